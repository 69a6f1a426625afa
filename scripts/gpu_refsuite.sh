#!/bin/bash
# The reference's own tests (baseline/_ref/pkg/tests, a git-ignored copy of
# the reference) against this package's public API on the B200
# (scripts/trilab_alias_plugin.py).  Out of scope: test_backends (numba /
# numpy registry), test_cli (the CLI).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
out=${1:-gpurun_out/refsuite.txt}
: > "$out"
for t in test_matrix test_ordering test_precond test_solver test_io test_properties test_acceptance; do
  echo "== $t" >> "$out"
  PYTHONPATH=. timeout 900 python -m pytest baseline/_ref/pkg/tests/$t.py -q -p scripts.trilab_alias_plugin \
      -p no:cacheprovider 2>&1 | tail -4 >> "$out"
done
cat "$out"
