"""pytest plugin: run the reference's OWN tests against this package's public
API (whole-path drop-in check): `trilab` and its public submodules resolve
to paper_1908_00741_b200.

    PYTHONPATH=. python -m pytest baseline/_ref/pkg/tests/test_<x>.py \\
        -p scripts.trilab_alias_plugin

Files that exercise the reference's CLI, its backend registry or its
private helpers are out of this drop-in's scope.
Integration check only; baseline/_ref is a git-ignored copy of the reference.
"""

import sys

# at import time: `-p` plugins load before the reference's conftest.py
import paper_1908_00741_b200 as P  # noqa: E402
from paper_1908_00741_b200 import io, matrix, ordering, precond, solver  # noqa: E402

sys.modules["trilab"] = P
for _name, _mod in (("matrix", matrix), ("ordering", ordering), ("precond", precond),
                    ("solver", solver), ("io", io)):
    sys.modules[f"trilab.{_name}"] = _mod
