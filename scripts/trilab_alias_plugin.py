"""pytest plugin: run the reference's OWN tests against this package's public
API (whole-path drop-in check): `trilab` and its public submodules resolve
to paper_1908_00741_b200.

    PYTHONPATH=. python -m pytest baseline/_ref/pkg/tests/test_<x>.py \\
        -p scripts.trilab_alias_plugin

Files that exercise the reference's CLI, its backend registry or its
private helpers are out of this drop-in's scope.  The
ordering / IC verifiers (src/ordering.py:283-346, src/precond.py:203-260) are
out of scope too: the plugin imports the reference's own and
exposes them next to this package's names, so its tests check this
package's orderings and factors with the reference's checkers.
Integration check only; baseline/_ref is a git-ignored copy of the reference.
"""

import os
import sys

# the reference's verifiers, imported before `trilab` is aliased
_REF_SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "baseline", "_ref", "pkg", "src")
sys.path.insert(0, _REF_SRC)
import trilab as _ref  # noqa: E402
import trilab.ordering as _ref_ordering  # noqa: E402
import trilab.precond as _ref_precond  # noqa: E402
import trilab._kernels.numba_backend  # noqa: E402,F401  (the verifiers' kernels)
sys.path.remove(_REF_SRC)
# the reference's kernel package keeps its name (this package has none): the
# verifiers import their kernels lazily from it
for _k in [k for k in sys.modules if (k == "trilab" or k.startswith("trilab."))
           and not k.startswith("trilab._kernels")]:
    sys.modules["_trilab_ref" + _k[len("trilab"):]] = sys.modules.pop(_k)

# at import time: `-p` plugins load before the reference's conftest.py
import paper_1908_00741_b200 as P  # noqa: E402
from paper_1908_00741_b200 import io, matrix, ordering, precond, solver  # noqa: E402

sys.modules["trilab"] = P
for _name, _mod in (("matrix", matrix), ("ordering", ordering), ("precond", precond),
                    ("solver", solver), ("io", io)):
    sys.modules[f"trilab.{_name}"] = _mod

_VERIFIERS = {
    ordering: ("OrderingGraph", "ErReport", "Level2Report", "build_ordering_graph",
               "check_er_condition", "check_level2_structure"),
    precond: ("ic_residual_on_pattern", "factor_equivalence_check"),
}
for _mod, _names in _VERIFIERS.items():
    _src = _ref_ordering if _mod is ordering else _ref_precond
    for _n in _names:
        setattr(_mod, _n, getattr(_src, _n))
        setattr(P, _n, getattr(_src, _n))
