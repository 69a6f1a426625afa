"""pytest plugin: run the reference's OWN test suite with this package's
kernel seam in place of trilab's numba backend.

    PYTHONPATH=baseline/_ref/pkg/src:. python -m pytest baseline/_ref/pkg/tests \\
        -p scripts.trilab_cuda_plugin

Every trilab entry point that resolves the "numba" backend (the default)
gets paper_1908_00741_b200.kernels: the 11 kernel functions, construction
kernels in the native host builder, SpMV / substitutions on the B200.  The
reference's cross-backend tests (T/test_backends.py) then compare this
backend against trilab's pure-numpy one bitwise.  Integration check only:
baseline/_ref is a git-ignored copy of the reference (never committed).
"""


def pytest_configure(config):
    import trilab._kernels as K

    import paper_1908_00741_b200.kernels as cuda
    K._BACKENDS["numba"] = cuda
    K._NUMBA_FAILED = False
