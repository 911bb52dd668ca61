import os
import sys

# The oracle's many small dense solves (numpy / OpenBLAS) run fastest single-threaded; a BLAS
# thread pool per call oversubscribes the host cores (measured: the scaled-config oracle tests
# 93 s -> 59 s on 8 cores).  oracle_core.c's OpenMP loops are not affected.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running oracle case")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    return oracle.load_library()
