import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle  # test infrastructure (the checker)

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref (reference build) not available")
    return Reference()


@pytest.fixture(scope="session")
def g():
    """The product package; on a GPU test it must load the CUDA library."""
    import paper_2509_19821_b200 as pkg

    return pkg


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_close(a, b, rtol=1e-5):
    """|a - b| <= rtol * max(1, |b|) elementwise (the north-star fp32 contract)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= rtol * np.maximum(1.0, np.abs(b))


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


REF_PROBLEMS = ([f"LIRCMOP{i}" for i in range(1, 15)] +
                ["C1-DTLZ1", "C1-DTLZ3", "C2-DTLZ2", "C3-DTLZ4", "DC1-DTLZ1", "DC1-DTLZ3",
                 "DC2-DTLZ1", "DC2-DTLZ3", "DC3-DTLZ1", "DC3-DTLZ3"] +
                [f"WTA-P{i}" for i in range(1, 11)])
MW_PROBLEMS = [f"MW{i}" for i in range(1, 15)]
DAS_PROBLEMS = [f"DASCMOP{i}" for i in range(1, 10)]
