"""CPU: the C-ABI library exists, loads, exports every symbol include/*.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gmpea_b200.h")
LIB = os.path.join(ROOT, "paper_2509_19821_b200", "libgmpea_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gmpea_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_operator_surface():
    syms = declared_symbols()
    for s in ("gmpea_evaluate", "gmpea_reproduce", "gmpea_environmental_selection", "gmpea_build_neighborhoods",
              "gmpea_reference_vectors", "gmpea_igd", "gmpea_hypervolume", "gmpea_metric_front",
              "gmpea_engine_create", "gmpea_engine_run", "gmpea_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    import paper_2509_19821_b200 as g
    from paper_2509_19821_b200._lib import CudaError

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(CudaError):
        g.make_problem("LIRCMOP1")
    # host-only metadata still works
    assert "LIRCMOP13" in g.problem_names() and "MW7" in g.problem_names()


def test_unknown_problem_is_invalid_argument():
    import paper_2509_19821_b200 as g

    with pytest.raises(ValueError, match="unknown problem"):
        g.make_problem("NOPE1")
