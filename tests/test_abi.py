"""Host-side checks of the C-ABI library (-m "not gpu"): it builds for sm_100a,
loads, exports every symbol include/nnls.h declares, carries real sm_100a
SASS with the FP64 tensor instruction, and fails loudly (no CPU fallback)
without a GPU."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import importlib
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_cs_0408029_b200"))
    import build as B  # noqa: E402
    B.build()
    sys.path.pop(0)
    import paper_cs_0408029_b200 as pkg
    return importlib.reload(pkg)


def test_exports_every_header_symbol(P):
    names = P.header_symbols()
    assert len(names) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only", P.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(P.lib, n)


def test_sass_is_sm100a_with_dmma(P):
    out = subprocess.check_output(["cuobjdump", "-sass", P.LIB_PATH]).decode(errors="replace")
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out          # FP64 tensor-core Cholesky update


def test_struct_layouts(P):
    assert ctypes.sizeof(P.Params) == 72
    assert ctypes.sizeof(P.Info) == 88
    assert ctypes.sizeof(P.IterRec) == 40
    p = P.default_params()
    assert p.zero_tol == 1e-12 and p.p_max == 3 and p.lsqr_mode == 1 and p.kkt == 1
    assert p.lsqr_atol == 1e-15 and p.lsqr_conlim == 1e8


def test_status_strings(P):
    for s in range(10):
        assert P.lib.nnls_status_string(s)


def test_no_cpu_fallback_without_gpu(P):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.NNLSError):
        P.Solver()
    with pytest.raises(P.NNLSError):
        P.device_info()


def test_product_never_imports_oracle():
    """The product package and the oracle share no code and never import each other."""
    pkg = os.path.join(ROOT, "paper_cs_0408029_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt
                assert "nnls_oracle" not in txt and "liboracle" not in txt
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_cs_0408029_b200" not in txt and "from paper_cs_0408029_b200" not in txt
            assert "#include \"../paper" not in txt and "common.cuh" not in txt


def test_invalid_args_rejected_before_device(P):
    # argument checks happen on the host before any device call
    st = P.lib.nnls_step_gram(0, 0, 0, None, None, None, None, None, 0, None, None)
    assert st == P.ERR_INVALID_ARG
    st = P.lib.nnls_step_dual(0, None, 0, None, None, None, None, 1e-12, None)
    assert st == P.ERR_INVALID_ARG
    h = ctypes.c_void_p()
    st = P.lib.nnls_setup(ctypes.byref(h), 3, 5, 0, None, None, None, None, None, None)
    assert st != P.OK and not h.value
