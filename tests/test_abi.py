"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and exports every
entry point include/polya.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "polya.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(polya_[A-Za-z_0-9]+)\s*\(", src)))


def test_library_builds_loads_and_exports_header_symbols():
    from paper_1411_3769_b200 import build as b
    lib_path = b.build()
    import paper_1411_3769_b200 as pb
    L = pb.lib()
    names = _declared()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(L, nm), nm
    assert set(pb.EXPORTS) <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}$", out, flags=re.M), nm


def test_sass_is_sm100a_and_uses_fp64_mma():
    from paper_1411_3769_b200 import build as b
    lib_path = b.build()
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out       # FP64 tensor-core MMA in the Schur / GEMM kernels


def test_invalid_arguments_are_rejected_without_a_gpu():
    import paper_1411_3769_b200 as pb
    L = pb.lib()
    h = ctypes.c_void_p()
    assert L.polya_setup(None, None, ctypes.byref(h)) == 1          # POLYA_EINVAL
    cfg = pb._Config(0, 2, 1, 1, 1, 1, 1e-3, 0, 1)                    # n = 0
    assert L.polya_setup(ctypes.byref(cfg), ctypes.c_void_p(1), ctypes.byref(h)) == 1
    cfg = pb._Config(4, 2, 1, 1, 1, 1, 0.0, 0, 1)                     # delta = 0
    assert L.polya_setup(ctypes.byref(cfg), ctypes.c_void_p(1), ctypes.byref(h)) == 1
    cfg = pb._Config(4, 2, 1, 1, 1, 1, 1e-3, 2, 2)                    # rank outside [0, nranks)
    assert L.polya_setup(ctypes.byref(cfg), ctypes.c_void_p(1), ctypes.byref(h)) == 1
    assert L.polya_strerror(2) == b"integer overflow in problem size"


def test_library_then_torch_import_order():
    """libpolya.so links the NCCL that PyTorch loads (rpath to the pip wheel), so loading the
    library BEFORE torch must not shadow torch's libnccl.so.2 with an older system copy."""
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1411_3769_b200 as pb; pb.lib(); "
            "import torch; import torch.distributed; print('ok')") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_setup_general_rejects_mixed_degrees_without_a_gpu():
    """polya_setup_general validates before touching the device: terms of different total degree
    (R18: one common degree cfg->da) are EINVAL."""
    import numpy as np
    import pytest
    import paper_1411_3769_b200 as pb
    n, l = 2, 2
    terms = [(np.zeros((2, n, n)), 1, np.zeros((2, n, n)), 1), (np.zeros((2, n, n)), 1, np.zeros((1, n, n)), 0)]
    with pytest.raises(pb.PolyaError, match="invalid argument"):
        pb.Polya.general(terms, n, l, 1, 1, 1)


def test_setup_general_rejects_lmi_order_below_n_without_a_gpu():
    """nlmi (the LMI order N) must be 0 (square) or >= n: EINVAL before any device call."""
    import ctypes

    import numpy as np
    import paper_1411_3769_b200 as pb
    L = pb.lib()
    cfg = pb._Config(3, 2, 1, 1, 1, 1, 1e-3, 0, 1, 0)
    At = np.zeros((2, 3, 3))
    Bt = np.zeros((1, 3, 3))
    da, db = np.array([1], dtype=np.int32), np.array([0], dtype=np.int32)
    h = ctypes.c_void_p()
    cp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.polya_setup_general(ctypes.byref(cfg), 2, 1, cp(da), cp(db), cp(At), cp(Bt), None, ctypes.byref(h))
    assert st == 1 and not h.value    # POLYA_EINVAL, no context
