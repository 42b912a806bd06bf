"""Host-side checks of the C ABI (no GPU): the built libhobf.so loads and exports
every symbol include/hobf.h declares; the oracle library builds and loads; the
product binding refuses to run without the CUDA library (no CPU fallback)."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2007_06563_b200", "libhobf.so")
HEADER = os.path.join(ROOT, "include", "hobf.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hobf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["hobf_pack", "hobf_unpack", "hobf_conv2d", "hobf_mac_planes", "hobf_quantize_pack",
              "hobf_gate_count", "hobf_status_str"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libhobf.so not built")
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    lib.hobf_nbits.restype = ctypes.c_int32
    assert lib.hobf_nbits(5, 3) == 11
    lib.hobf_nplanes.restype = ctypes.c_int32
    assert lib.hobf_nplanes(11) == 12 and lib.hobf_nplanes(12) == 12 and lib.hobf_nplanes(13) == 16
    lib.hobf_planes_words.restype = ctypes.c_int64
    lib.hobf_planes_words.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
    assert lib.hobf_planes_words(10, 33, 11) == 10 * 2 * 12


def test_binding_symbols_match_header():
    if not os.path.exists(LIB):
        pytest.skip("libhobf.so not built")
    sys.path.insert(0, ROOT)
    from paper_2007_06563_b200 import hobf
    assert sorted(hobf.SYMBOLS) == declared_symbols()
    g = hobf.gate_count(hobf.Fmt(5, 3, 0))  # host-only call: no device work
    assert g["mac"] > 0 and g["add"] > g["relu"]


def test_argument_errors_are_synchronous_and_need_no_gpu():
    if not os.path.exists(LIB):
        pytest.skip("libhobf.so not built")
    sys.path.insert(0, ROOT)
    from paper_2007_06563_b200 import hobf
    lib = hobf._lib
    f = hobf.Fmt(5, 3).c()
    # negative sizes -> EINVAL, unsupported format -> EUNSUPPORTED, bad shapes -> ESHAPE
    assert lib.hobf_pack(5, 3, None, -1, 4, None, None) == 1
    assert lib.hobf_conv2d(hobf.Fmt(7, 3).c(), None, 1, 4, 4, 4, None, 3, 3, 4, 1, 1, 0, None, None) == 3
    assert lib.hobf_conv2d(f, None, 1, 2, 2, 4, None, 5, 5, 4, 1, 0, 0, None, None) == 2
    assert lib.hobf_conv2d(f, None, 1, 4, 4, 4, None, 3, 3, 4, 0, 1, 0, None, None) == 1
    assert lib.hobf_mac_planes(f, None, None, None, 5, None) == 1
    assert lib.hobf_status_str(3) == b"unsupported format (no generated kernel)"
    # chaining epilogue / schedule validation happens before any launch: fake (never
    # dereferenced) 16-byte-aligned pointers reach the checks without a GPU
    P = 1 << 20
    E = hobf.hobf_epilogue
    bad = [E(hobf.OUT_NEXT_RECORDS, 0, 1), E(hobf.OUT_NEXT_RECORDS, 3, -1), E(hobf.OUT_NEXT_RECORDS, 12, 1),
           E(hobf.OUT_NEXT_PLANES, 30, 0), E(7, 3, 1)]
    for ep in bad:
        assert lib.hobf_conv2d_prepared_ex(f, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, ep, P, 0, None) == 1
        assert lib.hobf_conv2d_dw(f, P, 1, 4, 4, 8, P, 3, 3, 1, 1, 0, ep, P, None) == 1
    assert lib.hobf_conv2d_ex(f, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, E(hobf.OUT_NEXT_RECORDS, 3, 1), P, None) == 1
    assert lib.hobf_conv2d_prepared_ex(f, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, E(0, 0, 0), P, 16, None) == 1
    assert lib.hobf_conv2d_prepared_ex(f, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, E(0, 0, 0), P, 9, None) == 1
    assert lib.hobf_conv2d_dw(f, P, 1, 2, 2, 8, P, 5, 5, 1, 0, 0, E(0, 0, 0), P, None) == 2
    # beyond the launch grid's limits -> ESHAPE (not a launch failure)
    big = 2 ** 31 - 1
    assert lib.hobf_conv2d_prepared_ex(f, P, 1, 4, 4, 4, P, 3, 3, 65536 * 32, 1, 1, 0, E(0, 0, 0), P, 0, None) == 2
    assert lib.hobf_conv2d_prepared_ex(f, P, big, 4096, 4096, 4, P, 3, 3, 32, 1, 1, 0, E(0, 0, 0), P, 0, None) == 2
    assert lib.hobf_conv2d_ex(f, P, big, 4096, 4096, 4, P, 3, 3, 32, 1, 1, 0, E(0, 0, 0), P, None) == 2
    assert lib.hobf_conv2d_dw(f, P, big, 4096, 4096, 32, P, 3, 3, 1, 1, 0, E(0, 0, 0), P, None) == 2
    # the float32 output epilogue needs we <= 7 (exact float32 values); a misaligned output is refused
    f83 = hobf.Fmt(8, 3).c()
    assert lib.hobf_conv2d_ex(f83, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, E(hobf.OUT_F32, 0, 0), P, None) in (1, 3)
    assert lib.hobf_conv2d_ex(f, P, 1, 4, 4, 4, P, 3, 3, 8, 1, 1, 0, E(hobf.OUT_F32, 0, 0), P + 4, None) == 1
    # the kernel-info query checks its arguments like the conv calls
    info = hobf.hobf_kernel_info()
    assert lib.hobf_conv_kernel_info(3, f, 1, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 0, ctypes.byref(info)) == 1
    assert lib.hobf_conv_kernel_info(1, f, 1, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 0, None) == 1
    assert lib.hobf_conv_kernel_info(1, f, 1, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 16, ctypes.byref(info)) == 1
    assert lib.hobf_conv_kernel_info(0, f, 1, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 4, ctypes.byref(info)) == 1
    assert lib.hobf_conv_kernel_info(1, f, 1, 2, 2, 4, 5, 5, 8, 1, 0, E(0, 0, 0), 0, ctypes.byref(info)) == 2
    assert lib.hobf_conv_kernel_info(1, hobf.Fmt(7, 3).c(), 1, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 0,
                                     ctypes.byref(info)) == 3
    assert lib.hobf_conv_kernel_info(1, f, 0, 4, 4, 4, 3, 3, 8, 1, 1, E(0, 0, 0), 0, ctypes.byref(info)) == 0
    assert info.name == b""


def test_binding_fails_loudly_without_library(tmp_path):
    """Copy the binding next to no .so: importing must raise, not fall back."""
    pkg = tmp_path / "paper_2007_06563_b200"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "hobf.py").write_text(open(os.path.join(ROOT, "paper_2007_06563_b200", "hobf.py")).read())
    r = subprocess.run([sys.executable, "-c", "import paper_2007_06563_b200.hobf"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "libhobf.so is missing" in r.stderr


def test_oracle_is_independent_of_the_cuda_path():
    """The oracle shares no code with the product path and vice versa."""
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2007_06563_b200")):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in src and "from oracle" not in src and "hobf_ref" not in src, fn
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith((".py", ".c", ".h")):
            src = open(os.path.join(ROOT, "oracle", fn)).read()
            assert "import paper_2007_06563_b200" not in src and "from paper_2007_06563_b200" not in src, fn
