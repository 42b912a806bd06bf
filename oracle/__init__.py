"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/hobf_ref.c``: the plain scalar CPU emulation of the
HOBFLOPS format and MAC (arXiv 2007.06563) that the CUDA path is checked
against.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares
no code with ``paper_2007_06563_b200`` and never imports it.

Functions take and return numpy arrays of uint32 words; formats are (we, wf)
pairs and ``mode`` is 0 = RNE, 1 = RTZ (ledger L3/L4 in hobf_ref.c).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhobf_ref.so")
_lib = None

RNE = 0
RTZ = 1


def build(force: bool = False) -> str:
    """Compile hobf_ref.c with gcc (plain C, -O2)."""
    src = os.path.join(_HERE, "hobf_ref.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "libhobf_ref.so"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u32, i32, i64 = ctypes.c_uint32, ctypes.c_int, ctypes.c_int64
        P = ctypes.c_void_p
        L.ref_mul.restype = u32
        L.ref_mul.argtypes = [u32, u32, i32, i32, i32, i32]
        L.ref_add.restype = u32
        L.ref_add.argtypes = [u32, u32, i32, i32, i32]
        L.ref_relu.restype = u32
        L.ref_relu.argtypes = [u32, i32, i32]
        L.ref_canon.restype = u32
        L.ref_canon.argtypes = [u32, i32, i32]
        L.ref_encode_f32.restype = u32
        L.ref_encode_f32.argtypes = [ctypes.c_float, i32, i32, i32]
        L.ref_decode_f64.restype = ctypes.c_double
        L.ref_decode_f64.argtypes = [u32, i32, i32]
        L.ref_nbits.restype = i32
        L.ref_nbits.argtypes = [i32, i32]
        L.ref_mul_batch.argtypes = [P, P, P, i64, i32, i32, i32, i32]
        L.ref_add_batch.argtypes = [P, P, P, i64, i32, i32, i32]
        L.ref_relu_batch.argtypes = [P, P, i64, i32, i32]
        L.ref_canon_batch.argtypes = [P, P, i64, i32, i32]
        L.ref_encode_f32_batch.argtypes = [P, P, i64, i32, i32, i32]
        L.ref_convert_batch.argtypes = [P, P, i64, i32, i32, i32, i32]
        L.ref_decode_f64_batch.argtypes = [P, P, i64, i32, i32]
        L.ref_mac_batch.argtypes = [P, P, P, i64, i32, i32, i32, i32]
        L.ref_conv2d.restype = i32
        L.ref_conv2d.argtypes = [P, i32, i32, i32, i32, P, i32, i32, i32,
                                 i32, i32, i32, i32, i32, i32, i32, P, i32]
        L.ref_conv2d_dw.restype = i32
        L.ref_conv2d_dw.argtypes = [P, i32, i32, i32, i32, P, i32, i32, i32, i32, i32, i32, i32, i32, i32, P, i32]
        L.ref_conv2d_sample.restype = i32
        L.ref_conv2d_sample.argtypes = [P, i32, i32, i32, i32, P, i32, i32, i32,
                                        i32, i32, i32, i32, i32, i32, i32, P, i64, P]
        _lib = L
    return _lib


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def nbits(we: int, wf: int) -> int:
    return lib().ref_nbits(we, wf)


def mul(a, b, we, wf, wf_out, mode=RNE) -> np.ndarray:
    a, b = np.broadcast_arrays(_u32(a), _u32(b))
    a, b = _u32(a), _u32(b)
    out = np.empty(a.shape, np.uint32)
    lib().ref_mul_batch(_ptr(a), _ptr(b), _ptr(out), a.size, we, wf, wf_out, mode)
    return out


def add(a, b, we, wf, mode=RNE) -> np.ndarray:
    a, b = np.broadcast_arrays(_u32(a), _u32(b))
    a, b = _u32(a), _u32(b)
    out = np.empty(a.shape, np.uint32)
    lib().ref_add_batch(_ptr(a), _ptr(b), _ptr(out), a.size, we, wf, mode)
    return out


def mac(acc, a, b, we, wf, wf_out, mode=RNE) -> np.ndarray:
    acc, a, b = np.broadcast_arrays(_u32(acc), _u32(a), _u32(b))
    acc, a, b = _u32(acc).copy(), _u32(a), _u32(b)
    lib().ref_mac_batch(_ptr(acc), _ptr(a), _ptr(b), acc.size, we, wf, wf_out, mode)
    return acc


def relu(a, we, wf) -> np.ndarray:
    a = _u32(a)
    out = np.empty(a.shape, np.uint32)
    lib().ref_relu_batch(_ptr(a), _ptr(out), a.size, we, wf)
    return out


def canon(a, we, wf) -> np.ndarray:
    a = _u32(a)
    out = np.empty(a.shape, np.uint32)
    lib().ref_canon_batch(_ptr(a), _ptr(out), a.size, we, wf)
    return out


def convert(a, we, wf_in, wf_out, mode=RNE) -> np.ndarray:
    """Re-round F(we, wf_in) words into F(we, wf_out) (ref_convert: the layer
    epilogue of a chained network)."""
    a = _u32(a)
    out = np.empty_like(a)
    lib().ref_convert_batch(_ptr(a), _ptr(out), a.size, we, wf_in, wf_out, mode)
    return out


def conv_chain(x, layers, we, mode=RNE, nthreads=None) -> np.ndarray:
    """A chain of conv layers in the custom format: x = F(we, wf0) NHWC
    words; layers = [(w_words, wf, stride, pad, relu, extended), ...] where wf is
    that layer's input fraction width.  Each layer: conv2d at its MAC width,
    then (except after the last) convert to the next layer's wf.  Returns the
    last layer's accumulator-format words."""
    y = x
    for i, (wts, wf, stride, pad, relu, ext) in enumerate(layers):
        wf_out = 2 * wf + 1 if ext else wf + 1
        y = conv2d(y, wts, we, wf, wf_out, mode, stride, pad, relu, nthreads)
        if i + 1 < len(layers):
            y = convert(y, we, wf_out, layers[i + 1][1], mode)
    return y


def encode_f32(x, we, wf, mode=RNE) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    out = np.empty(x.shape, np.uint32)
    lib().ref_encode_f32_batch(_ptr(x), _ptr(out), x.size, we, wf, mode)
    return out


def decode_f64(w, we, wf) -> np.ndarray:
    w = _u32(w)
    out = np.empty(w.shape, np.float64)
    lib().ref_decode_f64_batch(_ptr(w), _ptr(out), w.size, we, wf)
    return out


def conv_out_hw(h, w, kh, kw, stride, pad):
    return (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1


def conv2d(x, wts, we, wf, wf_out, mode=RNE, stride=1, pad=1, relu=0, nthreads=None) -> np.ndarray:
    """x: [n,h,w,cin] words; wts: [kh,kw,cin,cout] words -> [n,ho,wo,cout] words in F(we, wf_out)."""
    x, wts = _u32(x), _u32(wts)
    n, h, w, cin = x.shape
    kh, kw, cin2, cout = wts.shape
    assert cin2 == cin
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    y = np.empty((n, ho, wo, cout), np.uint32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib().ref_conv2d(_ptr(x), n, h, w, cin, _ptr(wts), kh, kw, cout,
                          stride, pad, int(relu), we, wf, wf_out, mode, _ptr(y), int(nthreads))
    if rc != 0:
        raise ValueError("ref_conv2d: bad arguments")
    return y


def conv2d_dw(x, wts, we, wf, wf_out, mode=RNE, stride=1, pad=1, relu=0, nthreads=None) -> np.ndarray:
    """Depthwise conv (ref_conv2d_dw): x [n,h,w,c] words, wts [kh,kw,c] words ->
    [n,ho,wo,c] words in F(we, wf_out)."""
    x, wts = _u32(x), _u32(wts)
    n, h, w, c = x.shape
    kh, kw, c2 = wts.shape
    assert c2 == c
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    y = np.empty((n, ho, wo, c), dtype=np.uint32)
    nt = nthreads or os.cpu_count() or 1
    rc = lib().ref_conv2d_dw(_ptr(x), n, h, w, c, _ptr(wts), kh, kw, stride, pad, relu, we, wf, wf_out, mode,
                             _ptr(y), nt)
    assert rc == 0
    return y


def conv2d_sample(x, wts, idx, we, wf, wf_out, mode=RNE, stride=1, pad=1, relu=0) -> np.ndarray:
    """Outputs at flat indices idx of the [n,ho,wo,cout] result (single thread)."""
    x, wts = _u32(x), _u32(wts)
    n, h, w, cin = x.shape
    kh, kw, _, cout = wts.shape
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    y = np.empty(idx.shape, np.uint32)
    rc = lib().ref_conv2d_sample(_ptr(x), n, h, w, cin, _ptr(wts), kh, kw, cout,
                                 stride, pad, int(relu), we, wf, wf_out, mode, _ptr(idx), idx.size, _ptr(y))
    if rc != 0:
        raise ValueError("ref_conv2d_sample: bad arguments")
    return y
