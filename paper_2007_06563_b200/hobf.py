"""Thin Python binding of the C ABI in ``include/hobf.h`` (``libhobf.so``).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  Tensors are torch CUDA tensors; bit patterns are
carried in ``torch.int32`` tensors (same bits as the ABI's uint32).  There is
no CPU fallback: if the shared library is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhobf.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or `make -C paper_2007_06563_b200/csrc -j`)")

_lib = ctypes.CDLL(LIB_PATH)

RNE = 0
RTZ = 1

STATUS = {0: "ok", 1: "invalid argument", 2: "inconsistent shapes", 3: "unsupported format", 4: "CUDA launch error"}


class HobfError(RuntimeError):
    def __init__(self, fn, status):
        super().__init__(f"{fn}: {STATUS.get(status, status)} (status {status})")
        self.status = status


class hobf_fmt(ctypes.Structure):
    _fields_ = [("we", ctypes.c_int32), ("wf", ctypes.c_int32), ("round", ctypes.c_int32), ("extended", ctypes.c_int32)]


class hobf_epilogue(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("next_wf", ctypes.c_int32), ("next_pad", ctypes.c_int32)]


OUT_PLANES, OUT_NEXT_PLANES, OUT_NEXT_RECORDS, OUT_F32 = 0, 1, 2, 3


@dataclass(frozen=True)
class Next:
    """Layer-chaining epilogue (hobf_epilogue): write the output re-rounded into the
    next layer's F(we, wf) as planes (records=False, for hobf_conv2d) or as
    activation records padded by `pad` (records=True, for hobf_conv2d_prepared)."""
    wf: int
    records: bool = True
    pad: int = 1

    def c(self) -> hobf_epilogue:
        return hobf_epilogue(OUT_NEXT_RECORDS if self.records else OUT_NEXT_PLANES, self.wf, self.pad)


@dataclass(frozen=True)
class Float32Out:
    """Last-layer epilogue (HOBF_OUT_F32): the conv writes its outputs as exact
    float32 NHWC [n*ho*wo, cout] instead of planes (no unpack pass)."""
    records = False

    def c(self) -> hobf_epilogue:
        return hobf_epilogue(OUT_F32, 0, 0)


F32 = Float32Out()


@dataclass(frozen=True)
class Fmt:
    """Input format F(we, wf) plus MAC mode (round: 0 RNE / 1 RTZ; extended: 0 single)."""
    we: int
    wf: int
    round: int = RNE
    extended: int = 0

    def c(self) -> hobf_fmt:
        return hobf_fmt(self.we, self.wf, self.round, self.extended)

    @property
    def nin(self) -> int:
        return 3 + self.we + self.wf

    @property
    def wfo(self) -> int:
        return 2 * self.wf + 1 if self.extended else self.wf + 1

    @property
    def nout(self) -> int:
        return 3 + self.we + self.wfo


_i32, _i64, _p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
_lib.hobf_nbits.restype = _i32
_lib.hobf_nbits.argtypes = [_i32, _i32]
_lib.hobf_out_wf.restype = _i32
_lib.hobf_out_wf.argtypes = [hobf_fmt]
_lib.hobf_nplanes.restype = _i32
_lib.hobf_nplanes.argtypes = [_i32]
_lib.hobf_planes_words.restype = _i64
_lib.hobf_planes_words.argtypes = [_i64, _i64, _i32]
for _name in ("hobf_pack", "hobf_unpack"):
    getattr(_lib, _name).restype = _i32
    getattr(_lib, _name).argtypes = [_i32, _i32, _p, _i64, _i64, _p, _p]
_lib.hobf_quantize_pack.restype = _i32
_lib.hobf_quantize_pack.argtypes = [_i32, _i32, _i32, _p, _i64, _i64, _p, _p]
_lib.hobf_unpack_f32.restype = _i32
_lib.hobf_unpack_f32.argtypes = [_i32, _i32, _p, _i64, _i64, _p, _p]
_lib.hobf_conv2d.restype = _i32
_lib.hobf_conv2d.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32, _i32, _p, _p]
_lib.hobf_mac_planes.restype = _i32
_lib.hobf_mac_planes.argtypes = [hobf_fmt, _p, _p, _p, _i64, _p]
_lib.hobf_gate_count.restype = _i32
_lib.hobf_gate_count.argtypes = [hobf_fmt] + [ctypes.POINTER(_i32)] * 5
_lib.hobf_wtab_words.restype = _i64
_lib.hobf_wtab_words.argtypes = [hobf_fmt, _i32, _i32, _i32, _i32]
_lib.hobf_prepare_weights.restype = _i32
_lib.hobf_prepare_weights.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _p]
_lib.hobf_conv2d_prepared.restype = _i32
_lib.hobf_conv2d_prepared.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32, _i32,
                                      _p, _p]
_lib.hobf_conv2d_prepared_ex.restype = _i32
_lib.hobf_conv2d_prepared_ex.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32,
                                         _i32, hobf_epilogue, _p, _i32, _p]
_lib.hobf_conv2d_dw.restype = _i32
_lib.hobf_conv2d_dw.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32, hobf_epilogue,
                                _p, _p]
_lib.hobf_conv2d_ex.restype = _i32
_lib.hobf_conv2d_ex.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _p, _i32, _i32, _i32, _i32, _i32, _i32,
                                hobf_epilogue, _p, _p]
_lib.hobf_xrec_words.restype = _i64
_lib.hobf_xrec_words.argtypes = [_i32, _i32, _i32, _i32, _i32]
_lib.hobf_prepare_activations.restype = _i32
_lib.hobf_prepare_activations.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _i32, _p, _p]
_lib.hobf_quantize_activations.restype = _i32
_lib.hobf_quantize_activations.argtypes = [hobf_fmt, _p, _i32, _i32, _i32, _i32, _i32, _p, _p]
class hobf_kernel_info(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 256), ("variant", _i32), ("threads", _i32), ("dyn_smem", _i32),
                ("static_smem", _i32), ("regs", _i32), ("local_bytes", _i32), ("ctas_per_sm", _i32),
                ("blocks", _i64)]


_lib.hobf_conv_kernel_info.restype = _i32
_lib.hobf_conv_kernel_info.argtypes = [_i32, hobf_fmt, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                       hobf_epilogue, _i32, ctypes.POINTER(hobf_kernel_info)]
_lib.hobf_lop3_peak.restype = _i32
_lib.hobf_lop3_peak.argtypes = [_i32, _i32, _i32, _p, _p, ctypes.POINTER(_i64)]
_lib.hobf_last_launch_count.restype = _i32
_lib.hobf_status_str.restype = ctypes.c_char_p
_lib.hobf_status_str.argtypes = [_i32]
_lib.hobf_version.restype = ctypes.c_char_p

SYMBOLS = ["hobf_nbits", "hobf_out_wf", "hobf_nplanes", "hobf_planes_words", "hobf_pack", "hobf_quantize_pack",
           "hobf_unpack", "hobf_unpack_f32", "hobf_conv2d", "hobf_mac_planes", "hobf_gate_count",
           "hobf_lop3_peak", "hobf_last_launch_count", "hobf_status_str", "hobf_version",
           "hobf_wtab_words", "hobf_prepare_weights", "hobf_conv2d_prepared", "hobf_conv2d_prepared_ex", "hobf_conv2d_ex", "hobf_conv2d_dw", "hobf_xrec_words",
           "hobf_prepare_activations", "hobf_quantize_activations", "hobf_conv_kernel_info"]


def _check(fn, st):
    if st != 0:
        raise HobfError(fn, st)


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def nbits(we: int, wf: int) -> int:
    return _lib.hobf_nbits(we, wf)


def nplanes(nb: int) -> int:
    return _lib.hobf_nplanes(nb)


def planes_words(rows: int, c: int, nb: int) -> int:
    return _lib.hobf_planes_words(rows, c, nb)


def planes_shape(rows: int, c: int, nb: int):
    return (rows, (c + 31) // 32, nplanes(nb))


def last_launch_count() -> int:
    return _lib.hobf_last_launch_count()


def version() -> str:
    return _lib.hobf_version().decode()


def _new_planes(rows, c, nb, device, out=None):
    shape = planes_shape(rows, c, nb)
    if out is None:
        return torch.empty(shape, dtype=torch.int32, device=device)
    assert out.numel() == shape[0] * shape[1] * shape[2] and out.dtype == torch.int32
    return out


def pack(we: int, wf: int, words: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """words [rows, c] (int32 bit patterns, CUDA) -> planes [rows, ceil(c/32), NP]."""
    assert words.is_cuda and words.dtype == torch.int32 and words.is_contiguous()
    rows, c = words.shape
    out = _new_planes(rows, c, nbits(we, wf), words.device, out)
    _check("hobf_pack", _lib.hobf_pack(we, wf, _ptr(words), rows, c, _ptr(out), _stream(stream)))
    return out


def quantize_pack(we: int, wf: int, x: torch.Tensor, rnd: int = RNE, out=None, stream=None) -> torch.Tensor:
    """float32 [rows, c] (CUDA) -> planes in F(we, wf), quantised with rnd."""
    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
    rows, c = x.shape
    out = _new_planes(rows, c, nbits(we, wf), x.device, out)
    _check("hobf_quantize_pack", _lib.hobf_quantize_pack(we, wf, rnd, _ptr(x), rows, c, _ptr(out), _stream(stream)))
    return out


def unpack(we: int, wf: int, planes: torch.Tensor, rows: int, c: int, out=None, stream=None) -> torch.Tensor:
    assert planes.is_cuda and planes.dtype == torch.int32 and planes.is_contiguous()
    if out is None:
        out = torch.empty((rows, c), dtype=torch.int32, device=planes.device)
    _check("hobf_unpack", _lib.hobf_unpack(we, wf, _ptr(planes), rows, c, _ptr(out), _stream(stream)))
    return out


def unpack_f32(we: int, wf: int, planes: torch.Tensor, rows: int, c: int, out=None, stream=None) -> torch.Tensor:
    assert planes.is_cuda and planes.dtype == torch.int32 and planes.is_contiguous()
    if out is None:
        out = torch.empty((rows, c), dtype=torch.float32, device=planes.device)
    _check("hobf_unpack_f32", _lib.hobf_unpack_f32(we, wf, _ptr(planes), rows, c, _ptr(out), _stream(stream)))
    return out


def conv_out_hw(h, w, kh, kw, stride, pad):
    return (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1


def _next_out(f: Fmt, nxt, n, ho, wo, cout, device, out):
    """Output buffer of a conv with epilogue `nxt` (None = plain output planes)."""
    if nxt is None:
        return _new_planes(max(n * ho * wo, 0), cout, f.nout, device, out)
    if isinstance(nxt, Float32Out):
        if out is None:
            out = torch.empty((max(n * ho * wo, 0), cout), dtype=torch.float32, device=device)
        return out
    if not nxt.records:
        return _new_planes(max(n * ho * wo, 0), cout, nbits(f.we, nxt.wf), device, out)
    if out is None:  # the +0 border of the next layer's records: (2^wf) << 20
        out = torch.full((max(xrec_words(n, ho, wo, cout, nxt.pad), 4),), ((1 << nxt.wf) << 20),
                         dtype=torch.int32, device=device)
    return out


def conv2d(f: Fmt, x_planes: torch.Tensor, n: int, h: int, w: int, cin: int, w_planes: torch.Tensor,
           kh: int, kw: int, cout: int, stride: int = 1, pad: int = 1, relu: int = 0, out=None,
           stream=None, nxt: "Next | None" = None) -> torch.Tensor:
    """HOBFLOPS conv on planes; returns output planes [n*ho*wo, ceil(cout/32), NP(NOUT)],
    or with nxt = Next(wf, records=False) the next layer's input planes of F(we, wf)
    (hobf_conv2d_ex, fused re-rounding epilogue), or with nxt = F32 the exact float32
    outputs [n*ho*wo, cout] (HOBF_OUT_F32)."""
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    out = _next_out(f, nxt, n, ho, wo, cout, x_planes.device, out)
    if nxt is None:
        _check("hobf_conv2d", _lib.hobf_conv2d(f.c(), _ptr(x_planes), n, h, w, cin, _ptr(w_planes), kh, kw, cout,
                                               stride, pad, int(relu), _ptr(out), _stream(stream)))
    else:
        _check("hobf_conv2d_ex", _lib.hobf_conv2d_ex(f.c(), _ptr(x_planes), n, h, w, cin, _ptr(w_planes), kh, kw,
                                                     cout, stride, pad, int(relu), nxt.c(), _ptr(out),
                                                     _stream(stream)))
    return out


def conv2d_dw(f: Fmt, x_planes: torch.Tensor, n: int, h: int, w: int, c: int, w_planes: torch.Tensor,
              kh: int, kw: int, stride: int = 1, pad: int = 1, relu: int = 0, out=None, stream=None,
              nxt: "Next | None" = None) -> torch.Tensor:
    """Depthwise conv (hobf_conv2d_dw): x planes [n*h*w, G, NP], w planes of the
    [kh][kw][c] words -> output planes (or the next layer's planes / records, nxt)."""
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    out = _next_out(f, nxt, n, ho, wo, c, x_planes.device, out)
    ep = nxt.c() if nxt is not None else hobf_epilogue(OUT_PLANES, 0, 0)
    _check("hobf_conv2d_dw", _lib.hobf_conv2d_dw(f.c(), _ptr(x_planes), n, h, w, c, _ptr(w_planes), kh, kw, stride,
                                                 pad, int(relu), ep, _ptr(out), _stream(stream)))
    return out


def mac_planes(f: Fmt, acc: torch.Tensor, a: torch.Tensor, b: torch.Tensor, stream=None) -> torch.Tensor:
    """In place: acc = add(acc, mul(a, b)) lane-wise. acc [G, NP(NOUT)], a/b [G, NP(NIN)]."""
    n = acc.shape[0]
    assert a.shape[0] == n and b.shape[0] == n
    _check("hobf_mac_planes", _lib.hobf_mac_planes(f.c(), _ptr(acc), _ptr(a), _ptr(b), n, _stream(stream)))
    return acc


def gate_count(f: Fmt) -> dict:
    v = [_i32() for _ in range(5)]
    _check("hobf_gate_count", _lib.hobf_gate_count(f.c(), *[ctypes.byref(x) for x in v]))
    return {"mac": v[0].value, "mul": v[1].value, "add": v[2].value, "relu": v[3].value, "mac_tab": v[4].value}


def wtab_words(f: Fmt, kh: int, kw: int, cin: int, cout: int) -> int:
    """Size of the prepared-weight table in words, or -1 if the format has no table kernel."""
    return _lib.hobf_wtab_words(f.c(), kh, kw, cin, cout)


def prepare_weights(f: Fmt, w_planes: torch.Tensor, kh: int, kw: int, cin: int, cout: int, out=None,
                    stream=None) -> torch.Tensor:
    n = wtab_words(f, kh, kw, cin, cout)
    if n < 0:
        raise HobfError("hobf_wtab_words", 3)
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=w_planes.device)
    _check("hobf_prepare_weights", _lib.hobf_prepare_weights(f.c(), _ptr(w_planes), kh, kw, cin, cout, _ptr(out),
                                                             _stream(stream)))
    return out


def xrec_words(n: int, h: int, w: int, cin: int, pad: int) -> int:
    return _lib.hobf_xrec_words(n, h, w, cin, pad)


def prepare_activations(f: Fmt, x_planes: torch.Tensor, n: int, h: int, w: int, cin: int, pad: int, out=None,
                        stream=None) -> torch.Tensor:
    """Activation planes -> zero-padded [n][cin][h+2pad][w+2pad] records for conv2d_prepared."""
    if out is None:
        out = torch.empty(max(xrec_words(n, h, w, cin, pad), 1), dtype=torch.int32, device=x_planes.device)
    _check("hobf_prepare_activations", _lib.hobf_prepare_activations(f.c(), _ptr(x_planes), n, h, w, cin, pad,
                                                                     _ptr(out), _stream(stream)))
    return out


def quantize_activations(f: Fmt, x: torch.Tensor, pad: int, out=None, stream=None) -> torch.Tensor:
    """float32 NHWC [n,h,w,cin] (CUDA) -> records for conv2d_prepared, quantised with f.round."""
    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 4
    n, h, w, cin = x.shape
    if out is None:
        out = torch.empty(max(xrec_words(n, h, w, cin, pad), 1), dtype=torch.int32, device=x.device)
    _check("hobf_quantize_activations", _lib.hobf_quantize_activations(f.c(), _ptr(x), n, h, w, cin, pad, _ptr(out),
                                                                       _stream(stream)))
    return out


def conv2d_prepared(f: Fmt, xrec: torch.Tensor, n: int, h: int, w: int, cin: int, wtab: torch.Tensor,
                    kh: int, kw: int, cout: int, stride: int = 1, pad: int = 1, relu: int = 0, out=None,
                    stream=None, variant: int | None = None, nxt: "Next | None" = None) -> torch.Tensor:
    """Conv on prepared activations (same pad) and prepared weights -> output planes.
    variant: None = automatic kernel schedule, else that schedule (identical results);
    nxt: Next(wf, records=True, pad) writes the next layer's activation records
    (or planes) of F(we, wf) instead (hobf_conv2d_prepared_ex, fused re-rounding);
    nxt = F32 writes the exact float32 outputs [n*ho*wo, cout] (HOBF_OUT_F32)."""
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    out = _next_out(f, nxt, n, ho, wo, cout, xrec.device, out)
    if variant is None and nxt is None:
        _check("hobf_conv2d_prepared", _lib.hobf_conv2d_prepared(f.c(), _ptr(xrec), n, h, w, cin, _ptr(wtab), kh, kw,
                                                                 cout, stride, pad, int(relu), _ptr(out),
                                                                 _stream(stream)))
    else:
        ep = nxt.c() if nxt is not None else hobf_epilogue(OUT_PLANES, 0, 0)
        _check("hobf_conv2d_prepared_ex",
               _lib.hobf_conv2d_prepared_ex(f.c(), _ptr(xrec), n, h, w, cin, _ptr(wtab), kh, kw, cout, stride,
                                            pad, int(relu), ep, _ptr(out), int(variant or 0), _stream(stream)))
    return out


OP_CONV, OP_PREPARED, OP_DW = 0, 1, 2


def conv_kernel_info(op: int, f: Fmt, n: int, h: int, w: int, cin: int, kh: int, kw: int, cout: int,
                     stride: int = 1, pad: int = 1, nxt=None, variant: int = 0) -> dict:
    """The kernel (symbol, schedule, CTA shape, registers, spills, CTAs per SM) that the
    conv call with these arguments launches (hobf_conv_kernel_info; nothing is launched)."""
    info = hobf_kernel_info()
    ep = nxt.c() if nxt is not None else hobf_epilogue(OUT_PLANES, 0, 0)
    _check("hobf_conv_kernel_info", _lib.hobf_conv_kernel_info(op, f.c(), n, h, w, cin, kh, kw, cout, stride, pad, ep,
                                                               variant, ctypes.byref(info)))
    return {"name": info.name.decode(), "variant": info.variant, "threads": info.threads,
            "dyn_smem": info.dyn_smem, "static_smem": info.static_smem, "regs": info.regs,
            "local_bytes": info.local_bytes, "ctas_per_sm": info.ctas_per_sm, "blocks": info.blocks}


def lop3_peak(blocks: int, threads: int, iters: int, sink: torch.Tensor, stream=None) -> int:
    n = _i64()
    _check("hobf_lop3_peak", _lib.hobf_lop3_peak(blocks, threads, iters, _ptr(sink), _stream(stream), ctypes.byref(n)))
    return n.value


class Conv2d:
    """User-level HOBFLOPS convolution layer (the public API a user calls).

    Weights are quantised and bitsliced once at construction (the paper keeps
    kernels pre-transformed); ``__call__`` quantises + packs the float32
    NHWC input, runs the bitsliced conv and unpacks the NHWC float32 output
    (exact in float32), all in CUDA kernels."""

    def __init__(self, weight_f32: torch.Tensor, f: Fmt, stride: int = 1, pad: int = 1, relu: bool = False,
                 use_tables: bool = True):
        kh, kw, cin, cout = weight_f32.shape
        if not weight_f32.is_cuda:  # marshalling: the library works on device memory
            weight_f32 = weight_f32.to("cuda")
        weight_f32 = weight_f32.to(torch.float32)
        self.f, self.kh, self.kw, self.cin, self.cout = f, kh, kw, cin, cout
        self.stride, self.pad, self.relu = stride, pad, relu
        self.w_planes = quantize_pack(f.we, f.wf, weight_f32.reshape(kh * kw * cin, cout).contiguous(), f.round)
        self.wtab = None
        if use_tables and wtab_words(f, kh, kw, cin, cout) > 0:
            self.wtab = prepare_weights(f, self.w_planes, kh, kw, cin, cout)

    def forward_planes(self, x_planes, n, h, w, out=None, stream=None):
        if self.wtab is not None:
            xrec = prepare_activations(self.f, x_planes, n, h, w, self.cin, self.pad, stream=stream)
            return conv2d_prepared(self.f, xrec, n, h, w, self.cin, self.wtab, self.kh, self.kw, self.cout,
                                   self.stride, self.pad, int(self.relu), out=out, stream=stream)
        return conv2d(self.f, x_planes, n, h, w, self.cin, self.w_planes, self.kh, self.kw, self.cout,
                      self.stride, self.pad, int(self.relu), out=out, stream=stream)

    def __call__(self, x_f32: torch.Tensor) -> torch.Tensor:
        n, h, w, cin = x_f32.shape
        assert cin == self.cin
        if not x_f32.is_cuda:
            x_f32 = x_f32.to(self.w_planes.device)
        x_f32 = x_f32.to(torch.float32)
        # the conv's float32 epilogue writes the NHWC output directly (no plane round trip)
        if self.wtab is not None:
            xrec = quantize_activations(self.f, x_f32.contiguous(), self.pad)
            y = conv2d_prepared(self.f, xrec, n, h, w, cin, self.wtab, self.kh, self.kw, self.cout, self.stride,
                                self.pad, int(self.relu), nxt=F32)
        else:
            xp = quantize_pack(self.f.we, self.f.wf, x_f32.reshape(n * h * w, cin).contiguous(), self.f.round)
            y = conv2d(self.f, xp, n, h, w, cin, self.w_planes, self.kh, self.kw, self.cout, self.stride, self.pad,
                       int(self.relu), nxt=F32)
        ho, wo = conv_out_hw(h, w, self.kh, self.kw, self.stride, self.pad)
        return y.reshape(n, ho, wo, self.cout)


class Chain:
    """A chain of conv layers kept in the custom format between layers (the
    layer-chaining epilogue of P:262): the float32 input is quantised once into the
    first layer's activation records; every layer but the last re-rounds its
    outputs (after its ReLU) into the next layer's format and writes the next
    layer's records directly (HOBF_OUT_NEXT_RECORDS); the last layer writes exact
    float32 (HOBF_OUT_F32).  Layers are Conv2d objects on the weight-table path
    with one exponent width and one rounding mode; the result equals
    oracle.conv_chain.  Marshalling only: every step runs in the library."""

    def __init__(self, layers):
        if not layers:
            raise ValueError("empty chain")
        we, rnd = layers[0].f.we, layers[0].f.round
        for l in layers:
            if l.wtab is None:
                raise ValueError("every layer of a chain needs prepared weight tables (wf <= 10)")
            if l.f.we != we or l.f.round != rnd:
                raise ValueError("a chain keeps one exponent width and one rounding mode")
        for a, b in zip(layers, layers[1:]):
            if a.cout != b.cin:
                raise ValueError("channel counts of consecutive layers differ")
        self.layers = layers

    def __call__(self, x_f32: torch.Tensor) -> torch.Tensor:
        n, h, w, cin = x_f32.shape
        first = self.layers[0]
        if not x_f32.is_cuda:
            x_f32 = x_f32.to(first.wtab.device)
        rec = quantize_activations(first.f, x_f32.to(torch.float32).contiguous(), first.pad)
        for i, l in enumerate(self.layers):
            ho, wo = conv_out_hw(h, w, l.kh, l.kw, l.stride, l.pad)
            if i + 1 < len(self.layers):
                nx = self.layers[i + 1]
                rec = conv2d_prepared(l.f, rec, n, h, w, l.cin, l.wtab, l.kh, l.kw, l.cout, l.stride, l.pad,
                                      int(l.relu), nxt=Next(nx.f.wf, records=True, pad=nx.pad))
            else:
                y = conv2d_prepared(l.f, rec, n, h, w, l.cin, l.wtab, l.kh, l.kw, l.cout, l.stride, l.pad,
                                    int(l.relu), nxt=F32)
            h, w = ho, wo
        return y.reshape(n, h, w, self.layers[-1].cout)
