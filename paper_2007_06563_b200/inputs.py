"""Seeded synthetic inputs for the BASELINE.json configs.

This module holds NO method arithmetic: it only draws float32 tensors.  Both
the CUDA path (hobf_quantize_pack) and the oracle (ref_encode_f32) quantise
these floats into the custom format themselves.

Recipe (ledger L15/L16): ``numpy.random.Generator(PCG64(seed))``; draw the
activations first (float32, C order, NHWC), apply ReLU with ``np.maximum``
where the config says ReLU(N(0,1)), then draw the weights (KhKwCinCout) as
``standard_normal * float32(sigma)``; sigma is a standard deviation.
Uniform [0,4) is ``4 * random(float32)`` (exact).  Weak-scaling shard s > 0
draws its own activations from seed 1000 + s and reuses shard 0's weights.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class ConvConfig:
    name: str
    n: int
    h: int
    w: int
    cin: int
    cout: int
    formats: tuple           # ((we, wf), ...)
    x_dist: str              # "normal" | "relu_normal" | "uniform4"
    w_sigma: float
    kh: int = 3
    kw: int = 3
    stride: int = 1
    pad: int = 1
    text: str = ""
    dw: bool = False         # depthwise: cout == cin, weights [kh, kw, cin]

    @property
    def ho(self):
        return (self.h + 2 * self.pad - self.kh) // self.stride + 1

    @property
    def wo(self):
        return (self.w + 2 * self.pad - self.kw) // self.stride + 1

    def valid_macs(self, n=None):
        """MACs whose activation tap lies inside the image (padding taps excluded)."""
        n = self.n if n is None else n
        vy = sum(1 for oy in range(self.ho) for k in range(self.kh) if 0 <= oy * self.stride - self.pad + k < self.h)
        vx = sum(1 for ox in range(self.wo) for k in range(self.kw) if 0 <= ox * self.stride - self.pad + k < self.w)
        return n * vy * vx * self.cout * (1 if self.dw else self.cin)

    def macs(self, n=None):
        """Dense MACs (padding taps counted, ledger L11)."""
        n = self.n if n is None else n
        if self.dw:
            return n * self.ho * self.wo * self.cout * self.kh * self.kw
        return n * self.ho * self.wo * self.cout * self.cin * self.kh * self.kw


SWEEP = tuple((we, wf) for we in (4, 5, 6) for wf in range(2, 11))

CONFIGS = {
    "C1": ConvConfig("C1", 1, 8, 8, 16, 32, ((5, 10),), "normal", 0.25,
                     text="BASELINE configs[0]: 3x3 s1 p1, NHWC batch 1, 8x8x16 -> 32, e5m10, x N(0,1), w N(0,0.25)"),
    "C2": ConvConfig("C2", 1, 56, 56, 64, 64, ((5, 10),), "relu_normal", math.sqrt(2 / (9 * 64)),
                     text="BASELINE configs[1]: 3x3 s1 p1, batch 1, 56x56x64 -> 64, e5m10, x ReLU(N(0,1)), w N(0,sqrt(2/576))"),
    "C3": ConvConfig("C3", 32, 56, 56, 64, 64, ((5, 3),), "relu_normal", math.sqrt(2 / (9 * 64)),
                     text="BASELINE configs[2]: 3x3 s1 p1, batch 32, 56x56x64 -> 64, e5m3 (HOBFLOPS9)"),
    "C4": ConvConfig("C4", 256, 28, 28, 128, 128, ((4, 3),), "relu_normal", math.sqrt(2 / (9 * 128)),
                     text="BASELINE configs[3]: 3x3 s1 p1, batch 256, 28x28x128 -> 128, e4m3 (HOBFLOPSIEEE8)"),
    "C5": ConvConfig("C5", 64, 14, 14, 256, 256, SWEEP, "uniform4", 0.05,
                     text="BASELINE configs[4]: format sweep e4-6 m2-10, 3x3 s1 p1, batch 64, 14x14x256 -> 256"),
    # The paper's own workload shape: MobileNets
    # "Conv dw / s2" at 14x14x512, stride 2 -- as the paper runs it (a full conv of
    # M = 512 kernels over C = 512 channels, the IFM broadcast across the kernels,
    # P:257) and in its depthwise form.  The paper states no value distribution:
    # ReLU(N(0,1)) activations and He-normal weights like C2-C4; HOBFLOPS9 (e5m3).
    "MOB": ConvConfig("MOB", 128, 14, 14, 512, 512, ((5, 3),), "relu_normal", math.sqrt(2 / (9 * 512)),
                      stride=2, text="MobileNets Conv dw/s2 shape as a full conv (P:255): batch 128, 14x14x512 -> "
                                     "7x7x512, 3x3 s2 p1, e5m3"),
    "MOBDW": ConvConfig("MOBDW", 256, 14, 14, 512, 512, ((5, 3),), "relu_normal", math.sqrt(2 / 9),
                        stride=2, dw=True, text="MobileNets Conv dw/s2, depthwise (P:255): batch 256, 14x14x512 -> "
                                               "7x7x512, 3x3 s2 p1, e5m3"),
}


def draw(cfg: ConvConfig, n: int | None = None, shard: int = 0, seed: int = 0):
    """Return (x float32 [n,h,w,cin], w float32 [kh,kw,cin,cout])."""
    n = cfg.n if n is None else n
    rng = np.random.Generator(np.random.PCG64(seed))
    xs = _draw_x(rng, cfg, cfg.n)
    wshape = (cfg.kh, cfg.kw, cfg.cin) if cfg.dw else (cfg.kh, cfg.kw, cfg.cin, cfg.cout)
    wt = (rng.standard_normal(wshape, dtype=np.float32) * np.float32(cfg.w_sigma))
    if shard == 0 and n == cfg.n:
        return xs, wt
    if shard == 0:
        if n <= cfg.n:
            return xs[:n].copy(), wt
        rng2 = np.random.Generator(np.random.PCG64(seed + 1000))
        return np.concatenate([xs, _draw_x(rng2, cfg, n - cfg.n)]), wt
    rng2 = np.random.Generator(np.random.PCG64(seed + 1000 + shard))
    return _draw_x(rng2, cfg, n), wt


def _draw_x(rng, cfg: ConvConfig, n: int):
    shape = (n, cfg.h, cfg.w, cfg.cin)
    if cfg.x_dist == "normal":
        return rng.standard_normal(shape, dtype=np.float32)
    if cfg.x_dist == "relu_normal":
        return np.maximum(rng.standard_normal(shape, dtype=np.float32), np.float32(0))
    if cfg.x_dist == "uniform4":
        return np.float32(4) * rng.random(shape, dtype=np.float32)
    raise ValueError(cfg.x_dist)


def small_case(seed: int, n: int, h: int, w: int, cin: int, cout: int, dist: str = "normal",
               w_sigma: float = 0.5, kh: int = 3, kw: int = 3, dw: bool = False):
    """Small seeded case for parity tests (several tiles + ragged tails)."""
    cfg = ConvConfig("small", n, h, w, cin, cout, (), dist, w_sigma, kh, kw, dw=dw)
    return draw(cfg, seed=seed)
