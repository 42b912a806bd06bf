"""Kernel-only timing of the conv kernels (development tool, not the bench).

    python tools/conv_variants.py --config C3 [--kernel tables|gates] [--variant 3]
Prints one JSON line: conv ms (CUDA events, median of reps), MAC/s, lop3 frac.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2007_06563_b200 import hobf as H, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--format", default=None)
ap.add_argument("--kernel", default="tables")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--round", type=int, default=0)
ap.add_argument("--variant", type=int, default=0, help="hobf_conv2d_prepared_ex schedule (0 = automatic)")
ap.add_argument("--f32", action="store_true", help="float32 epilogue (the bench's output; variant 12 needs it)")
ap.add_argument("--n", type=int, default=0, help="batch override (a rank's share under the strong split)")
a = ap.parse_args()
cfg = inputs.CONFIGS[a.config]
if a.n:
    import dataclasses
    cfg = dataclasses.replace(cfg, n=a.n)
we, wf = cfg.formats[0] if not a.format else tuple(int(v) for v in a.format[1:].split("m"))
f = H.Fmt(we, wf, a.round)
x, w = inputs.draw(cfg)
xp = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, cfg.cin)).cuda(), f.round)
wp = H.quantize_pack(we, wf, torch.from_numpy(w.reshape(-1, cfg.cout)).cuda(), f.round)
g = H.gate_count(f)
if a.kernel == "tables":
    wt = H.prepare_weights(f, wp, 3, 3, cfg.cin, cfg.cout)
    xr = H.prepare_activations(f, xp, cfg.n, cfg.h, cfg.w, cfg.cin, cfg.pad)
    run = lambda: H.conv2d_prepared(f, xr, cfg.n, cfg.h, cfg.w, cfg.cin, wt, 3, 3, cfg.cout,  # noqa: E731
                                    cfg.stride, cfg.pad, variant=a.variant, nxt=H.F32 if a.f32 else None)
    G = g["mac_tab"]
else:
    run = lambda: H.conv2d(f, xp, cfg.n, cfg.h, cfg.w, cfg.cin, wp, 3, 3, cfg.cout, cfg.stride, cfg.pad)  # noqa: E731
    G = g["mac"]
y0 = run()
for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
macs = cfg.macs()
peak = 148 * 64 * 1.965e9
print(json.dumps({"config": a.config, "n": cfg.n, "format": f"e{we}m{wf}", "kernel": a.kernel,
                  "variant": a.variant, "f32": a.f32, "ms": ms,
                  "mac_per_s": macs / ms * 1e3, "G": G, "frac": macs * G / 32 / (ms * 1e-3) / peak,
                  "same_as_first": bool(torch.equal(y, y0))}))
