"""Development tool: conv2d_prepared throughput vs batch size (wave quantisation /
occupancy tail) and per-kernel times of one bench step.

    python tools/wave_scan.py --config C3 --ns 8,16,27,32,54,64
Prints one JSON line per batch size (CUDA events, median of reps).
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
ap.add_argument("--ns", default="32")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--round", type=int, default=0)
ap.add_argument("--const-x", type=float, default=None, help="every activation = this value (one table row)")
ap.add_argument("--steps", action="store_true", help="also time quantize_activations / unpack_f32 / prepare_weights")
a = ap.parse_args()
cfg = inputs.CONFIGS[a.config]
we, wf = cfg.formats[0] if not a.format else tuple(int(v) for v in a.format[1:].split("m"))
f = H.Fmt(we, wf, a.round)
G = H.gate_count(f)["mac_tab"]
peak = 148 * 64 * 1.965e9


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for n in [int(v) for v in a.ns.split(",")]:
    x, w = inputs.draw(cfg, n=n)
    if a.const_x is not None:
        x = np.full_like(x, a.const_x)
    xt = torch.from_numpy(x).cuda()
    wp = H.quantize_pack(we, wf, torch.from_numpy(w.reshape(-1, cfg.cout)).cuda(), f.round)
    wt = H.prepare_weights(f, wp, cfg.kh, cfg.kw, cfg.cin, cfg.cout)
    xr = H.quantize_activations(f, xt, cfg.pad)
    yp = H.conv2d_prepared(f, xr, n, cfg.h, cfg.w, cfg.cin, wt, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad)
    ms = timed(lambda: H.conv2d_prepared(f, xr, n, cfg.h, cfg.w, cfg.cin, wt, cfg.kh, cfg.kw, cfg.cout, cfg.stride,
                                         cfg.pad, out=yp), a.reps)
    macs = cfg.macs(n)
    warps = (n * cfg.ho * cfg.wo + 31) // 32 * ((cfg.cout + 31) // 32)
    rec = {"const_x": a.const_x, "config": a.config, "format": f"e{we}m{wf}", "n": n, "warps": warps, "warps_per_smsp": warps / 592,
           "ms": ms, "mac_per_s": macs / ms * 1e3, "G": G, "frac": macs * G / 32 / (ms * 1e-3) / peak}
    if a.steps:
        rows_y = n * cfg.ho * cfg.wo
        y = torch.empty((rows_y, cfg.cout), dtype=torch.float32, device="cuda")
        rec["quantize_activations_ms"] = timed(lambda: H.quantize_activations(f, xt, cfg.pad, out=xr), a.reps)
        rec["unpack_f32_ms"] = timed(lambda: H.unpack_f32(we, f.wfo, yp, rows_y, cfg.cout, out=y), a.reps)
        rec["prepare_weights_ms"] = timed(lambda: H.prepare_weights(f, wp, cfg.kh, cfg.kw, cfg.cin, cfg.cout, out=wt),
                                          a.reps)
        rec["wtab_MB"] = wt.numel() * 4 / 1e6
    print(json.dumps(rec), flush=True)
