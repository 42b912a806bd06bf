"""Kernel-only timing of the edge kernels (development tool, not the bench):
hobf_quantize_activations (float32 NHWC -> records) and hobf_quantize_pack
(float32 -> planes) on the configs' activation shapes, L2 flushed before every
launch, CUDA events, median of reps.

    python tools/edge_bench.py [--configs C3,C4,C5,MOB,MOBDW] [--reps 20]
Prints one line per (config, kernel): us, algorithmic bytes, GB/s, fraction of
MEASURED_PEAKS.json's HBM figure.
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
ap.add_argument("--configs", default="C3,C4,C5,MOB,MOBDW")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--round", type=int, default=0)
ap.add_argument("--flush", default="write", choices=["write", "read", "none"],
                help="L2 flush between launches: write 256 MiB (leaves dirty lines) or read it (clean)")
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
flush_sink = torch.zeros((), dtype=torch.int64, device="cuda")


def timed(run):
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        if a.flush == "write":
            flush.fill_(1)
        elif a.flush == "read":
            flush_sink.copy_(flush.view(torch.int64).sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)) * 1e3


for name in a.configs.split(","):
    cfg = inputs.CONFIGS[name]
    we, wf = cfg.formats[0]
    f = H.Fmt(we, wf, a.round)
    x, _ = inputs.draw(cfg)
    xt = torch.from_numpy(x).cuda()
    nin = int(xt.numel())
    rec = H.quantize_activations(f, xt, cfg.pad)
    us = timed(lambda: H.quantize_activations(f, xt, cfg.pad, out=rec))
    b = nin * 4 + rec.numel() * 4
    print(json.dumps({"config": name, "kernel": "quantize_activations", "us": round(us, 2), "bytes": b,
                      "GBps": round(b / us / 1e3, 1), "frac_hbm": round(b / us / 1e3 / peak, 3)}), flush=True)
    cp = torch.empty_like(xt)
    us = timed(lambda: cp.copy_(xt))
    b = nin * 8
    print(json.dumps({"config": name, "kernel": "torch copy_ (same bytes in)", "us": round(us, 2), "bytes": b,
                      "GBps": round(b / us / 1e3, 1), "frac_hbm": round(b / us / 1e3 / peak, 3)}), flush=True)
    x2 = xt.reshape(-1, cfg.cin)
    pl = H.quantize_pack(we, wf, x2, f.round)
    us = timed(lambda: H.quantize_pack(we, wf, x2, f.round, out=pl))
    b = nin * 4 + pl.numel() * 4
    print(json.dumps({"config": name, "kernel": "quantize_pack", "us": round(us, 2), "bytes": b,
                      "GBps": round(b / us / 1e3, 1), "frac_hbm": round(b / us / 1e3 / peak, 3)}), flush=True)
