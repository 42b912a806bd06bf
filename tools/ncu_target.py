"""Run the bench step of one config a few times (a target for ncu; development tool).

    ncu --set full -k regex:conv_tab --launch-skip 3 --launch-count 1 -o out \\
        python tools/ncu_target.py --config C5 --format e5m10

The step is bench.py's: quantize (records / planes) + conv with the float32
epilogue, weights prepared once; --variant forces a conv schedule.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_06563_b200 import hobf as H, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--format", default=None)
ap.add_argument("--round", type=int, default=0)
ap.add_argument("--extended", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="f32", choices=["f32", "planes"])
a = ap.parse_args()
cfg = inputs.CONFIGS[a.config]
we, wf = cfg.formats[0] if not a.format else tuple(int(v) for v in a.format[1:].split("m"))
f = H.Fmt(we, wf, a.round, extended=a.extended)
x, w = inputs.draw(cfg)
xt = torch.from_numpy(x).cuda()
wp = H.quantize_pack(we, wf, torch.from_numpy(w.reshape(-1, cfg.cout)).cuda(), f.round)
nxt = H.F32 if a.out == "f32" else None
if cfg.dw:
    for _ in range(a.reps):
        xp = H.quantize_pack(we, wf, xt.reshape(-1, cfg.cin), f.round)
        H.conv2d_dw(f, xp, cfg.n, cfg.h, cfg.w, cfg.cin, wp, cfg.kh, cfg.kw, cfg.stride, cfg.pad, 0, nxt=nxt)
else:
    tab = H.prepare_weights(f, wp, cfg.kh, cfg.kw, cfg.cin, cfg.cout)
    for _ in range(a.reps):
        xr = H.quantize_activations(f, xt, cfg.pad)
        H.conv2d_prepared(f, xr, cfg.n, cfg.h, cfg.w, cfg.cin, tab, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad, 0,
                          variant=a.variant, nxt=nxt)
torch.cuda.synchronize()
print("ok", a.config, f"e{we}m{wf}", H.conv_kernel_info(H.OP_DW if cfg.dw else H.OP_PREPARED, f, cfg.n, cfg.h, cfg.w,
                                                        cfg.cin, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad,
                                                        nxt=nxt, variant=a.variant))
