"""Small invocations of every kernel family, each schedule cross-checked
against the full-gate conv (development tool; meant for compute-sanitizer,
which is closed on this GPU pool -- the parity tests and these cross-checks
stand in for it).

    python tools/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_06563_b200 import hobf as H, inputs  # noqa: E402

n, h, w, cin, cout = 2, 9, 11, 40, 48
x, wt = inputs.small_case(5, n, h, w, cin, cout, "normal", 0.4)
for f in (H.Fmt(5, 3, 0), H.Fmt(5, 10, 1), H.Fmt(4, 3, 0, extended=1)):
    xt = torch.from_numpy(x).cuda()
    wp = H.quantize_pack(f.we, f.wf, torch.from_numpy(wt.reshape(-1, cout)).cuda(), f.round)
    xp = H.quantize_pack(f.we, f.wf, xt.reshape(-1, cin), f.round)
    y1 = H.conv2d(f, xp, n, h, w, cin, wp, 3, 3, cout, 1, 1, 1)
    if H.wtab_words(f, 3, 3, cin, cout) > 0:
        tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
        xr = H.quantize_activations(f, xt, 1)
        for v in (3, 4, 5, 6, 7, 8):
            y2 = H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, 1, variant=v)
            assert torch.equal(y1, y2), v
        r = H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, 1, nxt=H.Next(3, records=True, pad=1))
    H.unpack_f32(f.we, f.wfo, y1, n * h * w, cout)
    H.unpack(f.we, f.wfo, y1, n * h * w, cout)
    H.conv2d(f, xp, n, h, w, cin, wp, 3, 3, cout, 1, 1, 0, nxt=H.Next(3, records=False))
    _, wd = inputs.small_case(6, n, h, w, cin, cin, "normal", 0.4, dw=True)
    wdp = H.quantize_pack(f.we, f.wf, torch.from_numpy(wd.reshape(-1, cin)).cuda(), f.round)
    H.conv2d_dw(f, xp, n, h, w, cin, wdp, 3, 3, 2, 1, 0)
torch.cuda.synchronize()
print("sanitize_small ok")
