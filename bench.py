#!/usr/bin/env python3
"""Benchmark of the HOBFLOPS hot path on B200: bitsliced custom-FP conv MACs/s.

One step = the whole hot path over one batch: quantise the
float32 activations into the format's activation records (a0+a1), the
bitsliced conv (a3-a8: staging, broadcast, MUL and ADD circuits over the serial
(c,kh,kw) chain, ReLU) whose epilogue writes the exact float32 outputs NHWC
(a9; ``--out planes`` writes bit planes and unpacks them in a third kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

Multi-GPU: one process per GPU under
torchrun; the config's ONE global input is drawn on every rank and each rank
takes its shard (``paper_2007_06563_b200.shard``: images, then 32-lane output
channel groups, then output rows) -- strong scaling, no collective on the data
path.  After timing, the output words are gathered to rank 0 (NCCL point to
point, off the clock), hashed (``output_sha256``: identical for every N) and
sampled against the oracle.  ``--weak`` instead gives every rank a full batch of
its own (seed 1000 + rank).  Timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2007_06563_b200 import inputs  # noqa: E402  (no method arithmetic)
from paper_2007_06563_b200 import shard  # noqa: E402  (slicing / gathering only)

METRIC = "bitsliced custom-FP conv MACs/s per format at 1/2/4/8 B200; % of LOP3 roofline"
N_SM = 148
LOP3_PER_SM_CLK = 64          # 4 SMSPs x 16 lanes/clk on the ALU pipe (B300_MICROARCH rt_SMSP=2; measured 63.7)
SM_MAX_MHZ_FALLBACK = 1965.0  # B200_PROFILING.md clocks.max.sm
L2_BYTES = 126 * 1024 * 1024


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)  # C3: ~0.6 s of timed steps (>= 0.5 s)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hobf", choices=["hobf", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(inputs.CONFIGS))
    ap.add_argument("--format", default=None, help="override format, e.g. e5m10")
    ap.add_argument("--round", default="rne", choices=["rne", "rtz"])
    ap.add_argument("--relu", type=int, default=0)
    ap.add_argument("--extended", type=int, default=0, help="1 = extended MAC class (exact product, 2wF+1 accumulator)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "gates", "tables"],
                    help="conv kernel: gates = full lop3 MAC (hobf_conv2d); tables = prepared weights "
                         "(hobf_prepare_weights + hobf_conv2d_prepared); auto = tables when the format has them")
    ap.add_argument("--out", default="f32", choices=["f32", "planes"],
                    help="f32: the conv epilogue writes float32 NHWC; planes: output planes + hobf_unpack_f32")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank runs a full batch of its own (default: the config's "
                         "global batch split over the ranks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="time every format of the config (C5 format sweep)")
    ap.add_argument("--weights-per-step", action="store_true",
                    help="re-quantise and re-prepare the weights inside every timed step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sass", action="store_true", help="skip the cuobjdump opcode count of the conv kernel")
    ap.add_argument("--cpu-sample-macs", type=float, default=1.2e9,
                    help="MACs of the bounded oracle sample (about 10 s on 16 host cores)")
    return ap.parse_args(argv)


def measured_traffic(cfg_name, we, wf, use_tab, rtz=False, extended=False):
    """DRAM bytes per launch of the conv kernel from a committed ncu capture of this exact
    (config, format, rounding, MAC class, kernel), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    tag = f"e{we}m{wf}" + ("x" if extended else "") + ("_rtz" if rtz else "")
    return t.get(f"{cfg_name}/{tag}/{'conv2d_prepared' if use_tab else 'conv2d'}")


def fmt_of(cfg, override):
    if override:
        we, wf = override[1:].split("m")
        return int(we), int(wf)
    return cfg.formats[0]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------- distributed plumbing

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend):
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def _reduce(self, v: float, op) -> float:
        if not self.pg:
            return v
        import torch
        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.MAX if self.pg else None)

    def sum(self, v: float) -> float:
        return self._reduce(v, self.pg.ReduceOp.SUM if self.pg else None)

    def done(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, pw, reasons = [], [], [], set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            try:
                pw.append(float(p[2]))
            except ValueError:
                pass
            for name, v in zip(self.NAMES, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_index(dist):
    """One rank per GPU.  With more ranks than GPUs (HOBF_OVERSUBSCRIBE=1 only: a
    correctness run of the shard / gather path on a 1-GPU box, never a scaling
    measurement) ranks share devices round-robin."""
    import torch
    n = torch.cuda.device_count()
    if dist.local < n:
        return dist.local
    if os.environ.get("HOBF_OVERSUBSCRIBE") != "1":
        raise SystemExit(f"rank {dist.rank}: LOCAL_RANK {dist.local} but only {n} GPU(s) visible")
    return dist.local % n


# ----------------------------------------------------------------------------- the rank's problem

class Problem:
    """One rank's conv: its input slab, weight slab and shapes (strong scaling: a
    shard of the config's global layer; weak: a full batch of its own)."""

    def __init__(self, cfg, dist, weak: bool):
        self.cfg = cfg
        if weak or dist.world == 1:
            x, w = inputs.draw(cfg, shard=dist.rank) if weak else inputs.draw(cfg)
            self.shard = shard.plan(cfg.n, cfg.cout, cfg.ho, 1, 0)
            self.x, self.w, self.pad = x, w, cfg.pad
            self.x_global, self.w_global = x, w
        else:
            xg, wg = inputs.draw(cfg)
            self.shard = shard.plan(cfg.n, cfg.cout, cfg.ho, dist.world, dist.rank)
            self.x, self.w, self.pad = shard.slice_inputs(xg, wg, self.shard, cfg.stride, cfg.pad, cfg.dw)
            self.x_global, self.w_global = xg, wg
        self.n, self.h, self.wd, self.cin = self.x.shape
        self.cout = self.w.shape[-1]
        self.kh, self.kw, self.stride = cfg.kh, cfg.kw, cfg.stride
        self.ho = (self.h + 2 * self.pad - self.kh) // self.stride + 1
        self.wo = (self.wd + 2 * self.pad - self.kw) // self.stride + 1
        self.dw = cfg.dw

    def macs(self):
        return self.n * self.ho * self.wo * self.cout * (1 if self.dw else self.cin) * self.kh * self.kw


# ----------------------------------------------------------------------------- static SASS evidence

def sass_stats(lib_path, fmt_tag, kernel_symbol, g_per_mac):
    """Opcode counts of the conv kernel the bench ran: its format's cubin is extracted
    from libhobf.so (cuobjdump -xelf), disassembled, and the function with the exact
    symbol hobf_conv_kernel_info reported is counted -- whole function and its largest
    loop (LOP3 per tap there = G / 32 lanes); UBLKCP = cp.async.bulk (TMA), SYNCS =
    mbarrier operations."""
    if not kernel_symbol:
        return None
    cubin = f"hobf_fmt_{fmt_tag}.sm_100a.cubin"
    with tempfile.TemporaryDirectory() as td:
        r = subprocess.run(["cuobjdump", "-xelf", cubin, lib_path], cwd=td, capture_output=True, text=True)
        if r.returncode != 0 or not os.path.exists(os.path.join(td, cubin)):
            return {"error": "cuobjdump -xelf failed"}
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(td, cubin)], capture_output=True, text=True).stdout
    ins, cur = [], None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        if cur != kernel_symbol:
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    if not ins:
        return {"error": "symbol not found in the cubin"}

    def op(s):
        s = s.split(None, 1)[1] if s.startswith("@") else s
        return s.split()[0]

    def hist(body):
        h = {}
        for _, s in body:
            o = op(s).split(".")[0]
            h[o] = h.get(o, 0) + 1
        return h

    whole = hist(ins)
    best, best_d = None, -1.0
    for a, s in ins:  # the MAC loop: the backward-branch body with >= G LOP3 and the highest LOP3 density
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?(0x[0-9a-f]+)", s)
        if m and int(m.group(1), 16) < a:
            lo = int(m.group(1), 16)
            body = [(y, x) for y, x in ins if lo <= y <= a]
            nl = sum(1 for _, x in body if op(x).startswith("LOP3"))
            if g_per_mac and nl >= g_per_mac and nl / len(body) > best_d:
                best, best_d = body, nl / len(body)
    loop = hist(best) if best else {}
    lop3 = loop.get("LOP3", 0)
    return {"symbol": kernel_symbol, "instructions": len(ins), "LOP3": whole.get("LOP3", 0),
            "UBLKCP": whole.get("UBLKCP", 0), "SYNCS": whole.get("SYNCS", 0),
            "loop_instructions": len(best) if best else 0, "loop_LOP3": lop3,
            "loop_taps_at_G": round(lop3 / g_per_mac, 3) if g_per_mac else None,
            "loop_alu_share_LOP3": round(lop3 / max(1, sum(n for o, n in loop.items() if o in (
                "LOP3", "IADD3", "SHF", "PRMT", "ISETP", "SEL", "LEA", "PLOP3", "VIADD", "IMNMX"))), 4)}


# ----------------------------------------------------------------------------- reference arm (the oracle)

def run_reference(a, dist):
    """--impl reference: the CPU oracle, as it stands, on the host cores; rank 0 only."""
    if dist.rank != 0:
        return 0
    import oracle  # test infrastructure: allowed in bench.py's reference / cpu_baseline legs
    cfg = inputs.CONFIGS[a.config]
    we, wf = fmt_of(cfg, a.format)
    rnd = 0 if a.round == "rne" else 1
    cores = os.cpu_count() or 1
    x, w = inputs.draw(cfg, n=1)
    per_img = cfg.macs(1)
    # bounded sample per step: the conv of the first `rows` input rows of image 0
    # (an image of height `rows`), sized so that K+W steps take a few minutes at
    # the oracle's ~0.3e9 MAC/s: at most 0.4e9 MACs a step, 3.6e10 in all
    budget = min(0.4e9, 3.6e10 / max(1, a.steps + a.warmup))
    rows = max(1, min(cfg.h, int(round(cfg.h * min(1.0, budget / per_img)))))
    xq = oracle.encode_f32(x, we, wf, rnd)
    wq = oracle.encode_f32(w, we, wf, rnd)
    xin = np.ascontiguousarray(xq[:, :rows])
    ho_s = (rows + 2 * cfg.pad - cfg.kh) // cfg.stride + 1
    sample_macs = ho_s * cfg.wo * cfg.cout * (1 if cfg.dw else cfg.cin) * cfg.kh * cfg.kw
    conv = oracle.conv2d_dw if cfg.dw else oracle.conv2d

    def step():
        wfo = 2 * wf + 1 if a.extended else wf + 1
        y = conv(xin, wq, we, wf, wfo, rnd, cfg.stride, cfg.pad, a.relu, nthreads=cores)
        return y

    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    dt = time.perf_counter() - t0
    value = sample_macs * a.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MAC/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if a.weak else "strong", "vs_baseline": None, "dtype": f"e{we}m{wf}-exact-scalar",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.text}", "format": f"e{we}m{wf}", "round": a.round,
                   "batch": 1, "sample_output_rows": rows},
        "cpu_baseline": {"value": value, "unit": "MAC/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"conv of the first {rows} of {cfg.h} input rows of image 0 of {cfg.name} per step"},
        "e2e": {"value": value, "unit": "MAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, we, wf, wfo, rnd, relu, target_macs):
    """The oracle as it stands on the host cores (all threads), a bounded sample of the
    workload; plus its single-thread rate on a bounded sample of C2 (configs[1]), the
    paper's single-core measurement."""
    import oracle
    cores = os.cpu_count() or 1
    per_img = cfg.macs(1)
    n = max(1, min(cfg.n, int(round(target_macs / per_img))))
    x, w = inputs.draw(cfg, n=n)
    xq = oracle.encode_f32(x, we, wf, rnd)
    wq = oracle.encode_f32(w, we, wf, rnd)
    t0 = time.perf_counter()
    conv = oracle.conv2d_dw if cfg.dw else oracle.conv2d
    conv(xq, wq, we, wf, wfo, rnd, cfg.stride, cfg.pad, relu, nthreads=cores)
    dt = time.perf_counter() - t0
    # single thread: the first 8 input rows of C2 (e5m10, 8 x 56 x 64 x 64 x 9 MACs)
    c2 = inputs.CONFIGS["C2"]
    x2, w2 = inputs.draw(c2)
    rows = 8
    x2q = oracle.encode_f32(np.ascontiguousarray(x2[:, :rows]), 5, 10, 0)
    w2q = oracle.encode_f32(w2, 5, 10, 0)
    t1 = time.perf_counter()
    oracle.conv2d(x2q, w2q, 5, 10, 11, 0, 1, 1, 0, nthreads=1)
    dt1 = time.perf_counter() - t1
    macs1 = rows * c2.wo * c2.cout * c2.cin * 9
    return {"value": cfg.macs(n) / dt, "unit": "MAC/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{n} of {cfg.n} images of {cfg.name} (full conv, every output exact), {dt:.1f} s",
            "single_thread": {"value": macs1 / dt1, "unit": "MAC/s", "cores": 1,
                              "sample": f"C2 (e5m10 RNE) output rows 0-{rows - 1} of 56, {macs1:.3g} MACs, {dt1:.1f} s"}}


def parity_sample(cfg, we, wf, wfo, rnd, relu, y_words, x_f32, w_f32, k=256):
    import oracle
    xq = oracle.encode_f32(x_f32, we, wf, rnd)
    wq = oracle.encode_f32(w_f32, we, wf, rnd)
    rng = np.random.default_rng(123)
    idx = rng.integers(0, y_words.size, k)
    if cfg.dw:
        exp = oracle.conv2d_dw(xq, wq, we, wf, wfo, rnd, cfg.stride, cfg.pad, relu).ravel()[idx]
    else:
        exp = oracle.conv2d_sample(xq, wq, idx, we, wf, wfo, rnd, cfg.stride, cfg.pad, relu)
    return {"checked": int(k), "mismatches": int((y_words.ravel()[idx] != exp).sum())}


# ----------------------------------------------------------------------------- GPU arm

def run_gpu(a, dist):
    import torch
    from paper_2007_06563_b200 import hobf as H

    dev = torch.device("cuda", gpu_index(dist))
    torch.cuda.set_device(dev)
    cfg = inputs.CONFIGS[a.config]
    we, wf = fmt_of(cfg, a.format)
    rnd = 0 if a.round == "rne" else 1
    f = H.Fmt(we, wf, rnd, extended=a.extended)
    P = Problem(cfg, dist, a.weak)
    n, h, w, cin, cout, pad = P.n, P.h, P.wd, P.cin, P.cout, P.pad
    rows_x, rows_y = n * h * w, n * P.ho * P.wo
    rows_w = cfg.kh * cfg.kw * (1 if cfg.dw else cin)
    wt = torch.from_numpy(np.ascontiguousarray(P.w.reshape(rows_w, cout))).to(dev)
    wp = torch.empty(H.planes_shape(rows_w, cout, f.nin), dtype=torch.int32, device=dev)
    tab_words = 0 if cfg.dw else H.wtab_words(f, cfg.kh, cfg.kw, cin, cout)
    # depthwise: the activation is not broadcast (lanes = channels of both operands),
    # so there is no weight table: the full gate MAC (hobf_conv2d_dw)
    use_tab = not cfg.dw and (a.kernel == "tables" or (a.kernel == "auto" and tab_words > 0))
    f32_out = a.out == "f32"
    epi = H.F32 if f32_out else None
    wtab = torch.empty(max(tab_words, 4), dtype=torch.int32, device=dev) if use_tab else None
    # double-buffered per-step activations / outputs (the e2e leg overlaps copies with compute)
    xs = [torch.from_numpy(P.x).to(dev) for _ in range(2)]
    xps = [torch.empty(H.planes_shape(rows_x, cin, f.nin), dtype=torch.int32, device=dev)
           if not use_tab else None for _ in range(2)]
    xrecs = [torch.empty(max(H.xrec_words(n, h, w, cin, pad), 4), dtype=torch.int32, device=dev)
             if use_tab else None for _ in range(2)]
    yps = [torch.empty(H.planes_shape(rows_y, cout, f.nout), dtype=torch.int32, device=dev) for _ in range(2)]
    ys = [torch.empty((rows_y, cout), dtype=torch.float32, device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream()
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    launches = [0]

    def conv(b, st, nxt, out):
        x, xp, xrec = xs[b], xps[b], xrecs[b]
        if use_tab:
            H.conv2d_prepared(f, xrec, n, h, w, cin, wtab, cfg.kh, cfg.kw, cout, cfg.stride, pad, a.relu, out=out,
                              stream=st, nxt=nxt)
        elif cfg.dw:
            H.conv2d_dw(f, xp, n, h, w, cin, wp, cfg.kh, cfg.kw, cfg.stride, pad, a.relu, out=out, stream=st,
                        nxt=nxt)
        else:
            H.conv2d(f, xp, n, h, w, cin, wp, cfg.kh, cfg.kw, cout, cfg.stride, pad, a.relu, out=out, stream=st,
                     nxt=nxt)
        launches[0] += H.last_launch_count()

    def quantize(b, st):
        if use_tab:
            H.quantize_activations(f, xs[b], pad, out=xrecs[b], stream=st)
        else:
            H.quantize_pack(we, wf, xs[b].view(rows_x, cin), rnd, out=xps[b], stream=st)
        launches[0] += H.last_launch_count()

    def step(b=0, conv_ev=None, st=None):
        st = st or stream
        quantize(b, st)
        if a.weights_per_step:
            prep_weights(st)
        if conv_ev:
            conv_ev[0].record(st)
        conv(b, st, epi, ys[b] if f32_out else yps[b])
        if conv_ev:
            conv_ev[1].record(st)
        if not f32_out:
            H.unpack_f32(we, f.wfo, yps[b], rows_y, cout, out=ys[b], stream=st); launches[0] += H.last_launch_count()

    def prep_weights(st):
        # the layer's weights: quantise + bitslice (a1) and the per-weight product tables;
        # done once per layer (kernel data pre-transformed) unless --weights-per-step
        H.quantize_pack(we, wf, wt, rnd, out=wp, stream=st); launches[0] += H.last_launch_count()
        if use_tab:
            H.prepare_weights(f, wp, cfg.kh, cfg.kw, cin, cout, out=wtab, stream=st)
            launches[0] += H.last_launch_count()

    prep_weights(stream)
    torch.cuda.synchronize()
    pw0, pw1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.fill_(1)
    pw0.record(stream)
    prep_weights(stream)
    pw1.record(stream)
    torch.cuda.synchronize()
    weight_prep_ms = pw0.elapsed_time(pw1)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    K = a.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = ClockSampler(torch.cuda.current_device())
    launches[0] = 0
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.15)
    for k in range(K):
        flush.fill_(k)                      # evict L2 between timed steps (untimed)
        ev[k][0].record(stream)
        step(0, cev[k])
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    dist.barrier()
    step_t = [s.elapsed_time(e) for s, e in ev]
    conv_t = [s.elapsed_time(e) for s, e in cev]
    step_ms, conv_ms = sum(step_t), sum(conv_t)
    gpu_launches = launches[0]
    t_max = dist.max(step_ms) / 1e3
    conv_max = dist.max(conv_ms) / 1e3
    macs_rank = P.macs()
    macs_step = dist.sum(macs_rank) if not a.weak else dist.world * macs_rank
    value = macs_step * K / t_max
    # median of 5 repeats (consecutive blocks of the K timed steps; BASELINE.md report row)
    blocks = np.array_split(np.arange(K), 5) if K >= 5 else [np.arange(K)]
    rep = [macs_step * len(b) / (dist.max(sum(step_t[i] for i in b)) / 1e3) for b in blocks]

    # --- e2e through the public API with host buffers: every step copies its float32
    # activations from pinned host memory and reads its float32 output back; the copies
    # of step k+1 / k-1 run on a copy stream while step k computes (double buffers).
    e2e = None
    if not a.no_e2e:
        xh = torch.from_numpy(P.x).pin_memory()
        yh = [torch.empty((rows_y, cout), dtype=torch.float32).pin_memory() for _ in range(2)]
        cs = torch.cuda.Stream()
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        comp_done = [torch.cuda.Event() for _ in range(2)]
        d2h_done = [torch.cuda.Event() for _ in range(2)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def run_e2e(steps):
            with torch.cuda.stream(cs):
                xs[0].copy_(xh, non_blocking=True)
                h2d_done[0].record(cs)
            for k in range(steps):
                b = k % 2
                stream.wait_event(h2d_done[b])
                if k >= 2:
                    stream.wait_event(d2h_done[b])       # output buffer b read back
                step(b)
                comp_done[b].record(stream)
                with torch.cuda.stream(cs):
                    if k + 1 < steps:
                        if k >= 1:
                            cs.wait_event(comp_done[1 - b])   # buffer 1-b free again
                        xs[1 - b].copy_(xh, non_blocking=True)
                        h2d_done[1 - b].record(cs)
                    cs.wait_event(comp_done[b])
                    yh[b].copy_(ys[b], non_blocking=True)
                    d2h_done[b].record(cs)
            stream.wait_stream(cs)

        run_e2e(3)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        cs.wait_stream(stream)
        run_e2e(K)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_s = dist.max(e0.elapsed_time(e1) / 1e3)
        e2e = {"value": macs_step * K / e2e_s, "unit": "MAC/s",
               "h2d_bytes_per_step": int(xh.numel() * 4), "d2h_bytes_per_step": int(yh[0].numel() * 4),
               "ms_per_step": e2e_s / K * 1e3,
               "note": "per rank: pinned host float32 in/out every step; copies overlapped with compute (2 streams)"}

    # --- the output words (off the clock): the same conv with the planes epilogue, unpacked;
    # gathered to rank 0 (strong scaling) and hashed, so N = 1/2/4/8 can be compared
    conv(0, stream, None, yps[0])
    words = H.unpack(we, f.wfo, yps[0], rows_y, cout).cpu().numpy().view(np.uint32).reshape(n, P.ho, P.wo, cout)
    if f32_out:   # the float32 epilogue wrote exactly what unpack_f32 of these planes gives
        yd = H.unpack_f32(we, f.wfo, yps[0], rows_y, cout)
        step(0)
        torch.cuda.synchronize()
        f32_consistent = bool(torch.equal(yd.view(torch.int32), ys[0].view(torch.int32)))
    else:
        f32_consistent = None
    full = None
    if a.weak or dist.world == 1:
        full = words if dist.rank == 0 else None
    else:
        shards = shard.all_shards(cfg.n, cfg.cout, cfg.ho, dist.world)
        full = shard.gather_to_rank0(dist.pg, words, shards, cfg.wo, cfg.n, cfg.ho, cfg.cout, dist.rank,
                                     device=dev if dist.pg.get_backend() == "nccl" else None)

    # --- roofline of the dominant kernel (conv): algorithmic lop3 = MACs * G / 32
    g = H.gate_count(f)
    G = g["mac_tab"] if use_tab else g["mac"]
    op = H.OP_PREPARED if use_tab else (H.OP_DW if cfg.dw else H.OP_CONV)
    kinfo = H.conv_kernel_info(op, f, n, h, w, cin, cfg.kh, cfg.kw, cout, cfg.stride, pad, nxt=epi)
    lop3_per_launch = macs_rank * G / 32.0
    sm_mhz = clk["sm_max_mhz"] or SM_MAX_MHZ_FALLBACK
    peak = N_SM * LOP3_PER_SM_CLK * sm_mhz * 1e6
    achieved = lop3_per_launch * K / conv_max
    sink = torch.zeros(1024, dtype=torch.int32, device=dev)
    H.lop3_peak(N_SM * 4, 256, 200, sink)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    nops = H.lop3_peak(N_SM * 4, 256, 2000, sink)
    pe1.record(stream)
    torch.cuda.synchronize()
    measured_peak = nops / (pe0.elapsed_time(pe1) / 1e3)
    warps = kinfo["blocks"] * ((kinfo["threads"] + 31) // 32)

    # algorithmic bytes of the edge kernel(s): float32 activations in, records / planes out
    edge_bytes = P.x.nbytes + (4 * n * cin * (h + 2 * pad) * (w + 2 * pad) if use_tab
                               else 4 * rows_x * ((cin + 31) // 32) * ((f.nin + 3) // 4 * 4))
    if not f32_out:
        edge_bytes += 4 * rows_y * ((cout + 31) // 32) * ((f.nout + 3) // 4 * 4) + 4 * rows_y * cout
    if dist.rank != 0:
        return 0
    sass = None
    if not a.no_sass:
        try:
            sass = sass_stats(H.LIB_PATH, f"e{we}m{wf}", kinfo["name"], G)
        except (OSError, subprocess.SubprocessError) as e:  # cuobjdump missing or failing: evidence only
            sass = {"error": str(e)}
    s0 = P.shard
    line = {
        "metric": METRIC, "value": value, "unit": "MAC/s", "n_gpus": dist.world, "steps": K, "warmup": a.warmup,
        "ms_per_step": t_max / K * 1e3, "higher_is_better": True, "scaling": "weak" if a.weak else "strong",
        "vs_baseline": None,
        "dtype": f"e{we}m{wf}->e{we}m{f.wfo} custom FP, bitsliced u32 lop3", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.text}", "format": f"e{we}m{wf}", "round": a.round,
                   "mac_class": "extended" if a.extended else "single", "relu": a.relu,
                   "global_batch": cfg.n * (dist.world if a.weak else 1),
                   "per_gpu_batch": n, "dense_macs_per_step": int(macs_step),
                   "valid_tap_macs_per_step": cfg.valid_macs() * (dist.world if a.weak else 1),
                   "l2": "flushed (256 MiB write) between timed steps",
                   "step": (("quantize_activations(x) + conv2d_prepared" if use_tab else
                             "quantize_pack(x) + conv2d_dw" if cfg.dw else "quantize_pack(x) + conv2d") +
                            (" with the float32 output epilogue" if f32_out else " + unpack_f32(y)") +
                            (" + weight prep" if a.weights_per_step else
                             "; weights prepared once per layer (quantize_pack(w) + prepare_weights, P:203), "
                             "timed separately as weight_prep_ms")),
                   "weight_prep_ms": weight_prep_ms,
                   "parallelism": (f"dp{dist.world} weak (every rank a full batch of its own)" if a.weak else
                                   f"{dist.world} rank(s), split {s0.kind} (batch x cout-group x row factors "
                                   f"{list(s0.factors)}), no collective on the data path")},
        "repeats": {"mac_per_s": rep, "median_of_5": float(np.median(rep)),
                    "note": "the K timed steps in 5 consecutive blocks"},
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tlop3/s",
                     "frac": achieved / peak,
                     "traffic": measured_traffic(cfg.name, we, wf, use_tab, rnd == 1, bool(a.extended))
                     if (dist.world == 1 and not a.weak) or a.weak else None,
                     "kernel": "conv2d_prepared (weight tables)" if use_tab else
                               "conv2d_dw (depthwise, full lop3 MAC)" if cfg.dw else "conv2d (full lop3 MAC)",
                     "launch": kinfo,
                     "warps": int(warps), "smsp_occupied_frac": min(1.0, warps / (N_SM * 4)),
                     "gates_per_32lane_mac": G, "gates_full_mac": g["mac"],
                     "peak_source": f"derived: {N_SM} SM x {LOP3_PER_SM_CLK} lop3/clk x {sm_mhz:.0f} MHz",
                     "measured_lop3_peak": measured_peak / 1e12,
                     "conv_ms_per_step": conv_max / K * 1e3,
                     "conv_ms_median": float(np.median(conv_t)),
                     "mac_per_s_conv_only": macs_step * K / conv_max,
                     "paper_G257_roof_frac": (macs_rank * K / conv_max) / (peak * 32 / 257)},
        "edge": {  # the step minus the conv: quantise / layout of the activations (plus unpack with --out planes)
            "ms_per_step": (t_max - conv_max) / K * 1e3,
            "bytes_per_step": int(edge_bytes),
            "GBps": edge_bytes / max((t_max - conv_max) / K, 1e-12) / 1e9,
            "note": "algorithmic bytes (float32 in + records or planes out) / (step - conv) time; includes the "
                    "launch gap between the two kernels"},
        "paper_context": {"note": "single CPU core, other hardware (BASELINE.md): context, not a comparison",
                          "HOBFLOPS9_avx512_mac_per_s": 2e9, "HOBFLOPS9_src": "P:353 (Xeon Gold 5120, 512 lanes)",
                          "HOBFLOPS16_vs_SoftFP16_avx512": 8.2, "HOBFLOPS16_src": "P:353",
                          "HOBFLOPS9_neon_mac_per_s": 45e6, "HOBFLOPS9_neon_src": "P:33, P:360 (Cortex-A15)",
                          "HOBFLOPS8_avx512_gates": {"mul": 53, "add": 204, "src": "P:249"}},
        "sass": sass,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clk,
        "output_sha256": shard.words_sha256(full) if full is not None else None,
        "oversubscribed": os.environ.get("HOBF_OVERSUBSCRIBE") == "1" and dist.world > torch.cuda.device_count(),
        "f32_epilogue_equals_unpack_f32": f32_consistent,
    }
    if full is not None and not a.no_cpu_baseline:
        line["parity_sample"] = parity_sample(cfg, we, wf, f.wfo, rnd, a.relu, full, P.x_global, P.w_global)
    if dist.world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, we, wf, f.wfo, rnd, a.relu, a.cpu_sample_macs)
    print(json.dumps(line), flush=True)
    return 0


def run_sweep(a, dist):
    """--config C5 --sweep: every format of the sweep (configs[4]), each timed on the
    device like the main line (quantize + conv with the float32 epilogue per step);
    prints one JSON line whose value is all formats' dense MACs / their summed step
    time, with the per-format MAC/s and roofline fractions under "per_format".
    Strong scaling (the global batch split over the ranks) unless --weak."""
    import torch
    from paper_2007_06563_b200 import hobf as H

    dev = torch.device("cuda", gpu_index(dist))
    torch.cuda.set_device(dev)
    cfg = inputs.CONFIGS[a.config]
    rnd = 0 if a.round == "rne" else 1
    P = Problem(cfg, dist, a.weak)
    n, h, w, cin, cout, pad = P.n, P.h, P.wd, P.cin, P.cout, P.pad
    x = torch.from_numpy(P.x).to(dev)
    wt = torch.from_numpy(np.ascontiguousarray(P.w.reshape(-1, cout))).to(dev)
    rows_y = n * P.ho * P.wo
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    per, tot_ms, tot_macs, launches = {}, 0.0, 0, 0
    peak = N_SM * LOP3_PER_SM_CLK * SM_MAX_MHZ_FALLBACK * 1e6
    macs_step = dist.sum(P.macs()) if not a.weak else dist.world * P.macs()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for (we, wf) in cfg.formats:
        f = H.Fmt(we, wf, rnd, extended=a.extended)
        wp = H.quantize_pack(we, wf, wt, rnd)
        wtab = H.prepare_weights(f, wp, cfg.kh, cfg.kw, cin, cout)
        xrec = H.quantize_activations(f, x, pad)
        y = torch.empty((rows_y, cout), dtype=torch.float32, device=dev)

        def step(cev=None):
            n_l = 0
            H.quantize_activations(f, x, pad, out=xrec); n_l += H.last_launch_count()
            if a.weights_per_step:
                H.quantize_pack(we, wf, wt, rnd, out=wp); n_l += H.last_launch_count()
                H.prepare_weights(f, wp, cfg.kh, cfg.kw, cin, cout, out=wtab); n_l += H.last_launch_count()
            if cev:
                cev[0].record(stream)
            H.conv2d_prepared(f, xrec, n, h, w, cin, wtab, cfg.kh, cfg.kw, cout, cfg.stride, pad, a.relu, out=y,
                              nxt=H.F32); n_l += H.last_launch_count()
            if cev:
                cev[1].record(stream)
            return n_l

        for _ in range(a.warmup):
            step()
        K = a.steps
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        dist.barrier()
        torch.cuda.synchronize()
        for k in range(K):
            flush.fill_(k)
            ev[k][0].record(stream)
            launches += step(cev[k])
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        ms = dist.max(sum(s_.elapsed_time(e_) for s_, e_ in ev))
        cms = dist.max(sum(s_.elapsed_time(e_) for s_, e_ in cev))
        G = H.gate_count(f)["mac_tab"]
        macs = macs_step * K
        ki = H.conv_kernel_info(H.OP_PREPARED, f, n, h, w, cin, cfg.kh, cfg.kw, cout, cfg.stride, pad, nxt=H.F32)
        per[f"e{we}m{wf}"] = {"mac_per_s": macs / (ms / 1e3), "conv_mac_per_s": macs / (cms / 1e3), "G": G,
                             "roofline_frac": P.macs() * K * G / 32 / (cms / 1e3) / peak,
                             "variant": ki["variant"], "threads": ki["threads"], "ctas_per_sm": ki["ctas_per_sm"],
                             "regs": ki["regs"], "local_bytes": ki["local_bytes"]}
        tot_ms += ms
        tot_macs += macs
        del wtab, xrec, y, wp
    clk = clocks.stop()
    if dist.rank == 0:
        worst = min(v["roofline_frac"] for v in per.values())
        best = max(v["roofline_frac"] for v in per.values())
        print(json.dumps({
            "metric": METRIC, "value": tot_macs / (tot_ms / 1e3), "unit": "MAC/s", "n_gpus": dist.world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": tot_ms / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.weak else "strong", "vs_baseline": None,
            "dtype": "sweep e{4,5,6}m{2..10} custom FP, bitsliced u32 lop3", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.text}", "round": a.round, "formats": len(cfg.formats),
                       "global_batch": cfg.n * (dist.world if a.weak else 1), "per_gpu_batch": n,
                       "l2": "flushed (256 MiB write) between timed steps",
                       "step": "for every format: quantize_activations + conv2d_prepared (float32 epilogue; weights "
                               "prepared once per layer" + (", and again every step)" if a.weights_per_step else ")"),
                       "parallelism": f"{dist.world} rank(s), split {P.shard.kind}, no collective"},
            "roofline": {"bound": "alu", "unit": "fraction of LOP3 roof per format",
                         "frac_min": worst, "frac_max": best, "peak_tlop3_s": peak / 1e12},
            "per_format": per, "gpu_launches": launches, "clocks": clk}), flush=True)
    return 0


def main(argv=None):
    a = parse_args(argv)
    dist = Dist()
    if a.impl == "reference":
        rc = run_reference(a, dist)
        return rc
    import torch
    oversub = os.environ.get("HOBF_OVERSUBSCRIBE") == "1"
    dist.init("nccl" if torch.cuda.is_available() and not oversub else "gloo")
    try:
        if a.sweep:
            return run_sweep(a, dist)
        return run_gpu(a, dist)
    finally:
        dist.done()


if __name__ == "__main__":
    sys.exit(main())
