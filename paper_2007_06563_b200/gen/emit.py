"""Emit mapped circuits as straight-line sm_100a CUDA (PTX ``lop3.b32``).

This is the paper's domain-specific source-to-source generator:
a topologically sorted gate netlist becomes a sequence of bitwise operations,
one ``lop3.b32`` per mapped LUT; a 32-bit register holds one bit of 32 lanes
(the GPU analogue of the uint64 / __m512i operand types of P:247).

Usage (build time)::

    python -m paper_2007_06563_b200.gen.emit --out paper_2007_06563_b200/csrc/gen
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

from . import fpgen, sweep
from .lutmap import map_aig

RND_NAME = {0: "rne", 1: "rtz"}

# The format sweep of BASELINE configs[4] (exponent 4-6 x mantissa 2-10), which
# contains every other config's format (e5m10, e5m3, e4m3).
SWEEP = [(we, wf) for we in (4, 5, 6) for wf in range(2, 11)]


def np4(n: int) -> int:
    return (n + 3) // 4 * 4


def mapping_to_cuda(circuit, mapping, fname: str, out_arg: str, extra_doc: str = "") -> tuple[str, int]:
    """Return (device function source, number of lop3 emitted)."""
    g = circuit.g
    expr = {}
    node_of = {}
    loads = []
    for name, node in zip(g.input_names, g.input_nodes):
        local = "i_" + name.replace("[", "_").replace("]", "")
        expr[node] = local
        node_of[name] = node
        loads.append(f"  const uint32_t {local} = {name};")
    lut_nodes = {v for v, _, _ in mapping.luts}
    leaf_use = set()
    for v, leaves, tt in mapping.luts:
        leaf_use.update(leaves)
    # output polarity: flip a LUT's table when it only feeds complemented outputs
    out_pol = {}
    for o in circuit.outputs:
        out_pol.setdefault(o >> 1, set()).add(o & 1)
    flip = {v for v, pols in out_pol.items()
            if v in lut_nodes and pols == {1} and v not in leaf_use}
    lines = []
    n_ops = 0
    for v, leaves, tt in mapping.luts:
        ops = [expr[l] for l in leaves]
        while len(ops) < 3:
            ops.append(ops[0] if ops else "0u")
        if v in flip:
            tt ^= 0xFF
        # leaves[0] -> c, leaves[1] -> b, leaves[2] -> a  (index = 4a + 2b + c)
        lines.append(f"  const uint32_t t{v} = hobf_lop3<0x{tt:02x}>({ops[2]}, {ops[1]}, {ops[0]});")
        expr[v] = f"t{v}"
        n_ops += 1
    # inputs the network never reads (a plane the SDC sweep found equal to another) are not loaded
    used = set()
    for v, leaves, tt in mapping.luts:
        used.update(leaves)
    used.update(o >> 1 for o in circuit.outputs)
    loads = [ld for ld, node in zip(loads, g.input_nodes) if node in used]
    outs = []
    for i, o in enumerate(circuit.outputs):
        v, c = o >> 1, o & 1
        if v == 0:
            e = "0xffffffffu" if c else "0u"
        else:
            base = expr[v]
            if c and v not in flip:
                e = f"~{base}"
                n_ops += 1
            else:
                e = base
        outs.append(f"  {out_arg}[{i}] = {e};")
    args = ", ".join(f"const uint32_t* __restrict__ {name}" if name != out_arg else f"uint32_t* {name}"
                     for name, _ in circuit.inputs)
    if out_arg not in [n for n, _ in circuit.inputs]:
        args += f", uint32_t* {out_arg}"
    # all inputs are read into temporaries before any output is written (acc aliasing)
    src = [f"// {circuit.name}: {n_ops} lop3 per 32 lanes. {extra_doc}",
           f"__device__ __forceinline__ void {fname}({args}) {{"]
    src += loads + lines + outs + ["}"]
    return "\n".join(src), n_ops


def gen_format(we: int, wf: int, rnd: int, ext: int = 0) -> dict:
    """ext = 0: single class (product / accumulator wF+1); ext = 1: extended class
    (exact product, accumulator 2wF+1)."""
    t0 = time.time()
    wfo = 2 * wf + 1 if ext else wf + 1
    nin, nout = 3 + we + wf, 3 + we + wfo
    mac = fpgen.build_mac(we, wf, wfo, rnd)
    mul = fpgen.build_mul(we, wf, wfo, rnd)
    add = fpgen.build_add(we, wfo, rnd)
    mtab = fpgen.build_mac_tab(we, wf, rnd, wfo)
    if not ext:  # merge nodes equal on the valid input space (sweep.py: cached, proved exhaustively)
        cache = sweep.load_cache()
        mac = sweep.reduce("mac", mac, we, wf, rnd, wfo, cache)
        mul = sweep.reduce("mul", mul, we, wf, rnd, wfo, cache)
        add = sweep.reduce("add", add, we, wf, rnd, wfo, cache)
        mtab = sweep.reduce("mac_tab", mtab, we, wf, rnd, wfo, cache)
    else:        # extended-class table MACs: GPU-proved merges only (tools/sweep_gpu.py)
        mtab = sweep.reduce("mac_tab", mtab, we, wf, rnd, wfo, sweep.load_cache(), compute=False)
    mm = map_aig(mac.g, mac.outputs)
    mmul = map_aig(mul.g, mul.outputs)
    madd = map_aig(add.g, add.outputs)
    relu = fpgen.build_relu(we, wfo)
    mrelu = map_aig(relu.g, relu.outputs)
    mmtab = map_aig(mtab.g, mtab.outputs)
    tw = fpgen.tab_entry_width(we, wf, wfo)
    tag = f"e{we}m{wf}{'x' if ext else ''}_{RND_NAME[rnd]}"
    mac_src, g_mac = mapping_to_cuda(mac, mm, f"mac", "acc",
                                     "acc' = add(acc, mul(x, w)), S:555")
    relu_src, g_relu = mapping_to_cuda(relu, mrelu, f"relu", "r", "S:83-91")
    canon = fpgen.build_canon(we, wfo)
    canon_src, _ = mapping_to_cuda(canon, map_aig(canon.g, canon.outputs), "canon", "r",
                                   "canonical form after the mac_tab chain, S:38")
    tab_src, g_tab = mapping_to_cuda(mtab, mmtab, "mac_tab", "acc",
                                     "acc' = add(acc, product from the weight table row of x), S:555")
    body = f"""// GENERATED by paper_2007_06563_b200/gen/emit.py -- do not edit.
// HOBFLOPS {'extended' if ext else 'single'}-class MAC for F({we},{wf}) -> F({we},{wfo}), {RND_NAME[rnd].upper()}.
// NINBITS={nin}, NOUTBITS={nout} (P:257-260). Gate counts (lop3 per 32 lanes):
//   mac (mul+add jointly mapped) = {g_mac}; mul alone = {mmul.n_luts}; add alone = {madd.n_luts}; relu = {g_relu};
//   mac_tab (multiplier read from the per-weight table, fpgen.product_from_table; relaxed
//   accumulator, canonicalised once per output by canon) = {g_tab}.
#pragma once
#include "hobf_lop3.cuh"

namespace hobf_gen {{
struct F_{tag} {{
  static constexpr int WE = {we}, WF = {wf}, WFO = {wfo}, RND = {rnd}, EXT = {ext};
  static constexpr int NIN = {nin}, NOUT = {nout}, NPI = {np4(nin)}, NPO = {np4(nout)};
  static constexpr int G_MAC = {g_mac}, G_MUL = {mmul.n_luts}, G_ADD = {madd.n_luts}, G_RELU = {g_relu};
  static constexpr int G_TAB = {g_tab}, TAB_W = {tw}, NPT = {np4(tw)}, TAB_ROWS = {(1 << wf) + 3};
{indent(mac_src)}
{indent(tab_src)}
{indent(canon_src)}
{indent(relu_src)}
}};
}}  // namespace hobf_gen
"""
    return {"tag": tag, "we": we, "wf": wf, "rnd": rnd, "ext": ext, "src": body, "g_tab": g_tab,
            "g_mac": g_mac, "g_mul": mmul.n_luts, "g_add": madd.n_luts, "g_relu": g_relu,
            "secs": time.time() - t0}


def indent(s: str) -> str:
    return "\n".join(("  " + l if l else l) for l in s.split("\n")).replace("__device__ __forceinline__ void", "__device__ __forceinline__ static void")


def _job(args):
    return gen_format(*args)


def write_all(out_dir: str, formats=None, jobs: int | None = None) -> list[dict]:
    os.makedirs(out_dir, exist_ok=True)
    formats = formats or SWEEP
    todo = [(we, wf, rnd, ext) for (we, wf) in formats for ext in (0, 1) for rnd in (0, 1)]
    with ProcessPoolExecutor(max_workers=jobs or os.cpu_count()) as ex:
        results = list(ex.map(_job, todo))
    for r in results:
        path = os.path.join(out_dir, f"hobf_circuit_{r['tag']}.cuh")
        old = open(path).read() if os.path.exists(path) else None
        if old != r["src"]:
            with open(path, "w") as f:
                f.write(r["src"])
    # per-format translation units + dispatch table
    for (we, wf) in formats:
        path = os.path.join(out_dir, f"hobf_fmt_e{we}m{wf}.cu")
        src = f"""// GENERATED by paper_2007_06563_b200/gen/emit.py -- do not edit.
#include "hobf_circuit_e{we}m{wf}_rne.cuh"
#include "hobf_circuit_e{we}m{wf}_rtz.cuh"
#include "hobf_circuit_e{we}m{wf}x_rne.cuh"
#include "hobf_circuit_e{we}m{wf}x_rtz.cuh"
#include "../hobf_kernels.cuh"
HOBF_INSTANTIATE(e{we}m{wf}_rne, {we}, {wf}, 0)
HOBF_INSTANTIATE(e{we}m{wf}_rtz, {we}, {wf}, 1)
HOBF_INSTANTIATE(e{we}m{wf}x_rne, {we}, {wf}, 0)
HOBF_INSTANTIATE(e{we}m{wf}x_rtz, {we}, {wf}, 1)
"""
        old = open(path).read() if os.path.exists(path) else None
        if old != src:
            with open(path, "w") as f:
                f.write(src)
    table = ["// GENERATED by paper_2007_06563_b200/gen/emit.py -- do not edit.",
             "// {we, wf, rnd, g_mac, g_mul, g_add, g_relu, launch_conv, launch_mac}"]
    decl = []
    for r in sorted(results, key=lambda r: (r["we"], r["wf"], r["ext"], r["rnd"])):
        t = r["tag"]
        decl.append(f"HOBF_DECLARE({t})")
        table.append(f"HOBF_ENTRY({t}, {r['we']}, {r['wf']}, {r['rnd']}, {r['ext']}, {r['g_mac']}, {r['g_mul']}, "
                     f"{r['g_add']}, {r['g_relu']}, {r['g_tab']})")
    with open(os.path.join(out_dir, "hobf_table.inc"), "w") as f:
        f.write("\n".join(["// GENERATED -- declarations"] + decl) + "\n#define HOBF_TABLE_ENTRIES \\\n" +
                " \\\n".join(table[2:]) + "\n")
    counts = {r["tag"]: {k: r[k] for k in ("g_mac", "g_mul", "g_add", "g_relu", "g_tab")} for r in results}
    with open(os.path.join(out_dir, "gate_counts.json"), "w") as f:
        json.dump(counts, f, indent=1, sort_keys=True)
    return results


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "csrc", "gen"))
    ap.add_argument("--jobs", type=int, default=None)
    a = ap.parse_args(argv)
    res = write_all(a.out, jobs=a.jobs)
    for r in res:
        print(f"{r['tag']:14s} mac={r['g_mac']:4d} mul={r['g_mul']:4d} add={r['g_add']:4d} tab={r['g_tab']:4d} ({r['secs']:.1f}s)")


if __name__ == "__main__":
    sys.exit(main())
