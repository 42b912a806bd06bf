"""Static SASS evidence for the conv kernels (development tool).

    python tools/sass_loop_stats.py [fmt] [kernel-substring] > profiles/rNN_sass_<fmt>.txt

Disassembles paper_2007_06563_b200/csrc/build/hobf_fmt_<fmt>.o with cuobjdump,
finds every loop (backward branch) with more than 200 instructions in the
conv kernels, and prints its opcode histogram next to the generator's gate
count: LOP3 per loop body / taps per body = lop3 per 32-lane MAC.
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
fmt = sys.argv[1] if len(sys.argv) > 1 else "e5m3"
want = sys.argv[2] if len(sys.argv) > 2 else "conv_tab"
obj = os.path.join(ROOT, "paper_2007_06563_b200", "csrc", "build", f"hobf_fmt_{fmt.split('_')[0]}.o")
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
counts = json.load(open(os.path.join(ROOT, "paper_2007_06563_b200", "csrc", "gen", "gate_counts.json")))
print(f"# cuobjdump -sass {os.path.relpath(obj, ROOT)}: loops of the {want} kernels")
print(f"# generator gate counts (lop3 per 32-lane MAC): {fmt}_rne {counts[fmt + '_rne']}")
fn, lines = None, []
funcs = {}
for l in sass.splitlines():
    m = re.search(r"Function : (\S+)", l)
    if m:
        fn = m.group(1)
        funcs[fn] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
    if m and fn:
        funcs[fn].append((int(m.group(1), 16), m.group(2).strip()))
for fn, ins in funcs.items():
    tag = f"F_{fmt}_rne"
    if want not in fn or f"{len(tag)}{tag}" not in fn:
        continue
    for a, s in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?(0x[0-9a-f]+)", s)
        if not m or int(m.group(1), 16) >= a:
            continue
        lo = int(m.group(1), 16)
        body = [x for y, x in ins if lo <= y <= a]
        if len(body) < 200:
            continue
        ops = collections.Counter((x.split(None, 1)[1] if x.startswith("@") else x).split()[0] for x in body)
        lop3 = ops.get("LOP3.LUT", 0)
        alu = sum(n for o, n in ops.items() if o.split(".")[0] in ("LOP3", "IADD3", "SHF", "PRMT", "ISETP", "SEL",
                                                                      "LEA", "PLOP3", "VIADD", "IMNMX", "FMNMX"))
        g = counts[fmt + "_rne"]["g_tab"]
        print(f"\n{fn}\n  loop [{lo:#x}, {a:#x}]: {len(body)} instructions, LOP3 {lop3} "
              f"(= {lop3 / g:.2f} x G_tab {g}), ALU-pipe ops {alu}")
        print("  " + ", ".join(f"{o} {n}" for o, n in ops.most_common(16)))
