"""One line per kernel launch from an ncu --metrics launch list (development tool):
time, DRAM read / write, ALU-pipe %.   python tools/launch_summary.py profiles/r02_launches_*.csv"""
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    i_id, i_k, i_m, i_u, i_v = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    by = {}
    for r in rows[1:]:
        d = by.setdefault(int(r[i_id]), {"k": r[i_k]})
        v = float(r[i_v].replace(",", ""))
        u = r[i_u]
        if r[i_m] == "gpu__time_duration.sum":
            v = v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)   # -> us
        if r[i_m].startswith("dram__bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) / 1e6  # -> MB
        d[r[i_m]] = v
    print(path)
    for i in sorted(by):
        d = by[i]
        print(f"{i:3d} {d['k'][:60]:60s} {d.get('gpu__time_duration.sum', 0):9.1f} us  R {d.get('dram__bytes_read.sum', 0):8.1f} MB"
              f"  W {d.get('dram__bytes_write.sum', 0):8.1f} MB  alu {d.get('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 0):.2f}")
