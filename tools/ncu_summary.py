"""Summarise an ncu --set full report for profiles/ (development tool).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title line" > profiles/rNN_xxx.txt
Prints the launch geometry, pipe utilisation, DRAM traffic, cache hit rates and
the warp-stall breakdown (per-instruction samples from the source page).
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def main(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    print(f"# {title}")
    print(f"# source: {rep} (not committed)")
    print(f"{'Kernel Name':90s} {v[h.index('Kernel Name')]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:90s} {u[i]:10s} {v[i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    idx = {k: i for i, k in enumerate(hh)}
    tot = collections.Counter()
    for row in rows[2:]:
        if len(row) < len(hh):
            continue
        for k in hh:
            if k.startswith("stall_") and "(Not" not in k:
                tot[k] += int(row[idx[k]] or 0)
    s = sum(tot.values()) or 1
    print("# warp-state samples (fraction of all samples):")
    for k, n in tot.most_common(10):
        print(f"{k:90s} {n / s:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
