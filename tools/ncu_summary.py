"""Summaries of ncu captures for profiles/ (read here, after gpurun brings the
reports back).

  python tools/ncu_summary.py report <rep.ncu-rep> <title> <command>   -> per-kernel metric summary
  python tools/ncu_summary.py launches <launches.csv> <title>          -> launch list totals + sequence
"""
import collections
import csv
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_active.avg",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def report(rep, title, command):
    h, units, rows = raw(rep)
    print(title)
    print("command:", command)
    for r in rows:
        print("kernel:", r[h.index("Kernel Name")])
        for m in METRICS:
            if m in h:
                i = h.index(m)
                print(f"  {m:<86} {r[i]:>18} {units[i]}")
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith(STALL) and not name.endswith("_not_issued"):
                try:
                    stalls[name[len(STALL):]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values())
        if tot > 0:
            print("  stall reasons (pc samples, share):")
            for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
                print(f"    {k:<32} {100 * v / tot:5.1f}%")


def launches(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    seq = []
    for r in rows:
        us = float(r[vi].replace(",", "")) / 1000.0
        name = r[ki].split("(")[0]
        tot[name] += us
        cnt[name] += 1
        seq.append((name, us, r[gi] if gi is not None else ""))
    print(title)
    print("source: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)")
    s = sum(tot.values())
    print(f"total {s / 1000:.3f} ms over {len(rows)} launches")
    print(f"{'kernel':<48} {'launches':>8} {'ms':>10} {'share':>7}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:48]:<48} {cnt[k]:>8} {v / 1000:>10.3f} {100 * v / s:>6.1f}%")
    print("\nsequence (launches >= 40 us):")
    for i, (n, us, g) in enumerate(seq):
        if us >= 40:
            print(f"  {i:4d} {n[:44]:<44} {us:9.1f} us  grid {g}")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
