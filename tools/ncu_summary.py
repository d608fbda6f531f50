"""Summarise an .ncu-rep: key SOL / occupancy / scheduler metrics and the SASS
regions with the most executed instructions and stall samples.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--regions]"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Registers Per Thread",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Dynamic Shared Memory Per Block",
        "Block Limit Shared Mem", "Block Limit Registers", "Grid Size", "Block Size"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:38s} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if raw:
        h = raw[0]
        for r in raw[2:]:
            d = dict(zip(h, r))
            for kk in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                       "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"):
                if kk in d:
                    print(f"{'raw':40s} {kk:38s} {d[kk]}")
    if "--regions" in sys.argv:
        sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
        h, data = sass[1], sass[2:]
        ie = h.index("Instructions Executed")
        st = h.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(r[ie]) for r in data) or 1
        ts = sum(int(r[st]) for r in data) or 1
        for b in range(0, len(data), 40):
            c = sum(int(r[ie]) for r in data[b:b + 40])
            s = sum(int(r[st]) for r in data[b:b + 40])
            if c > tot * 0.01 or s > ts * 0.01:
                print(f"{b:5d} inst {100 * c / tot:5.1f}%  stall {100 * s / ts:5.1f}%  {data[b][1].strip()[:60]}")


if __name__ == "__main__":
    main()


def groups(rep, min_frac=0.01):
    """Runs of SASS instructions with equal execution counts (basic blocks)."""
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h, data = sass[1], sass[2:]
    ie = h.index("Instructions Executed")
    at = h.index("Avg. Threads Executed")
    tot = sum(int(r[ie]) for r in data)
    cur, start, acc = None, 0, 0
    out = []
    for i, r in enumerate(data + [["", "", "-1"] + [""] * len(h)]):
        c = int(r[ie]) if i < len(data) else -1
        if c != cur:
            if cur is not None and acc > tot * min_frac:
                out.append((start, i - 1, cur, acc, data[start][at], data[start][1].strip()[:50]))
            cur, start, acc = c, i, 0
        acc += max(c, 0)
    for s, e, c, a, t, txt in out:
        print(f"{s:5d}-{e:5d} n={e - s + 1:3d} exec={c:>11d} thr={t:>3s} share={100 * a / tot:5.1f}%  {txt}")
