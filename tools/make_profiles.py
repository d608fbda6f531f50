"""Turn raw ncu outputs from gpurun_out/ into the committed summaries in profiles/.

    python tools/make_profiles.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_r01.ncu-rep
writes profiles/<tag>_launches.txt, profiles/<tag>_ncu_<kernel>.txt and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * 1e-6)
    tot = sum(sum(v) for v in agg.values())
    what = ("# cold-cache serialised launches of `tools/recon_prof.py --reps 2` (two warm 20-iteration\n"
            "# c3 IRN-PICCS solves; shares, not absolutes, are comparable to the bench)"
            if "solver" in tag else
            "# cold-cache serialised launches of `bench.py --steps 2 --warmup 3 --skip-recon\n"
            "# --skip-cpu --skip-e2e --skip-fdk` (shares, not absolutes, are comparable to the bench)")
    lines = [f"# ncu launch list ({tag}): gpu__time_duration.sum, --clock-control none,", what,
             f"{'kernel':70s} {'n':>4s} {'total_ms':>10s} {'mean_ms':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:70]:70s} {len(v):4d} {sum(v):10.3f} {sum(v) / len(v):9.3f} "
                     f"{100 * sum(v) / tot:5.1f}%")
    # the step's own kernels: launched as often as the dominant kernel (once
    # per warm-up / timed step); setup kernels (nnz count, walk table) excluded
    top = max(agg.items(), key=lambda kv: sum(kv[1]))
    per_step = len(top[1])
    step = {k: v for k, v in agg.items() if len(v) == per_step}
    st = sum(sum(v) for v in step.values())
    lines += ["", f"# per bench step (kernels launched {per_step}x = once per step):",
              f"{'kernel':70s} {'mean_ms':>9s} {'share':>6s}"]
    for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:70]:70s} {sum(v) / len(v):9.3f} {100 * sum(v) / st:5.1f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(tag, rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        short = next((k for k in ("fwd_kernel", "adj_mirror_ws_kernel", "adj_mirror_kernel", "adj_brick_kernel") if k in name),
                     name.split("::")[-1].split("<")[0])
        lines = [f"# ncu --set full --clock-control none ({tag}): {name}",
                 "# c3 workload (tools/kprof.py): 256^3 @0.5 mm, 384^2 @0.5 mm, 60 views"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k:70s} {d[k]}")
        details = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "-k", d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]],
                                 capture_output=True, text=True).stdout
        open(os.path.join(PROF, f"{tag}_ncu_{short}.txt"), "w").write("\n".join(lines) + "\n")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            unit = rows[1][h.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            traffic[short] = (rd + wr) * scale
        except (KeyError, ValueError):
            pass
        print("\n".join(lines))
    if traffic:  # merged into the existing per-kernel table
        path = os.path.join(PROF, "ncu_traffic.json")
        allt = json.load(open(path)) if os.path.exists(path) else {}
        allt.update(traffic)
        json.dump(allt, open(path, "w"), indent=1)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    tag = sys.argv[1]
    launches(tag, sys.argv[2])
    full(tag, sys.argv[3])
