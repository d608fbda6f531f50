"""Per-source-line instruction / stall-sample totals from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
(ncu --page source --print-source cuda,sass; rows with a line number are
source-line aggregates.)"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          "regex:" + kern, "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], "", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or r[0] == "Function Name":
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")])
            ti = float(r[hdr.index("Thread Instructions Executed")])
            smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        rows.append((ie, ti, smp, f"{fname}:{r[0]}", r[1].strip()[:90]))
    tot_i = sum(x[0] for x in rows) or 1
    tot_s = sum(x[2] for x in rows) or 1
    print(f"total warp inst {tot_i:.3e}  samples {tot_s:.0f}")
    for ie, ti, smp, loc, src in sorted(rows, key=lambda x: -x[0])[:top]:
        print(f"{100*ie/tot_i:5.1f}% inst {100*smp/tot_s:5.1f}% smp  lanes {ti/max(ie,1):4.1f}  {loc:22s} {src}")


if __name__ == "__main__":
    main()
