"""Per-source-line instruction / stall attribution of one kernel in an ncu report.

    python profiles/ncu_lines.py report.ncu-rep [top_n]
"""
import collections
import csv
import io
import subprocess
import sys


def lines(path, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    src = {}
    cur = None
    iex = ist = None
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            iex = r.index("Instructions Executed")
            ist = r.index("Warp Stall Sampling (All Samples)")
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        try:
            agg[(cur, ln)][0] += float(r[iex] or 0)
            agg[(cur, ln)][1] += float(r[ist] or 0)
        except (ValueError, TypeError):
            pass
        src[(cur, ln)] = r[1][:90]
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {ti:.3e}")
    for (f, ln), (i, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"inst {i / ti * 100:5.1f}%  stall {s / ts * 100:5.1f}%  {f}:{ln}  {src[(f, ln)]}")


if __name__ == "__main__":
    lines(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
