"""Summarise an .ncu-rep: headline metrics per kernel and the hottest SASS lines (stall samples)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "Compute (SM) Throughput",
        "Waves Per SM"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, regex=None, top=20):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    for r in rows[1:]:
        if r[mi] in WANT:
            print(r[ii], r[ki][:40], r[mi], r[vi], r[ui])
    if regex:
        src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}"]))))
        body = src[2:]
        tot = sum(int(r[2] or 0) for r in body if r[2].isdigit())
        print("stall samples", tot)
        hot = sorted(((int(r[2]), i) for i, r in enumerate(body) if r[2].isdigit()), reverse=True)[:top]
        for n, i in sorted(hot, key=lambda x: x[1]):
            ctx = " | ".join(body[j][1].strip()[:50] for j in range(max(0, i - 2), i + 1))
            print(f"{n:6d} {i:5d} {ctx}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
