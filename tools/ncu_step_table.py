"""Per-launch table from an `ncu --set full` report of whole update steps: duration, grid, DRAM bytes,
L2 hit rate, tensor-pipe and SM throughput, achieved occupancy (markdown on stdout)."""
import csv
import io
import subprocess
import sys

METRICS = [("gpu__time_duration.sum", "us", 1.0), ("launch__grid_size", "grid", 1.0),
           ("dram__bytes_read.sum", "DRAM rd MB", None), ("dram__bytes_write.sum", "DRAM wr MB", None),
           ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
           ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor %", 1.0),
           ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1.0),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1.0)]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print("| # | kernel | " + " | ".join(m[1] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 2) + "|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("spz::", "").replace("unnamed>::", "")
        name = name.split("(")[0].replace("void ", "")[:40]
        vals = []
        for m, _, sc in METRICS:
            if m not in d:
                vals.append("-")
                continue
            v = float(d[m].replace(",", ""))
            u = units[h.index(m)]
            if sc is None:
                v *= SCALE.get(u, 1.0)
            elif m == "gpu__time_duration.sum":
                v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(u, 1.0)
            vals.append(f"{v:.3g}" if m != "launch__grid_size" else str(int(v)))
        print(f"| {d['ID']} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
