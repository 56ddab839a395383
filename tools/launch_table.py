"""Per-launch table from an `ncu --csv --log-file` metrics capture (one row per launch)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    launches = OrderedDict()
    for r in rows:
        k = r["ID"]
        d = launches.setdefault(k, {"name": r["Kernel Name"], "grid": r.get("Grid Size", "")})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        d[(r["Metric Name"], r["Metric Unit"])] = v
    return list(launches.values())


def short(name):
    n = name.replace("(anonymous namespace)::", "").replace("spz::", "")
    return n.split("(")[0][:44]


if __name__ == "__main__":
    ls = load(sys.argv[1])
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    count = int(sys.argv[3]) if len(sys.argv) > 3 else len(ls)
    tot = 0.0
    print("| # | kernel | us | grid | tensor % | DRAM rd MB | DRAM wr MB |")
    print("|---|---|---|---|---|---|---|")
    for i, d in enumerate(ls[first:first + count]):
        dur = next(v for (k, v) in d.items() if isinstance(k, tuple) and k[0] == "gpu__time_duration.sum")
        unit = next(k[1] for k in d if isinstance(k, tuple) and k[0] == "gpu__time_duration.sum")
        us = dur / 1000 if unit == "ns" else dur * (1000 if unit == "ms" else 1)
        tp = next((v for (k, v) in d.items() if isinstance(k, tuple) and k[0].startswith("sm__pipe_tensor")), 0)
        def mb(name):
            for k, v in d.items():
                if isinstance(k, tuple) and k[0] == name:
                    f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(k[1], 1e-6)
                    return v * f
            return 0
        grid = next((v for (k, v) in d.items() if isinstance(k, tuple) and k[0] == "launch__grid_size"), "")
        tot += us
        print(f"| {i} | `{short(d['name'])}` | {us:.1f} | {int(grid) if grid != '' else ''} | {tp:.1f} | {mb('dram__bytes_read.sum'):.2f} | {mb('dram__bytes_write.sum'):.2f} |")
    print(f"\nsum {tot:.1f} us over {count} launches")
