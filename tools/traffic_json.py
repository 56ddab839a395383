"""profiles/r02_traffic.json from an `ncu --set full` capture of one WLK update (tools/r02_capture.sh): per kernel
class, DRAM bytes read / written per launch, duration and tensor-pipe utilisation (bench.py's roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

CLASSES = {"tc_mlp_kernel<256, 1": "actor_fwd_mlp", "tc_mlp_pair_kernel": "critic_fwd_mlp", "critic_loss_kernel": "critic_loss",
           "tc_gemm_kernel<256, 0, 1, 6": "critic_dgrad_gemm", "tc_actor_bwd_kernel": "actor_bwd_fused",
           "tc_gemm_kernel<256, 1, 1, 7": "wgrad_gemm", "adam_polyak_kernel": "adam_polyak", "gather_kernel": "gather"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("spz::", "").replace("unnamed>::", "")
        name = name.replace("void ", "").replace("(int)", "").replace("(bool)", "")
        cls = next((c for k, c in CLASSES.items() if k in name), None)
        if cls is None or cls in res:
            continue
        f = lambda m: float(d[m].replace(",", "")) * SCALE.get(u[m], 1)
        res[cls] = {"dram_read": int(f("dram__bytes_read.sum")), "dram_write": int(f("dram__bytes_write.sum")),
                    "duration_us": float(d["gpu__time_duration.sum"].replace(",", "")) * (1e-3 if u["gpu__time_duration.sum"] == "nsecond" else 1),
                    "tensor_pipe_pct": float(d.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "0").replace(",", "") or 0),
                    "kernel": name.split("(")[0].strip()[:60]}
    doc = {"source": "ncu --set full --import-source on --clock-control none -s 60 -c 8 -o full python bench.py --steps 5 "
                     "--warmup 3 --reps 1 --min-time 0 --no-cpu-baseline --no-e2e --no-fp32 (tools/r02_capture.sh; one B200, "
                     "round 2, final build; report not committed: 8 launches of one WLK update)",
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, cold L2 (ncu flushes caches before each replay); "
                   "writes of the launch stay in the 126 MB L2 and are not yet written back when the launch ends",
           "walker": res}
    json.dump(doc, open(out, "w"), indent=2)
    print(json.dumps(res, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
