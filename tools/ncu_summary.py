"""Per-kernel summary CSV (+ traffic.json entries) from an `ncu --set full` report.

usage: python tools/ncu_summary.py report.ncu-rep out.csv [traffic.json [workload]]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "math_pipe_throttle", "mio_throttle", "wait",
          "lg_throttle", "not_selected", "selected"]
# bench.py kernel classes -> kernel-name prefixes
CLASSES = {"update": ("k_pass2_fused", "k_pass2_m8"), "contract_A": ("k_pass1",)}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    stall_metrics = [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS + stall_metrics)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    cols = [c for c in METRICS + stall_metrics if c in hdr]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["Kernel Name"] + [c.replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", "") for c in cols])
        w.writerow([""] + [units[hdr.index(c)] for c in cols])
        traffic = {}
        for r in rows[2:]:
            w.writerow([r[name_i]] + [r[hdr.index(c)] for c in cols])
            name = r[name_i].split("(")[0].replace("void ", "").replace("pasd::", "")
            rd, wr = float(r[hdr.index("dram__bytes_read.sum")]), float(r[hdr.index("dram__bytes_write.sum")])
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            b = rd * scale[units[hdr.index("dram__bytes_read.sum")]] + wr * scale[units[hdr.index("dram__bytes_write.sum")]]
            for cls, prefixes in CLASSES.items():
                if name.startswith(prefixes):
                    traffic.setdefault(cls, []).append(b)
    if len(sys.argv) > 3:  # merged into the file under the workload's name (bench.py keys it that way)
        wl = sys.argv[4] if len(sys.argv) > 4 else "c5_1000cube_r50"
        try:
            tj = json.load(open(sys.argv[3]))
        except (OSError, ValueError):
            tj = {}
        tj["_source"] = (f"ncu --set full --clock-control none ({rep}): dram__bytes_read.sum + "
                         "dram__bytes_write.sum per launch, mean over the captured launches of the class")
        tj["_keys"] = ("workload name -> kernel class -> DRAM bytes per launch; a workload or class not captured "
                       "is absent and bench.py reports roofline.traffic = null")
        tj[wl] = {cls: sum(v) / len(v) for cls, v in traffic.items()}
        with open(sys.argv[3], "w") as f:
            json.dump(tj, f, indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
