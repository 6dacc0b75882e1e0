"""Summarise an ncu report (--page raw) into the metrics this project tracks.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for i, h in enumerate(hdr):
            if h in KEYS or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    v = vals[i]
                d[h] = (v, units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(d["kernel"][:120])
        stalls = {k: v for k, v in d.items() if "stalled" in k}
        for k, v in d.items():
            if k != "kernel" and "stalled" not in k:
                print(f"  {k:70s} {v[0]} {v[1]}")
        top = sorted(stalls.items(), key=lambda kv: -kv[1][0])[:6]
        print("  top stalls (per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v[0]:.2f}" for k, v in top))
    if "--traffic" in sys.argv:  # --traffic CFG OUT.json: per-launch DRAM bytes of the (first) kernel
        cfg, out = sys.argv[sys.argv.index("--traffic") + 1], sys.argv[sys.argv.index("--traffic") + 2]
        d = res[0]
        rd = d["dram__bytes_read.sum"][0] * (1e6 if d["dram__bytes_read.sum"][1].startswith("M") else
                                              1e9 if d["dram__bytes_read.sum"][1].startswith("G") else 1.0)
        wr = d["dram__bytes_write.sum"][0] * (1e6 if d["dram__bytes_write.sum"][1].startswith("M") else
                                               1e9 if d["dram__bytes_write.sum"][1].startswith("G") else 1.0)
        t = d["gpu__time_duration.sum"]
        with open(out, "w") as f:
            json.dump({"config": cfg, "kernel": d["kernel"], "dram_bytes_read": rd, "dram_bytes_write": wr,
                       "dram_bytes_per_launch": rd + wr, "duration_under_ncu": f"{t[0]} {t[1]}",
                       "source": f"ncu --set full --clock-control none, one launch ({sys.argv[1]})"}, f, indent=1)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
