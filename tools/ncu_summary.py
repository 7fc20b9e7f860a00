"""Summarise an `ncu --set full` capture of the step kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_vN.ncu-rep profiles/ncu_step_kernel.json \
        --W 16384 --rows 16384 --label "round 1, kernel vN"

Writes the JSON bench.py reads for roofline.traffic (DRAM bytes per launch)
plus the headline counters (duration, issue, pipe utilisation, stalls).
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--W", type=int, default=16384)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(hdr, units, vals):
        if k in KEYS or k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                "_per_issue_active.ratio"):
            try:
                x = float(v)
            except ValueError:
                continue
            d[k] = x * SCALE.get(u, 1)
    rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
    sites = a.W * a.rows
    out = {
        "label": a.label, "report": a.rep, "W": a.W, "rows": a.rows,
        "kernel_seconds": d.get("gpu__time_duration.sum"),
        "dram_bytes_per_launch": rd + wr,
        "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_bytes_per_site": (rd + wr) / sites,
        "algorithmic_bytes_per_site": 1.875,
        "warp_instructions_per_site": d.get("smsp__inst_executed.sum", 0) / sites,
        "metrics": d,
        "note": "cold-cache, serialised ncu replay (--clock-control none); dirty lines still "
                "in L2 at kernel end make the write count a little low for one launch",
    }
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("kernel_seconds", "dram_bytes_per_site",
                                           "warp_instructions_per_site")}))


if __name__ == "__main__":
    main()
