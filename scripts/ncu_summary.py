#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of k_schur into a small JSON for profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep --config 4 --out profiles/r01/ncu_schur_cfg4.json
(reads the report with `ncu -i ... --page raw --csv`; no GPU needed)
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": a.report, "config": int(a.config) if a.config.isdigit() else a.config,
           "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None, "note": a.note}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                v = vals[i]
            out[name] = {"value": v, "unit": units[i]}
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
    rb = out.get("dram_read", {})
    wb = out.get("dram_write", {})
    if rb and wb:
        out["dram_bytes_per_launch"] = rb["value"] * scale.get(rb["unit"], 1) + wb["value"] * scale.get(wb["unit"], 1)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
