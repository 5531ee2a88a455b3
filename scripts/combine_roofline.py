#!/usr/bin/env python
"""Per-rank roofline of the block-sharded Schur complement with its combine, from the
library's own plan (polya_plan: no GPU needed).  The profiling guide's rule for a fused compute +
collective kernel: target time = max(FLOPs / FP64 peak, NVLink bytes / link bandwidth); the fused P2P
combine adds the owner's ordered sum (its N slots of G/N: the partial's size read + G/N written,
HBM-bound); output-tile sharding moves no bytes.  Peaks: the measured FP64 DMMA figure
(profiles/r01_fp64_peak.json), MEASURED_PEAKS.json's copy bandwidth, the guide's measured 770 GB/s
NVLink peer copy per direction.
Usage: python scripts/combine_roofline.py > profiles/r02/combine_roofline.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402

FP64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")))["dmma_tflops_sustained"] * 1e12
try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
except Exception:
    HBM = 6.65e12
NVLINK = 770e9

out = {"peaks": {"fp64_flops": FP64, "hbm_bytes_s": HBM, "nvlink_bytes_s_per_direction": NVLINK}, "configs": {}}
for cid in (4, 5):
    cfg = synth.CONFIGS[cid]
    d = pb.plan(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    wg, part = d["useful_flops_schur"], d["tiles_bytes"]   # W_G; a rank's partial G (all pair tiles)
    rows = {}
    for N in (1, 2, 4, 8):
        t_fp = wg / N / FP64
        t_link = (N - 1) / N * part / NVLINK
        t_sum = (part + part / N) / HBM
        rows[N] = {"tiles_ms": 1e3 * t_fp,
                   "blocks_fused_ms": 1e3 * (max(t_fp, t_link) + t_sum),
                   "compute_ms": 1e3 * t_fp, "nvlink_ms": 1e3 * t_link, "owner_sum_ms": 1e3 * t_sum,
                   "bound": "nvlink" if t_link > t_fp else "fp64"}
    out["configs"][f"cfg{cid}"] = {"W_G": wg, "partial_bytes": part, "by_N": rows}
print(json.dumps(out, indent=1))
