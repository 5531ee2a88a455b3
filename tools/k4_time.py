"""K4 timing / parity on arbitrary shapes (timing experiments; test infrastructure only).
usage: python tools/k4_time.py n l dp d1 d2 [reps] [--parity]
Times polya_schur (PAIR_TILES) with the library's phase events (precompute / assembly split) after a
256 MiB L2 flush, and with --parity compares the FULL G with the literal oracle (small n only)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402


def main():
    n, l, dp, d1, d2 = (int(v) for v in sys.argv[1:6])
    reps = int(sys.argv[6]) if len(sys.argv) > 6 and sys.argv[6].isdigit() else 5
    cfg = synth.small_config(n, l, dp, d1, d2)
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    ctx = pb.Polya(n, l, dp, d1, d2, A)
    X, W = synth.spd_blocks(n, ctx.nblocks, rng)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    out = {"shape": [n, l, dp, d1, d2], "lib": os.environ.get("POLYA_LIB", "default")}
    if "--parity" in sys.argv:
        from oracle import sdp as osdp
        P = osdp.build_problem(A, n, l, dp, d1, d2)
        G = ctx.schur(Xd, Wd).cpu().numpy()
        ref = osdp.schur_literal(P, X, W)
        out["parity_rel"] = float(np.linalg.norm(G - ref) / np.linalg.norm(ref))
    dims = ctx.dims
    N = dims["Ntil"]
    npl = dims["npairs_local"]
    G = torch.empty((max(npl, 1), N, N), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    ctx.set_timing(True)
    for _ in range(2):
        ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
    asm = []
    for _ in range(reps):
        flush.zero_()
        ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
        torch.cuda.synchronize()
        asm.append(ctx.timing())   # (ms precompute, ms assembly)
    ms = sorted(a[1] for a in asm)[len(asm) // 2]
    out["ms_assembly_median"] = ms
    out["tflops_assembly"] = dims["useful_flops_schur"] / (ms * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
