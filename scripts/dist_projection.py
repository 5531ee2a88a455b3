#!/usr/bin/env python
"""Projected time of the distributed factorisation (SHARD_CYCLIC) of config 5's
Schur complement (L0 = 21 tile rows of Ntil = 7260) on N = 1, 2, 4, 8 GPUs.

The per-tile operations are timed on the one available B200 with the library routines the
factorisation calls (cuSOLVER potrf, cuBLAS trsm / dgemm, reached here through torch, which calls
the same routines; syrk is charged as half a gemm), then the schedule of dist_potrf is replayed:
step k = owner's potrf, the broadcast of L_kk and the raw panel ((L0-k-1) tiles at an assumed NCCL
broadcast bandwidth), the panel solves split over the ranks (ceil((L0-k-1)/N) trsm on the busiest),
the broadcast of the solved tiles, then the slowest rank's trailing update of its own block
columns.  The schedule with all panel solves on the owner (the first version) is replayed beside it,
and the look-ahead schedule dist_potrf runs since round 2 (an event simulation: per rank one compute
engine; the panel work (potrf, trsm share) goes ahead of queued update work, which runs in stream
order -- block column k+1 of step k, then the rest of step k; broadcasts on the links at the assumed
bandwidth -- so step k+1's panel overlaps the rest of step k's trailing update).  A projection, not a multi-GPU measurement.
Usage: python scripts/dist_projection.py [bcast_GBps] [--timings FILE.json]   (JSON on stdout; with
--timings the per-tile times come from an earlier run's JSON instead of being measured)"""
import json
import sys

import torch

BW = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 400.0   # GB/s, NCCL broadcast over NVLink 5 (assumed)
T, N = 21, 7260


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


if "--timings" in sys.argv:
    prev = json.load(open(sys.argv[sys.argv.index("--timings") + 1]))
    t_potrf, t_trsm, t_gemm = prev["s_potrf"], prev["s_trsm"], prev["s_gemm"]
else:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g)
    S = A @ A.T / N + torch.eye(N, dtype=torch.float64, device="cuda")
    L = torch.linalg.cholesky(S)
    B = torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty_like(B)
    t_potrf = timed(lambda: torch.linalg.cholesky(S))
    t_trsm = timed(lambda: torch.linalg.solve_triangular(L, B.T, upper=False))
    t_gemm = timed(lambda: torch.matmul(A, B.T, out=C))
t_syrk = 0.5 * t_gemm
tile_bytes = N * N * 8

out = {"L0": T, "Ntil": N, "tile_GB": tile_bytes / 1e9, "bcast_GBps_assumed": BW,
       "s_potrf": t_potrf, "s_trsm": t_trsm, "s_gemm": t_gemm, "s_syrk_charged": t_syrk,
       "gemm_tflops": 2 * N ** 3 / t_gemm / 1e12, "runs": {}}
def replay(world, split):
    total = comm = 0.0
    for k in range(T):
        nq = T - k - 1
        one = 0.0 if world == 1 else tile_bytes / (BW * 1e9)
        if split:   # potrf; bcast L_kk + raw panel; split trsm; bcast solved tiles
            panel = t_potrf + -(-nq // world) * t_trsm
            bc = (1 + 2 * nq) * one if nq else 0.0
        else:       # potrf + all trsm on the owner; bcast solved panel
            panel = t_potrf + nq * t_trsm
            bc = nq * one
        upd = [0.0] * world
        for j in range(k + 1, T):
            upd[j % world] += t_syrk + (T - j - 1) * t_gemm
        total += panel + bc + max(upd)
        comm += bc
    return total, comm


def replay_lookahead(world):
    """Event simulation of dist_potrf with look-ahead (see the module docstring)."""
    one = 0.0 if world == 1 else tile_bytes / (BW * 1e9)
    free = [0.0] * world                 # each rank's compute engine
    col_ready = [0.0] * (T + 1)          # block column k fully updated (on its owner)
    upd_queue = [[] for _ in range(world)]   # (ready time, duration) of pending update work per rank
    def run_updates(r, until):
        """Run rank r's queued update work that is ready, while the engine is free before `until`."""
        while upd_queue[r] and max(free[r], upd_queue[r][0][0]) < until:
            ready, dur, tag = upd_queue[r].pop(0)
            free[r] = max(free[r], ready) + dur
            if tag is not None:
                col_ready[tag] = free[r]
    for k in range(T):
        o = k % world
        nq = T - k - 1
        # the owner factors L_kk as soon as column k is updated (its engine runs queued updates first,
        # but the column-k update was queued ahead of the rest, so it is done at col_ready[k])
        start = max(col_ready[k], 0.0)
        run_updates(o, start)
        free[o] = max(free[o], start) + t_potrf
        if nq == 0:
            break
        arrive = free[o] + (1 + nq) * one    # L_kk and the raw panel reach every rank
        done = []
        for r in range(world):
            ntr = len(range(r, nq, world))
            run_updates(r, arrive)
            free[r] = max(free[r], arrive) + ntr * t_trsm
            done.append(free[r])
        solved = max(done) + nq * one        # the solved tiles reach every rank
        for r in range(world):
            col1 = [(solved, t_syrk + (T - (k + 1) - 1) * t_gemm, k + 1)] if (k + 1) % world == r else []
            rest = sum(t_syrk + (T - j - 1) * t_gemm for j in range(k + 2, T) if j % world == r)
            # one in-order update stream per rank (as in dist_potrf): column k+1, then the rest of step k,
            # behind whatever of step k-1 is still queued
            upd_queue[r] = upd_queue[r] + col1 + ([(solved, rest, None)] if rest else [])
    for r in range(world):
        run_updates(r, float("inf"))
    return max(free)


for world in (1, 2, 4, 8):
    t_split, c_split = replay(world, True)
    t_owner, c_owner = replay(world, False)
    out["runs"][str(world)] = {"s_factorisation": t_split, "s_broadcast": c_split,
                               "s_factorisation_owner_trsm": t_owner,
                               "s_factorisation_lookahead": replay_lookahead(world)}
base = out["runs"]["1"]["s_factorisation"]
for w, r in out["runs"].items():
    r["speedup"] = base / r["s_factorisation"]
    r["efficiency"] = r["speedup"] / int(w)
    r["efficiency_owner_trsm"] = base / r["s_factorisation_owner_trsm"] / int(w)
    r["efficiency_lookahead"] = base / r["s_factorisation_lookahead"] / int(w)
print(json.dumps(out))
