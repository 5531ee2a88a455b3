#!/usr/bin/env python
"""Benchmark of the Polya/SDP hot path on B200 (BASELINE.json metric:
"Schur-complement assembly FP64 TFLOP/s and s per IPM iteration, 1/2/4/8 B200").

One *step* = one pass of the per-iteration hot path over the workload:
    polya_apply (B^T(y)), polya_adjoint (B(X)), polya_schur (SCM precompute + assembly of G)
on config 4 (n=100, l=4, dp=2, d1=d2=4; K=50,500, 204 Polya blocks) by default.
value = W_G / t_step (TFLOP/s), W_G = n^4 (sum nu^2 + 4 sum mu^2) the algorithmic FP64 FLOPs
of the Schur assembly; t_step is the max over ranks.

Launch: python bench.py [--gpus N --steps K --warmup W --config 4|5 --shard tiles|blocks|cyclic]
        torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU; default output-tile
        sharding of G: no inter-GPU traffic on the data path, NCCL only for the barrier and the
        max-over-ranks timing; --shard blocks: the paper's Polya-block partition with the partial
        G summed by NCCL ReduceScatter inside the step; --shard cyclic: the column-cyclic pair
        tiles of the distributed factorisation, whose IPM iteration is then timed at any N)
        python bench.py --impl reference ...   (the CPU oracle, rank 0 only)
The JSON line also carries the roofline of the dominant kernel (K4), the CPU-oracle baseline,
an end-to-end figure through the public API (pinned host inputs in, all of G back out, streamed
during the assembly), the seconds per IPM iteration (N = 1, or any N with --shard cyclic) and the SM clocks sampled during
the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Schur-complement assembly FP64 TFLOP/s"
UNIT = "TFLOP/s"
PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
NCU_FILE = os.path.join(ROOT, "profiles", "ncu_schur_latest.json")


def counts(cfg):
    """(L0, L, M) by Eq. (2) -- bench bookkeeping only (the library reports its own dims)."""
    from math import comb
    f = lambda l, d: comb(l + d - 1, l - 1)  # noqa: E731
    return f(cfg.l, cfg.dp), f(cfg.l, cfg.dp + cfg.d1), f(cfg.l, cfg.dp + 1 + cfg.d2)


def workload_name(cfg, cid):
    return (f"cfg{cid}: n={cfg.n}, l={cfg.l}, dp={cfg.dp}, da=1, d1={cfg.d1}, d2={cfg.d2} "
            f"({cfg.recipe} A_i, Wishart(n+5) X_b, Z_b^-1)")


def fp64_peak():
    try:
        d = json.load(open(PEAK_FILE))
        return float(d["dmma_tflops_sustained"]), "measured DMMA m8n8k4 f64 sustained (profiles/r01_fp64_peak.json)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal 148 SM x 64 FP64 FMA/clk x 1.965 GHz"


def hbm_peak():
    """MEASURED_PEAKS.json's copy bandwidth (GB/s), else the profiling guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------------
def oracle_rate(cfg, A, X, W, seconds, min_entries=4, seed=123, P=None):
    """Time the oracle (as it stands) computing literal G entries (Eq. T2, one trace product per
    block) on a bounded random sample; credit each entry with the algorithmic W_G / #entries of
    the upper triangle.  Returns (problem, entries, seconds, build_s)."""
    from oracle import sdp as osdp
    t0 = time.perf_counter()
    if P is None:
        P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    done, t_used = 0, 0.0
    while t_used < seconds or done < min_entries:
        i, j = (int(v) for v in rng.integers(0, P.K, size=2))
        t1 = time.perf_counter()
        osdp.schur_entries(P, X, W, [(min(i, j), max(i, j))])
        t_used += time.perf_counter() - t1
        done += 1
    return P, done, t_used, build_s


def oracle_rate_structured(cfg, A, X, W, seconds, seed=123, P=None, min_pairs=1):
    """Time the oracle's structured Schur assembly (oracle.sdp.schur_structured, SURVEY 8(c) O6'(iii):
    per pair (h, h') one library matmul over the rank-structured terms + the orientation fold) on a
    seeded random sample of pairs until `seconds` elapse; credit each pair with its share of W_G
    ((1 or 2) n^4 K_pair, K_pair = 4 mu + nu, the same count as the GPU's).  Returns
    (problem, flops credited, seconds, pairs done, build seconds)."""
    from oracle import sdp as osdp
    t0 = time.perf_counter()
    if P is None:
        P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    build_s = time.perf_counter() - t0
    pairs = [(h, h2) for h in range(P.L0) for h2 in range(h, P.L0)]
    order = np.random.default_rng(seed).permutation(len(pairs))
    actH = [[bool(np.any(P.H[h, m])) for m in range(P.M)] for h in range(P.L0)]
    n4 = float(P.n) ** 4
    flops, t_used, done = 0.0, 0.0, 0
    for q in order:
        if t_used >= seconds and done >= min_pairs:
            break
        h, h2 = pairs[q]
        mu = sum(actH[h][m] and actH[h2][m] for m in range(P.M))
        nu = int(((P.beta[h] != 0) & (P.beta[h2] != 0)).sum())
        t1 = time.perf_counter()
        osdp.schur_structured(P, X, W, pairs=[(h, h2)])
        t_used += time.perf_counter() - t1
        flops += (1.0 if h == h2 else 2.0) * n4 * (4 * mu + nu)
        done += 1
    return P, flops, t_used, done, build_s


def wg_flops(P):
    nu2 = sum(int((P.beta[:, j] != 0).sum()) ** 2 for j in range(P.L))
    mu2 = sum(int(sum(np.any(P.H[h, m] != 0) for h in range(P.L0))) ** 2 for m in range(P.M))
    return float(P.n) ** 4 * (nu2 + 4 * mu2)


def run_reference(args, cfg, cid):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    L0, L, M = counts(cfg)
    A, X, W = synth.make_case(cfg, L + M, seed=0)
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    P, _, _, _, _ = oracle_rate_structured(cfg, A, X, W, seconds=0.0)
    for w in range(args.warmup):
        oracle_rate_structured(cfg, A, X, W, seconds=0.0, P=P, seed=w)
    rates, times = [], []
    for s_ in range(args.steps):
        _, fl, t_used, done, _ = oracle_rate_structured(cfg, A, X, W, seconds=per_step, P=P, seed=1000 + s_)
        rates.append(fl / t_used / 1e12)
        times.append(t_used)
    value = statistics.mean(rates)
    cores = blas_threads()
    sample = (f"{args.steps} steps x ~{per_step:.0f} s of the oracle's structured Schur assembly "
              f"(oracle.sdp.schur_structured) on random pairs (h,h') of {workload_name(cfg, cid)}, credited "
              "(1|2) n^4 K_pair per pair")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(cfg, cid), "K": P.K, "nblocks": P.nblocks},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in out.strip().splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def reduce_over_ranks(x, op, device, world):
    """Max / sum of a per-rank scalar over the process group (NCCL on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def start_watchdog(seconds, emit, exit_fn=None):
    """Daemon timer for a leg that may hang inside a collective: after `seconds` it calls emit() (rank 0
    prints the JSON line with the leg marked as timed out) and ends the process with status 0 on its
    own clock (os._exit: a thread blocked in NCCL cannot be unwound).  cancel() it when the leg ends."""
    import threading

    def fire():
        try:
            emit()
        finally:
            sys.stdout.flush()
            sys.stderr.flush()
            (exit_fn or os._exit)(0)

    t = threading.Timer(seconds, fire)
    t.daemon = True
    t.start()
    return t


def run_gpu(args, cfg, cid):
    import torch
    import torch.distributed as dist

    import paper_1411_3769_b200 as pb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:   # NCCL INIT lines (comm nranks, NVLS / NVLink transport) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return reduce_over_ranks(x, "max", dev, world)

    def sum_over_ranks(x):
        return reduce_over_ranks(x, "sum", dev, world)

    L0, L, M = counts(cfg)
    A, X, W = synth.make_case(cfg, L + M, seed=0)
    t0 = time.perf_counter()
    blocks = args.shard == "blocks"
    cyclic = args.shard == "cyclic"
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=world,
                   shard=pb.SHARD_BLOCKS if blocks else pb.SHARD_CYCLIC if cyclic else pb.SHARD_TILES)
    setup_s = time.perf_counter() - t0
    if blocks or cyclic:   # NCCL communicator of the library (id from rank 0, distributed over the process group)
        uid = [pb.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0])
    p2p = blocks and args.combine == "p2p"
    if p2p:   # fused combine: exchange the receive slots' IPC handles, K4 stores into the owners' slots
        mine = ctx.p2p_export()
        hs = [None] * world
        if world > 1:
            dist.all_gather_object(hs, mine)
        else:
            hs = [mine]
        ctx.p2p_import(hs)
    K, N = ctx.K, ctx.Ntil
    npl = ctx.dims["npairs_local"]
    wg_rank = ctx.dims["useful_flops_schur"]
    wg_total = sum_over_ranks(wg_rank)
    wg_one = pb.plan(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)["useful_flops_schur"]   # the whole problem, one rank
    if abs(wg_total - wg_one) > 1e-9 * wg_one:
        raise SystemExit(f"bench.py: the ranks' shares sum to W_G = {wg_total:.6e}, the problem has {wg_one:.6e}")

    Xd = torch.from_numpy(X).to(dev)
    Wd = torch.from_numpy(W).to(dev)
    y = torch.from_numpy(np.random.default_rng(1).normal(size=K)).to(dev)
    if blocks:   # this rank's summed tiles (the partial G lives in two library-owned group slots)
        G = None
        Grecv = torch.empty(ctx.dims["reduce_count"], dtype=torch.float64, device=dev)
    else:
        G = torch.empty((max(npl, 1), N, N), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # 256 MiB > 126 MB L2
    ctx.set_timing(True)

    # B^T(y) and B(X) do not depend on G and share no workspace with the Schur assembly (separate arena
    # slots): they run on a side stream next to the precompute/assembly and join before the step ends
    side = torch.cuda.Stream(device=dev)
    Bt_buf = torch.empty((ctx.nblocks, ctx.bn, ctx.bn), dtype=torch.float64, device=dev)
    yv_buf = torch.empty(K, dtype=torch.float64, device=dev)

    def step():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        Bt = ctx.apply(y, out=Bt_buf, stream=side)
        yv = ctx.adjoint(Xd, out=yv_buf, stream=side)
        if p2p:      # fused: the assembly writes each partial tile into its owner's slot, owners sum
            ctx.schur_reduce_p2p(Xd, Wd, out=Grecv)
        elif blocks:   # pipelined: each tile group's ReduceScatter overlaps the next group's assembly
            ctx.schur_reduce(Xd, Wd, out=Grecv)
        else:
            ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
        cur.wait_stream(side)
        return Bt, yv

    for _ in range(args.warmup):
        step()
    if args.graph:   # the whole step as one CUDA graph (the library's calls are stream-ordered and capturable)
        if blocks:
            raise SystemExit("--graph: not with --shard blocks")
        torch.cuda.synchronize()
        ctx.set_timing(False)   # the phase events are not recorded inside the graph: time the whole step
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        step = graph.replay   # noqa: F811
        for _ in range(args.warmup):
            step()
    barrier()
    clk = ClockSampler(local)
    launches0 = ctx.launch_count()
    step_ms, pre_ms, asm_ms, comb_ms = [], [], [], []
    clk.start()
    time.sleep(0.3)
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        if args.graph:   # the step as a whole (the assembly dominates it beyond config 2)
            p, a = 0.0, e0.elapsed_time(e1)
        else:
            p, a = ctx.timing()                 # this step's schur events
        step_ms.append(e0.elapsed_time(e1))
        pre_ms.append(p)
        asm_ms.append(a)
        if blocks:
            comb_ms.append(ctx.combine_timing())
    barrier()
    clocks = clk.stop()
    launches = ctx.launch_count() - launches0
    launches_per_step = launches / args.steps

    t_step = max_over_ranks(statistics.mean(step_ms))
    t_asm_rank = statistics.mean(asm_ms)
    t_pre = max_over_ranks(statistics.mean(pre_ms))
    t_asm = max_over_ranks(t_asm_rank)
    t_comb = max_over_ranks(statistics.mean(comb_ms)) if blocks else 0.0
    value = wg_total / (t_step * 1e-3) / 1e12

    # ---- end to end through the public API: host (pinned) inputs -> device -> G back to host ----
    # G is streamed back in pair chunks while later chunks are assembled (polya_schur_prepare +
    # polya_schur_assemble on the compute stream, D2H copies on a second stream after each chunk's
    # event), so the PCIe transfer of the 11+ GB result overlaps the assembly.
    e2e = e2e_resident = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        Wh = torch.from_numpy(W).pin_memory()
        yh = y.cpu().pin_memory()
        Gres = Grecv if blocks else G          # the step's result on this rank
        Gh = torch.empty(Gres.shape, dtype=torch.float64).pin_memory()
        h2d = Xh.numel() * 8 + Wh.numel() * 8 + yh.numel() * 8
        d2h = Gh.numel() * 8
        comp = torch.cuda.current_stream()
        copy = torch.cuda.Stream()
        nch = 8 if (not blocks and npl >= 8) else 1
        cuts = [npl * q // nch for q in range(nch + 1)]
        barrier()
        e2e_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(comp)
            Xd.copy_(Xh, non_blocking=True)
            Wd.copy_(Wh, non_blocking=True)
            y.copy_(yh, non_blocking=True)
            ctx.apply(y)
            ctx.adjoint(Xd)
            if blocks:
                if p2p:
                    ctx.schur_reduce_p2p(Xd, Wd, out=Grecv)
                else:
                    ctx.schur_reduce(Xd, Wd, out=Grecv)
                Gh.copy_(Grecv, non_blocking=True)
                e1.record(comp)
            else:
                ctx.schur_prepare(Xd, Wd)
                for a_, b_ in zip(cuts[:-1], cuts[1:]):
                    ctx.schur_assemble(G, a_, b_, layout=pb.G_PAIR_TILES)
                    ev = torch.cuda.Event()
                    ev.record(comp)
                    copy.wait_event(ev)
                    with torch.cuda.stream(copy):
                        Gh[a_:b_].copy_(G[a_:b_], non_blocking=True)
                e1.record(copy)
            e1.synchronize()
            comp.wait_stream(copy)
            e2e_ms.append(e0.elapsed_time(e1))
        barrier()
        te = max_over_ranks(statistics.mean(e2e_ms))
        e2e = {"value": wg_total / (te * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": te,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "d2h_overlap": f"G streamed back in {nch} pair chunks while later chunks are assembled"}
        # the same public calls as in the IPM loop, where G is consumed on the device by the factorisation:
        # host inputs in every step, the step's small outputs (B^T(y), B(X)) back; G stays resident
        Bt = ctx.apply(y)
        Bh = torch.empty(Bt.shape, dtype=torch.float64).pin_memory()
        yvh = torch.empty(K, dtype=torch.float64).pin_memory()
        barrier()
        res_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            Xd.copy_(Xh, non_blocking=True)
            Wd.copy_(Wh, non_blocking=True)
            y.copy_(yh, non_blocking=True)
            ctx.apply(y, out=Bt)
            yv = ctx.adjoint(Xd)
            if p2p:
                ctx.schur_reduce_p2p(Xd, Wd, out=Grecv)
            elif blocks:
                ctx.schur_reduce(Xd, Wd, out=Grecv)
            else:
                ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
            Bh.copy_(Bt, non_blocking=True)
            yvh.copy_(yv, non_blocking=True)
            e1.record()
            e1.synchronize()
            res_ms.append(e0.elapsed_time(e1))
        barrier()
        tr = max_over_ranks(statistics.mean(res_ms))
        e2e_resident = {"value": wg_total / (tr * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": tr,
                        "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(Bh.numel() * 8 + yvh.numel() * 8),
                        "note": "inputs X, Z^-1, y from pinned host memory every step; B^T(y) and B(X) read back; G "
                                "stays on the device, where the IPM's factorisation consumes it (e2e_full_G also "
                                "copies all of G back)"}
        del Gh, Gres, Bh, yvh

    # ---- the per-iteration operators alone (HBM-bound for small n, FP64-bound for large):
    # algorithmic FLOPs (2 n^3 per nonzero H_{h,m} product, 2 n^2 per beta term) and compulsory HBM bytes
    # (inputs read once, outputs written once), each call timed with CUDA events after an L2 flush
    operators = None
    if flush is not None:
        d = ctx.dims
        n_ = cfg.n
        ops = {"apply": (lambda: ctx.apply(y), 2 * n_ ** 3 * d["nnz_H"] + 2 * n_ * n_ * d["nnz_beta"],
                         8 * (K + d["nnz_H"] * n_ * n_ + ctx.nblocks * n_ * n_)),
               "adjoint": (lambda: ctx.adjoint(Xd), 2 * n_ ** 3 * d["nnz_H"] + 2 * N * (d["nnz_H"] + d["nnz_beta"]),
                           8 * (ctx.nblocks * n_ * n_ + d["nnz_H"] * n_ * n_ + K))}
        operators = {"peaks": {"fp64_tflops": fp64_peak()[0], "hbm_gbs": hbm_peak()[0], "hbm_source": hbm_peak()[1]}}
        FP64_PEAK, HBM_PEAK = fp64_peak()[0], hbm_peak()[0]
        for name, (fn, flops, nbytes) in ops.items():
            ts = []
            for _ in range(5):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = max_over_ranks(statistics.median(ts))
            operators[name] = {"ms": t, "tflops": flops / (t * 1e-3) / 1e12, "gbs": nbytes / (t * 1e-3) / 1e9,
                               "frac_fp64": flops / (t * 1e-3) / 1e12 / FP64_PEAK, "frac_hbm": nbytes / (t * 1e-3) / 1e9 / HBM_PEAK,
                               "algorithmic_flops": flops, "compulsory_bytes": nbytes}

    def make_line(ipm, cpu):
        peak, peak_src = fp64_peak()
        achieved = wg_rank / (t_asm_rank * 1e-3) / 1e12
        traffic = None
        try:
            nc = json.load(open(NCU_FILE))
            if nc.get("config") == cid:
                traffic = nc.get("dram_bytes_per_launch")
        except Exception:
            pass
        return {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded synth/ generators; SURVEY 8(d))",
            "config": {"workload": workload_name(cfg, cid), "K": K, "nblocks": ctx.nblocks, "L0": ctx.L0,
                       "W_G": wg_one, "W_G_sum_over_ranks": wg_total,
                       "step": "polya_apply + polya_adjoint (side stream) + " + (
                           "polya_schur_reduce_p2p (precompute + assembly storing each partial tile into its "
                           "owner's slot over peer memory + the owners' ordered sums)" if p2p else
                           "polya_schur_reduce (precompute + assembly by tile groups, each group's NCCL "
                           "ReduceScatter on a comm stream overlapping the next group)" if blocks else
                           "polya_schur (precompute + assembly)"),
                       "layout": "G pair tiles (upper, row-panel ready)",
                       "cuda_graph": bool(args.graph),
                       "parallelism": (f"Polya-block shards x{world} + NCCL ReduceScatter of partial G" if blocks
                                       else f"column-cyclic pair-tile shards x{world} (distributed factorisation)"
                                       if cyclic else f"output-tile shards x{world}"),
                       "l2": "256 MiB memset between timed steps (outside the events); G write alone is "
                             f"{npl * N * N * 8 / 1e9:.1f} GB/step"},
            "breakdown_ms": {"schur_precompute": t_pre, "schur_assembly": t_asm,
                             "combine_nccl_exposed": t_comb,
                             "apply_adjoint_and_rest": t_step - t_pre - t_asm - t_comb, "setup_once_s": setup_s},
            "tflops_schur_assembly_only": wg_total / (t_asm * 1e-3) / 1e12,
            "roofline": {"bound": "tensor", "kernel": "k_schur (K4, FP64 DMMA)", "achieved": achieved, "peak": peak,
                         "unit": UNIT, "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_flops_per_launch": wg_rank, "peak_source": peak_src},
            "cpu_baseline": cpu,
            # e2e: the public calls of one Algorithm 2 iteration's operator work as the IPM makes them --
            # host inputs in, the step's host-side results out, G consumed on the device by the
            # factorisation; e2e_full_G: all of G back to the host as well (PCIe-bound)
            "e2e": e2e_resident,
            "e2e_full_G": e2e,
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "gpu_launches_per_step": launches_per_step,
            "clocks": clocks,
            "ipm_iteration": ipm,
            "operators": operators,
        }

    # ---- seconds per IPM iteration (Algorithm 2 step via polya_ipm_step) at every N: one rank uses the
    # dense (or, for config 5, tiled) factorisation; N > 1 ranks factor G distributed (SHARD_CYCLIC:
    # column-cyclic pair tiles, NCCL panel broadcasts) ----
    ipm = None
    watchdog = None
    if not args.no_ipm:
        # The N > 1 IPM leg runs the library's own NCCL communicator (panel broadcasts of the distributed
        # factorisation).  A hang there must not cost the Schur line measured above: after --ipm-timeout
        # seconds every rank gives up on its own clock, rank 0 prints the line with the IPM leg marked as
        # timed out, and all ranks exit.
        watchdog = start_watchdog(
            args.ipm_timeout,
            lambda: print(json.dumps(make_line({"error": f"IPM leg timed out after {args.ipm_timeout:g} s "
                                                         f"({world} rank(s))", "n_ranks": world}, None)),
                          flush=True) if rank == 0 else None)
        del G
        flush = None
        if blocks:
            del Grecv
        torch.cuda.empty_cache()
        ictx = ctx
        if world > 1 and not cyclic:   # the IPM context of N ranks: the distributed factorisation
            ictx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=world, shard=pb.SHARD_CYCLIC)
            uid = [pb.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ictx.nccl_init(uid[0])
        elif blocks:                   # one rank, block-sharded context: a plain one for the IPM leg
            ictx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
        Xi = torch.eye(cfg.n, dtype=torch.float64, device=dev).repeat(ictx.nblocks, 1, 1).contiguous()
        Zi = Xi.clone()
        yi = torch.zeros(K, dtype=torch.float64, device=dev)
        mu = 1.0 / 3.0                                                 # reading R4 at X = Z = I
        runs = []
        for it in range(2):                                            # the first call allocates G
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            st = ictx.ipm_step(Xi, Zi, yi, mu, it)
            e1.record()
            e1.synchronize()
            mu = st["mu"]
            runs.append((e0.elapsed_time(e1), st))
        ms, st = runs[-1]
        ms = max_over_ranks(ms)
        tiled = ictx.K * ictx.K * 8 > 0.45 * torch.cuda.get_device_properties(dev).total_memory
        dist_f = world > 1 or cyclic
        ipm = {"s_per_iteration": ms / 1e3, "n_ranks": world, "ms_schur": max_over_ranks(st["ms_schur"]),
               "ms_factorisation": max_over_ranks(st["ms_factor"]), "ms_other": max_over_ranks(st["ms_other"]),
               "factorisation": (f"distributed blocked Cholesky over {world} rank(s) (column-cyclic pair tiles, NCCL "
                                 "panel broadcasts, split panel solves; DESIGN.md 7.1)" if dist_f else
                                 "blocked Cholesky on the pair tiles (cuSOLVER dpotrf on diagonal tiles, cuBLAS "
                                 "dtrsm/dsyrk/dgemm) + blocked solves" if tiled else
                                 "cuSOLVER dpotrf + 2 dpotrs on the K x K SCM (FULL)"),
               "iteration_measured": 2, "gap": st["gap"], "tp": st["tp"], "td": st["td"]}
        # the factorisation against the FP64 roofline: K^3/3 flops of the Cholesky of the K x K SCM
        fl_chol = float(ictx.K) ** 3 / 3.0
        ipm["factorisation_tflops"] = fl_chol / (ipm["ms_factorisation"] * 1e-3) / 1e12
        ipm["factorisation_frac_fp64"] = ipm["factorisation_tflops"] / (fp64_peak()[0] * world)
        if ictx is not ctx:
            ictx.close()
        watchdog.cancel()

    # ---- CPU oracle baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        P, fl, t_used, done, build_s = oracle_rate_structured(cfg, A, X, W, seconds=args.cpu_seconds)
        _, ent, t_lit, _ = oracle_rate(cfg, A, X, W, seconds=min(3.0, args.cpu_seconds), P=P)
        per_entry = wg_total / (K * (K + 1) / 2)
        one = None
        try:   # the same oracle on one host thread (1 thread and all threads)
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                _, fl1, t1, done1, _ = oracle_rate_structured(cfg, A, X, W, seconds=min(6.0, args.cpu_seconds), P=P,
                                                              seed=321)
            one = {"value": fl1 / t1 / 1e12, "cores": 1, "sample": f"{done1} pair tiles in {t1:.1f} s"}
        except Exception as exc:   # threadpoolctl missing: say so
            one = {"unavailable": str(exc)}
        cpu = {"value": fl / t_used / 1e12, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
               "one_thread": one,
               "sample": f"{done} pair tiles (h,h') of G by the oracle's structured assembly (oracle.sdp."
                         f"schur_structured: one library matmul per pair + orientation fold) in {t_used:.1f} s, "
                         f"credited (1|2) n^4 K_pair each; oracle set-up {build_s:.1f} s excluded",
               "literal_entries_tflops": per_entry * ent / t_lit / 1e12,
               "literal_sample": f"{ent} literal G entries (Eq. T2, oracle.sdp.schur_entries) in {t_lit:.1f} s"}

    if rank == 0:
        print(json.dumps(make_line(ipm, cpu)), flush=True)
    barrier()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="tiles", choices=["tiles", "blocks", "cyclic"],
                    help="tiles: output-tile sharding, no data-path collective (default); blocks: the paper's "
                         "Polya-block sharding with the partial G summed by NCCL ReduceScatter; cyclic: "
                         "column-cyclic pair tiles, the layout of the distributed factorisation (IPM leg at any N)")
    ap.add_argument("--combine", default="nccl", choices=["nccl", "p2p"],
                    help="--shard blocks: the pipelined NCCL reduce-scatters (default) or the fused P2P combine "
                         "(K4 stores each partial tile into its owner's slot over NVLink peer memory)")
    ap.add_argument("--graph", action="store_true",
                    help="capture the step (apply + adjoint + schur) once as a CUDA graph and replay it (small configs "
                         "are launch-bound)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ipm", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ipm-timeout", type=float, default=None,
                    help="seconds before the IPM leg gives up (default 120; 1800 for config 5)")
    args = ap.parse_args()
    cid = int(args.config) if args.config.isdigit() else args.config
    cfg = synth.CONFIGS[cid]
    if args.ipm_timeout is None:
        args.ipm_timeout = 1800.0 if cid == 5 else 120.0
    if args.impl == "reference":
        return run_reference(args, cfg, cid)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)", file=sys.stderr)
        return 2
    return run_gpu(args, cfg, cid)


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: re-exec this script under torch.distributed.run with N
    ranks on this node (one per GPU); fails loudly when fewer than N GPUs are visible."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
