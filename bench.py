#!/usr/bin/env python
"""bench.py -- the hot path of arXiv 2301.01179 on B200: one step = one full FMM solve
(Algorithm 1: tree, P2M, M2M, tensors, S2L, L2L, L2P, near field) of the largest
single-GPU BASELINE.json configuration, configs[4] (C5: N = M = 4,194,304; sources uniform in arc
length on a torus and a sphere generating curve, fields on a 2048 x 2048 grid of (0,1] x [0,2],
modes n = 0..64, complex N(0,1) coefficients, p = 16, depth 10).  --config C2..C4 run the
smaller configurations (parity-test cases; C2 = configs[1] is the small FMM case).

Metric (BASELINE.json): FP64 modal source-field interactions per second, i.e. the
direct-equivalent rate (N_s N_f - skipped) K / t_solve, plus the solve time and the FP64
roofline fraction of the dominant kernel (per-phase CUDA events recorded by the library on the
streams the phases run on, inside the timed region: cylfmm_plan_set_profiling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cylfmm,reference}] [--config C5]

--impl reference times the CPU oracle (oracle/, plain FP64 C, OpenMP) as it stands on the host
cores -- this tier's reference arm (there is no reference implementation to install).
Under torchrun (N > 1, one process per GPU, NCCL) the field points are partitioned across ranks
by cost-weighted contiguous Morton ranges (cylfmm_partition_fields; north_star), each rank owns a
contiguous shard of the sources, and every timed step replicates the sources with an NCCL
all-gather before the rank's solve; the total problem is fixed ("scaling": "strong") and the
step time is the max over ranks.  Outputs stay sharded (each rank's potentials in its rows).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2301_01179_b200.inputs import CONFIGS  # noqa: E402

FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # DESIGN.md section 6 (derived, "alu")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# adaptive source tree per config (DESIGN R#26): (depth, leaf sources).  C4's
# clusters leave most of a uniform depth-8 tree's leaves either crowded or nearly empty; C5 (sources
# on curves, fields on a full grid) keeps the uniform depth-10 tree (pruning only adds S2L pairs).
ADAPTIVE = {"C4": (11, 224)}


def make_problem(name, args=None):
    """The config's synthetic inputs, with its tree: depth and adaptive leaf size (pr.leaf_src,
    0 = uniform) from ADAPTIVE unless --adaptive / --depth override them."""
    pr = CONFIGS[name]()
    a = getattr(args, "adaptive", None)
    pr.leaf_src = ADAPTIVE.get(name, (0, 0))[1] if a is None else a
    if getattr(args, "depth", 0):
        pr.depth = args.depth
    elif pr.leaf_src > 0 and name in ADAPTIVE:
        pr.depth = ADAPTIVE[name][0]
    return pr


def n_interactions(pr, skipped):
    return (len(pr.sr) * len(pr.fr) - skipped) * pr.K


def oracle_sample(pr, budget_s, cores):
    """Time the oracle FMM (all sources; upward pass in full) on a seeded sample of the field
    points sized so that one run takes about budget_s on this host.  Returns (m, seconds,
    skipped, sample indices)."""
    import oracle
    oracle.build()
    nf = len(pr.fr)
    order = np.random.default_rng(1234).permutation(nf)

    def run(m):
        idx = np.sort(order[:m])
        t0 = time.perf_counter()
        _, sk = oracle.fmm(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx], pr.p, pr.depth, pr.L,
                           pr.z0, nthreads=cores, leaf_src=pr.leaf_src)
        return time.perf_counter() - t0, sk, idx

    m0, m1 = min(nf, 16), min(nf, 64)
    t0, _, _ = run(m0)
    t1, sk, idx = run(m1)
    per = max((t1 - t0) / max(m1 - m0, 1), 1e-6)
    fixed = max(t1 - per * m1, 0.0)
    m = int(min(nf, max(m0, (budget_s - fixed) / per)))
    if m != m1:
        t1, sk, idx = run(m)
    return m, t1, sk, idx, fixed


def run_reference(args):
    """Reference arm: the CPU oracle FMM as it stands, on this host's cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cores = os.cpu_count() or 1
    if args.config == "C1":   # the oracle's direct sum, whole (about 0.1 s per step)
        oracle.build()
        pr = CONFIGS["C1"]()
        K = pr.S.shape[1]
        ts = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.direct(pr.sr, pr.sz, pr.S, pr.fr, pr.fz, nthreads=cores)
            if i >= args.warmup:
                ts.append(time.perf_counter() - t0)
        t = sum(ts) / len(ts)
        v = len(pr.sr) * len(pr.fr) * K / t
        print(json.dumps({
            "metric": "FP64 modal source-field interactions/s (direct sum)", "value": v,
            "unit": "interactions/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "replicas only", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"C1: {pr.name}", "n_src": len(pr.sr), "n_fld": len(pr.fr), "modes": K},
            "cpu_baseline": {"value": v, "unit": "interactions/s", "cores": cores, "kind": "oracle",
                             "sample": "the whole C1 direct sum per step"},
            "e2e": {"value": v, "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    pr = make_problem(args.config, args)
    m, _, _, idx, fixed = oracle_sample(pr, 4.0, cores)   # each step a bounded sample (~4 s)
    fr, fz = pr.fr[idx], pr.fz[idx]
    for _ in range(args.warmup):
        oracle.fmm(pr.sr, pr.sz, pr.S, fr, fz, pr.p, pr.depth, pr.L, pr.z0, nthreads=cores,
                   leaf_src=pr.leaf_src)
    ts = []
    sk = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, sk = oracle.fmm(pr.sr, pr.sz, pr.S, fr, fz, pr.p, pr.depth, pr.L, pr.z0, nthreads=cores,
                           leaf_src=pr.leaf_src)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    inter = (len(pr.sr) * m - sk) * pr.K
    v = inter / t
    sample = (f"oracle FMM (all {len(pr.sr)} sources, upward pass in full, ~{fixed:.1f} s of the "
              f"step) evaluated at a seeded sample of {m} of {len(pr.fr)} field points per step")
    line = {"metric": "FP64 modal source-field interactions/s (direct-equivalent, FMM solve)",
            "value": v, "unit": "interactions/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config}: {pr.name}", "n_src": len(pr.sr),
                       "n_fld": m, "modes": pr.K, "order": pr.p, "depth": pr.depth,
                       "adaptive_leaf": pr.leaf_src},
            "cpu_baseline": {"value": v, "unit": "interactions/s", "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(pr, budget_s=15.0):
    """The oracle as it stands, timed on this host's cores on a bounded sample of the workload."""
    cores = os.cpu_count() or 1
    m, t, sk, _, fixed = oracle_sample(pr, budget_s, cores)
    inter = (len(pr.sr) * m - sk) * pr.K
    return {"value": inter / t, "unit": "interactions/s", "cores": cores, "kind": "oracle",
            "sample": f"one oracle FMM solve: all {len(pr.sr)} sources (upward pass in full, "
                      f"~{fixed:.1f} s), a seeded sample of {m} of {len(pr.fr)} field points "
                      f"({t:.1f} s)"}


# Algorithmic FP64 work per unit: the dominant phase's
# achieved rate = these flops / its in-region CUDA-event time.
def phase_flops(pr, tm):
    K, p = pr.K, pr.p
    P = (p + 1) * (p + 2) // 2
    nf, ns = len(pr.fr), len(pr.sr)
    near = (tm["n_forward"] * (210 + 4 * (K - 2) + 5 * K) + tm["n_far"] * (60 + 14 * K) +
            tm["n_miller"] * (180 + 4 * (K - 1) + 5 * K) + 4 * tm["miller_steps"])
    return {"s2l": tm["n_s2l_pairs"] * 4 * P * P * K,
            "p2p": near,
            "l2p": nf * 4 * P * K,
            "p2m": ns * 4 * P * K}


KERNEL_OF = {"s2l": "s2l_batch_kernel (full batches at p > 12: s2l_batch_units_kernel) + s2l_reduce_kernel (S2L phase)",
             "p2p": "p2p_warp_kernel (near-field phase)",
             "l2p": "l2p_kernel (L2P phase)", "p2m": "p2m_kernel (P2M phase)"}
NCU_NAME = {"s2l": "s2l_batch_kernel", "p2p": "p2p_warp_kernel", "l2p": "l2p_kernel",
            "p2m": "p2m_kernel"}


def run_direct(args):
    """C1 (BASELINE configs[0]): the direct modal sum, I_direct = (N_s N_f - skipped) K / t
    (SURVEY 8(d)).  The sum is ~16 us of FP64 work, so a call is launch-latency bound: the step
    is one replay of a CUDA graph captured from cylfmm_direct_enqueue (launches only), timed
    with the L2 flushed between replays, plus 1000 replays back to back (inputs L2-resident:
    0.3 MB)."""
    import torch
    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200 import build as b
    if not b.up_to_date():
        b.build()
    pr = CONFIGS["C1"]()
    K = pr.S.shape[1]
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    d = [torch.as_tensor(np.ascontiguousarray(a), device=dev) for a in (pr.sr, pr.sz, pr.S, pr.fr, pr.fz)]
    ns, nf = len(pr.sr), len(pr.fr)
    out = torch.empty((nf, K), dtype=torch.complex128, device=dev)
    ws = torch.empty(g.direct_workspace_bytes(ns, nf, K), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        g.direct_enqueue(*d, out, ws)
    torch.cuda.synchronize()
    assert int(ws[:4].view(torch.int32).item()) == 0
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(stream)
    with torch.cuda.stream(cs):
        with torch.cuda.graph(gr, stream=cs):
            g.direct_enqueue(*d, out, ws)
    stream.wait_stream(cs)
    for _ in range(args.warmup):
        gr.replay()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.4)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        gr.replay()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    t_step = sum(a.elapsed_time(bb) for a, bb in ev) / args.steps
    R = 1000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(R):
        gr.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    t_rep = e0.elapsed_time(e1) / R
    # the plain synchronising call (allocation + flag read-back per call), for comparison
    e0.record(stream)
    for _ in range(50):
        g.direct(*d, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    t_call = e0.elapsed_time(e1) / 50
    clk = clocks.stop()
    inter = ns * nf * K     # independent field draws: no coincident pair (flag checked above)
    # e2e: host buffers in, potentials back, through the graph (pinned memory, copies timed)
    hs = [torch.as_tensor(np.ascontiguousarray(a)).pin_memory() for a in (pr.sr, pr.sz, pr.S, pr.fr, pr.fz)]
    hout = torch.empty((nf, K), dtype=torch.complex128).pin_memory()

    def e2e_step():
        for x, y in zip(d, hs):
            x.copy_(y, non_blocking=True)
        gr.replay()
        hout.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
    for _ in range(3):
        e2e_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    t_e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    flops = 600.0 * ns * nf   # W_pair ~ 600 flops at K = 9 (backward branch), 6e8 per sum
    ach = flops / (t_rep * 1e-3) / 1e12
    line = {"metric": "FP64 modal source-field interactions/s (direct sum)",
            "value": inter / (t_rep * 1e-3), "unit": "interactions/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_rep,
            "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C1: {pr.name}", "n_src": ns, "n_fld": nf, "modes": K,
                       "miller": "accurate", "l2": "resident (1000 CUDA-graph replays back to back; "
                       "the flushed single-replay time is ms_per_step_l2_flushed)"},
            "ms_per_step_l2_flushed": t_step, "value_l2_flushed": inter / (t_step * 1e-3),
            "ms_per_call_synchronous_api": t_call,
            "roofline": {"bound": "alu", "kernel": "p2p_warp_kernel + reduce_parts_kernel (direct sum)",
                         "achieved": ach, "peak": FP64_NOMINAL_TFLOPS, "unit": "TFLOP/s",
                         "frac": ach / FP64_NOMINAL_TFLOPS, "traffic": None,
                         "algorithmic_flops": flops,
                         "note": "one sum is 6e8 flops = 16 us at the FP64 nominal: launch / tail bound"},
            "clocks": clk,
            "e2e": {"value": inter / (t_e2e * 1e-3), "unit": "interactions/s", "ms_per_step": t_e2e,
                    "h2d_bytes_per_step": ns * (16 + 16 * K) + nf * 16, "d2h_bytes_per_step": nf * K * 16,
                    "api": "pinned copies + CUDA-graph replay of cylfmm_direct_enqueue"},
            "gpu_launches": 3 * R}
    if not args.no_cpu_baseline:
        import oracle
        oracle.build()
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 10.0:
            oracle.direct(pr.sr, pr.sz, pr.S, pr.fr, pr.fz, nthreads=cores)
            reps += 1
        t = (time.perf_counter() - t0) / reps
        line["cpu_baseline"] = {"value": inter / t, "unit": "interactions/s", "cores": cores,
                                "kind": "oracle", "sample": f"the whole C1 direct sum, {reps} repeats"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cylfmm", choices=["cylfmm", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--adaptive", type=int, default=None, metavar="SIGMA",
                    help="adaptive source tree (leaf <= SIGMA sources, SURVEY 8(f)-4); "
                         "0 = uniform; default: the config's (C4: 224 at depth 11)")
    ap.add_argument("--depth", type=int, default=0, help="override the config's depth")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "cylfmm" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "C1":
        return run_direct(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200 import build as b
    from paper_2301_01179_b200 import distributed as dd
    if not b.up_to_date():
        b.build()
    pr = make_problem(args.config, args)
    dev = torch.device("cuda", local)
    cfg = g.FMMConfig(n_modes=pr.K, order=pr.p, depth=pr.depth, L=pr.L, z0=pr.z0,
                      adaptive_leaf=pr.leaf_src)
    # fields: all of them on one GPU; on N GPUs the cost-weighted contiguous Morton range of this
    # rank (cylfmm_partition_fields, identical on every rank: planning, outside the timed region)
    if world > 1:
        part, _ = g.partition_fields(pr.sr, pr.sz, pr.fr, pr.fz, cfg, world)
        fidx = dd.my_fields(part, rank)
    else:
        fidx = np.arange(len(pr.fr))
    # sources: each rank owns a contiguous shard; N > 1: the library replicates them inside every
    # timed step (cylfmm_fmm_solve_dist: NCCL all-gather of the shard sizes, grouped broadcasts of
    # the shards, P2M split across the ranks + leaf-moment broadcasts) -- the north_star's
    # replication of the sources and the upper tree
    sl = dd.source_shard(len(pr.sr), rank, world)
    sr_loc = torch.as_tensor(pr.sr[sl], device=dev)
    sz_loc = torch.as_tensor(pr.sz[sl], device=dev)
    S_loc = torch.as_tensor(pr.S[sl], device=dev)
    same = pr.fields_are_sources and world == 1       # fields ARE the sources (C2-C4)
    fr, fz = pr.fr[fidx], pr.fz[fidx]
    fr_d = torch.as_tensor(np.ascontiguousarray(fr), device=dev)
    fz_d = torch.as_tensor(np.ascontiguousarray(fz), device=dev)
    out = torch.empty((len(fr), pr.K), dtype=torch.complex128, device=dev)
    if world > 1:   # the library-owned NCCL communicator (id from rank 0)
        from paper_2301_01179_b200.cylfmm import comm_unique_id
        uid = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        plan = g.Plan(cfg, dist=(world, rank, uid[0]))
    else:
        plan = g.Plan(cfg)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(timings=False):
        if world > 1:
            return plan.solve_dist(sr_loc, sz_loc, S_loc, fr_d, fz_d, out=out, timings=timings)
        a, bb = (sr_loc, sz_loc) if same else (fr_d, fz_d)
        return plan.solve(sr_loc, sz_loc, S_loc, a, bb, out=out, timings=timings)

    # warm-up, then one synchronising timings solve outside the timed region for the counts
    # (near-field branch mix, skipped pairs); the phase times come from the timed region
    for _ in range(args.warmup):
        step()
    _, tm = step(timings=True)
    launches_per_step = tm["kernel_launches"]
    skipped = tm["n_skipped"]
    plan.set_profiling(True)

    # timed region: K solves, L2 flushed between them (not timed), CUDA events on the stream
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    barrier()
    ms = [a.elapsed_time(bb) for a, bb in ev]
    clk = clocks.stop()
    phase = plan.read_timings()   # per-phase CUDA events of the K timed solves (averaged)
    plan.set_profiling(False)
    t_step = sum(ms) / len(ms)
    t_max = t_step
    if world > 1:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        sk = torch.tensor([skipped], device=dev, dtype=torch.int64)
        dist.all_reduce(sk)
        skipped = int(sk.item())
    inter_total = (len(pr.sr) * len(pr.fr) - skipped) * pr.K
    value = inter_total / (t_max * 1e-3)

    # fixed-geometry re-solves (new coefficients on the same rings: cylfmm_plan_set_geometry_cache):
    # the coefficient-dependent passes only, sync-free; then the same solve replayed as a CUDA graph
    reuse = None
    if world == 1 and not args.no_e2e:
        plan.set_geometry_cache(True)
        step()                                           # builds and remembers the geometry
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            step()
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        t_cached = sum(a.elapsed_time(bb) for a, bb in ev2) / args.steps
        gr = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step()
            with torch.cuda.graph(gr, stream=cs):
                step()
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            gr.replay()
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        t_graph = sum(a.elapsed_time(bb) for a, bb in ev2) / args.steps
        plan.set_geometry_cache(False)
        reuse = {"note": "fixed geometry, new coefficients each step: coordinate-only work reused "
                         "(cylfmm_plan_set_geometry_cache); not the headline step",
                 "ms_per_step": t_cached, "ms_per_step_cuda_graph": t_graph,
                 "value_cuda_graph": (len(pr.sr) * len(pr.fr) - skipped) * pr.K / (t_graph * 1e-3)}
    e2e = None
    if not args.no_e2e:
        # e2e through the host-buffer C-ABI call (pinned host memory, H2D + D2H inside the region):
        # the full source set and this rank's field points in, this rank's potentials out
        if world > 1:
            # this rank's source shard and field points from pinned host memory, the solve, its
            # potentials back to pinned host memory (the copies inside the timed region)
            hsh = [torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
                   for a in (pr.sr[sl], pr.sz[sl])]
            hSh = torch.as_tensor(np.ascontiguousarray(pr.S[sl])).pin_memory()
            hf = [torch.as_tensor(np.ascontiguousarray(a)).pin_memory() for a in (fr, fz)]
            hout = torch.empty((len(fr), pr.K), dtype=torch.complex128).pin_memory()

            def e2e_step():
                d = [x.to(dev, non_blocking=True) for x in (hsh[0], hsh[1], hSh, hf[0], hf[1])]
                o = plan.solve_dist(d[0], d[1], d[2], d[3], d[4], out=out)
                hout.copy_(o, non_blocking=True)
                torch.cuda.synchronize()
        else:
            hs = [torch.as_tensor(a).pin_memory() for a in (pr.sr, pr.sz)]
            hS = torch.as_tensor(pr.S).pin_memory()
            hf = hs if same else [torch.as_tensor(np.ascontiguousarray(a)).pin_memory() for a in (fr, fz)]
            hout = torch.empty((len(fr), pr.K), dtype=torch.complex128).pin_memory()

            def e2e_step():
                plan.solve_host(hs[0].numpy(), hs[1].numpy(), hS.numpy(), hf[0].numpy(),
                                hf[1].numpy(), out=hout.numpy())
        for _ in range(2):
            e2e_step()
        barrier()
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        t_e2e = sum(e2e_ms) / len(e2e_ms)
        t_sync = t_e2e
        if world == 1:
            # the streaming form of the same call (cylfmm_fmm_solve_host_async): K solves queued
            # back to back, each with its own upload and download (two device staging slots:
            # step i+1's upload and step i-1's download overlap step i's solve), one sync at the
            # end; the inputs (4.5 GB at C5) exceed L2, so no flush between steps
            args_h = (hs[0].numpy(), hs[1].numpy(), hS.numpy(), hf[0].numpy(), hf[1].numpy(),
                      hout.numpy())
            for _ in range(2):
                plan.solve_host_async(*args_h)
            plan.sync()
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                plan.solve_host_async(*args_h)
            plan.sync()
            t_e2e = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        nsl = sl.stop - sl.start if world > 1 else len(pr.sr)
        h2d = nsl * (16 + 16 * pr.K) + (0 if same else len(fr) * 16)
        d2h = len(fr) * pr.K * 16
        e2e = {"value": inter_total / (t_e2e * 1e-3), "unit": "interactions/s",
               "ms_per_step": t_e2e, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": ("cylfmm_fmm_solve_host_async (pipelined, sync after the K steps)"
                       if world == 1 else "pinned copies + cylfmm_fmm_solve_dist"),
               "ms_per_step_synchronous": t_sync}

    # roofline of the dominant kernel (FP64 CUDA-core arithmetic: "alu"): the compute phase
    # with the largest in-region time, its algorithmic flops (phase_flops) / that time
    fl = phase_flops(pr, tm)
    dom = max(fl, key=lambda k: phase["ms_" + k])
    ach = fl[dom] / (phase["ms_" + dom] * 1e-3) / 1e12 if phase["ms_" + dom] > 0 else None
    traffic = None
    try:   # dram read + write bytes per step of the dominant kernel(s), committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            per = json.load(f)["per_step_dram_bytes"][args.config]
            traffic = per.get(NCU_NAME[dom])
            if traffic is None and dom == "s2l":
                traffic = per.get("s2l_batch_units_kernel")
    except Exception:
        pass
    roof = {"bound": "alu", "kernel": KERNEL_OF[dom], "achieved": ach, "peak": FP64_NOMINAL_TFLOPS,
            "unit": "TFLOP/s", "frac": ach / FP64_NOMINAL_TFLOPS if ach else None,
            "traffic": traffic, "algorithmic_flops": fl[dom], "ms": phase["ms_" + dom],
            "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the phase's "
                            "kernel launches in one step (profiles/ncu_traffic.json)",
            "peak_note": "FP64 nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md 6); "
                         "MEASURED_PEAKS.json has no FP64 figure",
            "phase_frac": {k: (fl[k] / (phase["ms_" + k] * 1e-3) / 1e12 / FP64_NOMINAL_TFLOPS
                               if phase["ms_" + k] > 0 else None) for k in fl}}

    if rank == 0:
        line = {"metric": "FP64 modal source-field interactions/s (direct-equivalent, FMM solve)",
                "value": value, "unit": "interactions/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{args.config}: {pr.name}", "n_src": len(pr.sr),
                           "n_fld": len(pr.fr), "modes": pr.K, "order": pr.p, "depth": pr.depth,
                           "tree": (f"adaptive source tree, leaf <= {pr.leaf_src} sources"
                                    if pr.leaf_src > 0 else "uniform"),
                           "truncation": "double", "miller": "accurate", "l2": "flushed",
                           "parallelism": (f"field-partition x{world} (cost-weighted Morton ranges; "
                                           "library NCCL: source broadcast-all-gather, P2M split + "
                                           "leaf-moment broadcast)") if world > 1 else "single GPU"},
                "phase_ms": {k: round(v, 4) for k, v in phase.items() if k.startswith("ms_")},
                "near_branches": {k: tm[k] for k in ("n_forward", "n_far", "n_miller", "miller_steps")},
                "near_pairs": tm["n_near_pairs"], "s2l_box_pairs": tm["n_s2l_pairs"],
                "roofline": roof, "clocks": clk,
                "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps,
                "fixed_geometry": reuse}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(pr)
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
