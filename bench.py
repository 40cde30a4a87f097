#!/usr/bin/env python
"""bench.py — throughput of the FP8-LM data-parallel hot path on B200.

One "step" = one pass of the whole hot path over one
synthetic gradient set already resident in HBM:
  amax_scale_sync (A1 amax, A2 mu/scale/MIN) -> fp8_grad_allreduce (A3 quantize,
  A4/A5 reduce-scatter + FP32 reduce + all-gather, Eq. 6 scale, mu update) ->
  fp8_adam_step (A6 dequant + A7 two-pass JIT FP8 AdamW, FP8 weight copy).

Default workload: BASELINE.json configs[2], the GPT-7B gradient set (387 tensors, 6.65G
params, 26.6 GB of fp32 gradient) at N GPUs — the config the metric's "at 1/2/4/8 B200"
is quoted on.  --config gpt-125m is configs[1] (147 tensors, 123.69M params), c1 is
configs[0] (one 4096x4096 fp32 gradient, 2 simulated ranks on one GPU), gpt-13b with
--exchange zero is configs[3], gpt-175b-layer one transformer layer of GPT-175B (12
tensors, 1.81G params; north_star's "gradient sets shaped like GPT-7B/13B/175B layers").
N > 1 (torchrun): one rank per GPU, NCCL over NVLink, each rank holding its own full
gradient set (data parallelism: per-GPU work fixed -> "scaling": "weak").

metric (BASELINE.json): GB/s of algorithmic bytes moved per step, whole job (sum over
ranks) = N * bytes_per_rank / max-over-ranks step time, where bytes_per_rank = params
x (27 B at N = 1; 28 + 1/N + 2(N-1)/N B at N >= 2; 39 B for c1) — SURVEY §8(d).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 grad reduce+Adam step: GB/s & % HBM/NVLink roofline at 1/2/4/8 B200"
UNIT = "GB/s"
FALLBACK_HBM_GBS = 6650.0
NVLINK_PEER_GBS = 770.0   # measured peer copy per direction per GPU (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="gpt-7b",
                    choices=["gpt-7b", "gpt-125m", "gpt-13b", "gpt-175b-layer", "c1"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"], help="gradient dtype")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl", "zero"],
                    help="N > 1: fused peer-memory reduce-scatter/all-gather kernel (p2p), "
                         "NCCL all-to-all + all-gather around the reduce kernel (nccl), or "
                         "FP8 ZeRO whole-tensor owners over peer memory (zero, config C4)")
    ap.add_argument("--buckets", type=int, default=0,
                    help="N > 1, modes p2p / zero: split the tensors into this many buckets (one plan "
                         "each) and run the step in two phases per bucket (fp8lm_dp_step_split), so "
                         "the exchange of one bucket overlaps the HBM passes of the others.  0 = auto: "
                         "6 (p2p) or 4 (zero) for sets above 1G params, else 1 (small sets are launch-bound)")
    ap.add_argument("--bucket-lag", type=int, default=0,
                    help="split step issue order: 0 = phase 1 of every bucket then phase 2 of every "
                         "bucket; k = phase 2 of bucket b after phase 1 of bucket b + k")
    ap.add_argument("--lr", type=float, default=0.0,
                    help="0: the paper's max LR of the config (Table 1, P:279-282: 6e-4 for "
                         "GPT-125M, 3e-4 for 7B, 13B and C1, 6e-5 for 175B)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grad-sets", type=int, default=0,
                    help="gradient sets rotated step by step, in antithetic pairs when even (0: 4 for "
                         "GPT-125M, 2 for 7B, 1 for 13B)")
    ap.add_argument("--state-scaling", default="jit", choices=["jit", "delayed"],
                    help="optimizer-state scales: just-in-time (two AdamW passes, R19) or "
                         "delayed from a 16-step amax history (one pass, R25-R27)")
    ap.add_argument("--graph", action="store_true",
                    help="run the step as a CUDA graph (fp8lm_dp_step_graphed; single-plan steps)")
    ap.add_argument("--worst-case", action="store_true",
                    help="data-dependent worst case: lr 0.05 moves the largest weights far beyond the "
                         "amax(w') screen's margin, so pass 2's prologue recomputes pass 1 exactly for "
                         "(nearly) every tensor (DESIGN §5)")
    ap.add_argument("--quick", action="store_true",
                    help="profiling runs (ncu): no clock soak, no e2e, no cpu baseline")
    return ap.parse_args()


CONFIG_INDEX = {"c1": 0, "gpt-125m": 1, "gpt-7b": 2, "gpt-13b": 3, "gpt-175b-layer": None}
PAPER_LR = {"c1": 3e-4, "gpt-125m": 6e-4, "gpt-7b": 3e-4, "gpt-13b": 3e-4, "gpt-175b-layer": 6e-5}
C1_RANKS = 2
WORKLOAD = {
    "c1": "one 4096x4096 fp32 gradient tensor, 2 simulated ranks on one GPU (BASELINE.json configs[0])",
    "gpt-125m": "gpt-125m full gradient set (BASELINE.json configs[1])",
    "gpt-7b": "gpt-7b full gradient set (BASELINE.json configs[2])",
    "gpt-13b": "gpt-13b full gradient set (BASELINE.json configs[3])",
    "gpt-175b-layer": "one gpt-175b transformer layer (12 tensors, d = 12288; north_star's 175B layer shapes)",
}


def config_specs(config: str):
    """Tensor specs of a bench workload."""
    import synth
    if config == "c1":
        return synth.square_set(4096)
    if config == "gpt-175b-layer":
        return [s for s in synth.gpt_gradient_set("gpt-175b", 1) if s.name.startswith("layer0.")]
    return synth.gpt_gradient_set(config)


def alg_bytes_per_param(N: int, zero: bool = False, delayed: bool = False, sim: int = 0) -> float:
    """A1 4 + A3 5 + A7 18 at N = 1 (A4/A5 identity); at N >= 2 add the
    reduce (1 + 1/N) and the all-gather write 2(N-1)/N.  ZeRO owner mode (C4): every rank
    reads its gradient twice (A1 4, A3 5), the owner reduce reads N x n/N codes and writes
    n/N (1 + 1/N), AdamW runs on n/N parameters (18/N) and the w8 broadcast reads n/N and
    writes n (1/N + 1): 11 + 20/N.  Delayed state scaling (R25-R27) runs AdamW in one pass:
    A7 = read g8 1 + m1 1 + v 2 + master 2, write m1 1 + v 2 + master 2 + w8 1 = 12."""
    a7 = 12.0 if delayed else 18.0
    if sim:       # simulated ranks on one GPU (c1): A1 4N + A3 5N + reduce N + 1 + A7
        return 10.0 * sim + 1.0 + a7
    if zero:
        return 11.0 + (2.0 + a7) / N
    if N == 1:
        return 9.0 + a7
    return 10.0 + a7 + 1.0 / N + 2.0 * (N - 1) / N


# per-launch algorithmic bytes per parameter of each kernel (LOCAL / NCCL modes)
KERNEL_BYTES = {
    "amax": 4.0, "quantize": 5.0, "adam_pass1": 6.0, "adam_pass2": 12.0,
    "quantize+adam_pass1": 10.0,      # fused LOCAL kernel: read g 4, m1 1, v 2, master 2; write g8 1
    "adam_delayed": 12.0,             # single pass: read g8 1, m1 1, v 2, master 2; write 6
    "quantize+adam_delayed": 16.0,    # fused LOCAL: read g 4 + states 5; write g8 1 + states 5 + w8 1
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                index = int(vis.split(",")[index])
            except (ValueError, IndexError):
                pass
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(index), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), hw=parts[5], hwt=parts[6],
                                 swt=parts[7], pcap=parts[8]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        reasons = set()
        for r in rows:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                            ("swt", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in rows), "sm_max_mhz": max(r["smax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ oracle (CPU) legs
# The CPU oracle (oracle/, numpy, one core per process) as it stands, run on every host
# core: nothing in its arithmetic couples two tensors, so a fixed set of worker processes
# each owns whole tensors (assigned largest-first to the least-loaded worker) and keeps
# their optimizer state across steps.  Per step every worker generates its inputs
# (untimed), meets the others at a barrier, runs oracle.step.train_step on its tensors
# and reports its start / end time; the step time is the makespan max(end) - min(start).
def oracle_sample(specs, config, reference=False):
    """Bounded sample of the workload (tensor indices) for the oracle."""
    cores = len(os.sched_getaffinity(0))
    if config == "gpt-125m":
        # the whole C2 set ("timed fully for C1 and C2"); the reference arm,
        # which runs K + W steps, leaves out the 38.6M embedding (one core, ~20 s)
        return [t for t, s in enumerate(specs) if not (reference and s.name == "emb.w")]
    if config == "c1":
        return [0]
    # GPT-7B / 13B / 175B layer: the attention projections d x d of the first `cores` layers
    # (equal tensors: one per core; the smallest matrices of these sets), at most 16: the
    # oracle is memory-bound numpy, and more concurrent workers only slow each step (32
    # cores: 35 s per step against 18 s with 16)
    idx = [t for t, s in enumerate(specs) if s.name.endswith(".proj.w")]
    return idx[:max(1, min(cores, 16, len(idx)))]


def _oracle_worker(conn, barrier, tensors, nranks, delayed, lr):
    """One oracle process: tensors = [(t, numel)]; conn receives step numbers, None to stop."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    import torch
    torch.set_num_threads(1)
    import synth
    from oracle import adam as OA
    from oracle import step as OS
    states = []
    for t, n in tensors:
        w = torch.empty(n, dtype=torch.float32)
        synth.fill_weights(w, t)
        states.append(OA.init_state(w.numpy()))
    hists = [OA.init_history(st) for st in states] if delayed else None
    mus = [np.float32(1.0)] * len(tensors)
    conn.send("ready")
    while True:
        step = conn.recv()
        if step is None:
            break
        grads = []
        for r in range(nranks):
            row = []
            for t, n in tensors:
                g = torch.empty(n, dtype=torch.float32)
                synth.fill_gradient(g, step, t, r)
                row.append(g.numpy())
            grads.append(row)
        barrier.wait()
        t0 = time.monotonic()
        res = OS.train_step(grads, mus, states, OA.hyper_params(lr, step), hists=hists, step=step)
        t1 = time.monotonic()
        states, mus = res["states"], res["mu_next"]
        if delayed:
            hists = res["hists"]
        conn.send((t0, t1))


class OraclePool:
    """Worker processes (spawn: the parent may hold a CUDA context) over the sample."""

    def __init__(self, specs, idx, nranks=1, delayed=False, lr=3e-4, workers=None):
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        W = max(1, min(workers or len(os.sched_getaffinity(0)), len(idx)))
        load = [0] * W
        parts = [[] for _ in range(W)]
        for t in sorted(idx, key=lambda t: -specs[t].numel):      # largest first, least loaded
            j = min(range(W), key=lambda k: load[k])
            parts[j].append((t, specs[t].numel))
            load[j] += specs[t].numel
        self.params = sum(specs[t].numel for t in idx)
        self.max_part = max(load)
        self.barrier = ctx.Barrier(W)
        self.conns, self.procs = [], []
        for part in parts:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_oracle_worker, args=(b, self.barrier, part, nranks, delayed, lr),
                            daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"
        self.workers = W
        self.step_no = 0

    def step(self):
        """One oracle step of the whole sample -> (makespan s, per-worker busy s list)."""
        self.step_no += 1
        for c in self.conns:
            c.send(self.step_no)
        times = [c.recv() for c in self.conns]
        return max(t[1] for t in times) - min(t[0] for t in times), [t[1] - t[0] for t in times]

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=30)


def _oracle_line(args, specs, pool, secs, busy):
    nsim = C1_RANKS if args.config == "c1" else 0
    delayed = args.state_scaling == "delayed"
    bpp = alg_bytes_per_param(1, delayed=delayed, sim=nsim)
    value = bpp * pool.params / secs / 1e9
    # one core: the largest worker's own rate (its params over its busy time)
    one = bpp * pool.max_part / max(busy) / 1e9
    total = sum(s.numel for s in specs)
    cpu = os.popen("grep -m1 'model name' /proc/cpuinfo").read().split(":")[-1].strip()
    return value, {
        "value": value, "unit": UNIT, "cores": pool.workers, "kind": "oracle",
        "sample": (f"{pool.params} of {total} params of {args.config} ({len(specs)} tensors); "
                   f"whole tensors over {pool.workers} worker processes (one core each), makespan "
                   f"{secs:.2f} s per step"),
        "value_1thread": one, "host_cores_available": len(os.sched_getaffinity(0)), "cpu_model": cpu,
        "extrapolated_full_config_s": total * bpp / (value * 1e9)}


def cpu_baseline(args, specs):
    idx = oracle_sample(specs, args.config)
    pool = OraclePool(specs, idx, C1_RANKS if args.config == "c1" else 1,
                      args.state_scaling == "delayed", args.lr)
    try:
        secs, busy = pool.step()
    finally:
        pool.close()
    return _oracle_line(args, specs, pool, secs, busy)[1]


def run_reference(args, specs, world, rank):
    """--impl reference: the CPU oracle as the reference arm, same metric/config/unit."""
    if rank != 0:
        return
    idx = oracle_sample(specs, args.config, reference=True)
    pool = OraclePool(specs, idx, C1_RANKS if args.config == "c1" else 1,
                      args.state_scaling == "delayed", args.lr)
    try:
        for _ in range(args.warmup):
            pool.step()
        tot, busy_max = 0.0, []
        for _ in range(args.steps):
            secs, busy = pool.step()
            tot += secs
            busy_max.append(max(busy))
    finally:
        pool.close()
    ms = tot / args.steps * 1e3
    value, cpu = _oracle_line(args, specs, pool, ms / 1e3, [statistics.mean(busy_max)])
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} gradient set, oracle sample", "tensors": len(idx),
                       "params": pool.params, "state_scaling": args.state_scaling},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main
def main():
    args = parse()
    import synth
    if args.worst_case:
        args.lr = 0.05
    if not args.lr:
        args.lr = PAPER_LR[args.config]
    specs = config_specs(args.config)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, specs, world, rank)
        return

    import torch
    world, rank, local = dist_setup(args)
    import paper_2310_18313_b200 as B

    numels = [s.numel for s in specs]
    params = sum(numels)
    N = world
    sim = C1_RANKS if args.config == "c1" else 0
    if sim and N > 1:
        raise SystemExit("--config c1 is 2 simulated ranks on ONE GPU (BASELINE configs[0])")
    comm = B.Comm.from_torch_distributed() if N > 1 else None
    mode = ({"p2p": B.MODE_P2P, "nccl": B.MODE_NCCL, "zero": B.MODE_ZERO}[args.exchange]
            if N > 1 else (B.MODE_SIMULATED if sim else B.MODE_LOCAL))
    zero = mode == B.MODE_ZERO
    # auto: 6 buckets for P2P sets above 1G params, 4 for ZeRO (profiles/r2/split, zero_push)
    nb = args.buckets if args.buckets > 0 else ((4 if args.exchange == "zero" else 6) if params > 1e9 else 1)
    if not (N > 1 and args.exchange in ("p2p", "zero")):
        nb = 1
    groups = B.bucket_split(numels, nb) if nb > 1 else [list(range(len(numels)))]
    plans = [B.Plan([numels[t] for t in grp], mode=mode, nranks=sim or N, rank=rank) for grp in groups]
    plan = plans[0] if nb == 1 else None
    gdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    w0s = []
    for pl, grp in zip(plans, groups):
        w0 = pl.flat(torch.float32)
        for j, v in enumerate(pl.views(w0)):
            synth.fill_weights(v, grp[j])
        w0s.append(w0)
    R = args.grad_sets or {"gpt-125m": 4, "gpt-7b": 2, "gpt-13b": 1, "gpt-175b-layer": 2, "c1": 4}[args.config]
    # antithetic rotation G1, -G1, G2, -G2, ...: a gradient with a persistent mean drives
    # every weight to the sign-descent fixed point |w| = 1/wd within ~1e3 steps, a state
    # no real run reaches (the weights pile up at amax(w) and crowd the amax screen)
    # gsets[k]: the step input of gradient set k (one flat buffer; a list of the simulated
    # ranks' buffers; a list of the buckets' buffers); gbufs[k]: its device tensors
    gsets, gbufs = [], []
    for r_ in range(R):
        bufs = []
        for pl, grp in zip(plans, groups):
            for rk in (range(sim) if sim else [rank]):
                g = pl.flat(gdt)
                for j, v in enumerate(pl.views(g)):
                    synth.fill_gradient(v, 1 + r_ // 2, grp[j], rk)
                if R % 2 == 0 and r_ % 2 == 1:
                    g.neg_()
                bufs.append(g)
        gbufs.append(bufs)
        gsets.append(bufs if (sim or nb > 1) else bufs[0])
    grads = gsets[0]
    delayed = args.state_scaling == "delayed"
    if nb > 1:
        dp = B.BucketedDP(plans, w0s, comm=comm, lr=args.lr, state_scaling=args.state_scaling,
                          lag=args.bucket_lag)
    else:
        dp = B.FP8DataParallel(plans[0], w0s[0], comm=comm, lr=args.lr, state_scaling=args.state_scaling,
                               graphed=args.graph)
    dps = dp.dps if nb > 1 else [dp]
    del w0s
    torch.cuda.synchronize()
    nstep = [0]

    def step():
        dp.step(gsets[nstep[0] % R])
        nstep[0] += 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # clock sampler runs through a ~1 s untimed soak and the timed region.  Every rank
    # must run the SAME number of soak steps (each step is a collective), so the count is
    # derived from the warm-up's pace and agreed on (max over ranks) before the soak.
    sampler = None if args.quick else ClockSampler(local)
    if sampler is not None:
        t0 = time.perf_counter()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        per = max((time.perf_counter() - t0) / 3, 1e-5)
        n_soak = int(max_over_ranks(float(min(20000, max(1, int(1.0 / per)))), world))
        for _ in range(n_soak):
            step()
        torch.cuda.synchronize()

    # ---------------- timed region: K steps, CUDA events on the launch stream.  A clean
    # region gives ms_per_step / value; a second, instrumented region of K steps (every
    # library launch bracketed by events, which also serialises the PDL overlap of
    # consecutive kernels) gives the per-kernel times of the roofline
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world)

    barrier(world)
    torch.cuda.synchronize()
    for d_ in dps:           # per-kernel tracing needs the launches: the same kernels, eagerly
        d_.graphed = False
    B.prof_enable(True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    B.prof_enable(False)
    prof = B.prof_read()
    ms_prof_local = ev0.elapsed_time(ev1) / args.steps
    ms_prof = max_over_ranks(ms_prof_local, world)
    clocks = sampler.stop() if sampler is not None else None

    bytes_rank = alg_bytes_per_param(N, zero, delayed, sim) * params
    if args.dtype == "bf16":
        bytes_rank -= 2.0 * 2 * params * max(sim, 1)    # A1 and A3 read 2 B instead of 4
    value = N * bytes_rank / (ms / 1e3) / 1e9

    # ---------------- roofline of the dominant kernel (ours, largest device time)
    hbm, hbm_kind = peaks()
    ours = {k: v for k, v in prof.items() if v["ours"]}
    dom = max(ours, key=lambda k: ours[k]["ms"]) if ours else None
    roof = None
    kparams = sum(sum(d.layout.numels) for d in dps) if zero else params   # AdamW: owned tensors only
    # launches per step of the dominant kernel (buckets: one per bucket): bytes per launch
    # are the per-step bytes over that count
    lps = max(1.0, ours[dom]["launches"] / args.steps) if dom else 1.0
    if nb > 1:
        # split step: the exchange kernels of one bucket run beside the HBM passes of the
        # others, so a kernel's own event-bracketed time includes the time it shared the
        # GPU; the meaningful roofline is the whole step's (HBM-bound: every rank streams
        # its states and gradient once or twice, the NVLink traffic rides beside it)
        achieved = bytes_rank / (ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"whole step ({nb} buckets, overlapped kernels)",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_kind": hbm_kind, "traffic": None, "alg_bytes_per_launch": bytes_rank,
                "avg_launch_ms": ms, "share_of_step": 1.0,
                "note": "per rank; algorithmic bytes of SURVEY 8(d) (pass 1 counted whole although "
                        "each rank runs 1/N of it)"}
    elif zero and dom == "adam_pass2" and N > 1:
        # ZeRO dp_step: the owner's pass 2 also stores every w8 code into the N-1 peers'
        # windows, (N-1) bytes per owned parameter out of this GPU over NVLink, under its
        # own 12 B/param of HBM traffic; the link is the bound (the HBM fraction rides along)
        per_launch_ms = ours[dom]["ms"] / ours[dom]["launches"]
        nvb = (N - 1) * kparams / lps
        achieved = nvb / (per_launch_ms / 1e3) / 1e9
        hbm_ach = KERNEL_BYTES["adam_pass2"] * kparams / lps / (per_launch_ms / 1e3) / 1e9
        roof = {"bound": "nvlink", "kernel": dom, "achieved": achieved, "peak": NVLINK_PEER_GBS,
                "unit": "GB/s", "frac": achieved / NVLINK_PEER_GBS,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md); 900 nominal",
                "frac_of_nominal_900": achieved / 900.0, "traffic": None,
                "hbm_achieved": hbm_ach, "hbm_frac": hbm_ach / hbm,
                "alg_bytes_per_launch": nvb, "avg_launch_ms": per_launch_ms,
                "share_of_step": ours[dom]["ms"] / (ms_prof_local * args.steps)}
    elif dom == "reduce_p2p":
        # reduce-scatter over NVLink peer memory: every link direction carries (N-1)/N
        # bytes per parameter of read responses.  fp8lm_dp_step pulls the all-gather
        # inside the AdamW pass that encodes the states, so the exchange kernel moves
        # only those; the ZeRO owner reduce pulls (N-1)/N as well.
        per_launch_ms = ours[dom]["ms"] / ours[dom]["launches"]
        nvb = 1.0 * (N - 1) / N * params / lps
        achieved = nvb / (per_launch_ms / 1e3) / 1e9
        roof = {"bound": "nvlink", "kernel": dom, "achieved": achieved, "peak": NVLINK_PEER_GBS,
                "unit": "GB/s", "frac": achieved / NVLINK_PEER_GBS,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md); 900 nominal",
                "frac_of_nominal_900": achieved / 900.0, "traffic": None,
                "alg_bytes_per_launch": nvb, "avg_launch_ms": per_launch_ms,
                "share_of_step": ours[dom]["ms"] / (ms_prof_local * args.steps)}
    elif dom:
        per_launch_ms = ours[dom]["ms"] / ours[dom]["launches"]
        bpp = KERNEL_BYTES.get(dom)
        if sim and dom == "reduce":
            bpp = sim + 1.0                  # read the N simulated ranks' codes, write the sum
        if sim and dom == "quantize+adam_pass1":
            bpp = 4.0 * sim + 6.0            # fused: read N gradients + m1, v, master; write g8
        if sim and dom == "amax":
            bpp = 4.0 * sim                  # one launch reads every simulated rank's gradient
        if bpp is not None:
            if args.dtype == "bf16" and dom in ("amax", "quantize", "quantize+adam_pass1",
                                                "quantize+adam_delayed"):
                bpp -= 2.0 * (sim if sim and dom != "quantize" else 1)
            np_ = (kparams if dom.startswith("adam") else params) / lps
            achieved = bpp * np_ / (per_launch_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "peak_kind": hbm_kind, "traffic": None,
                    "alg_bytes_per_launch": bpp * np_, "avg_launch_ms": per_launch_ms,
                    "share_of_step": ours[dom]["ms"] / (ms_prof_local * args.steps)}
    if roof is not None:
        # DRAM bytes per launch of the same kernel on the same workload, from the committed
        # `ncu --set full` capture (tools/ncu_traffic.py); null when none was taken
        key = args.config + ("" if N == 1 else f"/n{N}/{args.exchange}") + \
            ("/delayed" if delayed else "") + ("/bf16" if args.dtype == "bf16" else "")
        for rnd in ("r2", "r1"):
            try:
                tr = json.load(open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")))
                ent = tr[key][dom]
            except (OSError, KeyError, ValueError):
                continue
            roof["traffic"] = ent["dram_bytes_per_launch"]
            roof["traffic_source"] = f"profiles/{rnd}/ncu_traffic.json [{key}] ({ent['source']})"
            break
    # our kernels launched inside the timed region (this rank): the instrumented pass runs
    # the same K steps, so its count is the timed region's
    launches = int(sum(v["launches"] for v in ours.values()))
    breakdown = {k: {"launches_per_step": v["launches"] / args.steps, "ms_per_step": v["ms"] / args.steps}
                 for k, v in prof.items()}
    if world > 1:
        # the same kernel on every rank: a spread here is cross-rank skew (a rank waiting in
        # the next step's scale exchange for a slower one), not kernel work
        for k in sorted(breakdown):
            v = breakdown[k]["ms_per_step"]
            breakdown[k]["ms_per_step_min_over_ranks"] = -max_over_ranks(-v, world)
            breakdown[k]["ms_per_step_max_over_ranks"] = max_over_ranks(v, world)

    # ---------------- e2e: host gradients (pinned) -> device, step, results -> host
    e2e = None
    if not args.no_e2e and not args.quick:
        host_sets = []
        dev_bufs = gbufs[0]
        set_bytes = sum(g.numel() * g.element_size() for g in dev_bufs)
        # large models: one pinned host copy (the H2D cost per step is the same)
        for bufs in (gbufs if set_bytes < 4e9 else gbufs[:1]):
            hs = []
            for g in bufs:
                h = torch.empty(g.numel(), dtype=gdt, pin_memory=True)
                h.copy_(g)
                hs.append(h)
            host_sets.append(hs)
        nres = sum(3 * d.plan.T + 1 for d in dps)
        out_h = torch.empty(nres, dtype=torch.float32, pin_memory=True)
        out_d = torch.empty(nres, dtype=torch.float32, device="cuda")
        ne = [0]

        def e2e_step():
            for d_, h_ in zip(dev_bufs, host_sets[ne[0] % len(host_sets)]):
                d_.copy_(h_, non_blocking=True)
            ne[0] += 1
            dp.step(grads)
            torch.cat([x for d in dps for x in (d.mu[:d.plan.T], d.s_g[:d.plan.T], d.sat[:d.plan.T].float(),
                                                d.skip.float())], out=out_d)
            out_h.copy_(out_d, non_blocking=True)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        e2e = {"value": N * bytes_rank / (ems / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": set_bytes,
               "d2h_bytes_per_step": out_h.numel() * 4}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline and not args.quick:
        cpu = cpu_baseline(args, specs)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config] + (", ZeRO owner mode (Alg. 1)" if zero else ""),
                       "tensors": len(numels), "params": params, "grad_dtype": args.dtype,
                       "buckets": nb, "bucket_lag": args.bucket_lag, "lr": args.lr,
                       "cuda_graph": bool(args.graph and nb == 1),
                       "case": "worst (amax(w') screen fallback)" if args.worst_case else "typical",
                       "alg_bytes_per_param_per_rank": bytes_rank / params,
                       "parallelism": f"dp{N}" if N > 1 else (f"{sim} simulated ranks" if sim else "single"), "state_scaling": args.state_scaling,
                       "exchange": (args.exchange if N > 1 else "none"),
                       "l2": "inputs larger than L2 (step moves %.2f GB/rank > 126 MB)" % (bytes_rank / 1e9),
                       "grad_sets_rotated": R, "grad_sets_antithetic": R % 2 == 0,
                       "hbm_frac_of_8tbs": value / N / 8000.0},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clocks, "kernels": breakdown,
            "ms_per_step_instrumented": ms_prof,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        import torch.distributed as dist
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
