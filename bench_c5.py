#!/usr/bin/env python
"""Config C5 (BASELINE.json configs[4]): FP8 gradient all-reduce message-size sweep vs
NCCL bf16, under torchrun on N GPUs of one box.

For every FP8 payload size n (bytes = elements) it times, max over ranks, CUDA events:
  p2p_full  — fp8lm_allreduce_jit (= amax_scale_sync + fp8_grad_allreduce) in mode P2P
              from an fp32 gradient: up to 1 MiB ONE kernel (amax, MIN of the scales
              through the peer pads, the one-shot exchange), above it amax + quantize + the
              fused peer-memory reduce-scatter + rank-order reduce + all-gather
  p2p_raw_full — up to 1 MiB: the one-handshake raw one-shot (k_oneshot_raw: every rank
              pulls the fp32 gradients and encodes them itself)
  p2p_rsag_full — up to 1 MiB: the same with the one-shot path off (quantize + RS + AG)
  p2p_xchg  — the fused exchange kernel alone (k_reduce_p2p, library launch tracing)
  nccl_full — the same arithmetic with NCCL transport (mode NCCL)
  nccl_bf16 — torch.distributed.all_reduce of n bf16 elements (NCCL, default algorithm)
  nccl_f32  — the same in fp32
and prints one JSON line per (size, impl) with time, algbw (payload bytes / time: n for
FP8, 2n for bf16, 4n for fp32) and busbw = algbw * 2(N-1)/N.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        bench_c5.py --min-log2 10 --max-log2 30 --stride 2
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def timed(fn, iters, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], dtype=torch.float32, device="cuda")   # NVLS: no f64
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() * 1e3          # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--stride", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--src-dtype", default="f32", choices=["f32", "bf16"],
                    help="gradient dtype of the FP8 rows (A1-A5 from fp32 or from bf16); the "
                         "NCCL rows are unchanged")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    import synth

    comm = B.Comm.from_torch_distributed()
    busf = 2.0 * (N - 1) / N
    rows = []
    for lg in range(args.min_log2, args.max_log2 + 1, args.stride):
        n = 1 << lg
        iters = max(5, min(args.iters, int(2e9 // n)))
        g = torch.empty(n, dtype=torch.float32, device="cuda")
        synth.fill_gradient(g, 1, 0, rank, amp=1e-3)
        if args.src_dtype == "bf16":
            g = g.to(torch.bfloat16)
        res = {}
        for mode_name, mode, oneshot in (("p2p_raw", B.MODE_P2P, "raw"), ("p2p", B.MODE_P2P, True),
                                         ("p2p_rsag", B.MODE_P2P, False), ("nccl", B.MODE_NCCL, False)):
            if mode_name in ("p2p_rsag", "p2p_raw") and n > (1 << 20):
                continue                       # above 1 MiB the p2p rows are the RS+AG path
            plan = B.Plan([n], mode=mode, nranks=N, rank=rank)
            if mode == B.MODE_P2P:
                plan.set_oneshot((1 << 20) if oneshot else 0)
                # p2p_raw: one handshake (k_oneshot_raw); p2p: two (k_oneshot_full)
                plan.set_oneshot_raw((1 << 20) if oneshot == "raw" else 0)
                plan.peer_setup(comm)
                g8 = plan.peer_g8()
                c = None
            else:
                g8 = plan.flat(torch.uint8, nbytes_like_g8=True)
                c = comm
            mu = torch.ones(1, device="cuda")
            amax = torch.zeros(1, device="cuda")
            s_g = torch.zeros(1, device="cuda")
            skip = torch.zeros(1, dtype=torch.int32, device="cuda")
            gs = torch.zeros(1, device="cuda")
            gsi = torch.zeros(1, device="cuda")
            sat = torch.zeros(1, dtype=torch.int32, device="cuda")

            def full():       # A1-A5: fp8lm_allreduce_jit (P2P small plans: one kernel)
                B.allreduce_jit(plan, g, mu, amax, s_g, skip, g8, gs, gsi, sat, comm=c)

            res[f"{mode_name}_full"] = timed(full, iters)
            if mode == B.MODE_P2P:
                # the same two calls captured in a CUDA graph: one host call per step (the
                # flag epochs live in device counters, so every replay is a new step)
                gr = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr):
                    full()
                res[f"{mode_name}_full_graph"] = timed(gr.replay, iters)
                del gr
            B.prof_enable(True)                  # a second, instrumented pass for the kernel
            timed(full, iters)
            B.prof_enable(False)
            prof = B.prof_read()
            if mode_name == "p2p" and "reduce_p2p" in prof:
                t = torch.tensor([prof["reduce_p2p"]["ms"] / prof["reduce_p2p"]["launches"]],
                                 dtype=torch.float32, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                res["p2p_xchg"] = t.item() * 1e3
            del plan, g8
        for dt, name, esz in ((torch.bfloat16, "nccl_bf16", 2), (torch.float32, "nccl_f32", 4)):
            x = torch.ones(n, dtype=dt, device="cuda")
            res[name] = timed(lambda: dist.all_reduce(x), iters)
            if dt == torch.bfloat16:
                gr = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.graph(gr):
                    dist.all_reduce(x)
                res[name + "_graph"] = timed(gr.replay, iters)
                del gr
            del x
        for impl, us in res.items():
            payload = n * (2 if impl.startswith("nccl_bf16") else 4 if impl == "nccl_f32" else 1)
            algbw = payload / (us * 1e-6) / 1e9
            row = {"config": "C5", "n_gpus": N, "elements": n, "fp8_bytes": n, "impl": impl,
                   "src_dtype": {"nccl_bf16": "bf16", "nccl_bf16_graph": "bf16", "nccl_f32": "f32"}.get(impl, args.src_dtype),
                   "nccl_algo": os.environ.get("NCCL_ALGO", "default"),
                   "us": us, "algbw_GBs": algbw, "busbw_GBs": algbw * busf,
                   "busbw_frac_of_900": algbw * busf / 900.0}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
        del g
        torch.cuda.empty_cache()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
