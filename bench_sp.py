#!/usr/bin/env python
"""FP8 activation converter g (§2.3, Fig. 5; Table 7) under torchrun:
the all-gather (forward) and reduce-scatter (backward) between the sequence- and
tensor-parallel regions, FP8 over NVLink peer memory (fp8lm_sp_*) against NCCL's bf16
all_gather_into_tensor / reduce_scatter_tensor on the same activation.

Workloads (Table 7 rows, one converter call per Transformer layer and direction):
  gpt13b_tp2   micro-batch 2 x seq 2048 x hidden 5120  (TP = 2)
  gpt175b_tp8  micro-batch 1 x seq 2048 x hidden 12288 (TP = 8, or the N available)
Each line: time per call (max over ranks, CUDA events), bytes each rank sends over
NVLink ((N-1) m for FP8, 2 (N-1) m for bf16) and the speed-up over NCCL bf16.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 bench_sp.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

WORKLOADS = {"gpt13b_tp2": (2 * 2048, 5120), "gpt175b_tp8": (1 * 2048, 12288)}


def timed(fn, iters, warm=5):
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
    t = torch.tensor([a.elapsed_time(b) / iters], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    comm = B.Comm.from_torch_distributed()
    total_max = max(t * h for t, h in WORKLOADS.values())
    conv = B.SPConverter(max_elems=total_max, comm=comm)
    for name, (tokens, hidden) in WORKLOADS.items():
        full = tokens * hidden                    # the gathered activation
        m = full // N
        g = torch.Generator(device="cuda")
        g.manual_seed(rank)
        x = torch.randn(m, generator=g, device="cuda").to(torch.bfloat16)
        dy = torch.randn(full, generator=g, device="cuda").to(torch.bfloat16)
        ag_out = torch.empty(full, dtype=torch.bfloat16, device="cuda")
        rs_out = torch.empty(m, dtype=torch.bfloat16, device="cuda")
        res = {
            "fp8_allgather": timed(lambda: conv.allgather(x, out=ag_out), args.iters),
            "nccl_bf16_allgather": timed(lambda: dist.all_gather_into_tensor(ag_out, x), args.iters),
            "fp8_reduce_scatter": timed(lambda: conv.reduce_scatter(dy, out=rs_out), args.iters),
            "nccl_bf16_reduce_scatter": timed(lambda: dist.reduce_scatter_tensor(rs_out, dy), args.iters),
        }
        B.prof_enable(True)
        for _ in range(10):
            conv.allgather(x, out=ag_out)
            conv.reduce_scatter(dy, out=rs_out)
        torch.cuda.synchronize()
        B.prof_enable(False)
        kern = {k: v["ms"] / v["launches"] * 1e3 for k, v in B.prof_read().items()}
        if rank == 0:
            for op in ("allgather", "reduce_scatter"):
                f8, bf = res[f"fp8_{op}"], res[f"nccl_bf16_{op}"]
                print(json.dumps({
                    "bench": "sp_converter", "workload": name, "n_gpus": N, "op": op,
                    "elements_full": full, "elements_per_rank": m,
                    "fp8_us": f8, "nccl_bf16_us": bf, "speedup": bf / f8,
                    "nvlink_bytes_per_rank": {"fp8": (N - 1) * m, "bf16": 2 * (N - 1) * m},
                    "fp8_nvlink_GBps": (N - 1) * m / (f8 * 1e-6) / 1e9,
                    "kernel_us": kern}), flush=True)
    conv.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
