#!/usr/bin/env python
"""Phase timeline of the one-shot all-reduce kernels (diagnostic; needs an experiment build
with -D FP8LM_OS_TRACE loaded through FP8LM_LIB):

  FP8LM_LIB=build_ab/lib_trace.so torchrun --nproc-per-node 2 tools/os_trace.py

For each size and variant (raw: k_oneshot_raw, one handshake; full: k_oneshot_full, two)
it times fp8lm_allreduce_jit back to back (CUDA events, max over ranks), then runs one
more call and prints that call's globaltimer stamps relative to the kernel start on
every rank: 1 amax done (CTA 0), 2 last CTA of the amax, 3 MIN handshake done, 4 CTA 0
released, 5 quantize done (CTA 0), 6 last CTA publishes "ready", 7 CTA 0 past the ready
wait, 8 CTA 0 done pulling, 9 tail CTA, 10 tail done.
"""
import ctypes
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    import synth
    fn = B.lib.fp8lm_debug_os_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p]
    comm = B.Comm.from_torch_distributed()
    for n in (1024, 65536, 1 << 20):
        for variant in ("raw", "full"):
            plan = B.Plan([n], mode=B.MODE_P2P, nranks=N, rank=rank)
            plan.set_oneshot(1 << 20)
            plan.set_oneshot_raw((1 << 20) if variant == "raw" else 0)
            plan.peer_setup(comm)
            g = torch.empty(n, dtype=torch.float32, device="cuda")
            synth.fill_gradient(g, 1, 0, rank, amp=1e-3)
            g8 = plan.peer_g8()
            z = lambda dt=torch.float32: torch.zeros(1, dtype=dt, device="cuda")
            mu = torch.ones(1, device="cuda")
            amax, s_g, gs, gsi = z(), z(), z(), z()
            skip, sat = z(torch.int32), z(torch.int32)

            def call():
                B.allreduce_jit(plan, g, mu, amax, s_g, skip, g8, gs, gsi, sat)

            for _ in range(5):
                call()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                call()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 50 * 1e3], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.barrier()
            call()
            torch.cuda.synchronize()
            buf = (ctypes.c_ulonglong * 16)()
            fn(ctypes.addressof(buf))
            st = [int(x) for x in buf]
            rel = {i: round((st[i] - st[0]) / 1e3, 2) for i in range(1, 11) if st[i] >= st[0] > 0}
            rows = [None] * N
            dist.all_gather_object(rows, {"rank": rank, "stamps_us": rel})
            if rank == 0:
                print(json.dumps({"n": n, "variant": variant, "n_gpus": N, "us_per_call": t.item(),
                                  "ranks": rows}), flush=True)
            del plan, g8
            dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
