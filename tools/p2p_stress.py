"""Stress the mode-P2P step under torchrun: many steps with a host synchronisation per
step (ranks drift against each other), reporting the step at which anything fails.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/p2p_stress.py
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--mode", default="p2p")
    ap.add_argument("--jitter", action="store_true", help="random host sleeps per rank")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    import synth
    specs = synth.gpt_gradient_set("gpt-125m", None)
    comm = B.Comm.from_torch_distributed()
    mode = {"p2p": B.MODE_P2P, "zero": B.MODE_ZERO}[args.mode]
    plan = B.Plan([s.numel for s in specs], mode=mode, nranks=N, rank=rank)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    gs = []
    for r_ in range(2):
        g = plan.flat(torch.float32)
        for t, v in enumerate(plan.views(g)):
            synth.fill_gradient(v, 1 + r_, t, rank)
        gs.append(g)
    dp = B.FP8DataParallel(plan, w0, comm=comm, lr=6e-4)
    import random
    rnd = random.Random(rank)
    t0 = time.time()
    for i in range(args.steps):
        dp.step(gs[i % 2])
        try:
            torch.cuda.synchronize()
        except Exception as e:
            print(f"rank {rank}: FAILED at step {i}: {e}", flush=True)
            raise
        if args.jitter and rnd.random() < 0.1:
            time.sleep(rnd.random() * 0.003)
        if i % 500 == 0 and rank == 0:
            print(f"step {i} ok ({time.time() - t0:.1f} s)", flush=True)
    print(f"rank {rank}: all {args.steps} steps ok", flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
