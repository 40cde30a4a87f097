"""torchrun worker for the multi-GPU parity test (tests/test_gpu_nccl.py).

Each rank runs the NCCL-mode hot path (fp8lm_amax_scale_sync -> fp8lm_grad_allreduce
[all-to-all, rank-order reduce, all-gather] -> fp8lm_adam_step) on its own synthetic
gradients, regenerates every other rank's gradients locally (synth is deterministic),
runs the N-rank CPU oracle and compares its own outputs element by element.  Exit code 0
iff every rank matched bit-exactly.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/dist_worker.py [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import adam as OA  # noqa: E402
from oracle import step as OS  # noqa: E402
from tests import _gpu_ref as R  # noqa: E402

F32 = np.float32
NUMELS = [3, 16, 17, 64, 1000, 16384, 16385, 40000, 70001, 5]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--lr", type=float, default=3e-4)
    ap.add_argument("--mode", choices=["nccl", "p2p", "zero"], default="nccl")
    ap.add_argument("--unfused", action="store_true",
                    help="the three ABI calls instead of fp8lm_dp_step")
    ap.add_argument("--delayed", action="store_true", help="delayed state scaling (R25-R27)")
    ap.add_argument("--oneshot", action="store_true", help="mode P2P: the one-shot small-message exchange")
    ap.add_argument("--raw", action="store_true", help="with --oneshot: the one-handshake raw one-shot")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B

    comm = B.Comm.from_torch_distributed()
    mode = {"p2p": B.MODE_P2P, "nccl": B.MODE_NCCL, "zero": B.MODE_ZERO}[args.mode]
    plan = B.Plan(NUMELS, mode=mode, nranks=N, rank=rank)
    plan.set_oneshot(1 << 40 if args.oneshot else 0)
    plan.set_oneshot_raw(1 << 40 if args.raw else 0)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    dp = B.FP8DataParallel(plan, w0, comm=comm, lr=args.lr, fused=not args.unfused,
                           state_scaling="delayed" if args.delayed else "jit")
    ref_states = R.oracle_init(plan, w0)
    mus = [F32(1.0)] * plan.T
    hists = [OA.init_history(st) for st in ref_states] if args.delayed else None
    ok = True
    msgs = []
    for step in range(1, args.steps + 1):
        # every rank's gradient, generated here (rank r's own buffer is the input)
        all_grads = []
        for r in range(N):
            flat = plan.flat(torch.float32)
            for t, v in enumerate(plan.views(flat)):
                synth.fill_gradient(v, step, t, r)
            if step == 2 and r == N - 1:
                flat[plan.offsets[4] + 7] = 3.0e5      # one huge value: sum saturates, mu halves
            all_grads.append(flat)
        dp.step(all_grads[rank], lr=args.lr)
        torch.cuda.synchronize()
        gnp = [R.to_np_f32(g) for g in all_grads]
        per_rank = [[g[plan.offsets[t]: plan.offsets[t] + plan.numels[t]] for t in range(plan.T)]
                    for g in gnp]
        res = OS.train_step(per_rank, mus, ref_states, OA.hyper_params(args.lr, step), hists=hists,
                            step=step)
        if args.delayed:
            hists = res["hists"]
        for m in R.compare_rank(B, plan, dp, res, rank, args.mode, not args.unfused and not args.oneshot):
            ok = False
            msgs.append(f"step {step}: {m}")
        mus = res["mu_next"]
        ref_states = res["states"]
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    for m in msgs[:10]:
        print(m, flush=True)
    if rank == 0:
        tag = args.mode.upper() + ("_UNFUSED" if args.unfused else "") + ("_DELAYED" if args.delayed else "") + \
            ("_ONESHOT" if args.oneshot else "") + ("_RAW" if args.raw else "")
        print(f"{tag} parity N={N}: {'OK' if flag.item() == 1 else 'MISMATCH'}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
