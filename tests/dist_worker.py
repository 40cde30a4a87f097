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


def check_zero(B, plan, dp, t, ref, where):
    """Mode ZERO: the owner's compact states of t, and every rank's replicated w8 of t."""
    w8 = dp.w8_full.cpu().numpy()[plan.offsets[t]: plan.offsets[t] + plan.numels[t]]
    sc = dp.w8_full_scalars.cpu().numpy()
    assert np.array_equal(w8, ref.w8.codes), f"{where}: replicated w8 differs"
    assert (F32(sc[0, t]), F32(sc[1, t]), F32(sc[2, t])) == (ref.w8.scale, ref.w8.scale_inv, ref.w8.amax), \
        f"{where}: replicated w8 scalars differ"
    if plan.owner(t) != dist.get_rank():
        return
    j = [tt for tt, _ in dp.layout.entries].index(t)
    o, n = dp.layout.offsets[j], plan.numels[t]
    st = dp.state
    got = dict(
        m1=st.m1.data[o:o + n].cpu().numpy(),
        v=st.v.data[o:o + n].cpu().view(torch.int16).numpy().view(np.uint16),
        master=st.master.data[o:o + n].cpu().view(torch.int16).numpy().view(np.uint16),
        w8=st.w8.data[o:o + n].cpu().numpy())
    for k in ("m1", "v", "master", "w8"):
        s_ = getattr(st, k)
        got[k + "_s"] = (F32(s_.scale[j].item()), F32(s_.scale_inv[j].item()), F32(s_.amax[j].item()))
    R.assert_state_equal(got, ref, where)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--lr", type=float, default=3e-4)
    ap.add_argument("--mode", choices=["nccl", "p2p", "zero"], default="nccl")
    ap.add_argument("--unfused", action="store_true",
                    help="the three ABI calls instead of fp8lm_dp_step")
    ap.add_argument("--delayed", action="store_true", help="delayed state scaling (R25-R27)")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B

    comm = B.Comm.from_torch_distributed()
    mode = {"p2p": B.MODE_P2P, "nccl": B.MODE_NCCL, "zero": B.MODE_ZERO}[args.mode]
    plan = B.Plan(NUMELS, mode=mode, nranks=N, rank=rank)
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
        g8 = dp.g8.cpu().numpy() if args.mode != "zero" else None
        s_g = dp.s_g.cpu().numpy()
        sat = dp.sat.cpu().numpy()
        mu = dp.mu.cpu().numpy()
        gs = dp.g_scale.cpu().numpy()
        if bool(dp.skip.item()) != res["skip"]:
            ok = False
            msgs.append(f"step {step}: skip differs")
        for t in range(plan.T):
            p = res["per_tensor"][t]
            sl = slice(plan.offsets[t], plan.offsets[t] + plan.numels[t])
            if g8 is not None and args.mode == "p2p" and not args.unfused:
                # fused P2P step: the all-gather is pulled inside pass 2, so this rank's
                # window holds its own shard's codes only (include/fp8lm.h, fp8lm_dp_step)
                lo, hi = plan.shard_begin(rank), plan.shard_begin(rank) + plan.shard_bytes
                a, b = max(lo, sl.start), min(hi, sl.stop)
                codes_ok = a >= b or np.array_equal(g8[a:b], p["codes"][a - sl.start:b - sl.start])
            elif g8 is not None:
                codes_ok = np.array_equal(g8[sl], p["codes"])
            elif plan.owner(t) == rank:                       # ZeRO: only the owner reduces t
                j = [tt for tt, _ in dp.layout.entries].index(t)
                o = dp.layout.offsets[j]
                codes_ok = np.array_equal(dp.g8.cpu().numpy()[o:o + plan.numels[t]], p["codes"])
            else:
                codes_ok = True
            checks = [
                ("codes", codes_ok),
                ("s_g", F32(s_g[t]) == p["s_g"]),
                ("sat", int(sat[t]) == p["sat"]),
                ("scale", F32(gs[t]) == p["scale"]),
                ("mu", F32(mu[t]) == res["mu_next"][t]),
            ]
            for name, good in checks:
                if not good:
                    ok = False
                    msgs.append(f"rank {rank} step {step} tensor {t}: {name} differs")
            try:
                if args.mode == "zero":
                    check_zero(B, plan, dp, t, res["states"][t], f"rank {rank} step {step} tensor {t}")
                else:
                    R.assert_state_equal(R.state_np(B, plan, dp.state, t), res["states"][t],
                                         f"rank {rank} step {step} tensor {t}")
            except AssertionError as e:
                ok = False
                msgs.append(str(e)[:300])
        mus = res["mu_next"]
        ref_states = res["states"]
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    for m in msgs[:10]:
        print(m, flush=True)
    if rank == 0:
        tag = args.mode.upper() + ("_UNFUSED" if args.unfused else "") + ("_DELAYED" if args.delayed else "")
        print(f"{tag} parity N={N}: {'OK' if flag.item() == 1 else 'MISMATCH'}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
