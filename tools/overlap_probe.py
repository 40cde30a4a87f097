"""Feasibility probe for overlapping the P2P exchange with HBM-bound AdamW work.

Times, per rank, (a) the mode-P2P all-reduce (quantize + fused exchange kernel) alone,
(b) a LOCAL-plan AdamW step (pass 1 + pass 2) on an independent state set alone, and
(c) both at once on two streams.  If (c) is close to max(a, b), a bucketed step that
runs pass 2 of bucket b under the exchange of bucket b+1 pays off.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/overlap_probe.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt-125m")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    import synth
    specs = synth.gpt_gradient_set(args.config, args.layers)
    numels = [s.numel for s in specs]
    comm = B.Comm.from_torch_distributed()
    pp = B.Plan(numels, mode=B.MODE_P2P, nranks=N, rank=rank)
    pl = B.Plan(numels, mode=B.MODE_LOCAL)
    g = pp.flat(torch.float32)
    for t, v in enumerate(pp.views(g)):
        synth.fill_gradient(v, 1, t, rank)
    w0 = pl.flat(torch.float32)
    for t, v in enumerate(pl.views(w0)):
        synth.fill_weights(v, t)
    dpp = B.FP8DataParallel(pp, w0, comm=comm, lr=3e-4)
    dpl = B.FP8DataParallel(pl, w0, lr=3e-4, fused=False)
    g8l = dpl.g8
    g8l.copy_(torch.randint(0, 0x7E, g8l.shape, dtype=torch.uint8, device=g8l.device))
    dpl.g_scale_inv.fill_(1e-4)
    sx = torch.cuda.Stream()
    sa = torch.cuda.Stream()
    T = len(numels)

    def exch():
        with torch.cuda.stream(sx):
            B.amax_scale_sync(pp, g, dpp.mu, dpp.amax, dpp.s_g, dpp.skip, None, sx)
            B.fp8_grad_allreduce(pp, g, dpp.s_g, dpp.skip, dpp.g8, dpp.g_scale, dpp.g_scale_inv,
                                 dpp.sat, dpp.mu, None, sx)

    def adam(t):
        with torch.cuda.stream(sa):
            hp = B.adam_hp(3e-4, t)
            B.fp8_adam_step(pl, g8l, dpl.g_scale_inv, dpl.state, hp, dpl.skip, sa)

    def timeit(fn):
        for i in range(3):
            fn(i + 1)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.iters):
            fn(i + 4)
        # join both side streams into the current stream
        ev = torch.cuda.Event()
        for s in (sx, sa):
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / args.iters], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    def both(i):
        # the side streams start after the current stream's e0
        ev = torch.cuda.Event()
        ev.record()
        sx.wait_event(ev)
        sa.wait_event(ev)
        exch()
        adam(i)
        ev2 = torch.cuda.Event()
        for s in (sx, sa):
            ev2.record(s)
            torch.cuda.current_stream().wait_event(ev2)

    def only_x(i):
        ev = torch.cuda.Event()
        ev.record()
        sx.wait_event(ev)
        exch()
        ev.record(sx)
        torch.cuda.current_stream().wait_event(ev)

    def only_a(i):
        ev = torch.cuda.Event()
        ev.record()
        sa.wait_event(ev)
        adam(i)
        ev.record(sa)
        torch.cuda.current_stream().wait_event(ev)

    a = timeit(only_x)
    b = timeit(only_a)
    c = timeit(both)
    if rank == 0:
        print(json.dumps({"config": args.config, "layers": args.layers,
                          "p2p_per_sm": os.environ.get("FP8LM_P2P_PER_SM"), "N": N, "T": T, "exchange_ms": a, "adam_ms": b,
                          "both_ms": c, "sum_ms": a + b, "max_ms": max(a, b)}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
