"""Fig. 6 of PAPER.md: SNR, underflow rate and overflow rate of pre-scaling,
post-scaling and automatic scaling for the FP8 gradient all-reduce, per Transformer block
of GPT-7B at data parallelism 128 — on synthetic gradients, through
fp8lm_allreduce_strategy.

Synthetic recipe: per block b of the 32 GPT-7B blocks and per weight
tensor of the block (qkv, proj, fc1, fc2), N = 128 ranks hold
    g_r = a (rho_b c + sqrt(1 - rho_b^2) z_r),   c, z_r ~ Student-t(3),
a sample of n elements per tensor (default 2^22), a fresh draw every step.  Per-tensor
scaling makes the statistics independent of the amplitude a, so blocks differ through
the cross-rank correlation rho_b, swept linearly from 0 (block 0) to 0.95 (block 31):
uncorrelated ranks sum like sqrt(N), correlated ranks like N, which is what separates
pre-scaling's underflow from post-scaling's overflow.  Auto-scaling runs `--steps`
steps per tensor (mu evolves, R1-R3); all three strategies are evaluated on the last
step's gradients.  Prints one JSON line per (block, strategy) and a summary line with
the strategy kernels' throughput (2 x 4 B per rank-element read).

    python tools/fig6.py [--blocks 0,4,...] [--n 4194304] [--steps 16]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

D_MODEL = 4096
TENSORS = ("qkv.w", "proj.w", "fc1.w", "fc2.w")


def student_t3(shape, gen, dev):
    z = torch.randn(shape, generator=gen, device=dev)
    chi = torch.randn((3,) + tuple(shape), generator=gen, device=dev).square_().sum(0)
    return z / torch.sqrt(chi / 3.0)


def draw(out, N, n, rho, seed, dist="t3", sigma=2.0):
    """t3: a (rho c + sqrt(1-rho^2) z_r), c, z_r ~ Student-t(3).
    lognormal: magnitudes a exp(sigma (rho c + sqrt(1-rho^2) z_r)) with signs
    sign(rho u + sqrt(1-rho^2) v_r), c, z_r, u, v_r ~ N(0, 1): correlated log-normal
    magnitudes and correlated signs across ranks, sigma = the spread in natural-log units."""
    gen = torch.Generator(device=out.device)
    gen.manual_seed(seed)
    k = math.sqrt(1.0 - rho * rho)
    if dist == "t3":
        c = student_t3((n,), gen, out.device)
        z = student_t3((N, n), gen, out.device)
        out.copy_(z.mul_(k).add_(c.mul_(rho)).mul_(1e-3))
        return
    c = torch.randn((n,), generator=gen, device=out.device)
    z = torch.randn((N, n), generator=gen, device=out.device)
    u = torch.randn((n,), generator=gen, device=out.device)
    v = torch.randn((N, n), generator=gen, device=out.device)
    mag = z.mul_(k).add_(c.mul_(rho)).mul_(sigma).exp_().mul_(1e-5)
    sgn = torch.sign(v.mul_(k).add_(u.mul_(rho)))
    out.copy_(mag.mul_(sgn))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=128)
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--blocks", default="0,4,8,12,16,20,24,28,31")
    ap.add_argument("--dist", default="t3", choices=["t3", "lognormal"])
    ap.add_argument("--sigma", type=float, default=2.0)
    args = ap.parse_args()
    import paper_2310_18313_b200 as B
    dev = torch.device("cuda")
    N, n = args.ranks, args.n
    g = torch.empty(N, n, dtype=torch.float32, device=dev)
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    st = B.commstats_buffer(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_ms, t_calls = 0.0, 0
    B.prof_enable(True)
    for b in [int(x) for x in args.blocks.split(",")]:
        rho = 0.95 * b / 31.0
        agg = {s: dict(sig2=0.0, err2=0.0, underflow=0, overflow=0, events=0) for s in B.STRATEGIES}
        mus = []
        for ti, name in enumerate(TENSORS):
            mu = torch.ones(1, device=dev)
            for step in range(args.steps):
                draw(g, N, n, rho, seed=(b * 16 + ti) * 1000 + step, dist=args.dist, sigma=args.sigma)
                last = step == args.steps - 1
                for strat in (("pre", "post", "auto") if last else ("auto",)):
                    torch.cuda.synchronize()
                    ev0.record()
                    B.allreduce_strategy(g, strat, mu, codes=codes, stats=st)
                    ev1.record()
                    torch.cuda.synchronize()
                    t_ms += ev0.elapsed_time(ev1)
                    t_calls += 1
                    if last:
                        d = B.commstats_read(st)
                        for k in agg[strat]:
                            agg[strat][k] += d[k]
                        if strat == "auto":
                            mus.append(d["mu_used"])
        for strat, a in agg.items():
            # the metrics of the summed statistics, computed by the library (R29-R30)
            snr, ur, orate = B.commstats_metrics(a["sig2"], a["err2"], int(a["underflow"]), int(a["overflow"]),
                                                 int(a["events"]))
            row = {"fig": 6, "model": "gpt-7b", "block": b, "rho": round(rho, 4), "dp": N,
                   "n_per_tensor": n, "tensors": list(TENSORS), "strategy": strat, "dist": args.dist,
                   "sigma": args.sigma if args.dist == "lognormal" else None,
                   "snr_db": snr, "underflow_rate": ur, "overflow_rate": orate}
            if strat == "auto":
                row["mu"] = mus
            print(json.dumps(row), flush=True)
    B.prof_enable(False)
    prof = {k: v["ms"] / v["launches"] for k, v in B.prof_read().items()}
    per_call = t_ms / t_calls
    gbs = 8.0 * N * n / (per_call / 1e3) / 1e9
    print(json.dumps({"summary": "strategy kernels", "ranks": N, "n": n,
                      "ms_per_call": per_call, "alg_GBps": gbs,
                      "alg_bytes_per_call": 8 * N * n,
                      "kernel_ms": prof,
                      "kernel_GBps": {k: 4.0 * N * n / (v / 1e3) / 1e9 for k, v in prof.items()},
                      "note": "amax pass + strategy pass, each reads the N x n fp32 block once"}),
          flush=True)


if __name__ == "__main__":
    main()
