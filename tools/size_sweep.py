"""Per-kernel time vs size at N = 1 (LOCAL dp_step, one tensor of n fp32 elements, or the
GPT-125M layout scaled): fits t = a + n * b per kernel, so a is the fixed cost of a launch
(ramp-up, tail, epilogue) and 1/b the asymptotic bandwidth.  Also times torch's own
read-only (max) and copy kernels on the same sizes.

    python tools/size_sweep.py [--state-scaling jit|delayed]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--state-scaling", default="jit")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--split", default="",
                    help="comma list of K: time n = 2^27 split into K equal tensors instead")
    args = ap.parse_args()
    import paper_2310_18313_b200 as B
    import synth
    rows = []
    cases = ([(1 << 27, int(k)) for k in args.split.split(",")] if args.split
             else [(1 << lg, 1) for lg in range(22, 30)])
    for n, K in cases:
        plan = B.Plan([n // K] * K, mode=B.MODE_LOCAL)
        w0 = plan.flat(torch.float32)
        for t, v in enumerate(plan.views(w0)):
            synth.fill_weights(v, t)
        gs = []
        for k in range(2):
            g = plan.flat(torch.float32)
            for t, v in enumerate(plan.views(g)):
                synth.fill_gradient(v, 1, t, 0, amp=1e-3)
            if k:
                g.neg_()
            gs.append(g)
        dp = B.FP8DataParallel(plan, w0, lr=6e-4, state_scaling=args.state_scaling)
        del w0
        for i in range(5):
            dp.step(gs[i % 2])
        torch.cuda.synchronize()
        B.prof_enable(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.steps):
            dp.step(gs[i % 2])
        b.record()
        torch.cuda.synchronize()
        B.prof_enable(False)
        prof = B.prof_read()
        row = {"n": n, "tensors": K, "step_us": a.elapsed_time(b) / args.steps * 1e3}
        for k, v in prof.items():
            row[k] = v["ms"] / v["launches"] * 1e3
        x = gs[0]
        y = torch.empty_like(x)
        for name, fn in (("torch_max", lambda: x.max()), ("torch_copy", lambda: y.copy_(x))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a.record()
            for _ in range(args.steps):
                fn()
            b.record()
            torch.cuda.synchronize()
            row[name] = a.elapsed_time(b) / args.steps * 1e3
        print(json.dumps(row), flush=True)
        rows.append(row)
        del dp, gs, x, y, plan
        torch.cuda.empty_cache()
    if args.split:
        return
    # least-squares fit over the 4 largest sizes
    import numpy as np
    keys = [k for k in rows[-1] if k not in ("n", "tensors")]
    fit = {}
    for k in keys:
        pts = [(r["n"], r[k]) for r in rows[-4:] if k in r]
        if len(pts) < 2:
            continue
        A = np.array([[1.0, p[0]] for p in pts])
        y_ = np.array([p[1] for p in pts])
        c, *_ = np.linalg.lstsq(A, y_, rcond=None)
        fit[k] = {"fixed_us": float(c[0]), "ns_per_elem": float(c[1] * 1e3)}
    print(json.dumps({"fit": fit}), flush=True)


if __name__ == "__main__":
    main()
