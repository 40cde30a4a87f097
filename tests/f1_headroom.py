"""f1 analysis: how much E4M3 / FP16 range the delayed state scales of
R25 give away against JIT (App. B), measured with the oracle over a 200-step
run of one 262144-element tensor, N = 1.  Not a test (no assertions); run as

    python -m tests.f1_headroom [--steps 200] [--alpha 0.0] > profiles/r2/f1_headroom.json

Variants (each its own trajectory from the same initial weights and gradient stream):
  jit       state scales from the exact amax of the new values (R18)
  prior     delayed, R25 as built in round 1: |m| <= 448 m_sinv, v <= 65504 v_sinv
  recorded  delayed, the previous step's exact recorded amax through its largest code
Gradients: the synthetic recipe (synth, Student-t(3), one tensor's amplitude) per step,
optionally AR(1)-correlated across steps (alpha) to mimic a persistent gradient mean.
Per step after a 50-step burn-in: headroom log2(B / A) of m1 and v (0 for JIT), the
fraction of m1 codes that are zero or subnormal (exponent field 0), and the relative
L2 error of the dequantized m1 / v against the exact binary32 m', v' of the step.
Reads the oracle (allowed: tests/ infrastructure); this is measurement, not parity."""
import argparse
import json
import math
import multiprocessing as mp

import numpy as np


def run(variant, steps, alpha, n, seed):
    import torch
    import synth
    from oracle import adam as OA
    from oracle.codec import E4M3, FP16, decode_f32, encode
    F32 = np.float32
    w = torch.empty(n)
    synth.fill_weights(w, 7)
    st = OA.init_state(w.numpy())
    hist = OA.init_history(st)
    g_prev = np.zeros(n, np.float32)
    out = []
    for step in range(1, steps + 1):
        z = torch.empty(n)
        synth.fill_gradient(z, step, 7, 0)
        g = (F32(alpha) * g_prev + F32(math.sqrt(1 - alpha * alpha)) * z.numpy()).astype(F32)
        g_prev = g
        # N = 1 JIT gradient quantization (the reduced codes and their scale_inv)
        a = F32(np.abs(g).max())
        s = F32(F32(448.0) / a)
        codes = encode(g * s, E4M3)
        gsi = F32(F32(1.0) / s)
        ghat = (decode_f32(codes, E4M3) * gsi).astype(F32)
        hp = OA.hyper_params(3e-4, step)
        if variant == "jit":
            res = OA.adam_step(ghat, st, hp)
            bm = bv = None
        else:
            bm, bv = OA.delayed_moment_bounds(st, gsi, hp, variant)
            res = OA.adam_step_delayed(ghat, st, hp, gsi, hist, step, bound=variant)
            hist = res["hist"]
        new = res["state"]
        if step > 50:
            m, v = res["m"].astype(np.float64), res["v"].astype(np.float64)
            am, av = float(np.abs(m).max()), float(v.max())
            mdq = new.m1.value().astype(np.float64)
            vdq = new.v.value().astype(np.float64)
            out.append(dict(
                step=step,
                head_m=0.0 if bm is None else math.log2(float(bm) / am),
                head_v=0.0 if bv is None else math.log2(float(bv) / av),
                m_zero_or_sub=float(np.mean((new.m1.codes & 0x78) == 0)),
                m_zero=float(np.mean((new.m1.codes & 0x7F) == 0)),
                v_zero_or_sub=float(np.mean((new.v.codes.astype(np.int64) & 0x7C00) == 0)),
                err_m=float(np.linalg.norm(mdq - m) / np.linalg.norm(m)),
                err_v=float(np.linalg.norm(vdq - v) / np.linalg.norm(v))))
        st = new
    return variant, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--n", type=int, default=1 << 18)
    ap.add_argument("--alphas", default="0.0,0.9")
    a = ap.parse_args()
    jobs = [(v, a.steps, float(al), a.n, 0) for al in a.alphas.split(",") for v in ("jit", "prior", "recorded")]
    with mp.get_context("spawn").Pool(len(jobs)) as pool:
        res = pool.starmap(run, jobs)
    report = {}
    for (v, _, al, _, _), (_, rows) in zip(jobs, res):
        key = f"alpha={al}"
        agg = {k: float(np.mean([r[k] for r in rows])) for k in rows[0] if k != "step"}
        agg["head_m_max"] = float(max(r["head_m"] for r in rows))
        report.setdefault(key, {})[v] = agg
    print(json.dumps({"what": "tests/f1_headroom.py: oracle, one 262144-element tensor, N = 1, "
                      f"{a.steps} steps (means over steps 51..{a.steps})", "results": report}, indent=1))


if __name__ == "__main__":
    main()
