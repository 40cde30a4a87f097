"""Every tensor of a big gradient set checked against the oracle in parallel (tests only).

Nothing in the method couples two tensors except the skip flag, so the
oracle runs per tensor: a pool of worker processes (one core each) owns the tensors
(largest first to the least loaded worker) and keeps their oracle state across steps.
Per step the parent writes the step's flat gradient and the device's outputs to files in
/dev/shm; every worker runs oracle.step.train_step on its tensors (N = 1) and compares
the device outputs with the oracle's element by element, returning mismatch messages.
"""
from __future__ import annotations

import os
import tempfile

import numpy as np

F32 = np.float32
STATE_KEYS = ("m1", "v", "master", "w8")


def _worker(conn, tensors, offsets, numels, w0_path, lr):
    import numpy as np
    from oracle import adam as OA
    from oracle import step as OS
    w0 = np.load(w0_path, mmap_mode="r")
    states = [OA.init_state(np.array(w0[offsets[t]: offsets[t] + numels[t]])) for t in tensors]
    mus = [F32(1.0)] * len(tensors)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        step, gpath, dpath = msg
        g = np.load(gpath, mmap_mode="r")
        dev = np.load(dpath)
        grads = [[np.array(g[offsets[t]: offsets[t] + numels[t]]) for t in tensors]]
        res = OS.train_step(grads, mus, states, OA.hyper_params(lr, step), step=step)
        bad = []
        for i, t in enumerate(tensors):
            p = res["per_tensor"][i]
            sl = slice(offsets[t], offsets[t] + numels[t])
            where = f"step {step} tensor {t} (n={numels[t]})"
            if not np.array_equal(dev["g8"][sl], p["codes"]):
                bad.append(f"{where}: reduced codes")
            for k, v in (("s_g", p["s_g"]), ("scale", p["scale"]), ("mu", res["mu_next"][i])):
                if F32(dev[k][t]) != F32(v):
                    bad.append(f"{where}: {k} {dev[k][t]} vs {v}")
            if int(dev["sat"][t]) != p["sat"]:
                bad.append(f"{where}: sat")
            st = res["states"][i]
            for k in STATE_KEYS:
                r = getattr(st, k)
                if not np.array_equal(dev[k][sl].astype(np.int64), r.codes.astype(np.int64)):
                    bad.append(f"{where}: {k} codes")
                got = (F32(dev[k + "_scale"][t]), F32(dev[k + "_scale_inv"][t]), F32(dev[k + "_amax"][t]))
                if got != (r.scale, r.scale_inv, r.amax):
                    bad.append(f"{where}: {k} scalars {got} vs {(r.scale, r.scale_inv, r.amax)}")
        states, mus = res["states"], res["mu_next"]
        conn.send(bad)


class OraclePool:
    def __init__(self, plan, w0_flat_np, lr, workers=None):
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        self.dir = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
        w0p = os.path.join(self.dir, "w0.npy")
        np.save(w0p, w0_flat_np)
        W = max(1, min(workers or len(os.sched_getaffinity(0)), plan.T))
        load = [0] * W
        parts = [[] for _ in range(W)]
        for t in sorted(range(plan.T), key=lambda t: -plan.numels[t]):
            j = min(range(W), key=lambda k: load[k])
            parts[j].append(t)
            load[j] += plan.numels[t]
        self.conns, self.procs = [], []
        for part in parts:
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_worker, args=(b, sorted(part), plan.offsets, plan.numels, w0p, lr),
                             daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for c in self.conns:
            assert c.recv() == "ready"

    def check(self, step, grad_flat_np, dev: dict):
        gp = os.path.join(self.dir, f"g{step}.npy")
        dp = os.path.join(self.dir, f"d{step}.npz")
        np.save(gp, grad_flat_np)
        np.savez(dp, **dev)
        for c in self.conns:
            c.send((step, gp, dp))
        bad = []
        for c in self.conns:
            bad += c.recv()
        os.unlink(gp)
        os.unlink(dp)
        return bad

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=60)
        import shutil
        shutil.rmtree(self.dir, ignore_errors=True)
