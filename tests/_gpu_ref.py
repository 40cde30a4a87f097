"""Helpers for the GPU parity tests: run the CUDA path through the binding and the
oracle on the SAME seeded inputs, and compare every output element by element."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import adam as OA
from oracle import pipeline as OP
from oracle import step as OS

F32 = np.float32


def make_grads(plan, nranks, step, device, dtype=torch.float32, specials=None, amp=None):
    """Per rank: a flat gradient buffer in plan layout filled with synth values."""
    out = []
    for r in range(nranks):
        flat = plan.flat(dtype)
        for t, v in enumerate(plan.views(flat)):
            if v.numel():
                synth.fill_gradient(v, step, t, r, amp=None if amp is None else amp[t])
        if specials is not None:
            specials(flat, r)
        out.append(flat)
    return out


def to_np_f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float32)


def state_np(B, plan, st, t):
    """One tensor's optimizer state from the device -> dict of numpy arrays/scalars."""
    g = lambda s: plan.gather(s.data, t).detach().cpu()
    sc = lambda s: (F32(s.scale[t].item()), F32(s.scale_inv[t].item()), F32(s.amax[t].item()))
    return dict(
        m1=g(st.m1).numpy().astype(np.uint8), m1_s=sc(st.m1),
        v=g(st.v).view(torch.int16).numpy().view(np.uint16), v_s=sc(st.v),
        master=g(st.master).view(torch.int16).numpy().view(np.uint16), master_s=sc(st.master),
        w8=g(st.w8).numpy().astype(np.uint8), w8_s=sc(st.w8),
    )


def assert_state_equal(dev, ref: OA.OptState, where=""):
    for name, key in (("m1", "m1"), ("v", "v"), ("master", "master"), ("w8", "w8")):
        r = getattr(ref, key)
        d = dev[name]
        assert d.shape == r.codes.shape, (where, name)
        bad = np.nonzero(d.astype(np.int64) != r.codes.astype(np.int64))[0]
        assert bad.size == 0, f"{where} {name}: {bad.size} codes differ, first {bad[:5]} dev {d[bad[:5]]} ref {r.codes[bad[:5]]}"
        s, si, a = dev[name + "_s"]
        assert (s, si, a) == (r.scale, r.scale_inv, r.amax), (where, name, (s, si, a), (r.scale, r.scale_inv, r.amax))


def oracle_init(plan, w0_flat, sub=None):
    """Oracle initial states of the tensors in `sub` (default: all), copying only their
    slices of the device buffer to the host."""
    sub = range(plan.T) if sub is None else sub
    return [OA.init_state(to_np_f32(w0_flat[plan.offsets[t]: plan.offsets[t] + plan.numels[t]])) for t in sub]


def compare_rank(B, plan, dp, res, rank, mode, fused, sub=None):
    """One rank's outputs of one step of modes P2P / ZERO / NCCL vs the N-rank oracle
    result `res` (of the tensors in `sub`, default all).  Returns a list of mismatch
    messages (empty = bit-exact).  mode: "p2p" | "zero" | "nccl"."""
    sub = list(range(plan.T)) if sub is None else list(sub)
    msgs = []
    s_g = dp.s_g.cpu().numpy()
    sat = dp.sat.cpu().numpy()
    mu = dp.mu.cpu().numpy()
    gs = dp.g_scale.cpu().numpy()
    g8 = dp.g8.cpu().numpy()
    if bool(dp.skip.item()) != res["skip"]:
        msgs.append(f"rank {rank}: skip differs")
    own = [tt for tt, _ in dp.layout.entries] if mode == "zero" else None
    for i, t in enumerate(sub):
        p = res["per_tensor"][i]
        sl = slice(plan.offsets[t], plan.offsets[t] + plan.numels[t])
        if mode == "p2p" and fused:
            # fused P2P step: the all-gather is pulled inside the AdamW pass, so this rank's
            # window holds its own shard's codes only (include/fp8lm.h, fp8lm_dp_step)
            lo = plan.shard_begin(rank)
            hi = lo + plan.shard_bytes
            a, b = max(lo, sl.start), min(hi, sl.stop)
            codes_ok = a >= b or np.array_equal(g8[a:b], p["codes"][a - sl.start:b - sl.start])
        elif mode == "zero":
            if plan.owner(t) == rank:                    # ZeRO: only the owner reduces t
                o = dp.layout.offsets[own.index(t)]
                codes_ok = np.array_equal(g8[o:o + plan.numels[t]], p["codes"])
            else:
                codes_ok = True
        else:
            codes_ok = np.array_equal(g8[sl], p["codes"])
        if p["skip"]:
            codes_ok = True
        checks = [("codes", codes_ok), ("s_g", F32(s_g[t]) == p["s_g"]),
                  ("sat", p["skip"] or int(sat[t]) == p["sat"]), ("scale", F32(gs[t]) == p["scale"]),
                  ("mu", F32(mu[t]) == res["mu_next"][i])]
        for name, good in checks:
            if not good:
                msgs.append(f"rank {rank} tensor {t}: {name} differs")
        where = f"rank {rank} tensor {t}"
        try:
            ref = res["states"][i]
            if mode == "zero":
                w8 = dp.w8_full.cpu().numpy()[sl]
                sc = dp.w8_full_scalars.cpu().numpy()
                assert np.array_equal(w8, ref.w8.codes), f"{where}: replicated w8 differs"
                assert (F32(sc[0, t]), F32(sc[1, t]), F32(sc[2, t])) == \
                    (ref.w8.scale, ref.w8.scale_inv, ref.w8.amax), f"{where}: replicated w8 scalars differ"
                if plan.owner(t) == rank:
                    j = own.index(t)
                    o, n = dp.layout.offsets[j], plan.numels[t]
                    st = dp.state
                    got = dict(
                        m1=st.m1.data[o:o + n].cpu().numpy(),
                        v=st.v.data[o:o + n].cpu().view(torch.int16).numpy().view(np.uint16),
                        master=st.master.data[o:o + n].cpu().view(torch.int16).numpy().view(np.uint16),
                        w8=st.w8.data[o:o + n].cpu().numpy())
                    for k in ("m1", "v", "master", "w8"):
                        s_ = getattr(st, k)
                        got[k + "_s"] = (F32(s_.scale[j].item()), F32(s_.scale_inv[j].item()),
                                         F32(s_.amax[j].item()))
                    assert_state_equal(got, ref, where)
            else:
                assert_state_equal(state_np(B, plan, dp.state, t), ref, where)
        except AssertionError as e:
            msgs.append(str(e)[:300])
    return msgs
