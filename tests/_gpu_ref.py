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
