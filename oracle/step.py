"""Oracle of one whole data-parallel step: the FP8 gradient all-reduce of every tensor
(§2.1) followed by the FP8 AdamW update (§2.2), for N simulated ranks.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Composition only — every arithmetic step lives in ``pipeline`` and ``adam``:
  for each tensor t:   allreduce_tensor (amax, s_r, s_g = min, quantize, rank-order
                       sum, requantize, sat, s = N*s_g)
  skip = any tensor has s_g == 0 (a non-finite gradient on some rank; R14)
  for each tensor t:   g_hat = dequantize; AdamW unless skip; mu_t <- mu_update
Data parallelism needs no change to the arithmetic; every rank applies the
same update, so the optimizer runs once here.
"""
from __future__ import annotations

from typing import List

import numpy as np

from . import adam as A
from . import pipeline as P


def train_step(grads_by_rank: List[List[np.ndarray]], mus: List[np.float32],
               states: List[A.OptState], hp: A.AdamHP, run_adam: bool = True,
               hists=None, step: int = 1):
    """grads_by_rank[r][t] -> dict(per_tensor=[...], skip, mu_next=[...], states=[...]).
    hists (list of amax(w) rings): delayed state scaling (App. B) instead of JIT;
    the updated rings are returned as "hists"."""
    N = len(grads_by_rank)
    T = len(grads_by_rank[0])
    per = []
    for t in range(T):
        per.append(P.allreduce_tensor([grads_by_rank[r][t] for r in range(N)], mus[t]))
    skip = any(p["skip"] for p in per)
    new_states = []
    for t in range(T):
        p = per[t]
        p["g_hat"] = P.dequantize(p["codes"], p["scale_inv"])
        if run_adam and hists is not None:
            res = A.adam_step_delayed(p["g_hat"], states[t], hp, p["scale_inv"], hists[t], step, skip)
            p["adam"] = res
            new_states.append(res["state"])
        elif run_adam:
            res = A.adam_step(p["g_hat"], states[t], hp, skip)
            p["adam"] = res
            new_states.append(res["state"])
    mu_next = [P.mu_update(mus[t], per[t]["sat"], per[t]["n"], skip) for t in range(T)]
    return dict(per_tensor=per, skip=skip, mu_next=mu_next,
                states=new_states if run_adam else states,
                hists=[p["adam"]["hist"] for p in per] if (run_adam and hists is not None) else None)
