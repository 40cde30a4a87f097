"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element,
on the same seeded inputs.  Bar (BASELINE.json north_star): FP8 codes, FP16 state bits,
scales, amax, mu, sat bit-exact; the pinned binary32 sequence (R16) makes that
achievable, so the tolerances of the north star are not used as a licence.
"""
import numpy as np
import pytest
import torch

from tests.conftest import gpu_available
from tests import _gpu_ref as R
from tests.test_oracle_codec import _probe_inputs

from oracle import adam as OA
from oracle import pipeline as OP
from oracle import step as OS
from oracle.codec import E4M3, E5M2, FP16, decode, encode

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

F32 = np.float32
DEV = "cuda"


@pytest.fixture(scope="module")
def B():
    import paper_2310_18313_b200 as b
    return b


# ----------------------------------------------------------------- codec (App. A)
@pytest.mark.parametrize("fmt", ["e4m3", "e5m2", "f16"])
def test_codec_unit_scale_vs_oracle(B, fmt):
    """Device encode of 1M random + every (exponent x top-5-mantissa x low-bit pattern)
    binary32 input, unit scale, vs the oracle: bit-exact (NaN: class only)."""
    fcode = {"e4m3": B.E4M3, "e5m2": B.E5M2, "f16": B.F16}[fmt]
    ofmt = {"e4m3": E4M3, "e5m2": E5M2, "f16": FP16}[fmt]
    x = _probe_inputs(seed=2)
    xt = torch.from_numpy(x).to(DEV)
    scale = torch.ones(1, device=DEV)
    codes, *_ = B.fp8_quantize(xt, fcode, jit=False, scale=scale)
    got = codes.view(torch.int16).cpu().numpy().view(np.uint16) if fmt == "f16" else codes.cpu().numpy()
    ref = encode(x, ofmt)
    nan = np.isnan(x)
    bad = np.nonzero(got[~nan].astype(np.int64) != ref[~nan].astype(np.int64))[0]
    assert bad.size == 0, (bad.size, x[~nan][bad[:8]], got[~nan][bad[:8]], ref[~nan][bad[:8]])
    assert np.all(np.isnan(decode(got[nan], ofmt)))


@pytest.mark.parametrize("fmt", ["e4m3", "e5m2", "f16"])
def test_dequantize_every_code(B, fmt):
    fcode = {"e4m3": B.E4M3, "e5m2": B.E5M2, "f16": B.F16}[fmt]
    ofmt = {"e4m3": E4M3, "e5m2": E5M2, "f16": FP16}[fmt]
    n = 1 << ofmt.nbits
    codes = np.arange(n, dtype=np.int64)
    si = F32(0.0078125 * 3)
    if fmt == "f16":
        ct = torch.from_numpy(codes.astype(np.uint16).view(np.int16)).to(DEV).view(torch.float16)
    else:
        ct = torch.from_numpy(codes.astype(np.uint8)).to(DEV)
    out = B.fp8_dequantize(ct, fcode, torch.tensor([si], device=DEV)).cpu().numpy()
    ref = decode(codes, ofmt).astype(F32) * si
    fin = np.isfinite(ref)
    assert np.array_equal(out[fin], ref[fin])
    assert np.array_equal(np.isnan(out), np.isnan(ref))


def test_jit_quantize_single_tensor(B):
    """fp8_quantize(jit): amax, scale = fl(448/amax), codes (App. B JIT)."""
    rng = np.random.default_rng(4)
    for n in (1, 15, 16, 17, 1000, 65536 + 7):
        x = (rng.standard_t(3, size=n) * 1e-3).astype(F32)
        codes, s, si, a, sat = B.fp8_quantize(torch.from_numpy(x).to(DEV), B.E4M3, jit=True, count_sat=True)
        ref = OA.encode_scaled(x, E4M3, OA.E4M3_MAX, F32(np.abs(x).max()))
        assert F32(a.item()) == ref.amax and F32(s.item()) == ref.scale and F32(si.item()) == ref.scale_inv
        assert np.array_equal(codes.cpu().numpy(), ref.codes)
        assert sat.item() == OP.sat_count(ref.codes)
    # bf16 source: exact widening
    xb = torch.from_numpy((rng.standard_normal(4097) * 3).astype(F32)).to(DEV).bfloat16()
    codes, s, si, a, _ = B.fp8_quantize(xb, B.E4M3, jit=True)
    xf = xb.float().cpu().numpy()
    ref = OA.encode_scaled(xf, E4M3, OA.E4M3_MAX, F32(np.abs(xf).max()))
    assert np.array_equal(codes.cpu().numpy(), ref.codes)


# ----------------------------------------------------------------- the whole step
RAGGED = [3, 16, 17, 64, 1000, 16384, 16385, 40000, 70001]


def _run_and_compare(B, numels, mode, nranks, steps, lr=3e-4, dtype=torch.float32,
                     specials=None, amp=None, check_tensors=None, fused=True, delayed=False,
                     graphed=False):
    """Run the device path for `steps` steps and the oracle on the same inputs; compare
    every per-tensor output of every step.  check_tensors: oracle runs only on this
    subset (valid because nothing couples two tensors except the skip flag, and the
    inputs of a subset run are finite)."""
    import synth
    plan = B.Plan(numels, mode=mode, nranks=nranks)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        if v.numel():
            synth.fill_weights(v, t)
    dp = B.FP8DataParallel(plan, w0, lr=lr, fused=fused,
                           state_scaling="delayed" if delayed else "jit", graphed=graphed)
    gbuf = None          # graphed: the captured step reads the same gradient buffers every step
    sub = list(range(plan.T)) if check_tensors is None else list(check_tensors)
    ref_states = R.oracle_init(plan, w0, sub)
    mus = [F32(1.0)] * len(sub)
    hists = [OA.init_history(st) for st in ref_states] if delayed else None
    torch.cuda.synchronize()
    for i, t in enumerate(sub):
        R.assert_state_equal(R.state_np(B, plan, dp.state, t), ref_states[i], f"init t={t}")
    for step in range(1, steps + 1):
        grads = R.make_grads(plan, nranks, step, DEV, dtype,
                             specials=(lambda f, r: specials(f, r, step)) if specials else None, amp=amp)
        if graphed:
            if gbuf is None:
                gbuf = [g.clone() for g in grads]
            for dst, src in zip(gbuf, grads):
                dst.copy_(src)
            torch.cuda.synchronize()
            dp.step(gbuf if mode == B.MODE_SIMULATED else gbuf[0], lr=lr)
        else:
            dp.step(grads if mode == B.MODE_SIMULATED else grads[0], lr=lr)
        torch.cuda.synchronize()
        per_rank = [[R.to_np_f32(g[plan.offsets[t]: plan.offsets[t] + plan.numels[t]]) for t in sub]
                    for g in grads]
        res = OS.train_step(per_rank, mus, ref_states, OA.hyper_params(lr, step), hists=hists,
                            step=step)
        assert bool(dp.skip.item()) == res["skip"], step
        if delayed:
            wh = dp.w_hist.cpu().numpy().reshape(16, -1)
            for i, t in enumerate(sub):
                assert np.array_equal(wh[:, t], res["hists"][i]), f"step {step} tensor {t}: history"
            hists = res["hists"]
        amax = dp.amax.cpu().numpy().reshape(-1, max(plan.T, 1))
        s_g = dp.s_g.cpu().numpy()
        g8 = {t: dp.g8[plan.offsets[t]: plan.offsets[t] + plan.numels[t]].cpu().numpy() for t in sub}
        gs = dp.g_scale.cpu().numpy()
        gsi = dp.g_scale_inv.cpu().numpy()
        sat = dp.sat.cpu().numpy()
        mu = dp.mu.cpu().numpy()
        for i, t in enumerate(sub):
            p = res["per_tensor"][i]
            where = f"step {step} tensor {t} (n={plan.numels[t]})"
            for r in range(amax.shape[0]):
                a_ref = p["amax"][r]
                assert (np.isnan(amax[r, t]) and np.isnan(a_ref)) or F32(amax[r, t]) == a_ref, where
            assert F32(s_g[t]) == p["s_g"], (where, s_g[t], p["s_g"])
            got = g8[t]
            if not p["skip"]:
                bad = np.nonzero(got != p["codes"])[0]
                assert bad.size == 0, f"{where}: {bad.size} reduced codes differ"
                assert int(sat[t]) == p["sat"], (where, sat[t], p["sat"])
            assert F32(gs[t]) == p["scale"], where
            assert F32(gsi[t]) == p["scale_inv"], where
            assert F32(mu[t]) == res["mu_next"][i], (where, mu[t], res["mu_next"][i])
            R.assert_state_equal(R.state_np(B, plan, dp.state, t), res["states"][i], where)
        mus = res["mu_next"]
        ref_states = res["states"]
    return plan, dp


@pytest.mark.parametrize("fused", [True, False], ids=["dp_step", "three_calls"])
def test_local_ragged_multistep(B, fused):
    """N = 1 (LOCAL): 9 ragged tensors spanning tiles + tails, 6 steps with mu dynamics,
    through fp8lm_dp_step (quantize + Adam pass 1 fused) and through the three calls."""
    _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=6, fused=fused)


@pytest.mark.parametrize("fused", [True, False], ids=["dp_step", "three_calls"])
def test_local_bf16_gradients(B, fused):
    _run_and_compare(B, RAGGED[:6], B.MODE_LOCAL, 1, steps=2, dtype=torch.bfloat16, fused=fused)


def test_local_fused_skip_and_screen_fallback(B):
    """Fused LOCAL step: an inf gradient (skip) and a large lr (screen fallback)."""
    def specials(flat, r, step):
        if step == 2:
            flat[11] = float("inf")
    _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=3, specials=specials, lr=0.05)


@pytest.mark.parametrize("fused,delayed", [(True, False), (False, False), (True, True)],
                         ids=["dp_step", "three_calls", "delayed"])
def test_local_tiny_moments_range_certificate(B, fused, delayed):
    """Tensors whose m' / v' can leave the branch-free sqrt / division cores' range
    (|m'| < 2^-60, 0 < v' < 2^-101: gradients of 1e-20 / 1e-30 / 1e-38) next to ordinary
    ones: the per-tensor a-priori certificate (kernels.cu range_cert) fails for the tiny
    ones, whose groups take the checked body with the exact intrinsics, and holds for the
    others, which skip the per-element checks."""
    amp = [1.0, 1e-20, 1e-30, 1e-12, 1e-3, 1e-38, 1.0, 1e-15, 1e-20]
    _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=3, amp=amp, fused=fused, delayed=delayed)


@pytest.mark.parametrize("N", [2, 3, 8])
def test_simulated_ranks_multistep(B, N):
    """N simulated ranks on one device (config C1 protocol): RS+AG degenerate to a local
    rank-order sum; correlated heavy-tailed gradients overflow the sum so sat
    and the mu halving path run."""
    _run_and_compare(B, RAGGED, B.MODE_SIMULATED, N, steps=4)


def test_edge_cases_empty_zero_and_tiny(B):
    """Empty tensor, all-zero tensor (s_g -> 1), sub-min-subnormal tensor."""
    numels = [0, 100, 33, 0, 5000, 77]
    amp = [1.0, 0.0, 1e-30, 1.0, 1e-3, 1e-38]
    _run_and_compare(B, numels, B.MODE_SIMULATED, 2, steps=2, amp=amp)


def test_nonfinite_gradient_skips(B):
    """inf on one rank / NaN on another: s_g = 0 -> skip, states unchanged, mu halves (R14)."""
    def specials(flat, r, step):
        if step == 2 and r == 1:
            flat[5] = float("inf")
        if step == 3 and r == 0:
            flat[70000] = float("nan")
    _run_and_compare(B, RAGGED, B.MODE_SIMULATED, 2, steps=4, specials=specials)


def test_determinism(B):
    numels = RAGGED
    outs = []
    for _ in range(2):
        plan, dp = _run_and_compare(B, numels, B.MODE_SIMULATED, 2, steps=1)
        outs.append((dp.g8.cpu().clone(), dp.state.master.data.cpu().clone(), dp.state.w8.data.cpu().clone()))
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                           b.view(torch.uint8) if b.dtype != torch.uint8 else b)


def test_c1_full_size_two_simulated_ranks(B):
    """Config C1 at full size (BASELINE.json configs[0]): one 4096x4096 fp32 gradient,
    2 simulated ranks, one full step compared element by element."""
    _run_and_compare(B, [4096 * 4096], B.MODE_SIMULATED, 2, steps=1)


def test_c2_full_set_sampled_tensors(B):
    """Config C2 (GPT-125M set, 147 tensors, 123.7M params) in the bench's launch
    configuration; per-tensor independence lets the oracle check a subset
    of tensors exactly: the 38.6M embedding, LayerNorms, biases, a 4d x d matrix, lnf."""
    import synth
    specs = synth.gpt_gradient_set("gpt-125m")
    numels = [s.numel for s in specs]
    pick = [0, 1, 2, 3, 4, 9, 10, len(specs) - 2, len(specs) - 1]
    _run_and_compare(B, numels, B.MODE_LOCAL, 1, steps=2, check_tensors=pick)


@pytest.mark.parametrize("state_scaling", ["jit", "delayed"])
def test_c3_full_set_sampled_tensors(B, state_scaling):
    """Config C3 (GPT-7B set, 387 tensors, 6.65G params, 26.6 GB of fp32 gradient) at
    N = 1 in the bench's launch configuration: the oracle checks layer 0's LayerNorms,
    biases and attention projection (16.8M), the last layer's fc2 bias and lnf exactly."""
    import synth
    specs = synth.gpt_gradient_set("gpt-7b")
    numels = [s.numel for s in specs]
    names = [s.name for s in specs]
    pick = [i for i, nm in enumerate(names) if nm.startswith("layer0.") and
            (len(specs[i].shape) == 1 or nm == "layer0.proj.w")]
    pick += [names.index("layer31.fc2.b"), len(specs) - 2, len(specs) - 1]
    _run_and_compare(B, numels, B.MODE_LOCAL, 1, steps=2, check_tensors=pick,
                     delayed=state_scaling == "delayed")


@pytest.mark.parametrize("fused", [True, False], ids=["dp_step", "three_calls"])
def test_delayed_scaling_local(B, fused):
    """Delayed state scaling (App. B, R25-R27): one AdamW pass; 20 steps so the
    16-slot amax(w) history wraps; fused (quantize + single pass) and separate calls."""
    _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=20, fused=fused, delayed=True)


def test_delayed_scaling_simulated_skip_bf16(B):
    def specials(flat, r, step):
        if step == 3 and r == 1:
            flat[20] = float("nan")
    _run_and_compare(B, RAGGED, B.MODE_SIMULATED, 2, steps=5, dtype=torch.bfloat16,
                     specials=specials, delayed=True)


def test_amax_screen_fallback_large_lr(B):
    """lr = 0.05 moves the largest weights by far more than the 2^-6 screen margin, so
    pass 1's certified amax(w') screen fails for most tensors and k_adam_wfix
    recomputes them exactly; results must still be bit-exact."""
    _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=3, lr=0.05)


def test_amax_screen_mixed_simulated(B):
    """Moderate lr: some tensors pass the screen, some fall back."""
    _run_and_compare(B, RAGGED, B.MODE_SIMULATED, 2, steps=3, lr=2e-3)


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_simulated_fused_reduce(B, N, dtype):
    """fp8lm_dp_step with 2..4 simulated ranks (config C1's path): one kernel quantizes
    every rank's staged gradient with the shared scale, sums the decoded codes in rank
    order, requantizes and runs Adam pass 1 — vs the oracle, with a NaN skip step and an
    overflowing sum (mu halves)."""
    def specials(flat, r, step):
        if step == 2 and r == N - 1:
            flat[70000] = float("nan")
        if step == 3 and r == 0:
            flat[1003] = 3.0e5
    _run_and_compare(B, RAGGED, B.MODE_SIMULATED, N, steps=4, dtype=dtype, specials=specials)


def _device_outputs(dp):
    """The step's outputs on the host, flat (plan layout) + [T] scalars."""
    st = dp.state
    d = dict(g8=dp.g8.cpu().numpy(), s_g=dp.s_g.cpu().numpy(), scale=dp.g_scale.cpu().numpy(),
             mu=dp.mu.cpu().numpy(), sat=dp.sat.cpu().numpy())
    for k in ("m1", "v", "master", "w8"):
        s_ = getattr(st, k)
        data = s_.data.cpu()
        d[k] = data.view(torch.int16).numpy().view(np.uint16) if data.dtype == torch.float16 else data.numpy()
        d[k + "_scale"] = s_.scale.cpu().numpy()
        d[k + "_scale_inv"] = s_.scale_inv.cpu().numpy()
        d[k + "_amax"] = s_.amax.cpu().numpy()
    return d


def test_c2_full_set_every_tensor(B):
    """Config C2 (GPT-125M, 147 tensors, 123.7M params) in the bench's launch
    configuration, EVERY tensor of every step checked against the oracle (which runs on
    all host cores, whole tensors per worker: tests/_oracle_pool.py): 3 steps, the
    38.6M embedding included."""
    import synth
    from tests._oracle_pool import OraclePool
    specs = synth.gpt_gradient_set("gpt-125m")
    numels = [s.numel for s in specs]
    lr = 6e-4
    plan = B.Plan(numels, mode=B.MODE_LOCAL, nranks=1)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    dp = B.FP8DataParallel(plan, w0, lr=lr)
    pool = OraclePool(plan, w0.cpu().numpy(), lr)
    try:
        for step in range(1, 4):
            g = R.make_grads(plan, 1, step, DEV)[0]
            dp.step(g, lr=lr)
            torch.cuda.synchronize()
            bad = pool.check(step, g.cpu().numpy(), _device_outputs(dp))
            assert not bad, "\n".join(bad[:10])
    finally:
        pool.close()


def test_mu_reaches_cap_on_device(B):
    """mu's growth rule (R2/R6) up to the cap on the device: tensor 1 has an all-zero
    gradient (s_g falls back to 1, nothing saturates), so from mu = 1.996 three clean steps
    take it to exactly 2.0 (min(2, fl(mu * fl(2^(1/1000))))) and it stays there; one huge
    element at step 7 saturates its sum and halves it to 1.0.  Tensor 0 (synthetic data)
    follows the oracle's mu_update on the device's saturation counts."""
    from oracle import pipeline as OP
    import synth
    numels = [1000, 4096]
    plan = B.Plan(numels, mode=B.MODE_LOCAL)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    dp = B.FP8DataParallel(plan, w0)
    mu0 = F32(1.996)
    dp.mu.fill_(float(mu0))
    mus = [mu0, mu0]
    for step in range(1, 9):
        g = R.make_grads(plan, 1, step, DEV)[0]
        g[plan.offsets[1]: plan.offsets[1] + numels[1]] = 0.0
        if step == 7:
            g[plan.offsets[1] + 5] = 1e30
        dp.step(g)
        torch.cuda.synchronize()
        sat = dp.sat.cpu().numpy()
        assert step == 7 or int(sat[1]) == 0
        mus = [OP.mu_update(mus[t], int(sat[t]), numels[t], False) for t in range(2)]
        got = [F32(x) for x in dp.mu.cpu().numpy()]
        assert got == mus, (step, got, mus)
        if step in (3, 4, 5, 6):
            assert got[1] == F32(2.0), (step, got)
        if step == 7:
            assert got[1] == F32(1.0), got


@pytest.mark.parametrize("case", ["local", "local_delayed", "local_bf16_skip", "simulated2"])
def test_graphed_step(B, case):
    """fp8lm_dp_step_graphed: eager on the first call, captured on the second, replayed from
    the third with the step's scalars (bias correction, history slot) patched into the
    AdamW nodes — bit-exact against the oracle every step (mu dynamics, a skip step, the
    16-slot history wrapping with delayed scaling, the fused simulated reduce)."""
    if case == "local":
        _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=6, graphed=True)
    elif case == "local_delayed":
        _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=20, delayed=True, graphed=True)
    elif case == "local_bf16_skip":
        def specials(flat, r, step):
            if step == 4:
                flat[11] = float("inf")
        _run_and_compare(B, RAGGED, B.MODE_LOCAL, 1, steps=6, dtype=torch.bfloat16, specials=specials,
                         graphed=True)
    else:
        _run_and_compare(B, RAGGED, B.MODE_SIMULATED, 2, steps=5, graphed=True)
