"""Modes P2P and ZERO on ONE GPU: N logical ranks in one process, each a plan of its own
whose peer table points at the other plans' local windows (fp8lm_peer_setup_loopback),
each rank's calls on its own stream.  The kernels are the multi-GPU ones — the fused
exchange + Adam pass 1 (k_reduce_p2p_a1), the pass-2 all-gather pull from the owners'
windows (k_adam<2, ., true>), the ZeRO owner reduce (k_reduce_owner_a1), the w8
broadcast inside pass 2 and k_w8_bcast, the scale MIN and the flag protocol through the
pads — so a single-GPU box runs the A5 all-gather and the A8 whole-tensor
ZeRO bit-exact against the N-rank oracle.  Grids are capped at #SMs / N
CTAs so the N ranks' kernels are resident together (their spin-waits need it)."""
import numpy as np
import pytest
import torch

from tests.conftest import gpu_available
from tests import _gpu_ref as R

from oracle import adam as OA
from oracle import step as OS

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

F32 = np.float32
RAGGED = [3, 16, 17, 64, 1000, 16384, 16385, 40000, 70001, 5]


@pytest.fixture(scope="module")
def B():
    import paper_2310_18313_b200 as b
    b.set_peer_timeout(120.0)          # a protocol bug traps instead of hanging the box
    # CUDA lazy loading: a kernel's first launch may wait for the device to go idle, which
    # never happens while another rank's kernel spins on a flag.  The library preloads its
    # own kernels in fp8lm_peer_setup_loopback; load torch's (fill, copy, the synthetic
    # generator) here by running the same host code once on a LOCAL plan.
    import synth
    plan = b.Plan(RAGGED, mode=b.MODE_LOCAL)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    for delayed in (False, True):
        dp = b.FP8DataParallel(plan, w0, state_scaling="delayed" if delayed else "jit")
        dp.step(R.make_grads(plan, 1, 1, "cuda")[0])
    b.CompactLayout.__new__(b.CompactLayout)
    x = plan.flat(torch.float32)
    x[3:1000].copy_(w0[64:1061])
    torch.cuda.synchronize()
    return b


def run_loopback(B, numels, mode, N, steps, fused=True, delayed=False, lr=3e-4, sub=None,
                 specials=None, oneshot=False, graphed=False, dtype=torch.float32):
    """oneshot: mode P2P's small-message exchange (fp8lm_plan_set_oneshot); off by
    default so that these small sets take the reduce-scatter / all-gather kernels.
    True: the two-handshake one-shot (raw variant off); "raw": the one-handshake raw
    one-shot (fp8lm_plan_set_oneshot_raw) where the call is fp8lm_allreduce_jit / dp_step."""
    import synth
    bmode = {"p2p": B.MODE_P2P, "zero": B.MODE_ZERO}[mode]
    plans = [B.Plan(numels, mode=bmode, nranks=N, rank=r) for r in range(N)]
    for p_ in plans:
        p_.set_oneshot(1 << 40 if oneshot else 0)
        p_.set_oneshot_raw(1 << 40 if oneshot == "raw" else 0)
    B.peer_setup_loopback(plans)
    streams = [torch.cuda.Stream() for _ in range(N)]
    w0 = plans[0].flat(torch.float32)
    for t, v in enumerate(plans[0].views(w0)):
        if v.numel():
            synth.fill_weights(v, t)
    torch.cuda.synchronize()
    dps = []
    for r in range(N):
        with torch.cuda.stream(streams[r]):
            dps.append(B.FP8DataParallel(plans[r], w0, lr=lr, fused=fused,
                                         state_scaling="delayed" if delayed else "jit", graphed=graphed))
    gbufs = None
    torch.cuda.synchronize()
    plan = plans[0]
    sub = list(range(plan.T)) if sub is None else list(sub)
    ref_states = R.oracle_init(plan, w0, sub)
    mus = [F32(1.0)] * len(sub)
    hists = [OA.init_history(st) for st in ref_states] if delayed else None
    msgs = []
    for step in range(1, steps + 1):
        grads = R.make_grads(plan, N, step, "cuda", dtype,
                             specials=(lambda f, r: specials(f, r, step)) if specials else None)
        torch.cuda.synchronize()
        if graphed:      # the captured steps read the same buffers every step
            if gbufs is None:
                gbufs = [g.clone() for g in grads]
            for dst, src in zip(gbufs, grads):
                dst.copy_(src)
            torch.cuda.synchronize()
        try:
            for r in range(N):
                with torch.cuda.stream(streams[r]):
                    dps[r].step(gbufs[r] if graphed else grads[r], lr=lr)
            torch.cuda.synchronize()
        except Exception as e:
            raise AssertionError(f"step {step}: {e}; watchdog report {B.peer_timeout_report()}") from e
        per_rank = [[R.to_np_f32(g[plan.offsets[t]: plan.offsets[t] + plan.numels[t]]) for t in sub]
                    for g in grads]
        res = OS.train_step(per_rank, mus, ref_states, OA.hyper_params(lr, step), hists=hists, step=step)
        for r in range(N):
            msgs += [f"step {step}: {m}" for m in
                     R.compare_rank(B, plans[r], dps[r], res, r, mode, fused and not oneshot, sub)]
        assert not msgs, "\n".join(msgs[:10])
        mus = res["mu_next"]
        ref_states = res["states"]
        if delayed:
            hists = res["hists"]
    assert B.peer_timeout_report()[0] == 0
    return plans, dps


def _huge(flat, r, step):
    # one huge value on the last rank at step 2: the sum saturates, mu halves
    if step == 2 and r == 1:
        flat[1000 + 7] = 3.0e5


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("variant", ["p2p", "p2p_unfused", "p2p_delayed", "zero", "zero_unfused",
                                     "zero_delayed"])
def test_loopback_bit_exact(B, N, variant):
    mode = variant.split("_")[0]
    run_loopback(B, RAGGED, mode, N, steps=3, fused="unfused" not in variant,
                 delayed="delayed" in variant, specials=_huge)


@pytest.mark.parametrize("variant", ["p2p", "p2p_unfused", "p2p_delayed", "zero", "zero_unfused",
                                     "p2p_oneshot", "p2p_oneshotraw"])
def test_loopback_eight_ranks(B, variant):
    """N = 8 (the largest group the kernels are instantiated for; gpurun offers at most 4
    GPUs): the NR = 8 exchange, one-shot and owner kernels, bit-exact on every rank."""
    mode = variant.split("_")[0]
    run_loopback(B, RAGGED, mode, 8, steps=3, fused="unfused" not in variant, delayed="delayed" in variant,
                 specials=_huge, oneshot=_oneshot_arg(variant))


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("numels", [[1500], [4096], [3, 64]], ids=["1500", "4096", "3+64"])
@pytest.mark.parametrize("variant", ["fused", "unfused", "raw"])
def test_loopback_oneshot_single_unit(B, N, numels, variant):
    """Plans of one 4096-element unit launch the one-shot kernels as ONE CTA, which skips
    the tickets and the phase word (k_oneshot, k_oneshot_full, k_oneshot_raw)."""
    def spec(flat, r, step):                  # one saturating sum at step 2
        if step == 2 and r == 1:
            flat[1] = 3.0e5
    run_loopback(B, numels, "p2p", N, steps=4, fused=variant != "unfused", specials=spec,
                 oneshot="raw" if variant == "raw" else True)


@pytest.mark.parametrize("N", [3, 4])
@pytest.mark.parametrize("variant", ["p2p", "p2p_unfused", "p2p_delayed", "zero", "zero_unfused"])
def test_loopback_tiny_shards(B, N, variant):
    """Shards smaller than a 16K-element work item: one item of the first tensor spans
    several shards, so the pushing quantize (P2P whole step / three calls) sends its
    16-code groups to several shard owners, and ZeRO owners get uneven loads."""
    mode = variant.split("_")[0]
    run_loopback(B, [20000, 5, 3000, 17, 64], mode, N, steps=3, fused="unfused" not in variant,
                 delayed="delayed" in variant, specials=_huge)


@pytest.mark.parametrize("N", [2, 3, 4])
@pytest.mark.parametrize("variant", ["fused", "unfused", "delayed", "raw", "raw_delayed"])
def test_loopback_oneshot(B, N, variant):
    """Mode P2P's one-shot small-message exchange (k_oneshot: quantize, one handshake,
    every rank pulls and reduces the whole set): bit-exact through fp8lm_dp_step (then
    both AdamW passes locally), the three calls and delayed scaling.  raw: the
    one-handshake kernel k_oneshot_raw (every rank pulls the gradients and encodes them
    itself; the window copy alternates halves step by step, so 4 steps wrap it twice)."""
    raw = variant.startswith("raw")
    run_loopback(B, RAGGED, "p2p", N, steps=4 if raw else 3, fused=variant != "unfused",
                 delayed=variant.endswith("delayed"), specials=_huge, oneshot="raw" if raw else True)


@pytest.mark.parametrize("mode", ["p2p", "zero"])
def test_loopback_skip_and_screen_fallback(B, mode):
    """A NaN on one rank (s_r = 0 -> every rank skips, mu halves) and lr = 0.05 (the
    amax(w') screen fails: adam_wfix's grid barrier inside the multi-GPU pass 2)."""
    def specials(flat, r, step):
        if step == 2 and r == 0:
            flat[17] = float("nan")
    run_loopback(B, RAGGED, mode, 2, steps=4, lr=0.05, specials=specials)


@pytest.mark.parametrize("mode,N", [("p2p", 2), ("p2p", 4), ("zero", 4)])
def test_loopback_gpt125m_sampled(B, mode, N):
    """The full-size paths (BASELINE configs[1] set at N ranks): work-order rotation wrap,
    pulls that straddle shard bounds, many items per CTA.  The oracle checks every tensor
    that straddles a shard bound plus small tensors from the first and last layers."""
    import synth
    specs = synth.gpt_gradient_set("gpt-125m")
    numels = [s.numel for s in specs]
    import paper_2310_18313_b200 as b
    probe = b.Plan(numels, mode=b.MODE_P2P, nranks=N, rank=0)
    bounds = [probe.shard_begin(r) for r in range(1, N)]
    straddle = [t for t in range(len(numels))
                if any(probe.offsets[t] < x < probe.offsets[t] + numels[t] for x in bounds)]
    del probe
    big = [t for t in straddle if numels[t] > 8_000_000]
    sub = sorted(set([t for t in straddle if t not in big][:3] + [1, 2, 3, 9, len(specs) - 2, len(specs) - 1]))
    run_loopback(B, numels, mode, N, steps=2, sub=sub)


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("variant", ["p2p", "p2p_delayed", "zero"])
def test_loopback_split_buckets(B, N, variant):
    """fp8lm_dp_step_split over 3 buckets (one plan each): phase 1 of every bucket (amax,
    MIN, quantize; the exchange on the plan's exchange stream), then phase 2 of every
    bucket (the AdamW pass with the pulled all-gather / the w8 broadcast).  Each bucket
    is an independent scaling group (R33), checked against the oracle on its tensors."""
    import synth
    mode = variant.split("_")[0]
    delayed = "delayed" in variant
    bmode = {"p2p": B.MODE_P2P, "zero": B.MODE_ZERO}[mode]
    groups = B.bucket_split(RAGGED, 3)
    assert len(groups) == 3
    plans = [[B.Plan([RAGGED[t] for t in grp], mode=bmode, nranks=N, rank=r) for grp in groups]
             for r in range(N)]
    for b in range(len(groups)):
        B.peer_setup_loopback([plans[r][b] for r in range(N)])
    streams = [torch.cuda.Stream() for _ in range(N)]
    w0s = []
    for b, grp in enumerate(groups):
        w = plans[0][b].flat(torch.float32)
        for j, v in enumerate(plans[0][b].views(w)):
            synth.fill_weights(v, grp[j])
        w0s.append(w)
    torch.cuda.synchronize()
    dps = []
    for r in range(N):
        with torch.cuda.stream(streams[r]):
            dps.append(B.BucketedDP(plans[r], w0s, state_scaling="delayed" if delayed else "jit"))
    torch.cuda.synchronize()
    refs = [R.oracle_init(plans[0][b], w0s[b]) for b in range(len(groups))]
    mus = [[F32(1.0)] * len(g) for g in groups]
    hists = [[OA.init_history(st) for st in rs] for rs in refs] if delayed else None
    for step in range(1, 4):
        grads = []
        for r in range(N):
            row = []
            for b, grp in enumerate(groups):
                flat = plans[0][b].flat(torch.float32)
                for j, v in enumerate(plans[0][b].views(flat)):
                    synth.fill_gradient(v, step, grp[j], r)
                if step == 2 and r == N - 1 and b == 1:
                    flat[plans[0][b].offsets[0] + 3] = 3.0e5      # bucket 1's sum saturates
                row.append(flat)
            grads.append(row)
        torch.cuda.synchronize()
        try:
            for r in range(N):
                with torch.cuda.stream(streams[r]):
                    dps[r].step(grads[r])
            torch.cuda.synchronize()
        except Exception as e:
            raise AssertionError(f"step {step}: {e}; watchdog report {B.peer_timeout_report()}") from e
        msgs = []
        for b, grp in enumerate(groups):
            plan = plans[0][b]
            per_rank = [[R.to_np_f32(grads[r][b][plan.offsets[j]: plan.offsets[j] + plan.numels[j]])
                         for j in range(plan.T)] for r in range(N)]
            res = OS.train_step(per_rank, mus[b], refs[b], OA.hyper_params(3e-4, step),
                                hists=hists[b] if delayed else None, step=step)
            for r in range(N):
                msgs += [f"step {step} bucket {b}: {m}" for m in
                         R.compare_rank(B, plans[r][b], dps[r].dps[b], res, r, mode, True)]
            mus[b], refs[b] = res["mu_next"], res["states"]
            if delayed:
                hists[b] = res["hists"]
        assert not msgs, "\n".join(msgs[:10])


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("oneshot,jit", [(True, False), (False, False), (True, True), (False, True), ("raw", True)],
                         ids=["oneshot", "rsag", "oneshot_jit", "rsag_jit", "oneshot_raw_jit"])
def test_loopback_graph_replay_allreduce(B, N, oneshot, jit):
    """The P2P exchange captured in a CUDA graph (one per rank, on its stream) and
    replayed: fp8lm_amax_scale_sync + fp8lm_grad_allreduce read their flag epochs from the
    pads' device counters (kPadCtl), so every replay is a new step.  Each replay's inputs
    are copied into the captured gradient buffer; results vs the N-rank oracle every step."""
    import synth
    from oracle import pipeline as OP
    plans = [B.Plan(RAGGED, mode=B.MODE_P2P, nranks=N, rank=r) for r in range(N)]
    for p_ in plans:
        p_.set_oneshot(1 << 40 if oneshot else 0)
        p_.set_oneshot_raw(1 << 40 if oneshot == "raw" else 0)
    B.peer_setup_loopback(plans)
    plan = plans[0]
    T = plan.T
    bufs = []
    for r in range(N):
        bufs.append(dict(g=plan.flat(torch.float32), g8=plans[r].peer_g8(),
                         mu=torch.ones(T, device="cuda"), amax=torch.zeros(T, device="cuda"),
                         s_g=torch.zeros(T, device="cuda"), skip=torch.zeros(1, dtype=torch.int32, device="cuda"),
                         gs=torch.zeros(T, device="cuda"), gsi=torch.zeros(T, device="cuda"),
                         sat=torch.zeros(T, dtype=torch.int32, device="cuda")))
    streams = [torch.cuda.Stream() for _ in range(N)]
    torch.cuda.synchronize()

    def call(r):
        b = bufs[r]
        if jit:      # fp8lm_allreduce_jit: one kernel for a small plan (k_oneshot_full)
            B.allreduce_jit(plans[r], b["g"], b["mu"], b["amax"], b["s_g"], b["skip"], b["g8"], b["gs"], b["gsi"],
                            b["sat"])
            return
        B.amax_scale_sync(plans[r], b["g"], b["mu"], b["amax"], b["s_g"], b["skip"])
        B.fp8_grad_allreduce(plans[r], b["g"], b["s_g"], b["skip"], b["g8"], b["gs"], b["gsi"], b["sat"], b["mu"])

    graphs = [torch.cuda.CUDAGraph() for _ in range(N)]
    # capture: the captured launches do not run; the device counters advance only on replay
    for r in range(N):
        with torch.cuda.graph(graphs[r], stream=streams[r]):
            call(r)
    torch.cuda.synchronize()
    mus = [F32(1.0)] * T
    for step in range(1, 5):
        grads = R.make_grads(plan, N, step, "cuda", specials=lambda f, r: _huge(f, r, step))
        for r in range(N):
            bufs[r]["g"].copy_(grads[r])
        torch.cuda.synchronize()
        for r in range(N):
            with torch.cuda.stream(streams[r]):
                graphs[r].replay()
        torch.cuda.synchronize()
        per_rank = [[R.to_np_f32(g[plan.offsets[t]: plan.offsets[t] + plan.numels[t]]) for t in range(T)]
                    for g in grads]
        for t in range(T):
            ref = OP.allreduce_tensor([per_rank[r][t] for r in range(N)], mus[t])
            for r in range(N):
                b = bufs[r]
                sl = slice(plan.offsets[t], plan.offsets[t] + plan.numels[t])
                # fp8lm_grad_allreduce leaves the whole reduced set in every rank's g8
                assert np.array_equal(b["g8"].cpu().numpy()[sl], ref["codes"]), (step, t, r)
                assert F32(b["s_g"][t].item()) == ref["s_g"] and int(b["sat"][t].item()) == ref["sat"], (step, t, r)
            mus[t] = OP.mu_update(mus[t], ref["sat"], ref["n"], False)
            assert F32(bufs[0]["mu"][t].item()) == mus[t], (step, t)
    assert B.peer_timeout_report()[0] == 0


@pytest.mark.parametrize("variant", ["p2p", "p2p_oneshot", "p2p_oneshotraw", "zero"])
def test_loopback_graphed_step(B, variant):
    """fp8lm_dp_step_graphed across N = 2 ranks on one GPU: each rank's step captured on
    its own stream (flag epochs from the pads' device counters, AdamW scalars patched per
    replay), bit-exact against the oracle over 5 steps."""
    mode = variant.split("_")[0]
    run_loopback(B, RAGGED, mode, 2, steps=5, specials=_huge, oneshot=_oneshot_arg(variant), graphed=True)


def _oneshot_arg(variant):
    return "raw" if "oneshotraw" in variant else "oneshot" in variant


@pytest.mark.parametrize("variant", ["p2p", "p2p_oneshot", "p2p_oneshotraw", "zero"])
def test_loopback_bf16_gradients(B, variant):
    """bf16 gradients (exact widening) through the multi-GPU kernels: the exchange's
    quantize, the one-kernel small-message path (k_oneshot_full), ZeRO's owner reduce."""
    run_loopback(B, RAGGED, variant.split("_")[0], 2, steps=3, specials=_huge, oneshot=_oneshot_arg(variant),
                 dtype=torch.bfloat16)
