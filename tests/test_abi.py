"""CPU tests of the C-ABI library: it loads, exports every symbol include/fp8lm.h
declares, and its host logic (hyper-parameter scalars, Alg. 1, plan layout, argument
checking) is right.  No compute calls here — those need a GPU (test_gpu_*.py)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fp8lm.h")


@pytest.fixture(scope="module")
def B():
    import paper_2310_18313_b200._binding as b
    return b


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fp8lm_[a-z0-9_]+)\s*\(", src)))


def test_header_parses_and_lists_the_four_calls():
    syms = declared_symbols()
    for name in ("fp8lm_quantize", "fp8lm_amax_scale_sync", "fp8lm_grad_allreduce", "fp8lm_adam_step"):
        assert name in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol(B):
    missing = [s for s in declared_symbols() if not hasattr(B.lib, s)]
    assert not missing, missing
    assert B.version() == 1
    assert B.has_nccl()


def test_library_is_sm100a(B):
    """The fatbin holds sm_100a SASS (cuobjdump), no generic PTX fallback needed."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", B.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_adam_hp_matches_oracle(B):
    from oracle.adam import hyper_params
    for lr, t, wd in ((3e-4, 1, 0.1), (6e-4, 7, 0.1), (1e-3, 1000, 0.0), (2.5e-5, 123457, 0.1)):
        hp = B.adam_hp(lr, t, weight_decay=wd)
        ref = hyper_params(lr, t, weight_decay=wd)
        for f in ("beta1", "beta2", "one_minus_beta1", "one_minus_beta2", "eps", "decay",
                  "step_size", "inv_bc2_sqrt"):
            assert np.float32(getattr(hp, f)) == getattr(ref, f), (f, lr, t)
    with pytest.raises(B.FP8LMError):
        B.adam_hp(1e-3, 0)


def test_zero_plan_matches_oracle(B):
    from oracle.zero import greedy_distribute
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(0, 80))
        m = int(rng.integers(1, 9))
        sizes = rng.integers(1, 50, size=n).tolist()      # many ties
        owner, load = B.zero_plan(sizes, m)
        o2, l2, _ = greedy_distribute(sizes, m)
        assert owner == o2 and load == l2
    # the GPT-13B set over 8 ranks (config C4)
    from synth import gpt_gradient_set
    sizes = [s.numel for s in gpt_gradient_set("gpt-13b")]
    owner, load = B.zero_plan(sizes, 8)
    o2, l2, _ = greedy_distribute(sizes, 8)
    assert owner == o2 and load == l2
    assert max(load) - min(load) <= max(sizes)


def _plan(B, numels, mode, nranks=1, rank=0):
    arr = (C.c_int64 * max(len(numels), 1))(*numels)
    h = C.c_void_p()
    rc = B.lib.fp8lm_plan_create(len(numels), arr, mode, nranks, rank, C.byref(h))
    return rc, h


def test_plan_layout(B):
    numels = [768, 5, 0, 50304 * 768, 17, 64]
    rc, h = _plan(B, numels, B.MODE_LOCAL)
    assert rc == 0
    offs = [B.lib.fp8lm_plan_offset(h, t) for t in range(len(numels))]
    total = B.lib.fp8lm_plan_total(h)
    assert offs[0] == 0
    for t in range(len(numels)):
        assert offs[t] % 64 == 0
        end = offs[t] + numels[t]
        nxt = offs[t + 1] if t + 1 < len(numels) else total
        assert end <= nxt and nxt - end < 64                 # tight packing, 64-aligned
    assert B.lib.fp8lm_plan_offset(h, len(numels)) == -1
    assert B.lib.fp8lm_plan_g8_bytes(h) == total
    B.lib.fp8lm_plan_destroy(h)


@pytest.mark.parametrize("N", [2, 3, 4, 8])
def test_plan_shards_partition_every_tensor(B, N):
    from synth import gpt_gradient_set
    numels = [s.numel for s in gpt_gradient_set("gpt-125m")]
    begins = []
    for r in range(N):
        rc, h = _plan(B, numels, B.MODE_NCCL, N, r)
        assert rc == 0
        S = B.lib.fp8lm_plan_shard_bytes(h)
        assert S % 64 == 0 and S * N >= B.lib.fp8lm_plan_total(h)
        assert B.lib.fp8lm_plan_g8_bytes(h) == S * N
        begins.append(B.lib.fp8lm_plan_shard_begin(h, r))
        B.lib.fp8lm_plan_destroy(h)
    assert begins == [r * S for r in range(N)]


def test_plan_argument_errors(B):
    assert _plan(B, [10], B.MODE_LOCAL, 2)[0] == B.EINVAL           # LOCAL needs nranks 1
    assert _plan(B, [10], B.MODE_NCCL, 2, 2)[0] == B.EINVAL         # rank out of range
    assert _plan(B, [10], B.MODE_SIMULATED, 17)[0] == B.EINVAL      # > 16 simulated ranks
    assert _plan(B, [-1], B.MODE_LOCAL)[0] == B.EINVAL
    assert b"numel" in B.lib.fp8lm_last_error()
    # unbound plan refuses hot-path calls before touching the GPU
    rc, h = _plan(B, [10], B.MODE_LOCAL)
    assert rc == 0
    rc = B.lib.fp8lm_amax_scale_sync(h, None, C.c_void_p(256), B.F32, C.c_void_p(256),
                                     C.c_void_p(256), C.c_void_p(256), C.c_void_p(256), None)
    assert rc == B.EWORKSPACE
    B.lib.fp8lm_plan_destroy(h)
    assert B.lib.fp8lm_quantize(None, B.F32, -1, B.E4M3, None, None, None, None, 1, None, None) == B.EINVAL
    # small-message thresholds: host setters, no GPU
    rc, h = _plan(B, [1000, 24], B.MODE_P2P, 2, 0)
    assert rc == 0
    assert B.lib.fp8lm_plan_set_oneshot(h, 1 << 20) == 0
    assert B.lib.fp8lm_plan_set_oneshot_raw(h, 0) == 0
    assert B.lib.fp8lm_plan_set_oneshot_raw(h, -1) == B.EINVAL
    assert B.lib.fp8lm_plan_set_oneshot(h, -1) == B.EINVAL
    B.lib.fp8lm_plan_destroy(h)
    assert B.lib.fp8lm_plan_set_oneshot_raw(None, 1) == B.EINVAL
    # ZeRO: every rank's owned layout is the Alg. 1 packing of its tensors
    numels = [5000, 70001, 3, 16384, 999, 64]
    owners = []
    for r in range(3):
        rc, h = _plan(B, numels, B.MODE_ZERO, 3, r)
        assert rc == 0
        owned = [t for t in range(len(numels)) if B.lib.fp8lm_plan_owned_offset(h, t) >= 0]
        assert B.lib.fp8lm_plan_owned_count(h) == len(owned)
        assert B.lib.fp8lm_plan_owned_total(h) == sum((numels[t] + 63) // 64 * 64 for t in owned)
        owners += owned
        B.lib.fp8lm_plan_destroy(h)
    assert sorted(owners) == list(range(len(numels)))      # every tensor has exactly one owner


def test_workspace_sizes(B):
    numels = [4096 * 4096]
    rc, h = _plan(B, numels, B.MODE_SIMULATED, 2)
    ws = B.lib.fp8lm_plan_workspace_bytes(h)
    assert ws >= 2 * 4096 * 4096            # the simulated ranks' code buffers
    B.lib.fp8lm_plan_destroy(h)
    rc, h = _plan(B, numels, B.MODE_NCCL, 4, 1)
    assert B.lib.fp8lm_plan_workspace_bytes(h) >= 2 * B.lib.fp8lm_plan_g8_bytes(h)   # send + recv
    B.lib.fp8lm_plan_destroy(h)


def test_sass_paired_fp32_has_no_contracted_products(B):
    """R16 needs every product of the AdamW sequence rounded on its own.  The paired
    FP32 bodies (device.cuh P2: FMUL2 / FFMA2) keep additions scalar because ptxas
    contracts a mul.rn.f32x2 feeding an add.rn.f32x2 into an FFMA2 even under
    --fmad=false; the only FFMA2 allowed are the 6 per lane pair inside the paired
    sqrt / division cores (2 + 4), i.e. 48 per 16-element group body: pass 2's body
    (k_adam<2, .>) and pass 1's certified exact screen (screen_exact_p2, in every kernel
    that runs pass 1: k_adam<1>, k_adam<3, ., ., NS>, the exchange kernels), one body per
    kernel.  A contracted product would show up as extra FFMA2 here (and as a parity
    failure on the GPU)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", B.LIB_PATH], capture_output=True, text=True).stdout
    counts, fn = {}, None
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
        elif "FFMA2" in line and fn:
            counts[fn] = counts.get(fn, 0) + 1
    assert counts, "no FFMA2 at all: the paired pass-2 body is missing"
    allowed = ("_ZN5fp8lm6k_adamILi1E", "_ZN5fp8lm6k_adamILi2E", "_ZN5fp8lm6k_adamILi3E",
               "_ZN5fp8lm15k_reduce_p2p_a1", "_ZN5fp8lm17k_reduce_owner_a1")
    for fn, c in counts.items():
        assert fn.startswith(allowed), (fn, c)
        assert c == 48, (fn, c)
    assert any(fn.startswith("_ZN5fp8lm6k_adamILi2E") for fn in counts)


def test_commstats_metrics_host(B):
    """fp8lm_commstats_metrics (R29-R30): SNR = 10 log10(sig2 / err2) and the event rates."""
    import struct
    import ctypes as C
    import math
    def metrics(sig2, err2, under, over, events):
        raw = struct.pack("<ddQQQIIffffff4I", sig2, err2, under, over, events, 0, 0, *([0.0] * 6), 0, 0, 0, 0)
        buf = (C.c_uint8 * len(raw)).from_buffer_copy(raw)
        out = (C.c_double * 3)()
        assert B.lib.fp8lm_commstats_metrics(C.cast(buf, C.c_void_p), out) == 0
        return list(out)
    snr, u, o = metrics(100.0, 1.0, 3, 1, 1000)
    assert snr == 20.0 and u == 0.003 and o == 0.001
    assert metrics(1.0, 0.0, 0, 0, 0)[0] == math.inf and metrics(1.0, 0.0, 0, 0, 0)[1:] == [0.0, 0.0]
    assert math.isnan(metrics(0.0, 0.0, 0, 0, 10)[0])
    assert metrics(0.0, 2.0, 0, 0, 10)[0] == -math.inf


def test_bucket_split_contiguous_balanced(B):
    """The split step's buckets (BucketedDP): contiguous groups covering every tensor once,
    in order, with about equal parameter counts (GPT-7B set into 6 buckets)."""
    import synth
    numels = [s.numel for s in synth.gpt_gradient_set("gpt-7b")]
    for nb in (1, 2, 3, 6, 8):
        groups = B.bucket_split(numels, nb)
        assert len(groups) == nb
        flat = [t for g in groups for t in g]
        assert flat == list(range(len(numels)))
        loads = [sum(numels[t] for t in g) for g in groups]
        # the largest tensor (the embedding, 3 % of the set) bounds the imbalance
        assert max(loads) <= sum(numels) / nb + max(numels)
    assert B.bucket_split([5, 1], 4) == [[0], [1]]
