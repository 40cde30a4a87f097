"""Thin ctypes binding over libfp8lm.so (include/fp8lm.h).

Argument marshalling only: PyTorch allocates device memory and supplies the stream
(and torch.distributed bootstraps the NCCL unique id); every step of the hot path
runs in the library's sm_100a kernels or in NCCL.  There is NO CPU fallback: if the
shared library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import math
import struct
import os
from typing import List, Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FP8LM_LIB: an experiment build of the same library (A/B timing runs, build.py --out)
LIB_PATH = os.environ.get("FP8LM_LIB") or os.path.join(_HERE, "libfp8lm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2310_18313_b200/build.py` "
        "(or __graft_entry__.build()); there is no fallback path")

lib = C.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants (fp8lm.h)
OK, EINVAL, ECUDA, ENCCL, EWORKSPACE, EUNSUPPORTED = 0, -1, -2, -3, -4, -5
E4M3, E5M2, F16, BF16, F32 = 0, 1, 2, 3, 4
MODE_LOCAL, MODE_SIMULATED, MODE_NCCL, MODE_P2P, MODE_ZERO = 0, 1, 2, 3, 4
ALIGN_ELEMS = 64
MAX_SIM_RANKS = 16

_p = C.c_void_p
_i32, _i64, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class AdamHP(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("beta1", "beta2", "one_minus_beta1", "one_minus_beta2",
                                          "eps", "decay", "step_size", "inv_bc2_sqrt")]


class STensors(C.Structure):
    _fields_ = [("data", _p), ("scale", _p), ("scale_inv", _p), ("amax", _p)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("fp8lm_version", C.c_int)
_sig("fp8lm_last_error", C.c_char_p)
_sig("fp8lm_has_nccl", C.c_int)
_sig("fp8lm_adam_hp_make", C.c_int, _f64, _f64, _f64, _f64, _f64, _i64, C.POINTER(AdamHP))
_sig("fp8lm_zero_plan", C.c_int, _i32, C.POINTER(_i64), _i32, C.POINTER(_i32), C.POINTER(_i64))
_sig("fp8lm_comm_unique_id", C.c_int, C.POINTER(C.c_uint8))
_sig("fp8lm_comm_init", C.c_int, _i32, _i32, C.POINTER(C.c_uint8), C.POINTER(_p))
_sig("fp8lm_comm_destroy", C.c_int, _p)
_sig("fp8lm_comm_attach", C.c_int, _p, _i32, _i32, C.POINTER(_p))
_sig("fp8lm_commstats_metrics", C.c_int, _p, C.POINTER(C.c_double))
_sig("fp8lm_plan_create", C.c_int, _i32, C.POINTER(_i64), _i32, _i32, _i32, C.POINTER(_p))
_sig("fp8lm_plan_destroy", C.c_int, _p)
_sig("fp8lm_plan_offset", _i64, _p, _i32)
_sig("fp8lm_plan_total", _i64, _p)
_sig("fp8lm_plan_g8_bytes", _i64, _p)
_sig("fp8lm_plan_shard_bytes", _i64, _p)
_sig("fp8lm_plan_shard_begin", _i64, _p, _i32)
_sig("fp8lm_plan_workspace_bytes", C.c_size_t, _p)
_sig("fp8lm_plan_bind", C.c_int, _p, _p, C.c_size_t, _p)
_sig("fp8lm_peer_setup", C.c_int, _p, _p, _p)
_sig("fp8lm_peer_setup_loopback", C.c_int, C.POINTER(_p), _i32, _p)
_sig("fp8lm_set_peer_timeout", C.c_int, _f64)
_sig("fp8lm_peer_timeout_report", C.c_int, C.POINTER(C.c_uint32))
_sig("fp8lm_plan_set_oneshot", C.c_int, _p, _i64)
_sig("fp8lm_plan_set_oneshot_raw", C.c_int, _p, _i64)
_sig("fp8lm_peer_g8", _p, _p)
_sig("fp8lm_peer_w8", _p, _p)
_sig("fp8lm_peer_w8_scalars", _p, _p)
_sig("fp8lm_plan_owner", _i32, _p, _i32)
_sig("fp8lm_plan_owned_offset", _i64, _p, _i32)
_sig("fp8lm_plan_owned_total", _i64, _p)
_sig("fp8lm_plan_owned_count", _i32, _p)
_sig("fp8lm_quantize", C.c_int, _p, _i32, _i64, _i32, _p, _p, _p, _p, _i32, _p, _p)
_sig("fp8lm_dequantize", C.c_int, _p, _i32, _i64, _p, _p, _p)
_sig("fp8lm_amax_scale_sync", C.c_int, _p, _p, _p, _i32, _p, _p, _p, _p, _p)
_sig("fp8lm_grad_allreduce", C.c_int, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p)
_sig("fp8lm_allreduce_jit", C.c_int, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p)
_sig("fp8lm_adam_step", C.c_int, _p, _p, _p, C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(STensors), C.POINTER(STensors), C.POINTER(AdamHP), _p, _p)
_sig("fp8lm_prof_enable", C.c_int, C.c_int)
_sig("fp8lm_prof_ids", C.c_int)
_sig("fp8lm_prof_read", C.c_int, _i32, C.POINTER(C.c_char_p), C.POINTER(_i64), C.POINTER(C.c_double),
     C.POINTER(_i32))
_sig("fp8lm_selftest_fastmath", C.c_int, _u64, _u64, C.POINTER(_u64))
_sig("fp8lm_dp_step", C.c_int, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
     C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(AdamHP), _p, _i32, _p)
_sig("fp8lm_dp_step_graphed", C.c_int, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
     C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(AdamHP), _p, _i32, _p)
_sig("fp8lm_dp_step_split", C.c_int, _p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
     C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(AdamHP), _p, _i32, _p)
_sig("fp8lm_adam_step_delayed", C.c_int, _p, _p, _p, C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(STensors), C.POINTER(STensors), C.POINTER(AdamHP), _p, _p, _i32, _p)
_sig("fp8lm_sp_create", C.c_int, _p, _i64, _p, C.POINTER(_p))
_sig("fp8lm_sp_destroy", C.c_int, _p)
_sig("fp8lm_sp_allgather", C.c_int, _p, _p, _i32, _i64, _p, _p, _i32, _p, _p)
_sig("fp8lm_sp_reduce_scatter", C.c_int, _p, _p, _i32, _i64, _p, _i32, _p, _p)
_sig("fp8lm_allreduce_strategy", C.c_int, _i32, _p, _i32, _i64, _p, _p, _p, _p)
_sig("fp8lm_state_init", C.c_int, _p, _p, C.POINTER(STensors), C.POINTER(STensors),
     C.POINTER(STensors), C.POINTER(STensors), _p)


class FP8LMError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != OK:
        msg = lib.fp8lm_last_error().decode(errors="replace")
        raise FP8LMError(f"{what} failed ({rc}): {msg}")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"gradients must be float32 or bfloat16, got {t.dtype}")


# ------------------------------------------------------------------ host helpers
def version() -> int:
    return lib.fp8lm_version()


def has_nccl() -> bool:
    return bool(lib.fp8lm_has_nccl())


def adam_hp(lr: float, step: int, beta1: float = 0.9, beta2: float = 0.95, eps: float = 1e-8,
            weight_decay: float = 0.1) -> AdamHP:
    """fp8lm_adam_hp_make (R24): scalars in double, rounded once to float."""
    hp = AdamHP()
    _check(lib.fp8lm_adam_hp_make(lr, beta1, beta2, eps, weight_decay, step, C.byref(hp)),
           "fp8lm_adam_hp_make")
    return hp


def zero_plan(numels: Sequence[int], nranks: int):
    """Alg. 1 -> (owner[T], load[nranks])."""
    T = len(numels)
    arr = (_i64 * max(T, 1))(*numels)
    owner = (_i32 * max(T, 1))()
    load = (_i64 * nranks)()
    _check(lib.fp8lm_zero_plan(T, arr, nranks, owner, load), "fp8lm_zero_plan")
    return list(owner)[:T], list(load)


def selftest_fastmath(div_pairs: int = 1 << 36, seed: int = 12345):
    """-> dict(sqrt_bad, sqrt_accepted, div_bad, div_accepted) (see fp8lm.h)."""
    out = (_u64 * 4)()
    _check(lib.fp8lm_selftest_fastmath(div_pairs, seed, out), "fp8lm_selftest_fastmath")
    return dict(sqrt_bad=out[0], sqrt_accepted=out[1], div_bad=out[2], div_accepted=out[3])


def prof_enable(on: bool = True):
    """Start (True) / stop (False) the library's per-launch CUDA-event tracing."""
    lib.fp8lm_prof_enable(1 if on else 0)


def prof_read():
    """-> {name: dict(launches, ms, ours)} for every id with at least one launch."""
    out = {}
    for i in range(lib.fp8lm_prof_ids()):
        name, n, ms, ours = C.c_char_p(), _i64(), C.c_double(), _i32()
        _check(lib.fp8lm_prof_read(i, C.byref(name), C.byref(n), C.byref(ms), C.byref(ours)),
               "fp8lm_prof_read")
        if n.value:
            out[name.value.decode()] = dict(launches=n.value, ms=ms.value, ours=bool(ours.value))
    return out


# ------------------------------------------------------------------ communicator
class Comm:
    """An NCCL communicator owned by the library, bootstrapped over torch.distributed."""

    def __init__(self, nranks: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = _p()
        _check(lib.fp8lm_comm_init(nranks, rank, buf, C.byref(h)), "fp8lm_comm_init")
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib.fp8lm_comm_unique_id(buf), "fp8lm_comm_unique_id")
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, group=None, attach: bool = True) -> "Comm":
        """attach=True: wrap torch.distributed's own NCCL communicator of `group`
        (ProcessGroupNCCL._comm_ptr(), fp8lm_comm_attach: one communicator per process);
        False, or when torch's communicator is not available: a new one of the library's
        own, bootstrapped over torch.distributed."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if attach:
            try:
                pg = group if group is not None else dist.distributed_c10d._get_default_group()
                backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
                ptr = backend._comm_ptr()
            except Exception:
                ptr = 0
            if ptr:
                obj = cls.__new__(cls)
                h = _p()
                _check(lib.fp8lm_comm_attach(C.c_void_p(ptr), world, rank, C.byref(h)), "fp8lm_comm_attach")
                obj.handle, obj.nranks, obj.rank, obj.attached = h, world, rank, True
                return obj
        obj: List[Optional[bytes]] = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(world, rank, obj[0])

    def close(self):
        if self.handle:
            lib.fp8lm_comm_destroy(self.handle)
            self.handle = None


# ------------------------------------------------------------------ plan
class Plan:
    """Flat layout of T tensors + bound device workspace (fp8lm_plan_*)."""

    def __init__(self, numels: Sequence[int], mode: int = MODE_LOCAL, nranks: int = 1, rank: int = 0,
                 device="cuda", stream=None):
        self.numels = [int(n) for n in numels]
        self.T = len(self.numels)
        self.mode, self.nranks, self.rank = mode, nranks, rank
        arr = (_i64 * max(self.T, 1))(*self.numels)
        h = _p()
        _check(lib.fp8lm_plan_create(self.T, arr, mode, nranks, rank, C.byref(h)), "fp8lm_plan_create")
        self.handle = h
        self.offsets = [lib.fp8lm_plan_offset(h, t) for t in range(self.T)]
        self.total = lib.fp8lm_plan_total(h)
        self.g8_bytes = lib.fp8lm_plan_g8_bytes(h)
        self.shard_bytes = lib.fp8lm_plan_shard_bytes(h)
        self.ws_bytes = lib.fp8lm_plan_workspace_bytes(h)
        self.device = torch.device(device)
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=self.device)
        _check(lib.fp8lm_plan_bind(h, _ptr(self.ws), self.ws.numel(), _stream(stream)), "fp8lm_plan_bind")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            lib.fp8lm_plan_destroy(h)
            self.handle = None

    peer_ready = False

    def peer_setup(self, comm: "Comm", stream=None):
        """Mode P2P: map every rank's windows (collective; see fp8lm_peer_setup)."""
        if self.peer_ready:
            return
        _check(lib.fp8lm_peer_setup(self.handle, comm.handle, _stream(stream)), "fp8lm_peer_setup")
        self.peer_ready = True

    def set_oneshot(self, max_bytes: int):
        """Mode P2P: the one-shot small-message exchange up to max_bytes (0 = off)."""
        _check(lib.fp8lm_plan_set_oneshot(self.handle, int(max_bytes)), "fp8lm_plan_set_oneshot")

    def set_oneshot_raw(self, max_bytes: int):
        """Mode P2P: the one-handshake raw one-shot up to max_bytes (0 = off; plans <= 1 MiB)."""
        _check(lib.fp8lm_plan_set_oneshot_raw(self.handle, int(max_bytes)), "fp8lm_plan_set_oneshot_raw")

    def _window(self, ptr, n, typestr):
        if not ptr:
            raise FP8LMError("peer window missing: fp8lm_peer_setup has not run")

        class _Win:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(_Win(), device=self.device)

    def peer_g8(self) -> torch.Tensor:
        """Mode P2P: this rank's g8 window as a uint8 tensor (no copy)."""
        return self._window(lib.fp8lm_peer_g8(self.handle), self.g8_bytes, "|u1")

    def peer_w8(self) -> torch.Tensor:
        """Mode ZERO: the replicated FP8 weight copy (full layout) as a uint8 tensor."""
        return self._window(lib.fp8lm_peer_w8(self.handle), max(self.total, 1), "|u1")

    def peer_w8_scalars(self) -> torch.Tensor:
        """Mode ZERO: [3, T] float rows (scale, scale_inv, amax) of the replicated w8."""
        return self._window(lib.fp8lm_peer_w8_scalars(self.handle), 3 * self.T, "<f4").view(3, self.T)

    # ---- mode ZERO: the compact layout of the owned tensors
    def owner(self, t: int) -> int:
        return lib.fp8lm_plan_owner(self.handle, t)

    def owned(self):
        """-> list of (t, compact offset) of the tensors this rank owns (ascending t)."""
        out = []
        for t in range(self.T):
            o = lib.fp8lm_plan_owned_offset(self.handle, t)
            if o >= 0:
                out.append((t, o))
        return out

    def compact(self) -> "CompactLayout":
        return CompactLayout(self)

    def shard_begin(self, rank: int) -> int:
        return lib.fp8lm_plan_shard_begin(self.handle, rank)

    # flat buffers in plan layout
    def flat(self, dtype, nbytes_like_g8: bool = False) -> torch.Tensor:
        n = self.g8_bytes if nbytes_like_g8 else self.total
        return torch.zeros(max(n, 1), dtype=dtype, device=self.device)

    def views(self, flat: torch.Tensor, shapes=None) -> List[torch.Tensor]:
        out = []
        for t in range(self.T):
            v = flat[self.offsets[t]: self.offsets[t] + self.numels[t]]
            out.append(v.view(shapes[t]) if shapes is not None else v)
        return out

    def gather(self, flat: torch.Tensor, t: int) -> torch.Tensor:
        return flat[self.offsets[t]: self.offsets[t] + self.numels[t]]


class CompactLayout:
    """Mode ZERO: flat layout of the owned tensors (optimizer state lives only here)."""

    def __init__(self, plan: Plan):
        self.plan = plan
        self.device = plan.device
        self.total = lib.fp8lm_plan_owned_total(plan.handle)
        self.T = lib.fp8lm_plan_owned_count(plan.handle)
        self.entries = plan.owned()                    # [(t, offset)]
        self.numels = [plan.numels[t] for t, _ in self.entries]
        self.offsets = [o for _, o in self.entries]

    def flat(self, dtype) -> torch.Tensor:
        return torch.zeros(max(self.total, 1), dtype=dtype, device=self.device)

    def gather(self, full_flat: torch.Tensor) -> torch.Tensor:
        """compact copy of the owned tensors of a full-layout buffer"""
        out = self.flat(full_flat.dtype)
        for (t, o), n in zip(self.entries, self.numels):
            out[o:o + n] = self.plan.gather(full_flat, t)
        return out


class STensorSet:
    """T scaling tensors packed flat: data + scale / scale_inv / amax [T]."""

    def __init__(self, plan: Plan, dtype: torch.dtype):
        self.data = plan.flat(dtype)
        dev = plan.device
        self.scale = torch.ones(max(plan.T, 1), dtype=torch.float32, device=dev)
        self.scale_inv = torch.ones(max(plan.T, 1), dtype=torch.float32, device=dev)
        self.amax = torch.zeros(max(plan.T, 1), dtype=torch.float32, device=dev)

    def c(self) -> STensors:
        return STensors(self.data.data_ptr(), self.scale.data_ptr(), self.scale_inv.data_ptr(),
                        self.amax.data_ptr())


class OptimizerState:
    """6 B/param FP8 optimizer state (Eq. 8) + the E4M3 weight copy."""

    def __init__(self, plan: Plan):
        self.m1 = STensorSet(plan, torch.uint8)        # E4M3
        self.v = STensorSet(plan, torch.float16)       # FP16 (scaled, R17)
        self.master = STensorSet(plan, torch.float16)  # FP16 (scaled)
        self.w8 = STensorSet(plan, torch.uint8)        # E4M3 weight copy

    def tensors(self):
        return dict(m1=self.m1, v=self.v, master=self.master, w8=self.w8)


def peer_setup_loopback(plans: Sequence[Plan], stream=None):
    """fp8lm_peer_setup_loopback: plans[r] (mode P2P or ZERO, nranks = len(plans),
    rank r) become the ranks of one single-process group on this GPU.  Each rank must then
    run its calls on its own stream (the ranks' kernels meet at peer flags)."""
    arr = (_p * len(plans))(*[p.handle.value for p in plans])
    _check(lib.fp8lm_peer_setup_loopback(arr, len(plans), _stream(stream)), "fp8lm_peer_setup_loopback")
    for p in plans:
        p.peer_ready = True


def set_peer_timeout(seconds: float):
    """Peer-wait watchdog (fp8lm_set_peer_timeout): 0 = wait forever."""
    _check(lib.fp8lm_set_peer_timeout(float(seconds)), "fp8lm_set_peer_timeout")


def peer_timeout_report():
    """-> (hit, flag index, epoch wanted, value seen) of the last watchdog trap, or zeros."""
    out = (C.c_uint32 * 4)()
    _check(lib.fp8lm_peer_timeout_report(out), "fp8lm_peer_timeout_report")
    return tuple(out)


# ------------------------------------------------------------------ the four calls
def fp8_quantize(src: torch.Tensor, fmt: int = E4M3, jit: bool = True, scale: torch.Tensor = None,
                 out: torch.Tensor = None, count_sat: bool = False, stream=None):
    """fp8lm_quantize on one tensor -> (codes, scale, scale_inv, amax, sat)."""
    src = src.contiguous()
    n = src.numel()
    dev = src.device
    if out is None:
        out = torch.empty(n, dtype=torch.uint8 if fmt != F16 else torch.float16, device=dev)
    if scale is None:
        scale = torch.ones(1, dtype=torch.float32, device=dev)
    scale_inv = torch.ones(1, dtype=torch.float32, device=dev)
    amax = torch.zeros(1, dtype=torch.float32, device=dev)
    sat = torch.zeros(1, dtype=torch.int32, device=dev) if count_sat else None
    _check(lib.fp8lm_quantize(_ptr(src), _dtype_code(src), n, fmt, _ptr(out), _ptr(scale),
                              _ptr(scale_inv), _ptr(amax), 1 if jit else 0, _ptr(sat), _stream(stream)),
           "fp8lm_quantize")
    return out, scale, scale_inv, amax, sat


def fp8_dequantize(codes: torch.Tensor, fmt: int, scale_inv: torch.Tensor, stream=None):
    out = torch.empty(codes.numel(), dtype=torch.float32, device=codes.device)
    _check(lib.fp8lm_dequantize(_ptr(codes), fmt, codes.numel(), _ptr(scale_inv), _ptr(out),
                                _stream(stream)), "fp8lm_dequantize")
    return out


# ------------------------------------------------------------------ SP converter (f4)
class SPConverter:
    """FP8 activation converter g between the sequence- and tensor-parallel regions
    (§2.3, Fig. 5): all-gather (forward) and reduce-scatter (backward) of activations in
    E4M3 over NVLink peer memory (fp8lm_sp_*).  comm=None: a single rank."""

    def __init__(self, max_elems: int, comm: Optional[Comm] = None, device=None, stream=None):
        self.nranks = comm.nranks if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        h = _p()
        _check(lib.fp8lm_sp_create(comm.handle if comm is not None else None, int(max_elems),
                                   _stream(stream), C.byref(h)), "fp8lm_sp_create")
        self.handle = h
        self.scale = torch.ones(2, dtype=torch.float32, device=self.device)

    def allgather(self, x: torch.Tensor, out_dtype=torch.bfloat16, codes: bool = False,
                  out: torch.Tensor = None, codes_out: torch.Tensor = None, stream=None):
        """x: this rank's partition (fp32 / bf16, m elements).  Returns (out [N m] of
        out_dtype or None, codes [N m] uint8 or None); self.scale = (s, 1/s)."""
        x = x.contiguous()
        m = x.numel()
        if out is None and out_dtype is not None:
            out = torch.empty(self.nranks * m, dtype=out_dtype, device=x.device)
        if codes and codes_out is None:
            codes_out = torch.empty(self.nranks * m, dtype=torch.uint8, device=x.device)
        _check(lib.fp8lm_sp_allgather(self.handle, _ptr(x), _dtype_code(x), m, _ptr(codes_out), _ptr(out),
                                      _dtype_code(out) if out is not None else F32, _ptr(self.scale),
                                      _stream(stream)), "fp8lm_sp_allgather")
        return out, codes_out

    def reduce_scatter(self, dy: torch.Tensor, out_dtype=torch.bfloat16, out: torch.Tensor = None,
                       stream=None):
        """dy: this rank's full gradient (N m elements).  Returns this rank's chunk [m] of
        the sum, in out_dtype."""
        dy = dy.contiguous()
        assert dy.numel() % self.nranks == 0
        m = dy.numel() // self.nranks
        if out is None:
            out = torch.empty(m, dtype=out_dtype, device=dy.device)
        _check(lib.fp8lm_sp_reduce_scatter(self.handle, _ptr(dy), _dtype_code(dy), m, _ptr(out),
                                           _dtype_code(out), _ptr(self.scale), _stream(stream)),
               "fp8lm_sp_reduce_scatter")
        return out

    def close(self):
        if self.handle:
            lib.fp8lm_sp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ strategies (f3)
STRATEGIES = {"pre": 0, "post": 1, "auto": 2}
# fp8lm_commstats (include/fp8lm.h): 5 x 8-byte fields, 2 u32, 6 f32, 4 u32 scratch
_COMMSTATS = struct.Struct("<ddQQQIIffffff4I")
COMMSTATS_BYTES = _COMMSTATS.size


def commstats_buffer(device) -> torch.Tensor:
    """A zero-initialised device fp8lm_commstats (reuse it across calls)."""
    return torch.zeros(COMMSTATS_BYTES // 8, dtype=torch.float64, device=device)


def commstats_read(buf: torch.Tensor) -> dict:
    """Host dict of one fp8lm_commstats (synchronises)."""
    v = _COMMSTATS.unpack(buf.detach().cpu().numpy().tobytes())
    keys = ("sig2", "err2", "underflow", "overflow", "events", "sat", "nonfinite", "amax", "s",
            "scale", "scale_inv", "mu_used", "mu_next")
    d = dict(zip(keys, v[:13]))
    raw = (C.c_uint8 * COMMSTATS_BYTES).from_buffer_copy(buf.detach().cpu().numpy().tobytes())
    out = (C.c_double * 3)()
    _check(lib.fp8lm_commstats_metrics(C.cast(raw, _p), out), "fp8lm_commstats_metrics")
    d["snr_db"], d["underflow_rate"], d["overflow_rate"] = out[0], out[1], out[2]
    return d


def commstats_metrics(sig2: float, err2: float, underflow: int, overflow: int, events: int):
    """fp8lm_commstats_metrics on aggregated sums (several calls' statistics added up):
    -> (snr_db, underflow_rate, overflow_rate)."""
    raw = _COMMSTATS.pack(sig2, err2, underflow, overflow, events, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0)
    buf = (C.c_uint8 * len(raw)).from_buffer_copy(raw)
    out = (C.c_double * 3)()
    _check(lib.fp8lm_commstats_metrics(C.cast(buf, _p), out), "fp8lm_commstats_metrics")
    return out[0], out[1], out[2]


def allreduce_strategy(grads: torch.Tensor, strategy, mu: torch.Tensor = None,
                       codes: torch.Tensor = None, stats: torch.Tensor = None, stream=None):
    """fp8lm_allreduce_strategy: N ranks' gradients as rows of a [N, n] fp32 device tensor;
    strategy "pre" | "post" | "auto" (Eq. 1 / Eq. 2 / Eq. 3-6).  Returns (codes, stats
    buffer); read the statistics with commstats_read.  mu (device float[1]) is updated in
    place by "auto"."""
    st = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    assert grads.dim() == 2 and grads.dtype == torch.float32 and grads.is_contiguous()
    N, n = grads.shape
    dev = grads.device
    if codes is None:
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
    if stats is None:
        stats = commstats_buffer(dev)
    if st == 2 and mu is None:
        raise ValueError("strategy auto needs mu")
    _check(lib.fp8lm_allreduce_strategy(st, _ptr(grads), N, n, _ptr(mu), _ptr(codes), _ptr(stats),
                                        _stream(stream)), "fp8lm_allreduce_strategy")
    return codes, stats


def _grads_arg(plan: Plan, grads):
    """mode SIMULATED: a list of flat per-rank buffers -> host pointer array."""
    if plan.mode == MODE_SIMULATED:
        assert len(grads) == plan.nranks
        arr = (_p * plan.nranks)(*[g.data_ptr() for g in grads])
        return C.cast(arr, _p), _dtype_code(grads[0]), arr
    return _ptr(grads), _dtype_code(grads), None


def amax_scale_sync(plan: Plan, grads, mu: torch.Tensor, amax_out: torch.Tensor, s_g: torch.Tensor,
                    skip: torch.Tensor, comm: Comm = None, stream=None):
    g, dt, keep = _grads_arg(plan, grads)
    _check(lib.fp8lm_amax_scale_sync(plan.handle, comm.handle if comm else None, g, dt, _ptr(mu),
                                     _ptr(amax_out), _ptr(s_g), _ptr(skip), _stream(stream)),
           "fp8lm_amax_scale_sync")
    del keep


def fp8_grad_allreduce(plan: Plan, grads, s_g: torch.Tensor, skip: torch.Tensor, g8: torch.Tensor,
                       g_scale: torch.Tensor, g_scale_inv: torch.Tensor, sat: torch.Tensor,
                       mu: torch.Tensor, comm: Comm = None, stream=None):
    g, dt, keep = _grads_arg(plan, grads)
    _check(lib.fp8lm_grad_allreduce(plan.handle, comm.handle if comm else None, g, dt, _ptr(s_g),
                                    _ptr(skip), _ptr(g8), _ptr(g_scale), _ptr(g_scale_inv),
                                    _ptr(sat), _ptr(mu), _stream(stream)),
           "fp8lm_grad_allreduce")
    del keep


def allreduce_jit(plan: Plan, grads, mu: torch.Tensor, amax_out: torch.Tensor, s_g: torch.Tensor,
                  skip: torch.Tensor, g8: torch.Tensor, g_scale: torch.Tensor, g_scale_inv: torch.Tensor,
                  sat: torch.Tensor, comm: Comm = None, stream=None):
    """fp8lm_allreduce_jit: amax_scale_sync + fp8_grad_allreduce in one call (mode P2P,
    small plans: one kernel)."""
    g, dt, keep = _grads_arg(plan, grads)
    _check(lib.fp8lm_allreduce_jit(plan.handle, comm.handle if comm else None, g, dt, _ptr(mu), _ptr(amax_out),
                                   _ptr(s_g), _ptr(skip), _ptr(g8), _ptr(g_scale), _ptr(g_scale_inv), _ptr(sat),
                                   _stream(stream)), "fp8lm_allreduce_jit")
    del keep


def fp8_adam_step(plan: Plan, g8: torch.Tensor, g_scale_inv: torch.Tensor, st: OptimizerState,
                  hp: AdamHP, skip: torch.Tensor, stream=None):
    m1, v, w, w8 = st.m1.c(), st.v.c(), st.master.c(), st.w8.c()
    _check(lib.fp8lm_adam_step(plan.handle, _ptr(g8), _ptr(g_scale_inv), C.byref(m1), C.byref(v),
                               C.byref(w), C.byref(w8), C.byref(hp), _ptr(skip), _stream(stream)),
           "fp8lm_adam_step")


def fp8_adam_step_delayed(plan: Plan, g8: torch.Tensor, g_scale_inv: torch.Tensor, st: OptimizerState,
                          hp: AdamHP, skip: torch.Tensor, w_hist: torch.Tensor, hist_slot: int,
                          stream=None):
    m1, v, w, w8 = st.m1.c(), st.v.c(), st.master.c(), st.w8.c()
    _check(lib.fp8lm_adam_step_delayed(plan.handle, _ptr(g8), _ptr(g_scale_inv), C.byref(m1), C.byref(v),
                                       C.byref(w), C.byref(w8), C.byref(hp), _ptr(skip), _ptr(w_hist),
                                       hist_slot, _stream(stream)), "fp8lm_adam_step_delayed")


def state_init(plan: Plan, w0_flat: torch.Tensor, st: OptimizerState, stream=None):
    m1, v, w, w8 = st.m1.c(), st.v.c(), st.master.c(), st.w8.c()
    _check(lib.fp8lm_state_init(plan.handle, _ptr(w0_flat), C.byref(m1), C.byref(v), C.byref(w),
                                C.byref(w8), _stream(stream)), "fp8lm_state_init")


# ------------------------------------------------------------------ the whole DP step
class FP8DataParallel:
    """The full hot path (§8a rows A1-A7) for one rank: owns the per-step device scalars.

    step(grads, lr): amax_scale_sync -> fp8_grad_allreduce -> fp8_adam_step, all on the
    current stream, no host synchronisation.  After it, .w8 (E4M3 weight copy) and its
    scale feed the next forward pass; .mu is already updated for the next step."""

    def __init__(self, plan: Plan, w0_flat: torch.Tensor, comm: Comm = None, lr: float = 3e-4,
                 betas=(0.9, 0.95), eps: float = 1e-8, weight_decay: float = 0.1,
                 fused: bool = True, state_scaling: str = "jit", graphed: bool = False):
        """graphed: fp8lm_dp_step_graphed — the step as a CUDA graph (captured on the
        second call with the same buffers, then replayed with the step's scalars patched)."""
        self.fused = fused
        self.graphed = graphed
        assert state_scaling in ("jit", "delayed")
        self.delayed = state_scaling == "delayed"
        self.plan, self.comm = plan, comm
        dev = plan.device
        T = max(plan.T, 1)
        nsim = plan.nranks if plan.mode == MODE_SIMULATED else 1
        self.mu = torch.ones(T, dtype=torch.float32, device=dev)
        self.amax = torch.zeros(nsim * T, dtype=torch.float32, device=dev)
        self.s_g = torch.zeros(T, dtype=torch.float32, device=dev)
        self.skip = torch.zeros(1, dtype=torch.int32, device=dev)
        self.layout = plan
        if plan.mode == MODE_P2P:
            plan.peer_setup(comm)       # no-op after peer_setup_loopback
            self.g8 = plan.peer_g8()
            self.comm = None            # the exchange runs in the library's kernels
        elif plan.mode == MODE_ZERO:
            plan.peer_setup(comm)
            self.comm = None
            self.layout = plan.compact()               # optimizer state: owned tensors only
            self.g8 = self.layout.flat(torch.uint8)
            w0_flat = self.layout.gather(w0_flat)
            self.w8_full = plan.peer_w8()
            self.w8_full_scalars = plan.peer_w8_scalars()
        else:
            self.g8 = plan.flat(torch.uint8, nbytes_like_g8=True)
        self.g_scale = torch.zeros(T, dtype=torch.float32, device=dev)
        self.g_scale_inv = torch.zeros(T, dtype=torch.float32, device=dev)
        self.sat = torch.zeros(T, dtype=torch.int32, device=dev)
        self.state = OptimizerState(self.layout)
        state_init(plan, w0_flat, self.state)
        self.w_hist = None
        if self.delayed:      # amax(w) history ring [16][T]: amax(w0) in slot 0 (R26)
            Tl = max(self.layout.T, 1)
            self.w_hist = torch.zeros(16 * Tl, dtype=torch.float32, device=dev)
            self.w_hist[:Tl].copy_(self.state.master.amax[:Tl])
        self.lr, self.betas, self.eps, self.wd = lr, betas, eps, weight_decay
        self.t = 0

    def step(self, grads, lr: float = None, stream=None):
        self.t += 1
        hp = adam_hp(self.lr if lr is None else lr, self.t, self.betas[0], self.betas[1], self.eps, self.wd)
        if self.fused:
            g, dt, keep = _grads_arg(self.plan, grads)
            st = self.state
            m1, v, w, w8 = st.m1.c(), st.v.c(), st.master.c(), st.w8.c()
            fn = lib.fp8lm_dp_step_graphed if self.graphed else lib.fp8lm_dp_step
            _check(fn(self.plan.handle, self.comm.handle if self.comm else None, g, dt,
                      _ptr(self.mu), _ptr(self.amax), _ptr(self.s_g), _ptr(self.skip),
                      _ptr(self.g8), _ptr(self.g_scale), _ptr(self.g_scale_inv),
                      _ptr(self.sat), C.byref(m1), C.byref(v), C.byref(w),
                      C.byref(w8), C.byref(hp), _ptr(self.w_hist), (self.t - 1) % 16,
                      _stream(stream)), "fp8lm_dp_step")
            del keep
            return
        self._three_calls(grads, hp, stream)

    def _split(self, phase: int, grads, hp: AdamHP, stream):
        g, dt, keep = _grads_arg(self.plan, grads) if grads is not None else (None, F32, None)
        st = self.state
        m1, v, w, w8 = st.m1.c(), st.v.c(), st.master.c(), st.w8.c()
        _check(lib.fp8lm_dp_step_split(self.plan.handle, phase, g, dt, _ptr(self.mu), _ptr(self.amax),
                                       _ptr(self.s_g), _ptr(self.skip), _ptr(self.g8), _ptr(self.g_scale),
                                       _ptr(self.g_scale_inv), _ptr(self.sat), C.byref(m1), C.byref(v),
                                       C.byref(w), C.byref(w8), C.byref(hp), _ptr(self.w_hist),
                                       (self.t - 1) % 16, _stream(stream)), "fp8lm_dp_step_split")
        del keep

    def step_begin(self, grads, lr: float = None, stream=None):
        """Phase 1 of fp8lm_dp_step_split (modes P2P / ZERO): amax, scale MIN and quantize on
        the stream, the exchange on the plan's exchange stream."""
        self.t += 1
        self._hp = adam_hp(self.lr if lr is None else lr, self.t, self.betas[0], self.betas[1], self.eps,
                           self.wd)
        self._split(1, grads, self._hp, stream)

    def step_end(self, stream=None):
        """Phase 2: wait for this plan's exchange, then the AdamW pass (pulled all-gather)."""
        self._split(2, None, self._hp, stream)

    def _three_calls(self, grads, hp, stream):
        amax_scale_sync(self.plan, grads, self.mu, self.amax, self.s_g, self.skip, self.comm, stream)
        fp8_grad_allreduce(self.plan, grads, self.s_g, self.skip, self.g8, self.g_scale,
                           self.g_scale_inv, self.sat, self.mu, self.comm, stream)
        if self.delayed:
            fp8_adam_step_delayed(self.plan, self.g8, self.g_scale_inv, self.state, hp, self.skip,
                                  self.w_hist, (self.t - 1) % 16, stream)
        else:
            fp8_adam_step(self.plan, self.g8, self.g_scale_inv, self.state, hp, self.skip, stream)


# ------------------------------------------------------------------ bucketed step (f2)
def bucket_split(numels: Sequence[int], buckets: int) -> List[List[int]]:
    """Contiguous groups of tensor indices with about equal parameter counts."""
    total = sum(numels)
    out, cur, acc = [], [], 0
    for t, n in enumerate(numels):
        cur.append(t)
        acc += n
        if len(out) < buckets - 1 and acc >= total * (len(out) + 1) / buckets:
            out.append(cur)
            cur = []
    if cur:
        out.append(cur)
    return out


class BucketedDP:
    """Modes P2P / ZERO with the tensors split into buckets (one plan each): every step
    issues phase 1 of every bucket, then phase 2 of every bucket (fp8lm_dp_step_split),
    so the exchange of bucket b runs on its exchange stream beside the amax / quantize of
    bucket b+1 and the AdamW pass of bucket b-1 on the caller's stream."""

    def __init__(self, plans: Sequence[Plan], w0s: Sequence[torch.Tensor], comm: Comm = None,
                 lag: int = 0, **kw):
        """lag: 0 = phase 1 of every bucket, then phase 2 of every bucket; k > 0 = phase 2 of
        bucket b is issued after phase 1 of bucket b + k (a software pipeline of depth k)."""
        self.plans = list(plans)
        self.lag = lag
        self.dps = [FP8DataParallel(p, w, comm=comm, **kw) for p, w in zip(self.plans, w0s)]

    def step(self, grads: Sequence[torch.Tensor], lr: float = None, stream=None):
        B = len(self.dps)
        lag = self.lag if self.lag > 0 else B
        done = 0
        for b, (dp, g) in enumerate(zip(self.dps, grads)):
            dp.step_begin(g, lr, stream)
            if b - done >= lag:
                self.dps[done].step_end(stream)
                done += 1
        for dp in self.dps[done:]:
            dp.step_end(stream)
