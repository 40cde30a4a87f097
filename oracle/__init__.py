"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct numpy implementation of the FP8-LM data-parallel
hot path (arXiv 2310.18313 §2.1-§2.3, App. A-B), written from PAPER.md with the
readings listed in DESIGN.md §3.  It shares no code with the CUDA path
(``paper_2310_18313_b200``) and neither imports the other.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.
The product path never routes through it.

Arithmetic model: every floating-point step is IEEE-754 binary32 with one
round-to-nearest-even per operation (numpy float32 elementwise ops; numpy never
contracts to FMA), because the method's outputs are FP8/FP16 codes whose rounding
decisions must be taken in the kernel's precision (task rule ③; R16).
The codec itself is computed exactly in float64 (every binary32 value and every
FP8/FP16 grid point is exact in float64).

Modules
  codec     — E4M3 / E5M2 / FP16 decode and saturating RNE encode (App. A)
  pipeline  — amax, mu controller, local/global scale, quantize, rank-order reduce,
              requantize, saturation count, dequantize (§2.1, Eq. 3-6)
  adam      — precision-decoupled AdamW, JIT state scaling (§2.2; App. B)
  zero      — Alg. 1 greedy whole-tensor distribution (§2.3)
  step      — the whole data-parallel step for N simulated ranks (composition)

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (see
DESIGN.md §4 "pins"); none is "parity unpinned".
"""
from . import codec, pipeline, adam, zero, step  # noqa: F401
