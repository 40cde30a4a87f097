"""The device encoder on EVERY binary32 bit pattern (2^32 inputs, unit scale) for E4M3,
E5M2 and FP16 against torch's clamp + cast on the same device — the third-party encoder
that tests/test_oracle_codec.py::test_vs_third_party_casts pins to the oracle's exact
codec (App. A, reading R11: saturating round-to-nearest-even).  NaN inputs:
only the NaN class is compared (R23).  SURVEY §4 T1."""
import pytest
import torch

from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _ref(x, fmt):
    if fmt == "e4m3":
        return x.clamp(-448, 448).to(torch.float8_e4m3fn).view(torch.uint8).to(torch.int32)
    if fmt == "e5m2":
        return x.clamp(-57344, 57344).to(torch.float8_e5m2).view(torch.uint8).to(torch.int32)
    return x.clamp(-65504, 65504).half().view(torch.int16).to(torch.int32) & 0xFFFF


@pytest.mark.parametrize("fmt", ["e4m3", "e5m2", "f16"])
def test_device_encoder_every_binary32(fmt):
    import paper_2310_18313_b200 as B
    code = {"e4m3": B.E4M3, "e5m2": B.E5M2, "f16": B.F16}[fmt]
    chunk = 1 << 28
    scale = torch.ones(1, device="cuda")
    out = torch.empty(chunk, dtype=torch.uint8 if fmt != "f16" else torch.float16, device="cuda")
    nan_max = {"e4m3": 0x7F, "e5m2": 0x7F, "f16": 0x7FFF}[fmt]
    nan_min = {"e4m3": 0x7F, "e5m2": 0x7D, "f16": 0x7C01}[fmt]
    checked = 0
    for lo in range(-(1 << 31), 1 << 31, chunk):
        bits = torch.arange(lo, lo + chunk, dtype=torch.int32, device="cuda")
        x = bits.view(torch.float32)
        codes, *_ = B.fp8_quantize(x, code, jit=False, scale=scale, out=out)
        got = (codes.view(torch.int16).to(torch.int32) & 0xFFFF) if fmt == "f16" else codes.to(torch.int32)
        ref = _ref(x, fmt)
        nan = torch.isnan(x)
        bad = (got != ref) & ~nan
        nbad = int(bad.sum().item())
        assert nbad == 0, (fmt, hex(lo & 0xFFFFFFFF), nbad,
                           bits[bad][:4].tolist(), got[bad][:4].tolist(), ref[bad][:4].tolist())
        mag = got[nan] & nan_max
        assert bool(((mag >= nan_min) & (mag <= nan_max)).all()), (fmt, "NaN class")
        checked += chunk
    assert checked == 1 << 32
