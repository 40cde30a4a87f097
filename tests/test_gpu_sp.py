"""GPU parity of the FP8 SP/TP activation converter g (fp8lm_sp_*; §2.3
P:193-200, Fig. 5; readings R31-R32) against oracle/sp.py: one rank on one GPU (the
degenerate N = 1 path through the same kernels), and N = 2, 4 GPUs under torchrun
(tests/sp_worker.py) — gathered codes, outputs and scales bit-exact."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import sp as SP
from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2310_18313_b200 as B
    return B


@pytest.mark.parametrize("m", [1, 15, 16, 1000, 65536, 1000003])
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_single_rank_converter(B, m, dt):
    conv = B.SPConverter(max_elems=2_000_000)
    g = torch.Generator()
    for rep in range(2):                                   # consecutive epochs
        g.manual_seed(m + rep)
        x = (torch.randn(m, generator=g) * 3e-2).to(dt)
        out, codes = conv.allgather(x.cuda(), out_dtype=torch.float32, codes=True)
        ref = SP.allgather_fp8([x.float().numpy()])
        assert np.array_equal(codes.cpu().numpy(), ref["codes"])
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref["out"].view(np.uint32))
        assert conv.scale[0].item() == ref["scale"] and conv.scale[1].item() == ref["scale_inv"]
        o = conv.reduce_scatter(x.cuda(), out_dtype=torch.bfloat16)
        r2 = SP.reduce_scatter_fp8([x.float().numpy()])
        assert np.array_equal(o.float().cpu().numpy().view(np.uint32),
                              SP.bf16_round(r2["out_by_rank"][0]).view(np.uint32))
    conv.close()


def test_zero_and_oversize(B):
    conv = B.SPConverter(max_elems=64)
    out, codes = conv.allgather(torch.zeros(64, device="cuda"), out_dtype=torch.float32, codes=True)
    assert conv.scale[0].item() == 1.0 and torch.all(out == 0) and torch.all(codes == 0)
    with pytest.raises(B.FP8LMError):
        conv.allgather(torch.zeros(65, device="cuda"))
    conv.close()


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_converter(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "sp_worker.py")]
    for _ in range(3):          # a freshly probed port can be taken before torchrun binds it
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
        cmd[cmd.index("--master-port") + 1] = str(_port())
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"SP parity N={n}: OK" in r.stdout
