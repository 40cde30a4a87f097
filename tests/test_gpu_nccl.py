"""Multi-GPU parity (one process per GPU, torchrun), bit-exact against the N-rank
oracle, for both exchange modes:
  nccl: amax -> MIN all-reduce -> quantize -> ncclAlltoAll -> rank-order reduce of the
        own shard -> in-place ncclAllGather + summed saturation counts -> mu -> AdamW;
  p2p:  the same arithmetic with the MIN exchanged through peer pads and reduce-scatter
        + reduce + all-gather fused in one kernel over NVLink peer memory;
  zero: FP8 ZeRO (Alg. 1): the owner of each whole tensor reduces it from every rank's
        send window and runs AdamW on it alone (through fp8lm_dp_step: pass 1 inside the
        owner reduce; "unfused": the three calls); w8 + scalars replicated by peer stores.
Needs >= 2 GPUs (gpurun --gpus 2 / 4)."""
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["nccl", "p2p", "p2p_unfused", "zero", "zero_unfused", "p2p_delayed",
                                  "zero_delayed", "p2p_oneshot", "p2p_unfused_oneshot", "p2p_oneshot_raw"])
@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_bit_exact(n, mode):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), "--steps", "3",
           "--mode", mode.split("_")[0]] + (["--unfused"] if "unfused" in mode else []) + \
          (["--delayed"] if "delayed" in mode else []) + (["--oneshot"] if "oneshot" in mode else []) + \
          (["--raw"] if "raw" in mode else [])
    env = dict(os.environ)
    for _ in range(3):          # a freshly probed port can be taken before torchrun binds it
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
        if "EADDRINUSE" not in r.stderr:
            break
        cmd[cmd.index("--master-port") + 1] = str(_port())
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"{mode.upper()} parity N={n}: OK" in r.stdout
