"""torchrun worker for the FP8 SP converter parity test (tests/test_gpu_sp.py): every
rank regenerates every rank's activations (seeded), runs fp8lm_sp_allgather and
fp8lm_sp_reduce_scatter over NVLink peer memory and compares its outputs bit for bit
with oracle/sp.py (§2.3; readings R31-R32).  Prints
"SP parity N=<n>: OK" iff every rank matched.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/sp_worker.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import sp as SP  # noqa: E402

# m values: vector sizes, ragged sizes, tiny, and one rank's activation of a GPT-13B
# TP=2 micro-batch slice (2048 tokens x 5120 / 2 ranks = 5.2M elements)
SIZES = [4096, 1000, 3, 16, 5242880, 65552]


def acts(r, m, seed, dtype):
    g = torch.Generator()
    g.manual_seed(1000 * seed + r)
    x = torch.randn(m, generator=g) * (10.0 ** ((seed % 5) - 2)) * (1 + r)
    return x.to(dtype)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import paper_2310_18313_b200 as B
    comm = B.Comm.from_torch_distributed()
    conv = B.SPConverter(max_elems=N * max(SIZES), comm=comm)
    ok = True
    for it, m in enumerate(SIZES):
        for in_dt, out_dt in ((torch.float32, torch.float32), (torch.bfloat16, torch.bfloat16)):
            # forward: all-gather of the sequence partitions
            parts = [acts(r, m, it, in_dt) for r in range(N)]
            out, codes = conv.allgather(parts[rank].cuda(), out_dtype=out_dt, codes=True)
            ref = SP.allgather_fp8([p.float().numpy() for p in parts])
            want = ref["out"] if out_dt == torch.float32 else SP.bf16_round(ref["out"])
            got = out.float().cpu().numpy()
            if not (np.array_equal(codes.cpu().numpy(), ref["codes"]) and
                    np.array_equal(got.view(np.uint32), want.view(np.uint32)) and
                    conv.scale[0].item() == ref["scale"]):
                print(f"rank {rank}: all-gather m={m} {in_dt} mismatch", flush=True)
                ok = False
            # backward: reduce-scatter of the full activation gradients
            full = [acts(r, N * m, 100 + it, in_dt) for r in range(N)]
            o = conv.reduce_scatter(full[rank].cuda(), out_dtype=out_dt)
            ref = SP.reduce_scatter_fp8([f.float().numpy() for f in full])
            want = ref["out_by_rank"][rank]
            if out_dt == torch.bfloat16:
                want = SP.bf16_round(want)
            if not (np.array_equal(o.float().cpu().numpy().view(np.uint32), want.view(np.uint32)) and
                    conv.scale[0].item() == ref["scale"]):
                print(f"rank {rank}: reduce-scatter m={m} {in_dt} mismatch", flush=True)
                ok = False
    torch.cuda.synchronize()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    conv.close()
    comm.close()
    if rank == 0:
        print(f"SP parity N={N}: {'OK' if flag.item() == 1 else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
