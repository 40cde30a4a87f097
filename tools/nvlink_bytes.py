#!/usr/bin/env python
"""NVLink bytes per step of the fused exchange kernels, from the NVML NVLink counters.

ncu cannot profile the exchange kernels (they spin on flags that another process's
kernel sets, and ncu serialises and replays kernels), so this reads the driver's
per-GPU NVLink byte counters around K steps instead:

  torchrun --nproc-per-node N tools/nvlink_bytes.py [--config gpt-125m] [--exchange p2p|zero]

Each rank reads its own GPU's counters (every NVLink field NVML exposes for bytes,
summed over the links; the return code is printed for fields the driver does not
support) before and after K steps of FP8DataParallel.step (unsplit), and rank 0 prints
one JSON line per rank: counter bytes per step against the algorithmic NVLink bytes per
step and rank — P2P: the reduce-scatter pulls (N-1)/N n plus the all-gather pulls
(N-1)/N n of codes; ZERO: the owner pulls (N-1)/N n plus the w8 broadcast (N-1)/N n
(both directions of every link carry the same amount).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def nvml_fields():
    import pynvml as p
    names = ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
             "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX",
             "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES"]
    return [(n, getattr(p, n)) for n in names if hasattr(p, n)]


def read_counters(handle, nlinks=18):
    """{field: (sum over links, ok_links, first error)} — per-link scope, then the
    aggregate scope (0xFFFFFFFF) if no link answered."""
    import pynvml as p
    out = {}
    for name, fid in nvml_fields():
        tot, ok, err = 0, 0, None
        for link in list(range(nlinks)) + [0xFFFFFFFF]:
            if link == 0xFFFFFFFF and ok:
                break
            try:
                v = p.nvmlDeviceGetFieldValues(handle, [(fid, link)])[0]
                if v.nvmlReturn != 0:
                    err = err or int(v.nvmlReturn)
                    continue
                tot += int(v.value.ullVal)
                ok += 1
            except Exception as e:  # noqa: BLE001 — report, do not fail the run
                err = err or repr(e)[:80]
        out[name] = (tot, ok, err)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt-125m")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "zero"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, N = dist.get_rank(), dist.get_world_size()
    import pynvml
    import paper_2310_18313_b200 as B
    import synth

    pynvml.nvmlInit()
    props = torch.cuda.get_device_properties(local)
    try:
        h = pynvml.nvmlDeviceGetHandleByPciBusId(
            f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0")
    except Exception:  # noqa: BLE001
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
    specs = synth.gpt_gradient_set(args.config)
    numels = [s.numel for s in specs]
    comm = B.Comm.from_torch_distributed()
    mode = {"p2p": B.MODE_P2P, "zero": B.MODE_ZERO}[args.exchange]
    plan = B.Plan(numels, mode=mode, nranks=N, rank=rank)
    plan.set_oneshot(0)
    w0 = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(w0)):
        synth.fill_weights(v, t)
    dp = B.FP8DataParallel(plan, w0, comm=comm)
    g = plan.flat(torch.float32)
    for t, v in enumerate(plan.views(g)):
        synth.fill_gradient(v, 1, t, rank)
    for _ in range(args.warmup):
        dp.step(g)
    torch.cuda.synchronize()
    dist.barrier()
    c0 = read_counters(h)
    for _ in range(args.steps):
        dp.step(g)
    torch.cuda.synchronize()
    dist.barrier()
    c1 = read_counters(h)
    n = plan.total
    alg = 2.0 * (N - 1) / N * n      # bytes per step and rank, each direction
    row = {"rank": rank, "n_gpus": N, "config": args.config, "exchange": args.exchange, "params": n,
           "alg_nvlink_bytes_per_step_each_direction": alg, "steps": args.steps, "fields": {}}
    for k in c0:
        d = c1[k][0] - c0[k][0]
        row["fields"][k] = {"delta": d, "per_step": d / args.steps, "per_step_over_alg": d / args.steps / alg,
                            "links": c1[k][1], "err": c1[k][2]}
    rows = [None] * N
    dist.all_gather_object(rows, row)
    if rank == 0:
        for r in rows:
            print(json.dumps(r), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
