"""N > 1 host logic on CPU (world_size 2, 3 and 8, gloo): the NCCL-mode data flow of
fp8lm_amax_scale_sync / fp8lm_grad_allreduce — MIN all-reduce of the local scales
(Eq. 4), the flat code buffer split into N shards by the library's plan (all-to-all
transport), rank-order reduction of the own shard, in-place all-gather, summed
saturation counts, mu update — replayed with gloo collectives and the oracle's
per-element arithmetic, then compared with the single-process N-rank oracle.

This pins the plan's shard map (fp8lm_plan_shard_bytes / _begin / offsets) and the
collective sequencing; the GPU kernels themselves are covered by test_gpu_*.py and
by `gpurun --gpus 2` runs of bench.py / test_gpu_nccl.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

F32 = np.float32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


NUMELS = [3, 16, 17, 1000, 16385, 40000, 64, 5]


def _local_grads(rank, step):
    import synth
    out = []
    for t, n in enumerate(NUMELS):
        g = torch.empty(n, dtype=torch.float32)
        synth.fill_gradient(g, step, t, rank)
        out.append(g.numpy())
    return out


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import ctypes as C
        import paper_2310_18313_b200._binding as B
        from oracle import pipeline as P
        from oracle.codec import E4M3, decode_f32, encode

        arr = (C.c_int64 * len(NUMELS))(*NUMELS)
        h = C.c_void_p()
        assert B.lib.fp8lm_plan_create(len(NUMELS), arr, B.MODE_NCCL, world, rank, C.byref(h)) == 0
        offs = [B.lib.fp8lm_plan_offset(h, t) for t in range(len(NUMELS))]
        S = B.lib.fp8lm_plan_shard_bytes(h)
        g8_bytes = B.lib.fp8lm_plan_g8_bytes(h)
        begin = B.lib.fp8lm_plan_shard_begin(h, rank)
        assert begin == rank * S and g8_bytes == world * S

        mus = [F32(1.0)] * len(NUMELS)
        results = []
        for step in (1, 2, 3):
            g = _local_grads(rank, step)
            # (2) amax_scale_sync: local scale, MIN all-reduce, fix-ups
            s_loc = torch.tensor([P.local_scale(*P.amax(x), mus[t]) for t, x in enumerate(g)], dtype=torch.float32)
            dist.all_reduce(s_loc, op=dist.ReduceOp.MIN)
            s_g = [P.global_scale([F32(v)])[0] for v in s_loc.numpy()]
            skip = any(F32(v) == 0 for v in s_loc.numpy())
            # (3) quantize into the flat send buffer (plan layout)
            send = torch.zeros(g8_bytes, dtype=torch.uint8)
            for t, x in enumerate(g):
                send[offs[t]: offs[t] + NUMELS[t]] = torch.from_numpy(P.quantize(x, s_g[t]).astype(np.uint8))
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)          # chunk j (S bytes) -> rank j
            # reduce the own shard, tensor piece by tensor piece, count saturation
            g8 = torch.zeros(g8_bytes, dtype=torch.uint8)
            sat = torch.zeros(len(NUMELS), dtype=torch.int64)
            lo, hi = rank * S, (rank + 1) * S
            for t in range(len(NUMELS)):
                a, b = max(lo, offs[t]), min(hi, offs[t] + NUMELS[t])
                if a >= b:
                    continue
                parts = [recv[r * S + (a - lo): r * S + (b - lo)].numpy() for r in range(world)]
                c = P.requantize(P.rank_order_sum(parts))
                g8[a:b] = torch.from_numpy(c.astype(np.uint8))
                sat[t] += P.sat_count(c)
            # in-place all-gather of the reduced shards + summed counts
            pieces = list(g8.chunk(world))
            dist.all_gather(pieces, g8[lo:hi].clone())
            g8 = torch.cat(pieces)
            dist.all_reduce(sat, op=dist.ReduceOp.SUM)
            mus = [P.mu_update(mus[t], int(sat[t]), NUMELS[t], skip) for t in range(len(NUMELS))]
            results.append(dict(g8=[g8[offs[t]: offs[t] + NUMELS[t]].numpy().copy() for t in range(len(NUMELS))],
                                sat=sat.tolist(), mu=[float(m) for m in mus], s_g=[float(s) for s in s_g]))
        B.lib.fp8lm_plan_destroy(h)
        q.put((rank, results))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_nccl_mode_protocol_matches_n_rank_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]

    from oracle import pipeline as P
    mus = [F32(1.0)] * len(NUMELS)
    for si, step in enumerate((1, 2, 3)):
        grads = [_local_grads(r, step) for r in range(world)]
        ref = [P.allreduce_tensor([grads[r][t] for r in range(world)], mus[t]) for t in range(len(NUMELS))]
        skip = any(x["skip"] for x in ref)
        for r in range(world):
            res = got[r][si]
            for t in range(len(NUMELS)):
                assert np.array_equal(res["g8"][t], ref[t]["codes"]), (r, step, t)
                assert res["sat"][t] == ref[t]["sat"]
                assert F32(res["s_g"][t]) == ref[t]["s_g"]
        mus = [P.mu_update(mus[t], ref[t]["sat"], NUMELS[t], skip) for t in range(len(NUMELS))]
        for r in range(world):
            assert [F32(m) for m in got[r][si]["mu"]] == mus


# ---------------------------------------------------------------- mode P2P dp_step (pull)
def _pull_worker(rank, world, port, q):
    """fp8lm_dp_step in mode P2P: the exchange kernel leaves each reduced shard in its
    owner's g8 window only, and AdamW pass 2 reads every tile's codes from the owners'
    windows — a tile [e, e + L) cut at the shard bounds, piece k from rank e_k // S —
    walking the items from the first one at or after rank * S (kernels.cu adam_issue /
    TileCursor rotation).  Replayed here: windows exchanged with gloo, the pulled view
    assembled tile by tile, compared with the N-rank oracle's reduced codes."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import ctypes as C
        import paper_2310_18313_b200._binding as B
        from oracle import pipeline as P

        arr = (C.c_int64 * len(NUMELS))(*NUMELS)
        h = C.c_void_p()
        assert B.lib.fp8lm_plan_create(len(NUMELS), arr, B.MODE_P2P, world, rank, C.byref(h)) == 0
        offs = [B.lib.fp8lm_plan_offset(h, t) for t in range(len(NUMELS))]
        S = B.lib.fp8lm_plan_shard_bytes(h)
        g8_bytes = B.lib.fp8lm_plan_g8_bytes(h)
        assert S % 64 == 0 and g8_bytes == world * S
        g = _local_grads(rank, 1)
        s_loc = torch.tensor([P.local_scale(*P.amax(x), F32(1.0)) for x in g], dtype=torch.float32)
        dist.all_reduce(s_loc, op=dist.ReduceOp.MIN)
        s_g = [P.global_scale([F32(v)])[0] for v in s_loc.numpy()]
        send = torch.zeros(g8_bytes, dtype=torch.uint8)
        for t, x in enumerate(g):
            send[offs[t]: offs[t] + NUMELS[t]] = torch.from_numpy(P.quantize(x, s_g[t]).astype(np.uint8))
        sends = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(sends, send)                  # the peers' send windows
        window = torch.zeros(g8_bytes, dtype=torch.uint8)   # this rank's g8 window
        lo, hi = rank * S, (rank + 1) * S
        for t in range(len(NUMELS)):
            a, b = max(lo, offs[t]), min(hi, offs[t] + NUMELS[t])
            if a < b:
                c = P.requantize(P.rank_order_sum([sends[r][a:b].numpy() for r in range(world)]))
                window[a:b] = torch.from_numpy(c.astype(np.uint8))
        windows = [torch.empty_like(window) for _ in range(world)]
        dist.all_gather(windows, window)              # what pass 2 can read over NVLink
        # pass 2: items of <= 16384 elements per tensor, tiles of 4096, pieces cut at
        # multiples of S; rotation starts at the first item at or after rank * S
        items = []
        for t in range(len(NUMELS)):
            for p0 in range(0, NUMELS[t], 16384):
                items.append((offs[t] + p0, min(16384, NUMELS[t] - p0)))
        rot = next((i for i, (pos, _) in enumerate(items) if pos >= lo), 0)
        pulled = torch.zeros(g8_bytes, dtype=torch.uint8)
        for i in range(len(items)):
            pos, n = items[(i + rot) % len(items)]
            for e0 in range(pos, pos + n, 4096):
                L = min(4096, pos + n - e0)
                Lr = (L + 15) // 16 * 16
                a = e0
                while a < e0 + Lr:
                    owner = a // S
                    m = min(e0 + Lr - a, (owner + 1) * S - a)
                    assert m % 16 == 0 and a % 16 == 0
                    pulled[a:a + m] = windows[owner][a:a + m]
                    a += m
        q.put((rank, [pulled[offs[t]: offs[t] + NUMELS[t]].numpy().copy() for t in range(len(NUMELS))]))
        B.lib.fp8lm_plan_destroy(h)
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_p2p_pull_allgather_matches_n_rank_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pull_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]
    from oracle import pipeline as P
    grads = [_local_grads(r, 1) for r in range(world)]
    for t in range(len(NUMELS)):
        ref = P.allreduce_tensor([grads[r][t] for r in range(world)], F32(1.0))
        for r in range(world):
            assert np.array_equal(got[r][t], ref["codes"]), (r, t)
