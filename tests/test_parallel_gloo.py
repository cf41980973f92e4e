"""x-slab decomposition host logic on CPU with world_size 2 (gloo): ring halo
exchange of face records, the MAX reduction of {lambda bits, error key}, and
the slab partition (mirrors csrc/aderdg_capi.cu adg_create)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_08682_b200.parallel import HaloExchange, slab_partition


def test_slab_partition_covers_grid():
    for K in (3, 9, 27, 81):
        for world in (1, 2, 3, 4, 8):
            if world > K:
                continue
            spans = [slab_partition(K, world, r) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == K
            for (a, n), (b, _) in zip(spans, spans[1:]):
                assert a + n == b
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, K, plane, rec, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plane0, P = slab_partition(K, world, rank)
    slots = (P + 2) * plane
    # record value encodes (global plane, face, cell-in-plane, element)
    tr = torch.full((4, slots, rec), -1.0, dtype=torch.float64)
    for lp in range(P):
        g = plane0 + lp
        for f in range(4):
            for c in range(plane):
                tr[f, (lp + 1) * plane + c] = 1e6 * g + 1e4 * f + 10 * c + torch.arange(rec)
    hx = HaloExchange(P, plane, rank, world)
    hx.exchange(tr)
    lo = tr[1, 0:plane].numpy().copy()
    hi = tr[0, (P + 1) * plane:(P + 2) * plane].numpy().copy()
    red = torch.tensor([rank * 10, 0x7FFFFFFFFFFFFFFF - (100 + rank)], dtype=torch.int64)
    hx.reduce(red)
    result_q.put((rank, plane0, P, lo, hi, red.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_and_reduction(world):
    K, plane, rec = 9, 4, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, plane, rec, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, plane0, P, lo, hi, red in res:
        g_lo = (plane0 - 1) % K          # periodic low neighbour plane: its high-x records (face 1)
        g_hi = (plane0 + P) % K          # high neighbour plane: its low-x records (face 0)
        for c in range(plane):
            assert np.array_equal(lo[c], 1e6 * g_lo + 1e4 * 1 + 10 * c + np.arange(rec))
            assert np.array_equal(hi[c], 1e6 * g_hi + 1e4 * 0 + 10 * c + np.arange(rec))
        assert red[0] == (world - 1) * 10
        assert 0x7FFFFFFFFFFFFFFF - red[1] == 100     # min error key wins
