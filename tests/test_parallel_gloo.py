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


class _FakeLib:
    """Stands in for the C library: rank 0's unique-id call succeeds or fails."""

    def __init__(self, ok):
        self.ok = ok

    def adg_nccl_unique_id(self, buf):
        if not self.ok:
            return 4
        for i in range(128):
            buf[i] = (7 * i + 3) % 256
        return 0


class _FakeHandle:
    def __init__(self, ok):
        self.lib = _FakeLib(ok)
        self.calls = []

    def call(self, name, *args):
        self.calls.append((name, bytes(args[0]), args[1], args[2]))


def _native_worker(rank, world, port, ok, result_q):
    from paper_1801_08682_b200.parallel import SlabDriver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    drv = object.__new__(SlabDriver)          # host logic only: no device handle
    drv.rank, drv.world = rank, world
    drv.handle = _FakeHandle(ok if rank == 0 else True)
    try:
        drv.init_native_comm()
        result_q.put((rank, "ok", drv.handle.calls))
    except RuntimeError:
        result_q.put((rank, "raised", drv.handle.calls))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ok", [True, False])
def test_native_comm_init_is_collective(ok):
    """SlabDriver.init_native_comm: rank 0's unique id (or its failure) reaches every
    rank, so all ranks open the library communicator with the same id or all fall
    back together (no rank left waiting in ncclCommInitRank)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_native_worker, args=(r, world, port, ok, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if ok:
        assert all(r[1] == "ok" for r in res)
        ids = {r[2][0][1] for r in res}
        assert len(ids) == 1 and len(next(iter(ids))) == 128
        assert [r[2][0][2] for r in res] == [0, 1] and all(r[2][0][3] == world for r in res)
    else:
        assert all(r[1] == "raised" and r[2] == [] for r in res)
