"""NCCL halo path on ONE GPU: a single-rank NCCL process group with the halo
slots forced on (halo_mode=1), so every step sends the slab-boundary face
records to itself with batched NCCL send/recv and all-reduces the
{lambda, error} pair through NCCL.  The result must equal the periodic
in-place run bitwise (this is the code path of the x-slab decomposition)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(port, out, inject, overlap, mode):
    import torch.distributed as dist
    from paper_1801_08682_b200 import scenarios
    from paper_1801_08682_b200.parallel import SlabDriver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    Q0 = scenarios.build("bump", 3, 2, 3, seed=5, noise=1e-2)
    a = SlabDriver(Q0, 3, 2, 3, 0, 1, 0, inject_rerun=inject, halo_mode=1, overlap=overlap,
                   mode=mode)
    a.run(4)
    qa = a.local_state()
    b = SlabDriver(Q0, 3, 2, 3, 0, 1, 0, inject_rerun=inject, mode=mode)
    b.run(4)
    qb = b.local_state()
    np.save(out, np.stack([qa, qb]))
    a.close()
    b.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("inject,overlap,mode", [(False, False, "fused"), (True, False, "fused"),
                                                 (False, True, "fused"), (True, True, "fused"),
                                                 (False, True, "straightforward")])
def test_nccl_self_halo_equals_periodic(cuda_ok, tmp_path, inject, overlap, mode):
    ctx = mp.get_context("spawn")
    out = str(tmp_path / "q.npy")
    p = ctx.Process(target=_run, args=(_port(), out, inject, overlap, mode))
    p.start()
    p.join(timeout=300)
    assert p.exitcode == 0
    qa, qb = np.load(out)
    assert np.array_equal(qa, qb)


def _run_native(port, out):
    import torch.distributed as dist
    from paper_1801_08682_b200 import scenarios
    from paper_1801_08682_b200.parallel import SlabDriver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    Q0 = scenarios.build("bump", 3, 2, 3, seed=5, noise=1e-2)
    a = SlabDriver(Q0, 3, 2, 3, 0, 1, 0, inject_rerun=True, halo_mode=1)
    a.init_native_comm()
    a.run(1)                      # priming step through the Python phase loop
    a.run_timed(2, flags=0)       # then whole steps enqueued from C over the library's comm
    a.run_timed(2)                # (without / with the per-launch kernel events)
    qa = a.local_state()
    b = SlabDriver(Q0, 3, 2, 3, 0, 1, 0, inject_rerun=True)
    b.run(5)
    qb = b.local_state()
    np.save(out, np.stack([qa, qb]))
    a.close()
    b.close()
    dist.destroy_process_group()


def test_native_nccl_steps_equal_periodic(cuda_ok, tmp_path):
    """adg_run_timed_mgpu: grouped ncclSend/ncclRecv of the boundary records on the
    library's own communicator (self exchange at world 1) + overlapped planes."""
    ctx = mp.get_context("spawn")
    out = str(tmp_path / "q.npy")
    p = ctx.Process(target=_run_native, args=(_port(), out))
    p.start()
    p.join(timeout=300)
    assert p.exitcode == 0
    qa, qb = np.load(out)
    assert np.array_equal(qa, qb)
