"""x-slab domain decomposition across GPUs (one process per GPU, NCCL).

The paper's distributed scheme (``PAPER.md:1585-1625``; not implemented by the
reference, ``SPEC.md:8,424``): non-overlapping subdomains of whole cell planes
along axis 0, face projections of the slab-boundary cells exchanged with the
two ring neighbours once per realisation step, boundary Riemann problems
solved redundantly on both sides, and one global reduction of the admissible
step (here: max of lambda, which gives dt_adm bitwise).

Per step and rank:  rerun (device-conditional)  ->  { halo exchange of the
trace parity the sweep will read  ||  sweep of the interior planes }  ->
sweep of the two boundary planes  ->  all-reduce MAX of {lambda bits,
INT64_MAX - error key}  ->  time control.  The exchange runs on NCCL's stream
while the interior planes (which read no halo slot and produce no record a
neighbour receives) run on the compute stream: the paper's transfer hiding
(``PAPER.md:1591-1597``).

Layout of the trace records (``include/aderdg_b200.h``): ``[2d faces][slots][REC]``
with ``slots = (planes_local + 2) * plane_cells``; slot plane 0 and
``planes_local + 1`` are the halos.  Face 0 = low-x side record of a cell,
face 1 = high-x side record, so every message is one contiguous slice.
"""

import numpy as np

from . import _lib
from .errors import ConfigurationError


def slab_partition(K, world, rank):
    """Planes of rank's slab: the first K % world ranks get one extra plane
    (mirrors adg_create in csrc/aderdg_capi.cu)."""
    if world < 1 or not 0 <= rank < world or world > K:
        raise ConfigurationError(f"bad slab decomposition: K={K} world={world} rank={rank}")
    base, extra = divmod(K, world)
    planes = base + (1 if rank < extra else 0)
    plane0 = rank * base + min(rank, extra)
    return plane0, planes


class HaloExchange:
    """Ring exchange of slab-boundary face records and the step reduction.

    Works on any torch tensors (CUDA with NCCL, CPU with gloo for tests)."""

    def __init__(self, planes_local, plane_cells, rank, world, group=None, staged=False):
        self.Pl, self.plane = planes_local, plane_cells
        self.rank, self.world, self.group = rank, world, group
        self.prev = (rank - 1) % world
        self.next = (rank + 1) % world
        # staged: device tensors go through host copies (gloo transport; used to
        # test the multi-slab device path with several ranks on one GPU)
        self.staged = staged
        self.force = False          # exchange even at world = 1 (self send/recv; halo test mode)

    def views(self, tr):
        """tr: tensor (2d, slots, REC).  Returns (send_to_prev, recv_from_prev,
        send_to_next, recv_from_next)."""
        P, n = self.Pl, self.plane
        send_prev = tr[0, n:2 * n]                    # low-x records of my first plane
        recv_next = tr[0, (P + 1) * n:(P + 2) * n]    # -> halo-hi: next rank's first-plane low-x
        send_next = tr[1, P * n:(P + 1) * n]          # high-x records of my last plane
        recv_prev = tr[1, 0:n]                        # -> halo-lo: prev rank's last-plane high-x
        return send_prev, recv_prev, send_next, recv_next

    def exchange(self, tr):
        self.wait(self.start(tr))

    def active(self):
        return self.world > 1 or self.force

    def start(self, tr):
        """Issue the ring exchange of ``tr``'s boundary records and return the
        pending works.  With NCCL the transfers run on NCCL's stream, ordered
        after the work already queued on the current stream; the caller keeps
        queueing independent kernels (the interior planes) and calls wait()
        before the halo readers.  The gloo-staged transport completes here."""
        import torch.distributed as dist
        if not self.active():
            return []
        send_prev, recv_prev, send_next, recv_next = self.views(tr)
        if self.staged:
            dev_recv = (recv_prev, recv_next)
            send_prev, send_next = send_prev.cpu(), send_next.cpu()
            recv_prev, recv_next = recv_prev.cpu(), recv_next.cpu()
        # order matters when prev == next (world 2): messages between one pair
        # are matched in issue order, so every rank sends "to next" first.
        ops = [dist.P2POp(dist.isend, send_next, self.next, self.group),
               dist.P2POp(dist.irecv, recv_prev, self.prev, self.group),
               dist.P2POp(dist.isend, send_prev, self.prev, self.group),
               dist.P2POp(dist.irecv, recv_next, self.next, self.group)]
        works = dist.batch_isend_irecv(ops)
        if self.staged:
            for r in works:
                r.wait()
            dev_recv[0].copy_(recv_prev)
            dev_recv[1].copy_(recv_next)
            return []
        return works

    @staticmethod
    def wait(works):
        """NCCL: the current stream waits for the transfers (no host block)."""
        for r in works:
            r.wait()

    def reduce(self, red):
        """red: int64[2] = {lambda bits, INT64_MAX - error key}; MAX over ranks."""
        import torch.distributed as dist
        if self.world == 1:
            return
        if self.staged:
            host = red.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.MAX, group=self.group)
            red.copy_(host)
            return
        dist.all_reduce(red, op=dist.ReduceOp.MAX, group=self.group)


class SlabDriver:
    """Fused driver over an x-slab of the periodic grid on this process's GPU.

    ``Q_global`` (reference layout) is sliced to the local cells; results are
    gathered on demand with ``local_state()``.  All ranks must call every
    method collectively.
    """

    def __init__(self, Q_global, d, L, p, rank, world, device, cfl=0.9, c_dt=0.99,
                 averaging="strict", forced_dt=None, inject_rerun=False,
                 spike_step=None, spike_factor=3.0, group=None, staged=False, halo_mode=0,
                 mode="fused", overlap=True, debug_checks=False):
        import torch
        from .basis import make_basis
        from .solver import upload_operators
        self.torch = torch
        self.d, self.L, self.p = d, L, p
        self.rank, self.world = rank, world
        self.dev = torch.device("cuda", device)
        cfg = _lib.AdgConfig()
        cfg.d, cfg.p, cfg.L = d, p, L
        cfg.cfl, cfg.c_dt = float(cfl), float(c_dt)
        cfg.creeping = 1 if averaging == "creeping" else 0
        cfg.forced_dt = float("nan") if forced_dt is None else float(forced_dt)
        cfg.inject_rerun = 1 if inject_rerun else 0
        cfg.spike_step = -1 if spike_step is None else int(spike_step)
        cfg.spike_factor = float(spike_factor)
        cfg.device, cfg.rank, cfg.world = int(device), int(rank), int(world)
        cfg.halo_mode = int(halo_mode)
        cfg.driver_mode = 1 if mode == "straightforward" else 0
        self.mode = mode
        self.overlap = bool(overlap)
        self.handle = _lib.Handle(cfg, debug=debug_checks)
        self._ops = upload_operators(self.handle, make_basis(p))
        self.lay = lay = self.handle.layout()
        self.stream = torch.cuda.current_stream(self.dev)
        self.handle.call("adg_set_stream", self.stream.cuda_stream)
        K = 3 ** L
        plane0, planes = slab_partition(K, world, rank)
        assert planes == lay.planes_local and plane0 * lay.plane_cells == lay.cell_offset
        self.cell_offset, self.n_local = lay.cell_offset, lay.n_cells_local
        self.halo = HaloExchange(lay.planes_local, lay.plane_cells, rank, world, group, staged)
        self.halo.force = bool(halo_mode)
        slots = (lay.planes_local + 2) * lay.plane_cells
        shape = (lay.faces_per_cell, slots, lay.record_doubles)
        self.tr = []
        for which in (_lib.ADG_BUF_TRACE0, _lib.ADG_BUF_TRACE1):
            ptr, nbytes = self.handle.buffer(which)
            assert nbytes == 8 * int(np.prod(shape))
            self.tr.append(torch.as_tensor(_lib.DeviceArray(ptr, shape, "<f8", self.dev), device=self.dev))
        rptr, _ = self.handle.buffer(_lib.ADG_BUF_REDUCE)
        self.red = torch.as_tensor(_lib.DeviceArray(rptr, (2,), "<i8", self.dev), device=self.dev)
        self.primed = False
        self.load(Q_global, reset=False)

    def load(self, Q_global, reset=True):
        """(Re)start from global initial data: upload the local slab and seed the
        time control (Driver._seed_time_control) with the global reduction."""
        if reset:
            self.handle.call("adg_reset")
            self.primed = False
        Ql = np.ascontiguousarray(Q_global[self.cell_offset:self.cell_offset + self.n_local],
                                  dtype=np.float64)
        self.handle.call("adg_load_state", _lib.dptr(Ql), Ql.size)
        self.handle.call("adg_phase_seed")
        self.halo.reduce(self.red)
        self.handle.call("adg_phase_seed_finish")
        self.handle.call("adg_sync")

    def enqueue_step(self):
        """Queue one realisation step without host synchronisation."""
        h = self.handle
        if not self.primed and self.mode != "straightforward":
            h.call("adg_phase_sweep")          # priming sweep (no traces read)
            self.halo.reduce(self.red)
            h.call("adg_phase_finish")
            self.primed = True
        h.call("adg_phase_rerun")
        tr = self.tr[h.lib.adg_trace_parity(h.h)]
        if self.overlap and self.halo.active():
            # the interior planes hide the face-record transfer
            pending = self.halo.start(tr)
            h.call("adg_phase_sweep_part", _lib.ADG_PART_INTERIOR)
            self.halo.wait(pending)
            h.call("adg_phase_sweep_part", _lib.ADG_PART_BOUNDARY)
        else:
            self.halo.exchange(tr)
            h.call("adg_phase_sweep")
        self.halo.reduce(self.red)
        h.call("adg_phase_finish")

    def run(self, steps):
        for _ in range(steps):
            self.enqueue_step()
        self.handle.call("adg_sync")
        return self.handle.lib.adg_step_count(self.handle.h)

    def init_native_comm(self, group=None):
        """Open the library's own NCCL communicator over the slab ranks
        (adg_nccl_init): rank 0 draws the unique id, torch.distributed broadcasts it.
        Afterwards run_timed() enqueues whole steps from C."""
        import ctypes
        uid = (ctypes.c_ubyte * 128)()
        ok = True
        if self.rank == 0:
            ok = self.handle.lib.adg_nccl_unique_id(uid) == 0
        if self.world > 1:
            # rank 0's verdict travels with the id, so every rank takes the same branch
            import torch.distributed as dist
            box = [bytes(uid) if ok else b""]
            dist.broadcast_object_list(box, src=0, group=group)
            ok = len(box[0]) == 128
            if ok:
                uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        if not ok:
            raise RuntimeError("adg_nccl_unique_id failed (libnccl.so.2 not loadable)")
        self.handle.call("adg_nccl_init", uid, self.rank, self.world)
        self.native_comm = True

    def run_timed(self, steps, flags=_lib.ADG_TIMED_KERNEL_EVENTS):
        """`steps` overlapped slab steps enqueued from C (adg_run_timed_mgpu_ex);
        returns (segment ms, sweep-kernel ms) measured on the launch stream (the
        kernel ms only with flags & ADG_TIMED_KERNEL_EVENTS, else 0)."""
        import ctypes
        out = (ctypes.c_double * 2)()
        self.handle.call("adg_run_timed_mgpu_ex", int(steps), int(flags), out)
        return out[0], out[1]

    def local_state(self):
        lay = self.lay
        Q = np.empty(lay.state_doubles)
        self.handle.call("adg_store_state", _lib.dptr(Q), Q.size)
        n = self.p + 1
        return Q.reshape((lay.n_cells_local,) + (n,) * self.d + (self.d + 2,))

    def time_control(self):
        return self.handle.time_control()

    def close(self):
        self.handle.close()


class SlabGroup:
    """N x-slab handles of one grid on N GPUs of this process (the reference's
    ``Driver(..., parallel=True, n_workers=N)`` seam, ``src/scheduler.py:92-95,126-130``).

    One NCCL clique over the handles (``adg_group_init`` -> ``ncclCommInitAll``);
    every call drives all slabs from one host thread per GPU inside the library
    (``adg_group_seed`` / ``adg_group_run``) with the per-rank step sequence of the
    one-process-per-GPU path: halo exchange hidden behind the interior planes, MAX
    all-reduce of the step reduction.  Max is exact, so the state equals the
    single-GPU state bitwise.
    """

    def __init__(self, make_cfg, devices, basis, d, p):
        import ctypes
        from .solver import upload_operators
        self.world = len(devices)
        self.d, self.p = d, p
        self.handles, self._ops = [], []
        for r, dev in enumerate(devices):
            cfg = make_cfg()
            cfg.rank, cfg.world, cfg.device = r, self.world, int(dev)
            h = _lib.Handle(cfg)
            self.handles.append(h)
            self._ops.append(upload_operators(h, basis))
        self.lays = [h.layout() for h in self.handles]
        self._arr = (ctypes.c_void_p * self.world)(*[h.h.value for h in self.handles])
        self.lib = self.handles[0].lib
        self._check(self.lib.adg_group_init(self._arr, self.world), "adg_group_init")

    @property
    def lead(self):
        return self.handles[0]

    def _check(self, st, what):
        self.handles[0].check(st, what)

    def load(self, Q_global):
        for h, lay in zip(self.handles, self.lays):
            Ql = np.ascontiguousarray(Q_global[lay.cell_offset:lay.cell_offset + lay.n_cells_local],
                                      dtype=np.float64)
            h.call("adg_load_state", _lib.dptr(Ql), Ql.size)

    def seed(self):
        self._check(self.lib.adg_group_seed(self._arr, self.world), "adg_group_seed")

    def run(self, steps, recs):
        """Status of ``adg_group_run`` (the caller maps it to an exception)."""
        return self.lib.adg_group_run(self._arr, self.world, int(steps), recs)

    def store(self, Q_global):
        for h, lay in zip(self.handles, self.lays):
            out = Q_global[lay.cell_offset:lay.cell_offset + lay.n_cells_local]
            if not out.flags.c_contiguous:
                raise ConfigurationError("grid.Q must stay C-contiguous")
            h.call("adg_store_state", _lib.dptr(out), out.size)

    def picard_histogram(self, bins=32):
        return sum(h.picard_histogram(bins) for h in self.handles)

    def close(self):
        for h in self.handles:
            h.close()
