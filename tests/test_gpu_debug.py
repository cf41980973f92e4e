"""Run-time correctness checks of the kernels (the debug library).

``libaderdg_b200_debug.so`` is the product sources built with ADG_DEBUG_CHECKS
(paper_1801_08682_b200/build.py).  On this GPU pool compute-sanitizer is closed, so
the hazards its tools look for are checked by the kernels themselves:

* stale data (racecheck across CTAs / sweeps): every face record carries the sweep
  that wrote it and every read is checked against the sweep that must have written
  it -- the reference's per-face sweep stamps (mesh.py:43-57, kernels.py:158-170,
  196-200); slot and cell indices are bounds-checked (memcheck);
* uninitialised shared memory (initcheck): dynamic shared memory is filled with NaN
  at kernel entry, so a read of an unwritten word poisons the result;
* intra-CTA races (racecheck / synccheck): every CTA barrier jitters its warps with a
  random sleep first, and the cells go to the CTAs in reverse order, so a missing
  barrier or a cross-CTA dependency changes the result.

Bar: the debug build produces the release build's state bitwise on every default
kernel and launch structure, and the stamp check fires on a corrupted record and on a
skipped halo exchange.
"""

import ctypes

import numpy as np
import pytest
import torch

from paper_1801_08682_b200 import (AdvectionSystem, DeviceError, Driver, EulerSystem, Kernels,
                                   SubcellLimiter, TimeControl, _lib, build_grid, make_basis,
                                   scenarios)

pytestmark = pytest.mark.gpu


def _run(d, L, p, steps, mode="fused", debug=False, system=None, scen="bump", limiter=False, **kw):
    system = system or EulerSystem(d)
    if scen == "bump":
        Q0 = scenarios.build("bump", d, L, p, seed=9, noise=1e-2)
    else:
        Q0 = scenarios.build(scen, d, L, p)
    grid = build_grid(d, L, p, system.m, boundary="outflow" if scen == "sod" else "periodic")
    grid.Q[...] = Q0
    basis = make_basis(p)
    lim = SubcellLimiter(system, basis, grid) if limiter else None
    drv = Driver(grid, Kernels(system, basis, grid, None), TimeControl(), mode, limiter=lim,
                 host_sync="run", debug_checks=debug, **kw)
    drv.run(steps=steps)
    recs = [(r["step"], r["T"], r["dt_new"], r["reruns"]) for r in drv.step_records]
    drv.close()
    return np.array(grid.Q), recs


CASES = [
    dict(d=3, L=2, p=3, steps=5, inject_rerun=True),           # sweep_kernel_p3, graph + rerun nodes
    dict(d=3, L=1, p=5, steps=3),                              # p=5 kernel
    dict(d=3, L=1, p=7, steps=2),                              # p=7 kernel (TMEM + smem state, DMMA tiles)
    dict(d=3, L=1, p=6, steps=2),                              # sweep_kernel_ho, TMEM time line
    dict(d=3, L=1, p=9, steps=2),                              # p=9 kernel (TMEM + smem state, line engine)
    dict(d=2, L=2, p=3, steps=5, spike_step=3),                # 2D p=3 kernel (fused time control) + speed spike
    dict(d=2, L=2, p=3, steps=4, inject_rerun=True),           # 2D p=3 kernel, rerun passes
    dict(d=2, L=2, p=2, steps=4),                              # generic 2D kernel
    dict(d=3, L=1, p=4, steps=3),                              # generic 3D kernel
    dict(d=3, L=2, p=3, steps=4, mode="straightforward"),      # straightforward passes
    dict(d=3, L=1, p=3, steps=3, scen="gauss"),                # advection plug-in
    dict(d=2, L=2, p=2, steps=8, mode="straightforward", limiter=True, scen="sod"),   # limiter, outflow
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_debug_build_equals_release_bitwise(cuda_ok, case):
    case = dict(case)
    if case.get("scen") == "gauss":
        case["system"] = AdvectionSystem(case["d"], (1.0, 0.5, 0.25))
    qa, ra = _run(**case)
    qb, rb = _run(debug=True, **case)
    assert np.array_equal(qa, qb)
    assert ra == rb


def test_debug_build_host_step_pipeline(cuda_ok):
    """adg_step_host (chunked H2D / sweep / D2H) under the debug checks."""
    out = []
    for debug in (False, True):
        Q0 = scenarios.build("bump", 3, 2, 3, seed=9, noise=1e-2)
        grid = build_grid(3, 2, 3, 5)
        grid.Q[...] = Q0
        drv = Driver(grid, Kernels(EulerSystem(3), make_basis(3), grid, None), TimeControl(), "fused",
                     host_sync="manual", debug_checks=debug)
        Q = np.ascontiguousarray(Q0)
        ptr = _lib.dptr(Q)
        for _ in range(4):
            drv.handle.call("adg_step_host", ptr, ptr, None)
        out.append(Q.copy())
        drv.close()
    assert np.array_equal(out[0], out[1])


def test_stale_record_is_detected(cuda_ok):
    """A face record whose stamp is not the previous sweep's is refused."""
    Q0 = scenarios.build("bump", 3, 1, 3, seed=9, noise=1e-2)
    grid = build_grid(3, 1, 3, 5)
    grid.Q[...] = Q0
    drv = Driver(grid, Kernels(EulerSystem(3), make_basis(3), grid, None), TimeControl(), "fused",
                 host_sync="manual", debug_checks=True)
    drv.step()                                   # priming + step 1
    h = drv.handle
    lay = h.layout()
    par = h.lib.adg_trace_parity(h.h)
    ptr, nbytes = h.buffer(_lib.ADG_BUF_TRACE0 + par)
    rec = lay.record_doubles
    slots = nbytes // 8 // (lay.faces_per_cell * rec)
    cell = 13
    own_slot = cell + lay.plane_cells
    word = (2 * slots + own_slot) * rec + rec - 1     # face 2 (axis 1 low side) stamp of cell 13
    bad = ctypes.c_double(12345.0)
    torch.cuda.init()
    t = torch.as_tensor(_lib.DeviceArray(ptr, (nbytes // 8,), "<f8", torch.device("cuda", 0)),
                        device="cuda:0")
    assert t[word].item() in (1.0, 2.0, 3.0, 4.0)   # a valid stamp (2s-1 / 2s)
    t[word] = bad.value
    torch.cuda.synchronize()
    with pytest.raises(DeviceError) as e:
        drv.step()
    # cell 13 reads it as its own record, cell 10 (its low neighbour along axis 1) as
    # the neighbour's; the smallest reader is reported
    assert "stale face record read by cell 10 at step 2" in str(e.value)
    drv.close()


def test_skipped_halo_exchange_is_detected(cuda_ok):
    """x-slab halos that were never exchanged carry no valid stamp."""
    from paper_1801_08682_b200.parallel import SlabDriver
    Q0 = scenarios.build("bump", 3, 1, 3, seed=9, noise=1e-2)
    drv = SlabDriver(Q0, 3, 1, 3, 0, 1, 0, halo_mode=1, debug_checks=True)
    h = drv.handle
    with pytest.raises(DeviceError) as e:
        h.call("adg_phase_sweep")                # priming (writes records, reads none)
        h.call("adg_phase_finish")
        h.call("adg_phase_rerun")
        h.call("adg_phase_sweep")                # reads the halo slots: no exchange happened
        h.call("adg_phase_finish")
        h.call("adg_sync")
    assert "stale face record" in str(e.value)
    drv.close()
