"""One small run of a product kernel path, for compute-sanitizer
(tools/sanitize.sh runs every case under memcheck / racecheck / synccheck / initcheck).

    python tools/sanitize_case.py <case>

Cases cover every default kernel instantiation and launch structure:
p3 (sweep_kernel_p3, graph steps + conditional rerun, inject_rerun), p5
(sweep_kernel_p5), p7 (sweep_kernel_p7), p9 (sweep_kernel_p9), gen2d (generic 2D kernel), p4 (generic 3D kernel), sf (straightforward
passes), adv (advection plug-in), lim (subcell limiter: detect / apply / lambda),
host (adg_step_host chunked H2D / sweep / D2H pipeline), stream (adg_run without graphs).
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_1801_08682_b200 import (AdvectionSystem, Driver, EulerSystem, Kernels,  # noqa: E402
                                   SubcellLimiter, TimeControl, _lib, build_grid, make_basis,
                                   scenarios)


def drive(d, L, p, steps, mode="fused", system=None, limiter=False, scen="bump", **kw):
    system = system or EulerSystem(d)
    if scen == "bump":
        Q0 = scenarios.build("bump", d, L, p, seed=3, noise=1e-2)
    else:
        Q0 = scenarios.build(scen, d, L, p)
    boundary = "outflow" if scen == "sod" else "periodic"
    grid = build_grid(d, L, p, system.m, boundary=boundary)
    grid.Q[...] = Q0 if system.m == Q0.shape[-1] else Q0[..., :1]
    basis = make_basis(p)
    lim = SubcellLimiter(system, basis, grid) if limiter else None
    drv = Driver(grid, Kernels(system, basis, grid, None), TimeControl(), mode, limiter=lim,
                 host_sync="run", **kw)
    return drv, steps


def main(case):
    if case == "p3":
        drv, n = drive(3, 1, 3, 4, inject_rerun=True)
    elif case == "p5":
        drv, n = drive(3, 1, 5, 3)
    elif case == "p7":
        drv, n = drive(3, 1, 7, 2)
    elif case == "p9":
        drv, n = drive(3, 1, 9, 2)
    elif case == "gen2d":
        drv, n = drive(2, 2, 3, 4, inject_rerun=True)
    elif case == "p4":
        drv, n = drive(3, 1, 4, 3)
    elif case == "sf":
        drv, n = drive(3, 1, 3, 3, mode="straightforward")
    elif case == "adv":
        drv, n = drive(3, 1, 3, 3, system=AdvectionSystem(3, (1.0, 0.5, 0.25)), scen="gauss")
    elif case == "lim":
        drv, n = drive(2, 2, 2, 6, mode="straightforward", limiter=True, scen="sod")
    elif case == "stream":
        drv, n = drive(3, 1, 3, 4, inject_rerun=True)
        drv.handle.call("adg_set_option", _lib.ADG_OPT_GRAPH, 0)
    elif case == "host":
        drv, _ = drive(3, 2, 3, 0)
        h = drv.handle
        Q = np.ascontiguousarray(drv.grid.Q)
        ptr = _lib.dptr(Q)
        for _ in range(4):
            h.call("adg_step_host", ptr, ptr, None)
        drv.close()
        print(f"{case}: ok")
        return
    else:
        raise SystemExit(f"unknown case {case}")
    drv.run(steps=n)
    assert np.all(np.isfinite(drv.grid.Q))
    drv.close()
    print(f"{case}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
