"""A/B numerics of a kernel experiment: the same seeded BASELINE-type state through the
product library and an A/B build (tools/build_ab.sh), compared after every step.

    python tools/ab_parity.py tools/ab/lib_<name>.so [d L p steps]

Each library runs in its own process (one CUDA library per process)."""
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def child(lib, d, L, p, steps, out):
    from paper_1801_08682_b200 import (Driver, EulerSystem, Kernels, TimeControl, _lib, build_grid, make_basis,
                                       scenarios)
    if lib != "product":
        _lib._lib = _lib.load_library(lib)
    Q0 = scenarios.build("bump", d, L, p)
    grid = build_grid(d, L, p, d + 2)
    grid.Q[...] = Q0
    drv = Driver(grid, Kernels(EulerSystem(d), make_basis(p), grid, None), TimeControl(), "fused", device=0,
                 host_sync="step")
    qs = []
    for _ in range(steps):
        drv.step()
        qs.append(np.array(grid.Q))
    np.savez(out, Q=np.stack(qs), hist=np.array(sorted(drv.picard_histogram().items())))


def main():
    if sys.argv[1] == "--child":
        lib, d, L, p, steps, out = sys.argv[2], *map(int, sys.argv[3:7]), sys.argv[7]
        return child(lib, d, L, p, steps, out)
    lib = sys.argv[1]
    d, L, p, steps = (int(x) for x in (sys.argv[2:6] if len(sys.argv) > 5 else (3, 1, 5, 4)))
    outs = []
    for which in ("product", lib):
        out = f"/tmp/ab_parity_{os.getpid()}_{len(outs)}.npz"
        subprocess.check_call([sys.executable, __file__, "--child", which, str(d), str(L), str(p), str(steps), out])
        outs.append(np.load(out))
        os.unlink(out)
    a, b = outs
    for s in range(steps):
        err = np.abs(a["Q"][s] - b["Q"][s]).max() / np.abs(a["Q"][s]).max()
        print(f"step {s + 1}: rel L-inf product vs {os.path.basename(lib)} {err:.3e}")
    print("picard histogram product", a["hist"].tolist())
    print("picard histogram variant", b["hist"].tolist())


if __name__ == "__main__":
    main()
