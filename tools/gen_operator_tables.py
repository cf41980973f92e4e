"""Generate paper_1801_08682_b200/data/operators.npz from the REFERENCE itself.

Runs only in the build container (``/root/reference`` present):

    python tools/gen_operator_tables.py

For p = 0..9 it stores the reference's 1-D collocation operators
(``make_basis``, src/basis.py:91-122: nodes, weights, diff, integ, left, right),
the subcell limiter's average matrix and least-squares lift
(``SubcellLimiter.__init__``, src/limiter.py:87-108: P, R) and the Lagrange
evaluation matrix at the 6-point Gauss rule used by the convergence study's
L2 error (src/cli.py:256-275: E6, with the rule's nodes / weights x6 / w6).
The product package only reads this table; tests/test_basis.py checks it
bitwise against the reference whenever the reference is importable.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1801_08682_b200", "data", "operators.npz")


def tables():
    sys.path.insert(0, REF)
    from aderdg.basis import lagrange_eval, make_basis
    from aderdg.limiter import SubcellLimiter
    from aderdg.mesh import build_grid
    from aderdg.pde import EulerSystem
    out = {}
    b6 = make_basis(5)
    out["x6"], out["w6"] = b6.nodes, b6.weights
    for p in range(10):
        b = make_basis(p)
        for f in ("nodes", "weights", "diff", "integ", "left", "right"):
            out[f"p{p}_{f}"] = np.asarray(getattr(b, f), dtype=np.float64)
        grid = build_grid(2, 1, p, 4, budget_bytes=1 << 40)
        lim = SubcellLimiter(EulerSystem(2), b, grid)
        out[f"p{p}_P"], out[f"p{p}_R"] = lim.P, lim.R
        out[f"p{p}_E6"] = lagrange_eval(b.nodes, b6.nodes)
    return out


if __name__ == "__main__":
    t = tables()
    np.savez(OUT, **t)
    print(f"wrote {len(t)} arrays to {OUT}")
