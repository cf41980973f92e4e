"""Algorithmic work and traffic of the fused ADER-DG sweep.

Counting convention: FMA = 2 flops; add/mul/div/sqrt/abs/max = 1.
``K`` = Picard iterations of a predict under the reference criterion
(``src/kernels.py:84-97``); the GPU counts them per cell and reports the sum.

Per cell and realisation step (n = p+1, N = n^d, NT = n^(d+1), m = d+2,
C_F = 2d^2+6d+3 flux flops per node as coded in ``src/pde.py:27-49``,
C_S = 2d+8 signal-speed flops per node, ``src/pde.py:51-57``)::

    predictor   K*NT*m*(2n(d+1)+d+3) + (K+1)*NT*C_F
    pred. side  2(d+1)*NT*m + 2d*NT*m + d*N*m + 8d*N*m + 4d*NT*m + 2d*N*C_S
    corrector   5d*n^(d-1)*m + 6d*N*m + N*m + d*N*C_S

Bytes (HBM, algorithmic, this implementation's data layout)::

    Q read+write, D read+write              4*N*m doubles
    face records: 2d written, 4d read       6d*(2*n^(d-1)*m + 2) doubles
"""


def shape(d, p):
    n = p + 1
    N = n ** d
    return n, N, N * n, d + 2


def flops_predict_iter(d, p):
    n, N, NT, m = shape(d, p)
    CF = 2 * d * d + 6 * d + 3
    return NT * m * (2 * n * (d + 1) + d + 3) + NT * CF


def flops_predict_fixed(d, p):
    """flops of one predict besides its K Picard iterations (final flux + pred. side)."""
    n, N, NT, m = shape(d, p)
    CF = 2 * d * d + 6 * d + 3
    CS = 2 * d + 8
    return (NT * CF + 2 * (d + 1) * NT * m + 2 * d * NT * m + d * N * m + 8 * d * N * m
            + 4 * d * NT * m + 2 * d * N * CS)


def flops_corrector(d, p):
    n, N, NT, m = shape(d, p)
    CS = 2 * d + 8
    return 5 * d * n ** (d - 1) * m + 6 * d * N * m + N * m + d * N * CS


def flops_step(d, p, cells, picard_iters, predicts):
    """Algorithmic flops of one realisation step (rerun pass included when
    ``predicts`` exceeds ``cells``)."""
    return (picard_iters * flops_predict_iter(d, p) + predicts * flops_predict_fixed(d, p)
            + cells * flops_corrector(d, p))


def bytes_step(d, p, cells, predicts=None):
    n, N, NT, m = shape(d, p)
    rec = 2 * n ** (d - 1) * m + 2
    per_cell = 8 * (4 * N * m + 6 * d * rec)
    extra = 0
    if predicts is not None and predicts > cells:       # rerun pass: read Q, write D + records
        extra = (predicts - cells) * 8 * (2 * N * m + 2 * d * rec)
    return cells * per_cell + extra


def dof(d, p, cells):
    n, N, NT, m = shape(d, p)
    return cells * N * m
