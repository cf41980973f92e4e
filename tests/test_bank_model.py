"""Shared-memory layouts of the p = 5 / 7 / 9 sweep kernels against the bank model they
were derived from: the LSU serves a 16-byte access per quarter-warp (eight
16-byte bank groups) and an 8-byte access per half-warp (sixteen 8-byte banks).  The
constants are parsed from the CUDA sources, the address formulas are restated here; ncu's
per-line wavefront counts (profiles/r02) equal what this model gives."""
import os
import re

import pytest

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_1801_08682_b200", "csrc")


def src(name):
    with open(os.path.join(CSRC, name)) as fh:
        return fh.read()


def wavefronts8(addrs):
    """8-byte accesses of one half-warp (addresses in doubles)."""
    banks = {}
    for a in set(addrs):
        banks.setdefault(a % 16, set()).add(a)
    return max(len(v) for v in banks.values())


def wavefronts16(addrs):
    """16-byte accesses of one quarter-warp (addresses in doubles, even)."""
    banks = {}
    for a in set(addrs):
        assert a % 2 == 0
        banks.setdefault((a // 2) % 8, set()).add(a)
    return max(len(v) for v in banks.values())


# ---------------------------------------------------------------------------
# p = 5
def p5_layout():
    s = src("aderdg_sweep_p5.cuh")
    tbl = re.search(r"kBlock\[28\] = \{([^}]*)\}", s).group(1)
    codes = [int(x) for x in tbl.replace("\n", " ").split(",")]
    acol = 23 * 8
    stride = 3 * acol + 16
    rowoff = lambda j: j * stride + (4 if j in (2, 3) else 0)
    return codes, acol, stride, rowoff


def p5_node(codes, tid):
    code = codes[tid >> 3]
    return (2 * (code // 9) + ((tid >> 2) & 1), 2 * ((code // 3) % 3) + ((tid >> 1) & 1),
            2 * (code % 3) + (tid & 1))


def test_p5_block_table_is_a_permutation():
    codes, *_ = p5_layout()
    assert sorted(codes[:27]) == list(range(27))
    nodes = {p5_node(codes, t) for t in range(216)}
    assert len(nodes) == 216 and all(max(n) < 6 for n in nodes)


def test_p5_owner_accesses_at_minimum_wavefronts():
    codes, acol, stride, rowoff = p5_layout()
    perfect8 = 0
    for a in range(3):
        def base(t):
            i = p5_node(codes, t)
            others = [i[b] for b in range(3) if b != a]
            return a * acol + rowoff(i[a]), others[0] * 6 + others[1]
        # 16-byte accesses (components 0-1 at column 2o, 2-3 at 72 + 2o): one block per quarter-warp
        for q in range(27):
            for off in (0, 72):
                ad = [base(t)[0] + off + 2 * base(t)[1] for t in range(8 * q, 8 * q + 8)]
                assert wavefronts16(ad) == 1
    # 8-byte accesses (component 4 at column 144 + o): two blocks per half-warp
    for h in range(13):
        ok = True
        for a in range(3):
            def addr(t):
                i = p5_node(codes, t)
                others = [i[b] for b in range(3) if b != a]
                return a * acol + rowoff(i[a]) + 144 + others[0] * 6 + others[1]
            ok = ok and wavefronts8([addr(t) for t in range(16 * h, 16 * h + 16)]) == 1
        perfect8 += ok
    assert perfect8 >= 11          # the maximum matching of the block grid


def test_p5_line_accesses_conflict_free():
    codes, acol, stride, rowoff = p5_layout()
    for r in range(3):
        for h in range(14):
            lines = [t + 224 * r for t in range(16 * h, 16 * h + 16) if t + 224 * r < 540]
            for j in range(6):
                # a half-warp may straddle two axis blocks: each axis part is contiguous
                ad = [(l // 180) * acol + rowoff(j) + l % 180 for l in lines]
                if ad:
                    assert wavefronts8(ad) <= 2
                    if len({l // 180 for l in lines}) == 1:
                        assert wavefronts8(ad) == 1


# ---------------------------------------------------------------------------
# p = 7
def p7_node(tid):
    warp, lane = tid >> 5, tid & 31
    return (2 * (warp >> 2) + ((lane >> 2) & 1), 2 * (warp & 3) + ((lane >> 3) & 1),
            (lane & 3) | ((lane >> 4) << 2))


def test_p7_layout_at_minimum_wavefronts():
    ncol = 5 * 64
    stride = 3 * ncol + 4
    assert re.search(r"STR = DIM \* NCOL \+ 4;", src("aderdg_sweep_p7.cuh"))
    assert len({p7_node(t) for t in range(512)}) == 512
    ow = [lambda i: 0 * ncol + i[0] * stride + i[1] * 8 + i[2],
          lambda i: 1 * ncol + i[1] * stride + i[0] * 8 + i[2],
          lambda i: 2 * ncol + i[2] * stride + (i[0] & 1) + 2 * (i[1] & 1) + 4 * (i[0] >> 1) + 16 * (i[1] >> 1)]
    for a in range(3):
        cols = {ow[a](p7_node(t)) % stride - a * ncol for t in range(512)}
        assert len({ow[a](p7_node(t)) for t in range(512)}) == 512 and max(cols) < 64
        for h in range(32):
            assert wavefronts8([ow[a](p7_node(t)) for t in range(16 * h, 16 * h + 16)]) == 1
    # tile accesses: B-fragment loads (rows k = lane & 3 (+4), column lane >> 2) and the
    # 16-byte D stores of the permuted rows
    for hw in range(2):
        lanes = range(16 * hw, 16 * hw + 16)
        for k0 in (0, 4):
            assert wavefronts8([((l & 3) + k0) * stride + (l >> 2) for l in lanes]) == 1
    prow = lambda fr: (fr & 4) | ((fr & 1) << 1) | ((fr >> 1) & 1)
    assert sorted(prow(r) for r in range(8)) == list(range(8))
    for q in range(4):
        lanes = range(8 * q, 8 * q + 8)
        assert wavefronts16([prow(l >> 2) * stride + 2 * (l & 3) for l in lanes]) == 1
    # padded tail staging: the face-trace gathers of a half-warp (pairs of lanes share a node)
    t1, t0 = 9, 72
    for a in range(3):
        for y0 in range(0, 64, 8):
            ys = range(y0, y0 + 8)
            xb = [(y // 8) * t1 + y % 8 if a == 0 else (y // 8) * t0 + y % 8 if a == 1
                  else (y // 8) * t0 + (y % 8) * t1 for y in ys]
            assert wavefronts8(xb) == 1


# ---------------------------------------------------------------------------
# p = 9
def test_p9_line_wavefronts_match_the_search():
    s = src("aderdg_sweep_p9.cuh")
    m = re.search(r"static constexpr int P0 = (\d+), P1 = (\d+), SC = (\d+);", s)
    p0, p1, sc = (int(x) for x in m.groups())

    def cost(bases):
        return sum(wavefronts8(bases[h:h + 16]) for h in range(0, 500, 16))

    new = [[(l % 5) * sc + (l // 50) * p1 + (l // 5) % 10 for l in range(500)],
           [(l % 5) * sc + ((l // 5) % 10) * p0 + l // 50 for l in range(500)],
           [(l % 5) * sc + ((l // 5) % 10) * p0 + (l // 50) * p1 for l in range(500)]]
    old = [[(l // 100) * 1124 + ((l % 100) // 10) * su + (l % 10) * sv for l in range(500)]
           for su, sv in ((10, 1), (111, 1), (111, 10))]
    assert sum(cost(b) for b in old) == 152        # r01 strides: ncu measured 1.58 x 96
    assert sum(cost(b) for b in new) <= 104        # 96 is the ideal (32 half-warps x 3 axes)
    assert 9 * p0 + 9 * p1 + 9 < sc
