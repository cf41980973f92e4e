"""Algorithmic flop/byte model used by bench.py's roofline."""

import pytest

from paper_1801_08682_b200 import roofline


@pytest.mark.parametrize("d,p,K,per_dof", [(2, 3, 5.8, 953), (3, 3, 5.77, 1267), (3, 5, 6.84, 2813),
                                           (3, 7, 7.09, 4756), (3, 9, 7.86, 7783)])
def test_flops_per_dof_matches_survey_table(d, p, K, per_dof):
    cells = 1000
    fl = roofline.flops_step(d, p, cells, K * cells, cells)
    got = fl / roofline.dof(d, p, cells)
    assert abs(got - per_dof) / per_dof < 0.01, got


def test_bytes_model_counts_rerun_extra():
    base = roofline.bytes_step(3, 3, 100, 100)
    assert roofline.bytes_step(3, 3, 100, 200) > base
