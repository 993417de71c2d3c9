"""Host pipeline grouping (paper_2007_08501_b200/pipeline.py): contiguous, covering, byte-balanced, ramped."""
import numpy as np

from paper_2007_08501_b200.pipeline import contiguous_groups, transfer_costs


def _check_cover(groups, n):
    assert groups[0][0] == 0 and groups[-1][1] == n
    for (a0, a1), (b0, b1) in zip(groups, groups[1:]):
        assert a1 == b0 and a0 < a1
    assert groups[-1][0] < groups[-1][1]


def test_groups_cover_and_balance():
    rng = np.random.default_rng(0)
    costs = rng.integers(1, 100, size=200).astype(float)
    for n_groups in (1, 2, 7, 16, 200, 500):
        g = contiguous_groups(costs, n_groups)
        _check_cover(g, len(costs))
        assert len(g) <= min(n_groups, len(costs))
    g = contiguous_groups(costs, 8)
    sums = [costs[a:b].sum() for a, b in g]
    assert max(sums) - min(sums) <= 2 * costs.max()


def test_ramp_makes_end_groups_smaller():
    costs = np.ones(1024)
    g = contiguous_groups(costs, 16, ramp=2)
    _check_cover(g, 1024)
    sizes = [b - a for a, b in g]
    assert sizes[0] < sizes[1] < sizes[5] and sizes[-1] < sizes[-2] < sizes[5]
    assert abs(sizes[0] * 4 - sizes[5]) <= 4 and abs(sizes[-1] * 4 - sizes[5]) <= 4


def test_transfer_costs():
    c = transfer_costs([10, 0], 4 * 4 * 2, backward=True)
    assert c.tolist() == [72 * 10 * 2 + 48 * 32, 48 * 32]
    c = transfer_costs([10], 32, backward=False)
    assert c.tolist() == [72 * 10 + 28 * 32]
