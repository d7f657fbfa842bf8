"""Pins of the seeded input generators (paper_1802_06215_b200/inputs.py):
the initial-belief marginals the paper states
by chi-square / binomial tests at K = 5000, and the layout facts."""
import math

import numpy as np

from paper_1802_06215_b200 import inputs


def chi2_p(counts, expected):
    """upper tail of the chi-square statistic (Wilson-Hilferty approximation)"""
    counts = np.asarray(counts, np.float64)
    expected = np.asarray(expected, np.float64)
    x2 = float(np.sum((counts - expected) ** 2 / expected))
    k = len(counts) - 1
    z = ((x2 / k) ** (1 / 3) - (1 - 2 / (9 * k))) / math.sqrt(2 / (9 * k))
    return 0.5 * math.erfc(z / math.sqrt(2))


def test_nav_start_cells_uniform_on_top_row_chi2():
    """K=5000 navigation start positions match the belief (uniform over
    the 13 top-border cells) at p > 0.01; gates uniform; unknown cells
    occupied w.p. 0.1"""
    st = inputs.nav_belief(5000, 1003)
    cells = st[0] & 0xFF
    assert np.all(cells < 13)  # top row y = 0
    counts = np.bincount(cells, minlength=13)
    assert chi2_p(counts, np.full(13, 5000 / 13)) > 0.01
    gate = (st[0] >> 8) & 1
    assert abs(gate.mean() - 0.5) < 5 * math.sqrt(0.25 / 5000)
    bits = np.unpackbits(st[1:].view(np.uint8), bitorder="little").reshape(-1)
    occ = bits.reshape(4, 5000, 32).transpose(1, 0, 2).reshape(5000, 128)[:, :124]
    assert abs(occ.mean() - 0.1) < 5 * math.sqrt(0.09 / occ.size)
    assert not np.any(bits.reshape(4, 5000, 32).transpose(1, 0, 2).reshape(5000, 128)[:, 124:])


def test_rock_good_rate_and_layout():
    st = inputs.rocksample_belief(15, 15, 2, 5000, 1002)
    good = (st[0][:, None] >> np.arange(15)) & 1
    assert abs(good.mean() - 0.5) < 5 * math.sqrt(0.25 / good.size)
    assert np.all(st[0] < (1 << 15))
    rocks, starts = inputs.rocksample_layout(15, 15, 2)
    assert len(set(rocks)) == 15 and starts == [(0, 5), (0, 10)]
    assert inputs.rocksample_layout(7, 8, 1) == (inputs.RS78_ROCKS, [inputs.RS78_START])


def test_car_goals_uniform_and_positions_shared():
    st = inputs.car_belief(5000, 1004)
    goals = np.concatenate([(st[2][:, None] >> (2 * np.arange(16))) & 3, (st[3][:, None] >> (2 * np.arange(4))) & 3],
                           axis=1)
    counts = np.bincount(goals.reshape(-1).astype(np.int64), minlength=4)
    assert chi2_p(counts, np.full(4, goals.size / 4)) > 0.01
    assert np.all(st[4:] == st[4:, :1])  # pedestrian positions are observed: identical in all scenarios


def test_weights_and_leaf_selection():
    w = inputs.weights(500)
    assert w.dtype == np.float32 and np.all(w == np.float32(1 / 500))
    wn = inputs.weights(500, 3, uniform=False)
    assert abs(float(wn.astype(np.float64).sum()) - 1.0) < 1e-5 and np.all(wn > 0)
    # leaf generator: sorted by (-N_c, action, ordinal)
    cb = np.array([0, 2, 3, 5])
    cc = np.array([3, 7, 9, 4, 7])
    assert inputs.select_leaves(cc, cb, 3, 4) == [(1, 0), (0, 1), (2, 1), (2, 0)]
