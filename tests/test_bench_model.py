"""CPU checks of bench.py's executed-relaxation model of query_grouped
(grouped_executed_relaxations): hand-computed task shapes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_single_bin_full_column_groups():
    # 5 queries of pair (0, 1): B1 = 20 rows, B2 = 64 columns (2 full groups)
    bsize = np.array([20, 64])
    c1 = np.zeros(5, np.int64)
    c2 = np.ones(5, np.int64)
    # slots 4 * ceil(5/4) = 8; cols 2 x 32; rows 16 + roundup4(4) = 20, + 1 combine pass
    assert bench.grouped_executed_relaxations(2, bsize, c1, c2) == 8 * 64 * 21


def test_half_tail_and_orientation():
    # pairs (1, 0) orient to (0, 1); B2 = 40: one 32-column group + an 8-column
    # tail run as a 16-column task with query slots in steps of 8
    bsize = np.array([18, 40])
    c1 = np.ones(3, np.int64)
    c2 = np.zeros(3, np.int64)
    rows = 16 + 4 + 1  # 18 rows: 16 + roundup4(2), + combine
    want = (4 * 32 + 8 * 16) * rows
    assert bench.grouped_executed_relaxations(2, bsize, c1, c2) == want


def test_balanced_split_of_a_large_bin():
    # 36 queries -> 2 items of 20 + 16 (not 32 + 4)
    bsize = np.array([16, 32])
    c1 = np.zeros(36, np.int64)
    c2 = np.ones(36, np.int64)
    rows = 16 + 1
    assert bench.grouped_executed_relaxations(2, bsize, c1, c2) == (20 + 16) * 32 * rows
