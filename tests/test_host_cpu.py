"""Host-side logic of the multi-GPU bench arm and the large-config input
generator (CPU; no GPU needed)."""
import numpy as np
import pytest
import torch

import bench
from paper_2110_12782_b200 import inputs


def test_partition_bounds_balanced_and_strict():
    n, s, t = inputs.small_graph("rmat", 4096, 3, edge_factor=8)
    src, dst = torch.from_numpy(s), torch.from_numpy(t)
    deg = np.bincount(s, minlength=n) + np.bincount(t, minlength=n)
    cost = deg + (deg > 0)
    for ws in (1, 2, 3, 8):
        b = bench.partition_bounds(n, src, dst, ws)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 1)
        per = [cost[b[r]:b[r + 1]].sum() for r in range(ws)]
        # contiguous split of a cumulative cost: no rank above its share by more than one row's cost
        assert max(per) <= cost.sum() / ws + deg.max() + 1


def test_partition_bounds_every_rank_gets_a_row():
    n = 10
    src = torch.tensor([0, 0, 0, 0], dtype=torch.int32)
    dst = torch.tensor([1, 2, 3, 4], dtype=torch.int32)
    b = bench.partition_bounds(n, src, dst, 8)
    assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 1)


def test_rmat_device_recipe_matches_numpy_statistics():
    """inputs.rmat_device draws the recipe of inputs.rmat (another random
    stream): same quadrant law at every bit level, so the per-level bit
    frequencies of the two agree within sampling error and match the law."""
    scale, ef, a, b_, c = 12, 16, 0.57, 0.19, 0.19
    s1, t1 = inputs.rmat_device(scale, ef, a, b_, c, 5, "cpu")
    s2, t2 = inputs.rmat(scale, ef, a, b_, c, 5)
    assert s1.dtype == torch.int32 and s1.numel() == ef << scale
    s1, t1 = s1.numpy(), t1.numpy()
    m = s1.size
    for lvl in range(scale):
        bit = 1 << lvl
        for x1, x2 in ((s1, s2), (t1, t2)):
            p1, p2 = ((x1 & bit) != 0).mean(), ((x2 & bit) != 0).mean()
            assert abs(p1 - p2) < 5 * np.sqrt(0.25 / m) + 1e-3
    # P(source bit set) = c + d, P(target bit set) = b + d at every level
    d = 1 - a - b_ - c
    assert abs(((s1 & 1) != 0).mean() - (c + d)) < 0.01
    assert abs(((t1 & 1) != 0).mean() - (b_ + d)) < 0.01
    # deterministic per seed
    s3, _ = inputs.rmat_device(scale, ef, a, b_, c, 5, "cpu")
    assert np.array_equal(s1, s3.numpy())
