"""Block-cyclic row-panel layout of the sharded sweep (distributed.RowPanels): ownership is a
partition of the rows, local ranges select exactly the owned rows of a global range, and the
per-rank shares of a set's complement stay balanced (the reason for the cyclic layout)."""

import numpy as np
import pytest

from paper_2502_06377_b200.distributed import RowPanels, map_indices


@pytest.mark.parametrize("p,world,panel", [(96, 2, 8), (100, 3, 8), (1000, 4, 64), (16384, 8, 128), (65536, 8, 128),
                                           (7, 3, 4), (5, 8, 128)])
def test_ownership_is_a_partition_and_cyclic(p, world, panel):
    lay = RowPanels(p, world, panel)
    allrows = np.concatenate(lay.rows)
    assert np.array_equal(np.sort(allrows), np.arange(p))
    for h, rows in enumerate(lay.rows):
        assert np.all((rows // panel) % world == h)
        assert np.all(np.diff(rows) > 0)
    assert np.array_equal(lay.owner, (np.arange(p) // panel) % world)


@pytest.mark.parametrize("p,world,panel,lo,hi", [(100, 3, 8, 13, 61), (1000, 4, 64, 0, 1000), (1000, 4, 64, 500, 500),
                                                 (16384, 8, 128, 1792, 4352), (65536, 8, 128, 60928, 65536)])
def test_local_range_selects_owned_rows_of_a_global_range(p, world, panel, lo, hi):
    lay = RowPanels(p, world, panel)
    total = 0
    for h in range(world):
        a, b = lay.local_range(h, lo, hi)
        sel = lay.rows[h][a:b]
        assert np.all((sel >= lo) & (sel < hi))
        rest = np.concatenate([lay.rows[h][:a], lay.rows[h][b:]])
        assert not np.any((rest >= lo) & (rest < hi))
        total += b - a
    assert total == hi - lo


def test_complement_shares_are_balanced_at_the_baseline_configs():
    """c4 / c5 with G = 8: every rank's share of a set's complement (its panel-GEMM columns)
    is within one panel of the mean; contiguous panels would leave the owners of I with b fewer."""
    for p, m, h, world in [(16384, 2048, 256, 8), (65536, 4096, 512, 8)]:
        lay = RowPanels(p, world, 128)
        for k in range(p // m):
            lo, hi = max(0, k * m - h), min(p, (k + 1) * m + h)
            shares = []
            for g in range(world):
                a, b = lay.local_range(g, lo, hi)
                shares.append(len(lay.rows[g]) - (b - a))
            assert max(shares) - min(shares) <= 128, (p, k, shares)


def test_map_indices_gap_map():
    assert list(map_indices((3, 0, 7), 6)) == [0, 1, 2, 7, 8, 9]
    assert list(map_indices(5, 3)) == [5, 6, 7]


def test_comm_model_conserves_bytes_and_matches_the_design_table():
    """ShardedSolver.comm_model: what the ranks send in the transpose exchange is what they receive,
    the GEMM flops add up to 2bc² + 2b²c, and the per-step figures quoted in DESIGN.md §6 hold."""
    from paper_2502_06377_b200.distributed import ShardedSolver

    table = {  # (p, lo, hi, world): (exchange MB, all-reduce MB, W all-gather MB) of DESIGN.md §6
        (16384, 1792, 4352, 8): (31, 92, 294), (16384, 1792, 4352, 2): (71, 52, 168),
        (65536, 3584, 8704, 8): (271, 367, 2350), (65536, 3584, 8704, 2): (619, 210, 1340),
    }
    for (p, lo, hi, world), (ex, ar, ag) in table.items():
        ms = [ShardedSolver.comm_model(p, lo, hi, world, r) for r in range(world)]
        b, c = hi - lo, p - (hi - lo)
        assert sum(m["exchange_out"] for m in ms) == sum(m["exchange_in"] for m in ms)
        assert sum(m["gemm_flops"] for m in ms) == 2 * b * c * c + 2 * b * b * c
        assert abs(sum(m["exchange_out"] for m in ms) / world / 1e6 - ex) <= 0.02 * ex      # mean over ranks
        assert abs(ms[0]["allreduce_top"] / 1e6 - ar) <= 0.02 * ar
        assert abs(max(m["allgather_w_in"] for m in ms) / 1e6 - ag) <= 0.02 * ag
        assert ShardedSolver.comm_model(p, lo, hi, world, 0, operands="replicated")["allgather_w_in"] == 0
