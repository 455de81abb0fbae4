"""Host logic of the slab partitions, no GPU: the apply's
layer ownership and the assembly's row blocks and coefficient halos."""

import pytest

from paper_1809_05471_b200.sharded import SlabAssembly, SlabPartition


@pytest.mark.parametrize("K,p,world", [(64, 4, 1), (64, 4, 2), (64, 4, 8), (10, 3, 3), (128, 6, 8), (9, 5, 2)])
def test_assembly_row_blocks_partition_rows_and_halo_covers_support(K, p, world):
    part = SlabPartition(K, p, world)
    n_layers = K + p - 1
    layer_rows = 7 * 5  # any N0·N1
    covered = []
    for r in range(world):
        sa = SlabAssembly(part, r)
        lo, hi = sa.row_range(layer_rows)
        a, b = sa.own_layers()
        assert (lo, hi) == (a * layer_rows, b * layer_rows)
        covered.append((a, b))
        e_lo, e_hi = sa.halo_elements()
        # rows of DoF layer m are sums over elements [m - p + 1, m] ∩ [0, K);
        # the one-pass symmetric kernel also forms the rows whose mirrored
        # entries land in the block: layers [a - p + 1, b + p - 1)
        need_lo, need_hi = max(0, a - 2 * (p - 1)), min(K, b + p - 1)
        assert (e_lo, e_hi) == (need_lo, need_hi)
        assert e_hi - e_lo <= (part.elements(r)[1] - part.elements(r)[0]) + 4 * (p - 1)
    assert covered[0][0] == 0 and covered[-1][1] == n_layers
    for (a0, b0), (a1, b1) in zip(covered, covered[1:]):
        assert b0 == a1 and a1 >= a0


def test_partition_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        SlabPartition(4, 3, 5)
