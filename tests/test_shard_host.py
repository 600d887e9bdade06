"""Host logic of pixel sharding, CPU only: the rank ranges partition the frame."""
import pytest

from paper_2007_14283_b200.dist import shard_range


@pytest.mark.parametrize("n,world", [(16384, 2), (16384, 3), (262144, 8), (24117248, 8), (9, 9), (1000, 7)])
def test_shard_ranges_partition(n, world):
    rs = [shard_range(n, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_shard_range_rejects_bad_args():
    for args in [(10, -1, 2), (10, 2, 2), (1, 0, 2)]:
        with pytest.raises(ValueError):
            shard_range(*args)
