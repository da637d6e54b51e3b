"""CPU: the {bitstring: count} dict of CountsTable (statevec.py:64-73 in the reference) built by
the CPython helper (csrc/counts_dict.c) equals the per-index bitstring() formatting, in
index order, for every width the planner accepts."""

import numpy as np
import pytest

from paper_2504_03967_b200 import statevec as sv


@pytest.mark.parametrize("n", [0, 1, 5, 8, 9, 17, 32, 33, 47, 62])
def test_counts_dict_matches_bitstring(n):
    from paper_2504_03967_b200._counts import counts_dict

    rng = np.random.default_rng(n)
    idx = np.unique(rng.integers(0, 1 << n, 300, dtype=np.int64)) if n else np.zeros(1, np.int64)
    cnt = rng.integers(1, 1 << 40, idx.size, dtype=np.int64)
    got = counts_dict(idx, cnt, n)
    ref = {sv.bitstring(int(i), n): int(c) for i, c in zip(idx, cnt)}
    assert got == ref and list(got) == list(ref)
    table = sv.counts_from_arrays(idx, cnt, int(cnt.sum()), n)
    assert table.counts == ref and table.total == int(cnt.sum())


def test_counts_dict_rejects_bad_arrays():
    from paper_2504_03967_b200._counts import counts_dict

    with pytest.raises(ValueError):
        counts_dict(np.zeros(3, np.int64), np.zeros(2, np.int64), 4)
    with pytest.raises(ValueError):
        counts_dict(np.zeros(3, np.int64), np.zeros(3, np.int64), 65)
