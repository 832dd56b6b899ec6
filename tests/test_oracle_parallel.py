"""The T-thread oracle replay (timing variant) equals the
1-thread replay bit for bit: verdicts, statuses, final A and V, leaks."""
import numpy as np
import pytest

import oracle
import tracegen as tg


def _both(tr, T):
    o1, v1, s1, l1 = oracle.replay_trace(tr)
    o2 = oracle.Oracle(tr.host_base, tr.host_size)
    v2, s2 = o2.replay_parallel(tr.events, tr.blob, threads=T)
    for f in v1.dtype.names:
        assert np.array_equal(v1[f], v2[f]), f
    assert np.array_equal(s1, s2)
    assert np.array_equal(o1.A, o2.A) and np.array_equal(o1.V, o2.V)
    l2 = o2.leaks()
    assert np.array_equal(l1, l2)


@pytest.mark.parametrize("T", [2, 3, 8])
@pytest.mark.parametrize("seed", range(10))
def test_parallel_tiny(seed, T):
    _both(tg.random_tiny(seed + 40000, arrays=seed % 2 == 0), T)


@pytest.mark.parametrize("seed", range(4))
def test_parallel_medium(seed):
    _both(tg.random_medium(seed + 600), 5)


def test_parallel_configs_scaled():
    _both(tg.toy(), 4)
    _both(tg.c2_small(n_copies=20000, n_allocs=2000), 8)
    _both(tg.c4_pitched(n_copies=1000, n_bufs=2, rows=128, inject_frac=0.05), 8)
    _both(tg.c5_sharded(scale=0.002), 8)
