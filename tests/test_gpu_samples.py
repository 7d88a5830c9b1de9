"""GPU parity of the raw-address ProfileWindow API:
stg_aggregate_samples vs the reference's aggregate_samples (samples.cpp:31-85,
oracle/_ref) — window bounds, first-seen record order and counts bit-exact —
plus the reference's own test cases (test_collector.cpp:43-99) restated, error
messages, the exact (comparator-sort) path, and size-independent properties at
sizes the reference would take minutes on.
"""
import numpy as np
import pytest

import paper_2603_29235_b200 as stg
from oracle import ref, strata_oracle as so
from tests.synth import oracle_stream, raw_stream

pytestmark = pytest.mark.gpu
need_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _gpu(ctx, ts, rk, off, pc, bn, drain, exact=False, device=False):
    if device:
        import torch
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
        got = ctx.aggregate_samples(t(ts, np.int64), t(off, np.int64), t(pc, np.int64), t(bn, np.int16),
                                    rank=None if rk is None else t(rk, np.int32), drain_interval_ns=drain,
                                    exact=exact)
    else:
        got = ctx.aggregate_samples(ts, off, pc, bn, rank=rk, drain_interval_ns=drain, exact=exact)
    return [(s, e, [(int(f), int(c)) for f, c in zip(fs, cs)]) for s, e, fs, cs in got]


@need_ref
@pytest.mark.parametrize("seed,drain,t0", [(1, 5_000_000_000, 3_000_000_000), (2, 1_000_000_000, -4_000_000_123),
                                           (3, 7, 0), (4, 10**15, 123), (5, 5_000_000_000, 5_000_000_000)])
@pytest.mark.parametrize("exact", [False, True])
def test_aggregate_matches_reference(ctx, seed, drain, t0, exact):
    ts, rk, off, pc, bn, ids = raw_stream(seed=seed, n=3000, t0=t0)
    exp = ref.aggregate_samples(ts, off, pc, bn, ids, rank=rk, drain=drain)
    got = _gpu(ctx, ts, rk, off, pc, bn, drain, exact=exact)
    assert got == [(s, e, recs) for _, s, e, recs in exp]


@need_ref
def test_aggregate_device_resident_input(ctx):
    ts, rk, off, pc, bn, ids = raw_stream(seed=9, n=5000)
    exp = ref.aggregate_samples(ts, off, pc, bn, ids, rank=rk)
    assert _gpu(ctx, ts, rk, off, pc, bn, 5_000_000_000, device=True) == [(s, e, r) for _, s, e, r in exp]


def _stream(samples):
    """[(ts, [offsets])] with one build id (test_collector.cpp:17-24)."""
    ts = np.array([t for t, _ in samples], np.int64)
    off = np.zeros(len(samples) + 1, np.uint64)
    off[1:] = np.cumsum([len(o) for _, o in samples])
    pc = np.array([x for _, o in samples for x in o], np.uint64)
    return ts, off, pc, np.zeros(len(pc), np.uint16)


def test_lossless_and_merging(ctx):  # test_collector.cpp:43-56
    ts, off, pc, bn = _stream([(0, [1, 2]), (10, [1, 2]), (20, [3]), (30, [1, 2])])
    got = _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000)
    assert got == [(0, 5_000_000_000, [(0, 3), (2, 1)])]


def test_drain_grid(ctx):  # test_collector.cpp:58-71
    ts, off, pc, bn = _stream([(1_000_000_000, [1]), (6_000_000_000, [1]), (6_500_000_000, [2]),
                               (22_000_000_000, [1])])
    got = _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000)
    assert [(s, e) for s, e, _ in got] == [(0, 5 * 10**9), (5 * 10**9, 10**10), (20 * 10**9, 25 * 10**9)]
    assert [r for _, _, r in got] == [[(0, 1)], [(1, 1), (2, 1)], [(3, 1)]]


def test_validation_messages(ctx):  # test_collector.cpp:73-82
    ts, off, pc, bn = _stream([(0, [8])])
    assert _gpu(ctx, ts[:0], None, off[:1], pc[:0], bn[:0], 5_000_000_000) == []
    with pytest.raises(stg.StgError, match="drain interval must be positive"):
        _gpu(ctx, ts, None, off, pc, bn, 0)
    ts, off, pc, bn = _stream([(0, [8]), (5, [8])])
    with pytest.raises(stg.StgError, match="aggregate_samples: mixed ranks"):
        _gpu(ctx, ts, np.array([0, 1], np.int32), off, pc, bn, 5_000_000_000)
    ts, off, pc, bn = _stream([(10, [8]), (5, [8])])
    with pytest.raises(stg.StgError, match="aggregate_samples: timestamps regressed"):
        _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000)
    ts, off, pc, bn = _stream([(0, [8]), (5, [])])
    with pytest.raises(stg.StgError, match="empty sample stack"):
        _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000)


@need_ref
@pytest.mark.parametrize("case", ["empty_then_regress", "regress_then_empty", "mixed_then_empty"])
def test_first_error_in_stream_order(ctx, case):
    ts, rk, off, pc, bn, ids = raw_stream(seed=4, n=400)
    ts, rk, off = ts.copy(), rk.copy(), off.astype(np.int64)
    a, b = (100, 200)

    def drop(i):
        nonlocal pc, bn, off
        f0, f1 = int(off[i]), int(off[i + 1])
        pc, bn = np.delete(pc, np.s_[f0:f1]), np.delete(bn, np.s_[f0:f1])
        off[i + 1:] -= f1 - f0

    if case == "empty_then_regress":
        drop(a)
        ts[b] = ts[b - 1] - 1
    elif case == "regress_then_empty":
        ts[a] = ts[a - 1] - 1
        drop(b)
    else:
        rk[a] = 99
        drop(b)
    off = off.astype(np.uint64)
    with pytest.raises(ref.RefError) as r:
        ref.aggregate_samples(ts, off, pc, bn, ids, rank=rk)
    with pytest.raises(stg.StgError) as g:
        _gpu(ctx, ts, rk, off, pc, bn, 5_000_000_000)
    assert str(g.value) == str(r.value)


def test_large_stream_properties(ctx):
    """2 M samples: the fingerprint path equals the exact comparator path, counts
    sum to the input, records are first-seen (each record's first sample is not
    preceded in its window by an equal stack — checked on a sample of records via
    the oracle on the window prefix), and windows tile the grid in order."""
    ts, rk, off, pc, bn, ids = raw_stream(seed=21, n=2_000_000, n_stacks=3000, max_depth=40, n_bins=3,
                                          span_ns=60_000_000_000)
    fast = _gpu(ctx, ts, rk, off, pc, bn, 5_000_000_000)
    exact = _gpu(ctx, ts, rk, off, pc, bn, 5_000_000_000, exact=True)
    assert fast == exact
    assert sum(c for _, _, r in fast for _, c in r) == len(ts)
    starts = [s for s, _, _ in fast]
    assert starts == sorted(starts) and all((s % 5_000_000_000) == 0 for s in starts)
    # first-seen order inside each window
    for _, _, r in fast:
        firsts = [f for f, _ in r]
        assert firsts == sorted(firsts)
    # oracle on the first window
    s0, e0, r0 = fast[0]
    n0 = int(np.searchsorted(ts, e0))
    stream = oracle_stream(ts[:n0], rk[:n0], off[:n0 + 1], pc, bn, ids)
    exp = so.aggregate_samples(stream)
    assert [c for _, c in exp[0][2]] == [c for _, c in r0]
    assert [stream[f][2] for f, _ in r0] == [fr for fr, _ in exp[0][2]]


@need_ref
def test_aggregate_unaligned_device_input(ctx):
    """frame arrays not 32/16-byte aligned take the scalar-load kernel variant."""
    import torch
    ts, rk, off, pc, bn, ids = raw_stream(seed=13, n=4000)
    exp = ref.aggregate_samples(ts, off, pc, bn, ids, rank=rk)
    pc_u = torch.from_numpy(np.concatenate([[0], pc]).astype(np.uint64).view(np.int64)).cuda()[1:]
    bn_u = torch.from_numpy(np.concatenate([[0], bn]).astype(np.uint16).view(np.int16)).cuda()[1:]
    assert pc_u.data_ptr() % 32 and bn_u.data_ptr() % 16
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
    got = ctx.aggregate_samples(t(ts, np.int64), t(off, np.int64), pc_u, bn_u, rank=t(rk, np.int32))
    got = [(s, e, [(int(f), int(c)) for f, c in zip(fs, cs)]) for s, e, fs, cs in got]
    assert got == [(s, e, r) for _, s, e, r in exp]


def test_aggregate_table_growth_all_distinct(ctx):
    """A stream of 1.5 M distinct stacks overflows the initial table several
    times (grow-and-retry); the result equals the exact path and every sample is
    its own record."""
    n = 1_500_000
    rng = np.random.default_rng(3)
    ts = np.sort(rng.integers(0, 20_000_000_000, size=n)).astype(np.int64)
    off = (np.arange(n + 1) * 3).astype(np.uint64)
    pc = np.stack([np.arange(n), rng.integers(0, 1 << 40, size=n), np.full(n, 7)], 1).reshape(-1).astype(np.uint64)
    bn = np.zeros(3 * n, np.uint16)
    fast = _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000)
    assert sum(len(r) for _, _, r in fast) == n
    assert [f for _, _, r in fast for f, _ in r] == list(range(n))
    assert fast == _gpu(ctx, ts, None, off, pc, bn, 5_000_000_000, exact=True)
