"""Error behaviour at the boundary: for invalid windows the C-ABI must refuse
with exactly the strata::Error message the reference throws (SURVEY.md §8(b):
"device-side validation must reproduce the same throw conditions"), and must
NOT throw where the reference does not (e.g. a regression outside the window).
"""
import numpy as np
import pytest

import paper_2603_29235_b200 as stg
from oracle import ref, strata_oracle as so
from tests.synth import pack_symr, build_id, small_window, with_empty_stacks

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _both(ctx, win):
    """(reference message or None, libstg message or None)."""
    try:
        ref.window_run(win, want_json=False)
        r = None
    except ref.RefError as e:
        r = str(e)
    try:
        ctx.window_run(win)
        g = None
    except stg.StgError as e:
        g = str(e)
    try:
        so.window_pipeline(win)
        o = None
    except so.StrataError as e:
        o = str(e)
    assert o == r, (o, r)
    return r, g


def _win(**kw):
    return small_window(seed=3, ranks=4, samples_per_rank=120, slow_rank=-1, iterations=20, **kw)


def test_entry_not_before_exit(ctx):
    w = _win()
    w.coll_exit = w.coll_exit.copy()
    w.coll_exit[17] = w.coll_entry[17]
    r, g = _both(ctx, w)
    assert r == g == "collective event with entry >= exit"


def test_entry_regression_within_rank(ctx):
    w = _win()
    w.coll_entry = w.coll_entry.copy()
    i = 4 * 7  # event of rank 0 in iteration 7
    w.coll_entry[i] = w.coll_entry[i - 4] - 1
    w.coll_exit = np.maximum(w.coll_exit, w.coll_entry + 1)
    r, g = _both(ctx, w)
    assert r == g == "collective events not time-ordered within rank"


def test_first_collective_error_wins(ctx):
    w = _win()
    w.coll_entry = w.coll_entry.copy()
    w.coll_exit = w.coll_exit.copy()
    w.coll_exit[30] = w.coll_entry[30]          # entry >= exit at index 30
    w.coll_entry[12] = w.coll_entry[8] - 1       # regression at index 12 (rank 0)
    r, g = _both(ctx, w)
    assert r == g


def _drop_frames(w, sample):
    f0, f1 = int(w.sample_frame_off[sample]), int(w.sample_frame_off[sample + 1])
    w.frame_pc = np.delete(w.frame_pc, np.s_[f0:f1])
    w.frame_bin = np.delete(w.frame_bin, np.s_[f0:f1])
    off = w.sample_frame_off.astype(np.int64)
    off[sample + 1:] -= f1 - f0
    w.sample_frame_off = off.astype(np.uint64)


def test_empty_stack_in_window(ctx):
    w = _win()
    _drop_frames(w, 200)  # rank 1, well inside the window
    r, g = _both(ctx, w)
    assert r == g == "empty sample stack"


def test_empty_stack_outside_window_is_ignored(ctx):
    w = _win()
    _drop_frames(w, 120)  # first sample of rank 1: before the window start
    r, g = _both(ctx, w)
    assert r is None and g is None


def test_timestamp_regression(ctx):
    w = _win()
    w.sample_ts = w.sample_ts.copy()
    w.sample_ts[300] = w.sample_ts[299] - 1000
    r, g = _both(ctx, w)
    assert r == g == "aggregate_samples: timestamps regressed"


def test_regression_before_window_is_ignored(ctx):
    w = _win()
    w.sample_ts = w.sample_ts.copy()
    w.sample_ts[121] = w.sample_ts[120] - 10  # rank 1, both out of the window
    r, g = _both(ctx, w)
    assert r is None and g is None


def test_empty_before_regression_in_same_rank(ctx):
    w = _win()
    w.sample_ts = w.sample_ts.copy()
    w.sample_ts[310] = w.sample_ts[309] - 1000
    _drop_frames(w, 305)
    r, g = _both(ctx, w)
    assert r == g == "empty sample stack"


def test_drain_interval_must_be_positive(ctx):
    w = _win()
    w.window_end_ns = w.window_start_ns - 2 * w.max_skew_ns
    r, g = _both(ctx, w)
    assert r == g == "drain interval must be positive"


@pytest.mark.parametrize("which", ["magic", "version", "count", "truncated", "unsorted", "name"])
def test_symr_validation_messages(ctx, which):
    good = pack_symr(build_id("err"), [0x10, 0x20], [4, 4], ["a", "b"])
    b = bytearray(good)
    if which == "magic":
        b[0] = ord("X")
    elif which == "version":
        b[4] = 99
    elif which == "count":
        b[28] = 77
    elif which == "truncated":
        b = b[:20]
    elif which == "unsorted":
        b[36:52], b[52:68] = good[52:68], good[36:52]
    elif which == "name":
        b[36 + 12] = 200  # name offset past the string table
    b = bytes(b)
    exp = ref.parse_error(b)
    assert exp is not None
    with pytest.raises(stg.StgError) as e:
        ctx.ingest(b)
    assert str(e.value) == exp


def test_ingest_key_mismatch_and_idempotence(ctx):
    p = pack_symr(build_id("k1"), [0x10], [4], ["a"])
    assert ctx.ingest(p, claimed_id=build_id("k1")) in (True, False)
    assert ctx.ingest(p, claimed_id=build_id("k1")) is False  # AlreadyPresent
    with pytest.raises(stg.StgError, match="symbol file build id does not match ingest key"):
        ctx.ingest(pack_symr(build_id("k2"), [0x10], [4], ["a"]), claimed_id=build_id("k3"))


def test_rank_with_only_empty_in_window_stacks(ctx):
    """A rank whose in-window samples ALL have empty stacks aggregates nothing,
    but the reference's aggregate_samples still throws on its first one."""
    w = with_empty_stacks(_win(), 2, "all")
    r, g = _both(ctx, w)
    assert r == g == "empty sample stack"


def test_empty_stack_in_last_rank(ctx):
    w = with_empty_stacks(_win(), 3, [40])
    r, g = _both(ctx, w)
    assert r == g == "empty sample stack"
