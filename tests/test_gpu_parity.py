"""GPU parity: libstg (C-ABI) vs the oracle on identical windows.

Bar: folded lines, counts, totals, symbol names, lateness, GPU/OS sums, flagged
ranks, verdicts and top paths are bit-exact; floating-point scores (fractions,
z-scores, evidence values) agree within 1e-6 relative (north_star tolerance).
"""
import numpy as np
import pytest

from oracle import ref, strata_oracle as so
from tests.compare import assert_close
from tests.synth import small_window

pytestmark = pytest.mark.gpu
REL = 1e-6  # north_star: floating-point scores within 1e-6 relative


def _check_window(ctx, win, against_ref=False):
    stats = ctx.window_run(win)
    gd = ctx.groupdata()
    rep = ctx.report()
    if against_ref:
        r, _, _ = ref.window_run(win)
        ogd, orep = r["groupdata"], r["report"]
    else:
        ogd, orep = so.window_pipeline(win)
    # integer / string / order results: exact
    assert gd["cpu_profiles"] == ogd["cpu_profiles"]
    assert gd["gpu_profiles"] == ogd["gpu_profiles"]
    assert gd["os_snapshots"] == ogd["os_snapshots"]
    assert rep["verdict"] == orep["verdict"]
    assert rep["flagged_ranks"] == orep["flagged_ranks"]
    assert rep["top_path"] == orep["top_path"]
    assert rep["reference_rank"] == orep["reference_rank"]
    assert rep["notes"] == orep["notes"]
    # lateness and iteration times are computed in the reference's FP order
    assert gd["lateness_per_instance"] == ogd["lateness_per_instance"]
    assert gd["iteration_times_ms"] == ogd["iteration_times_ms"]
    assert_close(gd, ogd, REL)
    assert_close(rep, orep, 0.0)  # the report is bit-exact (reference FP order)
    return stats, rep


@pytest.mark.parametrize("seed,slow", [(7, 3), (1, 4), (2, -1), (3, 0)])
def test_synthetic_window_matches_oracle(ctx, seed, slow):
    win = small_window(seed=seed, ranks=8, samples_per_rank=600, slow_rank=slow)
    _check_window(ctx, win)


def test_unknown_binaries_and_gaps(ctx):
    win = small_window(seed=11, ranks=6, samples_per_rank=500, slow_rank=2, unknown_frac=0.2, extra_bins=2)
    stats, _ = _check_window(ctx, win)
    assert stats["n_unknown"] > 0


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scenario", ["healthy", "thermal", "softirq", "dentry-lock", "logging",
                                      "io-bottleneck"])
@pytest.mark.parametrize("seed", [1, 2])
def test_simulator_scenarios_match_reference(ctx, scenario, seed):
    win = ref.simulate(scenario, seed)
    _, rep = _check_window(ctx, win, against_ref=True)
    # DiagnosisReport::to_json (dump(2)) and to_text: the reference's exact bytes
    r, _, _ = ref.window_run(win, want_json=False)
    assert ctx.report_json_text() == r["report_json_raw"]
    assert ctx.report_text() == r["report_text"]
    lab = win.labels
    if seed == 1:
        assert rep["verdict"] == lab["verdict"]


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_simulator_1024_ranks(ctx):
    win = ref.simulate("softirq", 5, ranks=1024, iterations=150)
    _check_window(ctx, win, against_ref=True)


@pytest.mark.parametrize("mode", [0, 1])
def test_resolve_matches_lookup(ctx, mode):
    rng = np.random.default_rng(5)
    from tests.synth import build_id, pack_symr
    n = 5000
    starts = np.unique(rng.integers(0, 1 << 40, size=n).astype(np.uint64))
    sizes = rng.integers(0, 4096, size=len(starts)).astype(np.uint32)
    names = [f"s{i}_{rng.integers(0, 1 << 30)}" for i in range(len(starts))]
    bid = build_id("resolve-test")
    symr = pack_symr(bid, starts, sizes, names)
    ctx.ingest(symr)
    f = so.SymbolFile.parse(symr)
    q = np.concatenate([starts[rng.integers(0, len(starts), 3000)] + rng.integers(0, 5000, 3000).astype(np.uint64),
                        rng.integers(0, 1 << 41, 2000).astype(np.uint64), starts[:10], np.array([0], np.uint64)])
    other = build_id("absent")
    bins = (rng.random(len(q)) < 0.05).astype(np.uint16)
    names_gpu, _ = ctx.resolve(q, bins, np.frombuffer(bid + other, np.uint8))
    repo = so.Repo([symr])
    exp = [repo.resolve_frame(bid if b == 0 else other, int(o), mode).decode() for o, b in zip(q, bins)]
    if mode == 0:
        assert names_gpu == exp
    else:
        names_gpu, _ = ctx.resolve(q, bins, np.frombuffer(bid + other, np.uint8), mode=1)
        assert names_gpu == exp


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,slow", [(7, 3), (4, 1)])
def test_waterline_matches_reference(ctx, seed, slow):
    """compute_waterline + flag_ranks (diagnosis.cpp:35-71) over the window's
    CPU profiles: means/stddevs within 1e-6, flagged (rank, function) exact."""
    win = small_window(seed=seed, ranks=8, samples_per_rank=600, slow_rank=slow)
    ctx.window_run(win, cfg={"want_waterline": 1})
    got = ctx.waterline()
    exp = ref.waterline(win)
    assert [f[0] for f in got["functions"]] == [f[0] for f in exp["functions"]]
    assert_close([f[1:] for f in got["functions"]], [f[1:] for f in exp["functions"]], REL)
    from tests.compare import assert_flags_match
    assert_flags_match(got["flags"], exp["flags"])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_c4_collectives_1024_ranks_match_reference(ctx):
    """C4 shape (1,024 ranks, alternating AllReduce/AllGather, NIC-softirq
    straggler) at 2,000 events per rank: instances, offsets, lateness, the
    straggler and the os-interference verdict exactly as the reference."""
    from tests.synth import c4_window
    win = c4_window(ranks=1024, events_per_rank=2000, seed=3)
    stats, rep = _check_window(ctx, win, against_ref=True)
    assert rep["verdict"] == "os-interference" and rep["flagged_ranks"] == [4]
    assert stats["n_windowed"] > 0


def test_collectives_irregular_streams_match_oracle(ctx):
    """Missing events and late joiners force the sequential greedy fallback."""
    from tests.synth import c4_window
    win = c4_window(ranks=16, events_per_rank=300, seed=5)
    keep = np.ones(len(win.coll_rank), bool)
    rng = np.random.default_rng(1)
    keep[rng.choice(len(keep), 40, replace=False)] = False  # drop events: partial instances
    for f in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur"):
        setattr(win, f, getattr(win, f)[keep])
    _check_window(ctx, win)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scenario,verdict", [("logging", "temporal-degradation"), ("thermal", None)])
def test_c5_4096_ranks_against_baseline(ctx, scenario, verdict):
    """C5: 4,096 ranks compared against the historical
    baseline.  All-rank thermal injection: target_ranks = all; the reference
    concludes `inconclusive` (temporal route is CPU-only) — parity, not the label."""
    win = ref.simulate(scenario, 7, ranks=4096)
    _, rep = _check_window(ctx, win, against_ref=True)
    if verdict:
        assert rep["verdict"] == verdict and len(rep["flagged_ranks"]) == 4096


def test_table_hints_grow_across_windows():
    """Tables sized from the previous window's counts (rank aggregation tables,
    sequence dedupe, prefix cache, unknown labels) must grow by retry when a later
    window needs more: a small window first, then one with 40x the distinct stacks,
    on a fresh context.  Both stay bit-exact against the oracle."""
    import paper_2603_29235_b200 as stg
    c = stg.Context(0)
    try:
        small = small_window(seed=21, ranks=4, samples_per_rank=300, slow_rank=1, pool=10)
        _check_window(c, small)
        big = small_window(seed=22, ranks=12, samples_per_rank=3000, slow_rank=5, pool=400, unknown_frac=0.05)
        stats, _ = _check_window(c, big)
        assert stats["agg_attempts"] > 1, "the aggregation tables should have grown by retry"
        # and shrinking back is exact too (tables larger than needed)
        _check_window(c, small_window(seed=23, ranks=4, samples_per_rank=300, slow_rank=2, pool=10))
    finally:
        c.close()


@pytest.mark.parametrize("depth", [3, 40, 70])
def test_stack_depths_and_alignments(ctx, depth):
    """Frame blocks of 8 are read at absolute alignment: stacks shorter than a block,
    spanning several blocks, and every f0 mod 8 (depths vary per sample) must all
    fold exactly."""
    win = small_window(seed=30 + depth, ranks=6, samples_per_rank=700, slow_rank=2, depth=depth, pool=150)
    _check_window(ctx, win)
