"""GPU parity of the output artifacts:
stg_result_folded_text = FoldedProfile::to_string (folded.cpp:33-43),
stg_result_diff_folded = diff_folded (folded.cpp:83-96), rendered on the device,
and the flame graphs stg_result_(diff_)flamegraph_svg = render_flamegraph /
render_diff_flamegraph (svg.cpp:157-172), against the reference's own texts
(oracle/_ref) and the oracle restatement.
Text is bytes: the bar is exact equality.
"""
import pytest

import paper_2603_29235_b200 as stg
from oracle import ref, strata_oracle as so
from tests.synth import small_window

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scenario", ["healthy", "softirq", "dentry-lock", "logging"])
def test_artifacts_match_reference(ctx, scenario):
    win = ref.simulate(scenario, 2)
    r, _, _ = ref.window_run(win, artifacts=True)
    ctx.window_run(win)
    art = r["artifacts"]
    for rank, text in art["folded"]:
        assert ctx.folded_text(rank) == text, rank
    for a, b, text in art["diffs"]:
        assert ctx.diff_folded(a, b) == text, (a, b)
    for rank, svg in art["svg"]:
        assert ctx.flamegraph_svg(rank, title=f"rank {rank}") == svg, rank
    for a, b, svg in art["svg_diffs"]:
        assert ctx.diff_flamegraph_svg(a, b, title=f"rank {a} vs rank {b}") == svg, (a, b)


def test_artifacts_with_unknown_labels_match_oracle(ctx):
    win = small_window(seed=11, ranks=6, samples_per_rank=500, slow_rank=2, unknown_frac=0.2, extra_bins=2)
    stats = ctx.window_run(win)
    assert stats["n_unknown"] > 0
    prof = so.build_group_data(win)["cpu_profiles"]
    ranks = sorted(prof)
    for rk in ranks:
        assert ctx.folded_text(rk) == prof[rk].to_string()
    for a in ranks[:3]:
        for b in ranks[:3]:
            assert ctx.diff_folded(a, b) == so.diff_folded(prof[a], prof[b])


def test_unknown_rank_is_refused(ctx):
    win = small_window(seed=3, ranks=4, samples_per_rank=200, slow_rank=-1)
    ctx.window_run(win)
    with pytest.raises(stg.StgError, match="unknown rank id: 999"):
        ctx.folded_text(999)
    with pytest.raises(stg.StgError, match="unknown rank id: 77"):
        ctx.diff_folded(0, 77)
    with pytest.raises(stg.StgError, match="unknown rank id: 5"):
        ctx.flamegraph_svg(5)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_flamegraphs_c1_scale_match_reference(ctx):
    """Deep, wide profiles (2k distinct stacks per rank, unknown labels, elided
    narrow frames) render to the reference's exact SVG bytes."""
    win = small_window(seed=2, ranks=4, samples_per_rank=30_000, slow_rank=1, depth=12, n_sym=2000, pool=2000,
                       unknown_frac=0.02)
    r, _, _ = ref.window_run(win, artifacts=True)
    ctx.window_run(win)
    art = r["artifacts"]
    assert art["svg"] and art["svg_diffs"]
    for rank, svg in art["svg"]:
        assert ctx.flamegraph_svg(rank, title=f"rank {rank}") == svg, rank
    for a, b, svg in art["svg_diffs"]:
        assert ctx.diff_flamegraph_svg(a, b, title=f"rank {a} vs rank {b}") == svg, (a, b)


def test_artifacts_large_window_properties(ctx):
    """At a size the oracle would take minutes on: line structure and count
    conservation — Σ counts of to_string = the rank's total, diff(a, a) repeats
    each count twice, diff(a, b) has union-many lines whose count columns
    reproduce both to_string texts."""
    win = small_window(seed=5, ranks=16, samples_per_rank=40_000, slow_rank=7, unknown_frac=0.05, extra_bins=1)
    ctx.window_run(win)
    folded = ctx.folded()
    a, b = sorted(folded)[:2]

    def parse(text, ncol):
        out = []
        for line in text.splitlines():
            parts = line.rsplit(" ", ncol)
            out.append((parts[0], tuple(int(x) for x in parts[1:])))
        return out

    ta = parse(ctx.folded_text(a), 1)
    tb = parse(ctx.folded_text(b), 1)
    assert sum(c for _, (c,) in ta) == folded[a][0]
    assert [";".join(n) for n, _ in folded[a][1]] == [k for k, _ in ta]
    same = parse(ctx.diff_folded(a, a), 2)
    assert [(k, (c, c)) for k, (c,) in ta] == same
    d = parse(ctx.diff_folded(a, b), 2)
    assert len(d) == len({k for k, _ in ta} | {k for k, _ in tb})
    assert [(k, (ca,)) for k, (ca, _) in d if ca] == ta
    assert [(k, (cb,)) for k, (_, cb) in d if cb] == tb
