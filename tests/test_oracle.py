"""Pins the oracle (oracle/strata_oracle.py) to the reference.

(1) The reference's own known-answer tests for this path, restated (each cites
    the reference test it restates: proj/tests/test_symbols.cpp,
    test_collector.cpp, test_diagnosis.cpp, acceptance.cpp).
(2) Golden fixtures in tests/golden/ produced by the compiled reference
    (tests/golden/make_golden.py): oracle output must equal them exactly.
(3) When oracle/_ref is built: oracle == reference on simulator windows.
CPU only.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import strata_oracle as so
from oracle.strata_oracle import EXACT_RANGE, NEAREST_LOWER, StrataError

GOLDEN = Path(__file__).resolve().parent / "golden"


def bid(c: str) -> bytes:
    """BuildId::digest(std::string(1, c)) — SHA-1 (build_id.cpp:96-105)."""
    import hashlib
    return hashlib.sha1(c.encode()).digest()


# ------------------------------------------------------------ test_symbols.cpp
def test_pack_parse_round_trip():  # test_symbols.cpp:53-70
    rng = np.random.default_rng(123)
    for trial in range(30):
        n = int(rng.integers(1, 200))
        starts = sorted(set(int(x) for x in rng.integers(0, 1 << 40, n)))
        ents = [(s, int(rng.integers(0, 4097)), "".join(chr(97 + int(c)) for c in rng.integers(0, 26, int(rng.integers(1, 65)))))
                for s in starts]
        b = so.pack_symbols(bid(chr(97 + trial % 26)), ents)
        f = so.SymbolFile.parse(b)
        assert f.build_id == bid(chr(97 + trial % 26))
        assert f.starts == [e[0] for e in ents] and f.sizes == [e[1] for e in ents]
        assert [n.decode() for n in f.names] == [e[2] for e in ents]
        assert so.pack_symbols(f.build_id, list(zip(f.starts, f.sizes, f.names))) == b


def test_pack_rejects():  # test_symbols.cpp:72-78
    with pytest.raises(StrataError):
        so.pack_symbols(bid("p"), [(0x10, 4, "a"), (0x10, 4, "b")])
    with pytest.raises(StrataError):
        so.pack_symbols(bid("p"), [(0x10, 4, "")])
    with pytest.raises(StrataError):
        so.pack_symbols(bid("p"), [(0x10, 4, "x" * 70000)])


def test_parse_rejects_corruption():  # test_symbols.cpp:80-101
    good = so.pack_symbols(bid("q"), [(0x10, 4, "a"), (0x20, 4, "b")])
    so.parse_symbols(good)

    def corrupt(i, v):
        b = bytearray(good)
        b[i] = v
        return bytes(b)

    for bad, msg in ((corrupt(0, ord("X")), "symbol file bad magic"),
                     (corrupt(4, 99), "unsupported symbol file version 99"),
                     (corrupt(28, 77), "symbol file bad string-table offset"),
                     (good[:20], "symbol file truncated header"),
                     (b"", "symbol file truncated header")):
        with pytest.raises(StrataError, match=msg):
            so.parse_symbols(bad)
    swapped = bytearray(good)
    swapped[36:52], swapped[52:68] = good[52:68], good[36:52]
    with pytest.raises(StrataError, match="not strictly sorted"):
        so.parse_symbols(bytes(swapped))


def test_lookup_modes():  # test_symbols.cpp:103-122
    f = so.SymbolFile(bid("l"), [0x100, 0x200, 0x300], [0x40, 0, 0x40], [b"f", b"marker", b"g"])
    E, N = EXACT_RANGE, NEAREST_LOWER
    assert f.lookup(0x100, E) == b"f" and f.lookup(0x13F, E) == b"f"
    assert f.lookup(0x140, E) is None and f.lookup(0x0FF, E) is None
    assert f.lookup(0x200, E) == b"marker" and f.lookup(0x201, E) is None
    assert f.lookup(0x140, N) == b"f" and f.lookup(0x2FF, N) == b"marker"
    assert f.lookup(0x10000, N) == b"g" and f.lookup(0x0FF, N) is None


def test_lookup_probe_bound():  # test_symbols.cpp:124-142
    for n in (1, 1000, 50_000):
        f = so.SymbolFile(bid("b"), [i * 64 for i in range(n)], [64] * n, [b"s"] * n)
        bound = 1 if n == 1 else math.ceil(math.log2(n)) + 1
        rng = np.random.default_rng(5)
        worst = max(f.lookup_index(int(x), EXACT_RANGE)[1] for x in rng.integers(0, n * 64, 2000))
        assert worst <= bound


def test_unknown_label():  # test_symbols.cpp:144-148
    assert so.unknown_frame_label(bid("u"), 0x1A2B) == b"[" + bid("u").hex().encode() + b"+0x1a2b]"


def test_resolve_falls_back_to_labels():  # test_symbols.cpp:209-222
    known, unknown = bid("k"), bid("z")
    repo = so.Repo([so.pack_symbols(known, [(0x100, 0x40, "f")])])
    names = repo.resolve_stack([(known, 0x110), (known, 0x900), (unknown, 0x10)], EXACT_RANGE)
    assert names == [b"f", so.unknown_frame_label(known, 0x900), so.unknown_frame_label(unknown, 0x10)]


# ---------------------------------------------------------- test_collector.cpp
def _smp(ts, offs, rank=0):
    return (ts, rank, tuple((bid("a"), o) for o in offs))


def test_aggregation_lossless():  # test_collector.cpp:43-56
    stream = [_smp(i * 100_000_000, [8, 16] if i % 3 == 0 else [8, 24]) for i in range(10)]
    w = so.aggregate_samples(stream)
    assert len(w) == 1 and len(w[0][2]) == 2
    assert sum(c for _, c in w[0][2]) == 10 and w[0][0] == 0 and w[0][1] == 5_000_000_000


def test_aggregation_grid():  # test_collector.cpp:58-71
    w = so.aggregate_samples([_smp(4_999_999_999, [8]), _smp(5_000_000_000, [8]), _smp(17_000_000_000, [8])])
    assert [x[0] for x in w] == [0, 5_000_000_000, 15_000_000_000]


def test_aggregation_validation():  # test_collector.cpp:73-82
    assert so.aggregate_samples([]) == []
    for bad in ([_smp(0, [8], 0), _smp(1, [8], 1)], [_smp(10, [8]), _smp(5, [8])], [_smp(0, [])]):
        with pytest.raises(StrataError):
            so.aggregate_samples(bad)
    with pytest.raises(StrataError):
        so.aggregate_samples([_smp(0, [8])], 0)


def test_folded_output_and_fractions():  # test_collector.cpp:101-122
    a = bid("a")
    repo = so.Repo([so.pack_symbols(a, [(0, 8, "main"), (8, 8, "leafA"), (16, 8, "work"), (24, 8, "leafB")])])
    f = so.to_folded([(0, 0, [(((a, 8), (a, 0)), 2), (((a, 24), (a, 16), (a, 0)), 1)])], repo, EXACT_RANGE)
    assert f.total == 3 and f.to_string() == "main;leafA 2\nmain;work;leafB 1\n"
    fr = f.inclusive_fractions()
    assert fr[b"main"] == 1.0
    assert fr[b"leafA"] == pytest.approx(2 / 3) and fr[b"work"] == pytest.approx(1 / 3)


def test_recursion_counts_once():  # test_collector.cpp:124-130
    fr = so.fold_symbolized([(["f", "f", "main"], 3), (["g", "main"], 1)]).inclusive_fractions()
    assert fr[b"f"] == pytest.approx(0.75) and fr[b"main"] == 1.0


def test_diff_folded():  # test_collector.cpp:132-137
    a = so.fold_symbolized([(["x", "main"], 4)])
    b = so.fold_symbolized([(["x", "main"], 1), (["y", "main"], 2)])
    assert so.diff_folded(a, b) == "main;x 4 1\nmain;y 0 2\n"


def test_matching_groups_instances():  # test_collector.cpp:139-158
    ev = [(r, 0, 0, 1_000_000 * it + 1_000 * r, 1_000_000 * it + 1_000 * r + 400_000)
          for it in range(5) for r in (0, 1, 2)]
    inst = so.match_collectives(ev, [0, 1, 2])
    assert len(inst) == 5 and all(not i.partial and len(i.events) == 3 for i in inst)
    for k, i in enumerate(inst):
        assert all(e[0] == 1_000_000 * k + 1_000 * r for r, e in i.events.items())


def test_matching_constant_shift():  # test_collector.cpp:160-173
    ev = []
    for it in range(4):
        b = 1_000_000 * it
        ev += [(0, 0, 0, b, b + 400_000), (1, 0, 0, b + 400_000_000, b + 400_400_000)]
    inst = so.match_collectives(ev, [0, 1])
    assert len(inst) == 4 and not any(i.partial for i in inst)


def test_partial_instance():  # test_collector.cpp:175-183
    inst = so.match_collectives([(0, 0, 0, 0, 400_000), (1, 0, 0, 1_000, 401_000)], [0, 1, 2])
    assert len(inst) == 1 and inst[0].partial and len(inst[0].events) == 2
    with pytest.raises(StrataError):
        so.entry_lateness(inst[0], {})


def test_matching_validation():  # test_collector.cpp:185-190
    with pytest.raises(StrataError):
        so.match_collectives([(0, 0, 0, 100, 100)], [0])
    with pytest.raises(StrataError):
        so.match_collectives([(0, 0, 0, 1_000_000, 1_400_000), (0, 0, 0, 0, 400_000)], [0])


def test_clock_alignment():  # test_collector.cpp:192-214
    skew = {0: -3_000_000, 1: 0, 2: 7_500_000}
    rng = np.random.default_rng(17)
    ev = []
    for it in range(101):
        te = 10_000_000 * (it + 1)
        for r, s in skew.items():
            ev.append((r, 0, 0, te - 500_000 + s, te + s + int(rng.integers(-50_000, 50_001))))
    off = so.align_clocks(so.match_collectives(ev, [0, 1, 2]))
    for r, s in skew.items():
        assert abs(off[r] - (s - 7_500_000)) <= 150_000
    assert so.align_clocks([]) is None


def test_entry_lateness():  # test_collector.cpp:216-235
    inst = so.Instance(0, 0, {r: (1_000_000 + (600_000 if r == 5 else 0), 1_400_000) for r in range(8)})
    lat = so.entry_lateness(inst, {})
    assert lat[0] == 0.0 and lat[5] == pytest.approx(0.6)
    sh = so.Instance(0, 0, {r: (e + 5_000_000, x + 5_000_000) for r, (e, x) in inst.events.items()})
    assert so.entry_lateness(sh, {}) == lat


# ---------------------------------------------------------- test_diagnosis.cpp
def _uniform(leaves):
    return so.fold_symbolized([([leaf, "main"], c) for leaf, c in leaves.items()])


def test_waterline_shift():  # test_diagnosis.cpp:20-40, acceptance c3
    for n in (2, 8, 64):
        per = {r: _uniform({"hot": 30 if r == 0 else 10, "base": 90}) for r in range(n)}
        wl = so.compute_waterline(per)
        exp = 0.1 + (30 / 120 - 0.1) / n
        assert abs(wl[b"hot"][0] - exp) < 1e-12
        assert wl[b"main"] == (1.0, 0.0)
    with pytest.raises(StrataError):
        so.compute_waterline({0: _uniform({"a": 1})})


def test_waterline_absent_zero():  # test_diagnosis.cpp:42-48
    wl = so.compute_waterline({0: _uniform({"only_here": 50, "shared": 50}), 1: _uniform({"shared": 100})})
    assert wl[b"only_here"][0] == pytest.approx(0.25)


def test_flag_strict():  # test_diagnosis.cpp:50-68
    per = {0: _uniform({"hot": 40, "base": 60})}
    per.update({r: _uniform({"hot": 10, "base": 90}) for r in range(1, 8)})
    flags = [(r, n) for r, n, _, _ in so.flag_ranks(so.compute_waterline(per), per) if n == b"hot"]
    assert flags == [(0, b"hot")]
    flat = {r: _uniform({"f": 10}) for r in range(4)}
    assert so.flag_ranks(so.compute_waterline(flat), flat) == []


def test_two_outliers_need_looser_k():  # test_diagnosis.cpp:70-88
    per = {r: _uniform({"hot": 30 if r < 2 else 10, "base": 90}) for r in range(8)}
    for k, want in ((2.0, 0), (1.0, 2)):
        wl = so.compute_waterline(per, k)
        assert sum(1 for f in so.flag_ranks(wl, per, k) if f[1] == b"hot") == want


def test_straggler_brute_force():  # test_diagnosis.cpp:90-119, acceptance c2
    inst = {r: 0.6 if r == 3 else 0.0 for r in range(8)}
    mu = 0.6 / 8
    sigma = math.sqrt((7 * mu * mu + (0.6 - mu) ** 2) / 8)
    a = so.detect_straggler([dict(inst) for _ in range(10)])
    assert len(a) == 1 and a[0].rank == 3 and a[0].flagged_instances == 10
    assert a[0].mean_lateness_ms == pytest.approx(0.6)
    assert abs(a[0].z_score - (0.6 - mu) / sigma) < 1e-9
    b = so.detect_straggler([{r: l + 5.0 for r, l in inst.items()} for _ in range(10)])
    assert b[0].rank == 3 and abs(b[0].z_score - a[0].z_score) < 1e-9


def test_straggler_persistence():  # test_diagnosis.cpp:121-134
    late = {r: 0.6 if r == 3 else 0.0 for r in range(8)}
    quiet = {r: 0.0 for r in range(8)}
    half = [late] * 5 + [quiet] * 5
    assert so.detect_straggler(half) == []
    a = so.detect_straggler(half + [late])
    assert len(a) == 1 and a[0].flagged_instances == 6


CFG = None


def _cfg():
    from paper_2603_29235_b200.abi import default_config
    return default_config()


def test_gpu_diff_cases():  # test_diagnosis.cpp:136-186
    ref = {"matmul": 800_000_000, "softmax": 300_000_000, "dropout": 200_000_000,
           "nccl_all_reduce": 900_000_000, "tiny": 500_000}
    s = {k: (int(v * 1.10) if k not in ("nccl_all_reduce", "tiny") else v) for k, v in ref.items()}
    v, slow, _ = so.gpu_diff(s, ref, _cfg())
    assert v == 1 and "nccl_all_reduce" not in slow and "tiny" not in slow
    s = dict(ref, matmul=1_600_000_000, softmax=312_000_000, dropout=206_000_000)
    v, _, top = so.gpu_diff(s, ref, _cfg())
    assert v == 2 and top == "matmul"
    assert so.gpu_diff(dict(ref, matmul=1_600_000_000), ref, _cfg())[0] == 0
    assert so.gpu_diff(ref, ref, _cfg())[0] == 0
    assert so.gpu_diff({}, ref, _cfg()) == (0, {}, "")


def test_cpu_diff_ties_and_paths():  # test_diagnosis.cpp:188-213
    s = so.fold_symbolized([(["spin_lock", "open", "main"], 30), (["read", "open", "main"], 10), (["compute", "main"], 60)])
    r = so.fold_symbolized([(["read", "open", "main"], 10), (["compute", "main"], 90)])
    d = so.cpu_diff(s, r, 0.005)
    assert [x[0] for x in d] == [b"open", b"spin_lock"]
    assert d[0][3] == pytest.approx(0.3)
    assert d[0][4] == d[1][4] == [b"main", b"open", b"spin_lock"]
    assert so.cpu_diff(r, r, 0.005) == []


def test_os_diff():  # test_diagnosis.cpp:215-245
    ref = {"interrupts": {"eth0": 2000}, "softirqs": {"NET_RX": 5000, "TIMER": 10000}, "p99": 400_000, "migrations": 0}
    s = {"interrupts": {"eth0": 16000}, "softirqs": {"NET_RX": 50000, "TIMER": 10500, "NEW_TYPE": 4000},
         "p99": 2_400_000, "migrations": 0}
    d = so.os_diff(s, ref, _cfg())
    assert len(d) == 4 and any(x[0] == "softirq:NEW_TYPE" and x[4] for x in d)
    assert all(x[0] != "softirq:TIMER" for x in d)
    z = {"interrupts": {}, "softirqs": {}, "p99": 0, "migrations": 0}
    assert so.os_diff(dict(z, interrupts={"x": 100}), dict(z, interrupts={"x": 10}), _cfg()) == []


def test_temporal_one_sided():  # test_diagnosis.cpp:247-263
    now = so.fold_symbolized([(["compute", "main"], 84), (["log", "main"], 4), (["new_path", "main"], 12)])
    c = so.temporal_diff(now, {b"main": 1.0, b"compute": 0.9, b"log": 0.01}, 0.005)
    assert [x[0] for x in c] == [b"new_path", b"log"] and c[0][2] == 0.0 and c[1][3] == pytest.approx(0.03)


def _gd(**kw):
    gd = {"group": 0, "cpu_profiles": {}, "gpu_profiles": {}, "os_snapshots": {}, "lateness_per_instance": [],
          "iteration_times_ms": [], "baseline": None, "baseline_iteration_ms": None}
    gd.update(kw)
    return gd


def test_diagnose_layer_routing():  # test_diagnosis.cpp:265-318
    inst = {r: 2.0 if r == 1 else 0.0 for r in range(8)}
    z = {"interrupts": {}, "softirqs": {}, "p50": 0, "p99": 0, "migrations": 0}
    base = dict(lateness_per_instance=[dict(inst) for _ in range(10)],
                gpu_profiles={r: {"matmul": 100_000_000} for r in range(8)},
                os_snapshots={r: dict(z) for r in range(8)},
                cpu_profiles={r: so.fold_symbolized([(["compute", "main"], 95)]) for r in range(8)})
    cp = dict(base["cpu_profiles"])
    cp[1] = so.fold_symbolized([(["compute", "main"], 80), (["spin", "sys", "main"], 20)])
    rep = so.diagnose(_gd(**dict(base, cpu_profiles=cp)))
    assert rep["verdict"] == "cpu-interference" and rep["flagged_ranks"] == [1]
    assert rep["reference_rank"] != 1 and rep["top_path"] == ["main", "sys", "spin"]
    gp = dict(base["gpu_profiles"])
    gp[1] = {"matmul": 118_000_000}
    assert so.diagnose(_gd(**dict(base, cpu_profiles=cp, gpu_profiles=gp)))["verdict"] == "gpu-uniform-slowdown"
    osn = {r: dict(z, softirqs={"NET_RX": 50_000 if r == 1 else 5_000}) for r in range(8)}
    assert so.diagnose(_gd(**dict(base, os_snapshots=osn)))["verdict"] == "os-interference"
    assert so.diagnose(_gd(**base))["verdict"] == "inconclusive"


def test_diagnose_temporal_gate():  # test_diagnosis.cpp:320-355
    cpu = {r: so.fold_symbolized([(["compute", "main"], 93), (["new_logging", "main"], 7)]) for r in range(4)}
    kw = dict(lateness_per_instance=[{r: 0.0 for r in range(4)}] * 10, cpu_profiles=cpu,
              baseline={"delta": 0.005, "fractions": {"main": 1.0, "compute": 1.0}}, baseline_iteration_ms=100.0)
    rep = so.diagnose(_gd(iteration_times_ms=[108.0] * 100, **kw))
    assert rep["verdict"] == "temporal-degradation" and rep["flagged_ranks"] == [0, 1, 2, 3]
    assert rep["top_path"] == ["main", "new_logging"]
    assert so.diagnose(_gd(iteration_times_ms=[101.0] * 100, **kw))["verdict"] == "healthy"
    kw["cpu_profiles"] = {r: so.fold_symbolized([(["compute", "main"], 100)]) for r in range(4)}
    assert so.diagnose(_gd(iteration_times_ms=[108.0] * 100, **kw))["verdict"] == "inconclusive"


# ------------------------------------------------------------- golden fixtures
def _load_fixture(path):
    from paper_2603_29235_b200.abi import Window
    d = json.loads(path.read_text())
    w = Window()
    for k, v in d["window"].items():
        if k in ("symr",):
            w.symr = [bytes.fromhex(x) for x in v]
        elif k in ("kernel_names", "counter_names", "baseline", "baseline_iteration_ms", "has_baseline",
                   "baseline_delta", "window_start_ns", "window_end_ns", "max_skew_ns", "group"):
            setattr(w, k, v)
        else:
            dt, vals = v
            setattr(w, k, np.asarray(vals, dtype=dt))
    w.bin_build_ids = w.bin_build_ids.reshape(-1, 20)
    return w, d["expected"]


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.json")), ids=lambda p: p.stem)
def test_golden_fixture(path):
    """Reference outputs captured by tests/golden/make_golden.py."""
    w, exp = _load_fixture(path)
    gd, rep = so.window_pipeline(w)
    assert gd == exp["groupdata"]
    assert rep == exp["report"]


def test_golden_fixtures_exist():
    assert len(list(GOLDEN.glob("*.json"))) >= 3


# ------------------------------------------------ live reference (if compiled)
@pytest.mark.parametrize("scenario", ["healthy", "thermal", "softirq", "dentry-lock", "logging", "io-bottleneck"])
def test_oracle_equals_reference_on_simulator(scenario):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = ref.simulate(scenario, 2)
    r, _, _ = ref.window_run(w)
    gd, rep = so.window_pipeline(w)
    assert gd == r["groupdata"] and rep == r["report"]


def test_oracle_equals_reference_on_synthetic():
    from oracle import ref
    from tests.synth import small_window
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for seed, slow in ((3, 2), (9, -1)):
        w = small_window(seed=seed, ranks=6, samples_per_rank=300, slow_rank=slow, unknown_frac=0.1, extra_bins=1)
        r, _, _ = ref.window_run(w)
        gd, rep = so.window_pipeline(w)
        assert gd == r["groupdata"] and rep == r["report"]


@pytest.mark.parametrize("scenario", ["softirq", "dentry-lock"])
def test_oracle_text_artifacts_equal_reference(scenario):
    """FoldedProfile::to_string and diff_folded texts (folded.cpp:33-43, 83-96)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = ref.simulate(scenario, 3)
    r, _, _ = ref.window_run(w, artifacts=True)
    gd = so.build_group_data(w)
    prof = gd["cpu_profiles"]
    art = r["artifacts"]
    assert [x[0] for x in art["folded"]] == sorted(prof)
    for rank, text in art["folded"]:
        assert prof[rank].to_string() == text
    assert art["diffs"]
    for a, b, text in art["diffs"]:
        assert so.diff_folded(prof[a], prof[b]) == text


@pytest.mark.parametrize("seed,drain", [(1, 5_000_000_000), (2, 1_000_000_000), (3, 7), (4, 10**15)])
def test_oracle_aggregate_samples_equals_reference(seed, drain):
    """aggregate_samples (samples.cpp:31-85): windows, first-seen record order, counts."""
    from oracle import ref
    from tests.synth import oracle_stream, raw_stream
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    ts, rk, off, pc, bn, ids = raw_stream(seed=seed, n=1500, t0=-4_000_000_123 if seed == 2 else 3_000_000_000)
    got = ref.aggregate_samples(ts, off, pc, bn, ids, rank=rk, drain=drain)
    stream = oracle_stream(ts, rk, off, pc, bn, ids)
    exp = so.aggregate_samples(stream, drain)
    assert [(g[1], g[2]) for g in got] == [(e[0], e[1]) for e in exp]
    for g, e in zip(got, exp):
        assert [c for _, c in g[3]] == [c for _, c in e[2]]
        assert [stream[f][2] for f, _ in g[3]] == [fr for fr, _ in e[2]]


def test_lookup_matches_reference_probes():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(9)
    starts = sorted(set(int(x) for x in rng.integers(0, 1 << 40, 500)))
    ents = [(s, int(rng.integers(0, 4096)), f"n{i}") for i, s in enumerate(starts)]
    b = so.pack_symbols(bid("r"), ents)
    assert ref.pack_symbols(bid("r"), ents) == b
    q = np.concatenate([rng.integers(0, 1 << 41, 3000), np.array(starts[:50])]).astype(np.uint64)
    f = so.SymbolFile.parse(b)
    for mode in (EXACT_RANGE, NEAREST_LOWER):
        idx, probes = ref.lookup(b, q, mode)
        mine = [f.lookup_index(int(x), mode) for x in q]
        assert [(-1 if i is None else i) for i, _ in mine] == idx.tolist()
        assert [p for _, p in mine] == probes.tolist()


@pytest.mark.skipif(not (Path(__file__).parent.parent / "oracle/_ref/libstrata_ref.so").exists(),
                    reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [3, 8])
def test_shared_cache_harness_equals_to_folded(seed):
    """The C2-scale parity tests symbolize the reference's records with its own
    resolve_stacks + fold_symbolized (one table cache per rank) instead of
    to_folded's per-record table reload: the GroupData and report must be
    identical to the as-is build_group_data."""
    from oracle import ref
    from tests.synth import small_window
    win = small_window(seed=seed, ranks=5, samples_per_rank=700, slow_rank=2, unknown_frac=0.05, extra_bins=1)
    a, _, _ = ref.window_run(win)
    b, _, _ = ref.window_run(win, threads=3, shared_cache=True)
    assert a == b


def test_c2_host_generator_shapes():
    """tests/synth.c2_samples_host (the reference arm's numpy C2 generator):
    shapes, per-rank time order, bins by level, the straggler's softirq leaf path."""
    from tests.synth import SOFTIRQ, c2_samples_host
    rng = np.random.default_rng(0)
    nsym = 5000
    tabs = []
    for b in range(3):
        sizes = rng.integers(16, 4096, nsym).astype(np.uint32)
        starts = (0x10000 + np.concatenate([[0], np.cumsum(sizes.astype(np.uint64) + 8)[:-1]])).astype(np.uint64)
        tabs.append((starts, sizes))
    cdf = np.cumsum(np.arange(1, 101, dtype=np.float64) ** -1.1)
    cdf /= cdf[-1]
    soft = tabs[2][0][:9] + 4
    ts, off, pc, bn = c2_samples_host(7, 3, 400, 64, 100, cdf, tabs, (nsym,) * 3, soft, 1, 0.3, 1000, 10_000,
                                      np.array([5, -3, 0]))
    assert len(ts) == 1200 and len(off) == 1201 and len(pc) == 1200 * 64 == len(bn)
    assert all(np.all(np.diff(ts[r * 400:(r + 1) * 400]) > 0) for r in range(3))
    b = bn.reshape(1200, 64)
    assert set(np.unique(b[:, 63])) == {0} and set(np.unique(b[:, 30])) == {1}  # root python, middle libtorch
    p = pc.reshape(1200, 64)
    soft_rows = np.all(p[:, :9][:, ::-1] == soft[None, :], axis=1)
    assert soft_rows[400:800].mean() > 0.15 and not soft_rows[:400].any() and not soft_rows[800:].any()
    assert len(SOFTIRQ) == 9
