"""GPU parity at the MEASURED configurations, against the
compiled reference (oracle/_ref) on identical inputs.

  C2  bench generator + c2_tables (3 x 1M-symbol tables, 64-frame stacks), at
      reduced ranks, both the bench's hot-function set and all functions hot;
      the reference symbolizes through its own resolve_stacks (one table cache
      per rank, symrepo.cpp:122-143) + fold_symbolized — the same folded
      profiles as to_folded, which would re-parse a 1M-entry table per record.
  C1  8 ranks x 100k samples, 10k-symbol table, 2k distinct stacks (Zipf).
  C3  simulate() at 1,024 ranks x 300 iterations, six scenarios x seeds, plus
      a C1-style 200-distinct-stack variant at 1,024 ranks.
  C4  1,024 ranks x 50k collective events.
Plus the fingerprint-safety cases: planted pc = B ^ K frames (the round-1
prefix-key annihilator) and forced prefix-key collisions caught by verify mode.

Bar: GroupData and report bit-exact (floats within 1e-6 relative where the
reference's own summation order is not reproduced, i.e. the GroupData's
fractions-free fields are exact; see test_gpu_parity._check_window).
"""
import types

import numpy as np
import pytest

from oracle import ref, strata_oracle as so
from tests.compare import assert_close
from tests.synth import c4_window, small_window

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]
REL = 1e-6


def _compare(ctx, win, cfg=None, ref_threads=8, shared_cache=False, oracle=False):
    stats = ctx.window_run(win, cfg=cfg)
    gd, rep = ctx.groupdata(), ctx.report()
    if oracle:
        ogd, orep = so.window_pipeline(win)
    else:
        r, _, _ = ref.window_run(win, threads=ref_threads, shared_cache=shared_cache)
        ogd, orep = r["groupdata"], r["report"]
    assert gd["cpu_profiles"] == ogd["cpu_profiles"]
    assert gd["gpu_profiles"] == ogd["gpu_profiles"]
    assert gd["os_snapshots"] == ogd["os_snapshots"]
    assert gd["lateness_per_instance"] == ogd["lateness_per_instance"]
    assert gd["iteration_times_ms"] == ogd["iteration_times_ms"]
    assert_close(gd, ogd, REL)
    assert_close(rep, orep, 0.0)
    return stats, rep


# ----------------------------------------------------------------------- C2
def _c2_workload(ranks, spr, hot):
    import bench
    a = types.SimpleNamespace(ranks=ranks, spr=spr, depth=64, pool=50_000, nsym=1_000_000, seed=42, hot=hot)
    return bench.Workload(a, 0, 1)


@pytest.fixture(scope="module")
def c2_small():
    return _c2_workload(4, 2000, "bench")


def test_c2_host_generator_matches_device(c2_small):
    """bench.py's reference arm generates its inputs with numpy (no repo .so):
    bit-identical to the CUDA bench generator."""
    import torch
    wl = c2_small
    for seed_off, period in ((0, 0), (17, 123_457)):
        dev = [t.cpu().numpy() for t in wl.generate(torch, 4, 2000, seed_off=seed_off, period=period)]
        host = wl.generate_host(4, 2000, seed_off=seed_off, period=period)
        assert np.array_equal(dev[0], host[0])
        assert np.array_equal(dev[1].view(np.uint64), host[1])
        assert np.array_equal(dev[2].view(np.uint64), host[2])
        assert np.array_equal(dev[3].view(np.uint16), host[3])


@pytest.mark.parametrize("hot,ranks,spr", [("bench", 4, 200_000), ("all", 4, 100_000)])
def test_c2_shape_matches_reference(ctx, hot, ranks, spr):
    """The headline workload's shape: 1M-entry bucket-indexed tables, 64-deep
    tree-structured stacks, prefix-cache hits, JIT unknown leaves, a straggler —
    device-resident inputs exactly as bench.py runs them, verify mode on."""
    import torch
    from paper_2603_29235_b200.abi import STG_MEM_DEVICE, STG_MEM_HOST
    wl = _c2_workload(ranks, spr, hot)
    arrays = wl.generate(torch, ranks, spr)
    win = wl.window(ranks, spr, arrays, STG_MEM_DEVICE)
    stats = ctx.window_run(win, cfg={"verify": 1, "want_waterline": 1})
    assert stats["verified"] == 1 and stats["verify_retries"] == 0
    assert stats["prefix_hits"] > 0                        # the cache is exercised
    assert stats["n_unknown"] > 0                          # JIT leaves
    gd, rep = ctx.groupdata(), ctx.report()
    host = (arrays[0].cpu().numpy(), arrays[1].cpu().numpy().view(np.uint64),
            arrays[2].cpu().numpy().view(np.uint64), arrays[3].cpu().numpy().view(np.uint16))
    del arrays
    hwin = wl.window(ranks, spr, host, STG_MEM_HOST)
    r, _, _ = ref.window_run(hwin, threads=ranks, shared_cache=True)
    assert gd["cpu_profiles"] == r["groupdata"]["cpu_profiles"]
    assert gd["gpu_profiles"] == r["groupdata"]["gpu_profiles"]
    assert gd["os_snapshots"] == r["groupdata"]["os_snapshots"]
    assert gd["lateness_per_instance"] == r["groupdata"]["lateness_per_instance"]
    assert_close(rep, r["report"], 0.0)
    # the same window through host buffers (the e2e path) gives the same result
    ctx.window_run(hwin, cfg={"want_waterline": 1})
    assert ctx.groupdata()["cpu_profiles"] == gd["cpu_profiles"]


# ----------------------------------------------------------------------- C1
def test_c1_full_scale_matches_reference(ctx):
    """8 ranks x 100k samples, 10k symbols, 2k distinct stacks."""
    win = small_window(seed=1, ranks=8, samples_per_rank=100_000, slow_rank=4, depth=12, n_sym=10_000, pool=2000)
    stats, rep = _compare(ctx, win, cfg={"verify": 1}, ref_threads=8)
    assert stats["verified"] == 1
    assert rep["verdict"] == "cpu-interference" and rep["flagged_ranks"] == [4]


# ----------------------------------------------------------------------- C3
@pytest.mark.parametrize("scenario", ["healthy", "thermal", "softirq", "dentry-lock", "logging", "io-bottleneck"])
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_c3_1024_ranks_matches_reference(ctx, scenario, seed):
    """§8(d) C3: simulate(default_spec(s, seed)) at 1,024 ranks x 300 iterations."""
    win = ref.simulate(scenario, seed, ranks=1024, iterations=300)
    _, rep = _compare(ctx, win)
    if seed == 1:
        assert rep["verdict"] == win.labels["verdict"]


def test_c3_rich_cpu_profiles_1024_ranks(ctx):
    """The richer C3 variant: C1-style CPU profiles (200 distinct stacks/rank) at 1,024 ranks."""
    win = small_window(seed=5, ranks=1024, samples_per_rank=3000, slow_rank=17, depth=12, n_sym=10_000, pool=200)
    _compare(ctx, win, cfg={"verify": 1}, ref_threads=16)


# ----------------------------------------------------------------------- C4
def test_c4_full_matches_reference(ctx):
    """§8(d) C4: 1,024 ranks x 50k AllReduce/AllGather events (51.2 M), NIC-softirq
    straggler; the reference takes ~1 min on one core."""
    win = c4_window(ranks=1024, events_per_rank=50_000, seed=1)
    stats, rep = _compare(ctx, win, ref_threads=1)
    assert stats["n_windowed"] > 0 and rep["flagged_ranks"] == [4]


# -------------------------------------------------------- fingerprint safety
def _same_leaf(w):
    """frame_pc with every sample's leaf set to the first sample's leaf: a wrong
    chain then shows up as a merged line (a differing leaf would give the sample
    a fingerprint of its own, re-materialised under its true names)."""
    off = np.asarray(w.sample_frame_off, np.uint64)
    pc = np.asarray(w.frame_pc, np.uint64).copy()
    bn = np.asarray(w.frame_bin, np.uint16).copy()
    leaf = off[:-1].astype(np.int64)
    pc[leaf] = pc[leaf[0]]
    bn[leaf] = bn[leaf[0]]
    w.frame_bin = bn
    return pc


def _annihilator_window(seed=21):
    """A C1 window in which every sample plants, at one non-leaf frame pair
    (slots 2m, 2m+1 of an aligned 8-frame block), pc = B(q) ^ K(slot) — the value
    that zeroed the round-1 block product — and draws the partner frame from two
    different functions.  Chains differing only in the partner must still fold
    under their own names (the reference full-compares, samples.cpp:67-76)."""
    w = small_window(seed=seed, ranks=4, samples_per_rank=60_000, slow_rank=-1, depth=12, n_sym=2000, pool=30)
    K = [0x243f6a8885a308d3, 0x13198a2e03707344, 0xa4093822299f31d0, 0x082efa98ec4e6c89,
         0x452821e638d01377, 0xbe5466cf34e90c6c, 0xc0ac29b7c97c50dd, 0x3f84d5b5b5470917]
    rng = np.random.default_rng(seed)
    off = np.asarray(w.sample_frame_off, np.uint64)
    pc = _same_leaf(w)
    partners = pc[int(off[0]) + 1:int(off[0]) + 3].copy()  # two pcs that resolve to real names
    M = (1 << 64) - 1
    for s in range(len(off) - 1):
        f0, f1 = int(off[s]), int(off[s + 1])
        a0 = f0 & ~7
        for j in range(f0 + 1, f1 - 1):
            if (j & 1) == 0 and j + 1 < f1:
                q = (j - a0) >> 3
                B = ((q + 1) * 0x9e3779b97f4a7c15) & M
                pc[j] = np.uint64(B ^ K[j & 7])
                pc[j + 1] = partners[rng.integers(0, 2)]
                break
    w.frame_pc = pc
    return w


def test_planted_annihilator_frames_fold_exactly(ctx):
    win = _annihilator_window()
    stats, _ = _compare(ctx, win, cfg={"verify": 1}, ref_threads=4)
    assert stats["verified"] == 1 and stats["verify_retries"] == 0 and stats["prefix_hits"] > 0


def test_forced_prefix_collisions_caught_by_verify(ctx):
    """4-bit prefix-cache keys make distinct call chains collide: without verify
    the folded profiles go wrong; verify mode detects it and re-runs without the
    cache, matching the oracle exactly."""
    # long enough that later batches find chains cached by earlier ones
    win = small_window(seed=9, ranks=4, samples_per_rank=100_000, slow_rank=1, depth=12, n_sym=2000, pool=400)
    win.frame_pc = _same_leaf(win)
    r, _, _ = ref.window_run(win, threads=4)
    st = ctx.window_run(win, cfg={"debug_weak_prefix_key": 1})
    assert st["prefix_hits"] > 0
    assert ctx.groupdata()["cpu_profiles"] != r["groupdata"]["cpu_profiles"]
    stats, _ = _compare(ctx, win, cfg={"debug_weak_prefix_key": 1, "verify": 1}, ref_threads=4)
    assert stats["verify_retries"] >= 1 and stats["verified"] == 1


def test_device_resident_side_streams(ctx):
    """coll_memory / side_memory = device: collectives, GPU kernel events and OS
    counters read from HBM give the same GroupData and report as host inputs."""
    import bench
    win = small_window(seed=4, ranks=6, samples_per_rank=3000, slow_rank=2, depth=12, n_sym=2000, pool=100)
    ctx.window_run(win)
    gd, rep = ctx.groupdata(), ctx.report()
    bench.side_to_device(win)
    ctx.window_run(win)
    assert ctx.groupdata() == gd and ctx.report() == rep
