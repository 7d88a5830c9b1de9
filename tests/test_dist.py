"""Multi-GPU path: one communication group spanning N GPUs.

CPU (gloo, world_size 2): rank sharding covers every rank exactly once and the
NCCL id is shipped through torch.distributed.
GPU (>= 2 devices): every process's report equals the single-process reference
report; the union of the processes' CPU profiles equals the reference's.
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

from paper_2603_29235_b200.dist import shard_bounds, shard_window
from tests.synth import small_window

ROOT = Path(__file__).resolve().parents[1]


def test_shard_bounds_cover_all_ranks():
    for n in (1, 7, 8, 1024):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                lo, hi = shard_bounds(n, world, r)
                got.extend(range(lo, hi))
            assert got == list(range(n))


def test_shard_window_reassembles():
    w = small_window(seed=2, ranks=5, samples_per_rank=50, slow_rank=1)
    parts = [shard_window(w, 2, r) for r in range(2)]
    assert np.concatenate([p.rank_ids for p in parts]).tolist() == w.rank_ids.tolist()
    assert np.concatenate([p.sample_ts for p in parts]).tolist() == w.sample_ts.tolist()
    assert np.concatenate([p.frame_pc for p in parts]).tolist() == w.frame_pc.tolist()
    for p in parts:
        assert int(p.rank_sample_off[-1]) == len(p.sample_ts)
        assert int(p.sample_frame_off[-1]) == len(p.frame_pc)
        assert p.coll_rank is w.coll_rank  # side streams stay replicated


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2603_29235_b200.dist import share_unique_id
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    uid = share_unique_id(dist, lambda: bytes(range(128)), device="cpu")
    out.put((rank, uid))
    dist.destroy_process_group()


def test_unique_id_shared_over_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == res[1] == bytes(range(128))


def _run_dist(case, n, shard=0):
    out = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 400),
           str(ROOT / "tests" / "dist_worker.py"), "--out", out, "--case", case, "--shard", str(shard)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [json.loads(Path(out, f"rank{i}.json").read_text()) for i in range(n)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["synthetic", "sim-softirq-1", "sim-logging-2", "sim-dentry-lock-3"])
def test_two_gpu_group_matches_reference(case):
    import torch
    from oracle import ref
    from tests.compare import assert_close
    from tests.dist_cases import make_case
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    if case.startswith("sim-") and not ref.available():
        pytest.skip("oracle/_ref not built")
    outs = _run_dist(case, 2)
    exp, _, _ = ref.window_run(make_case(case))
    for o in outs:
        assert o["report"] == exp["report"]  # bit-exact on every process
    prof = sorted((p for o in outs for p in o["groupdata"]["cpu_profiles"]), key=lambda p: p["rank"])
    assert prof == exp["groupdata"]["cpu_profiles"]
    for k in ("lateness_per_instance", "iteration_times_ms", "gpu_profiles", "os_snapshots"):
        assert outs[0]["groupdata"][k] == exp["groupdata"][k]
    wl = ref.waterline(make_case(case))
    got = outs[0]["waterline"]
    assert [f[0] for f in got["functions"]] == [f[0] for f in wl["functions"]]
    assert_close([f[1:] for f in got["functions"]], [f[1:] for f in wl["functions"]], 1e-6)
    from tests.compare import assert_flags_match
    assert_flags_match([f for o in outs for f in o["waterline"]["flags"]], wl["flags"])


def _merged_lateness(outs):
    """lateness_per_instance of a rank-sharded stage d: each process holds its own
    ranks' entries; the union per instance, in rank order."""
    n = len(outs[0]["groupdata"]["lateness_per_instance"])
    merged = []
    for i in range(n):
        d = {}
        for o in outs:
            lat = o["groupdata"]["lateness_per_instance"]
            assert len(lat) == n
            for r, v in lat[i]:
                assert d.get(r, v) == v
                d[r] = v
        merged.append([[r, d[r]] for r in sorted(d)])
    return merged


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [2, 4])
@pytest.mark.parametrize("case", ["synthetic", "sim-softirq-1", "sim-thermal-2", "c4-2000", "irregular"])
def test_sharded_stage_d_matches_reference(case, n_gpus):
    """Collectives and GPU/OS streams sharded by rank (STG_SHARD_COLL | STG_SHARD_SIDE):
    stage d runs on each GPU's own events with per-instance partials over NCCL and
    the straggler sums chained across GPUs in rank order; every process's report
    is bit-exact, and the union of the processes' lateness equals the reference's."""
    import torch
    from oracle import ref
    from tests.dist_cases import make_case
    if torch.cuda.device_count() < n_gpus:
        pytest.skip(f"needs {n_gpus} GPUs")
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    outs = _run_dist(case, n_gpus, shard=3)
    exp, _, _ = ref.window_run(make_case(case))
    for o in outs:
        assert "error" not in o, o.get("error")
        assert o["report"] == exp["report"]
        for k in ("iteration_times_ms", "gpu_profiles", "os_snapshots"):
            assert o["groupdata"][k] == exp["groupdata"][k]
    assert _merged_lateness(outs) == exp["groupdata"]["lateness_per_instance"]
    prof = sorted((p for o in outs for p in o["groupdata"]["cpu_profiles"]), key=lambda p: p["rank"])
    assert prof == exp["groupdata"]["cpu_profiles"]


@pytest.mark.gpu
def test_sharded_collective_error_agreed():
    """A bad collective event held only by the second GPU: both processes fail with
    the reference's message."""
    import torch
    from oracle import ref
    from tests.dist_cases import make_case
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    with pytest.raises(ref.RefError) as e:
        ref.window_run(make_case("err-coll-shard1"), want_json=False)
    outs = _run_dist("err-coll-shard1", 2, shard=1)
    assert [o.get("error") for o in outs] == [str(e.value)] * 2


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["err-empty-shard1", "err-empty-rank-shard1"])
def test_two_gpu_input_error_agreed(case):
    """An input error found only in the second GPU's shard: both processes fail
    with the reference's message instead of one throwing while the other waits
    in the next collective."""
    import torch
    from oracle import ref
    from tests.dist_cases import make_case
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    with pytest.raises(ref.RefError) as e:
        ref.window_run(make_case(case), want_json=False)
    outs = _run_dist(case, 2)
    assert [o.get("error") for o in outs] == [str(e.value)] * 2


def test_shard_window_streams_partition():
    """Sharded collectives / GPU events / OS records: every event lands on exactly
    one process, the owner of its rank interval, in input order."""
    from oracle import ref
    from paper_2603_29235_b200.dist import shard_rank_lo
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = ref.simulate("softirq", 2, ranks=32, iterations=150)
    for world in (2, 3):
        parts = [shard_window(w, world, r, streams=3) for r in range(world)]
        los = [shard_rank_lo(w.rank_ids, world, r) for r in range(world)]
        assert los == sorted(set(los)) and [p.shard_rank_lo for p in parts] == los
        for stream, fields in (("coll_rank", ("coll_rank", "coll_group", "coll_entry", "coll_exit")),
                               ("gpu_rank", ("gpu_rank", "gpu_kernel", "gpu_dur")),
                               ("os_rank", ("os_rank", "os_p50", "os_p99", "os_migrations"))):
            owner = np.searchsorted(los, np.asarray(getattr(w, stream)), "right") - 1
            for f in fields:
                exp = np.concatenate([np.asarray(getattr(w, f))[owner == q] for q in range(world)])
                assert np.concatenate([getattr(p, f) for p in parts]).tolist() == exp.tolist()
        for q, p in enumerate(parts):
            for key, off, val in (("os_irq_key", "os_irq_off", "os_irq_val"), ("os_sirq_key", "os_sirq_off", "os_sirq_val")):
                assert int(p.__dict__[off][-1]) == len(p.__dict__[key]) == len(p.__dict__[val])
                o_off = np.asarray(getattr(w, off), np.int64)
                rows = [i for i in range(len(w.os_rank)) if np.searchsorted(los, w.os_rank[i], "right") - 1 == q]
                exp = [int(x) for i in rows for x in np.asarray(getattr(w, val))[o_off[i]:o_off[i + 1]]]
                assert p.__dict__[val].tolist() == exp
