#!/usr/bin/env python3
"""bench.py — stack samples/s symbolized + aggregated + diffed (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): per GPU, 128 ranks x 1M CPU stack
samples, 64-frame stacks over three 1M-symbol tables (python, libtorch, cuda),
50k distinct symbolized stacks per rank drawn Zipf(1.1), leaf PCs uniform
inside their function, a straggler rank (softirq path + 0.6 ms late collective
entry), 100 AllReduce instances, GPU kernel and OS counter streams.  One step =
one full window through libstg: collective alignment -> fused symbolize +
aggregate -> fold/sort -> inclusive fractions / diff -> verdict.  Inputs are
resident in HBM (84 GB per GPU >> 126 MB L2, so no L2 flush is needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--ranks R] [--spr S] [--no-e2e] [--no-cpu-baseline]

N > 1: launched by torchrun, one process per GPU; the N GPUs analyse ONE
communication group of N x 128 ranks, each GPU holding the sample streams,
collective events and GPU / OS records of its own 128 ranks (weak scaling:
128 M samples per GPU; stg_window.shard_streams = STG_SHARD_COLL |
STG_SHARD_SIDE), with libstg's NCCL exchange inside the window; timing is the
max over ranks.  --config c3 / c4 shard one fixed 1,024-rank window over the
GPUs instead (strong scaling).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "stack samples/sec symbolized+aggregated+diffed"
UNIT = "samples/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--ranks", type=int, default=128)
    p.add_argument("--spr", type=int, default=1_000_000, help="samples per rank")
    p.add_argument("--depth", type=int, default=64)
    p.add_argument("--pool", type=int, default=50_000)
    p.add_argument("--nsym", type=int, default=1_000_000)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--hot", default="bench", choices=["all", "bench"],
                   help="functions the generator draws from: all of each 1M-symbol table, or 5k/20k/5k")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget-s", type=float, default=20.0)
    p.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "agg", "bundle"],
                   help="c2 = headline (samples/s); c3 = the north-star 1,024-rank window (C1-style CPU "
                        "stacks + GPU kernels + OS counters, sharded over the GPUs); "
                        "c4 = collective alignment, 1,024 ranks x 50k events; "
                        "agg = raw aggregate_samples on the BM_Aggregation stream shape; "
                        "bundle = load_bundle (JSONL) + analysis of a C1-scale bundle directory")
    p.add_argument("--agg-samples", type=int, default=64_000_000, help="agg: samples in the stream")
    p.add_argument("--bundle-spr", type=int, default=100_000, help="bundle: samples per rank (C1: 100k)")
    p.add_argument("--events", type=int, default=50_000, help="c4: events per rank")
    p.add_argument("--iterations", type=int, default=100, help="training iterations in the window (c3: 300)")
    return p.parse_args()


# --------------------------------------------------------------------- data
class Workload:
    """Symbol tables (host, SYMR) + side streams; samples generated on device."""

    def __init__(self, a, shard: int = 0, world: int = 1):
        """One communication group of world x a.ranks ranks; this process owns the
        samples of ranks [shard * a.ranks, (shard + 1) * a.ranks).  Collectives,
        GPU and OS streams cover the whole group (identical on every process)."""
        from tests.synth import c2_tables, side_streams
        self.a = a
        self.tables = c2_tables(a.seed, a.nsym)
        rng = np.random.default_rng(a.seed * 1000)
        self.period = 10_000  # ns between samples of a rank
        self.span = a.spr * self.period
        self.iterations = getattr(a, "iterations", 100)
        self.iter_ns = self.span // self.iterations
        self.group_size = world * a.ranks
        self.world = world
        self.skews_all = rng.integers(-10_000_000, 10_000_001, size=self.group_size).astype(np.int64)
        self.rank_base = shard * a.ranks
        self.skews = self.skews_all[self.rank_base:self.rank_base + a.ranks]
        self.slow_global = 4 if self.group_size > 4 else 0
        self.slow = self.slow_global - self.rank_base  # local index (may be out of range)
        self.side = side_streams(rng, self.group_size, self.iterations, self.iter_ns, self.span,
                                 self.slow_global, self.skews_all)
        w = np.arange(1, a.pool + 1, dtype=np.float64) ** -1.1
        self.zipf_cdf = np.cumsum(w / w.sum())
        self.zipf_cdf[-1] = 1.0

    def _gen_args(self, ranks: int):
        a = self.a
        # functions executed per binary: "bench" = 5k/20k/5k of the 1M (round-1
        # default), "all" = every function of each table can be drawn
        hot = (5000, 20000, 5000) if getattr(a, "hot", "bench") == "bench" else (a.nsym,) * 3
        return dict(depth=a.depth, pool=a.pool, zipf_cdf=self.zipf_cdf, hot=hot,
                    soft_pc=self.tables[2][1][:9] + 4, slow_rank=self.slow if 0 <= self.slow < ranks else -1,
                    soft_share=0.0174, jit_per_million=100, skew=self.skews[:ranks])

    def generate(self, torch, ranks: int, spr: int, seed_off: int = 0, period: int = 0):
        """Device tensors (ts, foff, pc, bin) for `ranks` x `spr` samples (bench-side CUDA
        generator, csrc/bench_gen.cu)."""
        a = self.a
        g = self._gen_args(ranks)
        lib = C.CDLL(str(ROOT / "paper_2603_29235_b200" / "libstg_bench.so"))
        dev = torch.device("cuda")
        n = ranks * spr
        ts = torch.empty(n, dtype=torch.int64, device=dev)
        foff = torch.empty(n + 1, dtype=torch.int64, device=dev)
        pc = torch.empty(n * a.depth, dtype=torch.int64, device=dev)
        bn = torch.empty(n * a.depth, dtype=torch.int16, device=dev)
        st = [torch.from_numpy(t[1].view(np.int64)).to(dev) for t in self.tables]
        sz = [torch.from_numpy(t[2].view(np.int32)).to(dev) for t in self.tables]
        cdf = torch.from_numpy(self.zipf_cdf).to(dev)
        skew = torch.from_numpy(g["skew"].copy()).to(dev)
        P = C.c_void_p
        starts = (P * 3)(*[t.data_ptr() for t in st])
        sizes = (P * 3)(*[t.data_ptr() for t in sz])
        nsym = (C.c_uint32 * 3)(*[a.nsym] * 3)
        hot = (C.c_uint32 * 3)(*g["hot"])
        softa = (C.c_uint64 * 9)(*[int(x) for x in g["soft_pc"]])
        lib.bench_gen_c2.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_uint32, P, P, P, P, P, P,
                                     C.c_int, C.c_double, C.c_uint32, C.c_int64, P, P, P, P, P, P]
        rc = lib.bench_gen_c2(a.seed + seed_off, ranks, spr, a.depth, a.pool, cdf.data_ptr(),
                              C.cast(starts, P), C.cast(sizes, P), C.cast(nsym, P), C.cast(hot, P),
                              C.cast(softa, P), g["slow_rank"], g["soft_share"], g["jit_per_million"],
                              period or self.period, skew.data_ptr(), ts.data_ptr(), foff.data_ptr(), pc.data_ptr(),
                              bn.data_ptr(), P(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, f"generator failed: {rc}"
        torch.cuda.synchronize()
        return ts, foff, pc, bn

    def generate_host(self, ranks: int, spr: int, seed_off: int = 0, period: int = 0):
        """The same samples as generate(), computed on the host with numpy
        (tests/synth.c2_samples_host) — the reference arm loads no repo library."""
        from tests.synth import c2_samples_host
        g = self._gen_args(ranks)
        return c2_samples_host(self.a.seed + seed_off, ranks, spr, self.a.depth, self.a.pool, g["zipf_cdf"],
                               [(t[1], t[2]) for t in self.tables], g["hot"], g["soft_pc"], g["slow_rank"],
                               g["soft_share"], g["jit_per_million"], period or self.period, g["skew"])

    def window(self, ranks: int, spr: int, arrays, memory: int):
        from paper_2603_29235_b200.abi import Window
        from tests.synth import apply_side
        a = self.a
        w = Window()
        w.memory = memory
        w.window_start_ns = int(self.iter_ns * 5)
        w.window_end_ns = int(self.span)
        w.max_skew_ns = 50_000_000
        w.rank_ids = np.arange(self.rank_base, self.rank_base + ranks, dtype=np.int32)
        w.rank_sample_off = (np.arange(ranks + 1, dtype=np.uint64) * spr)
        jit = bytes(20 * [0x7f])
        w.bin_build_ids = np.frombuffer(b"".join(t[0] for t in self.tables) + jit, np.uint8).reshape(-1, 20)
        w.sample_ts, w.sample_frame_off, w.frame_pc, w.frame_bin = arrays
        w.n_samples_ = ranks * spr
        w.n_frames_ = ranks * spr * a.depth
        if ranks == a.ranks:
            apply_side(w, self.side, self.group_size)
            if self.world > 1:  # collectives + GPU/OS streams sharded by rank like the samples
                from paper_2603_29235_b200.dist import keep_streams
                lo = self.rank_base if self.rank_base else None
                hi = self.rank_base + ranks if self.rank_base + ranks < self.group_size else None
                keep_streams(w, lo, hi, 3)
                w.shard_rank_lo = self.rank_base
        else:  # bounded sample: keep the side streams of the sampled ranks only
            from tests.synth import side_streams
            rng = np.random.default_rng(a.seed)
            side = side_streams(rng, ranks, self.iterations, self.iter_ns, self.span, self.slow_global,
                                self.skews_all, rank_base=self.rank_base)
            apply_side(w, side, ranks)
        w.has_baseline = True
        w.baseline_delta = 0.005
        w.baseline = {}
        w.baseline_iteration_ms = self.iter_ns / 1e6
        w.symr = [t[3] for t in self.tables]
        if memory == 1:  # STG_MEM_DEVICE: the side streams live in HBM too
            side_to_device(w)
        return w


def side_to_device(w):
    """Collectives, GPU kernel events and OS counter records as device tensors
    (stg_window.coll_memory / side_memory = STG_MEM_DEVICE): every input of the
    timed window is HBM-resident."""
    import torch
    cols = {"coll_rank": np.int32, "coll_group": np.int32, "coll_kind": np.uint8, "coll_entry": np.int64,
            "coll_exit": np.int64, "coll_gpu_dur": np.int64}
    side = {"gpu_rank": np.int32, "gpu_kernel": np.int32, "gpu_start": np.int64, "gpu_dur": np.int64,
            "os_rank": np.int32, "os_window_start": np.int64, "os_p50": np.int64, "os_p99": np.int64,
            "os_migrations": np.int64, "os_irq_off": np.int64, "os_irq_key": np.int32, "os_irq_val": np.int64,
            "os_sirq_off": np.int64, "os_sirq_key": np.int32, "os_sirq_val": np.int64}
    w.n_coll_ = len(w.coll_rank)
    w.n_gpu_ = len(w.gpu_rank)
    w.n_os_ = len(w.os_rank)
    for f, dt in {**cols, **side}.items():
        a = np.ascontiguousarray(np.asarray(getattr(w, f)).astype(dt))
        setattr(w, f, torch.from_numpy(a).cuda() if len(a) else torch.zeros(1, dtype=torch.int64).cuda())
    w.coll_memory = 1
    w.side_memory = 1


def c3_parity_sample(a, wl, ctx, arrays, k_ranks: int = 8):
    """Parity inside the c3 run: the folded texts (FoldedProfile::to_string) of
    the first k ranks (the straggler among them) from the GPU run just timed,
    against the reference's build_group_data on the same samples of those ranks
    with the whole group's collectives / GPU / OS streams (so the clock offsets
    and hence the window filter are the same).  The reference symbolizes with
    its resolve_stacks + fold_symbolized (one table cache per rank), see
    oracle/ref_harness.cpp."""
    from oracle import ref
    from paper_2603_29235_b200.abi import STG_MEM_HOST
    if not ref.available():
        return None
    spr, D = a.spr, a.depth
    n = k_ranks * spr
    host = (arrays[0][:n].cpu().numpy(), arrays[1][:n + 1].cpu().numpy().view(np.uint64),
            arrays[2][:n * D].cpu().numpy().view(np.uint64), arrays[3][:n * D].cpu().numpy().view(np.uint16))
    w = wl.window(a.ranks, spr, host, STG_MEM_HOST)
    w.rank_ids = w.rank_ids[:k_ranks].copy()
    w.rank_sample_off = w.rank_sample_off[:k_ranks + 1].copy()
    w.n_samples_, w.n_frames_ = n, n * D
    t0 = time.perf_counter()
    r, _, _ = ref.window_run(w, threads=k_ranks, want_json=False, artifacts=True, shared_cache=True)
    ref_s = time.perf_counter() - t0
    exp = {int(rk): txt for rk, txt in r["artifacts"]["folded"]}
    same = [ctx.folded_text(int(rk)) == exp.get(int(rk)) for rk in w.rank_ids]
    return {"ranks_checked": [int(x) for x in w.rank_ids], "folded_text_equal": all(same), "ref_seconds": round(ref_s, 1)}


def workload_name(a):
    if a.config == "c3":
        return ("C3 (north-star): one 1,024-rank window, 100k CPU samples/rank (12-frame stacks, 200 distinct "
                "stacks/rank, 3x10k-symbol tables), GPU kernel + OS counter streams, 300 iterations")
    return "C2: 128 ranks x 1M samples per GPU, 64-frame stacks, 3x1M-symbol tables"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            if self.recording:
                self.rows.append([x.strip() for x in line.split(",")])

    recording = False

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- reference
def reference_arm(a, wl, torch, threads: int, steps: int = 1, warmup: int = 0):
    """The reference's own CPU path (oracle/_ref: strata build_group_data +
    diagnose, compiled from /root/reference) on a bounded sample of the same
    workload, with its per-rank loop fanned over `threads` host threads.
    `warmup` untimed and `steps` timed runs, each a bounded sample sized so the
    whole leg stays within a few minutes (the reference's own timers: the
    build_group_data + diagnose calls, input marshalling excluded)."""
    from oracle import ref
    from paper_2603_29235_b200.abi import STG_MEM_HOST
    if not ref.available():
        return None
    # the reference reloads the 1M-entry tables for every aggregated record
    # (symrepo.cpp:99-120 via folded.cpp:24), so a step holds few samples per
    # rank.  Calibrate with every thread busy (table reloads contend for memory).
    def run(ranks, k):
        # spread the k samples over the whole window span
        arrays = wl.generate_host(ranks, k, seed_off=17, period=max(1, wl.span // k))
        w = wl.window(ranks, k, arrays, STG_MEM_HOST)
        t0 = time.perf_counter()
        res, tb, td = ref.window_run(w, threads=min(threads, ranks), want_json=False)
        return time.perf_counter() - t0, tb + td, ranks * k, res
    ranks = min(threads, a.ranks)
    w1, t1, _, _ = run(ranks, 2)
    budget = max(2.0, min(a.cpu_budget_s, 150.0 / max(1, steps + warmup)))
    k = max(1, int(2 * budget / max(w1, t1, 1e-6)))
    print(f"[bench ref] calibration: {ranks} ranks x 2 samples in {w1:.2f}s wall ({t1:.2f}s in the reference); "
          f"{k} samples per rank per step", file=sys.stderr, flush=True)
    for _ in range(warmup):
        run(ranks, k)
    tot_t = tot_n = 0.0
    res = None
    for i in range(max(1, steps)):
        w, t, n, res = run(ranks, k)
        tot_t += t
        tot_n += n
        print(f"[bench ref] step {i}: {n} samples in {t:.2f}s ({w:.2f}s wall)", file=sys.stderr, flush=True)
    return {"value": tot_n / tot_t, "unit": UNIT, "cores": ranks, "kind": "reference",
            "sample": f"{max(1, steps)} x ({ranks} ranks x {k} samples) of the {a.config.upper()} workload "
                      f"({a.depth}-frame stacks, 3x{a.nsym}-symbol tables), build_group_data+diagnose in "
                      f"{tot_t:.2f}s; the reference reloads the {a.nsym}-entry SYMR tables once per aggregated "
                      "record (resolve_stack cache is per call)",
            "verdict": res["report"]["verdict"]}


def peaks():
    try:
        return json.loads(PEAKS.read_text())
    except Exception:
        return {}


def ncu_traffic(kernel, algo_bytes):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture of this same workload (profiles/ncu_traffic.json,
    written by tools/ncu_summary.py --traffic-json); None when the capture was
    taken on a different workload size."""
    try:
        rec = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())[kernel]
    except Exception:
        return None
    if int(rec.get("algorithmic_bytes", -1)) != int(algo_bytes):
        return None
    return rec["dram_bytes"]


# ----------------------------------------------------------------------- c4
def bench_c4(a, torch, stg, rank, local, world, dist):
    """C4: NCCL collective-event alignment, 1,024 ranks x 50k AllReduce/AllGather
    events per GPU (device-resident), NIC-softirq straggler.  Metric: events/s."""
    from tests.synth import c4_window
    ranks = 1024
    E = a.events
    sharded = world > 1  # one 1,024-rank window, its ranks' events split over the GPUs (strong scaling)
    win = c4_window(ranks=ranks, events_per_rank=E, seed=1, device=True, torch=torch)
    if sharded:
        from paper_2603_29235_b200.dist import keep_streams, shard_bounds
        lo, hi = shard_bounds(ranks, world, rank)
        for f in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur"):
            setattr(win, f, getattr(win, f)[lo * E:hi * E].contiguous())  # rank-major events
        win.n_coll_ = (hi - lo) * E
        keep_streams(win, lo if rank else None, hi if rank + 1 < world else None, 2)
        win.shard_streams = 3
        win.shard_rank_lo = lo
    ctx = stg.Context(local)
    if sharded:
        from paper_2603_29235_b200.dist import share_unique_id
        ctx.dist_init(world, rank, share_unique_id(dist, stg.Context.dist_unique_id, device="cuda"))
    for _ in range(a.warmup):
        s = ctx.window_run(win)
        log(f"[c4 r{rank}] warmup {s['ms_total']:.2f} ms (collectives {s['ms_collectives']:.2f}) "
            f"instances={s['n_instances']} windowed={s['n_windowed']}")
    rep = ctx.report()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    coll = []
    e0.record()
    for _ in range(a.steps):
        s = ctx.window_run(win)
        coll.append(s["ms_collectives"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_ev = ranks * a.events  # events of the whole group per step (sharded) / per GPU (1 GPU)
    cm = float(np.median(coll))
    algo = 24 * n_ev // world  # per GPU: entry+exit read, lateness written (SURVEY.md §8(d) stage d)
    peak = peaks().get("hbm_gbs", 6650.0)
    line = {"metric": "collective events/sec aligned (match+align+lateness+straggler+verdict)",
            "value": n_ev / (ms / 1e3), "unit": "events/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"C4: {ranks} ranks x {a.events} events (AllReduce/AllGather), straggler rank 4",
                       "inputs": "collective arrays resident in HBM",
                       "parallelism": (f"one {ranks}-rank window, events sharded by rank over {world} GPUs "
                                       "(STG_SHARD_COLL: per-instance partials over NCCL, straggler sums "
                                       "chained in rank order)") if sharded else "1 GPU"},
            "verdict": rep["verdict"], "flagged_ranks": rep["flagged_ranks"],
            "stage_ms": {"collectives": cm, "total_device": s["ms_total"]},
            "roofline": {"bound": "hbm", "achieved": round(algo / (cm / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(algo / (cm / 1e3) / 1e9 / peak, 4), "traffic": None,
                         "kernel": "collective stage (k_coll_* + k_straggler_*)", "algorithmic_bytes": algo}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------- agg
def agg_stream(torch, n: int, seed: int, device: str):
    """The stream of the reference's BM_Aggregation (benchmarks/bench.cpp:79-95):
    16 stacks x 12 frames of one binary (offsets 0x1000 + s*64 + d*8), a sample
    every 10 us, stacks drawn uniformly — here n samples long."""
    g = torch.Generator(device=device).manual_seed(seed)
    pick = torch.randint(0, 16, (n,), generator=g, device=device, dtype=torch.int64)
    d = torch.arange(12, device=device, dtype=torch.int64)
    pc = (0x1000 + pick[:, None] * 64 + d[None, :] * 8).reshape(-1)
    ts = torch.arange(n, device=device, dtype=torch.int64) * 10_000
    off = torch.arange(n + 1, device=device, dtype=torch.int64) * 12
    bn = torch.zeros(n * 12, device=device, dtype=torch.int16)
    return ts, off, pc, bn


def bench_agg(a, torch, stg, rank, local, world, dist):
    """Raw-address aggregate_samples (samples.cpp:31-85, §8(f) row 4): one rank's
    stream per GPU, device-resident, drained every 5 s.  Metric: samples/s."""
    n = a.agg_samples
    ts, off, pc, bn = agg_stream(torch, n, 7 + rank, "cuda")
    ctx = stg.Context(local)
    for _ in range(a.warmup):
        wins = ctx.aggregate_samples(ts, off, pc, bn)
    nrec = sum(len(w[2]) for w in wins)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        ctx.aggregate_samples(ts, off, pc, bn)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # end to end: the stream in pinned host memory, copied in by the call, records copied out
    h = [x.cpu().pin_memory() for x in (ts, off, pc, bn)]
    ctx.aggregate_samples(*h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        ctx.aggregate_samples(*h)
    e2e_s = (time.perf_counter() - t0) / 2
    algo = n * (8 + 8 + 12 * 10)  # ts + frame offset + 12 frames x (8 B pc + 2 B bin), read once
    peak = peaks().get("hbm_gbs", 6650.0)
    cb = None
    if rank == 0 and not a.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            k = 2_000_000
            hs = [x[:k].cpu().numpy() for x in (ts,)] + [off[:k + 1].cpu().numpy().view(np.uint64),
                                                        pc[:12 * k].cpu().numpy().view(np.uint64),
                                                        bn[:12 * k].cpu().numpy().view(np.uint16)]
            from tests.synth import build_id
            t = ref.aggregate_samples(hs[0], hs[1], hs[2], hs[3], build_id("a"), time_only=True)
            cb = {"value": k / t, "unit": "samples/s", "cores": 1, "kind": "reference",
                  "sample": f"first {k} samples of the stream, strata::aggregate_samples alone "
                            "(single-threaded, as the reference runs it)"}
    line = {"metric": "raw samples/sec aggregated (aggregate_samples, 5 s drain)",
            "value": n * world / (ms / 1e3), "unit": "samples/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"BM_Aggregation stream shape (bench.cpp:79-95) x {n} samples per GPU",
                       "inputs": "stream resident in HBM (> L2)", "windows": len(wins), "records": nrec},
            "e2e": {"value": n * world / e2e_s, "unit": "samples/s",
                    "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in h)),
                    "d2h_bytes_per_step": int(nrec * 16 + len(wins) * 24)},
            "roofline": {"bound": "hbm", "achieved": round(algo / (ms / 1e3) / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(algo / (ms / 1e3) / 1e9 / peak, 4), "traffic": None,
                         "kernel": "whole call (k_agg_hash + k_agg_verify + compaction)",
                         "algorithmic_bytes": algo},
            "cpu_baseline": cb}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------- bundle
def write_bench_bundle(torch, wl, b, d: Path):
    """A write_bundle-format directory (bundle.cpp:83-164) for the workload."""
    from paper_2603_29235_b200.abi import STG_MEM_HOST
    ts, foff, pc, bn = wl.generate(torch, b.ranks, b.spr)
    host = (ts.cpu().numpy(), foff.cpu().numpy().view(np.uint64), pc.cpu().numpy().view(np.uint64),
            bn.cpu().numpy().view(np.uint16))
    w = wl.window(b.ranks, b.spr, host, STG_MEM_HOST)
    d.mkdir(parents=True, exist_ok=True)
    dump = lambda o: json.dumps(o, sort_keys=True, separators=(",", ":"))
    meta = {"scenario": "bench-c1", "seed": b.seed, "ranks": b.ranks, "iterations": wl.iterations,
            "sample_rate_hz": 1e9 / wl.period, "group": 0, "max_skew_ns": int(w.max_skew_ns),
            "window_start_ns": int(w.window_start_ns), "window_end_ns": int(w.window_end_ns),
            "baseline": {"epoch": "bench", "delta": 0.005, "iteration_ms": float(w.baseline_iteration_ms),
                         "fractions": {}},
            "group_ranks": [int(x) for x in w.group_ranks]}
    (d / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    with open(d / "gpu_events.jsonl", "w") as f:
        for i in range(len(w.gpu_rank)):
            f.write(dump({"rank": int(w.gpu_rank[i]), "iter": 0, "kernel": w.kernel_names[int(w.gpu_kernel[i])],
                          "start": int(w.gpu_start[i]), "dur": int(w.gpu_dur[i])}) + "\n")
    with open(d / "os_counters.jsonl", "w") as f:
        for i in range(len(w.os_rank)):
            irq = {w.counter_names[int(w.os_irq_key[k])]: int(w.os_irq_val[k])
                   for k in range(int(w.os_irq_off[i]), int(w.os_irq_off[i + 1]))}
            sirq = {w.counter_names[int(w.os_sirq_key[k])]: int(w.os_sirq_val[k])
                    for k in range(int(w.os_sirq_off[i]), int(w.os_sirq_off[i + 1]))}
            f.write(dump({"rank": int(w.os_rank[i]), "window_start": int(w.os_window_start[i]), "interrupts": irq,
                          "softirqs": sirq, "sched_delay_p50_ns": int(w.os_p50[i]),
                          "sched_delay_p99_ns": int(w.os_p99[i]), "numa_migrations": int(w.os_migrations[i])})
                    + "\n")
    for bid, _, _, symr in wl.tables:
        h = bid.hex()
        (d / "symbols" / h[:2]).mkdir(parents=True, exist_ok=True)
        (d / "symbols" / h[:2] / (h + ".symr")).write_bytes(symr)
    lib = C.CDLL(str(ROOT / "paper_2603_29235_b200" / "libstg_bench.so"))
    P = C.c_void_p
    lib.bench_write_jsonl.argtypes = [C.c_char_p, C.c_char_p, C.c_int, P, P, P, P, P, P, C.c_int, P, C.c_uint64,
                                      P, P, P, P, P, P]
    arr = lambda x, dt: np.ascontiguousarray(np.asarray(x).astype(dt))
    keep = [arr(w.rank_ids, np.int32), arr(w.rank_sample_off, np.uint64), host[0], host[1], host[2], host[3],
            arr(w.bin_build_ids, np.uint8), arr(w.coll_rank, np.int32), arr(w.coll_group, np.int32),
            arr(w.coll_kind, np.uint8), arr(w.coll_entry, np.int64), arr(w.coll_exit, np.int64),
            arr(w.coll_gpu_dur, np.int64)]
    rc = lib.bench_write_jsonl(str(d / "samples.jsonl").encode(), str(d / "collectives.jsonl").encode(),
                               len(keep[0]), *[k.ctypes.data for k in keep[:6]], len(keep[6]),
                               keep[6].ctypes.data, len(keep[7]), *[k.ctypes.data for k in keep[7:]])
    assert rc == 0
    return b.ranks * b.spr


def bench_bundle(a, torch, stg, rank, local, world, dist):
    """load_bundle (bundle.cpp:181-233) + build_group_data + diagnose of a C1-scale
    bundle directory (8 ranks x 100k samples, 12-frame stacks, 10k-symbol tables):
    JSONL bulk decoded on the GPU.  Metric: bundle samples/s, files to verdict."""
    import copy
    import shutil
    import tempfile
    b = copy.copy(a)
    b.ranks, b.spr, b.depth, b.nsym, b.pool = 8, a.bundle_spr, 12, 10_000, 2_000
    wl = Workload(b, rank, world)
    d = Path(tempfile.mkdtemp(prefix=f"stg_bundle_r{rank}_"))
    t0 = time.perf_counter()
    n = write_bench_bundle(torch, wl, b, d)
    log(f"[bundle r{rank}] wrote {d} in {time.perf_counter() - t0:.1f}s")
    ctx = stg.Context(local)
    for _ in range(a.warmup):
        info = ctx.load_bundle(d)
        log(f"[bundle r{rank}] warmup load: {info}")
        st = ctx.bundle_run()
    rep = ctx.report()
    log(f"[bundle r{rank}] verdict {rep['verdict']}")
    if dist:
        dist.barrier()
    times, infos = [], []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        infos.append(ctx.load_bundle(d))
        st = ctx.bundle_run()
        times.append(time.perf_counter() - t0)
    sec = float(np.mean(times))
    if dist:
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    dec = float(np.mean([i["decode_s"] for i in infos]))
    rd = float(np.mean([i["read_s"] for i in infos]))
    bulk = infos[-1]["bulk_bytes"]
    cb = None
    if rank == 0 and not a.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            tl, nref = ref.bundle_load_time(str(d))
            assert nref == n
            cb = {"value": n / tl, "unit": "samples/s", "cores": 1, "kind": "reference",
                  "sample": f"the same bundle directory through strata::load_bundle alone ({tl:.2f}s, "
                            "single-threaded); its build_group_data on this bundle is not timed: it reloads the "
                            "SYMR tables once per aggregated record (resolve_stack, symrepo.cpp:99-120) and "
                            "nearly every sample is its own record here (hours)",
                  "load_bundle_s": tl}
    line = {"metric": "bundle samples/sec (load_bundle JSONL + build_group_data + diagnose)",
            "value": n * world / sec, "unit": "samples/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": "C1-scale bundle directory: 8 ranks x 100k samples, 12-frame stacks, "
                                   "3 x 10k-symbol tables", "bulk_bytes": bulk},
            "verdict": rep["verdict"], "flagged_ranks": rep["flagged_ranks"],
            "stage_s": {"file_read": rd, "gpu_decode": dec, "analysis_device_ms": st["ms_total"]},
            "roofline": {"bound": "hbm", "achieved": round(bulk / dec / 1e9, 1), "peak": peaks().get("hbm_gbs", 6650.0),
                         "unit": "GB/s", "frac": round(bulk / dec / 1e9 / peaks().get("hbm_gbs", 6650.0), 4),
                         "traffic": None, "kernel": "JSONL decode incl. H2D of the file bytes (host-timed)",
                         "algorithmic_bytes": bulk},
            "e2e": {"value": n * world / sec, "unit": "samples/s", "h2d_bytes_per_step": bulk,
                    "d2h_bytes_per_step": 0},
            "cpu_baseline": cb}
    if rank == 0:
        print(json.dumps(line), flush=True)
    shutil.rmtree(d, ignore_errors=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------- main
def main():
    a = args_parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if a.impl == "reference":
        if a.config == "c3":
            a.ranks = 1024
            a.spr, a.depth, a.pool, a.nsym, a.hot, a.iterations = 100_000, 12, 200, 10_000, "all", 300
        if rank == 0:
            wl = Workload(a, 0)
            cb = reference_arm(a, wl, torch, os.cpu_count() or 1, steps=a.steps, warmup=a.warmup)
            if cb is None:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstrata_ref.so not built"}))
            else:
                line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
                        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "higher_is_better": True,
                        "scaling": "strong" if a.config == "c3" else "weak", "vs_baseline": None, "dtype": "u64",
                        "data": "synthetic",
                        "config": {"workload": workload_name(a),
                                   "ranks_per_gpu": a.ranks, "samples_per_rank": a.spr, "depth": a.depth,
                                   "distinct_stacks": a.pool, "symbols_per_table": a.nsym,
                                   "inputs": "host memory, bounded sample per step (see cpu_baseline.sample)"},
                        "cpu_baseline": cb,
                        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                "d2h_bytes_per_step": 0}}
                print(json.dumps(line), flush=True)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    if a.config == "c3":
        # north-star window (richer variant): 1,024 ranks in
        # one group, C1-style CPU profiles (100k samples/rank, 12-frame stacks,
        # 200 distinct stacks/rank, 10k-symbol tables), GPU kernel events and OS
        # counters of 300 iterations; the 1,024 ranks are sharded over the GPUs
        # (strong scaling: the window is fixed)
        a.ranks = 1024 // world
        a.spr, a.depth, a.pool, a.nsym, a.hot, a.iterations = 100_000, 12, 200, 10_000, "all", 300
    import paper_2603_29235_b200 as stg
    from paper_2603_29235_b200.abi import STG_MEM_DEVICE, STG_MEM_HOST
    if a.config == "c4":
        return bench_c4(a, torch, stg, rank, local, world, dist)
    if a.config == "agg":
        return bench_agg(a, torch, stg, rank, local, world, dist)
    if a.config == "bundle":
        return bench_bundle(a, torch, stg, rank, local, world, dist)
    wl = Workload(a, rank, world)
    ctx = stg.Context(local)
    if world > 1:  # one communication group spanning the GPUs: libstg's own NCCL group
        from paper_2603_29235_b200.dist import share_unique_id
        ctx.dist_init(world, rank, share_unique_id(dist, stg.Context.dist_unique_id, device="cuda"))
    # symbol-table ingest (SYMR parse + dictionary build, on the GPU; §8(f) row 2),
    # timed once: tables are ingested once per binary, not per window
    t0 = time.perf_counter()
    for _, _, _, symr in wl.tables:
        ctx.ingest(symr)
    t1 = time.perf_counter()
    ctx.resolve(np.zeros(1, np.uint64), np.zeros(1, np.uint16), np.zeros((1, 20), np.uint8))  # dictionary refresh
    t2 = time.perf_counter()
    ingest = {"tables": len(wl.tables), "symbols": a.nsym * len(wl.tables),
              "bytes": sum(len(t[3]) for t in wl.tables), "parse_s": round(t1 - t0, 4),
              "dictionary_s": round(t2 - t1, 4)}
    log(f"[bench r{rank}] tables ingested: parse {t1 - t0:.3f}s, dictionary {t2 - t1:.3f}s")
    t0 = time.time()
    arrays = wl.generate(torch, a.ranks, a.spr)
    win = wl.window(a.ranks, a.spr, arrays, STG_MEM_DEVICE)
    log(f"[bench r{rank}] generated {win.n_samples} samples / {win.n_frames} frames in {time.time() - t0:.1f}s")

    cfg = {"want_waterline": 1}  # every rank scored against its peers (compute_waterline + flag_ranks)

    def step():
        return ctx.window_run(win, cfg=cfg, ingest=False)

    clk = ClockSampler(local).__enter__()  # started before warm-up: NVML start-up stays untimed
    for i in range(a.warmup):
        s = step()
        log(f"[bench r{rank}] warmup {i}: {s['ms_total']:.2f} ms (sym {s['ms_symbolize']:.2f}) "
            f"verdict={stg.VERDICTS[s['verdict']]} lines={s['n_lines']} seqs={s['n_sequences']}")
    rep = ctx.report()
    sym_ms, tot_ms, launches = [], [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.recording = True
    e0.record()
    for _ in range(a.steps):
        s = step()
        sym_ms.append(s["ms_symbolize"])
        tot_ms.append(s["ms_total"])
        launches.append(s["kernel_launches"])
    e1.record()
    torch.cuda.synchronize()
    clk.recording = False
    clk.__exit__(None, None, None)
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1) / a.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_per_gpu = s["n_samples_in_window"]
    n_total = n_per_gpu
    if dist:  # in-window samples of the whole group (the shards differ slightly)
        t = torch.tensor([n_per_gpu], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        n_total = int(t.item())
    value = n_total / (ms / 1e3)
    # ---- roofline of the dominant kernel (fused symbolize+aggregate).  Algorithmic
    # bytes: every sample's ts + CSR row (16 B), and the frames of the IN-WINDOW
    # samples only (10 B each: 8 B pc + 2 B bin) — k_sym_agg never reads the frames
    # of a sample outside the window.  Stacks are a.depth frames deep.
    algo_bytes = 10 * n_per_gpu * a.depth + 16 * win.n_samples
    k_ms = float(np.median(sym_ms))
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    achieved = algo_bytes / (k_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": ncu_traffic("k_sym_agg_c3" if a.config == "c3" else "k_sym_agg", algo_bytes),
            "kernel": "k_sym_agg",
            "kernel_ms": round(k_ms, 3), "algorithmic_bytes": algo_bytes,
            "pipeline_frac": round(algo_bytes / (ms / 1e3) / 1e9 / peak, 4),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback 6.65 TB/s"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if a.config == "c3" else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_name(a),
                       "ranks_per_gpu": a.ranks, "samples_per_rank": a.spr, "depth": a.depth,
                       "distinct_stacks": a.pool, "symbols_per_table": a.nsym,
                       "functions_drawn": "5k/20k/5k per table" if a.hot == "bench" else "all 1M per table",
                       "inputs": f"resident in HBM, {(10 * win.n_frames + 16 * win.n_samples) / 1e9:.1f} GB/GPU "
                                 "> L2 (no flush needed)",
                       "group_ranks": wl.group_size,
                       "parallelism": (f"one {wl.group_size}-rank group sharded by rank over {world} GPUs "
                                       "(samples, collectives, GPU / OS streams); NCCL inside libstg: stage-d "
                                       "partials and straggler chains, cpu_diff fractions from their owners, "
                                       "waterline reductions") if world > 1 else
                                      f"one {wl.group_size}-rank group on 1 GPU"},
            "verdict": rep["verdict"], "flagged_ranks": rep["flagged_ranks"],
            "prefix_cache": {"hits": s["prefix_hits"], "misses": s["prefix_misses"]},
            "stage_ms": {"total_device": float(np.median(tot_ms)), "symbolize_aggregate": k_ms,
                         "collectives": s["ms_collectives"], "fold": s["ms_fold"], "diff": s["ms_diff"]},
            "roofline": roof, "ingest": ingest, "gpu_launches": int(np.median(launches)) * a.steps,
            "clocks": clk.summary()}
    if a.config == "c3":
        line["north_star"] = {"target": "full pipeline >= 0.40 of the HBM roofline on a 1,024-rank window",
                              "pipeline_frac": roof["pipeline_frac"], "met": roof["pipeline_frac"] >= 0.40}
        if rank == 0 and world == 1 and not a.no_cpu_baseline:
            try:
                line["parity_sample"] = c3_parity_sample(a, wl, ctx, arrays)
            except Exception as ex:
                line["parity_sample"] = {"error": str(ex)[:200]}
    # ---- end to end through the C-ABI with host buffers (H2D inside the timed region)
    e2e_ok = not a.no_e2e
    if e2e_ok and world > 1:
        try:
            import psutil
            need = world * (win.n_frames * 10 + win.n_samples * 16) * 1.25
            if psutil.virtual_memory().available < need:
                e2e_ok = False
                line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                               "reason": f"host RAM {psutil.virtual_memory().available / 1e9:.0f} GB < "
                                         f"{need / 1e9:.0f} GB of pinned inputs for {world} processes"}
        except ImportError:
            pass
        t = torch.tensor([1 if e2e_ok else 0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # every process takes the same branch
        if not t.item() and e2e_ok:
            e2e_ok = False
            line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                           "reason": "another process lacks host RAM for pinned inputs"}
    if e2e_ok:
        host = []
        for t in arrays:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            host.append(h)
        del arrays
        win = None
        torch.cuda.empty_cache()
        hwin = wl.window(a.ranks, a.spr, tuple(h.numpy().view(dt) for h, dt in
                                                zip(host, (np.int64, np.uint64, np.uint64, np.uint16))),
                         STG_MEM_HOST)
        ctx.window_run(hwin, cfg=cfg, ingest=False)  # warm
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(a.e2e_steps):
            st = ctx.window_run(hwin, cfg=cfg, ingest=False)
            r = ctx.report()
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
        el = (time.perf_counter() - t0) / a.e2e_steps
        if dist:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        line["e2e"] = {"value": n_total / el, "unit": UNIT,
                       "h2d_bytes_per_step": h2d // a.e2e_steps, "d2h_bytes_per_step": d2h // a.e2e_steps,
                       "ms_per_step": el * 1e3, "verdict": r["verdict"]}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            line["cpu_baseline"] = reference_arm(a, wl, torch, os.cpu_count() or 1)
        except Exception as ex:  # the baseline must not sink the GPU line
            line["cpu_baseline"] = {"error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
