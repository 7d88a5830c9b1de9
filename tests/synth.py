"""Seeded synthetic analysis windows (SURVEY.md §8(d) C1 shape), numpy only.

Used by tests, smoke() and bench.py.  Produces an abi.Window with SYMR symbol
tables, CPU stack samples with a Zipf stack mix, per-iteration AllReduce events
with per-rank clock skew, GPU kernel events, 5 s OS counter windows, and an
optional straggler rank (softirq path in its stacks, +0.6 ms collective entry
delay, NET_RX storm) — mirroring the fault model of the reference simulator
(simulate.cpp:164-182, 272-305) without depending on it.
"""
from __future__ import annotations

import hashlib
import struct

import numpy as np

from paper_2603_29235_b200.abi import Window

SIM_APP = ["main", "train_loop", "forward_pass", "matmul_dispatch", "softmax_dispatch",
           "backward_pass", "matmul_grad_dispatch", "bias_grad_dispatch", "allreduce_wait",
           "optimizer_step", "data_loader_next", "checkpoint_maybe", "log_metrics",
           "SLS::LogClient::Send", "SLS::LogClient::Serialize", "cpfs_checkpoint_write",
           "cpfs_write_block", "ossutils_download", "oss_http_get", "open64", "stat64", "unlink"]
SIM_KERNEL = ["asm_common_interrupt", "common_interrupt", "irq_exit_rcu", "__do_softirq",
              "net_rx_action", "napi_poll", "virtnet_poll", "virtnet_receive", "napi_gro_receive",
              "do_sys_openat2", "path_openat", "d_alloc_parallel", "queued_spin_lock_slowpath",
              "vfs_statx", "filename_lookup", "do_unlinkat", "d_invalidate"]
SOFTIRQ = SIM_KERNEL[:9]
KERNELS = ["dropout_kernel", "fused_matmul", "layernorm_kernel", "nccl_all_reduce", "softmax_kernel"]
COUNTERS = ["LOC", "NET_RX", "PCI-MSI-eth0", "RCU", "TIMER"]


def build_id(label: str) -> bytes:
    return hashlib.sha1(label.encode()).digest()


def pack_symr(bid: bytes, starts, sizes, names) -> bytes:
    """SYMR layout (symfile.hpp:13-18): header, sorted entries, u16-prefixed names."""
    order = np.argsort(np.asarray(starts, np.uint64), kind="stable")
    starts = np.asarray(starts, np.uint64)[order]
    sizes = np.asarray(sizes, np.uint32)[order]
    names = [names[i] for i in order]
    enc = [n.encode() if isinstance(n, str) else n for n in names]
    lens = np.array([len(e) for e in enc], np.int64)
    offs = np.zeros(len(enc), np.uint32)
    if len(enc):
        offs[1:] = np.cumsum(lens + 2)[:-1]
    n = len(enc)
    ent = np.zeros(n, dtype=[("s", "<u8"), ("z", "<u4"), ("o", "<u4")])
    ent["s"], ent["z"], ent["o"] = starts, sizes, offs
    strtab = b"".join(struct.pack("<H", len(e)) + e for e in enc)
    return b"SYMR" + struct.pack("<I", 1) + bid + struct.pack("<II", n, 36 + 16 * n) + ent.tobytes() + strtab


def small_window(seed: int = 1, ranks: int = 8, samples_per_rank: int = 2000, slow_rank: int = 4,
                 depth: int = 12, n_sym: int = 2000, pool: int = 200, unknown_frac: float = 0.01,
                 iterations: int = 100, softirq_share: float = 0.0174, entry_delay_ns: int = 600_000,
                 extra_bins: int = 0) -> Window:
    """C1-shaped window; slow_rank < 0 gives a healthy window."""
    rng = np.random.default_rng(seed)
    # ---- one application binary: symbols at 0x1000 + 64 i, size 48 (25 % gap)
    names = SIM_APP + SIM_KERNEL + [f"fn_{i}" for i in range(max(0, n_sym - len(SIM_APP) - len(SIM_KERNEL)))]
    n_sym = len(names)
    starts = 0x1000 + 64 * np.arange(n_sym, dtype=np.uint64)
    sizes = np.full(n_sym, 48, np.uint32)
    # distinct tables must carry distinct build ids (a context keeps the first
    # table ingested under an id, like SymbolRepository::ingest)
    bid = build_id(f"app-{seed}" if n_sym == 2000 else f"app-{seed}-n{n_sym}")
    symr = [pack_symr(bid, starts, sizes, names)]
    bids = [bid]
    for e in range(extra_bins):  # binaries without a symbol file: unknown labels
        bids.append(build_id(f"jit-{seed}-{e}"))
    idx = {n: i for i, n in enumerate(names)}
    # ---- stack pool (leaf-first lists of (bin, pc)); root is main;train_loop
    stacks = []
    for p in range(pool):
        d = int(rng.integers(max(3, depth - 4), depth + 5))
        mid = rng.integers(len(SIM_APP) + len(SIM_KERNEL), n_sym, size=d - 2)
        fr = [(0, int(starts[idx["main"]]) + 8), (0, int(starts[idx["train_loop"]]) + 8)]
        for m in mid:
            off = int(starts[m]) + (56 if rng.random() < unknown_frac else int(rng.integers(0, 48)))
            b = 0
            if extra_bins and rng.random() < 0.02:
                b = int(rng.integers(1, 1 + extra_bins))
            fr.append((b, off))
        stacks.append(fr[::-1])
    soft = [(0, int(starts[idx[n]]) + 4) for n in SOFTIRQ][::-1]
    zipf_w = 1.0 / np.arange(1, pool + 1) ** 1.1
    zipf_w /= zipf_w.sum()
    # ---- clocks
    period = 10_101_000 // 8  # ns between samples
    span = samples_per_rank * period
    iter_ns = span // iterations
    skews = rng.integers(-10_000_000, 10_000_001, size=ranks)
    ws = int(iter_ns * 5)  # analysis window starts after 5 iterations (true time)
    we = int(span)
    rank_ids = np.arange(ranks, dtype=np.int32)
    ts_all, foff, pcs, bins_ = [], [0], [], []
    rank_off = [0]
    for r in range(ranks):
        perm = rng.permutation(pool)
        choice = perm[rng.choice(pool, size=samples_per_rank, p=zipf_w)]
        t = np.cumsum(np.full(samples_per_rank, period) * (1 + rng.uniform(-0.02, 0.02, samples_per_rank)))
        t = t.astype(np.int64) + int(skews[r])
        for i in range(samples_per_rank):
            if r == slow_rank and rng.random() < softirq_share:
                fr = soft
            else:
                fr = stacks[int(choice[i])]
            for b, o in fr:
                bins_.append(b)
                pcs.append(o)
            foff.append(len(pcs))
        ts_all.append(t)
        rank_off.append(rank_off[-1] + samples_per_rank)
    side = side_streams(rng, ranks, iterations, iter_ns, we, slow_rank, skews, entry_delay_ns)
    w = Window()
    w.window_start_ns, w.window_end_ns, w.max_skew_ns = ws, we, 50_000_000
    w.rank_ids = rank_ids
    w.rank_sample_off = np.asarray(rank_off, np.uint64)
    w.bin_build_ids = np.frombuffer(b"".join(bids), np.uint8).reshape(-1, 20).copy()
    w.sample_ts = np.concatenate(ts_all).astype(np.int64)
    w.sample_frame_off = np.asarray(foff, np.uint64)
    w.frame_pc = np.asarray(pcs, np.uint64)
    w.frame_bin = np.asarray(bins_, np.uint16)
    apply_side(w, side, ranks)
    w.has_baseline = True
    w.baseline_delta = 0.005
    w.baseline = {"main": 1.0, "train_loop": 1.0}
    w.baseline_iteration_ms = iter_ns / 1e6
    w.symr = symr
    return w


def side_streams(rng, ranks, iterations, iter_ns, span_ns, slow_rank, skews, entry_delay_ns=600_000,
                 rank_base=0):
    """Collectives (one AllReduce per iteration), GPU kernel events and 5 s OS
    counter windows for `ranks` ranks with ids rank_base + r."""
    c_rank, c_entry, c_exit = [], [], []
    g_rank, g_kern, g_start, g_dur = [], [], [], []
    for k in range(iterations):
        t0 = k * iter_ns
        barrier = t0 + int(iter_ns * 0.8)
        comp = (int(iter_ns * 0.7) + rng.normal(0, 50_000, size=ranks)).astype(np.int64)
        jit = rng.integers(-25_000, 25_001, size=ranks)
        for r in range(ranks):
            delay = entry_delay_ns if r == slow_rank else 0
            entry = t0 + int(comp[r]) + delay
            ex = max(barrier, entry + 1000) + int(jit[r])
            c_rank.append(rank_base + r)
            c_entry.append(entry + int(skews[r]))
            c_exit.append(max(ex, entry + 1) + int(skews[r]))
            ks = t0
            for kk, share in ((1, 0.48), (4, 0.19), (0, 0.15), (2, 0.18)):
                du = int(share * int(comp[r]) * np.exp(rng.normal(0, 0.01)))
                g_rank.append(rank_base + r)
                g_kern.append(kk)
                g_start.append(ks + int(skews[r]))
                g_dur.append(du)
                ks += du
            g_rank.append(rank_base + r)
            g_kern.append(3)
            g_start.append(entry + int(skews[r]))
            g_dur.append(max(0, barrier - entry))
    o_rank, o_ws, o_p50, o_p99, o_mig = [], [], [], [], []
    irq_off, irq_k, irq_v, sirq_off, sirq_k, sirq_v = [0], [], [], [0], [], []
    for r in range(ranks):
        storm = r == slow_rank
        for wnd in range(int(np.ceil(span_ns / 5e9)) or 1):
            j = lambda: rng.uniform(0.98, 1.02)
            o_rank.append(rank_base + r)
            o_ws.append(wnd * 5_000_000_000 + int(skews[r]))
            o_p50.append(int(50_000 * j()))
            o_p99.append(int(400_000 * j() * (6 if storm else 1)))
            o_mig.append(int(5 * j()))
            irq_k += [0, 2]
            irq_v += [int(10000 * j()), int(2000 * j() * (8 if storm else 1))]
            irq_off.append(len(irq_k))
            sirq_k += [4, 3, 1]
            sirq_v += [int(8000 * j()), int(6000 * j()), int(5000 * j() * (10 if storm else 1))]
            sirq_off.append(len(sirq_k))
    return dict(c_rank=c_rank, c_entry=c_entry, c_exit=c_exit, g_rank=g_rank, g_kern=g_kern,
                g_start=g_start, g_dur=g_dur, o_rank=o_rank, o_ws=o_ws, o_p50=o_p50, o_p99=o_p99,
                o_mig=o_mig, irq_off=irq_off, irq_k=irq_k, irq_v=irq_v, sirq_off=sirq_off,
                sirq_k=sirq_k, sirq_v=sirq_v, rank_base=rank_base)


def apply_side(w: Window, side: dict, ranks: int):
    n = len(side["c_rank"])
    w.coll_rank = np.asarray(side["c_rank"], np.int32)
    w.coll_group = np.zeros(n, np.int32)
    w.coll_kind = np.zeros(n, np.uint8)
    w.coll_entry = np.asarray(side["c_entry"], np.int64)
    w.coll_exit = np.asarray(side["c_exit"], np.int64)
    w.coll_gpu_dur = w.coll_exit - w.coll_entry
    w.group_ranks = np.arange(side["rank_base"], side["rank_base"] + ranks, dtype=np.int32)
    w.gpu_rank = np.asarray(side["g_rank"], np.int32)
    w.gpu_kernel = np.asarray(side["g_kern"], np.uint32)
    w.gpu_start = np.asarray(side["g_start"], np.int64)
    w.gpu_dur = np.asarray(side["g_dur"], np.int64)
    w.kernel_names = list(KERNELS)
    w.os_rank = np.asarray(side["o_rank"], np.int32)
    w.os_window_start = np.asarray(side["o_ws"], np.int64)
    w.os_p50 = np.asarray(side["o_p50"], np.int64)
    w.os_p99 = np.asarray(side["o_p99"], np.int64)
    w.os_migrations = np.asarray(side["o_mig"], np.int64)
    w.os_irq_off = np.asarray(side["irq_off"], np.uint64)
    w.os_irq_key = np.asarray(side["irq_k"], np.uint32)
    w.os_irq_val = np.asarray(side["irq_v"], np.int64)
    w.os_sirq_off = np.asarray(side["sirq_off"], np.uint64)
    w.os_sirq_key = np.asarray(side["sirq_k"], np.uint32)
    w.os_sirq_val = np.asarray(side["sirq_v"], np.int64)
    w.counter_names = list(COUNTERS)


C2_BINARIES = (("python3.11", "py"), ("libtorch_cuda.so", "at::native"), ("libcuda.so", "cu"))


def c2_tables(seed: int = 42, nsym: int = 1_000_000):
    """Three 1M-symbol tables (python, libtorch, cuda): sizes log-uniform 16-4096 B,
    ~10 % gap fraction.  The cuda table's first 9 names are the softirq path.
    Returns [(build_id, starts, sizes, symr)]."""
    rng = np.random.default_rng(seed)
    out = []
    for b, (label, prefix) in enumerate(C2_BINARIES):
        sizes = np.exp(rng.uniform(np.log(16), np.log(4096), nsym)).astype(np.uint32)
        gaps = (sizes * rng.uniform(0.0, 0.22, nsym)).astype(np.uint64)
        starts = (0x10000 + np.concatenate([[0], np.cumsum(sizes.astype(np.uint64) + gaps)[:-1]])).astype(np.uint64)
        names = [f"{prefix}_{i:07d}" for i in range(nsym)]
        if b == 2:
            names[:9] = SOFTIRQ
        bid = build_id(f"c2-{label}-{seed}")
        out.append((bid, starts, sizes, pack_symr(bid, starts, sizes, names)))
    return out


def c4_window(ranks: int = 1024, events_per_rank: int = 2000, seed: int = 1, slow: int = 4,
              device: bool = False, torch=None) -> Window:
    """per rank, events alternating AllReduce/AllGather every
    2 ms, exit = t + 1.2 ms +- 25 us, entry +- 25 us, per-rank clock skew
    U[-10, +10] ms, the slow rank enters 0.6 ms late, NET_RX storm on its NIC.
    device=True builds the collective arrays with torch on the GPU."""
    rng = np.random.default_rng(seed)
    skews = rng.integers(-10_000_000, 10_000_001, size=ranks).astype(np.int64)
    E = events_per_rank
    w = Window()
    if device:
        g = torch.Generator(device="cuda").manual_seed(seed)
        dev = torch.device("cuda")
        r = torch.arange(ranks, device=dev, dtype=torch.int64).repeat_interleave(E)
        e = torch.arange(E, device=dev, dtype=torch.int64).repeat(ranks)
        t = e * 2_000_000
        sk = torch.from_numpy(skews).to(dev)[r]
        je = torch.randint(-25_000, 25_001, (ranks * E,), device=dev, generator=g)
        jx = torch.randint(-25_000, 25_001, (ranks * E,), device=dev, generator=g)
        entry = t + je + sk + (r == slow).to(torch.int64) * 600_000
        exit_ = t + 1_200_000 + jx + sk
        w.coll_memory = 1
        w.n_coll_ = ranks * E
        w.coll_rank = r.to(torch.int32)
        w.coll_group = torch.zeros(ranks * E, dtype=torch.int32, device=dev)
        w.coll_kind = ((e % 2) * 2).to(torch.uint8)
        w.coll_entry, w.coll_exit = entry, exit_
        w.coll_gpu_dur = exit_ - entry
    else:
        r = np.repeat(np.arange(ranks, dtype=np.int64), E)
        e = np.tile(np.arange(E, dtype=np.int64), ranks)
        t = e * 2_000_000
        entry = t + rng.integers(-25_000, 25_001, ranks * E) + skews[r] + (r == slow) * 600_000
        exit_ = t + 1_200_000 + rng.integers(-25_000, 25_001, ranks * E) + skews[r]
        w.coll_rank = r.astype(np.int32)
        w.coll_group = np.zeros(ranks * E, np.int32)
        w.coll_kind = ((e % 2) * 2).astype(np.uint8)
        w.coll_entry, w.coll_exit = entry.astype(np.int64), exit_.astype(np.int64)
        w.coll_gpu_dur = w.coll_exit - w.coll_entry
    w.group_ranks = np.arange(ranks, dtype=np.int32)
    span = E * 2_000_000
    w.window_start_ns = 20_000_000
    w.window_end_ns = span
    w.max_skew_ns = 50_000_000
    side = side_streams(rng, ranks, 1, span, span, slow, skews)
    for k in ("c_rank", "c_entry", "c_exit", "g_rank", "g_kern", "g_start", "g_dur"):
        side[k] = []
    coll = {k: getattr(w, k) for k in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit",
                                       "coll_gpu_dur", "group_ranks")}
    apply_side(w, side, ranks)
    for k, v in coll.items():
        setattr(w, k, v)
    w.symr = []
    return w


def raw_stream(seed: int = 1, n: int = 2000, n_stacks: int = 40, max_depth: int = 12, n_bins: int = 2,
               span_ns: int = 17_000_000_000, t0: int = 3_000_000_000, rank: int = 3):
    """One rank's raw sample stream for aggregate_samples (samples.cpp:31-85):
    stacks drawn from a small population (so records merge), shared prefixes and
    near-duplicates (same frames, different bin; one frame more/less) so that the
    merge is by full stack, timestamps non-decreasing with repeats and gaps wider
    than the drain interval.  Returns (ts, rank[], frame_off, pc, bin, bin_ids)."""
    rng = np.random.default_rng(seed)
    pop = []
    for k in range(n_stacks):
        d = int(rng.integers(1, max_depth + 1))
        pcs = rng.integers(0x1000, 0x1000 + 64 * 40, size=d).astype(np.uint64) & ~np.uint64(3)
        bins = rng.integers(0, n_bins, size=d).astype(np.uint16)
        pop.append((pcs, bins))
        if k % 7 == 3:  # near-duplicates
            b2 = bins.copy()
            b2[-1] = (b2[-1] + 1) % n_bins
            pop.append((pcs.copy(), b2))
            pop.append((pcs[:-1].copy() if d > 1 else pcs.copy(), bins[:-1].copy() if d > 1 else bins.copy()))
    w = rng.zipf(1.4, size=n) % len(pop)
    steps = rng.integers(0, 2 * span_ns // max(n, 1) + 1, size=n)
    steps[rng.random(n) < 0.1] = 0
    jumps = rng.random(n) < 0.002
    steps[jumps] += 11_000_000_000
    ts = (t0 + np.cumsum(steps)).astype(np.int64)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(pop[i][0]) for i in w])
    pc = np.concatenate([pop[i][0] for i in w]) if n else np.zeros(0, np.uint64)
    bn = np.concatenate([pop[i][1] for i in w]) if n else np.zeros(0, np.uint16)
    ids = b"".join(build_id(f"raw{b}") for b in range(n_bins))
    return ts, np.full(n, rank, np.int32), off, pc, bn, ids


def oracle_stream(ts, rank, off, pc, bn, ids: bytes):
    """The same stream in strata_oracle.aggregate_samples' form."""
    bids = [ids[20 * b:20 * b + 20] for b in range(len(ids) // 20)]
    out = []
    for i in range(len(ts)):
        fr = tuple((bids[int(bn[f])], int(pc[f])) for f in range(int(off[i]), int(off[i + 1])))
        out.append((int(ts[i]), int(rank[i]) if rank is not None else 0, fr))
    return out


# ------------------------------------------------------------------ C2 on the host
_U = np.uint64


def _h64(z):
    """The bench generator's mixer (csrc/bench_gen.cu h64), vectorised over uint64."""
    with np.errstate(over="ignore"):
        z = z + _U(0x9e3779b97f4a7c15)
        z = (z ^ (z >> _U(30))) * _U(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> _U(27))) * _U(0x94d049bb133111eb)
        return z ^ (z >> _U(31))


def c2_samples_host(seed: int, ranks: int, spr: int, depth: int, pool: int, zipf_cdf, tables, hot,
                    soft_pc, slow_rank: int, soft_share: float, jit_per_million: int, period_ns: int, skew):
    """numpy restatement of the C2 bench generator (csrc/bench_gen.cu k_gen), bit-identical to it, for
    callers that must not load any repo library (bench.py --impl reference).  tables = [(starts, sizes)]
    of the three binaries; returns (ts, frame_off, frame_pc, frame_bin) host arrays."""
    n = ranks * spr
    i = np.arange(n, dtype=_U)
    r = (i // _U(spr)).astype(np.int64)
    k = (i % _U(spr)).astype(np.int64)
    with np.errstate(over="ignore"):
        u = _h64(_U(seed) ^ (i * _U(0x2545f4914f6cdd1d)))
        x = (u >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        lo = np.searchsorted(np.asarray(zipf_cdf, np.float64), x, side="left").astype(np.int64)
        lo = np.minimum(lo, pool - 1)
        p = ((lo + r.astype(np.int64) * 7919) % pool).astype(np.uint64)
        soft = (r == slow_rank) & ((_h64(u) >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0) < soft_share)
        jit = ~soft & ((_h64(u ^ _U(0x77)) % _U(1000000)) < _U(jit_per_million))
        jit_pc = _U(0x7f0000000000) + (_h64(u ^ _U(0x99)) % _U(1000)) * _U(16)
        skew = np.asarray(skew, np.int64)
        ts = k * period_ns + (_h64(u ^ _U(0x55)) % _U(period_ns // 50 + 1)).astype(np.int64) + skew[r]
        D = depth
        pc = np.zeros((n, D), np.uint64)
        bn = np.zeros((n, D), np.uint16)
        a, b = D // 5, D - D // 5
        for j in range(D):
            q = D - 1 - j
            bj = 0 if j < a else (1 if j < b else 2)
            bits = (p & _U((1 << j) - 1)) if j < 16 else p
            node = _h64(_U(seed) ^ _U(j << 40) ^ (bits << _U(1)) ^ _U(0 if j < 16 else 1))
            f = (node % _U(hot[bj])).astype(np.uint64)
            f = (f * _U(2654435761)) % _U(len(tables[bj][0]))
            st = np.asarray(tables[bj][0], np.uint64)[f.astype(np.int64)]
            sz = np.asarray(tables[bj][1], np.uint32)[f.astype(np.int64)].astype(np.uint64)
            if j == D - 1:
                off = _h64(u ^ _U(j)) % sz
            elif j == D - 10:
                off = np.where(soft, _h64(u ^ _U(j)) % sz, _h64(node ^ _U(0x1234)) % sz)
            else:
                off = _h64(node ^ _U(0x1234)) % sz
            col = st + off
            colb = np.full(n, bj, np.uint16)
            if j >= D - 9:
                col = np.where(soft, _U(int(soft_pc[j - (D - 9)])), col)
                colb = np.where(soft, np.uint16(2), colb)
            if j == D - 1:
                col = np.where(jit, jit_pc, col)
                colb = np.where(jit, np.uint16(3), colb)
            pc[:, q] = col
            bn[:, q] = colb
    foff = (np.arange(n + 1, dtype=np.uint64) * _U(D))
    return ts, foff, pc.reshape(-1), bn.reshape(-1)


def with_empty_stacks(w: Window, rank_index: int, samples) -> Window:
    """Copy of a host window with the listed samples (rank-relative indices, or
    "all") of one rank stripped of every frame (an empty StackSample.frames)."""
    import copy
    out = copy.copy(w)
    soff = np.asarray(w.rank_sample_off, np.uint64)
    s0, s1 = int(soff[rank_index]), int(soff[rank_index + 1])
    ks = range(s1 - s0) if samples == "all" else samples
    foff = np.asarray(w.sample_frame_off, np.uint64).astype(np.int64)
    keep = np.ones(int(foff[-1]), bool)
    lens = np.diff(foff)
    for k in ks:
        s = s0 + k
        keep[foff[s]:foff[s + 1]] = False
        lens[s] = 0
    out.frame_pc = np.asarray(w.frame_pc)[keep].copy()
    out.frame_bin = np.asarray(w.frame_bin)[keep].copy()
    out.sample_frame_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    out.n_frames_ = None
    return out
