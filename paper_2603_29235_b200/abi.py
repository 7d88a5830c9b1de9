"""ctypes mirror of include/stg.h plus the numpy structure-of-arrays `Window`.

`Window` is the Python-side form of `stg_window` (the in-memory equivalent of the
reference's `strata::LoadedBundle`, proj/core/include/strata/bundle.hpp:23-42).
Arrays are numpy (host) or torch CUDA tensors (device-resident bulk arrays);
`Window.to_c()` produces the `StgWindow` struct plus a keep-alive list.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

STG_OK, STG_EINVAL, STG_ECUDA, STG_ENOMEM, STG_ESTATE, STG_ENOTFOUND = range(6)
STG_MEM_HOST, STG_MEM_DEVICE = 0, 1
LOOKUP_EXACT_RANGE, LOOKUP_NEAREST_LOWER = 0, 1

VERDICTS = [
    "healthy",
    "gpu-uniform-slowdown",
    "gpu-specific-kernel",
    "cpu-interference",
    "os-interference",
    "temporal-degradation",
    "inconclusive",
]
KINDS = ["AllReduce", "ReduceScatter", "AllGather", "Broadcast", "P2P"]

_p = C.c_void_p


class StgWindow(C.Structure):
    _fields_ = [
        ("memory", C.c_int32),
        ("group", C.c_int32),
        ("window_start_ns", C.c_int64),
        ("window_end_ns", C.c_int64),
        ("max_skew_ns", C.c_int64),
        ("n_ranks", C.c_int32),
        ("rank_ids", _p),
        ("rank_sample_off", _p),
        ("n_bins", C.c_int32),
        ("bin_build_ids", _p),
        ("n_samples", C.c_uint64),
        ("sample_ts", _p),
        ("sample_frame_off", _p),
        ("n_frames", C.c_uint64),
        ("frame_pc", _p),
        ("frame_bin", _p),
        ("n_coll", C.c_uint64),
        ("coll_rank", _p),
        ("coll_group", _p),
        ("coll_kind", _p),
        ("coll_entry", _p),
        ("coll_exit", _p),
        ("coll_gpu_dur", _p),
        ("n_group_ranks", C.c_int32),
        ("group_ranks", _p),
        ("n_gpu", C.c_uint64),
        ("gpu_rank", _p),
        ("gpu_kernel", _p),
        ("gpu_start", _p),
        ("gpu_dur", _p),
        ("n_kernel_names", C.c_uint32),
        ("kernel_names", _p),
        ("n_os", C.c_uint64),
        ("os_rank", _p),
        ("os_window_start", _p),
        ("os_p50", _p),
        ("os_p99", _p),
        ("os_migrations", _p),
        ("os_irq_off", _p),
        ("os_irq_key", _p),
        ("os_irq_val", _p),
        ("os_sirq_off", _p),
        ("os_sirq_key", _p),
        ("os_sirq_val", _p),
        ("n_counter_names", C.c_uint32),
        ("counter_names", _p),
        ("has_baseline", C.c_int32),
        ("baseline_delta", C.c_double),
        ("n_baseline", C.c_uint32),
        ("baseline_names", _p),
        ("baseline_fracs", _p),
        ("has_baseline_iteration", C.c_int32),
        ("baseline_iteration_ms", C.c_double),
        ("coll_memory", C.c_int32),
        ("side_memory", C.c_int32),
        ("shard_streams", C.c_int32),
        ("shard_rank_lo", C.c_int32),
    ]


class StgConfig(C.Structure):
    _fields_ = [
        ("window_iterations", C.c_int32),
        ("k", C.c_double),
        ("delta", C.c_double),
        ("iteration_regression_gate", C.c_double),
        ("gpu_median_uniform", C.c_double),
        ("gpu_cv_uniform", C.c_double),
        ("gpu_top_share_specific", C.c_double),
        ("gpu_median_none", C.c_double),
        ("gpu_ref_floor_ns", C.c_int64),
        ("gpu_exclude_prefix", C.c_char * 32),
        ("os_min_ratio", C.c_double),
        ("os_interrupt_floor", C.c_int64),
        ("os_sched_delay_floor_ns", C.c_int64),
        ("os_migration_floor", C.c_int64),
        ("lookup_mode", C.c_int32),
        ("want_waterline", C.c_int32),
        ("verify", C.c_int32),
        ("debug_weak_prefix_key", C.c_int32),
    ]


class StgSvgOptions(C.Structure):
    """stg_svg_options (SvgOptions, svg.hpp)."""
    _fields_ = [("width", C.c_int32), ("row_height", C.c_int32), ("min_fraction", C.c_double),
                ("title", C.c_char_p)]


class StgRunStats(C.Structure):
    _fields_ = [
        ("n_samples_in_window", C.c_uint64),
        ("n_lines", C.c_uint64),
        ("n_sequences", C.c_uint64),
        ("n_names", C.c_uint64),
        ("n_unknown", C.c_uint64),
        ("n_instances", C.c_uint64),
        ("n_windowed", C.c_uint64),
        ("n_cpu_ranks", C.c_uint64),
        ("verdict", C.c_int32),
        ("n_flagged", C.c_int32),
        ("ms_collectives", C.c_float),
        ("ms_symbolize", C.c_float),
        ("ms_fold", C.c_float),
        ("ms_diff", C.c_float),
        ("ms_total", C.c_float),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint32),
        ("agg_attempts", C.c_uint32),
        ("prefix_hits", C.c_uint64),
        ("prefix_misses", C.c_uint64),
        ("verified", C.c_uint32),
        ("verify_retries", C.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def default_config() -> dict:
    """DiagnosisConfig defaults (diagnosis.hpp:83-92,127-132,203-210)."""
    return dict(
        window_iterations=100,
        k=2.0,
        delta=0.005,
        iteration_regression_gate=0.03,
        gpu_median_uniform=0.03,
        gpu_cv_uniform=0.25,
        gpu_top_share_specific=0.60,
        gpu_median_none=0.01,
        gpu_ref_floor_ns=1_000_000,
        gpu_exclude_prefix="nccl",
        os_min_ratio=2.0,
        os_interrupt_floor=1000,
        os_sched_delay_floor_ns=1_000_000,
        os_migration_floor=100,
        lookup_mode=LOOKUP_EXACT_RANGE,
        want_waterline=0,
        verify=0,
        debug_weak_prefix_key=0,
    )


def config_struct(cfg: Optional[dict] = None) -> StgConfig:
    d = default_config()
    if cfg:
        d.update(cfg)
    c = StgConfig()
    for k, v in d.items():
        if k == "gpu_exclude_prefix":
            c.gpu_exclude_prefix = v.encode()
        else:
            setattr(c, k, v)
    return c


class StgStream(C.Structure):
    """stg_stream (include/stg.h): one rank's raw sample stream for aggregate_samples."""
    _fields_ = [
        ("memory", C.c_int32),
        ("n_samples", C.c_uint64),
        ("ts", _p),
        ("rank", _p),
        ("frame_off", _p),
        ("frame_pc", _p),
        ("frame_bin", _p),
    ]


STG_AGG_FORCE_EXACT = 1
STG_SHARD_COLL = 1
STG_SHARD_SIDE = 2


class StgBundleInfo(C.Structure):
    """stg_bundle_info (include/stg.h)."""
    _fields_ = [
        ("n_ranks", C.c_uint32), ("n_bins", C.c_uint32), ("n_tables_ingested", C.c_uint32), ("pad", C.c_uint32),
        ("n_samples", C.c_uint64), ("n_frames", C.c_uint64), ("n_coll", C.c_uint64), ("n_gpu", C.c_uint64),
        ("n_os", C.c_uint64), ("bulk_bytes", C.c_uint64), ("read_s", C.c_double), ("decode_s", C.c_double),
        ("total_s", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


def _ptr(a, keep: list):
    """Pointer to a numpy array (host) or torch tensor (device); None -> NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        keep.append(a)
        return a.data_ptr()
    a = np.ascontiguousarray(a)
    keep.append(a)
    return a.ctypes.data


def _strings(names: List[str], keep: list):
    arr = (C.c_char_p * max(len(names), 1))()
    enc = [n.encode() for n in names]
    keep.append(enc)
    for i, e in enumerate(enc):
        arr[i] = e
    keep.append(arr)
    return C.cast(arr, C.c_void_p).value


@dataclass
class Window:
    """Structure-of-arrays analysis window (stg_window)."""

    window_start_ns: int = 0
    window_end_ns: int = 0
    max_skew_ns: int = 50_000_000
    group: int = 0
    rank_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    rank_sample_off: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    bin_build_ids: np.ndarray = field(default_factory=lambda: np.zeros((0, 20), np.uint8))
    sample_ts: object = field(default_factory=lambda: np.zeros(0, np.int64))
    sample_frame_off: object = field(default_factory=lambda: np.zeros(1, np.uint64))
    frame_pc: object = field(default_factory=lambda: np.zeros(0, np.uint64))
    frame_bin: object = field(default_factory=lambda: np.zeros(0, np.uint16))
    memory: int = STG_MEM_HOST
    coll_memory: int = STG_MEM_HOST
    side_memory: int = STG_MEM_HOST
    shard_streams: int = 0  # STG_SHARD_COLL | STG_SHARD_SIDE (distributed mode)
    shard_rank_lo: int = 0
    n_gpu_: Optional[int] = None
    n_os_: Optional[int] = None
    n_coll_: Optional[int] = None
    n_samples_: Optional[int] = None
    n_frames_: Optional[int] = None
    # collectives
    coll_rank: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    coll_group: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    coll_kind: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    coll_entry: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    coll_exit: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    coll_gpu_dur: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    group_ranks: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    # gpu events
    gpu_rank: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    gpu_kernel: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    gpu_start: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    gpu_dur: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    kernel_names: List[str] = field(default_factory=list)
    # os counters
    os_rank: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    os_window_start: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    os_p50: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    os_p99: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    os_migrations: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    os_irq_off: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    os_irq_key: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    os_irq_val: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    os_sirq_off: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    os_sirq_key: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    os_sirq_val: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    counter_names: List[str] = field(default_factory=list)
    # baseline
    has_baseline: bool = False
    baseline_delta: float = 0.005
    baseline: Dict[str, float] = field(default_factory=dict)
    baseline_iteration_ms: Optional[float] = None
    # symbol tables (SYMR payloads) the window's binaries resolve against
    symr: List[bytes] = field(default_factory=list)
    labels: Optional[dict] = None

    @property
    def n_samples(self) -> int:
        if self.n_samples_ is not None:
            return self.n_samples_
        return int(len(self.sample_ts))

    @property
    def n_frames(self) -> int:
        if self.n_frames_ is not None:
            return self.n_frames_
        return int(len(self.frame_pc))

    def to_c(self):
        keep: list = []
        w = StgWindow()
        w.memory = self.memory
        w.group = self.group
        w.window_start_ns = int(self.window_start_ns)
        w.window_end_ns = int(self.window_end_ns)
        w.max_skew_ns = int(self.max_skew_ns)
        w.n_ranks = len(self.rank_ids)
        w.rank_ids = _ptr(np.asarray(self.rank_ids, np.int32), keep)
        w.rank_sample_off = _ptr(np.asarray(self.rank_sample_off, np.uint64), keep)
        bids = np.ascontiguousarray(np.asarray(self.bin_build_ids, np.uint8).reshape(-1, 20))
        w.n_bins = bids.shape[0]
        w.bin_build_ids = _ptr(bids, keep)
        w.n_samples = self.n_samples
        w.n_frames = self.n_frames
        if self.memory == STG_MEM_HOST:
            w.sample_ts = _ptr(np.asarray(self.sample_ts, np.int64), keep)
            w.sample_frame_off = _ptr(np.asarray(self.sample_frame_off, np.uint64), keep)
            w.frame_pc = _ptr(np.asarray(self.frame_pc, np.uint64), keep)
            w.frame_bin = _ptr(np.asarray(self.frame_bin, np.uint16), keep)
        else:
            w.sample_ts = _ptr(self.sample_ts, keep)
            w.sample_frame_off = _ptr(self.sample_frame_off, keep)
            w.frame_pc = _ptr(self.frame_pc, keep)
            w.frame_bin = _ptr(self.frame_bin, keep)
        w.coll_memory = self.coll_memory
        if self.coll_memory == STG_MEM_HOST:
            w.n_coll = len(self.coll_rank)
            w.coll_rank = _ptr(np.asarray(self.coll_rank, np.int32), keep)
            w.coll_group = _ptr(np.asarray(self.coll_group, np.int32), keep)
            w.coll_kind = _ptr(np.asarray(self.coll_kind, np.uint8), keep)
            w.coll_entry = _ptr(np.asarray(self.coll_entry, np.int64), keep)
            w.coll_exit = _ptr(np.asarray(self.coll_exit, np.int64), keep)
            w.coll_gpu_dur = _ptr(np.asarray(self.coll_gpu_dur, np.int64), keep)
        else:
            w.n_coll = self.n_coll_ if self.n_coll_ is not None else int(self.coll_rank.numel())
            for f in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur"):
                setattr(w, f, _ptr(getattr(self, f), keep))
        w.n_group_ranks = len(self.group_ranks)
        w.group_ranks = _ptr(np.asarray(self.group_ranks, np.int32), keep)
        w.side_memory = self.side_memory
        gpu_f = (("gpu_rank", np.int32), ("gpu_kernel", np.uint32), ("gpu_start", np.int64), ("gpu_dur", np.int64))
        os_f = (("os_rank", np.int32), ("os_window_start", np.int64), ("os_p50", np.int64), ("os_p99", np.int64),
                ("os_migrations", np.int64), ("os_irq_off", np.uint64), ("os_irq_key", np.uint32),
                ("os_irq_val", np.int64), ("os_sirq_off", np.uint64), ("os_sirq_key", np.uint32),
                ("os_sirq_val", np.int64))
        if self.side_memory == STG_MEM_HOST:
            w.n_gpu = len(self.gpu_rank)
            w.n_os = len(self.os_rank)
            for f, dt in gpu_f + os_f:
                setattr(w, f, _ptr(np.asarray(getattr(self, f), dt), keep))
        else:  # device tensors (data_ptr)
            w.n_gpu = self.n_gpu_ if self.n_gpu_ is not None else int(self.gpu_rank.numel())
            w.n_os = self.n_os_ if self.n_os_ is not None else int(self.os_rank.numel())
            for f, _ in gpu_f + os_f:
                setattr(w, f, _ptr(getattr(self, f), keep))
        w.n_kernel_names = len(self.kernel_names)
        w.kernel_names = _strings(self.kernel_names, keep)
        w.n_counter_names = len(self.counter_names)
        w.counter_names = _strings(self.counter_names, keep)
        w.has_baseline = int(bool(self.has_baseline))
        w.baseline_delta = float(self.baseline_delta)
        names = list(self.baseline.keys())
        w.n_baseline = len(names)
        w.baseline_names = _strings(names, keep)
        w.baseline_fracs = _ptr(np.array([self.baseline[n] for n in names], np.float64), keep)
        w.has_baseline_iteration = int(self.baseline_iteration_ms is not None)
        w.baseline_iteration_ms = float(self.baseline_iteration_ms or 0.0)
        w.shard_streams = int(self.shard_streams)
        w.shard_rank_lo = int(self.shard_rank_lo)
        return w, keep

    @staticmethod
    def from_c(w: StgWindow) -> "Window":
        """Deep-copies a host StgWindow (e.g. from the reference simulator)."""

        def arr(ptr, n, dt):
            if n == 0 or not ptr:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (n,)).copy()

        def strs(ptr, n):
            if n == 0:
                return []
            a = C.cast(ptr, C.POINTER(C.c_char_p))
            return [a[i].decode() for i in range(n)]

        out = Window()
        out.memory = STG_MEM_HOST
        out.group = w.group
        out.window_start_ns = w.window_start_ns
        out.window_end_ns = w.window_end_ns
        out.max_skew_ns = w.max_skew_ns
        out.rank_ids = arr(w.rank_ids, w.n_ranks, np.int32)
        out.rank_sample_off = arr(w.rank_sample_off, w.n_ranks + 1, np.uint64)
        out.bin_build_ids = arr(w.bin_build_ids, w.n_bins * 20, np.uint8).reshape(-1, 20)
        out.sample_ts = arr(w.sample_ts, w.n_samples, np.int64)
        out.sample_frame_off = arr(w.sample_frame_off, w.n_samples + 1, np.uint64)
        out.frame_pc = arr(w.frame_pc, w.n_frames, np.uint64)
        out.frame_bin = arr(w.frame_bin, w.n_frames, np.uint16)
        out.coll_rank = arr(w.coll_rank, w.n_coll, np.int32)
        out.coll_group = arr(w.coll_group, w.n_coll, np.int32)
        out.coll_kind = arr(w.coll_kind, w.n_coll, np.uint8)
        out.coll_entry = arr(w.coll_entry, w.n_coll, np.int64)
        out.coll_exit = arr(w.coll_exit, w.n_coll, np.int64)
        out.coll_gpu_dur = arr(w.coll_gpu_dur, w.n_coll, np.int64)
        out.group_ranks = arr(w.group_ranks, w.n_group_ranks, np.int32)
        out.gpu_rank = arr(w.gpu_rank, w.n_gpu, np.int32)
        out.gpu_kernel = arr(w.gpu_kernel, w.n_gpu, np.uint32)
        out.gpu_start = arr(w.gpu_start, w.n_gpu, np.int64)
        out.gpu_dur = arr(w.gpu_dur, w.n_gpu, np.int64)
        out.kernel_names = strs(w.kernel_names, w.n_kernel_names)
        out.os_rank = arr(w.os_rank, w.n_os, np.int32)
        out.os_window_start = arr(w.os_window_start, w.n_os, np.int64)
        out.os_p50 = arr(w.os_p50, w.n_os, np.int64)
        out.os_p99 = arr(w.os_p99, w.n_os, np.int64)
        out.os_migrations = arr(w.os_migrations, w.n_os, np.int64)
        out.os_irq_off = arr(w.os_irq_off, w.n_os + 1, np.uint64)
        n_irq = int(out.os_irq_off[-1]) if len(out.os_irq_off) else 0
        out.os_irq_key = arr(w.os_irq_key, n_irq, np.uint32)
        out.os_irq_val = arr(w.os_irq_val, n_irq, np.int64)
        out.os_sirq_off = arr(w.os_sirq_off, w.n_os + 1, np.uint64)
        n_sirq = int(out.os_sirq_off[-1]) if len(out.os_sirq_off) else 0
        out.os_sirq_key = arr(w.os_sirq_key, n_sirq, np.uint32)
        out.os_sirq_val = arr(w.os_sirq_val, n_sirq, np.int64)
        out.counter_names = strs(w.counter_names, w.n_counter_names)
        out.has_baseline = bool(w.has_baseline)
        out.baseline_delta = w.baseline_delta
        bn = strs(w.baseline_names, w.n_baseline)
        bf = arr(w.baseline_fracs, w.n_baseline, np.float64)
        out.baseline = {n: float(f) for n, f in zip(bn, bf)}
        out.baseline_iteration_ms = w.baseline_iteration_ms if w.has_baseline_iteration else None
        return out
