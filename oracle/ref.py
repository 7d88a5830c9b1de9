"""TEST INFRASTRUCTURE ONLY — ctypes driver for oracle/_ref/libstrata_ref.so.

libstrata_ref.so is the UNMODIFIED reference (strata, /root/reference/proj/core)
compiled in place by oracle/Makefile plus oracle/ref_harness.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
use this module; the product (paper_2603_29235_b200/) never imports oracle/.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile
from pathlib import Path
from typing import List, Optional

import numpy as np

from paper_2603_29235_b200.abi import StgWindow, Window

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libstrata_ref.so"
_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        l = C.CDLL(str(LIB_PATH))
        l.ref_sim_create.restype = C.c_void_p
        l.ref_sim_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_double,
                                     C.c_double, C.c_int, C.c_int, C.c_char_p, C.c_int]
        l.ref_sim_window.argtypes = [C.c_void_p, C.POINTER(StgWindow)]
        l.ref_sim_symr_count.argtypes = [C.c_void_p]
        l.ref_sim_symr.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
        l.ref_sim_labels_json.restype = C.c_char_p
        l.ref_sim_labels_json.argtypes = [C.c_void_p]
        l.ref_sim_free.argtypes = [C.c_void_p]
        l.ref_free.argtypes = [C.c_void_p]
        l.ref_window_run.argtypes = [C.POINTER(StgWindow), C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.c_char_p, C.c_int]
        l.ref_lookup.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int,
                                 C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
        l.ref_parse_symbols.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_int]
        l.ref_pack_symbols.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64),
                                       C.c_char_p, C.c_int]
        l.ref_unknown_label.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_int]
        l.ref_digest.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p]
        l.ref_collectives.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                      C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        l.ref_detect_straggler.argtypes = [C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_double, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        l.ref_waterline.argtypes = [C.POINTER(StgWindow), C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_char_p, C.c_double, C.POINTER(C.c_void_p), C.c_char_p,
                                    C.c_int]
        _lib = l
    return _lib


class RefError(Exception):
    """strata::Error raised by the reference."""


def _take_json(p: C.c_void_p):
    s = C.cast(p, C.c_char_p).value.decode()
    lib().ref_free(p)
    return json.loads(s)


def simulate(scenario: str, seed: int, ranks: int = 0, iterations: int = 0,
             sample_rate_hz: float = 0.0, magnitude: float = 0.0,
             onset_iteration: int = -1, analysis_window: int = 0) -> Window:
    """simulate(default_spec(scenario, seed)) with overrides -> Window (+ symr, labels)."""
    err = C.create_string_buffer(512)
    h = lib().ref_sim_create(scenario.encode(), seed, ranks, iterations, sample_rate_hz,
                             magnitude, onset_iteration, analysis_window, err, 512)
    if not h:
        raise RefError(err.value.decode())
    try:
        w = StgWindow()
        lib().ref_sim_window(h, C.byref(w))
        out = Window.from_c(w)
        syms = []
        for i in range(lib().ref_sim_symr_count(h)):
            p, n = C.c_void_p(), C.c_uint64()
            lib().ref_sim_symr(h, i, C.byref(p), C.byref(n))
            syms.append(C.string_at(p, n.value))
        out.symr = syms
        out.labels = json.loads(lib().ref_sim_labels_json(h).decode())
        return out
    finally:
        lib().ref_sim_free(h)


def window_run(win: Window, threads: int = 1, want_json: bool = True,
               tmpdir: Optional[str] = None, artifacts: bool = False, shared_cache: bool = False):
    """Reference build_group_data + diagnose.  Returns (result_json, t_build_s, t_diag_s).

    artifacts=True adds result_json["artifacts"]: FoldedProfile::to_string of every
    rank and diff_folded texts (see ref_harness.cpp).  shared_cache=True symbolizes
    each rank's records with the reference's resolve_stacks (one table cache per
    rank) + fold_symbolized instead of to_folded's per-record table reload: the
    same folded profiles (ref_harness.cpp build_group_data_threads), feasible on
    1M-symbol tables."""
    cw, keep = win.to_c()
    n = len(win.symr)
    bufs = [C.create_string_buffer(s, len(s)) for s in win.symr]
    ptrs = (C.c_void_p * max(n, 1))(*[C.cast(b, C.c_void_p) for b in bufs])
    lens = (C.c_uint64 * max(n, 1))(*[len(s) for s in win.symr])
    out = C.c_void_p()
    tb, td = C.c_double(), C.c_double()
    err = C.create_string_buffer(1024)
    tmp = tmpdir or tempfile.gettempdir()
    L = lib()
    L.ref_window_run_ex.argtypes = [C.POINTER(StgWindow), C.c_int, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int,
                                    C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.c_char_p, C.c_int]
    rc = L.ref_window_run_ex(C.byref(cw), n, ptrs, lens, tmp.encode(), threads, int(shared_cache),
                             2 if artifacts else int(want_json), C.byref(out), C.byref(tb), C.byref(td), err, 1024)
    if rc != 0:
        raise RefError(err.value.decode())
    return _take_json(out), tb.value, td.value


def waterline(win: Window, k: float = 2.0, tmpdir: Optional[str] = None):
    cw, keep = win.to_c()
    n = len(win.symr)
    bufs = [C.create_string_buffer(s, len(s)) for s in win.symr]
    ptrs = (C.c_void_p * max(n, 1))(*[C.cast(b, C.c_void_p) for b in bufs])
    lens = (C.c_uint64 * max(n, 1))(*[len(s) for s in win.symr])
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    tmp = tmpdir or tempfile.gettempdir()
    rc = lib().ref_waterline(C.byref(cw), n, ptrs, lens, tmp.encode(), k, C.byref(out), err, 1024)
    if rc != 0:
        raise RefError(err.value.decode())
    return _take_json(out)


def lookup(symr: bytes, offsets, mode: int):
    """SymbolFile::lookup over offsets -> (entry index or -1, probe counts)."""
    offs = np.ascontiguousarray(offsets, np.uint64)
    idx = np.zeros(len(offs), np.int64)
    probes = np.zeros(len(offs), np.uint64)
    err = C.create_string_buffer(512)
    rc = lib().ref_lookup(symr, len(symr), len(offs), offs.ctypes.data, mode,
                          idx.ctypes.data, probes.ctypes.data, err, 512)
    if rc != 0:
        raise RefError(err.value.decode())
    return idx, probes


def parse_error(symr: bytes) -> Optional[str]:
    err = C.create_string_buffer(512)
    rc = lib().ref_parse_symbols(symr, len(symr), err, 512)
    return None if rc == 0 else err.value.decode()


def pack_symbols(build_id: bytes, entries) -> bytes:
    """pack_symbols(id, [(start, size, name), ...])."""
    starts = np.array([e[0] for e in entries], np.uint64)
    sizes = np.array([e[1] for e in entries], np.uint32)
    blob = b"".join(e[2].encode() + b"\0" for e in entries) or b"\0"
    out, n = C.c_void_p(), C.c_uint64()
    err = C.create_string_buffer(512)
    bid = C.create_string_buffer(bytes(build_id), 20)
    rc = lib().ref_pack_symbols(bid, len(entries), starts.ctypes.data, sizes.ctypes.data, blob,
                                C.byref(out), C.byref(n), err, 512)
    if rc != 0:
        raise RefError(err.value.decode())
    data = C.string_at(out, n.value)
    lib().ref_free(out)
    return data


def unknown_label(build_id: bytes, off: int) -> str:
    buf = C.create_string_buffer(128)
    bid = C.create_string_buffer(bytes(build_id), 20)
    lib().ref_unknown_label(bid, off, buf, 128)
    return buf.value.decode()


def digest(data: bytes) -> bytes:
    out = C.create_string_buffer(20)
    lib().ref_digest(data, len(data), out)
    return out.raw


def collectives(rank, group, kind, entry, exit_, dur, group_ranks, max_skew=50_000_000):
    a = [np.ascontiguousarray(x, dt) for x, dt in
         ((rank, np.int32), (group, np.int32), (kind, np.uint8), (entry, np.int64),
          (exit_, np.int64), (dur, np.int64))]
    gr = np.ascontiguousarray(group_ranks, np.int32)
    out = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib().ref_collectives(len(a[0]), *[x.ctypes.data for x in a], len(gr), gr.ctypes.data,
                               max_skew, C.byref(out), err, 512)
    if rc != 0:
        raise RefError(err.value.decode())
    return _take_json(out)


def detect_straggler(lat: np.ndarray, ranks, k: float = 2.0):
    lat = np.ascontiguousarray(lat, np.float64)
    rk = np.ascontiguousarray(ranks, np.int32)
    out = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib().ref_detect_straggler(lat.shape[0], len(rk), rk.ctypes.data, lat.ctypes.data, k,
                                    C.byref(out), err, 512)
    if rc != 0:
        raise RefError(err.value.decode())
    return _take_json(out)


def aggregate_samples(ts, frame_off, frame_pc, frame_bin, bin_ids: bytes, rank=None,
                      drain: int = 5_000_000_000, time_only: bool = False):
    """Reference aggregate_samples (samples.cpp:31-85) on a raw SoA stream.
    Returns [(rank, start, end, [(first_sample, count), ...])], or with
    time_only=True the seconds spent inside aggregate_samples alone."""
    ts = np.ascontiguousarray(ts, np.int64)
    foff = np.ascontiguousarray(frame_off, np.uint64)
    pc = np.ascontiguousarray(frame_pc, np.uint64)
    bn = np.ascontiguousarray(frame_bin, np.uint16)
    rk = None if rank is None else np.ascontiguousarray(rank, np.int32)
    ids = np.frombuffer(bin_ids, np.uint8).copy()
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    L = lib()
    L.ref_aggregate_samples.argtypes = [C.c_uint64] + [C.c_void_p] * 5 + [C.c_int, C.c_void_p, C.c_int64,
                                                                         C.c_void_p, C.POINTER(C.c_double),
                                                                         C.c_char_p, C.c_int]
    t = C.c_double()
    rc = L.ref_aggregate_samples(len(ts), ts.ctypes.data, None if rk is None else rk.ctypes.data,
                                 foff.ctypes.data, pc.ctypes.data, bn.ctypes.data, len(ids) // 20,
                                 ids.ctypes.data, int(drain), None if time_only else C.addressof(out),
                                 C.byref(t), err, 1024)
    if rc != 0:
        raise RefError(err.value.decode())
    if time_only:
        return t.value
    j = _take_json(out)
    return [(w[0], w[1], w[2], [tuple(r) for r in w[3]]) for w in j["windows"]]


def write_bundle(scenario: str, seed: int, dirpath: str, ranks: int = 0, iterations: int = 0,
                 sample_rate_hz: float = 0.0):
    """Simulate a scenario and write_bundle (bundle.cpp:83-164) it to dirpath."""
    err = C.create_string_buffer(1024)
    h = lib().ref_sim_create(scenario.encode(), seed, ranks, iterations, sample_rate_hz, 0.0, -1, 0, err, 1024)
    if not h:
        raise RefError(err.value.decode())
    try:
        L = lib()
        L.ref_sim_write_bundle.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]
        if L.ref_sim_write_bundle(h, str(dirpath).encode(), err, 1024) != 0:
            raise RefError(err.value.decode())
    finally:
        lib().ref_sim_free(h)


def bundle_run(dirpath: str, want_json: bool = True):
    """Reference load_bundle + build_group_data + diagnose.
    Returns (result_json, t_load_s, t_build_s, t_diag_s)."""
    L = lib()
    L.ref_bundle_run.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_int]
    out = C.c_void_p()
    tl, tb, td = C.c_double(), C.c_double(), C.c_double()
    err = C.create_string_buffer(1024)
    if L.ref_bundle_run(str(dirpath).encode(), int(want_json), C.byref(out), C.byref(tl), C.byref(tb),
                        C.byref(td), err, 1024) != 0:
        raise RefError(err.value.decode())
    return _take_json(out), tl.value, tb.value, td.value


def bundle_load_time(dirpath: str):
    """Reference load_bundle alone: (seconds, samples)."""
    L = lib()
    L.ref_bundle_load_time.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_char_p,
                                       C.c_int]
    t, n = C.c_double(), C.c_uint64()
    err = C.create_string_buffer(1024)
    if L.ref_bundle_load_time(str(dirpath).encode(), C.byref(t), C.byref(n), err, 1024) != 0:
        raise RefError(err.value.decode())
    return t.value, n.value
