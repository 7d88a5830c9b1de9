"""paper_2603_29235_b200 — SysOM-AI's per-window analysis hot path on B200.

The product is libstg.so (include/stg.h): hand-written sm_100a CUDA behind a
C-ABI.  This module is the thin Python host binding used by tests and bench.py;
it mirrors the reference's verbs (proj/core/include/strata/*.hpp):

    Context.ingest(symr)            SymbolRepository::ingest / parse_symbols
    Context.resolve(...)            resolve_stacks
    Context.window_run(win)         build_group_data + diagnose
    Context.groupdata() / report()  GroupData / DiagnosisReport::to_json

There is no CPU fallback: if libstg.so is missing or no GPU is visible, every
call raises.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path
from typing import Optional

import numpy as np

from .abi import (STG_AGG_FORCE_EXACT, STG_MEM_DEVICE, STG_MEM_HOST, VERDICTS, StgBundleInfo, StgConfig,
                  StgRunStats, StgStream, StgSvgOptions, StgWindow, Window, _ptr, config_struct, default_config)

__all__ = ["Context", "StgError", "Window", "load_library", "LIB_PATH", "VERDICTS",
           "default_config"]

LIB_PATH = Path(__file__).resolve().parent / "libstg.so"
_lib = None


class StgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing — run `python -m paper_2603_29235_b200.build` "
                           "(there is no CPU fallback)")
    l = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    l.stg_last_error.restype = C.c_char_p
    l.stg_create.argtypes = [C.c_int, C.POINTER(P)]
    l.stg_destroy.argtypes = [P]
    l.stg_symtab_ingest.argtypes = [P, C.c_char_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_int)]
    l.stg_symtab_count.argtypes = [P, C.POINTER(C.c_uint32)]
    l.stg_resolve.argtypes = [P, C.c_uint64, P, P, C.c_int32, P, C.c_int, P]
    l.stg_name.argtypes = [P, C.c_uint32, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    l.stg_name_count.argtypes = [P, C.POINTER(C.c_uint32)]
    l.stg_config_default.argtypes = [C.POINTER(StgConfig)]
    l.stg_window_run.argtypes = [P, C.POINTER(StgWindow), C.POINTER(StgConfig), C.POINTER(StgRunStats)]
    for fn in ("stg_result_groupdata_json", "stg_result_report_json", "stg_result_waterline_json",
               "stg_result_report_text"):
        getattr(l, fn).argtypes = [P, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    l.stg_dist_unique_id.argtypes = [C.c_char_p]
    l.stg_dist_init.argtypes = [P, C.c_int, C.c_int, C.c_char_p]
    l.stg_result_folded_text.argtypes = [P, C.c_int32, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    l.stg_result_flamegraph_svg.argtypes = [P, C.c_int32, C.POINTER(StgSvgOptions), C.c_char_p, C.c_uint64,
                                            C.POINTER(C.c_uint64)]
    l.stg_result_diff_flamegraph_svg.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(StgSvgOptions), C.c_char_p,
                                                 C.c_uint64, C.POINTER(C.c_uint64)]
    l.stg_result_diff_folded.argtypes = [P, C.c_int32, C.c_int32, C.c_char_p, C.c_uint64,
                                         C.POINTER(C.c_uint64)]
    l.stg_bundle_load.argtypes = [P, C.c_char_p, C.POINTER(StgBundleInfo)]
    l.stg_bundle_window.argtypes = [P, C.POINTER(StgWindow)]
    l.stg_device_to_host.argtypes = [P, P, P, C.c_uint64]
    l.stg_aggregate_samples.argtypes = [P, C.POINTER(StgStream), C.c_int64, C.c_int, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]
    l.stg_aggregate_windows.argtypes = [P, P, P, P]
    l.stg_aggregate_records.argtypes = [P, P, P]
    l.stg_result_rank_count.argtypes = [P, C.POINTER(C.c_uint32)]
    l.stg_result_rank_info.argtypes = [P, C.c_uint32, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    l.stg_result_rank_lines.argtypes = [P, C.c_uint32, P, P, P]
    _lib = l
    return l


def _check(rc: int):
    if rc != 0:
        raise StgError(rc, load_library().stg_last_error().decode())


class Context:
    """One libstg context bound to one GPU."""

    def __init__(self, device: int = 0):
        self._l = load_library()
        self._h = C.c_void_p()
        _check(self._l.stg_create(device, C.byref(self._h)))
        self.last_stats: Optional[dict] = None

    def close(self):
        if self._h:
            self._l.stg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- distributed
    @staticmethod
    def dist_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(load_library().stg_dist_unique_id(buf))
        return buf.raw

    def dist_init(self, world: int, rank: int, uid: bytes):
        """Join an NCCL group spanning `world` contexts (see include/stg.h)."""
        assert len(uid) == 128
        _check(self._l.stg_dist_init(self._h, world, rank, uid))

    # ---------------------------------------------------------------- ingest
    def ingest(self, symr: bytes, claimed_id: Optional[bytes] = None) -> bool:
        stored = C.c_int(0)
        _check(self._l.stg_symtab_ingest(self._h, claimed_id, symr, len(symr), C.byref(stored)))
        return bool(stored.value)

    def table_count(self) -> int:
        n = C.c_uint32()
        _check(self._l.stg_symtab_count(self._h, C.byref(n)))
        return n.value

    # ------------------------------------------------------------- symbolize
    def resolve(self, pcs, bins, build_ids, mode: int = 0):
        """Frame-wise names (resolve_stacks); returns a list of strings."""
        pcs = np.ascontiguousarray(pcs, np.uint64)
        bins = np.ascontiguousarray(bins, np.uint16)
        ids = np.ascontiguousarray(np.asarray(build_ids, np.uint8).reshape(-1, 20))
        out = np.zeros(len(pcs), np.uint32)
        _check(self._l.stg_resolve(self._h, len(pcs), pcs.ctypes.data, bins.ctypes.data, ids.shape[0],
                                   ids.ctypes.data, mode, out.ctypes.data))
        return [self.name(int(k)) for k in out], out

    def name(self, key: int) -> str:
        need = C.c_uint64()
        _check(self._l.stg_name(self._h, key, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(self._l.stg_name(self._h, key, buf, need.value, C.byref(need)))
        # names are arbitrary bytes (NUL and non-UTF-8 included): keep them all
        return buf.raw[:need.value - 1].decode("utf-8", "surrogateescape")

    # ---------------------------------------------------------------- bundle
    def load_bundle(self, path) -> dict:
        """load_bundle (bundle.cpp:181-233) with the bulk files decoded on the GPU;
        the bundle's symbol tables are ingested.  Returns stg_bundle_info."""
        info = StgBundleInfo()
        _check(self._l.stg_bundle_load(self._h, str(path).encode(), C.byref(info)))
        return info.as_dict()

    def bundle_window(self) -> StgWindow:
        w = StgWindow()
        _check(self._l.stg_bundle_window(self._h, C.byref(w)))
        return w

    def bundle_run(self, cfg: Optional[dict] = None) -> dict:
        """build_group_data + diagnose on the loaded bundle (device-resident window)."""
        w = self.bundle_window()
        cc = config_struct(cfg)
        st = StgRunStats()
        _check(self._l.stg_window_run(self._h, C.byref(w), C.byref(cc), C.byref(st)))
        self.last_stats = st.as_dict()
        return self.last_stats

    def bundle_arrays(self) -> dict:
        """The loaded bundle's window with its device arrays copied to numpy (tests)."""
        w = self.bundle_window()

        def dev(ptr, n, dt):
            a = np.zeros(n, dt)
            if n:
                _check(self._l.stg_device_to_host(self._h, a.ctypes.data, ptr, a.nbytes))
            return a
        ns, nf, nc = w.n_samples, w.n_frames, w.n_coll
        return {
            "rank_ids": np.ctypeslib.as_array(C.cast(w.rank_ids, C.POINTER(C.c_int32)), (w.n_ranks,)).copy()
            if w.n_ranks else np.zeros(0, np.int32),
            "rank_sample_off": np.ctypeslib.as_array(C.cast(w.rank_sample_off, C.POINTER(C.c_uint64)),
                                                     (w.n_ranks + 1,)).copy(),
            "bin_build_ids": C.string_at(w.bin_build_ids, 20 * w.n_bins) if w.n_bins else b"",
            "sample_ts": dev(w.sample_ts, ns, np.int64),
            "sample_frame_off": dev(w.sample_frame_off, ns + 1 if ns else 0, np.uint64),
            "frame_pc": dev(w.frame_pc, nf, np.uint64),
            "frame_bin": dev(w.frame_bin, nf, np.uint16),
            "coll_rank": dev(w.coll_rank, nc, np.int32), "coll_group": dev(w.coll_group, nc, np.int32),
            "coll_kind": dev(w.coll_kind, nc, np.uint8), "coll_entry": dev(w.coll_entry, nc, np.int64),
            "coll_exit": dev(w.coll_exit, nc, np.int64), "coll_gpu_dur": dev(w.coll_gpu_dur, nc, np.int64),
        }

    # ------------------------------------------------------ raw aggregation
    def aggregate_samples(self, ts, frame_off, frame_pc, frame_bin, rank=None,
                          drain_interval_ns: int = 5_000_000_000, exact: bool = False):
        """aggregate_samples (samples.cpp:31-85) on the GPU for one rank's stream.

        Arrays are numpy (host) or torch CUDA tensors (device).  Returns a list of
        windows (start_ns, end_ns, first_sample[np.uint64], count[np.uint64]) —
        each record is the first-seen sample of its stack and its count."""
        keep: list = []
        dev = bool(getattr(ts, "is_cuda", False))
        st = StgStream()
        st.memory = STG_MEM_DEVICE if dev else STG_MEM_HOST
        st.n_samples = int(ts.shape[0] if dev else len(ts))
        if hasattr(ts, "data_ptr"):  # torch tensors (CUDA, or pinned host for end-to-end use)
            st.ts, st.rank = _ptr(ts, keep), _ptr(rank, keep)
            st.frame_off, st.frame_pc, st.frame_bin = (_ptr(frame_off, keep), _ptr(frame_pc, keep),
                                                       _ptr(frame_bin, keep))
        else:
            st.ts = _ptr(np.asarray(ts, np.int64), keep)
            st.rank = None if rank is None else _ptr(np.asarray(rank, np.int32), keep)
            st.frame_off = _ptr(np.asarray(frame_off, np.uint64), keep)
            st.frame_pc = _ptr(np.asarray(frame_pc, np.uint64), keep)
            st.frame_bin = _ptr(np.asarray(frame_bin, np.uint16), keep)
        nw, nr = C.c_uint64(), C.c_uint64()
        _check(self._l.stg_aggregate_samples(self._h, C.byref(st), int(drain_interval_ns),
                                             STG_AGG_FORCE_EXACT if exact else 0, C.byref(nw), C.byref(nr)))
        ws = np.zeros(nw.value, np.int64)
        we = np.zeros(nw.value, np.int64)
        ro = np.zeros(nw.value + 1, np.uint64)
        first = np.zeros(nr.value, np.uint64)
        cnt = np.zeros(nr.value, np.uint64)
        _check(self._l.stg_aggregate_windows(self._h, ws.ctypes.data, we.ctypes.data, ro.ctypes.data))
        _check(self._l.stg_aggregate_records(self._h, first.ctypes.data, cnt.ctypes.data))
        return [(int(ws[w]), int(we[w]), first[ro[w]:ro[w + 1]], cnt[ro[w]:ro[w + 1]])
                for w in range(nw.value)]

    # ---------------------------------------------------------------- window
    def window_run(self, win: Window, cfg: Optional[dict] = None, ingest: bool = True) -> dict:
        if ingest:
            for s in win.symr:
                self.ingest(s)
        cw, keep = win.to_c()
        cc = config_struct(cfg)
        st = StgRunStats()
        _check(self._l.stg_window_run(self._h, C.byref(cw), C.byref(cc), C.byref(st)))
        self.last_stats = st.as_dict()
        return self.last_stats

    def _json(self, fn) -> dict:
        need = C.c_uint64()
        _check(fn(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(fn(self._h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())

    def groupdata(self) -> dict:
        return self._json(self._l.stg_result_groupdata_json)

    def report(self) -> dict:
        return self._json(self._l.stg_result_report_json)

    def waterline(self) -> dict:
        return self._json(self._l.stg_result_waterline_json)

    def _text(self, fn, *args) -> str:
        need = C.c_uint64()
        _check(fn(self._h, *args, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(fn(self._h, *args, buf, need.value, C.byref(need)))
        return buf.raw[:need.value - 1].decode("utf-8", "surrogateescape")

    def report_json_text(self) -> str:
        """DiagnosisReport::to_json exactly as the reference writes it (nlohmann dump(2))."""
        return self._text(self._l.stg_result_report_json)

    def report_text(self) -> str:
        """DiagnosisReport::to_text (diagnosis.cpp:457-481)."""
        return self._text(self._l.stg_result_report_text)

    def folded_text(self, rank: int) -> str:
        """FoldedProfile::to_string of `rank`'s CPU profile (folded.cpp:33-43), rendered on the GPU."""
        return self._text(self._l.stg_result_folded_text, rank)

    def diff_folded(self, rank_a: int, rank_b: int) -> str:
        """diff_folded(profile(a), profile(b)) (folded.cpp:83-96), rendered on the GPU."""
        return self._text(self._l.stg_result_diff_folded, rank_a, rank_b)

    def flamegraph_svg(self, rank: int, title: str = "flame graph", width: int = 1200, row_height: int = 16,
                       min_fraction: float = 0.001) -> str:
        """render_flamegraph (svg.cpp:157-163) of `rank`'s CPU profile."""
        o = StgSvgOptions(width, row_height, min_fraction, title.encode())
        return self._text(self._l.stg_result_flamegraph_svg, rank, C.byref(o))

    def diff_flamegraph_svg(self, rank_before: int, rank_after: int, title: str = "flame graph", width: int = 1200,
                            row_height: int = 16, min_fraction: float = 0.001) -> str:
        """render_diff_flamegraph (svg.cpp:165-172) of two ranks' CPU profiles."""
        o = StgSvgOptions(width, row_height, min_fraction, title.encode())
        return self._text(self._l.stg_result_diff_flamegraph_svg, rank_before, rank_after, C.byref(o))

    def folded(self):
        """{rank: (total, [(names root-first, count), ...])} via the structured getters."""
        n = C.c_uint32()
        _check(self._l.stg_result_rank_count(self._h, C.byref(n)))
        out = {}
        for i in range(n.value):
            rank, nl, tot, nk = C.c_int32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            _check(self._l.stg_result_rank_info(self._h, i, C.byref(rank), C.byref(nl), C.byref(tot),
                                                C.byref(nk)))
            off = np.zeros(nl.value + 1, np.uint64)
            keys = np.zeros(max(nk.value, 1), np.uint32)
            cnt = np.zeros(max(nl.value, 1), np.uint64)
            _check(self._l.stg_result_rank_lines(self._h, i, off.ctypes.data, keys.ctypes.data,
                                                 cnt.ctypes.data))
            lines = []
            for l in range(nl.value):
                names = [self.name(int(k)) for k in keys[off[l]:off[l + 1]]]
                lines.append((names, int(cnt[l])))
            out[rank.value] = (tot.value, lines)
        return out
