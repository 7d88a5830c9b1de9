"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.

A plain-Python restatement of strata's per-window analysis (the reference at
/root/reference/proj/core, C++20), written from its semantics, not translated
line by line.  Each function cites the reference file:line it follows.  It is
the checker for the CUDA library in tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg; the product never imports it.

Parity pin: tests/test_oracle.py checks this module against (a) the known
answers of the reference's own unit/acceptance tests (restated) and golden
fixtures in tests/golden/, and (b) the reference itself compiled in place as
oracle/_ref/libstrata_ref.so (oracle/Makefile) on simulator windows.

Names are handled as `bytes` so that ordering is byte-wise like std::string
(char_traits<char>::lt compares as unsigned char); tuples of bytes order like
std::vector<std::string> (element-wise, shorter prefix first).  All floating
point is IEEE double evaluated in the reference's order, so results are
bit-identical to the reference, not merely close.
"""
from __future__ import annotations

import bisect
import math
import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

EXACT_RANGE, NEAREST_LOWER = 0, 1


class StrataError(Exception):
    """strata::Error (build_id.hpp:47-54)."""


# --------------------------------------------------------------------- SYMR
def parse_symbols(b: bytes):
    """parse_symbols (symfile.cpp:117-157): strict SYMR parse.

    Returns (build_id bytes, starts list, sizes list, names list of bytes)."""
    if len(b) < 36:
        raise StrataError("symbol file truncated header")
    if b[:4] != b"SYMR":
        raise StrataError("symbol file bad magic")
    version, = struct.unpack_from("<I", b, 4)
    if version != 1:
        raise StrataError(f"unsupported symbol file version {version}")
    bid = bytes(b[8:28])
    n, strtab_off = struct.unpack_from("<II", b, 28)
    if strtab_off != 36 + n * 16 or strtab_off > len(b):
        raise StrataError("symbol file bad string-table offset")
    strtab = b[strtab_off:]
    starts, sizes, names = [], [], []
    prev = 0
    for i in range(n):
        start, size, name_off = struct.unpack_from("<QII", b, 36 + 16 * i)
        if i > 0 and start <= prev:
            raise StrataError("symbol entries not strictly sorted")
        prev = start
        if name_off + 2 > len(strtab):
            raise StrataError("symbol name offset out of range")
        ln, = struct.unpack_from("<H", strtab, name_off)
        if ln == 0 or name_off + 2 + ln > len(strtab):
            raise StrataError("symbol name out of range")
        starts.append(start)
        sizes.append(size)
        names.append(bytes(strtab[name_off + 2:name_off + 2 + ln]))
    return bid, starts, sizes, names


def pack_symbols(build_id: bytes, entries) -> bytes:
    """pack_symbols (symfile.cpp:77-115); entries = [(start, size, name)]."""
    es = sorted(entries, key=lambda e: e[0])
    for a, b2 in zip(es, es[1:]):
        if a[0] == b2[0]:
            raise StrataError("duplicate symbol start")
    strtab = bytearray()
    offs = []
    for s, z, nm in es:
        nm = nm.encode() if isinstance(nm, str) else nm
        if not nm:
            raise StrataError("empty symbol name")
        if len(nm) > 0xFFFF:
            raise StrataError("symbol name too long")
        offs.append(len(strtab))
        strtab += struct.pack("<H", len(nm)) + nm
    out = bytearray(b"SYMR" + struct.pack("<I", 1) + bytes(build_id))
    out += struct.pack("<II", len(es), 36 + 16 * len(es))
    for (s, z, nm), o in zip(es, offs):
        out += struct.pack("<QII", s, z, o)
    return bytes(out + strtab)


@dataclass
class SymbolFile:
    """SymbolFile (symfile.hpp:20-41) — sorted starts, sizes, names."""

    build_id: bytes
    starts: List[int]
    sizes: List[int]
    names: List[bytes]

    @staticmethod
    def parse(b: bytes) -> "SymbolFile":
        return SymbolFile(*parse_symbols(b))

    def lookup_index(self, offset: int, mode: int) -> Tuple[Optional[int], int]:
        """SymbolFile::lookup (symfile.cpp:54-75): greatest start <= offset by
        bisection over [lo, hi); exact-range: size 0 matches only at start.
        Returns (entry index or None, probes)."""
        lo, hi, probes = 0, len(self.starts), 0
        while lo < hi:
            mid = lo + (hi - lo) // 2
            probes += 1
            if self.starts[mid] <= offset:
                lo = mid + 1
            else:
                hi = mid
        if lo == 0:
            return None, probes
        i = lo - 1
        if mode == EXACT_RANGE:
            st, sz = self.starts[i], self.sizes[i]
            # u64 wrap of start + size, as in the reference
            inside = offset == st if sz == 0 else offset < ((st + sz) & 0xFFFFFFFFFFFFFFFF)
            if not inside:
                return None, probes
        return i, probes

    def lookup(self, offset: int, mode: int) -> Optional[bytes]:
        i, _ = self.lookup_index(offset, mode)
        return None if i is None else self.names[i]


def unknown_frame_label(build_id: bytes, offset: int) -> bytes:
    """unknown_frame_label (symfile.cpp:159-163): "[<hex id>+0x<hex off>]"."""
    return b"[" + build_id.hex().encode() + b"+0x" + format(offset, "x").encode() + b"]"


class Repo:
    """SymbolRepository::load (symrepo.cpp:90-97) over in-memory SYMR payloads."""

    def __init__(self, payloads: Sequence[bytes] = ()):
        self.files: Dict[bytes, SymbolFile] = {}
        for p in payloads:
            f = SymbolFile.parse(p)
            self.files.setdefault(f.build_id, f)

    def resolve_frame(self, bid: bytes, off: int, mode: int) -> bytes:
        """One frame of resolve_stack (symrepo.cpp:99-120)."""
        f = self.files.get(bid)
        if f is not None:
            nm = f.lookup(off, mode)
            if nm is not None:
                return nm
        return unknown_frame_label(bid, off)

    def resolve_stack(self, frames, mode: int) -> List[bytes]:
        return [self.resolve_frame(b, o, mode) for b, o in frames]


# ------------------------------------------------------------- aggregation
def aggregate_samples(stream, drain: int = 5_000_000_000):
    """aggregate_samples (samples.cpp:31-85).  stream = [(ts, rank, frames)]
    with frames = tuple of (build_id, offset) leaf first.  Returns windows as
    (start, end, [(frames, count)] in first-seen order)."""
    if drain <= 0:
        raise StrataError("drain interval must be positive")
    out = []
    if not stream:
        return out
    ts0, rank0, _ = stream[0]
    start = ts0 - ((ts0 % drain + drain) % drain)  # Python % is floor-mod: same result
    end = start + drain
    rec: Dict[tuple, int] = {}
    prev = ts0
    for ts, rank, frames in stream:
        if not frames:
            raise StrataError("empty sample stack")
        if rank != rank0:
            raise StrataError("aggregate_samples: mixed ranks")
        if ts < prev:
            raise StrataError("aggregate_samples: timestamps regressed")
        prev = ts
        if ts >= end:
            if rec:
                out.append((start, end, list(rec.items())))
            rec = {}
            k = (ts - start) // drain  # ts >= start here, so floor == truncation
            start = start + k * drain
            end = start + drain
        rec[frames] = rec.get(frames, 0) + 1  # dict keeps first-seen order
    if rec:
        out.append((start, end, list(rec.items())))
    return out


@dataclass
class Folded:
    """FoldedProfile (folded.hpp:13-28): lines sorted lexicographically."""

    lines: List[Tuple[Tuple[bytes, ...], int]] = field(default_factory=list)
    total: int = 0

    def inclusive_fractions(self) -> Dict[bytes, float]:
        """folded.cpp:45-54: each distinct name of a line gets count/total,
        summed in line order."""
        out: Dict[bytes, float] = {}
        if self.total == 0:
            return out
        for frames, count in self.lines:
            for nm in sorted(set(frames)):
                out[nm] = out.get(nm, 0.0) + count / self.total
        return out

    def to_string(self) -> str:
        """folded.cpp:33-43"""
        return "".join(";".join(f.decode() for f in fr) + f" {c}\n" for fr, c in self.lines)


def _finish(merged: Dict[tuple, int]) -> Folded:
    """folded.cpp:11-19 — std::map order, total = Σ counts."""
    f = Folded()
    for frames in sorted(merged):
        f.lines.append((frames, merged[frames]))
        f.total += merged[frames]
    return f


def to_folded(windows, repo: Repo, mode: int) -> Folded:
    """to_folded over several windows (folded.cpp:61-71 with add_window :21-29)."""
    merged: Dict[tuple, int] = {}
    cache: Dict[tuple, bytes] = {}
    for _, _, records in windows:
        for frames, count in records:
            names = []
            for fr in frames:
                nm = cache.get(fr)
                if nm is None:
                    nm = cache[fr] = repo.resolve_frame(fr[0], fr[1], mode)
                names.append(nm)
            key = tuple(reversed(names))
            merged[key] = merged.get(key, 0) + count
    if not merged:
        raise StrataError("empty profile window")
    return _finish(merged)


def fold_symbolized(stacks) -> Folded:
    """fold_symbolized (folded.cpp:73-81): leaf-first input."""
    merged: Dict[tuple, int] = {}
    for frames, count in stacks:
        key = tuple(reversed([f if isinstance(f, bytes) else f.encode() for f in frames]))
        merged[key] = merged.get(key, 0) + count
    return _finish(merged)


def diff_folded(a: Folded, b: Folded) -> str:
    """diff_folded (folded.cpp:83-96)."""
    m: Dict[tuple, List[int]] = {}
    for fr, c in a.lines:
        m.setdefault(fr, [0, 0])[0] += c
    for fr, c in b.lines:
        m.setdefault(fr, [0, 0])[1] += c
    return "".join(";".join(f.decode() for f in fr) + f" {m[fr][0]} {m[fr][1]}\n" for fr in sorted(m))


# ------------------------------------------------------------- collectives
@dataclass
class Instance:
    group: int
    kind: int
    events: Dict[int, Tuple[int, int]]  # rank -> (entry, exit)
    partial: bool = False


def match_collectives(events, group_ranks, max_skew: int = 50_000_000) -> List[Instance]:
    """match_collectives (collective.cpp:29-103).  events = [(rank, group, kind,
    entry, exit)] in input order."""
    streams: Dict[Tuple[int, int], Dict[int, List[Tuple[int, int]]]] = {}
    for rank, group, kind, en, ex in events:
        if en >= ex:
            raise StrataError("collective event with entry >= exit")
        q = streams.setdefault((group, kind), {}).setdefault(rank, [])
        if q and en < q[-1][0]:
            raise StrataError("collective events not time-ordered within rank")
        q.append((en, ex))
    out: List[Instance] = []
    for gk in sorted(streams):
        per = streams[gk]
        ranks = sorted(per)
        mn = min(per[r][0][0] for r in ranks)
        coarse = {r: per[r][0][0] - mn for r in ranks}
        head = {r: 0 for r in ranks}
        while True:
            seed = None
            for r in ranks:  # min pre-aligned entry, ties -> lowest rank (strict <)
                if head[r] < len(per[r]):
                    e = per[r][head[r]][0] - coarse[r]
                    if seed is None or e < seed[0]:
                        seed = (e, per[r][head[r]][1] - coarse[r])
            if seed is None:
                break
            inst = Instance(gk[0], gk[1], {})
            for r in ranks:
                if head[r] < len(per[r]):
                    en, ex = per[r][head[r]]
                    if en - coarse[r] <= seed[1] + max_skew and ex - coarse[r] + max_skew >= seed[0]:
                        inst.events[r] = (en, ex)
                        head[r] += 1
            inst.partial = any(r not in inst.events for r in group_ranks)
            out.append(inst)
    # (min raw entry, group, kind) — collective.cpp:92-101 (std::sort, ties unspecified)
    out.sort(key=lambda x: (min(e for e, _ in x.events.values()), x.group, x.kind))
    return out


def _div_trunc(a: int, b: int) -> int:
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def align_clocks(instances) -> Optional[Dict[int, int]]:
    """align_clocks (collective.cpp:105-125): per-rank median of exit - max exit
    over complete instances; even count -> int64 truncating mean."""
    deltas: Dict[int, List[int]] = {}
    for inst in instances:
        if inst.partial:
            continue
        mx = max(ex for _, ex in inst.events.values())
        for r, (_, ex) in inst.events.items():
            deltas.setdefault(r, []).append(ex - mx)
    if not deltas:
        return None
    out = {}
    for r in sorted(deltas):
        v = sorted(deltas[r])
        n = len(v)
        out[r] = v[n // 2] if n % 2 else _div_trunc(v[n // 2 - 1] + v[n // 2], 2)
    return out


def entry_lateness(inst: Instance, offsets: Dict[int, int]) -> Dict[int, float]:
    """entry_lateness (collective.cpp:127-142)."""
    if inst.partial:
        raise StrataError("lateness requires a complete instance")
    adj = {r: en - offsets.get(r, 0) for r, (en, _) in inst.events.items()}
    mn = min(adj.values())
    return {r: (adj[r] - mn) / 1e6 for r in sorted(adj)}


# ---------------------------------------------------------------- diagnosis
def _mean(v):  # std::accumulate from 0.0 then / n (diagnosis.cpp:20-22)
    s = 0.0
    for x in v:
        s += x
    return s / len(v)


def _pstd(v, mu):  # diagnosis.cpp:14-18
    a = 0.0
    for x in v:
        a += (x - mu) * (x - mu)
    return math.sqrt(a / len(v))


def _median(v):  # diagnosis.cpp:24-28
    v = sorted(v)
    n = len(v)
    return v[n // 2] if n % 2 else (v[n // 2 - 1] + v[n // 2]) / 2.0


def compute_waterline(per_rank: Dict[int, Folded], k: float = 2.0):
    """compute_waterline (diagnosis.cpp:35-55) -> {name: (mean, stddev)}."""
    if len(per_rank) < 2:
        raise StrataError("waterline requires at least 2 ranks")
    fr: Dict[bytes, List[float]] = {}
    for r in sorted(per_rank):
        for nm, v in sorted(per_rank[r].inclusive_fractions().items()):
            fr.setdefault(nm, []).append(v)
    out = {}
    for nm in sorted(fr):
        v = fr[nm] + [0.0] * (len(per_rank) - len(fr[nm]))
        mu = _mean(v)
        out[nm] = (mu, _pstd(v, mu))
    return out


def flag_ranks(wl, per_rank: Dict[int, Folded], k: float = 2.0):
    """flag_ranks (diagnosis.cpp:57-71)."""
    out = []
    for r in sorted(per_rank):
        for nm, v in sorted(per_rank[r].inclusive_fractions().items()):
            if nm not in wl:
                continue
            thr = wl[nm][0] + k * wl[nm][1]
            if v > thr:
                out.append((r, nm, v, thr))
    return out


@dataclass
class Alert:
    rank: int
    mean_lateness_ms: float
    z_score: float
    flagged_instances: int
    window_instances: int


def detect_straggler(lat_per_instance: List[Dict[int, float]], k: float = 2.0) -> List[Alert]:
    """detect_straggler (diagnosis.cpp:76-111)."""
    flags: Dict[int, int] = {}
    lat: Dict[int, List[float]] = {}
    zs: Dict[int, List[float]] = {}
    for inst in lat_per_instance:
        if len(inst) < 2:
            continue
        v = [inst[r] for r in sorted(inst)]
        mu = _mean(v)
        sg = _pstd(v, mu)
        for r in sorted(inst):
            l = inst[r]
            lat.setdefault(r, []).append(l)
            if sg > 0.0 and l > mu + k * sg:
                flags[r] = flags.get(r, 0) + 1
                zs.setdefault(r, []).append((l - mu) / sg)
    n = len(lat_per_instance)
    return [Alert(r, _mean(lat[r]), _mean(zs[r]), c, n) for r, c in sorted(flags.items()) if c * 2 > n]


def median_lateness_rank(lat_per_instance, exclude) -> Optional[int]:
    """median_lateness_rank (diagnosis.cpp:284-297)."""
    lat: Dict[int, List[float]] = {}
    for inst in lat_per_instance:
        for r in sorted(inst):
            lat.setdefault(r, []).append(inst[r])
    means = sorted((_mean(v), r) for r, v in lat.items() if r not in exclude)
    return means[len(means) // 2][1] if means else None


def gpu_diff(s: Dict[str, int], ref: Dict[str, int], cfg: dict):
    """gpu_diff (diagnosis.cpp:122-172) -> (verdict 0/1/2, slowdown dict, top)."""
    slowdown, slows, total_added, top = {}, [], 0, ""
    for name in sorted(ref):
        t_ref = ref[name]
        if t_ref < cfg["gpu_ref_floor_ns"]:
            continue
        if cfg["gpu_exclude_prefix"] and name.startswith(cfg["gpu_exclude_prefix"]):
            continue
        if name not in s:
            continue
        x = s[name] / t_ref - 1.0
        slowdown[name] = x
        slows.append(x)
        added = s[name] - t_ref
        if added > 0:
            total_added += added
            if not top or added > s[top] - ref[top]:
                top = name
    if not slows:
        return 0, slowdown, top
    med = _median(slows)
    mu = _mean(slows)
    sg = _pstd(slows, mu)
    cv = abs(sg / mu) if mu != 0.0 else 0.0
    share = (s[top] - ref[top]) / total_added if top and total_added > 0 else 0.0
    if med <= cfg["gpu_median_none"]:
        return 0, slowdown, top
    if med > cfg["gpu_median_uniform"] and cv < cfg["gpu_cv_uniform"]:
        return 1, slowdown, top
    if share > cfg["gpu_top_share_specific"]:
        return 2, slowdown, top
    return 0, slowdown, top


def _hottest(prof: Folded, fn: bytes):
    best = None
    for fr, c in prof.lines:
        if fn in fr and (best is None or c > best[1]):
            best = (fr, c)
    return list(best[0]) if best else []


def cpu_diff(s: Folded, r: Folded, delta: float = 0.005):
    """cpu_diff (diagnosis.cpp:177-208) -> [(fn, fs, fr, d, hottest path)]."""
    fs_, fr_ = s.inclusive_fractions(), r.inclusive_fractions()
    out = []
    for fn in sorted(fs_):
        fs = fs_[fn]
        fr = fr_.get(fn, 0.0)
        d = fs - fr
        if d > delta:
            out.append((fn, fs, fr, d, _hottest(s, fn)))
    out.sort(key=lambda t: (-t[3], t[0]))
    return out


def os_diff(s: dict, r: dict, cfg: dict):
    """os_diff (diagnosis.cpp:213-243); snapshot dicts have interrupts,
    softirqs (name->count), p99, migrations."""
    out = []

    def check(name, sv, rv, floor):
        if sv - rv < floor:
            return
        if rv == 0:
            out.append((name, sv, rv, 0.0, True))
            return
        ratio = sv / rv
        if ratio >= cfg["os_min_ratio"]:
            out.append((name, sv, rv, ratio, False))

    for k in sorted(s["interrupts"]):
        check("interrupt:" + k, s["interrupts"][k], r["interrupts"].get(k, 0), cfg["os_interrupt_floor"])
    for k in sorted(s["softirqs"]):
        check("softirq:" + k, s["softirqs"][k], r["softirqs"].get(k, 0), cfg["os_interrupt_floor"])
    check("sched_delay_p99_ns", s["p99"], r["p99"], cfg["os_sched_delay_floor_ns"])
    check("numa_migrations", s["migrations"], r["migrations"], cfg["os_migration_floor"])
    return out


def temporal_diff(cur: Folded, baseline: Dict[bytes, float], delta: float):
    """temporal_diff (diagnosis.cpp:248-263)."""
    out = []
    for fn, now in sorted(cur.inclusive_fractions().items()):
        base = baseline.get(fn, 0.0)
        d = now - base
        if d > delta:
            out.append((fn, now, base, d))
    out.sort(key=lambda t: (-t[3], t[0]))
    return out


def diagnose(gd: dict, cfg: Optional[dict] = None) -> dict:
    """diagnose (diagnosis.cpp:301-432) over the oracle's GroupData dict;
    returns the DiagnosisReport::to_json layout (diagnosis.cpp:437-455)."""
    from paper_2603_29235_b200.abi import VERDICTS, default_config
    cfg = dict(default_config(), **(cfg or {}))
    rep = {"verdict": "healthy", "flagged_ranks": [], "evidence": [], "top_path": [], "notes": [],
           "reference_rank": None}
    lpi = gd["lateness_per_instance"]
    alerts = detect_straggler(lpi, cfg["k"])
    dec = lambda b: b.decode()
    if alerts:
        rep["flagged_ranks"] = sorted(a.rank for a in alerts)
        ref = median_lateness_rank(lpi, rep["flagged_ranks"])
        rep["reference_rank"] = ref
        if ref is None:
            rep["verdict"] = "inconclusive"
            rep["notes"].append("no reference rank available")
            return rep
        st = rep["flagged_ranks"][0]
        concluded = "inconclusive"
        gpu_ev, cpu_ev, os_ev = [], [], []
        gp = gd["gpu_profiles"]
        if st in gp and ref in gp:
            v, slow, top = gpu_diff(gp[st], gp[ref], cfg)
            for name in sorted(slow):
                gpu_ev.append({"layer": "gpu", "item": name, "straggler_value": float(gp[st][name]),
                               "reference_value": float(gp[ref][name]), "delta": slow[name]})
            if v == 1:
                concluded = "gpu-uniform-slowdown"
            elif v == 2:
                concluded = "gpu-specific-kernel"
                rep["top_path"] = [top]
        else:
            rep["notes"].append("gpu profiles missing; gpu layer skipped")
        cp = gd["cpu_profiles"]
        if st in cp and ref in cp:
            cd = cpu_diff(cp[st], cp[ref], cfg["delta"])
            for fn, fs, fr, d, _ in cd:
                cpu_ev.append({"layer": "cpu", "item": dec(fn), "straggler_value": fs,
                               "reference_value": fr, "delta": d})
            if concluded == "inconclusive" and cd:
                concluded = "cpu-interference"
                rep["top_path"] = [dec(x) for x in cd[0][4]]
        else:
            rep["notes"].append("cpu profiles missing; cpu layer skipped")
        osn = gd["os_snapshots"]
        if st in osn and ref in osn:
            od = os_diff(osn[st], osn[ref], cfg)
            for name, sv, rv, ratio, unb in od:
                os_ev.append({"layer": "os", "item": name, "straggler_value": float(sv),
                              "reference_value": float(rv), "delta": 0.0 if unb else ratio})
            if concluded == "inconclusive" and od:
                concluded = "os-interference"
        else:
            rep["notes"].append("os snapshots missing; os layer skipped")
        rep["verdict"] = concluded
        rep["evidence"] = gpu_ev + cpu_ev + os_ev
        if concluded == "inconclusive":
            rep["notes"].append("straggler detected but no layer concluded")
        return rep
    it = gd["iteration_times_ms"]
    if gd.get("baseline_iteration_ms") is not None and it:
        now = _mean(it)
        base = gd["baseline_iteration_ms"]
        if base > 0.0 and now > base * (1.0 + cfg["iteration_regression_gate"]):
            if gd.get("baseline") is None:
                rep["verdict"] = "inconclusive"
                rep["notes"].append("iteration time regressed but no baseline profile")
                return rep
            allst = []
            for r in sorted(gd["cpu_profiles"]):
                for fr, c in gd["cpu_profiles"][r].lines:
                    allst.append((list(reversed(fr)), c))
            merged = fold_symbolized(allst)
            bl = {k.encode() if isinstance(k, str) else k: v for k, v in gd["baseline"]["fractions"].items()}
            cands = temporal_diff(merged, bl, gd["baseline"]["delta"])
            if cands:
                rep["verdict"] = "temporal-degradation"
                rep["flagged_ranks"] = sorted(gd["cpu_profiles"])
                for fn, nw, b, d in cands:
                    rep["evidence"].append({"layer": "temporal", "item": dec(fn), "straggler_value": nw,
                                            "reference_value": b, "delta": d})
                rep["top_path"] = [dec(x) for x in _hottest(merged, cands[0][0])]
                return rep
            rep["verdict"] = "inconclusive"
            rep["notes"].append("iteration time regressed but no profile delta above delta")
            return rep
    rep["verdict"] = "healthy"
    return rep


# ----------------------------------------------------------- window batch
def build_group_data(win, mode: int = EXACT_RANGE) -> dict:
    """build_group_data (bundle.cpp:252-324) over an abi.Window (SoA)."""
    import numpy as np
    gd: dict = {"group": win.group}
    bids = [bytes(np.asarray(win.bin_build_ids, np.uint8).reshape(-1, 20)[i])
            for i in range(len(win.bin_build_ids))]
    ev = list(zip(win.coll_rank.tolist(), win.coll_group.tolist(), win.coll_kind.tolist(),
                  win.coll_entry.tolist(), win.coll_exit.tolist()))
    inst = match_collectives(ev, win.group_ranks.tolist(), win.max_skew_ns)
    off = align_clocks(inst) or {}
    oo = lambda r: off.get(r, 0)
    windowed = []
    for i in inst:
        if i.partial:
            continue
        mx = 0  # bundle.cpp:274 initialises the max to 0
        for r, (_, ex) in i.events.items():
            mx = max(mx, ex - oo(r))
        if mx >= win.window_start_ns:
            windowed.append((mx, i))
    windowed.sort(key=lambda t: t[0])
    gd["lateness_per_instance"] = [entry_lateness(i, off) for _, i in windowed]
    gd["iteration_times_ms"] = [(windowed[k][0] - windowed[k - 1][0]) / 1e6 for k in range(1, len(windowed))]
    repo = Repo(win.symr)
    cpu = {}
    drain = win.window_end_ns - win.window_start_ns + 2 * win.max_skew_ns
    ts = np.asarray(win.sample_ts)
    foff = np.asarray(win.sample_frame_off)
    pcs = np.asarray(win.frame_pc).tolist()
    bins = np.asarray(win.frame_bin).tolist()
    for ri, rank in enumerate(win.rank_ids.tolist()):
        a, b = int(win.rank_sample_off[ri]), int(win.rank_sample_off[ri + 1])
        stream = []
        for s in range(a, b):
            t = int(ts[s])
            if t - oo(rank) < win.window_start_ns:
                continue
            f0, f1 = int(foff[s]), int(foff[s + 1])
            frames = tuple((bids[bins[j]], pcs[j]) for j in range(f0, f1))
            stream.append((t, rank, frames))
        if not stream:
            continue
        cpu[rank] = to_folded(aggregate_samples(stream, drain), repo, mode)
    gd["cpu_profiles"] = cpu
    gp: Dict[int, Dict[str, int]] = {}
    for r, k, st, du in zip(win.gpu_rank.tolist(), win.gpu_kernel.tolist(), win.gpu_start.tolist(),
                            win.gpu_dur.tolist()):
        if st - oo(r) < win.window_start_ns:
            continue
        d = gp.setdefault(r, {})
        name = win.kernel_names[k]
        d[name] = d.get(name, 0) + du
    gd["gpu_profiles"] = gp
    osn: Dict[int, dict] = {}
    for i, r in enumerate(win.os_rank.tolist()):
        if int(win.os_window_start[i]) - oo(r) + 5_000_000_000 < win.window_start_ns:
            continue
        a = osn.setdefault(r, {"interrupts": {}, "softirqs": {}, "p50": 0, "p99": 0, "migrations": 0})
        for k in range(int(win.os_irq_off[i]), int(win.os_irq_off[i + 1])):
            nm = win.counter_names[int(win.os_irq_key[k])]
            a["interrupts"][nm] = a["interrupts"].get(nm, 0) + int(win.os_irq_val[k])
        for k in range(int(win.os_sirq_off[i]), int(win.os_sirq_off[i + 1])):
            nm = win.counter_names[int(win.os_sirq_key[k])]
            a["softirqs"][nm] = a["softirqs"].get(nm, 0) + int(win.os_sirq_val[k])
        a["p50"] = max(a["p50"], int(win.os_p50[i]))
        a["p99"] = max(a["p99"], int(win.os_p99[i]))
        a["migrations"] += int(win.os_migrations[i])
    gd["os_snapshots"] = osn
    # LoadedBundle always carries a baseline (bundle.hpp:37-38); build_group_data
    # copies it (bundle.cpp:257-258), empty / 0.0 when the bundle had none
    gd["baseline"] = {"delta": win.baseline_delta if win.has_baseline else 0.005, "fractions": dict(win.baseline)}
    gd["baseline_iteration_ms"] = win.baseline_iteration_ms if win.baseline_iteration_ms is not None else 0.0
    return gd


def groupdata_to_json(gd: dict) -> dict:
    """Canonical JSON layout shared with ref_harness.cpp and libstg."""
    return {
        "group": gd["group"],
        "cpu_profiles": [{"rank": r, "total": p.total,
                          "lines": [[[x.decode() for x in fr], c] for fr, c in p.lines]}
                         for r, p in sorted(gd["cpu_profiles"].items())],
        "gpu_profiles": [{"rank": r, "kernels": [[k, v] for k, v in sorted(m.items())]}
                         for r, m in sorted(gd["gpu_profiles"].items())],
        "os_snapshots": [{"rank": r, "interrupts": sorted([k, v] for k, v in a["interrupts"].items()),
                          "softirqs": sorted([k, v] for k, v in a["softirqs"].items()),
                          "p50": a["p50"], "p99": a["p99"], "migrations": a["migrations"]}
                         for r, a in sorted(gd["os_snapshots"].items())],
        "lateness_per_instance": [[[r, l] for r, l in sorted(i.items())] for i in gd["lateness_per_instance"]],
        "iteration_times_ms": gd["iteration_times_ms"],
        "baseline": None if gd["baseline"] is None else {
            "delta": gd["baseline"]["delta"],
            "fractions": sorted([k, v] for k, v in gd["baseline"]["fractions"].items())},
        "baseline_iteration_ms": gd["baseline_iteration_ms"],
    }


def window_pipeline(win, cfg: Optional[dict] = None):
    """build_group_data + diagnose -> (groupdata json, report)."""
    gd = build_group_data(win)
    return groupdata_to_json(gd), diagnose(gd, cfg)
