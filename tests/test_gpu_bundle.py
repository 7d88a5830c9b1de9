"""Bundle ingest on the GPU: stg_bundle_load decodes a
write_bundle directory (bundle.cpp:83-164) — samples.jsonl and collectives.jsonl
on the GPU — and the analysis of that device-resident window must equal the
reference's own load_bundle -> build_group_data -> diagnose (oracle/_ref) on the
same directory: GroupData and report bit-exact.  Decoded arrays are compared
with the reference's in-memory result, and malformed files must fail with the
reference's messages where it has its own (build ids, collective kinds, missing
files, nlohmann for the host-parsed files)."""
import json
import os
import shutil

import numpy as np
import pytest

import paper_2603_29235_b200 as stg
from oracle import ref
from tests.compare import assert_close

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _bundle(tmp_path, scenario, seed, **kw):
    d = tmp_path / f"{scenario}-{seed}"
    ref.write_bundle(scenario, seed, str(d), **kw)
    return d


def _check(ctx, d):
    info = ctx.load_bundle(d)
    ctx.bundle_run()
    gd, rep = ctx.groupdata(), ctx.report()
    r, _, _, _ = ref.bundle_run(d)
    assert gd["cpu_profiles"] == r["groupdata"]["cpu_profiles"]
    assert gd["lateness_per_instance"] == r["groupdata"]["lateness_per_instance"]
    assert_close(gd, r["groupdata"], 0.0)
    assert rep == r["report"]
    return info


@pytest.mark.parametrize("scenario", ["healthy", "thermal", "softirq", "dentry-lock", "logging", "io-bottleneck"])
def test_bundle_analysis_matches_reference(ctx, tmp_path, scenario):
    info = _check(ctx, _bundle(tmp_path, scenario, 2))
    assert info["n_samples"] > 0 and info["n_coll"] > 0 and info["n_tables_ingested"] >= 0


def test_decoded_arrays_match_simulation(ctx, tmp_path):
    d = _bundle(tmp_path, "softirq", 5)
    win = ref.simulate("softirq", 5)
    ctx.load_bundle(d)
    a = ctx.bundle_arrays()
    assert np.array_equal(a["rank_ids"], np.asarray(win.rank_ids, np.int32))
    assert np.array_equal(a["rank_sample_off"], np.asarray(win.rank_sample_off, np.uint64))
    assert np.array_equal(a["sample_ts"], np.asarray(win.sample_ts, np.int64))
    assert np.array_equal(a["sample_frame_off"], np.asarray(win.sample_frame_off, np.uint64))
    assert np.array_equal(a["frame_pc"], np.asarray(win.frame_pc, np.uint64))
    ids_g = [a["bin_build_ids"][20 * b:20 * b + 20] for b in a["frame_bin"]]
    wid = np.asarray(win.bin_build_ids, np.uint8).reshape(-1, 20)
    ids_r = [bytes(wid[b]) for b in np.asarray(win.frame_bin)]
    assert ids_g == ids_r
    for k, v in (("coll_rank", win.coll_rank), ("coll_group", win.coll_group), ("coll_kind", win.coll_kind),
                 ("coll_entry", win.coll_entry), ("coll_exit", win.coll_exit), ("coll_gpu_dur", win.coll_gpu_dur)):
        assert np.array_equal(a[k], np.asarray(v).astype(a[k].dtype)), k


def test_bundle_1024_ranks(ctx, tmp_path):
    info = _check(ctx, _bundle(tmp_path, "softirq", 5, ranks=1024, iterations=120))
    assert info["n_ranks"] == 1024


def _rewrite(path, fn):
    lines = open(path, "rb").read().split(b"\n")
    open(path, "wb").write(b"\n".join(fn(lines)))


def _ref_err(d):
    with pytest.raises(ref.RefError) as e:
        ref.bundle_run(d)
    return str(e.value)


def _stg_err(ctx, d):
    with pytest.raises(stg.StgError) as e:
        ctx.load_bundle(d)
    return str(e.value)


@pytest.mark.parametrize("case,same", [("hex_len", True), ("hex_char", True), ("kind", True), ("missing_file", True),
                                       ("meta_json", True), ("gpu_json", True), ("sample_json", False),
                                       ("sample_key", False)])
def test_bundle_errors(ctx, tmp_path, case, same):
    d = _bundle(tmp_path, "healthy", 1)
    s = d / "samples.jsonl"
    if case == "hex_len":
        _rewrite(s, lambda L: L[:50] + [L[50].replace(b'[["', b'[["ab', 1)] + L[51:])
    elif case == "hex_char":
        raw = open(s, "rb").read().split(b"\n")
        i = raw[70].index(b'[["') + 3
        raw[70] = raw[70][:i] + b"z" + raw[70][i + 1:]  # still 40 chars
        open(s, "wb").write(b"\n".join(raw))
    elif case == "kind":
        _rewrite(d / "collectives.jsonl", lambda L: L[:9] + [L[9].replace(b"AllReduce", b"AllToAll")] + L[10:])
    elif case == "missing_file":
        os.remove(d / "os_counters.jsonl")
    elif case == "meta_json":
        open(d / "meta.json", "w").write("{\"scenario\": ")
    elif case == "gpu_json":
        _rewrite(d / "gpu_events.jsonl", lambda L: L[:3] + [L[3][:-5]] + L[4:])
    elif case == "sample_json":
        _rewrite(s, lambda L: L[:20] + [L[20][:-3]] + L[21:])
    elif case == "sample_key":
        _rewrite(s, lambda L: L[:20] + [L[20].replace(b'"ts"', b'"tz"')] + L[21:])
    r = _ref_err(d)
    g = _stg_err(ctx, d)
    if same:
        assert g == r
    else:
        assert g.startswith("samples.jsonl line 21: "), g


def test_bundle_whitespace_crlf_and_key_order(ctx, tmp_path):
    """Valid JSON the writer does not produce: reordered keys, spaces, CRLF line
    ends and blank lines decode to the same analysis."""
    d = _bundle(tmp_path, "dentry-lock", 3)
    r0, _, _, _ = ref.bundle_run(d)
    for name in ("samples.jsonl", "collectives.jsonl"):
        out = []
        for line in open(d / name).read().split("\n"):
            if not line:
                continue
            j = json.loads(line)
            items = list(j.items())[::-1]
            out.append("{ " + " , ".join(f'{json.dumps(k)} : {json.dumps(v)}' for k, v in items) + " }\r")
            out.append("")
        open(d / name, "w").write("\n".join(out) + "\n")
    ctx.load_bundle(d)
    ctx.bundle_run()
    assert ctx.report() == r0["report"]
    assert ctx.groupdata()["cpu_profiles"] == r0["groupdata"]["cpu_profiles"]
