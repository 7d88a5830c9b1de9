"""The drop-in proof: the reference's own acceptance gate (proj/tests/acceptance.cpp,
compiled unchanged) relinked so that strata::build_group_data / resolve_stacks /
aggregate_samples / diagnose come from libstg's C++ shim
(paper_2603_29235_b200/csrc/shim/strata_stg.cpp) on the GPU — diagnose returns
the report the GPU computed in the same window run.  Every criterion that exercises the path (c1 scenario classification
over 60 simulator bundles, c7 symbolization round trip and misattribution, c9
clock alignment, c11 temporal threshold) must still PASS.
Built by oracle/Makefile `dropin` (needs /root/reference at build time only).
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
STG = ROOT / "oracle" / "_ref" / "acceptance_stg"


@pytest.mark.gpu
@pytest.mark.skipif(not STG.exists(), reason="oracle/_ref/acceptance_stg not built (make -C oracle dropin)")
def test_reference_acceptance_gate_relinked_on_gpu():
    r = subprocess.run([str(STG)], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = [l for l in r.stdout.splitlines() if "criterion" in l]
    assert len(lines) == 11, r.stdout + r.stderr
    assert all(l.startswith("PASS") for l in lines), r.stdout
    assert r.returncode == 0


DS = ROOT / "oracle" / "_ref" / "dropin_samples"


@pytest.mark.gpu
@pytest.mark.skipif(not DS.exists(), reason="oracle/_ref/dropin_samples not built (make -C oracle dropin)")
def test_aggregate_samples_relinked_on_gpu():
    """strata::aggregate_samples from the shim (GPU) equals the reference's own
    (samples.cpp compiled in place, renamed) on the BM_Aggregation stream of
    benchmarks/bench.cpp:79-100 and on random streams; errors carry the same text."""
    r = subprocess.run([str(DS)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout + r.stderr


SHIM = ROOT / "paper_2603_29235_b200" / "libstg_strata.so"


@pytest.mark.skipif(not (STG.exists() and SHIM.exists()), reason="drop-in not built")
def test_relinked_gate_takes_the_hot_path_from_the_shim():
    """The relinked binary imports the replaced strata:: functions, and the shim
    defines them (the reference objects in the link are compiled renamed)."""
    def syms(args, path):
        out = subprocess.run(["nm", "-D", *args, str(path)], capture_output=True, text=True).stdout
        return subprocess.run(["c++filt"], input=out, capture_output=True, text=True).stdout
    need = ["strata::build_group_data(", "strata::diagnose(", "strata::resolve_stacks", "strata::aggregate_samples("]
    imported = syms(["--undefined-only"], STG)
    defined = syms(["--defined-only"], SHIM)
    for n in need:
        assert n in imported, n
        assert n in defined, n
