"""Regenerates tests/golden/*.json from the reference itself.

Runs in this container only (needs oracle/_ref/libstrata_ref.so built from
/root/reference by oracle/Makefile).  Each fixture holds a small analysis window
(structure-of-arrays, include/stg.h layout) and the reference's outputs for it:
strata::build_group_data + strata::diagnose, rendered as canonical JSON.

    python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests.synth import small_window  # noqa: E402

ARRAYS = ["rank_ids", "rank_sample_off", "bin_build_ids", "sample_ts", "sample_frame_off", "frame_pc", "frame_bin",
          "coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur", "group_ranks",
          "gpu_rank", "gpu_kernel", "gpu_start", "gpu_dur", "os_rank", "os_window_start", "os_p50", "os_p99",
          "os_migrations", "os_irq_off", "os_irq_key", "os_irq_val", "os_sirq_off", "os_sirq_key", "os_sirq_val"]
SCALARS = ["kernel_names", "counter_names", "baseline", "baseline_iteration_ms", "has_baseline", "baseline_delta",
           "window_start_ns", "window_end_ns", "max_skew_ns", "group"]


def dump(name, win):
    res, _, _ = ref.window_run(win)
    d = {"source": "strata build_group_data + diagnose (oracle/_ref, compiled from /root/reference)",
         "window": {}, "expected": res}
    for k in ARRAYS:
        a = np.asarray(getattr(win, k))
        d["window"][k] = [str(a.dtype), a.reshape(-1).tolist()]
    for k in SCALARS:
        d["window"][k] = getattr(win, k)
    d["window"]["symr"] = [s.hex() for s in win.symr]
    out = Path(__file__).resolve().parent / f"{name}.json"
    out.write_text(json.dumps(d, separators=(",", ":")))
    print(out.name, out.stat().st_size, res["report"]["verdict"])


if __name__ == "__main__":
    for sc, seed in (("softirq", 1), ("thermal", 2), ("logging", 3), ("dentry-lock", 4), ("healthy", 5)):
        dump(f"sim_{sc}_{seed}", ref.simulate(sc, seed, ranks=8, iterations=40, sample_rate_hz=150.0,
                                              analysis_window=20))
    dump("synth_unknowns", small_window(seed=21, ranks=6, samples_per_rank=120, slow_rank=2, unknown_frac=0.15,
                                        extra_bins=2, n_sym=400, pool=40, iterations=30))
