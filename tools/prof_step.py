import sys, time
from pathlib import Path
sys.argv = ["bench.py", "--ranks", "128", "--no-e2e", "--no-cpu-baseline"]
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench, torch, ctypes as C
import paper_2603_29235_b200 as stg
from paper_2603_29235_b200.abi import STG_MEM_DEVICE, config_struct, StgRunStats
a = bench.args_parse()
wl = bench.Workload(a, 0)
ctx = stg.Context(0)
for _, _, _, symr in wl.tables: ctx.ingest(symr)
arrays = wl.generate(torch, a.ranks, a.spr)
win = wl.window(a.ranks, a.spr, arrays, STG_MEM_DEVICE)
for it in range(4):
    t0 = time.perf_counter(); cw, keep = win.to_c(); t1 = time.perf_counter()
    cc = config_struct({"want_waterline": 1}); st = StgRunStats()
    rc = ctx._l.stg_window_run(ctx._h, C.byref(cw), C.byref(cc), C.byref(st)); t2 = time.perf_counter()
    print(f"to_c {1e3*(t1-t0):.2f} ms  call {1e3*(t2-t1):.2f} ms  lib total {st.ms_total:.2f}", flush=True)
