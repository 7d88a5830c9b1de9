"""Worker for tests/test_dist.py: one process per GPU (torchrun).  Every process
builds the same window, keeps its rank shard, joins the libstg NCCL group and
writes its report / groupdata / waterline as JSON."""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

import paper_2603_29235_b200 as stg
from paper_2603_29235_b200.dist import share_unique_id, shard_window


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--case", required=True)
    ap.add_argument("--shard", type=int, default=0, help="stg_window.shard_streams (1 coll, 2 side)")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from tests.dist_cases import make_case
    win = make_case(a.case)
    ctx = stg.Context(local)
    ctx.dist_init(world, rank, share_unique_id(dist, stg.Context.dist_unique_id, device="cuda"))
    try:
        ctx.window_run(shard_window(win, world, rank, streams=a.shard), cfg={"want_waterline": 1})
        out = {"report": ctx.report(), "groupdata": ctx.groupdata(), "waterline": ctx.waterline()}
    except stg.StgError as e:  # every process must fail with the same error (no hang)
        out = {"error": str(e)}
    Path(a.out, f"rank{rank}.json").write_text(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
