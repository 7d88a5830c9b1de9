"""Host-side plumbing for one communication group spanning several GPUs.

One process per GPU (torchrun).  The window's CPU sample streams are sharded by
rank (contiguous blocks of the sorted rank ids); collectives, GPU events, OS
counters and the baseline stay identical on every process (include/stg.h,
"distributed").  torch.distributed only ships the 128-byte NCCL id; all
data-path exchanges happen inside libstg over its own NCCL communicator.
"""
from __future__ import annotations

import copy

import numpy as np


def shard_bounds(n_ranks: int, world: int, rank: int):
    """[lo, hi) of the rank block owned by `rank` (near-equal contiguous blocks)."""
    base, extra = divmod(n_ranks, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_window(win, world: int, rank: int):
    """Copy of a host Window keeping only this process's ranks' samples."""
    lo, hi = shard_bounds(len(win.rank_ids), world, rank)
    out = copy.copy(win)
    soff = np.asarray(win.rank_sample_off, np.uint64)
    s0, s1 = int(soff[lo]), int(soff[hi])
    foff = np.asarray(win.sample_frame_off, np.uint64)
    f0, f1 = int(foff[s0]), int(foff[s1])
    out.rank_ids = np.asarray(win.rank_ids, np.int32)[lo:hi].copy()
    out.rank_sample_off = (soff[lo:hi + 1] - soff[lo]).astype(np.uint64)
    out.sample_ts = np.asarray(win.sample_ts)[s0:s1].copy()
    out.sample_frame_off = (foff[s0:s1 + 1] - foff[s0]).astype(np.uint64)
    out.frame_pc = np.asarray(win.frame_pc)[f0:f1].copy()
    out.frame_bin = np.asarray(win.frame_bin)[f0:f1].copy()
    out.n_samples_ = None
    out.n_frames_ = None
    return out


def share_unique_id(dist, uid_fn, device=None) -> bytes:
    """World rank 0 creates the NCCL id (uid_fn), torch.distributed broadcasts it."""
    import torch
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(uid_fn()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())
