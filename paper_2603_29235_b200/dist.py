"""Host-side plumbing for one communication group spanning several GPUs.

One process per GPU (torchrun).  The window's CPU sample streams are sharded by
rank (contiguous blocks of the sorted rank ids).  Collectives and GPU / OS side
streams are either passed identically to every process, or sharded by the same
rank intervals (stg_window.shard_streams, include/stg.h): process p then owns
the ranks [shard_rank_lo(p), shard_rank_lo(p+1)).  The baseline is always
replicated.  torch.distributed only ships the 128-byte NCCL id; all data-path
exchanges happen inside libstg over its own NCCL communicator.
"""
from __future__ import annotations

import copy

import numpy as np


def shard_bounds(n_ranks: int, world: int, rank: int):
    """[lo, hi) of the rank block owned by `rank` (near-equal contiguous blocks)."""
    base, extra = divmod(n_ranks, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_rank_lo(rank_ids, world: int, rank: int) -> int:
    """First rank id owned by process `rank`: the first id of its block of the
    sorted CPU ranks (0 for process 0; past the last id for empty blocks), so
    the lower bounds increase with the process index."""
    ids = np.asarray(rank_ids, np.int64)
    if rank == 0:
        return 0
    lo, _ = shard_bounds(len(ids), world, rank)
    if lo < len(ids):
        return int(ids[lo])
    return int(ids[-1] if len(ids) else 0) + rank


def _keep(a, mask):
    return np.asarray(a)[mask].copy()


def _csr_keep(off, keys, vals, mask):
    off = np.asarray(off, np.uint64).astype(np.int64)
    lens = np.diff(off)[mask]
    new_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.arange(new_off[-1]) - np.repeat(new_off[:-1], lens) + np.repeat(off[:-1][mask], lens)
    return new_off.astype(np.uint64), np.asarray(keys)[idx].copy(), np.asarray(vals)[idx].copy()


def keep_streams(w, lo, hi, streams: int):
    """In place: keep only the collective events (streams & 1) and GPU / OS
    records (streams & 2) of ranks in [lo, hi) (None = unbounded)."""
    def own(r):
        r = np.asarray(r, np.int64)
        m = np.ones(len(r), bool)
        if lo is not None:
            m &= r >= lo
        if hi is not None:
            m &= r < hi
        return m
    w.shard_streams = int(streams)
    if streams & 1:
        m = own(w.coll_rank)
        for f in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur"):
            setattr(w, f, _keep(getattr(w, f), m))
    if streams & 2:
        m = own(w.gpu_rank)
        for f in ("gpu_rank", "gpu_kernel", "gpu_start", "gpu_dur"):
            setattr(w, f, _keep(getattr(w, f), m))
        m = own(w.os_rank)
        w.os_irq_off, w.os_irq_key, w.os_irq_val = _csr_keep(w.os_irq_off, w.os_irq_key, w.os_irq_val, m)
        w.os_sirq_off, w.os_sirq_key, w.os_sirq_val = _csr_keep(w.os_sirq_off, w.os_sirq_key, w.os_sirq_val, m)
        for f in ("os_rank", "os_window_start", "os_p50", "os_p99", "os_migrations"):
            setattr(w, f, _keep(getattr(w, f), m))


def shard_window(win, world: int, rank: int, streams: int = 0):
    """Copy of a host Window keeping only this process's ranks' samples, and with
    streams = STG_SHARD_COLL | STG_SHARD_SIDE also only its ranks' collective
    events / GPU events / OS counter records (shard_rank_lo intervals)."""
    lo, hi = shard_bounds(len(win.rank_ids), world, rank)
    out = copy.copy(win)
    if streams and world > 1:
        rlo = shard_rank_lo(win.rank_ids, world, rank)
        rhi = shard_rank_lo(win.rank_ids, world, rank + 1) if rank + 1 < world else None
        keep_streams(out, None if rank == 0 else rlo, rhi, streams)
        out.shard_rank_lo = int(rlo)
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
