"""Multi-GPU plumbing: frames shard across ranks, results gather to rank 0.

SURVEY.md 8(e): frames are independent, so frame f runs on rank
floor(f * G / N) (contiguous shards) with no collective on the compute path;
the only exchange is the per-box result gather (NCCL over NVLink on GPUs,
gloo in the CPU tests) into frame order on rank 0.  Sequential cross-frame
state (the rectification offset filter, autorect.hpp:77-90) is a host scan
between the two sharded passes (rect_shift_schedule).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def shard_bounds(n_frames: int, rank: int, world: int) -> Tuple[int, int]:
    """[begin, end) of the frames with floor(f * world / n_frames) == rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = -(-rank * n_frames // world)  # ceil(rank * N / G)
    hi = -(-(rank + 1) * n_frames // world)
    return lo, hi


def owner_of(frame: int, n_frames: int, world: int) -> int:
    return frame * world // n_frames


def gather_results(out: np.ndarray, counts: np.ndarray, n_frames: int, group=None, device=None
                   ) -> Optional[Tuple[np.ndarray, np.ndarray]]:
    """All ranks call with their shard's result records (rows = frames of the
    shard, any fixed record dtype) and counts; rank 0 returns the full
    (n_frames, ...) arrays in frame order, other ranks None.  Uses one padded
    all_gather of bytes (NCCL has no gather)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_frames // world)
    rec_bytes = out.dtype.itemsize * int(np.prod(out.shape[1:], dtype=np.int64))
    slab = np.zeros(per * rec_bytes + per * 4, np.uint8)
    lo, hi = shard_bounds(n_frames, rank, world)
    n = hi - lo
    if out.shape[0] != n or counts.shape[0] != n:
        raise ValueError("shard size mismatch")
    slab[:n * rec_bytes] = np.frombuffer(np.ascontiguousarray(out).tobytes(), np.uint8)
    slab[per * rec_bytes:per * rec_bytes + 4 * n] = np.frombuffer(counts.astype(np.int32).tobytes(), np.uint8)
    t = torch.from_numpy(slab)
    if device is not None:
        t = t.to(device)
    bufs = torch.zeros(world * t.numel(), dtype=torch.uint8, device=t.device)
    dist.all_gather_into_tensor(bufs, t, group=group)
    if rank != 0:
        return None
    allb = bufs.cpu().numpy().reshape(world, -1)
    full = np.zeros((n_frames,) + out.shape[1:], out.dtype)
    cnt = np.zeros(n_frames, np.int32)
    for r in range(world):
        a, b = shard_bounds(n_frames, r, world)
        k = b - a
        full[a:b] = np.frombuffer(allb[r, :k * rec_bytes].tobytes(), out.dtype).reshape((k,) + out.shape[1:])
        cnt[a:b] = np.frombuffer(allb[r, per * rec_bytes:per * rec_bytes + 4 * k].tobytes(), np.int32)
    return full, cnt


# ---------------------------------------------------------------- stream plumbing
# The bench's C5 stream and its ring steps run exactly these functions (with
# rg_range_frames as `range_chunk`); tests/test_dist_cpu.py runs them at world
# size 2 over gloo with the C oracle as `range_chunk`.

def stream_chunks(n_frames: int, rank: int, world: int, chunk: int) -> List[Tuple[int, int]]:
    """This rank's shard of an n_frames stream cut into chunks of <= chunk
    frames: [(global_lo, global_hi)], in frame order."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    lo, hi = shard_bounds(n_frames, rank, world)
    return [(c, min(hi, c + chunk)) for c in range(lo, hi, chunk)]


def slab_frames(n_frames: int, world: int) -> int:
    """Frames per rank slab of the padded gather (the largest shard)."""
    return -(-n_frames // world)


def alloc_slabs(n_frames: int, world: int, rec_bytes: int, device=None):
    """Per-rank result slab (uint8, slab_frames * rec_bytes) and counts
    (int32, slab_frames), plus the gathered buffers (world x the slab) --
    the shard's frames occupy the head of the slab in frame order."""
    import torch

    per = slab_frames(n_frames, world)
    out = torch.zeros(per * rec_bytes, dtype=torch.uint8, device=device)
    cnt = torch.zeros(per, dtype=torch.int32, device=device)
    g_out = torch.zeros(world * out.numel(), dtype=torch.uint8, device=device) if world > 1 else out
    g_cnt = torch.zeros(world * per, dtype=torch.int32, device=device) if world > 1 else cnt
    return out, cnt, g_out, g_cnt


def run_stream(range_chunk, n_frames: int, rank: int, world: int, chunk: int, out, cnt, rec_bytes: int) -> int:
    """Range this rank's shard chunk by chunk: range_chunk(glo, ghi, out_view,
    cnt_view) writes frames [glo, ghi)'s records and counts into the views of
    the slab.  No collective.  Returns the frames ranged."""
    lo, _ = shard_bounds(n_frames, rank, world)
    done = 0
    for glo, ghi in stream_chunks(n_frames, rank, world, chunk):
        a, b = glo - lo, ghi - lo
        range_chunk(glo, ghi, out[a * rec_bytes:b * rec_bytes], cnt[a:b])
        done += ghi - glo
    return done


def gather_slabs(out, cnt, g_out, g_cnt, world: int, group=None) -> None:
    """The only exchange: every rank's slab of records and counts to every
    rank (one all_gather each; NCCL over NVLink on GPUs, gloo on CPU)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_gather_into_tensor(g_out, out, group=group)
        dist.all_gather_into_tensor(g_cnt, cnt, group=group)


def frame_order(g_out, g_cnt, n_frames: int, world: int, rec_bytes: int):
    """Gathered slabs -> (records uint8 (n_frames, rec_bytes), counts int32
    (n_frames)) in global frame order (the reference's sequential order,
    pipeline.hpp:338-344)."""
    per = slab_frames(n_frames, world)
    ob = g_out.cpu().numpy().reshape(world, per, rec_bytes)
    cb = g_cnt.cpu().numpy().reshape(world, per)
    recs = np.zeros((n_frames, rec_bytes), np.uint8)
    cnt = np.zeros(n_frames, np.int32)
    for r in range(world):
        a, b = shard_bounds(n_frames, r, world)
        recs[a:b] = ob[r, :b - a]
        cnt[a:b] = cb[r, :b - a]
    return recs, cnt


def gathered_boxes(g_cnt, n_frames: int, world: int) -> int:
    """Boxes ranged over the whole stream (padding rows of short shards excluded)."""
    per = slab_frames(n_frames, world)
    cb = g_cnt.cpu().numpy().reshape(world, per)
    return int(sum(int(cb[r, :shard_bounds(n_frames, r, world)[1] - shard_bounds(n_frames, r, world)[0]].sum())
                   for r in range(world)))


def rect_shift_schedule(delta_stars: Sequence[int], window: int = 5, rate: float = 1.0) -> List[int]:
    """Two-pass rect schedule: from the per-frame search
    results delta*_t (pass A, computed sharded on the uncorrected pairs,
    pipeline.hpp:144-149), the left-image row shift applied to frame t is
    lround(current before frame t's filter update) (pipeline.hpp:135-138, 178)."""
    from .ranger import RectOffsetState, filter_offset

    st = RectOffsetState(window, rate)
    shifts = []
    for d in delta_stars:
        c = st.current
        shifts.append(int(np.floor(abs(c) + 0.5)) * (1 if c >= 0 else -1))  # std::lround
        filter_offset(st, int(d))
    return shifts
