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
