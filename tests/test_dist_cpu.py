"""CPU, world_size 2 (gloo): the bench's sharded stream plumbing
(shard.run_stream -> gather_slabs -> frame_order / gathered_boxes, the exact
functions bench.py's ring steps and C5 stream run) with the C oracle standing
in for rg_range_frames.  Frames shard across ranks with no compute-path
collective; the gathered per-box records equal the single-process records in
the reference's sequential frame order (pipeline.hpp:338-344)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

REC = 8 * 32  # out_stride 8 (C1) x rg_object_disparity


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame_records(f):
    """Frame f of the test stream (C1 scene, seed 100 + f) ranged by the oracle."""
    import oracle_lib
    from paper_2604_07980_b200 import _abi, synth as S

    sc, cfg = S.scene_c1(seed=100 + f, noise=2.0)
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    res, _ = oracle_lib.oracle().estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id)
                                                 for d in dets], cfg.to_c(), 2000.0, 0.3)
    return b"".join(bytes(r) for r in res), len(res)


def _run_shard(n_frames, rank, world, chunk):
    import torch
    from paper_2604_07980_b200 import shard

    out, cnt, g_out, g_cnt = shard.alloc_slabs(n_frames, world, REC)
    calls = []

    def range_chunk(glo, ghi, o, c):  # rg_range_frames stand-in: writes the chunk's slab rows
        calls.append((glo, ghi))
        for k, f in enumerate(range(glo, ghi)):
            b, n = _frame_records(f)
            o[k * REC:k * REC + len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8)
            c[k] = n

    done = shard.run_stream(range_chunk, n_frames, rank, world, chunk, out, cnt, REC)
    shard.gather_slabs(out, cnt, g_out, g_cnt, world)
    recs, counts = shard.frame_order(g_out, g_cnt, n_frames, world, REC)
    return recs, counts, shard.gathered_boxes(g_cnt, n_frames, world), calls, done


def _worker(rank, world, port, n_frames, chunk, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs, counts, boxes, calls, done = _run_shard(n_frames, rank, world, chunk)
    q.put((rank, recs.tobytes(), counts.tolist(), boxes, calls, done))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames,chunk", [(5, 2), (6, 4), (3, 8)])
def test_two_rank_stream_equals_single_process(n_frames, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process, world 1, same functions
    recs1, counts1, boxes1, calls1, done1 = _run_shard(n_frames, 0, 1, chunk)
    assert done1 == n_frames and calls1 == [(c, min(n_frames, c + chunk)) for c in range(0, n_frames, chunk)]
    want = np.zeros((n_frames, REC), np.uint8)
    for f in range(n_frames):
        b, n = _frame_records(f)
        want[f, :len(b)] = np.frombuffer(b, np.uint8)
    assert recs1.tobytes() == want.tobytes() and counts1.tolist() == [8] * n_frames
    for rank, recs, counts, boxes, calls, done in got:
        # every rank sees the whole stream in frame order after the gather
        assert recs == want.tobytes() and counts == [8] * n_frames and boxes == boxes1 == 8 * n_frames
        lo, hi = (0, (n_frames + 1) // 2) if rank == 0 else ((n_frames + 1) // 2, n_frames)
        assert done == hi - lo
        assert calls == [(c, min(hi, c + chunk)) for c in range(lo, hi, chunk)]  # contiguous, no overlap


def test_stream_chunks_cover_the_stream_once():
    from paper_2604_07980_b200 import shard

    for n in (0, 1, 7, 256, 4096):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                seen += [f for a, b in shard.stream_chunks(n, r, world, 256) for f in range(a, b)]
            assert seen == list(range(n))
            assert shard.slab_frames(n, world) == max(shard.shard_bounds(n, r, world)[1]
                                                      - shard.shard_bounds(n, r, world)[0] for r in range(world))
