"""CPU, world_size 2 (gloo): frames shard across ranks with no compute-path
collective; per-box results gather to rank 0 in frame order.  The per-rank
compute here is the C oracle (this test checks the host plumbing; the GPU
kernels are covered by the gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_frames, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_lib
    from paper_2604_07980_b200 import _abi, shard, synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE

    orc = oracle_lib.oracle()
    lo, hi = shard.shard_bounds(n_frames, rank, world)
    out = np.zeros((hi - lo, 8), OUT_DTYPE)
    cnt = np.zeros(hi - lo, np.int32)
    for k, f in enumerate(range(lo, hi)):
        sc, cfg = S.scene_c1(seed=100 + f, noise=2.0)
        L, R = S.render_stereo_pair(sc)
        dets = S.ground_truth_detections(sc)
        res, _ = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                              cfg.to_c(), 2000.0, 0.3)
        cnt[k] = len(res)
        out[k, :len(res)] = np.frombuffer(b"".join(bytes(r) for r in res), OUT_DTYPE)
    got = shard.gather_results(out, cnt, n_frames)
    if rank == 0:
        q.put((got[0].tobytes(), got[1].tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [5, 6])
def test_two_rank_shard_and_gather_equals_single_process(n_frames):
    import oracle_lib
    from paper_2604_07980_b200 import _abi, synth as S
    from paper_2604_07980_b200.engine import OUT_DTYPE

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, cnt = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = oracle_lib.oracle()
    want = np.zeros((n_frames, 8), OUT_DTYPE)
    for f in range(n_frames):
        sc, cfg = S.scene_c1(seed=100 + f, noise=2.0)
        L, R = S.render_stereo_pair(sc)
        dets = S.ground_truth_detections(sc)
        res, _ = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                              cfg.to_c(), 2000.0, 0.3)
        want[f, :len(res)] = np.frombuffer(b"".join(bytes(r) for r in res), OUT_DTYPE)
    assert full == want.tobytes() and cnt == [8] * n_frames
