"""GPU: the batched throughput APIs (rg_range_frames, rg_range_frames_host,
rg_auto_rect_frames) against the oracle frame by frame, and the drop-in proof
binaries (the reference's own unit + acceptance tests compiled against
include/ranger/)."""
import os
import subprocess

import numpy as np
import pytest

import oracle_lib
from paper_2604_07980_b200 import _abi, ranger as rg, synth as S
from paper_2604_07980_b200.engine import OUT_DTYPE, FrameEngine, pack_detections

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _frames(fn, n, **kw):
    Ls, Rs, D = [], [], []
    for i in range(n):
        sc, cfg = fn(seed=40 + i, noise=2.0, **kw)
        L, R = S.render_stereo_pair(sc)
        Ls.append(L)
        Rs.append(R)
        D.append(S.ground_truth_detections(sc))
    return np.stack(Ls), np.stack(Rs), D, cfg, sc


def _want(chk, L, R, dets, cfg):
    out, _ = chk.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                          cfg.to_c(), S.F_PX, S.BASELINE_M)
    return b"".join(bytes(o) for o in out)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_range_frames_device_and_host(ctx, chk, name):
    import torch

    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3}[name]
    n = 5 if name != "c3" else 3
    L, R, D, cfg, sc = _frames(fn, n)
    # vary the detection lists per frame: drop some boxes, permute others
    D = [d if i % 2 == 0 else list(reversed(d[: max(1, len(d) - i)])) for i, d in enumerate(D)]
    maxd = max(len(d) for d in D)
    eng = FrameEngine(sc.width, sc.height, cfg, maxd, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    dL, dR = torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev)
    out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(n, dtype=torch.int32, device=dev)
    eng.range_device(dL, dR, torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(n, eng.out_stride * 32)
    c = cnt.cpu().numpy()
    h_out = np.zeros(n * eng.out_stride, OUT_DTYPE)
    h_cnt = np.zeros(n, np.int32)
    eng.range_host(L, R, recs, offs, h_out, h_cnt, chunk=2)
    ho = h_out.view(np.uint8).reshape(n, eng.out_stride * 32)
    for f in range(n):
        want = _want(chk, L[f], R[f], D[f], cfg)
        assert int(c[f]) * 32 == len(want) and int(h_cnt[f]) == c[f]
        assert o[f, :len(want)].tobytes() == want
        assert ho[f, :len(want)].tobytes() == want


@pytest.mark.parametrize("name,n,wide,shift", [("c2", 12, False, False), ("c2", 13, False, True),
                                               ("c3", 12, False, False), ("c1", 16, True, True),
                                               ("c1", 16, False, False), ("c2", 1, False, False),
                                               ("c2", 3, False, True), ("c1", 2, True, False)])
def test_range_host_zero_copy_gather(ctx, chk, name, n, wide, shift):
    """rg_range_frames_host with pinned frames fetches only the image bytes
    the census reads for the matcher (gather_rows_kernel, zero-copy; batches
    of >= 12 frames take the ROI census, smaller ones the full-frame census
    over partly stale staging): the records equal the reference's, the
    staging buffers hold junk elsewhere (a previous batch of other frames),
    and fewer bytes than the frames cross the bus (rg_get_transfer)."""
    import torch

    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3}[name]
    L, R, D, cfg, sc = _frames(fn, n)
    cfg.census_9x7 = wide
    D = [d if i % 3 else list(reversed(d[: max(1, len(d) - i)])) for i, d in enumerate(D)]
    sh = ((np.arange(n) % 5) - 2).astype(np.int32) if shift else None
    maxd = max(len(d) for d in D)
    eng = FrameEngine(sc.width, sc.height, cfg, maxd, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)

    def pinned(a):
        t = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory()
        v = t.numpy().view(a.dtype).reshape(a.shape)
        v[...] = a
        return t, v
    keep = []
    for noise in (255 - L, L):  # first fill the staging with other frames
        tl, hL = pinned(noise if noise is not L else L)
        tr, hR = pinned(255 - R if noise is not L else R)
        keep += [tl, tr]
        h_out = np.zeros(n * eng.out_stride, OUT_DTYPE)
        h_cnt = np.zeros(n, np.int32)
        x0 = ctx.transfer()
        eng.range_host(hL, hR, recs, offs, h_out, h_cnt, chunk=n, left_shift=sh)
        x1 = ctx.transfer()
    assert 0 < x1[0] - x0[0] < L.nbytes + R.nbytes
    ho = h_out.view(np.uint8).reshape(n, eng.out_stride * 32)
    for f in range(n):
        Lf = L[f] if sh is None else np.ascontiguousarray(shift_vertical(L[f], int(sh[f])))
        want = _want(chk, Lf, R[f], D[f], cfg)
        assert int(h_cnt[f]) * 32 == len(want) and ho[f, :len(want)].tobytes() == want, (name, f)


def test_range_host_gather_padded_frames_and_partial_chunks(ctx, chk):
    """rg_range_frames_host over pinned frames with a padded pitch and frame
    stride (row and frame padding the gather must skip), 30 frames in chunks
    of 13 (a partial last chunk): records equal the reference's."""
    import ctypes as C
    import torch

    n, chunk = 30, 13
    L, R, D, cfg, sc = _frames(S.scene_c2, n)
    h, w = L.shape[1:]
    pitch, fstride = w + 64, (w + 64) * h + 4096
    eng = FrameEngine(w, h, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    bufs = []
    for img in (L, R):
        t = torch.zeros(n * fstride, dtype=torch.uint8).pin_memory()
        v = t.numpy()
        for f in range(n):
            v[f * fstride:f * fstride + pitch * h].reshape(h, pitch)[:, :w] = img[f]
        bufs.append(t)
    h_out = np.zeros(n * eng.out_stride, OUT_DTYPE)
    h_cnt = np.zeros(n, np.int32)
    b = eng._batch(n, pitch, fstride, bufs[0].data_ptr(), bufs[1].data_ptr(), recs.ctypes.data, offs.ctypes.data,
                   h_out.ctypes.data, h_cnt.ctypes.data)
    x0 = ctx.transfer()
    ctx.check(rg.lib().rg_range_frames_host(ctx.handle, C.byref(b), C.byref(eng._c), chunk, None))
    x1 = ctx.transfer()
    assert 0 < x1[0] - x0[0] < L.nbytes + R.nbytes
    ho = h_out.view(np.uint8).reshape(n, -1)
    for f in range(n):
        want = _want(chk, L[f], R[f], D[f], cfg)
        assert int(h_cnt[f]) * 32 == len(want) and ho[f, :len(want)].tobytes() == want, f


def test_census_rois_switch_same_records(ctx):
    """rg_set_census_rois(0) (full-frame census for every batch) and the
    default ROI tiles give byte-identical records on a 12-frame C2 batch."""
    import torch

    L, R, D, cfg, sc = _frames(S.scene_c2, 12)
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    args = (torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev), torch.from_numpy(recs.view(np.uint8)).to(dev),
            torch.from_numpy(offs).to(dev))
    outs = []
    for on in (True, False, True):
        ctx.set_census_rois(on)
        out = torch.zeros(12 * eng.out_stride * 32, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(12, dtype=torch.int32, device=dev)
        eng.range_device(*args, out, cnt)
        outs.append((out.cpu().numpy().tobytes(), cnt.cpu().numpy().tobytes()))
    ctx.set_census_rois(True)
    assert outs[0] == outs[1] == outs[2]


def shift_vertical(img, dy):
    """image.hpp:145-154: out(x, y) = in(x, clamp(y - dy, 0, H - 1))."""
    h = img.shape[0]
    return img[np.clip(np.arange(h) - dy, 0, h - 1)]


@pytest.mark.parametrize("name,wide", [("c1", False), ("c2", False), ("c1", True)])
def test_range_frames_left_shift(ctx, chk, name, wide):
    """Per-frame rect correction (pipeline.hpp:135-138) folded into the census
    row addressing == ranging shift_vertical(left, s) with the oracle."""
    import torch

    fn = {"c1": S.scene_c1, "c2": S.scene_c2}[name]
    shifts = np.array([-3, 0, 2, 5, -1], np.int32)
    n = len(shifts)
    L, R, D, cfg, sc = _frames(fn, n)
    cfg.census_9x7 = wide
    maxd = max(len(d) for d in D)
    eng = FrameEngine(sc.width, sc.height, cfg, maxd, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(n, dtype=torch.int32, device=dev)
    eng.range_device(torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev),
                     torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt,
                     left_shift=torch.from_numpy(shifts).to(dev))
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(n, eng.out_stride * 32)
    h_out = np.zeros(n * eng.out_stride, OUT_DTYPE)
    h_cnt = np.zeros(n, np.int32)
    eng.range_host(L, R, recs, offs, h_out, h_cnt, chunk=2, left_shift=shifts)
    ho = h_out.view(np.uint8).reshape(n, eng.out_stride * 32)
    for f in range(n):
        want = _want(chk, np.ascontiguousarray(shift_vertical(L[f], int(shifts[f]))), R[f], D[f], cfg)
        assert int(cnt[f]) * 32 == len(want) == int(h_cnt[f]) * 32
        assert o[f, :len(want)].tobytes() == want
        assert ho[f, :len(want)].tobytes() == want


def test_auto_rect_frames_equals_single(ctx):
    import torch

    n = 3
    Ls, Rs = [], []
    for i, voff in enumerate((-4, 0, 3)):
        sc = S.scene_c4(voff, seed=60 + i)
        L, R = S.render_stereo_pair(sc)
        Ls.append(L)
        Rs.append(R)
    L, R = np.stack(Ls), np.stack(Rs)
    cfg = rg.RangerConfig()
    eng = FrameEngine(1920, 1080, cfg, 1, ctx=ctx)
    dev = torch.device("cuda", 0)
    best = torch.zeros(n, dtype=torch.int32, device=dev)
    counts = torch.zeros(n * 17, dtype=torch.int64, device=dev)
    eng.auto_rect_device(torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev), S.C4_ROI, -8, 8, S.c4_bm(),
                         best, counts)
    torch.cuda.synchronize()
    for f in range(n):
        cs = []
        b = rg.auto_rect_search(L[f], R[f], rg.ImageRoi(*S.C4_ROI), -8, 8, S.c4_bm(), ctx=ctx, counts_out=cs)
        assert int(best[f]) == b == (-4, 0, 3)[f]
        assert counts[f * 17:(f + 1) * 17].cpu().tolist() == cs


@pytest.mark.parametrize("binary", ["unit_tests", "acceptance_tests"])
def test_reference_tests_pass_on_the_gpu_path(binary):
    exe = os.path.join(ROOT, "tests", "dropin", "_bin", binary)
    if not os.path.exists(exe):
        pytest.skip("drop-in binaries not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    if binary == "acceptance_tests":
        for c in (1, 3, 4, 5, 6, 7, 13, 14):
            assert f"criterion {c:2d}: PASS" in r.stdout
    else:  # census 9 + matching 10 + template_ranger 23 + autorect 8 + bm 9 + sgm 7 + pipeline 9 + radar_refiner 9
        assert "84 passed, 0 failed" in r.stdout, r.stdout[-3000:]


def test_integration_example_program():
    """INTEGRATION.md's C-ABI binding as a standalone C++ program
    (tests/dropin/integration_example.cpp): device frame loop + host records."""
    exe = os.path.join(ROOT, "tests", "dropin", "_bin", "integration_example")
    if not os.path.exists(exe):
        pytest.skip("integration example not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("frame ")]
    assert len(lines) == 6
    # the offset injected from frame 2 on is found and applied to later frames
    assert any("delta* 2" in l for l in lines) and "shift 0" in lines[0]


def _batch_vs_oracle(ctx, chk, L, R, D, cfg, focal=0.0, base=0.0, host=False):
    import torch

    n, h, w = L.shape
    maxd = max(1, max(len(d) for d in D))
    eng = FrameEngine(w, h, cfg, maxd, focal, base, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(n, dtype=torch.int32, device=dev)
    eng.range_device(torch.from_numpy(np.ascontiguousarray(L)).to(dev), torch.from_numpy(np.ascontiguousarray(R)).to(dev),
                     torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(n, eng.out_stride * 32)
    if host:  # the same batch from pinned host frames (zero-copy read-set gather when it applies)
        tl = torch.from_numpy(np.ascontiguousarray(L)).pin_memory()
        tr = torch.from_numpy(np.ascontiguousarray(R)).pin_memory()
        h_out = np.zeros(n * eng.out_stride, OUT_DTYPE)
        h_cnt = np.zeros(n, np.int32)
        eng.range_host(tl.numpy(), tr.numpy(), recs, offs, h_out, h_cnt, chunk=n)
        assert h_cnt.tobytes() == cnt.cpu().numpy().tobytes()
        ho = h_out.view(np.uint8).reshape(n, -1)
        for f in range(n):  # records past a frame's count are unspecified
            assert ho[f, :32 * int(h_cnt[f])].tobytes() == o[f, :32 * int(h_cnt[f])].tobytes(), f
    for f in range(n):
        got_n = int(cnt[f])
        if D[f]:
            want, _ = chk.estimate(np.ascontiguousarray(L[f]), np.ascontiguousarray(R[f]),
                                   [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in D[f]],
                                   cfg.to_c(), focal, base)
            want = b"".join(bytes(x) for x in want)
        else:
            want = b""
        assert got_n * 32 == len(want), (f, got_n, len(want))
        assert o[f, :len(want)].tobytes() == want, f


@pytest.mark.parametrize("batch", ["small", "roi"])
@pytest.mark.parametrize("case", ["odd_width", "empty_frames", "degenerate_boxes", "selection_overflow",
                                  "zero_range", "wide_range", "close_only_scale3"])
def test_range_frames_edge_cases(ctx, chk, case, batch):
    """Batched path vs the oracle on the shapes the planner/census/matcher
    special-case: non-multiple-of-4 widths (general census kernel), frames
    without detections, boxes leaving or degenerate in the image, more boxes
    than max_objects, one-candidate and >256-candidate search ranges, a
    non-half close scale (gather-mapped reduced raster).  batch "roi": the
    frames repeated to a 12+ frame batch (ROI-tile census, exact read sets)
    and also fed from pinned host frames (read-set gather)."""
    rng = np.random.default_rng(hash(case) % 1000)
    sc, cfg = S.scene_c1(seed=81, noise=2.0)
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    if case == "odd_width":
        L, R = L[:, :637], R[:, :637]
        frames = [(L, R, dets), (L, R, dets[::2])]
    elif case == "empty_frames":
        frames = [(L, R, []), (L, R, dets), (L, R, [])]
    elif case == "degenerate_boxes":
        bad = [rg.Detection(1.02, 0.5, 0.2, 0.2, 0, 900), rg.Detection(0.5, 0.5, 0.0, 0.3, 0, 901),
               rg.Detection(-0.05, 0.1, 0.2, 0.25, 1, 902), rg.Detection(0.5, 0.999, 0.3, 0.05, 0, 903),
               rg.Detection(0.5, 0.5, 1e-4, 1e-4, 0, 904)]
        frames = [(L, R, dets + bad), (L, R, bad)]
    elif case == "selection_overflow":
        cfg.max_objects = 3
        frames = [(L, R, dets), (L, R, list(reversed(dets)))]
    elif case == "zero_range":
        cfg.dx_max_far = 0
        cfg.dx_max_close = 0
        frames = [(L, R, dets)]
    elif case == "wide_range":
        cfg.dx_max_far = 300
        cfg.dx_max_close = 600
        frames = [(L, R, dets)]
    else:  # close_only_scale3
        cfg.close_scale = 3
        cfg.tau_s = 1e9  # everything CLOSE
        frames = [(L, R, dets)]
    if batch == "roi":
        frames = (frames * 12)[:max(12, len(frames))]
    Ls = np.stack([f[0] for f in frames])
    Rs = np.stack([f[1] for f in frames])
    _batch_vs_oracle(ctx, chk, Ls, Rs, [f[2] for f in frames], cfg, S.F_PX, S.BASELINE_M, host=batch == "roi")


@pytest.mark.parametrize("overlap", [True, False])
def test_range_frames_chunked_overlap_schedule(ctx, chk, overlap):
    """>= 32 frames take the chunked census/matcher overlap schedule (chunk
    rasters double-buffered across two streams); it must equal the oracle and
    the single-stream schedule frame by frame."""
    rng = np.random.default_rng(5)
    n = 37  # 4 chunks, the last one partial
    sc, cfg = S.scene_c1(seed=91, noise=2.0)
    L0, R0 = S.render_stereo_pair(sc)
    dets0 = S.ground_truth_detections(sc)
    L = np.stack([np.roll(L0, 3 * i, axis=1) for i in range(n)])
    R = np.stack([np.roll(R0, 3 * i, axis=1) for i in range(n)])
    D = [list(rng.permutation(dets0))[: 1 + (i % len(dets0))] for i in range(n)]
    ctx.set_overlap(overlap)
    try:
        _batch_vs_oracle(ctx, chk, L, R, D, cfg, S.F_PX, S.BASELINE_M)
    finally:
        ctx.set_overlap(False)


@pytest.mark.parametrize("name", ["c2", "c3s"])
def test_latency_and_throughput_matchers_agree(ctx, name):
    """Batches of <= 4 frames run the cooperative (CTA per FAR block) matcher,
    larger ones the warp-per-block one: the same frames give the same bytes
    either way, and repeated runs are bit-identical (determinism by
    construction: index-addressed writes, total-order argmin merges)."""
    import torch

    fn = {"c2": S.scene_c2, "c3s": lambda **k: S.scene_c3(stress=True, **k)}[name]
    L, R, D, cfg, sc = _frames(fn, 6)
    D = [d if i % 2 == 0 else list(reversed(d[: max(1, len(d) - 3 * i)])) for i, d in enumerate(D)]
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M, ctx=ctx)
    dev = torch.device("cuda", 0)

    def run(lo, hi):
        recs, offs = pack_detections(D[lo:hi])
        n = hi - lo
        out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        eng.range_device(torch.from_numpy(L[lo:hi]).to(dev), torch.from_numpy(R[lo:hi]).to(dev),
                         torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt)
        torch.cuda.synchronize()
        c = cnt.cpu().numpy()
        o = out.cpu().numpy().reshape(n, -1)
        return [o[f, :c[f] * 32].tobytes() for f in range(n)]

    big = run(0, 6)  # throughput matcher
    assert run(0, 6) == big  # repeat: bit-identical
    small = run(0, 1) + run(1, 3) + run(3, 6)  # latency matcher (1, 2, 3 frames)
    assert small == big


def _random_cfgs(n, seed=11):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        cfg = rg.RangerConfig(
            tau_s=float(rng.choice([20.0, 48.0, 100.0])), close_scale=int(rng.choice([1, 2, 3])),
            grid_side_points=int(rng.choice([2, 5, 8, 11])), max_total_points=int(rng.choice([4, 25, 64, 100])),
            close_block_side_points=int(rng.choice([2, 3, 5])), tau_d=float(rng.choice([0.5, 1.0, 3.0])),
            n_min=int(rng.choice([1, 3, 5])), tau_v=float(rng.choice([0.5, 1.0, 2.0])),
            max_objects=int(rng.choice([3, 8, 16])), dx_max_far=int(rng.choice([7, 33, 64, 100, 130])),
            dx_max_close=int(rng.choice([5, 64, 129, 192])))
        out.append(cfg)
    return out


@pytest.mark.parametrize("k", range(8))
def test_random_configs_both_matchers_match_oracle(ctx, chk, k):
    """Randomised RangerConfigs (ranges that are / are not multiples of 32,
    tails, tiny grids, close scales 1-3, selection budgets) on C1 frames:
    the latency (cooperative) matcher on a 1-frame batch and the throughput
    matcher on a 5-frame batch both equal the oracle frame by frame."""
    import torch

    cfg = _random_cfgs(8)[k]
    L, R, D, _, sc = _frames(S.scene_c1, 5)
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M, ctx=ctx)
    dev = torch.device("cuda", 0)

    def run(lo, hi):
        recs, offs = pack_detections(D[lo:hi])
        n = hi - lo
        out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        eng.range_device(torch.from_numpy(L[lo:hi]).to(dev), torch.from_numpy(R[lo:hi]).to(dev),
                         torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt)
        torch.cuda.synchronize()
        c = cnt.cpu().numpy()
        o = out.cpu().numpy().reshape(n, -1)
        return [o[f, :c[f] * 32].tobytes() for f in range(n)]

    big = run(0, 5)
    small = [run(f, f + 1)[0] for f in range(5)]
    for f in range(5):
        want = _want(chk, L[f], R[f], D[f], cfg)
        assert big[f] == want, (f, cfg)
        assert small[f] == want, (f, cfg)
    # a 15-frame batch (the 5 frames three times): the ROI-tile census with
    # the read sets of this config
    L, R, D = np.concatenate([L] * 3), np.concatenate([R] * 3), D * 3
    roi = run(0, 15)
    for f in range(15):
        assert roi[f] == big[f % 5], (f, cfg)


def test_multi_example_program():
    """The multi-GPU entry as a C++ program (tests/dropin/multi_example.cpp):
    frames sharded over every visible device, NCCL gather to device 0 and
    host copies, byte-equal to one context's rg_range_frames_host."""
    exe = os.path.join(ROOT, "tests", "dropin", "_bin", "multi_example")
    if not os.path.exists(exe):
        pytest.skip("multi example not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "multi ok" in r.stdout and "mismatches 0" in r.stdout


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_multi_ranger_matches_single_context_and_reference(ctx, chk, name):
    """MultiRanger on device 0 (one-rank NCCL communicator): host records and
    the device-0 gather equal FrameEngine.range_host and the reference."""
    import torch
    from paper_2604_07980_b200.engine import MultiRanger

    mk = S.scene_c1 if name == "c1" else S.scene_c2
    n = 9 if name == "c1" else 3
    scenes = [mk(seed=40 + f, noise=2.0) for f in range(n)]
    pairs = [S.render_stereo_pair(sc) for sc, _ in scenes]
    L = np.ascontiguousarray(np.stack([p[0] for p in pairs]))
    R = np.ascontiguousarray(np.stack([p[1] for p in pairs]))
    D = [S.ground_truth_detections(sc) for sc, _ in scenes]
    cfg = scenes[0][1]
    recs, offs = pack_detections(D)
    w, h = L.shape[2], L.shape[1]
    mr = MultiRanger([0], w, h, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M)
    out = np.zeros(n * mr.out_stride, OUT_DTYPE)
    cnt = np.zeros(n, np.int32)
    d_out = torch.zeros(n * mr.out_stride * 32, dtype=torch.uint8, device="cuda:0")
    d_cnt = torch.zeros(n, dtype=torch.int32, device="cuda:0")
    mr.range_host(L, R, recs, offs, out, cnt, d_out, d_cnt, chunk=2)
    mr.close()
    eng = FrameEngine(w, h, cfg, max(len(d) for d in D), S.F_PX, S.BASELINE_M, ctx=ctx)
    out1 = np.zeros(n * eng.out_stride, OUT_DTYPE)
    cnt1 = np.zeros(n, np.int32)
    eng.range_host(L, R, recs, offs, out1, cnt1, chunk=2)
    assert cnt.tolist() == cnt1.tolist() == d_cnt.cpu().tolist()
    assert out.tobytes() == out1.tobytes() == d_out.cpu().numpy().tobytes()
    for f in range(n):
        got = out.reshape(n, -1)[f][:cnt[f]]
        assert got.tobytes() == _want(chk, L[f], R[f], D[f], cfg)


@pytest.mark.parametrize("grid,maxp,frames", [(12, 144, 6), (12, 144, 2), (32, 1024, 6), (32, 1024, 1)])
def test_large_blocks_fit_the_device_matcher(ctx, chk, grid, maxp, frames):
    """Blocks of 144 and 1024 points (grid_side_points 12 / 32) through the
    batched matcher (throughput variant > 4 frames, latency variant <= 4):
    shared memory opts in for static + dynamic bytes and falls back to fewer
    warps per CTA when 16 warps' points do not fit."""
    import torch

    L, R, D, cfg, sc = _frames(S.scene_c1, frames)
    cfg.grid_side_points = grid
    cfg.max_total_points = maxp
    eng = FrameEngine(sc.width, sc.height, cfg, 8, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    out = torch.zeros(frames * eng.out_stride * 32, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(frames, dtype=torch.int32, device=dev)
    eng.range_device(torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev),
                     torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev), out, cnt)
    o = out.cpu().numpy().reshape(frames, -1)
    for f in range(frames):
        want = _want(chk, L[f], R[f], D[f], cfg)
        assert int(cnt[f]) * 32 == len(want) and o[f, :len(want)].tobytes() == want


@pytest.mark.parametrize("name,n,wide", [("c1", 16, False), ("c2", 12, False), ("c3", 12, False),
                                         ("c1", 16, True), ("c2", 12, True), ("c3", 12, True)])
def test_roi_census_batches_match_reference(ctx, chk, name, n, wide):
    """Batches of >= 12 frames take the ROI census (census_rows_kernel + the
    warp tile kernels over compacted tile lists; 9x7: census64_rowtile_kernel);
    a per-frame left shift (rect correction) and detection lists that differ
    per frame included.  Every record equals the reference's (9x7: the
    restatement's)."""
    import torch

    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3}[name]
    L, R, D, cfg, sc = _frames(fn, n)
    cfg.census_9x7 = wide
    D = [d if i % 3 else list(reversed(d[: max(1, len(d) - i)])) for i, d in enumerate(D)]
    shifts = ((np.arange(n) % 5) - 2).astype(np.int32)
    maxd = max(len(d) for d in D)
    eng = FrameEngine(sc.width, sc.height, cfg, maxd, S.F_PX, S.BASELINE_M, ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    dL, dR = torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev)
    d_recs, d_offs = torch.from_numpy(recs.view(np.uint8)).to(dev), torch.from_numpy(offs).to(dev)
    for sh in (None, shifts):
        out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        eng.range_device(dL, dR, d_recs, d_offs, out, cnt,
                         left_shift=torch.from_numpy(sh).to(dev) if sh is not None else None)
        o = out.cpu().numpy().reshape(n, -1)
        for f in range(n):
            Lf = L[f] if sh is None else np.ascontiguousarray(shift_vertical(L[f], int(sh[f])))
            want = _want(chk, Lf, R[f], D[f], cfg)
            assert int(cnt[f]) * 32 == len(want) and o[f, :len(want)].tobytes() == want, (name, f)
