"""GPU: census SGM (sgm.hpp:37-155) bit-exact against the
oracle (itself pinned to the reference's outputs in tests/golden), including
the detail:: building blocks the reference's own tests use."""
import ctypes as C

import numpy as np
import pytest

from paper_2604_07980_b200 import _abi, ranger as rg, synth as S

pytestmark = pytest.mark.gpu


def rand_img(rng, h, w):
    return rng.integers(0, 256, (h, w), dtype=np.uint8)


@pytest.mark.parametrize("w,h,nd,d_lo,p1,p2", [(40, 24, 16, 0, 8, 32), (33, 17, 8, -3, 0, 0), (64, 20, 24, 2, 3, 50),
                                               (90, 7, 32, -8, 8, 32), (70, 30, 40, 0, 8, 32),
                                               (50, 12, 96, -20, 5, 60), (1, 9, 4, 0, 8, 32),
                                               (80, 16, 48, -5, 4, 20), (120, 10, 64, -10, 8, 32),
                                               (70, 9, 64, 3, 100, 300)])
def test_sgm_random_matches_oracle(ctx, orc, w, h, nd, d_lo, p1, p2):
    rng = np.random.default_rng(w * 31 + nd)
    a, b = rand_img(rng, h, w), rand_img(rng, h, w)
    got = rg.sgm_disparity(a, b, rg.SgmParams(nd, d_lo, p1, p2), ctx=ctx)
    assert np.array_equal(got, orc.sgm(a, b, nd, d_lo, p1, p2))


def test_sgm_rendered_scene_matches_oracle(ctx, orc):
    sc = S.SceneConfig(width=256, height=120, background_contrast=90, seed=9,
                       objects=[S.SceneObject(id=1, position=(12.0, 0.5, 1.4), texture_seed=5)])
    L, R = S.render_stereo_pair(sc)
    got = rg.sgm_disparity(L, R, rg.SgmParams(64, 0, 8, 32), ctx=ctx)
    want = orc.sgm(L, R, 64, 0, 8, 32)
    assert np.array_equal(got, want)
    assert (got != -32768).mean() > 0.5


def test_sgm_detail_blocks_match_oracle(ctx, orc):
    lib = rg.lib()
    rng = np.random.default_rng(3)
    for (w, h, nd, p1, p2) in [(17, 9, 12, 3, 20), (8, 23, 40, 0, 5), (31, 5, 70, 7, 7)]:
        cost = rng.integers(0, 28, (h, w, nd), dtype=np.uint8)
        for sx, sy in [(1, 0), (0, 1), (1, 1), (-1, 1), (-1, 0), (0, -1), (1, -1), (-1, -1)]:
            acc0 = rng.integers(-5, 5, (h, w, nd)).astype(np.int32)
            got, want = acc0.copy(), acc0.copy()
            ctx.check(lib.rg_sgm_direction_pass(ctx.handle, cost.ctypes.data, w, h, nd, p1, p2, sx, sy,
                                                got.ctypes.data))
            assert orc.lib.orc_sgm_direction_pass(cost.ctypes.data, w, h, nd, p1, p2, sx, sy, want.ctypes.data) == 0
            assert np.array_equal(got, want), (w, h, nd, sx, sy)
    # cost volume from census codes (sgm.hpp:37-56)
    a, b = rand_img(rng, 11, 29), rand_img(rng, 11, 29)
    cl, cr = orc.census(a), orc.census(b)
    p = _abi.SgmParams(20, -4, 8, 32)
    cost = np.zeros((11, 29, 20), np.uint8)
    ctx.check(lib.rg_sgm_cost_volume(ctx.handle, cl.ctypes.data, cr.ctypes.data, 29, 11, C.byref(p),
                                     cost.ctypes.data))
    want = np.full((11, 29, 20), 27, np.uint8)
    for y in range(11):
        for x in range(29):
            for i in range(20):
                rx = x - (-4 + i)
                if 0 <= rx < 29:
                    want[y, x, i] = bin(int(cl[y, x]) ^ int(cr[y, rx])).count("1")
    assert np.array_equal(cost, want)


def test_sgm_frames_batched_equals_single(ctx):
    import torch

    rng = np.random.default_rng(11)
    n, h, w = 3, 40, 96
    L = np.stack([rand_img(rng, h, w) for _ in range(n)])
    R = np.stack([rand_img(rng, h, w) for _ in range(n)])
    p = rg.SgmParams(32, 0, 8, 32)
    dev = torch.device("cuda", 0)
    out = torch.zeros(n * h * w, dtype=torch.int16, device=dev)
    pc = p.to_c()
    dL, dR = torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev)  # alive until after the sync
    torch.cuda.synchronize()
    ctx.check(rg.lib().rg_sgm_frames(ctx.handle, dL.data_ptr(), dR.data_ptr(), n, h * w, w, w, h, C.byref(pc),
                                     out.data_ptr(), None))
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(n, h, w)
    for f in range(n):
        assert np.array_equal(got[f], rg.sgm_disparity(L[f], R[f], p, ctx=ctx))


def test_sgm_validation(ctx):
    img = np.zeros((8, 8), np.uint8)
    for bad in (rg.SgmParams(0, 0, 8, 32), rg.SgmParams(16, 0, -1, 32), rg.SgmParams(16, 0, 40, 32)):
        with pytest.raises(rg.InvalidArgument):
            rg.sgm_disparity(img, img, bad, ctx=ctx)
