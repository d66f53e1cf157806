"""GPU: the device frame source rg_render_frames_device
against the host renderer rg_render_stereo_pair, which tests/test_oracle_cpu.py
pins to the reference's render_stereo_pair (synth.hpp:142-230) by frame
hashes.  Whole frames must be byte-identical: background and object value
noise, far-to-near painting, the right image's sheared spans, the radiometric
map, the vertical offset and the mt19937_64 / normal_distribution noise."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2604_07980_b200 import ranger as rg, synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = rg.Context(0)
    yield c
    c.close()


def _device(ctx, scenes):
    w, h = scenes[0].width, scenes[0].height
    dev = torch.device("cuda", 0)
    L = torch.full((len(scenes), h, w), 7, dtype=torch.uint8, device=dev)
    R = torch.full_like(L, 7)
    S.render_frames_device(ctx, scenes, L, R)
    torch.cuda.synchronize()
    return L.cpu().numpy(), R.cpu().numpy()


def _check(ctx, scenes):
    L, R = _device(ctx, scenes)
    for f, sc in enumerate(scenes):
        hl, hr = S.render_stereo_pair(sc)
        assert np.array_equal(L[f], hl), f"left frame {f}: {int((L[f] != hl).sum())} bytes differ"
        assert np.array_equal(R[f], hr), f"right frame {f}: {int((R[f] != hr).sum())} bytes differ"


@pytest.mark.parametrize("noise", [0.0, 2.0])
def test_c1_frames(ctx, noise):
    _check(ctx, [S.scene_c1(seed=s, noise=noise)[0] for s in (1, 2, 3)])


def test_c2_batch_with_noise(ctx):
    _check(ctx, [S.scene_c2(seed=100 + s, noise=2.0)[0] for s in range(6)])


def test_c3_occluded_pairs(ctx):
    _check(ctx, [S.scene_c3(seed=5, noise=2.0)[0], S.scene_c3(seed=6, noise=0.0, stress=True)[0]])


def test_every_scene_knob(ctx):
    """Radiometric map, vertical offsets of both signs, texture quantisation,
    disparity bias, sloped objects, strong noise (clamping at 0 / 255)."""
    base, _ = S.scene_c1(seed=9, noise=0.0)
    variants = [
        dict(gain=1.2, rad_bias=-6.0, gamma=0.8, noise_sigma=1.5),
        dict(vertical_offset_px=3, noise_sigma=2.0),
        dict(vertical_offset_px=-5, gain=0.9),
        dict(texture_quant=4, disparity_bias_px=1.5, noise_sigma=0.7),
        dict(noise_sigma=60.0, background_contrast=120.0),
        dict(texture_cell_px=3.5, seed=2**63 + 11, noise_sigma=3.0),
    ]
    scenes = []
    for v in variants:
        sc = dataclasses.replace(base, objects=list(base.objects), **v)
        scenes.append(sc)
    # sloped objects (disparity_ramp) and an object partly outside the image
    sl = dataclasses.replace(base, objects=list(base.objects), noise_sigma=1.0)
    sl.objects[0] = dataclasses.replace(sl.objects[0], disparity_ramp=0.05)
    sl.objects[3] = dataclasses.replace(sl.objects[3], disparity_ramp=-0.08)
    sl.objects.append(S.place(sl, 99, 5.0, 470.0, 20.0))
    scenes.append(sl)
    _check(ctx, scenes)


def test_empty_scene_and_rejections(ctx):
    sc = S.SceneConfig(width=64, height=48, noise_sigma=2.0, seed=3)
    _check(ctx, [sc])
    dev = torch.device("cuda", 0)
    L = torch.zeros((2, 48, 64), dtype=torch.uint8, device=dev)
    R = torch.zeros_like(L)
    bad = dataclasses.replace(sc, gamma=0.0)
    with pytest.raises(rg.InvalidArgument):
        S.render_frames_device(ctx, [sc, bad], L, R)
    other = dataclasses.replace(sc, width=32)
    with pytest.raises(rg.InvalidArgument):
        S.render_frames_device(ctx, [sc, other], L, R)
    behind = dataclasses.replace(sc, objects=[S.SceneObject(id=1, position=(-5.0, 0.0, 1.0))])
    with pytest.raises(rg.InvalidArgument):
        S.render_frames_device(ctx, [behind], L, R)
