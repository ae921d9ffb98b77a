"""K1/K2 gather kernel: nearest is bit-exact with the reference cutter (via the golden
hashes produced by the reference and the oracle restatement), bilinear is bit-exact
with the integer restatement in oracle/resample_ref.py. Includes the reference's own
TestCutTile cases (test_detector.py:277-319): native copy, upscale, downscale sampling
positions, out-of-frame zero fill."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pipeline_ref, resample_ref
from paper_1810_10551_b200 import detector, kernels
from paper_1810_10551_b200.geometry import CropSpec, Rect

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _frame(h, w, seed):
    return np.random.default_rng(seed).integers(0, 255, (h, w, 3), np.uint8)


def _crop(x, y, side):
    return CropSpec(0, 0, 0, Rect(x, y, side, side), side / 608)


def test_nearest_matches_reference_golden_hashes(cuda):
    for case in GOLD["cut_tile"]:
        px = _frame(case["h"], case["w"], case["seed"])
        tile = detector.cut_tile(px, _crop(case["x"], case["y"], case["side"]))
        assert hashlib.sha256(tile.tobytes()).hexdigest() == case["sha256"], case


def test_reference_cut_tile_cases(cuda):
    px = _frame(700, 900, 0)
    assert np.array_equal(detector.cut_tile(px, _crop(120, 30, 608)), px[30:638, 120:728])
    px = _frame(400, 400, 0)
    src = (np.arange(608) * 304) // 608
    assert np.array_equal(detector.cut_tile(px, _crop(10, 20, 304)), px[20 + src][:, 10 + src])
    px = _frame(500, 500, 0)
    t = detector.cut_tile(px, _crop(450, 450, 608))
    assert np.array_equal(t[:50, :50], px[450:, 450:])
    assert not t[50:, :].any() and not t[:, 50:].any()
    with pytest.raises(ValueError):
        detector.cut_tile(np.zeros((100, 100), np.uint8), _crop(0, 0, 50))


@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
def test_batched_gather_matches_oracle(cuda, mode):
    torch = cuda
    rng = np.random.default_rng(7)
    H, W = 2160, 3840
    frames = rng.integers(0, 256, (2, H, W, 3), np.uint8)
    crops = [(0, 0, 2160), (1680, 0, 2160), (0, 0, 736), (3104, 1424, 736), (-30, 2000, 554),
             (3500, 2100, 1098), (0, 0, 3840), (100, 100, 300), (-500, -300, 4320),
             (3300, 700, 4320), (3833, 5, 608), (1000, 1000, 7000)]
    rows = [(f, 0, x, y, s, 0) for f in range(2) for (x, y, s) in crops]
    jobs = kernels.jobs_tensor(rows)
    dev = torch.from_numpy(frames).cuda()
    out = torch.empty((len(rows), 608, 608, 3), dtype=torch.uint8, device="cuda")
    kernels.gather(dev, H * W * 3, H, W, jobs, len(rows), mode, out_u8=out)
    got = out.cpu().numpy()
    for i, (f, _, x, y, s, _) in enumerate(rows):
        if mode == "nearest":
            ref = pipeline_ref.cut_tile_nearest(frames[f], (0, 0, 0, x, y, s, s / 608))
        else:
            ref = resample_ref.cut_tile_bilinear(frames[f], x, y, s)
        assert np.array_equal(got[i], ref), (mode, x, y, s)


def test_gather_bf16_activation_layout(cuda):
    torch = cuda
    rng = np.random.default_rng(9)
    frame = rng.integers(0, 256, (700, 900, 3), np.uint8)
    jobs = kernels.jobs_tensor([(0, 0, 50, 40, 640, 0)])
    act = torch.zeros((1, 610, 614, 4), dtype=torch.bfloat16, device="cuda")
    u8 = torch.empty((1, 608, 608, 3), dtype=torch.uint8, device="cuda")
    kernels.gather(torch.from_numpy(frame).cuda(), 0, 700, 900, jobs, 1, "bilinear", out_u8=u8,
                   out_act_ptr=act.data_ptr())
    ref = torch.from_numpy(resample_ref.cut_tile_bilinear(frame, 50, 40, 640)).float() / 255.0
    ref = ref.to(torch.bfloat16).float()
    _check_layout(act, ref)


def _check_layout(act, ref):
    """pixel (v, u) at [v+1][u+2] as rgb0; zero halo rows 0 / 609 and columns 0, 1, 610..613."""
    got = act[0, 1:-1].cpu().float()
    assert torch_equal(got[:, 2:610, 0:3], ref)
    assert got[:, :, 3].abs().max().item() == 0
    assert got[:, :2].abs().max().item() == 0 and got[:, 610:].abs().max().item() == 0
    assert act[0, 0].abs().max().item() == 0 and act[0, -1].abs().max().item() == 0


def torch_equal(a, b):
    import torch

    return torch.equal(a, b)


@pytest.mark.parametrize("mode", ["nearest", "bilinear"])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_gather_slot_layout_per_plan(cuda, mode, dtype):
    """Layer-0 input pixels in the parity plan (exact integer values) and the fp16 plan
    (value/255), crops partly outside the frame and down/up-scaled, both resample modes."""
    torch = cuda
    rng = np.random.default_rng(11)
    H, W = 2160, 3840
    frame = rng.integers(0, 256, (H, W, 3), np.uint8)
    for (x, y, s) in [(3104, 1424, 736), (-30, 2000, 554), (0, 0, 2160), (3500, 2100, 1098),
                      (100, 100, 300)]:
        jobs = kernels.jobs_tensor([(0, 0, x, y, s, 0)])
        act = torch.zeros((1, 610, 614, 4), dtype=torch.float16, device="cuda")
        kernels.gather(torch.from_numpy(frame).cuda(), 0, H, W, jobs, 1, mode,
                       out_act_ptr=act.data_ptr(), dtype=dtype)
        if mode == "nearest":
            tile = pipeline_ref.cut_tile_nearest(frame, (0, 0, 0, x, y, s, s / 608))
        else:
            tile = resample_ref.cut_tile_bilinear(frame, x, y, s)
        ref = torch.from_numpy(tile).float()
        if dtype == "fp16":
            ref = (ref / 255.0).to(torch.float16).float()
        _check_layout(act, ref)
