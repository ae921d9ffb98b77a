"""tcgen05 implicit-GEMM conv kernel vs a plain PyTorch fp32 conv of the same op.

Activations are compact NHWC [n][res][res][C] (the conv's zero padding is TMA
out-of-bounds fill). Inputs/weights are bf16/fp16 (exactly representable in fp32), the
reference accumulates in fp32 with TF32 off; the kernel accumulates in fp32 in TMEM and
rounds the output to 16 bits, so the tolerance is the output rounding (2^-8 / 2^-11
relative) plus accumulation-order noise.
"""

import numpy as np
import pytest

from oracle import yolo_ref

from paper_1810_10551_b200 import native, yolo

pytestmark = pytest.mark.gpu


DT = {"bf16": "bfloat16", "fp16": "float16"}


def _input(torch, n, res, c, seed, dtype="bf16"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(n, res, res, c, generator=g)
    return x.to(getattr(torch, DT[dtype])).cuda()


def _run_conv(torch, x, res, cin, cout, cout_pad, k, leaky, out_fp32=False, reorg=False,
              out_cstride=None, out_coff=0, seed=1, dtype="bf16", pool=False):
    n = x.shape[0]
    tdt = getattr(torch, DT[dtype])
    g = torch.Generator(device="cpu").manual_seed(seed)
    taps = k * k
    scale = (2.0 / (cin * taps)) ** 0.5
    w = torch.randn(cout, taps, cin, generator=g) * scale
    bias = torch.randn(cout, generator=g) * 0.1
    wpack = torch.zeros(cout_pad, taps * cin)
    wpack[:cout, : taps * cin] = w.reshape(cout, taps * cin)
    wpack = wpack.to(tdt).cuda()
    bpack = torch.zeros(cout_pad)
    bpack[:cout] = bias
    bpack = bpack.cuda()
    if out_cstride is None:
        out_cstride = cout_pad if out_fp32 else cout
    ores = res // 2 if (reorg or pool) else res
    out = torch.zeros(n, ores, ores, out_cstride,
                      dtype=torch.float32 if out_fp32 else tdt, device="cuda")
    native.call("tp_conv", native.ptr(x), n, res, cin, native.ptr(wpack), native.ptr(bpack),
                cout, cout_pad, k, int(leaky), native.ptr(out), out_cstride, out_coff,
                int(out_fp32), int(reorg), native.DTYPES[dtype], int(pool),
                native.stream_handle())
    torch.cuda.synchronize()
    # reference
    xin = x.float().permute(0, 3, 1, 2)
    wq = wpack[:cout, : taps * cin].float().reshape(cout, k, k, cin).permute(0, 3, 1, 2)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    ref = torch.nn.functional.conv2d(xin, wq, bias=bpack[:cout], padding=k // 2)
    if leaky:
        ref = torch.where(ref > 0, ref, 0.1 * ref)
    if pool:
        ref = torch.nn.functional.max_pool2d(ref, 2)
    ref = ref.permute(0, 2, 3, 1)  # n, res, res, cout
    return out, ref


def _check(torch, got, ref, rel=2e-2):
    got = got.float()
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err <= rel * scale, f"max err {err} vs scale {scale}"


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize(
    "cin,cout,k,res",
    [(32, 32, 3, 16), (32, 64, 3, 16), (64, 128, 3, 19), (128, 64, 1, 19), (256, 512, 3, 12),
     (64, 1024, 1, 7)],
)
def test_conv_matches_torch(cuda, cin, cout, k, res, dtype):
    torch = cuda
    x = _input(torch, 3, res, cin, seed=cin + cout, dtype=dtype)
    out, ref = _run_conv(torch, x, res, cin, cout, cout, k, leaky=True, dtype=dtype)
    _check(torch, out, ref, rel=2e-2 if dtype == "bf16" else 3e-3)


def test_conv_head_fp32_linear(cuda):
    torch = cuda
    x = _input(torch, 2, 19, 64, seed=5)
    out, ref = _run_conv(torch, x, 19, 64, 425, 448, 1, leaky=False, out_fp32=True)
    got = out[..., :425]
    err = (got - ref).abs().max().item()
    assert err <= 1e-3 * (ref.abs().max().item() + 1e-6)


def test_conv_reorg_and_channel_offset(cuda):
    torch = cuda
    x = _input(torch, 2, 38, 64, seed=9)
    out, ref = _run_conv(torch, x, 38, 64, 64, 64, 1, leaky=True, reorg=True, out_cstride=1280,
                         out_coff=0)
    # darknet reorg (reorg_cpu forward=0), restated in oracle/yolo_ref.reorg
    r = yolo_ref.reorg(ref.permute(0, 3, 1, 2).cpu()).permute(0, 2, 3, 1).to(ref.device)
    _check(torch, out[..., :256], r)
    assert out[..., 256:].abs().max().item() == 0
    out2, ref2 = _run_conv(torch, _input(torch, 2, 19, 128, seed=3), 19, 128, 64, 64, 3,
                           leaky=True, out_cstride=1280, out_coff=256)
    _check(torch, out2[..., 256:320], ref2)
    assert out2[..., :256].abs().max().item() == 0


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("cin,cout,res,n", [(32, 64, 32, 2), (64, 128, 40, 2), (128, 256, 76, 2),
                                            (64, 128, 152, 2), (128, 128, 48, 3),
                                            (128, 128, 152, 5)])
def test_conv_fused_pool_rect_tiles(cuda, cin, cout, res, n, dtype):
    """RECT 16x8 tiles (3-D TMA boxes) + 2x2 max pool in the epilogue, incl. partial tiles.
    cin = cout = 128 runs the swapped-operand kernel in 2-CTA clusters: 3 x 9 blocks of
    16x16 is an odd count (one CTA recomputes the last block and stores nothing), 5 x 100
    blocks give every cluster several tiles per accumulator buffer."""
    torch = cuda
    x = _input(torch, n, res, cin, seed=res, dtype=dtype)
    out, ref = _run_conv(torch, x, res, cin, cout, cout, 3, leaky=True, dtype=dtype, pool=True)
    _check(torch, out, ref, rel=2e-2 if dtype == "bf16" else 3e-3)


def test_conv_layer0_expanded_input(cuda):
    """Layer-0 mode: the gather's [res+2][res+6][rgb0] pixels (pixel (v, u) at [v+1][u+2],
    zero halo), read as overlapping 64-byte 8-pixel rows; compact pooled output."""
    torch = cuda
    n, res = 2, 64
    g = torch.Generator(device="cpu").manual_seed(4)
    img = torch.rand(n, res, res, 3, generator=g).half().float()
    ex = torch.zeros(n, res + 2, res + 6, 4)
    ex[:, 1:-1, 2:res + 2, 0:3] = img
    ex = ex.half().cuda()
    w = torch.randn(32, 3, 3, 3, generator=g) * 0.3  # cout, ky, kx, cin
    wpack = torch.from_numpy(yolo.pack_weight(0, w.permute(0, 3, 1, 2).numpy(), "fp16")).half().cuda()
    bias = (torch.randn(32, generator=g) * 0.1).cuda()
    out = torch.zeros(n, res // 2, res // 2, 32, dtype=torch.float16, device="cuda")
    native.call("tp_conv", native.ptr(ex), n, res, 16, native.ptr(wpack), native.ptr(bias), 32,
                32, 3, 1, native.ptr(out), 32, 0, 0, 0, native.DTYPES["fp16"], 1,
                native.stream_handle())
    torch.cuda.synchronize()
    wq = w.permute(0, 3, 1, 2).half().float().cuda()
    ref = torch.nn.functional.conv2d(img.cuda().permute(0, 3, 1, 2), wq, bias, padding=1)
    ref = torch.nn.functional.max_pool2d(torch.where(ref > 0, ref, 0.1 * ref), 2)
    _check(torch, out, ref.permute(0, 2, 3, 1), rel=3e-3)


def test_maxpool(cuda):
    torch = cuda
    x = _input(torch, 3, 16, 64, seed=2)
    out = torch.zeros(3, 8, 8, 64, dtype=torch.bfloat16, device="cuda")
    native.call("tp_maxpool2", native.ptr(x), 3, 16, 64, 0, native.ptr(out), native.stream_handle())
    torch.cuda.synchronize()
    ref = torch.nn.functional.max_pool2d(x.float().permute(0, 3, 1, 2), 2)
    assert torch.equal(out.float(), ref.permute(0, 2, 3, 1))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize(
    "cin,cout,res,pool",
    [(32, 64, 16, False), (64, 128, 24, False), (64, 128, 152, False), (32, 32, 40, False),
     (64, 128, 48, True), (64, 128, 152, True), (64, 256, 16, True),
     (32, 64, 32, True), (32, 64, 48, True), (64, 64, 32, True), (32, 64, 304, True)],
)
def test_conv_box_kernel(cuda, cin, cout, res, pool, dtype, monkeypatch):
    """Full-halo box kernel (one TMA box per 8x16 tile, taps as descriptor row offsets):
    plain, shuffle-pooled and pool-in-M (parity planes) epilogues, several images, partial
    last tile rows; must agree with torch and with the FLAT / RECT kernels (TP_BOX=0)."""
    torch = cuda
    n = 1 if res >= 152 else 3
    x = _input(torch, n, res, cin, seed=res + cin, dtype=dtype)
    out, ref = _run_conv(torch, x, res, cin, cout, cout, 3, leaky=True, dtype=dtype, pool=pool)
    _check(torch, out, ref, rel=2e-2 if dtype == "bf16" else 3e-3)
    monkeypatch.setenv("TP_BOX", "0")
    out0, _ = _run_conv(torch, x, res, cin, cout, cout, 3, leaky=True, dtype=dtype, pool=pool)
    # same fp32 accumulation order is not guaranteed across kernels: compare loosely
    _check(torch, out, out0.float(), rel=1e-2 if dtype == "bf16" else 2e-3)


@pytest.mark.parametrize("cin,cout,k,res,n", [(64, 128, 3, 19, 5), (128, 64, 1, 19, 5),
                                              (512, 1024, 3, 19, 3), (1024, 512, 1, 19, 3),
                                              (256, 512, 3, 38, 2), (128, 256, 3, 76, 1)])
def test_conv_im2col_tiles_cross_images(cuda, cin, cout, k, res, n):
    """FLAT tiles are 128 (or 256, CTA pair) consecutive compact pixels loaded with TMA
    im2col: tiles straddle image rows and image boundaries, taps outside an image must
    read zeros, and the last tile is partial."""
    torch = cuda
    x = _input(torch, n, res, cin, seed=cin * k + res, dtype="fp16")
    out, ref = _run_conv(torch, x, res, cin, cout, cout, k, leaky=True, dtype="fp16")
    _check(torch, out, ref, rel=3e-3)
