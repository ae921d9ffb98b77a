"""CPU restatement of the detector that sits behind the reference's Detector boundary
(TEST INFRASTRUCTURE — never on the product path).

The reference has no network: its Detector (pkg/src/tilepipe/detector.py:77-96) is an
abstract boundary and YOLO v2 is out of scope. The north star asks
for YOLO v2-608 behind that boundary, so this module restates yolov2-608.cfg (the
network PAPER.md:85,120 cites) as a torch-CPU fp32 forward plus a numpy region-layer
decode. "Parity unpinned by any reference test" applies to this file only: it is
pinned by the repo's own golden vectors (seeded weights, rendered synthetic tiles).

Weight format (shared with the GPU path, built by paper_1810_10551_b200/yolo.py):
  per conv (in LAYERS order) a bf16-valued matrix [cout_pad][K], K index = tap*cin + c,
  tap = ky*3 + kx (layer 0: [32][144] = ky x 3 window variants x 4 pixel slots x rgb0,
  variant 0 slots 1..3 = kx 0..2 — see paper_1810_10551_b200/yolo.py), BN folded,
  and a fp32 bias [cout_pad].
Activation precision: mode "bf16"/"fp16" rounds every stored activation to that 16-bit
type exactly like the GPU buffers (fp32 accumulation in between); "fp32" keeps fp32.
"""

from __future__ import annotations

import numpy as np

# (darknet index, cin, cout, ksize, input side); pooling after 0, 2, 6, 10, 16
LAYERS = [
    (0, 3, 32, 3, 608), (2, 32, 64, 3, 304), (4, 64, 128, 3, 152), (5, 128, 64, 1, 152),
    (6, 64, 128, 3, 152), (8, 128, 256, 3, 76), (9, 256, 128, 1, 76), (10, 128, 256, 3, 76),
    (12, 256, 512, 3, 38), (13, 512, 256, 1, 38), (14, 256, 512, 3, 38), (15, 512, 256, 1, 38),
    (16, 256, 512, 3, 38), (18, 512, 1024, 3, 19), (19, 1024, 512, 1, 19),
    (20, 512, 1024, 3, 19), (21, 1024, 512, 1, 19), (22, 512, 1024, 3, 19),
    (23, 1024, 1024, 3, 19), (24, 1024, 1024, 3, 19), (26, 512, 64, 1, 38),
    (29, 1280, 1024, 3, 19), (30, 1024, 425, 1, 19),
]
POOL_AFTER = {0, 2, 6, 10, 16}
ANCHORS = np.array([0.57273, 0.677385, 1.87446, 2.06253, 3.33843, 5.47434, 7.88282, 3.52778,
                    9.77052, 9.16828], dtype=np.float32)
N_CLASSES = 80


def _bf16(t):
    import torch

    return t.to(torch.bfloat16).to(torch.float32)


def _fp16(t):
    import torch

    return t.to(torch.float16).to(torch.float32)


ROUND = {"bf16": _bf16, "fp16": _fp16, "fp32": lambda t: t}


def unpack_weight(wpack, li):
    """[cout_pad][K] packed -> torch [cout][cin][k][k] (fp32)."""
    import torch

    _, cin, cout, k, _ = LAYERS[li]
    w = torch.as_tensor(np.asarray(wpack, dtype=np.float32))
    if li == 0:  # K = dy(3) x variant(3) x slot(4) x [rgb+pad]; variant 0 slots 1,2,3 = dx -1,0,1
        w = w[:cout, :144].reshape(cout, 3, 3, 4, 4)[:, :, 0, [1, 2, 3], :cin].reshape(cout, 9, cin)
    else:
        w = w[:cout, : k * k * cin].reshape(cout, k * k, cin)
    return w.reshape(cout, k, k, cin).permute(0, 3, 1, 2).contiguous()


def tiles_to_input(tiles_u8, mode="bf16"):
    """[n,608,608,3] uint8 -> NCHW fp32 holding x/255 rounded to the GPU's storage type."""
    import torch

    x = torch.as_tensor(np.asarray(tiles_u8)).to(torch.float32) / 255.0
    return ROUND[mode](x).permute(0, 3, 1, 2).contiguous()


def reorg(x):
    """[n,64,38,38] -> [n,256,19,19] exactly as darknet's yolov2-608 [reorg] stride=2 layer:
    forward_reorg_layer calls reorg_cpu(input, w, h, c, batch, stride, forward=0, output)
    (darknet src/reorg_layer.c, src/blas.c), whose loop over the input's (k, j, i) sets
    out[i + w*(j + h*k)] = in[w2 + 2w*(h2 + 2h*c2)] with c2 = k % (c/4), off = k / (c/4),
    w2 = 2i + off % 2, h2 = 2j + off / 2 — i.e. it reads the C x H x W input as
    C/4 x 2H x 2W memory; not a clean space-to-depth. Restated on flat NCHW indices."""
    n, c, h, w = x.shape
    k, j, i = np.meshgrid(np.arange(c), np.arange(h), np.arange(w), indexing="ij")
    out_c = c // 4
    c2, off = k % out_c, k // out_c
    w2, h2 = i * 2 + off % 2, j * 2 + off // 2
    src = (w2 + w * 2 * (h2 + h * 2 * c2)).reshape(-1)  # out[in_index] = x[out_index]
    flat = x.reshape(n, -1)[:, torch_index(src)]
    return flat.reshape(n, 4 * c, h // 2, w // 2)


def torch_index(a):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.long)


def forward(tiles_u8, weights, biases, mode="bf16", threads=None, return_features=False):
    """YOLO v2-608 forward on CPU. Returns the fp32 head [n,19,19,425] (channels last)."""
    import torch
    import torch.nn.functional as F

    if threads:
        torch.set_num_threads(threads)
    rnd = ROUND[mode]
    feats = {}
    with torch.no_grad():
        x = tiles_to_input(tiles_u8, mode)  # fp32: exact v/255, no rounding anywhere

        def conv(li, inp, linear=False):
            _, cin, cout, k, _ = LAYERS[li]
            w = unpack_weight(weights[li], li)
            b = torch.as_tensor(np.asarray(biases[li][:cout], dtype=np.float32))
            y = F.conv2d(inp, w, b, padding=k // 2)
            if not linear:
                y = torch.where(y > 0, y, 0.1 * y)
                y = rnd(y)
            return y

        li = 0
        route16 = None
        for li in range(20):  # darknet layers 0..24
            x = conv(li, x)
            if LAYERS[li][0] == 16:
                route16 = x
            if LAYERS[li][0] in POOL_AFTER:
                x = F.max_pool2d(x, 2)
        l24 = x
        r = reorg(conv(20, route16))
        x = torch.cat([r, l24], dim=1)
        x = conv(21, x)
        if return_features:
            feats["l29"] = x.permute(0, 2, 3, 1).contiguous().numpy()
        head = conv(22, x, linear=True)
    out = head.permute(0, 2, 3, 1).contiguous().numpy().astype(np.float32)
    return (out, feats) if return_features else out


def _sig(x):
    one = np.float32(1.0)
    return (one / (one + np.exp(-x))).astype(np.float32)


def region_decode(head, thresh, max_per_tile=1805):
    """head [n,19,19,425] fp32 -> per tile list of (local_rect, cls, conf) sorted by
    (-conf, cell*5+anchor). Same fp32 op sequence as csrc/tp_detect.cu decode_one."""
    n = head.shape[0]
    out = []
    f32 = np.float32
    rows = np.arange(19, dtype=np.float32)[:, None, None]
    cols = np.arange(19, dtype=np.float32)[None, :, None]
    for t in range(n):
        v = head[t].reshape(19, 19, 5, 85).astype(np.float32)
        obj = _sig(v[..., 4])
        logits = v[..., 5:]
        m = logits.max(axis=-1)
        best = logits.argmax(axis=-1)
        s = np.zeros(m.shape, dtype=np.float32)
        for k in range(N_CLASSES):  # sequential fp32 accumulation, like the kernel
            s = (s + np.exp((logits[..., k] - m).astype(f32))).astype(f32)
        conf = (obj / s).astype(f32)
        cx = ((cols + _sig(v[..., 0])) * f32(32.0)).astype(f32)
        cy = ((rows + _sig(v[..., 1])) * f32(32.0)).astype(f32)
        aw = ANCHORS[0::2][None, None, :]
        ah = ANCHORS[1::2][None, None, :]
        bw = ((aw * np.exp(v[..., 2])).astype(f32) * f32(32.0)).astype(f32)
        bh = ((ah * np.exp(v[..., 3])).astype(f32) * f32(32.0)).astype(f32)
        hw = (bw * f32(0.5)).astype(f32)
        hh = (bh * f32(0.5)).astype(f32)
        x1 = np.maximum(f32(0.0), (cx - hw).astype(f32))
        y1 = np.maximum(f32(0.0), (cy - hh).astype(f32))
        x2 = np.minimum(f32(608.0), (cx + hw).astype(f32))
        y2 = np.minimum(f32(608.0), (cy + hh).astype(f32))
        w = (x2 - x1).astype(f32)
        h = (y2 - y1).astype(f32)
        keep = (conf >= f32(thresh)) & (w > 0) & (h > 0)
        idx = np.nonzero(keep.reshape(-1))[0]
        c = conf.reshape(-1)[idx]
        order = np.lexsort((idx, -c.astype(np.float64)))
        idx = idx[order][:max_per_tile]
        dets = []
        for i in idx:
            dets.append(((float(x1.reshape(-1)[i]), float(y1.reshape(-1)[i]),
                          float(w.reshape(-1)[i]), float(h.reshape(-1)[i])),
                         int(best.reshape(-1)[i]), float(conf.reshape(-1)[i]), int(i)))
        out.append(dets)
    return out
