"""Integer bilinear crop resample (TEST INFRASTRUCTURE — the checker for K1/K2).

The reference only has the nearest-neighbour cutter (detector.py:223-247, restated as
pipeline_ref.cut_tile_nearest). The north star's ingest is a bilinear downscale; this
is its definition, in integer arithmetic so the CUDA kernel can match it bit for bit:

  for output index u in [0, 608):   num = max(0, (2u+1)*side - 608)
                                     s256 = num*256 // 1216      (8 fraction bits)
                                     i0 = s256 >> 8, f = s256 & 255, i1 = min(i0+1, side-1)
  source pixel (crop_x + i, crop_y + j) outside the frame reads as 0 (as in cut_tile)
  out = (p00*(256-fx)*(256-fy) + p01*fx*(256-fy) + p10*(256-fx)*fy + p11*fx*fy + 32768) >> 16
"""

from __future__ import annotations

import numpy as np

S = 608


def taps(side):
    u = np.arange(S, dtype=np.int64)
    num = np.maximum(0, (2 * u + 1) * side - S)
    s256 = (num * 256) // (2 * S)
    i0 = s256 >> 8
    f = s256 & 255
    i1 = np.minimum(i0 + 1, side - 1)
    return i0, i1, f


def _sample(pixels, ys, xs):
    H, W = pixels.shape[:2]
    yok = (ys >= 0) & (ys < H)
    xok = (xs >= 0) & (xs < W)
    v = pixels[np.clip(ys, 0, H - 1)][:, np.clip(xs, 0, W - 1)].astype(np.int64)
    v[~yok] = 0
    v[:, ~xok] = 0
    return v


def cut_tile_bilinear(pixels, x0, y0, side):
    i0, i1, f = taps(side)
    ys0, ys1 = y0 + i0, y0 + i1
    xs0, xs1 = x0 + i0, x0 + i1
    p00 = _sample(pixels, ys0, xs0)
    p01 = _sample(pixels, ys0, xs1)
    p10 = _sample(pixels, ys1, xs0)
    p11 = _sample(pixels, ys1, xs1)
    fx = f[None, :, None]
    fy = f[:, None, None]
    acc = (p00 * (256 - fx) * (256 - fy) + p01 * fx * (256 - fy) + p10 * (256 - fx) * fy
           + p11 * fx * fy + 32768) >> 16
    return acc.astype(np.uint8)
