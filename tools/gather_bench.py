"""Warm bandwidth of the crop gather (K1/K2) against the measured HBM peak.

    python tools/gather_bench.py [--frames 30] [--mode nearest] [--dtype fp32]

Cuts every final-grid crop (736-px squares at 4K P1; --grid attention: the 2160-px
stage-1 squares) of `--frames` synthetic 4K frames into the YOLO input, back to back,
timed with CUDA events. Two byte counts per launch:
  * algorithmic: read 3*min(side,608)^2 (nearest) or 3*min(side,1216)^2
    (bilinear) + write 608^2 * 3 * 2 B (16-bit rgb) per tile;
  * delivered: the 8-byte rgb0 pixels actually written (608^2 * 8 B per tile) + the
    source rows' bytes at 32-byte sector granularity (what DRAM must deliver);
each printed as GB/s and as a fraction of MEASURED_PEAKS.json hbm_gbs.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_10551_b200 import kernels, pipeline as P, yolo  # noqa: E402
from paper_1810_10551_b200.pipeline_types import GridPlan  # noqa: E402


def read_bytes(jobs, W, H, nearest=True):
    """DRAM bytes the source rows need, at 32-byte sector granularity."""
    total = 0
    for (_, _, x, y, side, _) in jobs:
        v = np.arange(608)
        if nearest:
            rows = np.unique(y + (v * side) // 608)
            cols = x + (np.arange(608) * side) // 608
        else:
            rows = np.unique(np.concatenate([y + (v * side) // 608, y + (v * side) // 608 + 1]))
            cols = np.concatenate([x + (np.arange(608) * side) // 608,
                                   x + (np.arange(608) * side) // 608 + 1])
        rows = rows[(rows >= 0) & (rows < H)]
        cols = cols[(cols >= 0) & (cols < W)]
        if len(rows) == 0 or len(cols) == 0:
            continue
        row_base = rows.astype(np.int64) * W * 3
        byte_idx = (row_base[:, None] + 3 * cols[None, :].astype(np.int64))
        sectors = np.unique(np.concatenate([byte_idx // 32, (byte_idx + 2) // 32], axis=None))
        total += len(sectors) * 32
    return total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--mode", default="nearest", choices=["nearest", "bilinear"])
    ap.add_argument("--dtype", default=yolo.DEFAULT_PRECISION)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", default="final", choices=["final", "attention"],
                    help="crop set: the final grid (~736 px squares at 4K) or the attention "
                         "grid (2160 px squares: the stage-1 downscale)")
    a = ap.parse_args()
    W, H = 3840, 2160
    plan = GridPlan.build(W, H, P.PipelineSettings.from_preset("1 att, 3 fin, 20 over"))
    jobs = [(f, c.crop_id, int(c.global_rect.x), int(c.global_rect.y), int(c.global_rect.w), 0)
            for f in range(a.frames)
            for c in (plan.final_grid if a.grid == "final" else plan.attention_grid).crops]
    n = len(jobs)
    frames = torch.randint(0, 256, (a.frames, H, W, 3), dtype=torch.uint8, device="cuda")
    net = yolo.YoloNet(n, dtype=a.dtype)
    jt = kernels.jobs_tensor(jobs)
    for _ in range(3):
        kernels.gather(frames, H * W * 3, H, W, jt, n, a.mode, out_act_ptr=net.input_ptr,
                       dtype=a.dtype)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        kernels.gather(frames, H * W * 3, H, W, jt, n, a.mode, out_act_ptr=net.input_ptr,
                       dtype=a.dtype)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    wr = n * 608 * 608 * 8
    rd = read_bytes(jobs, W, H, a.mode == "nearest")
    lim = 608 if a.mode == "nearest" else 1216
    alg = sum(3 * min(j[4], lim) ** 2 + 608 * 608 * 6 for j in jobs)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    gbs = (wr + rd) / ms / 1e6
    alg_gbs = alg / ms / 1e6
    print(json.dumps({"tiles": n, "grid": a.grid, "side": jobs[0][4], "mode": a.mode, "ms": ms,
                      "write_MB": wr / 1e6, "read_MB": rd / 1e6, "GB_per_s": gbs,
                      "frac": gbs / peak, "algorithmic_MB": alg / 1e6,
                      "algorithmic_GB_per_s": alg_gbs, "algorithmic_frac": alg_gbs / peak,
                      "hbm_peak_GB_per_s": peak}))


if __name__ == "__main__":
    main()
