"""Per-step CUDA-event timing of the YOLO v2 forward (warm, back-to-back launches).

    python tools/layer_times.py [--tiles 120] [--dtype fp16]

Prints each step's time, achieved TFLOP/s (algorithmic FLOPs) and effective GB/s of
its compulsory traffic (input read once + output written once).
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1810_10551_b200 import yolo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=120)
    ap.add_argument("--dtype", default=yolo.DEFAULT_PRECISION)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--unfused", action="store_true", help="layer 5 as its own launch")
    a = ap.parse_args()
    net = yolo.YoloNet(a.tiles, dtype=a.dtype)
    if a.unfused:
        net.set_fused(False)
    x = net.input_tensor(a.tiles)
    x[:, 1:-1, 1:-1, :] = torch.rand_like(x[:, 1:-1, 1:-1, :].float()).to(x.dtype)
    net.forward(a.tiles)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(yolo.STEPS) + 1)]
    times = [0.0] * len(yolo.STEPS)
    for _ in range(a.reps):
        for s in range(len(yolo.STEPS)):
            ev[s].record()
            net.forward_range(a.tiles, s, s)
        ev[-1].record()
        torch.cuda.synchronize()
        for s in range(len(yolo.STEPS)):
            times[s] += ev[s].elapsed_time(ev[s + 1]) / a.reps
    total = sum(times)
    li = -1
    print(f"{'step':>4} {'layer':>5} {'ms':>8} {'share':>6} {'TFLOP/s':>8}")
    for s, (kind, slot) in enumerate(yolo.STEPS):
        if kind == "conv":
            li += 1
            d, cin, cout, k, side = yolo.LAYERS[li]
            fl = 2.0 * side * side * cout * cin * k * k * a.tiles
            if s in net.fused_steps:  # ran inside the previous step's kernel
                print(f"{s:4d} {d:5d}    fused into step {s - 1}")
                continue
            print(f"{s:4d} {d:5d} {times[s]:8.3f} {100 * times[s] / total:5.1f}% "
                  f"{fl / times[s] / 1e9:8.1f}")
        else:
            print(f"{s:4d}  pool {times[s]:8.3f} {100 * times[s] / total:5.1f}%")
    fl = yolo.GFLOP_PER_TILE * 1e9 * a.tiles
    print(f"total {total:.3f} ms for {a.tiles} tiles: {fl / total / 1e9:.1f} TFLOP/s, "
          f"{total / a.tiles * 1e3:.1f} us/tile")


if __name__ == "__main__":
    main()
