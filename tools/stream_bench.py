"""Throughput of the §8f paths: run_stream over in-memory frames and over a PPM directory.

    python tools/stream_bench.py [--frames 96] [--batch 16] [--dir /tmp/tp_frames]

Renders a synthetic 4K clip (GPU renderer, copied to host), writes it as frame_%06d.ppm,
then times (wall clock, after one warm-up pass) run_stream(frames) and
run_stream(FrameSource.open(dir)) — host staging / disk reads overlapped with the GPU.
Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1810_10551_b200 import pipeline as P, synthetic  # noqa: E402
from paper_1810_10551_b200.frameio import FrameSource, frame_file_name, write_ppm  # noqa: E402
from paper_1810_10551_b200.stream import run_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=96)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--dir", default="/tmp/tp_stream_frames")
    ap.add_argument("--io-threads", type=int, default=8)
    a = ap.parse_args()
    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("mixed", W, H, a.frames, seed=0))
    dev = torch.empty((a.frames, H, W, 3), dtype=torch.uint8, device="cuda")
    for i in range(0, a.frames, 16):
        synthetic.render_frames_device(W, H, [gt[k] for k in range(i, min(i + 16, a.frames))],
                                       out=dev[i:i + 16])
    host = dev.cpu().numpy()
    frames = [P.Frame(i, W, H, host[i]) for i in range(a.frames)]
    os.makedirs(a.dir, exist_ok=True)
    for f in frames:
        write_ppm(os.path.join(a.dir, frame_file_name(f.frame_id)), f.pixels)
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    out = {"workload": f"{a.frames} synthetic 4K frames, batch {a.batch}, "
                       f"{a.io_threads} host threads ({os.cpu_count()} cores)"}
    for name, src in (("memory", frames), ("ppm_dir", None)):
        s = FrameSource.open(a.dir) if src is None else src
        run_stream(s if src is None else frames[: 2 * a.batch], settings, batch=a.batch,
                   io_threads=a.io_threads)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_stream(s, settings, batch=a.batch, io_threads=a.io_threads)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"frames_per_s": len(res) / dt, "frames": len(res)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
