"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of the library runs at least once at a small size.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--precision fp32]

One 4K dense frame through the engine (GPU render, gather, 23-conv YOLO on stage-1 and
stage-2 tiles, decode + to_global, attention boxes, select, build_jobs, collect,
postprocess), the bilinear gather, a crop-parallel run (slice / unslice) and the
isolated conv entry point on a 19x19 image per kernel family. Prints SANITIZE-OK."""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--skip-conv", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1810_10551_b200 import kernels, native, pipeline as P, synthetic
    from paper_1810_10551_b200.engine import AttentionPipelineB200

    torch.cuda.set_device(0)
    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 1, seed=0))[0]
    frames = synthetic.render_frames_device(W, H, [gt])
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, W, H, max_frames=1, precision=a.precision)
    eng.reset_history(())
    eng.run_device(1, frames=frames)
    (res, att), = eng.results([0])
    print(f"engine: {len(res.detections)} detections, {res.active_count} active crops")
    # bilinear gather into the stage-2 net's input slots
    jobs = kernels.jobs_tensor([(0, 2, 0, 0, 736, 0), (0, 3, 700, 300, 736, 1)])
    kernels.gather(frames, W * H * 3, H, W, jobs, 2, "bilinear", out_act_ptr=eng.net.input_ptr,
                   dtype=eng.dtype)
    # crop-parallel stage 2 (slice / compact exchange / unslice) with world 2 in turn
    ranks = [AttentionPipelineB200(settings, W, H, max_frames=1, net=eng.net,
                                   crop_shard=(r, 2)) for r in range(2)]
    for e in ranks:
        e.reset_history(())
        e.run_local(1, frames=frames)
    dets = torch.cat([e.local_results()[0] for e in ranks])
    counts = torch.cat([e.local_results()[1] for e in ranks])
    for e in ranks:
        e.all_dets.copy_(dets)
        e.all_counts.copy_(counts)
        e.finish_local()
    (res2, _), = ranks[0].results([0])
    assert res2.detections == res.detections
    if not a.skip_conv:  # isolated conv entry point, one small image per kernel family
        rng = np.random.default_rng(0)
        for cin, cout, k, res_, pool in ((32, 64, 3, 16, 1), (64, 128, 3, 16, 0),
                                         (128, 256, 3, 16, 0), (256, 512, 3, 12, 0),
                                         (128, 64, 1, 19, 0), (128, 256, 3, 16, 1)):
            x = torch.from_numpy(rng.standard_normal((1, res_, res_, cin)).astype(np.float16)).cuda()
            w = torch.from_numpy((rng.standard_normal((cout, k * k * cin)) * 0.05).astype(
                np.float16)).cuda()
            b = torch.zeros(cout, dtype=torch.float32, device="cuda")
            r_out = res_ // 2 if pool else res_
            out = torch.zeros((1, r_out, r_out, cout), dtype=torch.float16, device="cuda")
            native.call("tp_conv", native.ptr(x), 1, res_, cin, native.ptr(w), native.ptr(b),
                        cout, cout, k, 1, native.ptr(out), cout, 0, 0, 0, native.DTYPES["fp16"],
                        pool, native.stream_handle())
    torch.cuda.synchronize()
    print("SANITIZE-OK")


if __name__ == "__main__":
    main()
