"""tp_postprocess (K7: per-class greedy NMS + split merge + min_conf) at stress sizes.

    python tests/tools/post_bench.py [--frames 30] [--n 400 1000 2000] [--reps 20]

One launch handles --frames frames of n raw detections each (one CTA per frame, as in the
engine's batched step). Reports the CUDA-event time per launch, per frame, the bytes the
kernel must move (n x 56-byte tp_pdet_t records read + kept records written) and the
achieved GB/s against the measured HBM peak. The CPU reference time of one frame
(oracle restatement of postprocess.py, one host thread) is printed beside it. JSON lines.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--n", type=int, nargs="+", default=[400, 1000, 2000])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu", action="store_true", help="also time the CPU reference")
    a = ap.parse_args()
    import torch

    from oracle import e2e as E
    from oracle import pipeline_ref as R
    from paper_1810_10551_b200 import native
    from paper_1810_10551_b200.engine import MAX_PER_FRAME
    from paper_1810_10551_b200.postprocess import LabelTable, MergePolicy, ctypes_ref, \
        make_policy_struct

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.8) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.8
    W, H = 3840, 2160
    plan = R.Plan(W, H, 1, 3, 20)
    cells = R.cell_map(plan)
    labels = LabelTable(["person", "car"])
    pol = make_policy_struct(MergePolicy(), labels, 6, 18, min_conf=0.3)
    rec_b = native.PDET_DTYPE.itemsize
    for n in a.n:
        B = a.frames
        recs = np.zeros((B, MAX_PER_FRAME), dtype=native.PDET_DTYPE)
        raws = []
        for f in range(B):
            raw = E.synthetic_raw_detections(plan, n, seed=1000 * n + f)
            raws.append(raw)
            for i, (cid, (r, lab, conf)) in enumerate(raw):
                row, col = cells[cid]
                recs[f, i] = (r[0], r[1], r[2], r[3], conf, labels.id(lab), row * 6 + col, cid, i)
        dev_in = torch.from_numpy(recs.view(np.uint8).reshape(-1)).cuda()
        counts = torch.full((B,), n, dtype=torch.int32, device="cuda")
        dev_out = torch.empty_like(dev_in)
        out_counts = torch.zeros(B, dtype=torch.int32, device="cuda")

        def launch():
            native.call("tp_postprocess", native.ptr(dev_in), native.ptr(counts), B,
                        MAX_PER_FRAME, ctypes_ref(pol), native.ptr(dev_out),
                        native.ptr(out_counts), None, None, native.stream_handle())
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        kept = out_counts.cpu().numpy()
        # parity on frame 0 (bit-exact keep list / merged records vs the CPU restatement)
        want = R.finish(raws[0], cells, 0.3)
        got_rec = dev_out[: MAX_PER_FRAME * rec_b].cpu().numpy().view(native.PDET_DTYPE)[: kept[0]]
        got = [((int(r["x"]), int(r["y"]), int(r["w"]), int(r["h"])), labels.names[int(r["cls"])],
                float(r["conf"])) for r in got_rec]
        line = {"n_raw_per_frame": n, "frames_per_launch": B, "ms_per_launch": ms,
                "us_per_frame": 1e3 * ms / B, "kept_per_frame": float(kept.mean()),
                "bytes_per_launch": int(B * n * rec_b + kept.sum() * rec_b),
                "parity_frame0": got == want}
        line["achieved_GBps"] = line["bytes_per_launch"] / (ms / 1e3) / 1e9
        line["hbm_frac"] = line["achieved_GBps"] / peak
        if a.cpu:
            t0 = time.perf_counter()
            R.finish(raws[0], cells, 0.3)
            line["cpu_reference_ms_per_frame"] = 1e3 * (time.perf_counter() - t0)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
