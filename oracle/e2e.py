"""End-to-end parity helpers: the CPU reference pipeline with the CPU YOLO detector, and
the frame-level comparison against the GPU's FrameResults (TEST INFRASTRUCTURE —
imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs).

The CPU side is the oracle restatement of the reference pipeline (pipeline_ref: the
reference's pipeline.py:297-457 on tuples, pinned to reference goldens) with
oracle/yolo_ref's fp32 YOLO v2-608 + region decode as the detector
(detector.py:77-96 contract). The comparison implements the north-star contract:
  * crop-index selection and the NMS/merge keep-set must be identical;
  * boxes and scores within 1e-3 relative;
and accounts for the only legitimate differences, each counted and reported:
  * threshold-edge flips: a raw detection whose score lies within EDGE of a threshold
    (detector 0.25, min_confidence 0.3) may exist on one side only;
  * rounding-edge flips: an integer global coordinate (to_global's half-even rounding,
    geometry.py:237-256) may differ by 1 px when the exact value lies within ROUND_EDGE
    of a .5 boundary.
A frame whose inputs contain no such edge case must match exactly.
"""

from __future__ import annotations

import math

import numpy as np

from . import pipeline_ref as R
from . import yolo_ref

EDGE = 2e-3        # |score - threshold| below which a detection may flip sides
ROUND_EDGE = 0.02  # |frac(x) - 0.5| below which to_global's rounding may flip (px)
SCORE_REL = 1e-3   # north-star score tolerance


class CpuYolo:
    """detect(frame_id, crop) for pipeline_ref: cut_tile (nearest) + fp32 YOLO + decode,
    memoised per (frame, crop). `raw[(fid, crop_id)]` keeps the local detections."""

    def __init__(self, pixels_of, names, threshold=0.25, seed=0, threads=None):
        from paper_1810_10551_b200 import yolo  # weights generator (shared with the GPU)

        self.pixels_of = pixels_of
        self.names = names
        self.threshold = threshold
        self.wp, self.bs = yolo.make_weights(seed, dtype="fp16")
        self.threads = threads
        self.raw = {}
        self.tiles = {}

    def prefetch(self, fid, crops):
        """Batch the forward of several crops of one frame (faster on many cores)."""
        todo = [c for c in crops if (fid, c[0]) not in self.raw]
        if not todo:
            return
        px = self.pixels_of(fid)
        tiles = np.stack([R.cut_tile_nearest(px, c) for c in todo])
        head = yolo_ref.forward(tiles, self.wp, self.bs, mode="fp32", threads=self.threads)
        for c, t, dets in zip(todo, tiles, yolo_ref.region_decode(head, self.threshold)):
            self.tiles[(fid, c[0])] = t
            self.raw[(fid, c[0])] = [(r, self.names[k], conf) for r, k, conf, _ in dets]

    def __call__(self, fid, crop):
        if (fid, crop[0]) not in self.raw:
            self.prefetch(fid, [crop])
        return self.raw[(fid, crop[0])]


def reference_frame(plan, fid, det, history, window=2, margin=20, min_conf=0.3, **policy):
    """pipeline_ref.evaluate_frame with stage-2 prefetch (same result, batched forward)."""
    det.prefetch(fid, plan.att[3])
    att = R.attention_pass(plan, fid, det, min_conf)
    merged = R.merge_temporal([*history, att], window)
    active = R.select_active(plan.fin, merged, margin, plan.fw, plan.fh)
    det.prefetch(fid, [plan.by_id[c] for c in active])
    tagged = R.final_pass(plan, fid, active, det)
    dets = R.finish(tagged, R.cell_map(plan), min_conf, **policy)
    return dets, active, att


def edge_detections(det, fids, thresholds=(0.25, 0.3)):
    """Raw CPU detections of these frames whose score is within EDGE of a threshold."""
    out = []
    for (fid, cid), dets in det.raw.items():
        if fid not in fids:
            continue
        for r, lab, conf in dets:
            if any(abs(conf - t) < EDGE for t in thresholds):
                out.append((fid, cid, lab, conf))
    return out


def _rounding_edge(v):
    return abs((v - math.floor(v)) - 0.5) < ROUND_EDGE


def rounding_edges(plan, det, fids):
    """Raw CPU detections whose exact global coordinates sit on a rounding edge."""
    out = []
    for (fid, cid), dets in det.raw.items():
        if fid not in fids:
            continue
        crop = plan.by_id[cid]
        s = float(crop[6])
        for r, lab, conf in dets:
            xs = (crop[3] + r[0] * s, crop[4] + r[1] * s, crop[3] + (r[0] + r[2]) * s,
                  crop[4] + (r[1] + r[3]) * s)
            if any(_rounding_edge(v) for v in xs):
                out.append((fid, cid, lab, conf))
    return out


def compare_boxes(ref_boxes, gpu_boxes):
    """Attention box lists (int rects). Returns (exact, n_1px) — n_1px = boxes equal up
    to a 1-px rounding flip; exact False if anything else differs. The list order is
    crop-id order, then the detector's descending confidence (pipeline.py:297-316); two
    boxes of near-equal confidence may swap places (a score-tolerance order flip, as in
    compare_dets), which changes nothing downstream (merge_temporal dedups and
    select_active tests every box), so a positional mismatch falls back to matching the
    two lists as multisets."""
    if len(ref_boxes) != len(gpu_boxes):
        return False, 0
    n1 = 0
    for a, b in zip(ref_boxes, gpu_boxes):
        d = max(abs(p - q) for p, q in zip(a, b))
        if d > 1:
            break
        n1 += d == 1
    else:
        return True, n1
    free, n1 = list(gpu_boxes), 0
    for a in ref_boxes:
        cand = [(max(abs(p - q) for p, q in zip(a, b)), k) for k, b in enumerate(free)]
        d, k = min(cand)
        if d > 1:
            return False, n1
        n1 += d == 1
        free.pop(k)
    return True, n1


def compare_dets(ref_dets, gpu_dets):
    """Final detection lists [(rect, label, conf)] in output (keep) order.

    The keep-SET must be identical: every detection pairs with one of the other side of
    the same label, integer rect within 1 px (rounding edge) and score within SCORE_REL.
    The output order is the NMS order (-conf, index) (postprocess.py:54-73), so two
    kept detections whose scores differ by less than the score tolerance may swap
    places: counted as order flips.
    Returns dict(ok, n, n_1px, score_rel, order_flips[, first_diff])."""
    res = {"ok": len(ref_dets) == len(gpu_dets), "n": len(ref_dets), "n_1px": 0,
           "score_rel": 0.0, "order_flips": 0}
    if not res["ok"]:
        res["first_diff"] = ("lengths", len(ref_dets), len(gpu_dets))
        return res
    free = list(range(len(gpu_dets)))
    for i, (ra, la, ca) in enumerate(ref_dets):
        best = None
        for k in free:
            rb, lb, cb = gpu_dets[k]
            if lb != la:
                continue
            d = max(abs(p - q) for p, q in zip(ra, rb))
            rel = abs(ca - cb) / max(ca, 1e-12)
            if d <= 1 and rel <= SCORE_REL and (best is None or (d, rel) < best[1:]):
                best = (k, d, rel)
        if best is None:
            res["ok"] = False
            res["first_diff"] = ("unmatched", (ra, la, ca))
            return res
        k, d, rel = best
        free.remove(k)
        res["n_1px"] += d == 1
        res["score_rel"] = max(res["score_rel"], rel)
        if k != i:
            res["order_flips"] += 1
            ck = gpu_dets[i][2]
            # a swap is only legitimate between near-equal scores
            if abs(ck - ca) / max(ca, 1e-12) > 2 * SCORE_REL:
                res["ok"] = False
                res["first_diff"] = ("order", i, (ra, la, ca), gpu_dets[i])
                return res
    return res


def synthetic_raw_detections(plan, n, seed=0, labels=("person", "car")):
    """n raw stage-2 detections for one frame of `plan` shaped like the detector's output:
    clusters of jittered boxes around objects (so NMS suppresses and the split-merge rule
    fires across crop borders), each tagged with a final crop that contains its centre.
    Returns [(crop_id, (rect int tuple, label, conf))] in crop order — final_pass order."""
    rng = np.random.default_rng(seed)
    fw, fh = plan.fw, plan.fh
    fin = plan.fin[3]
    n_obj = max(1, n // 8)
    objs = []
    for _ in range(n_obj):
        w = int(rng.integers(40, 260))
        h = int(rng.integers(40, 360))
        objs.append((int(rng.integers(0, fw - w)), int(rng.integers(0, fh - h)), w, h,
                     labels[int(rng.integers(0, len(labels)))]))
    out = []
    for k in range(n):
        x, y, w, h, lab = objs[k % n_obj]
        jx, jy = rng.normal(0, 0.06 * w), rng.normal(0, 0.06 * h)
        sw, sh = rng.uniform(0.8, 1.2), rng.uniform(0.8, 1.2)
        x1 = int(min(max(0, x + jx), fw - 2))
        y1 = int(min(max(0, y + jy), fh - 2))
        ww = int(max(1, min(fw - x1, w * sw)))
        hh = int(max(1, min(fh - y1, h * sh)))
        cx, cy = x1 + ww / 2, y1 + hh / 2
        crops = [c for c in fin if c[3] <= cx < c[3] + c[5] and c[4] <= cy < c[4] + c[5]]
        crop = crops[int(rng.integers(0, len(crops)))]
        conf = float(np.float32(rng.uniform(0.25, 1.0)))
        out.append((crop[0], ((x1, y1, ww, hh), lab, conf)))
    out.sort(key=lambda t: t[0])  # final_pass: ascending crop id, detector order inside
    return out
