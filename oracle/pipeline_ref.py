"""CPU restatement of the reference attention-pipeline algorithm (TEST INFRASTRUCTURE).

This module is the parity oracle. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it, and only as the
checker / the timed CPU reference — never as part of the product path.

It restates, on plain tuples (rect = (x, y, w, h)), the reference functions of
``/root/reference/pkg/src/tilepipe``:

  geometry.py:151-164  crop_side_px         -> crop_side
  geometry.py:167-184  _axis_positions      -> axis_positions
  geometry.py:187-215  build_grid           -> build_grid
  geometry.py:218-234  to_local             -> to_local
  geometry.py:237-256  to_global            -> to_global
  geometry.py:80-91    intersects / iou     -> intersects / iou
  detector.py:223-247  cut_tile             -> cut_tile_nearest
  detector.py:99-135   mock_detect          -> mock_detect (scene-oracle detector fixture)
  pipeline.py:297-316  attention_pass       -> attention_pass
  pipeline.py:319-338  merge_temporal       -> merge_temporal
  pipeline.py:341-354  select_active        -> select_active
  pipeline.py:357-375  final_pass           -> final_pass
  pipeline.py:378-426  finish/evaluate      -> evaluate_frame, run_sequence
  pipeline.py:460-530  baselines            -> run_allcrops_baseline, run_downscale_baseline
  postprocess.py:54-73 nms_keep_indices     -> nms_keep_indices
  postprocess.py:81-163 merge_split         -> merge_split
  postprocess.py:166-187 postprocess        -> postprocess

It is pinned against golden vectors produced by running the reference itself
(tests/golden/make_golden.py) — see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

MODEL_SIDE = 608

# ----------------------------------------------------------------- geometry


def rect_ok(r):
    x, y, w, h = r
    return all(math.isfinite(v) for v in r) and w > 0 and h > 0


def x2(r):
    return r[0] + r[2]


def y2(r):
    return r[1] + r[3]


def area(r):
    return r[2] * r[3]


def intersection(a, b):
    lx, ly = max(a[0], b[0]), max(a[1], b[1])
    hx, hy = min(x2(a), x2(b)), min(y2(a), y2(b))
    if hx <= lx or hy <= ly:
        return None
    return (lx, ly, hx - lx, hy - ly)


def union_rect(a, b):
    lx, ly = min(a[0], b[0]), min(a[1], b[1])
    hx, hy = max(x2(a), x2(b)), max(y2(a), y2(b))
    return (lx, ly, hx - lx, hy - ly)


def dilated(r, margin, fw, fh):
    lx = max(0.0, r[0] - margin)
    ly = max(0.0, r[1] - margin)
    hx = min(float(fw), x2(r) + margin)
    hy = min(float(fh), y2(r) + margin)
    return (lx, ly, hx - lx, hy - ly)


def intersects(a, b):
    return min(x2(a), x2(b)) > max(a[0], b[0]) and min(y2(a), y2(b)) > max(a[1], b[1])


def iou(a, b):
    i = intersection(a, b)
    if i is None:
        return 0.0
    ia = area(i)
    return ia / (area(a) + area(b) - ia)


def crop_side(frame_h, rows, overlap):
    span = MODEL_SIDE * rows - overlap * (rows - 1)
    side = int(Fraction(frame_h * MODEL_SIDE, span) + Fraction(1, 2))
    return max(side, -(-frame_h // rows))


def axis_positions(extent, side, overlap, count):
    stride_numer = (MODEL_SIDE - overlap) * side
    last = max(0, extent - side)
    pos = []
    for i in range(count - 1):
        p = (i * stride_numer) // MODEL_SIDE
        p = max(p, extent - (count - i) * side, 0)
        pos.append(min(p, last))
    pos.append(last)
    return pos


def build_grid(frame_w, frame_h, rows, overlap, id_base=0):
    """Returns (side, rows, cols, crops) with crops = [(id, row, col, x, y, side, scale)]."""
    side = crop_side(frame_h, rows, overlap)
    numer = frame_w * MODEL_SIDE - overlap * side
    denom = (MODEL_SIDE - overlap) * side
    cols = max(1, -(-numer // denom))
    xs = axis_positions(frame_w, side, overlap, cols)
    ys = axis_positions(frame_h, side, overlap, rows)
    crops = []
    cid = id_base
    for r, y in enumerate(ys):
        for c, x in enumerate(xs):
            crops.append((cid, r, c, x, y, side, side / MODEL_SIDE))
            cid += 1
    return side, rows, cols, crops


def crop_rect(crop):
    return (crop[3], crop[4], crop[5], crop[5])


def to_local(r, crop):
    g = crop_rect(crop)
    inter = intersection(r, g)
    if inter is None:
        raise ValueError("no intersection")
    s = crop[6]
    lx1 = max(0.0, (inter[0] - g[0]) / s)
    ly1 = max(0.0, (inter[1] - g[1]) / s)
    lx2 = min(float(MODEL_SIDE), (x2(inter) - g[0]) / s)
    ly2 = min(float(MODEL_SIDE), (y2(inter) - g[1]) / s)
    return (lx1, ly1, lx2 - lx1, ly2 - ly1)


def to_global(r, crop, fw=None, fh=None):
    g = crop_rect(crop)
    s = crop[6]
    a1 = g[0] + r[0] * s
    b1 = g[1] + r[1] * s
    a2 = g[0] + x2(r) * s
    b2 = g[1] + y2(r) * s
    if fw is not None:
        a1, a2 = min(a1, fw - 1), min(a2, fw)
        b1, b2 = min(b1, fh - 1), min(b2, fh)
        a1, b1 = max(0.0, a1), max(0.0, b1)
    i1, j1 = round(a1), round(b1)
    i2, j2 = max(i1 + 1, round(a2)), max(j1 + 1, round(b2))
    return (i1, j1, i2 - i1, j2 - j1)


# ----------------------------------------------------------------- plan


class Plan:
    """Unified crop-id space (pipeline.py:209-269): attention, final, downscale."""

    def __init__(self, fw, fh, att_rows, fin_rows, overlap, fin_overlap=None):
        self.fw, self.fh = fw, fh
        fo = overlap if fin_overlap is None else fin_overlap
        self.att = build_grid(fw, fh, att_rows, overlap)
        self.fin = build_grid(fw, fh, fin_rows, fo, id_base=len(self.att[3]))
        side = max(fw, fh)
        self.down = (len(self.att[3]) + len(self.fin[3]), 0, 0, 0, 0, side, side / MODEL_SIDE)
        self.by_id = {c[0]: c for c in self.att[3] + self.fin[3]}
        self.by_id[self.down[0]] = self.down


# ----------------------------------------------------------------- tiles


def cut_tile_nearest(pixels, crop, input_side=MODEL_SIDE):
    H, W = pixels.shape[:2]
    side, x0, y0 = int(crop[5]), int(crop[3]), int(crop[4])
    src = (np.arange(input_side, dtype=np.int64) * side) // input_side
    xs, ys = x0 + src, y0 + src
    xok = (xs >= 0) & (xs < W)
    yok = (ys >= 0) & (ys < H)
    t = pixels[np.clip(ys, 0, H - 1)][:, np.clip(xs, 0, W - 1)].copy()
    t[~yok] = 0
    t[:, ~xok] = 0
    return t


# ----------------------------------------------------------------- detector fixture


def mock_detect(crop, gt, visibility=0.3, min_tile_px=8):
    """gt: [(rect, label)]; returns [(local_rect, label, conf)] sorted by -conf (stable)."""
    side = crop[5]
    g = crop_rect(crop)
    out = []
    for rect, label in gt:
        vis = intersection(rect, g)
        if vis is None:
            continue
        frac = area(vis) / area(rect)
        if frac < visibility:
            continue
        if min_tile_px > 0 and (vis[2] * MODEL_SIDE < min_tile_px * side or
                                vis[3] * MODEL_SIDE < min_tile_px * side):
            continue
        out.append((to_local(vis, crop), label, frac))
    out.sort(key=lambda d: -d[2])
    return out


# ----------------------------------------------------------------- stages


def attention_pass(plan, frame_id, detect, min_conf):
    """detect(frame_id, crop) -> [(local_rect, label, conf)] in detector order."""
    boxes = []
    for crop in plan.att[3]:
        for rect, label, conf in detect(frame_id, crop):
            if conf >= min_conf:
                boxes.append(to_global(rect, crop, plan.fw, plan.fh))
    return boxes


def merge_temporal(history_boxes, window):
    """history_boxes: list of box lists, oldest first; returns first-seen union."""
    out, seen = [], set()
    for boxes in history_boxes[-window:]:
        for b in boxes:
            if b not in seen:
                seen.add(b)
                out.append(b)
    return out


def select_active(fin_grid, boxes, margin, fw, fh):
    dil = [dilated(b, margin, fw, fh) for b in boxes]
    return sorted(c[0] for c in fin_grid[3] if any(intersects(crop_rect(c), d) for d in dil))


def final_pass(plan, frame_id, active_ids, detect):
    out = []
    for cid in sorted(active_ids):
        crop = plan.by_id[cid]
        for rect, label, conf in detect(frame_id, crop):
            out.append((cid, (to_global(rect, crop, plan.fw, plan.fh), label, conf)))
    return out


# ----------------------------------------------------------------- postprocess


def nms_keep_indices(dets, thr):
    """dets: [(rect, label, conf)]."""
    order = sorted(range(len(dets)), key=lambda i: (-dets[i][2], i))
    kept = []
    for i in order:
        ok = True
        for k in kept:
            if dets[k][1] == dets[i][1] and not (iou(dets[k][0], dets[i][0]) < thr):
                ok = False
                break
        if ok:
            kept.append(i)
    return kept


def _gap(lo1, hi1, lo2, hi2):
    return max(lo1, lo2) - min(hi1, hi2)


def _adjacent(ca, cb, vertical):
    dr, dc = (1, 0) if vertical else (0, 1)
    return any((r + dr, c + dc) in cb or (r - dr, c - dc) in cb for r, c in ca)


def _can_merge(a, ca, b, cb, rules, gap, tol):
    if a[1] != b[1]:
        return False
    rule = rules.get(a[1])
    if rule is None:
        return False
    ra, rb = a[0], b[0]
    if rule in ("vertical", "both") and _adjacent(ca, cb, True):
        if (_gap(ra[1], y2(ra), rb[1], y2(rb)) <= gap and abs(ra[0] - rb[0]) <= tol
                and abs(x2(ra) - x2(rb)) <= tol):
            return True
    if rule in ("horizontal", "both") and _adjacent(ca, cb, False):
        if (_gap(ra[0], x2(ra), rb[0], x2(rb)) <= gap and abs(ra[1] - rb[1]) <= tol
                and abs(y2(ra) - y2(rb)) <= tol):
            return True
    return False


def merge_split(tagged, cell_of, rules, gap=40, tol=30):
    """tagged: [(crop_id, det)], cell_of: crop_id -> (row, col)."""
    entries = [(frozenset({cell_of[cid]}), d) for cid, d in tagged]
    changed = True
    while changed:
        changed = False
        n = len(entries)
        for i in range(n):
            for j in range(i + 1, n):
                ci, di = entries[i]
                cj, dj = entries[j]
                if _can_merge(di, ci, dj, cj, rules, gap, tol):
                    entries[i] = (ci | cj, (union_rect(di[0], dj[0]), di[1], max(di[2], dj[2])))
                    del entries[j]
                    changed = True
                    break
            if changed:
                break
    return [d for _, d in entries]


def postprocess(tagged, cell_of, nms_iou=0.45, rules=None, gap=40, tol=30,
                merge_before_nms=False, nms_per_crop=False):
    rules = {"person": "vertical"} if rules is None else rules
    if nms_per_crop:
        groups = {}
        for idx, (cid, _) in enumerate(tagged):
            groups.setdefault(cid, []).append(idx)
        kept = []
        for cid, idxs in groups.items():
            ds = [tagged[i][1] for i in idxs]
            kept.extend((cid, ds[k]) for k in nms_keep_indices(ds, nms_iou))
        return merge_split(kept, cell_of, rules, gap, tol)
    if merge_before_nms:
        merged = merge_split(tagged, cell_of, rules, gap, tol)
        return [merged[i] for i in nms_keep_indices(merged, nms_iou)]
    keep = nms_keep_indices([d for _, d in tagged], nms_iou)
    return merge_split([tagged[i] for i in keep], cell_of, rules, gap, tol)


def finish(tagged, cell_of, min_conf, **policy):
    return [d for d in postprocess(tagged, cell_of, **policy) if d[2] >= min_conf]


# ----------------------------------------------------------------- orchestration


def cell_map(plan):
    out = {c[0]: (c[1], c[2]) for c in plan.fin[3]}
    out[plan.down[0]] = (0, 0)
    return out


def evaluate_frame(plan, frame_id, detect, history, window=2, margin=20, min_conf=0.3,
                   **policy):
    """Returns (dets, active_ids, att_boxes, merged_boxes)."""
    att = attention_pass(plan, frame_id, detect, min_conf)
    merged = merge_temporal([*history, att], window)
    active = select_active(plan.fin, merged, margin, plan.fw, plan.fh)
    tagged = final_pass(plan, frame_id, active, detect)
    dets = finish(tagged, cell_map(plan), min_conf, **policy)
    return dets, active, att, merged


def run_sequence(plan, frame_ids, detect, window=2, margin=20, min_conf=0.3, **policy):
    hist = []
    out = []
    for fid in frame_ids:
        dets, active, att, merged = evaluate_frame(plan, fid, detect, hist, window, margin,
                                                   min_conf, **policy)
        hist.append(att)
        del hist[: max(0, len(hist) - (window - 1))]
        out.append((fid, dets, active))
    return out


def run_allcrops_baseline(plan, frame_id, detect, min_conf=0.3, **policy):
    ids = [c[0] for c in plan.fin[3]]
    tagged = final_pass(plan, frame_id, ids, detect)
    return finish(tagged, cell_map(plan), min_conf, **policy)


def run_downscale_baseline(plan, frame_id, detect, min_conf=0.3, **policy):
    crop = plan.down
    tagged = [(crop[0], (to_global(r, crop, plan.fw, plan.fh), lab, conf))
              for r, lab, conf in detect(frame_id, crop)]
    return finish(tagged, {crop[0]: (0, 0)}, min_conf, **policy)
