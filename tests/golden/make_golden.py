"""Generate golden vectors by running the REAL reference (`tilepipe`) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json. The reference is not available on the GPU
box; tests read only the committed JSON. Every case records inputs and the
reference's outputs for a hot-path function.
"""

import hashlib
import json
import os
import random

import numpy as np

from tilepipe import geometry as G
from tilepipe import pipeline as P
from tilepipe import postprocess as PP
from tilepipe import synthetic as SY
from tilepipe.detector import Detection, cut_tile

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def rect(r):
    return [r.x, r.y, r.w, r.h]


def frame_pixels(h, w, seed):
    return np.random.default_rng(seed).integers(0, 255, (h, w, 3), np.uint8)


def main():
    gold = {}
    # 1. grids (Table I + extras)
    grids = []
    for fw, fh, rows, ov in [(3840, 2160, 1, 20), (3840, 2160, 2, 20), (3840, 2160, 3, 20),
                             (3840, 2160, 4, 20), (3840, 2160, 6, 20), (7680, 4320, 1, 20),
                             (7680, 4320, 2, 20), (7680, 4320, 3, 20), (7680, 4320, 4, 20),
                             (1280, 720, 3, 50), (1280, 720, 1, 50), (608, 608, 1, 0),
                             (1000, 300, 2, 100), (97, 61, 5, 7)]:
        g = G.build_grid(fw, fh, G.CropSettings(rows, ov))
        grids.append({"fw": fw, "fh": fh, "rows": rows, "overlap": ov, "side": g.crop_side,
                      "cols": g.cols,
                      "crops": [[c.crop_id, c.row, c.col, *rect(c.global_rect), c.scale]
                                for c in g.crops]})
    gold["grids"] = grids

    # 2. cut_tile (nearest) byte hashes
    tiles = []
    rng = random.Random(3)
    for case in range(24):
        h, w = rng.choice([(700, 900), (400, 400), (1000, 1000), (500, 500), (2160, 3840)])
        side = rng.choice([304, 608, 736, 912, 1098, 2160, 37])
        x = rng.randint(-50, w - 10)
        y = rng.randint(-50, h - 10)
        seed = 100 + case
        px = frame_pixels(h, w, seed)
        crop = G.CropSpec(0, 0, 0, G.Rect(x, y, side, side), side / 608)
        t = cut_tile(px, crop)
        tiles.append({"h": h, "w": w, "seed": seed, "x": x, "y": y, "side": side,
                      "sha256": hashlib.sha256(t.tobytes()).hexdigest()})
    gold["cut_tile"] = tiles

    # 3. to_global
    tg = []
    rng = random.Random(11)
    for _ in range(400):
        fw, fh = rng.choice([(3840, 2160), (7680, 4320), (1280, 720)])
        side = rng.choice([736, 2160, 1472, 554, 1098, 3840, 7680, 4320])
        cx = rng.randint(0, max(0, fw - side)) if side <= fw else 0
        cy = rng.randint(0, max(0, fh - side)) if side <= fh else 0
        crop = G.CropSpec(0, 0, 0, G.Rect(cx, cy, side, side), side / 608)
        lx = rng.uniform(0, 600)
        ly = rng.uniform(0, 600)
        lw = rng.uniform(0.01, 608 - lx)
        lh = rng.uniform(0.01, 608 - ly)
        if rng.random() < 0.2:  # float32-valued local rects like the decoder emits
            lx, ly, lw, lh = (float(np.float32(v)) for v in (lx, ly, lw, lh))
            if lw <= 0 or lh <= 0:
                continue
        r = G.Rect(lx, ly, lw, lh)
        clip = rng.random() < 0.8
        out = G.to_global(r, crop, fw, fh) if clip else G.to_global(r, crop)
        tg.append({"crop": [cx, cy, side], "fw": fw, "fh": fh, "clip": clip,
                   "local": rect(r), "out": rect(out)})
    gold["to_global"] = tg

    # 4. merge_temporal + select_active
    sel = []
    rng = random.Random(17)
    for case in range(150):
        fw, fh, preset = rng.choice([(1280, 720, "1 att, 3 fin, 50 over"),
                                     (3840, 2160, "1 att, 3 fin, 20 over"),
                                     (3840, 2160, "2 att, 4 fin, 20 over"),
                                     (7680, 4320, "1 att, 6 fin, 20 over")])
        s = P.PipelineSettings.from_preset(preset)
        plan = P.GridPlan.build(fw, fh, s)
        hist = []
        for fid in range(rng.randint(1, 3)):
            boxes = []
            for _ in range(rng.randint(0, 12)):
                w = rng.randint(1, fw // 6)
                h = rng.randint(1, fh // 6)
                boxes.append(G.Rect(rng.randint(0, fw - w), rng.randint(0, fh - h), w, h))
            if hist and rng.random() < 0.5 and hist[-1].boxes:
                boxes.append(rng.choice(hist[-1].boxes))  # duplicates across frames
            hist.append(P.AttentionModel(fid, tuple(boxes), (fid,)))
        window = rng.randint(1, 3)
        margin = rng.choice([0, 5, 20, 40])
        merged = P.merge_temporal(hist, window)
        active = P.select_active(plan.final_grid, merged, margin)
        sel.append({"fw": fw, "fh": fh, "preset": preset, "window": window, "margin": margin,
                    "history": [[rect(b) for b in m.boxes] for m in hist],
                    "merged": [rect(b) for b in merged.boxes],
                    "active": sorted(active.active_ids)})
    gold["select"] = sel

    # 5. NMS keep indices
    nms = []
    rng = random.Random(23)
    for case in range(150):
        dets = []
        for _ in range(rng.randint(0, 40)):
            x, y = rng.randint(0, 200), rng.randint(0, 200)
            conf = rng.choice([0.5, 0.6, 0.7, 0.9]) if rng.random() < 0.3 else round(rng.random(), 3)
            dets.append(Detection(G.Rect(x, y, rng.randint(5, 80), rng.randint(5, 80)),
                                  rng.choice(["person", "car", "bus"]), conf))
        thr = rng.choice([0.3, 0.45, 0.6])
        nms.append({"dets": [[*rect(d.rect), d.class_label, d.confidence] for d in dets],
                    "thr": thr, "keep": PP.nms_keep_indices(dets, thr)})
    # exact-threshold IoU case (equal suppresses)
    gold["nms"] = nms

    # 6. merge_split / postprocess with variants
    post = []
    rng = random.Random(29)
    grids = {"720": G.build_grid(1280, 720, G.CropSettings(3, 50)),
             "4k": G.build_grid(3840, 2160, G.CropSettings(3, 20))}
    policies = [{}, {"merge_before_nms": True}, {"nms_per_crop": True},
                {"mergeable_classes": {"person": "both", "car": "horizontal"}},
                {"nms_iou": 0.3, "vertical_gap_px": 10, "horizontal_alignment_tolerance_px": 5}]
    for case in range(200):
        gname = rng.choice(list(grids))
        grid = grids[gname]
        tagged = []
        for _ in range(rng.randint(0, 30)):
            spec = rng.choice(grid.crops)
            gx, gy = int(spec.global_rect.x), int(spec.global_rect.y)
            side = int(spec.global_rect.w)
            x = gx + rng.randint(0, side - 20)
            y = gy + rng.randint(0, side - 20)
            if rng.random() < 0.4:  # fragment touching a border
                y = gy + side - rng.randint(5, 40)
            tagged.append((spec.crop_id, Detection(
                G.Rect(x, y, rng.randint(10, 150), rng.randint(10, 150)),
                rng.choice(["person", "person", "car"]), round(rng.uniform(0.2, 1.0), 2))))
        pol = rng.choice(policies)
        out = PP.postprocess(tagged, grid, PP.MergePolicy(**pol))
        ms = PP.merge_split(tagged, grid, PP.MergePolicy(**pol))
        post.append({"grid": gname, "policy": pol,
                     "tagged": [[cid, *rect(d.rect), d.class_label, d.confidence]
                                for cid, d in tagged],
                     "out": [[*rect(d.rect), d.class_label, d.confidence] for d in out],
                     "merge_split": [[*rect(d.rect), d.class_label, d.confidence] for d in ms]})
    gold["postprocess"] = post

    # 7. synthetic scenes (GT) + render hashes, and full pipeline runs with the scene oracle
    scenes = []
    for kind, fw, fh, nfr in [("dense", 3840, 2160, 6), ("sparse", 3840, 2160, 4),
                              ("mixed", 7680, 4320, 3), ("straddle", 1280, 720, 4),
                              ("small", 3840, 2160, 2)]:
        spec = SY.SceneSpec(kind, fw, fh, nfr, seed=0)
        gt = SY.generate_scene(spec)
        renders = {}
        for fid in (0, nfr - 1):
            img = SY.render_frame(fw, fh, gt[fid])
            renders[str(fid)] = hashlib.sha256(img.tobytes()).hexdigest()
        settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
        oracle = P.oracle_for_scene(fw, fh, settings, gt)
        frames = [P.Frame(i, fw, fh) for i in range(nfr)]
        res = list(P.run_sequence(frames, settings, oracle))
        allc = [P.run_allcrops_baseline(f, settings, oracle) for f in frames[:2]]
        down = [P.run_downscale_baseline(f, oracle, settings) for f in frames[:2]]
        scenes.append({
            "kind": kind, "fw": fw, "fh": fh, "frames": nfr,
            "gt": {str(k): [[*rect(o.rect), o.class_label, o.object_id] for o in v]
                   for k, v in gt.items()},
            "render_sha256": renders,
            "pipeline": [{"dets": [[*rect(d.rect), d.class_label, d.confidence]
                                   for d in r.detections],
                          "active": r.active_count, "total": r.total_count} for r in res],
            "allcrops": [[[*rect(d.rect), d.class_label, d.confidence] for d in r.detections]
                         for r in allc],
            "downscale": [[[*rect(d.rect), d.class_label, d.confidence] for d in r.detections]
                          for r in down],
        })
    gold["scenes"] = scenes
    with open(OUT, "w") as fh:
        json.dump(gold, fh, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
