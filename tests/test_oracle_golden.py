"""Pin the CPU oracle (and the synthetic-scene port) to golden vectors produced by the
REAL reference (tests/golden/make_golden.py). CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pipeline_ref as R
from paper_1810_10551_b200 import synthetic

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _close(a, b):
    return all(x == y for x, y in zip(a, b)) and len(a) == len(b)


def test_grids_match_reference():
    for g in GOLD["grids"]:
        side, rows, cols, crops = R.build_grid(g["fw"], g["fh"], g["rows"], g["overlap"])
        assert (side, cols) == (g["side"], g["cols"])
        assert [list(c[:3]) + [c[3], c[4], c[5], c[5], c[6]] for c in crops] == g["crops"]


def test_cut_tile_nearest_matches_reference_hashes():
    for case in GOLD["cut_tile"]:
        px = np.random.default_rng(case["seed"]).integers(0, 255, (case["h"], case["w"], 3),
                                                          np.uint8)
        crop = (0, 0, 0, case["x"], case["y"], case["side"], case["side"] / 608)
        t = R.cut_tile_nearest(px, crop)
        assert hashlib.sha256(t.tobytes()).hexdigest() == case["sha256"]


def test_to_global_matches_reference():
    for c in GOLD["to_global"]:
        cx, cy, side = c["crop"]
        crop = (0, 0, 0, cx, cy, side, side / 608)
        if c["clip"]:
            out = R.to_global(tuple(c["local"]), crop, c["fw"], c["fh"])
        else:
            out = R.to_global(tuple(c["local"]), crop)
        assert list(out) == c["out"]


def _plan(c):
    a, f, o = (int(t.split()[0]) for t in c["preset"].split(","))
    return R.Plan(c["fw"], c["fh"], a, f, o)


def test_merge_temporal_and_select_match_reference():
    for c in GOLD["select"]:
        plan = _plan(c)
        hist = [[tuple(b) for b in m] for m in c["history"]]
        merged = R.merge_temporal(hist, c["window"])
        assert [list(b) for b in merged] == c["merged"]
        act = R.select_active(plan.fin, merged, c["margin"], c["fw"], c["fh"])
        assert act == c["active"]


def test_nms_matches_reference():
    for c in GOLD["nms"]:
        dets = [((d[0], d[1], d[2], d[3]), d[4], d[5]) for d in c["dets"]]
        assert R.nms_keep_indices(dets, c["thr"]) == c["keep"]


def _post_args(c):
    grid = {"720": R.build_grid(1280, 720, 3, 50), "4k": R.build_grid(3840, 2160, 3, 20)}[c["grid"]]
    cell_of = {cr[0]: (cr[1], cr[2]) for cr in grid[3]}
    tagged = [(t[0], ((t[1], t[2], t[3], t[4]), t[5], t[6])) for t in c["tagged"]]
    pol = c["policy"]
    kw = {"nms_iou": pol.get("nms_iou", 0.45),
          "rules": pol.get("mergeable_classes", {"person": "vertical"}),
          "gap": pol.get("vertical_gap_px", 40), "tol": pol.get("horizontal_alignment_tolerance_px", 30),
          "merge_before_nms": pol.get("merge_before_nms", False),
          "nms_per_crop": pol.get("nms_per_crop", False)}
    return tagged, cell_of, kw


def test_postprocess_and_merge_split_match_reference():
    for c in GOLD["postprocess"]:
        tagged, cell_of, kw = _post_args(c)
        out = R.postprocess(tagged, cell_of, **kw)
        assert [[*d[0], d[1], d[2]] for d in out] == c["out"]
        ms = R.merge_split(tagged, cell_of, kw["rules"], kw["gap"], kw["tol"])
        assert [[*d[0], d[1], d[2]] for d in ms] == c["merge_split"]


@pytest.mark.parametrize("idx", range(5))
def test_scene_generation_and_pipeline_match_reference(idx):
    sc = GOLD["scenes"][idx]
    spec = synthetic.SceneSpec(sc["kind"], sc["fw"], sc["fh"], sc["frames"], seed=0)
    gt = synthetic.generate_scene(spec)
    for fid, objs in sc["gt"].items():
        assert [[o.rect.x, o.rect.y, o.rect.w, o.rect.h, o.class_label, o.object_id]
                for o in gt[int(fid)]] == objs
    if sc["fw"] <= 3840:
        for fid, h in sc["render_sha256"].items():
            img = synthetic.render_frame(sc["fw"], sc["fh"], gt[int(fid)])
            assert hashlib.sha256(img.tobytes()).hexdigest() == h
    plan = R.Plan(sc["fw"], sc["fh"], 1, 3, 20)
    gtl = {f: [((o.rect.x, o.rect.y, o.rect.w, o.rect.h), o.class_label) for o in v]
           for f, v in gt.items()}

    def detect(fid, crop):
        return R.mock_detect(crop, gtl[fid])

    res = R.run_sequence(plan, range(sc["frames"]), detect)
    for (fid, dets, active), ref in zip(res, sc["pipeline"]):
        assert [[*d[0], d[1], d[2]] for d in dets] == ref["dets"]
        assert len(active) == ref["active"]
    for f, ref in enumerate(sc["allcrops"]):
        assert [[*d[0], d[1], d[2]] for d in R.run_allcrops_baseline(plan, f, detect)] == ref
    for f, ref in enumerate(sc["downscale"]):
        assert [[*d[0], d[1], d[2]] for d in R.run_downscale_baseline(plan, f, detect)] == ref
