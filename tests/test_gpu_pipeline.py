"""GPU kernels behind the reference-compatible API vs the REAL reference's outputs
(golden vectors) — bit-exact: to_global projection, merge_temporal + select_active,
NMS keep indices, merge_split and postprocess (all policy variants), and the whole
staged pipeline / baselines driven by the ground-truth scene detector."""

import json
import os
import random

import pytest

from paper_1810_10551_b200 import kernels, pipeline as P, synthetic
from paper_1810_10551_b200.detector import Detection, GroundTruthObject
from paper_1810_10551_b200.geometry import CropSettings, Rect, build_grid
from paper_1810_10551_b200.postprocess import MergePolicy, merge_split, nms, nms_keep_indices, \
    postprocess

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _row(d):
    return [d.rect.x, d.rect.y, d.rect.w, d.rect.h, d.class_label, d.confidence]


def test_projection_kernel_matches_reference(cuda):
    cases = GOLD["to_global"]
    for clip in (True, False):
        sub = [c for c in cases if c["clip"] == clip]
        fw = [c["fw"] for c in sub]
        # one launch per frame size (the kernel takes one frame size per call)
        for size in set(zip(fw, [c["fh"] for c in sub])):
            cs = [c for c in sub if (c["fw"], c["fh"]) == size]
            out = kernels.project_rects([c["local"] for c in cs], [c["crop"] for c in cs],
                                        size[0] if clip else None, size[1] if clip else None)
            assert [list(map(int, r)) for r in out] == [c["out"] for c in cs]


def test_select_and_merge_temporal_match_reference(cuda):
    for c in GOLD["select"]:
        s = P.PipelineSettings.from_preset(c["preset"])
        plan = P.GridPlan.build(c["fw"], c["fh"], s)
        hist = [P.AttentionModel(i, tuple(Rect(*b) for b in m), (i,))
                for i, m in enumerate(c["history"])]
        merged = P.merge_temporal(hist, c["window"])
        assert [[b.x, b.y, b.w, b.h] for b in merged.boxes] == c["merged"]
        act = P.select_active(plan.final_grid, merged, c["margin"])
        assert sorted(act.active_ids) == c["active"]


def test_nms_matches_reference(cuda):
    for c in GOLD["nms"]:
        dets = [Detection(Rect(*d[:4]), d[4], d[5]) for d in c["dets"]]
        assert nms_keep_indices(dets, c["thr"]) == c["keep"]


def test_reference_nms_cases(cuda):
    def det(x, y, w, h, conf, label="person"):
        return Detection(Rect(x, y, w, h), label, conf)

    d = [det(10, 10, 50, 50, 0.9), det(10, 10, 50, 50, 0.8)]
    assert nms(d, 0.45) == [d[0]]
    d = [det(0, 0, 10, 10, 0.9), det(0, 0, 10, 10, 0.8, "car")]
    assert len(nms(d, 0.45)) == 2
    # IoU exactly equal to the threshold suppresses: 10x10 boxes offset by 5 -> 50/150
    d = [det(0, 0, 10, 10, 0.9), det(5, 0, 10, 10, 0.8)]
    assert nms(d, 50 / 150) == [d[0]]
    d = [det(0, 0, 10, 10, 0.5), det(100, 0, 10, 10, 0.5), det(200, 0, 10, 10, 0.5)]
    assert nms_keep_indices(d, 0.45) == [0, 1, 2]


def test_postprocess_and_merge_split_match_reference(cuda):
    grids = {"720": build_grid(1280, 720, CropSettings(3, 50)),
             "4k": build_grid(3840, 2160, CropSettings(3, 20))}
    for c in GOLD["postprocess"]:
        grid = grids[c["grid"]]
        tagged = [(t[0], Detection(Rect(*t[1:5]), t[5], t[6])) for t in c["tagged"]]
        pol = MergePolicy(**c["policy"])
        assert [_row(d) for d in postprocess(tagged, grid, pol)] == c["out"]
        assert [_row(d) for d in merge_split(tagged, grid, pol)] == c["merge_split"]


def test_reference_merge_goldens(cuda):
    grid = build_grid(1280, 720, CropSettings(3, 50))

    def det(x, y, w, h, conf, label="person"):
        return Detection(Rect(x, y, w, h), label, conf)

    frags = [(0, det(50, 120, 60, 134, 0.67)), (grid.cols, det(50, 233, 60, 87, 0.435))]
    assert merge_split(frags, grid, MergePolicy()) == [det(50, 120, 60, 200, 0.67)]
    chain = [(0, det(60, 100, 50, 154, 0.4)), (grid.cols, det(60, 233, 50, 254, 0.64)),
             (2 * grid.cols, det(60, 466, 50, 34, 0.35))]
    assert merge_split(chain, grid, MergePolicy()) == [det(60, 100, 50, 400, 0.64)]
    near = [(0, det(50, 100, 60, 100, 0.7)), (grid.cols, det(50, 240, 60, 50, 0.6))]
    far = [(0, det(50, 100, 60, 100, 0.7)), (grid.cols, det(50, 241, 60, 50, 0.6))]
    assert len(merge_split(near, grid, MergePolicy())) == 1
    assert len(merge_split(far, grid, MergePolicy())) == 2
    ok = [(0, det(50, 120, 60, 134, 0.7)), (grid.cols, det(80, 233, 60, 87, 0.6))]
    off = [(0, det(50, 120, 60, 134, 0.7)), (grid.cols, det(81, 233, 60, 87, 0.6))]
    assert len(merge_split(ok, grid, MergePolicy())) == 1
    assert len(merge_split(off, grid, MergePolicy())) == 2
    assert postprocess([], grid, MergePolicy()) == []


@pytest.mark.parametrize("idx", range(5))
def test_staged_pipeline_with_scene_detector_matches_reference(cuda, idx):
    sc = GOLD["scenes"][idx]
    spec = synthetic.SceneSpec(sc["kind"], sc["fw"], sc["fh"], sc["frames"], seed=0)
    gt = synthetic.generate_scene(spec)
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    oracle = P.oracle_for_scene(sc["fw"], sc["fh"], settings, gt)
    frames = [P.Frame(i, sc["fw"], sc["fh"]) for i in range(sc["frames"])]
    res = list(P.run_sequence(frames, settings, oracle))
    for r, ref in zip(res, sc["pipeline"]):
        assert [_row(d) for d in r.detections] == ref["dets"]
        assert (r.active_count, r.total_count) == (ref["active"], ref["total"])
    for f, ref in enumerate(sc["allcrops"]):
        assert [_row(d) for d in P.run_allcrops_baseline(frames[f], settings, oracle).detections] \
            == ref
    for f, ref in enumerate(sc["downscale"]):
        assert [_row(d) for d in P.run_downscale_baseline(frames[f], oracle, settings).detections] \
            == ref


def test_staged_equals_allcrops_on_random_scenes(cuda):
    """Reference property test_pipeline.py:361-375 (30 attention-visible scenes)."""
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 50 over")
    rng = random.Random(71)
    for case in range(30):
        objs = []
        for i in range(rng.randint(1, 6)):
            w, h = rng.randint(40, 150), rng.randint(40, 150)
            objs.append(GroundTruthObject(Rect(rng.randint(0, 1280 - w), rng.randint(0, 720 - h),
                                               w, h), "person", f"{case}:{i}"))
        oracle = P.oracle_for_scene(1280, 720, settings, {0: objs})
        frame = P.Frame(0, 1280, 720)
        staged = P.run_frame(frame, settings, oracle)
        full = P.run_allcrops_baseline(frame, settings, oracle)
        assert staged.detections == full.detections
        assert staged.active_count <= full.active_count


def test_stage_failure_names_stage(cuda):
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 50 over")

    class Boom(P.SceneOracle):
        def detect(self, frame_id, crop_id, tile=None):
            raise RuntimeError("boom")

    plan = P.GridPlan.build(1280, 720, settings)
    det = Boom(plan.crops_by_id(), {3: []})
    with pytest.raises(P.StageFailure, match="attention stage failed on frame 3"):
        P.run_frame(P.Frame(3, 1280, 720), settings, det)
