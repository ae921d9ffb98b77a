"""NMS + merge (K7) at the survey's stress sizes: 400, 1,000 and 2,000 raw detections in
one frame (reference postprocess takes 140 ms / 1.6 s at 400 / 1,000),
every policy variant, bit-exact against the CPU restatement of the reference
(postprocess.py:54-187) — keep-set, order, merged rects and scores."""

import pytest

from oracle import e2e as E
from oracle import pipeline_ref as R
from paper_1810_10551_b200.detector import Detection
from paper_1810_10551_b200.geometry import CropSettings, Rect, build_grid
from paper_1810_10551_b200.postprocess import MergePolicy, postprocess

pytestmark = pytest.mark.gpu

W, H = 3840, 2160


@pytest.mark.parametrize("n,variant", [(400, "default"), (1000, "default"), (2000, "default"),
                                       (1000, "nms_per_crop"), (1000, "merge_before_nms")])
def test_postprocess_stress_matches_reference(cuda, n, variant):
    plan = R.Plan(W, H, 1, 3, 20)
    grid = build_grid(W, H, CropSettings(3, 20), id_base=len(plan.att[3]))
    raw = E.synthetic_raw_detections(plan, n, seed=n)
    kw = {} if variant == "default" else {variant: True}
    want = R.finish(raw, R.cell_map(plan), 0.3, **kw)
    tagged = [(cid, Detection(Rect(*r), lab, conf)) for cid, (r, lab, conf) in raw]
    got = postprocess(tagged, grid, MergePolicy(**kw), min_confidence=0.3)
    got = [((d.rect.x, d.rect.y, d.rect.w, d.rect.h), d.class_label, d.confidence) for d in got]
    assert got == want
    assert len(want) < n  # NMS suppressed and merged
