"""CPU-only checks: host value types / validation mirror the reference, the C-ABI
library loads and exports every symbol include/tilepipe_b200.h declares, and the
product package never imports the oracle."""

import ast
import json
import os
import re

import pytest

from paper_1810_10551_b200 import native
from paper_1810_10551_b200.geometry import (CropSettings, Rect, build_grid, crop_side_px,
                                            intersects, iou, to_global, to_local)
from paper_1810_10551_b200.pipeline_types import (ActiveSet, FrameResult, GridPlan,
                                                  PipelineSettings, TimingProfile)
from paper_1810_10551_b200.postprocess import MergePolicy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))


def test_grid_planning_matches_reference_golden():
    for g in GOLD["grids"]:
        grid = build_grid(g["fw"], g["fh"], CropSettings(g["rows"], g["overlap"]))
        assert (grid.crop_side, grid.cols) == (g["side"], g["cols"])
        got = [[c.crop_id, c.row, c.col, c.global_rect.x, c.global_rect.y, c.global_rect.w,
                c.global_rect.h, c.scale] for c in grid.crops]
        assert got == g["crops"]


def test_table_one_golden():
    for fh, rows, side in [(2160, 1, 2160), (2160, 2, 1098), (2160, 3, 736), (2160, 4, 554),
                           (2160, 6, 370), (4320, 1, 4320), (4320, 2, 2196), (4320, 3, 1472),
                           (4320, 4, 1107)]:
        assert crop_side_px(fh, CropSettings(rows, 20)) == side


def test_host_to_global_matches_reference_golden():
    from paper_1810_10551_b200.geometry import CropSpec

    for c in GOLD["to_global"]:
        cx, cy, side = c["crop"]
        crop = CropSpec(0, 0, 0, Rect(cx, cy, side, side), side / 608)
        r = Rect(*c["local"])
        out = to_global(r, crop, c["fw"], c["fh"]) if c["clip"] else to_global(r, crop)
        assert [out.x, out.y, out.w, out.h] == c["out"]


def test_rect_semantics():
    with pytest.raises(ValueError):
        Rect(0, 0, 0, 5)
    with pytest.raises(ValueError):
        Rect(float("nan"), 0, 1, 1)
    a, b = Rect(0, 0, 10, 10), Rect(10, 0, 5, 5)
    assert not intersects(a, b) and iou(a, b) == 0.0
    assert iou(a, a) == 1.0
    crop = build_grid(1216, 1216, CropSettings(1, 0)).crops[0]
    loc = to_local(crop.global_rect, crop)
    assert (loc.x, loc.y, loc.w, loc.h) == (0, 0, 608, 608)


def test_pipeline_settings_and_plan():
    s = PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    assert s.preset_name() == "1 att, 3 fin, 20 over"
    with pytest.raises(ValueError):
        PipelineSettings.from_preset("3 rows")
    with pytest.raises(ValueError):
        PipelineSettings(CropSettings(3), CropSettings(2))
    plan = GridPlan.build(3840, 2160, s)
    assert len(plan.attention_grid.crops) == 2 and len(plan.final_grid.crops) == 18
    assert plan.downscale_id == 20 and plan.downscale_crop.global_rect == Rect(0, 0, 3840, 3840)
    with pytest.raises(ValueError):
        ActiveSet(plan.final_grid, frozenset({999}))
    with pytest.raises(ValueError):
        FrameResult(0, (), 5, 2, TimingProfile())
    with pytest.raises(ValueError):
        TimingProfile(final_eval_ms=-1.0)
    with pytest.raises(ValueError):
        MergePolicy(nms_iou=1.0)
    with pytest.raises(ValueError):
        MergePolicy(mergeable_classes={"person": "diagonal"})


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "tilepipe_b200.h")).read()
    return set(re.findall(r"TP_API\s+[\w\s\*]+?\b(tp_\w+)\s*\(", src))


def test_library_loads_and_exports_every_header_symbol():
    lib = native.load()  # loading needs no GPU
    declared = _header_symbols()
    assert declared, "no TP_API declarations found"
    assert declared == set(native.SIGNATURES), declared ^ set(native.SIGNATURES)
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.tp_version() == 1
    assert lib.tp_yolo_workspace_bytes(1, 1) > 20_000_000
    # the fp32-parity plan doubles every activation buffer but the input slots and head
    assert lib.tp_yolo_workspace_bytes(1, 2) > 1.8 * lib.tp_yolo_workspace_bytes(1, 1)
    # the result gather rejects a missing communicator before touching NCCL or CUDA
    assert lib.tp_nccl_gather_dets(None, None, 0, None, 0, None, None, None) == 1
    assert b"bad argument" in lib.tp_last_error()


def test_product_never_imports_oracle():
    """No module of the package or its subpackages imports oracle/ (nor loads it by name
    through importlib / __import__)."""
    pkg = os.path.join(ROOT, "paper_1810_10551_b200")
    n = 0
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if not fn.endswith(".py"):
                continue
            path = os.path.join(dirpath, fn)
            src = open(path).read()
            tree = ast.parse(src)
            n += 1
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), path
                if isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", path
                if isinstance(node, ast.Constant) and isinstance(node.value, str):
                    assert not node.value.startswith("oracle."), path
    assert n >= 15  # walked the subpackages too (distribution/)


def test_ops_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    from paper_1810_10551_b200.detector import cut_tile
    from paper_1810_10551_b200.postprocess import nms

    crop = build_grid(608, 608, CropSettings(1, 0)).crops[0]
    with pytest.raises(native.NativeUnavailable):
        cut_tile(np.zeros((608, 608, 3), np.uint8), crop)
    from paper_1810_10551_b200.detector import Detection

    with pytest.raises(native.NativeUnavailable):
        nms([Detection(Rect(0, 0, 5, 5), "a", 0.5)], 0.45)


def test_result_line_is_byte_identical_to_reference_format():
    from paper_1810_10551_b200.detector import Detection
    from paper_1810_10551_b200.stream import result_line

    r = FrameResult(7, (Detection(Rect(10, 20, 30, 40), "person", 0.5),
                        Detection(Rect(1, 2, 3, 4), 'car "x"', 1.0)), 3, 18, TimingProfile())
    assert result_line(r) == (
        '{"active_count":3,"detections":[{"class":"person","confidence":0.500000,"h":40,"w":30,'
        '"x":10,"y":20},{"class":"car \\"x\\"","confidence":1.000000,"h":4,"w":3,"x":1,"y":2}],'
        '"frame_id":7,"total_count":18}')


def test_stream_ramp_chunks():
    """run_stream's batching: long streams ramp B/4, B/2, then B; order is kept."""
    from paper_1810_10551_b200.stream import ramp_chunks

    items = list(range(100))
    ch = ramp_chunks(items, 30)
    assert [len(c) for c in ch] == [7, 15, 30, 30, 18]
    assert [x for c in ch for x in c] == items
    assert [len(c) for c in ramp_chunks(items[:60], 30)] == [30, 30]  # not > 2B: no ramp
    assert [len(c) for c in ramp_chunks(items[:10], 2)] == [2] * 5     # B < 4: no ramp


def test_hl8_plan_tables():
    """The F16F8 (HL8) plan's host-side tables, without a GPU: every conv but layer 0 reads
    HL8 planes; the weight scales keep the fp16 hi-pass weights finite and the e4m3 lo-pass
    weights <= 240 with b = c - LO_EXP; the issued-work count is 1.5x K past layer 0."""
    import numpy as np

    from paper_1810_10551_b200 import yolo

    assert yolo.hl8_input_slots() == frozenset(range(1, len(yolo.LAYERS)))
    wpacks, _ = yolo.make_weights(0, dtype="fp16")
    for li in range(1, len(yolo.LAYERS)):
        c, b = yolo.hl8_scales(wpacks[li])
        wmax = float(np.abs(wpacks[li]).max())
        assert b == c - yolo.LO_EXP and wmax * 2.0 ** c <= 65504 and wmax * 2.0 ** b <= 240
        assert wmax * 2.0 ** (b + 1) > 240 or wmax * 2.0 ** (c + 1) > 65504  # the largest
        # hi-pass weights are the model's fp16 values scaled exactly by 2^c; the e4m3
        # lo-pass copy is within e4m3's 2^-4 relative rounding of w (normal range)
        whi, wlo, alpha = yolo.hl8_weights(wpacks[li])
        assert alpha == 2.0 ** -c
        assert np.array_equal(whi.astype(np.float16).astype(np.float32), whi)
        assert np.array_equal(whi * np.float32(alpha), np.asarray(wpacks[li], np.float32))
        lov = yolo.hl8_lo_weight_values(wpacks[li])
        w = np.asarray(wpacks[li], np.float32)
        big = np.abs(w) * 2.0 ** b >= 2.0 ** -6  # e4m3 normal range
        assert np.all(np.abs(lov - w)[big] <= np.abs(w)[big] * 2.0 ** -4 + 1e-12)
        assert wlo.dtype == np.uint8 and wlo.shape == w.shape
    g = [2.0 * s * s * co * ci * k * k / 1e9 for _, ci, co, k, s in yolo.LAYERS]
    assert abs(yolo.exec_gflop_per_tile("fp32") - (g[0] + 1.5 * sum(g[1:]))) < 1e-9
    assert abs(yolo.exec_gflop_per_tile("fp32x2") - (g[0] + 2.0 * sum(g[1:]))) < 1e-9
