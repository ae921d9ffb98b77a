"""Two-stage evaluation — reference-compatible entry points, GPU execution.

Mirrors ``tilepipe/pipeline.py`` name for name: ``oracle_for_scene`` (:272-288),
``attention_pass`` (:297-316), ``merge_temporal`` (:319-338), ``select_active``
(:341-354), ``final_pass`` (:357-375), ``finish_detections`` (:378-385),
``evaluate_frame`` / ``run_frame`` / ``run_sequence`` (:388-457) and both baselines
(:460-530), with the same signatures, defaults, ordering and ``StageFailure`` errors.

Two execution modes behind the same functions:
  * the detector is a ``YoloB200Detector``: the whole frame (or clip) runs in the
    device-resident batched engine (engine.AttentionPipelineB200);
  * any other ``Detector`` plugin: the detector is called per crop exactly as in the
    reference, and everything around it (tile cutting, to_global, temporal merge,
    selection, NMS + merge) runs on the GPU kernels.
There is no host compute fallback: without the CUDA library these functions raise.
"""

from __future__ import annotations

import time
from collections.abc import Iterable, Iterator, Mapping, Sequence

import numpy as np

from . import kernels
from .detector import Detection, Detector, GroundTruthObject, cut_tile
from .geometry import CropSettings, CropSpec, GridSpec, Rect
from .pipeline_types import (PRESET_RE, ActiveSet, AttentionModel, Frame, FrameResult, GridPlan,
                             PipelineSettings, StageFailure, TimingProfile)
from .postprocess import MergePolicy, postprocess
from .scene_oracle import SceneOracle

__all__ = [
    "PRESET_RE", "ActiveSet", "AttentionModel", "Frame", "FrameResult", "GridPlan",
    "PipelineSettings", "StageFailure", "TimingProfile", "oracle_for_scene", "attention_pass",
    "merge_temporal", "select_active", "final_pass", "finish_detections", "evaluate_frame",
    "run_frame", "run_sequence", "run_downscale_baseline", "run_allcrops_baseline",
]

MAX_WINDOW_BOXES = 512  # selection kernel capacity per frame window


def oracle_for_scene(frame_w: int, frame_h: int, settings: PipelineSettings,
                     gt_by_frame: Mapping[int, Sequence[GroundTruthObject]],
                     visibility_threshold: float = 0.3, *, min_tile_px: int = 8) -> SceneOracle:
    plan = GridPlan.build(frame_w, frame_h, settings)
    return SceneOracle(plan.crops_by_id(), gt_by_frame, visibility_threshold,
                       min_tile_px=min_tile_px)


def _is_yolo(det) -> bool:
    from .yolo import YoloB200Detector

    return isinstance(det, YoloB200Detector)


def _engine_for(det, settings: PipelineSettings, frame_w: int, frame_h: int,
                policy: MergePolicy | None):
    from .engine import AttentionPipelineB200

    cache = det.__dict__.setdefault("_engines", {})
    key = (settings, frame_w, frame_h, policy or MergePolicy())
    key = (key[0], key[1], key[2], repr(key[3]))
    eng = cache.get(key)
    if eng is None:
        eng = AttentionPipelineB200(settings, frame_w, frame_h, max_frames=4, seed=det.seed,
                                    threshold=det.threshold, policy=policy, head=det.head,
                                    precision=det.precision)
        cache[key] = eng
    return eng


def _detect_crops(frame: Frame, crops: Sequence[CropSpec], det: Detector, stage: str):
    """Per-crop plugin calls (reference order). Tiles are cut on the GPU in one batch."""
    tiles = None
    if frame.pixels is not None and crops:
        from .detector import cut_tiles

        tiles = cut_tiles(frame.pixels, list(crops)).cpu().numpy()
    out = []
    for i, crop in enumerate(crops):
        try:
            found = det.detect(frame.frame_id, crop.crop_id, None if tiles is None else tiles[i])
        except Exception as exc:
            raise StageFailure(stage, frame.frame_id) from exc
        out.append(found)
    return out


def _project(pairs, frame: Frame):
    """[(crop, Detection)] -> integer global Rects via the GPU to_global kernel."""
    loc = [[d.rect.x, d.rect.y, d.rect.w, d.rect.h] for _, d in pairs]
    crs = [[int(c.global_rect.x), int(c.global_rect.y), int(c.global_rect.w)] for c, _ in pairs]
    g = kernels.project_rects(loc, crs, frame.width, frame.height)
    return [Rect(int(r[0]), int(r[1]), int(r[2]), int(r[3])) for r in g]


def attention_pass(frame: Frame, settings: PipelineSettings, det: Detector, *,
                   plan: GridPlan | None = None) -> AttentionModel:
    if plan is None:
        plan = GridPlan.build(frame.width, frame.height, settings)
    crops = plan.attention_grid.crops
    if _is_yolo(det):
        if frame.pixels is None:
            raise StageFailure("attention", frame.frame_id) from ValueError("no pixels")
        eng = _engine_for(det, settings, frame.width, frame.height, None)
        return eng.attention_only(frame)
    found = _detect_crops(frame, crops, det, "attention")
    pairs = [(c, d) for c, ds in zip(crops, found) for d in ds
             if d.confidence >= settings.min_confidence]
    return AttentionModel(frame.frame_id, tuple(_project(pairs, frame)), (frame.frame_id,))


def merge_temporal(history: Sequence[AttentionModel], window: int) -> AttentionModel:
    if not history:
        raise ValueError("history must be non-empty")
    if window < 1:
        raise ValueError("window must be >= 1")
    ids = [m.frame_id for m in history]
    if ids != sorted(ids):
        raise ValueError(f"history must be ordered by frame_id, got {ids}")
    recent = list(history[-window:])
    slots = [[(b.x, b.y, b.w, b.h) for b in m.boxes] for m in recent]
    if sum(len(s) for s in slots) > MAX_WINDOW_BOXES:
        raise ValueError(f"more than {MAX_WINDOW_BOXES} boxes in the temporal window")
    # the select kernel de-duplicates in first-seen order; one dummy crop suffices
    (_, merged), = kernels.select(slots, len(slots), [[0.0, 0.0, 1.0, 1.0]], 0, 0.0, 1.0, 1.0,
                                  n_frames=1)
    boxes = tuple(_rect_like(m, recent) for m in merged)
    return AttentionModel(recent[-1].frame_id, boxes, tuple(m.frame_id for m in recent))


def _rect_like(vals, models):
    """Rebuild a Rect keeping the caller's int/float coordinate types."""
    for m in models:
        for b in m.boxes:
            if (b.x, b.y, b.w, b.h) == vals:
                return b
    return Rect(*vals)


def select_active(final_grid: GridSpec, att: AttentionModel, margin: int) -> ActiveSet:
    if margin < 0:
        raise ValueError("margin must be >= 0")
    if len(att.boxes) > MAX_WINDOW_BOXES:
        raise ValueError(f"more than {MAX_WINDOW_BOXES} attention boxes")
    for b in att.boxes:  # Rect.dilated would raise for a box entirely outside the frame
        b.dilated(margin, final_grid.frame_w, final_grid.frame_h)
    crops = [[c.global_rect.x, c.global_rect.y, c.global_rect.w, c.global_rect.h]
             for c in final_grid.crops]
    base = final_grid.crops[0].crop_id
    (ids, _), = kernels.select([[(b.x, b.y, b.w, b.h) for b in att.boxes]], 1, crops, base,
                               float(margin), final_grid.frame_w, final_grid.frame_h, n_frames=1)
    return ActiveSet(final_grid, frozenset(ids))


def final_pass(frame: Frame, active: ActiveSet, det: Detector) -> list[tuple[int, Detection]]:
    ids = sorted(active.active_ids)
    crops = [active.grid.crop_by_id(i) for i in ids]
    if _is_yolo(det):
        if frame.pixels is None:
            raise StageFailure("final", frame.frame_id) from ValueError("no pixels")
        from .engine import yolo_tagged

        try:
            return yolo_tagged(det, frame, crops)
        except Exception as exc:
            raise StageFailure("final", frame.frame_id) from exc
    found = _detect_crops(frame, crops, det, "final")
    pairs = [(c, d) for c, ds in zip(crops, found) for d in ds]
    rects = _project(pairs, frame)
    return [(c.crop_id, Detection(r, d.class_label, d.confidence))
            for (c, d), r in zip(pairs, rects)]


def finish_detections(tagged: Sequence[tuple[int, Detection]], grid: GridSpec,
                      policy: MergePolicy, min_confidence: float) -> tuple[Detection, ...]:
    return tuple(postprocess(tagged, grid, policy, min_confidence=min_confidence))


def evaluate_frame(frame: Frame, settings: PipelineSettings, det: Detector,
                   history: Sequence[AttentionModel] = (), policy: MergePolicy | None = None, *,
                   plan: GridPlan | None = None) -> tuple[FrameResult, AttentionModel]:
    if plan is None:
        plan = GridPlan.build(frame.width, frame.height, settings)
    if _is_yolo(det) and frame.pixels is not None:
        eng = _engine_for(det, settings, frame.width, frame.height, policy)
        return eng.evaluate_frames([frame], history)[0]
    policy = policy or MergePolicy()
    t0 = time.perf_counter()
    att = attention_pass(frame, settings, det, plan=plan)
    t1 = time.perf_counter()
    merged = merge_temporal([*history, att], settings.temporal_window)
    active = select_active(plan.final_grid, merged, settings.attention_margin_px)
    t2 = time.perf_counter()
    tagged = final_pass(frame, active, det)
    t3 = time.perf_counter()
    try:
        dets = finish_detections(tagged, plan.final_grid, policy, settings.min_confidence)
    except Exception as exc:
        raise StageFailure("postprocess", frame.frame_id) from exc
    t4 = time.perf_counter()
    timing = TimingProfile(attention_wait_ms=(t1 - t0) * 1e3, client_processing_ms=(t2 - t1) * 1e3,
                           final_eval_ms=(t3 - t2) * 1e3, postprocess_ms=(t4 - t3) * 1e3)
    res = FrameResult(frame.frame_id, dets, len(active.active_ids), len(plan.final_grid.crops),
                      timing)
    return res, att


def run_frame(frame: Frame, settings: PipelineSettings, det: Detector,
              history: Sequence[AttentionModel] = (), policy: MergePolicy | None = None, *,
              plan: GridPlan | None = None) -> FrameResult:
    return evaluate_frame(frame, settings, det, history, policy, plan=plan)[0]


def run_sequence(frames: Iterable[Frame], settings: PipelineSettings, det: Detector,
                 policy: MergePolicy | None = None, *, plan: GridPlan | None = None
                 ) -> Iterator[FrameResult]:
    if _is_yolo(det):
        yield from _run_sequence_batched(frames, settings, det, policy)
        return
    keep = settings.temporal_window - 1
    history: list[AttentionModel] = []
    for frame in frames:
        result, att = evaluate_frame(frame, settings, det, history, policy, plan=plan)
        history.append(att)
        del history[: max(0, len(history) - keep)]
        yield result


def _run_sequence_batched(frames, settings, det, policy):
    """Clip mode: frames go through the device engine in batches. The generator keeps its
    own attention history (the last K-1 AttentionModels, as the reference's run_sequence
    does, pipeline.py:442-457) and hands it to every batch, so interleaved generators and
    other callers sharing the cached engine cannot disturb each other; each batch holds
    the engine's lock (identical results to the per-frame loop)."""
    eng = None
    keep = settings.temporal_window - 1
    history: list[AttentionModel] = []
    batch: list[Frame] = []

    def flush():
        nonlocal history
        out = eng.evaluate_frames(batch, history)
        history = [*history, *(att for _, att in out)][-keep:] if keep > 0 else []
        return [res for res, _ in out]

    for fr in frames:
        if eng is None:
            eng = _engine_for(det, settings, fr.width, fr.height, policy)
        batch.append(fr)
        if len(batch) == eng.max_frames:
            yield from flush()
            batch = []
    if batch:
        yield from flush()


def run_downscale_baseline(frame: Frame, det: Detector, settings: PipelineSettings | None = None,
                           policy: MergePolicy | None = None, *, plan: GridPlan | None = None
                           ) -> FrameResult:
    if settings is None:
        settings = PipelineSettings(CropSettings(1), CropSettings(1))
    if plan is None:
        plan = GridPlan.build(frame.width, frame.height, settings)
    policy = policy or MergePolicy()
    crop = plan.downscale_crop
    t0 = time.perf_counter()
    if _is_yolo(det):
        from .engine import yolo_tagged

        try:
            tagged = yolo_tagged(det, frame, [crop])
        except Exception as exc:
            raise StageFailure("downscale", frame.frame_id) from exc
    else:
        (found,) = _detect_crops(frame, [crop], det, "downscale")
        rects = _project([(crop, d) for d in found], frame)
        tagged = [(crop.crop_id, Detection(r, d.class_label, d.confidence))
                  for d, r in zip(found, rects)]
    t1 = time.perf_counter()
    dets = finish_detections(tagged, plan.downscale_grid, policy, settings.min_confidence)
    t2 = time.perf_counter()
    timing = TimingProfile(final_eval_ms=(t1 - t0) * 1e3, postprocess_ms=(t2 - t1) * 1e3)
    return FrameResult(frame.frame_id, dets, 1, 1, timing)


def run_allcrops_baseline(frame: Frame, settings: PipelineSettings, det: Detector,
                          policy: MergePolicy | None = None, *, plan: GridPlan | None = None
                          ) -> FrameResult:
    if plan is None:
        plan = GridPlan.build(frame.width, frame.height, settings)
    policy = policy or MergePolicy()
    all_ids = frozenset(c.crop_id for c in plan.final_grid.crops)
    active = ActiveSet(plan.final_grid, all_ids)
    t0 = time.perf_counter()
    tagged = final_pass(frame, active, det)
    t1 = time.perf_counter()
    dets = finish_detections(tagged, plan.final_grid, policy, settings.min_confidence)
    t2 = time.perf_counter()
    timing = TimingProfile(final_eval_ms=(t1 - t0) * 1e3, postprocess_ms=(t2 - t1) * 1e3)
    return FrameResult(frame.frame_id, dets, len(all_ids), len(all_ids), timing)


def cut_tile_for(frame: Frame, crop: CropSpec) -> np.ndarray | None:
    """Reference `_tile_for` (pipeline.py:291-294), GPU cutter."""
    return None if frame.pixels is None else cut_tile(frame.pixels, crop)
