"""Ground-truth Detector plugins (API compatibility with the reference).

Same behaviour as the reference's ``mock_detect`` / ``SceneOracle`` / ``NoisyOracle``
(pkg/src/tilepipe/detector.py:99-220): a detector that answers from scene ground truth
instead of pixels. They are *plugins* behind the Detector boundary — the pipeline code
that calls them (tile cutting, projection, selection, NMS/merge) still runs on the GPU.
Used for stage-1 box injection and the reference's pipeline scenarios.
"""

from __future__ import annotations

import random
from collections.abc import Mapping, Sequence

import numpy as np

from .detector import Detection, Detector, DetectorProfile, GroundTruthObject
from .geometry import MODEL_SIDE, CropSpec, to_local


def mock_detect(crop: CropSpec, gt: Sequence[GroundTruthObject], visibility_threshold: float, *,
                min_tile_px: int = 8) -> list[Detection]:
    if not (0.0 < visibility_threshold <= 1.0):
        raise ValueError(f"visibility_threshold must be in (0, 1], got {visibility_threshold}")
    side = crop.global_rect.w
    found = []
    for obj in gt:
        seen = obj.rect.intersection(crop.global_rect)
        if seen is None:
            continue
        frac = seen.area / obj.rect.area
        if frac < visibility_threshold:
            continue
        too_small = (seen.w * MODEL_SIDE < min_tile_px * side or
                     seen.h * MODEL_SIDE < min_tile_px * side)
        if min_tile_px > 0 and too_small:
            continue
        found.append(Detection(to_local(seen, crop), obj.class_label, frac))
    found.sort(key=lambda d: -d.confidence)
    return found


class SceneOracle(Detector):
    def __init__(self, crops_by_id: Mapping[int, CropSpec],
                 gt_by_frame: Mapping[int, Sequence[GroundTruthObject]],
                 visibility_threshold: float = 0.3, *, min_tile_px: int = 8,
                 profile: DetectorProfile | None = None):
        if not (0.0 < visibility_threshold <= 1.0):
            raise ValueError(f"visibility_threshold must be in (0, 1], got {visibility_threshold}")
        if min_tile_px < 0:
            raise ValueError(f"min_tile_px must be >= 0, got {min_tile_px}")
        self._crops = dict(crops_by_id)
        self._gt = {fid: tuple(objs) for fid, objs in gt_by_frame.items()}
        self._vis = visibility_threshold
        self._min_px = min_tile_px
        if profile is None:
            profile = DetectorProfile(supported_classes=frozenset(
                o.class_label for objs in self._gt.values() for o in objs))
        self.profile = profile

    def detect(self, frame_id, crop_id, tile=None):
        if tile is not None:
            s = self.profile.input_side
            if not isinstance(tile, np.ndarray) or tile.shape != (s, s, 3):
                got = tile.shape if isinstance(tile, np.ndarray) else type(tile)
                raise ValueError(f"tile must be {s}x{s}x3, got {got}")
        if crop_id not in self._crops:
            raise ValueError(f"unknown crop_id: {crop_id}")
        dets = mock_detect(self._crops[crop_id], self._gt.get(frame_id, ()), self._vis,
                           min_tile_px=self._min_px)
        floor = self.profile.min_confidence
        if floor > 0.0:
            dets = [d for d in dets if d.confidence >= floor]
        if self.profile.supported_classes:
            dets = [d for d in dets if d.class_label in self.profile.supported_classes]
        return dets


class NoisyOracle(Detector):
    def __init__(self, base: Detector, miss_rate: float, seed: int = 0):
        if not (0.0 <= miss_rate <= 1.0):
            raise ValueError(f"miss_rate must be in [0, 1], got {miss_rate}")
        self._base, self._miss, self._seed = base, miss_rate, seed
        self.profile = base.profile

    def detect(self, frame_id, crop_id, tile=None):
        dets = self._base.detect(frame_id, crop_id, tile)
        if self._miss == 0.0:
            return dets
        rng = random.Random(f"{self._seed}:{frame_id}:{crop_id}")
        return [d for d in dets if rng.random() >= self._miss]
