"""Detector boundary (host types) and the GPU tile cutter.

Mirrors the reference ``tilepipe/detector.py``: ``Detection`` (:23-40),
``GroundTruthObject`` (:43-56), ``DetectorProfile`` (:57-74), the ``Detector`` plugin
ABC (:77-96) and ``cut_tile`` (:223-247). ``cut_tile`` here runs the K2 gather
kernel (``tp_gather_tiles``) — nearest mode is bit-exact with the reference cutter.
The YOLO v2 implementation of the boundary is ``yolo.YoloB200Detector``.
"""

from __future__ import annotations

from abc import ABC, abstractmethod
from dataclasses import dataclass, field

import numpy as np

from . import native
from .geometry import MODEL_SIDE, CropSpec, Rect


@dataclass(frozen=True)
class Detection:
    rect: Rect
    class_label: str
    confidence: float

    def __post_init__(self):
        if not self.class_label:
            raise ValueError("class_label must be non-empty")
        if not (0.0 <= self.confidence <= 1.0):
            raise ValueError(f"confidence must be in [0, 1], got {self.confidence}")


@dataclass(frozen=True)
class GroundTruthObject:
    rect: Rect
    class_label: str
    object_id: str

    def __post_init__(self):
        if not self.class_label:
            raise ValueError("class_label must be non-empty")
        if not self.object_id:
            raise ValueError("object_id must be non-empty")


@dataclass(frozen=True)
class DetectorProfile:
    input_side: int = MODEL_SIDE
    min_confidence: float = 0.0
    supported_classes: frozenset[str] = field(default_factory=frozenset)

    def __post_init__(self):
        if self.input_side < 1:
            raise ValueError(f"input_side must be >= 1, got {self.input_side}")
        if not (0.0 <= self.min_confidence <= 1.0):
            raise ValueError(f"min_confidence must be in [0, 1], got {self.min_confidence}")


class Detector(ABC):
    """Plugin interface: detect(frame_id, crop_id, tile) -> crop-local detections in
    608 space, sorted by descending confidence. Implementations must be safe for
    concurrent calls or document that calls are serialised."""

    profile: DetectorProfile

    @abstractmethod
    def detect(self, frame_id: int, crop_id: int, tile: np.ndarray | None = None
               ) -> list[Detection]:
        ...


def _check_pixels(pixels) -> None:
    if not isinstance(pixels, np.ndarray) or pixels.ndim != 3 or pixels.shape[2] != 3:
        shape = getattr(pixels, "shape", type(pixels))
        raise ValueError(f"pixels must be HxWx3, got shape {shape}")


def cut_tiles(pixels, crops, mode: str = "nearest"):
    """Cut many crops of one frame on the GPU. ``pixels``: HxWx3 uint8 numpy array or a
    CUDA uint8 tensor; ``crops``: CropSpec list or (x, y, side) tuples. Returns a CUDA
    uint8 tensor [n, 608, 608, 3]."""
    torch = native.require_cuda()
    if isinstance(pixels, np.ndarray):
        _check_pixels(pixels)
        dev = torch.from_numpy(np.ascontiguousarray(pixels, dtype=np.uint8)).cuda()
    else:
        dev = pixels
    H, W = int(dev.shape[0]), int(dev.shape[1])
    jobs = np.zeros(len(crops), dtype=native.JOB_DTYPE)
    for i, c in enumerate(crops):
        if isinstance(c, CropSpec):
            x, y, side = int(c.global_rect.x), int(c.global_rect.y), int(c.global_rect.w)
            jobs[i]["crop_id"] = c.crop_id
        else:
            x, y, side = (int(v) for v in c)
        jobs[i]["x"], jobs[i]["y"], jobs[i]["side"] = x, y, side
    out = torch.empty((len(crops), MODEL_SIDE, MODEL_SIDE, 3), dtype=torch.uint8, device="cuda")
    if len(crops) == 0:
        return out
    jobs_dev = torch.from_numpy(jobs.view(np.uint8)).cuda()
    native.call("tp_gather_tiles", native.ptr(dev), 0, H, W, native.ptr(jobs_dev), len(crops), None,
                native.RESAMPLE[mode], native.ptr(out), None, 0, native.stream_handle())
    return out


def cut_tile(pixels: np.ndarray, crop: CropSpec, input_side: int = MODEL_SIDE,
             mode: str = "nearest") -> np.ndarray:
    """Reference-compatible tile cutter (GPU): crop -> input_side^2 uint8 HWC tile."""
    _check_pixels(pixels)
    if input_side != MODEL_SIDE:
        raise ValueError(f"the B200 gather kernel produces {MODEL_SIDE}^2 tiles only")
    return cut_tiles(pixels, [crop], mode)[0].cpu().numpy()
