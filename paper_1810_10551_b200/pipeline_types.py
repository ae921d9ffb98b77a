"""Pipeline value types (host side), mirroring the reference ``tilepipe/pipeline.py``:
PipelineSettings (:38-87), Frame (:90-114), AttentionModel (:117-123), ActiveSet
(:126-137), TimingProfile (:140-180), FrameResult (:183-197), StageFailure (:200-206),
GridPlan (:209-269). Same fields, defaults, validation and error types."""

from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

from .geometry import MODEL_SIDE, CropSettings, CropSpec, GridSpec, Rect, build_grid

PRESET_RE = re.compile(r"^\s*(\d+)\s*att\s*,\s*(\d+)\s*fin\s*,\s*(\d+)\s*over\s*$")


@dataclass(frozen=True)
class PipelineSettings:
    attention: CropSettings
    final: CropSettings
    attention_margin_px: int = 20
    temporal_window: int = 2
    min_confidence: float = 0.3

    def __post_init__(self):
        if self.final.rows < self.attention.rows:
            raise ValueError(f"final rows ({self.final.rows}) must be >= attention rows "
                             f"({self.attention.rows})")
        if self.attention_margin_px < 0:
            raise ValueError("attention_margin_px must be >= 0")
        if self.temporal_window < 1:
            raise ValueError("temporal_window must be >= 1")
        if not (0.0 <= self.min_confidence <= 1.0):
            raise ValueError("min_confidence must be in [0, 1]")

    @property
    def overlap_px(self) -> int | None:
        a, f = self.attention.overlap_px, self.final.overlap_px
        return a if a == f else None

    @classmethod
    def from_preset(cls, text: str, **overrides) -> "PipelineSettings":
        m = PRESET_RE.match(text)
        if m is None:
            raise ValueError(f"bad preset {text!r}, expected like '1 att, 3 fin, 50 over'")
        a, f, o = (int(g) for g in m.groups())
        return cls(attention=CropSettings(a, o), final=CropSettings(f, o), **overrides)

    def preset_name(self) -> str | None:
        o = self.overlap_px
        if o is None:
            return None
        return f"{self.attention.rows} att, {self.final.rows} fin, {o} over"


@dataclass(frozen=True)
class Frame:
    frame_id: int
    width: int
    height: int
    pixels: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError(f"frame must be >= 1x1, got {self.width}x{self.height}")
        if self.pixels is not None and tuple(self.pixels.shape) != (self.height, self.width, 3):
            raise ValueError(f"pixels shape {tuple(self.pixels.shape)} does not match "
                             f"{self.height}x{self.width}x3")


@dataclass(frozen=True)
class AttentionModel:
    frame_id: int
    boxes: tuple[Rect, ...]
    source_window: tuple[int, ...]


@dataclass(frozen=True)
class ActiveSet:
    grid: GridSpec
    active_ids: frozenset[int]

    def __post_init__(self):
        known = {c.crop_id for c in self.grid.crops}
        bad = set(self.active_ids) - known
        if bad:
            raise ValueError(f"active ids not in grid: {sorted(bad)}")


@dataclass(frozen=True)
class TimingProfile:
    COLUMNS = ("io_ms", "attention_wait_ms", "client_processing_ms", "transfer_ms",
               "final_eval_ms", "postprocess_ms")

    io_ms: float = 0.0
    attention_wait_ms: float = 0.0
    client_processing_ms: float = 0.0
    transfer_ms: float = 0.0
    final_eval_ms: float = 0.0
    postprocess_ms: float = 0.0
    per_worker: tuple[tuple[str, float], ...] = ()

    def __post_init__(self):
        for name in self.COLUMNS:
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        for endpoint, busy in self.per_worker:
            if busy < 0:
                raise ValueError(f"busy_ms for {endpoint} must be >= 0")

    @property
    def total_ms(self) -> float:
        return sum(getattr(self, name) for name in self.COLUMNS)


@dataclass(frozen=True)
class FrameResult:
    frame_id: int
    detections: tuple
    active_count: int
    total_count: int
    timing: TimingProfile

    def __post_init__(self):
        if self.active_count > self.total_count:
            raise ValueError(f"active_count {self.active_count} > total_count {self.total_count}")


class StageFailure(RuntimeError):
    def __init__(self, stage: str, frame_id: int):
        super().__init__(f"{stage} stage failed on frame {frame_id}")
        self.stage = stage
        self.frame_id = frame_id


@dataclass(frozen=True)
class GridPlan:
    """Unified crop ids: attention 0..A-1, final A..A+F-1, downscale pseudo-crop A+F."""

    frame_w: int
    frame_h: int
    settings: PipelineSettings
    attention_grid: GridSpec
    final_grid: GridSpec
    downscale_crop: CropSpec

    @classmethod
    def build(cls, frame_w: int, frame_h: int, settings: PipelineSettings) -> "GridPlan":
        att = build_grid(frame_w, frame_h, settings.attention)
        fin = build_grid(frame_w, frame_h, settings.final, id_base=len(att.crops))
        side = max(frame_w, frame_h)
        down = CropSpec(len(att.crops) + len(fin.crops), 0, 0, Rect(0, 0, side, side),
                        side / MODEL_SIDE)
        return cls(frame_w, frame_h, settings, att, fin, down)

    @property
    def downscale_id(self) -> int:
        return self.downscale_crop.crop_id

    @property
    def downscale_grid(self) -> GridSpec:
        side = int(self.downscale_crop.global_rect.w)
        return GridSpec(self.frame_w, self.frame_h, CropSettings(rows=1, overlap_px=0), side, 1, 1,
                        (self.downscale_crop,))

    def crop_by_id(self, crop_id: int) -> CropSpec:
        if crop_id == self.downscale_crop.crop_id:
            return self.downscale_crop
        if crop_id < len(self.attention_grid.crops):
            return self.attention_grid.crop_by_id(crop_id)
        return self.final_grid.crop_by_id(crop_id)

    def crops_by_id(self) -> dict[int, CropSpec]:
        out = {c.crop_id: c for c in self.attention_grid.crops}
        out.update((c.crop_id, c) for c in self.final_grid.crops)
        out[self.downscale_crop.crop_id] = self.downscale_crop
        return out
