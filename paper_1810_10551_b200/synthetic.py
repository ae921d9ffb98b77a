"""Deterministic synthetic scenes (input generator for tests and bench).

Behaviour-identical restatement of the reference generator
(pkg/src/tilepipe/synthetic.py:24-196): same seeding string, same RNG call order,
same bounce rule and flat-colour renderer, so a scene spec yields the very same
ground truth and pixels on a GPU box where the reference is not installed. Pinned
by tests/test_oracle_golden.py against GT and render hashes from the reference.
``render_frames_device`` draws the same rectangles directly into a device batch
 so bench frames need not cross PCIe.
"""

from __future__ import annotations

import random
import zlib
from dataclasses import dataclass

import numpy as np

from .detector import GroundTruthObject
from .geometry import Rect

SCENE_KINDS = ("sparse", "dense", "small", "mixed", "straddle")
DEFAULT_COUNTS = {"sparse": 4, "dense": 24, "small": 8, "mixed": 10, "straddle": 5}
SMALL_SIZE = (0.014, 0.021)
NORMAL_SIZE = (0.037, 0.093)
PALETTE = {"person": (200, 60, 60), "car": (60, 120, 200), "bus": (220, 180, 40)}
BACKGROUND = (24, 24, 24)


def class_color(label: str) -> tuple[int, int, int]:
    if label in PALETTE:
        return PALETTE[label]
    c = zlib.crc32(label.encode("utf-8"))
    return (96 + (c & 0x7F), 96 + ((c >> 8) & 0x7F), 96 + ((c >> 16) & 0x7F))


@dataclass(frozen=True)
class SceneSpec:
    kind: str
    width: int
    height: int
    frame_count: int
    seed: int = 0
    object_count: int | None = None

    def __post_init__(self):
        if self.kind not in SCENE_KINDS:
            raise ValueError(f"kind must be one of {SCENE_KINDS}, got {self.kind!r}")
        if self.width < 64 or self.height < 64:
            raise ValueError("frame must be at least 64x64")
        if self.frame_count < 1:
            raise ValueError("frame_count must be >= 1")
        if self.object_count is not None and self.object_count < 1:
            raise ValueError("object_count must be >= 1")


class _Body:
    __slots__ = ("label", "w", "h", "x", "y", "vx", "vy", "oid")

    def __init__(self, label, w, h, x, y, vx, vy, oid):
        self.label, self.w, self.h = label, w, h
        self.x, self.y, self.vx, self.vy, self.oid = x, y, vx, vy, oid

    def advance(self, fw, fh):
        self.x += self.vx
        self.y += self.vy
        if self.x < 0 or self.x + self.w > fw:
            self.vx = -self.vx
            self.x = min(max(self.x, 0), fw - self.w)
        if self.y < 0 or self.y + self.h > fh:
            self.vy = -self.vy
            self.y = min(max(self.y, 0), fh - self.h)


def _side(rng, lohi, min_dim):
    return max(4, round(rng.uniform(*lohi) * min_dim))


def _bodies(spec: SceneSpec, rng: random.Random) -> list[_Body]:
    n = spec.object_count or DEFAULT_COUNTS[spec.kind]
    min_dim = min(spec.width, spec.height)
    speed = max(1, min_dim // 360)
    out = []
    for i in range(n):
        if spec.kind == "small" or (spec.kind == "mixed" and i % 2 == 0):
            lohi = SMALL_SIZE
        else:
            lohi = NORMAL_SIZE
        w = _side(rng, lohi, min_dim)
        h = _side(rng, lohi, min_dim)
        label = rng.choice(("person", "car"))
        if spec.kind == "straddle":
            label = "person"
            h = max(h, round(0.12 * min_dim))
            border = spec.height * (1 + i % 2) // 3
            x = rng.uniform(0, spec.width - w)
            y = min(max(border - h / 2, 0), spec.height - h)
        else:
            x = rng.uniform(0, spec.width - w)
            y = rng.uniform(0, spec.height - h)
        vx = rng.choice((-3, -2, -1, 1, 2, 3)) * speed
        vy = rng.choice((-3, -2, -1, 1, 2, 3)) * speed
        out.append(_Body(label, w, h, round(x), round(y), vx, vy, f"obj{i}"))
    return out


def generate_scene(spec: SceneSpec) -> dict[int, list[GroundTruthObject]]:
    rng = random.Random(f"{spec.kind}:{spec.width}x{spec.height}:{spec.seed}")
    bodies = _bodies(spec, rng)
    scene = {}
    for fid in range(spec.frame_count):
        scene[fid] = [GroundTruthObject(Rect(round(b.x), round(b.y), b.w, b.h), b.label, b.oid)
                      for b in bodies]
        for b in bodies:
            b.advance(spec.width, spec.height)
    return scene


CLIP_KINDS = ("sparse", "dense", "mixed")


def bench_clip(width: int, height: int, n_frames: int = 300, seed: int = 0
               ) -> list[list[GroundTruthObject]]:
    """The measurement clip of BASELINE configs[1]/[3]: n_frames // 3 frames
    each of a sparse, a dense and a mixed scene (generate_scene, this seed), in that
    order; clip frame i of the middle third is scene frame i - n_frames // 3, etc."""
    per = max(1, n_frames // len(CLIP_KINDS))
    out = []
    for kind in CLIP_KINDS:
        gt = generate_scene(SceneSpec(kind, width, height, per, seed=seed))
        out += [gt[i] for i in range(per)]
    return out


def _boxes(width, height, objects):
    for o in objects:
        x0, y0 = max(0, round(o.rect.x)), max(0, round(o.rect.y))
        x1, y1 = min(width, round(o.rect.x2)), min(height, round(o.rect.y2))
        if x1 > x0 and y1 > y0:
            yield x0, y0, x1, y1, class_color(o.class_label)


def render_frame(width: int, height: int, objects, background=BACKGROUND) -> np.ndarray:
    img = np.empty((height, width, 3), dtype=np.uint8)
    img[:, :] = background
    for x0, y0, x1, y1, col in _boxes(width, height, objects):
        img[y0:y1, x0:x1] = col
    return img


def render_frames_device(width, height, objects_per_frame, out=None, background=BACKGROUND):
    """Render a batch of frames straight into a CUDA uint8 [n, H, W, 3] tensor with the
    tp_render_frames kernel. Same painter's-order fills as render_frame, so the bytes are
    identical; only the rectangle list crosses PCIe."""
    from . import native

    torch = native.require_cuda()
    n = len(objects_per_frame)
    if out is None:
        out = torch.empty((n, height, width, 3), dtype=torch.uint8, device="cuda")
    if n == 0:
        return out
    boxes = [list(_boxes(width, height, objs)) for objs in objects_per_frame]
    m = max(1, max(len(b) for b in boxes))
    if m > 64:
        raise ValueError("at most 64 rectangles per frame")
    rects = np.zeros((n, m, 4), dtype=np.int32)
    cols = np.zeros((n, m, 3), dtype=np.uint8)
    cnt = np.zeros(n, dtype=np.int32)
    for i, bl in enumerate(boxes):
        cnt[i] = len(bl)
        for k, (x0, y0, x1, y1, col) in enumerate(bl):
            rects[i, k] = (x0, y0, x1, y1)
            cols[i, k] = col
    bg = background[0] | (background[1] << 8) | (background[2] << 16)
    r_d, c_d, n_d = (torch.from_numpy(a).cuda() for a in (rects, cols, cnt))
    native.call("tp_render_frames", native.ptr(r_d), native.ptr(c_d), native.ptr(n_d), n, m,
                height, width, bg, native.ptr(out), native.stream_handle())
    return out
