"""NMS and cross-border merging (reference-compatible API, GPU execution).

Mirrors ``tilepipe/postprocess.py``: ``MergePolicy`` (:21-51), ``nms_keep_indices``
(:54-73), ``nms`` (:76-78), ``merge_split`` (:127-163) and ``postprocess`` (:166-187).
Every call runs the K7 kernel (``tp_postprocess``, csrc/tp_post.cu) — one CTA per
frame, fp64 IoU with the reference op order, so keep-sets and merges are bit-exact.
"""

from __future__ import annotations

from collections.abc import Mapping, Sequence
from dataclasses import dataclass, field

import numpy as np

from . import native
from .detector import Detection
from .geometry import GridSpec, Rect

AXIS_RULES = ("vertical", "horizontal", "both")
MAX_ENTRIES = 2048  # per frame, kernel shared-memory capacity


@dataclass(frozen=True)
class MergePolicy:
    nms_iou: float = 0.45
    vertical_gap_px: int = 40
    horizontal_alignment_tolerance_px: int = 30
    mergeable_classes: Mapping[str, str] = field(default_factory=lambda: {"person": "vertical"})
    merge_before_nms: bool = False
    nms_per_crop: bool = False

    def __post_init__(self):
        if not (0.0 < self.nms_iou < 1.0):
            raise ValueError(f"nms_iou must be in (0, 1), got {self.nms_iou}")
        if self.vertical_gap_px < 0 or self.horizontal_alignment_tolerance_px < 0:
            raise ValueError("merge gaps must be >= 0")
        for label, rule in self.mergeable_classes.items():
            if rule not in AXIS_RULES:
                raise ValueError(f"unknown merge rule {rule!r} for class {label!r}")
        object.__setattr__(self, "mergeable_classes", dict(self.mergeable_classes))


class LabelTable:
    """Class label <-> small integer id used by the kernels."""

    def __init__(self, labels=()):
        self.ids: dict[str, int] = {}
        self.names: list[str] = []
        for lab in labels:
            self.id(lab)

    def id(self, label: str) -> int:
        k = self.ids.get(label)
        if k is None:
            k = len(self.names)
            if k >= native.TP_MAX_CLASSES:
                raise ValueError(f"more than {native.TP_MAX_CLASSES} distinct class labels")
            self.ids[label] = k
            self.names.append(label)
        return k


def make_policy_struct(policy: MergePolicy, labels: LabelTable, grid_cols: int, n_cells: int,
                       min_conf: float = -1.0, do_nms: bool = True, do_merge: bool = True):
    if n_cells > 256:
        raise ValueError(f"grid has {n_cells} cells; the merge kernel supports up to 256")
    p = native.PostPolicy()
    p.nms_iou = float(policy.nms_iou)
    p.gap_px = float(policy.vertical_gap_px)
    p.tol_px = float(policy.horizontal_alignment_tolerance_px)
    p.min_conf = float(min_conf)
    p.merge_before_nms = int(policy.merge_before_nms)
    p.nms_per_crop = int(policy.nms_per_crop)
    p.do_nms = int(do_nms)
    p.do_merge = int(do_merge)
    p.grid_cols = int(grid_cols)
    p.n_cells = int(n_cells)
    for label, rule in policy.mergeable_classes.items():
        if label in labels.ids:
            p.class_rule[labels.ids[label]] = native.RULES[rule]
    return p


def _all_int(dets) -> bool:
    return all(isinstance(v, int) for d in dets for v in (d.rect.x, d.rect.y, d.rect.w, d.rect.h))


def run_postprocess_kernel(tagged, cells, policy_struct, labels: LabelTable):
    """One-frame launch. tagged: [(crop_id, Detection)], cells: per-entry cell index.
    Returns (out records ndarray[PDET_DTYPE], keep indices list)."""
    torch = native.require_cuda()
    n = len(tagged)
    if n > MAX_ENTRIES:
        raise ValueError(f"{n} detections in one frame exceed the kernel capacity {MAX_ENTRIES}")
    rec = np.zeros(max(n, 1), dtype=native.PDET_DTYPE)
    for i, ((cid, d), cell) in enumerate(zip(tagged, cells)):
        rec[i] = (d.rect.x, d.rect.y, d.rect.w, d.rect.h, d.confidence, labels.id(d.class_label),
                  cell, cid, i)
    cap = max(n, 1)
    dev_in = torch.from_numpy(rec.view(np.uint8)).cuda()
    dev_out = torch.empty_like(dev_in)
    counts = torch.tensor([n], dtype=torch.int32, device="cuda")
    out_counts = torch.zeros(1, dtype=torch.int32, device="cuda")
    keep = torch.zeros(cap, dtype=torch.int32, device="cuda")
    keep_n = torch.zeros(1, dtype=torch.int32, device="cuda")
    native.call("tp_postprocess", native.ptr(dev_in), native.ptr(counts), 1, cap,
                ctypes_ref(policy_struct), native.ptr(dev_out), native.ptr(out_counts),
                native.ptr(keep), native.ptr(keep_n), native.stream_handle())
    m = int(out_counts.item())
    out = dev_out.cpu().numpy().view(native.PDET_DTYPE)[:m].copy()
    k = int(keep_n.item())
    return out, [int(v) for v in keep[:k].cpu().numpy()]


def ctypes_ref(struct):
    import ctypes

    return ctypes.cast(ctypes.pointer(struct), ctypes.c_void_p)


def records_to_detections(rec, labels: LabelTable, as_int: bool) -> list[Detection]:
    out = []
    for r in rec:
        vals = [float(r["x"]), float(r["y"]), float(r["w"]), float(r["h"])]
        if as_int:
            vals = [int(v) for v in vals]
        out.append(Detection(Rect(*vals), labels.names[int(r["cls"])], float(r["conf"])))
    return out


def nms_keep_indices(dets: Sequence[Detection], iou_threshold: float) -> list[int]:
    if not (0.0 < iou_threshold < 1.0):
        raise ValueError(f"iou_threshold must be in (0, 1), got {iou_threshold}")
    if not dets:
        return []
    labels = LabelTable(d.class_label for d in dets)
    pol = make_policy_struct(MergePolicy(nms_iou=iou_threshold, mergeable_classes={}), labels,
                             1, 1, do_nms=True, do_merge=False)
    _, keep = run_postprocess_kernel([(0, d) for d in dets], [0] * len(dets), pol, labels)
    return keep


def nms(dets: Sequence[Detection], iou_threshold: float) -> list[Detection]:
    return [dets[i] for i in nms_keep_indices(dets, iou_threshold)]


def _cells_for(tagged, grid: GridSpec):
    return [grid.crop_by_id(cid).row * grid.cols + grid.crop_by_id(cid).col for cid, _ in tagged]


def merge_split(tagged: Sequence[tuple[int, Detection]], grid: GridSpec, policy: MergePolicy
                ) -> list[Detection]:
    if not tagged:
        return []
    labels = LabelTable(d.class_label for _, d in tagged)
    cells = _cells_for(tagged, grid)
    pol = make_policy_struct(policy, labels, grid.cols, grid.rows * grid.cols, do_nms=False,
                             do_merge=True)
    rec, _ = run_postprocess_kernel(list(tagged), cells, pol, labels)
    return records_to_detections(rec, labels, _all_int([d for _, d in tagged]))


def postprocess(tagged: Sequence[tuple[int, Detection]], grid: GridSpec, policy: MergePolicy,
                min_confidence: float | None = None) -> list[Detection]:
    """NMS + merge chain (+ optional final confidence filter, fused on the GPU)."""
    if not tagged:
        return []
    labels = LabelTable(d.class_label for _, d in tagged)
    cells = _cells_for(tagged, grid)
    pol = make_policy_struct(policy, labels, grid.cols, grid.rows * grid.cols,
                             min_conf=-1.0 if min_confidence is None else min_confidence)
    rec, _ = run_postprocess_kernel(list(tagged), cells, pol, labels)
    return records_to_detections(rec, labels, _all_int([d for _, d in tagged]))
