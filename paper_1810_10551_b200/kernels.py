"""Thin typed wrappers over the C-ABI entry points (device tensors in, device tensors out).

Nothing here computes on the host; every function is one or more stream-ordered
launches of the native library.
"""

from __future__ import annotations

import numpy as np

from . import native
from .geometry import MODEL_SIDE

MAX_PER_TILE = 19 * 19 * 5  # every (cell, anchor) can be kept


def jobs_tensor(rows):
    """rows: iterable of (frame, crop_id, x, y, side, cell) -> CUDA uint8 [n*32] job table."""
    torch = native.require_cuda()
    rows = list(rows)
    arr = np.zeros(max(1, len(rows)), dtype=native.JOB_DTYPE)
    for i, (f, cid, x, y, side, cell) in enumerate(rows):
        arr[i] = (f, cid, x, y, side, cell, 0, 0)
    return torch.from_numpy(arr.view(np.uint8)).cuda()


def gather(frames_dev, frame_stride: int, H: int, W: int, jobs_dev, n_jobs: int, mode: str,
           out_u8=None, out_act_ptr: int = 0, n_jobs_dev=None, stream=None, dtype: str = "bf16"):
    native.call("tp_gather_tiles", native.ptr(frames_dev), int(frame_stride), H, W,
                native.ptr(jobs_dev), int(n_jobs), native.ptr(n_jobs_dev), native.RESAMPLE[mode],
                native.ptr(out_u8), out_act_ptr or None, native.DTYPES[dtype],
                native.stream_handle(stream))


def decode(net, n_tiles: int, jobs_dev, frame_w: int, frame_h: int, thresh: float, out, counts,
           n_tiles_dev=None, max_per_tile: int = MAX_PER_TILE, stream=None):
    from .yolo import ANCHORS

    anchors = np.ascontiguousarray(ANCHORS, dtype=np.float32)
    native.call("tp_region_decode", net.head_ptr, net.head_cstride, int(n_tiles),
                native.ptr(n_tiles_dev), native.ptr(jobs_dev), int(frame_w), int(frame_h),
                float(thresh), anchors.ctypes.data, native.ptr(out), int(max_per_tile),
                native.ptr(counts), native.stream_handle(stream))


def alloc_dets(n_tiles: int, max_per_tile: int = MAX_PER_TILE):
    torch = native.require_cuda()
    out = torch.empty(max(1, n_tiles) * max_per_tile * native.DET_DTYPE.itemsize,
                      dtype=torch.uint8, device="cuda")
    counts = torch.zeros(max(1, n_tiles), dtype=torch.int32, device="cuda")
    return out, counts


def dets_to_host(out, counts, n_tiles: int, max_per_tile: int = MAX_PER_TILE):
    c = counts[:n_tiles].cpu().numpy()
    recs = out[: n_tiles * max_per_tile * native.DET_DTYPE.itemsize].cpu().numpy().view(
        native.DET_DTYPE).reshape(n_tiles, max_per_tile)
    return recs, c


def detect_tiles_device(net, tiles_dev, thresh: float):
    """Run YOLO on [n,608,608,3] uint8 device tiles (n <= net.max_tiles).

    The tiles are fed through the gather kernel as identity crops of a 608x608 "frame"
    so the layer-0 input normalisation is the same kernel as the pipeline's."""
    n = int(tiles_dev.shape[0])
    jobs = jobs_tensor((i, 0, 0, 0, MODEL_SIDE, 0) for i in range(n))
    gather(tiles_dev, MODEL_SIDE * MODEL_SIDE * 3, MODEL_SIDE, MODEL_SIDE, jobs, n,
           "nearest", out_act_ptr=net.input_ptr, dtype=net.dtype)
    net.forward(n)
    out, counts = alloc_dets(n)
    decode(net, n, jobs, MODEL_SIDE, MODEL_SIDE, thresh, out, counts)
    return dets_to_host(out, counts, n)


def project_rects(local_rects, crops_xyside, frame_w=None, frame_h=None):
    """to_global on the GPU for host detector output. local: [n,4] float64, crops [n,3]."""
    torch = native.require_cuda()
    n = len(local_rects)
    if n == 0:
        return np.zeros((0, 4), dtype=np.int64)
    loc = torch.from_numpy(np.ascontiguousarray(local_rects, dtype=np.float64)).cuda()
    cr = torch.from_numpy(np.ascontiguousarray(crops_xyside, dtype=np.int32)).cuda()
    out = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    fw = -1 if frame_w is None else int(frame_w)
    fh = -1 if frame_h is None else int(frame_h)
    native.call("tp_project_rects", native.ptr(loc), native.ptr(cr), n, fw, fh, native.ptr(out),
                native.stream_handle())
    return out.cpu().numpy().astype(np.int64)


def select(boxes_slots, window: int, crops_rects, crop_id_base: int, margin: float, frame_w,
           frame_h, n_frames: int | None = None, max_merged: int = 512):
    """merge_temporal + select_active on the GPU for host box lists.

    boxes_slots: list (oldest first) of [(x,y,w,h)] lists; returns per frame
    (active ids, merged boxes) for frames window-1 .. len-1 (slot-relative)."""
    torch = native.require_cuda()
    n_slots = len(boxes_slots)
    if n_frames is None:
        n_frames = n_slots - (window - 1)
    max_boxes = max(1, max((len(b) for b in boxes_slots), default=1))
    arr = np.zeros((n_slots, max_boxes, 4), dtype=np.float64)
    cnt = np.zeros(n_slots, dtype=np.int32)
    for s, bl in enumerate(boxes_slots):
        cnt[s] = len(bl)
        for k, b in enumerate(bl):
            arr[s, k] = b
    n_crops = len(crops_rects)
    words = (n_crops + 31) // 32
    boxes_d = torch.from_numpy(arr).cuda()
    cnt_d = torch.from_numpy(cnt).cuda()
    crops_d = torch.from_numpy(np.ascontiguousarray(crops_rects, dtype=np.float64)).cuda()
    mask = torch.zeros((n_frames, words), dtype=torch.int32, device="cuda")
    ids = torch.zeros((n_frames, n_crops), dtype=torch.int32, device="cuda")
    acnt = torch.zeros(n_frames, dtype=torch.int32, device="cuda")
    merged = torch.zeros((n_frames, max_merged, 4), dtype=torch.float64, device="cuda")
    mcnt = torch.zeros(n_frames, dtype=torch.int32, device="cuda")
    native.call("tp_select_active", native.ptr(boxes_d), native.ptr(cnt_d), max_boxes, n_frames,
                window, native.ptr(crops_d), n_crops, crop_id_base, float(margin), float(frame_w),
                float(frame_h), native.ptr(mask), words, native.ptr(ids), native.ptr(acnt),
                native.ptr(merged), native.ptr(mcnt), max_merged, native.stream_handle())
    ids_h, acnt_h = ids.cpu().numpy(), acnt.cpu().numpy()
    merged_h, mcnt_h = merged.cpu().numpy(), mcnt.cpu().numpy()
    res = []
    for f in range(n_frames):
        if mcnt_h[f] > max_merged:
            raise ValueError(f"more than {max_merged} merged attention boxes")
        res.append(([int(v) for v in ids_h[f, : acnt_h[f]]],
                    [tuple(float(v) for v in merged_h[f, k]) for k in range(mcnt_h[f])]))
    return res
