"""Streaming scheduler and byte-stable results output (§8f-3).

``run_stream`` is the B200 counterpart of the reference's remote ``run_stream``
(pkg/src/tilepipe/distribution/client.py:294-377): frames in, ``FrameResult`` s out in
input order, a failure raises ``StreamAborted(cursor, completed, reason)`` carrying every
frame finished before it. Instead of attention workers over TCP it overlaps the host->
device copy of batch i+1 (pinned staging, dedicated copy stream) with the device
pipeline of batch i; ``TimingProfile`` keeps the reference meaning: ``io_ms`` is the
frame's share of the H2D copy, ``attention_wait_ms`` its share of stage 1, ...,
``per_worker`` names the device and its busy time.

``result_line`` / ``write_results`` reproduce the reference's canonical JSON lines
(frameio.py:227-258) byte for byte.
"""

from __future__ import annotations

import json
from collections.abc import Sequence
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import native
from .pipeline_types import FrameResult, PipelineSettings, TimingProfile
from .postprocess import MergePolicy


class StreamAborted(RuntimeError):
    """A stage failed mid-stream; carries the resume cursor and the completed results."""

    def __init__(self, cursor: int, completed: Sequence[FrameResult], reason: str):
        super().__init__(f"stream aborted at frame index {cursor}: {reason}")
        self.cursor = cursor
        self.completed = tuple(completed)


def run_stream(frames, settings: PipelineSettings, det=None,
               policy: MergePolicy | None = None, *, batch: int = 16, engine=None,
               io_threads: int = 8) -> list[FrameResult]:
    """Evaluate a frame stream on the GPU, in input order, with ingest overlapped.

    ``frames`` is an iterable of ``Frame`` s or a ``frameio.FrameSource`` (a directory of
    PPM files): source frames are read from disk straight into the pinned staging buffer
    on ``io_threads`` host threads while the GPU runs the previous batch."""
    from .engine import AttentionPipelineB200
    from .yolo import YoloB200Detector

    torch = native.require_cuda()
    if hasattr(frames, "load_into"):  # FrameSource
        source = frames
        W, H = source.width, source.height
        items = [(fid, (lambda out, i=i: source.load_into(i, out)))
                 for i, fid in enumerate(source.frame_ids)]
    else:
        frames = list(frames)
        if not frames:
            return []
        W, H = frames[0].width, frames[0].height
        items = [(fr.frame_id, _frame_loader(fr, W, H)) for fr in frames]
    if not items:
        return []
    if engine is None:
        det = det or YoloB200Detector()
        engine = AttentionPipelineB200(settings, W, H, max_frames=batch, seed=det.seed,
                                       threshold=det.threshold, policy=policy, head=det.head,
                                       precision=det.precision)
    B = engine.max_frames
    dev_name = f"cuda:{torch.cuda.current_device()}"
    stage = [torch.empty((B, H, W, 3), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    dev = [torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    copy_start = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    results: list[FrameResult] = []
    chunks = [items[i:i + B] for i in range(0, len(items), B)]
    pool = ThreadPoolExecutor(max_workers=max(1, io_threads))

    def stage_chunk(k: int) -> None:
        slot = k % 2
        chunk = chunks[k]
        copied[slot].synchronize()  # the H2D that last read this staging slot is done
        futs = [pool.submit(load, stage[slot][j].numpy()) for j, (_, load) in enumerate(chunk)]
        for f in futs:
            f.result()  # re-raises the first decode / dimension / missing-file error
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(used[slot])
            copy_start[slot].record(copy_stream)
            dev[slot][: len(chunk)].copy_(stage[slot][: len(chunk)], non_blocking=True)
            copied[slot].record(copy_stream)

    engine.reset_history(())
    ev_sets = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(2)]
    cursor = 0

    def emit(k: int, snap) -> None:
        """Results of batch k (its snapshot and events; the GPU may run batch k+1)."""
        nonlocal cursor
        slot = k % 2
        chunk = chunks[k]
        n = len(chunk)
        res = engine.results_from(snap, [fid for fid, _ in chunk])
        e = ev_sets[slot]
        t = [e[i].elapsed_time(e[i + 1]) / n for i in range(4)]
        io = copy_start[slot].elapsed_time(copied[slot]) / n
        timing = TimingProfile(io_ms=io, attention_wait_ms=t[0], client_processing_ms=t[1],
                               final_eval_ms=t[2], postprocess_ms=t[3],
                               per_worker=((dev_name, sum(t)),))
        for r, _ in res:
            results.append(FrameResult(r.frame_id, r.detections, r.active_count, r.total_count,
                                       timing))
        cursor += n

    try:
        stage_chunk(0)
        pending = None  # (batch index, snapshot) launched but not yet emitted
        for k in range(len(chunks)):
            slot = k % 2
            n = len(chunks[k])
            torch.cuda.current_stream().wait_event(copied[slot])
            engine.events = ev_sets[slot]
            engine.run_device(n, frames=dev[slot], timed=True)
            used[slot].record()
            snap = engine.snapshot(slot)
            if pending is not None:  # batch k-1 finishes while batch k is queued
                emit(*pending)
            pending = (k, snap)
            if k + 1 < len(chunks):
                try:  # host packing + H2D of the next batch overlap batch k on the GPU
                    stage_chunk(k + 1)
                except Exception:
                    emit(*pending)  # keep the finished batch's results, then abort
                    pending = None
                    raise
        if pending is not None:
            emit(*pending)
    except Exception as exc:
        raise StreamAborted(cursor, results, str(exc)) from exc
    finally:
        pool.shutdown(wait=True)
    return results


def _frame_loader(fr, W: int, H: int):
    """Staging callback for an in-memory Frame (validated when it is staged)."""
    def load(out) -> None:
        if fr.width != W or fr.height != H:
            raise ValueError(f"frame {fr.frame_id} is {fr.width}x{fr.height}, "
                             f"stream is {W}x{H}")
        if fr.pixels is None:
            raise ValueError(f"frame {fr.frame_id} has no pixels")
        out[...] = fr.pixels
    return load


def _detection_json(d) -> str:
    return '{"class":%s,"confidence":%.6f,"h":%d,"w":%d,"x":%d,"y":%d}' % (
        json.dumps(d.class_label), d.confidence, round(d.rect.h), round(d.rect.w),
        round(d.rect.x), round(d.rect.y))


def result_line(result: FrameResult) -> str:
    """Canonical one-line JSON of a frame's results (reference frameio.py:241-250)."""
    dets = ",".join(_detection_json(d) for d in result.detections)
    return '{"active_count":%d,"detections":[%s],"frame_id":%d,"total_count":%d}' % (
        result.active_count, dets, result.frame_id, result.total_count)


def write_results(results: Sequence[FrameResult], path) -> None:
    with open(path, "w", newline="\n") as fh:
        for r in results:
            fh.write(result_line(r))
            fh.write("\n")


__all__ = ["StreamAborted", "run_stream", "result_line", "write_results", "np"]
