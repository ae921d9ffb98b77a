"""Streaming scheduler and byte-stable results output (§8f-3).

``run_stream`` is the B200 counterpart of the reference's remote ``run_stream``
(pkg/src/tilepipe/distribution/client.py:294-377): frames in, ``FrameResult`` s out in
input order, a failure raises ``StreamAborted(cursor, completed, reason)`` carrying every
frame finished before it.

Schedule (the reference's attention pipelining, client.py:312-338, on one device):
  * ingest — batch k+1's frames are read / staged on host threads and copied H2D on a
    copy stream while the GPU runs batch k (pinned caller frames are copied directly);
  * attention look-ahead — stage 1 of batch k+1 runs on its own stream and its own
    YoloNet workspace while batch k's selection, stage 2 and postprocess run on the main
    stream, exactly as the reference's attention workers compute frame t+1 while the
    final workers finish frame t;
  * results — batch k's records are copied to pinned host memory on the stream and
    turned into FrameResults while the GPU runs batch k+1.

``TimingProfile`` keeps the reference meaning per frame (batch values / batch size):
``attention_wait_ms`` is only the part of stage 1 that was NOT hidden behind the previous
batch's final stage (the whole stage 1 for the first batch, or without look-ahead),
``client_processing_ms`` the selection, ``final_eval_ms`` stage 2, ``postprocess_ms``
NMS + merge, ``io_ms`` the H2D copy, ``per_worker`` = ((device, busy_ms),) with busy_ms
the device's stage-2 time (final_eval_ms equals the largest busy_ms, as in
client.py:202). The multi-GPU version (frame shards, NCCL result gather) is
``distributed.run_stream_sharded``, built on the same driver.

``result_line`` / ``write_results`` reproduce the reference's canonical JSON lines
(frameio.py:227-258) byte for byte.
"""

from __future__ import annotations

import json
import os
import sys
import time
from collections.abc import Sequence
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import native
from .pipeline_types import FrameResult, PipelineSettings, TimingProfile
from .postprocess import MergePolicy

N_DEV_SLOTS = 3  # device frame buffers: batch k+2's H2D never waits for batch k+1


class StreamAborted(RuntimeError):
    """A stage failed mid-stream; carries the resume cursor and the completed results."""

    def __init__(self, cursor: int, completed: Sequence[FrameResult], reason: str):
        super().__init__(f"stream aborted at frame index {cursor}: {reason}")
        self.cursor = cursor
        self.completed = tuple(completed)


def stream_items(frames):
    """(width, height, items) for a Frame iterable or a frameio.FrameSource; an item is
    (frame_id, load(out_np) callback, pinned source tensor or None)."""
    torch = native.require_cuda()
    if hasattr(frames, "load_into"):  # FrameSource: read straight into pinned staging
        source = frames
        items = [(fid, (lambda out, i=i: source.load_into(i, out)), None)
                 for i, fid in enumerate(source.frame_ids)]
        return source.width, source.height, items
    frames = list(frames)
    if not frames:
        return 0, 0, []
    W, H = frames[0].width, frames[0].height
    items = []
    for fr in frames:
        src = None
        px = fr.pixels
        if (px is not None and fr.width == W and fr.height == H and isinstance(px, np.ndarray)
                and px.flags.c_contiguous and px.shape == (H, W, 3)):
            t = torch.from_numpy(px)
            if t.is_pinned():  # caller-pinned frame: DMA it directly, no staging copy
                src = t
        items.append((fr.frame_id, _frame_loader(fr, W, H), src))
    return W, H, items


class StreamDriver:
    """One engine, a list of batches of items, the ingest / look-ahead / results
    overlap described in the module docstring. `sink` turns finished batches into
    results (default: FrameResults of this device)."""

    def __init__(self, engine, W: int, H: int, *, io_threads: int = 8, lookahead: bool = True):
        torch = native.require_cuda()
        self.torch = torch
        self.engine = engine
        self.W, self.H = W, H
        B = engine.max_frames
        self.B = B
        self.lookahead = lookahead and engine.net1 is not engine.net
        self.stage = [torch.empty((B, H, W, 3), dtype=torch.uint8, pin_memory=True)
                      for _ in range(2)]
        self.dev = [torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda")
                    for _ in range(N_DEV_SLOTS)]
        self.copy_stream = torch.cuda.Stream()
        self.att_stream = torch.cuda.Stream() if self.lookahead else None
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        self.copied = [ev() for _ in range(N_DEV_SLOTS)]
        self.copy_start = [ev() for _ in range(N_DEV_SLOTS)]
        self.staged = [torch.cuda.Event() for _ in range(2)]  # H2D done reading stage slot
        self.used = [torch.cuda.Event() for _ in range(N_DEV_SLOTS)]
        self.att_ev = [(ev(), ev()) for _ in range(3)]  # k % 3: k+2 is queued before k emits
        self.fin_ev = [[ev() for _ in range(5)] for _ in range(2)]
        self.fin_end = [ev() for _ in range(3)]  # batch k -> k % 3 (read two batches later)
        self.pool = ThreadPoolExecutor(max_workers=max(1, io_threads))
        self.dev_name = f"cuda:{torch.cuda.current_device()}"
        # TP_STREAM_TRACE=1: host seconds per phase of run(), printed to stderr at the end
        self.trace = {} if os.environ.get("TP_STREAM_TRACE") else None

    def close(self):
        self.pool.shutdown(wait=True)

    # ---- ingest
    def load(self, k: int, chunk) -> None:
        """Host-stage (if needed) and H2D-copy batch k into device slot k % 3."""
        torch = self.torch
        slot, sslot = k % N_DEV_SLOTS, k % 2
        direct = all(src is not None for _, _, src in chunk)
        if not direct:
            self.staged[sslot].synchronize()  # the H2D that last read this staging slot
            futs = [self.pool.submit(load, self.stage[sslot][j].numpy())
                    for j, (_, load, _) in enumerate(chunk)]
            for f in futs:
                f.result()  # re-raises the first decode / dimension / missing-file error
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.used[slot])
            self.copy_start[slot].record(self.copy_stream)
            if direct:
                for j, (_, _, src) in enumerate(chunk):
                    self.dev[slot][j].copy_(src, non_blocking=True)
            else:
                self.dev[slot][: len(chunk)].copy_(self.stage[sslot][: len(chunk)],
                                                   non_blocking=True)
                self.staged[sslot].record(self.copy_stream)
            self.copied[slot].record(self.copy_stream)

    # ---- device work
    def stage1(self, k: int, n: int) -> None:
        torch = self.torch
        slot, bank = k % N_DEV_SLOTS, (self.base + k) % 2
        st = self.att_stream if self.lookahead else torch.cuda.current_stream()
        st.wait_event(self.copied[slot])
        if self.lookahead and k >= 2:  # bank k%2 was last read by batch k-2's selection
            st.wait_event(self.fin_end[(k - 2) % 3])
        with torch.cuda.stream(st):
            self.engine.stage1(n, self.dev[slot], stream=st, bank=bank,
                               events=self.att_ev[k % 3])

    def finish(self, k: int, n: int) -> None:
        torch = self.torch
        slot, bank = k % N_DEV_SLOTS, (self.base + k) % 2
        cur = torch.cuda.current_stream()
        cur.wait_event(self.copied[slot])
        cur.wait_event(self.att_ev[k % 3][1])
        eng = self.engine
        eng.events = self.fin_ev[k % 2]
        eng.finish(n, self.dev[slot], bank=bank, timed=True)
        self.fin_end[k % 3].record()
        self.used[slot].record()

    def timing(self, k: int, n: int) -> TimingProfile:
        """Per-frame TimingProfile of batch k (its events must have completed)."""
        slot = k % N_DEV_SLOTS
        e = self.fin_ev[k % 2]
        a0, a1 = self.att_ev[k % 3]
        att = a0.elapsed_time(a1)
        if self.lookahead and k > 0:  # only the part not hidden behind batch k-1's finish
            wait = max(0.0, self.fin_end[(k - 1) % 3].elapsed_time(a1))
        else:
            wait = att
        sel, fin, post = (e[i].elapsed_time(e[i + 1]) for i in (1, 2, 3))
        io = self.copy_start[slot].elapsed_time(self.copied[slot])
        return TimingProfile(io_ms=io / n, attention_wait_ms=min(wait, att) / n,
                             client_processing_ms=sel / n, final_eval_ms=fin / n,
                             postprocess_ms=post / n, per_worker=((self.dev_name, fin / n),))

    def run(self, chunks, sink, n_batches: int | None = None, failed=None):
        """Drive every batch through the device. sink.after_finish(k, n, chunk, failed) is
        called on the main stream after batch k's finish (n = 0 for padding batches up to
        n_batches and after a local failure); sink.emit(k, n, chunk, timing) once batch
        k's results are final (timing None when n = 0); sink.check(k, failed) after batch
        k+1 was launched (a collective sink raises there once any rank failed)."""
        nb = len(chunks) if n_batches is None else max(n_batches, len(chunks))
        self.base = self.engine._next  # box bank of batch 0 (holds the seeded history)
        if chunks and failed is None:
            try:
                self.load(0, chunks[0])
                self.stage1(0, len(chunks[0]))
            except Exception as exc:
                if not sink.collective:
                    raise
                failed = exc
        elif failed is not None and not sink.collective:
            raise failed
        pending = None
        for k in range(nb):
            chunk = chunks[k] if k < len(chunks) else []
            n = len(chunk) if failed is None else 0
            t0 = time.perf_counter()
            if n:
                try:
                    self.finish(k, n)
                except Exception as exc:
                    failed, n = exc, 0
            sink.after_finish(k, n, chunk, failed)
            t1 = time.perf_counter()
            if self.trace is not None:
                self._tr("finish_enqueue", t1 - t0)
            if failed is None and k + 1 < len(chunks):
                # host packing + H2D + stage 1 of batch k+1 are queued BEFORE batch k-1's
                # results are built on the host, so the copy and the look-ahead never wait
                # for Python result objects (slots and banks are guarded by events)
                try:
                    self.load(k + 1, chunks[k + 1])
                    self.stage1(k + 1, len(chunks[k + 1]))
                except Exception as exc:
                    failed = exc
                if self.trace is not None:
                    self._tr("load_stage1_enqueue", time.perf_counter() - t1)
            if pending is not None:  # batch k-1 finishes while batch k is queued
                self._emit(sink, *pending)
                pending = None
            pending = (k, n, chunk)
            if failed is not None and not sink.collective:
                self._emit(sink, *pending)  # keep the finished batch, then abort
                raise failed
            # collective sinks: every rank keeps issuing its per-batch exchange (with a
            # failure status) until all ranks have seen the failure, then all stop together
            sink.check(k, failed)
        if pending is not None:
            self._emit(sink, *pending)
        sink.check(nb, failed)
        if self.trace is not None:
            print("stream trace (host s): " + ", ".join(f"{k} {v:.4f}" for k, v in self.trace.items())
                  + f", batches {nb}", file=sys.stderr)

    def _emit(self, sink, k, n, chunk):
        t0 = time.perf_counter()
        if n:
            self.fin_end[k % 3].synchronize()
        t1 = time.perf_counter()
        sink.emit(k, n, chunk, self.timing(k, n) if n else None)
        if self.trace is not None:
            self._tr("emit_wait", t1 - t0)
            self._tr("emit_build", time.perf_counter() - t1)

    def _tr(self, key, dt):
        self.trace[key] = self.trace.get(key, 0.0) + dt


class LocalSink:
    """Default sink: FrameResults of this engine's batches, in order."""

    collective = False

    def __init__(self, engine):
        self.engine = engine
        self.results: list[FrameResult] = []
        self.snaps = {}

    def after_finish(self, k, n, chunk, failed=None):
        if n:
            self.snaps[k] = self.engine.snapshot(k % 2)

    def emit(self, k, n, chunk, timing):
        if not n:
            return
        res = self.engine.results_from(self.snaps.pop(k), [fid for fid, _, _ in chunk])
        for r, _ in res:
            self.results.append(FrameResult(r.frame_id, r.detections, r.active_count,
                                            r.total_count, timing))

    def check(self, k, failed=None):
        if failed is not None:
            raise failed


def make_engine(settings, W, H, det=None, policy=None, batch=16):
    from .engine import AttentionPipelineB200
    from .yolo import YoloB200Detector

    det = det or YoloB200Detector()
    return AttentionPipelineB200(settings, W, H, max_frames=batch, seed=det.seed,
                                 threshold=det.threshold, policy=policy, head=det.head,
                                 precision=det.precision)


def run_stream(frames, settings: PipelineSettings, det=None,
               policy: MergePolicy | None = None, *, batch: int = 16, engine=None,
               io_threads: int = 8, history=(), lookahead: bool = True) -> list[FrameResult]:
    """Evaluate a frame stream on the GPU, in input order, with ingest and attention
    overlapped (module docstring).

    ``frames`` is an iterable of ``Frame`` s or a ``frameio.FrameSource`` (a directory of
    PPM files): source frames are read from disk straight into the pinned staging buffer
    on ``io_threads`` host threads while the GPU runs the previous batch; Frames whose
    pixels live in pinned memory are copied to the device directly. ``history``: the
    AttentionModels of the frames before the stream (default: none)."""
    W, H, items = stream_items(frames)
    if not items:
        return []
    if engine is None:
        engine = make_engine(settings, W, H, det, policy, batch)
    chunks = ramp_chunks(items, engine.max_frames)
    drv = StreamDriver(engine, W, H, io_threads=io_threads, lookahead=lookahead)
    sink = LocalSink(engine)
    with engine.lock:
        engine.reset_history(history)
        try:
            drv.run(chunks, sink)
        except Exception as exc:
            raise StreamAborted(len(sink.results), sink.results, str(exc)) from exc
        finally:
            drv.close()
    return sink.results


def ramp_chunks(items, B: int) -> list:
    """Batches of a stream: B frames each, except that a long stream (> 2B frames) starts
    with B/4 and B/2 so the first batch's H2D copy and stage 1 — the only ones no earlier
    batch hides — are short; each ramp batch's compute then covers the next one's copy.
    Results do not depend on the batching (attention history stays on the device)."""
    sizes = []
    if len(items) > 2 * B and B >= 4:
        sizes = [B // 4, B // 2]
    chunks, i = [], 0
    for n in sizes:
        chunks.append(items[i:i + n])
        i += n
    chunks += [items[j:j + B] for j in range(i, len(items), B)]
    return chunks


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


__all__ = ["StreamAborted", "StreamDriver", "LocalSink", "run_stream", "result_line",
           "write_results", "stream_items", "make_engine", "ramp_chunks"]
