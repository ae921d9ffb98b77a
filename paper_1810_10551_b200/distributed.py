"""Frame-parallel sharding across GPUs (one process per GPU, torch.distributed).

The path partitions by frame: attention for frame t depends only on
frame t, selection on frames t-K+1..t, and the final pass never feeds back. A clip is
split into contiguous shards whose sizes differ by at most one (the reference's
``dispatch`` rule, distribution/client.py:82-96: ``shard_ranges``). A rank seeds its
temporal window by re-running stage 1 on the K-1 frames just before its shard
(``history_frames`` -> ``AttentionPipelineB200.prime_history``; 2 attention tiles per
frame at preset P1) instead of exchanging attention boxes, so the data path has no
collective. The only collective is the per-batch result gather (``ShardSink``): every
rank's compact batch results — a status/count header plus up to ``gather_cap`` final
records per frame — all-gathered in one fused NCCL launch through the C-ABI
(``tp_nccl_gather_dets`` on torch.distributed's own communicator; gloo on CPU), so rank 0
holds every frame's FrameResult in frame order (the reference's in-order results of
``run_stream``, client.py:294-377). A frame above the cap, or a failure on any rank,
makes every rank raise at the same batch (no rank is left waiting in a collective).
"""

from __future__ import annotations

import numpy as np

GATHER_CAP = 512  # final detections per frame carried by the result gather


def shard_ranges(n_frames: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, stop) chunks, sizes differing by at most one, in rank order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_frames, world)
    out, s = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((s, s + n))
        s += n
    return out


def history_frames(start: int, window: int) -> list[int]:
    """Frames whose attention a chunk starting at `start` needs before its first frame."""
    return list(range(max(0, start - (window - 1)), start))


def pack_records(rows: list[np.ndarray], max_rows: int, dtype: np.dtype) -> tuple[np.ndarray, np.ndarray]:
    """Per-frame record arrays -> (counts[n], padded [n, max_rows] records)."""
    counts = np.array([len(r) for r in rows], dtype=np.int32)
    if (counts > max_rows).any():
        raise ValueError(f"a frame has more than {max_rows} records")
    buf = np.zeros((len(rows), max_rows), dtype=dtype)
    for i, r in enumerate(rows):
        buf[i, : len(r)] = r
    return counts, buf


_warned = False


def nccl_comm(group=None) -> int:
    """The ncclComm_t torch.distributed holds for this rank's device (borrowed, never
    freed here). torch creates communicators lazily; one tiny all-reduce forces it."""
    import torch
    import torch.distributed as dist

    backend = (group or dist.group.WORLD)._get_backend(torch.device("cuda"))
    try:
        ptr = int(backend._comm_ptr())
    except RuntimeError:
        ptr = 0
    if not ptr:
        dist.all_reduce(torch.zeros(1, device="cuda"), group=group)
        ptr = int(backend._comm_ptr())
    if not ptr:
        raise RuntimeError("torch.distributed exposes no NCCL communicator for this device")
    return ptr


_comm_ok: dict = {}


def _fused_ok(group) -> bool:
    """Whether every rank can use the fused C-ABI gather (agreed collectively once per
    group: a rank without a communicator pointer would otherwise issue a different
    collective sequence from its peers and hang them)."""
    import torch
    import torch.distributed as dist

    key = id(group)
    if key not in _comm_ok:
        try:
            nccl_comm(group)
            mine = 1
        except (RuntimeError, AttributeError):
            mine = 0
        t = torch.tensor([mine], dtype=torch.int32, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        _comm_ok[key] = bool(int(t.item()))
    return _comm_ok[key]


def nccl_all_gather(local_recs, all_recs, local_counts, all_counts, group=None, stream=None):
    """Rank-order all-gather of a record slice and its counts in one fused NCCL launch on
    `stream` (tp_nccl_gather_dets). Shapes: all_* = world x local_*.

    If any rank's torch build exposes no communicator pointer (agreed collectively), all
    ranks use the same two all-gathers through torch.distributed's NCCL (one warning)."""
    import torch.distributed as dist

    from . import native

    if not _fused_ok(group):
        global _warned
        if not _warned:
            import warnings

            warnings.warn("tp_nccl_gather_dets unavailable on some rank; using torch NCCL "
                          "all-gathers")
            _warned = True
        if local_recs is not None:
            dist.all_gather_into_tensor(all_recs.view(-1), local_recs.reshape(-1), group=group)
        if local_counts is not None:
            dist.all_gather_into_tensor(all_counts.view(-1), local_counts.reshape(-1), group=group)
        return
    comm = nccl_comm(group)
    native.call("tp_nccl_gather_dets", comm, native.ptr(local_recs),
                int(local_recs.numel() * local_recs.element_size()) if local_recs is not None else 0,
                native.ptr(local_counts), int(local_counts.numel()) if local_counts is not None else 0,
                native.ptr(all_recs), native.ptr(all_counts), native.stream_handle(stream))


def all_gather_pair(local_recs, all_recs, local_counts, all_counts, group=None):
    """Backend-neutral rank-order all-gather of (records, counts): fused NCCL on GPUs,
    host tensors over gloo."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        nccl_all_gather(local_recs, all_recs, local_counts, all_counts, group)
        return
    for loc, out in ((local_recs, all_recs), (local_counts, all_counts)):
        host = out.cpu()
        dist.all_gather_into_tensor(host.view(-1), loc.reshape(-1).cpu(), group=group)
        out.copy_(host)


def gather_records(counts, records, frames_per_rank: list[int], group=None, to_host=True):
    """All-gather per-frame (count, padded records) from every rank; returns the
    concatenation in rank (= frame) order as a list of per-frame record arrays.

    `counts` int32 [n_local]; `records` uint8 [n_local, rec_bytes] tensors on the
    backend's device. Ranks may hold different frame counts: buffers are padded to
    the largest shard."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_max = max(frames_per_rank)
    dev = counts.device
    c = torch.zeros(n_max, dtype=torch.int32, device=dev)
    c[: counts.numel()] = counts
    r = torch.zeros((n_max, records.shape[1]), dtype=torch.uint8, device=dev)
    r[: records.shape[0]] = records
    call = torch.empty(world * n_max, dtype=torch.int32, device=dev)
    rall = torch.empty((world * n_max, records.shape[1]), dtype=torch.uint8, device=dev)
    all_gather_pair(r, rall, c, call, group)
    if not to_host:  # stay on device (no host sync): [world*n_max] counts, records
        return call, rall
    call = call.cpu().numpy().reshape(world, n_max)
    rall = rall.cpu().numpy().reshape(world, n_max, -1)
    out = []
    for rank in range(world):
        for f in range(frames_per_rank[rank]):
            out.append((int(call[rank, f]), rall[rank, f]))
    return out


class BatchGather:
    """Device-side per-batch result gather for frame shards. Per rank and batch: an int32
    header [status, n, 0, 0 | final counts (B) | active counts (B)] and the first `cap`
    final records (56 B, tp_pdet_t) of each frame, all-gathered in rank order; the
    received buffers are copied to pinned host memory (double-buffered) so the host
    reads batch k while the device runs batch k+1."""

    HDR = 4

    def __init__(self, B: int, world: int, group=None, cap: int = GATHER_CAP, records=True):
        import torch

        from . import native
        from .engine import MAX_PER_FRAME

        if not (1 <= cap <= MAX_PER_FRAME):
            raise ValueError(f"gather cap must be 1..{MAX_PER_FRAME}")
        self.torch, self.B, self.world, self.group, self.cap = torch, B, world, group, cap
        self.rec = native.PDET_DTYPE.itemsize
        self.nh = self.HDR + 2 * B
        nrb = B * cap * self.rec if records else 0
        self.records = records
        dev = "cuda"
        self.hdr = torch.zeros(self.nh, dtype=torch.int32, device=dev)
        self.recs = torch.zeros(max(nrb, 1), dtype=torch.uint8, device=dev)
        self.all_hdr = torch.zeros(world * self.nh, dtype=torch.int32, device=dev)
        self.all_recs = torch.zeros(world * max(nrb, 1), dtype=torch.uint8, device=dev)
        pin = dict(pin_memory=True)
        self.host = [{"hdr": torch.empty(world * self.nh, dtype=torch.int32, **pin),
                      "recs": torch.empty(world * max(nrb, 1), dtype=torch.uint8, **pin),
                      "event": torch.cuda.Event()} for _ in range(2)]

    def launch(self, engine, k: int, n: int, failed: bool, want_records: bool) -> None:
        """Pack this rank's batch k (on the current stream) and all-gather it."""
        from .engine import MAX_PER_FRAME

        B = self.B
        self.hdr.zero_()
        self.hdr[0] = 1 if failed else 0
        self.hdr[1] = n
        if n:
            self.hdr[self.HDR:self.HDR + n].copy_(engine.ocounts[:n])
            self.hdr[self.HDR + B:self.HDR + B + n].copy_(engine.active_counts[:n])
            if self.records:
                src = engine.outp[: n * MAX_PER_FRAME * self.rec].view(
                    n, MAX_PER_FRAME * self.rec)[:, : self.cap * self.rec]
                self.recs[: n * self.cap * self.rec].view(n, self.cap * self.rec).copy_(src)
        all_gather_pair(self.recs, self.all_recs, self.hdr, self.all_hdr, self.group)
        h = self.host[k % 2]
        h["hdr"].copy_(self.all_hdr, non_blocking=True)
        if want_records and self.records:
            h["recs"].copy_(self.all_recs, non_blocking=True)
        h["event"].record()

    def read(self, k: int):
        """(headers [world][nh] int32, records [world][B][cap] tp_pdet_t) of batch k."""
        from . import native

        h = self.host[k % 2]
        h["event"].synchronize()
        hdr = h["hdr"].numpy().reshape(self.world, self.nh).copy()
        recs = None
        if self.records:
            recs = h["recs"].numpy().view(native.PDET_DTYPE).reshape(
                self.world, self.B, self.cap).copy()
        return hdr, recs


class ShardSink:
    """Result sink of a frame-sharded stream (see module docstring). Rank 0 assembles
    every rank's FrameResults; each rank keeps its own frames' TimingProfiles, which are
    exchanged once at the end (host objects, a few KB)."""

    collective = True

    def __init__(self, engine, items, ranges, rank: int, world: int, group=None,
                 cap: int = GATHER_CAP):
        from .engine import MAX_PER_FRAME  # noqa: F401

        self.engine, self.items, self.ranges = engine, items, ranges
        self.rank, self.world, self.group = rank, world, group
        self.B = engine.max_frames
        self.gather = BatchGather(self.B, world, group, cap)
        self.cap = cap
        self.records: dict[int, tuple] = {}  # global frame index -> (dets, active_count)
        self.timings: dict[int, object] = {}  # local frame index -> TimingProfile
        self.failed_at = None  # (rank, batch) of the first failure seen
        self.overflow = None

    def after_finish(self, k, n, chunk, failed=None):
        self.gather.launch(self.engine, k, n, failed is not None, want_records=self.rank == 0)

    def emit(self, k, n, chunk, timing):
        from .engine import records_to_detections

        hdr, recs = self.gather.read(k)
        B, H = self.B, BatchGather.HDR
        for r in range(self.world):
            status, nr = int(hdr[r, 0]), int(hdr[r, 1])
            if status and self.failed_at is None:
                self.failed_at = (r, k)
            for j in range(nr):
                oc, ac = int(hdr[r, H + j]), int(hdr[r, H + B + j])
                g = self.ranges[r][0] + k * B + j
                if oc > self.cap and self.overflow is None:
                    self.overflow = (g, oc)
                if self.rank == 0 and oc <= self.cap:
                    self.records[g] = (records_to_detections(recs[r, j, :oc],
                                                             self.engine.labels.names), ac)
        if n and timing is not None:
            for j in range(n):
                self.timings[self.ranges[self.rank][0] + k * B + j] = timing

    def check(self, k, failed=None):
        if self.failed_at is not None or self.overflow is not None:
            raise _ShardFailure(self.failed_at, self.overflow, failed)


class _ShardFailure(RuntimeError):
    def __init__(self, failed_at, overflow, local):
        if overflow is not None:
            msg = (f"frame index {overflow[0]} has {overflow[1]} final detections, above the "
                   "result gather cap (raise gather_cap)")
        else:
            msg = f"rank {failed_at[0]} failed at batch {failed_at[1]}"
            if local is not None:
                msg += f": {local}"
        super().__init__(msg)


def run_stream_sharded(frames, settings, det=None, policy=None, *, batch: int = 16,
                       group=None, engine=None, io_threads: int = 8, lookahead: bool = True,
                       gather_cap: int = GATHER_CAP):
    """Multi-GPU run_stream (reference client.py:294-377 semantics). Every rank passes the
    same `frames` (Frames or a FrameSource); rank r evaluates shard_ranges(n, world)[r]
    after seeding its window from the K-1 frames before the shard (stage 1 only), with the
    single-GPU scheduler (stream.StreamDriver: ingest, attention look-ahead and results
    overlapped). Per batch the compact results are all-gathered over NCCL, so rank 0
    returns every frame's FrameResult in input order (other ranks return []). A failure
    anywhere raises StreamAborted on every rank (rank 0's carries the completed prefix)."""
    import torch
    import torch.distributed as dist

    from .pipeline_types import FrameResult
    from .stream import StreamAborted, StreamDriver, make_engine, stream_items

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    W, H, items = stream_items(frames)
    if not items:
        return []
    if engine is None:
        engine = make_engine(settings, W, H, det, policy, batch)
    B = engine.max_frames
    ranges = shard_ranges(len(items), world)
    s, e = ranges[rank]
    mine = items[s:e]
    chunks = [mine[i:i + B] for i in range(0, len(mine), B)]
    n_batches = max(-(-(b - a) // B) for a, b in ranges)
    hist = history_frames(s, engine.K)
    drv = StreamDriver(engine, W, H, io_threads=io_threads, lookahead=lookahead)
    sink = ShardSink(engine, items, ranges, rank, world, group, gather_cap)
    with engine.lock:
        prime_err = None
        try:
            engine.reset_history(())
            if hist and mine:  # the window's frames before the shard: stage 1 only
                drv.load(0, [items[i] for i in hist])
                torch.cuda.current_stream().wait_event(drv.copied[0])
                engine.prime_history(drv.dev[0], len(hist))
        except Exception as exc:  # noqa: BLE001 — reported through the batch protocol
            prime_err = exc
        try:
            drv.run(chunks, sink, n_batches=n_batches, failed=prime_err)
            err = None
        except Exception as exc:  # noqa: BLE001 — every rank raised at the same batch
            err = exc
        finally:
            drv.close()
    # per-frame timings travel once, as host objects, after the last collective
    if err is None:
        gathered = [None] * world
        dist.all_gather_object(gathered, sink.timings, group=group)
    if err is not None:
        done = sorted(sink.records) if rank == 0 else sorted(sink.timings)
        cursor = next((i for i, g in enumerate(done) if g != (done[0] + i if done else 0)),
                      len(done))
        completed = [FrameResult(items[g][0], *sink.records[g], engine.F,
                                 sink.timings.get(g) or _blank())
                     for g in done[:cursor]] if rank == 0 else []
        raise StreamAborted(cursor, completed, str(err)) from err
    timings = {}
    for t in gathered:
        timings.update(t)
    if rank != 0:
        return []
    return [FrameResult(items[g][0], sink.records[g][0], sink.records[g][1], engine.F,
                        timings[g]) for g in range(len(items))]


def _blank():
    from .pipeline_types import TimingProfile

    return TimingProfile()
