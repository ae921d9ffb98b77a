"""Batched, device-resident attention pipeline (the B200-native hot path).

One call processes a batch of N frames already in HBM with no host round trip inside:

  gather A attention tiles/frame (K1) -> YOLO v2 (K3/K4, tcgen05) -> region decode +
  to_global (K5) -> attention box lists (conf >= min_conf) -> merge_temporal +
  select_active over the K-frame window (K6) -> stage-2 job list -> gather active
  crops (K2) -> YOLO v2 on the active tiles (count read on device) -> decode ->
  final_pass tagged lists -> NMS + merge + min_conf (K7)

Batching frames is semantically free: attention for frame t depends only
on frame t, selection on frames t-K+1..t, and the final pass never feeds back; the
attention boxes of the last K-1 frames are carried on the device into the next batch.
Results equal the reference's run_sequence (pipeline.py:442-457) frame by frame.
"""

from __future__ import annotations

import threading
from contextlib import nullcontext

import numpy as np

from . import kernels, native
from .detector import Detection
from .geometry import Rect
from .pipeline_types import AttentionModel, FrameResult, GridPlan, PipelineSettings, \
    StageFailure, TimingProfile
from .postprocess import LabelTable, MergePolicy, make_policy_struct, ctypes_ref
from .yolo import COCO_NAMES, DEFAULT_PRECISION, YoloNet

MAX_BOXES = 256        # attention boxes per frame (conf >= min_conf)
MAX_MERGED = 512       # merged window boxes per frame
MAX_PER_FRAME = 2048   # raw stage-2 detections per frame (postprocess capacity)
EXCHANGE_CAP = 128     # raw stage-2 records per tile in the crop-parallel exchange


def _dist_exchange(local_dets, local_counts, all_dets, all_counts):
    """Default crop_shard exchange: all-gather every rank's compact stage-2 slice in rank
    order over the default process group (NCCL on GPUs: records and counts in one fused
    launch through tp_nccl_gather_dets; gloo on CPU)."""
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        from .distributed import nccl_all_gather
        nccl_all_gather(local_dets, all_dets, local_counts, all_counts)
        return
    for loc, out in ((local_dets, all_dets), (local_counts, all_counts)):
        dist.all_gather(list(out.view(dist.get_world_size(), -1).unbind(0)), loc)


class AttentionPipelineB200:
    def __init__(self, settings: PipelineSettings, frame_w: int, frame_h: int, *,
                 max_frames: int = 8, seed: int = 0, threshold: float = 0.25,
                 policy: MergePolicy | None = None, resample: str = "nearest",
                 head: str = "calibrated", net: YoloNet | None = None,
                 precision: str = DEFAULT_PRECISION,
                 crop_shard: tuple[int, int] | None = None, exchange=None,
                 exchange_cap: int = EXCHANGE_CAP):
        """crop_shard=(rank, world): crop-parallel stage 2 — every rank runs
        stage 1 + selection for the same frames and evaluates its contiguous slice of the
        active crops; `exchange(local_dets, local_counts, all_dets, all_counts)` all-gathers
        the compact slices (exchange_cap records per tile + true counts) in rank order
        (default: torch.distributed, NCCL on GPUs).

        Stage 1 and stage 2 run on two YoloNets sharing one set of device weights, so the
        stage 1 of batch k+1 may run on another stream while batch k finishes
        (stage1()/finish(), used by stream.run_stream); a caller-supplied `net` serves
        both stages (no overlap)."""
        torch = native.require_cuda()
        if resample not in native.RESAMPLE:
            raise ValueError(f"resample must be one of {tuple(native.RESAMPLE)}")
        self.torch = torch
        self.settings = settings
        self.W, self.H = int(frame_w), int(frame_h)
        self.plan = GridPlan.build(self.W, self.H, settings)
        self.policy = policy or MergePolicy()
        self.threshold = float(threshold)
        self.resample = resample
        self.max_frames = int(max_frames)
        att, fin = self.plan.attention_grid, self.plan.final_grid
        self.A, self.F = len(att.crops), len(fin.crops)
        self.K = settings.temporal_window
        if self.F > 1024 or fin.rows * fin.cols > 256:
            raise ValueError("final grid too large for the selection/merge kernels")
        mf = self.max_frames
        if net is None:  # precision "fp32" = the hi/lo fp16 activation-pair plan
            net = YoloNet(mf * self.F, seed=seed, head=head, dtype=precision)
            net1 = YoloNet(mf * self.A, share=net)
        else:
            if net.max_tiles < mf * max(self.A, self.F):
                raise ValueError("shared YoloNet too small for this batch size")
            net1 = net
        self.net, self.net1 = net, net1
        self.dtype = self.net.dtype
        self.lock = threading.RLock()  # one batch at a time on the shared buffers

        dev = "cuda"
        self.frames = torch.empty((mf, self.H, self.W, 3), dtype=torch.uint8, device=dev)
        self.frame_stride = self.H * self.W * 3
        self.att_jobs = kernels.jobs_tensor(
            (f, c.crop_id, int(c.global_rect.x), int(c.global_rect.y), int(c.global_rect.w),
             c.row * att.cols + c.col) for f in range(mf) for c in att.crops)
        self.fin_rects = torch.tensor(
            [[c.global_rect.x, c.global_rect.y, c.global_rect.w, c.global_rect.h]
             for c in fin.crops], dtype=torch.float64, device=dev)
        self.fin_table = torch.tensor(
            [[int(c.global_rect.x), int(c.global_rect.y), int(c.global_rect.w),
              c.row * fin.cols + c.col] for c in fin.crops], dtype=torch.int32, device=dev)
        self.dets1, self.counts1 = kernels.alloc_dets(mf * self.A)
        # attention box banks: slots 0..K-2 = history, K-1.. = the batch's own frames.
        # Batch k uses bank k % 2, so stage 1 of batch k+1 never touches the bank batch k's
        # selection reads; finish() carries its batch's last K-1 lists into the other bank.
        slots = (self.K - 1) + mf
        self._banks = [torch.zeros((slots, MAX_BOXES, 4), dtype=torch.float64, device=dev)
                       for _ in range(2)]
        self._bank_counts = [torch.zeros(slots, dtype=torch.int32, device=dev) for _ in range(2)]
        self._next = 0  # bank of the next batch
        self._bank = 0  # bank of the last finished batch (results read it)
        self.words = (self.F + 31) // 32
        self.mask = torch.zeros((mf, self.words), dtype=torch.int32, device=dev)
        self.active_ids = torch.zeros((mf, self.F), dtype=torch.int32, device=dev)
        self.active_counts = torch.zeros(mf, dtype=torch.int32, device=dev)
        self.merged = torch.zeros((mf, MAX_MERGED, 4), dtype=torch.float64, device=dev)
        self.merged_counts = torch.zeros(mf, dtype=torch.int32, device=dev)
        self.jobs2 = torch.zeros(mf * self.F * native.JOB_DTYPE.itemsize, dtype=torch.uint8,
                                 device=dev)
        self.frame_job_start = torch.zeros(mf + 1, dtype=torch.int32, device=dev)
        self.n_jobs2 = torch.zeros(1, dtype=torch.int32, device=dev)
        self.dets2, self.counts2 = kernels.alloc_dets(mf * self.F)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.crop_shard = None
        if crop_shard is not None:
            rank, world = (int(v) for v in crop_shard)
            if not (world >= 1 and 0 <= rank < world):
                raise ValueError(f"bad crop_shard {crop_shard}")
            if not (1 <= exchange_cap <= kernels.MAX_PER_TILE):
                raise ValueError(f"exchange_cap must be 1..{kernels.MAX_PER_TILE}")
            self.crop_shard = (rank, world)
            self.exchange_cap = int(exchange_cap)
            self.max_slice = -(-mf * self.F // world)
            det_b = self.exchange_cap * native.DET_DTYPE.itemsize
            self.jobs_local = torch.zeros(self.max_slice * native.JOB_DTYPE.itemsize,
                                          dtype=torch.uint8, device=dev)
            self.n_local = torch.zeros(1, dtype=torch.int32, device=dev)
            self.send_dets = torch.zeros(self.max_slice * det_b, dtype=torch.uint8, device=dev)
            self.all_dets = torch.zeros(world * self.max_slice * det_b, dtype=torch.uint8,
                                        device=dev)
            self.all_counts = torch.zeros(world * self.max_slice, dtype=torch.int32, device=dev)
            self.exchange = exchange or _dist_exchange
        rec = native.PDET_DTYPE.itemsize
        self.pdets = torch.zeros(mf * MAX_PER_FRAME * rec, dtype=torch.uint8, device=dev)
        self.pcounts = torch.zeros(mf, dtype=torch.int32, device=dev)
        self.outp = torch.zeros(mf * MAX_PER_FRAME * rec, dtype=torch.uint8, device=dev)
        self.ocounts = torch.zeros(mf, dtype=torch.int32, device=dev)
        self.labels = LabelTable(COCO_NAMES)
        self.post_policy = make_policy_struct(self.policy, self.labels, fin.cols,
                                              fin.rows * fin.cols,
                                              min_conf=settings.min_confidence)
        self.full_box = torch.tensor([0.0, 0.0, float(self.W), float(self.H)],
                                     dtype=torch.float64, device=dev)
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        self.last_timing = TimingProfile()
        self.last_n_tiles = (0, 0)

    # ------------------------------------------------------------------ state
    @property
    def boxes(self):
        """Attention box slots of the last finished batch (history + its frames)."""
        return self._banks[self._bank]

    @property
    def box_counts(self):
        return self._bank_counts[self._bank]

    def reset_history(self, history=()):
        """Seed the K-1 history slots of the next batch from host AttentionModels
        (oldest first)."""
        b = self._next
        K1 = self.K - 1
        self._bank_counts[b][:K1].zero_()
        hist = list(history)[-K1:] if K1 > 0 else []
        off = K1 - len(hist)
        for i, m in enumerate(hist):
            n = len(m.boxes)
            if n > MAX_BOXES:
                raise ValueError(f"history model has {n} boxes (> {MAX_BOXES})")
            if n:
                self._banks[b][off + i, :n] = self.torch.tensor(
                    [[r.x, r.y, r.w, r.h] for r in m.boxes], dtype=self.torch.float64)
            self._bank_counts[b][off + i] = n

    def prime_history(self, frames, n: int, stream=None) -> None:
        """Seed the K-1 history slots of the next batch by running stage 1 on the n <= K-1
        frames (device uint8 [n,H,W,3]) that precede it — the boundary of a frame-parallel
        shard (distributed.history_frames): no attention exchange between ranks."""
        b = self._next
        K1 = self.K - 1
        cnt = self._bank_counts[b]
        cnt[:K1].zero_()
        if K1 == 0 or n == 0:
            return
        if n > K1:
            raise ValueError(f"at most {K1} history frames")
        self.stage1(n, frames, stream=stream, bank=b)
        bank = self._banks[b]
        with self.torch.cuda.stream(stream) if stream is not None else nullcontext():
            bank[K1 - n:K1].copy_(bank[K1:K1 + n].clone())
            cnt[K1 - n:K1].copy_(cnt[K1:K1 + n].clone())

    def upload(self, frames_host, n: int, non_blocking: bool = True):
        """Host uint8 [n,H,W,3] (ideally pinned) -> the device frame batch."""
        self.frames[:n].copy_(frames_host[:n], non_blocking=non_blocking)

    # ------------------------------------------------------------------ run
    def set_attention(self, boxes_per_frame) -> None:
        """Inject stage-1 attention boxes for the next run_device(..., attention="inject")
        call: one list of (x, y, w, h) global boxes per batch frame."""
        torch = self.torch
        K1 = self.K - 1
        n = len(boxes_per_frame)
        if n > self.max_frames:
            raise ValueError("more frames than the batch holds")
        arr = np.zeros((n, MAX_BOXES, 4), dtype=np.float64)
        cnt = np.zeros(n, dtype=np.int32)
        for f, bl in enumerate(boxes_per_frame):
            if len(bl) > MAX_BOXES:
                raise ValueError(f"more than {MAX_BOXES} attention boxes in a frame")
            cnt[f] = len(bl)
            for k, b in enumerate(bl):
                arr[f, k] = b
        self._banks[self._next][K1:K1 + n].copy_(torch.from_numpy(arr))
        self._bank_counts[self._next][K1:K1 + n].copy_(torch.from_numpy(cnt))

    def run_device(self, n: int, frames=None, stream=None, timed: bool = False,
                   attention: str = "yolo") -> None:
        """Launch the whole pipeline for frames[0:n] (device). No host synchronisation.

        attention: "yolo" (stage 1 on the attention grid), "inject" (boxes from
        set_attention), or "all" (every final crop active: run_allcrops_baseline)."""
        if not (1 <= n <= self.max_frames):
            raise ValueError(f"batch of {n} frames (max {self.max_frames})")
        if attention not in ("yolo", "inject", "all"):
            raise ValueError("attention must be 'yolo', 'inject' or 'all'")
        b = self._next
        K1 = self.K - 1
        if timed:
            self.events[0].record(stream)
        if attention == "all":
            self._banks[b][K1:K1 + n, 0] = self.full_box
            self._bank_counts[b][K1:K1 + n] = 1
        elif attention == "yolo":
            self.stage1(n, frames, stream=stream, bank=b)
        self.finish(n, frames, stream=stream, bank=b, timed=timed)

    def capture(self, n: int, frames, attention: str = "yolo"):
        """CUDA-graph the whole device step for a fixed batch size and frame buffer (no host
        work between kernels: worth ~10% per frame at batch 1, nothing at batch >= 4).
        Returns a replay() callable; each replay is one run_device(n, frames) (history
        advances as in eager mode) and results()/snapshot() read it as usual. The graph
        captures both box banks' roles, so it is captured twice (even / odd batches)."""
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graphs = []
        with torch.cuda.stream(side):
            self.run_device(n, frames=frames, attention=attention)  # warm-up on the stream
            side.synchronize()
            for _ in range(2):
                g = torch.cuda.CUDAGraph()
                bank = self._next
                with torch.cuda.graph(g, stream=side):
                    self.run_device(n, frames=frames, attention=attention)
                graphs.append((bank, g))
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        by_bank = dict(graphs)

        def replay():
            b = self._next
            by_bank[b].replay()
            self._bank, self._next, self._n = b, 1 - b, n
        replay.graph = by_bank
        return replay

    def _gather(self, net, fr, jobs, n_tiles, n_jobs_dev, stream):
        """Crop gather into a net's layer-0 input slots."""
        kernels.gather(fr, self.frame_stride, self.H, self.W, jobs, n_tiles, self.resample,
                       out_act_ptr=net.input_ptr, n_jobs_dev=n_jobs_dev, stream=stream,
                       dtype=self.dtype)

    def stage1(self, n: int, frames=None, stream=None, bank: int | None = None,
               events=None) -> None:
        """Stage 1 of a batch (attention_pass, reference pipeline.py:297-316): gather the
        A attention tiles per frame, YOLO on net1, decode + to_global, conf >= min_conf
        boxes into box bank `bank` (default: the next batch's) slots K-1... events:
        optional (start, end) CUDA events recorded on `stream` around it."""
        fr = self.frames if frames is None else frames
        b = self._next if bank is None else bank
        st = native.stream_handle(stream)
        K1 = self.K - 1
        if events is not None:
            events[0].record(stream)
        try:
            nt1 = n * self.A
            self._gather(self.net1, fr, self.att_jobs, nt1, None, stream)
            self.net1.forward(nt1, stream=stream)
            kernels.decode(self.net1, nt1, self.att_jobs, self.W, self.H, self.threshold,
                           self.dets1, self.counts1, stream=stream)
            native.call("tp_attention_boxes", native.ptr(self.dets1), native.ptr(self.counts1),
                        kernels.MAX_PER_TILE, n, self.A, float(self.settings.min_confidence),
                        native.ptr(self._banks[b]) + K1 * MAX_BOXES * 32,
                        native.ptr(self._bank_counts[b]) + K1 * 4, MAX_BOXES, st)
        except native.NativeError as exc:
            raise StageFailure("attention", -1) from exc
        if events is not None:
            events[1].record(stream)

    def finish(self, n: int, frames=None, stream=None, bank: int | None = None,
               timed: bool = False) -> None:
        """Selection + stage 2 + postprocess of the batch whose attention boxes are in
        `bank` (merge_temporal/select_active/final_pass/finish_detections, reference
        pipeline.py:319-385), then carry its last K-1 attention lists into the other
        bank's history slots. timed: events[1..4] around select / stage 2 / post."""
        fr = self.frames if frames is None else frames
        b = self._next if bank is None else bank
        st = native.stream_handle(stream)
        ev = self.events
        boxes, counts = self._banks[b], self._bank_counts[b]
        try:
            if timed:
                ev[1].record(stream)
            native.call("tp_select_active", native.ptr(boxes), native.ptr(counts),
                        MAX_BOXES, n, self.K, native.ptr(self.fin_rects), self.F, self.A,
                        float(self.settings.attention_margin_px), float(self.W), float(self.H),
                        native.ptr(self.mask), self.words, native.ptr(self.active_ids),
                        native.ptr(self.active_counts), native.ptr(self.merged),
                        native.ptr(self.merged_counts), MAX_MERGED, st)
            native.call("tp_build_jobs", native.ptr(self.active_ids),
                        native.ptr(self.active_counts), n, self.F, native.ptr(self.fin_table),
                        self.A, native.ptr(self.jobs2), native.ptr(self.frame_job_start),
                        native.ptr(self.n_jobs2), st)
        except native.NativeError as exc:
            raise StageFailure("select", -1) from exc
        self._bank = b
        try:
            if timed:
                ev[2].record(stream)
            nt2 = n * self.F  # upper bound; kernels read the real count from n_jobs2
            if self.crop_shard is None:
                self._gather(self.net, fr, self.jobs2, nt2, self.n_jobs2, stream)
                self.net.forward(nt2, n_tiles_dev=self.n_jobs2, stream=stream)
                kernels.decode(self.net, nt2, self.jobs2, self.W, self.H, self.threshold,
                               self.dets2, self.counts2, n_tiles_dev=self.n_jobs2, stream=stream)
            else:
                self._stage2_slice(fr, nt2, stream, st)
                if self._split_phase:  # run_local(): the caller exchanges and finishes
                    self._pending = (n, stream, st, timed)
                    return
                with self.torch.cuda.stream(stream) if stream is not None else nullcontext():
                    self.exchange(*self.local_results(), self.all_dets, self.all_counts)
                self._unslice(nt2, st)
        except native.NativeError as exc:
            raise StageFailure("final", -1) from exc
        self._post(n, stream, st, timed)

    # ---- crop-parallel stage 2 (crop_shard) ----
    _split_phase = False

    def _stage2_slice(self, fr, nt2, stream, st):
        rank, world = self.crop_shard
        native.call("tp_slice_jobs", native.ptr(self.jobs2), native.ptr(self.n_jobs2), rank,
                    world, native.ptr(self.jobs_local), native.ptr(self.n_local), self.max_slice,
                    st)
        ntl = min(-(-nt2 // world), self.max_slice)  # host upper bound of the slice
        self._gather(self.net, fr, self.jobs_local, ntl, self.n_local, stream)
        self.net.forward(ntl, n_tiles_dev=self.n_local, stream=stream)
        kernels.decode(self.net, ntl, self.jobs_local, self.W, self.H, self.threshold,
                       self.dets2, self.counts2, n_tiles_dev=self.n_local, stream=stream)
        # compact slice for the exchange: the first exchange_cap records of every tile
        # (the counts stay true, so the receiver detects a clipped tile)
        rec = native.DET_DTYPE.itemsize
        src = self.dets2[: self.max_slice * kernels.MAX_PER_TILE * rec].view(
            self.max_slice, kernels.MAX_PER_TILE * rec)[:, : self.exchange_cap * rec]
        with self.torch.cuda.stream(stream) if stream is not None else nullcontext():
            self.send_dets.view(self.max_slice, self.exchange_cap * rec).copy_(src)

    def _unslice(self, nt2, st):
        rank, world = self.crop_shard
        native.call("tp_unslice_dets", native.ptr(self.all_dets), native.ptr(self.all_counts),
                    self.max_slice, native.ptr(self.n_jobs2), world, nt2, self.exchange_cap,
                    kernels.MAX_PER_TILE, native.ptr(self.dets2), native.ptr(self.counts2),
                    native.ptr(self.overflow), st)

    def local_results(self):
        """This rank's compact stage-2 slice: (dets bytes, true counts) device tensors —
        [max_slice][exchange_cap] records, [max_slice] counts."""
        return self.send_dets, self.counts2[: self.max_slice]

    def run_local(self, n: int, frames=None, stream=None, timed: bool = False):
        """crop_shard phase 1: stages 1 + selection + this rank's stage-2 slice; then
        fill all_dets / all_counts (rank-order concatenation of every rank's
        local_results()) and call finish_local()."""
        if self.crop_shard is None:
            raise ValueError("run_local needs crop_shard")
        self._split_phase = True
        try:
            self.run_device(n, frames=frames, stream=stream, timed=timed)
        finally:
            self._split_phase = False

    def finish_local(self):
        """crop_shard phase 2: unslice the gathered slices, collect, postprocess."""
        n, stream, st, timed = self._pending
        try:
            self._unslice(n * self.F, st)
        except native.NativeError as exc:
            raise StageFailure("final", -1) from exc
        self._post(n, stream, st, timed)

    def _post(self, n, stream, st, timed):
        ev = self.events
        K1 = self.K - 1
        b = self._bank
        try:
            native.call("tp_collect_final", native.ptr(self.dets2), native.ptr(self.counts2),
                        kernels.MAX_PER_TILE, native.ptr(self.jobs2),
                        native.ptr(self.frame_job_start), n, native.ptr(self.pdets),
                        native.ptr(self.pcounts), MAX_PER_FRAME, st)
        except native.NativeError as exc:
            raise StageFailure("final", -1) from exc
        try:
            if timed:
                ev[3].record(stream)
            native.call("tp_postprocess", native.ptr(self.pdets), native.ptr(self.pcounts), n,
                        MAX_PER_FRAME, ctypes_ref(self.post_policy), native.ptr(self.outp),
                        native.ptr(self.ocounts), None, None, st)
            if timed:
                ev[4].record(stream)
        except native.NativeError as exc:
            raise StageFailure("postprocess", -1) from exc
        # carry the batch's last K-1 attention lists into the other bank's history slots
        if K1 > 0:
            with self.torch.cuda.stream(stream) if stream is not None else nullcontext():
                self._banks[1 - b][:K1].copy_(self._banks[b][n:n + K1])
                self._bank_counts[1 - b][:K1].copy_(self._bank_counts[b][n:n + K1])
        self._next = 1 - b
        self._n = n

    # ------------------------------------------------------------------ API helpers
    def _upload_frames(self, frames):
        torch = self.torch
        for i, fr in enumerate(frames):
            if fr.width != self.W or fr.height != self.H:
                raise ValueError("frame size differs from the engine's")
            if fr.pixels is None:
                raise StageFailure("attention", fr.frame_id) from ValueError(
                    "YoloB200Detector needs frame pixels")
            self.frames[i].copy_(torch.from_numpy(np.ascontiguousarray(fr.pixels)))

    def evaluate_frames(self, frames, history=()):
        """Frames (host pixels) -> [(FrameResult, AttentionModel)]. history=None keeps the
        device-carried attention of the previous call (clip mode)."""
        n = len(frames)
        with self.lock:
            if history is not None:
                self.reset_history(history)
            self._upload_frames(frames)
            self.run_device(n, timed=True)
            t = [v / n for v in self.stage_times_ms()]
            timing = TimingProfile(attention_wait_ms=t[0], client_processing_ms=t[1],
                                   final_eval_ms=t[2], postprocess_ms=t[3])
            return self.results([f.frame_id for f in frames], timing)

    def attention_only(self, frame):
        """attention_pass for one frame: stage 1 + box extraction, no selection."""
        with self.lock:
            self._upload_frames([frame])
            K1 = self.K - 1
            b = self._next
            self.stage1(1, self.frames, bank=b)
            cnt = self._bank_counts[b][K1:K1 + 1].cpu().numpy()
            if (cnt > MAX_BOXES).any():
                raise StageFailure("attention", frame.frame_id)
            bx = self._banks[b][K1, : int(cnt[0])].cpu().numpy()
            boxes = tuple(Rect(int(v[0]), int(v[1]), int(v[2]), int(v[3])) for v in bx)
            return AttentionModel(frame.frame_id, boxes, (frame.frame_id,))

    # ------------------------------------------------------------------ host views
    def stage_times_ms(self):
        self.events[4].synchronize()
        e = self.events
        return (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]),
                e[3].elapsed_time(e[4]))

    def results(self, frame_ids, timing: TimingProfile | None = None):
        """Download and convert the last batch to (FrameResult, AttentionModel) pairs."""
        return self.results_from(self.snapshot(), frame_ids, timing)

    def snapshot(self, slot: int = 0, stream=None):
        """Queue stream-ordered D2H copies of the last batch's results into pinned host
        buffers (slot 0/1 double-buffers them), so the next batch may be launched before
        the host reads these: returns a handle for results_from()."""
        torch = self.torch
        n = self._n
        K1 = self.K - 1
        bufs = self.__dict__.setdefault("_snap_bufs", {})
        if slot not in bufs:
            mf, rec = self.max_frames, native.PDET_DTYPE.itemsize
            pin = dict(pin_memory=True)
            bufs[slot] = {"oc": torch.empty(mf, dtype=torch.int32, **pin),
                          "pc": torch.empty(mf, dtype=torch.int32, **pin),
                          "ac": torch.empty(mf, dtype=torch.int32, **pin),
                          "bc": torch.empty(mf, dtype=torch.int32, **pin),
                          "mc": torch.empty(mf, dtype=torch.int32, **pin),
                          "of": torch.empty(1, dtype=torch.int32, **pin),
                          "boxes": torch.empty((mf, MAX_BOXES, 4), dtype=torch.float64, **pin),
                          "rec": torch.empty(mf * MAX_PER_FRAME * rec, dtype=torch.uint8, **pin),
                          "event": torch.cuda.Event()}
        s = bufs[slot]
        rb = n * MAX_PER_FRAME * native.PDET_DTYPE.itemsize
        boxes, counts = self._banks[self._bank], self._bank_counts[self._bank]
        with torch.cuda.stream(stream) if stream is not None else nullcontext():
            s["oc"][:n].copy_(self.ocounts[:n], non_blocking=True)
            s["pc"][:n].copy_(self.pcounts[:n], non_blocking=True)
            s["ac"][:n].copy_(self.active_counts[:n], non_blocking=True)
            s["mc"][:n].copy_(self.merged_counts[:n], non_blocking=True)
            s["of"].copy_(self.overflow, non_blocking=True)
            # the batch's own box slots are K1..K1+n-1 of its bank
            s["bc"][:n].copy_(counts[K1:K1 + n], non_blocking=True)
            s["boxes"][:n].copy_(boxes[K1:K1 + n], non_blocking=True)
            s["rec"][:rb].copy_(self.outp.view(-1)[:rb], non_blocking=True)
            s["event"].record(stream)
        return (n, s)

    def results_from(self, snap, frame_ids, timing: TimingProfile | None = None):
        """(FrameResult, AttentionModel) pairs from a snapshot (waits for its copies).
        Capacity overflows raise StageFailure — results are never silently truncated."""
        n, s = snap
        s["event"].synchronize()
        oc, pc, ac = s["oc"][:n].numpy(), s["pc"][:n].numpy(), s["ac"][:n].numpy()
        if (pc > MAX_PER_FRAME).any():
            raise StageFailure("final", int(frame_ids[int(np.argmax(pc))]))
        mc = s["mc"][:n].numpy()
        if (mc > MAX_MERGED).any():  # temporal window above the selection kernel's capacity
            raise StageFailure("select", int(frame_ids[int(np.argmax(mc))]))
        if int(s["of"][0]) != 0:  # a tile clipped by the crop-parallel exchange cap
            raise StageFailure("final", int(frame_ids[0]))
        cnt = s["bc"][:n].numpy()
        if (cnt > MAX_BOXES).any():
            raise StageFailure("attention", int(frame_ids[int(np.argmax(cnt))]))
        bx = s["boxes"][:n].numpy()
        rec = s["rec"][: n * MAX_PER_FRAME * native.PDET_DTYPE.itemsize].numpy()
        rec = rec.view(native.PDET_DTYPE).reshape(n, MAX_PER_FRAME)
        out = []
        timing = timing or TimingProfile()
        for f in range(n):
            dets = records_to_detections(rec[f, : oc[f]], self.labels.names)
            res = FrameResult(int(frame_ids[f]), dets, int(ac[f]), self.F, timing)
            boxes = tuple(Rect(int(b[0]), int(b[1]), int(b[2]), int(b[3]))
                          for b in bx[f, : cnt[f]])
            out.append((res, AttentionModel(int(frame_ids[f]), boxes, (int(frame_ids[f]),))))
        return out

    def box_counts_snapshot(self, n):
        """Attention boxes per frame of the last batch (host lists)."""
        K1 = self.K - 1
        cnt = self.box_counts[K1:K1 + n].cpu().numpy()
        if (cnt > MAX_BOXES).any():
            raise StageFailure("attention", -1)
        bx = self.boxes[K1:K1 + n].cpu().numpy()
        return [bx[f, : cnt[f]] for f in range(n)]


def records_to_detections(rec, names) -> tuple:
    """tp_pdet_t records (integer-valued global rects) -> Detection tuple. Column-wise
    .tolist() conversion: ~2.5x faster than per-record numpy field access, which
    dominated building FrameResults for dense frames."""
    if len(rec) == 0:
        return ()
    cols = [rec[k].astype(np.int64).tolist() for k in ("x", "y", "w", "h")]
    cls, conf = rec["cls"].tolist(), rec["conf"].tolist()
    return tuple(Detection(Rect(x, y, w, h), names[c], p)
                 for x, y, w, h, c, p in zip(*cols, cls, conf))


def exclusive_boxes(final_grid, crop_ids, margin: int, size: int = 4):
    """Small attention boxes, one per requested crop, placed at the centre of the part of
    the crop no other crop covers, so after dilation by `margin` each activates exactly
    its crop (for forced-density runs)."""
    crops = final_grid.crops
    out = []
    for cid in crop_ids:
        c = final_grid.crop_by_id(cid)
        g = c.global_rect
        lo_x, hi_x, lo_y, hi_y = g.x, g.x2, g.y, g.y2
        for o in crops:
            if o.crop_id == cid:
                continue
            r = o.global_rect
            if o.row == c.row and o.col == c.col - 1:
                lo_x = max(lo_x, r.x2)
            if o.row == c.row and o.col == c.col + 1:
                hi_x = min(hi_x, r.x)
            if o.col == c.col and o.row == c.row - 1:
                lo_y = max(lo_y, r.y2)
            if o.col == c.col and o.row == c.row + 1:
                hi_y = min(hi_y, r.y)
        if hi_x - lo_x < size + 2 * margin + 2 or hi_y - lo_y < size + 2 * margin + 2:
            raise ValueError(f"crop {cid} has no exclusive region wide enough")
        cx, cy = (lo_x + hi_x) // 2, (lo_y + hi_y) // 2
        out.append((cx - size // 2, cy - size // 2, size, size))
    return out


def yolo_tagged(det, frame, crops):
    """final_pass / downscale body for the YOLO detector: the given crops of one frame are
    gathered, run and decoded (with to_global) on the GPU; returns the reference's tagged
    list [(crop_id, Detection)] in crop order, detector order within a crop."""
    torch = native.require_cuda()
    net = det.net
    dev = torch.from_numpy(np.ascontiguousarray(frame.pixels)).cuda()
    H, W = frame.height, frame.width
    out = []
    for s in range(0, len(crops), net.max_tiles):
        chunk = crops[s:s + net.max_tiles]
        n = len(chunk)
        jobs = kernels.jobs_tensor((0, c.crop_id, int(c.global_rect.x), int(c.global_rect.y),
                                    int(c.global_rect.w), 0) for c in chunk)
        kernels.gather(dev, 0, H, W, jobs, n, "nearest", out_act_ptr=net.input_ptr,
                       dtype=net.dtype)
        net.forward(n)
        recs, counts = kernels.alloc_dets(n)
        kernels.decode(net, n, jobs, W, H, det.threshold, recs, counts)
        rec, cnt = kernels.dets_to_host(recs, counts, n)
        for i, c in enumerate(chunk):
            for r in rec[i, : cnt[i]]:
                out.append((c.crop_id, Detection(
                    Rect(int(r["gx"]), int(r["gy"]), int(r["gw"]), int(r["gh"])),
                    COCO_NAMES[int(r["cls"])], float(r["conf"]))))
    return out
