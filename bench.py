"""Benchmark: synthetic 4K attention-pipeline stream, frames/sec (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Workload (BASELINE.json configs[1]): the 300-frame synthetic 3840x2160 clip of
synthetic.bench_clip (frames 0-99 sparse, 100-199 dense, 200-299 mixed scenes, seed 0;
the reference generator's semantics), preset "1 att, 3 fin, 20 over", random-init
YOLO v2-608 (seed 0). One step = one batch of --batch frames through the full two-stage
pipeline (stage-1 YOLO on 2 attention tiles/frame, selection, stage-2 YOLO on the active
crops, NMS + merge). With N GPUs the clip is N x 300 frames (segment r = bench_clip with
seed r) sharded contiguously over the ranks (frame-DP; rank r > 0 seeds its temporal
window by recomputing stage 1 on the frame before its shard); weak scaling.

* value: frames/sec with the clip resident in HBM (each batch's input is 30 4K frames,
  746 MB > 126 MB L2, so no flush is needed between steps); stage 1 of batch k+1 runs on
  a second stream while batch k finishes (the run_stream schedule); at N > 1 every batch's
  results are all-gathered over NCCL (the fused C-ABI gather) inside the timed region.
* e2e: the same metric through the drop-in API — stream.run_stream (N = 1) /
  distributed.run_stream_sharded (N > 1) — with HOST frames in pinned memory: per step
  the H2D copy of the batch, the D2H of its results and the construction of every
  FrameResult / Detection object are inside the timed region.
* precision (default "fp32"): the fp32-parity plan — activations as exact fp16 hi/lo
  pairs, fp32 accumulation — the mode inside the north-star 1e-3 score tolerance
  (tests/test_gpu_e2e_parity.py); --precision fp16 runs the ~2x faster 16-bit mode.
* roofline: the dominant kernel family is the tcgen05 implicit-GEMM conv (23 launches per
  YOLO forward + 1 maxpool): achieved = 62.938 GFLOP x tiles / the union of the measured
  forward intervals (algorithmic FLOPs; `executed_tflops` counts the parity plan's K).
* cpu_baseline / --impl reference: the reference pipeline (oracle/pipeline_ref, pinned to
  reference goldens) with the fp32 CPU YOLO (oracle/yolo_ref) on the box's host cores, on
  frames spread over the same sparse/dense/mixed clip; the GPU arm's cpu_baseline also
  checks those frames' results against the GPU's.
* sub_results (N = 1): BASELINE configs[2] (all-crops), [3] (8K), [4] (density 0.5,
  injected stage 1) and the fp16 mode, each a short timed run with its own clock record.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PRESET = "1 att, 3 fin, 20 over"
FRAMES = {"4k": (3840, 2160), "8k": (7680, 4320)}
METRIC = "frames/sec, synthetic 4K & 8K video, 1/2/4/8 B200; crops/sec; % roofline"
# our kernels per step (CUPTI table, profiles/r02_step_kernel_table.txt): a YOLO forward is
# 23 convs + the route max pool + the reorg gather, minus the convs fused into their
# producer (fp32 plan: layer 5 inside layer 4's kernel -> 24); stage 1 = gather + forward +
# decode + attention boxes; finish = select + build jobs + gather + forward + decode +
# collect + postprocess


def launches_per_step(fwd: int) -> int:
    return (1 + fwd + 1 + 1) + (1 + 1 + 1 + fwd + 1 + 1 + 1)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=30)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--resample", default="nearest", choices=["nearest", "bilinear"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp32x2", "fp16", "bf16"],
                    help="activation precision: fp32 = the parity plan (default: fp16 hi/lo "
                         "pairs up to 152^2, then fp16 hi + e4m3 lo planes); fp32x2 = hi/lo "
                         "fp16 pairs on every layer; fp16/bf16 = 16-bit activations")
    ap.add_argument("--profile", action="store_true",
                    help="CUPTI kernel table of the timed steps to stderr (not a bench run)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub_results runs")
    ap.add_argument("--no-lookahead", action="store_true",
                    help="stage 1 and 2 of a batch back to back on one stream")
    ap.add_argument("--frame", default="4k", choices=sorted(FRAMES))
    ap.add_argument("--preset", default=PRESET)
    ap.add_argument("--mode", default="pipeline", choices=["pipeline", "allcrops"],
                    help="allcrops = the run_allcrops_baseline comparator (config 3)")
    ap.add_argument("--density", type=float, default=None,
                    help="inject stage-1 boxes activating this fraction of the final grid "
                         "(config 5 density sweep; stage 1 is skipped)")
    ap.add_argument("--clip-frames", type=int, default=300)
    return ap.parse_args(argv)


# --------------------------------------------------------------------------- launch


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_launch_ranks(args) -> bool:
    """`--gpus N` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run and return True (this process only waits). Fails loudly when
    the box has fewer GPUs than asked."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and os.environ.get("TP_BENCH_SHARED_GPU") != "1":
        sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def arm_config(args, world: int) -> dict:
    """Workload description, identical for the B200 arm and the reference arm."""
    W, H = FRAMES[args.frame]
    kind = "all-crops baseline" if args.mode == "allcrops" else "attention pipeline"
    dens = "" if args.density is None else f" (injected stage 1, density {args.density})"
    return {"workload": f"{args.frame.upper()} {kind}{dens} on the synthetic bench clip "
                        f"({args.clip_frames} frames per GPU: sparse/dense/mixed thirds, "
                        f"segment r = seed r), preset '{args.preset}', random-init YOLO "
                        "v2-608 (seed 0, calibrated head)",
            "frame": [W, H], "frames_per_step": args.batch, "per_gpu_frames": args.clip_frames,
            "resample": args.resample, "parallelism": f"frame-dp{world}",
            "precision": args.precision}


def lscpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region (NVML in-process every
    20 ms; nvidia-smi every 200 ms if NVML is unavailable)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                   "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.nvml = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.nvml = pynvml
        except Exception:
            self.nvml = None

    def _sample_nvml(self):
        nv = self.nvml
        mhz = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
        bits = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
        flags = ["Active" if bits & self.REASON_BITS[k] else "Not Active"
                 for k in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                           "sw_power_cap")]
        return [str(mhz), str(self.max_mhz)] + flags

    def _run(self):
        while not self.stop.is_set():
            try:
                if self.nvml is not None:
                    self.samples.append(self._sample_nvml())
                    self.stop.wait(0.02)
                    continue
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self.nvml else "nvidia-smi"}


# --------------------------------------------------------------------------- CPU arm


def sample_frames(n_clip: int, k: int) -> list[int]:
    """k frame indices spread evenly over the clip (sparse / dense / mixed thirds)."""
    return [min(n_clip - 1, int((i + 0.5) * n_clip / k)) for i in range(k)]


def cpu_reference_frames(args, fids, objs, threads=None):
    """The reference pipeline + fp32 CPU YOLO on the given clip frames (each with its
    K=2 history: the previous frame's attention, computed outside the timing — in a
    sequential run it belongs to the previous frame's step). Returns per-frame seconds,
    results and tiles."""
    import torch

    from oracle import e2e as E
    from oracle import pipeline_ref as R
    from paper_1810_10551_b200 import synthetic, yolo

    W, H = FRAMES[args.frame]
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cache = {}

    def pixels_of(f):
        if f not in cache:
            cache[f] = synthetic.render_frame(W, H, objs[f])
        return cache[f]
    det = E.CpuYolo(pixels_of, yolo.COCO_NAMES, threads=threads)
    plan = R.Plan(W, H, 1, 3, 20)
    out = []
    for f in fids:
        hist = []
        if f > 0:
            det.prefetch(f - 1, plan.att[3])
            hist = [R.attention_pass(plan, f - 1, det, 0.3)]
        t0 = time.perf_counter()
        dets, active, att = E.reference_frame(plan, f, det, hist)
        dt = time.perf_counter() - t0
        out.append({"frame": f, "seconds": dt, "dets": dets, "active": active, "att": att,
                    "tiles": len(plan.att[3]) + len(active)})
        for k in [k for k in det.raw if k[0] < f - 1]:  # bounded memory
            det.raw.pop(k, None)
            det.tiles.pop(k, None)
    return out, threads


def run_reference(args, rank, world):
    """--impl reference: the reference pipeline on the host cores, one clip frame per
    step, frames spread over the sparse/dense/mixed clip (same config as the GPU arm)."""
    if rank != 0:
        return
    from paper_1810_10551_b200 import synthetic

    W, H = FRAMES[args.frame]
    objs = synthetic.bench_clip(W, H, args.clip_frames, seed=0)
    n = args.warmup + args.steps
    fids = sample_frames(len(objs), n)
    res, threads = cpu_reference_frames(args, fids, objs)
    timed = res[args.warmup:]
    total = sum(r["seconds"] for r in timed)
    v = args.steps / total
    tiles = sum(r["tiles"] for r in timed) / len(timed)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(args, world),
            "step": "one clip frame per step (bounded CPU sample of the workload): frames "
                    f"{[r['frame'] for r in timed]} spread over the sparse/dense/mixed clip",
            "workload_stats": {"tiles_per_frame": tiles},
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads,
                             "kind": "port", "cpu": lscpu_model(),
                             "sample": f"{args.steps} frames spread over the clip: oracle "
                                       "reference pipeline + torch-CPU fp32 YOLO v2-608"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_with_parity(args, objs):
    """GPU arm's cpu_baseline: 3 frames (one per scene kind), timed on the host cores,
    and their results compared with the GPU's (oracle.e2e contract)."""
    from oracle import e2e as E
    from paper_1810_10551_b200 import pipeline as P, synthetic, yolo

    W, H = FRAMES[args.frame]
    n = len(objs)
    fids = [n // 6, n // 2, 5 * n // 6]
    res, threads = cpu_reference_frames(args, fids, objs)
    total = sum(r["seconds"] for r in res)
    settings = P.PipelineSettings.from_preset(args.preset)
    gdet = yolo.YoloB200Detector(precision=args.precision)
    exact = 0
    notes = []
    for r in res:
        f = r["frame"]
        fr = [P.Frame(i, W, H, synthetic.render_frame(W, H, objs[i]))
              for i in ([f - 1] if f else []) + [f]]
        g = list(P.run_sequence(fr, settings, gdet))[-1]
        got = [((d.rect.x, d.rect.y, d.rect.w, d.rect.h), d.class_label, d.confidence)
               for d in g.detections]
        cmp = E.compare_dets(r["dets"], got)
        ok = cmp["ok"] and g.active_count == len(r["active"])
        exact += ok
        notes.append({"frame": f, "match": bool(ok), "dets": cmp["n"],
                      "score_rel": cmp["score_rel"], "order_flips": cmp["order_flips"],
                      "rounding_1px": cmp["n_1px"]})
    return {"value": len(res) / total, "unit": "frames/s", "cores": threads, "kind": "port",
            "cpu": lscpu_model(),
            "sample": f"frames {fids} (sparse, dense, mixed), {total:.1f} s: oracle reference "
                      "pipeline + torch-CPU fp32 YOLO v2-608, all host threads",
            "parity": {"frames": len(res), "match": exact, "detail": notes}}


# --------------------------------------------------------------------------- GPU arm


class DeviceLoop:
    """The device-resident step loop: batch k's stage 1 on `att` (look-ahead) while batch
    k-1 finishes on the main stream; at world > 1 the batch's results are all-gathered
    (distributed.BatchGather, fused NCCL) after its finish. Conv forwards are bracketed
    by events on their own streams for the roofline."""

    def __init__(self, eng, clip, B, mode, density, lookahead, world, group=None):
        import torch

        self.torch, self.eng, self.clip, self.B = torch, eng, clip, B
        self.mode, self.lookahead = mode, lookahead and eng.net1 is not eng.net
        self.att = torch.cuda.Stream() if self.lookahead else None
        self.att_done = [torch.cuda.Event() for _ in range(2)]
        self.fin_done = [torch.cuda.Event() for _ in range(2)]
        self.gather = None
        if world > 1:
            from paper_1810_10551_b200.distributed import BatchGather
            self.gather = BatchGather(B, world, group)
        self.fwd = []  # (start, end, tiles or None=device count, step)
        self.n2 = []   # per step: device tensor holding the stage-2 tile count
        self.injected = []
        if density is not None:  # boxes at the centres of round(d*F) crops per frame
            import random as _random

            from paper_1810_10551_b200.engine import exclusive_boxes
            fin = eng.plan.final_grid.crops
            k = int(round(density * len(fin)))
            rng = _random.Random(1234)
            for _ in range(4):  # 4 batches of injected boxes, uploaded once
                boxes = [exclusive_boxes(
                    eng.plan.final_grid, [fin[c].crop_id for c in sorted(rng.sample(range(len(fin)), k))],
                    eng.settings.attention_margin_px) for _ in range(B)]
                arr = np.zeros((B, 256, 4))
                cnt = np.zeros(B, dtype=np.int32)
                for f, bl in enumerate(boxes):
                    cnt[f] = len(bl)
                    arr[f, : len(bl)] = bl
                self.injected.append((torch.from_numpy(arr).cuda(), torch.from_numpy(cnt).cuda()))
        self.density = density
        self._wrap(eng.net)
        if eng.net1 is not eng.net:
            self._wrap(eng.net1)
        self.record = False

    def _wrap(self, net):
        orig = net.forward
        torch = self.torch

        def timed(n, n_tiles_dev=None, stream=None):
            if not self.record:
                return orig(n, n_tiles_dev=n_tiles_dev, stream=stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            orig(n, n_tiles_dev=n_tiles_dev, stream=stream)
            b.record(stream)
            self.fwd.append((a, b, None if n_tiles_dev is not None else n))
        net.forward = timed

    def frames(self, i):
        s = (i * self.B) % self.clip.shape[0]
        return self.clip[s:s + self.B]

    def stage1(self, i):
        torch, eng = self.torch, self.eng
        bank = (self.base + i) % 2
        if self.mode != "pipeline" or self.density is not None:
            K1 = eng.K - 1
            if self.density is not None:
                arr, cnt = self.injected[i % len(self.injected)]
                eng._banks[bank][K1:K1 + self.B].copy_(arr)
                eng._bank_counts[bank][K1:K1 + self.B].copy_(cnt)
            else:  # all-crops: one full-frame box per frame
                eng._banks[bank][K1:K1 + self.B, 0] = eng.full_box
                eng._bank_counts[bank][K1:K1 + self.B] = 1
            self.att_done[i % 2].record()
            return
        st = self.att if self.lookahead else torch.cuda.current_stream()
        if self.lookahead and i >= 2:
            st.wait_event(self.fin_done[i % 2])  # bank reuse: batch i-2's selection read it
        with torch.cuda.stream(st):
            eng.stage1(self.B, self.frames(i), stream=st, bank=bank)
            self.att_done[i % 2].record(st)

    def finish(self, i):
        torch, eng = self.torch, self.eng
        cur = torch.cuda.current_stream()
        cur.wait_event(self.att_done[i % 2])
        eng.finish(self.B, self.frames(i), bank=(self.base + i) % 2)
        if self.record:
            n2 = torch.empty(1, dtype=torch.int32, device="cuda")
            n2.copy_(eng.n_jobs2)
            self.n2.append(n2)
        if self.gather is not None:
            self.gather.launch(eng, i, self.B, False, want_records=False)
        self.fin_done[i % 2].record()

    def run(self, first, last):
        """Steps first..last-1 (stage 1 of `first` must not have been launched)."""
        self.base = self.eng._next - first  # bank of step i = (base + i) % 2
        self.stage1(first)
        for i in range(first, last):
            if self.lookahead and i + 1 < last:
                self.stage1(i + 1)
                self.finish(i)
            else:
                self.finish(i)
                if i + 1 < last:
                    self.stage1(i + 1)

    def conv_stats(self, t0):
        """(union of forward intervals in ms, algorithmic FLOPs) over the recorded steps."""
        from paper_1810_10551_b200 import yolo

        n2 = [int(t.item()) for t in self.n2]
        iv, flops, k2 = [], 0.0, 0
        for a, b, n in self.fwd:
            if n is None:  # stage-2 forward: device-side tile count, in step order
                n = n2[k2] if k2 < len(n2) else 0
                k2 += 1
            iv.append((t0.elapsed_time(a), t0.elapsed_time(b)))
            flops += n * yolo.GFLOP_PER_TILE * 1e9
        iv.sort()
        busy, end = 0.0, -1e30
        for s, e in iv:
            if e <= end:
                continue
            busy += e - max(s, end)
            end = e
        return busy, flops, sum(n2)


def gpu_run(args, rank, world, local, shared_gpu, group, sub=False):
    """One GPU-arm measurement: (line fields, eng, clip objects) — the device-resident
    timed loop; the caller adds e2e / cpu_baseline / sub_results."""
    import torch
    import torch.distributed as dist

    from paper_1810_10551_b200 import pipeline as P, synthetic, yolo
    from paper_1810_10551_b200.engine import AttentionPipelineB200

    W, H = FRAMES[args.frame]
    B = args.batch
    objs = synthetic.bench_clip(W, H, args.clip_frames, seed=rank)
    objs = [objs[k % len(objs)] for k in range(-(-len(objs) // B) * B)]
    n_clip = len(objs)
    settings = P.PipelineSettings.from_preset(args.preset)
    eng = AttentionPipelineB200(settings, W, H, max_frames=B, resample=args.resample,
                                precision=args.precision)
    clip = torch.empty((n_clip, H, W, 3), dtype=torch.uint8, device="cuda")
    for i in range(0, n_clip, 10):
        synthetic.render_frames_device(W, H, objs[i:i + 10], out=clip[i:i + 10])
    eng.reset_history(())
    if rank > 0 and args.mode == "pipeline" and args.density is None:
        # frame-DP boundary: the frame before this shard is the last of segment r-1
        prev = synthetic.bench_clip(W, H, args.clip_frames, seed=rank - 1)[-1]
        pf = synthetic.render_frames_device(W, H, [prev])
        eng.prime_history(pf, 1)
    mode = "allcrops" if args.mode == "allcrops" else "pipeline"
    loop = DeviceLoop(eng, clip, B, mode, args.density, not args.no_lookahead, world, group)
    n_steps = args.warmup + args.steps
    loop.run(0, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = None
    if args.profile:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
        prof.__enter__()
    loop.record = True
    with ClockSampler(0 if shared_gpu else local) as clocks:
        torch.cuda.synchronize()
        t0.record()
        loop.run(args.warmup, n_steps)
        t1.record()
        torch.cuda.synchronize()
    loop.record = False
    ms = t0.elapsed_time(t1)
    if prof is not None:
        prof.__exit__(None, None, None)
        kernel_table(prof, ms, args.steps)
    if world > 1:
        mt = torch.tensor([ms], device="cuda")
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())
    value = args.steps * B * world / (ms / 1e3)
    busy, flops, tiles2 = loop.conv_stats(t0)
    conv_tflops = flops / (busy / 1e3) / 1e12
    stage1 = eng.A * B * args.steps if mode == "pipeline" and args.density is None else 0
    tiles_per_frame = (stage1 + tiles2) / (args.steps * B)
    fields = {"value": value, "ms_per_step": ms / args.steps, "clocks": clocks.summary(),
              "conv_tflops": conv_tflops, "conv_busy_ms": busy, "tiles_per_frame": tiles_per_frame,
              "kernels": eng.net.kernel_summary(),
              "forward_launches": 25 - len(eng.net.fused_steps)}
    return fields, eng, objs, clip


PRECISION_NOTE = {
    "fp32": "fp32-parity (HL8): every activation but the layer-0 pixels and the fp32 head is "
            "an fp16 hi plane + an e4m3 lo plane e4m3((x - hi) * 2^11); each conv runs "
            "kind::f16 MMAs on hi and kind::f8f6f4 MMAs on lo into one fp32 accumulator; fp32 "
            "epilogue; layer 5 runs inside layer 4's kernel",
    "fp32x2": "fp32-parity: activations as fp16 hi/lo pairs on every layer (2x K), fp32 "
              "accumulation and epilogue",
}
EXECUTED_NOTE = {
    "fp32": "tensor-core work issued, in kind::f16-rate GFLOP: fp16 hi + e4m3 lo (f8f6f4 at "
            "2x rate) make 1.5x K on every layer but layer 0 ({:.1f} GFLOP per tile)",
    "fp32x2": "tensor-core FLOPs issued: hi/lo activations double K on every layer but "
              "layer 0 ({:.1f} GFLOP per tile)",
}


def measured_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def peak_tflops() -> float:
    """Dense bf16 (= fp16) TFLOP/s sustained, MEASURED_PEAKS.json (driver-written), else the
    profiling recipe's fallback."""
    return float(measured_peaks().get("bf16_tflops_sustained", 1391.0))


def roofline(args, f):
    from paper_1810_10551_b200 import yolo

    peaks = measured_peaks()
    peak = peak_tflops()
    traffic = {}
    tfile = {"fp32": "r02h_conv_traffic_fp32.json",
             "fp32x2": "r01_conv_traffic_fp32.json"}.get(args.precision, "r01_conv_traffic.json")
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", tfile)))
    except Exception:
        pass
    exec_gf = yolo.exec_gflop_per_tile(args.precision)
    exec_scale = exec_gf / yolo.GFLOP_PER_TILE
    a = f["conv_tflops"]
    return {"bound": "tensor", "kernel": "YOLO v2 conv stack: 23 tcgen05 launches per forward "
                                         f"({f['kernels']}) + 1 maxpool",
            "achieved": a, "peak": peak, "unit": "TFLOP/s", "frac": a / peak,
            "traffic": traffic.get("dram_MB_per_tile", 0) * 1e6 if traffic else None,
            "traffic_unit": f"DRAM bytes per 608^2 tile, ncu --set full (profiles/{tfile})",
            "algorithmic_bytes_per_tile": traffic.get("algorithmic_MB_per_tile", 0) * 1e6
            if traffic else None,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else
                           "B200_PROFILING.md fallback",
            "algorithmic": f"{yolo.GFLOP_PER_TILE:.3f} GFLOP per 608^2 tile",
            "timing": "union of the CUDA-event intervals of every YOLO forward in the timed "
                      "steps (stage 1 and stage 2 overlap on two streams)",
            "executed_tflops": a * exec_scale, "executed_frac": a * exec_scale / peak,
            "executed": EXECUTED_NOTE.get(args.precision, "same as algorithmic").format(exec_gf),
            "conv_share_of_step": f["conv_busy_ms"] / (f["ms_per_step"] * args.steps)}


def run_e2e(args, eng, objs, clip, rank, world, group):
    """The same metric through the drop-in API with pinned HOST frames: run_stream
    (N = 1) / run_stream_sharded (N > 1) over steps x batch frames per rank, FrameResults
    built on the host. Wall clock around the call, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1810_10551_b200 import distributed as D, native, pipeline as P, synthetic
    from paper_1810_10551_b200.engine import MAX_PER_FRAME
    from paper_1810_10551_b200.stream import run_stream

    W, H = FRAMES[args.frame]
    B = args.batch
    settings = P.PipelineSettings.from_preset(args.preset)
    frame_bytes = W * H * 3
    # pinned host copy of the rank's clip: all of it up to 16 GB (4 GB per rank when
    # several ranks share the host); a capped copy takes evenly spaced frames so the
    # sparse / dense / mixed mix is kept
    cap_bytes = (16 << 30) if world == 1 else (4 << 30)
    n_host = min(clip.shape[0], max(B, cap_bytes // frame_bytes))
    pick = np.linspace(0, clip.shape[0] - 1, n_host).round().astype(np.int64)
    host = torch.empty((n_host, H, W, 3), dtype=torch.uint8, pin_memory=True)
    for i in range(0, n_host, 16):
        host[i:i + 16].copy_(clip[torch.from_numpy(pick[i:i + 16]).cuda()].cpu())
    prev = None
    if rank > 0:
        p = synthetic.bench_clip(W, H, args.clip_frames, seed=rank - 1)[-1]
        prev = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
        prev.copy_(synthetic.render_frames_device(W, H, [p])[0].cpu())

    def frames_for(n_per_rank, base_id):
        """Global clip of world x n_per_rank frames; only this rank's shard (and the
        frame before it) carries pixels."""
        out = []
        for r in range(world):
            for j in range(n_per_rank):
                fid = base_id + r * n_per_rank + j
                px = None
                if r == rank:
                    px = host[j % n_host].numpy()
                elif r == rank - 1 and j == n_per_rank - 1:
                    px = prev.numpy()
                out.append(P.Frame(fid, W, H, px))
        return out

    def call(frames):
        if world == 1:
            return run_stream(frames, settings, engine=eng)
        return D.run_stream_sharded(frames, settings, engine=eng, group=group)

    call(frames_for(args.warmup * B, 10 ** 6))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    frames = frames_for(args.steps * B, 0)
    t0 = time.perf_counter()
    res = call(frames)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        mt = torch.tensor([dt], device="cuda")
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        dt = float(mt.item())
    n_dets = sum(len(r.detections) for r in res)
    rec = native.PDET_DTYPE.itemsize
    d2h = B * (MAX_PER_FRAME * rec + 5 * 4) + 256 * 32 * B  # records, counts, box lists
    if world > 1:
        d2h = world * (B * D.GATHER_CAP * rec + 4 * (4 + 2 * B)) if rank == 0 else 0
    return {"value": args.steps * B * world / dt, "unit": "frames/s",
            "h2d_bytes_per_step": B * frame_bytes, "d2h_bytes_per_step": int(d2h),
            "api": "stream.run_stream" if world == 1 else "distributed.run_stream_sharded",
            "frame_results": len(res), "detections": n_dets,
            "timing": "host wall clock around the API call (pinned host frames in, "
                      "FrameResults out; H2D, D2H and result objects inside), max over ranks"}


def sub_results(args, rank, world, local, shared_gpu, group):
    """BASELINE configs[2], [3], [4] and the fp16 mode as short timed runs (N = 1)."""
    import gc

    import torch

    runs = [
        ("configs[2]: all-crops baseline, 4K", ["--mode", "allcrops"]),
        ("configs[3]: attention pipeline, 8K (60-frame clip)", ["--frame", "8k", "--clip-frames", "60"]),
        ("configs[4]: density 0.5 (injected stage 1), 4K", ["--density", "0.5"]),
        ("configs[4]: density 0.5 (injected stage 1), 8K", ["--density", "0.5", "--frame", "8k",
                                                            "--clip-frames", "60"]),
        ("fp16 fast mode (scores within ~5e-3), 4K", ["--precision", "fp16"]),
    ]
    out = []
    for name, extra in runs:
        sa = parse(["--steps", "5", "--warmup", "2", "--batch", str(args.batch)] + extra)
        try:
            f, eng, _, clip = gpu_run(sa, rank, world, local, shared_gpu, group, sub=True)
        except Exception as exc:  # a sub-run must never sink the headline line
            out.append({"config": name, "error": str(exc)[:300]})
            continue
        out.append({"config": name, "args": " ".join(extra), "value": f["value"],
                    "unit": "frames/s", "ms_per_step": f["ms_per_step"], "steps": sa.steps,
                    "warmup": sa.warmup, "tiles_per_frame": f["tiles_per_frame"],
                    "crops_per_sec": f["value"] * f["tiles_per_frame"],
                    "roofline_frac": f["conv_tflops"] / peak_tflops(),
                    "conv_tflops": f["conv_tflops"], "clocks": f["clocks"]})
        del eng, clip
        gc.collect()
        torch.cuda.empty_cache()
    return out


def kernel_table(prof, ms: float, steps: int) -> None:
    """Per-kernel device time over the timed steps (warm, real overlap), to stderr."""
    import torch

    agg: dict[str, list] = {}
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ev.time_range.elapsed_us() / 1e3
        a[1] += 1
    busy = sum(v[0] for v in agg.values())
    print(f"# kernel table: {steps} steps, {ms:.3f} ms wall (device), {busy:.3f} ms kernel busy",
          file=sys.stderr)
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{100 * t / ms:6.2f}% {t / steps:9.3f} ms/step {n // steps:5d}/step  {k}",
              file=sys.stderr)


def main():
    args = parse()
    if maybe_launch_ranks(args):
        return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist

    # TP_BENCH_SHARED_GPU=1: logic check of the multi-rank path on a one-GPU box (every
    # rank on cuda:0, gloo collectives, ranks never wait on each other's kernels); such a
    # run is flagged in its line and is not a scaling measurement
    shared_gpu = os.environ.get("TP_BENCH_SHARED_GPU") == "1"
    if not shared_gpu and torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks but {torch.cuda.device_count()} GPUs")
    dev_idx = 0 if shared_gpu else local
    torch.cuda.set_device(dev_idx)
    group = None
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    f, eng, objs, clip = gpu_run(args, rank, world, local, shared_gpu, group)
    e2e = None if args.no_e2e else run_e2e(args, eng, objs, clip, rank, world, group)
    cpu = None
    subs = None
    if rank == 0 and world == 1:
        del clip
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_with_parity(args, objs[: args.clip_frames])
    if world == 1 and not args.no_sub and args.mode == "pipeline" and args.density is None \
            and args.frame == "4k" and args.precision == "fp32":
        del eng
        subs = sub_results(args, rank, world, local, shared_gpu, group)
    if rank == 0:
        line = {
            "metric": METRIC, "value": f["value"], "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": f["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "precision": PRECISION_NOTE.get(
                args.precision, f"{args.precision} operands/activations, fp32 accumulation "
                                "(tcgen05 kind::f16)"),
            "config": arm_config(args, world),
            "workload_stats": {"tiles_per_frame": f["tiles_per_frame"],
                               "crops_per_sec": f["value"] * f["tiles_per_frame"],
                               "l2": f"inputs exceed L2 ({args.batch * FRAMES[args.frame][0] * FRAMES[args.frame][1] * 3 / 1e6:.0f} MB per step)",
                               "schedule": "stage-1 look-ahead on a second stream"
                               if not args.no_lookahead else "sequential stages",
                               **({"shared_gpu_logic_check": "all ranks on cuda:0 over gloo: "
                                   "not a scaling measurement"} if shared_gpu else {})},
            "roofline": roofline(args, f),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step(f["forward_launches"]) * args.steps,
            "clocks": f["clocks"],
        }
        if subs is not None:
            line["sub_results"] = subs
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
