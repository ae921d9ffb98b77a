"""``run`` entry point: the reference's ``cmd_run``
(pkg/src/tilepipe/cli.py:159-200) with a ``yolo-b200`` detector kind.

    python -m paper_1810_10551_b200.cli run --config run.ini [--mode pipeline|allcrops|downscale]
        [--results out.jsonl] [--timing out.csv]

Config: the reference's INI schema (``frameio.read_run_config``): ``[pipeline]`` preset or
rows/overlaps, ``[detector] kind = yolo-b200 | oracle`` (+ ``batch`` for yolo-b200),
``[paths] frames / ground_truth / results / timing``, optional ``[frame]``. A yolo-b200
pipeline run streams the frames directory through ``run_stream`` (disk -> pinned -> HBM
overlapped with the GPU); an oracle run is the reference's ground-truth detector called per
crop with every other stage on the GPU kernels. Output: byte-stable results JSON lines,
the timing CSV, and the reference's summary lines.
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time
from pathlib import Path

from . import frameio
from . import pipeline as P

RUN_MODES = ("pipeline", "allcrops", "downscale")


class UsageError(Exception):
    pass


def _print_run_summary(results, wall_s: float, mode: str) -> None:
    count = len(results)
    fps = count / wall_s if wall_s > 0 else 0.0
    print(f"mode={mode} frames={count} wall_s={wall_s:.3f} fps={fps:.2f}")
    if results:
        per_frame = [r.timing.total_ms for r in results]
        print("per_frame_ms"
              f" min={min(per_frame):.1f}"
              f" mean={statistics.fmean(per_frame):.1f}"
              f" p50={statistics.median(per_frame):.1f}"
              f" max={max(per_frame):.1f}")
        active = sum(r.active_count for r in results)
        total = sum(r.total_count for r in results)
        share = active / total if total else 0.0
        print(f"crops active={active} total={total} active_share={share:.3f}")


def _frames(config: frameio.RunConfig, gt_by_frame):
    if config.frames_dir is not None:
        source = frameio.FrameSource.open(config.frames_dir)
        if config.frame_width is not None and (
                (config.frame_width, config.frame_height) != (source.width, source.height)):
            raise UsageError(f"config says {config.frame_width}x{config.frame_height} but "
                             f"frames are {source.width}x{source.height}")
        return source, source.width, source.height
    w, h = config.frame_width, config.frame_height
    return [P.Frame(fid, w, h) for fid in sorted(gt_by_frame)], w, h


def run(config: frameio.RunConfig, mode: str = "pipeline"):
    """Evaluate a configured run; returns the FrameResults in frame order."""
    from .stream import run_stream
    from .yolo import YoloB200Detector

    if mode not in RUN_MODES:
        raise UsageError(f"mode must be one of {RUN_MODES}, got {mode!r}")
    settings = config.settings
    gt_by_frame = {}
    if config.ground_truth_path is not None:
        gt_by_frame = frameio.read_ground_truth(config.ground_truth_path)
    source, width, height = _frames(config, gt_by_frame)
    if config.detector == "yolo-b200":
        if mode == "pipeline":
            return run_stream(source, settings, batch=config.batch)
        det = YoloB200Detector()
    else:
        det = P.oracle_for_scene(width, height, settings, gt_by_frame,
                                 config.visibility_threshold, min_tile_px=config.min_tile_px)
        if mode == "pipeline":
            frames = source.frames() if hasattr(source, "frames") else source
            return list(P.run_sequence(frames, settings, det))
    frames = source.frames() if hasattr(source, "frames") else source
    if mode == "downscale":
        return [P.run_downscale_baseline(f, det, settings) for f in frames]
    return [P.run_allcrops_baseline(f, settings, det) for f in frames]


def cmd_run(args) -> int:
    try:
        config = frameio.read_run_config(args.config)
    except (OSError, ValueError) as exc:
        raise UsageError(str(exc)) from exc
    results_path = Path(args.results) if args.results else config.results_path
    if args.timing:
        timing_path = Path(args.timing)
    elif config.timing_path is not None:
        timing_path = config.timing_path
    else:
        timing_path = results_path.with_name(results_path.stem + "_timing.csv")
    started = time.perf_counter()
    results = run(config, args.mode)
    wall_s = time.perf_counter() - started
    frameio.write_results(results, results_path)
    frameio.write_timing_csv(results, timing_path)
    _print_run_summary(results, wall_s, args.mode)
    print(f"results={results_path} timing={timing_path}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1810_10551_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="evaluate a configured frame sequence")
    r.add_argument("--config", required=True)
    r.add_argument("--mode", default="pipeline", choices=RUN_MODES)
    r.add_argument("--results")
    r.add_argument("--timing")
    args = ap.parse_args(argv)
    try:
        return cmd_run(args)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
