"""Frame-sharded run_stream (reference dispatch rule
distribution/client.py:82-96 and run_stream :294-377): a clip split into contiguous
shards over ranks, each rank seeding its K=2 window by recomputing stage 1 on the frame
before its shard, results all-gathered per batch so rank 0 holds every FrameResult in
order.

* world 2 on one GPU: two processes share cuda:0 over gloo (host-side collectives: no
  rank ever waits on another rank's kernel), rank 0's results must equal a single-process
  run_sequence of the same clip — including the frame right after the shard boundary;
  a bad frame on rank 1 makes both ranks raise StreamAborted (no hang);
* world 1 over NCCL: the same code through the fused C-ABI gather (tp_nccl_gather_dets).
Each run is a subprocess so process groups never leak into other tests."""

import os
import pickle
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent("""
    import os, pickle, sys, numpy as np, torch, torch.distributed as dist
    from paper_1810_10551_b200 import synthetic, pipeline as P
    from paper_1810_10551_b200.distributed import run_stream_sharded
    from paper_1810_10551_b200.stream import StreamAborted
    backend, out, bad = sys.argv[1], sys.argv[2], int(sys.argv[3])
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo")
    rank = dist.get_rank()
    W, H = 3840, 2160
    objs = synthetic.bench_clip(W, H, 9, seed=0)[:7]      # sparse, dense, mixed frames
    frames = [P.Frame(100 + i, W, H, synthetic.render_frame(W, H, o)) for i, o in enumerate(objs)]
    if bad >= 0:
        frames[bad] = P.Frame(100 + bad, 1280, 720, np.zeros((720, 1280, 3), np.uint8))
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    try:
        res = run_stream_sharded(frames, settings, batch=2)
        payload = ("ok", [(r.frame_id, r.detections, r.active_count, r.total_count,
                           r.timing.per_worker[0][0]) for r in res])
    except StreamAborted as exc:
        payload = ("aborted", exc.cursor, [r.frame_id for r in exc.completed], str(exc))
    with open(out + f".{rank}", "wb") as fh:
        pickle.dump(payload, fh)
    dist.destroy_process_group()
""")


def _launch(tmp_path, backend, world, bad=-1, port=29531):
    out = str(tmp_path / f"res_{backend}_{bad}")
    procs = []
    for r in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER, backend, out, str(bad)],
                                      cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    logs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("sharded stream hung")
        logs.append(o[-1000:] + e[-3000:])
        assert p.returncode == 0, "\n".join(logs)
    return [pickle.load(open(out + f".{r}", "rb")) for r in range(world)]


@pytest.fixture(scope="module")
def reference_results(cuda):
    """Single-process drop-in API on the same 7-frame clip."""
    from paper_1810_10551_b200 import pipeline as P, synthetic, yolo

    W, H = 3840, 2160
    objs = synthetic.bench_clip(W, H, 9, seed=0)[:7]
    frames = [P.Frame(100 + i, W, H, synthetic.render_frame(W, H, o)) for i, o in enumerate(objs)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    res = list(P.run_sequence(frames, settings, yolo.YoloB200Detector()))
    return [(r.frame_id, r.detections, r.active_count, r.total_count) for r in res]


def test_sharded_stream_world2_gloo_equals_run_sequence(tmp_path, reference_results):
    r0, r1 = _launch(tmp_path, "gloo", 2)
    assert r0[0] == "ok" and r1 == ("ok", [])
    got = [t[:4] for t in r0[1]]
    assert got == reference_results  # shards [0,4) and [4,7): frame 4 primed from frame 3
    assert all(t[4].startswith("cuda:") for t in r0[1])
    assert any(t[1] for t in got)


def test_sharded_stream_failure_aborts_every_rank(tmp_path, reference_results):
    r0, r1 = _launch(tmp_path, "gloo", 2, bad=5, port=29533)  # frame 5: rank 1's 2nd frame
    assert r0[0] == "aborted" and r1[0] == "aborted"
    # rank 0 finished its whole shard [0,4) before the failure surfaced
    assert r0[2] == [100, 101, 102, 103][: len(r0[2])] and r0[1] == len(r0[2])


def test_sharded_stream_world1_nccl_fused_gather(tmp_path, reference_results):
    (r0,) = _launch(tmp_path, "nccl", 1, port=29535)
    assert r0[0] == "ok" and [t[:4] for t in r0[1]] == reference_results
