"""Multi-process (world_size 2, gloo, CPU) checks of the frame-sharding host logic:
contiguous dispatch, boundary history frames, and the padded result gather restoring
global frame order — the same code the NCCL path runs on GPUs."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1810_10551_b200 import distributed as D
from paper_1810_10551_b200 import native


def test_shard_ranges_match_dispatch_rule():
    assert D.shard_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert D.shard_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for n in range(0, 40):
        for w in range(1, 9):
            rs = D.shard_ranges(n, w)
            sizes = [b - a for a, b in rs]
            assert sum(sizes) == n and max(sizes) - min(sizes) <= 1
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))


def test_history_frames():
    assert D.history_frames(0, 2) == []
    assert D.history_frames(10, 2) == [9]
    assert D.history_frames(10, 3) == [8, 9]
    assert D.history_frames(1, 3) == [0]


def _frame_records(f):
    rng = np.random.default_rng(f)
    n = int(rng.integers(0, 5))
    rec = np.zeros(n, dtype=native.PDET_DTYPE)
    rec["x"] = rng.integers(0, 3000, n)
    rec["conf"] = rng.random(n)
    rec["src"] = f
    return rec


def _worker(rank, world, port, n_frames, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges = D.shard_ranges(n_frames, world)
    a, b = ranges[rank]
    rows = [_frame_records(f) for f in range(a, b)]
    counts, buf = D.pack_records(rows, 8, native.PDET_DTYPE)
    out = D.gather_records(torch.from_numpy(counts), torch.from_numpy(buf.view(np.uint8)),
                           [r[1] - r[0] for r in ranges])
    if rank == 0:
        q.put([(c, bytes(r)) for c, r in out])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [7, 2])
def test_gather_restores_global_frame_order(n_frames):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + n_frames + os.getpid() % 500
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got) == n_frames
    for f, (c, raw) in enumerate(got):
        exp = _frame_records(f)
        assert c == len(exp)
        rec = np.frombuffer(raw, dtype=native.PDET_DTYPE)[:c]
        assert (rec == exp).all()
