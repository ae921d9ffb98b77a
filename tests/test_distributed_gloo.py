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


# ---- crop-parallel stage 2 (engine crop_shard): rank-order exchange of padded slices ----

def _crop_worker(rank, world, port, n_jobs, max_slice, per_tile, q):
    import torch
    import torch.distributed as dist

    from paper_1810_10551_b200.engine import _dist_exchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = D.shard_ranges(n_jobs, world)[rank]  # == tp_shard.cu slice_of()
    dets = torch.full((max_slice, per_tile), -1, dtype=torch.int32)
    counts = torch.zeros(max_slice, dtype=torch.int32)
    for i, j in enumerate(range(a, b)):  # job j's "records": j*100 + k
        counts[i] = j % (per_tile + 1)
        dets[i, : counts[i]] = j * 100 + torch.arange(int(counts[i]), dtype=torch.int32)
    all_dets = torch.empty(world * max_slice * per_tile, dtype=torch.int32)
    all_counts = torch.empty(world * max_slice, dtype=torch.int32)
    _dist_exchange(dets.view(-1), counts, all_dets, all_counts)
    if rank == 0:
        q.put((all_dets.tolist(), all_counts.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def _unslice(all_dets, all_counts, n_jobs, world, max_slice, per_tile):
    """Restatement of tp_shard.cu unslice_kernel's job -> (rank, index) map."""
    base, extra = divmod(n_jobs, world)
    out = []
    for j in range(n_jobs):
        if j < extra * (base + 1):
            r, i = divmod(j, base + 1)
        else:
            jj = j - extra * (base + 1)
            r = extra + jj // base
            i = jj - (r - extra) * base
        s = r * max_slice + i
        c = all_counts[s]
        out.append(all_dets[s * per_tile: s * per_tile + c])
    return out


@pytest.mark.parametrize("n_jobs", [11, 1])
def test_crop_exchange_rank_order_and_unslice(n_jobs):
    world, per_tile = 2, 3
    max_slice = -(-16 // world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + n_jobs + os.getpid() % 500
    procs = [ctx.Process(target=_crop_worker,
                         args=(r, world, port, n_jobs, max_slice, per_tile, q))
             for r in range(world)]
    for p in procs:
        p.start()
    all_dets, all_counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = _unslice(all_dets, all_counts, n_jobs, world, max_slice, per_tile)
    assert got == [[j * 100 + k for k in range(j % (per_tile + 1))] for j in range(n_jobs)]
