"""Frame-parallel sharding across GPUs (one process per GPU, torch.distributed).

The path partitions by frame: attention for frame t depends only on
frame t, selection on frames t-K+1..t, and the final pass never feeds back. A clip is
split into contiguous chunks whose sizes differ by at most one (the reference's
``dispatch`` rule, distribution/client.py:82-96). A rank seeds its temporal window by
re-running stage 1 on the K-1 frames just before its chunk (2 tiles per frame at
preset P1) instead of exchanging attention boxes, so the data path has no collective;
the only collective is the result gather to rank 0 (``gather_records``), a fixed-size
padded all-gather: on GPUs one fused NCCL launch through the C-ABI
(``tp_nccl_gather_dets`` on torch.distributed's own communicator), gloo on CPU.
"""

from __future__ import annotations

import numpy as np


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


def nccl_all_gather(local_recs, all_recs, local_counts, all_counts, group=None, stream=None):
    """Rank-order all-gather of a padded record slice and its counts in one fused NCCL
    launch on `stream` (tp_nccl_gather_dets). Shapes: all_* = world x local_*.

    If this torch build exposes no communicator pointer, the same two all-gathers go
    through torch.distributed's own NCCL calls (still on the GPU; one warning)."""
    import torch.distributed as dist

    from . import native

    try:
        comm = nccl_comm(group)
    except (RuntimeError, AttributeError) as exc:
        global _warned
        if not _warned:
            import warnings

            warnings.warn(f"tp_nccl_gather_dets unavailable ({exc}); using torch NCCL all-gathers")
            _warned = True
        if local_recs is not None:
            dist.all_gather_into_tensor(all_recs.view(-1), local_recs.reshape(-1), group=group)
        if local_counts is not None:
            dist.all_gather_into_tensor(all_counts.view(-1), local_counts.reshape(-1), group=group)
        return
    native.call("tp_nccl_gather_dets", comm, native.ptr(local_recs),
                int(local_recs.numel() * local_recs.element_size()) if local_recs is not None else 0,
                native.ptr(local_counts), int(local_counts.numel()) if local_counts is not None else 0,
                native.ptr(all_recs), native.ptr(all_counts), native.stream_handle(stream))


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
    if dist.get_backend(group) == "nccl":
        nccl_all_gather(r, rall, c, call, group)
    else:  # gloo gathers host tensors
        ch, rh = call.cpu(), rall.cpu()
        dist.all_gather_into_tensor(ch, c.cpu(), group=group)
        dist.all_gather_into_tensor(rh, r.cpu(), group=group)
        call.copy_(ch)
        rall.copy_(rh)
    if not to_host:  # stay on device (no host sync): [world*n_max] counts, records
        return call, rall
    call = call.cpu().numpy().reshape(world, n_max)
    rall = rall.cpu().numpy().reshape(world, n_max, -1)
    out = []
    for rank in range(world):
        for f in range(frames_per_rank[rank]):
            out.append((int(call[rank, f]), rall[rank, f]))
    return out
