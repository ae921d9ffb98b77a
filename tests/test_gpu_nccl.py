"""Result gather through the C-ABI (tp_nccl_gather_dets) on torch.distributed's own NCCL
communicator. One GPU is lent, so the process group has world size 1 (the collective
still runs through NCCL: ncclGroupStart, two ncclAllGather, ncclGroupEnd); the
rank-order semantics for world > 1 are covered with gloo in test_distributed_gloo.py.
Runs in a subprocess so the process group does not leak into other tests."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import numpy as np, torch, torch.distributed as dist
    from paper_1810_10551_b200 import native, synthetic, pipeline as P
    from paper_1810_10551_b200 import distributed as D
    from paper_1810_10551_b200.engine import AttentionPipelineB200
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    assert native.load().tp_nccl_available() == 1
    assert D.nccl_comm() != 0
    g = torch.Generator(device="cuda").manual_seed(5)
    recs = torch.randint(0, 256, (7, 1000), dtype=torch.uint8, device="cuda", generator=g)
    counts = torch.arange(7, dtype=torch.int32, device="cuda") * 3
    all_recs = torch.zeros_like(recs)
    all_counts = torch.full_like(counts, -1)
    D.nccl_all_gather(recs, all_recs, counts, all_counts)
    torch.cuda.synchronize()
    assert torch.equal(all_recs, recs) and torch.equal(all_counts, counts)
    out = D.gather_records(counts, recs, [7])
    assert [c for c, _ in out] == counts.tolist()
    assert all(np.array_equal(r, recs[i].cpu().numpy()) for i, (_, r) in enumerate(out))
    # crop-parallel engine with the default (NCCL, C-ABI) exchange equals the plain engine
    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 2, seed=4))
    clip = [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(2)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    single = AttentionPipelineB200(settings, W, H, max_frames=2)
    want = [(r.frame_id, r.active_count, r.detections) for r, _ in single.evaluate_frames(clip, history=())]
    shard = AttentionPipelineB200(settings, W, H, max_frames=2, net=single.net, crop_shard=(0, 1))
    got = [(r.frame_id, r.active_count, r.detections) for r, _ in shard.evaluate_frames(clip, history=())]
    assert got == want
    dist.destroy_process_group()
    print("NCCL-OK")
""")


def test_nccl_result_gather_through_c_abi(cuda):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29517", PYTHONPATH=ROOT)
    p = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0 and "NCCL-OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
