"""Crop-parallel stage 2 (reference dispatch rule
pkg/src/tilepipe/distribution/client.py:82-96): R ranks each evaluate a contiguous slice of
the same device job list; after the rank-order all-gather and tp_unslice_dets every rank's
FrameResults equal the single-GPU engine's. One GPU: the R ranks are R engines run in
turn in one process and the all-gather is a rank-order concatenation (no rank waits on
another rank's kernel)."""

import numpy as np
import pytest

from paper_1810_10551_b200 import pipeline as P, synthetic
from paper_1810_10551_b200.engine import AttentionPipelineB200

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def clip():
    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 4, seed=3))
    return [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(4)]


def _key(out):
    return [(r.frame_id, r.active_count, r.detections) for r, _ in out]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_crop_sharded_stage2_equals_single_gpu(cuda, clip, world):
    torch = cuda
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    single = AttentionPipelineB200(settings, 3840, 2160, max_frames=2)
    want = _key(single.evaluate_frames(clip[:2], history=()))
    want += _key(single.evaluate_frames(clip[2:], history=None))
    ranks = [AttentionPipelineB200(settings, 3840, 2160, max_frames=2, net=single.net,
                                   crop_shard=(r, world)) for r in range(world)]
    frames = torch.from_numpy(np.stack([f.pixels for f in clip])).cuda()
    got = []
    for b in (0, 2):
        for e in ranks:
            if b == 0:
                e.reset_history(())
            e.run_local(2, frames=frames[b:b + 2])
        torch.cuda.synchronize()
        dets = torch.cat([e.local_results()[0] for e in ranks])
        counts = torch.cat([e.local_results()[1] for e in ranks])
        assert int(sum(int(e.n_local.item()) for e in ranks)) == int(ranks[0].n_jobs2.item())
        per_rank = []
        for e in ranks:
            e.all_dets.copy_(dets)
            e.all_counts.copy_(counts)
            e.finish_local()
            per_rank.append(_key(e.results([b, b + 1])))
        assert all(k == per_rank[0] for k in per_rank)
        got += per_rank[0]
    assert got == want
    assert any(d for _, _, d in want)


def test_crop_shard_default_path_with_injected_exchange(cuda, clip):
    """world 1 through evaluate_frames with an injected (identity) exchange: the
    non-split branch of _finish."""
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    single = AttentionPipelineB200(settings, 3840, 2160, max_frames=2)
    want = _key(single.evaluate_frames(clip[:2], history=()))
    calls = []

    def exchange(ld, lc, ad, ac):
        calls.append(1)
        ad.copy_(ld)
        ac.copy_(lc)

    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=2, net=single.net,
                                crop_shard=(0, 1), exchange=exchange)
    assert _key(eng.evaluate_frames(clip[:2], history=())) == want and calls


def test_crop_shard_rejects_bad_rank(cuda):
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    with pytest.raises(ValueError):
        AttentionPipelineB200(settings, 3840, 2160, max_frames=1, crop_shard=(2, 2))
