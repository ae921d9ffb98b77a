"""Region decode (K5) in isolation: ONE head tensor fed to both decoders.

The GPU kernel (csrc/tp_detect.cu decode_kernel, fused to_global) and the CPU
restatement (oracle/yolo_ref.region_decode) decode the same fp32 head — the network's
own heads of real tiles and random heads whose scores crowd the threshold — so any
difference is the decoder's alone. Contract: the same kept (cell, anchor) set up to
candidates whose score lies within 1e-6 of the threshold; classes equal; local rects
and scores within a few fp32 ulps (CUDA expf vs numpy's exp are the only non-IEEE-exact
ops; the rest is the same correctly rounded op sequence); order = (-conf, index); and
the projected global rects bit-exact with the reference's to_global (geometry.py:237-256)
applied to the GPU's own local rects.
"""

import numpy as np
import pytest

from oracle import pipeline_ref as R
from oracle import yolo_ref
from paper_1810_10551_b200 import kernels, native, pipeline as P, synthetic, yolo

pytestmark = pytest.mark.gpu

W, H = 3840, 2160


def _heads(n_real, n_rand, seed=0):
    """Real heads (the network on bench-clip tiles) + random heads with crowded scores."""
    net = yolo.YoloNet(n_real)
    objs = synthetic.bench_clip(W, H, 300, seed=0)
    fr = synthetic.render_frames_device(W, H, [objs[i] for i in (120, 250)])
    plan = P.GridPlan.build(W, H, P.PipelineSettings.from_preset("1 att, 3 fin, 20 over"))
    crops = list(plan.final_grid.crops)[4:4 + n_real]
    jobs = kernels.jobs_tensor((i % 2, c.crop_id, int(c.global_rect.x), int(c.global_rect.y),
                                int(c.global_rect.w), 0) for i, c in enumerate(crops))
    kernels.gather(fr, W * H * 3, H, W, jobs, n_real, "nearest", out_act_ptr=net.input_ptr,
                   dtype=net.dtype)
    net.forward(n_real)
    real = net.head_tensor(n_real)[..., :425].cpu().numpy()
    rng = np.random.default_rng(seed)
    rand = rng.normal(0.0, 2.0, (n_rand, 19, 19, 425)).astype(np.float32)
    v = rand.reshape(n_rand, 19, 19, 5, 85)
    v[..., 4] = rng.normal(0.5, 1.5, v.shape[:-1])    # objectness around the thresholds
    v[..., 5:] *= 0.5
    best = rng.integers(0, 80, v.shape[:-1])              # one dominant class per candidate
    np.put_along_axis(v[..., 5:], best[..., None],
                      np.take_along_axis(v[..., 5:], best[..., None], -1)
                      + rng.uniform(2.0, 8.0, best.shape)[..., None], -1)
    return np.concatenate([real, rand]), crops


def _decode_gpu(heads, crops, thr):
    torch = native.require_cuda()
    n = heads.shape[0]
    net = yolo.YoloNet(n)
    h = net.head_tensor(n)
    h.zero_()
    h[..., :425].copy_(torch.from_numpy(heads))
    jobs = kernels.jobs_tensor((0, c.crop_id, int(c.global_rect.x), int(c.global_rect.y),
                                int(c.global_rect.w), 0) for c in (crops * n)[:n])
    out, counts = kernels.alloc_dets(n)
    kernels.decode(net, n, jobs, W, H, thr, out, counts)
    return kernels.dets_to_host(out, counts, n)


@pytest.mark.parametrize("thr", [0.25, 0.3])
def test_decode_same_head_both_decoders(cuda, thr):
    heads, crops = _heads(4, 6)
    recs, counts = _decode_gpu(heads, crops, thr)
    ref = yolo_ref.region_decode(heads, thr)
    n_cmp = n_edge = n_exact = 0
    max_rect, max_conf = 0.0, 0.0
    crops_n = (crops * len(heads))[: len(heads)]
    for t, r_list in enumerate(ref):
        g = recs[t, : counts[t]]
        g_list = [((float(x["lx"]), float(x["ly"]), float(x["lw"]), float(x["lh"])),
                   int(x["cls"]), float(x["conf"])) for x in g]
        # pair every GPU detection with a CPU one: same class, rect and score within a few
        # ulps (hash on rounded values, linear fallback); unpaired ones must sit on the
        # threshold edge
        def key(rr, c):
            return (c,) + tuple(round(v, 2) for v in rr)
        pool = {}
        for k, d in enumerate(r_list):
            pool.setdefault(key(d[0], d[1]), []).append(k)
        used = set()
        for rr, c, s in g_list:
            cand = [k for k in pool.get(key(rr, c), []) if k not in used]
            if not cand:
                cand = [k for k, d in enumerate(r_list) if k not in used and d[1] == c and
                        max(abs(a - b) for a, b in zip(rr, d[0])) <= 1e-3]
            if not cand:
                assert abs(s - thr) < 1e-6, (t, rr, c, s)
                n_edge += 1
                continue
            j = min(cand, key=lambda k: abs(s - r_list[k][2]))
            used.add(j)
            d = r_list[j]
            dr = max(abs(a - b) for a, b in zip(rr, d[0]))
            dc = abs(s - d[2]) / d[2]
            max_rect, max_conf = max(max_rect, dr), max(max_conf, dc)
            n_exact += (dr == 0.0 and dc == 0.0)
            n_cmp += 1
        for k, d in enumerate(r_list):
            if k not in used:
                assert abs(d[2] - thr) < 1e-6, (t, d)
                n_edge += 1
        # output order: scores non-increasing (ties by cell/anchor index)
        confs = [s for _, _, s in g_list]
        assert all(a >= b for a, b in zip(confs, confs[1:]))
        # projection: bit-exact to_global of the GPU's own local rect
        crop = crops_n[t]
        rc = (crop.crop_id, 0, 0, int(crop.global_rect.x), int(crop.global_rect.y),
              int(crop.global_rect.w), crop.global_rect.w / 608)
        for x in g:
            want = R.to_global((float(x["lx"]), float(x["ly"]), float(x["lw"]), float(x["lh"])),
                               rc, W, H)
            assert (int(x["gx"]), int(x["gy"]), int(x["gw"]), int(x["gh"])) == tuple(want)
    print(f"thr {thr}: {n_cmp} detections compared ({n_exact} bit-identical), "
          f"max |d rect| {max_rect:.2e} px, max score rel {max_conf:.2e}, edge {n_edge}")
    assert n_cmp > 500
    assert max_rect <= 1e-3 and max_conf <= 1e-5
