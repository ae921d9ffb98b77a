"""Per-tensor precision study for the YOLO v2 stack (CPU, torch fp32 emulation).

Question: which stored activations need the fp32-parity hi/lo pair, and which can be a
single fp16 value, while the decoded scores stay within the north-star 1e-3 relative of
the fp32 reference? Each conv slot's OUTPUT is rounded as chosen ("fp32" exact, "hilo" =
hi + fp16(x - hi) as the GPU's parity buffers store it, "fp16" = one RNE fp16), the rest
of the forward is fp32, and the decoded detections are compared with the all-fp32 run.

  python tests/tools/precision_study.py [--tiles 8] [--greedy]
  python tests/tools/precision_study.py --lo8        # the HL8 plan (fp16 hi + e4m3 lo on every input)

Prints per-slot sensitivity (only that slot fp16) and the executed-FLOP saving of a plan.
--lo8 emulates the "fp32" plan exactly: every conv input x (but layer 0's) as
hi = fp16(x) times the fp16 weights plus e4m3((x - hi) 2^a) 2^-a times e4m3(w 2^b) 2^-b,
with b from yolo.hl8_scales (a = LO_EXP; also a = 9, 10, 12 for comparison).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pipeline_ref as R  # noqa: E402
from oracle import yolo_ref  # noqa: E402
from paper_1810_10551_b200 import synthetic, yolo  # noqa: E402

# FLOPs of the consumers of each producing slot (GFLOP per tile) — the K that doubles when
# that slot's output is stored as a hi/lo pair
LAY = yolo.LAYERS


def layer_gflop(li):
    _, cin, cout, k, s = LAY[li]
    return 2.0 * s * s * cout * cin * k * k / 1e9


CONSUMERS = {s: [s + 1] for s in range(22)}
CONSUMERS[12] = [13, 20]          # L16 -> L18 (pooled) and L26
CONSUMERS[19] = [(21, 1024)]      # L24 -> L29 channels [256, 1280)
CONSUMERS[20] = [(21, 256)]       # L26 (reorg) -> L29 channels [0, 256)
CONSUMERS[21] = [22]


def consumer_gflop(s):
    g = 0.0
    for c in CONSUMERS[s]:
        if isinstance(c, tuple):
            li, ch = c
            g += layer_gflop(li) * ch / LAY[li][1]
        else:
            g += layer_gflop(c)
    return g


def make_tiles(n):
    W, H = 3840, 2160
    plan = R.Plan(W, H, 1, 3, 20)
    tiles = []
    for kind, fid in (("dense", 0), ("mixed", 3), ("sparse", 1)):
        gt = synthetic.generate_scene(synthetic.SceneSpec(kind, W, H, fid + 1, seed=0))
        px = synthetic.render_frame(W, H, gt[fid])
        crops = list(plan.att[3]) + [plan.fin[3][k] for k in (1, 4, 7, 8, 10, 13, 16)]
        tiles += [R.cut_tile_nearest(px, c) for c in crops]
    return np.stack(tiles[:n])


def forward(tiles, wp, bs, rounds):
    """yolo_ref.forward with a per-slot output rounding."""
    import torch
    import torch.nn.functional as F

    def rnd(t, mode):
        if mode == "fp32":
            return t
        hi = t.to(torch.float16).to(torch.float32)
        if mode == "fp16":
            return hi
        return hi + (t - hi).to(torch.float16).to(torch.float32)

    with torch.no_grad():
        x = yolo_ref.tiles_to_input(tiles, "fp32")

        def conv(li, inp, linear=False):
            _, cin, cout, k, _ = LAY[li]
            w = yolo_ref.unpack_weight(wp[li], li)
            b = torch.as_tensor(np.asarray(bs[li][:cout], dtype=np.float32))
            y = F.conv2d(inp, w, b, padding=k // 2)
            if not linear:
                y = torch.where(y > 0, y, 0.1 * y)
                y = rnd(y, rounds[li])
            return y

        route16 = None
        for li in range(20):
            x = conv(li, x)
            if LAY[li][0] == 16:
                route16 = x
            if LAY[li][0] in yolo_ref.POOL_AFTER:
                x = F.max_pool2d(x, 2)
        x = torch.cat([yolo_ref.reorg(conv(20, route16)), x], dim=1)
        x = conv(21, x)
        head = conv(22, x, linear=True)
    return head.permute(0, 2, 3, 1).contiguous().numpy()


def forward_lo8(tiles, wp, bs, a):
    """The HL8 plan's forward (see module docstring), everything else fp32."""
    import torch
    import torch.nn.functional as F

    def e4m3(t):
        return t.clamp(-448, 448).to(torch.float8_e4m3fn).to(torch.float32)

    with torch.no_grad():
        x = yolo_ref.tiles_to_input(tiles, "fp32")

        def conv(li, inp, linear=False):
            _, cin, cout, k, _ = LAY[li]
            w = yolo_ref.unpack_weight(wp[li], li)
            b = torch.as_tensor(np.asarray(bs[li][:cout], dtype=np.float32))
            if li == 0:
                y = F.conv2d(inp, w, b, padding=k // 2)
            else:
                hi = inp.to(torch.float16).to(torch.float32)
                lo = e4m3((inp - hi) * 2.0 ** a) / 2.0 ** a
                wm = float(w.abs().max())
                be = min(int(np.floor(np.log2(240.0 / wm))), int(np.floor(np.log2(65504.0 / wm))) - a)
                wlo = e4m3(w * 2.0 ** be) / 2.0 ** be
                y = F.conv2d(hi, w, b, padding=k // 2) + F.conv2d(lo, wlo, None, padding=k // 2)
            if not linear:
                y = torch.where(y > 0, y, 0.1 * y)
            return y

        route16 = None
        for li in range(20):
            x = conv(li, x)
            if LAY[li][0] == 16:
                route16 = x
            if LAY[li][0] in yolo_ref.POOL_AFTER:
                x = F.max_pool2d(x, 2)
        x = torch.cat([yolo_ref.reorg(conv(20, route16)), x], dim=1)
        x = conv(21, x)
        head = conv(22, x, linear=True)
    return head.permute(0, 2, 3, 1).contiguous().numpy()


def compare(ref_head, head, thr=0.25):
    """max relative score error over detections present in both, max box err / 608,
    number of threshold flips (detection on one side only)."""
    ra = yolo_ref.region_decode(ref_head, thr)
    ga = yolo_ref.region_decode(head, thr)
    cerr, berr, flips, n = 0.0, 0.0, 0, 0
    for r_list, g_list in zip(ra, ga):
        rmap = {d[3]: d for d in r_list}
        gmap = {d[3]: d for d in g_list}
        for k in set(rmap) | set(gmap):
            if k not in rmap or k not in gmap:
                flips += 1
                continue
            a, b = rmap[k], gmap[k]
            n += 1
            cerr = max(cerr, abs(a[2] - b[2]) / a[2])
            berr = max(berr, max(abs(p - q) for p, q in zip(a[0], b[0])) / 608)
    # logit error on object cells: head channels 4 (+85k) objectness, full-head max abs
    return cerr, berr, flips, n, float(np.abs(head - ref_head).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=8)
    ap.add_argument("--greedy", action="store_true")
    ap.add_argument("--plan", default="", help="comma list of slots stored as single fp16")
    ap.add_argument("--lo8", action="store_true", help="emulate the HL8 (fp32) plan")
    args = ap.parse_args()
    import torch

    torch.set_num_threads(os.cpu_count())
    tiles = make_tiles(args.tiles)
    wp, bs = yolo.make_weights(0, dtype="fp16")
    t0 = time.time()
    ref = forward(tiles, wp, bs, ["fp32"] * 23)
    print(f"fp32 reference: {time.time() - t0:.1f} s for {len(tiles)} tiles", flush=True)
    hilo = forward(tiles, wp, bs, ["hilo"] * 23)
    print("all hilo (parity plan):  score %.2e box %.2e flips %d n %d head %.2e" % compare(ref, hilo))
    if args.lo8:
        for a in (yolo.LO_EXP, 9, 10, 12):
            print(f"HL8 lo exponent {a}:        score %.2e box %.2e flips %d n %d head %.2e"
                  % compare(ref, forward_lo8(tiles, wp, bs, a)), flush=True)
        return
    allf = forward(tiles, wp, bs, ["fp16"] * 23)
    print("all fp16 (fast plan):    score %.2e box %.2e flips %d n %d head %.2e" % compare(ref, allf))
    total = yolo.GFLOP_PER_TILE
    if args.plan:
        single = {int(s) for s in args.plan.split(",")}
        r = ["fp16" if s in single else "hilo" for s in range(23)]
        saved = sum(consumer_gflop(s) for s in single)
        print(f"plan {sorted(single)}: executed {2 * total - 0.64 - saved:.1f} GFLOP/tile;"
              " score %.2e box %.2e flips %d n %d head %.2e" % compare(ref, forward(tiles, wp, bs, r)))
        return
    sens = []
    for s in range(22):
        r = ["hilo"] * 23
        r[s] = "fp16"
        c = compare(ref, forward(tiles, wp, bs, r))
        sens.append((s, c))
        print(f"slot {s:2d} (L{LAY[s][0]:2d}) fp16 only: consumers {consumer_gflop(s):5.2f} GFLOP"
              "  score %.2e box %.2e flips %d n %d head %.2e" % c, flush=True)
    if args.greedy:
        order = sorted(range(22), key=lambda s: sens[s][1][0] / max(consumer_gflop(s), 1e-3))
        single = set()
        for s in order:
            trial = single | {s}
            r = ["fp16" if q in trial else "hilo" for q in range(23)]
            c = compare(ref, forward(tiles, wp, bs, r))
            ok = c[0] < 5e-4 and c[1] < 5e-4
            print(f"  + slot {s:2d}: score %.2e box %.2e flips %d -> {'keep' if ok else 'reject'}"
                  % c[:3], flush=True)
            if ok:
                single = trial
        saved = sum(consumer_gflop(s) for s in single)
        print(f"greedy single-fp16 slots {sorted(single)}: saves {saved:.1f} of "
              f"{2 * total:.1f} executed GFLOP/tile")


if __name__ == "__main__":
    main()
