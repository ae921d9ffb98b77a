"""Build the committed YOLO head for a seed: a deterministic linear probe on the random
backbone's layer-29 features (dev tool; its output is data, not code on the hot path).

    python tests/tools/calibrate_head.py [--seed 0]

Why: a random-init YOLO v2 never reaches the pipeline's 0.3 score threshold (SURVEY
§0.4), so stage 1 would select nothing. The probe keeps the backbone random (seeded,
shared with the oracle) and fits only the 1x1 head on synthetic scenes:
  * objectness (anchor 2 only; the other anchors are disabled): ridge-LDA direction
    between cells containing an object centre and cells touching no object;
  * class: ridge-LDA person-vs-car on the positive cells (other classes biased off);
  * tx, ty, tw, th: ridge regression to the YOLO v2 targets of the positive cells.
Features come from the CPU oracle network in fp32 (oracle/yolo_ref.py).
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pipeline_ref, yolo_ref  # noqa: E402
from paper_1810_10551_b200 import synthetic, yolo  # noqa: E402

ANCHOR = 2
REG_OBJ = 1.0   # strong ridge: a smoother probe amplifies 16-bit activation rounding less
REG_CLS = 2.0
SCENES = [("dense", 3840, 2160, 1), ("sparse", 3840, 2160, 2), ("mixed", 3840, 2160, 3),
          ("dense", 7680, 4320, 4), ("straddle", 3840, 2160, 5)]


def tiles_and_labels():
    tiles, infos = [], []
    for kind, W, H, seed in SCENES:
        gt = synthetic.generate_scene(synthetic.SceneSpec(kind, W, H, 1, seed=seed))[0]
        px = synthetic.render_frame(W, H, gt)
        plan = pipeline_ref.Plan(W, H, 1, 3, 20)
        crops = plan.att[3] + plan.fin[3][::3]
        for c in crops:
            tiles.append(pipeline_ref.cut_tile_nearest(px, c))
            s = c[6]
            objs = [((o.rect.x - c[3]) / s, (o.rect.y - c[4]) / s, o.rect.w / s, o.rect.h / s,
                     o.class_label) for o in gt]
            infos.append(objs)
    return np.stack(tiles), infos


def cell_targets(objs):
    """Per cell: label (1 pos, 0 neg, -1 ignore), class, box targets."""
    lab = np.zeros((19, 19), np.int8)
    cls = np.zeros((19, 19), np.int8)
    tgt = np.zeros((19, 19, 4), np.float32)
    for x, y, w, h, c in objs:
        x1, y1, x2, y2 = max(0, x), max(0, y), min(608, x + w), min(608, y + h)
        if x2 <= x1 or y2 <= y1:
            continue
        r0, r1 = int(max(0, y1 // 32)), int(min(18, (y2 - 1) // 32))
        c0, c1 = int(max(0, x1 // 32)), int(min(18, (x2 - 1) // 32))
        lab[r0:r1 + 1, c0:c1 + 1] = np.where(lab[r0:r1 + 1, c0:c1 + 1] == 1, 1, -1)
        cx, cy = (x1 + x2) / 2, (y1 + y2) / 2
        ri, ci = int(cy // 32), int(cx // 32)
        if 0 <= ri < 19 and 0 <= ci < 19:
            lab[ri, ci] = 1
            cls[ri, ci] = 0 if c == "person" else 1
            fx = np.clip(cx / 32 - ci, 0.05, 0.95)
            fy = np.clip(cy / 32 - ri, 0.05, 0.95)
            aw, ah = yolo.ANCHORS[2 * ANCHOR], yolo.ANCHORS[2 * ANCHOR + 1]
            tgt[ri, ci] = (np.log(fx / (1 - fx)), np.log(fy / (1 - fy)),
                           np.log((x2 - x1) / 32 / aw), np.log((y2 - y1) / 32 / ah))
    return lab, cls, tgt


def ridge_lda(a, b, reg):
    mu_a, mu_b = a.mean(0), b.mean(0)
    cov = np.cov(b, rowvar=False) if len(b) > 1 else np.eye(a.shape[1])
    lam = reg * np.trace(cov) / cov.shape[0]
    return np.linalg.solve(cov + lam * np.eye(cov.shape[0]), mu_a - mu_b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    t0 = time.time()
    wpacks, biases = yolo.make_weights(args.seed, head="random")
    tiles, infos = tiles_and_labels()
    feats = []
    for i in range(0, len(tiles), 4):
        _, f = yolo_ref.forward(tiles[i:i + 4], wpacks, biases, mode=yolo.DEFAULT_PRECISION,
                                threads=os.cpu_count(), return_features=True)
        feats.append(f["l29"])
    feats = np.concatenate(feats).astype(np.float64)  # n,19,19,1024
    print(f"features for {len(tiles)} tiles in {time.time() - t0:.1f}s")
    labs, clss, tgts = zip(*(cell_targets(o) for o in infos))
    lab = np.stack(labs).reshape(-1)
    cls = np.stack(clss).reshape(-1)
    tgt = np.stack(tgts).reshape(-1, 4)
    F = feats.reshape(-1, 1024)
    pos, neg = F[lab == 1], F[lab == 0]
    print("positive cells", len(pos), "negative cells", len(neg))

    w_obj = ridge_lda(pos, neg, REG_OBJ)
    p_pos, p_neg = pos @ w_obj, neg @ w_obj
    m_pos, m_neg = np.median(p_pos), np.median(p_neg)
    a = 10.0 / (m_pos - m_neg)
    obj_w, obj_b = a * w_obj, -a * m_neg - 6.0
    lp, ln = pos @ obj_w + obj_b, neg @ obj_w + obj_b
    print(f"objectness: pos>0 {np.mean(lp > 0):.3f}  neg>0 {np.mean(ln > 0):.4f}")

    pcls = cls[lab == 1]
    per, car = pos[pcls == 0], pos[pcls == 1]
    w_c = ridge_lda(per, car, REG_CLS) if len(per) and len(car) else np.zeros(1024)
    q_p, q_c = per @ w_c, car @ w_c
    mid, half = (np.mean(q_p) + np.mean(q_c)) / 2, (np.mean(q_p) - np.mean(q_c)) / 2
    cw, cb = 2.0 * w_c / half, -2.0 * mid / half
    s = pos @ cw + cb
    print(f"class: person acc {np.mean(s[pcls == 0] > 0):.3f} car acc {np.mean(s[pcls == 1] < 0):.3f}")

    X = np.concatenate([pos, np.ones((len(pos), 1))], 1)
    lam = 0.5 * np.trace(X.T @ X) / X.shape[1]
    reg = np.linalg.solve(X.T @ X + lam * np.eye(X.shape[1]), X.T @ tgt[lab == 1])
    res = X @ reg - tgt[lab == 1]
    print("box regression rmse", np.sqrt((res ** 2).mean(0)))

    W = np.zeros((425, 1024), np.float64)
    B = np.zeros(425, np.float64)
    for an in range(5):
        base = an * 85
        if an != ANCHOR:
            B[base + 4] = -30.0
            continue
        W[base:base + 4] = reg[:1024].T
        B[base:base + 4] = reg[1024]
        W[base + 4], B[base + 4] = obj_w, obj_b
        B[base + 5:base + 85] = -6.0
        W[base + 5 + 0], B[base + 5 + 0] = cw, 2.0 + cb       # person
        W[base + 5 + 2], B[base + 5 + 2] = -cw, 2.0 - cb      # car
    os.makedirs(yolo.DATA_DIR, exist_ok=True)
    out = yolo.head_path(args.seed)
    np.savez_compressed(out, w=W.astype(np.float32), b=B.astype(np.float32))
    print("wrote", out, f"({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main()
