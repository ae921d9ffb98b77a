"""The B200 detector behind the reference wire protocol: one EVAL_REQUEST
carrying several 608x608 tiles is answered from ONE batched device call, with exactly
the detections a direct detect_tiles / per-crop detect gives; concurrent clients get
the same answers (the detector serialises its shared workspace)."""

import json
import socket
import struct
import threading

import numpy as np
import pytest

from paper_1810_10551_b200 import pipeline as P, synthetic
from paper_1810_10551_b200.detector import cut_tile
from paper_1810_10551_b200.distribution import DetectorServer, wire
from paper_1810_10551_b200.yolo import YoloB200Detector

pytestmark = pytest.mark.gpu


def _ask(endpoint, msg):
    host, _, port = endpoint.rpartition(":")
    with socket.create_connection((host, int(port)), timeout=60) as sock:
        sock.sendall(msg)
        head = wire._recv_exact(sock, 4)
        (n,) = struct.unpack(">I", head)
        return json.loads(wire._recv_exact(sock, n))


def _rows(dets):
    return [{"x": d.rect.x, "y": d.rect.y, "w": d.rect.w, "h": d.rect.h,
             "class": d.class_label, "confidence": d.confidence} for d in dets]


def test_yolo_worker_batched_equals_direct(cuda):
    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 1, seed=2))
    px = synthetic.render_frame(W, H, gt[0])
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    plan = P.GridPlan.build(W, H, settings)
    crops = [c for _, c in sorted(plan.crops_by_id().items())][:6]
    tiles = [cut_tile(px, c) for c in crops]
    det = YoloB200Detector()
    want = det.detect_tiles(np.stack(tiles))
    assert sum(len(w) for w in want) > 0
    assert _rows(det.detect(0, crops[1].crop_id, tiles[1])) == _rows(want[1])
    msg = wire.eval_request(
        0, [{"crop_id": c.crop_id, "width": 608, "height": 608} for c in crops],
        b"".join(t.tobytes() for t in tiles))
    with DetectorServer(det) as server:
        reply = _ask(server.endpoint, msg)
        assert reply["type"] == "EVAL_RESPONSE"
        assert [r["crop_id"] for r in reply["results"]] == [c.crop_id for c in crops]
        for r, w in zip(reply["results"], want):
            assert r["detections"] == _rows(w)
        # concurrent clients: identical answers
        outs = [None] * 4

        def run(k):
            outs[k] = _ask(server.endpoint, msg)

        ths = [threading.Thread(target=run, args=(k,)) for k in range(4)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert all(o == reply for o in outs)
        # a wrong-size tile is rejected before any device work, with detect's message
        bad = _ask(server.endpoint, wire.eval_request(
            0, [{"crop_id": 1, "width": 608, "height": 608}, {"crop_id": 2, "width": 10,
                                                               "height": 10}],
            tiles[0].tobytes() + bytes(300)))
        assert bad["code"] == "detector_failure" and bad["message"].startswith("crop_id 2: tile must")
