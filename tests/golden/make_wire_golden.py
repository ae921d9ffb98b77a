"""Golden transcript of the reference worker: run HERE, where the
reference package is importable; the fixture is committed and the tests never read
/root/reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_wire_golden.py

Records (a) wire encodings of a few headers and (b) the raw reply bytes of the
reference DetectorServer serving the reference SceneOracle for a seeded 4K scene, to a
fixed list of request messages on one connection (HEALTH, raster-free EVAL_REQUESTs for
every crop, an EVAL_REQUEST with 608x608 tiles, an unknown crop id, an unknown type).
"""

import json
import os
import socket
import struct

import numpy as np
from tilepipe import pipeline as P, synthetic
from tilepipe.distribution import wire
from tilepipe.distribution.worker import DetectorServer

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "wire_golden.json")
W, H = 3840, 2160


def requests():
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    plan = P.GridPlan.build(W, H, settings)
    ids = sorted(plan.crops_by_id())
    msgs = [wire.encode_message({"type": "HEALTH"}), wire.eval_request(0, [])]
    for f in (0, 1, 2):
        msgs.append(wire.eval_request(f, [{"crop_id": c, "width": 0, "height": 0} for c in ids]))
    rng = np.random.default_rng(3)
    tiles = rng.integers(0, 256, (2, 608, 608, 3), np.uint8)
    msgs.append(wire.eval_request(1, [{"crop_id": ids[0], "width": 608, "height": 608},
                                      {"crop_id": ids[3], "width": 608, "height": 608}],
                                  tiles.tobytes()))
    msgs.append(wire.eval_request(0, [{"crop_id": 999, "width": 0, "height": 0}]))
    msgs.append(wire.encode_message({"type": "BOGUS"}))
    return settings, msgs


def main():
    settings, msgs = requests()
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 3, seed=0))
    oracle = P.oracle_for_scene(W, H, settings, gt)
    with DetectorServer(oracle) as server:
        host, _, port = server.endpoint.rpartition(":")
        replies = []
        with socket.create_connection((host, int(port)), timeout=10) as sock:
            for m in msgs:
                sock.sendall(m)
                head = wire._recv_exact(sock, 4)
                (n,) = struct.unpack(">I", head)
                replies.append((head + wire._recv_exact(sock, n)).hex())
    enc = []
    for h in ({"type": "HEALTH"}, {"type": "ERROR", "code": "x", "message": "é"},
              {"type": "EVAL_RESPONSE", "frame_id": 3, "results": [
                  {"crop_id": 2, "detections": [{"x": 1.5, "y": 2, "w": 3, "h": 4,
                                                 "class": "car", "confidence": 0.25}]}]}):
        enc.append({"header": h, "bytes": wire.encode_message(h).hex()})
    import hashlib

    # the tile-carrying request is rebuilt by the test from its seed (2.2 MB of pixels);
    # its sha256 pins the rebuild
    reqs = [{"hex": m.hex()} if len(m) < 65536 else
            {"tiles_seed": 3, "sha256": hashlib.sha256(m).hexdigest()} for m in msgs]
    json.dump({"scene": {"kind": "dense", "W": W, "H": H, "frames": 3, "seed": 0,
                         "preset": "1 att, 3 fin, 20 over"},
               "requests": reqs, "replies": replies, "encodings": enc}, open(OUT, "w"))
    print(f"wrote {OUT}: {len(msgs)} requests, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
