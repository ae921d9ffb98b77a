"""Remote worker: the reference's wire protocol and worker behaviour,
pinned to a transcript of the REFERENCE worker (tests/golden/make_wire_golden.py ->
wire_golden.json: reply bytes of tilepipe's DetectorServer serving tilepipe's
SceneOracle). CPU only: the batched path is exercised with a stub detector; the GPU
detector behind the same server is in test_gpu_remote.py."""

import hashlib
import json
import os
import socket
import struct

import numpy as np
import pytest

from paper_1810_10551_b200 import pipeline as P, synthetic
from paper_1810_10551_b200.detector import Detection, DetectorProfile
from paper_1810_10551_b200.distribution import DetectorServer, wire
from paper_1810_10551_b200.geometry import Rect

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "wire_golden.json")))


def _exchange(endpoint, msgs):
    host, _, port = endpoint.rpartition(":")
    out = []
    with socket.create_connection((host, int(port)), timeout=10) as sock:
        for m in msgs:
            sock.sendall(m)
            head = wire._recv_exact(sock, 4)
            (n,) = struct.unpack(">I", head)
            out.append(head + wire._recv_exact(sock, n))
    return out


def _requests(plan):
    ids = sorted(plan.crops_by_id())
    msgs = []
    for r in GOLD["requests"]:
        if "hex" in r:
            msgs.append(bytes.fromhex(r["hex"]))
            continue
        tiles = np.random.default_rng(r["tiles_seed"]).integers(0, 256, (2, 608, 608, 3), np.uint8)
        m = wire.eval_request(1, [{"crop_id": ids[0], "width": 608, "height": 608},
                                  {"crop_id": ids[3], "width": 608, "height": 608}],
                              tiles.tobytes())
        assert hashlib.sha256(m).hexdigest() == r["sha256"]
        msgs.append(m)
    return msgs


def test_encodings_are_byte_identical_to_reference():
    for e in GOLD["encodings"]:
        assert wire.encode_message(e["header"]).hex() == e["bytes"]
    with pytest.raises(wire.ProtocolError):
        wire.encode_message({"type": "EVAL_REQUEST", "crops": [{"crop_id": 0, "width": 1,
                                                                 "height": 1}]})


def test_worker_transcript_matches_reference_worker():
    sc = GOLD["scene"]
    settings = P.PipelineSettings.from_preset(sc["preset"])
    gt = synthetic.generate_scene(synthetic.SceneSpec(sc["kind"], sc["W"], sc["H"], sc["frames"],
                                                      seed=sc["seed"]))
    oracle = P.oracle_for_scene(sc["W"], sc["H"], settings, gt)
    plan = P.GridPlan.build(sc["W"], sc["H"], settings)
    with DetectorServer(oracle) as server:
        got = _exchange(server.endpoint, _requests(plan))
    assert [g.hex() for g in got] == GOLD["replies"]


class _StubBatched:
    """A batched detector: one detection per tile carrying the tile's mean as conf."""

    def __init__(self):
        self.profile = DetectorProfile(input_side=4, supported_classes=frozenset({"car"}))
        self.calls = []

    def check_tile(self, tile):
        if tile is None or tile.shape != (4, 4, 3):
            raise ValueError(f"bad tile {None if tile is None else tile.shape}")

    def detect_tiles(self, tiles):
        self.calls.append(len(tiles))
        return [[Detection(Rect(1, 2, 3, 4), "car", float(t.mean()) / 255.0)] for t in tiles]

    def detect(self, frame_id, crop_id, tile):  # the worker must not fall back to this
        raise AssertionError("per-crop detect called on a batched detector")


def test_batched_worker_one_call_order_and_errors():
    det = _StubBatched()
    tiles = [np.full((4, 4, 3), v, np.uint8) for v in (10, 200, 50)]
    crops = [{"crop_id": c, "width": 4, "height": 4} for c in (7, 3, 9)]
    with DetectorServer(det) as server:
        ok, bad, health = _exchange(server.endpoint, [
            wire.eval_request(5, crops, b"".join(t.tobytes() for t in tiles)),
            wire.eval_request(6, [crops[0], {"crop_id": 4, "width": 0, "height": 0}, crops[2]],
                              tiles[0].tobytes() + tiles[2].tobytes()),
            wire.encode_message({"type": "HEALTH"})])
    assert det.calls == [3]  # one device call for the whole request; none for the bad one
    head = json.loads(ok[4:])
    assert head["frame_id"] == 5 and [r["crop_id"] for r in head["results"]] == [7, 3, 9]
    assert [r["detections"][0]["confidence"] for r in head["results"]] == \
        [10 / 255.0, 200 / 255.0, 50 / 255.0]
    err = json.loads(bad[4:])
    assert err == {"type": "ERROR", "code": "detector_failure", "message": "crop_id 4: bad tile None"}
    assert json.loads(health[4:]) == {"type": "HEALTH_OK", "input_side": 4, "classes": ["car"]}


def test_unframed_garbage_reports_malformed_and_closes():
    det = _StubBatched()
    with DetectorServer(det) as server:
        host, _, port = server.endpoint.rpartition(":")
        with socket.create_connection((host, int(port)), timeout=10) as sock:
            body = b"{not json"
            sock.sendall(struct.pack(">I", len(body)) + body)
            header, _ = wire.recv_message(sock)
            assert header["type"] == "ERROR" and header["code"] == "malformed"
            assert sock.recv(1) == b""  # the server closed the connection


def test_message_parser_streamed_and_malformed():
    """The I/O-free parser the client and the worker share: a request fed one byte at a
    time round-trips, and each malformed form raises ProtocolError with the reference's
    message (wire.py recv_message)."""
    tiles = np.arange(2 * 3 * 3, dtype=np.uint8).tobytes()
    msg = wire.eval_request(7, [{"crop_id": 1, "width": 3, "height": 2}], tiles)
    stream = iter(msg)
    header, payload = wire.drive(wire.message_steps(),
                                 lambda n: bytes(next(stream) for _ in range(n)))
    assert header == {"type": "EVAL_REQUEST", "frame_id": 7,
                      "crops": [{"crop_id": 1, "width": 3, "height": 2}]}
    assert payload == tiles and next(stream, None) is None

    def parse(raw):
        buf = memoryview(raw)
        pos = [0]

        def read(n):
            chunk = bytes(buf[pos[0]:pos[0] + n])
            pos[0] += n
            return chunk
        return wire.drive(wire.message_steps(), read)

    def framed(body):
        return struct.pack(">I", len(body)) + body

    for raw, text in [(struct.pack(">I", wire.MAX_HEADER_BYTES + 1), "exceeds limit"),
                      (framed(b"\xff\xfe"), "not valid JSON"),
                      (framed(b"[1,2]"), "'type' field"),
                      (framed(b'{"crops":[{"width":1}],"type":"EVAL_REQUEST"}'),
                       "malformed crop list")]:
        with pytest.raises(wire.ProtocolError, match=text):
            parse(raw)
    assert parse(framed(b'{"type":"HEALTH"}')) == ({"type": "HEALTH"}, b"")
