"""frameio: PPM frames, FrameSource, result/timing files (reference frameio.py semantics;
behaviours follow pkg/tests/test_frameio.py) + the zero-copy read_ppm_into."""

import csv

import numpy as np
import pytest

from paper_1810_10551_b200.detector import Detection
from paper_1810_10551_b200.frameio import (TIMING_CSV_COLUMNS, FrameDecodeError,
                                           FrameDimensionError, FrameSource, frame_file_name,
                                           read_ppm, read_ppm_into, read_results, write_ppm,
                                           write_results, write_timing_csv)
from paper_1810_10551_b200.geometry import Rect
from paper_1810_10551_b200.pipeline_types import FrameResult, TimingProfile


def _seq(d, ids, w=16, h=8):
    d.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(3)
    out = {}
    for i in ids:
        px = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        write_ppm(d / frame_file_name(i), px)
        out[i] = px
    return out


def test_ppm_round_trip_and_header(tmp_path):
    px = np.random.default_rng(1).integers(0, 256, (5, 7, 3), dtype=np.uint8)
    write_ppm(tmp_path / "a.ppm", px)
    raw = (tmp_path / "a.ppm").read_bytes()
    assert raw.startswith(b"P6\n7 5\n255\n") and len(raw) == len(b"P6\n7 5\n255\n") + 105
    assert np.array_equal(read_ppm(tmp_path / "a.ppm"), px)


def test_ppm_comments_and_errors(tmp_path):
    p = tmp_path / "c.ppm"
    p.write_bytes(b"P6\n# a comment\n2 2\n255\n" + bytes(12))
    assert read_ppm(p).shape == (2, 2, 3)
    cases = {b"P5\n2 2\n255\n" + bytes(4): "magic", b"P6\n2 2\n65535\n" + bytes(24): "maxval",
             b"P6\n4 4\n255\n" + bytes(10): "truncated", b"garbage": "header",
             b"P6\nx 2\n255\n": "non-numeric", b"P6\n# open comment": "comment"}
    for data, _why in cases.items():
        p.write_bytes(data)
        with pytest.raises(FrameDecodeError):
            read_ppm(p)
        with pytest.raises(FrameDecodeError):
            read_ppm_into(p, np.empty(4096, np.uint8))
    with pytest.raises(ValueError):
        write_ppm(tmp_path / "x.ppm", np.zeros((2, 2), np.uint8))


def test_read_does_not_alias_the_file(tmp_path):
    p = tmp_path / "a.ppm"
    write_ppm(p, np.full((2, 2, 3), 7, np.uint8))
    a = read_ppm(p)
    a[...] = 0
    assert read_ppm(p).max() == 7


def test_read_ppm_into_matches_read_ppm(tmp_path):
    px = _seq(tmp_path, [4], w=33, h=9)[4]
    buf = np.full(33 * 9 * 3 + 5, 255, np.uint8)
    assert read_ppm_into(tmp_path / frame_file_name(4), buf) == (33, 9)
    assert np.array_equal(buf[: 33 * 9 * 3].reshape(9, 33, 3), px)
    assert (buf[-5:] == 255).all()  # nothing written past the raster
    with pytest.raises(ValueError):
        read_ppm_into(tmp_path / frame_file_name(4), np.empty(10, np.uint8))


def test_frame_source(tmp_path):
    d = tmp_path / "frames"
    px = _seq(d, [10, 0, 2])
    (d / "notes.txt").write_text("ignored")
    src = FrameSource.open(d)
    assert src.frame_ids == (0, 2, 10) and (src.width, src.height) == (16, 8) and len(src) == 3
    frames = list(src.frames())
    assert [f.frame_id for f in frames] == [0, 2, 10]
    assert all(np.array_equal(f.pixels, px[f.frame_id]) for f in frames)
    out = np.empty((8, 16, 3), np.uint8)
    src.load_into(2, out)
    assert np.array_equal(out, px[10])
    with pytest.raises(IndexError):
        src.frame(3)
    write_ppm(d / frame_file_name(2), np.zeros((9, 16, 3), np.uint8))
    with pytest.raises(FrameDimensionError):
        src.frame(1)
    with pytest.raises(FrameDimensionError):
        src.load_into(1, np.empty((9, 16, 3), np.uint8))
    (d / frame_file_name(10)).unlink()
    with pytest.raises(FileNotFoundError):
        src.frame(2)
    (d / frame_file_name(0)).write_bytes(b"junk")
    with pytest.raises(FrameDecodeError):
        src.frame(0)
    (tmp_path / "empty").mkdir()
    with pytest.raises(FileNotFoundError):
        FrameSource.open(tmp_path / "empty")
    with pytest.raises(FileNotFoundError):
        FrameSource.open(tmp_path / "missing")


def test_results_and_timing_files(tmp_path):
    res = [FrameResult(3, (Detection(Rect(10, 20, 30, 40), "car", 0.9876543),
                           Detection(Rect(1, 2, 3, 4), "person", 0.5)), 4, 18,
                       TimingProfile(io_ms=1.0, final_eval_ms=2.5, per_worker=(("cuda:0", 3.5),))),
           FrameResult(4, (), 0, 18, TimingProfile())]
    write_results(res, tmp_path / "r.jsonl")
    lines = (tmp_path / "r.jsonl").read_text().splitlines()
    assert lines[0] == ('{"active_count":4,"detections":[{"class":"car","confidence":0.987654,'
                        '"h":40,"w":30,"x":10,"y":20},{"class":"person","confidence":0.500000,'
                        '"h":4,"w":3,"x":1,"y":2}],"frame_id":3,"total_count":18}')
    back = read_results(tmp_path / "r.jsonl")
    assert [r.frame_id for r in back] == [3, 4] and back[0].detections[0].class_label == "car"
    write_results(back, tmp_path / "r2.jsonl")
    assert (tmp_path / "r2.jsonl").read_bytes() == (tmp_path / "r.jsonl").read_bytes()
    write_timing_csv(res, tmp_path / "t.csv")
    rows = list(csv.reader(open(tmp_path / "t.csv")))
    assert tuple(rows[0]) == TIMING_CSV_COLUMNS and len(rows) == 3
    assert rows[1][-1] == "cuda:0=3.500" and rows[1][TIMING_CSV_COLUMNS.index("total_ms")] == "3.500"
    (tmp_path / "bad.jsonl").write_text('{"frame_id": 1}\n')
    with pytest.raises(ValueError):
        read_results(tmp_path / "bad.jsonl")


def test_ground_truth_round_trip_and_run_config(tmp_path):
    from paper_1810_10551_b200.detector import GroundTruthObject
    from paper_1810_10551_b200.frameio import read_ground_truth, read_run_config, write_ground_truth

    gt = {2: [GroundTruthObject(Rect(10, 20, 30.5, 40), "car", "c1")],
          0: [GroundTruthObject(Rect(1, 2, 3, 4), "person", "p1")]}
    write_ground_truth(gt, tmp_path / "gt.jsonl")
    first = (tmp_path / "gt.jsonl").read_text().splitlines()[0]
    assert first == '{"class":"person","frame_id":0,"h":4,"object_id":"p1","w":3,"x":1,"y":2}'
    back = read_ground_truth(tmp_path / "gt.jsonl")
    assert sorted(back) == [0, 2] and back[2][0].rect.w == 30.5
    (tmp_path / "frames").mkdir()
    write_ppm(tmp_path / "frames" / frame_file_name(0), np.zeros((8, 16, 3), np.uint8))
    cfg = tmp_path / "run.ini"
    cfg.write_text("[pipeline]\npreset = 1 att, 3 fin, 20 over\n[detector]\nkind = yolo-b200\n"
                   "batch = 4\n[paths]\nframes = frames\nresults = out.jsonl\n")
    rc = read_run_config(cfg)
    assert rc.detector == "yolo-b200" and rc.batch == 4 and rc.ground_truth_path is None
    assert rc.frames_dir == (tmp_path / "frames").resolve()
    cfg.write_text("[pipeline]\npreset = 1 att, 3 fin, 20 over\n[detector]\nkind = oracle\n"
                   "[paths]\nresults = out.jsonl\n[frame]\nwidth = 64\nheight = 32\n")
    with pytest.raises(ValueError):  # oracle needs ground truth
        read_run_config(cfg)
    cfg.write_text("[pipeline]\npreset = 1 att, 3 fin, 20 over\n[detector]\nkind = remote\n"
                   "[paths]\nground_truth = gt.jsonl\nresults = out.jsonl\n[frame]\nwidth = 64\n"
                   "height = 32\n")
    with pytest.raises(ValueError, match="remote"):
        read_run_config(cfg)
    cfg.write_text("[pipeline]\nattention_rows = 1\nfinal_rows = 3\noverlap_px = 20\n"
                   "[detector]\nkind = oracle\nvisibility_threshold = 0.5\n[paths]\n"
                   "ground_truth = gt.jsonl\nresults = out.jsonl\n[frame]\nwidth = 64\nheight = 32\n")
    rc = read_run_config(cfg)
    assert rc.settings.preset_name() == "1 att, 3 fin, 20 over" and rc.visibility_threshold == 0.5
