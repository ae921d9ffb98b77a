"""Batched YOLO engine vs the CPU oracle on the same synthetic frames and weights.

North-star parity contract:
  * crop-index selection is bit-exact given identical stage-1 boxes (the GPU's stage-1
    boxes are fed to the oracle's merge_temporal/select_active);
  * the NMS/merge keep-set is bit-exact given identical raw detections (the GPU's raw
    stage-2 tagged lists are fed to the oracle's postprocess);
  * decoded boxes and scores match the oracle network (bf16 activation storage, fp32
    accumulation) within BOX_REL / CONF_ABS below; detections within CONF_ABS of the
    threshold may legitimately appear on one side only.
"""

import numpy as np
import pytest

from oracle import pipeline_ref as R
from oracle import yolo_ref
from paper_1810_10551_b200 import kernels, native, pipeline as P, synthetic, yolo
from paper_1810_10551_b200.engine import MAX_PER_FRAME, AttentionPipelineB200

pytestmark = pytest.mark.gpu

# 16-bit activation storage (default fp16 operands, fp32 accumulation): rounding flips
# caused by a different fp32 accumulation order propagate through 23 layers.
BOX_REL = 1e-3     # |d coord| / 608 (608-space local rects)
# Measured on B200 with fp16 operands: boxes 1.8e-4 (inside the north-star 1e-3), scores
# up to 4.9e-3 relative for low-confidence detections (sigmoid slope x fp16 activation
# rounding through 23 layers); the north-star 1e-3 score bar needs fp32 activation storage.
CONF_REL = 6e-3    # |d score| / score
CONF_ABS = 2e-3    # a detection this close to the threshold may exist on one side only


@pytest.fixture(scope="module")
def clip():
    W, H = 3840, 2160
    spec = synthetic.SceneSpec("dense", W, H, 3, seed=0)
    gt = synthetic.generate_scene(spec)
    frames = [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(3)]
    return frames


@pytest.fixture(scope="module")
def engine(cuda):
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    return AttentionPipelineB200(settings, 3840, 2160, max_frames=2)


def _run_clip(engine, clip):
    out = engine.evaluate_frames(clip[:2], history=())
    out += engine.evaluate_frames(clip[2:], history=None)  # history carried on device
    return out


def test_engine_runs_and_finds_objects(engine, clip):
    out = _run_clip(engine, clip)
    assert len(out) == 3
    for res, att in out:
        assert res.total_count == 18
        assert 0 < res.active_count <= 18
        assert len(att.boxes) > 0
        assert len(res.detections) > 0
        for d in res.detections:
            assert d.confidence >= 0.3


def test_selection_bit_exact_given_gpu_stage1_boxes(engine, clip):
    out = _run_clip(engine, clip)
    plan = R.Plan(3840, 2160, 1, 3, 20)
    hist = []
    for res, att in out:
        boxes = [(b.x, b.y, b.w, b.h) for b in att.boxes]
        merged = R.merge_temporal(hist + [boxes], 2)
        act = R.select_active(plan.fin, merged, 20, 3840, 2160)
        assert len(act) == res.active_count
        hist = [boxes]
    # last batch's per-frame active id lists
    ids = engine.active_ids.cpu().numpy()
    cnt = engine.active_counts.cpu().numpy()
    assert sorted(ids[0, : cnt[0]].tolist()) == act


def test_nms_keep_set_bit_exact_given_gpu_raw_detections(engine, clip):
    engine.evaluate_frames(clip[:2], history=())
    torch = native.require_cuda()
    n = 2
    pc = engine.pcounts[:n].cpu().numpy()
    raw = engine.pdets.view(-1)[: n * MAX_PER_FRAME * 56].cpu().numpy().view(
        native.PDET_DTYPE).reshape(n, MAX_PER_FRAME)
    oc = engine.ocounts[:n].cpu().numpy()
    out = engine.outp.view(-1)[: n * MAX_PER_FRAME * 56].cpu().numpy().view(
        native.PDET_DTYPE).reshape(n, MAX_PER_FRAME)
    plan = R.Plan(3840, 2160, 1, 3, 20)
    cell_of = R.cell_map(plan)
    for f in range(n):
        tagged = [(int(r["crop_id"]), ((float(r["x"]), float(r["y"]), float(r["w"]),
                                        float(r["h"])), yolo.COCO_NAMES[int(r["cls"])],
                                       float(r["conf"]))) for r in raw[f, : pc[f]]]
        ref = R.finish(tagged, cell_of, 0.3)
        got = [((float(r["x"]), float(r["y"]), float(r["w"]), float(r["h"])),
                yolo.COCO_NAMES[int(r["cls"])], float(r["conf"])) for r in out[f, : oc[f]]]
        assert got == ref
        assert len(tagged) > 0
    del torch


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_boxes_and_scores_match_cpu_oracle(engine, clip, precision):
    """Stage-1 tiles of frame 0 through both networks; decoded detections compared.
    fp16: 16-bit activations on both sides (CONF_REL); fp32: the hi/lo parity mode against
    the fp32 reference at the north-star bar (1e-3 relative for boxes and scores)."""
    fr = clip[0]
    plan = R.Plan(3840, 2160, 1, 3, 20)
    tiles = np.stack([R.cut_tile_nearest(fr.pixels, c) for c in plan.att[3]]
                     + [R.cut_tile_nearest(fr.pixels, plan.fin[3][k]) for k in (7, 8)])
    det = yolo.YoloB200Detector(max_tiles=4, precision=precision)
    gpu = det.detect_tiles(tiles)
    wpacks, biases = yolo.make_weights(0, dtype="fp16")
    head = yolo_ref.forward(tiles, wpacks, biases, mode=precision)
    ref = yolo_ref.region_decode(head, det.threshold)
    n_match, conf_err, box_err = 0, 0.0, 0.0
    for g_list, r_list in zip(gpu, ref):
        r_used = set()
        for g in g_list:
            gc = np.array([g.rect.x, g.rect.y, g.rect.w, g.rect.h])
            best, bd = None, 1e9
            for k, (rr, cls, conf, idx) in enumerate(r_list):
                if k in r_used or yolo.COCO_NAMES[cls] != g.class_label:
                    continue
                d = np.abs(np.array(rr) - gc).max()
                if d < bd:
                    best, bd = k, d
            if best is None or bd / 608 > BOX_REL:
                assert abs(g.confidence - det.threshold) < CONF_ABS, (g, bd)
                continue
            r_used.add(best)
            conf_err = max(conf_err, abs(r_list[best][2] - g.confidence) / r_list[best][2])
            box_err = max(box_err, bd / 608)
            n_match += 1
        for k, (rr, cls, conf, idx) in enumerate(r_list):
            if k not in r_used:
                assert abs(conf - det.threshold) < CONF_ABS, (rr, conf)
    print(f"{precision}: matched {n_match}: max score rel err {conf_err:.2e}, "
          f"max box err/608 {box_err:.2e}")
    assert n_match > 0
    assert conf_err <= (CONF_REL if precision == "fp16" else 1e-3) and box_err <= BOX_REL


def _check_selection_and_nms(engine, out, W, H, n):
    """Selection bit-exact given the GPU's stage-1 boxes; NMS/merge bit-exact given the
    GPU's raw stage-2 detections (last batch of n frames)."""
    plan = R.Plan(W, H, engine.settings.attention.rows, engine.settings.final.rows,
                  engine.settings.final.overlap_px)
    hist, acts = [], []
    for res, att in out:
        boxes = [(b.x, b.y, b.w, b.h) for b in att.boxes]
        merged = R.merge_temporal(hist + [boxes], engine.K)
        act = R.select_active(plan.fin, merged, engine.settings.attention_margin_px, W, H)
        assert len(act) == res.active_count
        acts.append(act)
        hist = (hist + [boxes])[-(engine.K - 1):] if engine.K > 1 else []
    # the id sets (not just counts) of the last batch, read from the device
    ids = engine.active_ids[:n].cpu().numpy()
    cnt = engine.active_counts[:n].cpu().numpy()
    for f in range(n):
        assert sorted(ids[f, : cnt[f]].tolist()) == acts[len(acts) - n + f]
    pc = engine.pcounts[:n].cpu().numpy()
    raw = engine.pdets.view(-1)[: n * MAX_PER_FRAME * 56].cpu().numpy().view(
        native.PDET_DTYPE).reshape(n, MAX_PER_FRAME)
    cell_of = R.cell_map(plan)
    for f, (res, _) in enumerate(out[-n:]):
        tagged = [(int(r["crop_id"]), ((float(r["x"]), float(r["y"]), float(r["w"]),
                                        float(r["h"])), yolo.COCO_NAMES[int(r["cls"])],
                                       float(r["conf"]))) for r in raw[f, : pc[f]]]
        ref = R.finish(tagged, cell_of, engine.settings.min_confidence)
        got = [((d.rect.x, d.rect.y, d.rect.w, d.rect.h), d.class_label, d.confidence)
               for d in res.detections]
        assert got == ref


def test_8k_engine_parity(cuda):
    """BASELINE config 4 frames (7680x4320): same parity contract at 8K."""
    W, H = 7680, 4320
    gt = synthetic.generate_scene(synthetic.SceneSpec("mixed", W, H, 2, seed=0))
    frames = [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(2)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, W, H, max_frames=2)
    out = eng.evaluate_frames(frames, history=())
    assert all(r.total_count == 18 and r.active_count > 0 for r, _ in out)
    _check_selection_and_nms(eng, out, W, H, 2)


def test_allcrops_mode_equals_api_allcrops_baseline(cuda, clip):
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=1)
    eng._upload_frames(clip[:1])
    eng.run_device(1, attention="all")
    (res, _), = eng.results([clip[0].frame_id])
    assert res.active_count == res.total_count == 18
    det = yolo.YoloB200Detector(max_tiles=18)
    api = P.run_allcrops_baseline(clip[0], settings, det)
    assert res.detections == api.detections and len(api.detections) > 0


def test_injected_density_activates_exactly_k_crops(cuda, clip):
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=2)
    eng._upload_frames(clip[:2])
    fin = eng.plan.final_grid.crops
    for k in (1, 5, 18):
        from paper_1810_10551_b200.engine import exclusive_boxes

        boxes = [exclusive_boxes(eng.plan.final_grid, [c.crop_id for c in fin[:k]], 20)] * 2
        eng.reset_history(())
        eng.set_attention(boxes)
        eng.run_device(2, attention="inject")
        cnt = eng.active_counts[:2].cpu().tolist()
        assert cnt == [k, k]
        ids = eng.active_ids[0, :k].cpu().tolist()
        assert ids == [c.crop_id for c in fin[:k]]


def test_device_renderer_matches_reference_render(cuda):
    import hashlib
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "reference_golden.json")))
    for sc in gold["scenes"]:
        gt = synthetic.generate_scene(synthetic.SceneSpec(sc["kind"], sc["fw"], sc["fh"],
                                                          sc["frames"], seed=0))
        fids = [int(f) for f in sc["render_sha256"]]
        out = synthetic.render_frames_device(sc["fw"], sc["fh"], [gt[f] for f in fids])
        for i, f in enumerate(fids):
            h = hashlib.sha256(out[i].cpu().numpy().tobytes()).hexdigest()
            if sc["fw"] <= 3840:
                assert h == sc["render_sha256"][str(f)]
            else:  # 8K golden not stored: compare with the host restatement
                ref = synthetic.render_frame(sc["fw"], sc["fh"], gt[f])
                assert h == hashlib.sha256(ref.tobytes()).hexdigest()


def test_run_stream_equals_run_sequence_and_aborts_with_cursor(cuda, clip):
    from paper_1810_10551_b200.stream import StreamAborted, run_stream

    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    det = yolo.YoloB200Detector()
    seq = list(P.run_sequence(clip, settings, det))
    streamed = run_stream(clip, settings, batch=2)
    assert [(r.frame_id, r.detections, r.active_count) for r in streamed] == \
        [(r.frame_id, r.detections, r.active_count) for r in seq]
    t = streamed[0].timing
    assert t.io_ms > 0 and t.final_eval_ms > 0 and t.per_worker[0][0].startswith("cuda:")
    bad = list(clip[:2]) + [P.Frame(9, 1280, 720, np.zeros((720, 1280, 3), np.uint8))]
    with pytest.raises(StreamAborted) as ei:
        run_stream(bad, settings, batch=2)
    assert ei.value.cursor == 2 and len(ei.value.completed) == 2


def test_run_stream_ramped_batches_equal_run_sequence(cuda):
    """A stream longer than 2 batches starts with B/4 and B/2 frames (stream.ramp_chunks):
    batches of 1, 2, 4, 4, 1 frames must give run_sequence's results."""
    from paper_1810_10551_b200.stream import ramp_chunks, run_stream

    W, H = 3840, 2160
    gt = synthetic.generate_scene(synthetic.SceneSpec("mixed", W, H, 12, seed=3))
    frames = [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(12)]
    assert [len(c) for c in ramp_chunks(frames, 4)] == [1, 2, 4, 4, 1]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    seq = list(P.run_sequence(frames, settings, yolo.YoloB200Detector()))
    streamed = run_stream(frames, settings, batch=4)
    assert [(r.frame_id, r.detections, r.active_count) for r in streamed] == \
        [(r.frame_id, r.detections, r.active_count) for r in seq]


def test_run_stream_from_disk_equals_in_memory(cuda, clip, tmp_path):
    """§8f-2: a FrameSource (PPM directory) streamed from disk straight into pinned staging
    gives the same results as the in-memory frames; a corrupt file aborts at its batch."""
    from paper_1810_10551_b200.frameio import FrameSource, frame_file_name, write_ppm
    from paper_1810_10551_b200.stream import StreamAborted, run_stream

    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    for fr in clip:
        write_ppm(tmp_path / frame_file_name(fr.frame_id), fr.pixels)
    src = FrameSource.open(tmp_path)
    mem = run_stream(clip, settings, batch=2)
    disk = run_stream(src, settings, batch=2)
    assert [(r.frame_id, r.detections, r.active_count, r.total_count) for r in disk] == \
        [(r.frame_id, r.detections, r.active_count, r.total_count) for r in mem]
    (tmp_path / frame_file_name(clip[2].frame_id)).write_bytes(b"P6\n1 1\n255\n")
    with pytest.raises(StreamAborted) as ei:
        run_stream(FrameSource.open(tmp_path), settings, batch=2)
    assert ei.value.cursor == 2 and len(ei.value.completed) == 2


def test_cli_run_yolo_b200_and_oracle(cuda, clip, tmp_path, capsys):
    """§8f-3: `cli run` with detector kind yolo-b200 (frames dir -> run_stream) writes the
    same result lines as run_stream; kind oracle equals run_sequence with the scene oracle."""
    from paper_1810_10551_b200 import cli
    from paper_1810_10551_b200.frameio import (frame_file_name, read_results, write_ground_truth,
                                               write_ppm)
    from paper_1810_10551_b200.stream import result_line, run_stream

    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    (tmp_path / "frames").mkdir()
    for fr in clip:
        write_ppm(tmp_path / "frames" / frame_file_name(fr.frame_id), fr.pixels)
    (tmp_path / "y.ini").write_text(
        "[pipeline]\npreset = 1 att, 3 fin, 20 over\n[detector]\nkind = yolo-b200\nbatch = 2\n"
        "[paths]\nframes = frames\nresults = y.jsonl\n")
    assert cli.main(["run", "--config", str(tmp_path / "y.ini")]) == 0
    assert "mode=pipeline frames=3" in capsys.readouterr().out
    ref = [result_line(r) for r in run_stream(clip, settings, batch=2)]
    assert (tmp_path / "y.jsonl").read_text().splitlines() == ref
    assert (tmp_path / "y_timing.csv").is_file()

    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", 3840, 2160, 3, seed=0))
    write_ground_truth(gt, tmp_path / "gt.jsonl")
    (tmp_path / "o.ini").write_text(
        "[pipeline]\npreset = 1 att, 3 fin, 20 over\n[detector]\nkind = oracle\n"
        "[paths]\nground_truth = gt.jsonl\nresults = o.jsonl\n[frame]\nwidth = 3840\n"
        "height = 2160\n")
    assert cli.main(["run", "--config", str(tmp_path / "o.ini")]) == 0
    oracle = P.oracle_for_scene(3840, 2160, settings, gt)
    frames = [P.Frame(i, 3840, 2160) for i in sorted(gt)]
    want = [result_line(r) for r in P.run_sequence(frames, settings, oracle)]
    assert (tmp_path / "o.jsonl").read_text().splitlines() == want
    assert [r.frame_id for r in read_results(tmp_path / "o.jsonl")] == sorted(gt)


def test_fp32_parity_engine(cuda, clip):
    """precision="fp32" (hi/lo activations) through the whole batched pipeline: selection
    and NMS/merge exact as in fp16 mode, stage-1 detections vs the fp32 CPU network within
    the north-star 1e-3, and the same detections as run_sequence with the fp32 detector."""
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=2, precision="fp32")
    out = eng.evaluate_frames(clip[:2], history=())
    assert all(r.total_count == 18 and r.active_count > 0 and r.detections for r, _ in out)
    _check_selection_and_nms(eng, out, 3840, 2160, 2)
    # stage-1 boxes of frame 0 vs the fp32 oracle network on the same attention tile
    plan = R.Plan(3840, 2160, 1, 3, 20)
    tile = R.cut_tile_nearest(clip[0].pixels, plan.att[3][0])
    wpacks, biases = yolo.make_weights(0, dtype="fp16")
    ref = yolo_ref.region_decode(yolo_ref.forward(tile[None], wpacks, biases, mode="fp32"),
                                 0.25)[0]
    crop = plan.att[3][0]
    ref_boxes = [R.to_global(tuple(r[0]), crop, 3840, 2160) for r in ref if r[2] >= 0.3 + 1e-3]
    got_boxes = [(b.x, b.y, b.w, b.h) for b in out[0][1].boxes]
    assert ref_boxes
    for rb in ref_boxes:  # every clearly-above-threshold oracle box is a GPU attention box
        assert any(max(abs(a - b) for a, b in zip(rb, g)) <= 1 for g in got_boxes), rb
    det = yolo.YoloB200Detector(precision="fp32")
    seq = list(P.run_sequence(clip[:2], settings, det))
    assert [r.detections for r in seq] == [r.detections for r, _ in out]


def test_batch_with_empty_frames(cuda, clip):
    """Frames with zero raw detections mixed into a batch (the density-0.1 sweep case):
    every stage must handle per-frame counts of 0; results stay exact for the others."""
    W, H = 3840, 2160
    blank = P.Frame(100, W, H, synthetic.render_frame(W, H, []))
    frames = [blank, clip[0], P.Frame(101, W, H, blank.pixels), clip[1],
              P.Frame(102, W, H, blank.pixels), P.Frame(103, W, H, blank.pixels)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, W, H, max_frames=6)
    for _ in range(3):  # repeated launches reuse shared memory left by other kernels
        out = eng.evaluate_frames(frames, history=())
        for k in (0, 2, 4, 5):  # blank frames may inherit active crops (temporal window)
            assert out[k][0].detections == ()
        assert out[0][0].active_count == 0 and out[5][0].active_count == 0
        assert out[1][0].detections and out[3][0].detections
    _check_selection_and_nms(eng, out, W, H, 6)


@pytest.mark.timeout(120)
def test_all_blank_batch_has_no_stage2_tiles(cuda):
    """A batch with no attention boxes at all: stage 2 has zero tiles (device count 0), so
    every conv CTA owns no tile — kernels must exit instead of waiting for weights."""
    W, H = 3840, 2160
    blank = synthetic.render_frame(W, H, [])
    frames = [P.Frame(200 + i, W, H, blank) for i in range(3)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, W, H, max_frames=3)
    out = eng.evaluate_frames(frames, history=())
    assert [(r.active_count, r.detections) for r, _ in out] == [(0, ())] * 3
    assert int(eng.n_jobs2.item()) == 0


def test_bilinear_resample_engine_parity(cuda, clip):
    """resample="bilinear" (the north-star ingest downscale, integer fixed point) through
    the whole engine: same selection / NMS exactness contract as nearest."""
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=2, resample="bilinear")
    out = eng.evaluate_frames(clip[:2], history=())
    assert all(r.total_count == 18 and r.active_count > 0 and r.detections for r, _ in out)
    _check_selection_and_nms(eng, out, 3840, 2160, 2)


def test_capacity_overflow_fails_loudly(cuda, clip):
    """Maximum sizes: with detector threshold 0 every candidate (1805 per tile) survives
    decode, so a frame's raw stage-2 detections exceed the 2048-record postprocess capacity;
    the engine must raise StageFailure instead of silently truncating."""
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=1, threshold=0.0)
    with pytest.raises(P.StageFailure):
        eng.evaluate_frames(clip[:1], history=())


@pytest.mark.parametrize("W,H,precision", [(1280, 720, "fp16"), (1920, 1080, "bf16")])
def test_engine_other_sizes_and_bf16(cuda, W, H, precision):
    """720p / 1080p frames (other crop sides, partial edge crops) and bf16 activations:
    same selection / NMS exactness contract."""
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 2, seed=1))
    frames = [P.Frame(i, W, H, synthetic.render_frame(W, H, gt[i])) for i in range(2)]
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    eng = AttentionPipelineB200(settings, W, H, max_frames=2, precision=precision)
    out = eng.evaluate_frames(frames, history=())
    assert all(r.total_count == eng.F for r, _ in out)
    _check_selection_and_nms(eng, out, W, H, 2)


def test_cuda_graph_step_matches_eager(cuda, clip):
    """engine.capture(): a CUDA-graph replay of the device step gives the eager results."""
    torch = cuda
    settings = P.PipelineSettings.from_preset("1 att, 3 fin, 20 over")
    frames = torch.from_numpy(np.stack([f.pixels for f in clip[:1]])).cuda()
    eager = AttentionPipelineB200(settings, 3840, 2160, max_frames=1)
    eager.reset_history(())
    want = []
    for _ in range(3):
        eager.run_device(1, frames=frames)
        want.append([(r.detections, r.active_count) for r, _ in eager.results([0])])
    eng = AttentionPipelineB200(settings, 3840, 2160, max_frames=1)
    eng.reset_history(())
    step = eng.capture(1, frames)  # capture performs one warm-up step (history advances)
    eng.reset_history(())
    got = []
    for _ in range(3):
        step()
        got.append([(r.detections, r.active_count) for r, _ in eng.results([0])])
    assert got == want and want[0][0][0]
