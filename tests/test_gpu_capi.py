"""The C-ABI from plain C (tests/capi/tp_capi_demo.c, built here with gcc against
include/tilepipe_b200.h and the in-tree library): one 4K frame's two attention tiles
through tp_gather_tiles -> tp_yolo_create_ex / tp_yolo_forward (the default fp32-parity
plan) -> tp_region_decode, with cudaMalloc'd memory and no Python or torch in the process.
Its head and detection records must equal the Python engine path's bit for bit (same
kernels, same inputs)."""

import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

from paper_1810_10551_b200 import kernels, native, synthetic, yolo

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W, H = 3840, 2160


def _build(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "tp_capi_demo")
    lib_dir = os.path.dirname(native.LIB_PATH)
    cuda = "/usr/local/cuda"
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-o", exe,
                    os.path.join(ROOT, "tests", "capi", "tp_capi_demo.c"),
                    f"-I{cuda}/include", f"-L{cuda}/lib64", "-lcudart", f"-L{lib_dir}",
                    "-ltilepipe_b200", f"-Wl,-rpath,{lib_dir}:{cuda}/lib64"], check=True)
    return exe


def _blob(net, path):
    with open(path, "wb") as f:
        f.write(b"TPW1" + struct.pack("<i", len(yolo.LAYERS)))
        for li in range(len(yolo.LAYERS)):
            hi = net.w_dev[li].cpu().numpy().tobytes()
            lo = b"" if net.wlo_dev[li] is None else net.wlo_dev[li].cpu().numpy().tobytes()
            b = net.b_dev[li].cpu().numpy().astype(np.float32).tobytes()
            for chunk in (hi, lo, b):
                f.write(struct.pack("<Q", len(chunk)) + chunk)
            f.write(struct.pack("<f", float(net.alphas[li])))


def test_c_program_matches_python_engine(cuda, tmp_path):
    torch = cuda
    exe = _build(tmp_path)
    gt = synthetic.generate_scene(synthetic.SceneSpec("dense", W, H, 1, seed=0))[0]
    px = synthetic.render_frame(W, H, gt)
    (tmp_path / "frame.raw").write_bytes(px.tobytes())
    net = yolo.YoloNet(2)  # default precision: the HL8 parity plan
    _blob(net, tmp_path / "w.blob")
    out = subprocess.run([exe, str(tmp_path / "w.blob"), str(tmp_path / "frame.raw"), str(W),
                          str(H), str(tmp_path / "head.f32"), str(tmp_path / "dets.bin")],
                         capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stderr
    c_head = np.fromfile(tmp_path / "head.f32", dtype=np.float32).reshape(2, 19, 19, -1)
    raw = (tmp_path / "dets.bin").read_bytes()
    c_counts = np.frombuffer(raw[:8], dtype=np.int32)
    c_recs = np.frombuffer(raw[8:], dtype=native.DET_DTYPE)

    # the same two crops through the Python side of the same library
    frame = torch.from_numpy(px).cuda()
    jobs = kernels.jobs_tensor([(0, 0, 0, 0, H, 0), (0, 1, W - H, 0, H, 1)])
    kernels.gather(frame, W * H * 3, H, W, jobs, 2, "nearest", out_act_ptr=net.input_ptr,
                   dtype=net.dtype)
    net.forward(2)
    det_out, det_counts = kernels.alloc_dets(2)
    kernels.decode(net, 2, jobs, W, H, 0.25, det_out, det_counts)
    torch.cuda.synchronize()
    py_head = net.head_tensor(2).cpu().numpy()
    recs, counts = kernels.dets_to_host(det_out, det_counts, 2)
    assert np.array_equal(c_head, py_head)
    assert c_counts.tolist() == counts.tolist() and counts.sum() > 0
    py_recs = np.concatenate([recs[t, : counts[t]] for t in range(2)])
    assert c_recs.tobytes() == py_recs.tobytes()
