"""Phase cycles of the fused layer 4 -> 5 swap kernel (TP_CONV_DEBUG=32), per CTA.

    TP_CONV_DEBUG=32 python tools/fused_phases.py [--tiles 120]

x4 wait = waiting for the shared staging buffer, staging = layer 4's HL8 values into it,
mma wait = waiting for the 1x1's MMAs, epilogue = the 1x1's HL8 output (all summed over the
two epilogue groups' warp 0); MMA issuer: total, waiting for a drained accumulator (tempty),
waiting for operands (full)."""

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1810_10551_b200 import native, yolo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=120)
    a = ap.parse_args()
    if not int(os.environ.get("TP_CONV_DEBUG", "0")) & 32:
        sys.exit("set TP_CONV_DEBUG=32")
    lib = native.load()
    net = yolo.YoloNet(a.tiles)
    assert net.fused_steps, "plan is not fused"
    step = min(net.fused_steps) - 1
    x = net.input_tensor(a.tiles)
    x[:, 1:-1, 1:-1, :] = torch.rand_like(x[:, 1:-1, 1:-1, :].float()).to(x.dtype)
    net.forward(a.tiles)
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 8)()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lib.tp_debug_conv_counters(None, 0, 1)
    net.forward_range(a.tiles, step, step)
    torch.cuda.synchronize()
    lib.tp_debug_conv_counters(buf, 8, 0)
    c = [v / sms / 1e3 for v in buf]
    print(f"per CTA (kcycles): MMA issuer {c[2]:.1f} (tempty wait {c[3]:.1f}, full wait {c[4]:.1f})")
    print(f"epilogue warp 0 of both groups: x4 wait {c[0]:.1f}, staging {c[1]:.1f}, "
          f"mma wait {c[5]:.1f}, epilogue {c[6]:.1f}")


if __name__ == "__main__":
    main()
