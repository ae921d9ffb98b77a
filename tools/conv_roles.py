"""Per-role cycle breakdown of the conv kernels (TP_CONV_DEBUG bit 32 counters).

    TP_CONV_DEBUG=32 python tools/conv_roles.py [--tiles 120]

For each conv step of the YOLO forward prints, averaged over CTAs: the MMA issuer's
total cycles and the share it spent waiting for a free accumulator (tempty) and for a
loaded stage (full), the producer's share waiting for a free stage (empty), and the
epilogue warp 0's share waiting for a finished accumulator (tfull). All conv kernels carry
the counters; for the CTA-pair kernel only the leader CTAs count, so its kcyc columns read
half the per-SM value (the percentages are unaffected). An issuer waiting on `full` is not
an idle tensor pipe: MMAs are queued asynchronously (check ncu tensor-pipe activity).
"""

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
    x = net.input_tensor(a.tiles)
    x[:, 1:-1, 1:-1, :] = torch.rand_like(x[:, 1:-1, 1:-1, :].float()).to(x.dtype)
    net.forward(a.tiles)
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 8)()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    print(f"{'step':>4} {'layer':>5} {'ms':>7} {'mma_kcyc':>9} {'tempty%':>8} {'full%':>6} "
          f"{'prod_empty%':>11} {'epi_kcyc':>9} {'epi_tfull%':>10}")
    li = -1
    for s, (kind, _slot) in enumerate(yolo.STEPS):
        if kind != "conv":
            continue
        li += 1
        lib.tp_debug_conv_counters(None, 0, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        net.forward_range(a.tiles, s, s)
        e1.record()
        torch.cuda.synchronize()
        lib.tp_debug_conv_counters(buf, 8, 0)
        c = list(buf)
        n = max(c[7], 1) * sms
        mma, te, fu = c[2] / n, c[3] / n, c[4] / n
        pr, pe = c[0] / n, c[1] / n
        ep, ew = c[5] / n, c[6] / n
        pct = lambda u, v: 100.0 * u / v if v else 0.0  # noqa: E731
        print(f"{s:4d} {yolo.LAYERS[li][0]:5d} {e0.elapsed_time(e1):7.3f} {mma / 1e3:9.1f} "
              f"{pct(te, mma):8.1f} {pct(fu, mma):6.1f} {pct(pe, pr):11.1f} {ep / 1e3:9.1f} "
              f"{pct(ew, ep):10.1f}")


if __name__ == "__main__":
    main()
