"""Compulsory HBM bytes per 608^2 tile of one YOLO v2 forward (the roofline's
`algorithmic_bytes_per_tile`): every activation buffer read once by its consumer and
written once by its producer, in the stored layout of each plan (csrc/tp_conv.cu kBufs /
kSteps): compact NHWC 16-bit, the layer-0 input as [610][614][4] rgb0 pixels, the head fp32
[19][19][448]; the fp32x2 plan doubles every activation but the input and head (hi/lo fp16
pairs), the fp32 plan (HL8) stores them as 3 bytes per element (fp16 hi + e4m3 lo planes).
Weights are amortised over the batch and reported separately. The fp32 plan runs layer 5
inside layer 4's kernel (csrc/tp_conv.cu swap_fused_1x1): layer 4's output never reaches
HBM, so its write and read drop out ("fp32" = fused default, "fp32-unfused" = both kept).

    python tools/algorithmic_bytes.py
"""

import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1810_10551_b200 import yolo  # noqa: E402

# buffer: (stored side, channels, bytes per element)
BUFS = {"I608": (610, 4, 2), "P304": (304, 32, 2), "P152": (152, 64, 2), "A152": (152, 128, 2),
        "B152": (152, 64, 2), "P76": (76, 128, 2), "A76": (76, 256, 2), "B76": (76, 128, 2),
        "P38": (38, 256, 2), "A38": (38, 512, 2), "B38": (38, 256, 2), "E38": (38, 512, 2),
        "P19": (19, 512, 2), "A19": (19, 1024, 2), "B19": (19, 512, 2), "C19": (19, 1024, 2),
        "CAT19": (19, 1280, 2), "HEAD": (19, 448, 4)}
# (input buffer, output buffer, channels written) per step, as kSteps
STEPS = [("I608", "P304", 32), ("P304", "P152", 64), ("P152", "A152", 128),
         ("A152", "B152", 64), ("B152", "P76", 128), ("P76", "A76", 256), ("A76", "B76", 128),
         ("B76", "P38", 256), ("P38", "A38", 512), ("A38", "B38", 256), ("B38", "A38", 512),
         ("A38", "B38", 256), ("B38", "E38", 512), ("E38", "P19", 512), ("P19", "A19", 1024),
         ("A19", "B19", 512), ("B19", "C19", 1024), ("C19", "B19", 512), ("B19", "A19", 1024),
         ("A19", "C19", 1024), ("C19", "CAT19", 1024), ("E38", "CAT19", 256),
         ("CAT19", "A19", 1024), ("A19", "HEAD", 448)]


MULT = {"fp16": 1.0, "fp32x2": 2.0, "fp32": 1.5, "fp32-unfused": 1.5}  # bytes per element / 2
ON_CHIP = {"fp32": {"A152"}}  # buffers a plan keeps on chip (fused producer -> consumer)


def activation_mb(plan: str) -> float:
    def mult(b):
        return MULT[plan] if b not in ("I608", "HEAD") else 1

    total = 0
    for src, dst, och in STEPS:
        if dst in ON_CHIP.get(plan, ()):  # the fused kernel reads src, writes the consumer's dst
            continue
        if src in ON_CHIP.get(plan, ()):
            src = next(a for a, b, _ in STEPS if b == src)
        s, c, e = BUFS[src]
        total += (610 * 614 * 4 * 2 if src == "I608" else s * s * c * e * mult(src))
        s, _, e = BUFS[dst]
        total += s * s * och * e * mult(dst)
    return total / 1e6


def weights_mb(plan: str) -> float:
    total = 0
    for li, (_, cin, cout, k, _) in enumerate(yolo.LAYERS):
        cpad = yolo.HEAD_CPAD if li == yolo.HEAD else cout
        kk = 144 * 2 if li == 0 else k * k * cin * 2 * MULT[plan]
        total += cpad * kk
    return total / 1e6


if __name__ == "__main__":
    for plan in ("fp16", "fp32", "fp32-unfused", "fp32x2"):
        print(f"{plan}: activations {activation_mb(plan):.2f} MB per tile, "
              f"weights {weights_mb(plan):.1f} MB per forward")
