"""Conv DRAM traffic per tile from an ncu --set full raw export of one stage-2 forward
(tools/profile_round.sh conv_raw_<tag>.csv.gz) -> profiles/<tag>_conv_traffic_fp32.json,
the file bench.py reads for roofline.traffic.

    python tools/conv_traffic.py gpurun_out/conv_raw_r02h.csv.gz r02h "<capture command>"

The tile count is inferred from the first launch whose input is HBM-cold and known: the
fused layer 4 + 5 kernel reads layer 3's pooled HL8 output (152^2 x 64 x 3 B per tile) plus
its weights, so tiles = its DRAM reads / that size (writes still in L2 when a kernel ends are
counted by later kernels, as in any per-kernel DRAM split)."""

import csv
import gzip
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.algorithmic_bytes import activation_mb, weights_mb  # noqa: E402

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
P152_HL8_MB = 152 * 152 * 64 * 3 / 1e6


def main():
    path, tag, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
    hdr, units, data = rows[0], rows[1], rows[2:]

    def col(r, name):
        i = hdr.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    rd = [col(r, "dram__bytes_read.sum") for r in data]
    wr = [col(r, "dram__bytes_write.sum") for r in data]
    ms = sum(col(r, "gpu__time_duration.sum") for r in data)
    assert len(data) == 22, f"expected the fused plan's 22 conv launches, got {len(data)}"
    tiles = round(rd[2] / P152_HL8_MB)
    total = sum(rd) + sum(wr)
    out = {
        "capture": cmd,
        "tiles": tiles,
        "tiles_note": "from the fused layer 4+5 kernel's DRAM reads / 4.435 MB of HL8 input per tile",
        "forward_ms_ncu": round(ms, 2),
        "dram_MB": round(total, 1),
        "dram_MB_per_tile": round(total / tiles, 2),
        "algorithmic_MB_per_tile": round(activation_mb("fp32"), 2),
        "weights_MB_per_forward": round(weights_mb("fp32"), 1),
        "note": "algorithmic = every HBM-resident activation (HL8: 3 bytes per element) read once "
                "+ written once per tile, layer 4's output kept on chip by the fused kernel "
                "(tools/algorithmic_bytes.py); weights amortised over the batch. Per-layer: "
                f"profiles/{tag}_conv_layers_ncu.csv.",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
