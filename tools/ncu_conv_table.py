"""Per-layer summary of an `ncu --set full` capture of one YOLO forward's conv launches.

    python tools/ncu_conv_table.py gpurun_out/conv_full_r01c.ncu-rep > profiles/r01_conv_layers_ncu.csv

Columns: darknet layer, kernel, duration, share, DRAM read/write MB, tensor-pipe active %
(realtime, of elapsed), SM throughput %, grid. Durations are ncu's serialised cold-cache
replays: compare shares, not absolutes (profiling recipe).
"""

import csv
import io
import subprocess
import sys

LAYERS = [0, 2, 4, 5, 6, 8, 9, 10, 12, 13, 14, 15, 16, 18, 19, 20, 21, 22, 23, 24, 26, 29, 30]
# the fp32 (HL8) plan runs layer 5 inside layer 4's kernel: 22 launches
LAYERS_FUSED = [0, 2, "4+5"] + LAYERS[4:]
COLS = {
    "name": "Kernel Name",
    "ms": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "tensor": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
}
SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "byte": 1e-6, "B": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0,
         "Gbyte": 1e3, "GB": 1e3}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {k: hdr.index(v) for k, v in COLS.items()}

    def val(r, k):
        s = r[idx[k]].replace(",", "")
        try:
            return float(s) * SCALE.get(units[idx[k]], 1.0)
        except ValueError:
            return float("nan")

    tot = sum(val(r, "ms") for r in data)
    rd_tot = sum(val(r, "rd") + val(r, "wr") for r in data)
    print(f"# ncu --set full --clock-control none: {len(data)} conv launches of one YOLO forward ({rep})")
    print("layer,kernel,ms,share_pct,dram_read_MB,dram_write_MB,tensor_active_pct,sm_throughput_pct,grid")
    for i, r in enumerate(data):
        name = r[idx["name"]].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        layer = (LAYERS[i] if len(data) == len(LAYERS)
                 else LAYERS_FUSED[i] if len(data) == len(LAYERS_FUSED) else i)
        print(f"{layer},{name.replace(',', ';')},{val(r, 'ms'):.3f},{100 * val(r, 'ms') / tot:.1f},"
              f"{val(r, 'rd'):.1f},{val(r, 'wr'):.1f},{val(r, 'tensor'):.1f},{val(r, 'sm'):.1f},"
              f"{int(val(r, 'grid'))}")
    print(f"# forward total {tot:.3f} ms, DRAM traffic {rd_tot:.1f} MB")


if __name__ == "__main__":
    main()
