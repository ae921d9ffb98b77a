"""Density-sweep table (BASELINE configs 3 and 5) from tools/density_sweep.sh output.

    python tools/sweep_table.py gpurun_out/sweep4k.jsonl gpurun_out/sweep8k.jsonl

One CSV row per bench line: frame, workload, frames/s, crops/s, tiles per frame, conv
TFLOP/s on algorithmic FLOPs and in issued f16-rate work, median SM clock under load.
"""

import json
import sys


def main():
    print("frame,workload,frames_per_s,crops_per_s,tiles_per_frame,conv_TFLOPs_algorithmic,"
          "conv_TFLOPs_executed,sm_mhz")
    for path in sys.argv[1:]:
        for line in open(path):
            line = line.strip()
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            cfg, ws, r = d["config"], d["workload_stats"], d["roofline"]
            w = cfg["workload"]
            wl = (w.split("density ")[1].split(")")[0] if "density " in w else None)
            wl = (f"density {wl}" if wl is not None
                  else "allcrops" if "all-crops" in w else "attention (yolo stage 1)")
            print(f"{cfg['frame'][0] == 7680 and '8k' or '4k'},{wl},{d['value']:.1f},"
                  f"{ws['crops_per_sec']:.0f},{ws['tiles_per_frame']:.2f},{r['achieved']:.0f},"
                  f"{r['executed_tflops']:.0f},{d['clocks']['sm_mhz']:.0f}")


if __name__ == "__main__":
    main()
