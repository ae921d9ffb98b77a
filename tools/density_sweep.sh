#!/bin/bash
# BASELINE config 5 (density sweep) and config 3 (all-crops comparator) on 1 GPU:
# stage-1 boxes injected so that round(d*F) final crops are active per frame.
# Usage (under gpurun): tools/density_sweep.sh [4k|8k] > gpurun_out/sweep.jsonl
FRAME=${1:-4k}
for d in 0.1 0.2 0.3 0.4 0.5 0.6 0.7 0.8 0.9 1.0; do
  python bench.py --frame $FRAME --steps 5 --warmup 3 --clip-frames 90 --density $d \
      --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
done
python bench.py --frame $FRAME --steps 5 --warmup 3 --clip-frames 90 --mode allcrops \
    --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
python bench.py --frame $FRAME --steps 5 --warmup 3 --clip-frames 90 \
    --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
