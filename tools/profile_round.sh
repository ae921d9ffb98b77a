#!/bin/bash
# Profiling recipe for one round (run under gpurun on ONE GPU):
#   plain bench -> launch list (gpu__time_duration per launch) -> ncu --set full on the
#   conv kernel launches of one YOLO forward. Outputs land in gpurun_out/.
set -u
CMD="python bench.py --steps 2 --warmup 3 --batch 8 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
tail -1 gpurun_out/plain.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
# conv launches: each step = 2 forwards x 23 conv launches; skip step 0's stage-1 forward
ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 23 -c 23 \
    -o gpurun_out/conv_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ls -la gpurun_out/
