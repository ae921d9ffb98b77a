#!/bin/bash
# Profiling recipe for one round (run under gpurun on ONE GPU):
#   plain bench -> launch list of OUR kernels (gpu__time_duration per launch) ->
#   ncu --set full on the 23 conv launches of one stage-2 YOLO forward.
# Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 1 --batch 30 --no-e2e --no-cpu-baseline"
KERN='regex:conv_tc_kernel|conv_pair_kernel|conv_l0_kernel|conv_box_kernel|gather_kernel|decode_kernel|select_kernel|postprocess_kernel|maxpool2_kernel|maxpool2_split_kernel|collect_final_kernel|slice_jobs_kernel|unslice_kernel|attention_boxes_kernel|build_jobs_kernel'
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
tail -1 gpurun_out/plain_$TAG.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KERN" --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
# conv launches: warm-up step = 2 forwards (46 launches); timed step stage-1 = 23 more
ncu --set full --clock-control none --import-source on -k regex:conv_ -s 69 -c 23 \
    -o gpurun_out/conv_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
