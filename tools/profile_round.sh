#!/bin/bash
# Profiling recipe for one round (run under gpurun on ONE GPU):
#   plain bench -> launch list of OUR kernels (gpu__time_duration per launch) ->
#   ncu --set full on the conv launches of one stage-2 YOLO forward (22 in the default fp32
#   plan: layer 5 runs inside layer 4's kernel; NCONV=23 for the other plans).
# Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 1 --batch 30 --no-e2e --no-cpu-baseline --no-sub"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
tail -1 gpurun_out/plain_$TAG.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
# conv launches: warm-up step = 2 forwards; timed step stage-1 = one more
NCONV=${NCONV:-22}
ncu --set full --clock-control none --import-source on -k regex:conv_ -s $((3 * NCONV)) -c $NCONV \
    -o gpurun_out/conv_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
# HBM-bound side kernels (gather, decode, select, postprocess) of the same command
ncu --set full --clock-control none --import-source on \
    -k 'regex:gather_kernel|decode_kernel|select_kernel|postprocess_kernel|build_jobs_kernel|collect_final_kernel|maxpool2' \
    -c 16 -o gpurun_out/aux_full_$TAG $CMD > gpurun_out/ncu_aux_$TAG.log 2>&1
echo "aux rc=$?"
python tools/layer_times.py --tiles 120 > gpurun_out/layer_times_$TAG.txt 2>&1
echo "layer_times rc=$?"
# summaries on the box (the .ncu-rep files exceed what gpurun brings back)
python tools/launch_summary.py gpurun_out/launches_$TAG.csv "$TAG" "$CMD" > gpurun_out/launch_summary_$TAG.txt
python tools/ncu_conv_table.py gpurun_out/conv_full_$TAG.ncu-rep > gpurun_out/conv_layers_$TAG.csv
ncu -i gpurun_out/conv_full_$TAG.ncu-rep --page raw --csv > gpurun_out/conv_raw_$TAG.csv
ncu -i gpurun_out/aux_full_$TAG.ncu-rep --page raw --csv > gpurun_out/aux_raw_$TAG.csv
gzip -f gpurun_out/conv_raw_$TAG.csv gpurun_out/aux_raw_$TAG.csv
[ "$NCONV" = 22 ] && python tools/conv_traffic.py gpurun_out/conv_raw_$TAG.csv.gz "$TAG" \
    "ncu --set full --clock-control none -k regex:conv_ -s 66 -c 22 on $CMD" > gpurun_out/conv_traffic_$TAG.json
ls -la gpurun_out/*.ncu-rep
rm -f gpurun_out/*.ncu-rep
