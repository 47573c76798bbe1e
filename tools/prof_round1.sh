#!/bin/bash
# Round-1 GPU measurement: full bench (with CPU baseline), launch list of the
# bench command under ncu, and one --set full capture of the gather kernel on
# a 10k-document C5 instance (15 GB, so ncu's replay save/restore fits).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_r1.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?"
kill $SMI
CMD="python bench.py --no-cpu-baseline --no-build --steps 2 --warmup 1"
timeout 600 $CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
SMALL="python bench.py --c5-docs 10000 --queries 10000 --no-cpu-baseline --no-build --steps 1 --warmup 1"
timeout 600 $SMALL > gpurun_out/plain_small.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 1 -c 1 \
    -o gpurun_out/gather_r1 $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
