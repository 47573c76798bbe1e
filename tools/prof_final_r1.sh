#!/bin/bash
# End-of-round captures with the final code: the bench launch list (ncu
# gpu__time_duration, cold, serialised) and one --set full capture each of
# the gather and termize kernels on a 10k-document C5 instance (15 GB, so
# ncu's replay save/restore fits).  Each command first runs without ncu.
mkdir -p gpurun_out
CMD="python bench.py --no-cpu-baseline --no-build --steps 2 --warmup 1"
timeout 600 $CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
SMALL="python bench.py --c5-docs 10000 --queries 10000 --no-cpu-baseline --no-build --steps 1 --warmup 1"
timeout 600 $SMALL > gpurun_out/plain_small.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel|termize" -c 2 \
    -o gpurun_out/kernels_final $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
