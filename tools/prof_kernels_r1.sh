#!/bin/bash
# ncu --set full captures of kernel 1 (termize) and kernel 4 (count, fill)
# on small instances (C5 10k docs / 10k queries; C1 build), after the same
# commands exited 0 without ncu.
set -x
Q="python bench.py --c5-docs 10000 --queries 10000 --no-cpu-baseline --no-build --steps 1 --warmup 1"
timeout 600 $Q > gpurun_out/plain_q.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:termize -s 1 -c 1 \
    -o gpurun_out/termize_r1 $Q > gpurun_out/ncu_termize.log 2>&1
echo "termize rc=$?"
B="python tools/config_runs.py c1 --docs 1 --queries 1 --out gpurun_out/c1_prof.json"
timeout 600 $B > gpurun_out/plain_b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_kernel|fill_kernel" -c 2 \
    -o gpurun_out/build_r1 $B > gpurun_out/ncu_build.log 2>&1
echo "build rc=$?"
