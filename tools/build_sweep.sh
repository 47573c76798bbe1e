#!/bin/bash
# count-pass load factor / wave size sweep on config 3 (two builds each, warm)
for cfg in "3 96 96" "4 96 96" "6 192 96" "4 192 48" "4 192 192"; do
  set -- $cfg
  COBS_COUNT_LOAD_DIV=$1 COBS_COUNT_WAVE_MB=$2 COBS_SLAB_WAVE_MB=$3 timeout 900 python tools/config_runs.py c3 --docs 1 --queries 1 --repeat 2 --out gpurun_out/sweep_$1_$2_$3.json > gpurun_out/sweep_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"
done
