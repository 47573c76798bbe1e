#!/bin/bash
# A/B of the query bench on one box: tools/ab_bench.sh <libA> <libB> [extra bench args]
A=$1; B=$2; shift 2
for rep in 1 2; do
  for L in "$A" "$B"; do
    COBS_GPU_LIB=$L python bench.py --no-build --no-cpu-baseline "$@" > /tmp/abb.json 2>/tmp/abb.err
    python -c "
import json; d=json.load(open('/tmp/abb.json'))
print('$(basename $L)', 'value %.1f M  gather %.1f GB/s  frac %.3f  clk %s' % (d['value']/1e6, d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz']))" || tail -3 /tmp/abb.err
  done
done
