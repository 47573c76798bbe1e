#!/bin/bash
# A/B build timing on one box: tools/ab_build.sh <libA> <libB> <configs...>
# (alternates the two libraries twice per config; prints count/fill ms)
A=$1; B=$2; shift 2
for cfg in "$@"; do
  for rep in 1 2; do
    for L in "$A" "$B"; do
      COBS_GPU_LIB=$L python tools/config_runs.py $cfg --build-only --repeat 2 --out /tmp/ab.json > /tmp/ab.log 2>&1
      python -c "
import json,sys; r=json.load(open('/tmp/ab.json'))[0]['build']
print('$cfg', '$(basename $L)', 'count %.1f fill %.1f total %.1f' % (r['ms_count'], r['ms_fill'], r['ms_total_call']))"
    done
  done
done
