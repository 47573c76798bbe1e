#!/bin/bash
# A/B of a build knob given as an environment assignment, same library:
#   tools/ab_env_build.sh "VAR=a" "VAR=b" <configs...>
A=$1; B=$2; shift 2
for cfg in "$@"; do
  for rep in 1 2; do
    for E in "$A" "$B"; do
      env $E python tools/config_runs.py $cfg --build-only --repeat 2 --out /tmp/ab.json > /tmp/ab.log 2>&1 || tail -3 /tmp/ab.log
      python -c "
import json; r=json.load(open('/tmp/ab.json'))[0]['build']
print('$cfg', '$E', 'count %.1f fill %.1f total %.1f' % (r['ms_count'], r['ms_fill'], r['ms_total_call']))"
    done
  done
done
