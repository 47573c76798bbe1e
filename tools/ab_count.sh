#!/bin/bash
# A/B of the partitioned count's dedup knobs on the full C3 build (one box):
#   tools/ab_count.sh "ENV=1 ENV2=2" "ENV=3" ...
# prints ms_count / ms_fill per variant (median of 3 builds after a warm-up)
for v in "$@"; do
  echo "== $v"
  env $v COBS_BUILD_DEBUG=1 python tools/config_runs.py ${CFG:-c3} --build-only --repeat 4 --out /tmp/ab.json 2>&1 | grep -E "count .* ms" | tail -3
done
