#!/bin/bash
# A/B of compile-time build knobs on one box: tools/ab_build.sh "-DCOBS_X=1" "-DCOBS_X=2" ...
# (rebuilds the library per variant; C3 by default, CFG=c2|c4 to change)
for v in "$@"; do
  echo "== $v"
  touch paper_1905_09624_b200/csrc/build.cu
  make -j8 lib EXTRA="$v" > /dev/null 2>&1 || { echo "build failed"; continue; }
  COBS_BUILD_DEBUG=1 python tools/config_runs.py ${CFG:-c3} --build-only --repeat 4 --out /tmp/ab.json 2>&1 | grep -E "count .* ms|ms_fill" | tail -3 | cut -c1-300
done
