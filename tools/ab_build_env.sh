#!/bin/bash
# A/B of compile-time knobs x environment knobs on one box:
#   tools/ab_build_env.sh "-DCOBS_X=1|ENV=a ENV2=b" "-DCOBS_X=2|" ...
# (rebuilds the library when the compile part changes; C3 by default, CFG=c2|c4)
last=""
for v in "$@"; do
  def="${v%%|*}"; envs="${v#*|}"
  echo "== $def | $envs"
  if [ "$def" != "$last" ]; then
    touch paper_1905_09624_b200/csrc/build.cu
    make -j8 lib EXTRA="$def" > /dev/null 2>&1 || { echo "build failed"; continue; }
    last="$def"
  fi
  env $envs COBS_BUILD_DEBUG=1 python tools/config_runs.py ${CFG:-c3} --build-only --repeat 3 --out /tmp/ab.json 2>&1 | grep -E "count .* ms" | tail -2 | cut -c1-120
  python -c "import json; b=json.load(open('/tmp/ab.json'))[0]['build']; print('  last build: count %.1f fill %.1f total %.1f ms' % (b['ms_count'], b['ms_fill'], b['ms_total_call']))"
done
