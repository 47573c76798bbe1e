#!/bin/bash
# Build-path timing and per-kernel launch list (used on the GPU box).
#   tools/build_prof.sh c3 [tag]
set -u
cfg=${1:-c3}; tag=${2:-x}
python tools/config_runs.py $cfg --build-only --repeat 2 --out gpurun_out/build_${cfg}_${tag}.json > gpurun_out/build_${cfg}_${tag}.log 2>&1 || exit 1
cut -c1-420 gpurun_out/build_${cfg}_${tag}.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pc_|count_kernel|slab|unit_copy|DeviceScan" --csv \
    --log-file gpurun_out/launch_${cfg}_${tag}.csv python tools/config_runs.py $cfg --build-only \
    --out gpurun_out/build_${cfg}_${tag}_ncu.json > gpurun_out/ncu_${cfg}_${tag}.log 2>&1
python - "$cfg" "$tag" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(f"gpurun_out/launch_{sys.argv[1]}_{sys.argv[2]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split("(")[0][-40:]; agg[k][0] += 1; agg[k][1] += float(r[vi].replace(",", ""))
for k, (n, t) in agg.items():
    print(f"{k:42s} {n:5d} {t/1e6:10.2f} ms")
PY
