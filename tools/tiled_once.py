# one tiled batch on a config-5-shaped index (for ncu captures; tools only)
import os, sys
sys.path.insert(0, '.')
import paper_1905_09624_b200 as cb
from workloads import synth
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 26000
median = float(sys.argv[3]) if len(sys.argv) > 3 else 2.4e6
view = cb.synth_c5(7, docs, 1024, median, 0.5, 0.3, device=0)
cfg = synth.replace(synth.CONFIGS["c5"], n_docs=100, n_queries=nq)
qb, qo = synth.queries(cfg)
for rep in range(2):
    b = cb.query_batch_raw(view, qb, qo, 0.8, 0, keep_device=True)
    print("path", b.gather_path, "gather_ms", b.ms_gather, "GB/s", b.row_bytes / b.ms_gather / 1e6, flush=True)
