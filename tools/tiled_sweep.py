# A/B sweep of the tiled gather's knobs on a config-5-shaped index (tools only)
import json, os, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1905_09624_b200 as cb
from workloads import synth
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 26000
view = cb.synth_c5(7, docs, 1024, 2.4e6, 0.5, 0.3, device=0)
cfg = synth.replace(synth.CONFIGS["c5"], n_docs=100, n_queries=nq)
qb, qo = synth.queries(cfg)
variants = [dict(COBS_TILED="0", **v) for v in (
    {}, {"COBS_EF": "0"}, {"COBS_QT": "26000"}, {"COBS_QT": "26000", "COBS_EF": "0"}, {"COBS_QT": "2048"},
    {"COBS_QT": "2048", "COBS_EF": "0"})]
for kv in variants:
    for k in ("COBS_TILED", "COBS_TILE_LAG", "COBS_TILE_SHIFT", "COBS_TILE_WARPS", "COBS_TILE_QS", "COBS_EF", "COBS_QT"):
        os.environ.pop(k, None)
    os.environ.update(kv)
    ts = []
    for rep in range(3):
        b = cb.query_batch_raw(view, qb, qo, 0.8, 0, keep_device=True)
        ts.append(b.ms_gather)
    print(json.dumps({"kv": kv, "path": b.gather_path, "gather_ms": ts, "row_bytes": b.row_bytes,
                      "GBs": b.row_bytes / (min(ts) / 1e3) / 1e9}), flush=True)
