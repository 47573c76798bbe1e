# A/B of a bin-sorted, clock-rotated gather_kernel variant (COBS_SORT /
# COBS_SORT_MODE / COBS_SORT_TSHIFT) on one C5-shaped index (tools only).  The
# variant was measured slower and removed ("HBM page locality");
# this script documents the A/B.  usage: sort_sweep.py [docs] [queries]
import json, os, sys
sys.path.insert(0, '.')
import paper_1905_09624_b200 as cb
from workloads import synth
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
view = cb.synth_c5(1905_09624, docs, 1024, 2.4e6, 0.5, 0.3, device=0)
cfg = synth.replace(synth.CONFIGS["c5"], n_docs=100, n_queries=nq)
qb, qo = synth.queries(cfg)
variants = [{"COBS_SORT": "0"}, {"COBS_SORT": "1", "COBS_SORT_MODE": "1"}, {"COBS_SORT": "1", "COBS_SORT_MODE": "2"},
            {"COBS_SORT": "1", "COBS_SORT_MODE": "0", "COBS_SORT_TSHIFT": "13"}, {"COBS_SORT": "0"}]
ref = None
for kv in variants:
    os.environ.update(kv)
    ts = []
    for rep in range(3):
        b = cb.query_batch_raw(view, qb, qo, 0.8, 0)
        ts.append(b.ms_gather)
    if ref is None:
        ref = (b.hit_n.copy(), b.docs.copy(), b.scores.copy())
    same = bool((b.hit_n == ref[0]).all() and (b.docs == ref[1]).all() and (b.scores == ref[2]).all())
    print(json.dumps({"kv": kv, "gather_ms": [round(t, 2) for t in ts], "GBs": round(b.row_bytes / (min(ts) / 1e3) / 1e9),
                      "hits": int(b.hit_n.sum()), "same_hits": same}), flush=True)
