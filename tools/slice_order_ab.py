# A/B of the gather's CTA order (COBS_SLICE_INNER: (block, query group, slice)
# instead of (task, query group); the variant was not kept) on
# full-size C2 / C4 indexes built on the device (tools only).  usage: slice_order_ab.py c2|c4
import os, sys, json
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1905_09624_b200 as cb
from paper_1905_09624_b200 import synth
name = sys.argv[1]
cfg = synth.CONFIGS[name]
lengths = synth.doc_lengths(cfg)
dev = torch.empty(int(lengths.sum()), dtype=torch.uint8, device="cuda:0")
cb.synth_docs_device(cfg.seed, cfg.alpha, lengths, dev.data_ptr(), 0)
seg_off = np.zeros(cfg.n_docs + 1, np.uint64)
np.cumsum(lengths, out=seg_off[1:])
params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical, block_size=cfg.block_size)
view, _ = cb.build_device(dev.data_ptr(), seg_off, np.arange(cfg.n_docs + 1), synth.doc_names(cfg), params,
                          cfg.kind, device=0, seqs_on_device=True)
del dev
torch.cuda.empty_cache()
qb, qo = synth.queries(cfg, lengths=lengths)
ref = None
for kv in ({"COBS_SLICE_INNER": "0"}, {"COBS_SLICE_INNER": "1"}) * 2:
    os.environ.update(kv)
    ts = []
    for rep in range(4):
        b = cb.query_batch_raw(view, qb, qo, cfg.K, scores=False)
        ts.append(b.ms_gather)
    if ref is None:
        ref = (b.hit_n.copy(), b.docs.copy(), b.scores.copy())
    same = bool(np.array_equal(b.hit_n, ref[0]) and np.array_equal(b.docs, ref[1]) and np.array_equal(b.scores, ref[2]))
    print(json.dumps({"cfg": name, "kv": kv, "gather_ms": [round(t, 3) for t in ts],
                      "GBs": round(b.row_bytes / (min(ts) / 1e3) / 1e9), "same_hits": same}), flush=True)
