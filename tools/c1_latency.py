# per-call wall and event time of the C1 query batch (tools only)
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1905_09624_b200 as cb
from workloads import synth
cfg = synth.CONFIGS["c1"]
buf, off = synth.docs(cfg)
names = synth.doc_names(cfg)
docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
img = cb.build_classic(docs, cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p), device=0)
view = cb.open_image(img, 0)
qb, qo = synth.queries(cfg)
stream = torch.cuda.Stream()
view.set_stream(stream.cuda_stream)
for rep in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0.record(stream)
    out = cb.query_batch_raw(view, qb, qo, cfg.K)
    e1.record(stream)
    torch.cuda.synchronize()
    print("wall %.2f ms  events %.2f ms  lib total %.2f" % ((time.perf_counter() - t) * 1e3, e0.elapsed_time(e1), out.ms_total), flush=True)
