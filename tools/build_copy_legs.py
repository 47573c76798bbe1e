# Copy legs of an end-to-end build call (host sequences -> file image): H2D,
# kernels, D2H (tools only).  usage: build_copy_legs.py [c1|c2s]
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1905_09624_b200 as cb
from workloads import synth
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = synth.CONFIGS["c1"] if name == "c1" else synth.scaled(synth.CONFIGS["c2"], 2000)
buf, off = synth.docs(cfg)
names = synth.doc_names(cfg)
docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p)
for rep in range(3):
    t = time.perf_counter()
    img = cb.build_classic(docs, params, device=0)
    wall = (time.perf_counter() - t) * 1e3
    print(name, "corpus MB %.0f image MB %.0f" % (buf.nbytes / 1e6, len(img) / 1e6),
          {k: round(v, 2) for k, v in cb.last_build_timing_ex().items()}, "wall %.1f" % wall, flush=True)
