#!/usr/bin/env python
"""Where the e2e step's time goes on the C5 batch (tools only): wall time of
the C-ABI call from Python vs the library's own event span (H2D of the
patterns through the last D2H), per step, for host (pinned) input."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_09624_b200 as cb  # noqa: E402
from workloads import synth  # noqa: E402

cfg = synth.CONFIGS["c5"]
view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
qb, qo = synth.queries(cfg, np.arange(cfg.n_queries, dtype=np.uint64))
h_pat = torch.from_numpy(qb).pin_memory().numpy()
h_off = torch.from_numpy(qo.view(np.int64)).pin_memory().numpy().view(np.uint64)
for i in range(6):
    t = time.perf_counter()
    r = cb.query_batch_raw(view, h_pat, h_off, cfg.K)
    wall = (time.perf_counter() - t) * 1e3
    print("wall %.1f ms  events %.1f ms (termize %.1f gather %.1f order %.2f)  host %.1f ms"
          % (wall, r.ms_total, r.ms_termize, r.ms_gather, r.ms_order, wall - r.ms_total), flush=True)
