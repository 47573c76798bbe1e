#!/usr/bin/env python
"""One C5 query batch on the ~100 GB procedural index (for ncu captures of
the real benched configuration; tools only).

    python tools/c5_once.py [--queries 100000]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1905_09624_b200 as cb  # noqa: E402
from workloads import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--queries", type=int, default=100_000)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
cfg = synth.CONFIGS["c5"]
view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
qb, qo = synth.queries(cfg, np.arange(a.queries, dtype=np.uint64))
for _ in range(a.repeat):
    r = cb.query_batch_raw(view, qb, qo, cfg.K)
    print("gather ms %.2f (path %d, %d launches), row bytes %d, %.1f GB/s algorithmic, hits %d"
          % (r.ms_gather, r.gather_path, r.launches, r.row_bytes, r.row_bytes / r.ms_gather / 1e6,
             int(r.hit_n.sum())), flush=True)
view.close()
