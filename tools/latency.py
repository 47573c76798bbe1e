#!/usr/bin/env python
"""Per-call latency of the batch query through the C-ABI on the config-5
index (100,000 documents, ~99 GB in HBM): batches of 1 .. 4,096 random
1,000-bp queries from host memory, hit lists back to the host.

    python tools/latency.py [--out gpurun_out/latency.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1905_09624_b200 as cb  # noqa: E402
from workloads import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "latency.json"))
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    cfg = synth.CONFIGS["c5"]
    view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    res = {"index_bytes_hbm": view.device_bytes(), "batches": []}
    for n in (1, 8, 64, 512, 4096):
        qb, qo = synth.queries(cfg, np.arange(n, dtype=np.uint64))
        for _ in range(3):
            cb.query_batch_raw(view, qb, qo, cfg.K)
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            r = cb.query_batch_raw(view, qb, qo, cfg.K)
            ts.append((time.perf_counter() - t) * 1e3)
        med = statistics.median(ts)
        res["batches"].append({"queries": n, "ms_median": med, "ms_min": min(ts),
                               "ms_device_total": r.ms_total, "ms_termize": r.ms_termize,
                               "ms_gather": r.ms_gather, "ms_order": r.ms_order,
                               "queries_per_s": n / (med / 1e3),
                               "launches": r.launches})
        print(json.dumps(res["batches"][-1]), flush=True)
    view.close()
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
