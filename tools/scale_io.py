#!/usr/bin/env python
"""At-scale timings the bench does not cover (verdict r1 items 6 and 10):

  * kernel 3 under dense hits: the C5 index queried with K = 1e-12 (tau = 1:
    every document with score >= 1 is a hit, ~100,000 hits per query) for a
    1,000-query batch -- gather vs ordering time, hits/s;
  * the resident open of a written ~100 GB C5 file: write_index (D2H +
    file write), then open_resident of the file (parse + read + pitched
    upload), load GB/s; the reopened index answers a batch identically.

    python tools/scale_io.py [--dir /tmp] [--queries 1000] [--out gpurun_out/scale_io.json]
"""
import argparse
import json
import os
import shutil
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1905_09624_b200 as cb  # noqa: E402
from workloads import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--skip-file", action="store_true")
    ap.add_argument("--file-docs", type=int, default=70_000, help="documents of the C5 index written to disk")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "scale_io.json"))
    a = ap.parse_args()
    cfg = synth.CONFIGS["c5"]
    out = {"config": "c5", "n_docs": cfg.n_docs}
    t = time.perf_counter()
    view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    out["synth_s"] = time.perf_counter() - t
    qb, qo = synth.queries(cfg, np.arange(a.queries, dtype=np.uint64))

    # ---- kernel 3 under dense hits ---------------------------------------
    dense = {}
    for K in (0.8, 1e-12):
        cb.query_batch_raw(view, qb, qo, K)  # warm-up (workspace sized)
        t = time.perf_counter()
        r = cb.query_batch_raw(view, qb, qo, K)
        wall = time.perf_counter() - t
        hits = int(r.hit_n.sum())
        dense[str(K)] = {"queries": a.queries, "hits": hits, "hits_per_query": hits / a.queries,
                         "ms_termize": r.ms_termize, "ms_gather": r.ms_gather, "ms_order": r.ms_order,
                         "ms_call_wall": wall * 1e3, "ms_total_events": r.ms_total,
                         "order_hits_per_s": hits / (r.ms_order / 1e3) if r.ms_order else None,
                         "order_share_of_kernels": r.ms_order / (r.ms_termize + r.ms_gather + r.ms_order)}
        print(K, dense[str(K)], flush=True)
    out["dense_hits"] = dense
    ref_batch = cb.query_batch_raw(view, qb, qo, 0.3, 10)

    # ---- write the file, then the resident open ---------------------------
    # (the GPU box's disk holds ~80 GB: the file leg uses --file-docs
    # documents of the same C5 shape, ~0.99 GB per 1,000 documents)
    if a.file_docs and a.file_docs != cfg.n_docs:
        view.close()
        view = cb.synth_c5(cfg.seed, a.file_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
        ref_batch = cb.query_batch_raw(view, qb, qo, 0.3, 10)
        out["file_docs"] = a.file_docs
    if not a.skip_file:
        path = os.path.join(a.dir, "c5_scale.cobs")
        free = shutil.disk_usage(a.dir).free
        size = view.device_bytes()
        out["disk_free_bytes"] = free
        if free < size * 1.1:
            out["file"] = {"skipped": f"{free} bytes free in {a.dir}, need ~{size}"}
        else:
            t = time.perf_counter()
            cb.write_index(view, path)
            wt = time.perf_counter() - t
            fsize = os.path.getsize(path)
            view.close()
            view = None
            t = time.perf_counter()
            v2 = cb.open_resident(path)
            ot = time.perf_counter() - t
            r2 = cb.query_batch_raw(v2, qb, qo, 0.3, 10)
            same = (np.array_equal(r2.hit_n, ref_batch.hit_n) and np.array_equal(r2.ell, ref_batch.ell)
                    and all(np.array_equal(r2.hits(i)[0], ref_batch.hits(i)[0]) for i in range(len(qo) - 1)))
            out["file"] = {"bytes": fsize, "write_s": wt, "write_gbs": fsize / wt / 1e9,
                           "open_resident_s": ot, "open_resident_gbs": fsize / ot / 1e9,
                           "reopened_answers_identical": bool(same),
                           "note": "file written right before the open: it may be (partly) in the page cache"}
            print(out["file"], flush=True)
            v2.close()
            os.remove(path)
    if view is not None:
        view.close()
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
