#!/usr/bin/env python
"""Full-size runs of BASELINE.json configs 1-4 on one B200: build the index
on the device from the seeded corpus (documents generated in HBM), query the
config's whole batch, and check parity with the CPU oracle:

  * the file: every byte of the GPU-built image (header and payload) against
    the streamed oracle build of the same corpus (oracle/cobs_stream.c,
    orc_stream_check -- the reference's extract_terms / build_* / write_index
    restated one 64-document column group at a time);
  * dense scores (K = 1e-12, every document's score) of a seeded 1% query
    sample, and their l / skipped, against the oracle querying that image
    (once the image equals the oracle's build, this is the oracle's query);
  * the hit lists of the same sample at the config's K from the full batch.

    python tools/config_runs.py c2 c3 c4 [--out gpurun_out/configs.json]
"""
import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_09624_b200 as cb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads import synth  # noqa: E402


def run(name: str, n_queries: int = 0, repeat: int = 1, build_only: bool = False):
    cfg = synth.CONFIGS[name]
    if n_queries:
        cfg = synth.replace(cfg, n_queries=n_queries)
    res = {"config": name, "n_docs": cfg.n_docs}
    lengths = synth.doc_lengths(cfg)
    total = int(lengths.sum())
    res["corpus_bytes"] = total
    dev = torch.empty(total, dtype=torch.uint8, device="cuda")
    t = time.perf_counter()
    cb.synth_docs_device(cfg.seed, cfg.alpha, lengths, dev.data_ptr())
    res["gen_s"] = time.perf_counter() - t
    seg_off = np.zeros(cfg.n_docs + 1, np.uint64)
    np.cumsum(lengths, out=seg_off[1:])
    doc_segs = np.arange(cfg.n_docs + 1, dtype=np.uint64)
    names = synth.doc_names(cfg)
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                            block_size=cfg.block_size)
    torch.cuda.synchronize()
    for rep in range(repeat):  # the last build is reported (earlier ones warm up)
        if rep:
            view.close()
        t = time.perf_counter()
        view, _ = cb.build_device(dev.data_ptr(), seg_off, doc_segs, names, params, cfg.kind,
                                  seqs_on_device=True)
        wall = time.perf_counter() - t
    c, f, tot = cb.last_build_timing()
    res["build"] = {"ms_count": c, "ms_fill": f, "ms_total_call": tot, "wall_s": wall,
                    "docs_per_s_kernels": cfg.n_docs / ((c + f) / 1e3),
                    "docs_per_s_call": cfg.n_docs / (tot / 1e3),
                    "index_bytes_hbm": view.device_bytes()}
    del dev
    torch.cuda.empty_cache()
    if build_only:
        view.close()
        return res

    # ---- the config's query batch --------------------------------------
    qb, qo = synth.queries(cfg, lengths=lengths)
    stream = torch.cuda.Stream()
    view.set_stream(stream.cuda_stream)
    cb.query_batch_raw(view, qb, qo, cfg.K)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = cb.query_batch_raw(view, qb, qo, cfg.K)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    grams = int(out.ell.astype(np.uint64).sum())
    res["query"] = {"n_queries": len(qo) - 1, "ms_e2e": ms, "qgrams_per_s_e2e": grams / (ms / 1e3),
                    "ms_termize": out.ms_termize, "ms_gather": out.ms_gather,
                    "ms_order": out.ms_order, "row_bytes": out.row_bytes,
                    "gather_gbs": out.row_bytes / (out.ms_gather / 1e3) / 1e9,
                    "hits_total": int(out.hit_n.sum())}

    # ---- parity: the whole file, then a seeded 1% of the queries --------
    t = time.perf_counter()
    img = cb.index_image_array(view)  # the file image, straight into one host array
    res["image_bytes"] = int(len(img))
    res["image_d2h_s"] = time.perf_counter() - t
    t = time.perf_counter()
    rep = O.stream_check(cfg.seed, cfg.alpha, lengths, img, q=cfg.q, k=cfg.k, p=cfg.p,
                         canonical=cfg.canonical, block_size=cfg.block_size, kind=cfg.kind,
                         threads=os.cpu_count() or 1)
    checks = {"file_header_equal": rep["header_equal"],
              "file_payload_bad_bytes": int(rep["payload_bad_bytes"]),
              "file_term_count_mismatch": int(rep["term_count_mismatch"]),
              "oracle_windows": int(rep["windows"]),
              "file_check_s": time.perf_counter() - t,
              "file_check_threads": os.cpu_count() or 1}
    checks["file_byte_identical"] = (rep["header_equal"] and rep["payload_bad_bytes"] == 0
                                     and rep["term_count_mismatch"] == 0)
    if not build_only:
        t = time.perf_counter()
        idx = O.OracleIndex.parse_array(img)
        n_q = len(qo) - 1
        rng = np.random.default_rng(cfg.seed)
        sample = np.sort(rng.choice(n_q, size=max(1, n_q // 100), replace=False)).astype(np.uint64)
        sb, so = synth.queries(cfg, sample, lengths=lengths)
        # dense scores (K = 1e-12: tau = 1, every score exported) of the sample
        g = cb.query_batch_raw(view, sb, so, 1e-12, scores=True, hits=False)
        ell, sk, st, _, dense = idx.query_batch(sb, so, 1e-12, scores=True, threads=os.cpu_count() or 1)
        checks["dense_sample_queries"] = int(len(sample))
        checks["dense_scores_equal"] = bool(np.array_equal(g.dense.astype(np.uint32), dense)
                                            and np.array_equal(g.ell.astype(np.uint64), ell)
                                            and np.array_equal(g.skipped.astype(np.uint64), sk))
        checks["dense_nonzero_frac"] = float((dense > 0).mean())
        # hit lists at the config's K: the full batch's answers for the sample
        ok_q, n_hits = True, 0
        for j, i in enumerate(sample.tolist()):
            pat = sb[int(so[j]):int(so[j + 1])].tobytes()
            try:
                ell_i, sk_i, hits, _ = idx.query(pat, cfg.K)
            except O.OracleError as e:
                ok_q &= int(out.status[i]) == e.code
                continue
            d_, s_ = out.hits(i)
            ok_q &= (int(out.ell[i]), int(out.skipped[i])) == (ell_i, sk_i)
            ok_q &= [(int(a), int(b)) for a, b in zip(d_, s_)] == hits
            n_hits += len(hits)
        checks["sample_hits_equal"] = ok_q
        checks["sample_hits_total"] = n_hits
        checks["query_check_s"] = time.perf_counter() - t
        del idx
    res["checks"] = checks
    del img
    view.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--build-only", action="store_true")
    a = ap.parse_args()
    results = []
    for c in a.configs:
        r = run(c, a.batch, a.repeat, a.build_only)
        print(json.dumps(r), flush=True)
        results.append(r)
        json.dump(results, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
