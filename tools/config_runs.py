#!/usr/bin/env python
"""Full-size runs of BASELINE.json configs 1-4 on one B200: build the index
on the device from the seeded corpus (documents generated in HBM), query the
config's batch, and check parity against the CPU oracle through properties
that do not need an oracle-sized build:

  * header: widths == size_filter(block max term_count) (oracle's sizing),
    compact order (term_count, name) non-decreasing;
  * sampled documents: term_count == the oracle's extract_terms, and the
    document's whole bit column == the oracle's single-document build with the
    same forced width (every row, exact);
  * sampled queries: dense scores / l / hits == the oracle querying the
    GPU-built file image.

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


def column_bits(img: bytes, idx: O.OracleIndex, block: int, col: int) -> np.ndarray:
    dc, w, base = idx.blocks()[block]
    rb = (dc + 7) // 8
    off = idx.x.blocks[block].offset
    rows = np.frombuffer(img, dtype=np.uint8, count=w * rb, offset=off).reshape(w, rb)
    return (rows[:, col // 8] >> (col % 8)) & 1


def run(name: str, n_sample_docs: int, n_sample_queries: int, n_queries: int = 0, repeat: int = 1,
        build_only: bool = False):
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

    # ---- parity through properties + samples ----------------------------
    t = time.perf_counter()
    img = cb.index_image(view)
    idx = O.OracleIndex.parse(img)
    checks = {}
    blocks = idx.blocks()
    tcs = np.asarray(idx.term_counts(), dtype=np.uint64)
    checks["widths_sized_by_oracle"] = all(
        w == O.size_filter(int(tcs[base:base + dc].max()), cfg.p, cfg.k) for dc, w, base in blocks)
    if cfg.kind == 1:
        nms = idx.names()
        checks["compact_order"] = all((tcs[i], nms[i]) <= (tcs[i + 1], nms[i + 1])
                                      for i in range(len(nms) - 1))
    name_to_col = {n: i for i, n in enumerate(idx.names())}
    rng = random.Random(7)
    sample = rng.sample(range(cfg.n_docs), n_sample_docs)
    ok_tc = ok_col = True
    for d in sample:
        buf, off = synth.docs(cfg, [d], lengths=lengths)
        content = [buf.tobytes()]
        terms, sk, occ = O.extract_terms(content, cfg.q, cfg.canonical)
        g = name_to_col[names[d]]
        b = next(i for i, (dc, w, base) in enumerate(blocks) if base <= g < base + dc)
        dc, w, base = blocks[b]
        ok_tc &= int(tcs[g]) == len(terms)
        one = O.build_image([(names[d], content)], q=cfg.q, k=cfg.k, p=cfg.p,
                            canonical=cfg.canonical, kind=0, forced_w=w)
        one_idx = O.OracleIndex.parse(one)
        want = column_bits(one, one_idx, 0, 0)
        got = column_bits(img, idx, b, g - base)
        ok_col &= bool(np.array_equal(want, got))
    checks["sampled_term_counts"] = ok_tc
    checks["sampled_columns_exact"] = ok_col
    qs = sorted(rng.sample(range(len(qo) - 1), n_sample_queries))
    ok_q = True
    for i in qs:
        pat = qb[int(qo[i]):int(qo[i + 1])].tobytes()
        try:
            ell, sk, hits, _ = idx.query(pat, cfg.K)
        except O.OracleError as e:
            ok_q &= int(out.status[i]) == e.code
            continue
        d_, s_ = out.hits(i)
        ok_q &= (int(out.ell[i]), int(out.skipped[i])) == (ell, sk)
        ok_q &= [(int(a), int(b)) for a, b in zip(d_, s_)] == hits
    checks["sampled_queries_hits"] = ok_q
    checks["n_sample_docs"] = n_sample_docs
    checks["n_sample_queries"] = n_sample_queries
    checks["check_s"] = time.perf_counter() - t
    res["checks"] = checks
    view.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--docs", type=int, default=4)
    ap.add_argument("--queries", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--build-only", action="store_true")
    a = ap.parse_args()
    results = []
    for c in a.configs:
        r = run(c, a.docs, a.queries, a.batch, a.repeat, a.build_only)
        print(json.dumps(r), flush=True)
        results.append(r)
        json.dump(results, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
