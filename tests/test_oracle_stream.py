"""The full-size streaming check (oracle/cobs_stream.c) pinned against the
plain restatement (orc_build_image, itself pinned against the reference):
on scaled instances of configs 2-4 (same shapes, small sizes) the streamed
check of orc_build_image's file passes with every byte, and a flipped
payload bit, a changed term count or a wrong width are each caught.  CPU
only; the GPU test (test_gpu_full_configs.py) runs it at full size."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import synth


def scaled_image(name, n_docs, len_scale, **kw):
    cfg = synth.scaled(synth.CONFIGS[name], n_docs, len_scale, **kw)
    lengths = synth.doc_lengths(cfg)
    buf, off = synth.docs(cfg, lengths=lengths)
    names = synth.doc_names(cfg)
    docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
    img = O.build_image(docs, q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                        block_size=cfg.block_size, kind=cfg.kind)
    return cfg, lengths, docs, img


def check(cfg, lengths, img, threads=4):
    return O.stream_check(cfg.seed, cfg.alpha, lengths, img, q=cfg.q, k=cfg.k, p=cfg.p,
                          canonical=cfg.canonical, block_size=cfg.block_size, kind=cfg.kind,
                          threads=threads)


@pytest.mark.parametrize("name,n_docs,scale,block", [
    ("c2", 150, 0.004, 0), ("c3", 300, 0.002, 64), ("c4", 200, 0.002, 0), ("c1", 70, 0.05, 0)])
def test_stream_check_equals_restatement(name, n_docs, scale, block):
    kw = {"block_size": block} if block else {}
    cfg, lengths, docs, img = scaled_image(name, n_docs, scale, **kw)
    r = check(cfg, lengths, img)
    assert r["header_equal"] and r["payload_bad_bytes"] == 0 and r["term_count_mismatch"] == 0, r
    want_tc = [len(O.extract_terms(c, cfg.q, cfg.canonical)[0]) for _, c in docs]
    assert list(r["term_counts"]) == want_tc
    assert r["windows"] == int(np.maximum(lengths.astype(np.int64) - cfg.q + 1, 0).sum())


def test_stream_check_catches_corruption():
    cfg, lengths, docs, img = scaled_image("c4", 150, 0.002)
    idx = O.OracleIndex.parse(img)
    b0 = idx.x.blocks[0]
    arr = np.frombuffer(img, np.uint8).copy()
    # one payload bit: row 7, byte 3
    pos = b0.offset + 7 * b0.row_bytes + 3
    arr[pos] ^= 0x10
    r = check(cfg, lengths, arr)
    assert r["header_equal"] and r["payload_bad_bytes"] == 1
    assert (r["bad_block"], r["bad_row"], r["bad_byte"]) == (0, 7, 3)
    # a term count in the header (the first document's, last byte of its u64)
    arr = np.frombuffer(img, np.uint8).copy()
    tc_pos = 52 + 16 + 2 + len(idx.names()[0])
    arr[tc_pos] ^= 1
    r = check(cfg, lengths, arr)
    assert not r["header_equal"] and r["term_count_mismatch"] == 1
    # unknown document name
    arr = np.frombuffer(img, np.uint8).copy()
    arr[52 + 16 + 2] = ord("x")
    with pytest.raises(O.OracleError):
        check(cfg, lengths, arr)
