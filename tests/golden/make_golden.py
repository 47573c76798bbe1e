"""Regenerate the golden fixtures in this directory from the REFERENCE ITSELF
(oracle/_ref = /root/reference/proj sources compiled unmodified).

    python tests/golden/make_golden.py

Writes small index files built and serialised by the reference's
build_classic / build_compact / write_index, and golden.json holding the
reference query() results for a fixed set of patterns (hits at several K /
top_t, error code + message, and dense scores through the K = 1e-12
export).  The fixtures travel with the repo, so the GPU box (where
/root/reference does not exist) still checks against reference outputs.
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def rand(rng, n, alphabet=b"ACGT"):
    return bytes(rng.choice(alphabet) for _ in range(n))


def corpus(rng, n, lo, hi, noisy=False, prefix=b"doc"):
    docs = []
    for i in range(n):
        alpha = b"ACGTN" if noisy and i % 4 == 0 else b"ACGT"
        segs = [rand(rng, rng.randint(lo, hi), alpha) for _ in range(1 + (i % 3 == 0))]
        docs.append((prefix + b"%04d" % i, segs))
    return docs


SPECS = {
    # name: (seed, n_docs, lo, hi, noisy, params)
    "tiny": None,
    "classic_k2": (11, 12, 80, 600, False, dict(k=2, kind=0)),
    "compact_canon": (12, 14, 60, 900, True, dict(k=1, canonical=True, block_size=4, kind=1)),
    "compact_k3": (13, 10, 31, 400, False, dict(k=3, block_size=3, kind=1)),
    "classic_q10_aa": (14, 9, 30, 500, False, dict(q=10, k=2, p=0.1, kind=0)),
}


def main():
    out = {"files": {}, "patterns": [], "results": {}}
    pats_rng = random.Random(2024)
    for name, spec in SPECS.items():
        path = os.path.join(HERE, name + ".cobs")
        if spec is None:
            docs, params = [(b"d", [b"A" * 31])], dict(kind=0)
        else:
            seed, n, lo, hi, noisy, params = spec
            rng = random.Random(seed)
            if name.endswith("_aa"):
                docs = [(b"p%03d" % i, [rand(rng, rng.randint(lo, hi), b"ACDEFGHIKLMNPQRSTVWY")])
                        for i in range(n)]
            else:
                docs = corpus(rng, n, lo, hi, noisy)
        O.ref_build_write(docs, path, **params)
        out["files"][name] = {"docs": [[d[0].decode(), [s.decode() for s in d[1]]] for d in docs],
                              "params": params}
        # patterns: substrings, random, an N-split one, a too-short one
        pats = []
        for i in range(6):
            src = docs[i % len(docs)][1][0]
            ln = min(len(src), 60 + 30 * i)
            st = pats_rng.randrange(len(src) - ln + 1)
            pats.append(src[st:st + ln])
        alpha = b"ACDEFGHIKLMNPQRSTVWY" if name.endswith("_aa") else b"ACGT"
        pats.append(rand(pats_rng, 120, alpha))
        pats.append(pats[1][:30] + b"N" + pats[1][31:])
        pats.append(b"ACGT")
        pats.append(b"N" * 40)
        ref = O.RefIndex.open(path)
        res = []
        for pat in pats:
            for K, top_t in [(1.0, 0), (0.5, 0), (0.8, 2), (1e-12, 0)]:
                try:
                    ell, sk, hits = ref.query(pat, K, top_t)
                    res.append({"pat": pat.decode(), "K": K, "top_t": top_t, "ell": ell,
                                "skipped": sk, "hits": hits})
                except O.OracleError as e:
                    res.append({"pat": pat.decode(), "K": K, "top_t": top_t, "error": e.code,
                                "msg": e.msg})
        out["results"][name] = res
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
