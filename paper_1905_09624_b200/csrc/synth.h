/* Seeded synthetic workloads for the five BASELINE.json configs.
 *
 * This is INPUT generation, not part of the COBS path: the product library
 * (device generators), the CPU oracle and the bench all include this one
 * header so every consumer sees the same documents, queries and procedural
 * (config-5) index bits.  Everything here is integer-only and counter based
 * (splitmix64 finaliser keyed by (seed, stream, index)), so the host and the
 * device produce identical bytes.  The only floating point (log-normal /
 * log-uniform document lengths, config-5 term counts) is host-only and is
 * computed once, then passed to whoever needs it.
 *
 * Plain C99 so oracle/ (gcc) can include it; compiles as CUDA host+device.
 */
#ifndef COBS_SYNTH_H
#define COBS_SYNTH_H

#include <stddef.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- counter-based RNG ------------------------------------------------ */

SYN_HD uint64_t syn_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Key of an independent stream: (seed, stream) -> 64-bit key. */
SYN_HD uint64_t syn_key(uint64_t seed, uint64_t stream) {
    return syn_mix64(syn_mix64(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}

/* i-th 64-bit draw of a stream. */
SYN_HD uint64_t syn_u64(uint64_t key, uint64_t i) {
    return syn_mix64(key ^ (i * 0xA0761D6478BD642FULL));
}

/* Stream ids. Documents use SYN_S_DOC + doc, queries SYN_S_QUERY + query. */
#define SYN_S_DOC 0x1000000000ULL
#define SYN_S_QUERY 0x2000000000ULL
#define SYN_S_LEN 0x3000000000ULL
#define SYN_S_C5BITS 0x4000000000ULL
#define SYN_S_C5TC 0x5000000000ULL

/* DNA letters, and the fixed 20-letter amino-acid alphabet of config 4
 * (pinned: the letters change the hashes). */
#define SYN_DNA_LETTERS "ACGT"
#define SYN_AA_LETTERS "ACDEFGHIKLMNPQRSTVWY"

/* Document alphabets. */
#define SYN_ALPHA_DNA 0
#define SYN_ALPHA_AA 1

/* Symbol index (0..3 DNA, 0..19 AA) of position i of document `doc`. */
SYN_HD uint32_t syn_doc_sym(uint64_t seed, int alpha, uint64_t doc, uint64_t i) {
    uint64_t key = syn_key(seed, SYN_S_DOC + doc);
    if (alpha == SYN_ALPHA_DNA) {
        uint64_t w = syn_u64(key, i >> 5);
        return (uint32_t)(w >> (2 * (i & 31))) & 3u;
    }
    uint64_t w = syn_u64(key, i >> 1);
    uint32_t half = (uint32_t)(w >> (32 * (i & 1)));
    return (uint32_t)(((uint64_t)half * 20u) >> 32);
}

SYN_HD char syn_sym_char(int alpha, uint32_t s) {
    return alpha == SYN_ALPHA_DNA ? SYN_DNA_LETTERS[s] : SYN_AA_LETTERS[s];
}

/* Bytes [lo, lo+n) of document `doc`. */
SYN_HD void syn_doc_bytes(uint64_t seed, int alpha, uint64_t doc, uint64_t lo, uint64_t n,
                          char* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = syn_sym_char(alpha, syn_doc_sym(seed, alpha, doc, lo + i));
}

/* ---- queries ----------------------------------------------------------- */

/* Query kinds. */
#define SYN_Q_RANDOM 0  /* uniform random symbols */
#define SYN_Q_SUBST 1   /* substring of a document + per-symbol substitutions */
#define SYN_Q_INDEL 2   /* substring + substitution/insertion/deletion edits (1/3 each) */

/* Description of a query batch (host-side). Half the queries (even ids when
 * mixed=1, i.e. ids 0,2,4,...) are drawn from documents; the rest random. */
typedef struct syn_query_spec {
    uint64_t seed;
    int alpha;
    uint64_t n_queries;
    uint64_t qlen;          /* output length of every query */
    int kind;               /* SYN_Q_SUBST or SYN_Q_INDEL for the drawn half */
    uint32_t edit_per_65536; /* per-symbol edit probability * 65536 */
    int mixed;              /* 1: half drawn, half random; 0: all random */
} syn_query_spec;

/* Generate query `j` into out[0..qlen). `doc_len` gives each document's length
 * (n_docs entries); drawn queries pick a document long enough. */
static inline void syn_query(const syn_query_spec* s, const uint64_t* doc_len, uint64_t n_docs,
                             uint64_t j, char* out) {
    uint64_t key = syn_key(s->seed, SYN_S_QUERY + j);
    uint64_t ctr = 0;
    uint32_t nsym = s->alpha == SYN_ALPHA_DNA ? 4u : 20u;
    int drawn = s->mixed && (j % 2 == 0);
    if (!drawn) {
        for (uint64_t i = 0; i < s->qlen; ++i) {
            uint64_t u = syn_u64(key, ctr++);
            out[i] = syn_sym_char(s->alpha, (uint32_t)(((u >> 32) * nsym) >> 32));
        }
        return;
    }
    /* pick a document whose length fits the query (with indel slack) */
    uint64_t need = s->kind == SYN_Q_INDEL ? s->qlen + s->qlen / 4 + 64 : s->qlen;
    uint64_t doc = 0;
    for (int tries = 0; tries < 1000; ++tries) {
        doc = syn_u64(key, ctr++) % n_docs;
        if (doc_len[doc] >= need) break;
    }
    uint64_t span = doc_len[doc] >= need ? doc_len[doc] - need + 1 : 1;
    uint64_t pos = syn_u64(key, ctr++) % span;
    uint64_t src = pos, i = 0;
    while (i < s->qlen) {
        uint64_t u = syn_u64(key, ctr++);
        uint32_t r16 = (uint32_t)(u & 0xFFFF);
        uint32_t op = (uint32_t)((u >> 16) % 3);   /* 0 sub, 1 ins, 2 del */
        uint32_t alt = (uint32_t)((u >> 32) % (nsym - 1)) + 1;
        uint32_t cur = src < doc_len[doc] ? syn_doc_sym(s->seed, s->alpha, doc, src) : 0;
        if (r16 < s->edit_per_65536) {
            if (s->kind == SYN_Q_SUBST || op == 0) {
                out[i++] = syn_sym_char(s->alpha, (cur + alt) % nsym);
                ++src;
            } else if (op == 1) {
                out[i++] = syn_sym_char(s->alpha, (uint32_t)((u >> 40) % nsym));
            } else {
                ++src;
            }
        } else {
            out[i++] = syn_sym_char(s->alpha, cur);
            ++src;
        }
    }
}

/* ---- config-5 procedural compact index --------------------------------- */

/* Bits of row r of block b: 16-bit uniforms against the block threshold
 * (density * 65536), four per 64-bit draw; padding columns (>= doc_count)
 * are zero. Byte j of the row covers columns 8j..8j+7 (LSB first). */
SYN_HD uint64_t syn_c5_key(uint64_t seed, uint64_t block) {
    return syn_key(seed, SYN_S_C5BITS + block);
}

SYN_HD uint8_t syn_c5_byte_k(uint64_t key, uint64_t row, uint64_t j, uint32_t thr16,
                             uint64_t doc_count) {
    uint64_t base = row * 0x100000000ULL + j * 2; /* two draws per byte */
    uint8_t out = 0;
    for (int h = 0; h < 2; ++h) {
        uint64_t u = syn_u64(key, base + (uint64_t)h);
        for (int t = 0; t < 4; ++t) {
            uint32_t v = (uint32_t)(u >> (16 * t)) & 0xFFFFu;
            uint64_t col = 8 * j + (uint64_t)(4 * h + t);
            if (v < thr16 && col < doc_count) out |= (uint8_t)(1u << (4 * h + t));
        }
    }
    return out;
}

SYN_HD uint8_t syn_c5_byte(uint64_t seed, uint64_t block, uint64_t row, uint64_t j,
                           uint32_t thr16, uint64_t doc_count) {
    return syn_c5_byte_k(syn_c5_key(seed, block), row, j, thr16, doc_count);
}

/* ---- host-only length / term-count distributions ----------------------- */
#include <math.h>

/* Uniform double in (0,1) from one draw. */
static inline double syn_unit(uint64_t u) {
    return ((double)(u >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* Standard normal (Box-Muller, cosine branch) from draws 2i, 2i+1. */
static inline double syn_normal(uint64_t key, uint64_t i) {
    double u1 = syn_unit(syn_u64(key, 2 * i));
    double u2 = syn_unit(syn_u64(key, 2 * i + 1));
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Document lengths.  dist 0: fixed `a`; 1: floor(exp(U(ln a, ln b)))
 * (log-uniform, config 2); 2: floor(exp(N(ln a, b))) (log-normal with
 * median a and sigma b, config 3).  Lengths are clamped to >= minlen. */
static inline void syn_doc_lengths(uint64_t seed, uint64_t n, int dist, double a, double b,
                                   uint64_t minlen, uint64_t* out) {
    uint64_t key = syn_key(seed, SYN_S_LEN);
    for (uint64_t i = 0; i < n; ++i) {
        double len;
        if (dist == 0)
            len = a;
        else if (dist == 1)
            len = floor(exp(log(a) + (log(b) - log(a)) * syn_unit(syn_u64(key, i))));
        else
            len = floor(exp(log(a) + b * syn_normal(key, i)));
        uint64_t l = (uint64_t)len;
        out[i] = l < minlen ? minlen : l;
    }
}

/* Config-5 per-document distinct term counts, log-normal (median, sigma),
 * in draw order (document i is named "doc%06llu" % i). */
static inline void syn_c5_term_counts(uint64_t seed, uint64_t n, double median, double sigma,
                                      uint64_t* out) {
    uint64_t key = syn_key(seed, SYN_S_C5TC);
    for (uint64_t i = 0; i < n; ++i) {
        double v = floor(exp(log(median) + sigma * syn_normal(key, i)));
        out[i] = v < 1.0 ? 1 : (uint64_t)v;
    }
}

/* Config-5 block fill density 1-(1-1/w)^n as a 16-bit threshold. */
static inline uint32_t syn_c5_thr16(uint64_t w, uint64_t n) {
    double density = -expm1((double)n * log1p(-1.0 / (double)w));
    double t = floor(density * 65536.0 + 0.5);
    return t >= 65536.0 ? 65536u : (uint32_t)t;
}

/* Config-5 document name of draw index i. */
static inline int syn_c5_name(uint64_t i, char* out /* >= 24 bytes */) {
    int n = 0;
    char digits[24];
    int nd = 0;
    do {
        digits[nd++] = (char)('0' + (int)(i % 10));
        i /= 10;
    } while (i);
    out[n++] = 'd'; out[n++] = 'o'; out[n++] = 'c';
    for (int z = nd; z < 6; ++z) out[n++] = '0';
    while (nd) out[n++] = digits[--nd];
    return n;
}

#ifdef __cplusplus
}
#endif

#endif /* COBS_SYNTH_H */
