/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see cobs_oracle.h).
 *
 * Plain-C restatement of the reference's query and construction path.  Each
 * function cites the reference file:line it restates (paths relative to
 * /root/reference).  Parity is pinned against the reference's golden vectors
 * and against the reference itself (oracle/_ref), see tests/.
 */
#define _GNU_SOURCE
#include "cobs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_1905_09624_b200/csrc/synth.h"

#define SET_ERR(...)                                 \
    do {                                             \
        if (err && errlen) snprintf(err, errlen, __VA_ARGS__); \
    } while (0)

void orc_free(void* p) { free(p); }

/* ---- XXH64: proj/include/cobs/xxhash64.hpp:17-95 ----------------------- */

#define P1 0x9E3779B185EBCA87ULL
#define P2 0xC2B2AE3D27D4EB4FULL
#define P3 0x165667B19E3779F9ULL
#define P4 0x85EBCA77C2B2AE63ULL
#define P5 0x27D4EB2F165667C5ULL

static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static uint64_t ld64(const uint8_t* p) { /* xxhash64.hpp:23-28, little endian */
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}
static uint32_t ld32(const uint8_t* p) { /* xxhash64.hpp:30-33 */
    return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
static uint64_t xround(uint64_t acc, uint64_t lane) { /* :35-37 */
    return rotl64(acc + lane * P2, 31) * P1;
}
static uint64_t xmerge(uint64_t acc, uint64_t lane) { /* :39-41 */
    return (acc ^ xround(0, lane)) * P1 + P4;
}

uint64_t orc_xxh64(const void* data, size_t len, uint64_t seed) { /* :45-95 */
    const uint8_t* p = (const uint8_t*)data;
    const uint8_t* end = p + len;
    uint64_t acc;
    if (len >= 32) {
        uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        do {
            v1 = xround(v1, ld64(p));
            v2 = xround(v2, ld64(p + 8));
            v3 = xround(v3, ld64(p + 16));
            v4 = xround(v4, ld64(p + 24));
            p += 32;
        } while (p + 32 <= end);
        acc = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        acc = xmerge(acc, v1);
        acc = xmerge(acc, v2);
        acc = xmerge(acc, v3);
        acc = xmerge(acc, v4);
    } else {
        acc = seed + P5;
    }
    acc += (uint64_t)len;
    while (p + 8 <= end) {
        acc ^= xround(0, ld64(p));
        acc = rotl64(acc, 27) * P1 + P4;
        p += 8;
    }
    if (p + 4 <= end) {
        acc ^= (uint64_t)ld32(p) * P1;
        acc = rotl64(acc, 23) * P2 + P3;
        p += 4;
    }
    while (p < end) {
        acc ^= (uint64_t)(*p++) * P5;
        acc = rotl64(acc, 11) * P1;
    }
    acc ^= acc >> 33;
    acc *= P2;
    acc ^= acc >> 29;
    acc *= P3;
    acc ^= acc >> 32;
    return acc;
}

/* ---- bloom math: proj/src/bloom.cpp ------------------------------------ */

double orc_fpr_approx(uint64_t w, uint32_t k, uint64_t v) { /* bloom.cpp:42-48 */
    if (v == 0) return 0.0;
    double a = -(double)k * (double)v / (double)w;
    double miss = -expm1(a);
    return exp((double)k * log(miss));
}

int orc_size_filter(uint64_t v, double p, uint32_t k, uint64_t* out) { /* bloom.cpp:50-66 */
    if (!(p > 0.0 && p < 1.0)) return 1;
    if (k < 1) return 1;
    if (v == 0) {
        *out = 1;
        return 0;
    }
    double root = pow(p, 1.0 / (double)k);
    if (root >= 1.0) return 1;
    double denom = -log1p(-root);
    uint64_t w = (uint64_t)ceil((double)k * (double)v / denom);
    if (w < 1) w = 1;
    while (w > 1 && orc_fpr_approx(w - 1, k, v) <= p) --w;
    while (orc_fpr_approx(w, k, v) > p) ++w;
    *out = w;
    return 0;
}

uint64_t orc_score_threshold(uint64_t ell, double K) { /* bloom.cpp:120-123 */
    uint64_t t = (uint64_t)ceil(K * (double)ell - 1e-9);
    return t < 1 ? 1 : t;
}

/* ---- termizer: proj/src/termizer.cpp:18-30,92-129 ---------------------- */

static char complement(uint8_t c) { /* termizer.cpp:18-26 */
    switch (c) {
    case 'A': return 'T';
    case 'C': return 'G';
    case 'G': return 'C';
    case 'T': return 'A';
    default: return 0;
    }
}

static int cmp_q(const void* a, const void* b, void* q) {
    return memcmp(a, b, *(const uint32_t*)q);
}

int orc_extract_terms(const uint8_t* const* segs, const uint64_t* lens, size_t nseg, uint32_t q,
                      int canonical, uint8_t** terms_out, uint64_t* ell, uint64_t* skipped_out,
                      uint64_t* occ_out) {
    if (q < 1) return 1; /* termizer.cpp:105 */
    uint64_t cap = 0;
    for (size_t s = 0; s < nseg; ++s)
        if (lens[s] >= q) cap += lens[s] - q + 1;
    uint8_t* terms = (uint8_t*)malloc(cap * q + 1);
    uint64_t n = 0, skipped = 0, occ = 0;
    for (size_t s = 0; s < nseg; ++s) { /* termizer.cpp:108-125 */
        const uint8_t* t = segs[s];
        if (lens[s] < q) continue;
        for (uint64_t i = 0; i + q <= lens[s]; ++i) {
            const uint8_t* gram = t + i;
            uint8_t* dst = terms + n * q;
            if (canonical) {
                int ok = 1;
                for (uint32_t j = 0; j < q; ++j)
                    if (!complement(gram[j])) { ok = 0; break; }
                if (!ok) { ++skipped; continue; } /* :113-116 */
                for (uint32_t j = 0; j < q; ++j) dst[j] = (uint8_t)complement(gram[q - 1 - j]);
                if (!(memcmp(dst, gram, q) < 0)) memcpy(dst, gram, q); /* :117-119 */
            } else {
                memcpy(dst, gram, q);
            }
            ++n;
            ++occ;
        }
    }
    /* sort + unique: termizer.cpp:126-127 (bytewise, as std::string <) */
    uint32_t qq = q;
    if (n > 1) qsort_r(terms, n, q, cmp_q, &qq);
    uint64_t u = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (u == 0 || memcmp(terms + (u - 1) * q, terms + i * q, q) != 0) {
            if (u != i) memmove(terms + u * q, terms + i * q, q);
            ++u;
        }
    *terms_out = terms;
    *ell = u;
    if (skipped_out) *skipped_out = skipped;
    if (occ_out) *occ_out = occ;
    return 0;
}

/* ---- file parse: proj/src/storage.cpp:182-280 --------------------------- */

typedef struct cursor {
    const uint8_t* img;
    uint64_t size, pos;
} cursor;

static int cur_read(cursor* c, void* dst, uint64_t n) { /* storage.cpp:118-131 */
    if (n > c->size - c->pos) return -1;
    memcpy(dst, c->img + c->pos, n);
    c->pos += n;
    return 0;
}
static uint64_t rd_le(const uint8_t* b, int n) {
    uint64_t v = 0;
    for (int i = n - 1; i >= 0; --i) v = (v << 8) | b[i];
    return v;
}

#define TRUNC(c)                                                                 \
    do {                                                                         \
        SET_ERR("index file %s is truncated", path);                             \
        goto fail;                                                               \
    } while (0)
#define BAD(...)                                                                 \
    do {                                                                         \
        char what_[512];                                                         \
        snprintf(what_, sizeof what_, __VA_ARGS__);                              \
        SET_ERR("index file %s: %s", path, what_);                              \
        goto fail;                                                               \
    } while (0)

static int cmp_name_idx(const void* a, const void* b, void* ctx) {
    const orc_index* x = (const orc_index*)ctx;
    uint64_t i = *(const uint64_t*)a, j = *(const uint64_t*)b;
    uint16_t li = x->name_len[i], lj = x->name_len[j];
    int c = memcmp(x->names[i], x->names[j], li < lj ? li : lj);
    if (c) return c;
    return li < lj ? -1 : li > lj;
}

/* Sorted global indices by name (bytewise, std::string order). */
static uint64_t* name_order(const orc_index* x) {
    uint64_t* ord = (uint64_t*)malloc(sizeof(uint64_t) * (x->num_docs + 1));
    for (uint64_t i = 0; i < x->num_docs; ++i) ord[i] = i;
    qsort_r(ord, x->num_docs, sizeof(uint64_t), cmp_name_idx, (void*)x);
    return ord;
}

static int names_equal(const orc_index* x, uint64_t i, uint64_t j) {
    return x->name_len[i] == x->name_len[j] &&
           memcmp(x->names[i], x->names[j], x->name_len[i]) == 0;
}

int orc_parse(const uint8_t* img, uint64_t len, const char* path, orc_index* out, char* err,
              size_t errlen) {
    memset(out, 0, sizeof *out);
    cursor c = {img, len, 0};
    uint8_t b[8];
    out->file_size = len;
    if (len < 52) BAD("too small to be an index file");             /* :185 */
    cur_read(&c, b, 8);
    if (memcmp(b, "COBSIDX1", 8) != 0) BAD("bad magic");             /* :190 */
    cur_read(&c, b, 1);
    if (b[0] != 1) BAD("unsupported format version %u", b[0]);      /* :192-193 */
    cur_read(&c, b, 1);
    out->kind = b[0];
    if (out->kind != 0 && out->kind != 1) BAD("unknown index kind %u", b[0]);
    cur_read(&c, b, 1);
    out->params.hash_scheme = b[0];
    if (b[0] != 0) BAD("unknown hash scheme %u", b[0]);
    cur_read(&c, b, 1);
    if (b[0] > 1) BAD("bad canonical flag");
    out->params.canonical = b[0];
    cur_read(&c, b, 4);
    out->params.q = (uint32_t)rd_le(b, 4);
    cur_read(&c, b, 4);
    out->params.k = (uint32_t)rd_le(b, 4);
    cur_read(&c, b, 8);
    {
        uint64_t bits = rd_le(b, 8);
        memcpy(&out->params.p, &bits, 8);
    }
    cur_read(&c, b, 8);
    out->params.block_size = rd_le(b, 8);
    cur_read(&c, b, 8);
    uint64_t nb = rd_le(b, 8);
    cur_read(&c, b, 8);
    uint64_t nd = rd_le(b, 8);
    if (out->params.q < 1 || out->params.k < 1) BAD("bad q/k parameters");       /* :209 */
    if (!(out->params.p > 0.0 && out->params.p < 1.0)) BAD("target FPR out of range");
    if (out->params.block_size < 1) BAD("bad block size");
    if (nb < 1) BAD("no blocks");
    if (out->kind == 0 && nb != 1) BAD("classic index must have exactly one block");
    if (nb > len / 17) BAD("block count exceeds file size");                     /* :218 */
    out->num_blocks = nb;
    out->blocks = (orc_block*)calloc(nb, sizeof(orc_block));
    /* document tables: :220-238.  Grow the per-document arrays as we go. */
    uint64_t cap = 16, seen = 0;
    out->names = (const uint8_t**)malloc(cap * sizeof(void*));
    out->name_len = (uint16_t*)malloc(cap * sizeof(uint16_t));
    out->term_count = (uint64_t*)malloc(cap * sizeof(uint64_t));
    for (uint64_t bi = 0; bi < nb; ++bi) {
        orc_block* B = &out->blocks[bi];
        if (cur_read(&c, b, 8)) TRUNC(c);
        B->doc_count = rd_le(b, 8);
        if (cur_read(&c, b, 8)) TRUNC(c);
        B->w = rd_le(b, 8);
        if (B->doc_count < 1) BAD("empty block");
        if (B->w < 1) BAD("zero block width");
        if (B->doc_count > (c.size - c.pos) / 10) BAD("document table exceeds file size");
        B->row_bytes = (B->doc_count + 7) / 8;
        B->doc_base = seen;
        for (uint64_t i = 0; i < B->doc_count; ++i) {
            if (seen == cap) {
                cap *= 2;
                out->names = (const uint8_t**)realloc(out->names, cap * sizeof(void*));
                out->name_len = (uint16_t*)realloc(out->name_len, cap * sizeof(uint16_t));
                out->term_count = (uint64_t*)realloc(out->term_count, cap * sizeof(uint64_t));
            }
            if (cur_read(&c, b, 2)) TRUNC(c);
            uint16_t nl = (uint16_t)rd_le(b, 2);
            if (nl > c.size - c.pos) TRUNC(c);
            out->names[seen] = img + c.pos;
            out->name_len[seen] = nl;
            c.pos += nl;
            if (cur_read(&c, b, 8)) TRUNC(c);
            out->term_count[seen] = rd_le(b, 8);
            ++seen;
        }
    }
    out->num_docs = seen;
    if (seen != nd) BAD("document count mismatch");                              /* :238 */
    for (uint64_t bi = 0; bi < nb; ++bi) {                                        /* :240-250 */
        if (cur_read(&c, b, 8)) TRUNC(c);
        out->blocks[bi].offset = rd_le(b, 8);
    }
    out->payload_start = c.pos;
    uint64_t expected = c.pos;
    for (uint64_t bi = 0; bi < nb; ++bi) {
        const orc_block* B = &out->blocks[bi];
        uint64_t pb = B->w * B->row_bytes; /* wraps like the reference's u64 */
        if (B->offset != expected) BAD("payload offsets not contiguous");
        if (pb > len - expected) BAD("payload exceeds file size");
        expected += pb;
    }
    if (expected != len) BAD("trailing bytes after payload");
    if (out->kind == 1) { /* :253-265 */
        uint64_t pw = 0, ptc = 0, g = 0;
        for (uint64_t bi = 0; bi < nb; ++bi) {
            if (out->blocks[bi].w < pw) BAD("block widths decrease");
            pw = out->blocks[bi].w;
            for (uint64_t i = 0; i < out->blocks[bi].doc_count; ++i, ++g) {
                if (out->term_count[g] < ptc) BAD("document term counts not sorted");
                ptc = out->term_count[g];
            }
        }
    }
    { /* :267-277 */
        uint64_t* ord = name_order(out);
        for (uint64_t i = 1; i < seen; ++i)
            if (names_equal(out, ord[i - 1], ord[i])) {
                char nm[300];
                uint16_t l = out->name_len[ord[i]];
                if (l > 255) l = 255;
                memcpy(nm, out->names[ord[i]], l);
                nm[l] = 0;
                free(ord);
                BAD("duplicate document name %s", nm);
            }
        free(ord);
    }
    out->payload = img + out->payload_start;
    return 0;
fail:
    orc_index_free(out);
    return 2;
}

void orc_index_free(orc_index* x) {
    free(x->blocks);
    free((void*)x->names);
    free(x->name_len);
    free(x->term_count);
    free(x->name_pool);
    free(x->c5_thr16);
    memset(x, 0, sizeof *x);
}

/* ---- row access: ResidentView::row_data (storage.cpp:309-314) or the
 *      config-5 procedural rows ---------------------------------------- */

static const uint8_t* row_data(const orc_index* x, uint64_t b, uint64_t r, uint8_t* scratch) {
    const orc_block* B = &x->blocks[b];
    if (x->payload)
        return x->payload + (B->offset - x->payload_start) + r * B->row_bytes;
    for (uint64_t j = 0; j < B->row_bytes; ++j)
        scratch[j] = syn_c5_byte(x->c5_seed, b, r, j, x->c5_thr16[b], B->doc_count);
    return scratch;
}

/* ---- query: proj/src/query.cpp:49-164 ---------------------------------- */

typedef struct hit_sort_ctx {
    const orc_index* x;
    const orc_hit* hits;
} hit_sort_ctx;

static int cmp_hit(const void* a, const void* b, void* ctx) { /* query.cpp:156-160 */
    const orc_index* x = (const orc_index*)ctx;
    const orc_hit* h1 = (const orc_hit*)a;
    const orc_hit* h2 = (const orc_hit*)b;
    if (h1->score != h2->score) return h1->score > h2->score ? -1 : 1;
    uint64_t i = h1->doc, j = h2->doc;
    return cmp_name_idx(&i, &j, (void*)x);
}

int orc_query(const orc_index* x, const uint8_t* pat, uint64_t len, double K, uint64_t top_t,
              uint32_t* scores, uint64_t* ell_out, uint64_t* skipped_out, orc_hit** hits_out,
              uint64_t* n_hits, char* err, size_t errlen) {
    if (hits_out) *hits_out = NULL;
    if (n_hits) *n_hits = 0;
    if (!(K > 0.0 && K <= 1.0)) { /* query.cpp:125-126 */
        SET_ERR("query: K must be in (0,1]");
        return 1;
    }
    uint32_t q = x->params.q, k = x->params.k;
    uint8_t* terms;
    uint64_t ell, skipped;
    const uint8_t* segs[1] = {pat};
    uint64_t lens[1] = {len};
    orc_extract_terms(segs, lens, 1, q, x->params.canonical, &terms, &ell, &skipped, NULL);
    if (ell_out) *ell_out = ell;
    if (skipped_out) *skipped_out = skipped;
    if (ell == 0) { /* query.cpp:133-138 */
        free(terms);
        if (skipped > 0)
            SET_ERR("query: all %llu pattern grams were skipped by canonicalization",
                    (unsigned long long)skipped);
        else
            SET_ERR("query: pattern shorter than q = %u", q);
        return 2;
    }
    uint64_t* h = (uint64_t*)malloc(sizeof(uint64_t) * ell * k); /* :141-144 */
    for (uint64_t t = 0; t < ell; ++t)
        for (uint32_t s = 0; s < k; ++s) h[t * k + s] = orc_xxh64(terms + t * q, q, s);
    free(terms);
    uint64_t tau = orc_score_threshold(ell, K); /* :146 */
    uint64_t nh = 0, hcap = 0;
    orc_hit* hits = NULL;
    for (uint64_t bi = 0; bi < x->num_blocks; ++bi) { /* :149-154 -> score_range :49-89 */
        const orc_block* B = &x->blocks[bi];
        uint64_t rb = B->row_bytes, w = B->w;
        uint32_t* cnt = (uint32_t*)calloc(rb * 8, sizeof(uint32_t));
        uint8_t* acc = (uint8_t*)malloc(rb);
        uint8_t* scratch = (uint8_t*)malloc(rb);
        for (uint64_t t = 0; t < ell; ++t) {
            const uint8_t* src = row_data(x, bi, h[t * k] % w, scratch);
            memcpy(acc, src, rb);
            for (uint32_t s = 1; s < k; ++s) { /* :65-73 */
                const uint8_t* r = row_data(x, bi, h[t * k + s] % w, scratch);
                for (uint64_t j = 0; j < rb; ++j) acc[j] &= r[j];
            }
            for (uint64_t j = 0; j < rb; ++j) /* :74-81 */
                if (acc[j])
                    for (int i = 0; i < 8; ++i) cnt[j * 8 + i] += (acc[j] >> i) & 1u;
        }
        for (uint64_t d = 0; d < B->doc_count; ++d) { /* :83-88 (d < dc) */
            if (scores) scores[B->doc_base + d] = cnt[d];
            if (cnt[d] >= tau) {
                if (nh == hcap) {
                    hcap = hcap ? 2 * hcap : 64;
                    hits = (orc_hit*)realloc(hits, hcap * sizeof(orc_hit));
                }
                hits[nh].doc = B->doc_base + d;
                hits[nh].score = cnt[d];
                ++nh;
            }
        }
        free(cnt);
        free(acc);
        free(scratch);
    }
    free(h);
    if (nh > 1) qsort_r(hits, nh, sizeof(orc_hit), cmp_hit, (void*)x); /* :156-160 */
    if (top_t > 0 && nh > top_t) nh = top_t;                            /* :161-162 */
    if (n_hits) *n_hits = nh;
    if (hits_out)
        *hits_out = hits;
    else
        free(hits);
    return 0;
}

typedef struct batch_ctx {
    const orc_index* x;
    const uint8_t* pats;
    const uint64_t* off;
    size_t n;
    double K;
    uint32_t* scores;
    uint64_t *ell, *skipped, *n_hits;
    int* status;
    size_t next;
    pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
    batch_ctx* c = (batch_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        size_t i = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (i >= c->n) break;
        uint64_t nh = 0;
        c->status[i] = orc_query(c->x, c->pats + c->off[i], c->off[i + 1] - c->off[i], c->K, 0,
                                 c->scores ? c->scores + i * c->x->num_docs : NULL, &c->ell[i],
                                 &c->skipped[i], NULL, &nh, NULL, 0);
        if (c->n_hits) c->n_hits[i] = nh;
    }
    return NULL;
}

int orc_query_batch(const orc_index* x, const uint8_t* pats, const uint64_t* offsets, size_t n,
                    double K, uint32_t* scores, uint64_t* ell, uint64_t* skipped, int* status,
                    uint64_t* n_hits, int threads) {
    batch_ctx c = {x, pats, offsets, n, K, scores, ell, skipped, n_hits, status, 0,
                   PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &c);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return 0;
}

/* ---- build + write ------------------------------------------------------ */

typedef struct bdoc {
    const char* name;
    uint64_t name_len;
    uint8_t* terms;
    uint64_t ell;
} bdoc;

static int cmp_bdoc_name(const bdoc* a, const bdoc* b) {
    uint64_t l = a->name_len < b->name_len ? a->name_len : b->name_len;
    int c = memcmp(a->name, b->name, l);
    if (c) return c;
    return a->name_len < b->name_len ? -1 : a->name_len > b->name_len;
}
static int cmp_bdoc_ptr_name(const void* a, const void* b) {
    return cmp_bdoc_name(*(const bdoc* const*)a, *(const bdoc* const*)b);
}
static int cmp_bdoc_ptr_tc(const void* a, const void* b) { /* compact_index.cpp:27-30 */
    const bdoc* x = *(const bdoc* const*)a;
    const bdoc* y = *(const bdoc* const*)b;
    if (x->ell != y->ell) return x->ell < y->ell ? -1 : 1;
    return cmp_bdoc_name(x, y);
}

typedef struct bbuf {
    uint8_t* p;
    uint64_t n, cap;
} bbuf;
static void put(bbuf* b, const void* src, uint64_t n) {
    if (b->n + n > b->cap) {
        while (b->n + n > b->cap) b->cap = b->cap ? 2 * b->cap : 4096;
        b->p = (uint8_t*)realloc(b->p, b->cap);
    }
    memcpy(b->p + b->n, src, n);
    b->n += n;
}
static void put_le(bbuf* b, uint64_t v, int n) { /* storage.cpp:28-43 */
    uint8_t t[8];
    for (int i = 0; i < n; ++i) t[i] = (uint8_t)(v >> (8 * i));
    put(b, t, (uint64_t)n);
}

int orc_build_image(const uint8_t* const* segs, const uint64_t* lens, const uint64_t* doc_seg,
                    const char* const* names, size_t n_docs, const orc_params* P, int kind,
                    uint64_t forced_w, uint8_t** img, uint64_t* img_len, char* err,
                    size_t errlen) {
    /* params.hpp:26-35 */
    if (P->q < 1 || P->k < 1 || !(P->p > 0.0 && P->p < 1.0) || P->block_size < 1 ||
        P->hash_scheme != 0) {
        SET_ERR("params: invalid");
        return 1;
    }
    if (n_docs == 0) { /* classic_index.cpp:44 / compact_index.cpp:22 */
        SET_ERR("build: no documents");
        return 2;
    }
    bdoc* docs = (bdoc*)calloc(n_docs, sizeof(bdoc));
    for (size_t d = 0; d < n_docs; ++d) { /* extract_terms per document */
        docs[d].name = names[d];
        docs[d].name_len = strlen(names[d]);
        orc_extract_terms(segs + doc_seg[d], lens + doc_seg[d], doc_seg[d + 1] - doc_seg[d], P->q,
                          P->canonical, &docs[d].terms, &docs[d].ell, NULL, NULL);
    }
    bdoc** order = (bdoc**)malloc(n_docs * sizeof(bdoc*));
    for (size_t d = 0; d < n_docs; ++d) order[d] = &docs[d];
    int rc = 0;
    { /* duplicate names: classic_index.cpp:17-22, compact_index.cpp:33-40 */
        bdoc** byname = (bdoc**)malloc(n_docs * sizeof(bdoc*));
        memcpy(byname, order, n_docs * sizeof(bdoc*));
        qsort(byname, n_docs, sizeof(bdoc*), cmp_bdoc_ptr_name);
        for (size_t i = 1; i < n_docs; ++i)
            if (cmp_bdoc_name(byname[i - 1], byname[i]) == 0) {
                SET_ERR("duplicate document name: %s", byname[i]->name);
                rc = 2;
                break;
            }
        free(byname);
    }
    uint64_t nb = 1, B = n_docs;
    if (rc == 0 && kind == 1) {
        qsort(order, n_docs, sizeof(bdoc*), cmp_bdoc_ptr_tc);
        B = P->block_size;
        nb = (n_docs + B - 1) / B; /* compact_index.cpp:41-42 */
    }
    uint64_t* widths = (uint64_t*)calloc(nb, sizeof(uint64_t));
    for (uint64_t b = 0; rc == 0 && b < nb; ++b) { /* classic_index.cpp:48-61 per block */
        uint64_t lo = b * B, hi = lo + B < n_docs ? lo + B : n_docs, mx = 0;
        for (uint64_t i = lo; i < hi; ++i)
            if (order[i]->ell > mx) mx = order[i]->ell;
        if (kind == 0 && forced_w)
            widths[b] = forced_w;
        else if (orc_size_filter(mx, P->p, P->k, &widths[b])) {
            SET_ERR("bloom: bad sizing arguments");
            rc = 1;
        }
    }
    if (rc) {
        for (size_t d = 0; d < n_docs; ++d) free(docs[d].terms);
        free(docs);
        free(order);
        free(widths);
        return rc;
    }
    /* header: storage.cpp:345-380 */
    bbuf out = {0, 0, 0};
    put(&out, "COBSIDX1", 8);
    put_le(&out, 1, 1);
    put_le(&out, (uint64_t)kind, 1);
    put_le(&out, P->hash_scheme, 1);
    put_le(&out, P->canonical ? 1 : 0, 1);
    put_le(&out, P->q, 4);
    put_le(&out, P->k, 4);
    {
        uint64_t bits;
        memcpy(&bits, &P->p, 8);
        put_le(&out, bits, 8);
    }
    put_le(&out, P->block_size, 8);
    put_le(&out, nb, 8);
    put_le(&out, n_docs, 8);
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = b * B, hi = lo + B < n_docs ? lo + B : n_docs;
        put_le(&out, hi - lo, 8);
        put_le(&out, widths[b], 8);
        for (uint64_t i = lo; i < hi; ++i) {
            if (order[i]->name_len > 65535) { /* storage.cpp:368-369 */
                SET_ERR("document name too long to store: %s", order[i]->name);
                rc = 2;
            }
            put_le(&out, order[i]->name_len, 2);
            put(&out, order[i]->name, order[i]->name_len);
            put_le(&out, order[i]->ell, 8);
        }
    }
    uint64_t off = out.n + 8 * nb; /* storage.cpp:376-380 */
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = b * B, hi = lo + B < n_docs ? lo + B : n_docs;
        put_le(&out, off, 8);
        off += widths[b] * ((hi - lo + 7) / 8);
    }
    /* payload: fill_columns (classic_index.cpp:26-36) per block, rows in order */
    for (uint64_t b = 0; rc == 0 && b < nb; ++b) {
        uint64_t lo = b * B, hi = lo + B < n_docs ? lo + B : n_docs;
        uint64_t rb = (hi - lo + 7) / 8, w = widths[b];
        uint8_t* m = (uint8_t*)calloc(w * rb, 1);
        for (uint64_t c = lo; c < hi; ++c)
            for (uint64_t t = 0; t < order[c]->ell; ++t)
                for (uint32_t s = 0; s < P->k; ++s) {
                    uint64_t r = orc_xxh64(order[c]->terms + t * P->q, P->q, s) % w;
                    m[r * rb + (c - lo) / 8] |= (uint8_t)(1u << ((c - lo) % 8)); /* bit_matrix.hpp:25-27 */
                }
        put(&out, m, w * rb);
        free(m);
    }
    for (size_t d = 0; d < n_docs; ++d) free(docs[d].terms);
    free(docs);
    free(order);
    free(widths);
    if (rc) {
        free(out.p);
        return rc;
    }
    *img = out.p;
    *img_len = out.n;
    return 0;
}

/* ---- config 5 ----------------------------------------------------------- */

typedef struct c5doc {
    uint64_t tc, id;
} c5doc;
static int cmp_c5(const void* a, const void* b) { /* (term_count, name) with zero-padded names */
    const c5doc* x = (const c5doc*)a;
    const c5doc* y = (const c5doc*)b;
    if (x->tc != y->tc) return x->tc < y->tc ? -1 : 1;
    char nx[24], ny[24];
    int lx = syn_c5_name(x->id, nx), ly = syn_c5_name(y->id, ny);
    int c = memcmp(nx, ny, (size_t)(lx < ly ? lx : ly));
    if (c) return c;
    return lx < ly ? -1 : lx > ly;
}

int orc_c5_make(uint64_t seed, uint64_t n, uint64_t B, double median, double sigma, double p,
                orc_index* x) {
    memset(x, 0, sizeof *x);
    uint64_t* tc = (uint64_t*)malloc(n * sizeof(uint64_t));
    syn_c5_term_counts(seed, n, median, sigma, tc);
    c5doc* d = (c5doc*)malloc(n * sizeof(c5doc));
    for (uint64_t i = 0; i < n; ++i) d[i].tc = tc[i], d[i].id = i;
    free(tc);
    qsort(d, n, sizeof(c5doc), cmp_c5);
    uint64_t nb = (n + B - 1) / B;
    x->params.q = 31;
    x->params.k = 1;
    x->params.p = p;
    x->params.canonical = 0;
    x->params.block_size = B;
    x->kind = 1;
    x->num_blocks = nb;
    x->num_docs = n;
    x->blocks = (orc_block*)calloc(nb, sizeof(orc_block));
    x->c5_thr16 = (uint32_t*)calloc(nb, sizeof(uint32_t));
    x->names = (const uint8_t**)malloc(n * sizeof(void*));
    x->name_len = (uint16_t*)malloc(n * sizeof(uint16_t));
    x->term_count = (uint64_t*)malloc(n * sizeof(uint64_t));
    x->name_pool = (char*)malloc(n * 24);
    x->c5_seed = seed;
    for (uint64_t i = 0; i < n; ++i) {
        char* nm = x->name_pool + i * 24;
        x->name_len[i] = (uint16_t)syn_c5_name(d[i].id, nm);
        x->names[i] = (const uint8_t*)nm;
        x->term_count[i] = d[i].tc;
    }
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = b * B, hi = lo + B < n ? lo + B : n, mx = 0;
        for (uint64_t i = lo; i < hi; ++i)
            if (d[i].tc > mx) mx = d[i].tc;
        x->blocks[b].doc_count = hi - lo;
        x->blocks[b].row_bytes = (hi - lo + 7) / 8;
        x->blocks[b].doc_base = lo;
        orc_size_filter(mx, p, 1, &x->blocks[b].w);
        x->c5_thr16[b] = syn_c5_thr16(x->blocks[b].w, mx);
    }
    free(d);
    /* offsets as the writer would lay them out */
    uint64_t head = 52 + 8 * nb;
    for (uint64_t b = 0; b < nb; ++b) {
        head += 16;
        for (uint64_t i = 0; i < x->blocks[b].doc_count; ++i)
            head += 10 + x->name_len[x->blocks[b].doc_base + i];
    }
    x->payload_start = head;
    uint64_t off = head;
    for (uint64_t b = 0; b < nb; ++b) {
        x->blocks[b].offset = off;
        off += x->blocks[b].w * x->blocks[b].row_bytes;
    }
    x->file_size = off;
    return 0;
}

int orc_header_image(const orc_index* x, uint8_t** img, uint64_t* len) {
    bbuf out = {0, 0, 0};
    put(&out, "COBSIDX1", 8);
    put_le(&out, 1, 1);
    put_le(&out, x->kind, 1);
    put_le(&out, x->params.hash_scheme, 1);
    put_le(&out, x->params.canonical ? 1 : 0, 1);
    put_le(&out, x->params.q, 4);
    put_le(&out, x->params.k, 4);
    uint64_t bits;
    memcpy(&bits, &x->params.p, 8);
    put_le(&out, bits, 8);
    put_le(&out, x->params.block_size, 8);
    put_le(&out, x->num_blocks, 8);
    put_le(&out, x->num_docs, 8);
    for (uint64_t b = 0; b < x->num_blocks; ++b) {
        put_le(&out, x->blocks[b].doc_count, 8);
        put_le(&out, x->blocks[b].w, 8);
        for (uint64_t i = 0; i < x->blocks[b].doc_count; ++i) {
            uint64_t g = x->blocks[b].doc_base + i;
            put_le(&out, x->name_len[g], 2);
            put(&out, x->names[g], x->name_len[g]);
            put_le(&out, x->term_count[g], 8);
        }
    }
    uint64_t off = out.n + 8 * x->num_blocks;
    for (uint64_t b = 0; b < x->num_blocks; ++b) {
        put_le(&out, off, 8);
        off += x->blocks[b].w * x->blocks[b].row_bytes;
    }
    *img = out.p;
    *len = out.n;
    return 0;
}
