/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see cobs_oracle.h).
 *
 * Full-size check of a built index image against the seeded synthetic
 * corpus it was built from (workloads/synth: BASELINE.json configs 2-4).
 * The configs' corpora (11-72 GB of sequence, 10-35 GB indexes) are far
 * beyond orc_build_image, which materialises every TermSet; this restates
 * the same build -- extract_terms (termizer.cpp:103-129) -> term_count,
 * build_classic / build_compact (classic_index.cpp:26-64,
 * compact_index.cpp:19-52) -> header (storage.cpp:345-380) and payload bits
 * (bit_matrix.hpp:25-27) -- one 64-document column group at a time, and
 * compares every payload byte and the whole header against the image.
 *
 *   * a unit is (block b, column group g): the <= 64 documents whose bits
 *     are byte columns [8g, 8g+8) of block b's rows.  The unit's documents
 *     are regenerated from the seed, every window's term is hashed with
 *     orc_xxh64 (the pinned XXH64) for every seed and `% w_b` sets bit
 *     (row, column) in a w_b x 64-bit slab, and the slab is compared with
 *     those 8 byte columns of the image, row by row;
 *   * the same pass counts each document's distinct terms exactly (its
 *     window keys -- the 2-bit DNA code, or 5-bit residue indices for the
 *     20-letter alphabet; injective for q <= 31 / q*5 <= 60 -- partitioned by
 *     a bijective mix and counted in small hash sets);
 *   * which documents form which block, and the block widths, are read from
 *     the image's header for the payload comparison; the header itself is
 *     then rebuilt from the oracle's own term counts (classic: input order;
 *     compact: (term_count, name) order in blocks of block_size; widths
 *     size_filter(block max)) and compared byte for byte, so a header that
 *     passes vouches for the layout the payload was compared under.
 *
 * Canonical mode (DNA only): the term is min(gram, revcomp(gram)) bytewise
 * (termizer.cpp:117-119); for A/C/G/T windows bytewise order equals 2-bit
 * code order, and the reverse-complement bytes are read from the
 * document's reverse complement.  Supported: DNA with q <= 31 (or q = 32
 * canonical), the 20-letter alphabet non-canonical with q <= 12 -- the
 * configs' shapes; anything else is refused (return 1).  Pinned against
 * orc_build_image on scaled configs by tests/test_oracle_stream.py.
 */
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cobs_oracle.h"
#include "../paper_1905_09624_b200/csrc/synth.h"

#define SET_ERR(...)                                  \
    do {                                              \
        if (err && errlen) snprintf(err, errlen, __VA_ARGS__); \
    } while (0)

typedef struct unit {
    uint64_t block, group, cost;
} unit;

typedef struct shared {
    const orc_stream_spec* s;
    const orc_index* x;      /* the image, parsed (pinned parser) */
    const uint8_t* img;
    const uint64_t* col_id;  /* file column -> draw index */
    unit* units;
    uint64_t n_units;
    uint64_t next;           /* atomic */
    uint64_t max_len, max_w;
    uint64_t* tc;            /* oracle term count by draw index */
    pthread_mutex_t mu;
    orc_stream_report rep;
    int fail;
    char msg[256];
} shared;

static uint64_t mix64(uint64_t z) { /* splitmix64 finaliser: a bijection */
    z ^= z >> 31;
    z *= 0x7FB5D329728EA185ULL;
    z ^= z >> 27;
    z *= 0x81DADEF4BC2DD44DULL;
    return z ^ (z >> 33);
}

static uint64_t pow2_at_least(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

/* Distinct keys of keys[0..n): a direct set for short lists, else a
 * partition by the top bits of mix64(key) (equal keys meet in one part)
 * into parts of ~16k keys, each counted in an L2-sized set. */
typedef struct counter {
    uint64_t *tmp, *tab;
    uint64_t tmp_cap, tab_cap;
    uint32_t* hist;
} counter;

static uint64_t count_set(counter* c, const uint64_t* k, uint64_t n) {
    if (!n) return 0;
    uint64_t S = pow2_at_least(2 * n);
    if (S > c->tab_cap) {
        free(c->tab);
        c->tab = (uint64_t*)malloc(S * sizeof(uint64_t));
        c->tab_cap = S;
    }
    memset(c->tab, 0xff, S * sizeof(uint64_t)); /* all ones = empty */
    uint64_t distinct = 0;
    int ones_seen = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t key = k[i];
        if (key == ~0ULL) { /* the empty marker itself: counted aside */
            distinct += !ones_seen;
            ones_seen = 1;
            continue;
        }
        uint64_t slot = mix64(key) & (S - 1);
        for (;;) {
            uint64_t cur = c->tab[slot];
            if (cur == ~0ULL) {
                c->tab[slot] = key;
                ++distinct;
                break;
            }
            if (cur == key) break;
            slot = (slot + 1) & (S - 1);
        }
    }
    return distinct;
}

static uint64_t count_distinct(counter* c, const uint64_t* k, uint64_t n) {
    if (n <= (1u << 15)) return count_set(c, k, n);
    uint32_t bits = 0;
    while ((1ULL << bits) < (n >> 14)) ++bits;
    const uint64_t nb = 1ULL << bits;
    if (n > c->tmp_cap) {
        free(c->tmp);
        c->tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
        c->tmp_cap = n;
    }
    c->hist = (uint32_t*)realloc(c->hist, (nb + 1) * sizeof(uint32_t));
    memset(c->hist, 0, (nb + 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) ++c->hist[(mix64(k[i]) >> (64 - bits)) + 1];
    for (uint64_t b = 0; b < nb; ++b) c->hist[b + 1] += c->hist[b];
    uint32_t* cur = (uint32_t*)malloc(nb * sizeof(uint32_t));
    memcpy(cur, c->hist, nb * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) c->tmp[cur[mix64(k[i]) >> (64 - bits)]++] = k[i];
    free(cur);
    uint64_t total = 0;
    for (uint64_t b = 0; b < nb; ++b) total += count_set(c, c->tmp + c->hist[b], c->hist[b + 1] - c->hist[b]);
    return total;
}

/* Document bytes of draw index `doc` (synth.h syn_doc_sym, one 64-bit draw
 * per 32 bases / 2 residues instead of one per symbol). */
static void gen_doc(uint64_t seed, int alpha, uint64_t doc, uint64_t len, uint8_t* out, uint8_t* sym) {
    const uint64_t key = syn_key(seed, SYN_S_DOC + doc);
    if (alpha == SYN_ALPHA_DNA) {
        for (uint64_t i = 0; i < len; i += 32) {
            uint64_t w = syn_u64(key, i >> 5);
            uint64_t e = len - i < 32 ? len - i : 32;
            for (uint64_t j = 0; j < e; ++j) {
                uint32_t s = (uint32_t)(w >> (2 * j)) & 3u;
                sym[i + j] = (uint8_t)s;
                out[i + j] = (uint8_t)SYN_DNA_LETTERS[s];
            }
        }
    } else {
        for (uint64_t i = 0; i < len; i += 2) {
            uint64_t w = syn_u64(key, i >> 1);
            for (uint64_t j = 0; j < 2 && i + j < len; ++j) {
                uint32_t half = (uint32_t)(w >> (32 * j));
                uint32_t s = (uint32_t)(((uint64_t)half * 20u) >> 32);
                sym[i + j] = (uint8_t)s;
                out[i + j] = (uint8_t)SYN_AA_LETTERS[s];
            }
        }
    }
}

static uint8_t comp(uint8_t c) { /* termizer.cpp:18-26 for A/C/G/T */
    switch (c) {
    case 'A': return 'T';
    case 'C': return 'G';
    case 'G': return 'C';
    default: return 'A';
    }
}

typedef struct worker {
    shared* sh;
    uint8_t *fwd, *rc, *sym;
    uint64_t* keys;
    uint64_t* slab;
    counter cnt;
} worker;

#define ROW_BATCH 64

static void* work(void* arg) {
    worker* W = (worker*)arg;
    shared* sh = W->sh;
    const orc_stream_spec* s = sh->s;
    const orc_index* x = sh->x;
    const uint32_t q = s->params.q, k = s->params.k;
    const int canon = s->params.canonical != 0;
    const int dna = s->alpha == SYN_ALPHA_DNA;
    const uint32_t sb = dna ? 2 : 5;
    const uint64_t mask = q * sb >= 64 ? ~0ULL : ((1ULL << (q * sb)) - 1);
    uint64_t rows[ROW_BATCH];
    uint64_t windows = 0;
    for (;;) {
        uint64_t u = __atomic_fetch_add(&sh->next, 1, __ATOMIC_RELAXED);
        if (u >= sh->n_units) break;
        const orc_block* B = &x->blocks[sh->units[u].block];
        const uint64_t g = sh->units[u].group, w = B->w, rb = B->row_bytes;
        const uint64_t c0 = 64 * g, c1 = c0 + 64 < B->doc_count ? c0 + 64 : B->doc_count;
        memset(W->slab, 0, w * sizeof(uint64_t));
        for (uint64_t c = c0; c < c1; ++c) {
            const uint64_t id = sh->col_id[B->doc_base + c];
            const uint64_t L = s->doc_len[id];
            gen_doc(s->seed, s->alpha, id, L, W->fwd, W->sym);
            if (canon)
                for (uint64_t i = 0; i < L; ++i) W->rc[i] = comp(W->fwd[L - 1 - i]);
            const uint64_t bit = 1ULL << (c - c0);
            uint64_t cf = 0, cr = 0, nk = 0, nrow = 0;
            const uint64_t nwin = L >= q ? L - q + 1 : 0;
            for (uint64_t i = 0; i + 1 < q && i < L; ++i) {
                cf = ((cf << sb) | W->sym[i]) & mask;
                if (canon) cr = (cr >> 2) | ((uint64_t)(3u - W->sym[i]) << (2 * (q - 1)));
            }
            for (uint64_t j = 0; j < nwin; ++j) {
                const uint8_t sy = W->sym[j + q - 1];
                cf = ((cf << sb) | sy) & mask;
                const uint8_t* term = W->fwd + j;
                uint64_t key = cf;
                if (canon) {
                    cr = (cr >> 2) | ((uint64_t)(3u - sy) << (2 * (q - 1)));
                    if (cr < cf) { /* revcomp strictly smaller (termizer.cpp:117-118) */
                        key = cr;
                        term = W->rc + (L - j - q);
                    }
                }
                W->keys[nk++] = key;
                for (uint32_t sd = 0; sd < k; ++sd) { /* classic_index.cpp:28-35 */
                    const uint64_t r = orc_xxh64(term, q, sd) % w;
                    __builtin_prefetch(W->slab + r, 1);
                    rows[nrow++] = r;
                    if (nrow == ROW_BATCH) {
                        for (uint64_t t = 0; t < nrow; ++t) W->slab[rows[t]] |= bit;
                        nrow = 0;
                    }
                }
            }
            for (uint64_t t = 0; t < nrow; ++t) W->slab[rows[t]] |= bit;
            windows += nwin;
            sh->tc[id] = count_distinct(&W->cnt, W->keys, nk); /* termizer.cpp:126-127 */
        }
        /* the unit's byte columns of the image vs the slab */
        const uint64_t nbytes = rb - 8 * g < 8 ? rb - 8 * g : 8;
        const uint8_t* base = sh->img + B->offset + 8 * g;
        uint64_t bad = 0, bad_row = 0, bad_byte = 0;
        for (uint64_t r = 0; r < w; ++r) {
            uint64_t got = 0;
            if (nbytes == 8)
                memcpy(&got, base + r * rb, 8);
            else
                memcpy(&got, base + r * rb, nbytes);
            const uint64_t want = W->slab[r];
            if (got != want) {
                for (uint64_t b = 0; b < nbytes; ++b)
                    if (((got ^ want) >> (8 * b)) & 0xff) {
                        if (!bad) bad_row = r, bad_byte = 8 * g + b;
                        ++bad;
                    }
            }
        }
        pthread_mutex_lock(&sh->mu);
        if (bad) {
            const uint64_t blk = sh->units[u].block;
            orc_stream_report* R = &sh->rep;
            if (!R->payload_bad_bytes || blk < R->bad_block ||
                (blk == R->bad_block && (bad_row < R->bad_row || (bad_row == R->bad_row && bad_byte < R->bad_byte)))) {
                R->bad_block = blk;
                R->bad_row = bad_row;
                R->bad_byte = bad_byte;
            }
            R->payload_bad_bytes += bad;
        }
        pthread_mutex_unlock(&sh->mu);
    }
    __atomic_fetch_add(&sh->rep.windows, windows, __ATOMIC_RELAXED);
    return NULL;
}

static int cmp_unit(const void* a, const void* b) { /* costliest first */
    const unit* x = (const unit*)a;
    const unit* y = (const unit*)b;
    return x->cost > y->cost ? -1 : x->cost < y->cost;
}

typedef struct ord {
    uint64_t tc, id;
} ord;
static int cmp_ord(const void* a, const void* b) { /* compact_index.cpp:27-30; names zero-padded */
    const ord* x = (const ord*)a;
    const ord* y = (const ord*)b;
    if (x->tc != y->tc) return x->tc < y->tc ? -1 : 1;
    return x->id < y->id ? -1 : x->id > y->id; /* equal width => numeric order == bytewise order */
}

static int doc_name(uint64_t id, uint32_t width, char* out) {
    return sprintf(out, "doc%0*llu", (int)width, (unsigned long long)id);
}

int orc_stream_check(const orc_stream_spec* s, const uint8_t* img, uint64_t img_len, int threads,
                     orc_stream_report* rep, uint64_t* term_counts, char* err, size_t errlen) {
    memset(rep, 0, sizeof *rep);
    const uint32_t q = s->params.q;
    if (!((s->alpha == SYN_ALPHA_DNA && (q <= 31 || (q == 32 && s->params.canonical))) ||
          (s->alpha == SYN_ALPHA_AA && !s->params.canonical && q <= 12)) ||
        q < 1 || s->params.k < 1 || s->n_docs == 0) {
        SET_ERR("stream check: unsupported shape (alpha %d, q %u, canonical %d)", s->alpha, q,
                s->params.canonical);
        return 1;
    }
    orc_index x;
    if (orc_parse(img, img_len, "<image>", &x, err, errlen)) return 2;
    int rc = 0;
    const uint64_t n = s->n_docs;
    uint32_t width = 4;
    {
        char t[32];
        int l = sprintf(t, "%llu", (unsigned long long)(n - 1));
        if ((uint32_t)l > width) width = (uint32_t)l;
    }
    shared sh;
    memset(&sh, 0, sizeof sh);
    sh.s = s;
    sh.x = &x;
    sh.img = img;
    pthread_mutex_init(&sh.mu, NULL);
    uint64_t* col_id = (uint64_t*)malloc((x.num_docs ? x.num_docs : 1) * sizeof(uint64_t));
    uint8_t* seen = (uint8_t*)calloc(n, 1);
    sh.tc = (uint64_t*)calloc(n, sizeof(uint64_t));
    if (x.num_docs != n) {
        SET_ERR("stream check: image has %llu documents, corpus %llu", (unsigned long long)x.num_docs,
                (unsigned long long)n);
        rc = 3;
    }
    for (uint64_t c = 0; rc == 0 && c < x.num_docs; ++c) { /* column -> draw index by name */
        char nm[48];
        const uint8_t* p = x.names[c];
        uint64_t id = 0;
        int ok = x.name_len[c] > 3 && x.name_len[c] < 40 && memcmp(p, "doc", 3) == 0;
        for (uint16_t i = 3; ok && i < x.name_len[c]; ++i) {
            ok = p[i] >= '0' && p[i] <= '9';
            id = id * 10 + (uint64_t)(p[i] - '0');
        }
        ok = ok && id < n && !seen[id];
        if (ok) {
            int l = doc_name(id, width, nm);
            ok = l == x.name_len[c] && memcmp(nm, p, (size_t)l) == 0;
        }
        if (!ok) {
            SET_ERR("stream check: column %llu has an unexpected or repeated name", (unsigned long long)c);
            rc = 3;
            break;
        }
        seen[id] = 1;
        col_id[c] = id;
    }
    free(seen);
    if (rc == 0) {
        sh.col_id = col_id;
        for (uint64_t b = 0; b < x.num_blocks; ++b) {
            const orc_block* B = &x.blocks[b];
            if (B->w > sh.max_w) sh.max_w = B->w;
            for (uint64_t g = 0; 64 * g < B->doc_count; ++g) {
                uint64_t c1 = 64 * g + 64 < B->doc_count ? 64 * g + 64 : B->doc_count, bases = 0;
                for (uint64_t c = 64 * g; c < c1; ++c) bases += s->doc_len[col_id[B->doc_base + c]];
                sh.units = (unit*)realloc(sh.units, (sh.n_units + 1) * sizeof(unit));
                sh.units[sh.n_units++] = (unit){b, g, bases * s->params.k + B->w};
            }
        }
        for (uint64_t i = 0; i < n; ++i)
            if (s->doc_len[i] > sh.max_len) sh.max_len = s->doc_len[i];
        qsort(sh.units, sh.n_units, sizeof(unit), cmp_unit);
        if (threads < 1) threads = 1;
        worker* ws = (worker*)calloc((size_t)threads, sizeof(worker));
        pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
        int started = 0;
        for (int t = 0; t < threads; ++t) {
            worker* W = &ws[t];
            W->sh = &sh;
            W->fwd = (uint8_t*)malloc(sh.max_len + 1);
            W->rc = (uint8_t*)malloc(sh.max_len + 1);
            W->sym = (uint8_t*)malloc(sh.max_len + 1);
            W->keys = (uint64_t*)malloc((sh.max_len + 1) * sizeof(uint64_t));
            W->slab = (uint64_t*)malloc((sh.max_w ? sh.max_w : 1) * sizeof(uint64_t));
            if (!W->fwd || !W->rc || !W->sym || !W->keys || !W->slab) {
                SET_ERR("stream check: out of host memory");
                rc = 4;
                break;
            }
        }
        for (int t = 0; rc == 0 && t < threads; ++t, ++started) pthread_create(&th[t], NULL, work, &ws[t]);
        for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
        for (int t = 0; t < threads; ++t) {
            free(ws[t].fwd);
            free(ws[t].rc);
            free(ws[t].sym);
            free(ws[t].keys);
            free(ws[t].slab);
            free(ws[t].cnt.tmp);
            free(ws[t].cnt.tab);
            free(ws[t].cnt.hist);
        }
        free(ws);
        free(th);
        free(sh.units);
    }
    if (rc == 0) {
        /* term counts vs the image's, then the oracle's own header */
        for (uint64_t c = 0; c < x.num_docs; ++c) rep->term_count_mismatch += sh.tc[col_id[c]] != x.term_count[c];
        ord* o = (ord*)malloc(n * sizeof(ord));
        for (uint64_t i = 0; i < n; ++i) o[i] = (ord){sh.tc[i], i};
        const uint64_t B = s->kind == 1 ? s->params.block_size : n;
        if (s->kind == 1) qsort(o, n, sizeof(ord), cmp_ord);
        orc_index y;
        memset(&y, 0, sizeof y);
        y.params = s->params;
        y.kind = (uint8_t)s->kind;
        y.num_docs = n;
        y.num_blocks = (n + B - 1) / B; /* compact_index.cpp:41-42; classic: one block */
        y.blocks = (orc_block*)calloc(y.num_blocks, sizeof(orc_block));
        y.names = (const uint8_t**)malloc(n * sizeof(void*));
        y.name_len = (uint16_t*)malloc(n * sizeof(uint16_t));
        y.term_count = (uint64_t*)malloc(n * sizeof(uint64_t));
        char* pool = (char*)malloc(n * 48);
        for (uint64_t i = 0; i < n; ++i) {
            y.name_len[i] = (uint16_t)doc_name(o[i].id, width, pool + 48 * i);
            y.names[i] = (const uint8_t*)(pool + 48 * i);
            y.term_count[i] = o[i].tc;
        }
        uint64_t expect = 0;
        for (uint64_t b = 0; b < y.num_blocks; ++b) {
            uint64_t lo = b * B, hi = lo + B < n ? lo + B : n, mx = 0;
            for (uint64_t i = lo; i < hi; ++i)
                if (o[i].tc > mx) mx = o[i].tc;
            y.blocks[b].doc_count = hi - lo;
            y.blocks[b].row_bytes = (hi - lo + 7) / 8;
            y.blocks[b].doc_base = lo;
            orc_size_filter(mx, s->params.p, s->params.k, &y.blocks[b].w); /* bloom.cpp:50-66 */
            expect += y.blocks[b].w * y.blocks[b].row_bytes;
        }
        uint8_t* head = NULL;
        uint64_t hlen = 0;
        orc_header_image(&y, &head, &hlen);
        rep->header_len = hlen;
        rep->image_len_expected = hlen + expect;
        rep->header_equal = hlen <= img_len && memcmp(head, img, hlen) == 0 && hlen + expect == img_len;
        if (term_counts)
            for (uint64_t i = 0; i < n; ++i) term_counts[i] = sh.tc[i];
        orc_free(head);
        free(pool);
        free(y.blocks);
        free(y.names);
        free(y.name_len);
        free(y.term_count);
        free(o);
        rep->payload_bad_bytes = sh.rep.payload_bad_bytes;
        rep->bad_block = sh.rep.bad_block;
        rep->bad_row = sh.rep.bad_row;
        rep->bad_byte = sh.rep.bad_byte;
        rep->windows = sh.rep.windows;
    }
    free(col_id);
    free(sh.tc);
    pthread_mutex_destroy(&sh.mu);
    orc_index_free(&x);
    return rc;
}
