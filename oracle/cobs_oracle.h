/* CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference COBS query and construction path
 * (/root/reference/proj, clean-room C++20).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker.  The product (paper_1905_09624_b200) never links or calls it.
 *
 * Pinned by: tests/test_oracle_golden.py (XXH64 / size_filter / score_threshold
 * / termizer / 90-byte file golden vectors from the reference's own tests and
 * FORMAT.md) and tests/test_oracle_vs_ref.py (bit-exact against the reference
 * sources compiled into oracle/_ref/ by oracle/Makefile).
 *
 * Return codes mirror the reference's exception taxonomy as the CLI maps it
 * (proj/src/cli.cpp:448-454): 0 ok, 1 std::invalid_argument, 2 cobs::DataError.
 */
#ifndef COBS_ORACLE_H
#define COBS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/cobs/xxhash64.hpp:45-95 */
uint64_t orc_xxh64(const void* data, size_t len, uint64_t seed);
/* proj/src/bloom.cpp:42-48 */
double orc_fpr_approx(uint64_t w, uint32_t k, uint64_t v);
/* proj/src/bloom.cpp:50-66; returns 0 ok / 1 invalid argument */
int orc_size_filter(uint64_t v, double p, uint32_t k, uint64_t* w);
/* proj/src/bloom.cpp:120-123 */
uint64_t orc_score_threshold(uint64_t ell, double K);

/* proj/src/termizer.cpp:103-129 over `nseg` content strings.  *terms receives
 * ell*q bytes (sorted, distinct; malloc'd, free with orc_free). */
int orc_extract_terms(const uint8_t* const* segs, const uint64_t* lens, size_t nseg, uint32_t q,
                      int canonical, uint8_t** terms, uint64_t* ell, uint64_t* skipped,
                      uint64_t* occurrences);

typedef struct orc_params {
    uint32_t q, k;
    double p;
    int canonical;
    uint64_t block_size;
    uint8_t hash_scheme;
} orc_params;

typedef struct orc_block {
    uint64_t doc_count, w, row_bytes;
    uint64_t offset;   /* absolute file offset of the payload */
    uint64_t doc_base; /* global column index of the block's first document */
} orc_block;

/* Parsed index (file image or procedural). Names point into `img` (file) or
 * into `name_pool` (procedural). */
typedef struct orc_index {
    orc_params params;
    uint8_t kind;
    uint64_t num_blocks, num_docs;
    orc_block* blocks;
    const uint8_t** names;
    uint16_t* name_len;
    uint64_t* term_count;
    const uint8_t* payload; /* image payload (NULL for procedural) */
    uint64_t payload_start, file_size;
    char* name_pool;
    /* config-5 procedural rows */
    uint64_t c5_seed;
    uint32_t* c5_thr16;
} orc_index;

/* proj/src/storage.cpp:182-280 (parse_index) over an in-memory file image.
 * The image must outlive the index. */
int orc_parse(const uint8_t* img, uint64_t len, const char* path, orc_index* out, char* err,
              size_t errlen);
void orc_index_free(orc_index* idx);

typedef struct orc_hit {
    uint64_t doc; /* global column index */
    uint64_t score;
} orc_hit;

/* proj/src/query.cpp:123-164.  `scores` (num_docs entries, may be NULL)
 * receives every document's score; `hits` (malloc'd) the documents with
 * score >= tau ordered by (score desc, name asc) truncated to top_t. */
int orc_query(const orc_index* idx, const uint8_t* pat, uint64_t len, double K, uint64_t top_t,
              uint32_t* scores, uint64_t* ell, uint64_t* skipped, orc_hit** hits,
              uint64_t* n_hits, char* err, size_t errlen);

/* Batch of queries on `threads` threads (one query per thread at a time,
 * like proj/src/cli.cpp:205-221).  scores: n x num_docs (may be NULL);
 * status[i]: 0/1/2.  Hits are not returned (timing / score export use). */
int orc_query_batch(const orc_index* idx, const uint8_t* pats, const uint64_t* offsets, size_t n,
                    double K, uint32_t* scores, uint64_t* ell, uint64_t* skipped, int* status,
                    uint64_t* n_hits, int threads);

/* Build + serialise: proj/src/classic_index.cpp:40-94,
 * proj/src/compact_index.cpp:19-71, proj/src/storage.cpp:345-397.
 * Document d owns content strings [doc_seg[d], doc_seg[d+1]) of (segs, lens).
 * kind 0 classic / 1 compact.  *img is malloc'd. */
int orc_build_image(const uint8_t* const* segs, const uint64_t* lens, const uint64_t* doc_seg,
                    const char* const* names, size_t n_docs, const orc_params* params, int kind,
                    uint64_t forced_w, uint8_t** img, uint64_t* img_len, char* err, size_t errlen);

/* Config-5 procedural compact index (no payload; rows regenerated from the
 * seed with synth.h).  Header semantics follow proj/src/compact_index.cpp:27-52. */
int orc_c5_make(uint64_t seed, uint64_t n_docs, uint64_t block_size, double median, double sigma,
                double p, orc_index* out);
/* Header bytes (everything before the payload) of any orc_index, as
 * proj/src/storage.cpp:345-380 writes them. */
int orc_header_image(const orc_index* idx, uint8_t** img, uint64_t* len);

/* Full-size streaming check (oracle/cobs_stream.c): the index image `img`
 * of the seeded synthetic corpus (synth.h documents 0..n_docs-1, lengths
 * doc_len[], names "doc" + zero-padded draw index) against the build the
 * reference would make of it -- every payload byte and the whole header --
 * without materialising the corpus or a second index.  Returns 0 (report
 * filled), 1 unsupported shape, 2 image unparsable, 3 documents/names do not
 * match the corpus, 4 out of memory. */
typedef struct orc_stream_spec {
    uint64_t seed;
    int alpha; /* 0 DNA, 1 the 20-letter amino-acid alphabet */
    uint64_t n_docs;
    const uint64_t* doc_len;
    orc_params params;
    int kind; /* 0 classic, 1 compact */
} orc_stream_spec;

typedef struct orc_stream_report {
    int header_equal;            /* oracle header == image header, and lengths agree */
    uint64_t header_len, image_len_expected;
    uint64_t term_count_mismatch; /* documents whose term_count differs from the image's */
    uint64_t payload_bad_bytes;   /* payload bytes that differ */
    uint64_t bad_block, bad_row, bad_byte; /* the first (lowest) differing payload byte */
    uint64_t windows;
} orc_stream_report;

int orc_stream_check(const orc_stream_spec* spec, const uint8_t* img, uint64_t img_len, int threads,
                     orc_stream_report* rep, uint64_t* term_counts, char* err, size_t errlen);

void orc_free(void* p);

#ifdef __cplusplus
}
#endif

#endif
