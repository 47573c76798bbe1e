/* cobs_gpu.h — C-ABI of the B200-native COBS query / construction path.
 *
 * This is the drop-in boundary.  The reference exposes its path as a C++ API
 * (/root/reference/proj/include/cobs); every entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only: no C++ or
 * torch types cross this boundary, no exceptions escape it.
 *
 * Return codes mirror the reference's exception taxonomy as its CLI maps
 * it (proj/src/cli.cpp:448-454):
 *   COBS_OK (0)     success
 *   COBS_EUSAGE (1) std::invalid_argument  (bad K, bad params, ...)
 *   COBS_EDATA (2)  cobs::DataError        (corrupt file, empty corpus,
 *                                           duplicate names, l = 0 pattern)
 *   COBS_ECUDA (4)  device failure (no reference equivalent)
 * Error text (same wording as the reference's exception messages) goes to
 * `err` (may be NULL) truncated to `errlen`.
 *
 * Threading: one CUDA stream per index handle; calls on one handle are
 * serialised by the library; distinct handles are independent.  Results are
 * library-allocated and freed by the library.
 */
#ifndef COBS_GPU_H
#define COBS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COBS_OK 0
#define COBS_EUSAGE 1
#define COBS_EDATA 2
#define COBS_ECUDA 4

#define COBS_KIND_CLASSIC 0 /* proj/include/cobs/index_view.hpp:13 */
#define COBS_KIND_COMPACT 1 /* proj/include/cobs/index_view.hpp:14 */

/* proj/include/cobs/params.hpp:17-38 (IndexParams) */
typedef struct cobs_index_params {
    uint32_t q;
    uint32_t k;
    double p;
    uint64_t block_size;
    uint8_t canonical;
    uint8_t hash_scheme;
    uint8_t reserved[6];
} cobs_index_params;

typedef struct cobs_gpu_index cobs_gpu_index;
typedef struct cobs_gpu_results cobs_gpu_results;

/* ---- library ---------------------------------------------------------- */

/* Version string of this library. */
const char* cobs_gpu_version(void);

/* ---- index lifecycle -------------------------------------------------- */

/* Replaces cobs::open_resident (proj/include/cobs/storage.hpp:19,
 * proj/src/storage.cpp:407-411): parse + validate with the same rejection
 * matrix as parse_index (proj/src/storage.cpp:182-280), then upload every
 * block payload to HBM on `device` (rows re-pitched to 32-byte multiples). */
int cobs_gpu_index_open(const char* path, int device, cobs_gpu_index** out, char* err,
                        size_t errlen);

/* Same with an HBM budget (bytes).  If the pitched payload exceeds a
 * non-zero budget the index opens in the host-resident streaming mode
 * (the counterpart of open_random_access,
 * storage.hpp:21-23): the payload stays in pinned host memory and each query
 * batch streams it through two staging buffers of budget/2 bytes, copies
 * overlapping the gather.  Results are identical to the resident mode. */
int cobs_gpu_index_open_ex(const char* path, int device, uint64_t hbm_budget, cobs_gpu_index** out,
                           char* err, size_t errlen);
/* cobs_gpu_index_open_ex from an in-memory file image. */
int cobs_gpu_index_open_image_ex(const uint8_t* image, uint64_t len, const char* path, int device,
                                 uint64_t hbm_budget, cobs_gpu_index** out, char* err, size_t errlen);
/* 1 if the index is in the host-resident streaming mode. */
int cobs_gpu_index_streaming(const cobs_gpu_index* index);

/* cobs::open_random_access (storage.hpp:23, storage.cpp:320-341) in its own
 * spirit: when the pitched payload exceeds hbm_budget the payload is NOT
 * copied to host memory -- every batch reads it from the file (host
 * threads, pread + repack into pinned group images) and streams it through
 * two HBM staging buffers, so indexes larger than host RAM work too.
 * Within the budget the index is resident, as cobs_gpu_index_open. */
int cobs_gpu_index_open_file(const char* path, int device, uint64_t hbm_budget, cobs_gpu_index** out,
                             char* err, size_t errlen);

/* Block sharding of a compact index (the reference has no
 * sharded reader): blocks [block_lo, block_hi) of the file at `path` as a
 * standalone compact index in HBM -- same params, those blocks and their
 * documents, the whole header validated as by cobs_gpu_index_open.  Hit
 * columns of a shard are local; add cobs_gpu_index_column_offset for the
 * file column.  Per query, the union of every shard's hits ordered by
 * (score desc, name asc) and cut to top_t equals the unsharded result.
 * COBS_EUSAGE for an empty/out-of-range block range or a classic index
 * split into parts. */
int cobs_gpu_index_open_blocks(const char* path, int device, uint64_t block_lo, uint64_t block_hi,
                               cobs_gpu_index** out, char* err, size_t errlen);
uint64_t cobs_gpu_index_column_offset(const cobs_gpu_index* index);

/* Same, from an in-memory file image (`path` is only used in messages). */
int cobs_gpu_index_open_image(const uint8_t* image, uint64_t len, const char* path, int device,
                              cobs_gpu_index** out, char* err, size_t errlen);

/* Launch this handle's work on a caller-owned CUDA stream (a cudaStream_t
 * passed as void*; NULL restores the handle's own stream), so callers can
 * bracket batches with their own events.  The caller keeps the stream alive. */
int cobs_gpu_index_set_stream(cobs_gpu_index* index, void* stream);

/* Releases HBM and host state.  NULL is a no-op. */
void cobs_gpu_index_close(cobs_gpu_index* index);

/* IndexView metadata (proj/include/cobs/index_view.hpp:22-35). */
int cobs_gpu_index_params(const cobs_gpu_index* index, cobs_index_params* out);
uint8_t cobs_gpu_index_kind(const cobs_gpu_index* index);
uint64_t cobs_gpu_index_block_count(const cobs_gpu_index* index);
uint64_t cobs_gpu_index_doc_count(const cobs_gpu_index* index, uint64_t block);
uint64_t cobs_gpu_index_width(const cobs_gpu_index* index, uint64_t block);
uint64_t cobs_gpu_index_row_bytes(const cobs_gpu_index* index, uint64_t block);
uint64_t cobs_gpu_index_total_docs(const cobs_gpu_index* index);
/* IndexView::doc(b, i) (index_view.hpp:27).  `name` stays valid until close. */
int cobs_gpu_index_doc(const cobs_gpu_index* index, uint64_t block, uint64_t i, const char** name,
                       uint64_t* name_len, uint64_t* term_count);
/* Global column (file column order, block-major) of document (block, i). */
uint64_t cobs_gpu_index_doc_global(const cobs_gpu_index* index, uint64_t block, uint64_t i);
/* HBM bytes held by the payload (pitched) and by the whole index. */
uint64_t cobs_gpu_index_device_bytes(const cobs_gpu_index* index);
/* IndexView::row_data (index_view.hpp:41-42) served from HBM by a D2H copy of
 * bytes [byte_lo, byte_hi) of row r (slow; tools and tests). */
int cobs_gpu_index_row(const cobs_gpu_index* index, uint64_t block, uint64_t r, uint64_t byte_lo,
                       uint64_t byte_hi, uint8_t* out);
/* Replaces cobs::write_index(const IndexView&, path) (storage.hpp:14,
 * proj/src/storage.cpp:345-397) for a device-resident index: the payload is
 * read back from HBM and the file is byte-identical to the reference's. */
int cobs_gpu_index_write(const cobs_gpu_index* index, const char* path, char* err, size_t errlen);

/* The same bytes as cobs_gpu_index_write, returned in memory (free with
 * cobs_gpu_free). */
int cobs_gpu_index_image(const cobs_gpu_index* index, uint8_t** image, uint64_t* image_len, char* err,
                         size_t errlen);

/* The same image written into a caller buffer (no library allocation, no
 * intermediate copy: for images of tens of GB).  *image_len receives the
 * size; with dst == NULL or cap < size nothing is written and 1 returned
 * (query the size with dst == NULL). */
int cobs_gpu_index_image_into(const cobs_gpu_index* index, uint8_t* dst, uint64_t cap, uint64_t* image_len,
                              char* err, size_t errlen);

/* ---- batch query ------------------------------------------------------ */

/* flags */
#define COBS_Q_HITS 1u          /* ordered, thresholded hit lists */
#define COBS_Q_SCORES 2u        /* dense per-document score matrix n x total_docs */
#define COBS_Q_DEVICE_INPUT 4u  /* patterns / offsets are device pointers */
#define COBS_Q_KEEP_DEVICE 8u   /* leave results in HBM (no D2H); for timing */
#define COBS_Q_PRUNE 16u        /* hits only: stop reading a (query, slice)'s rows once no
                                   document there can still reach tau; identical hit lists,
                                   fewer row bytes (not in the reference) */

/* Replaces cobs::query (proj/include/cobs/query.hpp:46-47,
 * proj/src/query.cpp:123-164) over a batch, the way the CLI batch mode
 * calls it (proj/src/cli.cpp:205-221): query i is pattern bytes
 * [offsets[i], offsets[i+1]).  Patterns are raw bytes (not uppercased), as
 * query() takes them.  K outside (0,1] -> COBS_EUSAGE for the whole batch
 * (query.cpp:125-126); a pattern with l = 0 gets status COBS_EDATA and the
 * reference's message in its result (query.cpp:133-138), as the CLI's inline
 * "ERR" line does, and does not abort the batch. */
int cobs_gpu_query_batch(cobs_gpu_index* index, const uint8_t* patterns, const uint64_t* offsets,
                         uint64_t n, double K, uint64_t top_t, uint32_t flags,
                         cobs_gpu_results** out, char* err, size_t errlen);

uint64_t cobs_gpu_results_count(const cobs_gpu_results* r);
/* QueryResult fields (query.hpp:31-39) of query i: ell, skipped, status
 * (0 / COBS_EDATA), message (empty when ok), number of hits after top_t. */
int cobs_gpu_results_query(const cobs_gpu_results* r, uint64_t i, uint64_t* ell, uint64_t* skipped,
                           int* status, const char** message, uint64_t* n_hits);
/* Hits of query i ordered by (score desc, name asc) (query.cpp:156-162):
 * global document columns and scores.  Pointers valid until free. */
int cobs_gpu_results_hits(const cobs_gpu_results* r, uint64_t i, const uint32_t** docs,
                          const uint32_t** scores);
/* Bulk view of all n queries (for array-oriented hosts): ell[n], skipped[n],
 * status[n], hit_off[n] / hit_n[n] index into doc/score[total_hits]. */
int cobs_gpu_results_arrays(const cobs_gpu_results* r, const uint32_t** ell, const uint64_t** skipped,
                            const int** status, const uint64_t** hit_off, const uint64_t** hit_n,
                            const uint32_t** docs, const uint32_t** scores, uint64_t* total_hits);
/* Dense score matrix (COBS_Q_SCORES): n x total_docs values of
 * `*score_bytes` (2 when every l <= 65535, else 4, as query.cpp:150-153
 * picks uint16/uint32 counters), row i = query i, columns in file order. */
const void* cobs_gpu_results_scores(const cobs_gpu_results* r, uint32_t* score_bytes);
/* Device-side timings of the batch (ms, CUDA events on the index's stream):
 * termize+hash, gather, order, and the whole call from before the H2D of
 * the patterns to after the D2H of the results. */
int cobs_gpu_results_timing(const cobs_gpu_results* r, double* ms_termize, double* ms_gather,
                            double* ms_order, double* ms_total);
/* Kernels of this library launched by the batch (library sorts excluded). */
uint32_t cobs_gpu_results_launches(const cobs_gpu_results* r);
/* Algorithmic row bytes of the batch: sum_i k * l_i * sum_b row_bytes_b
 * (the random-access reader's bytes_read accounting, storage.cpp:325-331). */
uint64_t cobs_gpu_results_row_bytes(const cobs_gpu_results* r);
/* Streaming mode: index payload bytes copied host -> HBM by the batch (the
 * analogue of RandomAccessView::bytes_read, index_view.hpp:44-46). */
uint64_t cobs_gpu_results_h2d_index_bytes(const cobs_gpu_results* r);
/* Where kernel 2 read the index rows from: 0 = HBM-resident payload, 1 =
 * the host-resident (pinned) payload directly over PCIe (zero-copy: only the
 * addressed rows), 2 = the host-resident payload streamed through HBM staging
 * buffers (the whole payload per batch).  All compute the same scores and
 * hits (query.cpp:49-89);
 * h2d_index_bytes counts the index bytes moved. */
uint32_t cobs_gpu_results_gather_path(const cobs_gpu_results* r);
void cobs_gpu_results_free(cobs_gpu_results* r);

/* ---- build ------------------------------------------------------------ */

/* Replaces extract_terms + build_classic / build_compact + write_index
 * (termizer.hpp:37-38, classic_index.hpp:37-44, compact_index.hpp:26-27,
 * storage.hpp:14-16).  Content strings i are bytes [seg_offsets[i],
 * seg_offsets[i+1]) of `seqs`; document d owns strings
 * [doc_segs[d], doc_segs[d+1]) (grams never span strings); names[d] is a
 * NUL-terminated name (so build names cannot contain NUL bytes; the reader
 * accepts any name bytes the format allows).  kind: COBS_KIND_CLASSIC (documents in input order,
 * width forced_w or sized for the largest document) or COBS_KIND_COMPACT
 * (sorted by (term_count, name), blocks of block_size).  The image written
 * to `out_path` (if non-NULL) and/or returned through `image`/`image_len`
 * (if non-NULL; free with cobs_gpu_free) is byte-identical to the
 * reference writer's. */
int cobs_gpu_build(const uint8_t* seqs, const uint64_t* seg_offsets, uint64_t n_segs,
                   const uint64_t* doc_segs, const char* const* names, uint64_t n_docs,
                   const cobs_index_params* params, int kind, uint64_t forced_w, int device,
                   const char* out_path, uint8_t** image, uint64_t* image_len, char* err,
                   size_t errlen);

/* build flags */
#define COBS_B_DEVICE_INPUT 1u /* `seqs` is a device pointer (seg/doc arrays stay on the host) */
/* Every segment is one pre-extracted term -- the reference's TermSet input
 * (termizer.hpp:14-26) to build_classic / build_compact
 * (classic_index.hpp:37-44, compact_index.hpp:26-27): terms are hashed as
 * given (no windowing, canonicalisation or skipping), term_count = number of
 * terms, and a term whose length is not q returns COBS_EUSAGE with the
 * reference's message (classic_index.cpp:49-56). */
#define COBS_B_TERMS 2u
/* `seqs` is `const uint8_t* const*`: n_segs host pointers, string i of
 * seg_offsets[i+1] - seg_offsets[i] bytes (the offsets still describe the
 * packed layout).  The strings are gathered into HBM through the library's
 * pinned staging buffers, so a caller holding separate strings (the
 * reference's vector<string> contents) needs no packed host copy.  Not
 * with COBS_B_DEVICE_INPUT. */
#define COBS_B_SEGMENT_PTRS 4u

/* cobs_gpu_build with flags, optionally returning the built index resident
 * in HBM (`index_out`, ready to query; close with cobs_gpu_index_close)
 * instead of, or as well as, the file image / file. */
int cobs_gpu_build_ex(const uint8_t* seqs, const uint64_t* seg_offsets, uint64_t n_segs,
                      const uint64_t* doc_segs, const char* const* names, uint64_t n_docs,
                      const cobs_index_params* params, int kind, uint64_t forced_w, int device,
                      uint32_t flags, const char* out_path, uint8_t** image, uint64_t* image_len,
                      cobs_gpu_index** index_out, char* err, size_t errlen);

/* Replaces cobs::merge_classic (proj/include/cobs/classic_index.hpp:46-49,
 * proj/src/classic_index.cpp:96-115): documents of `a` then `b`, every row the
 * bit-concatenation of a's and b's (bit_matrix.cpp:10-23), computed on the
 * device into a new device-resident index.  COBS_EDATA on differing
 * parameters / widths or duplicate names (same messages); COBS_EUSAGE unless
 * both are classic and resident on `device`. */
int cobs_gpu_merge_classic(const cobs_gpu_index* a, const cobs_gpu_index* b, int device,
                           cobs_gpu_index** out, char* err, size_t errlen);

/* Build timings (ms) of the calling thread's last cobs_gpu_build: term
 * counting, fill (sequences in HBM -> finished matrix), total incl. H2D,
 * D2H and serialisation. */
int cobs_gpu_build_timing(double* ms_count, double* ms_fill, double* ms_total);
/* The same plus the host<->device copy legs of the last build: sequences
 * H2D (0 when they were already on the device) and the index image D2H
 * (0 when the index stayed in HBM). */
int cobs_gpu_build_timing_ex(double* ms_h2d, double* ms_count, double* ms_fill, double* ms_d2h,
                             double* ms_total);
/* The count leg of the last build split up: its kernels alone (CUDA events
 * after the workspace allocation and before its release), and the host time
 * of the workspace's cudaMalloc and cudaFree calls (both inside ms_count). */
int cobs_gpu_build_timing_count(double* ms_kernels, double* ms_alloc, double* ms_free);

/* Releases the device memory the library keeps between calls: the build's
 * count workspace (<= 17 GB: two key buffers and per-wave arrays, kept so
 * that repeated builds skip their cudaMalloc / cudaFree; COBS_BUILD_CACHE=0
 * frees it after every build).  The library also releases it by itself when
 * one of its own device allocations runs out of memory.  Returns the bytes
 * released. */
uint64_t cobs_gpu_trim(void);

void cobs_gpu_free(void* p);

/* ---- file front ends ------------------------------ */

#define COBS_FORMAT_AUTO 0  /* by extension: .fa/.fasta/.fna -> FASTA, else text */
#define COBS_FORMAT_FASTA 1
#define COBS_FORMAT_TEXT 2

/* `cobs query index -F queries.fa -K K -t top_t` (proj/src/cli.cpp:192-223):
 * FASTA records read as read_fasta_named does (termizer.cpp:150-162:
 * uppercased sequence lines, name = header up to the first blank,
 * "query_<N>" for empty headers), queried as one batch, and the CLI's batch
 * output returned byte for byte: per record "*name	N
" then N lines
 * "doc	score	ell
", or "*name	ERR	<message>
" (cli.cpp:187-190,214-218).
 * *tsv is NUL-terminated; free with cobs_gpu_free. */
int cobs_gpu_query_fasta(cobs_gpu_index* index, const char* fasta_path, double K, uint64_t top_t,
                         char** tsv, uint64_t* tsv_len, char* err, size_t errlen);

/* `cobs build inputs... --mode classic|compact --format F` (cli.cpp:112-166):
 * directories expand recursively in lexicographic path order, every file is
 * one document named by its stem (load_document, termizer.cpp:168-172),
 * FASTA records are separate content strings.  Output as cobs_gpu_build. */
int cobs_gpu_build_files(const char* const* inputs, uint64_t n_inputs, const cobs_index_params* params,
                         int kind, int format, int device, const char* out_path, uint8_t** image,
                         uint64_t* image_len, char* err, size_t errlen);

/* ---- synthetic workloads (bench / tests; not part of the reference
 *      boundary) ----------------------------------------------------- */

/* Config-5 procedural compact index generated directly in HBM from a seed
 * (paper_1905_09624_b200/csrc/synth.h): n_docs documents with log-normal
 * (median, sigma) term counts sorted into blocks of block_size, widths
 * size_filter(block max, p, 1), i.i.d. Bernoulli bits of density
 * 1-(1-1/w)^n per block.  Equivalent to opening the file the reference
 * writer would produce for the same header and rows. */
int cobs_gpu_index_synth_c5(uint64_t seed, uint64_t n_docs, uint64_t block_size, double median,
                            double sigma, double p, int device, cobs_gpu_index** out, char* err,
                            size_t errlen);

/* Blocks [block_lo, block_hi) of the same config-5 index as a block shard
 * (cobs_gpu_index_open_blocks semantics: hit columns are local,
 * cobs_gpu_index_column_offset maps them to file columns). */
int cobs_gpu_index_synth_c5_blocks(uint64_t seed, uint64_t n_docs, uint64_t block_size, double median,
                                   double sigma, double p, uint64_t block_lo, uint64_t block_hi, int device,
                                   cobs_gpu_index** out, char* err, size_t errlen);

/* Generate documents [doc_lo, doc_hi) of a synthetic corpus on the device
 * into `dev_out` (device pointer, sum of lengths bytes, concatenated in
 * document order). alpha: 0 DNA, 1 amino acids. */
int cobs_gpu_synth_docs(uint64_t seed, int alpha, const uint64_t* doc_len, uint64_t doc_lo,
                        uint64_t doc_hi, uint8_t* dev_out, int device);

/* Roofline calibration on this GPU (bench/tools; not a reference
 * interface): HBM read GB/s for a streaming read and for random 128-byte
 * lines in the gather kernel's access shape, over a power-of-two buffer of
 * <= `bytes` (>= 1 GiB) allocated for the call. */
int cobs_gpu_calibrate(int device, uint64_t bytes, double* stream_gbs, double* random128_gbs);

#ifdef __cplusplus
}
#endif

#endif /* COBS_GPU_H */
