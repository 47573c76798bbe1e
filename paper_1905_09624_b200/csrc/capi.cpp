// extern "C" boundary (include/cobs_gpu.h).  Exceptions never cross it: the
// reference's taxonomy maps to return codes exactly as its CLI does
// (proj/src/cli.cpp:448-454).
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <memory>

#include "../../include/cobs_gpu.h"
#include "build.hpp"
#include "frontend.hpp"
#include "index.hpp"
#include "merge.hpp"

namespace cobsg {
void calibrate(int device, uint64_t bytes, double* stream_gbs, double* random128_gbs); // calib.cu
}

struct cobs_gpu_index {
    std::unique_ptr<cobsg::DeviceIndex> ix;
};
struct cobs_gpu_results {
    cobsg::QueryResults r;
};

namespace {

void set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) std::snprintf(err, errlen, "%s", msg);
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        if (err && errlen) err[0] = 0;
        return COBS_OK;
    } catch (const cobsg::DataError& e) {
        set_err(err, errlen, e.what());
        return COBS_EDATA;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return COBS_EUSAGE;
    } catch (const cobsg::CudaError& e) {
        set_err(err, errlen, e.what());
        return COBS_ECUDA;
    } catch (const std::bad_alloc&) {
        set_err(err, errlen, "out of host memory");
        return COBS_ECUDA;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return COBS_ECUDA;
    }
}

cobsg::Params to_params(const cobs_index_params* p) {
    cobsg::Params P;
    P.q = p->q;
    P.k = p->k;
    P.p = p->p;
    P.block_size = p->block_size;
    P.canonical = p->canonical != 0;
    P.hash_scheme = p->hash_scheme;
    return P;
}

} // namespace

extern "C" {

const char* cobs_gpu_version(void) { return "cobs-b200 0.1 (sm_100a)"; }

int cobs_gpu_index_open_ex(const char* path, int device, uint64_t hbm_budget, cobs_gpu_index** out,
                           char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index(cobsg::file_source(path), device, hbm_budget);
        *out = h.release();
    });
}

int cobs_gpu_index_open_file(const char* path, int device, uint64_t hbm_budget, cobs_gpu_index** out,
                             char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index(cobsg::file_source(path), device, hbm_budget, /*file_backed=*/true);
        *out = h.release();
    });
}

int cobs_gpu_index_open_blocks(const char* path, int device, uint64_t block_lo, uint64_t block_hi,
                               cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index_blocks(cobsg::file_source(path), device, block_lo, block_hi);
        *out = h.release();
    });
}

uint64_t cobs_gpu_index_column_offset(const cobs_gpu_index* index) { return index->ix->column_offset; }

int cobs_gpu_index_open_image_ex(const uint8_t* image, uint64_t len, const char* path, int device,
                                 uint64_t hbm_budget, cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index(cobsg::memory_source(image, len, path ? path : "<memory>"), device,
                                  hbm_budget);
        *out = h.release();
    });
}

int cobs_gpu_index_streaming(const cobs_gpu_index* index) { return index->ix->streaming() ? 1 : 0; }

int cobs_gpu_index_open(const char* path, int device, cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index(cobsg::file_source(path), device);
        *out = h.release();
    });
}

int cobs_gpu_index_open_image(const uint8_t* image, uint64_t len, const char* path, int device,
                              cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::open_index(cobsg::memory_source(image, len, path ? path : "<memory>"), device);
        *out = h.release();
    });
}

void cobs_gpu_index_close(cobs_gpu_index* index) { delete index; }

int cobs_gpu_index_set_stream(cobs_gpu_index* index, void* stream) {
    std::lock_guard<std::mutex> lock(index->ix->mu);
    index->ix->user_stream = static_cast<cudaStream_t>(stream);
    return COBS_OK;
}

int cobs_gpu_index_params(const cobs_gpu_index* index, cobs_index_params* out) {
    const cobsg::Params& P = index->ix->meta.params;
    std::memset(out, 0, sizeof *out);
    out->q = P.q;
    out->k = P.k;
    out->p = P.p;
    out->block_size = P.block_size;
    out->canonical = P.canonical ? 1 : 0;
    out->hash_scheme = P.hash_scheme;
    return COBS_OK;
}

uint8_t cobs_gpu_index_kind(const cobs_gpu_index* index) { return index->ix->meta.kind; }
uint64_t cobs_gpu_index_block_count(const cobs_gpu_index* index) { return index->ix->meta.blocks.size(); }
uint64_t cobs_gpu_index_doc_count(const cobs_gpu_index* index, uint64_t b) {
    return b < index->ix->meta.blocks.size() ? index->ix->meta.blocks[b].doc_count : 0;
}
uint64_t cobs_gpu_index_width(const cobs_gpu_index* index, uint64_t b) {
    return b < index->ix->meta.blocks.size() ? index->ix->meta.blocks[b].w : 0;
}
uint64_t cobs_gpu_index_row_bytes(const cobs_gpu_index* index, uint64_t b) {
    return b < index->ix->meta.blocks.size() ? index->ix->meta.blocks[b].row_bytes() : 0;
}
uint64_t cobs_gpu_index_total_docs(const cobs_gpu_index* index) { return index->ix->meta.total_docs(); }

int cobs_gpu_index_doc(const cobs_gpu_index* index, uint64_t b, uint64_t i, const char** name,
                       uint64_t* name_len, uint64_t* term_count) {
    const cobsg::IndexMeta& m = index->ix->meta;
    if (b >= m.blocks.size() || i >= m.blocks[b].doc_count) return COBS_EUSAGE;
    const cobsg::DocEntry& d = m.docs[m.blocks[b].doc_base + i];
    *name = d.name.data();
    *name_len = d.name.size();
    *term_count = d.term_count;
    return COBS_OK;
}

uint64_t cobs_gpu_index_doc_global(const cobs_gpu_index* index, uint64_t b, uint64_t i) {
    return index->ix->meta.blocks[b].doc_base + i;
}

uint64_t cobs_gpu_index_device_bytes(const cobs_gpu_index* index) {
    const cobsg::DeviceIndex& ix = *index->ix;
    return ix.streaming() ? 2 * ix.hs->staging_bytes : ix.payload_bytes;
}

int cobs_gpu_index_row(const cobs_gpu_index* index, uint64_t b, uint64_t r, uint64_t lo, uint64_t hi,
                       uint8_t* out) {
    return guarded(nullptr, 0, [&] {
        const cobsg::DeviceIndex& ix = *index->ix;
        if (b >= ix.blocks.size() || r >= ix.blocks[b].w || lo > hi || hi > ix.blocks[b].rb)
            throw cobsg::UsageError("row: out of range");
        if (ix.streaming()) {
            ix.hs->read_payload(ix.hs->block_off[b] + r * ix.blocks[b].rb + lo, out, hi - lo);
            return;
        }
        COBS_CUDA(cudaSetDevice(ix.device));
        COBS_CUDA(cudaMemcpy(out, ix.payload + ix.blocks[b].base + r * ix.blocks[b].pitch + lo, hi - lo,
                             cudaMemcpyDeviceToHost));
    });
}

int cobs_gpu_index_write(const cobs_gpu_index* index, const char* path, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const cobsg::DeviceIndex& ix = *index->ix;
        COBS_CUDA(cudaSetDevice(ix.device));
        std::vector<uint8_t> head = ix.meta.header_bytes();
        FILE* f = std::fopen(path, "wb");
        if (!f) throw cobsg::DataError(std::string("cannot create index file: ") + path);
        std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
        if (std::fwrite(head.data(), 1, head.size(), f) != head.size())
            throw cobsg::DataError(std::string("error writing index file: ") + path);
        if (ix.streaming()) { // payload in file layout: host copy or the source file
            std::vector<uint8_t> chunk(std::min<uint64_t>(ix.hs->host_bytes, 64ull << 20));
            for (uint64_t o = 0; o < ix.hs->host_bytes; o += chunk.size()) {
                const uint64_t len = std::min<uint64_t>(chunk.size(), ix.hs->host_bytes - o);
                ix.hs->read_payload(o, chunk.data(), len);
                if (std::fwrite(chunk.data(), 1, len, f) != len)
                    throw cobsg::DataError(std::string("error writing index file: ") + path);
            }
            return;
        }
        std::vector<uint8_t> buf;
        for (const cobsg::DevBlock& d : ix.blocks) {
            uint64_t rows_per = std::max<uint64_t>(1, (64ull << 20) / d.rb);
            for (uint64_t r0 = 0; r0 < d.w; r0 += rows_per) {
                uint64_t rows = std::min(rows_per, d.w - r0);
                buf.resize(rows * d.rb);
                COBS_CUDA(cudaMemcpy2D(buf.data(), d.rb, ix.payload + d.base + r0 * d.pitch, d.pitch, d.rb,
                                       rows, cudaMemcpyDeviceToHost));
                if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size())
                    throw cobsg::DataError(std::string("error writing index file: ") + path);
            }
        }
    });
}

int cobs_gpu_index_image(const cobs_gpu_index* index, uint8_t** image, uint64_t* image_len, char* err,
                         size_t errlen) {
    *image = nullptr;
    *image_len = 0;
    return guarded(err, errlen, [&] {
        std::vector<uint8_t> img = cobsg::index_image(*index->ix);
        *image = static_cast<uint8_t*>(std::malloc(std::max<size_t>(img.size(), 1)));
        if (!*image) throw std::bad_alloc();
        std::memcpy(*image, img.data(), img.size());
        *image_len = img.size();
    });
}

int cobs_gpu_index_image_into(const cobs_gpu_index* index, uint8_t* dst, uint64_t cap, uint64_t* image_len,
                              char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const uint64_t size = cobsg::index_image_size(*index->ix);
        if (image_len) *image_len = size;
        if (!dst || cap < size) throw cobsg::UsageError("index_image_into: buffer of " + std::to_string(cap) +
                                                        " bytes, image needs " + std::to_string(size));
        cobsg::index_image_into(*index->ix, dst);
    });
}

int cobs_gpu_query_batch(cobs_gpu_index* index, const uint8_t* patterns, const uint64_t* offsets,
                         uint64_t n, double K, uint64_t top_t, uint32_t flags, cobs_gpu_results** out,
                         char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto r = std::make_unique<cobs_gpu_results>();
        cobsg::query_batch(*index->ix, patterns, offsets, n, K, top_t, flags, r->r);
        *out = r.release();
    });
}

uint64_t cobs_gpu_results_count(const cobs_gpu_results* r) { return r->r.n; }

int cobs_gpu_results_query(const cobs_gpu_results* r, uint64_t i, uint64_t* ell, uint64_t* skipped,
                           int* status, const char** message, uint64_t* n_hits) {
    const cobsg::QueryResults& R = r->r;
    if (i >= R.n || i >= R.ell.size()) return COBS_EUSAGE;
    if (ell) *ell = R.ell[i];
    if (skipped) *skipped = R.skipped[i];
    if (status) *status = R.status[i];
    if (message) *message = R.message[i].c_str();
    if (n_hits) *n_hits = R.hit_n[i];
    return COBS_OK;
}

int cobs_gpu_results_hits(const cobs_gpu_results* r, uint64_t i, const uint32_t** docs,
                          const uint32_t** scores) {
    const cobsg::QueryResults& R = r->r;
    if (i >= R.n || i >= R.hit_off.size()) return COBS_EUSAGE;
    static const uint32_t empty = 0;
    if (R.doc.empty()) {
        *docs = &empty;
        *scores = &empty;
        return COBS_OK;
    }
    *docs = R.doc.data() + R.hit_off[i];
    *scores = R.score.data() + R.hit_off[i];
    return COBS_OK;
}

int cobs_gpu_results_arrays(const cobs_gpu_results* r, const uint32_t** ell, const uint64_t** skipped,
                            const int** status, const uint64_t** hit_off, const uint64_t** hit_n,
                            const uint32_t** docs, const uint32_t** scores, uint64_t* total_hits) {
    const cobsg::QueryResults& R = r->r;
    *ell = R.ell.data();
    *skipped = R.skipped.data();
    *status = R.status.data();
    *hit_off = R.hit_off.data();
    *hit_n = R.hit_n.data();
    *docs = R.doc.data();
    *scores = R.score.data();
    *total_hits = R.doc.size();
    return COBS_OK;
}

const void* cobs_gpu_results_scores(const cobs_gpu_results* r, uint32_t* score_bytes) {
    if (score_bytes) *score_bytes = r->r.score_bytes;
    return r->r.scores.empty() ? nullptr : r->r.scores.data();
}

int cobs_gpu_results_timing(const cobs_gpu_results* r, double* a, double* b, double* c, double* d) {
    if (a) *a = r->r.ms_termize;
    if (b) *b = r->r.ms_gather;
    if (c) *c = r->r.ms_order;
    if (d) *d = r->r.ms_total;
    return COBS_OK;
}

uint32_t cobs_gpu_results_launches(const cobs_gpu_results* r) { return r->r.launches; }

uint64_t cobs_gpu_results_row_bytes(const cobs_gpu_results* r) { return r->r.row_bytes; }

uint32_t cobs_gpu_results_gather_path(const cobs_gpu_results* r) {
    return r->r.zero_copy ? 1u : r->r.h2d_index_bytes ? 2u : 0u;
}

uint64_t cobs_gpu_results_h2d_index_bytes(const cobs_gpu_results* r) { return r->r.h2d_index_bytes; }

void cobs_gpu_results_free(cobs_gpu_results* r) { delete r; }

int cobs_gpu_build_ex(const uint8_t* seqs, const uint64_t* seg_offsets, uint64_t n_segs,
                      const uint64_t* doc_segs, const char* const* names, uint64_t n_docs,
                      const cobs_index_params* params, int kind, uint64_t forced_w, int device,
                      uint32_t flags, const char* out_path, uint8_t** image, uint64_t* image_len,
                      cobs_gpu_index** index_out, char* err, size_t errlen) {
    if (image) *image = nullptr;
    if (image_len) *image_len = 0;
    if (index_out) *index_out = nullptr;
    return guarded(err, errlen, [&] {
        if ((flags & COBS_B_SEGMENT_PTRS) && (flags & COBS_B_DEVICE_INPUT))
            throw cobsg::UsageError("build: COBS_B_SEGMENT_PTRS needs host strings");
        std::vector<std::string> nm(n_docs);
        for (uint64_t d = 0; d < n_docs; ++d) nm[d] = names[d];
        auto ix = cobsg::build_device_index(seqs, seg_offsets, n_segs, doc_segs, nm, to_params(params),
                                            static_cast<uint8_t>(kind), forced_w, device,
                                            (flags & COBS_B_DEVICE_INPUT) != 0, (flags & COBS_B_TERMS) != 0,
                                            (flags & COBS_B_SEGMENT_PTRS) != 0);
        if (out_path || image) { // the image is made once, straight into the returned buffer
            const auto t0 = std::chrono::steady_clock::now();
            const uint64_t size = cobsg::index_image_size(*ix);
            uint8_t* buf = static_cast<uint8_t*>(std::malloc(std::max<size_t>(size, 1)));
            if (!buf) throw std::bad_alloc();
            std::unique_ptr<uint8_t, decltype(&std::free)> hold(buf, &std::free);
            cobsg::index_image_into(*ix, buf);
            cobsg::note_image_ms(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            if (out_path) cobsg::write_image(buf, size, out_path);
            if (image) {
                *image = hold.release();
                *image_len = size;
            }
        }
        if (index_out) {
            auto h = std::make_unique<cobs_gpu_index>();
            h->ix = std::move(ix);
            *index_out = h.release();
        }
    });
}

int cobs_gpu_build(const uint8_t* seqs, const uint64_t* seg_offsets, uint64_t n_segs,
                   const uint64_t* doc_segs, const char* const* names, uint64_t n_docs,
                   const cobs_index_params* params, int kind, uint64_t forced_w, int device,
                   const char* out_path, uint8_t** image, uint64_t* image_len, char* err,
                   size_t errlen) {
    return cobs_gpu_build_ex(seqs, seg_offsets, n_segs, doc_segs, names, n_docs, params, kind,
                             forced_w, device, 0, out_path, image, image_len, nullptr, err, errlen);
}

int cobs_gpu_merge_classic(const cobs_gpu_index* a, const cobs_gpu_index* b, int device,
                           cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::merge_classic(*a->ix, *b->ix, device);
        *out = h.release();
    });
}

int cobs_gpu_query_fasta(cobs_gpu_index* index, const char* fasta_path, double K, uint64_t top_t,
                         char** tsv, uint64_t* tsv_len, char* err, size_t errlen) {
    *tsv = nullptr;
    *tsv_len = 0;
    return guarded(err, errlen, [&] {
        std::string out = cobsg::query_fasta_tsv(*index->ix, fasta_path, K, top_t);
        *tsv = static_cast<char*>(std::malloc(out.size() + 1));
        if (!*tsv) throw std::bad_alloc();
        std::memcpy(*tsv, out.c_str(), out.size() + 1);
        *tsv_len = out.size();
    });
}

int cobs_gpu_build_files(const char* const* inputs, uint64_t n_inputs, const cobs_index_params* params,
                         int kind, int format, int device, const char* out_path, uint8_t** image,
                         uint64_t* image_len, char* err, size_t errlen) {
    if (image) *image = nullptr;
    if (image_len) *image_len = 0;
    return guarded(err, errlen, [&] {
        if (format < COBS_FORMAT_AUTO || format > COBS_FORMAT_TEXT) throw cobsg::UsageError("unknown input format");
        std::vector<std::string> in(inputs, inputs + n_inputs);
        std::vector<uint8_t> img =
            cobsg::build_from_files(in, to_params(params), static_cast<uint8_t>(kind), format, device);
        if (out_path) cobsg::write_image(img, out_path);
        if (image) {
            *image = static_cast<uint8_t*>(std::malloc(std::max<size_t>(img.size(), 1)));
            if (!*image) throw std::bad_alloc();
            std::memcpy(*image, img.data(), img.size());
            *image_len = img.size();
        }
    });
}

int cobs_gpu_build_timing(double* ms_count, double* ms_fill, double* ms_total) {
    const cobsg::BuildTiming& t = cobsg::last_build_timing();
    if (ms_count) *ms_count = t.ms_count;
    if (ms_fill) *ms_fill = t.ms_fill;
    if (ms_total) *ms_total = t.ms_total;
    return COBS_OK;
}

int cobs_gpu_build_timing_ex(double* ms_h2d, double* ms_count, double* ms_fill, double* ms_d2h,
                             double* ms_total) {
    const cobsg::BuildTiming& t = cobsg::last_build_timing();
    if (ms_h2d) *ms_h2d = t.ms_h2d;
    if (ms_count) *ms_count = t.ms_count;
    if (ms_fill) *ms_fill = t.ms_fill;
    if (ms_d2h) *ms_d2h = t.ms_d2h;
    if (ms_total) *ms_total = t.ms_total;
    return COBS_OK;
}

int cobs_gpu_build_timing_count(double* ms_kernels, double* ms_alloc, double* ms_free) {
    const cobsg::BuildTiming& t = cobsg::last_build_timing();
    if (ms_kernels) *ms_kernels = t.ms_count_kernels;
    if (ms_alloc) *ms_alloc = t.ms_count_alloc;
    if (ms_free) *ms_free = t.ms_count_free;
    return COBS_OK;
}

uint64_t cobs_gpu_trim(void) { return cobsg::trim_device_caches(); }

void cobs_gpu_free(void* p) { std::free(p); }

int cobs_gpu_index_synth_c5(uint64_t seed, uint64_t n_docs, uint64_t block_size, double median,
                            double sigma, double p, int device, cobs_gpu_index** out, char* err,
                            size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::synth_c5_index(seed, n_docs, block_size, median, sigma, p, device);
        *out = h.release();
    });
}

int cobs_gpu_index_synth_c5_blocks(uint64_t seed, uint64_t n_docs, uint64_t block_size, double median,
                                   double sigma, double p, uint64_t block_lo, uint64_t block_hi, int device,
                                   cobs_gpu_index** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(err, errlen, [&] {
        auto h = std::make_unique<cobs_gpu_index>();
        h->ix = cobsg::synth_c5_index(seed, n_docs, block_size, median, sigma, p, device, block_lo, block_hi);
        *out = h.release();
    });
}

int cobs_gpu_synth_docs(uint64_t seed, int alpha, const uint64_t* doc_len, uint64_t doc_lo,
                        uint64_t doc_hi, uint8_t* dev_out, int device) {
    return guarded(nullptr, 0, [&] { cobsg::synth_docs(seed, alpha, doc_len, doc_lo, doc_hi, dev_out, device); });
}

int cobs_gpu_calibrate(int device, uint64_t bytes, double* stream_gbs, double* random128_gbs) {
    return guarded(nullptr, 0, [&] { cobsg::calibrate(device, bytes, stream_gbs, random128_gbs); });
}

} // extern "C"
