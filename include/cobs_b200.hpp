// cobs_b200.hpp — header-only C++20 host API over the C-ABI (cobs_gpu.h),
// mirroring the reference's C++ interface for this path
// (/root/reference/proj/include/cobs: index_view.hpp, storage.hpp, query.hpp,
// classic_index.hpp, compact_index.hpp) with the same names, argument meaning
// and error behaviour: cobs_b200::DataError where the reference throws
// cobs::DataError, std::invalid_argument where it throws that.
//
// One difference of shape, not meaning: the device build fuses extract_terms
// (termizer.hpp:37-38) into build_classic / build_compact, so they take
// documents (name + content strings) instead of pre-extracted TermSets, and
// return a device-resident, queryable index.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "cobs_gpu.h"

namespace cobs_b200 {

// proj/include/cobs/error.hpp:12-14
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// device failure (no reference equivalent)
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
[[noreturn]] inline void raise(int rc, const char* err) {
    if (rc == COBS_EDATA) throw DataError(err);
    if (rc == COBS_EUSAGE) throw std::invalid_argument(err);
    throw DeviceError(err);
}
inline void check(int rc, const char* err) {
    if (rc != COBS_OK) raise(rc, err);
}
} // namespace detail

inline constexpr uint8_t kKindClassic = COBS_KIND_CLASSIC; // index_view.hpp:13
inline constexpr uint8_t kKindCompact = COBS_KIND_COMPACT; // index_view.hpp:14

// proj/include/cobs/params.hpp:17-38
struct IndexParams {
    uint32_t q = 31;
    uint32_t k = 1;
    double p = 0.3;
    bool canonical = false;
    uint64_t block_size = 1024;
    uint8_t hash_scheme = 0;
    bool operator==(const IndexParams&) const = default;
    cobs_index_params c() const {
        cobs_index_params x{};
        x.q = q;
        x.k = k;
        x.p = p;
        x.block_size = block_size;
        x.canonical = canonical ? 1 : 0;
        x.hash_scheme = hash_scheme;
        return x;
    }
};

// classic_index.hpp:15-20
struct DocEntry {
    std::string name;
    uint64_t term_count = 0;
    bool operator==(const DocEntry&) const = default;
};

// query.hpp:15-39
struct ScoredHit {
    std::string doc_name;
    uint64_t score = 0;
    bool operator==(const ScoredHit&) const = default;
};
struct QueryOptions {
    double K = 0.9;
    uint64_t top_t = 0;
    uint32_t workers = 1; // no meaning on the device; kept for signature parity
};
struct QueryResult {
    uint64_t ell = 0;
    uint64_t skipped = 0;
    std::vector<ScoredHit> hits;
};

// A document for the fused extract + build: termizer.hpp:37-38's arguments.
struct Document {
    std::string name;
    std::vector<std::string> content;
};

// IndexView (index_view.hpp:18-47) over an index resident in HBM (or
// host-resident in streaming mode).  Immutable; safe for concurrent queries
// (the library serialises calls on one handle).
class GpuIndexView {
public:
    explicit GpuIndexView(cobs_gpu_index* h) : h_(h) {
        for (uint64_t b = 0; b < block_count(); ++b)
            for (uint64_t i = 0; i < doc_count(b); ++i) {
                const char* name;
                uint64_t len, tc;
                cobs_gpu_index_doc(h_, b, i, &name, &len, &tc);
                docs_.push_back({std::string(name, len), tc});
            }
        block_base_.push_back(0);
        for (uint64_t b = 0; b < block_count(); ++b) block_base_.push_back(block_base_.back() + doc_count(b));
        cobs_index_params c;
        cobs_gpu_index_params(h_, &c);
        params_ = {c.q, c.k, c.p, c.canonical != 0, c.block_size, c.hash_scheme};
    }
    ~GpuIndexView() { cobs_gpu_index_close(h_); }
    GpuIndexView(const GpuIndexView&) = delete;
    GpuIndexView& operator=(const GpuIndexView&) = delete;

    const IndexParams& params() const { return params_; }
    uint8_t kind() const { return cobs_gpu_index_kind(h_); }
    size_t block_count() const { return cobs_gpu_index_block_count(h_); }
    uint64_t doc_count(size_t b) const { return cobs_gpu_index_doc_count(h_, b); }
    uint64_t width(size_t b) const { return cobs_gpu_index_width(h_, b); }
    size_t row_bytes(size_t b) const { return cobs_gpu_index_row_bytes(h_, b); }
    uint64_t total_docs() const { return docs_.size(); }
    const DocEntry& doc(size_t b, uint64_t i) const { return docs_[block_base_[b] + i]; }
    // bytes [lo, hi) of row r, copied from HBM into `scratch` (index_view.hpp:41-42)
    const uint8_t* row_data(size_t b, uint64_t r, size_t lo, size_t hi, uint8_t* scratch) const {
        if (cobs_gpu_index_row(h_, b, r, lo, hi, scratch) != COBS_OK)
            throw std::out_of_range("row_data: out of range");
        return scratch;
    }
    bool streaming() const { return cobs_gpu_index_streaming(h_) != 0; }
    const std::string& global_name(uint64_t col) const { return docs_[col].name; }
    cobs_gpu_index* handle() const { return h_; }

private:
    cobs_gpu_index* h_;
    IndexParams params_;
    std::vector<DocEntry> docs_;
    std::vector<uint64_t> block_base_;
};

// storage.hpp:19 — parse + validate (same rejection matrix), upload to HBM.
inline std::unique_ptr<GpuIndexView> open_resident(const std::string& path, int device = 0) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    detail::check(cobs_gpu_index_open(path.c_str(), device, &h, err, sizeof err), err);
    return std::make_unique<GpuIndexView>(h);
}

// storage.hpp:23 — for indexes larger than HBM: streamed per batch from
// pinned host memory, or (from_file) read from the file every batch.
inline std::unique_ptr<GpuIndexView> open_random_access(const std::string& path, uint64_t hbm_budget,
                                                        int device = 0, bool from_file = false) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    detail::check(from_file ? cobs_gpu_index_open_file(path.c_str(), device, hbm_budget, &h, err, sizeof err)
                            : cobs_gpu_index_open_ex(path.c_str(), device, hbm_budget, &h, err, sizeof err),
                  err);
    return std::make_unique<GpuIndexView>(h);
}

// Block sharding: blocks [block_lo, block_hi) of a compact
// index as a standalone compact index; column_offset() maps its columns to
// the file's.  Merge shard hit lists by (score desc, name asc), cut to top_t.
inline std::unique_ptr<GpuIndexView> open_blocks(const std::string& path, uint64_t block_lo, uint64_t block_hi,
                                                 int device = 0) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    detail::check(cobs_gpu_index_open_blocks(path.c_str(), device, block_lo, block_hi, &h, err, sizeof err), err);
    return std::make_unique<GpuIndexView>(h);
}
inline uint64_t column_offset(const GpuIndexView& v) { return cobs_gpu_index_column_offset(v.handle()); }

// storage.hpp:14 — byte-identical to the reference writer.
inline void write_index(const GpuIndexView& index, const std::string& path) {
    char err[1024];
    detail::check(cobs_gpu_index_write(index.handle(), path.c_str(), err, sizeof err), err);
}

// query() over a batch, the CLI batch mode's semantics (cli.cpp:205-221):
// a pattern without usable terms puts the reference's DataError message in
// errors[i] (if given) and leaves results[i] empty instead of aborting.
inline std::vector<QueryResult> query_batch(const GpuIndexView& index, const std::vector<std::string>& patterns,
                                            const QueryOptions& opts, std::vector<std::string>* errors) {
    std::string bytes;
    std::vector<uint64_t> off{0};
    for (const std::string& p : patterns) {
        bytes += p;
        off.push_back(bytes.size());
    }
    char err[1024];
    cobs_gpu_results* r = nullptr;
    detail::check(cobs_gpu_query_batch(index.handle(), reinterpret_cast<const uint8_t*>(bytes.data()),
                                       off.data(), patterns.size(), opts.K, opts.top_t, COBS_Q_HITS, &r,
                                       err, sizeof err),
                  err);
    std::unique_ptr<cobs_gpu_results, void (*)(cobs_gpu_results*)> guard(r, cobs_gpu_results_free);
    std::vector<QueryResult> out(patterns.size());
    if (errors) errors->assign(patterns.size(), std::string());
    for (uint64_t i = 0; i < patterns.size(); ++i) {
        uint64_t ell, skipped, n;
        int status;
        const char* msg;
        cobs_gpu_results_query(r, i, &ell, &skipped, &status, &msg, &n);
        out[i].ell = ell;
        out[i].skipped = skipped;
        if (status != COBS_OK) {
            if (errors) (*errors)[i] = msg;
            continue;
        }
        const uint32_t *docs, *scores;
        cobs_gpu_results_hits(r, i, &docs, &scores);
        for (uint64_t j = 0; j < n; ++j) out[i].hits.push_back({index.global_name(docs[j]), scores[j]});
    }
    return out;
}

// query.hpp:46-47: invalid_argument for K outside (0,1]; DataError when the
// pattern yields no terms (query.cpp:125-138).
inline QueryResult query(const GpuIndexView& index, std::string_view pattern, const QueryOptions& opts = {}) {
    std::vector<std::string> errors;
    std::vector<QueryResult> r = query_batch(index, {std::string(pattern)}, opts, &errors);
    if (!errors[0].empty()) throw DataError(errors[0]);
    return std::move(r[0]);
}

namespace detail {
inline std::unique_ptr<GpuIndexView> build(const std::vector<Document>& docs, const IndexParams& params, int kind,
                                           uint64_t forced_w, int device) {
    // the strings stay where they are: one pointer per string (COBS_B_SEGMENT_PTRS)
    std::vector<const uint8_t*> seqs;
    std::vector<uint64_t> seg{0}, doc_segs{0};
    std::vector<const char*> names;
    for (const Document& d : docs) {
        for (const std::string& c : d.content) {
            seqs.push_back(reinterpret_cast<const uint8_t*>(c.data()));
            seg.push_back(seg.back() + c.size());
        }
        doc_segs.push_back(seg.size() - 1);
        names.push_back(d.name.c_str());
    }
    cobs_index_params c = params.c();
    char err[1024];
    cobs_gpu_index* h = nullptr;
    check(cobs_gpu_build_ex(reinterpret_cast<const uint8_t*>(seqs.data()), seg.data(), seg.size() - 1,
                            doc_segs.data(), names.data(), names.size(), &c, kind, forced_w, device,
                            COBS_B_SEGMENT_PTRS,
                            nullptr, nullptr, nullptr, &h, err, sizeof err),
          err);
    return std::make_unique<GpuIndexView>(h);
}
} // namespace detail

// extract_terms + build_classic (classic_index.hpp:37-39): documents in input
// order, width forced_w or sized for the largest document.
inline std::unique_ptr<GpuIndexView> build_classic(const std::vector<Document>& docs, const IndexParams& params,
                                                   uint64_t forced_w = 0, int device = 0) {
    return detail::build(docs, params, kKindClassic, forced_w, device);
}

// extract_terms + build_compact (compact_index.hpp:26-27).
inline std::unique_ptr<GpuIndexView> build_compact(const std::vector<Document>& docs, const IndexParams& params,
                                                   int device = 0) {
    return detail::build(docs, params, kKindCompact, 0, device);
}

// classic_index.hpp:46-49
inline std::unique_ptr<GpuIndexView> merge_classic(const GpuIndexView& a, const GpuIndexView& b, int device = 0) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    detail::check(cobs_gpu_merge_classic(a.handle(), b.handle(), device, &h, err, sizeof err), err);
    return std::make_unique<GpuIndexView>(h);
}

// Releases the device memory kept between calls (the build's count workspace,
// cobs_gpu_trim); returns the bytes released.
inline uint64_t trim() { return cobs_gpu_trim(); }

} // namespace cobs_b200
