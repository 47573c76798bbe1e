// cobs_gpu_binding.hpp -- the binding a reference maintainer adds to the
// reference tree (e.g. as proj/include/cobs/gpu.hpp) to put the B200 path
// behind the reference's OWN C++ interface.  It compiles against the
// reference headers (proj/include/cobs) and links libcobs_gpu.so; it is not
// part of this repo's product library (which has no reference dependency).
//
//  * cobs::gpu::DeviceIndexView is a cobs::IndexView (index_view.hpp:18-47)
//    whose payload lives in HBM.  Every reference caller that takes an
//    IndexView -- cobs::query (query.hpp:46-47), cobs::write_index
//    (storage.hpp:14), cobs::run_validation / oracle_query (validate.hpp) --
//    runs on it unchanged; row_data (index_view.hpp:37-42) is served by a D2H
//    copy into the caller's scratch, or, after mirror(), from a host copy of
//    the payload read back once.
//  * cobs::gpu::open_resident / open_random_access mirror storage.hpp:19,23.
//  * cobs::gpu::query / query_batch are the device engine with cobs::query's
//    signature and exceptions (query.cpp:123-164): the drop-in for the CLI's
//    batch loop (cli.cpp:205-221).
//  * cobs::gpu::build_classic / build_compact take the reference's TermSets
//    (classic_index.hpp:37-44, compact_index.hpp:26-27) and return the index
//    resident in HBM; cobs::gpu::merge_classic mirrors classic_index.hpp:46-49.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "cobs/error.hpp"
#include "cobs/index_view.hpp"
#include "cobs/query.hpp"
#include "cobs/termizer.hpp"
#include "cobs_gpu.h"

namespace cobs::gpu {

// C-ABI return codes -> the reference's exception taxonomy (cli.cpp:448-454)
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] inline void raise(int rc, const char* err) {
    if (rc == COBS_EDATA) throw DataError(err);
    if (rc == COBS_EUSAGE) throw std::invalid_argument(err);
    throw DeviceError(err);
}

inline void check(int rc, const char* err) {
    if (rc != COBS_OK) raise(rc, err);
}

class DeviceIndexView final : public IndexView {
public:
    //! Takes ownership of an open C-ABI handle.
    explicit DeviceIndexView(cobs_gpu_index* h) : h_(h) {
        cobs_index_params c{};
        cobs_gpu_index_params(h_, &c);
        params_.q = c.q;
        params_.k = c.k;
        params_.p = c.p;
        params_.canonical = c.canonical != 0;
        params_.block_size = c.block_size;
        params_.hash_scheme = c.hash_scheme;
        const uint64_t nb = cobs_gpu_index_block_count(h_);
        base_.push_back(0);
        for (uint64_t b = 0; b < nb; ++b) {
            const uint64_t dc = cobs_gpu_index_doc_count(h_, b);
            widths_.push_back(cobs_gpu_index_width(h_, b));
            for (uint64_t i = 0; i < dc; ++i) {
                const char* name = nullptr;
                uint64_t len = 0, tc = 0;
                cobs_gpu_index_doc(h_, b, i, &name, &len, &tc);
                docs_.push_back(DocEntry{std::string(name, len), tc});
            }
            base_.push_back(docs_.size());
        }
    }
    ~DeviceIndexView() override { cobs_gpu_index_close(h_); }
    DeviceIndexView(const DeviceIndexView&) = delete;
    DeviceIndexView& operator=(const DeviceIndexView&) = delete;

    const IndexParams& params() const override { return params_; }
    uint8_t kind() const override { return cobs_gpu_index_kind(h_); }
    size_t block_count() const override { return widths_.size(); }
    uint64_t doc_count(size_t b) const override { return base_[b + 1] - base_[b]; }
    uint64_t width(size_t b) const override { return widths_[b]; }
    const DocEntry& doc(size_t b, uint64_t i) const override { return docs_[base_[b] + i]; }

    const uint8_t* row_data(size_t b, uint64_t r, size_t lo, size_t hi, uint8_t* scratch) const override {
        if (b >= widths_.size() || r >= widths_[b] || lo > hi || hi > row_bytes(b))
            throw std::out_of_range("row_data: out of range");
        if (!mirror_.empty()) return mirror_.data() + block_off_[b] + r * row_bytes(b) + lo;
        if (hi == lo) return scratch;
        if (cobs_gpu_index_row(h_, b, r, lo, hi, scratch) != COBS_OK)
            throw DeviceError("row_data: device read failed");
        return scratch;
    }

    //! Read the whole payload back once; row_data is then served from host
    //! memory (pointers into it, like ResidentView, storage.cpp:309-314).
    void mirror() {
        uint8_t* img = nullptr;
        uint64_t len = 0;
        char err[1024];
        check(cobs_gpu_index_image(h_, &img, &len, err, sizeof err), err);
        uint64_t payload = 0;
        block_off_.clear();
        for (size_t b = 0; b < widths_.size(); ++b) {
            block_off_.push_back(payload);
            payload += widths_[b] * row_bytes(b);
        }
        mirror_.assign(img + (len - payload), img + len); // payload is the file's tail
        cobs_gpu_free(img);
    }

    //! Global column (file column order) -> document entry.
    const DocEntry& global_doc(uint64_t col) const { return docs_[col]; }
    cobs_gpu_index* handle() const { return h_; }
    bool streaming() const { return cobs_gpu_index_streaming(h_) != 0; }

private:
    cobs_gpu_index* h_;
    IndexParams params_;
    std::vector<uint64_t> widths_, base_, block_off_;
    std::vector<DocEntry> docs_;
    std::vector<uint8_t> mirror_;
};

//! storage.hpp:19 -- parse + validate (the reference's rejection matrix and
//! messages), upload to HBM.
inline std::unique_ptr<DeviceIndexView> open_resident(const std::string& path, int device = 0) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    check(cobs_gpu_index_open(path.c_str(), device, &h, err, sizeof err), err);
    return std::make_unique<DeviceIndexView>(h);
}

//! storage.hpp:23 -- an index larger than the HBM budget is streamed through
//! HBM per batch, read from the file every batch like the reference's
//! RandomAccessView (storage.cpp:320-341), or with from_file = false kept in
//! pinned host memory.
inline std::unique_ptr<DeviceIndexView> open_random_access(const std::string& path, uint64_t hbm_budget,
                                                           int device = 0, bool from_file = true) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    check(from_file ? cobs_gpu_index_open_file(path.c_str(), device, hbm_budget, &h, err, sizeof err)
                    : cobs_gpu_index_open_ex(path.c_str(), device, hbm_budget, &h, err, sizeof err),
          err);
    return std::make_unique<DeviceIndexView>(h);
}

//! cobs::query over a whole batch on the device (cli.cpp:205-221).  A pattern
//! without usable terms throws DataError from query(); here its message goes
//! to errors[i] (the CLI's inline ERR line) unless errors is null, in which
//! case the first such error is thrown.
inline std::vector<QueryResult> query_batch(const DeviceIndexView& index, const std::vector<std::string>& patterns,
                                            const QueryOptions& opts, std::vector<std::string>* errors = nullptr) {
    std::string bytes;
    std::vector<uint64_t> off{0};
    for (const std::string& p : patterns) {
        bytes += p;
        off.push_back(bytes.size());
    }
    char err[1024];
    cobs_gpu_results* r = nullptr;
    check(cobs_gpu_query_batch(index.handle(), reinterpret_cast<const uint8_t*>(bytes.data()), off.data(),
                               patterns.size(), opts.K, opts.top_t, COBS_Q_HITS, &r, err, sizeof err),
          err);
    std::unique_ptr<cobs_gpu_results, void (*)(cobs_gpu_results*)> guard(r, cobs_gpu_results_free);
    std::vector<QueryResult> out(patterns.size());
    if (errors) errors->assign(patterns.size(), std::string());
    for (uint64_t i = 0; i < patterns.size(); ++i) {
        uint64_t ell = 0, skipped = 0, n = 0;
        int status = 0;
        const char* msg = nullptr;
        cobs_gpu_results_query(r, i, &ell, &skipped, &status, &msg, &n);
        if (status != COBS_OK) {
            if (!errors) throw DataError(msg);
            (*errors)[i] = msg;
            continue;
        }
        out[i].ell = ell;
        out[i].skipped = skipped;
        const uint32_t *docs = nullptr, *scores = nullptr;
        cobs_gpu_results_hits(r, i, &docs, &scores);
        out[i].hits.reserve(n);
        for (uint64_t j = 0; j < n; ++j) out[i].hits.push_back({index.global_doc(docs[j]).name, scores[j]});
    }
    return out;
}

//! cobs::query (query.hpp:46-47) on the device: same result, same
//! exceptions (invalid_argument for K outside (0,1], DataError for l = 0).
inline QueryResult query(const DeviceIndexView& index, std::string_view pattern, const QueryOptions& opts = {}) {
    return std::move(query_batch(index, {std::string(pattern)}, opts, nullptr)[0]);
}

namespace detail {
inline std::unique_ptr<DeviceIndexView> build(const std::vector<TermSet>& documents, const IndexParams& params,
                                              int kind, uint64_t forced_w, int device) {
    // the terms stay where they are: one pointer per term (COBS_B_SEGMENT_PTRS)
    std::vector<const uint8_t*> terms;
    std::vector<uint64_t> seg{0}, doc_segs{0};
    std::vector<const char*> names;
    for (const TermSet& d : documents) {
        for (const std::string& t : d.terms) {
            terms.push_back(reinterpret_cast<const uint8_t*>(t.data()));
            seg.push_back(seg.back() + t.size());
        }
        doc_segs.push_back(seg.size() - 1);
        names.push_back(d.name.c_str());
    }
    cobs_index_params c{};
    c.q = params.q;
    c.k = params.k;
    c.p = params.p;
    c.canonical = params.canonical ? 1 : 0;
    c.block_size = params.block_size;
    c.hash_scheme = params.hash_scheme;
    char err[1024];
    cobs_gpu_index* h = nullptr;
    check(cobs_gpu_build_ex(reinterpret_cast<const uint8_t*>(terms.data()), seg.data(), seg.size() - 1,
                            doc_segs.data(), names.data(), names.size(), &c, kind, forced_w, device,
                            COBS_B_TERMS | COBS_B_SEGMENT_PTRS,
                            nullptr, nullptr, nullptr, &h, err, sizeof err),
          err);
    return std::make_unique<DeviceIndexView>(h);
}
} // namespace detail

//! classic_index.hpp:37-39 (workers has no meaning on the device).
inline std::unique_ptr<DeviceIndexView> build_classic(const std::vector<TermSet>& documents,
                                                      const IndexParams& params, uint32_t /*workers*/ = 1,
                                                      uint64_t forced_w = 0, int device = 0) {
    return detail::build(documents, params, COBS_KIND_CLASSIC, forced_w, device);
}

//! compact_index.hpp:26-27
inline std::unique_ptr<DeviceIndexView> build_compact(const std::vector<TermSet>& documents,
                                                      const IndexParams& params, uint32_t /*workers*/ = 1,
                                                      int device = 0) {
    return detail::build(documents, params, COBS_KIND_COMPACT, 0, device);
}

//! classic_index.hpp:46-49, both inputs resident on `device`.
inline std::unique_ptr<DeviceIndexView> merge_classic(const DeviceIndexView& a, const DeviceIndexView& b,
                                                      int device = 0) {
    char err[1024];
    cobs_gpu_index* h = nullptr;
    check(cobs_gpu_merge_classic(a.handle(), b.handle(), device, &h, err, sizeof err), err);
    return std::make_unique<DeviceIndexView>(h);
}

} // namespace cobs::gpu
