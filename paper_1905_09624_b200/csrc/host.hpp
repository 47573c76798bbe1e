// Host-side C++ core of the B200 COBS path: parameters, error taxonomy, the
// sizing math, and the FORMAT.md reader/writer.  Own implementation from
// /root/reference/proj/FORMAT.md and SPEC.md; citations are to the reference
// code whose behaviour each piece must match bit for bit.
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace cobsg {

// proj/include/cobs/error.hpp:12-14 — bad data; maps to exit/return code 2.
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// std::invalid_argument in the reference — maps to code 1.
struct UsageError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
// Device failure — code 4 (no reference equivalent).
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// proj/include/cobs/params.hpp:17-38
struct Params {
    uint32_t q = 31;
    uint32_t k = 1;
    double p = 0.3;
    bool canonical = false;
    uint64_t block_size = 1024;
    uint8_t hash_scheme = 0;

    void validate() const; // params.hpp:26-35
};

constexpr uint8_t kKindClassic = 0; // index_view.hpp:13
constexpr uint8_t kKindCompact = 1; // index_view.hpp:14

namespace bloom {
double fpr_approx(uint64_t w, uint32_t k, uint64_t v);  // bloom.cpp:42-48
uint64_t size_filter(uint64_t v, double p, uint32_t k); // bloom.cpp:50-66
uint64_t score_threshold(uint64_t ell, double K);       // bloom.cpp:120-123
} // namespace bloom

// Host twin of the device XXH64 (FORMAT.md "Term hashing").
uint64_t xxh64(const void* data, size_t len, uint64_t seed);

struct DocEntry {
    std::string name;
    uint64_t term_count = 0;
};

struct BlockMeta {
    uint64_t doc_count = 0;
    uint64_t w = 0;
    uint64_t offset = 0;   // absolute file offset of the payload
    uint64_t doc_base = 0; // global column of the block's first document
    uint64_t row_bytes() const { return (doc_count + 7) / 8; }
    uint64_t payload_bytes() const { return w * row_bytes(); }
};

// Everything in a COBS file except the payload rows.
struct IndexMeta {
    Params params;
    uint8_t kind = kKindClassic;
    std::vector<BlockMeta> blocks;
    std::vector<DocEntry> docs; // all documents, file column order
    uint64_t payload_start = 0;
    uint64_t file_size = 0;

    uint64_t total_docs() const { return docs.size(); }
    // Rank of each document's name in bytewise order (std::string <), used
    // for the (score desc, name asc) tie-break on the device.
    std::vector<uint32_t> name_ranks() const;
    // Header bytes (head + tables + offsets) exactly as the reference writer
    // emits them (storage.cpp:345-380); recomputes offsets/payload_start.
    std::vector<uint8_t> header_bytes() const;
    // Fill doc_base / offsets / payload_start / file_size from the tables.
    void layout();
};

// Random-access byte source for the parser (file via pread, or memory).
struct ByteSource {
    uint64_t size = 0;
    std::string path;
    std::function<void(uint64_t, void*, uint64_t)> read_at;
};
ByteSource file_source(const std::string& path); // storage.cpp:67-109 semantics
ByteSource memory_source(const uint8_t* data, uint64_t len, const std::string& path);

// parse_index (proj/src/storage.cpp:182-280): identical acceptance and
// rejection, DataError with the reference's messages.
IndexMeta parse_index(const ByteSource& src);

} // namespace cobsg
