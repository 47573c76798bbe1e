// Device-resident COBS index (the HBM equivalent of the reference's
// ResidentView, proj/src/storage.cpp:301-318) and the per-batch query
// workspace.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dev.cuh"

namespace cobsg {

// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    ~DevBuf();
};

struct PinnedBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    ~PinnedBuf();
};

struct QueryWorkspace {
    DevBuf pats, offs, win_base, tab_off, gtab, hashes, ell, skipped, tau;
    DevBuf hit_count, hit_total, hit_q, hit_doc, hit_score;
    DevBuf key64, key64_alt, key32, key32_alt, perm, perm_alt, out_doc, out_score;
    DevBuf scores, cub_tmp;
    PinnedBuf h_small;
    uint64_t hit_cap = 0;
};

struct DeviceIndex {
    IndexMeta meta;
    int device = 0;
    cudaStream_t stream = nullptr;      // the handle's own stream
    cudaStream_t user_stream = nullptr; // caller-owned override
    cudaStream_t work_stream() const { return user_stream ? user_stream : stream; }
    uint8_t* payload = nullptr; // pitched rows of every block
    uint64_t payload_bytes = 0;
    std::vector<DevBlock> blocks;
    DevBlock* d_blocks = nullptr;
    // column tasks: (block, 1024-document slice)
    std::vector<uint32_t> ct_block, ct_slice;
    uint32_t* d_ct = nullptr; // [2*nct]: block, slice
    uint32_t* d_name_rank = nullptr;
    uint64_t sum_row_bytes = 0; // sum_b row_bytes_b
    bool evict_first = false;   // payload far larger than L2
    std::mutex mu;
    QueryWorkspace ws;

    ~DeviceIndex();
    // Set up blocks / tasks / ranks from `meta` and allocate the payload.
    void allocate();
    void finish_upload(); // block table, tasks, ranks -> HBM
};

// Open from a byte source: parse, allocate, stream rows into pitched HBM.
std::unique_ptr<DeviceIndex> open_index(const ByteSource& src, int device);
// Config-5 procedural index generated in HBM.
std::unique_ptr<DeviceIndex> synth_c5_index(uint64_t seed, uint64_t n_docs, uint64_t block_size,
                                            double median, double sigma, double p, int device);

struct QueryResults {
    uint64_t n = 0;
    std::vector<uint32_t> ell, tau;
    std::vector<uint64_t> skipped;
    std::vector<int> status;
    std::vector<std::string> message;
    std::vector<uint64_t> hit_off, hit_n; // per query, into doc/score (after top_t)
    std::vector<uint32_t> doc, score;
    std::vector<uint8_t> scores; // dense, n x D x score_bytes
    uint32_t score_bytes = 2;
    double ms_termize = 0, ms_gather = 0, ms_order = 0, ms_total = 0;
    uint32_t launches = 0; // kernels of ours launched by the batch
    uint64_t row_bytes = 0;
};

// The batch query path (kernels 1-3).  Throws UsageError for bad K.
void query_batch(DeviceIndex& ix, const uint8_t* patterns, const uint64_t* offsets, uint64_t n,
                 double K, uint64_t top_t, uint32_t flags, QueryResults& out);

} // namespace cobsg
