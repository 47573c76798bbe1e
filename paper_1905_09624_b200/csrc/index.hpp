// Device-resident COBS index (the HBM equivalent of the reference's
// ResidentView, proj/src/storage.cpp:301-318) and the per-batch query
// workspace.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dev.cuh"
#include "host.hpp"

namespace cobsg {

// Grow-only device buffer (owning, move-only).
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void reserve(size_t n);
    void release(); // free now
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    ~DevBuf();
};

// Frees the device memory the library keeps between calls (the build's count
// workspace, see build.cu); DevBuf::reserve calls it and retries once when
// cudaMalloc runs out of memory.  Returns the bytes released.
size_t trim_device_caches();

struct PinnedBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    void reserve(size_t n);
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    ~PinnedBuf();
};

struct QueryWorkspace {
    DevBuf pats, offs, win_base, tab_off, gtab, hashes, ell, skipped, tau;
    DevBuf hit_count, hit_total, hit_q, hit_doc, hit_score, starts;
    DevBuf key64, key64_alt, key32, key32_alt, perm, perm_alt, out_doc, out_score;
    DevBuf scores, cub_tmp;
    PinnedBuf h_small;
    uint64_t hit_cap = 0;
};

// Host-resident (out-of-core) mode: the payload stays in
// pinned host memory (pitched) or in the index file, and a query batch either
// streams it through two HBM staging buffers in "slabs" (a block's rows
// restricted to a range of 1,024-document slices), copy of slab group g+1
// overlapping the gather of group g, or -- pinned, small batches -- reads
// only the addressed rows over PCIe (zero-copy).  The counterpart of the
// reference's random-access reader (storage.cpp:320-341) for indexes larger
// than HBM.
struct Slab {
    uint32_t block, s0, ns; // slices [s0, s0+ns) of `block`
    uint64_t base;          // offset inside the staging buffer
    uint32_t width, pitch;  // row bytes copied / device row stride
    bool direct;            // whole rows in one 1D copy (the source row stride == pitch)
};
struct StreamGroup {
    uint32_t slab_lo, slab_hi, ct_lo, ct_hi;
};
struct HostStream {
    // Pinned variant: the payload in mapped pinned host memory, in the
    // device's pitched layout (block b at DevBlock::base, rows DevBlock::pitch
    // apart, zero padding), so the gather can also read the addressed rows
    // straight over PCIe (zero-copy, host_dev) when a batch touches far less
    // than the whole payload.
    uint8_t* host = nullptr;         // pinned, mapped; pitched payload
    uint8_t* host_dev = nullptr;     // its device alias
    const std::vector<DevBlock>* layout = nullptr; // the pitched layout of `host`
    uint64_t host_bytes = 0;         // payload bytes in file layout
    std::vector<uint64_t> block_off; // file-layout payload offset of each block
    std::vector<Slab> slabs;
    std::vector<StreamGroup> groups;
    DevBlock* d_slab_blocks = nullptr;
    uint32_t* d_slab_ct = nullptr;   // (slab, local slice) pairs, group by group
    uint8_t* staging[2] = {nullptr, nullptr};
    uint64_t staging_bytes = 0;
    cudaStream_t copy = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    // File-backed variant: no host copy of the payload; each batch the host
    // reads every group from the file (threads: pread + repack into the
    // group's device layout, in a pinned image) and sends it with one DMA.
    bool file_backed = false;
    ByteSource src;                              // the index file (file-backed)
    uint64_t payload_start = 0;                  // file offset of the payload
    uint8_t* hstage[2] = {nullptr, nullptr};     // pinned group images
    cudaEvent_t h2d_done[2] = {nullptr, nullptr};
    bool hstage_busy[2] = {false, false};
    std::vector<uint64_t> group_bytes;           // staging bytes each group occupies
    // payload bytes [off, off + len) in file layout, from host memory or the file
    void read_payload(uint64_t off, void* dst, uint64_t len) const;
    // file-backed: group gi's slabs, in device-staging layout, into dst
    void stage_group(const std::vector<DevBlock>& blocks, size_t gi, uint8_t* dst) const;
    ~HostStream();
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
    uint64_t column_offset = 0; // block shard: file column of this index's first document
    bool evict_first = false;   // payload far larger than L2
    uint64_t free_hbm_seen = 0; // the last free-HBM reading of a query batch (0: none yet)
    std::mutex mu;
    QueryWorkspace ws;
    std::unique_ptr<HostStream> hs; // non-null: host-resident (streaming) mode
    bool streaming() const { return hs != nullptr; }

    ~DeviceIndex();
    // Block table, column tasks and pitched layout from `meta` (no memory).
    void plan();
    // plan() + allocate the pitched payload in HBM.
    void allocate();
    void finish_upload(); // block table, tasks, ranks -> HBM
};

// Host <-> device copies of large pageable host buffers through a cached
// pair of pinned staging buffers: host threads copy chunk i+1 between the
// caller's memory and pinned memory while the copy engine moves chunk i
// (the driver's own pageable path is one thread and a narrow 2D copy engine
// path is slower still).  Pinned sources/destinations are copied directly.
void h2d_staged(void* dst_dev, const void* src_host, uint64_t bytes, cudaStream_t st);
// The packed layout seg_off[0..n_segs] gathered from one host pointer per
// string (no packed host copy), through the same pinned staging pair.
void h2d_gather_staged(void* dst_dev, const uint8_t* const* seg_ptrs, const uint64_t* seg_off, uint64_t n_segs,
                       cudaStream_t st);
// Device -> pageable host through the same pinned pair, host threads copying
// chunk i out while chunk i+1 is in flight (the driver's pageable D2H path
// runs at ~2 GB/s into freshly allocated memory).  Synchronous.
void d2h_staged(void* dst_host, const void* src_dev, uint64_t bytes, cudaStream_t st);
// Rows [0, rows) of a pitched device matrix (row_bytes of each pitch-byte
// row) into a packed host array: pitched 1D chunks D2H, un-pitched by host
// threads (no narrow-row 2D copies).  Synchronous.
void d2h_unpitch(void* dst_host, const uint8_t* src_dev, uint64_t rows, uint32_t row_bytes, uint32_t pitch,
                 cudaStream_t st);

// Open from a byte source: parse, allocate, stream rows into pitched HBM.
// With hbm_budget > 0 and a pitched payload larger than it, open in the
// host-resident streaming mode with two staging buffers of hbm_budget/2.
std::unique_ptr<DeviceIndex> open_index(const ByteSource& src, int device, uint64_t hbm_budget = 0,
                                        bool file_backed = false);
// Blocks [block_lo, block_hi) of a compact index as a standalone compact
// index resident in HBM (SURVEY.md §8e block sharding): same params, those
// blocks and their documents; column_offset = the file column of its first
// document.  The whole header is parsed and validated as by open_index.
std::unique_ptr<DeviceIndex> open_index_blocks(const ByteSource& src, int device, uint64_t block_lo,
                                               uint64_t block_hi);
// Config-5 procedural index generated in HBM.
std::unique_ptr<DeviceIndex> synth_c5_index(uint64_t seed, uint64_t n_docs, uint64_t block_size,
                                            double median, double sigma, double p, int device,
                                            uint64_t block_lo = 0, uint64_t block_hi = ~0ull);

// Host memory for large result buffers: 2 MB aligned and advised for
// transparent huge pages (the first touch of fresh 4 KB pages costs more than
// the copy that fills them: ~0.3 s for 800 MB of hits).
void* result_alloc(size_t bytes);
void result_free(void* p) noexcept;

// std::vector storage without value-initialisation (result buffers that a
// device copy overwrites at once), large ones on huge pages
template <typename T>
struct NoInitAlloc : std::allocator<T> {
    template <typename U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <typename U>
    NoInitAlloc(const NoInitAlloc<U>&) {}
    T* allocate(size_t n) { return static_cast<T*>(result_alloc(n * sizeof(T))); }
    void deallocate(T* p, size_t) noexcept { result_free(p); }
    template <typename U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <typename U, typename... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <typename T>
using RawVec = std::vector<T, NoInitAlloc<T>>;

struct QueryResults {
    uint64_t n = 0;
    std::vector<uint32_t> ell, tau;
    std::vector<uint64_t> skipped;
    std::vector<int> status;
    std::vector<std::string> message;
    std::vector<uint64_t> hit_off, hit_n; // per query, into doc/score (after top_t)
    RawVec<uint32_t> doc, score;
    RawVec<uint8_t> scores; // dense, n x D x score_bytes
    uint32_t score_bytes = 2;
    double ms_termize = 0, ms_gather = 0, ms_order = 0, ms_total = 0;
    uint32_t launches = 0; // kernels of ours launched by the batch
    uint64_t h2d_index_bytes = 0; // host-resident modes: index bytes moved host -> GPU
    bool zero_copy = false;       // host-resident: rows read from mapped host memory
    uint64_t row_bytes = 0;
};

// The batch query path (kernels 1-3).  Throws UsageError for bad K.
void query_batch(DeviceIndex& ix, const uint8_t* patterns, const uint64_t* offsets, uint64_t n,
                 double K, uint64_t top_t, uint32_t flags, QueryResults& out);

} // namespace cobsg
