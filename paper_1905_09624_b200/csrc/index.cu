// Device-resident index: open (parse + pitched HBM upload) and the config-5
// procedural generator.  The HBM layout is described in DESIGN.md §3.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <numeric>
#include <thread>

#include <sys/mman.h>

#include "index.hpp"
#include "synth.h"

namespace cobsg {

void DevBuf::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    if (n == 0) return;
    cudaError_t e = cudaMalloc(&ptr, n);
    if (e == cudaErrorMemoryAllocation && trim_device_caches() > 0) { // the cached count workspace may be in the way
        cudaGetLastError();
        e = cudaMalloc(&ptr, n);
    }
    COBS_CUDA(e);
    bytes = n;
}
void DevBuf::release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
}
DevBuf::~DevBuf() {
    if (ptr) cudaFree(ptr);
}
void PinnedBuf::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    COBS_CUDA(cudaHostAlloc(&ptr, n, cudaHostAllocPortable)); // pinned for every device's context
    bytes = n;
}
PinnedBuf::~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
}

namespace {

// Process-wide pinned staging (two buffers, allocated once: cudaMallocHost of
// this size costs milliseconds, far more than a copy of it).
constexpr uint64_t kStageBytes = 64ull << 20;
struct StagePool {
    std::mutex mu;
    PinnedBuf buf[2];
};
StagePool& stage_pool() {
    static StagePool p;
    return p;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// f(lo, hi) over [0, n) split across up to 8 host threads (small n: inline)
template <typename F>
void host_parallel(uint64_t n, uint64_t grain, F&& f) {
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const uint64_t parts = std::min<uint64_t>(hw, (n + grain - 1) / std::max<uint64_t>(grain, 1));
    if (parts <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const uint64_t per = (n + parts - 1) / parts;
    for (uint64_t i = 1; i < parts; ++i)
        th.emplace_back([&, i] { f(std::min(n, i * per), std::min(n, (i + 1) * per)); });
    f(0, std::min(n, per));
    for (auto& t : th) t.join();
}

} // namespace

void h2d_staged(void* dst_dev, const void* src_host, uint64_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes <= (4ull << 20) || is_pinned(src_host)) {
        COBS_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    StagePool& P = stage_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    Event done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
    bool busy[2] = {false, false};
    const uint8_t* src = static_cast<const uint8_t*>(src_host);
    uint8_t* dst = static_cast<uint8_t*>(dst_dev);
    for (uint64_t off = 0, i = 0; off < bytes; off += kStageBytes, ++i) {
        const int b = static_cast<int>(i & 1);
        const uint64_t len = std::min(kStageBytes, bytes - off);
        P.buf[b].reserve(kStageBytes);
        if (busy[b]) COBS_CUDA(cudaEventSynchronize(done[b])); // its last DMA has drained
        uint8_t* stage = P.buf[b].as<uint8_t>();
        host_parallel(len, 8ull << 20, [&](uint64_t lo, uint64_t hi) { std::memcpy(stage + lo, src + off + lo, hi - lo); });
        COBS_CUDA(cudaMemcpyAsync(dst + off, stage, len, cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaEventRecord(done[b], st));
        busy[b] = true;
    }
    for (int b = 0; b < 2; ++b)
        if (busy[b]) COBS_CUDA(cudaEventSynchronize(done[b])); // the pool is reused after return
}

void h2d_gather_staged(void* dst_dev, const uint8_t* const* seg_ptrs, const uint64_t* seg_off, uint64_t n_segs,
                       cudaStream_t st) {
    const uint64_t bytes = n_segs ? seg_off[n_segs] - seg_off[0] : 0;
    if (bytes == 0) return;
    StagePool& P = stage_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    Event done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
    bool busy[2] = {false, false};
    uint8_t* dst = static_cast<uint8_t*>(dst_dev);
    const uint64_t base = seg_off[0];
    for (uint64_t off = 0, i = 0; off < bytes; off += kStageBytes, ++i) {
        const int b = static_cast<int>(i & 1);
        const uint64_t len = std::min(kStageBytes, bytes - off);
        P.buf[b].reserve(kStageBytes);
        if (busy[b]) COBS_CUDA(cudaEventSynchronize(done[b])); // its last DMA has drained
        uint8_t* stage = P.buf[b].as<uint8_t>();
        // packed bytes [off + lo, off + hi) from the strings that hold them
        host_parallel(len, 8ull << 20, [&](uint64_t lo, uint64_t hi) {
            uint64_t pos = base + off + lo;
            const uint64_t end = base + off + hi;
            uint64_t s = static_cast<uint64_t>(std::upper_bound(seg_off, seg_off + n_segs + 1, pos) - seg_off) - 1;
            while (pos < end) {
                const uint64_t take = std::min(end, seg_off[s + 1]) - pos;
                if (take) std::memcpy(stage + (pos - base - off), seg_ptrs[s] + (pos - seg_off[s]), take);
                pos += take;
                ++s;
            }
        });
        COBS_CUDA(cudaMemcpyAsync(dst + off, stage, len, cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaEventRecord(done[b], st));
        busy[b] = true;
    }
    for (int b = 0; b < 2; ++b)
        if (busy[b]) COBS_CUDA(cudaEventSynchronize(done[b])); // the pool is reused after return
}

void* result_alloc(size_t bytes) {
    constexpr size_t kHuge = 2u << 20;
    if (bytes < kHuge) {
        void* p = std::malloc(std::max<size_t>(bytes, 1));
        if (!p) throw std::bad_alloc();
        return p;
    }
    const size_t len = (bytes + kHuge - 1) / kHuge * kHuge;
    void* p = std::aligned_alloc(kHuge, len);
    if (!p) throw std::bad_alloc();
    madvise(p, len, MADV_HUGEPAGE); // best effort
    return p;
}
void result_free(void* p) noexcept { std::free(p); }

void d2h_staged(void* dst_host, const void* src_dev, uint64_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes <= (4ull << 20) || is_pinned(dst_host)) {
        COBS_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        return;
    }
    StagePool& P = stage_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    Event done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
    const uint8_t* src = static_cast<const uint8_t*>(src_dev);
    uint8_t* dst = static_cast<uint8_t*>(dst_host);
    const uint64_t nchunks = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](uint64_t c) {
        const int b = static_cast<int>(c & 1);
        P.buf[b].reserve(kStageBytes);
        COBS_CUDA(cudaMemcpyAsync(P.buf[b].ptr, src + c * kStageBytes, std::min(kStageBytes, bytes - c * kStageBytes),
                                  cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaEventRecord(done[b], st));
    };
    issue(0);
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int b = static_cast<int>(c & 1);
        COBS_CUDA(cudaEventSynchronize(done[b]));
        if (c + 1 < nchunks) issue(c + 1); // the next chunk's DMA runs while this one is copied out
        const uint8_t* stage = P.buf[b].as<uint8_t>();
        const uint64_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
        host_parallel(len, 8ull << 20, [&](uint64_t lo, uint64_t hi) { std::memcpy(dst + off + lo, stage + lo, hi - lo); });
    }
}

void d2h_unpitch(void* dst_host, const uint8_t* src_dev, uint64_t rows, uint32_t row_bytes, uint32_t pitch,
                 cudaStream_t st) {
    if (rows == 0 || row_bytes == 0) return;
    uint8_t* dst = static_cast<uint8_t*>(dst_host);
    const uint64_t chunk_rows = std::max<uint64_t>(1, kStageBytes / pitch);
    if (pitch == row_bytes && is_pinned(dst_host)) {
        COBS_CUDA(cudaMemcpyAsync(dst, src_dev, rows * pitch, cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        return;
    }
    StagePool& P = stage_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    Event done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
    const uint64_t nchunks = (rows + chunk_rows - 1) / chunk_rows;
    auto issue = [&](uint64_t c) {
        const int b = static_cast<int>(c & 1);
        const uint64_t r0 = c * chunk_rows, n = std::min(chunk_rows, rows - r0);
        P.buf[b].reserve(kStageBytes);
        COBS_CUDA(cudaMemcpyAsync(P.buf[b].ptr, src_dev + r0 * pitch, n * pitch, cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaEventRecord(done[b], st));
    };
    issue(0);
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int b = static_cast<int>(c & 1);
        COBS_CUDA(cudaEventSynchronize(done[b]));
        if (c + 1 < nchunks) issue(c + 1); // the next chunk's DMA runs while this one is unpacked
        const uint64_t r0 = c * chunk_rows, n = std::min(chunk_rows, rows - r0);
        const uint8_t* stage = P.buf[b].as<uint8_t>();
        if (pitch == row_bytes)
            host_parallel(n * pitch, 8ull << 20, [&](uint64_t lo, uint64_t hi) {
                std::memcpy(dst + r0 * row_bytes + lo, stage + lo, hi - lo);
            });
        else
            host_parallel(n, (8ull << 20) / pitch + 1, [&](uint64_t lo, uint64_t hi) {
                for (uint64_t r = lo; r < hi; ++r)
                    std::memcpy(dst + (r0 + r) * row_bytes, stage + r * pitch, row_bytes);
            });
    }
}

DeviceIndex::~DeviceIndex() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (payload) cudaFree(payload);
    if (d_blocks) cudaFree(d_blocks);
    if (d_ct) cudaFree(d_ct);
    if (d_name_rank) cudaFree(d_name_rank);
    if (stream) cudaStreamDestroy(stream);
}

HostStream::~HostStream() {
    if (copy) cudaStreamSynchronize(copy);
    for (int i = 0; i < 2; ++i) {
        if (staging[i]) cudaFree(staging[i]);
        if (copied[i]) cudaEventDestroy(copied[i]);
        if (consumed[i]) cudaEventDestroy(consumed[i]);
    }
    if (d_slab_blocks) cudaFree(d_slab_blocks);
    if (d_slab_ct) cudaFree(d_slab_ct);
    if (host) cudaFreeHost(host);
    for (int i = 0; i < 2; ++i) {
        if (hstage[i]) cudaFreeHost(hstage[i]);
        if (h2d_done[i]) cudaEventDestroy(h2d_done[i]);
    }
    if (copy) cudaStreamDestroy(copy);
}

void HostStream::read_payload(uint64_t off, void* dst, uint64_t len) const {
    if (file_backed) {
        src.read_at(payload_start + off, dst, len);
        return;
    }
    // file layout [off, off + len) from the pitched host copy, row by row
    uint8_t* out = static_cast<uint8_t*>(dst);
    for (size_t b = 0; b < block_off.size() && len; ++b) {
        const DevBlock& d = (*layout)[b];
        const uint64_t bytes = d.w * d.rb;
        if (off >= block_off[b] + bytes) continue;
        uint64_t rel = off - block_off[b];
        while (len && rel < bytes) {
            const uint64_t r = rel / d.rb, c = rel - r * d.rb;
            const uint64_t n = std::min<uint64_t>(d.rb - c, len);
            std::memcpy(out, host + d.base + r * d.pitch + c, n);
            out += n;
            off += n;
            rel += n;
            len -= n;
        }
    }
}

void HostStream::stage_group(const std::vector<DevBlock>& blocks, size_t gi, uint8_t* dst) const {
    // work items: (slab, byte range of a direct slab | row range of a window slab)
    struct Item {
        uint32_t slab;
        uint64_t lo, hi;
    };
    constexpr uint64_t kPiece = 8ull << 20;
    std::vector<Item> items;
    const StreamGroup& G = groups[gi];
    for (uint32_t si = G.slab_lo; si < G.slab_hi; ++si) {
        const Slab& sl = slabs[si];
        const DevBlock& d = blocks[sl.block];
        if (sl.direct) {
            for (uint64_t o = 0; o < d.w * d.rb; o += kPiece) items.push_back({si, o, std::min(d.w * d.rb, o + kPiece)});
        } else {
            const uint64_t rows = std::max<uint64_t>(1, kPiece / d.rb);
            for (uint64_t r = 0; r < d.w; r += rows) items.push_back({si, r, std::min(d.w, r + rows)});
        }
    }
    std::atomic<size_t> next{0};
    std::exception_ptr failure;
    std::mutex fail_mu;
    auto work = [&] {
        std::vector<uint8_t> tmp;
        try {
            for (size_t i = next.fetch_add(1); i < items.size(); i = next.fetch_add(1)) {
                const Item& it = items[i];
                const Slab& sl = slabs[it.slab];
                const DevBlock& d = blocks[sl.block];
                if (sl.direct) {
                    read_payload(block_off[sl.block] + it.lo, dst + sl.base + it.lo, it.hi - it.lo);
                } else { // whole rows from the file, this slab's column window into the image
                    tmp.resize((it.hi - it.lo) * d.rb);
                    read_payload(block_off[sl.block] + it.lo * d.rb, tmp.data(), tmp.size());
                    for (uint64_t r = it.lo; r < it.hi; ++r)
                        std::memcpy(dst + sl.base + r * sl.pitch, tmp.data() + (r - it.lo) * d.rb + sl.s0 * 128ull,
                                    sl.width);
                }
            }
        } catch (...) {
            std::lock_guard<std::mutex> g(fail_mu);
            failure = std::current_exception();
        }
    };
    const size_t nt = std::min<size_t>(items.size(), std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    if (failure) std::rethrow_exception(failure);
}

void DeviceIndex::plan() {
    COBS_CUDA(cudaSetDevice(device));
    if (!stream) COBS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (meta.total_docs() >= (1ull << 32))
        throw DataError("index has more than 2^32 documents; the device path indexes columns in 32 bits");
    uint64_t off = 0;
    sum_row_bytes = 0;
    blocks.clear();
    ct_block.clear();
    ct_slice.clear();
    for (size_t b = 0; b < meta.blocks.size(); ++b) {
        const BlockMeta& m = meta.blocks[b];
        DevBlock d{};
        d.rb = static_cast<uint32_t>(m.row_bytes());
        d.pitch = (d.rb + 31u) & ~31u;
        d.w = m.w;
        d.magic = mod_magic(m.w);
        d.dc = static_cast<uint32_t>(m.doc_count);
        d.doc_base = static_cast<uint32_t>(m.doc_base);
        d.base = off;
        uint64_t bytes = m.w * d.pitch;
        if (m.w != 0 && bytes / m.w != d.pitch) throw DataError("block payload too large for the device");
        off += (bytes + 255) & ~255ull;
        sum_row_bytes += d.rb;
        blocks.push_back(d);
        uint32_t slices = (d.rb + 127u) / 128u;
        for (uint32_t s = 0; s < slices; ++s) {
            ct_block.push_back(static_cast<uint32_t>(b));
            ct_slice.push_back(s);
        }
    }
    payload_bytes = off;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    evict_first = payload_bytes > 4ull * static_cast<uint64_t>(l2);
}

void DeviceIndex::allocate() {
    plan();
    bool any_pad = false;
    for (const DevBlock& d : blocks) any_pad |= d.pitch != d.rb;
    size_t free_b = 0, total_b = 0;
    COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (payload_bytes + (256ull << 20) > free_b)
        throw DataError("index payload (" + std::to_string(payload_bytes) +
                        " bytes pitched) does not fit in free device memory (" +
                        std::to_string(free_b) + " bytes)");
    COBS_CUDA(cudaMalloc(&payload, std::max<uint64_t>(payload_bytes, 256)));
    if (any_pad) {
        for (const DevBlock& d : blocks)
            if (d.pitch != d.rb)
                COBS_CUDA(cudaMemsetAsync(payload + d.base, 0, d.w * d.pitch, stream));
    }
}

void DeviceIndex::finish_upload() {
    COBS_CUDA(cudaMalloc(&d_blocks, sizeof(DevBlock) * blocks.size()));
    COBS_CUDA(cudaMemcpyAsync(d_blocks, blocks.data(), sizeof(DevBlock) * blocks.size(),
                              cudaMemcpyHostToDevice, stream));
    std::vector<uint32_t> ct(2 * ct_block.size());
    for (size_t i = 0; i < ct_block.size(); ++i) {
        ct[2 * i] = ct_block[i];
        ct[2 * i + 1] = ct_slice[i];
    }
    COBS_CUDA(cudaMalloc(&d_ct, sizeof(uint32_t) * std::max<size_t>(ct.size(), 2)));
    COBS_CUDA(cudaMemcpyAsync(d_ct, ct.data(), sizeof(uint32_t) * ct.size(), cudaMemcpyHostToDevice,
                              stream));
    std::vector<uint32_t> rank = meta.name_ranks();
    COBS_CUDA(cudaMalloc(&d_name_rank, sizeof(uint32_t) * std::max<size_t>(rank.size(), 1)));
    COBS_CUDA(cudaMemcpyAsync(d_name_rank, rank.data(), sizeof(uint32_t) * rank.size(),
                              cudaMemcpyHostToDevice, stream));
    COBS_CUDA(cudaStreamSynchronize(stream));
}

namespace {

// Host-resident mode: read the payload into pinned memory, cut blocks into
// slabs of whole 1,024-document slices that fit half the budget, pack slabs
// into groups (one staging buffer each), upload the slab tables.
void open_streaming(DeviceIndex& ix, const ByteSource& src, uint64_t budget, bool file_backed) {
    auto hs = std::make_unique<HostStream>();
    const IndexMeta& m = ix.meta;
    hs->host_bytes = m.file_size - m.payload_start;
    hs->payload_start = m.payload_start;
    hs->file_backed = file_backed;
    for (size_t b = 0; b < ix.blocks.size(); ++b) hs->block_off.push_back(m.blocks[b].offset - m.payload_start);
    if (file_backed) {
        hs->src = src;
    } else { // pitched, mapped pinned copy: rows read in 64 MB pieces, re-pitched by host threads
        COBS_CUDA(cudaHostAlloc(&hs->host, std::max<uint64_t>(ix.payload_bytes, 1),
                                cudaHostAllocMapped | cudaHostAllocPortable));
        COBS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hs->host_dev), hs->host, 0));
        hs->layout = &ix.blocks;
        struct Piece { size_t b; uint64_t r0, r1; };
        std::vector<Piece> pieces;
        for (size_t b = 0; b < ix.blocks.size(); ++b) {
            const DevBlock& d = ix.blocks[b];
            const uint64_t rows = std::max<uint64_t>(1, (64ull << 20) / std::max<uint32_t>(d.rb, 1));
            for (uint64_t r = 0; r < d.w; r += rows) pieces.push_back({b, r, std::min(d.w, r + rows)});
        }
        std::atomic<size_t> next{0};
        std::exception_ptr failure;
        std::mutex fail_mu;
        auto work = [&] {
            std::vector<uint8_t> tmp;
            try {
                for (size_t i = next.fetch_add(1); i < pieces.size(); i = next.fetch_add(1)) {
                    const Piece& p = pieces[i];
                    const DevBlock& d = ix.blocks[p.b];
                    uint8_t* dst = hs->host + d.base + p.r0 * d.pitch;
                    if (d.pitch == d.rb) {
                        src.read_at(m.blocks[p.b].offset + p.r0 * d.rb, dst, (p.r1 - p.r0) * d.rb);
                        continue;
                    }
                    tmp.resize((p.r1 - p.r0) * d.rb);
                    src.read_at(m.blocks[p.b].offset + p.r0 * d.rb, tmp.data(), tmp.size());
                    for (uint64_t r = p.r0; r < p.r1; ++r) {
                        std::memcpy(dst + (r - p.r0) * d.pitch, tmp.data() + (r - p.r0) * d.rb, d.rb);
                        std::memset(dst + (r - p.r0) * d.pitch + d.rb, 0, d.pitch - d.rb);
                    }
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(fail_mu);
                failure = std::current_exception();
            }
        };
        const size_t nt = std::min<size_t>(pieces.size(), std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
        std::vector<std::thread> th;
        for (size_t t = 1; t < nt; ++t) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
        if (failure) std::rethrow_exception(failure);
    }
    const uint64_t half = (budget / 2) & ~255ull;
    hs->staging_bytes = half;
    std::vector<DevBlock> sblocks;
    std::vector<uint32_t> sct;
    StreamGroup g{0, 0, 0, 0};
    uint64_t used = 0;
    for (size_t b = 0; b < ix.blocks.size(); ++b) {
        const DevBlock& d = ix.blocks[b];
        const uint32_t nsl = (d.rb + 127u) / 128u;
        const uint64_t per_slice = d.w * 128ull;
        uint32_t s_max = static_cast<uint32_t>(std::max<uint64_t>(1, half / std::max<uint64_t>(per_slice, 1)));
        for (uint32_t s0 = 0; s0 < nsl; s0 += s_max) {
            Slab sl{};
            sl.block = static_cast<uint32_t>(b);
            sl.s0 = s0;
            sl.ns = std::min(s_max, nsl - s0);
            sl.width = std::min<uint32_t>(d.rb - s0 * 128u, sl.ns * 128u);
            // whole rows go over as one contiguous copy at the source's own
            // row stride (narrow 2D DMA rows crawl over PCIe): the pitched host
            // copy's pitch, or the file's row length when 4-byte aligned
            if (file_backed) {
                sl.direct = s0 == 0 && sl.width == d.rb && (d.rb & 3u) == 0;
                sl.pitch = sl.direct ? sl.width : ((sl.width + 31u) & ~31u);
            } else {
                sl.direct = s0 == 0 && sl.width == d.rb;
                sl.pitch = sl.direct ? d.pitch : ((sl.width + 31u) & ~31u);
            }
            const uint64_t bytes = ((d.w * sl.pitch) + 255) & ~255ull;
            if (bytes > half)
                throw DataError("block " + std::to_string(b) + " needs " + std::to_string(bytes) +
                                " bytes of HBM per slice, more than half the budget");
            if (used + bytes > half) { // close the group
                g.slab_hi = static_cast<uint32_t>(hs->slabs.size());
                g.ct_hi = static_cast<uint32_t>(sct.size() / 2);
                hs->groups.push_back(g);
                hs->group_bytes.push_back(used);
                g = StreamGroup{g.slab_hi, 0, g.ct_hi, 0};
                used = 0;
            }
            sl.base = used;
            used += bytes;
            DevBlock sd = d;
            sd.base = sl.base;
            sd.pitch = sl.pitch;
            sd.rb = sl.width;
            sd.dc = std::min<uint32_t>(d.dc - s0 * 1024u, sl.ns * 1024u);
            sd.doc_base = d.doc_base + s0 * 1024u;
            const uint32_t idx = static_cast<uint32_t>(hs->slabs.size());
            for (uint32_t j = 0; j < sl.ns; ++j) {
                sct.push_back(idx);
                sct.push_back(j);
            }
            hs->slabs.push_back(sl);
            sblocks.push_back(sd);
        }
    }
    g.slab_hi = static_cast<uint32_t>(hs->slabs.size());
    g.ct_hi = static_cast<uint32_t>(sct.size() / 2);
    if (g.slab_hi > g.slab_lo) {
        hs->groups.push_back(g);
        hs->group_bytes.push_back(used);
    }
    COBS_CUDA(cudaMalloc(&hs->d_slab_blocks, sizeof(DevBlock) * std::max<size_t>(sblocks.size(), 1)));
    COBS_CUDA(cudaMalloc(&hs->d_slab_ct, sizeof(uint32_t) * std::max<size_t>(sct.size(), 2)));
    COBS_CUDA(cudaMemcpy(hs->d_slab_blocks, sblocks.data(), sizeof(DevBlock) * sblocks.size(),
                         cudaMemcpyHostToDevice));
    COBS_CUDA(cudaMemcpy(hs->d_slab_ct, sct.data(), sizeof(uint32_t) * sct.size(), cudaMemcpyHostToDevice));
    for (int i = 0; i < 2; ++i) {
        if (file_backed) {
            COBS_CUDA(cudaHostAlloc(&hs->hstage[i], std::max<uint64_t>(half, 256), cudaHostAllocDefault));
            COBS_CUDA(cudaEventCreateWithFlags(&hs->h2d_done[i], cudaEventDisableTiming));
        }
        COBS_CUDA(cudaMalloc(&hs->staging[i], std::max<uint64_t>(half, 256)));
        COBS_CUDA(cudaEventCreateWithFlags(&hs->copied[i], cudaEventDisableTiming));
        COBS_CUDA(cudaEventCreateWithFlags(&hs->consumed[i], cudaEventDisableTiming));
    }
    COBS_CUDA(cudaStreamCreateWithFlags(&hs->copy, cudaStreamNonBlocking));
    ix.evict_first = true;
    ix.hs = std::move(hs);
}

} // namespace

namespace {

// Rows of every block into the pitched HBM payload through two pinned
// staging buffers (re-pitched on the copy engine), the next chunk read from
// the source while the previous one is copied.  src_offset[b]: file offset of
// block b's payload.
void upload_rows(DeviceIndex& ix, const ByteSource& src, const std::vector<uint64_t>& src_offset) {
    const size_t kStage = 64ull << 20;
    PinnedBuf stage[2];
    stage[0].reserve(kStage);
    stage[1].reserve(kStage);
    Event done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
    int cur = 0;
    bool used[2] = {false, false};
    for (size_t b = 0; b < ix.blocks.size(); ++b) {
        const DevBlock& d = ix.blocks[b];
        uint64_t rows_per = std::max<uint64_t>(1, kStage / d.rb);
        for (uint64_t r0 = 0; r0 < d.w; r0 += rows_per) {
            uint64_t rows = std::min(rows_per, d.w - r0);
            if (used[cur]) COBS_CUDA(cudaEventSynchronize(done[cur]));
            if (rows * d.rb > stage[cur].bytes) stage[cur].reserve(rows * d.rb);
            src.read_at(src_offset[b] + r0 * d.rb, stage[cur].ptr, rows * d.rb);
            uint8_t* dst = ix.payload + d.base + r0 * d.pitch;
            if (d.pitch == d.rb)
                COBS_CUDA(cudaMemcpyAsync(dst, stage[cur].ptr, rows * d.rb, cudaMemcpyHostToDevice, ix.stream));
            else
                COBS_CUDA(cudaMemcpy2DAsync(dst, d.pitch, stage[cur].ptr, d.rb, d.rb, rows, cudaMemcpyHostToDevice,
                                            ix.stream));
            COBS_CUDA(cudaEventRecord(done[cur], ix.stream));
            used[cur] = true;
            cur ^= 1;
        }
    }
    COBS_CUDA(cudaStreamSynchronize(ix.stream));
}

} // namespace

std::unique_ptr<DeviceIndex> open_index(const ByteSource& src, int device, uint64_t hbm_budget, bool file_backed) {
    auto ix = std::make_unique<DeviceIndex>();
    ix->meta = parse_index(src);
    ix->device = device;
    ix->plan();
    if (hbm_budget > 0 && ix->payload_bytes > hbm_budget) {
        open_streaming(*ix, src, hbm_budget, file_backed);
        ix->finish_upload();
        return ix;
    }
    ix->allocate();
    std::vector<uint64_t> offs;
    for (const BlockMeta& m : ix->meta.blocks) offs.push_back(m.offset);
    upload_rows(*ix, src, offs);
    ix->finish_upload();
    return ix;
}

std::unique_ptr<DeviceIndex> open_index_blocks(const ByteSource& src, int device, uint64_t block_lo,
                                               uint64_t block_hi) {
    IndexMeta full = parse_index(src);
    const uint64_t nb = full.blocks.size();
    if (!(block_lo < block_hi && block_hi <= nb))
        throw UsageError("open_blocks: block range [" + std::to_string(block_lo) + ", " + std::to_string(block_hi) +
                         ") outside [0, " + std::to_string(nb) + ")");
    if (full.kind != kKindCompact && !(block_lo == 0 && block_hi == nb))
        throw UsageError("open_blocks: block sharding needs a compact index");
    auto ix = std::make_unique<DeviceIndex>();
    IndexMeta& m = ix->meta;
    m.params = full.params;
    m.kind = full.kind;
    std::vector<uint64_t> offs;
    for (uint64_t b = block_lo; b < block_hi; ++b) {
        const BlockMeta& fb = full.blocks[b];
        offs.push_back(fb.offset);
        m.blocks.push_back(fb);
        m.docs.insert(m.docs.end(), full.docs.begin() + fb.doc_base, full.docs.begin() + fb.doc_base + fb.doc_count);
    }
    m.layout(); // offsets of the shard as a standalone file (for write / image)
    ix->column_offset = full.blocks[block_lo].doc_base;
    ix->device = device;
    ix->plan();
    ix->allocate();
    upload_rows(*ix, src, offs);
    ix->finish_upload();
    return ix;
}

// ---- config-5 procedural payload ---------------------------------------

__global__ void c5_fill_kernel(uint32_t* rows, uint64_t words, uint32_t words_per_row, uint64_t key,
                               uint32_t thr16, uint32_t dc) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < words;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = g / words_per_row;
        uint32_t wj = static_cast<uint32_t>(g - r * words_per_row);
        uint32_t v = 0;
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t)
            v |= (uint32_t)syn_c5_byte_k(key, r, 4u * wj + t, thr16, dc) << (8 * t);
        rows[g] = v;
    }
}

std::unique_ptr<DeviceIndex> synth_c5_index(uint64_t seed, uint64_t n, uint64_t B, double median,
                                            double sigma, double p, int device, uint64_t block_lo,
                                            uint64_t block_hi) {
    if (n == 0 || B == 0) throw UsageError("synth_c5: n_docs and block_size must be >= 1");
    const uint64_t nb_all = (n + B - 1) / B;
    if (block_hi > nb_all) block_hi = nb_all;
    if (!(block_lo < block_hi))
        throw UsageError("synth_c5: block range [" + std::to_string(block_lo) + ", " + std::to_string(block_hi) +
                         ") outside [0, " + std::to_string(nb_all) + ")");
    auto ix = std::make_unique<DeviceIndex>();
    ix->device = device;
    IndexMeta& m = ix->meta;
    m.kind = kKindCompact;
    m.params.q = 31;
    m.params.k = 1;
    m.params.p = p;
    m.params.canonical = false;
    m.params.block_size = B;
    std::vector<uint64_t> tc(n);
    syn_c5_term_counts(seed, n, median, sigma, tc.data());
    std::vector<uint64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<std::string> names(n);
    for (uint64_t i = 0; i < n; ++i) {
        char nm[24];
        int l = syn_c5_name(i, nm);
        names[i].assign(nm, static_cast<size_t>(l));
    }
    // (term_count, name) order: compact_index.cpp:27-30
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
        if (tc[a] != tc[b]) return tc[a] < tc[b];
        return names[a] < names[b];
    });
    // blocks [block_lo, block_hi) only: a block shard of the same index
    // (open_index_blocks semantics; column_offset maps its columns)
    const uint64_t nb = block_hi - block_lo;
    std::vector<uint32_t> thr(nb);
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = (block_lo + b) * B, hi = std::min(n, lo + B), mx = 0;
        BlockMeta bm;
        bm.doc_count = hi - lo;
        for (uint64_t i = lo; i < hi; ++i) {
            m.docs.push_back({names[order[i]], tc[order[i]]});
            mx = std::max(mx, tc[order[i]]);
        }
        bm.w = bloom::size_filter(mx, p, 1); // classic_index.cpp:61 per block
        thr[b] = syn_c5_thr16(bm.w, mx);
        m.blocks.push_back(bm);
    }
    m.layout();
    ix->column_offset = block_lo * B;
    ix->allocate();
    for (uint64_t b = 0; b < nb; ++b) {
        const DevBlock& d = ix->blocks[b];
        uint64_t words = d.w * (d.pitch / 4);
        c5_fill_kernel<<<148 * 16, 256, 0, ix->stream>>>(
            reinterpret_cast<uint32_t*>(ix->payload + d.base), words, d.pitch / 4,
            syn_c5_key(seed, block_lo + b), thr[b], d.dc);
        COBS_CUDA(cudaGetLastError());
    }
    ix->finish_upload();
    return ix;
}

} // namespace cobsg
