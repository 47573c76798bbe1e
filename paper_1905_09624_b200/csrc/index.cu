// Device-resident index: open (parse + pitched HBM upload) and the config-5
// procedural generator.  The HBM layout is described in DESIGN.md §3.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "index.hpp"
#include "synth.h"

namespace cobsg {

void DevBuf::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    if (n == 0) return;
    COBS_CUDA(cudaMalloc(&ptr, n));
    bytes = n;
}
DevBuf::~DevBuf() {
    if (ptr) cudaFree(ptr);
}
void PinnedBuf::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    COBS_CUDA(cudaMallocHost(&ptr, n));
    bytes = n;
}
PinnedBuf::~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
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

void DeviceIndex::allocate() {
    COBS_CUDA(cudaSetDevice(device));
    COBS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (meta.total_docs() >= (1ull << 32))
        throw DataError("index has more than 2^32 documents; the device path indexes columns in 32 bits");
    uint64_t off = 0;
    sum_row_bytes = 0;
    blocks.clear();
    ct_block.clear();
    ct_slice.clear();
    bool any_pad = false;
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
        any_pad |= d.pitch != d.rb;
        sum_row_bytes += d.rb;
        blocks.push_back(d);
        uint32_t slices = (d.rb + 127u) / 128u;
        for (uint32_t s = 0; s < slices; ++s) {
            ct_block.push_back(static_cast<uint32_t>(b));
            ct_slice.push_back(s);
        }
    }
    payload_bytes = off;
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
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    evict_first = payload_bytes > 4ull * static_cast<uint64_t>(l2);
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

std::unique_ptr<DeviceIndex> open_index(const ByteSource& src, int device) {
    auto ix = std::make_unique<DeviceIndex>();
    ix->meta = parse_index(src);
    ix->device = device;
    ix->allocate();
    // Stream rows through two pinned staging buffers, re-pitching on the copy
    // engine (cudaMemcpy2DAsync), while the next chunk is read from the file.
    const size_t kStage = 64ull << 20;
    PinnedBuf stage[2];
    stage[0].reserve(kStage);
    stage[1].reserve(kStage);
    cudaEvent_t done[2];
    COBS_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    COBS_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    int cur = 0;
    bool used[2] = {false, false};
    for (size_t b = 0; b < ix->blocks.size(); ++b) {
        const DevBlock& d = ix->blocks[b];
        const BlockMeta& m = ix->meta.blocks[b];
        uint64_t rows_per = std::max<uint64_t>(1, kStage / d.rb);
        for (uint64_t r0 = 0; r0 < d.w; r0 += rows_per) {
            uint64_t rows = std::min(rows_per, d.w - r0);
            if (used[cur]) COBS_CUDA(cudaEventSynchronize(done[cur]));
            if (rows * d.rb > stage[cur].bytes) stage[cur].reserve(rows * d.rb);
            src.read_at(m.offset + r0 * d.rb, stage[cur].ptr, rows * d.rb);
            uint8_t* dst = ix->payload + d.base + r0 * d.pitch;
            if (d.pitch == d.rb)
                COBS_CUDA(cudaMemcpyAsync(dst, stage[cur].ptr, rows * d.rb, cudaMemcpyHostToDevice,
                                          ix->stream));
            else
                COBS_CUDA(cudaMemcpy2DAsync(dst, d.pitch, stage[cur].ptr, d.rb, d.rb, rows,
                                            cudaMemcpyHostToDevice, ix->stream));
            COBS_CUDA(cudaEventRecord(done[cur], ix->stream));
            used[cur] = true;
            cur ^= 1;
        }
    }
    COBS_CUDA(cudaStreamSynchronize(ix->stream));
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
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
                                            double sigma, double p, int device) {
    if (n == 0 || B == 0) throw UsageError("synth_c5: n_docs and block_size must be >= 1");
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
    uint64_t nb = (n + B - 1) / B;
    std::vector<uint32_t> thr(nb);
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = b * B, hi = std::min(n, lo + B), mx = 0;
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
    ix->allocate();
    for (uint64_t b = 0; b < nb; ++b) {
        const DevBlock& d = ix->blocks[b];
        uint64_t words = d.w * (d.pitch / 4);
        c5_fill_kernel<<<148 * 16, 256, 0, ix->stream>>>(
            reinterpret_cast<uint32_t*>(ix->payload + d.base), words, d.pitch / 4,
            syn_c5_key(seed, b), thr[b], d.dc);
        COBS_CUDA(cudaGetLastError());
    }
    ix->finish_upload();
    return ix;
}

} // namespace cobsg
