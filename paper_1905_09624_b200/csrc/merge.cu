// merge_classic on the device: column concatenation of two
// classic indexes with equal parameters and width
// (proj/src/classic_index.cpp:96-115, proj/src/bit_matrix.cpp:10-23).
//
// Byte-exact with the reference's BitMatrix::concat_columns: the left
// index's row bytes are copied verbatim; the right index's bits are either
// copied verbatim (left column count a multiple of 8, the memcpy branch) or
// OR-ed in bit by bit at column a.cols + c for c < b.cols (so its padding
// bits are not carried over).
#include <algorithm>

#include "index.hpp"
#include "merge.hpp"

namespace cobsg {

namespace {

__global__ void concat_kernel(const uint8_t* a, uint32_t pa, uint32_t ra, uint64_t ca, const uint8_t* b,
                              uint32_t pb, uint64_t cb, uint8_t* out, uint32_t po, uint32_t ro,
                              uint64_t rows) {
    const uint64_t total = rows * ro;
    const bool aligned = (ca & 7) == 0;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = g / ro;
        const uint32_t j = static_cast<uint32_t>(g - r * ro);
        const uint8_t* arow = a + r * pa;
        const uint8_t* brow = b + r * pb;
        uint32_t v = j < ra ? arow[j] : 0u; // memcpy(out.row(r), a.row(r), a.row_bytes())
        if (aligned) {
            if (j >= ra) v = brow[j - ra]; // memcpy of b's row (bit_matrix.cpp:16)
        } else {
            // out bit 8j+t <- b bit (8j+t-ca) for 0 <= 8j+t-ca < cb (bit_matrix.cpp:18-19)
            const int64_t c0 = static_cast<int64_t>(8ull * j) - static_cast<int64_t>(ca);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int64_t c = c0 + t;
                if (c >= 0 && c < static_cast<int64_t>(cb)) v |= ((brow[c >> 3] >> (c & 7)) & 1u) << t;
            }
        }
        out[r * po + j] = static_cast<uint8_t>(v);
    }
}

} // namespace

std::unique_ptr<DeviceIndex> merge_classic(const DeviceIndex& A, const DeviceIndex& B, int device) {
    const IndexMeta& a = A.meta;
    const IndexMeta& b = B.meta;
    if (A.streaming() || B.streaming())
        throw UsageError("merge: host-resident (streaming) indexes are not supported");
    if (a.kind != kKindClassic || b.kind != kKindClassic)
        throw UsageError("merge: only classic indexes can be merged");
    const Params &pa = a.params, &pb = b.params; // IndexParams::operator== (params.hpp:37)
    if (!(pa.q == pb.q && pa.k == pb.k && pa.p == pb.p && pa.canonical == pb.canonical &&
          pa.block_size == pb.block_size && pa.hash_scheme == pb.hash_scheme))
        throw DataError("merge: index parameters differ"); // classic_index.cpp:97-98
    const uint64_t wa = a.blocks[0].w, wb = b.blocks[0].w;
    if (wa != wb) // classic_index.cpp:99-101
        throw DataError("merge: widths differ (" + std::to_string(wa) + " vs " + std::to_string(wb) +
                        "); rebuild with a common forced width");
    { // classic_index.cpp:102-106 -> check_unique_names (:17-22)
        std::vector<const std::string*> names;
        for (const DocEntry& d : a.docs) names.push_back(&d.name);
        for (const DocEntry& d : b.docs) names.push_back(&d.name);
        std::sort(names.begin(), names.end(),
                  [](const std::string* x, const std::string* y) { return *x < *y; });
        for (size_t i = 1; i < names.size(); ++i)
            if (*names[i - 1] == *names[i]) throw DataError("duplicate document name: " + *names[i]);
    }
    if (A.device != device || B.device != device)
        throw UsageError("merge: both indexes must be resident on the output device");
    auto ix = std::make_unique<DeviceIndex>();
    ix->device = device;
    IndexMeta& m = ix->meta;
    m.params = pa;
    m.kind = kKindClassic;
    m.docs = a.docs;
    m.docs.insert(m.docs.end(), b.docs.begin(), b.docs.end());
    BlockMeta bm;
    bm.doc_count = m.docs.size();
    bm.w = wa;
    m.blocks.push_back(bm);
    m.layout();
    ix->allocate();
    const DevBlock &da = A.blocks[0], &db = B.blocks[0], &dout = ix->blocks[0];
    if (dout.pitch != dout.rb)
        COBS_CUDA(cudaMemsetAsync(ix->payload + dout.base, 0, dout.w * dout.pitch, ix->stream));
    const uint8_t* pa_dev = A.payload + da.base;
    const uint8_t* pb_dev = B.payload + db.base;
    if (dout.w * dout.rb > 0)
        concat_kernel<<<148 * 16, 256, 0, ix->stream>>>(pa_dev, da.pitch, da.rb, a.blocks[0].doc_count, pb_dev,
                                                        db.pitch, b.blocks[0].doc_count,
                                                        ix->payload + dout.base, dout.pitch, dout.rb, dout.w);
    COBS_CUDA(cudaGetLastError());
    COBS_CUDA(cudaStreamSynchronize(ix->stream));
    ix->finish_upload();
    return ix;
}

} // namespace cobsg
