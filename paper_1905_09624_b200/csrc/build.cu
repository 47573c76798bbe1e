// Kernel 4: index construction on the device.
//
//   count pass  one thread per window (flattened over all documents, so
//               skewed document sizes load-balance): canonicalise, XXH64,
//               exact per-document distinct count through the lock-free set
//               of dev.cuh -> term_count   (termizer.cpp:103-129,
//               termizer.hpp:25)
//   host        classic width / compact (term_count, name) sort, blocks of
//               B, per-block widths        (classic_index.cpp:40-64,
//               compact_index.cpp:19-52, bloom.cpp:50-66)
//   fill pass   for every window and seed, bit (XXH64 % w_b, column)
//               (classic_index.cpp:26-36, bit_matrix.hpp:25-27): 32
//               consecutive columns of a block are one u32 per row, so waves
//               of such column "slabs" (L2-sized) are filled with atomicOr and
//               then copied into the pitched HBM layout of the query index
//               (a built index is queryable in place; the file payload is its
//               un-pitched D2H copy).  OR is idempotent, so every window is
//               filled, not just the distinct ones.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>

#include "build.hpp"
#include "dev.cuh"
#include "index.hpp"
#include "synth.h"

namespace cobsg {

namespace {

thread_local BuildTiming g_timing;

constexpr int kBRun = 8; // consecutive windows rolled by one thread

struct WinArgs {
    const uint8_t* seqs;
    const uint64_t* seg_off;   // n_segs+1 byte offsets into seqs
    const uint64_t* seg_rbase; // n_segs+1 prefix of runs (kBRun windows) per segment
    const uint32_t* seg_doc;   // document of each segment
    const uint64_t* doc_start; // byte offset of each document's first segment
    uint64_t seg_lo, seg_hi;   // segment range of this pass
    uint64_t r_lo, r_hi;       // run range of this pass
    uint32_t q, k;
    int canonical;
    uint32_t tag_mask; // all ones (tests may narrow it to force tag collisions)
};

// run g -> segment (seg_rbase[s] <= g < seg_rbase[s+1]), searched in [lo, hi)
__device__ __forceinline__ uint64_t find_seg_in(const WinArgs& a, uint64_t g, uint64_t lo, uint64_t hi) {
    while (hi - lo > 1) {
        uint64_t mid = (lo + hi) >> 1;
        if (a.seg_rbase[mid] <= g)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint64_t find_seg(const WinArgs& a, uint64_t g) {
    return find_seg_in(a, g, a.seg_lo, a.seg_hi);
}

// Runs are handed to CTAs in contiguous chunks so the segment range of a
// chunk is searched once (by one thread) and each run's search is over the
// few segments the chunk spans, not the whole corpus.
constexpr uint64_t kChunkRuns = 512;

// Calls f(j, dna, code) for the windows [j0, j1) of segment bytes `sb`
// (dna: all-ACGT window with q <= 32, code: its canonical/forward code).
template <int QC, typename F>
__device__ __forceinline__ void roll_windows(const uint8_t* sb, uint64_t j0, uint64_t j1, uint32_t q_rt,
                                             bool canonical, F&& f) {
    const uint32_t q = QC ? QC : q_rt;
    if (q <= 32) {
        Roller R(q);
        for (uint32_t i = 0; i + 1 < q; ++i) R.push(__ldg(sb + j0 + i));
        for (uint64_t j = j0; j < j1; ++j) {
            R.push(__ldg(sb + j + q - 1));
            f(j, R.dna(), canonical ? R.canon() : R.fwd);
        }
    } else {
        for (uint64_t j = j0; j < j1; ++j) f(j, false, 0ull);
    }
}

template <int QC>
__global__ void __launch_bounds__(256) count_kernel(WinArgs a, unsigned long long* tab,
                                                    const uint64_t* tab_off, const uint64_t* tab_slots,
                                                    unsigned long long* term_count) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t q = QC ? QC : a.q;
    __shared__ uint64_t s_seg[2];
    const uint64_t nchunks = (a.r_hi - a.r_lo + kChunkRuns - 1) / kChunkRuns;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t r0 = a.r_lo + c * kChunkRuns, r1 = min(a.r_hi, r0 + kChunkRuns);
    __syncthreads();
    if (threadIdx.x == 0) {
        s_seg[0] = find_seg(a, r0);
        s_seg[1] = find_seg(a, r1 - 1) + 1;
    }
    __syncthreads();
    const uint64_t slo = s_seg[0], shi = s_seg[1];
    for (uint64_t base = r0 + (threadIdx.x >> 5) * 32; base < r1; base += blockDim.x) {
        const uint64_t g = base + lane;
        uint32_t cnt = 0, doc = 0xffffffffu;
        if (g < r1) {
            const uint64_t s = find_seg_in(a, g, slo, shi);
            doc = a.seg_doc[s];
            const uint64_t len = a.seg_off[s + 1] - a.seg_off[s];
            const uint64_t W = len >= q ? len - q + 1 : 0;
            const uint64_t j0 = (g - a.seg_rbase[s]) * kBRun;
            const uint64_t j1 = min(W, j0 + kBRun);
            const uint8_t* sb = a.seqs + a.seg_off[s];
            const uint8_t* dbase = a.seqs + a.doc_start[doc];
            unsigned long long* t = tab + tab_off[doc];
            const uint64_t mask = tab_slots[doc] - 1;
            roll_windows<QC>(sb, j0, j1, q, a.canonical != 0, [&](uint64_t j, bool dna, uint64_t code) {
                const uint8_t* w = sb + j;
                const uint32_t pos = static_cast<uint32_t>(w - dbase);
                if (dna) { // the slot only needs a well-mixed hash of the exact code
                    cnt += set_insert_code(t, mask, mix_code(code), code);
                } else if (a.canonical) {
                    if (q <= 32 || !window_acgt(w, q)) return; // skipped (termizer.cpp:113-116)
                    const bool rc = choose_rc(w, q);
                    cnt += set_insert(t, mask, xxh64_term(w, q, rc, 0), pos, dbase, q, true, rc, a.tag_mask);
                } else {
                    const uint64_t h = xxh64_term(w, q, false, 0);
                    cnt += q <= 32 ? set_insert_tagged(t, mask, h, pos, dbase, q, a.tag_mask)
                                   : set_insert(t, mask, h, pos, dbase, q, false, false, a.tag_mask);
                }
            });
        }
        // one atomic per (warp, document)
        const unsigned peers = __match_any_sync(0xffffffffu, doc);
        const uint32_t sum = __reduce_add_sync(peers, cnt);
        if (g < r1 && sum && lane == (uint32_t)(__ffs(peers) - 1))
            atomicAdd(term_count + doc, (unsigned long long)sum);
    }
    }
}

// ---- slab fill: the bits of 32 consecutive columns of a block are one u32
// per row -- a dense "slab" of w words.  A wave of such slabs (sized to stay
// L2-resident) is filled with atomicOr, then copied into the matrix's 4-byte
// column positions (one strided u32 store per row), instead of random
// read-modify-writes straight into the whole (HBM-sized) matrix.

struct SlabDoc {
    uint64_t run_lo, seg_lo, seg_hi; // first run and segment range of the document
    uint64_t slab;                   // u32 index of its slab's row 0 in the wave buffer
    uint64_t w, magic;
    uint32_t bit;                    // column % 32
};
struct SlabGroup {
    uint64_t src;   // u32 index of row 0 in the wave buffer
    uint64_t dst;   // payload byte offset of (row 0, byte 4 * group)
    uint64_t w;
    uint32_t pitch;
};

template <int QC>
__global__ void __launch_bounds__(256) slab_fill_kernel(WinArgs a, const SlabDoc* docs,
                                                        const uint64_t* run_prefix, uint32_t ndocs,
                                                        unsigned int* slab) {
    const uint32_t q = QC ? QC : a.q;
    const uint64_t total = run_prefix[ndocs];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = ndocs; // run_prefix[lo] <= t < run_prefix[hi]
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (run_prefix[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        const SlabDoc D = docs[lo];
        const uint64_t g = D.run_lo + (t - run_prefix[lo]);
        const uint64_t s = find_seg_in(a, g, D.seg_lo, D.seg_hi);
        const uint64_t len = a.seg_off[s + 1] - a.seg_off[s];
        const uint64_t W = len >= q ? len - q + 1 : 0;
        const uint64_t j0 = (g - a.seg_rbase[s]) * kBRun;
        const uint64_t j1 = min(W, j0 + kBRun);
        const uint8_t* sb = a.seqs + a.seg_off[s];
        unsigned int* col = slab + D.slab;
        const unsigned int bit = 1u << D.bit;
        roll_windows<QC>(sb, j0, j1, q, a.canonical != 0, [&](uint64_t j, bool dna, uint64_t code) {
            const uint8_t* w = sb + j;
            if (dna) {
                for (uint32_t seed = 0; seed < a.k; ++seed)
                    atomicOr(col + fastmod(xxh64_code<QC>(code, q, seed), D.w, D.magic), bit);
            } else if (a.canonical) {
                if (q <= 32 || !window_acgt(w, q)) return;
                const bool rc = choose_rc(w, q);
                for (uint32_t seed = 0; seed < a.k; ++seed)
                    atomicOr(col + fastmod(xxh64_term(w, q, rc, seed), D.w, D.magic), bit);
            } else {
                for (uint32_t seed = 0; seed < a.k; ++seed)
                    atomicOr(col + fastmod(xxh64_term(w, q, false, seed), D.w, D.magic), bit);
            }
        });
    }
}

__global__ void slab_copy_kernel(const SlabGroup* groups, const uint64_t* row_prefix, uint32_t ngroups,
                                 const unsigned int* slab, uint8_t* payload) {
    const uint64_t total = row_prefix[ngroups];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = ngroups;
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (row_prefix[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        const SlabGroup G = groups[lo];
        const uint64_t r = t - row_prefix[lo];
        *reinterpret_cast<unsigned int*>(payload + G.dst + r * G.pitch) = slab[G.src + r];
    }
}

inline uint64_t next_pow2(uint64_t x) {
    uint64_t p = 2;
    while (p < x) p <<= 1;
    return p;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

} // namespace

const BuildTiming& last_build_timing() { return g_timing; }

std::unique_ptr<DeviceIndex> build_device_index(const uint8_t* seqs, const uint64_t* seg_off,
                                                uint64_t n_segs, const uint64_t* doc_segs,
                                                const std::vector<std::string>& names, const Params& P,
                                                uint8_t kind, uint64_t forced_w, int device,
                                                bool seqs_on_device, bool terms_input) {
    auto t_start = std::chrono::steady_clock::now();
    g_timing = BuildTiming();
    P.validate();                                             // params.hpp:26-35
    const uint64_t n_docs = names.size();
    if (n_docs == 0) throw DataError("build: no documents"); // classic_index.cpp:44
    if (kind != kKindClassic && kind != kKindCompact) throw UsageError("build: unknown index kind");
    for (uint64_t d = 0; d < n_docs; ++d)
        if (doc_segs[d + 1] < doc_segs[d] || doc_segs[d + 1] > n_segs)
            throw UsageError("build: bad document segment ranges");
    if (doc_segs[0] != 0 || doc_segs[n_docs] != n_segs)
        throw UsageError("build: document segment ranges must cover all segments in order");
    // Pre-extracted terms (one segment = one TermSet entry): the reference's
    // term-length check, in its order -- input order for classic
    // (classic_index.cpp:49-56, before the name check), sorted order for
    // compact (each block re-runs build_classic after the name check,
    // compact_index.cpp:27-52).
    auto check_terms = [&](const std::vector<uint64_t>& docs_in_order) {
        for (uint64_t d : docs_in_order)
            for (uint64_t s = doc_segs[d]; s < doc_segs[d + 1]; ++s)
                if (seg_off[s + 1] - seg_off[s] != P.q)
                    throw UsageError("build: term length != q in document " + names[d]);
    };
    std::vector<uint64_t> input_order(n_docs);
    std::iota(input_order.begin(), input_order.end(), 0);
    if (terms_input && kind == kKindClassic) check_terms(input_order);
    {
        std::vector<const std::string*> sorted(n_docs);
        for (uint64_t d = 0; d < n_docs; ++d) sorted[d] = &names[d];
        std::sort(sorted.begin(), sorted.end(),
                  [](const std::string* a, const std::string* b) { return *a < *b; });
        for (uint64_t i = 1; i < n_docs; ++i)
            if (*sorted[i - 1] == *sorted[i]) // classic_index.cpp:17-22
                throw DataError("duplicate document name: " + *sorted[i]);
    }
    if (terms_input && kind == kKindCompact) {
        std::vector<uint64_t> by_count = input_order;
        std::sort(by_count.begin(), by_count.end(), [&](uint64_t a, uint64_t b) {
            const uint64_t ta = doc_segs[a + 1] - doc_segs[a], tb = doc_segs[b + 1] - doc_segs[b];
            return ta != tb ? ta < tb : names[a] < names[b];
        });
        check_terms(by_count);
    }
    const uint32_t q = P.q;

    COBS_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    COBS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};

    // windows per segment / document
    std::vector<uint64_t> seg_rbase(n_segs + 1, 0), doc_start(n_docs), doc_w(n_docs, 0);
    std::vector<uint32_t> seg_doc(n_segs);
    for (uint64_t d = 0; d < n_docs; ++d) {
        doc_start[d] = n_segs ? seg_off[doc_segs[d]] : 0;
        for (uint64_t s = doc_segs[d]; s < doc_segs[d + 1]; ++s) {
            seg_doc[s] = static_cast<uint32_t>(d);
            uint64_t len = seg_off[s + 1] - seg_off[s];
            uint64_t W = len >= q ? len - q + 1 : 0;
            seg_rbase[s + 1] = seg_rbase[s] + (W + kBRun - 1) / kBRun;
            doc_w[d] += W;
        }
        if (seg_off[doc_segs[d + 1]] - doc_start[d] >= 0xffffffffull)
            throw UsageError("build: documents larger than 4 GiB are not supported");
    }
    const uint64_t total_bytes = n_segs ? seg_off[n_segs] : 0;
    const uint64_t total_runs = seg_rbase[n_segs];

    DevBuf d_seqs, d_segoff, d_segw, d_segdoc, d_docstart, d_tab, d_taboff, d_tabslots, d_tc;
    if (!seqs_on_device) d_seqs.reserve(std::max<uint64_t>(total_bytes, 1));
    d_segoff.reserve(8 * (n_segs + 1));
    d_segw.reserve(8 * (n_segs + 1));
    d_segdoc.reserve(4 * std::max<uint64_t>(n_segs, 1));
    d_docstart.reserve(8 * n_docs);
    d_tc.reserve(8 * n_docs);
    auto t_h2d = std::chrono::steady_clock::now();
    if (!seqs_on_device)
        COBS_CUDA(cudaMemcpyAsync(d_seqs.ptr, seqs, total_bytes, cudaMemcpyHostToDevice, st));
    COBS_CUDA(cudaMemcpyAsync(d_segoff.ptr, seg_off, 8 * (n_segs + 1), cudaMemcpyHostToDevice, st));
    COBS_CUDA(cudaMemcpyAsync(d_segw.ptr, seg_rbase.data(), 8 * (n_segs + 1), cudaMemcpyHostToDevice, st));
    if (n_segs)
        COBS_CUDA(cudaMemcpyAsync(d_segdoc.ptr, seg_doc.data(), 4 * n_segs, cudaMemcpyHostToDevice, st));
    COBS_CUDA(cudaMemcpyAsync(d_docstart.ptr, doc_start.data(), 8 * n_docs, cudaMemcpyHostToDevice, st));
    COBS_CUDA(cudaMemsetAsync(d_tc.ptr, 0, 8 * n_docs, st));
    COBS_CUDA(cudaStreamSynchronize(st));
    g_timing.ms_h2d = ms_since(t_h2d);

    WinArgs wa{};
    wa.seqs = seqs_on_device ? seqs : d_seqs.as<uint8_t>();
    wa.seg_off = d_segoff.as<uint64_t>();
    wa.seg_rbase = d_segw.as<uint64_t>();
    wa.seg_doc = d_segdoc.as<uint32_t>();
    wa.doc_start = d_docstart.as<uint64_t>();
    wa.q = q;
    wa.k = P.k;
    wa.canonical = (P.canonical && !terms_input) ? 1 : 0; // terms are hashed as given
    wa.tag_mask = debug_tag_mask();

    Event e0, e1, e2, e3;

    // ---- count pass, in waves of documents whose sets fit in L2 ---------
    // (random CAS into L2-resident sets instead of DRAM; a document larger
    // than a wave gets a wave of its own)
    uint64_t slab_wave_bytes = 96ull << 20;
    if (const char* e = std::getenv("COBS_SLAB_WAVE_MB")) slab_wave_bytes = std::strtoull(e, nullptr, 10) << 20;
    std::vector<uint64_t> tc(n_docs);
    if (terms_input) { // TermSet::term_count() = terms.size() (termizer.hpp:25)
        for (uint64_t d = 0; d < n_docs; ++d) tc[d] = doc_segs[d + 1] - doc_segs[d];
    } else {
        std::vector<uint64_t> tab_off(n_docs), tab_slots(n_docs);
        uint64_t load_div = 4; // slots >= load_div/2 * windows (load <= 2/load_div)
        if (const char* e = std::getenv("COBS_COUNT_LOAD_DIV")) load_div = std::max<uint64_t>(2, std::strtoull(e, nullptr, 10));
        for (uint64_t d = 0; d < n_docs; ++d) tab_slots[d] = next_pow2(doc_w[d] * load_div / 2 + 1);
        size_t free_b = 0, total_b = 0;
        COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
        uint64_t wave_bytes = 192ull << 20;
        if (const char* e = std::getenv("COBS_COUNT_WAVE_MB")) wave_bytes = std::strtoull(e, nullptr, 10) << 20;
        const uint64_t budget_slots = std::max<uint64_t>(std::min<uint64_t>((free_b / 3) / 8, wave_bytes / 8), 1ull << 16);
        std::vector<uint64_t> wave_lo{0};
        uint64_t max_slots = 0;
        for (uint64_t d0 = 0; d0 < n_docs;) {
            uint64_t d1 = d0, slots = 0;
            while (d1 < n_docs && (d1 == d0 || slots + tab_slots[d1] <= budget_slots)) {
                tab_off[d1] = slots; // relative to the wave's tables
                slots += tab_slots[d1];
                ++d1;
            }
            max_slots = std::max(max_slots, slots);
            wave_lo.push_back(d1);
            d0 = d1;
        }
        d_taboff.reserve(8 * n_docs);
        d_tabslots.reserve(8 * n_docs);
        d_tab.reserve(8 * max_slots);
        COBS_CUDA(cudaMemcpyAsync(d_tabslots.ptr, tab_slots.data(), 8 * n_docs, cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_taboff.ptr, tab_off.data(), 8 * n_docs, cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaEventRecord(e0, st));
        auto ck = q == 31 ? count_kernel<31> : count_kernel<0>;
        for (size_t wv = 0; wv + 1 < wave_lo.size(); ++wv) {
            const uint64_t d0 = wave_lo[wv], d1 = wave_lo[wv + 1];
            const uint64_t slots = tab_off[d1 - 1] + tab_slots[d1 - 1];
            COBS_CUDA(cudaMemsetAsync(d_tab.ptr, 0, 8 * slots, st));
            wa.seg_lo = doc_segs[d0];
            wa.seg_hi = doc_segs[d1];
            wa.r_lo = seg_rbase[wa.seg_lo];
            wa.r_hi = seg_rbase[wa.seg_hi];
            if (wa.r_hi > wa.r_lo) {
                const uint64_t runs = wa.r_hi - wa.r_lo;
                const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(148 * 8, (runs + kChunkRuns - 1) / kChunkRuns));
                ck<<<grid, 256, 0, st>>>(wa, d_tab.as<unsigned long long>(), d_taboff.as<uint64_t>(),
                                         d_tabslots.as<uint64_t>(), d_tc.as<unsigned long long>());
                COBS_CUDA(cudaGetLastError());
            }
        }
        COBS_CUDA(cudaEventRecord(e1, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        float ms_count = 0;
        cudaEventElapsedTime(&ms_count, e0, e1);
        g_timing.ms_count = ms_count;
        COBS_CUDA(cudaMemcpy(tc.data(), d_tc.ptr, 8 * n_docs, cudaMemcpyDeviceToHost));
        d_tab = DevBuf();
    }

    // ---- host: order, blocks, widths ------------------------------------
    IndexMeta meta;
    meta.params = P;
    meta.kind = kind;
    std::vector<uint64_t> order(n_docs);
    std::iota(order.begin(), order.end(), 0);
    uint64_t B = n_docs;
    if (kind == kKindCompact) {
        std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { // compact_index.cpp:27-30
            if (tc[a] != tc[b]) return tc[a] < tc[b];
            return names[a] < names[b];
        });
        B = P.block_size;
    }
    const uint64_t nb = (n_docs + B - 1) / B;
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t lo = b * B, hi = std::min(n_docs, lo + B), mx = 0;
        BlockMeta bm;
        bm.doc_count = hi - lo;
        for (uint64_t i = lo; i < hi; ++i) {
            uint64_t d = order[i];
            meta.docs.push_back({names[d], tc[d]});
            mx = std::max(mx, tc[d]);
        }
        bm.w = (kind == kKindClassic && forced_w != 0) ? forced_w : bloom::size_filter(mx, P.p, P.k);
        meta.blocks.push_back(bm);
    }
    meta.layout();
    (void)meta.header_bytes(); // DataError for names longer than 65,535 bytes (storage.cpp:368)

    // ---- fill pass, straight into the pitched HBM layout of a DeviceIndex
    auto ix = std::make_unique<DeviceIndex>();
    ix->meta = std::move(meta);
    ix->device = device;
    ix->allocate(); // refuses a matrix that does not fit in free HBM
    COBS_CUDA(cudaMemsetAsync(ix->payload, 0, ix->payload_bytes, ix->stream));
    COBS_CUDA(cudaStreamSynchronize(ix->stream));
    COBS_CUDA(cudaEventRecord(e2, st));
    wa.seg_lo = 0;
    wa.seg_hi = n_segs;
    if (total_runs > 0) {
        // waves of whole 32-column groups, block-major, slabs <= wave_bytes
        std::vector<SlabDoc> sdocs;
        std::vector<uint64_t> run_prefix;   // per wave: ndocs+1 entries (concatenated)
        std::vector<SlabGroup> sgroups;
        std::vector<uint64_t> row_prefix;   // per wave: ngroups+1 entries (concatenated)
        struct Wave { size_t doc0, ndocs, rp0, grp0, ngroups, gp0; uint64_t words; };
        std::vector<Wave> waves;
        Wave cur{0, 0, 0, 0, 0, 0, 0};
        uint64_t max_words = 0;
        auto close_wave = [&] {
            if (cur.ngroups == 0) return;
            max_words = std::max(max_words, cur.words);
            waves.push_back(cur);
            cur = Wave{sdocs.size(), 0, run_prefix.size(), sgroups.size(), 0, row_prefix.size(), 0};
        };
        const uint64_t wave_words = std::max<uint64_t>(slab_wave_bytes / 4, 1);
        for (uint64_t b = 0; b < nb; ++b) {
            const DevBlock& d = ix->blocks[b];
            const uint64_t ngr = (d.dc + 31) / 32;
            for (uint64_t gi = 0; gi < ngr; ++gi) {
                if (cur.ngroups > 0 && cur.words + d.w > wave_words) close_wave();
                if (cur.ngroups == 0) { // open: prefix starts
                    cur.rp0 = run_prefix.size();
                    cur.gp0 = row_prefix.size();
                    run_prefix.push_back(0);
                    row_prefix.push_back(0);
                }
                SlabGroup G{cur.words, d.base + 4 * gi, d.w, d.pitch};
                sgroups.push_back(G);
                row_prefix.push_back(row_prefix.back() + d.w);
                for (uint64_t c = 32 * gi; c < std::min<uint64_t>(d.dc, 32 * gi + 32); ++c) {
                    const uint64_t doc = order[d.doc_base + c];
                    SlabDoc D{};
                    D.seg_lo = doc_segs[doc];
                    D.seg_hi = doc_segs[doc + 1];
                    D.run_lo = seg_rbase[D.seg_lo];
                    D.slab = cur.words;
                    D.w = d.w;
                    D.magic = d.magic;
                    D.bit = static_cast<uint32_t>(c % 32);
                    sdocs.push_back(D);
                    run_prefix.push_back(run_prefix.back() + (seg_rbase[D.seg_hi] - D.run_lo));
                    ++cur.ndocs;
                }
                cur.words += d.w;
                ++cur.ngroups;
            }
        }
        close_wave();
        DevBuf d_sdocs, d_rp, d_sgroups, d_gp, d_slab;
        d_sdocs.reserve(sizeof(SlabDoc) * std::max<size_t>(sdocs.size(), 1));
        d_rp.reserve(8 * run_prefix.size());
        d_sgroups.reserve(sizeof(SlabGroup) * std::max<size_t>(sgroups.size(), 1));
        d_gp.reserve(8 * row_prefix.size());
        d_slab.reserve(4 * std::max<uint64_t>(max_words, 1));
        COBS_CUDA(cudaMemcpyAsync(d_sdocs.ptr, sdocs.data(), sizeof(SlabDoc) * sdocs.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_rp.ptr, run_prefix.data(), 8 * run_prefix.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_sgroups.ptr, sgroups.data(), sizeof(SlabGroup) * sgroups.size(),
                                  cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_gp.ptr, row_prefix.data(), 8 * row_prefix.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaEventRecord(e2, st));
        auto fk = q == 31 ? slab_fill_kernel<31> : slab_fill_kernel<0>;
        for (const Wave& wv : waves) {
            COBS_CUDA(cudaMemsetAsync(d_slab.ptr, 0, 4 * wv.words, st));
            const uint64_t runs = run_prefix[wv.rp0 + wv.ndocs];
            if (runs > 0)
                fk<<<static_cast<unsigned>(std::min<uint64_t>(148 * 16, (runs + 255) / 256)), 256, 0, st>>>(
                    wa, d_sdocs.as<SlabDoc>() + wv.doc0, d_rp.as<uint64_t>() + wv.rp0,
                    static_cast<uint32_t>(wv.ndocs), d_slab.as<unsigned int>());
            slab_copy_kernel<<<static_cast<unsigned>(std::min<uint64_t>(148 * 16, (wv.words + 255) / 256)), 256, 0,
                               st>>>(d_sgroups.as<SlabGroup>() + wv.grp0, d_gp.as<uint64_t>() + wv.gp0,
                                     static_cast<uint32_t>(wv.ngroups), d_slab.as<unsigned int>(), ix->payload);
            COBS_CUDA(cudaGetLastError());
        }
        COBS_CUDA(cudaEventRecord(e3, st));
        COBS_CUDA(cudaStreamSynchronize(st));
    }
    COBS_CUDA(cudaEventRecord(e3, st));
    COBS_CUDA(cudaStreamSynchronize(st));
    float ms_fill = 0;
    cudaEventElapsedTime(&ms_fill, e2, e3);
    g_timing.ms_fill = ms_fill;
    ix->finish_upload();
    g_timing.ms_total = ms_since(t_start);
    return ix;
}

std::vector<uint8_t> index_image(const DeviceIndex& ix) {
    std::vector<uint8_t> header = ix.meta.header_bytes();
    const uint64_t payload = ix.meta.file_size - ix.meta.payload_start;
    std::vector<uint8_t> image(header.size() + payload);
    std::memcpy(image.data(), header.data(), header.size());
    if (ix.streaming()) { // host-resident: the payload is already in file layout
        std::memcpy(image.data() + header.size(), ix.hs->host, payload);
        return image;
    }
    COBS_CUDA(cudaSetDevice(ix.device));
    uint64_t off = header.size();
    for (const DevBlock& d : ix.blocks) { // un-pitch on the copy engine
        if (d.w)
            COBS_CUDA(cudaMemcpy2D(image.data() + off, d.rb, ix.payload + d.base, d.pitch, d.rb, d.w,
                                   cudaMemcpyDeviceToHost));
        off += d.w * d.rb;
    }
    return image;
}

std::vector<uint8_t> build_index(const uint8_t* seqs, const uint64_t* seg_off, uint64_t n_segs,
                                 const uint64_t* doc_segs, const std::vector<std::string>& names,
                                 const Params& P, uint8_t kind, uint64_t forced_w, int device) {
    auto t0 = std::chrono::steady_clock::now();
    auto ix = build_device_index(seqs, seg_off, n_segs, doc_segs, names, P, kind, forced_w, device, false, false);
    auto t_d2h = std::chrono::steady_clock::now();
    std::vector<uint8_t> image = index_image(*ix);
    g_timing.ms_d2h = ms_since(t_d2h);
    g_timing.ms_total = ms_since(t0);
    return image;
}

void write_image(const std::vector<uint8_t>& image, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc); // storage.cpp:382-396
    if (!out) throw DataError("cannot create index file: " + path);
    out.write(reinterpret_cast<const char*>(image.data()), static_cast<std::streamsize>(image.size()));
    out.flush();
    if (!out) throw DataError("error writing index file: " + path);
}

// ---- synthetic documents on the device ---------------------------------

__global__ void synth_docs_kernel(uint64_t seed, int alpha, const uint64_t* doc_off, uint64_t doc_lo,
                                  uint64_t n_docs, uint64_t total, uint8_t* out) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n_docs; // doc_off[lo] <= g < doc_off[hi]
        while (hi - lo > 1) {
            uint64_t mid = (lo + hi) >> 1;
            if (doc_off[mid] <= g)
                lo = mid;
            else
                hi = mid;
        }
        out[g] = static_cast<uint8_t>(
            syn_sym_char(alpha, syn_doc_sym(seed, alpha, doc_lo + lo, g - doc_off[lo])));
    }
}

void synth_docs(uint64_t seed, int alpha, const uint64_t* doc_len, uint64_t doc_lo, uint64_t doc_hi,
                uint8_t* dev_out, int device) {
    COBS_CUDA(cudaSetDevice(device));
    uint64_t n = doc_hi - doc_lo;
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + doc_len[doc_lo + i];
    DevBuf d_off;
    d_off.reserve(8 * (n + 1));
    COBS_CUDA(cudaMemcpy(d_off.ptr, off.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    if (off[n] > 0) synth_docs_kernel<<<148 * 16, 256>>>(seed, alpha, d_off.as<uint64_t>(), doc_lo, n, off[n], dev_out);
    COBS_CUDA(cudaGetLastError());
    COBS_CUDA(cudaDeviceSynchronize());
}

} // namespace cobsg
