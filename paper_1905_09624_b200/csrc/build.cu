// Kernel 4: index construction on the device.
//
//   count pass  exact per-document distinct count -> term_count
//               (termizer.cpp:103-129, termizer.hpp:25), windows rolled as
//               2-bit codes (canonical = min(fwd, revcomp)):
//               * partitioned (q <= 32, large corpora): codes mixed by a
//                 bijection and split into per-document buckets (shared-
//                 memory histograms, scan, a two-level scatter), each bucket
//                 deduplicated in a shared-memory set of 32-bit
//                 fingerprint|index slots over its keys staged by the bulk-
//                 copy engine -- pc_*_kernel;
//               * hash sets (any q, byte-path windows, small corpora):
//                 per-document lock-free sets in L2-sized waves -- count_kernel.
//   host        classic width / compact (term_count, name) sort, blocks of
//               B, per-block widths        (classic_index.cpp:40-64,
//               compact_index.cpp:19-52, bloom.cpp:50-66)
//   fill pass   for every window and seed, bit (XXH64 % w_b, column)
//               (classic_index.cpp:26-36, bit_matrix.hpp:25-27): 32
//               consecutive columns of a block are one u32 per row, so waves
//               of such column "slabs" (L2-sized) are filled with atomicOr,
//               then copied 8 groups (32 bytes per row) at a time into the
//               pitched HBM layout of the query index (a built index is
//               queryable in place; the file payload is its un-pitched D2H
//               copy).  OR is idempotent, so every window is filled, not just
//               the distinct ones.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <type_traits>

#include <cub/cub.cuh>

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

#ifndef COBS_PC_PREFETCH
#define COBS_PC_PREFETCH 1
#endif
constexpr bool kPcPrefetch = COBS_PC_PREFETCH != 0;

// ---- packed rolling for 2-bit DNA codes (the count pass's hot loop) ----
//
// 16 bases enter at once: their bytes become 2-bit codes four at a time
// (one multiply packs a word's four codes), and three shift registers hold
// the recent bases -- forward codes newest-lowest (R, 128 bits), complement
// codes newest-highest (T, 128 bits: reverse-complement codes read out
// without any per-base reversal) and a 1-bit-per-base non-ACGT mask (Bm).
// Each of the 16 windows ending in the chunk is then a constant-shift
// extract of R and T (funnel shifts) and a mask test of Bm: ~13 integer ops
// per window instead of a 64-bit shift/or/and chain per byte.
struct U128 {
    uint64_t hi, lo;
};
// low 64 bits of x >> s (0 <= s < 128)
__device__ __forceinline__ uint64_t shr128(const U128& x, uint32_t s) {
    if (s == 0) return x.lo;
    if (s < 64) return (x.lo >> s) | (x.hi << (64 - s));
    return x.hi >> (s - 64);
}
// codes of 4 A/C/G/T bytes packed into 8 bits, the first byte most significant
__device__ __forceinline__ uint32_t pack4(uint32_t w) {
    const uint32_t c = ((w >> 1) ^ (w >> 2)) & 0x03030303u; // base_code per byte
    return (c * 0x40100401u) >> 24;
}
// 4 bits: bit 3 = byte 0 ... bit 0 = byte 3 is not one of A, C, G, T
__device__ __forceinline__ uint32_t bad4(uint32_t w) {
    const uint32_t c = ((w >> 1) ^ (w >> 2)) & 0x03030303u;
    const uint32_t sel = (c | (c >> 4)) & 0x00ff00ffu; // nibble k = code of byte k
    const uint32_t expect = __byte_perm(0x54474341u, 0u, (sel & 0xffu) | ((sel >> 8) & 0xff00u));
    const uint32_t x = expect ^ w; // nonzero bytes: not the letter of their own code
    if (x == 0u) return 0u;
    const uint32_t nz = (((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
    return (((nz >> 7) * 0x08040201u) >> 24) & 0xfu;
}

template <int QC, typename F>
__device__ __forceinline__ void roll_range_packed(const uint8_t* sb, uint64_t j0, uint64_t j1, uint32_t q_rt,
                                                  bool canonical, F&& f) {
    const uint32_t q = QC ? QC : q_rt;
    const uint64_t mask = q >= 32 ? ~0ull : ((1ull << (2 * q)) - 1);
    const uint64_t qmask = q >= 64 ? ~0ull : ((1ull << q) - 1);
    const uint64_t end = j1 + q - 1, first = j0 + q - 1; // bytes [j0, end); windows end at >= first
    U128 R{0, 0}, T{0, 0};
    uint64_t Bm = 0;
    uint64_t i = j0;
    // window ending at byte e (pushed t bytes ago): emit if e >= first
    auto emit = [&](uint64_t e, uint32_t t) {
        if (e < first) return;
        const bool ok = ((Bm >> t) & qmask) == 0;
        uint64_t code = shr128(R, 2 * t) & mask;
        if (canonical) { // min(gram, revcomp) bytewise == min of the codes
            const uint64_t rc = shr128(T, 128 - 2 * q - 2 * t) & mask;
            code = rc < code ? rc : code;
        }
        f(e - (q - 1), ok, code);
    };
    auto push1 = [&](uint32_t c) {
        const uint32_t b = base_code(c);
        R.hi = (R.hi << 2) | (R.lo >> 62);
        R.lo = (R.lo << 2) | b;
        T.lo = (T.lo >> 2) | (T.hi << 62);
        T.hi = (T.hi >> 2) | (static_cast<uint64_t>(3u - b) << 62);
        Bm = (Bm << 1) | (acgt_bit(c) ^ 1u);
        emit(i, 0);
        ++i;
    };
    while (i < end && (reinterpret_cast<uintptr_t>(sb + i) & 15u)) push1(__ldg(sb + i));
    // the 16 bytes after the current ones are loaded while these are rolled
    // (A/B knob COBS_PC_PREFETCH: C3 super-bucket scatter 451 -> 407 ms, count
    // 1,510-1,542 -> 1,460-1,470 ms; the histogram pass unchanged)
    uint4 vn = make_uint4(0u, 0u, 0u, 0u);
    if (kPcPrefetch && i + 16 <= end) vn = __ldg(reinterpret_cast<const uint4*>(sb + i));
    while (i + 16 <= end) {
        uint4 v;
        if (kPcPrefetch) {
            v = vn;
            if (i + 32 <= end) vn = __ldg(reinterpret_cast<const uint4*>(sb + i + 16));
        } else {
            v = __ldg(reinterpret_cast<const uint4*>(sb + i));
        }
        const uint32_t P = (pack4(v.x) << 24) | (pack4(v.y) << 16) | (pack4(v.z) << 8) | pack4(v.w);
        uint32_t rp = __brev(P); // complement codes, first base lowest
        rp = ~(((rp >> 1) & 0x55555555u) | ((rp & 0x55555555u) << 1));
        const uint32_t bad = (bad4(v.x) << 12) | (bad4(v.y) << 8) | (bad4(v.z) << 4) | bad4(v.w);
        R.hi = (R.hi << 32) | (R.lo >> 32);
        R.lo = (R.lo << 32) | P;
        T.lo = (T.lo >> 32) | (T.hi << 32);
        T.hi = (T.hi >> 32) | (static_cast<uint64_t>(rp) << 32);
        Bm = (Bm << 16) | bad;
        i += 16;
#pragma unroll
        for (int t = 15; t >= 0; --t) emit(i - 1 - static_cast<uint32_t>(t), static_cast<uint32_t>(t));
    }
    while (i < end) push1(__ldg(sb + i));
}

// roll_windows over a long range with 16-byte loads: the segment bytes
// [j0, j1 + q - 1) are pushed in order (aligned uint4 loads for the body,
// bytes at the ragged ends), f(j, dna, code) after every complete window j
// in [j0, j1).  Only for q <= 32.  PACKED: 2-bit DNA codes 16 bases at a
// time (roll_range_packed; small callbacks only -- it inlines f 16 times).
template <int QC, int UNROLL = 4, int SB = 0, bool PACKED = false, typename F>
__device__ __forceinline__ void roll_range(const uint8_t* sb, uint64_t j0, uint64_t j1, uint32_t q_rt,
                                           bool canonical, F&& f, const uint8_t* symtab = nullptr) {
    const uint32_t q = QC ? QC : q_rt;
    if (j1 <= j0) return;
    if constexpr (PACKED && SB == 0) {
        roll_range_packed<QC>(sb, j0, j1, q, canonical, f);
        return;
    }
    // SB > 0: small-alphabet symbol codes (non-canonical raw bytes), else 2-bit DNA codes
    typename std::conditional<SB == 0, Roller, SymRoller<SB ? SB : 1>>::type R = [&] {
        if constexpr (SB == 0) return Roller(q);
        else return SymRoller<SB>(q, symtab);
    }();
    const uint64_t end = j1 + q - 1, first = j0 + q - 1;
    uint64_t i = j0;
    auto push = [&](uint32_t c) {
        R.push(c);
        if (i >= first) f(i - (q - 1), R.dna(), canonical ? R.canon() : R.fwd);
        ++i;
    };
    while (i < end && (reinterpret_cast<uintptr_t>(sb + i) & 15u)) push(__ldg(sb + i));
    if (i + 16 <= end) { // the next 16 bytes are loaded while these are rolled
        uint4 v = __ldg(reinterpret_cast<const uint4*>(sb + i));
        for (;;) {
            const bool more = i + 32 <= end;
            uint4 nx = v;
            if (more) nx = __ldg(reinterpret_cast<const uint4*>(sb + i + 16));
            const uint64_t lo = v.x | static_cast<uint64_t>(v.y) << 32, hi = v.z | static_cast<uint64_t>(v.w) << 32;
            // (a bounded unroll: the callback may be large, and 16 inlined
            // copies of it overflow the instruction cache)
#pragma unroll UNROLL
            for (int k = 0; k < 16; ++k) push(static_cast<uint32_t>((k < 8 ? lo >> (8 * k) : hi >> (8 * (k - 8))) & 0xffu));
            if (!more) break;
            v = nx;
        }
    }
    while (i < end) push(__ldg(sb + i));
}

template <int QC>
__global__ void __launch_bounds__(256) count_kernel(WinArgs a, unsigned long long* tab,
                                                    const uint64_t* tab_off, const uint64_t* tab_slots,
                                                    unsigned long long* term_count) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t q = QC ? QC : a.q;
    const bool codes = codes_exact(q, a.canonical != 0); // else q = 32 raw: byte path
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
                if (dna && codes) { // the slot only needs a well-mixed hash of the exact code
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

// ---- partitioned distinct count (q <= 32: every counted window is a 2-bit
// code).  Instead of one random L2/DRAM CAS per window into a per-document
// hash set, each document's codes are mixed by a bijection (the keys) and
// split by the keys' top bits into buckets of ~4,096 keys (chunk histograms
// in shared memory, one global atomic per (chunk, bucket)), scattered into a
// key buffer in two levels, and every bucket is deduplicated by one CTA in a
// shared-memory set.  Exact: a code lands in exactly one bucket, and equal
// codes always in the same one.
#ifndef COBS_PC_RUNS
#define COBS_PC_RUNS 16
#endif
constexpr uint32_t kPcRunsPerThread = COBS_PC_RUNS; // consecutive runs one thread rolls through
constexpr uint32_t kPcRuns = 256 * kPcRunsPerThread; // runs (x kBRun windows) per chunk
constexpr uint32_t kPcHist = 8192;   // buckets a chunk histogram keeps in shared memory
constexpr uint64_t kPcTarget = 4096;    // keys per bucket: nbk = next_pow2(ceil(W / kPcTarget)) <= kPcHist
                                        // (A/B, fingerprint sets: 2,048 / 3,072 / 4,096 / 8,192 -> C3 count
                                        // 1.78-1.91 / 1.49-1.52 / 1.41-1.50 / 1.74-1.78 s)
constexpr uint64_t kPcWaveKeys = 1000000000; // windows per wave (A/B knob COBS_PC_WAVE_KEYS)
constexpr uint32_t kPcMaxSlotsFp = 32768;  // largest fingerprint set (128 KB of shared memory)
                                        // (A/B with 1x-mean sets: 1,024 / 2,048 / 4,096 -> C3 count 1.81 / 1.65 / 1.61 s)

struct PcDoc {
    uint64_t run_lo, run_hi; // global run range of the document
    uint64_t seg_lo, seg_hi; // its segments
    uint64_t chunk0;         // first chunk (wave-relative prefix)
    uint64_t bucket0;        // first bucket (wave-relative prefix)
    uint32_t nbk;            // buckets (a power of two)
    uint32_t shift;          // 64 - log2(nbk); 64 = a single bucket
    uint32_t doc;            // global document index
    uint32_t sb0;            // two-level scatter: first super-bucket (wave-relative prefix)
    uint32_t tpr;            // runs per thread in this document's chunks (a chunk = 256 x tpr runs)
};

struct PcArgs {
    WinArgs a;
    const PcDoc* docs;
    uint32_t ndocs;
    uint64_t nchunks;
    uint32_t* bucket_cnt;     // per bucket (histogram pass)
    unsigned long long* keys; // mix_code(code) (a bijection), grouped by (super-)bucket
    unsigned long long* bad;  // non-ACGT windows without canonicalisation (byte path needed)
    uint32_t* chunk_sup;      // two-level: per (chunk, super-bucket) key counts [chunk][kSup], or null
    const uint8_t* symtab;    // SB > 0: byte -> symbol index (256 entries)
    unsigned long long* work; // the wave's work counters (zeroed): [0] histogram chunks, [1] scatter chunks, [2] super-buckets
};

// Persistent CTAs take their next unit (chunk, super-bucket) from a global
// counter instead of striding by the grid: the grids below ask for more
// CTAs than fit an SM (registers), and the histogram pass shares the SMs
// with the previous wave's kernels, so a fixed stride left the late CTAs'
// whole share to run on mostly empty SMs.  Call with all threads; includes
// the barrier that ends the previous unit's use of shared memory.
__device__ __forceinline__ uint64_t pc_next_unit(unsigned long long* counter, unsigned long long* s_slot) {
    __syncthreads();
    if (threadIdx.x == 0) *s_slot = atomicAdd(counter, 1ull);
    __syncthreads();
    return *s_slot;
}

#ifndef COBS_PC_MIX_LIGHT
#define COBS_PC_MIX_LIGHT 1
#endif
// the partitioned count's key of a code: a bijection whose top bits (bucket),
// low bits (set group) and bits 32..46 (fingerprint) all depend on the whole code
__device__ __forceinline__ uint64_t pc_mix(uint64_t z) {
    if (COBS_PC_MIX_LIGHT) { // one multiply + one fold (A/B vs the splitmix64 finaliser: C3 count 1,038 vs 1,057 ms, C4 211 vs 217)
        z *= 0x9E3779B97F4A7C15ULL;
        return z ^ (z >> 32);
    }
    return mix_code(z);
}
__device__ __forceinline__ uint32_t pc_bucket(uint64_t code, uint32_t shift) {
    return shift >= 64 ? 0u : static_cast<uint32_t>(pc_mix(code) >> shift);
}

constexpr int kSymBits = 5;                  // symbol codes: <= 32 distinct byte values, q <= 12
#ifndef COBS_PC_PACKED
#define COBS_PC_PACKED 1
#endif
constexpr bool kPcPacked = COBS_PC_PACKED != 0; // 2-bit codes rolled 16 bases at a time (roll_range_packed)
#ifndef COBS_PC_SUPLOG2
#define COBS_PC_SUPLOG2 4
#endif
constexpr uint32_t kSupLog2 = COBS_PC_SUPLOG2; // two-level scatter: <= 16 super-buckets per document (A/B, C3 count: 8 -> 1,211 ms,
                                               // 16 -> 998, 32 -> 1,052; 64 and 256 slower still): fewer runs = more lanes of a
                                               // warp's store in one 128-byte line
constexpr uint32_t kSup = 1u << kSupLog2;
#ifndef COBS_PC_BPSLOG2
#define COBS_PC_BPSLOG2 4
#endif
// log2(buckets per super-bucket) of a document with 2^lg buckets: <= kSup
// super-buckets, and >= 2^COBS_PC_BPSLOG2 buckets in each where the document has that many
__host__ __device__ __forceinline__ uint32_t pc_super_shift_lg(uint32_t lg) {
    const uint32_t a = lg - (lg < kSupLog2 ? lg : kSupLog2);
    constexpr uint32_t kBps = COBS_PC_BPSLOG2;
    const uint32_t b = kBps == 0u ? 0u : (lg < kBps ? lg : kBps);
    return a > b ? a : b;
}
__device__ __forceinline__ uint32_t pc_super_shift(const PcDoc& D) { // bucket >> this = super-bucket
    return pc_super_shift_lg(64u - D.shift);                         // (64 - shift = log2(nbk))
}

// chunk c -> its document (last i with docs[i].chunk0 <= c, skipping empty ones)
__device__ __forceinline__ uint32_t pc_chunk_doc(const PcDoc* docs, uint32_t n, uint64_t c) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (docs[mid].chunk0 <= c)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// runs [r0, r1) of chunk c of document D (256 threads x D.tpr runs)
__device__ __forceinline__ void pc_chunk_runs(const PcDoc& D, uint64_t c, uint64_t& r0, uint64_t& r1) {
    r0 = D.run_lo + (c - D.chunk0) * (256ull * D.tpr);
    r1 = min(D.run_hi, r0 + static_cast<uint64_t>(256ull * D.tpr));
}

// f(dna, code) for every window of the chunk's runs; each thread rolls
// through D.tpr consecutive runs (256 threads per CTA)
template <int QC, int SB = 0, typename F>
__device__ __forceinline__ void pc_windows(const WinArgs& a, const PcDoc& D, uint64_t r0, uint64_t r1, F&& f,
                                           const uint8_t* symtab = nullptr) {
    const uint32_t q = QC ? QC : a.q;
    uint64_t g = r0 + static_cast<uint64_t>(threadIdx.x) * D.tpr;
    const uint64_t ge = min(r1, g + static_cast<uint64_t>(D.tpr));
    while (g < ge) {
        const uint64_t s = find_seg_in(a, g, D.seg_lo, D.seg_hi);
        const uint64_t rb = a.seg_rbase[s];
        const uint64_t len = a.seg_off[s + 1] - a.seg_off[s];
        const uint64_t W = len >= q ? len - q + 1 : 0;
        const uint64_t gend = min(ge, a.seg_rbase[s + 1]);
        roll_range<QC, 4, SB, kPcPacked>(a.seqs + a.seg_off[s], (g - rb) * kBRun, min(W, (gend - rb) * kBRun), q,
                                         a.canonical != 0, [&](uint64_t, bool dna, uint64_t code) { f(dna, code); },
                                         symtab);
        g = gend;
    }
}

// (min CTAs per SM, A/B: 4 -> 55-56 registers; 5 -> 48 registers: C3 count
// 1,158 vs 1,116 ms; 6 -> 40 registers and spills: 1,241 ms)
#ifndef COBS_PC_HIST_MINB
#define COBS_PC_HIST_MINB 4
#endif
#ifndef COBS_PC_SCAT_MINB
#define COBS_PC_SCAT_MINB 4
#endif
template <int QC, int SB = 0>
__global__ void __launch_bounds__(256, COBS_PC_HIST_MINB) pc_hist_kernel(PcArgs p) {
    __shared__ uint32_t s_hist[kPcHist];
    __shared__ uint32_t s_doc;
    __shared__ unsigned long long s_bad;
    __shared__ uint8_t s_sym[256];
    __shared__ unsigned long long s_unit;
    if (SB) s_sym[threadIdx.x] = p.symtab[threadIdx.x]; // (256 threads)
    for (;;) {
        const uint64_t c = pc_next_unit(p.work + 0, &s_unit);
        if (c >= p.nchunks) break;
        if (threadIdx.x == 0) {
            s_doc = pc_chunk_doc(p.docs, p.ndocs, c);
            s_bad = 0;
        }
        __syncthreads();
        const PcDoc D = p.docs[s_doc]; // (D.nbk <= kPcHist)
        for (uint32_t j = threadIdx.x; j < D.nbk; j += blockDim.x) s_hist[j] = 0;
        __syncthreads();
        uint64_t r0, r1;
        pc_chunk_runs(D, c, r0, r1);
        uint32_t bad = 0;
        pc_windows<QC, SB>(p.a, D, r0, r1, [&](bool dna, uint64_t code) {
            if (!dna) { // canonical: skipped (termizer.cpp:113-116); else needs the byte path
                bad += p.a.canonical ? 0u : 1u;
                return;
            }
            atomicAdd(&s_hist[pc_bucket(code, D.shift)], 1u);
        }, s_sym);
        if (bad) atomicAdd(&s_bad, (unsigned long long)bad);
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < D.nbk; j += blockDim.x)
            if (s_hist[j]) atomicAdd(&p.bucket_cnt[D.bucket0 + j], s_hist[j]);
        { // the super-bucket scatter's per-chunk reservation sizes
            const uint32_t sbs = pc_super_shift(D), nsb = D.nbk >> sbs;
            if (threadIdx.x < nsb) {
                uint32_t sum = 0;
                for (uint32_t j = threadIdx.x << sbs; j < (threadIdx.x + 1u) << sbs; ++j) sum += s_hist[j];
                p.chunk_sup[c * kSup + threadIdx.x] = sum;
            }
        }
        if (threadIdx.x == 0 && s_bad) atomicAdd(p.bad, s_bad);
    }
}

// ---- two-level scatter: keys first into <= kSup super-buckets per document
// (a super-bucket = consecutive buckets, so its region is theirs in the
// final layout), long runs per chunk; then one CTA per super-bucket places
// its keys into their buckets.  A chunk's runs are then ~512 keys instead of
// ~16, so DRAM sees whole sectors instead of read-modify-writes of sectors
// shared with runs written by other CTAs much later.

// super-bucket cursors = offset of its first bucket; super -> document map
__global__ void pc_super_init_kernel(const PcDoc* docs, uint32_t ndocs, const uint32_t* off, uint32_t* sup_cursor,
                                     uint32_t* sup_doc) {
    for (uint32_t i = blockIdx.x; i < ndocs; i += gridDim.x) {
        const PcDoc D = docs[i];
        const uint32_t sbs = pc_super_shift(D), nsb = D.nbk >> sbs;
        for (uint32_t j = threadIdx.x; j < nsb; j += blockDim.x) {
            sup_cursor[D.sb0 + j] = off[D.bucket0 + (static_cast<uint64_t>(j) << sbs)];
            sup_doc[D.sb0 + j] = i;
        }
    }
}

template <int QC, int SB = 0>
__global__ void __launch_bounds__(256, COBS_PC_SCAT_MINB) pc_scatter_super_kernel(PcArgs p, uint32_t* sup_cursor) {
    __shared__ uint32_t s_cnt[kSup], s_base[kSup];
    __shared__ uint32_t s_doc;
    __shared__ uint8_t s_sym[256];
    __shared__ unsigned long long s_unit;
    if (SB) s_sym[threadIdx.x] = p.symtab[threadIdx.x]; // (256 threads)
    for (;;) {
        const uint64_t c = pc_next_unit(p.work + 1, &s_unit);
        if (c >= p.nchunks) break;
        if (threadIdx.x == 0) s_doc = pc_chunk_doc(p.docs, p.ndocs, c);
        __syncthreads();
        const PcDoc D = p.docs[s_doc];
        uint64_t r0, r1;
        pc_chunk_runs(D, c, r0, r1);
        const uint32_t sbs = pc_super_shift(D), nsb = D.nbk >> sbs;
        if (threadIdx.x < nsb) { // (the histogram pass left the chunk's counts)
            const uint32_t n = p.chunk_sup[c * kSup + threadIdx.x];
            if (n) s_base[threadIdx.x] = atomicAdd(&sup_cursor[D.sb0 + threadIdx.x], n);
            s_cnt[threadIdx.x] = 0;
        }
        __syncthreads();
        pc_windows<QC, SB>(p.a, D, r0, r1, [&](bool dna, uint64_t code) {
            if (!dna) return;
            const uint64_t m = pc_mix(code);
            const uint32_t sb = (D.shift >= 64 ? 0u : static_cast<uint32_t>(m >> D.shift)) >> sbs;
            p.keys[s_base[sb] + atomicAdd(&s_cnt[sb], 1u)] = m;
        }, s_sym);
    }
}

// one CTA per super-bucket: its keys (in keys_a) into their buckets (keys_b),
// a tile of kFinTile keys at a time: counting-sorted by bucket in shared
// memory, then each bucket's run of the tile written with coalesced stores
// (whole sectors, no read-modify-write of partially written ones).
#ifndef COBS_FIN_TILE
#define COBS_FIN_TILE 4096
#endif
constexpr uint32_t kFinTile = COBS_FIN_TILE;
constexpr uint32_t kFinPer = kFinTile / 256; // keys per thread per tile
__global__ void __launch_bounds__(256) pc_scatter_final_kernel(const PcDoc* docs, const uint32_t* sup_doc,
                                                               uint64_t nsup, const uint32_t* off,
                                                               const unsigned long long* keys_a,
                                                               unsigned long long* keys_b, unsigned long long* work) {
    constexpr uint32_t kMaxB = kPcHist / kSup > 128 ? kPcHist / kSup : 128; // buckets per super-bucket
    __shared__ uint32_t s_cur[kMaxB], s_cnt[kMaxB], s_off[kMaxB];
    __shared__ uint16_t s_start[kMaxB]; // (< kFinTile)
    __shared__ unsigned long long s_sorted[kFinTile];
    __shared__ unsigned long long s_unit;
    for (;;) {
        const uint64_t g = pc_next_unit(work, &s_unit);
        if (g >= nsup) break;
        const PcDoc D = docs[sup_doc[g]];
        const uint32_t sbs = pc_super_shift(D), bps = 1u << sbs;
        const uint64_t b_lo = D.bucket0 + ((g - D.sb0) << sbs);
        for (uint32_t t = threadIdx.x; t < bps; t += blockDim.x) s_cur[t] = off[b_lo + t];
        const uint32_t k0 = off[b_lo], k1 = off[b_lo + bps];
        // (loading the next tile's keys while this one is placed: 122
        // registers instead of 71, C3 placement 314 -> 360 ms; not kept)
        for (uint32_t tile = k0; tile < k1; tile += kFinTile) {
            const uint32_t n = min(kFinTile, k1 - tile);
            for (uint32_t t = threadIdx.x; t < bps; t += blockDim.x) s_cnt[t] = 0;
            __syncthreads();
            unsigned long long kv[kFinPer];
            uint32_t lr[kFinPer]; // bucket (low 12 bits) | rank within the tile's bucket << 12
#pragma unroll
            for (uint32_t u = 0; u < kFinPer; ++u) {
                const uint32_t i = threadIdx.x + u * blockDim.x;
                kv[u] = i < n ? __ldcs(keys_a + tile + i) : 0ull;
            }
#pragma unroll
            for (uint32_t u = 0; u < kFinPer; ++u) {
                lr[u] = 0;
                if (threadIdx.x + u * blockDim.x < n) {
                    const uint32_t lb = (D.shift >= 64 ? 0u : static_cast<uint32_t>(kv[u] >> D.shift)) & (bps - 1u);
                    lr[u] = lb | (atomicAdd(&s_cnt[lb], 1u) << 12);
                }
            }
            __syncthreads();
            if (threadIdx.x < 32) { // exclusive scan of the tile's bucket counts (<= kMaxB)
                uint32_t carry = 0;
                for (uint32_t c0 = 0; c0 < bps; c0 += 32) {
                    const uint32_t v = c0 + threadIdx.x < bps ? s_cnt[c0 + threadIdx.x] : 0u;
                    uint32_t incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (threadIdx.x >= static_cast<uint32_t>(o)) incl += y;
                    }
                    if (c0 + threadIdx.x < bps) {
                        s_start[c0 + threadIdx.x] = static_cast<uint16_t>(carry + incl - v);
                        // sorted position i of the tile -> its place in keys_b (mod 2^32)
                        s_off[c0 + threadIdx.x] = s_cur[c0 + threadIdx.x] - (carry + incl - v);
                    }
                    carry += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            __syncthreads();
#pragma unroll
            for (uint32_t u = 0; u < kFinPer; ++u)
                if (threadIdx.x + u * blockDim.x < n) {
                    s_sorted[s_start[lr[u] & 0xfffu] + (lr[u] >> 12)] = kv[u];
                }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) { // consecutive i -> consecutive addresses per run
                const unsigned long long k = s_sorted[i];            // (its bucket again from the key itself)
                const uint32_t lb = (D.shift >= 64 ? 0u : static_cast<uint32_t>(k >> D.shift)) & (bps - 1u);
                keys_b[s_off[lb] + i] = k;
            }
            __syncthreads();
            for (uint32_t t = threadIdx.x; t < bps; t += blockDim.x) s_cur[t] += s_cnt[t];
        }
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(phase)
                 : "memory");
}

// key i of a bucket staged in shared memory (SMEM) or read from global memory
template <bool SMEM>
__device__ __forceinline__ unsigned long long dd_key(uint32_t s_base, const unsigned long long* g, uint32_t i) {
    if constexpr (SMEM) {
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(s_base + 8u * i));
        return v;
    } else {
        return __ldg(g + i);
    }
}

// A key's fingerprint: its bits [16 + ib, 47) under fmask (= ~imask; tests
// narrow it) with bit 31 set, so it is never 0 (an empty slot) and above
// every index mask (ib <= 28).
__device__ __forceinline__ uint32_t dd_fp(unsigned long long m, uint32_t fmask) {
    return (static_cast<uint32_t>(m >> 16) & fmask) | 0x80000000u;
}

// One probe of a key of the fingerprint set (see pc_dedup_fp_kernel):
// returns true once the key is settled (new -> ++mine, duplicate, or
// stuck = every group full).
struct DdKey {
    unsigned long long m;
    uint32_t i, probes;
};
template <bool SMEM>
__device__ __forceinline__ bool dd_probe(DdKey& k, uint32_t sg, uint32_t gmask, uint32_t imask, uint32_t fmask,
                                         uint32_t s_keys,
                                         const unsigned long long* g_keys, uint32_t& mine, bool& stuck) {
    const uint32_t fp = dd_fp(k.m, fmask);
    const uint32_t gaddr = sg + 16u * ((static_cast<uint32_t>(k.m) + k.probes) & gmask);
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(gaddr));
    // slot j holds this fingerprint iff (slot ^ fp) <= imask (an empty slot never does: fp > imask)
    if (((v.x ^ fp) <= imask) | ((v.y ^ fp) <= imask) | ((v.z ^ fp) <= imask) | ((v.w ^ fp) <= imask)) {
        const uint32_t sl[4] = {v.x, v.y, v.z, v.w}; // (rare: a duplicate, or a fingerprint accident)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((sl[j] ^ fp) <= imask && dd_key<SMEM>(s_keys, g_keys, sl[j] & imask) == k.m) return true;
    }
    const uint32_t occ = (v.x != 0u) + (v.y != 0u) + (v.z != 0u) + (v.w != 0u); // occupied slots are a prefix
    if (occ < 4u) {
        uint32_t cur;
        asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(cur) : "r"(gaddr + 4u * occ), "r"(0u), "r"(fp | k.i)
                     : "memory");
        if (cur == 0u) {
            ++mine;
            return true;
        }
        return (cur ^ fp) <= imask && dd_key<SMEM>(s_keys, g_keys, cur & imask) == k.m;
        // (else another key took the slot: the next probe looks at the group again)
    }
    if (++k.probes > gmask) { // every group full: the wave is recounted
        stuck = true;
        return true;
    }
    return false;
}

// The keys of one bucket, each thread walking i = tid, tid + T, ... with
// kDdInFlight keys in flight (each gets one probe per trip; a settled key is
// replaced by the thread's next one).  (A warp-sliced variant refilling
// lanes by ballot kept more lanes busy but issued more instructions: C3
// dedup wave 25.0 vs 23.0 ms.)
#ifndef COBS_DD_INFLIGHT
#define COBS_DD_INFLIGHT 2
#endif
constexpr int kDdInFlight = COBS_DD_INFLIGHT;
template <int THREADS, bool SMEM>
__device__ __forceinline__ void dd_bucket(uint32_t n, uint32_t sg, uint32_t gmask, uint32_t imask, uint32_t fmask,
                                          uint32_t s_keys, const unsigned long long* g_keys, uint32_t& mine,
                                          bool& stuck) {
    uint32_t next = threadIdx.x;
    DdKey key[kDdInFlight];
    bool live[kDdInFlight];
#pragma unroll
    for (int j = 0; j < kDdInFlight; ++j) {
        key[j] = DdKey{0, next, 0};
        next += THREADS;
        live[j] = key[j].i < n;
        if (live[j]) key[j].m = dd_key<SMEM>(s_keys, g_keys, key[j].i);
    }
    for (;;) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < kDdInFlight; ++j) any |= live[j];
        if (!any) break;
#pragma unroll
        for (int j = 0; j < kDdInFlight; ++j)
            if (live[j] && dd_probe<SMEM>(key[j], sg, gmask, imask, fmask, s_keys, g_keys, mine, stuck)) {
                key[j] = DdKey{0, next, 0};
                next += THREADS;
                live[j] = key[j].i < n;
                if (live[j]) key[j].m = dd_key<SMEM>(s_keys, g_keys, key[j].i);
            }
    }
}

// The same for a staged bucket, first probes as straight-line code: each
// thread takes kDdU keys per step (i = base + u * T), loads their groups
// back to back, and claims the first empty slot of a group that shows no
// equal fingerprint with one CAS.  Everything else -- an equal fingerprint
// (a duplicate or an accident), a full group, a lost CAS (another key took
// the slot after the group was read; also a second key of this thread in the
// same group, whose view is stale) -- is left pending: its index goes to the
// warp's queue in shared memory, and whenever 32 are queued the warp settles
// them with the probe loop of dd_probe, one per lane (settling each thread's
// own pending keys right after the step ran that loop at ~15 % lane
// activity and was slower than the per-key loop: C3 count 1,498 vs 1,328
// ms).  Exact by the same invariant:
// slots of a group fill in order, and a CAS on slot s is only tried by a
// thread that saw the slots before s occupied and unequal, so it succeeds
// only if nothing was inserted into the group since the thread read it.
// (C3 dedup wave: 4.1 warp instructions per key in the per-key loop, 21 of
// 32 lanes active; here all lanes run the first probe.)
#ifndef COBS_DD_U
#define COBS_DD_U 1
#endif
constexpr int kDdU = COBS_DD_U;
#ifndef COBS_DD_LOAD
#define COBS_DD_LOAD 4
#endif
constexpr uint32_t kDdLoadNum = COBS_DD_LOAD; // set slots >= kDdLoadNum / 2 x keys where the launch's slots allow
constexpr uint32_t kDdQueue = 32u * kDdU + 32u; // pending keys a warp can hold (u16 indices)
template <int THREADS, bool SMEM>
__device__ __forceinline__ void dd_bucket_fast(uint32_t n, uint32_t sg, uint32_t gmask, uint32_t imask, uint32_t fmask,
                                               uint32_t s_keys, const unsigned long long* g_keys, uint16_t* s_queue,
                                               uint32_t& mine, bool& stuck) {
    const uint32_t lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    uint16_t* q = s_queue + (threadIdx.x >> 5) * kDdQueue;
    uint32_t qn = 0; // (warp-uniform)
    auto settle = [&](uint32_t i) {
        DdKey k{dd_key<SMEM>(s_keys, g_keys, i), i, 0};
        while (!dd_probe<SMEM>(k, sg, gmask, imask, fmask, s_keys, g_keys, mine, stuck)) {
        }
    };
    // keys of step `b` (clamped: a valid address; not used beyond n); keys read
    // from global memory are loaded one step ahead
    auto load = [&](uint32_t b, unsigned long long (&k)[kDdU]) {
#pragma unroll
        for (int u = 0; u < kDdU; ++u) k[u] = dd_key<SMEM>(s_keys, g_keys, min(b + u * THREADS, n - 1u));
    };
    unsigned long long nxt[kDdU];
    if (!SMEM) load(threadIdx.x, nxt);
    for (uint32_t wbase = threadIdx.x - lane; wbase < n; wbase += kDdU * THREADS) { // (warp-uniform trip count)
        const uint32_t base = wbase + lane;
        unsigned long long m[kDdU];
        uint32_t ga[kDdU];
        uint4 v[kDdU];
        if (SMEM) {
            load(base, m);
        } else {
#pragma unroll
            for (int u = 0; u < kDdU; ++u) m[u] = nxt[u];
            load(base + kDdU * THREADS, nxt);
        }
#pragma unroll
        for (int u = 0; u < kDdU; ++u) {
            ga[u] = sg + 16u * (static_cast<uint32_t>(m[u]) & gmask);
            asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "r"(ga[u]));
        }
#pragma unroll
        for (int u = 0; u < kDdU; ++u) {
            const uint32_t i = base + u * THREADS;
            bool pending = false;
            if (i < n) {
                const uint32_t fp = dd_fp(m[u], fmask);
                const uint32_t nearest = min(min(v[u].x ^ fp, v[u].y ^ fp), min(v[u].z ^ fp, v[u].w ^ fp));
                const uint32_t occ = (v[u].x >> 31) + (v[u].y >> 31) + (v[u].z >> 31) + (v[u].w >> 31); // a prefix
                uint32_t cur = 1u;
                if (nearest > imask && occ < 4u)
                    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(cur) : "r"(ga[u] + 4u * occ), "r"(0u), "r"(fp | i)
                                 : "memory");
                if (cur == 0u)
                    ++mine;
                else
                    pending = true;
            }
            const uint32_t pb = __ballot_sync(0xffffffffu, pending);
            if (pending) q[qn + __popc(pb & lt)] = static_cast<uint16_t>(i);
            qn += __popc(pb);
        }
        __syncwarp();
        while (qn >= 32u) { // a full warp of pending keys
            qn -= 32u;
            const uint32_t i = q[qn + lane];
            __syncwarp();
            settle(i);
        }
    }
    if (lane < qn) settle(q[lane]);
}

// One CTA per bucket: the distinct count of its n mixed keys through a
// shared-memory set of 32-bit slots.  A slot holds (fingerprint | index of
// the key in the bucket); the keys themselves are staged in shared memory
// by the bulk-copy engine (nbuf = 2: the next bucket's keys arrive while
// this one is inserted), so a slot is 4 bytes (a group of 4 slots = one
// LDS.128, the claim one 32-bit CAS) and a key is compared in full only on
// a fingerprint match (a duplicate, or a 2^-(32-ib) accident).  ib = index
// bits = max(16, bits(n - 1)); the fingerprint is the key's bits
// [16 + ib, 48) (the bucket is its top bits, the group its low bits), never
// 0, so 0 marks an empty slot.  Slots of a group fill in order and never
// empty, so a key can only sit before its group's first empty slot: the set
// is exact.  Buckets larger than a staging buffer read their keys from
// global memory.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) pc_dedup_fp_kernel(const uint32_t* off, uint64_t nbuckets,
                                                          const unsigned long long* keys, const uint32_t* bucket_doc,
                                                          unsigned long long* term_count, unsigned int* overflow,
                                                          uint32_t slots, uint32_t kcap, uint32_t nbuf,
                                                          uint32_t fp_test_mask, uint32_t fast) {
    extern __shared__ __align__(16) uint8_t dd_smem[];
    uint4* s_grp = reinterpret_cast<uint4*>(dd_smem);                                          // slots / 4 groups
    unsigned long long* s_buf = reinterpret_cast<unsigned long long*>(dd_smem + 4ull * slots); // nbuf x kcap keys
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_buf + static_cast<uint64_t>(nbuf) * kcap); // nbuf mbarriers
    uint16_t* s_queue = reinterpret_cast<uint16_t*>(s_bar + nbuf); // per warp: kDdQueue pending key indices
    if (threadIdx.x == 0) {
        for (uint32_t j = 0; j < nbuf; ++j) mbar_init(&s_bar[j], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t sg = static_cast<uint32_t>(__cvta_generic_to_shared(s_grp));
    // keys [o0, o0 + n) staged from the 16-byte aligned key o0 & ~1 (keys is 256-byte aligned)
    auto staged = [&](uint32_t o0, uint32_t n) { return n > 0 && ((n + (o0 & 1u) + 1u) & ~1u) <= kcap; };
    auto prefetch = [&](uint64_t t, uint32_t b) {
        const uint32_t o0 = off[t], n = off[t + 1] - o0;
        if (staged(o0, n)) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // (after the generic reads of the buffer)
            bulk_load(s_buf + b * kcap, keys + (o0 & ~1u), 8u * ((n + (o0 & 1u) + 1u) & ~1u), &s_bar[b]);
        }
    };
    if (threadIdx.x == 0 && blockIdx.x < nbuckets) prefetch(blockIdx.x, 0);
    uint32_t phase = 0; // parity bit per buffer
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < nbuckets; t += gridDim.x, ++it) {
        const uint32_t b = nbuf > 1 ? (it & 1u) : 0u;
        // (buffer b ^ 1 was released by the barrier that ended the previous bucket)
        if (nbuf > 1 && threadIdx.x == 0 && t + gridDim.x < nbuckets) prefetch(t + gridDim.x, b ^ 1u);
        const uint32_t o0 = off[t], n = off[t + 1] - o0;
        if (n == 0) {
            if (nbuf == 1 && threadIdx.x == 0 && t + gridDim.x < nbuckets) prefetch(t + gridDim.x, 0);
            continue; // uniform over the CTA
        }
        const uint32_t ib = max(16, 32 - __clz(static_cast<int>(n - 1)));
        uint32_t G = 64; // groups: load <= 2/3 where the launch's slots allow
        while (G * 4 < kDdLoadNum * n / 2 && G * 4 < slots) G <<= 1;
        for (uint32_t j = threadIdx.x; j < G; j += THREADS) s_grp[j] = make_uint4(0u, 0u, 0u, 0u);
        const bool st = staged(o0, n);
        if (st) {
            mbar_wait(&s_bar[b], (phase >> b) & 1u);
            phase ^= 1u << b;
        }
        __syncthreads(); // set cleared, keys staged
        uint32_t mine = 0;
        bool stuck = ib > 28; // (a bucket of > 2^28 keys: the wave is recounted)
        if (!stuck) {
            const uint32_t imask = (1u << ib) - 1u;
            if (st && fast)
                dd_bucket_fast<THREADS, true>(n, sg, G - 1u, imask, ~imask & fp_test_mask,
                                              static_cast<uint32_t>(__cvta_generic_to_shared(s_buf + b * kcap + (o0 & 1u))),
                                              nullptr, s_queue, mine, stuck);
            else if (fast && n <= 65536u) // (queue entries are 16-bit key indices)
                dd_bucket_fast<THREADS, false>(n, sg, G - 1u, imask, ~imask & fp_test_mask, 0u, keys + o0, s_queue, mine,
                                               stuck);
            else if (st)
                dd_bucket<THREADS, true>(n, sg, G - 1u, imask, ~imask & fp_test_mask,
                                         static_cast<uint32_t>(__cvta_generic_to_shared(s_buf + b * kcap + (o0 & 1u))),
                                         nullptr, mine, stuck);
            else
                dd_bucket<THREADS, false>(n, sg, G - 1u, imask, ~imask & fp_test_mask, 0u, keys + o0, mine, stuck);
        }
        mine = __reduce_add_sync(0xffffffffu, mine);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&term_count[bucket_doc[t]], (unsigned long long)mine);
        if (stuck) atomicOr(overflow, 1u);
        __syncthreads(); // the set and buffer b are free again
        if (nbuf == 1 && threadIdx.x == 0 && t + gridDim.x < nbuckets) prefetch(t + gridDim.x, 0);
    }
}

// any byte outside {A,C,G,T} in [0, n)?  (without canonicalisation such
// windows need the byte path, which the partitioned count does not have)
__global__ void any_non_acgt_kernel(const uint8_t* p, uint64_t n, unsigned int* found) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t bad = 0;
    const uint64_t align = (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15;
    const uint64_t head = n < align ? n : align;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < head; i += stride) bad |= !acgt_bit(p[i]);
    const uint4* v = reinterpret_cast<const uint4*>(p + head);
    const uint64_t nv = (n - head) / 16;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 x = __ldcs(v + i);
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 16; ++k) bad |= !acgt_bit((w[k >> 2] >> (8 * (k & 3))) & 0xffu);
    }
    for (uint64_t i = head + nv * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        bad |= !acgt_bit(p[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(found, 1u);
}

// the set of byte values in [0, n) as a 256-bit mask (8 words)
__global__ void byte_set_kernel(const uint8_t* p, uint64_t n, unsigned int* set) {
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto add = [&](uint32_t b) {
        const uint32_t bit = 1u << (b & 31u), w = b >> 5;
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] |= w == static_cast<uint32_t>(k) ? bit : 0u;
    };
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t align = (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15;
    const uint64_t head = n < align ? n : align;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < head; i += stride) add(p[i]);
    const uint4* v = reinterpret_cast<const uint4*>(p + head);
    const uint64_t nv = (n - head) / 16;
    uint64_t mid = 0; // byte values 64..127 (letters): one 64-bit shift per byte instead of the 8-way select
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 x = __ldcs(v + i);
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((w[j] & 0xc0c0c0c0u) == 0x40404040u) {
#pragma unroll
                for (int k = 0; k < 4; ++k) mid |= 1ull << ((w[j] >> (8 * k)) & 63u);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) add((w[j] >> (8 * k)) & 0xffu);
            }
        }
    }
    m[2] |= static_cast<uint32_t>(mid);
    m[3] |= static_cast<uint32_t>(mid >> 32);
    for (uint64_t i = head + nv * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) add(p[i]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t r = __reduce_or_sync(0xffffffffu, m[k]);
        if ((threadIdx.x & 31) == 0 && r) atomicOr(set + k, r);
    }
}

// bucket -> document of a wave
__global__ void pc_bdoc_kernel(const PcDoc* docs, uint32_t ndocs, uint32_t* bucket_doc) {
    for (uint32_t i = blockIdx.x; i < ndocs; i += gridDim.x) {
        const PcDoc D = docs[i];
        for (uint32_t j = threadIdx.x; j < D.nbk; j += blockDim.x) bucket_doc[D.bucket0 + j] = D.doc;
    }
}

// ---- slab fill: the bits of 32 consecutive columns of a block are one u32
// per row -- a dense "slab" of w words.  A wave of such slabs (sized to stay
// L2-resident) is filled with atomicOr, then copied into the matrix's 4-byte
// column positions (one strided u32 store per row), instead of random
// read-modify-writes straight into the whole (HBM-sized) matrix.

struct SlabDoc {
    uint64_t run_lo, run_hi, seg_lo, seg_hi; // run and segment ranges of the document
    uint64_t slab;                   // u32 index of its slab's row 0 in the wave buffer
    uint64_t w, magic;
    uint32_t bit;                    // column % 32
};
// A run of <= kUnitGroups consecutive 32-column groups of one block, their
// slabs consecutive (group-major) in the stage buffer: copied into the
// payload row by row, 4 * ng contiguous bytes per row (whole 32-byte sectors
// when ng = 8, so DRAM sees no partial-sector writes).
struct CopyUnit {
    uint64_t src; // u32 index of the first group's row 0 in the stage
    uint64_t dst; // payload byte offset of (row 0, first group)
    uint64_t w;
    uint32_t ng, pitch;
};
constexpr uint32_t kUnitGroups = 8;

// Consecutive runs one fill thread rolls through: 16 when the windows are
// 2-bit codes (one roller warm-up per 128 windows), 1 when they may need the
// byte path (the window bytes are re-read, and neighbouring lanes should then
// read neighbouring bytes).
constexpr uint32_t kFillRunsDna = 16;

// every window of a document -> k bits of its slab column; one thread per
// `rpt` consecutive runs of one document (run_prefix counts those spans)
template <int QC>
#ifndef COBS_FILL_MINB
#define COBS_FILL_MINB 3
#endif
__global__ void __launch_bounds__(256, COBS_FILL_MINB) slab_fill_kernel(WinArgs a, const SlabDoc* docs,
                                                        const uint64_t* run_prefix, uint32_t ndocs,
                                                        unsigned int* slab, uint32_t rpt) {
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
        unsigned int* col = slab + D.slab;
        const unsigned int bit = 1u << D.bit;
        uint64_t g = D.run_lo + (t - run_prefix[lo]) * rpt;
        const uint64_t ge = min(D.run_hi, g + rpt);
        while (g < ge) {
            const uint64_t s = find_seg_in(a, g, D.seg_lo, D.seg_hi);
            const uint64_t rb = a.seg_rbase[s];
            const uint64_t len = a.seg_off[s + 1] - a.seg_off[s];
            const uint64_t W = len >= q ? len - q + 1 : 0;
            const uint64_t gend = min(ge, a.seg_rbase[s + 1]);
            const uint64_t j0 = (g - rb) * kBRun, j1 = min(W, (gend - rb) * kBRun);
            const uint8_t* sb = a.seqs + a.seg_off[s];
            auto put = [&](uint64_t j, bool dna, uint64_t code) {
                const uint8_t* w = sb + j;
                if (dna) {
                    if (a.k > 1 && q < 32) { // the seeds share the seed-independent multiplies
                        const XxhShort x = xxh_short_code<QC>(code, q);
                        for (uint32_t seed = 0; seed < a.k; ++seed)
                            atomicOr(col + fastmod(xxh_short_seed<QC>(x, q, seed), D.w, D.magic), bit);
                    } else {
                        for (uint32_t seed = 0; seed < a.k; ++seed)
                            atomicOr(col + fastmod(xxh64_code<QC>(code, q, seed), D.w, D.magic), bit);
                    }
                } else if (a.canonical) {
                    if (q <= 32 || !window_acgt(w, q)) return; // skipped (termizer.cpp:113-116)
                    const bool rc = choose_rc(w, q);
                    for (uint32_t seed = 0; seed < a.k; ++seed)
                        atomicOr(col + fastmod(xxh64_term(w, q, rc, seed), D.w, D.magic), bit);
                } else {
                    if (a.k > 1 && q < 32) {
                        const XxhShort x = xxh_short_term(w, q, false);
                        for (uint32_t seed = 0; seed < a.k; ++seed)
                            atomicOr(col + fastmod(xxh_short_seed<0>(x, q, seed), D.w, D.magic), bit);
                    } else {
                        for (uint32_t seed = 0; seed < a.k; ++seed)
                            atomicOr(col + fastmod(xxh64_term(w, q, false, seed), D.w, D.magic), bit);
                    }
                }
            };
            if (rpt == 1)
                roll_windows<QC>(sb, j0, j1, q, a.canonical != 0, put);
            else if (q <= 32)
                roll_range<QC, 1>(sb, j0, j1, q, a.canonical != 0, put);
            else
                for (uint64_t j = j0; j < j1; ++j) put(j, false, 0ull);
            g = gend;
        }
    }
}

__global__ void unit_copy_kernel(const CopyUnit* units, const uint64_t* prefix, uint32_t nunits,
                                 const unsigned int* stage, uint8_t* payload) {
    const uint64_t total = prefix[nunits];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nunits;
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (prefix[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        const CopyUnit U = units[lo];
        const uint64_t local = t - prefix[lo];
        const uint64_t r = local / U.ng, x = local - r * U.ng;
        *reinterpret_cast<unsigned int*>(payload + U.dst + r * U.pitch + 4 * x) = stage[U.src + x * U.w + r];
    }
}

// a sub-range of a DevBuf
struct BufView {
    void* ptr = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

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

// The partitioned count's workspace (two key buffers of <= 8 GB each and the
// per-wave arrays) is kept between builds: cudaFree of these buffers took
// 6-20 ms usually but 100-600 ms on some builds (profiles/r2/session5:
// free_timing.log, the `free=` column of the A/B logs), cudaMalloc 2-130 ms.
// One workspace per process, handed to one build at a time (a concurrent
// build allocates its own and frees it); released by cobs_gpu_trim(), by
// DevBuf::reserve when an allocation of this library runs out of memory, or
// with COBS_BUILD_CACHE=0 after every build.
struct CountWorkspace {
    DevBuf keys, keys_a, small;
    int device = -1;
    size_t bytes() const { return keys.bytes + keys_a.bytes + small.bytes; }
};
namespace {
std::mutex g_ws_mu;
CountWorkspace* g_ws = nullptr; // (leaked at exit: the runtime may be gone when statics die)
std::unique_ptr<CountWorkspace> acquire_count_ws(int device) {
    std::unique_ptr<CountWorkspace> ws;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        ws.reset(g_ws);
        g_ws = nullptr;
    }
    if (ws && ws->device != device) ws.reset(); // (its buffers are freed)
    if (!ws) {
        ws = std::make_unique<CountWorkspace>();
        ws->device = device;
    }
    return ws;
}
void release_count_ws(std::unique_ptr<CountWorkspace> ws) {
    const char* e = std::getenv("COBS_BUILD_CACHE");
    if (e && e[0] == '0') return; // freed here
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (!g_ws) g_ws = ws.release();
}
} // namespace
size_t trim_device_caches() {
    std::unique_ptr<CountWorkspace> ws;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        ws.reset(g_ws);
        g_ws = nullptr;
    }
    return ws ? ws->bytes() : 0;
}

std::unique_ptr<DeviceIndex> build_device_index(const uint8_t* seqs, const uint64_t* seg_off,
                                                uint64_t n_segs, const uint64_t* doc_segs,
                                                const std::vector<std::string>& names, const Params& P,
                                                uint8_t kind, uint64_t forced_w, int device,
                                                bool seqs_on_device, bool terms_input, bool seg_ptrs) {
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

    DevBuf d_seqs, d_segoff, d_segw, d_segdoc, d_docstart, d_tc;
    if (!seqs_on_device) d_seqs.reserve(std::max<uint64_t>(total_bytes, 1));
    d_segoff.reserve(8 * (n_segs + 1));
    d_segw.reserve(8 * (n_segs + 1));
    d_segdoc.reserve(4 * std::max<uint64_t>(n_segs, 1));
    d_docstart.reserve(8 * n_docs);
    d_tc.reserve(8 * n_docs);
    auto t_h2d = std::chrono::steady_clock::now();
    if (seg_ptrs) // one host pointer per string (COBS_B_SEGMENT_PTRS)
        h2d_gather_staged(d_seqs.ptr, reinterpret_cast<const uint8_t* const*>(seqs), seg_off, n_segs, st);
    else if (!seqs_on_device)
        h2d_staged(d_seqs.ptr, seqs, total_bytes, st);
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

    NvtxPhase phase;
    phase.begin("cobs.build.count");
    // ---- count pass, in waves of documents whose sets fit in L2 ---------
    // (random CAS into L2-resident sets instead of DRAM; a document larger
    // than a wave gets a wave of its own)
    uint64_t slab_wave_bytes = 96ull << 20;
    if (const char* e = std::getenv("COBS_SLAB_WAVE_MB")) slab_wave_bytes = std::strtoull(e, nullptr, 10) << 20;
    std::vector<uint64_t> tc(n_docs);
    std::chrono::steady_clock::time_point t_count0 = std::chrono::steady_clock::now();
    uint32_t fill_rpt = 1; // kFillRunsDna once the count has seen only 2-bit-code windows
    if (terms_input) { // TermSet::term_count() = terms.size() (termizer.hpp:25)
        for (uint64_t d = 0; d < n_docs; ++d) tc[d] = doc_segs[d + 1] - doc_segs[d];
    } else {
        size_t free_b = 0, total_b = 0;
        // exact distinct counts by hash-set insertion (any q, any bytes) for
        // documents [d_lo, d_hi), in waves whose sets stay L2-resident
        auto hashset_count = [&](uint64_t d_lo, uint64_t d_hi) {
            std::vector<uint64_t> tab_off(n_docs), tab_slots(n_docs);
            uint64_t load_div = 4; // slots >= load_div/2 * windows (load <= 2/load_div)
            if (const char* e = std::getenv("COBS_COUNT_LOAD_DIV")) load_div = std::max<uint64_t>(2, std::strtoull(e, nullptr, 10));
            for (uint64_t d = d_lo; d < d_hi; ++d) tab_slots[d] = next_pow2(doc_w[d] * load_div / 2 + 1);
            COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
            uint64_t wave_bytes = 192ull << 20;
            if (const char* e = std::getenv("COBS_COUNT_WAVE_MB")) wave_bytes = std::strtoull(e, nullptr, 10) << 20;
            const uint64_t budget_slots = std::max<uint64_t>(std::min<uint64_t>((free_b / 3) / 8, wave_bytes / 8), 1ull << 16);
            std::vector<uint64_t> wave_lo{d_lo};
            uint64_t max_slots = 0;
            for (uint64_t d0 = d_lo; d0 < d_hi;) {
                uint64_t d1 = d0, slots = 0;
                while (d1 < d_hi && (d1 == d0 || slots + tab_slots[d1] <= budget_slots)) {
                    tab_off[d1] = slots; // relative to the wave's tables
                    slots += tab_slots[d1];
                    ++d1;
                }
                max_slots = std::max(max_slots, slots);
                wave_lo.push_back(d1);
                d0 = d1;
            }
            DevBuf d_tab, d_taboff, d_tabslots;
            d_taboff.reserve(8 * n_docs);
            d_tabslots.reserve(8 * n_docs);
            d_tab.reserve(8 * std::max<uint64_t>(max_slots, 1));
            COBS_CUDA(cudaMemcpyAsync(d_tabslots.ptr, tab_slots.data(), 8 * n_docs, cudaMemcpyHostToDevice, st));
            COBS_CUDA(cudaMemcpyAsync(d_taboff.ptr, tab_off.data(), 8 * n_docs, cudaMemcpyHostToDevice, st));
            // (short runs per lane on purpose: a CTA's windows stay within one
            // or two documents, so the sets it touches stay L2-resident)
            auto ck = q == 31 ? count_kernel<31> : count_kernel<0>;
            const uint64_t span = kChunkRuns;
            for (size_t wv = 0; wv + 1 < wave_lo.size(); ++wv) {
                const uint64_t d0 = wave_lo[wv], d1 = wave_lo[wv + 1];
                const uint64_t slots = tab_off[d1 - 1] + tab_slots[d1 - 1];
                COBS_CUDA(cudaMemsetAsync(d_tab.ptr, 0, 8 * slots, st));
                WinArgs w = wa;
                w.seg_lo = doc_segs[d0];
                w.seg_hi = doc_segs[d1];
                w.r_lo = seg_rbase[w.seg_lo];
                w.r_hi = seg_rbase[w.seg_hi];
                if (w.r_hi > w.r_lo) {
                    const uint64_t runs = w.r_hi - w.r_lo;
                    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(148 * 8, (runs + span - 1) / span));
                    ck<<<grid, 256, 0, st>>>(w, d_tab.as<unsigned long long>(), d_taboff.as<uint64_t>(),
                                             d_tabslots.as<uint64_t>(), d_tc.as<unsigned long long>());
                    COBS_CUDA(cudaGetLastError());
                }
            }
            COBS_CUDA(cudaStreamSynchronize(st)); // tables die with this scope
        };

        // symbol codes for raw-byte corpora over a small alphabet (see SymRoller)
        uint32_t sym_bits = 0;
        DevBuf d_symtab;
        d_symtab.reserve(256);

        // partitioned count for q <= 32 (see pc_hist_kernel), in waves of
        // documents whose windows fit the key buffer; a wave that meets a
        // window needing the byte path (non-ACGT, no canonicalisation) or a
        // bucket too skewed for its set is recounted by hashset_count
        auto partitioned_count = [&] {
            COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
            // two key buffers (super-bucket scatter, final placement), 16 bytes
            // per window.  A wave holds <= kPcWaveKeys windows (16 GB of key
            // buffers): the kernels' time does not depend on the wave size
            // (C3: 1,316-1,320 ms with 85 GB / 20 waves, 1,327-1,333 ms with
            // 16 GB / 73 waves), but cudaFree of the 85 GB took 500+ ms on
            // about one build in five (6-20 ms otherwise; profiles/r2/free_timing)
            // against 6-8 ms for 16 GB, and the caller keeps its HBM.
            // (a document larger than that still gets a wave of its own while it fits half the free HBM)
            const uint64_t kmem = std::min<uint64_t>((free_b / 2) / 16, 0xffffffffull);
            uint64_t kmax = std::min(kmem, std::max(kPcWaveKeys, doc_w.empty() ? 0 : *std::max_element(doc_w.begin(), doc_w.end())));
            if (const char* e = std::getenv("COBS_PC_WAVE_KEYS")) kmax = std::min<uint64_t>(kmem, std::strtoull(e, nullptr, 10));
            kmax = std::max<uint64_t>(kmax, 1);
            uint64_t target = kPcTarget; // keys per bucket (A/B knob COBS_PC_TARGET)
            if (const char* e = std::getenv("COBS_PC_TARGET")) target = std::max<uint64_t>(64, std::strtoull(e, nullptr, 10));
            const uint64_t max_buckets = kmax / (target / 2) + 2 * n_docs + 1;
            // plan every wave up front (documents in order, keys <= kmax); the
            // waves then run back to back without a host round trip
            struct PcWave { uint64_t d0, d1, doc0, nbuck, nchunk, slots, keys, nsup, kcap; };
            std::vector<PcWave> pw;
            std::vector<PcDoc> pd;
            std::vector<std::pair<uint64_t, uint64_t>> oversize; // documents beyond the key buffer
            for (uint64_t d0 = 0; d0 < n_docs;) {
                PcWave wv{d0, d0, pd.size(), 0, 0, 256, 0, 0, 2};
                uint64_t d1 = d0;
                while (d1 < n_docs) {
                    const uint64_t W = doc_w[d1];
                    uint64_t nbk = 1;
                    while (nbk * target < W && nbk < kPcHist) nbk <<= 1;
                    // the set must hold a bucket's distinct keys: mean W / nbk
                    // + 6 sigma of a bucket's key count, at load <= 2/3
                    const uint64_t mean = (W + nbk - 1) / nbk;
                    const double fullest = mean + 6.0 * std::sqrt(static_cast<double>(mean));
                    uint64_t slots = 256;
                    while (slots < 1.5 * fullest + 256 && slots < kPcMaxSlotsFp) slots <<= 1;
                    if (const char* e = std::getenv("COBS_PC_SLOTS_CAP")) // tests: sets too small -> recount
                        slots = std::max<uint64_t>(256, std::min<uint64_t>(slots, std::strtoull(e, nullptr, 10)));
                    if (d1 > d0 && (wv.keys + W > kmax || wv.nbuck + nbk > max_buckets)) break;
                    wv.slots = std::max(wv.slots, slots);
                    wv.kcap = std::max<uint64_t>(wv.kcap, (static_cast<uint64_t>(fullest) + 4) & ~1ull);
                    PcDoc D{};
                    D.seg_lo = doc_segs[d1];
                    D.seg_hi = doc_segs[d1 + 1];
                    D.run_lo = seg_rbase[D.seg_lo];
                    D.run_hi = seg_rbase[D.seg_hi];
                    D.chunk0 = wv.nchunk;
                    D.bucket0 = wv.nbuck;
                    D.nbk = static_cast<uint32_t>(nbk);
                    D.shift = 64 - static_cast<uint32_t>(__builtin_ctzll(nbk));
                    D.doc = static_cast<uint32_t>(d1);
                    D.sb0 = static_cast<uint32_t>(wv.nsup);
                    D.tpr = kPcRunsPerThread;
                    pd.push_back(D);
                    wv.nsup += nbk >> pc_super_shift_lg(static_cast<uint32_t>(__builtin_ctzll(nbk)));
                    wv.keys += W;
                    wv.nbuck += nbk;
                    wv.nchunk += (D.run_hi - D.run_lo + kPcRuns - 1) / kPcRuns;
                    ++d1;
                }
                wv.d1 = d1;
                if (wv.keys > kmax || wv.nbuck > max_buckets) {
                    pd.resize(wv.doc0);
                    oversize.push_back({d0, d1});
                } else {
                    pw.push_back(wv);
                }
                d0 = d1;
            }
            uint64_t max_keys = 1, max_nbuck = 1, max_nsup = 1, max_nchunk = 1;
            for (const PcWave& wv : pw) {
                max_keys = std::max(max_keys, wv.keys);
                max_nbuck = std::max(max_nbuck, wv.nbuck);
                max_nsup = std::max(max_nsup, wv.nsup);
                max_nchunk = std::max(max_nchunk, wv.nchunk);
            }
            // Wave i's histogram pass (+ scan, super-bucket cursors) runs on a
            // second stream while wave i-1 is scattered and deduplicated, so
            // its rolling overlaps their memory/latency-bound kernels; the
            // per-wave arrays are double-buffered (A/B knob COBS_PC_OVERLAP=0).
            const auto t_alloc = std::chrono::steady_clock::now();
            const char* ov_env = std::getenv("COBS_PC_OVERLAP");
            const bool overlap = !(ov_env && ov_env[0] == '0');
            std::unique_ptr<CountWorkspace> cws = acquire_count_ws(device);
            DevBuf &d_keys = cws->keys, &d_keys_a = cws->keys_a, &d_small = cws->small;
            d_keys.reserve(8 * max_keys + 16); // (+16: the dedup's 16-byte staged copies may read one key past the end)
            d_keys_a.reserve(8 * max_keys);
            // the per-wave arrays: views into one allocation (one cudaMalloc / cudaFree instead of ~20)
            BufView d_docs, d_flags, d_sup_cur[2], d_sup_doc[2], d_cnt[2], d_off[2], d_tmp[2], d_bdoc[2], d_chunk_sup[2];
            size_t tmp_bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                          static_cast<int>(max_nbuck + 1), st);
            std::vector<std::pair<BufView*, size_t>> plan{{&d_flags, 64 * std::max<size_t>(pw.size(), 1)}, // per wave: bad, overflow, 3 work counters
                                                       {&d_docs, sizeof(PcDoc) * std::max<size_t>(pd.size(), 1)}};
            for (int b = 0; b < (overlap ? 2 : 1); ++b) {
                plan.push_back({&d_chunk_sup[b], 4ull * kSup * max_nchunk});
                plan.push_back({&d_sup_cur[b], 4 * max_nsup});
                plan.push_back({&d_sup_doc[b], 4 * max_nsup});
                plan.push_back({&d_cnt[b], 4 * (max_nbuck + 1)});
                plan.push_back({&d_off[b], 4 * (max_nbuck + 1)});
                plan.push_back({&d_bdoc[b], 4 * (max_nbuck + 1)});
                plan.push_back({&d_tmp[b], std::max<size_t>(tmp_bytes, 16)});
            }
            size_t arena = 0;
            for (auto& v : plan) arena += (v.second + 255) & ~size_t(255);
            d_small.reserve(arena);
            size_t o = 0;
            for (auto& v : plan) {
                v.first->ptr = static_cast<uint8_t*>(d_small.ptr) + o;
                v.first->bytes = v.second;
                o += (v.second + 255) & ~size_t(255);
            }
            g_timing.ms_count_alloc = ms_since(t_alloc);
            Event ek0, ek1; // the kernels alone: after the allocation, before the frees
            COBS_CUDA(cudaEventRecord(ek0, st));
            if (!pd.empty())
                COBS_CUDA(cudaMemcpyAsync(d_docs.ptr, pd.data(), sizeof(PcDoc) * pd.size(), cudaMemcpyHostToDevice, st));
            COBS_CUDA(cudaMemsetAsync(d_flags.ptr, 0, 64 * std::max<size_t>(pw.size(), 1), st));
            cudaStream_t hs = st;
            if (overlap) COBS_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
            struct HsGuard {
                cudaStream_t s, main;
                ~HsGuard() {
                    if (s != main) cudaStreamDestroy(s);
                }
            } hsg{hs, st};
            Event ev_ready(cudaEventDisableTiming), ev_hist[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)},
                  ev_done[2] = {Event(cudaEventDisableTiming), Event(cudaEventDisableTiming)};
            COBS_CUDA(cudaEventRecord(ev_ready, st));
            COBS_CUDA(cudaStreamWaitEvent(hs, ev_ready, 0));
            auto hist = sym_bits ? pc_hist_kernel<0, kSymBits> : q == 31 ? pc_hist_kernel<31> : pc_hist_kernel<0>;
            auto scat = sym_bits ? pc_scatter_super_kernel<0, kSymBits>
                        : q == 31 ? pc_scatter_super_kernel<31> : pc_scatter_super_kernel<0>;
            // dedup CTA size (A/B knob COBS_PC_DEDUP_THREADS = 256 / 512: within noise)
            const char* dt_env = std::getenv("COBS_PC_DEDUP_THREADS");
            const bool dd512 = dt_env && std::atoi(dt_env) >= 512;
            auto dedup = dd512 ? pc_dedup_fp_kernel<512> : pc_dedup_fp_kernel<256>;
            // set + key staging buffer(s) + mbarrier(s) (a wave's kcap is capped so this fits)
            uint32_t nbuf = 1; // key staging buffers (A/B knob COBS_PC_DD_NBUF = 1 / 2; 1: more CTAs per SM, faster)
            if (const char* e = std::getenv("COBS_PC_DD_NBUF")) nbuf = std::atoi(e) == 1 ? 1u : 2u;
            const uint64_t dd_queue = 2ull * kDdQueue * ((dd512 ? 512 : 256) / 32); // the warps' pending-key queues
            auto dd_smem = [&](uint64_t slots, uint64_t kcap) {
                return static_cast<size_t>(4 * slots + nbuf * (8 * kcap + 8) + dd_queue);
            };
            COBS_CUDA(cudaFuncSetAttribute(dedup, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            // tests narrow the fingerprints to force accidental matches (COBS_PC_FP_MASK, e.g. 0x30000)
            const uint32_t fp_test_mask = std::getenv("COBS_PC_FP_MASK")
                                              ? static_cast<uint32_t>(std::strtoul(std::getenv("COBS_PC_FP_MASK"), nullptr, 0))
                                              : 0xffffffffu;
            // straight-line first probes in the dedup (A/B knob COBS_PC_DD_FAST=0: the per-key probe loop)
            const char* df_env = std::getenv("COBS_PC_DD_FAST");
            const uint32_t dd_fast = !(df_env && df_env[0] == '0');
            // keys read from global memory one step ahead, or (A/B knob COBS_PC_DD_STAGE=1) staged in shared
            // memory by the bulk-copy engine: twice the shared memory per CTA, half the warps per SM
            // (C3 count kernels 1,173 vs 1,246 ms)
            const char* ds_env = std::getenv("COBS_PC_DD_STAGE");
            const bool dd_stage = ds_env && ds_env[0] == '1';
            for (size_t i = 0; i < pw.size(); ++i) {
                const PcWave& wv = pw[i];
                if (!wv.nchunk) continue;
                const int b = overlap ? static_cast<int>(i & 1) : 0;
                const uint32_t nd = static_cast<uint32_t>(wv.d1 - wv.d0);
                unsigned long long* flags = d_flags.as<unsigned long long>() + 8 * i;
                PcArgs pa{};
                pa.a = wa;
                pa.docs = d_docs.as<PcDoc>() + wv.doc0;
                pa.ndocs = nd;
                pa.nchunks = wv.nchunk;
                pa.bucket_cnt = d_cnt[b].as<uint32_t>();
                pa.keys = d_keys_a.as<unsigned long long>();
                pa.bad = flags;
                pa.chunk_sup = d_chunk_sup[b].as<uint32_t>();
                pa.symtab = d_symtab.as<uint8_t>();
                pa.work = flags + 2;
                const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(148 * 6, wv.nchunk)));
                // histogram side (buffers b are free once wave i-2's dedup is done)
                COBS_CUDA(cudaStreamWaitEvent(hs, ev_done[b], 0));
                COBS_CUDA(cudaMemsetAsync(d_cnt[b].ptr, 0, 4 * (wv.nbuck + 1), hs));
                pc_bdoc_kernel<<<std::min<uint32_t>(nd, 148 * 8), 256, 0, hs>>>(d_docs.as<PcDoc>() + wv.doc0, nd,
                                                                               d_bdoc[b].as<uint32_t>());
                hist<<<grid, 256, 0, hs>>>(pa);
                size_t tb = d_tmp[b].bytes;
                COBS_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp[b].ptr, tb, d_cnt[b].as<uint32_t>(), d_off[b].as<uint32_t>(),
                                                        static_cast<int>(wv.nbuck + 1), hs));
                pc_super_init_kernel<<<std::min<uint32_t>(nd, 148 * 8), kSup, 0, hs>>>(
                    d_docs.as<PcDoc>() + wv.doc0, nd, d_off[b].as<uint32_t>(), d_sup_cur[b].as<uint32_t>(),
                    d_sup_doc[b].as<uint32_t>());
                COBS_CUDA(cudaEventRecord(ev_hist[b], hs));
                // key side
                COBS_CUDA(cudaStreamWaitEvent(st, ev_hist[b], 0));
                scat<<<grid, 256, 0, st>>>(pa, d_sup_cur[b].as<uint32_t>());
                pc_scatter_final_kernel<<<static_cast<unsigned>(std::min<uint64_t>(148 * 8, wv.nsup)), 256, 0, st>>>(
                    d_docs.as<PcDoc>() + wv.doc0, d_sup_doc[b].as<uint32_t>(), wv.nsup, d_off[b].as<uint32_t>(),
                    d_keys_a.as<unsigned long long>(), d_keys.as<unsigned long long>(), flags + 4);
                const uint64_t kcap = !dd_stage ? 0 : std::min<uint64_t>(wv.kcap, ((227 * 1024 - dd_queue - 4 * wv.slots) / nbuf / 8 - 1) & ~1ull);
                dedup<<<static_cast<unsigned>(std::min<uint64_t>(148 * 64, wv.nbuck)), dd512 ? 512 : 256,
                        dd_smem(wv.slots, kcap), st>>>(
                    d_off[b].as<uint32_t>(), wv.nbuck, d_keys.as<unsigned long long>(), d_bdoc[b].as<uint32_t>(),
                    d_tc.as<unsigned long long>(), reinterpret_cast<unsigned int*>(flags + 1),
                    static_cast<uint32_t>(wv.slots), static_cast<uint32_t>(kcap), nbuf, fp_test_mask, dd_fast);
                COBS_CUDA(cudaEventRecord(ev_done[b], st));
                COBS_CUDA(cudaGetLastError());
            }
            g_timing.count_waves = static_cast<uint32_t>(pw.size());
            std::vector<uint64_t> flags(8 * pw.size());
            if (!pw.empty())
                COBS_CUDA(cudaMemcpyAsync(flags.data(), d_flags.ptr, 64 * pw.size(), cudaMemcpyDeviceToHost, st));
            COBS_CUDA(cudaEventRecord(ek1, st));
            COBS_CUDA(cudaStreamSynchronize(st));
            {
                float ms_k = 0;
                cudaEventElapsedTime(&ms_k, ek0, ek1);
                g_timing.ms_count_kernels = ms_k;
            }
            g_timing.ms_count_sync = ms_since(t_count0);
            const auto t_free = std::chrono::steady_clock::now();
            // (a recount that runs out of memory gets it back through DevBuf::reserve)
            if (cws->bytes() <= 16 * kPcWaveKeys + (1ull << 30))
                release_count_ws(std::move(cws)); // kept for the next build
            cws.reset();
            g_timing.ms_count_free = ms_since(t_free);
            bool byte_windows = !oversize.empty() || sym_bits; // symbol-coded windows hash their bytes in the fill
            for (size_t i = 0; i < pw.size(); ++i) byte_windows |= flags[8 * i] != 0;
            if (!byte_windows) fill_rpt = kFillRunsDna;
            const auto t_recount = std::chrono::steady_clock::now();
            for (size_t i = 0; i < pw.size(); ++i)
                if (flags[8 * i] || (flags[8 * i + 1] & 0xffffffffull)) { // recount this wave exactly
                    COBS_CUDA(cudaMemsetAsync(d_tc.as<unsigned long long>() + pw[i].d0, 0, 8 * (pw[i].d1 - pw[i].d0), st));
                    hashset_count(pw[i].d0, pw[i].d1);
                    ++g_timing.count_fallback_waves;
                }
            for (const auto& r : oversize) hashset_count(r.first, r.second);
            if (g_timing.count_fallback_waves || !oversize.empty()) g_timing.ms_count_kernels += ms_since(t_recount);
        };

        COBS_CUDA(cudaEventRecord(e0, st));
        t_count0 = std::chrono::steady_clock::now();
        const char* pc_env = std::getenv("COBS_COUNT_PARTITION");
        // (small corpora: the hash sets are L2-resident anyway and need no
        // key buffer; COBS_COUNT_PARTITION=1 forces the partitioned count)
        uint64_t total_w = 0;
        for (uint64_t d = 0; d < n_docs; ++d) total_w += doc_w[d];
        // (codes_exact: q = 32 without canonicalisation has no spare key value)
        bool use_pc = codes_exact(q, wa.canonical != 0) &&
                      (pc_env ? pc_env[0] == '1' : total_w >= (1ull << 30));
        const char* scan_env = std::getenv("COBS_PC_NO_SCAN"); // tests: reach the per-wave fallback
        if (use_pc && !wa.canonical && total_bytes && !(scan_env && scan_env[0] == '1')) {
            // byte-path windows ahead? then the hash sets straight away
            DevBuf d_found;
            d_found.reserve(4);
            COBS_CUDA(cudaMemsetAsync(d_found.ptr, 0, 4, st));
            any_non_acgt_kernel<<<148 * 8, 256, 0, st>>>(wa.seqs, total_bytes, d_found.as<unsigned int>());
            uint32_t found = 0;
            COBS_CUDA(cudaMemcpyAsync(&found, d_found.ptr, 4, cudaMemcpyDeviceToHost, st));
            COBS_CUDA(cudaStreamSynchronize(st));
            use_pc = found == 0;
            const char* sym_env = std::getenv("COBS_PC_SYMBOLS");
            if (found && q * kSymBits <= 62 && !(sym_env && sym_env[0] == '0')) {
                // raw bytes: if the corpus has <= 2^kSymBits distinct byte values, every
                // window is an exact kSymBits-per-symbol code and the partitioned count applies
                DevBuf d_set;
                d_set.reserve(32);
                COBS_CUDA(cudaMemsetAsync(d_set.ptr, 0, 32, st));
                byte_set_kernel<<<148 * 8, 256, 0, st>>>(wa.seqs, total_bytes, d_set.as<unsigned int>());
                uint32_t set[8];
                COBS_CUDA(cudaMemcpyAsync(set, d_set.ptr, 32, cudaMemcpyDeviceToHost, st));
                COBS_CUDA(cudaStreamSynchronize(st));
                std::vector<uint8_t> tab(256, 0xff);
                uint32_t nsym = 0;
                for (uint32_t b = 0; b < 256; ++b)
                    if ((set[b >> 5] >> (b & 31)) & 1u) tab[b] = static_cast<uint8_t>(nsym++);
                if (nsym <= (1u << kSymBits)) {
                    COBS_CUDA(cudaMemcpyAsync(d_symtab.ptr, tab.data(), 256, cudaMemcpyHostToDevice, st));
                    sym_bits = kSymBits;
                    use_pc = true;
                }
            }
        }
        if (use_pc)
            partitioned_count();
        else
            hashset_count(0, n_docs);
        COBS_CUDA(cudaEventRecord(e1, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        float ms_count = 0;
        cudaEventElapsedTime(&ms_count, e0, e1);
        g_timing.ms_count = ms_count;
        if (!use_pc) g_timing.ms_count_kernels = ms_count; // (hash sets: small tables, allocation included)
        if (std::getenv("COBS_BUILD_DEBUG"))
            std::fprintf(stderr, "[cobs build] count %.1f ms (kernels %.1f): partitioned=%d waves=%u recounted=%u fill_rpt=%u alloc=%.1f sync=%.1f free=%.1f ms\n",
                         ms_count, g_timing.ms_count_kernels, use_pc ? 1 : 0, g_timing.count_waves,
                         g_timing.count_fallback_waves, fill_rpt, g_timing.ms_count_alloc, g_timing.ms_count_sync,
                         g_timing.ms_count_free);
        COBS_CUDA(cudaMemcpy(tc.data(), d_tc.ptr, 8 * n_docs, cudaMemcpyDeviceToHost));
    }

    const double ms_at_count_end = ms_since(t_start);
    phase.begin("cobs.build.sizing");
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

    phase.begin("cobs.build.fill");
    // ---- fill pass, straight into the pitched HBM layout of a DeviceIndex
    const double ms_at_sizing_end = ms_since(t_start);
    auto ix = std::make_unique<DeviceIndex>();
    ix->meta = std::move(meta);
    ix->device = device;
    ix->allocate(); // refuses a matrix that does not fit in free HBM
    const double ms_at_alloc_end = ms_since(t_start);
    COBS_CUDA(cudaMemsetAsync(ix->payload, 0, ix->payload_bytes, ix->stream));
    COBS_CUDA(cudaStreamSynchronize(ix->stream));
    const double ms_at_memset_end = ms_since(t_start);
    COBS_CUDA(cudaEventRecord(e2, st));
    wa.seg_lo = 0;
    wa.seg_hi = n_segs;
    if (total_runs > 0) {
        // Stage batches of whole copy units (<= 8 consecutive groups of one
        // block, slabs group-major); inside a batch, fill waves of whole
        // groups whose slabs stay L2-resident (<= slab_wave_bytes); after a
        // batch's waves, one unit_copy launch moves it into the payload.
        std::vector<SlabDoc> sdocs;
        std::vector<uint64_t> run_prefix; // per fill wave: ndocs+1 entries (concatenated)
        std::vector<CopyUnit> units;
        std::vector<uint64_t> unit_prefix; // per batch: nunits+1 entries (concatenated)
        struct Wave { size_t doc0, ndocs, rp0; uint64_t w_lo, w_hi; };
        struct Batch { size_t wave0, nwaves, unit0, nunits, up0; };
        std::vector<Wave> waves;
        std::vector<Batch> batches;
        uint64_t max_w = 1;
        for (uint64_t b = 0; b < nb; ++b) max_w = std::max<uint64_t>(max_w, ix->blocks[b].w);
        const uint64_t wave_words = std::max<uint64_t>(slab_wave_bytes / 4, 1);
        const uint64_t stage_words = std::max<uint64_t>(kUnitGroups * max_w, std::max<uint64_t>(wave_words, 64ull << 20));
        uint64_t words = 0, max_words = 0; // stage fill of the open batch
        bool wave_open = false, batch_open = false;
        auto close_wave = [&] {
            if (!wave_open) return;
            waves.back().w_hi = words;
            wave_open = false;
        };
        auto close_batch = [&] {
            if (!batch_open) return;
            close_wave();
            Batch& B = batches.back();
            B.nwaves = waves.size() - B.wave0;
            B.nunits = units.size() - B.unit0;
            max_words = std::max(max_words, words);
            words = 0;
            batch_open = false;
        };
        for (uint64_t b = 0; b < nb; ++b) {
            const DevBlock& d = ix->blocks[b];
            const uint64_t ngr = (d.dc + 31) / 32;
            for (uint64_t g0 = 0; g0 < ngr; g0 += kUnitGroups) {
                const uint32_t ng = static_cast<uint32_t>(std::min<uint64_t>(kUnitGroups, ngr - g0));
                if (batch_open && words + ng * d.w > stage_words) close_batch();
                if (!batch_open) {
                    batches.push_back(Batch{waves.size(), 0, units.size(), 0, unit_prefix.size()});
                    unit_prefix.push_back(0);
                    batch_open = true;
                }
                units.push_back(CopyUnit{words, d.base + 4 * g0, d.w, ng, d.pitch});
                unit_prefix.push_back(unit_prefix.back() + ng * d.w);
                for (uint64_t gi = g0; gi < g0 + ng; ++gi) {
                    if (wave_open && words + d.w - waves.back().w_lo > wave_words) close_wave();
                    if (!wave_open) {
                        waves.push_back(Wave{sdocs.size(), 0, run_prefix.size(), words, words});
                        run_prefix.push_back(0);
                        wave_open = true;
                    }
                    Wave& wv = waves.back();
                    for (uint64_t c = 32 * gi; c < std::min<uint64_t>(d.dc, 32 * gi + 32); ++c) {
                        const uint64_t doc = order[d.doc_base + c];
                        SlabDoc D{};
                        D.seg_lo = doc_segs[doc];
                        D.seg_hi = doc_segs[doc + 1];
                        D.run_lo = seg_rbase[D.seg_lo];
                        D.run_hi = seg_rbase[D.seg_hi];
                        D.slab = words;
                        D.w = d.w;
                        D.magic = d.magic;
                        D.bit = static_cast<uint32_t>(c % 32);
                        sdocs.push_back(D);
                        run_prefix.push_back(run_prefix.back() + (D.run_hi - D.run_lo + fill_rpt - 1) / fill_rpt);
                        ++wv.ndocs;
                    }
                    words += d.w;
                }
            }
        }
        close_batch();
        DevBuf d_sdocs, d_rp, d_units, d_up, d_slab;
        d_sdocs.reserve(sizeof(SlabDoc) * std::max<size_t>(sdocs.size(), 1));
        d_rp.reserve(8 * run_prefix.size());
        d_units.reserve(sizeof(CopyUnit) * std::max<size_t>(units.size(), 1));
        d_up.reserve(8 * unit_prefix.size());
        d_slab.reserve(4 * std::max<uint64_t>(max_words, 1));
        COBS_CUDA(cudaMemcpyAsync(d_sdocs.ptr, sdocs.data(), sizeof(SlabDoc) * sdocs.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_rp.ptr, run_prefix.data(), 8 * run_prefix.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_units.ptr, units.data(), sizeof(CopyUnit) * units.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaMemcpyAsync(d_up.ptr, unit_prefix.data(), 8 * unit_prefix.size(), cudaMemcpyHostToDevice, st));
        COBS_CUDA(cudaEventRecord(e2, st));
        auto fk = q == 31 ? slab_fill_kernel<31> : slab_fill_kernel<0>;
        // (a grid of one resident round, 148 x 3 CTAs, measured slower: C3 fill 1,076 vs 1,017 ms, C4 273 vs 254)
        const uint64_t fill_grid = 148 * 16;
        for (const Batch& B : batches) {
            for (size_t i = B.wave0; i < B.wave0 + B.nwaves; ++i) {
                const Wave& wv = waves[i];
                COBS_CUDA(cudaMemsetAsync(d_slab.as<unsigned int>() + wv.w_lo, 0, 4 * (wv.w_hi - wv.w_lo), st));
                const uint64_t runs = run_prefix[wv.rp0 + wv.ndocs];
                if (runs > 0)
                    fk<<<static_cast<unsigned>(std::min<uint64_t>(fill_grid, (runs + 255) / 256)), 256, 0, st>>>(
                        wa, d_sdocs.as<SlabDoc>() + wv.doc0, d_rp.as<uint64_t>() + wv.rp0,
                        static_cast<uint32_t>(wv.ndocs), d_slab.as<unsigned int>(), fill_rpt);
                COBS_CUDA(cudaGetLastError());
            }
            const uint64_t total = unit_prefix[B.up0 + B.nunits];
            unit_copy_kernel<<<static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(148 * 16, (total + 255) / 256))),
                               256, 0, st>>>(d_units.as<CopyUnit>() + B.unit0, d_up.as<uint64_t>() + B.up0,
                                             static_cast<uint32_t>(B.nunits), d_slab.as<unsigned int>(), ix->payload);
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
    const double ms_at_fill_end = ms_since(t_start);
    ix->finish_upload();
    g_timing.ms_total = ms_since(t_start);
    if (std::getenv("COBS_BUILD_DEBUG"))
        std::fprintf(stderr, "[cobs build] call %.1f ms: count done at %.1f, sizing %.1f, matrix alloc %.1f, memset %.1f, "
                             "fill (setup + kernels %.1f) done at %.1f, finish %.1f\n",
                     g_timing.ms_total, ms_at_count_end, ms_at_sizing_end - ms_at_count_end,
                     ms_at_alloc_end - ms_at_sizing_end, ms_at_memset_end - ms_at_alloc_end, ms_fill, ms_at_fill_end,
                     g_timing.ms_total - ms_at_fill_end);
    return ix;
}

uint64_t index_image_size(const DeviceIndex& ix) {
    return ix.meta.header_bytes().size() + (ix.meta.file_size - ix.meta.payload_start);
}

void index_image_into(const DeviceIndex& ix, uint8_t* dst) {
    const std::vector<uint8_t> header = ix.meta.header_bytes();
    const uint64_t payload = ix.meta.file_size - ix.meta.payload_start;
    std::memcpy(dst, header.data(), header.size());
    if (ix.streaming()) { // host-resident: the payload is already in file layout
        ix.hs->read_payload(0, dst + header.size(), payload);
        return;
    }
    COBS_CUDA(cudaSetDevice(ix.device));
    uint64_t off = header.size();
    for (const DevBlock& d : ix.blocks) { // pitched 1D chunks, un-pitched on the host
        d2h_unpitch(dst + off, ix.payload + d.base, d.w, d.rb, d.pitch, ix.stream);
        off += d.w * d.rb;
    }
}

std::vector<uint8_t> index_image(const DeviceIndex& ix) {
    std::vector<uint8_t> image(index_image_size(ix));
    index_image_into(ix, image.data());
    return image;
}

void note_image_ms(double ms) {
    g_timing.ms_d2h = ms;
    g_timing.ms_total += ms;
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
    write_image(image.data(), image.size(), path);
}

void write_image(const uint8_t* image, uint64_t size, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc); // storage.cpp:382-396
    if (!out) throw DataError("cannot create index file: " + path);
    out.write(reinterpret_cast<const char*>(image), static_cast<std::streamsize>(size));
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
