// The COBS query hot path on sm_100a: three kernels behind one batch call.
//
//   kernel 1  termize_hash_kernel   windows -> canonical terms -> XXH64 ->
//             exact per-query dedup (lock-free set) -> seed-major hashes, l,
//             skipped, tau.            (reference: query.cpp:127-146,
//             termizer.cpp:103-129, xxhash64.hpp:45-95, bloom.cpp:120-123)
//   kernel 2  gather_kernel         one warp per (query, block, 1024-document
//             slice): stream the k rows of every term (128-byte coalesced
//             loads), AND them, add the 32-bit document masks into bit-sliced
//             counters with a carry-save (Harley-Seal) adder, then threshold
//             and compact hits; optional dense scores.  Small batches split
//             one query's terms over a CTA's 8 warps (counts added
//             bit-sliced); an index streamed from host memory or the file
//             is gathered slab group by slab group.
//                                      (reference: query.cpp:49-119)
//   kernel 3  ordering              CUB radix sorts on (query, score desc,
//             name rank asc) (reference: query.cpp:156-162).
// A host batch too large for the free HBM runs as sub-batches (results
// concatenated, one dense score width).
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdlib>
#include <cub/cub.cuh>
#include <type_traits>

#include "../../include/cobs_gpu.h"
#include "gather_common.cuh"
#include "index.hpp"

namespace cobsg {

namespace {

#ifndef COBS_GATHER_MINB
#define COBS_GATHER_MINB 3
#endif
constexpr int kTermizeThreads = 256;
constexpr uint32_t kSmemSlots = 16384; // <= 128 KB of shared set per CTA
constexpr uint64_t kNoGtab = ~0ull;

inline uint64_t next_pow2(uint64_t x) {
    uint64_t p = 2;
    while (p < x) p <<= 1;
    return p;
}

// ---- kernel 1 -----------------------------------------------------------

struct TermizeArgs {
    const uint8_t* pats;
    const uint64_t* off;
    const uint64_t* win_base; // n+1 prefix of windows
    const uint64_t* tab_off;  // per query: slot offset into gtab, or kNoGtab
    unsigned long long* gtab;
    uint64_t n;
    uint32_t q, k;
    int canonical;
    double K;
    uint32_t smem_slots; // shared-memory set capacity (tile arrays follow it)
    uint32_t tag_mask;   // all ones (tests may narrow it to force tag collisions)
    uint64_t* hashes; // [win_total * k]
    uint32_t* ell;
    uint64_t* skipped;
    uint32_t* tau;
};

// Set size for W windows: load factor <= 2/3 (same formula on the host).
__host__ __device__ __forceinline__ uint64_t set_slots(uint64_t W) {
    uint64_t x = W + W / 2 + 1, p = 2;
    while (p < x) p <<= 1;
    return p;
}

// Tile of the pattern in shared memory with per-position codes of runs of
// 1, 2, 4, 8, 16 bases and their all-ACGT flags, built by doubling
// (c2L[j] = cL[j] << 2L | cL[j+L]); a window's code is then 5 lookups.
constexpr int kTile = 2048;           // windows per tile
constexpr int kTileP = kTile + 32;    // positions per tile
constexpr size_t kTileBytes = (size_t)kTileP * (4 + 2 + 1 + 1 + 1) + (size_t)kTileP * 5;

struct TileView {
    uint32_t* c16;
    uint16_t* c8;
    uint8_t *c4, *c2, *c1;
    uint8_t* ok[5]; // ok[b][j]: bases [j, j + 2^b) are all A/C/G/T
    __device__ explicit TileView(uint8_t* base) {
        c16 = reinterpret_cast<uint32_t*>(base);
        c8 = reinterpret_cast<uint16_t*>(c16 + kTileP);
        c4 = reinterpret_cast<uint8_t*>(c8 + kTileP);
        c2 = c4 + kTileP;
        c1 = c2 + kTileP;
        for (int b = 0; b < 5; ++b) ok[b] = c1 + kTileP * (b + 1);
    }
    // code and validity of the q-base window at tile position j (q <= 32)
    __device__ __forceinline__ uint64_t window(uint32_t j, uint32_t q, bool& valid) const {
        uint64_t code = 0;
        uint32_t off = j, good = 1;
        if (q & 32) {
            code = (static_cast<uint64_t>(c16[off]) << 32) | c16[off + 16];
            good = ok[4][off] & ok[4][off + 16];
            off += 32;
        }
        if (q & 16) { code = (code << 32) | c16[off]; good &= ok[4][off]; off += 16; }
        if (q & 8) { code = (code << 16) | c8[off]; good &= ok[3][off]; off += 8; }
        if (q & 4) { code = (code << 8) | c4[off]; good &= ok[2][off]; off += 4; }
        if (q & 2) { code = (code << 4) | c2[off]; good &= ok[1][off]; off += 2; }
        if (q & 1) { code = (code << 2) | c1[off]; good &= ok[0][off]; }
        valid = good != 0;
        return code;
    }
};

// Reverse complement of a q-base code: complement every base (xor 3), then
// reverse the order of the 2-bit groups.
__device__ __forceinline__ uint64_t revcomp_code(uint64_t code, uint32_t q) {
    uint64_t x = __brevll(~code);
    x = ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
    return x >> (64 - 2 * q);
}

// One CTA per query.  The pattern is staged tile by tile into shared memory;
// every thread then takes 8 consecutive windows: all-ACGT windows (q <= 32)
// get their code from the tile (canonical = min(code, revcomp)), XXH64 from
// the code and an exact code-keyed insert; other windows take the byte path.
// The distinct terms are compacted in window order.  QC: 31 or 0.
template <int QC, int THREADS>
__global__ void __launch_bounds__(THREADS) termize_hash_kernel(TermizeArgs a) {
    extern __shared__ __align__(16) unsigned long long s_dyn[];
    using Reduce = cub::BlockReduce<uint64_t, THREADS>;
    __shared__ typename Reduce::TempStorage tmp_reduce;
    __shared__ uint32_t s_count; // distinct terms of the current query
    const uint32_t q = QC ? QC : a.q, k = a.k;
    // DNA windows carried as 2-bit codes.  Not for q = 32 without
    // canonicalisation: there a code spans all 64 bits, so the poly-T code
    // 2^64-1 would make the key code+1 wrap to the empty marker, and codes
    // with bit 63 set would share the key space of the byte-path keys --
    // those patterns take the byte path (exact byte compares) instead.
    // (Canonical codes at q = 32 are never all ones: revcomp(T^32) = A^32.)
    const bool code_path = codes_exact(q, a.canonical != 0);
    unsigned long long* s_tab = s_dyn;
    TileView T(reinterpret_cast<uint8_t*>(s_dyn + a.smem_slots));
    for (uint64_t qi = blockIdx.x; qi < a.n; qi += gridDim.x) {
        const uint64_t W = a.win_base[qi + 1] - a.win_base[qi];
        const uint64_t L = a.off[qi + 1] - a.off[qi];
        const uint8_t* pat = a.pats + a.off[qi];
        const uint64_t S = set_slots(W);
        unsigned long long* tab = a.tab_off[qi] == kNoGtab ? s_tab : a.gtab + a.tab_off[qi];
        for (uint64_t s = threadIdx.x; s < S; s += blockDim.x) tab[s] = 0ull;
        uint64_t* out = a.hashes + a.win_base[qi] * k;
        uint64_t skipped = 0;
        if (threadIdx.x == 0) s_count = 0;
        for (uint64_t tb = 0; tb < W; tb += kTile) {
            __syncthreads(); // table cleared / previous tile consumed
            const uint32_t nwin = static_cast<uint32_t>(W - tb < (uint64_t)kTile ? W - tb : (uint64_t)kTile);
            if (code_path) {
                // positions needed: nwin + q - 1 (rounded so every level is defined)
                const uint32_t np = nwin + 32 < (uint32_t)kTileP ? nwin + 32 : (uint32_t)kTileP;
                for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
                    const uint32_t c = tb + i < L ? __ldg(pat + tb + i) : 'A';
                    T.c1[i] = static_cast<uint8_t>(base_code(c));
                    T.ok[0][i] = static_cast<uint8_t>(acgt_bit(c));
                }
                __syncthreads();
                for (uint32_t i = threadIdx.x; i + 1 < np; i += blockDim.x) {
                    T.c2[i] = static_cast<uint8_t>((T.c1[i] << 2) | T.c1[i + 1]);
                    T.ok[1][i] = T.ok[0][i] & T.ok[0][i + 1];
                }
                __syncthreads();
                for (uint32_t i = threadIdx.x; i + 3 < np; i += blockDim.x) {
                    T.c4[i] = static_cast<uint8_t>((T.c2[i] << 4) | T.c2[i + 2]);
                    T.ok[2][i] = T.ok[1][i] & T.ok[1][i + 2];
                }
                __syncthreads();
                for (uint32_t i = threadIdx.x; i + 7 < np; i += blockDim.x) {
                    T.c8[i] = static_cast<uint16_t>((T.c4[i] << 8) | T.c4[i + 4]);
                    T.ok[3][i] = T.ok[2][i] & T.ok[2][i + 4];
                }
                __syncthreads();
                for (uint32_t i = threadIdx.x; i + 15 < np; i += blockDim.x) {
                    T.c16[i] = (static_cast<uint32_t>(T.c8[i]) << 16) | T.c8[i + 8];
                    T.ok[4][i] = T.ok[3][i] & T.ok[3][i + 8];
                }
                __syncthreads();
            }
            // window r*threads + tid: every thread busy even for short patterns;
            // winners are appended with one shared atomic per warp and round
            // (term order inside the list is irrelevant: scores are sums)
            for (uint32_t r0 = 0; r0 < nwin; r0 += THREADS) {
                const uint32_t jl = r0 + threadIdx.x;
                const bool active = jl < nwin;
                const uint64_t j = tb + jl;
                const uint8_t* w = pat + j;
                bool won = false, bytep = false, rc = false;
                uint64_t h = 0, code = 0;
                if (active) {
                    bool dna = false;
                    if (code_path) code = T.window(jl, q, dna);
                    if (dna) {
                        if (a.canonical) { // termizer.cpp:117-119: min(gram, revcomp)
                            const uint64_t rcc = revcomp_code(code, q);
                            code = rcc < code ? rcc : code;
                        }
                        h = xxh64_code<QC>(code, q, 0);
                        won = set_insert_code(tab, S - 1, h, code);
                    } else if (a.canonical) {
                        // non-ACGT window: skipped (termizer.cpp:113-116); for q > 32
                        // the ACGT windows take the canonical byte path
                        if (code_path || !window_acgt(w, q)) {
                            ++skipped;
                        } else {
                            rc = choose_rc(w, q);
                            h = xxh64_term(w, q, rc, 0);
                            bytep = true;
                            won = set_insert(tab, S - 1, h, static_cast<uint32_t>(j), pat, q, true, rc,
                                             a.tag_mask);
                        }
                    } else { // raw bytes (any alphabet): termizer.cpp:120-122
                        h = xxh64_term(w, q, false, 0);
                        bytep = true;
                        won = code_path
                                  ? set_insert_tagged(tab, S - 1, h, static_cast<uint32_t>(j), pat, q, a.tag_mask)
                                  : set_insert(tab, S - 1, h, static_cast<uint32_t>(j), pat, q, false, false,
                                               a.tag_mask);
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, won);
                if (m) {
                    const uint32_t lane = threadIdx.x & 31u;
                    uint32_t base = 0;
                    if (lane == 0) base = atomicAdd(&s_count, static_cast<uint32_t>(__popc(m)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (won) { // seed-major per term: query.cpp:141-144
                        uint64_t* dst = out + static_cast<uint64_t>(base + __popc(m & ((1u << lane) - 1u))) * k;
                        dst[0] = h;
                        for (uint32_t s = 1; s < k; ++s)
                            dst[s] = bytep ? xxh64_term(w, q, rc, s) : xxh64_code<QC>(code, q, s);
                    }
                }
            }
        }
        __syncthreads();
        const uint64_t ell = s_count;
        uint64_t skip_total = Reduce(tmp_reduce).Sum(skipped);
        if (threadIdx.x == 0) {
            a.ell[qi] = static_cast<uint32_t>(ell);
            a.skipped[qi] = skip_total;
            // bloom.cpp:120-123 with the host's separate roundings (no FMA)
            double t = ceil(__dsub_rn(__dmul_rn(a.K, (double)ell), 1e-9));
            uint64_t tau = t < 1.0 ? 1 : static_cast<uint64_t>(t);
            a.tau[qi] = ell ? static_cast<uint32_t>(tau) : 0u;
        }
        __syncthreads();
    }
}

// ---- kernel 2 -----------------------------------------------------------

struct GatherArgs {
    const uint8_t* payload;
    const DevBlock* blocks;
    const uint32_t* ct; // (block, slice) pairs
    uint32_t nct;
    const uint64_t* hashes;
    const uint64_t* win_base;
    const uint32_t* ell;
    const uint32_t* tau;
    uint64_t n;
    uint32_t k;
    uint32_t qt; // queries per tile (multiple of 8)
    uint32_t split; // 1: one warp per (query, column task); 8: the CTA's 8 warps split one query's terms
    uint64_t D;
    void* scores; // dense [n][D] (uint16 or uint32) or null
    int want_hits;
    int prune;    // threshold pruning (hits only, no dense scores)
    uint32_t* hit_count; // per query
    unsigned long long* hit_total;
    uint64_t hit_cap;
    uint32_t* hit_q;
    uint32_t* hit_doc;
    uint32_t* hit_score;
};

// One warp = one (query, column task): 32 lanes x 4 bytes = the 128-byte,
// 1024-document slice of every addressed row.  Per chunk of CH terms the
// lanes compute the CH rows (exact modulo, one term per lane) into a
// warp-private shared-memory list, then every lane issues CH independent
// 4-byte loads (each warp load = one coalesced 128-byte line), reading the
// row list with 128-bit broadcast LDS; the next chunk's hashes are
// prefetched while this chunk's rows are in flight.
//
// NT = NP + 4 bit planes in total (the batch's max window count is < 2^NT).
// KT = 1: k = 1 and every width < 2^32 (32-bit rows); KT = 0: runtime k,
// 64-bit rows.  EF: L2 evict-first row loads (index far larger than L2).
template <int NP, int KT, bool EF>
__global__ void __launch_bounds__(256, COBS_GATHER_MINB) gather_kernel(GatherArgs a) {
    constexpr int NT = NP + 4;
    constexpr int CH = (NT <= 16 && KT == 1) ? 32 : 16; // terms per chunk
    constexpr int LCH = CH == 32 ? 5 : 4;     // log2(CH): weight of the planes P
    constexpr int NPP = NT - LCH;             // planes above the carry-save levels
    constexpr int KS = KT ? KT : 1;           // row lists per chunk held in smem
    using RowT = typename std::conditional<KT != 0, uint32_t, uint64_t>::type;
    __shared__ __align__(16) RowT s_rows[8][KS * CH];

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // split = 8 (small batches): the CTA's warps take every 8th chunk of one
    // query's terms and their counts are added at the end (more warps in
    // flight per query when there are too few queries to fill the GPU)
    const uint32_t S = a.split;
    const uint32_t qpc = S == 1 ? 8u : 1u; // queries per CTA
    const uint32_t groups = (a.qt + qpc - 1) / qpc;
    const uint32_t per_tile = groups * a.nct;
    const uint32_t bid = blockIdx.x;
    const uint32_t tile = bid / per_tile;
    const uint32_t r = bid - tile * per_tile;
    const uint32_t cti = r / groups;
    const uint32_t qg = r - cti * groups;
    const uint32_t qin = S == 1 ? qg * 8 + warp : qg;
    const uint32_t sub = S == 1 ? 0u : warp; // this warp's first chunk
    const uint64_t qi = static_cast<uint64_t>(tile) * a.qt + qin;
    if (qin >= a.qt || qi >= a.n) return;
    const uint32_t ell = a.ell[qi];
    if (ell == 0) return; // DataError query: no scores, no hits
    const uint32_t k = KT ? KT : a.k;
    const DevBlock B = a.blocks[a.ct[2 * cti]];
    const uint32_t slice = a.ct[2 * cti + 1];
    // Lanes past the row's pitch re-read an in-row word: their documents are
    // >= doc_count and are masked out below, so no per-load predicate.
    const uint32_t lane_byte = min(slice * 128u + lane * 4u, B.pitch - 4u);
    const uint8_t* rowbase = a.payload + B.base + lane_byte;
    const uint64_t* hq = a.hashes + a.win_base[qi] * k;
    uint64_t policy = 0;
    if (EF) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    RowT* rows = s_rows[warp];

    uint32_t ones = 0, twos = 0, fours = 0, eights = 0, sixteens = 0;
    uint32_t P[NPP];
#pragma unroll
    for (int p = 0; p < NPP; ++p) P[p] = 0;

    const uint32_t stride = S * CH; // terms from one of this warp's chunks to its next
    uint64_t hnext[KS];
#pragma unroll
    for (int s = 0; s < KS; ++s)
        hnext[s] = (KT != 0 && lane < CH && sub * CH + lane < ell) ? __ldg(hq + (uint64_t)(sub * CH + lane) * KS + s)
                                                                   : 0;
    // One chunk of CH terms; TAIL (the last, partial chunk only) zeroes the
    // masks of the padding terms, so full chunks carry no per-term predicate.
    auto chunk = [&](uint32_t t0, auto tail_c) {
        constexpr bool TAIL = decltype(tail_c)::value;
        const uint32_t tl = t0 + lane;
        uint32_t v[CH];
        if constexpr (KT != 0) { // k = KT, 32-bit rows; the k rows are ANDed (query.cpp:65-73)
            uint64_t h[KS];
#pragma unroll
            for (int s = 0; s < KS; ++s) h[s] = hnext[s];
            if (lane < CH && tl + stride < ell) { // prefetch the next chunk's hashes
#pragma unroll
                for (int s = 0; s < KS; ++s) hnext[s] = __ldg(hq + (uint64_t)(tl + stride) * KS + s);
            }
            if (lane < CH) {
#pragma unroll
                for (int s = 0; s < KS; ++s)
                    rows[s * CH + lane] =
                        (!TAIL || tl < ell) ? static_cast<RowT>(fastmod(h[s], B.w, B.magic)) : 0;
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < CH; u += 4) {
                uint4 r4 = *reinterpret_cast<const uint4*>(rows + u);
                v[u + 0] = ld_row<EF>(row_addr(rowbase, r4.x, B.pitch), policy);
                v[u + 1] = ld_row<EF>(row_addr(rowbase, r4.y, B.pitch), policy);
                v[u + 2] = ld_row<EF>(row_addr(rowbase, r4.z, B.pitch), policy);
                v[u + 3] = ld_row<EF>(row_addr(rowbase, r4.w, B.pitch), policy);
#pragma unroll
                for (int s = 1; s < KS; ++s) {
                    r4 = *reinterpret_cast<const uint4*>(rows + s * CH + u);
                    v[u + 0] &= ld_row<EF>(row_addr(rowbase, r4.x, B.pitch), policy);
                    v[u + 1] &= ld_row<EF>(row_addr(rowbase, r4.y, B.pitch), policy);
                    v[u + 2] &= ld_row<EF>(row_addr(rowbase, r4.z, B.pitch), policy);
                    v[u + 3] &= ld_row<EF>(row_addr(rowbase, r4.w, B.pitch), policy);
                }
            }
            __syncwarp();
        } else {
            for (uint32_t s = 0; s < k; ++s) { // AND the k rows: query.cpp:65-73
                if (lane < CH)
                    rows[lane] = (!TAIL || tl < ell)
                                     ? static_cast<RowT>(fastmod(__ldg(hq + (uint64_t)tl * k + s), B.w, B.magic))
                                     : 0;
                __syncwarp();
#pragma unroll
                for (int u = 0; u < CH; u += 2) {
                    const ulonglong2 r2 = *reinterpret_cast<const ulonglong2*>(rows + u);
                    uint32_t x0 = ld_row<EF>(rowbase + r2.x * B.pitch, policy);
                    uint32_t x1 = ld_row<EF>(rowbase + r2.y * B.pitch, policy);
                    v[u] = s ? (v[u] & x0) : x0;
                    v[u + 1] = s ? (v[u + 1] & x1) : x1;
                }
                __syncwarp();
            }
        }
        if constexpr (TAIL) {
#pragma unroll
            for (int u = 0; u < CH; ++u)
                if (t0 + u >= ell) v[u] = 0;
        }
        uint32_t carry = csa16(v, ones, twos, fours, eights);
        if constexpr (CH == 32) {
            uint32_t c2 = csa16(v + 16, ones, twos, fours, eights);
            csa(carry, sixteens, sixteens, carry, c2); // carry now has weight 32
        }
#pragma unroll
        for (int p = 0; p < NPP; ++p) { // ripple the weight-CH carry
            uint32_t c = P[p] & carry;
            P[p] ^= carry;
            carry = c;
        }
    };
    // Documents d < dc only: padding columns never count (query.cpp:84-86).
    const uint32_t d0 = slice * 1024u + lane * 32u; // this lane's first document
    uint32_t valid = 0;
    if (d0 < B.dc) valid = (B.dc - d0 >= 32u) ? 0xffffffffu : ((1u << (B.dc - d0)) - 1u);
    const uint64_t gdoc0 = static_cast<uint64_t>(B.doc_base) + d0;
    const uint32_t tau = a.tau[qi];
    // Flush the carry-save state into plain bit planes F (weight 2^p).
    uint32_t F[NT];
    auto flush = [&]() {
#pragma unroll
        for (int p = 0; p < LCH; ++p) F[p] = 0;
#pragma unroll
        for (int p = 0; p < NPP; ++p) F[p + LCH] = P[p];
        if constexpr (CH == 32) add_at<NT>(F, 4, sixteens);
        add_at<NT>(F, 3, eights);
        add_at<NT>(F, 2, fours);
        add_at<NT>(F, 1, twos);
        add_at<NT>(F, 0, ones);
    };

    uint32_t t0 = sub * CH;
    for (; t0 + CH <= ell; t0 += stride) {
        chunk(t0, std::false_type{});
        // Optional threshold pruning (hits only): every 2 chunks, if no document
        // of this slice can still reach tau with all remaining terms, its hit
        // list is empty whatever those rows hold -- stop reading them.
        if (a.prune && S == 1 && ((t0 / CH) & 1u) == 1u) {
            const uint32_t rem = ell - (t0 + CH);
            if (tau > rem) {
                flush();
                if (!__any_sync(0xffffffffu, ge_mask<NT>(F, tau - rem) & valid)) return;
            }
        }
    }
    if (t0 < ell) chunk(t0, std::true_type{}); // the partial last chunk, if it is this warp's
    flush();
    if (S > 1) { // add the warps' counts: bit-sliced ripple-carry adds in warp 0
        extern __shared__ uint32_t s_planes[]; // [8][NT][32]
#pragma unroll
        for (int p = 0; p < NT; ++p) s_planes[(warp * NT + p) * 32 + lane] = F[p];
        __syncthreads();
        if (warp != 0) return;
        for (uint32_t w = 1; w < 8; ++w) {
            uint32_t c = 0;
#pragma unroll
            for (int p = 0; p < NT; ++p) {
                const uint32_t g = s_planes[(w * NT + p) * 32 + lane];
                const uint32_t x = F[p] ^ g;
                const uint32_t sum = x ^ c;
                c = (F[p] & g) | (x & c);
                F[p] = sum;
            }
        }
    }

    const EmitArgs e{a.scores, a.D, a.want_hits, a.hit_count, a.hit_total, a.hit_cap, a.hit_q, a.hit_doc, a.hit_score};
    emit_slice<NT>(e, qi, gdoc0, valid, tau, F, lane);
}

// ---- kernel 3 helpers ---------------------------------------------------

__global__ void make_keys_kernel(uint64_t m, const uint32_t* score, const uint32_t* doc,
                                 const uint32_t* rank, int rbits, uint32_t smask, uint64_t* key,
                                 uint32_t* perm) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    // (score desc, name asc) as one ascending key
    key[i] = (static_cast<uint64_t>(~score[i] & smask) << rbits) | rank[doc[i]];
    perm[i] = static_cast<uint32_t>(i);
}

// One ascending key for the whole batch order (query, score desc, name asc):
// query id above the (score, name rank) key of make_keys_kernel.
__global__ void make_qkeys_kernel(uint64_t m, const uint32_t* q, const uint32_t* score, const uint32_t* doc,
                                  const uint32_t* rank, int rbits, int sbits, uint32_t smask, uint64_t* key,
                                  uint32_t* perm) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    key[i] = (static_cast<uint64_t>(q[i]) << (sbits + rbits)) |
             (static_cast<uint64_t>(~score[i] & smask) << rbits) | rank[doc[i]];
    perm[i] = static_cast<uint32_t>(i);
}

// top_t on the device: hit i of the sorted batch (query q = its segment, rank
// j inside it) is kept iff j < top_t, at out_start[q] + j (query.cpp:161-162);
// seg_start / out_start are the exclusive scans of the per-query counts and
// of min(count, top_t).
__global__ void truncate_kernel(uint64_t m, uint64_t n, const uint64_t* seg_start, const uint64_t* out_start,
                                uint64_t top_t, const uint32_t* perm, const uint32_t* doc, const uint32_t* score,
                                uint32_t* out_doc, uint32_t* out_score) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint64_t lo = 0, hi = n; // seg_start[lo] <= i < seg_start[hi]
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (seg_start[mid] <= i)
            lo = mid;
        else
            hi = mid;
    }
    const uint64_t j = i - seg_start[lo];
    if (j >= top_t) return;
    out_doc[out_start[lo] + j] = doc[perm[i]];
    out_score[out_start[lo] + j] = score[perm[i]];
}

__global__ void gather_u32_kernel(uint64_t m, const uint32_t* perm, const uint32_t* src,
                                  uint32_t* dst) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < m) dst[i] = src[perm[i]];
}

int bits_for(uint64_t v) { // bits to represent values 0..v
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return std::max(b, 1);
}

using GatherFn = void (*)(GatherArgs);

template <int NP, int KT>
GatherFn pick_ef(bool ef) {
    return ef ? gather_kernel<NP, KT, true> : gather_kernel<NP, KT, false>;
}

// kt: 1..3 with every width < 2^32 (32-bit rows), else 0 (runtime k, 64-bit rows)
template <int NP>
GatherFn pick_k(int kt, bool ef) {
    switch (kt) {
    case 1: return pick_ef<NP, 1>(ef);
    case 2: return pick_ef<NP, 2>(ef);
    case 3: return pick_ef<NP, 3>(ef);
    default: return pick_ef<NP, 0>(ef);
    }
}

GatherFn pick_gather(int nt_needed, int kt, bool ef) {
    if (nt_needed <= 8) return pick_k<4>(kt, ef);
    if (nt_needed <= 12) return pick_k<8>(kt, ef);
    if (nt_needed <= 16) return pick_k<12>(kt, ef);
    return pick_k<28>(kt, ef);
}

} // namespace

namespace {

// More hits than one ordering pass may hold: kernel 3's sorts take an int
// item count, and every hit needs ~12 bytes in the gather's pool plus ~40 in
// the sort buffers.  query_batch re-runs such a batch as two halves.
struct HitsOverflow {
    uint64_t hits;
};
uint64_t hit_limit() {
    if (const char* e = std::getenv("COBS_HIT_LIMIT")) return std::strtoull(e, nullptr, 10); // tests
    size_t free_b = 0, total_b = 0;
    COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return std::min<uint64_t>(0x7fffffffull, free_b / 64);
}

// One batch through kernels 1-3; the caller holds ix.mu.  min_nt: at least
// this many count bits (dense score width agreed over sub-batches).
void query_batch_one(DeviceIndex& ix, const uint8_t* patterns, const uint64_t* offsets, uint64_t n,
                     double K, uint64_t top_t, uint32_t flags, int min_nt, QueryResults& R) {
    QueryWorkspace& ws = ix.ws;
    cudaStream_t st = ix.work_stream();
    const Params& P = ix.meta.params;
    const uint32_t q = P.q, k = P.k;
    const uint64_t D = ix.meta.total_docs();
    const bool dev_in = flags & COBS_Q_DEVICE_INPUT;
    R = QueryResults();
    R.n = n;
    if (n == 0) return;

    // Host-side window accounting (needs the offsets on the host).
    std::vector<uint64_t> h_off(n + 1);
    if (dev_in) {
        COBS_CUDA(cudaMemcpyAsync(h_off.data(), offsets, sizeof(uint64_t) * (n + 1),
                                  cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaStreamSynchronize(st));
    }
    else
        std::copy(offsets, offsets + n + 1, h_off.begin());
    std::vector<uint64_t> win_base(n + 1), tab_off(n);
    uint64_t wmax = 0, gslots = 0;
    win_base[0] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t len = h_off[i + 1] - h_off[i];
        uint64_t W = len >= q ? len - q + 1 : 0; // termizer.cpp:109-110
        if (W >= 0xffffffffull) throw UsageError("query: pattern longer than 2^32-2 grams");
        win_base[i + 1] = win_base[i] + W;
        wmax = std::max(wmax, W);
        uint64_t S = set_slots(W);
        if (S <= kSmemSlots) {
            tab_off[i] = kNoGtab;
        } else {
            tab_off[i] = gslots;
            gslots += S;
        }
    }
    const uint64_t wtot = win_base[n];
    const uint64_t pat_bytes = h_off[n] - h_off[0];

    Event ev_begin, ev_end;
    COBS_CUDA(cudaEventRecord(ev_begin, st));

    // Buffers
    const uint8_t* d_pats;
    const uint64_t* d_off;
    if (dev_in) {
        d_pats = patterns;
        d_off = offsets;
    } else {
        ws.pats.reserve(std::max<uint64_t>(h_off[n], 1));
        ws.offs.reserve(sizeof(uint64_t) * (n + 1));
        h2d_staged(ws.pats.ptr, patterns, h_off[n], st); // pinned: one async copy; pageable: staged
        COBS_CUDA(cudaMemcpyAsync(ws.offs.ptr, offsets, sizeof(uint64_t) * (n + 1),
                                  cudaMemcpyHostToDevice, st));
        d_pats = ws.pats.as<uint8_t>();
        d_off = ws.offs.as<uint64_t>();
    }
    (void)pat_bytes;
    ws.win_base.reserve(sizeof(uint64_t) * (n + 1));
    ws.tab_off.reserve(sizeof(uint64_t) * n);
    ws.gtab.reserve(std::max<uint64_t>(gslots, 1) * 8);
    ws.hashes.reserve(std::max<uint64_t>(wtot * k, 1) * 8);
    ws.ell.reserve(4 * n);
    ws.skipped.reserve(8 * n);
    ws.tau.reserve(4 * n);
    ws.hit_count.reserve(4 * n);
    ws.hit_total.reserve(8);
    COBS_CUDA(cudaMemcpyAsync(ws.win_base.ptr, win_base.data(), 8 * (n + 1), cudaMemcpyHostToDevice, st));
    COBS_CUDA(cudaMemcpyAsync(ws.tab_off.ptr, tab_off.data(), 8 * n, cudaMemcpyHostToDevice, st));

    Event ev[4];
    COBS_CUDA(cudaEventRecord(ev[0], st));

    NvtxPhase phase;
    phase.begin("cobs.query.termize");
    // kernel 1
    TermizeArgs ta{};
    ta.pats = d_pats;
    ta.off = d_off;
    ta.win_base = ws.win_base.as<uint64_t>();
    ta.tab_off = ws.tab_off.as<uint64_t>();
    ta.gtab = ws.gtab.as<unsigned long long>();
    ta.n = n;
    ta.q = q;
    ta.k = k;
    ta.canonical = P.canonical ? 1 : 0;
    ta.K = K;
    ta.tag_mask = debug_tag_mask();
    ta.hashes = ws.hashes.as<uint64_t>();
    ta.ell = ws.ell.as<uint32_t>();
    ta.skipped = ws.skipped.as<uint64_t>();
    ta.tau = ws.tau.as<uint32_t>();
    uint64_t small_S = 2;
    for (uint64_t i = 0; i < n; ++i)
        if (tab_off[i] == kNoGtab) small_S = std::max(small_S, set_slots(win_base[i + 1] - win_base[i]));
    ta.smem_slots = static_cast<uint32_t>(std::min<uint64_t>(small_S, kSmemSlots));
    size_t smem = static_cast<size_t>(ta.smem_slots) * 8 + kTileBytes;
    // long patterns (large shared sets, few CTAs per SM) get 1,024 threads
    const bool wide = smem > (64u << 10);
    auto k1 = q == 31 ? (wide ? termize_hash_kernel<31, 1024> : termize_hash_kernel<31, kTermizeThreads>)
                      : (wide ? termize_hash_kernel<0, 1024> : termize_hash_kernel<0, kTermizeThreads>);
    COBS_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    unsigned grid1 = static_cast<unsigned>(std::min<uint64_t>(n, 1u << 30));
    k1<<<grid1, wide ? 1024 : kTermizeThreads, smem, st>>>(ta);
    COBS_CUDA(cudaGetLastError());
    R.launches += 1;
    COBS_CUDA(cudaEventRecord(ev[1], st));

    phase.begin("cobs.query.gather");
    // kernel 2
    const bool want_scores = flags & COBS_Q_SCORES;
    const bool want_hits = (flags & COBS_Q_HITS) || !(flags & COBS_Q_SCORES);
    int nt_needed = std::max(bits_for(wmax), min_nt);
    R.score_bytes = nt_needed <= 16 ? 2 : 4;
    if (want_scores) {
        ws.scores.reserve(std::max<uint64_t>(n * D * R.score_bytes, 1));
        COBS_CUDA(cudaMemsetAsync(ws.scores.ptr, 0, n * D * R.score_bytes, st));
    }
    if (ws.hit_cap == 0) {
        ws.hit_cap = 1u << 20;
        ws.hit_q.reserve(4 * ws.hit_cap);
        ws.hit_doc.reserve(4 * ws.hit_cap);
        ws.hit_score.reserve(4 * ws.hit_cap);
    }
    GatherArgs ga{};
    ga.payload = ix.payload;
    ga.blocks = ix.d_blocks;
    ga.ct = ix.d_ct;
    ga.nct = static_cast<uint32_t>(ix.ct_block.size());
    ga.hashes = ws.hashes.as<uint64_t>();
    ga.win_base = ws.win_base.as<uint64_t>();
    ga.ell = ws.ell.as<uint32_t>();
    ga.tau = ws.tau.as<uint32_t>();
    ga.n = n;
    ga.k = k;
    uint64_t qt = 8192;
    if (const char* e = std::getenv("COBS_QT")) qt = std::max<uint64_t>(8, std::strtoull(e, nullptr, 10));
    qt = std::min<uint64_t>((qt + 7) / 8 * 8, (n + 7) / 8 * 8);
    ga.qt = static_cast<uint32_t>(qt);
    ga.D = D;
    ga.scores = want_scores ? ws.scores.ptr : nullptr;
    ga.want_hits = want_hits ? 1 : 0;
    ga.prune = ((flags & COBS_Q_PRUNE) && want_hits && !want_scores) ? 1 : 0;
    ga.hit_count = ws.hit_count.as<uint32_t>();
    ga.hit_total = ws.hit_total.as<unsigned long long>();
    bool w32 = true;
    for (const DevBlock& d : ix.blocks) w32 &= d.w <= 0xffffffffull;
    bool ef = ix.evict_first;
    if (const char* e = std::getenv("COBS_EF")) ef = std::atoi(e) != 0; // A/B of the L2 policy
    GatherFn fn = pick_gather(nt_needed, (w32 && k <= 3) ? static_cast<int>(k) : 0, ef);
    // Term split for batches too small to fill the GPU with one warp per
    // (query, column task): fewer than ~4 resident waves of warps.
    ga.split = static_cast<uint64_t>(n) * ga.nct < 4ull * 148 * 24 ? 8 : 1;
    if (const char* e = std::getenv("COBS_SPLIT")) ga.split = std::strtoul(e, nullptr, 10) == 8 ? 8 : 1;
    const uint32_t qpc = ga.split == 1 ? 8 : 1;
    const size_t split_smem = ga.split == 1 ? 0 : 8 * 32 * 32 * 4; // [8 warps][NT <= 32][32 lanes]
    const uint64_t tiles = (n + qt - 1) / qt;
    const uint64_t grid2 = tiles * ((qt + qpc - 1) / qpc) * ga.nct;
    if (grid2 >= (1ull << 31)) throw UsageError("query batch too large for one launch; split it");
    // Host-resident (pinned) index: stream the whole payload through HBM, or
    // -- when the batch addresses far fewer bytes -- let the gather read its
    // rows straight from the mapped host copy over PCIe (zero-copy; random
    // 128-byte reads cost ~kZcCost times a bulk DMA byte).  The bound uses
    // windows for terms (l <= windows).  COBS_ZC=0/1 forces a mode (tests).
    bool zc = false;
    if (ix.streaming() && !ix.hs->file_backed) {
        constexpr uint64_t kZcCost = 4;
        uint64_t stream_bytes = 0;
        for (uint64_t g : ix.hs->group_bytes) stream_bytes += g;
        const uint64_t zc_bytes = wtot * k * ix.sum_row_bytes;
        zc = zc_bytes * kZcCost < stream_bytes;
        if (const char* e = std::getenv("COBS_ZC")) zc = e[0] == '1';
    }
    R.zero_copy = zc;
    const bool resident_gather = !ix.streaming() || zc;
    if (zc) ga.payload = ix.hs->host_dev;
    unsigned long long h_total = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        ga.hit_cap = ws.hit_cap;
        ga.hit_q = ws.hit_q.as<uint32_t>();
        ga.hit_doc = ws.hit_doc.as<uint32_t>();
        ga.hit_score = ws.hit_score.as<uint32_t>();
        COBS_CUDA(cudaMemsetAsync(ws.hit_count.ptr, 0, 4 * n, st));
        COBS_CUDA(cudaMemsetAsync(ws.hit_total.ptr, 0, 8, st));
        if (attempt == 0) COBS_CUDA(cudaEventRecord(ev[1], st));
        if (resident_gather) {
            if (grid2 > 0) {
                fn<<<static_cast<unsigned>(grid2), 256, split_smem, st>>>(ga);
                R.launches += 1;
            }
        } else { // host-resident index: stream slab groups through two staging buffers
            HostStream& hs = *ix.hs;
            for (size_t gi = 0; gi < hs.groups.size(); ++gi) {
                const StreamGroup& G = hs.groups[gi];
                const int buf = static_cast<int>(gi & 1);
                if (hs.file_backed) { // host stages the group from the file while the GPU runs the last one
                    if (hs.hstage_busy[buf]) COBS_CUDA(cudaEventSynchronize(hs.h2d_done[buf]));
                    hs.stage_group(ix.blocks, gi, hs.hstage[buf]);
                }
                COBS_CUDA(cudaStreamWaitEvent(hs.copy, hs.consumed[buf], 0)); // buffer free again
                if (hs.file_backed) {
                    COBS_CUDA(cudaMemcpyAsync(hs.staging[buf], hs.hstage[buf], hs.group_bytes[gi],
                                              cudaMemcpyHostToDevice, hs.copy));
                    COBS_CUDA(cudaEventRecord(hs.h2d_done[buf], hs.copy));
                    hs.hstage_busy[buf] = true;
                    for (uint32_t si = G.slab_lo; si < G.slab_hi; ++si)
                        R.h2d_index_bytes += ix.blocks[hs.slabs[si].block].w * hs.slabs[si].width;
                }
                for (uint32_t si = G.slab_lo; si < (hs.file_backed ? G.slab_lo : G.slab_hi); ++si) {
                    const Slab& sl = hs.slabs[si];
                    const DevBlock& d = ix.blocks[sl.block]; // (the pitched host copy's layout too)
                    if (sl.direct)
                        COBS_CUDA(cudaMemcpyAsync(hs.staging[buf] + sl.base, hs.host + d.base, d.w * d.pitch,
                                                  cudaMemcpyHostToDevice, hs.copy));
                    else
                        COBS_CUDA(cudaMemcpy2DAsync(hs.staging[buf] + sl.base, sl.pitch,
                                                    hs.host + d.base + sl.s0 * 128ull, d.pitch, sl.width, d.w,
                                                    cudaMemcpyHostToDevice, hs.copy));
                    R.h2d_index_bytes += d.w * sl.width;
                }
                COBS_CUDA(cudaEventRecord(hs.copied[buf], hs.copy));
                COBS_CUDA(cudaStreamWaitEvent(st, hs.copied[buf], 0));
                GatherArgs gg = ga;
                gg.payload = hs.staging[buf];
                gg.blocks = hs.d_slab_blocks;
                gg.ct = hs.d_slab_ct + 2ull * G.ct_lo;
                gg.nct = G.ct_hi - G.ct_lo;
                const uint64_t grid_g = tiles * ((qt + qpc - 1) / qpc) * gg.nct;
                if (grid_g >= (1ull << 31)) throw UsageError("query batch too large for one launch; split it");
                if (grid_g > 0) {
                    fn<<<static_cast<unsigned>(grid_g), 256, split_smem, st>>>(gg);
                    R.launches += 1;
                }
                COBS_CUDA(cudaEventRecord(hs.consumed[buf], st));
            }
        }
        COBS_CUDA(cudaGetLastError());
        COBS_CUDA(cudaEventRecord(ev[2], st));
        COBS_CUDA(cudaMemcpyAsync(&h_total, ws.hit_total.ptr, 8, cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        // (the limit queries free HBM -- a driver call -- so only for big hit counts)
        if (want_hits && h_total > (std::getenv("COBS_HIT_LIMIT") ? 0ull : (1ull << 24)) && h_total > hit_limit())
            throw HitsOverflow{h_total};
        if (h_total <= ws.hit_cap) break;
        ws.hit_cap = h_total + h_total / 8;
        ws.hit_q.reserve(4 * ws.hit_cap);
        ws.hit_doc.reserve(4 * ws.hit_cap);
        ws.hit_score.reserve(4 * ws.hit_cap);
    }

    phase.begin("cobs.query.order");
    // kernel 3: order hits by (query, score desc, name asc): one radix sort
    // of (query | ~score | name rank) keys with the hit index as the value,
    // then the kept hits gathered -- all of them, or the first top_t of each
    // query cut on the device so only those cross PCIe
    const uint64_t m = h_total;
    std::vector<uint32_t> cnt(n);
    uint64_t m_out = 0;
    if (want_hits && m > 0) {
        ws.key64.reserve(8 * m);
        ws.key64_alt.reserve(8 * m);
        ws.perm.reserve(4 * m);
        ws.perm_alt.reserve(4 * m);
        ws.out_doc.reserve(4 * m);
        ws.out_score.reserve(4 * m);
        const int rbits = bits_for(D ? D - 1 : 0), sbits = nt_needed, qbits = bits_for(n ? n - 1 : 0);
        const uint32_t smask = sbits >= 32 ? 0xffffffffu : ((1u << sbits) - 1u);
        const unsigned g = static_cast<unsigned>((m + 255) / 256);
        cub::DoubleBuffer<uint64_t> k64(ws.key64.as<uint64_t>(), ws.key64_alt.as<uint64_t>());
        cub::DoubleBuffer<uint32_t> pv(ws.perm.as<uint32_t>(), ws.perm_alt.as<uint32_t>());
        if (qbits + sbits + rbits <= 64) {
            make_qkeys_kernel<<<g, 256, 0, st>>>(m, ws.hit_q.as<uint32_t>(), ws.hit_score.as<uint32_t>(),
                                                 ws.hit_doc.as<uint32_t>(), ix.d_name_rank, rbits, sbits, smask,
                                                 ws.key64.as<uint64_t>(), ws.perm.as<uint32_t>());
            COBS_CUDA(cudaGetLastError());
            size_t tmp = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp, k64, pv, static_cast<int>(m), 0, qbits + sbits + rbits, st);
            ws.cub_tmp.reserve(tmp);
            tmp = ws.cub_tmp.bytes;
            COBS_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.ptr, tmp, k64, pv, static_cast<int>(m), 0,
                                                      qbits + sbits + rbits, st));
            R.launches += 2;
        } else { // (> 64 key bits) score+name sort, then a stable sort by query
            ws.key32.reserve(4 * m);
            ws.key32_alt.reserve(4 * m);
            make_keys_kernel<<<g, 256, 0, st>>>(m, ws.hit_score.as<uint32_t>(), ws.hit_doc.as<uint32_t>(),
                                                ix.d_name_rank, rbits, smask, ws.key64.as<uint64_t>(),
                                                ws.perm.as<uint32_t>());
            COBS_CUDA(cudaGetLastError());
            size_t tmp1 = 0, tmp2 = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp1, k64, pv, static_cast<int>(m), 0, rbits + sbits, st);
            cub::DoubleBuffer<uint32_t> k32(ws.key32.as<uint32_t>(), ws.key32_alt.as<uint32_t>());
            cub::DeviceRadixSort::SortPairs(nullptr, tmp2, k32, pv, static_cast<int>(m), 0, qbits, st);
            ws.cub_tmp.reserve(std::max(tmp1, tmp2));
            tmp1 = ws.cub_tmp.bytes;
            COBS_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.ptr, tmp1, k64, pv, static_cast<int>(m), 0,
                                                      rbits + sbits, st));
            gather_u32_kernel<<<g, 256, 0, st>>>(m, pv.Current(), ws.hit_q.as<uint32_t>(), k32.Current());
            tmp2 = ws.cub_tmp.bytes;
            COBS_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub_tmp.ptr, tmp2, k32, pv, static_cast<int>(m), 0, qbits,
                                                      st));
            R.launches += 4;
        }
        // per-query counts decide whether top_t shrinks what comes back
        COBS_CUDA(cudaMemcpyAsync(cnt.data(), ws.hit_count.ptr, 4 * n, cudaMemcpyDeviceToHost, st));
        COBS_CUDA(cudaStreamSynchronize(st));
        uint64_t kept = 0;
        for (uint64_t i = 0; i < n; ++i) kept += (top_t > 0 && cnt[i] > top_t) ? top_t : cnt[i];
        if (kept < m) { // cut every query to its first top_t on the device
            std::vector<uint64_t> starts(2 * (n + 1), 0);
            for (uint64_t i = 0; i < n; ++i) {
                starts[i + 1] = starts[i] + cnt[i];
                starts[n + 1 + i + 1] = starts[n + 1 + i] + std::min<uint64_t>(cnt[i], top_t);
            }
            ws.starts.reserve(8 * starts.size());
            COBS_CUDA(cudaMemcpyAsync(ws.starts.ptr, starts.data(), 8 * starts.size(), cudaMemcpyHostToDevice, st));
            truncate_kernel<<<g, 256, 0, st>>>(m, n, ws.starts.as<uint64_t>(), ws.starts.as<uint64_t>() + n + 1, top_t,
                                               pv.Current(), ws.hit_doc.as<uint32_t>(), ws.hit_score.as<uint32_t>(),
                                               ws.out_doc.as<uint32_t>(), ws.out_score.as<uint32_t>());
            R.launches += 1;
        } else {
            gather_u32_kernel<<<g, 256, 0, st>>>(m, pv.Current(), ws.hit_doc.as<uint32_t>(),
                                                 ws.out_doc.as<uint32_t>());
            gather_u32_kernel<<<g, 256, 0, st>>>(m, pv.Current(), ws.hit_score.as<uint32_t>(),
                                                 ws.out_score.as<uint32_t>());
            R.launches += 2;
        }
        COBS_CUDA(cudaGetLastError());
        m_out = kept;
    }
    COBS_CUDA(cudaEventRecord(ev[3], st));

    // D2H: per-query metadata always (small); hits and scores unless the
    // caller keeps results on the device.
    const bool keep = flags & COBS_Q_KEEP_DEVICE;
    R.ell.resize(n);
    R.tau.resize(n);
    R.skipped.resize(n);
    COBS_CUDA(cudaMemcpyAsync(R.ell.data(), ws.ell.ptr, 4 * n, cudaMemcpyDeviceToHost, st));
    COBS_CUDA(cudaMemcpyAsync(R.tau.data(), ws.tau.ptr, 4 * n, cudaMemcpyDeviceToHost, st));
    COBS_CUDA(cudaMemcpyAsync(R.skipped.data(), ws.skipped.ptr, 8 * n, cudaMemcpyDeviceToHost, st));
    if (!(want_hits && m > 0)) COBS_CUDA(cudaMemcpyAsync(cnt.data(), ws.hit_count.ptr, 4 * n, cudaMemcpyDeviceToHost, st));
    // large results: pinned staging + host threads (d2h_staged)
    if (!keep && want_hits && m_out > 0) {
        R.doc.resize(m_out); // (default-initialised: no zero fill before the copy)
        R.score.resize(m_out);
        d2h_staged(R.doc.data(), ws.out_doc.ptr, 4 * m_out, st);
        d2h_staged(R.score.data(), ws.out_score.ptr, 4 * m_out, st);
    }
    if (!keep && want_scores) {
        R.scores.resize(n * D * R.score_bytes);
        d2h_staged(R.scores.data(), ws.scores.ptr, R.scores.size(), st);
    }
    COBS_CUDA(cudaEventRecord(ev_end, st));
    COBS_CUDA(cudaStreamSynchronize(st));
    R.status.assign(n, 0);
    R.message.assign(n, std::string());
    R.hit_off.resize(n);
    R.hit_n.resize(n);
    uint64_t o = 0;
    const bool cut = m_out < m; // the device already kept only the first top_t per query
    for (uint64_t i = 0; i < n; ++i) {
        R.hit_off[i] = o;
        uint64_t c = want_hits ? cnt[i] : 0;
        R.hit_n[i] = keep ? 0 : ((top_t > 0 && c > top_t) ? top_t : c); // query.cpp:161-162
        o += cut ? R.hit_n[i] : c;
        if (R.ell[i] == 0) { // query.cpp:133-138
            R.status[i] = COBS_EDATA;
            R.message[i] = R.skipped[i] > 0
                               ? "query: all " + std::to_string(R.skipped[i]) +
                                     " pattern grams were skipped by canonicalization"
                               : "query: pattern shorter than q = " + std::to_string(q);
        }
        R.row_bytes += static_cast<uint64_t>(k) * R.ell[i] * ix.sum_row_bytes;
    }
    if (zc) R.h2d_index_bytes = R.row_bytes; // the addressed rows, read over PCIe
    float t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t12, ev[1], ev[2]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    R.ms_termize = t01;
    R.ms_gather = t12;
    R.ms_order = t23;
    float ttot = 0;
    cudaEventElapsedTime(&ttot, ev_begin, ev_end);
    R.ms_total = ttot;
}

void append_results(QueryResults& R, QueryResults&& S) {
    const uint64_t base = R.doc.size();
    R.n += S.n;
    R.ell.insert(R.ell.end(), S.ell.begin(), S.ell.end());
    R.tau.insert(R.tau.end(), S.tau.begin(), S.tau.end());
    R.skipped.insert(R.skipped.end(), S.skipped.begin(), S.skipped.end());
    R.status.insert(R.status.end(), S.status.begin(), S.status.end());
    for (auto& m : S.message) R.message.push_back(std::move(m));
    for (uint64_t o : S.hit_off) R.hit_off.push_back(o + base);
    R.hit_n.insert(R.hit_n.end(), S.hit_n.begin(), S.hit_n.end());
    R.doc.insert(R.doc.end(), S.doc.begin(), S.doc.end());
    R.score.insert(R.score.end(), S.score.begin(), S.score.end());
    R.scores.insert(R.scores.end(), S.scores.begin(), S.scores.end());
    R.score_bytes = S.score_bytes;
    R.ms_termize += S.ms_termize;
    R.ms_gather += S.ms_gather;
    R.ms_order += S.ms_order;
    R.ms_total += S.ms_total;
    R.launches += S.launches;
    R.h2d_index_bytes += S.h2d_index_bytes;
    R.zero_copy = R.zero_copy || S.zero_copy;
    R.row_bytes += S.row_bytes;
}

} // namespace

// A host batch whose per-window buffers (hashes, sets) and dense scores would
// not fit in half of the free HBM is run as consecutive sub-batches and the
// results concatenated (same answers, same dense score width).
void query_batch(DeviceIndex& ix, const uint8_t* patterns, const uint64_t* offsets, uint64_t n,
                 double K, uint64_t top_t, uint32_t flags, QueryResults& R) {
    if (!(K > 0.0 && K <= 1.0)) throw UsageError("query: K must be in (0,1]"); // query.cpp:125
    std::lock_guard<std::mutex> lock(ix.mu);
    COBS_CUDA(cudaSetDevice(ix.device));
    if ((flags & (COBS_Q_DEVICE_INPUT | COBS_Q_KEEP_DEVICE)) || n <= 1) {
        try {
            query_batch_one(ix, patterns, offsets, n, K, top_t, flags, 1, R);
        } catch (const HitsOverflow& h) {
            throw UsageError("query: " + std::to_string(h.hits) +
                             " hits exceed one ordering pass; submit the batch in parts");
        }
        return;
    }
    const uint32_t q = ix.meta.params.q, k = ix.meta.params.k;
    const uint64_t D = ix.meta.total_docs();
    const bool want_scores = flags & COBS_Q_SCORES;
    std::vector<uint64_t> cost(n); // device bytes per query, roughly
    uint64_t total = 0, wmax = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t len = offsets[i + 1] - offsets[i];
        const uint64_t W = len >= q ? len - q + 1 : 0;
        wmax = std::max(wmax, W);
        cost[i] = len + W * (8ull * k + 24) + (want_scores ? 4 * D : 0) + 64;
        total += cost[i];
    }
    // free HBM (a driver call: ~1.7 ms with a 100 GB index resident) is
    // re-read only when the batch could come near half of the last reading
    size_t free_b = ix.free_hbm_seen, total_b = 0;
    if (free_b == 0 || 4 * total > free_b) {
        COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
        ix.free_hbm_seen = free_b;
    }
    uint64_t budget = std::max<uint64_t>(free_b / 2, 64ull << 20);
    if (const char* e = std::getenv("COBS_QUERY_BUDGET")) budget = std::strtoull(e, nullptr, 10);
    const int nt = bits_for(wmax);
    R = QueryResults();
    std::vector<uint64_t> sub_off;
    // queries [a, b) as one sub-batch; halved while their hits overflow
    std::function<void(uint64_t, uint64_t)> run = [&](uint64_t a, uint64_t b) {
        sub_off.assign(offsets + a, offsets + b + 1);
        const uint64_t base = sub_off[0];
        for (uint64_t& o : sub_off) o -= base;
        QueryResults S;
        try {
            query_batch_one(ix, patterns + base, sub_off.data(), b - a, K, top_t, flags, nt, S);
        } catch (const HitsOverflow& h) {
            if (b - a == 1)
                throw UsageError("query: " + std::to_string(h.hits) + " hits of one pattern exceed one ordering pass");
            const uint64_t mid = a + (b - a) / 2;
            run(a, mid);
            run(mid, b);
            return;
        }
        append_results(R, std::move(S));
    };
    if (total <= budget) {
        run(0, n);
        return;
    }
    for (uint64_t a = 0; a < n;) {
        uint64_t b = a, c = 0;
        while (b < n && (b == a || c + cost[b] <= budget)) c += cost[b++];
        run(a, b);
        a = b;
    }
}

} // namespace cobsg
