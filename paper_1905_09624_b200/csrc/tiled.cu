// L2-tiled row gather: kernel 2 for batches whose terms address every row of
// a block many times over (config 5: 100,000 queries x 970 terms per block
// against ~7.9 M rows, each row read ~12 times).
//
// The reference's score_range (query.cpp:49-89) walks one query's terms and
// reads each term's row of the block.  gather_kernel (query.cu) does the same
// with one warp per (query, slice); its reads are uniformly random 128-byte
// lines over the whole index, so they run at the HBM random-line rate
// (~5.7 TB/s) and every repeat of a row is another HBM read.  Here the work
// of a *wave* of queries is reordered instead:
//
//   bucket_kernel  one warp per query of the wave: for every block, the
//                  rows h % w_b of the query's terms (exact fastmod), grouped
//                  by row range (2^shift rows, <= 64 ranges per block) with a
//                  per-lane counting sort, written as one list per
//                  (block, query).
//   tile_kernel    one persistent CTA per SM; the CTA owns `qs` queries of
//                  the wave and keeps their bit-sliced counters (carry-save
//                  state, NT words x 32 lanes) in shared memory.  For every
//                  column task (block, 1,024-document slice) the grid walks
//                  the block's row ranges in lockstep (a phase counter per
//                  range; a warp may run at most `lag` phases ahead of the
//                  slowest), and each warp adds, for each of its queries, the
//                  rows of the current range.  A range (32 MB of 128-byte
//                  lines at shift 18) is fetched from HBM once and then
//                  served from L2 to all the wave's queries.  After the last
//                  range the counters are thresholded exactly as in
//                  gather_kernel (same hits, same dense scores).
//
// Counts are sums of the same masks in a different order, so results are
// identical to gather_kernel and to the reference.  Eligible batches: k = 1,
// 32-bit rows, every query <= 1,024 windows (NT <= 12), resident index.
//
// Status: opt-in (COBS_TILED=1), never chosen automatically.  Measured on a
// B200 it is 1.7-2.6x slower than gather_kernel, even with an L2-resident
// index: at L2-sized ranges a query has only ~15-30 rows per range, so the
// per-(query, range) work (state in/out of shared memory, list chunk, phase
// arrival) is as large as the row work, and the grid-wide range lockstep
// leaves warps waiting (profiles/r1/tiled_gather.md).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "gather_common.cuh"
#include "tiled.hpp"

namespace cobsg {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kBins = 64;        // row ranges per block, at most
constexpr int kLPL = 32;         // terms per lane in the bucket kernel -> l <= 1,024
constexpr int kBucketWarps = 8;
constexpr size_t kBucketSmemPerWarp = (kBins + 1024) * 4;
constexpr uint32_t kMaxLag = 7;  // phase arrival slots per CTA: 8

struct BucketArgs {
    const uint64_t* hashes;
    const uint64_t* win_base;
    const uint32_t* ell;
    uint64_t q0;
    uint32_t nq;
    const DevBlock* blocks;
    const uint8_t* shift;
    uint32_t nb;
    uint32_t* lists;
    uint64_t slots;
};

// One warp per query.  The query's hashes stay in registers; for each block:
// rows (exact h mod w_b), a shared atomic per row on its range's counter
// gives the row's rank within the range, a warp scan of the (<= 64) counts
// gives the range offsets, and the rows are placed into a shared staging
// list and written out coalesced.  Within a range the order is arbitrary
// (counts are sums, they commute).
__global__ void __launch_bounds__(kBucketWarps * 32, 2) bucket_kernel(BucketArgs a) {
    extern __shared__ uint32_t bsm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t qi = a.q0 + static_cast<uint64_t>(blockIdx.x) * kBucketWarps + warp;
    if (qi >= a.q0 + a.nq) return;
    const uint32_t ell = a.ell[qi];
    if (ell == 0) return;
    uint32_t* cnt = bsm + warp * (kBins + 1024); // per range: count, then offset
    uint32_t* stage = cnt + kBins;
    const uint64_t* hq = a.hashes + a.win_base[qi]; // k = 1: one hash per term
    uint64_t h[kLPL];
#pragma unroll
    for (int j = 0; j < kLPL; ++j) {
        const uint32_t t = j * 32 + lane;
        h[j] = t < ell ? __ldg(hq + t) : 0;
    }
    uint32_t* out0 = a.lists + (a.win_base[qi] - a.win_base[a.q0]);
    for (uint32_t b = 0; b < a.nb; ++b) {
        const DevBlock B = a.blocks[b];
        const uint32_t sh = a.shift[b];
#pragma unroll
        for (int k = 0; k < kBins / 32; ++k) cnt[lane + 32 * k] = 0;
        __syncwarp();
        uint32_t row[kLPL], rank[kLPL / 2]; // two 16-bit ranks per word (l <= 1,024)
#pragma unroll
        for (int j = 0; j < kLPL; ++j) {
            const uint32_t t = j * 32 + lane;
            uint32_t rk = 0;
            row[j] = 0;
            if (t < ell) {
                row[j] = static_cast<uint32_t>(fastmod(h[j], B.w, B.magic)); // query.cpp:63
                rk = atomicAdd(&cnt[row[j] >> sh], 1u);
            }
            if (j & 1) rank[j / 2] |= rk << 16;
            else rank[j / 2] = rk;
        }
        __syncwarp();
        // exclusive offsets of the ranges: lane l scans ranges 8l .. 8l+7, then a warp scan
        uint32_t cv[kBins / 32], run = 0;
#pragma unroll
        for (int k = 0; k < kBins / 32; ++k) {
            cv[k] = cnt[lane * (kBins / 32) + k];
            run += cv[k];
        }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        __syncwarp();
        uint32_t off = incl - run;
#pragma unroll
        for (int k = 0; k < kBins / 32; ++k) {
            cnt[lane * (kBins / 32) + k] = off;
            off += cv[k];
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kLPL; ++j) {
            const uint32_t t = j * 32 + lane;
            if (t < ell) stage[cnt[row[j] >> sh] + ((rank[j / 2] >> ((j & 1) * 16)) & 0xffffu)] = row[j];
        }
        __syncwarp();
        uint32_t* out = out0 + static_cast<uint64_t>(b) * a.slots;
        for (uint32_t t = lane; t < ell; t += 32) __stcs(out + t, stage[t]);
        __syncwarp();
    }
}

struct TileArgs {
    const uint8_t* payload;
    const DevBlock* blocks;
    const uint32_t* ct;
    uint32_t nct;
    const uint8_t* shift;
    const uint32_t* lists;
    uint64_t slots;
    const uint64_t* win_base;
    const uint32_t* ell;
    const uint32_t* tau;
    uint64_t q0;
    uint32_t nq;
    uint32_t qs;
    uint64_t D;
    void* scores;
    int want_hits;
    uint32_t* hit_count;
    unsigned long long* hit_total;
    uint64_t hit_cap;
    uint32_t* hit_q;
    uint32_t* hit_doc;
    uint32_t* hit_score;
    uint32_t* done; // per phase: CTAs whose warps all finished it
    uint32_t lag;
};

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait until every CTA finished phase p.  Bounded: the guard only shapes L2
// locality, so after 20 ms it gives up rather than ever hang.
__device__ __forceinline__ void wait_phase(const uint32_t* p, uint32_t target) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) return;
    const uint64_t t0 = globaltimer();
    do {
        __nanosleep(64);
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    } while (v < target && globaltimer() - t0 < 20000000ull);
}

// Bulk (copy-engine) prefetch of [p, p + bytes) into L2; bytes % 16 == 0.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// This CTA's share of the rows of phase (column task ci, range r): the whole
// range is brought into L2 by the grid one phase before it is gathered, so
// HBM streams the index sequentially and the gather hits L2.

// Predicated row load (no memory access when !pred).
__device__ __forceinline__ uint32_t ld_row_if(const uint8_t* p, uint32_t pred) {
    uint32_t v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.L1::no_allocate.b32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "l"(p), "r"(pred));
    return v;
}

// One persistent CTA per SM, W warps; warp w owns the CTA's queries w, w+W,
// ... (at most QPW).  Per phase (one row range of one column task) a warp
// walks its queries with a two-deep pipeline: the row loads of query i+1 are
// issued before the carry-save adds of query i.  Each query's list chunk for
// the next phase is loaded (into a register per query) right after its
// cursor moves, a whole phase ahead of use.
__device__ __forceinline__ void prefetch_phase(const TileArgs& a, uint32_t ci, uint32_t r) {
    const uint32_t b = a.ct[2 * ci], sl = a.ct[2 * ci + 1];
    const DevBlock B = a.blocks[b];
    const uint32_t sh = a.shift[b];
    const uint64_t row0 = static_cast<uint64_t>(r) << sh;
    const uint64_t row1 = min(B.w, static_cast<uint64_t>(r + 1) << sh);
    const uint8_t* base = a.payload + B.base;
    if (B.pitch <= 128u) { // one slice: the range is one contiguous run of rows
        const uint64_t lo = row0 * B.pitch, hi = row1 * B.pitch;
        const uint64_t per = ((hi - lo + gridDim.x - 1) / gridDim.x + 4095) & ~4095ull;
        const uint64_t c0 = lo + blockIdx.x * per, c1 = min(hi, c0 + per);
        for (uint64_t o = c0 + threadIdx.x * 4096ull; o < c1; o += blockDim.x * 4096ull)
            bulk_prefetch_l2(base + o, static_cast<uint32_t>(min(static_cast<uint64_t>(4096), c1 - o)));
    } else { // this slice's 128 bytes of every row of the range
        const uint32_t len = min(128u, B.pitch - sl * 128u);
        const uint64_t per = (row1 - row0 + gridDim.x - 1) / gridDim.x;
        const uint64_t q0 = row0 + blockIdx.x * per, q1 = min(row1, q0 + per);
        for (uint64_t rr = q0 + threadIdx.x; rr < q1; rr += blockDim.x)
            bulk_prefetch_l2(base + rr * B.pitch + sl * 128u, len);
    }
}

template <int NT, int W, int QPW>
__global__ void __launch_bounds__(W * 32, 1) tile_kernel(TileArgs a) {
    constexpr int LCH = 5;        // carry-save levels ones..sixteens
    constexpr int NPP = NT - LCH; // planes of weight 32, 64, ...
    extern __shared__ __align__(16) uint32_t tsm[];
    __shared__ uint32_t s_arrive[kMaxLag + 1];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x <= kMaxLag) s_arrive[threadIdx.x] = 0;
    __syncthreads();
    uint32_t* rs = tsm + a.qs * NT * 32 + warp * 32; // this warp's row broadcast list
    const uint64_t qb = a.q0 + static_cast<uint64_t>(blockIdx.x) * a.qs;
    const uint64_t qend = a.q0 + a.nq;
    const uint32_t nown = qb >= qend ? 0u : static_cast<uint32_t>(min(static_cast<uint64_t>(a.qs), qend - qb));
    const uint32_t nmine = warp < nown ? min((nown - warp + W - 1) / W, static_cast<uint32_t>(QPW)) : 0u;
    // lane i holds the warp's i-th query: l, list offset, cursor
    uint32_t my_ell = 0, my_lo = 0, my_cur = 0;
    if (lane < nmine) {
        const uint64_t qi = qb + warp + lane * W;
        my_ell = a.ell[qi];
        my_lo = static_cast<uint32_t>(a.win_base[qi] - a.win_base[a.q0]);
    }
    const uint32_t target = gridDim.x;
    uint32_t g = 0; // global phase index
    if (a.nct) prefetch_phase(a, 0, 0);
    for (uint32_t ci = 0; ci < a.nct; ++ci) {
        const uint32_t bidx = a.ct[2 * ci], slice = a.ct[2 * ci + 1];
        const DevBlock B = a.blocks[bidx];
        const uint32_t sh = a.shift[bidx];
        const uint32_t nbins = static_cast<uint32_t>((B.w - 1) >> sh) + 1u;
        // lanes past the pitch re-read an in-row word (their documents are masked)
        const uint32_t lane_byte = min(slice * 128u + lane * 4u, B.pitch - 4u);
        const uint8_t* rowbase = a.payload + B.base + lane_byte;
        const uint32_t* Lb = a.lists + static_cast<uint64_t>(bidx) * a.slots;
        my_cur = 0;
        // the 32 list entries of query i from position c (all lanes call it)
        auto list_at = [&](uint32_t i, uint32_t c) -> uint32_t {
            const uint32_t e = __shfl_sync(kFull, my_ell, i);
            const uint32_t lo = __shfl_sync(kFull, my_lo, i);
            return c + lane < e ? __ldcs(Lb + lo + c + lane) : 0xffffffffu;
        };
        uint32_t L[QPW];
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
            if (i < static_cast<int>(nmine)) {
                uint32_t* s = tsm + (warp + i * W) * NT * 32 + lane;
#pragma unroll
                for (int p = 0; p < NT; ++p) s[p * 32] = 0;
                L[i] = list_at(i, 0);
            }
        }
        for (uint32_t r = 0; r < nbins; ++r, ++g) {
            if (g >= a.lag) {
                if (lane == 0) wait_phase(a.done + (g - a.lag), target);
                __syncwarp();
            }
            if (r + 1 < nbins) prefetch_phase(a, ci, r + 1); // next range into L2 meanwhile
            else if (ci + 1 < a.nct) prefetch_phase(a, ci + 1, 0);
            // rows of range r at the head of a chunk (lists are range-sorted)
            auto count = [&](uint32_t i, uint32_t rowv) -> uint32_t {
                const uint32_t c = __shfl_sync(kFull, my_cur, i), e = __shfl_sync(kFull, my_ell, i);
                return __popc(__ballot_sync(kFull, c + lane < e && (rowv >> sh) == r));
            };
            auto issue = [&](uint32_t rowv, uint32_t n, uint32_t(&v)[32]) {
                rs[lane] = rowv;
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 32; u += 4) {
                    if (u < static_cast<int>(n)) { // uniform: only the groups that hold rows issue
                        const uint4 r4 = *reinterpret_cast<const uint4*>(rs + u);
                        v[u + 0] = ld_row_if(row_addr(rowbase, r4.x, B.pitch), 1u);
                        v[u + 1] = ld_row_if(row_addr(rowbase, r4.y, B.pitch), u + 1 < static_cast<int>(n));
                        v[u + 2] = ld_row_if(row_addr(rowbase, r4.z, B.pitch), u + 2 < static_cast<int>(n));
                        v[u + 3] = ld_row_if(row_addr(rowbase, r4.w, B.pitch), u + 3 < static_cast<int>(n));
                    } else {
                        v[u + 0] = v[u + 1] = v[u + 2] = v[u + 3] = 0;
                    }
                }
                __syncwarp();
            };
            // query i: its rows of range r (already in flight in v, n of them)
            // into its carry-save state; more than one chunk (rare) synchronously
            auto consume = [&](int i, uint32_t(&v)[32], uint32_t n) {
                uint32_t c = __shfl_sync(kFull, my_cur, i);
                uint32_t* s = tsm + (warp + i * W) * NT * 32 + lane;
                uint32_t ones = s[0], twos = s[32], fours = s[64], eights = s[96], sixteens = s[128];
                uint32_t P[NPP];
#pragma unroll
                for (int p = 0; p < NPP; ++p) P[p] = s[(LCH + p) * 32];
                auto add = [&](const uint32_t(&x)[32], uint32_t m) {
                    uint32_t carry = csa16(x, ones, twos, fours, eights);
                    if (m > 16) {
                        const uint32_t c2 = csa16(x + 16, ones, twos, fours, eights);
                        csa(carry, sixteens, sixteens, carry, c2); // weight 32
                    } else {
                        const uint32_t t = sixteens & carry;
                        sixteens ^= carry;
                        carry = t;
                    }
#pragma unroll
                    for (int p = 0; p < NPP; ++p) {
                        const uint32_t t = P[p] & carry;
                        P[p] ^= carry;
                        carry = t;
                    }
                };
                if (n) add(v, n);
                c += n;
                while (n == 32) { // more of range r than one chunk (rare)
                    const uint32_t rowv = list_at(i, c);
                    n = __popc(__ballot_sync(kFull, c + lane < __shfl_sync(kFull, my_ell, i) && (rowv >> sh) == r));
                    if (n) {
                        issue(rowv, n, v);
                        add(v, n);
                    }
                    c += n;
                }
                s[0] = ones;
                s[32] = twos;
                s[64] = fours;
                s[96] = eights;
                s[128] = sixteens;
#pragma unroll
                for (int p = 0; p < NPP; ++p) s[(LCH + p) * 32] = P[p];
                if (lane == static_cast<uint32_t>(i)) my_cur = c;
                L[i] = list_at(i, c); // next phase's chunk, a phase ahead
            };
            // two-deep pipeline over the warp's queries, ping-pong buffers
            uint32_t va[32], vb[32], na = 0, nb = 0;
            if (nmine) {
                na = count(0, L[0]);
                issue(L[0], na, va);
            }
#pragma unroll
            for (int i = 0; i < QPW; i += 2) {
                if (i < static_cast<int>(nmine)) {
                    if (i + 1 < static_cast<int>(nmine)) {
                        nb = count(i + 1, L[i + 1]);
                        issue(L[i + 1], nb, vb);
                    }
                    consume(i, va, na);
                }
                if (i + 1 < static_cast<int>(nmine)) {
                    if (i + 2 < static_cast<int>(nmine) && i + 2 < QPW) {
                        na = count(i + 2, L[(i + 2) % QPW]);
                        issue(L[(i + 2) % QPW], na, va);
                    }
                    consume(i + 1, vb, nb);
                }
            }
            __syncwarp();
            if (lane == 0) { // the CTA's last warp to finish the phase signals it
                const uint32_t old = atomicAdd(&s_arrive[g & kMaxLag], 1u);
                if (old == W - 1) {
                    s_arrive[g & kMaxLag] = 0;
                    atomicAdd(a.done + g, 1u);
                }
            }
        }
        // thresholds, hits and dense scores of this column task (as gather_kernel)
        const uint32_t d0 = slice * 1024u + lane * 32u;
        uint32_t valid = 0;
        if (d0 < B.dc) valid = (B.dc - d0 >= 32u) ? 0xffffffffu : ((1u << (B.dc - d0)) - 1u);
        const uint64_t gdoc0 = static_cast<uint64_t>(B.doc_base) + d0;
        for (uint32_t i = 0; i < nmine; ++i) {
            const uint64_t qi = qb + warp + i * W;
            if (__shfl_sync(kFull, my_ell, i) == 0) continue; // DataError query
            const uint32_t* s = tsm + (warp + i * W) * NT * 32 + lane;
            uint32_t F[NT];
#pragma unroll
            for (int p = 0; p < LCH; ++p) F[p] = 0;
#pragma unroll
            for (int p = 0; p < NPP; ++p) F[LCH + p] = s[(LCH + p) * 32];
            add_at<NT>(F, 4, s[128]);
            add_at<NT>(F, 3, s[96]);
            add_at<NT>(F, 2, s[64]);
            add_at<NT>(F, 1, s[32]);
            add_at<NT>(F, 0, s[0]);
            if (a.scores) {
                uint16_t* row = static_cast<uint16_t*>(a.scores) + qi * a.D + gdoc0; // NT <= 16
                for (int b = 0; b < 32; ++b)
                    if ((valid >> b) & 1u) row[b] = static_cast<uint16_t>(extract<NT>(F, b));
            }
            if (!a.want_hits) continue;
            uint32_t hits = ge_mask<NT>(F, a.tau[qi]) & valid;
            const uint32_t cnt = __popc(hits);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, o);
                if (lane >= static_cast<uint32_t>(o)) incl += y;
            }
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            if (total == 0) continue;
            unsigned long long base = 0;
            if (lane == 31) {
                base = atomicAdd(a.hit_total, static_cast<unsigned long long>(total));
                atomicAdd(a.hit_count + qi, total);
            }
            base = __shfl_sync(kFull, base, 31);
            uint64_t idx = base + incl - cnt;
            while (hits) {
                const int b = __ffs(hits) - 1;
                hits &= hits - 1;
                if (idx < a.hit_cap) {
                    a.hit_q[idx] = static_cast<uint32_t>(qi);
                    a.hit_doc[idx] = static_cast<uint32_t>(gdoc0 + b);
                    a.hit_score[idx] = extract<NT>(F, b);
                }
                ++idx;
            }
        }
    }
}

using TileFn = void (*)(TileArgs);

constexpr int kQPW16 = 11; // queries per warp at 16 warps (<= 176 per CTA)
constexpr int kQPW24 = 8;  // at 24 warps

TileFn pick_tile(int nt, int warps) {
    if (nt == 10) return warps == 24 ? tile_kernel<10, 24, kQPW24> : tile_kernel<10, 16, kQPW16>;
    return warps == 24 ? tile_kernel<12, 24, kQPW24> : tile_kernel<12, 16, kQPW16>;
}

size_t tile_smem(int nt, int warps, uint32_t qs) {
    return static_cast<size_t>(qs) * nt * 32 * 4 + static_cast<size_t>(warps) * 32 * 4;
}

} // namespace

TiledPlan tiled_plan(DeviceIndex& ix, const std::vector<uint64_t>& win_base, uint64_t n, int nt_needed,
                     bool prune) {
    TiledPlan tp;
    const char* env = std::getenv("COBS_TILED");
    const int mode = env ? std::atoi(env) : -1; // 0 off, 1 force (when eligible), -1 auto
    // Measured slower than gather_kernel on every shape tried (DESIGN.md
    // section 2, "L2-tiled gather"): opt-in only, auto never selects it --
    // and returns before any CUDA query, so the default batch pays nothing.
    if (mode != 1) return tp.why = mode == 0 ? "off" : "auto: the warp-per-query gather is faster", tp;
    const Params& P = ix.meta.params;
    if (ix.streaming()) return tp.why = "streaming index", tp;
    if (P.k != 1) return tp.why = "k > 1", tp;
    if (prune) return tp.why = "pruning", tp;
    if (nt_needed > 12) return tp.why = "windows > 4095", tp;
    uint64_t wmax = 0, sum_w = 0;
    for (uint64_t i = 0; i < n; ++i) wmax = std::max(wmax, win_base[i + 1] - win_base[i]);
    if (wmax > 1024) return tp.why = "windows > 1024", tp;
    for (const DevBlock& d : ix.blocks) {
        if (d.w > 0xffffffffull) return tp.why = "width >= 2^32", tp;
        sum_w += d.w;
    }
    tp.nt = nt_needed <= 10 ? 10 : 12;
    if (const char* e = std::getenv("COBS_TILE_WARPS")) tp.warps = std::atoi(e) == 24 ? 24 : 16;
    if (const char* e = std::getenv("COBS_TILE_SHIFT")) tp.base_shift = std::max(10, std::min(28, std::atoi(e)));
    if (const char* e = std::getenv("COBS_TILE_LAG")) tp.lag = std::max(1, std::min<int>(kMaxLag, std::atoi(e)));
    int nsm = 0, smem_max = 0;
    COBS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ix.device));
    COBS_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix.device));
    const uint64_t per_q = static_cast<uint64_t>(tp.nt) * 32 * 4;
    uint64_t qs_max = (static_cast<uint64_t>(smem_max) - tile_smem(tp.nt, tp.warps, 0)) / per_q;
    qs_max = std::min<uint64_t>(qs_max, static_cast<uint64_t>(tp.warps) * (tp.warps == 24 ? kQPW24 : kQPW16));
    // list memory: nb x (slots of a wave) x 4 bytes
    size_t free_b = 0, total_b = 0;
    COBS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t nb = ix.blocks.size();
    const uint64_t avg_w = std::max<uint64_t>(1, win_base[n] / std::max<uint64_t>(n, 1));
    const uint64_t avail = free_b + ix.ws.tlist.bytes; // the list buffer is reused across batches
    const uint64_t budget = avail > (2ull << 30) ? avail - (2ull << 30) : 0;
    uint64_t qs_mem = budget / std::max<uint64_t>(1, nb * avg_w * 4 * 2 * nsm); // 2x: slack for uneven windows
    uint64_t qs_cap = std::min(qs_max, qs_mem);
    if (const char* e = std::getenv("COBS_TILE_QS")) qs_cap = std::min<uint64_t>(qs_cap, std::max(1, std::atoi(e)));
    if (qs_cap < 1 || (mode < 0 && qs_cap < static_cast<uint64_t>(tp.warps))) return tp.why = "no room for the lists", tp;
    const uint64_t waves = (n + qs_cap * nsm - 1) / (qs_cap * nsm);
    // balanced waves, queries per CTA a multiple of the warps when possible
    uint64_t qs = (n + waves * nsm - 1) / (waves * nsm);
    qs = std::min(qs_cap, qs >= static_cast<uint64_t>(tp.warps) ? (qs + tp.warps - 1) / tp.warps * tp.warps : qs);
    const uint64_t per_wave = qs * nsm;
    // auto: tile only when the wave reads each row several times and the
    // index is far larger than L2 (a small index is L2-resident anyway)
    const double reuse = static_cast<double>(std::min<uint64_t>(per_wave, n)) * avg_w /
                         (static_cast<double>(sum_w) / std::max<uint64_t>(nb, 1));
    (void)reuse; // (a future auto mode would require reuse >= 2 and an index far larger than L2)
    tp.qs = static_cast<uint32_t>(qs);
    tp.grid = static_cast<uint32_t>(nsm);
    for (uint64_t q0 = 0; q0 < n; q0 += per_wave) {
        tp.wave_q0.push_back(q0);
        tp.slots = std::max(tp.slots, win_base[std::min(n, q0 + per_wave)] - win_base[q0]);
    }
    tp.wave_q0.push_back(n);
    if (nb * tp.slots * 4 > budget || tp.slots >= (1ull << 32)) return tp.why = "no room for the lists", tp;
    tp.shift.resize(nb);
    tp.phases = 0;
    for (uint64_t b = 0; b < nb; ++b) {
        uint32_t s = tp.base_shift;
        while (((ix.blocks[b].w - 1) >> s) >= static_cast<uint64_t>(kBins)) ++s;
        tp.shift[b] = static_cast<uint8_t>(s);
    }
    for (uint32_t b : ix.ct_block) tp.phases += static_cast<uint32_t>((ix.blocks[b].w - 1) >> tp.shift[b]) + 1u;
    tp.use = true;
    tp.why = "tiled";
    if (std::getenv("COBS_TILE_VERBOSE")) {
        std::fprintf(stderr, "tiled: nt %d warps %d qs %u waves %zu slots %llu phases %u lag %u\n", tp.nt, tp.warps, tp.qs,
                     tp.wave_q0.size() - 1, static_cast<unsigned long long>(tp.slots), tp.phases, tp.lag);
        for (uint64_t b = 0; b < nb; ++b)
            std::fprintf(stderr, "  block %llu w %llu shift %u ranges %llu range_MB %.1f\n", static_cast<unsigned long long>(b),
                         static_cast<unsigned long long>(ix.blocks[b].w), tp.shift[b],
                         static_cast<unsigned long long>(((ix.blocks[b].w - 1) >> tp.shift[b]) + 1),
                         (1ull << tp.shift[b]) * 128.0 / 1e6);
    }
    return tp;
}

uint32_t tiled_gather(DeviceIndex& ix, const TiledPlan& tp, cudaStream_t st, const TiledIO& io) {
    QueryWorkspace& ws = ix.ws;
    const uint32_t nb = static_cast<uint32_t>(ix.blocks.size());
    ws.tlist.reserve(std::max<uint64_t>(nb * tp.slots * 4, 4));
    ws.tdone.reserve(std::max<uint64_t>(tp.phases * 4ull, 4));
    ws.tshift.reserve(std::max<uint64_t>(nb, 1));
    COBS_CUDA(cudaMemcpyAsync(ws.tshift.ptr, tp.shift.data(), nb, cudaMemcpyHostToDevice, st));
    const size_t bsmem = kBucketWarps * kBucketSmemPerWarp;
    COBS_CUDA(cudaFuncSetAttribute(bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bsmem)));
    TileFn tf = pick_tile(tp.nt, tp.warps);
    const size_t tsmem = tile_smem(tp.nt, tp.warps, tp.qs);
    COBS_CUDA(cudaFuncSetAttribute(tf, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem)));
    uint32_t launches = 0;
    for (size_t w = 0; w + 1 < tp.wave_q0.size(); ++w) {
        const uint64_t q0 = tp.wave_q0[w];
        const uint32_t nq = static_cast<uint32_t>(tp.wave_q0[w + 1] - q0);
        BucketArgs ba{};
        ba.hashes = io.hashes;
        ba.win_base = io.win_base;
        ba.ell = io.ell;
        ba.q0 = q0;
        ba.nq = nq;
        ba.blocks = ix.d_blocks;
        ba.shift = ws.tshift.as<uint8_t>();
        ba.nb = nb;
        ba.lists = ws.tlist.as<uint32_t>();
        ba.slots = tp.slots;
        bucket_kernel<<<(nq + kBucketWarps - 1) / kBucketWarps, kBucketWarps * 32, bsmem, st>>>(ba);
        const cudaError_t bucket_launch = cudaGetLastError();
        COBS_CUDA(bucket_launch);
        if (std::getenv("COBS_TILE_SYNC")) COBS_CUDA(cudaStreamSynchronize(st)); // debug: fault location
        COBS_CUDA(cudaMemsetAsync(ws.tdone.ptr, 0, tp.phases * 4ull, st));
        TileArgs ta{};
        ta.payload = ix.payload;
        ta.blocks = ix.d_blocks;
        ta.ct = ix.d_ct;
        ta.nct = static_cast<uint32_t>(ix.ct_block.size());
        ta.shift = ws.tshift.as<uint8_t>();
        ta.lists = ws.tlist.as<uint32_t>();
        ta.slots = tp.slots;
        ta.win_base = io.win_base;
        ta.ell = io.ell;
        ta.tau = io.tau;
        ta.q0 = q0;
        ta.nq = nq;
        ta.qs = tp.qs;
        ta.D = io.D;
        ta.scores = io.scores;
        ta.want_hits = io.want_hits;
        ta.hit_count = io.hit_count;
        ta.hit_total = io.hit_total;
        ta.hit_cap = io.hit_cap;
        ta.hit_q = io.hit_q;
        ta.hit_doc = io.hit_doc;
        ta.hit_score = io.hit_score;
        ta.done = ws.tdone.as<uint32_t>();
        ta.lag = tp.lag;
        const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(tp.grid, (nq + tp.qs - 1) / tp.qs));
        void* args[] = {&ta};
        // co-resident CTAs (one per SM) so the phase guard never waits on an unscheduled CTA
        cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tf), dim3(grid),
                                                    dim3(tp.warps * 32), args, tsmem, st);
        if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
            (void)cudaGetLastError();
            tf<<<grid, tp.warps * 32, tsmem, st>>>(ta); // the guard times out instead of hanging
            e = cudaGetLastError();
        }
        const cudaError_t tile_launch = e;
        COBS_CUDA(tile_launch);
        if (std::getenv("COBS_TILE_SYNC")) COBS_CUDA(cudaStreamSynchronize(st));
        launches += 2;
    }
    return launches;
}

} // namespace cobsg
