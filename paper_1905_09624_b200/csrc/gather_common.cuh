// Bit-sliced counting helpers shared by the row-gather kernels (query.cu:
// gather_kernel).  The reference counts with a
// 256 x 8 expand table per AND byte (query.cpp:25-45,74-81); here 32
// documents' counts live as bit planes of one 32-bit word per lane and
// masks are added with carry-save (Harley-Seal) adders.
#pragma once

#include <cstdint>

namespace cobsg {

// Carry-save adder: (hi, lo) = a + b + c.
__device__ __forceinline__ void csa(uint32_t& hi, uint32_t& lo, uint32_t a, uint32_t b, uint32_t c) {
    uint32_t u = a ^ b;
    hi = (a & b) | (u & c);
    lo = u ^ c;
}

template <bool EF>
__device__ __forceinline__ uint32_t ld_row(const uint8_t* p, uint64_t policy) {
    uint32_t v;
    if (EF)
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
            : "=r"(v)
            : "l"(p), "l"(policy));
    else
        asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// rowbase + row * pitch in one IMAD.WIDE.U32.
__device__ __forceinline__ const uint8_t* row_addr(const uint8_t* base, uint32_t row, uint32_t pitch) {
    const uint8_t* p;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(row), "r"(pitch), "l"(base));
    return p;
}

// Bit-sliced counters: a document's count is sum_p 2^p * bit(F[p]).
template <int NT>
__device__ __forceinline__ void add_at(uint32_t (&F)[NT], int level, uint32_t x) {
#pragma unroll
    for (int p = 0; p < NT; ++p) {
        if (p >= level) {
            uint32_t t = F[p] & x;
            F[p] ^= x;
            x = t;
        }
    }
}

template <int NT>
__device__ __forceinline__ uint32_t extract(const uint32_t (&F)[NT], int i) {
    uint32_t s = 0;
#pragma unroll
    for (int p = 0; p < NT; ++p) s |= ((F[p] >> i) & 1u) << p;
    return s;
}

// Bit-sliced F >= T over the 32 documents of a lane at once.
template <int NT>
__device__ __forceinline__ uint32_t ge_mask(const uint32_t (&F)[NT], uint32_t T) {
    uint32_t gt = 0, eq = 0xffffffffu;
#pragma unroll
    for (int p = NT - 1; p >= 0; --p) {
        const uint32_t tb = ((T >> p) & 1u) ? 0xffffffffu : 0u;
        gt |= eq & F[p] & ~tb;
        eq &= ~(F[p] ^ tb);
    }
    if constexpr (NT < 32) {
        if ((T >> NT) != 0u) return 0u; // T beyond the representable counts
    }
    return gt | eq;
}

// Harley-Seal step: 16 document masks into the carry-save accumulators;
// returns the weight-16 carry.
__device__ __forceinline__ uint32_t csa16(const uint32_t* v, uint32_t& ones, uint32_t& twos,
                                          uint32_t& fours, uint32_t& eights) {
    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
    csa(twosA, ones, ones, v[0], v[1]);
    csa(twosB, ones, ones, v[2], v[3]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, v[4], v[5]);
    csa(twosB, ones, ones, v[6], v[7]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsA, fours, fours, foursA, foursB);
    csa(twosA, ones, ones, v[8], v[9]);
    csa(twosB, ones, ones, v[10], v[11]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, v[12], v[13]);
    csa(twosB, ones, ones, v[14], v[15]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsB, fours, fours, foursA, foursB);
    csa(sixteens, eights, eights, eightsA, eightsB);
    return sixteens;
}

// Where a gather writes a finished (query, slice)'s results: dense scores
// and/or hits (document order within the slice; kernel 3 orders them).
struct EmitArgs {
    void* scores; // dense [n][D] (uint16 when NT <= 16, else uint32) or null
    uint64_t D;
    int want_hits;
    uint32_t* hit_count; // per query
    unsigned long long* hit_total;
    uint64_t hit_cap;
    uint32_t* hit_q;
    uint32_t* hit_doc;
    uint32_t* hit_score;
};

// The 32 documents of a lane (global columns gdoc0.., `valid` of them real)
// with counts F: dense scores, then F >= tau bit-sliced over all 32 at once,
// compacted with a warp scan and one atomic per warp (query.cpp:83-88).
template <int NT>
__device__ __forceinline__ void emit_slice(const EmitArgs& a, uint64_t qi, uint64_t gdoc0, uint32_t valid,
                                           uint32_t tau, const uint32_t (&F)[NT], uint32_t lane) {
    if (a.scores) {
        if (NT <= 16) {
            uint16_t* row = static_cast<uint16_t*>(a.scores) + qi * a.D + gdoc0;
            for (int i = 0; i < 32; ++i)
                if ((valid >> i) & 1u) row[i] = static_cast<uint16_t>(extract<NT>(F, i));
        } else {
            uint32_t* row = static_cast<uint32_t*>(a.scores) + qi * a.D + gdoc0;
            for (int i = 0; i < 32; ++i)
                if ((valid >> i) & 1u) row[i] = extract<NT>(F, i);
        }
    }
    if (!a.want_hits) return;
    uint32_t hits = ge_mask<NT>(F, tau) & valid;
    uint32_t cnt = __popc(hits);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    unsigned long long base = 0;
    if (lane == 31) {
        base = atomicAdd(a.hit_total, (unsigned long long)total);
        atomicAdd(a.hit_count + qi, total);
    }
    base = __shfl_sync(0xffffffffu, base, 31);
    uint64_t idx = base + incl - cnt;
    while (hits) {
        int i = __ffs(hits) - 1;
        hits &= hits - 1;
        if (idx < a.hit_cap) {
            a.hit_q[idx] = static_cast<uint32_t>(qi);
            a.hit_doc[idx] = static_cast<uint32_t>(gdoc0 + i);
            a.hit_score[idx] = extract<NT>(F, i);
        }
        ++idx;
    }
}

} // namespace cobsg
