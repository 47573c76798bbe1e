// Device-side building blocks shared by the query and build kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "host.hpp"

namespace cobsg {

#define COBS_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::cobsg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

// One block of the device-resident index.  Rows are re-pitched to a 32-byte
// multiple so a warp's 128-byte column slice never straddles an extra DRAM
// sector; bytes [row_bytes, pitch) of every row are zero.
struct DevBlock {
    uint64_t base;  // byte offset of row 0 in the payload allocation
    uint64_t w;     // rows (Bloom width)
    uint64_t magic; // floor((2^64-1)/w) for the exact modulo below
    uint32_t pitch; // device bytes per row
    uint32_t rb;    // file bytes per row = ceil(doc_count/8)
    uint32_t dc;    // documents
    uint32_t doc_base;
};

// h mod w, exact for all 64-bit h and w >= 1: the magic quotient is at most
// two below the true one, so two conditional subtractions
// finish it.  Replaces the reference's `% w` (query.cpp:63,68,
// termizer.cpp:135) without a 64-bit divide.
__host__ __device__ __forceinline__ uint64_t fastmod(uint64_t h, uint64_t w, uint64_t magic) {
#ifdef __CUDA_ARCH__
    uint64_t q = __umul64hi(h, magic);
#else
    uint64_t q = (uint64_t)(((unsigned __int128)h * magic) >> 64);
#endif
    uint64_t r = h - q * w;
    if (r >= w) r -= w;
    if (r >= w) r -= w;
    return r;
}
inline uint64_t mod_magic(uint64_t w) { return ~0ULL / w; }

// ---- XXH64 (FORMAT.md "Term hashing"; reference xxhash64.hpp:45-95) ----

namespace xx {
constexpr uint64_t P1 = 0x9E3779B185EBCA87ULL, P2 = 0xC2B2AE3D27D4EB4FULL,
                   P3 = 0x165667B19E3779F9ULL, P4 = 0x85EBCA77C2B2AE63ULL,
                   P5 = 0x27D4EB2F165667C5ULL;
__device__ __forceinline__ uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__device__ __forceinline__ uint64_t rnd(uint64_t acc, uint64_t lane) {
    return rotl(acc + lane * P2, 31) * P1;
}
} // namespace xx

// Complement of an A/C/G/T byte (termizer.cpp:18-26), branch-free: bit 1 is
// set for C/G (xor 0x04 swaps them) and clear for A/T (xor 0x15 swaps them).
__device__ __forceinline__ uint32_t comp_byte(uint32_t c) { return c ^ ((c & 2u) ? 0x04u : 0x15u); }

__device__ __forceinline__ bool is_acgt(uint32_t c) {
    return c == 'A' || c == 'C' || c == 'G' || c == 'T';
}

// Byte i of a window as the termizer would emit it: forward bytes, or the
// reverse complement when `rc` (termizer.cpp:117-119).
__device__ __forceinline__ uint32_t term_byte(const uint8_t* w, uint32_t q, bool rc, uint32_t i) {
    return rc ? comp_byte(w[q - 1 - i]) : (uint32_t)w[i];
}

__device__ __forceinline__ uint64_t term_lane64(const uint8_t* w, uint32_t q, bool rc, uint32_t i) {
    uint64_t v = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) v = (v << 8) | term_byte(w, q, rc, i + (uint32_t)b);
    return v;
}

// XXH64(term bytes, seed) of a window, reading the window in place.
__device__ __forceinline__ uint64_t xxh64_term(const uint8_t* w, uint32_t q, bool rc, uint64_t seed) {
    using namespace xx;
    uint32_t i = 0;
    uint64_t h;
    if (q >= 32) {
        uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        do {
            v1 = rnd(v1, term_lane64(w, q, rc, i));
            v2 = rnd(v2, term_lane64(w, q, rc, i + 8));
            v3 = rnd(v3, term_lane64(w, q, rc, i + 16));
            v4 = rnd(v4, term_lane64(w, q, rc, i + 24));
            i += 32;
        } while (i + 32 <= q);
        h = rotl(v1, 1) + rotl(v2, 7) + rotl(v3, 12) + rotl(v4, 18);
        h = (h ^ rnd(0, v1)) * P1 + P4;
        h = (h ^ rnd(0, v2)) * P1 + P4;
        h = (h ^ rnd(0, v3)) * P1 + P4;
        h = (h ^ rnd(0, v4)) * P1 + P4;
    } else {
        h = seed + P5;
    }
    h += q;
    for (; i + 8 <= q; i += 8) h = rotl(h ^ rnd(0, term_lane64(w, q, rc, i)), 27) * P1 + P4;
    if (i + 4 <= q) {
        uint32_t l = 0;
#pragma unroll
        for (int b = 3; b >= 0; --b) l = (l << 8) | term_byte(w, q, rc, i + (uint32_t)b);
        h = rotl(h ^ ((uint64_t)l * P1), 23) * P2 + P3;
        i += 4;
    }
    for (; i < q; ++i) h = rotl(h ^ ((uint64_t)term_byte(w, q, rc, i) * P5), 11) * P1;
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// Canonical orientation of an all-ACGT window: true iff revcomp < gram
// bytewise (termizer.cpp:117-118: rc is kept only when strictly smaller).
__device__ __forceinline__ bool choose_rc(const uint8_t* w, uint32_t q) {
    for (uint32_t i = 0; i < q; ++i) {
        uint32_t f = w[i], r = comp_byte(w[q - 1 - i]);
        if (r != f) return r < f;
    }
    return false;
}

// Window has only A/C/G/T bytes (termizer.cpp:28-30, 113).
__device__ __forceinline__ bool window_acgt(const uint8_t* w, uint32_t q) {
    for (uint32_t i = 0; i < q; ++i)
        if (!is_acgt(w[i])) return false;
    return true;
}

// Two windows emit the same term bytes.
__device__ __forceinline__ bool terms_equal(const uint8_t* a, bool rca, const uint8_t* b, bool rcb,
                                            uint32_t q) {
    for (uint32_t i = 0; i < q; ++i)
        if (term_byte(a, q, rca, i) != term_byte(b, q, rcb, i)) return false;
    return true;
}

// Lock-free exact set insert of window `pos` with hash h.  Slot words are
// (h >> 32) << 32 | (pos + 1); 0 is empty.  Equal 32-bit tags are resolved
// by comparing the window bytes, so distinct terms with colliding hashes
// each get their own slot and the count of winners is the exact number of
// distinct terms.  Returns true iff this window owns a new slot.
__device__ __forceinline__ bool set_insert(unsigned long long* tab, uint64_t mask, uint64_t h,
                                           uint32_t pos, const uint8_t* win_base, uint32_t q,
                                           bool canonical, bool rc) {
    unsigned long long key = ((unsigned long long)(h >> 32) << 32) | (unsigned long long)(pos + 1u);
    uint64_t slot = h & mask;
    const uint8_t* mine = win_base + pos;
    for (;;) {
        unsigned long long cur = *((volatile unsigned long long*)&tab[slot]);
        if (cur == 0ULL) {
            cur = atomicCAS(&tab[slot], 0ULL, key);
            if (cur == 0ULL) return true;
        }
        if ((cur >> 32) == (key >> 32)) {
            const uint8_t* other = win_base + ((uint32_t)cur - 1u);
            bool orc = canonical ? choose_rc(other, q) : false;
            if (terms_equal(mine, rc, other, orc, q)) return false;
        }
        slot = (slot + 1) & mask;
    }
}

} // namespace cobsg
