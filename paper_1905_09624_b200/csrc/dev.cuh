// Device-side building blocks shared by the query and build kernels.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "host.hpp"

namespace cobsg {

#define COBS_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::cobsg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

// RAII CUDA event (destroyed on every exit path).
// NVTX phase ranges (header-only NVTX3; free unless a profiler attaches):
// begin() closes the previous phase, the destructor the last one.
struct NvtxPhase {
    bool on = false;
    void begin(const char* name) {
        end();
        nvtxRangePushA(name);
        on = true;
    }
    void end() {
        if (on) nvtxRangePop();
        on = false;
    }
    ~NvtxPhase() { end(); }
};

struct Event {
    cudaEvent_t e = nullptr;
    explicit Event(unsigned flags = cudaEventDefault) {
        COBS_CUDA(cudaEventCreateWithFlags(&e, flags));
    }
    ~Event() {
        if (e) cudaEventDestroy(e);
    }
    Event(const Event&) = delete;
    Event& operator=(const Event&) = delete;
    operator cudaEvent_t() const { return e; }
};

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

// Tag bits of the byte-path dedup keys: all of them, unless the test-only
// COBS_DEBUG_TAG_BITS narrows them so distinct terms collide on the tag and
// the exact byte comparison decides (tests/test_gpu_edge.py).
inline uint32_t debug_tag_mask() {
    if (const char* e = std::getenv("COBS_DEBUG_TAG_BITS")) {
        int b = std::atoi(e);
        if (b >= 0 && b < 32) return (1u << b) - 1u;
    }
    return 0xffffffffu;
}

// ---- XXH64 (FORMAT.md "Term hashing"; reference xxhash64.hpp:45-95) ----

namespace xx {
constexpr uint64_t P1 = 0x9E3779B185EBCA87ULL, P2 = 0xC2B2AE3D27D4EB4FULL,
                   P3 = 0x165667B19E3779F9ULL, P4 = 0x85EBCA77C2B2AE63ULL,
                   P5 = 0x27D4EB2F165667C5ULL;
// 64-bit rotate left by 0 < r < 32 as two funnel shifts (SHF.L.W); the plain
// shift/or form was lowered to ~6 instructions.
__device__ __forceinline__ uint64_t rotl(uint64_t x, int r) {
    const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
    const uint32_t nhi = __funnelshift_l(lo, hi, r); // high word of (hi:lo) << r
    const uint32_t nlo = __funnelshift_l(hi, lo, r); // high word of (lo:hi) << r
    return (static_cast<uint64_t>(nhi) << 32) | nlo;
}
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
                                           bool canonical, bool rc, uint32_t tag_mask = 0xffffffffu) {
    // tag_mask < all-ones only in tests: forces tag collisions onto the byte compare
    unsigned long long key = ((unsigned long long)((h >> 32) & tag_mask) << 32) | (unsigned long long)(pos + 1u);
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

namespace cobsg {

// ---- DNA fast path: 2-bit codes ---------------------------------------
//
// For windows of only A/C/G/T bytes and q <= 32 the term is carried as a
// 2q-bit code (A=0 < C=1 < G=2 < T=3, first base most significant), so
//   * integer order of codes == bytewise order of the ASCII terms, which makes
//     the canonical min(gram, revcomp) (termizer.cpp:117-118) a 64-bit min;
//   * the code is an exact (injective) dedup key -- no byte compares;
//   * forward and reverse-complement codes roll in O(1) per window;
//   * the ASCII bytes XXH64 needs are rebuilt from the code in registers
//     (bases spread to nibbles, one PRMT per 4 bases).
// Windows with any other byte take the byte path above.

// 1 iff c is one of 'A','C','G','T': all four lie in 0x40..0x5f at bit
// positions 1, 3, 7 and 20 of the low 5 bits.
__device__ __forceinline__ uint32_t acgt_bit(uint32_t c) {
    return ((c & 0xe0u) == 0x40u) ? (0x10008au >> (c & 31u)) & 1u : 0u;
}
// 2-bit code of an A/C/G/T byte: ((c >> 1) ^ (c >> 2)) & 3 maps A,C,G,T to 0..3.
__device__ __forceinline__ uint32_t base_code(uint32_t c) { return ((c >> 1) ^ (c >> 2)) & 3u; }

// The term's bases in little-endian order: base j of a q-base code in bits
// 2j, 2j+1 (the code has base 0 most significant).
__device__ __forceinline__ uint64_t code_le(uint64_t code, uint32_t q) {
    uint64_t x = __brevll(code); // reverses the bases and the 2 bits within each
    x = ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
    return x >> (64 - 2 * q);
}
// ASCII of bases [i, i+8) / [i, i+4) / i of a little-endian code: each base's
// 2 bits are spread to a nibble (shift-or-mask steps), and PRMT selects
// "ACGT"[nibble] for 4 bytes at a time.
__device__ __forceinline__ uint64_t le_lane64(uint64_t le, uint32_t i) {
    uint32_t x = static_cast<uint32_t>(le >> (2 * i)) & 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u; // nibble k = base i + k
    return static_cast<uint64_t>(__byte_perm(0x54474341u, 0u, x)) |
           (static_cast<uint64_t>(__byte_perm(0x54474341u, 0u, x >> 16)) << 32);
}
__device__ __forceinline__ uint32_t le_word(uint64_t le, uint32_t i) {
    uint32_t x = static_cast<uint32_t>(le >> (2 * i)) & 0xffu;
    x = (x | (x << 4)) & 0x0f0fu;
    x = (x | (x << 2)) & 0x3333u;
    return __byte_perm(0x54474341u, 0u, x);
}
__device__ __forceinline__ uint32_t le_byte(uint64_t le, uint32_t i) {
    return __byte_perm(0x54474341u, 0u, static_cast<uint32_t>(le >> (2 * i)) & 3u) & 0xffu;
}

// XXH64 of the ASCII bytes of a q-base code, 1 <= q <= 32 (QC = q when known
// at compile time, else 0).  Same arithmetic as xxh64_term / xxhash64.hpp:45-95.
template <int QC>
__device__ __forceinline__ uint64_t xxh64_code(uint64_t code, uint32_t q_rt, uint64_t seed) {
    using namespace xx;
    const uint32_t q = QC ? QC : q_rt;
    const uint64_t le = code_le(code, q);
    uint32_t i = 0;
    uint64_t h;
    if (q == 32) { // one 32-byte stripe
        uint64_t v1 = rnd(seed + P1 + P2, le_lane64(le, 0));
        uint64_t v2 = rnd(seed + P2, le_lane64(le, 8));
        uint64_t v3 = rnd(seed, le_lane64(le, 16));
        uint64_t v4 = rnd(seed - P1, le_lane64(le, 24));
        h = rotl(v1, 1) + rotl(v2, 7) + rotl(v3, 12) + rotl(v4, 18);
        h = (h ^ rnd(0, v1)) * P1 + P4;
        h = (h ^ rnd(0, v2)) * P1 + P4;
        h = (h ^ rnd(0, v3)) * P1 + P4;
        h = (h ^ rnd(0, v4)) * P1 + P4;
        i = 32;
    } else {
        h = seed + P5;
    }
    h += q;
#pragma unroll
    for (int l = 0; l < 4; ++l)
        if (i + 8 <= q) {
            h = rotl(h ^ rnd(0, le_lane64(le, i)), 27) * P1 + P4;
            i += 8;
        }
    if (i + 4 <= q) {
        h = rotl(h ^ (static_cast<uint64_t>(le_word(le, i)) * P1), 23) * P2 + P3;
        i += 4;
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
        if (i < q) {
            h = rotl(h ^ (static_cast<uint64_t>(le_byte(le, i)) * P5), 11) * P1;
            ++i;
        }
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// XXH64 of an input shorter than 32 bytes (xxhash64.hpp:68-93) splits into
// a seed-independent part -- round(0, lane) of each 8-byte lane, word * P1
// of the 4-byte tail, byte * P5 of each last byte: 12 of the 19 multiplies
// at q = 31 -- and the accumulator chain that starts at seed + P5 + len.
// Several seeds of one term (k > 1) share the first part.
struct XxhShort {
    uint64_t k8[3], k4, k1[3];
};
template <int QC>
__device__ __forceinline__ XxhShort xxh_short_code(uint64_t code, uint32_t q_rt) { // 1 <= q < 32
    using namespace xx;
    const uint32_t q = QC ? QC : q_rt;
    const uint64_t le = code_le(code, q);
    XxhShort x{};
    uint32_t i = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l)
        if (i + 8 <= q) {
            x.k8[l] = rnd(0, le_lane64(le, i));
            i += 8;
        }
    if (i + 4 <= q) {
        x.k4 = static_cast<uint64_t>(le_word(le, i)) * P1;
        i += 4;
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
        if (i < q) {
            x.k1[b] = static_cast<uint64_t>(le_byte(le, i)) * P5;
            ++i;
        }
    return x;
}
__device__ __forceinline__ XxhShort xxh_short_term(const uint8_t* w, uint32_t q, bool rc) { // 1 <= q < 32
    using namespace xx;
    XxhShort x{};
    uint32_t i = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l)
        if (i + 8 <= q) {
            x.k8[l] = rnd(0, term_lane64(w, q, rc, i));
            i += 8;
        }
    if (i + 4 <= q) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 3; b >= 0; --b) v = (v << 8) | term_byte(w, q, rc, i + static_cast<uint32_t>(b));
        x.k4 = static_cast<uint64_t>(v) * P1;
        i += 4;
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
        if (i < q) {
            x.k1[b] = static_cast<uint64_t>(term_byte(w, q, rc, i)) * P5;
            ++i;
        }
    return x;
}
template <int QC>
__device__ __forceinline__ uint64_t xxh_short_seed(const XxhShort& x, uint32_t q_rt, uint64_t seed) {
    using namespace xx;
    const uint32_t q = QC ? QC : q_rt;
    uint64_t h = seed + P5 + q;
    uint32_t i = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l)
        if (i + 8 <= q) {
            h = rotl(h ^ x.k8[l], 27) * P1 + P4;
            i += 8;
        }
    if (i + 4 <= q) {
        h = rotl(h ^ x.k4, 23) * P2 + P3;
        i += 4;
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
        if (i < q) {
            h = rotl(h ^ x.k1[b], 11) * P1;
            ++i;
        }
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// Rolling 2-bit codes over a run of windows.  push() consumes one byte;
// after q pushes without a non-ACGT byte in the last q, fwd/rev hold the
// window's forward and reverse-complement codes.
struct Roller {
    uint64_t fwd = 0, rev = 0, mask;
    uint32_t q, since_bad; // bytes since the last non-ACGT byte
    __device__ explicit Roller(uint32_t q_) : mask(q_ >= 32 ? ~0ull : ((1ull << (2 * q_)) - 1)), q(q_), since_bad(0) {}
    __device__ __forceinline__ void push(uint32_t c) {
        uint32_t ok = acgt_bit(c);
        uint64_t code = base_code(c);
        fwd = ((fwd << 2) | code) & mask;
        rev = (rev >> 2) | ((3ull - code) << (2 * (q - 1)));
        since_bad = ok ? since_bad + 1 : 0;
    }
    __device__ __forceinline__ bool dna() const { return since_bad >= q; }
    // canonical term code: min(gram, revcomp) bytewise == min of the codes
    __device__ __forceinline__ uint64_t canon() const { return fwd < rev ? fwd : rev; }
};

// Rolling codes of windows over a small alphabet (<= 2^SB byte values, q*SB
// <= 62 bits): a window's code is its q symbols' SB-bit indices (table
// `tab`: byte -> index, 0xff = not in the alphabet), first symbol most
// significant.  An exact (injective) key for raw-byte windows, used only to
// count distinct windows; the row hashes still come from the bytes.
template <int SB>
struct SymRoller {
    uint64_t fwd = 0, mask;
    uint32_t q, since_bad = 0;
    const uint8_t* tab;
    __device__ SymRoller(uint32_t q_, const uint8_t* t)
        : mask(q_ * SB >= 64 ? ~0ull : ((1ull << (q_ * SB)) - 1)), q(q_), tab(t) {}
    __device__ __forceinline__ void push(uint32_t c) {
        const uint32_t sym = tab[c];
        fwd = ((fwd << SB) | (sym & ((1u << SB) - 1u))) & mask;
        since_bad = sym != 0xffu ? since_bad + 1 : 0;
    }
    __device__ __forceinline__ bool dna() const { return since_bad >= q; } // (a complete window)
    __device__ __forceinline__ uint64_t canon() const { return fwd; }
};

// Slot hash for code-keyed sets where the XXH64 row hash is not needed
// (the splitmix64 finaliser: two multiplies).
__device__ __forceinline__ uint64_t mix_code(uint64_t z) {
    z ^= z >> 31;
    z *= 0x7FB5D329728EA185ULL;
    z ^= z >> 27;
    z *= 0x81DADEF4BC2DD44DULL;
    return z ^ (z >> 33);
}

// 2-bit codes are exact, collision-free set keys (code + 1, 0 = empty) iff
// q < 32, or q = 32 with canonicalisation (min(fwd, revcomp) is never
// 2^64-1, and canonical mode skips every byte-path window, so no tagged key
// shares the table).  Non-canonical q = 32 windows take the byte path.
__host__ __device__ __forceinline__ bool codes_exact(uint32_t q, bool canonical) {
    return q < 32 || (q == 32 && canonical);
}

// Exact set insert keyed by the 2-bit code (+1 keeps 0 empty; see
// codes_exact for when this is collision-free).  When q < 32 the code has
// bit 63 clear, and byte-path keys sharing a table (set_insert_tagged)
// always have bit 63 set, so the key spaces never collide.
__device__ __forceinline__ bool set_insert_code(unsigned long long* tab, uint64_t mask, uint64_t h,
                                                uint64_t code) {
    const unsigned long long key = static_cast<unsigned long long>(code) + 1ull;
    uint64_t slot = h & mask;
    for (;;) {
        unsigned long long cur = *((volatile unsigned long long*)&tab[slot]);
        if (cur == 0ull) {
            cur = atomicCAS(&tab[slot], 0ull, key);
            if (cur == 0ull) return true;
        }
        if (cur == key) return false;
        slot = (slot + 1) & mask;
    }
}

// Byte-path insert for tables shared with code keys: key bit 63 set, 31-bit
// hash tag, 32-bit position+1; equal tags are resolved by the window bytes.
__device__ __forceinline__ bool set_insert_tagged(unsigned long long* tab, uint64_t mask, uint64_t h,
                                                  uint32_t pos, const uint8_t* win_base, uint32_t q,
                                                  uint32_t tag_mask = 0xffffffffu) {
    const unsigned long long key = (1ull << 63) |
                                   ((unsigned long long)((h >> 33) & 0x7fffffffu & tag_mask) << 32) |
                                   (unsigned long long)(pos + 1u);
    uint64_t slot = h & mask;
    const uint8_t* mine = win_base + pos;
    for (;;) {
        unsigned long long cur = *((volatile unsigned long long*)&tab[slot]);
        if (cur == 0ull) {
            cur = atomicCAS(&tab[slot], 0ull, key);
            if (cur == 0ull) return true;
        }
        if ((cur >> 32) == (key >> 32)) {
            const uint8_t* other = win_base + ((uint32_t)cur - 1u);
            if (terms_equal(mine, false, other, false, q)) return false;
        }
        slot = (slot + 1) & mask;
    }
}

} // namespace cobsg
