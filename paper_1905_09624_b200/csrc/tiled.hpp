// L2-tiled row gather (kernel 2, large batches): the batch's rows of each
// block are visited range by range so every row is fetched from HBM about
// once per wave of queries and re-read from L2 by the wave's other terms.
// Same counts, scores and hits as gather_kernel (query.cu), which is the
// reference's score_range loop (query.cpp:49-89).
#pragma once

#include <cstdint>
#include <vector>

#include "index.hpp"

namespace cobsg {

struct TiledPlan {
    bool use = false;
    int nt = 0;            // bit planes (10 or 12)
    int warps = 16;        // warps per CTA of the tile kernel
    uint32_t qs = 0;       // queries per CTA (per SM) in a wave
    uint32_t grid = 0;     // CTAs (one per SM)
    uint32_t lag = 2;      // a warp may start phase g once every warp finished g - lag
    uint32_t base_shift = 18;
    std::vector<uint64_t> wave_q0; // first query of each wave (+ n at the end)
    uint64_t slots = 0;    // window slots of the largest wave (list stride per block)
    std::vector<uint8_t> shift; // per block: rows per range = 2^shift (<= 64 ranges)
    uint32_t phases = 0;   // sum over column tasks of the block's range count
    const char* why = "";  // reason when not used
};

// Decide whether (and how) a batch runs through the tiled gather.  win_base:
// host window prefix of the batch (n + 1 entries).
TiledPlan tiled_plan(DeviceIndex& ix, const std::vector<uint64_t>& win_base, uint64_t n, int nt_needed,
                     bool prune);

struct TiledIO {
    const uint64_t* hashes;   // seed-major term hashes (k = 1)
    const uint64_t* win_base; // per query window prefix (device)
    const uint32_t* ell;
    const uint32_t* tau;
    uint64_t D;
    void* scores; // dense [n][D] or null
    int want_hits;
    uint32_t* hit_count;
    unsigned long long* hit_total;
    uint64_t hit_cap;
    uint32_t* hit_q;
    uint32_t* hit_doc;
    uint32_t* hit_score;
};

// Runs every wave (bucket kernel + tile kernel) on `st`; returns the number
// of kernel launches.
uint32_t tiled_gather(DeviceIndex& ix, const TiledPlan& tp, cudaStream_t st, const TiledIO& io);

} // namespace cobsg
