// Same-box roofline calibration for the bench (not on the query path): the
// HBM read bandwidth this GPU sustains for (a) a streaming read and (b)
// random 128-byte lines in kernel 2's access shape (one warp load = one
// line, 16 independent lines in flight per warp).  bench.py reports the
// gather kernel against (b) measured in the same process, next to the
// MEASURED_PEAKS.json copy peak the contract asks for.
#include <cstdint>

#include "dev.cuh"

namespace cobsg {

namespace {

__device__ __forceinline__ uint64_t cal_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void cal_stream_kernel(const uint4* p, uint64_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
}

constexpr int kCalLines = 16;

__global__ void cal_random_kernel(const uint8_t* p, uint64_t lines, uint64_t per_warp, uint64_t seed,
                                  uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    const uint64_t ctr = warp * per_warp;
    for (uint64_t it = 0; it < per_warp; it += kCalLines) {
        const uint32_t mine = static_cast<uint32_t>(cal_mix(seed ^ (ctr + it + (lane % kCalLines))) & (lines - 1));
        uint32_t v[kCalLines];
#pragma unroll
        for (int u = 0; u < kCalLines; ++u) {
            const uint32_t line = __shfl_sync(0xffffffffu, mine, u);
            v[u] = __ldcs(reinterpret_cast<const uint32_t*>(p + (uint64_t)line * 128) + lane);
        }
#pragma unroll
        for (int u = 0; u < kCalLines; ++u) acc ^= v[u];
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
}

} // namespace

// bytes is rounded down to a power of two >= 1 GiB
void calibrate(int device, uint64_t bytes, double* stream_gbs, double* random128_gbs) {
    COBS_CUDA(cudaSetDevice(device));
    uint64_t b = 1ull << 30;
    while (b * 2 <= bytes) b *= 2;
    uint8_t* p = nullptr;
    uint32_t* out = nullptr;
    COBS_CUDA(cudaMalloc(&p, b));
    COBS_CUDA(cudaMalloc(&out, 4));
    struct Free {
        void* a;
        void* b;
        ~Free() {
            cudaFree(a);
            cudaFree(b);
        }
    } guard{p, out};
    COBS_CUDA(cudaMemset(p, 1, b));
    Event e0, e1;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) { // last of three (the first warms up)
        COBS_CUDA(cudaEventRecord(e0, 0));
        cal_stream_kernel<<<148 * 8, 512>>>(reinterpret_cast<const uint4*>(p), b / 16, out);
        COBS_CUDA(cudaEventRecord(e1, 0));
        COBS_CUDA(cudaEventSynchronize(e1));
        COBS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    *stream_gbs = b / (ms / 1e3) / 1e9;
    const uint64_t warps = 148ull * 64 * 8, per_warp = 2048;
    for (int rep = 0; rep < 3; ++rep) {
        COBS_CUDA(cudaEventRecord(e0, 0));
        cal_random_kernel<<<static_cast<unsigned>(warps * 32 / 256), 256>>>(p, b / 128, per_warp, 1234 + rep, out);
        COBS_CUDA(cudaEventRecord(e1, 0));
        COBS_CUDA(cudaEventSynchronize(e1));
        COBS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    COBS_CUDA(cudaGetLastError());
    *random128_gbs = warps * per_warp * 128.0 / (ms / 1e3) / 1e9;
}

} // namespace cobsg
