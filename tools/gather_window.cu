// Calibration microbenchmark (not product code): do random 128-byte line
// reads get faster when the lines in flight across the GPU are confined to a
// window that moves through the buffer over time (DRAM page locality), as
// opposed to uniformly random lines over the whole buffer?
//
// Each warp issues U independent random line loads per step (one warp load =
// one 128-byte line, like gather_kernel); the line is drawn uniformly from
// [base, base + window) where base advances with %globaltimer (one window
// width per `period` ns), wrapping over the buffer.  window = buffer size is
// the plain random case.  Run under ncu to check dram__bytes_read ~= bytes
// requested (no L2 reuse).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_window tools/gather_window.cu
//   tools/gather_window
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int U>
__global__ void window_lines(const uint8_t* p, uint64_t lines, uint64_t win_lines, uint32_t period_shift,
                             uint64_t per_warp, uint64_t t0, uint32_t* out, uint64_t seed) {
    // lines and win_lines are powers of two: masks, no divisions
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    for (uint64_t it = 0; it < per_warp; it += U) {
        // window base from the global clock: all warps share it
        const uint64_t now = __shfl_sync(0xffffffffu, gtimer(), 0);
        const uint64_t base = win_lines >= lines ? 0 : (((now - t0) >> period_shift) * (win_lines / 2)) & (lines - 1);
        const uint64_t r = mix(seed ^ (warp * per_warp + it + (lane % U)));
        const uint64_t mine = (base + (r & (win_lines - 1))) & (lines - 1);
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t line = __shfl_sync(0xffffffffu, mine, u);
            v[u] = __ldcs(reinterpret_cast<const uint32_t*>(p + line * 128) + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    const double gib = 16.0; // a power of two of lines (masks)
    (void)argc; (void)argv;
    const uint64_t bytes = (uint64_t)(gib * (1ull << 30));
    uint8_t* p;
    uint32_t* out;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMalloc(&out, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t lines = bytes / 128;
    const int threads = 256;
    const uint64_t warps = 148ull * 64 * 8;
    const uint64_t per_warp = 4096;
    const int blocks = (int)(warps * 32 / threads);
    const double req_gb = warps * per_warp * 128.0 / 1e9;
    printf("{\"gib\": %.1f, \"requested_GB\": %.2f, \"rows\": [", gib, req_gb);
    const uint64_t wins_mb[] = {32, 128, 256, 1024, 4096, 0};
    const uint32_t periods_log2ns[] = {11, 13, 15}; // ~2, 8, 33 us per half-window step
    bool first = true;
    for (uint64_t wmb : wins_mb) {
        const uint64_t wl = wmb ? (wmb << 20) / 128 : lines;
        for (uint32_t per : periods_log2ns) {
            if (!wmb && per != periods_log2ns[0]) continue;
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                uint64_t t0 = 0;
                cudaEventRecord(a);
                window_lines<16><<<blocks, threads>>>(p, lines, wl, per, per_warp, t0, out, 99 + rep);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
            }
            printf("%s{\"window_MB\": %llu, \"period_us\": %.1f, \"gbs\": %.1f}", first ? "" : ", ",
                   (unsigned long long)(wmb ? wmb : bytes >> 20), (1u << per) / 1000.0,
                   req_gb / (ms / 1e3));
            first = false;
        }
    }
    printf("]}\n");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("cuda error %s\n", cudaGetErrorString(e));
    return 0;
}
