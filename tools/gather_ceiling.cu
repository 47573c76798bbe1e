// Calibration microbenchmark (not product code): what HBM read bandwidth a
// B200 sustains for (a) a streaming read and (b) random 128-byte line reads
// with the gather kernel's access shape (one warp = one 128-byte line per
// load, 32 independent loads per warp in flight).  Used to put the gather
// kernel's roofline fraction in context.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gc tools/gather_ceiling.cu
//   /tmp/gc [GiB=64]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void stream_read(const uint4* p, uint64_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void random_lines(const uint8_t* p, uint64_t lines, uint64_t per_warp, uint32_t* out, uint64_t seed) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    uint64_t ctr = warp * per_warp;
    for (uint64_t it = 0; it < per_warp; it += U) {
        // lane u draws line u of this batch (like the gather kernel's one row per lane)
        const uint32_t mine = static_cast<uint32_t>(mix(seed ^ (ctr + it + (lane % U))) & (lines - 1));
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t line = __shfl_sync(0xffffffffu, mine, u);
            v[u] = __ldcs(reinterpret_cast<const uint32_t*>(p + (uint64_t)line * 128) + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// Same random 128-byte lines staged by the bulk-copy engine
// (cp.async.bulk, one elected lane per warp, mbarrier completion, two
// 32-line buffers per warp) and consumed from shared memory.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(phase)
                 : "memory");
}

__global__ void __launch_bounds__(256) random_lines_bulk(const uint8_t* p, uint64_t lines, uint64_t per_warp,
                                                         uint32_t* out, uint64_t seed) {
    extern __shared__ __align__(128) uint8_t dyn[];
    auto buf = reinterpret_cast<uint8_t(*)[2][32 * 128]>(dyn);
    auto bars = reinterpret_cast<uint64_t(*)[2]>(dyn + 8 * 2 * 32 * 128);
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) {
        mbar_init(&bars[w][0], 1);
        mbar_init(&bars[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint64_t ctr = warp * per_warp;
    auto issue = [&](uint64_t it, int b) {
        const uint32_t mine = static_cast<uint32_t>(mix(seed ^ (ctr + it * 32 + lane)) & (lines - 1));
        if (lane == 0) mbar_expect(&bars[w][b], 32 * 128);
        __syncwarp();
        // every lane issues its own line's bulk copy
        bulk_copy(&buf[w][b][lane * 128], p + (uint64_t)mine * 128, 128, &bars[w][b]);
    };
    const uint64_t iters = per_warp / 32;
    uint32_t acc = 0;
    issue(0, 0);
    for (uint64_t it = 0; it < iters; ++it) {
        const int b = it & 1;
        if (it + 1 < iters) issue(it + 1, b ^ 1);
        mbar_wait(&bars[w][b], (it >> 1) & 1);
#pragma unroll 8
        for (int u = 0; u < 32; ++u) acc ^= reinterpret_cast<const uint32_t*>(&buf[w][b][u * 128])[lane];
        __syncwarp();
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    double gib = argc > 1 ? atof(argv[1]) : 64.0;
    uint64_t bytes = (uint64_t)(gib * (1ull << 30));
    uint8_t* p;
    uint32_t* out;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        stream_read<<<148 * 8, 512>>>(reinterpret_cast<const uint4*>(p), bytes / 16, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    printf("{\"stream_read_gbs\": %.1f, ", bytes / (ms / 1e3) / 1e9);
    const uint64_t lines = bytes / 128;
    const int threads = 256;
    const uint64_t warps = 148ull * 64 * 8;
    const uint64_t per_warp = 2048;
    const int blocks = (int)(warps * 32 / threads);
    auto run = [&](auto kern, const char* name) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            kern<<<blocks, threads>>>(p, lines, per_warp, out, 1234 + rep);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("\"%s\": %.1f, ", name, warps * per_warp * 128.0 / (ms / 1e3) / 1e9);
    };
    run(random_lines<8>, "random128_u8_gbs");
    run(random_lines<16>, "random128_u16_gbs");
    run(random_lines<32>, "random128_u32_gbs");
    {
        const int smem = 8 * 2 * 32 * 128 + 8 * 2 * 8;
        cudaFuncSetAttribute(random_lines_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            random_lines_bulk<<<blocks, threads, smem>>>(p, lines, per_warp, out, 1234 + rep);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        cudaError_t e = cudaGetLastError();
        printf("\"random128_bulk_copy_gbs\": %.1f, \"bulk_err\": \"%s\", ", warps * per_warp * 128.0 / (ms / 1e3) / 1e9,
               cudaGetErrorString(e));
    }
    printf("\"gib\": %.1f}\n", gib);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("cuda error %s\n", cudaGetErrorString(e));
    return 0;
}
