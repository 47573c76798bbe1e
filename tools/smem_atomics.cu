// Shared-memory operation throughput on random slots (calibration for the
// build's dedup / histogram kernels): ops per SM per cycle for
// ATOMS.CAS.64, ATOMS.CAS.32, ATOMS.ADD.32, LDS.64 + STS.64, and
// warp-synchronous claim (match.any + STS).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd(uint32_t& x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

template <int OP>
__global__ void __launch_bounds__(256) kern(int iters, unsigned long long* out) {
    __shared__ unsigned long long tab[4096];
    unsigned int* t32 = reinterpret_cast<unsigned int*>(tab);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
        const uint32_t s = rnd(x) & 4095;
        if (OP == 0) acc += atomicCAS(&tab[s], 0ull, (unsigned long long)x | 1ull);
        if (OP == 1) acc += atomicCAS(&t32[s], 0u, x | 1u);
        if (OP == 2) acc += atomicAdd(&t32[s], 1u);
        if (OP == 3) { unsigned long long v = tab[s]; acc += v; if (v == 0) tab[s] = x | 1ull; }
        if (OP == 4) { const unsigned peers = __match_any_sync(0xffffffffu, s); unsigned long long v = tab[s];
                       if (v == 0 && (threadIdx.x & 31) == __ffs(peers) - 1) tab[s] = x | 1ull; acc += v; }
        if (OP == 5) acc += tab[s];
        if ((i & 1023) == 1023) { __syncthreads(); for (int j = threadIdx.x; j < 4096; j += blockDim.x) tab[j] = 0; __syncthreads(); }
    }
    if (acc == 0x1234567) out[0] = acc;
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 8);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = 148 * 4, iters = 1 << 14;
    const char* names[] = {"cas64", "cas32", "add32", "lds_sts64", "match_sts64", "lds64"};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{");
    for (int op = 0; op < 6; ++op) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            switch (op) {
            case 0: kern<0><<<blocks, 256>>>(iters, out); break;
            case 1: kern<1><<<blocks, 256>>>(iters, out); break;
            case 2: kern<2><<<blocks, 256>>>(iters, out); break;
            case 3: kern<3><<<blocks, 256>>>(iters, out); break;
            case 4: kern<4><<<blocks, 256>>>(iters, out); break;
            case 5: kern<5><<<blocks, 256>>>(iters, out); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        const double ops = (double)blocks * 256 * iters;
        printf("\"%s_Gops\": %.1f, \"%s_per_sm_clk\": %.2f, ", names[op], ops / ms / 1e6, names[op],
               ops / (ms * 1e-3) / 148 / (clk_khz * 1e3));
    }
    printf("\"clock_khz\": %d}\n", clk_khz);
    return 0;
}
