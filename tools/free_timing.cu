// How long do cudaMalloc / cudaFree of the count pass's key buffers take, and
// what avoids the slow frees seen in the build (profiles/r2/count_fp:
// 16-19 ms usually, 100-600 ms on some builds)?  Variants, 8 rounds each:
//   plain   : cudaMalloc 2 x G GiB, write them, cudaFree both, then cudaMalloc + free F GiB (the fill's matrix)
//   pool    : the same through cudaMallocAsync / cudaFreeAsync on a pool that keeps its memory
//   pooltrim: pool, trimmed to 0 after every round
//   chunks  : the G GiB as 1 GiB cudaMalloc pieces
// nvcc -O2 -arch=sm_100a -o free_timing tools/free_timing.cu
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

__global__ void touch(unsigned long long* p, size_t n, unsigned long long v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v + i;
}

int main(int argc, char** argv) {
    const size_t G = (argc > 1 ? std::atoll(argv[1]) : 40) << 30; // each key buffer
    const size_t F = (argc > 2 ? std::atoll(argv[2]) : 35) << 30; // the later allocation
    const size_t R = (argc > 3 ? std::atoll(argv[3]) : 70) << 30; // resident corpus stand-in
    const int rounds = 8;
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    void* resident = nullptr;
    CK(cudaMalloc(&resident, R));
    touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)resident, R / 8, 1);
    CK(cudaStreamSynchronize(st));

    std::printf("== plain (2 x %zu GiB, then %zu GiB)\n", G >> 30, F >> 30);
    for (int r = 0; r < rounds; ++r) {
        void *a, *b, *f;
        double t0 = now_ms();
        CK(cudaMalloc(&a, G));
        CK(cudaMalloc(&b, G));
        double t1 = now_ms();
        touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)a, G / 8, r);
        touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)b, G / 8, r);
        CK(cudaStreamSynchronize(st));
        double t2 = now_ms();
        CK(cudaFree(a));
        double t3 = now_ms();
        CK(cudaFree(b));
        double t4 = now_ms();
        CK(cudaMalloc(&f, F));
        double t5 = now_ms();
        touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)f, F / 8, r);
        CK(cudaStreamSynchronize(st));
        double t6 = now_ms();
        CK(cudaFree(f));
        double t7 = now_ms();
        std::printf("round %d: malloc %.1f  touch %.1f  freeA %.1f  freeB %.1f  mallocF %.1f  touchF %.1f  freeF %.1f ms\n", r,
                    t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6);
    }

    for (int trim = 0; trim < 2; ++trim) {
        std::printf("== pool%s\n", trim ? " trimmed every round" : " (memory kept)");
        cudaMemPool_t pool;
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = 0;
        CK(cudaMemPoolCreate(&pool, &props));
        unsigned long long thr = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        for (int r = 0; r < rounds; ++r) {
            void *a, *b, *f;
            double t0 = now_ms();
            CK(cudaMallocFromPoolAsync(&a, G, pool, st));
            CK(cudaMallocFromPoolAsync(&b, G, pool, st));
            CK(cudaStreamSynchronize(st));
            double t1 = now_ms();
            touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)a, G / 8, r);
            touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)b, G / 8, r);
            CK(cudaStreamSynchronize(st));
            double t2 = now_ms();
            CK(cudaFreeAsync(a, st));
            CK(cudaFreeAsync(b, st));
            CK(cudaStreamSynchronize(st));
            double t4 = now_ms();
            CK(cudaMallocFromPoolAsync(&f, F, pool, st));
            CK(cudaStreamSynchronize(st));
            double t5 = now_ms();
            touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)f, F / 8, r);
            CK(cudaStreamSynchronize(st));
            double t6 = now_ms();
            CK(cudaFreeAsync(f, st));
            CK(cudaStreamSynchronize(st));
            double t7 = now_ms();
            double t8 = t7;
            if (trim) {
                CK(cudaMemPoolTrimTo(pool, 0));
                t8 = now_ms();
            }
            std::printf("round %d: malloc %.1f  touch %.1f  free %.1f  mallocF %.1f  touchF %.1f  freeF %.1f  trim %.1f ms\n", r,
                        t1 - t0, t2 - t1, t4 - t2, t5 - t4, t6 - t5, t7 - t6, t8 - t7);
        }
        double t0 = now_ms();
        CK(cudaMemPoolDestroy(pool));
        std::printf("pool destroy %.1f ms\n", now_ms() - t0);
    }

    std::printf("== chunks of 1 GiB\n");
    for (int r = 0; r < rounds; ++r) {
        std::vector<void*> v(2 * (G >> 30));
        double t0 = now_ms();
        for (auto& p : v) CK(cudaMalloc(&p, 1ull << 30));
        double t1 = now_ms();
        for (auto& p : v) touch<<<148 * 8, 256, 0, st>>>((unsigned long long*)p, (1ull << 30) / 8, r);
        CK(cudaStreamSynchronize(st));
        double t2 = now_ms();
        double worst = 0;
        for (auto& p : v) {
            double a = now_ms();
            CK(cudaFree(p));
            worst = std::max(worst, now_ms() - a);
        }
        double t3 = now_ms();
        std::printf("round %d: malloc %.1f  touch %.1f  free %.1f (worst piece %.1f) ms\n", r, t1 - t0, t2 - t1, t3 - t2, worst);
    }
    CK(cudaFree(resident));
    return 0;
}
