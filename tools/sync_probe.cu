// Latency probe (development aid): cooperative launch, grid.sync, a hand-rolled
// counter barrier over G CTAs, and small D2H copies (pageable vs pinned).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
#include <chrono>
namespace cg = cooperative_groups;
__global__ void k_gsync(int n, int *dummy) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; i++) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) dummy[0] = n;
}
__global__ void k_ctrbar(int n, unsigned *ctr) {
    // one arrival per CTA per step, spin until all arrived
    for (int i = 0; i < n; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            const unsigned target = (unsigned)(i + 1) * gridDim.x;
            while (true) {
                unsigned v;
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr));
                if (v >= target) break;
            }
        }
        __syncthreads();
    }
}
__global__ void k_empty() {}
int main() {
    int *d; unsigned *ctr; cudaMalloc(&d, 4); cudaMalloc(&ctr, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int G : {148, 74, 37, 16}) {
        for (int n : {1, 25}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; rep++) {
                void *args[] = {&n, &d};
                cudaEventRecord(a, s);
                cudaLaunchCooperativeKernel((void *)k_gsync, G, 256, args, 0, s);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
            }
            printf("grid.sync G=%3d n=%2d: %.2f us\n", G, n, best * 1e3);
            best = 1e9;
            for (int rep = 0; rep < 5; rep++) {
                cudaMemsetAsync(ctr, 0, 4, s);
                cudaEventRecord(a, s);
                k_ctrbar<<<G, 256, 0, s>>>(n, ctr);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
            }
            printf("ctrbar    G=%3d n=%2d: %.2f us\n", G, n, best * 1e3);
        }
    }
    // D2H small copies + sync, wall clock
    char *h_page = (char *)malloc(4096), *h_pin; cudaMallocHost(&h_pin, 4096);
    char *dbuf; cudaMalloc(&dbuf, 4096);
    for (int mode = 0; mode < 4; mode++) {
        double best = 1e9;
        for (int rep = 0; rep < 20; rep++) {
            auto t0 = std::chrono::high_resolution_clock::now();
            if (mode == 0) { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }
            if (mode == 1) { cudaMemcpyAsync(h_page, dbuf, 256, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
            if (mode == 2) { cudaMemcpyAsync(h_pin, dbuf, 256, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
            if (mode == 3) { for (int i = 0; i < 3; i++) cudaMemcpyAsync(h_page + 64 * i, dbuf, 64, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
            auto t1 = std::chrono::high_resolution_clock::now();
            best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        const char *nm[] = {"empty kernel + sync", "D2H 256B pageable + sync", "D2H 256B pinned + sync", "3x D2H pageable + sync"};
        printf("%s: %.1f us\n", nm[mode], best);
    }
    // cooperative launch overhead alone (n=0)
    {
        int n = 0; void *args[] = {&n, &d};
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(a, s);
            cudaLaunchCooperativeKernel((void *)k_gsync, 148, 256, args, 0, s);
            cudaEventRecord(b, s); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
        }
        printf("coop launch n=0: %.2f us\n", best * 1e3);
    }
    return 0;
}
