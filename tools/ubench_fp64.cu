// FP64 throughput on this B200 (development aid; gives the fp64 roofline of the
// NEXT-row kernels): DFMA and fmin(double) per clock per SM, 8 independent chains
// per thread, full occupancy.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *out, int n, double a, double b)
{
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < n; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = OP == 0 ? fma(x[i], a, b) : fmin(x[i], b + i) + a;
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main()
{
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n = 4096, blocks = sms * 8, threads = 256;
    for (int op = 0; op < 2; op++) {
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(o, n, 0.999, 1e-3);
            else k<1><<<blocks, threads>>>(o, n, 1e-9, 0.5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double ops = (double)blocks * threads * n * 8;
        // op 1 counts one fmin + one add per element
        printf("%s: %.3f ms, %.2f T elem-ops/s, %.1f per clk per SM at %d MHz\n",
               op == 0 ? "DFMA" : "fmin(double)+DADD", best, ops / best / 1e9,
               ops / (best * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
