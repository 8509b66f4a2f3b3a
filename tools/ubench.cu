// ubench.cu -- B12 microbenchmarks: sustained issue rate of the instructions the
// exhaustive (min,+) kernel is built from, per SM per clock, on the whole chip.
// Each thread runs 16 independent chains of the op in a loop; grid = SMs x 4
// blocks x 256 threads.  Rate = ops / (elapsed SM clocks x #SMs).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench tools/ubench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CH 16
#define ITERS 4096

template <int OP>
__global__ void __launch_bounds__(256) kern(float *out, const float *in, unsigned long long *clk)
{
    float a[CH], b[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) {
        a[i] = __ldcg(in + (threadIdx.x * 2 * CH + i) % 4096);
        b[i] = __ldcg(in + (threadIdx.x * 2 * CH + CH + i) % 4096);
    }
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < CH; i++) {
            if (OP == 0) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));              // FMNMX
            if (OP == 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));              // FADD
            if (OP == 2) asm volatile("fma.rn.f32 %0, %1, 0f3F800000, %0;" : "+f"(a[i]) : "f"(b[i]));  // FFMA imm
            if (OP == 3) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 1) % CH]));  // FFMA 3-reg
            if (OP == 4) {  // FMNMX + FADD pair (the kernel's inner loop)
                float m;
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m) : "f"(a[i]), "f"(b[i]));
                asm volatile("add.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(m));
            }
            if (OP == 5) {  // FMNMX + FFMA(imm 1.0) pair
                float m;
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m) : "f"(a[i]), "f"(b[i]));
                asm volatile("fma.rn.f32 %0, %1, 0f3F800000, %0;" : "+f"(b[i]) : "f"(m));
            }
            if (OP == 6 && (i & 1) == 0) {  // 2x FMNMX + FADD2 (packed accumulate)
                float m0, m1;
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m0) : "f"(a[i]), "f"(b[i]));
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m1) : "f"(a[i + 1]), "f"(b[i]));
                asm volatile("{.reg .b64 x, y; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %3}; add.rn.f32x2 x, x, y; mov.b64 {%0, %1}, x;}"
                             : "+f"(b[i]), "+f"(b[i + 1]) : "f"(m0), "f"(m1));
            }
            if (OP == 7 && (i & 1) == 0)  // FADD2 alone
                asm volatile("{.reg .b64 x, y; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %3}; add.rn.f32x2 x, x, y; mov.b64 {%0, %1}, x;}"
                             : "+f"(a[i]), "+f"(a[i + 1]) : "f"(b[i]), "f"(b[i + 1]));
            if (OP == 8) asm volatile("min.s32 %0, %0, %1;" : "+r"(*(int *)&a[i]) : "r"(*(int *)&b[i]));   // IMNMX
            if (OP == 9) asm volatile("min.f16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));  // HMNMX2
            if (OP == 12) asm volatile("min.u16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));  // VIMNMX.U16x2
            if (OP == 13) {   // alternate HMNMX2 / VIMNMX.U16x2: do they share a pipe?
                if (i & 1) asm volatile("min.u16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));
                else asm volatile("min.f16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));
            }
            if (OP == 14) asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 1) % CH]));  // FMNMX3
            if (OP == 15) {   // alternate HMNMX2 / HADD2 (ALU + FMA pipes)
                if (i & 1) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));
                else asm volatile("min.f16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));
            }
            if (OP == 16) asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]), "r"(*(unsigned *)&b[(i + 1) % CH]));  // VABSDIFF4.ACC
            if (OP == 17) asm volatile("dp4a.u32.u32 %0, %1, %2, %0;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]), "r"(*(unsigned *)&b[(i + 1) % CH]));  // IDP.4A
            if (OP == 18) {   // alternate VABSDIFF4 / HMNMX2: do they share a pipe?
                if (i & 1) asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]), "r"(*(unsigned *)&b[(i + 1) % CH]));
                else asm volatile("min.f16x2 %0, %0, %1;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]));
            }
            if (OP == 19) {   // alternate VABSDIFF4 / IMAD (FMA pipe)
                if (i & 1) asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]), "r"(*(unsigned *)&b[(i + 1) % CH]));
                else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(*(unsigned *)&a[i]) : "r"(*(unsigned *)&b[i]), "r"(*(unsigned *)&b[(i + 1) % CH]));
            }
            if (OP == 10) {  // |a-b| accumulate: FADD + FADD(|.|)
                float d;
                asm volatile("sub.f32 %0, %1, %2;" : "=f"(d) : "f"(a[i]), "f"(b[i]));
                asm volatile("{.reg .f32 t; abs.f32 t, %1; add.f32 %0, %0, t;}" : "+f"(a[(i + 1) % CH]) : "f"(d));
            }
            if (OP == 11 && (i & 1) == 0) {  // 2x FMNMX + FFMA2 (packed, imm 1.0)
                float m0, m1;
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m0) : "f"(a[i]), "f"(b[i]));
                asm volatile("min.f32 %0, %1, %2;" : "=f"(m1) : "f"(a[i + 1]), "f"(b[i]));
                asm volatile("{.reg .b64 x, y, o; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %3}; mov.b64 o, {0f3F800000, 0f3F800000}; fma.rn.f32x2 x, y, o, x; mov.b64 {%0, %1}, x;}"
                             : "+f"(b[i]), "+f"(b[i + 1]) : "f"(m0), "f"(m1));
            }
        }
    }
    unsigned long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < CH; i++) s += a[i] + b[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) atomicMax(clk, t1 - t0);
}

template <int OP>
void run(const char *name, double evals_per_op, int nsm)
{
    float *out, *in;
    unsigned long long *clk;
    const int blocks = nsm * 4;
    cudaMalloc(&out, sizeof(float) * blocks * 256);
    cudaMalloc(&in, sizeof(float) * 4096);
    cudaMemset(in, 0, sizeof(float) * 4096);
    cudaMalloc(&clk, sizeof(unsigned long long));
    kern<OP><<<blocks, 256>>>(out, in, clk);
    cudaMemset(clk, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<OP><<<blocks, 256>>>(out, in, clk);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double warp_instr = (double)blocks * 8 * ITERS * CH;   // per "op slot"
    const double lanes = warp_instr * 32 * evals_per_op;
    printf("%-28s %7.2f lane-ops/clk/SM  (%.3f ms, %.0f MHz effective)\n", name,
           lanes / ((double)c * nsm), ms, (double)c / (ms * 1e3));
    cudaFree(out);
    cudaFree(clk);
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs: %d\n", nsm);
    run<0>("FMNMX", 1, nsm);
    run<1>("FADD", 1, nsm);
    run<2>("FFMA imm", 1, nsm);
    run<3>("FFMA 3reg", 1, nsm);
    run<4>("FMNMX+FADD (evals)", 1, nsm);
    run<5>("FMNMX+FFMA-imm (evals)", 1, nsm);
    run<6>("2FMNMX+FADD2 (evals)", 1, nsm);
    run<11>("2FMNMX+FFMA2 (evals)", 1, nsm);
    run<7>("FADD2 (fp32 lanes)", 1, nsm);
    run<8>("IMNMX", 1, nsm);
    run<9>("HMNMX2 (f16x2 words)", 1, nsm);
    run<10>("sub+abs-add (evals)", 1, nsm);
    run<12>("VIMNMX.U16x2 (words)", 1, nsm);
    run<13>("HMNMX2|VIMNMX.U16x2 alt", 1, nsm);
    run<14>("FMNMX3", 1, nsm);
    run<15>("HMNMX2|HADD2 alt", 1, nsm);
    run<16>("VABSDIFF4.ACC (words)", 1, nsm);
    run<17>("IDP.4A (words)", 1, nsm);
    run<18>("VABSDIFF4|HMNMX2 alt", 1, nsm);
    run<19>("VABSDIFF4|IMAD alt", 1, nsm);
    return 0;
}
