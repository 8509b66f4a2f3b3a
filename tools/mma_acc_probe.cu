// mma_acc_probe.cu -- accumulation precision of mma.sync.m16n8k16 f16 -> f32 on
// this GPU (SASS HMMA.16816.F32), used to size the error window of the
// tensor-summed exhaustive kernel.
//
// With B a 0/1 selector (B[k][n] = 1 iff (k < 8) == (n even)) every output is
//     d = c + sum of 8 fp16 values (products by 1.0 are exact)
// and the probe compares d with the exact sum (fp64) over
//   (1) c = 2^j, all addends 1.0                      (big accumulator)
//   (2) c = 1.0, all addends 2^-j                     (where small addends vanish)
//   (3) random c in [0, 2^j), addends random fp16 in [0, 8) -- max error in ulp(d)
// and reports max |d - exact| / ulp(exact) and / exact.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mma_acc_probe tools/mma_acc_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

// one warp: in[32][4] A-fragment regs (f16x2), c_in[32][4], out[32][4]
__global__ void k_mma(const uint32_t *a_in, const float *c_in, float *out, int n_tiles)
{
    const int lane = threadIdx.x & 31, g = lane >> 2;
    const uint32_t one = 0x3C003C00u;
    const uint32_t b0 = (g & 1) ? 0u : one, b1 = (g & 1) ? one : 0u;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint32_t *a = a_in + (size_t)t * 128 + lane * 4;
        const float *c = c_in + (size_t)t * 128 + lane * 4;
        float d0 = c[0], d1 = c[1], d2 = c[2], d3 = c[3];
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
        float *o = out + (size_t)t * 128 + lane * 4;
        o[0] = d0;
        o[1] = d1;
        o[2] = d2;
        o[3] = d3;
    }
}

static float h2f(uint16_t h)
{
    __half_raw r;
    r.x = h;
    return __half2float(__half(r));
}
static uint16_t f2h(float f)
{
    __half_raw r = __half(__float2half_rn(f));
    return r.x;
}

// exact d for lane/reg: output reg j of lane (g, q): rows g / g+8, cols even/odd
static double exact(const uint32_t *A, const float *Cin, int t, int lane, int j)
{
    const int g = lane >> 2;
    const int row = (j < 2) ? g : g + 8;
    const bool odd = (j & 1);
    double s = Cin[(size_t)t * 128 + lane * 4 + j];
    // A[row][k]: lanes (g', q) hold reg0 = (g', k 2q..), reg1 = (g'+8, k 2q..), reg2 = (g', k 2q+8..), reg3 = (g'+8, ..)
    for (int q = 0; q < 4; q++) {
        const int ln = (row & 7) * 4 + q;
        const int reg = (row < 8 ? 0 : 1) + (odd ? 2 : 0);
        const uint32_t w = A[(size_t)t * 128 + ln * 4 + reg];
        s += h2f(w & 0xffff) + h2f(w >> 16);
    }
    return s;
}

static double ulp(double x)
{
    int e;
    frexp(x, &e);
    return ldexp(1.0, e - 24);
}

static void run(const char *name, int n_tiles, uint32_t *hA, float *hC)
{
    uint32_t *dA;
    float *dC, *dO;
    cudaMalloc(&dA, sizeof(uint32_t) * 128 * n_tiles);
    cudaMalloc(&dC, sizeof(float) * 128 * n_tiles);
    cudaMalloc(&dO, sizeof(float) * 128 * n_tiles);
    cudaMemcpy(dA, hA, sizeof(uint32_t) * 128 * n_tiles, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, hC, sizeof(float) * 128 * n_tiles, cudaMemcpyHostToDevice);
    k_mma<<<256, 32>>>(dA, dC, dO, n_tiles);
    float *hO = (float *)malloc(sizeof(float) * 128 * n_tiles);
    cudaMemcpy(hO, dO, sizeof(float) * 128 * n_tiles, cudaMemcpyDeviceToHost);
    double max_ulp = 0, max_rel = 0, max_rel_sum = 0;
    int n_over = 0, n_under = 0;
    for (int t = 0; t < n_tiles; t++)
        for (int lane = 0; lane < 32; lane++)
            for (int j = 0; j < 4; j++) {
                const double ex = exact(hA, hC, t, lane, j);
                const double d = hO[(size_t)t * 128 + lane * 4 + j];
                const double err = d - ex;
                if (err > 0) n_over++;
                if (err < 0) n_under++;
                if (ex > 0) {
                    max_ulp = fmax(max_ulp, fabs(err) / ulp(ex));
                    max_rel = fmax(max_rel, fabs(err) / ex);
                }
            }
    (void)max_rel_sum;
    printf("%-44s max_err=%.3f ulp  rel=%.3e (=2^%.2f)  above=%d below=%d\n", name, max_ulp, max_rel,
           max_rel > 0 ? log2(max_rel) : -999.0, n_over, n_under);
    free(hO);
    cudaFree(dA);
    cudaFree(dC);
    cudaFree(dO);
}

int main()
{
    const int NT = 4096;
    uint32_t *A = (uint32_t *)malloc(sizeof(uint32_t) * 128 * NT);
    float *C = (float *)malloc(sizeof(float) * 128 * NT);
    srand(12345);
    auto fill_A = [&](int t, float v) {
        const uint16_t h = f2h(v);
        for (int i = 0; i < 128; i++) A[(size_t)t * 128 + i] = (uint32_t)h | ((uint32_t)h << 16);
    };
    char name[128];
    // (1) big accumulator, addends 1.0
    for (int j = 0; j <= 24; j += 4) {
        for (int t = 0; t < 8; t++) {
            fill_A(t, 1.0f);
            for (int i = 0; i < 128; i++) C[t * 128 + i] = ldexpf(1.0f, j) + (float)(i % 7);
        }
        snprintf(name, sizeof name, "(1) c=2^%d(+i), 8 addends 1.0", j);
        run(name, 8, A, C);
    }
    // (2) c = 1, addends 2^-j
    for (int j = 4; j <= 28; j += 4) {
        for (int t = 0; t < 8; t++) {
            fill_A(t, ldexpf(1.0f, -j > -24 ? -j : -24));
            for (int i = 0; i < 128; i++) C[t * 128 + i] = 1.0f;
        }
        snprintf(name, sizeof name, "(2) c=1, 8 addends 2^-%d", j);
        run(name, 8, A, C);
    }
    // (3) random
    for (int j = 0; j <= 16; j += 4) {
        for (int t = 0; t < NT; t++)
            for (int i = 0; i < 128; i++) {
                const float a = (float)rand() / RAND_MAX * 8.0f, b = (float)rand() / RAND_MAX * 8.0f;
                A[(size_t)t * 128 + i] = (uint32_t)f2h(a) | ((uint32_t)f2h(b) << 16);
                C[(size_t)t * 128 + i] = (float)rand() / RAND_MAX * ldexpf(1.0f, j);
            }
        snprintf(name, sizeof name, "(3) random c<2^%d, addends [0,8)", j);
        run(name, NT, A, C);
    }
    // (4) random with wide addend exponents (incl. subnormal fp16)
    for (int t = 0; t < NT; t++)
        for (int i = 0; i < 128; i++) {
            const float a = ldexpf((float)rand() / RAND_MAX, -(rand() % 26));
            const float b = ldexpf((float)rand() / RAND_MAX, -(rand() % 26));
            A[(size_t)t * 128 + i] = (uint32_t)f2h(a) | ((uint32_t)f2h(b) << 16);
            C[(size_t)t * 128 + i] = ldexpf((float)rand() / RAND_MAX, (rand() % 12) - 6);
        }
    run("(4) random wide exponents", NT, A, C);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
