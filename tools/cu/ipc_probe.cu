// Throughput of candidate epilogue instructions on sm_100a (8 independent chains per thread).
#include <cstdio>
#include <cstdint>
#define N_IT 4096
template <int OP>
__global__ void k(float* out, float a0, uint32_t ai) {
    float x[8]; uint32_t u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = a0 + threadIdx.x + i; u[i] = ai + threadIdx.x * 7 + i; }
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = fminf(x[i], x[(i + 1) & 7] + 0.0f);                 // FMNMX
            if (OP == 1) { float r; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x[i]), "f"(x[(i+1)&7]), "f"(x[(i+2)&7])); x[i] = r; }  // FMNMX3
            if (OP == 2) { uint32_t r; asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(u[i]), "r"(u[(i+1)&7]), "r"(u[(i+2)&7])); u[i] = r; }  // LOP3
            if (OP == 3) { uint32_t r; asm volatile("mul.hi.u32 %0, %1, 134217728;" : "=r"(r) : "r"(u[i])); u[i] = r + 3; }   // IMAD.HI (+IADD)
            if (OP == 4) x[i] = x[i] - x[(i + 3) & 7];                                   // FADD
            if (OP == 5) { uint32_t r; asm volatile("mad.lo.u32 %0, %1, 32, %2;" : "=r"(r) : "r"(u[i]), "r"(u[(i+1)&7])); u[i] = r; }   // IMAD/LEA
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i] + (float)u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> void run(const char* name, float* d) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int blocks = 148 * 4, threads = 512;
    k<OP><<<blocks, threads>>>(d, 1.0f, 3u);
    cudaEventRecord(a); k<OP><<<blocks, threads>>>(d, 1.0f, 3u); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = (double)blocks * threads / 32 * N_IT * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double per_smsp_clk = warp_instr / (148.0 * 4) / (ms * 1e-3 * clk * 1e3);
    printf("%-10s %8.3f ms  %.3f warp-instr/clk/SMSP (at %d MHz max)\n", name, ms, per_smsp_clk, clk / 1000);
}
int main() {
    float* d; cudaMalloc(&d, 148 * 4 * 512 * 4);
    run<0>("FMNMX", d); run<1>("FMNMX3", d); run<2>("LOP3", d); run<3>("IMAD.HI", d); run<4>("FADD", d); run<5>("IMAD", d);
    return 0;
}
