// probe_issue_mix.cu -- does an FMA-pipe instruction (IMAD) issued between LOP3s cost ALU-pipe throughput?
// W warps per SM (one CTA per SM), each thread runs ITER iterations of a body with NL LOP3 and NI IMAD on
// independent accumulators.  Prints cycles per body per sub-partition for several mixes; if the pipes overlap,
// adding IMADs up to one per LOP3 leaves the time at 2 cycles per LOP3.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_issue_mix tools/cuda/probe_issue_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__constant__ uint32_t c_one = 1u;
template <int NL, int NI>
__global__ void __launch_bounds__(256, 1) mix(uint32_t *out, int iters, uint32_t seed)
{
    uint32_t a[16], m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { a[i] = seed * (threadIdx.x + i + 1); m[i] = seed ^ (i * 77u + threadIdx.x); }
    const uint32_t one = c_one;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {   // 16 rounds; per round NL/16 LOP3 and NI/16 IMAD
#pragma unroll
            for (int j = 0; j < NL / 16; ++j) {
                const int k = (r * (NL / 16) + j) % 16;
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(a[(k + 5) % 16]), "r"(a[(k + 11) % 16]));
            }
#pragma unroll
            for (int j = 0; j < NI / 16; ++j) {
                const int k = (r * (NI / 16) + j) % 16;
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(m[k]) : "r"(one), "r"(m[(k + 3) % 16]));
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= a[i] ^ m[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
template <int NL, int NI>
void run(int warps, uint32_t *out, int sms, double ghz)
{
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    mix<NL, NI><<<sms, 32 * warps>>>(out, 100, 3);
    cudaEventRecord(e0);
    mix<NL, NI><<<sms, 32 * warps>>>(out, iters, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * ghz * 1e9 / iters;             // cycles per body (all warps of a sub-partition in parallel)
    const double per_smsp = cyc / ((warps + 3) / 4);               // per warp-body on one sub-partition
    printf("warps/SM %d  LOP3 %3d  IMAD %3d : %.1f cycles per body per warp slot  (%.2f per LOP3)\n", warps, NL, NI, per_smsp, per_smsp / NL);
}
int main()
{
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz / 1e6;
    uint32_t *out; cudaMalloc(&out, 256 * 256 * 4);
    for (int w : {4, 8}) {
        run<256, 0>(w, out, p.multiProcessorCount, ghz);
        run<256, 64>(w, out, p.multiProcessorCount, ghz);
        run<256, 128>(w, out, p.multiProcessorCount, ghz);
        run<256, 256>(w, out, p.multiProcessorCount, ghz);
        run<128, 256>(w, out, p.multiProcessorCount, ghz);
    }
    return 0;
}
