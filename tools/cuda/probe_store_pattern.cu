// Store-pattern probe for the row-major kernels (Grain v1 is store-pattern-bound):
// W persistent warps; a thread owns 32 instance rows of PITCH bytes and, once per "drain", writes RUN
// contiguous bytes to each of them (16-byte stores), advancing RUN bytes along the row -- the DRAM-side
// pattern of row_drain() with a staging tile of 8 * RUN clocks.  Reports the achieved store bandwidth for
// RUN = 32 / 64 / 128 and the evict_last L2 hint, with a dummy ALU delay between drains that matches the
// generation rate (so that lines are open for as long as in the real kernel).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_store tools/cuda/probe_store_pattern.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int RUN, bool KEEP>
__global__ void __launch_bounds__(256, 1)
store_kernel(unsigned char *out, unsigned long long pitch, unsigned nchains, unsigned row_bytes, int delay, unsigned *ticket)
{
    const unsigned lane = threadIdx.x & 31;
    for (;;) {
        unsigned chain = 0;
        if (lane == 0) chain = atomicAdd(ticket, 1u);
        chain = __shfl_sync(0xFFFFFFFFu, chain, 0);
        if (chain >= nchains) break;
        unsigned char *rows = out + ((unsigned long long)chain * 1024 + lane * 32) * pitch;
        unsigned x = chain * 2654435761u + lane;
        for (unsigned off = 0; off < row_bytes; off += RUN) {
            for (int d = 0; d < delay; ++d) x = x * 1664525u + 1013904223u;  // stands for the clocks of one tile
            for (int r = 0; r < 32; ++r) {
                unsigned char *p = rows + (unsigned long long)r * pitch + off;
#pragma unroll
                for (int q = 0; q < RUN / 16; ++q) {
                    const uint4 v = make_uint4(x, x ^ r, x + q, off);
                    if (KEEP) {
                        unsigned long long pol;
                        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p + 16 * q), "r"(v.x),
                                     "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                                     : "memory");
                    } else {
                        *reinterpret_cast<uint4 *>(p + 16 * q) = v;
                    }
                }
            }
        }
    }
}

template <int RUN, bool KEEP>
float run(unsigned char *out, unsigned long long pitch, unsigned nchains, unsigned row_bytes, int delay, unsigned *ticket, int warps)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(ticket, 0, 4);
        cudaEventRecord(e0);
        store_kernel<RUN, KEEP><<<148, 32 * warps>>>(out, pitch, nchains, row_bytes, delay, ticket);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char **argv)
{
    const unsigned nchains = 4096;            // 2^22 rows
    const unsigned row_bytes = 8192;          // 64 Kbit per instance
    const unsigned long long pitch = row_bytes;
    unsigned char *out;
    unsigned *ticket;
    cudaMalloc(&out, (size_t)nchains * 1024 * pitch);
    cudaMalloc(&ticket, 4);
    const double gb = (double)nchains * 1024 * row_bytes / 1e9;
    printf("rows 2^22 x %u B (%.1f GB), 148 CTAs; GB/s by contiguous run per row and drain, delay = dummy ALU work between drains\n", row_bytes, gb);
    for (int warps : {7, 8})
        for (int delay : {2000, 8000, 16000}) {
            printf("warps/SM %d delay %5d:", warps, delay);
            printf("  run32 %7.0f", gb / run<32, false>(out, pitch, nchains, row_bytes, delay, ticket, warps) * 1e3);
            printf("  run32+keep %7.0f", gb / run<32, true>(out, pitch, nchains, row_bytes, delay, ticket, warps) * 1e3);
            printf("  run48 %7.0f", gb * (8160.0 / 8192.0) / run<48, false>(out, pitch, nchains, 8160, delay * 3 / 2, ticket, warps) * 1e3);
            printf("  run48+keep %7.0f", gb * (8160.0 / 8192.0) / run<48, true>(out, pitch, nchains, 8160, delay * 3 / 2, ticket, warps) * 1e3);
            printf("  run64 %7.0f", gb / run<64, false>(out, pitch, nchains, row_bytes, delay * 2, ticket, warps) * 1e3);
            printf("  run64+keep %7.0f", gb / run<64, true>(out, pitch, nchains, row_bytes, delay * 2, ticket, warps) * 1e3);
            printf("  run128 %7.0f", gb / run<128, false>(out, pitch, nchains, row_bytes, delay * 4, ticket, warps) * 1e3);
            printf("  run128+keep %7.0f\n", gb / run<128, true>(out, pitch, nchains, row_bytes, delay * 4, ticket, warps) * 1e3);
        }
    return 0;
}
