// probe_grain_lockstep.cu -- is the 80-clock circular-buffer body of Grain v1 (no realignment moves, ~56 KB of
// code) instruction-fetch bound because the warps of an SM run it at different phases?  Static chains (one per
// warp, no scheduler), column-major stores, three variants on identical work:
//   0  sliding window (16-clock body + 160 moves)   1  circular buffer, warps free-running
//   2  circular buffer, the CTA's warps held in lockstep with a barrier per 16-clock segment
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_1909_04750_b200/csrc -I include ...
#include <cstdio>
#include "mk2_grain.cuh"
using namespace mk2;
using namespace mk2::grain;

template <int MODE>
__global__ void __launch_bounds__(256, 1) run(uint32_t *out, uint64_t stride, uint32_t T, uint32_t seed)
{
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t *p = out + g;
    uint32_t x = 0;
    if constexpr (MODE == 0) {
        uint32_t b[GW], s[GW];
#pragma unroll
        for (int i = 0; i < GW; ++i) { b[i] = seed * (g + i + 1); s[i] = (seed + i) ^ (g * 2654435761u); }
#pragma unroll 1
        for (uint32_t t = 0; t < T; t += WIN) {
            grain::static_for_up<0, WIN>([&](auto ic) {
                const uint32_t z = step<decltype(ic)::value, false>(b, s);
                *p = z; p += stride; x += z;
            });
            realign<WIN>(b, s);
        }
    } else {
        uint32_t b[GB], s[GB];
#pragma unroll
        for (int i = 0; i < GB; ++i) { b[i] = seed * (g + i + 1); s[i] = (seed + i) ^ (g * 2654435761u); }
        auto seg = [&](auto pc) {
            grain::static_for_up<0, WIN>([&](auto ic) {
                const uint32_t z = step<decltype(pc)::value + decltype(ic)::value, false, GB, true>(b, s);
                *p = z; p += stride; x += z;
            });
            if constexpr (MODE == 2) __syncthreads();
        };
#pragma unroll 1
        for (uint32_t t = 0; t < T; t += 5 * WIN) {
            seg(std::integral_constant<int, 0>{});
            seg(std::integral_constant<int, 16>{});
            seg(std::integral_constant<int, 32>{});
            seg(std::integral_constant<int, 48>{});
            seg(std::integral_constant<int, 64>{});
        }
    }
    if (x == 0x12345678u) out[0] = x;
}

int main()
{
    cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    const uint32_t T = 5 * 16 * 100;  // 8000 clocks
    for (int warps : {8, 4}) {
        const uint64_t G = (uint64_t)sms * warps * 32;
        uint32_t *out; cudaMalloc(&out, G * T * 4);
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                if (mode == 0) run<0><<<sms, 32 * warps>>>(out, G, T, 7);
                if (mode == 1) run<1><<<sms, 32 * warps>>>(out, G, T, 7);
                if (mode == 2) run<2><<<sms, 32 * warps>>>(out, G, T, 7);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep && ms < best) best = ms;
            }
            printf("warps/SM %d mode %d: %.3f ms  %.2f Tb/s\n", warps, mode, best, G * 32.0 * T / best / 1e9);
        }
        cudaFree(out);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
