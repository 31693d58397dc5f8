// mk2_grain_row8.cuh -- Grain v1 row-major keystream with EIGHT worker warps per SM.
//
// Reference: pkg/src/slicerng/kernels.py:268-292 (Grain's compiled loop) + :600-621 (lane-major bytes).
//
// The default row-major kernel (grain::gen_rowmajor_kernel) keeps a 256-clock tile per thread in shared memory:
// 32 KiB per warp, seven warps in 227 KiB, so one sub-partition of every SM is left with a lone warp, which runs
// Grain at ~80% of what two warps sharing a sub-partition reach (profiles/r02_probe_grain_lone_warps.txt).  Here
// every thread keeps 28 of the tile's 32 eight-clock groups in shared memory (8 warps x 28 KiB = 224 KiB) and the
// last four in TENSOR memory (32 columns per warp, tcgen05.st / tcgen05.ld; no MMA anywhere): one code path, eight
// warps, and only an eighth of the tile traffic goes through tensor memory (the all-tensor-memory tile was measured
// in round 1 and lost to its read bandwidth).  As in the default kernel the 8 x 32 bit transposes run in registers
// on each group as it is produced, the drain is the byte-transposing second pass only, and the sector that
// completes a 128-byte line is written evict_first.
// Measured (B200, 2^22 instances x 65536 clocks; profiles/r02_probe_grain_lone_warps.txt, section 15): bit-exact and
// 10.6-10.8 Tb/s against 11.4 for the seven-warp default -- the eighth warp brings 155 MB of open 128-byte row lines
// instead of 136 MB, more than L2 holds, and the store pattern takes back more than the filled sub-partition gives.
// Opt-in: mk2_set_row_staging(ctx, 5).
// tcgen05 instructions are warp-collective, so only whole chains come here (N a multiple of 1024), with full
// tiles and 32-byte aligned rows; mk2_api.cu falls back to the default kernel otherwise.
#pragma once
#include "mk2_grain.cuh"
#include "mk2_tmem.cuh"

namespace mk2 {
namespace grain {
namespace row8 {

constexpr int THREADS = 256;
constexpr int SMEM_GROUPS = 28;                       // groups 0..27 of a tile: shared memory
constexpr int TMEM_GROUPS = 4;                        // groups 28..31: tensor memory, column = 8 * (group - 28) + k
constexpr uint32_t TS = THREADS;
constexpr int SMEM_BYTES = SMEM_GROUPS * 8 * THREADS * 4;  // 229 376
constexpr uint32_t TMEM_COLS = 64;                    // two warps per lane quadrant x 32 columns
static_assert(WIN == 16, "two groups per window");

template <bool LSB>
__global__ void __launch_bounds__(THREADS, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out, unsigned long long *acc_out,
                    uint8_t *__restrict__ out, uint64_t pitch, uint64_t G, uint64_t T, uint32_t chunk,
                    uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress,
                    uint32_t chain_base)
{
    extern __shared__ uint32_t tile[];  // [28 groups][8 k][256 threads]
    __shared__ uint32_t tmem_base_slot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem::alloc(&tmem_base_slot, TMEM_COLS);
    tmem::fence_before_sync();
    __syncthreads();
    tmem::fence_after_sync();
    const uint32_t tcol = tmem_base_slot + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 32u;

    uint32_t *col = tile + threadIdx.x;
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);  // exists: whole chains only
        const uint64_t c0 = (uint64_t)k * chunk;  // chunk and T are multiples of 256 clocks
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        {
            uint32_t b[GW], s[GW];
            unsigned long long a;
            load_state<OFF>(state, acc, G, g, b, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
#pragma unroll 1
            for (uint64_t t0 = 0; t0 < tc; t0 += 256) {
                uint32_t *zp = col;
                HalfSums hs;  // 256 words per tile
#pragma unroll 1
                for (int w = 0; w < 16; ++w) {
                    window_begin(b, s);
                    uint32_t zz[WIN];
                    static_for_up<0, WIN>([&](auto ic) {
                        constexpr int c = decltype(ic)::value;
                        zz[c] = step<c, false>(b, s);
                        hs.add(zz[c]);
                    });
                    uint32_t z0[8], z1[8];
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        z0[LSB ? m : 7 - m] = zz[m];  // clock m -> bit 7 - m (MSB-first) or m
                        z1[LSB ? m : 7 - m] = zz[8 + m];
                    }
                    transpose8x32(z0);  // z[k]: byte q = output byte of instance 8 q + k for this group
                    transpose8x32(z1);
                    if (w < SMEM_GROUPS / 2) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            zp[kk * TS] = z0[kk];
                            zp[(8 + kk) * TS] = z1[kk];
                        }
                        zp += WIN * TS;
                    } else {
                        const uint32_t tc0 = tcol + (uint32_t)(w - SMEM_GROUPS / 2) * 16u;
                        tmem::st8(tc0, z0);
                        tmem::st8(tc0 + 8u, z1);
                    }
                    window_end(b, s);
                }
                hs.fold(a);
                tmem::wait_st();
                // ---- drain: 32 bytes per instance row, one 256-bit store per row
                uint8_t *dst = rows + (t0 >> 3);
#pragma unroll 1
                for (int kk = 0; kk < 8; ++kk) {
                    uint32_t xt[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) xt[u] = tmem::ld1(tcol + (uint32_t)(8 * u + kk));
                    uint32_t y[8][4];  // [g4][q]
#pragma unroll
                    for (int g4 = 0; g4 < 7; ++g4) {
                        uint32_t x[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) x[u] = col[((4 * g4 + u) * 8 + kk) * TS];
                        bytes4x4(x, y[g4]);
                    }
                    // one wait for the four loads; the registers are threaded through it so that no consumer is
                    // scheduled ahead of it
                    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(xt[0]), "+r"(xt[1]), "+r"(xt[2]), "+r"(xt[3])::"memory");
                    bytes4x4(xt, y[7]);
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const uint32_t v[8] = {y[0][qq], y[1][qq], y[2][qq], y[3][qq], y[4][qq], y[5][qq], y[6][qq], y[7][qq]};
                        store32_line(dst + (uint64_t)(8 * qq + kk) * pitch, v);
                    }
                }
            }
            store_state<OFF>(state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }

    tmem::fence_before_sync();
    __syncthreads();
    tmem::fence_after_sync();
    if (warp == 0) tmem::dealloc(tmem_base_slot, TMEM_COLS);
}

}  // namespace row8
}  // namespace grain
}  // namespace mk2
