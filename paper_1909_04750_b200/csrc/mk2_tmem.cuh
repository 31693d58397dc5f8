// mk2_tmem.cuh -- row-major keystream with the staging tile in TENSOR MEMORY.
//
// The row-major kernel parks 256 keystream words per thread (1 KiB) between two drains so
// that every instance row receives whole 32-byte sectors.  In shared memory that is 32 KiB
// per warp, and 227 KiB fit only seven worker warps per SM: one sub-partition is left with
// a lone warp and nobody to hide its drain behind.  The SM's 256 KiB of tensor memory are
// idle in this integer path (no MMA anywhere), and they are exactly eight such tiles:
// 128 lanes x 512 columns x 32 bit.  A warp may touch the 32 TMEM lanes of its quadrant
// (warp id % 4), so warp w owns lanes 32 (w % 4) .. +31, columns 256 (w / 4) .. +255:
// thread = lane, column = clock within the tile.  tcgen05.st / tcgen05.ld move registers
// to and from it (no tensor-core instruction is involved), 12 cycles of latency instead of
// shared memory's ~30, and shared memory is not used at all.
//
// Same bits as gen_rowmajor_kernel (kernels.py:604-621 layout) and the launch planner's default
// for MICKEY: +1.8% at 2^24 instances (profiles/r01b_probe_row_staging.txt).  Grain v1 stays on
// shared memory: at 40 LOP3 per clock it drains eight times as often, and the tile reads
// (64 B/clk of TMEM read bandwidth per SM against 128 B/clk of LDS) cost more than the eighth
// warp brings (measured 7.9 against 9.3 Tb/s).
#pragma once
#include "mk2_kernels.cuh"

namespace mk2 {
namespace tmem {

#ifndef MK2_RBLOCK_ROW_TMEM
#define MK2_RBLOCK_ROW_TMEM MK2_RBLOCK_ROW
#endif
constexpr int RBLOCK = MK2_RBLOCK_ROW_TMEM;  // clocks per clock_block in this kernel

// ---- allocation: one full warp allocates / frees, the address travels through shared memory
// (ncols: 256 for up to four worker warps, 512 = the SM's whole tensor memory for eight)
__device__ __forceinline__ void alloc(uint32_t *smem_slot, uint32_t ncols)
{
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem_slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---- register <-> TMEM, shape 32x32b: thread i of the warp <-> lane i of its quadrant, N consecutive columns
__device__ __forceinline__ void st1(uint32_t taddr, uint32_t v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ uint32_t ld1(uint32_t taddr)
{
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
    return v;
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// The loaded registers are threaded through the wait so that no consumer can be scheduled ahead of it.
__device__ __forceinline__ void wait_ld(uint32_t &v)
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v)::"memory");
}
template <int N>
__device__ __forceinline__ void wait_ld(uint32_t (&v)[N])
{
    static_assert(N == 8 || N == 16, "8 or 16 registers");
    if constexpr (N == 8)
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])::"memory");
    else
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                       "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])::"memory");
}

// Drain of one staging tile (ngrp 8-clock groups in the thread's TMEM lane, columns tcol ..) into the
// instance rows at `dst`: row_drain() of mk2_kernels.cuh with tensor memory in place of the smem column.
// Executed by all 32 threads of the warp (tcgen05 ld / st are warp-collective); `store` is false for
// threads whose group does not exist.
// LSB selects the byte packing: first bit in the MSB (library default, bitops.py:20-23) or in the LSB (Grain's
// published convention, grain.py:13-16).
template <bool ALIGNED16, bool LSB = false>
__device__ __forceinline__ void row_drain(uint32_t tcol, uint8_t *dst, uint64_t pitch, int ngrp, uint64_t nrows)
{
    // ---- pass 1: 8x32 bit transposes, in place
#pragma unroll 1
    for (int grp = 0; grp < ngrp; ++grp) {
        uint32_t v[8], z[8];
        ld8(tcol + 8 * grp, v);
        wait_ld(v);
#pragma unroll
        for (int m = 0; m < 8; ++m) z[LSB ? m : 7 - m] = v[m];  // clock m -> bit 7 - m (MSB-first) or m
        transpose8x32(z);                             // z[k]: byte q = output byte of instance 8 q + k
        st8(tcol + 8 * grp, z);
    }
    wait_st();
    // ---- pass 2: 32 bytes per instance row, as two back-to-back 16-byte stores
    if (ALIGNED16 && ngrp == 32 && __all_sync(0xFFFFFFFFu, nrows == 32)) {
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                uint32_t x[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = ld1(tcol + (16 * half + i) * 8 + kk);
                wait_ld(x);
                uint32_t y[4][4];  // [g4][q]
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) {
                    const uint32_t x4[4] = {x[4 * g4], x[4 * g4 + 1], x[4 * g4 + 2], x[4 * g4 + 3]};
                    bytes4x4(x4, y[g4]);
                }
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    store16<0>(dst + (uint64_t)(8 * qq + kk) * pitch + 16 * half,
                                              make_uint4(y[0][qq], y[1][qq], y[2][qq], y[3][qq]));
            }
        }
    } else {
        // ragged edge: short tail, partial last group or unaligned rows (nrows = 0: nothing is stored)
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll 1
            for (int grp = 0; grp < ngrp; ++grp) {
                uint32_t x = ld1(tcol + grp * 8 + kk);
                wait_ld(x);
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    if ((uint64_t)(8 * qq + kk) < nrows)
                        dst[(uint64_t)(8 * qq + kk) * pitch + grp] = (uint8_t)(x >> (8 * qq));
            }
    }
}

constexpr int TILE_CLOCKS = 256;

// Kernel prologue / epilogue: allocate the CTA's columns and return this warp's tile address
// (lane quadrant in bits 31:16, column half in bits 15:0); free them after every warp is done.
__device__ __forceinline__ uint32_t open_tile(uint32_t *smem_slot)
{
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) alloc(smem_slot, blockDim.x > 128 ? 512u : 256u);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    return *smem_slot + (((warp & 3u) * 32u) << 16) + (warp >> 2) * (uint32_t)TILE_CLOCKS;
}
__device__ __forceinline__ void close_tile(const uint32_t *smem_slot)
{
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if ((threadIdx.x >> 5) == 0) dealloc(*smem_slot, blockDim.x > 128 ? 512u : 256u);
}

template <bool ALIGNED16, bool LSB = false>
__global__ void __launch_bounds__(BLOCK, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                    unsigned long long *acc_out, uint8_t *__restrict__ out, uint64_t pitch, uint64_t N, uint64_t G,
                    uint64_t T, uint32_t chunk, uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots,
                    uint32_t mask, uint32_t *progress, uint32_t chain_base)
{
    __shared__ uint32_t tmem_base_slot;
    const uint32_t tcol = open_tile(&tmem_base_slot);

    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g_own = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);
        // tcgen05 ld / st are warp-collective: a thread whose group does not exist (last, partial chain)
        // runs along on the last real group and stores nothing
        const bool real = g_own < G;
        const uint64_t g = real ? g_own : G - 1;
        const uint64_t c0 = (uint64_t)k * chunk;  // chunk is a multiple of 256 clocks
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        {
            uint32_t r[NBITS], s[NBITS];
            unsigned long long a;
            load_state(state, acc, G, g, r, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
            const uint64_t nrows = !real ? 0 : (N - 32 * g < 32 ? N - 32 * g : 32);

#pragma unroll 1
            for (uint64_t t0 = 0; t0 < tc; t0 += TILE_CLOCKS) {
                const int nclk = (tc - t0) >= TILE_CLOCKS ? TILE_CLOCKS : (int)(tc - t0);
                const int ngrp = nclk >> 3;
                uint32_t tz = tcol;
                int t = 0;
                HalfSums hs;  // a tile is at most 256 words
                if constexpr (RBLOCK > 1) {
#pragma unroll 1
                    for (; t + RBLOCK <= nclk; t += RBLOCK) {
                        clock_block<RBLOCK, false, false, true>(r, s, NoInput{}, [&](auto kc, uint32_t z) {
                            st1(tz + decltype(kc)::value, z);
                            hs.add(z);
                        });
                        tz += RBLOCK;
                    }
                }
#pragma unroll 1
                for (; t < nclk; ++t) {
                    const uint32_t z = keystream_word(r, s);
                    st1(tz, z);
                    tz += 1;
                    hs.add(z);
                    clock<false, false>(r, s, 0u);
                }
                hs.fold(a);
                wait_st();
                row_drain<ALIGNED16, LSB>(tcol, rows + (t0 >> 3), pitch, ngrp, nrows);
            }
            if (real) store_state(state_out, acc_out, G, g, r, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }

    close_tile(&tmem_base_slot);
}

}  // namespace tmem
}  // namespace mk2
