// mk2_grain_row64.cuh -- Grain v1 row-major keystream with 64 contiguous bytes per instance row and drain.
//
// Why: the row-major store pattern, not the ALU pipe, bounds Grain (38 LOP3 per clock).  With 256-clock
// staging tiles every drain writes one isolated 32-byte sector per instance row, 8 KB apart, and seven
// warps per SM keep 136 MB of 128-byte lines open -- more than L2 holds -- so the sectors reach DRAM one by
// one at 1.2-1.3 TB/s (10.4 Tb/s of keystream).  tools/cuda/probe_store_pattern.cu reproduces the pattern
// without the cipher (profiles/r02_probe_store_pattern.txt): 32-byte runs 1.16-1.24 TB/s at seven warps
// per SM, 64-byte runs 2.0 TB/s, which is above what the cipher's LOP3s can produce (1.73 TB/s).
//
// A 64-byte run per row needs a 512-clock tile = 2 KiB per thread, 64 KiB per warp: shared memory (227 KiB)
// holds three such tiles, the SM's tensor memory (128 lanes x 512 columns x 32 bit, idle in this integer
// path) exactly four.  So the CTA is eight worker warps, two per SM sub-partition: warps 0-3 park their tile
// in tensor memory (lane quadrant w, all 512 columns), warps 4-6 in shared memory, and warp 7 gets the 32 KiB
// of shared memory that are left: a 256-clock tile, 32 bytes per row and drain (an eighth of the traffic).
// Same persistent chain / chunk scheduler, state parking and checksum as the other keystream kernels.
//
// The drain is also cheaper than row_drain()'s two passes: the 8x32 bit transpose of a group of eight
// keystream words is done in registers right after the eight clocks that produce them (Grain's window leaves
// room for eight more live words; MICKEY's 200 state words do not), and the transposed words go straight to
// the tile at [k][group], so that the drain reads sixteen consecutive words per instance-row piece -- one
// tcgen05.ld.x16 or sixteen conflict-free LDS -- with no second pass over the tile.
#pragma once
#include "mk2_grain.cuh"
#include "mk2_tmem.cuh"

namespace mk2 {
namespace grain {
namespace row64 {

#ifndef MK2_GRAIN_ROW64_WIN
#define MK2_GRAIN_ROW64_WIN 16
#endif
constexpr int RWIN = MK2_GRAIN_ROW64_WIN;   // clocks per window realignment in this kernel: 8 or 16
constexpr int RGW = GB + RWIN;              // window length
constexpr int TILE_CLOCKS = 512;            // clocks per drain of a full-size tile = 64 bytes per instance row
constexpr int NGRP = TILE_CLOCKS / 8;       // 8-clock groups per full-size tile
constexpr int TMEM_WARPS = 4, SMEM_WARPS = 3, HALF_WARPS = 1;
constexpr int THREADS = 32 * (TMEM_WARPS + SMEM_WARPS + HALF_WARPS);
constexpr int SMEM_TS = 32 * SMEM_WARPS;    // tile stride in shared memory: consecutive threads -> consecutive banks
constexpr int SMEM_BYTES = TILE_CLOCKS * SMEM_TS * 4 + (TILE_CLOCKS / 2) * 32 * 4;  // three full tiles + one half tile

// A warp's staging tile.  Transposed word k (0..7) of group grp lives at word index k * ngrp + grp.  ONE code
// path serves the three kinds of tile (tensor memory / shared memory, 64 or 32 groups): the kind is a
// warp-uniform runtime value, so that the two warps that share an SM sub-partition (always one tensor-memory
// warp and one shared-memory warp: a warp reaches the tensor-memory lanes of quadrant warp % 4 only) run the
// same instructions and do not evict each other's loop from the instruction cache.
struct Tile {
    static constexpr int OUT_POLICY = 1;  // row stores ask L2 to keep the line (see store16)
    bool tm;         // tensor memory (else shared memory)
    uint32_t taddr;  // tensor memory: lane quadrant in bits 31:16, column 0
    uint32_t *col;   // shared memory: this thread's column
    int ts;          // shared memory: words between consecutive tile words (threads sharing the tile)
    int ngrp;        // 8-clock groups per tile: 64 (64 bytes per row and drain) or 32

    // The eight transposed words of one group, w[k] -> word index k * ngrp + grp.  ONE warp-uniform branch per
    // group: a branch per store would cut the clock loop into basic blocks of one clock each and cost the LOP3
    // stream its scheduling freedom (predicated tcgen05.st are turned into branches by ptxas as well).
    __device__ __forceinline__ void store8(int grp, const uint32_t (&w)[8]) const
    {
        if (tm) {
#pragma unroll
            for (int k = 0; k < 8; ++k) tmem::st1(taddr + (uint32_t)(k * ngrp + grp), w[k]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) col[(k * ngrp + grp) * ts] = w[k];
        }
    }
    __device__ __forceinline__ uint32_t load1(int idx) const
    {
        if (tm) {
            uint32_t v = tmem::ld1(taddr + (uint32_t)idx);
            tmem::wait_ld(v);
            return v;
        }
        return col[idx * ts];
    }
    __device__ __forceinline__ void load16(int first, uint32_t (&x)[16]) const
    {
        if (tm) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
                  "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
                : "r"(taddr + (uint32_t)first)
                : "memory");
            tmem::wait_ld(x);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = col[(first + i) * ts];
        }
    }
    __device__ __forceinline__ void stores_done() const
    {
        if (tm) tmem::wait_st();
    }
};

// The same tile in GLOBAL memory, sized and hinted to stay in L2 (mk2_set_row_staging(ctx, 3)): eight worker
// warps per SM x 64 KiB = 74 MB of scratch for the whole GPU against 126 MB of L2.  A thread only ever reads
// back the words it wrote itself (its own lane of [k][group][lane]), so there is nothing to synchronise: this
// is a register spill area with a known address, written with one coalesced 128-byte store per warp and word
// and read back the same way.  What it buys: no shared or tensor memory at all (eight warps, no STTM / LDTM,
// no allocation barrier) and still 64 contiguous bytes per instance row and drain.  What it costs: the
// keystream crosses the SM <-> L2 fabric three times (tile store, tile load, row store) instead of once.
#ifndef MK2_L2TILE_ST_POLICY
#define MK2_L2TILE_ST_POLICY 1   // tile stores: 0 = st.cg, 1 = L2 evict_last hint
#endif
#ifndef MK2_L2TILE_OUT_POLICY
#define MK2_L2TILE_OUT_POLICY 2  // row stores: 0 = plain, 1 = L2 evict_last, 2 = L2 evict_first
#endif
struct L2Tile {
    static constexpr int OUT_POLICY = MK2_L2TILE_OUT_POLICY;
    uint32_t *col;   // this thread's lane of the warp's scratch slot
    int ngrp;        // 8-clock groups per tile

    __device__ __forceinline__ void store8(int grp, const uint32_t (&w)[8]) const
    {
        uint32_t *p = col + grp * 32;
#if MK2_L2TILE_ST_POLICY == 1
        unsigned long long pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p + k * ngrp * 32), "r"(w[k]), "l"(pol) : "memory");
#else
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcg(p + k * ngrp * 32, w[k]);
#endif
    }
    __device__ __forceinline__ uint32_t load1(int idx) const { return __ldcg(col + idx * 32); }
    __device__ __forceinline__ void load16(int first, uint32_t (&x)[16]) const
    {
        const uint32_t *p = col + first * 32;
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = __ldcg(p + i * 32);
    }
    __device__ __forceinline__ void stores_done() const {}
};

// Eight keystream words of one 8-clock group -> bit transpose -> tile.  z[m] = keystream word of clock m.
template <bool LSB, class TT>
__device__ __forceinline__ void park_group(const TT &tile, int grp, const uint32_t (&z)[8])
{
    uint32_t w[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) w[LSB ? m : 7 - m] = z[m];  // clock m -> bit 7 - m (MSB-first) or m
    transpose8x32(w);                                       // w[k]: byte q = output byte of instance 8 q + k
    tile.store8(grp, w);
}

// Tile -> instance rows.  Whole tiles of complete, 16-byte aligned groups take the fast path: per k and per
// sixteen groups, sixteen consecutive words -> four 4x4 byte transposes -> one 16-byte store to each of the
// rows 8 q + k; the pieces of a row's 64-byte run follow one another within a few hundred cycles.
template <class TT>
__device__ __forceinline__ void drain(const TT &tile, uint8_t *dst, uint64_t pitch, int ngrp, uint64_t nrows, bool aligned)
{
    tile.stores_done();
    if (aligned && ngrp == tile.ngrp && __all_sync(0xFFFFFFFFu, nrows == 32)) {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
#pragma unroll 1
            for (int piece = 0; piece < ngrp; piece += 16) {
                uint32_t x[16];
                tile.load16(k * ngrp + piece, x);
                uint32_t y[4][4];  // [g4][q]
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) {
                    const uint32_t x4[4] = {x[4 * g4], x[4 * g4 + 1], x[4 * g4 + 2], x[4 * g4 + 3]};
                    bytes4x4(x4, y[g4]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    store16<TT::OUT_POLICY>(dst + (uint64_t)(8 * q + k) * pitch + piece, make_uint4(y[0][q], y[1][q], y[2][q], y[3][q]));
            }
        }
    } else {
        // ragged edge: short last tile, partial last group of instances, unaligned rows (nrows = 0: nothing stored)
#pragma unroll 1
        for (int k = 0; k < 8; ++k)
#pragma unroll 1
            for (int grp = 0; grp < ngrp; ++grp) {
                const uint32_t x = tile.load1(k * tile.ngrp + grp);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if ((uint64_t)(8 * q + k) < nrows) dst[(uint64_t)(8 * q + k) * pitch + grp] = (uint8_t)(x >> (8 * q));
            }
    }
}

// One worker warp: pop chains, run chunks of clocks, park keystream in `tile`, drain every 8 * tile.ngrp clocks.
// Every thread of the warp runs along (the tensor-memory loads and stores are warp-collective): a thread whose
// group does not exist (last, partial chain) works on the last real group and stores nothing.
template <bool LSB, class TT>
__device__ __forceinline__ void worker(const TT &tile, const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                                       unsigned long long *acc_out, uint8_t *out, uint64_t pitch, uint64_t N, uint64_t G, uint64_t T,
                                       uint32_t chunk, uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots,
                                       uint32_t mask, uint32_t *progress, uint32_t chain_base, bool aligned)
{
    const int tile_clocks = 8 * tile.ngrp;
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g_own = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);
        const bool real = g_own < G;
        const uint64_t g = real ? g_own : G - 1;
        const uint64_t c0 = (uint64_t)k * chunk;  // chunk is a multiple of TILE_CLOCKS
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        {
            // Window of 80 + RWIN words per register, RWIN / 8 groups per loop iteration.  Measured on the B200 at
            // 2^22 instances (profiles/r02_probe_grain_row64.txt): RWIN 16 beats RWIN 8, whose 20 register copies
            // per clock (IMAD.MOV on the half-rate FMA pipe) cost more than its spill-free 245 registers return.
            uint32_t b[RGW], s[RGW];
            unsigned long long a;
            load_state(state, acc, G, g, b, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
            const uint64_t nrows = !real ? 0 : (N - 32 * g < 32 ? N - 32 * g : 32);
#pragma unroll 1
            for (uint64_t t0 = 0; t0 < tc; t0 += tile_clocks) {
                const int nclk = (tc - t0) >= (uint64_t)tile_clocks ? tile_clocks : (int)(tc - t0);  // a multiple of 8
                HalfSums hs;  // checksum on the FMA pipe; a tile is at most 512 words
                int grp = 0;
                static_assert(RWIN == 8 || RWIN == 16, "whole 8-clock groups per window");
#pragma unroll 1
                for (; grp + RWIN / 8 <= (nclk >> 3); grp += RWIN / 8) {
                    static_for_up<0, RWIN / 8>([&](auto hc) {
                        constexpr int h = decltype(hc)::value;
                        uint32_t z[8];
                        static_for_up<0, 8>([&](auto ic) {
                            constexpr int c = decltype(ic)::value;
                            z[c] = step<8 * h + c, false>(b, s);
                            hs.add(z[c]);
                        });
                        park_group<LSB>(tile, grp + h, z);
                    });
                    realign<RWIN>(b, s);
                }
                if (grp < (nclk >> 3)) {  // RWIN 16: one more group of eight clocks
                    uint32_t z[8];
                    static_for_up<0, 8>([&](auto ic) {
                        constexpr int c = decltype(ic)::value;
                        z[c] = step<c, false>(b, s);
                        hs.add(z[c]);
                    });
                    park_group<LSB>(tile, grp, z);
                    realign<8>(b, s);
                }
                hs.fold(a);
                drain(tile, rows + (t0 >> 3), pitch, nclk >> 3, nrows, aligned);
            }
            if (real) store_state(state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

template <bool LSB>
__global__ void __launch_bounds__(THREADS, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out, unsigned long long *acc_out,
                    uint8_t *__restrict__ out, uint64_t pitch, uint64_t N, uint64_t G, uint64_t T, uint32_t chunk,
                    uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress,
                    uint32_t chain_base, bool aligned)
{
    extern __shared__ uint32_t smem_tile[];  // [TILE_CLOCKS][SMEM_TS] for warps 4..6, then [TILE_CLOCKS / 2][32] for warp 7
    __shared__ uint32_t tmem_base_slot;
    const uint32_t warp = threadIdx.x >> 5;
    // the whole tensor memory of the SM: one persistent CTA per SM, so there is never a second allocator
    if (warp == 0) tmem::alloc(&tmem_base_slot, 512u);
    tmem::fence_before_sync();
    __syncthreads();
    tmem::fence_after_sync();

    Tile tile;
    tile.tm = warp < TMEM_WARPS;
    tile.taddr = tmem_base_slot + (((warp & 3u) * 32u) << 16);
    if (warp < TMEM_WARPS + SMEM_WARPS) {  // warps 4..6: full tiles side by side in shared memory
        tile.col = smem_tile + (threadIdx.x - 32 * TMEM_WARPS);
        tile.ts = SMEM_TS;
        tile.ngrp = NGRP;
    } else {                               // warp 7: the half tile behind them
        tile.col = smem_tile + TILE_CLOCKS * SMEM_TS + (threadIdx.x & 31u);
        tile.ts = 32;
        tile.ngrp = NGRP / 2;
    }
    worker<LSB>(tile, state, acc, state_out, acc_out, out, pitch, N, G, T, chunk, chunks_per_chain, q, slots, mask, progress,
                chain_base, aligned);

    tmem::fence_before_sync();
    __syncthreads();
    tmem::fence_after_sync();
    if (warp == 0) tmem::dealloc(tmem_base_slot, 512u);
}

// Every worker warp with its tile in L2-resident scratch: scratch[(CTA * 8 + warp)][k][group][lane].
constexpr size_t L2TILE_BYTES_PER_WARP = (size_t)TILE_CLOCKS * 32 * 4;
template <bool LSB>
__global__ void __launch_bounds__(BLOCK, 1)
gen_rowmajor_l2_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out, unsigned long long *acc_out,
                       uint8_t *__restrict__ out, uint64_t pitch, uint64_t N, uint64_t G, uint64_t T, uint32_t chunk,
                       uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress,
                       uint32_t chain_base, bool aligned, uint32_t *scratch)
{
    L2Tile tile;
    const uint32_t warp = threadIdx.x >> 5;
    tile.col = scratch + ((size_t)blockIdx.x * (BLOCK / 32) + warp) * (L2TILE_BYTES_PER_WARP / 4) + (threadIdx.x & 31u);
    tile.ngrp = NGRP;
    worker<LSB>(tile, state, acc, state_out, acc_out, out, pitch, N, G, T, chunk, chunks_per_chain, q, slots, mask, progress,
                chain_base, aligned);
}

}  // namespace row64
}  // namespace grain
}  // namespace mk2
