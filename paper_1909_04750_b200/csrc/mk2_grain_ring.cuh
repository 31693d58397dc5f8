// mk2_grain_ring.cuh -- Grain v1 row-major keystream for LONE warps: four worker warps per SM, one per
// sub-partition, the drain of a staging tile software-pipelined into the generation of the next one.
//
// Reference: pkg/src/slicerng/kernels.py:268-292 (Grain's compiled loop) + :600-621 (lane-major bytes).
//
// Why: the row-major drains leave one 32-byte sector per instance row and tile, and how fast those reach
// DRAM depends on how many rows are open at once (profiles/r02_probe_store_pattern.txt: with the L2
// evict_last hint, 1.9-2.0 TB/s at four warps per SM against 1.1-1.2 at seven or eight -- Grain needs 1.73).
// Four warps per SM means nobody hides a warp's latencies for it, so this kernel never stops to drain:
//   * the 8 x 32 bit transposes run in registers on the keystream words of each 8-clock group, inside the
//     16-clock window body (no load / transpose / store pass over the tile);
//   * the tile lives in a ring of three 16-group blocks per thread (48 groups, 1.5 KiB; 192 KiB per CTA):
//     tile i occupies two blocks, tile i + 1 starts in the third and only re-enters tile i's first block in
//     its ninth window -- so windows 0..7 of tile i + 1 each carry one eighth of tile i's drain (the 32 words
//     of one k, byte-transposed into four 32-byte row pieces), whose shared-memory loads and PRMTs the
//     scheduler interleaves with the cipher's LOP3s.
// Only full tiles, whole groups of 32 instances and 32-byte aligned rows come here (mk2_api.cu falls back to
// grain::gen_rowmajor_kernel otherwise), so there is no ragged code in the loop.
// Measured (B200, 2^22 instances x 65536 clocks): 10.5-10.6 Tb/s, level with the seven-warp default kernel before
// that one learnt the in-register transposes (11.4 now) -- lone warps lose to their own latencies what the better
// store pattern returns.  Opt-in: mk2_set_row_staging(ctx, 4).
#pragma once
#include "mk2_grain.cuh"

namespace mk2 {
namespace grain {
namespace ring {

constexpr int THREADS = 128;                     // four worker warps, one per sub-partition
constexpr int TILE_GROUPS = 32;                  // 256 clocks: one 32-byte sector per row and tile
constexpr int BLOCK_GROUPS = 16;                 // ring block
constexpr int RING_BLOCKS = 3;
constexpr uint32_t TS = THREADS;                 // word stride between a thread's consecutive tile words
constexpr uint32_t BLOCK_WORDS = BLOCK_GROUPS * 8 * TS;
constexpr int SMEM_BYTES = RING_BLOCKS * BLOCK_WORDS * 4;  // 196 608
constexpr int WINDOWS = 8 * TILE_GROUPS / WIN;   // 16 windows of 16 clocks per tile

// store32_keep() of mk2_kernels.cuh without the "memory" clobber: the row pieces are register values nobody in
// the kernel reads back, so the compiler and ptxas may move shared-memory traffic and the cipher across them.
__device__ __forceinline__ void store32_keep_free(uint8_t *p, const uint32_t (&v)[8])
{
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol));
}

// One eighth of a tile's drain: the 32 words of one k (rows 8 q + k, q = 0..3), 16 groups from each of the
// tile's two ring blocks (p0 / p1 already point at word k of the block's first group), as two passes that
// each build two rows, so that only 16 output words are live at a time.
__device__ __forceinline__ void drain_unit(const uint32_t *p0, const uint32_t *p1, uint8_t *dst, uint64_t pitch, bool store)
{
#pragma unroll
    for (int qh = 0; qh < 2; ++qh) {
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int g4 = 0; g4 < 8; ++g4) {
            const uint32_t *p = (g4 < 4 ? p0 : p1) + (4 * (g4 & 3)) * 8 * TS;
            const uint32_t x0 = p[0], x1 = p[8 * TS], x2 = p[16 * TS], x3 = p[24 * TS];
            const uint32_t a = prmt(x0, x1, qh ? 0x7362 : 0x5140);  // bytes 2q', 2q'+1 of the pair, interleaved
            const uint32_t b = prmt(x2, x3, qh ? 0x7362 : 0x5140);
            lo[g4] = prmt(a, b, 0x5410);  // row q = 2 qh:     bytes of groups 4 g4 .. 4 g4 + 3
            hi[g4] = prmt(a, b, 0x7632);  // row q = 2 qh + 1
        }
        if (store) {
            store32_keep_free(dst + (uint64_t)(16 * qh) * pitch, lo);
            store32_keep_free(dst + (uint64_t)(16 * qh + 8) * pitch, hi);
        }
    }
}

// One 16-clock window: keystream words -> two in-register 8 x 32 transposes -> ring slots at zp; with DRAIN,
// one unit of the previous tile's drain rides along.
template <bool LSB, bool DRAIN>
__device__ __forceinline__ void window(uint32_t (&b)[GW], uint32_t (&s)[GW], HalfSums &hs, uint32_t *zp, const uint32_t *p0,
                                       const uint32_t *p1, uint8_t *dst, uint64_t pitch, bool store)
{
    // The drain unit comes first (its loads read ring blocks this window does not write).  Its stores are guarded
    // (`store`: a chunk's first tile has no predecessor), which makes the unit a region of its own in front of the
    // cipher's instructions.  The branch-free form -- unit and cipher in one basic block -- was measured and is
    // SLOWER (10.1-10.2 against 10.5-10.6 Tb/s): ptxas then issues all 32 LDS and most of the 64 PRMT before the
    // first LOP3 of the window (profiles/r02_probe_grain_lone_warps.txt, section 5).
    if constexpr (DRAIN) drain_unit(p0, p1, dst, pitch, store);
    window_begin(b, s);
    uint32_t zz[WIN];
    static_for_up<0, WIN>([&](auto ic) {
        constexpr int c = decltype(ic)::value;
        zz[c] = step<c, false>(b, s);
        hs.add(zz[c]);
    });
#pragma unroll
    for (int h = 0; h < WIN / 8; ++h) {
        uint32_t z[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) z[LSB ? m : 7 - m] = zz[8 * h + m];  // clock m -> bit 7 - m (MSB-first) or m
        transpose8x32(z);  // z[k]: byte q = output byte of instance 8 q + k for this group
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) zp[(8 * h + kk) * TS] = z[kk];
    }
    window_end(b, s);
}

template <bool LSB>
__global__ void __launch_bounds__(THREADS, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out, unsigned long long *acc_out,
                    uint8_t *__restrict__ out, uint64_t pitch, uint64_t G, uint64_t T, uint32_t chunk,
                    uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress,
                    uint32_t chain_base)
{
    extern __shared__ uint32_t tile[];  // [3 blocks][16 groups][8 k][128 threads]
    uint32_t *col = tile + threadIdx.x;
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);
        const uint64_t c0 = (uint64_t)k * chunk;  // chunk and T are multiples of 256 clocks
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        if (g < G) {
            uint32_t b[GW], s[GW];
            unsigned long long a;
            load_state<OFF>(state, acc, G, g, b, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
            const uint32_t ntiles = (uint32_t)(tc >> 8);
            uint32_t bx = 0;          // ring block of the first half of the tile being generated
            uint32_t px = 0, py = 0;  // the previous tile's blocks
            uint8_t *prev = rows;
#pragma unroll 1
            for (uint32_t ti = 0; ti < ntiles; ++ti) {
                const uint32_t by = bx == RING_BLOCKS - 1 ? 0 : bx + 1;
                const bool store = ti != 0;  // the chunk's first tile has no predecessor to drain
                HalfSums hs;  // 256 words per tile
                {
                    uint32_t *zp = col + bx * BLOCK_WORDS;
                    const uint32_t *p0 = col + px * BLOCK_WORDS, *p1 = col + py * BLOCK_WORDS;
                    uint8_t *dst = prev;
#pragma unroll 1
                    for (int w = 0; w < WINDOWS / 2; ++w) {
                        window<LSB, true>(b, s, hs, zp, p0, p1, dst, pitch, store);
                        zp += WIN * TS;
                        p0 += TS;
                        p1 += TS;
                        dst += pitch;
                    }
                }
                {
                    uint32_t *zp = col + by * BLOCK_WORDS;
#pragma unroll 1
                    for (int w = 0; w < WINDOWS / 2; ++w) {
                        window<LSB, false>(b, s, hs, zp, nullptr, nullptr, nullptr, 0, false);
                        zp += WIN * TS;
                    }
                }
                hs.fold(a);
                prev = rows + (uint64_t)ti * (8 * TILE_GROUPS / 8);
                px = bx;
                py = by;
                bx = by == RING_BLOCKS - 1 ? 0 : by + 1;
            }
            // the chunk's last tile has no successor to ride on
            if (ntiles) {
                const uint32_t *p0 = col + px * BLOCK_WORDS, *p1 = col + py * BLOCK_WORDS;
#pragma unroll 1
                for (int kk = 0; kk < 8; ++kk) {
                    drain_unit(p0, p1, prev, pitch, true);
                    p0 += TS;
                    p1 += TS;
                    prev += pitch;
                }
            }
            store_state<OFF>(state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

}  // namespace ring
}  // namespace grain
}  // namespace mk2
