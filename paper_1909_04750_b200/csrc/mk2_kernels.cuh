// mk2_kernels.cuh -- sm_100a kernels of the bitsliced MICKEY 2.0 path.
//
// Data layout in HBM (all little-endian uint32 words, G = N/32 groups):
//   state[200][G]   word i   (i < 100)  = R bit i of the 32 instances of group g
//                   word 100+i          = S bit i            (mickey.py:236-243)
//   mat[c][G]       input word of load clock c (bit j = instance j's IV/key bit,
//                   mickey.py:291-301); ragged sets append activity masks
//   acc[G]          per-group uint64 sum of every keystream word emitted
//   out (column)    uint32 out[t][stride]  bit j of out[t][g] = z_t of inst 32g+j
//   out (row)       uint8  out[n][pitch]   MSB-first bytes   (kernels.py:604-621)
// Consecutive threads own consecutive groups g, so every access to state / mat /
// column-major output is a fully coalesced 128-byte warp transaction.
#pragma once
#include <cuda_runtime.h>

#include "mk2_clock.cuh"
#include "mk2_bits.cuh"

#ifndef MK2_RBLOCK_COL
#define MK2_RBLOCK_COL 6
#endif
#ifndef MK2_RBLOCK_ROW
#define MK2_RBLOCK_ROW 5
#endif
#ifndef MK2_RBLOCK_INIT
#define MK2_RBLOCK_INIT 4
#endif

namespace mk2 {

// Clocks per clock_block (deferred R reduction, mk2_clock.cuh) in the column-major, row-major and
// init kernels.  1 = the plain one-clock body.  Build-time knobs: the longer the block, the fewer
// LOP3 per clock (4: 303.8, 5: 301.2, 6: 299.7) and the larger the loop body (4.9 KB per clock).
// Defaults from the A/B on B200 (profiles/r01b_probe_rblock.txt): column-major gains up to 6;
// row-major and init start spilling inside the block at 6 / 5.
// Column-major loop: output addressing (0 = 64-bit pointer bump, 1 = 32-bit index) and checksum (0 = mad.wide
// accumulate, 1 = IDP.2A half sums); row-major loop: checksum likewise.  See gen_colmajor_kernel.
#ifndef MK2_COL_ADDR
#define MK2_COL_ADDR 0
#endif
#ifndef MK2_COL_SUM
#define MK2_COL_SUM 0
#endif
#ifndef MK2_ROW_SUM
#define MK2_ROW_SUM 1
#endif
#ifndef MK2_DRAIN_UNROLL_HALF
#define MK2_DRAIN_UNROLL_HALF 1
#endif
#ifndef MK2_COL_LOOP_UNROLL
#define MK2_COL_LOOP_UNROLL 1
#endif
constexpr int COL_LOOP_UNROLL = MK2_COL_LOOP_UNROLL;  // clock_blocks per iteration of the column-major loop
constexpr int DRAIN_UNROLL_HALF = MK2_DRAIN_UNROLL_HALF;  // row drain, pass 2: sector halves per iteration
constexpr int RBLOCK_COL = MK2_RBLOCK_COL;
constexpr int RBLOCK_ROW = MK2_RBLOCK_ROW;
constexpr int RBLOCK_INIT = MK2_RBLOCK_INIT;
constexpr int BLOCK = 256;           // 8 warps = 2 per SM sub-partition at 255 regs/thread
// Row-major staging: TG 8-clock groups per drain = TG bytes per instance row per drain.
// TG = 32 (256 clocks, a full 32-byte sector per row) needs 1 KiB of shared memory per
// thread, i.e. at most 6 worker warps per SM; TG = 16 allows 8 warps but writes half
// sectors (measured: 4x the algorithmic DRAM traffic from read-modify-write).
constexpr int row_smem_bytes(int tg, int threads) { return 8 * tg * threads * 4; }

// ---------------------------------------------------------------------------
// 8 x 32 bit-matrix transpose, in place: afterwards bit (8q + k) of w[b] is the
// old bit (8q + b) of w[k]  (four independent 8x8 transposes, one per byte
// column).  Three half-block swap stages, the log-step scheme of the
// reference's _square_transpose (pkg/src/slicerng/bitslab.py:183-200)
// restricted to the last three stages.  2 shifts (FMA pipe) + 2 LOP3 per pair.
// ---------------------------------------------------------------------------
// Both shifts are issued on the FMA pipe, which the keystream kernels leave idle: the left shift as
// IMAD.SHL (ptxas' own choice), the right shift as IMAD.HI with the multiplier 2^(32-S) read from
// constant memory (a literal would be strength-reduced back to an ALU-pipe SHF).  Each merge is ONE
// LOP3 with the mask as its third operand; written as (x & M) | (y & ~M), ptxas emits two.
__constant__ uint32_t shr_mul[5] = {0u, 1u << 31, 1u << 30, 0u, 1u << 28};  // [S] = 2^(32-S), S in {1, 2, 4}
template <int S>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x)
{
    return __umulhi(x, shr_mul[S]);
}
template <int S, uint32_t M>
__device__ __forceinline__ void swap_stage(uint32_t &a, uint32_t &b)
{
    constexpr unsigned SEL = ((LA & LC) | (LB & ~LC)) & 0xFF;  // (x & m) | (y & ~m)
    const uint32_t na = lop3<SEL>(a, b << S, M);
    const uint32_t nb = lop3<SEL>(shr_fma<S>(a), b, M);
    a = na;
    b = nb;
}
__device__ __forceinline__ void transpose8x32(uint32_t (&w)[8])
{
    swap_stage<4, 0x0F0F0F0Fu>(w[0], w[4]);
    swap_stage<4, 0x0F0F0F0Fu>(w[1], w[5]);
    swap_stage<4, 0x0F0F0F0Fu>(w[2], w[6]);
    swap_stage<4, 0x0F0F0F0Fu>(w[3], w[7]);
    swap_stage<2, 0x33333333u>(w[0], w[2]);
    swap_stage<2, 0x33333333u>(w[1], w[3]);
    swap_stage<2, 0x33333333u>(w[4], w[6]);
    swap_stage<2, 0x33333333u>(w[5], w[7]);
    swap_stage<1, 0x55555555u>(w[0], w[1]);
    swap_stage<1, 0x55555555u>(w[2], w[3]);
    swap_stage<1, 0x55555555u>(w[4], w[5]);
    swap_stage<1, 0x55555555u>(w[6], w[7]);
}

struct NoInput {  // clock_block's input source when no input word is injected
    template <class KC>
    __device__ __forceinline__ uint32_t operator()(KC) const { return 0u; }
};

// ---------------------------------------------------------------------------
// Material packing: row-major key/IV bytes -> one bitsliced input word per load
// clock (the word-wide load of mickey.py:291-301, for 32 lanes per thread).
// nbytes byte columns of `src` (row stride `stride`) become clocks
// c0 .. c0 + nbits - 1, MSB-first per byte (bitops.py:33-36).  Rows >= N read
// as zero: the reference's unused lanes (zero material).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pack_bytes_to_clocks(const uint8_t *__restrict__ src, uint32_t stride,
                                                     uint64_t first_row, uint64_t N, int nbits,
                                                     uint32_t *__restrict__ mat, uint64_t G, uint64_t g, int c0)
{
    const int nbytes = (nbits + 7) >> 3;
    for (int b = 0; b < nbytes; ++b) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t v = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t row = first_row + 8 * q + k;
                const uint32_t byte = row < N ? src[row * stride + b] : 0u;
                v |= byte << (8 * q);
            }
            w[k] = v;
        }
        transpose8x32(w);  // w[bit] = bit `bit` of byte b across the 32 instances
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int c = 8 * b + m;  // clock within this field; bit 7-m of the byte
            if (c < nbits) mat[(uint64_t)(c0 + c) * G + g] = w[7 - m];
        }
    }
}

// The same for 10-byte records (keys; IVs stored u8[N][10]) of a complete group whose 320 bytes are 16-byte
// aligned: twenty 128-bit loads bring the thread's 32 records into registers and every byte is picked with
// compile-time PRMT selectors, instead of 320 single-byte loads that each touch 32 sectors per warp
// (2^26 pairs: 2.6 -> 0.6 ms).
__device__ __forceinline__ void pack_records10_to_clocks(const uint8_t *__restrict__ src, int nbits, uint32_t *__restrict__ mat,
                                                         uint64_t G, uint64_t g, int c0)
{
    uint32_t rec[80];  // bytes 0..319 = records 32 g .. 32 g + 31
    const uint4 *p = reinterpret_cast<const uint4 *>(src + 320 * g);
#pragma unroll
    for (int i = 0; i < 20; ++i) {
        const uint4 v = __ldg(p + i);
        rec[4 * i] = v.x;
        rec[4 * i + 1] = v.y;
        rec[4 * i + 2] = v.z;
        rec[4 * i + 3] = v.w;
    }
    const int nbytes = (nbits + 7) >> 3;
    static_for_up<0, 9>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        if (b < nbytes) {
            uint32_t w[8];
            static_for_up<0, 7>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                // byte q of w[k] = byte b of record 8 q + k, at byte offset 10 (8 q + k) + b of rec[]
                constexpr int o0 = 10 * k + b, o1 = 10 * (8 + k) + b, o2 = 10 * (16 + k) + b, o3 = 10 * (24 + k) + b;
                const uint32_t lo = __byte_perm(rec[o0 >> 2], rec[o1 >> 2], (o0 & 3) | ((4 + (o1 & 3)) << 4));
                const uint32_t hi = __byte_perm(rec[o2 >> 2], rec[o3 >> 2], (o2 & 3) | ((4 + (o3 & 3)) << 4));
                w[k] = __byte_perm(lo, hi, 0x5410);
            });
            transpose8x32(w);  // w[bit] = bit `bit` of byte b across the 32 instances
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = 8 * b + m;  // clock within this field; bit 7 - m of the byte
                if (c < nbits) mat[(uint64_t)(c0 + c) * G + g] = w[7 - m];
            }
        }
    });
}

// fast10: both arrays are 16-byte aligned and the IVs are stored 10 bytes apart
__global__ void __launch_bounds__(BLOCK)
pack_uniform_kernel(const uint8_t *__restrict__ keys, const uint8_t *__restrict__ ivs, uint32_t iv_stride,
                    int iv_bits, uint64_t N, uint64_t G, uint32_t *__restrict__ mat, bool fast10)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    if (fast10 && 32 * g + 32 <= N) {
        if (iv_bits) pack_records10_to_clocks(ivs, iv_bits, mat, G, g, 0);
        pack_records10_to_clocks(keys, KEY_BITS, mat, G, g, iv_bits);
        return;
    }
    pack_bytes_to_clocks(ivs, iv_stride, 32 * g, N, iv_bits, mat, G, g, 0);
    pack_bytes_to_clocks(keys, 10, 32 * g, N, KEY_BITS, mat, G, g, iv_bits);
}

// Ragged IV lengths (mickey.py:287-289 falls back to per-lane scalar init; here
// the lanes stay bitsliced): lane j with L_j IV bits idles in the all-zero
// state for Lmax - L_j clocks and then loads normally, so all lanes finish the
// IV phase together.  nbits[row] in 0..80, or 0xFF for an unused lane that
// must end in the all-zero state (from_scalar_states, mickey.py:306-316).
// mat rows: [0, Lmax+80) input words; [Lmax+80, 2 Lmax+80) activity masks
// (bit j set once lane j has started); row 2 Lmax+80: final lane mask.
// fast10 (complete groups, 10-byte IV records, 16-byte aligned arrays): the group's 320 IV bytes and 32
// lengths come in with 128-bit loads, every lane's bit string is shifted to its start clock with funnel
// shifts and three 32x32 bit transposes per array turn lanes into clock words (mk2_bits.cuh) -- instead of
// one byte load and a handful of ALU ops per (lane, clock).
__global__ void __launch_bounds__(BLOCK)
pack_ragged_kernel(const uint8_t *__restrict__ keys, const uint8_t *__restrict__ ivs, uint32_t iv_stride,
                   const uint8_t *__restrict__ nbits, int lmax, uint64_t N, uint64_t G,
                   uint32_t *__restrict__ mat, bool fast10)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    if (fast10 && 32 * g + 32 <= N) {
        uint32_t len[8];
        {
            const uint4 *pl = reinterpret_cast<const uint4 *>(nbits + 32 * g);
            const uint4 a = __ldg(pl), b = __ldg(pl + 1);
            len[0] = a.x; len[1] = a.y; len[2] = a.z; len[3] = a.w;
            len[4] = b.x; len[5] = b.y; len[6] = b.z; len[7] = b.w;
        }
        uint32_t used = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) used |= (((len[j >> 2] >> (8 * (j & 3))) & 0xFFu) <= 80u ? 1u : 0u) << j;
        if (lmax > 0) {
            uint32_t rec[80];
            const uint4 *p = reinterpret_cast<const uint4 *>(ivs + 320 * g);
#pragma unroll
            for (int i = 0; i < 20; ++i) {
                const uint4 v = __ldg(p + i);
                rec[4 * i] = v.x; rec[4 * i + 1] = v.y; rec[4 * i + 2] = v.z; rec[4 * i + 3] = v.w;
            }
#pragma unroll 1
            for (int k = 0; 32 * k < lmax; ++k) {
                uint32_t in[32], act[32];
                ragged_group_words(rec, len, lmax, k, in, act);
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    const int c = 32 * k + b;
                    if (c < lmax) {
                        mat[(uint64_t)c * G + g] = in[b];
                        mat[(uint64_t)(lmax + KEY_BITS + c) * G + g] = act[b];
                    }
                }
            }
        }
        mat[(uint64_t)(2 * lmax + KEY_BITS) * G + g] = used;
        pack_records10_to_clocks(keys, KEY_BITS, mat, G, g, lmax);
        return;
    }
    uint32_t used = 0;
    int len[32];
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {
        const uint64_t row = 32 * g + j;
        const int l = row < N ? nbits[row] : 0xFF;
        len[j] = l;
        if (l <= 80) used |= 1u << j;
    }
    for (int c = 0; c < lmax; ++c) {
        uint32_t w = 0, act = 0;
        for (int j = 0; j < 32; ++j) {
            const int l = len[j];
            if (l > 80) continue;
            const int start = lmax - l;
            if (c >= start) {
                act |= 1u << j;
                const int cc = c - start;
                const uint32_t byte = ivs[(32 * g + j) * (uint64_t)iv_stride + (cc >> 3)];
                w |= ((byte >> (7 - (cc & 7))) & 1u) << j;
            }
        }
        mat[(uint64_t)c * G + g] = w;
        mat[(uint64_t)(lmax + KEY_BITS + c) * G + g] = act;
    }
    mat[(uint64_t)(2 * lmax + KEY_BITS) * G + g] = used;
    pack_bytes_to_clocks(keys, 10, 32 * g, N, KEY_BITS, mat, G, g, lmax);
}

// Counter-IV synthetic set: one key for every instance,
// IV_k = the 80-bit big-endian value of the global instance index
// k = first + 32 g + j (first % 32 == 0), so load clock c carries bit 79 - c of
// k: the five low bits are fixed lane patterns, the rest are uniform words.
__global__ void __launch_bounds__(BLOCK)
pack_counter_kernel(uint64_t key_hi16, uint64_t key_lo64, uint64_t first, uint64_t G, uint32_t *__restrict__ mat)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    const uint64_t base = first + 32 * g;
    for (int c = 0; c < 80; ++c) {
        const int p = 79 - c;
        uint32_t w;
        if (p >= 64) w = 0u;
        else if (p >= 5) w = ((base >> p) & 1ull) ? 0xFFFFFFFFu : 0u;
        else w = p == 0 ? 0xAAAAAAAAu : p == 1 ? 0xCCCCCCCCu : p == 2 ? 0xF0F0F0F0u : p == 3 ? 0xFF00FF00u : 0xFFFF0000u;
        mat[(uint64_t)c * G + g] = w;
    }
    for (int c = 0; c < 80; ++c) {  // key bit c, MSB-first over the 10 key bytes
        const int p = 79 - c;
        const uint64_t bit = p >= 64 ? (key_hi16 >> (p - 64)) & 1ull : (key_lo64 >> p) & 1ull;
        mat[(uint64_t)(80 + c) * G + g] = bit ? 0xFFFFFFFFu : 0u;
    }
}

// ---------------------------------------------------------------------------
// Key/IV load + pre-clock (mickey.py:141-151 / :291-303), 32 instances per
// thread, one input word per load clock.  RAGGED adds the activity masking
// described at pack_ragged_kernel.
// ---------------------------------------------------------------------------
template <bool RAGGED>
__global__ void __launch_bounds__(BLOCK, 1)
init_kernel(const uint32_t *__restrict__ mat, int load_clocks, int lmax, uint64_t G,
            uint32_t *__restrict__ state, unsigned long long *__restrict__ acc)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    uint32_t r[NBITS], s[NBITS];
#pragma unroll
    for (int i = 0; i < NBITS; ++i) r[i] = s[i] = 0u;

    // input words are fetched one clock ahead so the load latency hides behind a clock's LOP3s
    const uint32_t *p = mat + g;
    int c = 0;
    uint32_t in_next = load_clocks > 0 ? __ldg(p) : 0u;
    if constexpr (RAGGED) {
        // IV phase of a group whose lanes start at different clocks: masked blocks (clock_block_masked holds
        // the lanes that have not started in the all-zero state for 5 extra LOP3 per clock), the next block's
        // input and activity words in flight while this one runs
        const uint32_t *pa = mat + (uint64_t)(lmax + KEY_BITS) * G + g;
        constexpr int KB = RBLOCK_INIT > 4 ? 4 : RBLOCK_INIT;
        uint32_t nx[KB], na[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            nx[k] = k < lmax ? __ldg(p + (uint64_t)k * G) : 0u;
            na[k] = k < lmax ? __ldg(pa + (uint64_t)k * G) : 0u;
        }
#pragma unroll 1
        for (; c + KB <= lmax; c += KB) {
            uint32_t cur[KB], act[KB];
            p += (uint64_t)KB * G;
            pa += (uint64_t)KB * G;
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                cur[k] = nx[k];
                act[k] = na[k];
                nx[k] = c + KB + k < lmax ? __ldg(p + (uint64_t)k * G) : 0u;
                na[k] = c + KB + k < lmax ? __ldg(pa + (uint64_t)k * G) : 0u;
            }
            clock_block_masked<KB>(
                r, s, [&](auto kc) { return cur[decltype(kc)::value]; }, [&](auto kc) { return act[decltype(kc)::value]; });
        }
#pragma unroll 1
        for (int k = 0; c < lmax; ++c, ++k) {  // up to KB - 1 single masked clocks; nx / na already hold their words
            uint32_t w = nx[0], a = na[0];
#pragma unroll
            for (int q = 1; q < KB; ++q)
                if (k == q) { w = nx[q]; a = na[q]; }
            p += G;
            clock_block_masked<1>(r, s, [&](auto) { return w; }, [&](auto) { return a; });
        }
        in_next = c < load_clocks ? __ldg(p) : 0u;
    }
    if constexpr (RBLOCK_INIT > 1) {
        // blocks of RBLOCK_INIT load clocks (deferred R reduction); the next block's input words are in flight
        // while this one runs
        uint32_t nx[RBLOCK_INIT];
        nx[0] = in_next;
#pragma unroll
        for (int k = 1; k < RBLOCK_INIT; ++k) nx[k] = c + k < load_clocks ? __ldg(p + (uint64_t)k * G) : 0u;
#pragma unroll 1
        for (; c + RBLOCK_INIT <= load_clocks; c += RBLOCK_INIT) {
            uint32_t cur[RBLOCK_INIT];
            p += (uint64_t)RBLOCK_INIT * G;
#pragma unroll
            for (int k = 0; k < RBLOCK_INIT; ++k) {
                cur[k] = nx[k];
                nx[k] = c + RBLOCK_INIT + k < load_clocks ? __ldg(p + (uint64_t)k * G) : 0u;
            }
            clock_block<RBLOCK_INIT, true, true, false>(
                r, s, [&](auto kc) { return cur[decltype(kc)::value]; }, [](auto, uint32_t) {});
        }
        in_next = nx[0];
    }
#pragma unroll 1
    for (; c < load_clocks; ++c) {
        const uint32_t in = in_next;
        p += G;
        if (c + 1 < load_clocks) in_next = __ldg(p);
        clock<true, true>(r, s, in);
    }
    {
        int k = 0;
        if constexpr (RBLOCK_INIT > 1) {
#pragma unroll 1
            for (; k + RBLOCK_INIT <= PRECLOCKS; k += RBLOCK_INIT)
                clock_block<RBLOCK_INIT, true, false, false>(r, s, NoInput{}, [](auto, uint32_t) {});
        }
#pragma unroll 1
        for (; k < PRECLOCKS; ++k) clock<true, false>(r, s, 0u);
    }

    if constexpr (RAGGED) {
        const uint32_t used = mat[(uint64_t)(2 * lmax + KEY_BITS) * G + g];
#pragma unroll
        for (int i = 0; i < NBITS; ++i) { r[i] &= used; s[i] &= used; }
    }
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        state[(uint64_t)i * G + g] = r[i];
        state[(uint64_t)(NBITS + i) * G + g] = s[i];
    }
    acc[g] = 0ull;
}

// ---------------------------------------------------------------------------
// Generic stepping: n CLOCK_KG calls with caller-supplied input words and
// mixing flag, no output (MickeySliced.clock_kg, mickey.py:329-360).  Used by
// the host mirror's clock_kg(); not a throughput path.
// ---------------------------------------------------------------------------
template <bool MIXING>
__global__ void __launch_bounds__(BLOCK, 1)
clock_kernel(uint32_t *__restrict__ state, const uint32_t *__restrict__ in_words, uint64_t n, uint64_t G)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    uint32_t r[NBITS], s[NBITS];
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        r[i] = state[(uint64_t)i * G + g];
        s[i] = state[(uint64_t)(NBITS + i) * G + g];
    }
#pragma unroll 1
    for (uint64_t c = 0; c < n; ++c) clock<MIXING, true>(r, s, in_words ? in_words[c * G + g] : 0u);
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        state[(uint64_t)i * G + g] = r[i];
        state[(uint64_t)(NBITS + i) * G + g] = s[i];
    }
}

// 64-bit accumulate on the FMA pipe (IMAD.WIDE.U32) so the checksum does not
// take ALU-pipe slots from the LOP3 stream.
__device__ __forceinline__ void acc_add(unsigned long long &acc, uint32_t z)
{
    asm("mad.wide.u32 %0, %1, 1, %0;" : "+l"(acc) : "r"(z));
}
// The same checksum without any ALU-pipe instruction: ptxas re-associates consecutive mad.wide
// accumulations into 3-input IADD3 + IADD3.X (one ALU slot per clock); integer dot products run on
// the FMA pipe and are left alone.  Two IDP.2A per keystream word keep the sums of its low and high
// 16-bit halves in 32-bit registers, exact for up to 65536 words; fold() adds them to the 64-bit sum.
struct HalfSums {
    uint32_t lo = 0, hi = 0;
    __device__ __forceinline__ void add(uint32_t z)
    {
        asm("dp2a.lo.u32.u32 %0, %1, %2, %0;" : "+r"(lo) : "r"(z), "r"(0x00000001));  // += z & 0xFFFF
        asm("dp2a.lo.u32.u32 %0, %1, %2, %0;" : "+r"(hi) : "r"(z), "r"(0x00000100));  // += z >> 16
    }
    __device__ __forceinline__ void fold(unsigned long long &acc)
    {
        acc += (unsigned long long)lo + ((unsigned long long)hi << 16);
        lo = hi = 0;
    }
};
constexpr uint32_t HALFSUM_MAX_WORDS = 65536;
static_assert((unsigned long long)HALFSUM_MAX_WORDS * 0xFFFFull <= 0xFFFFFFFFull, "half sums must fit 32 bits");
// pointer += bytes: as a mad.wide ptxas puts the carry half on the FMA pipe (IADD3 + IMAD.X)
template <class P>
__device__ __forceinline__ void ptr_add(P *&p, uint32_t bytes)
{
    asm("mad.wide.u32 %0, %1, 1, %0;" : "+l"(p) : "r"(bytes));
}

// ---------------------------------------------------------------------------
// Persistent scheduling of the keystream kernels.
//
// A "chain" is one warp's worth of groups (32 threads x 32 instances = 1024
// instances); its clocks are strictly serial, chains are independent.  The
// keystream of a chain is cut into chunks of `chunk` clocks.  Worker warps (one
// persistent CTA per SM) pull READY chains from a device-side FIFO ring, run one
// chunk (state in registers), park the state in HBM and push the chain back.
// With fewer chains than resident warps x sub-partition capacity (BASELINE
// config 2: 1024 chains on 592 sub-partitions) a static launch idles 14% of the
// ALU pipes; the FIFO hands a finished chain to the longest-idle worker, so
// load follows free sub-partitions.  With many chains it is a plain dynamic
// tile scheduler with a short tail.
//
// Ring entry = (ticket + 1) << 32 | chain, written with one 64-bit store, so a
// consumer spinning on its ticket's slot needs no separate flag.  State handed
// between SMs goes through L2 (ld.cg / st.cg + __threadfence on both sides).
// ---------------------------------------------------------------------------
struct SchedQueue {
    unsigned long long head;        // next pop ticket
    unsigned long long tail;        // next push ticket
    unsigned long long total_jobs;  // chains * chunks_per_chain
    unsigned long long pad;
};

// Optional per-job trace (mk2_set_trace): who ran which chunk where and when.
struct TraceRec {
    uint32_t chain, k, smid, warp;
    unsigned long long t_pop, t_start, t_end;  // %globaltimer, ns
    unsigned long long pad;
};
struct Trace {
    TraceRec *rec;
    unsigned long long *count;
    unsigned long long capacity;
};
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid()
{
    uint32_t v;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    return v;
}
__device__ __forceinline__ void trace_job(const Trace &tr, uint32_t chain, uint32_t k, unsigned long long t_pop,
                                          unsigned long long t_start, unsigned long long t_end)
{
    if (tr.rec && (threadIdx.x & 31u) == 0) {
        const unsigned long long i = atomicAdd(tr.count, 1ull);
        if (i < tr.capacity) {
            TraceRec r;
            r.chain = chain; r.k = k; r.smid = smid(); r.warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
            r.t_pop = t_pop; r.t_start = t_start; r.t_end = t_end; r.pad = 0;
            tr.rec[i] = r;
        }
    }
    __syncwarp();
}

__global__ void sched_init_kernel(SchedQueue *q, unsigned long long *slots, uint32_t *progress, uint32_t chains,
                                  uint32_t chunks_per_chain, uint32_t ring)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        q->pad = 0ull;
        q->head = 0ull;
        q->tail = chains;
        q->total_jobs = (unsigned long long)chains * chunks_per_chain;
    }
    // tickets 0..chains-1 are pre-filled; every other slot is cleared so that an
    // entry left by an earlier launch can never match a ticket of this one
    if (i < ring) slots[i] = i < chains ? (((unsigned long long)(i + 1) << 32) | i) : 0ull;
    if (i < chains) progress[i] = 0u;
}

// Memory-ordering helpers (PTX memory model, gpu scope).  st.release compiles to
// MEMBAR.ALL.GPU + a strong store and, unlike __threadfence(), does not
// invalidate L1; ld.acquire is a strong load followed by one L1 invalidate.
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Returns false when all work has been handed out.  The whole warp executes
// every instruction here (lane 0's atomic is predicated, the poll is one
// broadcast load): a lane-0-only polling loop was measured to leave the warp
// running its next job at half speed.
__device__ __forceinline__ bool sched_pop(SchedQueue *q, const unsigned long long *slots, uint32_t mask,
                                          uint32_t &chain)
{
    const unsigned lane = threadIdx.x & 31u;
    unsigned long long t = 0ull;
    if (lane == 0) t = atomicAdd(&q->head, 1ull);
    t = __shfl_sync(0xFFFFFFFFu, t, 0);
    if (t >= ld_relaxed_u64(&q->total_jobs)) return false;
    const unsigned long long *slot = slots + (t & mask);
    const unsigned long long want = (t + 1) & 0xFFFFFFFFull;
    unsigned ns = 32;
    while ((ld_relaxed_u64(slot) >> 32) != want) {
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
    }
    const unsigned long long e = ld_acquire_u64(slot);  // acquire: the chain's parked state is visible
    chain = (uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)e, 0);
    return true;
}

// Every lane has already published its share of the chain's state with a
// release store (store_state); lane 0 hands the chain to the next worker.
__device__ __forceinline__ void sched_push(SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress,
                                           uint32_t chain, uint32_t k_done, uint32_t chunks_per_chain)
{
    __syncwarp();
    if ((threadIdx.x & 31u) == 0) {
        __stcg(progress + chain, k_done);
        if (k_done < chunks_per_chain) {
            const unsigned long long t = atomicAdd(&q->tail, 1ull);
            st_release_u64(slots + (t & mask), ((t + 1) << 32) | chain);
        }
    }
    __syncwarp();
}

// State moves between SMs through L2: ld.cg / st.cg, addresses by pointer
// bumping.  The kernels receive the state / accumulator base twice (an input
// and an output parameter holding the same address): otherwise ptxas keeps the
// 200 load addresses alive across the clock loop to reuse them for the
// stores, and spills every one of them.  The accumulator store doubles as the
// lane's release fence for everything it wrote in this job.
__device__ __forceinline__ void bump(const uint32_t *&p, uint64_t stride)
{
    p += stride;
    asm volatile("" : "+l"(p));
}
__device__ __forceinline__ void load_state(const uint32_t *__restrict__ state, const unsigned long long *acc,
                                           uint64_t G, uint64_t g, uint32_t (&r)[NBITS], uint32_t (&s)[NBITS],
                                           unsigned long long &a)
{
    const uint32_t *p = state + g;
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        r[i] = __ldcg(p);
        bump(p, G);
    }
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        s[i] = __ldcg(p);
        bump(p, G);
    }
    a = __ldcg(acc + g);
}
__device__ __forceinline__ void store_state(uint32_t *__restrict__ state, unsigned long long *acc, uint64_t G,
                                            uint64_t g, const uint32_t (&r)[NBITS], const uint32_t (&s)[NBITS],
                                            unsigned long long a)
{
    const uint32_t *p = state + g;
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        __stcg(const_cast<uint32_t *>(p), r[i]);
        bump(p, G);
    }
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        __stcg(const_cast<uint32_t *>(p), s[i]);
        bump(p, G);
    }
    st_release_u64(acc + g, a);
}

// ---------------------------------------------------------------------------
// Keystream, column-major: out[t * stride + g] = z_t (mickey.py:362-368; the
// compiled loop kernels.py:46-95).  Resumable: state and the checksum
// accumulator live in HBM between chunks and between calls.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK, 1)
gen_colmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                    unsigned long long *acc_out, uint32_t *__restrict__ out, uint64_t stride, uint64_t G, uint64_t T, uint32_t chunk,
                    uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask,
                    uint32_t *progress, Trace tr)
{
    uint32_t chain;
    for (;;) {
        const unsigned long long t_pop = tr.rec ? gtime() : 0ull;
        if (!sched_pop(q, slots, mask, chain)) break;
        const unsigned long long t_start = tr.rec ? gtime() : 0ull;
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)chain * 32 + (threadIdx.x & 31u);
        const uint64_t t0 = (uint64_t)k * chunk;
        const uint64_t tc = T - t0 < chunk ? T - t0 : chunk;
        if (g < G) {
            uint32_t r[NBITS], s[NBITS];
            unsigned long long a;
            load_state(state, acc, G, g, r, s, a);
            // Build-time experiment knobs (profiles/r01b_probe_col_row_variants.txt).  MK2_COL_ADDR 1: a
            // 64-bit base and a 32-bit element index (index * 4 + base is one IMAD.WIDE, the index bump a
            // uniform-datapath IMAD) instead of a 64-bit pointer bump (IADD3 + IMAD.X per clock);
            // MK2_COL_SUM 1: IDP.2A half sums instead of the mad.wide accumulate (3-input IADD3 + IADD3.X
            // per two clocks).  Both remove every non-LOP3 instruction from the ALU pipe (1810 -> 1798 per
            // six clocks) and both are SLOWER by 0.3-0.7% on the B200 in this loop, so the defaults are 0/0;
            // the row-major loop, with its shared-memory stores, gains 1.5% from the half sums at 2^24 instances.
            uint32_t *base = out + t0 * stride + g;
            const uint32_t stride32 = (uint32_t)stride;  // host side guarantees stride < 2^30
            uint32_t seg_max = 0xFFFFFFFFu / stride32;
            if (seg_max > HALFSUM_MAX_WORDS) seg_max = HALFSUM_MAX_WORDS;
            if (seg_max > RBLOCK_COL) seg_max -= seg_max % RBLOCK_COL;
            uint64_t t = 0;
#pragma unroll 1
            while (t < tc) {
                const uint32_t nseg = tc - t < seg_max ? (uint32_t)(tc - t) : seg_max;
                [[maybe_unused]] uint32_t idx = 0;
                [[maybe_unused]] uint32_t *p = base;
                uint32_t u = 0;
                HalfSums hs;
                auto emit = [&](uint32_t z) {
#if MK2_COL_ADDR
                    base[idx] = z;
                    idx += stride32;
#else
                    *p = z;
                    ptr_add(p, stride32 * 4u);
#endif
#if MK2_COL_SUM
                    hs.add(z);
#else
                    acc_add(a, z);
#endif
                };
                if constexpr (RBLOCK_COL > 1) {
#pragma unroll COL_LOOP_UNROLL
                    for (; u + RBLOCK_COL <= nseg; u += RBLOCK_COL)
                        clock_block<RBLOCK_COL, false, false, true>(r, s, NoInput{}, [&](auto, uint32_t z) { emit(z); });
                }
#pragma unroll 1
                for (; u < nseg; ++u) {
                    emit(keystream_word(r, s));
                    clock<false, false>(r, s, 0u);
                }
                hs.fold(a);
                base += (uint64_t)nseg * stride;
                t += nseg;
            }
            store_state(state_out, acc_out, G, g, r, s, a);
        }
        const unsigned long long t_end = tr.rec ? gtime() : 0ull;  // before the chain is handed on
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
        trace_job(tr, chain, k, t_pop, t_start, t_end);
    }
}

// ---------------------------------------------------------------------------
// Keystream, row-major: out[(32 g + j) * pitch + t / 8], MSB-first bytes
// (kernels.py:604-621, bitops.py:20-23).
//
// The clock loop is the blocked loop of the column-major kernel, except that z_t goes to
// a per-thread staging tile instead of HBM: the 200 state words leave no registers to
// hold keystream.  This kernel keeps the tile in a private shared-memory column
// (tile[t][tid], conflict-free); the default for MICKEY, tmem::gen_rowmajor_kernel in
// mk2_tmem.cuh, keeps it in tensor memory with the same two-pass drain.  Every 8 * TG
// clocks (256 = a full 32-byte sector per instance row) the thread drains its tile:
//   pass 1  per 8 clocks: 8 words back into registers, 8x32 bit transpose
//           (word k, byte q = the output byte of instance 8q + k), back in place;
//   pass 2  per k: 16 words (one per 8-clock group) -> 4x4 byte transposes with
//           PRMT -> one 16-byte store per instance row, the two halves of a sector
//           back to back.
// Each thread only ever reads what it wrote, so no barrier is needed; the drain loops
// are not unrolled further, which keeps the code inside the instruction cache.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    return __byte_perm(a, b, sel);
}

// x[0..3]: words of 4 consecutive groups for fixed k; y[q] = bytes q of x[0..3]
// in ascending group (= address) order.
__device__ __forceinline__ void bytes4x4(const uint32_t (&x)[4], uint32_t (&y)[4])
{
    const uint32_t a01 = prmt(x[0], x[1], 0x5140);  // [x0.b0, x1.b0, x0.b1, x1.b1]
    const uint32_t a23 = prmt(x[2], x[3], 0x5140);
    const uint32_t b01 = prmt(x[0], x[1], 0x7362);  // [x0.b2, x1.b2, x0.b3, x1.b3]
    const uint32_t b23 = prmt(x[2], x[3], 0x7362);
    y[0] = prmt(a01, a23, 0x5410);
    y[1] = prmt(a01, a23, 0x7632);
    y[2] = prmt(b01, b23, 0x5410);
    y[3] = prmt(b01, b23, 0x7632);
}

// 16-byte row store.  POLICY 1 asks L2 to keep the line (evict_last): the four sectors of a row's
// 128-byte line arrive one drain apart, and lines that survive in L2 until they are complete reach
// DRAM as one 128-byte write instead of four isolated sectors.
// Measured: Grain v1's row-major kernel, whose stores reach DRAM at 1.2 TB/s, gains 6.6% (its caller passes
// POLICY 1); MICKEY's, at 0.24 TB/s, is indifferent (POLICY 0).
template <int POLICY>
__device__ __forceinline__ void store16(uint8_t *p, uint4 v)
{
    if constexpr (POLICY == 1) {
        unsigned long long pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w), "l"(pol)
                     : "memory");
    } else if constexpr (POLICY == 2) {
        // streaming: the row piece is complete when it is written, L2 may write it back first
        unsigned long long pol;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w), "l"(pol)
                     : "memory");
    } else {
        *reinterpret_cast<uint4 *>(p) = v;
    }
}

// One 32-byte (256-bit, sm_100) row store with the same L2 hint: a whole sector in a single request.
__device__ __forceinline__ void store32_keep(uint8_t *p, const uint32_t (&v)[8])
{
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol)
                 : "memory");
}

// The same store, but the sector that COMPLETES a 128-byte line (address bits 6:5 = 3) is written evict_first:
// a complete line has nothing left to wait for in L2 and should make room for the open ones.
__device__ __forceinline__ void store32_line(uint8_t *p, const uint32_t (&v)[8])
{
    unsigned long long keep, go;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(go));
    const unsigned long long pol = (reinterpret_cast<uintptr_t>(p) & 96) == 96 ? go : keep;
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol)
                 : "memory");
}

// Drain of one staging tile (ngrp 8-clock groups of keystream words in the thread's smem
// column `col`, stride TS) into the instance rows at `dst`.  Shared by every cipher's
// row-major kernel.  LSB selects the byte packing: first bit in the MSB (library default,
// bitops.py:20-23) or in the LSB (Grain's published convention, grain.py:13-16).
template <bool ALIGNED16, int TG, int TS, bool LSB, int STORE_POLICY = 0, bool PRE_TRANSPOSED = false>
__device__ __forceinline__ void row_drain(uint32_t *col, uint8_t *dst, uint64_t pitch, int ngrp, uint64_t nrows)
{
    constexpr uint32_t ts = TS;
    // ---- pass 1: bit transposes, in place in the smem column; the next group's 8 words
    // are fetched while the current group is transposed (a lone warp has nobody else to
    // hide the LDS latency behind).  PRE_TRANSPOSED: the producer already stored the
    // transposed words of every group (Grain's full tiles).
    if constexpr (!PRE_TRANSPOSED) {
        uint32_t nx[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) nx[m] = col[m * ts];
#pragma unroll 1
        for (int grp = 0; grp < ngrp; ++grp) {
            uint32_t z[8];
            uint32_t *gp = col + grp * 8 * ts;
#pragma unroll
            for (int m = 0; m < 8; ++m) z[LSB ? m : 7 - m] = nx[m];  // clock m -> bit 7 - m (MSB-first) or m
            if (grp + 1 < ngrp) {
#pragma unroll
                for (int m = 0; m < 8; ++m) nx[m] = gp[(8 + m) * ts];
            }
            transpose8x32(z);  // z[k]: byte q = output byte of instance 8 q + k
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) gp[kk * ts] = z[kk];
        }
    }
    // ---- pass 2: TG bytes (or the tail) per instance row, 16 bytes per store; the two
    // halves of a 32-byte sector are stored back to back so they merge in L2
    if (STORE_POLICY >= 2 && TG == 32 && ALIGNED16 && ngrp == TG && nrows == 32 &&
        ((reinterpret_cast<uintptr_t>(dst) | pitch) & 31) == 0) {
        // whole 32-byte sectors in one store each
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t y[8][4];  // [g4][q]
#pragma unroll
            for (int g4 = 0; g4 < 8; ++g4) {
                uint32_t x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = col[((4 * g4 + u) * 8 + kk) * ts];
                bytes4x4(x, y[g4]);
            }
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const uint32_t v[8] = {y[0][qq], y[1][qq], y[2][qq], y[3][qq], y[4][qq], y[5][qq], y[6][qq], y[7][qq]};
                if constexpr (STORE_POLICY == 3) store32_line(dst + (uint64_t)(8 * qq + kk) * pitch, v);
                else store32_keep(dst + (uint64_t)(8 * qq + kk) * pitch, v);
            }
        }
    } else if (ALIGNED16 && ngrp == TG && nrows == 32) {
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll DRAIN_UNROLL_HALF
            for (int half = 0; half < TG / 16; ++half) {
                uint32_t y[4][4];  // [g4][q]
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) {
                    uint32_t x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) x[u] = col[((16 * half + 4 * g4 + u) * 8 + kk) * ts];
                    bytes4x4(x, y[g4]);
                }
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    store16<(STORE_POLICY != 0)>(dst + (uint64_t)(8 * qq + kk) * pitch + 16 * half,
                                              make_uint4(y[0][qq], y[1][qq], y[2][qq], y[3][qq]));
            }
        }
    } else {
        // ragged edge: short tail, partial last group or unaligned rows
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll 1
            for (int grp = 0; grp < ngrp; ++grp) {
                const uint32_t x = col[(grp * 8 + kk) * ts];
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    if ((uint64_t)(8 * qq + kk) < nrows)
                        dst[(uint64_t)(8 * qq + kk) * pitch + grp] = (uint8_t)(x >> (8 * qq));
            }
    }
}

template <bool ALIGNED16, int TG, int TS, bool LSB = false>
__global__ void __launch_bounds__(BLOCK, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                    unsigned long long *acc_out, uint8_t *__restrict__ out,
                    uint64_t pitch, uint64_t N, uint64_t G, uint64_t T, uint32_t chunk, uint32_t chunks_per_chain,
                    SchedQueue *q, unsigned long long *slots, uint32_t mask, uint32_t *progress, uint32_t chain_base)
{
    extern __shared__ uint32_t tile[];  // [8 * TG clocks][TS], TS >= blockDim.x
    constexpr uint32_t ts = TS;         // tile stride: consecutive threads -> consecutive banks
    uint32_t *col = tile + threadIdx.x;
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        // chains [chain_base, chain_base + n) are scheduled; `out` row 0 is the first instance of chain_base
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);
        const uint64_t c0 = (uint64_t)k * chunk;  // chunk is a multiple of 8 * TG clocks
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        if (g < G) {
            uint32_t r[NBITS], s[NBITS];
            unsigned long long a;
            load_state(state, acc, G, g, r, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
            const uint64_t nrows = N - 32 * g < 32 ? N - 32 * g : 32;  // rows of this group that exist

#pragma unroll 1
            for (uint64_t t0 = 0; t0 < tc; t0 += 8 * TG) {
                const int nclk = (tc - t0) >= 8 * TG ? 8 * TG : (int)(tc - t0);
                const int ngrp = nclk >> 3;
                uint32_t *zp = col;
                int t = 0;
                HalfSums hs;  // a tile is at most 256 words
                if constexpr (RBLOCK_ROW > 1) {
#pragma unroll 1
                    for (; t + RBLOCK_ROW <= nclk; t += RBLOCK_ROW) {
                        clock_block<RBLOCK_ROW, false, false, true>(r, s, NoInput{}, [&](auto kc, uint32_t z) {
                            zp[decltype(kc)::value * ts] = z;
#if MK2_ROW_SUM
                            hs.add(z);
#else
                            acc_add(a, z);
#endif
                        });
                        zp += RBLOCK_ROW * ts;
                    }
                }
#pragma unroll 1
                for (; t < nclk; ++t) {
                    const uint32_t z = keystream_word(r, s);
                    *zp = z;
                    zp += ts;
#if MK2_ROW_SUM
                    hs.add(z);
#else
                    acc_add(a, z);
#endif
                    clock<false, false>(r, s, 0u);
                }
                hs.fold(a);
                row_drain<ALIGNED16, TG, TS, LSB>(col, rows + (t0 >> 3), pitch, ngrp, nrows);
            }
            store_state(state_out, acc_out, G, g, r, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

// ---------------------------------------------------------------------------
// Checksum fold: sum_g acc[g] << (32 * ((g + g_offset) & 1))  mod 2^64, i.e. the
// column-major buffer of everything emitted so far, read as little-endian
// uint64 words and summed (the cross-GPU invariant of SURVEY.md 8(e)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK)
checksum_kernel(const unsigned long long *__restrict__ acc, uint64_t G, uint64_t g_offset,
                unsigned long long *__restrict__ result)
{
    unsigned long long v = 0;
    for (uint64_t g = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; g < G; g += (uint64_t)gridDim.x * BLOCK)
        v += acc[g] << (32 * ((g + g_offset) & 1));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(result, v);
}

// ---------------------------------------------------------------------------
// LOP3 issue-rate probe: the roofline denominator.  16
// independent non-linear chains per thread, nothing but LOP3 in the loop.
// lane-ops = threads * iters * 16 * UNROLL.
// ---------------------------------------------------------------------------
constexpr int PEAK_UNROLL = 16;
__global__ void __launch_bounds__(BLOCK)
lop3_peak_kernel(uint32_t *__restrict__ out, uint32_t seed, int iters)
{
    uint32_t x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = seed * (2654435761u + k) + threadIdx.x * (k + 1) + blockIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < PEAK_UNROLL; ++u) {
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = lop3<0x6A>(x[k], x[(k + 5) & 15], x[(k + 11) & 15]);  // c ^ (a & b)
        }
    }
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) v ^= x[k];
    if (v == 0x12345u) out[blockIdx.x * BLOCK + threadIdx.x] = v;  // practically never: keeps the chains live
}

}  // namespace mk2
