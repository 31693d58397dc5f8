// mk2_grain.cuh -- bitsliced Grain v1 (the paper's second stream cipher).
//
// Reference: pkg/src/slicerng/grain.py (engines), kernels.py:268-292 (compiled sliding-window
// loop).  One thread = 32 instances: b[i] / s[i] hold bit i of the 80-bit NFSR / LFSR.
// Both registers shift every clock, so unlike MICKEY the state MOVES: the kernel keeps a
// sliding window of 80 + WIN words per register in registers, runs WIN clocks against
// compile-time offsets and then realigns the window with WIN-position moves (the same
// amortised register swap as the reference's numba loop, kernels.py:268-287).  The moves
// are plain register copies, which ptxas issues on the otherwise idle FMA pipe, so the
// ALU pipe only sees the 38 LOP3s of f, g, h and z per clock.
//
//   f(s) = s62^s51^s38^s23^s13^s0                      grain.py:33-34
//   g(b) = 11 linear taps ^ 11 product terms           grain.py:36-52
//   h    = 5-input filter over s3,s25,s46,s64,b63      grain.py:54-56, 96-103
//   z    = h ^ b1^b2^b4^b10^b31^b43^b56                grain.py:58-59, 127-133
//   init: b = key bits, s = IV bits || ones, 160 clocks with z fed back into both (grain.py:147-156);
//   key / IV bits are taken LSB-first per byte (grain.py:88-92).
#pragma once
#include "mk2_kernels.cuh"

namespace mk2 {
namespace grain {

constexpr int GB = 80;           // bits per register (grain.py:29)
#ifndef MK2_GRAIN_STORE_POLICY
#define MK2_GRAIN_STORE_POLICY 3
#endif
constexpr int GRAIN_STORE_POLICY = MK2_GRAIN_STORE_POLICY;  // row stores: 1 = 2 x 16 B, 2 = 1 x 32 B, both L2 evict_last;
                                                            // 3 = 1 x 32 B, evict_last except for the sector that completes a 128-byte line
#ifndef MK2_GRAIN_ROW_FUSED_T
#define MK2_GRAIN_ROW_FUSED_T 1
#endif
constexpr int WIN = 16;          // clocks per window realignment
constexpr int GW = GB + WIN;     // window length
constexpr int INIT_CLOCKS = 160; // grain.py:30

// LOP3 truth tables used below (inputs a = 0xF0, b = 0xCC, c = 0xAA).
constexpr unsigned L_XOR3 = 0x96, L_XOR2 = 0x3C, L_AND2 = 0xC0, L_AND3 = 0x80, L_MAJ = 0xE8;
constexpr unsigned L_A_XOR_BC = 0x78;    // a ^ (b & c)
constexpr unsigned L_AXORB_AND_C = 0x28; // (a ^ b) & c

// One clock at window offset C: returns z, appends the two feedback words at C + 80.
// Hand-mapped onto 3-input LUTs: 38 LOP3 per clock (f 3, z 9, g 26); nvcc's own mapping of the
// textbook expressions (grain.py:96-117) needed 43.
//   h = A ^ x2 D with A = x1 ^ x4 ^ t, t = x3 (x0 ^ x4), D = t ^ x3 ^ MAJ(x0, x1, x4)   (Shannon on x2)
//   g = 12 linear taps ^ P1..P11 with the shared pairs b63b60, b37b33, b15b9, b52b45, b28b21; products
//       of three or more taps are reduced to a pair and folded in as acc ^ (p & q).
template <int C, bool INIT, int NW, bool CIRC = false>
__device__ __forceinline__ uint32_t step(uint32_t (&b)[NW], uint32_t (&s)[NW])
{
    // CIRC: the registers are a circular buffer of GB words (bit i at clock t lives in word (t + i) mod GB, the
    // feedback overwrites the word bit 0 leaves) instead of a sliding window: nothing ever has to be moved
    static_assert(CIRC ? (NW == GB && C < GB) : (C + GB < NW), "window too short for this offset");
    constexpr auto ix = [](int i) constexpr { return CIRC ? (C + i) % GB : C + i; };
    // ---- output z (grain.py:127-133)
    const uint32_t x0 = s[ix(3)], x1 = s[ix(25)], x2 = s[ix(46)], x3 = s[ix(64)], x4 = b[ix(63)];
    const uint32_t t = lop3<L_AXORB_AND_C>(x0, x4, x3);
    const uint32_t m = lop3<L_MAJ>(x0, x1, x4);
    const uint32_t D = lop3<L_XOR3>(t, x3, m);
    const uint32_t p1 = lop3<L_XOR3>(b[ix(1)], b[ix(2)], b[ix(4)]);
    const uint32_t p2 = lop3<L_XOR3>(b[ix(10)], b[ix(31)], b[ix(43)]);
    const uint32_t p3 = lop3<L_XOR3>(b[ix(56)], t, x1);
    const uint32_t p4 = lop3<L_XOR3>(p1, p2, x4);
    const uint32_t p5 = lop3<L_A_XOR_BC>(p3, x2, D);
    const uint32_t z = p4 ^ p5;
    // ---- LFSR feedback f (grain.py:120-124)
    const uint32_t f1 = lop3<L_XOR3>(s[ix(62)], s[ix(51)], s[ix(38)]);
    const uint32_t f2 = lop3<L_XOR3>(s[ix(23)], s[ix(13)], s[ix(0)]);
    // ---- NFSR feedback g ^ s0 (grain.py:106-117)
    const uint32_t P1 = b[ix(63)] & b[ix(60)], P2 = b[ix(37)] & b[ix(33)], P3 = b[ix(15)] & b[ix(9)];
    const uint32_t pa = b[ix(52)] & b[ix(45)], pc = b[ix(28)] & b[ix(21)];
    const uint32_t P5 = b[ix(33)] & pc;
    const uint32_t h6 = lop3<L_AND3>(b[ix(63)], b[ix(45)], b[ix(28)]);
    const uint32_t h7 = b[ix(60)] & b[ix(52)], h8 = b[ix(21)] & b[ix(15)], h9 = P1 & pa, h11 = pa & P2;
    const uint32_t l1 = lop3<L_XOR3>(s[ix(0)], b[ix(62)], b[ix(60)]);
    const uint32_t l2 = lop3<L_XOR3>(b[ix(52)], b[ix(45)], b[ix(37)]);
    const uint32_t l3 = lop3<L_XOR3>(b[ix(33)], b[ix(28)], b[ix(21)]);
    const uint32_t l4 = lop3<L_XOR3>(b[ix(14)], b[ix(9)], b[ix(0)]);
    const uint32_t l5 = lop3<L_XOR3>(P1, P2, P3);
    uint32_t accA = lop3<L_XOR3>(l1, l2, l3);
    uint32_t accB = lop3<L_XOR3>(l4, l5, P5);
    accA = lop3<L_A_XOR_BC>(accA, b[ix(60)], pa);  // P4  = b60 b52 b45
    accA = lop3<L_A_XOR_BC>(accA, h6, b[ix(9)]);   // P6  = b63 b45 b28 b9
    accA = lop3<L_A_XOR_BC>(accA, h7, P2);         // P7  = b60 b52 b37 b33
    accA = lop3<L_A_XOR_BC>(accA, h8, P1);         // P8  = b63 b60 b21 b15
    accB = lop3<L_A_XOR_BC>(accB, h9, b[ix(37)]);  // P9  = b63 b60 b52 b45 b37
    accB = lop3<L_A_XOR_BC>(accB, P5, P3);         // P10 = b33 b28 b21 b15 b9
    accB = lop3<L_A_XOR_BC>(accB, h11, pc);        // P11 = b52 b45 b37 b33 b28 b21
    uint32_t fl, fn;
    if (INIT) {  // z is fed back into both registers (grain.py:150-155)
        fl = lop3<L_XOR3>(f1, f2, z);
        fn = lop3<L_XOR3>(accA, accB, z);
    } else {
        fl = f1 ^ f2;
        fn = accA ^ accB;
    }
    s[ix(GB)] = fl;
    b[ix(GB)] = fn;
    return z;
}

template <int N, int NW>
__device__ __forceinline__ void realign(uint32_t (&b)[NW], uint32_t (&s)[NW])
{
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        b[i] = b[i + N];
        s[i] = s[i + N];
    }
}

// Realignment at the TOP of a window, through a copy ptxas cannot see through (an IMAD by a 1 read from constant
// memory).  A plain b[i] = b[i + WIN] is copy-propagated into its readers and left without successors in the
// loop body, so the list scheduler parks all ~160 moves behind the last LOP3 -- dead time for a warp that has its
// sub-partition to itself.  As real producers of the window's first operands they are issued where they are
// needed, between the LOP3s.  The state is then carried in words WIN .. WIN + 79 between windows.
#ifndef MK2_GRAIN_TOP
#define MK2_GRAIN_TOP 1
#endif
constexpr int OFF = MK2_GRAIN_TOP ? WIN : 0;  // where the state sits between two windows
// the column-major loop may use a longer window (it has registers to spare): half the copies per clock
#ifndef MK2_GRAIN_COL_WIN
#define MK2_GRAIN_COL_WIN 32
#endif
#ifndef MK2_GRAIN_ROW_WIN
#define MK2_GRAIN_ROW_WIN 16
#endif
constexpr int RWIN_ = MK2_GRAIN_ROW_WIN;      // window of the default row-major kernel (a divisor of 256, a multiple of 8)
constexpr int RGW_ = GB + RWIN_;
constexpr int ROFF_ = MK2_GRAIN_TOP ? RWIN_ : 0;
constexpr int CWIN = MK2_GRAIN_COL_WIN;
constexpr int CGW = GB + CWIN;
constexpr int COFF = MK2_GRAIN_TOP ? CWIN : 0;
__constant__ uint32_t opaque_one = 1u;
__device__ __forceinline__ uint32_t opaque_copy(uint32_t x)
{
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(d) : "r"(x), "r"(opaque_one));
    return d;
}
template <int W = WIN, int NW>
__device__ __forceinline__ void realign_top(uint32_t (&b)[NW], uint32_t (&s)[NW])
{
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        b[i] = opaque_copy(b[i + W]);
        s[i] = opaque_copy(s[i + W]);
    }
}
// window prologue / epilogue of the keystream loops, and the switch between the two conventions around a tail
template <int W = WIN, int NW>
__device__ __forceinline__ void window_begin(uint32_t (&b)[NW], uint32_t (&s)[NW])
{
    if constexpr (MK2_GRAIN_TOP) realign_top<W>(b, s);
}
template <int W = WIN, int NW>
__device__ __forceinline__ void window_end(uint32_t (&b)[NW], uint32_t (&s)[NW])
{
    if constexpr (!MK2_GRAIN_TOP) realign<W>(b, s);
}
template <int W = WIN, int NW>
__device__ __forceinline__ void tail_begin(uint32_t (&b)[NW], uint32_t (&s)[NW])  // state to words 0 .. 79
{
    if constexpr (MK2_GRAIN_TOP) realign<W>(b, s);
}
template <int W = WIN, int NW>
__device__ __forceinline__ void tail_end(uint32_t (&b)[NW], uint32_t (&s)[NW])  // and back to W .. W + 79
{
    if constexpr (MK2_GRAIN_TOP) {
#pragma unroll
        for (int i = GB - 1; i >= 0; --i) {
            b[i + W] = b[i];
            s[i + W] = s[i];
        }
    }
}

// Checksum accumulator of the Grain loops: HalfSums (two IDP.2A per word) or, with MK2_GRAIN_WIDESUM, ONE 64-bit
// multiply-add per word by a 1 read from constant memory (IMAD.WIDE; ptxas cannot turn it back into ALU-pipe adds).
#ifndef MK2_GRAIN_WIDESUM
#define MK2_GRAIN_WIDESUM 0
#endif
struct WideSum {
    unsigned long long v = 0;
    __device__ __forceinline__ void add(uint32_t z) { asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(v) : "r"(z), "r"(opaque_one)); }
    __device__ __forceinline__ void fold(unsigned long long &acc)
    {
        acc += v;
        v = 0;
    }
};
#if MK2_GRAIN_WIDESUM
using GrainSum = WideSum;
#else
using GrainSum = HalfSums;
#endif

template <int Lo, int Hi, class F>
__device__ __forceinline__ void static_for_up(F &&f)
{
    if constexpr (Lo < Hi) {
        f(std::integral_constant<int, Lo>{});
        static_for_up<Lo + 1, Hi>(f);
    }
}

// state[160][G]: words 0..79 = NFSR, 80..159 = LFSR (same coalesced layout as MICKEY's)
template <int O = 0, int NW>
__device__ __forceinline__ void load_state(const uint32_t *state, const unsigned long long *acc, uint64_t G, uint64_t g,
                                           uint32_t (&b)[NW], uint32_t (&s)[NW], unsigned long long &a)
{
    const uint32_t *p = state + g;
    constexpr int o = O;  // first state word: OFF in the sliding-window kernels of this file
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        b[o + i] = __ldcg(p);
        bump(p, G);
    }
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        s[o + i] = __ldcg(p);
        bump(p, G);
    }
    a = __ldcg(acc + g);
}
template <int O = 0, int NW>
__device__ __forceinline__ void store_state(uint32_t *state, unsigned long long *acc, uint64_t G, uint64_t g,
                                            const uint32_t (&b)[NW], const uint32_t (&s)[NW], unsigned long long a)
{
    const uint32_t *p = state + g;
    constexpr int o = O;  // first state word: OFF in the sliding-window kernels of this file
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        __stcg(const_cast<uint32_t *>(p), b[o + i]);
        bump(p, G);
    }
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        __stcg(const_cast<uint32_t *>(p), s[o + i]);
        bump(p, G);
    }
    st_release_u64(acc + g, a);
}

// ---------------------------------------------------------------------------
// Key/IV load + 160 init clocks (GrainSliced.from_key_ivs, grain.py:250-277).  The 32
// instances' key / IV bytes are transposed straight into the registers that ARE the
// initial state; the 16 top LFSR words are ones only in lanes that exist.
// ---------------------------------------------------------------------------
template <int NBYTES>
__device__ __forceinline__ void load_bits_lsb(const uint8_t *__restrict__ src, uint64_t first_row, uint64_t N,
                                              uint32_t *dst /* NBYTES * 8 words */)
{
#pragma unroll
    for (int p = 0; p < NBYTES; ++p) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t v = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t row = first_row + 8 * q + k;
                const uint32_t byte = row < N ? src[row * NBYTES + p] : 0u;
                v |= byte << (8 * q);
            }
            w[k] = v;
        }
        transpose8x32(w);  // w[bit] = bit `bit` of byte p across the 32 instances
#pragma unroll
        for (int m = 0; m < 8; ++m) dst[8 * p + m] = w[m];  // LSB-first: bit m of byte p is register bit 8p + m
    }
}

__global__ void __launch_bounds__(BLOCK, 1)
init_kernel(const uint8_t *__restrict__ keys, const uint8_t *__restrict__ ivs, uint64_t N, uint64_t G,
            uint32_t *__restrict__ state, unsigned long long *__restrict__ acc)
{
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= G) return;
    uint32_t b[GW], s[GW];
    load_bits_lsb<10>(keys, 32 * g, N, b);
    load_bits_lsb<8>(ivs, 32 * g, N, s);
    const uint64_t left = N - 32 * g;
    const uint32_t lanes = left >= 32 ? 0xFFFFFFFFu : ((1u << left) - 1u);
#pragma unroll
    for (int i = 64; i < GB; ++i) s[i] = lanes;
#pragma unroll 1
    for (int w = 0; w < INIT_CLOCKS / WIN; ++w) {
        static_for_up<0, WIN>([&](auto ic) { (void)step<decltype(ic)::value, true>(b, s); });
        realign<WIN>(b, s);
    }
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        state[(uint64_t)i * G + g] = b[i];
        state[(uint64_t)(GB + i) * G + g] = s[i];
    }
    acc[g] = 0ull;
}

// ---------------------------------------------------------------------------
// Keystream kernels: same persistent chain / chunk scheduler as MICKEY's.  `chunk` is a
// multiple of WIN (column-major) or of the staging tile (row-major); only the very last
// chunk of a chain can end in a tail of < WIN clocks, run one clock at a time.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK, 1)
gen_colmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                    unsigned long long *acc_out, uint32_t *__restrict__ out, uint64_t stride, uint64_t G, uint64_t T,
                    uint32_t chunk, uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask,
                    uint32_t *progress)
{
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)chain * 32 + (threadIdx.x & 31u);
        const uint64_t t0 = (uint64_t)k * chunk;
        const uint64_t tc = T - t0 < chunk ? T - t0 : chunk;
        if (g < G) {
            uint32_t b[CGW], s[CGW];
            unsigned long long a;
            load_state<COFF>(state, acc, G, g, b, s, a);
#ifndef MK2_GRAIN_COL_FMA
#define MK2_GRAIN_COL_FMA 1
#endif
#if MK2_GRAIN_COL_FMA
            // Output addressing and checksum off the ALU pipe (a 64-bit pointer bump and a 64-bit accumulate are
            // 3 of 40 ALU-pipe instructions per clock here): 64-bit base + 32-bit element index (IMAD.WIDE, the
            // index lives on the uniform datapath) and IDP.2A half sums; segments of < 2^32 elements, <= 65536 words.
            uint32_t *base = out + t0 * stride + g;
            const uint32_t stride32 = (uint32_t)stride;  // host side guarantees stride < 2^30
            uint32_t seg_max = 0xFFFFFFFFu / stride32;
            if (seg_max > HALFSUM_MAX_WORDS) seg_max = HALFSUM_MAX_WORDS;
            if (seg_max > CWIN) seg_max -= seg_max % CWIN;
            uint64_t t = 0;
#pragma unroll 1
            while (t < tc) {
                const uint32_t nseg = tc - t < seg_max ? (uint32_t)(tc - t) : seg_max;
                uint32_t idx = 0, u = 0;
                GrainSum hs;
#pragma unroll 1
                for (; u + CWIN <= nseg; u += CWIN) {
                    window_begin<CWIN>(b, s);
                    static_for_up<0, CWIN>([&](auto ic) {
                        const uint32_t z = step<decltype(ic)::value, false>(b, s);
                        base[idx] = z;
                        idx += stride32;
                        hs.add(z);
                    });
                    window_end<CWIN>(b, s);
                }
                if (u < nseg) {
                    tail_begin<CWIN>(b, s);
#pragma unroll 1
                    for (; u < nseg; ++u) {
                        const uint32_t z = step<0, false>(b, s);
                        base[idx] = z;
                        idx += stride32;
                        hs.add(z);
                        realign<1>(b, s);
                    }
                    tail_end<CWIN>(b, s);
                }
                hs.fold(a);
                base += (uint64_t)nseg * stride;
                t += nseg;
            }
#else
            uint32_t *p = out + t0 * stride + g;
            uint64_t t = 0;
#pragma unroll 1
            for (; t + CWIN <= tc; t += CWIN) {
                window_begin<CWIN>(b, s);
                static_for_up<0, CWIN>([&](auto ic) {
                    const uint32_t z = step<decltype(ic)::value, false>(b, s);
                    *p = z;
                    p += stride;
                    acc_add(a, z);
                });
                window_end<CWIN>(b, s);
            }
            if (t < tc) {
                tail_begin<CWIN>(b, s);
#pragma unroll 1
                for (; t < tc; ++t) {
                    const uint32_t z = step<0, false>(b, s);
                    *p = z;
                    p += stride;
                    acc_add(a, z);
                    realign<1>(b, s);
                }
                tail_end<CWIN>(b, s);
            }
#endif
            store_state<COFF>(state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

// ---------------------------------------------------------------------------
// Circular-buffer clocking: 80 words per register and NO realignment.  Clock t at compile-time phase
// P = t mod 80 reads word (P + tap) mod 80 and overwrites word P, so the loop body is five 16-clock segments
// (phases 0, 16, .. 64) dispatched by a slot counter; a chunk may stop after any segment and the state is
// parked from the rotation it is left in.  What it buys: the 164 register moves per 16 clocks of the sliding
// window are gone (a lone warp per sub-partition cannot overlap them with its LOP3s) and 32 registers are
// free.  What it costs: a 5 x longer body (instruction cache).
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void store_state_rot(uint32_t *state, unsigned long long *acc, uint64_t G, uint64_t g,
                                                const uint32_t (&b)[GB], const uint32_t (&s)[GB], unsigned long long a)
{
    const uint32_t *p = state + g;
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        __stcg(const_cast<uint32_t *>(p), b[(R + i) % GB]);
        bump(p, G);
    }
#pragma unroll
    for (int i = 0; i < GB; ++i) {
        __stcg(const_cast<uint32_t *>(p), s[(R + i) % GB]);
        bump(p, G);
    }
    st_release_u64(acc + g, a);
}
__device__ __forceinline__ void store_state_slot(uint32_t slot, uint32_t *state, unsigned long long *acc, uint64_t G, uint64_t g,
                                                 const uint32_t (&b)[GB], const uint32_t (&s)[GB], unsigned long long a)
{
    switch (slot) {
    case 0: store_state_rot<0>(state, acc, G, g, b, s, a); break;
    case 1: store_state_rot<16>(state, acc, G, g, b, s, a); break;
    case 2: store_state_rot<32>(state, acc, G, g, b, s, a); break;
    case 3: store_state_rot<48>(state, acc, G, g, b, s, a); break;
    default: store_state_rot<64>(state, acc, G, g, b, s, a); break;
    }
}

// Column-major keystream on the circular buffer (T a multiple of 16 clocks).
__global__ void __launch_bounds__(BLOCK, 1)
gen_colmajor_circ_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                         unsigned long long *acc_out, uint32_t *__restrict__ out, uint64_t stride, uint64_t G, uint64_t T,
                         uint32_t chunk, uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots, uint32_t mask,
                         uint32_t *progress)
{
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)chain * 32 + (threadIdx.x & 31u);
        const uint64_t t0 = (uint64_t)k * chunk;
        const uint64_t tc = T - t0 < chunk ? T - t0 : chunk;
        if (g < G) {
            uint32_t b[GB], s[GB];
            unsigned long long a;
            load_state(state, acc, G, g, b, s, a);
            uint32_t *base = out + t0 * stride + g;
            const uint32_t stride32 = (uint32_t)stride;  // host side guarantees stride < 2^30
            uint32_t seg_max = 0xFFFFFFFFu / stride32;
            if (seg_max > HALFSUM_MAX_WORDS) seg_max = HALFSUM_MAX_WORDS;
            seg_max -= seg_max % WIN;
            uint32_t slot = 0;
            uint64_t t = 0;
#pragma unroll 1
            while (t < tc) {
                const uint32_t nseg = tc - t < seg_max ? (uint32_t)(tc - t) : seg_max;
                uint32_t idx = 0;
                GrainSum hs;
                auto seg = [&](auto pc) {
                    static_for_up<0, WIN>([&](auto ic) {
                        const uint32_t z = step<decltype(pc)::value + decltype(ic)::value, false, GB, true>(b, s);
                        base[idx] = z;
                        idx += stride32;
                        hs.add(z);
                    });
                };
#pragma unroll 1
                for (uint32_t left = nseg / WIN; left; --left) {
                    switch (slot) {
                    case 0: seg(std::integral_constant<int, 0>{}); break;
                    case 1: seg(std::integral_constant<int, 16>{}); break;
                    case 2: seg(std::integral_constant<int, 32>{}); break;
                    case 3: seg(std::integral_constant<int, 48>{}); break;
                    default: seg(std::integral_constant<int, 64>{}); break;
                    }
                    slot = slot == 4 ? 0 : slot + 1;
                }
                hs.fold(a);
                base += (uint64_t)nseg * stride;
                t += nseg;
            }
            store_state_slot(slot, state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

template <bool ALIGNED16, int TG, int TS, bool LSB>
__global__ void __launch_bounds__(BLOCK, 1)
gen_rowmajor_kernel(const uint32_t *state, const unsigned long long *acc, uint32_t *state_out,
                    unsigned long long *acc_out, uint8_t *__restrict__ out, uint64_t pitch, uint64_t N, uint64_t G,
                    uint64_t T, uint32_t chunk, uint32_t chunks_per_chain, SchedQueue *q, unsigned long long *slots,
                    uint32_t mask, uint32_t *progress, uint32_t chain_base)
{
    extern __shared__ uint32_t tile[];  // [8 * TG clocks][TS]
    constexpr uint32_t ts = TS;
    uint32_t *col = tile + threadIdx.x;
    uint32_t chain;
    while (sched_pop(q, slots, mask, chain)) {
        const uint32_t k = __ldcg(progress + chain);
        const uint64_t g = (uint64_t)(chain_base + chain) * 32 + (threadIdx.x & 31u);
        const uint64_t c0 = (uint64_t)k * chunk;
        const uint64_t tc = T - c0 < chunk ? T - c0 : chunk;
        if (g < G) {
            uint32_t b[RGW_], s[RGW_];
            unsigned long long a;
            load_state<ROFF_>(state, acc, G, g, b, s, a);
            uint8_t *rows = out + 32 * (g - (uint64_t)chain_base * 32) * pitch + (c0 >> 3);
            const uint64_t nrows = N - 32 * g < 32 ? N - 32 * g : 32;
#pragma unroll 1
            for (uint64_t t0 = 0; t0 < tc; t0 += 8 * TG) {
                const int nclk = (tc - t0) >= 8 * TG ? 8 * TG : (int)(tc - t0);  // a multiple of 8
                uint32_t *zp = col;
                int t = 0;
                GrainSum hs;  // checksum on the FMA pipe; a tile is at most 256 words
#if MK2_GRAIN_ROW_FUSED_T
                if (nclk == 8 * TG) {
                    // full tile: the 8 x 32 bit transposes run in registers on each 8-clock group as it is
                    // produced, so the drain has no load / transpose / store pass over the tile
#pragma unroll 1
                    for (; t < nclk; t += RWIN_) {
                        window_begin<RWIN_>(b, s);
                        uint32_t zz[RWIN_];
                        static_for_up<0, RWIN_>([&](auto ic) {
                            constexpr int c = decltype(ic)::value;
                            zz[c] = step<c, false>(b, s);
                            hs.add(zz[c]);
                        });
#pragma unroll
                        for (int h = 0; h < RWIN_ / 8; ++h) {
                            uint32_t z[8];
#pragma unroll
                            for (int m = 0; m < 8; ++m) z[LSB ? m : 7 - m] = zz[8 * h + m];
                            transpose8x32(z);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk) zp[(8 * h + kk) * ts] = z[kk];
                        }
                        zp += RWIN_ * ts;
                        window_end<RWIN_>(b, s);
                    }
                    hs.fold(a);
                    row_drain<ALIGNED16, TG, TS, LSB, GRAIN_STORE_POLICY, true>(col, rows + (t0 >> 3), pitch, nclk >> 3, nrows);
                    continue;
                }
#endif
#pragma unroll 1
                for (; t + RWIN_ <= nclk; t += RWIN_) {
                    window_begin<RWIN_>(b, s);
                    static_for_up<0, RWIN_>([&](auto ic) {
                        constexpr int c = decltype(ic)::value;
                        const uint32_t z = step<c, false>(b, s);
                        zp[c * ts] = z;
                        hs.add(z);
                    });
                    zp += RWIN_ * ts;
                    window_end<RWIN_>(b, s);
                }
                if (t < nclk) {
                    tail_begin<RWIN_>(b, s);
#pragma unroll 1
                    for (; t < nclk; ++t) {
                        const uint32_t z = step<0, false>(b, s);
                        *zp = z;
                        zp += ts;
                        hs.add(z);
                        realign<1>(b, s);
                    }
                    tail_end<RWIN_>(b, s);
                }
                hs.fold(a);
                row_drain<ALIGNED16, TG, TS, LSB, GRAIN_STORE_POLICY>(col, rows + (t0 >> 3), pitch, nclk >> 3, nrows);
            }
            store_state<ROFF_>(state_out, acc_out, G, g, b, s, a);
        }
        sched_push(q, slots, mask, progress, chain, k + 1, chunks_per_chain);
    }
}

}  // namespace grain
}  // namespace mk2
