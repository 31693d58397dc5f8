// mk2_coop.cuh -- small batches: one WARP per 32-instance group, the 200 state bits spread over the lanes.
//
// The throughput kernels give a thread all 200 state words of its 32 instances: ~300 LOP3 per clock and thread,
// and a warp can issue one LOP3 every two cycles, so a clock takes 600 cycles however few of the warp's threads
// have a group.  That is the right shape when there are thousands of chains to overlap; it is the wrong one for
// the reference's own calling unit -- mickey_sliced_words on 64 lanes (kernels.py:189-200; cli.py:219-231 batches
// by 64) is two threads of one warp clocking serially: 1.4 ms for 4096 clocks on a GPU that is otherwise idle,
// where the reference's numba loop needs 0.3 ms.
//
// Here lane l of a warp owns positions 4l .. 4l+3 of R and of S (lanes 0..24; 25..31 ride along with zeros) of
// ONE group.  A clock is then 8 positions of work per lane instead of 200: the three neighbour words a lane needs
// (r[4l-1], s[4l-1], s[4l+4]) and the taps (r0^s0, s34^r67, s67^r33, r99, s99, s50) travel by warp shuffles.  The
// tables are no longer compile-time per position -- every lane runs the same instructions -- so they are five
// per-lane mask words per position, and a position costs 7 LOP3 (R 2, S 5) instead of ~3.  Per clock and warp:
// ~40 LOP3 + 11 shuffles, ~110 cycles instead of 600.  Same state layout in HBM (state[200][G], acc[G]) as every
// other kernel, so a context can be initialised here and continued by the throughput kernels or vice versa.
//
// Used by the launch planner for G <= COOP_MAX_GROUPS (mk2_api.cu; mk2_set_small_batch turns it off).
#pragma once
#include "mk2_kernels.cuh"

namespace mk2 {
namespace coop {

constexpr int PB = 4;               // positions per lane
constexpr int LANES = NBITS / PB;   // 25 lanes carry state
constexpr int WARPS = 4;            // warps per CTA: one per SM sub-partition
static_assert(NBITS % PB == 0, "whole lanes");
// which lane / slot holds a position
MK2_CX int lane_of(int pos) { return pos / PB; }
MK2_CX int slot_of(int pos) { return pos % PB; }

constexpr unsigned FULL = 0xFFFFFFFFu;
#ifndef MK2_COOP_UNROLL
#define MK2_COOP_UNROLL 8
#endif
constexpr int COOP_UNROLL = MK2_COOP_UNROLL;  // clocks per loop iteration: lets the next clock's shuffles overlap this clock's LOP3s

// Per-lane table words: all-ones where the lane's position k has the table bit set.
struct LaneTables {
    uint32_t taps[PB], c0[PB], c1[PB], f0[PB], f1[PB];
    uint32_t inner[PB];   // 1 <= position <= 98: the AND term of CLOCK_S exists (mickey.py:347-349)
    uint32_t first;       // all-ones in lanes > 0: the lane has a left neighbour
};
__device__ __forceinline__ LaneTables make_tables(unsigned lane)
{
    LaneTables t;
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        const int p = (int)lane * PB + k;
        const bool live = p < NBITS;
        const int q = live ? p : 0;
        t.taps[k] = live && tbit(T_RTAPS, q) ? FULL : 0u;
        t.c0[k] = live && tbit(T_COMP0, q) ? FULL : 0u;
        t.c1[k] = live && tbit(T_COMP1, q) ? FULL : 0u;
        t.f0[k] = live && tbit(T_FB0, q) ? FULL : 0u;
        t.f1[k] = live && tbit(T_FB1, q) ? FULL : 0u;
        t.inner[k] = live && p >= 1 && p <= 98 ? FULL : 0u;
    }
    t.first = lane > 0 ? FULL : 0u;
    return t;
}

// One CLOCK_KG (mickey.py:329-360) of the warp's group.  r[k] / s[k] = bit 4 lane + k of R / S for the 32
// instances; `in` = the input word (same in every lane).  Returns nothing: z is taken before the clock.
template <bool MIXING, bool INPUT>
__device__ __forceinline__ void clock(uint32_t (&r)[PB], uint32_t (&s)[PB], uint32_t in, const LaneTables &t, unsigned lane)
{
    // taps: each is a word of one lane, fetched by every lane
    const uint32_t s34 = __shfl_sync(FULL, s[slot_of(CTRL_R_S_TAP)], lane_of(CTRL_R_S_TAP));
    const uint32_t r67 = __shfl_sync(FULL, r[slot_of(CTRL_R_R_TAP)], lane_of(CTRL_R_R_TAP));
    const uint32_t s67 = __shfl_sync(FULL, s[slot_of(CTRL_S_S_TAP)], lane_of(CTRL_S_S_TAP));
    const uint32_t r33 = __shfl_sync(FULL, r[slot_of(CTRL_S_R_TAP)], lane_of(CTRL_S_R_TAP));
    const uint32_t r99 = __shfl_sync(FULL, r[slot_of(99)], lane_of(99));
    const uint32_t s99 = __shfl_sync(FULL, s[slot_of(99)], lane_of(99));
    // neighbours across the lane boundary (old values)
    const uint32_t r_left = __shfl_up_sync(FULL, r[PB - 1], 1) & t.first;   // position 0: nothing shifts in
    const uint32_t s_left = __shfl_up_sync(FULL, s[PB - 1], 1) & t.first;
    const uint32_t s_right = __shfl_down_sync(FULL, s[0], 1);               // lane 24, slot 3 = position 99: unused (inner = 0)
    const uint32_t ctrl_r = s34 ^ r67, ctrl_s = s67 ^ r33;
    uint32_t fb_r = r99, fb_s = s99;
    if constexpr (MIXING) fb_r ^= __shfl_sync(FULL, s[slot_of(MIXING_S_TAP)], lane_of(MIXING_S_TAP));
    if constexpr (INPUT) {
        fb_r ^= in;
        fb_s ^= in;
    }
    // ---- R: r'[i] = r[i-1] ^ (ctrl_r & r[i]) ^ (fb_r on RTAPS)                           mickey.py:338-343
    constexpr unsigned A_XOR_BC = (LA ^ (LB & LC)) & 0xFF;
    uint32_t nr[PB], ns[PB];
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        const uint32_t left = k == 0 ? r_left : r[k - 1];
        const uint32_t x = lop3<A_XOR_BC>(left, ctrl_r, r[k]);
        nr[k] = lop3<A_XOR_BC>(x, fb_r, t.taps[k]);
    }
    // ---- S: s'[i] = s[i-1] ^ ((s[i]^COMP0_i) & (s[i+1]^COMP1_i)) ^ fb_s & (ctrl_s ? FB1_i : FB0_i)   mickey.py:345-358
    constexpr unsigned XOR_AND = ((LA ^ LB) & LC) & 0xFF;        // (a ^ b) & c
    constexpr unsigned AND_XOR = ((LA & LB) ^ LC) & 0xFF;        // (a & b) ^ c
    constexpr unsigned MUX = ((LA & ~LC) | (LB & LC)) & 0xFF;    // c ? b : a
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        const uint32_t left = k == 0 ? s_left : s[k - 1];
        const uint32_t right = k == PB - 1 ? s_right : s[k + 1];
        const uint32_t g1 = s[k] ^ t.c0[k];
        const uint32_t g2 = lop3<XOR_AND>(right, t.c1[k], t.inner[k]);
        const uint32_t g3 = lop3<AND_XOR>(g1, g2, left);
        const uint32_t sel = lop3<MUX>(t.f0[k], t.f1[k], ctrl_s);
        ns[k] = lop3<A_XOR_BC>(g3, fb_s, sel);
    }
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        r[k] = nr[k];
        s[k] = ns[k];
    }
}

__device__ __forceinline__ void load_state(const uint32_t *state, uint64_t G, uint64_t g, unsigned lane, uint32_t (&r)[PB], uint32_t (&s)[PB])
{
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        const unsigned p = lane * PB + k;
        r[k] = p < NBITS ? __ldcg(state + (uint64_t)p * G + g) : 0u;
        s[k] = p < NBITS ? __ldcg(state + (uint64_t)(NBITS + p) * G + g) : 0u;
    }
}
__device__ __forceinline__ void store_state(uint32_t *state, uint64_t G, uint64_t g, unsigned lane, const uint32_t (&r)[PB], const uint32_t (&s)[PB])
{
#pragma unroll
    for (int k = 0; k < PB; ++k) {
        const unsigned p = lane * PB + k;
        if (p < NBITS) {
            state[(uint64_t)p * G + g] = r[k];
            state[(uint64_t)(NBITS + p) * G + g] = s[k];
        }
    }
}

// Key/IV load + pre-clocks (init_kernel<false>): input words mat[c][G] as written by the pack kernels.
__global__ void __launch_bounds__(32 * WARPS)
init_kernel(const uint32_t *__restrict__ mat, int load_clocks, uint64_t G, uint32_t *__restrict__ state,
            unsigned long long *__restrict__ acc)
{
    const unsigned lane = threadIdx.x & 31u;
    const LaneTables t = make_tables(lane);
    for (uint64_t g = (uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); g < G; g += (uint64_t)gridDim.x * WARPS) {
        uint32_t r[PB] = {0u, 0u, 0u, 0u}, s[PB] = {0u, 0u, 0u, 0u};
        // 32 input words at a time: lane j fetches the word of clock c0 + j, the clocks pick them up by shuffle
        for (int c0 = 0; c0 < load_clocks; c0 += 32) {
            const int n = load_clocks - c0 < 32 ? load_clocks - c0 : 32;
            const uint32_t mine = (int)lane < n ? __ldg(mat + (uint64_t)(c0 + lane) * G + g) : 0u;
#pragma unroll COOP_UNROLL
            for (int j = 0; j < n; ++j) clock<true, true>(r, s, __shfl_sync(FULL, mine, j), t, lane);
        }
#pragma unroll COOP_UNROLL
        for (int k = 0; k < PRECLOCKS; ++k) clock<true, false>(r, s, 0u, t, lane);
        store_state(state, G, g, lane, r, s);
        if (lane == 0) acc[g] = 0ull;
    }
}

// Column-major keystream (gen_colmajor_kernel): out[t][g] for t in [0, T); state and checksum carried on.
__global__ void __launch_bounds__(32 * WARPS)
gen_colmajor_kernel(uint32_t *__restrict__ state, unsigned long long *__restrict__ acc, uint32_t *__restrict__ out,
                    uint64_t stride, uint64_t G, uint64_t T)
{
    const unsigned lane = threadIdx.x & 31u;
    const LaneTables t = make_tables(lane);
    for (uint64_t g = (uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); g < G; g += (uint64_t)gridDim.x * WARPS) {
        uint32_t r[PB], s[PB];
        load_state(state, G, g, lane, r, s);
        unsigned long long sum = 0;
        uint32_t *o = out + g;
        for (uint64_t t0 = 0; t0 < T; t0 += 32) {
            const int n = T - t0 < 32 ? (int)(T - t0) : 32;
            uint32_t mine = 0;  // keystream word of clock t0 + lane
#pragma unroll COOP_UNROLL
            for (int j = 0; j < n; ++j) {
                const uint32_t z = __shfl_sync(FULL, r[0] ^ s[0], 0);   // z_t = r0 ^ s0, sampled before the clock (mickey.py:153-157)
                if ((int)lane == j) mine = z;
                clock<false, false>(r, s, 0u, t, lane);
            }
            if ((int)lane < n) {
                o[(t0 + lane) * stride] = mine;
                sum += mine;
            }
        }
        store_state(state, G, g, lane, r, s);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_down_sync(FULL, sum, d);
        if (lane == 0) acc[g] += sum;
    }
}

// 32 x 32 bit transpose across the warp: in: lane j holds word j; out: lane i holds column i (bit k = bit i of
// word k).  Five butterfly stages (the log-step half-block swaps of bitslab.py:183-200 with the partner word in
// another lane instead of another register).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, unsigned lane)
{
#pragma unroll
    for (int st = 4; st >= 0; --st) {
        const unsigned sh = 1u << st;
        const uint32_t m = st == 4 ? 0xFFFF0000u : st == 3 ? 0xFF00FF00u : st == 2 ? 0xF0F0F0F0u : st == 1 ? 0xCCCCCCCCu : 0xAAAAAAAAu;
        const uint32_t y = __shfl_xor_sync(FULL, x, sh);
        x = (lane & sh) ? ((x & m) | ((y & m) >> sh)) : ((x & ~m) | ((y & ~m) << sh));
    }
    return x;
}

// Row-major keystream (kernels.py:604-621 layout; tmem::gen_rowmajor_kernel for small batches): every 32 clocks
// the warp's 32 keystream words are bit-transposed across the lanes and lane i writes four bytes of instance
// 32 g + i's row.  T is a multiple of 8.  LSB: first bit in the least significant position of a byte.
template <bool LSB>
__global__ void __launch_bounds__(32 * WARPS)
gen_rowmajor_kernel(uint32_t *__restrict__ state, unsigned long long *__restrict__ acc, uint8_t *__restrict__ out, uint64_t pitch,
                    uint64_t N, uint64_t G, uint64_t T)
{
    const unsigned lane = threadIdx.x & 31u;
    const LaneTables t = make_tables(lane);
    const bool word_stores = ((reinterpret_cast<uintptr_t>(out) | pitch) & 3u) == 0;
    for (uint64_t g = (uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); g < G; g += (uint64_t)gridDim.x * WARPS) {
        uint32_t r[PB], s[PB];
        load_state(state, G, g, lane, r, s);
        unsigned long long sum = 0;
        const uint64_t row = 32 * g + lane;
        uint8_t *dst = out + row * pitch;
        for (uint64_t t0 = 0; t0 < T; t0 += 32) {
            const int n = T - t0 < 32 ? (int)(T - t0) : 32;
            uint32_t mine = 0;  // keystream word of clock t0 + lane
#pragma unroll COOP_UNROLL
            for (int j = 0; j < n; ++j) {
                const uint32_t z = __shfl_sync(FULL, r[0] ^ s[0], 0);
                if ((int)lane == j) mine = z;
                clock<false, false>(r, s, 0u, t, lane);
            }
            sum += mine;
            uint32_t w = warp_transpose32(mine, lane);  // bit k = z_{t0 + k} of instance 32 g + lane
            if (!LSB) w = __byte_perm(__brev(w), 0u, 0x0123);  // MSB-first bytes in ascending address order (bitops.py:20-23)
            if (row < N) {
                uint8_t *p = dst + (t0 >> 3);
                if (n == 32 && word_stores) {
                    *reinterpret_cast<uint32_t *>(p) = w;
                } else {
                    for (int b = 0; b < (n >> 3); ++b) p[b] = (uint8_t)(w >> (8 * b));
                }
            }
        }
        store_state(state, G, g, lane, r, s);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_down_sync(FULL, sum, d);
        if (lane == 0) acc[g] += sum;
    }
}

}  // namespace coop
}  // namespace mk2
