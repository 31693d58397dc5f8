// mk2_bits.cuh -- bit-matrix helpers of the key/IV packing kernels.
//
// Host-compilable like mk2_clock.cuh (tests/host_clock_check.cpp evaluates the same template code in
// software, so the ragged packing can be checked without a GPU); the product only runs the device build.
#pragma once
#include <cstdint>

#include "mk2_clock.cuh"

namespace mk2 {

MK2_HD uint32_t bit_reverse(uint32_t x)
{
#ifdef __CUDA_ARCH__
    return __brev(x);
#else
    uint32_t r = 0;
    for (int i = 0; i < 32; ++i) r |= ((x >> i) & 1u) << (31 - i);
    return r;
#endif
}

// bytes 0..3 of x are indices 0..3, bytes of y indices 4..7; result byte i = index nibble i of sel
MK2_HD uint32_t byte_pick(uint32_t x, uint32_t y, uint32_t sel)
{
#ifdef __CUDA_ARCH__
    return __byte_perm(x, y, sel);
#else
    const uint64_t v = ((uint64_t)y << 32) | x;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)((v >> (8 * ((sel >> (4 * i)) & 7u))) & 0xFFu) << (8 * i);
    return r;
#endif
}

// 32 x 32 bit-matrix transpose in place: afterwards bit j of a[b] is the old bit b of a[j].
// Five half-block swap stages, the scheme of the reference's _square_transpose
// (pkg/src/slicerng/bitslab.py:183-200); every index is a compile-time constant.
template <int J, uint32_t M>
MK2_HD void transpose32_stage(uint32_t (&a)[32])
{
    static_for_up<0, 31>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr ((k & J) == 0) {
            const uint32_t t = ((a[k] >> J) ^ a[k + J]) & M;
            a[k] ^= t << J;
            a[k + J] ^= t;
        }
    });
}
MK2_HD void transpose32(uint32_t (&a)[32])
{
    transpose32_stage<16, 0x0000FFFFu>(a);
    transpose32_stage<8, 0x00FF00FFu>(a);
    transpose32_stage<4, 0x0F0F0F0Fu>(a);
    transpose32_stage<2, 0x33333333u>(a);
    transpose32_stage<1, 0x55555555u>(a);
}

MK2_HD uint32_t low_mask(int n) { return n >= 32 ? 0xFFFFFFFFu : n <= 0 ? 0u : (1u << n) - 1u; }

// One lane of a group with ragged IV lengths (mickey.py:287-289 gives such lanes a per-lane scalar init;
// here they stay bitsliced).  The lane's IV is b0 b1 b2 (big-endian: IV byte 0 in the top byte of b0, bytes
// 8, 9 in the top half of b2), L its bit length (0..80, or > 80 for an unused lane).  The group clocks
// lmax IV-phase clocks; this lane idles in the all-zero state for start = lmax - L clocks and then loads
// its L bits, so that every lane reaches the key phase together.  Returns word k (clocks 32 k .. 32 k + 31,
// clock c in bit c % 32) of the lane's input bit string and of its activity string (bit c set from the
// lane's first load clock on).
MK2_HD void ragged_lane_words(uint32_t b0, uint32_t b1, uint32_t b2, int L, int lmax, int k, uint32_t &in_k, uint32_t &act_k)
{
    if (L > 80) {
        in_k = act_k = 0u;
        return;
    }
    const uint32_t w0 = bit_reverse(b0) & low_mask(L), w1 = bit_reverse(b1) & low_mask(L - 32),
                   w2 = bit_reverse(b2) & low_mask(L - 64);  // IV bit c in bit c % 32 of word c / 32
    const int start = lmax - L, ws = start >> 5, bs = start & 31;
    // (w2 : w1 : w0) << start, word k of the result; nothing falls off the top because L + start = lmax <= 80
    const int src = k - ws;  // word of the unshifted string that lands in word k (with its lower neighbour)
    const uint32_t hi = src == 0 ? w0 : src == 1 ? w1 : src == 2 ? w2 : 0u;
    const uint32_t lo = src == 1 ? w0 : src == 2 ? w1 : src == 3 ? w2 : 0u;
    in_k = bs ? (hi << bs) | (lo >> (32 - bs)) : hi;
    act_k = low_mask(lmax - 32 * k) & ~low_mask(start - 32 * k);
}

// byte_pick selector: the four bytes starting at byte `sh` of the pair, as a big-endian word
MK2_CX uint32_t be_sel(int sh) { return (uint32_t)((sh + 3) | ((sh + 2) << 4) | ((sh + 1) << 8) | (sh << 12)); }

// The fast path of pack_ragged_kernel for one complete group: rec[] = the group's 32 IV records of 10
// bytes (320 bytes as 80 little-endian words), len[] = the 32 bit lengths packed four per word.  Produces
// the 32 input words and 32 activity words of clocks 32 k .. 32 k + 31 (index = clock % 32).
MK2_HD void ragged_group_words(const uint32_t (&rec)[80], const uint32_t (&len)[8], int lmax, int k, uint32_t (&in)[32],
                               uint32_t (&act)[32])
{
    static_for_up<0, 31>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        constexpr int o = 10 * j;  // byte offset of lane j's record
        // big-endian words: result byte 3 = record byte 0, ...
        constexpr int i0 = o >> 2, s0 = o & 3, i1 = (o + 4) >> 2, s1 = (o + 4) & 3, i2 = (o + 8) >> 2, s2 = (o + 8) & 3;
        const uint32_t b0 = byte_pick(rec[i0], rec[i0 + 1 < 80 ? i0 + 1 : 79], be_sel(s0));
        const uint32_t b1 = byte_pick(rec[i1], rec[i1 + 1 < 80 ? i1 + 1 : 79], be_sel(s1));
        // bytes 8, 9 -> top half; the two low bytes are whatever follows in memory (masked away: L <= 80)
        const uint32_t b2 = byte_pick(rec[i2], rec[i2 + 1 < 80 ? i2 + 1 : 79], be_sel(s2));
        static_assert(s0 <= 2 && s1 <= 2 && s2 <= 2, "10-byte records start at even offsets");
        const int L = (int)((len[j >> 2] >> (8 * (j & 3))) & 0xFFu);
        ragged_lane_words(b0, b1, b2, L, lmax, k, in[j], act[j]);
    });
    transpose32(in);
    transpose32(act);
}

}  // namespace mk2
