// mk2_clock.cuh -- the bitsliced MICKEY 2.0 clock as straight-line LOP3 code.
//
// One thread owns 32 independent MICKEY 2.0 instances in column-major form:
// r[i] / s[i] hold bit i of the 100-bit R / S registers of those 32 instances
// (lane j of the word = instance j), the layout of the reference's
// MickeySliced engine (pkg/src/slicerng/mickey.py:236-243, bitslab.py:3-6).
//
// clock<MIXING, INPUT>() is the word form of CLOCK_KG
// (pkg/src/slicerng/mickey.py:329-360), re-derived for a 3-input-LUT machine:
//   * every table (RTAPS, COMP0, COMP1, FB0, FB1; mickey.py:35-39) is a
//     compile-time predicate of the position, so it costs no instruction and
//     no register: it only selects the LOP3 truth table / whether an XOR exists;
//   * both registers are updated IN PLACE (R from position 99 down; S likewise
//     with one carried word), so the "shift" is pure register renaming;
//   * per clock: R = 149 LOP3, S = 174, control = 4, z = 1.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>

namespace mk2 {

constexpr int NBITS = 100;      // mickey.py:31 STATE_BITS
constexpr int PRECLOCKS = 100;  // mickey.py:32
constexpr int KEY_BITS = 80;

// Packed tables: bit i = word i/32, bit i%32 (mickey.py:35-39).
enum Table { T_RTAPS = 0, T_COMP0, T_COMP1, T_FB0, T_FB1 };

__host__ __device__ constexpr uint32_t table_word(int tab, int w)
{
    switch (tab * 4 + w) {
    case 0: return 0x1279327Bu; case 1: return 0xB5546660u; case 2: return 0xDF87818Fu; case 3: return 0x00000003u;
    case 4: return 0x6AA97A30u; case 5: return 0x7942A809u; case 6: return 0x057EBFEAu; case 7: return 0x00000006u;
    case 8: return 0xDD629E9Au; case 9: return 0xE3A21D63u; case 10: return 0x91C23DD7u; case 11: return 0x00000001u;
    case 12: return 0x9FFA7FAFu; case 13: return 0xAF4A9381u; case 14: return 0x9CEC5802u; case 15: return 0x00000001u;
    case 16: return 0x4C8CB877u; case 17: return 0x4911B063u; case 18: return 0x40FBC52Bu; case 19: return 0x00000008u;
    default: return 0u;
    }
}
__host__ __device__ constexpr bool tbit(int tab, int i) { return (table_word(tab, i >> 5) >> (i & 31)) & 1u; }

// tap positions (mickey.py:42-46)
constexpr int CTRL_R_S_TAP = 34, CTRL_R_R_TAP = 67, CTRL_S_S_TAP = 67, CTRL_S_R_TAP = 33, MIXING_S_TAP = 50;

// ---- LOP3 with a compile-time truth table (a = 0xF0, b = 0xCC, c = 0xAA) ----
template <unsigned LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}
constexpr unsigned LA = 0xF0, LB = 0xCC, LC = 0xAA;
constexpr unsigned LUT_XOR3 = (LA ^ LB ^ LC) & 0xFF;        // a ^ b ^ c
constexpr unsigned LUT_A_XOR_BC = (LA ^ (LB & LC)) & 0xFF;  // a ^ (b & c)
constexpr unsigned LUT_A_AND_NOT_B = (LA & ~LB) & 0xFF;     // a & ~b (c ignored)
// S-hat truth table for position i: a ^ ((b ^ COMP0_i) & (c ^ COMP1_i))
__host__ __device__ constexpr unsigned shat_lut(int i)
{
    return (LA ^ ((LB ^ (tbit(T_COMP0, i) ? 0xFFu : 0u)) & (LC ^ (tbit(T_COMP1, i) ? 0xFFu : 0u)))) & 0xFF;
}

// compile-time descending loop: f(integral_constant<int, I>) for I = Hi .. Lo
template <int Hi, int Lo, class F>
__device__ __forceinline__ void static_for_down(F &&f)
{
    if constexpr (Hi >= Lo) {
        f(std::integral_constant<int, Hi>{});
        static_for_down<Hi - 1, Lo>(f);
    }
}

// One CLOCK_KG of 32 instances.  MIXING: mickey.py:334 (input_r ^= s[50]);
// INPUT: whether an input word is injected (key/IV load) or is zero.
template <bool MIXING, bool INPUT>
__device__ __forceinline__ void clock(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], uint32_t in)
{
    // control words (mickey.py:332-333)
    const uint32_t ctrl_r = s[CTRL_R_S_TAP] ^ r[CTRL_R_R_TAP];
    const uint32_t ctrl_s = s[CTRL_S_S_TAP] ^ r[CTRL_S_R_TAP];
    // feedback words (mickey.py:336, 345)
    uint32_t fb_r, fb_s;
    if constexpr (MIXING && INPUT) fb_r = lop3<LUT_XOR3>(r[99], s[MIXING_S_TAP], in);
    else if constexpr (MIXING) fb_r = r[99] ^ s[MIXING_S_TAP];
    else if constexpr (INPUT) fb_r = r[99] ^ in;
    else fb_r = r[99];
    if constexpr (INPUT) fb_s = s[99] ^ in;
    else fb_s = s[99];
    const uint32_t fb1 = fb_s & ctrl_s;   // FB1-only positions (mickey.py:351)
    const uint32_t fb0 = fb_s & ~ctrl_s;  // FB0-only positions (mickey.py:352)

    // ---- R: r'[i] = r[i-1] ^ (ctrl_r & r[i]) (^ fb_r on RTAPS) ; mickey.py:338-343
    static_for_down<99, 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        uint32_t t = lop3<LUT_A_XOR_BC>(r[i - 1], ctrl_r, r[i]);
        if constexpr (tbit(T_RTAPS, i)) t ^= fb_r;
        r[i] = t;
    });
    static_assert(tbit(T_RTAPS, 0), "position 0 is an R tap");
    r[0] = lop3<LUT_A_XOR_BC>(fb_r, ctrl_r, r[0]);

    // ---- S: s'[i] = s[i-1] ^ ((s[i]^COMP0_i) & (s[i+1]^COMP1_i)) ^ FB ; mickey.py:346-358
    auto fbmix = [&](auto ic, uint32_t t) -> uint32_t {
        constexpr int i = decltype(ic)::value;
        constexpr bool f0 = tbit(T_FB0, i), f1 = tbit(T_FB1, i);
        if constexpr (f0 && f1) return t ^ fb_s;
        else if constexpr (f0) return t ^ fb0;
        else if constexpr (f1) return t ^ fb1;
        else return t;
    };
    uint32_t up = s[99];  // old s[i+1] carried down the in-place sweep
    s[99] = fbmix(std::integral_constant<int, 99>{}, s[98]);
    static_for_down<98, 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const uint32_t t = lop3<shat_lut(i)>(s[i - 1], s[i], up);
        up = s[i];
        s[i] = fbmix(ic, t);
    });
    s[0] = fbmix(std::integral_constant<int, 0>{}, 0u);
}

// keystream word z_t = r0 ^ s0, sampled before the clock (mickey.py:365-367)
__device__ __forceinline__ uint32_t keystream_word(const uint32_t (&r)[NBITS], const uint32_t (&s)[NBITS])
{
    return r[0] ^ s[0];
}

}  // namespace mk2
