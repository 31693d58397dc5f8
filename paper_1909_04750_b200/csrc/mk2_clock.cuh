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
//
// clock_block<K, ...>() runs K clocks with R's feedback DEFERRED (see below):
// R costs (100 + k) LOP3 in clock k of the block plus one ~93-LOP3 reduction
// per block instead of 149 per clock -- 126 per clock at K = 4.
//
// The header also compiles as plain host C++ (tests/host_clock_check.cpp): the
// truth tables are then evaluated in software.  That build exists only so the
// test suite can check the template code without a GPU; the product library
// never runs it.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>

#ifndef __CUDACC__
#define MK2_HD inline
#else
#define MK2_HD __host__ __device__ __forceinline__
#endif
#ifdef __CUDACC__
#define MK2_CX __host__ __device__ constexpr
#else
#define MK2_CX constexpr
#endif

namespace mk2 {

constexpr int NBITS = 100;      // mickey.py:31 STATE_BITS
constexpr int PRECLOCKS = 100;  // mickey.py:32
constexpr int KEY_BITS = 80;

// Packed tables: bit i = word i/32, bit i%32 (mickey.py:35-39).
enum Table { T_RTAPS = 0, T_COMP0, T_COMP1, T_FB0, T_FB1 };

MK2_CX uint32_t table_word(int tab, int w)
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
MK2_CX bool tbit(int tab, int i) { return (table_word(tab, i >> 5) >> (i & 31)) & 1u; }

// tap positions (mickey.py:42-46)
constexpr int CTRL_R_S_TAP = 34, CTRL_R_R_TAP = 67, CTRL_S_S_TAP = 67, CTRL_S_R_TAP = 33, MIXING_S_TAP = 50;

// ---- LOP3 with a compile-time truth table (a = 0xF0, b = 0xCC, c = 0xAA) ----
template <unsigned LUT>
MK2_HD uint32_t lop3(uint32_t a, uint32_t b, uint32_t c)
{
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
#else
    uint32_t d = 0;  // host check build: evaluate the truth table minterm by minterm
    for (unsigned m = 0; m < 8; ++m)
        if ((LUT >> m) & 1u) d |= ((m & 4u) ? a : ~a) & ((m & 2u) ? b : ~b) & ((m & 1u) ? c : ~c);
    return d;
#endif
}
constexpr unsigned LA = 0xF0, LB = 0xCC, LC = 0xAA;
constexpr unsigned LUT_XOR3 = (LA ^ LB ^ LC) & 0xFF;        // a ^ b ^ c
constexpr unsigned LUT_A_XOR_BC = (LA ^ (LB & LC)) & 0xFF;  // a ^ (b & c)
constexpr unsigned LUT_A_AND_NOT_B = (LA & ~LB) & 0xFF;     // a & ~b (c ignored)
// S-hat truth table for position i: a ^ ((b ^ COMP0_i) & (c ^ COMP1_i))
MK2_CX unsigned shat_lut(int i)
{
    return (LA ^ ((LB ^ (tbit(T_COMP0, i) ? 0xFFu : 0u)) & (LC ^ (tbit(T_COMP1, i) ? 0xFFu : 0u)))) & 0xFF;
}

// compile-time descending loop: f(integral_constant<int, I>) for I = Hi .. Lo
template <int Hi, int Lo, class F>
MK2_HD void static_for_down(F &&f)
{
    if constexpr (Hi >= Lo) {
        f(std::integral_constant<int, Hi>{});
        static_for_down<Hi - 1, Lo>(f);
    }
}
// ascending: f(integral_constant<int, I>) for I = Lo .. Hi
template <int Lo, int Hi, class F>
MK2_HD void static_for_up(F &&f)
{
    if constexpr (Lo <= Hi) {
        f(std::integral_constant<int, Lo>{});
        static_for_up<Lo + 1, Hi>(f);
    }
}

// Positions where an all-zero lane does NOT stay all-zero under a zero-input clock: with s = 0 and no
// feedback, s'[i] = COMP0_i & COMP1_i.  Everything else of CLOCK_KG maps the zero state to itself (R is
// linear, the control and feedback bits are state bits), so a lane can be held in the zero state by
// masking these positions only.
MK2_CX bool zero_leak(int i) { return i >= 1 && i <= 98 && tbit(T_COMP0, i) && tbit(T_COMP1, i); }
MK2_CX int zero_leak_extra_ops()
{
    int n = 0;  // leak positions without a feedback XOR to fold the mask into
    for (int i = 1; i <= 98; ++i) n += (zero_leak(i) && !tbit(T_FB0, i) && !tbit(T_FB1, i)) ? 1 : 0;
    return n;
}

// CLOCK_S of 32 instances, in place (mickey.py:345-358).  fb0 / fb1 are fb_s masked by
// ~ctrl_s / ctrl_s: the words XORed into FB0-only / FB1-only positions.
// MASKED: lanes whose `act` bit is clear are lanes still in the all-zero state that must stay there
// (ragged IV lengths: a lane with a shorter IV starts later); see zero_leak().  The mask rides in the
// feedback XOR's LOP3 where there is one, so it costs zero_leak_extra_ops() extra LOP3 per clock.
template <bool MASKED = false>
MK2_HD void clock_s(uint32_t (&s)[NBITS], uint32_t fb_s, uint32_t fb0, uint32_t fb1, uint32_t act = 0xFFFFFFFFu)
{
    // s'[i] = s[i-1] ^ ((s[i]^COMP0_i) & (s[i+1]^COMP1_i)) ^ FB
    auto fbmix = [&](auto ic, uint32_t t) -> uint32_t {
        constexpr int i = decltype(ic)::value;
        constexpr bool f0 = tbit(T_FB0, i), f1 = tbit(T_FB1, i);
        if constexpr (MASKED && zero_leak(i)) {
            constexpr unsigned XOR_AND = ((LA ^ LB) & LC) & 0xFF;  // (a ^ b) & c
            if constexpr (f0 && f1) return lop3<XOR_AND>(t, fb_s, act);
            else if constexpr (f0) return lop3<XOR_AND>(t, fb0, act);
            else if constexpr (f1) return lop3<XOR_AND>(t, fb1, act);
            else return t & act;
        } else if constexpr (f0 && f1) return t ^ fb_s;
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

// One CLOCK_KG of 32 instances.  MIXING: mickey.py:334 (input_r ^= s[50]);
// INPUT: whether an input word is injected (key/IV load) or is zero.
template <bool MIXING, bool INPUT>
MK2_HD void clock(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], uint32_t in)
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

    clock_s(s, fb_s, fb0, fb1);
}

// ---------------------------------------------------------------------------
// K clocks with R's feedback deferred.
//
// R is a Galois register: with p(x) = x^100 + T(x), T = RTAPS, one CLOCK_R is
//     r <- x r + ctrl_r r + in_r T(x)            (mod p)       (mickey.py:336-343)
// and the only part of that which is not one 3-input function per position is
// the reduction x^100 -> T(x), i.e. the fb_r XOR into the 50 tap positions.
// clock_block keeps R UNREDUCED inside a block: the coefficient that falls off
// position 99 in clock k becomes an extra word o[0], earlier ones move up
// (o[j] = coefficient of x^(100+j)), and every position, overflow words
// included, just does a'[i] = a[i-1] ^ (ctrl_r & a[i]).  The true register is
//     r[i] ^ XOR_j Q_j[i] & o[j],     Q_j = x^(100+j) mod p  (compile-time),
// which the clock needs at three taps only (r0 for z, r33, r67 for the control
// bits; r99 is needed for nothing but fb_r) and which is restored for all 100
// positions once per block: one XOR3 per position against two precomputed
// combinations of the overflow words.  R per clock: 100 + k, + ~93 / K; the
// result is identical to K calls of clock<>() (tests/test_clock_host.py,
// GPU parity tests).
// ---------------------------------------------------------------------------
constexpr int MAX_RBLOCK = 6;
struct QTable {
    uint32_t w[MAX_RBLOCK][4];
};
MK2_CX QTable make_qtable()
{
    QTable t{};
    for (int w = 0; w < 4; ++w) t.w[0][w] = table_word(T_RTAPS, w);
    for (int j = 1; j < MAX_RBLOCK; ++j) {
        uint32_t carry = 0;
        for (int w = 0; w < 4; ++w) {
            const uint32_t v = t.w[j - 1][w];
            t.w[j][w] = (v << 1) | carry;
            carry = v >> 31;
        }
        if ((t.w[j][3] >> 4) & 1u) {  // bit 100 set: fold x^100 -> T(x)
            t.w[j][3] &= 0xFu;
            for (int w = 0; w < 4; ++w) t.w[j][w] ^= table_word(T_RTAPS, w);
        }
    }
    return t;
}
constexpr QTable QTAB = make_qtable();
MK2_CX bool qbit(int j, int i) { return (QTAB.w[j][i >> 5] >> (i & 31)) & 1u; }
// bit mask over j in [lo, hi) of Q_j[i]
MK2_CX unsigned qmask(int i, int lo, int hi)
{
    unsigned m = 0;
    for (int j = lo; j < hi; ++j)
        if (qbit(j, i)) m |= 1u << (j - lo);
    return m;
}

// XOR of every subset of up to three words, index = subset mask.  The pair / triple sums
// go through asm LOP3s so that the compiler neither re-derives them per use nor
// re-associates them into the consumers; unused entries are dead code.
template <int H>
MK2_HD void subset_xors(const uint32_t *w, uint32_t (&c)[8])
{
    static_assert(H >= 0 && H <= 3, "at most three words per half");
    c[0] = 0u;
    if constexpr (H >= 1) c[1] = w[0];
    if constexpr (H >= 2) {
        c[2] = w[1];
        c[3] = lop3<(LA ^ LB) & 0xFF>(w[0], w[1], 0u);
    }
    if constexpr (H >= 3) {
        c[4] = w[2];
        c[5] = lop3<(LA ^ LB) & 0xFF>(w[0], w[2], 0u);
        c[6] = lop3<(LA ^ LB) & 0xFF>(w[1], w[2], 0u);
        c[7] = lop3<LUT_XOR3>(w[0], w[1], w[2]);
    }
}

// stored tap word ^ pending overflow words: the true R bit at position TAP in clock KCUR
template <int TAP, int KCUR, int K>
MK2_HD uint32_t r_tap(uint32_t x, const uint32_t (&r)[NBITS], const uint32_t (&o)[K])
{
    uint32_t v = x ^ r[TAP];
    static_for_up<0, KCUR - 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        if constexpr (qbit(j, TAP)) v ^= o[j];
    });
    return v;
}

// LOP3 count of one keystream clock_block<K> (no input, no mixing, z emitted), from the same
// tables the code is generated from: the figure bench.py's roofline uses and
// tests/test_structure.py compares with the SASS.
MK2_CX int xor_ops(int n) { return n / 2; }  // XOR of n >= 2 words with 3-input LUTs
MK2_CX int pending(int tap, int k)
{
    int n = 0;
    for (int j = 0; j < k; ++j) n += qbit(j, tap) ? 1 : 0;
    return n;
}
MK2_CX int block_lop3_count(int K)
{
    int ops = 0;
    for (int k = 0; k < K; ++k) {
        ops += xor_ops(2 + pending(0, k));                                            // z
        ops += xor_ops(2 + pending(CTRL_R_R_TAP, k));                                 // ctrl_r
        ops += pending(CTRL_S_R_TAP, k) ? xor_ops(2 + pending(CTRL_S_R_TAP, k)) : 0;  // ctrl_s, else inside fb0 / fb1
        ops += 2;                                                                     // fb0, fb1
        ops += 100 + k;                                                               // R, unreduced
        ops += 174;                                                                   // S
    }
    const int HA = (K + 1) / 2;
    bool used_a[8] = {}, used_b[8] = {};
    for (int i = 0; i < NBITS; ++i) {
        const unsigned ma = qmask(i, 0, HA), mb = qmask(i, HA, K);
        if (ma | mb) ++ops;  // one XOR (or XOR3) per position with pending overflow
        used_a[ma] = true;
        used_b[mb] = true;
    }
    for (int m = 3; m < 8; ++m)
        if (m != 4) ops += (used_a[m] ? 1 : 0) + (used_b[m] ? 1 : 0);  // multi-word combinations
    return ops;
}

// K x CLOCK_KG.  in_word(k) supplies clock k's input word (INPUT), emit(k, z) receives
// z = r0 ^ s0 sampled before clock k (EMIT).  Reduced state in, reduced state out.
template <int K, bool MIXING, bool INPUT, bool EMIT, bool MASKED, class In, class Emit, class Act>
MK2_HD void clock_block_impl(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], In &&in_word, Emit &&emit, Act &&act_word)
{
    static_assert(K >= 1 && K <= MAX_RBLOCK, "block length");
    uint32_t o[K];
    static_for_up<0, K - 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr (EMIT) emit(kc, r_tap<0, k, K>(s[0], r, o));
        const uint32_t ctrl_r = r_tap<CTRL_R_R_TAP, k, K>(s[CTRL_R_S_TAP], r, o);
        [[maybe_unused]] uint32_t in = 0u;
        if constexpr (INPUT) in = in_word(kc);
        uint32_t fb_s;
        if constexpr (INPUT) fb_s = s[99] ^ in;
        else fb_s = s[99];
        uint32_t fb0, fb1;
        if constexpr (pending(CTRL_S_R_TAP, k) == 0) {  // ctrl_s = s67 ^ r33 folds into the two masks
            fb1 = lop3<(LA & (LB ^ LC)) & 0xFF>(fb_s, s[CTRL_S_S_TAP], r[CTRL_S_R_TAP]);
            fb0 = lop3<(LA & ~(LB ^ LC)) & 0xFF>(fb_s, s[CTRL_S_S_TAP], r[CTRL_S_R_TAP]);
        } else {
            const uint32_t ctrl_s = r_tap<CTRL_S_R_TAP, k, K>(s[CTRL_S_S_TAP], r, o);
            fb1 = fb_s & ctrl_s;
            fb0 = fb_s & ~ctrl_s;
        }

        // ---- R, unreduced: a'[i] = a[i-1] ^ (ctrl_r & a[i]), a = r[0..99] o[0..k-1]; in_r enters at x^100
        uint32_t top = r[99];  // a[99] ^ in_r: what moves into position 100
        if constexpr (MIXING && INPUT) top = lop3<LUT_XOR3>(r[99], s[MIXING_S_TAP], in);
        else if constexpr (MIXING) top = r[99] ^ s[MIXING_S_TAP];
        else if constexpr (INPUT) top = r[99] ^ in;
        if constexpr (k == 0) {
            o[0] = top;
        } else {
            o[k] = o[k - 1];
            static_for_down<k - 1, 1>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                o[j] = lop3<LUT_A_XOR_BC>(o[j - 1], ctrl_r, o[j]);
            });
            o[0] = lop3<LUT_A_XOR_BC>(top, ctrl_r, o[0]);
        }
        static_for_down<99, 1>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            r[i] = lop3<LUT_A_XOR_BC>(r[i - 1], ctrl_r, r[i]);
        });
        r[0] &= ctrl_r;

        if constexpr (MASKED) clock_s<true>(s, fb_s, fb0, fb1, act_word(kc));
        else clock_s(s, fb_s, fb0, fb1);
    });

    // ---- reduce: r[i] ^= XOR_j Q_j[i] & o[j], the overflow words split in two halves
    constexpr int HA = (K + 1) / 2, HB = K - HA;
    uint32_t ca[8], cb[8];
    subset_xors<HA>(o, ca);
    subset_xors<HB>(o + HA, cb);
    static_for_down<99, 0>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr unsigned ma = qmask(i, 0, HA), mb = qmask(i, HA, K);
        if constexpr (ma != 0 && mb != 0) r[i] = lop3<LUT_XOR3>(r[i], ca[ma], cb[mb]);
        else if constexpr (ma != 0) r[i] ^= ca[ma];
        else if constexpr (mb != 0) r[i] ^= cb[mb];
    });
}

struct NoAct {
    template <class KC>
    MK2_HD uint32_t operator()(KC) const { return 0xFFFFFFFFu; }
};
template <int K, bool MIXING, bool INPUT, bool EMIT, class In, class Emit>
MK2_HD void clock_block(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], In &&in_word, Emit &&emit)
{
    clock_block_impl<K, MIXING, INPUT, EMIT, false>(r, s, in_word, emit, NoAct{});
}
// K load clocks (mixing, input word in_word(k)) for a group whose lanes start at different clocks:
// lanes whose bit in act_word(k) is clear are still in the all-zero state, carry a zero input bit and
// stay in the zero state through clock k.  Costs zero_leak_extra_ops() LOP3 per clock over clock_block.
template <int K, class In, class Act>
MK2_HD void clock_block_masked(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], In &&in_word, Act &&act_word)
{
    clock_block_impl<K, true, true, false, true>(r, s, in_word, [](auto, uint32_t) {}, act_word);
}

// keystream word z_t = r0 ^ s0, sampled before the clock (mickey.py:365-367)
MK2_HD uint32_t keystream_word(const uint32_t (&r)[NBITS], const uint32_t (&s)[NBITS])
{
    return r[0] ^ s[0];
}

}  // namespace mk2
