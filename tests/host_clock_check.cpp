// Host build of csrc/mk2_clock.cuh for tests/test_clock_host.py: the same template code the
// kernels are generated from, with the LOP3 truth tables evaluated in software, so the block
// clock (deferred R reduction) can be compared with the one-clock form and with the oracle on
// a machine without a GPU.  Test infrastructure only: nothing in the product links this.
#include <cstdint>

#include "../paper_1909_04750_b200/csrc/mk2_clock.cuh"
#include "../paper_1909_04750_b200/csrc/mk2_bits.cuh"

using namespace mk2;

namespace {
template <bool MIX, bool INP>
void plain(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], const uint32_t *in, int n, uint32_t *z)
{
    for (int k = 0; k < n; ++k) {
        z[k] = keystream_word(r, s);
        clock<MIX, INP>(r, s, INP ? in[k] : 0u);
    }
}
template <int K, bool MIX, bool INP>
void block(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], const uint32_t *in, uint32_t *z)
{
    clock_block<K, MIX, INP, true>(
        r, s, [&](auto kc) { return in[decltype(kc)::value]; }, [&](auto kc, uint32_t w) { z[decltype(kc)::value] = w; });
}
template <int K>
void block_k(uint32_t (&r)[NBITS], uint32_t (&s)[NBITS], int mixing, int has_in, const uint32_t *in, uint32_t *z)
{
    if (mixing && has_in) block<K, true, true>(r, s, in, z);
    else if (mixing) block<K, true, false>(r, s, in, z);
    else if (has_in) block<K, false, true>(r, s, in, z);
    else block<K, false, false>(r, s, in, z);
}
}  // namespace

extern "C" {
// n one-clock steps; z[k] = r0 ^ s0 before step k
void hc_plain(uint32_t *r, uint32_t *s, int mixing, int has_in, const uint32_t *in, int n, uint32_t *z)
{
    auto &R = *reinterpret_cast<uint32_t(*)[NBITS]>(r);
    auto &S = *reinterpret_cast<uint32_t(*)[NBITS]>(s);
    if (mixing && has_in) plain<true, true>(R, S, in, n, z);
    else if (mixing) plain<true, false>(R, S, in, n, z);
    else if (has_in) plain<false, true>(R, S, in, n, z);
    else plain<false, false>(R, S, in, n, z);
}
// one clock_block<K>; returns 0, or -1 for an unsupported K
int hc_block(int K, uint32_t *r, uint32_t *s, int mixing, int has_in, const uint32_t *in, uint32_t *z)
{
    auto &R = *reinterpret_cast<uint32_t(*)[NBITS]>(r);
    auto &S = *reinterpret_cast<uint32_t(*)[NBITS]>(s);
    switch (K) {
    case 1: block_k<1>(R, S, mixing, has_in, in, z); return 0;
    case 2: block_k<2>(R, S, mixing, has_in, in, z); return 0;
    case 3: block_k<3>(R, S, mixing, has_in, in, z); return 0;
    case 4: block_k<4>(R, S, mixing, has_in, in, z); return 0;
    case 5: block_k<5>(R, S, mixing, has_in, in, z); return 0;
    case 6: block_k<6>(R, S, mixing, has_in, in, z); return 0;
    default: return -1;
    }
}
// one clock_block_masked<K> (load clocks of a ragged group: lanes with a clear act bit stay in the zero state)
int hc_block_masked(int K, uint32_t *r, uint32_t *s, const uint32_t *in, const uint32_t *act)
{
    auto &R = *reinterpret_cast<uint32_t(*)[NBITS]>(r);
    auto &S = *reinterpret_cast<uint32_t(*)[NBITS]>(s);
    auto inw = [&](auto kc) { return in[decltype(kc)::value]; };
    auto actw = [&](auto kc) { return act[decltype(kc)::value]; };
    switch (K) {
    case 1: clock_block_masked<1>(R, S, inw, actw); return 0;
    case 2: clock_block_masked<2>(R, S, inw, actw); return 0;
    case 3: clock_block_masked<3>(R, S, inw, actw); return 0;
    case 4: clock_block_masked<4>(R, S, inw, actw); return 0;
    default: return -1;
    }
}
void hc_transpose32(uint32_t *a) { transpose32(*reinterpret_cast<uint32_t(*)[32]>(a)); }
// fast path of pack_ragged_kernel for one group: 96 input words + 96 activity words (clock-major)
void hc_ragged_group(const uint32_t *rec, const uint32_t *len, int lmax, uint32_t *in96, uint32_t *act96)
{
    for (int k = 0; k < 3; ++k)
        ragged_group_words(*reinterpret_cast<const uint32_t(*)[80]>(rec), *reinterpret_cast<const uint32_t(*)[8]>(len), lmax, k,
                           *reinterpret_cast<uint32_t(*)[32]>(in96 + 32 * k), *reinterpret_cast<uint32_t(*)[32]>(act96 + 32 * k));
}
int hc_zero_leak_extra_ops() { return zero_leak_extra_ops(); }
int hc_block_lop3_count(int K) { return K >= 1 && K <= MAX_RBLOCK ? block_lop3_count(K) : -1; }
int hc_q_bit(int j, int i) { return qbit(j, i) ? 1 : 0; }
}
