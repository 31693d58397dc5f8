// mk2_seedgen.cuh -- per-lane key/IV derivation from a 256-bit master seed on the GPU.
//
// The reference derives lane material with AES-128 in a counter construction
// (pkg/src/slicerng/seedgen.py:57-86) and caps a seed at 64 lanes (:22) because
// its AES is Python; here one thread derives one lane, so a seed can feed the
// millions of lanes the MICKEY kernels run:
//   dk      = AES_{seed[0:16]}(seed[16:32])                       (seedgen.py:57-60)
//   block_c = tag || lane (4 B, big-endian) || c (4 B, BE) || 0^7  (seedgen.py:72-78)
//   stream  = AES_dk(block_0) || AES_dk(block_1);  key = stream[0:10], iv = stream[10:20]
// AES-128 is plain FIPS-197 (the reference's AesScalarTable,
// pkg/src/slicerng/aes_ctr.py:193-219): byte i of a block is state row i % 4,
// column i / 4.  The S-box is computed once per CTA into shared memory from the
// GF(2^8) inverse + affine map, so no table literal is carried in the source; the
// per-lane kernel runs on a bank-replicated SubBytes + MixColumns table built from it.
#pragma once
#include <cstdint>

namespace mk2 {

__device__ __forceinline__ uint8_t gf_xtime(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1B : 0)); }

__device__ inline uint8_t gf_mul(uint8_t a, uint8_t b)
{
    uint8_t p = 0;
    for (int i = 0; i < 8; ++i) {
        if (b & 1) p ^= a;
        a = gf_xtime(a);
        b >>= 1;
    }
    return p;
}

// S-box entry for x: inverse by x^254 (square-and-multiply), then the affine map.
__device__ inline uint8_t aes_sbox_compute(uint8_t x)
{
    uint8_t x2 = gf_mul(x, x), x4 = gf_mul(x2, x2), x8 = gf_mul(x4, x4), x16 = gf_mul(x8, x8);
    uint8_t x32 = gf_mul(x16, x16), x64 = gf_mul(x32, x32), x128 = gf_mul(x64, x64);
    uint8_t inv = gf_mul(gf_mul(gf_mul(x128, x64), gf_mul(x32, x16)), gf_mul(gf_mul(x8, x4), x2));  // x^254
    uint8_t r = inv, v = inv;
    for (int k = 0; k < 4; ++k) {
        r = (uint8_t)((r << 1) | (r >> 7));
        v ^= r;
    }
    return v ^ 0x63;
}

__device__ inline void aes_expand_key(const uint8_t *sbox, const uint8_t key[16], uint8_t rk[11][16])
{
    for (int i = 0; i < 16; ++i) rk[0][i] = key[i];
    uint8_t rcon = 1;
    for (int r = 1; r <= 10; ++r) {
        const uint8_t *p = rk[r - 1];
        uint8_t t[4] = {(uint8_t)(sbox[p[13]] ^ rcon), sbox[p[14]], sbox[p[15]], sbox[p[12]]};
        rcon = gf_xtime(rcon);
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 4; ++b) rk[r][4 * c + b] = p[4 * c + b] ^ (c ? rk[r][4 * (c - 1) + b] : t[b]);
    }
}

// One block; state as four column words (byte k of word c = state row k, column c).
__device__ __forceinline__ void aes_encrypt_block(const uint8_t *sbox, const uint32_t *rk /*[44]*/, uint32_t (&st)[4])
{
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] ^= rk[c];
#pragma unroll 1
    for (int r = 1; r <= 10; ++r) {
        uint32_t t[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // SubBytes + ShiftRows: row k of column c comes from column (c + k) & 3
            const uint32_t b0 = sbox[st[c] & 0xFF];
            const uint32_t b1 = sbox[(st[(c + 1) & 3] >> 8) & 0xFF];
            const uint32_t b2 = sbox[(st[(c + 2) & 3] >> 16) & 0xFF];
            const uint32_t b3 = sbox[(st[(c + 3) & 3] >> 24) & 0xFF];
            t[c] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
        }
        if (r < 10) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // MixColumns on packed bytes: a ^ all ^ xtime(a ^ rot(a))
                const uint32_t a = t[c];
                const uint32_t rot = (a >> 8) | (a << 24);  // byte k <- byte k + 1
                const uint32_t x = a ^ rot;
                const uint32_t xt = ((x & 0x7F7F7F7Fu) << 1) ^ (((x >> 7) & 0x01010101u) * 0x1Bu);
                const uint32_t all = x ^ ((x >> 16) | (x << 16));  // a0^a1^a2^a3 in every byte
                t[c] = a ^ all ^ xt;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) st[c] = t[c] ^ rk[4 * r + c];
    }
}

// The bulk path: the same block function on a combined SubBytes + MixColumns table.
//   T0[x] = (2 s, s, s, 3 s) as bytes 0..3 with s = sbox[x]: the MixColumns image of a row-0 byte; a byte of
//   row k contributes T0 rotated left by k bytes, so one 256-word table and three rotations replace four.
// The table is replicated 32 times in shared memory -- entry x of lane l lives at word 32 x + l, i.e. always in
// bank l -- so the 16 data-dependent lookups of a round never conflict (the byte-wide S-box above is 64 words
// for 32 lanes).  `tbl` points at this lane's column.
__device__ __forceinline__ uint32_t rotl8(uint32_t w, int k) { return k ? __funnelshift_l(w, w, 8 * k) : w; }
template <int K>
__device__ __forceinline__ uint32_t tt(const uint32_t *tbl, uint32_t word)
{
    // byte K of `word`, times 32 words: (word >> 8 K & 0xFF) << 5
    const uint32_t off = K == 0 ? (word << 5) & 0x1FE0u : (word >> (8 * K - 5)) & 0x1FE0u;
    return tbl[off];
}
__device__ __forceinline__ void aes_encrypt_block_tt(const uint32_t *tbl, const uint32_t *rk /*[44]*/, uint32_t (&st)[4])
{
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] ^= rk[c];
#pragma unroll 1
    for (int r = 1; r < 10; ++r) {
        uint32_t t[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)  // row k of output column c comes from column (c + k) & 3 (ShiftRows)
            t[c] = tt<0>(tbl, st[c]) ^ rotl8(tt<1>(tbl, st[(c + 1) & 3]), 1) ^ rotl8(tt<2>(tbl, st[(c + 2) & 3]), 2) ^
                   rotl8(tt<3>(tbl, st[(c + 3) & 3]), 3) ^ rk[4 * r + c];
#pragma unroll
        for (int c = 0; c < 4; ++c) st[c] = t[c];
    }
    uint32_t t[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // last round: SubBytes + ShiftRows only; s is byte 1 of T0
        const uint32_t b0 = (tt<0>(tbl, st[c]) >> 8) & 0xFFu;
        const uint32_t b1 = tt<1>(tbl, st[(c + 1) & 3]) & 0xFF00u;
        const uint32_t b2 = (tt<2>(tbl, st[(c + 2) & 3]) << 8) & 0xFF0000u;
        const uint32_t b3 = (tt<3>(tbl, st[(c + 3) & 3]) << 16) & 0xFF000000u;
        t[c] = (b0 | b1 | b2 | b3) ^ rk[40 + c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] = t[c];
}

// 1 thread: derivation key and its round keys (as little-endian column words).
__global__ void seed_setup_kernel(const uint8_t *__restrict__ seed /*[32]*/, uint32_t *__restrict__ rk_out /*[44]*/)
{
    __shared__ uint8_t sbox[256];
    for (int x = threadIdx.x; x < 256; x += blockDim.x) sbox[x] = aes_sbox_compute((uint8_t)x);
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint8_t key[16], rkb[11][16];
    for (int i = 0; i < 16; ++i) key[i] = seed[i];
    aes_expand_key(sbox, key, rkb);
    uint32_t rkw[44];
    for (int i = 0; i < 44; ++i) {
        const uint8_t *p = &rkb[0][0] + 4 * i;
        rkw[i] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
    }
    uint32_t st[4];
    for (int c = 0; c < 4; ++c)
        st[c] = seed[16 + 4 * c] | (seed[17 + 4 * c] << 8) | (seed[18 + 4 * c] << 16) | ((uint32_t)seed[19 + 4 * c] << 24);
    aes_encrypt_block(sbox, rkw, st);
    for (int c = 0; c < 4; ++c)
        for (int b = 0; b < 4; ++b) key[4 * c + b] = (uint8_t)(st[c] >> (8 * b));
    aes_expand_key(sbox, key, rkb);
    for (int i = 0; i < 44; ++i) {
        const uint8_t *p = &rkb[0][0] + 4 * i;
        rk_out[i] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
    }
}

// One thread per lane: two AES blocks -> 10 key bytes + iv_len IV bytes (10 for mickey, 8 for grain:
// seedgen.py:24-29); the IV rows are iv_len bytes apart.
__global__ void __launch_bounds__(256)
seed_derive_kernel(const uint32_t *__restrict__ rk_in, uint32_t tag, uint64_t first_lane, uint64_t n, int iv_len,
                   uint8_t *__restrict__ keys, uint8_t *__restrict__ ivs)
{
    __shared__ uint32_t t0r[256 * 32];  // T0, one copy per bank (32 KB)
    __shared__ uint32_t rk[44];
    for (int x = threadIdx.x; x < 256; x += blockDim.x) {
        const uint32_t sb = aes_sbox_compute((uint8_t)x), s2 = gf_xtime((uint8_t)sb);
        const uint32_t w = s2 | (sb << 8) | (sb << 16) | ((s2 ^ sb) << 24);
        for (int l = 0; l < 32; ++l) t0r[32 * x + l] = w;
    }
    if (threadIdx.x < 44) rk[threadIdx.x] = rk_in[threadIdx.x];
    __syncthreads();
    const uint32_t *tbl = t0r + (threadIdx.x & 31);
    const bool even = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(ivs)) & 1u) == 0;
    // grid-stride over lanes: the table build (an S-box inversion per thread) is paid once per CTA, not per 256 lanes
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t lane = (uint32_t)(first_lane + j);
        uint32_t stream[8];
#pragma unroll
        for (uint32_t c = 0; c < 2; ++c) {
            // bytes: [tag, lane>>24, lane>>16, lane>>8 | lane, 0, 0, 0 | c, 0, 0, 0 | 0, 0, 0, 0]
            uint32_t st[4] = {tag | ((lane >> 24) << 8) | (((lane >> 16) & 0xFF) << 16) | (((lane >> 8) & 0xFF) << 24),
                              lane & 0xFF, c, 0u};
            aes_encrypt_block_tt(tbl, rk, st);
#pragma unroll
            for (int w = 0; w < 4; ++w) stream[4 * c + w] = st[w];
        }
        uint8_t *k = keys + 10 * j, *v = ivs + (uint64_t)iv_len * j;
        if (iv_len != 10) {
#pragma unroll
            for (int b = 0; b < 10; ++b) k[b] = (uint8_t)(stream[b >> 2] >> (8 * (b & 3)));
#pragma unroll
            for (int b = 10; b < 20; ++b)
                if (b - 10 < iv_len) v[b - 10] = (uint8_t)(stream[b >> 2] >> (8 * (b & 3)));
        } else if (even) {  // 10-byte records at even addresses: five 16-bit stores each instead of ten byte stores
#pragma unroll
            for (int u = 0; u < 5; ++u) reinterpret_cast<uint16_t *>(k)[u] = (uint16_t)(stream[u >> 1] >> (16 * (u & 1)));
#pragma unroll
            for (int u = 5; u < 10; ++u) reinterpret_cast<uint16_t *>(v)[u - 5] = (uint16_t)(stream[u >> 1] >> (16 * (u & 1)));
        } else {
#pragma unroll
            for (int b = 0; b < 10; ++b) k[b] = (uint8_t)(stream[b >> 2] >> (8 * (b & 3)));
#pragma unroll
            for (int b = 10; b < 20; ++b) v[b - 10] = (uint8_t)(stream[b >> 2] >> (8 * (b & 3)));
        }
    }
}

}  // namespace mk2
