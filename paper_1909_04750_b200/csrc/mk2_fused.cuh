// mk2_fused.cuh -- one-shot bulk generation in ONE kernel: key/IV bytes -> rows of keystream bytes.
//
// kernels.mickey_sliced_words + words_lane_major_bytes of the reference (kernels.py:189-200, :615-621): every
// call restarts from the key/IV load, so for an init-dominated batch (BASELINE config 5: 2^26 fresh key/IV
// pairs x 1 Kbit) the path is   pack -> 160 load clocks -> 100 pre-clocks -> T keystream clocks -> rows.
// As three kernels (pack_uniform_kernel, init_kernel, tmem::gen_rowmajor_kernel) the bitsliced input words
// and the 200-word state of every 32 instances make a round trip through HBM in between: 11.98 GB of DRAM
// traffic for 8.59 GB of keystream + 1.34 GB of key/IV bytes (ncu), three launch tails, and a separate packing
// pass.  Here a worker warp does all of it for one chain (1024 instances) without leaving the SM:
//
//   A  the thread's 32 key and 32 IV records (2 x 320 bytes, twenty 128-bit loads each) are turned into
//      bitsliced input words (PRMT byte picks + 8x32 bit transposes, as pack_records10_to_clocks) and parked
//      in the warp's TENSOR MEMORY tile, column = load clock -- the tile is idle until the keystream starts;
//   B  load clocks in blocks of four (next block's four words in flight: one tcgen05.ld.x4), pre-clocks;
//   C  the keystream loop and 256-clock tile drains of tmem::gen_rowmajor_kernel; the state never exists
//      outside registers (it is written out at the end only when the caller wants to resume).
//
// The three phases are three loops of 19-24 KB of code each.  Two warps of an SM in different loops would
// evict each other from the 32 KB instruction cache (measured for larger bodies: -20..30%), so the eight
// warps of the CTA take eight consecutive chains at a time (one CTA barrier per job): they start together, do the
// same work and therefore run the same loop.  Measured on the config-5 batch (tools/probe_fused.py): per-warp
// jobs, i.e. warps drifting into different loops, 49.7 ms; CTA-wide jobs 46.6 ms.
#pragma once
#include "mk2_tmem.cuh"

namespace mk2 {
namespace fused {

__device__ __forceinline__ void ld4(uint32_t taddr, uint32_t (&v)[4])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void wait_ld4(uint32_t (&v)[4])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])::"memory");
}

// The 320 bytes of a group's 32 ten-byte records -> rec[80], twenty 128-bit loads.  In the last, partial group
// of the batch only `valid` < 320 bytes exist: whole 16-byte pieces are loaded the same way, the ragged piece
// byte by byte, the rest is zero -- rows past N carry zero material (mickey.py:273-276, unused lanes).
__device__ __noinline__ uint4 load_piece_tail(const uint8_t *__restrict__ src, uint32_t nbytes)
{
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (uint32_t b = 0; b < nbytes; ++b) {
        const uint32_t v = (uint32_t)src[b] << (8 * (b & 3));
        if (b < 4) w[0] |= v;
        else if (b < 8) w[1] |= v;
        else if (b < 12) w[2] |= v;
        else w[3] |= v;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void load_records(const uint8_t *__restrict__ src, uint32_t valid, uint32_t (&rec)[80])
{
    const uint4 *p = reinterpret_cast<const uint4 *>(src);
#pragma unroll
    for (int i = 0; i < 20; ++i) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (16u * i + 16u <= valid) v = __ldg(p + i);
        else if (16u * i < valid) v = load_piece_tail(src + 16 * i, valid - 16u * i);
        rec[4 * i] = v.x;
        rec[4 * i + 1] = v.y;
        rec[4 * i + 2] = v.z;
        rec[4 * i + 3] = v.w;
    }
}

// nbytes byte columns of the records -> tile columns c0 .. c0 + 8 nbytes - 1 (column = load clock, MSB-first
// per byte, bitops.py:33-36).  Warp-collective (tcgen05.st): every thread of the warp runs it.
__device__ __forceinline__ void park_records(const uint32_t (&rec)[80], int nbytes, uint32_t tcol)
{
    static_for_up<0, 9>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        if (b < nbytes) {  // warp-uniform
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
            const uint32_t v[8] = {w[7], w[6], w[5], w[4], w[3], w[2], w[1], w[0]};  // clock 8 b + m carries bit 7 - m
            tmem::st8(tcol + 8 * b, v);
        }
    });
}

// iv_bytes = IV length in bytes (0..10; the host side routes IV lengths that are not whole bytes, IV strides
// other than 10 and unaligned arrays to the three-kernel path).  ticket: zeroed before the launch.
// state_out / acc_out: null, or where to leave the state for a resuming mk2_generate_* call.
// sum: += what checksum_kernel would compute for the batch (sum of acc << 32 * (global group parity)).
//
// Jobs.  Ticket t < full_jobs: the eight chains 8 t .. 8 t + 7, one per warp.  The host makes full_jobs a multiple
// of the grid size, i.e. whole rounds in which every SM is busy.  What is left (fewer jobs than SMs: a last round
// that would leave the other SMs idle for a whole job) is handed out as HALF jobs: four chains on warps 0..3, one
// per SM sub-partition, where a lone warp runs almost twice as fast (97.8% of the LOP3 rate alone against
// 98.6% for two) -- the last round then takes half the time on twice as many SMs (config 5: 55.5 rounds, not 56).
template <bool ALIGNED16>
__global__ void __launch_bounds__(BLOCK, 1)
bulk_rowmajor_kernel(const uint8_t *__restrict__ keys, const uint8_t *__restrict__ ivs, int iv_bytes, uint64_t N, uint64_t G,
                     uint64_t T, uint8_t *__restrict__ out, uint64_t pitch, unsigned long long *ticket,
                     unsigned long long full_jobs, unsigned long long *sum, uint64_t g_offset,
                     uint32_t *__restrict__ state_out, unsigned long long *__restrict__ acc_out)
{
    __shared__ uint32_t tmem_base_slot;
    __shared__ unsigned long long job_slot;
    const uint32_t tcol = tmem::open_tile(&tmem_base_slot);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t chains = (G + 31) / 32;
    const int load_clocks = 8 * iv_bytes + KEY_BITS;

    for (;;) {
        if (threadIdx.x == 0) job_slot = atomicAdd(ticket, 1ull);
        __syncthreads();
        const uint64_t job = job_slot;
        const bool whole = job < full_jobs;
        const uint64_t chain0 = whole ? job * 8 : full_jobs * 8 + (job - full_jobs) * 4;
        if (chain0 >= chains) break;  // CTA-uniform
        // Warps without a chain in this job wait at the barrier below.  The predicate comes out of a vote so that
        // it is warp-uniform by construction: under a branch the compiler cannot prove uniform the loops lose the
        // uniform datapath (tile address and loop counters in vector registers, one R2UR per tile store).
        const uint64_t chain = chain0 + warp;
        if (__all_sync(0xFFFFFFFFu, chain < chains && (whole || warp < 4))) {
            const uint64_t g_own = chain * 32 + lane;
            // tcgen05 ld / st are warp-collective: a thread whose group does not exist (last, partial chain) runs
            // along on the last real group and stores nothing
            const bool real = g_own < G;
            const uint64_t g = real ? g_own : G - 1;
            const uint64_t left = N - 32 * g;  // instances of this group that exist
            const uint32_t valid = left >= 32 ? 320u : (uint32_t)left * 10u;

            // ---- A: key/IV records -> input words in the tile (IV bits first, then the key: mickey.py:145-148)
            {
                uint32_t rec[80];
                if (iv_bytes) {
                    load_records(ivs + 320 * g, valid, rec);
                    park_records(rec, iv_bytes, tcol);
                }
                load_records(keys + 320 * g, valid, rec);
                park_records(rec, 10, tcol + 8 * iv_bytes);
                tmem::wait_st();
            }

            // ---- B: load clocks + pre-clocks (init_kernel<false> with the input words read from the tile).  ONE loop
            // for both (a pre-clock is a load clock with a zero input word: 1217 against 1216 LOP3 per block): one
            // 19.8 KB body to fetch per job instead of two.  No barrier between the phases: the warps of a job start
            // together and do the same work, so they stay in the same loop anyway.
            uint32_t r[NBITS], s[NBITS];
#pragma unroll
            for (int i = 0; i < NBITS; ++i) r[i] = s[i] = 0u;
            {
                static_assert(RBLOCK_INIT == 4 && PRECLOCKS % 4 == 0, "four input words per block, whole blocks");
                uint32_t nx[4];
                ld4(tcol, nx);
                wait_ld4(nx);
#pragma unroll 1
                for (int c = 0; c < load_clocks + PRECLOCKS; c += 4) {  // load_clocks is a multiple of 8
                    const uint32_t cur[4] = {nx[0], nx[1], nx[2], nx[3]};
                    if (c + 4 < load_clocks) {
                        ld4(tcol + c + 4, nx);
                    } else {
                        nx[0] = nx[1] = nx[2] = nx[3] = 0u;
                    }
                    clock_block<4, true, true, false>(
                        r, s, [&](auto kc) { return cur[decltype(kc)::value]; }, [](auto, uint32_t) {});
                    wait_ld4(nx);
                }
            }

            // ---- C: keystream, 256-clock tiles, row drains (tmem::gen_rowmajor_kernel's loop)
            unsigned long long a = 0;
            uint8_t *rows = out + 32 * g * pitch;
            const uint64_t nrows = !real ? 0 : (left < 32 ? left : 32);
#pragma unroll 1
            for (uint64_t t0 = 0; t0 < T; t0 += tmem::TILE_CLOCKS) {
                const int nclk = (T - t0) >= tmem::TILE_CLOCKS ? tmem::TILE_CLOCKS : (int)(T - t0);
                uint32_t tz = tcol;
                int t = 0;
                HalfSums hs;
#pragma unroll 1
                for (; t + tmem::RBLOCK <= nclk; t += tmem::RBLOCK) {
                    clock_block<tmem::RBLOCK, false, false, true>(r, s, NoInput{}, [&](auto kc, uint32_t z) {
                        tmem::st1(tz + decltype(kc)::value, z);
                        hs.add(z);
                    });
                    tz += tmem::RBLOCK;
                }
#pragma unroll 1
                for (; t < nclk; ++t) {
                    const uint32_t z = keystream_word(r, s);
                    tmem::st1(tz, z);
                    tz += 1;
                    hs.add(z);
                    clock<false, false>(r, s, 0u);
                }
                hs.fold(a);
                tmem::wait_st();
                tmem::row_drain<ALIGNED16, false>(tcol, rows + (t0 >> 3), pitch, nclk >> 3, nrows);
            }
            if (real && state_out) {
#pragma unroll
                for (int i = 0; i < NBITS; ++i) {
                    state_out[(uint64_t)i * G + g] = r[i];
                    state_out[(uint64_t)(NBITS + i) * G + g] = s[i];
                }
                acc_out[g] = a;
            }
            // checksum of the batch, as checksum_kernel folds the per-group sums
            unsigned long long v = real ? a << (32 * ((g + g_offset) & 1)) : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
            if (lane == 0) atomicAdd(sum, v);
        }
        __syncthreads();  // job_slot is rewritten at the top
    }
    tmem::close_tile(&tmem_base_slot);
}

}  // namespace fused
}  // namespace mk2
