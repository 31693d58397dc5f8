// mk2_api.cu -- C-ABI shim (include/mk2.h) over the sm_100a kernels.
// Host side only does pointer classification, chunking and launches; all
// cipher work is in mk2_clock.cuh / mk2_kernels.cuh (MICKEY 2.0), mk2_grain.cuh (Grain v1) and
// mk2_seedgen.cuh (seed derivation).  No CPU fallback exists in this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>

#include "../../include/mk2.h"
#include "mk2_kernels.cuh"
#include "mk2_tmem.cuh"
#include "mk2_grain.cuh"
#include "mk2_grain_row64.cuh"
#include "mk2_grain_ring.cuh"
#include "mk2_grain_row8.cuh"
#include "mk2_fused.cuh"
#include "mk2_coop.cuh"
#include "mk2_seedgen.cuh"
#include "mk2_host_lanes.h"

using namespace mk2;
using mk2::host::HostCopyLanes;

namespace {
thread_local std::string g_create_error;  // text of this thread's last failed mk2_create
// Per staging buffer for host outputs (two in flight).  Column-major tiles are plain 1-D copies: small
// tiles shorten the pipeline fill (measured on B200, 2 GiB per call: 32 MiB 54.8 GB/s, 256 MiB 53.0 GB/s).
// Row-major tiles are 2-D copies whose rows must stay >= 512 B wide (64 B rows: 16 GB/s), so they are
// 16x larger (profiles/r01b_probe_e2e_stage.txt).
constexpr size_t STAGE_BYTES = size_t(32) << 20;
constexpr size_t ROW_TILE_FACTOR = 16;
// Pageable host outputs below this size are left to the driver's own staged copy (no lanes, no page-locking).
constexpr uint64_t BOUNCE_MIN_BYTES = uint64_t(64) << 20;

// Restores the caller's current device when an entry point returns: a process that drives torch on cuda:0 and
// an mk2 context on device 1 keeps its own current device.
struct DeviceGuard {
    int prev = -1, dev;
    bool ok = true;
    explicit DeviceGuard(int device) : dev(device)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard()
    {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

}  // namespace

struct mk2_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own = nullptr, stream = nullptr, copy = nullptr, h2d = nullptr;  // h2d: mk2_bulk_rowmajor only (lazy)
    cudaEvent_t h2d_done[2] = {nullptr, nullptr}, mat_used[2] = {nullptr, nullptr};
    void *d_bulk_in[2] = {nullptr, nullptr};  // material staging of mk2_bulk_rowmajor
    size_t bulk_in_bytes = 0;
    cudaMemPool_t pool = nullptr;  // private stream-ordered pool for scratch (kept warm: no trim at sync points)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t gen_done[2] = {nullptr, nullptr}, copy_done[2] = {nullptr, nullptr};
    bool copy_pending[2] = {false, false};
    uint64_t N = 0, G = 0, cap = 0, g_offset = 0, clocks = 0;
    uint32_t *d_state = nullptr;
    unsigned long long *d_acc = nullptr, *d_sum = nullptr;
    SchedQueue *d_queue = nullptr;       // persistent-kernel scheduler (mk2_kernels.cuh)
    unsigned long long *d_slots = nullptr;
    uint32_t *d_progress = nullptr;
    uint32_t ring = 0;                   // ring size (power of two >= 2 x chains)
    uint32_t chunk_user = 0;             // user override of clocks per scheduling chunk (0 = automatic)
    int block_user = 0;                  // user override of threads per persistent CTA (0 = automatic)
    size_t stage_target = STAGE_BYTES;   // bytes per host-output staging tile (mk2_set_stage_bytes)
    bool stage_user = false;             // ... set by the caller (honoured as is for pageable outputs too)
    int row_staging = 0;                 // row-major staging tile: 0 = automatic, 1 = shared memory, 2 = tensor memory,
                                         // 3 = L2-resident scratch (Grain only)
    uint32_t *d_rowscratch = nullptr;    // staging mode 3: one 64 KiB tile per worker warp (lazy)
    int bulk_fused = 1;                  // mk2_bulk_rowmajor with device buffers, one-kernel path: 0 never, 1 automatic
                                         // (init-dominated calls, T <= FUSED_MAX_CLOCKS), 2 whenever eligible
    int small_batch = 1;                 // 1 = warp-per-group kernels (mk2_coop.cuh) for G <= COOP_MAX_GROUPS
    int last_plan_block = 0;
    uint32_t last_plan_chunk = 0;
    Trace trace = {nullptr, nullptr, 0}; // optional per-job trace (device buffers owned by the ctx)
    unsigned max_grid = 0;               // debug knob: cap on persistent CTAs (0 = one per SM slot)
    void *d_stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    HostCopyLanes *lanes = nullptr;          // copy lanes for PAGEABLE host outputs (lazy)
    int host_threads = 0;                    // number of lanes; 0 = automatic
    bool ready = false, async = false, timing_open = false;
    int cipher = 0;        // 0 = MICKEY 2.0, 1 = Grain v1 (which kernels the state belongs to)
    bool row_lsb = false;  // Grain row-major byte packing of the current call
    float last_ms = 0.f;
    int last_launches = 0;
    int block = BLOCK;  // threads per CTA of the clocking kernels (tunable, <= BLOCK)
    std::string err;
};

namespace {

int fail(mk2_ctx *c, int code, const std::string &msg)
{
    if (c) c->err = msg;
    else g_create_error = msg;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            cudaGetLastError(); /* clear a non-sticky error so that it is not reported twice */    \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? MK2_E_NOMEM : MK2_E_CUDA,            \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                       \
        }                                                                                          \
    } while (0)

enum class Mem { Device, Pinned, Pageable };
Mem classify(const void *p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return Mem::Pageable;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return Mem::Device;
    return a.type == cudaMemoryTypeHost ? Mem::Pinned : Mem::Pageable;
}
bool is_device_ptr(const void *p) { return classify(p) == Mem::Device; }

// Stream-ordered scratch of one call: whatever was allocated is given back to the pool on EVERY exit path
// (cudaFreeAsync on the launch stream orders the free after the kernels that use it).
struct Scratch {
    mk2_ctx *ctx;
    void *ptr[8] = {};
    int n = 0;
    explicit Scratch(mk2_ctx *c) : ctx(c) {}
    ~Scratch()
    {
        for (int i = 0; i < n; ++i)
            if (ptr[i]) cudaFreeAsync(ptr[i], ctx->stream);
    }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    int alloc(void **out, size_t bytes)
    {
        *out = nullptr;
        if (n == 8) return fail(ctx, MK2_E_ARG, "internal: scratch list full");
        CK(cudaMallocFromPoolAsync(out, bytes, ctx->pool, ctx->stream));
        ptr[n++] = *out;
        return MK2_OK;
    }
};

inline unsigned blocks_for(uint64_t G, int block = BLOCK) { return (unsigned)((G + block - 1) / block); }

int begin_timing(mk2_ctx *ctx)
{
    ctx->last_launches = 0;
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    return MK2_OK;
}

int end_timing(mk2_ctx *ctx)
{
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->timing_open = true;
    if (!ctx->async) {
        CK(cudaEventSynchronize(ctx->ev1));
        CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
        ctx->timing_open = false;
    }
    return MK2_OK;
}

int ensure_capacity(mk2_ctx *ctx, uint64_t G)
{
    if (G <= ctx->cap) return MK2_OK;
    // whatever happens below, the old state is gone: no later call may launch on freed (or null) buffers
    ctx->ready = false;
    ctx->N = ctx->G = 0;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->d_state) cudaFree(ctx->d_state);
    if (ctx->d_acc) cudaFree(ctx->d_acc);
    if (ctx->d_slots) cudaFree(ctx->d_slots);
    if (ctx->d_progress) cudaFree(ctx->d_progress);
    ctx->d_state = nullptr;
    ctx->d_acc = nullptr;
    ctx->d_slots = nullptr;
    ctx->d_progress = nullptr;
    ctx->cap = 0;
    const uint64_t chains = (G + 31) / 32;
    uint64_t ring = 64;  // power of two >= 2 x chains: a slot is never rewritten while its reader may still poll it
    while (ring < 2 * chains) ring <<= 1;
    if (ring > 0x80000000ull) return fail(ctx, MK2_E_ARG, "too many instances for one context");
    CK(cudaMalloc(&ctx->d_state, sizeof(uint32_t) * 2 * NBITS * G));
    CK(cudaMalloc(&ctx->d_acc, sizeof(unsigned long long) * G));
    CK(cudaMalloc(&ctx->d_slots, sizeof(unsigned long long) * ring));
    CK(cudaMalloc(&ctx->d_progress, sizeof(uint32_t) * chains));
    ctx->ring = (uint32_t)ring;
    ctx->cap = G;
    return MK2_OK;
}

int ensure_stage(mk2_ctx *ctx, size_t bytes)
{
    if (bytes <= ctx->stage_bytes) return MK2_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->copy));
    for (int b = 0; b < 2; ++b) {
        if (ctx->d_stage[b]) cudaFree(ctx->d_stage[b]);
        ctx->d_stage[b] = nullptr;
        ctx->copy_pending[b] = false;
    }
    ctx->stage_bytes = 0;
    for (int b = 0; b < 2; ++b) CK(cudaMalloc(&ctx->d_stage[b], bytes));
    ctx->stage_bytes = bytes;
    return MK2_OK;
}

// Copy lanes for pageable host outputs (see HostCopyLanes, HostTiles).
int ensure_lanes(mk2_ctx *ctx)
{
    if (ctx->lanes) return MK2_OK;
    int n = ctx->host_threads;
    if (n <= 0) {
        // one lane per hardware thread, 2..16; a tile uses as many of them as suit its shape (HostCopyLanes::post)
        const unsigned hw = std::thread::hardware_concurrency();
        n = (int)std::min<unsigned>(16u, std::max<unsigned>(2u, hw));
    }
    ctx->lanes = new (std::nothrow) HostCopyLanes(ctx->device, n);
    if (!ctx->lanes) return fail(ctx, MK2_E_NOMEM, "out of host memory");
    return MK2_OK;
}

// Bring a host-or-device input array onto the device (stream ordered).
int stage_input(mk2_ctx *ctx, Scratch &scratch, const void *src, size_t bytes, const uint8_t **dev)
{
    if (bytes == 0 || src == nullptr) {
        *dev = nullptr;
        return MK2_OK;
    }
    if (is_device_ptr(src)) {
        *dev = static_cast<const uint8_t *>(src);
        return MK2_OK;
    }
    void *owned = nullptr;
    int rc = scratch.alloc(&owned, bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(owned, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *dev = static_cast<const uint8_t *>(owned);
    return MK2_OK;
}

// Small batches (the reference's own 64-lane calling unit up to a few thousand groups): one warp per group with
// the state spread over its lanes clocks ~5x faster than a thread per group, as long as the GPU has idle
// sub-partitions to put the warps on.  Measured crossover: tools/probe_small_batch.py.
constexpr uint64_t COOP_MAX_GROUPS = 2048;
inline unsigned coop_grid(const mk2_ctx *ctx) { return (unsigned)((ctx->G + coop::WARPS - 1) / coop::WARPS); }

int launch_init(mk2_ctx *ctx, const uint32_t *mat, int load_clocks, int lmax, bool ragged)
{
    const unsigned nb = blocks_for(ctx->G, ctx->block);
    if (!ragged && ctx->small_batch && ctx->G <= COOP_MAX_GROUPS)
        coop::init_kernel<<<coop_grid(ctx), 32 * coop::WARPS, 0, ctx->stream>>>(mat, load_clocks, ctx->G, ctx->d_state, ctx->d_acc);
    else if (ragged)
        init_kernel<true><<<nb, ctx->block, 0, ctx->stream>>>(mat, load_clocks, lmax, ctx->G, ctx->d_state, ctx->d_acc);
    else
        init_kernel<false><<<nb, ctx->block, 0, ctx->stream>>>(mat, load_clocks, lmax, ctx->G, ctx->d_state, ctx->d_acc);
    CK(cudaGetLastError());
    ctx->last_launches++;
    ctx->clocks = 0;
    ctx->cipher = 0;
    ctx->ready = true;
    return MK2_OK;
}

// ---------------------------------------------------------------------------
// Schedule of one keystream launch: how many worker warps per SM and how the T
// clocks of every chain (= 1024 instances) are cut into chunks.
//
// Measured on B200 (profiles/): one warp alone on an SM sub-partition already
// runs the clock loop at 98.9% of the LOP3 issue rate, two warps share it at
// 99.1%, and parking / reloading a chain's state costs nothing measurable even
// for 512-clock chunks.  So:
//   * plenty of chains (>= 2 x 8 warps x SMs): 8 worker warps per SM, fixed
//     chunk; the FIFO is a dynamic tile scheduler with a short tail;
//   * fewer chains (BASELINE config 2: 1024 chains, 592 sub-partitions): one
//     worker warp per sub-partition and the chunk COUNT K chosen so that
//     chains x K is as close as possible below a multiple of the worker count
//     (1024 x 37 = 592 x 64): every sub-partition stays busy to the end
//     instead of 1024 warps sitting unevenly on 592 sub-partitions (-14%).
// mk2_set_block_threads / mk2_set_chunk_clocks override the automatic choice.
// ---------------------------------------------------------------------------
struct Plan {
    int tg;           // row-major only: 8-clock groups per drain (16 or 32)
    int block;        // threads per CTA (4, 7 or 8 worker warps unless overridden), one CTA per SM
    uint32_t chunk;   // clocks per chunk
    uint32_t cpc;     // chunks per chain
    unsigned grid;
    bool tmem;        // row-major only: staging tile in tensor memory (mk2_tmem.cuh)
    bool row64;       // Grain row-major: 512-clock tiles, 64 bytes per row and drain (mk2_grain_row64.cuh)
    bool rowl2;       // ... with every warp's tile in L2-resident global scratch
    bool ring;        // Grain row-major: four lone warps per SM, drains pipelined into the next tile (mk2_grain_ring.cuh)
    bool row8;        // Grain row-major: eight warps per SM, 28 groups of the tile in shared + 4 in tensor memory
};

Plan make_plan(const mk2_ctx *ctx, uint64_t T, bool rowmajor, uint64_t chains, bool ring_ok = false)
{
    const uint64_t sms = (uint64_t)ctx->sm_count;
    Plan p{};
    // row-major: 7 warps per SM x 1 KiB per thread = 224 KiB of the 227 KiB shared memory leave room
    // for 256-clock (full 32-byte sector) staging tiles
    // row-major staging in tensor memory (MICKEY only): eight 256-clock tiles fit, shared memory holds seven
    p.tmem = rowmajor && ctx->cipher == 0 && ctx->row_staging != 1;
    p.block = ctx->block_user ? ctx->block_user : (chains >= 16 * sms ? (rowmajor && !p.tmem ? 224 : 256) : 128);
    p.tg = p.tmem || p.block <= 224 ? 32 : 16;  // smem strides: <= 128 -> 128, <= 192 -> 192, <= 224 -> 224, else (16, 256)
    // Grain row-major with mk2_set_row_staging(ctx, 2): 512-clock tiles (64 contiguous bytes per row and drain),
    // four in tensor memory and three and a half in shared memory.  NOT the default: it takes DRAM out of the
    // picture (17% busy instead of the limiter) but its staging instructions cost what that returns
    // (9.9-10.1 Tb/s against 10.4 for the 256-clock shared-memory kernel, Grain section).
    p.row64 = rowmajor && ctx->cipher == 1 && ctx->row_staging == 2 && !ctx->block_user;
    p.rowl2 = rowmajor && ctx->cipher == 1 && ctx->row_staging == 3;
    if (p.row64) {
        p.block = grain::row64::THREADS;
        p.tg = grain::row64::NGRP;
    }
    if (p.rowl2) {
        p.block = ctx->block_user ? ctx->block_user : BLOCK;
        p.tg = grain::row64::NGRP;
    }
    p.ring = ring_ok && rowmajor && ctx->cipher == 1 && ctx->row_staging == 4;
    if (p.ring) {
        p.block = grain::ring::THREADS;
        p.tg = grain::ring::TILE_GROUPS;
    }
    // whole chains only (tcgen05 is warp-collective); plenty of chains, or it has no eighth warp to fill
    p.row8 = ring_ok && rowmajor && ctx->cipher == 1 && ctx->row_staging == 5 && ctx->N % 1024 == 0 && !ctx->block_user;
    if (p.row8) {
        p.block = grain::row8::THREADS;
        p.tg = 32;
    }
    const uint32_t granule = rowmajor ? 8u * (uint32_t)p.tg : (ctx->cipher == 1 ? (uint32_t)grain::CWIN : 1u);
    auto round_chunk = [&](uint64_t c) {
        c = std::max<uint64_t>(c, granule);
        c = (c + granule - 1) / granule * granule;
        return (uint32_t)std::min<uint64_t>(c, 0x7FFFFF00ull);
    };
    const uint64_t workers = sms * (uint64_t)(p.block / 32);
    if (ctx->chunk_user) {
        p.chunk = round_chunk(ctx->chunk_user);
    } else if (chains >= 2 * workers || chains <= workers) {
        // Grain row-major: longer chunks (fewer state reloads at 37 LOP3 per clock; measured 9.9 -> 10.1 Tb/s)
        const uint64_t many = rowmajor && ctx->cipher == 1 ? 16384 : 4096;
        p.chunk = round_chunk(std::min<uint64_t>(T, chains <= workers ? T : many));
    } else {
        // workers < chains < 2 x workers: pick K for the least idle time in the last round
        const uint64_t kmax = std::max<uint64_t>(1, std::min<uint64_t>(128, T / 1024));
        double best = 1e30;
        uint64_t best_k = 1;
        for (uint64_t k = 1; k <= kmax; ++k) {
            const uint32_t c = round_chunk((T + k - 1) / k);
            const uint64_t keff = (T + c - 1) / c;
            const uint64_t jobs = chains * keff;
            const double rounds = (double)((jobs + workers - 1) / workers);
            // time ~ rounds x (chunk length + hand-off); a hand-off costs about 30 clocks' worth
            // (~10 us, exposed because a lone warp has no partner to overlap it with)
            const double cost = rounds * ((double)c + 30.0);
            if (cost < best * 0.998) {
                best = cost;
                best_k = k;
            }
        }
        p.chunk = round_chunk((T + best_k - 1) / best_k);
    }
    p.cpc = (uint32_t)((T + p.chunk - 1) / p.chunk);
    p.grid = (unsigned)std::min<uint64_t>(sms, (chains + p.block / 32 - 1) / (p.block / 32));
    if (chains > workers) p.grid = (unsigned)sms;
    if (ctx->max_grid) p.grid = std::min(p.grid, ctx->max_grid);
    return p;
}

// Scheduler reset for one launch.
int launch_sched(mk2_ctx *ctx, const Plan &p, uint64_t chains)
{
    if ((uint64_t)p.cpc * chains >= 0xFFFFFFFFull) return fail(ctx, MK2_E_ARG, "too many chunks: raise mk2_set_chunk_clocks");
    sched_init_kernel<<<(ctx->ring + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_queue, ctx->d_slots, ctx->d_progress,
                                                                        (uint32_t)chains, p.cpc, ctx->ring);
    CK(cudaGetLastError());
    ctx->last_launches++;
    ctx->last_plan_block = p.block;
    ctx->last_plan_chunk = p.chunk;
    return MK2_OK;
}

int launch_col(mk2_ctx *ctx, uint64_t T, uint32_t *out, uint64_t stride)
{
    const uint64_t chains = (ctx->G + 31) / 32;
    if (ctx->cipher == 0 && ctx->small_batch && ctx->G <= COOP_MAX_GROUPS && !ctx->trace.rec) {
        coop::gen_colmajor_kernel<<<coop_grid(ctx), 32 * coop::WARPS, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, out, stride,
                                                                                        ctx->G, T);
        CK(cudaGetLastError());
        ctx->last_launches++;
        ctx->last_plan_block = 32 * coop::WARPS;
        ctx->last_plan_chunk = (uint32_t)std::min<uint64_t>(T, 0x7FFFFF00ull);
        return MK2_OK;
    }
    const Plan p = make_plan(ctx, T, false, chains);
    int rc = launch_sched(ctx, p, chains);
    if (rc) return rc;
    if (ctx->cipher == 1 && ctx->row_staging == 4 && T % grain::WIN == 0)
        grain::gen_colmajor_circ_kernel<<<p.grid, p.block, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc,
                                                                             out, stride, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                                                                             ctx->d_slots, ctx->ring - 1, ctx->d_progress);
    else if (ctx->cipher == 1)
        grain::gen_colmajor_kernel<<<p.grid, p.block, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc,
                                                                        out, stride, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                                                                        ctx->d_slots, ctx->ring - 1, ctx->d_progress);
    else
        gen_colmajor_kernel<<<p.grid, p.block, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out,
                                                                 stride, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                                                                 ctx->d_slots, ctx->ring - 1, ctx->d_progress, ctx->trace);
    CK(cudaGetLastError());
    ctx->last_launches++;
    return MK2_OK;
}

// Row-major keystream of chains [chain_base, chain_base + nchains); `out` = row of the first
// instance of chain_base.
int launch_row(mk2_ctx *ctx, uint64_t T, uint8_t *out, uint64_t pitch, uint64_t chain_base, uint64_t nchains)
{
    if (ctx->cipher == 0 && ctx->small_batch && ctx->G <= COOP_MAX_GROUPS && chain_base == 0 && nchains == (ctx->G + 31) / 32) {
        if (ctx->row_lsb)
            coop::gen_rowmajor_kernel<true><<<coop_grid(ctx), 32 * coop::WARPS, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, out, pitch,
                                                                                               ctx->N, ctx->G, T);
        else
            coop::gen_rowmajor_kernel<false><<<coop_grid(ctx), 32 * coop::WARPS, 0, ctx->stream>>>(ctx->d_state, ctx->d_acc, out, pitch,
                                                                                                ctx->N, ctx->G, T);
        CK(cudaGetLastError());
        ctx->last_launches++;
        ctx->last_plan_block = 32 * coop::WARPS;
        ctx->last_plan_chunk = (uint32_t)std::min<uint64_t>(T, 0x7FFFFF00ull);
        return MK2_OK;
    }
    const bool aligned = (reinterpret_cast<uintptr_t>(out) % 16 == 0) && (pitch % 16 == 0);
    // the lone-warp ring kernel takes only full tiles, whole groups and 32-byte aligned rows
    const bool ring_ok = (reinterpret_cast<uintptr_t>(out) % 32 == 0) && (pitch % 32 == 0) && T % 256 == 0 && ctx->N % 32 == 0;
    const Plan p = make_plan(ctx, T, true, nchains, ring_ok);  // chunks are whole staging tiles
    int rc = launch_sched(ctx, p, nchains);
    if (rc) return rc;
    if (p.row8) {
        if (ctx->row_lsb)
            grain::row8::gen_rowmajor_kernel<true><<<p.grid, p.block, grain::row8::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base);
        else
            grain::row8::gen_rowmajor_kernel<false><<<p.grid, p.block, grain::row8::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base);
        CK(cudaGetLastError());
        ctx->last_launches++;
        return MK2_OK;
    }
    if (p.ring) {
        if (ctx->row_lsb)
            grain::ring::gen_rowmajor_kernel<true><<<p.grid, p.block, grain::ring::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base);
        else
            grain::ring::gen_rowmajor_kernel<false><<<p.grid, p.block, grain::ring::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base);
        CK(cudaGetLastError());
        ctx->last_launches++;
        return MK2_OK;
    }
    if (p.rowl2) {
        if (!ctx->d_rowscratch)
            CK(cudaMalloc(&ctx->d_rowscratch, (size_t)ctx->sm_count * (BLOCK / 32) * grain::row64::L2TILE_BYTES_PER_WARP));
        if (ctx->row_lsb)
            grain::row64::gen_rowmajor_l2_kernel<true><<<p.grid, p.block, 0, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base, aligned, ctx->d_rowscratch);
        else
            grain::row64::gen_rowmajor_l2_kernel<false><<<p.grid, p.block, 0, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base, aligned, ctx->d_rowscratch);
        CK(cudaGetLastError());
        ctx->last_launches++;
        return MK2_OK;
    }
    if (p.row64) {
        if (ctx->row_lsb)
            grain::row64::gen_rowmajor_kernel<true><<<p.grid, p.block, grain::row64::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base, aligned);
        else
            grain::row64::gen_rowmajor_kernel<false><<<p.grid, p.block, grain::row64::SMEM_BYTES, ctx->stream>>>(
                ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc, ctx->d_queue,
                ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base, aligned);
        CK(cudaGetLastError());
        ctx->last_launches++;
        return MK2_OK;
    }
    // staging geometry: (TG, stride) = (32, 128) | (32, 192) | (32, 224) | (16, 256); the stride is a template
    // parameter so that every smem offset in the drain loops is an immediate
    const int ts = p.tg == 32 ? (p.block <= 128 ? 128 : p.block <= 192 ? 192 : 224) : 256;
    const size_t smem = (size_t)row_smem_bytes(p.tg, ts);
#define MK2_ROW_LAUNCH1(AL, TGV, TSV, LSBV)                                                                  \
    gen_rowmajor_kernel<AL, TGV, TSV, LSBV><<<p.grid, p.block, smem, ctx->stream>>>(                        \
        ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc,  \
        ctx->d_queue, ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base)
#define MK2_ROW_LAUNCH(AL, TGV, TSV)                          \
    do {                                                      \
        if (ctx->row_lsb) MK2_ROW_LAUNCH1(AL, TGV, TSV, true); \
        else MK2_ROW_LAUNCH1(AL, TGV, TSV, false);            \
    } while (0)
#define MK2_GRAIN_ROW_LAUNCH(AL, TGV, TSV, LSBV)                                                              \
    grain::gen_rowmajor_kernel<AL, TGV, TSV, LSBV><<<p.grid, p.block, smem, ctx->stream>>>(                  \
        ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc,  \
        ctx->d_queue, ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base)
#define MK2_GRAIN_ROW_PICK(TGV, TSV)                                                   \
    do {                                                                               \
        if (aligned && ctx->row_lsb) MK2_GRAIN_ROW_LAUNCH(true, TGV, TSV, true);       \
        else if (aligned) MK2_GRAIN_ROW_LAUNCH(true, TGV, TSV, false);                 \
        else if (ctx->row_lsb) MK2_GRAIN_ROW_LAUNCH(false, TGV, TSV, true);            \
        else MK2_GRAIN_ROW_LAUNCH(false, TGV, TSV, false);                             \
    } while (0)
#define MK2_TMEM_ROW_LAUNCH(AL, LSBV)                                                                        \
    tmem::gen_rowmajor_kernel<AL, LSBV><<<p.grid, p.block, 0, ctx->stream>>>(                                \
        ctx->d_state, ctx->d_acc, ctx->d_state, ctx->d_acc, out, pitch, ctx->N, ctx->G, T, p.chunk, p.cpc,  \
        ctx->d_queue, ctx->d_slots, ctx->ring - 1, ctx->d_progress, (uint32_t)chain_base)
    if (p.tmem) {
        if (aligned && ctx->row_lsb) MK2_TMEM_ROW_LAUNCH(true, true);
        else if (aligned) MK2_TMEM_ROW_LAUNCH(true, false);
        else if (ctx->row_lsb) MK2_TMEM_ROW_LAUNCH(false, true);
        else MK2_TMEM_ROW_LAUNCH(false, false);
    } else if (ctx->cipher == 1) {
        if (ts == 128) MK2_GRAIN_ROW_PICK(32, 128);
        else if (ts == 192) MK2_GRAIN_ROW_PICK(32, 192);
        else if (ts == 224) MK2_GRAIN_ROW_PICK(32, 224);
        else MK2_GRAIN_ROW_PICK(16, 256);
    } else if (ts == 128) {
        if (aligned) MK2_ROW_LAUNCH(true, 32, 128); else MK2_ROW_LAUNCH(false, 32, 128);
    } else if (ts == 192) {
        if (aligned) MK2_ROW_LAUNCH(true, 32, 192); else MK2_ROW_LAUNCH(false, 32, 192);
    } else if (ts == 224) {
        if (aligned) MK2_ROW_LAUNCH(true, 32, 224); else MK2_ROW_LAUNCH(false, 32, 224);
    } else {
        if (aligned) MK2_ROW_LAUNCH(true, 16, 256); else MK2_ROW_LAUNCH(false, 16, 256);
    }
#undef MK2_TMEM_ROW_LAUNCH
#undef MK2_ROW_LAUNCH
#undef MK2_ROW_LAUNCH1
#undef MK2_GRAIN_ROW_PICK
#undef MK2_GRAIN_ROW_LAUNCH
    CK(cudaGetLastError());
    ctx->last_launches++;
    return MK2_OK;
}

// host-output helper: make staging buffer b safe to overwrite
int acquire_stage(mk2_ctx *ctx, int b)
{
    if (ctx->copy_pending[b]) {
        CK(cudaStreamWaitEvent(ctx->stream, ctx->copy_done[b], 0));
        ctx->copy_pending[b] = false;
    }
    return MK2_OK;
}

int drain_copies(mk2_ctx *ctx)
{
    CK(cudaStreamSynchronize(ctx->copy));
    ctx->copy_pending[0] = ctx->copy_pending[1] = false;
    return MK2_OK;
}

// D2H side of a host-output call.  Tile i is generated into device staging buffer b = i & 1; the caller does
//     b = next(); acquire(b); <launch the kernel into d_stage[b]>; copy_out(b, ...)
//   pinned destination   -> one async (2-D) copy on the copy stream, straight into the array; acquire() makes the
//                           launch stream wait for the copy that last read the buffer;
//   pageable destination -> the tile is queued for the copy lanes (HostCopyLanes), which start on it as soon as
//                           its kernel has finished; acquire() blocks the calling thread until the lanes have
//                           moved the tile that last used the buffer.
// finish() waits for everything (the API returns with the array complete).
class HostTiles {
public:
    // Small pageable outputs are not worth the lanes: the driver's own staged copy handles them.
    HostTiles(mk2_ctx *c, Mem dst, uint64_t total_bytes) : ctx(c), bounce(dst == Mem::Pageable && total_bytes >= BOUNCE_MIN_BYTES) {}
    ~HostTiles()
    {
        // never leave lanes writing into the caller's array (or reading a staging buffer) after the call returned
        if (bounce && ctx->lanes)
            for (auto &t : inflight) ctx->lanes->wait(t);
    }
    bool pageable() const { return bounce; }
    int prepare() { return bounce ? ensure_lanes(ctx) : MK2_OK; }
    int next() { return (int)(count++ & 1); }
    int acquire(int b)
    {
        if (!bounce) return acquire_stage(ctx, b);
        return reclaim(b);
    }
    // rows x width bytes from staging buffer b (pitch spitch) to dst (pitch dpitch)
    int copy_out(int b, uint8_t *dst, size_t dpitch, size_t spitch, size_t width, size_t rows)
    {
        CK(cudaEventRecord(ctx->gen_done[b], ctx->stream));
        if (bounce) {
            inflight[b] = ctx->lanes->post(ctx->d_stage[b], spitch, dst, dpitch, width, rows, ctx->gen_done[b]);
            return MK2_OK;
        }
        CK(cudaStreamWaitEvent(ctx->copy, ctx->gen_done[b], 0));
        if (dpitch == width && spitch == width)
            CK(cudaMemcpyAsync(dst, ctx->d_stage[b], width * rows, cudaMemcpyDeviceToHost, ctx->copy));
        else
            CK(cudaMemcpy2DAsync(dst, dpitch, ctx->d_stage[b], spitch, width, rows, cudaMemcpyDeviceToHost, ctx->copy));
        CK(cudaEventRecord(ctx->copy_done[b], ctx->copy));
        ctx->copy_pending[b] = true;
        return MK2_OK;
    }
    int finish()
    {
        if (bounce) {
            int rc;
            const int last = (int)((count + 1) & 1);  // older tile first
            if ((rc = reclaim(last ^ 1)) || (rc = reclaim(last))) return rc;
            return MK2_OK;
        }
        return drain_copies(ctx);
    }

private:
    int reclaim(int b)
    {
        if (!inflight[b]) return MK2_OK;
        const int e = ctx->lanes->wait(inflight[b]);
        inflight[b].reset();
        if (e) return fail(ctx, MK2_E_CUDA, std::string("copy lane: ") + cudaGetErrorString((cudaError_t)e));
        return MK2_OK;
    }
    mk2_ctx *ctx;
    bool bounce;
    uint64_t count = 0;
    HostCopyLanes::TilePtr inflight[2];
};

int check_ready(mk2_ctx *ctx)
{
    if (!ctx) return MK2_E_ARG;
    if (!ctx->ready) return fail(ctx, MK2_E_STATE, "context holds no key/IV material: call mk2_init_* first");
    return MK2_OK;
}

// Every entry point that touches CUDA: NULL check, then run on the context's device and put the caller's
// current device back on return.
#define MK2_ENTER(c)                                                                   \
    if (!(c)) return MK2_E_ARG;                                                        \
    DeviceGuard device_guard_((c)->device);                                            \
    if (!device_guard_.ok) return fail((c), MK2_E_CUDA, "cudaSetDevice failed")

// Opt-in to > 48 KiB of dynamic shared memory for the shared-memory row-major kernels: a per-device function
// attribute, set once per process and device instead of 24 cudaFuncSetAttribute calls per context.
cudaError_t opt_in_row_kernels(int device)
{
    static std::mutex m;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lk(m);
    if (device >= 0 && device < 64 && done[device]) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    const int row_smem_max = row_smem_bytes(32, 224);  // the largest staging tile: 224 KiB
    auto opt_in = [&](auto kernel) {
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, row_smem_max);
    };
#define MK2_OPT_IN_MICKEY(TGV, TSV)                          \
    opt_in(gen_rowmajor_kernel<true, TGV, TSV, true>);       \
    opt_in(gen_rowmajor_kernel<true, TGV, TSV, false>);      \
    opt_in(gen_rowmajor_kernel<false, TGV, TSV, true>);      \
    opt_in(gen_rowmajor_kernel<false, TGV, TSV, false>)
    MK2_OPT_IN_MICKEY(32, 128);
    MK2_OPT_IN_MICKEY(32, 192);
    MK2_OPT_IN_MICKEY(32, 224);
    MK2_OPT_IN_MICKEY(16, 256);
#undef MK2_OPT_IN_MICKEY
#define MK2_OPT_IN_GRAIN(TGV, TSV)                                  \
    opt_in(grain::gen_rowmajor_kernel<true, TGV, TSV, true>);       \
    opt_in(grain::gen_rowmajor_kernel<true, TGV, TSV, false>);      \
    opt_in(grain::gen_rowmajor_kernel<false, TGV, TSV, true>);      \
    opt_in(grain::gen_rowmajor_kernel<false, TGV, TSV, false>)
    MK2_OPT_IN_GRAIN(32, 128);
    MK2_OPT_IN_GRAIN(32, 192);
    MK2_OPT_IN_GRAIN(32, 224);
    MK2_OPT_IN_GRAIN(16, 256);
#undef MK2_OPT_IN_GRAIN
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::row8::gen_rowmajor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::row8::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::row8::gen_rowmajor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::row8::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::ring::gen_rowmajor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::ring::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::ring::gen_rowmajor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::ring::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::row64::gen_rowmajor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::row64::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grain::row64::gen_rowmajor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 grain::row64::SMEM_BYTES);
    if (e == cudaSuccess && device >= 0 && device < 64) done[device] = true;
    return e;
}

}  // namespace

extern "C" {

int mk2_abi_version(void) { return 2; }

int mk2_lop3_per_clock(void) { return 327; }
static int rblock_of(int kernel)
{
    return kernel == 1 ? mk2::tmem::RBLOCK : kernel == 2 ? mk2::RBLOCK_INIT : mk2::RBLOCK_COL;
}
int mk2_rblock(int kernel) { return rblock_of(kernel); }
int mk2_lop3_per_block(int kernel)
{
    // evaluated at compile time from the tables the clock code is generated from
    static constexpr int count[mk2::MAX_RBLOCK + 1] = {0, 327, mk2::block_lop3_count(2), mk2::block_lop3_count(3),
                                                       mk2::block_lop3_count(4), mk2::block_lop3_count(5),
                                                       mk2::block_lop3_count(6)};
    return count[rblock_of(kernel)];
}

int mk2_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int mk2_create(int device, mk2_ctx **out)
{
    mk2_ctx *ctx = nullptr;  // CK() reports into g_create_error while ctx == nullptr
    if (!out) return fail(nullptr, MK2_E_ARG, "out is NULL");
    *out = nullptr;
    int n = mk2_device_count();
    if (n <= 0) return fail(nullptr, MK2_E_NODEVICE, "no CUDA device visible; this library has no CPU fallback");
    if (device < 0 || device >= n) return fail(nullptr, MK2_E_ARG, "device index out of range");
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(nullptr, MK2_E_NODEVICE,
                    std::string("device is sm_") + std::to_string(prop.major) + std::to_string(prop.minor) +
                        "; the kernels are built for sm_100a only");
    DeviceGuard guard(device);
    if (!guard.ok) return fail(nullptr, MK2_E_CUDA, "cudaSetDevice failed");
    mk2_ctx *c = new (std::nothrow) mk2_ctx();
    if (!c) return fail(nullptr, MK2_E_NOMEM, "out of host memory");
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    // experiment knob (tools/probe_grain_l2_persist.sh): L2 set-aside for persisting (evict_last) lines, in MiB
    if (const char *v = std::getenv("MK2_L2_PERSIST_MB")) {
        const size_t want = std::min<size_t>((size_t)std::strtoull(v, nullptr, 0) << 20, (size_t)prop.persistingL2CacheMaxSize);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
        std::fprintf(stderr, "mk2: persisting L2 set-aside %zu MiB (max %d MiB, L2 %d MiB)\n", got >> 20,
                     prop.persistingL2CacheMaxSize >> 20, prop.l2CacheSize >> 20);
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&c->gen_done[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->copy_done[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        e = cudaMemPoolCreate(&c->pool, &props);
        if (e == cudaSuccess) {
            // scratch freed with cudaFreeAsync stays in the pool instead of being unmapped at the next
            // synchronisation (the default pool's behaviour cost ~40 ms per 1.3 GB re-allocation)
            unsigned long long keep = ~0ull;
            e = cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_sum, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_queue, sizeof(SchedQueue));
    if (e == cudaSuccess) e = opt_in_row_kernels(device);
    if (e != cudaSuccess) {
        std::string msg = std::string("context setup: ") + cudaGetErrorString(e);
        mk2_destroy(c);
        return fail(nullptr, MK2_E_CUDA, msg);
    }
    c->stream = c->own;
    *out = c;
    return MK2_OK;
}

int mk2_destroy(mk2_ctx *ctx)
{
    if (!ctx) return MK2_OK;
    DeviceGuard guard(ctx->device);
    delete ctx->lanes;
    ctx->lanes = nullptr;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy) cudaStreamSynchronize(ctx->copy);
    if (ctx->h2d) cudaStreamSynchronize(ctx->h2d);
    for (int b = 0; b < 2; ++b) {
        if (ctx->d_bulk_in[b]) cudaFree(ctx->d_bulk_in[b]);
        if (ctx->h2d_done[b]) cudaEventDestroy(ctx->h2d_done[b]);
        if (ctx->mat_used[b]) cudaEventDestroy(ctx->mat_used[b]);
        if (ctx->d_stage[b]) cudaFree(ctx->d_stage[b]);
        if (ctx->gen_done[b]) cudaEventDestroy(ctx->gen_done[b]);
        if (ctx->copy_done[b]) cudaEventDestroy(ctx->copy_done[b]);
    }
    if (ctx->d_state) cudaFree(ctx->d_state);
    if (ctx->d_acc) cudaFree(ctx->d_acc);
    if (ctx->d_sum) cudaFree(ctx->d_sum);
    if (ctx->d_queue) cudaFree(ctx->d_queue);
    if (ctx->d_rowscratch) cudaFree(ctx->d_rowscratch);
    if (ctx->trace.rec) cudaFree(ctx->trace.rec);
    if (ctx->trace.count) cudaFree(ctx->trace.count);
    if (ctx->d_slots) cudaFree(ctx->d_slots);
    if (ctx->d_progress) cudaFree(ctx->d_progress);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    delete ctx;
    return MK2_OK;
}

int mk2_set_stream(mk2_ctx *ctx, void *cuda_stream)
{
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);  // 0 is a real stream: the legacy default stream
    return MK2_OK;
}

int mk2_use_own_stream(mk2_ctx *ctx)
{
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stream = ctx->own;
    return MK2_OK;
}

int mk2_set_trace(mk2_ctx *ctx, uint64_t capacity)
{
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->trace.rec) cudaFree(ctx->trace.rec);
    if (ctx->trace.count) cudaFree(ctx->trace.count);
    ctx->trace = {nullptr, nullptr, 0};
    if (capacity) {
        CK(cudaMalloc(&ctx->trace.rec, sizeof(TraceRec) * capacity));
        CK(cudaMalloc(&ctx->trace.count, sizeof(unsigned long long)));
        CK(cudaMemset(ctx->trace.count, 0, sizeof(unsigned long long)));
        ctx->trace.capacity = capacity;
    }
    return MK2_OK;
}

int mk2_read_trace(mk2_ctx *ctx, void *records, uint64_t max_records, uint64_t *count)
{
    if (!ctx || !count) return MK2_E_ARG;
    *count = 0;
    if (!ctx->trace.rec) return MK2_OK;
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    unsigned long long n = 0;
    CK(cudaMemcpy(&n, ctx->trace.count, sizeof n, cudaMemcpyDeviceToHost));
    n = std::min<unsigned long long>(n, std::min<unsigned long long>(ctx->trace.capacity, max_records));
    if (n && records) CK(cudaMemcpy(records, ctx->trace.rec, sizeof(TraceRec) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemset(ctx->trace.count, 0, sizeof(unsigned long long)));
    *count = n;
    return MK2_OK;
}

int mk2_last_plan(const mk2_ctx *ctx, int *block_threads, uint32_t *chunk_clocks)
{
    if (!ctx) return MK2_E_ARG;
    if (block_threads) *block_threads = ctx->last_plan_block;
    if (chunk_clocks) *chunk_clocks = ctx->last_plan_chunk;
    return MK2_OK;
}

int mk2_set_max_ctas(mk2_ctx *ctx, uint32_t ctas)
{
    if (!ctx) return MK2_E_ARG;
    ctx->max_grid = ctas;
    return MK2_OK;
}

int mk2_set_chunk_clocks(mk2_ctx *ctx, uint32_t clocks)
{
    if (!ctx) return MK2_E_ARG;
    if (clocks != 0 && clocks < 128) return fail(ctx, MK2_E_ARG, "chunk must be 0 (auto) or at least 128 clocks");
    ctx->chunk_user = clocks;
    return MK2_OK;
}

int mk2_set_row_staging(mk2_ctx *ctx, int mode)
{
    if (!ctx) return MK2_E_ARG;
    if (mode < 0 || mode > 5)
        return fail(ctx, MK2_E_ARG,
                    "row staging mode must be 0 (automatic), 1 (shared memory), 2 (tensor memory), 3 (L2 scratch), 4 (Grain ring) "
                    "or 5 (Grain, eight warps)");
    ctx->row_staging = mode;
    return MK2_OK;
}

int mk2_set_small_batch(mk2_ctx *ctx, int enable)
{
    if (!ctx) return MK2_E_ARG;
    ctx->small_batch = enable ? 1 : 0;
    return MK2_OK;
}

int mk2_set_bulk_fused(mk2_ctx *ctx, int mode)
{
    if (!ctx) return MK2_E_ARG;
    if (mode < 0 || mode > 2) return fail(ctx, MK2_E_ARG, "bulk fused mode must be 0 (never), 1 (automatic) or 2 (whenever eligible)");
    ctx->bulk_fused = mode;
    return MK2_OK;
}

int mk2_set_stage_bytes(mk2_ctx *ctx, uint64_t bytes)
{
    if (!ctx) return MK2_E_ARG;
    if (bytes && bytes < (1u << 20)) return fail(ctx, MK2_E_ARG, "stage bytes must be 0 (default) or at least 1 MiB");
    ctx->stage_target = bytes ? (size_t)bytes : STAGE_BYTES;
    ctx->stage_user = bytes != 0;
    return MK2_OK;
}

int mk2_set_block_threads(mk2_ctx *ctx, int threads)
{
    if (!ctx) return MK2_E_ARG;
    if (threads == 0) {
        ctx->block_user = 0;
        return MK2_OK;
    }
    if (threads < 32 || threads > BLOCK || threads % 32) return fail(ctx, MK2_E_ARG, "threads per CTA must be 0 (auto) or 32..256 in steps of 32");
    ctx->block_user = threads;
    return MK2_OK;
}

int mk2_set_host_threads(mk2_ctx *ctx, int threads)
{
    if (!ctx) return MK2_E_ARG;
    if (threads < 0 || threads > 256) return fail(ctx, MK2_E_ARG, "host threads must be 0 (automatic) or 1..256");
    if (threads != ctx->host_threads) {
        delete ctx->lanes;  // idle between calls; re-created with the new size on next use
        ctx->lanes = nullptr;
        ctx->host_threads = threads;
    }
    return MK2_OK;
}

int mk2_host_alloc(size_t bytes, void **out)
{
    if (!out) return MK2_E_ARG;
    *out = nullptr;
    if (bytes == 0) return MK2_OK;
    const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(nullptr, e == cudaErrorMemoryAllocation ? MK2_E_NOMEM : MK2_E_CUDA,
                    std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    return MK2_OK;
}

int mk2_host_free(void *p)
{
    if (!p) return MK2_OK;
    if (cudaFreeHost(p) != cudaSuccess) {
        cudaGetLastError();
        return MK2_E_CUDA;
    }
    return MK2_OK;
}

int mk2_set_async(mk2_ctx *ctx, int async)
{
    if (!ctx) return MK2_E_ARG;
    ctx->async = async != 0;
    return MK2_OK;
}

int mk2_trim(mk2_ctx *ctx)
{
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->copy));
    for (int b = 0; b < 2; ++b) {
        if (ctx->d_stage[b]) cudaFree(ctx->d_stage[b]);
        ctx->d_stage[b] = nullptr;
        ctx->copy_pending[b] = false;
    }
    ctx->stage_bytes = 0;
    CK(cudaMemPoolTrimTo(ctx->pool, 0));
    return MK2_OK;
}

int mk2_sync(mk2_ctx *ctx)
{
    MK2_ENTER(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->copy));
    if (ctx->timing_open) {
        CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
        ctx->timing_open = false;
    }
    return MK2_OK;
}

const char *mk2_last_error(const mk2_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int mk2_set_group_offset(mk2_ctx *ctx, uint64_t group_offset)
{
    if (!ctx) return MK2_E_ARG;
    ctx->g_offset = group_offset;
    return MK2_OK;
}

int mk2_query(const mk2_ctx *ctx, uint64_t *N, uint64_t *G, uint64_t *clocks)
{
    if (!ctx) return MK2_E_ARG;
    if (N) *N = ctx->N;
    if (G) *G = ctx->G;
    if (clocks) *clocks = ctx->clocks;
    return MK2_OK;
}

float mk2_last_kernel_ms(const mk2_ctx *ctx) { return ctx ? ctx->last_ms : -1.f; }
int mk2_last_kernel_launches(const mk2_ctx *ctx) { return ctx ? ctx->last_launches : 0; }

static int init_common(mk2_ctx *ctx, uint64_t N)
{
    if (N == 0) return fail(ctx, MK2_E_ARG, "at least one lane is required");
    const uint64_t G = (N + 31) / 32;
    ctx->ready = false;  // whatever happens from here on, the previous state is no longer valid
    int rc = ensure_capacity(ctx, G);
    if (rc) return rc;
    ctx->N = N;
    ctx->G = G;
    return MK2_OK;
}

// pack + key/IV load + pre-clock of the ctx->N instances whose material is on the device
static int init_uniform_device(mk2_ctx *ctx, const uint8_t *dk, const uint8_t *di, uint32_t iv_stride, uint32_t iv_bits)
{
    int rc;
    Scratch scratch(ctx);
    void *matp = nullptr;
    const int load = (int)iv_bits + KEY_BITS;
    if ((rc = scratch.alloc(&matp, sizeof(uint32_t) * (size_t)load * ctx->G))) return rc;
    uint32_t *mat = static_cast<uint32_t *>(matp);
    const bool fast10 = reinterpret_cast<uintptr_t>(dk) % 16 == 0 &&
                        (!iv_bits || (iv_stride == 10 && reinterpret_cast<uintptr_t>(di) % 16 == 0));
    pack_uniform_kernel<<<blocks_for(ctx->G), BLOCK, 0, ctx->stream>>>(dk, di, iv_stride, (int)iv_bits, ctx->N, ctx->G, mat,
                                                                        fast10);
    CK(cudaGetLastError());
    ctx->last_launches++;
    return launch_init(ctx, mat, load, 0, false);
}

int mk2_init_from_material(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride,
                           uint32_t iv_bits, uint64_t N)
{
    MK2_ENTER(ctx);
    if (!keys) return fail(ctx, MK2_E_ARG, "keys is NULL");
    if (iv_bits > 80) return fail(ctx, MK2_E_ARG, "IV must be at most 80 bits");
    if (iv_bits && (!ivs || iv_stride < (iv_bits + 7) / 8)) return fail(ctx, MK2_E_ARG, "ivs/iv_stride too small for iv_bits");
    int rc = init_common(ctx, N);
    if (rc) return rc;
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    const uint8_t *dk = nullptr, *di = nullptr;
    if ((rc = stage_input(ctx, scratch, keys, N * 10, &dk))) return rc;
    if ((rc = stage_input(ctx, scratch, iv_bits ? ivs : nullptr, N * (size_t)iv_stride, &di))) return rc;
    if ((rc = init_uniform_device(ctx, dk, di, iv_stride, iv_bits))) return rc;
    return end_timing(ctx);
}

int mk2_init_ragged(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride,
                    const uint8_t *iv_nbits, uint64_t N)
{
    MK2_ENTER(ctx);
    if (!keys || !iv_nbits) return fail(ctx, MK2_E_ARG, "keys / iv_nbits is NULL");
    if (N == 0) return fail(ctx, MK2_E_ARG, "at least one lane is required");
    // the lengths steer the launch, so they are needed on the host
    std::string lens(N, '\0');
    if (is_device_ptr(iv_nbits)) {
        CK(cudaMemcpyAsync(&lens[0], iv_nbits, N, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    } else {
        std::memcpy(&lens[0], iv_nbits, N);
    }
    int lmax = 0;
    for (uint64_t n = 0; n < N; ++n) {
        const unsigned l = (unsigned char)lens[n];
        if (l == MK2_IV_UNUSED) continue;
        if (l > 80) return fail(ctx, MK2_E_ARG, "lane " + std::to_string(n) + ": IV must be at most 80 bits");
        lmax = std::max(lmax, (int)l);
    }
    if (lmax && (!ivs || iv_stride < (uint32_t)(lmax + 7) / 8)) return fail(ctx, MK2_E_ARG, "ivs/iv_stride too small");
    int rc = init_common(ctx, N);
    if (rc) return rc;
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    const uint8_t *dk = nullptr, *di = nullptr, *dn = nullptr;
    void *matp = nullptr;
    if ((rc = stage_input(ctx, scratch, keys, N * 10, &dk))) return rc;
    if ((rc = stage_input(ctx, scratch, lmax ? ivs : nullptr, N * (size_t)iv_stride, &di))) return rc;
    if ((rc = stage_input(ctx, scratch, iv_nbits, N, &dn))) return rc;
    const int load = lmax + KEY_BITS;
    if ((rc = scratch.alloc(&matp, sizeof(uint32_t) * (size_t)(2 * lmax + KEY_BITS + 1) * ctx->G))) return rc;
    uint32_t *mat = static_cast<uint32_t *>(matp);
    auto al16 = [](const void *q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
    const bool fast10 = al16(dk) && al16(dn) && (!lmax || (iv_stride == 10 && al16(di)));
    pack_ragged_kernel<<<blocks_for(ctx->G), BLOCK, 0, ctx->stream>>>(dk, di, iv_stride, dn, lmax, N, ctx->G, mat, fast10);
    CK(cudaGetLastError());
    ctx->last_launches++;
    if ((rc = launch_init(ctx, mat, load, lmax, true))) return rc;
    return end_timing(ctx);
}

int mk2_init_counter_iv(mk2_ctx *ctx, const uint8_t key[10], uint64_t first_index, uint64_t N)
{
    MK2_ENTER(ctx);
    if (!key) return fail(ctx, MK2_E_ARG, "key is NULL");
    if (first_index % 32) return fail(ctx, MK2_E_ARG, "first_index must be a multiple of 32");
    if (first_index + N < first_index) return fail(ctx, MK2_E_ARG, "instance index range overflows 64 bits");
    int rc = init_common(ctx, N);
    if (rc) return rc;
    uint64_t hi = ((uint64_t)key[0] << 8) | key[1], lo = 0;
    for (int i = 2; i < 10; ++i) lo = (lo << 8) | key[i];
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    void *matp = nullptr;
    if ((rc = scratch.alloc(&matp, sizeof(uint32_t) * (size_t)160 * ctx->G))) return rc;
    uint32_t *mat = static_cast<uint32_t *>(matp);
    pack_counter_kernel<<<blocks_for(ctx->G), BLOCK, 0, ctx->stream>>>(hi, lo, first_index, ctx->G, mat);
    CK(cudaGetLastError());
    ctx->last_launches++;
    if ((rc = launch_init(ctx, mat, 160, 0, false))) return rc;
    return end_timing(ctx);
}

// IV bytes per lane of a derivation tag (seedgen.py:24-31, _SIZES / _ALGO_TAGS): 2 = grain (10 + 8),
// 3 = mickey (10 + 10).  Tag 1 (aes-ctr: 16-byte key + 12-byte nonce) is not on this library's path.
static int derive_iv_len(uint32_t tag) { return tag == 3u ? 10 : tag == 2u ? 8 : 0; }

static int derive_check(mk2_ctx *ctx, const uint8_t seed[32], uint32_t tag, uint64_t first_lane, uint64_t N)
{
    if (!seed) return fail(ctx, MK2_E_ARG, "seed is NULL");
    if (!derive_iv_len(tag)) return fail(ctx, MK2_E_ARG, "algo_tag must be 2 (grain) or 3 (mickey)");
    if (N == 0) return fail(ctx, MK2_E_ARG, "at least one lane is required");
    if (first_lane + N > (1ull << 32) || first_lane + N < first_lane)
        return fail(ctx, MK2_E_ARG, "lane index must fit the 32-bit field of the derivation block");
    bool nonzero = false;
    for (int i = 0; i < 32; ++i) nonzero |= seed[i] != 0;
    if (!nonzero) return fail(ctx, MK2_E_ARG, "all-zero master seed rejected");
    return MK2_OK;
}

// Derive key/IV rows for lanes [first_lane, first_lane + N) into device buffers (stream ordered); arguments
// already validated by derive_check.
static int derive_to_device(mk2_ctx *ctx, Scratch &scratch, const uint8_t seed[32], uint32_t tag, uint64_t first_lane,
                            uint64_t N, uint8_t *d_keys, uint8_t *d_ivs)
{
    int rc;
    void *d_seed = nullptr, *d_rk = nullptr;
    if ((rc = scratch.alloc(&d_seed, 32))) return rc;
    if ((rc = scratch.alloc(&d_rk, 44 * sizeof(uint32_t)))) return rc;
    CK(cudaMemcpyAsync(d_seed, seed, 32, cudaMemcpyHostToDevice, ctx->stream));
    seed_setup_kernel<<<1, 256, 0, ctx->stream>>>(static_cast<const uint8_t *>(d_seed), static_cast<uint32_t *>(d_rk));
    CK(cudaGetLastError());
    // grid-stride kernel: six 256-thread CTAs per SM (32 KB of table each) cover any N
    const unsigned derive_grid = (unsigned)std::min<uint64_t>((N + 255) / 256, 6ull * (uint64_t)ctx->sm_count);
    seed_derive_kernel<<<derive_grid, 256, 0, ctx->stream>>>(static_cast<const uint32_t *>(d_rk), tag, first_lane, N,
                                                             derive_iv_len(tag), d_keys, d_ivs);
    CK(cudaGetLastError());
    ctx->last_launches += 2;
    return MK2_OK;
}

int mk2_derive_material(mk2_ctx *ctx, const uint8_t seed[32], uint32_t algo_tag, uint64_t first_lane, uint64_t N,
                        uint8_t *keys, uint8_t *ivs)
{
    MK2_ENTER(ctx);
    if (!keys || !ivs) return fail(ctx, MK2_E_ARG, "keys / ivs is NULL");
    int rc = derive_check(ctx, seed, algo_tag, first_lane, N);
    if (rc) return rc;
    if ((rc = begin_timing(ctx))) return rc;
    const size_t iv_len = (size_t)derive_iv_len(algo_tag);
    const bool dk = is_device_ptr(keys), di = is_device_ptr(ivs);
    Scratch scratch(ctx);
    void *tk = nullptr, *ti = nullptr;
    if (!dk && (rc = scratch.alloc(&tk, N * 10))) return rc;
    if (!di && (rc = scratch.alloc(&ti, N * iv_len))) return rc;
    uint8_t *pk = dk ? keys : static_cast<uint8_t *>(tk), *pi = di ? ivs : static_cast<uint8_t *>(ti);
    if ((rc = derive_to_device(ctx, scratch, seed, algo_tag, first_lane, N, pk, pi))) return rc;
    if (!dk) CK(cudaMemcpyAsync(keys, tk, N * 10, cudaMemcpyDeviceToHost, ctx->stream));
    if (!di) CK(cudaMemcpyAsync(ivs, ti, N * iv_len, cudaMemcpyDeviceToHost, ctx->stream));
    if ((rc = end_timing(ctx))) return rc;
    if (!dk || !di) CK(cudaStreamSynchronize(ctx->stream));
    return MK2_OK;
}

int mk2_init_from_seed(mk2_ctx *ctx, const uint8_t seed[32], uint64_t first_lane, uint64_t N)
{
    MK2_ENTER(ctx);
    int rc = derive_check(ctx, seed, 3u /* mickey */, first_lane, N);
    if (rc) return rc;
    if ((rc = init_common(ctx, N))) return rc;
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    void *dk = nullptr, *di = nullptr;
    if ((rc = scratch.alloc(&dk, N * 10))) return rc;
    if ((rc = scratch.alloc(&di, N * 10))) return rc;
    if ((rc = derive_to_device(ctx, scratch, seed, 3u, first_lane, N, static_cast<uint8_t *>(dk), static_cast<uint8_t *>(di))))
        return rc;
    if ((rc = init_uniform_device(ctx, static_cast<const uint8_t *>(dk), static_cast<const uint8_t *>(di), 10, 80))) return rc;
    return end_timing(ctx);
}

static int generate_colmajor_impl(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words);
static int generate_rowmajor_impl(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes);

static int check_cipher(mk2_ctx *ctx, int cipher)
{
    int rc = check_ready(ctx);
    if (rc) return rc;
    if (ctx->cipher != cipher)
        return fail(ctx, MK2_E_STATE, cipher ? "context holds MICKEY state: call mk2_grain_init_from_material first"
                                             : "context holds Grain state: call a MICKEY mk2_init_* first");
    return MK2_OK;
}

int mk2_generate_colmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 0);
    return rc ? rc : generate_colmajor_impl(ctx, T, out, stride_words);
}

int mk2_generate_rowmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes)
{
    return mk2_generate_rowmajor_order(ctx, T, out, pitch_bytes, 0);
}

int mk2_generate_rowmajor_order(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes, int lsb_first)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 0);
    if (rc) return rc;
    ctx->row_lsb = lsb_first != 0;
    return generate_rowmajor_impl(ctx, T, out, pitch_bytes);
}

int mk2_grain_init_from_material(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint64_t N)
{
    MK2_ENTER(ctx);
    if (!keys || !ivs) return fail(ctx, MK2_E_ARG, "keys / ivs is NULL");
    int rc = init_common(ctx, N);
    if (rc) return rc;
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    const uint8_t *dk = nullptr, *di = nullptr;
    if ((rc = stage_input(ctx, scratch, keys, N * 10, &dk))) return rc;
    if ((rc = stage_input(ctx, scratch, ivs, N * 8, &di))) return rc;
    grain::init_kernel<<<blocks_for(ctx->G, ctx->block), ctx->block, 0, ctx->stream>>>(dk, di, N, ctx->G, ctx->d_state,
                                                                                        ctx->d_acc);
    CK(cudaGetLastError());
    ctx->last_launches++;
    ctx->clocks = 0;
    ctx->cipher = 1;
    ctx->ready = true;
    return end_timing(ctx);
}

int mk2_grain_generate_colmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 1);
    return rc ? rc : generate_colmajor_impl(ctx, T, out, stride_words);
}

int mk2_grain_generate_rowmajor(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes, int lsb_first)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 1);
    if (rc) return rc;
    ctx->row_lsb = lsb_first != 0;
    return generate_rowmajor_impl(ctx, T, out, pitch_bytes);
}

static int generate_colmajor_impl(mk2_ctx *ctx, uint64_t T, void *out, uint64_t stride_words)
{
    int rc = check_ready(ctx);
    if (rc) return rc;
    if (T == 0) {  // zero-length request leaves the state untouched (tests/test_mickey.py:167-171)
        ctx->last_ms = 0.f;
        ctx->last_launches = 0;
        return MK2_OK;
    }
    if (!out) return fail(ctx, MK2_E_ARG, "out is NULL");
    if (stride_words < ctx->G) return fail(ctx, MK2_E_ARG, "stride_words smaller than the group count");
    if (stride_words >= (1ull << 30)) return fail(ctx, MK2_E_ARG, "stride_words must be below 2^30");  // 32-bit byte strides in the kernels
    if (reinterpret_cast<uintptr_t>(out) % 4) return fail(ctx, MK2_E_ARG, "out must be 4-byte aligned");
    if ((rc = begin_timing(ctx))) return rc;
    const Mem mem = classify(out);
    if (mem == Mem::Device) {
        if ((rc = launch_col(ctx, T, static_cast<uint32_t *>(out), stride_words))) return rc;
    } else {
        // Host output: keystream tiles are produced in two device staging buffers and copied out on a second
        // stream while the next tile is generated.  Pinned destinations take the D2H copy directly; pageable
        // ones go through the pinned bounce buffers and the copy workers (HostTiles).
        const size_t row_bytes = ctx->G * sizeof(uint32_t);
        HostTiles tiles(ctx, mem, T * row_bytes);
        // copy lanes work on 8 MiB sub-chunks: give them tiles of at least 128 MiB to spread over
        // Pinned destinations: the D2H stream moves 128 MiB copies at 57.2 GB/s and 32 MiB ones at 56.85
        // (profiles/r02b_probe_e2e_link.txt), but the link idles while the FIRST tile is generated -- so the tiles
        // grow: 4 MiB, 8, ... up to 128 MiB (a 2 GiB call: 0.2 ms of fixed cost and 56.86 GB/s -> 0.07 ms and 57.1).
        const bool ramp = !tiles.pageable() && !ctx->stage_user;
        const size_t target = !ctx->stage_user ? std::max<size_t>(ctx->stage_target, size_t(128) << 20) : ctx->stage_target;
        const size_t want = std::max<size_t>(std::min<size_t>(target, T * row_bytes), row_bytes);
        if ((rc = ensure_stage(ctx, want))) return rc;
        if ((rc = tiles.prepare())) return rc;
        const uint64_t chunk_max = std::max<uint64_t>(1, ctx->stage_bytes / row_bytes);
        uint64_t chunk = ramp ? std::min<uint64_t>(chunk_max, std::max<uint64_t>(1, (size_t(4) << 20) / row_bytes)) : chunk_max;
        for (uint64_t t0 = 0, tc = 0; t0 < T; t0 += tc, chunk = std::min(chunk_max, 2 * chunk)) {
            tc = std::min(chunk, T - t0);
            const int b = tiles.next();
            if ((rc = tiles.acquire(b))) return rc;
            if ((rc = launch_col(ctx, tc, static_cast<uint32_t *>(ctx->d_stage[b]), ctx->G))) return rc;
            uint8_t *dst = static_cast<uint8_t *>(out) + t0 * stride_words * sizeof(uint32_t);
            if ((rc = tiles.copy_out(b, dst, stride_words * sizeof(uint32_t), row_bytes, row_bytes, tc))) return rc;
        }
        if ((rc = tiles.finish())) return rc;
    }
    ctx->clocks += T;
    return end_timing(ctx);
}

// Host row-major output of every chain of the context: 2-D tiles [block of chains] x [time chunk]
// through two device staging buffers (`b` = which one comes next; copies are left in flight:
// drain_copies).  A tile is a contiguous run of instance rows, each >= 512 B wide whenever T allows,
// so the D2H copy is one wide 2-D (or plain 1-D) transfer; a chain block is large enough to occupy
// every worker warp.  Chains stay strictly serial in time because the time loop is the inner one.
static int rowmajor_to_host(mk2_ctx *ctx, uint64_t T, uint8_t *out, uint64_t pitch_bytes, HostTiles &tiles)
{
    int rc;
    const uint64_t chains = (ctx->G + 31) / 32;
    // tile = [block_chains x 1024 rows] x [tc_max clocks] of about ROW_TILE_FACTOR x stage_target bytes, rows at
    // least 512 B wide when T allows (narrower 2-D copies collapse: 192 B rows 37 GB/s, 64 B rows 16 GB/s), and
    // between one and two chains per worker warp of a full launch
    // Pageable destinations: the copy lanes memcpy row pieces into the caller's pitched array, and 512-byte pieces
    // move at two thirds of the rate of 1 KiB ones (profiles/r02_probe_host_buffers.txt), so rows are 1 KiB wide
    // and the chain block is halved instead (half the worker warps still generate at twice the link rate).
    const bool pageable = tiles.pageable();
    // Pinned destinations: a chain block of ONE chain per SM sub-partition and 256 MiB tiles.  A lone warp runs at
    // twice the speed, so the call's first tile -- during which the link idles -- is ready in half the time, and half
    // the worker warps still generate at several times the link rate.  Measured on one box, 2 GiB per call
    // (tools/probe_e2e_row.py; before: two chains per sub-partition, 512 MiB tiles): 2^20 x 16384 bits 40.68 -> 39.61 ms,
    // 2^24 x 1024 40.66 -> 40.14, 2^22 x 4096 41.66 -> 40.30.  Making the later tiles of a call wider (2-D copies of
    // wider rows are more efficient in isolation) was measured too and loses 4-6% (MK2_ROW_WIDE = 2, 4, 8).
    static const uint64_t env_factor = std::getenv("MK2_ROW_TILE_FACTOR") ? std::strtoull(std::getenv("MK2_ROW_TILE_FACTOR"), nullptr, 0) : 0;
    static const uint64_t env_workers = std::getenv("MK2_ROW_WORKERS") ? std::strtoull(std::getenv("MK2_ROW_WORKERS"), nullptr, 0) : 0;
    static const uint64_t env_wide = std::getenv("MK2_ROW_WIDE") ? std::strtoull(std::getenv("MK2_ROW_WIDE"), nullptr, 0) : 0;
    const uint64_t tile_bytes = (env_factor ? env_factor : (pageable ? ROW_TILE_FACTOR : ROW_TILE_FACTOR / 2)) * ctx->stage_target;
    const uint64_t min_clocks = std::min<uint64_t>((T + 255) / 256 * 256, pageable ? 8192 : 4096);
    const uint64_t workers = (env_workers ? env_workers : 4ull) * (uint64_t)ctx->sm_count;
    const uint64_t want_chains = std::min<uint64_t>(2 * workers, std::max<uint64_t>(workers, tile_bytes / (min_clocks / 8) / 1024));
    const uint64_t block_chains = std::min<uint64_t>(chains, want_chains);
    const uint64_t block_rows = block_chains * 1024;
    uint64_t tc_max = std::max<uint64_t>(min_clocks, tile_bytes / block_rows / 32 * 256);
    tc_max = std::min<uint64_t>(tc_max, (T + 255) / 256 * 256);
    // later tiles of a pinned call: up to `wide` x the first tile's width, within 1 GiB per staging buffer
    const uint64_t wide = pageable || ctx->stage_user ? 1 : (env_wide ? env_wide : 1);
    uint64_t tc_wide = std::min<uint64_t>(wide * tc_max, (T + 255) / 256 * 256);
    while (tc_wide > tc_max && block_rows * (tc_wide / 8) > (size_t(1) << 30)) tc_wide -= 256;
    // a later block of a bulk call never needs larger staging buffers than the first one, but if it ever did the
    // copy lanes must be done with the old buffers before they are replaced (ensure_stage only knows the streams)
    if (block_rows * (tc_wide / 8) > ctx->stage_bytes && (rc = tiles.finish())) return rc;
    if ((rc = ensure_stage(ctx, block_rows * (tc_wide / 8)))) return rc;
    if ((rc = tiles.prepare())) return rc;
    bool first_tile = !ctx->copy_pending[0] && !ctx->copy_pending[1];  // nothing in flight: the link is idle
    for (uint64_t c0 = 0; c0 < chains; c0 += block_chains) {
        const uint64_t nch = std::min(block_chains, chains - c0);
        const uint64_t row0 = c0 * 1024;
        const uint64_t nrows = std::min<uint64_t>(nch * 1024, ctx->N - row0);
        for (uint64_t t0 = 0, tc = 0; t0 < T; t0 += tc) {
            tc = std::min(first_tile ? tc_max : tc_wide, T - t0);
            first_tile = false;
            const uint64_t sp = (tc / 8 + 15) / 16 * 16;  // staging pitch, 16-byte multiple
            const int b = tiles.next();
            if ((rc = tiles.acquire(b))) return rc;
            if ((rc = launch_row(ctx, tc, static_cast<uint8_t *>(ctx->d_stage[b]), sp, c0, nch))) return rc;
            if ((rc = tiles.copy_out(b, out + row0 * pitch_bytes + t0 / 8, pitch_bytes, sp, tc / 8, nrows))) return rc;
        }
    }
    return MK2_OK;
}

static int generate_rowmajor_impl(mk2_ctx *ctx, uint64_t T, void *out, uint64_t pitch_bytes)
{
    int rc = check_ready(ctx);
    if (rc) return rc;
    if (T % 8) return fail(ctx, MK2_E_ARG, "bit count must be a multiple of 8");
    if (T == 0) {
        ctx->last_ms = 0.f;
        ctx->last_launches = 0;
        return MK2_OK;
    }
    if (!out) return fail(ctx, MK2_E_ARG, "out is NULL");
    if (pitch_bytes < T / 8) return fail(ctx, MK2_E_ARG, "pitch_bytes smaller than T/8");
    if ((rc = begin_timing(ctx))) return rc;
    const uint64_t chains = (ctx->G + 31) / 32;
    const Mem mem = classify(out);
    if (mem == Mem::Device) {
        if ((rc = launch_row(ctx, T, static_cast<uint8_t *>(out), pitch_bytes, 0, chains))) return rc;
    } else {
        HostTiles tiles(ctx, mem, ctx->N * (T / 8));
        if ((rc = rowmajor_to_host(ctx, T, static_cast<uint8_t *>(out), pitch_bytes, tiles))) return rc;
        if ((rc = tiles.finish())) return rc;
    }
    ctx->clocks += T;
    return end_timing(ctx);
}

// ---------------------------------------------------------------------------
// One-shot bulk generation, row-major: init + keystream of N instances x T bits
// in one call (what kernels.mickey_sliced_words + words_lane_major_bytes do in the
// reference, kernels.py:189-200 / :615-621).  With host buffers the instances are
// processed in blocks and the three stages of consecutive blocks overlap:
//     H2D of block b+1's key/IV bytes | pack + init + keystream of block b | D2H of block b-1
// on three streams, so the upload and the init hide behind the (link-bound) download.
// The context keeps no resumable state afterwards.
// ---------------------------------------------------------------------------
static int bulk_rowmajor_impl(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride, uint32_t iv_bits,
                             uint64_t N, uint64_t T, void *out, uint64_t pitch_bytes, uint64_t *checksum);

int mk2_bulk_rowmajor(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride, uint32_t iv_bits,
                      uint64_t N, uint64_t T, void *out, uint64_t pitch_bytes, uint64_t *checksum)
{
    MK2_ENTER(ctx);
    const int rc = bulk_rowmajor_impl(ctx, keys, ivs, iv_stride, iv_bits, N, T, out, pitch_bytes, checksum);
    if (rc && rc != MK2_E_ARG) {
        // a failure part-way through the block pipeline: whatever state is on the device belongs to an arbitrary
        // block, so the context holds nothing resumable; quiesce the three streams before handing it back
        ctx->ready = false;
        ctx->N = ctx->G = 0;
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->copy);
        if (ctx->h2d) cudaStreamSynchronize(ctx->h2d);
        ctx->copy_pending[0] = ctx->copy_pending[1] = false;
        cudaGetLastError();
    }
    return rc;
}

static int bulk_rowmajor_impl(mk2_ctx *ctx, const uint8_t *keys, const uint8_t *ivs, uint32_t iv_stride, uint32_t iv_bits,
                             uint64_t N, uint64_t T, void *out, uint64_t pitch_bytes, uint64_t *checksum)
{
    if (!keys) return fail(ctx, MK2_E_ARG, "keys is NULL");
    if (N == 0) return fail(ctx, MK2_E_ARG, "at least one instance is required");
    if (iv_bits > 80) return fail(ctx, MK2_E_ARG, "IV must be at most 80 bits");
    if (iv_bits && (!ivs || iv_stride < (iv_bits + 7) / 8)) return fail(ctx, MK2_E_ARG, "ivs/iv_stride too small for iv_bits");
    if (T == 0 || T % 8) return fail(ctx, MK2_E_ARG, "bit count must be a positive multiple of 8");
    if (!out) return fail(ctx, MK2_E_ARG, "out is NULL");
    if (pitch_bytes < T / 8) return fail(ctx, MK2_E_ARG, "pitch_bytes smaller than T/8");
    int rc;
    const Mem out_mem = classify(out);
    const bool in_dev = is_device_ptr(keys), out_dev = out_mem == Mem::Device;
    if (iv_bits && is_device_ptr(ivs) != in_dev) return fail(ctx, MK2_E_ARG, "keys and ivs must both be host or both be device pointers");
    uint64_t block_inst = 2ull * 8ull * (uint64_t)ctx->sm_count * 1024ull;  // two chains per worker warp
    // Everything on the device already.  Init-dominated calls (T <= FUSED_MAX_CLOCKS; BASELINE config 5) run as ONE
    // kernel for the whole batch (mk2_fused.cuh): input words and state never leave the SM.  It wants whole IV bytes,
    // 10-byte IV records and 16-byte aligned arrays (what the 128-bit record loads need).  Keystream-dominated calls
    // gain nothing from fusing the 260 init clocks and lose the chunk scheduler's short tail (measured, 2^24 x 65536:
    // fused 590.7 ms, blocks 583.9, one block 579.6): they run as ONE block -- pack + init + persistent keystream
    // kernel over all N, the state of all N on the device (48 B per instance with the packed input words) -- as long
    // as that fits a modest budget; beyond it, and with host buffers, the block pipeline below.
    constexpr uint64_t FUSED_MAX_CLOCKS = 1024, ONE_BLOCK_STATE_BUDGET = 16ull << 30;
    const bool small = ctx->small_batch && (N + 31) / 32 <= COOP_MAX_GROUPS;  // the warp-per-group kernels are quicker there
    if (in_dev && out_dev && N * 48 <= ONE_BLOCK_STATE_BUDGET) block_inst = std::max(block_inst, N);
    if (in_dev && out_dev && (ctx->bulk_fused == 2 || (ctx->bulk_fused == 1 && T <= FUSED_MAX_CLOCKS)) && !small &&
        ctx->row_staging != 1 && iv_bits % 8 == 0 &&
        reinterpret_cast<uintptr_t>(keys) % 16 == 0 &&
        (iv_bits == 0 || (iv_stride == 10 && reinterpret_cast<uintptr_t>(ivs) % 16 == 0))) {
        const bool resume = N <= 2ull * 8ull * (uint64_t)ctx->sm_count * 1024ull;  // small enough to keep its state
        const uint64_t G = (N + 31) / 32;
        ctx->ready = false;
        if (resume) {
            if ((rc = init_common(ctx, N))) return rc;
        } else {
            ctx->N = ctx->G = 0;
        }
        ctx->last_launches = 0;
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        CK(cudaMemsetAsync(ctx->d_sum, 0, sizeof(unsigned long long), ctx->stream));
        CK(cudaMemsetAsync(ctx->d_queue, 0, sizeof(SchedQueue), ctx->stream));
        const uint64_t jobs = ((G + 31) / 32 + BLOCK / 32 - 1) / (BLOCK / 32);
        const uint64_t sms = ctx->max_grid ? std::min<uint64_t>(ctx->max_grid, (uint64_t)ctx->sm_count) : (uint64_t)ctx->sm_count;
        // whole rounds as eight-chain jobs; a last round that would occupy at most half of the SMs as four-chain jobs
        const uint64_t rem = jobs % sms;
        const unsigned long long full_jobs = rem && 2 * rem <= sms ? jobs - rem : jobs;
        const unsigned grid = (unsigned)std::min<uint64_t>(sms, full_jobs + 2 * (jobs - full_jobs));
        uint32_t *st = resume ? ctx->d_state : nullptr;
        unsigned long long *ac = resume ? ctx->d_acc : nullptr;
        const bool aligned = reinterpret_cast<uintptr_t>(out) % 16 == 0 && pitch_bytes % 16 == 0;
        if (aligned)
            fused::bulk_rowmajor_kernel<true><<<grid, BLOCK, 0, ctx->stream>>>(keys, ivs, (int)iv_bits / 8, N, G, T,
                static_cast<uint8_t *>(out), pitch_bytes, &ctx->d_queue->head, full_jobs, ctx->d_sum, ctx->g_offset, st, ac);
        else
            fused::bulk_rowmajor_kernel<false><<<grid, BLOCK, 0, ctx->stream>>>(keys, ivs, (int)iv_bits / 8, N, G, T,
                static_cast<uint8_t *>(out), pitch_bytes, &ctx->d_queue->head, full_jobs, ctx->d_sum, ctx->g_offset, st, ac);
        CK(cudaGetLastError());
        unsigned long long v = 0;
        CK(cudaMemcpyAsync(&v, ctx->d_sum, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
        ctx->timing_open = false;
        ctx->last_launches = 1;
        ctx->last_plan_block = BLOCK;
        ctx->last_plan_chunk = (uint32_t)std::min<uint64_t>(T, 0x7FFFFF00ull);
        if (checksum) *checksum = v;
        if (resume) {
            ctx->clocks = T;
            ctx->cipher = 0;
            ctx->ready = true;
        }
        return MK2_OK;
    }
    if (!ctx->h2d) {
        CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&ctx->h2d_done[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->mat_used[i], cudaEventDisableTiming));
        }
    }
    const size_t in_row = 10 + (iv_bits ? (size_t)iv_stride : 0);
    const size_t in_bytes = (size_t)std::min<uint64_t>(N, block_inst) * in_row;
    if (!in_dev && in_bytes > ctx->bulk_in_bytes) {
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaStreamSynchronize(ctx->h2d));
        for (int i = 0; i < 2; ++i) {
            if (ctx->d_bulk_in[i]) cudaFree(ctx->d_bulk_in[i]);
            ctx->d_bulk_in[i] = nullptr;
        }
        ctx->bulk_in_bytes = 0;
        for (int i = 0; i < 2; ++i) CK(cudaMalloc(&ctx->d_bulk_in[i], in_bytes));
        ctx->bulk_in_bytes = in_bytes;
    }
    if ((rc = init_common(ctx, std::min<uint64_t>(N, block_inst)))) return rc;
    ctx->last_launches = 0;
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_sum, 0, sizeof(unsigned long long), ctx->stream));
    CK(cudaEventRecord(ctx->mat_used[0], ctx->stream));  // everything queued before this call is ahead of the uploads
    CK(cudaStreamWaitEvent(ctx->h2d, ctx->mat_used[0], 0));
    HostTiles tiles(ctx, out_mem, N * (T / 8));
    ctx->row_lsb = false;
    int launches = 0;
    uint64_t nblk = 0;
    // Host buffers: the download cannot start before the first block's keys have been uploaded and its keystream
    // generated, so for short keystreams the blocks GROW -- an eighth of the full size first, doubling (whole chains, so
    // that block starts stay multiples of 64 instances): the link idles for 0.6 ms instead of 3 ms at the start of a
    // call (2 GiB calls, tools/probe_e2e_row.py: 2^24 x 1024 bits 41.3 -> 40.4 ms, 2^22 x 4096 41.1 -> 40.4).  Long
    // keystreams are the opposite case -- a small first block is a long serial job on a mostly idle GPU (2^20 x 16384:
    // 39.9 -> 43.2 ms) -- and keep full blocks.
    static const uint64_t env_ramp = std::getenv("MK2_BULK_RAMP") ? std::strtoull(std::getenv("MK2_BULK_RAMP"), nullptr, 0) : 0;
    const uint64_t ramp = in_dev && out_dev ? 1 : (env_ramp ? env_ramp : (T <= 4096 ? 8 : 1));
    uint64_t blk = std::max<uint64_t>(1024, block_inst / ramp / 1024 * 1024);
    for (uint64_t row0 = 0, n = 0; row0 < N; row0 += n, ++nblk, blk = std::min(block_inst, 2 * blk)) {
        n = std::min(blk, N - row0);
        ctx->last_launches = 0;
        const int i = (int)(nblk & 1);
        const uint8_t *dk, *di = nullptr;
        if (in_dev) {
            dk = keys + row0 * 10;
            if (iv_bits) di = ivs + row0 * (uint64_t)iv_stride;
        } else {
            uint8_t *buf = static_cast<uint8_t *>(ctx->d_bulk_in[i]);
            if (nblk >= 2) CK(cudaStreamWaitEvent(ctx->h2d, ctx->mat_used[i], 0));  // block b-2 has been packed
            CK(cudaMemcpyAsync(buf, keys + row0 * 10, n * 10, cudaMemcpyHostToDevice, ctx->h2d));
            if (iv_bits)
                CK(cudaMemcpyAsync(buf + n * 10, ivs + row0 * (uint64_t)iv_stride, n * (size_t)iv_stride,
                                   cudaMemcpyHostToDevice, ctx->h2d));
            CK(cudaEventRecord(ctx->h2d_done[i], ctx->h2d));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->h2d_done[i], 0));
            dk = buf;
            if (iv_bits) di = buf + n * 10;
        }
        ctx->N = n;
        ctx->G = (n + 31) / 32;
        if ((rc = init_uniform_device(ctx, dk, di, iv_stride, iv_bits))) return rc;
        if (!in_dev) CK(cudaEventRecord(ctx->mat_used[i], ctx->stream));
        uint8_t *dst = static_cast<uint8_t *>(out) + row0 * pitch_bytes;
        if (out_dev) {
            if ((rc = launch_row(ctx, T, dst, pitch_bytes, 0, (ctx->G + 31) / 32))) return rc;
        } else {
            if ((rc = rowmajor_to_host(ctx, T, dst, pitch_bytes, tiles))) return rc;
        }
        // checksum of the whole call: block sums accumulate in d_sum (block starts are multiples of 64 instances,
        // so the parity term of checksum_kernel is that of the global group index)
        const unsigned nb = std::min<unsigned>(blocks_for(ctx->G), 4u * (unsigned)ctx->sm_count);
        checksum_kernel<<<nb, BLOCK, 0, ctx->stream>>>(ctx->d_acc, ctx->G, ctx->g_offset + row0 / 32, ctx->d_sum);
        CK(cudaGetLastError());
        launches += ctx->last_launches + 1;
    }
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, ctx->d_sum, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (!out_dev && (rc = tiles.finish())) return rc;
    CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
    ctx->timing_open = false;
    ctx->last_launches = launches;
    if (checksum) *checksum = v;
    if (nblk > 1) {  // only the last block's state is on the device: nothing to resume from
        ctx->ready = false;
        ctx->N = ctx->G = 0;
    } else {
        ctx->clocks = T;
    }
    return MK2_OK;
}

int mk2_clock(mk2_ctx *ctx, int mixing, const uint32_t *input_words, uint64_t n)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 0);
    if (rc) return rc;
    if (n == 0) return MK2_OK;
    if ((rc = begin_timing(ctx))) return rc;
    Scratch scratch(ctx);
    const uint8_t *din = nullptr;
    if ((rc = stage_input(ctx, scratch, input_words, input_words ? sizeof(uint32_t) * n * ctx->G : 0, &din))) return rc;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(din);
    if (mixing)
        clock_kernel<true><<<blocks_for(ctx->G, ctx->block), ctx->block, 0, ctx->stream>>>(ctx->d_state, w, n, ctx->G);
    else
        clock_kernel<false><<<blocks_for(ctx->G, ctx->block), ctx->block, 0, ctx->stream>>>(ctx->d_state, w, n, ctx->G);
    CK(cudaGetLastError());
    ctx->last_launches++;
    return end_timing(ctx);
}

int mk2_state_export(mk2_ctx *ctx, uint32_t *rs)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 0);
    if (rc) return rc;
    if (!rs) return fail(ctx, MK2_E_ARG, "rs is NULL");
    const size_t bytes = sizeof(uint32_t) * 2 * NBITS * ctx->G;
    CK(cudaMemcpyAsync(rs, ctx->d_state, bytes, is_device_ptr(rs) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return MK2_OK;
}

int mk2_state_import(mk2_ctx *ctx, const uint32_t *rs, uint64_t N)
{
    MK2_ENTER(ctx);
    if (!rs) return fail(ctx, MK2_E_ARG, "rs is NULL");
    int rc = init_common(ctx, N);
    if (rc) return rc;
    const size_t bytes = sizeof(uint32_t) * 2 * NBITS * ctx->G;
    CK(cudaMemcpyAsync(ctx->d_state, rs, bytes, is_device_ptr(rs) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemsetAsync(ctx->d_acc, 0, sizeof(unsigned long long) * ctx->G, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->clocks = 0;
    ctx->cipher = 0;
    ctx->ready = true;
    return MK2_OK;
}

int mk2_grain_state_export(mk2_ctx *ctx, uint32_t *bs)
{
    MK2_ENTER(ctx);
    int rc = check_cipher(ctx, 1);
    if (rc) return rc;
    if (!bs) return fail(ctx, MK2_E_ARG, "bs is NULL");
    const size_t bytes = sizeof(uint32_t) * 2 * grain::GB * ctx->G;
    CK(cudaMemcpyAsync(bs, ctx->d_state, bytes, is_device_ptr(bs) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return MK2_OK;
}

int mk2_checksum(mk2_ctx *ctx, uint64_t *sum)
{
    MK2_ENTER(ctx);
    int rc = check_ready(ctx);
    if (rc) return rc;
    if (!sum) return fail(ctx, MK2_E_ARG, "sum is NULL");
    CK(cudaMemsetAsync(ctx->d_sum, 0, sizeof(unsigned long long), ctx->stream));
    const unsigned nb = std::min<unsigned>(blocks_for(ctx->G), 4u * (unsigned)ctx->sm_count);
    checksum_kernel<<<nb, BLOCK, 0, ctx->stream>>>(ctx->d_acc, ctx->G, ctx->g_offset, ctx->d_sum);
    CK(cudaGetLastError());
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, ctx->d_sum, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *sum = v;
    return MK2_OK;
}

int mk2_lop3_peak(mk2_ctx *ctx, double *lane_ops_per_s, float *ms_out)
{
    if (!lane_ops_per_s) return MK2_E_ARG;
    MK2_ENTER(ctx);
    uint32_t *sink = nullptr;
    const unsigned nb = 8u * (unsigned)ctx->sm_count;
    CK(cudaMalloc(&sink, sizeof(uint32_t) * nb * BLOCK));
    const int iters = 2048;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {  // first repetition is the warm-up
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        lop3_peak_kernel<<<nb, BLOCK, 0, ctx->stream>>>(sink, 12345u + rep, iters);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        if (rep > 0) best = std::min(best, ms);
    }
    CK(cudaFree(sink));
    const double ops = (double)nb * BLOCK * 32.0 / 32.0 * (double)iters * 16.0 * PEAK_UNROLL;
    *lane_ops_per_s = ops / (best * 1e-3);
    if (ms_out) *ms_out = best;
    return MK2_OK;
}

}  // extern "C"
