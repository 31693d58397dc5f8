// mk2_host_lanes.h -- host side of PAGEABLE output buffers (plain C++ + CUDA runtime; no device code).
//
// Included by mk2_api.cu only.  See HostTiles there for how tiles are produced and queued.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace mk2 {
namespace host {

// ---------------------------------------------------------------------------
// Host side of PAGEABLE output buffers.  A D2H copy into pageable memory is staged by the driver
// through its own small pinned buffers on the calling thread (measured on this box: 10-13 GB/s against
// 56 GB/s into pinned memory).  Here a few independent COPY LANES do it in parallel: a lane is a host
// thread with its own CUDA stream, two events and two page-locked slots.  A device staging tile is cut
// into sub-chunks of LANE_BYTES; every lane repeatedly claims the next sub-chunk, starts its device ->
// slot copy on its stream, and meanwhile memcpy's the sub-chunk that landed in its other slot into the
// caller's array (a fresh numpy array takes its first-touch page faults there, spread over the lanes).
// The link stays busy with the lanes' copies; tiles are queued, so the lanes run on into the next tile
// while the calling thread is launching kernels.
// ---------------------------------------------------------------------------
// Sub-chunk size and store flavour, measured on the 16-core B200 host with 2 GiB outputs
// (profiles/r02_probe_copy_lanes.txt; pinned destination: 56.5 GB/s column-major, 51 GB/s row-major):
//   contiguous destination (column-major tiles): 8 MiB sub-chunks moved with non-temporal stores 51 GB/s from
//       8 lanes on; 2 MiB sub-chunks 46 GB/s with plain memcpy, 36 GB/s with non-temporal stores;
//   pitched destination (row-major tiles, 1 KiB row pieces): 2 MiB sub-chunks 46 GB/s at 16 lanes (either
//       store flavour), 8 MiB sub-chunks 36 GB/s.
constexpr size_t LANE_BYTES_WIDE = size_t(8) << 20;
constexpr size_t LANE_BYTES_PITCHED = size_t(2) << 20;

#if defined(__x86_64__) && defined(__GNUC__)
#include <immintrin.h>
// memcpy with non-temporal stores: the destination (the caller's result array) is written once and not read
// back by these threads, so the lines need not be fetched for ownership nor kept in cache.
__attribute__((target("avx2"))) inline void stream_copy(uint8_t *dst, const uint8_t *src, size_t n)
{
    const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
    if (n < 4096 || head > n) {
        std::memcpy(dst, src, n);
        return;
    }
    std::memcpy(dst, src, head);
    dst += head; src += head; n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 96), d);
    }
    _mm_sfence();
    std::memcpy(dst + i, src + i, n - i);
}
inline bool cpu_has_avx2() { return __builtin_cpu_supports("avx2"); }
#else
inline void stream_copy(uint8_t *dst, const uint8_t *src, size_t n) { std::memcpy(dst, src, n); }
inline bool cpu_has_avx2() { return false; }
#endif

class HostCopyLanes {
public:
    struct Tile {
        const uint8_t *src = nullptr;  // device staging buffer
        uint8_t *dst = nullptr;        // caller's (pageable) array
        size_t spitch = 0, dpitch = 0, width = 0, rows = 0;
        cudaEvent_t ready = nullptr;   // recorded after the kernel that fills src
        size_t rows_per_sub = 1, cols_per_sub = 1, col_subs = 1, nsub = 0;
        std::atomic<size_t> next{0};
        std::atomic<size_t> remaining{0};
        size_t sub_bytes = 0;          // page-locked slot space one sub-chunk needs
        bool nt = false;               // move it with non-temporal stores
        std::atomic<int> error{0};     // first cudaError_t seen by a lane
        unsigned long long id = 0;     // never reused (a freed tile's address can be)
        int lanes_wanted = 1 << 30;    // lanes with a higher index leave this tile to the others
    };
    using TilePtr = std::shared_ptr<Tile>;

    HostCopyLanes(int device, int nlanes) : device_(device)
    {
        // experiment knobs (tools/probe_lanes.py): sub-chunk size and store flavour of the lanes
        if (const char *v = std::getenv("MK2_LANE_BYTES")) lane_bytes_ = std::max<size_t>(65536, std::strtoull(v, nullptr, 0));
        avx2_ = cpu_has_avx2();
        if (const char *v = std::getenv("MK2_LANE_NT")) nt_override_ = std::atoi(v) != 0 ? 1 : 0;
        lanes_override_ = std::getenv("MK2_LANE_ALL") != nullptr;
        if (const char *v = std::getenv("MK2_LANE_WIDE")) wide_lanes_ = std::max(1, std::atoi(v));
        for (int i = 0; i < nlanes; ++i) lanes_.emplace_back([this, i] { run(i); });
    }
    ~HostCopyLanes()
    {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : lanes_) t.join();
    }
    // rows x width bytes at src (pitch spitch, device) -> dst (pitch dpitch, host), once `ready` has happened
    TilePtr post(const void *src, size_t spitch, void *dst, size_t dpitch, size_t width, size_t rows, cudaEvent_t ready)
    {
        auto t = std::make_shared<Tile>();
        t->src = static_cast<const uint8_t *>(src);
        t->dst = static_cast<uint8_t *>(dst);
        t->spitch = spitch; t->dpitch = dpitch; t->width = width; t->rows = rows; t->ready = ready;
        // sub-chunks: whole rows (narrow rows) or pieces of one row (rows wider than a slot)
        const bool wide = dpitch == width;  // the tile is one contiguous run in the caller's array
        const size_t lane_bytes = lane_bytes_ ? lane_bytes_ : (wide ? LANE_BYTES_WIDE : LANE_BYTES_PITCHED);
        t->nt = avx2_ && (nt_override_ >= 0 ? nt_override_ != 0 : wide);
        // contiguous tiles are at their best with 6-8 lanes (8 MiB non-temporal sub-chunks saturate the memory
        // system; more lanes only compete), pitched row tiles keep gaining up to 16 (profiles/r02_probe_copy_lanes.txt)
        if (wide && !lanes_override_) t->lanes_wanted = wide_lanes_;
        t->rows_per_sub = std::max<size_t>(1, lane_bytes / width);
        t->cols_per_sub = std::min(width, lane_bytes);
        t->sub_bytes = t->rows_per_sub * t->cols_per_sub;
        t->col_subs = (width + t->cols_per_sub - 1) / t->cols_per_sub;
        t->nsub = ((rows + t->rows_per_sub - 1) / t->rows_per_sub) * t->col_subs;
        t->remaining.store(t->nsub);
        if (t->nsub == 0) return t;
        {
            std::lock_guard<std::mutex> lk(m_);
            t->id = ++last_id_;
            queue_.push_back(t);
        }
        cv_.notify_all();
        return t;
    }
    // blocks until every sub-chunk of the tile is in the caller's array; returns the first CUDA error (0 = none)
    int wait(const TilePtr &t)
    {
        if (!t) return 0;
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return t->remaining.load() == 0; });
        return t->error.load();
    }

private:
    struct Sub {
        TilePtr t;
        size_t r0 = 0, nr = 0, c0 = 0, nc = 0;
        int slot = 0;
        cudaError_t e = cudaSuccess;
    };
    // Next unclaimed sub-chunk of the oldest unfinished tile; with `block` it sleeps until there is one (or the
    // lanes are shut down), without it returns false at once when the queue is empty.
    bool claim(bool block, Sub &s, int lane)
    {
        for (;;) {
            TilePtr t;
            {
                std::unique_lock<std::mutex> lk(m_);
                for (;;) {
                    while (!queue_.empty() && queue_.front()->next.load() >= queue_.front()->nsub) queue_.pop_front();
                    // the oldest unfinished tile this lane may work on
                    t.reset();
                    for (const auto &q : queue_)
                        if (lane < q->lanes_wanted && q->next.load() < q->nsub) {
                            t = q;
                            break;
                        }
                    if (stop_ || t || !block) break;
                    cv_.wait(lk);
                }
                if (stop_ || !t) return false;
            }
            const size_t i = t->next.fetch_add(1);
            if (i >= t->nsub) continue;
            s.r0 = (i / t->col_subs) * t->rows_per_sub;
            s.nr = std::min(t->rows_per_sub, t->rows - s.r0);
            s.c0 = (i % t->col_subs) * t->cols_per_sub;
            s.nc = std::min(t->cols_per_sub, t->width - s.c0);
            s.t = std::move(t);
            return true;
        }
    }
    void run(int lane)
    {
        // a lane = this thread, one stream, two page-locked slots: the D2H copy of its next sub-chunk is in flight
        // while it moves the current one into the caller's array
        cudaStream_t stream = nullptr;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        void *slots = nullptr;   // two page-locked slots of slot_bytes each, grown to the largest sub-chunk seen
        size_t slot_bytes = 0;
        const bool ok = cudaSetDevice(device_) == cudaSuccess &&
                        cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) == cudaSuccess &&
                        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) == cudaSuccess &&
                        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) == cudaSuccess;
        unsigned long long synced = 0;  // id of the tile whose `ready` event this lane's stream already waits on
        Sub cur, nxt;
        bool have_cur = false;
        auto land = [&] {  // wait for the current sub-chunk's D2H copy and move it into the caller's array
            Tile &t = *cur.t;
            cudaError_t e = cur.e;
            if (e == cudaSuccess) e = cudaEventSynchronize(ev[cur.slot]);
            if (e == cudaSuccess) {
                uint8_t *d = t.dst + cur.r0 * t.dpitch + cur.c0;
                const uint8_t *h = static_cast<const uint8_t *>(slots) + (size_t)cur.slot * slot_bytes;
                if (!t.nt) {
                    if (t.dpitch == cur.nc) std::memcpy(d, h, cur.nc * cur.nr);
                    else
                        for (size_t r = 0; r < cur.nr; ++r) std::memcpy(d + r * t.dpitch, h + r * cur.nc, cur.nc);
                } else if (t.dpitch == cur.nc) {
                    stream_copy(d, h, cur.nc * cur.nr);
                } else {
                    for (size_t r = 0; r < cur.nr; ++r) stream_copy(d + r * t.dpitch, h + r * cur.nc, cur.nc);
                }
            } else {
                int zero = 0;
                t.error.compare_exchange_strong(zero, (int)e);
                cudaGetLastError();
            }
            if (t.remaining.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> lk(m_);
                done_.notify_all();
            }
            cur.t.reset();
            have_cur = false;
        };
        for (;;) {
            const bool have_nxt = claim(!have_cur, nxt, lane);
            if (!have_nxt && !have_cur) break;  // shut down (a blocking claim only fails on stop)
            if (have_nxt) {
                Tile &t = *nxt.t;
                cudaError_t e = ok ? cudaSuccess : cudaErrorInitializationError;
                if (t.sub_bytes > slot_bytes) {  // larger slots needed: nothing may be in flight in the old ones
                    if (have_cur) land();
                    if (slots) cudaFreeHost(slots);
                    slots = nullptr;
                    slot_bytes = 0;
                    if (e == cudaSuccess) e = cudaHostAlloc(&slots, 2 * t.sub_bytes, cudaHostAllocDefault);
                    if (e == cudaSuccess) slot_bytes = t.sub_bytes;
                }
                // start its D2H copy into the slot `cur` does not use
                nxt.slot = have_cur ? cur.slot ^ 1 : 0;
                uint8_t *h = static_cast<uint8_t *>(slots) + (size_t)nxt.slot * slot_bytes;
                if (e == cudaSuccess && synced != t.id) {
                    e = cudaStreamWaitEvent(stream, t.ready, 0);
                    synced = t.id;
                }
                if (e == cudaSuccess) {
                    if (t.spitch == nxt.nc)
                        e = cudaMemcpyAsync(h, t.src + nxt.r0 * t.spitch, nxt.nc * nxt.nr, cudaMemcpyDeviceToHost, stream);
                    else
                        e = cudaMemcpy2DAsync(h, nxt.nc, t.src + nxt.r0 * t.spitch + nxt.c0, t.spitch, nxt.nc, nxt.nr,
                                              cudaMemcpyDeviceToHost, stream);
                }
                if (e == cudaSuccess) e = cudaEventRecord(ev[nxt.slot], stream);
                nxt.e = e;
            }
            if (have_cur) land();
            if (have_nxt) {
                cur = std::move(nxt);
                have_cur = true;
                nxt = Sub{};
            }
        }
        if (slots) cudaFreeHost(slots);
        for (auto &e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
    int device_;
    size_t lane_bytes_ = 0;   // 0 = by tile shape
    bool avx2_ = false;
    int nt_override_ = -1;
    bool lanes_override_ = false;
    int wide_lanes_ = 8;          // lanes a contiguous tile uses (MK2_LANE_WIDE)
    std::vector<std::thread> lanes_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::deque<TilePtr> queue_;
    unsigned long long last_id_ = 0;
    bool stop_ = false;
};

}  // namespace host
}  // namespace mk2
