// sg_xfer.cu -- the API boundary's host <-> device copies of index arrays.
//
// The reference's arrays are int64 (SuccessorList.succ, EdgeGraph.edges,
// the returned ranks and labels, core.py:77-110); the device works on
// 32-bit ids.  Moving int64 over PCIe and narrowing on the device moves
// twice the bytes the kernels need.  These copies narrow / widen on the host
// instead, pipelined against the DMA:
//
//   h2d:  host threads narrow chunk k+1 (int64 -> u32, range-checked against
//         `bound`) into a pinned staging slot while chunk k is copied;
//   d2h:  chunk k is copied into a pinned slot while host threads widen
//         chunk k-1 (u32 -> int64) into the caller's array.
//
// Measured on the B200 box (tools/probe_hostconv.py, 2^28 elements, 16 host
// threads): int64 H2D 38.6 ms vs u32 H2D 19.3 ms + narrowing 23-30 ms
// overlapped; int64 D2H 37.8 ms vs u32 D2H 18.8 ms + widening ~30 ms.
// Data conversion only -- no ranking or labelling is computed here.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <emmintrin.h>  // SSE2 (x86-64 baseline): 16-B non-temporal stores
#include <sched.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "sg_internal.cuh"

namespace sg {
namespace {

// host CPUs this process may actually run on: the affinity mask (what
// hardware_concurrency ignores: it counts the machine's online CPUs), capped
// by a cgroup CPU quota (v2 cpu.max, v1 cfs_quota_us / cfs_period_us).  More
// spinning workers than usable CPUs would time-slice against each other.
int usable_cpus() {
    int n = 0;
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
    if (n <= 0) n = (int)std::max(1u, std::thread::hardware_concurrency());
    long long quota = -1, period = 0;
    if (FILE* f = fopen("/sys/fs/cgroup/cpu.max", "r")) {
        char q[32] = {0};
        if (fscanf(f, "%31s %lld", q, &period) == 2 && strcmp(q, "max") != 0) quota = atoll(q);
        fclose(f);
    } else if (FILE* fq = fopen("/sys/fs/cgroup/cpu/cpu.cfs_quota_us", "r")) {
        if (fscanf(fq, "%lld", &quota) != 1) quota = -1;
        fclose(fq);
        if (FILE* fp = fopen("/sys/fs/cgroup/cpu/cpu.cfs_period_us", "r")) {
            if (fscanf(fp, "%lld", &period) != 1) period = 0;
            fclose(fp);
        }
    }
    if (quota > 0 && period > 0) n = std::min<long long>(n, std::max(1LL, quota / period));
    return n;
}

// fixed pool of host threads running one parallel-for at a time.  A pipelined
// copy calls run() once per chunk (every ~0.3-0.5 ms), so workers spin on the
// generation counter for a while before sleeping on the condition variable:
// a condition-variable wake-up per chunk and per worker cost ~1-3 ms per
// 2^28-id transfer.
class Pool {
  public:
    Pool() {
        nthreads_ = std::max(1, std::min(usable_cpus(), 32));
        if (const char* e = getenv("SG_XFER_THREADS")) {  // experiment switch (read once, at first use)
            const int v = atoi(e);
            if (v >= 1 && v <= 256) nthreads_ = v;
        }
        if (const char* e = getenv("SG_XFER_SPIN")) kSpin = std::max(0, atoi(e));
        for (int i = 1; i < nthreads_; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_.store(true);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    int size() const { return nthreads_; }
    // fn(part, parts) on every thread (the caller is part 0); returns when all are done
    void run(const std::function<void(int, int)>& fn) {
        std::unique_lock<std::mutex> call(call_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            pending_.store(nthreads_ - 1, std::memory_order_relaxed);
            gen_.fetch_add(1, std::memory_order_release);  // spinning workers see fn_ with it
        }
        cv_.notify_all();
        fn(0, nthreads_);
        for (int i = 0; pending_.load(std::memory_order_acquire) != 0; ++i) {
            if (i < kSpin) {
                _mm_pause();
                continue;
            }
            std::unique_lock<std::mutex> lk(mu_);
            done_cv_.wait(lk, [this] { return pending_.load(std::memory_order_acquire) == 0; });
            break;
        }
        fn_ = nullptr;
    }

  private:
    int kSpin = 1 << 16;  // pause loops before sleeping (~ms); SG_XFER_SPIN=0: sleep at once
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            uint64_t g = gen_.load(std::memory_order_acquire);
            for (int i = 0; g == seen && i < kSpin; ++i) {
                _mm_pause();
                g = gen_.load(std::memory_order_acquire);
            }
            if (g == seen) {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                g = gen_.load(std::memory_order_acquire);
            }
            seen = g;
            if (stop_.load()) return;
            (*fn_)(id, nthreads_);
            if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> lk(mu_);  // a waiter may be asleep on done_cv_
                done_cv_.notify_one();
            }
        }
    }
    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)>* fn_ = nullptr;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> pending_{0};
    std::atomic<bool> stop_{false};
};

Pool& pool() {
    static Pool p;
    return p;
}

constexpr int kSlots = 4;
// ids per pipelined chunk: the first chunk's conversion and the last chunk's
// copy are not overlapped, so smaller chunks shorten the ends of the pipe
// (SG_XFER_CHUNK_MI: Mi ids per chunk, 1..16, read once at first use)
size_t chunk_ids() {
    static const size_t v = [] {
        size_t x = size_t(4) << 20;
        if (const char* e = getenv("SG_XFER_CHUNK_MI")) {
            const int m = atoi(e);
            if (m >= 1 && m <= 16) x = size_t(m) << 20;
        }
        return x;
    }();
    return v;
}

// pinned staging ring of one device (u32 slots big enough for either direction)
struct Ring {
    uint32_t* slot[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    bool ok = false;
};

std::mutex g_ring_mu;
Ring g_rings[64];

Ring* ring_for_current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    Ring& r = g_rings[dev];
    if (r.ok) return &r;
    for (int k = 0; k < kSlots; ++k) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&r.slot[k]), chunk_ids() * sizeof(uint32_t), cudaHostAllocPortable) !=
                cudaSuccess ||
            cudaEventCreateWithFlags(&r.ev[k], cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
    }
    r.ok = true;
    return &r;
}

// [lo, hi) of part p out of parts, in whole cache lines of u32
inline void split(size_t n, int p, int parts, size_t& lo, size_t& hi) {
    const size_t per = ((n + parts - 1) / parts + 15) & ~size_t(15);
    lo = std::min(n, per * (size_t)p);
    hi = std::min(n, lo + per);
}


// int64 -> u32 over [0, len): returns nonzero if any value lies outside
// [0, bound) (bound <= 2^31).  dst (pinned staging) gets 16-B non-temporal
// stores: it is DMA'd next, so there is no point in reading it for
// ownership or keeping it in the host caches.
inline uint64_t narrow_range(const int64_t* src, uint32_t* dst, size_t len, uint64_t bound) {
    uint64_t acc = 0;
    size_t i = 0;
    for (; i < len && ((uintptr_t)(dst + i) & 15); ++i) {
        const uint64_t v = (uint64_t)src[i];
        acc |= (uint64_t)(v >= bound);
        dst[i] = (uint32_t)v;
    }
    const __m128i bm1 = _mm_set1_epi32((int)(bound - 1));  // bound - 1 < 2^31: a signed compare works
    __m128i hi_any = _mm_setzero_si128();  // any nonzero high word: out of range
    __m128i sgn = _mm_setzero_si128();     // sign bits: low word >= 2^31, or low word > bound - 1
    for (; i + 4 <= len; i += 4) {
        const __m128 a = _mm_castsi128_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
        const __m128 b = _mm_castsi128_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 2)));
        const __m128i lo = _mm_castps_si128(_mm_shuffle_ps(a, b, _MM_SHUFFLE(2, 0, 2, 0)));
        const __m128i hi = _mm_castps_si128(_mm_shuffle_ps(a, b, _MM_SHUFFLE(3, 1, 3, 1)));
        hi_any = _mm_or_si128(hi_any, hi);
        sgn = _mm_or_si128(sgn, _mm_or_si128(lo, _mm_cmpgt_epi32(lo, bm1)));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), lo);
    }
    acc |= (uint64_t)(_mm_movemask_epi8(_mm_cmpeq_epi32(hi_any, _mm_setzero_si128())) != 0xFFFF);
    acc |= (uint64_t)(_mm_movemask_ps(_mm_castsi128_ps(sgn)) != 0);
    for (; i < len; ++i) {
        const uint64_t v = (uint64_t)src[i];
        acc |= (uint64_t)(v >= bound);
        dst[i] = (uint32_t)v;
    }
    return acc;
}

// u32 -> int64 over [0, len), 16-B non-temporal stores into the caller's array
inline void widen(const uint32_t* src, int64_t* dst, size_t len) {
    size_t i = 0;
    for (; i < len && ((uintptr_t)(dst + i) & 15); ++i) dst[i] = (int64_t)src[i];
    const __m128i z = _mm_setzero_si128();
    for (; i + 4 <= len; i += 4) {
        const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_unpacklo_epi32(x, z));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2), _mm_unpackhi_epi32(x, z));
    }
    for (; i < len; ++i) dst[i] = (int64_t)src[i];
}
}  // namespace
}  // namespace sg

extern "C" {

int sg_xfer_threads(void) { return sg::pool().size(); }

int sg_h2d_narrow_i64(const int64_t* host, uint64_t count, uint32_t* dev, uint64_t bound, void* stream,
                      int* in_range) {
    using namespace sg;
    *in_range = 1;
    if (count == 0) return SG_OK;
    if (!host || !dev) return SG_ERR_VALUE;
    std::lock_guard<std::mutex> lk(g_ring_mu);  // one pipelined copy at a time per process
    Ring* r = ring_for_current_device();
    if (!r) {
        cudaGetLastError();
        return SG_ERR_CUDA;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t kChunkV = chunk_ids();
    std::atomic<int> bad{0};
    const uint64_t nchunks = (count + kChunkV - 1) / kChunkV;
    for (uint64_t k = 0; k < nchunks; ++k) {
        const int sl = (int)(k % kSlots);
        const size_t off = k * kChunkV;
        const size_t len = std::min<uint64_t>(kChunkV, count - off);
        SG_CUDA(cudaEventSynchronize(r->ev[sl]));  // the slot's previous DMA has finished
        uint32_t* dst = r->slot[sl];
        const int64_t* src = host + off;
        pool().run([&](int p, int parts) {
            size_t lo, hi;
            split(len, p, parts, lo, hi);
            if (narrow_range(src + lo, dst + lo, hi - lo, bound)) bad.store(1, std::memory_order_relaxed);
            _mm_sfence();  // the non-temporal stores are visible before the DMA reads the slot
        });
        if (bad.load(std::memory_order_relaxed)) {
            *in_range = 0;  // the caller copies int64 instead; the device reports the exact error
            return SG_OK;
        }
        SG_CUDA(cudaMemcpyAsync(dev + off, dst, len * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        SG_CUDA(cudaEventRecord(r->ev[sl], s));
    }
    return SG_OK;
}

int sg_d2h_widen_u32(const uint32_t* dev, uint64_t count, int64_t* host, void* stream) {
    using namespace sg;
    if (count == 0) return SG_OK;
    if (!host || !dev) return SG_ERR_VALUE;
    std::lock_guard<std::mutex> lk(g_ring_mu);
    Ring* r = ring_for_current_device();
    if (!r) {
        cudaGetLastError();
        return SG_ERR_CUDA;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t kChunkV = chunk_ids();
    const uint64_t nchunks = (count + kChunkV - 1) / kChunkV;
    auto widen_chunk = [&](uint64_t k) -> int {
        const int sl = (int)(k % kSlots);
        const size_t off = k * kChunkV;
        const size_t len = std::min<uint64_t>(kChunkV, count - off);
        SG_CUDA(cudaEventSynchronize(r->ev[sl]));
        const uint32_t* src = r->slot[sl];
        int64_t* dst = host + off;
        pool().run([&](int p, int parts) {
            size_t lo, hi;
            split(len, p, parts, lo, hi);
            widen(src + lo, dst + lo, hi - lo);
            _mm_sfence();
        });
        return SG_OK;
    };
    // keep kSlots - 1 copies in flight ahead of the widening
    for (uint64_t k = 0; k < nchunks; ++k) {
        const int sl = (int)(k % kSlots);
        if (k >= (uint64_t)kSlots) {
            const int rc = widen_chunk(k - kSlots);  // frees slot sl
            if (rc != SG_OK) return rc;
        }
        const size_t off = k * kChunkV;
        const size_t len = std::min<uint64_t>(kChunkV, count - off);
        SG_CUDA(cudaMemcpyAsync(r->slot[sl], dev + off, len * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaEventRecord(r->ev[sl], s));
    }
    for (uint64_t k = nchunks > (uint64_t)kSlots ? nchunks - kSlots : 0; k < nchunks; ++k) {
        const int rc = widen_chunk(k);
        if (rc != SG_OK) return rc;
    }
    return SG_OK;
}

}  // extern "C"
