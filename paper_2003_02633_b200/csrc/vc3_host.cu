// vc3_host.cu — host-buffer entry points of the C ABI (include/vc3_b200.h).
//
// The reference API takes host arrays (numpy) and returns host arrays
// (codec.py:189-228, bench.py:41-51).  These entry points give the same
// contract from C: the input is streamed to the device in chunks on three
// CUDA streams so that the host->device copy of chunk k+1, the kernel on chunk
// k and the device->host copy of chunk k-1 overlap (separate copy engines).
// Device staging comes from a library-private stream-ordered memory pool that
// keeps its memory between calls, so repeated calls do not pay cudaMalloc.
//
// Pageable host buffers (plain numpy arrays, the reference's callers) cannot
// be DMA'd directly: the driver would stage them one piece at a time on one
// CPU thread.  For those the pipeline stages through its own pinned ring
// (kept between calls): a pool of host threads copies chunk k + 1 into, and
// chunk k - 2 out of, pinned buffers while the copy engines and the kernel
// work on the chunks in between.
#include <cuda_runtime.h>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/vc3_b200.h"

namespace {

#ifndef VC3_HOST_STREAMS
#define VC3_HOST_STREAMS 3
#endif
#ifndef VC3_HOST_CHUNK_LOG2
#define VC3_HOST_CHUNK_LOG2 23
#endif
constexpr int kStreams = VC3_HOST_STREAMS;
constexpr int64_t kChunk = int64_t(1) << VC3_HOST_CHUNK_LOG2;  // vectors per chunk (2^23: 64 MiB of words)

#ifndef VC3_HOST_STAGE_CHUNK_LOG2
#define VC3_HOST_STAGE_CHUNK_LOG2 21
#endif
constexpr int64_t kStageChunk = int64_t(1) << VC3_HOST_STAGE_CHUNK_LOG2;  // vectors per staged chunk
constexpr int kMaxIo = 3;  // host operands + result per call
#ifndef VC3_HOST_COPY_THREADS
#define VC3_HOST_COPY_THREADS 16u  // staging memcpy threads (capped by the host's cores)
#endif

// Staging copy with streaming (non-temporal) stores: the destination lines
// are written without being read first (a plain memcpy of a few-MB slice
// reads every destination line for ownership, 3 bytes of DRAM traffic per
// byte instead of 2) and do not evict the cache.  The trailing sfence makes
// the stores globally visible before the slice is reported done (the DMA or
// the caller reads them next).
void copy_stream(void* dst, const void* src, size_t n) {
#if defined(__x86_64__)
    char* d = (char*)dst;
    const char* s = (const char*)src;
    const size_t head = std::min(n, (size_t)((16 - ((uintptr_t)d & 15)) & 15));
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    for (; n >= 64; n -= 64, d += 64, s += 64) {
        const __m128i a = _mm_loadu_si128((const __m128i*)s), b = _mm_loadu_si128((const __m128i*)(s + 16)),
                      c = _mm_loadu_si128((const __m128i*)(s + 32)), e = _mm_loadu_si128((const __m128i*)(s + 48));
        _mm_stream_si128((__m128i*)d, a);
        _mm_stream_si128((__m128i*)(d + 16), b);
        _mm_stream_si128((__m128i*)(d + 32), c);
        _mm_stream_si128((__m128i*)(d + 48), e);
    }
    std::memcpy(d, s, n);
    _mm_sfence();
#else
    std::memcpy(dst, src, n);
#endif
}

// Copies into the pinned ring: streaming stores (1) or plain stores (0: the
// ring's lines can stay in the last-level cache, where the copy engine's
// reads find them when the slots are small)
#ifndef VC3_HOST_NT_IN
#define VC3_HOST_NT_IN 1
#endif

// A small pool of host threads for the staging copies (memcpy into / out of
// the pinned ring): one memcpy thread reaches ~10 GB/s, PCIe 5 ~55 GB/s.
class CopyPool {
  public:
    static CopyPool& get() {
        // never destroyed: its workers stay blocked on the condition variable
        // until the process exits (a static object's destructor would tear
        // the mutex down under them at exit)
        static CopyPool* pool = new CopyPool();
        return *pool;
    }
    // copy `bytes` in `nthreads_` slices; returns when all slices are done
    void copy(void* dst, const void* src, size_t bytes, bool nt) {
        const int parts = (int)std::max<size_t>(1, std::min<size_t>(workers_.size() + 1, bytes >> 20));
        const size_t step = (bytes + parts - 1) / parts;
        {
            std::lock_guard<std::mutex> lock(mu_);
            for (int i = 1; i < parts; ++i) {
                const size_t lo = std::min(bytes, step * i), hi = std::min(bytes, lo + step);
                if (hi > lo) {
                    ++pending_;
                    tasks_.push_back([=] {
                        if (nt)
                            copy_stream((char*)dst + lo, (const char*)src + lo, hi - lo);
                        else
                            std::memcpy((char*)dst + lo, (const char*)src + lo, hi - lo);
                    });
                }
            }
        }
        cv_.notify_all();
        if (nt)  // this thread's slice
            copy_stream(dst, src, std::min(bytes, step));
        else
            std::memcpy(dst, src, std::min(bytes, step));
        std::unique_lock<std::mutex> lock(mu_);
        done_cv_.wait(lock, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(VC3_HOST_COPY_THREADS, std::max(1u, hw)) - 1;
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
        for (auto& t : workers_) t.detach();
    }
    void run() {
        for (;;) {
            std::function<void()> task;
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return !tasks_.empty(); });
                task = std::move(tasks_.back());
                tasks_.pop_back();
            }
            task();
            {
                std::lock_guard<std::mutex> lock(mu_);
                --pending_;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::vector<std::function<void()>> tasks_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    int pending_ = 0;
};

struct DeviceCtx {
    cudaMemPool_t pool = nullptr;
    cudaStream_t streams[kStreams] = {};
    char* stage[kStreams][kMaxIo] = {};  // pinned staging ring (pageable callers), grown on demand
    size_t stage_bytes[kStreams][kMaxIo] = {};
    int32_t* d_bad = nullptr;  // non-finite counter of vc3_compress_host (allocated once)
    std::recursive_mutex call_mu;  // one host-buffer call at a time per device (shared streams)
    bool ready = false;
};

std::mutex g_mu;
DeviceCtx g_ctx[64];

int ctx_for(int device, DeviceCtx** out) {
    if (device < 0 || device >= 64) return VC3_ERR_ARG;
    std::lock_guard<std::mutex> lock(g_mu);
    DeviceCtx& c = g_ctx[device];
    if (!c.ready) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&c.pool, &props) != cudaSuccess) return VC3_ERR_CUDA;
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(c.pool, cudaMemPoolAttrReleaseThreshold, &keep);
        for (auto& s : c.streams)
            if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
                return VC3_ERR_CUDA;
        {
            int prev = 0;
            cudaGetDevice(&prev);
            const bool ok = cudaSetDevice(device) == cudaSuccess &&
                            cudaMalloc((void**)&c.d_bad, sizeof(int32_t)) == cudaSuccess;
            cudaSetDevice(prev);
            if (!ok) return VC3_ERR_CUDA;
        }
        c.ready = true;
    }
    *out = &c;
    return VC3_OK;
}

struct DeviceGuard {
    int prev = 0;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear: a plain host pointer is not an error
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int ensure_stage(DeviceCtx* ctx, int slot, int k, size_t bytes) {
    if (ctx->stage_bytes[slot][k] >= bytes) return VC3_OK;
    if (ctx->stage[slot][k]) cudaFreeHost(ctx->stage[slot][k]);
    ctx->stage[slot][k] = nullptr;
    ctx->stage_bytes[slot][k] = 0;
    if (cudaHostAlloc((void**)&ctx->stage[slot][k], bytes, cudaHostAllocPortable) != cudaSuccess)
        return VC3_ERR_CUDA;
    ctx->stage_bytes[slot][k] = bytes;
    return VC3_OK;
}

// Generic chunked pipeline: per chunk, `in_bytes` lists the host inputs'
// bytes per element, the kernel callback runs on device copies, and one output
// of `out_bytes` per element comes back.  Pinned host buffers are copied
// directly; pageable ones go through the pinned staging ring.
template <int NIN, typename Kernel>
int pipeline(const void* const (&in)[NIN], const int (&in_bytes)[NIN], void* out, int out_bytes,
             int64_t n, int device, Kernel kernel) {
    static_assert(NIN + 1 <= kMaxIo, "staging ring holds NIN inputs + 1 output");
    if (n < 0) return VC3_ERR_ARG;
    if (n == 0) return VC3_OK;
    DeviceGuard guard(device);
    if (!guard.ok) return VC3_ERR_CUDA;
    DeviceCtx* ctx = nullptr;
    int st = ctx_for(device, &ctx);
    if (st) return st;
    std::lock_guard<std::recursive_mutex> call_lock(ctx->call_mu);
    bool staged = !is_pinned(out);
    for (int i = 0; i < NIN; ++i) staged = staged || !is_pinned(in[i]);
    const int64_t chunk = std::min(n, staged ? kStageChunk : kChunk);
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const int nbuf = (int)std::min<int64_t>(kStreams, nchunks);
    char* dev_in[kStreams][NIN] = {};
    char* dev_out[kStreams] = {};
    for (int b = 0; b < nbuf && !st; ++b) {
        for (int k = 0; k < NIN && !st; ++k)
            if (cudaMallocFromPoolAsync((void**)&dev_in[b][k], chunk * in_bytes[k], ctx->pool,
                                        ctx->streams[b]) != cudaSuccess)
                st = VC3_ERR_CUDA;
        if (!st && cudaMallocFromPoolAsync((void**)&dev_out[b], chunk * out_bytes, ctx->pool,
                                           ctx->streams[b]) != cudaSuccess)
            st = VC3_ERR_CUDA;
        if (staged) {
            for (int k = 0; k < NIN && !st; ++k) st = ensure_stage(ctx, b, k, chunk * in_bytes[k]);
            if (!st) st = ensure_stage(ctx, b, NIN, chunk * out_bytes);
        }
    }
    CopyPool& pool = CopyPool::get();
    // staged: copy a finished chunk's result out of its pinned slot
    auto retire = [&](int64_t kk) {
        const int b = (int)(kk % nbuf);
        const int64_t off = kk * chunk, cnt = std::min(chunk, n - off);
        if (cudaStreamSynchronize(ctx->streams[b]) != cudaSuccess) return VC3_ERR_CUDA;
        pool.copy((char*)out + off * out_bytes, ctx->stage[b][NIN], cnt * out_bytes, true);
        return VC3_OK;
    };
    for (int64_t k = 0; k < nchunks && !st; ++k) {
        const int b = (int)(k % nbuf);
        cudaStream_t s = ctx->streams[b];
        const int64_t off = k * chunk, cnt = std::min(chunk, n - off);
        if (staged && k >= nbuf) st = retire(k - nbuf);  // slot b's previous chunk
        if (st) break;
        for (int i = 0; i < NIN; ++i) {
            const char* src = (const char*)in[i] + off * in_bytes[i];
            if (staged) {
                pool.copy(ctx->stage[b][i], src, cnt * in_bytes[i], VC3_HOST_NT_IN != 0);
                src = ctx->stage[b][i];
            }
            if (cudaMemcpyAsync(dev_in[b][i], src, cnt * in_bytes[i], cudaMemcpyHostToDevice, s) !=
                cudaSuccess)
                st = VC3_ERR_CUDA;
        }
        if (!st) st = kernel((const void* const*)dev_in[b], (void*)dev_out[b], cnt, s);
        char* dst = staged ? ctx->stage[b][NIN] : (char*)out + off * out_bytes;
        if (!st && cudaMemcpyAsync(dst, dev_out[b], cnt * out_bytes, cudaMemcpyDeviceToHost, s) !=
                       cudaSuccess)
            st = VC3_ERR_CUDA;
    }
    if (staged && !st)
        for (int64_t k = std::max<int64_t>(0, nchunks - nbuf); k < nchunks && !st; ++k) st = retire(k);
    for (int b = 0; b < nbuf; ++b) {
        for (int k = 0; k < NIN; ++k)
            if (dev_in[b][k]) cudaFreeAsync(dev_in[b][k], ctx->streams[b]);
        if (dev_out[b]) cudaFreeAsync(dev_out[b], ctx->streams[b]);
    }
    for (int b = 0; b < nbuf; ++b)
        if (cudaStreamSynchronize(ctx->streams[b]) != cudaSuccess && !st) st = VC3_ERR_CUDA;
    return st;
}

}  // namespace

extern "C" {

int vc3_add_compressed_host(const uint64_t* a_host, const uint64_t* b_host, uint64_t* c_host,
                            int64_t n, vc3_layout layout, uint32_t policy, int32_t device) {
    if (vc3_validate_layout(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u || (n > 0 && (!a_host || !b_host || !c_host))) return VC3_ERR_ARG;
    const void* const in[2] = {a_host, b_host};
    const int bytes[2] = {8, 8};
    return pipeline<2>(in, bytes, c_host, 8, n, device,
                       [&](const void* const* d, void* o, int64_t cnt, cudaStream_t s) {
                           return vc3_add_compressed((const uint64_t*)d[0], (const uint64_t*)d[1],
                                                     (uint64_t*)o, cnt, layout, policy, s);
                       });
}

int vc3_compress_host(const float* xyz_host, uint64_t* words_host, int64_t n, vc3_layout layout,
                      uint32_t policy, int64_t* nonfinite_out, int32_t device) {
    if (vc3_validate_layout(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u || (n > 0 && (!xyz_host || !words_host))) return VC3_ERR_ARG;
    if (nonfinite_out) *nonfinite_out = 0;
    if (n == 0) return VC3_OK;
    DeviceCtx* ctx = nullptr;
    int st = ctx_for(device, &ctx);
    if (st) return st;
    int32_t* d_bad = ctx->d_bad;
    std::lock_guard<std::recursive_mutex> call_lock(ctx->call_mu);  // held across the pipeline
    {
        // zeroed and synchronised before any pipeline stream touches it
        DeviceGuard guard(device);
        if (!guard.ok || cudaMemsetAsync(d_bad, 0, sizeof(int32_t), ctx->streams[0]) != cudaSuccess ||
            cudaStreamSynchronize(ctx->streams[0]) != cudaSuccess)
            return VC3_ERR_CUDA;
    }
    const void* const in[1] = {xyz_host};
    const int bytes[1] = {12};
    st = pipeline<1>(in, bytes, words_host, 8, n, device,
                     [&](const void* const* d, void* o, int64_t cnt, cudaStream_t s) {
                         return vc3_compress((const float*)d[0], (uint64_t*)o, cnt, layout, policy,
                                             d_bad, s);
                     });
    // the pipeline synchronised its streams: the count is final
    DeviceGuard guard(device);
    int32_t bad = 0;
    if (cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->streams[0]) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->streams[0]) != cudaSuccess) {
        if (!st) st = VC3_ERR_CUDA;
    }
    if (nonfinite_out) *nonfinite_out = bad;
    if (!st && bad > 0) st = VC3_ERR_NONFINITE;
    return st;
}

int vc3_decompress_host(const uint64_t* words_host, float* xyz_host, int64_t n, vc3_layout layout,
                        int32_t device) {
    if (vc3_validate_layout(layout)) return VC3_ERR_LAYOUT;
    if (n > 0 && (!words_host || !xyz_host)) return VC3_ERR_ARG;
    const void* const in[1] = {words_host};
    const int bytes[1] = {8};
    return pipeline<1>(in, bytes, xyz_host, 12, n, device,
                       [&](const void* const* d, void* o, int64_t cnt, cudaStream_t s) {
                           return vc3_decompress((const uint64_t*)d[0], (float*)o, cnt, layout, s);
                       });
}

}  // extern "C"
