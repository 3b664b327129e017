// vc3_host.cu — host-buffer entry points of the C ABI (include/vc3_b200.h).
//
// The reference API takes host arrays (numpy) and returns host arrays
// (codec.py:189-228, bench.py:41-51).  These entry points give the same
// contract from C: the input is streamed to the device in chunks on three
// CUDA streams so that the host->device copy of chunk k+1, the kernel on chunk
// k and the device->host copy of chunk k-1 overlap (separate copy engines).
// Device staging comes from a library-private stream-ordered memory pool that
// keeps its memory between calls, so repeated calls do not pay cudaMalloc.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

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

struct DeviceCtx {
    cudaMemPool_t pool = nullptr;
    cudaStream_t streams[kStreams] = {};
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

// Generic chunked pipeline: per chunk, `in_bytes` lists the host inputs'
// bytes per element, the kernel callback runs on device copies, and one output
// of `out_bytes` per element comes back.
template <int NIN, typename Kernel>
int pipeline(const void* const (&in)[NIN], const int (&in_bytes)[NIN], void* out, int out_bytes,
             int64_t n, int device, Kernel kernel) {
    if (n < 0) return VC3_ERR_ARG;
    if (n == 0) return VC3_OK;
    DeviceGuard guard(device);
    if (!guard.ok) return VC3_ERR_CUDA;
    DeviceCtx* ctx = nullptr;
    int st = ctx_for(device, &ctx);
    if (st) return st;
    std::lock_guard<std::recursive_mutex> call_lock(ctx->call_mu);
    const int64_t chunk = std::min(n, kChunk);
    const int nbuf = (int)std::min<int64_t>(kStreams, (n + chunk - 1) / chunk);
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
    }
    for (int64_t off = 0, k = 0; off < n && !st; off += chunk, ++k) {
        const int b = (int)(k % nbuf);
        cudaStream_t s = ctx->streams[b];
        const int64_t cnt = std::min(chunk, n - off);
        for (int i = 0; i < NIN; ++i)
            if (cudaMemcpyAsync(dev_in[b][i], (const char*)in[i] + off * in_bytes[i],
                                cnt * in_bytes[i], cudaMemcpyHostToDevice, s) != cudaSuccess)
                st = VC3_ERR_CUDA;
        if (!st) st = kernel((const void* const*)dev_in[b], (void*)dev_out[b], cnt, s);
        if (!st && cudaMemcpyAsync((char*)out + off * out_bytes, dev_out[b], cnt * out_bytes,
                                   cudaMemcpyDeviceToHost, s) != cudaSuccess)
            st = VC3_ERR_CUDA;
    }
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
