// umma_bench.cu — tcgen05.mma kind::tf32 issue-rate microbenchmark on one
// CTA per SM: back-to-back M=128, K=8 MMAs with N = 64/128/256 from shared
// memory (no-swizzle K-major), reports dense TF32 TFLOP/s over all SMs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
    return (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) |
           ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_bench(int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    float* f = reinterpret_cast<float*>(sm);
    for (int i = threadIdx.x; i < (128 + N) * 8 * 2; i += blockDim.x) f[i] = 1.0f / (1 + (i & 7));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint64_t a = desc(sm), b = desc(sm + 128 * 8 * 4);
        const uint32_t id = idesc(128, N);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (TS)  // A from TMEM (columns 256.. of the allocation)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
                             "r"(tmem + 256u), "l"(b), "r"(id), "r"(i));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                             "l"(a), "l"(b), "r"(id), "r"(i));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}"
                         : "=r"(done) : "r"(smem_u32(&bar)));
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS>
void run(int sms) {
    const int iters = 20000;
    unsigned long long* d;
    cudaMalloc(&d, sms * 8);
    const size_t smem = (size_t)(128 + N) * 8 * 4 * 2 + 1024;
    cudaFuncSetAttribute(k_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<N, TS><<<sms, 128, smem>>>(100, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_bench<N, TS><<<sms, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 8 * (double)iters * sms;
    printf("%s N=%3d: %.1f TFLOP/s tf32 dense (%.1f cycles per MMA on SM0) err=%s\n", TS ? "A:tmem" : "A:smem", N, flops / (ms * 1e-3) / 1e12,
           (double)c / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, false>(sms);
    run<128, false>(sms);
    run<256, false>(sms);
    run<128, true>(sms);
    run<256, true>(sms);
    return 0;
}
