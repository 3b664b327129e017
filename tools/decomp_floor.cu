// Decompress floor microbenchmark: what the memory side of
// k_decompress allows before any decode arithmetic.  Same launch shape as the
// shipped kernel (512 threads, 2 CTAs per SM, 4 words per thread step, the
// 49 KB default-layout table in shared memory, per-warp output staging):
//
//   copy     : 8 B in, 12 B out per word (integer ops only), staged output
//   lookup   : copy + the two random 16-byte table loads per word the decode
//              does (theta grid entry nt >> 7, phi grid entry nph >> 7), summed
//   lookup2  : copy + four loads per word (the fused path's two-level form)
//
// Build and run (one GPU):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/decomp_floor tools/decomp_floor.cu
//   /tmp/decomp_floor            # prints Gword/s per variant, 2^28 random words
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kThreads = 512;
constexpr int kTabN = 2049 + 1025;  // theta grid + endpoint, phi grid + pole (default layout)

struct u64x4 {
    unsigned long long x, y, z, w;
};
__device__ __forceinline__ u64x4 ld4(const unsigned long long* p) {
    u64x4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w)
                 : "l"(p));
    return v;
}

template <int LOOKUPS>
__global__ void __launch_bounds__(kThreads, 2)
    k_floor(const unsigned long long* __restrict__ w, float* __restrict__ xyz, int64_t n,
            const double2* __restrict__ gtab) {
    extern __shared__ double2 s_tab[];
    for (int i = threadIdx.x; i < kTabN + 128 * 2; i += blockDim.x) s_tab[i] = gtab[i % kTabN];
    __syncthreads();
    float4* stage = reinterpret_cast<float4*>(s_tab + kTabN + 256) + (threadIdx.x >> 5) * 96;
    const int lane = threadIdx.x & 31;
    const int64_t groups = n / 4, stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t gw_end = ((groups + 31) / 32) * 32;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < gw_end; g += stride) {
        u64x4 u = {0, 0, 0, 0};
        if (g < groups) u = ld4(w + 4 * g);
        const unsigned long long ws[4] = {u.x, u.y, u.z, u.w};
        float o[12];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned nt = (unsigned)ws[k] & 0x3ffffu, np = (unsigned)(ws[k] >> 18) & 0x1ffffu;
            float a = __uint_as_float(((unsigned)(ws[k] >> 40) & 0x7fffffu) | 0x3f800000u);
            float b = __uint_as_float((nt & 0x7fffffu) | 0x3f800000u), c = __uint_as_float(np | 0x3f800000u);
            if (LOOKUPS >= 2) {
                const double2 A = s_tab[nt >> 7], B = s_tab[2049 + (np >> 7)];
                a += (float)(A.x + B.y);
                b += (float)(A.y + B.x);
            }
            if (LOOKUPS >= 4) {
                const double2 R = s_tab[kTabN + (nt & 127)], S = s_tab[kTabN + 128 + (np & 127)];
                c += (float)(R.x + S.y + R.y + S.x);
            }
            o[3 * k] = a;
            o[3 * k + 1] = b;
            o[3 * k + 2] = c;
        }
        stage[3 * lane] = make_float4(o[0], o[1], o[2], o[3]);
        stage[3 * lane + 1] = make_float4(o[4], o[5], o[6], o[7]);
        stage[3 * lane + 2] = make_float4(o[8], o[9], o[10], o[11]);
        __syncwarp();
        const int64_t g0 = g - lane;
        float4* base = reinterpret_cast<float4*>(xyz + 12 * g0);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int idx = 32 * k + lane;
            if (g0 + idx / 3 < groups) base[idx] = stage[idx];
        }
        __syncwarp();
    }
}

template <int L>
float run(const unsigned long long* w, float* xyz, int64_t n, const double2* tab, int sms) {
    const size_t smem = (size_t)(kTabN + 256) * 16 + kThreads * 48;
    cudaFuncSetAttribute(k_floor<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_floor<L>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int grid = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k_floor<L><<<grid, kThreads, smem>>>(w, xyz, n, tab);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) k_floor<L><<<grid, kThreads, smem>>>(w, xyz, n, tab);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return (float)(n / (ms / reps * 1e-3) / 1e9);
}

int main() {
    const int64_t n = int64_t(1) << 28;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* w;
    float* xyz;
    double2* tab;
    cudaMalloc(&w, n * 8);
    cudaMalloc(&xyz, n * 12);
    cudaMalloc(&tab, kTabN * 16);
    std::vector<unsigned long long> h(1 << 20);
    unsigned long long s = 0x9E3779B97F4A7C15ull;
    for (auto& v : h) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        v = s;
    }
    for (int64_t off = 0; off < n; off += (int64_t)h.size())
        cudaMemcpy(w + off, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double2> ht(kTabN);
    for (int i = 0; i < kTabN; ++i) ht[i] = make_double2(0.001 * i, 1.0 - 0.0001 * i);
    cudaMemcpy(tab, ht.data(), kTabN * 16, cudaMemcpyHostToDevice);
    const float c = run<0>(w, xyz, n, tab, sms), l = run<2>(w, xyz, n, tab, sms), l2 = run<4>(w, xyz, n, tab, sms);
    printf("{\"copy_gword_s\": %.1f, \"lookup2_gword_s\": %.1f, \"lookup4_gword_s\": %.1f, "
           "\"hbm_ceiling_gword_s\": %.1f}\n",
           c, l, l2, 6448.1 / 20.0);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
