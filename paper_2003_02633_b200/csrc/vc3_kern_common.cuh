// vc3_kern_common.cuh — launch helpers, streaming load/store wrappers and the
// shared-memory table loader used by every kernel translation unit of the
// library (vc3_kernels.cu, vc3_fused.cu).  Internal: not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"
#include "vc3_rt.h"

namespace {

using namespace vc3;
using namespace vc3::rt;

constexpr int kThreads = 256;
// measured on B200 (tools/occupancy_sweep.py): 4 vectors per thread step and
// >= 4 resident CTAs per SM (<= 64 registers) give the best fused-add issue rate
#ifndef VC3_FUSED_MIN_BLOCKS
#define VC3_FUSED_MIN_BLOCKS 4
#endif
// the RK stage's exact mode keeps the two-conversion boundary test (ICV field:
// DESIGN §9); the add and axpy use the conversion-free cell test
#ifndef VC3_RK_CELL
#define VC3_RK_CELL 0
#endif
#ifndef VC3_DECOMP_STAGE
#define VC3_DECOMP_STAGE 1
#endif
// grid caps in CTAs per SM for the streaming kernels (grid-stride beyond);
// more CTAs than resident slots balance the tail across SMs (measured)
#ifndef VC3_DECOMP_CELL
#define VC3_DECOMP_CELL 0  // decompress's boundary test: 0 two-conversion, 1 cell test (vc3_device.cuh)
#endif
#ifndef VC3_ADD_CTAS_PER_SM
#define VC3_ADD_CTAS_PER_SM 48
#endif
// grid cap of the all-single table kernels (3 resident per SM; 12 per SM
// measured 120.5 vs 118.8 Gvec/s contract, 105.6 vs 105.4 exact at 48)
#ifndef VC3_AS_CTAS_PER_SM
#define VC3_AS_CTAS_PER_SM 12
#endif
#ifndef VC3_AS1_CTAS_PER_SM
#define VC3_AS1_CTAS_PER_SM 1  // CFG 1, 2 (one 768-thread CTA per SM: persistent)
#endif
#ifndef VC3_COMPRESS_CTAS_PER_SM
#define VC3_COMPRESS_CTAS_PER_SM 48
#endif
#ifndef VC3_DECOMP_CTAS_PER_SM
#define VC3_DECOMP_CTAS_PER_SM 4
#endif
// decompress CTAs: the 49 KB table is shared by more threads per CTA
#ifndef VC3_DECOMP_THREADS
#define VC3_DECOMP_THREADS 512
#endif
#ifndef VC3_DECOMP_MIN_BLOCKS
#define VC3_DECOMP_MIN_BLOCKS 2
#endif


// grid for `items` work items of one thread each: at most `per_sm` CTAs per
// SM (grid-stride beyond that), at least one.
unsigned grid_for(int64_t items, int per_sm = 8) {
    int64_t blocks = (items + kThreads - 1) / kThreads;
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}

// launch a table kernel: opt in to its shared-memory size first
#define VC3_LAUNCH_TABLE(KERNEL, GRID, SMEM, STREAM, ...)                          \
    do {                                                                           \
        const int st_ = ensure_smem((const void*)(KERNEL), (SMEM));                \
        if (st_) return st_;                                                       \
        KERNEL<<<(GRID), kThreads, (SMEM), (STREAM)>>>(__VA_ARGS__);               \
    } while (0)

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
inline bool aligned32(const void* p) { return ((uintptr_t)p & 31u) == 0; }

// ----- streaming loads/stores (read-once data: keep it out of L1) ----------
__device__ __forceinline__ ulonglong2 ld_stream_u2(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
// sm_100 256-bit global accesses (LDG/STG .256): four words per instruction
struct u64x4 {
    unsigned long long x, y, z, w;
};
__device__ __forceinline__ u64x4 ld_stream_u4(const unsigned long long* p) {
    u64x4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_u4(unsigned long long* p, unsigned long long a,
                                      unsigned long long b, unsigned long long c,
                                      unsigned long long d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c),
                 "l"(d)
                 : "memory");
}
__device__ __forceinline__ void st_u2(unsigned long long* p, unsigned long long a,
                                      unsigned long long b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_f4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

__device__ __forceinline__ int64_t gtid() {
    return (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// Copy the decode table into shared memory (once per CTA; grids are capped
// at a few CTAs per SM, so the copy is amortised over the whole stream).
// the decode's boundary tolerance (relative to the magnitude), stored after
// the reference's tables by get_full_table
// CELL: the cell test (needs_exact<true>) takes the doubled tolerance
template <bool CELL = false>
__device__ __forceinline__ double exact_tol(const double2* __restrict__ full, const Params& P) {
    const double t = full ? __ldg(full + (P.ntmax + 1) + (P.npmax + 1)).x : 0.0;
    return CELL ? __dadd_rn(t, t) : t;
}

template <bool TABLE>
__device__ __forceinline__ void load_table(double2* sm, const double2* __restrict__ g,
                                           const Params& P) {
    if (TABLE) {
        const int n = P.tab_n;
        for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = g[i];
        __syncthreads();
    }
}

__device__ __forceinline__ void load_table_fused(double2* sm, const double2* __restrict__ g, const Params& P,
                                                 const FusedCopy& F) {
    for (int i = threadIdx.x; i < F.n; i += blockDim.x) {
        const int src = i < F.tp    ? (i >> F.tg)
                        : i < F.trt ? P.p_base + ((i - F.tp) >> F.pg)
                        : i < F.trp ? P.rt_base + ((i - F.trt) >> F.rt)
                                    : P.rp_base + ((i - F.trp) >> F.rp);
        sm[i] = g[src];
    }
    __syncthreads();
}

// ----- dispatch helpers ----------------------------------------------------------
template <template <unsigned> class F, typename... A>
int by_policy(uint32_t pol, A... args) {
    switch (pol & 7u) {
        case 0: return F<0>::run(args...);
        case 1: return F<1>::run(args...);
        case 2: return F<2>::run(args...);
        case 3: return F<3>::run(args...);
        case 4: return F<4>::run(args...);
        case 5: return F<5>::run(args...);
        case 6: return F<6>::run(args...);
        default: return F<7>::run(args...);
    }
}

#define VC3_CHECK_N(n) \
    if ((n) < 0) return VC3_ERR_ARG; \
    if ((n) == 0) return VC3_OK;

}  // namespace
