// Per-stage SASS budget probes for the fused path (tools/sass_loop.py reads
// the loop bodies).  Each kernel is one stage of the fused add's per-vector
// work in the same 4-vectors-per-thread loop as the product kernel; the rare
// slow paths are replaced by a token so only the hot path remains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -cubin \
//        -I include -o /tmp/sass_probe.cubin tools/sass_probe.cu
#include "../paper_2003_02633_b200/csrc/vc3_device.cuh"
#include "../paper_2003_02633_b200/csrc/vc3_fused.cuh"

using namespace vc3;
using Lay = DefaultLayout;

struct u64x4p {
    unsigned long long x, y, z, w;
};
__device__ __forceinline__ u64x4p ld4(const unsigned long long* p) {
    u64x4p v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(unsigned long long* p, unsigned long long a, unsigned long long b,
                                    unsigned long long c, unsigned long long d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
                 : "memory");
}

#define PROBE_PROLOGUE                                 \
    Params P = Pin;                                    \
    Lay::apply(P);                                     \
    extern __shared__ double2 s_tab[];                 \
    const DecTab T = dec_tab(s_tab, fused_copy<0>(P)); \
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;

// stage: two decodes of the fused add (contract / exact), sums stored as floats
template <bool EXACT>
__global__ void __launch_bounds__(256, 4) probe_decode2(const unsigned long long* a, const unsigned long long* b,
                                                        float* out, int64_t groups, Params Pin,
                                                        const double2* full, double tol2) {
    PROBE_PROLOGUE
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const u64x4p u = ld4(a + 4 * g), v = ld4(b + 4 * g);
        const unsigned long long wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
        float o[12];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float x1, y1, z1, x2, y2, z2;
            if (decode_fused<EXACT>(wa[k], P, T, tol2, x1, y1, z1)) x1 = -x1;
            if (decode_fused<EXACT>(wb[k], P, T, tol2, x2, y2, z2)) x2 = -x2;
            o[3 * k] = __fadd_rn(x1, x2);
            o[3 * k + 1] = __fadd_rn(y1, y2);
            o[3 * k + 2] = __fadd_rn(z1, z2);
        }
        float4* d = reinterpret_cast<float4*>(out + 12 * g);
        d[0] = make_float4(o[0], o[1], o[2], o[3]);
        d[1] = make_float4(o[4], o[5], o[6], o[7]);
        d[2] = make_float4(o[8], o[9], o[10], o[11]);
    }
}

// stage: the all-single compress of four vectors (fast path only)
__global__ void __launch_bounds__(256, 4) probe_compress(const float* in, unsigned long long* out,
                                                         int64_t groups, Params Pin) {
    PROBE_PROLOGUE
    (void)T;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const float4* s = reinterpret_cast<const float4*>(in + 12 * g);
        const float4 A = s[0], B = s[1], C = s[2];
        const float x[4] = {A.x, A.w, B.z, C.y}, y[4] = {A.y, B.x, B.w, C.z}, z[4] = {A.z, B.y, C.x, C.w};
        unsigned long long w[4];
        bool slow[4];
        compress_as2(x, y, z, P, w, slow);
        compress_as2(x + 2, y + 2, z + 2, P, w + 2, slow + 2);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (slow[k]) w[k] = ~w[k];
        st4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
}

// stage: the round-1 generic compress (compress_one<ALL_SINGLE>) for comparison
__global__ void __launch_bounds__(256, 4) probe_compress_r1(const float* in, unsigned long long* out,
                                                            int64_t groups, Params Pin) {
    PROBE_PROLOGUE
    (void)T;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const float4* s = reinterpret_cast<const float4*>(in + 12 * g);
        const float4 A = s[0], B = s[1], C = s[2];
        st4(out + 4 * g, compress_one<7, true, true>(A.x, A.y, A.z, P),
            compress_one<7, true, true>(A.w, B.x, B.y, P), compress_one<7, true, true>(B.z, B.w, C.x, P),
            compress_one<7, true, true>(C.y, C.z, C.w, P));
    }
}

// the whole fused add (hot path only)
template <bool EXACT>
__global__ void __launch_bounds__(256, 4) probe_add(const unsigned long long* a, const unsigned long long* b,
                                                    unsigned long long* c, int64_t groups, Params Pin,
                                                    const double2* full, double tol2) {
    PROBE_PROLOGUE
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const u64x4p u = ld4(a + 4 * g), v = ld4(b + 4 * g);
        const unsigned long long wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
        float xa[4], ya[4], za[4], xb[4], yb[4], zb[4], x[4], y[4], z[4];
        unsigned redo = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            redo |= (unsigned)decode_fused<EXACT>(wa[k], P, T, tol2, xa[k], ya[k], za[k]) << k;
            redo |= (unsigned)decode_fused<EXACT>(wb[k], P, T, tol2, xb[k], yb[k], zb[k]) << (k + 4);
        }
        if (EXACT && __any_sync(__activemask(), redo != 0u)) xa[0] = -xa[0];
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
            upk(add2(pk(xa[k], xa[k + 1]), pk(xb[k], xb[k + 1])), x[k], x[k + 1]);
            upk(add2(pk(ya[k], ya[k + 1]), pk(yb[k], yb[k + 1])), y[k], y[k + 1]);
            upk(add2(pk(za[k], za[k + 1]), pk(zb[k], zb[k + 1])), z[k], z[k + 1]);
        }
        unsigned long long w[4];
        bool slow[4];
        compress_as2<true>(x, y, z, P, w, slow);
        compress_as2<true>(x + 2, y + 2, z + 2, P, w + 2, slow + 2);
        if (__any_sync(__activemask(), slow[0] | slow[1] | slow[2] | slow[3])) w[0] = ~w[0];
        st4(c + 4 * g, w[0], w[1], w[2], w[3]);
    }
}


// stage probes: each reads four vectors (48 B) and writes four words, so the
// loop overhead is the same as probe_copy's
__device__ __forceinline__ void ld12(const float* in, int64_t g, float x[4], float y[4], float z[4]) {
    const float4* s = reinterpret_cast<const float4*>(in + 12 * g);
    const float4 A = s[0], B = s[1], C = s[2];
    x[0] = A.x; y[0] = A.y; z[0] = A.z; x[1] = A.w; y[1] = B.x; z[1] = B.y;
    x[2] = B.z; y[2] = B.w; z[2] = C.x; x[3] = C.y; y[3] = C.z; z[3] = C.w;
}

__global__ void __launch_bounds__(256, 3) probe_copy(const float* in, unsigned long long* out, int64_t groups) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        float x[4], y[4], z[4];
        ld12(in, g, x, y, z);
        unsigned long long w[4];
        for (int k = 0; k < 4; ++k)
            w[k] = ((unsigned long long)__float_as_uint(x[k]) << 32) ^ __float_as_uint(y[k]) ^ __float_as_uint(z[k]);
        st4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(256, 3) probe_theta(const float* in, unsigned long long* out, int64_t groups,
                                                      Params Pin) {
    PROBE_PROLOGUE
    (void)T;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        float x[4], y[4], z[4];
        ld12(in, g, x, y, z);
        int nt[4];
        bool slow[4];
        theta2<true>(x, y, P, nt, slow);
        theta2<true>(x + 2, y + 2, P, nt + 2, slow + 2);
        unsigned long long w[4];
        for (int k = 0; k < 4; ++k) w[k] = (unsigned long long)nt[k] ^ __float_as_uint(z[k]) ^ slow[k];
        st4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(256, 3) probe_phi(const float* in, unsigned long long* out, int64_t groups,
                                                    Params Pin) {
    PROBE_PROLOGUE
    (void)T;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        float x[4], y[4], z[4];
        ld12(in, g, x, y, z);
        int nph[4];
        bool slow[4] = {false, false, false, false};
        phi2<true>(x, y, z, P, nph, slow);
        phi2<true>(x + 2, y + 2, z + 2, P, nph + 2, slow + 2);
        unsigned long long w[4];
        for (int k = 0; k < 4; ++k) w[k] = (unsigned long long)nph[k] ^ slow[k];
        st4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(256, 3) probe_mag(const float* in, unsigned long long* out, int64_t groups,
                                                    Params Pin) {
    PROBE_PROLOGUE
    (void)T;
    for (int64_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        float x[4], y[4], z[4];
        ld12(in, g, x, y, z);
        unsigned long long w[4];
        for (int k = 0; k < 4; ++k) {
            bool slow = false;
            w[k] = (unsigned long long)mag_field_fast(x[k], y[k], z[k], P, slow) ^ slow;
        }
        st4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
}

template __global__ void probe_decode2<false>(const unsigned long long*, const unsigned long long*, float*,
                                              int64_t, Params, const double2*, double);
template __global__ void probe_decode2<true>(const unsigned long long*, const unsigned long long*, float*,
                                             int64_t, Params, const double2*, double);
template __global__ void probe_add<false>(const unsigned long long*, const unsigned long long*,
                                          unsigned long long*, int64_t, Params, const double2*, double);
template __global__ void probe_add<true>(const unsigned long long*, const unsigned long long*,
                                         unsigned long long*, int64_t, Params, const double2*, double);
