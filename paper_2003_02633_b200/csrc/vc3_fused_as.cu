// vc3_fused_as.cu — the fused operations' all-single path on table layouts
// (the reference benchmark's configuration, bench.py:41-69): four vectors per
// thread step through the restructured decode / compress of vc3_fused.cuh.
// Dispatched from vc3_fused.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"
#include "vc3_fused.cuh"
#include "vc3_kern_common.cuh"
#include "vc3_rt.h"

namespace {

constexpr unsigned kAllSingle = 7u;

// ===================== all-single path on table layouts ======================
// Four vectors per thread step: eight fast table decodes, float32 sums, two
// compress_as2 pairs.  The rare exceptions take warp-uniform branches (one
// vote each per step, so the exception code is never predicated into the
// hot path): the exact mode's boundary redo (decode_redo, ~1e-5 of words) and
// the compress range exceptions (the generic bit-exact compress_one).
template <bool EXACT>
__device__ __forceinline__ void decode4(const unsigned long long w[4], const Params& P,
                                        const DecTab& T, const double2* full, double tol2,
                                        float x[4], float y[4], float z[4]) {
    unsigned redo = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        redo |= (unsigned)decode_fused<EXACT>(w[k], P, T, tol2, x[k], y[k], z[k]) << k;
    if (EXACT && __any_sync(__activemask(), redo != 0u)) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((redo >> k) & 1u) decode_redo(w[k], P, full, x[k], y[k], z[k]);
    }
}

// BOUNDED: the inputs are float32 sums of decoded default-layout vectors
// (|component| < 2^48), so the overflow range tests can be skipped.
template <bool BOUNDED = false>
__device__ __forceinline__ void encode4(const float x[4], const float y[4], const float z[4],
                                        const Params& P, unsigned long long w[4]) {
    bool slow[4];
    compress_as2<BOUNDED>(x, y, z, P, w, slow);
    compress_as2<BOUNDED>(x + 2, y + 2, z + 2, P, w + 2, slow + 2);
    if (__any_sync(__activemask(), slow[0] | slow[1] | slow[2] | slow[3])) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (slow[k]) w[k] = compress_one<kAllSingle, true, true>(x[k], y[k], z[k], P);
    }
}

// float32 sums of two decoded pairs (one FADD2 per component pair)
__device__ __forceinline__ void add_pairs(const float a[2], const float b[2], float out[2]) {
    upk(add2(pk(a[0], a[1]), pk(b[0], b[1])), out[0], out[1]);
}

// sums / combinations of two decoded words stay below 2^61 only for the
// default layout's magnitudes (< 2^47); runtime layouts keep every range test
template <class LAY>
constexpr bool kBounded = std::is_same<LAY, DefaultLayout>::value;

#ifndef VC3_ADD_AS_MIN_BLOCKS
#define VC3_ADD_AS_MIN_BLOCKS 3  // measured: 3 resident CTAs (80 registers, no spills) beat 4 (64, spills)
#endif
// CFG: the shared-memory copy and CTA shape (fused_copy): 0 = 3 CTAs x 256
// threads per SM; 1, 2 = one CTA x 768 threads per SM with replicated grids
// (theta x2 / phi x4, or theta x4 / phi x4)
template <int CFG>
constexpr int kAsThreads = CFG ? 768 : kThreads;
template <int CFG>
constexpr int kAsMinBlocks = CFG ? 1 : VC3_ADD_AS_MIN_BLOCKS;

template <bool EXACT, class LAY, int CFG = 0>
__global__ void __launch_bounds__(kAsThreads<CFG>, kAsMinBlocks<CFG>)
    k_add_as(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
             unsigned long long* __restrict__ c, int64_t n, Params Pin, bool vec,
             const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    const FusedCopy F = fused_copy<CFG>(P);
    load_table_fused(s_tab, gtab, P, F);
    const DecTab T = dec_tab(s_tab, F);
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        const u64x4 u = ld_stream_u4(a + 4 * g), v = ld_stream_u4(b + 4 * g);
        const unsigned long long wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
        float xa[4], ya[4], za[4], xb[4], yb[4], zb[4], x[4], y[4], z[4];
        decode4<EXACT>(wa, P, T, full, tol2, xa, ya, za);
        decode4<EXACT>(wb, P, T, full, tol2, xb, yb, zb);
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
            add_pairs(xa + k, xb + k, x + k);
            add_pairs(ya + k, yb + k, y + k);
            add_pairs(za + k, zb + k, z + k);
        }
        unsigned long long w[4];
        encode4<kBounded<LAY>>(x, y, z, P, w);
        st_u4(c + 4 * g, w[0], w[1], w[2], w[3]);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float x1, y1, z1, x2, y2, z2;
        const unsigned long long wa = a[i], wb = b[i];
        if (decode_fused<EXACT>(wa, P, T, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, T, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
        c[i] = compress_one<kAllSingle, true, true>(__fadd_rn(x1, x2), __fadd_rn(y1, y2),
                                                    __fadd_rn(z1, z2), P);
    }
}

// K4 axpy, all-single: y' = compress(alpha * decode(x) + decode(y)), the
// float32 product and sum rounded separately (scalar: a packed product may
// not feed a packed sum, vc3_fused.cuh).  y may alias y_out.
template <bool EXACT, class LAY, int CFG = 0>
__global__ void __launch_bounds__(kAsThreads<CFG>, kAsMinBlocks<CFG>)
    k_axpy_as(float al, const unsigned long long* __restrict__ xw, const unsigned long long* yw,
              unsigned long long* yo, int64_t n, Params Pin, bool vec,
              const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    const FusedCopy F = fused_copy<CFG>(P);
    load_table_fused(s_tab, gtab, P, F);
    const DecTab T = dec_tab(s_tab, F);
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        const u64x4 u = ld_stream_u4(xw + 4 * g);
        u64x4 v;
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w)
                     : "l"(yw + 4 * g));
        const unsigned long long wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
        float xa[4], ya[4], za[4], xb[4], yb[4], zb[4], x[4], y[4], z[4];
        decode4<EXACT>(wa, P, T, full, tol2, xa, ya, za);
        decode4<EXACT>(wb, P, T, full, tol2, xb, yb, zb);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[k] = __fadd_rn(__fmul_rn(al, xa[k]), xb[k]);
            y[k] = __fadd_rn(__fmul_rn(al, ya[k]), yb[k]);
            z[k] = __fadd_rn(__fmul_rn(al, za[k]), zb[k]);
        }
        unsigned long long w[4];
        encode4(x, y, z, P, w);
        st_u4(yo + 4 * g, w[0], w[1], w[2], w[3]);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float x1, y1, z1, x2, y2, z2;
        const unsigned long long wa = xw[i], wb = yw[i];
        if (decode_fused<EXACT>(wa, P, T, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, T, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
        yo[i] = compress_one<kAllSingle, true, true>(__fadd_rn(__fmul_rn(al, x1), x2),
                                                     __fadd_rn(__fmul_rn(al, y1), y2),
                                                     __fadd_rn(__fmul_rn(al, z1), z2), P);
    }
}

// K4b low-storage RK stage, all-single: dq' = a*dq + dt*R ; q' = q + b*dq'
// (float32, each product and sum rounded; q' uses the register dq').
template <bool EXACT>
__device__ __forceinline__ void rk_math(float ca, float cb, float dt, float& q, float& d, float r) {
    d = __fadd_rn(__fmul_rn(ca, d), __fmul_rn(dt, r));
    q = __fadd_rn(q, __fmul_rn(cb, d));
}

template <bool EXACT, class LAY, int CFG = 0>
__global__ void __launch_bounds__(kAsThreads<CFG>, kAsMinBlocks<CFG>)
    k_rk_as(float ca, float cb, float dt, unsigned long long* __restrict__ q,
            unsigned long long* __restrict__ dq, const unsigned long long* __restrict__ R, int64_t n,
            Params Pin, bool vec, const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    const FusedCopy F = fused_copy<CFG>(P);
    load_table_fused(s_tab, gtab, P, F);
    const DecTab T = dec_tab(s_tab, F);
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        u64x4 uq, ud;
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(uq.x), "=l"(uq.y), "=l"(uq.z), "=l"(uq.w) : "l"(q + 4 * g));
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(ud.x), "=l"(ud.y), "=l"(ud.z), "=l"(ud.w) : "l"(dq + 4 * g));
        const u64x4 ur = ld_stream_u4(R + 4 * g);
        const unsigned long long wq[4] = {uq.x, uq.y, uq.z, uq.w}, wd[4] = {ud.x, ud.y, ud.z, ud.w},
                                 wr[4] = {ur.x, ur.y, ur.z, ur.w};
        float qx[4], qy[4], qz[4], dx[4], dy[4], dz[4], rx[4], ry[4], rz[4];
        decode4<EXACT>(wq, P, T, full, tol2, qx, qy, qz);
        decode4<EXACT>(wd, P, T, full, tol2, dx, dy, dz);
        decode4<EXACT>(wr, P, T, full, tol2, rx, ry, rz);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            rk_math<EXACT>(ca, cb, dt, qx[k], dx[k], rx[k]);
            rk_math<EXACT>(ca, cb, dt, qy[k], dy[k], ry[k]);
            rk_math<EXACT>(ca, cb, dt, qz[k], dz[k], rz[k]);
        }
        unsigned long long w[4];
        encode4(dx, dy, dz, P, w);
        st_u4(dq + 4 * g, w[0], w[1], w[2], w[3]);
        encode4(qx, qy, qz, P, w);
        st_u4(q + 4 * g, w[0], w[1], w[2], w[3]);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float q0, q1, q2, d0, d1, d2, r0, r1, r2;
        const unsigned long long wq = q[i], wd = dq[i], wr = R[i];
        if (decode_fused<EXACT>(wq, P, T, tol2, q0, q1, q2)) decode_redo(wq, P, full, q0, q1, q2);
        if (decode_fused<EXACT>(wd, P, T, tol2, d0, d1, d2)) decode_redo(wd, P, full, d0, d1, d2);
        if (decode_fused<EXACT>(wr, P, T, tol2, r0, r1, r2)) decode_redo(wr, P, full, r0, r1, r2);
        rk_math<EXACT>(ca, cb, dt, q0, d0, r0);
        rk_math<EXACT>(ca, cb, dt, q1, d1, r1);
        rk_math<EXACT>(ca, cb, dt, q2, d2, r2);
        dq[i] = compress_one<kAllSingle, true, true>(d0, d1, d2, P);
        q[i] = compress_one<kAllSingle, true, true>(q0, q1, q2, P);
    }
}

// K1 compress, all-single policy: 4 vectors (48 B in, 32 B out) per thread
// step through two compress_as2 pairs; the range exceptions take the generic
// compress_one (warp-uniform branch).  Non-finite inputs are counted (the
// host raises NonFiniteInput; their words are unspecified, as in vc3_compress).
template <class LAY>
__global__ void __launch_bounds__(kThreads, VC3_FUSED_MIN_BLOCKS)
    k_compress_as(const float* __restrict__ xyz, unsigned long long* __restrict__ out, int64_t n,
                  Params Pin, bool vec, int32_t* __restrict__ nonfinite) {
    Params P = Pin;
    LAY::apply(P);
    int bad = 0;
    const int64_t groups = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        const float4 A = ld_stream_f4(xyz + 12 * g), B = ld_stream_f4(xyz + 12 * g + 4),
                     C = ld_stream_f4(xyz + 12 * g + 8);
        const float x[4] = {A.x, A.w, B.z, C.y}, y[4] = {A.y, B.x, B.w, C.z}, z[4] = {A.z, B.y, C.x, C.w};
        bad += !finite3(x[0], y[0], z[0]) + !finite3(x[1], y[1], z[1]) + !finite3(x[2], y[2], z[2]) +
               !finite3(x[3], y[3], z[3]);
        unsigned long long w[4];
        encode4(x, y, z, P, w);
        st_u4(out + 4 * g, w[0], w[1], w[2], w[3]);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        bad += !finite3(x, y, z);
        out[i] = compress_one<kAllSingle, true, true>(x, y, z, P);
    }
    if (bad && nonfinite) atomicAdd(nonfinite, bad);
}

}  // namespace

namespace vc3 {
namespace as {

// Shared memory of the fused kernels: the table copy (fused_copy<CFG>).
template <int CFG>
size_t fused_smem(const Params& P) { return (size_t)fused_copy<CFG>(P).n * sizeof(double2); }

template <int CFG, typename KFn, typename... Args>
int launch_table_kernel(KFn fn, const Params& P, int64_t n, bool vec, cudaStream_t s, Args... args) {
    const size_t smem = fused_smem<CFG>(P);
    if (const int st = ensure_smem((const void*)fn, smem)) return st;
    const int threads = kAsThreads<CFG>;
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + threads - 1) / threads;
    int per_sm = CFG ? VC3_AS1_CTAS_PER_SM : VC3_AS_CTAS_PER_SM;
#ifdef VC3_TUNE
    static const int tune_grid = getenv("VC3_TUNE_GRID") ? atoi(getenv("VC3_TUNE_GRID")) : 0;
    if (tune_grid > 0) per_sm = tune_grid;
#endif
    const int64_t cap = (int64_t)sm_count() * per_sm;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    fn<<<(unsigned)blocks, threads, smem, s>>>(args...);
    return launch_status();
}

// Copy configuration per operation and mode (fused_copy; measured on 2^28
// vectors, Gvec/s exact / contract): add 113.3 / 130.0 with CFG 2, 110.4 /
// 131.1 with CFG 1, 105.4 / 120.4 with CFG 0 (3 x 256 threads); axpy 108.9 /
// 126.2 (CFG 1) vs 109.1 / 120.4 (CFG 2); RK 60.2 / 67.8 (CFG 2) vs 58.9 /
// 64.8 (CFG 1).  CFG 2's copy layout is instantiated for the default layout
// only; other layouts take CFG 1.
enum AsOp { kOpAdd, kOpAxpy, kOpRk };
static int as_cfg(AsOp op, bool exact, bool def) {
    int c = op == kOpAdd ? (exact ? 2 : 1) : (op == kOpAxpy ? 1 : 2);
#ifdef VC3_TUNE
    static const int t = getenv("VC3_TUNE_CFG") ? atoi(getenv("VC3_TUNE_CFG")) : -1;
    if (t >= 0) c = t;
#endif
    return c == 2 && !def ? 1 : c;
}

// Launch the all-single fused add (table layouts).  Returns a vc3_status.
int launch_add(const unsigned long long* a, const unsigned long long* b, unsigned long long* c,
               int64_t n, const Params& P, bool def, bool exact, bool vec, const double2* tab,
               const double2* full, cudaStream_t s) {
    const int cfg = as_cfg(kOpAdd, exact, def);
    if (cfg == 2) {
        auto fn = exact ? k_add_as<true, DefaultLayout, 2> : k_add_as<false, DefaultLayout, 2>;
        return launch_table_kernel<2>(fn, P, n, vec, s, a, b, c, n, P, vec, tab, full);
    }
#ifdef VC3_TUNE
    if (cfg == 0) {  // the round's first form, 3 x 256 threads (A/B builds only)
        auto fn = def ? (exact ? k_add_as<true, DefaultLayout> : k_add_as<false, DefaultLayout>)
                      : (exact ? k_add_as<true, RuntimeLayout> : k_add_as<false, RuntimeLayout>);
        return launch_table_kernel<0>(fn, P, n, vec, s, a, b, c, n, P, vec, tab, full);
    }
#endif
    auto fn = def ? (exact ? k_add_as<true, DefaultLayout, 1> : k_add_as<false, DefaultLayout, 1>)
                  : (exact ? k_add_as<true, RuntimeLayout, 1> : k_add_as<false, RuntimeLayout, 1>);
    return launch_table_kernel<1>(fn, P, n, vec, s, a, b, c, n, P, vec, tab, full);
}

int launch_axpy(float al, const unsigned long long* x, const unsigned long long* y,
                unsigned long long* yo, int64_t n, const Params& P, bool def, bool exact, bool vec,
                const double2* tab, const double2* full, cudaStream_t s) {
    const int cfg = as_cfg(kOpAxpy, exact, def);
    if (cfg == 2) {
        auto fn = exact ? k_axpy_as<true, DefaultLayout, 2> : k_axpy_as<false, DefaultLayout, 2>;
        return launch_table_kernel<2>(fn, P, n, vec, s, al, x, y, yo, n, P, vec, tab, full);
    }
#ifdef VC3_TUNE
    if (cfg == 0) {  // the round's first form, 3 x 256 threads (A/B builds only)
        auto fn = def ? (exact ? k_axpy_as<true, DefaultLayout> : k_axpy_as<false, DefaultLayout>)
                      : (exact ? k_axpy_as<true, RuntimeLayout> : k_axpy_as<false, RuntimeLayout>);
        return launch_table_kernel<0>(fn, P, n, vec, s, al, x, y, yo, n, P, vec, tab, full);
    }
#endif
    auto fn = def ? (exact ? k_axpy_as<true, DefaultLayout, 1> : k_axpy_as<false, DefaultLayout, 1>)
                  : (exact ? k_axpy_as<true, RuntimeLayout, 1> : k_axpy_as<false, RuntimeLayout, 1>);
    return launch_table_kernel<1>(fn, P, n, vec, s, al, x, y, yo, n, P, vec, tab, full);
}

int launch_rk(float ca, float cb, float dt, unsigned long long* q, unsigned long long* dq,
              const unsigned long long* R, int64_t n, const Params& P, bool def, bool exact,
              bool vec, const double2* tab, const double2* full, cudaStream_t s) {
    const int cfg = as_cfg(kOpRk, exact, def);
    if (cfg == 2) {
        auto fn = exact ? k_rk_as<true, DefaultLayout, 2> : k_rk_as<false, DefaultLayout, 2>;
        return launch_table_kernel<2>(fn, P, n, vec, s, ca, cb, dt, q, dq, R, n, P, vec, tab, full);
    }
#ifdef VC3_TUNE
    if (cfg == 0) {  // the round's first form, 3 x 256 threads (A/B builds only)
        auto fn = def ? (exact ? k_rk_as<true, DefaultLayout> : k_rk_as<false, DefaultLayout>)
                      : (exact ? k_rk_as<true, RuntimeLayout> : k_rk_as<false, RuntimeLayout>);
        return launch_table_kernel<0>(fn, P, n, vec, s, ca, cb, dt, q, dq, R, n, P, vec, tab, full);
    }
#endif
    auto fn = def ? (exact ? k_rk_as<true, DefaultLayout, 1> : k_rk_as<false, DefaultLayout, 1>)
                  : (exact ? k_rk_as<true, RuntimeLayout, 1> : k_rk_as<false, RuntimeLayout, 1>);
    return launch_table_kernel<1>(fn, P, n, vec, s, ca, cb, dt, q, dq, R, n, P, vec, tab, full);
}

// The all-single compress (layouts with t <= 25, p <= 24: clamp-free buckets).
int launch_compress(const float* xyz, unsigned long long* w, int64_t n, const Params& P, bool def,
                    bool vec, int32_t* nonfinite, cudaStream_t s) {
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sm_count() * VC3_COMPRESS_CTAS_PER_SM;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    if (def)
        k_compress_as<DefaultLayout><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else
        k_compress_as<RuntimeLayout><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    return launch_status();
}
}  // namespace as
}  // namespace vc3
