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
                                        const double2* tt, const double2* tp, const double2* full,
                                        double tol2, float x[4], float y[4], float z[4]) {
    unsigned redo = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        redo |= (unsigned)decode_fused<EXACT>(w[k], P, tt, tp, tol2, x[k], y[k], z[k]) << k;
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
template <bool EXACT, class LAY, int MINB = VC3_ADD_AS_MIN_BLOCKS, int PREFETCH = 0>
__global__ void __launch_bounds__(kThreads, MINB)
    k_add_as(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
             unsigned long long* __restrict__ c, int64_t n, Params Pin, bool vec,
             const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<true>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    // PREFETCH 1: the next step's words are loaded before this step's decode
    // (register double buffering); 2: loaded after the decodes, so their
    // latency hides behind the compress half while the decode's registers
    // are free
    int64_t g = gtid();
    u64x4 un = {0, 0, 0, 0}, vn = un;
    if ((PREFETCH == 1 || PREFETCH == 2) && g < groups) {
        un = ld_stream_u4(a + 4 * g);
        vn = ld_stream_u4(b + 4 * g);
    }
    for (; g < groups; g += gstride()) {
        u64x4 u, v;
        const int64_t gn = g + gstride();
        if (PREFETCH >= 3) {
            // 3 / 4: the words of the step one / two grid strides ahead are
            // prefetched into L2, so this thread's next loads hit L2
            const int64_t gp = g + (PREFETCH - 2) * gstride();
            if (gp < groups) {
                prefetch_l2(a + 4 * gp);
                prefetch_l2(b + 4 * gp);
            }
        }
        if (PREFETCH == 1 || PREFETCH == 2) {
            u = un;
            v = vn;
            if (PREFETCH == 1 && gn < groups) {
                un = ld_stream_u4(a + 4 * gn);
                vn = ld_stream_u4(b + 4 * gn);
            }
        } else {
            u = ld_stream_u4(a + 4 * g);
            v = ld_stream_u4(b + 4 * g);
        }
        const unsigned long long wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
        float xa[4], ya[4], za[4], xb[4], yb[4], zb[4], x[4], y[4], z[4];
        decode4<EXACT>(wa, P, tt, tp, full, tol2, xa, ya, za);
        decode4<EXACT>(wb, P, tt, tp, full, tol2, xb, yb, zb);
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
            add_pairs(xa + k, xb + k, x + k);
            add_pairs(ya + k, yb + k, y + k);
            add_pairs(za + k, zb + k, z + k);
        }
        if (PREFETCH == 2 && gn < groups) {
            un = ld_stream_u4(a + 4 * gn);
            vn = ld_stream_u4(b + 4 * gn);
        }
        unsigned long long w[4];
        encode4<kBounded<LAY>>(x, y, z, P, w);
        st_u4(c + 4 * g, w[0], w[1], w[2], w[3]);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float x1, y1, z1, x2, y2, z2;
        const unsigned long long wa = a[i], wb = b[i];
        if (decode_fused<EXACT>(wa, P, tt, tp, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, tt, tp, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
        c[i] = compress_one<kAllSingle, true, true>(__fadd_rn(x1, x2), __fadd_rn(y1, y2),
                                                    __fadd_rn(z1, z2), P);
    }
}

// Words staged through shared memory by cp.async (LDGSTS), two stages: the
// next step's 64 bytes per thread are in flight while this step computes,
// with no registers held for them.  Stage layout chunk-major (16-byte chunk k
// of thread t at (k * T + t) * 16) so the copies and the LDS.128 reads are
// bank-conflict free.
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <bool EXACT, class LAY, int T, int MINB>
__global__ void __launch_bounds__(T, MINB)
    k_add_as_cp(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
                unsigned long long* __restrict__ c, int64_t n, Params Pin, bool vec,
                const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<true>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    const uint4* stage = reinterpret_cast<const uint4*>(s_tab + P.tab_n);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage) + threadIdx.x * 16u;
    auto issue = [&](int64_t gi, int st) {
        const uint32_t s0 = sbase + (uint32_t)(st * 4 * T * 16);
        const unsigned long long* pa = a + 4 * gi;
        const unsigned long long* pb = b + 4 * gi;
        if (gi < groups) {
            cp_async16(s0, pa);
            cp_async16(s0 + T * 16, pa + 2);
            cp_async16(s0 + 2 * T * 16, pb);
            cp_async16(s0 + 3 * T * 16, pb + 2);
        }
        cp_async_commit();  // (an empty group at the end keeps wait_group 1 uniform)
    };
    int64_t g = gtid();
    issue(g, 0);
    int st = 0;
    for (; g < groups; g += gstride(), st ^= 1) {
        issue(g + gstride(), st ^ 1);
        cp_async_wait1();  // this step's group (own slots only: no barrier needed)
        const uint4* q = stage + st * 4 * T + threadIdx.x;
        const uint4 q0 = q[0], q1 = q[T], q2 = q[2 * T], q3 = q[3 * T];
        const unsigned long long wa[4] = {((unsigned long long)q0.y << 32) | q0.x, ((unsigned long long)q0.w << 32) | q0.z,
                                          ((unsigned long long)q1.y << 32) | q1.x, ((unsigned long long)q1.w << 32) | q1.z};
        const unsigned long long wb[4] = {((unsigned long long)q2.y << 32) | q2.x, ((unsigned long long)q2.w << 32) | q2.z,
                                          ((unsigned long long)q3.y << 32) | q3.x, ((unsigned long long)q3.w << 32) | q3.z};
        float xa[4], ya[4], za[4], xb[4], yb[4], zb[4], x[4], y[4], z[4];
        decode4<EXACT>(wa, P, tt, tp, full, tol2, xa, ya, za);
        decode4<EXACT>(wb, P, tt, tp, full, tol2, xb, yb, zb);
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
    asm volatile("cp.async.wait_all;" ::: "memory");
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float x1, y1, z1, x2, y2, z2;
        const unsigned long long wa = a[i], wb = b[i];
        if (decode_fused<EXACT>(wa, P, tt, tp, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, tt, tp, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
        c[i] = compress_one<kAllSingle, true, true>(__fadd_rn(x1, x2), __fadd_rn(y1, y2),
                                                    __fadd_rn(z1, z2), P);
    }
}

// Two vectors per thread step (one compress pair): half the live state of
// k_add_as, 16-byte word accesses.
template <bool EXACT, class LAY, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_add_as2(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
              unsigned long long* __restrict__ c, int64_t n, Params Pin, bool vec,
              const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<true>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol2 = EXACT ? exact_tol<true>(full, P) : 0.0;
    const int64_t pairs = vec ? n / 2 : 0;
    for (int64_t g = gtid(); g < pairs; g += gstride()) {
        const ulonglong2 u = ld_stream_u2(a + 2 * g), v = ld_stream_u2(b + 2 * g);
        const unsigned long long w4[4] = {u.x, u.y, v.x, v.y};
        float xs[4], ys[4], zs[4], x[2], y[2], z[2];
        decode4<EXACT>(w4, P, tt, tp, full, tol2, xs, ys, zs);
        add_pairs(xs, xs + 2, x);
        add_pairs(ys, ys + 2, y);
        add_pairs(zs, zs + 2, z);
        unsigned long long w[2];
        bool slow[2];
        compress_as2(x, y, z, P, w, slow);
        if (__any_sync(__activemask(), slow[0] | slow[1])) {
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (slow[k]) w[k] = compress_one<kAllSingle, true, true>(x[k], y[k], z[k], P);
        }
        st_u2(c + 2 * g, w[0], w[1]);
    }
    for (int64_t i = pairs * 2 + gtid(); i < n; i += gstride()) {
        float x1, y1, z1, x2, y2, z2;
        const unsigned long long wa = a[i], wb = b[i];
        if (decode_fused<EXACT>(wa, P, tt, tp, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, tt, tp, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
        c[i] = compress_one<kAllSingle, true, true>(__fadd_rn(x1, x2), __fadd_rn(y1, y2),
                                                    __fadd_rn(z1, z2), P);
    }
}

// K4 axpy, all-single: y' = compress(alpha * decode(x) + decode(y)), the
// float32 product and sum rounded separately (scalar: a packed product may
// not feed a packed sum, vc3_fused.cuh).  y may alias y_out.
template <bool EXACT, class LAY>
__global__ void __launch_bounds__(kThreads, VC3_ADD_AS_MIN_BLOCKS)
    k_axpy_as(float al, const unsigned long long* __restrict__ xw, const unsigned long long* yw,
              unsigned long long* yo, int64_t n, Params Pin, bool vec,
              const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<true>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
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
        decode4<EXACT>(wa, P, tt, tp, full, tol2, xa, ya, za);
        decode4<EXACT>(wb, P, tt, tp, full, tol2, xb, yb, zb);
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
        if (decode_fused<EXACT>(wa, P, tt, tp, tol2, x1, y1, z1)) decode_redo(wa, P, full, x1, y1, z1);
        if (decode_fused<EXACT>(wb, P, tt, tp, tol2, x2, y2, z2)) decode_redo(wb, P, full, x2, y2, z2);
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

template <bool EXACT, class LAY>
__global__ void __launch_bounds__(kThreads, VC3_ADD_AS_MIN_BLOCKS)
    k_rk_as(float ca, float cb, float dt, unsigned long long* __restrict__ q,
            unsigned long long* __restrict__ dq, const unsigned long long* __restrict__ R, int64_t n,
            Params Pin, bool vec, const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<true>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
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
        decode4<EXACT>(wq, P, tt, tp, full, tol2, qx, qy, qz);
        decode4<EXACT>(wd, P, tt, tp, full, tol2, dx, dy, dz);
        decode4<EXACT>(wr, P, tt, tp, full, tol2, rx, ry, rz);
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
        if (decode_fused<EXACT>(wq, P, tt, tp, tol2, q0, q1, q2)) decode_redo(wq, P, full, q0, q1, q2);
        if (decode_fused<EXACT>(wd, P, tt, tp, tol2, d0, d1, d2)) decode_redo(wd, P, full, d0, d1, d2);
        if (decode_fused<EXACT>(wr, P, tt, tp, tol2, r0, r1, r2)) decode_redo(wr, P, full, r0, r1, r2);
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
#ifndef VC3_COMPRESS_PF
#define VC3_COMPRESS_PF 0
#endif
template <class LAY, int MINB = VC3_FUSED_MIN_BLOCKS, int PF = VC3_COMPRESS_PF>
__global__ void __launch_bounds__(kThreads, MINB)
    k_compress_as(const float* __restrict__ xyz, unsigned long long* __restrict__ out, int64_t n,
                  Params Pin, bool vec, int32_t* __restrict__ nonfinite) {
    Params P = Pin;
    LAY::apply(P);
    int bad = 0;
    const int64_t groups = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        if (PF) {  // L2 prefetch of the 48 bytes PF grid strides ahead
            const int64_t gp = g + PF * gstride();
            if (gp < groups) {
                prefetch_l2(xyz + 12 * gp);
                prefetch_l2(xyz + 12 * gp + 8);
            }
        }
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
// Launch the all-single fused add (table layouts).  Returns a vc3_status.
int launch_add(const unsigned long long* a, const unsigned long long* b, unsigned long long* c,
               int64_t n, const Params& P, bool def, bool exact, bool vec, const double2* tab,
               const double2* full, cudaStream_t s) {
    using Fn = void (*)(const unsigned long long*, const unsigned long long*, unsigned long long*,
                        int64_t, Params, bool, const double2*, const double2*);
    Fn fn;
    int threads = kThreads, per_sm = VC3_ADD_CTAS_PER_SM;
    size_t smem = table_smem(P);
    int v = 0;
#ifdef VC3_TUNE
    static const int tune = getenv("VC3_TUNE") ? atoi(getenv("VC3_TUNE")) : 0;
    v = tune;
#endif
    if (def && v == 7) {
        fn = exact ? k_add_as_cp<true, DefaultLayout, 512, 2> : k_add_as_cp<false, DefaultLayout, 512, 2>;
        threads = 512;
        per_sm = 2;
        smem += 2 * 4 * 512 * 16;
    } else if (def && v == 8) {
        fn = exact ? k_add_as_cp<true, DefaultLayout, 256, 3> : k_add_as_cp<false, DefaultLayout, 256, 3>;
        per_sm = 3;
        smem += 2 * 4 * 256 * 16;
    } else if (def && v == 9) {
        fn = exact ? k_add_as_cp<true, DefaultLayout, 512, 2> : k_add_as_cp<false, DefaultLayout, 512, 2>;
        threads = 512;
        per_sm = 24;
        smem += 2 * 4 * 512 * 16;
    } else if (def) {
        switch (v) {
            case 1: fn = exact ? k_add_as<true, DefaultLayout, 3> : k_add_as<false, DefaultLayout, 3>; break;
            case 2: fn = exact ? k_add_as<true, DefaultLayout, 3, 2> : k_add_as<false, DefaultLayout, 3, 2>; break;
            case 4: fn = exact ? k_add_as<true, DefaultLayout, 4, 2> : k_add_as<false, DefaultLayout, 4, 2>; break;
            case 5: fn = exact ? k_add_as<true, DefaultLayout, 2, 2> : k_add_as<false, DefaultLayout, 2, 2>; break;
            case 3: fn = exact ? k_add_as2<true, DefaultLayout, 4> : k_add_as2<false, DefaultLayout, 4>; break;
            case 10: fn = exact ? k_add_as<true, DefaultLayout, 3, 3> : k_add_as<false, DefaultLayout, 3, 3>; break;
            case 11: fn = exact ? k_add_as<true, DefaultLayout, 3, 4> : k_add_as<false, DefaultLayout, 3, 4>; break;
            default: fn = exact ? k_add_as<true, DefaultLayout> : k_add_as<false, DefaultLayout>;
        }
    } else {
        fn = exact ? k_add_as<true, RuntimeLayout> : k_add_as<false, RuntimeLayout>;
    }
    if (const int st = ensure_smem((const void*)fn, smem)) return st;
#ifdef VC3_TUNE
    static const int tune_grid = getenv("VC3_TUNE_GRID") ? atoi(getenv("VC3_TUNE_GRID")) : 0;
    if (tune_grid) per_sm = tune_grid;
#endif
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    fn<<<(unsigned)blocks, threads, smem, s>>>(a, b, c, n, P, vec, tab, full);
    return launch_status();
}

template <typename KFn, typename... Args>
int launch_table_kernel(KFn fn, const Params& P, int64_t n, bool vec, cudaStream_t s, Args... args) {
    const size_t smem = table_smem(P);
    if (const int st = ensure_smem((const void*)fn, smem)) return st;
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sm_count() * VC3_ADD_CTAS_PER_SM;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    fn<<<(unsigned)blocks, kThreads, smem, s>>>(args...);
    return launch_status();
}

int launch_axpy(float al, const unsigned long long* x, const unsigned long long* y,
                unsigned long long* yo, int64_t n, const Params& P, bool def, bool exact, bool vec,
                const double2* tab, const double2* full, cudaStream_t s) {
    auto fn = def ? (exact ? k_axpy_as<true, DefaultLayout> : k_axpy_as<false, DefaultLayout>)
                  : (exact ? k_axpy_as<true, RuntimeLayout> : k_axpy_as<false, RuntimeLayout>);
    return launch_table_kernel(fn, P, n, vec, s, al, x, y, yo, n, P, vec, tab, full);
}

int launch_rk(float ca, float cb, float dt, unsigned long long* q, unsigned long long* dq,
              const unsigned long long* R, int64_t n, const Params& P, bool def, bool exact,
              bool vec, const double2* tab, const double2* full, cudaStream_t s) {
    auto fn = def ? (exact ? k_rk_as<true, DefaultLayout> : k_rk_as<false, DefaultLayout>)
                  : (exact ? k_rk_as<true, RuntimeLayout> : k_rk_as<false, RuntimeLayout>);
    return launch_table_kernel(fn, P, n, vec, s, ca, cb, dt, q, dq, R, n, P, vec, tab, full);
}

// The all-single compress (layouts with t <= 25, p <= 24: clamp-free buckets).
int launch_compress(const float* xyz, unsigned long long* w, int64_t n, const Params& P, bool def,
                    bool vec, int32_t* nonfinite, cudaStream_t s) {
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sm_count() * VC3_COMPRESS_CTAS_PER_SM;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    int v = 0;
#ifdef VC3_TUNE
    static const int tune = getenv("VC3_TUNE_C") ? atoi(getenv("VC3_TUNE_C")) : 0;
    v = tune;
#endif
    if (def && v == 1)
        k_compress_as<DefaultLayout, 3><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else if (def && v == 2)
        k_compress_as<DefaultLayout, 4, 1><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else if (def && v == 3)
        k_compress_as<DefaultLayout, 3, 1><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else if (def && v == 4)
        k_compress_as<DefaultLayout, 4, 2><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else if (def)
        k_compress_as<DefaultLayout><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    else
        k_compress_as<RuntimeLayout><<<(unsigned)blocks, kThreads, 0, s>>>(xyz, w, n, P, vec, nonfinite);
    return launch_status();
}
}  // namespace as
}  // namespace vc3
