// vc3_fused.cu — the fused streaming operations on compressed words:
// c = a + b (K3, the headline), y = alpha*x + y (K4 axpy) and the low-storage
// RK stage (K4b), each decode -> float32 op -> encode in one pass so nothing
// uncompressed touches HBM.
//
// Two numerics modes, selected per call (include/vc3_b200.h):
//   VC3_EXACT    every decode is bit-identical to the reference's (boundary
//                components redone from its own tables), so output words are
//                the reference's;
//   VC3_CONTRACT the fast table decode without that test (a component may be
//                one ulp off, a word may move one bin at a tie).
// Two code paths:
//   * all-single policy on a table layout (the reference benchmark's
//     configuration, bench.py:41-69): the restructured path of vc3_fused.cuh
//     (packed float32 pairs, range-tested fast divides / square roots);
//   * every other policy / layout: the generic per-vector routines of
//     vc3_device.cuh.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"
#include "vc3_kern_common.cuh"
#include "vc3_rt.h"

// the all-single kernels live in vc3_fused_as.cu
namespace vc3 {
namespace as {
int launch_add(const unsigned long long* a, const unsigned long long* b, unsigned long long* c,
               int64_t n, const Params& P, bool def, bool exact, bool vec, const double2* tab,
               const double2* full, cudaStream_t s);
int launch_axpy(float al, const unsigned long long* x, const unsigned long long* y,
                unsigned long long* yo, int64_t n, const Params& P, bool def, bool exact, bool vec,
                const double2* tab, const double2* full, cudaStream_t s);
int launch_rk(float ca, float cb, float dt, unsigned long long* q, unsigned long long* dq,
              const unsigned long long* R, int64_t n, const Params& P, bool def, bool exact,
              bool vec, const double2* tab, const double2* full, cudaStream_t s);
}  // namespace as
}  // namespace vc3

#ifndef VC3_USE_FMA
#define VC3_USE_FMA 1
#endif

namespace {

constexpr bool kFmaF = VC3_USE_FMA != 0;
constexpr unsigned kAllSingle = 7u;

// ===================== generic path (any policy, any layout) ==================
// A zero field may decode to signed zeros (SIGNED_ZERO_OK) only when the
// re-compress maps every +-0 pattern alike: the float32 atan2 of the
// theta-single policies does; libm's double atan2 (theta-double) does not.
template <unsigned POLICY>
constexpr bool kSignedZeroOk = (POLICY & kThetaSingle) != 0;

// K3 fused add: c = compress(decompress(a) + decompress(b)) (_kernels.py:348-359)
template <unsigned POLICY, bool TABLE, bool EXACT>
__device__ __forceinline__ unsigned long long add_one(unsigned long long a, unsigned long long b,
                                                      const Params& P, const double2* tt,
                                                      const double2* tp, const double2* full,
                                                      double tol) {
    float x1, y1, z1, x2, y2, z2;
    decompress_one<TABLE, kSignedZeroOk<POLICY>, EXACT>(a, P, tt, tp, x1, y1, z1, full, tol);
    decompress_one<TABLE, kSignedZeroOk<POLICY>, EXACT>(b, P, tt, tp, x2, y2, z2, full, tol);
    return compress_one<POLICY, kFmaF, TABLE>(__fadd_rn(x1, x2), __fadd_rn(y1, y2),
                                              __fadd_rn(z1, z2), P);
}

template <unsigned POLICY, bool TABLE, class LAY, bool EXACT>
__global__ void __launch_bounds__(kThreads, VC3_FUSED_MIN_BLOCKS)
    k_add(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
          unsigned long long* __restrict__ c, int64_t n, Params Pin, bool vec,
          const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<TABLE>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol = EXACT ? exact_tol<VC3_CELL_CHECK>(full, P) : 0.0;
    // four independent vectors per thread step give the scheduler ILP across
    // the long FP64 chains; words move with sm_100 256-bit accesses
    constexpr int kV = 4;
    const int64_t groups = vec ? n / kV : 0;
    for (int64_t g = gtid(); g < groups; g += gstride()) {
        const u64x4 u = ld_stream_u4(a + kV * g), v = ld_stream_u4(b + kV * g);
        const unsigned long long c0 = add_one<POLICY, TABLE, EXACT>(u.x, v.x, P, tt, tp, full, tol);
        const unsigned long long c1 = add_one<POLICY, TABLE, EXACT>(u.y, v.y, P, tt, tp, full, tol);
        const unsigned long long c2 = add_one<POLICY, TABLE, EXACT>(u.z, v.z, P, tt, tp, full, tol);
        const unsigned long long c3 = add_one<POLICY, TABLE, EXACT>(u.w, v.w, P, tt, tp, full, tol);
        st_u4(c + kV * g, c0, c1, c2, c3);
    }
    for (int64_t i = groups * kV + gtid(); i < n; i += gstride())
        c[i] = add_one<POLICY, TABLE, EXACT>(a[i], b[i], P, tt, tp, full, tol);
}

// K4 axpy: y' = compress(alpha*decode(x) + decode(y))
template <unsigned POLICY, bool TABLE, bool EXACT>
__device__ __forceinline__ unsigned long long axpy_one(float al, unsigned long long x,
                                                       unsigned long long y, const Params& P,
                                                       const double2* tt, const double2* tp,
                                                       const double2* full, double tol) {
    float x1, y1, z1, x2, y2, z2;
    decompress_one<TABLE, kSignedZeroOk<POLICY>, EXACT>(x, P, tt, tp, x1, y1, z1, full, tol);
    decompress_one<TABLE, kSignedZeroOk<POLICY>, EXACT>(y, P, tt, tp, x2, y2, z2, full, tol);
    return compress_one<POLICY, kFmaF, TABLE>(__fadd_rn(__fmul_rn(al, x1), x2),
                                              __fadd_rn(__fmul_rn(al, y1), y2),
                                              __fadd_rn(__fmul_rn(al, z1), z2), P);
}

template <unsigned POLICY, bool TABLE, class LAY, bool EXACT>
__global__ void __launch_bounds__(kThreads, VC3_FUSED_MIN_BLOCKS)
    k_axpy(float al, const unsigned long long* __restrict__ x, const unsigned long long* y,
           unsigned long long* yo, int64_t n, Params Pin, bool vec,
           const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<TABLE>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol = EXACT ? exact_tol<VC3_CELL_CHECK>(full, P) : 0.0;
    const int64_t pairs = vec ? n / 2 : 0;
    for (int64_t g = gtid(); g < pairs; g += gstride()) {
        const ulonglong2 u = ld_stream_u2(x + 2 * g);
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(y + 2 * g);  // may alias yo
        st_u2(yo + 2 * g, axpy_one<POLICY, TABLE, EXACT>(al, u.x, v.x, P, tt, tp, full, tol),
              axpy_one<POLICY, TABLE, EXACT>(al, u.y, v.y, P, tt, tp, full, tol));
    }
    for (int64_t i = pairs * 2 + gtid(); i < n; i += gstride())
        yo[i] = axpy_one<POLICY, TABLE, EXACT>(al, x[i], y[i], P, tt, tp, full, tol);
}

// K4b low-storage RK stage: dq' = a*dq + dt*R ; q' = q + b*dq'
template <unsigned POLICY, bool TABLE, bool EXACT>
__device__ __forceinline__ void rk_one(float ca, float cb, float dt, unsigned long long& q,
                                       unsigned long long& dq, unsigned long long r,
                                       const Params& P, const double2* tt, const double2* tp,
                                       const double2* full, double tol) {
    float q0, q1, q2, d0, d1, d2, r0, r1, r2;
    constexpr bool SZ = kSignedZeroOk<POLICY>;
    decompress_one<TABLE, SZ, EXACT, VC3_RK_CELL>(q, P, tt, tp, q0, q1, q2, full, tol);
    decompress_one<TABLE, SZ, EXACT, VC3_RK_CELL>(dq, P, tt, tp, d0, d1, d2, full, tol);
    decompress_one<TABLE, SZ, EXACT, VC3_RK_CELL>(r, P, tt, tp, r0, r1, r2, full, tol);
    d0 = __fadd_rn(__fmul_rn(ca, d0), __fmul_rn(dt, r0));
    d1 = __fadd_rn(__fmul_rn(ca, d1), __fmul_rn(dt, r1));
    d2 = __fadd_rn(__fmul_rn(ca, d2), __fmul_rn(dt, r2));
    q0 = __fadd_rn(q0, __fmul_rn(cb, d0));
    q1 = __fadd_rn(q1, __fmul_rn(cb, d1));
    q2 = __fadd_rn(q2, __fmul_rn(cb, d2));
    dq = compress_one<POLICY, kFmaF, TABLE>(d0, d1, d2, P);
    q = compress_one<POLICY, kFmaF, TABLE>(q0, q1, q2, P);
}

template <unsigned POLICY, bool TABLE, class LAY, bool EXACT>
__global__ void __launch_bounds__(kThreads, VC3_FUSED_MIN_BLOCKS)
    k_rk(float ca, float cb, float dt, unsigned long long* __restrict__ q,
         unsigned long long* __restrict__ dq, const unsigned long long* __restrict__ R, int64_t n,
         Params Pin, bool vec, const double2* __restrict__ gtab, const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    load_table<TABLE>(s_tab, gtab, P);
    const double2* tt = s_tab;
    const double2* tp = s_tab + P.p_base;
    const double tol = EXACT ? exact_tol<VC3_RK_CELL>(full, P) : 0.0;
    const int64_t pairs = vec ? n / 2 : 0;
    for (int64_t g = gtid(); g < pairs; g += gstride()) {
        ulonglong2 u = *reinterpret_cast<const ulonglong2*>(q + 2 * g);
        ulonglong2 v = *reinterpret_cast<const ulonglong2*>(dq + 2 * g);
        const ulonglong2 r = ld_stream_u2(R + 2 * g);
        rk_one<POLICY, TABLE, EXACT>(ca, cb, dt, u.x, v.x, r.x, P, tt, tp, full, tol);
        rk_one<POLICY, TABLE, EXACT>(ca, cb, dt, u.y, v.y, r.y, P, tt, tp, full, tol);
        st_u2(q + 2 * g, u.x, u.y);
        st_u2(dq + 2 * g, v.x, v.y);
    }
    for (int64_t i = pairs * 2 + gtid(); i < n; i += gstride()) {
        unsigned long long qq = q[i], dd = dq[i];
        rk_one<POLICY, TABLE, EXACT>(ca, cb, dt, qq, dd, R[i], P, tt, tp, full, tol);
        q[i] = qq;
        dq[i] = dd;
    }
}

// ===================== dispatch ================================================
int full_table_for(const Params& P, bool exact, const double2** full) {
    *full = nullptr;
    return (exact && P.table_mode) ? get_full_table(P, full) : VC3_OK;
}

// one kernel pointer per (policy, layout class, mode); the caller launches it
template <unsigned POL>
struct AddKernel {
    using Fn = void (*)(const unsigned long long*, const unsigned long long*, unsigned long long*,
                        int64_t, Params, bool, const double2*, const double2*);
    static Fn pick(const Params& P, bool def, bool exact) {
        if (!P.table_mode) return k_add<POL, false, RuntimeLayout, true>;
        if constexpr (POL == kAllSingle) {
            return nullptr;  // table layouts: vc3::as::launch_add (vc3_fused_as.cu)
        } else {
            if (def) return exact ? k_add<POL, true, DefaultLayout, true> : k_add<POL, true, DefaultLayout, false>;
            return exact ? k_add<POL, true, RuntimeLayout, true> : k_add<POL, true, RuntimeLayout, false>;
        }
    }
};

template <unsigned POL>
struct RunAdd {
    static int run(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n, const Params& P,
                   bool def, bool exact, const double2* tab, cudaStream_t s) {
        const bool vec = aligned32(a) && aligned32(b) && aligned32(c);
        const unsigned grid = grid_for(vec ? (n + 3) / 4 : n, VC3_ADD_CTAS_PER_SM);
        const double2* full = nullptr;
        if (const int st = full_table_for(P, exact, &full)) return st;
        if (POL == kAllSingle && P.table_mode)
            return vc3::as::launch_add((const unsigned long long*)a, (const unsigned long long*)b,
                                       (unsigned long long*)c, n, P, def, exact, vec, tab, full, s);
        const auto fn = AddKernel<POL>::pick(P, def, exact);
        const size_t smem = table_smem(P);
        if (const int st = ensure_smem((const void*)fn, smem)) return st;
        fn<<<grid, kThreads, smem, s>>>((const unsigned long long*)a, (const unsigned long long*)b,
                                        (unsigned long long*)c, n, P, vec, tab, full);
        return launch_status();
    }
};

template <unsigned POL>
struct RunAxpy {
    static int run(float al, const uint64_t* x, const uint64_t* y, uint64_t* yo, int64_t n,
                   const Params& P, bool def, bool exact, const double2* tab, cudaStream_t s) {
        auto X = (const unsigned long long*)x, Y = (const unsigned long long*)y;
        auto O = (unsigned long long*)yo;
        const double2* full = nullptr;
        if (const int st = full_table_for(P, exact, &full)) return st;
        if (POL == kAllSingle && P.table_mode)
            return vc3::as::launch_axpy(al, X, Y, O, n, P, def, exact,
                                        aligned32(x) && aligned32(y) && aligned32(yo), tab, full, s);
        const bool vec = aligned16(x) && aligned16(y) && aligned16(yo);
        const unsigned grid = grid_for(vec ? (n + 1) / 2 : n, VC3_ADD_CTAS_PER_SM);
        using Fn = void (*)(float, const unsigned long long*, const unsigned long long*,
                            unsigned long long*, int64_t, Params, bool, const double2*, const double2*);
        Fn fn;
        if constexpr (POL == kAllSingle) {
            fn = k_axpy<POL, false, RuntimeLayout, true>;  // wide layouts only (tables: vc3_fused_as.cu)
        } else {
            if (!P.table_mode) fn = k_axpy<POL, false, RuntimeLayout, true>;
            else if (def) fn = exact ? k_axpy<POL, true, DefaultLayout, true> : k_axpy<POL, true, DefaultLayout, false>;
            else fn = exact ? k_axpy<POL, true, RuntimeLayout, true> : k_axpy<POL, true, RuntimeLayout, false>;
        }
        const size_t smem = table_smem(P);
        if (const int st = ensure_smem((const void*)fn, smem)) return st;
        fn<<<grid, kThreads, smem, s>>>(al, X, Y, O, n, P, vec, tab, full);
        return launch_status();
    }
};

template <unsigned POL>
struct RunRk {
    static int run(float ca, float cb, float dt, uint64_t* q, uint64_t* dq, const uint64_t* R,
                   int64_t n, const Params& P, bool def, bool exact, const double2* tab,
                   cudaStream_t s) {
        auto Q = (unsigned long long*)q, D = (unsigned long long*)dq;
        auto RR = (const unsigned long long*)R;
        const double2* full = nullptr;
        if (const int st = full_table_for(P, exact, &full)) return st;
        if (POL == kAllSingle && P.table_mode)
            return vc3::as::launch_rk(ca, cb, dt, Q, D, RR, n, P, def, exact,
                                      aligned32(q) && aligned32(dq) && aligned32(R), tab, full, s);
        const bool vec = aligned16(q) && aligned16(dq) && aligned16(R);
        const unsigned grid = grid_for(vec ? (n + 1) / 2 : n, VC3_ADD_CTAS_PER_SM);
        using Fn = void (*)(float, float, float, unsigned long long*, unsigned long long*,
                            const unsigned long long*, int64_t, Params, bool, const double2*,
                            const double2*);
        Fn fn;
        if constexpr (POL == kAllSingle) {
            fn = k_rk<POL, false, RuntimeLayout, true>;  // wide layouts only (tables: vc3_fused_as.cu)
        } else {
            if (!P.table_mode) fn = k_rk<POL, false, RuntimeLayout, true>;
            else if (def) fn = exact ? k_rk<POL, true, DefaultLayout, true> : k_rk<POL, true, DefaultLayout, false>;
            else fn = exact ? k_rk<POL, true, RuntimeLayout, true> : k_rk<POL, true, RuntimeLayout, false>;
        }
        const size_t smem = table_smem(P);
        if (const int st = ensure_smem((const void*)fn, smem)) return st;
        fn<<<grid, kThreads, smem, s>>>(ca, cb, dt, Q, D, RR, n, P, vec, tab, full);
        return launch_status();
    }
};

}  // namespace

// ===================== extern "C" boundary ====================================
extern "C" {

int vc3_add_compressed_ex(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n,
                          vc3_layout layout, uint32_t policy, uint32_t flags, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u || (flags & ~VC3_FLAGS_ALL)) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!a || !b || !c) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    const double2* tab = nullptr;
    if (const int st = get_table(P, &tab)) return st;
    return by_policy<RunAdd>(policy, a, b, c, n, P, is_default_layout(layout),
                             !(flags & VC3_CONTRACT), tab, (cudaStream_t)stream);
}

int vc3_add_compressed(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n,
                       vc3_layout layout, uint32_t policy, void* stream) {
    return vc3_add_compressed_ex(a, b, c, n, layout, policy, VC3_EXACT, stream);
}

int vc3_axpy_ex(float alpha, const uint64_t* x, const uint64_t* y, uint64_t* y_out, int64_t n,
                vc3_layout layout, uint32_t policy, uint32_t flags, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u || (flags & ~VC3_FLAGS_ALL)) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!x || !y || !y_out) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    const double2* tab = nullptr;
    if (const int st = get_table(P, &tab)) return st;
    return by_policy<RunAxpy>(policy, alpha, x, y, y_out, n, P, is_default_layout(layout),
                              !(flags & VC3_CONTRACT), tab, (cudaStream_t)stream);
}

int vc3_axpy(float alpha, const uint64_t* x, const uint64_t* y, uint64_t* y_out, int64_t n,
             vc3_layout layout, uint32_t policy, void* stream) {
    return vc3_axpy_ex(alpha, x, y, y_out, n, layout, policy, VC3_EXACT, stream);
}

int vc3_rk_stage_ex(float a, float b, float dt, uint64_t* q, uint64_t* dq, const uint64_t* R,
                    int64_t n, vc3_layout layout, uint32_t policy, uint32_t flags, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u || (flags & ~VC3_FLAGS_ALL)) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!q || !dq || !R) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    const double2* tab = nullptr;
    if (const int st = get_table(P, &tab)) return st;
    return by_policy<RunRk>(policy, a, b, dt, q, dq, R, n, P, is_default_layout(layout),
                            !(flags & VC3_CONTRACT), tab, (cudaStream_t)stream);
}

int vc3_rk_stage(float a, float b, float dt, uint64_t* q, uint64_t* dq, const uint64_t* R,
                 int64_t n, vc3_layout layout, uint32_t policy, void* stream) {
    return vc3_rk_stage_ex(a, b, dt, q, dq, R, n, layout, policy, VC3_EXACT, stream);
}

}  // extern "C"
