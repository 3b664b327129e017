// vc3_kernels.cu — sm_100a kernels of the inline 3-vector codec and the
// extern "C" boundary declared in include/vc3_b200.h.
//
// Memory layout in HBM: compressed words are contiguous uint64
// arrays moved as 32-byte groups of four (sm_100 256-bit LDG/STG; 16-byte
// pairs in the axpy / RK kernels); vectors are the caller's array-of-structs
// float32 [n][3] moved as three 16-byte float4 per group of four vectors.
// Every kernel is a grid-stride streaming loop over a grid sized to a
// multiple of the SM count; nothing uncompressed touches HBM in the fused
// operations.  Decoding kernels first copy the layout's sin/cos table (49 KB
// at the default layout, opt-in shared memory) from global memory into
// shared memory.
#include <cuda_runtime.h>
#include <cstdlib>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"
#include "vc3_rt.h"

using namespace vc3;

#ifndef VC3_USE_FMA
// Fused Horner / bucket FMAs: enabled after tools/exhaustive.cu proved them
// bit-identical to the reference's unfused sequence over every float32 input.
#define VC3_USE_FMA 1
#endif
constexpr bool kFma = VC3_USE_FMA != 0;

// Host runtime shared with the other translation units (vc3_rt.h).
namespace vc3 {
namespace rt {

thread_local int g_last_cuda = 0;

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return VC3_OK;
    g_last_cuda = (int)e;
    return VC3_ERR_CUDA;
}

int launch_status() { return cuda_status(cudaGetLastError()); }

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int sm_count() {
    static std::mutex mu;
    static std::map<int, int> counts;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    auto it = counts.find(dev);
    if (it != counts.end()) return it->second;
    int count = 0;
    if (cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || count <= 0)
        count = 148;
    counts[dev] = count;
    return count;
}

bool layout_ok(const vc3_layout& L) {
    const int s = L.sign_bits, e = L.exponent_bits, m = L.mantissa_bits, p = L.phi_bits,
              t = L.theta_bits;
    if (s != 0 && s != 1) return false;
    if (e < 1 || e > 8 || m < 1 || m > 23 || p < 1 || p > 32 || t < 1 || t > 32) return false;
    if (s + e + m + p + t != 64) return false;
    if (e == 8 && L.exponent_bias != 127) return false;
    if (L.exponent_bias < 0 || L.exponent_bias > 128) return false;
    return true;
}

// Host derivation of the by-value parameter block.  The double expressions
// of the bucket arithmetic are the reference's (_kernels.py:139-140)
// evaluated in IEEE double; the doubled forms are exact scalings of them.
Params make_params(const vc3_layout& L) {
    Params P{};
    P.e = L.exponent_bits;
    P.m = L.mantissa_bits;
    P.p = L.phi_bits;
    P.t = L.theta_bits;
    P.bias = L.exponent_bias;
    derive_int_fields(P);
    const volatile double pi = kPi;  // keep host arithmetic plain IEEE double
    P.nt_half = (double)P.ntmax / 2.0;
    P.t_scale = (double)P.ntmax / (2.0 * pi);
    P.p_scale = (double)P.npmax / pi;
    P.nt_half2 = 2.0 * P.nt_half;
    P.t_scale2 = 2.0 * P.t_scale;
    P.p_scale2 = 2.0 * P.p_scale;
    const long double pid = (long double)kPi;
    P.t_delta = (double)(2.0L * pid / (long double)P.ntmax);
    P.p_delta = (double)(pid / (long double)P.npmax);
    P.t_rcp = 1.0 / (double)P.ntmax;
    P.p_rcp = 1.0 / (double)P.npmax;
    P.resid_hi = 0x43300000u;
    return P;
}

bool is_default_layout(const vc3_layout& L) {
    return L.sign_bits == 0 && L.exponent_bits == 7 && L.mantissa_bits == 22 && L.phi_bits == 17 &&
           L.theta_bits == 18 && L.exponent_bias == 80;
}

// sin/cos(RN(pi) * k / b) to double accuracy: exact quarter-turn reduction,
// then long double libm.  Entries near a zero crossing keep full relative
// accuracy because pi - RN(pi) enters separately.
void sincos_host(long long k, long long b, double* s, double* c) {
    const long double pid = (long double)kPi;
    const long double tail = 1.2246467991473531772e-16L;  // pi - RN(pi)
    const long long ak = k < 0 ? -k : k;
    long long j = (4 * ak + b) / (2 * b);
    if (k < 0) j = -j;
    const long long m = 2 * k - j * b;
    const long double psi = pid * (long double)m / (2.0L * (long double)b) - (long double)j * tail / 2.0L;
    const long double sp = sinl(psi), cp = cosl(psi);
    long double ss, cc;
    switch (((j % 4) + 4) % 4) {
        case 0: ss = sp; cc = cp; break;
        case 1: ss = cp; cc = -sp; break;
        case 2: ss = -sp; cc = -cp; break;
        default: ss = -cp; cc = sp; break;
    }
    *s = (double)ss;
    *c = (double)cc;
}

// Device-resident decode tables, built once per (device, t, p) and kept.
struct TableKey {
    int dev, t, p;
    bool operator<(const TableKey& o) const {
        return dev != o.dev ? dev < o.dev : (t != o.t ? t < o.t : p < o.p);
    }
};
std::mutex g_tab_mu;
std::map<TableKey, double2*> g_tabs;

// Upload a host table into fresh device memory, safe on first use inside a
// caller's CUDA-graph capture and independent of the caller's stream: the
// thread switches to relaxed capture mode for the allocation, and the copy
// runs on a library-private non-blocking stream that is synchronised before
// returning (so no later kernel on any stream can see the memory early).
int upload_table(const void* h, size_t bytes, double2** out) {
    *out = nullptr;
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    static std::mutex smu;
    static std::map<int, cudaStream_t> streams;
    cudaStream_t s = nullptr;
    int st = VC3_OK;
    {
        std::lock_guard<std::mutex> lock(smu);
        const int dev = current_device();
        auto it = streams.find(dev);
        if (it == streams.end()) {
            st = cuda_status(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            if (!st) streams[dev] = s;
        } else {
            s = it->second;
        }
    }
    double2* d = nullptr;
    if (!st) st = cuda_status(cudaMalloc((void**)&d, bytes));
    if (!st) st = cuda_status(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    if (!st) st = cuda_status(cudaStreamSynchronize(s));
    if (st && d) cudaFree(d);
    cudaThreadExchangeStreamCaptureMode(&mode);  // restore the caller's mode
    if (!st) *out = d;
    return st;
}

// layout of the fast table: [theta grid (t_n - 1)][theta endpoint nt = ntmax]
// [phi grid (p_n - 1)][phi pole]
std::vector<double2> fast_table_host(const Params& P) {
    std::vector<double2> h((size_t)P.tab_n);
    for (int i = 0; i < P.t_n - 1; ++i) {
        double s, c;
        sincos_host(2 * ((long long)i << P.t_shift) - P.ntmax, P.ntmax, &s, &c);
        h[i] = make_double2(s, c);
    }
    h[P.t_n - 1] = make_double2(kPiTail, -1.0);  // nt = ntmax: sin(+RN(pi)), cos(+RN(pi))
    for (int i = 0; i < P.p_n - 1; ++i) {
        double s, c;
        sincos_host((long long)i << P.p_shift, P.npmax, &s, &c);
        h[P.p_base + i] = make_double2(s, c);
    }
    h[P.p_base + P.p_n - 1] = make_double2(0.0, -1.0);  // nph = npmax: the reference's exact pole
    // residual sections: (sin(l * D), cos(l * D) - 1) for every residual index
    // l, D = 2 RN(pi) / ntmax (theta) or RN(pi) / npmax (phi), in long double
    const long double pid = (long double)kPi;
    for (int l = 0; l < (1 << P.t_shift); ++l) {
        const long double psi = (long double)l * (2.0L * pid / (long double)P.ntmax);
        h[P.rt_base + l] = make_double2((double)sinl(psi), (double)(-2.0L * sinl(psi / 2) * sinl(psi / 2)));
    }
    for (int l = 0; l < (1 << P.p_shift); ++l) {
        const long double psi = (long double)l * (pid / (long double)P.npmax);
        h[P.rp_base + l] = make_double2((double)sinl(psi), (double)(-2.0L * sinl(psi / 2) * sinl(psi / 2)));
    }
    return h;
}

int get_table(const Params& P, const double2** out) {
    *out = nullptr;
    if (!P.table_mode) return VC3_OK;
    const TableKey key{current_device(), P.t, P.p};
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto it = g_tabs.find(key);
    if (it != g_tabs.end()) {
        *out = it->second;
        return VC3_OK;
    }
    const std::vector<double2> h = fast_table_host(P);
    double2* d = nullptr;
    if (const int st = upload_table(h.data(), h.size() * sizeof(double2), &d)) return st;
    g_tabs[key] = d;
    *out = d;
    return VC3_OK;
}

// The reference's own decode tables (_kernels.py:252-273): glibc sin/cos of
// th = _PI*(2n/ntmax - 1) and ph = _PI*n/npmax, exact pole; 6 MB at the
// default layout, device-resident, read only for the rare boundary cases of
// the bit-identical decodes.
std::map<TableKey, double2*> g_full;
std::map<TableKey, double> g_tol;

// The device's table + residual evaluation (sincos_resid, vc3_device.cuh)
// restated on the host: every step is one IEEE double operation (std::fma is
// correctly rounded; the host build has no FMA contraction), so the results
// are the device's bit for bit.
void sincos_resid_host(double2 A, int lo, double delta, double* s, double* c) {
    const double psi = std::fma((double)(4503599627370496LL + lo), delta, -4503599627370496.0 * delta);
    const volatile double u = psi * psi;
    const volatile double pu = psi * u;
    const double sps = std::fma(pu, -1.0 / 6.0, psi);
    const volatile double cq = std::fma(u, 1.0 / 24.0, -0.5);
    const volatile double cm1 = u * cq;
    *s = std::fma(A.y, sps, std::fma(A.x, cm1, A.x));
    *c = std::fma(-A.x, sps, std::fma(A.y, cm1, A.y));
}

// The two-level form (decode_fused, vc3_fused.cuh): the residual's
// (sin psi, cos psi - 1) come from the residual table section.
void sincos_two_level_host(double2 A, double2 Rs, double* s, double* c) {
    *s = std::fma(A.y, Rs.x, std::fma(A.x, Rs.y, A.x));
    *c = std::fma(-A.x, Rs.x, std::fma(A.y, Rs.y, A.y));
}

// Decode tolerance (relative to r): a decoded component fl(fl(r*c')*s') vs
// the reference's fl(fl(r*c)*s) with |c - c'| <= et, |s - s'| <= ep differs
// by at most r*(et + ep + et*ep + 4u(1 + et)(1 + ep)), u = 2^-53; the
// boundary test's own d +- e roundings move its ends by <= r*2^-53 more.
double decode_tolerance(double et, double ep) { return (et + ep) * (1.0 + 0x1p-20) + 0x1p-49; }

int get_full_table(const Params& P, const double2** out) {
    *out = nullptr;
    if (!P.table_mode) return VC3_OK;
    const double2* seed = nullptr;
    if (const int st0 = get_table(P, &seed)) return st0;
    const TableKey key{current_device(), P.t, P.p};
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto it = g_full.find(key);
    if (it != g_full.end()) {
        *out = it->second;
        return VC3_OK;
    }
    // [theta: ntmax + 1][phi: npmax + 1][tolerance]
    std::vector<double2> h((size_t)(P.ntmax + 1 + P.npmax + 1 + 1));
    const volatile double pi = kPi;
    for (long long n = 0; n <= P.ntmax; ++n) {
        const double th = pi * (2.0 * (double)n / (double)P.ntmax - 1.0);
        h[(size_t)n] = make_double2(std::sin(th), std::cos(th));
    }
    for (long long n = 0; n <= P.npmax; ++n) {
        const double ph = pi * (double)n / (double)P.npmax;
        h[(size_t)(P.ntmax + 1 + n)] = make_double2(std::sin(ph), std::cos(ph));
    }
    h[(size_t)(P.ntmax + 1 + P.npmax)] = make_double2(0.0, -1.0);
    // largest |fast table sin/cos - reference sin/cos| over every theta index
    // (et) and every phi index (ep), indexed as the decodes index the table
    const std::vector<double2> fast = fast_table_host(P);
    double et = 0.0, ep = 0.0;
    // both decode forms share the tolerance: the residual polynomial
    // (decompress_one) and the two-level table (decode_fused)
    for (long long nt = 0; nt <= P.ntmax; ++nt) {
        const long long b = nt + (nt == P.ntmax ? 1 : 0);
        const int lo = (int)(b & ((1 << P.t_shift) - 1));
        const double2 A = fast[(size_t)(b >> P.t_shift)], Rf = h[(size_t)nt];
        double s, c, s2, c2;
        sincos_resid_host(A, lo, P.t_delta, &s, &c);
        sincos_two_level_host(A, fast[(size_t)(P.rt_base + lo)], &s2, &c2);
        et = std::fmax(et, std::fmax(std::fmax(std::fabs(s - Rf.x), std::fabs(c - Rf.y)),
                                     std::fmax(std::fabs(s2 - Rf.x), std::fabs(c2 - Rf.y))));
    }
    for (long long nph = 0; nph <= P.npmax; ++nph) {
        const long long b = nph + (nph == P.npmax ? 1 : 0);
        const int lo = (int)(b & ((1 << P.p_shift) - 1));
        const double2 A = fast[(size_t)(P.p_base + (b >> P.p_shift))];
        const double2 R = h[(size_t)(P.ntmax + 1 + nph)];
        double s, c, s2, c2;
        sincos_resid_host(A, lo, P.p_delta, &s, &c);
        sincos_two_level_host(A, fast[(size_t)(P.rp_base + lo)], &s2, &c2);
        ep = std::fmax(ep, std::fmax(std::fmax(std::fabs(s - R.x), std::fabs(c - R.y)),
                                     std::fmax(std::fabs(s2 - R.x), std::fabs(c2 - R.y))));
    }
    const double tol = decode_tolerance(et, ep);
    h.back() = make_double2(tol, 0.0);
    double2* d = nullptr;
    if (const int st = upload_table(h.data(), h.size() * sizeof(double2), &d)) return st;
    g_full[key] = d;
    g_tol[key] = tol;
    *out = d;
    return VC3_OK;
}

double full_table_tolerance(const Params& P) {
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto it = g_tol.find(TableKey{current_device(), P.t, P.p});
    return it == g_tol.end() ? 0.0 : it->second;
}

size_t table_smem(const Params& P) { return P.table_mode ? (size_t)P.tab_n * sizeof(double2) : 0; }

// Opt a kernel into more than 48 KB of dynamic shared memory (the default
// layout's table is 49 KB), once per (device, kernel).
int ensure_smem(const void* func, size_t bytes) {
    if (bytes <= 48 * 1024) return VC3_OK;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    const auto key = std::make_pair(current_device(), func);
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return VC3_OK;
    int st = cuda_status(
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    // all of the unified L1 as shared memory: several table copies per SM
    // (the streams bypass L1: ld.global.nc.L1::no_allocate)
    if (st == VC3_OK)
        st = cuda_status(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (st == VC3_OK) done[key] = bytes;
    return st;
}

}  // namespace rt
}  // namespace vc3

#include "vc3_fused.cuh"
#include "vc3_kern_common.cuh"

namespace {

// ===================== kernels ==============================================

// K1 compress: 4 vectors (48 B in, 32 B out) per thread per step.
// EV: also count the magnitude events (K8, codec.py:241-262) in the same pass.
template <unsigned POLICY, bool NARROW, class LAY, bool EV = false>
__global__ void __launch_bounds__(kThreads, VC3_FUSED_MIN_BLOCKS) k_compress(const float* __restrict__ xyz,
                                                       unsigned long long* __restrict__ out,
                                                       int64_t n, Params Pin, bool vec,
                                                       int32_t* __restrict__ nonfinite,
                                                       unsigned long long* __restrict__ events = nullptr) {
    Params P = Pin;
    LAY::apply(P);
    int bad = 0;
    unsigned ev[2] = {0u, 0u};
    const int64_t groups = vec ? n / 4 : 0;
    // (shared-memory staging of this input was measured slower: the kernel
    // is issue-bound, so the 16-byte strided loads stay; the next step's
    // loads are issued before this step's compute)
    int64_t g = gtid();
    float4 an = make_float4(0, 0, 0, 0), bn = an, cn = an;
    if (g < groups) {
        an = ld_stream_f4(xyz + 12 * g); bn = ld_stream_f4(xyz + 12 * g + 4); cn = ld_stream_f4(xyz + 12 * g + 8);
    }
    for (; g < groups; g += gstride()) {
        const float4 a = an, b = bn, c = cn;
        const int64_t gn = g + gstride();
        if (gn < groups) {
            an = ld_stream_f4(xyz + 12 * gn); bn = ld_stream_f4(xyz + 12 * gn + 4); cn = ld_stream_f4(xyz + 12 * gn + 8);
        }
        bad += !finite3(a.x, a.y, a.z) + !finite3(a.w, b.x, b.y) + !finite3(b.z, b.w, c.x) +
               !finite3(c.y, c.z, c.w);
        const unsigned long long w0 = compress_one<POLICY, kFma, NARROW, EV>(a.x, a.y, a.z, P, ev);
        const unsigned long long w1 = compress_one<POLICY, kFma, NARROW, EV>(a.w, b.x, b.y, P, ev);
        const unsigned long long w2 = compress_one<POLICY, kFma, NARROW, EV>(b.z, b.w, c.x, P, ev);
        const unsigned long long w3 = compress_one<POLICY, kFma, NARROW, EV>(c.y, c.z, c.w, P, ev);
        st_u4(out + 4 * g, w0, w1, w2, w3);
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        bad += !finite3(x, y, z);
        out[i] = compress_one<POLICY, kFma, NARROW, EV>(x, y, z, P, ev);
    }
    if (bad && nonfinite) atomicAdd(nonfinite, bad);
    if (EV) {
        if (ev[0]) atomicAdd(events, (unsigned long long)ev[0]);
        if (ev[1]) atomicAdd(events + 1, (unsigned long long)ev[1]);
    }
}

// K2 decompress: 4 words (32 B in, 48 B out) per thread per step.
// EXACT: bit-identical to the reference's libm decode (boundary components
// redone from its own tables); !EXACT: the fast table decode, each component
// the reference's float32 or one ulp from it.
// STAGE: the per-warp shared staging of the output (measured: contract mode
// 264 staged vs 243 direct, exact mode 248 staged vs 262 direct Gword/s).
// PREP: log2 replication of the phi grid (lane L reads copy L mod 2^PREP):
// fewer bank conflicts on its random lookups; MINB: resident CTAs per SM.
// Contract mode: PREP 2, one CTA per SM (275.5 vs 264.8 Gword/s); exact
// mode keeps the unreplicated table at 2 CTAs per SM (262 vs 261).
template <bool TABLE, class LAY, bool EXACT = true, bool STAGE = VC3_DECOMP_STAGE != 0, int PREP_ = 0,
          int MINB = VC3_DECOMP_MIN_BLOCKS, int TREP_ = 0, int THREADS = VC3_DECOMP_THREADS>
__global__ void __launch_bounds__(THREADS, MINB) k_decompress(const unsigned long long* __restrict__ w,
                                                         float* __restrict__ xyz, int64_t n,
                                                         Params Pin, bool vec,
                                                         const double2* __restrict__ gtab,
                                                         const double2* __restrict__ full) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ double2 s_tab[];
    constexpr int PREP = TABLE ? PREP_ : 0, TREP = TABLE ? TREP_ : 0;
    const int pb = P.t_n << TREP;  // phi grid start in the (replicated) copy
    const int tab_n = TABLE ? (PREP || TREP ? pb + (P.p_n << PREP) : P.tab_n) : 0;
    if (TABLE && (PREP || TREP)) {
        for (int i = threadIdx.x; i < tab_n; i += blockDim.x)
            s_tab[i] = gtab[i < pb ? (i >> TREP) : P.p_base + ((i - pb) >> PREP)];
        __syncthreads();
    } else {
        load_table<TABLE>(s_tab, gtab, P);
    }
    const double2* tt = s_tab + (TREP ? (threadIdx.x & ((1 << TREP) - 1)) : 0);
    const double2* tp = s_tab + (PREP || TREP ? pb : P.p_base) + (PREP ? (threadIdx.x & ((1 << PREP) - 1)) : 0);
    // the boundary test and its tolerance form must agree: the cell test
    // takes the doubled tolerance (exact_tol<true>), the two-conversion test
    // the plain one
    const double tol = EXACT ? exact_tol<VC3_DECOMP_CELL != 0>(full, P) : 0.0;
    const int64_t groups = vec ? n / 4 : 0;
    // per-warp shared staging of the array-of-structs output: each lane's 48 B
    // go to shared memory, then the warp writes 3 x 512 contiguous bytes
    float4* stage = !STAGE ? nullptr : reinterpret_cast<float4*>(s_tab + tab_n) + (threadIdx.x >> 5) * 96;
    const int lane = threadIdx.x & 31;
    (void)stage;
    (void)lane;
    // register double buffering: the next step's words are in flight while
    // this step decodes (one CTA holds only 1024 threads at 49 KB of table)
    int64_t g = gtid();
    u64x4 wn = {0, 0, 0, 0};
    if (g < groups) wn = ld_stream_u4(w + 4 * g);
    // whole warps step together so the staged stores stay warp-uniform
    const int64_t gw_end = ((groups + 31) / 32) * 32;
    for (; g < gw_end; g += gstride()) {
        const u64x4 u = wn;
        const int64_t gn = g + gstride();
        if (gn < groups) wn = ld_stream_u4(w + 4 * gn);
        float o[12];
        {
            decompress_one<TABLE, false, EXACT, VC3_DECOMP_CELL != 0, PREP, TREP>(u.x, P, tt, tp, o[0], o[1], o[2], full, tol);
            decompress_one<TABLE, false, EXACT, VC3_DECOMP_CELL != 0, PREP, TREP>(u.y, P, tt, tp, o[3], o[4], o[5], full, tol);
            decompress_one<TABLE, false, EXACT, VC3_DECOMP_CELL != 0, PREP, TREP>(u.z, P, tt, tp, o[6], o[7], o[8], full, tol);
            decompress_one<TABLE, false, EXACT, VC3_DECOMP_CELL != 0, PREP, TREP>(u.w, P, tt, tp, o[9], o[10], o[11], full, tol);
        }
        if constexpr (STAGE) {
        stage[3 * lane] = make_float4(o[0], o[1], o[2], o[3]);
        stage[3 * lane + 1] = make_float4(o[4], o[5], o[6], o[7]);
        stage[3 * lane + 2] = make_float4(o[8], o[9], o[10], o[11]);
        __syncwarp();
        const int64_t g0 = g - lane;  // first group of this warp
        float* base = xyz + 12 * g0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int idx = 32 * k + lane;  // float4 index within the warp's 1536 B
            VC3_DCHECK(idx < 96 && (threadIdx.x >> 5) * 96 + idx < (blockDim.x >> 5) * 96);
            if (g0 + idx / 3 < groups) {
                const float4 f = stage[idx];
                st_f4(base + 4 * idx, f.x, f.y, f.z, f.w);
            }
        }
        __syncwarp();
        } else {
        if (g < groups) {
            float* dst = xyz + 12 * g;
            st_f4(dst, o[0], o[1], o[2], o[3]);
            st_f4(dst + 4, o[4], o[5], o[6], o[7]);
            st_f4(dst + 8, o[8], o[9], o[10], o[11]);
        }
        }
    }
    for (int64_t i = groups * 4 + gtid(); i < n; i += gstride()) {
        float x, y, z;
        decompress_one<TABLE, false, EXACT, VC3_DECOMP_CELL != 0, PREP, TREP>(w[i], P, tt, tp, x, y, z, full, tol);
        xyz[3 * i] = x;
        xyz[3 * i + 1] = y;
        xyz[3 * i + 2] = z;
    }
}

// K5 uncompressed baseline: flat float32 add (_kernels.py:341-345)
__global__ void __launch_bounds__(kThreads) k_add_raw(const float* __restrict__ a,
                                                      const float* __restrict__ b,
                                                      float* __restrict__ c, int64_t n, bool vec) {
    const int64_t quads = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < quads; g += gstride()) {
        const float4 u = ld_stream_f4(a + 4 * g), v = ld_stream_f4(b + 4 * g);
        st_f4(c + 4 * g, __fadd_rn(u.x, v.x), __fadd_rn(u.y, v.y), __fadd_rn(u.z, v.z),
              __fadd_rn(u.w, v.w));
    }
    for (int64_t i = quads * 4 + gtid(); i < n; i += gstride()) c[i] = __fadd_rn(a[i], b[i]);
}

// K5b uncompressed RK-stage baseline: dq' = a*dq + dt*R ; q' = q + b*dq' (flat float32)
__global__ void __launch_bounds__(kThreads) k_rk_f32(float ca, float cb, float dt,
                                                     float* __restrict__ q, float* __restrict__ dq,
                                                     const float* __restrict__ R, int64_t n,
                                                     bool vec) {
    const int64_t quads = vec ? n / 4 : 0;
    for (int64_t g = gtid(); g < quads; g += gstride()) {
        float4 qv = *reinterpret_cast<const float4*>(q + 4 * g);
        float4 dv = *reinterpret_cast<const float4*>(dq + 4 * g);
        const float4 rv = ld_stream_f4(R + 4 * g);
        dv.x = __fadd_rn(__fmul_rn(ca, dv.x), __fmul_rn(dt, rv.x));
        dv.y = __fadd_rn(__fmul_rn(ca, dv.y), __fmul_rn(dt, rv.y));
        dv.z = __fadd_rn(__fmul_rn(ca, dv.z), __fmul_rn(dt, rv.z));
        dv.w = __fadd_rn(__fmul_rn(ca, dv.w), __fmul_rn(dt, rv.w));
        qv.x = __fadd_rn(qv.x, __fmul_rn(cb, dv.x));
        qv.y = __fadd_rn(qv.y, __fmul_rn(cb, dv.y));
        qv.z = __fadd_rn(qv.z, __fmul_rn(cb, dv.z));
        qv.w = __fadd_rn(qv.w, __fmul_rn(cb, dv.w));
        st_f4(dq + 4 * g, dv.x, dv.y, dv.z, dv.w);
        st_f4(q + 4 * g, qv.x, qv.y, qv.z, qv.w);
    }
    for (int64_t i = quads * 4 + gtid(); i < n; i += gstride()) {
        const float d = __fadd_rn(__fmul_rn(ca, dq[i]), __fmul_rn(dt, R[i]));
        dq[i] = d;
        q[i] = __fadd_rn(q[i], __fmul_rn(cb, d));
    }
}

// ----- pieces ----------------------------------------------------------------
template <unsigned POLICY>
__global__ void __launch_bounds__(kThreads) k_spherical(const float* __restrict__ xyz,
                                                        double* __restrict__ r,
                                                        double* __restrict__ th,
                                                        double* __restrict__ ph, int64_t n,
                                                        int32_t* nonfinite) {
    constexpr bool TS = POLICY & kThetaSingle, PS = POLICY & kPhiSingle;
    int bad = 0;
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        bad += !finite3(x, y, z);
        const double xd = x, yd = y, zd = z;
        const double s = __fma_rn(zd, zd, __fma_rn(yd, yd, __dmul_rn(xd, xd)));
        double rr = 0.0, t = 0.0, p = 0.0;
        if (s != 0.0) {
            rr = __dsqrt_rn(s);
            t = TS ? (double)atan2_f32<kFma>(y, x) : atan2(yd, xd);
            if (PS) {
                const float sq =
                    __fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z));
                const float rq = __fsqrt_rn(sq);
                float w = 1.0f;
                if (rq > 0.0f) w = fminf(fmaxf(__fdiv_rn(z, rq), -1.0f), 1.0f);
                p = (double)acos_f32<kFma>(w);
            } else {
                p = acos(fmin(fmax(__ddiv_rn(zd, rr), -1.0), 1.0));
            }
        }
        r[i] = rr;
        th[i] = t;
        ph[i] = p;
    }
    if (bad && nonfinite) atomicAdd(nonfinite, bad);
}

__global__ void __launch_bounds__(kThreads) k_quantize(const double* __restrict__ th,
                                                       const double* __restrict__ ph,
                                                       long long* __restrict__ nt,
                                                       long long* __restrict__ nph, int64_t n,
                                                       Params P, int quant_single) {
    // Arbitrary caller angles: the unfused reference sequence (no FMA proof applies).
    for (int64_t i = gtid(); i < n; i += gstride()) {
        long long a, b;
        quantize<false>(th[i], ph[i], quant_single != 0, P, a, b);
        nt[i] = a;
        nph[i] = b;
    }
}

__global__ void __launch_bounds__(kThreads) k_dequantize(const long long* __restrict__ nt,
                                                         const long long* __restrict__ nph,
                                                         double* __restrict__ th,
                                                         double* __restrict__ ph, int64_t n,
                                                         Params P) {
    // dequantize_kernel (_kernels.py:334-338): pi*(2n/nmax - 1), pi*n/nmax
    for (int64_t i = gtid(); i < n; i += gstride()) {
        th[i] = __dmul_rn(kPi, __dsub_rn(__ddiv_rn(__dmul_rn(2.0, (double)nt[i]), (double)P.ntmax), 1.0));
        ph[i] = __ddiv_rn(__dmul_rn(kPi, (double)nph[i]), (double)P.npmax);
    }
}

__global__ void __launch_bounds__(kThreads) k_encode_mag(const double* __restrict__ r,
                                                         unsigned long long* __restrict__ f,
                                                         int64_t n, Params P) {
    for (int64_t i = gtid(); i < n; i += gstride()) f[i] = encode_mag(r[i], P);
}

__global__ void __launch_bounds__(kThreads) k_decode_mag(const long long* __restrict__ f,
                                                         float* __restrict__ r, int64_t n,
                                                         Params P) {
    for (int64_t i = gtid(); i < n; i += gstride()) r[i] = decode_mag((unsigned long long)f[i], P);
}

__global__ void __launch_bounds__(kThreads) k_mag_events(const float* __restrict__ xyz, int64_t n,
                                                         Params P,
                                                         unsigned long long* __restrict__ counts,
                                                         int32_t* __restrict__ nonfinite) {
    unsigned long long fl = 0, sat = 0;
    int bad = 0;
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        bad += !finite3(x, y, z);
        const double xd = x, yd = y, zd = z;
        const double r = __dsqrt_rn(__fma_rn(zd, zd, __fma_rn(yd, yd, __dmul_rn(xd, xd))));
        if (r > 0.0) {
            const unsigned u = __float_as_uint(__double2float_ru(r));
            const int e7 = (int)((u >> 23) & 0xFFu) - 127 + P.bias;
            fl += e7 <= 1;
            sat += e7 >= P.emax;
        }
    }
    if (fl) atomicAdd(counts, fl);
    if (sat) atomicAdd(counts + 1, sat);
    if (bad && nonfinite) atomicAdd(nonfinite, bad);
}

// ----- K6 error statistics (analysis.py:118-167) ------------------------------
// Stage 1: each block reduces a contiguous slice of one chunk to (n, mean, M2, max)
// with per-thread Welford and Chan merges in a fixed order (deterministic).
struct Moments {
    double n, mean, m2, max;
};

__device__ __forceinline__ Moments chan(Moments a, Moments b) {
    if (a.n == 0) return b;
    if (b.n == 0) return a;
    const double n = a.n + b.n, d = b.mean - a.mean;
    Moments r;
    r.n = n;
    r.mean = a.mean + d * (b.n / n);
    r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / n);
    r.max = fmax(a.max, b.max);
    return r;
}

// Error metrics (include/vc3_b200.h VC3_ERR_*), double precision, every
// operation rounded in the order written (the tests' numpy restatement
// follows the same order):
//   0 L2:        e = ||v - vh||
//   1 L2/|v|:    e = ||v - vh|| / ||v||            (||v|| = 0 -> / 1)
//   2 angular:   e = atan2(||v x vh||, v . vh)     (radians; 0 for zero vectors)
//   3 rel. mag.: e = | ||vh|| - ||v|| | / ||v||    (||v|| = 0 -> 0)
__device__ __forceinline__ double norm3(double x, double y, double z) {
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

__device__ __forceinline__ double err_one(const float* v, const float* vh, int64_t i, int kind) {
    const double x = v[3 * i], y = v[3 * i + 1], z = v[3 * i + 2];
    const double a = vh[3 * i], b = vh[3 * i + 1], c = vh[3 * i + 2];
    if (kind == VC3_ERR_ANGULAR) {
        const double cx = __dsub_rn(__dmul_rn(y, c), __dmul_rn(z, b));
        const double cy = __dsub_rn(__dmul_rn(z, a), __dmul_rn(x, c));
        const double cz = __dsub_rn(__dmul_rn(x, b), __dmul_rn(y, a));
        const double dot = __dadd_rn(__dadd_rn(__dmul_rn(x, a), __dmul_rn(y, b)), __dmul_rn(z, c));
        return atan2(norm3(cx, cy, cz), dot);
    }
    const double nv = norm3(x, y, z);
    if (kind == VC3_ERR_REL_MAGNITUDE) {
        return nv > 0.0 ? __ddiv_rn(fabs(__dsub_rn(norm3(a, b, c), nv)), nv) : 0.0;
    }
    double e = norm3(__dsub_rn(x, a), __dsub_rn(y, b), __dsub_rn(z, c));
    if (kind == VC3_ERR_L2_NORMALISED) e = __ddiv_rn(e, nv > 0.0 ? nv : 1.0);
    return e;
}

constexpr int kStatThreads = 256;
constexpr int kStatSlice = 8192;  // vectors per block slice

__global__ void __launch_bounds__(kStatThreads) k_err_partial(const float* __restrict__ v,
                                                              const float* __restrict__ vh,
                                                              int64_t n, int kind,
                                                              int64_t chunk, int slices_per_chunk,
                                                              Moments* __restrict__ part) {
    const int64_t c = blockIdx.y, s = blockIdx.x;
    const int64_t c0 = c * chunk, c1 = min(n, c0 + chunk);
    const int64_t lo = c0 + s * (int64_t)kStatSlice, hi = min(c1, lo + kStatSlice);
    Moments m = {0, 0, 0, 0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += kStatThreads) {
        const double e = err_one(v, vh, i, kind);
        m.n += 1;
        const double d = e - m.mean;
        m.mean += d / m.n;
        m.m2 += d * (e - m.mean);
        m.max = fmax(m.max, e);
    }
    __shared__ Moments sh[kStatThreads];
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int w = kStatThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] = chan(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[c * slices_per_chunk + s] = sh[0];
}

__global__ void k_err_final(const Moments* __restrict__ part, int64_t nchunks,
                            int slices_per_chunk, double* __restrict__ out) {
    for (int64_t c = gtid(); c < nchunks; c += gstride()) {
        Moments m = {0, 0, 0, 0};
        for (int s = 0; s < slices_per_chunk; ++s) m = chan(m, part[c * slices_per_chunk + s]);
        out[4 * c] = m.n;
        out[4 * c + 1] = m.mean;
        out[4 * c + 2] = m.m2;
        out[4 * c + 3] = m.max;
    }
}

}  // namespace
namespace vc3 {
namespace as {  // vc3_fused_as.cu
int launch_compress(const float* xyz, unsigned long long* w, int64_t n, const Params& P, bool def,
                    bool vec, int32_t* nonfinite, cudaStream_t s);
}  // namespace as
}  // namespace vc3
namespace {

template <unsigned POL>
struct RunCompress {
    static int run(const float* x, uint64_t* w, int64_t n, const Params& P, bool def, int32_t* nf,
                   unsigned long long* ev, cudaStream_t s) {
        const bool vec = aligned16(x) && aligned32(w);
        // all-single policy: the restructured compress of vc3_fused.cuh
        if (POL == 7u && !ev && P.t <= 25 && P.p <= 24)
            return vc3::as::launch_compress(x, (unsigned long long*)w, n, P, def, vec, nf, s);
        const unsigned grid = grid_for(vec ? (n + 3) / 4 : n, VC3_COMPRESS_CTAS_PER_SM);
        auto W = (unsigned long long*)w;
        if (ev) {
            if (def)
                k_compress<POL, true, DefaultLayout, true><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf, ev);
            else if (P.t <= 29 && P.p <= 29)
                k_compress<POL, true, RuntimeLayout, true><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf, ev);
            else
                k_compress<POL, false, RuntimeLayout, true><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf, ev);
        } else if (def) {
            k_compress<POL, true, DefaultLayout><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf);
        } else if (P.t <= 29 && P.p <= 29) {
            k_compress<POL, true, RuntimeLayout><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf);
        } else {
            k_compress<POL, false, RuntimeLayout><<<grid, kThreads, 0, s>>>(x, W, n, P, vec, nf);
        }
        return launch_status();
    }
};

template <unsigned POL>
struct RunSpherical {
    static int run(const float* x, double* r, double* t, double* p, int64_t n, int32_t* nf,
                   cudaStream_t s) {
        k_spherical<POL & 3u><<<grid_for(n), kThreads, 0, s>>>(x, r, t, p, n, nf);
        return launch_status();
    }
};

}  // namespace

// ===================== extern "C" boundary ====================================
namespace {
// One k_decompress configuration: replication of the phi / theta grids
// (PREP / TREP, log2), CTA size, resident CTAs, grid cap per SM.
template <bool TABLE, class LAY, bool EXACT, bool STAGE, int PREP, int TREP, int THREADS, int MINB>
int decomp_launch(const unsigned long long* W, float* xyz, int64_t n, const Params& P, bool vec,
                  const double2* tab, const double2* full, int per_sm, cudaStream_t s) {
    auto fn = k_decompress<TABLE, LAY, EXACT, STAGE, PREP, MINB, TREP, THREADS>;
    const size_t tab_bytes =
        !TABLE ? 0
               : (PREP || TREP ? (size_t)((P.t_n << TREP) + (P.p_n << PREP)) * sizeof(double2) : table_smem(P));
    const size_t smem = tab_bytes + (STAGE ? (size_t)THREADS * 48 : 0);  // staging: 1.5 KB per warp
    if (const int st = ensure_smem((const void*)fn, smem)) return st;
    const int64_t items = vec ? (n + 3) / 4 : n;
    int64_t blocks = (items + THREADS - 1) / THREADS;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    blocks = blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
    fn<<<(unsigned)blocks, THREADS, smem, s>>>(W, xyz, n, P, vec, tab, full);
    return launch_status();
}

}  // namespace

extern "C" {

const char* vc3_version(void) { return "vc3-b200 0.2.0 (sm_100a)"; }

const char* vc3_status_string(int status) {
    switch (status) {
        case VC3_OK: return "ok";
        case VC3_ERR_LAYOUT: return "invalid bit layout";
        case VC3_ERR_ARG: return "invalid argument";
        case VC3_ERR_CUDA: return "CUDA error";
        case VC3_ERR_NONFINITE: return "non-finite input";
        case VC3_ERR_LENGTH: return "length mismatch";
        default: return "unknown status";
    }
}

int vc3_last_cuda_error(void) { return g_last_cuda; }

int vc3_validate_layout(vc3_layout layout) { return layout_ok(layout) ? VC3_OK : VC3_ERR_LAYOUT; }

int vc3_compress(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout, uint32_t policy,
                 int32_t* d_nonfinite, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!xyz || !words) return VC3_ERR_ARG;
    return by_policy<RunCompress>(policy, xyz, words, n, make_params(layout),
                                  is_default_layout(layout), d_nonfinite,
                                  (unsigned long long*)nullptr, (cudaStream_t)stream);
}

int vc3_compress_events(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout,
                        uint32_t policy, int32_t* d_nonfinite, uint64_t* d_events, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!xyz || !words || !d_events) return VC3_ERR_ARG;
    return by_policy<RunCompress>(policy, xyz, words, n, make_params(layout),
                                  is_default_layout(layout), d_nonfinite,
                                  (unsigned long long*)d_events, (cudaStream_t)stream);
}

int vc3_decode_tolerance(vc3_layout layout, double* tol) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (!tol) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    *tol = 0.0;
    const double2* full = nullptr;
    const int st = get_full_table(P, &full);
    if (st || !full) return st;
    *tol = full_table_tolerance(P);
    return VC3_OK;
}

int vc3_prepare_layout(vc3_layout layout, uint32_t flags) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (flags & ~VC3_FLAGS_ALL) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    const double2* tab = nullptr;
    if (const int st = get_table(P, &tab)) return st;
    if (!(flags & VC3_CONTRACT)) {
        const double2* full = nullptr;
        if (const int st = get_full_table(P, &full)) return st;
    }
    return VC3_OK;
}

int vc3_decompress_ex(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout,
                      uint32_t flags, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (flags & ~VC3_FLAGS_ALL) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!xyz || !words) return VC3_ERR_ARG;
    const Params P = make_params(layout);
    const double2* tab = nullptr;
    int st = get_table(P, &tab);
    if (st) return st;
    const bool exact = !(flags & VC3_CONTRACT);
    const double2* full = nullptr;
    if (exact) {
        st = get_full_table(P, &full);
        if (st) return st;
    }
    auto W = (const unsigned long long*)words;
    const bool vec = aligned32(words) && aligned16(xyz);
    cudaStream_t s = (cudaStream_t)stream;
    const bool def = is_default_layout(layout);
    if (!P.table_mode)  // wide layouts: the reference-angle polynomial (no table, no exactness test)
        return decomp_launch<false, RuntimeLayout, true, true, 0, 0, VC3_DECOMP_THREADS, VC3_DECOMP_MIN_BLOCKS>(
            W, xyz, n, P, vec, tab, full, VC3_DECOMP_CTAS_PER_SM, s);
    // measured (2^28 words, Gword/s exact / contract): cfg 0 255.3 / 255.6,
    // cfg 1 259.2 / 275.3, cfg 2 262.2 / 273.0, cfg 3 270.4 / 272.3
    int cfg = exact ? 3 : 1;
#ifdef VC3_TUNE
    static const int tune = getenv("VC3_TUNE_DEC") ? atoi(getenv("VC3_TUNE_DEC")) : -1;
    if (tune >= 0) cfg = tune;
#endif
#define VC3_DEC_GO(LAY)                                                                                   \
    switch (cfg) {                                                                                        \
        case 0: /* 2 x 512 threads, unreplicated table */                                                 \
            return exact ? decomp_launch<true, LAY, true, false, 0, 0, 512, 2>(W, xyz, n, P, vec, tab, full, 4, s) \
                         : decomp_launch<true, LAY, false, true, 0, 0, 512, 2>(W, xyz, n, P, vec, tab, full, 4, s); \
        case 1: /* 1 x 512 threads, phi grid x4 */                                                        \
            return exact ? decomp_launch<true, LAY, true, false, 2, 0, 512, 1>(W, xyz, n, P, vec, tab, full, 2, s) \
                         : decomp_launch<true, LAY, false, true, 2, 0, 512, 1>(W, xyz, n, P, vec, tab, full, 2, s); \
        case 2: /* 1 x 768 threads, theta grid x2, phi grid x4 */                                         \
            return exact ? decomp_launch<true, LAY, true, false, 2, 1, 768, 1>(W, xyz, n, P, vec, tab, full, 1, s) \
                         : decomp_launch<true, LAY, false, true, 2, 1, 768, 1>(W, xyz, n, P, vec, tab, full, 1, s); \
        default: /* 1 x 768 threads, theta grid x4, phi grid x2 */                                        \
            return exact ? decomp_launch<true, LAY, true, false, 1, 2, 768, 1>(W, xyz, n, P, vec, tab, full, 1, s) \
                         : decomp_launch<true, LAY, false, true, 1, 2, 768, 1>(W, xyz, n, P, vec, tab, full, 1, s); \
    }
    if (def) {
        VC3_DEC_GO(DefaultLayout)
    } else {
        VC3_DEC_GO(RuntimeLayout)
    }
#undef VC3_DEC_GO
}

int vc3_decompress(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout, void* stream) {
    return vc3_decompress_ex(words, xyz, n, layout, VC3_EXACT, stream);
}

int vc3_add_raw(const float* a, const float* b, float* c, int64_t n_floats, void* stream) {
    VC3_CHECK_N(n_floats);
    if (!a || !b || !c) return VC3_ERR_ARG;
    const bool vec = aligned16(a) && aligned16(b) && aligned16(c);
    k_add_raw<<<grid_for(vec ? (n_floats + 3) / 4 : n_floats), kThreads, 0, (cudaStream_t)stream>>>(
        a, b, c, n_floats, vec);
    return launch_status();
}

int vc3_rk_stage_f32(float a, float b, float dt, float* q, float* dq, const float* R,
                     int64_t n_floats, void* stream) {
    VC3_CHECK_N(n_floats);
    if (!q || !dq || !R) return VC3_ERR_ARG;
    const bool vec = aligned16(q) && aligned16(dq) && aligned16(R);
    k_rk_f32<<<grid_for(vec ? (n_floats + 3) / 4 : n_floats), kThreads, 0, (cudaStream_t)stream>>>(
        a, b, dt, q, dq, R, n_floats, vec);
    return launch_status();
}

int vc3_to_spherical(const float* xyz, double* r, double* theta, double* phi, int64_t n,
                     uint32_t policy, int32_t* d_nonfinite, void* stream) {
    if (policy > 7u) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!xyz || !r || !theta || !phi) return VC3_ERR_ARG;
    return by_policy<RunSpherical>(policy, xyz, r, theta, phi, n, d_nonfinite,
                                   (cudaStream_t)stream);
}

int vc3_quantize_angles(const double* theta, const double* phi, int64_t* n_theta, int64_t* n_phi,
                        int64_t n, vc3_layout layout, uint32_t policy, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    if (policy > 7u) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!theta || !phi || !n_theta || !n_phi) return VC3_ERR_ARG;
    k_quantize<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        theta, phi, (long long*)n_theta, (long long*)n_phi, n, make_params(layout),
        (policy & VC3_QUANT_SINGLE) ? 1 : 0);
    return launch_status();
}

int vc3_dequantize_angles(const int64_t* n_theta, const int64_t* n_phi, double* theta, double* phi,
                          int64_t n, vc3_layout layout, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    VC3_CHECK_N(n);
    if (!theta || !phi || !n_theta || !n_phi) return VC3_ERR_ARG;
    k_dequantize<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        (const long long*)n_theta, (const long long*)n_phi, theta, phi, n, make_params(layout));
    return launch_status();
}

int vc3_encode_magnitude(const double* r, uint64_t* field, int64_t n, vc3_layout layout,
                         void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    VC3_CHECK_N(n);
    if (!r || !field) return VC3_ERR_ARG;
    k_encode_mag<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        r, (unsigned long long*)field, n, make_params(layout));
    return launch_status();
}

int vc3_decode_magnitude(const int64_t* field, float* r, int64_t n, vc3_layout layout,
                         void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    VC3_CHECK_N(n);
    if (!r || !field) return VC3_ERR_ARG;
    k_decode_mag<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>((const long long*)field, r, n,
                                                                    make_params(layout));
    return launch_status();
}

int vc3_magnitude_events_checked(const float* xyz, int64_t n, vc3_layout layout,
                                 unsigned long long* d_counts, int32_t* d_nonfinite, void* stream) {
    if (!layout_ok(layout)) return VC3_ERR_LAYOUT;
    VC3_CHECK_N(n);
    if (!xyz || !d_counts) return VC3_ERR_ARG;
    k_mag_events<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(xyz, n, make_params(layout),
                                                                    d_counts, d_nonfinite);
    return launch_status();
}

int vc3_magnitude_events(const float* xyz, int64_t n, vc3_layout layout,
                         unsigned long long* d_counts, void* stream) {
    return vc3_magnitude_events_checked(xyz, n, layout, d_counts, nullptr, stream);
}

int vc3_error_stats_workspace(int64_t n, int64_t chunk, uint64_t* bytes) {
    if (n < 0 || chunk <= 0 || !bytes) return VC3_ERR_ARG;
    const int64_t nchunks = n ? (n + chunk - 1) / chunk : 0;
    const int64_t slices = n ? (std::min(chunk, n) + kStatSlice - 1) / kStatSlice : 0;
    *bytes = (uint64_t)(sizeof(Moments) * slices * nchunks);
    return VC3_OK;
}

int vc3_error_stats_ws(const float* v, const float* vh, int64_t n, int32_t kind, int64_t chunk,
                       double* d_chunk_stats, void* d_work, uint64_t work_bytes, void* stream) {
    if (kind < VC3_ERR_L2 || kind > VC3_ERR_REL_MAGNITUDE) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!v || !vh || !d_chunk_stats || chunk <= 0) return VC3_ERR_ARG;
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const int64_t slices64 = (std::min(chunk, n) + kStatSlice - 1) / kStatSlice;
    if (slices64 > 65535 || nchunks > 65535) return VC3_ERR_ARG;
    if (!d_work || work_bytes < sizeof(Moments) * slices64 * nchunks) return VC3_ERR_ARG;
    const int slices = (int)slices64;
    cudaStream_t s = (cudaStream_t)stream;
    Moments* part = (Moments*)d_work;
    k_err_partial<<<dim3(slices, (unsigned)nchunks), kStatThreads, 0, s>>>(v, vh, n, kind,
                                                                          chunk, slices, part);
    k_err_final<<<grid_for(nchunks), kThreads, 0, s>>>(part, nchunks, slices, d_chunk_stats);
    return launch_status();
}

int vc3_error_stats(const float* v, const float* vh, int64_t n, int32_t kind, int64_t chunk,
                    double* d_chunk_stats, void* stream) {
    if (kind < VC3_ERR_L2 || kind > VC3_ERR_REL_MAGNITUDE) return VC3_ERR_ARG;
    VC3_CHECK_N(n);
    if (!v || !vh || !d_chunk_stats || chunk <= 0) return VC3_ERR_ARG;
    uint64_t bytes = 0;
    vc3_error_stats_workspace(n, chunk, &bytes);
    cudaStream_t s = (cudaStream_t)stream;
    // stream-ordered scratch from the device's default memory pool (no
    // device-wide synchronisation; legal inside graph capture)
    void* part = nullptr;
    int st = cuda_status(cudaMallocAsync(&part, bytes, s));
    if (st) return st;
    st = vc3_error_stats_ws(v, vh, n, kind, chunk, d_chunk_stats, part, bytes, stream);
    cudaFreeAsync(part, s);
    return st;
}

}  // extern "C"
