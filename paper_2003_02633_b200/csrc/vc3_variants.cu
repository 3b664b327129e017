// vc3_variants.cu — K7: companded and fractionally split angle coding
// (/root/reference/pkg/src/vc3/analysis.py:259-417) on sm_100a.
//
// The reference evaluates both variants only inside its studies
// (compand_study, split_sweep), with double-precision spherical angles
// (ORACLE policy), numpy double transcendental functions and a float32
// reconstruction.  Here each variant is a word format with a compress and a
// decompress kernel, so the studies (and any caller) run on the device:
//   compander (uniform / cosine / tanh):  [magnitude | n_phi | n_theta], the
//       layout's packing with companded indices;
//   split: [magnitude (64 - total_bits) | J], J = n_phi*(n_theta_max+1) + n_theta
//       (analysis.py:284-291), the format SURVEY H6 proposes.
// Double transcendental functions come from CUDA's libm (<= 2 ulp), so a
// bucket index can differ from the reference's only at ties; tests count them.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"

using namespace vc3;

namespace {

constexpr int kThreads = 256;

struct VParams {
    int kind;                  // VC3_VARIANT_*
    double gamma, c, m;        // tanh compander: c = tanh(gamma), m = 1/(2c) (host glibc, like math.tanh)
    long long nt_max, np_max;  // bucket maxima (split: derived; compander: the layout's)
    int t, p, shift;           // compander packing widths; split: shift = total_bits
    int e, mb, bias, emax;     // magnitude field
    unsigned field_low, field_high;
};

__device__ __forceinline__ long long nint_d(double v) {
    // ceil(floor(2v)/2) (analysis.py:306, :378)
    return (__double2ll_rd(__dmul_rn(2.0, v)) + 1) >> 1;
}

__device__ __forceinline__ long long clip_ll(long long v, long long hi) {
    return v < 0 ? 0 : (v > hi ? hi : v);
}

// Compander.encode (analysis.py:364-378)
template <int KIND>
__device__ __forceinline__ long long compand_encode(double psi, long long n_max, const VParams& V) {
    const double nm = (double)n_max;
    double raw;
    if (KIND == VC3_VARIANT_COSINE) {
        raw = __ddiv_rn(__dmul_rn(nm, __dsub_rn(1.0, cos(__dmul_rn(kPi, psi)))), 2.0);
    } else if (KIND == VC3_VARIANT_TANH) {
        const double t = tanh(__dmul_rn(V.gamma, __dsub_rn(__dmul_rn(2.0, psi), 1.0)));
        raw = __dmul_rn(__dmul_rn(V.m, nm), __dadd_rn(t, V.c));
    } else {
        raw = __dmul_rn(psi, nm);
    }
    return clip_ll(nint_d(raw), n_max);
}

// Compander.decode (analysis.py:380-393)
template <int KIND>
__device__ __forceinline__ double compand_decode(long long n, long long n_max, const VParams& V) {
    const double nd = (double)n, nm = (double)n_max;
    if (KIND == VC3_VARIANT_COSINE) {
        const double arg = fmin(fmax(__dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, nd), nm)), -1.0), 1.0);
        return __ddiv_rn(acos(arg), kPi);
    }
    if (KIND == VC3_VARIANT_TANH) {
        const double u = fmin(fmax(__dsub_rn(__ddiv_rn(nd, __dmul_rn(V.m, nm)), V.c), -V.c), V.c);
        const double psi = __ddiv_rn(__dadd_rn(__ddiv_rn(atanh(u), V.gamma), 1.0), 2.0);
        return fmin(fmax(psi, 0.0), 1.0);
    }
    return __ddiv_rn(nd, nm);
}

__device__ __forceinline__ unsigned encode_field(double r64, const VParams& V) {
    if (r64 == 0.0) return 0u;
    const unsigned u = __float_as_uint(__double2float_ru(r64));
    const int e7 = (int)((u >> 23) & 0xFFu) - 127 + V.bias;
    if (e7 <= 1) return V.field_low;
    if (e7 >= V.emax) return V.field_high;
    return ((unsigned)e7 << V.mb) | ((u & 0x7FFFFFu) >> (23 - V.mb));
}

__device__ __forceinline__ float decode_field(unsigned long long field, const VParams& V) {
    if (field == 0ull) return 0.0f;
    const int e7 = (int)((field >> V.mb) & (unsigned long long)V.emax);
    const unsigned mant = (unsigned)(field & ((1ull << V.mb) - 1ull));
    int e8 = e7 - V.bias + 127;
    e8 = e8 < 0 ? 0 : (e8 > 254 ? 254 : e8);
    return __uint_as_float(((unsigned)e8 << 23) | (mant << (23 - V.mb)));
}

// KIND: the variant, a template parameter so each kernel carries one code path
template <int KIND>
__global__ void __launch_bounds__(kThreads) k_compress_variant(const float* __restrict__ xyz,
                                                               unsigned long long* __restrict__ out,
                                                               int64_t n, VParams V,
                                                               int32_t* nonfinite) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        bad += !finite3(x, y, z);
        // to_spherical under the ORACLE policy (_kernels.py:89-126)
        const double xd = x, yd = y, zd = z;
        const double s = __fma_rn(zd, zd, __fma_rn(yd, yd, __dmul_rn(xd, xd)));
        const double r64 = __dsqrt_rn(s);
        double th = 0.0, ph = 0.0;
        if (r64 != 0.0) {
            th = atan2(yd, xd);
            ph = acos(fmin(fmax(__ddiv_rn(zd, r64), -1.0), 1.0));
        }
        long long nt, nph;
        unsigned long long angles;
        if (KIND == VC3_VARIANT_SPLIT) {
            // _quantize_free (analysis.py:300-306), then joint_encode (:284-291)
            const double ntm = (double)V.nt_max, npm = (double)V.np_max;
            const double vt = __dadd_rn(__ddiv_rn(ntm, 2.0), __dmul_rn(th, __ddiv_rn(ntm, __dmul_rn(2.0, kPi))));
            const double vp = __dmul_rn(ph, __ddiv_rn(npm, kPi));
            nt = clip_ll(nint_d(vt), V.nt_max);
            nph = clip_ll(nint_d(vp), V.np_max);
            angles = (unsigned long long)nph * (unsigned long long)(V.nt_max + 1) + (unsigned long long)nt;
        } else {
            // compand_study (analysis.py:404-405)
            const double psi_t = __ddiv_rn(__dadd_rn(th, kPi), __dmul_rn(2.0, kPi));
            nt = compand_encode<KIND>(psi_t, V.nt_max, V);
            nph = compand_encode<KIND>(__ddiv_rn(ph, kPi), V.np_max, V);
            angles = ((unsigned long long)nph << V.t) | (unsigned long long)nt;
        }
        const unsigned long long field = encode_field(r64, V);
        out[i] = r64 == 0.0 ? 0ull : ((field << V.shift) | angles);
    }
    if (bad && nonfinite) atomicAdd(nonfinite, bad);
}

// The reconstruction angles are formed as multiples of pi and their sin/cos
// taken with sincospi: theta = pi q_t, phi = pi q_p with q_t = 2 psi_t - 1
// (compander) or 2 n_t / n_t_max - 1 (split), q_p = psi_p or n_p / n_p_max.
// The reference rounds pi q first and calls sin / cos; the two differ by
// about one double ulp, so a float32 component differs (by one ulp) only
// where its double lies within that of a rounding boundary (tests: <= 2 ulp,
// >= 99.9 % exact).
template <int KIND>
__global__ void __launch_bounds__(kThreads) k_decompress_variant(const unsigned long long* __restrict__ w,
                                                                 float* __restrict__ xyz, int64_t n,
                                                                 VParams V) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long word = w[i];
        const unsigned long long field = word >> V.shift;
        const unsigned long long angles = word & ((1ull << V.shift) - 1ull);
        double qt, qp;
        if (KIND == VC3_VARIANT_SPLIT) {
            // joint_decode (analysis.py:294-297) and the reconstruction (:326-333)
            const unsigned long long nt1 = (unsigned long long)(V.nt_max + 1);
            const long long nph = (long long)(angles / nt1), nt = (long long)(angles % nt1);
            qt = __dsub_rn(__ddiv_rn(__dmul_rn(2.0, (double)nt), (double)V.nt_max), 1.0);
            qp = __ddiv_rn((double)nph, (double)V.np_max);
        } else {
            // compand_study reconstruction (analysis.py:406-414)
            const long long nt = (long long)(angles & ((1ull << V.t) - 1ull));
            const long long nph = (long long)((angles >> V.t) & ((1ull << V.p) - 1ull));
            qt = __dsub_rn(__dmul_rn(2.0, compand_decode<KIND>(nt, V.nt_max, V)), 1.0);
            qp = compand_decode<KIND>(nph, V.np_max, V);
        }
        const double rh = (double)decode_field(field, V);
        double st, ct, sp, cp;
        sincospi(qt, &st, &ct);
        sincospi(qp, &sp, &cp);
        xyz[3 * i] = __double2float_rn(__dmul_rn(__dmul_rn(rh, ct), sp));
        xyz[3 * i + 1] = __double2float_rn(__dmul_rn(__dmul_rn(rh, st), sp));
        xyz[3 * i + 2] = __double2float_rn(__dmul_rn(rh, cp));
    }
}

int make_vparams(const vc3_layout& L, const vc3_variant& var, VParams* out) {
    if (vc3_validate_layout(L) != VC3_OK) return VC3_ERR_LAYOUT;
    VParams V{};
    V.kind = var.kind;
    V.e = L.exponent_bits;
    V.mb = L.mantissa_bits;
    V.bias = L.exponent_bias;
    V.emax = (1 << V.e) - 1;
    V.field_low = 2u << V.mb;
    V.field_high = ((unsigned)(V.emax - 1) << V.mb) | ((1u << V.mb) - 1u);
    V.t = L.theta_bits;
    V.p = L.phi_bits;
    V.shift = L.phi_bits + L.theta_bits;
    if (var.kind == VC3_VARIANT_SPLIT) {
        // SplitConfig (analysis.py:259-281); the joint index must fill the
        // layout's angle bits so the magnitude field keeps its width.
        const int tb = var.total_bits;
        if (tb != V.shift || tb < 2 || tb > 62 || var.n_phi_max < 1) return VC3_ERR_ARG;
        const long long cap = 1LL << tb;
        const long long nt1 = cap / (var.n_phi_max + 1);
        if (nt1 < 2) return VC3_ERR_ARG;
        V.np_max = var.n_phi_max;
        V.nt_max = nt1 - 1;
        if ((V.np_max + 1) * (V.nt_max + 1) - 1 >= cap) return VC3_ERR_ARG;
    } else if (var.kind == VC3_VARIANT_UNIFORM || var.kind == VC3_VARIANT_COSINE ||
               var.kind == VC3_VARIANT_TANH) {
        V.nt_max = (1LL << V.t) - 1;
        V.np_max = (1LL << V.p) - 1;
        if (var.kind == VC3_VARIANT_TANH) {
            if (!(var.gamma > 0.0)) return VC3_ERR_ARG;
            V.gamma = var.gamma;
            V.c = tanh(var.gamma);
            V.m = 1.0 / (2.0 * V.c);
        }
    } else {
        return VC3_ERR_ARG;
    }
    *out = V;
    return VC3_OK;
}

unsigned grid_for_n(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t b = (n + kThreads - 1) / kThreads, cap = (int64_t)sms * 8;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

extern "C" {

int vc3_compress_variant(const float* xyz, uint64_t* words, int64_t n, vc3_layout layout,
                         vc3_variant variant, int32_t* d_nonfinite, void* stream) {
    VParams V;
    int st = make_vparams(layout, variant, &V);
    if (st) return st;
    if (n < 0) return VC3_ERR_ARG;
    if (n == 0) return VC3_OK;
    if (!xyz || !words) return VC3_ERR_ARG;
    const unsigned g = grid_for_n(n);
    cudaStream_t s = (cudaStream_t)stream;
    auto out = (unsigned long long*)words;
    switch (V.kind) {
        case VC3_VARIANT_COSINE: k_compress_variant<VC3_VARIANT_COSINE><<<g, kThreads, 0, s>>>(xyz, out, n, V, d_nonfinite); break;
        case VC3_VARIANT_TANH: k_compress_variant<VC3_VARIANT_TANH><<<g, kThreads, 0, s>>>(xyz, out, n, V, d_nonfinite); break;
        case VC3_VARIANT_SPLIT: k_compress_variant<VC3_VARIANT_SPLIT><<<g, kThreads, 0, s>>>(xyz, out, n, V, d_nonfinite); break;
        default: k_compress_variant<VC3_VARIANT_UNIFORM><<<g, kThreads, 0, s>>>(xyz, out, n, V, d_nonfinite);
    }
    return cudaGetLastError() == cudaSuccess ? VC3_OK : VC3_ERR_CUDA;
}

int vc3_decompress_variant(const uint64_t* words, float* xyz, int64_t n, vc3_layout layout,
                           vc3_variant variant, void* stream) {
    VParams V;
    int st = make_vparams(layout, variant, &V);
    if (st) return st;
    if (n < 0) return VC3_ERR_ARG;
    if (n == 0) return VC3_OK;
    if (!xyz || !words) return VC3_ERR_ARG;
    const unsigned g = grid_for_n(n);
    cudaStream_t s = (cudaStream_t)stream;
    auto in = (const unsigned long long*)words;
    switch (V.kind) {
        case VC3_VARIANT_COSINE: k_decompress_variant<VC3_VARIANT_COSINE><<<g, kThreads, 0, s>>>(in, xyz, n, V); break;
        case VC3_VARIANT_TANH: k_decompress_variant<VC3_VARIANT_TANH><<<g, kThreads, 0, s>>>(in, xyz, n, V); break;
        case VC3_VARIANT_SPLIT: k_decompress_variant<VC3_VARIANT_SPLIT><<<g, kThreads, 0, s>>>(in, xyz, n, V); break;
        default: k_decompress_variant<VC3_VARIANT_UNIFORM><<<g, kThreads, 0, s>>>(in, xyz, n, V);
    }
    return cudaGetLastError() == cudaSuccess ? VC3_OK : VC3_ERR_CUDA;
}

int vc3_variant_maxima(vc3_layout layout, vc3_variant variant, int64_t* n_theta_max,
                       int64_t* n_phi_max) {
    VParams V;
    int st = make_vparams(layout, variant, &V);
    if (st) return st;
    if (n_theta_max) *n_theta_max = V.nt_max;
    if (n_phi_max) *n_phi_max = V.np_max;
    return VC3_OK;
}

}  // extern "C"
