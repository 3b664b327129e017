// exhaustive.cu — proof-by-enumeration that the FMA forms used by the
// compress kernels give bit-identical results to the reference's unfused
// operation sequence, for EVERY float32 input the kernels can see.
//
//   1. atan2_f32 core: a = F32(td + td*z*Q_atan(z)), td = t in [0, 1]
//      (_kernels.py:39-61; t = lo/hi is an IEEE float32 quotient in [0, 1]).
//   2. acos_f32(w) for every float32 w in [-1, 1]            (_kernels.py:64-80)
//   3. theta bucket nint(ntmax/2 + th*(ntmax/(2 pi))) for every float32 th in
//      [-F32(pi), F32(pi)] and every theta width t = 1..32   (_kernels.py:129-147);
//      the kernels use the fused form for t <= 29 only (t = 30, 32 show ties).
//
// Prints one line per check: "<name> checked=<N> mismatches=<M>" and exits 0
// only when every mismatch count is zero.  tests/test_exhaustive.py runs it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -ftz=false
//        -prec-div=true -prec-sqrt=true -I include -o tools/exhaustive tools/exhaustive.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_2003_02633_b200/csrc/vc3_device.cuh"

using namespace vc3;

__global__ void k_atan(unsigned lo, unsigned hi, unsigned long long* bad, unsigned* first) {
    for (unsigned long long b = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         b <= hi; b += (unsigned long long)gridDim.x * blockDim.x) {
        const float t = __uint_as_float((unsigned)b);
        const float a = __double2float_rn(atan_core<true>((double)t));
        const float r = __double2float_rn(atan_core<false>((double)t));
        if (__float_as_uint(a) != __float_as_uint(r)) {
            atomicAdd(bad, 1ull);
            atomicMin(first, (unsigned)b);
        }
    }
}

__global__ void k_acos(unsigned lo, unsigned hi, unsigned long long* bad, unsigned* first) {
    for (unsigned long long b = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         b <= hi; b += (unsigned long long)gridDim.x * blockDim.x) {
        const float w = __uint_as_float((unsigned)b);
        if (__float_as_uint(acos_f32<true>(w)) != __float_as_uint(acos_f32<false>(w))) {
            atomicAdd(bad, 1ull);
            atomicMin(first, (unsigned)b);
        }
    }
}

__global__ void k_theta(unsigned lo, unsigned hi, Params P, unsigned long long* bad,
                        unsigned* first) {
    for (unsigned long long b = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         b <= hi; b += (unsigned long long)gridDim.x * blockDim.x) {
        const double th = (double)__uint_as_float((unsigned)b);
        const long long nt1 = clampll((floor_ll(__fma_rn(th, P.t_scale2, P.nt_half2)) + 1) >> 1, P.ntmax);
        const long long nt2 =
            clampll((floor_ll(__dadd_rn(P.nt_half2, __dmul_rn(th, P.t_scale2))) + 1) >> 1, P.ntmax);
        if (nt1 != nt2) {
            atomicAdd(bad, 1ull);
            atomicMin(first, (unsigned)b);
        }
    }
}

__global__ void k_sqrt(unsigned lo, unsigned hi, unsigned long long* bad, unsigned* first) {
    for (unsigned long long b = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         b <= hi; b += (unsigned long long)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((unsigned)b);
        if (__float_as_uint(sqrt_rn_normal(x)) != __float_as_uint(__fsqrt_rn(x))) {
            atomicAdd(bad, 1ull);
            atomicMin(first, (unsigned)b);
        }
    }
}

static Params params_for_t(int t) {
    Params P = {};
    P.t = t;
    P.ntmax = (1LL << t) - 1;
    P.npmax = 1;
    const volatile double pi = kPi;
    P.nt_half = (double)P.ntmax / 2.0;
    P.t_scale = (double)P.ntmax / (2.0 * pi);
    P.p_scale = (double)P.npmax / pi;
    P.nt_half2 = 2.0 * P.nt_half;
    P.t_scale2 = 2.0 * P.t_scale;
    return P;
}

static unsigned long long g_total_bad = 0;   // forms the kernels use
static bool g_count = true;

template <typename F>
static void run(const char* name, unsigned lo, unsigned hi, F launch) {
    unsigned long long* bad;
    unsigned* first;
    cudaMalloc(&bad, sizeof(*bad));
    cudaMalloc(&first, sizeof(*first));
    cudaMemset(bad, 0, sizeof(*bad));
    cudaMemset(first, 0xff, sizeof(*first));
    launch(lo, hi, bad, first);
    unsigned long long hbad = 0;
    unsigned hfirst = 0;
    cudaError_t e = cudaMemcpy(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost);
    cudaMemcpy(&hfirst, first, sizeof(hfirst), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("%s CUDA error %s\n", name, cudaGetErrorString(e));
        exit(2);
    }
    printf("%s checked=%llu mismatches=%llu first=0x%08x\n", name,
           (unsigned long long)hi - lo + 1, hbad, hbad ? hfirst : 0u);
    if (g_count) g_total_bad += hbad;
    cudaFree(bad);
    cudaFree(first);
}

int main() {
    const dim3 grid(148 * 16), block(256);
    const unsigned ONE = 0x3f800000u, NEG_ONE = 0xbf800000u, PI_BITS = 0x40490fdbu;  // F32(pi)
    run("atan_core[t in +0..1]", 0u, ONE, [&](unsigned lo, unsigned hi, auto bad, auto first) {
        k_atan<<<grid, block>>>(lo, hi, bad, first);
    });
    run("acos_f32[w in +0..1]", 0u, ONE, [&](unsigned lo, unsigned hi, auto bad, auto first) {
        k_acos<<<grid, block>>>(lo, hi, bad, first);
    });
    run("acos_f32[w in -0..-1]", 0x80000000u, NEG_ONE,
        [&](unsigned lo, unsigned hi, auto bad, auto first) {
            k_acos<<<grid, block>>>(lo, hi, bad, first);
        });
    // branch-free sqrt on acos_f32's argument range [2^-25, 0.25]
    run("sqrt_rn_normal[x in 2^-25..0.25]", 0x33000000u, 0x3E800000u,
        [&](unsigned lo, unsigned hi, auto bad, auto first) {
            k_sqrt<<<grid, block>>>(lo, hi, bad, first);
        });
    for (int t = 1; t <= 32; ++t) {
        // the kernels use the fused theta form only for t <= 29 (Params::theta_fma)
        g_count = t <= 29;
        char name[64];
        const Params P = params_for_t(t);
        snprintf(name, sizeof name, "theta_bucket[t=%d, th in +0..pi]", t);
        run(name, 0u, PI_BITS, [&](unsigned lo, unsigned hi, auto bad, auto first) {
            k_theta<<<grid, block>>>(lo, hi, P, bad, first);
        });
        snprintf(name, sizeof name, "theta_bucket[t=%d, th in -0..-pi]", t);
        run(name, 0x80000000u, 0x80000000u | PI_BITS,
            [&](unsigned lo, unsigned hi, auto bad, auto first) {
                k_theta<<<grid, block>>>(lo, hi, P, bad, first);
            });
    }
    printf("(widths 30..32 are reported only: the kernels keep the unfused form there)\n");
    printf("TOTAL mismatches=%llu\n", g_total_bad);
    return g_total_bad == 0 ? 0 : 1;
}
