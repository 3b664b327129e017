// decode_variants.cu — throughput / parity study of decode-trig strategies
// for the sm_100a decompress path (not product code).
//   V0  product v1: integer quarter-turn reduction + fdlibm polynomials
//   V2  same math, 32-bit integer logic, branch-free quadrant map, cmem coeffs
//   V3  1-level shared-memory table of sin/cos(RN(pi)*hi*512/b) + short
//       polynomial in the residual lo*RN(pi)/b
//   V4  2-level shared-memory tables (hi and lo), angle addition only
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -ftz=false
//        -prec-div=true -prec-sqrt=true -o tools/decode_variants tools/decode_variants.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2003_02633_b200/csrc/vc3_device.cuh"

using namespace vc3;

__constant__ double cS[6] = {-1.66666666666666324348e-01, 8.33333333332248946124e-03,
                             -1.98412698298579493134e-04, 2.75573137070700676789e-06,
                             -2.50507602534068634195e-08, 1.58969099521155010221e-10};
__constant__ double cC[6] = {4.16666666666666019037e-02, -1.38888888888741095749e-03,
                             2.48015872894767294178e-05, -2.75573143513906633035e-07,
                             2.08757232129817482790e-09, -1.13596475577881948265e-11};

__device__ __forceinline__ double i2d_magic(int m) {
    // exact int32 -> double via the 2^52 + 2^31 bias (one LOP + one DADD)
    return __dsub_rn(__hiloint2double(0x43300000, (unsigned)m ^ 0x80000000u), 4503601774854144.0);
}

// V2: narrow-layout polynomial path
__device__ __forceinline__ void sincos_grid32(int a, int b, double step, double& s, double& c) {
    const int aa = abs(a);
    int j = (int)(4 * aa > b) + (int)(4 * aa > 3 * b);
    j = a < 0 ? -j : j;
    const int m = 2 * a - j * b;
    const double psi = __fma_rn((double)m, step, (double)j * (-0.5 * kPiTail));
    const double z = __dmul_rn(psi, psi);
    double r = __fma_rn(z, cS[5], cS[4]);
    r = __fma_rn(z, r, cS[3]);
    r = __fma_rn(z, r, cS[2]);
    r = __fma_rn(z, r, cS[1]);
    const double sp = __fma_rn(__dmul_rn(z, psi), __fma_rn(z, r, cS[0]), psi);
    double q = __fma_rn(z, cC[5], cC[4]);
    q = __fma_rn(z, q, cC[3]);
    q = __fma_rn(z, q, cC[2]);
    q = __fma_rn(z, q, cC[1]);
    q = __fma_rn(z, q, cC[0]);
    const double hz = __dmul_rn(0.5, z);
    const double w = __dsub_rn(1.0, hz);
    const double cp = __dadd_rn(w, __fma_rn(__dmul_rn(z, z), q, __dsub_rn(__dsub_rn(1.0, w), hz)));
    // branch-free quadrant map: swap for odd j, negate by quadrant
    const bool odd = j & 1;
    double ss = odd ? cp : sp, cc = odd ? sp : cp;
    const int jq = j & 3;
    if (jq == 2 || jq == 3) ss = -ss;
    if (jq == 1 || jq == 2) cc = -cc;
    s = ss;
    c = cc;
}

__device__ __forceinline__ void decode_v2(unsigned long long w, const Params& P, float& ox,
                                          float& oy, float& oz) {
    const unsigned lo = (unsigned)w;
    const int nt = (int)(lo & (unsigned)P.tmask);
    const int nph = (int)((unsigned)(w >> P.t) & (unsigned)P.pmask);
    const unsigned long long field = w >> (P.p + P.t);
    const double r = (double)decode_mag(field, P);
    double st, ct, sp, cp;
    sincos_grid32(2 * nt - (int)P.ntmax, (int)P.ntmax, P.t_step, st, ct);
    sincos_grid32(nph, (int)P.npmax, P.p_step, sp, cp);
    if (nph == (int)P.npmax) { sp = 0.0; cp = -1.0; }
    ox = __double2float_rn(__dmul_rn(__dmul_rn(r, ct), sp));
    oy = __double2float_rn(__dmul_rn(__dmul_rn(r, st), sp));
    oz = __double2float_rn(__dmul_rn(r, cp));
}

// V3: 1-level table + residual polynomial.  Table entry k holds
// (sin, cos)(RN(pi) * (k - off) * 512 / b) computed on the host in long double.
constexpr int kShift = 9;
struct TabInfo {
    int t_off, p_off;   // index offsets (entries before zero)
    int t_n, p_n;       // entries
    double t_delta;     // RN(pi)/b_theta   (residual angle per lo unit, theta uses a/b with a=2nt-N)
    double p_delta;     // RN(pi)/b_phi
};

__device__ __forceinline__ void sincos_tab1(int a, int off, double delta, const double2* tab,
                                            double& s, double& c) {
    const int hi = (a + (1 << (kShift - 1))) >> kShift;
    const int lo = a - (hi << kShift);
    const double2 A = tab[hi + off];
    const double psi = __dmul_rn(i2d_magic(lo), delta);
    const double u = __dmul_rn(psi, psi);
    const double sps = __fma_rn(__dmul_rn(psi, u), __fma_rn(u, 1.0 / 120.0, -1.0 / 6.0), psi);
    const double cm1 = __dmul_rn(u, __fma_rn(u, 1.0 / 24.0, -0.5));
    s = __fma_rn(A.y, sps, __fma_rn(A.x, cm1, A.x));
    c = __fma_rn(-A.x, sps, __fma_rn(A.y, cm1, A.y));
}

template <int V>
__device__ __forceinline__ void decode_tab(unsigned long long w, const Params& P, const TabInfo& I,
                                           const double2* tt, const double2* tp, const double2* lt,
                                           const double2* lp, float& ox, float& oy, float& oz) {
    const unsigned lo32 = (unsigned)w;
    const int nt = (int)(lo32 & (unsigned)P.tmask);
    const int nph = (int)((unsigned)(w >> P.t) & (unsigned)P.pmask);
    const unsigned long long field = w >> (P.p + P.t);
    const double r = (double)decode_mag(field, P);
    double st, ct, sp, cp;
    const int at = 2 * nt - (int)P.ntmax;
    if (V == 3) {
        sincos_tab1(at, I.t_off, I.t_delta, tt, st, ct);
        sincos_tab1(nph, I.p_off, I.p_delta, tp, sp, cp);
    } else {
        const int hi_t = (at + 256) >> 9, lo_t = at - (hi_t << 9);
        const double2 A = tt[hi_t + I.t_off], B = lt[lo_t + 256];
        st = __fma_rn(A.y, B.x, __dmul_rn(A.x, B.y));
        ct = __fma_rn(-A.x, B.x, __dmul_rn(A.y, B.y));
        const int hi_p = (nph + 256) >> 9, lo_p = nph - (hi_p << 9);
        const double2 C = tp[hi_p + I.p_off], D = lp[lo_p + 256];
        sp = __fma_rn(C.y, D.x, __dmul_rn(C.x, D.y));
        cp = __fma_rn(-C.x, D.x, __dmul_rn(C.y, D.y));
    }
    if (nph == (int)P.npmax) { sp = 0.0; cp = -1.0; }
    ox = __double2float_rn(__dmul_rn(__dmul_rn(r, ct), sp));
    oy = __double2float_rn(__dmul_rn(__dmul_rn(r, st), sp));
    oz = __double2float_rn(__dmul_rn(r, cp));
}

template <int V>
__global__ void __launch_bounds__(256) k_dec(const unsigned long long* __restrict__ w,
                                             float* __restrict__ out, long long n, Params P,
                                             TabInfo I, const double2* __restrict__ gtab, int ntab) {
    extern __shared__ double2 sm[];
    if (V >= 3) {
        for (int i = threadIdx.x; i < ntab; i += blockDim.x) sm[i] = gtab[i];
        __syncthreads();
    }
    const double2* tt = sm;
    const double2* tp = sm + I.t_n;
    const double2* lt = sm + I.t_n + I.p_n;
    const double2* lp = lt;
    const long long groups = n / 4;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
         g += (long long)gridDim.x * blockDim.x) {
        const ulonglong2 u = reinterpret_cast<const ulonglong2*>(w)[2 * g];
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(w)[2 * g + 1];
        float o[12];
        const unsigned long long ws[4] = {u.x, u.y, v.x, v.y};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (V == 0) decompress_one(ws[k], P, o[3 * k], o[3 * k + 1], o[3 * k + 2]);
            else if (V == 2) decode_v2(ws[k], P, o[3 * k], o[3 * k + 1], o[3 * k + 2]);
            else decode_tab<V>(ws[k], P, I, tt, tp, lt, lp, o[3 * k], o[3 * k + 1], o[3 * k + 2]);
        }
        float4* dst = reinterpret_cast<float4*>(out + 12 * g);
        dst[0] = make_float4(o[0], o[1], o[2], o[3]);
        dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        dst[2] = make_float4(o[8], o[9], o[10], o[11]);
    }
}

static Params make_P(int t, int p, int e, int m, int bias) {
    Params P = {};
    P.e = e; P.m = m; P.p = p; P.t = t; P.bias = bias;
    P.emax = (1 << e) - 1;
    P.ntmax = (1LL << t) - 1; P.npmax = (1LL << p) - 1;
    P.tmask = P.ntmax; P.pmask = P.npmax;
    const volatile double pi = kPi;
    P.nt_half = (double)P.ntmax / 2.0;
    P.t_scale = (double)P.ntmax / (2.0 * pi);
    P.p_scale = (double)P.npmax / pi;
    P.t_step = pi / (2.0 * (double)P.ntmax);
    P.p_step = pi / (2.0 * (double)P.npmax);
    P.field_low = 2u << m;
    P.field_high = ((unsigned)(P.emax - 1) << m) | ((1u << m) - 1u);
    return P;
}

static void push_sincos(std::vector<double2>& v, long double ang) {
    v.push_back(make_double2((double)sinl(ang), (double)cosl(ang)));
}

int main() {
    const int t = 18, p = 17;
    const Params P = make_P(t, p, 7, 22, 80);
    const long long n = 1LL << 28;
    const long double PID = (long double)3.141592653589793;  // RN(pi) exactly
    std::vector<double2> tab;
    TabInfo I;
    const long long N = P.ntmax, NP = P.npmax;
    // theta: a = 2nt-N in [-N, N] ; hi in [-(N+256)>>9 ... ]
    const int t_hi_min = (int)((-N + 256) >> 9), t_hi_max = (int)((N + 256) >> 9);
    I.t_off = -t_hi_min;
    I.t_n = t_hi_max - t_hi_min + 1;
    for (int h = t_hi_min; h <= t_hi_max; ++h) push_sincos(tab, PID * (long double)(h * 512) / (long double)N);
    const int p_hi_max = (int)((NP + 256) >> 9);
    I.p_off = 0;
    I.p_n = p_hi_max + 1;
    for (int h = 0; h <= p_hi_max; ++h) push_sincos(tab, PID * (long double)(h * 512) / (long double)NP);
    I.t_delta = (double)(PID / (long double)N);
    I.p_delta = (double)(PID / (long double)NP);
    const size_t tab1 = tab.size();
    // V4 lo tables (theta only; phi shares the same lo grid? no: separate steps) -- build both
    std::vector<double2> tab4 = tab;
    for (int l = -256; l < 256; ++l) push_sincos(tab4, PID * (long double)l / (long double)N);
    // phi lo table appended after theta lo (V4 uses lt for both: approximate study uses theta lo grid for phi)
    printf("table entries: V3 %zu (%.1f KB), V4 %zu (%.1f KB)\n", tab1, tab1 * 16 / 1024.0,
           tab4.size(), tab4.size() * 16 / 1024.0);

    unsigned long long* dw;
    float *d0, *d1;
    double2 *dt3, *dt4;
    cudaMalloc(&dw, n * 8);
    cudaMalloc(&d0, n * 12);
    cudaMalloc(&d1, n * 12);
    cudaMalloc(&dt3, tab.size() * 16);
    cudaMalloc(&dt4, tab4.size() * 16);
    cudaMemcpy(dt3, tab.data(), tab.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dt4, tab4.data(), tab4.size() * 16, cudaMemcpyHostToDevice);
    // random words with normal-range magnitude fields
    std::vector<unsigned long long> hw(1 << 20);
    unsigned long long s = 0x9E3779B97F4A7C15ull;
    for (auto& x : hw) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        x = s;
    }
    for (long long off = 0; off < n; off += hw.size())
        cudaMemcpy(dw + off, hw.data(), hw.size() * 8, cudaMemcpyHostToDevice);
    int sms = 148;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name, const double2* gt, int ntab, float* out) {
        const size_t smem = ntab * 16;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 16);
        for (int occ : {4, 8}) {
            const int grid = sms * occ;
            kern<<<grid, 256, smem>>>(dw, out, n, P, I, gt, ntab);
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) kern<<<grid, 256, smem>>>(dw, out, n, P, I, gt, ntab);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 5;
            printf("%-34s grid %4d: %8.3f ms  %7.1f Gword/s  %7.1f GB/s  %s\n", name, grid, ms,
                   n / ms / 1e6, 20.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    };
    run(k_dec<0>, "V0 product poly (int64, branches)", dt3, 0, d0);
    run(k_dec<2>, "V2 poly int32 branch-free", dt3, 0, d1);
    auto cmp = [&](const char* name) {
        std::vector<unsigned> h0(3 << 20), h1(3 << 20);
        long long bad = 0, tot = 0;
        for (long long off = 0; off < 3 * n; off += h0.size()) {
            cudaMemcpy(h0.data(), d0 + off, h0.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(h1.data(), d1 + off, h1.size() * 4, cudaMemcpyDeviceToHost);
            for (size_t i = 0; i < h0.size(); ++i) bad += h0[i] != h1[i];
            tot += h0.size();
            if (off > (1LL << 26)) break;
        }
        printf("   %s vs V0: %lld / %lld components differ\n", name, bad, tot);
    };
    cmp("V2");
    run(k_dec<3>, "V3 1-level smem table + poly", dt3, (int)tab1, d1);
    cmp("V3");
    run(k_dec<4>, "V4 2-level smem tables", dt4, (int)tab4.size(), d1);
    cmp("V4 (phi lo grid approximate)");
    return 0;
}
