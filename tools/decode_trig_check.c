// Offline study: how closely do candidate GPU decode-trig algorithms reproduce
// the reference's libm sin/cos tables (/root/reference/pkg/src/vc3/_kernels.py:252-273)?
// Emulates the device arithmetic with C fma() so the same op sequence can be
// ported to CUDA bit-for-bit.  Prints ulp histograms and the resulting float32
// component mismatch rate on random magnitudes.
// gcc -O2 -ffp-contract=off -o decode_trig_check decode_trig_check.c -lm
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double PI_ = 3.141592653589793;

// fdlibm-style kernels on |x| <= pi/4 (coefficients re-derived below by fit check)
static const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                    S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                    S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
static const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                    C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                    C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;

static inline void ksincos(double x, double* s, double* c) {
    double z = x * x;
    double r = fma(z, fma(z, fma(z, fma(z, S6, S5), S4), S3), S2);
    double v = z * x;
    *s = fma(v, fma(z, r, S1), x);
    double q = fma(z, fma(z, fma(z, fma(z, fma(z, C6, C5), C4), C3), C2), C1);
    // cos = 1 - z/2 + z^2 q ; evaluate as w + ((1-w) - hz + z*z*q) for accuracy
    double hz = 0.5 * z;
    double w = 1.0 - hz;
    *c = w + fma(z * z, q, (1.0 - w) - hz);
}

static const double PIO2_HI = 1.5707963267948966;         // RN(pi/2)
static const double PIO2_LO = 6.123233995736766e-17;      // RN(pi/2 - PIO2_HI)
static const double PI_RES = 1.2246467991473532e-16;      // pi - RN(pi)

// Variant A: integer-domain reduction of alpha = pi_d * a / b  (b > 0)
static void sincos_grid_int(int64_t a, int64_t b, double* s, double* c) {
    int64_t aa = a < 0 ? -a : a;
    int j = (4 * aa > b) + (4 * aa > 3 * b);
    if (a < 0) j = -j;
    int64_t m = 2 * a - (int64_t)j * b;
    double C1g = PI_ / (2.0 * (double)b);
    // alpha - j*pi/2 = pi_d*m/(2b) - j*(pi - pi_d)/2
    double psi = fma((double)m, C1g, -(double)j * (PI_RES * 0.5));
    double sp, cp;
    ksincos(psi, &sp, &cp);
    switch (j & 3) {
        case 0: *s = sp; *c = cp; break;
        case 1: *s = cp; *c = -sp; break;
        case 2: *s = -sp; *c = -cp; break;
        default: *s = -cp; *c = sp; break;
    }
}

// correctly rounded x/b for integers via reciprocal + fma correction (Markstein)
static inline double div_cr(double x, double b, double rb) {
    double q0 = x * rb;
    double r = fma(-q0, b, x);
    return fma(r, rb, q0);
}

// Variant B: reproduce the reference's double angle exactly, then Cody-Waite.
static void sincos_ref_angle(double ang, int j, double* s, double* c) {
    double d = fma(-(double)j, PIO2_HI, ang);
    double psi = fma(-(double)j, PIO2_LO, d);
    double sp, cp;
    ksincos(psi, &sp, &cp);
    switch (j & 3) {
        case 0: *s = sp; *c = cp; break;
        case 1: *s = cp; *c = -sp; break;
        case 2: *s = -sp; *c = -cp; break;
        default: *s = -cp; *c = sp; break;
    }
}

static int64_t ulpdiff(double a, double b) {
    if (a == b) return 0;
    int64_t ia, ib;
    memcpy(&ia, &a, 8); memcpy(&ib, &b, 8);
    if (ia < 0) ia = INT64_MIN - ia;
    if (ib < 0) ib = INT64_MIN - ib;
    int64_t d = ia - ib;
    return d < 0 ? -d : d;
}

typedef struct { int64_t h[6]; int64_t max; double maxrel; } hist_t;
static void hadd(hist_t* H, double got, double ref) {
    int64_t u = ulpdiff(got, ref);
    int k = u == 0 ? 0 : u == 1 ? 1 : u == 2 ? 2 : u <= 16 ? 3 : u <= 1 << 20 ? 4 : 5;
    H->h[k]++;
    if (u > H->max) H->max = u;
    double rel = ref != 0 ? fabs(got - ref) / fabs(ref) : fabs(got);
    if (rel > H->maxrel) H->maxrel = rel;
}
static void hprint(const char* name, hist_t* H) {
    printf("  %-26s 0ulp %lld  1ulp %lld  2ulp %lld  <=16 %lld  <=2^20 %lld  more %lld  max %lld  maxrel %.3g\n",
           name, (long long)H->h[0], (long long)H->h[1], (long long)H->h[2], (long long)H->h[3],
           (long long)H->h[4], (long long)H->h[5], (long long)H->max, H->maxrel);
}

// Variant C: 1-level table + residual polynomial (the product decode).
// Table entry for hi: (sin, cos)(RN(pi) * hi * 2^sh / b), evaluated in long double
// after an exact quarter-turn reduction (so entries near zero crossings keep
// full relative accuracy).  theta endpoints are special-cased by the caller.
static void sincos_ld(int64_t k, int64_t b, double* s, double* c) {
    // alpha = pi_d * k / b ; j = round(2k/b) ; residual = pi_d*(2k - j b)/(2b) - j*(pi - pi_d)/2
    const long double PID = (long double)PI_;
    const long double TAIL = 1.2246467991473531772e-16L;  // pi - RN(pi)
    int64_t ak = k < 0 ? -k : k;
    int64_t j = (4 * ak + b) / (2 * b);  // round(2|k|/b)
    if (k < 0) j = -j;
    int64_t m = 2 * k - j * b;
    long double psi = PID * (long double)m / (2.0L * (long double)b) - (long double)j * TAIL / 2.0L;
    long double sp = sinl(psi), cp = cosl(psi);
    long double ss, cc;
    switch (((j % 4) + 4) % 4) {
        case 0: ss = sp; cc = cp; break;
        case 1: ss = cp; cc = -sp; break;
        case 2: ss = -sp; cc = -cp; break;
        default: ss = -cp; cc = sp; break;
    }
    *s = (double)ss; *c = (double)cc;
}

static void sincos_tab1(int64_t a, int64_t b, int sh, double* s, double* c) {
    const long double PID = (long double)PI_;
    int64_t half = sh ? (1LL << (sh - 1)) : 0;
    int64_t hi = (a + half) >> sh, lo = a - (hi << sh);
    double sA, cA;
    sincos_ld(hi << sh, b, &sA, &cA);
    double delta = (double)(PID / (long double)b);
    double psi = (double)lo * delta;
    double u = psi * psi;
    double sps = fma(psi * u, fma(u, 1.0 / 120.0, -1.0 / 6.0), psi);
    double cm1 = u * fma(u, 1.0 / 24.0, -0.5);
    *s = fma(cA, sps, fma(sA, cm1, sA));
    *c = fma(-sA, sps, fma(cA, cm1, cA));
}

// Variant D (product since round 1b): plain bit split, index = n >> sh,
// residual = n & (2^sh - 1) >= 0.  theta entry h: RN(pi)*(2h*2^sh - N)/N,
// residual angle lo*RN(2 RN(pi)/N); phi entry h: RN(pi)*h*2^sh/NP.
static void sincos_tabD(int64_t k_entry, int64_t b, int64_t lo, double delta, double* s, double* c) {
    double sA, cA;
    sincos_ld(k_entry, b, &sA, &cA);
    double psi = (double)lo * delta;
    double u = psi * psi;
    double sps = fma(psi * u, fma(u, 1.0 / 120.0, -1.0 / 6.0), psi);
    double cm1 = u * fma(u, 1.0 / 24.0, -0.5);
    *s = fma(cA, sps, fma(sA, cm1, sA));
    *c = fma(-sA, sps, fma(cA, cm1, cA));
}

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t rng(void) { rng_state ^= rng_state << 13; rng_state ^= rng_state >> 7; rng_state ^= rng_state << 17; return rng_state; }

static int e2e(void) {
    const int t = 18, p = 17;
    const int64_t N = (1LL << t) - 1, NP = (1LL << p) - 1;
    double *st = malloc(8 * (N + 1)), *ct = malloc(8 * (N + 1)), *sp = malloc(8 * (NP + 1)), *cp = malloc(8 * (NP + 1));
    for (int64_t n = 0; n <= N; ++n) { double th = PI_ * (2.0 * (double)n / (double)N - 1.0); st[n] = sin(th); ct[n] = cos(th); }
    for (int64_t n = 0; n <= NP; ++n) { double ph = PI_ * (double)n / (double)NP; sp[n] = sin(ph); cp[n] = cos(ph); }
    sp[NP] = 0.0; cp[NP] = -1.0;
    double rN = 1.0 / (double)N, rNP = 1.0 / (double)NP;
    int64_t total = 0, misA = 0, misB = 0, misC = 0, misD = 0;
    for (int64_t i = 0; i < 20000000; ++i) {
        if ((i & 3) == 0) { /* force endpoints sometimes */ }
        uint64_t w = rng();
        int64_t nt = w & N, nph = (w >> t) & NP;
        uint32_t mant = (uint32_t)(w >> 40) & 0x7fffff;
        float r = 0; uint32_t rb = (127u << 23) | mant; memcpy(&r, &rb, 4);
        double R = r;
        float ref[3] = {(float)(R * ct[nt] * sp[nph]), (float)(R * st[nt] * sp[nph]), (float)(R * cp[nph])};
        double sA, cA, spA, cpA, sB, cB, spB, cpB;
        sincos_grid_int(2 * nt - N, N, &sA, &cA);
        if (nph == NP) { spA = 0; cpA = -1; } else sincos_grid_int(nph, NP, &spA, &cpA);
        double q = div_cr(2.0 * (double)nt, (double)N, rN);
        int64_t a = 2 * nt - N, aa = a < 0 ? -a : a;
        int j = (4 * aa > N) + (4 * aa > 3 * N); if (a < 0) j = -j;
        sincos_ref_angle(PI_ * (q - 1.0), j, &sB, &cB);
        if (nph == NP) { spB = 0; cpB = -1; }
        else { double qp = div_cr(PI_ * (double)nph, (double)NP, rNP); int jp = (4 * nph > NP) + (4 * nph > 3 * NP); sincos_ref_angle(qp, jp, &spB, &cpB); }
        double sC, cC, spC, cpC;
        sincos_tab1(2 * nt - N, N, 9, &sC, &cC);
        if (nt == 0) { sC = -1.2246467991473532e-16; cC = -1.0; }
        if (nt == N) { sC = 1.2246467991473532e-16; cC = -1.0; }
        if (nph == NP) { spC = 0; cpC = -1; } else sincos_tab1(nph, NP, 9, &spC, &cpC);
        float C[3] = {(float)(R * cC * spC), (float)(R * sC * spC), (float)(R * cpC)};
        for (int k = 0; k < 3; ++k) misC += C[k] != ref[k];
        {
            double sD, cD, spD, cpD;
            const double dt2 = (double)(2.0L * (long double)PI_ / (long double)N), dp = (double)((long double)PI_ / (long double)NP);
            if (nt == N) { sD = 1.2246467991473532e-16; cD = -1.0; }
            else sincos_tabD(2 * ((nt >> 7) << 7) - N, N, nt & 127, dt2, &sD, &cD);
            if (nph == NP) { spD = 0; cpD = -1; }
            else sincos_tabD((nph >> 7) << 7, NP, nph & 127, dp, &spD, &cpD);
            float D[3] = {(float)(R * cD * spD), (float)(R * sD * spD), (float)(R * cpD)};
            for (int k = 0; k < 3; ++k) misD += D[k] != ref[k];
        }
        float A[3] = {(float)(R * cA * spA), (float)(R * sA * spA), (float)(R * cpA)};
        float B[3] = {(float)(R * cB * spB), (float)(R * sB * spB), (float)(R * cpB)};
        for (int k = 0; k < 3; ++k) {
            total++;
            int64_t dA = ulpdiff(A[k], ref[k]), dB = ulpdiff(B[k], ref[k]);
            if (A[k] != ref[k]) { misA++; }
            if (B[k] != ref[k]) { misB++; }
            (void)dA; (void)dB;
        }
    }
    printf("variant C (table) mismatches %lld, variant D (plain split table) %lld\n", (long long)misC, (long long)misD);
    printf("components %lld: variant A mismatches %lld (%.3g), variant B mismatches %lld (%.3g)\n",
           (long long)total, (long long)misA, (double)misA / total, (long long)misB, (double)misB / total);
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1) return e2e();
    int layouts[][2] = {{18, 17}, {16, 16}, {17, 16}, {17, 17}, {25, 10}, {8, 8}, {3, 2}};
    for (int li = 0; li < 7; ++li) {
        int t = layouts[li][0], p = layouts[li][1];
        int64_t N = (1LL << t) - 1, NP = (1LL << p) - 1;
        printf("layout t=%d p=%d\n", t, p);
        hist_t hsA = {0}, hcA = {0}, hsB = {0}, hcB = {0}, hdiv = {0};
        double rN = 1.0 / (double)N, rNP = 1.0 / (double)NP;
        int64_t divbad = 0, divbad_p = 0;
        for (int64_t n = 0; n <= N; ++n) {
            double th = PI_ * (2.0 * (double)n / (double)N - 1.0);
            double rs = sin(th), rc = cos(th);
            double s, c;
            sincos_grid_int(2 * n - N, N, &s, &c);
            hadd(&hsA, s, rs); hadd(&hcA, c, rc);
            double q = div_cr(2.0 * (double)n, (double)N, rN);
            if (q != 2.0 * (double)n / (double)N) divbad++;
            double ang = PI_ * (q - 1.0);
            int64_t a = 2 * n - N, aa = a < 0 ? -a : a;
            int j = (4 * aa > N) + (4 * aa > 3 * N);
            if (a < 0) j = -j;
            sincos_ref_angle(ang, j, &s, &c);
            hadd(&hsB, s, rs); hadd(&hcB, c, rc);
        }
        printf(" theta (%lld entries), div_cr mismatches %lld\n", (long long)(N + 1), (long long)divbad);
        {
            hist_t hs = {0}, hc = {0};
            int shown = 0;
            for (int64_t n = 0; n <= N; ++n) {
                double th = PI_ * (2.0 * (double)n / (double)N - 1.0);
                double rs = sin(th), rc = cos(th), s2, c2;
                sincos_tab1(2 * n - N, N, t > 9 ? t - 9 : 0, &s2, &c2);
                if (n == 0) { s2 = -1.2246467991473532e-16; c2 = -1.0; }
                if (n == N) { s2 = 1.2246467991473532e-16; c2 = -1.0; }
                hadd(&hs, s2, rs); hadd(&hc, c2, rc);
                if ((ulpdiff(s2, rs) > 4 || ulpdiff(c2, rc) > 4) && shown < 6) {
                    printf("    n=%lld a=%lld sin ref %.17g got %.17g (%lld ulp) cos ref %.17g got %.17g (%lld ulp)\n", (long long)n, (long long)(2*n-N), rs, s2, (long long)ulpdiff(s2, rs), rc, c2, (long long)ulpdiff(c2, rc));
                    shown++;
                }
            }
            hprint("C table1 sin", &hs); hprint("C table1 cos", &hc);
        }
        {
            hist_t hs = {0}, hc = {0};
            const int sh = t > 11 ? t - 11 : 0;
            const double dlt = (double)(2.0L * (long double)PI_ / (long double)N);
            for (int64_t n = 0; n <= N; ++n) {
                double th = PI_ * (2.0 * (double)n / (double)N - 1.0);
                double s2, c2;
                if (n == N) { s2 = 1.2246467991473532e-16; c2 = -1.0; }
                else {
                    int64_t hi = n >> sh, lo = n & ((1LL << sh) - 1);
                    sincos_tabD(2 * (hi << sh) - N, N, lo, dlt, &s2, &c2);
                }
                hadd(&hs, s2, sin(th)); hadd(&hc, c2, cos(th));
            }
            hprint("D theta sin", &hs); hprint("D theta cos", &hc);
        }
        hprint("A int-reduce sin", &hsA); hprint("A int-reduce cos", &hcA);
        hprint("B ref-angle sin", &hsB); hprint("B ref-angle cos", &hcB);
        hist_t psA = {0}, pcA = {0}, psB = {0}, pcB = {0};
        for (int64_t n = 0; n < NP; ++n) {  // endpoint forced separately
            double ph = PI_ * (double)n / (double)NP;
            double rs = sin(ph), rc = cos(ph);
            double s, c;
            sincos_grid_int(n, NP, &s, &c);
            hadd(&psA, s, rs); hadd(&pcA, c, rc);
            double q = div_cr(PI_ * (double)n, (double)NP, rNP);
            if (q != ph) divbad_p++;
            int j = (4 * n > NP) + (4 * n > 3 * NP);
            sincos_ref_angle(q, j, &s, &c);
            hadd(&psB, s, rs); hadd(&pcB, c, rc);
        }
        printf(" phi (%lld entries), div_cr mismatches %lld\n", (long long)NP, (long long)divbad_p);
        {
            hist_t hs = {0}, hc = {0};
            for (int64_t n = 0; n < NP; ++n) {
                double ph = PI_ * (double)n / (double)NP;
                double s2, c2;
                sincos_tab1(n, NP, p > 9 ? p - 9 : 0, &s2, &c2);
                hadd(&hs, s2, sin(ph)); hadd(&hc, c2, cos(ph));
            }
            hprint("C table1 sin", &hs); hprint("C table1 cos", &hc);
        }
        hprint("A int-reduce sin", &psA); hprint("A int-reduce cos", &pcA);
        hprint("B ref-angle sin", &psB); hprint("B ref-angle cos", &pcB);
    }
    return 0;
}

// ---- end-to-end component mismatch rate on random words (default layout) ----
// build with -DE2E to run instead of the table study
