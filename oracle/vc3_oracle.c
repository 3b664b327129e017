/*
 * vc3_oracle.c — CPU restatement of the reference codec's numeric core.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline timed by bench.py (cpu_baseline leg and
 * `--impl reference`).  Only tests/, __graft_entry__.smoke() and bench.py may
 * load it.  The product library (paper_2003_02633_b200/csrc) never links it.
 *
 * It restates /root/reference/pkg/src/vc3/_kernels.py (numba @njit, no fast
 * math, no FMA contraction) in plain C99 compiled with -ffp-contract=off, so
 * every float32/float64 operation rounds exactly where the numba code rounds.
 * Double-precision trig goes through the host libm, as numba's does
 * (`math.atan2`, `math.acos`, `math.sin`, `math.cos` lower to libm calls).
 *
 * Pinned against the reference: the fixtures in tests/golden were produced by importing
 * the reference package (tests/golden/make_golden.py) and tests/test_oracle.py
 * checks this file against them bit for bit.
 *
 * Batch entry points take an `nthreads` argument and split the index range
 * into contiguous chunks over pthreads (the reference runs one thread; the
 * per-element results do not depend on the split).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef float F32;
static const double PI_ = 3.141592653589793;    /* _kernels.py:18 */
static const double PI_2_ = 1.5707963267948966;  /* _kernels.py:19 */

/* _trig.py:16-25 */
static const double ATAN_Q[8] = {
    -0x1.5554ee890806fp-2, 0x1.997b7924aa8f1p-3, -0x1.231c3e32e0e58p-3,
    0x1.b55760bdb2d66p-4, -0x1.36309347af22dp-4, 0x1.63b9fa6a62bfdp-5,
    -0x1.0e02eab0b70f2p-6, 0x1.81fc37099279bp-9,
};
/* _trig.py:28-34 */
static const double ASIN_Q[5] = {
    0x1.5555bd6f47f8dp-3, 0x1.330560cdcb21cp-4, 0x1.742c47410ba97p-5,
    0x1.8f2b9cb95b714p-6, 0x1.56eddb3a21eebp-5,
};

/* _kernels.py:23-28 — Horner, q = q*z + C[i] (two roundings per step) */
static inline double atan_q(double z) {
    double q = ATAN_Q[7];
    for (int i = 6; i >= 0; --i) q = q * z + ATAN_Q[i];
    return q;
}

/* _kernels.py:31-36 */
static inline double asin_q(double z) {
    double q = ASIN_Q[4];
    for (int i = 3; i >= 0; --i) q = q * z + ASIN_Q[i];
    return q;
}

/* _kernels.py:39-61 */
F32 vc3o_atan2_f32(F32 y, F32 x) {
    F32 ax = fabsf(x), ay = fabsf(y);
    F32 hi = ax > ay ? ax : ay;
    F32 lo = ax > ay ? ay : ax;
    F32 t = hi > 0.0f ? lo / hi : 0.0f;
    double td = (double)t;
    double z = td * td;
    F32 a = (F32)(td + td * z * atan_q(z));
    if (ay > ax) a = (F32)PI_2_ - a;
    if (x < 0.0f) a = (F32)PI_ - a;
    if (y < 0.0f) a = -a;
    if (y == 0.0f) a = x < 0.0f ? (F32)PI_ : 0.0f;
    return a;
}

/* _kernels.py:64-80 */
F32 vc3o_acos_f32(F32 w) {
    F32 aw = fabsf(w);
    if (aw <= 0.5f) {
        F32 z32 = w * w;
        double xd = (double)w, z = (double)z32;
        double asn = xd + xd * z * asin_q(z);
        return (F32)(PI_2_ - asn);
    }
    F32 zs = (1.0f - aw) * 0.5f;
    F32 xs = (F32)sqrt((double)zs);
    double xd = (double)xs, z = (double)zs;
    double asn = xd + xd * z * asin_q(z);
    F32 big = (F32)(2.0 * asn);
    return w > 0.0f ? big : (F32)PI_ - big;
}

/* _kernels.py:83-86 — ceil(floor(2x)/2) */
static inline int64_t nint_f64(double x) { return (int64_t)ceil(floor(2.0 * x) / 2.0); }

/* _kernels.py:89-126; returns r64, writes theta/phi */
static inline double spherical(F32 x, F32 y, F32 z, int theta_single, int phi_single,
                               double* th_out, double* ph_out) {
    double xd = x, yd = y, zd = z;
    double r64 = sqrt(xd * xd + yd * yd + zd * zd);
    if (r64 == 0.0) { *th_out = 0.0; *ph_out = 0.0; return 0.0; }
    double th, ph;
    if (theta_single) th = (double)vc3o_atan2_f32(y, x);
    else th = atan2(yd, xd);
    if (phi_single) {
        F32 s = (x * x + y * y) + z * z;
        F32 rq = (F32)sqrt((double)s);
        F32 w;
        if (rq > 0.0f) {
            w = z / rq;
            if (w > 1.0f) w = 1.0f;
            if (w < -1.0f) w = -1.0f;
        } else {
            w = 1.0f;
        }
        ph = (double)vc3o_acos_f32(w);
    } else {
        double w64 = zd / r64;
        if (w64 > 1.0) w64 = 1.0;
        if (w64 < -1.0) w64 = -1.0;
        ph = acos(w64);
    }
    *th_out = th;
    *ph_out = ph;
    return r64;
}

/* _kernels.py:129-147 */
static inline void quantize(double th, double ph, int64_t ntmax, int64_t npmax, int quant_single,
                            int64_t* nt_out, int64_t* nph_out) {
    if (quant_single) { th = (double)(F32)th; ph = (double)(F32)ph; }
    double vt = (double)ntmax / 2.0 + th * ((double)ntmax / (2.0 * PI_));
    double vp = ph * ((double)npmax / PI_);
    int64_t nt = nint_f64(vt), nph = nint_f64(vp);
    if (nt < 0) nt = 0;
    if (nt > ntmax) nt = ntmax;
    if (nph < 0) nph = 0;
    if (nph > npmax) nph = npmax;
    *nt_out = nt;
    *nph_out = nph;
}

static inline uint32_t f2u(F32 f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline F32 u2f(uint32_t u) { F32 f; memcpy(&f, &u, 4); return f; }

/* _kernels.py:150-175 */
int64_t vc3o_encode_mag(double r64, int e_bits, int m_bits, int bias) {
    if (r64 == 0.0) return 0;
    F32 r32 = (F32)r64;
    if ((double)r32 < r64) r32 = nextafterf(r32, INFINITY);
    int64_t u = (int64_t)f2u(r32);
    int64_t e8 = (u >> 23) & 0xFF;
    int64_t tail = u & 0x7FFFFF;
    int64_t e7 = e8 - 127 + bias;
    int64_t emax = ((int64_t)1 << e_bits) - 1;
    if (e7 <= 1) return (int64_t)2 << m_bits;
    if (e7 >= emax) return ((emax - 1) << m_bits) | (((int64_t)1 << m_bits) - 1);
    return (e7 << m_bits) | (tail >> (23 - m_bits));
}

/* _kernels.py:178-195 */
F32 vc3o_decode_mag(int64_t field, int e_bits, int m_bits, int bias) {
    if (field == 0) return 0.0f;
    int64_t e7 = (field >> m_bits) & (((int64_t)1 << e_bits) - 1);
    int64_t mant = field & (((int64_t)1 << m_bits) - 1);
    int64_t e8 = e7 - bias + 127;
    if (e8 < 0) e8 = 0;
    if (e8 > 254) e8 = 254;
    return u2f((uint32_t)((e8 << 23) | (mant << (23 - m_bits))));
}

typedef struct { int e, m, p, t, bias; } lay_t;

/* _kernels.py:198-212 */
static inline uint64_t compress_one(F32 x, F32 y, F32 z, lay_t L, int ts, int ps, int qs) {
    double th, ph;
    double r64 = spherical(x, y, z, ts, ps, &th, &ph);
    if (r64 == 0.0) return 0;
    int64_t ntmax = ((int64_t)1 << L.t) - 1, npmax = ((int64_t)1 << L.p) - 1;
    int64_t nt, nph;
    quantize(th, ph, ntmax, npmax, qs, &nt, &nph);
    int64_t field = vc3o_encode_mag(r64, L.e, L.m, L.bias);
    return ((uint64_t)field << (L.p + L.t)) | ((uint64_t)nph << L.t) | (uint64_t)nt;
}

/* _kernels.py:252-273 — sin/cos of every reconstructed angle (libm) */
typedef struct { int t, p; double *sin_t, *cos_t, *sin_p, *cos_p; } tables_t;

static void build_tables(tables_t* T, int t, int p) {
    int64_t ntmax = ((int64_t)1 << t) - 1, npmax = ((int64_t)1 << p) - 1;
    T->t = t; T->p = p;
    T->sin_t = (double*)malloc(sizeof(double) * (ntmax + 1));
    T->cos_t = (double*)malloc(sizeof(double) * (ntmax + 1));
    T->sin_p = (double*)malloc(sizeof(double) * (npmax + 1));
    T->cos_p = (double*)malloc(sizeof(double) * (npmax + 1));
    for (int64_t n = 0; n <= ntmax; ++n) {
        double th = PI_ * (2.0 * (double)n / (double)ntmax - 1.0);
        T->sin_t[n] = sin(th);
        T->cos_t[n] = cos(th);
    }
    for (int64_t n = 0; n <= npmax; ++n) {
        double ph = PI_ * (double)n / (double)npmax;
        T->sin_p[n] = sin(ph);
        T->cos_p[n] = cos(ph);
    }
    T->sin_p[npmax] = 0.0;
    T->cos_p[npmax] = -1.0;
}

/* One cached table set (the reference caches per (t, p), codec.py:42,51-63). */
static pthread_mutex_t g_tab_mu = PTHREAD_MUTEX_INITIALIZER;
static tables_t g_tab = {0, 0, 0, 0, 0, 0};

static const tables_t* get_tables(int t, int p) {
    pthread_mutex_lock(&g_tab_mu);
    if (!g_tab.sin_t || g_tab.t != t || g_tab.p != p) {
        free(g_tab.sin_t); free(g_tab.cos_t); free(g_tab.sin_p); free(g_tab.cos_p);
        build_tables(&g_tab, t, p);
    }
    pthread_mutex_unlock(&g_tab_mu);
    return &g_tab;
}

/* codec.py:39-40,66-67 */
static int has_tables(int t, int p) { return ((1LL << t) + (1LL << p)) <= (1LL << 21); }

/* _kernels.py:276-290 */
static inline void decompress_one_tab(uint64_t w, lay_t L, const tables_t* T, F32* o) {
    uint64_t tmask = ((uint64_t)1 << L.t) - 1, pmask = ((uint64_t)1 << L.p) - 1;
    int64_t nt = (int64_t)(w & tmask);
    int64_t nph = (int64_t)((w >> L.t) & pmask);
    int64_t field = (int64_t)(w >> (L.p + L.t));
    if (field == 0) { o[0] = o[1] = o[2] = 0.0f; return; }
    double r = (double)vc3o_decode_mag(field, L.e, L.m, L.bias);
    o[0] = (F32)(r * T->cos_t[nt] * T->sin_p[nph]);
    o[1] = (F32)(r * T->sin_t[nt] * T->sin_p[nph]);
    o[2] = (F32)(r * T->cos_p[nph]);
}

/* _kernels.py:304-331 */
static inline void decompress_one_direct(uint64_t w, lay_t L, F32* o) {
    uint64_t tmask = ((uint64_t)1 << L.t) - 1, pmask = ((uint64_t)1 << L.p) - 1;
    int64_t ntmax = ((int64_t)1 << L.t) - 1, npmax = ((int64_t)1 << L.p) - 1;
    int64_t nt = (int64_t)(w & tmask);
    int64_t nph = (int64_t)((w >> L.t) & pmask);
    int64_t field = (int64_t)(w >> (L.p + L.t));
    if (field == 0) { o[0] = o[1] = o[2] = 0.0f; return; }
    double r = (double)vc3o_decode_mag(field, L.e, L.m, L.bias);
    double th = PI_ * (2.0 * (double)nt / (double)ntmax - 1.0);
    double ph = PI_ * (double)nph / (double)npmax;
    double st = sin(th), ct = cos(th), sp, cp;
    if (nph == npmax) { sp = 0.0; cp = -1.0; }
    else { sp = sin(ph); cp = cos(ph); }
    o[0] = (F32)(r * ct * sp);
    o[1] = (F32)(r * st * sp);
    o[2] = (F32)(r * cp);
}

static inline void decompress_one(uint64_t w, lay_t L, const tables_t* T, F32* o) {
    if (T) decompress_one_tab(w, L, T, o);
    else decompress_one_direct(w, L, o);
}

/* ---- batch drivers (contiguous chunks over pthreads) ---------------------- */

typedef struct {
    int op;
    int64_t lo, hi;
    const void *a, *b, *c;
    void* out;
    void* out2;
    lay_t L;
    int ts, ps, qs;
    const tables_t* T;
    float alpha;
} job_t;

enum { OP_COMPRESS, OP_DECOMPRESS, OP_ADD, OP_ADD_RAW, OP_AXPY, OP_RK };

static void run_range(job_t* j) {
    const lay_t L = j->L;
    switch (j->op) {
    case OP_COMPRESS: {
        const F32* v = (const F32*)j->a;
        uint64_t* o = (uint64_t*)j->out;
        for (int64_t i = j->lo; i < j->hi; ++i)
            o[i] = compress_one(v[3 * i], v[3 * i + 1], v[3 * i + 2], L, j->ts, j->ps, j->qs);
        break;
    }
    case OP_DECOMPRESS: {
        const uint64_t* w = (const uint64_t*)j->a;
        F32* o = (F32*)j->out;
        for (int64_t i = j->lo; i < j->hi; ++i) decompress_one(w[i], L, j->T, o + 3 * i);
        break;
    }
    case OP_ADD: { /* _kernels.py:348-359 */
        const uint64_t *a = (const uint64_t*)j->a, *b = (const uint64_t*)j->b;
        uint64_t* c = (uint64_t*)j->out;
        for (int64_t i = j->lo; i < j->hi; ++i) {
            F32 p[3], q[3];
            decompress_one(a[i], L, j->T, p);
            decompress_one(b[i], L, j->T, q);
            c[i] = compress_one(p[0] + q[0], p[1] + q[1], p[2] + q[2], L, j->ts, j->ps, j->qs);
        }
        break;
    }
    case OP_ADD_RAW: { /* _kernels.py:341-345 (flat float32) */
        const F32 *a = (const F32*)j->a, *b = (const F32*)j->b;
        F32* c = (F32*)j->out;
        for (int64_t i = j->lo; i < j->hi; ++i) c[i] = a[i] + b[i];
        break;
    }
    case OP_AXPY: { /* composition oracle for y <- compress(alpha*decode(x) + decode(y)) */
        const uint64_t *x = (const uint64_t*)j->a, *y = (const uint64_t*)j->b;
        uint64_t* o = (uint64_t*)j->out;
        const F32 al = j->alpha;
        for (int64_t i = j->lo; i < j->hi; ++i) {
            F32 p[3], q[3];
            decompress_one(x[i], L, j->T, p);
            decompress_one(y[i], L, j->T, q);
            o[i] = compress_one(al * p[0] + q[0], al * p[1] + q[1], al * p[2] + q[2],
                                L, j->ts, j->ps, j->qs);
        }
        break;
    }
    }
}

static void* thread_main(void* arg) { run_range((job_t*)arg); return NULL; }

static void run_parallel(job_t proto, int64_t n, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
    if (nthreads == 1) { proto.lo = 0; proto.hi = n; run_range(&proto); return; }
    pthread_t th[256];
    job_t jobs[256];
    int64_t per = (n + nthreads - 1) / nthreads;
    for (int k = 0; k < nthreads; ++k) {
        jobs[k] = proto;
        jobs[k].lo = (int64_t)k * per < n ? (int64_t)k * per : n;
        jobs[k].hi = (int64_t)(k + 1) * per < n ? (int64_t)(k + 1) * per : n;
        pthread_create(&th[k], NULL, thread_main, &jobs[k]);
    }
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
}

static lay_t mk(int e, int m, int p, int t, int bias) { lay_t L = {e, m, p, t, bias}; return L; }

/* ---- exported API ---------------------------------------------------------- */

/* codec.py:189-202 / _kernels.py:215-220 ; array-of-structs float32 input */
void vc3o_compress(const float* xyz, uint64_t* out, int64_t n, int e, int m, int p, int t,
                   int bias, int ts, int ps, int qs, int nthreads) {
    job_t j; memset(&j, 0, sizeof j);
    j.op = OP_COMPRESS; j.a = xyz; j.out = out; j.L = mk(e, m, p, t, bias);
    j.ts = ts; j.ps = ps; j.qs = qs;
    run_parallel(j, n, nthreads);
}

/* codec.py:205-228 ; array-of-structs float32 output */
void vc3o_decompress(const uint64_t* w, float* xyz, int64_t n, int e, int m, int p, int t,
                     int bias, int nthreads) {
    job_t j; memset(&j, 0, sizeof j);
    j.op = OP_DECOMPRESS; j.a = w; j.out = xyz; j.L = mk(e, m, p, t, bias);
    j.T = has_tables(t, p) ? get_tables(t, p) : NULL;
    run_parallel(j, n, nthreads);
}

/* bench.py:41-69 / _kernels.py:348-359 (the reference's wide-layout fallback
 * composes the batch codec, which is the same per-element arithmetic) */
void vc3o_add_compressed(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n, int e,
                         int m, int p, int t, int bias, int ts, int ps, int qs, int nthreads) {
    job_t j; memset(&j, 0, sizeof j);
    j.op = OP_ADD; j.a = a; j.b = b; j.out = c; j.L = mk(e, m, p, t, bias);
    j.ts = ts; j.ps = ps; j.qs = qs;
    j.T = has_tables(t, p) ? get_tables(t, p) : NULL;
    run_parallel(j, n, nthreads);
}

/* bench.py:30-38 / _kernels.py:341-345 ; n_floats = 3 * n_vectors */
void vc3o_add_raw(const float* a, const float* b, float* c, int64_t n_floats, int nthreads) {
    job_t j; memset(&j, 0, sizeof j);
    j.op = OP_ADD_RAW; j.a = a; j.b = b; j.out = c;
    run_parallel(j, n_floats, nthreads);
}

/* No reference symbol: y <- compress(alpha*decompress(x) + decompress(y)),
 * float32 ops in the order written (a multiply then an add, two roundings). */
void vc3o_axpy(float alpha, const uint64_t* x, const uint64_t* y, uint64_t* out, int64_t n,
               int e, int m, int p, int t, int bias, int ts, int ps, int qs, int nthreads) {
    job_t j; memset(&j, 0, sizeof j);
    j.op = OP_AXPY; j.a = x; j.b = y; j.out = out; j.L = mk(e, m, p, t, bias);
    j.ts = ts; j.ps = ps; j.qs = qs; j.alpha = alpha;
    j.T = has_tables(t, p) ? get_tables(t, p) : NULL;
    run_parallel(j, n, nthreads);
}

/* pieces: codec.py:99-186 */
void vc3o_spherical(const float* xyz, double* r, double* th, double* ph, int64_t n, int ts,
                    int ps) {
    for (int64_t i = 0; i < n; ++i)
        r[i] = spherical(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], ts, ps, &th[i], &ph[i]);
}

void vc3o_quantize(const double* th, const double* ph, int64_t* nt, int64_t* nph, int64_t n,
                   int64_t ntmax, int64_t npmax, int qs) {
    for (int64_t i = 0; i < n; ++i) quantize(th[i], ph[i], ntmax, npmax, qs, &nt[i], &nph[i]);
}

void vc3o_encode_mag_batch(const double* r, int64_t* out, int64_t n, int e, int m, int bias) {
    for (int64_t i = 0; i < n; ++i) out[i] = vc3o_encode_mag(r[i], e, m, bias);
}

void vc3o_decode_mag_batch(const int64_t* f, float* out, int64_t n, int e, int m, int bias) {
    for (int64_t i = 0; i < n; ++i) out[i] = vc3o_decode_mag(f[i], e, m, bias);
}

/* sin/cos tables exactly as the reference builds them (for parity analysis) */
void vc3o_angle_tables(int t, int p, double* sin_t, double* cos_t, double* sin_p, double* cos_p) {
    tables_t T;
    build_tables(&T, t, p);
    memcpy(sin_t, T.sin_t, sizeof(double) << t);
    memcpy(cos_t, T.cos_t, sizeof(double) << t);
    memcpy(sin_p, T.sin_p, sizeof(double) << p);
    memcpy(cos_p, T.cos_p, sizeof(double) << p);
    free(T.sin_t); free(T.cos_t); free(T.sin_p); free(T.cos_p);
}
