// vc3_fr.cu — flux-reconstruction flux divergence on compressed fluxes
// (Alg. 1), on the sm_100a tensor cores.
//
//   div[k][c][i] = sum_j sum_d D[d*ns + j][k] * X[j][c][i][d],
//   X[j][c][i] = decompress(words[(j*n_vars + c)*ld + i])      (a 3-vector)
//
// i = element, c = equation (variable), j/k = solution points, d = dimension.
// For each equation this is a GEMM  Out_c (n_elem x ns) = A_c (n_elem x 3ns)
// * D' (3ns x ns), with the decode of the compressed flux as the producer of
// the A operand.  At k = 4 (ns = 125) it is 93,750 flops per element-equation
// against 1,500 B of compressed input and output — beyond the FP32 CUDA-core
// rate at HBM speed — so the contraction runs on tcgen05:
//
//  * persistent CTAs (one per SM), tiles of 256 elements of one equation as
//    two UMMA M = 128 halves; 16 decode warps, 4 epilogue warps, one
//    operator-load warp (cp.async.bulk of the pre-split operator slice from
//    L2), one flux-row warp (cp.async.bulk of each stage's 8 rows into a
//    shared-memory ring) and one MMA warp (a single thread issues
//    tcgen05.mma);
//  * K is walked in stages of 8 solution points (24 k-values): the decode
//    warps write the stage's A slice straight into shared memory in the
//    canonical no-swizzle K-major UMMA layout (8-row x 16-byte core
//    matrices), the MMA warp accumulates into TMEM (two halves x npad fp32
//    columns, double-buffered across tiles), stages ring through mbarriers;
//  * the operand decode is float32 (MUFU sin/cos, decode_f32): the GEMM's
//    own rounding is larger than its error;
//  * fp32 accuracy on TF32 tensor cores by operand splitting (3xTF32):
//    a = a_hi + a_lo, b = b_hi + b_lo with a_hi the top 19 bits, and
//    a*b ~ a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (relative error ~2^-21);
//  * epilogue warps: tcgen05.ld of the accumulator (lane = element, column =
//    point), coalesced 128-byte stores per output point, overlapping the
//    next tile's mainloop.
//
// The uncompressed baseline (float32 [j][c][i][3] fluxes) runs the same
// kernel with plain loads in place of the decode.  For tensor-product
// hexahedra the sum-factorised kernels at the end of this file apply the
// 1D derivative matrix per direction on the CUDA cores instead.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"
#include "vc3_rt.h"

using namespace vc3;
using namespace vc3::rt;

namespace {

#ifndef VC3_FR_HEX_REG
#define VC3_FR_HEX_REG 1
#endif

constexpr int kRows = 256;             // elements per tile: two UMMA M = 128 halves
constexpr int kHalf = 128;
constexpr int kPts = 8;                // solution points per K stage
constexpr int kDecodeWarps = 16;       // 2 threads per element, 4 points each
constexpr int kEpiWarps = 4;           // TMEM -> global, one per TMEM lane quarter
constexpr int kThreadsFr = (kDecodeWarps + kEpiWarps + 3) * 32;
constexpr int kLoadWarp = kDecodeWarps + kEpiWarps;
constexpr int kMmaWarp = kDecodeWarps + kEpiWarps + 1;
constexpr int kRawWarp = kDecodeWarps + kEpiWarps + 2;  // flux rows -> shared memory (BULK)
constexpr int kASliceBytes = kHalf * kPts * 4;  // one half, one dimension, hi or lo: 4 KB

__host__ __device__ constexpr int b_slice_bytes(int npad) { return npad * kPts * 4; }
// stage: A slices [hi|lo][half m][dimension d] (12 x 4 KB), then B slices
// [hi|lo][d] (6 x npad x 32 B)
__host__ __device__ constexpr int stage_bytes(int npad) {
    return 12 * kASliceBytes + 6 * b_slice_bytes(npad);
}
__host__ __device__ constexpr int a_slice(int lo, int m, int d) { return ((lo * 2 + m) * 3 + d) * kASliceBytes; }

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// canonical no-swizzle K-major shared-memory matrix descriptor (sm_100 format:
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), layout 0)
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
           ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = npad
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// fp32 decode for the contraction.  The GEMM rounds each product to ~2^-21
// (3xTF32), so the operand needs no more than that: the angles are formed in
// float32 (|error| ~ 2^-22) and their sin/cos come from the hardware
// (MUFU.SIN/COS, |error| <= 2^-21.4 on [-pi, pi]).  No shared-memory table:
// the table gathers of the exact decode were this kernel's bottleneck
// (compressed FR at k = 4: 2.07 -> 2.38 G elem-eq/s).  Agreement with
// vc3_decompress: |dx| <= ~2^-21 |x| per component (tests/test_fr.py bounds
// the divergence at 2^-18 sum |D||X|).
template <class LAY>
__device__ __forceinline__ void decode_f32(unsigned long long w, const Params& P, float& ox, float& oy,
                                           float& oz) {
    const unsigned long long field = w >> (P.p + P.t);
    const unsigned nt = (unsigned)(w & P.tmask);
    const unsigned nph = (unsigned)((w >> P.t) & P.pmask);
    float st, ct, sp, cp;
    const float th = __fmaf_rn(__uint2float_rn(nt), (float)(2.0 * 3.141592653589793 / (double)P.ntmax),
                               -3.14159265358979f);
    const float ph = __fmul_rn(__uint2float_rn(nph), (float)(3.141592653589793 / (double)P.npmax));
    __sincosf(th, &st, &ct);
    __sincosf(ph, &sp, &cp);
    float r;
    if (P.dec_normal) {
        // every exponent maps to a normal float32: re-bias the field's bits
        const unsigned f = (unsigned)field & ((1u << (P.e + P.m)) - 1u);
        r = field ? __uint_as_float((f << (23 - P.m)) + ((unsigned)(127 - P.bias) << 23)) : 0.0f;
    } else {
        r = decode_mag(field, P);  // exact float32 magnitude, 0 for a zero field
    }
    ox = __fmul_rn(__fmul_rn(r, ct), sp);
    oy = __fmul_rn(__fmul_rn(r, st), sp);
    oz = __fmul_rn(r, cp);
}

// offset of (row, kk) inside one canonical K-major slice of 8 k-values:
// core matrices of 8 rows x 16 B; LBO (next 4 k-values) = 128 B, SBO (next
// 8 rows) = 256 B
__host__ __device__ constexpr int canon_off(int row, int kk) {
    return (row >> 3) * 256 + (kk >> 2) * 128 + (row & 7) * 16 + (kk & 3) * 4;
}

// ---- operator preparation -----------------------------------------------------
// Bprep[s][hi|lo][d][canonical npad x 8] from D[3ns][ns] (row d*ns + j, column k)
__global__ void k_fr_prepare(const float* __restrict__ D, int ns, int npad, int nst,
                             float* __restrict__ out) {
    const int per_stage = 6 * npad * kPts;
    const int total = nst * per_stage;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int s = idx / per_stage;
        int r = idx - s * per_stage;
        const int part = r / (npad * kPts);  // 0..2 hi d0..d2, 3..5 lo d0..d2
        r -= part * npad * kPts;
        const int n = r / kPts, kk = r - n * kPts;
        const int d = part % 3;
        const int j = s * kPts + kk;
        const float v = (j < ns && n < ns) ? D[(size_t)(d * ns + j) * ns + n] : 0.0f;
        const float hi = tf32_hi(v);
        out[(size_t)s * per_stage + part * npad * kPts + canon_off(n, kk) / 4] = part < 3 ? hi : v - hi;
    }
}

// ---- the fused kernel -----------------------------------------------------------
struct FrArgs {
    const unsigned long long* words;  // compressed fluxes [ns][n_vars][ld]
    const float* raw;                 // or float32 fluxes [ns][n_vars][ld][3]
    const float* bprep;               // k_fr_prepare output
    float* out;                       // [ns][n_vars][ld]
    int64_t n_elem, ld;
    int n_vars, ns, npad, nst, nbuf, nraw;
};

// BULK: the flux rows of each stage (8 points x 256 elements, contiguous per
// point) are brought into a shared-memory ring by cp.async.bulk from one
// producer thread, so the decode warps never wait on HBM latency; otherwise
// (strides not 16-byte aligned) the decode warps prefetch into registers.
template <bool RAW, bool BULK, class LAY>
__global__ void __launch_bounds__(kThreadsFr, 1) k_fr_div(FrArgs a, Params Pin) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sbytes = stage_bytes(a.npad);
    constexpr int esize = RAW ? 12 : 8;
    constexpr int rbytes = kPts * kRows * esize;  // one raw-ring slot
    unsigned char* stages = smem;
    unsigned char* rawbuf = smem + (size_t)a.nbuf * sbytes;
    unsigned char* meta = rawbuf + (BULK ? (size_t)a.nraw * rbytes : 0);
    uint64_t* full = reinterpret_cast<uint64_t*>(meta);
    uint64_t* empty = full + a.nbuf;
    uint64_t* acc_full = empty + a.nbuf;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint64_t* raw_full = acc_empty + 2;   // [nraw]
    uint64_t* raw_empty = raw_full + 8;   // [nraw]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + 8);
    // accumulators: [buffer][half] x npad fp32 columns; two buffers when they fit
    const int nacc = 4 * a.npad <= 512 ? 2 : 1;
    const uint32_t tmem_cols = nacc * 2 * a.npad <= 256 ? 256 : 512;

    const int64_t tiles_per_var = (a.n_elem + kRows - 1) / kRows;
    const int64_t ntiles = tiles_per_var * a.n_vars;

    if (threadIdx.x == 0) {
        for (int b = 0; b < a.nbuf; ++b) {
            mbar_init(&full[b], kDecodeWarps + 1);
            mbar_init(&empty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kEpiWarps);
        }
        if (BULK) {
            for (int r = 0; r < a.nraw; ++r) {
                mbar_init(&raw_full[r], 1);
                mbar_init(&raw_empty[r], kDecodeWarps);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < kDecodeWarps) {
        // ---------------- producers of A (decode), all tiles of this CTA ----------------
        const int row = threadIdx.x & (kRows - 1), h = threadIdx.x / kRows;
        const int m = row / kHalf;
        const int64_t plane = (int64_t)a.n_vars * a.ld;  // stride between solution points
        const int64_t plane2 = 2 * plane, plane3 = 3 * plane, step = (int64_t)kPts * plane;
        // register fetch cursor (!BULK): runs two stages ahead of the decode,
        // across tile boundaries
        int64_t ftile = blockIdx.x;
        int fstage = 0;
        const unsigned long long* wp = nullptr;
        const float* fp = nullptr;
        bool flive = false;
        auto begin_tile = [&](int64_t t) {
            const int c = (int)(t / tiles_per_var);
            const int64_t i = (t - (int64_t)c * tiles_per_var) * kRows + row;
            flive = t < ntiles && i < a.n_elem;
            const int64_t base = (int64_t)c * a.ld + i + (int64_t)(4 * h) * plane;
            wp = a.words + (RAW ? 0 : base);
            fp = a.raw + (RAW ? 3 * base : 0);
        };
        unsigned long long w1[4], w2[4];
        float3 f1[4], f2[4];
        auto fetch = [&](unsigned long long* w, float3* f) {
            const int jn = fstage * kPts + 4 * h;
            const int nv = flive ? min(max(a.ns - jn, 0), 4) : 0;
            if (RAW) {
                const float* pq[4] = {fp, fp + 3 * plane, fp + 3 * plane2, fp + 3 * plane3};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    f[q] = q < nv ? make_float3(__ldg(pq[q]), __ldg(pq[q] + 1), __ldg(pq[q] + 2))
                                  : make_float3(0.f, 0.f, 0.f);
                fp += 3 * step;
            } else {
                const unsigned long long* pq[4] = {wp, wp + plane, wp + plane2, wp + plane3};
#pragma unroll
                for (int q = 0; q < 4; ++q) w[q] = q < nv ? __ldg(pq[q]) : 0ull;
                wp += step;
            }
            if (++fstage == a.nst) {
                fstage = 0;
                ftile += gridDim.x;
                begin_tile(ftile);
            }
        };
        if (!BULK) {
            begin_tile(ftile);
            fetch(w1, f1);
            fetch(w2, f2);
        }
        const int off = canon_off(row & (kHalf - 1), 4 * h);
        int b = 0, use = 0;  // A-ring slot and how often it has been filled before
        int r = 0, ruse = 0; // raw-ring slot (BULK)
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 0; s < a.nst; ++s) {
                unsigned long long w[4];
                float3 f[4];
                if (BULK) {
                    // points 8s + 4h + q of this element from the raw ring
                    const int nv = min(max(a.ns - (s * kPts + 4 * h), 0), 4);
                    mbar_wait(&raw_full[r], ruse & 1);
                    const unsigned char* rb = rawbuf + (size_t)r * rbytes;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const unsigned char* e = rb + ((size_t)(4 * h + q) * kRows + row) * esize;
                        if (RAW) {
                            const float* ef = reinterpret_cast<const float*>(e);
                            f[q] = q < nv ? make_float3(ef[0], ef[1], ef[2]) : make_float3(0.f, 0.f, 0.f);
                        } else {
                            w[q] = q < nv ? *reinterpret_cast<const unsigned long long*>(e) : 0ull;
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&raw_empty[r]);
                    if (++r == a.nraw) { r = 0; ++ruse; }
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        w[q] = w1[q]; f[q] = f1[q];
                        w1[q] = w2[q]; f1[q] = f2[q];
                    }
                    fetch(w2, f2);
                }
                float x[4], y[4], z[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (RAW) {
                        x[q] = f[q].x; y[q] = f[q].y; z[q] = f[q].z;
                    } else {
                        // zero words (and padding) decode to exact zeros
                        decode_f32<LAY>(w[q], P, x[q], y[q], z[q]);
                    }
                }
                if (use > 0) mbar_wait(&empty[b], (use - 1) & 1);
                unsigned char* st = stages + (size_t)b * sbytes;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const float* v = d == 0 ? x : (d == 1 ? y : z);
                    float4 hi, lo;
                    hi.x = tf32_hi(v[0]); lo.x = v[0] - hi.x;
                    hi.y = tf32_hi(v[1]); lo.y = v[1] - hi.y;
                    hi.z = tf32_hi(v[2]); lo.z = v[2] - hi.z;
                    hi.w = tf32_hi(v[3]); lo.w = v[3] - hi.w;
                    *reinterpret_cast<float4*>(st + a_slice(0, m, d) + off) = hi;
                    *reinterpret_cast<float4*>(st + a_slice(1, m, d) + off) = lo;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[b]);
                if (++b == a.nbuf) { b = 0; ++use; }
            }
        }
    } else if (warp < kDecodeWarps + kEpiWarps) {
        // ---------------- epilogue: TMEM -> global, overlapping the next tile ----------------
        const int ew = warp - kDecodeWarps;  // == warp % 4: TMEM lane quarter
        const int64_t cstride = (int64_t)a.n_vars * a.ld;
        int lt = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
            const int ab = nacc == 2 ? (lt & 1) : 0;
            const int au = nacc == 2 ? (lt >> 1) : lt;
            mbar_wait(&acc_full[ab], au & 1);
            tc_fence_after();
            const int c = (int)(t / tiles_per_var);
            const int64_t i0 = (t - (int64_t)c * tiles_per_var) * kRows;
#pragma unroll 1
            for (int em = 0; em < 2; ++em) {
                const int64_t ei = i0 + em * kHalf + ew * 32 + lane;
                const bool elive = ei < a.n_elem;
                float* op = a.out + (int64_t)c * a.ld + ei;
                const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)((ab * 2 + em) * a.npad);
                for (int c0 = 0; c0 < a.npad; c0 += 16) {
                    float v[16];
                    tmem_ld16(tbase + (uint32_t)c0, v);
                    const int kn = min(16, a.ns - c0);
                    if (elive) {
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            if (q < kn) op[0] = v[q];
                            op += cstride;
                        }
                    } else {
                        op += 16 * cstride;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
        }
    } else if (warp == kLoadWarp) {
        // ---------------- operator slices (L2 -> smem, bulk async copy) ----------------
        if (lane == 0) {
            const uint32_t bbytes = 6 * b_slice_bytes(a.npad);
            int b = 0, use = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int s = 0; s < a.nst; ++s) {
                    if (use > 0) mbar_wait(&empty[b], (use - 1) & 1);
                    unsigned char* dst = stages + (size_t)b * sbytes + 12 * kASliceBytes;
                    mbar_arrive_tx(&full[b], bbytes);
                    bulk_g2s(dst, a.bprep + (size_t)s * (bbytes / 4), bbytes, &full[b]);
                    if (++b == a.nbuf) { b = 0; ++use; }
                }
            }
        }
        __syncwarp();
    } else if (BULK && warp == kRawWarp) {
        // ---------------- flux rows (HBM -> smem ring, bulk async copy) ----------------
        if (lane == 0) {
            const int64_t plane = (int64_t)a.n_vars * a.ld;
            const unsigned char* src0 = RAW ? reinterpret_cast<const unsigned char*>(a.raw)
                                            : reinterpret_cast<const unsigned char*>(a.words);
            int r = 0, ruse = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int c = (int)(t / tiles_per_var);
                const int64_t i0 = (t - (int64_t)c * tiles_per_var) * kRows;
                const int64_t cnt = a.ld - i0 < kRows ? a.ld - i0 : kRows;  // rows are ld long
                const uint32_t row_bytes = (uint32_t)(cnt * esize);
                for (int s = 0; s < a.nst; ++s) {
                    if (ruse > 0) mbar_wait(&raw_empty[r], (ruse - 1) & 1);
                    const int nrows = min(kPts, a.ns - s * kPts);
                    unsigned char* dst = rawbuf + (size_t)r * rbytes;
                    mbar_arrive_tx(&raw_full[r], (uint32_t)nrows * row_bytes);
                    for (int jj = 0; jj < nrows; ++jj) {
                        const int64_t j = (int64_t)s * kPts + jj;
                        bulk_g2s(dst + (size_t)jj * kRows * esize,
                                 src0 + ((j * plane) + (int64_t)c * a.ld + i0) * esize, row_bytes,
                                 &raw_full[r]);
                    }
                    if (++r == a.nraw) { r = 0; ++ruse; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issue (one thread) ----------------
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(kHalf, a.npad);
            const int bsl = b_slice_bytes(a.npad);
            const uint64_t desc0 = smem_desc(stages, 128, 256);
            int b = 0, use = 0, lt = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
                const int ab = nacc == 2 ? (lt & 1) : 0;
                const int au = nacc == 2 ? (lt >> 1) : lt;
                if (au > 0) mbar_wait(&acc_empty[ab], (au - 1) & 1);  // epilogue drained it
                tc_fence_after();
                for (int s = 0; s < a.nst; ++s) {
                    mbar_wait(&full[b], use & 1);
                    tc_fence_after();
                    // descriptors = slot base descriptor + (byte offset >> 4): one
                    // add each (the MMA thread shares its scheduler with decode
                    // warps, so its instruction count per MMA matters)
                    const uint64_t sd = desc0 + (uint64_t)(((uint32_t)b * (uint32_t)sbytes) >> 4);
                    const uint64_t bd = sd + (uint64_t)((12 * kASliceBytes) >> 4);
                    const uint32_t acc0 = tmem + (uint32_t)(ab * 2 * a.npad);
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const uint64_t bhi = bd + (uint64_t)((uint32_t)(d * bsl) >> 4);
                        const uint64_t blo = bd + (uint64_t)((uint32_t)((3 + d) * bsl) >> 4);
#pragma unroll
                        for (int m = 0; m < 2; ++m) {
                            const uint32_t acc = acc0 + (uint32_t)(m * a.npad);
                            const uint64_t ahi = sd + (uint64_t)(a_slice(0, m, d) >> 4);
                            const uint64_t alo = sd + (uint64_t)(a_slice(1, m, d) >> 4);
                            mma_tf32(acc, alo, bhi, idesc, (s | d) != 0);
                            mma_tf32(acc, ahi, blo, idesc, 1);
                            mma_tf32(acc, ahi, bhi, idesc, 1);
                        }
                    }
                    mma_commit(&empty[b]);
                    if (++b == a.nbuf) { b = 0; ++use; }
                }
                mma_commit(&acc_full[ab]);
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
    }
}

// ---- the CTA-pair kernel (tcgen05 cta_group::2) ------------------------------
// Two CTAs of a cluster share one UMMA M = 256 product per (dimension, split):
// each holds the A operand of its own 128 elements and half of the operator
// slice (N / 2 columns), the leader issues the MMA for both, and each CTA's
// TMEM receives the accumulator rows of its elements.  Per 128 elements the
// tensor core then reads 4 KB of A and 2 KB of B per MMA instead of 4 + 4, and
// each CTA copies half of each operator slice: this kernel is bound by
// shared-memory bandwidth (tensor-core operand reads + decode stores).
// The peer's stage and accumulator hand-offs reach the leader's barriers
// through one relay thread (the peer's MMA warp): it waits on the peer's own
// barrier and arrives on the leader's at cluster scope.
constexpr int kPairRows = 128;  // elements per CTA; a pair's tile is 256
constexpr int kPairDecodeWarps = 8;  // 2 threads per element, 4 points each

__host__ __device__ constexpr int pair_half_bytes(int npad) { return npad * kPts * 4 / 2; }
__host__ __device__ constexpr int pair_stage_bytes(int npad) {
    return 6 * kASliceBytes + 6 * pair_half_bytes(npad);
}
__host__ __device__ constexpr int pa_slice(int lo, int d) { return (lo * 3 + d) * kASliceBytes; }

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_rank(uint64_t* bar, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mma2_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma2_commit_both(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}

template <bool RAW, class LAY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsFr, 1) k_fr_div2(FrArgs a, Params Pin) {
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int sbytes = pair_stage_bytes(a.npad);
    const int hb = pair_half_bytes(a.npad);
    constexpr int esize = RAW ? 12 : 8;
    constexpr int rbytes = kPts * kPairRows * esize;  // one raw-ring slot
    unsigned char* stages = smem;
    unsigned char* rawbuf = smem + (size_t)a.nbuf * sbytes;
    unsigned char* meta = rawbuf + (size_t)a.nraw * rbytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(meta);
    uint64_t* empty = full + a.nbuf;
    uint64_t* acc_full = empty + a.nbuf;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint64_t* raw_full = acc_empty + 2;   // [nraw]
    uint64_t* raw_empty = raw_full + 8;   // [nraw]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + 8);
    const uint32_t tmem_cols = 2 * a.npad <= 32 ? 32 : 2 * a.npad <= 64 ? 64 : 2 * a.npad <= 128 ? 128
                             : 2 * a.npad <= 256 ? 256 : 512;
    const int64_t tiles_per_var = (a.n_elem + 2 * kPairRows - 1) / (2 * kPairRows);
    const int64_t ntiles = tiles_per_var * a.n_vars;
    const int64_t pair0 = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int b = 0; b < a.nbuf; ++b) {
            mbar_init(&full[b], kPairDecodeWarps + 1 + (leader ? 1 : 0));  // + the peer's relay
            mbar_init(&empty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kEpiWarps + (leader ? 1 : 0));
        }
        for (int r = 0; r < a.nraw; ++r) {
            mbar_init(&raw_full[r], 1);
            mbar_init(&raw_empty[r], kPairDecodeWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < kPairDecodeWarps) {
        // ---------------- producers of A (decode): 2 threads per element, 4 points each
        // (warps kPairDecodeWarps..kDecodeWarps-1 of the shared CTA shape idle)
        const int row = threadIdx.x & (kPairRows - 1), h = threadIdx.x / kPairRows;  // h in 0..1
        const int off = canon_off(row, 4 * h);
        int b = 0, use = 0, r = 0, ruse = 0;
        for (int64_t t = pair0; t < ntiles; t += npairs) {
            for (int s = 0; s < a.nst; ++s) {
                const int nv = min(max(a.ns - (s * kPts + 4 * h), 0), 4);
                mbar_wait(&raw_full[r], ruse & 1);
                const unsigned char* rb = rawbuf + (size_t)r * rbytes;
                float x[4], y[4], z[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned char* e = rb + ((size_t)(4 * h + q) * kPairRows + row) * esize;
                    if (RAW) {
                        const float* ef = reinterpret_cast<const float*>(e);
                        x[q] = q < nv ? ef[0] : 0.f;
                        y[q] = q < nv ? ef[1] : 0.f;
                        z[q] = q < nv ? ef[2] : 0.f;
                    } else {
                        const unsigned long long wq = q < nv ? *reinterpret_cast<const unsigned long long*>(e) : 0ull;
                        decode_f32<LAY>(wq, P, x[q], y[q], z[q]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&raw_empty[r]);
                if (++r == a.nraw) { r = 0; ++ruse; }
                if (use > 0) mbar_wait(&empty[b], (use - 1) & 1);
                unsigned char* st = stages + (size_t)b * sbytes;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const float* v = d == 0 ? x : (d == 1 ? y : z);
                    float4 hi, lo;
                    hi.x = tf32_hi(v[0]); lo.x = v[0] - hi.x;
                    hi.y = tf32_hi(v[1]); lo.y = v[1] - hi.y;
                    hi.z = tf32_hi(v[2]); lo.z = v[2] - hi.z;
                    hi.w = tf32_hi(v[3]); lo.w = v[3] - hi.w;
                    *reinterpret_cast<float4*>(st + pa_slice(0, d) + off) = hi;
                    *reinterpret_cast<float4*>(st + pa_slice(1, d) + off) = lo;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[b]);
                if (++b == a.nbuf) { b = 0; ++use; }
            }
        }
    } else if (warp < kDecodeWarps) {
        // idle
    } else if (warp < kDecodeWarps + kEpiWarps) {
        // ---------------- epilogue: this CTA's 128 elements from its TMEM
        const int ew = warp - kDecodeWarps;  // == warp % 4: TMEM lane quarter
        const int64_t cstride = (int64_t)a.n_vars * a.ld;
        int lt = 0;
        for (int64_t t = pair0; t < ntiles; t += npairs, ++lt) {
            const int ab = lt & 1, au = lt >> 1;
            mbar_wait(&acc_full[ab], au & 1);
            tc_fence_after();
            const int c = (int)(t / tiles_per_var);
            const int64_t ei = (t - (int64_t)c * tiles_per_var) * (2 * kPairRows) + rank * kPairRows + ew * 32 + lane;
            const bool elive = ei < a.n_elem;
            float* op = a.out + (int64_t)c * a.ld + ei;
            const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(ab * a.npad);
            for (int c0 = 0; c0 < a.npad; c0 += 16) {
                float v[16];
                tmem_ld16(tbase + (uint32_t)c0, v);
                const int kn = min(16, a.ns - c0);
                if (elive) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (q < kn) op[0] = v[q];
                        op += cstride;
                    }
                } else {
                    op += 16 * cstride;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
        }
    } else if (warp == kLoadWarp) {
        // ---------------- this CTA's half of each operator slice
        if (lane == 0) {
            int b = 0, use = 0;
            for (int64_t t = pair0; t < ntiles; t += npairs) {
                for (int s = 0; s < a.nst; ++s) {
                    if (use > 0) mbar_wait(&empty[b], (use - 1) & 1);
                    unsigned char* dst = stages + (size_t)b * sbytes + 6 * kASliceBytes;
                    mbar_arrive_tx(&full[b], 6 * hb);
                    const float* src = a.bprep + (size_t)s * 6 * a.npad * kPts + (size_t)rank * (hb / 4);
#pragma unroll 1
                    for (int part = 0; part < 6; ++part)
                        bulk_g2s(dst + part * hb, src + (size_t)part * a.npad * kPts, hb, &full[b]);
                    if (++b == a.nbuf) { b = 0; ++use; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kRawWarp) {
        // ---------------- flux rows of this CTA's 128 elements
        if (lane == 0) {
            const int64_t plane = (int64_t)a.n_vars * a.ld;
            const unsigned char* src0 = RAW ? reinterpret_cast<const unsigned char*>(a.raw)
                                            : reinterpret_cast<const unsigned char*>(a.words);
            int r = 0, ruse = 0;
            for (int64_t t = pair0; t < ntiles; t += npairs) {
                const int c = (int)(t / tiles_per_var);
                const int64_t i0 = (t - (int64_t)c * tiles_per_var) * (2 * kPairRows) + rank * kPairRows;
                const int64_t left = a.ld - i0;
                const int64_t cnt = left <= 0 ? 0 : (left < kPairRows ? left : kPairRows);
                const uint32_t row_bytes = (uint32_t)(cnt * esize);
                for (int s = 0; s < a.nst; ++s) {
                    if (ruse > 0) mbar_wait(&raw_empty[r], (ruse - 1) & 1);
                    const int nrows = min(kPts, a.ns - s * kPts);
                    unsigned char* dst = rawbuf + (size_t)r * rbytes;
                    mbar_arrive_tx(&raw_full[r], (uint32_t)nrows * row_bytes);
                    if (row_bytes)
                        for (int jj = 0; jj < nrows; ++jj) {
                            const int64_t j = (int64_t)s * kPts + jj;
                            bulk_g2s(dst + (size_t)jj * kPairRows * esize,
                                     src0 + ((j * plane) + (int64_t)c * a.ld + i0) * esize, row_bytes,
                                     &raw_full[r]);
                        }
                    if (++r == a.nraw) { r = 0; ++ruse; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        if (lane == 0 && leader) {
            // ---------------- MMA issue for the pair (one thread of the leader)
            const uint32_t idesc = idesc_tf32(2 * kPairRows, a.npad);
            const uint64_t desc0 = smem_desc(stages, 128, 256);
            int b = 0, use = 0, lt = 0;
            for (int64_t t = pair0; t < ntiles; t += npairs, ++lt) {
                const int ab = lt & 1, au = lt >> 1;
                if (au > 0) mbar_wait(&acc_empty[ab], (au - 1) & 1);  // both epilogues drained it
                tc_fence_after();
                for (int s = 0; s < a.nst; ++s) {
                    mbar_wait(&full[b], use & 1);  // both CTAs' stage b
                    tc_fence_after();
                    const uint64_t sd = desc0 + (uint64_t)(((uint32_t)b * (uint32_t)sbytes) >> 4);
                    const uint64_t bd = sd + (uint64_t)((6 * kASliceBytes) >> 4);
                    const uint32_t acc = tmem + (uint32_t)(ab * a.npad);
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const uint64_t bhi = bd + (uint64_t)((uint32_t)(d * hb) >> 4);
                        const uint64_t blo = bd + (uint64_t)((uint32_t)((3 + d) * hb) >> 4);
                        const uint64_t ahi = sd + (uint64_t)(pa_slice(0, d) >> 4);
                        const uint64_t alo = sd + (uint64_t)(pa_slice(1, d) >> 4);
                        mma2_tf32(acc, alo, bhi, idesc, (s | d) != 0);
                        mma2_tf32(acc, ahi, blo, idesc, 1);
                        mma2_tf32(acc, ahi, bhi, idesc, 1);
                    }
                    mma2_commit_both(&empty[b]);
                    if (++b == a.nbuf) { b = 0; ++use; }
                }
                mma2_commit_both(&acc_full[ab]);
            }
        } else if (lane == 0) {
            // ---------------- the peer's relay to the leader's barriers
            int b = 0, use = 0, lt = 0;
            for (int64_t t = pair0; t < ntiles; t += npairs, ++lt) {
                const int ab = lt & 1, au = lt >> 1;
                if (au > 0) {
                    mbar_wait(&acc_empty[ab], (au - 1) & 1);
                    mbar_arrive_rank(&acc_empty[ab], 0);
                }
                for (int s = 0; s < a.nst; ++s) {
                    mbar_wait(&full[b], use & 1);
                    mbar_arrive_rank(&full[b], 0);
                    if (++b == a.nbuf) { b = 0; ++use; }
                }
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
    }
}

int npad_for(int ns) { return ((ns + 15) / 16) * 16; }
int nst_for(int ns) { return (ns + kPts - 1) / kPts; }

int fr_launch(const unsigned long long* words, const float* raw, const float* bprep, float* out,
              int64_t n_elem, int n_vars, int64_t ld, int ns, const vc3_layout* layout, cudaStream_t s) {
    if (n_elem < 0 || n_vars < 1 || ns < 1 || ns > 256 || ld < n_elem) return VC3_ERR_ARG;
    if (!bprep || !out || (!words && !raw)) return VC3_ERR_ARG;
    if (((uintptr_t)bprep & 15u) != 0) return VC3_ERR_ARG;
    if (n_elem == 0) return VC3_OK;
    FrArgs a{};
    a.words = words;
    a.raw = raw;
    a.bprep = bprep;
    a.out = out;
    a.n_elem = n_elem;
    a.ld = ld;
    a.n_vars = n_vars;
    a.ns = ns;
    a.npad = npad_for(ns);
    a.nst = nst_for(ns);
    Params P{};
    if (!raw) {
        if (!layout_ok(*layout)) return VC3_ERR_LAYOUT;
        P = make_params(*layout);
    }
    // the CTA-pair kernel is opt-in (VC3_FR_PAIR=1 in the environment): it is
    // correct but measured slower
    static const bool pair_on = [] {
        const char* e = getenv("VC3_FR_PAIR");
        return e && e[0] == '1';
    }();
    const size_t budget = 227 * 1024 - 1024;
    {
        // the CTA-pair kernel (k_fr_div2): bulk flux rows (16-byte aligned
        // rows), an even grid of clusters
        const int esize_p = raw ? 12 : 8;
        const void* src_p = raw ? (const void*)raw : (const void*)words;
        const bool bulk_p = ((uintptr_t)src_p & 15u) == 0 && (ld % 4) == 0;
        if (pair_on && bulk_p && sm_count() >= 2) {
            const size_t sbp = (size_t)pair_stage_bytes(a.npad);
            const size_t rbp = (size_t)kPts * kPairRows * esize_p;
            int nbuf = (int)((budget - 2 * rbp) / sbp);
            if (nbuf > 4) nbuf = 4;
            if (nbuf > a.nst) nbuf = a.nst;
            if (nbuf >= 1) {
                int nraw = (int)((budget - (size_t)nbuf * sbp) / rbp);
                if (nraw > 8) nraw = 8;
                a.nbuf = nbuf;
                a.nraw = nraw;
                const size_t smem = (size_t)nbuf * sbp + (size_t)nraw * rbp + 1024;
                const int64_t tiles = ((n_elem + 2 * kPairRows - 1) / (2 * kPairRows)) * n_vars;
                const int64_t pairs = tiles < sm_count() / 2 ? tiles : sm_count() / 2;
                const unsigned grid = (unsigned)(2 * pairs);
#define VC3_FR_GO2(R, L)                                                                 \
    do {                                                                                 \
        const int st_ = ensure_smem((const void*)k_fr_div2<R, L>, smem);                \
        if (st_) return st_;                                                             \
        k_fr_div2<R, L><<<grid, kThreadsFr, smem, s>>>(a, P);                           \
    } while (0)
                if (raw) VC3_FR_GO2(true, RuntimeLayout);
                else if (is_default_layout(*layout)) VC3_FR_GO2(false, DefaultLayout);
                else VC3_FR_GO2(false, RuntimeLayout);
#undef VC3_FR_GO2
                return launch_status();
            }
        }
    }
    const size_t sb = (size_t)stage_bytes(a.npad);
    // the raw ring needs 16-byte aligned rows: base pointer, ld multiple of 4
    const int esize = raw ? 12 : 8;
    const void* src = raw ? (const void*)raw : (const void*)words;
    const size_t rbytes = (size_t)kPts * kRows * esize;
    bool bulk = ((uintptr_t)src & 15u) == 0 && (ld % 4) == 0;
    // two A/B stages (decode of s+1 overlaps the MMA of s) come first, more
    // when they fit beside a raw ring of >= 2 slots; the ring takes the rest
    int nbuf = (int)(budget / sb);
    if (nbuf > a.nst) nbuf = a.nst;
    if (nbuf < 1) return VC3_ERR_ARG;
    const int nbuf2 = nbuf < 2 ? nbuf : 2;
    int more = budget > 3 * rbytes ? (int)((budget - 3 * rbytes) / sb) : 0;
    if (more > 4) more = 4;
    if (more > a.nst) more = a.nst;
    nbuf = more > nbuf2 ? more : nbuf2;
    int nraw = (int)((budget - (size_t)nbuf * sb) / rbytes);
    if (nraw > 8) nraw = 8;
    if (nraw < 2) bulk = false;
    a.nbuf = nbuf;
    a.nraw = bulk ? nraw : 0;
    const size_t smem = (size_t)nbuf * sb + (size_t)a.nraw * rbytes + 1024;
    const int64_t tiles = ((n_elem + kRows - 1) / kRows) * n_vars;
    const int64_t grid = tiles < sm_count() ? tiles : sm_count();  // persistent: one CTA per SM
#define VC3_FR_GO(R, B, L)                                                               \
    do {                                                                                 \
        const int st_ = ensure_smem((const void*)k_fr_div<R, B, L>, smem);               \
        if (st_) return st_;                                                             \
        k_fr_div<R, B, L><<<(unsigned)grid, kThreadsFr, smem, s>>>(a, P);               \
    } while (0)
    if (raw) {
        if (bulk) VC3_FR_GO(true, true, RuntimeLayout);
        else VC3_FR_GO(true, false, RuntimeLayout);
    } else if (is_default_layout(*layout)) {
        if (bulk) VC3_FR_GO(false, true, DefaultLayout);
        else VC3_FR_GO(false, false, DefaultLayout);
    } else {
        if (bulk) VC3_FR_GO(false, true, RuntimeLayout);
        else VC3_FR_GO(false, false, RuntimeLayout);
    }
#undef VC3_FR_GO
    return launch_status();
}

// ---- sum-factorised divergence for tensor-product hexahedra ---------------------
// For D built from a 1D derivative matrix M (M[a][m] = l_m'(x_a), k+1 Gauss
// points per direction, point index p = px + n py + n^2 pz), Alg. 1 reduces to
//   div[k] = sum_a M[kx][a] X_(a,ky,kz).x + M[ky][a] X_(kx,a,kz).y
//                                        + M[kz][a] X_(kx,ky,a).z,
// 3(k+1) multiply-adds per output instead of 3 ns.  fp32 fluxes: one thread
// per (element, equation) streams its ns points in order and scatters the
// three components into ns accumulators held in registers (indices are
// compile-time: the point loop is fully unrolled); HBM-bound.
struct HexOp {
    float m[6][6];
};

template <int K, bool COMP, class LAY>
__global__ void __launch_bounds__(128, 3) k_fr_hex_reg(const float* __restrict__ raw, float* __restrict__ out,
                                                    int64_t n_elem, int n_vars, int64_t ld, HexOp op,
                                                    const unsigned long long* __restrict__ words = nullptr,
                                                    Params Pin = Params{}) {
    constexpr int N1 = K + 1, NS = N1 * N1 * N1, PF = 8;
    Params P = Pin;
    if (COMP) LAY::apply(P);
    const int c = blockIdx.y;
    const int64_t plane = (int64_t)n_vars * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_elem;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = (int64_t)c * ld + i;
        float acc[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) acc[k] = 0.0f;
        float3 pf[PF];  // the next PF points' fluxes are in flight
        unsigned long long pw[PF];
#pragma unroll
        for (int q = 0; q < PF; ++q) {
            if (COMP) {
                pw[q] = __ldg(words + base + q * plane);
            } else {
                const float* p = raw + 3 * (base + q * plane);
                pf[q] = make_float3(__ldg(p), __ldg(p + 1), __ldg(p + 2));
            }
        }
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            float x, y, z;
            if (COMP) {
                decode_f32<LAY>(pw[j % PF], P, x, y, z);
            } else {
                x = pf[j % PF].x; y = pf[j % PF].y; z = pf[j % PF].z;
            }
            if (j + PF < NS) {
                if (COMP) {
                    pw[j % PF] = __ldg(words + base + (j + PF) * plane);
                } else {
                    const float* p = raw + 3 * (base + (j + PF) * plane);
                    pf[j % PF] = make_float3(__ldg(p), __ldg(p + 1), __ldg(p + 2));
                }
            }
        const int jx = j % N1, jy = (j / N1) % N1, jz = j / (N1 * N1);
#pragma unroll
            for (int a = 0; a < N1; ++a) {
                acc[a + N1 * jy + N1 * N1 * jz] = __fmaf_rn(op.m[a][jx], x, acc[a + N1 * jy + N1 * N1 * jz]);
                acc[jx + N1 * a + N1 * N1 * jz] = __fmaf_rn(op.m[a][jy], y, acc[jx + N1 * a + N1 * N1 * jz]);
                acc[jx + N1 * jy + N1 * N1 * a] = __fmaf_rn(op.m[a][jz], z, acc[jx + N1 * jy + N1 * N1 * a]);
            }
        }
        float* o = out + base;
#pragma unroll
        for (int k = 0; k < NS; ++k) o[k * plane] = acc[k];
    }
}

// Compressed fluxes: decoding inside that register-heavy loop is latency-bound
// (measured 0.67 G elem-eq/s at k = 4: all ns accumulators live in registers,
// 2 warps per scheduler).  Here a CTA takes
// 32 elements of one equation: phase A decodes the tile's 32 x ns words with
// all 8 warps (loads issued up front, lane = element) into shared memory as
// [dimension][point][element] floats; phase B applies the sum-factorised
// operator from shared memory (15 conflict-free loads + 15 FMAs per output at
// k = 4), lane = element, so global loads and stores stay 256/128-byte
// coalesced rows.
constexpr int kHexE = 32;
constexpr int kHexThreads = 256;

template <int K, class LAY>
__global__ void __launch_bounds__(kHexThreads, 4) k_fr_hex_staged(
    const unsigned long long* __restrict__ words, float* __restrict__ out, int64_t n_elem, int n_vars,
    int64_t ld, HexOp op, Params Pin) {
    constexpr int N1 = K + 1, NS = N1 * N1 * N1, NW = kHexThreads / 32;
    constexpr int NJ = (NS + NW - 1) / NW;  // points per warp in phase A
    Params P = Pin;
    LAY::apply(P);
    extern __shared__ float xs[];  // [3][NS][kHexE]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t blocks_per_var = (n_elem + kHexE - 1) / kHexE;
    const int64_t ntiles = blocks_per_var * n_vars;
    const int64_t plane = (int64_t)n_vars * ld;
    // the next tile's words are loaded while this tile runs phase B
    unsigned long long w[NJ];
    auto load_tile = [&](int64_t t) {
        const int c = (int)(t / blocks_per_var);
        const int64_t i = (t - (int64_t)c * blocks_per_var) * kHexE + lane;
        const bool ok = t < ntiles && i < n_elem;
        const unsigned long long* wp = words + (int64_t)c * ld + i + warp * plane;
        const int64_t wstep = NW * plane;
#pragma unroll
        for (int r = 0; r < NJ; ++r) {
            const int j = warp + NW * r;
            w[r] = (ok && j < NS) ? __ldg(wp) : 0ull;
            wp += wstep;
        }
    };
    load_tile(blockIdx.x);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int c = (int)(t / blocks_per_var);
        const int64_t i = (t - (int64_t)c * blocks_per_var) * kHexE + lane;
        const bool live = i < n_elem;
        // phase A: decode
#pragma unroll
        for (int r = 0; r < NJ; ++r) {
            const int j = warp + NW * r;
            if (j < NS) {
                float x, y, z;
                decode_f32<LAY>(w[r], P, x, y, z);
                xs[(0 * NS + j) * kHexE + lane] = x;
                xs[(1 * NS + j) * kHexE + lane] = y;
                xs[(2 * NS + j) * kHexE + lane] = z;
            }
        }
        load_tile(t + gridDim.x);
        __syncthreads();
        // phase B: sum-factorised operator; a thread computes one x-line
        // (ky, kz) of its element: the x-part reuses the line's N1 values,
        // the 1D matrix rows of ky and kz are loaded once per line
        float* op_out = out + (int64_t)c * ld + i;
        for (int L = warp; L < N1 * N1; L += NW) {
            const int ky = L % N1, kz = L / N1;
            // row bases: every inner offset below is a compile-time constant
            const float* xl = xs + (N1 * L) * kHexE + lane;
            const float* yl = xs + (NS + N1 * N1 * kz) * kHexE + lane;
            const float* zl = xs + (2 * NS + N1 * ky) * kHexE + lane;
            float my[N1], mz[N1], xv[N1], acc[N1];
#pragma unroll
            for (int a = 0; a < N1; ++a) {
                my[a] = op.m[ky][a];
                mz[a] = op.m[kz][a];
                xv[a] = xl[a * kHexE];
            }
#pragma unroll
            for (int kx = 0; kx < N1; ++kx) {
                float t = 0.0f;
#pragma unroll
                for (int a = 0; a < N1; ++a) t = __fmaf_rn(op.m[kx][a], xv[a], t);
#pragma unroll
                for (int a = 0; a < N1; ++a) t = __fmaf_rn(my[a], yl[(kx + N1 * a) * kHexE], t);
#pragma unroll
                for (int a = 0; a < N1; ++a) t = __fmaf_rn(mz[a], zl[(kx + N1 * N1 * a) * kHexE], t);
                acc[kx] = t;
            }
            if (live) {
                float* o = op_out + (int64_t)(N1 * L) * plane;
#pragma unroll
                for (int kx = 0; kx < N1; ++kx) {
                    o[0] = acc[kx];
                    o += plane;
                }
            }
        }
        __syncthreads();
    }
}

template <int K>
int hex_launch_k(const unsigned long long* words, const float* raw, float* out, int64_t n_elem,
                 int n_vars, int64_t ld, const HexOp& op, const vc3_layout* layout, cudaStream_t s) {
    Params P{};
    size_t smem = 0;
    if (!raw) P = make_params(*layout);
    int64_t blocks = (n_elem + 127) / 128;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    const dim3 grid((unsigned)blocks, (unsigned)n_vars);
    if (raw) {
        k_fr_hex_reg<K, false, RuntimeLayout><<<grid, 128, 0, s>>>(raw, out, n_elem, n_vars, ld, op);
    } else if (VC3_FR_HEX_REG && K != 3) {
        // register-resident accumulators with the MUFU decode in the point
        // loop; at k = 3 the compiler's schedule spills, the staged kernel wins
        if (is_default_layout(*layout))
            k_fr_hex_reg<K, true, DefaultLayout><<<grid, 128, 0, s>>>(nullptr, out, n_elem, n_vars, ld, op, words, P);
        else
            k_fr_hex_reg<K, true, RuntimeLayout><<<grid, 128, 0, s>>>(nullptr, out, n_elem, n_vars, ld, op, words, P);
    } else {
        constexpr int NS = (K + 1) * (K + 1) * (K + 1);
        smem += (size_t)3 * NS * kHexE * sizeof(float);
        const int64_t tiles = ((n_elem + kHexE - 1) / kHexE) * n_vars;
        const int64_t cap3 = (int64_t)sm_count() * 4;  // four 48-KB CTAs per SM at k = 4
        const unsigned g = (unsigned)(tiles < cap3 ? tiles : cap3);
        if (is_default_layout(*layout)) {
            const int st = ensure_smem((const void*)k_fr_hex_staged<K, DefaultLayout>, smem);
            if (st) return st;
            cudaFuncSetAttribute((const void*)k_fr_hex_staged<K, DefaultLayout>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            k_fr_hex_staged<K, DefaultLayout><<<g, kHexThreads, smem, s>>>(words, out, n_elem, n_vars, ld, op, P);
        } else {
            const int st = ensure_smem((const void*)k_fr_hex_staged<K, RuntimeLayout>, smem);
            if (st) return st;
            k_fr_hex_staged<K, RuntimeLayout><<<g, kHexThreads, smem, s>>>(words, out, n_elem, n_vars, ld, op, P);
        }
    }
    return launch_status();
}

int hex_launch(const unsigned long long* words, const float* raw, const float* m1d, int degree,
               float* out, int64_t n_elem, int n_vars, int64_t ld, const vc3_layout* layout,
               cudaStream_t s) {
    if (degree < 1 || degree > 4 || n_elem < 0 || n_vars < 1 || n_vars > 65535 || ld < n_elem)
        return VC3_ERR_ARG;
    if (!m1d || !out || (!words && !raw)) return VC3_ERR_ARG;
    if (!raw && !layout_ok(*layout)) return VC3_ERR_LAYOUT;
    if (n_elem == 0) return VC3_OK;
    HexOp op{};
    for (int a = 0; a <= degree; ++a)
        for (int b = 0; b <= degree; ++b) op.m[a][b] = m1d[a * (degree + 1) + b];
    switch (degree) {
        case 1: return hex_launch_k<1>(words, raw, out, n_elem, n_vars, ld, op, layout, s);
        case 2: return hex_launch_k<2>(words, raw, out, n_elem, n_vars, ld, op, layout, s);
        case 3: return hex_launch_k<3>(words, raw, out, n_elem, n_vars, ld, op, layout, s);
        default: return hex_launch_k<4>(words, raw, out, n_elem, n_vars, ld, op, layout, s);
    }
}

}  // namespace

extern "C" {

int64_t vc3_fr_operator_floats(int n_points) {
    if (n_points < 1 || n_points > 256) return -1;
    return (int64_t)nst_for(n_points) * 6 * npad_for(n_points) * kPts;
}

int vc3_fr_prepare_operator(const float* D, int n_points, float* op, void* stream) {
    if (!D || !op || n_points < 1 || n_points > 256) return VC3_ERR_ARG;
    const int64_t total = vc3_fr_operator_floats(n_points);
    const int grid = (int)((total + 255) / 256);
    k_fr_prepare<<<grid, 256, 0, (cudaStream_t)stream>>>(D, n_points, npad_for(n_points),
                                                          nst_for(n_points), op);
    return launch_status();
}

int vc3_fr_divergence(const uint64_t* words, const float* op, float* div, int64_t n_elem,
                      int n_vars, int64_t ld, int n_points, vc3_layout layout, void* stream) {
    if (!words) return VC3_ERR_ARG;
    return fr_launch((const unsigned long long*)words, nullptr, op, div, n_elem, n_vars, ld, n_points,
                     &layout, (cudaStream_t)stream);
}

int vc3_fr_divergence_f32(const float* flux, const float* op, float* div, int64_t n_elem,
                          int n_vars, int64_t ld, int n_points, void* stream) {
    if (!flux) return VC3_ERR_ARG;
    return fr_launch(nullptr, flux, op, div, n_elem, n_vars, ld, n_points, nullptr,
                     (cudaStream_t)stream);
}

int vc3_fr_divergence_hex(const uint64_t* words, const float* m1d, int degree, float* div,
                          int64_t n_elem, int n_vars, int64_t ld, vc3_layout layout, void* stream) {
    if (!words) return VC3_ERR_ARG;
    return hex_launch((const unsigned long long*)words, nullptr, m1d, degree, div, n_elem, n_vars, ld,
                      &layout, (cudaStream_t)stream);
}

int vc3_fr_divergence_hex_f32(const float* flux, const float* m1d, int degree, float* div,
                              int64_t n_elem, int n_vars, int64_t ld, void* stream) {
    if (!flux) return VC3_ERR_ARG;
    return hex_launch(nullptr, flux, m1d, degree, div, n_elem, n_vars, ld, nullptr,
                      (cudaStream_t)stream);
}

}  // extern "C"
