// Issue-rate micro-benchmark of the sm_100a instructions the fused codec
// kernels are built from (round 2).  Each thread runs ILP independent chains
// of one instruction (inline PTX so the SASS is exactly that instruction),
// 8 CTAs x 256 threads per SM; prints warp-instructions per clock per SM
// (peak issue is 4: one per SMSP) from CUDA-event time x the SM clock measured
// under load (clock64 vs globaltimer).
// Mixed entries interleave two instruction kinds 1:1 to show whether their
// pipes overlap.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench2 pipebench2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define ILP 8
#define ITERS 2048

enum Op {
    FFMA, FFMA_IMM, FFMA2, FADD2, FMUL2, DFMA, DMUL, DADD, F2F_D_F, F2F_F_D, F2F_F_D_RU, MUFU_RCP,
    MUFU_RSQ, MUFU_RSQ64H, LOP3, IADD3, SHF, IMAD, FSEL, FMNMX, DSETP, LDS128, LDS64, MIX_DFMA_FFMA2,
    MIX_DFMA_LOP3, MIX_DFMA_IMAD, MIX_FFMA2_LOP3, MIX_F2F_DFMA, MIX_DFMA_FFMA, NOPS
};
static const char* kNames[] = {
    "FFMA (3 reg)", "FFMA (imm)", "FFMA2", "FADD2", "FMUL2", "DFMA", "DMUL", "DADD",
    "F2F.F64.F32", "F2F.F32.F64", "F2F.F32.F64.RP", "MUFU.RCP", "MUFU.RSQ", "MUFU.RSQ64H",
    "LOP3", "IADD3", "SHF", "IMAD", "FSEL", "FMNMX", "DSETP", "LDS.128 random", "LDS.64 random",
    "DFMA+FFMA2 1:1", "DFMA+LOP3 1:1", "DFMA+IMAD 1:1", "FFMA2+LOP3 1:1", "F2F.F64.F32+DFMA 1:1",
    "DFMA+FFMA 1:1"};

template <int OP>
__global__ void __launch_bounds__(256) kbench(double* out, long long* cyc, float seedf) {
    double d[ILP];
    float f[ILP];
    unsigned long long p[ILP];
    unsigned u[ILP];
    __shared__ double2 tab[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_double2(i * 0.5, i * 0.25);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
        d[j] = 1.0 + 1e-3 * (threadIdx.x + j);
        f[j] = seedf + 1e-3f * (threadIdx.x + j);
        float2 t = make_float2(f[j], f[j] * 0.5f);
        p[j] = *reinterpret_cast<unsigned long long*>(&t);
        u[j] = threadIdx.x * 7 + j;
    }
    const float cf = 0.9999f;
    const unsigned long long c2 = p[0] ^ 0x10001ull;
    const double cd = 0.999999;
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (OP == FFMA) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[j]) : "f"(cf), "f"(f[(j + 1) % ILP]));
            if (OP == FFMA_IMM) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f33D6BF95;" : "+f"(f[j]));
            if (OP == FFMA2) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[j]) : "l"(c2));
            if (OP == FADD2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[j]) : "l"(c2));
            if (OP == FMUL2) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[j]) : "l"(c2));
            if (OP == DFMA) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(cd));
            if (OP == DMUL) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[j]) : "d"(cd));
            if (OP == DADD) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[j]) : "d"(cd));
            if (OP == F2F_D_F) asm volatile("{.reg .f64 t; cvt.f64.f32 t, %0; cvt.rn.f32.f64 %0, t;}" : "+f"(f[j]));
            if (OP == F2F_F_D) asm volatile("{.reg .f32 t; cvt.rn.f32.f64 t, %0; cvt.f64.f32 %0, t;}" : "+d"(d[j]));
            if (OP == F2F_F_D_RU) asm volatile("{.reg .f32 t; cvt.rp.f32.f64 t, %0; cvt.f64.f32 %0, t;}" : "+d"(d[j]));
            if (OP == MUFU_RCP) asm volatile("{.reg .f32 t; rcp.approx.ftz.f32 t, %0; fma.rn.f32 %0, t, 0f3F7FFFFF, 0f3F800000;}" : "+f"(f[j]));
            if (OP == MUFU_RSQ) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
            if (OP == MUFU_RSQ64H) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(d[j]));
            if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]), "r"(u[(j + 2) % ILP]));
            if (OP == IADD3) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]));
            if (OP == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]));
            if (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]), "r"(u[(j + 2) % ILP]));
            if (OP == FSEL) asm volatile("{.reg .pred q; setp.lt.f32 q, %1, 0f3F800000; selp.f32 %0, %0, %1, q;}" : "+f"(f[j]) : "f"(f[(j + 1) % ILP]));
            if (OP == FMNMX) asm volatile("max.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(f[(j + 1) % ILP]));
            if (OP == DSETP) asm volatile("{.reg .pred q; setp.lt.f64 q, %1, 0d3FF0000000000000; selp.b32 %0, %0, 3, q; add.rn.f64 %1, %1, 0d3E112E0BE826D695;}" : "+r"(u[j]), "+d"(d[j]));
            if (OP == LDS128) { const double2 v = tab[u[j] & 2047]; u[j] = u[j] * 1103515245u + 12345u + (unsigned)__double2hiint(v.x); d[j] += v.y; }
            if (OP == LDS64) { const double v = reinterpret_cast<const double*>(tab)[u[j] & 4095]; u[j] = u[j] * 1103515245u + 12345u + (unsigned)__double2hiint(v); }
            if (OP == MIX_DFMA_FFMA2) {
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(cd));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[j]) : "l"(c2));
            }
            if (OP == MIX_DFMA_LOP3) {
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(cd));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]), "r"(u[(j + 2) % ILP]));
            }
            if (OP == MIX_DFMA_IMAD) {
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(cd));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]), "r"(u[(j + 2) % ILP]));
            }
            if (OP == MIX_FFMA2_LOP3) {
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[j]) : "l"(c2));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[j]) : "r"(u[(j + 1) % ILP]), "r"(u[(j + 2) % ILP]));
            }
            if (OP == MIX_F2F_DFMA) {
                asm volatile("{.reg .f64 t; cvt.f64.f32 t, %0; add.rn.f64 %1, %1, t;}" : "+f"(f[j]), "+d"(d[j]));
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[(j + 3) % ILP]) : "d"(cd));
            }
            if (OP == MIX_DFMA_FFMA) {
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(cd));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[j]) : "f"(cf), "f"(f[(j + 1) % ILP]));
            }
        }
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc += d[j] + f[j] + (double)u[j] + (double)(p[j] & 0xffff);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static int instr_per_step(int op) {
    switch (op) {
        case F2F_D_F: case F2F_F_D: case F2F_F_D_RU: return 2;  // a conversion pair
        case FSEL: case MUFU_RCP: return 2;
        case DSETP: return 3;                          // setp + select
        case MIX_DFMA_FFMA2: case MIX_DFMA_LOP3: case MIX_DFMA_IMAD: case MIX_FFMA2_LOP3:
        case MIX_DFMA_FFMA: return 2;
        case MIX_F2F_DFMA: return 3;
        default: return 1;
    }
}

template <int OP>
void run(int nsm, double clk_hz) {
    const int blocks = nsm * 8, threads = 256;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    kbench<OP><<<blocks, threads>>>(out, cyc, 1.5f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kbench<OP><<<blocks, threads>>>(out, cyc, 1.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_steps = (double)blocks * (threads / 32) * ILP * ITERS;
    const double clks = ms * 1e-3 * clk_hz;
    const double ipc = warp_steps * instr_per_step(OP) / nsm / clks;
    printf("%-24s %6.3f warp-instr/clk/SM  (%5.2f steps/clk/SM, %.3f ms)  %s\n", kNames[OP], ipc,
           warp_steps / nsm / clks, ms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

// SM clock under load: clock64 against globaltimer over a busy loop
__global__ void kclk(double* hz) {
    unsigned long long g0, g1;
    long long c0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    float f = 1.0f;
    for (int i = 0; i < 4000000; ++i) f = fmaf(f, 0.9999999f, 1e-7f);
    long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) hz[blockIdx.x] = (double)(c1 - c0) / (double)(g1 - g0) * 1e9 + (f == 0.0f);
}

template <int... OPS>
void run_all(int nsm, double hz, std::integer_sequence<int, OPS...>) {
    (run<OPS>(nsm, hz), ...);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* dh;
    cudaMalloc(&dh, sizeof(double) * p.multiProcessorCount);
    kclk<<<p.multiProcessorCount, 32>>>(dh);
    double hz = 0;
    cudaMemcpy(&hz, dh, sizeof(double), cudaMemcpyDeviceToHost);
    printf("%s SMs=%d  SM clock under load %.0f MHz\n", p.name, p.multiProcessorCount, hz / 1e6);
    run_all(p.multiProcessorCount, hz, std::make_integer_sequence<int, NOPS>{});
    return 0;
}
