// Micro-benchmark of the sm_100a pipes the codec leans on: FP64 FMA/ADD,
// 64-bit <-> 32-bit conversions, double sqrt, IEEE float division and random
// 16-byte shared-memory table lookups.  Prints per-SM per-clock throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench pipebench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

template <int OP>
__global__ void __launch_bounds__(256) kbench(double* out, long long* cyc, float seedf) {
    double d[ILP];
    float f[ILP];
    long long l[ILP];
    __shared__ double2 tab[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = make_double2(i * 0.5, i * 0.25);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
        d[j] = 1.0 + 1e-3 * (threadIdx.x + j);
        f[j] = seedf + 1e-3f * (threadIdx.x + j);
        l[j] = threadIdx.x * 7 + j;
    }
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (OP == 0) d[j] = fma(d[j], 0.999999, 1e-7);                  // DFMA
            if (OP == 1) d[j] = d[j] + 1e-9;                                 // DADD
            if (OP == 2) { f[j] = f[j] * 1.0000001f; d[j] += (double)f[j]; } // F2F.F64.F32 (+DADD)
            if (OP == 3) { f[j] = f[j] + (float)d[j]; }                      // F2F.F32.F64 (+FADD)
            if (OP == 4) { l[j] += __double2ll_rd(d[j]); d[j] += 1e-9; }    // F2I.S64.F64 (+DADD)
            if (OP == 5) { d[j] += __ll2double_rn(l[j]); l[j] += 3; }       // I2F.F64.S64
            if (OP == 6) f[j] = fmaf(f[j], 0.9999f, 1e-7f);                 // FFMA
            if (OP == 7) { double2 v = tab[(l[j] & 1023)]; l[j] = l[j] * 1103515245 + 12345 + (long long)v.x; d[j] += v.y; }  // LDS.128 random
            if (OP == 8) d[j] = sqrt(d[j]) + 1.0;                            // DSQRT (IEEE)
            if (OP == 9) f[j] = __fdiv_rn(1.0f, f[j]) + 1.0f;                // IEEE f32 div
            if (OP == 10) { f[j] = f[j] + __double2float_ru(d[j]); d[j] += 1e-9; } // F2F.F32.F64.RP
            if (OP == 11) { d[j] = __dadd_rd(d[j], 6755399441055744.0) - 6755399441055744.0 + 0.5; } // DADD.RM magic floor
            if (OP == 12) { l[j] = (l[j] * 3 + 1) ^ (l[j] >> 3); }           // 64-bit int mix (IMAD/SHF/LOP)
            if (OP == 13) { unsigned u = __float_as_uint(f[j]); unsigned hi = ((u & 0x80000000u) | ((u & 0x7fffffffu) >> 3)) + 0x38000000u; d[j] += __hiloint2double(hi, u << 29); f[j] += 1e-7f; } // int f32->f64
        }
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc += d[j] + f[j] + (double)l[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int nsm) {
    int blocks = nsm * 8, threads = 256;
    double* out; long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    kbench<OP><<<blocks, threads>>>(out, cyc, 1.5f);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kbench<OP><<<blocks, threads>>>(out, cyc, 1.5f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mc = 0; for (int i = 0; i < blocks; ++i) mc = mc > h[i] ? mc : (double)h[i];
    double ops = (double)blocks * threads * ILP * ITERS;
    // per-SM per-clock using the in-kernel cycle count of the slowest CTA (8 CTAs/SM co-resident)
    printf("%-28s %8.3f ms  %9.1f Gop/s  %6.1f op/clk/SM (clk64)  %s\n", name, ms, ops / ms / 1e6,
           ops / nsm / mc, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc); delete[] h;
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
    int n = p.multiProcessorCount;
    run<0>("DFMA", n);
    run<1>("DADD", n);
    run<2>("F2F.F64.F32 (+DADD)", n);
    run<3>("F2F.F32.F64 (+FADD)", n);
    run<4>("F2I.S64.F64.FLOOR (+DADD)", n);
    run<5>("I2F.F64.S64 (+DADD)", n);
    run<6>("FFMA", n);
    run<7>("LDS.128 random (+int,DADD)", n);
    run<8>("DSQRT ieee (+DADD)", n);
    run<9>("FDIV ieee (+FADD)", n);
    run<10>("F2F.F32.F64.RP (+FADD,DADD)", n);
    run<11>("DADD.RM magic floor (3 DADD)", n);
    run<12>("int64 mix", n);
    run<13>("int f32->f64 (+DADD,FADD)", n);
    return 0;
}
