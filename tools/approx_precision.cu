// approx_precision.cu — measures the worst relative error of the sm_100a
// approximate FP64 reciprocal square root (rsqrt.approx.ftz.f64, MUFU.RSQ64H)
// and reciprocal (rcp.approx.ftz.f64, MUFU.RCP64H) over every 20-bit high
// mantissa (the units read only the high word), both exponent parities and
// both extreme low words.  The compress kernel's fast magnitude path relies on
// the rsqrt bound.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_approx(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

__global__ void k(double* worst) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;  // 2^23 cases
    const unsigned mant_hi = i & 0xFFFFF;
    const unsigned expo = 1023 + ((i >> 20) & 1) + ((i >> 21) & 1 ? 200 : -200);
    const unsigned lo = (i >> 22) & 1 ? 0xFFFFFFFFu : 0u;
    const double x = __hiloint2double((int)((expo << 20) | mant_hi), (int)lo);
    // reference values to ~1 ulp
    const double s = __dsqrt_rn(x);
    const double rs = __ddiv_rn(1.0, s);
    const double rc = __ddiv_rn(1.0, x);
    const double e1 = fabs(rsqrt_approx(x) - rs) / rs;
    const double e2 = fabs(rcp_approx(x) - rc) / rc;
    atomicMax((unsigned long long*)&worst[0], __double_as_longlong(e1));
    atomicMax((unsigned long long*)&worst[1], __double_as_longlong(e2));
}

int main() {
    double* d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    k<<<(1 << 23) / 256, 256>>>(d);
    double h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("rsqrt.approx.ftz.f64 max rel err %.3e (2^%.2f)\n", h[0], log2(h[0]));
    printf("rcp.approx.ftz.f64   max rel err %.3e (2^%.2f)\n", h[1], log2(h[1]));
    return 0;
}
