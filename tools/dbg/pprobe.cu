// debug: packed phi pipeline intermediates vs scalar
#include <cstdio>
#include <cstring>
#include "../../paper_2003_02633_b200/csrc/vc3_device.cuh"
#include "../../paper_2003_02633_b200/csrc/vc3_fused.cuh"
using namespace vc3;
__global__ void k(const float* v, unsigned* out) {
  float z[2] = {v[0], v[1]}, sqv[2] = {v[2], v[3]};
  const f2 ONE = splat2(1.0f), HALF = splat2(0.5f), NHALF = splat2(-0.5f);
  const f2 SQ = pk(sqv[0], sqv[1]), Z = pk(z[0], z[1]);
  float rs[2]; for (int k = 0; k < 2; ++k) rs[k] = rsqrt_approx(sqv[k]);
  const f2 RS = pk(rs[0], rs[1]);
  const f2 YQ = mul2(SQ, RS);
  const f2 RQ = fma2(fnma2(YQ, YQ, SQ), mul2(RS, HALF), YQ);
  float rq[2], ri[2]; upk(RQ, rq[0], rq[1]);
  for (int k = 0; k < 2; ++k) ri[k] = rcp_approx(rq[k]);
  const f2 RI0 = pk(ri[0], ri[1]);
  const f2 RI = fma2(RI0, fnma2(RQ, RI0, ONE), RI0);
  const f2 WQ = mul2(Z, RI);
  const f2 W = fma2(fnma2(RQ, WQ, Z), RI, WQ);
  float wv[2], aw[2]; upk(W, wv[0], wv[1]);
  for (int k = 0; k < 2; ++k) { wv[k] = fminf(fmaxf(wv[k], -1.0f), 1.0f); aw[k] = fabsf(wv[k]); }
  const f2 ZS = fma2(pk(aw[0], aw[1]), NHALF, HALF);
  float zs[2], rz[2]; upk(ZS, zs[0], zs[1]);
  for (int k = 0; k < 2; ++k) rz[k] = rsqrt_approx(zs[k]);
  const f2 RZ = pk(rz[0], rz[1]);
  const f2 YS = mul2(ZS, RZ);
  const f2 XS = fma2(fnma2(YS, YS, ZS), mul2(RZ, HALF), YS);
  float xs[2]; upk(XS, xs[0], xs[1]);
  for (int k = 0; k < 2; ++k) {
    out[8*k] = __float_as_uint(rq[k]); out[8*k+1] = __float_as_uint(__fsqrt_rn(sqv[k]));
    out[8*k+2] = __float_as_uint(wv[k]); out[8*k+3] = __float_as_uint(__fdiv_rn(z[k], __fsqrt_rn(sqv[k])));
    out[8*k+4] = __float_as_uint(zs[k]); out[8*k+5] = __float_as_uint(__fmul_rn(__fsub_rn(1.0f, aw[k]), 0.5f));
    out[8*k+6] = __float_as_uint(xs[k]); out[8*k+7] = __float_as_uint(__fsqrt_rn(zs[k]));
  }
}
int main() {
  // z and sq of the two failing vectors
  unsigned hz[4] = {0xbfebc0da, 0xbfb11ee3, 0, 0};
  float h[4]; memcpy(h, hz, 8);
  h[2] = 4.791524f; h[3] = 2.0314183f;
  // exact sq from the float ops
  float* d; unsigned* o; cudaMalloc(&d, 16); cudaMalloc(&o, 64);
  cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
  k<<<1, 1>>>(d, o);
  unsigned r[16]; cudaMemcpy(r, o, 64, cudaMemcpyDeviceToHost);
  for (int k = 0; k < 2; ++k) printf("rq %08x/%08x w %08x/%08x zs %08x/%08x xs %08x/%08x\n", r[8*k], r[8*k+1], r[8*k+2], r[8*k+3], r[8*k+4], r[8*k+5], r[8*k+6], r[8*k+7]);
}
