// debug: compress_as2 vs compress_one on given float triples, with intermediates
#include <cstdio>
#include <cstring>

#include "../../paper_2003_02633_b200/csrc/vc3_device.cuh"
#include "../../paper_2003_02633_b200/csrc/vc3_fused.cuh"
using namespace vc3;
__global__ void k(const float* v, int n, Params Pin, unsigned long long* out) {
  Params P = Pin; DefaultLayout::apply(P);
  int i = threadIdx.x;
  if (2 * i + 1 >= n) return;
  float x[2] = {v[6*i], v[6*i+3]}, y[2] = {v[6*i+1], v[6*i+4]}, z[2] = {v[6*i+2], v[6*i+5]};
  unsigned long long w[2]; bool slow[2];
  compress_as2(x, y, z, P, w, slow);
  for (int k = 0; k < 2; ++k) {
    out[4*(2*i+k)] = w[k];
    out[4*(2*i+k)+1] = compress_one<7, true, true>(x[k], y[k], z[k], P);
    out[4*(2*i+k)+2] = slow[k];
    // intermediates via scalar float IEEE ops
    float sq = __fadd_rn(__fadd_rn(__fmul_rn(x[k],x[k]), __fmul_rn(y[k],y[k])), __fmul_rn(z[k],z[k]));
    float rq = __fsqrt_rn(sq); float wq = __fdiv_rn(z[k], rq);
    out[4*(2*i+k)+3] = ((unsigned long long)__float_as_uint(rq) << 32) | __float_as_uint(wq);
  }
}
int main(int argc, char** argv) {
  float h[600]; int n = 0;
  unsigned hx; while (n < 600 && scanf("%x", &hx) == 1) { memcpy(&h[n], &hx, 4); ++n; }
  n /= 3;
  float* d; unsigned long long* o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8 * 4 * 200);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  Params P{}; P.e=7;P.m=22;P.p=17;P.t=18;P.bias=80; derive_int_fields(P);
  const double pi = 3.141592653589793;
  P.nt_half=(double)P.ntmax/2.0; P.t_scale=(double)P.ntmax/(2.0*pi); P.p_scale=(double)P.npmax/pi;
  P.nt_half2=2*P.nt_half; P.t_scale2=2*P.t_scale; P.p_scale2=2*P.p_scale;
  k<<<1, 1>>>(d, n, P, o);
  unsigned long long r[800]; cudaMemcpy(r, o, 8*4*n, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("%d fast=%016llx gen=%016llx slow=%llu rq=%08x w=%08x %s\n", i, r[4*i], r[4*i+1], r[4*i+2], (unsigned)(r[4*i+3]>>32), (unsigned)r[4*i+3], r[4*i]==r[4*i+1]?"":"DIFF");
}
