// Throughput (per SM) of the FP64 ops in the relaxation: DFMA/DADD and the
// MUFU.RCP64H / MUFU.RSQ64H seeds.  One CTA of 256 threads per SM, 8
// independent chains per thread; prints warp-instructions per cycle per SM.
#include <cstdio>
#include <cstdint>
#include "../../paper_2305_07030_b200/csrc/frb_arith.cuh"
template <int OP>
__global__ void thr(double* out, double a, long long* cyc) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = a + k + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 512; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __fma_rn(x[k], 0.999, 1e-3);
      if (OP == 1) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x[k]));
      if (OP == 2) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x[k]));
      if (OP == 3) x[k] = __dadd_rn(x[k], 1e-3);
      if (OP == 4) x[k] = __dmul_rn(x[k], 0.999);
      if (OP == 5) {  // one F1 element: sqrt_fast + div_fast chain
        bool o1, o2;
        const double l = frb_arith::sqrt_fast(__dadd_rn(__dmul_rn(x[k], x[k]), 1.0), o1);
        const double q = frb_arith::div_fast(__dmul_rn(2.0, __dsub_rn(l, 1.5)), __dmul_rn(1.5, l), o2);
        x[k] = __dadd_rn(q, (o1 && o2) ? 1.0 : 2.0);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[OP] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8); cudaMallocManaged(&c, 128);
  for (int T : {128, 256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      thr<0><<<148, T>>>(o, 1.0, c); thr<1><<<148, T>>>(o, 1.5, c); thr<2><<<148, T>>>(o, 1.5, c);
      thr<3><<<148, T>>>(o, 1.0, c); thr<4><<<148, T>>>(o, 1.5, c); thr<5><<<148, T>>>(o, 1.5, c);
      cudaDeviceSynchronize();
    }
    const double wi = 512.0 * 8 * T / 32;
    printf("T=%d  DFMA %.3f  RCP64H %.3f  RSQ64H %.3f DADD %.3f DMUL %.3f warp-instr/clk/SM; F1 element %.3f thread-elements/clk/SM\n", T, wi / c[0], wi / c[1], wi / c[2], wi / c[3], wi / c[4], 512.0 * 8 * T / c[5]);
  }
  return 0;
}
