// Throughput (per SM) of the FP64 ops in the relaxation: DFMA/DADD and the
// MUFU.RCP64H / MUFU.RSQ64H seeds.  One CTA of 256 threads per SM, 8
// independent chains per thread; prints warp-instructions per cycle per SM.
#include <cstdio>
#include <cstdint>
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
      if (OP == 3) x[k] = __fmaf_rn(__int_as_float(__double2hiint(x[k])), 0.f, __int_as_float(__double2loint(x[k]))) + x[k];
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
  double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8); cudaMallocManaged(&c, 64);
  for (int T : {128, 256, 512, 1024}) {
    thr<0><<<148, T>>>(o, 1.0, c); thr<1><<<148, T>>>(o, 1.5, c); thr<2><<<148, T>>>(o, 1.5, c);
    cudaDeviceSynchronize();
    thr<0><<<148, T>>>(o, 1.0, c); thr<1><<<148, T>>>(o, 1.5, c); thr<2><<<148, T>>>(o, 1.5, c);
    cudaDeviceSynchronize();
    const double wi = 512.0 * 8 * T / 32;
    printf("T=%d  DFMA %.3f  RCP64H %.3f  RSQ64H %.3f warp-instr/clk/SM (cycles %lld %lld %lld)\n", T, wi / c[0], wi / c[1], wi / c[2], c[0], c[1], c[2]);
  }
  return 0;
}
