// Cycles of the real C3 (32^3, 16 ranks) local and top tree programs replayed
// by one warp (run_prog of frb_relax.cuh), alone on the SM: isolates the
// program's cost from the kernel context. Programs come from plan.py
// (tools/ubench/c3_prog*.bin written by the build-container script).
#include <cstdio>
#include <vector>
#include "../../paper_2305_07030_b200/csrc/frb_relax.cuh"
namespace frb_tu { thread_local char g_err[512]; }

__global__ void bench(const int* progs, int lw, int tw, int LS, int TS, long long* out) {
  int* lp = reinterpret_cast<int*>(g_smem + 3 * (LS + TS));
  int* tp = lp + lw + (lw & 1);
  for (int k = threadIdx.x; k < lw; k += blockDim.x) lp[k] = progs[k];
  for (int k = threadIdx.x; k < tw; k += blockDim.x) tp[k] = progs[lw + k];
  for (int k = threadIdx.x; k < 3 * (LS + TS); k += blockDim.x) g_smem[k] = 1.0 + 1e-3 * k;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    run_prog(lp, 0, threadIdx.x);
    long long t1 = clock64();
    run_prog(tp, 3 * LS, threadIdx.x);
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
  }
}

int main() {
  int hdr[4];
  FILE* f = fopen("tools/ubench/c3_prog_hdr.bin", "rb"); fread(hdr, 4, 4, f); fclose(f);
  std::vector<int> p(hdr[2] + hdr[3]);
  f = fopen("tools/ubench/c3_prog.bin", "rb"); fread(p.data(), 4, p.size(), f); fclose(f);
  int* dp; long long* dout;
  cudaMalloc(&dp, p.size() * 4); cudaMalloc(&dout, 16);
  cudaMemcpy(dp, p.data(), p.size() * 4, cudaMemcpyHostToDevice);
  size_t smem = 8 * 3 * (hdr[0] + hdr[1]) + 4 * (p.size() + 2);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    bench<<<1, 512, smem>>>(dp, hdr[2], hdr[3], hdr[0], hdr[1], dout);
    long long h[2]; cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
    printf("local program %lld cycles (%d rounds), top program %lld cycles (%d rounds) %s\n", h[0], p[0], h[1],
           p[hdr[2]], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
