#include <vector>
#include <cstdio>
// Cycles per round of the tree-program replay (run_prog in frb_relax.cuh):
// one warp replays a synthetic program of R rounds (each lane adds two slots
// of the previous level into a new slot), alone on the SM and with 23
// other warps streaming FP64 work (the shadow (-f)/m of the T phase).
#include "../../paper_2305_07030_b200/csrc/frb_relax.cuh"

namespace frb_tu { thread_local char g_err[512]; }

__global__ void bench(const int* prog_g, int words, int n_slots, int busy, long long* out) {
  int* prog = reinterpret_cast<int*>(g_smem + 3 * n_slots);
  for (int k = threadIdx.x; k < words; k += blockDim.x) prog[k] = prog_g[k];
  for (int k = threadIdx.x; k < 3 * n_slots; k += blockDim.x) g_smem[k] = 1.0 + k;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int rep = 0; rep < 8; ++rep) run_prog(prog, 0, threadIdx.x & 31);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / 8;
  } else if (busy) {
    double x = threadIdx.x, y = 1.0000001;
    for (int i = 0; i < 4000; ++i) x = __dadd_rn(__dmul_rn(x, y), 1e-9);
    if (x == 0.5) out[1] = 1;
  }
}

int main() {
  for (int R : {1, 4, 10, 20}) {
    // round r: lane l combines slots (r*64 + 2l, r*64 + 2l + 1) into slot (r+1)*64 + l (slot indices x3)
    std::vector<int> p(2 + (R + 1) * 64, 0);
    p[0] = R;
    for (int r = 0; r <= R; ++r)
      for (int l = 0; l < 32; ++l) {
        int a = r * 64 + 2 * l, b = a + 1, d = (r + 1) * 64 + l;
        if (r == R) { a = b = d = 8 * 64 + l; }
        p[2 + 64 * r + 2 * l] = 3 * d;
        p[2 + 64 * r + 2 * l + 1] = (3 * a) | ((3 * b) << 16);
      }
    int n_slots = (R + 2) * 64;
    int *dp; long long* dout;
    cudaMalloc(&dp, p.size() * 4); cudaMalloc(&dout, 16);
    cudaMemcpy(dp, p.data(), p.size() * 4, cudaMemcpyHostToDevice);
    size_t smem = 8 * 3 * n_slots + 4 * p.size();
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int busy = 0; busy < 2; ++busy) {
      bench<<<1, 768, smem>>>(dp, (int)p.size(), n_slots, busy, dout);
      long long h[2]; cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
      printf("rounds %2d busy %d: %lld cycles per replay, %.0f per round (%s)\n", R, busy, h[0], (double)h[0] / R,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
