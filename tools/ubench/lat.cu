// Micro-benchmarks of the latencies that bound one relaxation iteration on
// B200: dependent FP64 chains, IEEE div/sqrt, LDS, L2-hit LDG, CTA barrier,
// and a DSMEM st.async + mbarrier ping-pong between the 2 CTAs of a cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void fp64_chain(double* out, double a, double b, long long* cyc) {
  double x = a, y = b;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = __dadd_rn(x, y); }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = __dmul_rn(x, y); }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = __fma_rn(x, y, a); }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) { x = __ddiv_rn(y, x); }
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) { x = __dsqrt_rn(x); }
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = (t4 - t3) * 10; cyc[4] = (t5 - t4) * 10; }
}

__global__ void mem_chain(const int* __restrict__ g, int* out, long long* cyc, int n) {
  __shared__ int s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (i * 7 + 1) & 4095;
  __syncthreads();
  int p = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) p = s[p];
  long long t1 = clock64();
  int q = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) q = __ldg(g + q);
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) __syncthreads();
  long long t3 = clock64();
  out[threadIdx.x] = p + q;
  if (threadIdx.x == 0) { cyc[5] = t1 - t0; cyc[6] = (t2 - t1) * 5; cyc[7] = t3 - t2; }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) pingpong(long long* cyc, int iters) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ double buf[4];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  uint32_t peer_buf, peer_bar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_buf) : "r"(smem_u32(buf)), "r"(rank ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_bar) : "r"(smem_u32(&bar)), "r"(rank ^ 1));
  uint32_t ph = 0;
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" :: "r"(smem_u32(&bar)) : "memory");
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (rank == (unsigned)(i & 1)) {
      if (threadIdx.x == 0)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(peer_buf), "l"((long long)i), "r"(peer_bar) : "memory");
    } else {
      uint32_t done = 0;
      while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" :: "r"(smem_u32(&bar)) : "memory");
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (rank == 0 && threadIdx.x == 0) cyc[8] = (t1 - t0) / iters;  // one-way hop incl. re-arm
  cl.sync();
}

int main() {
  double* d; long long* c; int* g; int* o;
  cudaMalloc(&d, 1 << 16); cudaMalloc(&c, 1024); cudaMalloc(&o, 1 << 16);
  const int n = 1 << 20;
  cudaMalloc(&g, n * sizeof(int));
  int* h = (int*)malloc(n * sizeof(int));
  for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 7919 + 104729) % n);
  cudaMemcpy(g, h, n * sizeof(int), cudaMemcpyHostToDevice);
  fp64_chain<<<1, 32>>>(d, 1.0000001, 1e-9, c);
  mem_chain<<<1, 512>>>(g, o, c, n);
  mem_chain<<<1, 512>>>(g, o, c, n);  // second run: L2 warm
  pingpong<<<2, 32>>>(c, 2000);
  cudaDeviceSynchronize();
  long long hc[16];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("cycles per op: DADD %.1f DMUL %.1f DFMA %.1f DDIV(ieee) %.1f DSQRT(ieee) %.1f LDS %.1f LDG(L2) %.1f BAR.SYNC(512) %.1f st.async->mbarrier hop %lld\n",
         hc[0] / 1000.0, hc[1] / 1000.0, hc[2] / 1000.0, hc[3] / 1000.0, hc[4] / 1000.0, hc[5] / 1000.0, hc[6] / 1000.0, hc[7] / 1000.0, hc[8]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
