// pipe_bench.cu -- the fused kernel's load ring in isolation: a producer lane streams stages of
// (V copy of vb bytes, optional W' copy of wb bytes) into a ring of R stages; a consumer lane waits
// for each stage and releases it (plain mbarrier arrive, or tcgen05.commit like the MMA warp).
// 148 CTAs; groups of 4 consecutive CTAs read the same V addresses (4 cout blocks of a tile block);
// W' is shared by all CTAs.  Prints ns per stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}
extern __shared__ __align__(1024) uint8_t dsm[];
__global__ void k(const uint8_t* V, const uint8_t* W, int n, int R, int vb, int wb, int commit, int share,
                  long long* cyc, int nprod) {
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int stage = vb + wb;
  const uint8_t* vbase = V + (long long)(blockIdx.x / share) * n * (long long)vb % (30ll << 20);
  long long t0 = clock64();
  if (warp >= 2 && warp < 2 + nprod && lane == 0) {
    for (int it = warp - 2; it < n; it += nprod) {
      const int s = it % R;
      wait(su32(&empty[s]), ((it / R) & 1) ^ 1);
      const uint32_t f = su32(&full[s]), dst = su32(dsm) + s * stage;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(f), "r"(vb + wb) : "memory");
      const uint8_t* vs = V + ((vbase - V) + (long long)it * vb) % (30ll << 20);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "l"(vs), "r"(vb), "r"(f) : "memory");
      if (wb)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst + vb), "l"(W + ((long long)it * wb) % (448 << 10)), "r"(wb), "r"(f) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < n; it++) {
      const int s = it % R;
      wait(su32(&full[s]), (it / R) & 1);
      if (commit)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&empty[s])) : "memory");
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[s])) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(32));
}
int main() {
  uint8_t *V, *W; cudaMalloc(&V, 32 << 20); cudaMalloc(&W, 1 << 20);
  cudaMemset(V, 1, 32 << 20); cudaMemset(W, 2, 1 << 20);
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct C { int R, vb, wb, commit, share; const char* note; };
  C cs[] = {{4, 32768, 8192, 0, 4, "fused now (arrive)"}, {4, 32768, 0, 0, 4, "V only"},
            {8, 16384, 4096, 0, 4, "8 x 20K"}, {4, 16384, 2048, 0, 4, "real-group size"}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 400;
  for (int nctas : {148, 1})
  for (int np : {1, 2, 4})
  for (auto c : cs) {
    int smem = c.R * (c.vb + c.wb);
    k<<<nctas, 192, smem>>>(V, W, n, c.R, c.vb, c.wb, c.commit, c.share, cyc, np);
    cudaEventRecord(e0);
    k<<<nctas, 192, smem>>>(V, W, n, c.R, c.vb, c.wb, c.commit, c.share, cyc, np);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("ctas %3d nprod %d R=%d V=%5d W=%5d %-6s share=%d: %6.1f ns/stage %6.1f B/cyc/SM (%s) %s\n", nctas, np,
           c.R, c.vb, c.wb, c.commit ? "commit" : "arrive", c.share, ms * 1e6 / n,
           (double)(c.vb + c.wb) * n / (ms * 1e-3 * 1.965e9), c.note, cudaGetErrorString(err));
  }
  return 0;
}
