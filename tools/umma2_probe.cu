// umma2_probe.cu -- standalone check of the 2-SM (CTA pair) tcgen05.mma.cta_group::2.kind::i8 conventions a
// paired staged GEMM would use: a cluster of 2 CTAs, each holding its own 128 rows of A and one half of the N
// rows of B in shared memory (same offsets in both CTAs); the leader (rank 0) issues the MMA with M = 256; a
// multicast commit arrives on both CTAs' mbarriers; each CTA reads its 128 x N accumulator rows from its TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma2_probe umma2_probe.cu && ./umma2_probe [N]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 2; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}

// a_img: per rank, 128 x K bytes in the canonical K-major layout ([kstep][rowgroup][khalf][8][16]);
// b_img: per rank, (N/2) x K bytes, same layout
__global__ void __cluster_dims__(2, 1, 1) probe2(const int8_t* a_img, const int8_t* b_img, int a_bytes, int b_bytes,
                                               int N, int nk, uint32_t idesc, int32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + ((a_bytes + 1023) / 1024) * 1024;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const uint32_t rank = cta_rank();
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  const int8_t* ai = a_img + (size_t)rank * a_bytes;
  const int8_t* bi = b_img + (size_t)rank * b_bytes;
  for (int i = tid * 16; i < a_bytes; i += blockDim.x * 16) *(int4*)(sa + i) = *(const int4*)(ai + i);
  for (int i = tid * 16; i < b_bytes; i += blockDim.x * 16) *(int4*)(sb + i) = *(const int4*)(bi + i);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  if (rank == 0 && tid == 0) {
    for (int k = 0; k < nk; k++) {
      const uint64_t ad = desc(smem_u32(sa) + k * 128 * 32, 128, 256);
      const uint64_t bd = desc(smem_u32(sb) + k * (N / 2) * 32, 128, 256);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p; }"
                   :: "r"(tb), "l"(ad), "l"(bd), "r"(idesc), "r"(k));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(&bar)), "h"((uint16_t)3));
  }
  if (tid == 0) wait_parity(smem_u32(&bar), 0);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      const uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; i++) out[((size_t)rank * 128 + row) * N + c0 + i] = (int32_t)r[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(256));
}

static void pack(const std::vector<int>& src, int r0, int R, int K, std::vector<int8_t>& img, size_t base) {
  for (int r = 0; r < R; r++)
    for (int k = 0; k < K; k++) {
      const int ks = k / 32, kh = (k % 32) / 16, kb = k % 16;
      img[base + (size_t)ks * R * 32 + (r / 8) * 256 + kh * 128 + (r % 8) * 16 + kb] = (int8_t)src[(size_t)(r0 + r) * K + k];
    }
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 128;
  const int M = 256, K = 64;
  srand(4321);
  std::vector<int> A((size_t)M * K), B((size_t)N * K);
  for (auto& v : A) v = (rand() % 256) - 128;
  for (auto& v : B) v = (rand() % 256) - 128;
  const int a_bytes = 128 * K, b_bytes = (N / 2) * K;
  std::vector<int8_t> ai(2 * (size_t)a_bytes), bi(2 * (size_t)b_bytes);
  for (int rk = 0; rk < 2; rk++) {
    pack(A, rk * 128, 128, K, ai, (size_t)rk * a_bytes);
    pack(B, rk * (N / 2), N / 2, K, bi, (size_t)rk * b_bytes);
  }
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  int8_t *da, *db; int32_t* dout;
  CK(cudaMalloc(&da, ai.size())); CK(cudaMalloc(&db, bi.size())); CK(cudaMalloc(&dout, (size_t)M * N * 4));
  CK(cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dout, 0, (size_t)M * N * 4));
  const int smem = 64 * 1024;
  CK(cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe2<<<2, 128, smem>>>(da, db, a_bytes, b_bytes, N, K / 32, idesc, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> out((size_t)M * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      long long s = 0;
      for (int k = 0; k < K; k++) s += (long long)A[(size_t)m * K + k] * B[(size_t)n * K + k];
      if (s != out[(size_t)m * N + n]) {
        if (bad < 4) printf("  mismatch m=%d n=%d want %lld got %d\n", m, n, s, out[(size_t)m * N + n]);
        bad++;
      }
    }
  printf("cta_group::2 kind::i8 M=256 N=%d K=%d: %s (%d bad of %d)\n", N, K, bad ? "FAIL" : "PASS", bad, M * N);
  return bad ? 1 : 0;
}
