// umma_probe.cu -- standalone check of the tcgen05.mma.kind::i8 operand
// descriptor conventions used by k_gemm.cu (K-major, no swizzle, core
// matrices of 8 rows x 16 bytes).  Each variant runs in its own process
// (argv[1]) so an illegal-instruction fault cannot poison the others.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 2; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}

// A: M x K bytes, B: N x K bytes, both pre-laid-out in smem image order.
// D[m][n] = sum_k A[m][k] * B[n][k]  (int32).  nk = K / 32 MMAs.
__global__ void probe_kernel(const int8_t* a_img, const int8_t* b_img, int a_bytes, int b_bytes,
                             int M, int N, int nk, uint32_t idesc, uint32_t a_lbo, uint32_t a_sbo,
                             uint32_t b_lbo, uint32_t b_sbo, uint32_t a_kstride, uint32_t b_kstride,
                             int32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + ((a_bytes + 1023) / 1024) * 1024;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid * 16; i < a_bytes; i += blockDim.x * 16) *(int4*)(sa + i) = *(const int4*)(a_img + i);
  for (int i = tid * 16; i < b_bytes; i += blockDim.x * 16) *(int4*)(sb + i) = *(const int4*)(b_img + i);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tb = tmem_base;
  if (tid == 0) {
    for (int k = 0; k < nk; k++) {
      uint32_t aaddr = smem_u32(sa) + k * a_kstride, baddr = smem_u32(sb) + k * b_kstride;
      uint64_t ad = (uint64_t)((aaddr & 0x3FFFF) >> 4) | ((uint64_t)(a_lbo >> 4) << 16) |
                    ((uint64_t)(a_sbo >> 4) << 32) | (1ull << 46);
      uint64_t bd = (uint64_t)((baddr & 0x3FFFF) >> 4) | ((uint64_t)(b_lbo >> 4) << 16) |
                    ((uint64_t)(b_sbo >> 4) << 32) | (1ull << 46);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                   :: "r"(tb), "l"(ad), "l"(bd), "r"(idesc), "r"(k));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    wait_parity(smem_u32(&bar), 0);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      uint32_t taddr = tb + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (row < M)
        for (int i = 0; i < 8; i++) out[row * N + c0 + i] = (int32_t)r[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(256));
}

// layout 0: [kstep][rowgroup][khalf][8][16]      (khalf stride 128, rowgroup stride 256)
// layout 1: [kstep][khalf][rowgroup][8][16]      (rowgroup stride 128, khalf stride R*16)
static void pack(const std::vector<int>& src, int R, int K, int layout, std::vector<int8_t>& img) {
  img.assign((size_t)R * K, 0);
  for (int r = 0; r < R; r++)
    for (int k = 0; k < K; k++) {
      int ks = k / 32, kh = (k % 32) / 16, kb = k % 16;
      size_t base = (size_t)ks * R * 32, off;
      if (layout == 0) off = base + (r / 8) * 256 + kh * 128 + (r % 8) * 16 + kb;
      else off = base + kh * (R * 16) + (r / 8) * 128 + (r % 8) * 16 + kb;
      img[off] = (int8_t)src[(size_t)r * K + k];
    }
}

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int N = argc > 2 ? atoi(argv[2]) : 64;
  int asgn = argc > 3 ? atoi(argv[3]) : 1, bsgn = argc > 4 ? atoi(argv[4]) : 1;
  int M = 128, K = 64;
  // variant bits: 0 -> layout (0/1); 1 -> swap lbo/sbo fields; 2 -> M field at bit 23 instead of 24
  int layout = variant & 1, swap = (variant >> 1) & 1, mbit = (variant & 4) ? 23 : 24;
  srand(1234 + variant);
  std::vector<int> A((size_t)M * K), B((size_t)N * K);
  for (auto& v : A) v = asgn ? (rand() % 256) - 128 : rand() % 256;
  for (auto& v : B) v = bsgn ? (rand() % 256) - 128 : rand() % 256;
  std::vector<int8_t> ai, bi;
  pack(A, M, K, layout, ai); pack(B, N, K, layout, bi);
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo;   // "lbo" = K-direction core-matrix stride, "sbo" = row-group stride
  if (layout == 0) { a_lbo = 128; a_sbo = 256; b_lbo = 128; b_sbo = 256; }
  else { a_lbo = M * 16; a_sbo = 128; b_lbo = N * 16; b_sbo = 128; }
  if (swap) { std::swap(a_lbo, a_sbo); std::swap(b_lbo, b_sbo); }
  uint32_t idesc = (2u << 4) | ((uint32_t)asgn << 7) | ((uint32_t)bsgn << 10) | ((uint32_t)(N >> 3) << 17) |
                   ((uint32_t)(M >> 4) << mbit);
  int8_t *da, *db; int32_t* dout;
  CK(cudaMalloc(&da, ai.size())); CK(cudaMalloc(&db, bi.size())); CK(cudaMalloc(&dout, (size_t)M * N * 4));
  CK(cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dout, 0, (size_t)M * N * 4));
  int smem = 64 * 1024;
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<<<1, 128, smem>>>(da, db, (int)ai.size(), (int)bi.size(), M, N, K / 32, idesc, a_lbo, a_sbo, b_lbo, b_sbo,
                                 M * 32, N * 32, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> out((size_t)M * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      long long s = 0;
      for (int k = 0; k < K; k++) s += (long long)A[(size_t)m * K + k] * B[(size_t)n * K + k];
      if (s != out[(size_t)m * N + n]) { if (bad < 3) printf("  mismatch m=%d n=%d want %lld got %d\n", m, n, s, out[(size_t)m * N + n]); bad++; }
    }
  printf("variant %d (layout %d swap %d mbit %d) N=%d a_s8=%d b_s8=%d: %s (%d bad)\n", variant, layout, swap, mbit, N,
         asgn, bsgn, bad ? "FAIL" : "PASS", bad);
  return bad ? 1 : 0;
}
