// k_gemm.cu -- K3: the Winograd-domain channel contraction: for
// each of the 46 operand planes p, M_p[tiles x Cout] = V_p[tiles x Cin] .
// W'_p[Cin x Cout], on the tcgen05 tensor cores (kind::i8, int32 accumulation
// in TMEM).  Every operand is split into an s8 high and a u8 low piece
// (layout.cuh), so one plane is four UMMAs per 32-channel K step into three
// TMEM accumulators:
//     acc_hh += Vhi . Whi          (weight 2^16)
//     acc_x  += Vhi . Wlo + Vlo . Whi   (weight 2^8)
//     acc_ll += Vlo . Wlo          (weight 1)
// and the epilogue forms M = 2^16 acc_hh + 2^8 acc_x + acc_ll (exact mod
// 2^32; the true |M| < 2^31 for Cin <= 896, A23).
//
// CTA = 128 threads, one (plane, 128-tile block, n_block-cout block):
//   warp 0 lane 0  producer: 1-D bulk copies (TMA engine) of whole pre-tiled
//                  K stages into shared memory, mbarrier complete_tx
//   warp 1 lane 0  MMA issuer: tcgen05.mma per K step, tcgen05.commit frees
//                  the stage
//   warps 0..3     epilogue: tcgen05.ld (warp w owns TMEM lanes 32w..32w+31)
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kStages = 4;
constexpr int kKStepsPerStage = 2;
constexpr uint32_t kABytesPerKStep = kMBlock * kKStep;   // 4096

__host__ __device__ inline uint32_t gemm_stage_bytes(int nblk) {
  return 2u * kKStepsPerStage * kABytesPerKStep + 2u * kKStepsPerStage * (uint32_t)nblk * kKStep;
}
__host__ __device__ inline uint32_t gemm_tmem_cols(int nblk) {
  uint32_t need = 3u * (uint32_t)nblk, c = 32;
  while (c < need) c <<= 1;
  return c;
}
inline size_t gemm_smem_bytes(int nblk) { return (size_t)kStages * gemm_stage_bytes(nblk) + 1024; }

__global__ void __launch_bounds__(128, 1)
    k_gemm(const int8_t* __restrict__ V, const int8_t* __restrict__ W, int32_t* __restrict__ M, int ksteps,
           long long tiles_pad, int cout_pad, int cin_pad, int nblk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tb = blockIdx.x, nb = blockIdx.y, plane = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_bytes = kKStepsPerStage * kABytesPerKStep;
  const uint32_t b_bytes = kKStepsPerStage * (uint32_t)nblk * kKStep;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages), done = smem_u32(bars + 2 * kStages);
  const uint32_t tmem_cols = gemm_tmem_cols(nblk);

  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), tmem_cols);
    tmem_relinquish();
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_it = (ksteps + kKStepsPerStage - 1) / kKStepsPerStage;

  if (warp == 0 && lane == 0) {
    // ---------------- producer
    const int8_t* vh = V + (long long)(2 * plane) * tiles_pad * cin_pad + (long long)tb * ksteps * kABytesPerKStep;
    const int8_t* vl = vh + tiles_pad * cin_pad;
    const int8_t* wh = W + (long long)(2 * plane) * cout_pad * cin_pad + (long long)nb * ksteps * nblk * kKStep;
    const int8_t* wl = wh + (long long)cout_pad * cin_pad;
    for (int it = 0; it < n_it; ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      mbar_wait(empty0 + 8 * s, ph ^ 1);
      const int k0 = it * kKStepsPerStage;
      const int kn = min(kKStepsPerStage, ksteps - k0);
      const uint32_t ab = kn * kABytesPerKStep, bb = kn * (uint32_t)nblk * kKStep;
      const uint32_t st = sbase + s * stage_bytes;
      mbar_arrive_expect_tx(full0 + 8 * s, 2 * ab + 2 * bb);
      bulk_g2s(st, vh + (long long)k0 * kABytesPerKStep, ab, full0 + 8 * s);
      bulk_g2s(st + a_bytes, vl + (long long)k0 * kABytesPerKStep, ab, full0 + 8 * s);
      bulk_g2s(st + 2 * a_bytes, wh + (long long)k0 * nblk * kKStep, bb, full0 + 8 * s);
      bulk_g2s(st + 2 * a_bytes + b_bytes, wl + (long long)k0 * nblk * kKStep, bb, full0 + 8 * s);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    const uint32_t id_ss = idesc_i8(kMBlock, nblk, 1, 1), id_su = idesc_i8(kMBlock, nblk, 1, 0);
    const uint32_t id_us = idesc_i8(kMBlock, nblk, 0, 1), id_uu = idesc_i8(kMBlock, nblk, 0, 0);
    const uint32_t acc_hh = tmem, acc_x = tmem + nblk, acc_ll = tmem + 2 * nblk;
    for (int it = 0; it < n_it; ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      const int k0 = it * kKStepsPerStage;
      const int kn = min(kKStepsPerStage, ksteps - k0);
      const uint32_t st = sbase + s * stage_bytes;
      for (int kk = 0; kk < kn; ++kk) {
        const uint32_t acc = (k0 + kk) > 0;
        const uint64_t a_hi = umma_desc(st + kk * kABytesPerKStep, 128, 256);
        const uint64_t a_lo = umma_desc(st + a_bytes + kk * kABytesPerKStep, 128, 256);
        const uint64_t b_hi = umma_desc(st + 2 * a_bytes + kk * nblk * kKStep, 128, 256);
        const uint64_t b_lo = umma_desc(st + 2 * a_bytes + b_bytes + kk * nblk * kKStep, 128, 256);
        umma_i8(acc_hh, a_hi, b_hi, id_ss, acc);
        umma_i8(acc_x, a_hi, b_lo, id_su, acc);
        umma_i8(acc_x, a_lo, b_hi, id_us, 1);
        umma_i8(acc_ll, a_lo, b_lo, id_uu, acc);
      }
      umma_commit(empty0 + 8 * s);   // stage reusable once these MMAs have read it
    }
    umma_commit(done);
  }
  __syncwarp();

  // ---------------- epilogue: M = 2^16 hh + 2^8 x + ll, int32 row-major [tile][cout]
  mbar_wait(done, 0);
  tc_fence_after();
  const long long row = (long long)tb * kMBlock + warp * 32 + lane;
  int32_t* mrow = M + ((long long)plane * tiles_pad + row) * cout_pad + (long long)nb * nblk;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < nblk; c0 += 16) {
    uint32_t h[16], x[16], l[16];
    tmem_ld16(lane_base + c0, h);
    tmem_ld16(lane_base + nblk + c0, x);
    tmem_ld16(lane_base + 2 * nblk + c0, l);
    tmem_ld_wait();
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] = (h[j] << 16) + (x[j] << 8) + l[j];
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<int4*>(mrow + c0 + j) = make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols);
}

cudaError_t launch_gemm(const Geom& g, long long tiles_pad_launch, const int8_t* vimg, const int8_t* wimg, int32_t* m,
                        cudaStream_t st) {
  dim3 grid((unsigned)(tiles_pad_launch / kMBlock), g.cout_pad / g.nblk, kPlanes);
  k_gemm<<<grid, 128, gemm_smem_bytes(g.nblk), st>>>(vimg, wimg, m, g.ksteps, g.chunk_tiles_pad, g.cout_pad, g.cin_pad,
                                                    g.nblk);
  return cudaGetLastError();
}

cudaError_t setup_gemm() {
  return cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes(128));
}

}  // namespace wino
