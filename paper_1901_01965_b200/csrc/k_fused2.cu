// k_fused2.cu -- K3F2: the rational F(2x2,3x3) path as ONE kernel from the
// Winograd-domain operands to the output: the 16 real GEMM planes on tcgen05 (kind::i8, int32 in
// TMEM), the reverse scaling M'' = rha(M m / 2^q), Y = A^T M'' A (A^T = [[1,1,1,0],
// [0,1,-1,-1]], A25), out32 = rha(Y / 4) (A26), requantisation (A14), crop and store.  M''
// never leaves the SM; the staged F(2x2) path writes and re-reads 64 B of it per (tile, cout).
//
// Operands: V in the staged F(2x2) layout ([tile block][plane][K step][hi, lo][4 KB], K2 unchanged);
// W' in the fused F(2x2) layout [32-cout block][plane][K step][W hi rows | W lo rows] (layout.cuh
// w_offset), so the two planes of a pair are contiguous in both.  Balanced s8 pieces, v = 256 hi + lo.
//
// Work unit = (128-tile block, 32-cout block): the 16 planes as 8 pairs; the output state is Y (4 words
// per (tile, cout)), 32 registers per epilogue thread, so the unit can be 32 couts wide (twice the
// complex fused kernel's) and its UMMAs are N = 64.  Per K step and plane: A_hi . [W hi | W lo] into
// [s16 | s8] and A_lo . [W hi | W lo] into [s8 | s0] (the plane's first lo UMMA overwrites [s8 | s0];
// the s16 block starts at zero and is re-zeroed by the epilogue after each read).
//
// Persistent CTAs (fewest for the unit rounds), 19 warps (<= 96 registers: 5 warps on some SM sub-partition):
//   warps 0..15  epilogue: TMEM lane quadrant w % 4 (32 tiles), couts 8 (w / 4) .. +7
//   warps 16, 17 producers (one elected lane each, alternate stages): V and W' bulk copies
//   warp 18      MMA issuer (one elected lane)
// Ring: 4 stages of 40 KB (one pair, 2 K steps) or, at K >= 4 steps, 2 stages of 80 KB (one pair,
// 4 K steps); a stage holding the pair's whole K range is one V copy and one W' copy.
// TMEM: 4 slots of 96 columns (one plane: [s16 | s8 | s0] x 32 couts), 128 columns spare.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <utility>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

// Debug-only subtraction switches (tools/README.md): 0 in every product build
#ifndef WINO_F2_NOFEED
#define WINO_F2_NOFEED 0   // no copies, no UMMAs: the epilogue and the barrier skeleton alone
#endif
#ifndef WINO_F2_NOFOLD
#define WINO_F2_NOFOLD 0   // no reverse scaling / output-transform arithmetic
#endif

namespace wino {

namespace {

constexpr int kN2 = 32;                         // couts per unit
constexpr int kC2 = 8;                          // couts per epilogue thread
constexpr int kE2Warps = 16, kP2Warps = 2;
constexpr int kP2Warp = kE2Warps, kM2Warp = kE2Warps + kP2Warps;
constexpr int kT2Threads = 32 * (kE2Warps + kP2Warps + 1);
constexpr uint32_t kRing2 = 163840;             // 160 KB of stages
constexpr int kSlots2 = 4, kSlotCols2 = 96;
constexpr uint32_t kPlaneW = 2 * kN2 * kKStep;  // W' bytes per plane and K step (64 rows x 32 B)
constexpr uint32_t kPlaneV = 2 * kVBlockBytes;  // V bytes per plane and K step (hi + lo)
constexpr int kE2Bar = 1;

inline size_t fused2_smem_bytes() { return kRing2 + 16 * kN2 * 4 + 1024; }

__device__ __forceinline__ void e2_barrier() {
  asm volatile("bar.sync %0, %1;" ::"n"(kE2Bar), "n"(kE2Warps * 32) : "memory");
}
__device__ __forceinline__ void tld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tzero8(uint32_t taddr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr), "r"(0)
               : "memory");
}
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// M'' = rha(v m / 2^q) as rha(v m' / 2^7), m' = m 2^(7-q) (q >= 3: m' <= 4080); m' = 128 is the identity
__device__ __forceinline__ int32_t rscale7(int32_t v, uint32_t mq) { return rha_mul_shr7(v, mq); }
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <typename F>
__device__ __forceinline__ void static_for16(F&& f) { static_for_impl(f, std::make_integer_sequence<int, 16>{}); }
// A[k][i] of the F(2,3) output transform, A^T = [[1,1,1,0],[0,1,-1,-1]]
__host__ __device__ constexpr int a2(int k, int i) { return i == 0 ? (k < 3 ? 1 : 0) : (k == 0 ? 0 : (k == 1 ? 1 : -1)); }

}  // namespace

// KC: K steps per stage (2 -> four 40 KB stages, 4 -> two 80 KB stages)
template <bool NHWC, bool OUT8, int KC>
__global__ void __launch_bounds__(kT2Threads, 1)
    k_fused2(const int8_t* __restrict__ V, const int8_t* __restrict__ W, const uint8_t* __restrict__ codes, Geom g,
             int n0, int imgs, int tblocks, int32_t rq_mult, int rq_shift, void* __restrict__ y) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kStg = KC == 2 ? 4 : 2;
  constexpr uint32_t kStgBytes = kRing2 / kStg, kStgV = 2 * KC * kPlaneV;   // V of a pair, then W' of the pair
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;   // warp-uniform: TMEM addresses in uniform registers
  uint32_t* etab = reinterpret_cast<uint32_t*>(smem + kRing2);           // [16 positions][32 couts] m'
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kRing2 + 16 * kN2 * 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStg + 2 * kSlots2);
  uint32_t* lut = tmem_slot + 4;                                          // 64: code -> m'
  const uint32_t sbase = smem_u32(smem);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStg);
  const uint32_t tfull0 = smem_u32(bars + 2 * kStg), tempty0 = smem_u32(bars + 2 * kStg + kSlots2);
  const int nblocks = g.cout_pad / kN2;
  const int n_units = tblocks * nblocks;
  const int ksteps = g.ksteps;

  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  if (threadIdx.x == 32 * kP2Warp) {
    for (int s = 0; s < kStg; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < kSlots2; b++) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, kE2Warps);
    }
    fence_mbar_init();
  }
  pdl_trigger();
  if (threadIdx.x < 64) {   // inverse factor of every 6-bit code (A8/A27); code 0 -> m' = 128
    int n, p, m = 128, q = 7;
    decode_code(threadIdx.x, n, p);
    if (n >= 8) inverse_factor(n, p, m, q);
    lut[threadIdx.x] = (uint32_t)m << (7 - q);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (warp < kE2Warps) {   // accumulator slots start at zero (the epilogue re-zeroes each after reading)
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * kC2;
    for (int b = 0; b < kSlots2; b++)
#pragma unroll
      for (int blk = 0; blk < 1; blk++) tzero8(lb + b * kSlotCols2 + blk * kN2);   // s16 blocks
    tst_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();   // V, W' and the codes come from the kernels just before

  if (warp >= kP2Warp && warp < kP2Warp + kP2Warps) {
    // ------------------------------------------------ producers: warp p issues the stages it with it % 2 == p
    const int pw = warp - kP2Warp;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int tb = u / nblocks, nb = u - tb * nblocks;
      for (int pr = 0; pr < 8; pr++) {
        const int8_t* v0 = V + ((long long)tb * 16 + 2 * pr) * ksteps * kPlaneV;
        const int8_t* w0 = W + ((long long)nb * 16 + 2 * pr) * ksteps * kPlaneW;
        for (int k0 = 0; k0 < ksteps; k0 += KC, it++) {
          if (it % kP2Warps != pw || WINO_F2_NOFEED) continue;
          const int s = it % kStg;
          mbar_wait(empty0 + 8 * s, ((it / kStg) & 1) ^ 1);
          const int kn = min(KC, ksteps - k0);
          const uint32_t st = sbase + s * kStgBytes;
          if (elect_one()) {
            const uint32_t vb = kn * kPlaneV, wb = kn * kPlaneW;
            mbar_arrive_expect_tx(full0 + 8 * s, 2 * (vb + wb));
            if (kn == ksteps) {   // the pair's whole K range: contiguous in V and in W'
              bulk_g2s(st, v0, 2 * vb, full0 + 8 * s);
              bulk_g2s(st + kStgV, w0, 2 * wb, full0 + 8 * s);
            } else {              // plane q at q * KC steps in the stage
              for (int q = 0; q < 2; q++) {
                bulk_g2s(st + q * KC * kPlaneV, v0 + ((long long)q * ksteps + k0) * kPlaneV, vb, full0 + 8 * s);
                bulk_g2s(st + kStgV + q * KC * kPlaneW, w0 + ((long long)q * ksteps + k0) * kPlaneW, wb,
                         full0 + 8 * s);
              }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == kM2Warp) {
    // ------------------------------------------------ MMA issuer (warp-uniform loop, one elected lane issues)
    const uint32_t id64 = idesc_i8(kMBlock, 2 * kN2, 1, 1);
    int it = 0, pc = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      for (int pr = 0; pr < 8; pr++, pc += 2) {
        const int b0 = pc % kSlots2, b1 = (pc + 1) % kSlots2;   // the pair's two slots
        mbar_wait(tempty0 + 8 * b0, ((pc / kSlots2) & 1) ^ 1);
        mbar_wait(tempty0 + 8 * b1, (((pc + 1) / kSlots2) & 1) ^ 1);
        tc_fence_after();
        for (int k0 = 0; k0 < ksteps; k0 += KC, it++) {
          const int s = it % kStg;
          if (!WINO_F2_NOFEED) mbar_wait(full0 + 8 * s, (it / kStg) & 1);
          tc_fence_after();
          const int kn = min(KC, ksteps - k0);
          const uint32_t st = sbase + s * kStgBytes;
          // stage layout: whole-K stages hold plane q at q * ksteps steps, chunked ones at q * KC steps
          const int qs = kn == ksteps ? ksteps : KC;
          if (!WINO_F2_NOFEED && elect_one()) {
            for (int q = 0; q < 2; ++q) {
              const uint32_t d = tmem + (q ? b1 : b0) * kSlotCols2;
              const uint32_t va = st + (uint32_t)(q * qs) * kPlaneV, wa = st + kStgV + (uint32_t)(q * qs) * kPlaneW;
              for (int kk = 0; kk < kn; ++kk) {
                const uint64_t ah = umma_desc(va + kk * kPlaneV, 128, 256);
                const uint64_t al = umma_desc(va + kk * kPlaneV + kVBlockBytes, 128, 256);
                const uint64_t bb = umma_desc(wa + kk * kPlaneW, 128, 256);
                // the plane's first K step overwrites [s8 | s0] (columns 32..95); s16 (0..31) was zeroed
                // by the epilogue, so only one of the three column blocks needs a TMEM store
                umma_i8(d + kN2, al, bb, id64, (k0 + kk) > 0);   // [s8 | s0]  (+)= lo . [W hi | W lo]
                umma_i8(d, ah, bb, id64, 1u);                    // [s16 | s8] +=   hi . [W hi | W lo]
              }
            }
            umma_commit(empty0 + 8 * s);   // stage reusable once these MMAs have read it
          }
          __syncwarp();
        }
        if (elect_one()) {
          umma_commit(tfull0 + 8 * (b0 >> 1));   // one commit for the pair's two slots (commits cost ~200 cycles)
        }
        __syncwarp();
      }
    }
  } else if (warp < kE2Warps) {
    // ------------------------------------------------ epilogue: thread = tile row x 8 couts
    const int quad = warp & 3, cw = warp >> 2;
    const int row = quad * 32 + lane;
    const int etid = threadIdx.x;                       // 0..511
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + cw * kC2;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int tb = u / nblocks, nb = u - tb * nblocks;
      e2_barrier();   // the previous unit's etab reads are done
      {               // this unit's reverse-scale entries: [16 positions][32 couts]
        const int p = etid / kN2, c = etid % kN2;
        const int co = nb * kN2 + c;
        const int code = (g.scaling && co < g.cout) ? codes[(long long)co * 16 + p] : 0;
        etab[etid] = lut[code & 63];
      }
      e2_barrier();
      int32_t Y[2][2][kC2];
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
          for (int c = 0; c < kC2; c++) Y[i][j][c] = 0;
      // Software-pipelined over the 16 planes: the TMEM loads of plane p + 1 are in flight while plane
      // p is scaled and folded into Y.  16 planes per unit over 4 slots: slot p % 4, phase (p / 4) & 1.
      uint32_t h[8], x[8], l[8];
      int32_t v[kC2];   // M of the plane being folded
      auto fetch = [&](auto pc) {   // wait for plane P's slot and start its three 8-column loads
        constexpr int P = decltype(pc)::value;
        // pair barrier (P / 2) % 2 (the pair's slots are 2 (P / 2 % 2) and +1), phase (P / 4) & 1
        if constexpr ((P & 1) == 0) mbar_wait(tfull0 + 8 * ((P >> 1) & 1), (P / kSlots2) & 1);
        tc_fence_after();
        const uint32_t a = lane_base + (P & (kSlots2 - 1)) * kSlotCols2;
        tld8(a, h);
        tld8(a + kN2, x);
        tld8(a + 2 * kN2, l);
      };
      auto land = [&](auto pc) {    // loads landed: re-zero s16, release the slot, compose M
        constexpr int P = decltype(pc)::value;
        tmem_ld_wait();
        tzero8(lane_base + (P & (kSlots2 - 1)) * kSlotCols2);   // s16 only: the first K step overwrites s8, s0
        tst_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty0 + 8 * (P & (kSlots2 - 1)));
#pragma unroll
        for (int c = 0; c < kC2; c++) v[c] = (int32_t)((h[c] << 16) + (x[c] << 8) + l[c]);
      };
      auto fold = [&](auto pc) {    // Y[i][j] += A[r][i] A[cc][j] M'' with M'' = rha(M m / 2^q)
        constexpr int P = decltype(pc)::value, r = P >> 2, cc = P & 3;
        if (WINO_F2_NOFOLD) return;
        const uint32_t* mm = etab + P * kN2 + cw * kC2;
#pragma unroll
        for (int c = 0; c < kC2; c++) {
          const int32_t mv = rscale7(v[c], mm[c]);
#pragma unroll
          for (int i = 0; i < 2; i++)
#pragma unroll
            for (int j = 0; j < 2; j++) {
              const int coef = a2(r, i) * a2(cc, j);   // in {-1, 0, 1}
              Y[i][j][c] += coef * mv;
            }
        }
      };
      fetch(std::integral_constant<int, 0>{});
      land(std::integral_constant<int, 0>{});
      static_for16([&](auto pc) {
        constexpr int P = decltype(pc)::value;
        if constexpr (P + 1 < 16) fetch(std::integral_constant<int, P + 1>{});
        fold(pc);
        if constexpr (P + 1 < 16) land(std::integral_constant<int, P + 1>{});
      });
      // ---- out32 = rha(Y / 4) (A26), requantisation (A14), crop, store
      const int t = tb * kMBlock + row;
      if (t >= imgs * g.tpi) continue;
      const int ti = fdiv(t, g.dv_tpi), rem = t - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
      const int img = n0 + ti, oy0 = 2 * ty, ox0 = 2 * (rem - ty * g.tw);
      const int ni = min(2, g.ho - oy0), nj = min(2, g.wo - ox0);
      const int co0 = nb * kN2 + cw * kC2;
      auto outv = [&](int32_t yv) -> int32_t {
        const int32_t o32 = (yv + 2 + (yv >> 31)) >> 2;   // rha(Y / 4)
        if (!OUT8) return o32;
        const long long pr = (long long)o32 * rq_mult;
        long long rr = pr;
        if (rq_shift > 0) {
          const long long aa = pr < 0 ? -pr : pr;
          const long long qq = (aa + (1ll << (rq_shift - 1))) >> rq_shift;
          rr = pr < 0 ? -qq : qq;
        }
        return (int32_t)(rr > 127 ? 127 : (rr < -128 ? -128 : rr));
      };
#pragma unroll
      for (int i = 0; i < 2; i++) {
        if (i >= ni) continue;
#pragma unroll
        for (int j = 0; j < 2; j++) {
          if (j >= nj) continue;
          const int oy = oy0 + i, ox = ox0 + j;
          if (NHWC) {
            const long long pix = ((long long)img * g.ho + oy) * g.wo + ox;
            if (OUT8) {
              int8_t* dst = static_cast<int8_t*>(y) + pix * g.cout + co0;
              if ((g.cout & 7) == 0 && co0 < g.cout) {
                uint32_t w0 = 0, w1 = 0;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                  w0 |= ((uint32_t)outv(Y[i][j][c]) & 0xffu) << (8 * c);
                  w1 |= ((uint32_t)outv(Y[i][j][c + 4]) & 0xffu) << (8 * c);
                }
                *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
              } else {
#pragma unroll
                for (int c = 0; c < kC2; c++)
                  if (co0 + c < g.cout) dst[c] = (int8_t)outv(Y[i][j][c]);
              }
            } else {
              int32_t* dst = static_cast<int32_t*>(y) + pix * g.cout + co0;
#pragma unroll
              for (int c = 0; c < kC2; c++)
                if (co0 + c < g.cout) dst[c] = outv(Y[i][j][c]);
            }
          } else {
#pragma unroll
            for (int c = 0; c < kC2; c++) {
              const int co = co0 + c;
              if (co >= g.cout) continue;
              const long long off = (((long long)img * g.cout + co) * g.ho + oy) * g.wo + ox;
              if (OUT8) static_cast<int8_t*>(y)[off] = (int8_t)outv(Y[i][j][c]);
              else static_cast<int32_t*>(y)[off] = outv(Y[i][j][c]);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

static int g_fused2_sms = 0;

cudaError_t launch_fused2(const Geom& g, long long tiles_pad_launch, int n0, int imgs, const int8_t* vimg,
                          const int8_t* wimg, const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y,
                          cudaStream_t st) {
  if (g.nblk != kN2 || g.alg != 1) return cudaErrorInvalidValue;
  const int tblocks = (int)(tiles_pad_launch / kMBlock);
  const int n_units = tblocks * (g.cout_pad / kN2);
  int grid = n_units < g_fused2_sms ? n_units : g_fused2_sms;
  const int rounds = (n_units + grid - 1) / grid;   // fewest CTAs for the same number of unit rounds
  grid = (n_units + rounds - 1) / rounds;
  const size_t smem = fused2_smem_bytes();
  const bool nhwc = g.layout == 1, out8 = g.out_mode == 0, k4 = g.ksteps >= 4;
  cudaError_t e;
#define WINO_KF2(A, B)                                                                                          \
  e = k4 ? launch_pdl(k_fused2<A, B, 4>, dim3(grid), dim3(kT2Threads), smem, st, vimg, wimg, codes, g, n0, imgs, \
                      tblocks, rq_mult, rq_shift, y)                                                            \
         : launch_pdl(k_fused2<A, B, 2>, dim3(grid), dim3(kT2Threads), smem, st, vimg, wimg, codes, g, n0, imgs, \
                      tblocks, rq_mult, rq_shift, y)
  if (nhwc) {
    if (out8) WINO_KF2(true, true);
    else WINO_KF2(true, false);
  } else {
    if (out8) WINO_KF2(false, true);
    else WINO_KF2(false, false);
  }
#undef WINO_KF2
  return e;
}

cudaError_t setup_fused2() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_fused2_sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = (int)fused2_smem_bytes();
#define WINO_KF2_ATTR(A, B)                                                                                     \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused2<A, B, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused2<A, B, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
  WINO_KF2_ATTR(true, true);
  WINO_KF2_ATTR(true, false);
  WINO_KF2_ATTR(false, true);
  WINO_KF2_ATTR(false, false);
#undef WINO_KF2_ATTR
  return e;
}

}  // namespace wino
