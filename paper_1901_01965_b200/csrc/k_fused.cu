// k_fused.cu -- K3F: the Winograd-domain channel contraction on the
// tcgen05 tensor cores FUSED with the Karatsuba recombination,
// the reverse scaling M'' = rha(M m / 2^q), the real-only
// output transform Y = A^T M'' A, out32 = rha(Y / 16)
// (A2, A11), crop, requantisation (A14) and the store.  M'' never leaves the SM:
// the staged path (k_gemm.cu + k_output.cu) writes and re-reads 144 bytes per
// (tile, cout) through HBM, this kernel writes 1 (int8) or 4 (int32).
//
// Work unit = (128-tile block, 16-cout block).  A unit runs all 46 GEMM planes
// (16 real positions, 10 complex primaries x 3 Karatsuba planes) of its tiles
// and couts, row by row of the 6x6 Winograd grid, in the order
//   rows r = 0, 5, 1, 2: real (r,0) (r,1) (r,2) (r,5), then the primary (r,3)
//   row 3:               primaries (3,0) (3,1) (3,2) (3,5) (3,3) (3,4)
// Operand pieces and UMMA layouts are those of layout.cuh: per plane and
// 32-channel K step four kind::i8 UMMAs (M = 128 tiles, N = 16 couts, K = 32)
// into three int32 TMEM accumulators hh / x / ll, so
//   M_p = 2^16 hh + 2^8 x + ll  (exact mod 2^32; true values fit, A23).
//
// Output transform (A^T rows a_0 = (1,1,1,1,1,0), a_1 = (0,1,-1,i,-i,0),
// a_2 = (0,1,1,-1,-1,0), a_3 = (0,1,-1,-i,i,1); a_j[4] = conj a_j[3]), done as
// in k_output.cu but row by row as the rows arrive:
//   Z_r[j] = sum_c M''[r][c] a_j[c]   (real for r in {0,1,2,5}: the pair at
//            columns 3/4 gives 2 Re(i^j z); complex for r = 3)
//   Y[0] = Z_0 + P + 2 Re Z_3   Y[1] = Q - 2 Im Z_3   Y[2] = P - 2 Re Z_3
//   Y[3] = Q + Z_5 + 2 Im Z_3,  P = Z_1 + Z_2, Q = Z_1 - Z_2
// (row 4 = conj row 3 is never formed).  Z_0, Z_5, P, Q are parked in
// spare TMEM columns as soon as they are complete, Re/Im Z_3 stay in registers,
// and the unit ends by reading them back once and storing y.
//
// Persistent CTA per SM, warp-specialised (18 warps, <= 96 registers):
//   warps 0..15  epilogue: warp w owns TMEM lane quadrant w % 4 (32 tiles) and
//                couts 4 (w / 4) .. +3 of the unit; thread = (tile, 4 couts)
//   warp 16      producer (1 lane): 1-D bulk copies (TMA engine) of the pre-tiled
//                V blocks and W' rows into a kFStages-deep shared-memory ring
//   warp 17      MMA issuer (1 lane): tcgen05.mma into a ring of kFAccSlots plane
//                accumulators (3 x 16 TMEM columns each), tcgen05.commit ->
//                stage free / accumulator full
// TMEM: columns [0, 240) accumulator ring, [256, 512) row partials
// [Z_0 | P | Q | Z_5][cw 0..3][j 0..3][c 0..3].
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kFN = 16;                       // couts per unit = UMMA N
constexpr int kFEpiWarps = 16;                // 4 per TMEM lane quadrant
constexpr int kFC = kFN / (kFEpiWarps / 4);   // couts per epilogue thread (4)
constexpr int kFProducerWarp = kFEpiWarps, kFMmaWarp = kFEpiWarps + 1;
constexpr int kFThreads = 32 * (kFEpiWarps + 2);
constexpr int kFStages = 8;
constexpr int kFKPerStage = 2;                // K steps (32 channels each) per ring stage
constexpr int kFAccSlots = 5;                 // TMEM plane-accumulator ring
constexpr int kFAccCols = 3 * kFN;            // hh, x, ll
constexpr uint32_t kFPartCol = 256;           // row partials Z_0, P, Q, Z_5 (64 columns each)
constexpr int kFPlanes = 46;
constexpr int kFGroups = 26;                  // 16 real positions + 10 primaries
constexpr uint32_t kFA = kFKPerStage * kMBlock * kKStep;     // one A piece per stage (8 KB)
constexpr uint32_t kFB = kFKPerStage * kFN * kKStep;         // one B piece per stage (1 KB)
constexpr uint32_t kFStageBytes = 2 * kFA + 2 * kFB;
constexpr uint32_t kFStagingBytes = kMBlock * 16 * kFN;      // int8 output tile: [16 px][128 tiles][16 couts]
constexpr uint32_t kFETabBytes = 2 * kFGroups * kFN * 4;     // m' per (group, cout), 2 units
constexpr int kFEpiBar = 1;
static_assert(kFAccSlots * kFAccCols <= (int)kFPartCol, "accumulator ring overlaps the partials");

inline size_t fused_smem_bytes() {
  return (size_t)kFStages * kFStageBytes + kFStagingBytes + kFETabBytes + 512;
}

// real rows in processing order (index ri into R = {0,1,2,5}): r = 0, 5, 1, 2
__host__ __device__ constexpr int frow(int k) { return k == 0 ? 0 : (k == 1 ? 3 : k - 1); }
// i-th plane of a unit in processing order
__host__ __device__ constexpr int fplane(int i) {
  return i < 28 ? ((i % 7) < 4 ? frow(i / 7) * 4 + (i % 7) : kRealPlanes + 3 * frow(i / 7) + (i % 7) - 4) : i;
}
// position index (r*6 + c) of group g: g < 20: real row ri = g/5, slot g%5 (4 = primary (R[ri],3));
// g >= 20: primary 4 + g-20
__device__ __forceinline__ int fgroup_pos(int g) {
  return g < 20 ? ((g % 5) < 4 ? real_pos((g / 5) * 4 + g % 5) : cpx_pos(g / 5)) : cpx_pos(4 + g - 20);
}

__device__ __forceinline__ void fepi_barrier() {
  asm volatile("bar.sync %0, %1;" ::"n"(kFEpiBar), "n"(kFEpiWarps * 32) : "memory");
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const int32_t (&v)[4][4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0][0]), "r"(v[0][1]), "r"(v[0][2]), "r"(v[0][3]), "r"(v[1][0]), "r"(v[1][1]), "r"(v[1][2]),
      "r"(v[1][3]), "r"(v[2][0]), "r"(v[2][1]), "r"(v[2][2]), "r"(v[2][3]), "r"(v[3][0]), "r"(v[3][1]),
      "r"(v[3][2]), "r"(v[3][3])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[4][4]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]),
        "=r"(v[1][3]), "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[3][0]), "=r"(v[3][1]),
        "=r"(v[3][2]), "=r"(v[3][3])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// M'' = rha(v m / 2^q) (A9) evaluated as rha(v m' / 2^7) with
// m' = m 2^(7-q) (q in [4,7], so m' <= 2040): one constant per (position, cout)
// and a fixed shift.  rha(p / 2^7) = (p + 64 - [p < 0]) >> 7 (floor shift).  The
// unscaled code is m' = 128, which returns v.
__device__ __forceinline__ int32_t frscale(int32_t v, uint32_t mq) {
  const long long p = (long long)v * (long long)mq + (long long)(64 + (v >> 31));
  return (int32_t)(p >> 7);
}

__device__ __forceinline__ void fwait(uint32_t bar, uint32_t parity, int dbg) {
  if (dbg & 64) mbar_spin(bar, parity); else mbar_wait(bar, parity);
}

// a_k[c] for the real indices c in {0,1,2,5}
__host__ __device__ constexpr int areal(int k, int c) {
  return c == 0 ? (k == 0) : (c == 1 ? 1 : (c == 2 ? ((k & 1) ? -1 : 1) : (k == 3)));
}
// i^n (x + iy) = (re_x x + re_y y) + i (im_x x + im_y y)
__host__ __device__ constexpr int re_x(int n) { return (n & 3) == 0 ? 1 : ((n & 3) == 2 ? -1 : 0); }
__host__ __device__ constexpr int re_y(int n) { return (n & 3) == 1 ? -1 : ((n & 3) == 3 ? 1 : 0); }
__host__ __device__ constexpr int im_x(int n) { return (n & 3) == 1 ? 1 : ((n & 3) == 3 ? -1 : 0); }
__host__ __device__ constexpr int im_y(int n) { return re_x(n); }

template <bool NHWC, bool OUT8, bool RQFAST>
__global__ void __launch_bounds__(kFThreads, 1)
    k_fused(const int8_t* __restrict__ V, const int8_t* __restrict__ W, const uint8_t* __restrict__ codes, Geom g,
            int n0, int imgs, int tblocks, int32_t rq_mult, int rq_shift, void* __restrict__ y, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* staging = smem + kFStages * kFStageBytes;
  uint32_t* etab = reinterpret_cast<uint32_t*>(staging + kFStagingBytes);    // [2][26][16] m'
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(etab) + kFETabBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kFStages + 2 * kFAccSlots);
  uint32_t* lut = tmem_slot + 4;                                             // 64: code -> m' = m 2^(7-q)
  const uint32_t sbase = smem_u32(smem);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kFStages);
  const uint32_t tfull0 = smem_u32(bars + 2 * kFStages), tempty0 = smem_u32(bars + 2 * kFStages + kFAccSlots);
  const int nblocks = g.cout_pad / kFN;
  const int n_units = tblocks * nblocks;
  const int ksteps = g.ksteps;
  const int n_it = (ksteps + kFKPerStage - 1) / kFKPerStage;

  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  if (threadIdx.x == 32 * kFProducerWarp) {
    for (int s = 0; s < kFStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < kFAccSlots; b++) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, kFEpiWarps);
    }
    fence_mbar_init();
  }
  pdl_trigger();
  if (threadIdx.x < 64) {   // inverse factor of every 6-bit code (A8); code 0 -> m' = 128: identity
    int n, p, m = 128, q = 7;
    decode_code(threadIdx.x, n, p);
    if (n >= 8) inverse_factor(n, p, m, q);
    lut[threadIdx.x] = (uint32_t)m << (7 - q);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // V (and W', codes) come from the kernels just before

  if (warp == kFProducerWarp) {
    if (lane == 0) {
      // ------------------------------------------------ producer
      const long long pstride = (long long)g.cout_pad * g.cin_pad;   // one W' plane-piece
      int it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int tb = u / nblocks, nb = u - tb * nblocks;
        const int8_t* vt = V + (long long)tb * ksteps * (2 * kPlanes) * kVBlockBytes;
        const int8_t* wt = W + (long long)nb * ksteps * kFN * kKStep;
        for (int i = 0; i < kFPlanes; i++) {
          const int plane = fplane(i);
          const int8_t* vblk = vt + (long long)(2 * plane) * kVBlockBytes;
          const int8_t* wh = wt + (long long)(2 * plane) * pstride;
          for (int ks = 0; ks < n_it; ks++, it++) {
            const int s = it % kFStages;
            fwait(empty0 + 8 * s, ((it / kFStages) & 1) ^ 1, dbg);
            const int k0 = ks * kFKPerStage;
            const int kn = min(kFKPerStage, ksteps - k0);
            const uint32_t st = sbase + s * kFStageBytes;
            if (dbg & 32) {   // debug: no copies (synchronisation cost only)
              mbar_arrive(full0 + 8 * s);
              continue;
            }
            mbar_arrive_expect_tx(full0 + 8 * s, kn * (2 * kVBlockBytes + 2 * kFN * kKStep));
            if (dbg & 16) {   // debug: the same bytes as one contiguous copy
              bulk_g2s(st, vt + (long long)(it & 63) * kFStageBytes, kn * (2 * kVBlockBytes + 2 * kFN * kKStep),
                       full0 + 8 * s);
              continue;
            }
            for (int kk = 0; kk < kn; kk++) {
              const int8_t* src = vblk + (long long)(k0 + kk) * (2 * kPlanes) * kVBlockBytes;
              bulk_g2s(st + kk * kVBlockBytes, src, kVBlockBytes, full0 + 8 * s);                       // hi
              bulk_g2s(st + kFA + kk * kVBlockBytes, src + kVBlockBytes, kVBlockBytes, full0 + 8 * s);  // lo
            }
            const uint32_t bb = kn * kFN * kKStep;
            bulk_g2s(st + 2 * kFA, wh + (long long)k0 * kFN * kKStep, bb, full0 + 8 * s);
            bulk_g2s(st + 2 * kFA + kFB, wh + pstride + (long long)k0 * kFN * kKStep, bb, full0 + 8 * s);
          }
        }
      }
    }
  } else if (warp == kFMmaWarp) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      const uint32_t id_ss = idesc_i8(kMBlock, kFN, 1, 1), id_su = idesc_i8(kMBlock, kFN, 1, 0);
      const uint32_t id_us = idesc_i8(kMBlock, kFN, 0, 1), id_uu = idesc_i8(kMBlock, kFN, 0, 0);
      int it = 0, pc = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        for (int i = 0; i < kFPlanes; i++, pc++) {
          const int b = pc % kFAccSlots;
          fwait(tempty0 + 8 * b, ((pc / kFAccSlots) & 1) ^ 1, dbg);   // epilogue drained this slot
          tc_fence_after();
          const uint32_t acc_hh = tmem + b * kFAccCols, acc_x = acc_hh + kFN, acc_ll = acc_hh + 2 * kFN;
          for (int ks = 0; ks < n_it; ks++, it++) {
            const int s = it % kFStages;
            fwait(full0 + 8 * s, (it / kFStages) & 1, dbg);
            tc_fence_after();
            const int k0 = ks * kFKPerStage;
            const int kn = min(kFKPerStage, ksteps - k0);
            const uint32_t st = sbase + s * kFStageBytes;
            for (int kk = 0; kk < kn && !(dbg & 2); ++kk) {
              const uint32_t acc = (k0 + kk) > 0;
              const uint64_t a_hi = umma_desc(st + kk * kVBlockBytes, 128, 256);
              const uint64_t a_lo = umma_desc(st + kFA + kk * kVBlockBytes, 128, 256);
              const uint64_t b_hi = umma_desc(st + 2 * kFA + kk * kFN * kKStep, 128, 256);
              const uint64_t b_lo = umma_desc(st + 2 * kFA + kFB + kk * kFN * kKStep, 128, 256);
              umma_i8(acc_hh, a_hi, b_hi, id_ss, acc);
              umma_i8(acc_x, a_hi, b_lo, id_su, acc);
              umma_i8(acc_x, a_lo, b_hi, id_us, 1);
              umma_i8(acc_ll, a_lo, b_lo, id_uu, acc);
            }
            umma_commit(empty0 + 8 * s);   // stage reusable once these MMAs have read it
          }
          umma_commit(tfull0 + 8 * b);     // plane accumulator complete
        }
      }
    }
  } else if (warp < kFEpiWarps) {
    // ------------------------------------------------ epilogue
    const int quad = warp & 3, cw = warp >> 2;
    const int row = quad * 32 + lane;                 // tile within the unit
    const int etid = threadIdx.x;                     // 0..511
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + cw * kFC;
    const uint32_t part = tmem + ((uint32_t)(quad * 32) << 16) + kFPartCol + cw * 16;
    int pc = 0;
    // one plane: M = 2^16 hh + 2^8 x + ll for this thread's 4 couts
    auto take = [&](int32_t (&v)[kFC]) {
      const int b = pc % kFAccSlots;
      fwait(tfull0 + 8 * b, (pc / kFAccSlots) & 1, dbg);
      tc_fence_after();
      const uint32_t a = lane_base + b * kFAccCols;
      uint32_t h[kFC], x[kFC], l[kFC];
      tmem_ld4(a, h);
      tmem_ld4(a + kFN, x);
      tmem_ld4(a + 2 * kFN, l);
      if (!(dbg & 4)) tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * b);
#pragma unroll
      for (int j = 0; j < kFC; j++) v[j] = (int32_t)((h[j] << 16) + (x[j] << 8) + l[j]);
      pc++;
    };
    // fill the m' table of unit u into buffer buf
    auto fill_etab = [&](int u, int buf) {
      if (u < n_units && etid < kFGroups * kFN) {
        const int grp = etid / kFN, c = etid % kFN;
        const int co = (u % nblocks) * kFN + c;
        const int code = (g.scaling && co < g.cout) ? codes[(long long)co * 36 + fgroup_pos(grp)] : 0;
        etab[buf * kFGroups * kFN + etid] = lut[code & 63];
      }
    };
    auto rscale = [&](int32_t (&v)[kFC], const uint32_t* tb, int grp) {
      const uint4 m = *reinterpret_cast<const uint4*>(tb + grp * kFN + cw * kFC);
      v[0] = frscale(v[0], m.x);
      v[1] = frscale(v[1], m.y);
      v[2] = frscale(v[2], m.z);
      v[3] = frscale(v[3], m.w);
    };
    // Karatsuba primary: P0 = Re.Re, P1 = Im.Im, P2 = (Re+Im)(Re+Im) -> Re = P0 - P1, Im = P2 - P0 - P1,
    // then the reverse scale on Re and Im (A10)
    auto take_cpx = [&](int32_t (&re)[kFC], int32_t (&im)[kFC], const uint32_t* tb, int grp) {
      int32_t v[kFC];
      take(re);
      take(v);
#pragma unroll
      for (int j = 0; j < kFC; j++) { re[j] -= v[j]; v[j] = re[j] + 2 * v[j]; }   // Re = P0 - P1; v = P0 + P1
      take(im);
#pragma unroll
      for (int j = 0; j < kFC; j++) im[j] -= v[j];
      rscale(re, tb, grp);
      rscale(im, tb, grp);
    };
    // Z_r[j][c] of real row R[ri]: real (r, cc) adds a_j[cc] M''; the pair at (r,3)/(r,4) adds 2 Re(i^j z)
    auto real_row = [&](auto ric, int32_t (&Z)[4][kFC], const uint32_t* tb) {
      constexpr int ri = decltype(ric)::value;
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < kFC; c++) Z[j][c] = 0;
#pragma unroll
      for (int s = 0; s < 4; s++) {
        const int cc = s == 3 ? 5 : s;
        int32_t m[kFC];
        take(m);
        rscale(m, tb, ri * 5 + s);
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int c = 0; c < kFC; c++) Z[j][c] += areal(j, cc) * m[c];
      }
      int32_t re[kFC], im[kFC];
      take_cpx(re, im, tb, ri * 5 + 4);
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < kFC; c++) Z[j][c] += 2 * re_x(j) * re[c] + 2 * re_y(j) * im[c];
    };

    if (dbg & 8) {   // debug: accumulator handshake only
      for (int u = blockIdx.x; u < n_units; u += gridDim.x)
        for (int i = 0; i < kFPlanes; i++, pc++) {
          const int b = pc % kFAccSlots;
          fwait(tfull0 + 8 * b, (pc / kFAccSlots) & 1, dbg);
          tc_fence_after();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty0 + 8 * b);
        }
    } else {
    fill_etab(blockIdx.x, 0);
    int k = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, k++) {
      fepi_barrier();                                  // etab[k & 1] visible; staging free
      fill_etab(u + gridDim.x, (k + 1) & 1);
      const uint32_t* tb = etab + (k & 1) * kFGroups * kFN;
      {
        int32_t Z[4][kFC];
        real_row(std::integral_constant<int, 0>{}, Z, tb);   // row 0
        tmem_st16(part + 0 * 64, Z);
        real_row(std::integral_constant<int, 3>{}, Z, tb);   // row 5
        tmem_st16(part + 3 * 64, Z);
      }
      {
        int32_t Z1[4][kFC], Z2[4][kFC];
        real_row(std::integral_constant<int, 1>{}, Z1, tb);  // row 1
        real_row(std::integral_constant<int, 2>{}, Z2, tb);  // row 2
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int c = 0; c < kFC; c++) {
            const int32_t p = Z1[j][c] + Z2[j][c], q = Z1[j][c] - Z2[j][c];
            Z1[j][c] = p;
            Z2[j][c] = q;
          }
        tmem_st16(part + 1 * 64, Z1);   // P
        tmem_st16(part + 2 * 64, Z2);   // Q
      }
      // ---- row 3: Z_3[j] = sum_cc M''[3][cc] a_j[cc], cc = 0,1,2,5 (real a), 3 (i^j), 4 (i^-j)
      int32_t zr[4][kFC], zi[4][kFC];
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < kFC; c++) zr[j][c] = zi[j][c] = 0;
      auto cpx_row = [&](auto kkc) {
        constexpr int kk = decltype(kkc)::value;
        int32_t re[kFC], im[kFC];
        take_cpx(re, im, tb, 20 + kk);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int n = kk == 4 ? j : (4 - j);   // power of i for (3,3) / (3,4)
          const int ax = kk < 4 ? areal(j, kk == 3 ? 5 : kk) : 0;
          const int rx = kk < 4 ? ax : re_x(n), ry = kk < 4 ? 0 : re_y(n);
          const int ix = kk < 4 ? 0 : im_x(n), iy = kk < 4 ? ax : im_y(n);
#pragma unroll
          for (int c = 0; c < kFC; c++) {
            zr[j][c] += rx * re[c] + ry * im[c];
            zi[j][c] += ix * re[c] + iy * im[c];
          }
        }
      };
      cpx_row(std::integral_constant<int, 0>{});
      cpx_row(std::integral_constant<int, 1>{});
      cpx_row(std::integral_constant<int, 2>{});
      cpx_row(std::integral_constant<int, 3>{});
      cpx_row(std::integral_constant<int, 4>{});
      cpx_row(std::integral_constant<int, 5>{});
      tmem_st_wait();

      if (dbg & 1) continue;   // debug: no output (pipeline timing)
      // ---- out32 = rha(Y / 16) (A11), optional requantisation (A14), crop, store
      const int tb_i = u / nblocks, nb = u - tb_i * nblocks;
      const int t = tb_i * kMBlock + row;              // chunk tile
      const bool tvalid = t < imgs * g.tpi;
      int img = 0, oy0 = 0, ox0 = 0, ni = 0, nj = 0;
      if (tvalid) {
        const int rem = t % g.tpi, ty = rem / g.tw;
        img = n0 + t / g.tpi;
        oy0 = 4 * ty;
        ox0 = 4 * (rem - ty * g.tw);
        ni = min(4, g.ho - oy0);
        nj = min(4, g.wo - ox0);
      }
      const int co0 = nb * kFN + cw * kFC;
      auto outv = [&](int32_t yv) -> int32_t {
        const int32_t t31 = yv >> 31;
        if (!OUT8) return (yv + 8 + t31) >> 4;                         // rha(Y / 16), |Y| < 2^31 - 8
        if (RQFAST) {                                                   // rha(rha(Y/16) / 2^S), S <= 20
          const int32_t kpos = rq_shift > 0 ? 8 + (1 << (rq_shift + 3)) : 8;
          const int32_t kneg = rq_shift > 0 ? 17 : 1;
          const int32_t r = (yv + kpos + t31 * kneg) >> (rq_shift + 4);
          return max(-128, min(127, r));
        }
        const int32_t o32 = (yv + 8 + t31) >> 4;
        const long long pr = (long long)o32 * rq_mult;
        long long r = pr;
        if (rq_shift > 0) {
          const long long a = pr < 0 ? -pr : pr;
          const long long q = (a + (1ll << (rq_shift - 1))) >> rq_shift;
          r = pr < 0 ? -q : q;
        }
        return (int32_t)(r > 127 ? 127 : (r < -128 ? -128 : r));
      };
      const bool stage8 = NHWC && OUT8 && (g.cout & 15) == 0;
      // store output row i (Yi[j][c] = Y[i][j] of couts co0 + c)
      auto emit_row = [&](int i, const int32_t (&Yi)[4][kFC]) {
        if (stage8) {   // stage [px][tile][16 couts] bytes; 16-byte chunks leave after the barrier
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t w = ((uint32_t)outv(Yi[j][0]) & 0xffu) | (((uint32_t)outv(Yi[j][1]) & 0xffu) << 8) |
                               (((uint32_t)outv(Yi[j][2]) & 0xffu) << 16) | ((uint32_t)outv(Yi[j][3]) << 24);
            *reinterpret_cast<uint32_t*>(staging + ((i * 4 + j) * kMBlock + row) * 16 + cw * kFC) = w;
          }
          return;
        }
        if (!tvalid || i >= ni) return;
        if (NHWC) {
#pragma unroll
          for (int j = 0; j < 4; j++) {
            if (j >= nj) continue;
            const long long pix = ((long long)img * g.ho + oy0 + i) * g.wo + ox0 + j;
            if (OUT8) {
              int8_t* dst = static_cast<int8_t*>(y) + pix * g.cout;
#pragma unroll
              for (int c = 0; c < kFC; c++)
                if (co0 + c < g.cout) dst[co0 + c] = (int8_t)outv(Yi[j][c]);
            } else {
              int32_t* dst = static_cast<int32_t*>(y) + pix * g.cout;
              if ((g.cout & 3) == 0 && co0 < g.cout) {
                *reinterpret_cast<int4*>(dst + co0) =
                    make_int4(outv(Yi[j][0]), outv(Yi[j][1]), outv(Yi[j][2]), outv(Yi[j][3]));
              } else {
#pragma unroll
                for (int c = 0; c < kFC; c++)
                  if (co0 + c < g.cout) dst[co0 + c] = outv(Yi[j][c]);
              }
            }
          }
        } else {   // NCHW: per cout, 4 consecutive pixels of output row oy0 + i
          const bool vec = (g.wo & 3) == 0 && nj == 4;
#pragma unroll
          for (int c = 0; c < kFC; c++) {
            const int co = co0 + c;
            if (co >= g.cout) continue;
            const long long off = (((long long)img * g.cout + co) * g.ho + oy0 + i) * g.wo + ox0;
            if (OUT8) {
              int8_t* dst = static_cast<int8_t*>(y) + off;
              if (vec) {
                *reinterpret_cast<uint32_t*>(dst) =
                    ((uint32_t)outv(Yi[0][c]) & 0xffu) | (((uint32_t)outv(Yi[1][c]) & 0xffu) << 8) |
                    (((uint32_t)outv(Yi[2][c]) & 0xffu) << 16) | ((uint32_t)outv(Yi[3][c]) << 24);
              } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                  if (j < nj) dst[j] = (int8_t)outv(Yi[j][c]);
              }
            } else {
              int32_t* dst = static_cast<int32_t*>(y) + off;
              if (vec) {
                *reinterpret_cast<int4*>(dst) = make_int4(outv(Yi[0][c]), outv(Yi[1][c]), outv(Yi[2][c]), outv(Yi[3][c]));
              } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                  if (j < nj) dst[j] = outv(Yi[j][c]);
              }
            }
          }
        }
      };
      {
        int32_t A[4][kFC], B[4][kFC];
        tmem_ld16(part + 0 * 64, A);   // Z_0
        tmem_ld16(part + 1 * 64, B);   // P
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int c = 0; c < kFC; c++) {
            const int32_t r2 = 2 * zr[j][c];
            A[j][c] += B[j][c] + r2;   // Y[0] = Z_0 + P + 2 Re Z_3
            B[j][c] -= r2;             // Y[2] = P - 2 Re Z_3
          }
        emit_row(0, A);
        emit_row(2, B);
        tmem_ld16(part + 2 * 64, A);   // Q
        tmem_ld16(part + 3 * 64, B);   // Z_5
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int c = 0; c < kFC; c++) {
            const int32_t i2 = 2 * zi[j][c];
            B[j][c] += A[j][c] + i2;   // Y[3] = Q + Z_5 + 2 Im Z_3
            A[j][c] -= i2;             // Y[1] = Q - 2 Im Z_3
          }
        emit_row(1, A);
        emit_row(3, B);
      }
      if (stage8) {
        fepi_barrier();
#pragma unroll
        for (int q = 0; q < (16 * kMBlock) / (kFEpiWarps * 32); q++) {
          const int ch = etid + q * kFEpiWarps * 32;
          const int px = ch >> 7, rr = ch & (kMBlock - 1);
          const int tt = tb_i * kMBlock + rr;
          if (tt >= imgs * g.tpi) continue;
          const int rem = tt % g.tpi, ty = rem / g.tw;
          const int oy = 4 * ty + (px >> 2), ox = 4 * (rem - ty * g.tw) + (px & 3);
          if (oy >= g.ho || ox >= g.wo) continue;
          const uint4 val = *reinterpret_cast<const uint4*>(staging + ch * 16);
          int8_t* dst = static_cast<int8_t*>(y) +
                        (((long long)(n0 + tt / g.tpi) * g.ho + oy) * g.wo + ox) * g.cout + nb * kFN;
          *reinterpret_cast<uint4*>(dst) = val;
        }
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

static int g_fused_sms = 0;
static int g_fused_dbg = 0;   // WINO_FUSED_DBG (debug timing only): 1 no output, 2 no MMAs, 4 no TMEM-load wait

cudaError_t launch_fused(const Geom& g, long long tiles_pad_launch, int n0, int imgs, const int8_t* vimg,
                         const int8_t* wimg, const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y,
                         cudaStream_t st) {
  if (g.nblk != kFN) return cudaErrorInvalidValue;
  const int tblocks = (int)(tiles_pad_launch / kMBlock);
  const int n_units = tblocks * (g.cout_pad / kFN);
  const int grid = n_units < g_fused_sms ? n_units : g_fused_sms;
  const size_t smem = fused_smem_bytes();
  const bool nhwc = g.layout == 1, out8 = g.out_mode == 0, fast = rq_mult == 1 && rq_shift <= 20;
  cudaError_t e;
#define WINO_KF(A, B, C) \
  e = launch_pdl(k_fused<A, B, C>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs, tblocks, rq_mult, rq_shift, y, g_fused_dbg)
  if (nhwc) {
    if (!out8) WINO_KF(true, false, false);
    else if (fast) WINO_KF(true, true, true);
    else WINO_KF(true, true, false);
  } else {
    if (!out8) WINO_KF(false, false, false);
    else if (fast) WINO_KF(false, true, true);
    else WINO_KF(false, true, false);
  }
#undef WINO_KF
  return e;
}

cudaError_t setup_fused() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_fused_sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char* d = std::getenv("WINO_FUSED_DBG")) g_fused_dbg = std::atoi(d);
  const int smem = (int)fused_smem_bytes();
#define WINO_KF_ATTR(A, B, C) \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
  WINO_KF_ATTR(true, false, false);
  WINO_KF_ATTR(true, true, true);
  WINO_KF_ATTR(true, true, false);
  WINO_KF_ATTR(false, false, false);
  WINO_KF_ATTR(false, true, true);
  WINO_KF_ATTR(false, true, false);
#undef WINO_KF_ATTR
  return e;
}

}  // namespace wino
