// k_fused.cu -- K3F: the Winograd-domain channel contraction on the
// tcgen05 tensor cores FUSED with the reverse scaling M'' = rha(M m / 2^q)
// (P:312), the real-only output transform Y = A^T M'' A (P:163-170,
// P:237), out32 = rha(Y / 16) (A2, A11), crop, requantisation (A14) and the
// store.  M'' never leaves the SM: the staged path (k_gemm.cu + k_output.cu)
// writes and re-reads 144 bytes per (tile, cout) through HBM; this kernel writes
// the output only.
//
// Operands (layout.cuh, "fused-path operand layouts"): per GROUP (a real
// position, or a complex primary with its conjugate mirror implied),
// pieces v = 256 hi + lo (V: hi = v >> 8 s8, lo = v & 255 u8, read as an unsigned
// A operand; W': balanced s8 hi and lo), group-contiguous so a stage is ONE bulk
// copy of V (<= 32 KB) and one of W'.  At c_in <= 8 two slot-groups share a K step
// (quarter-K packing, layout.cuh, MG = 5).  The complex product uses the
// 4-multiplication form as K/N-concatenated real GEMMs (identical integers to
// the Karatsuba form of P:83-86, which the staged path implements):
//   Re = Vr Wr - Vi Wi,  Im = Vr Wi + Vi Wr.
// Pieces are concatenated along N so that each UMMA is as wide as possible
// (kind::i8 costs ~45 cycles per M=128, K=32 UMMA for any N <= 64):
//   real group, per K step:     A = V hi . [W hi | W lo]  -> D[s16 | s8]
//                               A = V lo . [W hi | W lo]  -> D[s8 | s0]   (D offset 16)
//   complex group, per K step:  A = Vr hi . B0, A = Vr lo . B0 (offset 32),
//                               A = Vi hi . B1, A = Vi lo . B1 (offset 32)
//   B0 = [Wr hi | Wi hi | Wr lo | Wi lo], B1 = [-Wi hi | Wr hi | -Wi lo | Wr lo]
//   -> D[Re16 | Im16 | Re8 | Im8 | Re0 | Im0]; M = 2^16 s16 + 2^8 s8 + s0 (mod 2^32
//   exact; the true values fit, A23).  MG = 0: on the first K step the overlapping
//   column blocks are initialised by splitting one UMMA (accumulate flag is per
//   UMMA, not per column); MG > 0: every slot starts at zero (the epilogue re-zeroes
//   what it read) and every UMMA accumulates.
//
// Work unit = (128-tile block, 16-cout block): all 26 groups, row by row of the
// 6x6 Winograd grid in the order rows 0, 5, 1, 2 (real (r,0) (r,1) (r,2) (r,5),
// then primary (r,3)), then row 3 (primaries (3,0) (3,1) (3,2) (3,5) (3,3) (3,4)).
// Output transform (A^T rows a_0 = (1,1,1,1,1,0), a_1 = (0,1,-1,i,-i,0),
// a_2 = (0,1,1,-1,-1,0), a_3 = (0,1,-1,-i,i,1); a_j[4] = conj a_j[3]):
//   Z_r[j] = sum_c M''[r][c] a_j[c]  (real for r in {0,1,2,5}: the pair at
//            columns 3/4 gives 2 Re(i^j z); complex for r = 3)
//   Y[0] = Z_0 + P + 2 Re Z_3   Y[1] = Q - 2 Im Z_3   Y[2] = P - 2 Re Z_3
//   Y[3] = Q + Z_5 + 2 Im Z_3,  P = Z_1 + Z_2, Q = Z_1 - Z_2   (row 4 never formed)
// Z_0, Z_5 are parked in shared memory, P, Q in TMEM, Re/Im Z_3 in registers.
//
// Persistent CTAs (the fewest that keep the number of unit rounds), warp-specialised (19 warps,
// <= 96 registers):
//   warps 0..15  epilogue: TMEM lane quadrant w % 4 (32 tiles), couts 4 (w / 4) .. +3
//   warps 16, 17 producers (one elected lane each, alternate stages): bulk copies into the ring
//   warp 18      MMA issuer (one elected lane): tcgen05.mma into 4 TMEM accumulator slots of 96
//                columns (one complex group or two real groups each)
// Ring (160 KB): MG = 0 four 40 KB stages (a group's K chunk each), MG = 1 four 40 KB stages and
// MG = 2 two 80 KB stages (one slot-group each), MG = 3 two 80 KB stages (4 K steps of a slot-group),
// MG = 4 (one K step) four 40 KB stages of two slot-groups each, MG = 5 (quarter-K packing) four stages
// of one 13 KB pack each (two slot-groups, one N = 160 UMMA pair).
// TMEM: [0, 384) accumulator slots, [384, 448) P, [448, 512) Q.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kFN = kFN16;                    // couts per unit
constexpr int kFEpiWarps = 16;                // 4 per TMEM lane quadrant
constexpr int kFC = 4;                        // couts per epilogue thread
constexpr int kFProducers = 2;                // producer warps, alternating stages (the per-thread
                                              // issue cost of a stage's bulk copies is ~0.27 us)
constexpr int kFProducerWarp = kFEpiWarps, kFMmaWarp = kFEpiWarps + kFProducers;
constexpr int kFThreads = 32 * (kFEpiWarps + kFProducers + 1);
constexpr int kFStages = 4;
constexpr uint32_t kFStageV = 32768;          // V part of a stage (<= 32 KB)
constexpr uint32_t kFStageBytes = kFStageV + 8192;
constexpr int kFSlots = 4;                    // TMEM accumulator slots
constexpr int kFSlotCols = 96;
constexpr uint32_t kFPCol = 384, kFQCol = 448;
constexpr int kFSlotGroups = 18;              // per unit: 4 rows x (2 real pairs + 1 complex) + 6 complex
constexpr uint32_t kFPartBytes = 65536;       // Z_0, Z_5 partials; aliased by the int8 output staging tile
constexpr uint32_t kFETabBytes = kFGroupsN * kFN * 4;
constexpr int kFEpiBar = 1;
constexpr uint32_t kQkStage = kQkPackV + kQkPackW;   // MG = 5 ring stage (13 KB, packed back to back)

inline size_t fused_smem_bytes() {
  return (size_t)kFStages * kFStageBytes + kFPartBytes + kFETabBytes + 512;
}

// K steps per stage of group gi (V of a stage <= 32 KB)
__host__ __device__ constexpr int fg_kchunk(int gi) { return fg_complex(gi) ? 2 : 4; }
// slot-group sg -> first group and group count
__device__ __forceinline__ int sg_first(int sg) { return sg < 12 ? (sg / 3) * 5 + (sg % 3) * 2 : 20 + sg - 12; }
__device__ __forceinline__ int sg_count(int sg) { return (sg < 12 && sg % 3 < 2) ? 2 : 1; }
// MG = 4 (one K step): V and W' bytes of slot-group sg (a real pair: 2 x 2 pieces, 2 W' units; a complex
// group: 4 pieces, 4 W' units)
__device__ __forceinline__ uint32_t sg_vbytes1(int sg) { return 4u * kVBlockBytes; }
__device__ __forceinline__ uint32_t sg_wbytes1(int sg) { return sg_count(sg) == 2 ? 2048u : 4096u; }
// position index (r*6 + c) of group gi
__device__ __forceinline__ int fg_pos(int gi) {
  return fg_complex(gi) ? cpx_pos(fg_primary(gi)) : real_pos(fg_real_plane(gi));
}

// barrier waits of the MMA issuer and of the epilogue's accumulator handshake: suspending try_wait, or a
// non-suspending test_wait poll (no wake-up latency after the phase flips) under WINO_SPIN_MMA / WINO_SPIN_EPI
__device__ __forceinline__ void mma_wait(uint32_t bar, uint32_t parity) {
#ifdef WINO_SPIN_MMA
  mbar_spin(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void epi_wait(uint32_t bar, uint32_t parity) {
#ifdef WINO_SPIN_EPI
  mbar_spin(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
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
// zero 4 columns of this warp's lane quadrant (accumulators of the MG variants start from zero, so every
// UMMA accumulates and the first K step needs no split)
__device__ __forceinline__ void tmem_zero4(uint32_t taddr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(taddr), "r"(0) : "memory");
}

// M'' = rha(v m / 2^q) (A9) evaluated as rha(v m' / 2^7) with
// m' = m 2^(7-q) (q in [4,7], so m' <= 2040): one constant per (position, cout)
// and a fixed shift.  rha(p / 2^7) = (p + 64 - [p < 0]) >> 7 (floor shift).  The
// unscaled code is m' = 128, which returns v.
__device__ __forceinline__ int32_t frscale(int32_t v, uint32_t mq) { return rha_mul_shr7(v, mq); }

// a_k[c] for the real indices c in {0,1,2,5}
__host__ __device__ constexpr int areal(int k, int c) {
  return c == 0 ? (k == 0) : (c == 1 ? 1 : (c == 2 ? ((k & 1) ? -1 : 1) : (k == 3)));
}
// i^n (x + iy) = (re_x x + re_y y) + i (im_x x + im_y y)
__host__ __device__ constexpr int re_x(int n) { return (n & 3) == 0 ? 1 : ((n & 3) == 2 ? -1 : 0); }
__host__ __device__ constexpr int re_y(int n) { return (n & 3) == 1 ? -1 : ((n & 3) == 3 ? 1 : 0); }
__host__ __device__ constexpr int im_x(int n) { return (n & 3) == 1 ? 1 : ((n & 3) == 3 ? -1 : 0); }
__host__ __device__ constexpr int im_y(int n) { return re_x(n); }

// MG > 0: ONE ring stage per slot-group (a real pair's or a complex group's whole K range; the pair's
// V and W' are contiguous), 18 stages per unit instead of 26 (c_in <= 64) or 36 (c_in <= 128) -- each
// stage costs ~350 cycles of copy issue plus a commit.  MG = 1 (c_in <= 64): 4 stages of
// 40 KB; MG = 2 (c_in <= 128): 2 stages of 80 KB (the same 160 KB); MG = 3 (c_in > 128): 2 stages of 80 KB,
// each 4 K steps of a slot-group (faster than the general loops at every c_in measured, 256..768).  The MG
// loops are separate code; the general loops (MG = 0) remain for WINO_FUSED_MERGE=0 (experiments).
template <bool NHWC, bool OUT8, bool RQFAST, int MG>
__global__ void __launch_bounds__(kFThreads, 1)
    k_fused(const int8_t* __restrict__ V, const int8_t* __restrict__ W, const uint8_t* __restrict__ codes, Geom g,
            int n0, int imgs, int tblocks, int32_t rq_mult, int rq_shift, void* __restrict__ y, int dbg,
            uint64_t* __restrict__ trace) {
#ifdef WINO_FUSED_TRACE
  // per CTA: [stage it < 64][4]: 0 producer issued, 1 MMA saw data, 2 MMA committed; [64 + slot-group < 32][4]:
  // 0 MMA got slot, 1 epilogue warp 0 saw accumulators, 2 epilogue warp 0 released
  uint64_t* tr = trace ? trace + (size_t)blockIdx.x * 96 * 4 : nullptr;
#define FTRACE(i, ev) do { if (tr && (i) < 96) { tr[(i) * 4 + (ev)] = clock64(); } } while (0)   // SM cycles
#else
  (void)trace;
#define FTRACE(i, ev) do { } while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem[];
#ifndef WINO_FUSED_DBG
  dbg = 0;   // the WINO_FUSED_DBG ablation modes exist only in debug builds (-DWINO_FUSED_DBG)
#endif
  // warp index broadcast from lane 0: warp-uniform to the compiler, so the TMEM addresses derived from it
  // live in uniform registers (no per-access R2UR moves before LDTM / STTM)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* part = smem + kFStages * kFStageBytes;                            // Z_0 / Z_5 | output staging
  uint32_t* etab = reinterpret_cast<uint32_t*>(part + kFPartBytes);          // [26 groups][16 couts] m'
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(etab) + kFETabBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kFStages + 2 * kFSlots);
  uint32_t* lut = tmem_slot + 4;                                             // 64: code -> m'
  const uint32_t sbase = smem_u32(smem);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kFStages);
  const uint32_t tfull0 = smem_u32(bars + 2 * kFStages), tempty0 = smem_u32(bars + 2 * kFStages + kFSlots);
  const int nblocks = g.cout_pad / kFN;
  const int n_units = tblocks * nblocks;
  const int ksteps = g.ksteps;
  // quarter-K pairing (MG = 5, int8 NHWC staged output, an even number of cout blocks): the two cout blocks
  // that share a 32-byte sector of each output pixel run back to back on one CTA, their outputs are staged
  // side by side and leave as whole sectors (a lane pair per sector) instead of two half-sector stores
  const bool qpair = MG == 5 && NHWC && OUT8 && (g.cout & 15) == 0 && !g.pool2 && (nblocks & 1) == 0;
  const int u_first = qpair ? 2 * (int)blockIdx.x : (int)blockIdx.x;
  auto u_next = [&](int u) -> int { return qpair ? ((u & 1) ? u + 2 * (int)gridDim.x - 1 : u + 1) : u + (int)gridDim.x; };

  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  if (threadIdx.x == 32 * kFProducerWarp) {
    for (int s = 0; s < kFStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < kFSlots; b++) {
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
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if constexpr (MG > 0) {   // every accumulator slot starts at zero (the epilogue re-zeroes each after reading)
    if (warp < kFEpiWarps) {
      const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * kFC;
      for (int b = 0; b < kFSlots; b++)
#pragma unroll
        for (int blk = 0; blk < 6; blk++) tmem_zero4(lb + b * kFSlotCols + blk * 16);
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  pdl_wait();   // V (and W', codes) come from the kernels just before

  if (warp >= kFProducerWarp && warp < kFProducerWarp + kFProducers) {
    {   // warp-uniform loop, one elected lane issues (operands stay in uniform registers)
      // ------------------------------------------------ producers: warp p issues the stages it with it % P == p
      const int pw = warp - kFProducerWarp;
      int it = 0;
      if constexpr (MG == 5) {
        // quarter-K packing (c_in <= 8, layout.cuh): one stage per pack (8 KB of V + 5 KB of W': two slot-groups),
        // released by its own commit
        for (int u = u_first; u < n_units; u = u_next(u)) {
          const int tb = u / nblocks, nb = u - tb * nblocks;
          for (int pk = 0; pk < kQkPacks; pk++, it++) {
            if (it % kFProducers != pw) continue;
            const int s = it % kFStages;
            mbar_wait(empty0 + 8 * s, ((it / kFStages) & 1) ^ 1);
            const uint32_t st = sbase + s * kQkStage;
            if (elect_one()) {
              if (dbg & 4) {   // debug builds only: no copies
                mbar_arrive(full0 + 8 * s);
              } else {
                mbar_arrive_expect_tx(full0 + 8 * s, kQkPackV + kQkPackW);
                bulk_g2s(st, V + ((long long)tb * kQkPacks + pk) * kQkPackV, kQkPackV, full0 + 8 * s);
                bulk_g2s(st + kQkPackV, W + ((long long)nb * kQkPacks + pk) * kQkPackW, kQkPackW, full0 + 8 * s);
              }
              if (it < 64) FTRACE(it, 0);
            }
            __syncwarp();
          }
        }
      } else if constexpr (MG == 4) {
        // one K step (c_in <= 32): a 40 KB stage holds TWO consecutive slot-groups (their groups are
        // contiguous in V and W'), one V and one W' copy per stage, 9 stages per unit instead of 18; the
        // stage is released by its own commit (empty barrier) after the second slot-group's UMMAs
        constexpr uint32_t kSV = 32768;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          const int tb = u / nblocks, nb = u - tb * nblocks;
          for (int pr = 0; pr < kFSlotGroups / 2; pr++, it++) {
            if (it % kFProducers != pw) continue;
            const int s = it % kFStages;
            mbar_wait(empty0 + 8 * s, ((it / kFStages) & 1) ^ 1);
            const int g0 = sg_first(2 * pr);
            const uint32_t vb = sg_vbytes1(2 * pr) + sg_vbytes1(2 * pr + 1);
            const uint32_t wb = sg_wbytes1(2 * pr) + sg_wbytes1(2 * pr + 1);
            const int8_t* vg = V + ((long long)tb * kVPiecesF + fg_vprefix(g0)) * kVBlockBytes;
            const int8_t* wg = W + ((long long)nb * kWRowUnitsF + fg_wprefix(g0)) * 1024;
            const uint32_t st = sbase + s * kFStageBytes;
            if (elect_one()) {
              if (dbg & 4) {   // debug builds only: no copies
                mbar_arrive(full0 + 8 * s);
              } else {
                mbar_arrive_expect_tx(full0 + 8 * s, vb + wb);
                bulk_g2s(st, vg, vb, full0 + 8 * s);
                bulk_g2s(st + kSV, wg, wb, full0 + 8 * s);
              }
              if (it < 64) FTRACE(it, 0);
            }
            __syncwarp();
          }
        }
      } else if constexpr (MG == 3) {
        // two 80 KB stages, each 4 K steps of one slot-group (a pair: both groups' chunks, 2 + 2 copies),
        // released by stage commits as in the general loops
        constexpr uint32_t kSB = kFStages * kFStageBytes / 2, kSV = 65536;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          const int tb = u / nblocks, nb = u - tb * nblocks;
          for (int sg = 0; sg < kFSlotGroups; sg++) {
            const int g0 = sg_first(sg), ng = sg_count(sg);
            for (int k0 = 0; k0 < ksteps; k0 += 4, it++) {
              if (it % kFProducers != pw) continue;
              const int s = it & 1;
              mbar_wait(empty0 + 8 * s, ((it >> 1) & 1) ^ 1);
              const int kn = min(4, ksteps - k0);
              const uint32_t st = sbase + s * kSB;
              if (elect_one()) {
                if (ng == 2) {   // group q: V at q * 32 KB, W' at kSV + q * 4 KB
                  const uint32_t vbq = (uint32_t)(kn * 2) * kVBlockBytes, wbq = (uint32_t)kn * 1024;
                  mbar_arrive_expect_tx(full0 + 8 * s, 2 * (vbq + wbq));
                  for (int q = 0; q < 2; q++) {
                    const int gi = g0 + q;
                    const int8_t* vg = V + ((long long)tb * kVPiecesF + fg_vprefix(gi)) * ksteps * kVBlockBytes +
                                       (long long)k0 * 2 * kVBlockBytes;
                    const int8_t* wg = W + ((long long)nb * kWRowUnitsF + fg_wprefix(gi)) * ksteps * 1024 +
                                       (long long)k0 * 1024;
                    bulk_g2s(st + q * 32768u, vg, vbq, full0 + 8 * s);
                    bulk_g2s(st + kSV + q * 4096u, wg, wbq, full0 + 8 * s);
                  }
                } else {
                  const uint32_t vb = (uint32_t)(kn * 4) * kVBlockBytes, wb = (uint32_t)(kn * 4) * 1024;
                  const int8_t* vg = V + ((long long)tb * kVPiecesF + fg_vprefix(g0)) * ksteps * kVBlockBytes +
                                     (long long)k0 * 4 * kVBlockBytes;
                  const int8_t* wg = W + ((long long)nb * kWRowUnitsF + fg_wprefix(g0)) * ksteps * 1024 +
                                     (long long)k0 * 4 * 1024;
                  mbar_arrive_expect_tx(full0 + 8 * s, vb + wb);
                  bulk_g2s(st, vg, vb, full0 + 8 * s);
                  bulk_g2s(st + kSV, wg, wb, full0 + 8 * s);
                }
              }
              __syncwarp();
            }
          }
        }
      } else if constexpr (MG > 0) {
        constexpr int kMgStages = MG == 2 ? 2 : 4;
        constexpr uint32_t kMgStageBytes = kFStages * kFStageBytes / kMgStages, kMgStageV = MG == 2 ? 65536 : kFStageV;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          const int tb = u / nblocks, nb = u - tb * nblocks;
          for (int sg = 0; sg < kFSlotGroups; sg++) {
            const int g0 = sg_first(sg), ng = sg_count(sg);
            for (int q = 0; q < (ng == 2 ? 1 : ng); q++, it++) {   // one stage per slot-group
              if (it % kFProducers != pw) continue;
              const int gi = g0 + q;
              const int8_t* vg = V + ((long long)tb * kVPiecesF + fg_vprefix(gi)) * ksteps * kVBlockBytes;
              const int8_t* wg = W + ((long long)nb * kWRowUnitsF + fg_wprefix(gi)) * ksteps * 1024;
              const int s = it % kMgStages;
              // stage s last held slot-group it - kMgStages: its accumulator commit (tfull) also covers the
              // MMAs that read the stage, so no separate stage commit is needed (tfull cannot have moved on:
              // its next commit is slot-group it - kMgStages + 4 >= it's, whose operands are loaded here)
              static_assert(kMgStages <= kFSlots, "stage reuse must precede the slot's next commit");
              if (it >= kMgStages)
                mbar_wait(tfull0 + 8 * ((it - kMgStages) % kFSlots), ((it - kMgStages) / kFSlots) & 1);
              // pair: pieces 2 + 2, W' units 1 + 1; complex group: 4 pieces, 4 W' units (all K steps)
              const int pcs = ng == 2 ? 4 : fg_pieces(gi), wu = ng == 2 ? 2 : fg_wunits(gi);
              const uint32_t vb = (uint32_t)(ksteps * pcs) * kVBlockBytes, wb = (uint32_t)(ksteps * wu) * 1024;
              const uint32_t st = sbase + s * kMgStageBytes;
              if (elect_one()) {
                if (dbg & 4) {   // debug builds only: no copies (the stage is marked full at once)
                  mbar_arrive(full0 + 8 * s);
                } else {
                  mbar_arrive_expect_tx(full0 + 8 * s, vb + wb);
                  bulk_g2s(st, vg, vb, full0 + 8 * s);
                  bulk_g2s(st + kMgStageV, wg, wb, full0 + 8 * s);
                }
                if (it < 64) FTRACE(it, 0);
              }
              __syncwarp();
            }
          }
        }
      } else
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int tb = u / nblocks, nb = u - tb * nblocks;
        for (int gi = 0; gi < kFGroupsN; gi++) {
          const int pcs = fg_pieces(gi), wu = fg_wunits(gi), kc = fg_kchunk(gi);
          const int8_t* vg = V + ((long long)tb * kVPiecesF + fg_vprefix(gi)) * ksteps * kVBlockBytes;
          const int8_t* wg = W + ((long long)nb * kWRowUnitsF + fg_wprefix(gi)) * ksteps * 1024;
          for (int k0 = 0; k0 < ksteps; k0 += kc, it++) {
            if (it % kFProducers != pw) continue;
            const int s = it % kFStages;
            mbar_wait(empty0 + 8 * s, ((it / kFStages) & 1) ^ 1);
            const int kn = min(kc, ksteps - k0);
            const uint32_t vb = (uint32_t)(kn * pcs) * kVBlockBytes, wb = (uint32_t)(kn * wu) * 1024;
            const uint32_t st = sbase + s * kFStageBytes;
            if (elect_one()) {
              mbar_arrive_expect_tx(full0 + 8 * s, vb + wb);
              bulk_g2s(st, vg + (long long)k0 * pcs * kVBlockBytes, vb, full0 + 8 * s);
              bulk_g2s(st + kFStageV, wg + (long long)k0 * wu * 1024, wb, full0 + 8 * s);
              if (it < 64) FTRACE(it, 0);
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == kFMmaWarp) {
    {   // warp-uniform loop, one elected lane issues
      // ------------------------------------------------ MMA issuer
      const uint32_t id16 = idesc_i8(kMBlock, 16, 1, 1), id32 = idesc_i8(kMBlock, 32, 1, 1),
                     id64 = idesc_i8(kMBlock, 64, 1, 1);
      // lo pieces of V are u8 (v = 256 hi + lo, lo = v & 255; K2F, layout.cuh): unsigned A operand
      const uint32_t id16u = idesc_i8(kMBlock, 16, 0, 1), id32u = idesc_i8(kMBlock, 32, 0, 1),
                     id64u = idesc_i8(kMBlock, 64, 0, 1);
      int it = 0, sgc = 0;
      if constexpr (MG == 5) {
        // one N = 160 UMMA pair per pack fills two adjacent TMEM slots (layout.cuh quarter-K packing)
        const uint32_t id160 = idesc_i8(kMBlock, kQkRows, 1, 1), id160u = idesc_i8(kMBlock, kQkRows, 0, 1);
        const uint64_t D0 = umma_desc(sbase, 128, 256);
        const uint32_t d0lo = (uint32_t)D0, d0hi = (uint32_t)(D0 >> 32);
        auto dsc = [&](uint32_t off) -> uint64_t { return ((uint64_t)d0hi << 32) | (uint64_t)(d0lo + (off >> 4)); };
        for (int u = u_first; u < n_units; u = u_next(u)) {
          for (int pk = 0; pk < kQkPacks; pk++, it++, sgc += 2) {
            const int s = it % kFStages;
            const int b = sgc % kFSlots;            // even: slots b, b + 1 are adjacent
            mma_wait(tempty0 + 8 * b, ((sgc / kFSlots) & 1) ^ 1);
            mma_wait(tempty0 + 8 * (b + 1), (((sgc + 1) / kFSlots) & 1) ^ 1);
            mma_wait(full0 + 8 * s, (it / kFStages) & 1);
            tc_fence_after();
            if (it < 64 && lane == 0) FTRACE(it, 1);
            if (sgc < 32 && lane == 0) FTRACE(64 + sgc, 0);
            const uint32_t st = s * kQkStage;
            const uint32_t d0 = tmem + b * kFSlotCols;
            if (elect_one()) {
              if (!(dbg & 2)) {
                const uint64_t bw = dsc(st + kQkPackV);
                // hi, accumulate off: writes columns [0, 160) of the slot pair (slot b whole, its s0 block from the
                // zero rows; slot b+1 s16 / s8), so only slot b+1's s0 block [160, 192) must start at zero
                umma_i8(d0, dsc(st), bw, id160, 0u);                       // hi: [slot b: ... | 0 | slot b+1]
                umma_i8(d0 + 32, dsc(st + kVBlockBytes), bw, id160u, 1u);  // lo (u8) at the piece offset 32
              }
              umma_commit(tfull0 + 8 * b);
              umma_commit(tfull0 + 8 * (b + 1));
              umma_commit(empty0 + 8 * s);
              if (it < 64) FTRACE(it, 2);
            }
            __syncwarp();
          }
        }
      } else
      if constexpr (MG == 4) {
        constexpr uint32_t kSV = 32768;
        const uint64_t D0 = umma_desc(sbase, 128, 256);   // + (offset >> 4): see the MG 1..3 loop below
        const uint32_t d0lo = (uint32_t)D0, d0hi = (uint32_t)(D0 >> 32);
        auto dsc = [&](uint32_t off) -> uint64_t { return ((uint64_t)d0hi << 32) | (uint64_t)(d0lo + (off >> 4)); };
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          for (int pr = 0; pr < kFSlotGroups / 2; pr++, it++) {
            const int s = it % kFStages;
            mma_wait(full0 + 8 * s, (it / kFStages) & 1);
            tc_fence_after();
            if (it < 64 && lane == 0) FTRACE(it, 1);
            uint32_t voff = s * kFStageBytes, woff = s * kFStageBytes + kSV;
#pragma unroll
            for (int h = 0; h < 2; h++, sgc++) {
              const int sg = 2 * pr + h;
              const int b = sgc % kFSlots;
              mma_wait(tempty0 + 8 * b, ((sgc / kFSlots) & 1) ^ 1);
              tc_fence_after();
              if (sgc < 32 && lane == 0) FTRACE(64 + sgc, 0);
              const uint32_t d0 = tmem + b * kFSlotCols;
              if (elect_one()) {
                if (dbg & 2) {   // debug builds only: no UMMAs
                } else if (sg_count(sg) == 2) {   // real pair: group q's pieces at q * 8 KB, W' at q * 1 KB
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const uint64_t bb = dsc(woff + q * 1024);
                    umma_i8(d0 + q * 48, dsc(voff + (2 * q) * kVBlockBytes), bb, id32, 1u);
                    umma_i8(d0 + q * 48 + 16, dsc(voff + (2 * q + 1) * kVBlockBytes), bb, id32u, 1u);
                  }
                } else {
                  const uint64_t b0 = dsc(woff), b1 = dsc(woff + 2048);
                  umma_i8(d0, dsc(voff), b0, id64, 1u);
                  umma_i8(d0 + 32, dsc(voff + kVBlockBytes), b0, id64u, 1u);
                  umma_i8(d0, dsc(voff + 2 * kVBlockBytes), b1, id64, 1u);
                  umma_i8(d0 + 32, dsc(voff + 3 * kVBlockBytes), b1, id64u, 1u);
                }
                umma_commit(tfull0 + 8 * b);   // slot complete
              }
              __syncwarp();
              voff += sg_vbytes1(sg);
              woff += sg_wbytes1(sg);
            }
            if (elect_one()) umma_commit(empty0 + 8 * s);   // both slot-groups' UMMAs read: stage free
            __syncwarp();
            if (it < 64 && lane == 0) FTRACE(it, 2);
          }
        }
      } else
      if constexpr (MG == 3) {
        constexpr uint32_t kSB = kFStages * kFStageBytes / 2, kSV = 65536;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          for (int sg = 0; sg < kFSlotGroups; sg++, sgc++) {
            const int b = sgc % kFSlots;
            mma_wait(tempty0 + 8 * b, ((sgc / kFSlots) & 1) ^ 1);
            tc_fence_after();
            const int g0 = sg_first(sg), ng = sg_count(sg);
            const uint32_t d0 = tmem + b * kFSlotCols;
            for (int k0 = 0; k0 < ksteps; k0 += 4, it++) {
              const int s = it & 1;
              mma_wait(full0 + 8 * s, (it >> 1) & 1);
              tc_fence_after();
              const int kn = min(4, ksteps - k0);
              const uint32_t st = sbase + s * kSB;
              if (elect_one()) {
                if (ng == 2) {
                  for (int q = 0; q < 2; ++q) {
                    const uint32_t d = d0 + q * 48;
                    const uint32_t va = st + q * 32768u, wa = st + kSV + q * 4096u;
                    for (int kk = 0; kk < kn; ++kk) {   // slots start at zero: every UMMA accumulates
                      const uint64_t ah = umma_desc(va + (2 * kk) * kVBlockBytes, 128, 256);
                      const uint64_t al = umma_desc(va + (2 * kk + 1) * kVBlockBytes, 128, 256);
                      const uint64_t bb = umma_desc(wa + kk * 1024, 128, 256);
                      umma_i8(d, ah, bb, id32, 1u);
                      umma_i8(d + 16, al, bb, id32u, 1u);
                    }
                  }
                } else {
                  for (int kk = 0; kk < kn; ++kk) {
                    const uint32_t a0 = st + (4 * kk) * kVBlockBytes;
                    const uint64_t rh = umma_desc(a0, 128, 256), rl = umma_desc(a0 + kVBlockBytes, 128, 256);
                    const uint64_t ih = umma_desc(a0 + 2 * kVBlockBytes, 128, 256),
                                   il = umma_desc(a0 + 3 * kVBlockBytes, 128, 256);
                    const uint32_t bw = st + kSV + kk * 4096;
                    const uint64_t b0 = umma_desc(bw, 128, 256), b1 = umma_desc(bw + 2048, 128, 256);
                    umma_i8(d0, rh, b0, id64, 1u);
                    umma_i8(d0 + 32, rl, b0, id64u, 1u);
                    umma_i8(d0, ih, b1, id64, 1u);
                    umma_i8(d0 + 32, il, b1, id64u, 1u);
                  }
                }
                umma_commit(empty0 + 8 * s);   // stage reusable once these MMAs have read it
              }
              __syncwarp();
            }
            if (elect_one()) umma_commit(tfull0 + 8 * b);   // slot complete
            __syncwarp();
          }
        }
      } else if constexpr (MG > 0) {
        constexpr int kMgStages = MG == 2 ? 2 : 4;
        constexpr uint32_t kMgStageBytes = kFStages * kFStageBytes / kMgStages, kMgStageV = MG == 2 ? 65536 : kFStageV;
        // every operand of this loop is K-major, no swizzle, LBO 128 / SBO 256: its descriptor is the ring
        // base's plus (offset >> 4) in the 14-bit address field (no carry: shared memory < 256 KB), so each
        // descriptor costs one uniform add instead of a shift / mask / or chain per UMMA
        const uint64_t D0 = umma_desc(sbase, 128, 256);
        const uint32_t d0lo = (uint32_t)D0, d0hi = (uint32_t)(D0 >> 32);
        auto dsc = [&](uint32_t off) -> uint64_t { return ((uint64_t)d0hi << 32) | (uint64_t)(d0lo + (off >> 4)); };
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
          for (int sg = 0; sg < kFSlotGroups; sg++, sgc++, it++) {   // one stage per slot-group
            const int b = sgc % kFSlots;
            mma_wait(tempty0 + 8 * b, ((sgc / kFSlots) & 1) ^ 1);
            tc_fence_after();
            if (sgc < 32 && lane == 0) FTRACE(64 + sgc, 0);
            const int ng = sg_count(sg);
            const int s = it % kMgStages;
            mma_wait(full0 + 8 * s, (it / kMgStages) & 1);
            tc_fence_after();
            if (it < 64 && lane == 0) FTRACE(it, 1);
            const uint32_t st = s * kMgStageBytes;   // stage offset from the ring base
            const uint32_t d0 = tmem + b * kFSlotCols;
            if (elect_one()) {
              if (dbg & 2) {   // debug builds only: no UMMAs
              } else if (ng == 2) {   // real pair: group q's V at q * 2 ksteps blocks, W' at q * ksteps KB
                for (int q = 0; q < 2; ++q) {
                  const uint32_t d = d0 + q * 48;
                  const uint32_t va = st + (uint32_t)(q * 2 * ksteps) * kVBlockBytes;
                  const uint32_t wa = st + kMgStageV + (uint32_t)(q * ksteps) * 1024;
                  for (int kk = 0; kk < ksteps; ++kk) {   // slots start at zero: every UMMA accumulates
                    const uint64_t bb = dsc(wa + kk * 1024);
                    umma_i8(d, dsc(va + (2 * kk) * kVBlockBytes), bb, id32, 1u);        // [s16 | s8] += hi . [W hi | W lo]
                    if (dbg & 64) break;   // debug builds only: one UMMA per group (timing)
                    umma_i8(d + 16, dsc(va + (2 * kk + 1) * kVBlockBytes), bb, id32u, 1u);   // [s8 | s0] += lo . [W hi | W lo]
                  }
                }
              } else {         // complex group: all K steps in the stage
                for (int kk = 0; kk < ksteps; ++kk) {
                  const uint32_t a0 = st + (4 * kk) * kVBlockBytes;
                  const uint32_t bw = st + kMgStageV + kk * 4096;
                  const uint64_t b0 = dsc(bw), b1 = dsc(bw + 2048);
                  umma_i8(d0, dsc(a0), b0, id64, 1u);                           // [Re16 Im16 Re8 Im8] += Vr hi . B0
                  if (dbg & 64) break;   // debug builds only: one UMMA per group (timing)
                  umma_i8(d0 + 32, dsc(a0 + kVBlockBytes), b0, id64u, 1u);      // [Re8 Im8 Re0 Im0]   += Vr lo . B0
                  umma_i8(d0, dsc(a0 + 2 * kVBlockBytes), b1, id64, 1u);
                  umma_i8(d0 + 32, dsc(a0 + 3 * kVBlockBytes), b1, id64u, 1u);
                }
              }
              umma_commit(tfull0 + 8 * b);    // slot complete (and stage s free, see the producer)
              if (it < 64) FTRACE(it, 2);
            }
            __syncwarp();
          }
        }
      } else
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        for (int sg = 0; sg < kFSlotGroups; sg++, sgc++) {
          const int b = sgc % kFSlots;
          mma_wait(tempty0 + 8 * b, ((sgc / kFSlots) & 1) ^ 1);   // epilogue drained this slot
          tc_fence_after();
          if (sgc < 32 && lane == 0) FTRACE(64 + sgc, 0);
          const int g0 = sg_first(sg), ng = sg_count(sg);
          for (int q = 0; q < ng; q++) {
            const int gi = g0 + q;
            const bool cpx = fg_complex(gi);
            const int kc = fg_kchunk(gi);
            const uint32_t d = tmem + b * kFSlotCols + q * 48;
            for (int k0 = 0; k0 < ksteps; k0 += kc, it++) {
              const int s = it % kFStages;
              mma_wait(full0 + 8 * s, (it / kFStages) & 1);
              tc_fence_after();
              if (it < 64 && lane == 0) FTRACE(it, 1);
              const int kn = min(kc, ksteps - k0);
              const uint32_t st = sbase + s * kFStageBytes;
              if (!(dbg & 2) && elect_one()) {
                for (int kk = 0; kk < kn; ++kk) {
                  const bool first = (k0 + kk) == 0;
                  if (!cpx) {
                    const uint64_t ah = umma_desc(st + (2 * kk) * kVBlockBytes, 128, 256);
                    const uint64_t al = umma_desc(st + (2 * kk + 1) * kVBlockBytes, 128, 256);
                    const uint32_t bw = st + kFStageV + kk * 1024;
                    const uint64_t bb = umma_desc(bw, 128, 256), bl = umma_desc(bw + 512, 128, 256);
                    umma_i8(d, ah, bb, id32, first ? 0u : 1u);                // [s16 | s8]
                    if (first) {
                      umma_i8(d + 32, al, bl, id16u, 0u);                      // s0
                      umma_i8(d + 16, al, bb, id16u, 1u);                      // s8 += lo.hi
                    } else {
                      umma_i8(d + 16, al, bb, id32u, 1u);                      // [s8 | s0]
                    }
                  } else {
                    const uint32_t a0 = st + (4 * kk) * kVBlockBytes;
                    const uint64_t rh = umma_desc(a0, 128, 256), rl = umma_desc(a0 + kVBlockBytes, 128, 256);
                    const uint64_t ih = umma_desc(a0 + 2 * kVBlockBytes, 128, 256),
                                   il = umma_desc(a0 + 3 * kVBlockBytes, 128, 256);
                    const uint32_t bw = st + kFStageV + kk * 4096;
                    const uint64_t b0 = umma_desc(bw, 128, 256), b0l = umma_desc(bw + 1024, 128, 256);
                    const uint64_t b1 = umma_desc(bw + 2048, 128, 256);
                    umma_i8(d, rh, b0, id64, first ? 0u : 1u);                // [Re16 Im16 Re8 Im8]
                    if (first) {
                      umma_i8(d + 64, rl, b0l, id32u, 0u);                     // [Re0 Im0]
                      umma_i8(d + 32, rl, b0, id32u, 1u);                      // [Re8 Im8] += lo.hi
                    } else {
                      umma_i8(d + 32, rl, b0, id64u, 1u);                      // [Re8 Im8 Re0 Im0]
                    }
                    umma_i8(d, ih, b1, id64, 1u);
                    umma_i8(d + 32, il, b1, id64u, 1u);
                  }
                }
              }
              __syncwarp();
              if (elect_one()) umma_commit(empty0 + 8 * s);   // stage reusable once these MMAs have read it
              __syncwarp();
              if (it < 64 && lane == 0) FTRACE(it, 2);
            }
          }
          if (elect_one()) umma_commit(tfull0 + 8 * b);       // slot complete
          __syncwarp();
        }
      }
    }
  } else if (warp < kFEpiWarps) {
    // ------------------------------------------------ epilogue
    const int quad = warp & 3, cw = warp >> 2;
    const int row = quad * 32 + lane;                 // tile within the unit
    const int etid = threadIdx.x;                     // 0..511
    const uint32_t lane_tm = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t lane_base = lane_tm + cw * kFC;
    // Z_0 / Z_5 partials of this thread: 4 x 16-byte chunks each, conflict-free [slot][cw][q][row]
    auto part_ptr = [&](int slot, int q) {
      return reinterpret_cast<int4*>(part + ((((slot * 4 + cw) * 4 + q) * kMBlock + row) << 4));
    };
    int sgc = 0;
    auto combine = [&](const uint32_t (&h)[4], const uint32_t (&x)[4], const uint32_t (&l)[4], int32_t (&v)[4]) {
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = (int32_t)((h[j] << 16) + (x[j] << 8) + l[j]);
    };
    auto slot_wait = [&]() -> uint32_t {
      const int b = sgc % kFSlots;
      epi_wait(tfull0 + 8 * b, (sgc / kFSlots) & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0 && sgc < 32) FTRACE(64 + sgc, 1);
      return lane_base + b * kFSlotCols;
    };
    auto zero_slot = [&](uint32_t a) {   // MG variants: the columns this warp read, back to zero
      if (dbg & 16) return;              // debug builds only: no re-zeroing (results wrong; timing)
      if constexpr (MG == 5) {   // the pack's first UMMA overwrites all but the odd slot's s0 block
        if (sgc & 1) {
          tmem_zero4(a + 64);
          tmem_zero4(a + 80);
          tmem_st_wait();
        }
      } else if constexpr (MG > 0) {
#pragma unroll
        for (int blk = 0; blk < 6; blk++) tmem_zero4(a + blk * 16);
        tmem_st_wait();
      }
    };
    auto slot_release = [&]() {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * (sgc % kFSlots));
      if (warp == 0 && lane == 0 && sgc < 32) FTRACE(64 + sgc, 2);
      sgc++;
    };
    auto etab_ld = [&](int gi) -> uint4 { return *reinterpret_cast<const uint4*>(etab + gi * kFN + cw * kFC); };
    auto rscale = [&](int32_t (&v)[4], const uint4 m) {
      if (dbg & 128) {   // debug builds only: no reverse scaling (results wrong; timing)
        v[0] += m.x; v[1] += m.y; v[2] += m.z; v[3] += m.w;
        return;
      }
      v[0] = frscale(v[0], m.x);
      v[1] = frscale(v[1], m.y);
      v[2] = frscale(v[2], m.z);
      v[3] = frscale(v[3], m.w);
    };
    // two real groups of one slot: M of both, reverse scaled
    auto take_real2 = [&](int gi, int32_t (&m0)[4], int32_t (&m1)[4]) {
      // the m' loads go ahead of the slot wait (the barrier asm is a compiler fence): their latency hides there
      const uint4 ma = etab_ld(gi), mb = etab_ld(gi + 1);
      const uint32_t a = slot_wait();
      uint32_t h0[4], x0[4], l0[4], h1[4], x1[4], l1[4];
      if (dbg & 32) {   // debug builds only: no accumulator loads (results wrong; timing)
#pragma unroll
        for (int j = 0; j < 4; j++) { h0[j] = x0[j] = l0[j] = h1[j] = x1[j] = l1[j] = (uint32_t)(a + j); }
      } else {
        // MG 5 (quarter-K packing): the pair's piece blocks interleave [g0 s16 | g1 s16 | g0 s8 | g1 s8 | ...]
        constexpr uint32_t kO1 = MG == 5 ? 16 : 48, kOs = MG == 5 ? 32 : 16;
        tmem_ld4(a, h0);
        tmem_ld4(a + kOs, x0);
        tmem_ld4(a + 2 * kOs, l0);
        tmem_ld4(a + kO1, h1);
        tmem_ld4(a + kO1 + kOs, x1);
        tmem_ld4(a + kO1 + 2 * kOs, l1);
        tmem_ld_wait();
      }
      zero_slot(a);
      slot_release();
      combine(h0, x0, l0, m0);
      combine(h1, x1, l1, m1);
      rscale(m0, ma);
      rscale(m1, mb);
    };
    auto take_cpx = [&](int gi, int32_t (&re)[4], int32_t (&im)[4]) {
      const uint4 m = etab_ld(gi);
      const uint32_t a = slot_wait();
      uint32_t rh[4], ih[4], rx[4], ix[4], rl[4], il[4];
      if (dbg & 32) {   // debug builds only: no accumulator loads (results wrong; timing)
#pragma unroll
        for (int j = 0; j < 4; j++) { rh[j] = ih[j] = rx[j] = ix[j] = rl[j] = il[j] = (uint32_t)(a + j); }
      } else {
        tmem_ld4(a, rh);
        tmem_ld4(a + 16, ih);
        tmem_ld4(a + 32, rx);
        tmem_ld4(a + 48, ix);
        tmem_ld4(a + 64, rl);
        tmem_ld4(a + 80, il);
        tmem_ld_wait();
      }
      zero_slot(a);
      slot_release();
      combine(rh, rx, rl, re);
      combine(ih, ix, il, im);
      rscale(re, m);
      rscale(im, m);
    };
    // Z of real row R[ri] (processing slot k): real (r, cc) adds a_j[cc] M''; the pair adds 2 Re(i^j z)
    // int8 NHWC output of a unit, staged in `part` as [px][tile][16 couts]: 16-byte chunks to global.
    // Deferred into the NEXT unit's row 0 (after its first two slot-groups, before Z_0 overwrites the
    // staging), so the accumulators of that unit are drained meanwhile instead of stalling its MMAs.
    const bool stage8 = NHWC && OUT8 && (g.cout & 15) == 0;
    // staging tile: the 4-byte word of couts 4cw..4cw+3 of a (pixel, tile) chunk sits at word cw ^ ((tile >> 3) & 3)
    // of its 16-byte chunk, so the 32 rows of a warp store into 32 different banks (the unswizzled layout was a
    // 4-way conflict per store); store_staged puts the words back in cout order
    const uint32_t stg_word = (uint32_t)((cw ^ ((row >> 3) & 3)) * kFC);
    auto unswizzle = [](uint4 v, int rr) -> uint4 {
      const int k = (rr >> 3) & 3;
      if (k & 1) v = make_uint4(v.y, v.x, v.w, v.z);
      if (k & 2) v = make_uint4(v.z, v.w, v.x, v.y);
      return v;
    };
    bool pending = false, staged_read = false;
    int pend_tb = 0, pend_nb = 0;
    auto store_staged = [&](int tb_i, int nb) {
      if (g.pool2) {   // fused 2x2/2 max pool: staged as [pooled px 4][tile][16 couts], one chunk per thread
        const int rr = etid & (kMBlock - 1), ppx = etid >> 7;
        const int tt = tb_i * kMBlock + rr;
        if (tt < imgs * g.tpi) {
          const int ti = fdiv(tt, g.dv_tpi), rem = tt - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
          const int pho = g.ho >> 1, pwo = g.wo >> 1;
          const int py = 2 * ty + (ppx >> 1), px = 2 * (rem - ty * g.tw) + (ppx & 1);
          if (py < pho && px < pwo) {
            int8_t* dst = static_cast<int8_t*>(y) + (((long long)(n0 + ti) * pho + py) * pwo + px) * g.cout + nb * kFN;
            *reinterpret_cast<uint4*>(dst) = unswizzle(*reinterpret_cast<const uint4*>(part + etid * 16), rr);
          }
        }
        return;
      }
      // chunk ch = etid + q * 512: tile rr = etid % 128 for every q (512 = 4 x 128), pixel px = ch / 128
      const int rr = etid & (kMBlock - 1);
      const int tt = tb_i * kMBlock + rr;
      if (tt < imgs * g.tpi) {
        const int ti = fdiv(tt, g.dv_tpi), rem = tt - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
        const int oyb = 4 * ty, oxb = 4 * (rem - ty * g.tw);
        int8_t* base = static_cast<int8_t*>(y) + (long long)(n0 + ti) * g.ho * g.wo * g.cout + nb * kFN;
        constexpr int kQ = (16 * kMBlock) / (kFEpiWarps * 32);
        uint4 val[kQ];
#pragma unroll
        for (int q = 0; q < kQ; q++)   // all staging loads first: one LDS latency instead of kQ
          val[q] = *reinterpret_cast<const uint4*>(part + (etid + q * kFEpiWarps * 32) * 16);
#pragma unroll
        for (int q = 0; q < kQ; q++) {
          const int px = (etid + q * kFEpiWarps * 32) >> 7;
          const int oy = oyb + (px >> 2), ox = oxb + (px & 3);
          if (oy >= g.ho || ox >= g.wo) continue;
          if (dbg & 4096) {   // debug: the same stores to linear (fully coalesced) addresses
            *reinterpret_cast<uint4*>(static_cast<int8_t*>(y) +
                                      ((((long long)tb_i * (g.cout_pad / kFN) + nb) * kQ + q) * 512 + etid) * 16) = val[q];
            continue;
          }
          if (dbg & 8192) {   // debug: streaming (evict-first) stores
            __stcs(reinterpret_cast<uint4*>(base + ((long long)oy * g.wo + ox) * g.cout), unswizzle(val[q], rr));
            continue;
          }
          *reinterpret_cast<uint4*>(base + ((long long)oy * g.wo + ox) * g.cout) = unswizzle(val[q], rr);
        }
      }
    };
    // quarter-K pairing: the sector-pair staging [px 16][tile 128][32 B] behind the 4 x 13 KB ring; the unit of
    // the even cout block fills bytes 0-15 of each 32-byte chunk, the odd one bytes 16-31 (16-byte halves
    // swapped by tile bit 2 and words by tile bits 3-4, so both the staging writes and the reads are
    // conflict-free); after the odd unit a lane pair writes each tile pixel's whole sector
    uint8_t* pstg = smem + kFStages * kQkStage;
    auto store_pair = [&](int tb_i, int nb0) {
      const int half = etid & 1, rr = (etid >> 1) & (kMBlock - 1);
      const int tt = tb_i * kMBlock + rr;
      if (tt >= imgs * g.tpi) return;
      const int ti = fdiv(tt, g.dv_tpi), rem = tt - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
      const int oyb = 4 * ty, oxb = 4 * (rem - ty * g.tw);
      int8_t* base = static_cast<int8_t*>(y) + (long long)(n0 + ti) * g.ho * g.wo * g.cout + (nb0 + half) * kFN;
      uint4 val[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int px = (etid >> 8) + 2 * k;
        val[k] = *reinterpret_cast<const uint4*>(pstg + (px * kMBlock + rr) * 32 + ((half ^ ((rr >> 2) & 1)) * 16));
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int px = (etid >> 8) + 2 * k;
        const int oy = oyb + (px >> 2), ox = oxb + (px & 3);
        if (oy >= g.ho || ox >= g.wo) continue;
        *reinterpret_cast<uint4*>(base + ((long long)oy * g.wo + ox) * g.cout) = unswizzle(val[k], rr);
      }
    };
    auto real_row = [&](int k, int32_t (&Z)[4][4]) {
      const int gb = 5 * k;
      int32_t m0[4], m1[4];
      take_real2(gb, m0, m1);   // cc = 0, 1
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < 4; c++) Z[j][c] = areal(j, 0) * m0[c] + areal(j, 1) * m1[c];
      take_real2(gb + 2, m0, m1);   // cc = 2, 5
      if (k == 0 && pending) {      // the previous unit's output, then nobody reads the staging any more
        if (!(dbg & (256 | 2048))) {
          if (qpair) store_pair(pend_tb, pend_nb);
          else store_staged(pend_tb, pend_nb);
        }
        // the staging (aliased by Z_0, except in pair mode) is free once every thread has read it: the barrier
        // sits just before the Z_0 parking, so the skew of the stores is absorbed by the row's complex group
        staged_read = !qpair;
        pending = false;
      }
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < 4; c++) Z[j][c] += areal(j, 2) * m0[c] + areal(j, 5) * m1[c];
      take_cpx(gb + 4, m0, m1);
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < 4; c++) Z[j][c] += 2 * re_x(j) * m0[c] + 2 * re_y(j) * m1[c];
    };
    // this thread's etab entry (group etid / 16, cout etid % 16) of unit u: the code is loaded from
    // global memory one unit ahead (load_code at the start of a unit, fill_etab at its end), so the
    // load latency never stalls the epilogue
    auto load_code = [&](int u) -> int {
      if (u < n_units && etid < kFGroupsN * kFN) {
        const int gi = etid / kFN, c = etid % kFN;
        const int co = (u % nblocks) * kFN + c;
        return (g.scaling && co < g.cout) ? codes[(long long)co * 36 + fg_pos(gi)] : 0;
      }
      return 0;
    };
    auto fill_etab = [&](int code) {
      if (etid < kFGroupsN * kFN) etab[etid] = lut[code & 63];
    };

    if (dbg & 8) {   // debug: accumulator handshake only
      for (int u = u_first; u < n_units; u = u_next(u))
        for (int sg = 0; sg < kFSlotGroups; sg++) {
          slot_wait();
          slot_release();
        }
    } else {
      fill_etab(load_code(u_first));
      int uc = 0;   // units done (trace index)
      for (int u = u_first; u < n_units; u = u_next(u), uc++) {
        fepi_barrier();                                // etab visible; staging of the previous unit drained
        const int next_code = load_code(u_next(u));
        {
          int32_t Z[4][4];
          real_row(0, Z);                              // row 0 -> Z_0
          if (staged_read) {
            fepi_barrier();
            staged_read = false;
          }
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (!(dbg & (256 | 512))) *part_ptr(0, j) = make_int4(Z[j][0], Z[j][1], Z[j][2], Z[j][3]);
          real_row(1, Z);                              // row 5 -> Z_5
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (!(dbg & (256 | 512))) *part_ptr(1, j) = make_int4(Z[j][0], Z[j][1], Z[j][2], Z[j][3]);
        }
        {
          int32_t Z1[4][4], Z2[4][4];
          real_row(2, Z1);                             // row 1
          real_row(3, Z2);                             // row 2
#pragma unroll
          for (int j = 0; j < 4; j++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
              const int32_t p = Z1[j][c] + Z2[j][c], q = Z1[j][c] - Z2[j][c];
              Z1[j][c] = p;
              Z2[j][c] = q;
            }
          tmem_st16(lane_tm + kFPCol + cw * 16, Z1);   // P
          tmem_st16(lane_tm + kFQCol + cw * 16, Z2);   // Q
        }
        // ---- row 3: Z_3[j] = sum_cc M''[3][cc] a_j[cc], cc = 0,1,2,5 (real a), 3 (i^j), 4 (i^-j)
        int32_t zr[4][4], zi[4][4];
        auto cpx_row = [&](auto kkc) {
          constexpr int kk = decltype(kkc)::value;
          int32_t re[4], im[4];
          take_cpx(20 + kk, re, im);
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int n = kk == 4 ? j : (4 - j);   // power of i for (3,3) / (3,4)
            const int ax = kk < 4 ? areal(j, kk == 3 ? 5 : kk) : 0;
            const int rx = kk < 4 ? ax : re_x(n), ry = kk < 4 ? 0 : re_y(n);
            const int ix = kk < 4 ? 0 : im_x(n), iy = kk < 4 ? ax : im_y(n);
#pragma unroll
            for (int c = 0; c < 4; c++) {
              if (kk == 0) {
                zr[j][c] = rx * re[c] + ry * im[c];
                zi[j][c] = ix * re[c] + iy * im[c];
              } else {
                zr[j][c] += rx * re[c] + ry * im[c];
                zi[j][c] += ix * re[c] + iy * im[c];
              }
            }
          }
        };
        cpx_row(std::integral_constant<int, 0>{});
        cpx_row(std::integral_constant<int, 1>{});
        cpx_row(std::integral_constant<int, 2>{});
        cpx_row(std::integral_constant<int, 3>{});
        cpx_row(std::integral_constant<int, 4>{});
        cpx_row(std::integral_constant<int, 5>{});
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 0, 3);
        tmem_st_wait();

        // ---- Y rows: Y0 = Z_0 + P + 2 Re Z_3, Y2 = P - 2 Re Z_3, Y1 = Q - 2 Im Z_3, Y3 = Q + Z_5 + 2 Im Z_3
        int32_t Y0[4][4], Y1[4][4], Y2[4][4], Y3[4][4];
        tmem_ld16(lane_tm + kFPCol + cw * 16, Y2);     // P
        tmem_ld16(lane_tm + kFQCol + cw * 16, Y1);     // Q
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int4 z0 = (dbg & (256 | 512)) ? make_int4(j, 0, 0, 0) : *part_ptr(0, j);
          const int4 z5 = (dbg & (256 | 512)) ? make_int4(0, j, 0, 0) : *part_ptr(1, j);
          const int32_t a0[4] = {z0.x, z0.y, z0.z, z0.w}, a5[4] = {z5.x, z5.y, z5.z, z5.w};
#pragma unroll
          for (int c = 0; c < 4; c++) {
            const int32_t r2 = 2 * zr[j][c], i2 = 2 * zi[j][c];
            Y0[j][c] = a0[c] + Y2[j][c] + r2;
            Y2[j][c] -= r2;
            Y3[j][c] = Y1[j][c] + a5[c] + i2;
            Y1[j][c] -= i2;
          }
        }
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 1, 3);
        fepi_barrier();                                // every Z_0 / Z_5 read before the staging overwrites them
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 2, 3);
        fill_etab(next_code);                          // this unit's reverse scales are all done

        // ---- out32 = rha(Y / 16) (A11), optional requantisation (A14), crop, store
        const int tb_i = u / nblocks, nb = u - tb_i * nblocks;
        const int t = tb_i * kMBlock + row;            // chunk tile
        const bool tvalid = t < imgs * g.tpi;
        int img = 0, oy0 = 0, ox0 = 0, ni = 0, nj = 0;
        if (tvalid) {
          const int ti = fdiv(t, g.dv_tpi), rem = t - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
          img = n0 + ti;
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
        // RQFAST without the clamp: cvt.pack.sat saturates while packing four values into bytes
        auto outv_unclamped = [&](int32_t yv) -> int32_t {
          const int32_t kpos = rq_shift > 0 ? 8 + (1 << (rq_shift + 3)) : 8;
          const int32_t kneg = rq_shift > 0 ? 17 : 1;
          return (yv + kpos + (yv >> 31) * kneg) >> (rq_shift + 4);
        };
        auto pack_sat4 = [](int32_t a, int32_t b, int32_t c, int32_t d) -> uint32_t {   // bytes [a, b, c, d]
          uint32_t hi, w;
          asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
          asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(b), "r"(a), "r"(hi));
          return w;
        };
        // store output row i (Yi[j][c] = Y[i][j] of couts co0 + c)
        auto emit_row = [&](int i, const int32_t (&Yi)[4][4]) {
          if (stage8) {   // stage [px][tile][16 couts] bytes; 16-byte chunks leave after the barrier
#pragma unroll
            for (int j = 0; j < 4; j++) {
              const uint32_t w = RQFAST ? pack_sat4(outv_unclamped(Yi[j][0]), outv_unclamped(Yi[j][1]),
                                                    outv_unclamped(Yi[j][2]), outv_unclamped(Yi[j][3]))
                                        : __byte_perm(__byte_perm((uint32_t)outv(Yi[j][0]), (uint32_t)outv(Yi[j][1]), 0x0040),
                                                      __byte_perm((uint32_t)outv(Yi[j][2]), (uint32_t)outv(Yi[j][3]), 0x0040),
                                                      0x5410);
              if (dbg & (256 | 1024)) {   // debug bits 256/1024: no staging (kept live)
                if (w == 0x12345678u) *reinterpret_cast<uint32_t*>(part) = w;
              } else if (qpair) {
                *reinterpret_cast<uint32_t*>(pstg + ((i * 4 + j) * kMBlock + row) * 32 +
                                             (((nb & 1) ^ ((row >> 2) & 1)) * 16) + stg_word) = w;
              } else {
                *reinterpret_cast<uint32_t*>(part + ((i * 4 + j) * kMBlock + row) * 16 + stg_word) = w;
              }
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
                  *reinterpret_cast<int4*>(dst) =
                      make_int4(outv(Yi[0][c]), outv(Yi[1][c]), outv(Yi[2][c]), outv(Yi[3][c]));
                } else {
#pragma unroll
                  for (int j = 0; j < 4; j++)
                    if (j < nj) dst[j] = outv(Yi[j][c]);
                }
              }
            }
          }
        };
        if (stage8 && g.pool2) {   // int8 words of the 4 x 4 block, then the 2 x 2 pooled block (signed byte max)
          auto word = [&](const int32_t (&Yi)[4][4], int j) -> uint32_t {
            return RQFAST ? pack_sat4(outv_unclamped(Yi[j][0]), outv_unclamped(Yi[j][1]), outv_unclamped(Yi[j][2]),
                                      outv_unclamped(Yi[j][3]))
                          : __byte_perm(__byte_perm((uint32_t)outv(Yi[j][0]), (uint32_t)outv(Yi[j][1]), 0x0040),
                                        __byte_perm((uint32_t)outv(Yi[j][2]), (uint32_t)outv(Yi[j][3]), 0x0040), 0x5410);
          };
#pragma unroll
          for (int pj = 0; pj < 2; pj++) {
            const uint32_t top = __vmaxs4(__vmaxs4(word(Y0, 2 * pj), word(Y0, 2 * pj + 1)),
                                          __vmaxs4(word(Y1, 2 * pj), word(Y1, 2 * pj + 1)));
            const uint32_t bot = __vmaxs4(__vmaxs4(word(Y2, 2 * pj), word(Y2, 2 * pj + 1)),
                                          __vmaxs4(word(Y3, 2 * pj), word(Y3, 2 * pj + 1)));
            *reinterpret_cast<uint32_t*>(part + ((0 * 2 + pj) * kMBlock + row) * 16 + stg_word) = top;
            *reinterpret_cast<uint32_t*>(part + ((1 * 2 + pj) * kMBlock + row) * 16 + stg_word) = bot;
          }
        } else {
          emit_row(0, Y0);
          emit_row(1, Y1);
          emit_row(2, Y2);
          emit_row(3, Y3);
        }
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 3, 3);
        fepi_barrier();                                // staging complete; etab of the next unit visible
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 4, 3);
        if (stage8 && (!qpair || (nb & 1))) {   // stored during the next unit's row 0 (or after the last unit)
          pending = true;
          pend_tb = tb_i;
          pend_nb = qpair ? nb - 1 : nb;
        }
        if (warp == 0 && lane == 0) FTRACE(uc * 8 + 5, 3);
      }
      if (pending && !(dbg & (256 | 2048))) {
        if (qpair) store_pair(pend_tb, pend_nb);
        else store_staged(pend_tb, pend_nb);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
#undef FTRACE
}

static int g_fused_sms = 0;
static uint64_t* g_fused_trace = nullptr;
void set_fused_trace(void* buf) { g_fused_trace = static_cast<uint64_t*>(buf); }
// WINO_FUSED_DBG env (debug builds with -DWINO_FUSED_DBG only): 2 no MMAs, 4 no copies (MG > 0), 8 epilogue
// handshake only, 16 no TMEM re-zeroing, 32 no accumulator loads, 64 one UMMA per group, 128 no reverse-scale
// multiply, 256 no epilogue shared-memory traffic (= 512 no Z_0/Z_5 parking + 1024 no output staging + 2048 no
// staged output stores), 4096 output stores to linear addresses, 8192 streaming (.cs) output stores
static int g_fused_dbg = 0;
// fewest CTAs for the same number of unit rounds (C2: 196 units -> 98 CTAs x 2 instead of 148 + 48): the
// freed SMs run the other streams' kernels for the whole launch (C2 190.7 -> 203.1, C3 310.7 -> 332.1 TOPS
// with three batches in flight); WINO_FUSED_BALANCE=0 restores the full grid (experiments)
static int g_fused_balance = 1;
// WINO_FUSED_MAXCTA: cap on the fused kernel's grid, leaving SMs to the other lanes' kernels (experiments)
static int g_fused_maxcta = 0;
static int g_fused_merge = 4;   // WINO_FUSED_MERGE: 4 also two slot-groups per stage at c_in <= 32; 0 general loops only, 1 merged stages at c_in <= 64,
                                // 2 also at c_in <= 128, 3 also 4-K-step slot-group stages above

cudaError_t launch_fused(const Geom& g, long long tiles_pad_launch, int n0, int imgs, const int8_t* vimg,
                         const int8_t* wimg, const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y,
                         cudaStream_t st) {
  if (g.nblk != kFN) return cudaErrorInvalidValue;
  const int tblocks = (int)(tiles_pad_launch / kMBlock);
  const int n_units = tblocks * (g.cout_pad / kFN);
  const int cap = g_fused_maxcta > 0 && g_fused_maxcta < g_fused_sms ? g_fused_maxcta : g_fused_sms;
  // quarter-K pairing (see k_fused): a CTA takes pairs of units
  const bool qpair = g.qk && g.layout == 1 && g.out_mode == 0 && (g.cout & 15) == 0 && !g.pool2 &&
                     (g.cout_pad / kFN) % 2 == 0;
  const int work = qpair ? n_units / 2 : n_units;
  int grid = work < cap ? work : cap;
  if (g_fused_balance) {   // fewest CTAs with the same number of unit rounds: the rest of the SMs stay free
    const int rounds = (work + grid - 1) / grid;
    grid = (work + rounds - 1) / rounds;
  }
  const size_t smem = fused_smem_bytes();
  const bool nhwc = g.layout == 1, out8 = g.out_mode == 0, fast = rq_mult == 1 && rq_shift <= 20;
  cudaError_t e;
#define WINO_KF(A, B, C)                                                                                       \
  e = g.qk                                                                                                      \
          ? launch_pdl(k_fused<A, B, C, 5>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)                                \
      : g.ksteps == 1 && g_fused_merge >= 4                                                                        \
          ? launch_pdl(k_fused<A, B, C, 4>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)                                \
      : g.ksteps <= 2 && g_fused_merge >= 1                                                                        \
          ? launch_pdl(k_fused<A, B, C, 1>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)                                \
      : g.ksteps <= 4 && g_fused_merge >= 2                                                                      \
          ? launch_pdl(k_fused<A, B, C, 2>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)                                \
      : g_fused_merge >= 3                                                                                       \
          ? launch_pdl(k_fused<A, B, C, 3>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)                                \
          : launch_pdl(k_fused<A, B, C, 0>, dim3(grid), dim3(kFThreads), smem, st, vimg, wimg, codes, g, n0, imgs,    \
                       tblocks, rq_mult, rq_shift, y, g_fused_dbg, g_fused_trace)
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
  if (const char* d = std::getenv("WINO_FUSED_BALANCE")) g_fused_balance = std::atoi(d);
  if (const char* d = std::getenv("WINO_FUSED_MERGE")) g_fused_merge = std::atoi(d);
  if (const char* d = std::getenv("WINO_FUSED_MAXCTA")) g_fused_maxcta = std::atoi(d);
  const int smem = (int)fused_smem_bytes();
#define WINO_KF_ATTR(A, B, C)                                                                                     \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<A, B, C, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
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
