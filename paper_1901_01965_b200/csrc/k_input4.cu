// k_input4.cu -- K2F for NHWC int8 input: the input-tile gather + D = B^T d B of the
// fused path, four channels per thread in 16-bit SWAR lanes.
//
// Thread = (tile, 4 consecutive channels); warp = 8 consecutive tiles (one 8-row core-matrix group of the
// UMMA layout) x 16 channels (one 16-byte K half), so each 4-byte store of a warp fills one contiguous
// 128-byte run.  Per pixel one 4-byte load; the four int8 values become offset-binary bytes x + 128
// (XOR 0x80) and two SWAR words A = u0 + 2^16 u1, B = u2 + 2^16 u3 (exact integers; every transform step
// is an add or subtract of such words, exact as long as |lane| < 2^15, which the 12-bit range of D
// guarantees, Appendix A).  The offset-binary bias reaches a single Winograd position: B^T 1 = 4 e_1, so
// D(x + 128) = D(x) + 2048 [position (1,1)], removed there with one subtraction.
//
// Piece encoding of the fused V image (layout.cuh): v = 256 hi + lo with lo = v & 255 (u8) and
// hi = v >> 8 (s8, [-8, 7]); the fused GEMM reads lo pieces as unsigned A operands.  From a SWAR word
// P = L0 + 2^16 L1: lo(L0), hi(L0) are bytes 0, 1 of P (the low lane is exact modulo 2^16) and lo(L1),
// hi(L1) bytes 2, 3 of P + 2048 (L0 + 2048 >= 0 carries no borrow into the high lane).
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kI4Warps = 8;
constexpr int kI4TilesPerWarp = 8;
constexpr int kI4TilesPerCta = kI4Warps * kI4TilesPerWarp;   // 64
constexpr int kI4ChPerCta = 16;

// the two 4-byte piece words (lo, hi) of four channels from the SWAR words A (channels 0, 1), B (2, 3)
__device__ __forceinline__ void pieces4(uint32_t A, uint32_t B, uint32_t& lo, uint32_t& hi) {
  const uint32_t t1 = __byte_perm(A, A + 2048u, 0x7160);   // [lo0, lo1, hi0, hi1]
  const uint32_t t2 = __byte_perm(B, B + 2048u, 0x7160);   // [lo2, lo3, hi2, hi3]
  lo = __byte_perm(t1, t2, 0x5410);
  hi = __byte_perm(t1, t2, 0x7632);
}

__device__ __forceinline__ void st32(int8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
__device__ __forceinline__ void st32d(int8_t* p, uint32_t v, int dbg) {
  if (!(dbg & 1) || v == 0x7f7f7f7fu) st32(p, v);   // debug: stores skipped (kept live by the impossible test)
}

// store the value (A, B) of a group's value slot: pieces at p (hi) and p + 4 KB (lo)
__device__ __forceinline__ void store_val(int8_t* p_hi, uint32_t A, uint32_t B, int dbg) {
  uint32_t lo, hi;
  pieces4(A, B, lo, hi);
  st32d(p_hi, hi, dbg);
  st32d(p_hi + kVBlockBytes, lo, dbg);
}

// D = B^T d B of one (tile t, 4 channels c) patch w (SWAR-ready words: 4 int8 channels per pixel, 0 outside the
// map) and the stores of its 36 values' pieces into the fused V image (or the quarter-K packed image, QK)
template <int KS, bool QK>
__device__ __forceinline__ void k2f_transform_store(const Geom& g, const uint32_t (&w)[36], int8_t* __restrict__ vimg,
                                                    int t, int c, int dbg) {
  const int ksteps = KS ? KS : g.ksteps;
  const long long kst = (long long)ksteps * kVBlockBytes;
  int8_t* base = vimg + (long long)(t / kMBlock) * kVPiecesF * kst + tiled_offset(t % kMBlock, c & 31, kMBlock);
  int8_t* base2 = base + (long long)((c >> 5) * 2) * kVBlockBytes;   // real groups: 2 pieces per K step
  int8_t* base4 = base + (long long)((c >> 5) * 4) * kVBlockBytes;   // complex groups: 4 pieces
  auto gp = [&](int gi) { return (fg_pieces(gi) == 2 ? base2 : base4) + fg_vprefix(gi) * kst; };
  // QK: (t / 128) pack blocks, row r, channel slot c; value part vp of group gi at byte qk_kbyte(gi, vp, c)
  int8_t* qbase = vimg + (long long)(t / kMBlock) * kQkPacks * kQkPackV + tiled_offset(t % kMBlock, c, kMBlock);
  // hi-piece address of value part vp (0; 1 = a complex group's Im) of group gi (lo piece 4 KB after it)
  auto vp_addr = [&](int gi, int vp) -> int8_t* {
    if constexpr (QK) {
      const int kb = qk_kbyte(gi, vp, 0);
      return qbase + (qk_sg_of(gi) / 2) * kQkPackV + (kb >> 4) * 128 + (kb & 15);
    } else {
      return gp(gi) + vp * 2 * kVBlockBytes;
    }
  };
  // ---- d' = B^T d per column on SWAR words: rows e0, e1, e2, e5 real, row 3 = ra + i rb
  uint32_t e0[6][2], e1[6][2], e2[6][2], e5[6][2], ra[6][2], rb[6][2];
#pragma unroll
  for (int j = 0; j < 6; j++) {
    uint32_t P[6][2];
#pragma unroll
    for (int a = 0; a < 6; a++) {
      const uint32_t u = w[a * 6 + j] ^ 0x80808080u;   // offset binary x + 128
      P[a][0] = __byte_perm(u, 0u, 0x4140);            // channels 0, 1 in 16-bit lanes
      P[a][1] = __byte_perm(u, 0u, 0x4342);            // channels 2, 3
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t s24 = P[2][h] + P[4][h], s13 = P[1][h] + P[3][h];
      e0[j][h] = P[0][h] - P[4][h];
      e1[j][h] = s13 + s24;
      e2[j][h] = s24 - s13;
      ra[j][h] = P[4][h] - P[2][h];    // Re d'[3][j]
      rb[j][h] = P[3][h] - P[1][h];    // Im d'[3][j]
      e5[j][h] = P[5][h] - P[1][h];
    }
  }

  // ---- D = d' B along each real row (R[ri], .): 4 real positions and the primary (R[ri], 3)
  auto real_row = [&](auto ric, const uint32_t (&e)[6][2]) {
    constexpr int ri = decltype(ric)::value;
    uint32_t v[6][2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t s24 = e[2][h] + e[4][h], s13 = e[1][h] + e[3][h];
      v[0][h] = e[0][h] - e[4][h];      // (R[ri], 0)
      v[1][h] = s13 + s24;              // (R[ri], 1)
      v[2][h] = s24 - s13;              // (R[ri], 2)
      v[3][h] = e[5][h] - e[1][h];      // (R[ri], 5)
      v[4][h] = e[4][h] - e[2][h];      // Re (R[ri], 3)
      v[5][h] = e[3][h] - e[1][h];      // Im (R[ri], 3)
    }
    if constexpr (ri == 1) {            // position (1,1): remove the offset-binary bias 2048 from both lanes
      v[1][0] -= 0x08000800u;
      v[1][1] -= 0x08000800u;
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
      const int gi = fg_of_real(ri * 4 + s);
      store_val(vp_addr(gi, QK ? gi - qk_sg_first(qk_sg_of(gi)) : 0), v[s][0], v[s][1], dbg);
    }
    store_val(vp_addr(fg_of_primary(ri), 0), v[4][0], v[4][1], dbg);   // Re: pieces 0 (hi), 1 (lo)
    store_val(vp_addr(fg_of_primary(ri), 1), v[5][0], v[5][1], dbg);   // Im: pieces 2, 3 (QK: value part 1)
  };
  real_row(std::integral_constant<int, 0>{}, e0);
  real_row(std::integral_constant<int, 1>{}, e1);
  real_row(std::integral_constant<int, 2>{}, e2);
  real_row(std::integral_constant<int, 3>{}, e5);

  // ---- complex row 3 = a + i b: (3,0) (3,1) (3,2) (3,5) -> primaries 4..7, (3,3) -> 8, (3,4) -> 9
  uint32_t re[4][2], im[4][2], q[4][2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    auto A = [&](int j) { return ra[j][h]; };
    auto Bv = [&](int j) { return rb[j][h]; };
    const uint32_t as24 = A(2) + A(4), as13 = A(1) + A(3), bs24 = Bv(2) + Bv(4), bs13 = Bv(1) + Bv(3);
    re[0][h] = A(0) - A(4); re[1][h] = as13 + as24; re[2][h] = as24 - as13; re[3][h] = A(5) - A(1);
    im[0][h] = Bv(0) - Bv(4); im[1][h] = bs13 + bs24; im[2][h] = bs24 - bs13; im[3][h] = Bv(5) - Bv(1);
    // (3,3) = (e4 - e2) + i (e3 - e1), (3,4) = (e4 - e2) - i (e3 - e1), e = a + i b
    q[0][h] = A(4) - A(2) - Bv(3) + Bv(1);
    q[1][h] = Bv(4) - Bv(2) + A(3) - A(1);
    q[2][h] = A(4) - A(2) + Bv(3) - Bv(1);
    q[3][h] = Bv(4) - Bv(2) - A(3) + A(1);
  }
#pragma unroll
  for (int j = 0; j < 4; j++) {
    store_val(vp_addr(fg_of_primary(4 + j), 0), re[j][0], re[j][1], dbg);
    store_val(vp_addr(fg_of_primary(4 + j), 1), im[j][0], im[j][1], dbg);
  }
  store_val(vp_addr(fg_of_primary(8), 0), q[0][0], q[0][1], dbg);
  store_val(vp_addr(fg_of_primary(8), 1), q[1][0], q[1][1], dbg);
  store_val(vp_addr(fg_of_primary(9), 0), q[2][0], q[2][1], dbg);
  store_val(vp_addr(fg_of_primary(9), 1), q[3][0], q[3][1], dbg);
}

// a 16-channel slice past c_in: V = 0 (both pieces of every group) for (tile t, channels c..c+3)
template <int KS>
__device__ __forceinline__ void k2f_zero_slice(const Geom& g, int8_t* __restrict__ vimg, int t, int c) {
  const int ksteps = KS ? KS : g.ksteps;
  const long long kst = (long long)ksteps * kVBlockBytes;
  int8_t* base = vimg + (long long)(t / kMBlock) * kVPiecesF * kst + tiled_offset(t % kMBlock, c & 31, kMBlock);
  int8_t* base2 = base + (long long)((c >> 5) * 2) * kVBlockBytes;
  int8_t* base4 = base + (long long)((c >> 5) * 4) * kVBlockBytes;
#pragma unroll
  for (int gi = 0; gi < kFGroupsN; gi++) {
    int8_t* p = (fg_pieces(gi) == 2 ? base2 : base4) + fg_vprefix(gi) * kst;
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (q < fg_pieces(gi)) st32(p + q * kVBlockBytes, 0u);
  }
}

// c_in < 4: the 6 pixels of each of the 6 patch rows from aligned words (see the QK gather below)
template <int CIN>
__device__ __forceinline__ void gather_rows_small(const int8_t* p0, long long rstride, uint32_t (&w)[36]) {
  constexpr uint32_t kMask = (1u << (8 * CIN)) - 1u;
#pragma unroll
  for (int a = 0; a < 6; a++) {
    const int8_t* rp = p0 + a * rstride;
    const uint32_t off = (uint32_t)(reinterpret_cast<uintptr_t>(rp) & 3u);
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp - off);
    uint32_t W[6], R[5];
#pragma unroll
    for (int k = 0; k < 6; k++) W[k] = __ldg(wp + k);
#pragma unroll
    for (int k = 0; k < 5; k++) R[k] = __funnelshift_r(W[k], W[k + 1], off * 8u);   // row bytes from byte 0
#pragma unroll
    for (int b = 0; b < 6; b++) {
      const int B = b * CIN;   // compile-time after unrolling
      const uint32_t v = (B & 3) == 0 ? R[B >> 2] : __funnelshift_r(R[B >> 2], R[(B >> 2) + 1], (B & 3) * 8);
      w[a * 6 + b] = v & kMask;
    }
  }
}

// QK: the quarter-K packed V image (c_in <= 8, layout.cuh): thread = (tile, 4 of the 8 channel slots), warp =
// 16 tiles, CTA = one 128-tile block; the (group, value part) of a value selects its pack and K byte
template <int KS, int MINB, bool QK = false>   // KS: g.ksteps as a compile-time constant (1, 2, 4, 8, 16; 0 = runtime)
__global__ void __launch_bounds__(kI4Warps * 32, MINB)
    k_input_transform_f4(Geom g, const int8_t* __restrict__ x, int n0, int imgs, int8_t* __restrict__ vimg, int dbg,
                         int spc) {
#ifndef WINO_K2_DBG
  dbg = 0;   // ablation bits (debug builds only): 1 no V stores, 2 no x loads
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // spc 16-channel slices per CTA (warp w: tile group w / spc, slice w % spc), so the warps that read the
  // same pixels' bytes share the CTA's L1 (WINO_K2F4_SPC)
  const int slice = QK ? 0 : blockIdx.y * spc + warp % spc;
  const int t = QK ? blockIdx.x * kMBlock + warp * 16 + (lane >> 1)
                   : blockIdx.x * (kI4TilesPerCta / spc) + (warp / spc) * kI4TilesPerWarp + (lane >> 2);
  const int c = QK ? 4 * (lane & 1) : slice * kI4ChPerCta + 4 * (lane & 3);
  pdl_trigger();
  pdl_wait();   // x may come from the previous kernel; V may still be read by the previous GEMM

  const int tiles = imgs * g.tpi;
  if (!QK && slice * kI4ChPerCta >= g.cin) {   // a slice of padding channels only: V = 0 (both pieces)
    k2f_zero_slice<KS>(g, vimg, t, c);
    return;
  }

  // ---- gather the zero-padded 6x6 patch (4 channels per pixel word; 0 outside the map / past c_in)
  uint32_t w[36];
  {
    int img = 0, iy0 = -1000000, ix0 = -1000000;
    if (t < tiles) {
      const int ti = fdiv(t, g.dv_tpi), rem = t - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
      img = n0 + ti;
      iy0 = 4 * ty - g.pad;
      ix0 = 4 * (rem - ty * g.tw) - g.pad;
    }
    const long long rstride = (long long)g.w * g.cin;
    const int8_t* p0 = x + ((long long)img * g.h * g.w + (long long)iy0 * g.w + ix0) * g.cin + c;
    const bool inside = t < tiles && c + 4 <= g.cin && iy0 >= 0 && iy0 + 6 <= g.h && ix0 >= 0 && ix0 + 6 <= g.w;
    if (dbg & 2) {   // debug: no loads (a lane-dependent pattern instead)
#pragma unroll
      for (int i = 0; i < 36; i++) w[i] = (uint32_t)(t * 0x01010101u + i);
    } else if (QK && g.cin < 4 && __all_sync(0xffffffffu, t >= tiles || c > 0 ||
                                                 (iy0 >= 0 && iy0 + 6 < g.h && ix0 >= 0 && ix0 + 6 <= g.w))) {
      // c_in < 4 (VGG-16 layer 1: 3 bytes per pixel): a patch row is 6 c_in contiguous bytes; read it as the
      // 6 aligned 4-byte words covering it, realign them with funnel shifts and cut the pixels out at static
      // byte offsets (6 loads per row instead of 6 c_in byte loads); the row below exists (iy0 + 6 < h), so the
      // last word stays inside the tensor
#pragma unroll
      for (int i = 0; i < 36; i++) w[i] = 0u;
      if (t < tiles && c == 0) {
        if (g.cin == 3) gather_rows_small<3>(p0, rstride, w);
        else if (g.cin == 2) gather_rows_small<2>(p0, rstride, w);
        else gather_rows_small<1>(p0, rstride, w);
      }
    } else if ((g.cin & 3) == 0 && __all_sync(0xffffffffu, inside)) {
      // interior warp: unpredicated 4-byte loads; column offsets b * c_in are immediates when c_in = 32 KS
      const int cst = (KS > 0 && g.cin == 32 * KS) ? 32 * KS : g.cin;
#pragma unroll
      for (int a = 0; a < 6; a++) {
        const int8_t* rp = p0 + a * rstride;
#pragma unroll
        for (int b = 0; b < 6; b++) w[a * 6 + b] = __ldg(reinterpret_cast<const uint32_t*>(rp + b * cst));
      }
    } else {
      bool vx[6];
#pragma unroll
      for (int b = 0; b < 6; b++) vx[b] = t < tiles && ix0 + b >= 0 && ix0 + b < g.w;
      const bool vec = (g.cin & 3) == 0 && c + 4 <= g.cin;
#pragma unroll
      for (int a = 0; a < 6; a++) {
        const bool vy = iy0 + a >= 0 && iy0 + a < g.h;
        const int8_t* rp = p0 + a * rstride;
#pragma unroll
        for (int b = 0; b < 6; b++) {
          uint32_t v = 0u;
          if (vy && vx[b]) {
            const int8_t* pp = rp + (long long)b * g.cin;
            if (vec) {
              v = __ldg(reinterpret_cast<const uint32_t*>(pp));
            } else {   // c_in % 4 != 0 or a partial quad: byte loads of the channels below c_in
#pragma unroll
              for (int j = 0; j < 4; j++)
                if (c + j < g.cin) v |= (uint32_t)(uint8_t)__ldg(pp + j) << (8 * j);
            }
          }
          w[a * 6 + b] = v;
        }
      }
    }
  }
  k2f_transform_store<KS, QK>(g, w, vimg, t, c, dbg);
}

cudaError_t launch_input_transform_f4(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg,
                                      cudaStream_t st) {
  const long long tiles = (long long)imgs * g.tpi;
  const long long tiles_pad = (tiles + kMBlock - 1) / kMBlock * kMBlock;
  // 16-channel slices per CTA: 4 (2 when c_in_pad is not a multiple of 64) -- the four warps that read a
  // pixel's 64 channel bytes (two 32-byte sectors) sit in one CTA and share its L1 instead of four CTAs each
  // pulling the sectors from L2: a batch-512 C2-shaped layer 144 -> 103 us, VGG-16 layers 2-5 K2 -33 %,
  // C5 526 -> 555 TOPS; WINO_K2F4_SPC = 1 / 2 / 4 overrides (experiments)
  static const int spc_env = [] { const char* e = std::getenv("WINO_K2F4_SPC"); return e ? std::atoi(e) : 4; }();
  const int spc = (spc_env == 4 && g.cin_pad % 64 == 0) ? 4 : (spc_env >= 2 ? 2 : 1);
  dim3 grid((unsigned)(tiles_pad / (kI4TilesPerCta / spc)), g.cin_pad / (kI4ChPerCta * spc));
  // CTAs per SM the register budget targets (WINO_K2F4_MINB; 3 measured best at C2 and the VGG-16 stack)
  static const int dbg = [] { const char* e = std::getenv("WINO_K2_DBG"); return e ? std::atoi(e) : 0; }();
  static const int minb = [] { const char* e = std::getenv("WINO_K2F4_MINB"); return e ? std::atoi(e) : 3; }();
#define WINO_K2F4(K, M) \
  launch_pdl_co(k_input_transform_f4<K, M>, grid, dim3(kI4Warps * 32), 0, st, kCarveL1, g, x, n0, imgs, vimg, dbg, spc)
#define WINO_K2F4_M(M)              \
  switch (g.ksteps) {               \
    case 1: return WINO_K2F4(1, M);   \
    case 2: return WINO_K2F4(2, M);   \
    case 4: return WINO_K2F4(4, M);   \
    case 8: return WINO_K2F4(8, M);   \
    case 16: return WINO_K2F4(16, M); \
    default: return WINO_K2F4(0, M);  \
  }
  if (g.qk) {   // quarter-K packed V (c_in <= 8): one CTA per 128-tile block
    return launch_pdl_co(k_input_transform_f4<1, 3, true>, dim3((unsigned)(tiles_pad / kMBlock)),
                         dim3(kI4Warps * 32), 0, st, kCarveL1, g, x, n0, imgs, vimg, dbg, 1);
  }
  if (minb >= 4) { WINO_K2F4_M(4) }
  if (minb == 3) { WINO_K2F4_M(3) }
  WINO_K2F4_M(2)
#undef WINO_K2F4_M
#undef WINO_K2F4
}

}  // namespace wino
