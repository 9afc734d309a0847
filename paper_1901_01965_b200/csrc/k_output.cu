// k_output.cu -- K4: on the 36 values per (tile, cout) that K3 leaves (M'':
// 16 real, 10 Re, 10 Im after Karatsuba recombination and reverse scaling), the
// real-only output transform Y = A^T M'' A that never forms the imaginary
// coefficients, out32 = rha(Y / 16) (G used as 4G,
// DESIGN.md A2/A11), crop, optional requantisation (A14) and the store.
//
// One thread per (tile, output channel); consecutive threads take
// consecutive channels, so the 36 slot reads of M (layout.cuh) are coalesced.
//
// Real-only transform.  A^T rows are a_0 = (1,1,1,1,1,0), a_1 = (0,1,-1,i,-i,0),
// a_2 = (0,1,1,-1,-1,0), a_3 = (0,1,-1,-i,i,1); a_j4 = conj(a_j3).  For a row
// r in {0,1,2,5} with real entries M0,M1,M2,M5 and primary z = x + iy at
// column 3 (column 4 holds conj z):
//   Z[r][0] = M0+M1+M2+2x   Z[r][1] = M1-M2-2y   Z[r][2] = M1+M2-2x   Z[r][3] = M1-M2+M5+2y
// Row 3 is complex (w_c at c in {0,1,2,5}, w3 = M[3][3], w4 = M[3][4]) and
// row 4 is its conjugate, so
//   Y[0][j] = Z0+Z1+Z2+2Re Z3   Y[1][j] = Z1-Z2-2Im Z3
//   Y[2][j] = Z1+Z2-2Re Z3      Y[3][j] = Z1-Z2+Z5+2Im Z3.
// All sums are int32 with wrap-around: exact because the true Y fits (A23).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kOutCoBlock = 64;                       // couts per CTA
constexpr int kOutTiles = 256 / kOutCoBlock;            // tiles per CTA

// |Y| < 2^31 - 8 for every supported plan (16 * 128^2 * 9 * 896 < 2^31 - 8),
// so rha(Y / 16) is exact in 32-bit arithmetic.
__device__ __forceinline__ int32_t rha16_32(uint32_t yv) {
  const int32_t y = (int32_t)yv;
  const int32_t r = (abs(y) + 8) >> 4;
  return y < 0 ? -r : r;
}

// NHWC: layout 1 / 0; OUT8: int8 (requantised) / int32 output; RQFAST: multiplier 1
// and shift <= 30, so requantisation fits 32-bit arithmetic.
template <bool NHWC, bool OUT8, bool RQFAST>
__global__ void __launch_bounds__(256) k_output_transform(Geom g, const int32_t* __restrict__ M, int n0, int imgs,
                                                          int32_t rq_mult, int rq_shift, void* __restrict__ y) {
  const int tl = threadIdx.x / kOutCoBlock, cl = threadIdx.x % kOutCoBlock;
  const int t = blockIdx.x * kOutTiles + tl;              // chunk tile
  const int co = blockIdx.y * kOutCoBlock + cl;
  pdl_trigger();
  pdl_wait();   // M'' comes from the GEMM just before
  if (t >= imgs * g.tpi || co >= g.cout) return;
  const long long ps = g.chunk_tiles_pad * (long long)g.cout_pad;
  const int32_t* mp = M + m_offset(g, t, co);

  uint32_t mr[16], cr[10], cim[10];
#pragma unroll
  for (int s = 0; s < 16; s++) mr[s] = (uint32_t)__ldg(mp + s * ps);
#pragma unroll
  for (int k = 0; k < 10; k++) {
    cr[k] = (uint32_t)__ldg(mp + (16 + k) * ps);
    cim[k] = (uint32_t)__ldg(mp + (26 + k) * ps);
  }
  // Z = M'' A  (rows 0,1,2,5 real; row 3 complex)
  uint32_t Z[4][4], zr[4], zi[4];
#pragma unroll
  for (int ri = 0; ri < 4; ri++) {
    uint32_t M0 = mr[ri * 4], M1 = mr[ri * 4 + 1], M2 = mr[ri * 4 + 2], M5 = mr[ri * 4 + 3];
    uint32_t x2 = 2 * cr[ri], y2 = 2 * cim[ri];
    Z[ri][0] = M0 + M1 + M2 + x2;
    Z[ri][1] = M1 - M2 - y2;
    Z[ri][2] = M1 + M2 - x2;
    Z[ri][3] = M1 - M2 + M5 + y2;
  }
  {
    uint32_t w0r = cr[4], w1r = cr[5], w2r = cr[6], w5r = cr[7], w3r = cr[8], w4r = cr[9];
    uint32_t w0i = cim[4], w1i = cim[5], w2i = cim[6], w5i = cim[7], w3i = cim[8], w4i = cim[9];
    zr[0] = w0r + w1r + w2r + w3r + w4r;        zi[0] = w0i + w1i + w2i + w3i + w4i;
    zr[1] = w1r - w2r - w3i + w4i;              zi[1] = w1i - w2i + w3r - w4r;
    zr[2] = w1r + w2r - w3r - w4r;              zi[2] = w1i + w2i - w3i - w4i;
    zr[3] = w1r - w2r + w3i - w4i + w5r;        zi[3] = w1i - w2i - w3r + w4r + w5i;
  }
  const int ti = fdiv(t, g.dv_tpi), img = n0 + ti, rem = t - ti * g.tpi;
  const int ty = fdiv(rem, g.dv_tw), tx = rem - ty * g.tw;
  const int oy0 = 4 * ty, ox0 = 4 * tx;
  const int ni = min(4, g.ho - oy0), nj = min(4, g.wo - ox0);
  // output element (oy0 + i, ox0 + j) = ybase + i * ystride + j * xstride (element units)
  const int xstride = NHWC ? g.cout : 1, ystride = NHWC ? g.wo * g.cout : g.wo;
  const long long ybase = NHWC ? (((long long)img * g.ho + oy0) * g.wo + ox0) * g.cout + co
                               : (((long long)img * g.cout + co) * g.ho + oy0) * g.wo + ox0;
  int8_t* y8 = static_cast<int8_t*>(y) + (OUT8 ? ybase : 0);
  int32_t* y32 = static_cast<int32_t*>(y) + (OUT8 ? 0 : ybase);
  const uint32_t rq_half = rq_shift > 0 ? (1u << (rq_shift - 1)) : 0u;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    uint32_t Yc[4];
    Yc[0] = Z[0][j] + Z[1][j] + Z[2][j] + 2 * zr[j];
    Yc[1] = Z[1][j] - Z[2][j] - 2 * zi[j];
    Yc[2] = Z[1][j] + Z[2][j] - 2 * zr[j];
    Yc[3] = Z[1][j] - Z[2][j] + Z[3][j] + 2 * zi[j];
    if (j >= nj) break;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      if (i >= ni) break;
      const int32_t o32 = rha16_32(Yc[i]);   // rha(Y / 16)
      const int off = i * ystride + j * xstride;
      if (!OUT8) {
        y32[off] = o32;
      } else if (RQFAST) {
        const uint32_t a = (uint32_t)abs(o32);
        const int32_t r = (int32_t)((a + rq_half) >> rq_shift);   // |o32| + 2^29 < 2^32
        y8[off] = (int8_t)(o32 < 0 ? max(-r, -128) : min(r, 127));
      } else {
        long long r = rq_shift > 0 ? rha_shift64((long long)o32 * rq_mult, rq_shift) : (long long)o32 * rq_mult;
        y8[off] = (int8_t)(r > 127 ? 127 : (r < -128 ? -128 : r));
      }
    }
  }
}

// Same transform, one thread per (tile, 4 consecutive couts): the 36 slot reads are 16-byte loads
// (4 couts share one 16-byte chunk of an M'' tile row, layout.cuh), 16 threads cover a tile row of
// 64 couts (256 contiguous bytes).  Requires cout % 4 == 0.
constexpr int kOut4Quads = 16, kOut4Tiles = 16;   // 256 threads: 16 tiles x 64 couts
template <bool NHWC, bool OUT8, bool RQFAST, bool POOL = false>
__global__ void __launch_bounds__(256, 2) k_output_transform4(Geom g, const int32_t* __restrict__ M, int n0, int imgs,
                                                           int32_t rq_mult, int rq_shift, void* __restrict__ y) {
  const int tl = threadIdx.x / kOut4Quads, ql = threadIdx.x % kOut4Quads;
  const int t = blockIdx.x * kOut4Tiles + tl;
  const int co0 = (blockIdx.y * kOut4Quads + ql) * 4;
  pdl_trigger();
  pdl_wait();   // M'' comes from the GEMM just before
  if (t >= imgs * g.tpi || co0 >= g.cout) return;
  const long long ps = g.chunk_tiles_pad * (long long)g.cout_pad;
  const int4* mp = reinterpret_cast<const int4*>(M + m_offset(g, t, co0));
  const long long ps4 = ps / 4;
  int4 v[36];
#pragma unroll
  for (int s = 0; s < 36; s++) v[s] = __ldg(mp + s * ps4);
  const int ti = fdiv(t, g.dv_tpi), img = n0 + ti, rem = t - ti * g.tpi;
  const int ty = fdiv(rem, g.dv_tw), tx = rem - ty * g.tw;
  const int oy0 = 4 * ty, ox0 = 4 * tx;
  const int ni = min(4, g.ho - oy0), nj = min(4, g.wo - ox0);
  const uint32_t rq_half = rq_shift > 0 ? (1u << (rq_shift - 1)) : 0u;
  auto comp = [](const int4& q, int c) -> uint32_t {
    return (uint32_t)(c == 0 ? q.x : (c == 1 ? q.y : (c == 2 ? q.z : q.w)));
  };
  auto requant = [&](uint32_t yv) -> int32_t {
    const int32_t o32 = rha16_32(yv);
    if (!OUT8) return o32;
    if (RQFAST) {
      const uint32_t a = (uint32_t)abs(o32);
      const int32_t r = (int32_t)((a + rq_half) >> rq_shift);
      return o32 < 0 ? max(-r, -128) : min(r, 127);
    }
    long long r = rq_shift > 0 ? rha_shift64((long long)o32 * rq_mult, rq_shift) : (long long)o32 * rq_mult;
    return (int32_t)(r > 127 ? 127 : (r < -128 ? -128 : r));
  };
  uint32_t out[4][4][4];   // [c][i][j]
#pragma unroll
  for (int c = 0; c < 4; c++) {
    uint32_t Z[4][4], zr[4], zi[4];
#pragma unroll
    for (int ri = 0; ri < 4; ri++) {
      const uint32_t M0 = comp(v[ri * 4], c), M1 = comp(v[ri * 4 + 1], c), M2 = comp(v[ri * 4 + 2], c),
                     M5 = comp(v[ri * 4 + 3], c);
      const uint32_t x2 = 2 * comp(v[16 + ri], c), y2 = 2 * comp(v[26 + ri], c);
      Z[ri][0] = M0 + M1 + M2 + x2;
      Z[ri][1] = M1 - M2 - y2;
      Z[ri][2] = M1 + M2 - x2;
      Z[ri][3] = M1 - M2 + M5 + y2;
    }
    {
      const uint32_t w0r = comp(v[20], c), w1r = comp(v[21], c), w2r = comp(v[22], c), w5r = comp(v[23], c),
                     w3r = comp(v[24], c), w4r = comp(v[25], c);
      const uint32_t w0i = comp(v[30], c), w1i = comp(v[31], c), w2i = comp(v[32], c), w5i = comp(v[33], c),
                     w3i = comp(v[34], c), w4i = comp(v[35], c);
      zr[0] = w0r + w1r + w2r + w3r + w4r;        zi[0] = w0i + w1i + w2i + w3i + w4i;
      zr[1] = w1r - w2r - w3i + w4i;              zi[1] = w1i - w2i + w3r - w4r;
      zr[2] = w1r + w2r - w3r - w4r;              zi[2] = w1i + w2i - w3i - w4i;
      zr[3] = w1r - w2r + w3i - w4i + w5r;        zi[3] = w1i - w2i - w3r + w4r + w5i;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      out[c][0][j] = (uint32_t)requant(Z[0][j] + Z[1][j] + Z[2][j] + 2 * zr[j]);
      out[c][1][j] = (uint32_t)requant(Z[1][j] - Z[2][j] - 2 * zi[j]);
      out[c][2][j] = (uint32_t)requant(Z[1][j] + Z[2][j] - 2 * zr[j]);
      out[c][3][j] = (uint32_t)requant(Z[1][j] - Z[2][j] + Z[3][j] + 2 * zi[j]);
    }
  }
  if constexpr (POOL) {   // NHWC int8 with the fused 2x2/2 max pool (g.pool2): the tile's 2x2 pooled block
    const int pho = g.ho >> 1, pwo = g.wo >> 1;
#pragma unroll
    for (int pi = 0; pi < 2; pi++) {
      const int py = 2 * ty + pi;
      if (py >= pho) break;
#pragma unroll
      for (int pj = 0; pj < 2; pj++) {
        const int px = 2 * tx + pj;
        if (px >= pwo) break;
        uint32_t word = 0;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const int m = max(max((int)out[c][2 * pi][2 * pj], (int)out[c][2 * pi][2 * pj + 1]),
                            max((int)out[c][2 * pi + 1][2 * pj], (int)out[c][2 * pi + 1][2 * pj + 1]));
          word |= ((uint32_t)m & 0xffu) << (8 * c);
        }
        *reinterpret_cast<uint32_t*>(static_cast<int8_t*>(y) + (((long long)img * pho + py) * pwo + px) * g.cout +
                                     co0) = word;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    if (i >= ni) break;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j >= nj) break;
      if (NHWC) {
        const long long pix = ((long long)img * g.ho + oy0 + i) * g.wo + ox0 + j;
        if (OUT8) {
          *reinterpret_cast<uint32_t*>(static_cast<int8_t*>(y) + pix * g.cout + co0) =
              (out[0][i][j] & 0xffu) | ((out[1][i][j] & 0xffu) << 8) | ((out[2][i][j] & 0xffu) << 16) |
              (out[3][i][j] << 24);
        } else {
          *reinterpret_cast<int4*>(static_cast<int32_t*>(y) + pix * g.cout + co0) =
              make_int4((int)out[0][i][j], (int)out[1][i][j], (int)out[2][i][j], (int)out[3][i][j]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const long long off = (((long long)img * g.cout + co0 + c) * g.ho + oy0 + i) * g.wo + ox0 + j;
          if (OUT8) static_cast<int8_t*>(y)[off] = (int8_t)out[c][i][j];
          else static_cast<int32_t*>(y)[off] = (int32_t)out[c][i][j];
        }
      }
    }
  }
}

// ---- rational F(2x2,3x3): Y = A^T M'' A with A^T = [[1,1,1,0],[0,1,-1,-1]] (A25)
// on the 16 M'' slots (position i*4 + j), out32 = rha(Y / 4) (A26), requantisation, 2x2 store.
template <bool NHWC, bool OUT8, bool RQFAST>
__global__ void __launch_bounds__(256) k_output_transform2(Geom g, const int32_t* __restrict__ M, int n0, int imgs,
                                                           int32_t rq_mult, int rq_shift, void* __restrict__ y) {
  const int tl = threadIdx.x / kOutCoBlock, cl = threadIdx.x % kOutCoBlock;
  const int t = blockIdx.x * kOutTiles + tl;
  const int co = blockIdx.y * kOutCoBlock + cl;
  pdl_trigger();
  pdl_wait();
  if (t >= imgs * g.tpi || co >= g.cout) return;
  const long long ps = g.chunk_tiles_pad * (long long)g.cout_pad;
  const int32_t* mp = M + m_offset(g, t, co);
  uint32_t m[16];
#pragma unroll
  for (int s = 0; s < 16; s++) m[s] = (uint32_t)__ldg(mp + s * ps);
  uint32_t Z[2][4];   // A^T M''
#pragma unroll
  for (int j = 0; j < 4; j++) {
    Z[0][j] = m[0 * 4 + j] + m[1 * 4 + j] + m[2 * 4 + j];
    Z[1][j] = m[1 * 4 + j] - m[2 * 4 + j] - m[3 * 4 + j];
  }
  const int ti = fdiv(t, g.dv_tpi), img = n0 + ti, rem = t - ti * g.tpi;
  const int ty = fdiv(rem, g.dv_tw), tx = rem - ty * g.tw;
  const int oy0 = 2 * ty, ox0 = 2 * tx;
  const int ni = min(2, g.ho - oy0), nj = min(2, g.wo - ox0);
  const uint32_t rq_half = rq_shift > 0 ? (1u << (rq_shift - 1)) : 0u;
#pragma unroll
  for (int i = 0; i < 2; i++) {
    if (i >= ni) break;
    const uint32_t Yr[2] = {Z[i][0] + Z[i][1] + Z[i][2], Z[i][1] - Z[i][2] - Z[i][3]};   // (A^T M'') A
#pragma unroll
    for (int j = 0; j < 2; j++) {
      if (j >= nj) break;
      const int32_t yv = (int32_t)Yr[j];
      const int32_t o32 = (yv + 2 + (yv >> 31)) >> 2;   // rha(Y / 4), |Y| < 2^31 - 2
      const long long yi = NHWC ? (((long long)img * g.ho + oy0 + i) * g.wo + ox0 + j) * g.cout + co
                                : (((long long)img * g.cout + co) * g.ho + oy0 + i) * g.wo + ox0 + j;
      if (!OUT8) {
        static_cast<int32_t*>(y)[yi] = o32;
      } else if (RQFAST) {
        const uint32_t a = (uint32_t)abs(o32);
        const int32_t r = (int32_t)((a + rq_half) >> rq_shift);
        static_cast<int8_t*>(y)[yi] = (int8_t)(o32 < 0 ? max(-r, -128) : min(r, 127));
      } else {
        long long r = rq_shift > 0 ? rha_shift64((long long)o32 * rq_mult, rq_shift) : (long long)o32 * rq_mult;
        static_cast<int8_t*>(y)[yi] = (int8_t)(r > 127 ? 127 : (r < -128 ? -128 : r));
      }
    }
  }
}

cudaError_t launch_output_transform(const Geom& g, const int32_t* m, int n0, int imgs, int32_t rq_mult,
                                    int rq_shift, void* y, cudaStream_t st) {
  const int tiles = imgs * g.tpi;
  dim3 grid((unsigned)((tiles + kOutTiles - 1) / kOutTiles), (unsigned)((g.cout + kOutCoBlock - 1) / kOutCoBlock));
  const bool nhwc = g.layout == 1, out8 = g.out_mode == 0, fast = rq_mult == 1 && rq_shift <= 30;
  cudaError_t e;
  if (g.alg == 1) {   // rational F(2x2)
#define WINO_K42(A, B, C) e = launch_pdl_co(k_output_transform2<A, B, C>, grid, dim3(256), 0, st, kCarveL1, g, m, n0, imgs, rq_mult, rq_shift, y)
    if (nhwc) {
      if (!out8) WINO_K42(true, false, false);
      else if (fast) WINO_K42(true, true, true);
      else WINO_K42(true, true, false);
    } else {
      if (!out8) WINO_K42(false, false, false);
      else if (fast) WINO_K42(false, true, true);
      else WINO_K42(false, true, false);
    }
#undef WINO_K42
    return e;
  }
  if (nhwc && (g.cout & 3) == 0) {   // vectorised variant (NHWC; NCHW keeps one cout per thread)
    dim3 grid4((unsigned)((tiles + kOut4Tiles - 1) / kOut4Tiles), (unsigned)((g.cout + 63) / 64));
#define WINO_K4V(B, C) e = launch_pdl_co(k_output_transform4<true, B, C>, grid4, dim3(256), 0, st, kCarveL1, g, m, n0, imgs, rq_mult, rq_shift, y)
    if (g.pool2) {
      if (fast) e = launch_pdl_co(k_output_transform4<true, true, true, true>, grid4, dim3(256), 0, st, kCarveL1, g, m,
                                  n0, imgs, rq_mult, rq_shift, y);
      else e = launch_pdl_co(k_output_transform4<true, true, false, true>, grid4, dim3(256), 0, st, kCarveL1, g, m, n0,
                             imgs, rq_mult, rq_shift, y);
      return e;
    }
    if (!out8) WINO_K4V(false, false);
    else if (fast) WINO_K4V(true, true);
    else WINO_K4V(true, false);
#undef WINO_K4V
    return e;
  }
#define WINO_K4(A, B, C) e = launch_pdl_co(k_output_transform<A, B, C>, grid, dim3(256), 0, st, kCarveL1, g, m, n0, imgs, rq_mult, rq_shift, y)
  if (nhwc) {
    if (!out8) WINO_K4(true, false, false);
    else if (fast) WINO_K4(true, true, true);
    else WINO_K4(true, true, false);
  } else {
    if (!out8) WINO_K4(false, false, false);
    else if (fast) WINO_K4(false, true, true);
    else WINO_K4(false, true, false);
  }
#undef WINO_K4
  return e;
}

cudaError_t setup_output_transform() { return cudaSuccess; }

// ------------------------------------------------------------------ misc
// valid: 0, or a 6-bit code with n in [8,15]; int8-native target (f3): a 7-bit code with n in [8,15], p in [4,8]
__global__ void k_check_codes(const uint8_t* __restrict__ codes, int count, int code7, int32_t* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    int c = codes[i];
    const bool ok = c == 0 || (code7 ? (c < 128 && (c >> 3) >= 8 && (c & 7) <= 4) : (c < 64 && (c >> 2) >= 8));
    if (!ok) atomicOr(bad, 1);
  }
}
cudaError_t launch_check_codes(const uint8_t* codes, int count, int code7, int32_t* bad, cudaStream_t st) {
  k_check_codes<<<(count + 255) / 256, 256, 0, st>>>(codes, count, code7, bad);
  return cudaGetLastError();
}

__global__ void k_maxpool2(const int8_t* __restrict__ x, int n, int h, int w, int c, int layout, int8_t* __restrict__ y) {
  const int ho = h / 2, wo = w / 2;
  const long long total = (long long)n * ho * wo * c;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int ci, ox, oy, img;
  if (layout == 1) {
    ci = (int)(i % c); long long r = i / c; ox = (int)(r % wo); r /= wo; oy = (int)(r % ho); img = (int)(r / ho);
  } else {
    ox = (int)(i % wo); long long r = i / wo; oy = (int)(r % ho); r /= ho; ci = (int)(r % c); img = (int)(r / c);
  }
  int m = -128;
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      int yy = 2 * oy + a, xx = 2 * ox + b;
      int v = layout == 1 ? x[(((long long)img * h + yy) * w + xx) * c + ci] : x[(((long long)img * c + ci) * h + yy) * w + xx];
      m = v > m ? v : m;
    }
  y[i] = (int8_t)m;
}
// NHWC with c % 16 == 0 and 16-byte aligned tensors: thread = (output pixel, 16 channels), four 16-byte
// loads, per-byte signed max, one 16-byte store (bandwidth-bound; the per-element kernel above spent
// ~10x the time in index arithmetic and byte loads)
__global__ void k_maxpool2_nhwc16(const uint4* __restrict__ x, int h, int w, int c16, long long total,
                                  uint4* __restrict__ y) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int wo = w >> 1, ho = h >> 1;
  const int cg = (int)(i % c16);
  long long r = i / c16;
  const int ox = (int)(r % wo);
  r /= wo;
  const int oy = (int)(r % ho);
  const long long img = r / ho;
  const long long p00 = ((img * h + 2 * oy) * w + 2 * ox) * c16 + cg;
  const long long rowst = (long long)w * c16;
  const uint4 a = __ldg(x + p00), b = __ldg(x + p00 + c16), d = __ldg(x + p00 + rowst),
              e = __ldg(x + p00 + rowst + c16);
  uint4 m;
  m.x = __vmaxs4(__vmaxs4(a.x, b.x), __vmaxs4(d.x, e.x));
  m.y = __vmaxs4(__vmaxs4(a.y, b.y), __vmaxs4(d.y, e.y));
  m.z = __vmaxs4(__vmaxs4(a.z, b.z), __vmaxs4(d.z, e.z));
  m.w = __vmaxs4(__vmaxs4(a.w, b.w), __vmaxs4(d.w, e.w));
  y[i] = m;
}

cudaError_t launch_maxpool2(const int8_t* x, int n, int h, int w, int c, int layout, int8_t* y, cudaStream_t st) {
  if (layout == 1 && (c & 15) == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
    const long long total = (long long)n * (h / 2) * (w / 2) * (c / 16);
    k_maxpool2_nhwc16<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(x), h, w,
                                                                        c / 16, total, reinterpret_cast<uint4*>(y));
    return cudaGetLastError();
  }
  long long total = (long long)n * (h / 2) * (w / 2) * c;
  k_maxpool2<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(x, n, h, w, c, layout, y);
  return cudaGetLastError();
}

}  // namespace wino
