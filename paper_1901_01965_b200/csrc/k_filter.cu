// k_filter.cu -- K1: offline filter transform W = G_int g G_int^T, the
// paper's per-(OFM, position) integer scale factors, downscale, Karatsuba
// operand planes and int8 piece split.
//
// One warp per output channel (see k_filter_transform); the transform is
// recomputed in the second pass instead of being stored.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

// Slot order inside one channel's 36 values:
//   0..15  real positions (R[s/4], R[s%4]), R = {0,1,2,5}
//   16+2k, 17+2k   re, im of complex primary k (layout.cuh order)
__device__ __forceinline__ void filter_tile_transform(const int g[3][3], int out[36]) {
  // u = G_int g  (rows 0,1,2,5 real; row 3 = a + i b), G_int rows
  // (4,0,0) (1,1,1) (1,-1,1) (1,i,-1) [(1,-i,-1)] (0,0,4)   -- P:154-160 times 4
  int u0[3], u1[3], u2[3], u5[3], a[3], b[3];
#pragma unroll
  for (int j = 0; j < 3; j++) {
    u0[j] = 4 * g[0][j];
    u1[j] = g[0][j] + g[1][j] + g[2][j];
    u2[j] = g[0][j] - g[1][j] + g[2][j];
    a[j] = g[0][j] - g[2][j];
    b[j] = g[1][j];
    u5[j] = 4 * g[2][j];
  }
  // W = u G_int^T, row by row; for a real row e: W[.][0]=4e0, W[.][1]=e0+e1+e2,
  // W[.][2]=e0-e1+e2, W[.][5]=4e2, W[.][3]=(e0-e2) + i e1.
  const int* rows[4] = {u0, u1, u2, u5};
#pragma unroll
  for (int ri = 0; ri < 4; ri++) {
    const int* e = rows[ri];
    out[ri * 4 + 0] = 4 * e[0];
    out[ri * 4 + 1] = e[0] + e[1] + e[2];
    out[ri * 4 + 2] = e[0] - e[1] + e[2];
    out[ri * 4 + 3] = 4 * e[2];
    out[16 + 2 * ri] = e[0] - e[2];   // primary k = ri : (R[ri], 3)
    out[17 + 2 * ri] = e[1];
  }
  // complex row 3: e = a + i b
  // (3,0)=4e0  (3,1)=e0+e1+e2  (3,2)=e0-e1+e2  (3,5)=4e2
  out[16 + 8] = 4 * a[0];             out[17 + 8] = 4 * b[0];
  out[16 + 10] = a[0] + a[1] + a[2];  out[17 + 10] = b[0] + b[1] + b[2];
  out[16 + 12] = a[0] - a[1] + a[2];  out[17 + 12] = b[0] - b[1] + b[2];
  out[16 + 14] = 4 * a[2];            out[17 + 14] = 4 * b[2];
  // (3,3) = (e0 - e2) + i e1 ;  (3,4) = (e0 - e2) - i e1
  out[16 + 16] = a[0] - a[2] - b[1];  out[17 + 16] = b[0] - b[2] + a[1];
  out[16 + 18] = a[0] - a[2] + b[1];  out[17 + 18] = b[0] - b[2] - a[1];
}

__device__ __forceinline__ int rha_mul_shift(int v, int n, int p) {  // rha(v n / 2^p)
  int prod = v * n;
  int a = prod < 0 ? -prod : prod;
  int r = (a + (1 << (p - 1))) >> p;
  return prod < 0 ? -r : r;
}

constexpr int kFilterWarps = 8;   // warps per CTA; one CTA per output channel

// Scaled operand planes of one (cout, cin) filter: 46 values.
__device__ __forceinline__ void scaled_planes(const int t[36], const int* sn, const int* sp, int vals[46]) {
#pragma unroll
  for (int s = 0; s < 16; s++) vals[s] = sn[s] ? rha_mul_shift(t[s], sn[s], sp[s]) : t[s];   // W' = rha(W n / 2^p)
#pragma unroll
  for (int k = 0; k < 10; k++) {
    const int n = sn[16 + k], p = sp[16 + k];
    const int re = n ? rha_mul_shift(t[16 + 2 * k], n, p) : t[16 + 2 * k];
    const int im = n ? rha_mul_shift(t[17 + 2 * k], n, p) : t[17 + 2 * k];
    vals[16 + 3 * k + 0] = re;
    vals[16 + 3 * k + 1] = im;
    vals[16 + 3 * k + 2] = re + im;
  }
}

// One 3x3 filter as int values: int8 w, or uint8 w minus its zero point (int9, f2, A28).
__device__ __forceinline__ void load_filter(const Geom& g, const int8_t* __restrict__ w, int co, int ci, int gg[3][3]) {
#pragma unroll
  for (int u = 0; u < 3; u++)
#pragma unroll
    for (int v = 0; v < 3; v++) {
      const int8_t raw = g.layout == 0 ? w[((long long)co * g.cin + ci) * 9 + u * 3 + v]
                                       : w[((long long)co * 9 + u * 3 + v) * g.cin + ci];
      gg[u][v] = g.in_u8 ? (int)(uint8_t)raw - g.zw : (int)raw;
    }
}

// One CTA per output channel (the unit the paper scales: "applied to
// the filters used to generate one output feature map"), channels split over
// its warps.
//   pass 1: transform every input channel (thread-strided), max magnitude per
//           position across channels, codes (P:322-330 read as A3);
//   pass 2: per 32-channel group (one per warp), recompute, scale, split and
//           stage the 92 operand bytes per channel in shared memory, then write
//           whole 16-byte rows of the pre-tiled W image.
//   FUSED: the fused path's group layout instead (layout.cuh): per group the rows
//   real [W hi, W lo], complex [Wr hi, Wi hi, Wr lo, Wi lo, -Wi hi, Wr hi, -Wi lo, Wr lo]
//   (balanced s8 pieces), 112 staged rows per channel.
//   W1: the int8-native target (A29): real positions bound |W| by 127,
//   complex ones |Re| + |Im| by 126, x = floor(target 256 / max), p = 11 - y, 7-bit codes; each
//   of the 46 planes is ONE s8 operand (w1_offset), 46 staged rows per channel.
template <bool FUSED, bool W1 = false>
__global__ void __launch_bounds__(kFilterWarps * 32) k_filter_transform(Geom g, const int8_t* __restrict__ w,
                                                                         int8_t* __restrict__ wimg,
                                                                         uint8_t* __restrict__ codes) {
  constexpr int kRows = FUSED ? 2 * kWRowUnitsF : (W1 ? kPlanes : 2 * kPlanes);
  __shared__ __align__(16) int8_t s_stage[kFilterWarps][kRows][32];
  __shared__ int s_max[kFilterWarps][26];
  __shared__ int s_n[26], s_p[26];
  __shared__ uint8_t s_gi[FUSED ? kRows : 1];   // FUSED: group of each staged row (read after pass 1's barriers)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int co = blockIdx.x;
  const bool live = co < g.cout;
  pdl_trigger();
  if constexpr (FUSED) {
    for (int sr = threadIdx.x; sr < kRows; sr += blockDim.x) {   // the last group whose 2 * wprefix <= sr
      int gi = 0;
      for (int q = 1; q < kFGroupsN; q++) gi += (2 * fg_wprefix(q) <= sr) ? 1 : 0;
      s_gi[sr] = (uint8_t)gi;
    }
  }
  pdl_wait();   // w_wino / codes are read by the previous step's GEMM

  int mx[26];
#pragma unroll
  for (int i = 0; i < 26; i++) mx[i] = 0;
  // the transform of this thread's first channel (ci = threadIdx.x) stays in registers for pass 2,
  // whose first iteration handles the same channel (every channel when cin <= blockDim)
  int t0[36];
#pragma unroll
  for (int i = 0; i < 36; i++) t0[i] = 0;
  if (live) {
    for (int ci = threadIdx.x; ci < g.cin; ci += blockDim.x) {
      int gg[3][3], t[36];
      load_filter(g, w, co, ci, gg);
      filter_tile_transform(gg, t);
      if (ci == (int)threadIdx.x) {
#pragma unroll
        for (int i = 0; i < 36; i++) t0[i] = t[i];
      }
#pragma unroll
      for (int s = 0; s < 16; s++) mx[s] = max(mx[s], abs(t[s]));
#pragma unroll
      for (int k = 0; k < 10; k++)
        mx[16 + k] = max(mx[16 + k], W1 ? abs(t[16 + 2 * k]) + abs(t[17 + 2 * k])
                                        : max(abs(t[16 + 2 * k]), abs(t[17 + 2 * k])));
    }
  }
#pragma unroll
  for (int i = 0; i < 26; i++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[i] = max(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
    if (lane == 0) s_max[warp][i] = mx[i];
  }
  __syncthreads();
  if (threadIdx.x < 26) {
    int m = 0;
#pragma unroll
    for (int wv = 0; wv < kFilterWarps; wv++) m = max(m, s_max[wv][threadIdx.x]);
    int n = 0, p = 0;
    const int tgt = W1 ? (threadIdx.x < 16 ? 127 : 126) : g.target;
    if (g.scaling && m > tgt) {
      // P:322-329 read per DESIGN.md A3: x = floor(255*128/max), y = floor(log2 x),
      // n = x >> (y - 3) (4-bit, in [8, 15]), p = 10 - y (in [4, 7]).  W1 (A29): one more
      // bit, x = floor(tgt*256/max), p = 11 - y (in [4, 8]).
      const int x = (tgt * (W1 ? 256 : 128)) / m;
      const int y = 31 - __clz(x);
      n = y >= 3 ? (x >> (y - 3)) : (x << (3 - y));
      p = (W1 ? 11 : 10) - y;
    }
    s_n[threadIdx.x] = n;
    s_p[threadIdx.x] = p;
    if (live) {
      const int i = threadIdx.x;
      // 6-bit code, W1 7-bit (A29); 0 = unscaled
      const uint8_t code = (uint8_t)(n ? (W1 ? ((n << 3) | (p - 4)) : ((n << 2) | (p - 4))) : 0);
      if (i < 16) {
        codes[co * 36 + real_pos(i)] = code;
      } else {
        codes[co * 36 + cpx_pos(i - 16)] = code;
        codes[co * 36 + cpx_mirror_pos(i - 16)] = code;   // mirrors share the factor
      }
    }
  }
  __syncthreads();
  int sn[26], sp[26];
#pragma unroll
  for (int i = 0; i < 26; i++) { sn[i] = s_n[i]; sp[i] = s_p[i]; }

  for (int c0 = warp * 32; c0 < g.cin_pad; c0 += kFilterWarps * 32) {
    const int ci = c0 + lane;
    int vals[46];
    if (live && ci < g.cin) {
      if (c0 == warp * 32) {   // ci == threadIdx.x: transformed in pass 1
        scaled_planes(t0, sn, sp, vals);
      } else {
        int gg[3][3], t[36];
        load_filter(g, w, co, ci, gg);
        filter_tile_transform(gg, t);
        scaled_planes(t, sn, sp, vals);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 46; i++) vals[i] = 0;
    }
    if constexpr (W1) {
#pragma unroll
      for (int pl = 0; pl < 46; pl++) s_stage[warp][pl][lane] = (int8_t)vals[pl];   // |W'| <= 127 (A29)
      __syncwarp();
      for (int idx = lane; idx < kPlanes * 2; idx += 32) {   // (plane, 16-channel half)
        const int pl = idx >> 1, hf = idx & 1;
        const int4 v = *reinterpret_cast<const int4*>(&s_stage[warp][pl][hf * 16]);
        *reinterpret_cast<int4*>(wimg + w1_offset(g, pl, co, c0 + hf * 16)) = v;
      }
    } else if constexpr (!FUSED) {
#pragma unroll
      for (int pl = 0; pl < 46; pl++) {
        s_stage[warp][2 * pl + 0][lane] = (int8_t)bal_hi(vals[pl]);   // balanced s8 pieces (layout.cuh)
        s_stage[warp][2 * pl + 1][lane] = (int8_t)bal_lo(vals[pl]);
      }
      __syncwarp();
      for (int idx = lane; idx < 2 * kPlanes * 2; idx += 32) {   // (piece-plane, 16-channel half)
        const int pp = idx >> 1, hf = idx & 1;
        const int4 v = *reinterpret_cast<const int4*>(&s_stage[warp][pp][hf * 16]);
        *reinterpret_cast<int4*>(wimg + w_offset(g, pp >> 1, pp & 1, co, c0 + hf * 16)) = v;
      }
    } else if (g.qk) {
      // quarter-K packing (c_in <= 8, layout.cuh): this cout's 10 rows of each pack's B (4 rows of slot 2P,
      // 2 zero rows, 4 rows of slot 2P+1), 32 K bytes each, channel ci at byte part * 8 + ci of its slot half
      int8_t (*st8)[32] = s_stage[warp];
      for (int i = lane; i < kQkPacks * 10 * 8; i += 32) reinterpret_cast<int*>(st8)[i] = 0;
      __syncwarp();
      if (ci < 8) {
#pragma unroll
        for (int pk = 0; pk < kQkPacks; pk++)
#pragma unroll
          for (int sp = 0; sp < 2; sp++) {
            const int sg = 2 * pk + sp, g0 = qk_sg_first(sg);
            int8_t (*r)[32] = st8 + pk * 10 + (sp ? 6 : 0);   // the slot's 4 rows
            const int b0 = sp * 16 + ci, b1 = b0 + 8;          // value parts 0 and 1
            if (!fg_complex(g0)) {
              const int v0 = vals[fg_real_plane(g0)], v1 = vals[fg_real_plane(g0 + 1)];
              r[0][b0] = (int8_t)bal_hi(v0);
              r[1][b1] = (int8_t)bal_hi(v1);
              r[2][b0] = (int8_t)bal_lo(v0);
              r[3][b1] = (int8_t)bal_lo(v1);
            } else {
              const int k = fg_primary(g0);
              const int wr = vals[16 + 3 * k], wi = vals[16 + 3 * k + 1], nwi = -wi;
              r[0][b0] = (int8_t)bal_hi(wr);  r[0][b1] = (int8_t)bal_hi(nwi);   // Re16: Vr Wr - Vi Wi
              r[1][b0] = (int8_t)bal_hi(wi);  r[1][b1] = (int8_t)bal_hi(wr);    // Im16: Vr Wi + Vi Wr
              r[2][b0] = (int8_t)bal_lo(wr);  r[2][b1] = (int8_t)bal_lo(nwi);
              r[3][b0] = (int8_t)bal_lo(wi);  r[3][b1] = (int8_t)bal_lo(wr);
            }
          }
      }
      __syncwarp();
      if (c0 == 0) {
        const int nb = co / kFN16, cr = co % kFN16;
        for (int idx = lane; idx < kQkPacks * 10 * 2; idx += 32) {   // (pack, staged row, 16-byte K half)
          const int pk = idx / 20, j = (idx >> 1) % 10, kh = idx & 1;
          const int row = (j < 4 ? 16 * j : (j < 6 ? 64 + 16 * (j - 4) : 96 + 16 * (j - 6))) + cr;
          const int4 v = *reinterpret_cast<const int4*>(&st8[pk * 10 + j][kh * 16]);
          *reinterpret_cast<int4*>(wimg + wq_offset(nb, pk, row, kh * 16)) = v;
        }
      }
    } else {
      // staged row 2 * wprefix(gi) + j holds piece-row j of group gi for this cout
#pragma unroll
      for (int s = 0; s < 16; s++) {
        const int r0 = 2 * fg_wprefix(fg_of_real(s));
        s_stage[warp][r0 + 0][lane] = (int8_t)bal_hi(vals[s]);
        s_stage[warp][r0 + 1][lane] = (int8_t)bal_lo(vals[s]);
      }
#pragma unroll
      for (int k = 0; k < 10; k++) {
        const int r0 = 2 * fg_wprefix(fg_of_primary(k));
        const int wr = vals[16 + 3 * k], wi = vals[16 + 3 * k + 1], nwi = -wi;
        s_stage[warp][r0 + 0][lane] = (int8_t)bal_hi(wr);
        s_stage[warp][r0 + 1][lane] = (int8_t)bal_hi(wi);
        s_stage[warp][r0 + 2][lane] = (int8_t)bal_lo(wr);
        s_stage[warp][r0 + 3][lane] = (int8_t)bal_lo(wi);
        s_stage[warp][r0 + 4][lane] = (int8_t)bal_hi(nwi);
        s_stage[warp][r0 + 5][lane] = (int8_t)bal_hi(wr);
        s_stage[warp][r0 + 6][lane] = (int8_t)bal_lo(nwi);
        s_stage[warp][r0 + 7][lane] = (int8_t)bal_lo(wr);
      }
      __syncwarp();
      const int nb = co / kFN16, cr = co % kFN16;
      for (int idx = lane; idx < kRows * 2; idx += 32) {   // (staged row, 16-channel half)
        const int sr = idx >> 1, hf = idx & 1;
        const int gi = s_gi[sr];   // group of staged row sr
        const int j = sr - 2 * fg_wprefix(gi);
        const int4 v = *reinterpret_cast<const int4*>(&s_stage[warp][sr][hf * 16]);
        *reinterpret_cast<int4*>(wimg + wf_offset(g, gi, nb, j * kFN16 + cr, c0 + hf * 16)) = v;
      }
    }
    __syncwarp();
  }
}

// ---- rational F(2x2,3x3): W = G' g G'^T, G' = 2G, 16 real positions
// (row-major 4x4), the same per-(OFM, position) scaling, staged W' layout with 16 planes.
__device__ __forceinline__ void filter_tile_transform2(const int g[3][3], int out[16]) {
  int u[4][3];   // G' g: rows 2 g0 | g0 + g1 + g2 | g0 - g1 + g2 | 2 g2
#pragma unroll
  for (int j = 0; j < 3; j++) {
    u[0][j] = 2 * g[0][j];
    u[1][j] = g[0][j] + g[1][j] + g[2][j];
    u[2][j] = g[0][j] - g[1][j] + g[2][j];
    u[3][j] = 2 * g[2][j];
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {   // (G' g) G'^T row by row
    out[i * 4 + 0] = 2 * u[i][0];
    out[i * 4 + 1] = u[i][0] + u[i][1] + u[i][2];
    out[i * 4 + 2] = u[i][0] - u[i][1] + u[i][2];
    out[i * 4 + 3] = 2 * u[i][2];
  }
}

__global__ void __launch_bounds__(kFilterWarps * 32) k_filter_transform2(Geom g, const int8_t* __restrict__ w,
                                                                          int8_t* __restrict__ wimg,
                                                                          uint8_t* __restrict__ codes) {
  __shared__ __align__(16) int8_t s_stage[kFilterWarps][32][32];   // 16 planes x 2 pieces per channel
  __shared__ int s_max[kFilterWarps][16];
  __shared__ int s_n[16], s_p[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int co = blockIdx.x;
  const bool live = co < g.cout;
  pdl_trigger();
  pdl_wait();
  int mx[16];
#pragma unroll
  for (int i = 0; i < 16; i++) mx[i] = 0;
  if (live) {
    for (int ci = threadIdx.x; ci < g.cin; ci += blockDim.x) {   // steps 1-2: transform, max magnitude
      int gg[3][3], t[16];
      load_filter(g, w, co, ci, gg);
      filter_tile_transform2(gg, t);
#pragma unroll
      for (int s = 0; s < 16; s++) mx[s] = max(mx[s], abs(t[s]));
    }
  }
#pragma unroll
  for (int i = 0; i < 16; i++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[i] = max(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
    if (lane == 0) s_max[warp][i] = mx[i];
  }
  __syncthreads();
  if (threadIdx.x < 16) {   // steps 3-4 (read as DESIGN.md A3)
    int m = 0;
#pragma unroll
    for (int wv = 0; wv < kFilterWarps; wv++) m = max(m, s_max[wv][threadIdx.x]);
    int n = 0, p = 0;
    if (g.scaling && m > g.target) {
      const int x = (g.target * 128) / m;
      const int y = 31 - __clz(x);
      n = y >= 3 ? (x >> (y - 3)) : (x << (3 - y));
      p = 10 - y;
    }
    s_n[threadIdx.x] = n;
    s_p[threadIdx.x] = p;
    if (live) codes[co * 16 + threadIdx.x] = (uint8_t)(n ? ((n << 2) | (p - 4)) : 0);
  }
  __syncthreads();
  int sn[16], sp[16];
#pragma unroll
  for (int i = 0; i < 16; i++) { sn[i] = s_n[i]; sp[i] = s_p[i]; }
  for (int c0 = warp * 32; c0 < g.cin_pad; c0 += kFilterWarps * 32) {
    const int ci = c0 + lane;
    int vals[16];
    if (live && ci < g.cin) {
      int gg[3][3];
      load_filter(g, w, co, ci, gg);
      filter_tile_transform2(gg, vals);
#pragma unroll
      for (int s = 0; s < 16; s++) vals[s] = sn[s] ? rha_mul_shift(vals[s], sn[s], sp[s]) : vals[s];
    } else {
#pragma unroll
      for (int s = 0; s < 16; s++) vals[s] = 0;
    }
#pragma unroll
    for (int s = 0; s < 16; s++) {
      s_stage[warp][2 * s + 0][lane] = (int8_t)bal_hi(vals[s]);
      s_stage[warp][2 * s + 1][lane] = (int8_t)bal_lo(vals[s]);
    }
    __syncwarp();
    for (int idx = lane; idx < 32 * 2; idx += 32) {   // (piece-plane, 16-channel half)
      const int pp = idx >> 1, hf = idx & 1;
      const int4 v = *reinterpret_cast<const int4*>(&s_stage[warp][pp][hf * 16]);
      *reinterpret_cast<int4*>(wimg + w_offset(g, pp >> 1, pp & 1, co, c0 + hf * 16)) = v;
    }
    __syncwarp();
  }
}

static int g_carve_filter = kCarveFilter;

cudaError_t launch_filter_transform(const Geom& g, const int8_t* w, int8_t* wimg, uint8_t* codes, cudaStream_t st) {
  if (g.alg == 1)
    return launch_pdl_co(k_filter_transform2, dim3(g.cout_pad), dim3(kFilterWarps * 32), 0, st, g_carve_filter, g, w, wimg, codes);
  if (g.path == 0)
    return launch_pdl_co(k_filter_transform<true>, dim3(g.cout_pad), dim3(kFilterWarps * 32), 0, st, g_carve_filter, g, w, wimg, codes);
  if (g.w1)
    return launch_pdl_co(k_filter_transform<false, true>, dim3(g.cout_pad), dim3(kFilterWarps * 32), 0, st, g_carve_filter, g, w, wimg,
                      codes);
  return launch_pdl_co(k_filter_transform<false>, dim3(g.cout_pad), dim3(kFilterWarps * 32), 0, st, g_carve_filter, g, w, wimg, codes);
}

cudaError_t setup_filter_transform() {
  if (const char* c = std::getenv("WINO_CARVE_K1")) g_carve_filter = std::atoi(c);   // experiments
  return cudaSuccess;
}

}  // namespace wino
