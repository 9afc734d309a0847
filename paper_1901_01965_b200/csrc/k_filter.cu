// k_filter.cu -- K1: offline filter transform W = G_int g G_int^T, the
// paper's per-(OFM, position) integer scale factors, downscale, Karatsuba
// operand planes and int8 piece split.
//
// One CTA per output channel (the unit the paper scales: "applied to
// the filters used to generate one output feature map").  Each thread
// transforms a strided subset of the input channels into shared memory
// (36 int16 per channel: 16 real values + 10 complex primaries as re,im),
// the CTA reduces the per-position max magnitude across channels, threads
// 0..25 derive the 6-bit codes, and every thread then writes its channels'
// scaled, split operand bytes into the pre-tiled W image.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

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

__global__ void __launch_bounds__(256) k_filter_transform(Geom g, const int8_t* __restrict__ w,
                                                          int8_t* __restrict__ wimg, uint8_t* __restrict__ codes) {
  extern __shared__ int16_t s_w[];      // [cin][36]
  __shared__ int s_max[8][26];
  __shared__ int s_n[26], s_p[26];
  const int co = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool live = co < g.cout;

  int mx[26];
#pragma unroll
  for (int i = 0; i < 26; i++) mx[i] = 0;
  if (live) {
    for (int ci = tid; ci < g.cin; ci += blockDim.x) {
      int gg[3][3];
#pragma unroll
      for (int u = 0; u < 3; u++)
#pragma unroll
        for (int v = 0; v < 3; v++)
          gg[u][v] = g.layout == 0 ? w[((long long)co * g.cin + ci) * 9 + u * 3 + v]
                                   : w[((long long)co * 9 + u * 3 + v) * g.cin + ci];
      int t[36];
      filter_tile_transform(gg, t);
#pragma unroll
      for (int i = 0; i < 36; i++) s_w[ci * 36 + i] = (int16_t)t[i];
#pragma unroll
      for (int s = 0; s < 16; s++) mx[s] = max(mx[s], abs(t[s]));
#pragma unroll
      for (int k = 0; k < 10; k++) mx[16 + k] = max(mx[16 + k], max(abs(t[16 + 2 * k]), abs(t[17 + 2 * k])));
    }
  }
  // max over input channels per position
#pragma unroll
  for (int i = 0; i < 26; i++) {
    int v = mx[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_max[warp][i] = v;
  }
  __syncthreads();
  if (tid < 26) {
    int m = 0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); wv++) m = max(m, s_max[wv][tid]);
    int n = 0, p = 0;
    if (g.scaling && m > g.target) {
      // P:322-329 read per DESIGN.md A3: x = floor(255*128/max), y = floor(log2 x),
      // n = x >> (y - 3) (4-bit, in [8, 15]), p = 10 - y (in [4, 7]).
      int x = (g.target * 128) / m;
      int y = 31 - __clz(x);
      n = y >= 3 ? (x >> (y - 3)) : (x << (3 - y));
      p = 10 - y;
    }
    s_n[tid] = n;
    s_p[tid] = p;
    if (live) {
      int code = n ? ((n << 2) | (p - 4)) : 0;   // 6-bit code, 0 = unscaled
      if (tid < 16) {
        codes[co * 36 + real_pos(tid)] = (uint8_t)code;
      } else {
        codes[co * 36 + cpx_pos(tid - 16)] = (uint8_t)code;
        codes[co * 36 + cpx_mirror_pos(tid - 16)] = (uint8_t)code;   // mirrors share the factor
      }
    }
  }
  __syncthreads();

  // Scaled operand planes, split into int8 pieces, into the pre-tiled image.
  const long long pp_stride = (long long)g.cout_pad * g.cin_pad;
  const long long base0 = w_offset(g, 0, co, 0);   // pp = 0 offset of (co, k = 0)
  for (int ci = tid; ci < g.cin_pad; ci += blockDim.x) {
    const long long off = base0 + tiled_offset(co % g.nblk, ci, g.nblk) - tiled_offset(co % g.nblk, 0, g.nblk);
    int vals[46];
    if (live && ci < g.cin) {
      int sv[36];
#pragma unroll
      for (int i = 0; i < 36; i++) sv[i] = s_w[ci * 36 + i];
#pragma unroll
      for (int s = 0; s < 16; s++) {
        int n = s_n[s];
        vals[s] = n ? rha_mul_shift(sv[s], n, s_p[s]) : sv[s];        // W' = rha(W n / 2^p)
      }
#pragma unroll
      for (int k = 0; k < 10; k++) {
        int n = s_n[16 + k], p = s_p[16 + k];
        int re = n ? rha_mul_shift(sv[16 + 2 * k], n, p) : sv[16 + 2 * k];
        int im = n ? rha_mul_shift(sv[17 + 2 * k], n, p) : sv[17 + 2 * k];
        vals[16 + 3 * k + 0] = re;          // Karatsuba operands
        vals[16 + 3 * k + 1] = im;
        vals[16 + 3 * k + 2] = re + im;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 46; i++) vals[i] = 0;
    }
#pragma unroll
    for (int pl = 0; pl < 46; pl++) {
      int v = vals[pl];
      wimg[off + (2 * pl + 0) * pp_stride] = (int8_t)(v >> 8);            // hi, s8
      wimg[off + (2 * pl + 1) * pp_stride] = (int8_t)(uint8_t)(v & 255);  // lo, u8
    }
  }
}

cudaError_t launch_filter_transform(const Geom& g, const int8_t* w, int8_t* wimg, uint8_t* codes, cudaStream_t st) {
  size_t smem = (size_t)g.cin * 36 * sizeof(int16_t);
  k_filter_transform<<<g.cout_pad, 256, smem, st>>>(g, w, wimg, codes);
  return cudaGetLastError();
}

cudaError_t setup_filter_transform() {
  return cudaFuncSetAttribute(k_filter_transform, cudaFuncAttributeMaxDynamicSharedMemorySize, 896 * 36 * 2);
}

}  // namespace wino
