// k_input.cu -- K2: input-tile gather + D = B^T d B in exact integer
// Gaussian arithmetic, Karatsuba operand planes and
// int8 piece split, written in the pre-tiled UMMA layout (layout.cuh).
//
// CTA = 256 threads = 16 tiles x 16 input channels (one 16-byte K half of a
// core-matrix row).  Phase 1 stages the 16 overlapping 6x6 patches in shared
// memory (one 16-byte vector per pixel for NHWC with Cin % 16 == 0),
// phase 2 transforms one (tile, channel) per thread -- only the 16 real
// values and the 10 conjugate primaries are formed -- and stages
// the 92 output bytes, phase 3 writes whole 16-byte core-matrix rows.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace wino {

constexpr int kTilesPerCta = 16;
constexpr int kChPerCta = 16;

__global__ void __launch_bounds__(256) k_input_transform(Geom g, const int8_t* __restrict__ x, int n0, int imgs,
                                                         int8_t* __restrict__ vimg) {
  __shared__ __align__(16) int8_t s_patch[kTilesPerCta][36][kChPerCta];
  __shared__ __align__(16) int8_t s_out[2 * kPlanes][kTilesPerCta][kChPerCta];
  const int tid = threadIdx.x;
  const long long t0 = (long long)blockIdx.x * kTilesPerCta;
  const int ci0 = blockIdx.y * kChPerCta;
  const long long tiles = (long long)imgs * g.tpi;

  // ---- phase 1: gather the zero-padded 6x6 patches (origin (4ty - pad, 4tx - pad))
  const bool vec = (g.layout == 1) && (g.cin % 16 == 0);
  if (vec) {
    for (int idx = tid; idx < kTilesPerCta * 36; idx += blockDim.x) {
      int tl = idx / 36, pix = idx % 36;
      long long t = t0 + tl;
      int4 v = make_int4(0, 0, 0, 0);
      if (t < tiles) {
        int img = n0 + (int)(t / g.tpi), rem = (int)(t % g.tpi);
        int iy = 4 * (rem / g.tw) - g.pad + pix / 6, ix = 4 * (rem % g.tw) - g.pad + pix % 6;
        if (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w)
          v = __ldg(reinterpret_cast<const int4*>(x + (((long long)img * g.h + iy) * g.w + ix) * g.cin + ci0));
      }
      *reinterpret_cast<int4*>(&s_patch[tl][pix][0]) = v;
    }
  } else {
    for (int idx = tid; idx < kTilesPerCta * 36 * kChPerCta; idx += blockDim.x) {
      int tl = idx / (36 * kChPerCta), rest = idx % (36 * kChPerCta);
      int ch, pix;
      if (g.layout == 0) { ch = rest / 36; pix = rest % 36; }   // NCHW: spatial fastest
      else { pix = rest / kChPerCta; ch = rest % kChPerCta; }
      long long t = t0 + tl;
      int c = ci0 + ch;
      int8_t v = 0;
      if (t < tiles && c < g.cin) {
        int img = n0 + (int)(t / g.tpi), rem = (int)(t % g.tpi);
        int iy = 4 * (rem / g.tw) - g.pad + pix / 6, ix = 4 * (rem % g.tw) - g.pad + pix % 6;
        if (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w)
          v = g.layout == 0 ? x[(((long long)img * g.cin + c) * g.h + iy) * g.w + ix]
                            : x[(((long long)img * g.h + iy) * g.w + ix) * g.cin + c];
      }
      s_patch[tl][pix][ch] = v;
    }
  }
  __syncthreads();

  // ---- phase 2: one (tile, channel) per thread
  {
    const int tl = tid >> 4, ch = tid & 15;
    int d[6][6];
#pragma unroll
    for (int a = 0; a < 6; a++)
#pragma unroll
      for (int b = 0; b < 6; b++) d[a][b] = s_patch[tl][a * 6 + b][ch];
    // d' = B^T d, row formulas of P:184-189 (row 4 = conj(row 3) is not formed)
    int e0[6], e1[6], e2[6], e5[6], ra[6], rb[6];
#pragma unroll
    for (int j = 0; j < 6; j++) {
      int s24 = d[2][j] + d[4][j], s13 = d[1][j] + d[3][j];
      e0[j] = d[0][j] - d[4][j];
      e1[j] = s13 + s24;
      e2[j] = s24 - s13;
      ra[j] = d[4][j] - d[2][j];     // Re d'[3][j]
      rb[j] = d[3][j] - d[1][j];     // Im d'[3][j]
      e5[j] = d[5][j] - d[1][j];
    }
    int v[46];
    // D = d' B: the same combinations along each row; real rows first
    const int* rows[4] = {e0, e1, e2, e5};
#pragma unroll
    for (int ri = 0; ri < 4; ri++) {
      const int* e = rows[ri];
      int s24 = e[2] + e[4], s13 = e[1] + e[3];
      v[ri * 4 + 0] = e[0] - e[4];
      v[ri * 4 + 1] = s13 + s24;
      v[ri * 4 + 2] = s24 - s13;
      v[ri * 4 + 3] = e[5] - e[1];
      int re = e[4] - e[2], im = e[3] - e[1];        // primary k = ri : (R[ri], 3)
      v[16 + 3 * ri + 0] = re;
      v[16 + 3 * ri + 1] = im;
      v[16 + 3 * ri + 2] = re + im;
    }
    // complex row 3 (a + i b): columns 0, 1, 2, 5 -> primaries k = 4..7
    {
      int as24 = ra[2] + ra[4], as13 = ra[1] + ra[3], bs24 = rb[2] + rb[4], bs13 = rb[1] + rb[3];
      int re[4] = {ra[0] - ra[4], as13 + as24, as24 - as13, ra[5] - ra[1]};
      int im[4] = {rb[0] - rb[4], bs13 + bs24, bs24 - bs13, rb[5] - rb[1]};
#pragma unroll
      for (int c = 0; c < 4; c++) {
        v[16 + 3 * (4 + c) + 0] = re[c];
        v[16 + 3 * (4 + c) + 1] = im[c];
        v[16 + 3 * (4 + c) + 2] = re[c] + im[c];
      }
      // (3,3) = (e4 - e2) + i (e3 - e1),  (3,4) = (e4 - e2) - i (e3 - e1), e = a + i b
      int r33 = ra[4] - ra[2] - rb[3] + rb[1], i33 = rb[4] - rb[2] + ra[3] - ra[1];
      int r34 = ra[4] - ra[2] + rb[3] - rb[1], i34 = rb[4] - rb[2] - ra[3] + ra[1];
      v[16 + 3 * 8 + 0] = r33; v[16 + 3 * 8 + 1] = i33; v[16 + 3 * 8 + 2] = r33 + i33;
      v[16 + 3 * 9 + 0] = r34; v[16 + 3 * 9 + 1] = i34; v[16 + 3 * 9 + 2] = r34 + i34;
    }
#pragma unroll
    for (int pl = 0; pl < kPlanes; pl++) {
      s_out[2 * pl + 0][tl][ch] = (int8_t)(v[pl] >> 8);             // hi, s8
      s_out[2 * pl + 1][tl][ch] = (int8_t)(uint8_t)(v[pl] & 255);   // lo, u8
    }
  }
  __syncthreads();

  // ---- phase 3: 16-byte rows of the pre-tiled V image
  for (int idx = tid; idx < 2 * kPlanes * kTilesPerCta; idx += blockDim.x) {
    int pp = idx / kTilesPerCta, tl = idx % kTilesPerCta;
    int4 val = *reinterpret_cast<const int4*>(&s_out[pp][tl][0]);
    *reinterpret_cast<int4*>(vimg + v_offset(g, pp, t0 + tl, ci0)) = val;
  }
}

cudaError_t launch_input_transform(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st) {
  long long tiles = (long long)imgs * g.tpi;
  long long tiles_pad = (tiles + kMBlock - 1) / kMBlock * kMBlock;
  dim3 grid((unsigned)(tiles_pad / kTilesPerCta), g.cin_pad / kChPerCta);
  k_input_transform<<<grid, 256, 0, st>>>(g, x, n0, imgs, vimg);
  return cudaGetLastError();
}

cudaError_t setup_input_transform() { return cudaSuccess; }

}  // namespace wino
