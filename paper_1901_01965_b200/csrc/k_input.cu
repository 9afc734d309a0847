// k_input.cu -- K2: input-tile gather + D = B^T d B in exact integer
// Gaussian arithmetic, Karatsuba operand planes and
// int8 piece split, written in the pre-tiled UMMA layout (layout.cuh).
//
// Thread = (tile, pair of adjacent input channels).  A warp covers 4
// consecutive tiles (4 consecutive rows of one core matrix) x 16 channels
// (one 16-byte K half), so every 2-byte store of the warp lands in one
// contiguous 64-byte run.  Per channel only the 16 real values and the 10
// conjugate primaries are formed: d' = B^T d column by column,
// then the same combinations along each row of d'.  The two channels'
// values v0, v1 of a plane become balanced s8 pieces v = 256 hi + lo
// (lo = byte 0 of v read as s8, hi = byte 1 of v + 128: two PRMTs on v + 128)
// stored as two 16-bit pairs [hi0, hi1] and [lo0, lo1], 4 KB apart (staged
// layout; the fused layout's two-channel variant below keeps lo = v & 255 as
// u8 and hi = v >> 8).  All 92 plane-pieces of a (tile block, K step) are
// 4 KB apart, so every store is an immediate offset from one base pointer.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"
#include "ptx.cuh"

namespace wino {

constexpr int kInWarps = 8;
constexpr int kInTilesPerWarp = 4;
constexpr int kInTilesPerCta = kInWarps * kInTilesPerWarp;   // 32
constexpr int kInChPerCta = 16;

// Sign-extend byte `b` of w: PTX prmt default mode replicates the byte's msb
// for selector nibbles with bit 3 set (CUDA's __byte_perm masks that bit off).
__device__ __forceinline__ int sbyte(uint32_t w, int b) {
  const uint32_t sel = b == 0 ? 0x8880u : (b == 1 ? 0x9991u : (b == 2 ? 0xAAA2u : 0xBBB3u));
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
  return (int)r;
}

// Activation value of channel byte `ch` of a gathered pixel pair: int8, or uint8 minus the zero
// point (int9, f2).
template <bool U8>
__device__ __forceinline__ int dval(const Geom& g, uint32_t w, int ch) {
  if constexpr (U8) return (int)((w >> (8 * ch)) & 0xffu) - g.zx;
  else return sbyte(w, ch);
}

// The 46 operand-plane values of one channel from d' rows (e0, e1, e2, e5 real;
// row 3 = ra + i rb), in plane order (layout.cuh).
struct Rows {
  int e0[6], e1[6], e2[6], e5[6], ra[6], rb[6];
};

template <int RI>
__device__ __forceinline__ void real_row_planes(const int (&e)[6], int (&v)[7]) {
  const int s24 = e[2] + e[4], s13 = e[1] + e[3];
  v[0] = e[0] - e[4];          // (R[RI], 0)
  v[1] = s13 + s24;            // (R[RI], 1)
  v[2] = s24 - s13;            // (R[RI], 2)
  v[3] = e[5] - e[1];          // (R[RI], 5)
  v[4] = e[4] - e[2];          // Re (R[RI], 3)
  v[5] = e[3] - e[1];          // Im (R[RI], 3)
  v[6] = v[4] + v[5];          // Re + Im
}

__device__ __forceinline__ void st16(int8_t* p, uint32_t v) { *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; }

// Store plane `PL` for both channels: balanced s8 pieces hi = byte 1 of v + 128 and lo =
// byte 0 of v (layout.cuh), hi at the plane's K-step block, lo 4 KB after it.
template <int PL>
__device__ __forceinline__ void store_plane(int8_t* base, long long pstride, int v0, int v1) {
  int8_t* p = base + PL * pstride;
  const uint32_t w0 = (uint32_t)(v0 + 128), w1 = (uint32_t)(v1 + 128);   // byte 0 of v + 128 = lo ^ 0x80
  st16(p, __byte_perm(w0, w1, 0x0051));                                  // [hi0, hi1]
  st16(p + 4096, __byte_perm(w0, w1, 0x0040) ^ 0x8080u);                 // [lo0, lo1]
}

// Gather the zero-padded 6x6 patch of chunk tile t for channels c, c+1 and form
// d' = B^T d column by column for both channels.
template <bool U8, int KS = 0>
__device__ __forceinline__ void input_rows(const Geom& g, const int8_t* __restrict__ x, int n0, int imgs, int t, int c,
                                           Rows (&r)[2]) {
  const int tiles = imgs * g.tpi;

  // ---- gather the zero-padded 6x6 patch at origin (4ty - pad, 4tx - pad): 2 channels per pixel.
  // uint8 input (f2): out-of-map pixels and channels past Cin read the zero point, so that
  // d = u8 - zx = 0 there (padding is the real value 0, A28).
  const uint32_t zpair = U8 ? (uint32_t)(g.zx | (g.zx << 8)) : 0u;
  uint32_t w[36];
  {
    int img = 0, iy0 = -1000000, ix0 = -1000000;   // padding tiles read nothing
    if (t < tiles) {
      const int ti = fdiv(t, g.dv_tpi), rem = t - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
      img = n0 + ti;
      iy0 = 4 * ty - g.pad;
      ix0 = 4 * (rem - ty * g.tw) - g.pad;
    }
    const bool cok = c < g.cin;
    bool vx[6];
#pragma unroll
    for (int b = 0; b < 6; b++) vx[b] = cok && ix0 + b >= 0 && ix0 + b < g.w;
    if (g.layout == 1 && (g.cin & 1) == 0) {
      // NHWC, even Cin: one 16-bit load per pixel; row pointer hoisted, column offsets b*Cin
      const int8_t* p0 = x + ((long long)img * g.h * g.w + (long long)iy0 * g.w + ix0) * g.cin + c;
      const long long rstride = (long long)g.w * g.cin;
      // interior warps (every lane's patch inside the map) with c_in = 32 KS: unpredicated loads at
      // immediate column offsets b * c_in (the border test and address arithmetic were ~6 instructions per load)
      const bool inside = cok && iy0 >= 0 && iy0 + 6 <= g.h && ix0 >= 0 && ix0 + 6 <= g.w;
      if (KS > 0 && g.cin == 32 * KS && __all_sync(0xffffffffu, inside)) {
#pragma unroll
        for (int a = 0; a < 6; a++) {
          const uint16_t* rp = reinterpret_cast<const uint16_t*>(p0 + a * rstride);
#pragma unroll
          for (int b = 0; b < 6; b++) w[a * 6 + b] = (uint32_t)__ldg(rp + b * 16 * KS);
        }
      } else {
#pragma unroll
        for (int a = 0; a < 6; a++) {
          const bool vy = iy0 + a >= 0 && iy0 + a < g.h;
          const uint16_t* rp = reinterpret_cast<const uint16_t*>(p0 + a * rstride);
#pragma unroll
          for (int b = 0; b < 6; b++) w[a * 6 + b] = (vy && vx[b]) ? (uint32_t)__ldg(rp + (b * g.cin >> 1)) : zpair;
        }
      }
    } else {
      // generic path (NCHW or odd Cin): byte loads
      const long long cstep = g.layout == 1 ? 1 : (long long)g.h * g.w;
#pragma unroll
      for (int a = 0; a < 6; a++)
#pragma unroll
        for (int b = 0; b < 6; b++) {
          const int iy = iy0 + a, ix = ix0 + b;
          uint32_t v = zpair;
          if (vx[b] && iy >= 0 && iy < g.h) {
            const long long i0 = g.layout == 1 ? (((long long)img * g.h + iy) * g.w + ix) * g.cin + c
                                               : (((long long)img * g.cin + c) * g.h + iy) * g.w + ix;
            v = (uint8_t)__ldg(x + i0);
            v |= (c + 1 < g.cin) ? (uint32_t)(uint8_t)__ldg(x + i0 + cstep) << 8 : (zpair & 0xff00u);
          }
          w[a * 6 + b] = v;
        }
    }
  }

  // ---- d' = B^T d per column, for both channels
#pragma unroll
  for (int j = 0; j < 6; j++) {
#pragma unroll
    for (int ch = 0; ch < 2; ch++) {
      const int d0 = dval<U8>(g, w[0 * 6 + j], ch), d1 = dval<U8>(g, w[1 * 6 + j], ch), d2 = dval<U8>(g, w[2 * 6 + j], ch);
      const int d3 = dval<U8>(g, w[3 * 6 + j], ch), d4 = dval<U8>(g, w[4 * 6 + j], ch), d5 = dval<U8>(g, w[5 * 6 + j], ch);
      const int s24 = d2 + d4, s13 = d1 + d3;
      r[ch].e0[j] = d0 - d4;
      r[ch].e1[j] = s13 + s24;
      r[ch].e2[j] = s24 - s13;
      r[ch].ra[j] = d4 - d2;     // Re d'[3][j]
      r[ch].rb[j] = d3 - d1;     // Im d'[3][j]
      r[ch].e5[j] = d5 - d1;
    }
  }
}

// 16-channel slices per CTA (4 when c_in_pad is a multiple of 64, else 2; WINO_K2_SPC overrides)
inline int k2_slices_per_cta(int cin_pad) {
  static const int env = [] { const char* e = std::getenv("WINO_K2_SPC"); return e ? std::atoi(e) : 4; }();
  return (env == 4 && cin_pad % 64 == 0) ? 4 : (env >= 2 ? 2 : 1);
}

template <bool U8, int KS>   // KS: g.ksteps at compile time (0 = runtime), as in K2F
__global__ void __launch_bounds__(kInWarps * 32) k_input_transform(Geom g, const int8_t* __restrict__ x, int n0,
                                                                   int imgs, int8_t* __restrict__ vimg, int spc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = lane >> 3, cp = lane & 7;                      // tile within warp, channel pair
  // spc 16-channel slices per CTA (warp w: tile group w / spc, slice w % spc): the warps reading a pixel's
  // channel bytes share the CTA's L1 (k_input4.cu)
  const int t = blockIdx.x * (kInTilesPerCta / spc) + (warp / spc) * kInTilesPerWarp + tl;   // chunk tile
  const int c = (blockIdx.y * spc + warp % spc) * kInChPerCta + 2 * cp;   // first channel of the pair
  pdl_trigger();
  pdl_wait();   // x may come from the previous kernel (layer stacks); V may still be read by the previous GEMM
  Rows r[2];
  input_rows<U8, KS>(g, x, n0, imgs, t, c, r);

  // ---- D = d' B along rows; store every plane as soon as it is formed
  const long long tb = t / kMBlock;
  const int row = t % kMBlock;
  const int k = c;   // channel index inside cin_pad
  // plane p, piece q of this (tile, channel) at base + p * pstride + q * 4 KB (v_offset, layout.cuh)
  const long long pstride = (long long)(KS ? KS : g.ksteps) * 2 * kVBlockBytes;
  int8_t* base = vimg + tb * kPlanes * pstride + (long long)(k >> 5) * 2 * kVBlockBytes +
                 tiled_offset(row, k & 31, kMBlock);
  {
    int v0[7], v1[7];
    real_row_planes<0>(r[0].e0, v0); real_row_planes<0>(r[1].e0, v1);
    store_plane<0>(base, pstride, v0[0], v1[0]); store_plane<1>(base, pstride, v0[1], v1[1]);
    store_plane<2>(base, pstride, v0[2], v1[2]); store_plane<3>(base, pstride, v0[3], v1[3]);
    store_plane<16>(base, pstride, v0[4], v1[4]); store_plane<17>(base, pstride, v0[5], v1[5]); store_plane<18>(base, pstride, v0[6], v1[6]);
    real_row_planes<1>(r[0].e1, v0); real_row_planes<1>(r[1].e1, v1);
    store_plane<4>(base, pstride, v0[0], v1[0]); store_plane<5>(base, pstride, v0[1], v1[1]);
    store_plane<6>(base, pstride, v0[2], v1[2]); store_plane<7>(base, pstride, v0[3], v1[3]);
    store_plane<19>(base, pstride, v0[4], v1[4]); store_plane<20>(base, pstride, v0[5], v1[5]); store_plane<21>(base, pstride, v0[6], v1[6]);
    real_row_planes<2>(r[0].e2, v0); real_row_planes<2>(r[1].e2, v1);
    store_plane<8>(base, pstride, v0[0], v1[0]); store_plane<9>(base, pstride, v0[1], v1[1]);
    store_plane<10>(base, pstride, v0[2], v1[2]); store_plane<11>(base, pstride, v0[3], v1[3]);
    store_plane<22>(base, pstride, v0[4], v1[4]); store_plane<23>(base, pstride, v0[5], v1[5]); store_plane<24>(base, pstride, v0[6], v1[6]);
    real_row_planes<3>(r[0].e5, v0); real_row_planes<3>(r[1].e5, v1);
    store_plane<12>(base, pstride, v0[0], v1[0]); store_plane<13>(base, pstride, v0[1], v1[1]);
    store_plane<14>(base, pstride, v0[2], v1[2]); store_plane<15>(base, pstride, v0[3], v1[3]);
    store_plane<25>(base, pstride, v0[4], v1[4]); store_plane<26>(base, pstride, v0[5], v1[5]); store_plane<27>(base, pstride, v0[6], v1[6]);
  }
  // complex row 3 = a + i b: columns 0, 1, 2, 5 -> primaries 4..7; (3,3) -> 8; (3,4) -> 9
  {
    int re[2][4], im[2][4], q[2][4];
#pragma unroll
    for (int ch = 0; ch < 2; ch++) {
      const int* a = r[ch].ra;
      const int* b = r[ch].rb;
      const int as24 = a[2] + a[4], as13 = a[1] + a[3], bs24 = b[2] + b[4], bs13 = b[1] + b[3];
      re[ch][0] = a[0] - a[4]; re[ch][1] = as13 + as24; re[ch][2] = as24 - as13; re[ch][3] = a[5] - a[1];
      im[ch][0] = b[0] - b[4]; im[ch][1] = bs13 + bs24; im[ch][2] = bs24 - bs13; im[ch][3] = b[5] - b[1];
      // (3,3) = (e4 - e2) + i (e3 - e1),  (3,4) = (e4 - e2) - i (e3 - e1), e = a + i b
      q[ch][0] = a[4] - a[2] - b[3] + b[1];
      q[ch][1] = b[4] - b[2] + a[3] - a[1];
      q[ch][2] = a[4] - a[2] + b[3] - b[1];
      q[ch][3] = b[4] - b[2] - a[3] + a[1];
    }
    store_plane<28>(base, pstride, re[0][0], re[1][0]); store_plane<29>(base, pstride, im[0][0], im[1][0]);
    store_plane<30>(base, pstride, re[0][0] + im[0][0], re[1][0] + im[1][0]);
    store_plane<31>(base, pstride, re[0][1], re[1][1]); store_plane<32>(base, pstride, im[0][1], im[1][1]);
    store_plane<33>(base, pstride, re[0][1] + im[0][1], re[1][1] + im[1][1]);
    store_plane<34>(base, pstride, re[0][2], re[1][2]); store_plane<35>(base, pstride, im[0][2], im[1][2]);
    store_plane<36>(base, pstride, re[0][2] + im[0][2], re[1][2] + im[1][2]);
    store_plane<37>(base, pstride, re[0][3], re[1][3]); store_plane<38>(base, pstride, im[0][3], im[1][3]);
    store_plane<39>(base, pstride, re[0][3] + im[0][3], re[1][3] + im[1][3]);
    store_plane<40>(base, pstride, q[0][0], q[1][0]); store_plane<41>(base, pstride, q[0][1], q[1][1]);
    store_plane<42>(base, pstride, q[0][0] + q[0][1], q[1][0] + q[1][1]);
    store_plane<43>(base, pstride, q[0][2], q[1][2]); store_plane<44>(base, pstride, q[0][3], q[1][3]);
    store_plane<45>(base, pstride, q[0][2] + q[0][3], q[1][2] + q[1][3]);
  }
}

// ---- fused-path V image (layout.cuh "fused-path operand layouts"): per group, pieces hi = v >> 8 (s8,
// byte 1 of v) and lo = v & 255 (u8, byte 0 of v; the fused GEMM reads lo as an unsigned A operand),
// stored for both channels.  (NCHW and uint8 input; NHWC int8 runs k_input4.cu.)
__device__ __forceinline__ void st_fused(int8_t* p_hi, int v0, int v1) {
  st16(p_hi, __byte_perm((uint32_t)v0, (uint32_t)v1, 0x0051));          // [hi0, hi1]
  st16(p_hi + 4096, __byte_perm((uint32_t)v0, (uint32_t)v1, 0x0040));   // [lo0, lo1]
}

// KS: g.ksteps as a compile-time constant (1, 2, 4, 8, 16; 0 = runtime), so that every piece's store
// offset from the thread's base pointer is an immediate
template <bool U8, int KS>
__global__ void __launch_bounds__(kInWarps * 32) k_input_transform_f(Geom g, const int8_t* __restrict__ x, int n0,
                                                                     int imgs, int8_t* __restrict__ vimg, int spc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = lane >> 3, cp = lane & 7;
  // spc 16-channel slices per CTA (warp w: tile group w / spc, slice w % spc): the warps reading a pixel's
  // channel bytes share the CTA's L1 (k_input4.cu)
  const int t = blockIdx.x * (kInTilesPerCta / spc) + (warp / spc) * kInTilesPerWarp + tl;   // chunk tile
  const int c = (blockIdx.y * spc + warp % spc) * kInChPerCta + 2 * cp;   // first channel of the pair
  pdl_trigger();
  pdl_wait();
  Rows r[2];
  input_rows<U8, KS>(g, x, n0, imgs, t, c, r);

  const long long tb = t / kMBlock;
  const int row = t % kMBlock;
  const long long kst = (long long)(KS ? KS : g.ksteps) * kVBlockBytes;
  int8_t* base = vimg + tb * kVPiecesF * kst + tiled_offset(row, c & 31, kMBlock);
  const int ks = c >> 5;
  int8_t* base2 = base + (long long)(ks * 2) * kVBlockBytes;   // groups of 2 pieces (real)
  int8_t* base4 = base + (long long)(ks * 4) * kVBlockBytes;   // groups of 4 pieces (complex)
  // first (hi) piece of group gi for this K step
  auto gp = [&](int gi) { return (fg_pieces(gi) == 2 ? base2 : base4) + fg_vprefix(gi) * kst; };
  auto real_row = [&](auto ric, const int (&e0)[6], const int (&e1)[6]) {
    constexpr int ri = decltype(ric)::value;
    int v0[7], v1[7];
    real_row_planes<ri>(e0, v0);
    real_row_planes<ri>(e1, v1);
#pragma unroll
    for (int s = 0; s < 4; s++) st_fused(gp(fg_of_real(ri * 4 + s)), v0[s], v1[s]);
    int8_t* pc = gp(fg_of_primary(ri));
    st_fused(pc, v0[4], v1[4]);                      // Re (R[ri], 3)
    st_fused(pc + 2 * kVBlockBytes, v0[5], v1[5]);   // Im
  };
  real_row(std::integral_constant<int, 0>{}, r[0].e0, r[1].e0);
  real_row(std::integral_constant<int, 1>{}, r[0].e1, r[1].e1);
  real_row(std::integral_constant<int, 2>{}, r[0].e2, r[1].e2);
  real_row(std::integral_constant<int, 3>{}, r[0].e5, r[1].e5);
  // complex row 3 = a + i b: (3,0) (3,1) (3,2) (3,5) -> primaries 4..7, (3,3) -> 8, (3,4) -> 9
  int re[2][4], im[2][4], q[2][4];
#pragma unroll
  for (int ch = 0; ch < 2; ch++) {
    const int* a = r[ch].ra;
    const int* b = r[ch].rb;
    const int as24 = a[2] + a[4], as13 = a[1] + a[3], bs24 = b[2] + b[4], bs13 = b[1] + b[3];
    re[ch][0] = a[0] - a[4]; re[ch][1] = as13 + as24; re[ch][2] = as24 - as13; re[ch][3] = a[5] - a[1];
    im[ch][0] = b[0] - b[4]; im[ch][1] = bs13 + bs24; im[ch][2] = bs24 - bs13; im[ch][3] = b[5] - b[1];
    q[ch][0] = a[4] - a[2] - b[3] + b[1];
    q[ch][1] = b[4] - b[2] + a[3] - a[1];
    q[ch][2] = a[4] - a[2] + b[3] - b[1];
    q[ch][3] = b[4] - b[2] - a[3] + a[1];
  }
#pragma unroll
  for (int j = 0; j < 4; j++) {
    int8_t* pc = gp(fg_of_primary(4 + j));
    st_fused(pc, re[0][j], re[1][j]);
    st_fused(pc + 2 * kVBlockBytes, im[0][j], im[1][j]);
  }
  {
    int8_t* pc = gp(fg_of_primary(8));
    st_fused(pc, q[0][0], q[1][0]);
    st_fused(pc + 2 * kVBlockBytes, q[0][1], q[1][1]);
    pc = gp(fg_of_primary(9));
    st_fused(pc, q[0][2], q[1][2]);
    st_fused(pc + 2 * kVBlockBytes, q[0][3], q[1][3]);
  }
}

cudaError_t launch_input_transform_f(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st) {
  const long long tiles = (long long)imgs * g.tpi;
  const long long tiles_pad = (tiles + kMBlock - 1) / kMBlock * kMBlock;
  const int spc = k2_slices_per_cta(g.cin_pad);
  dim3 grid((unsigned)(tiles_pad / (kInTilesPerCta / spc)), g.cin_pad / (kInChPerCta * spc));
#define WINO_K2F(U, K) launch_pdl_co(k_input_transform_f<U, K>, grid, dim3(kInWarps * 32), 0, st, kCarveL1, g, x, n0, imgs, vimg, spc)
#define WINO_K2F_KS(U)                                                                                          \
  switch (g.ksteps) {                                                                                           \
    case 1: return WINO_K2F(U, 1);                                                                              \
    case 2: return WINO_K2F(U, 2);                                                                              \
    case 4: return WINO_K2F(U, 4);                                                                              \
    case 8: return WINO_K2F(U, 8);                                                                              \
    case 16: return WINO_K2F(U, 16);                                                                            \
    default: return WINO_K2F(U, 0);                                                                             \
  }
  if (g.in_u8) { WINO_K2F_KS(true) }   // uint8 + zero point (f2, A28)
  WINO_K2F_KS(false)
#undef WINO_K2F_KS
#undef WINO_K2F
}

// ---- rational F(2x2,3x3): 4x4 patch at (2ty - pad, 2tx - pad), D = B^T d B with the
// F(2,3) matrix B^T = [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]] (A25), 16 real planes
// (position i*4 + j), balanced pieces, staged V layout (plane stride = g.planes = 16).
template <bool U8, int KS>   // uint8 + zero point (f2, A28): out-of-map pixels read the zero point (d = 0)
__global__ void __launch_bounds__(kInWarps * 32) k_input_transform2(Geom g, const int8_t* __restrict__ x, int n0,
                                                                    int imgs, int8_t* __restrict__ vimg, int spc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tl = lane >> 3, cp = lane & 7;
  // spc 16-channel slices per CTA (warp w: tile group w / spc, slice w % spc): the warps reading a pixel's
  // channel bytes share the CTA's L1 (k_input4.cu)
  const int t = blockIdx.x * (kInTilesPerCta / spc) + (warp / spc) * kInTilesPerWarp + tl;   // chunk tile
  const int c = (blockIdx.y * spc + warp % spc) * kInChPerCta + 2 * cp;   // first channel of the pair
  pdl_trigger();
  pdl_wait();
  uint32_t w[16];   // 2 channels per pixel
  const uint32_t zpair = U8 ? (uint32_t)(g.zx | (g.zx << 8)) : 0u;
  {
    int img = 0, iy0 = -1000000, ix0 = -1000000;
    if (t < imgs * g.tpi) {
      const int ti = fdiv(t, g.dv_tpi), rem = t - ti * g.tpi, ty = fdiv(rem, g.dv_tw);
      img = n0 + ti;
      iy0 = 2 * ty - g.pad;
      ix0 = 2 * (rem - ty * g.tw) - g.pad;
    }
    const bool cok = c < g.cin;
    bool vx[4];
#pragma unroll
    for (int b = 0; b < 4; b++) vx[b] = cok && ix0 + b >= 0 && ix0 + b < g.w;
    if (g.layout == 1 && (g.cin & 1) == 0) {
      // NHWC, even Cin: one 16-bit load per pixel; row pointer hoisted, column offsets b*Cin (as in K2)
      const int8_t* p0 = x + ((long long)img * g.h * g.w + (long long)iy0 * g.w + ix0) * g.cin + c;
      const long long rstride = (long long)g.w * g.cin;
      const bool inside = cok && iy0 >= 0 && iy0 + 4 <= g.h && ix0 >= 0 && ix0 + 4 <= g.w;
      if (KS > 0 && g.cin == 32 * KS && __all_sync(0xffffffffu, inside)) {   // interior warp: as in K2F
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const uint16_t* rp = reinterpret_cast<const uint16_t*>(p0 + a * rstride);
#pragma unroll
          for (int b = 0; b < 4; b++) w[a * 4 + b] = (uint32_t)__ldg(rp + b * 16 * KS);
        }
      } else {
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const bool vy = iy0 + a >= 0 && iy0 + a < g.h;
          const uint16_t* rp = reinterpret_cast<const uint16_t*>(p0 + a * rstride);
#pragma unroll
          for (int b = 0; b < 4; b++) w[a * 4 + b] = (vy && vx[b]) ? (uint32_t)__ldg(rp + (b * g.cin >> 1)) : zpair;
        }
      }
    } else {
      const long long cstep = g.layout == 1 ? 1 : (long long)g.h * g.w;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
          const int iy = iy0 + a, ix = ix0 + b;
          uint32_t v = zpair;
          if (vx[b] && iy >= 0 && iy < g.h) {
            const long long i0 = g.layout == 1 ? (((long long)img * g.h + iy) * g.w + ix) * g.cin + c
                                               : (((long long)img * g.cin + c) * g.h + iy) * g.w + ix;
            v = (uint8_t)__ldg(x + i0);
            v |= (c + 1 < g.cin) ? (uint32_t)(uint8_t)__ldg(x + i0 + cstep) << 8 : (zpair & 0xff00u);
          }
          w[a * 4 + b] = v;
        }
    }
  }
  const long long pstride = (long long)(KS ? KS : g.ksteps) * 2 * kVBlockBytes;
  int8_t* base = vimg + (t / kMBlock) * g.planes * pstride + (long long)(c >> 5) * 2 * kVBlockBytes +
                 tiled_offset(t % kMBlock, c & 31, kMBlock);
  int Dv[2][16];
#pragma unroll
  for (int ch = 0; ch < 2; ch++) {
    int r[4][4];   // d' = B^T d, column by column
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int d0 = dval<U8>(g, w[0 * 4 + j], ch), d1 = dval<U8>(g, w[1 * 4 + j], ch),
                d2 = dval<U8>(g, w[2 * 4 + j], ch), d3 = dval<U8>(g, w[3 * 4 + j], ch);
      r[0][j] = d0 - d2; r[1][j] = d1 + d2; r[2][j] = d2 - d1; r[3][j] = d1 - d3;
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {   // D = d' B, row by row
      Dv[ch][i * 4 + 0] = r[i][0] - r[i][2];
      Dv[ch][i * 4 + 1] = r[i][1] + r[i][2];
      Dv[ch][i * 4 + 2] = r[i][2] - r[i][1];
      Dv[ch][i * 4 + 3] = r[i][1] - r[i][3];
    }
  }
#pragma unroll
  for (int pos = 0; pos < 16; pos++) {
    int8_t* p = base + pos * pstride;
    st16(p, __byte_perm((uint32_t)(Dv[0][pos] + 128), (uint32_t)(Dv[1][pos] + 128), 0x0051));   // [hi0, hi1]
    st16(p + kVBlockBytes, __byte_perm((uint32_t)Dv[0][pos], (uint32_t)Dv[1][pos], 0x0040));      // [lo0, lo1]
  }
}

cudaError_t launch_input_transform(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st) {
  const long long tiles = (long long)imgs * g.tpi;
  const long long tiles_pad = (tiles + kMBlock - 1) / kMBlock * kMBlock;
  const int spc = k2_slices_per_cta(g.cin_pad);
  dim3 grid((unsigned)(tiles_pad / (kInTilesPerCta / spc)), g.cin_pad / (kInChPerCta * spc));
#define WINO_K22(U, K) launch_pdl_co(k_input_transform2<U, K>, grid, dim3(kInWarps * 32), 0, st, kCarveL1, g, x, n0, imgs, vimg, spc)
#define WINO_K22_KS(U)                                                                                          \
  switch (g.ksteps) {                                                                                           \
    case 1: return WINO_K22(U, 1);                                                                              \
    case 2: return WINO_K22(U, 2);                                                                              \
    case 4: return WINO_K22(U, 4);                                                                              \
    case 8: return WINO_K22(U, 8);                                                                              \
    case 16: return WINO_K22(U, 16);                                                                            \
    default: return WINO_K22(U, 0);                                                                             \
  }
  if (g.alg == 1 && g.in_u8) { WINO_K22_KS(true) }
  if (g.alg == 1) { WINO_K22_KS(false) }
#undef WINO_K22_KS
#undef WINO_K22
#define WINO_K2S(U, K) launch_pdl_co(k_input_transform<U, K>, grid, dim3(kInWarps * 32), 0, st, kCarveL1, g, x, n0, imgs, vimg, spc)
#define WINO_K2S_KS(U)                                                                                          \
  switch (g.ksteps) {                                                                                           \
    case 1: return WINO_K2S(U, 1);                                                                              \
    case 2: return WINO_K2S(U, 2);                                                                              \
    case 4: return WINO_K2S(U, 4);                                                                              \
    case 8: return WINO_K2S(U, 8);                                                                              \
    case 16: return WINO_K2S(U, 16);                                                                            \
    default: return WINO_K2S(U, 0);                                                                             \
  }
  if (g.in_u8) { WINO_K2S_KS(true) }
  WINO_K2S_KS(false)
#undef WINO_K2S_KS
#undef WINO_K2S
}

cudaError_t setup_input_transform() { return cudaSuccess; }

}  // namespace wino
