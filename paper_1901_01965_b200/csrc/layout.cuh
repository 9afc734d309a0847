// layout.cuh -- geometry, plane numbering and HBM operand layouts of the
// CUDA path.  (The CPU oracle has its own, independent definitions.)
//
// Winograd-domain positions: the 6x6 grid has 16 always-real
// positions R x R, R = {0,1,2,5}, and 10 conjugate pairs whose primaries are
//   (0,3) (1,3) (2,3) (5,3) (3,0) (3,1) (3,2) (3,5) (3,3) (3,4)
// mirrored (swap 3<->4 in each index in {3,4}) to
//   (0,4) (1,4) (2,4) (5,4) (4,0) (4,1) (4,2) (4,5) (4,4) (4,3).
// GEMM planes (46 = 16 + 10 x 3):
//   plane s       (s < 16)  real position (R[s/4], R[s%4])
//   plane 16+3k+0           Re of primary k   (Karatsuba P0 = Re V * Re W)
//   plane 16+3k+1           Im of primary k   (P1 = Im V * Im W)
//   plane 16+3k+2           Re + Im           (P2 = (Re V + Im V)(Re W + Im W))
// Every operand value v (|v| <= 2048) is split into two BALANCED s8 pieces
//   lo = ((v + 128) & 255) - 128 (the low byte of v),  hi = (v - lo) / 256 = (v + 128) >> 8
// so v = 256 hi + lo, both pieces s8 (hi in [-8, 8]), and a plane product is
//   V W = 65536 hh + 256 (hl + lh) + ll     (exact mod 2^32).
//
// Operand images are stored pre-tiled in the UMMA canonical K-major
// no-swizzle layout so one 1-D bulk copy moves a whole stage:
//   block of R rows and K = 32 bytes (one K step): byte (row r, k) at
//     (r / 8) * 256  +  (k / 16) * 128  +  (r % 8) * 16  +  k % 16
//   (core matrix = 8 rows x 16 B; LBO = 128, SBO = 256).
//   V image: [tile_block][plane][K step][piece hi, lo][128 rows x 32 B] -- a
//            plane's K steps are contiguous (one bulk copy per stage)
//   W image: [plane][cout_block][K step][2 n_block rows x 32 B], rows
//            [W hi of the n_block couts | W lo]: the B operand of one UMMA
//            A_piece . [W hi | W lo] (N = 2 n_block) whose two column halves
//            land at scales 2^(8+8a) and 2^(8a) (a = 1 for the hi piece of V)
//   M      : [slot 36][tile_block][cout_block][128 rows][n_block] int32 -- GEMM
//            results after the Karatsuba recombination and the reverse scaling
//            (M'', read by K4): slot s < 16 real position s, 16+k = Re and 26+k = Im of
//            complex primary k; within a 128 x n_block tile, element
//            (r, c) sits at r * n_block + ((c / 4) ^ (r & swz)) * 4 + c % 4 with
//            swz = min(n_block / 4, 8) - 1 (16-byte chunks XOR-swizzled by row,
//            so K3's shared-memory staging is bank-conflict free and the tile
//            leaves with one bulk copy)
#pragma once
#include <cstdint>

namespace wino {

constexpr int kPlanes = 46;
constexpr int kRealPlanes = 16;
constexpr int kPrimaries = 10;
constexpr int kPieces = 2;
constexpr int kSlots = 36;    // M'' values per (tile, cout)
constexpr int kMBlock = 128;   // GEMM M (tiles per CTA) = TMEM lanes
constexpr int kKStep = 32;     // int8 MMA K
constexpr int kMaxLanes = 8;   // concurrent chunk pipelines of one conv call (wino_conv_desc.lanes)

// Division by a plan constant d >= 1 for 0 <= n < 2^31 without the ~25-instruction integer divide:
// q = (n m) >> (31 + s), s = ceil(log2 d), m = ceil(2^(31+s) / d) < 2^32.  Exact: with m d = 2^(31+s) + e,
// 0 <= e < d <= 2^s, n m / 2^(31+s) = n / d + n e / (d 2^(31+s)) and the error term is < 1/d.
struct FastDiv {
  uint32_t m;
  int s;
};
inline FastDiv make_fastdiv(int d) {
  int s = 0;
  while ((1ll << s) < d) s++;
  const unsigned long long num = 1ull << (31 + s);
  return FastDiv{(uint32_t)((num + (unsigned long long)d - 1) / (unsigned long long)d), s};
}
__host__ __device__ __forceinline__ int fdiv(int n, FastDiv f) {
  return (int)(((unsigned long long)(uint32_t)n * f.m) >> (31 + f.s));
}

struct Geom {
  int n, h, w, cin, cout, pad, layout;
  int ho, wo, th, tw, tpi;     // output size, tiles per row/col, tiles per image
  FastDiv dv_tw, dv_tpi;       // divisions by tw and tpi (tile decode in K2)
  int cin_pad, cout_pad, nblk, ksteps;
  int scaling, target, out_mode;   // out_mode: WINO_OUT_INT8 or WINO_OUT_INT32 (the pooled mode maps to INT8)
  int pool2;                   // 2x2/2 max pool of the int8 output fused into the output stage (NHWC)
  int path;                    // WINO_PATH_FUSED (0) or WINO_PATH_STAGED (1)
  int alg;                     // WINO_ALG_F4X4 (0) or WINO_ALG_F2X2 (1)
  int tile;                    // output tile edge (4 or 2)
  int npos;                    // Winograd positions = M'' slots = codes per cout (36 or 16)
  int planes;                  // staged GEMM planes per (tile, channel) (46 or 16)
  int in_u8, zx, zw;           // uint8 x/w with zero points (f2, A28); 0, 0, 0 for int8
  int w1;                      // int8-native target (f3, A29): W' is ONE s8 piece per plane, 7-bit codes
  int qk;                      // fused path, quarter-K packing (c_in <= 8, NHWC int8): V / W' per pack (above)
  int chunk_imgs;
  long long chunk_tiles_pad;   // multiple of kMBlock
};

__host__ __device__ __forceinline__ long long tiled_offset(int r, int k, int R) {
  return (long long)(k >> 5) * R * 32 + (r >> 3) * 256 + ((k >> 4) & 1) * 128 + (r & 7) * 16 + (k & 15);
}

constexpr int kVBlockBytes = kMBlock * kKStep;   // one (plane-piece, tile block, K step) block = 4 KB
// Byte offset of V piece `piece` (0 hi, 1 lo) of plane `plane`, chunk tile t, channel k (staged path).
__host__ __device__ __forceinline__ long long v_offset(const Geom& g, int plane, int piece, long long t, int k) {
  const long long blk = t / kMBlock;
  const int r = (int)(t % kMBlock);
  return (((blk * g.planes + plane) * g.ksteps + (k >> 5)) * 2 + piece) * kVBlockBytes + tiled_offset(r, k & 31, kMBlock);
}
// Element offset of (chunk tile t, cout co) inside one plane of M.
__host__ __device__ __forceinline__ long long m_offset(const Geom& g, long long t, int co) {
  const int r = (int)(t & (kMBlock - 1)), c = co % g.nblk, nb = co / g.nblk;
  const int cpr = g.nblk >> 2, swz = (cpr < 8 ? cpr : 8) - 1;
  return ((t >> 7) * (long long)(g.cout_pad / g.nblk) + nb) * (kMBlock * g.nblk) + r * g.nblk +
         (((c >> 2) ^ (r & swz)) << 2) + (c & 3);
}
// Byte offset of W piece `piece` (0 hi, 1 lo) of plane `plane`, output channel co, input channel k (staged).
// Staged path: [plane][cout block][K step][W hi rows | W lo rows]; the fused F(2x2) path (k_fused2.cu)
// orders [cout block][plane][K step][...] so that the two planes of a pair are contiguous.
__host__ __device__ __forceinline__ long long w_offset(const Geom& g, int plane, int piece, int co, int k) {
  const int nb = co / g.nblk, r = co % g.nblk;
  const long long blk = g.path == 0 ? (long long)nb * g.planes + plane : (long long)plane * (g.cout_pad / g.nblk) + nb;
  return (blk * g.ksteps + (k >> 5)) * (2 * g.nblk * kKStep) + tiled_offset(piece * g.nblk + r, k & 31, 2 * g.nblk);
}

// ---------------------------------------------------------------- fused-path (K3F) operand layouts
// The fused path stores the Winograd-domain operands by GROUP: a real position
// (one real value) or a complex primary (Re and Im, the 4-multiplication complex
// product Re = VrWr - ViWi, Im = VrWi + ViWr expressed as K/N-concatenated real
// GEMMs).  Groups are numbered in the fused kernel's processing order gi:
//   gi = 5k + s, k = 0..3 -> row R[frow(k)] (rows 0, 5, 1, 2): s < 4 real (R[ri], R[s]),
//                                                            s = 4 primary ri
//   gi = 20..25            -> primaries 4..9 (row 3)
// Every value v is split into two BALANCED s8 pieces: lo = ((v + 128) & 255) - 128,
// hi = (v - lo) / 256, so v = 256 hi + lo and one UMMA signedness (s8 x s8) fits all.
// V (per 128-tile block): [group gi][K step][piece][128 rows x 32 B] with pieces
//   real (hi, lo), complex (Re hi, Re lo, Im hi, Im lo)  -> 72 pieces per K step;
//   a group's K steps are contiguous, so one bulk copy moves a whole stage.
// W' (per 16-cout block): [group gi][K step][B rows x 32 B] with
//   real: 32 rows [W hi (16 couts) | W lo (16)]
//   complex: 128 rows: B0 = [Wr hi | Wi hi | Wr lo | Wi lo], B1 = [-Wi hi | Wr hi | -Wi lo | Wr lo]
//   -> 56 x 32 rows per K step.
constexpr int kFN16 = 16;            // couts per fused unit
constexpr int kFGroupsN = 26;
constexpr int kVPiecesF = 72;        // V pieces per (tile block, K step)
constexpr int kWRowUnitsF = 56;      // 32-row W' units per (cout block, K step)
__host__ __device__ constexpr int frow(int k) { return k == 0 ? 0 : (k == 1 ? 3 : k - 1); }
__host__ __device__ constexpr bool fg_complex(int gi) { return gi >= 20 || gi % 5 == 4; }
__host__ __device__ constexpr int fg_pieces(int gi) { return fg_complex(gi) ? 4 : 2; }
__host__ __device__ constexpr int fg_wunits(int gi) { return fg_complex(gi) ? 4 : 1; }   // 32-row units
__host__ __device__ constexpr int fg_vprefix(int gi) { return gi < 20 ? (gi / 5) * 12 + (gi % 5) * 2 : 48 + (gi - 20) * 4; }
__host__ __device__ constexpr int fg_wprefix(int gi) { return gi < 20 ? (gi / 5) * 8 + (gi % 5) : 32 + (gi - 20) * 4; }
// real plane index (R[ri]*... numbering of layout: ri*4 + s) or primary index of a group
__host__ __device__ constexpr int fg_real_plane(int gi) { return frow(gi / 5) * 4 + gi % 5; }
__host__ __device__ constexpr int fg_primary(int gi) { return gi < 20 ? frow(gi / 5) : 4 + gi - 20; }
// group of real plane s (= ri*4 + c) / of primary k
__host__ __device__ constexpr int fg_of_real(int s) {
  return ((s >> 2) == 0 ? 0 : ((s >> 2) == 3 ? 1 : (s >> 2) + 1)) * 5 + (s & 3);
}
__host__ __device__ constexpr int fg_of_primary(int k) {
  return k < 4 ? (k == 0 ? 0 : (k == 3 ? 1 : k + 1)) * 5 + 4 : 20 + k - 4;
}
// balanced s8 split
__host__ __device__ __forceinline__ int bal_lo(int v) { return ((v + 128) & 255) - 128; }
__host__ __device__ __forceinline__ int bal_hi(int v) { return (v - bal_lo(v)) >> 8; }
// byte offset of V piece `piece` of group gi, chunk tile t, channel k (fused layout)
__host__ __device__ __forceinline__ long long vf_offset(const Geom& g, int gi, int piece, long long t, int k) {
  const long long blk = t / kMBlock;
  const int r = (int)(t % kMBlock);
  return ((blk * kVPiecesF + fg_vprefix(gi)) * g.ksteps + (long long)(k >> 5) * fg_pieces(gi) + piece) * kVBlockBytes +
         tiled_offset(r, k & 31, kMBlock);
}
// byte offset of W' row `row` (within the group's 32- or 128-row block) of group gi, cout block nb, channel k
__host__ __device__ __forceinline__ long long wf_offset(const Geom& g, int gi, int nb, int row, int k) {
  const int rows = 32 * fg_wunits(gi);
  return ((long long)(nb * kWRowUnitsF + fg_wprefix(gi)) * g.ksteps + (long long)(k >> 5) * fg_wunits(gi)) * 1024 +
         tiled_offset(row, k & 31, rows);
}

// ---------------------------------------------------------------- fused path, quarter-K packing (c_in <= 8)
// With one K step and at most 8 input channels, a 32-byte K row carries TWO slot-groups (a "pack"): slot-group
// 2P in bytes 0..15 and 2P+1 in bytes 16..31, each as two 8-channel value parts -- a real pair's groups g0, g1,
// or a complex group's Re and Im.  V (per 128-tile block): [pack 0..8][piece hi, lo][128 rows x 32 B] = 72 KB
// (4x less than the unpacked 288 KB at c_in_pad 32).  W' (per 16-cout block): [pack][160 rows x 32 B], the
// block-diagonal B of one N = 160 UMMA pair that fills two adjacent TMEM slots at once: rows 0..63 slot 2P,
// 64..95 zero, 96..159 slot 2P+1; a slot's 64 rows are (cout = row % 16)
//   real pair (interleaved slot [g0 s16 | g1 s16 | g0 s8 | g1 s8 | g0 s0 | g1 s0]):
//     rows 0-15 W hi(g0) in part 0, 16-31 W hi(g1) in part 1, 32-47 W lo(g0) part 0, 48-63 W lo(g1) part 1
//   complex (slot [Re16 | Im16 | Re8 | Im8 | Re0 | Im0], A = [Vr | Vi] along K):
//     rows 0-15 [Wr hi | (-Wi) hi], 16-31 [Wi hi | Wr hi], 32-47 [Wr lo | (-Wi) lo], 48-63 [Wi lo | Wr lo]
// A = the pack's hi (or lo) block, at TMEM slot 2P's column 0 (hi) and 32 (lo): one UMMA pair per two
// slot-groups (K = 32, N = 160) instead of 2 or 4 per slot-group.
constexpr int kQkPacks = 9;
constexpr int kQkRows = 160;
constexpr uint32_t kQkPackW = kQkRows * 32;        // 5120 B of W' per (pack, 16-cout block)
constexpr uint32_t kQkPackV = 2 * kVBlockBytes;    // 8 KB of V per (pack, tile block)
// slot-group of fused group gi (processing order of k_fused.cu: rows 0, 5, 1, 2 as pair, pair, complex;
// then row 3's six complex groups), its first group and its group count
__host__ __device__ constexpr int qk_sg_of(int gi) {
  return gi < 20 ? (gi / 5) * 3 + ((gi % 5) < 4 ? (gi % 5) / 2 : 2) : 12 + gi - 20;
}
__host__ __device__ constexpr int qk_sg_first(int sg) { return sg < 12 ? (sg / 3) * 5 + (sg % 3) * 2 : 20 + sg - 12; }
// byte of value part vp (0/1) of group gi's slot-group inside the pack's 32-byte K row, channel ch (< 8)
__host__ __device__ constexpr int qk_kbyte(int gi, int vp, int ch) { return (qk_sg_of(gi) % 2) * 16 + vp * 8 + ch; }
__host__ __device__ __forceinline__ long long vq_offset(long long t, int pack, int piece, int kbyte) {
  return ((t / kMBlock) * kQkPacks + pack) * (long long)kQkPackV + piece * kVBlockBytes +
         tiled_offset((int)(t % kMBlock), kbyte, kMBlock);
}
__host__ __device__ __forceinline__ long long wq_offset(int nb, int pack, int row, int kbyte) {
  return (long long)(nb * kQkPacks + pack) * kQkPackW + tiled_offset(row, kbyte, kQkRows);
}

// Byte offset of the single s8 W' piece (int8-native target, f3) of plane `plane`, cout co, channel k:
// [plane][cout block][K step][n_block rows x 32 B].
__host__ __device__ __forceinline__ long long w1_offset(const Geom& g, int plane, int co, int k) {
  const int nb = co / g.nblk, r = co % g.nblk;
  return (((long long)plane * (g.cout_pad / g.nblk) + nb) * g.ksteps + (k >> 5)) * (g.nblk * kKStep) +
         tiled_offset(r, k & 31, g.nblk);
}

// Position index (r*6+c) of real plane s and of complex primary k / its mirror
// (arithmetic, so no local-memory tables; R = {0,1,2,5} -> R[i] = i + 2 (i == 3)).
__host__ __device__ __forceinline__ int rsel(int i) { return i + (i == 3 ? 2 : 0); }
__host__ __device__ __forceinline__ int real_pos(int s) { return rsel(s >> 2) * 6 + rsel(s & 3); }
__host__ __device__ __forceinline__ int cpx_pos(int k) {      // (R[k],3) | (3,R[k-4]) | (3,3) | (3,4)
  return k < 4 ? rsel(k) * 6 + 3 : (k < 8 ? 18 + rsel(k - 4) : 21 + (k - 8));
}
__host__ __device__ __forceinline__ int cpx_mirror_pos(int k) {   // (R[k],4) | (4,R[k-4]) | (4,4) | (4,3)
  return k < 4 ? rsel(k) * 6 + 4 : (k < 8 ? 24 + rsel(k - 4) : 28 - (k - 8));
}

// round-half-away-from-zero of v / 2^k (k >= 1), 64-bit.
__device__ __forceinline__ long long rha_shift64(long long v, int k) {
  long long a = v < 0 ? -v : v;
  long long r = (a + (1ll << (k - 1))) >> k;
  return v < 0 ? -r : r;
}

// Decode a 6-bit code (n << 2 | (p - 4)); 0 = unscaled.
__device__ __forceinline__ void decode_code(int code, int& n, int& p) {
  n = code >> 2;
  p = (code & 3) + 4;
}
// Decode a 7-bit code of the int8-native target (f3, A29): (n << 3) | (p - 4), p in [4,8].
__device__ __forceinline__ void decode_code7(int code, int& n, int& p) {
  n = code >> 3;
  p = (code & 7) + 4;
}
// Inverse factor (A8/A27): the largest q in {7..3} with m = rha(2^(q+p)/n) <= 255
// (q = 3 only for the 8/128 factor that int9 weights reach).
__device__ __forceinline__ void inverse_factor(int n, int p, int& m, int& q) {
  for (q = 7; q >= 3; --q) {
    long long num = 1ll << (q + p);
    m = (int)((2 * num + n) / (2 * n));
    if (m <= 255) return;
  }
  q = 4;
  m = 255;   // unreachable for valid codes (n >= 8)
}

}  // namespace wino
