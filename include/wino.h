/*
 * wino.h -- C ABI of the B200-native complex-Winograd int8 convolution.
 *
 * Method: Meng & Brothers, "Efficient Winograd Convolution via Integer
 * Arithmetic" (arXiv 1901.01965).  "P:n" cites line n of the paper text
 * (reference PAPER.md); "A<n>" cites a reading recorded in DESIGN.md.
 *
 * What the library computes (all integer, bit-exact, no CPU fallback):
 *   y = 3x3 stride-1 dilation-1 correlation of x with w, zero padding `pad`,
 *   evaluated as the complex Winograd F(4x4,3x3) over the Gaussian integers
 *   with interpolation points {0, +-1, +-i}:
 *       Y = A^T [ (G g G^T) (.) (B^T d B) ] A
 *   with the conjugate-pair / real-split savings (16 real + 10 Karatsuba
 *   complex products = 46 general multiplications per tile),
 *   the imaginary output skipped, and, when filter_scaling != 0, the
 *   paper's integer filter-precision scaling of the Winograd-domain filters
 *   (n / 2^p downscale with 6-bit codes, 8-bit m / 2^q reverse scale before
 *   the output transform), composed with the complex
 *   F(4x4) as an extension (A17).  G is used scaled by 4 (A2) so one final
 *   out32 = rha(Re Y / 16) recovers the convolution (A11).
 *
 * Conventions
 *   - Every function returns a wino_status; nothing aborts or throws.
 *   - All tensor pointers passed to wino_transform_filter / wino_conv2d_int8
 *     are DEVICE pointers on the plan's device, 16-byte aligned, owned by
 *     the caller (the library never allocates or frees device memory).
 *   - Scale codes are validated at the boundary (P:330 read as A4: 0, or
 *     (n << 2) | (p - 4) with n in [8, 15]): a code buffer is checked on the
 *     device, synchronously, the first time a plan sees it (or by
 *     wino_validate_codes), and an invalid entry returns WINO_ERR_RANGE
 *     before any kernel of the conv is enqueued.  Buffers written by the
 *     plan's own wino_transform_filter are valid by construction.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Work is enqueued asynchronously; launch errors are returned
 *     at once, device faults surface at the caller's next synchronisation.
 *   - Calls on different streams are safe when each uses its own workspace.
 *   - int8 tensors are two's-complement with no zero points (A12); uint8
 *     input (input_type) carries explicit zero points (A28).
 */
#ifndef WINO_H
#define WINO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    WINO_OK = 0,
    WINO_ERR_INVALID_ARG = -1,   /* NULL / misaligned pointer, bad enum, wrong device  */
    WINO_ERR_UNSUPPORTED = -2,   /* shape or flag outside the supported set            */
    WINO_ERR_SHAPE = -3,         /* inconsistent sizes                                  */
    WINO_ERR_RANGE = -4,         /* invalid scale code; requant shift out of [0, 62] or
                                    multiplier < 1                                      */
    WINO_ERR_CUDA = -5,          /* a CUDA runtime call failed (launch or attribute)    */
    WINO_ERR_NOMEM = -6          /* host allocation of the plan failed                  */
} wino_status;

/* Tensor layouts; x and y share the layout of the plan.
 *   WINO_NCHW: x [N][Cin][H][W],  w [Cout][Cin][3][3] (OIHW), y [N][Cout][Ho][Wo]
 *   WINO_NHWC: x [N][H][W][Cin],  w [Cout][3][3][Cin] (OHWI), y [N][Ho][Wo][Cout]
 * with Ho = H + 2 pad - 2, Wo = W + 2 pad - 2.                                   */
enum { WINO_NCHW = 0, WINO_NHWC = 1 };

/* Output element type.
 *   WINO_OUT_INT32: y = out32 = rha(Re Y / 16)  (the convolution itself when
 *                   unscaled; int32, wraps never: |y| < 2^31 for Cin <= 896).
 *   WINO_OUT_INT8:  y = clamp(rha(out32 * requant_mult / 2^requant_shift),
 *                   -128, 127) with a 64-bit product (A14).                     */
enum { WINO_OUT_INT8 = 0, WINO_OUT_INT32 = 1, WINO_OUT_INT8_POOL2 = 2 };
/*   WINO_OUT_INT8_POOL2: the int8 output above followed by the 2x2 stride-2 max
 *                   pool of the VGG stack (A22), fused into the output stage:
 *                   y [N][Ho/2][Wo/2][Cout] (floor); NHWC, complex F(4x4),
 *                   c_out % 16 == 0 (fused path) or % 4 == 0 (staged path),
 *                   else WINO_ERR_UNSUPPORTED.  Identical to wino_maxpool2_int8
 *                   applied to the WINO_OUT_INT8 result (requantisation is
 *                   monotone, so the pool commutes with it).                  */

typedef struct {
    int n, h, w;          /* batch and input spatial size, each >= 1                  */
    int c_in, c_out;      /* 1 <= c_in <= 896 (768 scaled; int32 exactness, A23),
                             1 <= c_out <= 2048                                       */
    int pad;              /* 0 or 1; h + 2 pad >= 3 and w + 2 pad >= 3                 */
    int layout;           /* WINO_NCHW or WINO_NHWC                                    */
    int filter_scaling;   /* 0: exact (codes all 0); 1: the paper's scheme */
    int filter_target_max;/* 255: the paper's int9 target (A6, the default);
                             127: the int8-native target (needs
                             filter_scaling, the staged path, F4x4 and int8 input)   */
    int out_mode;         /* WINO_OUT_INT8, WINO_OUT_INT32 or WINO_OUT_INT8_POOL2       */
    int workspace_mb;     /* batch-chunk budget for V (+ M) in MiB; 0 = default (128, or
                             env WINO_CHUNK_MB).  Larger = fewer, longer launches.     */
    int path;             /* WINO_PATH_AUTO (0, the default everywhere -- this ABI, the
                             Python WinoConv2d and ConvStack): fused for F2x2, and for
                             F4x4 when c_in <= 128 (target 255), else staged;
                             wino_plan_info.path reports the choice.
                             WINO_PATH_FUSED (1): K2 input transform, then ONE kernel for
                             the GEMMs (4-multiplication complex form, 36 planes) +
                             reverse scaling + output transform + store (M'' on chip).
                             WINO_PATH_STAGED (2): K2, K3 GEMMs (46 planes: 16 real +
                             10 Karatsuba x 3) -> M'' in the workspace,
                             K4 output transform (M'' inspectable, wino_plan_info).   */
    int algorithm;        /* WINO_ALG_F4X4 (0, default): complex F(4x4,3x3) over the
                             Gaussian integers, points {0, +-1, +-i};
                             WINO_ALG_F2X2 (1): rational F(2x2,3x3), G' = 2G,
                             the configuration the paper evaluates; either path.
                             Codes are [c_out][36] (F4x4) or [c_out][16] (F2x2).      */
    int input_type;       /* WINO_IN_INT8 (0, default) or WINO_IN_UINT8 (1): x and w are
                             uint8 with the zero points below (the paper's affine model,
                             P:251); the convolution is that of the int9 values x - zx,
                             w - zw, padding = real 0 (A28).  c_in <= 224
                             (int32 exactness); either algorithm, either path.        */
    int x_zero_point;     /* [0, 255], uint8 input only                                  */
    int w_zero_point;     /* [0, 255], uint8 input only                                  */
    int lanes;            /* 0 or 1: the chunks of a call run one after another on the
                             caller's stream.  2..8: chunk c runs on lane c % lanes, each
                             lane with its own V (+ M'') buffer in the workspace and its
                             own stream (the plan's, forked from and joined back into the
                             caller's stream with events, so CUDA-graph capture works);
                             one chunk's input transform then overlaps another's GEMM.
                             Capped at the chunk count.  Results are identical.         */
} wino_conv_desc;

/* Hot-path kernel structure (wino_conv_desc.path). */
enum { WINO_PATH_AUTO = 0, WINO_PATH_FUSED = 1, WINO_PATH_STAGED = 2 };

/* Winograd algorithm (wino_conv_desc.algorithm). */
enum { WINO_ALG_F4X4 = 0, WINO_ALG_F2X2 = 1 };

/* Element type of x and w (wino_conv_desc.input_type). */
enum { WINO_IN_INT8 = 0, WINO_IN_UINT8 = 1 };

typedef struct wino_plan_s *wino_plan_t;

/* Geometry and workspace layout of a plan (read-only, for tests and tools). */
typedef struct {
    int ho, wo;                 /* output spatial size                                */
    int tiles_h, tiles_w;       /* ceil(ho/4), ceil(wo/4)                             */
    long long tiles;            /* T = n * tiles_h * tiles_w                          */
    int cin_pad;                /* c_in rounded up to 32 (one int8 MMA K step)        */
    int cout_pad;               /* c_out rounded up to n_block                        */
    int n_block;                /* GEMM N tile (couts per CTA)                         */
    int m_block;                /* GEMM M tile (tiles per CTA) = 128                   */
    int planes;                 /* staged F4x4: 46 = 16 real + 10 x {re, im, re+im}
                                   (P:228); fused F4x4: 36 = 16 real + 10 x {re, im};
                                   F2x2: 16                                            */
    int pieces;                 /* 2 int8 pieces per operand value, v = 256 hi + lo:
                                   balanced s8 (lo = low byte of v read as s8), except
                                   the fused path's V (lo = v & 255 as u8) */
    int chunk_images;           /* images per workspace chunk                          */
    int n_chunks;
    int lanes;                  /* chunk pipelines actually used (<= n_chunks)          */
    size_t lane_bytes;          /* workspace bytes per lane (V + M'' of one chunk)     */
    int packing;                /* 1; 4 = the fused path's quarter-K packing at c_in <= 8
                                   (two slot-groups per 32-byte K row)    */
    long long chunk_tiles_pad;  /* tiles per chunk rounded up to m_block               */
    int path;                   /* WINO_PATH_FUSED or WINO_PATH_STAGED (AUTO resolved)  */
    int stages;                 /* kernels per chunk: 2 (fused) or 3 (staged)          */
    int algorithm;              /* WINO_ALG_F4X4 or WINO_ALG_F2X2                      */
    int tile;                   /* output tile edge: 4 (F4x4) or 2 (F2x2)             */
    int positions;              /* Winograd positions = codes per c_out: 36 or 16     */
    size_t v_offset, v_bytes;   /* V  = B^T d B operand planes inside the workspace (lane 0;
                                   lane k at + k * lane_bytes; chunk c on lane c % lanes) */
    size_t m_offset, m_bytes;   /* M'' = 36 int32 per (tile, cout) after Karatsuba and
                                   reverse scaling; swizzled tiles; staged
                                   path only (m_bytes = 0 on the fused path)           */
    size_t workspace_bytes;     /* lanes x lane_bytes + a 256-byte status block (the
                                   code-validation flag)                               */
    size_t filter_bytes;        /* transformed-filter buffer (w_wino)                  */
    size_t codes_bytes;         /* c_out * positions bytes (36 F4x4, 16 F2x2)         */
    size_t x_bytes, y_bytes;    /* input / output tensor sizes in bytes                */
} wino_plan_info;

/* Human-readable text for a status code (static storage, never NULL). */
const char *wino_status_string(wino_status s);

/* Text of the CUDA runtime error behind the calling thread's most recent
 * WINO_ERR_CUDA ("no error" if none); static storage, never NULL.        */
const char *wino_last_cuda_error(void);

/* Validate `desc` and build an immutable plan for CUDA device `device`.
 * The plan holds host metadata only.  Returns WINO_ERR_UNSUPPORTED for
 * pad not in {0,1}, n/h/w/c < 1, h + 2 pad < 3 or w + 2 pad < 3,
 * c_in > 896 (> 768 with filter_scaling; > 224 for uint8 input), c_out > 2048,
 * filter_target_max not in {255, 127} (127 only with scaling, staged, F4x4,
 * int8), and WINO_ERR_INVALID_ARG for bad enums or NULL pointers.  The device
 * must be sm_100 (B200).  A plan's only mutable state is its set of known-valid
 * code buffers (thread-safe).                                            */
wino_status wino_plan(const wino_conv_desc *desc, int device, wino_plan_t *out);
wino_status wino_plan_destroy(wino_plan_t plan);
wino_status wino_plan_query(wino_plan_t plan, wino_plan_info *info);

/* Sizes of the caller-allocated device buffers (0 on a NULL plan). */
size_t wino_filter_bytes(wino_plan_t plan);     /* w_wino                      */
size_t wino_codes_bytes(wino_plan_t plan);      /* scale_codes = c_out * positions */
size_t wino_workspace_bytes(wino_plan_t plan);  /* V and M of one batch chunk + status */
size_t wino_output_bytes(wino_plan_t plan);     /* y                            */

/* Offline filter transform: for every output channel,
 *   W = G_int g G_int^T (G_int = 4G) for all input channels;
 *   per position (X-Y location) the max over input channels of
 *   max(|Re W|, |Im W|) (A5) selects the code (n, p) of P:317-330 read as A3
 *   (code = (n << 2) | (p - 4), 0 = unscaled, A4; mirrors share their
 *   primary's code; 7-bit (n << 3) | (p - 4) for target 127, A29);
 *   W' = rha(W n / 2^p) (A7); then the GEMM operand planes split into balanced
 *   int8 pieces: staged path 46 planes (16 real, and re, im, re+im per complex
 *   primary for the Karatsuba product), fused path 16 real planes +
 *   the [Wr | Wi] / [-Wi | Wr] blocks of the 4-multiplication complex product
 *   (identical integers).  F2x2: W = G' g G'^T (G' = 2G),
 *   16 real planes, 16 codes per c_out.  The codes buffer is recorded as valid
 *   for this plan.
 *   w           device, int8, layout per desc (OIHW or OHWI)
 *   w_wino      device, wino_filter_bytes(plan) bytes, written (opaque layout,
 *               documented in DESIGN.md "HBM layout")
 *   scale_codes device, [c_out][positions] uint8, written (all 0 when
 *               filter_scaling == 0)                                        */
wino_status wino_transform_filter(wino_plan_t plan, const int8_t *w, void *w_wino,
                                  uint8_t *scale_codes, void *stream);

/* The convolution hot path:
 * input transform D = B^T d B per tile and channel, 46 Winograd-domain
 * int8 GEMMs [tiles x Cin] x [Cin x Cout] on the tcgen05 tensor cores with
 * int32 accumulation, Karatsuba recombination, reverse scaling
 * M'' = rha(M m / 2^q) with (m, q) derived from `scale_codes` on the device
 * (A8), real-only output transform, rha(./16), crop, optional
 * requantisation, store.
 *   x            device, int8 input, layout per desc
 *   w_wino       device, produced by wino_transform_filter for this plan
 *   scale_codes  device, [c_out][positions] 6-bit codes -- THE explicit
 *                filter-scale parameter: the codes W' was scaled with (from
 *                wino_transform_filter, or any codes applied consistently).
 *                Every entry must be 0 or decode to n in [8,15] (A4; 7-bit
 *                codes, p in [4,8], for target 127): on the first call with a
 *                buffer the plan has not seen, the codes are checked on the
 *                device and the stream is synchronised; an invalid entry
 *                returns WINO_ERR_RANGE and nothing is enqueued.  A caller
 *                that rewrites a buffer the plan has already accepted with
 *                codes of its own re-checks it with wino_validate_codes.
 *   requant_mult, requant_shift  used for WINO_OUT_INT8 only: mult >= 1,
 *                shift in [0, 62], else WINO_ERR_RANGE
 *   y            device, wino_output_bytes(plan) bytes, written
 *   workspace    device, wino_workspace_bytes(plan) bytes, scratch (holds
 *                V and M of the last chunk afterwards, see wino_plan_info) */
wino_status wino_conv2d_int8(wino_plan_t plan, const int8_t *x, const void *w_wino,
                             const uint8_t *scale_codes, int32_t requant_mult, int requant_shift,
                             void *y, void *workspace, void *stream);

/* End-to-end variant with HOST tensors: enqueues the host-to-device copy of
 * x (x_host -> x_dev), wino_conv2d_int8, and the device-to-host copy of y
 * (y_dev -> y_host) on `stream`.  x_host / y_host should be pinned
 * (cudaHostAlloc) for asynchronous copies; x_dev / y_dev are caller-owned
 * device staging buffers of wino_plan_info.x_bytes / y_bytes.  The caller
 * synchronises the stream before reading y_host.                          */
wino_status wino_conv2d_int8_host(wino_plan_t plan, const int8_t *x_host, const void *w_wino,
                                  const uint8_t *scale_codes, int32_t requant_mult,
                                  int requant_shift, void *y_host, int8_t *x_dev, void *y_dev,
                                  void *workspace, void *stream);

/* Profiling / testing entry point: enqueue ONE kernel of the hot path for
 * batch chunk `chunk` (0 <= chunk < wino_plan_info.n_chunks):
 *   stage 2 = input transform (x -> V in the workspace),
 *   fused path:  stage 3 = GEMMs + Karatsuba + reverse scaling + output
 *                transform + store (V, w_wino, scale_codes -> y);
 *   staged path: stage 3 = Winograd-domain GEMMs + Karatsuba + reverse
 *                scaling (V, w_wino, scale_codes -> M'' in the workspace),
 *                stage 4 = output transform (M'' -> y).
 * Running stages 2 .. 1 + wino_plan_info.stages for every chunk in order is
 * exactly wino_conv2d_int8.  Arguments as for wino_conv2d_int8; WINO_ERR_INVALID_ARG
 * for a bad stage or chunk.                                               */
wino_status wino_conv2d_int8_stage(wino_plan_t plan, int stage, int chunk, const int8_t *x,
                                   const void *w_wino, const uint8_t *scale_codes,
                                   int32_t requant_mult, int requant_shift, void *y,
                                   void *workspace, void *stream);

/* Synchronous validation of a code buffer against this plan (A4):
 * checks all c_out * positions entries on the device (flag in the workspace's
 * status block), synchronises `stream`, and returns WINO_OK (and records the
 * buffer as valid for the plan) or WINO_ERR_RANGE (and forgets it).
 * codes and workspace are device pointers as for wino_conv2d_int8.         */
wino_status wino_validate_codes(wino_plan_t plan, const uint8_t *scale_codes, void *workspace, void *stream);

/* Asynchronous device-side check of a code table: writes 1 to *bad_flag
 * (device int32, caller-zeroed) if any of the c_out * positions codes is
 * neither 0 nor a valid code (n in [8,15]).                               */
wino_status wino_check_codes(wino_plan_t plan, const uint8_t *scale_codes, int32_t *bad_flag,
                             void *stream);

/* Debug only (effective when libwino is built with -DWINO_K3_TRACE, e.g.
 * WINO_NVCC_FLAGS=-DWINO_K3_TRACE python paper_1901_01965_b200/build.py --force):
 * when `device_buffer` is non-NULL, subsequent GEMM (K3) launches
 * write a per-CTA timeline of globaltimer stamps into it (uint64
 * [grid][16 planes][6 events]: producer issued, MMA saw data, MMA got TMEM
 * buffer, MMA committed, epilogue saw accumulators, epilogue finished unit).
 * The buffer must hold num_SMs * 96 uint64.  NULL turns tracing off.      */
wino_status wino_debug_set_trace(void *device_buffer);

/* Debug / test only: floor(n / d) through the plan-constant fast division the
 * kernels use for their tile decode (layout.cuh FastDiv), evaluated on the host.
 * n in [0, 2^31), d >= 1; returns -1 for arguments outside that range.     */
int wino_debug_fastdiv(int n, int d);

/* Harness op for the VGG stack (A22): 2x2 stride-2 max pool on int8,
 * layout per `layout`, y [N][C][H/2][W/2] or [N][H/2][W/2][C].           */
wino_status wino_maxpool2_int8(const int8_t *x, int n, int h, int w, int c, int layout,
                               int8_t *y, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* WINO_H */
