// wino_abi.cu -- the C ABI declared in include/wino.h: plan validation,
// workspace sizing (batch chunks sized to stay L2-resident), and sequencing of
// the K2 -> K3 -> K4 launches per chunk on the caller's stream.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/wino.h"
#include "kernels.cuh"
#include "layout.cuh"

struct wino_plan_s {
  wino_conv_desc d;           // as given (d.path may be WINO_PATH_AUTO)
  int device = 0;
  wino::Geom g{};             // g.path: the kernel path, 0 fused / 1 staged (layout.cuh)
  int n_chunks = 0;
  size_t v_bytes = 0, m_bytes = 0, status_offset = 0, ws_bytes = 0, f_bytes = 0, x_bytes = 0, y_bytes = 0;
  // scale-code buffers known to hold valid codes (written by wino_transform_filter of this plan, or
  // checked by wino_validate_codes); the only mutable state of a plan, guarded by `mu`
  std::mutex mu;
  std::vector<const uint8_t*> valid_codes;
  // chunk pipelines (wino_conv_desc.lanes): chunk c runs on lane c % lanes with its own V (+ M'') buffer
  // at workspace + lane * lane_bytes; lane 0 is the caller's stream, lanes 1.. are the plan's own streams,
  // forked from and joined back into the caller's stream with events (graph-capture safe)
  int lanes = 1;
  size_t lane_bytes = 0;
  std::mutex lane_mu;
  bool lane_init = false;
  cudaStream_t aux[wino::kMaxLanes] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[wino::kMaxLanes] = {};
  ~wino_plan_s() {
    for (int i = 0; i < wino::kMaxLanes; i++) {
      if (aux[i]) cudaStreamDestroy(aux[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
  }
};

namespace {

thread_local cudaError_t g_last_cuda_error = cudaSuccess;
wino_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return WINO_OK;
  g_last_cuda_error = e;
  return WINO_ERR_CUDA;
}

std::mutex g_setup_mu;
bool g_setup_done[64] = {};

wino_status setup_device(int device) {
  std::lock_guard<std::mutex> lk(g_setup_mu);
  if (device < 0 || device >= 64) return WINO_ERR_INVALID_ARG;
  if (g_setup_done[device]) return WINO_OK;
  int old = -1;
  if (cudaGetDevice(&old) != cudaSuccess) return WINO_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return WINO_ERR_CUDA;
  cudaError_t e = wino::setup_filter_transform();
  if (e == cudaSuccess) e = wino::setup_input_transform();
  if (e == cudaSuccess) e = wino::setup_gemm();
  if (e == cudaSuccess) e = wino::setup_output_transform();
  if (e == cudaSuccess) e = wino::setup_fused();
  if (e == cudaSuccess) e = wino::setup_fused2();
  cudaSetDevice(old);
  if (e != cudaSuccess) return cuda_status(e);
  g_setup_done[device] = true;
  return WINO_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

wino_status check_device(const wino_plan_s* p) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return WINO_ERR_CUDA;
  return cur == p->device ? WINO_OK : WINO_ERR_INVALID_ARG;
}

long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// WINO_K2F_LEGACY=1: the two-channel K2F for NHWC int8 as well (A/B experiments)
// WINO_QK_OFF=1: no quarter-K packing at c_in <= 8 (A/B experiments)
bool qk_off() {
  static const bool v = [] { const char* e = std::getenv("WINO_QK_OFF"); return e && std::atoi(e) != 0; }();
  return v;
}
bool k2f_legacy() {
  static const bool v = [] { const char* e = std::getenv("WINO_K2F_LEGACY"); return e && std::atoi(e) != 0; }();
  return v;
}

// WINO_PATH_AUTO's c_in limit for the fused path; WINO_AUTO_FUSED_CIN overrides (experiments)
int auto_fused_max_cin() {
  const char* env = std::getenv("WINO_AUTO_FUSED_CIN");
  return env ? std::atoi(env) : 128;
}

size_t chunk_budget_bytes(int desc_mb) {
  const char* env = std::getenv("WINO_CHUNK_MB");
  long mb = desc_mb > 0 ? desc_mb : (env ? std::atol(env) : 128);
  if (mb < 1) mb = 1;
  return (size_t)mb << 20;
}

}  // namespace

// ---------------------------------------------------------------- scale-code validation (wino.h)
static bool codes_known_valid(wino_plan_s* p, const uint8_t* codes) {
  std::lock_guard<std::mutex> lk(p->mu);
  for (const uint8_t* c : p->valid_codes)
    if (c == codes) return true;
  return false;
}
static void codes_mark(wino_plan_s* p, const uint8_t* codes, bool valid) {
  std::lock_guard<std::mutex> lk(p->mu);
  for (size_t i = 0; i < p->valid_codes.size(); i++)
    if (p->valid_codes[i] == codes) {
      if (!valid) p->valid_codes.erase(p->valid_codes.begin() + (long)i);
      return;
    }
  if (!valid) return;
  if (p->valid_codes.size() >= 64) p->valid_codes.erase(p->valid_codes.begin());   // oldest out
  p->valid_codes.push_back(codes);
}
// Synchronous device check of c_out * positions codes: the flag lives in the workspace's status block.
static wino_status validate_codes(wino_plan_s* p, const uint8_t* codes, void* workspace, cudaStream_t s) {
  int32_t* flag = reinterpret_cast<int32_t*>(static_cast<int8_t*>(workspace) + p->status_offset);
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) e = wino::launch_check_codes(codes, p->d.c_out * p->g.npos, p->g.w1, flag, s);
  int32_t bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, flag, sizeof(bad), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e);
  codes_mark(p, codes, bad == 0);
  return bad ? WINO_ERR_RANGE : WINO_OK;
}

extern "C" {

const char* wino_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda_error); }

const char* wino_status_string(wino_status s) {
  switch (s) {
    case WINO_OK: return "ok";
    case WINO_ERR_INVALID_ARG: return "invalid argument (null/misaligned pointer, bad enum or wrong device)";
    case WINO_ERR_UNSUPPORTED: return "unsupported shape or flag";
    case WINO_ERR_SHAPE: return "inconsistent sizes";
    case WINO_ERR_RANGE: return "value out of range (invalid scale code, or requant multiplier/shift)";
    case WINO_ERR_CUDA: return "CUDA runtime error";
    case WINO_ERR_NOMEM: return "out of host memory";
  }
  return "unknown status";
}

wino_status wino_plan(const wino_conv_desc* desc, int device, wino_plan_t* out) {
  if (!desc || !out) return WINO_ERR_INVALID_ARG;
  *out = nullptr;
  if (desc->path != WINO_PATH_FUSED && desc->path != WINO_PATH_STAGED && desc->path != WINO_PATH_AUTO)
    return WINO_ERR_INVALID_ARG;
  // WINO_PATH_AUTO (the default, 0): the fused kernels where they measured faster -- the complex F(4x4) one at
  // c_in <= 128 (C2, C3, VGG-16 layers 1-5; at c_in = 256 the staged path won in r02: C4 435 vs 420 TOPS,
  // VGG-16 layers 6-8 1348 / 1327 / 636 vs 1538 / 1484 / 657 us), the rational F(2x2) one everywhere (C2-C4:
  // 1.4-1.7x the staged path) -- for target 255; else staged
  wino_conv_desc dr = *desc;
  if (dr.path == WINO_PATH_AUTO)
    dr.path = (dr.filter_target_max == 255 &&
               (dr.algorithm == WINO_ALG_F2X2 || dr.c_in <= auto_fused_max_cin()))
                  ? WINO_PATH_FUSED
                  : WINO_PATH_STAGED;
  const wino_conv_desc& d = dr;
  if (d.layout != WINO_NCHW && d.layout != WINO_NHWC) return WINO_ERR_INVALID_ARG;
  if (d.out_mode != WINO_OUT_INT8 && d.out_mode != WINO_OUT_INT32 && d.out_mode != WINO_OUT_INT8_POOL2)
    return WINO_ERR_INVALID_ARG;
  if (d.filter_scaling != 0 && d.filter_scaling != 1) return WINO_ERR_INVALID_ARG;
  if (d.workspace_mb < 0) return WINO_ERR_INVALID_ARG;
  if (d.path != WINO_PATH_FUSED && d.path != WINO_PATH_STAGED) return WINO_ERR_INVALID_ARG;
  if (d.algorithm != WINO_ALG_F4X4 && d.algorithm != WINO_ALG_F2X2) return WINO_ERR_INVALID_ARG;
  if (d.input_type != WINO_IN_INT8 && d.input_type != WINO_IN_UINT8) return WINO_ERR_INVALID_ARG;
  if (d.input_type == WINO_IN_UINT8) {
    if (d.x_zero_point < 0 || d.x_zero_point > 255 || d.w_zero_point < 0 || d.w_zero_point > 255)
      return WINO_ERR_INVALID_ARG;
    if (d.c_in > 224) return WINO_ERR_UNSUPPORTED;   // int32 exactness of Y for int9 values (A28)
  }
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c_in < 1 || d.c_out < 1) return WINO_ERR_UNSUPPORTED;
  if (d.pad != 0 && d.pad != 1) return WINO_ERR_UNSUPPORTED;
  if (d.h + 2 * d.pad < 3 || d.w + 2 * d.pad < 3) return WINO_ERR_UNSUPPORTED;
  // int32 exactness of M'' and Y (A23): 896 unscaled, 768 scaled
  if (d.c_in > (d.filter_scaling ? 768 : 896)) return WINO_ERR_UNSUPPORTED;
  if (d.filter_target_max != 255 && d.filter_target_max != 127) return WINO_ERR_UNSUPPORTED;
  // int8-native target (f3, A29): single-piece W' needs scaling, the staged complex F(4x4), int8 input
  if (d.filter_target_max == 127 && (!d.filter_scaling || d.path != WINO_PATH_STAGED || d.algorithm != WINO_ALG_F4X4 ||
                                     d.input_type != WINO_IN_INT8))
    return WINO_ERR_UNSUPPORTED;
  if (d.c_out > 2048 || (long long)d.n * d.h * d.w > (1ll << 40)) return WINO_ERR_UNSUPPORTED;
  if (d.lanes < 0 || d.lanes > wino::kMaxLanes) return WINO_ERR_INVALID_ARG;
  // int8 output with the 2x2/2 max pool fused into the output stage (the VGG stack's pools, A22): NHWC,
  // complex F(4x4); fused path with c_out % 16 == 0, staged path with c_out % 4 == 0
  if (d.out_mode == WINO_OUT_INT8_POOL2 &&
      (d.layout != WINO_NHWC || d.algorithm != WINO_ALG_F4X4 || d.h + 2 * d.pad - 2 < 2 || d.w + 2 * d.pad - 2 < 2 ||
       (d.c_out % (d.path == WINO_PATH_FUSED ? 16 : 4)) != 0))
    return WINO_ERR_UNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) return WINO_ERR_CUDA;
  if (device < 0 || device >= ndev) return WINO_ERR_INVALID_ARG;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return WINO_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return WINO_ERR_UNSUPPORTED;   // sm_100a cubin only
  wino_status st = setup_device(device);
  if (st != WINO_OK) return st;

  wino_plan_s* p = new (std::nothrow) wino_plan_s();
  if (!p) return WINO_ERR_NOMEM;
  p->d = *desc;
  p->device = device;
  wino::Geom& g = p->g;
  g.n = d.n; g.h = d.h; g.w = d.w; g.cin = d.c_in; g.cout = d.c_out; g.pad = d.pad; g.layout = d.layout;
  g.ho = d.h + 2 * d.pad - 2;
  g.wo = d.w + 2 * d.pad - 2;
  g.alg = d.algorithm;
  g.tile = d.algorithm == WINO_ALG_F2X2 ? 2 : 4;
  g.npos = d.algorithm == WINO_ALG_F2X2 ? 16 : 36;
  g.planes = d.algorithm == WINO_ALG_F2X2 ? 16 : wino::kPlanes;
  g.w1 = d.filter_target_max == 127;
  g.in_u8 = d.input_type == WINO_IN_UINT8;
  g.zx = g.in_u8 ? d.x_zero_point : 0;
  g.zw = g.in_u8 ? d.w_zero_point : 0;
  g.th = (g.ho + g.tile - 1) / g.tile;
  g.tw = (g.wo + g.tile - 1) / g.tile;
  g.tpi = g.th * g.tw;
  g.dv_tw = wino::make_fastdiv(g.tw);
  g.dv_tpi = wino::make_fastdiv(g.tpi);
  g.cin_pad = (int)round_up(d.c_in, wino::kKStep);
  // quarter-K packing of the fused complex path at c_in <= 8 (layout.cuh): NHWC int8 (the SWAR K2)
  g.qk = d.path == WINO_PATH_FUSED && d.algorithm == WINO_ALG_F4X4 && d.layout == WINO_NHWC &&
         d.input_type == WINO_IN_INT8 && d.c_in <= 8 && !k2f_legacy() && !qk_off();
  const int cout16 = (int)round_up(d.c_out, 16);
  g.path = d.path == WINO_PATH_FUSED ? 0 : 1;
  // fused path: 16-cout units (UMMA N = 16); staged path: widest N that the cout count fills
  g.nblk = d.path == WINO_PATH_FUSED ? (d.algorithm == WINO_ALG_F2X2 ? 32 : 16)
                                     : (cout16 <= 16 ? 16 : (cout16 <= 32 ? 32 : 64));
  g.cout_pad = (int)round_up(d.c_out, g.nblk);
  g.ksteps = g.cin_pad / wino::kKStep;
  g.scaling = d.filter_scaling;
  g.target = d.filter_target_max;
  g.pool2 = d.out_mode == WINO_OUT_INT8_POOL2;
  g.out_mode = g.pool2 ? WINO_OUT_INT8 : d.out_mode;   // the kernels requantise to int8 either way
  // batch chunk: V (+ M on the staged path) of one chunk within the budget
  const size_t m_per_tile = d.path == WINO_PATH_STAGED ? (size_t)g.npos * 4 * (size_t)g.cout_pad : 0;
  const bool fused_f4 = d.path == WINO_PATH_FUSED && d.algorithm == WINO_ALG_F4X4;
  const size_t v_per_tile_ch = fused_f4 ? wino::kVPiecesF : 2 * (size_t)g.planes;
  const size_t per_img = g.qk ? (size_t)g.tpi * (wino::kQkPacks * wino::kQkPackV / wino::kMBlock)
                              : (size_t)g.tpi * (v_per_tile_ch * (size_t)g.cin_pad + m_per_tile);
  long long imgs = (long long)(chunk_budget_bytes(d.workspace_mb) / (per_img ? per_img : 1));
  if (imgs < 1) imgs = 1;
  if (imgs > d.n) imgs = d.n;
  g.chunk_imgs = (int)imgs;
  g.chunk_tiles_pad = round_up((long long)imgs * g.tpi, wino::kMBlock);
  p->n_chunks = (int)((d.n + imgs - 1) / imgs);
  p->v_bytes = g.qk ? (size_t)(g.chunk_tiles_pad / wino::kMBlock) * wino::kQkPacks * wino::kQkPackV
                   : v_per_tile_ch * g.chunk_tiles_pad * g.cin_pad;
  p->m_bytes = d.path == WINO_PATH_STAGED ? (size_t)g.npos * g.chunk_tiles_pad * g.cout_pad * 4 : 0;
  // + one 256-byte status block (the code-validation flag of wino_validate_codes)
  p->lanes = d.lanes > 1 ? (d.lanes < p->n_chunks ? d.lanes : p->n_chunks) : 1;
  p->lane_bytes = (size_t)round_up((long long)(p->v_bytes + p->m_bytes), 256);
  p->status_offset = p->lane_bytes * p->lanes;
  p->ws_bytes = p->status_offset + 256;
  // W': 92 B per (cin, cout) staged (46 planes x 2 pieces); 112 B fused (56 rows x 2 couts-halves, layout.cuh)
  p->f_bytes = g.qk ? (size_t)(g.cout_pad / 16) * wino::kQkPacks * wino::kQkPackW
                   : (size_t)(fused_f4 ? 2 * wino::kWRowUnitsF : (g.w1 ? 1 : 2) * g.planes) * g.cout_pad * g.cin_pad;
  p->x_bytes = (size_t)d.n * d.h * d.w * d.c_in;
  p->y_bytes = g.pool2 ? (size_t)d.n * (g.ho / 2) * (g.wo / 2) * d.c_out
                       : (size_t)d.n * g.ho * g.wo * d.c_out * (d.out_mode == WINO_OUT_INT32 ? 4 : 1);
  *out = p;
  return WINO_OK;
}

wino_status wino_plan_destroy(wino_plan_t plan) {
  if (!plan) return WINO_ERR_INVALID_ARG;
  delete plan;
  return WINO_OK;
}

wino_status wino_plan_query(wino_plan_t p, wino_plan_info* info) {
  if (!p || !info) return WINO_ERR_INVALID_ARG;
  std::memset(info, 0, sizeof(*info));
  info->ho = p->g.ho; info->wo = p->g.wo;
  info->tiles_h = p->g.th; info->tiles_w = p->g.tw;
  info->tiles = (long long)p->d.n * p->g.tpi;
  info->cin_pad = p->g.cin_pad; info->cout_pad = p->g.cout_pad;
  info->n_block = p->g.nblk; info->m_block = wino::kMBlock;
  info->planes = p->g.path == 0 && p->g.alg == 0 ? 36 : p->g.planes;   // fused F4: 16 + 10 x (re, im)
  info->algorithm = p->g.alg; info->tile = p->g.tile; info->positions = p->g.npos;
  info->pieces = wino::kPieces;
  info->chunk_images = p->g.chunk_imgs; info->n_chunks = p->n_chunks;
  info->lanes = p->lanes; info->lane_bytes = p->lane_bytes;
  info->packing = p->g.qk ? 4 : 1;
  info->chunk_tiles_pad = p->g.chunk_tiles_pad;
  info->path = p->g.path == 0 ? WINO_PATH_FUSED : WINO_PATH_STAGED;
  info->stages = p->g.path == 0 ? 2 : 3;
  info->v_offset = 0; info->v_bytes = p->v_bytes;
  info->m_offset = p->v_bytes; info->m_bytes = p->m_bytes;
  info->workspace_bytes = p->ws_bytes;
  info->filter_bytes = p->f_bytes;
  info->codes_bytes = (size_t)p->d.c_out * p->g.npos;
  info->x_bytes = p->x_bytes; info->y_bytes = p->y_bytes;
  return WINO_OK;
}

size_t wino_filter_bytes(wino_plan_t p) { return p ? p->f_bytes : 0; }
size_t wino_codes_bytes(wino_plan_t p) { return p ? (size_t)p->d.c_out * p->g.npos : 0; }
size_t wino_workspace_bytes(wino_plan_t p) { return p ? p->ws_bytes : 0; }
size_t wino_output_bytes(wino_plan_t p) { return p ? p->y_bytes : 0; }

wino_status wino_transform_filter(wino_plan_t p, const int8_t* w, void* w_wino, uint8_t* codes, void* stream) {
  if (!p || !w || !w_wino || !codes) return WINO_ERR_INVALID_ARG;
  if (!aligned16(w_wino)) return WINO_ERR_INVALID_ARG;
  wino_status st = check_device(p);
  if (st != WINO_OK) return st;
  cudaError_t e = wino::launch_filter_transform(p->g, w, static_cast<int8_t*>(w_wino), codes,
                                                static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) codes_mark(p, codes, true);   // K1 writes valid codes by construction
  return cuda_status(e);
}

static wino_status run_stage(const wino_plan_s* p, int stage, int chunk, const int8_t* x, const void* w_wino,
                             const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y, void* workspace,
                             cudaStream_t s) {
  const wino::Geom& g = p->g;
  const int n0 = chunk * g.chunk_imgs;
  const int imgs = p->d.n - n0 < g.chunk_imgs ? p->d.n - n0 : g.chunk_imgs;
  const long long tiles_pad = round_up((long long)imgs * g.tpi, wino::kMBlock);
  int8_t* vimg = static_cast<int8_t*>(workspace) + (size_t)(chunk % p->lanes) * p->lane_bytes;
  int32_t* m = reinterpret_cast<int32_t*>(vimg + p->v_bytes);
  cudaError_t e = cudaErrorInvalidValue;
  if (stage == 2)
    e = g.path == 0 && g.alg == 0 ? (g.layout == WINO_NHWC && !g.in_u8 && !k2f_legacy()
                                         ? wino::launch_input_transform_f4(g, x, n0, imgs, vimg, s)
                                         : wino::launch_input_transform_f(g, x, n0, imgs, vimg, s))
                                  : wino::launch_input_transform(g, x, n0, imgs, vimg, s);
  if (g.path == 0) {
    if (stage == 3)
      e = g.alg == 1 ? wino::launch_fused2(g, tiles_pad, n0, imgs, vimg, static_cast<const int8_t*>(w_wino), codes,
                                           rq_mult, rq_shift, y, s)
                     : wino::launch_fused(g, tiles_pad, n0, imgs, vimg, static_cast<const int8_t*>(w_wino), codes,
                                          rq_mult, rq_shift, y, s);
  } else {
    if (stage == 3) e = wino::launch_gemm(g, tiles_pad, vimg, static_cast<const int8_t*>(w_wino), codes, m, s);
    if (stage == 4) e = wino::launch_output_transform(g, m, n0, imgs, rq_mult, rq_shift, y, s);
  }
  return cuda_status(e);
}

static wino_status check_conv_args(const wino_plan_s* p, const int8_t* x, const void* w_wino, const uint8_t* codes,
                                   int32_t rq_mult, int rq_shift, void* y, void* workspace) {
  if (!p || !x || !w_wino || !codes || !y || !workspace) return WINO_ERR_INVALID_ARG;
  if (!aligned16(x) || !aligned16(w_wino) || !aligned16(y) || !aligned16(workspace)) return WINO_ERR_INVALID_ARG;
  if (p->g.out_mode == WINO_OUT_INT8 && (rq_mult < 1 || rq_shift < 0 || rq_shift > 62)) return WINO_ERR_RANGE;
  return check_device(p);
}

wino_status wino_conv2d_int8(wino_plan_t p, const int8_t* x, const void* w_wino, const uint8_t* codes,
                             int32_t rq_mult, int rq_shift, void* y, void* workspace, void* stream) {
  wino_status st = check_conv_args(p, x, w_wino, codes, rq_mult, rq_shift, y, workspace);
  if (st != WINO_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!codes_known_valid(p, codes)) {   // first use of this code buffer: synchronous check (wino.h)
    st = validate_codes(p, codes, workspace, s);
    if (st != WINO_OK) return st;
  }
  const int last = p->g.path == 0 ? 3 : 4;
  if (p->lanes <= 1) {
    for (int c = 0; c < p->n_chunks; c++)
      for (int stage = 2; stage <= last; stage++) {
        st = run_stage(p, stage, c, x, w_wino, codes, rq_mult, rq_shift, y, workspace, s);
        if (st != WINO_OK) return st;
      }
    return WINO_OK;
  }
  // chunk pipelines: lane k runs chunks k, k + lanes, ... in order on its stream (its V buffer is reused,
  // each chunk's K2 waits for the lane's previous GEMM through stream order); lanes run concurrently, so
  // one chunk's input transform overlaps another's GEMM and the launch tails fill in
  std::lock_guard<std::mutex> lk(p->lane_mu);
  cudaError_t e = cudaSuccess;
  if (!p->lane_init) {
    e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming);
    for (int i = 1; i < p->lanes && e == cudaSuccess; i++) {
      e = cudaStreamCreateWithFlags(&p->aux[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_join[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_status(e);
    p->lane_init = true;
  }
  e = cudaEventRecord(p->ev_fork, s);
  for (int i = 1; i < p->lanes && e == cudaSuccess; i++) e = cudaStreamWaitEvent(p->aux[i], p->ev_fork, 0);
  if (e != cudaSuccess) return cuda_status(e);
  for (int c = 0; c < p->n_chunks; c++) {
    const int lane = c % p->lanes;
    cudaStream_t ls = lane == 0 ? s : p->aux[lane];
    for (int stage = 2; stage <= last; stage++) {
      st = run_stage(p, stage, c, x, w_wino, codes, rq_mult, rq_shift, y, workspace, ls);
      if (st != WINO_OK) return st;
    }
  }
  for (int i = 1; i < p->lanes && e == cudaSuccess; i++) {
    e = cudaEventRecord(p->ev_join[i], p->aux[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, p->ev_join[i], 0);
  }
  return cuda_status(e);
}

wino_status wino_conv2d_int8_stage(wino_plan_t p, int stage, int chunk, const int8_t* x, const void* w_wino,
                                   const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y, void* workspace,
                                   void* stream) {
  wino_status st = check_conv_args(p, x, w_wino, codes, rq_mult, rq_shift, y, workspace);
  if (st != WINO_OK) return st;
  const int last = p->g.path == 0 ? 3 : 4;
  if (stage < 2 || stage > last || chunk < 0 || chunk >= p->n_chunks) return WINO_ERR_INVALID_ARG;
  if (stage >= 3 && !codes_known_valid(p, codes)) {
    st = validate_codes(p, codes, workspace, static_cast<cudaStream_t>(stream));
    if (st != WINO_OK) return st;
  }
  return run_stage(p, stage, chunk, x, w_wino, codes, rq_mult, rq_shift, y, workspace,
                   static_cast<cudaStream_t>(stream));
}

wino_status wino_conv2d_int8_host(wino_plan_t p, const int8_t* x_host, const void* w_wino, const uint8_t* codes,
                                  int32_t rq_mult, int rq_shift, void* y_host, int8_t* x_dev, void* y_dev,
                                  void* workspace, void* stream) {
  if (!p || !x_host || !y_host || !x_dev || !y_dev) return WINO_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t ce = cudaMemcpyAsync(x_dev, x_host, p->x_bytes, cudaMemcpyHostToDevice, s);
  if (ce != cudaSuccess) return cuda_status(ce);
  wino_status st = wino_conv2d_int8(p, x_dev, w_wino, codes, rq_mult, rq_shift, y_dev, workspace, stream);
  if (st != WINO_OK) return st;
  ce = cudaMemcpyAsync(y_host, y_dev, p->y_bytes, cudaMemcpyDeviceToHost, s);
  if (ce != cudaSuccess) return cuda_status(ce);
  return WINO_OK;
}

wino_status wino_check_codes(wino_plan_t p, const uint8_t* codes, int32_t* bad_flag, void* stream) {
  if (!p || !codes || !bad_flag) return WINO_ERR_INVALID_ARG;
  wino_status st = check_device(p);
  if (st != WINO_OK) return st;
  return cuda_status(wino::launch_check_codes(codes, p->d.c_out * p->g.npos, p->g.w1, bad_flag,
                                              static_cast<cudaStream_t>(stream)));
}

wino_status wino_validate_codes(wino_plan_t p, const uint8_t* codes, void* workspace, void* stream) {
  if (!p || !codes || !workspace || !aligned16(workspace)) return WINO_ERR_INVALID_ARG;
  wino_status st = check_device(p);
  if (st != WINO_OK) return st;
  return validate_codes(p, codes, workspace, static_cast<cudaStream_t>(stream));
}

int wino_debug_fastdiv(int n, int d) {
  if (n < 0 || d < 1) return -1;
  return wino::fdiv(n, wino::make_fastdiv(d));
}

wino_status wino_debug_set_trace(void* device_buffer) {
  wino::set_gemm_trace(device_buffer);
  wino::set_fused_trace(device_buffer);
  return WINO_OK;
}

wino_status wino_maxpool2_int8(const int8_t* x, int n, int h, int w, int c, int layout, int8_t* y, void* stream) {
  if (!x || !y || n < 1 || h < 2 || w < 2 || c < 1) return WINO_ERR_INVALID_ARG;
  if (layout != WINO_NCHW && layout != WINO_NHWC) return WINO_ERR_INVALID_ARG;
  return cuda_status(wino::launch_maxpool2(x, n, h, w, c, layout, y, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
