// kernels.cuh -- launchers of the four hot-path kernels (internal to libwino).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "layout.cuh"

namespace wino {

// Launch with programmatic stream serialization (PDL): the kernel may start while
// the previous kernel in the stream finishes; it calls pdl_wait() before touching
// global memory the previous kernels produce or consume.
// Launch with programmatic dependent launch (the kernel calls pdl_wait before reading its
// predecessor's output) and, if carveout >= 0, a preferred L1/shared-memory split (percent of the
// maximum shared memory).  Measured at C2 with three batches in flight next to the GEMM's ~210 KB of
// shared memory: K2/K4 at 0 (maximum L1) and K1 at 25 (room for its 2 resident CTAs) take the step
// from 146 to 159 TOPS and K1 from 3.7 to 3.1 us; the default preference re-splits the SMs between them.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_co(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 int carveout, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
  attr[1].val.sharedMemCarveout = carveout < 0 ? 0u : (unsigned)carveout;
  cfg.attrs = attr;
  cfg.numAttrs = carveout < 0 ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  return launch_pdl_co(kernel, grid, block, smem, st, -1, args...);
}
constexpr int kCarveL1 = 0, kCarveFilter = 25;

// Same with a 1-D thread-block cluster of `cluster` CTAs (grid.x a multiple of it).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// K1: filter transform + scaling + operand planes (k_filter.cu)
cudaError_t setup_filter_transform();
cudaError_t launch_filter_transform(const Geom& g, const int8_t* w, int8_t* wimg, uint8_t* codes, cudaStream_t st);

// K2: input gather + B^T d B + operand planes (k_input.cu)
//   x: whole input tensor; images [n0, n0 + imgs) form the chunk.
cudaError_t setup_input_transform();
cudaError_t launch_input_transform(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st);
//   fused-path V image (group layout, balanced pieces; layout.cuh)
cudaError_t launch_input_transform_f(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st);
// NHWC int8 input, 4 channels per thread in 16-bit SWAR lanes (k_input4.cu); same V image as the above
cudaError_t launch_input_transform_f4(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st);

// K3: 46 Winograd-domain int8 GEMMs on tcgen05 + Karatsuba + reverse scaling -> M'' (k_gemm.cu)
cudaError_t setup_gemm();
cudaError_t launch_gemm(const Geom& g, long long tiles_pad_launch, const int8_t* vimg, const int8_t* wimg,
                        const uint8_t* codes, int32_t* mpp, cudaStream_t st);

void set_gemm_trace(void* buf);   // debug timeline buffer (nullptr = off)

// K4: A^T M'' A + /16 + requant + store (k_output.cu)
cudaError_t setup_output_transform();
cudaError_t launch_output_transform(const Geom& g, const int32_t* mpp, int n0, int imgs, int32_t rq_mult,
                                    int rq_shift, void* y, cudaStream_t st);

// K3F: fused GEMMs + Karatsuba + reverse scaling + output transform + store (k_fused.cu);
//   requires g.nblk == 16.  V of the chunk -> y directly (no M'' in HBM).
// K3F2: fused rational F(2x2) GEMMs + reverse scaling + output transform + store (k_fused2.cu)
cudaError_t setup_fused2();
cudaError_t launch_fused2(const Geom& g, long long tiles_pad_launch, int n0, int imgs, const int8_t* vimg,
                          const int8_t* wimg, const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y,
                          cudaStream_t st);
cudaError_t setup_fused();
void set_fused_trace(void* buf);   // debug timeline (-DWINO_FUSED_TRACE), nullptr = off
cudaError_t launch_fused(const Geom& g, long long tiles_pad_launch, int n0, int imgs, const int8_t* vimg,
                         const int8_t* wimg, const uint8_t* codes, int32_t rq_mult, int rq_shift, void* y,
                         cudaStream_t st);

// misc (k_misc.cu)
cudaError_t launch_check_codes(const uint8_t* codes, int count, int code7, int32_t* bad, cudaStream_t st);
cudaError_t launch_maxpool2(const int8_t* x, int n, int h, int w, int c, int layout, int8_t* y, cudaStream_t st);

}  // namespace wino
