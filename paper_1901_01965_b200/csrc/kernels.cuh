// kernels.cuh -- launchers of the four hot-path kernels (internal to libwino).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "layout.cuh"

namespace wino {

// K1: filter transform + scaling + operand planes (k_filter.cu)
cudaError_t setup_filter_transform();
cudaError_t launch_filter_transform(const Geom& g, const int8_t* w, int8_t* wimg, uint8_t* codes, cudaStream_t st);

// K2: input gather + B^T d B + operand planes (k_input.cu)
//   x: whole input tensor; images [n0, n0 + imgs) form the chunk.
cudaError_t setup_input_transform();
cudaError_t launch_input_transform(const Geom& g, const int8_t* x, int n0, int imgs, int8_t* vimg, cudaStream_t st);

// K3: 46 Winograd-domain int8 GEMMs on tcgen05 -> raw per-plane M (k_gemm.cu)
cudaError_t setup_gemm();
cudaError_t launch_gemm(const Geom& g, long long tiles_pad_launch, const int8_t* vimg, const int8_t* wimg,
                        int32_t* mraw, cudaStream_t st);

void set_gemm_trace(void* buf);   // debug timeline buffer (nullptr = off)

// K4: Karatsuba + reverse scaling + A^T M'' A + /16 + requant + store (k_output.cu)
cudaError_t setup_output_transform();
cudaError_t launch_output_transform(const Geom& g, const int32_t* mraw, const uint8_t* codes, int n0, int imgs,
                                    int32_t rq_mult, int rq_shift, void* y, cudaStream_t st);

// misc (k_misc.cu)
cudaError_t launch_check_codes(const uint8_t* codes, int count, int32_t* bad, cudaStream_t st);
cudaError_t launch_maxpool2(const int8_t* x, int n, int h, int w, int c, int layout, int8_t* y, cudaStream_t st);

}  // namespace wino
