// conv_tc.cu -- tcgen05 / TMEM / TMA TF32 convolution kernels (sm_100a).
// (placeholder until the tensor-core path lands: every entry declines.)
#include "ck_handle.hpp"

namespace ck {
bool conv_tc_available() { return false; }
bool conv_tc_forward(ck_handle*, const float*, const float*, const float*, float*,
                     const ConvDims&, int, cudaStream_t) { return false; }
bool conv_tc_dgrad(ck_handle*, const float*, const float*, float*, const ConvDims&, int,
                   cudaStream_t) { return false; }
bool conv_tc_wgrad(ck_handle*, const float*, const float*, float*, const ConvDims&, int,
                   cudaStream_t) { return false; }
void conv_tc_release(ck_handle*) {}
}  // namespace ck
