// Internal launch API of the coarse-level-staging dense FAST kernel
// (msda_dense_slice.cu).
#pragma once
#include "msda_common.cuh"

namespace msda {

bool plan_slice(const int32_t* shape_host, int cams, int L, int C, int esz, int G, int& VEC, int& first_staged,
                int* staged_off, int& stage_bytes);
cudaError_t launch_dense_slice(const msda_features_t& f, int Q, int P, int G, const float* loc, const float* w,
                               bool project, const float* anchors, const float* offsets, const msda_cameras_t* cams,
                               const float* strides, float dt, bool h2, bool normalize, float* out, DevStatus* st,
                               int VEC, int first_staged, const int* staged_off, int stage_bytes, int num_sms,
                               cudaStream_t s);

}  // namespace msda
