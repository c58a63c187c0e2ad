// Placeholder entry points (replaced by the dense / projection / OAE kernels).
#include "msda_common.cuh"
extern "C" {
size_t msda_dense_workspace_size(int32_t, int32_t, int32_t, int32_t, int32_t, int32_t, int32_t) { return 256; }
int32_t msda_dense(const msda_features_t*, int32_t, int32_t, int32_t, const float*, const float*, int32_t, int32_t, float*, void*, size_t, void*) { return MSDA_BAD_ARG; }
int32_t msda_dense_project(const msda_features_t*, int32_t, const float*, int32_t, const float*, const msda_cameras_t*, const float*, float, int32_t, const float*, int32_t, float*, void*, size_t, void*) { return MSDA_BAD_ARG; }
int32_t msda_oae_pool(const msda_features_t*, int32_t, const float*, int32_t, const float*, const msda_cameras_t*, const float*, const float*, const float*, const float*, float*, uint8_t*, void*, size_t, void*) { return MSDA_BAD_ARG; }
size_t msda_oae_workspace_size(int32_t, int32_t, int32_t) { return 256; }
}
