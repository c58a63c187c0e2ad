// Internal launch API of the exact CSR path (msda_exact.cu).
#pragma once
#include "msda_common.cuh"

namespace msda {

struct ExactWorkspace {
  DevStatus* status;
  SampleRec* rec;
  float* wn;
  unsigned long long* g_hi;
  unsigned long long* g_lo;
  int32_t* g_idx;
  float* qsum;  // [n_queries] per-query weight sums written by the plan
};

size_t exact_workspace_bytes(int64_t n_queries, int64_t n_samples);
cudaError_t reset_exact_workspace(const ExactWorkspace& w, cudaStream_t stream);
ExactWorkspace carve_exact_workspace(void* ws, int64_t n_samples);
cudaError_t launch_plan_canon(const msda_features_t& f, const msda_csr_plan_t& p, int normalize,
                              const ExactWorkspace& w, int num_sms, cudaStream_t stream,
                              int64_t queries_per_batch = 0);
cudaError_t launch_gather_exact(const msda_features_t& f, const msda_csr_plan_t& p, int precision,
                                const ExactWorkspace& w, float* out, uint8_t* empty, cudaStream_t stream,
                                int c_off = 0, int c_count = 0, int fast_normalize = -1, int n_groups = 1,
                                int normalize = 1);
// FAST on the CSR plan: one gather launch straight from the raw plan arrays
// (fast_normalize = normalize flag); cudaErrorNotSupported when the channel
// slice does not span whole warps (the caller then runs the exact stages).
inline cudaError_t launch_csr_fast(const msda_features_t& f, const msda_csr_plan_t& p, int normalize,
                                   const ExactWorkspace& w, float* out, uint8_t* empty, cudaStream_t stream) {
  return launch_gather_exact(f, p, MSDA_FAST, w, out, empty, stream, 0, 0, normalize ? 1 : 0);
}

// FAST on the dense Sparse4D layout through the pipelined gather (records
// built from the sampling locations on the fly, no plan pass).
// cudaErrorNotSupported when the shape does not fit (G > 8, a lane's channels
// straddling groups, misalignment): the caller then uses its own kernel.
struct DenseFastSpec {
  const float* loc;  // [batch * Q, P, cams, 2]
  const float* w;    // [batch * Q, P, cams, L, G]
  int32_t Q, P, G, normalize;
  float* wsum_out;      // [batch * Q, G] or null
  float* wsum_scratch;  // [batch * Q, G] device scratch for split normalisation
  bool h2;              // FAST_H2: half2 accumulation per camera (f16 storage; other dtypes ignore it)
  const float2* proj_cell = nullptr;  // fused projection: cells [batch * Q, P, cams, L] (NaN: behind), or null
  int32_t n_lv = 0;        // gather only levels [0, n_lv) (0: all)
  bool accumulate = false;  // out / wsum are zeroed by the caller: always red.add, the caller normalises
  bool prezeroed = false;   // out / wsum already zeroed by the caller (a camera split needs no memsets)
};
// *normalize_pending: the cameras were split across warps and out holds
// unnormalised sums; the caller divides by wsum (out or scratch) per group.
cudaError_t launch_gather_dense_fast(const msda_features_t& f, const DenseFastSpec& d, DevStatus* status, float* out,
                                     cudaStream_t stream, bool* normalize_pending);

// Coarse levels of the dense FAST call from on-chip staged maps
// (msda_staged.cu).  dense_staged_fine_levels: the number of leading (fine)
// levels left to the gather when the split applies to this shape (the
// trailing levels of every camera fit the stage budget), else -1.
// launch_dense_coarse red.add's the coarse levels' partial sums into the
// zeroed out / wsum.
int dense_staged_fine_levels(const msda_features_t& f, int G, int P);
cudaError_t launch_dense_coarse(const msda_features_t& f, const DenseFastSpec& d, int n_fine, float* out,
                                float* wsum, cudaStream_t stream);

// Dense EXACT without normalisation in one pass: the gather warp ranks each
// (camera, level) run itself (msda_dense_exact.cu).  cudaErrorNotSupported
// when the shape does not fit (the caller takes the two-pass path).
// status: reset by the kernel (the call's only kernel; nothing reports into it)
cudaError_t launch_dense_exact_fused(const msda_features_t& f, const float* loc, const float* w, int Q, int P, int G,
                                     float* out, DevStatus* status, cudaStream_t stream);

}  // namespace msda
