// Tracker association cost (tracker.py:105-142) — sm_100a.
//
// The consumer of the pooled embeddings: for every (query, detection) pair
//   geo  = |c_q - c_d|_2                      (3-vectors)
//   emb  = |m_q - e_d|_2                      (D-vectors, D = embedding dim)
//   admissible = geo <= gate_radius
//   cost = alpha_emb * emb + alpha_geo * geo / gate   (gate = 1 if not finite)
//   solver_cost = admissible ? cost : 1e9     (tracker.py:32, 126)
// in f64 with numpy's exact operation order: np.linalg.norm is
// sqrt(add.reduce(x * x)) and add.reduce on a contiguous float64 row is
// numpy's pairwise sum (sequential below 8 terms; 8 running partial sums
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail up to
// 128 terms; halves above that).  Every operation is separately rounded, so
// the matrices equal the reference's bit for bit; the Hungarian solve
// (scipy linear_sum_assignment) stays on the host.
//
// One thread per pair, 16 x 16 pairs per CTA (8 x 8 above D ~ 800); the
// CTA's query and detection embedding rows are staged in shared memory (rows
// padded to an even pitch with a 16-B bank skew; read two doubles at a time).
#include <algorithm>

#include "msda_common.cuh"

namespace msda {
namespace {

constexpr int kMaxDim = 1024;

struct AssocArgs {
  const double* qc;  // [n_q, 3]
  const double* dc;  // [n_d, 3]
  const double* qe;  // [n_q, D]
  const double* de;  // [n_d, D]
  int32_t n_q, n_d, D;
  double gate_radius, alpha_emb, alpha_geo;
  double* cost;         // [n_q, n_d]
  double* solver_cost;  // [n_q, n_d]
  uint8_t* admissible;  // [n_q, n_d]
};

__device__ __forceinline__ double sqdiff(const double* a, const double* b, int i) {
  const double d = __dsub_rn(a[i], b[i]);
  return __dmul_rn(d, d);
}

// numpy pairwise_sum of (a[i] - b[i])^2 over [0, n), n <= 128
__device__ double pairwise_block(const double* a, const double* b, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, i));
    return res;
  }
  // rows are 16-B aligned: two doubles per shared-memory load
  auto sq8 = [&](int i0, double* v) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const double2 x = *reinterpret_cast<const double2*>(a + i0 + j);
      const double2 y = *reinterpret_cast<const double2*>(b + i0 + j);
      const double d0 = __dsub_rn(x.x, y.x), d1 = __dsub_rn(x.y, y.y);
      v[j] = __dmul_rn(d0, d0);
      v[j + 1] = __dmul_rn(d1, d1);
    }
  };
  double r[8];
  sq8(0, r);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    double t[8];
    sq8(i, t);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], t[j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, i));
  return res;
}

// the recursive halving above 128 terms, unrolled as an explicit stack
__device__ double pairwise_sum_sq(const double* a, const double* b, int n) {
  if (n <= 128) return pairwise_block(a, b, n);
  if (n <= 256) {  // one halving, both halves <= 128: no stack (stays in registers)
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pairwise_block(a, b, n2), pairwise_block(a + n2, b + n2, n - n2));
  }
  // leaves in left-to-right order, combined bottom-up exactly like the recursion
  struct Node {
    int off, n, state;
    double left;
  };
  Node st[16];
  int sp = 0;
  st[sp++] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (sp > 0) {
    Node& nd = st[sp - 1];
    if (nd.n <= 128) {
      ret = pairwise_block(a + nd.off, b + nd.off, nd.n);
      --sp;
      continue;
    }
    int n2 = nd.n / 2;
    n2 -= n2 % 8;
    if (nd.state == 0) {  // descend left
      nd.state = 1;
      st[sp++] = {nd.off, n2, 0, 0.0};
    } else if (nd.state == 1) {  // left done: descend right
      nd.left = ret;
      nd.state = 2;
      st[sp++] = {nd.off + n2, nd.n - n2, 0, 0.0};
    } else {  // both done
      ret = __dadd_rn(nd.left, ret);
      --sp;
    }
  }
  return ret;
}

template <int kTile>
__global__ void __launch_bounds__(kTile * kTile) assoc_cost_kernel(AssocArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int pitch = a.D + 2 + (a.D & 1);  // even (16-B aligned rows), 16 B of bank skew per row
  double* s_q = sm;
  double* s_d = sm + kTile * pitch;
  const int q0 = blockIdx.y * kTile, d0 = blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile * a.D; i += blockDim.x) {
    const int r = i / a.D, k = i - r * a.D;
    if (q0 + r < a.n_q) s_q[r * pitch + k] = a.qe[(int64_t)(q0 + r) * a.D + k];
    if (d0 + r < a.n_d) s_d[r * pitch + k] = a.de[(int64_t)(d0 + r) * a.D + k];
  }
  __syncthreads();
  const int ti = threadIdx.x / kTile, tj = threadIdx.x % kTile;
  const int q = q0 + ti, d = d0 + tj;
  if (q >= a.n_q || d >= a.n_d) return;
  const double* qc = a.qc + (int64_t)q * 3;
  const double* dc = a.dc + (int64_t)d * 3;
  const double geo = __dsqrt_rn(__dadd_rn(__dadd_rn(sqdiff(qc, dc, 0), sqdiff(qc, dc, 1)), sqdiff(qc, dc, 2)));
  const double emb = __dsqrt_rn(pairwise_sum_sq(s_q + ti * pitch, s_d + tj * pitch, a.D));
  const bool adm = geo <= a.gate_radius;
  const double gate = isfinite(a.gate_radius) ? a.gate_radius : 1.0;
  const double cost = __dadd_rn(__dmul_rn(a.alpha_emb, emb), __ddiv_rn(__dmul_rn(a.alpha_geo, geo), gate));
  const int64_t o = (int64_t)q * a.n_d + d;
  a.cost[o] = cost;
  a.solver_cost[o] = adm ? cost : 1e9;
  a.admissible[o] = adm ? 1 : 0;
}

}  // namespace
}  // namespace msda

using namespace msda;

extern "C" {

int32_t msda_assoc_cost(const double* q_centers, const double* d_centers, const double* q_embeddings,
                        const double* d_embeddings, int32_t n_q, int32_t n_d, int32_t dim, double gate_radius,
                        double alpha_emb, double alpha_geo, double* cost, double* solver_cost, uint8_t* admissible,
                        void* stream) {
  if (n_q < 0 || n_d < 0 || dim <= 0 || dim > kMaxDim) return MSDA_BAD_ARG;
  if (n_q == 0 || n_d == 0) return MSDA_OK;
  if (!q_centers || !d_centers || !q_embeddings || !d_embeddings || !cost || !solver_cost || !admissible)
    return MSDA_BAD_ARG;
  if (gate_radius != gate_radius) return MSDA_BAD_ARG;  // NaN gate
  AssocArgs a{q_centers, d_centers, q_embeddings, d_embeddings, n_q,  n_d,        dim,       gate_radius,
              alpha_emb, alpha_geo, cost,         solver_cost,  admissible};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // 16 x 16 pairs per CTA while both 16-row tiles fit in shared memory, else 8 x 8
  const int pitch = dim + 2 + (dim & 1);
  const size_t smem16 = 2 * (size_t)16 * pitch * sizeof(double);
  if (smem16 <= 200 * 1024) {
    if (smem16 > 48 * 1024 && cudaFuncSetAttribute(assoc_cost_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem16) != cudaSuccess)
      return MSDA_CUDA_ERROR;
    const dim3 grid((unsigned)((n_d + 15) / 16), (unsigned)((n_q + 15) / 16));
    assoc_cost_kernel<16><<<grid, 256, smem16, s>>>(a);
  } else {
    const size_t smem8 = 2 * (size_t)8 * pitch * sizeof(double);
    if (cudaFuncSetAttribute(assoc_cost_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8) !=
        cudaSuccess)
      return MSDA_CUDA_ERROR;
    const dim3 grid((unsigned)((n_d + 7) / 8), (unsigned)((n_q + 7) / 8));
    assoc_cost_kernel<8><<<grid, 64, smem8, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

}  // extern "C"
