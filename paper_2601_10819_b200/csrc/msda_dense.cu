// Dense Sparse4D-layout MSDA (deformable_aggregation) and the fused
// keypoint-projection variant — sm_100a.
//
// FAST mode (the throughput path): one CTA per (batch, anchor).  The CTA
// walks the anchor's P x cams x L samples in chunks of kChunk:
//   phase A  all threads build the chunk's 32-B SampleRecs (bilinear corner
//            rows + f32 interpolation weights; cell = loc*W - 0.5, the
//            reference convention features.py:20-24) and stage the chunk's
//            [kChunk, G] group weights in shared memory with coalesced loads.
//            In PROJECT mode the sample location comes from the anchor's
//            keypoints (geometry.py:207-255) projected through the camera
//            (geometry.py:162-182, f64), behind-camera samples get weight 0.
//   phase B  the CTA is split into n_split sub-groups of C/VEC lanes; each
//            sub-group takes every n_split-th sample, gathers the four
//            corner rows with 16-B loads (channel-last rows, full 32-B
//            sectors) and FMAs them into f32 accumulators with the combined
//            weights iw_k * w_g.
// A shared-memory reduction over the sub-groups and the optional
// per-(anchor, group) renormalisation finish the anchor.
//
// EXACT mode expands the dense inputs into one CSR plan per channel group and
// runs the bit-faithful CSR kernels (msda_exact.cu) on that channel slice.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "msda_common.cuh"
#include "msda_exact.cuh"

namespace msda {
namespace {

constexpr int kDenseThreads = 256;
constexpr int kChunk = 128;
constexpr int kMaxGroups = 32;
constexpr int kMaxPoints = 64;

struct DenseArgs {
  const void* feat;
  int64_t n_rows;  // rows per batch item
  int32_t C, bs, Q, P, cams, L, G;
  const int32_t* shape;
  const int64_t* start;
  const float* loc;  // [bs, Q, P, cams, 2]            (LOC mode)
  const float* w;    // [bs, Q, P, cams, L, G]
  int32_t normalize;
  float* out;        // [bs, Q, C]
  float* wsum_out;   // [bs, Q, G] per-(anchor, group) weight sums, or null (camera-sharded partials)
  DevStatus* status;
  // PROJECT mode
  const float* anchors;  // [bs, Q, 10]
  int32_t n_learned;
  const float* offsets;  // [n_learned, 3]
  const double* K;       // [cams, 4]
  const double* R;       // [cams, 9]
  const double* T;       // [cams, 3]
  const float* strides;  // [L]
  float dt;
};

// Keypoints of one anchor into shared memory (P x 3 doubles).
__device__ void anchor_keypoints(const DenseArgs& a, int64_t bq, double* kp, DevStatus* st) {
  for (int p = threadIdx.x; p < a.P; p += blockDim.x)
    if (!anchor_keypoint(a.anchors + bq * 10, p, a.offsets, a.dt, kp + 3 * p)) set_status(st, MSDA_OFFSET_RANGE, p);
}

__device__ __forceinline__ bool project_point(const DenseArgs& a, int cam, const double* p, double& u, double& v) {
  return project_f64(a.K + cam * 4, a.R + cam * 9, a.T + cam * 3, p, u, v);
}

template <typename T, int VEC, bool PROJECT>
__global__ void __launch_bounds__(kDenseThreads) dense_fast_kernel(DenseArgs a) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  __shared__ SampleRec s_rec[kChunk];
  __shared__ float s_w[kChunk * kMaxGroups];
  __shared__ float s_red[kDenseThreads * VEC];
  __shared__ float s_wsum[kDenseThreads / 2 * 2];
  __shared__ double s_kp[PROJECT ? kMaxPoints * 3 : 1];

  const int64_t bq = blockIdx.x;  // flattened (batch, anchor)
  const int b = (int)(bq / a.Q);
  const int S = a.P * a.cams * a.L;
  const int lpr = a.C / VEC;                  // lanes per feature row
  const int n_split = kDenseThreads / lpr;    // sample sub-groups
  const int sub = threadIdx.x / lpr;
  const int lane = threadIdx.x - sub * lpr;
  const bool active = sub < n_split;
  const int c0 = lane * VEC;
  const int cpg = a.C / a.G;
  const int g = c0 / cpg;
  const bool group_head = (c0 % cpg) == 0;
  const int64_t row_base = (int64_t)b * a.n_rows;
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)c0 * sizeof(T);
  const size_t row_bytes = (size_t)a.C * sizeof(T);
  const float* wq = a.w + bq * (int64_t)S * a.G;

  if constexpr (PROJECT) {
    anchor_keypoints(a, bq, s_kp, a.status);
    __syncthreads();
  }

  float acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;
  float wsum = 0.0f;

  for (int base = 0; base < S; base += kChunk) {
    const int n = min(kChunk, S - base);
    // ---- phase A: records + staged group weights ----
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int s = base + i;
      const int l = s % a.L;
      const int pc = s / a.L;
      const int cam = pc % a.cams;
      const int p = pc / a.cams;
      const int t = cam * a.L + l;
      const int H = a.shape[2 * t], W = a.shape[2 * t + 1];
      float u, v;
      bool valid = true;
      if constexpr (PROJECT) {
        double up, vp;
        valid = project_point(a, cam, s_kp + 3 * p, up, vp);
        const double st = (double)a.strides[l];
        u = valid ? (float)(up / st - 0.5) : -4.0f;
        v = valid ? (float)(vp / st - 0.5) : -4.0f;
      } else {
        const float* lp = a.loc + ((bq * a.P + p) * a.cams + cam) * 2;
        u = __fsub_rn(__fmul_rn(lp[0], (float)W), 0.5f);
        v = __fsub_rn(__fmul_rn(lp[1], (float)H), 0.5f);
      }
      SampleRec r = make_record(u, v, row_base + a.start[t], H, W);
      if (!valid) r.iw[0] = r.iw[1] = r.iw[2] = r.iw[3] = 0.0f;
      s_rec[i] = r;
    }
    for (int j = threadIdx.x; j < n * a.G; j += blockDim.x) s_w[j] = __ldg(wq + (int64_t)base * a.G + j);
    __syncthreads();
    if constexpr (PROJECT) {  // behind-camera samples leave the plan: zero weight
      for (int j = threadIdx.x; j < n * a.G; j += blockDim.x) {
        const SampleRec& r = s_rec[j / a.G];
        if (r.iw[0] == 0.0f && r.iw[1] == 0.0f && r.iw[2] == 0.0f && r.iw[3] == 0.0f) s_w[j] = 0.0f;
      }
      __syncthreads();
    }
    // ---- phase B: gather + FMA ----
    if (active) {
      int i = sub;
      for (; i + n_split < n; i += 2 * n_split) {
        const SampleRec r0 = s_rec[i], r1 = s_rec[i + n_split];
        const float w0 = s_w[i * a.G + g], w1 = s_w[(i + n_split) * a.G + g];
        RawVec<BYTES> c[2][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          c[0][k] = r0.row[k] >= 0 ? ldg_vec<BYTES>(feat + (size_t)r0.row[k] * row_bytes) : zero_vec<BYTES>();
          c[1][k] = r1.row[k] >= 0 ? ldg_vec<BYTES>(feat + (size_t)r1.row[k] * row_bytes) : zero_vec<BYTES>();
        }
        wsum += w0 + w1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float f0[VEC], f1[VEC];
          to_f32<T, VEC>(c[0][k], f0);
          to_f32<T, VEC>(c[1][k], f1);
          const float cw0 = r0.iw[k] * w0, cw1 = r1.iw[k] * w1;
#pragma unroll
          for (int e = 0; e < VEC; e += 2) {  // FFMA2: two channels per instruction
            float2 p = __ffma2_rn(make_float2(f0[e], f0[e + 1]), make_float2(cw0, cw0),
                                  make_float2(acc[e], acc[e + 1]));
            p = __ffma2_rn(make_float2(f1[e], f1[e + 1]), make_float2(cw1, cw1), p);
            acc[e] = p.x;
            acc[e + 1] = p.y;
          }
        }
      }
      for (; i < n; i += n_split) {
        const SampleRec r0 = s_rec[i];
        const float w0 = s_w[i * a.G + g];
        wsum += w0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (r0.row[k] < 0) continue;
          float f0[VEC];
          to_f32<T, VEC>(ldg_vec<BYTES>(feat + (size_t)r0.row[k] * row_bytes), f0);
          const float cw0 = r0.iw[k] * w0;
#pragma unroll
          for (int e = 0; e < VEC; e += 2) {
            const float2 p = __ffma2_rn(make_float2(f0[e], f0[e + 1]), make_float2(cw0, cw0),
                                        make_float2(acc[e], acc[e + 1]));
            acc[e] = p.x;
            acc[e + 1] = p.y;
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- reduce sub-groups, renormalise, write ----
  if (active) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) s_red[sub * a.C + c0 + e] = acc[e];
    if (group_head) s_wsum[sub * a.G + g] = wsum;
  }
  __syncthreads();
  float* o = a.out + bq * a.C;
  for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
    float sum = 0.0f;
    for (int j = 0; j < n_split; ++j) sum += s_red[j * a.C + c];
    if (a.normalize || a.wsum_out) {
      const int gg = c / cpg;
      float ws = 0.0f;
      for (int j = 0; j < n_split; ++j) ws += s_wsum[j * a.G + gg];
      if (a.wsum_out && c == gg * cpg) a.wsum_out[bq * a.G + gg] = ws;
      if (a.normalize) {
        if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, bq);
        sum = sum / ws;
      }
    }
    o[c] = sum;
  }
}

// ---------------------------------------------------------------------------
// FAST, production shape (C == 32 * VEC): one CTA of kWcWarps warps per
// anchor; warp w aggregates cameras w, w + kWcWarps, ... in camera-major,
// level-minor order, so all resident anchors sweep the cameras in lockstep and
// the live working set is a few cameras' maps (L2-resident): each touched cell
// comes from HBM about once.  Per camera, lanes build 32 sample records and
// stage the group weights in warp-private shared memory (__syncwarp only, no
// CTA barrier), then the whole warp gathers each sample's four corner rows
// (lane = VEC channels, 16/32-B vector loads, full sectors) and FMAs them with
// iw_k * w_g: FFMA2 in f32, or HFMA2 into a per-camera half2 partial that is
// flushed to f32 after every camera (HACC, f16 storage; the paper's half2
// accumulation, bounded to 52-sample runs).

constexpr int kWcWarps = 4;
constexpr int kWcMaxGroups = 32;

template <typename T, int VEC, bool PROJECT, bool HACC>
__global__ void __launch_bounds__(kWcWarps * 32) dense_warpcam_kernel(DenseArgs a) {
  constexpr int NV = VEC * (int)sizeof(T) / 16;
  static_assert(NV >= 1 && NV * 16 == VEC * (int)sizeof(T), "16-B multiples");
  __shared__ SampleRec s_rec[kWcWarps][32];
  __shared__ float s_w[kWcWarps][32 * kWcMaxGroups];
  __shared__ float s_red[kWcWarps][32 * VEC];
  __shared__ float s_ws[kWcWarps][kWcMaxGroups];
  __shared__ double s_kp[PROJECT ? kMaxPoints * 3 : 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bq = blockIdx.x;
  const int b = (int)(bq / a.Q);
  const int G = a.G;
  const int cpg = a.C / G;
  const int c0 = lane * VEC;
  const int g = c0 / cpg;
  const bool group_head = (c0 % cpg) == 0;
  const int64_t row_base = (int64_t)b * a.n_rows;
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)c0 * sizeof(T);
  const uint32_t row_bytes = (uint32_t)(a.C * (int)sizeof(T));
  const int n_cs = a.P * a.L;  // samples per camera

  if constexpr (PROJECT) {
    anchor_keypoints(a, bq, s_kp, a.status);
    __syncthreads();
  }

  float acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;
  float wsum = 0.0f;

  for (int cam = warp; cam < a.cams; cam += kWcWarps) {
    __half2 hacc[VEC / 2];
    if constexpr (HACC) {
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) hacc[e] = __float2half2_rn(0.0f);
    }
    for (int base = 0; base < n_cs; base += 32) {
      const int n = min(32, n_cs - base);
      if (lane < n) {
        const int s = base + lane;
        const int l = s / a.P, p = s - l * a.P;
        const int t = cam * a.L + l;
        const int H = a.shape[2 * t], W = a.shape[2 * t + 1];
        float u, v;
        bool valid = true;
        if constexpr (PROJECT) {
          double up, vp;
          valid = project_point(a, cam, s_kp + 3 * p, up, vp);
          const double st = (double)a.strides[l];
          u = valid ? (float)(up / st - 0.5) : -4.0f;
          v = valid ? (float)(vp / st - 0.5) : -4.0f;
        } else {
          const float* lp = a.loc + ((bq * a.P + p) * a.cams + cam) * 2;
          u = __fsub_rn(__fmul_rn(lp[0], (float)W), 0.5f);
          v = __fsub_rn(__fmul_rn(lp[1], (float)H), 0.5f);
        }
        s_rec[warp][lane] = make_record(u, v, row_base + a.start[t], H, W);
        const float* wp = a.w + (((bq * a.P + p) * a.cams + cam) * a.L + l) * (int64_t)G;
        for (int gg = 0; gg < G; ++gg) s_w[warp][lane * G + gg] = valid ? __ldg(wp + gg) : 0.0f;
      }
      __syncwarp();
      for (int i = 0; i < n; i += 2) {
        const bool two = i + 1 < n;
        const SampleRec r0 = s_rec[warp][i];
        const SampleRec r1 = s_rec[warp][two ? i + 1 : i];
        const float w0 = s_w[warp][i * G + g];
        const float w1 = two ? s_w[warp][(i + 1) * G + g] : 0.0f;
        Row<NV> c[2][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (r0.row[k] >= 0) c[0][k] = ld_row<NV>(feat + (size_t)r0.row[k] * row_bytes);
          else
#pragma unroll
            for (int j = 0; j < NV; ++j) c[0][k].v[j] = make_uint4(0, 0, 0, 0);
          if (two && r1.row[k] >= 0) c[1][k] = ld_row<NV>(feat + (size_t)r1.row[k] * row_bytes);
          else
#pragma unroll
            for (int j = 0; j < NV; ++j) c[1][k].v[j] = make_uint4(0, 0, 0, 0);
        }
        wsum += w0 + w1;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const SampleRec& r = j ? r1 : r0;
          const float wg = j ? w1 : w0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float cw = r.iw[k] * wg;
            const uint32_t* raw = reinterpret_cast<const uint32_t*>(c[j][k].v);
            if constexpr (HACC) {
              const __half2 cwh = __float2half2_rn(cw);
#pragma unroll
              for (int e = 0; e < VEC / 2; ++e)
                hacc[e] = __hfma2(*reinterpret_cast<const __half2*>(&raw[e]), cwh, hacc[e]);
            } else {
              float f[VEC];
              raw_to_f32<T, VEC>(raw, f);
#pragma unroll
              for (int e = 0; e < VEC; e += 2) {
                const float2 pr = __ffma2_rn(make_float2(f[e], f[e + 1]), make_float2(cw, cw),
                                             make_float2(acc[e], acc[e + 1]));
                acc[e] = pr.x;
                acc[e + 1] = pr.y;
              }
            }
          }
        }
      }
      __syncwarp();
    }
    if constexpr (HACC) {
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        const float2 f = __half22float2(hacc[e]);
        acc[2 * e] += f.x;
        acc[2 * e + 1] += f.y;
      }
    }
  }

#pragma unroll
  for (int e = 0; e < VEC; ++e) s_red[warp][c0 + e] = acc[e];
  if (group_head) s_ws[warp][g] = wsum;
  __syncthreads();
  float* o = a.out + bq * a.C;
  for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
    float sum = 0.0f;
#pragma unroll
    for (int j = 0; j < kWcWarps; ++j) sum += s_red[j][c];
    if (a.normalize || a.wsum_out) {
      const int gg = c / cpg;
      float ws = 0.0f;
#pragma unroll
      for (int j = 0; j < kWcWarps; ++j) ws += s_ws[j][gg];
      if (a.wsum_out && c == gg * cpg) a.wsum_out[bq * a.G + gg] = ws;
      if (a.normalize) {
        if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, bq);
        sum = sum / ws;
      }
    }
    o[c] = sum;
  }
}

template <typename T, int VEC, bool PROJECT, bool HACC>
cudaError_t launch_warpcam(const DenseArgs& a, cudaStream_t s) {
  const int64_t grid = (int64_t)a.bs * a.Q;
  if (grid == 0) return cudaSuccess;
  dense_warpcam_kernel<T, VEC, PROJECT, HACC><<<(unsigned)grid, kWcWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int VEC, bool PROJECT>
cudaError_t launch_dense_fast_t(const DenseArgs& a, cudaStream_t s) {
  const int64_t grid = (int64_t)a.bs * a.Q;
  if (grid == 0) return cudaSuccess;
  dense_fast_kernel<T, VEC, PROJECT><<<(unsigned)grid, kDenseThreads, 0, s>>>(a);
  return cudaGetLastError();
}

template <bool PROJECT>
cudaError_t launch_dense_fast(const DenseArgs& a, int dtype, bool h2, cudaStream_t s) {
  const int cpg = a.C / a.G;
  const auto fits = [&](int vec) { return a.C % vec == 0 && cpg % vec == 0 && a.C / vec <= kDenseThreads; };
  const uintptr_t al = reinterpret_cast<uintptr_t>(a.feat);
  const auto warpcam = [&](int vec, int esz) {
    return a.C == 32 * vec && cpg % vec == 0 && a.G <= kWcMaxGroups && al % 16 == 0 && (a.C * esz) % 16 == 0;
  };
  switch (dtype) {
    case MSDA_F32:
      if (warpcam(8, 4)) return launch_warpcam<float, 8, PROJECT, false>(a, s);
      if (warpcam(4, 4)) return launch_warpcam<float, 4, PROJECT, false>(a, s);
      break;
    case MSDA_F16:
      if (warpcam(8, 2) && h2) return launch_warpcam<__half, 8, PROJECT, true>(a, s);
      if (warpcam(8, 2)) return launch_warpcam<__half, 8, PROJECT, false>(a, s);
      break;
    default:
      if (warpcam(8, 2)) return launch_warpcam<__nv_bfloat16, 8, PROJECT, false>(a, s);
      break;
  }
  switch (dtype) {
    case MSDA_F32:
      if (fits(4)) return launch_dense_fast_t<float, 4, PROJECT>(a, s);
      return launch_dense_fast_t<float, 2, PROJECT>(a, s);
    case MSDA_F16:
      if (fits(8)) return launch_dense_fast_t<__half, 8, PROJECT>(a, s);
      if (fits(4)) return launch_dense_fast_t<__half, 4, PROJECT>(a, s);
      return launch_dense_fast_t<__half, 2, PROJECT>(a, s);
    default:
      if (fits(8)) return launch_dense_fast_t<__nv_bfloat16, 8, PROJECT>(a, s);
      if (fits(4)) return launch_dense_fast_t<__nv_bfloat16, 4, PROJECT>(a, s);
      return launch_dense_fast_t<__nv_bfloat16, 2, PROJECT>(a, s);
  }
}

// ---------------------------------------------------------------------------
// EXACT: dense -> CSR plan for one channel group

template <bool PROJECT>
__global__ void dense_expand_kernel(DenseArgs a, int group, int64_t* offsets, int32_t* cam_o, int32_t* lvl_o,
                                    float* u_o, float* v_o, float* w_o) {
  __shared__ double s_kp[PROJECT ? kMaxPoints * 3 : 1];
  const int S = a.P * a.cams * a.L;
  const int64_t bq = blockIdx.x;
  if constexpr (PROJECT) {
    anchor_keypoints(a, bq, s_kp, a.status);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offsets[bq] = bq * S;
    if (bq == (int64_t)a.bs * a.Q - 1) offsets[bq + 1] = (bq + 1) * S;
  }
  // emitted camera-major, level, point: already grouped by (camera, level),
  // so the canonicaliser takes its rank-within-run path
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int p = s % a.P;
    const int cl = s / a.P;
    const int l = cl % a.L;
    const int cam = cl / a.L;
    const int t = cam * a.L + l;
    const int64_t o = bq * S + s;
    const int64_t wi = ((bq * a.P + p) * a.cams + cam) * a.L + l;
    float u, v, w = a.w[wi * a.G + group];
    if constexpr (PROJECT) {
      double up, vp;
      if (project_point(a, cam, s_kp + 3 * p, up, vp)) {
        const double st = (double)a.strides[l];
        u = (float)(up / st - 0.5);
        v = (float)(vp / st - 0.5);
      } else {  // behind the camera: a zero-weight, fully outside sample adds nothing
        u = v = -4.0f;
        w = 0.0f;
      }
    } else {
      const float* lp = a.loc + ((bq * a.P + p) * a.cams + cam) * 2;
      u = __fsub_rn(__fmul_rn(lp[0], (float)a.shape[2 * t + 1]), 0.5f);
      v = __fsub_rn(__fmul_rn(lp[1], (float)a.shape[2 * t]), 0.5f);
    }
    cam_o[o] = cam;
    lvl_o[o] = l;
    u_o[o] = u;
    v_o[o] = v;
    w_o[o] = w;
  }
}

// ---------------------------------------------------------------------------
// EXACT with channel groups in one pass.  The canonical order (camera, level,
// v, u, w; features.py:261-263) differs between groups only among samples
// whose (camera, level, v, u) tie — and tied samples share one bilinear
// record — so one canonicalisation serves every group: records are written
// once at the shared slot; each group's weight goes to its own slot, the
// tied ones ranked by that group's weight (then position).  Per-group
// sequential f32 weight sums (threads 0..G-1, in each group's canonical
// order) normalise in place, and one gather over all channels reads the
// lane's group weight: bit-identical to G separate plans.
// Samples are indexed i = (camera * L + level) * P + point, so the
// (camera, level) run of i is [i - i % P, i - i % P + P).

template <bool PROJECT>
__global__ void __launch_bounds__(128) dense_canon_kernel(DenseArgs a, SampleRec* rec, float* wn, int normalize) {
  extern __shared__ __align__(16) unsigned long long s_kp[];  // [n] (ord(v) << 32) | ord(u), then [n] valid bytes
  __shared__ double s_kpt[PROJECT ? kMaxPoints * 3 : 1];
  __shared__ float s_ws[kMaxGroups];
  const int n = a.P * a.cams * a.L;
  const int64_t bq = blockIdx.x;
  const int b = (int)(bq / a.Q);
  const int64_t lo = bq * n;
  const int G = a.G;
  const int64_t row_base = (int64_t)b * a.n_rows;
  unsigned char* s_valid = reinterpret_cast<unsigned char*>(s_kp + n);
  asm volatile("griddepcontrol.launch_dependents;");  // the gather may launch early (it waits for completion)
  if constexpr (PROJECT) {
    anchor_keypoints(a, bq, s_kpt, a.status);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int p = i % a.P, t = i / a.P, cam = t / a.L, l = t - cam * a.L;
    float u, v;
    bool valid = true;
    if constexpr (PROJECT) {
      double up, vp;
      valid = project_point(a, cam, s_kpt + 3 * p, up, vp);
      if (valid) {
        const double st = (double)a.strides[l];
        u = (float)(up / st - 0.5);
        v = (float)(vp / st - 0.5);
      } else {  // behind the camera: outside every grid and weight 0 (the plan keeps it, it adds nothing)
        u = v = -4.0f;
      }
    } else {
      const float* lp = a.loc + ((bq * a.P + p) * a.cams + cam) * 2;
      u = __fsub_rn(__fmul_rn(lp[0], (float)a.shape[2 * t + 1]), 0.5f);
      v = __fsub_rn(__fmul_rn(lp[1], (float)a.shape[2 * t]), 0.5f);
    }
    s_kp[i] = ((unsigned long long)ord_f32(v) << 32) | ord_f32(u);
    s_valid[i] = valid ? 1 : 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int p = i % a.P, t = i / a.P, cam = t / a.L, l = t - cam * a.L;
    const int r0 = i - p;
    const unsigned long long ki = s_kp[i];
    int below = 0;
    bool tie = false;
    for (int j = r0; j < r0 + a.P; ++j) {
      const unsigned long long kj = s_kp[j];
      below += kj < ki ? 1 : 0;
      tie |= (kj == ki) & (j != i);
    }
    const float u = unord_f32((uint32_t)(ki & 0xffffffffu)), v = unord_f32((uint32_t)(ki >> 32));
    const bool valid = s_valid[i] != 0;
    const int slot = r0 + below;  // first slot of this (v, u) value inside the run
    const float* wp = a.w + (((bq * a.P + p) * a.cams + cam) * a.L + l) * (int64_t)G;
    int eq_before = 0;  // rank among exact (v, u) ties by position: tied records are identical
    if (tie)
      for (int j = r0; j < i; ++j) eq_before += s_kp[j] == ki ? 1 : 0;
    rec[lo + slot + eq_before] = make_record(u, v, row_base + a.start[t], a.shape[2 * t], a.shape[2 * t + 1]);
    for (int g = 0; g < G; ++g) {
      const float wg = valid ? __ldg(wp + g) : 0.0f;
      int sg = slot;
      if (tie) {  // rank inside the tie by this group's weight, then position
        const uint32_t oi = ord_f32(wg);
        for (int j = r0; j < r0 + a.P; ++j) {
          if (j == i || s_kp[j] != ki) continue;
          const float* wpj = a.w + (((bq * a.P + (j - r0)) * a.cams + cam) * a.L + l) * (int64_t)G;
          const uint32_t oj = ord_f32(s_valid[j] ? __ldg(wpj + g) : 0.0f);
          sg += (oj < oi || (oj == oi && j < i)) ? 1 : 0;
        }
      }
      wn[(lo + sg) * G + g] = wg;
    }
  }
  __syncthreads();
  if (normalize) {
    if (threadIdx.x < G) {  // sequential f32 sum in this group's canonical order (features.py:264-269)
      float ws = 0.0f;
      const float* wg = wn + lo * G + threadIdx.x;
      for (int s2 = 0; s2 < n; ++s2) ws = __fadd_rn(ws, wg[(int64_t)s2 * G]);
      if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, bq);
      s_ws[threadIdx.x] = ws;
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < (int64_t)n * G; k += blockDim.x)
      wn[lo * G + k] = __fdiv_rn(wn[lo * G + k], s_ws[k % G]);
  }
}

__global__ void dense_offsets_kernel(int64_t* off, int64_t nq, int n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nq; i += (int64_t)gridDim.x * blockDim.x)
    off[i] = i * n;
}

cudaError_t launch_dense_offsets(int64_t* off, int64_t nq, int n, cudaStream_t s) {
  dense_offsets_kernel<<<(unsigned)std::min<int64_t>((nq + 256) / 256, 1024), 256, 0, s>>>(off, nq, n);
  return cudaGetLastError();
}

// Projection pre-pass of the fused FAST path: one thread per (batch, anchor,
// keypoint, camera) builds the keypoint (geometry.py:207-255, f64), projects
// it (geometry.py:162-182, f64) and writes every level's cell coordinate
// cell[((bq * P + p) * cams + cam) * L + l] = f32(pixel / stride_l - 0.5)
// (features.py:45-47), or NaN when depth <= 1e-6 (the sample leaves the plan).
// (optionally also zeroing the split call's totals: out as float4 and the
// weight sums, saving the memset launches in front of the split)
__global__ void project_prepass_kernel(DenseArgs a, float2* cell, float4* zero4, int64_t n_zero4, float* zero1,
                                       int64_t n_zero1) {
  // the call's status reset and its keypoint-offset check, both by one thread
  // (the check depends on the learned offsets only, geometry.py:241-244): no
  // other thread of any kernel of the call reports before this grid completes
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.status = DevStatus{};
    for (int p = 7; p < a.P; ++p) {
      const float* o = a.offsets + (p - 7) * 3;
      if (!(fabsf(o[0]) <= 1.0f && fabsf(o[1]) <= 1.0f && fabsf(o[2]) <= 1.0f)) {
        set_status(a.status, MSDA_OFFSET_RANGE, p);
        break;
      }
    }
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_zero4; i += (int64_t)gridDim.x * blockDim.x)
    zero4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_zero1; i += (int64_t)gridDim.x * blockDim.x)
    zero1[i] = 0.0f;
  const int64_t n = (int64_t)a.bs * a.Q * a.P * a.cams;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int cam = (int)(i % a.cams);
    const int64_t bqp = i / a.cams;
    const int64_t bq = bqp / a.P;
    const int p = (int)(bqp - bq * a.P);
    double kp[3];
    anchor_keypoint(a.anchors + bq * 10, p, a.offsets, a.dt, kp);  // range reported above
    double u, v;
    const bool ok = project_point(a, cam, kp, u, v);
    for (int l = 0; l < a.L; ++l) {
      const double st = (double)a.strides[l];
      cell[i * a.L + l] = ok ? make_float2((float)(u / st - 0.5), (float)(v / st - 0.5))
                             : make_float2(__int_as_float(0x7fc00000), 0.0f);
    }
  }
}

// the split FAST call's one zeroing launch: status block, totals, weight sums
// (instead of three memset nodes ahead of the two accumulating kernels)
__global__ void zero_totals_kernel(DevStatus* st, float4* z4, int64_t n4, float* z1, int64_t n1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  if (t == 0) *st = DevStatus{};
  for (int64_t i = t; i < n4; i += stride) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = t; i < n1; i += stride) z1[i] = 0.0f;
}

// out[q, c] /= weight_sums[q, c / (C / G)] (camera-sharded partials after the all-reduce)
__global__ void group_normalize_kernel(float* out, const float* wsum, int64_t n_q, int C, int G, DevStatus* st) {
  const int cpg = C / G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_q * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / C;
    const float ws = wsum[q * G + (int)(i - q * C) / cpg];
    if (ws == 0.0f) set_status(st, MSDA_ZERO_WEIGHT_SUM, q);
    out[i] = out[i] / ws;
  }
}

size_t dense_exact_extra_bytes(int64_t n_queries, int64_t n_samples) {
  return align_up((size_t)(n_queries + 1) * 8, 256) + 5 * align_up((size_t)n_samples * 4, 256);
}

int32_t run_dense(const msda_features_t* f, int32_t Q, int32_t P, int32_t G, const float* loc, const float* w,
                  int32_t precision, int32_t normalize, float* out, void* ws, size_t ws_bytes, cudaStream_t s,
                  bool project, const float* anchors, int32_t n_learned, const float* offsets,
                  const msda_cameras_t* cams, const float* strides, float dt, float* wsum_out = nullptr);

// A forked stream for work that overlaps the caller's stream inside one call
// (fork / join events recorded per call).  One per host thread and device:
// calls from different threads never share it.
struct AuxStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false, tried = false;
};
const AuxStream& aux_stream() {
  thread_local AuxStream per_dev[64];
  static const AuxStream none{};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return none;
  AuxStream& x = per_dev[dev];
  if (!x.tried) {
    x.tried = true;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    x.ok = cudaStreamCreateWithPriority(&x.stream, cudaStreamNonBlocking, hi) == cudaSuccess &&
           cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) == cudaSuccess;
    if (!x.ok) cudaGetLastError();  // not sticky: the call runs both parts on the caller's stream
  }
  return x;
}


}  // namespace
}  // namespace msda

using namespace msda;

namespace {

int32_t validate_dense(const msda_features_t* f, int32_t Q, int32_t P, int32_t G) {
  if (!f || !f->data || !f->spatial_shape || !f->scale_start_index) return MSDA_BAD_ARG;
  if (f->n_cams <= 0 || f->n_levels <= 0 || f->channels <= 0 || f->batch <= 0 || Q < 0 || P <= 0) return MSDA_BAD_ARG;
  if (f->dtype < MSDA_F32 || f->dtype > MSDA_BF16) return MSDA_BAD_ARG;
  if (f->channels % 2) return MSDA_ODD_CHANNELS;
  if (G <= 0 || G > kMaxGroups || f->channels % G || (f->channels / G) % 2) return MSDA_BAD_ARG;
  if (f->n_rows <= 0 || (int64_t)f->batch * f->n_rows >= (int64_t(1) << 31)) return MSDA_BAD_ARG;
  const int esz = f->dtype == MSDA_F32 ? 4 : 2;
  if (f->channels / 2 > kDenseThreads || (reinterpret_cast<uintptr_t>(f->data) % 4) || (f->channels * esz) % 4)
    return MSDA_BAD_ARG;
  return MSDA_OK;
}

size_t dense_ws(int32_t batch, int32_t Q, int32_t P, int32_t cams, int32_t L) {
  const int64_t nq = (int64_t)batch * Q;
  const int64_t S = nq * P * cams * L;
  return exact_workspace_bytes(nq, S) + dense_exact_extra_bytes(nq, S);
}

}  // namespace

namespace msda {
namespace {

int32_t run_dense(const msda_features_t* f, int32_t Q, int32_t P, int32_t G, const float* loc, const float* w,
                  int32_t precision, int32_t normalize, float* out, void* ws, size_t ws_bytes, cudaStream_t s,
                  bool project, const float* anchors, int32_t n_learned, const float* offsets,
                  const msda_cameras_t* cams, const float* strides, float dt, float* wsum_out) {
  DenseArgs a{};
  a.wsum_out = wsum_out;
  a.feat = f->data;
  a.n_rows = f->n_rows;
  a.C = f->channels;
  a.bs = f->batch;
  a.Q = Q;
  a.P = P;
  a.cams = f->n_cams;
  a.L = f->n_levels;
  a.G = G;
  a.shape = f->spatial_shape;
  a.start = f->scale_start_index;
  a.loc = loc;
  a.w = w;
  a.normalize = normalize;
  a.out = out;
  if (project) {
    a.anchors = anchors;
    a.n_learned = n_learned;
    a.offsets = offsets;
    a.K = reinterpret_cast<const double*>(cams->K);
    a.R = reinterpret_cast<const double*>(cams->R);
    a.T = reinterpret_cast<const double*>(cams->t);
    a.strides = strides;
    a.dt = dt;
  }
  const int64_t nq = (int64_t)a.bs * Q;
  const int64_t S = nq * P * a.cams * a.L;
  if (ws_bytes < exact_workspace_bytes(nq, S) + dense_exact_extra_bytes(nq, S)) return MSDA_BAD_ARG;
  ExactWorkspace ew = carve_exact_workspace(ws, S);
  a.status = ew.status;
  const bool fast = precision == MSDA_FAST || precision == MSDA_FAST_H2;
  const int n_fine = fast && nq > 0 ? dense_staged_fine_levels(*f, G, P) : -1;
  const bool aligned_out = a.C % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
  // FAST totals are zeroed by one kernel: the projection pre-pass, or (plain
  // calls) zero_totals_kernel, which also resets the status block (a split
  // over levels or cameras red.adds into them; an unsplit gather overwrites)
  const bool zeroed = fast && nq > 0 && aligned_out;
  // the status block is reset by the first kernel of the call where one of
  // ours comes first (projection pre-pass, zeroing kernel), else by a memset
  const bool fused_exact = precision == MSDA_EXACT && !normalize && !project;
  const bool kernel_reset = nq > 0 && ((fast && (project || zeroed)) || fused_exact);
  if (!kernel_reset && reset_exact_workspace(ew, s) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (nq == 0) return MSDA_OK;
  if (fast) {
    const bool h2 = precision == MSDA_FAST_H2;
    // the exact records' space is free in FAST: it holds the split weight sums
    float* scratch = reinterpret_cast<float*>(ew.rec);
    DenseFastSpec d{loc, w, Q, P, G, normalize, wsum_out, scratch, h2};
    float* wsum = wsum_out ? wsum_out : (normalize ? scratch : nullptr);
    if (zeroed && !project) {
      const int blocks = (int)std::min<int64_t>((nq * a.C / 4 + 255) / 256, 148 * 4);
      zero_totals_kernel<<<blocks, 256, 0, s>>>(ew.status, reinterpret_cast<float4*>(out), nq * a.C / 4, wsum,
                                                wsum ? nq * G : 0);
      if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
    }
    if (project) {  // projection pre-pass (f64): per-level cells of every (anchor, keypoint, camera)
      float2* uv = reinterpret_cast<float2*>(ew.g_hi);  // the exact sort scratch (8 B per sample) is free in FAST
      const int64_t n = nq * P * a.cams;
      const int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 32);
      project_prepass_kernel<<<blocks, 128, 0, s>>>(a, uv, reinterpret_cast<float4*>(out), zeroed ? nq * a.C / 4 : 0,
                                                    wsum, (zeroed && wsum) ? nq * G : 0);
      if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
      d.loc = nullptr;
      d.proj_cell = uv;
    }
    // pipelined gather (msda_exact.cu); shapes it does not take use the warp-camera kernel
    bool pending = false;
    cudaError_t e = cudaErrorNotSupported;
    if (n_fine > 0) {  // coarse levels from on-chip staged maps, fine levels by the pipelined gather
      e = cudaSuccess;
      if (!zeroed) {
        e = cudaMemsetAsync(out, 0, (size_t)nq * a.C * 4, s);
        if (e == cudaSuccess && wsum) e = cudaMemsetAsync(wsum, 0, (size_t)nq * G * 4, s);
      }
      // coarse levels (shared-memory-bound, no L2 gathers) on a forked
      // high-priority stream beside the fine levels' gather (L2-bound):
      // one 256-thread coarse CTA per SM, the gather's one-warp CTAs fill
      // the rest; both red.add into the zeroed totals, the join orders
      // them before whatever follows on s (capturable in a CUDA graph)
      const AuxStream& x = aux_stream();
      if (e == cudaSuccess && x.ok) {
        e = cudaEventRecord(x.fork, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(x.stream, x.fork, 0);
        if (e == cudaSuccess) e = launch_dense_coarse(*f, d, n_fine, out, wsum, x.stream);
        if (e == cudaSuccess) e = cudaEventRecord(x.join, x.stream);
      } else if (e == cudaSuccess) {
        e = launch_dense_coarse(*f, d, n_fine, out, wsum, s);
      }
      if (e == cudaSuccess) {
        DenseFastSpec fine = d;
        fine.n_lv = n_fine;
        fine.accumulate = true;
        e = launch_gather_dense_fast(*f, fine, ew.status, out, s, &pending);
        if (e == cudaErrorNotSupported) return MSDA_CUDA_ERROR;  // the staged plan implies the gather fits
      }
      if (e == cudaSuccess && x.ok) e = cudaStreamWaitEvent(s, x.join, 0);
      if (e != cudaSuccess) return MSDA_CUDA_ERROR;
    } else {
      d.prezeroed = zeroed;
      e = launch_gather_dense_fast(*f, d, ew.status, out, s, &pending);
    }
    if (e == cudaSuccess) {
      if (pending) {
        const int64_t total = nq * a.C;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
        group_normalize_kernel<<<blocks, 256, 0, s>>>(out, wsum_out ? wsum_out : scratch, nq, a.C, G, ew.status);
        if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
      }
      return MSDA_OK;
    }
    if (e != cudaErrorNotSupported) return MSDA_CUDA_ERROR;
    // shapes the pipelined gather does not take: the warp-camera kernel (projecting itself)
    e = project ? launch_dense_fast<true>(a, f->dtype, h2, s) : launch_dense_fast<false>(a, f->dtype, h2, s);
    return e == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
  }
  if (precision == MSDA_EXACT_HALF && f->dtype != MSDA_F16) return MSDA_BAD_ARG;
  if (precision == MSDA_EXACT && !normalize && !project) {  // one fused pass: runs ranked in the gather warp
    const cudaError_t e = launch_dense_exact_fused(*f, loc, w, Q, P, G, out, ew.status, s);
    if (e == cudaSuccess) return MSDA_OK;
    if (e != cudaErrorNotSupported) return MSDA_CUDA_ERROR;
    if (reset_exact_workspace(ew, s) != cudaSuccess) return MSDA_CUDA_ERROR;  // the fallback's kernels report
  }
  {  // EXACT, one pass for every group (bit-identical to the per-group plans below)
    const int n = P * a.cams * a.L;
    const size_t smem = (size_t)n * 9;
    SampleRec* rec = ew.rec;
    float* wn_g = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + exact_workspace_bytes(nq, S) +
                                           dense_exact_extra_bytes(nq, S));
    if (G <= 8 && smem <= 200 * 1024 && ws_bytes >= dense_ws(a.bs, Q, P, a.cams, a.L) + (size_t)S * G * 4) {
      msda_csr_plan_t plan1{nq, S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
      // offsets: every query owns n consecutive canonical slots
      int64_t* d_off = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(ws) + exact_workspace_bytes(nq, S));
      plan1.offsets = d_off;
      if (launch_dense_offsets(d_off, nq, n, s) != cudaSuccess) return MSDA_CUDA_ERROR;
      auto kern = project ? dense_canon_kernel<true> : dense_canon_kernel<false>;
      if (smem > 48 * 1024 &&
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MSDA_CUDA_ERROR;
      kern<<<(unsigned)nq, 128, smem, s>>>(a, rec, wn_g, normalize);
      if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
      ExactWorkspace ew1 = ew;
      ew1.wn = wn_g;
      // weights arrive normalised per group (dense_canon_kernel): no division in the gather
      const cudaError_t e = launch_gather_exact(*f, plan1, precision, ew1, out, nullptr, s, 0, 0, -1, G, 0);
      if (e == cudaSuccess) return MSDA_OK;
      if (e != cudaErrorNotSupported) return MSDA_CUDA_ERROR;
    }
  }
  // EXACT / EXACT_HALF: one canonical CSR plan per group, exact kernels on its channel slice
  char* p = reinterpret_cast<char*>(ws) + exact_workspace_bytes(nq, S);
  int64_t* d_off = reinterpret_cast<int64_t*>(p);
  p += align_up((size_t)(nq + 1) * 8, 256);
  const size_t sb = align_up((size_t)S * 4, 256);
  int32_t* d_cam = reinterpret_cast<int32_t*>(p);
  int32_t* d_lvl = reinterpret_cast<int32_t*>(p + sb);
  float* d_u = reinterpret_cast<float*>(p + 2 * sb);
  float* d_v = reinterpret_cast<float*>(p + 3 * sb);
  float* d_w = reinterpret_cast<float*>(p + 4 * sb);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  msda_csr_plan_t plan{nq, S, d_off, d_cam, d_lvl, d_u, d_v, d_w};
  const int cpg = a.C / G;
  for (int g = 0; g < G; ++g) {
    if (project)
      dense_expand_kernel<true><<<(unsigned)nq, 256, 0, s>>>(a, g, d_off, d_cam, d_lvl, d_u, d_v, d_w);
    else
      dense_expand_kernel<false><<<(unsigned)nq, 256, 0, s>>>(a, g, d_off, d_cam, d_lvl, d_u, d_v, d_w);
    if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
    if (launch_plan_canon(*f, plan, normalize, ew, sms, s, Q) != cudaSuccess) return MSDA_CUDA_ERROR;
    if (launch_gather_exact(*f, plan, precision, ew, out, nullptr, s, g * cpg, cpg, -1, 1, normalize) != cudaSuccess)
      return MSDA_CUDA_ERROR;
  }
  return MSDA_OK;
}

}  // namespace
}  // namespace msda

extern "C" {

size_t msda_dense_workspace_size(int32_t batch, int32_t n_queries, int32_t n_points, int32_t n_cams,
                                 int32_t n_levels, int32_t n_groups, int32_t channels) {
  (void)channels;
  const int64_t S = (int64_t)batch * n_queries * n_points * n_cams * n_levels;
  return dense_ws(batch, n_queries, n_points, n_cams, n_levels) + (size_t)S * std::max(1, (int)n_groups) * 4;
}

int32_t msda_dense(const msda_features_t* feat, int32_t n_queries, int32_t n_points, int32_t n_groups,
                   const float* sampling_location, const float* weights, int32_t precision, int32_t normalize,
                   float* out, void* workspace, size_t workspace_bytes, void* stream) {
  int32_t st = validate_dense(feat, n_queries, n_points, n_groups);
  if (st != MSDA_OK) return st;
  if (precision < MSDA_EXACT || precision > MSDA_FAST_H2) return MSDA_BAD_PRECISION;
  if (n_queries == 0) return MSDA_OK;  // nothing to aggregate (empty tensors may carry null pointers)
  if (!sampling_location || !weights || !out || !workspace) return MSDA_BAD_ARG;
  return run_dense(feat, n_queries, n_points, n_groups, sampling_location, weights, precision, normalize, out,
                   workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream), false, nullptr, 0, nullptr,
                   nullptr, nullptr, 0.0f);
}

int32_t msda_dense_partial(const msda_features_t* feat, int32_t n_queries, int32_t n_points, int32_t n_groups,
                           const float* sampling_location, const float* weights, int32_t precision, float* out,
                           float* weight_sums, void* workspace, size_t workspace_bytes, void* stream) {
  int32_t st = validate_dense(feat, n_queries, n_points, n_groups);
  if (st != MSDA_OK) return st;
  if (precision != MSDA_FAST && precision != MSDA_FAST_H2) return MSDA_BAD_PRECISION;
  if (n_queries == 0) return MSDA_OK;
  if (!sampling_location || !weights || !out || !weight_sums || !workspace) return MSDA_BAD_ARG;
  return run_dense(feat, n_queries, n_points, n_groups, sampling_location, weights, precision, 0, out, workspace,
                   workspace_bytes, reinterpret_cast<cudaStream_t>(stream), false, nullptr, 0, nullptr, nullptr,
                   nullptr, 0.0f, weight_sums);
}

int32_t msda_dense_normalize(float* out, const float* weight_sums, int64_t n_queries, int32_t channels,
                             int32_t n_groups, void* workspace, void* stream) {
  if (!out || !weight_sums || !workspace || n_queries < 0 || channels <= 0 || n_groups <= 0 ||
      channels % n_groups)
    return MSDA_BAD_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DevStatus* status = reinterpret_cast<DevStatus*>(workspace);
  if (cudaMemsetAsync(status, 0, sizeof(DevStatus), s) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (n_queries == 0) return MSDA_OK;
  const int64_t total = n_queries * channels;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  group_normalize_kernel<<<blocks, 256, 0, s>>>(out, weight_sums, n_queries, channels, n_groups, status);
  return cudaGetLastError() == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

int32_t msda_dense_project(const msda_features_t* feat, int32_t n_queries, const float* anchors, int32_t n_learned,
                           const float* learned_offsets, const msda_cameras_t* cams, const float* strides, float dt,
                           int32_t n_groups, const float* weights, int32_t precision, int32_t normalize, float* out,
                           void* workspace, size_t workspace_bytes, void* stream) {
  const int32_t P = 7 + n_learned;
  int32_t st = validate_dense(feat, n_queries, P, n_groups);
  if (st != MSDA_OK) return st;
  if (precision < MSDA_EXACT || precision > MSDA_FAST_H2) return MSDA_BAD_PRECISION;
  if (n_learned < 0 || P > kMaxPoints || (n_learned > 0 && !learned_offsets)) return MSDA_BAD_ARG;
  if (n_queries == 0) return MSDA_OK;
  if (!anchors || !cams || !cams->K || !cams->R || !cams->t || !strides || !weights || !out || !workspace)
    return MSDA_BAD_ARG;
  return run_dense(feat, n_queries, P, n_groups, nullptr, weights, precision, normalize, out, workspace,
                   workspace_bytes, reinterpret_cast<cudaStream_t>(stream), true, anchors, n_learned,
                   learned_offsets, cams, strides, dt);
}

}  // extern "C"
