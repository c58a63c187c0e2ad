// Dense FAST MSDA with the coarse pyramid levels staged on chip — sm_100a.
//
// The 4-corner gathers of coarse levels re-read the same few cells hundreds of
// times (cfg1 shape: 266 corner touches per level-3 cell, 66 per level-2
// cell), so through L2 they cost far more than their bytes.  This kernel
// decomposes FAST (order-free) aggregation by camera instead of by anchor:
//
//   CTA (anchor block, channel slice of SC = 32*VEC channels, batch x camera)
//     1. stage the slice of this camera's coarsest levels (all cells) into
//        shared memory with cp.async (16-B chunks of the channel-last rows);
//     2. each warp takes anchors of the block; lanes build 32 sample records
//        at a time (cell = loc*W - 0.5 or the fused keypoint projection) and
//        stage the slice's group weights in warp-private shared memory;
//     3. the warp walks the anchor's P*L samples of this camera: staged levels
//        read corners from shared memory, the rest gather from global (L2);
//        FFMA2 into f32 (or HFMA2 into a half2 partial, FAST_H2);
//     4. the anchor's slice partial is added into out with red.global.add.v4
//        / .v2 (out zeroed first): cameras are summed in any order (FAST).
// Normalisation (per anchor and group) is a second small pass.
#include <algorithm>

#include "msda_common.cuh"

namespace msda {
namespace {

constexpr int kSliceWarps = 16;
constexpr int kSliceMaxGroups = 8;  // groups inside one channel slice
constexpr int kSliceMaxLevels = 8;
constexpr int kSliceStageBudget = 180 * 1024;  // dynamic smem for staged levels (static part ~33 KB)

struct SliceArgs {
  const void* feat;
  int64_t n_rows;
  int32_t C, bs, Q, P, cams, L, G;
  const int32_t* shape;
  const int64_t* start;
  const float* loc;
  const float* w;
  float* out;
  // PROJECT
  const float* anchors;
  const float* offsets;
  const double* K;
  const double* R;
  const double* T;
  const float* strides;
  float dt;
  DevStatus* status;
  // slicing
  int32_t first_staged;                  // levels >= first_staged live in smem
  int32_t staged_off[kSliceMaxLevels];   // byte offset of each staged level in smem
  int32_t anchors_per_block;
  int32_t stage_bytes;
};

template <int N>
struct VecT;
template <>
struct VecT<4> { using t = uint32_t; };
template <>
struct VecT<8> { using t = uint2; };
template <>
struct VecT<16> { using t = uint4; };

__device__ __forceinline__ void red_add(float* p, const float* v, int n) {
  if (n == 4) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3])
                 : "memory");
  } else if (n == 2) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v[0]), "f"(v[1]) : "memory");
  } else {
    for (int i = 0; i < n; ++i) atomicAdd(p + i, v[i]);
  }
}

template <typename T, int VEC, bool PROJECT, bool H2>
__global__ void __launch_bounds__(kSliceWarps * 32, 1) dense_slice_kernel(SliceArgs a) {
  constexpr int LB = VEC * (int)sizeof(T);  // bytes per lane per row slice
  using LV = typename VecT<LB>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SampleRec s_rec[kSliceWarps][32];
  __shared__ uint8_t s_lvl[kSliceWarps][32];
  __shared__ float s_w[kSliceWarps][32 * kSliceMaxGroups];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SC = 32 * VEC;
  const int slice = blockIdx.y;
  const int b = blockIdx.z / a.cams, cam = blockIdx.z % a.cams;
  const int c_base = slice * SC;
  const int cpg = a.C / a.G;
  const int g0 = c_base / cpg;                  // first group of the slice
  const int ng = max(1, SC / cpg);              // groups in the slice
  const int g_lane = (c_base + lane * VEC) / cpg - g0;
  const int esz = (int)sizeof(T);
  const int64_t row_base = (int64_t)b * a.n_rows;
  const char* feat = reinterpret_cast<const char*>(a.feat);
  const size_t row_bytes = (size_t)a.C * esz;

  // ---- 1. stage this camera's coarse levels (channel slice) ----
  {
    const int chunks = SC * esz / 16;
    for (int l = a.first_staged; l < a.L; ++l) {
      const int t = cam * a.L + l;
      const int cells = a.shape[2 * t] * a.shape[2 * t + 1];
      const char* src0 = feat + ((size_t)(row_base + a.start[t]) * a.C + c_base) * esz;
      const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(smem_raw + a.staged_off[l]);
      for (int i = threadIdx.x; i < cells * chunks; i += blockDim.x) {
        const int cell = i / chunks, ch = i - cell * chunks;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + (uint32_t)(cell * SC * esz + ch * 16)),
                     "l"(src0 + (size_t)cell * row_bytes + ch * 16));
      }
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }

  const char* featc = feat + (size_t)(c_base + lane * VEC) * esz;
  const int n_cs = a.P * a.L;
  const int q_lo = blockIdx.x * a.anchors_per_block;
  const int q_hi = min(a.Q, q_lo + a.anchors_per_block);
  for (int q = q_lo + warp; q < q_hi; q += kSliceWarps) {
    const int64_t bq = (int64_t)b * a.Q + q;
    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;
    __half2 hacc[VEC / 2 > 0 ? VEC / 2 : 1];
    if constexpr (H2) {
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
          double kp[3], up, vp;
          valid = anchor_keypoint(a.anchors + bq * 10, p, a.offsets, a.dt, kp);
          if (!valid) set_status(a.status, MSDA_OFFSET_RANGE, p);
          valid = valid && project_f64(a.K + cam * 4, a.R + cam * 9, a.T + cam * 3, kp, up, vp);
          const double st = (double)a.strides[l];
          u = valid ? (float)(up / st - 0.5) : -4.0f;
          v = valid ? (float)(vp / st - 0.5) : -4.0f;
        } else {
          const float* lp = a.loc + ((bq * a.P + p) * a.cams + cam) * 2;
          u = __fsub_rn(__fmul_rn(lp[0], (float)W), 0.5f);
          v = __fsub_rn(__fmul_rn(lp[1], (float)H), 0.5f);
        }
        const bool staged = l >= a.first_staged;
        s_rec[warp][lane] = make_record(u, v, staged ? 0 : row_base + a.start[t], H, W);
        s_lvl[warp][lane] = (uint8_t)l;
        const float* wp = a.w + (((bq * a.P + p) * a.cams + cam) * a.L + l) * (int64_t)a.G + g0;
        for (int gg = 0; gg < ng; ++gg) s_w[warp][lane * kSliceMaxGroups + gg] = valid ? __ldg(wp + gg) : 0.0f;
      }
      __syncwarp();
      // kUnroll samples per step: all their corner loads are issued before
      // any of them is consumed (memory-level parallelism per warp)
      constexpr int kUnroll = 4;
      for (int i0 = 0; i0 < n; i0 += kUnroll) {
        SampleRec rr[kUnroll];
        float wgs[kUnroll];
        LV cc[kUnroll][4];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          const int i = i0 + j;
          if (i >= n) {
            wgs[j] = 0.0f;
#pragma unroll
            for (int k = 0; k < 4; ++k) cc[j][k] = LV{};
            continue;
          }
          rr[j] = s_rec[warp][i];
          wgs[j] = s_w[warp][i * kSliceMaxGroups + g_lane];
          const int l = s_lvl[warp][i];
          if (l >= a.first_staged) {
            const unsigned char* lv = smem_raw + a.staged_off[l] + lane * LB;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              cc[j][k] = rr[j].row[k] >= 0 ? *reinterpret_cast<const LV*>(lv + (size_t)rr[j].row[k] * SC * esz)
                                           : LV{};
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              cc[j][k] = rr[j].row[k] >= 0
                             ? __ldg(reinterpret_cast<const LV*>(featc + (size_t)rr[j].row[k] * row_bytes))
                             : LV{};
          }
        }
#pragma unroll
        for (int j = 0; j < kUnroll; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i0 + j >= n) break;
          const float cw = rr[j].iw[k] * wgs[j];
          const uint32_t* raw = reinterpret_cast<const uint32_t*>(&cc[j][k]);
          if constexpr (H2) {
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
      __syncwarp();
    }
    if constexpr (H2) {
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        const float2 f = __half22float2(hacc[e]);
        acc[2 * e] = f.x;
        acc[2 * e + 1] = f.y;
      }
    }
    float* o = a.out + bq * a.C + c_base + lane * VEC;
#pragma unroll
    for (int e = 0; e < VEC; e += 4) red_add(o + e, acc + e, VEC - e >= 4 ? 4 : VEC - e);
  }
}

// out[b, q, c] /= sum over (p, cam, l) of w[b, q, p, cam, l, g(c)]
__global__ void normalize_kernel(const float* w, int64_t bq_n, int S, int G, int C, float* out, DevStatus* st) {
  const int64_t bq = blockIdx.x;
  __shared__ float s_sum[kSliceMaxGroups * 4];
  if (bq >= bq_n) return;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    float acc = 0.0f;
    for (int s = 0; s < S; ++s) acc += w[(bq * S + s) * G + g];
    s_sum[g] = acc;
    if (acc == 0.0f) set_status(st, MSDA_ZERO_WEIGHT_SUM, bq);
  }
  __syncthreads();
  const int cpg = C / G;
  for (int c = threadIdx.x; c < C; c += blockDim.x) out[bq * C + c] /= s_sum[c / cpg];
}

template <typename T, int VEC, bool PROJECT, bool H2>
cudaError_t launch_slice_t(const SliceArgs& a, int smem, int n_blocks, cudaStream_t s) {
  const int dyn = smem;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(dense_slice_kernel<T, VEC, PROJECT, H2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceStageBudget);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((unsigned)n_blocks, (unsigned)(a.C / (32 * VEC)), (unsigned)(a.bs * a.cams));
  dense_slice_kernel<T, VEC, PROJECT, H2><<<grid, kSliceWarps * 32, dyn, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

// Plan the slicing on the host from the level shapes: widest slice whose
// coarse levels (at least the coarsest) fit in shared memory.  Returns false
// when nothing useful fits (the caller keeps the per-anchor kernel).
bool plan_slice(const int32_t* shape_host, int cams, int L, int C, int esz, int G, int& VEC, int& first_staged,
                int* staged_off, int& stage_bytes) {
  if (L > kSliceMaxLevels) return false;
  for (int c = 1; c < cams; ++c)  // one staging layout for every camera
    for (int i = 0; i < 2 * L; ++i)
      if (shape_host[2 * L * c + i] != shape_host[i]) return false;
  const int budget = kSliceStageBudget;
  const int cpg = C / G;
  // the slice width that keeps the most levels on chip wins; ties go to the
  // widest slice (fewer, larger lane loads)
  int best_vec = 0, best_fs = L;
  for (int vec : {8, 4, 2}) {
    const int SC = 32 * vec;
    if (C % SC || vec * esz < 4 || vec * esz > 16 || SC % cpg && cpg % SC) continue;
    if (SC / cpg > kSliceMaxGroups) continue;
    // stage from the coarsest level down while it fits
    int bytes = 0, fs = L;
    for (int l = L - 1; l >= 1; --l) {  // never stage level 0 (finest; little reuse)
      const int need = shape_host[2 * l] * shape_host[2 * l + 1] * SC * esz;
      if (bytes + need > budget) break;
      bytes += need;
      fs = l;
    }
    if (fs < best_fs) {
      best_fs = fs;
      best_vec = vec;
    }
  }
  if (best_fs >= L) return false;
  VEC = best_vec;
  first_staged = best_fs;
  const int SC = 32 * best_vec;
  int off = 0;
  for (int l = 0; l < kSliceMaxLevels; ++l) staged_off[l] = 0;
  for (int l = best_fs; l < L; ++l) {
    staged_off[l] = off;
    off += shape_host[2 * l] * shape_host[2 * l + 1] * SC * esz;
  }
  stage_bytes = off;
  return true;
}

cudaError_t launch_dense_slice(const msda_features_t& f, int Q, int P, int G, const float* loc, const float* w,
                               bool project, const float* anchors, const float* offsets, const msda_cameras_t* cams,
                               const float* strides, float dt, bool h2, bool normalize, float* out, DevStatus* st,
                               int VEC, int first_staged, const int* staged_off, int stage_bytes, int num_sms,
                               cudaStream_t s) {
  SliceArgs a{};
  a.feat = f.data;
  a.n_rows = f.n_rows;
  a.C = f.channels;
  a.bs = f.batch;
  a.Q = Q;
  a.P = P;
  a.cams = f.n_cams;
  a.L = f.n_levels;
  a.G = G;
  a.shape = f.spatial_shape;
  a.start = f.scale_start_index;
  a.loc = loc;
  a.w = w;
  a.out = out;
  a.status = st;
  if (project) {
    a.anchors = anchors;
    a.offsets = offsets;
    a.K = cams->K;
    a.R = cams->R;
    a.T = cams->t;
    a.strides = strides;
    a.dt = dt;
  }
  a.first_staged = first_staged;
  for (int l = 0; l < kSliceMaxLevels; ++l) a.staged_off[l] = staged_off[l];
  a.stage_bytes = stage_bytes;
  // anchor blocks: enough CTAs to fill the device about twice
  const int slices = f.channels / (32 * VEC);
  const int64_t base_ctas = (int64_t)slices * f.batch * f.n_cams;
  int n_blocks = (int)std::max<int64_t>(1, (2 * num_sms + base_ctas - 1) / base_ctas);
  n_blocks = std::min(n_blocks, std::max(1, Q / kSliceWarps));
  a.anchors_per_block = (Q + n_blocks - 1) / n_blocks;
  n_blocks = (Q + a.anchors_per_block - 1) / a.anchors_per_block;
  cudaError_t e = cudaMemsetAsync(out, 0, (size_t)f.batch * Q * f.channels * sizeof(float), s);
  if (e != cudaSuccess) return e;
  const int esz = f.dtype == MSDA_F32 ? 4 : 2;
#define MSDA_SLICE_CASE(TT, V)                                                                        \
  if (VEC == V) {                                                                                     \
    if (project) e = h2 ? launch_slice_t<TT, V, true, true>(a, stage_bytes, n_blocks, s)              \
                        : launch_slice_t<TT, V, true, false>(a, stage_bytes, n_blocks, s);            \
    else e = h2 ? launch_slice_t<TT, V, false, true>(a, stage_bytes, n_blocks, s)                     \
                : launch_slice_t<TT, V, false, false>(a, stage_bytes, n_blocks, s);                   \
  }
  if (esz == 4) {
    MSDA_SLICE_CASE(float, 4)
    else MSDA_SLICE_CASE(float, 2)
  } else if (f.dtype == MSDA_F16) {
    MSDA_SLICE_CASE(__half, 8)
    else MSDA_SLICE_CASE(__half, 4)
    else MSDA_SLICE_CASE(__half, 2)
  } else {
    MSDA_SLICE_CASE(__nv_bfloat16, 8)
    else MSDA_SLICE_CASE(__nv_bfloat16, 4)
    else MSDA_SLICE_CASE(__nv_bfloat16, 2)
  }
#undef MSDA_SLICE_CASE
  if (e != cudaSuccess) return e;
  if (normalize) {
    normalize_kernel<<<(unsigned)((int64_t)f.batch * Q), 128, 0, s>>>(w, (int64_t)f.batch * Q,
                                                                     P * f.n_cams * f.n_levels, G, f.channels, out,
                                                                     st);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace msda
