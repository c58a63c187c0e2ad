// Occlusion-aware embedding pooling (cfg4), fused after the keypoint
// sampling — sm_100a.
//
// Restates mvtrack3d.oae (oae.py:81-164) on the device, one CTA per query:
//   for every camera
//     for every keypoint (geometry.py:207-255 in f64) in front of the camera
//       g_k = mean over levels of the f32 bilinear read at
//             cell = pixel / stride - 0.5                  (oae.py:103-112)
//     a = softmax_k(desc . g_k / sqrt(D)); view = sum_k a_k g_k (oae.py:117-122)
//   fused = sum_c v_c view_c / sum_c v_c over valid views    (oae.py:125-151)
//   |fused|_2 normalised; sum v <= 1e-3 -> memory, all_occluded (oae.py:154-164)
// oae_warp_kernel (below) is the production kernel; oae_pool_kernel is the
// generic fallback (threads own VEC consecutive channels, g_k staged in f64
// shared memory, block-reduced dot products) for channel counts that do not
// fill one warp row.
#include <algorithm>

#include "msda_common.cuh"

namespace msda {
namespace {

constexpr int kOaeMaxPoints = 64;
constexpr int kOaeMaxC = 1024;

struct OaeArgs {
  const void* feat;
  int32_t C, cams, L, Q;
  const int32_t* shape;
  const int64_t* start;
  const float* anchors;  // [Q, 10]
  const float* offsets;  // [n_learned, 3]
  int32_t P;
  const double* K;
  const double* R;
  const double* T;
  const float* strides;  // [L]
  const float* desc;     // [Q, C]
  const float* vis;      // [Q, cams]
  const float* memory;   // [Q, C]
  float* out;            // [Q, C]
  uint8_t* occluded;     // [Q]
  DevStatus* status;
  // camera groups (oae_warp_kernel<.., SPLIT>): CTA (q, grp) takes cameras
  // [grp * kOaeWarps, (grp + 1) * kOaeWarps) and writes its partial sums
  int32_t n_grp;
  double* part;     // [Q, n_grp, C] sum_c v_c view_c over the group's valid views
  double* part_vt;  // [Q, n_grp] sum_c v_c over the same views
};

// block-wide sum of one double per thread (blockDim multiple of 32, <= 1024)
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

template <typename T, int VEC>
__global__ void oae_pool_kernel(OaeArgs a) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_g = reinterpret_cast<double*>(smem_raw);  // [P][C]
  __shared__ double s_kp[kOaeMaxPoints * 3];
  __shared__ double s_red[32];
  __shared__ double s_score[kOaeMaxPoints];
  __shared__ int s_valid[kOaeMaxPoints];

  const int q = blockIdx.x;
  const int c0 = threadIdx.x * VEC;
  const bool active = c0 < a.C;
  const size_t row_bytes = (size_t)a.C * sizeof(T);
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)(active ? c0 : 0) * sizeof(T);

  for (int p = threadIdx.x; p < a.P; p += blockDim.x)
    if (!anchor_keypoint(a.anchors + (int64_t)q * 10, p, a.offsets, 0.0f, s_kp + 3 * p))
      set_status(a.status, MSDA_OFFSET_RANGE, p);
  __syncthreads();

  double d[VEC], fused[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    d[e] = active ? (double)a.desc[(int64_t)q * a.C + c0 + e] : 0.0;
    fused[e] = 0.0;
  }
  const double inv_sqrt_d = 1.0 / sqrt((double)a.C);
  double vis_total = 0.0;

  for (int cam = 0; cam < a.cams; ++cam) {
    int n_valid = 0;
    for (int p = 0; p < a.P; ++p) {
      double up, vp;
      const bool ok = project_f64(a.K + cam * 4, a.R + cam * 9, a.T + cam * 3, s_kp + 3 * p, up, vp);
      if (threadIdx.x == 0) s_valid[p] = ok;
      if (!ok) continue;
      ++n_valid;
      double g[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) g[e] = 0.0;
      for (int l = 0; l < a.L; ++l) {
        const int t = cam * a.L + l;
        const double st = (double)a.strides[l];
        const SampleRec r = make_record((float)(up / st - 0.5), (float)(vp / st - 0.5), a.start[t],
                                        a.shape[2 * t], a.shape[2 * t + 1]);
        float c[4][VEC];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const RawVec<BYTES> raw = (active && r.row[k] >= 0) ? ldg_vec<BYTES>(feat + (size_t)r.row[k] * row_bytes)
                                                              : zero_vec<BYTES>();
          to_f32<T, VEC>(raw, c[k]);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float b = __fadd_rn(__fadd_rn(__fmul_rn(c[0][e], r.iw[0]), __fmul_rn(c[1][e], r.iw[1])),
                                    __fadd_rn(__fmul_rn(c[2][e], r.iw[2]), __fmul_rn(c[3][e], r.iw[3])));
          g[e] += (double)b;
        }
      }
      double dot = 0.0;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        g[e] /= (double)a.L;  // level mean (oae.py:112)
        if (active) s_g[(size_t)p * a.C + c0 + e] = g[e];
        dot += g[e] * d[e];
      }
      dot = block_sum(dot, s_red);
      if (threadIdx.x == 0) s_score[p] = dot * inv_sqrt_d;
    }
    __syncthreads();
    if (n_valid == 0) continue;  // invalid view: zero visibility weight (oae.py:141-143)
    double mx = -INFINITY;
    for (int p = 0; p < a.P; ++p)
      if (s_valid[p]) mx = fmax(mx, s_score[p]);
    double z = 0.0;
    for (int p = 0; p < a.P; ++p)
      if (s_valid[p]) z += exp(s_score[p] - mx);
    double view[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) view[e] = 0.0;
    for (int p = 0; p < a.P; ++p) {
      if (!s_valid[p]) continue;
      const double wgt = exp(s_score[p] - mx) / z;
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (active) view[e] += wgt * s_g[(size_t)p * a.C + c0 + e];
    }
    const double v = (double)a.vis[(int64_t)q * a.cams + cam];
    vis_total += v;
#pragma unroll
    for (int e = 0; e < VEC; ++e) fused[e] += v * view[e];
    __syncthreads();
  }

  float* o = a.out + (int64_t)q * a.C;
  if (!(vis_total > 1e-3)) {  // AllOccluded -> keep the memory embedding
    if (active)
      for (int e = 0; e < VEC; ++e) o[c0 + e] = a.memory[(int64_t)q * a.C + c0 + e];
    if (threadIdx.x == 0) a.occluded[q] = 1;
    return;
  }
  double sq = 0.0;
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    fused[e] /= vis_total;
    sq += fused[e] * fused[e];
  }
  const double norm = sqrt(block_sum(active ? sq : 0.0, s_red));
  if (!(norm >= 1e-12)) set_status(a.status, MSDA_BAD_ARG, q);  // cannot normalise (oae.py:47-49)
  if (active)
    for (int e = 0; e < VEC; ++e) o[c0 + e] = (float)(fused[e] / norm);
  if (threadIdx.x == 0) a.occluded[q] = 0;
}

// ---------------------------------------------------------------------------
// Production shape (C == 32 * VEC): one CTA of kOaeWarps warps per query, warp
// w takes cameras w, w + kOaeWarps, ...; a whole warp covers the channel row.
// Per valid keypoint the 4 levels x 4 corner rows are loaded together, the
// level mean (FFMA2, the 1/L folded into the bilinear weights) and the
// descriptor score (per-lane FFMA2, f64 warp all-reduce) follow, and the
// keypoint softmax is accumulated online in f32 (running max / sum, weighted
// vector), so no keypoint features are staged.  Tolerance parity: fused
// products and f32 softmax vs the reference's f64 (<= 1e-4 on the unit
// embedding, tests/test_gpu_dense.py).  Per-warp camera partials are
// summed across warps at the end (tolerance-level reassociation of Eq. 2).

constexpr int kOaeWarps = 8;
__device__ __align__(16) unsigned char g_oae_zero_row[kOaeMaxC * 4];  // zero-initialised at module load
constexpr int kOaeLevels = 4;   // levels loaded together (more are looped)
constexpr int kOaeMaxRecs = 64;  // keypoints x levels staged per camera

// SPLIT: with many cameras one CTA per query leaves a ragged last wave (900
// CTAs at 2 per SM = 3.04 waves on 148 SMs); CTAs of (query, group of
// kOaeWarps cameras) — one camera per warp — write per-group partials (f64,
// fixed order) that oae_finish_kernel reduces in group order: deterministic.
template <typename T, int VEC, bool SPLIT = false>
__global__ void __launch_bounds__(kOaeWarps * 32, 2) oae_warp_kernel(OaeArgs a) {
  constexpr int NV = VEC * (int)sizeof(T) / 16;
  constexpr int LV = NV >= 2 ? 2 : kOaeLevels;  // levels in flight: bounded by registers
  __shared__ double s_kp[kOaeMaxPoints * 3];
  __shared__ SampleRec s_rec[kOaeWarps][kOaeMaxRecs];  // per camera: every (keypoint, level) record
  __shared__ float s_fused[kOaeWarps][32 * VEC];
  __shared__ double s_vt[kOaeWarps];
  __shared__ double s_red[kOaeWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = SPLIT ? (int)(blockIdx.x / a.n_grp) : (int)blockIdx.x;
  const int grp = SPLIT ? (int)(blockIdx.x - (int64_t)q * a.n_grp) : 0;
  const int cam_end = SPLIT ? min(a.cams, (grp + 1) * kOaeWarps) : a.cams;
  const int c0 = lane * VEC;
  const size_t row_bytes = (size_t)a.C * sizeof(T);
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)c0 * sizeof(T);
  const char* zrow = reinterpret_cast<const char*>(g_oae_zero_row) + (size_t)c0 * sizeof(T);
  const int units16 = (int)(row_bytes >> 4);  // row_bytes % 16 == 0 (C = 32 * VEC, 16-B lanes)

  if constexpr (SPLIT) {
    // split launch: nothing else of this grid reports (the finishing kernel
    // reports after it), so the call's status reset and the offset check
    // (offsets only, geometry.py:241-244) are one thread's
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
    for (int p = threadIdx.x; p < a.P; p += blockDim.x)
      anchor_keypoint(a.anchors + (int64_t)q * 10, p, a.offsets, 0.0f, s_kp + 3 * p);
  } else {
    for (int p = threadIdx.x; p < a.P; p += blockDim.x)
      if (!anchor_keypoint(a.anchors + (int64_t)q * 10, p, a.offsets, 0.0f, s_kp + 3 * p))
        set_status(a.status, MSDA_OFFSET_RANGE, p);
  }
  __syncthreads();

  float2 d2[VEC / 2];
  float fused[VEC];
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    d2[e / 2] = make_float2(a.desc[(int64_t)q * a.C + c0 + e], a.desc[(int64_t)q * a.C + c0 + e + 1]);
    fused[e] = fused[e + 1] = 0.0f;
  }
  const float inv_sqrt_d = (float)(1.0 / sqrt((double)a.C));
  const float inv_l = 1.0f / (float)a.L;  // level mean folded into the bilinear weights
  double vt = 0.0;

  for (int cam = grp * kOaeWarps + warp; cam < cam_end; cam += kOaeWarps) {
    double up = 0.0, vp = 0.0;
    const bool ok = lane < a.P &&
                    project_f64(a.K + cam * 4, a.R + cam * 9, a.T + cam * 3, s_kp + 3 * min(lane, a.P - 1), up, vp);
    unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (mask == 0u) continue;  // every keypoint behind: invalid view, zero weight (oae.py:114-115, 141-143)
    // every (keypoint, level) record of this camera, one per lane, staged in
    // warp-private shared memory: cell = pixel / stride - 0.5 (features.py:45-47)
    for (int s0 = 0; s0 < a.P * a.L; s0 += 32) {
      const int s = s0 + lane;
      const int kp = min(s, a.P * a.L - 1) / a.L, l = min(s, a.P * a.L - 1) % a.L;
      const double u = __shfl_sync(0xffffffffu, up, kp), v = __shfl_sync(0xffffffffu, vp, kp);
      if (s < a.P * a.L) {
        const int t = cam * a.L + l;
        const double st = (double)a.strides[l];
        SampleRec rec = make_record((float)(u / st - 0.5), (float)(v / st - 0.5), a.start[t], a.shape[2 * t],
                                    a.shape[2 * t + 1]);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // rows -> 16-B units: one shift per corner address in the load stream
          rec.row[k] = rec.row[k] >= 0 ? rec.row[k] * units16 : -1;
        s_rec[warp][s] = rec;
      }
    }
    __syncwarp();
    float m = -INFINITY, z = 0.0f;
    float2 acc[VEC / 2];
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) acc[e] = make_float2(0.0f, 0.0f);
    // two keypoints per step: their row loads are in flight together and the
    // two score reductions interleave; the softmax update stays in keypoint order
    auto online = [&](const float2* g, float dotf) {
      const float sc = dotf * inv_sqrt_d;
      const float m2 = fmaxf(m, sc);
      const float scale = expf(m - m2), w = expf(sc - m2);  // online softmax (oae.py:117-122)
      z = z * scale + w;
      const float2 s2 = make_float2(scale, scale), w2 = make_float2(w, w);
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) acc[e] = __ffma2_rn(g[e], w2, __fmul2_rn(acc[e], s2));
      m = m2;
    };
    while (mask) {
      const int pa = __ffs(mask) - 1;
      mask &= mask - 1;
      const bool has_b = mask != 0;
      const int pb = has_b ? __ffs(mask) - 1 : pa;
      if (has_b) mask &= mask - 1;
      float2 ga[VEC / 2], gb[VEC / 2];
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) ga[e] = gb[e] = make_float2(0.0f, 0.0f);
      constexpr int LP = LV >= 2 ? LV / 2 : 1;  // levels per keypoint per load round
      for (int l0 = 0; l0 < a.L; l0 += LP) {
        SampleRec r[2][LP];
        Row<NV> c[2][LP][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int j = 0; j < LP; ++j) {
            const int l = l0 + j;
            const bool use = l < a.L && (h == 0 || has_b);
            if (use) {
              r[h][j] = s_rec[warp][(h ? pb : pa) * a.L + l];
            } else {
              r[h][j].row[0] = r[h][j].row[1] = r[h][j].row[2] = r[h][j].row[3] = -1;
              r[h][j].iw[0] = r[h][j].iw[1] = r[h][j].iw[2] = r[h][j].iw[3] = 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // out-of-grid corners read a static zero row (L1-resident): no
              // predication or register zero-fill in the load stream
              const int row = r[h][j].row[k];
              c[h][j][k] = ld_row<NV>(row >= 0 ? feat + ((size_t)(uint32_t)row << 4) : zrow);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float2* g = h ? gb : ga;
#pragma unroll
          for (int j = 0; j < LP; ++j) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float f[VEC];
              raw_to_f32<T, VEC>(reinterpret_cast<const uint32_t*>(c[h][j][k].v), f);
              const float cw = r[h][j].iw[k] * inv_l;
              const float2 w2 = make_float2(cw, cw);
#pragma unroll
              for (int e = 0; e < VEC / 2; ++e) g[e] = __ffma2_rn(make_float2(f[2 * e], f[2 * e + 1]), w2, g[e]);
            }
          }
        }
      }
      float2 da = make_float2(0.0f, 0.0f), db = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        da = __ffma2_rn(ga[e], d2[e], da);
        db = __ffma2_rn(gb[e], d2[e], db);
      }
      float sa = da.x + da.y, sb = db.x + db.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {  // two warp all-reduces, interleaved
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
      }
      online(ga, sa);
      if (has_b) online(gb, sb);
    }
    __syncwarp();  // the next camera restages s_rec
    const double vis = (double)a.vis[(int64_t)q * a.cams + cam];
    vt += vis;
    const float vz = (float)(vis / (double)z);
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) {
      fused[2 * e] += vz * acc[e].x;
      fused[2 * e + 1] += vz * acc[e].y;
    }
  }

#pragma unroll
  for (int e = 0; e < VEC; ++e) s_fused[warp][c0 + e] = fused[e];
  if (lane == 0) s_vt[warp] = vt;
  __syncthreads();
  double total = 0.0;
#pragma unroll
  for (int w = 0; w < kOaeWarps; ++w) total += s_vt[w];
  if constexpr (SPLIT) {  // the group's partials; oae_finish_kernel completes the query
    double* pp = a.part + ((int64_t)q * a.n_grp + grp) * a.C;
    for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
      double f = 0.0;
#pragma unroll
      for (int w = 0; w < kOaeWarps; ++w) f += (double)s_fused[w][c];
      pp[c] = f;
    }
    if (threadIdx.x == 0) a.part_vt[(int64_t)q * a.n_grp + grp] = total;
    return;
  }
  float* o = a.out + (int64_t)q * a.C;
  if (!(total > 1e-3)) {  // AllOccluded -> keep the memory embedding (oae.py:159-164)
    for (int c = threadIdx.x; c < a.C; c += blockDim.x) o[c] = a.memory[(int64_t)q * a.C + c];
    if (threadIdx.x == 0) a.occluded[q] = 1;
    return;
  }
  // fused / total, then L2 normalise (oae.py:151, 44-50)
  double sq = 0.0;
  for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
    double f = 0.0;
#pragma unroll
    for (int w = 0; w < kOaeWarps; ++w) f += (double)s_fused[w][c];
    f /= total;
    s_fused[0][c] = (float)f;  // each c is owned by one thread: safe in place after the sum
    sq += f * f;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o2);
  if (lane == 0) s_red[warp] = sq;
  __syncthreads();
  double norm2 = 0.0;
#pragma unroll
  for (int w = 0; w < kOaeWarps; ++w) norm2 += s_red[w];
  const double norm = sqrt(norm2);
  if (!(norm >= 1e-12)) set_status(a.status, MSDA_BAD_ARG, q);
  for (int c = threadIdx.x; c < a.C; c += blockDim.x) o[c] = (float)((double)s_fused[0][c] / norm);
  if (threadIdx.x == 0) a.occluded[q] = 0;
}

// one CTA per query: sum the groups' partials in group order, then the
// fused / total, AllOccluded and L2-normalisation steps of oae_warp_kernel
__global__ void __launch_bounds__(256) oae_finish_kernel(OaeArgs a) {
  __shared__ double s_red[8];
  const int q = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* pv = a.part_vt + (int64_t)q * a.n_grp;
  double total = 0.0;
  for (int g = 0; g < a.n_grp; ++g) total += pv[g];
  float* o = a.out + (int64_t)q * a.C;
  if (!(total > 1e-3)) {  // AllOccluded -> keep the memory embedding (oae.py:159-164)
    for (int c = threadIdx.x; c < a.C; c += blockDim.x) o[c] = a.memory[(int64_t)q * a.C + c];
    if (threadIdx.x == 0) a.occluded[q] = 1;
    return;
  }
  const double* pp = a.part + (int64_t)q * a.n_grp * a.C;
  double sq = 0.0;
  double f[4];  // C <= 4 * 256 (kOaeMaxC)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * 256;
    f[i] = 0.0;
    if (c < a.C) {
      for (int g = 0; g < a.n_grp; ++g) f[i] += pp[(int64_t)g * a.C + c];
      f[i] /= total;
      sq += f[i] * f[i];
    }
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o2);
  if (lane == 0) s_red[warp] = sq;
  __syncthreads();
  double norm2 = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) norm2 += s_red[w];
  const double norm = sqrt(norm2);
  if (!(norm >= 1e-12)) set_status(a.status, MSDA_BAD_ARG, q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c < a.C) o[c] = (float)(f[i] / norm);
  }
  if (threadIdx.x == 0) a.occluded[q] = 0;
}

template <typename T, int VEC>
cudaError_t launch_oae_warp(const OaeArgs& a, cudaStream_t s) {
  if (a.Q == 0) return cudaSuccess;
  if (a.n_grp > 1) {
    oae_warp_kernel<T, VEC, true><<<(unsigned)((int64_t)a.Q * a.n_grp), kOaeWarps * 32, 0, s>>>(a);
    if (cudaGetLastError() != cudaSuccess) return cudaErrorLaunchFailure;
    oae_finish_kernel<<<a.Q, 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  oae_warp_kernel<T, VEC><<<a.Q, kOaeWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int VEC>
cudaError_t launch_oae_t(const OaeArgs& a, cudaStream_t s) {
  const int lanes = a.C / VEC;
  const int block = std::max(32, (lanes + 31) / 32 * 32);
  const size_t smem = (size_t)a.P * a.C * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(oae_pool_kernel<T, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (a.Q == 0) return cudaSuccess;
  oae_pool_kernel<T, VEC><<<a.Q, block, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace
}  // namespace msda

using namespace msda;

extern "C" {

// status | per-(query, camera group) partials (split path, cams > kOaeWarps)
static size_t oae_groups(int32_t n_cams) { return n_cams > kOaeWarps ? (n_cams + kOaeWarps - 1) / kOaeWarps : 1; }

size_t msda_oae_workspace_size(int32_t n_queries, int32_t n_cams, int32_t channels) {
  const size_t g = oae_groups(n_cams);
  if (g <= 1 || n_queries <= 0 || channels <= 0) return kStatusBytes;
  return kStatusBytes + align_up((size_t)n_queries * g * channels * 8, 256) + align_up((size_t)n_queries * g * 8, 256);
}

int32_t msda_oae_pool(const msda_features_t* f, int32_t n_queries, const float* anchors, int32_t n_learned,
                      const float* learned_offsets, const msda_cameras_t* cams, const float* strides,
                      const float* descriptors, const float* visibility, const float* memory, float* out,
                      uint8_t* all_occluded, void* workspace, size_t workspace_bytes, void* stream) {
  if (!f || !f->data || !f->spatial_shape || !f->scale_start_index || f->batch != 1) return MSDA_BAD_ARG;
  if (f->n_cams <= 0 || f->n_levels <= 0 || f->channels <= 0 || n_queries < 0 || n_learned < 0) return MSDA_BAD_ARG;
  if (f->channels % 2) return MSDA_ODD_CHANNELS;
  if (f->channels > kOaeMaxC || 7 + n_learned > kOaeMaxPoints) return MSDA_BAD_ARG;
  if (n_queries == 0) return MSDA_OK;  // empty tensors may carry null pointers
  if (!anchors || !cams || !cams->K || !cams->R || !cams->t || !strides || !descriptors || !visibility ||
      !memory || !out || !all_occluded || !workspace || workspace_bytes < kStatusBytes)
    return MSDA_BAD_ARG;
  if (n_learned > 0 && !learned_offsets) return MSDA_BAD_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  OaeArgs a{};
  a.feat = f->data;
  a.C = f->channels;
  a.cams = f->n_cams;
  a.L = f->n_levels;
  a.Q = n_queries;
  a.shape = f->spatial_shape;
  a.start = f->scale_start_index;
  a.anchors = anchors;
  a.offsets = learned_offsets;
  a.P = 7 + n_learned;
  a.K = cams->K;
  a.R = cams->R;
  a.T = cams->t;
  a.strides = strides;
  a.desc = descriptors;
  a.vis = visibility;
  a.memory = memory;
  a.out = out;
  a.occluded = all_occluded;
  a.status = reinterpret_cast<DevStatus*>(workspace);
  a.n_grp = 1;
  if (oae_groups(f->n_cams) > 1 && workspace_bytes >= msda_oae_workspace_size(n_queries, f->n_cams, f->channels)) {
    a.n_grp = (int32_t)oae_groups(f->n_cams);
    char* p = reinterpret_cast<char*>(workspace) + kStatusBytes;
    a.part = reinterpret_cast<double*>(p);
    a.part_vt = reinterpret_cast<double*>(p + align_up((size_t)n_queries * a.n_grp * f->channels * 8, 256));
  }
  const uintptr_t al = reinterpret_cast<uintptr_t>(f->data);
  cudaError_t e;
  const int C = f->channels;
  const bool al16 = al % 16 == 0;
  // 16-B-unit row offsets in int32 (oae_warp_kernel): the table must stay below 32 GB
  // the warp kernel projects one keypoint per lane (32-bit ballot): P <= 32
  const bool recs_fit = a.P <= 32 && a.P * a.L <= kOaeMaxRecs && (double)f->n_rows * f->channels * (f->dtype == MSDA_F32 ? 4 : 2) <
                                                        (double)(1ll << 35);
  // the split warp kernel resets the status itself (its first thread); every other launch after a memset
  const bool warp_path = recs_fit && al16 && ((f->dtype == MSDA_F32 && (C == 256 || C == 128)) ||
                                              (f->dtype != MSDA_F32 && C == 256));
  if (!(warp_path && a.n_grp > 1 && a.Q > 0) && cudaMemsetAsync(workspace, 0, sizeof(DevStatus), s) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  if (recs_fit && al16 && f->dtype == MSDA_F32 && C == 256) return launch_oae_warp<float, 8>(a, s) == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
  if (recs_fit && al16 && f->dtype == MSDA_F32 && C == 128) return launch_oae_warp<float, 4>(a, s) == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
  if (recs_fit && al16 && f->dtype == MSDA_F16 && C == 256) return launch_oae_warp<__half, 8>(a, s) == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
  if (recs_fit && al16 && f->dtype == MSDA_BF16 && C == 256)
    return launch_oae_warp<__nv_bfloat16, 8>(a, s) == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
  switch (f->dtype) {
    case MSDA_F32:
      e = (C % 4 == 0 && al16) ? launch_oae_t<float, 4>(a, s) : launch_oae_t<float, 2>(a, s);
      break;
    case MSDA_F16:
      e = (C % 8 == 0 && al % 16 == 0) ? launch_oae_t<__half, 8>(a, s) : launch_oae_t<__half, 2>(a, s);
      break;
    default:
      e = (C % 8 == 0 && al % 16 == 0) ? launch_oae_t<__nv_bfloat16, 8>(a, s)
                                       : launch_oae_t<__nv_bfloat16, 2>(a, s);
  }
  return e == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

}  // extern "C"
