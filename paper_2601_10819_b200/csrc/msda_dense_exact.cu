// Dense EXACT (bit-faithful) deformable_aggregation in one pass — sm_100a.
//
// The reference's contract is per-query bit identity with msda_reference
// (features.py:241-276): for every (query, channel) one sequential f32 sum
// over the query's samples in canonical order (camera, level, v, u, weight;
// features.py:261-263) of ((c00*w00 + c10*w10) + (c01*w01 + c11*w11)) * w,
// each product and sum rounded once.  With channel groups (Sparse4D), group
// g's channels use the plan with weights[..., g] (SURVEY §8(c) "Groups G").
//
// In the dense layout a query's samples come as (camera, level) runs of P
// keypoints, so canonicalising a query is ranking P keys inside each run —
// no global sort.  This kernel does it in the gather warp itself, one camera
// ahead of the accumulation, instead of a separate canonicalisation pass that
// writes records and per-group weights to HBM and reads them back:
//   * loader (per camera, per level run): lane p < P loads its keypoint's
//     location once per camera, builds the level's (v, u) key and record,
//     ranks it with P shuffles, and stages record + the G group weights at
//     its canonical slot in the warp's shared memory.  Exact (v, u) ties —
//     identical records — are ordered per group by that group's weight, then
//     position (the lexsort's last keys), exactly as the reference orders them;
//   * accumulation: the pipelined gather of msda_exact.cu (corner rows D
//     samples ahead with cp.async into a per-warp ring), every lane adding its
//     channels' exact tree (FFMA2 with -0 / 1 operands from kernel
//     parameters, exact_accumulate) with its group's weight, in slot order.
// normalize = False only (Sparse4D's softmaxed weights); normalising calls
// take the two-pass path, whose per-group weight sums need the whole
// canonical order first.
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "msda_common.cuh"
#include "msda_exact.cuh"

namespace msda {
namespace {

constexpr int kMaxRun = 32;      // keypoints per (camera, level) run: one lane each
constexpr int kMaxCamRun = 128;  // samples per camera (levels x keypoints) staged at once
constexpr int kGW = 8;           // group weights staged per sample
constexpr int kMaxLv = 4;        // levels per camera

struct DenseExactArgs {
  const void* feat;
  int64_t n_rows;  // rows per batch item
  int32_t C, Q, P, cams, L, G, cpg;
  const int32_t* shape;
  const int64_t* start;
  const float* loc;  // [bs, Q, P, cams, 2]
  const float* w;    // [bs, Q, P, cams, L, G]
  float* out;        // [bs, Q, C]
  int64_t n_queries;
  int32_t ncs_pad;   // staged samples per camera buffer (levels x keypoints, rounded up to 4)
  float2 one2, nz2;  // FFMA2 operands that make exact adds / products (parameters: never fused)
  DevStatus* status;  // reset by the first thread (no kernel of this call reports into it)
};

// per-warp shared memory: the corner ring, then two camera buffers of
// ncs_pad records (int4 rows, float4 iw) and kGW weights each
template <int BYTES, int D>
struct DxSmem {
  static constexpr int kSlot = 4 * 32 * BYTES;
  static constexpr int kRing = D * kSlot;
  static constexpr int bytes(int ncs_pad) { return kRing + 2 * ncs_pad * (16 + 16 + kGW * 4); }
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Canonicalise the keypoint run (camera cam, level l) of a query: lane p < P
// holds keypoint p's location lp and group weights pwl; each record goes to
// its canonical slot run0 + rank (features.py:261-263).  Exact (v, u) ties —
// identical records — are ordered per group by that group's weight, then
// position (the lexsort's last keys).
__device__ __forceinline__ void stage_run(const DenseExactArgs& a, int lane, bool act, float2 lp,
                                          const float (&pwl)[kGW], int cam, int l, int64_t row_base, int run0,
                                          int4* rows_w, float4* iw_w, float* wn_w) {
  const int t = cam * a.L + l;
  const int H = a.shape[2 * t], W = a.shape[2 * t + 1];
  const float u = __fsub_rn(__fmul_rn(lp.x, (float)W), 0.5f);  // cell = loc * W - 0.5 (features.py:20-24)
  const float v = __fsub_rn(__fmul_rn(lp.y, (float)H), 0.5f);
  const unsigned long long key = ((unsigned long long)ord_f32(v) << 32) | ord_f32(u);
  int below = 0, eq_before = 0;
  bool tie = false;
  for (int j = 0; j < a.P; ++j) {
    const unsigned long long kj = __shfl_sync(0xffffffffu, key, j);
    below += kj < key ? 1 : 0;
    tie |= (kj == key) & (j != lane);
    eq_before += (kj == key) & (j < lane) ? 1 : 0;
  }
  const SampleRec r = make_record(u, v, row_base + a.start[t], H, W);
  if (act) {  // tied records are identical: any slot of the tie set holds the same record
    rows_w[run0 + below + eq_before] = make_int4(r.row[0], r.row[1], r.row[2], r.row[3]);
    iw_w[run0 + below + eq_before] = make_float4(r.iw[0], r.iw[1], r.iw[2], r.iw[3]);
  }
  if (!__any_sync(0xffffffffu, act && tie)) {
    if (act) {
      float4* dst = reinterpret_cast<float4*>(wn_w + (run0 + below) * kGW);
      dst[0] = make_float4(pwl[0], pwl[1], pwl[2], pwl[3]);
      dst[1] = make_float4(pwl[4], pwl[5], pwl[6], pwl[7]);
    }
  } else {
    uint32_t oi[kGW];
    int sg[kGW];
#pragma unroll
    for (int g = 0; g < kGW; ++g) {
      oi[g] = ord_f32(pwl[g]);
      sg[g] = below;
    }
#pragma unroll 1
    for (int j = 0; j < a.P; ++j) {
      const unsigned long long kj = __shfl_sync(0xffffffffu, key, j);
      const bool same = j != lane && kj == key;
#pragma unroll
      for (int g = 0; g < kGW; ++g) {
        const uint32_t oj = __shfl_sync(0xffffffffu, oi[g], j);
        sg[g] += (same && (oj < oi[g] || (oj == oi[g] && j < lane))) ? 1 : 0;
      }
    }
    if (act)
#pragma unroll
      for (int g = 0; g < kGW; ++g) wn_w[(run0 + sg[g]) * kGW + g] = pwl[g];
  }
}

template <typename T, int VEC, int D>
__global__ void __launch_bounds__(32) dense_exact_kernel(const DenseExactArgs a) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.status) *a.status = DevStatus{};
  constexpr int BYTES = VEC * (int)sizeof(T);
  static_assert(BYTES == 16 || BYTES == 8, "8- or 16-B lanes");  // (8-B lanes, two warps per query: 1268 vs 957 us at cfg3)
  using SM = DxSmem<BYTES, D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  static_assert((D & (D - 1)) == 0, "ring depth: a power of two");
  const int NB = a.ncs_pad;  // samples per camera buffer
  const int lane = threadIdx.x;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t ring = sbase + lane * BYTES;           // + slot * kSlot + corner * 32 * BYTES
  const unsigned char* ring_ptr = smem_raw + lane * BYTES;
  const uint32_t s_rows = sbase + SM::kRing;            // int4 [2][NB]
  int4* rows_w = reinterpret_cast<int4*>(smem_raw + SM::kRing);
  float4* iw_w = reinterpret_cast<float4*>(smem_raw + SM::kRing + 2 * NB * 16);
  float* wn_w = reinterpret_cast<float*>(smem_raw + SM::kRing + 4 * NB * 16);

  const int warps_per_q = a.C / VEC / 32;
  const int64_t q = (int64_t)blockIdx.x / warps_per_q;
  if (q >= a.n_queries) return;
  const int c0 = (int)(blockIdx.x - q * warps_per_q) * 32 * VEC + lane * VEC;
  const int gl = c0 / a.cpg;  // this lane's channel group
  const int64_t row_base = (q / a.Q) * a.n_rows;
  const char* featc = reinterpret_cast<const char*>(a.feat) + (size_t)c0 * sizeof(T);
  const uint32_t row_bytes = (uint32_t)a.C * (uint32_t)sizeof(T);
  const int n_cs = a.L * a.P;  // samples per camera
  const int n = a.cams * n_cs;
  const bool act = lane < a.P;

  // a camera's keypoint location and group weights, loaded one camera before
  // they are staged (their HBM latency stays off the gather's path)
  float2 pl;
  float pw[kMaxLv][kGW];
  auto prefetch_camera = [&](int cam) {
    const int64_t pc = (q * a.P + (act ? lane : 0)) * a.cams + min(cam, a.cams - 1);
    pl = __ldg(reinterpret_cast<const float2*>(a.loc) + pc);
#pragma unroll
    for (int l = 0; l < kMaxLv; ++l)
#pragma unroll
      for (int g = 0; g < kGW; ++g)
        pw[l][g] = (l < a.L && g < a.G) ? __ldg(a.w + (pc * a.L + l) * a.G + g) : 0.0f;
  };
  // stage camera `cam`'s runs in canonical order into buffer `buf` from the prefetched inputs
  auto stage_camera = [&](int cam, int buf) {
#pragma unroll
    for (int l = 0; l < kMaxLv; ++l) {
      if (l >= a.L) break;
      stage_run(a, lane, act, pl, pw[l], cam, l, row_base, buf * NB + l * a.P, rows_w, iw_w, wn_w);
    }
    __syncwarp();
  };
  // corner rows of staged sample `idx` (buffer-major index) into ring slot `slot_addr`
  auto issue = [&](int idx, uint32_t slot_addr) {
    const uint4 rr = lds128(s_rows + idx * 16);
    const int rows[4] = {(int)rr.x, (int)rr.y, (int)rr.z, (int)rr.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      cp_async_zfill<BYTES>(slot_addr + k * 32 * BYTES, featc + (size_t)(uint32_t)max(rows[k], 0) * row_bytes,
                            rows[k] >= 0);
  };

  prefetch_camera(0);
  stage_camera(0, 0);
  prefetch_camera(1);
  // prologue: the first D samples (all in camera 0: D < levels x keypoints)
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < n) issue(k, ring + k * SM::kSlot);
    cp_async_commit();
  }
  float acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;
  uint32_t g = 0;  // global sample index; ring slot = g % D
  // one sample: its exact tree (products, sums, weight) — independent of acc
  auto tree = [&](int idx, uint32_t slot, float (&tw)[VEC]) {
    const uint4 iwr = *reinterpret_cast<const uint4*>(iw_w + idx);
    const float wn = wn_w[idx * kGW + gl];
    float c[4][VEC];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      RawVec<BYTES> cv;
      if constexpr (BYTES == 16) {
        cv.v = *reinterpret_cast<const uint4*>(ring_ptr + slot * SM::kSlot + k * 32 * BYTES);
      } else {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];"
                     : "=r"(cv.v.x), "=r"(cv.v.y)
                     : "r"(ring + slot * SM::kSlot + k * 32 * BYTES));
      }
      to_f32<T, VEC>(cv, c[k]);
    }
    const float2 w0 = make_float2(__uint_as_float(iwr.x), __uint_as_float(iwr.x));
    const float2 w1 = make_float2(__uint_as_float(iwr.y), __uint_as_float(iwr.y));
    const float2 w2 = make_float2(__uint_as_float(iwr.z), __uint_as_float(iwr.z));
    const float2 w3 = make_float2(__uint_as_float(iwr.w), __uint_as_float(iwr.w));
    const float2 ws = make_float2(wn, wn);
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {  // ((c00*w00 + c10*w10) + (c01*w01 + c11*w11)) * w, each op rounded once
      const float2 p0 = __ffma2_rn(make_float2(c[0][e], c[0][e + 1]), w0, a.nz2);
      const float2 p1 = __ffma2_rn(make_float2(c[1][e], c[1][e + 1]), w1, a.nz2);
      const float2 p2 = __ffma2_rn(make_float2(c[2][e], c[2][e + 1]), w2, a.nz2);
      const float2 p3 = __ffma2_rn(make_float2(c[3][e], c[3][e + 1]), w3, a.nz2);
      const float2 t = __ffma2_rn(__ffma2_rn(p0, a.one2, p1), a.one2, __ffma2_rn(p2, a.one2, p3));
      const float2 r = __ffma2_rn(t, ws, a.nz2);
      tw[e] = r.x;
      tw[e + 1] = r.y;
    }
  };
  // N samples' trees interleaved channel pair by channel pair: all 4 N
  // corner loads first, then for each pair the N samples' products and
  // sums side by side (independent chains in program order), so the
  // scheduler can cover FFMA2 / conversion latency with one warp per query
  auto treeN = [&](auto nsm, int idx0, uint32_t g0, float (&tw)[decltype(nsm)::value][VEC]) {
    constexpr int NS = decltype(nsm)::value;
    uint4 iwr[NS];
    float wn[NS];
    RawVec<BYTES> cv[NS][4];
#pragma unroll
    for (int sm = 0; sm < NS; ++sm) {
      iwr[sm] = *reinterpret_cast<const uint4*>(iw_w + idx0 + sm);
      wn[sm] = wn_w[(idx0 + sm) * kGW + gl];
      const uint32_t slot = (g0 + sm) % D;
#pragma unroll
      for (int k = 0; k < 4; ++k) cv[sm][k] = *reinterpret_cast<const RawVec<BYTES>*>(ring_ptr + slot * SM::kSlot + k * 32 * BYTES);
    }
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
#pragma unroll
      for (int sm = 0; sm < NS; ++sm) {
        float2 c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float f[VEC];
          to_f32<T, VEC>(cv[sm][k], f);
          c[k] = make_float2(f[e], f[e + 1]);
        }
        const float2 p0 = __ffma2_rn(c[0], make_float2(__uint_as_float(iwr[sm].x), __uint_as_float(iwr[sm].x)), a.nz2);
        const float2 p1 = __ffma2_rn(c[1], make_float2(__uint_as_float(iwr[sm].y), __uint_as_float(iwr[sm].y)), a.nz2);
        const float2 p2 = __ffma2_rn(c[2], make_float2(__uint_as_float(iwr[sm].z), __uint_as_float(iwr[sm].z)), a.nz2);
        const float2 p3 = __ffma2_rn(c[3], make_float2(__uint_as_float(iwr[sm].w), __uint_as_float(iwr[sm].w)), a.nz2);
        const float2 t = __ffma2_rn(__ffma2_rn(p0, a.one2, p1), a.one2, __ffma2_rn(p2, a.one2, p3));
        const float2 r = __ffma2_rn(t, make_float2(wn[sm], wn[sm]), a.nz2);
        tw[sm][e] = r.x;
        tw[sm][e + 1] = r.y;
      }
    }
  };
  auto add = [&](const float (&tw)[VEC]) {  // acc + tw: the sequential sum (features.py:271-274)
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const float2 r = __ffma2_rn(make_float2(tw[e], tw[e + 1]), a.one2, make_float2(acc[e], acc[e + 1]));
      acc[e] = r.x;
      acc[e + 1] = r.y;
    }
  };
  for (int cam = 0; cam < a.cams; ++cam) {
    const bool has_next = cam + 1 < a.cams;
    if (has_next) {  // stage camera c + 1 (its inputs were loaded a camera ago), prefetch c + 2
      stage_camera(cam + 1, (cam + 1) & 1);
      prefetch_camera(cam + 2);
    }
    const int buf = (cam & 1) * NB, nbuf = ((cam + 1) & 1) * NB;
    // the sample D ahead of (cam, j): this camera's buffer, then the next one's
    auto refill = [&](int j, uint32_t slot) {
      const int ja = j + D;
      if (ja < n_cs) issue(buf + ja, ring + slot * SM::kSlot);
      else if (has_next) issue(nbuf + ja - n_cs, ring + slot * SM::kSlot);
      cp_async_commit();
    };
    int j = 0;
    if constexpr (D >= 8) {  // four samples per step: their trees overlap, the adds stay in order
      for (; j + 3 < n_cs; j += 4, g += 4) {
        cp_async_wait<D - 4>();
        float tt[4][VEC];
        treeN(std::integral_constant<int, 4>{}, buf + j, g, tt);
        add(tt[0]);
        add(tt[1]);
        add(tt[2]);
        add(tt[3]);
        refill(j, g % D);
        refill(j + 1, (g + 1) % D);
        refill(j + 2, (g + 2) % D);
        refill(j + 3, (g + 3) % D);
      }
    }
    for (; j + 1 < n_cs; j += 2, g += 2) {  // two samples: their trees overlap, the adds stay in order
      cp_async_wait<D - 2>();
      float tt[2][VEC];
      treeN(std::integral_constant<int, 2>{}, buf + j, g, tt);
      add(tt[0]);
      add(tt[1]);
      refill(j, g % D);
      refill(j + 1, (g + 1) % D);
    }
    if (j < n_cs) {
      cp_async_wait<D - 1>();
      float t0[VEC];
      tree(buf + j, g % D, t0);
      add(t0);
      refill(j, g % D);
      ++g;
    }
  }
  cp_async_wait<0>();
  float* o = a.out + q * a.C + c0;
#pragma unroll
  for (int e = 0; e < VEC; e += 4)
    *reinterpret_cast<float4*>(o + e) = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
}

// resident one-warp CTAs of dense_exact_kernel<T, VEC, D> on the device
template <typename T, int VEC, int D>
int64_t dx_slots(int smem) {
  int per_sm = 0, sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaFuncSetAttribute(dense_exact_kernel<T, VEC, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_exact_kernel<T, VEC, D>, 32, smem) != cudaSuccess)
    per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int64_t)per_sm * sms;
}

template <typename T, int VEC, int D>
cudaError_t launch_dx(const DenseExactArgs& a, cudaStream_t s) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int smem = DxSmem<BYTES, D>::bytes(a.ncs_pad);
  static std::atomic<bool> attr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
    const cudaError_t e =
        cudaFuncSetAttribute(dense_exact_kernel<T, VEC, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_release);
  }
  const int64_t grid = a.n_queries * (a.C / VEC / 32);
  if (grid == 0) return cudaSuccess;
  dense_exact_kernel<T, VEC, D><<<(unsigned)grid, 32, smem, s>>>(a);
  return cudaGetLastError();
}

// one sequential chain per warp: a warp that misses the first wave costs a
// whole extra chain, so take the deepest ring whose residency still holds
// every warp at once (else the shallowest)
template <typename T, int VEC>
cudaError_t launch_dx_depth(const DenseExactArgs& a, cudaStream_t s) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int64_t warps = a.n_queries * (a.C / VEC / 32);
  const int n_cs = a.L * a.P;
  if (n_cs > 16 && warps <= dx_slots<T, VEC, 16>(DxSmem<BYTES, 16>::bytes(a.ncs_pad))) return launch_dx<T, VEC, 16>(a, s);
  if (n_cs > 8 && warps <= dx_slots<T, VEC, 8>(DxSmem<BYTES, 8>::bytes(a.ncs_pad))) return launch_dx<T, VEC, 8>(a, s);
  if (n_cs > 4) return launch_dx<T, VEC, 4>(a, s);
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t launch_dense_exact_fused(const msda_features_t& f, const float* loc, const float* w, int Q, int P, int G,
                                     float* out, DevStatus* status, cudaStream_t stream) {
  const int C = f.channels;
  const int esz = f.dtype == MSDA_F32 ? 4 : 2;
  if (G < 1 || G > kGW || C % G || P < 1 || P > kMaxRun || f.n_levels > kMaxLv || f.n_levels * P > kMaxCamRun)
    return cudaErrorNotSupported;
  const int vec = f.dtype == MSDA_F32 ? 4 : 8;  // 16-B lanes
  if (C % (32 * vec) || (C / G) % vec) return cudaErrorNotSupported;  // whole warps; a lane in one group
  if (reinterpret_cast<uintptr_t>(f.data) % 16 || (C * esz) % 16 || reinterpret_cast<uintptr_t>(out) % 16 ||
      reinterpret_cast<uintptr_t>(loc) % 8)
    return cudaErrorNotSupported;
  DenseExactArgs a{};
  a.feat = f.data;
  a.n_rows = f.n_rows;
  a.C = C;
  a.Q = Q;
  a.P = P;
  a.cams = f.n_cams;
  a.L = f.n_levels;
  a.G = G;
  a.cpg = C / G;
  a.shape = f.spatial_shape;
  a.start = f.scale_start_index;
  a.loc = loc;
  a.w = w;
  a.out = out;
  a.n_queries = (int64_t)f.batch * Q;
  a.one2 = make_float2(1.0f, 1.0f);
  a.nz2 = make_float2(-0.0f, -0.0f);
  a.ncs_pad = (f.n_levels * P + 3) / 4 * 4;
  a.status = status;
  switch (f.dtype) {  // the ring stays within one camera ahead of the consumer (D < levels x keypoints)
    case MSDA_F32: return launch_dx_depth<float, 4>(a, stream);
    case MSDA_F16: return launch_dx_depth<__half, 8>(a, stream);
    default: return launch_dx_depth<__nv_bfloat16, 8>(a, stream);
  }
}

}  // namespace msda
