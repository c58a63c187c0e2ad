// Exact (bit-faithful) MSDA over a CSR sample plan — sm_100a.
//
// Two kernels per call:
//   plan_canon_kernel  one CTA per query: canonical sort of the query's
//                      samples by (camera, level, v, u, weight)
//                      (features.py:261-263), sequential f32 weight sum in that
//                      order (features.py:264-269), then one 32-B SampleRec +
//                      normalised weight per sample, written back in canonical
//                      order.  Sort is a bitonic network on 128-bit keys in
//                      shared memory (global scratch for very long queries).
//   gather_exact_kernel one thread per (query, VEC-channel slice): walks the
//                      query's records in canonical order, 16-B vector gathers
//                      of the four corner rows (channel-last layout), the
//                      reference f32 expression tree
//                      ((c00*w00 + c10*w10) + (c01*w01 + c11*w11)) * wn, and a
//                      sequential f32 accumulate (features.py:219, 271-274).
//                      Every op is separately rounded (__fmul_rn/__fadd_rn), so
//                      the output is bit-identical to msda_reference.  The
//                      EXACT_HALF variant does the same in __half2 with
//                      __hmul2_rn/__hadd2_rn, i.e. msda_optimized(PACKED_HALF)
//                      (features.py:306-359).
#include <algorithm>
#include <type_traits>

#include "msda_common.cuh"
#include "msda_exact.cuh"

namespace msda {

namespace {

constexpr int kPlanThreads = 256;

struct PlanArgs {
  const int64_t* offsets;
  const int32_t* cam;
  const int32_t* lvl;
  const float* u;
  const float* v;
  const float* w;
  int64_t n_queries;
  int32_t n_cams, n_levels;
  const int32_t* shape;
  const int64_t* start;
  int32_t normalize;
  int32_t smem_cap;
  SampleRec* rec;
  float* wn;
  unsigned long long* g_hi;  // global sort scratch [S] (long queries only)
  unsigned long long* g_lo;
  DevStatus* status;
};

__device__ __forceinline__ bool key_gt(unsigned long long ah, unsigned long long al, unsigned long long bh,
                                       unsigned long long bl) {
  return ah > bh || (ah == bh && al > bl);
}

// Always-ascending bitonic network over n keys, virtually padded with +inf to
// the next power of two (a compare with a padded partner is a no-op, so no
// padding is ever stored).
__device__ void bitonic_sort(unsigned long long* hi, unsigned long long* lo, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (N >> 1); t += blockDim.x) {
        const int i = (t / j) * 2 * j + (t % j);
        const int p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i + j);
        if (p < n) {
          unsigned long long ih = hi[i], il = lo[i], ph = hi[p], pl = lo[p];
          if (key_gt(ih, il, ph, pl)) {
            hi[i] = ph;
            lo[i] = pl;
            hi[p] = ih;
            lo[p] = il;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kPlanThreads) plan_canon_kernel(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* s_hi = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* s_lo = s_hi + a.smem_cap;
  __shared__ float s_wsum;
  const int n_tiles = a.n_cams * a.n_levels;

  for (int64_t q = blockIdx.x; q < a.n_queries; q += gridDim.x) {
    const int64_t lo = a.offsets[q], hi = a.offsets[q + 1];
    const int n = (int)(hi - lo);
    if (n <= 0) continue;
    unsigned long long* khi = (n <= a.smem_cap) ? s_hi : a.g_hi + lo;
    unsigned long long* klo = (n <= a.smem_cap) ? s_lo : a.g_lo + lo;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t s = lo + i;
      int c = a.cam[s], l = a.lvl[s];
      const float uu = a.u[s], vv = a.v[s], ww = a.w[s];
      if (c < 0 || c >= a.n_cams || l < 0 || l >= a.n_levels) {
        set_status(a.status, MSDA_BAD_TARGET, s);
        c = 0;
        l = 0;
      }
      if (!(isfinite(uu) && isfinite(vv) && isfinite(ww))) set_status(a.status, MSDA_NONFINITE, s);
      const unsigned long long tile = (unsigned long long)(c * a.n_levels + l);
      khi[i] = (tile << 32) | ord_f32(vv);
      klo[i] = ((unsigned long long)ord_f32(uu) << 32) | ord_f32(ww);
    }
    __syncthreads();
    bitonic_sort(khi, klo, n);
    if (threadIdx.x == 0) {
      float ws = 0.0f;
      if (a.normalize) {
        // sequential float32 sum in canonical order (features.py:264-267)
        for (int i = 0; i < n; ++i) ws = __fadd_rn(ws, unord_f32((uint32_t)(klo[i] & 0xffffffffu)));
        if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, q);
      }
      s_wsum = ws;
    }
    __syncthreads();
    const float wsum = s_wsum;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long kh = khi[i], kl = klo[i];
      const int t = (int)(kh >> 32);
      const float vv = unord_f32((uint32_t)(kh & 0xffffffffu));
      const float uu = unord_f32((uint32_t)(kl >> 32));
      const float ww = unord_f32((uint32_t)(kl & 0xffffffffu));
      const int tt = t < n_tiles ? t : 0;
      a.rec[lo + i] = make_record(uu, vv, a.start[tt], a.shape[2 * tt], a.shape[2 * tt + 1]);
      a.wn[lo + i] = a.normalize ? __fdiv_rn(ww, wsum) : ww;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// gather / accumulate

struct GatherArgs {
  const void* feat;
  int32_t C;
  int64_t n_queries;
  const int64_t* offsets;
  const SampleRec* rec;
  const float* wn;
  float* out;
  uint8_t* empty;
};

__device__ __forceinline__ SampleRec ld_rec(const SampleRec* p) {
  SampleRec r;
  asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.row[0]), "=r"(r.row[1]), "=r"(r.row[2]), "=r"(r.row[3])
               : "l"(p));
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.iw[0]), "=f"(r.iw[1]), "=f"(r.iw[2]), "=f"(r.iw[3])
               : "l"(reinterpret_cast<const char*>(p) + 16));
  return r;
}

// T: storage type; VEC: channels per thread; HALF: f16 arithmetic.
template <typename T, int VEC, bool HALF, int UNROLL>
__global__ void __launch_bounds__(256) gather_exact_kernel(GatherArgs a) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int lanes_per_q = a.C / VEC;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t q = gtid / lanes_per_q;
  if (q >= a.n_queries) return;
  const int c0 = (int)(gtid - q * lanes_per_q) * VEC;
  const int64_t lo = a.offsets[q], hi = a.offsets[q + 1];
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)c0 * sizeof(T);
  const size_t row_bytes = (size_t)a.C * sizeof(T);

  float accf[VEC];
  __half2 acch[VEC / 2 > 0 ? VEC / 2 : 1];
#pragma unroll
  for (int e = 0; e < VEC; ++e) accf[e] = 0.0f;
#pragma unroll
  for (int e = 0; e < (VEC / 2 > 0 ? VEC / 2 : 1); ++e) acch[e] = __float2half2_rn(0.0f);

  int64_t i = lo;
  for (; i < hi; i += UNROLL) {
    SampleRec r[UNROLL];
    float s[UNROLL];
    RawVec<BYTES> cv[UNROLL][4];
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      if (i + j < hi) {
        r[j] = ld_rec(a.rec + i + j);
        s[j] = __ldg(a.wn + i + j);
      } else {
        r[j].row[0] = r[j].row[1] = r[j].row[2] = r[j].row[3] = -1;
        r[j].iw[0] = r[j].iw[1] = r[j].iw[2] = r[j].iw[3] = 0.0f;
        s[j] = 0.0f;
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cv[j][k] = (r[j].row[k] >= 0) ? ldg_vec<BYTES>(feat + (size_t)r[j].row[k] * row_bytes) : zero_vec<BYTES>();
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      if (i + j >= hi) break;
      if constexpr (!HALF) {
        float c[4][VEC];
#pragma unroll
        for (int k = 0; k < 4; ++k) to_f32<T, VEC>(cv[j][k], c[k]);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float t = __fadd_rn(__fadd_rn(__fmul_rn(c[0][e], r[j].iw[0]), __fmul_rn(c[1][e], r[j].iw[1])),
                                    __fadd_rn(__fmul_rn(c[2][e], r[j].iw[2]), __fmul_rn(c[3][e], r[j].iw[3])));
          accf[e] = __fadd_rn(accf[e], __fmul_rn(s[j], t));
        }
      } else {
        const __half2 hw0 = __float2half2_rn(r[j].iw[0]);
        const __half2 hw1 = __float2half2_rn(r[j].iw[1]);
        const __half2 hw2 = __float2half2_rn(r[j].iw[2]);
        const __half2 hw3 = __float2half2_rn(r[j].iw[3]);
        const __half2 hs = __float2half2_rn(s[j]);
        const __half2* h0 = reinterpret_cast<const __half2*>(&cv[j][0]);
        const __half2* h1 = reinterpret_cast<const __half2*>(&cv[j][1]);
        const __half2* h2 = reinterpret_cast<const __half2*>(&cv[j][2]);
        const __half2* h3 = reinterpret_cast<const __half2*>(&cv[j][3]);
#pragma unroll
        for (int e = 0; e < VEC / 2; ++e) {
          const __half2 t = __hadd2_rn(__hadd2_rn(__hmul2_rn(h0[e], hw0), __hmul2_rn(h1[e], hw1)),
                                       __hadd2_rn(__hmul2_rn(h2[e], hw2), __hmul2_rn(h3[e], hw3)));
          acch[e] = __hadd2_rn(acch[e], __hmul2_rn(t, hs));
        }
      }
    }
  }

  float* o = a.out + q * a.C + c0;
  if constexpr (!HALF) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) o[e] = accf[e];
  } else {
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) {
      const float2 f = __half22float2(acch[e]);
      o[2 * e] = f.x;
      o[2 * e + 1] = f.y;
    }
  }
  if (c0 == 0 && a.empty) a.empty[q] = (hi == lo) ? 1 : 0;
}

template <typename T, int VEC, bool HALF>
cudaError_t launch_gather(const GatherArgs& g, cudaStream_t stream) {
  const int lanes = g.C / VEC;
  const int64_t threads = g.n_queries * lanes;
  const int block = 256;
  const int64_t grid = (threads + block - 1) / block;
  if (grid == 0) return cudaSuccess;
  gather_exact_kernel<T, VEC, HALF, 4><<<(unsigned)grid, block, 0, stream>>>(g);
  return cudaGetLastError();
}

}  // namespace

size_t exact_workspace_bytes(int64_t n_queries, int64_t n_samples) {
  (void)n_queries;
  size_t b = kStatusBytes;
  b += align_up((size_t)n_samples * sizeof(SampleRec), 256);
  b += align_up((size_t)n_samples * sizeof(float), 256);
  b += 2 * align_up((size_t)n_samples * sizeof(unsigned long long), 256);
  return b;
}

ExactWorkspace carve_exact_workspace(void* ws, int64_t n_samples) {
  ExactWorkspace w;
  char* p = reinterpret_cast<char*>(ws);
  w.status = reinterpret_cast<DevStatus*>(p);
  p += kStatusBytes;
  w.rec = reinterpret_cast<SampleRec*>(p);
  p += align_up((size_t)n_samples * sizeof(SampleRec), 256);
  w.wn = reinterpret_cast<float*>(p);
  p += align_up((size_t)n_samples * sizeof(float), 256);
  w.g_hi = reinterpret_cast<unsigned long long*>(p);
  p += align_up((size_t)n_samples * sizeof(unsigned long long), 256);
  w.g_lo = reinterpret_cast<unsigned long long*>(p);
  return w;
}

cudaError_t launch_plan_canon(const msda_features_t& f, const msda_csr_plan_t& p, int normalize,
                              const ExactWorkspace& w, int num_sms, cudaStream_t stream) {
  if (p.n_queries == 0) return cudaSuccess;
  PlanArgs a;
  a.offsets = p.offsets;
  a.cam = p.camera_index;
  a.lvl = p.level;
  a.u = p.u;
  a.v = p.v;
  a.w = p.weight;
  a.n_queries = p.n_queries;
  a.n_cams = f.n_cams;
  a.n_levels = f.n_levels;
  a.shape = f.spatial_shape;
  a.start = f.scale_start_index;
  a.normalize = normalize;
  a.smem_cap = 2048;  // 32 KB of keys per CTA; longer queries sort in global scratch
  a.rec = w.rec;
  a.wn = w.wn;
  a.g_hi = w.g_hi;
  a.g_lo = w.g_lo;
  a.status = w.status;
  const size_t smem = (size_t)a.smem_cap * 2 * sizeof(unsigned long long);
  const int64_t grid = std::min<int64_t>(p.n_queries, (int64_t)num_sms * 16);
  plan_canon_kernel<<<(unsigned)grid, kPlanThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather_exact(const msda_features_t& f, const msda_csr_plan_t& p, int precision,
                                const ExactWorkspace& w, float* out, uint8_t* empty, cudaStream_t stream) {
  GatherArgs g;
  g.feat = f.data;
  g.C = f.channels;
  g.n_queries = p.n_queries;
  g.offsets = p.offsets;
  g.rec = w.rec;
  g.wn = w.wn;
  g.out = out;
  g.empty = empty;
  const uintptr_t base = reinterpret_cast<uintptr_t>(f.data);
  const int C = f.channels;
  if (precision == MSDA_EXACT_HALF) {
    if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, true>(g, stream);
    if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, true>(g, stream);
    return launch_gather<__half, 2, true>(g, stream);
  }
  switch (f.dtype) {
    case MSDA_F32:
      if (C % 4 == 0 && base % 16 == 0) return launch_gather<float, 4, false>(g, stream);
      return launch_gather<float, 2, false>(g, stream);
    case MSDA_F16:
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, false>(g, stream);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, false>(g, stream);
      return launch_gather<__half, 2, false>(g, stream);
    default:
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__nv_bfloat16, 8, false>(g, stream);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__nv_bfloat16, 4, false>(g, stream);
      return launch_gather<__nv_bfloat16, 2, false>(g, stream);
  }
}

}  // namespace msda
