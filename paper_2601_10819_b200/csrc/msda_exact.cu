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
  int64_t queries_per_batch;  // query q reads batch q / queries_per_batch ...
  int64_t rows_per_batch;     // ... whose table starts rows_per_batch rows later
  SampleRec* rec;
  float* wn;
  unsigned long long* g_hi;  // global sort scratch [S] (long queries only)
  unsigned long long* g_lo;
  DevStatus* status;
};

template <typename K>
__device__ __forceinline__ bool key_gt(K ah, K al, K bh, K bl) {
  return ah > bh || (ah == bh && al > bl);
}

// Always-ascending bitonic network over n keys, virtually padded with +inf to
// the next power of two (a compare with a padded partner is a no-op, so no
// padding is ever stored).  j is a power of two: index math is shifts/masks.
template <typename K>
__device__ void bitonic_sort(K* hi, K* lo, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int lj = __ffs(j) - 1;
      const bool flip = (j == (k >> 1));
      for (int t = threadIdx.x; t < (N >> 1); t += blockDim.x) {
        const int i = ((t >> lj) << (lj + 1)) | (t & (j - 1));
        const int p = flip ? (i ^ (k - 1)) : (i + j);
        if (p < n) {
          const K ih = hi[i], il = lo[i], ph = hi[p], pl = lo[p];
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

constexpr int kRunCap = 128;  // longest (camera, level) run the rank path handles

// first index in [0, n) whose tile (key_hi >> 32) is >= t (keys tile-sorted)
template <typename K>
__device__ __forceinline__ int tile_lower_bound(const K* hi, int n, uint32_t t) {
  int a = 0, b = n;
  while (a < b) {
    const int m = (a + b) >> 1;
    if ((uint32_t)(hi[m] >> 32) < t) a = m + 1; else b = m;
  }
  return a;
}

// Canonicalise one query whose keys sit in (khi, klo): sorted keys end up in
// (shi, slo).  When the samples already arrive grouped by (camera, level) —
// the reference bench generator and every dense expansion do — each sample's
// final slot is its run start plus its rank inside the run, computed in
// parallel; otherwise a bitonic sort.  Returns the sequential f32 weight sum.
template <typename K>
__device__ float canon_query(const PlanArgs& a, int64_t q, int n, K* khi, K* klo, K* shi, K* slo, float* s_wsum,
                             int* s_flag) {
  // tile-sortedness and longest run
  bool bad = false;
  for (int i = threadIdx.x + 1; i < n; i += blockDim.x) bad |= (khi[i] >> 32) < (khi[i - 1] >> 32);
  const bool tile_sorted = !__syncthreads_or(bad);
  bool rank_path = tile_sorted;
  if (tile_sorted) {
    bool long_run = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (i > 0 && (khi[i] >> 32) == (khi[i - 1] >> 32)) continue;  // only run heads probe
      const uint32_t t = (uint32_t)(khi[i] >> 32);
      long_run |= (tile_lower_bound(khi, n, t + 1) - i) > kRunCap;
    }
    rank_path = !__syncthreads_or(long_run);
  }
  if (rank_path) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const K ih = khi[i], il = klo[i];
      const uint32_t t = (uint32_t)(ih >> 32);
      const int rs = tile_lower_bound(khi, n, t);
      const int re = tile_lower_bound(khi, n, t + 1);
      int rank = 0;
      for (int j = rs; j < re; ++j) {
        const K jh = khi[j], jl = klo[j];
        rank += (jh < ih || (jh == ih && (jl < il || (jl == il && j < i)))) ? 1 : 0;
      }
      shi[rs + rank] = ih;
      slo[rs + rank] = il;
    }
  } else {
    bitonic_sort(khi, klo, n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      shi[i] = khi[i];
      slo[i] = klo[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float ws = 0.0f;
    if (a.normalize) {
      // sequential float32 sum in canonical order (features.py:264-267);
      // loads run ahead of the dependent add chain
      int i = 0;
      for (; i + 4 <= n; i += 4) {
        const K k0 = slo[i], k1 = slo[i + 1], k2 = slo[i + 2], k3 = slo[i + 3];
        ws = __fadd_rn(ws, unord_f32((uint32_t)(k0 & 0xffffffffu)));
        ws = __fadd_rn(ws, unord_f32((uint32_t)(k1 & 0xffffffffu)));
        ws = __fadd_rn(ws, unord_f32((uint32_t)(k2 & 0xffffffffu)));
        ws = __fadd_rn(ws, unord_f32((uint32_t)(k3 & 0xffffffffu)));
      }
      for (; i < n; ++i) ws = __fadd_rn(ws, unord_f32((uint32_t)(slo[i] & 0xffffffffu)));
      if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, q);
    }
    *s_wsum = ws;
  }
  __syncthreads();
  (void)s_flag;
  return *s_wsum;
}

__global__ void __launch_bounds__(kPlanThreads) plan_canon_kernel(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* s_hi = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* s_lo = s_hi + a.smem_cap;
  unsigned long long* s_shi = s_lo + a.smem_cap;
  unsigned long long* s_slo = s_shi + a.smem_cap;
  __shared__ float s_wsum;
  __shared__ int s_flag;
  const int n_tiles = a.n_cams * a.n_levels;

  for (int64_t q = blockIdx.x; q < a.n_queries; q += gridDim.x) {
    const int64_t lo = a.offsets[q], hi = a.offsets[q + 1];
    const int n = (int)(hi - lo);
    if (n <= 0) continue;
    const bool in_smem = n <= a.smem_cap;
    unsigned long long* khi = in_smem ? s_hi : a.g_hi + lo;
    unsigned long long* klo = in_smem ? s_lo : a.g_lo + lo;
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
    // sorted keys: shared memory, or (long queries) the record area as scratch
    // — records are written after the keys are consumed, one slot per sample.
    unsigned long long* shi;
    unsigned long long* slo;
    float wsum;
    if (in_smem) {
      shi = s_shi;
      slo = s_slo;
      wsum = canon_query(a, q, n, s_hi, s_lo, s_shi, s_slo, &s_wsum, &s_flag);
    } else {
      shi = reinterpret_cast<unsigned long long*>(a.rec + lo);  // 32 B/sample holds 16 B of key
      slo = shi + n;
      wsum = canon_query(a, q, n, khi, klo, shi, slo, &s_wsum, &s_flag);
      // keys may not live in the record area while records are written:
      // move them back into the key scratch first
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        khi[i] = shi[i];
        klo[i] = slo[i];
      }
      __syncthreads();
      shi = khi;
      slo = klo;
    }
    const int64_t row_base = (q / a.queries_per_batch) * a.rows_per_batch;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long kh = shi[i], kl = slo[i];
      const int t = (int)(kh >> 32);
      const float vv = unord_f32((uint32_t)(kh & 0xffffffffu));
      const float uu = unord_f32((uint32_t)(kl >> 32));
      const float ww = unord_f32((uint32_t)(kl & 0xffffffffu));
      const int tt = t < n_tiles ? t : 0;
      a.rec[lo + i] = make_record(uu, vv, row_base + a.start[tt], a.shape[2 * tt], a.shape[2 * tt + 1]);
      a.wn[lo + i] = a.normalize ? __fdiv_rn(ww, wsum) : ww;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// gather / accumulate

struct GatherArgs {
  const void* feat;
  int32_t C;          // channels processed (slice width)
  int32_t row_elems;  // elements per feature row (full C)
  int32_t c_off;      // first channel of the slice
  int32_t out_stride; // floats per output row
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
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)(a.c_off + c0) * sizeof(T);
  const size_t row_bytes = (size_t)a.row_elems * sizeof(T);

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

  float* o = a.out + q * a.out_stride + a.c_off + c0;
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

// ---------------------------------------------------------------------------
// Pipelined gather (the production path when a query's channel slice spans
// whole warps).  Same arithmetic and order as gather_exact_kernel; the
// difference is memory-level parallelism: each lane keeps D samples' corner
// rows in flight with cp.async (LDGSTS, zero-fill for out-of-grid corners)
// into a per-warp shared-memory ring, and the query's records are staged 32 at
// a time in shared memory (one coalesced load per lane, read back as warp
// broadcasts), fetched one batch ahead.  Registers stay low, so the ring depth
// — not the register file — sets the bytes in flight per SM.

template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? BYTES : 0;
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "r"(n));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

template <int BYTES, int D>
struct PipeSmem {
  static constexpr int kCorner = D * 4 * 32 * BYTES;        // corner ring
  static constexpr int kRows = 2 * 32 * 16;                 // int4 rows[2][32]
  static constexpr int kIw = 2 * 32 * 16;                   // float4 iw[2][32]
  static constexpr int kWn = 2 * 32 * 4;                    // float wn[2][32]
  static constexpr int kPerWarp = kCorner + kRows + kIw + kWn;
};

constexpr int kPipeWarps = 2;

template <typename T, int VEC, bool HALF, int D>
__global__ void __launch_bounds__(kPipeWarps * 32) gather_pipe_kernel(GatherArgs a) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  using SM = PipeSmem<BYTES, D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + warp * SM::kPerWarp;
  int4* s_rows = reinterpret_cast<int4*>(base + SM::kCorner);
  float4* s_iw = reinterpret_cast<float4*>(base + SM::kCorner + SM::kRows);
  float* s_wn = reinterpret_cast<float*>(base + SM::kCorner + SM::kRows + SM::kIw);
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(base) + lane * BYTES;

  const int warps_per_q = a.C / VEC / 32;
  const int64_t gw = (int64_t)blockIdx.x * kPipeWarps + warp;
  const int64_t q = gw / warps_per_q;
  if (q >= a.n_queries) return;
  const int c0 = (int)(gw - q * warps_per_q) * 32 * VEC + lane * VEC;
  const int64_t lo = a.offsets[q], hi = a.offsets[q + 1];
  const int64_t n = hi - lo;
  const char* featc = reinterpret_cast<const char*>(a.feat) + (size_t)(a.c_off + c0) * sizeof(T);
  const size_t row_bytes = (size_t)a.row_elems * sizeof(T);

  // record batch b: lane j holds sample lo + 32 b + j
  int4 r_rows = make_int4(-1, -1, -1, -1);
  float4 r_iw = make_float4(0.f, 0.f, 0.f, 0.f);
  float r_wn = 0.0f;
  auto load_batch = [&](int64_t b) {
    const int64_t s = lo + b * 32 + lane;
    if (s < hi) {
      const SampleRec r = ld_rec(a.rec + s);
      r_rows = make_int4(r.row[0], r.row[1], r.row[2], r.row[3]);
      r_iw = make_float4(r.iw[0], r.iw[1], r.iw[2], r.iw[3]);
      r_wn = __ldg(a.wn + s);
    }
  };
  auto store_batch = [&](int buf) {
    s_rows[buf * 32 + lane] = r_rows;
    s_iw[buf * 32 + lane] = r_iw;
    s_wn[buf * 32 + lane] = r_wn;
  };
  auto issue = [&](int64_t k) {
    const int buf = (int)((k >> 5) & 1), j = (int)(k & 31);
    const int4 rows = s_rows[buf * 32 + j];
    const uint32_t dst = ring + (uint32_t)((k % D) * 4 * 32 * BYTES);
    cp_async_zfill<BYTES>(dst, rows.x >= 0 ? featc + (size_t)rows.x * row_bytes : featc, rows.x >= 0);
    cp_async_zfill<BYTES>(dst + 32 * BYTES, rows.y >= 0 ? featc + (size_t)rows.y * row_bytes : featc, rows.y >= 0);
    cp_async_zfill<BYTES>(dst + 64 * BYTES, rows.z >= 0 ? featc + (size_t)rows.z * row_bytes : featc, rows.z >= 0);
    cp_async_zfill<BYTES>(dst + 96 * BYTES, rows.w >= 0 ? featc + (size_t)rows.w * row_bytes : featc, rows.w >= 0);
  };

  load_batch(0);
  store_batch(0);
  __syncwarp();
  load_batch(1);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < n) issue(k);
    cp_async_commit();
  }

  float accf[VEC];
  __half2 acch[VEC / 2 > 0 ? VEC / 2 : 1];
#pragma unroll
  for (int e = 0; e < VEC; ++e) accf[e] = 0.0f;
#pragma unroll
  for (int e = 0; e < (VEC / 2 > 0 ? VEC / 2 : 1); ++e) acch[e] = __float2half2_rn(0.0f);

  for (int64_t i = 0; i < n; ++i) {
    cp_async_wait<D - 1>();
    const int buf = (int)((i >> 5) & 1), j = (int)(i & 31);
    const float4 iw = s_iw[buf * 32 + j];
    const float wn = s_wn[buf * 32 + j];
    const unsigned char* src = base + (size_t)((i % D) * 4 * 32 + lane) * BYTES;
    RawVec<BYTES> cv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cv[k] = *reinterpret_cast<const RawVec<BYTES>*>(src + k * 32 * BYTES);
    if constexpr (!HALF) {
      float c[4][VEC];
#pragma unroll
      for (int k = 0; k < 4; ++k) to_f32<T, VEC>(cv[k], c[k]);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const float t = __fadd_rn(__fadd_rn(__fmul_rn(c[0][e], iw.x), __fmul_rn(c[1][e], iw.y)),
                                  __fadd_rn(__fmul_rn(c[2][e], iw.z), __fmul_rn(c[3][e], iw.w)));
        accf[e] = __fadd_rn(accf[e], __fmul_rn(wn, t));
      }
    } else {
      const __half2 hw0 = __float2half2_rn(iw.x), hw1 = __float2half2_rn(iw.y);
      const __half2 hw2 = __float2half2_rn(iw.z), hw3 = __float2half2_rn(iw.w);
      const __half2 hs = __float2half2_rn(wn);
      const __half2* h0 = reinterpret_cast<const __half2*>(&cv[0]);
      const __half2* h1 = reinterpret_cast<const __half2*>(&cv[1]);
      const __half2* h2 = reinterpret_cast<const __half2*>(&cv[2]);
      const __half2* h3 = reinterpret_cast<const __half2*>(&cv[3]);
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        const __half2 t = __hadd2_rn(__hadd2_rn(__hmul2_rn(h0[e], hw0), __hmul2_rn(h1[e], hw1)),
                                     __hadd2_rn(__hmul2_rn(h2[e], hw2), __hmul2_rn(h3[e], hw3)));
        acch[e] = __hadd2_rn(acch[e], __hmul2_rn(t, hs));
      }
    }
    const int64_t k = i + D;
    if (k < n) {
      if ((k & 31) == 0) {  // entering record batch k/32: publish it, prefetch the next
        __syncwarp();
        store_batch((int)((k >> 5) & 1));
        __syncwarp();
        load_batch((k >> 5) + 1);
      }
      issue(k);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();

  float* o = a.out + q * a.out_stride + a.c_off + c0;
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
  if (c0 == 0 && a.empty) a.empty[q] = (n == 0) ? 1 : 0;
}

template <typename T, int VEC, bool HALF, int D>
cudaError_t launch_gather_pipe(const GatherArgs& g, cudaStream_t stream) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int smem = kPipeWarps * PipeSmem<BYTES, D>::kPerWarp;
  static bool attr_set = false;  // per instantiation; benign race (idempotent)
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gather_pipe_kernel<T, VEC, HALF, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t warps = g.n_queries * (g.C / VEC / 32);
  const int64_t grid = (warps + kPipeWarps - 1) / kPipeWarps;
  if (grid == 0) return cudaSuccess;
  gather_pipe_kernel<T, VEC, HALF, D><<<(unsigned)grid, kPipeWarps * 32, smem, stream>>>(g);
  return cudaGetLastError();
}

template <typename T, int VEC, bool HALF>
cudaError_t launch_gather(const GatherArgs& g, cudaStream_t stream) {
  if ((g.C / VEC) % 32 == 0 && g.C % VEC == 0) {
    if constexpr (VEC * sizeof(T) == 16) return launch_gather_pipe<T, VEC, HALF, 6>(g, stream);
    else return launch_gather_pipe<T, VEC, HALF, 8>(g, stream);
  }
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
                              const ExactWorkspace& w, int num_sms, cudaStream_t stream,
                              int64_t queries_per_batch) {
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
  a.smem_cap = 1024;  // 32 KB of keys (unsorted + sorted) per CTA; longer queries use global scratch
  a.queries_per_batch = queries_per_batch > 0 ? queries_per_batch : (p.n_queries > 0 ? p.n_queries : 1);
  a.rows_per_batch = f.n_rows;
  a.rec = w.rec;
  a.wn = w.wn;
  a.g_hi = w.g_hi;
  a.g_lo = w.g_lo;
  a.status = w.status;
  const size_t smem = (size_t)a.smem_cap * 4 * sizeof(unsigned long long);
  const int64_t grid = std::min<int64_t>(p.n_queries, (int64_t)num_sms * 16);
  plan_canon_kernel<<<(unsigned)grid, kPlanThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather_exact(const msda_features_t& f, const msda_csr_plan_t& p, int precision,
                                const ExactWorkspace& w, float* out, uint8_t* empty, cudaStream_t stream,
                                int c_off, int c_count) {
  GatherArgs g;
  g.feat = f.data;
  if (c_count <= 0) {
    c_off = 0;
    c_count = f.channels;
  }
  g.C = c_count;
  g.row_elems = f.channels;
  g.c_off = c_off;
  g.out_stride = f.channels;
  g.n_queries = p.n_queries;
  g.offsets = p.offsets;
  g.rec = w.rec;
  g.wn = w.wn;
  g.out = out;
  g.empty = empty;
  const size_t esz = f.dtype == MSDA_F32 ? 4 : 2;
  // vector width must divide the slice and keep every row access aligned
  const uintptr_t base = reinterpret_cast<uintptr_t>(f.data) | ((size_t)c_off * esz) | ((size_t)f.channels * esz);
  const int C = c_count;
  if (precision == MSDA_EXACT_HALF) {
    if (C % 128 == 0 && base % 8 == 0) return launch_gather<__half, 4, true>(g, stream);
    if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, true>(g, stream);
    if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, true>(g, stream);
    return launch_gather<__half, 2, true>(g, stream);
  }
  switch (f.dtype) {
    case MSDA_F32:
      if (C % 4 == 0 && base % 16 == 0) return launch_gather<float, 4, false>(g, stream);
      if (C % 64 == 0 && base % 8 == 0) return launch_gather<float, 2, false>(g, stream);
      return launch_gather<float, 2, false>(g, stream);
    case MSDA_F16:
      if (C % 128 == 0 && base % 8 == 0) return launch_gather<__half, 4, false>(g, stream);
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, false>(g, stream);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, false>(g, stream);
      return launch_gather<__half, 2, false>(g, stream);
    default:
      if (C % 128 == 0 && base % 8 == 0) return launch_gather<__nv_bfloat16, 4, false>(g, stream);
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__nv_bfloat16, 8, false>(g, stream);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__nv_bfloat16, 4, false>(g, stream);
      return launch_gather<__nv_bfloat16, 2, false>(g, stream);
  }
}

}  // namespace msda
