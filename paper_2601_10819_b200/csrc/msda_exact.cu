// Exact (bit-faithful) MSDA over a CSR sample plan — sm_100a.
//
// Two kernels per call:
//
//   plan_canon_kernel   one 128-thread CTA per query.  Builds 128-bit keys
//                       (tile = camera*L + level, v, u, weight) with an
//                       order-preserving float map, i.e. the canonical order
//                       of features.py:261-263.  When the query arrives grouped
//                       by (camera, level) — the reference bench generator and
//                       every dense expansion do — each sample's canonical
//                       slot is its run start (a shared-memory table built in
//                       the same pass that checks the grouping) plus its rank
//                       in the run (one 64-bit (v, u) compare per run member),
//                       and its 32-B SampleRec and raw weight are written there
//                       in that pass; otherwise a bitonic sort.  Then the
//                       sequential f32 weight sum in canonical order
//                       (features.py:264-269), one float per query.
//
//   gather_pipe_kernel  one warp per (query, 32*VEC channels): walks the
//                       query's records in canonical order (its batch loader
//                       turns each raw weight into w / sum, features.py:271-
//                       273).  Corner rows
//                       (channel-last, 16-B per lane, whole 32-B sectors) are
//                       prefetched D samples ahead with cp.async (LDGSTS,
//                       zero-fill for out-of-grid corners) into a per-warp
//                       shared-memory ring; records are staged 32 at a time.
//                       The reference f32 expression tree
//                       ((c00*w00 + c10*w10) + (c01*w01 + c11*w11)) * wn and
//                       the sequential accumulate (features.py:219, 271-274)
//                       are evaluated two channels per instruction with FFMA2,
//                       every product and sum separately rounded (the 1.0 and
//                       -0.0 operands come from kernel parameters so ptxas
//                       cannot fuse them) — bit-identical to msda_reference.
//                       The PACKED_HALF variant does the same with
//                       __hmul2_rn/__hadd2_rn (features.py:306-359).
//
//   gather_exact_kernel register-pipelined fallback for channel slices that do
//                       not span whole warps (small C in tests / odd groups).
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "msda_common.cuh"
#include "msda_exact.cuh"

#ifdef MSDA_PLAN_TL  // builder-only timeline (tools/plan_timeline.py): globaltimer stamps, never shipped
__device__ unsigned long long g_msda_tl[8192][8];
#define MSDA_TL(slot, k)                                                              \
  do {                                                                                \
    if ((threadIdx.x & 31) == 0 && (slot) < 8192) {                                   \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_msda_tl[(slot)][(k)] = t_;                                                    \
    }                                                                                 \
  } while (0)
#define MSDA_TL_SMID(slot)                                                            \
  do {                                                                                \
    uint32_t s_;                                                                      \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));                                  \
    if ((threadIdx.x & 31) == 0 && (slot) < 8192) g_msda_tl[(slot)][3] = s_;          \
  } while (0)
extern "C" int msda_debug_timeline(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_msda_tl, bytes < sizeof(g_msda_tl) ? bytes : sizeof(g_msda_tl));
}
#else
#define MSDA_TL(slot, k) \
  do {                   \
  } while (0)
#define MSDA_TL_SMID(slot) \
  do {                     \
  } while (0)
#endif
#define MSDA_TL_WARP (2048 + (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)))

namespace msda {

namespace {

constexpr int kPlanThreads = 128;
constexpr int kPlanSmemCap = 1024;  // samples per query canonicalised in shared memory
constexpr int kRunCap = 256;        // longest (camera, level) run the rank path handles

using u64 = unsigned long long;

struct PlanArgs {
  const int64_t* offsets;
  const int32_t* cam;
  const int32_t* lvl;
  const float* u;
  const float* v;
  const float* w;
  int64_t n_queries;
  int64_t n_samples;  // offsets must satisfy 0 <= offsets[q] <= offsets[q + 1] <= n_samples
  int32_t n_cams, n_levels;
  const int32_t* shape;
  const int64_t* start;
  int32_t normalize;
  int64_t queries_per_batch;  // query q reads batch q / queries_per_batch ...
  int64_t rows_per_batch;     // ... whose table starts rows_per_batch rows later
  SampleRec* rec;
  float* wn;    // [S] raw weights in canonical order (the gather divides by qsum)
  float* qsum;  // [n_queries] sequential f32 weight sum per query (normalize)
  u64* g_hi;  // global scratch [S] for queries longer than kPlanSmemCap
  u64* g_lo;
  int32_t* g_idx;
  DevStatus* status;
};

__device__ __forceinline__ float key_weight(u64 lo) { return unord_f32((uint32_t)(lo & 0xffffffffu)); }

constexpr int kRunTable = 1024;  // tiles whose runs are tabulated in shared memory

// Keys are stored as two words: kt = (tile << 32) | ord(w), kp = (ord(v) << 32)
// | ord(u), so that inside a (camera, level) run one 64-bit compare of kp
// orders (v, u); the weight (and then position) only breaks exact ties.
__device__ __forceinline__ bool canon_gt(u64 at, u64 ap, u64 bt, u64 bp) {
  const uint32_t ta = (uint32_t)(at >> 32), tb = (uint32_t)(bt >> 32);
  if (ta != tb) return ta > tb;
  if (ap != bp) return ap > bp;
  return (uint32_t)at > (uint32_t)bt;
}

// Always-ascending bitonic network on (kt, kp) in canonical order, virtually
// padded with +inf to the next power of two (a compare with a padded partner
// is a no-op, so no padding is stored); j is a power of two: shifts/masks.
__device__ void bitonic_sort_canon(u64* kt, u64* kp, int n) {
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
          const u64 it = kt[i], ip = kp[i], pt = kt[p], pp = kp[p];
          if (canon_gt(it, ip, pt, pp)) {
            kt[i] = pt;
            kp[i] = pp;
            kt[p] = it;
            kp[p] = ip;
          }
        }
      }
      __syncthreads();
    }
  }
}

// sequential float32 sum in canonical order (features.py:264-267): one
// thread, loads issued well ahead of the dependent add chain
__device__ __forceinline__ float sequential_sum(const float* sw, int n, bool vec_ok) {
  float ws = 0.0f;
  int i = 0;
  if (vec_ok) {  // 32 values loaded ahead of each 32-add stretch of the dependent chain
    for (; i + 32 <= n; i += 32) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = *reinterpret_cast<const float4*>(sw + i + 4 * k);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ws = __fadd_rn(ws, v[k].x);
        ws = __fadd_rn(ws, v[k].y);
        ws = __fadd_rn(ws, v[k].z);
        ws = __fadd_rn(ws, v[k].w);
      }
    }
  }
  for (; i < n; ++i) ws = __fadd_rn(ws, sw[i]);
  return ws;
}

constexpr int kTileTab = 256;  // tiles whose (first row, H, W) a plan CTA keeps in shared memory

// per-CTA shared tables of the plan kernel beside the key arrays (dynamic
// shared memory sized by the tile count: cfg2 23.5 KB per CTA)
struct PlanShared {
  int16_t* run;   // [2 n_run] (first, one past last) position of each tile's run; n_run = 0: no rank path
  int16_t* slot;  // [kPlanSmemCap] rank path: the canonical slot of the key at each position
  int32_t* tstart;  // [n_tab] tile table: first row (batch offset not included); n_tab = 0: read global
  int2* thw;        // [n_tab] (H, W)
  int n_run, n_tab;
};

__host__ __device__ constexpr size_t plan_smem_bytes(int n_tiles) {
  return (size_t)kPlanSmemCap * (8 + 8 + 4 + 2) + (n_tiles <= kRunTable ? 4 * (size_t)n_tiles : 0) +
         (n_tiles <= kTileTab ? 12 * (size_t)n_tiles : 0) + 16;
}

template <bool SMEM>
__device__ __forceinline__ void canon_query(const PlanArgs& a, int64_t q, int64_t lo, int n, int n_tiles, u64* khi,
                                            u64* klo, float* sw, const PlanShared& sh);

__global__ void __launch_bounds__(kPlanThreads, 7) plan_canon_kernel(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char plan_smem[];
  const int n_tiles = a.n_cams * a.n_levels;
  u64* s_hi = reinterpret_cast<u64*>(plan_smem);
  u64* s_lo = s_hi + kPlanSmemCap;
  float* s_w = reinterpret_cast<float*>(s_lo + kPlanSmemCap);
  PlanShared sh;
  sh.slot = reinterpret_cast<int16_t*>(s_w + kPlanSmemCap);
  sh.n_run = n_tiles <= kRunTable ? n_tiles : 0;
  sh.n_tab = n_tiles <= kTileTab ? n_tiles : 0;
  sh.run = sh.slot + kPlanSmemCap;
  sh.thw = reinterpret_cast<int2*>(plan_smem + ((kPlanSmemCap * 22 + 4 * sh.n_run + 7) & ~7));
  sh.tstart = reinterpret_cast<int32_t*>(sh.thw + sh.n_tab);
  // the tile table, read by every record this CTA writes (made visible by the
  // first query's post-load barrier)
  for (int t = threadIdx.x; t < sh.n_tab; t += blockDim.x) {
    sh.tstart[t] = (int32_t)a.start[t];
    sh.thw[t] = make_int2(a.shape[2 * t], a.shape[2 * t + 1]);
  }
  // programmatic dependent launch: the gather grid may be scheduled now; it
  // waits (griddepcontrol.wait) for this grid's completion and memory flush
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) MSDA_TL(blockIdx.x, 0);

  for (int64_t q = blockIdx.x; q < a.n_queries; q += gridDim.x) {
    const int64_t lo = a.offsets[q], hi = a.offsets[q + 1];
    if (lo < 0 || hi < lo || hi > a.n_samples) {  // malformed CSR offsets: report, touch nothing
      if (threadIdx.x == 0) set_status(a.status, MSDA_BAD_ARG, q);
      continue;
    }
    const int n = (int)(hi - lo);
    if (n <= 0) continue;
    // two inlined copies so the shared-memory one compiles to LDS/STS (a
    // pointer chosen at run time between smem and global would be generic)
    if (n <= kPlanSmemCap)
      canon_query<true>(a, q, lo, n, n_tiles, s_hi, s_lo, s_w, sh);
    else  // long query: global scratch (the wn slots double as its weight scratch)
      canon_query<false>(a, q, lo, n, n_tiles, a.g_hi + lo, a.g_lo + lo, a.wn + lo, sh);
  }
  if (threadIdx.x == 0) MSDA_TL(blockIdx.x, 5);
}

template <bool SMEM>
__device__ __forceinline__ void canon_query(const PlanArgs& a, int64_t q, int64_t lo, int n, int n_tiles, u64* khi,
                                            u64* klo, float* sw, const PlanShared& sh) {
  int16_t* s_run = sh.run;
  {
    constexpr int U = 4;  // samples per thread whose loads are in flight together
    for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
      int c[U], l[U];
      float uu[U], vv[U], ww[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = i0 + j * (int)blockDim.x;
        if (i < n) {
          const int64_t s = lo + i;
          c[j] = __ldg(a.cam + s);
          l[j] = __ldg(a.lvl + s);
          uu[j] = __ldg(a.u + s);
          vv[j] = __ldg(a.v + s);
          ww[j] = __ldg(a.w + s);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = i0 + j * (int)blockDim.x;
        if (i < n) {
          if (c[j] < 0 || c[j] >= a.n_cams || l[j] < 0 || l[j] >= a.n_levels) {
            set_status(a.status, MSDA_BAD_TARGET, lo + i);
            c[j] = 0;
            l[j] = 0;
          }
          if (!(isfinite(uu[j]) && isfinite(vv[j]) && isfinite(ww[j]))) set_status(a.status, MSDA_NONFINITE, lo + i);
          khi[i] = ((u64)(c[j] * a.n_levels + l[j]) << 32) | ord_f32(ww[j]);  // kt: tile, weight
          klo[i] = ((u64)ord_f32(vv[j]) << 32) | ord_f32(uu[j]);               // kp: v, u
        }
      }
    }
    __syncthreads();
    if (q == blockIdx.x && threadIdx.x == 0) MSDA_TL(blockIdx.x, 1);
    const int64_t row_base = (q / a.queries_per_batch) * a.rows_per_batch;
    // record + raw weight of the key at canonical slot `slot`
    auto record = [&](u64 kt, u64 kp) {
      const int t = (int)(kt >> 32);
      const float vv = unord_f32((uint32_t)(kp >> 32));
      const float uu = unord_f32((uint32_t)(kp & 0xffffffffu));
      const int tt = t < n_tiles ? t : 0;
      if (sh.n_tab) {  // shared tile table: no dependent global load per record
        const int2 hw = sh.thw[tt];
        return make_record(uu, vv, row_base + sh.tstart[tt], hw.x, hw.y);
      }
      return make_record(uu, vv, row_base + a.start[tt], a.shape[2 * tt], a.shape[2 * tt + 1]);
    };
    auto emit = [&](u64 kt, u64 kp, int slot) {
      a.rec[lo + slot] = record(kt, kp);
      a.wn[lo + slot] = key_weight(kt);
      sw[slot] = key_weight(kt);
    };
    // grouped by (camera, level)?  run heads / tails record their run in the same pass
    bool bad = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t t = (uint32_t)(khi[i] >> 32);
      const uint32_t tp = i > 0 ? (uint32_t)(khi[i - 1] >> 32) : 0xffffffffu;
      const uint32_t tn = i + 1 < n ? (uint32_t)(khi[i + 1] >> 32) : 0xffffffffu;
      bad |= i > 0 && t < tp;
      if (t < (uint32_t)sh.n_run) {
        if (t != tp) s_run[2 * t] = (int16_t)i;
        if (t != tn) s_run[2 * t + 1] = (int16_t)(i + 1);
      }
    }
    bool rank_path = !__syncthreads_or(bad) && sh.n_run > 0 && n <= 32767;
    if (q == blockIdx.x && threadIdx.x == 0) MSDA_TL(blockIdx.x, 2);
    if (rank_path) {  // canonical slot = run start + rank of (v, u) in the run
      bool long_run = false;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const u64 it = khi[i], ip = klo[i];
        const uint32_t t = (uint32_t)(it >> 32);
        const int rs = s_run[2 * t], re = s_run[2 * t + 1];
        if (re - rs > kRunCap) {  // quadratic ranks would be too slow: sort instead
          long_run = true;
          continue;
        }
        // v first: one 32-bit compare per run member (the high words of the
        // (v, u) keys); members with the same v (rare for float
        // coordinates) send the sample to the full (v, u, weight, position)
        // comparison
        const uint32_t* kv = reinterpret_cast<const uint32_t*>(klo) + 1;  // kv[2 j] = ord(v) of key j
        const uint32_t iv = (uint32_t)(ip >> 32);
        int rank = 0;
        bool same_v = false;
#pragma unroll 4
        for (int j = rs; j < re; ++j) {
          const uint32_t jv = kv[2 * j];
          rank += jv < iv ? 1 : 0;
          same_v |= (jv == iv) & (j != i);
        }
        bool tie = false;
        if (same_v) {  // redo with the 64-bit (v, u) keys
          rank = 0;
          for (int j = rs; j < re; ++j) {
            const u64 jp = klo[j];
            rank += jp < ip ? 1 : 0;
            tie |= (jp == ip) & (j != i);
          }
        }
        if (tie) {  // exact (v, u) tie (rare): weight, then position
          const uint32_t wi = (uint32_t)it;
          for (int j = rs; j < re; ++j) {
            if (j == i || klo[j] != ip) continue;
            const uint32_t wj = (uint32_t)khi[j];
            rank += (wj < wi || (wj == wi && j < i)) ? 1 : 0;
          }
        }
        if constexpr (SMEM) {  // records are written below, beside the weight sum
          sh.slot[i] = (int16_t)(rs + rank);
          sw[rs + rank] = key_weight(it);
        } else {
          emit(it, ip, rs + rank);
        }
      }
      rank_path = !__syncthreads_or(long_run);
    }
    if (q == blockIdx.x && threadIdx.x == 0) MSDA_TL(blockIdx.x, 3);
    if (!rank_path) {  // ungrouped or long runs: full bitonic sort, slots = sorted order
      bitonic_sort_canon(khi, klo, n);
      for (int i = threadIdx.x; i < n; i += blockDim.x) emit(khi[i], klo[i], i);
      __syncthreads();
    }
    // sequential f32 sum in canonical order (features.py:264-269) by one
    // thread; on the shared-memory rank path warps 1.. write the records and
    // raw weights meanwhile
    if (SMEM && rank_path && threadIdx.x >= 32) {
      for (int i = threadIdx.x - 32; i < n; i += blockDim.x - 32) {
        const int slot = sh.slot[i];
        const u64 kt = khi[i];
        a.rec[lo + slot] = record(kt, klo[i]);
        a.wn[lo + slot] = key_weight(kt);
      }
    }
    if (threadIdx.x == 0 && a.normalize) {
      const float ws = sequential_sum(sw, n, SMEM);
      if (ws == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, q);
      a.qsum[q] = ws;
    }
    if (q == blockIdx.x && threadIdx.x == 0) MSDA_TL(blockIdx.x, 4);
    __syncthreads();  // shared memory is reused by the next query
  }
}

// ---------------------------------------------------------------------------
// gather / accumulate

struct GatherArgs {
  const void* feat;
  int32_t C;           // channels processed (slice width)
  int32_t row_elems;   // elements per feature row (full C)
  int32_t c_off;       // first channel of the slice
  int32_t out_stride;  // floats per output row
  int64_t n_queries;
  int64_t n_samples;  // CSR offsets are clamped to [0, n_samples] (the plan kernel reports bad ones)
  const int64_t* offsets;
  const SampleRec* rec;
  const float* wn;
  const float* qsum;  // per-query weight sums of the canonical plan (wn holds raw weights), or null
  float* out;
  uint8_t* empty;
  float2 one2;  // (1, 1)   — FFMA2 operands that make exact adds / products;
  float2 nz2;   // (-0, -0)   passed as parameters so ptxas cannot fuse them
  // FAST (RAW): the raw plan, read directly — no canonicalisation
  const int32_t* cam;
  const int32_t* lvl;
  const float* u;
  const float* v;
  const float* w;
  const int32_t* shape;
  const int64_t* start;
  int32_t n_cams, n_levels, normalize;
  DevStatus* status;
  // dense EXACT with channel groups: wn is [S, n_groups], channel c uses group c / cpg
  int32_t n_groups, cpg;
  // DENSE (FAST on the Sparse4D layout): query q = (batch, anchor) owns the
  // P x cams x L samples of loc [q, P, cams, 2] / w [q, P, cams, L, G]
  const float* loc;
  int32_t P;
  int64_t q_per_batch, rows_per_batch;
  float* wsum_out;  // [q, G] per-group weight sums, or null
  // cameras split across warps: split k takes cameras [k cps, (k + 1) cps);
  // with n_split > 1 the partial sums are red.add-ed into out / wsum_out
  // (zeroed first) and normalised by a separate pass
  int32_t cps, n_split;
  int32_t n_lv;        // DENSE: levels [0, n_lv) of every camera
  int32_t accumulate;  // DENSE: always red.add into the zeroed totals (another kernel adds to them too)
  // DENSE with fused projection: cell coordinates [q, P, cams, L] from the
  // projection pre-pass (f32(pixel / stride_l - 0.5) in f64; NaN = behind the
  // camera: outside every grid, weight 0) instead of loc
  const float2* proj_cell;
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

// DENSE record of sample s of the warp (anchor q, cameras from cam_lo), in
// camera-major, level, point order; wg = the sample's G group weights
template <int GW>
__device__ __forceinline__ SampleRec dense_record(const GatherArgs& a, int64_t q, int cam_lo, int s, float (&wg)[GW]) {
  const int per_cam = a.n_lv * a.P;
  const int cs = s / per_cam, rem = s - cs * per_cam;
  const int cam = cam_lo + cs;
  const int l = rem / a.P, p = rem - l * a.P;
  const int t = cam * a.n_levels + l;
  const int H = a.shape[2 * t], W = a.shape[2 * t + 1];
  const int64_t pc = (q * a.P + p) * a.n_cams + cam;
  float uu, vv;
  bool valid = true;
  if (a.proj_cell) {  // projected keypoint (geometry.py:162-182), cell = pixel / stride - 0.5
    const float2 cl = a.proj_cell[pc * a.n_levels + l];
    valid = !isnan(cl.x);
    uu = valid ? cl.x : -4.0f;
    vv = valid ? cl.y : -4.0f;
  } else {
    const float2 lp = __ldg(reinterpret_cast<const float2*>(a.loc) + pc);
    uu = __fsub_rn(__fmul_rn(lp.x, (float)W), 0.5f);
    vv = __fsub_rn(__fmul_rn(lp.y, (float)H), 0.5f);
  }
  const float* wp = a.w + (pc * a.n_levels + l) * a.n_groups;
  if (GW == 8 && a.n_groups == 8 && (reinterpret_cast<uintptr_t>(wp) & 15) == 0) {
    const float4 w0 = __ldg(reinterpret_cast<const float4*>(wp)), w1 = __ldg(reinterpret_cast<const float4*>(wp) + 1);
    const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int k = 0; k < GW; ++k) wg[k] = valid ? ww[k % 8] : 0.0f;
  } else {
#pragma unroll
    for (int k = 0; k < GW; ++k) wg[k] = (valid && k < a.n_groups) ? __ldg(wp + k) : 0.0f;  // behind the camera: out of the plan
  }
  return make_record(uu, vv, (q / a.q_per_batch) * a.rows_per_batch + a.start[t], H, W);
}

template <int VEC>
__device__ __forceinline__ void half_accumulate(__half2* acch, const void* const* cvp, const float4 iw, const float wn) {
  const __half2 hw0 = __float2half2_rn(iw.x), hw1 = __float2half2_rn(iw.y);
  const __half2 hw2 = __float2half2_rn(iw.z), hw3 = __float2half2_rn(iw.w);
  const __half2 hs = __float2half2_rn(wn);
  const __half2* h0 = reinterpret_cast<const __half2*>(cvp[0]);
  const __half2* h1 = reinterpret_cast<const __half2*>(cvp[1]);
  const __half2* h2 = reinterpret_cast<const __half2*>(cvp[2]);
  const __half2* h3 = reinterpret_cast<const __half2*>(cvp[3]);
#pragma unroll
  for (int e = 0; e < VEC / 2; ++e) {
    const __half2 t = __hadd2_rn(__hadd2_rn(__hmul2_rn(h0[e], hw0), __hmul2_rn(h1[e], hw1)),
                                 __hadd2_rn(__hmul2_rn(h2[e], hw2), __hmul2_rn(h3[e], hw3)));
    acch[e] = __hadd2_rn(acch[e], __hmul2_rn(t, hs));
  }
}

// T: storage type; VEC: channels per thread; HALF: f16 arithmetic.
template <typename T, int VEC, bool HALF, int UNROLL>
__global__ void __launch_bounds__(256) gather_exact_kernel(GatherArgs a) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  if (a.status && *reinterpret_cast<volatile const int32_t*>(&a.status->code) == MSDA_BAD_ARG) return;
  const int lanes_per_q = a.C / VEC;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t q = gtid / lanes_per_q;
  if (q >= a.n_queries) return;
  const int c0 = (int)(gtid - q * lanes_per_q) * VEC;
  const int64_t lo = min(max(a.offsets[q], (int64_t)0), a.n_samples);
  const int64_t hi = min(max(a.offsets[q + 1], lo), a.n_samples);
  const char* feat = reinterpret_cast<const char*>(a.feat) + (size_t)(a.c_off + c0) * sizeof(T);
  const size_t row_bytes = (size_t)a.row_elems * sizeof(T);

  float accf[VEC];
  __half2 acch[VEC / 2];
#pragma unroll
  for (int e = 0; e < VEC; ++e) accf[e] = 0.0f;
#pragma unroll
  for (int e = 0; e < VEC / 2; ++e) acch[e] = __float2half2_rn(0.0f);

  for (int64_t i = lo; i < hi; i += UNROLL) {
    SampleRec r[UNROLL];
    float s[UNROLL];
    RawVec<BYTES> cv[UNROLL][4];
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      if (i + j < hi) {
        r[j] = ld_rec(a.rec + i + j);
        s[j] = __ldg(a.wn + i + j);
        if (a.qsum && a.normalize) s[j] = __fdiv_rn(s[j], a.qsum[q]);
      } else {
        r[j].row[0] = r[j].row[1] = r[j].row[2] = r[j].row[3] = -1;
        r[j].iw[0] = r[j].iw[1] = r[j].iw[2] = r[j].iw[3] = 0.0f;
        s[j] = 0.0f;
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        cv[j][k] = (r[j].row[k] >= 0) ? ldg_vec<BYTES>(feat + (size_t)r[j].row[k] * row_bytes) : zero_vec<BYTES>();
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      if (i + j >= hi) break;
      const float4 iw = make_float4(r[j].iw[0], r[j].iw[1], r[j].iw[2], r[j].iw[3]);
      if constexpr (!HALF) {
        float c[4][VEC];
#pragma unroll
        for (int k = 0; k < 4; ++k) to_f32<T, VEC>(cv[j][k], c[k]);
        exact_accumulate<VEC>(accf, c, iw, s[j], a.one2, a.nz2);
      } else {
        const void* cvp[4] = {&cv[j][0], &cv[j][1], &cv[j][2], &cv[j][3]};
        half_accumulate<VEC>(acch, cvp, iw, s[j]);
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
// rows in flight with cp.async into a per-warp shared-memory ring, and the
// query's records are staged 32 at a time (one coalesced load per lane, read
// back as warp broadcasts), fetched one batch ahead.  Registers stay low, so
// the ring depth — not the register file — sets the bytes in flight per SM.

template <int BYTES, int D, int GW = 1>
struct PipeSmem {
  static constexpr int kSlot = 4 * 32 * BYTES;  // one sample: 4 corners x 32 lanes
  static constexpr int kCorner = D * kSlot;      // corner ring
  static constexpr int kRows = 2 * 32 * 16;      // int4 rows[2][32]
  static constexpr int kIw = 2 * 32 * 16;        // float4 iw[2][32]
  static constexpr int kWn = 2 * 32 * 4 * GW;    // float wn[2][32][GW] (GW weights per sample: channel groups)
  static constexpr int kPerWarp = kCorner + kRows + kIw + kWn;
};

constexpr int kPipeWarps = 1;  // one warp per CTA: finest shared-memory granularity per SM
constexpr int kDenseSplitSamples = 208;  // DENSE: target samples per warp (4 cameras of 4 levels x 13 points)

// FAST: acc += (iw_k * wn) * c_k, fused, any order
template <int VEC>
__device__ __forceinline__ void fast_accumulate(float* acc, const float (*c)[VEC], const float4 iw, const float wn) {
  const float cw[4] = {iw.x * wn, iw.y * wn, iw.z * wn, iw.w * wn};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 w2 = make_float2(cw[k], cw[k]);
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const float2 r = __ffma2_rn(make_float2(c[k][e], c[k][e + 1]), w2, make_float2(acc[e], acc[e + 1]));
      acc[e] = r.x;
      acc[e + 1] = r.y;
    }
  }
}

// RAW = FAST on the CSR plan: records are built from the plan arrays in the
// batch loader and the weight sum is a warp reduction (any order), so no
// canonicalisation pass runs; the gather pipeline is the exact path's.
//
// DENSE = FAST on the Sparse4D layout (deformable_aggregation): records are
// built from the anchor's normalised sampling locations (cell = loc * W - 0.5,
// features.py:20-24) in camera-major, level, point order — every resident
// anchor sweeps the cameras at about the same pace, so the live working set
// is a few cameras' maps — and the lane's channel-group weight is summed on
// the fly for the per-(anchor, group) normalisation at the end.
// HACC (DENSE, f16 storage, FAST_H2): the paper's half2 accumulation — HFMA2
// of the stored f16 pairs with half(iw_k * w_g) into a per-camera half2
// partial, flushed into the f32 accumulator after every camera (runs of
// L x P samples), as the warp-camera kernel does (msda_dense.cu).
template <typename T, int VEC, bool HALF, int D, bool RAW, int GW, bool DENSE = false, bool HACC = false>
__global__ void __launch_bounds__(kPipeWarps * 32) gather_pipe_kernel(GatherArgs a) {
  static_assert(!DENSE || (RAW && GW > 1), "DENSE builds raw records with per-group weights");
  static_assert(!HACC || (DENSE && !HALF && std::is_same<T, __half>::value), "HACC: dense f16");
  constexpr int BYTES = VEC * (int)sizeof(T);
  using SM = PipeSmem<BYTES, D, GW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // launched programmatically after the canonicaliser: its records, weights
  // and sums are visible once the primary grid has completed (a no-op when
  // launched normally)
  if constexpr (!DENSE && !RAW) MSDA_TL(MSDA_TL_WARP, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if constexpr (!DENSE && !RAW) MSDA_TL(MSDA_TL_WARP, 1);
  // malformed CSR offsets (reported by the plan kernel): the workspace
  // records are not all written, read none of them
  if (!RAW && a.status && *reinterpret_cast<volatile const int32_t*>(&a.status->code) == MSDA_BAD_ARG) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + warp * SM::kPerWarp;
  int4* s_rows = reinterpret_cast<int4*>(base + SM::kCorner);
  float4* s_iw = reinterpret_cast<float4*>(base + SM::kCorner + SM::kRows);
  float* s_wn = reinterpret_cast<float*>(base + SM::kCorner + SM::kRows + SM::kIw);
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(base) + lane * BYTES;
  const unsigned char* ring_ptr = base + lane * BYTES;

  const int warps_per_q = a.C / VEC / 32;
  int64_t gw = (int64_t)blockIdx.x * kPipeWarps + warp;
  int cam_lo = 0, n_cam = 0;
  if constexpr (DENSE) {  // split-major: the first waves sweep the first cameras of every anchor
    const int64_t per_split = a.n_queries * warps_per_q;
    const int split = (int)(gw / per_split);
    if (split >= a.n_split) return;
    gw -= split * per_split;
    cam_lo = split * a.cps;
    n_cam = min(a.cps, a.n_cams - cam_lo);
  }
  const int64_t q = gw / warps_per_q;
  if (q >= a.n_queries) return;
  const int c0 = (int)(gw - q * warps_per_q) * 32 * VEC + lane * VEC;
  const int nd = DENSE ? a.P * n_cam * a.n_lv : 0;  // samples of this dense split
  const int64_t lo = DENSE ? 0 : min(max(a.offsets[q], (int64_t)0), a.n_samples);
  const int n = DENSE ? nd : (int)(min(max(a.offsets[q + 1], lo), a.n_samples) - lo);
  const SampleRec* rec = a.rec + lo;
  const float* wnp = a.wn + lo * (GW > 1 ? a.n_groups : 1);
  const int gl = GW > 1 ? (a.c_off + c0) / a.cpg : 0;  // this lane's channel group
  const char* featc = reinterpret_cast<const char*>(a.feat) + (size_t)(a.c_off + c0) * sizeof(T);
  const uint32_t row_bytes = (uint32_t)a.row_elems * (uint32_t)sizeof(T);

  const bool head = c0 == lane * VEC;  // the query's first channel-slice warp reports plan errors
  const float wq = (!RAW && a.qsum && a.normalize && n > 0) ? a.qsum[q] : 1.0f;
  float wsum = 1.0f;
  float wsum_g = 0.0f;  // DENSE: this lane's group weight sum
  if constexpr (RAW && !DENSE) {
    // no plan kernel runs in FAST: the gather reports malformed offsets itself
    if (head && lane == 0 && (a.offsets[q] < 0 || a.offsets[q + 1] < a.offsets[q] || a.offsets[q + 1] > a.n_samples))
      set_status(a.status, MSDA_BAD_ARG, q);
    if (a.normalize) {  // per-query weight sum, any order (FAST)
      float t = 0.0f;
      for (int s = lane; s < n; s += 32) t += __ldg(a.w + lo + s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      wsum = t;
      if (n > 0 && wsum == 0.0f && head && lane == 0) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, q);
    }
  }

  // record batch b: lane j holds sample 32 b + j
  int4 r_rows = make_int4(-1, -1, -1, -1);
  float4 r_iw = make_float4(0.f, 0.f, 0.f, 0.f);
  float r_wn = 0.0f;
  float r_wg[GW];
#pragma unroll
  for (int k = 0; k < GW; ++k) r_wg[k] = 0.0f;
  auto load_batch = [&](int b) {
    const int s = b * 32 + lane;
    if (s < n) {
      SampleRec r;
      if constexpr (DENSE) {
        r = dense_record<GW>(a, q, cam_lo, s, r_wg);
      } else if constexpr (RAW) {
        const int64_t si = lo + s;
        int c = __ldg(a.cam + si), l = __ldg(a.lvl + si);
        const float uu = __ldg(a.u + si), vv = __ldg(a.v + si), ww = __ldg(a.w + si);
        if (c < 0 || c >= a.n_cams || l < 0 || l >= a.n_levels) {
          if (head) set_status(a.status, MSDA_BAD_TARGET, si);
          c = 0;
          l = 0;
        }
        if (!(isfinite(uu) && isfinite(vv) && isfinite(ww)) && head) set_status(a.status, MSDA_NONFINITE, si);
        const int t = c * a.n_levels + l;
        r = make_record(uu, vv, a.start[t], a.shape[2 * t], a.shape[2 * t + 1]);
        r_wn = a.normalize ? ww / wsum : ww;
      } else {
        r = ld_rec(rec + s);
        if constexpr (GW == 1) {
          r_wn = __ldg(wnp + s);  // raw weight: divided when the batch is published (no load-use stall here)
        } else {
#pragma unroll
          for (int k = 0; k < GW; ++k)
            if (k < a.n_groups) r_wg[k] = __ldg(wnp + (int64_t)s * a.n_groups + k);
        }
      }
      r_rows = make_int4(r.row[0], r.row[1], r.row[2], r.row[3]);
      r_iw = make_float4(r.iw[0], r.iw[1], r.iw[2], r.iw[3]);
    }
  };
  auto store_batch = [&](int buf) {
    s_rows[buf * 32 + lane] = r_rows;
    s_iw[buf * 32 + lane] = r_iw;
    if constexpr (GW == 1) {
      // w / sum (features.py:271-273); RAW batches arrive already divided
      s_wn[buf * 32 + lane] = (!RAW && a.qsum && a.normalize) ? __fdiv_rn(r_wn, wq) : r_wn;
    } else {
#pragma unroll
      for (int k = 0; k < GW; ++k) s_wn[(buf * 32 + lane) * GW + k] = r_wg[k];
    }
  };
  auto issue = [&](int k, uint32_t slot_off) {
    const int4 rows = s_rows[((k >> 5) & 1) * 32 + (k & 31)];
    const uint32_t dst = ring + slot_off;
    const int r0 = max(rows.x, 0), r1 = max(rows.y, 0), r2 = max(rows.z, 0), r3 = max(rows.w, 0);
    cp_async_zfill<BYTES>(dst, featc + (size_t)r0 * row_bytes, rows.x >= 0);
    cp_async_zfill<BYTES>(dst + 32 * BYTES, featc + (size_t)r1 * row_bytes, rows.y >= 0);
    cp_async_zfill<BYTES>(dst + 64 * BYTES, featc + (size_t)r2 * row_bytes, rows.z >= 0);
    cp_async_zfill<BYTES>(dst + 96 * BYTES, featc + (size_t)r3 * row_bytes, rows.w >= 0);
  };

  load_batch(0);
  store_batch(0);
  __syncwarp();
  load_batch(1);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < n) issue(k, (uint32_t)(k * SM::kSlot));
    cp_async_commit();
  }
  uint32_t read_off = 0;

  float accf[VEC];
  __half2 acch[VEC / 2];
#pragma unroll
  for (int e = 0; e < VEC; ++e) accf[e] = 0.0f;
#pragma unroll
  for (int e = 0; e < VEC / 2; ++e) acch[e] = __float2half2_rn(0.0f);

  __half2 hacc[HACC ? VEC / 2 : 1];
#pragma unroll
  for (int e = 0; e < (HACC ? VEC / 2 : 1); ++e) hacc[e] = __float2half2_rn(0.0f);
  int run_left = HACC ? a.n_lv * a.P : 0;  // samples left in the current camera
  auto hacc_sample = [&](const RawVec<BYTES>* cv, const float4 iw, const float wn) {
    const float cw[4] = {iw.x * wn, iw.y * wn, iw.z * wn, iw.w * wn};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __half2 cwh = __float2half2_rn(cw[k]);
      const __half2* h = reinterpret_cast<const __half2*>(&cv[k]);
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) hacc[e] = __hfma2(h[e], cwh, hacc[e]);
    }
    if (--run_left == 0) {  // camera done: flush the half2 partial
#pragma unroll
      for (int e = 0; e < VEC / 2; ++e) {
        const float2 f = __half22float2(hacc[e]);
        accf[2 * e] += f.x;
        accf[2 * e + 1] += f.y;
        hacc[e] = __float2half2_rn(0.0f);
      }
      run_left = a.n_lv * a.P;
    }
  };

  // two samples per iteration: their shared-memory reads and products overlap;
  // the accumulation itself stays strictly sequential (i, then i + 1)
  static_assert(D >= 2, "ring depth");
  for (int i = 0; i < n; i += 2) {
    cp_async_wait<D - 2>();  // groups i and i + 1 have landed
    const bool two = i + 1 < n;
    const int b0 = ((i >> 5) & 1) * 32 + (i & 31);
    const int b1 = (((i + 1) >> 5) & 1) * 32 + ((i + 1) & 31);
    const float4 iw0 = s_iw[b0], iw1 = s_iw[b1];
    const float wn0 = s_wn[b0 * GW + gl], wn1 = s_wn[b1 * GW + gl];
    const uint32_t off1 = (read_off + SM::kSlot == (uint32_t)SM::kCorner) ? 0u : read_off + SM::kSlot;
    RawVec<BYTES> cv0[4], cv1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cv0[k] = *reinterpret_cast<const RawVec<BYTES>*>(ring_ptr + read_off + k * 32 * BYTES);
      cv1[k] = *reinterpret_cast<const RawVec<BYTES>*>(ring_ptr + off1 + k * 32 * BYTES);
    }
    if constexpr (HACC) {
      hacc_sample(cv0, iw0, wn0);
      if (two) hacc_sample(cv1, iw1, wn1);
      wsum_g += two ? wn0 + wn1 : wn0;
    } else if constexpr (!HALF) {
      float c0[4][VEC], c1[4][VEC];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        to_f32<T, VEC>(cv0[k], c0[k]);
        to_f32<T, VEC>(cv1[k], c1[k]);
      }
      if constexpr (RAW) {
        fast_accumulate<VEC>(accf, c0, iw0, wn0);
        if (two) fast_accumulate<VEC>(accf, c1, iw1, wn1);
        if constexpr (DENSE) wsum_g += two ? wn0 + wn1 : wn0;
      } else {
        exact_accumulate2<VEC>(accf, c0, iw0, wn0, c1, iw1, wn1, two, a.one2, a.nz2);
      }
    } else {
      const void* p0[4] = {&cv0[0], &cv0[1], &cv0[2], &cv0[3]};
      const void* p1[4] = {&cv1[0], &cv1[1], &cv1[2], &cv1[3]};
      half_accumulate<VEC>(acch, p0, iw0, wn0);
      if (two) half_accumulate<VEC>(acch, p1, iw1, wn1);
    }
    // refill the two consumed slots with samples i + D and i + D + 1
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = i + D + j;
      if (k < n) {
        if ((k & 31) == 0) {  // entering record batch k/32: publish it, prefetch the next
          __syncwarp();
          store_batch((k >> 5) & 1);
          __syncwarp();
          load_batch((k >> 5) + 1);
        }
        issue(k, read_off);
      }
      cp_async_commit();
      read_off += SM::kSlot;
      if (read_off == (uint32_t)SM::kCorner) read_off = 0;
    }
  }
  cp_async_wait<0>();

  float* o = a.out + q * a.out_stride + a.c_off + c0;
  if constexpr (DENSE) {  // per-(anchor, group) renormalisation (FAST: sum in any order)
    const bool ghead = (a.c_off + c0) % a.cpg == 0;  // the group's first lane reports
    if (a.n_split > 1 || a.accumulate) {  // partial over a camera range: add into the zeroed totals
      if (ghead && a.wsum_out) atomicAdd(a.wsum_out + q * a.n_groups + gl, wsum_g);
      static_assert(VEC % 4 == 0, "float4 partials");
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        atomicAdd(reinterpret_cast<float4*>(o + e), make_float4(accf[e], accf[e + 1], accf[e + 2], accf[e + 3]));
      return;
    }
    if (ghead) {
      if (a.wsum_out) a.wsum_out[q * a.n_groups + gl] = wsum_g;
      if (a.normalize && wsum_g == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, q);
    }
    if (a.normalize) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) accf[e] = accf[e] / wsum_g;
    }
  }
  if constexpr (!HALF) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        *reinterpret_cast<float4*>(o + e) = make_float4(accf[e], accf[e + 1], accf[e + 2], accf[e + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) o[e] = accf[e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) {
      const float2 f = __half22float2(acch[e]);
      o[2 * e] = f.x;
      o[2 * e + 1] = f.y;
    }
  }
  if (c0 == 0 && a.empty) a.empty[q] = (n == 0) ? 1 : 0;
  if constexpr (!DENSE && !RAW) {
    MSDA_TL(MSDA_TL_WARP, 2);
    MSDA_TL_SMID(MSDA_TL_WARP);
  }
}

template <typename T, int VEC, bool HALF, int D, bool RAW, int GW = 1, bool DENSE = false, bool HACC = false>
cudaError_t launch_gather_pipe(const GatherArgs& g, cudaStream_t stream) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int smem = kPipeWarps * PipeSmem<BYTES, D, GW>::kPerWarp;
  static std::atomic<bool> attr_set[64];  // per instantiation and device (function attributes are per device)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(gather_pipe_kernel<T, VEC, HALF, D, RAW, GW, DENSE, HACC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev].store(true, std::memory_order_release);
  }
  const int64_t warps = g.n_queries * (g.C / VEC / 32) * (DENSE ? g.n_split : 1);
  const int64_t grid = (warps + kPipeWarps - 1) / kPipeWarps;
  if (grid == 0) return cudaSuccess;
  // programmatic stream serialisation: the launch overlaps the tail of the
  // preceding canonicaliser (which triggers early); correctness rests on the
  // kernel's griddepcontrol.wait
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kPipeWarps * 32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gather_pipe_kernel<T, VEC, HALF, D, RAW, GW, DENSE, HACC>, g);
}

// resident one-warp CTAs of gather_pipe_kernel<..., D, ..., GW> on the device
template <typename T, int VEC, bool HALF, int D, int GW>
int64_t pipe_slots() {
  static std::atomic<int64_t> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) {
    const int64_t c = cached[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  constexpr int BYTES = VEC * (int)sizeof(T);
  const int smem = kPipeWarps * PipeSmem<BYTES, D, GW>::kPerWarp;
  int per_sm = 0, sms = 148;
  cudaFuncSetAttribute(gather_pipe_kernel<T, VEC, HALF, D, false, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_pipe_kernel<T, VEC, HALF, D, false, GW>,
                                                    kPipeWarps * 32, smem) != cudaSuccess)
    per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = (int64_t)per_sm * sms * kPipeWarps;
  if (dev >= 0 && dev < 64 && slots > 0) cached[dev].store(slots, std::memory_order_relaxed);
  return slots;
}

// EXACT (16-B lanes): a query's canonical accumulation is one sequential
// chain per warp, so a grid that spills a few warps into a second wave costs
// a whole extra chain (cfg1 dense EXACT: 1800 warps vs 12 x 148 resident at
// ring depth 7 -> 160.6 us; depth 6, 13 per SM -> 126 us).  Use the deepest
// ring whose residency still holds every warp at once.
template <typename T, int VEC, bool HALF, int GW>
cudaError_t launch_exact_pipe(const GatherArgs& g, cudaStream_t stream) {
  const int64_t warps = g.n_queries * (g.C / VEC / 32);
  if (warps > pipe_slots<T, VEC, HALF, 7, GW>()) {
    if (warps <= pipe_slots<T, VEC, HALF, 6, GW>()) return launch_gather_pipe<T, VEC, HALF, 6, false, GW>(g, stream);
    if (warps <= pipe_slots<T, VEC, HALF, 5, GW>()) return launch_gather_pipe<T, VEC, HALF, 5, false, GW>(g, stream);
  }
  return launch_gather_pipe<T, VEC, HALF, 7, false, GW>(g, stream);
}

template <typename T, int VEC, bool HALF>
cudaError_t launch_gather(const GatherArgs& g, cudaStream_t stream, bool raw) {
  if (g.n_groups > 1) {  // per-group weights (dense EXACT, one pass): pipelined kernel only
    if ((g.C / VEC) % 32 != 0 || g.C % VEC != 0 || g.n_groups > 8) return cudaErrorNotSupported;
    if constexpr (VEC * sizeof(T) == 16) return launch_exact_pipe<T, VEC, HALF, 8>(g, stream);
    else return launch_gather_pipe<T, VEC, HALF, 12, false, 8>(g, stream);
  }
  if ((g.C / VEC) % 32 == 0 && g.C % VEC == 0) {
    if constexpr (!HALF) {
      if (raw) {
        if constexpr (VEC * sizeof(T) == 16) return launch_gather_pipe<T, VEC, HALF, 7, true>(g, stream);
        else return launch_gather_pipe<T, VEC, HALF, 12, true>(g, stream);
      }
    }
    if constexpr (VEC * sizeof(T) == 16) return launch_exact_pipe<T, VEC, HALF, 1>(g, stream);
    else return launch_gather_pipe<T, VEC, HALF, 12, false>(g, stream);
  }
  if (raw) return cudaErrorNotSupported;
  const int lanes = g.C / VEC;
  const int64_t threads = g.n_queries * lanes;
  const int block = 256;
  const int64_t grid = (threads + block - 1) / block;
  if (grid == 0) return cudaSuccess;
  gather_exact_kernel<T, VEC, HALF, 4><<<(unsigned)grid, block, 0, stream>>>(g);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather_dense_fast(const msda_features_t& f, const DenseFastSpec& d, DevStatus* status, float* out,
                                     cudaStream_t stream, bool* normalize_pending) {
  *normalize_pending = false;
  const int C = f.channels, G = d.G;
  const size_t esz = f.dtype == MSDA_F32 ? 4 : 2;
  if (G < 1 || G > 8 || C % G) return cudaErrorNotSupported;
  const int cpg = C / G;
  GatherArgs g{};
  g.feat = f.data;
  g.C = C;
  g.row_elems = C;
  g.c_off = 0;
  g.out_stride = C;
  g.n_queries = (int64_t)f.batch * d.Q;
  g.out = out;
  g.w = d.w;
  g.loc = d.loc;
  g.proj_cell = d.proj_cell;
  g.P = d.P;
  g.q_per_batch = d.Q > 0 ? d.Q : 1;
  g.rows_per_batch = f.n_rows;
  g.wsum_out = d.wsum_out;
  g.shape = f.spatial_shape;
  g.start = f.scale_start_index;
  g.n_cams = f.n_cams;
  g.n_levels = f.n_levels;
  g.normalize = d.normalize;
  g.status = status;
  g.n_groups = G;
  g.cpg = cpg;
  if (reinterpret_cast<uintptr_t>(f.data) % 16 || (C * esz) % 16 || reinterpret_cast<uintptr_t>(out) % 16 ||
      (!d.proj_cell && reinterpret_cast<uintptr_t>(d.loc) % 8))
    return cudaErrorNotSupported;
  // a lane's channels must share one group, a query's channels span whole warps
  const int vec = f.dtype == MSDA_F32 ? 4 : 8;  // 16-B lanes
  if (C % (32 * vec) || cpg % vec) return cudaErrorNotSupported;
  // cameras per warp: about kDenseSplitSamples samples per warp, so that
  // short per-warp chains and many resident warps keep the gather fed
  g.n_lv = d.n_lv > 0 ? std::min(d.n_lv, f.n_levels) : f.n_levels;
  g.accumulate = d.accumulate ? 1 : 0;
  const int per_cam = d.P * g.n_lv;
  // fine levels beside the staged kernel: chains of 104 samples, halved
  // (down to 26) while the grid has fewer than ~20 k warps — small calls are
  // latency-bound and want more, shorter chains; large batches pay for the
  // extra partial red.adds.  Measured 26 / 52 / 104 / 156: cfg3 FAST_H2
  // 371 / 365 / 369 / — us, cfg4 FAST 221 / 222 / 229 us, cfg1 f16 FAST_H2
  // 51 / 53 / 57 / 60 us; cfg5-stream (16 scenes x 32 cameras) 3.68 ms at 52
  // vs 3.58 ms at 104
  int split_samples = d.accumulate ? kDenseSplitSamples / 2 : kDenseSplitSamples;
  if (d.accumulate)
    while (split_samples > kDenseSplitSamples / 8 &&
           g.n_queries * ((f.n_cams * per_cam + split_samples - 1) / split_samples) < 20000)
      split_samples /= 2;
  const int want = std::max(1, (f.n_cams * per_cam + split_samples - 1) / split_samples);
  g.cps = (f.n_cams + want - 1) / want;
  g.n_split = (f.n_cams + g.cps - 1) / g.cps;
  if (g.n_split > 1 || d.accumulate) {
    if (!d.wsum_out && d.normalize && !d.wsum_scratch) return cudaErrorNotSupported;
    if (!d.wsum_out && d.normalize) g.wsum_out = d.wsum_scratch;
    if (!d.accumulate && !d.prezeroed) {
      if (cudaMemsetAsync(out, 0, (size_t)g.n_queries * C * 4, stream) != cudaSuccess) return cudaErrorUnknown;
      if (g.wsum_out && cudaMemsetAsync(g.wsum_out, 0, (size_t)g.n_queries * G * 4, stream) != cudaSuccess)
        return cudaErrorUnknown;
    }
    *normalize_pending = d.normalize != 0;
  }
  // ring depth 2: the dense gather is issue-bound (bf16/f16 -> f32 per
  // channel-corner), so more resident warps (28 per SM at 8 KB of shared
  // memory each) beat a deeper per-warp ring (D = 7: 12 per SM); measured at
  // cfg1-cfg4, D in {2, 3, 4, 5, 7} x split in {104, 156, 208, 416} samples
  if (d.accumulate) {
    // fine levels only (the coarse ones come from the staged kernel): every
    // corner row is an L2 miss or a far L2 hit, so a deeper ring than the
    // all-level gather's and shorter chains (26-104 samples per warp, above)
    // win — cfg3 FAST_H2 fine part 227 vs 300 us (D = 2, 208 then).  With the
    // adaptive chains, D = 2 / 3 / 4 / 5 / 6: cfg3 FAST_H2 371 / 363 / 365 /
    // 369 / 387 us, cfg3 FAST 456 / 463 / 467 / 475 / 498 us, cfg4 FAST 217 /
    // 217 / 219 / 221 / 234 us
    switch (f.dtype) {
      case MSDA_F16:
        if (d.h2) return launch_gather_pipe<__half, 8, false, 3, true, 8, true, true>(g, stream);
        return launch_gather_pipe<__half, 8, false, 3, true, 8, true>(g, stream);
      case MSDA_BF16: return launch_gather_pipe<__nv_bfloat16, 8, false, 3, true, 8, true>(g, stream);
      case MSDA_F32: return launch_gather_pipe<float, 4, false, 3, true, 8, true>(g, stream);
      default: return cudaErrorNotSupported;
    }
  }
  switch (f.dtype) {
    case MSDA_F32: return launch_gather_pipe<float, 4, false, 2, true, 8, true>(g, stream);
    case MSDA_F16:
      if (d.h2) return launch_gather_pipe<__half, 8, false, 2, true, 8, true, true>(g, stream);
      return launch_gather_pipe<__half, 8, false, 2, true, 8, true>(g, stream);
    default: return launch_gather_pipe<__nv_bfloat16, 8, false, 2, true, 8, true>(g, stream);
  }
}

cudaError_t reset_exact_workspace(const ExactWorkspace& w, cudaStream_t stream) {
  return cudaMemsetAsync(w.status, 0, sizeof(DevStatus), stream);
}

size_t exact_workspace_bytes(int64_t n_queries, int64_t n_samples) {
  size_t b = kStatusBytes;
  b += align_up((size_t)n_samples * sizeof(SampleRec), 256);
  b += align_up((size_t)n_samples * sizeof(float), 256);
  b += 2 * align_up((size_t)n_samples * sizeof(u64), 256);
  b += align_up((size_t)n_samples * sizeof(int32_t), 256);
  b += align_up((size_t)n_queries * sizeof(float), 256);  // per-query weight sums
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
  w.g_hi = reinterpret_cast<u64*>(p);
  p += align_up((size_t)n_samples * sizeof(u64), 256);
  w.g_lo = reinterpret_cast<u64*>(p);
  p += align_up((size_t)n_samples * sizeof(u64), 256);
  w.g_idx = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)n_samples * sizeof(int32_t), 256);
  w.qsum = reinterpret_cast<float*>(p);
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
  a.n_samples = p.n_samples;
  a.n_cams = f.n_cams;
  a.n_levels = f.n_levels;
  a.shape = f.spatial_shape;
  a.start = f.scale_start_index;
  a.normalize = normalize;
  a.queries_per_batch = queries_per_batch > 0 ? queries_per_batch : (p.n_queries > 0 ? p.n_queries : 1);
  a.rows_per_batch = f.n_rows;
  a.rec = w.rec;
  a.wn = w.wn;
  a.g_hi = w.g_hi;
  a.g_lo = w.g_lo;
  a.g_idx = w.g_idx;
  a.qsum = w.qsum;
  a.status = w.status;
  // one CTA per query while they all fit on the device at once
  const int64_t grid = std::min<int64_t>(p.n_queries, (int64_t)num_sms * 8);
  plan_canon_kernel<<<(unsigned)grid, kPlanThreads, plan_smem_bytes(f.n_cams * f.n_levels), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather_exact(const msda_features_t& f, const msda_csr_plan_t& p, int precision,
                                const ExactWorkspace& w, float* out, uint8_t* empty, cudaStream_t stream,
                                int c_off, int c_count, int fast_normalize, int n_groups, int normalize) {
  const bool raw = fast_normalize >= 0;  // FAST on the raw plan (no canonicalisation pass)
  GatherArgs g{};
  g.n_groups = n_groups;
  g.cpg = f.channels / std::max(1, n_groups);
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
  g.n_samples = p.n_samples;
  g.offsets = p.offsets;
  g.rec = w.rec;
  g.wn = w.wn;
  g.qsum = n_groups > 1 ? nullptr : w.qsum;
  g.out = out;
  g.empty = empty;
  g.one2 = make_float2(1.0f, 1.0f);
  g.nz2 = make_float2(-0.0f, -0.0f);
  g.cam = p.camera_index;
  g.lvl = p.level;
  g.u = p.u;
  g.v = p.v;
  g.w = p.weight;
  g.shape = f.spatial_shape;
  g.start = f.scale_start_index;
  g.n_cams = f.n_cams;
  g.n_levels = f.n_levels;
  g.normalize = raw ? fast_normalize : normalize;
  g.status = w.status;
  const size_t esz = f.dtype == MSDA_F32 ? 4 : 2;
  // vector width must divide the slice and keep every row (and output) access aligned
  const uintptr_t base = reinterpret_cast<uintptr_t>(f.data) | ((size_t)c_off * esz) | ((size_t)f.channels * esz);
  const uintptr_t obase = reinterpret_cast<uintptr_t>(out) | ((size_t)c_off * 4) | ((size_t)f.channels * 4);
  const int C = c_count;
  if (precision == MSDA_EXACT_HALF) {
    if (C % 128 == 0 && base % 8 == 0) return launch_gather<__half, 4, true>(g, stream, raw);
    if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, true>(g, stream, raw);
    if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, true>(g, stream, raw);
    return launch_gather<__half, 2, true>(g, stream, raw);
  }
  switch (f.dtype) {
    case MSDA_F32:
      // two warps per 256 channels (16-B lanes; 8-B lanes measured slower)
      if (C % 4 == 0 && base % 16 == 0 && obase % 16 == 0) return launch_gather<float, 4, false>(g, stream, raw);
      return launch_gather<float, 2, false>(g, stream, raw);
    case MSDA_F16:
      if (C % 128 == 0 && base % 8 == 0) return launch_gather<__half, 4, false>(g, stream, raw);
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__half, 8, false>(g, stream, raw);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__half, 4, false>(g, stream, raw);
      return launch_gather<__half, 2, false>(g, stream, raw);
    default:
      if (C % 128 == 0 && base % 8 == 0) return launch_gather<__nv_bfloat16, 4, false>(g, stream, raw);
      if (C % 8 == 0 && base % 16 == 0) return launch_gather<__nv_bfloat16, 8, false>(g, stream, raw);
      if (C % 4 == 0 && base % 8 == 0) return launch_gather<__nv_bfloat16, 4, false>(g, stream, raw);
      return launch_gather<__nv_bfloat16, 2, false>(g, stream, raw);
  }
}

}  // namespace msda
