// C ABI of msda_b200 (include/msda_b200.h): argument validation, workspace
// carving, status mapping and the host-buffer context.  No torch types cross
// this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <vector>

#include "msda_common.cuh"
#include "msda_exact.cuh"

using namespace msda;

namespace {

__global__ void f32_to_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}

// ---- touched-row fetch for the host-buffer path ----
// Large, sparsely sampled grids (the finest levels: at cfg2 a level-0 cell is
// read 0.36 times per call) are not copied whole: when the caller's host
// buffer is pinned (device-visible through UVA), one warp per plan sample
// claims each in-grid corner row in a bitmap and copies only the rows no one
// claimed before, straight from host memory over PCIe into the device table.
// Same bilinear corner rule as the plan (make_record), so every row the
// gather reads is present; the other rows are never read.
struct FetchArgs {
  const int32_t* cam;
  const int32_t* lvl;
  const float* u;
  const float* v;
  int64_t n_samples;
  int32_t n_cams, n_levels;
  const int32_t* shape;
  const int64_t* start;
  const unsigned long long* src;  // [n_tiles] device-visible host address of each fetched tile, 0 = copied whole
  char* table;                    // device table
  uint32_t* claimed;              // [rows / 32 + 1] bitmap, zeroed
  unsigned long long* fetched;    // rows fetched (bytes = rows * row_bytes)
  int32_t row_bytes;
};

__global__ void __launch_bounds__(256) fetch_rows_kernel(FetchArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t sidx = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sidx < a.n_samples;
       sidx += warps) {
    const int c = a.cam[sidx], l = a.lvl[sidx];
    if (c < 0 || c >= a.n_cams || l < 0 || l >= a.n_levels) continue;  // the plan kernel reports it
    const int t = c * a.n_levels + l;
    const unsigned long long src = a.src[t];
    if (!src) continue;
    const float uu = a.u[sidx], vv = a.v[sidx];
    if (!(isfinite(uu) && isfinite(vv))) continue;
    const SampleRec r = make_record(uu, vv, 0, a.shape[2 * t], a.shape[2 * t + 1]);  // tile-local rows
    unsigned todo = 0;
    if (lane < 4 && r.row[lane] >= 0) {
      const int64_t g = a.start[t] + r.row[lane];
      const uint32_t bit = 1u << (g & 31);
      todo = (atomicOr(a.claimed + (g >> 5), bit) & bit) ? 0u : 1u;
    }
    unsigned mask = __ballot_sync(0xffffffffu, todo) & 0xfu;
    while (mask) {
      const int k = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t row = r.row[k];
      const char* from = reinterpret_cast<const char*>(src) + (size_t)row * a.row_bytes;
      char* to = a.table + (size_t)(a.start[t] + row) * a.row_bytes;
      for (int off = lane * 16; off < a.row_bytes; off += 32 * 16)
        *reinterpret_cast<uint4*>(to + off) = *reinterpret_cast<const uint4*>(from + off);
      if (lane == 0) atomicAdd(a.fetched, 1ull);
    }
  }
}

// bilinear_sample (features.py:184-219) for n (u, v) cell coordinates on one
// (H, W, C) grid: one warp per sample, the reference's f32 tree
// ((c00*w00 + c10*w10) + (c01*w01 + c11*w11)), each product and sum rounded
// once, out-of-grid corners read as +0 rows.  `grid` is device memory or a
// device-visible pinned host buffer.
__global__ void bilinear_kernel(const float* __restrict__ grid, int H, int W, int C, const float* __restrict__ u,
                                const float* __restrict__ v, int64_t n, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const SampleRec r = make_record(u[i], v[i], 0, H, W);
    for (int c = lane; c < C; c += 32) {
      float cv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) cv[k] = r.row[k] >= 0 ? grid[(size_t)r.row[k] * C + c] : 0.0f;
      const float a = __fadd_rn(__fmul_rn(cv[0], r.iw[0]), __fmul_rn(cv[1], r.iw[1]));
      const float b = __fadd_rn(__fmul_rn(cv[2], r.iw[2]), __fmul_rn(cv[3], r.iw[3]));
      out[i * C + c] = __fadd_rn(a, b);
    }
  }
}

cudaError_t launch_f32_to_f16(const float* src, __half* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
  f32_to_f16_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

int g_num_sms_cache[64] = {0};

int num_sms_for_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev >= 0 && dev < 64 && g_num_sms_cache[dev] > 0) return g_num_sms_cache[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) g_num_sms_cache[dev] = n;
  return n;
}

int32_t validate_features(const msda_features_t* f) {
  if (!f || !f->data || !f->spatial_shape || !f->scale_start_index) return MSDA_BAD_ARG;
  if (f->n_cams <= 0 || f->n_levels <= 0 || f->channels <= 0 || f->batch <= 0) return MSDA_BAD_ARG;
  if (f->dtype < MSDA_F32 || f->dtype > MSDA_BF16) return MSDA_BAD_ARG;
  if (f->n_rows <= 0 || f->n_rows >= (int64_t(1) << 31)) return MSDA_BAD_ARG;
  if (f->channels % 2 != 0) return MSDA_ODD_CHANNELS;
  return MSDA_OK;
}

}  // namespace

extern "C" {

int32_t msda_abi_version(void) { return 2; }

const char* msda_status_string(int32_t s) {
  switch (s) {
    case MSDA_OK: return "ok";
    case MSDA_ODD_CHANNELS: return "channel count is odd; packed pairs need an even count";
    case MSDA_NONFINITE: return "plan weights and coordinates must be finite";
    case MSDA_BAD_TARGET: return "plan references an unknown camera id or a missing level";
    case MSDA_ZERO_WEIGHT_SUM: return "plan weights sum to zero, cannot renormalize";
    case MSDA_BAD_PRECISION: return "unknown precision mode";
    case MSDA_CHANNEL_MISMATCH: return "pyramid channel count does not match the descriptor length";
    case MSDA_CUDA_ERROR: return "CUDA runtime error";
    case MSDA_BAD_ARG: return "invalid argument";
    case MSDA_OFFSET_RANGE: return "learned keypoint offset component outside [-1, 1]";
    default: return "unknown status";
  }
}

size_t msda_csr_workspace_size(int64_t n_queries, int64_t n_samples, int32_t channels) {
  (void)channels;
  return exact_workspace_bytes(n_queries, n_samples);
}

int32_t msda_csr(const msda_features_t* feat, const msda_csr_plan_t* plan, int32_t precision, int32_t normalize,
                 float* out, uint8_t* empty, void* workspace, size_t workspace_bytes, void* stream_) {
  return msda_csr_stages(feat, plan, precision, normalize, out, empty, workspace, workspace_bytes, stream_, 3);
}

int32_t msda_csr_stages(const msda_features_t* feat, const msda_csr_plan_t* plan, int32_t precision,
                        int32_t normalize, float* out, uint8_t* empty, void* workspace, size_t workspace_bytes,
                        void* stream_, int32_t stage_mask) {
  int32_t st = validate_features(feat);
  if (st != MSDA_OK) return st;
  if (!plan || plan->n_queries < 0 || plan->n_samples < 0) return MSDA_BAD_ARG;
  if (precision < MSDA_EXACT || precision > MSDA_FAST_H2) return MSDA_BAD_PRECISION;
  if (precision == MSDA_EXACT_HALF && feat->dtype != MSDA_F16) return MSDA_BAD_ARG;
  if (!workspace || workspace_bytes < msda_csr_workspace_size(plan->n_queries, plan->n_samples, feat->channels))
    return MSDA_BAD_ARG;
  if (plan->n_queries > 0 && (!plan->offsets || !out)) return MSDA_BAD_ARG;
  if (plan->n_samples > 0 &&
      (!plan->camera_index || !plan->level || !plan->u || !plan->v || !plan->weight))
    return MSDA_BAD_ARG;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  ExactWorkspace w = carve_exact_workspace(workspace, plan->n_samples);
  if ((stage_mask & 1) && reset_exact_workspace(w, stream) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (plan->n_queries == 0) return MSDA_OK;
  // FAST: any summation order, so no canonicalisation — one gather launch
  // from the raw plan (stage 2; stage 1 only resets the status word)
  if (precision >= MSDA_FAST && feat->batch == 1) {
    if (!(stage_mask & 2)) return MSDA_OK;
    const cudaError_t e = launch_csr_fast(*feat, *plan, normalize, w, out, empty, stream);
    if (e == cudaSuccess) return MSDA_OK;
    if (e != cudaErrorNotSupported) return MSDA_CUDA_ERROR;
  }
  const int prec = precision >= MSDA_FAST ? MSDA_EXACT : precision;
  if ((stage_mask & 1) &&
      launch_plan_canon(*feat, *plan, normalize, w, num_sms_for_current_device(), stream) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  if ((stage_mask & 2) &&
      launch_gather_exact(*feat, *plan, prec, w, out, empty, stream, 0, 0, -1, 1, normalize) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  return MSDA_OK;
}

int32_t msda_read_status(const void* workspace, void* stream_, int32_t* status, int64_t* detail) {
  if (!workspace) return MSDA_BAD_ARG;
  DevStatus h{};
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, stream) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (status) *status = h.code;
  if (detail) *detail = status_detail(h);
  return MSDA_OK;
}

// ---------------------------------------------------------------------------
// host-buffer context (end-to-end entry point)

struct msda_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // whole-grid copies, concurrent with the row fetch on `stream`
  cudaEvent_t fork = nullptr, join = nullptr;
  void* arena = nullptr;
  size_t arena_bytes = 0;
  long long last_h2d_bytes = 0;  // host->device bytes moved by the last msda_csr_host call
  long long last_detail = -1;    // offending query / sample of the last call's status, or -1
};

long long msda_context_last_detail(const msda_context_t* ctx) { return ctx ? ctx->last_detail : -1; }

long long msda_context_last_h2d_bytes(const msda_context_t* ctx) { return ctx ? ctx->last_h2d_bytes : -1; }

// Page-lock an existing host range (e.g. a memory-mapped FPYR file) so that
// copies from it are single DMA transfers; read_only for PROT_READ mappings.
int32_t msda_host_register(void* ptr, size_t bytes, int32_t read_only) {
  if (!ptr || bytes == 0) return MSDA_BAD_ARG;
  unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
  if (cudaHostRegister(ptr, bytes, flags) != cudaSuccess) {
    cudaGetLastError();  // not sticky: the caller stages through a pinned buffer instead
    return MSDA_CUDA_ERROR;
  }
  return MSDA_OK;
}

int32_t msda_host_unregister(void* ptr) {
  if (!ptr) return MSDA_BAD_ARG;
  if (cudaHostUnregister(ptr) != cudaSuccess) {
    cudaGetLastError();
    return MSDA_CUDA_ERROR;
  }
  return MSDA_OK;
}

int32_t msda_context_create(int32_t device, msda_context_t** ctx) {
  if (!ctx) return MSDA_BAD_ARG;
  auto* c = new (std::nothrow) msda_context();
  if (!c) return MSDA_BAD_ARG;
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming) != cudaSuccess) {
    msda_context_destroy(c);
    return MSDA_CUDA_ERROR;
  }
  *ctx = c;
  return MSDA_OK;
}

void msda_context_destroy(msda_context_t* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  delete ctx;
}

static int32_t ctx_reserve(msda_context_t* ctx, size_t bytes) {
  if (bytes <= ctx->arena_bytes) return MSDA_OK;
  if (ctx->arena) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->copy_stream);
    cudaFree(ctx->arena);
    ctx->arena = nullptr;
    ctx->arena_bytes = 0;
  }
  size_t want = std::max(bytes, ctx->arena_bytes + ctx->arena_bytes / 2);
  if (cudaMalloc(&ctx->arena, want) != cudaSuccess) return MSDA_CUDA_ERROR;
  ctx->arena_bytes = want;
  return MSDA_OK;
}

int32_t msda_csr_host(msda_context_t* ctx, const void* const* level_data, const int32_t* spatial_shape,
                      int32_t n_cams, int32_t n_levels, int32_t channels, int32_t dtype, int64_t n_queries,
                      const int64_t* offsets, const int32_t* camera_index, const int32_t* level, const float* u,
                      const float* v, const float* weight, int32_t precision, int32_t normalize, float* out,
                      uint8_t* empty) {
  if (!ctx || !level_data || !spatial_shape || !offsets || n_cams <= 0 || n_levels <= 0 || channels <= 0 ||
      n_queries < 0)
    return MSDA_BAD_ARG;
  if (channels % 2) return MSDA_ODD_CHANNELS;
  if (dtype < MSDA_F32 || dtype > MSDA_BF16) return MSDA_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MSDA_CUDA_ERROR;
  ctx->last_detail = -1;
  // CSR offsets (HOST): offsets[0] == 0 and non-decreasing, else the plan
  // arrays' extent (offsets[n_queries] samples) is not what the caller holds
  if (offsets[0] != 0) return MSDA_BAD_ARG;
  for (int64_t q = 0; q < n_queries; ++q)
    if (offsets[q + 1] < offsets[q]) {
      ctx->last_detail = q;
      return MSDA_BAD_ARG;
    }
  const size_t esz = dtype == MSDA_F32 ? 4 : 2;
  const int n_tiles = n_cams * n_levels;
  std::vector<int64_t> start(n_tiles);
  int64_t rows = 0;
  for (int t = 0; t < n_tiles; ++t) {
    if (spatial_shape[2 * t] < 0 || spatial_shape[2 * t + 1] < 0) return MSDA_BAD_ARG;
    if ((int64_t)spatial_shape[2 * t] * spatial_shape[2 * t + 1] > 0 && !level_data[t]) return MSDA_BAD_ARG;
    start[t] = rows;
    rows += (int64_t)spatial_shape[2 * t] * spatial_shape[2 * t + 1];
  }
  const int64_t S = offsets[n_queries];
  // PACKED_HALF stores features as f16 (features.py:398): f32 host grids are
  // copied in and rounded to f16 on the device.
  const bool cvt_half = (precision == MSDA_EXACT_HALF && dtype == MSDA_F32);
  const int32_t dev_dtype = cvt_half ? MSDA_F16 : dtype;
  const size_t half_b = cvt_half ? align_up((size_t)rows * channels * 2, 256) : 0;
  // tiles fetched row by row instead of copied whole: pinned (device-visible)
  // host buffers of grids with more cells than 2 x the mean samples per tile
  // (4 corner reads per sample touch < ~85 % of such a grid; measured at cfg2:
  // fetching levels 0-1 beats copying them)
  std::vector<unsigned long long> src(n_tiles, 0ull);
  const int64_t per_tile = n_tiles > 0 ? S / n_tiles : 0;
  const bool fetch_ok = !cvt_half && (channels * esz) % 16 == 0;
  for (int t = 0; t < n_tiles && fetch_ok; ++t) {
    const int64_t cells = (int64_t)spatial_shape[2 * t] * spatial_shape[2 * t + 1];
    if (cells <= 2 * per_tile || !level_data[t]) continue;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, level_data[t]) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (pa.type == cudaMemoryTypeHost && pa.devicePointer && reinterpret_cast<uintptr_t>(pa.devicePointer) % 16 == 0)
      src[t] = reinterpret_cast<unsigned long long>(pa.devicePointer);
  }
  bool any_fetch = false;
  for (int t = 0; t < n_tiles; ++t) any_fetch |= src[t] != 0;
  // arena: [workspace | table | shape | start | offsets | cam | lvl | u | v | w | out | empty | src | bitmap | count]
  const size_t src_b = align_up((size_t)n_tiles * 8, 256), bm_b = align_up((size_t)(rows / 32 + 1) * 4, 256);
  const size_t ws_b = align_up(msda_csr_workspace_size(n_queries, S, channels), 256);
  const size_t tab_b = align_up((size_t)rows * channels * esz, 256);
  const size_t shp_b = align_up((size_t)n_tiles * 2 * 4, 256), st_b = align_up((size_t)n_tiles * 8, 256);
  const size_t off_b = align_up((size_t)(n_queries + 1) * 8, 256), i_b = align_up((size_t)S * 4, 256);
  const size_t out_b = align_up((size_t)n_queries * channels * 4, 256), emp_b = align_up((size_t)n_queries, 256);
  const size_t total = ws_b + tab_b + half_b + shp_b + st_b + off_b + 5 * i_b + out_b + emp_b + src_b + bm_b + 256;
  int32_t st = ctx_reserve(ctx, total);
  if (st != MSDA_OK) return st;
  char* p = reinterpret_cast<char*>(ctx->arena);
  void* d_ws = p; p += ws_b;
  char* d_tab = p; p += tab_b;
  char* d_half = p; p += half_b;
  int32_t* d_shape = reinterpret_cast<int32_t*>(p); p += shp_b;
  int64_t* d_start = reinterpret_cast<int64_t*>(p); p += st_b;
  int64_t* d_off = reinterpret_cast<int64_t*>(p); p += off_b;
  int32_t* d_cam = reinterpret_cast<int32_t*>(p); p += i_b;
  int32_t* d_lvl = reinterpret_cast<int32_t*>(p); p += i_b;
  float* d_u = reinterpret_cast<float*>(p); p += i_b;
  float* d_v = reinterpret_cast<float*>(p); p += i_b;
  float* d_w = reinterpret_cast<float*>(p); p += i_b;
  float* d_out = reinterpret_cast<float*>(p); p += out_b;
  uint8_t* d_emp = reinterpret_cast<uint8_t*>(p); p += emp_b;
  unsigned long long* d_src = reinterpret_cast<unsigned long long*>(p); p += src_b;
  uint32_t* d_bm = reinterpret_cast<uint32_t*>(p); p += bm_b;
  unsigned long long* d_fetched = reinterpret_cast<unsigned long long*>(p);
  cudaStream_t s = ctx->stream;
  bool ok = true;
  long long h2d = 0;
  // Whole grids go by copy engine on the copy stream while the fetch kernel
  // pulls the sparse grids' touched rows on `stream`: PCIe carries both at
  // once (measured 53.4 GB/s together vs 55.6 copy-engine-only / 51.5
  // zero-copy-only, profiles/r1/pcie_ceiling.txt).  The plan inputs go first
  // on `stream` since the fetch needs them.
  ok = cudaEventRecord(ctx->fork, s) == cudaSuccess && cudaStreamWaitEvent(ctx->copy_stream, ctx->fork, 0) ==
       cudaSuccess;
  for (int t = 0; t < n_tiles && ok; ++t) {
    if (src[t]) continue;  // fetched row by row below
    const size_t nb = (size_t)spatial_shape[2 * t] * spatial_shape[2 * t + 1] * channels * esz;
    if (nb == 0) continue;
    ok = cudaMemcpyAsync(d_tab + (size_t)start[t] * channels * esz, level_data[t], nb, cudaMemcpyHostToDevice,
                         ctx->copy_stream) == cudaSuccess;
    h2d += (long long)nb;
  }
  ok = ok && cudaEventRecord(ctx->join, ctx->copy_stream) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(d_shape, spatial_shape, (size_t)n_tiles * 8, cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(d_start, start.data(), (size_t)n_tiles * 8, cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(d_off, offsets, (size_t)(n_queries + 1) * 8, cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (S > 0) {
    ok = ok && cudaMemcpyAsync(d_cam, camera_index, S * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(d_lvl, level, S * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(d_u, u, S * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(d_v, v, S * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(d_w, weight, S * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
  }
  if (!ok) {
    cudaStreamSynchronize(ctx->copy_stream);
    return MSDA_CUDA_ERROR;
  }
  h2d += (long long)(n_tiles * 16 + (n_queries + 1) * 8 + S * 20);
  if (any_fetch) {
    ok = cudaMemcpyAsync(d_src, src.data(), (size_t)n_tiles * 8, cudaMemcpyHostToDevice, s) == cudaSuccess &&
         cudaMemsetAsync(d_bm, 0, bm_b + 256, s) == cudaSuccess;  // bitmap + counter
    FetchArgs fa{d_cam, d_lvl, d_u, d_v, S, n_cams, n_levels, d_shape, d_start, d_src, d_tab, d_bm, d_fetched,
                 (int32_t)(channels * esz)};
    const int64_t blocks = std::min<int64_t>((S + 7) / 8, (int64_t)num_sms_for_current_device() * 16);
    if (ok && blocks > 0) fetch_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(fa);
    ok = ok && cudaGetLastError() == cudaSuccess;
  }
  ok = ok && cudaStreamWaitEvent(s, ctx->join, 0) == cudaSuccess;
  if (!ok) {
    cudaStreamSynchronize(ctx->copy_stream);
    return MSDA_CUDA_ERROR;
  }
  // every return from here on first drains both streams: the caller's host
  // buffers may still be the source of in-flight DMAs
  auto fail = [&](int32_t code) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamSynchronize(s);
    return code;
  };
  if (cvt_half) {
    if (launch_f32_to_f16(reinterpret_cast<const float*>(d_tab), reinterpret_cast<__half*>(d_half),
                          rows * (int64_t)channels, s) != cudaSuccess)
      return fail(MSDA_CUDA_ERROR);
  }
  msda_features_t f{};
  f.data = cvt_half ? d_half : d_tab;
  f.dtype = dev_dtype;
  f.batch = 1;
  f.n_cams = n_cams;
  f.n_levels = n_levels;
  f.channels = channels;
  f.n_rows = rows;
  f.spatial_shape = d_shape;
  f.scale_start_index = d_start;
  f.spatial_shape_host = spatial_shape;
  msda_csr_plan_t pl{n_queries, S, d_off, d_cam, d_lvl, d_u, d_v, d_w};
  st = msda_csr(&f, &pl, precision, normalize, d_out, d_emp, d_ws, ws_b, s);
  if (st != MSDA_OK) return fail(st);
  if (cudaMemcpyAsync(out, d_out, (size_t)n_queries * channels * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail(MSDA_CUDA_ERROR);
  if (empty && cudaMemcpyAsync(empty, d_emp, (size_t)n_queries, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail(MSDA_CUDA_ERROR);
  int32_t dev_status = 0;
  int64_t detail = -1;
  st = msda_read_status(d_ws, s, &dev_status, &detail);  // synchronises the stream
  if (st != MSDA_OK) return fail(st);
  ctx->last_detail = detail;
  if (any_fetch) {
    unsigned long long rows_fetched = 0;
    if (cudaMemcpy(&rows_fetched, d_fetched, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return fail(MSDA_CUDA_ERROR);
    h2d += (long long)(rows_fetched * channels * esz);
  }
  ctx->last_h2d_bytes = h2d;
  return dev_status;
}


// bilinear_sample over HOST buffers: grid (H, W, C) f32, n coordinates, out
// [n, C].  A page-locked grid is read in place by the kernel (only the corner
// rows cross PCIe); a pageable one is copied whole into the context arena.
int32_t msda_bilinear_host(msda_context_t* ctx, const float* grid, int32_t H, int32_t W, int32_t C, int64_t n,
                           const float* u, const float* v, float* out) {
  if (!ctx || !grid || H <= 0 || W <= 0 || C <= 0 || n < 0 || (n > 0 && (!u || !v || !out))) return MSDA_BAD_ARG;
  if ((int64_t)H * W >= (int64_t(1) << 31)) return MSDA_BAD_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return MSDA_CUDA_ERROR;
  ctx->last_detail = -1;
  if (n == 0) return MSDA_OK;
  const size_t grid_b = (size_t)H * W * C * 4;
  const float* d_grid = nullptr;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, grid) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
    d_grid = reinterpret_cast<const float*>(pa.devicePointer);
  else
    cudaGetLastError();
  const size_t gb = d_grid ? 0 : align_up(grid_b, 256), cb = align_up((size_t)n * 4, 256);
  const size_t ob = align_up((size_t)n * C * 4, 256);
  int32_t st = ctx_reserve(ctx, gb + 2 * cb + ob);
  if (st != MSDA_OK) return st;
  char* p = reinterpret_cast<char*>(ctx->arena);
  cudaStream_t s = ctx->stream;
  long long h2d = 2 * n * 4;
  bool ok = true;
  if (!d_grid) {
    ok = cudaMemcpyAsync(p, grid, grid_b, cudaMemcpyHostToDevice, s) == cudaSuccess;
    d_grid = reinterpret_cast<const float*>(p);
    h2d += (long long)grid_b;
  }
  float* d_u = reinterpret_cast<float*>(p + gb);
  float* d_v = reinterpret_cast<float*>(p + gb + cb);
  float* d_out = reinterpret_cast<float*>(p + gb + 2 * cb);
  ok = ok && cudaMemcpyAsync(d_u, u, (size_t)n * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(d_v, v, (size_t)n * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (ok) {
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)num_sms_for_current_device() * 16);
    bilinear_kernel<<<(unsigned)blocks, 256, 0, s>>>(d_grid, H, W, C, d_u, d_v, n, d_out);
    ok = cudaGetLastError() == cudaSuccess;
  }
  ok = ok && cudaMemcpyAsync(out, d_out, (size_t)n * C * 4, cudaMemcpyDeviceToHost, s) == cudaSuccess;
  const bool synced = cudaStreamSynchronize(s) == cudaSuccess;
  ctx->last_h2d_bytes = h2d;
  return ok && synced ? MSDA_OK : MSDA_CUDA_ERROR;
}

}  // extern "C"
