// Occlusion visibility v_i for every (camera, object) pair — sm_100a.
//
// Restates mvtrack3d.visibility (visibility.py:46-115), batched:
//   rect_kernel      one thread per (camera, object): the eight box corners
//                    (geometry.py:195-204: bit 0 -> +l/2, bit 1 -> +w/2,
//                    bit 2 -> +h/2, rotated by yaw, translated), projected in
//                    f64 with behind-camera corners skipped (geometry.py:162-
//                    182); axis-aligned bounds + mean corner depth, or
//                    "fully behind" when no corner projects.
//   visible_kernel   one CTA per (camera, target): blockers = every other
//                    object of that camera whose rect exists and whose mean
//                    depth is strictly smaller, compacted into shared memory;
//                    grid^2 sample points at cell centres of the target rect
//                    are visible when inside [0, W) x [0, H) and outside every
//                    blocker rect (closed bounds); the count is block-reduced.
// Bit-exact with the reference on the same host arithmetic: cos / sin of the
// yaw come from the caller (Python's math.cos / math.sin in rot_z,
// geometry.py:50-53 — the device libm differs in the last bit); the two
// numpy matrix products follow the OpenBLAS (SkylakeX) kernels numpy calls,
// measured here bit for bit: `local @ rot_z(yaw).T` (geometry.py:205) is the
// FMA chain k = 0, 1, 2 per output, `R @ p` (geometry.py:176) is
// fma(R2, p2, fma(R0, p0, R1 * p1)); the rest is separately rounded
// (__dmul_rn / __dadd_rn / __ddiv_rn) like numpy's scalar ops.
#include <algorithm>

#include "msda_common.cuh"

namespace msda {
namespace {

struct Rect {
  double u0, u1, v0, v1, depth;
  int valid;
  int pad;
};

struct VisArgs {
  const double* K;    // [cams, 4]
  const double* R;    // [cams, 9]
  const double* T;    // [cams, 3]
  const int32_t* wh;  // [cams, 2] image width, height
  const double* obj;  // [n_obj, 9] x, y, z, w, l, h, yaw, cos(yaw), sin(yaw) (host libm)
  int32_t cams, n_obj, grid;
  Rect* rects;        // [cams, n_obj]
  float* vis;         // [cams, n_obj]
  uint8_t* behind;    // [cams, n_obj]
};

// one row of numpy's `R @ p` for a 3x3 R (OpenBLAS dgemv order)
__device__ __forceinline__ double dot3(const double* r, double x, double y, double z) {
  return __fma_rn(r[2], z, __fma_rn(r[0], x, __dmul_rn(r[1], y)));
}

__global__ void rect_kernel(VisArgs a) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)a.cams * a.n_obj) return;
  const int cam = (int)(id / a.n_obj), o = (int)(id % a.n_obj);
  const double* s = a.obj + (int64_t)o * 9;
  const double c = s[7], sn = s[8];
  const double hl = s[4] / 2.0, hw = s[3] / 2.0, hh = s[5] / 2.0;
  const double* R = a.R + cam * 9;
  const double* T = a.T + cam * 3;
  const double* K = a.K + cam * 4;
  Rect r{INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0, 0, 0};
  double d[8];
  int n = 0;
  for (int i = 0; i < 8; ++i) {
    const double lx = (i & 1) ? hl : -hl, ly = (i & 2) ? hw : -hw, lz = (i & 4) ? hh : -hh;
    // local @ rot_z(yaw)^T + centre: per output the FMA chain over the rows
    // of rot_z = [[c, -s, 0], [s, c, 0], [0, 0, 1]] (OpenBLAS dgemm order)
    const double px = __dadd_rn(__fma_rn(lz, 0.0, __fma_rn(ly, -sn, __dmul_rn(lx, c))), s[0]);
    const double py = __dadd_rn(__fma_rn(lz, 0.0, __fma_rn(ly, c, __dmul_rn(lx, sn))), s[1]);
    const double pz = __dadd_rn(__fma_rn(lz, 1.0, __fma_rn(ly, 0.0, __dmul_rn(lx, 0.0))), s[2]);
    const double xc = __dadd_rn(dot3(R, px, py, pz), T[0]);
    const double yc = __dadd_rn(dot3(R + 3, px, py, pz), T[1]);
    const double zc = __dadd_rn(dot3(R + 6, px, py, pz), T[2]);
    if (!(zc > 1e-6)) continue;
    const double u = __dadd_rn(__ddiv_rn(__dmul_rn(K[0], xc), zc), K[2]);
    const double v = __dadd_rn(__ddiv_rn(__dmul_rn(K[1], yc), zc), K[3]);
    r.u0 = fmin(r.u0, u);
    r.u1 = fmax(r.u1, u);
    r.v0 = fmin(r.v0, v);
    r.v1 = fmax(r.v1, v);
    d[n++] = zc;
  }
  // np.mean: a sequential sum below 8 values, numpy's 8-way pairwise tree at 8
  double dsum = 0.0;
  if (n == 8) {
    dsum = __dadd_rn(__dadd_rn(__dadd_rn(d[0], d[1]), __dadd_rn(d[2], d[3])),
                     __dadd_rn(__dadd_rn(d[4], d[5]), __dadd_rn(d[6], d[7])));
  } else {
    for (int i = 0; i < n; ++i) dsum = __dadd_rn(dsum, d[i]);
  }
  r.valid = n > 0;
  r.depth = n > 0 ? __ddiv_rn(dsum, (double)n) : 0.0;
  a.rects[id] = r;
}

__global__ void __launch_bounds__(256) visible_kernel(VisArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Rect* s_b = reinterpret_cast<Rect*>(smem_raw);
  __shared__ int s_nb;
  __shared__ int s_cnt[8];
  const int cam = blockIdx.y, t = blockIdx.x;
  const Rect* cr = a.rects + (int64_t)cam * a.n_obj;
  const Rect tr = cr[t];
  const int64_t out = (int64_t)cam * a.n_obj + t;
  if (!tr.valid) {
    if (threadIdx.x == 0) {
      a.vis[out] = 0.0f;
      a.behind[out] = 1;
    }
    return;
  }
  if (threadIdx.x == 0) s_nb = 0;
  __syncthreads();
  for (int o = threadIdx.x; o < a.n_obj; o += blockDim.x) {
    const Rect b = cr[o];
    if (o != t && b.valid && b.depth < tr.depth) s_b[atomicAdd(&s_nb, 1)] = b;
  }
  __syncthreads();
  const int nb = s_nb;
  const double W = (double)a.wh[2 * cam], H = (double)a.wh[2 * cam + 1];
  const int g = a.grid;
  const double du = __dadd_rn(tr.u1, -tr.u0), dv = __dadd_rn(tr.v1, -tr.v0);
  int cnt = 0;
  for (int p = threadIdx.x; p < g * g; p += blockDim.x) {
    const int iy = p / g, ix = p - iy * g;
    const double su = __ddiv_rn((double)ix + 0.5, (double)g), sv = __ddiv_rn((double)iy + 0.5, (double)g);
    const double u = __dadd_rn(tr.u0, __dmul_rn(su, du));
    const double v = __dadd_rn(tr.v0, __dmul_rn(sv, dv));
    bool vis = u >= 0.0 && u < W && v >= 0.0 && v < H;
    for (int b = 0; b < nb && vis; ++b)
      vis = !(s_b[b].u0 <= u && u <= s_b[b].u1 && s_b[b].v0 <= v && v <= s_b[b].v1);
    cnt += vis ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += s_cnt[w];
    a.vis[out] = (float)((double)total / (double)(g * g));
    a.behind[out] = 0;
  }
}

// ---------------------------------------------------------------------------
// Feature painting (simulator.py:249-289): the producer
// of the pyramids the MSDA path reads, written straight into the
// channel-last concatenated table (mc_ms_feat) in the compute dtype.
//   cell centre (x + 0.5) * stride, (y + 0.5) * stride (f64, simulator.py:
//   275-277); winner = the nearest (strictly smaller mean depth, first in
//   entity order on ties) rect containing it (closed bounds, visibility.py:
//   32-33); moving objects add their f64 signature, occluders nothing
//   (simulator.py:283-288); value = f32(background + signature).
// The background is the caller's f64 grid (bit-identical to the reference
// given the reference's numpy draw) or, when absent, drawn on device:
// Philox4x32-10 (counter = element / 4, tile, frame; key = seed) and a
// Box-Muller transform — the same N(0, sigma) law, not the same numbers.

struct PaintArgs {
  const Rect* rects;        // [cams, n_ent]
  const double* strides;    // [L]
  const int32_t* shape;     // [cams, L, 2]
  const int64_t* start;     // [cams, L]
  const double* sig;        // [n_obj, C]
  const double* bg;         // [rows, C] or null
  void* out;                // [rows, C]
  int32_t cams, L, C, n_ent, n_obj, dtype, frame;
  float sigma;
  uint32_t key0, key1;
};

constexpr int kPaintCells = 64;  // cells per CTA

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ k0, lo1, hi0 ^ ctr.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ctr;
}

__device__ __forceinline__ void store4(void* out, int dtype, int64_t i, const float* f) {
  if (dtype == MSDA_F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + i) = make_float4(f[0], f[1], f[2], f[3]);
  } else if (dtype == MSDA_F16) {
    const __half2 a = __halves2half2(__float2half_rn(f[0]), __float2half_rn(f[1]));
    const __half2 b = __halves2half2(__float2half_rn(f[2]), __float2half_rn(f[3]));
    *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(out) + i) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  } else {
    const __nv_bfloat162 a = __halves2bfloat162(__float2bfloat16_rn(f[0]), __float2bfloat16_rn(f[1]));
    const __nv_bfloat162 b = __halves2bfloat162(__float2bfloat16_rn(f[2]), __float2bfloat16_rn(f[3]));
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + i) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}

// CTA = 64 cells of one (camera, level) grid.  Four threads per cell run the
// depth contest (a quarter of the entities each); then every thread owns a fixed 4-channel chunk
// (C % 4 == 0) and walks the cells with stride blockDim / (C / 4).
__global__ void __launch_bounds__(256) paint_kernel(PaintArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Rect* s_r = reinterpret_cast<Rect*>(smem_raw);
  __shared__ int s_win[kPaintCells];
  const int t = blockIdx.y;  // tile = cam * L + level
  const int cam = t / a.L, level = t - cam * a.L;
  const int H = a.shape[2 * t], W = a.shape[2 * t + 1];
  const int cell0 = blockIdx.x * kPaintCells;
  if (cell0 >= H * W) return;
  for (int e = threadIdx.x; e < a.n_ent; e += blockDim.x) s_r[e] = a.rects[(int64_t)cam * a.n_ent + e];
  __syncthreads();
  const double stride = a.strides[level];
  {  // depth contest: 4 threads per cell, each a quarter of the entities, then the
     // lexicographic minimum (depth, entity index) == the first strictly-nearest
    const int cl = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int cell = cell0 + cl;
    int win = -1;
    double best = INFINITY;
    if (cell < H * W) {
      const int y = cell / W, x = cell - y * W;
      const double u = __dmul_rn((double)x + 0.5, stride), v = __dmul_rn((double)y + 0.5, stride);
      for (int e = part; e < a.n_ent; e += 4) {
        const Rect r = s_r[e];
        if (r.valid && r.u0 <= u && u <= r.u1 && r.v0 <= v && v <= r.v1 && r.depth < best) {
          best = r.depth;
          win = e;
        }
      }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ow = __shfl_xor_sync(0xffffffffu, win, o);
      if (ow >= 0 && (win < 0 || ob < best || (ob == best && ow < win))) {
        best = ob;
        win = ow;
      }
    }
    if (part == 0) s_win[cl] = win < a.n_obj ? win : -1;  // occluders paint nothing
  }
  __syncthreads();
  const int n_cells = min(kPaintCells, H * W - cell0);
  const int chunks = a.C >> 2;  // 4-channel chunks per cell
  const int c4 = threadIdx.x % chunks;
  const int cstep = blockDim.x / chunks;
  if ((int)threadIdx.x >= cstep * chunks) return;
  const int64_t row0 = a.start[t] + cell0;
  for (int cl = threadIdx.x / chunks; cl < n_cells; cl += cstep) {
    const int64_t o = (row0 + cl) * a.C + 4 * c4;
    double v[4];
    if (a.bg) {
      const double4 b = *reinterpret_cast<const double4*>(a.bg + o);  // f64 background row chunk
      v[0] = b.x;
      v[1] = b.y;
      v[2] = b.z;
      v[3] = b.w;
    } else {  // device background: one Philox4x32-10 draw -> four N(0, sigma) (Box-Muller, f32)
      const uint4 r = philox4x32_10(make_uint4((uint32_t)(o >> 2), (uint32_t)(o >> 34), (uint32_t)t,
                                               (uint32_t)a.frame), a.key0, a.key1);
      // 23-bit uniforms via the exponent trick: (0, 1] for the logs, [0, 1) for the angles
      const float u1 = 2.0f - __uint_as_float((r.x >> 9) | 0x3f800000u);
      const float u3 = 2.0f - __uint_as_float((r.z >> 9) | 0x3f800000u);
      const float a1 = __uint_as_float((r.y >> 9) | 0x3f800000u) - 1.0f;
      const float a2 = __uint_as_float((r.w >> 9) | 0x3f800000u) - 1.0f;
      const float m1 = sqrtf(-2.0f * __logf(u1)) * a.sigma, m2 = sqrtf(-2.0f * __logf(u3)) * a.sigma;
      float s1, c1, s2, c2;
      __sincosf(6.283185307f * a1, &s1, &c1);
      __sincosf(6.283185307f * a2, &s2, &c2);
      const int w = s_win[cl];
      if (w < 0) {  // background only: straight to the storage dtype
        const float nz[4] = {m1 * c1, m1 * s1, m2 * c2, m2 * s2};
        store4(a.out, a.dtype, o, nz);
        continue;
      }
      v[0] = m1 * c1;
      v[1] = m1 * s1;
      v[2] = m2 * c2;
      v[3] = m2 * s2;
    }
    const int w = s_win[cl];
    if (w >= 0) {  // simulator.py:288 values[mask] += signature (f64)
      const double4 sg = *reinterpret_cast<const double4*>(a.sig + (int64_t)w * a.C + 4 * c4);
      v[0] = __dadd_rn(v[0], sg.x);
      v[1] = __dadd_rn(v[1], sg.y);
      v[2] = __dadd_rn(v[2], sg.z);
      v[3] = __dadd_rn(v[3], sg.w);
    }
    float f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = __double2float_rn(v[j]);  // simulator.py:289 astype(np.float32)
    store4(a.out, a.dtype, o, f);
  }
}

}  // namespace
}  // namespace msda

using namespace msda;

extern "C" {

size_t msda_visibility_workspace_size(int32_t n_cams, int32_t n_objects) {
  return align_up((size_t)n_cams * n_objects * sizeof(Rect), 256);
}

int32_t msda_visibility(const msda_cameras_t* cams, const int32_t* image_wh, int32_t n_cams, const double* objects,
                        int32_t n_objects, int32_t grid, float* visibility, uint8_t* fully_behind, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!cams || !cams->K || !cams->R || !cams->t || !image_wh || n_cams < 0 || n_objects < 0) return MSDA_BAD_ARG;
  if (grid < 2 || grid > 4096) return MSDA_BAD_ARG;
  if (n_cams == 0 || n_objects == 0) return MSDA_OK;
  if (!objects || !visibility || !fully_behind || !workspace ||
      workspace_bytes < msda_visibility_workspace_size(n_cams, n_objects))
    return MSDA_BAD_ARG;
  const size_t smem = (size_t)n_objects * sizeof(Rect);
  if (smem > 200 * 1024) return MSDA_BAD_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  VisArgs a{cams->K, cams->R, cams->t, image_wh, objects, n_cams, n_objects, grid,
            reinterpret_cast<Rect*>(workspace), visibility, fully_behind};
  const int64_t pairs = (int64_t)n_cams * n_objects;
  rect_kernel<<<(unsigned)((pairs + 127) / 128), 128, 0, s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(visible_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  visible_kernel<<<dim3((unsigned)n_objects, (unsigned)n_cams), 256, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

size_t msda_paint_workspace_size(int32_t n_cams, int32_t n_entities) {
  return align_up((size_t)n_cams * n_entities * sizeof(Rect), 256);
}

int32_t msda_paint(const msda_cameras_t* cams, int32_t n_cams, int32_t n_levels, const double* strides,
                   const int32_t* spatial_shape, const int32_t* spatial_shape_host, const int64_t* scale_start_index,
                   int32_t channels, const double* entities, int32_t n_objects, int32_t n_occluders,
                   const double* signatures, const double* background, float sigma, uint64_t seed, int32_t frame,
                   int32_t out_dtype, void* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!cams || !cams->K || !cams->R || !cams->t || n_cams <= 0 || n_levels <= 0 || channels <= 0) return MSDA_BAD_ARG;
  if (!strides || !spatial_shape || !spatial_shape_host || !scale_start_index || !out) return MSDA_BAD_ARG;
  if (n_objects < 0 || n_occluders < 0 || out_dtype < MSDA_F32 || out_dtype > MSDA_BF16) return MSDA_BAD_ARG;
  const int32_t n_ent = n_objects + n_occluders;
  if (n_ent > 0 && (!entities || !workspace || workspace_bytes < msda_paint_workspace_size(n_cams, n_ent)))
    return MSDA_BAD_ARG;
  if (n_objects > 0 && !signatures) return MSDA_BAD_ARG;
  if (channels % 4 || channels / 4 > 256) return MSDA_BAD_ARG;  // 4-channel chunks, one pass of a CTA per cell
  // vector access: 4 channels per thread (double4 reads, 16/8-B writes)
  if (reinterpret_cast<uintptr_t>(out) % 16 || reinterpret_cast<uintptr_t>(background) % 32 ||
      reinterpret_cast<uintptr_t>(signatures) % 32)
    return MSDA_BAD_ARG;
  const size_t smem = (size_t)n_ent * sizeof(Rect);
  if (smem > 200 * 1024) return MSDA_BAD_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Rect* rects = reinterpret_cast<Rect*>(workspace);
  if (n_ent > 0) {
    VisArgs va{cams->K, cams->R, cams->t, nullptr, entities, n_cams, n_ent, 2, rects, nullptr, nullptr};
    const int64_t pairs = (int64_t)n_cams * n_ent;
    rect_kernel<<<(unsigned)((pairs + 127) / 128), 128, 0, s>>>(va);
    if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
  }
  int max_cells = 0;
  for (int i = 0; i < n_cams * n_levels; ++i) {
    if (spatial_shape_host[2 * i] <= 0 || spatial_shape_host[2 * i + 1] <= 0) return MSDA_BAD_ARG;
    max_cells = std::max(max_cells, spatial_shape_host[2 * i] * spatial_shape_host[2 * i + 1]);
  }
  PaintArgs a{rects, strides, spatial_shape, scale_start_index, signatures, background, out, n_cams, n_levels,
              channels, n_ent, n_objects, out_dtype, frame, sigma, (uint32_t)seed, (uint32_t)(seed >> 32)};
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(paint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  const dim3 grid((unsigned)((max_cells + kPaintCells - 1) / kPaintCells), (unsigned)(n_cams * n_levels));
  paint_kernel<<<grid, 256, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

}  // extern "C"
