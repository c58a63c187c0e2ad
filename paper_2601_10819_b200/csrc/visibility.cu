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
// The f64 arithmetic is separately rounded (__dmul_rn/__dadd_rn) like numpy's.
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
  const double* obj;  // [n_obj, 7] x, y, z, w, l, h, yaw
  int32_t cams, n_obj, grid;
  Rect* rects;        // [cams, n_obj]
  float* vis;         // [cams, n_obj]
  uint8_t* behind;    // [cams, n_obj]
};

__device__ __forceinline__ double dot3(const double* r, double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(r[0], x), __dmul_rn(r[1], y)), __dmul_rn(r[2], z));
}

__global__ void rect_kernel(VisArgs a) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)a.cams * a.n_obj) return;
  const int cam = (int)(id / a.n_obj), o = (int)(id % a.n_obj);
  const double* s = a.obj + (int64_t)o * 7;
  const double c = cos(s[6]), sn = sin(s[6]);
  const double hl = s[4] / 2.0, hw = s[3] / 2.0, hh = s[5] / 2.0;
  const double* R = a.R + cam * 9;
  const double* T = a.T + cam * 3;
  const double* K = a.K + cam * 4;
  Rect r{INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0, 0, 0};
  double d[8];
  int n = 0;
  for (int i = 0; i < 8; ++i) {
    const double lx = (i & 1) ? hl : -hl, ly = (i & 2) ? hw : -hw, lz = (i & 4) ? hh : -hh;
    // local @ rot_z(yaw)^T + centre
    const double px = __dadd_rn(__dadd_rn(__dmul_rn(lx, c), __dmul_rn(ly, -sn)), s[0]);
    const double py = __dadd_rn(__dadd_rn(__dmul_rn(lx, sn), __dmul_rn(ly, c)), s[1]);
    const double pz = __dadd_rn(lz, s[2]);
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

}  // extern "C"
