// Shared device helpers for the msda_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/msda_b200.h"

namespace msda {

// Per-sample record produced by the plan stage and consumed by the gather
// stage: absolute feature rows of the four bilinear corners (-1 = outside the
// grid, reads as zero, features.py:214-217) and the four f32 interpolation
// weights w00, w10, w01, w11 (features.py:199-208).  32 bytes, 16-B aligned.
struct __align__(16) SampleRec {
  int32_t row[4];
  float iw[4];
};

// Device status word at the head of every workspace (zeroed before a call).
// The first error code wins; among reports of that code the smallest detail
// (query / sample index) is kept, so the message names the first offending
// query as the reference's sequential loop does (features.py:264-269).
// detail_enc holds ~detail (0 = none) so that atomicMax keeps the minimum.
struct DevStatus {
  int32_t code;
  int32_t pad;
  unsigned long long detail_enc;
};
constexpr size_t kStatusBytes = 256;

__device__ __forceinline__ void set_status(DevStatus* st, int code, long long detail) {
  const int prev = atomicCAS(&st->code, 0, code);
  if ((prev == 0 || prev == code) && detail >= 0) atomicMax(&st->detail_enc, ~(unsigned long long)detail);
}
__host__ __device__ inline long long status_detail(const DevStatus& st) {
  return (st.code && st.detail_enc) ? (long long)~st.detail_enc : -1;
}

// Order-preserving float -> uint32 map (ascending float order == ascending
// key order).  -0.0 is canonicalised to +0.0 first, matching numpy's sort,
// which treats them as equal (features.py:261-263); all reference arithmetic
// is insensitive to the sign of a zero coordinate or weight here.
__device__ __forceinline__ uint32_t ord_f32(float f) {
  uint32_t b = __float_as_uint(f);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Bilinear record for cell coordinates (u, v) on a grid of H x W rows
// starting at `start`: the float32 arithmetic of features.py:197-208 and the
// float in-bounds tests of features.py:318-321 (no integer overflow for huge
// coordinates), separately rounded (no FMA contraction).
__device__ __forceinline__ SampleRec make_record(float u, float v, int64_t start, int H, int W) {
  SampleRec r;
  const float x0f = floorf(u), y0f = floorf(v);
  const float fu = __fsub_rn(u, x0f), fv = __fsub_rn(v, y0f);
  const float omu = __fsub_rn(1.0f, fu), omv = __fsub_rn(1.0f, fv);
  r.iw[0] = __fmul_rn(omu, omv);
  r.iw[1] = __fmul_rn(fu, omv);
  r.iw[2] = __fmul_rn(omu, fv);
  r.iw[3] = __fmul_rn(fu, fv);
  const bool inx0 = (x0f >= 0.0f) && (x0f <= (float)(W - 1));
  const bool inx1 = (x0f >= -1.0f) && (x0f <= (float)(W - 2));
  const bool iny0 = (y0f >= 0.0f) && (y0f <= (float)(H - 1));
  const bool iny1 = (y0f >= -1.0f) && (y0f <= (float)(H - 2));
  const int x0 = (inx0 || inx1) ? (int)x0f : 0;
  const int y0 = (iny0 || iny1) ? (int)y0f : 0;
  const int64_t base = start + (int64_t)y0 * W + x0;
  r.row[0] = (inx0 && iny0) ? (int32_t)base : -1;
  r.row[1] = (inx1 && iny0) ? (int32_t)(base + 1) : -1;
  r.row[2] = (inx0 && iny1) ? (int32_t)(base + W) : -1;
  r.row[3] = (inx1 && iny1) ? (int32_t)(base + W + 1) : -1;
  return r;
}

// ---- vector loads of VEC channels (read-only, streaming through L1) ----
template <int BYTES>
struct RawVec;
template <>
struct RawVec<16> { uint4 v; };
template <>
struct RawVec<8> { uint2 v; };
template <>
struct RawVec<4> { uint32_t v; };

template <int BYTES>
__device__ __forceinline__ RawVec<BYTES> ldg_vec(const void* p);
template <>
__device__ __forceinline__ RawVec<16> ldg_vec<16>(const void* p) {
  RawVec<16> r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.v.x), "=r"(r.v.y), "=r"(r.v.z), "=r"(r.v.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ RawVec<8> ldg_vec<8>(const void* p) {
  RawVec<8> r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.v.x), "=r"(r.v.y) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ RawVec<4> ldg_vec<4>(const void* p) {
  RawVec<4> r;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r.v) : "l"(p));
  return r;
}

template <int BYTES>
__device__ __forceinline__ RawVec<BYTES> zero_vec() {
  RawVec<BYTES> r;
  uint32_t* w = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < BYTES / 4; ++i) w[i] = 0u;
  return r;
}

// Widen VEC stored elements to f32 (exact for f16 / bf16).
template <typename T, int VEC>
__device__ __forceinline__ void to_f32(const RawVec<VEC * sizeof(T)>& r, float* out) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&r);
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) out[i] = __uint_as_float(w[i]);
  } else if constexpr (std::is_same<T, __half>::value) {
#pragma unroll
    for (int i = 0; i < VEC / 2; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f = __half22float2(h);
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC / 2; ++i) {  // bf16 -> f32 is a 16-bit shift
      out[2 * i] = __uint_as_float(w[i] << 16);
      out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}

// ---- whole-lane row slices: NV x 16 B per lane (read-only path) ----
template <int NV>
struct Row {
  uint4 v[NV];
};

template <int NV>
__device__ __forceinline__ Row<NV> ld_row(const char* p) {
  Row<NV> r;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.v[i].x), "=r"(r.v[i].y), "=r"(r.v[i].z), "=r"(r.v[i].w)
                 : "l"(p + 16 * i));
  return r;
}

// VEC stored elements (packed in 32-bit words) -> f32, exact
template <typename T, int VEC>
__device__ __forceinline__ void raw_to_f32(const uint32_t* raw, float* f) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) f[e] = __uint_as_float(raw[e]);
  } else if constexpr (std::is_same<T, __half>::value) {
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) {
      const float2 p = __half22float2(*reinterpret_cast<const __half2*>(&raw[e]));
      f[2 * e] = p.x;
      f[2 * e + 1] = p.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) {  // bf16 -> f32 is a 16-bit shift
      f[2 * e] = __uint_as_float(raw[e] << 16);
      f[2 * e + 1] = __uint_as_float(raw[e] & 0xffff0000u);
    }
  }
}

// Keypoint p of an anchor (x, y, z, w, l, h, yaw, vx, vy, vz), float64:
// p = 0 centre, 1..6 the face centres (+l, -l, +w, -w, +h, -h halves),
// p >= 7 learned offsets scaled by the half extents (geometry.py:207-247),
// rotated by yaw, shifted by velocity * dt (geometry.py:250-255).
// Returns false when a learned offset component leaves [-1, 1].
__device__ inline bool anchor_keypoint(const float* an, int p, const float* offsets, float dt, double* out) {
  const double x = an[0], y = an[1], z = an[2], w = an[3], l = an[4], h = an[5], yaw = an[6];
  const double c = cos(yaw), s = sin(yaw);
  const double hl = l / 2.0, hw = w / 2.0, hh = h / 2.0;
  double lx = 0.0, ly = 0.0, lz = 0.0;
  bool ok = true;
  switch (p) {
    case 0: break;
    case 1: lx = hl; break;
    case 2: lx = -hl; break;
    case 3: ly = hw; break;
    case 4: ly = -hw; break;
    case 5: lz = hh; break;
    case 6: lz = -hh; break;
    default: {
      const float* o = offsets + (p - 7) * 3;
      ok = fabsf(o[0]) <= 1.0f && fabsf(o[1]) <= 1.0f && fabsf(o[2]) <= 1.0f;
      lx = (double)o[0] * hl;
      ly = (double)o[1] * hw;
      lz = (double)o[2] * hh;
    }
  }
  out[0] = (c * lx - s * ly) + x + (double)an[7] * (double)dt;
  out[1] = (s * lx + c * ly) + y + (double)an[8] * (double)dt;
  out[2] = lz + z + (double)an[9] * (double)dt;
  return ok;
}

// Pinhole projection (geometry.py:162-182), float64: p_cam = R p + t; a point
// with depth <= 1e-6 is behind the camera (returns false); u = fx*x/z + cx.
__device__ inline bool project_f64(const double* K, const double* R, const double* T, const double* p, double& u,
                                   double& v) {
  const double xc = (R[0] * p[0] + R[1] * p[1] + R[2] * p[2]) + T[0];
  const double yc = (R[3] * p[0] + R[4] * p[1] + R[5] * p[2]) + T[1];
  const double zc = (R[6] * p[0] + R[7] * p[1] + R[8] * p[2]) + T[2];
  if (!(zc > 1e-6)) return false;
  u = K[0] * xc / zc + K[2];
  v = K[1] * yc / zc + K[3];
  return true;
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- cp.async (LDGSTS) with zero-fill for out-of-grid corners ----
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
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- the reference's exact f32 expression tree ----
// Two samples' trees side by side (independent chains in program order), then
// the two sequential adds: acc = (acc + t0) + t1, each rounded once — the same
// bits as two exact_accumulate calls, with more instruction-level parallelism.
template <int VEC>
__device__ __forceinline__ void exact_accumulate2(float* acc, const float (*c0)[VEC], const float4 iw0, const float wn0,
                                                  const float (*c1)[VEC], const float4 iw1, const float wn1, bool two,
                                                  const float2 one2, const float2 nz2) {
  static_assert(VEC % 2 == 0, "pairs");
  float2 tw0[VEC / 2], tw1[VEC / 2];
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const float2 a0 = __ffma2_rn(make_float2(c0[0][e], c0[0][e + 1]), make_float2(iw0.x, iw0.x), nz2);
    const float2 a1 = __ffma2_rn(make_float2(c1[0][e], c1[0][e + 1]), make_float2(iw1.x, iw1.x), nz2);
    const float2 b0 = __ffma2_rn(make_float2(c0[1][e], c0[1][e + 1]), make_float2(iw0.y, iw0.y), nz2);
    const float2 b1 = __ffma2_rn(make_float2(c1[1][e], c1[1][e + 1]), make_float2(iw1.y, iw1.y), nz2);
    const float2 d0 = __ffma2_rn(make_float2(c0[2][e], c0[2][e + 1]), make_float2(iw0.z, iw0.z), nz2);
    const float2 d1 = __ffma2_rn(make_float2(c1[2][e], c1[2][e + 1]), make_float2(iw1.z, iw1.z), nz2);
    const float2 f0 = __ffma2_rn(make_float2(c0[3][e], c0[3][e + 1]), make_float2(iw0.w, iw0.w), nz2);
    const float2 f1 = __ffma2_rn(make_float2(c1[3][e], c1[3][e + 1]), make_float2(iw1.w, iw1.w), nz2);
    const float2 t0 = __ffma2_rn(__ffma2_rn(a0, one2, b0), one2, __ffma2_rn(d0, one2, f0));
    const float2 t1 = __ffma2_rn(__ffma2_rn(a1, one2, b1), one2, __ffma2_rn(d1, one2, f1));
    tw0[e / 2] = __ffma2_rn(t0, make_float2(wn0, wn0), nz2);
    tw1[e / 2] = __ffma2_rn(t1, make_float2(wn1, wn1), nz2);
  }
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    float2 r = __ffma2_rn(tw0[e / 2], one2, make_float2(acc[e], acc[e + 1]));
    if (two) r = __ffma2_rn(tw1[e / 2], one2, r);
    acc[e] = r.x;
    acc[e + 1] = r.y;
  }
}

// acc[e] += wn * ((c0*w0 + c1*w1) + (c2*w2 + c3*w3)), two channels per FFMA2,
// every product and sum rounded once (x*y + -0 == round(x*y); x*1 + y ==
// round(x + y)).
template <int VEC>
__device__ __forceinline__ void exact_accumulate(float* acc, const float (*c)[VEC], const float4 iw, const float wn,
                                                 const float2 one2, const float2 nz2) {
  static_assert(VEC % 2 == 0, "pairs");
  const float2 w0 = make_float2(iw.x, iw.x), w1 = make_float2(iw.y, iw.y);
  const float2 w2 = make_float2(iw.z, iw.z), w3 = make_float2(iw.w, iw.w);
  const float2 ws = make_float2(wn, wn);
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const float2 a = __ffma2_rn(make_float2(c[0][e], c[0][e + 1]), w0, nz2);
    const float2 b = __ffma2_rn(make_float2(c[1][e], c[1][e + 1]), w1, nz2);
    const float2 d = __ffma2_rn(make_float2(c[2][e], c[2][e + 1]), w2, nz2);
    const float2 f = __ffma2_rn(make_float2(c[3][e], c[3][e + 1]), w3, nz2);
    const float2 ab = __ffma2_rn(a, one2, b);
    const float2 df = __ffma2_rn(d, one2, f);
    const float2 t = __ffma2_rn(ab, one2, df);
    const float2 tw = __ffma2_rn(t, ws, nz2);
    const float2 r = __ffma2_rn(tw, one2, make_float2(acc[e], acc[e + 1]));
    acc[e] = r.x;
    acc[e + 1] = r.y;
  }
}



}  // namespace msda
