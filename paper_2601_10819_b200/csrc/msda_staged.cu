// Coarse-level dense FAST aggregation from on-chip staged maps
// (deformable_aggregation, Sparse4D layout) — sm_100a.
//
// Why: the anchor-major gather moves every in-grid corner row of every
// sample from L2 to the SMs (cfg3: 6.1 GB per layer, ~10x the algorithmic
// bytes) at the chip's L2-slice throughput cap.  Half of those rows belong to
// the two coarse levels, which are tiny and hot: at the cfg1/cfg3 shape a
// level-3 cell is read ~266 times per camera per call, a level-2 cell ~66
// times.  So the dense FAST call is split by level:
//   * fine levels (0, 1): the anchor-major pipelined gather (msda_exact.cu,
//     full 512-B / 1-KB rows per warp instruction), restricted to them;
//   * coarse levels (this kernel): per work item = (batch b, camera c,
//     128-byte channel slice s, anchor chunk), one elected thread stages the
//     slice of the camera's coarse levels — every row x 128 B, 880 rows =
//     112.6 KB at the cfg1 shape — into shared memory with TMA
//     (cp.async.bulk.tensor.2d, mbarrier complete_tx); the 16 warps then read
//     corner rows with conflict-free LDS.128 (8 lanes x 16 B per row).
// Both parts red.add their partial sums into the zeroed output (and weight
// sums); normalisation, if asked, is the separate group_normalize pass.
//
// Coarse kernel mapping: a row slice is 4 lanes x 32 B, so a warp holds 8
// groups; group g of a warp walks one anchor (the warp takes anchors in
// blocks of 8) through its P keypoints x the coarse levels, all groups in
// lockstep.  A sample's record (cell = loc * W - 0.5, the reference
// convention features.py:20-24; zero padding features.py:214-217) is built
// by the group's 4 lanes; out-of-grid corners read a zero row.  Keypoints
// p + 1 and p + 2 have their locations and weights in flight while p is
// summed.  At the anchor's end each group red.add's its slice partial: no
// cross-lane reduction.
#include <cuda.h>

#include <algorithm>
#include <atomic>

#include "msda_common.cuh"
#include "msda_exact.cuh"

namespace msda {
namespace {

// 8 warps: the coarse kernel runs beside the fine gather (forked stream), and
// a 256-thread CTA leaves registers for ~8 gather warps per SM (16 warps
// alone: 160 us; 8 warps beside the gather: cfg3 FAST_H2 382 vs 397 us total)
constexpr int kStWarps = 8;
constexpr int kStThreads = kStWarps * 32;
constexpr int kSliceBytes = 128;  // staged row slice: one 128-B line, 8 lanes x 16 B
constexpr int kBoxRows = 64;      // TMA box: 64 rows x 128 B
constexpr int kMaxLevels = 4;
constexpr int kStageBudget = 120 * 1024;
constexpr int kCoarse = 2;   // staged levels: the last two (levels 2, 3 of 4)
constexpr int kFine = kMaxLevels - kCoarse;

struct StagedArgs {
  int64_t n_rows;  // rows per batch item
  int32_t C, bs, Q, P, cams, G, cpg;
  const int32_t* shape;  // [cams, 4, 2]
  const int64_t* start;  // [cams, 4]
  const float* loc;      // [bs, Q, P, cams, 2]
  const float* w;        // [bs, Q, P, cams, 4, G]
  float* out;            // [bs, Q, C], zeroed
  float* wsum;           // [bs, Q, G], zeroed, or null
  const float2* proj_cell;  // fused projection: cells [bs, Q, P, cams, 4] (NaN: behind the camera), or null
  int32_t n_slices, n_chunks, chunk;  // slices per row, anchor chunks, anchors per chunk
  int64_t n_items;
  int32_t zero_off;  // byte offset of the 128-B zero row (the stage area [0, kStageBudget) precedes it)
  int32_t bar_off;   // byte offset of the stage mbarrier
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int r0, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// T: storage type; HACC: half2 products/partials (f16 only).
// A lane owns LB = 32 bytes of the 128-B row slice (two 16-B chunks), so a
// row is 4 lanes and a warp's 8 groups take 8 samples per step: the record
// work per sample is shared by 4 lanes, not 8.  The two chunk loads of odd
// groups are issued in swapped order, which keeps every quarter-warp phase of
// an LDS.128 on 32 distinct banks.
template <typename T, bool HACC, bool PROJ>
__global__ void __launch_bounds__(kStThreads, 1)
    staged_coarse_kernel(const __grid_constant__ CUtensorMap tmap, const StagedArgs a) {
  constexpr int LB = 32;                               // bytes per lane
  constexpr int NC = LB / 16;                          // 16-B chunks per lane
  constexpr int LPR = kSliceBytes / LB;                // lanes per row slice
  constexpr int NG = 32 / LPR;                         // sample groups per warp
  constexpr int VEC = LB / (int)sizeof(T);             // elements per lane
  constexpr int SLICE = kSliceBytes / (int)sizeof(T);  // elements per slice
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LPR, li = lane % LPR;  // keypoint group, lane within the row slice
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + a.bar_off;
  const uint32_t lane_off = li * LB + (grp & 1) * 16;  // first chunk this lane loads (second: xor 16)
  const uint32_t zero_row = sbase + a.zero_off + lane_off;
  if (threadIdx.x < kSliceBytes / 4) reinterpret_cast<uint32_t*>(smem + a.zero_off)[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint32_t parity = 0;
  for (int64_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    // camera-major: consecutive items share a camera (then batch item)
    int64_t r = item;
    const int chunk = (int)(r % a.n_chunks);
    r /= a.n_chunks;
    const int slice = (int)(r % a.n_slices);
    r /= a.n_slices;
    const int b = (int)(r % a.bs);
    const int cam = (int)(r / a.bs);
    const int64_t row_base = (int64_t)b * a.n_rows;
    __syncthreads();  // every warp is done with the previous item's staged rows
    if (threadIdx.x == 0) {  // the coarse levels' row slices, coarsest first, each padded to whole boxes
      uint32_t bytes = 0;
      for (int l = kFine; l < kMaxLevels; ++l) {
        const int rows = a.shape[2 * (cam * kMaxLevels + l)] * a.shape[2 * (cam * kMaxLevels + l) + 1];
        bytes += (rows + kBoxRows - 1) / kBoxRows * kBoxRows * kSliceBytes;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, bytes);
      uint32_t off = 0;
      for (int l = kMaxLevels - 1; l >= kFine; --l) {
        const int rows = a.shape[2 * (cam * kMaxLevels + l)] * a.shape[2 * (cam * kMaxLevels + l) + 1];
        const int64_t r0 = row_base + a.start[cam * kMaxLevels + l];
        for (int k = 0; k * kBoxRows < rows; ++k, off += kBoxRows * kSliceBytes)
          tma_load_2d(sbase + off, &tmap, slice * SLICE, (int)(r0 + k * kBoxRows), bar);
      }
    }
    // per-level constants of this camera (coarse level kFine + k, staged coarsest first)
    int lW[kCoarse], lH[kCoarse];
    uint32_t lbase[kCoarse];
    {
      uint32_t off = 0;
#pragma unroll
      for (int k = kCoarse - 1; k >= 0; --k) {
        lH[k] = a.shape[2 * (cam * kMaxLevels + kFine + k)];
        lW[k] = a.shape[2 * (cam * kMaxLevels + kFine + k) + 1];
        lbase[k] = sbase + off + lane_off;
        off += (lH[k] * lW[k] + kBoxRows - 1) / kBoxRows * kBoxRows * kSliceBytes;
      }
    }
    const int c_lane = slice * SLICE + li * VEC;  // first channel of this lane
    const int g_lane = c_lane / a.cpg;
    const int q0 = chunk * a.chunk;
    const int n_anchor = max(0, min(a.chunk, a.Q - q0));
    mbar_wait(bar, parity);
    parity ^= 1u;

    // a warp takes blocks of NG anchors; group g walks anchor q0 + NG * blk + g
    // through its P keypoints x the coarse levels (all groups in lockstep), so
    // no cross-group reduction is needed
    const int n_blocks = (n_anchor + NG - 1) / NG;
    for (int blk = warp; blk < n_blocks; blk += kStWarps) {
      const int qi = blk * NG + grp;
      const bool valid = qi < n_anchor;
      const int64_t bq = (int64_t)b * a.Q + q0 + (valid ? qi : 0);
      const int64_t pc0 = bq * a.P * a.cams + cam;  // (bq, p = 0, cam); p adds a.cams
      // locations (or, fused projection, the pre-pass's cells of the coarse
      // levels) and weights of keypoints p and p + 1 in flight (two buffers)
      float2 bl[2][PROJ ? kCoarse : 1];
      float bw[2][kCoarse];
      auto load_pt = [&](int p, int k2) {
        const int64_t pc = pc0 + (int64_t)min(p, a.P - 1) * a.cams;
        if constexpr (PROJ) {
#pragma unroll
          for (int k = 0; k < kCoarse; ++k) bl[k2][k] = __ldg(a.proj_cell + pc * kMaxLevels + kFine + k);
        } else {
          bl[k2][0] = __ldg(reinterpret_cast<const float2*>(a.loc) + pc);
        }
#pragma unroll
        for (int k = 0; k < kCoarse; ++k) bw[k2][k] = __ldg(a.w + (pc * kMaxLevels + kFine + k) * a.G + g_lane);
      };
      load_pt(0, 0);
      load_pt(1, 1);
      float acc[VEC];
      __half2 hacc[HACC ? VEC / 2 : 1];
      float wacc = 0.0f;
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;
#pragma unroll
      for (int e = 0; e < (HACC ? VEC / 2 : 1); ++e) hacc[e] = __float2half2_rn(0.0f);
      for (int p0 = 0; p0 < a.P; p0 += 2) {
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          if (p0 + k2 >= a.P) break;
          float2 lp[PROJ ? kCoarse : 1];
          float wl[kCoarse];
#pragma unroll
          for (int k = 0; k < (PROJ ? kCoarse : 1); ++k) lp[k] = bl[k2][k];
#pragma unroll
          for (int k = 0; k < kCoarse; ++k) wl[k] = bw[k2][k];
          load_pt(p0 + k2 + 2, k2);  // keypoint p + 2 into this buffer (clamped past P)
#pragma unroll
          for (int l = kCoarse - 1; l >= 0; --l) {
            const int W = lW[l], H = lH[l];
            float u, v, wg = wl[l];
            if constexpr (PROJ) {  // cell = f32(pixel / stride - 0.5) from the pre-pass; NaN: behind, out of the plan
              const bool ok = !isnan(lp[l].x);
              u = ok ? lp[l].x : -4.0f;
              v = ok ? lp[l].y : -4.0f;
              wg = ok ? wg : 0.0f;
            } else {  // cell = loc * W - 0.5 (features.py:20-24)
              u = __fsub_rn(__fmul_rn(lp[0].x, (float)W), 0.5f);
              v = __fsub_rn(__fmul_rn(lp[0].y, (float)H), 0.5f);
            }
            const float uc = fminf(fmaxf(u, -2.0f), (float)W + 1.0f);  // keeps the integer conversion in range
            const float vc = fminf(fmaxf(v, -2.0f), (float)H + 1.0f);
            const float x0f = floorf(uc), y0f = floorf(vc);
            const float fu = uc - x0f, fv = vc - y0f;
            const int x0 = (int)x0f, y0 = (int)y0f;
            const bool vx0 = (unsigned)x0 < (unsigned)W, vx1 = (unsigned)(x0 + 1) < (unsigned)W;
            const bool vy0 = (unsigned)y0 < (unsigned)H, vy1 = (unsigned)(y0 + 1) < (unsigned)H;
            const uint32_t rb = lbase[l] + (uint32_t)(y0 * W + x0) * kSliceBytes;
            const uint32_t addr[4] = {vx0 && vy0 ? rb : zero_row, vx1 && vy0 ? rb + kSliceBytes : zero_row,
                                      vx0 && vy1 ? rb + W * kSliceBytes : zero_row,
                                      vx1 && vy1 ? rb + (W + 1) * kSliceBytes : zero_row};
            const float omu = 1.0f - fu, omv = 1.0f - fv;
            const float c[4] = {omu * omv * wg, fu * omv * wg, omu * fv * wg, fu * fv * wg};
            wacc += wg;
            uint4 cv[4][NC];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int h = 0; h < NC; ++h)
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(cv[k][h].x), "=r"(cv[k][h].y), "=r"(cv[k][h].z), "=r"(cv[k][h].w)
                             : "r"(addr[k] ^ (uint32_t)(h * 16)));
            // accumulate in load order: chunk h of an odd group's lane holds
            // the lane's elements of chunk h ^ 1 (swapped back at the end)
            constexpr int CV = 16 / (int)sizeof(T);  // elements per chunk
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
              for (int h = 0; h < NC; ++h) {
                if constexpr (HACC) {
                  const __half2 cwh = __float2half2_rn(c[k]);
                  const __half2* hv = reinterpret_cast<const __half2*>(&cv[k][h]);
#pragma unroll
                  for (int e = 0; e < CV / 2; ++e) hacc[h * CV / 2 + e] = __hfma2(hv[e], cwh, hacc[h * CV / 2 + e]);
                } else {
                  float f[CV];
                  raw_to_f32<T, CV>(reinterpret_cast<const uint32_t*>(&cv[k][h]), f);
                  const float2 cw2 = make_float2(c[k], c[k]);
#pragma unroll
                  for (int e = 0; e < CV; e += 2) {
                    const float2 r2 = __ffma2_rn(make_float2(f[e], f[e + 1]), cw2,
                                                 make_float2(acc[h * CV + e], acc[h * CV + e + 1]));
                    acc[h * CV + e] = r2.x;
                    acc[h * CV + e + 1] = r2.y;
                  }
                }
              }
            }
          }
        }
      }
      if constexpr (HACC) {
#pragma unroll
        for (int e = 0; e < VEC / 2; ++e) {
          const float2 f2 = __half22float2(hacc[e]);
          acc[2 * e] = f2.x;
          acc[2 * e + 1] = f2.y;
        }
      }
      if (grp & 1) {  // back to element order
#pragma unroll
        for (int e = 0; e < VEC / 2; ++e) {
          const float t = acc[e];
          acc[e] = acc[VEC / 2 + e];
          acc[VEC / 2 + e] = t;
        }
      }
      if (valid) {  // this anchor's slice partial over the camera's coarse levels
        float* o = a.out + bq * a.C + c_lane;
#pragma unroll
        for (int e = 0; e < VEC; e += 4) red_add_v4(o + e, acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
        if (a.wsum && (c_lane % a.cpg) == 0) atomicAdd(a.wsum + bq * a.G + g_lane, wacc);
      }
    }
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiled>(nullptr);
    }
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

template <typename T, bool HACC, bool PROJ>
cudaError_t launch_coarse_p(const CUtensorMap& map, const StagedArgs& a, size_t smem, cudaStream_t s) {
  static std::atomic<bool> attr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
    const cudaError_t e =
        cudaFuncSetAttribute(staged_coarse_kernel<T, HACC, PROJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_release);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(a.n_items, sms);
  staged_coarse_kernel<T, HACC, PROJ><<<(unsigned)grid, kStThreads, smem, s>>>(map, a);
  return cudaGetLastError();
}

template <typename T, bool HACC>
cudaError_t launch_coarse_t(const CUtensorMap& map, const StagedArgs& a, size_t smem, cudaStream_t s) {
  return a.proj_cell ? launch_coarse_p<T, HACC, true>(map, a, smem, s) : launch_coarse_p<T, HACC, false>(map, a, smem, s);
}

}  // namespace

int dense_staged_fine_levels(const msda_features_t& f, int G, int P) {
  // f32 too: 128-B slices of 32 channels (cfg1 f32 FAST 94 -> 86 us once the
  // anchor chunks are whole warp blocks; it measured 108 us with ragged ones)
  const int esz = f.dtype == MSDA_F32 ? 4 : 2;
  const int C = f.channels;
  if (f.n_levels != kMaxLevels || !f.spatial_shape_host || P < 1 || G < 1 || C % G ||
      (C * esz) % kSliceBytes || (C / G) % (32 / esz))
    return -1;
  // the fine levels' gather takes whole 16-B-lane warps over a row, each lane in one group
  if (C % (32 * (16 / esz)) || (C / G) % (16 / esz)) return -1;
  if (reinterpret_cast<uintptr_t>(f.data) % 16 || (int64_t)f.batch * f.n_rows >= (int64_t(1) << 31)) return -1;
  if (!encode_fn()) return -1;
  // the coarsest levels whose 128-B row slices (padded to whole TMA boxes)
  // fit the stage budget, the same for every camera
  int n_fine = -1;
  for (int c = 0; c < f.n_cams; ++c) {
    int64_t off = 0;
    int nf = kMaxLevels;
    for (int l = kMaxLevels - 1; l >= 0; --l) {
      const int64_t rows =
          (int64_t)f.spatial_shape_host[2 * (c * kMaxLevels + l)] * f.spatial_shape_host[2 * (c * kMaxLevels + l) + 1];
      const int64_t bytes = (rows + kBoxRows - 1) / kBoxRows * kBoxRows * kSliceBytes;
      if (off + bytes > kStageBudget) break;
      off += bytes;
      nf = l;
    }
    if (c > 0 && nf != n_fine) return -1;
    n_fine = nf;
  }
  // the kernel stages exactly the last two levels (a level-3+2 budget that
  // also fits level 1 would still leave it to the gather)
  return n_fine <= kFine ? kFine : -1;
}

cudaError_t launch_dense_coarse(const msda_features_t& f, const DenseFastSpec& d, int n_fine, float* out,
                                float* wsum, cudaStream_t stream) {
  const int esz = f.dtype == MSDA_F32 ? 4 : 2;
  const int C = f.channels;
  const int slice_elems = kSliceBytes / esz;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {(cuuint64_t)C, (cuuint64_t)((int64_t)f.batch * f.n_rows)};
  const cuuint64_t gstride[1] = {(cuuint64_t)C * esz};
  const cuuint32_t box[2] = {(cuuint32_t)slice_elems, (cuuint32_t)kBoxRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = f.dtype == MSDA_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : f.dtype == MSDA_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (encode_fn()(&map, dt, 2, const_cast<void*>(f.data), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  StagedArgs a{};
  a.n_rows = f.n_rows;
  a.C = C;
  a.bs = f.batch;
  a.Q = d.Q;
  a.P = d.P;
  a.cams = f.n_cams;
  a.G = d.G;
  a.cpg = C / d.G;
  (void)n_fine;
  a.shape = f.spatial_shape;
  a.start = f.scale_start_index;
  a.loc = d.loc;
  a.w = d.w;
  a.proj_cell = d.proj_cell;
  a.out = out;
  a.wsum = wsum;
  a.n_slices = C / slice_elems;
  // anchor chunks: every warp of an item takes whole 8-anchor blocks, so a
  // chunk is a multiple of kStWarps x 8 anchors (65-anchor chunks at cfg1 ran
  // 9 blocks on 8 warps: a lone second round per item); among those, the
  // fewest rounds of (block rounds per item + a staging) over the SMs
  const int64_t pairs = (int64_t)f.batch * f.n_cams * a.n_slices;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int kBlockAnchors = kStWarps * 8;
  double best = 1e30;
  a.chunk = kBlockAnchors;
  for (int c = kBlockAnchors;; c += kBlockAnchors) {
    const int64_t items = pairs * ((d.Q + c - 1) / c);
    // (staging weight 0.5 / 1 / 2 measured alike; 0.25 picks smaller chunks, cfg3 375 vs 369 us)
    const double cost = (double)((items + sms - 1) / sms) * ((c / kBlockAnchors) + 0.5);
    if (cost < best - 1e-9) {
      best = cost;
      a.chunk = c;
    }
    if (c >= d.Q) break;
  }
  a.n_chunks = (d.Q + a.chunk - 1) / a.chunk;
  a.n_items = pairs * a.n_chunks;
  a.zero_off = kStageBudget;
  a.bar_off = a.zero_off + kSliceBytes;
  const size_t smem = (size_t)a.bar_off + 16;
  if (d.Q == 0) return cudaSuccess;
  switch (f.dtype) {
    case MSDA_F16:
      return d.h2 ? launch_coarse_t<__half, true>(map, a, smem, stream)
                  : launch_coarse_t<__half, false>(map, a, smem, stream);
    case MSDA_BF16: return launch_coarse_t<__nv_bfloat16, false>(map, a, smem, stream);
    case MSDA_F32: return launch_coarse_t<float, false>(map, a, smem, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace msda
