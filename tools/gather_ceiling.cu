// Gather-bandwidth ceilings on this B200 for the cfg2 access pattern.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_ceiling tools/gather_ceiling.cu
//   ./tools/gather_ceiling
//
// Table: cfg2 geometry (16 cams x 4 levels, 270x480 .. 33x60, C=256 f32,
// 2.82 GB).  Samples: 900 queries x 16 cams x 4 levels x 13 points, cell
// coordinates uniform like the reference bench generator, visited per query in
// (camera, level) order — the same rows, order and concurrency as the exact
// gather, but with no arithmetic beyond one add per loaded word:
//   stream      : sequential read of the whole table (copy-style ceiling)
//   corners_ldg : warp per (query, 128 ch), 4 corner rows per sample, LDG.128,
//                 U samples unrolled
// Prints GB/s for the unique touched bytes and for the bytes moved.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

struct Geo { int H[4], W[4]; long long start[16][4]; };

__global__ void make_rows(Geo g, int Q, int P, int4* rows) {
  long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long S = (long long)Q * 16 * 4 * P;
  if (s >= S) return;
  int p = s % P, l = (s / P) % 4, c = (s / (P * 4)) % 16;
  uint32_t h1 = hash((uint32_t)s * 2 + 1), h2 = hash((uint32_t)s * 2 + 2);
  float u = -1.0f + (g.W[l] + 1.0f) * (h1 * (1.0f / 4294967296.0f));
  float v = -1.0f + (g.H[l] + 1.0f) * (h2 * (1.0f / 4294967296.0f));
  int x0 = (int)floorf(u), y0 = (int)floorf(v);
  int r[4];
  for (int k = 0; k < 4; ++k) {
    int x = x0 + (k & 1), y = y0 + (k >> 1);
    r[k] = (x >= 0 && x < g.W[l] && y >= 0 && y < g.H[l]) ? (int)(g.start[c][l] + (long long)y * g.W[l] + x) : -1;
  }
  rows[s] = make_int4(r[0], r[1], r[2], r[3]);
  (void)p;
}

__global__ void stream_read(const float4* __restrict__ t, long long n, float* out) {
  float acc = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(t + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int U>
__global__ void corners_ldg(const float4* __restrict__ t, const int4* __restrict__ rows, int per_q, int Q, float* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int q = warp >> 1;
  if (q >= Q) return;
  const int half = warp & 1;
  const float4* base = t + half * 32 + lane;  // 64 float4 per 1 KB row
  const int4* rq = rows + (long long)q * per_q;
  float acc = 0.f;
  for (int i = 0; i < per_q; i += U) {
    float4 v[U][4];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int4 r = rq[min(i + j, per_q - 1)];
      const int rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) v[j][k] = rr[k] >= 0 ? __ldg(base + (long long)rr[k] * 64) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += v[j][k].x + v[j][k].y + v[j][k].z + v[j][k].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// The production exact-gather structure (1-warp CTAs, cp.async zero-fill
// ring of D samples x 4 corner rows per lane) with MATH = 0: one add per word,
// MATH = 1: the 9 separately rounded FFMA2 ops per channel pair of the exact
// kernel (1.0 / -0.0 operands from parameters).
template <int D, int MATH>
__global__ void __launch_bounds__(32) corners_pipe(const float4* __restrict__ t, const int4* __restrict__ rows,
                                                   int per_q, int Q, float2 one2, float2 nz2, float* out) {
  __shared__ __align__(16) float4 ring[D][4][32];
  const int lane = threadIdx.x;
  const int q = blockIdx.x >> 1, half = blockIdx.x & 1;
  if (q >= Q) return;
  const char* base = reinterpret_cast<const char*>(t + half * 32 + lane);
  const int4* rq = rows + (long long)q * per_q;
  auto issue = [&](int k, int slot) {
    const int4 r = rq[k];
    const int rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[slot][c][lane]);
      const char* src = base + (size_t)max(rr[c], 0) * 1024;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(rr[c] >= 0 ? 16 : 0));
    }
  };
  for (int k = 0; k < D; ++k) {
    if (k < per_q) issue(k, k);
    asm volatile("cp.async.commit_group;");
  }
  float acc[4] = {0, 0, 0, 0};
  int slot = 0;
  for (int i = 0; i < per_q; ++i) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1));
    float4 c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = ring[slot][k][lane];
    if (MATH) {
      const float w = 0.25f, wn = 0.001f;
      const float2 w2 = make_float2(w, w), ws = make_float2(wn, wn);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float2 x0 = e ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y);
        const float2 x1 = e ? make_float2(c[1].z, c[1].w) : make_float2(c[1].x, c[1].y);
        const float2 x2 = e ? make_float2(c[2].z, c[2].w) : make_float2(c[2].x, c[2].y);
        const float2 x3 = e ? make_float2(c[3].z, c[3].w) : make_float2(c[3].x, c[3].y);
        const float2 a = __ffma2_rn(x0, w2, nz2), b = __ffma2_rn(x1, w2, nz2);
        const float2 d = __ffma2_rn(x2, w2, nz2), f = __ffma2_rn(x3, w2, nz2);
        const float2 tt = __ffma2_rn(__ffma2_rn(a, one2, b), one2, __ffma2_rn(d, one2, f));
        const float2 r = __ffma2_rn(__ffma2_rn(tt, ws, nz2), one2, make_float2(acc[2 * e], acc[2 * e + 1]));
        acc[2 * e] = r.x;
        acc[2 * e + 1] = r.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[0] += c[k].x + c[k].y + c[k].z + c[k].w;
    }
    if (i + D < per_q) issue(i + D, slot);
    asm volatile("cp.async.commit_group;");
    slot = slot + 1 == D ? 0 : slot + 1;
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 12345.f) out[0] = acc[0];
}

int main() {
  Geo g{};
  const int H[4] = {270, 135, 67, 33}, W[4] = {480, 240, 120, 60};
  long long r = 0;
  for (int c = 0; c < 16; ++c)
    for (int l = 0; l < 4; ++l) {
      g.H[l] = H[l]; g.W[l] = W[l]; g.start[c][l] = r; r += (long long)H[l] * W[l];
    }
  const long long rows = r, C = 256;
  const int Q = 900, P = 13, per_q = 16 * 4 * P;
  const long long S = (long long)Q * per_q;
  float4* table; int4* rws; float* out;
  CK(cudaMalloc(&table, rows * C * 4));
  CK(cudaMemset(table, 0, rows * C * 4));
  CK(cudaMalloc(&rws, S * sizeof(int4)));
  CK(cudaMalloc(&out, 4));
  make_rows<<<(S + 255) / 256, 256>>>(g, Q, P, rws);
  CK(cudaDeviceSynchronize());
  std::vector<int4> h(S);
  CK(cudaMemcpy(h.data(), rws, S * sizeof(int4), cudaMemcpyDeviceToHost));
  std::vector<char> seen(rows, 0);
  long long touched = 0, moved = 0;
  for (auto& x : h) for (int v : {x.x, x.y, x.z, x.w}) if (v >= 0) { moved++; if (!seen[v]) { seen[v] = 1; touched++; } }
  printf("rows %lld, touched %lld (%.1f%%), moved rows %lld, unique %.3f GB, moved %.3f GB\n", rows, touched,
         100.0 * touched / rows, moved, touched * 1024.0 / 1e9, moved * 1024.0 / 1e9);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch, double bytes, double moved_bytes) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("%-14s %8.1f us  unique %7.1f GB/s  moved %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           moved_bytes / (ms * 1e-3) / 1e9);
  };
  const double tb = rows * C * 4.0;
  timeit("stream", [&] { stream_read<<<148 * 16, 256>>>(table, rows * C / 4, out); }, tb, tb);
  const double ub = touched * 1024.0, mb = moved * 1024.0;
  timeit("corners_u2", [&] { corners_ldg<2><<<(Q * 2 * 32 + 63) / 64, 64>>>(table, rws, per_q, Q, out); }, ub, mb);
  timeit("corners_u4", [&] { corners_ldg<4><<<(Q * 2 * 32 + 63) / 64, 64>>>(table, rws, per_q, Q, out); }, ub, mb);
  timeit("corners_u8", [&] { corners_ldg<8><<<(Q * 2 * 32 + 63) / 64, 64>>>(table, rws, per_q, Q, out); }, ub, mb);
  const float2 one2 = make_float2(1.f, 1.f), nz2 = make_float2(-0.f, -0.f);
  timeit("pipe_d4", [&] { corners_pipe<4, 0><<<Q * 2, 32>>>(table, rws, per_q, Q, one2, nz2, out); }, ub, mb);
  timeit("pipe_d7", [&] { corners_pipe<7, 0><<<Q * 2, 32>>>(table, rws, per_q, Q, one2, nz2, out); }, ub, mb);
  timeit("pipe_d12", [&] { corners_pipe<12, 0><<<Q * 2, 32>>>(table, rws, per_q, Q, one2, nz2, out); }, ub, mb);
  timeit("pipe_d7_math", [&] { corners_pipe<7, 1><<<Q * 2, 32>>>(table, rws, per_q, Q, one2, nz2, out); }, ub, mb);
  timeit("pipe_d12_math", [&] { corners_pipe<12, 1><<<Q * 2, 32>>>(table, rws, per_q, Q, one2, nz2, out); }, ub, mb);
  return 0;
}
