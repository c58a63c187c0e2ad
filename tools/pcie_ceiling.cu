// Host->device ceilings on this box for the e2e path (msda_csr_host).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_ceiling tools/pcie_ceiling.cu
//   ./tools/pcie_ceiling
//
// The e2e leg of bench.py moves ~1.22 GB per call from pinned host memory:
// whole grids by copy engine (cudaMemcpyAsync) and touched 1 KB rows of the
// sparse grids by device warps reading the pinned buffer through UVA
// (fetch_rows_kernel).  This measures, on 1 GiB of pinned memory:
//   memcpy_h2d      : one cudaMemcpyAsync (copy engine)
//   memcpy_d2h      : the reverse
//   zc_seq_rowN     : warp-per-row zero-copy reads, rows in order, N KB rows
//   zc_rand_1k      : warp-per-row zero-copy reads of 1 KB rows in hashed order
//   zc_rand_1k_x2   : the same with two rows in flight per warp
//   bulk_*          : one cp.async.bulk (TMA bulk copy) per row into shared, then stored
//   memcpy+zc       : memcpy of half on one stream, zero-copy of the other half on another
// Result on this pool's B200s (profiles/r1/pcie_ceiling.txt): copy engine
// 55.6 GB/s; every SM-side read (any row size, order, in-flight depth, LDG or
// bulk) 51.5 GB/s; both at once 53.4 GB/s.
// Prints GB/s (best of 5, CUDA events).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// warp per row (row_bytes multiple of 512), rows [0, n) in order or permuted
// by an odd multiplier mod n (n a power of two) so consecutive warps hit
// scattered host pages; `inflight` rows per warp iteration
template <int INFLIGHT>
__global__ void __launch_bounds__(256) zc_rows(const char* __restrict__ src, char* __restrict__ dst, int64_t n,
                                               int row_bytes, int permute) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t i = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * INFLIGHT; i < n; i += warps * INFLIGHT) {
    uint4 buf[INFLIGHT][2];
    int64_t rows[INFLIGHT];
#pragma unroll
    for (int k = 0; k < INFLIGHT; ++k) {
      const int64_t j = i + k < n ? i + k : n - 1;
      rows[k] = permute ? (int64_t)((uint64_t)(j * 2654435761ull + hash((uint32_t)permute)) & (uint64_t)(n - 1)) : j;
    }
    for (int off = lane * 16; off < row_bytes; off += 1024) {
#pragma unroll
      for (int k = 0; k < INFLIGHT; ++k) {
        buf[k][0] = *reinterpret_cast<const uint4*>(src + rows[k] * row_bytes + off);
        buf[k][1] = off + 512 < row_bytes ? *reinterpret_cast<const uint4*>(src + rows[k] * row_bytes + off + 512)
                                          : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < INFLIGHT; ++k) {
        if (i + k >= n) break;
        *reinterpret_cast<uint4*>(dst + rows[k] * row_bytes + off) = buf[k][0];
        if (off + 512 < row_bytes) *reinterpret_cast<uint4*>(dst + rows[k] * row_bytes + off + 512) = buf[k][1];
      }
    }
  }
}

// one elected thread per warp pulls a whole row host -> shared with one
// cp.async.bulk (TMA bulk copy, mbarrier completion), then the warp stores it
// to the device table: does the bulk engine issue larger PCIe reads than LDG?
__global__ void __launch_bounds__(256) zc_bulk(const char* __restrict__ src, char* __restrict__ dst, int64_t n,
                                               int row_bytes, int permute) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  char* buf = smem + wid * row_bytes;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[wid]);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf);
  if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  uint32_t phase = 0;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t i = (int64_t)blockIdx.x * 8 + wid; i < n; i += warps) {
    const int64_t row = permute ? (int64_t)((uint64_t)(i * 2654435761ull + hash((uint32_t)permute)) & (uint64_t)(n - 1)) : i;
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(row_bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sb), "l"(src + row * row_bytes), "r"(row_bytes), "r"(b) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(b), "r"(phase) : "memory");
    phase ^= 1;
    for (int off = lane * 16; off < row_bytes; off += 512)
      *reinterpret_cast<uint4*>(dst + row * row_bytes + off) = *reinterpret_cast<const uint4*>(buf + off);
    __syncwarp();
  }
}

int main() {
  const size_t bytes = size_t(1) << 30;
  char *h = nullptr, *d = nullptr, *hdev = nullptr;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)i;
  CK(cudaHostGetDevicePointer(&hdev, h, 0));
  CK(cudaMalloc(&d, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, j1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&j1));
  auto timeit = [&](auto&& body, double gb) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0, s0);
      body();
      cudaEventRecord(e1, s0);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    return gb / (best * 1e-3);
  };
  const double gb = bytes / 1e9;
  const unsigned grid = sms * 16;
  printf("memcpy_h2d      %8.1f GB/s\n", timeit([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s0); }, gb));
  printf("memcpy_d2h      %8.1f GB/s\n", timeit([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s0); }, gb));
  for (int rb : {512, 1024, 4096}) {
    const int64_t n = bytes / rb;
    printf("zc_seq_row%-5d %8.1f GB/s\n", rb,
           timeit([&] { zc_rows<1><<<grid, 256, 0, s0>>>(hdev, d, n, rb, 0); }, gb));
  }
  const int64_t n1k = bytes / 1024;
  printf("zc_rand_1k      %8.1f GB/s\n", timeit([&] { zc_rows<1><<<grid, 256, 0, s0>>>(hdev, d, n1k, 1024, 7); }, gb));
  printf("zc_rand_1k_x2   %8.1f GB/s\n", timeit([&] { zc_rows<2><<<grid, 256, 0, s0>>>(hdev, d, n1k, 1024, 7); }, gb));
  printf("zc_rand_1k_g4   %8.1f GB/s  (4 CTAs per SM)\n",
         timeit([&] { zc_rows<1><<<sms * 4, 256, 0, s0>>>(hdev, d, n1k, 1024, 7); }, gb));
  CK(cudaFuncSetAttribute(zc_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
  printf("bulk_rand_1k    %8.1f GB/s\n",
         timeit([&] { zc_bulk<<<grid / 2, 256, 8 * 1024, s0>>>(hdev, d, n1k, 1024, 7); }, gb));
  printf("bulk_seq_4k     %8.1f GB/s\n",
         timeit([&] { zc_bulk<<<sms * 4, 256, 8 * 4096, s0>>>(hdev, d, bytes / 4096, 4096, 0); }, gb));
  CK(cudaGetLastError());
  printf("memcpy+zc       %8.1f GB/s\n", timeit([&] {
           cudaEventRecord(j1, s0);
           cudaStreamWaitEvent(s1, j1, 0);
           cudaMemcpyAsync(d, h, bytes / 2, cudaMemcpyHostToDevice, s1);
           zc_rows<1><<<grid, 256, 0, s0>>>(hdev + bytes / 2, d + bytes / 2, n1k / 2, 1024, 0);
           cudaEventRecord(j1, s1);
           cudaStreamWaitEvent(s0, j1, 0);
         }, gb));
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
