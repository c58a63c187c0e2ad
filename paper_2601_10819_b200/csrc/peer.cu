// Camera-sharded partial-sum all-reduce over peer memory — sm_100a.
//
// one scene's cameras split across ranks; every rank holds the
// un-normalised numerators [rows, C] and per-(anchor, group) weight sums
// [rows, G] of its cameras, and every rank needs the normalised sum.  Instead
// of an NCCL all-reduce followed by a separate normalising launch, each rank
// pushes its partial straight into every peer's accumulation buffer over
// NVLink (float4 `red.global.add` through CUDA-IPC mappings), signals with a
// system-scope release counter, and one kernel per rank waits for every
// rank's signal and writes the normalised result (the zero-sum check of
// features.py:268-269 included).
//
// Symmetric buffer (one per rank, cudaMalloc'd by msda_peer_alloc so that its
// IPC handle maps the whole allocation): two halves, used by alternate
// epochs, each [rows * C] numerators | [rows * G] weight sums | arrival
// counter.  Epoch e (identical on every rank) uses half b = e & 1:
//   1. zero half b ^ 1 (the previous epoch's, already consumed here);
//   2. exchange: add the local partial into half b of every rank, then, per
//      CTA, fence.sys + one release increment of every rank's counter;
//   3. wait until this rank's counter reaches world x (exchange CTAs), then
//      out = num / wsum per group.
// A peer can only reach epoch e + 1 (and touch half b ^ 1 here) after its
// step 3 saw this rank's epoch-e signal, which stream order places after
// this rank's step 1 — so no add lands in a half before it is zeroed and no
// half is zeroed while a peer may still add to it.  The wait is bounded: a
// missing peer reports MSDA_CUDA_ERROR instead of hanging the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "msda_common.cuh"

namespace msda {
namespace {

constexpr int kMaxPeers = 8;
constexpr int kExchangeThreads = 256;

struct PeerLayout {
  size_t num_floats, wsum_floats, half_bytes;  // per half
  size_t wsum_off, flag_off;                   // byte offsets inside a half
};

PeerLayout peer_layout(int64_t rows, int32_t channels, int32_t groups) {
  PeerLayout l;
  l.num_floats = (size_t)rows * channels;
  l.wsum_floats = (size_t)rows * groups;
  l.wsum_off = align_up(l.num_floats * 4, 256);
  l.flag_off = l.wsum_off + align_up(l.wsum_floats * 4, 256);
  l.half_bytes = l.flag_off + 256;
  return l;
}

struct ExchangeArgs {
  const float* num;   // local partial numerators [rows * C]
  const float* wsum;  // local partial weight sums [rows * G] (or null)
  char* peer_half[kMaxPeers];  // half b of every rank's buffer (own included)
  int32_t world;
  int64_t num4;       // rows * C / 4
  int64_t wsum_n;     // rows * G
  size_t wsum_off, flag_off;
};

__global__ void __launch_bounds__(kExchangeThreads) peer_exchange_kernel(ExchangeArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float4* src4 = reinterpret_cast<const float4*>(a.num);
  for (int64_t i = t0; i < a.num4; i += stride) {
    const float4 v = src4[i];
    for (int p = 0; p < a.world; ++p) atomicAdd(reinterpret_cast<float4*>(a.peer_half[p]) + i, v);
  }
  if (a.wsum) {
    for (int64_t i = t0; i < a.wsum_n; i += stride) {
      const float v = a.wsum[i];
      for (int p = 0; p < a.world; ++p) atomicAdd(reinterpret_cast<float*>(a.peer_half[p] + a.wsum_off) + i, v);
    }
  }
  __threadfence_system();  // every thread's adds are performed system-wide ...
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // ... before the CTA's signal
    for (int p = 0; p < a.world; ++p) {
      uint32_t* flag = reinterpret_cast<uint32_t*>(a.peer_half[p] + a.flag_off);
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
    }
  }
}

struct FinishArgs {
  const char* half;  // this rank's half b
  size_t wsum_off, flag_off;
  uint32_t expected;  // world x exchange CTAs
  int64_t rows;
  int32_t C, G, normalize;
  float* out;       // [rows, C]
  float* wsum_out;  // [rows, G] or null
  DevStatus* status;
};

__global__ void __launch_bounds__(256) peer_finish_kernel(FinishArgs a) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const uint32_t* flag = reinterpret_cast<const uint32_t*>(a.half + a.flag_off);
    const long long t0 = clock64();
    uint32_t v = 0;
    int ok = 1;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v >= a.expected) break;
      if (clock64() - t0 > (1ll << 33)) {  // ~4 s: a rank never arrived
        set_status(a.status, MSDA_CUDA_ERROR, -1);
        ok = 0;
        break;
      }
      __nanosleep(256);
    }
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  const float* num = reinterpret_cast<const float*>(a.half);
  const float* ws = reinterpret_cast<const float*>(a.half + a.wsum_off);
  const int cpg = a.C / a.G;
  const int64_t total = a.rows * a.C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / a.C;
    const int g = (int)(i - r * a.C) / cpg;
    const float s = __ldcg(ws + r * a.G + g);
    float v = __ldcg(num + i);
    if (a.normalize) {
      if (s == 0.0f) set_status(a.status, MSDA_ZERO_WEIGHT_SUM, r);
      v = v / s;
    }
    a.out[i] = v;
    if (a.wsum_out && (i - r * a.C) % cpg == 0) a.wsum_out[r * a.G + g] = s;
  }
}

}  // namespace
}  // namespace msda

using namespace msda;

extern "C" {

size_t msda_peer_buffer_size(int64_t rows, int32_t channels, int32_t groups) {
  if (rows < 0 || channels <= 0 || groups <= 0) return 0;
  return 2 * peer_layout(rows, channels, groups).half_bytes;
}

int32_t msda_peer_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return MSDA_BAD_ARG;
  *ptr = nullptr;
  if (cudaMalloc(ptr, bytes) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (cudaMemset(*ptr, 0, bytes) != cudaSuccess) return MSDA_CUDA_ERROR;
  return MSDA_OK;
}

int32_t msda_peer_free(void* ptr) {
  if (ptr && cudaFree(ptr) != cudaSuccess) return MSDA_CUDA_ERROR;
  return MSDA_OK;
}

int32_t msda_ipc_handle(const void* ptr, void* handle /* MSDA_IPC_HANDLE_BYTES */) {
  if (!ptr || !handle) return MSDA_BAD_ARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)) != cudaSuccess) return MSDA_CUDA_ERROR;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, sizeof(h));
  return MSDA_OK;
}

int32_t msda_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return MSDA_BAD_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr = nullptr;
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return MSDA_CUDA_ERROR;
  return MSDA_OK;
}

int32_t msda_ipc_close(void* ptr) {
  if (ptr && cudaIpcCloseMemHandle(ptr) != cudaSuccess) return MSDA_CUDA_ERROR;
  return MSDA_OK;
}

int32_t msda_peer_allreduce_normalize(const float* num, const float* weight_sums, void* const* peer_buffers,
                                      int32_t world, int32_t rank, uint32_t epoch, int64_t rows, int32_t channels,
                                      int32_t groups, int32_t normalize, float* out, float* wsum_out,
                                      void* workspace, void* stream_) {
  if (!num || !peer_buffers || !out || !workspace || world < 1 || world > kMaxPeers || rank < 0 || rank >= world ||
      rows < 0 || channels <= 0 || groups <= 0 || channels % groups || channels % 4)
    return MSDA_BAD_ARG;
  if (normalize && !weight_sums) return MSDA_BAD_ARG;
  for (int p = 0; p < world; ++p)
    if (!peer_buffers[p]) return MSDA_BAD_ARG;
  if ((reinterpret_cast<uintptr_t>(num) | reinterpret_cast<uintptr_t>(out)) % 16) return MSDA_BAD_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
  DevStatus* status = reinterpret_cast<DevStatus*>(workspace);
  if (cudaMemsetAsync(status, 0, sizeof(DevStatus), s) != cudaSuccess) return MSDA_CUDA_ERROR;
  if (rows == 0) return MSDA_OK;
  const PeerLayout l = peer_layout(rows, channels, groups);
  const int b = (int)(epoch & 1u);
  char* own = reinterpret_cast<char*>(peer_buffers[rank]);
  // 1. the other half (consumed by this rank's previous epoch) back to zero
  if (cudaMemsetAsync(own + (size_t)(b ^ 1) * l.half_bytes, 0, l.half_bytes, s) != cudaSuccess)
    return MSDA_CUDA_ERROR;
  // 2. push the local partial into half b of every rank, then signal
  ExchangeArgs ea{};
  ea.num = num;
  ea.wsum = weight_sums;
  ea.world = world;
  for (int p = 0; p < world; ++p) ea.peer_half[p] = reinterpret_cast<char*>(peer_buffers[p]) + (size_t)b * l.half_bytes;
  ea.num4 = (int64_t)(l.num_floats / 4);
  ea.wsum_n = weight_sums ? (int64_t)l.wsum_floats : 0;
  ea.wsum_off = l.wsum_off;
  ea.flag_off = l.flag_off;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a grid every rank computes identically (the arrival count depends on it)
  const int64_t want = (ea.num4 + kExchangeThreads - 1) / kExchangeThreads;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, 256));
  peer_exchange_kernel<<<grid, kExchangeThreads, 0, s>>>(ea);
  if (cudaGetLastError() != cudaSuccess) return MSDA_CUDA_ERROR;
  // 3. wait for every rank, then normalise into out
  FinishArgs fa{};
  fa.half = own + (size_t)b * l.half_bytes;
  fa.wsum_off = l.wsum_off;
  fa.flag_off = l.flag_off;
  fa.expected = (uint32_t)world * grid;
  fa.rows = rows;
  fa.C = channels;
  fa.G = groups;
  fa.normalize = normalize;
  fa.out = out;
  fa.wsum_out = wsum_out;
  fa.status = status;
  const int64_t total = rows * channels;
  const unsigned fgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sms * 2));
  peer_finish_kernel<<<fgrid, 256, 0, s>>>(fa);
  return cudaGetLastError() == cudaSuccess ? MSDA_OK : MSDA_CUDA_ERROR;
}

}  // extern "C"
