// Error reporting, mix64, device/peer/IPC utilities and a device int64 scan.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "hmf_common.cuh"
#include "hmf_internal.h"

namespace hmf {

static thread_local char g_last_error[256] = "";

int64_t set_error(int64_t code, const char* msg) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
  return code;
}

int64_t set_cuda_error(cudaError_t e) {
  std::snprintf(g_last_error, sizeof(g_last_error), "CUDA error %d: %s", int(e),
                cudaGetErrorString(e));
  return HMF_ERR_CUDA;
}

int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Function attributes (the dynamic shared-memory opt-in above 48 KB) are per
// device: set them and query the occupancy once per (kernel, device, shape).
cudaError_t kernel_occupancy(const void* kern, int threads, int smem, int* per_sm) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  // the dynamic shared-memory limit set per (kernel, device): it only ever
  // grows, so a launch with less shared memory never lowers it under one
  // whose occupancy was cached with more
  static std::map<std::pair<const void*, int>, int> limit;
  const auto key = std::make_tuple(kern, dev, threads, smem);
  std::lock_guard<std::mutex> lock(mu);
  if (smem > 48 * 1024) {
    int& lim = limit[std::make_pair(kern, dev)];
    if (smem > lim) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      lim = smem;
    }
  }
  auto it = cache.find(key);
  if (it != cache.end()) {
    *per_sm = it->second;
    return cudaSuccess;
  }
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, size_t(smem));
  if (e != cudaSuccess) return e;
  if (n < 1) n = 1;
  cache[key] = n;
  *per_sm = n;
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Exclusive scan of int64: per-block sums -> single-block scan of block sums
// -> per-block rescan with carry-in.  Deterministic.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ inline int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < int(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += y;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  const int64_t warp_prefix = warp > 0 ? warp_sums[warp - 1] : 0;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void scan_tile_sums(const int64_t* in, int64_t n, int64_t* tile_sums) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  int64_t s = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + int64_t(threadIdx.x) * kScanItems + j;
    if (i < n) s += in[i];
  }
  int64_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// One block scans all tile sums in place (n_tiles arbitrary: serial chunks).
__global__ void scan_tile_prefix(int64_t* tile_sums, int64_t n_tiles) {
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n_tiles; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < n_tiles ? tile_sums[i] : 0;
    int64_t total;
    const int64_t ex = block_exclusive_scan(v, &total);
    if (i < n_tiles) tile_sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

__global__ void scan_tile_apply(const int64_t* in, int64_t* out, int64_t n,
                                const int64_t* tile_prefix) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  int64_t vals[kScanItems];
  int64_t s = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + int64_t(threadIdx.x) * kScanItems + j;
    vals[j] = i < n ? in[i] : 0;
    s += vals[j];
  }
  int64_t run = tile_prefix[blockIdx.x] + block_exclusive_scan(s, nullptr);
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + int64_t(threadIdx.x) * kScanItems + j;
    if (i < n) out[i] = run;
    run += vals[j];
  }
}

cudaError_t scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  int64_t* sums = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sums), size_t(tiles) * 8, stream);
  if (e != cudaSuccess) return e;
  scan_tile_sums<<<unsigned(tiles), kScanThreads, 0, stream>>>(in, n, sums);
  scan_tile_prefix<<<1, kScanThreads, 0, stream>>>(sums, tiles);
  scan_tile_apply<<<unsigned(tiles), kScanThreads, 0, stream>>>(in, out, n, sums);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(sums, stream);
  return e != cudaSuccess ? e : e2;
}

}  // namespace hmf

extern "C" {

int hmf_abi_version(void) { return HMF_ABI_VERSION; }

const char* hmf_last_error(void) { return hmf::g_last_error; }

// kernels.mix64 (hetmf/kernels.py:32-48).
uint64_t hmf_mix64(const uint64_t* parts, int32_t n_parts) {
  uint64_t h = 0x6A09E667F3BCC909ull;
  for (int32_t i = 0; i < n_parts; ++i) {
    h ^= parts[i];
    h += hmf::kGolden;
    h = hmf::splitmix_finalize(h);
  }
  return h & 0x7FFFFFFFFFFFFFFFull;
}

int hmf_device_count(int32_t* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *n = 0;
    return int(hmf::set_cuda_error(e));
  }
  *n = c;
  return HMF_OK;
}

int hmf_set_device(int32_t dev) {
  cudaError_t e = cudaSetDevice(dev);
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_enable_peer_access(int32_t dev, int32_t peer) {
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, dev, peer);
  if (e != cudaSuccess) return int(hmf::set_cuda_error(e));
  if (!can) return int(hmf::set_error(HMF_ERR_UNSUPPORTED, "peer access not supported"));
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return HMF_OK;
  }
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_memcpy_peer_async(void* dst, int32_t dst_dev, const void* src, int32_t src_dev,
                          int64_t bytes, void* stream) {
  if (bytes < 0) return int(hmf::set_error(HMF_ERR_ARG, "negative byte count"));
  if (bytes == 0) return HMF_OK;
  // a negative device means "locate by unified address" (e.g. an IPC-mapped
  // peer allocation): the driver routes the copy over NVLink
  cudaError_t e =
      (dst_dev < 0 || src_dev < 0)
          ? cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDefault,
                            static_cast<cudaStream_t>(stream))
          : cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, size_t(bytes),
                                static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_stream_synchronize(void* stream) {
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

// IPC handles name whole allocations; a pointer from a caching allocator may
// sit inside one.  The allocation base comes from the driver's
// cuMemGetAddressRange (fetched through the runtime's entry-point query, so
// the library keeps no link-time dependency on libcuda).
typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

int hmf_ipc_get_handle(const void* dptr, uint8_t* handle64, int64_t* offset) {
  static MemGetAddressRangeFn range_fn = nullptr;
  if (!range_fn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return int(hmf::set_error(HMF_ERR_CUDA, "no cuMemGetAddressRange"));
    range_fn = reinterpret_cast<MemGetAddressRangeFn>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0)
    return int(hmf::set_error(HMF_ERR_CUDA, "cuMemGetAddressRange failed"));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return int(hmf::set_cuda_error(e));
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  std::memcpy(handle64, &h, 64);
  *offset = int64_t(reinterpret_cast<unsigned long long>(dptr) - base);
  return HMF_OK;
}

int hmf_ipc_open_handle(const uint8_t* handle64, void** dptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_ipc_close_handle(void* dptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

}  // extern "C"
