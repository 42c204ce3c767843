// The reference visit order of sgd_range (hetmf/kernels.py:77-119), on device.
//
// The reference draws one splitmix64 stream from state seed ^ 0xD1B54A32D192ED03:
// first nw-1 draws Fisher-Yates the window order (kernels.py:81-89), then each
// window, in visit order, copies its triples to scratch and Fisher-Yates them
// with the next span-1 draws (kernels.py:96-119).  The t-th draw is a pure
// function of t (state advances by the golden constant), and every window but
// the last holds exactly W = 4096 triples, so the draw offset and output offset
// of every visited window are closed-form: windows are shuffled in parallel,
// one warp each.  Within a window the swap indices j = z % (i+1) are computed
// 32 at a time by the lanes and applied serially by lane 0 in shared memory.
#include "hmf_common.cuh"
#include "hmf_internal.h"

namespace hmf {

constexpr int kOrderWarps = 2;

// Window permutation (single thread; nw-1 sequential swaps).  worder[nw]
// receives the visit position of the short last window (index nw-1).
__global__ void window_order_kernel(int64_t nw, uint64_t s0, int32_t* worder) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int64_t i = 0; i < nw; ++i) worder[i] = int32_t(i);
  uint64_t t = 0;
  for (int64_t i = nw - 1; i > 0; --i) {
    const uint64_t z = rand_z(s0, ++t);
    const int64_t j = int64_t(z % uint64_t(i + 1));
    const int32_t tmp = worder[i];
    worder[i] = worder[j];
    worder[j] = tmp;
  }
  int32_t last_pos = 0;
  for (int64_t i = 0; i < nw; ++i)
    if (worder[i] == int32_t(nw - 1)) last_pos = int32_t(i);
  worder[nw] = last_pos;
}

__global__ void __launch_bounds__(kOrderWarps * 32)
    window_shuffle_kernel(int64_t n, int64_t nw, uint64_t s0, const int32_t* __restrict__ worder,
                          int32_t* __restrict__ perm) {
  __shared__ int32_t scratch[kOrderWarps][kShuffleWindow];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * kOrderWarps + warp;  // visit position
  if (w >= nw) return;
  constexpr int64_t W = kShuffleWindow;
  const int64_t wid = worder[w];
  const int64_t lo = wid * W;
  const int64_t span = (n - lo) < W ? (n - lo) : W;
  const int64_t last_pos = worder[nw];
  const int64_t span_last = n - (nw - 1) * W;
  const int64_t short_before = (last_pos < w) ? (W - span_last) : 0;
  const uint64_t draw0 = uint64_t(nw - 1) + uint64_t(w * (W - 1) - short_before);
  const int64_t out_base = w * W - short_before;
  int32_t* s = scratch[warp];
  for (int64_t i = lane; i < span; i += 32) s[i] = int32_t(lo + i);
  __syncwarp();
  // Step st (0-based) handles i = span-1-st and uses draw number draw0+st+1.
  for (int64_t sb = 0; sb < span - 1; sb += 32) {
    const int64_t st = sb + lane;
    int32_t j = 0;
    if (st < span - 1) {
      const int64_t i = span - 1 - st;
      j = int32_t(rand_z(s0, draw0 + uint64_t(st) + 1) % uint64_t(i + 1));
    }
    const int64_t cnt = (span - 1 - sb) < 32 ? (span - 1 - sb) : 32;
    for (int l = 0; l < cnt; ++l) {
      const int32_t jl = __shfl_sync(0xffffffffu, j, l);
      if (lane == 0) {
        const int64_t i = span - 1 - (sb + l);
        const int32_t a = s[i];
        s[i] = s[jl];
        s[jl] = a;
      }
    }
    __syncwarp();
  }
  for (int64_t i = lane; i < span; i += 32) perm[out_base + i] = s[i];
}

cudaError_t launch_visit_order(int64_t n, uint64_t seed, int32_t* perm, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const uint64_t s0 = seed ^ kOrderSalt;
  const int64_t nw = (n + kShuffleWindow - 1) / kShuffleWindow;
  int32_t* worder = nullptr;
  cudaError_t e =
      cudaMallocAsync(reinterpret_cast<void**>(&worder), size_t(nw + 1) * sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  window_order_kernel<<<1, 1, 0, stream>>>(nw, s0, worder);
  const int64_t blocks = (nw + kOrderWarps - 1) / kOrderWarps;
  window_shuffle_kernel<<<unsigned(blocks), kOrderWarps * 32, 0, stream>>>(n, nw, s0, worder,
                                                                             perm);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(worder, stream);
  return e != cudaSuccess ? e : e2;
}

}  // namespace hmf

extern "C" int hmf_visit_order(int64_t n, uint64_t seed, int32_t* perm, void* stream) {
  if (n < 0 || n > INT32_MAX) return int(hmf::set_error(HMF_ERR_ARG, "n out of range"));
  if (n > 0 && !perm) return int(hmf::set_error(HMF_ERR_ARG, "null perm"));
  cudaError_t e = hmf::launch_visit_order(n, seed, perm, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}
