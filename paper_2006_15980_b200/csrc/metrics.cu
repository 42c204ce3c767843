// Residual sums for RMSE and the regularized loss (hetmf/sgd.py:134-188), in f64.
//
// Same lane-group row layout as the update kernel (16-byte vectors, shuffle
// reduction), but the products and sums are taken in f64 so the result is
// within rounding of the reference's f64 numpy evaluation on the same values.
// Per-block partials are written to a scratch array and summed in a fixed order
// by a second kernel, so the result is deterministic for a given n and device.
#include <map>
#include <mutex>
#include <utility>

#include "hmf_common.cuh"
#include "hmf_internal.h"

namespace hmf {

constexpr int kMetricThreads = 256;

__device__ inline void block_sum3(double& a, double& b, double& c) {
  __shared__ double red[3][kMetricThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
    red[2][warp] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = b = c = 0.0;
    for (int w = 0; w < kMetricThreads / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
      c += red[2][w];
    }
  }
}

template <int K, typename S>
__global__ void __launch_bounds__(kMetricThreads)
    residual_kernel(const S* __restrict__ P, const S* __restrict__ Q,
                    const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                    const typename RatingOf<S>::T* __restrict__ vals, int64_t n, int64_t row_base,
                    int64_t col_base, int with_reg, double* __restrict__ partials) {
  using G = Geo<K, S>;
  using ST = Storage<S>;
  using C = typename ST::C;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G::LPR, lane_g = lane % G::LPR;
  const int64_t gw = (int64_t(blockIdx.x) * kMetricThreads + threadIdx.x) >> 5;
  const int64_t tw = (int64_t(gridDim.x) * kMetricThreads) >> 5;
  double sq = 0.0, pp = 0.0, qq = 0.0;
  for (int64_t base = gw * G::RPW; base < n; base += tw * G::RPW) {
    const int64_t i = base + grp;
    const bool ok = i < n;
    double dot = 0.0;
    if (ok) {
      const S* prow = P + (int64_t(rows[i]) - row_base) * K;
      const S* qrow = Q + (int64_t(cols[i]) - col_base) * K;
#pragma unroll
      for (int v = 0; v < G::NV; ++v) {
        C p[G::VE], q[G::VE];
        ST::load(prow + (v * G::LPR + lane_g) * G::VE, p);
        ST::load(qrow + (v * G::LPR + lane_g) * G::VE, q);
#pragma unroll
        for (int e = 0; e < G::VE; ++e) {
          dot += double(p[e]) * double(q[e]);
          if (with_reg) {
            pp += double(p[e]) * double(p[e]);
            qq += double(q[e]) * double(q[e]);
          }
        }
      }
    }
    dot = group_sum<G::LPR>(dot);
    if (ok && lane_g == 0) {
      const double err = double(vals[i]) - dot;
      sq += err * err;
    }
  }
  block_sum3(sq, pp, qq);
  if (threadIdx.x == 0) {
    partials[3 * blockIdx.x + 0] = sq;
    partials[3 * blockIdx.x + 1] = pp;
    partials[3 * blockIdx.x + 2] = qq;
  }
}

template <typename S>
__global__ void __launch_bounds__(kMetricThreads)
    residual_generic_kernel(const S* __restrict__ P, const S* __restrict__ Q,
                            const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                            const typename RatingOf<S>::T* __restrict__ vals, int64_t n, int k,
                            int64_t row_base, int64_t col_base, int with_reg,
                            double* __restrict__ partials) {
  using ST = Storage<S>;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * kMetricThreads + threadIdx.x) >> 5;
  const int64_t tw = (int64_t(gridDim.x) * kMetricThreads) >> 5;
  double sq = 0.0, pp = 0.0, qq = 0.0;
  for (int64_t i = gw; i < n; i += tw) {
    const S* prow = P + (int64_t(rows[i]) - row_base) * k;
    const S* qrow = Q + (int64_t(cols[i]) - col_base) * k;
    double dot = 0.0;
    for (int f = lane; f < k; f += 32) {
      const double p = double(ST::load1(prow + f)), q = double(ST::load1(qrow + f));
      dot += p * q;
      if (with_reg) {
        pp += p * p;
        qq += q * q;
      }
    }
    dot = group_sum<32>(dot);
    if (lane == 0) {
      const double err = double(vals[i]) - dot;
      sq += err * err;
    }
  }
  block_sum3(sq, pp, qq);
  if (threadIdx.x == 0) {
    partials[3 * blockIdx.x + 0] = sq;
    partials[3 * blockIdx.x + 1] = pp;
    partials[3 * blockIdx.x + 2] = qq;
  }
}

__global__ void __launch_bounds__(kMetricThreads)
    finalize_sums_kernel(const double* __restrict__ partials, int blocks, double* out) {
  double a = 0.0, b = 0.0, c = 0.0;
  // fixed assignment: thread t sums blocks t, t+T, ... in order
  for (int i = threadIdx.x; i < blocks; i += kMetricThreads) {
    a += partials[3 * i];
    b += partials[3 * i + 1];
    c += partials[3 * i + 2];
  }
  block_sum3(a, b, c);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
    out[2] = c;
  }
}

// Per-(device, stream) partial-sum scratch, allocated once: launches on one
// stream are ordered, so they can share it.  (A cudaMallocAsync per call
// occasionally blocked the host for hundreds of ms on the GPU boxes, stalling
// the per-epoch RMSE read of the streamed e2e loop.)
static cudaError_t partials_for(cudaStream_t stream, size_t bytes, double** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<double*, size_t>> bufs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto& b = bufs[{dev, stream}];
  if (b.second < bytes) {
    if (b.first) {
      e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return e;
      cudaFree(b.first);
      b = {nullptr, 0};
    }
    e = cudaMalloc(reinterpret_cast<void**>(&b.first), bytes);
    if (e != cudaSuccess) return e;
    b.second = bytes;
  }
  *out = b.first;
  return cudaSuccess;
}

template <typename S>
static int residual_sums(const S* P, const S* Q, int64_t k, const int32_t* rows,
                         const int32_t* cols, const typename RatingOf<S>::T* vals, int64_t n,
                         int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                         cudaStream_t stream) {
  if (k < 1 || n < 0) return int(set_error(HMF_ERR_ARG, "bad k or n"));
  if (!out) return int(set_error(HMF_ERR_ARG, "null out"));
  const int64_t want = (n * 32 + kMetricThreads - 1) / kMetricThreads;
  int64_t blocks = int64_t(device_sm_count()) * 8;
  if (want < blocks) blocks = want;
  if (blocks < 1) blocks = 1;
  double* partials = nullptr;
  cudaError_t e = partials_for(stream, size_t(device_sm_count()) * 8 * 3 * sizeof(double),
                               &partials);
  if (e != cudaSuccess) return int(set_cuda_error(e));
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) == 0;
  const unsigned g = unsigned(blocks);
  bool done = false;
  if (aligned) {
    switch (k) {
#define HMF_RES_CASE(KK)                                                                         \
  case KK:                                                                                       \
    residual_kernel<KK, S><<<g, kMetricThreads, 0, stream>>>(P, Q, rows, cols, vals, n, row_base, \
                                                            col_base, with_reg, partials);       \
    done = true;                                                                                 \
    break;
      HMF_RES_CASE(32)
      HMF_RES_CASE(64)
      HMF_RES_CASE(128)
      HMF_RES_CASE(256)
#undef HMF_RES_CASE
      default: break;
    }
  }
  if (!done)
    residual_generic_kernel<S><<<g, kMetricThreads, 0, stream>>>(
        P, Q, rows, cols, vals, n, int(k), row_base, col_base, with_reg, partials);
  finalize_sums_kernel<<<1, kMetricThreads, 0, stream>>>(partials, int(blocks), out);
  e = cudaGetLastError();
  return e == cudaSuccess ? HMF_OK : int(set_cuda_error(e));
}

}  // namespace hmf

extern "C" {

int hmf_residual_sums_f32(const float* user_f, const float* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream) {
  return hmf::residual_sums<float>(user_f, item_f, k, rows, cols, vals, n, row_base, col_base,
                                   with_reg, out, static_cast<cudaStream_t>(stream));
}

int hmf_residual_sums_f16(const uint16_t* user_f, const uint16_t* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream) {
  return hmf::residual_sums<__half>(reinterpret_cast<const __half*>(user_f),
                                    reinterpret_cast<const __half*>(item_f), k, rows, cols, vals,
                                    n, row_base, col_base, with_reg, out,
                                    static_cast<cudaStream_t>(stream));
}

int hmf_residual_sums_f64(const double* user_f, const double* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const double* vals, int64_t n,
                          int64_t row_base, int64_t col_base, int32_t with_reg, double* out,
                          void* stream) {
  return hmf::residual_sums<double>(user_f, item_f, k, rows, cols, vals, n, row_base, col_base,
                                    with_reg, out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
