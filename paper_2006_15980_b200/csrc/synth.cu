// Synthetic instance generator with the law of data.synthetic_ratings
// (hetmf/data.py:311-336): unique cells uniform over the matrix, ratings
// sum_r A[u,r] B[v,r] + N(0, noise), A/B ~ U[0, factor_scale/sqrt(rank)].
//
// The reference draws cells with numpy (np.unique over rejection draws), which
// takes 326 s at 100 M cells and cannot produce 3.1 B; here every cell is
// selected independently with probability p by geometric skipping along its
// row (one thread per row, counter-based RNG), so the selected set is uniform
// given its size; the host then permutes it and keeps the exact target count,
// mirroring the reference's permutation(chosen)[:target].
#include <math.h>

#include "hmf_common.cuh"
#include "hmf_internal.h"

namespace hmf {

__device__ inline uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return splitmix_finalize(splitmix_finalize(seed ^ (a * kGolden + 0x632BE59BD9B4E019ull)) +
                           b * kMixA + kGolden);
}

// Uniform on (0, 1].
__device__ inline double unit_open(uint64_t h) {
  return (double((h >> 11) + 1ull)) * 0x1.0p-53;
}

// Next selected column after `col` in row `row` (draw number j), or >= n_cols.
__device__ inline int64_t next_cell(int64_t col, double log_q, uint64_t seed, int64_t row,
                                    uint64_t j) {
  if (log_q == 0.0) return col + 1;  // p >= 1: every cell
  const double u = unit_open(hash3(seed, uint64_t(row), j));
  const double skip = floor(log(u) / log_q);
  if (skip > 9.0e15) return INT64_MAX / 2;
  return col + 1 + int64_t(skip);
}

__global__ void synth_count_kernel(int64_t n_rows, int64_t n_cols, double log_q, uint64_t seed,
                                   int64_t row_base, int64_t* row_cnt) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n_rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    int64_t col = -1, cnt = 0;
    uint64_t j = 0;
    while (true) {
      col = next_cell(col, log_q, seed, row_base + row, j++);
      if (col >= n_cols) break;
      ++cnt;
    }
    row_cnt[row] = cnt;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) row_cnt[n_rows] = 0;
}

__global__ void synth_cells_kernel(int64_t n_rows, int64_t n_cols, double log_q, uint64_t seed,
                                   int64_t row_base, const int64_t* __restrict__ row_ptr,
                                   int32_t* out_rows, int32_t* out_cols) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n_rows;
       row += int64_t(gridDim.x) * blockDim.x) {
    int64_t col = -1, pos = row_ptr[row];
    uint64_t j = 0;
    while (true) {
      col = next_cell(col, log_q, seed, row_base + row, j++);
      if (col >= n_cols) break;
      out_rows[pos] = int32_t(row_base + row);
      out_cols[pos] = int32_t(col);
      ++pos;
    }
  }
}

__global__ void synth_fill_kernel(const int32_t* __restrict__ rows,
                                  const int32_t* __restrict__ cols, int64_t n, int rank,
                                  double noise, double hi, uint64_t seed, float* __restrict__ vals) {
  const uint64_t seed_a = splitmix_finalize(seed + 1), seed_b = splitmix_finalize(seed + 2),
                 seed_n = splitmix_finalize(seed + 3);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = uint64_t(rows[i]), v = uint64_t(cols[i]);
    double acc = 0.0;
    for (int r = 0; r < rank; ++r) {
      const double a = (unit_open(hash3(seed_a, u, uint64_t(r))) - 0x1.0p-53) * hi;
      const double b = (unit_open(hash3(seed_b, v, uint64_t(r))) - 0x1.0p-53) * hi;
      acc += a * b;
    }
    if (noise > 0.0) {
      // keyed by the cell, not its position: a row band generated alone
      // (hmf_synthetic_count with row_base) gets the same values as the
      // whole matrix
      const double u1 = unit_open(hash3(seed_n, u, v));
      const double u2 = unit_open(hash3(seed_n ^ kMixB, u, v));
      acc += noise * sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    vals[i] = float(acc);
  }
}

// Keyed pseudo-random permutation of [0, n): a 4-round balanced Feistel
// network over [0, 4^h) >= n with cycle walking (expected < 4 steps), so a
// random reordering of billions of cells needs no sort and no index array.
struct Feistel {
  uint32_t half_bits;
  uint64_t mask, keys[4];
  __device__ uint64_t round(uint64_t r, int i) const {
    return splitmix_finalize(r * kGolden ^ keys[i]) & mask;
  }
  __device__ uint64_t once(uint64_t x) const {
    uint64_t l = x >> half_bits, r = x & mask;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t t = l ^ round(r, i);
      l = r;
      r = t;
    }
    return (l << half_bits) | r;
  }
  __device__ uint64_t operator()(uint64_t x, uint64_t n) const {
    do { x = once(x); } while (x >= n);
    return x;
  }
};

__global__ void permute_cells_kernel(const int32_t* __restrict__ in_rows,
                                     const int32_t* __restrict__ in_cols, int64_t n_in,
                                     int32_t* __restrict__ out_rows, int32_t* __restrict__ out_cols,
                                     int64_t n_out, Feistel f) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_out;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = int64_t(f(uint64_t(i), uint64_t(n_in)));
    out_rows[i] = in_rows[j];
    out_cols[i] = in_cols[j];
  }
}

// Held-out split keyed by the cell: mask[i] = 1 iff hash(seed, row, col) <
// fraction, so every row band of a matrix agrees with the whole on which
// cells are test cells.
__global__ void cell_mask_kernel(const int32_t* __restrict__ rows,
                                 const int32_t* __restrict__ cols, int64_t n, double fraction,
                                 uint64_t seed, uint8_t* __restrict__ mask) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    mask[i] = unit_open(hash3(seed, uint64_t(rows[i]), uint64_t(cols[i]))) <= fraction ? 1 : 0;
}

static double log_keep(double p) {
  if (p >= 1.0) return 0.0;
  return log1p(-p);
}

}  // namespace hmf

extern "C" {

int64_t hmf_synthetic_count(int64_t n_rows, int64_t n_cols, double p, uint64_t seed,
                            int64_t row_base, int64_t* row_ptr, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || n_cols < 0 || row_base < 0 || !(p > 0.0) || !row_ptr)
    return hmf::set_error(HMF_ERR_ARG, "bad generator arguments");
  const int64_t blocks = n_rows > 0 ? (n_rows + 255) / 256 : 1;
  hmf::synth_count_kernel<<<unsigned(blocks < 65535 * 16 ? blocks : 65535 * 16), 256, 0, stream>>>(
      n_rows, n_cols, hmf::log_keep(p), seed, row_base, row_ptr);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = hmf::scan_exclusive_i64(row_ptr, row_ptr, n_rows + 1, stream);
  int64_t total = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&total, row_ptr + n_rows, 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return hmf::set_cuda_error(e);
  return total;
}

int hmf_synthetic_cells(int64_t n_rows, int64_t n_cols, double p, uint64_t seed,
                        int64_t row_base, const int64_t* row_ptr, int32_t* out_rows,
                        int32_t* out_cols, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n_rows < 0 || n_cols < 0 || row_base < 0 || !(p > 0.0) || !row_ptr)
    return int(hmf::set_error(HMF_ERR_ARG, "bad generator arguments"));
  if (row_base + n_rows > INT32_MAX || n_cols > INT32_MAX)
    return int(hmf::set_error(HMF_ERR_ARG, "indices must fit int32"));
  const int64_t blocks = n_rows > 0 ? (n_rows + 255) / 256 : 1;
  hmf::synth_cells_kernel<<<unsigned(blocks < 65535 * 16 ? blocks : 65535 * 16), 256, 0, stream>>>(
      n_rows, n_cols, hmf::log_keep(p), seed, row_base, row_ptr, out_rows, out_cols);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_permute_cells(const int32_t* in_rows, const int32_t* in_cols, int64_t n_in,
                      int32_t* out_rows, int32_t* out_cols, int64_t n_out, uint64_t seed,
                      void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n_in < 0 || n_out < 0 || n_out > n_in)
    return int(hmf::set_error(HMF_ERR_ARG, "need 0 <= n_out <= n_in"));
  if (n_out == 0) return HMF_OK;
  hmf::Feistel f;
  uint32_t bits = 1;
  while ((uint64_t(1) << (2 * bits)) < uint64_t(n_in)) ++bits;
  f.half_bits = bits;
  f.mask = (uint64_t(1) << bits) - 1;
  for (int i = 0; i < 4; ++i) f.keys[i] = hmf::splitmix_finalize(seed + uint64_t(i + 1) * hmf::kMixB);
  int64_t blocks = (n_out + 255) / 256;
  const int64_t cap = int64_t(hmf::device_sm_count()) * 32;
  if (blocks > cap) blocks = cap;
  hmf::permute_cells_kernel<<<unsigned(blocks), 256, 0, stream>>>(in_rows, in_cols, n_in, out_rows,
                                                                  out_cols, n_out, f);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_synthetic_fill(const int32_t* rows, const int32_t* cols, int64_t n, int32_t rank,
                       double noise, double factor_scale, uint64_t seed, float* vals,
                       void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n < 0 || rank < 1) return int(hmf::set_error(HMF_ERR_ARG, "bad fill arguments"));
  if (n == 0) return HMF_OK;
  const double hi = factor_scale / sqrt(double(rank));
  int64_t blocks = (n + 255) / 256;
  if (blocks > int64_t(hmf::device_sm_count()) * 32) blocks = int64_t(hmf::device_sm_count()) * 32;
  hmf::synth_fill_kernel<<<unsigned(blocks), 256, 0, stream>>>(rows, cols, n, rank, noise, hi, seed,
                                                               vals);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

int hmf_cell_mask(const int32_t* rows, const int32_t* cols, int64_t n, double fraction,
                  uint64_t seed, uint8_t* mask, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (n < 0 || !(fraction >= 0.0) || fraction > 1.0)
    return int(hmf::set_error(HMF_ERR_ARG, "bad mask arguments"));
  if (n == 0) return HMF_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > int64_t(hmf::device_sm_count()) * 32) blocks = int64_t(hmf::device_sm_count()) * 32;
  hmf::cell_mask_kernel<<<unsigned(blocks), 256, 0, stream>>>(rows, cols, n, fraction, seed, mask);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HMF_OK : int(hmf::set_cuda_error(e));
}

}  // extern "C"
