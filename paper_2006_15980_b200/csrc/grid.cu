// Block bucketing: the device form of data.build_grid (hetmf/data.py:238-280).
//
// The reference computes block ids by searchsorted on the cuts and applies a
// stable argsort; here the stable partition is done in three passes over
// warp-sized tiles:
//   1. count   each warp walks its tile 32 triples at a time; __match_any_sync
//              groups lanes with equal block id and the group leader adds the
//              group size to a per-warp shared-memory histogram, written out as
//              column `tile` of a [n_blocks][n_tiles] count matrix;
//   2. scan    one exclusive scan over the flattened matrix gives, for every
//              (block, tile), the output offset of that tile's first triple of
//              that block (block-major, tiles in input order => stable);
//   3. scatter each warp re-walks its tile, a lane's position being the running
//              offset of its block plus its rank among equal-id lanes below it.
#include "hmf_common.cuh"
#include "hmf_internal.h"

namespace hmf {

__device__ inline int band_of(const int64_t* cuts, int n_bands, int64_t x) {
  // largest b with cuts[b] <= x  (searchsorted(cuts, x, side="right") - 1)
  int lo = 0, hi = n_bands;  // answer in [0, n_bands)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(cuts + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

struct BucketGeo {
  const int64_t* row_cuts;
  const int64_t* col_cuts;
  int n_row_bands, n_col_bands, n_blocks;
  int64_t n, tile, n_tiles;
};

__global__ void bucket_count_kernel(const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ cols, BucketGeo g,
                                    int64_t* __restrict__ counts) {
  extern __shared__ int64_t hist_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (tile >= g.n_tiles) return;
  int64_t* hist = hist_smem + int64_t(warp) * g.n_blocks;
  for (int b = lane; b < g.n_blocks; b += 32) hist[b] = 0;
  __syncwarp();
  const int64_t beg = tile * g.tile;
  const int64_t end = min(beg + g.tile, g.n);
  for (int64_t base = beg; base < end; base += 32) {
    const int64_t i = base + lane;
    const bool ok = i < end;
    int bid = -1;
    if (ok)
      bid = band_of(g.row_cuts, g.n_row_bands, rows[i]) * g.n_col_bands +
            band_of(g.col_cuts, g.n_col_bands, cols[i]);
    const unsigned peers = __match_any_sync(0xffffffffu, bid);
    if (ok && lane == __ffs(peers) - 1) hist[bid] += __popc(peers);
    __syncwarp();
  }
  for (int b = lane; b < g.n_blocks; b += 32) counts[int64_t(b) * g.n_tiles + tile] = hist[b];
}

__global__ void bucket_scatter_kernel(const int32_t* __restrict__ rows,
                                      const int32_t* __restrict__ cols,
                                      const float* __restrict__ vals, BucketGeo g,
                                      const int64_t* __restrict__ offsets,
                                      int32_t* __restrict__ out_rows,
                                      int32_t* __restrict__ out_cols,
                                      float* __restrict__ out_vals) {
  extern __shared__ int64_t run_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (tile >= g.n_tiles) return;
  int64_t* run = run_smem + int64_t(warp) * g.n_blocks;
  for (int b = lane; b < g.n_blocks; b += 32) run[b] = offsets[int64_t(b) * g.n_tiles + tile];
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t beg = tile * g.tile;
  const int64_t end = min(beg + g.tile, g.n);
  for (int64_t base = beg; base < end; base += 32) {
    const int64_t i = base + lane;
    const bool ok = i < end;
    int bid = -1;
    int32_t r = 0, c = 0;
    float v = 0.f;
    if (ok) {
      r = rows[i];
      c = cols[i];
      v = vals[i];
      bid = band_of(g.row_cuts, g.n_row_bands, r) * g.n_col_bands +
            band_of(g.col_cuts, g.n_col_bands, c);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bid);
    if (ok) {
      const int64_t pos = run[bid] + __popc(peers & lt);
      out_rows[pos] = r;
      out_cols[pos] = c;
      out_vals[pos] = v;
    }
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) run[bid] += __popc(peers);
    __syncwarp();
  }
}

__global__ void bucket_ptr_kernel(const int64_t* __restrict__ offsets, BucketGeo g,
                                  int64_t* __restrict__ block_ptr) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= g.n_blocks;
       b += gridDim.x * blockDim.x) {
    if (b == g.n_blocks) block_ptr[b] = g.n;
    else block_ptr[b] = g.n_tiles > 0 ? offsets[int64_t(b) * g.n_tiles] : 0;
  }
}

static int bucket(const int32_t* rows, const int32_t* cols, const float* vals, int64_t n,
                  const int64_t* row_cuts, int n_row_bands, const int64_t* col_cuts,
                  int n_col_bands, int32_t* out_rows, int32_t* out_cols, float* out_vals,
                  int64_t* block_ptr, cudaStream_t stream) {
  if (n < 0 || n_row_bands < 1 || n_col_bands < 1)
    return int(set_error(HMF_ERR_ARG, "bad sizes"));
  const int64_t n_blocks = int64_t(n_row_bands) * n_col_bands;
  if (n_blocks > 12288) return int(set_error(HMF_ERR_UNSUPPORTED, "too many blocks (> 12288)"));
  BucketGeo g;
  g.row_cuts = row_cuts;
  g.col_cuts = col_cuts;
  g.n_row_bands = n_row_bands;
  g.n_col_bands = n_col_bands;
  g.n_blocks = int(n_blocks);
  g.n = n;
  // tiles of >= 2048 triples, at most 65536 tiles (count matrix <= 65536 x n_blocks)
  int64_t tile = 2048;
  if ((n + tile - 1) / tile > 65536) tile = (((n + 65535) / 65536) + 31) / 32 * 32;
  g.tile = tile;
  g.n_tiles = (n + tile - 1) / tile;
  cudaError_t e = cudaSuccess;
  if (g.n_tiles == 0) {
    bucket_ptr_kernel<<<1, 256, 0, stream>>>(nullptr, g, block_ptr);
    e = cudaGetLastError();
    return e == cudaSuccess ? HMF_OK : int(set_cuda_error(e));
  }
  int warps = int((96 * 1024) / (n_blocks * 8));
  if (warps > 8) warps = 8;
  if (warps < 1) warps = 1;
  const size_t smem = size_t(warps) * size_t(n_blocks) * 8;
  if (smem > 48 * 1024) {
    int per_sm = 0;  // sets the shared-memory opt-in on this device
    cudaError_t ea = kernel_occupancy(reinterpret_cast<const void*>(bucket_count_kernel),
                                      warps * 32, int(smem), &per_sm);
    if (ea == cudaSuccess)
      ea = kernel_occupancy(reinterpret_cast<const void*>(bucket_scatter_kernel), warps * 32,
                            int(smem), &per_sm);
    if (ea != cudaSuccess) return int(set_cuda_error(ea));
  }
  int64_t* counts = nullptr;
  const size_t cells = size_t(n_blocks) * size_t(g.n_tiles);
  e = cudaMallocAsync(reinterpret_cast<void**>(&counts), cells * 8, stream);
  if (e != cudaSuccess) return int(set_cuda_error(e));
  const unsigned grid = unsigned((g.n_tiles + warps - 1) / warps);
  bucket_count_kernel<<<grid, warps * 32, smem, stream>>>(rows, cols, g, counts);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = scan_exclusive_i64(counts, counts, int64_t(cells), stream);
  if (e == cudaSuccess) {
    bucket_scatter_kernel<<<grid, warps * 32, smem, stream>>>(rows, cols, vals, g, counts,
                                                              out_rows, out_cols, out_vals);
    bucket_ptr_kernel<<<unsigned((n_blocks + 256) / 256), 256, 0, stream>>>(counts, g, block_ptr);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(counts, stream);
  if (e == cudaSuccess) e = e2;
  return e == cudaSuccess ? HMF_OK : int(set_cuda_error(e));
}

}  // namespace hmf

extern "C" int hmf_bucket_triples(const int32_t* rows, const int32_t* cols, const float* vals,
                                  int64_t n, const int64_t* row_cuts, int32_t n_row_bands,
                                  const int64_t* col_cuts, int32_t n_col_bands,
                                  int32_t* out_rows, int32_t* out_cols, float* out_vals,
                                  int64_t* block_ptr, void* stream) {
  return hmf::bucket(rows, cols, vals, n, row_cuts, n_row_bands, col_cuts, n_col_bands, out_rows,
                     out_cols, out_vals, block_ptr, static_cast<cudaStream_t>(stream));
}
