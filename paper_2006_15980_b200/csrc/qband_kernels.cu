// Q-band-stationary block update: the staged item band of the reference's
// BatchEngine (workers.py:186-202, "triples plus the touched item-factor
// columns") held in shared memory on B200.
//
// A block of the division plan is split into S column sub-bands (equal item
// width).  Its triples are bucketed by sub-band (stable), so sub-band s is the
// contiguous range [sub_ptr[s], sub_ptr[s+1]) and touches only items
// [sub_cuts[s], sub_cuts[s+1]).  Warp w owns sub-bands w, w + TW, ...:
//   1. copy the sub-band's Q rows into its private shared-memory slice (fp32),
//   2. stream the sub-band's triples through a 2-stage cp.async.bulk ring,
//   3. per rating: P row from HBM (16-byte vectors, prefetched one group of U
//      ratings ahead), Q row from shared memory, __shfl_xor dot, update; the Q
//      row is rewritten in shared memory (exact sequential SGD for Q — no
//      other warp can touch it), the P delta is added with a vector
//      reduction (red.global.add.v4.f32; other warps may share the user),
//   4. write the Q slice back (rounded to the storage type once).
// Versus the global-Q HOGWILD kernel this removes the Q loads and Q
// reductions from the SM->L2 path (half of its traffic, the binding unit in
// the r01 ncu profile) and all races on Q.
//
// Row tiles (L2 residency of P).  The block's user span is cut into n_tiles
// equal row tiles sized to sit in L2; triples are bucketed tile-major, so
// sub-band s of tile t is [sub_ptr[t*n_sub+s], sub_ptr[t*n_sub+s+1]).  All
// warps walk the tiles in one seeded rotation: the P rows live at any moment
// are about one tile's, so P reads and reductions hit L2 instead of HBM.
// Sub-band s belongs to the same warp in every tile, so Q stays race-free.
#include "hmf_common.cuh"
#include "hmf_internal.h"
#include "lanevec.cuh"

namespace hmf {

namespace qs {

constexpr int kWarps = 16;           // warps per CTA
constexpr int kChunk = 128;          // triples per staging stage
constexpr int kSliceBytes = 4096;    // fp32 Q slice per warp

// Row layout: RowLay<K, S> (lanevec.cuh) — 32 lanes, K/32 elements each,
// vectorised for every storage width; the fp32 Q slice uses the same
// element interleave.
template <int K, typename S> using Lay = RowLay<K, S>;

constexpr int stage_bytes = kChunk * 12;
constexpr int warp_bytes = kSliceBytes + 2 * stage_bytes + 16;

// i-th row tile of an epoch: the same seeded rotation for every warp
__device__ inline int tile_at(int i, int n_tiles, uint64_t seed) {
  if (n_tiles <= 1) return 0;
  const int rot = int(splitmix_finalize(seed ^ 0x5851F42D4C957F2DULL) % uint64_t(n_tiles));
  const int t = i + rot;
  return t >= n_tiles ? t - n_tiles : t;
}

}  // namespace qs
}  // namespace hmf

#include "qchain.cuh"
#include "runs.cuh"

namespace hmf {
namespace qs {

struct Ring {
  int32_t* rows;
  int32_t* cols;
  float* vals;
};

__device__ inline Ring ring_at(unsigned char* base, int b) {
  unsigned char* p = base + kSliceBytes + b * stage_bytes;
  return Ring{reinterpret_cast<int32_t*>(p), reinterpret_cast<int32_t*>(p + kChunk * 4),
              reinterpret_cast<float*>(p + kChunk * 8)};
}

__device__ inline void stage(const Ring& r, uint64_t* bar, const int32_t* rows,
                             const int32_t* cols, const float* vals, int64_t beg, int64_t end,
                             bool bulk_ok, int lane) {
  const int n = int(end - beg);
  const int n_bulk = bulk_ok ? (n & ~3) : 0;
  if (lane == 0) {
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, uint32_t(n_bulk) * 12u);
    if (n_bulk > 0) {
      bulk_g2s(r.rows, rows + beg, n_bulk * 4, bar);
      bulk_g2s(r.cols, cols + beg, n_bulk * 4, bar);
      bulk_g2s(r.vals, vals + beg, n_bulk * 4, bar);
    }
  }
  for (int i = n_bulk + lane; i < n; i += 32) {
    r.rows[i] = __ldg(rows + beg + i);
    r.cols[i] = __ldg(cols + beg + i);
    r.vals[i] = __ldg(vals + beg + i);
  }
}

template <int K, typename S, int U, int MINB = 2>
__global__ void __launch_bounds__(kWarps * 32, MINB)
    qband_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const int32_t* __restrict__ rows,
                 const int32_t* __restrict__ cols, const float* __restrict__ vals,
                 const int64_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_cuts,
                 int n_sub, int n_tiles, float lr, float ru, float ri, uint64_t seed) {
  using L = Lay<K, S>;
  constexpr int E = L::EPL;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * warp_bytes;
  float* qslice = reinterpret_cast<float*>(wbase);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + kSliceBytes + 2 * stage_bytes);
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int tw = gridDim.x * kWarps;
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(cols) |
                         reinterpret_cast<uintptr_t>(vals)) & 15u) == 0;
  uint32_t phase[2] = {0u, 0u};

  for (int ti = 0; ti < n_tiles; ++ti) {
  const int tile = tile_at(ti, n_tiles, seed);
  const int64_t* sp = sub_ptr + int64_t(tile) * n_sub;
  const uint64_t bin0 = uint64_t(tile) * uint64_t(n_sub);
  for (int s = blockIdx.x * kWarps + warp; s < n_sub; s += tw) {
    const int c_lo = sub_cuts[s];
    const int n_items = sub_cuts[s + 1] - c_lo;
    if (n_items > kSliceBytes / (K * 4)) __trap();  // host contract: slice fits
    if (sp[s + 1] <= sp[s]) continue;  // no triples in this tile: nothing to stage
    S* qrow0 = Qb + int64_t(c_lo) * K;
    // 1. Q slice -> shared memory (fp32)
    for (int it = 0; it < n_items; ++it) {
      float t[E];
      Lay<K, S>::ldg(qrow0 + int64_t(it) * K, lane, t);
      Lay<K, S>::stsf(qslice + it * K, lane, t);
    }
    const int64_t beg = sp[s], end = sp[s + 1];
    const int64_t a0 = beg & ~int64_t(3);
    const int64_t n_chunks = (end - a0 + kChunk - 1) / kChunk;
    // seeded rotation of the chunk visit order (fresh order every epoch)
    const int64_t rot =
        n_chunks > 0
            ? int64_t(splitmix_finalize(seed + (bin0 + uint64_t(s)) * kGolden) % uint64_t(n_chunks))
            : 0;
    auto chunk_begin = [&](int64_t x) -> int64_t {
      int64_t c = x + rot;
      if (c >= n_chunks) c -= n_chunks;
      return a0 + c * kChunk;
    };
    if (n_chunks > 0) {
      const int64_t cb = chunk_begin(0);
      stage(ring_at(wbase, 0), &bars[0], rows, cols, vals, cb, min(cb + kChunk, end), bulk_ok,
            lane);
    }
    int qcur = -1;  // slice index of the Q row held in q[]
    float q[E];
    __syncwarp();
    for (int64_t x = 0; x < n_chunks; ++x) {
      const int b = int(x & 1);
      if (x + 1 < n_chunks) {
        const int64_t nb = chunk_begin(x + 1);
        stage(ring_at(wbase, b ^ 1), &bars[b ^ 1], rows, cols, vals, nb, min(nb + kChunk, end),
              bulk_ok, lane);
      }
      const int64_t cb = chunk_begin(x);
      const int lo = int(max(beg - cb, int64_t(0)));
      const int hi = int(min(cb + kChunk, end) - cb);
      mbar_wait(&bars[b], phase[b]);
      phase[b] ^= 1u;
      __syncwarp();
      const Ring r = ring_at(wbase, b);

      float pc[U][E], pn[U][E];
      int32_t uc[U], un[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = lo + j;
        uc[j] = i < hi ? r.rows[i] : -1;
        if (uc[j] >= 0) Lay<K, S>::ldg(Pb + int64_t(uc[j]) * K, lane, pc[j]);
      }
      for (int base = lo; base < hi; base += U) {
        // prefetch the next group's P rows
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int i = base + U + j;
          un[j] = i < hi ? r.rows[i] : -1;
          if (un[j] >= 0) Lay<K, S>::ldg(Pb + int64_t(un[j]) * K, lane, pn[j]);
        }
        // the current group, sequentially on the shared-memory Q slice
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (uc[j] >= 0) {
            const int i = base + j;
            // item runs: the current item's Q row stays in registers; the
            // shared slice is touched only when the item changes (warp-uniform)
            const int v = r.cols[i] - c_lo;
            if (v != qcur) {
              if (qcur >= 0) Lay<K, S>::stsf(qslice + qcur * K, lane, q);
              Lay<K, S>::ldsf(qslice + v * K, lane, q);
              qcur = v;
            }
            float d = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) d += pc[j][e] * q[e];
            d = group_sum<32>(d);
            const float err = r.vals[i] - d;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const float pu = pc[j][e], qv = q[e];
              pc[j][e] = lr * (err * qv - ru * pu);
              q[e] = qv + lr * (err * pu - ri * qv);
            }
            Lay<K, S>::red(Pb + int64_t(uc[j]) * K, lane, pc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          uc[j] = un[j];
#pragma unroll
          for (int e = 0; e < E; ++e) pc[j][e] = pn[j][e];
        }
      }
      __syncwarp();
    }
    if (qcur >= 0) Lay<K, S>::stsf(qslice + qcur * K, lane, q);
    __syncwarp();
    // 4. Q slice back to HBM (rounded to the storage type once per lease)
    for (int it = 0; it < n_items; ++it) {
      float t[E];
      Lay<K, S>::ldsf(qslice + it * K, lane, t);
      Lay<K, S>::stg(qrow0 + int64_t(it) * K, lane, t);
    }
    __syncwarp();
  }
  }  // tiles
}


// ---------------------------------------------------------------------------
// Host side.  Implementation 0 is the warp-per-rating kernel above (the
// north star's "one warp per rating"); 4-6 are the chained item-run kernels
// (qchain.cuh), 5 the default.  Round 1's implementations 1 (TMA P-row ring,
// 3.0 G upd/s at NF k=128), 2 (per-lane cp.async ring) and 3 (implementation
// 0 at one CTA per SM) lost to 4/5 at every k and are gone
// (profiles/r02/impl_sweep_nf_k128.jsonl, r01_tma_variant/).
// ---------------------------------------------------------------------------
template <int K> struct RegCfg {  // ratings per prefetch group
  static constexpr int U = (K / 32) >= 4 ? 2 : 4;
};

template <int K, typename S>
static cudaError_t warp_slots_per_sm(int* out) {
  auto kern = qband_kernel<K, S, RegCfg<K>::U>;
  int per_sm = 0;
  const cudaError_t e = kernel_occupancy(reinterpret_cast<const void*>(kern), kWarps * 32,
                                         kWarps * warp_bytes, &per_sm);
  *out = per_sm * kWarps;
  return e;
}

template <int K, typename S>
static cudaError_t launch_warp(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                               const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                               int n_sub, int n_tiles, double lr, double ru, double ri,
                               uint64_t seed, int64_t row_base, int64_t col_base,
                               cudaStream_t stream, const LaunchOpts& o) {
  // P rows prefetched one group ahead: 2 x U x (K/32) floats per lane in flight
  auto kern = qband_kernel<K, S, RegCfg<K>::U>;
  const int smem = kWarps * warp_bytes;
  int per_sm = 0;
  const cudaError_t e =
      kernel_occupancy(reinterpret_cast<const void*>(kern), kWarps * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int want = (n_sub + kWarps - 1) / kWarps;
  const int cap = grid_share(device_sm_count() * per_sm, o.share);
  const int grid = want < cap ? want : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kWarps * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                            sub_ptr, sub_cuts, n_sub, n_tiles, float(lr), float(ru),
                                            float(ri), seed);
  return cudaGetLastError();
}

constexpr int kDefaultImpl = 5;
constexpr int kDefaultQsync = 32;

// hmf_qband_opts -> LaunchOpts (NULL or -1 fields: defaults).  Returns
// HMF_OK or a negative code with the message set.
static int64_t resolve_opts(const hmf_qband_opts* in, int64_t k, bool f16, LaunchOpts* o) {
  o->impl = in && in->impl >= 0 ? in->impl : kDefaultImpl;
  if (in && in->impl < -1) return set_error(HMF_ERR_ARG, "impl must be -1, 0, 4..6 or 8");
  if (o->impl != 0 && (o->impl < 4 || o->impl > 8 || o->impl == 7))
    return set_error(HMF_ERR_ARG, "impl must be -1, 0, 4..6 or 8");
  o->cfg = in && in->chain_cfg >= 0 ? in->chain_cfg : auto_chain_cfg(int(k), f16);
  if (!chain_cfg_ok(o->cfg) || (in && in->chain_cfg < -1))
    return set_error(HMF_ERR_ARG, "chain_cfg must be -1, 2, 4, 5 or 6");
  if (in && (in->pstore < -1 || in->pstore > 1))
    return set_error(HMF_ERR_ARG, "pstore must be -1, 0 or 1");
  o->pstore = in && in->pstore == 1 ? 1 : 0;
  if (in && in->qsync < -1) return set_error(HMF_ERR_ARG, "qsync must be >= -1");
  o->qsync = in && in->qsync >= 0 ? in->qsync : kDefaultQsync;
  if (in && (in->grid_share < -1 || in->grid_share == 0 || in->grid_share > 64))
    return set_error(HMF_ERR_ARG, "grid_share must be -1 or 1..64");
  o->share = in && in->grid_share >= 1 ? in->grid_share : 1;
  if (in && (in->lockstep < -1 || in->lockstep > 3))
    return set_error(HMF_ERR_ARG, "lockstep must be -1..3");
  o->lockstep = in && in->lockstep >= 0 ? in->lockstep : 3;
  if (in && (in->runs_wide < -1 || in->runs_wide > 1))
    return set_error(HMF_ERR_ARG, "runs_wide must be -1, 0 or 1");
  o->wide = in && in->runs_wide == 1 ? 1 : 0;
  return HMF_OK;
}

static int64_t check_block_args(const void* P, const void* Q, const void* rows, const void* vals,
                                const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                int64_t n_tiles) {
  if (n_sub * n_tiles > (int64_t(1) << 31))
    return set_error(HMF_ERR_ARG, "n_sub * n_tiles too large");
  if (!P || !Q || !rows || !vals || !sub_ptr || !sub_cuts)
    return set_error(HMF_ERR_ARG, "null pointer");
  if (((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) != 0)
    return set_error(HMF_ERR_ARG, "factor arrays must be 16-byte aligned");
  return HMF_OK;
}

template <typename S>
static int64_t run(S* P, S* Q, int64_t k, const int32_t* rows, const int32_t* cols,
                   const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                   int64_t n_sub, int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                   double ru, double ri, uint64_t seed, int64_t row_base, int64_t col_base,
                   cudaStream_t stream) {
  LaunchOpts o;
  int64_t rc = resolve_opts(opts, k, sizeof(S) == 2, &o);
  if (rc != HMF_OK) return rc;
  if (n_sub <= 0 || n_tiles <= 0) return 0;
  rc = check_block_args(P, Q, rows, vals, sub_ptr, sub_cuts, n_sub, n_tiles);
  if (rc != HMF_OK) return rc;
  if (o.impl == 8)
    return set_error(HMF_ERR_ARG, "implementation 8 runs through hmf_sgd_block_runs_*");
  // cols == nullptr: every sub-band is one item, sub_cuts[s] (chained kernel only)
  if (!cols && o.impl == 0)
    return set_error(HMF_ERR_ARG, "cols may be null only for implementations 4-6");
  cudaError_t e;
  switch (k) {
#define HMF_QB_CASE(KK)                                                                      \
  case KK:                                                                                   \
    e = o.impl == 0                                                                          \
            ? launch_warp<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),      \
                                 int(n_tiles), lr, ru, ri, seed, row_base, col_base, stream, \
                                 o)                                                          \
            : launch_chain<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),     \
                                  int(n_tiles), lr, ru, ri, seed, row_base, col_base, stream, \
                                  o);                                                        \
    break;
    HMF_QB_CASE(32)
    HMF_QB_CASE(64)
    HMF_QB_CASE(128)
    HMF_QB_CASE(256)
#undef HMF_QB_CASE
    default: return set_error(HMF_ERR_UNSUPPORTED, "Q-band kernel needs k in {32,64,128,256}");
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return 0;
}

// the chained kernel with uint16 row ids (row tile relative, see launch_chain)
template <typename S>
static int64_t run_u16(S* P, S* Q, int64_t k, const uint16_t* rows, const int32_t* cols,
                       const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                       int64_t n_sub, int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                       double ru, double ri, uint64_t seed, int64_t row_base, int64_t col_base,
                       cudaStream_t stream, const int32_t* tile_row0 = nullptr) {
  LaunchOpts o;
  int64_t rc = resolve_opts(opts, k, sizeof(S) == 2, &o);
  if (rc != HMF_OK) return rc;
  if (n_sub <= 0 || n_tiles <= 0) return 0;
  rc = check_block_args(P, Q, rows, vals, sub_ptr, sub_cuts, n_sub, n_tiles);
  if (rc != HMF_OK) return rc;
  if (o.impl == 0 || o.impl >= 7)
    return set_error(HMF_ERR_UNSUPPORTED, "uint16 row ids need implementation 4, 5 or 6");
  cudaError_t e;
  switch (k) {
#define HMF_QB_CASE(KK)                                                                     \
  case KK:                                                                                  \
    e = launch_chain<KK, S, uint16_t>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub), \
                                      int(n_tiles), lr, ru, ri, seed, row_base, col_base,   \
                                      stream, o, tile_row0);                                \
    break;
    HMF_QB_CASE(32)
    HMF_QB_CASE(64)
    HMF_QB_CASE(128)
    HMF_QB_CASE(256)
#undef HMF_QB_CASE
    default: return set_error(HMF_ERR_UNSUPPORTED, "Q-band kernel needs k in {32,64,128,256}");
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return 0;
}

// implementation 8: run groups over a tile-resident P (runs.cuh)
template <int K, typename S, typename RowT, bool Wide = false>
static cudaError_t launch_runs(S* P, S* Q, const RowT* rows, const float* vals,
                               const int32_t* runs, const int32_t* tile_run,
                               const int32_t* tile_cut, int n_tiles,
                               int max_rows, double lr, double ru, double ri, uint64_t seed,
                               int64_t row_base, int64_t col_base, cudaStream_t stream,
                               const LaunchOpts& o) {
  if constexpr (K == 32 && !Wide) {
    if (o.wide)
      return launch_runs<K, S, RowT, true>(P, Q, rows, vals, runs, tile_run, tile_cut, n_tiles,
                                           max_rows, lr, ru, ri, seed, row_base, col_base,
                                           stream, o);
  }
  using C = RunsCfg<K, S, Wide>;
  auto kern = runs_kernel<K, S, C::LPC, C::WPB, RowT>;
  const int smem = max_rows * K * int(sizeof(S));
  int per_sm = 0;
  cudaError_t e = kernel_occupancy(reinterpret_cast<const void*>(kern), C::WPB * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int cap = grid_share(device_sm_count() * per_sm, o.share);
  const int grid = n_tiles < cap ? n_tiles : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, C::WPB * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, vals,
                                            reinterpret_cast<const int4*>(runs), tile_run,
                                            tile_cut, n_tiles, float(lr), float(ru), float(ri),
                                            uint32_t(seed ^ (seed >> 32)));
  return cudaGetLastError();
}

template <typename S, typename RowT>
static int64_t run_runs(S* P, S* Q, int64_t k, const RowT* rows, const float* vals,
                        const int32_t* runs, const int32_t* tile_run,
                        const int32_t* tile_cut, int64_t n_tiles, int32_t max_rows,
                        const hmf_qband_opts* opts, double lr, double ru, double ri,
                        uint64_t seed, int64_t row_base, int64_t col_base, cudaStream_t stream) {
  LaunchOpts o;
  int64_t rc = resolve_opts(opts, k, sizeof(S) == 2, &o);
  if (rc != HMF_OK) return rc;
  if (opts && opts->impl >= 0 && opts->impl != 8)
    return set_error(HMF_ERR_ARG, "hmf_sgd_block_runs_* runs implementation 8");
  if (n_tiles <= 0) return 0;
  if (!P || !Q || !rows || !vals || !runs || !tile_run || !tile_cut)
    return set_error(HMF_ERR_ARG, "null pointer");
  if ((reinterpret_cast<uintptr_t>(runs) & 15u) != 0)
    return set_error(HMF_ERR_ARG, "run descriptors must be 16-byte aligned");
  if (((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) != 0)
    return set_error(HMF_ERR_ARG, "factor arrays must be 16-byte aligned");
  if (n_tiles > (int64_t(1) << 30)) return set_error(HMF_ERR_ARG, "n_tiles too large");
  if (max_rows <= 0 || int64_t(max_rows) * k * int64_t(sizeof(S)) > kPTileBytes)
    return set_error(HMF_ERR_ARG, "a tile's P rows must fit hmf_ptile_max_rows(k, f16)");
  if (sizeof(RowT) == 2 && max_rows > 65536)
    return set_error(HMF_ERR_ARG, "uint16 row ids need tiles of at most 65536 rows");
  if (sizeof(RowT) == 1 && max_rows > 256)
    return set_error(HMF_ERR_ARG, "uint8 row ids need tiles of at most 256 rows");
  cudaError_t e;
  switch (k) {
#define HMF_RN_CASE(KK)                                                                      \
  case KK:                                                                                   \
    e = launch_runs<KK, S, RowT>(P, Q, rows, vals, runs, tile_run, tile_cut,                 \
                                 int(n_tiles), max_rows, lr, ru, ri, seed, row_base,          \
                                 col_base, stream, o);                                        \
    break;
    HMF_RN_CASE(32)
    HMF_RN_CASE(64)
    HMF_RN_CASE(128)
    HMF_RN_CASE(256)
#undef HMF_RN_CASE
    default: return set_error(HMF_ERR_UNSUPPORTED, "Q-band kernel needs k in {32,64,128,256}");
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return 0;
}

template <typename S>
static int slots_per_sm(int64_t k, const hmf_qband_opts* opts) {
  LaunchOpts o;
  if (resolve_opts(opts, k, sizeof(S) == 2, &o) != HMF_OK) return 0;
  int n = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (k) {
#define HMF_WPS(KK)                                                                        \
  case KK:                                                                                 \
    e = o.impl == 0 ? warp_slots_per_sm<KK, S>(&n)                                         \
        : o.impl == 8 ? (n = o.wide && KK == 32                                            \
                             ? RunsCfg<KK, S, true>::WPB * 32 / RunsCfg<KK, S, true>::LPC       \
                             : RunsCfg<KK, S>::WPB * 32 / RunsCfg<KK, S>::LPC,                  \
                         cudaSuccess)         \
                      : chain_slots_per_sm<KK, S>(o.cfg, &n);                                \
    break;
    HMF_WPS(32)
    HMF_WPS(64)
    HMF_WPS(128)
    HMF_WPS(256)
#undef HMF_WPS
    default: break;
  }
  if (e != cudaSuccess) return int(set_cuda_error(e));
  return n;
}

}  // namespace qs
}  // namespace hmf

extern "C" {

int32_t hmf_qband_slots_per_sm(int64_t k, int32_t f16, const hmf_qband_opts* opts) {
  return f16 ? hmf::qs::slots_per_sm<__half>(k, opts) : hmf::qs::slots_per_sm<float>(k, opts);
}

int32_t hmf_qband_resolve_impl(int64_t k, int32_t f16) {
  (void)k;
  (void)f16;
  return hmf::qs::kDefaultImpl;
}

int32_t hmf_qband_resolve_chain_cfg(int64_t k, int32_t f16) {
  return hmf::qs::auto_chain_cfg(int(k), f16 != 0);
}

int32_t hmf_qband_chain_lanes(int64_t k, int32_t f16, int32_t cfg) {
  const int c = cfg >= 0 ? cfg : hmf::qs::auto_chain_cfg(int(k), f16 != 0);
  if (!hmf::qs::chain_cfg_ok(c)) return int32_t(hmf::set_error(HMF_ERR_ARG, "bad chain_cfg"));
  return hmf::qs::chain_lanes(int(k), c);
}

int32_t hmf_qband_max_items(int64_t k, int32_t f16, int32_t impl) {
  (void)f16;
  if (k != 32 && k != 64 && k != 128 && k != 256) return 0;
  if (impl != 0) return int32_t(1 << 30);  // chained: Q rows in registers, no slice bound
  return int32_t(hmf::qs::kSliceBytes / (k * 4));
}

int64_t hmf_sgd_block_qband_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                                const int32_t* cols, const float* vals, const int64_t* sub_ptr,
                                const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                const hmf_qband_opts* opts, double lr, double reg_user,
                                double reg_item, uint64_t seed, int64_t row_base, int64_t col_base,
                                void* stream) {
  return hmf::qs::run<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                             n_tiles, opts, lr, reg_user, reg_item, seed, row_base, col_base,
                             static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                const int32_t* rows, const int32_t* cols, const float* vals,
                                const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                double reg_user, double reg_item, uint64_t seed, int64_t row_base,
                                int64_t col_base, void* stream) {
  return hmf::qs::run<__half>(reinterpret_cast<__half*>(user_f), reinterpret_cast<__half*>(item_f),
                              k, rows, cols, vals, sub_ptr, sub_cuts, n_sub, n_tiles, opts, lr,
                              reg_user, reg_item, seed, row_base, col_base,
                              static_cast<cudaStream_t>(stream));
}

int32_t hmf_ptile_max_rows(int64_t k, int32_t f16) {
  if (k != 32 && k != 64 && k != 128 && k != 256) return 0;
  return int32_t(hmf::qs::kPTileBytes / (k * (f16 ? 2 : 4)));
}

int32_t hmf_runs_chains_per_warp(int64_t k, int32_t f16) {
  using hmf::qs::RunsCfg;
#define HMF_RUNS_NC(KK) \
  case KK: return 32 / (f16 ? RunsCfg<KK, __half>::LPC : RunsCfg<KK, float>::LPC);
  switch (k) {
    HMF_RUNS_NC(32)
    HMF_RUNS_NC(64)
    HMF_RUNS_NC(128)
    HMF_RUNS_NC(256)
    default: return 0;
  }
#undef HMF_RUNS_NC
}

int64_t hmf_sgd_block_runs_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                               const float* vals, const int32_t* runs, const int32_t* tile_run,
                               const int32_t* tile_cut, int64_t n_tiles, int32_t max_tile_rows,
                               const hmf_qband_opts* opts, double lr, double reg_user,
                               double reg_item, uint64_t seed, int64_t row_base, int64_t col_base,
                               void* stream) {
  return hmf::qs::run_runs<float, int32_t>(user_f, item_f, k, rows, vals, runs, tile_run,
                                           tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user,
                                           reg_item, seed, row_base, col_base,
                                           static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_runs_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                               const int32_t* rows, const float* vals, const int32_t* runs,
                               const int32_t* tile_run, const int32_t* tile_cut, int64_t n_tiles,
                               int32_t max_tile_rows, const hmf_qband_opts* opts, double lr,
                               double reg_user, double reg_item, uint64_t seed, int64_t row_base,
                               int64_t col_base, void* stream) {
  return hmf::qs::run_runs<__half, int32_t>(
      reinterpret_cast<__half*>(user_f), reinterpret_cast<__half*>(item_f), k, rows, vals, runs,
      tile_run, tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user, reg_item, seed, row_base,
      col_base, static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_runs_u16_f32(float* user_f, float* item_f, int64_t k, const uint16_t* rows,
                                   const float* vals, const int32_t* runs,
                                   const int32_t* tile_run, const int32_t* tile_cut,
                                   int64_t n_tiles, int32_t max_tile_rows,
                                   const hmf_qband_opts* opts, double lr, double reg_user,
                                   double reg_item, uint64_t seed, int64_t row_base,
                                   int64_t col_base, void* stream) {
  return hmf::qs::run_runs<float, uint16_t>(user_f, item_f, k, rows, vals, runs, tile_run,
                                            tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user,
                                            reg_item, seed, row_base, col_base,
                                            static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_runs_u16_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                   const uint16_t* rows, const float* vals, const int32_t* runs,
                                   const int32_t* tile_run, const int32_t* tile_cut,
                                   int64_t n_tiles, int32_t max_tile_rows,
                                   const hmf_qband_opts* opts, double lr, double reg_user,
                                   double reg_item, uint64_t seed, int64_t row_base,
                                   int64_t col_base, void* stream) {
  return hmf::qs::run_runs<__half, uint16_t>(
      reinterpret_cast<__half*>(user_f), reinterpret_cast<__half*>(item_f), k, rows, vals, runs,
      tile_run, tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user, reg_item, seed, row_base,
      col_base, static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_runs_u8_f32(float* user_f, float* item_f, int64_t k, const uint8_t* rows,
                                  const float* vals, const int32_t* runs, const int32_t* tile_run,
                                  const int32_t* tile_cut, int64_t n_tiles, int32_t max_tile_rows,
                                  const hmf_qband_opts* opts, double lr, double reg_user,
                                  double reg_item, uint64_t seed, int64_t row_base,
                                  int64_t col_base, void* stream) {
  return hmf::qs::run_runs<float, uint8_t>(user_f, item_f, k, rows, vals, runs, tile_run,
                                           tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user,
                                           reg_item, seed, row_base, col_base,
                                           static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_runs_u8_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                  const uint8_t* rows, const float* vals, const int32_t* runs,
                                  const int32_t* tile_run, const int32_t* tile_cut,
                                  int64_t n_tiles, int32_t max_tile_rows,
                                  const hmf_qband_opts* opts, double lr, double reg_user,
                                  double reg_item, uint64_t seed, int64_t row_base,
                                  int64_t col_base, void* stream) {
  return hmf::qs::run_runs<__half, uint8_t>(
      reinterpret_cast<__half*>(user_f), reinterpret_cast<__half*>(item_f), k, rows, vals, runs,
      tile_run, tile_cut, n_tiles, max_tile_rows, opts, lr, reg_user, reg_item, seed, row_base,
      col_base, static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_f32(float* user_f, float* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                    double reg_user, double reg_item, uint64_t seed,
                                    int64_t row_base, int64_t col_base, void* stream) {
  return hmf::qs::run_u16<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                                 n_tiles, opts, lr, reg_user, reg_item, seed, row_base, col_base,
                                 static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, const hmf_qband_opts* opts, double lr,
                                    double reg_user, double reg_item, uint64_t seed,
                                    int64_t row_base, int64_t col_base, void* stream) {
  return hmf::qs::run_u16<__half>(reinterpret_cast<__half*>(user_f),
                                  reinterpret_cast<__half*>(item_f), k, rows, cols, vals, sub_ptr,
                                  sub_cuts, n_sub, n_tiles, opts, lr, reg_user, reg_item, seed,
                                  row_base, col_base, static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_tiles_f32(float* user_f, float* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, const hmf_qband_opts* opts,
                                          double lr, double reg_user, double reg_item,
                                          uint64_t seed, int64_t col_base, void* stream) {
  if (!tile_row0 && n_sub > 0 && n_tiles > 0) return hmf::set_error(HMF_ERR_ARG, "null pointer");
  return hmf::qs::run_u16<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                                 n_tiles, opts, lr, reg_user, reg_item, seed, 0, col_base,
                                 static_cast<cudaStream_t>(stream), tile_row0);
}

int64_t hmf_sgd_block_qband_u16_tiles_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, const hmf_qband_opts* opts,
                                          double lr, double reg_user, double reg_item,
                                          uint64_t seed, int64_t col_base, void* stream) {
  if (!tile_row0 && n_sub > 0 && n_tiles > 0) return hmf::set_error(HMF_ERR_ARG, "null pointer");
  return hmf::qs::run_u16<__half>(reinterpret_cast<__half*>(user_f),
                                  reinterpret_cast<__half*>(item_f), k, rows, cols, vals, sub_ptr,
                                  sub_cuts, n_sub, n_tiles, opts, lr, reg_user, reg_item, seed, 0,
                                  col_base, static_cast<cudaStream_t>(stream), tile_row0);
}

}  // extern "C"
