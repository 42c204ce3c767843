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
#include <atomic>
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
// TMA-pipelined variant.  Same ownership scheme (one warp per item sub-band,
// Q slice in shared memory), but every global transfer is a bulk async copy
// issued by one lane:
//   * P rows are fetched D ratings ahead into a per-warp shared-memory ring
//     (cp.async.bulk global->shared, one mbarrier per slot), so a warp keeps D
//     rows in flight without holding them in registers;
//   * P deltas are written to a small ring and added to HBM by TMA bulk
//     reductions (cp.reduce.async.bulk .add.f32 -> UBLKRED), E in flight;
//   * triples arrive through the 2-stage bulk ring as before.
// Lanes only touch shared memory and registers: the per-lane LDG/RED traffic
// of the register-prefetch variant (the SM->L2 request path bound in the r01
// profile) moves to the TMA engine.
// ---------------------------------------------------------------------------
template <int K, typename S, int D, int E> struct TmaLayout {
  static constexpr int ROWB = K * int(sizeof(S));
  static constexpr int TRIP = 2 * stage_bytes;
  static constexpr int PRING = D * ROWB;
  static constexpr int DRING = E * ROWB;
  static constexpr int O_TRIP = kSliceBytes;
  static constexpr int O_PRING = O_TRIP + TRIP;
  static constexpr int O_DRING = O_PRING + PRING;
  static constexpr int O_BARS = O_DRING + DRING;
  static constexpr int BYTES = ((O_BARS + (2 + D) * 8) + 127) / 128 * 128;
};

__device__ inline void bulk_reduce_add(float* dst, const void* src, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
      "r"(smem_addr(src)), "r"(bytes)
      : "memory");
}
__device__ inline void bulk_reduce_add(__half* dst, const void* src, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.noftz.f16 [%0], [%1], %2;" ::"l"(
          dst),
      "r"(smem_addr(src)), "r"(bytes)
      : "memory");
}
__device__ inline void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ inline void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ inline void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int K, typename S, int D, int E, int WPB, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB)
    qtma_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const int32_t* __restrict__ rows,
                const int32_t* __restrict__ cols, const float* __restrict__ vals,
                const int64_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_cuts,
                int n_sub, int n_tiles, float lr, float ru, float ri, uint64_t seed) {
  using T = TmaLayout<K, S, D, E>;
  constexpr int EL = Lay<K, S>::EPL;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * T::BYTES;
  float* qslice = reinterpret_cast<float*>(wbase);
  S* pring = reinterpret_cast<S*>(wbase + T::O_PRING);
  S* dring = reinterpret_cast<S*>(wbase + T::O_DRING);
  uint64_t* tbar = reinterpret_cast<uint64_t*>(wbase + T::O_BARS);  // 2 triple stages
  uint64_t* pbar = tbar + 2;                                         // D P slots
  if (lane == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    for (int i = 0; i < D; ++i) mbar_init(&pbar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int tw = gridDim.x * WPB;
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(cols) |
                         reinterpret_cast<uintptr_t>(vals)) & 15u) == 0;
  uint32_t tpar[2] = {0u, 0u};  // wait parity per triple stage
  uint32_t issued = 0, consumed = 0;

  for (int ti = 0; ti < n_tiles; ++ti) {
  const int tile = tile_at(ti, n_tiles, seed);
  const int64_t* sp = sub_ptr + int64_t(tile) * n_sub;
  const uint64_t bin0 = uint64_t(tile) * uint64_t(n_sub);
  for (int s = blockIdx.x * WPB + warp; s < n_sub; s += tw) {
    const int c_lo = sub_cuts[s];
    const int n_items = sub_cuts[s + 1] - c_lo;
    if (n_items > kSliceBytes / (K * 4)) __trap();
    if (sp[s + 1] <= sp[s]) continue;  // no triples: nothing to stage
    S* qrow0 = Qb + int64_t(c_lo) * K;
    for (int it = 0; it < n_items; ++it) {
      float t[EL];
      Lay<K, S>::ldg(qrow0 + int64_t(it) * K, lane, t);
      Lay<K, S>::stsf(qslice + it * K, lane, t);
    }
    const int64_t beg = sp[s], end = sp[s + 1];
    const int64_t a0 = beg & ~int64_t(3);
    const int n_chunks = int((end - a0 + kChunk - 1) / kChunk);
    if (n_chunks <= 0) continue;
    const int rot = int(splitmix_finalize(seed + (bin0 + uint64_t(s)) * kGolden) % uint64_t(n_chunks));
    auto cbeg = [&](int x) -> int64_t {
      int c = x + rot;
      if (c >= n_chunks) c -= n_chunks;
      return a0 + int64_t(c) * kChunk;
    };
    auto clo = [&](int x) -> int { return int(max(beg - cbeg(x), int64_t(0))); };
    auto chi = [&](int x) -> int { return int(min(cbeg(x) + kChunk, end) - cbeg(x)); };
    auto stage_x = [&](int x) {
      const int64_t b0 = cbeg(x);
      stage(ring_at(wbase, x & 1), &tbar[x & 1], rows, cols, vals, b0, min(b0 + kChunk, end),
            bulk_ok, lane);
    };
    auto wait_x = [&](int x) {
      mbar_wait(&tbar[x & 1], tpar[x & 1]);
      tpar[x & 1] ^= 1u;
      __syncwarp();
    };
    // prefetch cursor (px, pi) runs up to D ratings ahead of the consume
    // cursor (cx, ci) and never more than one chunk ahead (only chunks cx and
    // cx+1 are staged)
    stage_x(0);
    if (n_chunks > 1) stage_x(1);
    __syncwarp();
    wait_x(0);
    int px = 0, pi = clo(0);
    int cx = 0, ci = clo(0);
    bool px_ready = true;  // chunk px's triples waited (chunk 0 just was)
    auto issue = [&]() {
      // Wait for a chunk lazily, at its first issue: issues are guarded by
      // px <= cx + 1, so the chunk has been staged by then.
      if (!px_ready) {
        wait_x(px);
        px_ready = true;
      }
      if (lane == 0) {
        const int slot = int(issued % D);
        const int32_t u = ring_at(wbase, px & 1).rows[pi];
        fence_proxy_async();
        mbar_arrive_expect_tx(&pbar[slot], uint32_t(T::ROWB));
        bulk_g2s(pring + slot * K, Pb + int64_t(u) * K, uint32_t(T::ROWB), &pbar[slot]);
      }
      ++issued;
      if (++pi >= chi(px)) {
        ++px;
        px_ready = false;
        if (px < n_chunks) pi = clo(px);
      }
    };
    while (px < n_chunks && px <= cx + 1 && issued - consumed < uint32_t(D)) issue();
    while (cx < n_chunks) {
      const Ring r = ring_at(wbase, cx & 1);
      const int slot = int(consumed % D);
      mbar_wait(&pbar[slot], (consumed / D) & 1u);
      float p[EL], q[EL];
      Lay<K, S>::lds(pring + slot * K, lane, p);
      const int vloc = r.cols[ci] - c_lo;
      float* qs_row = qslice + vloc * K;
      Lay<K, S>::ldsf(qs_row, lane, q);
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < EL; ++e) d += p[e] * q[e];
      d = group_sum<32>(d);
      const float err = r.vals[ci] - d;
#pragma unroll
      for (int e = 0; e < EL; ++e) {
        const float pu = p[e], qv = q[e];
        p[e] = lr * (err * qv - ru * pu);
        q[e] = qv + lr * (err * pu - ri * qv);
      }
      Lay<K, S>::stsf(qs_row, lane, q);
      // delta ring slot: the reduction that last read it must be done reading
      const int dslot = int(consumed % E);
      if (lane == 0 && consumed >= uint32_t(E)) bulk_wait_read<E - 1>();
      __syncwarp();
      Lay<K, S>::sts(dring + dslot * K, lane, p);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        bulk_reduce_add(Pb + int64_t(r.rows[ci]) * K, dring + dslot * K, uint32_t(T::ROWB));
        bulk_commit();
      }
      ++consumed;
      if (++ci >= chi(cx)) {
        ++cx;
        if (cx + 1 < n_chunks) {
          __syncwarp();
          stage_x(cx + 1);  // buffer (cx+1)&1 held chunk cx-1: fully consumed
        }
        if (cx < n_chunks) ci = clo(cx);
      }
      while (px < n_chunks && px <= cx + 1 && issued - consumed < uint32_t(D)) issue();
    }
    // Q slice back to HBM
    for (int it = 0; it < n_items; ++it) {
      float t[EL];
      Lay<K, S>::ldsf(qslice + it * K, lane, t);
      Lay<K, S>::stg(qrow0 + int64_t(it) * K, lane, t);
    }
    __syncwarp();
  }
  }  // tiles
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// (D, E, WPB, MINB) per K: ~13-14 KB of shared memory per warp, 16 warps/SM
template <int K, typename S> struct TmaCfg {
  static constexpr int ROWB = K * int(sizeof(S));
  static constexpr int D0 = 4096 / ROWB;
  static constexpr int D = D0 < 4 ? 4 : (D0 > 16 ? 16 : D0);
  static constexpr int E = D / 2;
  static constexpr int WPB = 8, MINB = 2;
};

template <int K, typename S>
static cudaError_t launch_tma(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                              const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                              int n_sub, int n_tiles, double lr, double ru, double ri, uint64_t seed,
                              int64_t row_base, int64_t col_base, cudaStream_t stream) {
  using C = TmaCfg<K, S>;
  using T = TmaLayout<K, S, C::D, C::E>;
  auto kern = qtma_kernel<K, S, C::D, C::E, C::WPB, C::MINB>;
  const int smem = C::WPB * T::BYTES;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  const int want = (n_sub + C::WPB - 1) / C::WPB;
  const int cap = grid_share(device_sm_count() * per_sm);
  const int grid = want < cap ? want : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, C::WPB * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                            sub_ptr, sub_cuts, n_sub, n_tiles, float(lr), float(ru),
                                            float(ri), seed);
  return cudaGetLastError();
}

template <int K, typename S>
static int tma_warps_per_sm() {
  using C = TmaCfg<K, S>;
  using T = TmaLayout<K, S, C::D, C::E>;
  auto kern = qtma_kernel<K, S, C::D, C::E, C::WPB, C::MINB>;
  const int smem = C::WPB * T::BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, smem);
  return per_sm * C::WPB;
}

// register-prefetch configurations: impl 0 = 2 CTAs/SM, U ratings per group;
// impl 3 = 1 CTA/SM with twice the registers and a group twice as deep
template <int K, bool Deep> struct RegCfg {
  static constexpr int U = ((K / 32) >= 4 ? 2 : 4) * (Deep ? 2 : 1);
  static constexpr int MINB = Deep ? 1 : 2;
};

template <int K, typename S, bool Deep = false>
static int reg_warps_per_sm() {
  using C = RegCfg<K, Deep>;
  auto kern = qband_kernel<K, S, C::U, C::MINB>;
  const int smem = kWarps * warp_bytes;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  return per_sm * kWarps;
}

// process default implementation; -1 = automatic (resolve_impl)
static std::atomic<int> g_qband_impl{-1};

// Implementation for a launch: an explicit impl >= 0, else the process
// default, else automatic: the chained kernel with Q deltas (5).  With whole
// item runs per sub-band it is the chained kernel (4), on the L2
// load+reduction ceiling at k >= 128 (profiles/r02/l2_rowbench.jsonl); with
// item runs split over chains it also beats the warp-per-rating kernel (0)
// on narrow blocks and small k (ML-1M 12.1 vs 6.5, NF k=32 fp32 21.1 vs 16.5
// G upd/s; profiles/r02/impl5_*.jsonl).
static int resolve_impl(int impl, int64_t k, bool f16) {
  (void)k;
  (void)f16;
  if (impl < 0) impl = g_qband_impl;
  if (impl < 0) impl = 5;
  return impl;
}

// ---------------------------------------------------------------------------
// Async-copy ring variant (impl 2).  Same ownership scheme; the P rows of the
// next D-1 ratings are in flight as per-lane cp.async copies (LDGSTS) into a
// per-warp shared-memory ring instead of registers.  Each lane copies and
// later reads back only its own vector of a row, so a lane's own
// cp.async.wait_group is the only synchronisation: no proxy fences, no
// mbarriers, no cross-lane barriers on the P path.  Registers no longer bound
// the prefetch depth, so D rows per warp stay in flight.
// ---------------------------------------------------------------------------
template <int K, typename S, int D> struct AsyncLayout {
  static constexpr int ROWB = K * int(sizeof(S));
  static constexpr int SLICE = 2048;  // fp32 Q slice per warp
  static constexpr int O_TRIP = SLICE;
  static constexpr int O_RING = O_TRIP + 2 * stage_bytes;
  static constexpr int O_BARS = O_RING + D * ROWB;
  static constexpr int BYTES = ((O_BARS + 16) + 127) / 128 * 128;
};

template <int BYTES> __device__ inline void cp_async(void* smem_dst, const void* gsrc) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_dst)),
                 "l"(gsrc)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(smem_dst)),
                 "l"(gsrc), "n"(BYTES)
                 : "memory");
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ inline void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int K, typename S, int D, int WPB, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB)
    qasync_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const int32_t* __restrict__ rows,
                  const int32_t* __restrict__ cols, const float* __restrict__ vals,
                  const int64_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_cuts,
                  int n_sub, int n_tiles, float lr, float ru, float ri, uint64_t seed) {
  using L = Lay<K, S>;
  using AL = AsyncLayout<K, S, D>;
  constexpr int E = L::EPL;
  constexpr int VB = L::W * int(sizeof(S));  // bytes per lane vector
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * AL::BYTES;
  float* qslice = reinterpret_cast<float*>(wbase);
  S* ring = reinterpret_cast<S*>(wbase + AL::O_RING);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + AL::O_BARS);
  auto rstage = [&](int b) -> Ring {
    unsigned char* p = wbase + AL::O_TRIP + b * stage_bytes;
    return Ring{reinterpret_cast<int32_t*>(p), reinterpret_cast<int32_t*>(p + kChunk * 4),
                reinterpret_cast<float*>(p + kChunk * 8)};
  };
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int tw = gridDim.x * WPB;
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(cols) |
                         reinterpret_cast<uintptr_t>(vals)) & 15u) == 0;
  uint32_t phase[2] = {0u, 0u};

  // issue the P row of user u into ring slot `slot` (this lane's vectors)
  auto fetch = [&](int32_t u, int slot) {
    const S* src = Pb + int64_t(u) * K;
    S* dst = ring + slot * K;
#pragma unroll
    for (int v = 0; v < L::NV; ++v) cp_async<VB>(dst + L::off(v, lane), src + L::off(v, lane));
  };

  for (int ti = 0; ti < n_tiles; ++ti) {
  const int tile = tile_at(ti, n_tiles, seed);
  const int64_t* sp = sub_ptr + int64_t(tile) * n_sub;
  const uint64_t bin0 = uint64_t(tile) * uint64_t(n_sub);
  for (int s = blockIdx.x * WPB + warp; s < n_sub; s += tw) {
    const int c_lo = sub_cuts[s];
    const int n_items = sub_cuts[s + 1] - c_lo;
    if (n_items * K * 4 > AL::SLICE) __trap();  // host contract: slice fits
    const int64_t beg = sp[s], end = sp[s + 1];
    if (end <= beg) continue;
    S* qrow0 = Qb + int64_t(c_lo) * K;
    for (int it = 0; it < n_items; ++it) {
      float t[E];
      L::ldg(qrow0 + int64_t(it) * K, lane, t);
      L::stsf(qslice + it * K, lane, t);
    }
    const int64_t a0 = beg & ~int64_t(3);
    const int64_t n_chunks = (end - a0 + kChunk - 1) / kChunk;
    const int64_t rot = int64_t(splitmix_finalize(seed + (bin0 + uint64_t(s)) * kGolden) % uint64_t(n_chunks));
    auto chunk_begin = [&](int64_t x) -> int64_t {
      int64_t c = x + rot;
      if (c >= n_chunks) c -= n_chunks;
      return a0 + c * kChunk;
    };
    {
      const int64_t cb = chunk_begin(0);
      stage(rstage(0), &bars[0], rows, cols, vals, cb, min(cb + kChunk, end), bulk_ok, lane);
    }
    __syncwarp();
    for (int64_t x = 0; x < n_chunks; ++x) {
      const int b = int(x & 1);
      if (x + 1 < n_chunks) {
        const int64_t nb = chunk_begin(x + 1);
        stage(rstage(b ^ 1), &bars[b ^ 1], rows, cols, vals, nb, min(nb + kChunk, end), bulk_ok,
              lane);
      }
      const int64_t cb = chunk_begin(x);
      const int lo = int(max(beg - cb, int64_t(0)));
      const int hi = int(min(cb + kChunk, end) - cb);
      mbar_wait(&bars[b], phase[b]);
      phase[b] ^= 1u;
      __syncwarp();
      const Ring r = rstage(b);
      // prologue: D-1 rows in flight, one commit group per rating
#pragma unroll
      for (int j = 0; j < D - 1; ++j) {
        if (lo + j < hi) fetch(r.rows[lo + j], (lo + j) % D);
        cp_async_commit();
      }
      for (int i = lo; i < hi; ++i) {
        if (i + D - 1 < hi) fetch(r.rows[i + D - 1], (i + D - 1) % D);
        cp_async_commit();
        cp_async_wait<D - 1>();  // this lane's copy of row i has landed
        float p[E], q[E];
        L::lds(ring + (i % D) * K, lane, p);
        float* qs_row = qslice + (r.cols[i] - c_lo) * K;
        L::ldsf(qs_row, lane, q);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) d += p[e] * q[e];
        d = group_sum<32>(d);
        const float err = r.vals[i] - d;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float pu = p[e], qv = q[e];
          p[e] = lr * (err * qv - ru * pu);
          q[e] = qv + lr * (err * pu - ri * qv);
        }
        L::stsf(qs_row, lane, q);
        L::red(Pb + int64_t(r.rows[i]) * K, lane, p);
      }
      cp_async_wait<0>();
      __syncwarp();
    }
    for (int it = 0; it < n_items; ++it) {
      float t[E];
      L::ldsf(qslice + it * K, lane, t);
      L::stg(qrow0 + int64_t(it) * K, lane, t);
    }
    __syncwarp();
  }
  }  // tiles
}

template <int K, typename S> struct AsyncCfg {
  static constexpr int ROWB = K * int(sizeof(S));
  static constexpr int D0 = 3072 / ROWB;
  static constexpr int D = D0 < 4 ? 4 : (D0 > 16 ? 16 : D0);
  static constexpr int WPB = 8, MINB = 3;
};

template <int K, typename S>
static cudaError_t launch_async(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                                int n_sub, int n_tiles, double lr, double ru, double ri, uint64_t seed,
                                int64_t row_base, int64_t col_base, cudaStream_t stream) {
  using C = AsyncCfg<K, S>;
  using AL = AsyncLayout<K, S, C::D>;
  auto kern = qasync_kernel<K, S, C::D, C::WPB, C::MINB>;
  const int smem = C::WPB * AL::BYTES;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  const int want = (n_sub + C::WPB - 1) / C::WPB;
  const int cap = grid_share(device_sm_count() * per_sm);
  const int grid = want < cap ? want : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, C::WPB * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                            sub_ptr, sub_cuts, n_sub, n_tiles, float(lr), float(ru),
                                            float(ri), seed);
  return cudaGetLastError();
}

template <int K, typename S>
static int async_warps_per_sm() {
  using C = AsyncCfg<K, S>;
  using AL = AsyncLayout<K, S, C::D>;
  auto kern = qasync_kernel<K, S, C::D, C::WPB, C::MINB>;
  const int smem = C::WPB * AL::BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, smem);
  return per_sm * C::WPB;
}

// impl 2 needs >= 4-byte lane vectors (cp.async sizes 4/8/16): not K=32 fp16
template <int K, typename S> constexpr bool async_ok() {
  return Lay<K, S>::W * int(sizeof(S)) >= 4;
}

template <int K, typename S>
static cudaError_t launch_async_if(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                   const float* vals, const int64_t* sub_ptr,
                                   const int32_t* sub_cuts, int n_sub, int n_tiles, double lr, double ru,
                                   double ri, uint64_t seed, int64_t row_base, int64_t col_base,
                                   cudaStream_t stream) {
  if constexpr (async_ok<K, S>())
    return launch_async<K, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, n_sub, n_tiles, lr, ru, ri, seed,
                              row_base, col_base, stream);
  else
    return cudaErrorNotSupported;
}

template <int K, typename S>
static int async_warps_per_sm_if() {
  if constexpr (async_ok<K, S>()) return async_warps_per_sm<K, S>();
  else return 0;
}

template <int K, typename S>
constexpr int max_items() {
  return kSliceBytes / (K * 4);
}

template <int K, typename S, bool Deep = false>
static cudaError_t launch(S* P, S* Q, const int32_t* rows, const int32_t* cols, const float* vals,
                          const int64_t* sub_ptr, const int32_t* sub_cuts, int n_sub, int n_tiles,
                          double lr, double ru, double ri, uint64_t seed, int64_t row_base,
                          int64_t col_base, cudaStream_t stream) {
  // P rows prefetched one group ahead: 2 x U x (K/32) floats per lane in flight
  using C = RegCfg<K, Deep>;
  auto kern = qband_kernel<K, S, C::U, C::MINB>;
  const int smem = kWarps * warp_bytes;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  const int want = (n_sub + kWarps - 1) / kWarps;
  const int cap = grid_share(device_sm_count() * per_sm);
  const int grid = want < cap ? want : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kWarps * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                            sub_ptr, sub_cuts, n_sub, n_tiles, float(lr), float(ru),
                                            float(ri), seed);
  return cudaGetLastError();
}

template <typename S>
static int64_t run(S* P, S* Q, int64_t k, const int32_t* rows, const int32_t* cols,
                   const float* vals, const int64_t* sub_ptr, const int32_t* sub_cuts,
                   int64_t n_sub, int64_t n_tiles, int impl_req, double lr, double ru, double ri,
                   uint64_t seed, int64_t row_base, int64_t col_base, cudaStream_t stream) {
  if (n_sub <= 0 || n_tiles <= 0) return 0;
  if (impl_req > 6) return set_error(HMF_ERR_ARG, "impl must be -1..6");
  if (n_sub * n_tiles > (int64_t(1) << 31))
    return set_error(HMF_ERR_ARG, "n_sub * n_tiles too large");
  if (!P || !Q || !rows || !vals || !sub_ptr || !sub_cuts)
    return set_error(HMF_ERR_ARG, "null pointer");
  if (((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) != 0)
    return set_error(HMF_ERR_ARG, "factor arrays must be 16-byte aligned");
  cudaError_t e;
  const int impl = resolve_impl(impl_req, k, sizeof(S) == 2);
  // cols == nullptr: every sub-band is one item, sub_cuts[s] (chained kernel only)
  if (!cols && impl < 4)
    return set_error(HMF_ERR_ARG, "cols may be null only for implementations 4-6");
  switch (k) {
#define HMF_QB_CASE(KK)                                                                    \
  case KK:                                                                                 \
    if (impl == 2 && async_ok<KK, S>())                                                    \
      e = launch_async_if<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),    \
                                 int(n_tiles), lr, ru, ri, seed, row_base, col_base,       \
                                 stream);                                                  \
    else if (impl >= 4)                                                                    \
      e = launch_chain<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),       \
                              int(n_tiles), lr, ru, ri, seed, row_base, col_base, stream,  \
                              impl == 4 ? 0 : (impl == 5 ? 1 : 2));                        \
    else if (impl == 3)                                                                    \
      e = launch<KK, S, true>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),       \
                              int(n_tiles), lr, ru, ri, seed, row_base, col_base, stream); \
    else if (impl == 1)                                                                    \
      e = launch_tma<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub),         \
                            int(n_tiles), lr, ru, ri, seed, row_base, col_base, stream);   \
    else                                                                                   \
      e = launch<KK, S>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, int(n_sub), int(n_tiles), \
                        lr, ru, ri, seed, row_base, col_base, stream);                     \
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
                       int64_t n_sub, int64_t n_tiles, int impl_req, double lr, double ru,
                       double ri, uint64_t seed, int64_t row_base, int64_t col_base,
                       cudaStream_t stream, const int32_t* tile_row0 = nullptr) {
  if (n_sub <= 0 || n_tiles <= 0) return 0;
  if (n_sub * n_tiles > (int64_t(1) << 31))
    return set_error(HMF_ERR_ARG, "n_sub * n_tiles too large");
  if (!P || !Q || !rows || !vals || !sub_ptr || !sub_cuts)
    return set_error(HMF_ERR_ARG, "null pointer");
  if (((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) != 0)
    return set_error(HMF_ERR_ARG, "factor arrays must be 16-byte aligned");
  const int set = g_chain_cfg.load();
  const int cfg = set >= 0 ? set : auto_chain_cfg(int(k), sizeof(S) == 2);
  if (cfg != 2 && (cfg < 4 || cfg > 6))
    return set_error(HMF_ERR_UNSUPPORTED, "uint16 row ids need chain configuration 2, 4, 5 or 6");
  const int impl = resolve_impl(impl_req, k, sizeof(S) == 2);
  if (impl < 4)
    return set_error(HMF_ERR_UNSUPPORTED, "uint16 row ids need implementation 4, 5 or 6");
  const int qdelta = impl == 4 ? 0 : (impl == 5 ? 1 : 2);
  cudaError_t e;
  switch (k) {
    case 32: e = launch_chain<32, S, uint16_t>(P, Q, rows, cols, vals, sub_ptr, sub_cuts,
                                                int(n_sub), int(n_tiles), lr, ru, ri, seed,
                                                row_base, col_base, stream, qdelta, tile_row0); break;
    case 64: e = launch_chain<64, S, uint16_t>(P, Q, rows, cols, vals, sub_ptr, sub_cuts,
                                                int(n_sub), int(n_tiles), lr, ru, ri, seed,
                                                row_base, col_base, stream, qdelta, tile_row0); break;
    case 128: e = launch_chain<128, S, uint16_t>(P, Q, rows, cols, vals, sub_ptr, sub_cuts,
                                                  int(n_sub), int(n_tiles), lr, ru, ri, seed,
                                                  row_base, col_base, stream, qdelta, tile_row0); break;
    case 256: e = launch_chain<256, S, uint16_t>(P, Q, rows, cols, vals, sub_ptr, sub_cuts,
                                                  int(n_sub), int(n_tiles), lr, ru, ri, seed,
                                                  row_base, col_base, stream, qdelta, tile_row0); break;
    default: return set_error(HMF_ERR_UNSUPPORTED, "Q-band kernel needs k in {32,64,128,256}");
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return 0;
}

template <typename S>
static int warps_per_sm(int64_t k, int impl) {
  impl = resolve_impl(impl, k, sizeof(S) == 2);
  switch (k) {
#define HMF_WPS(KK)                                                                   \
  case KK:                                                                            \
    if (impl == 2 && async_ok<KK, S>()) return async_warps_per_sm_if<KK, S>();        \
    if (impl == 3) return reg_warps_per_sm<KK, S, true>();                            \
    if (impl >= 4) return chain_slots_per_sm<KK, S>();                                \
    return impl == 1 ? tma_warps_per_sm<KK, S>() : reg_warps_per_sm<KK, S>();
    HMF_WPS(32)
    HMF_WPS(64)
    HMF_WPS(128)
    HMF_WPS(256)
#undef HMF_WPS
    default: return 0;
  }
}

// Q-slice budget of the active implementation (bytes of fp32 Q per warp)
template <typename S>
static int slice_bytes(int64_t k, int impl) {
  impl = resolve_impl(impl, k, sizeof(S) == 2);
  if (impl >= 4) return 1 << 30;  // Q rows in registers: no slice bound
  if (impl != 2) return kSliceBytes;
  switch (k) {
    case 32: return async_ok<32, S>() ? AsyncLayout<32, S, 4>::SLICE : kSliceBytes;
    case 64: return async_ok<64, S>() ? AsyncLayout<64, S, 4>::SLICE : kSliceBytes;
    case 128: return async_ok<128, S>() ? AsyncLayout<128, S, 4>::SLICE : kSliceBytes;
    case 256: return async_ok<256, S>() ? AsyncLayout<256, S, 4>::SLICE : kSliceBytes;
    default: return kSliceBytes;
  }
}

}  // namespace qs
}  // namespace hmf

extern "C" {

int32_t hmf_qband_slots_per_sm(int64_t k, int32_t f16, int32_t impl) {
  return f16 ? hmf::qs::warps_per_sm<__half>(k, impl) : hmf::qs::warps_per_sm<float>(k, impl);
}

int32_t hmf_qband_warps_per_sm(int64_t k, int32_t f16) {
  return hmf_qband_slots_per_sm(k, f16, -1);
}

int32_t hmf_qband_resolve_impl(int64_t k, int32_t f16) {
  return hmf::qs::resolve_impl(-1, k, f16 != 0);
}

int32_t hmf_qband_get_impl() { return hmf::qs::g_qband_impl; }

int hmf_qband_set_chain_cfg(int32_t cfg) {
  if (cfg < -1 || cfg >= hmf::qs::kChainCfgs)
    return int(hmf::set_error(HMF_ERR_ARG, "chain configuration out of range"));
  hmf::qs::g_chain_cfg = cfg;
  return HMF_OK;
}

int hmf_qband_set_chain_lockstep(int32_t bits) {
  if (bits < 0 || bits > 3) return int(hmf::set_error(HMF_ERR_ARG, "lockstep bits must be 0..3"));
  hmf::qs::g_chain_lockstep = bits;
  return HMF_OK;
}

int hmf_qband_set_pstore(int32_t mode) {
  if (mode < -1 || mode > 1) return int(hmf::set_error(HMF_ERR_ARG, "pstore must be -1..1"));
  hmf::qs::g_chain_pstore = mode;
  return HMF_OK;
}

int32_t hmf_qband_get_pstore(void) { return hmf::qs::g_chain_pstore; }

int32_t hmf_qband_get_chain_cfg(void) { return hmf::qs::g_chain_cfg; }

int hmf_qband_set_qsync(int32_t steps) {
  if (steps < 0) return int(hmf::set_error(HMF_ERR_ARG, "qsync steps must be >= 0"));
  hmf::qs::g_qsync_steps = steps;
  return HMF_OK;
}

int hmf_qband_set_grid_share(int32_t div) {
  if (div < 1 || div > 64) return int(hmf::set_error(HMF_ERR_ARG, "grid share must be 1..64"));
  hmf::qs::g_grid_div = div;
  return HMF_OK;
}

int32_t hmf_qband_chain_lanes_for(int64_t k, int32_t f16) {
  const int set = hmf::qs::g_chain_cfg.load();
  const int cfg = set >= 0 ? set : hmf::qs::auto_chain_cfg(int(k), f16 != 0);
  if (cfg == 5 || cfg == 6) return k >= 256 ? 16 : 8;
  const int per = (cfg == 2 || cfg == 3) ? 8 : 16;  // elements per lane
  const int lpc = int(k) / per;
  return lpc < 4 ? 4 : (lpc > 32 ? 32 : lpc);
}

int32_t hmf_qband_chain_lanes(int64_t k) { return hmf_qband_chain_lanes_for(k, 0); }

int hmf_qband_set_impl(int32_t impl) {
  if (impl < -1 || impl > 6)
    return int(hmf::set_error(HMF_ERR_ARG, "impl must be -1..6"));
  hmf::qs::g_qband_impl = impl;
  return HMF_OK;
}

int32_t hmf_qband_max_items_for(int64_t k, int32_t f16, int32_t impl) {
  if (k != 32 && k != 64 && k != 128 && k != 256) return 0;
  const int b = f16 ? hmf::qs::slice_bytes<__half>(k, impl) : hmf::qs::slice_bytes<float>(k, impl);
  return b >= (1 << 30) ? int32_t(1 << 30) : int32_t(b / (k * 4));
}

int32_t hmf_qband_max_items(int64_t k) {
  // the tighter of the fp32 / fp16 budgets of the default implementation
  const int32_t a = hmf_qband_max_items_for(k, 0, -1), b = hmf_qband_max_items_for(k, 1, -1);
  return a < b ? a : b;
}

int64_t hmf_sgd_block_qband_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                                const int32_t* cols, const float* vals, const int64_t* sub_ptr,
                                const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                int32_t impl, double lr, double reg_user, double reg_item,
                                uint64_t seed, int64_t row_base, int64_t col_base, void* stream) {
  return hmf::qs::run<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                             n_tiles, impl, lr, reg_user, reg_item, seed, row_base, col_base,
                             static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                const int32_t* rows, const int32_t* cols, const float* vals,
                                const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                int64_t n_tiles, int32_t impl, double lr, double reg_user,
                                double reg_item, uint64_t seed, int64_t row_base, int64_t col_base,
                                void* stream) {
  return hmf::qs::run<__half>(reinterpret_cast<__half*>(user_f), reinterpret_cast<__half*>(item_f),
                              k, rows, cols, vals, sub_ptr, sub_cuts, n_sub, n_tiles, impl, lr,
                              reg_user, reg_item, seed, row_base, col_base,
                              static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_f32(float* user_f, float* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, int32_t impl, double lr, double reg_user,
                                    double reg_item, uint64_t seed, int64_t row_base,
                                    int64_t col_base, void* stream) {
  return hmf::qs::run_u16<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                                 n_tiles, impl, lr, reg_user, reg_item, seed, row_base, col_base,
                                 static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                    const uint16_t* rows, const int32_t* cols, const float* vals,
                                    const int64_t* sub_ptr, const int32_t* sub_cuts, int64_t n_sub,
                                    int64_t n_tiles, int32_t impl, double lr, double reg_user,
                                    double reg_item, uint64_t seed, int64_t row_base,
                                    int64_t col_base, void* stream) {
  return hmf::qs::run_u16<__half>(reinterpret_cast<__half*>(user_f),
                                  reinterpret_cast<__half*>(item_f), k, rows, cols, vals, sub_ptr,
                                  sub_cuts, n_sub, n_tiles, impl, lr, reg_user, reg_item, seed,
                                  row_base, col_base, static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_block_qband_u16_tiles_f32(float* user_f, float* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, int32_t impl, double lr,
                                          double reg_user, double reg_item, uint64_t seed,
                                          int64_t col_base, void* stream) {
  if (!tile_row0 && n_sub > 0 && n_tiles > 0) return hmf::set_error(HMF_ERR_ARG, "null pointer");
  return hmf::qs::run_u16<float>(user_f, item_f, k, rows, cols, vals, sub_ptr, sub_cuts, n_sub,
                                 n_tiles, impl, lr, reg_user, reg_item, seed, 0, col_base,
                                 static_cast<cudaStream_t>(stream), tile_row0);
}

int64_t hmf_sgd_block_qband_u16_tiles_f16(uint16_t* user_f, uint16_t* item_f, int64_t k,
                                          const uint16_t* rows, const int32_t* cols,
                                          const float* vals, const int64_t* sub_ptr,
                                          const int32_t* sub_cuts, int64_t n_sub, int64_t n_tiles,
                                          const int32_t* tile_row0, int32_t impl, double lr,
                                          double reg_user, double reg_item, uint64_t seed,
                                          int64_t col_base, void* stream) {
  if (!tile_row0 && n_sub > 0 && n_tiles > 0) return hmf::set_error(HMF_ERR_ARG, "null pointer");
  return hmf::qs::run_u16<__half>(reinterpret_cast<__half*>(user_f),
                                  reinterpret_cast<__half*>(item_f), k, rows, cols, vals, sub_ptr,
                                  sub_cuts, n_sub, n_tiles, impl, lr, reg_user, reg_item, seed, 0,
                                  col_base, static_cast<cudaStream_t>(stream), tile_row0);
}

}  // extern "C"
