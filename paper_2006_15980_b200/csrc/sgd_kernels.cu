// Per-rating SGD update kernels: the B200 replacement for the reference's
// numba kernel `sgd_range` (hetmf/kernels.py:61-133).
//
// Update rule (hetmf/kernels.py:120-131), per rating (u, v, r):
//   err    = r - sum_f P[u,f] * Q[v,f]
//   P[u,f] = pu + lr * (err * qv - reg_user * pu)
//   Q[v,f] = qv + lr * (err * pu - reg_item * qv)      (pu, qv pre-update)
// with u = rows[i] - row_base, v = cols[i] - col_base (kernels.py:105-106).
//
// Modes:
//   HOGWILD  many warps, each lane group owns one rating at a time; rows are
//            updated lock-free: each update's deltas are added with vector
//            reductions at L2 (red.global.add.v4.f32), so concurrent updates
//            of a row never overwrite each other (reads may be stale).  The
//            B200 analogue of the reference's racing batch lanes
//            (workers.py:222-266).
//   HOGWILD_LWW  the same, written back with plain stores: last writer wins
//            per component, exactly the reference lanes' race.  Triples are
//            staged into per-warp shared-memory rings by cp.async.bulk (TMA)
//            with mbarrier completion, P/Q rows move as 16-byte vectors and the
//            dot product is a __shfl_xor butterfly.
//   ORDERED  one warp walks the reference's exact visit order (windowed
//            Fisher-Yates, kernels.py:77-119) with the same fp32 arithmetic as
//            HOGWILD: the fixed-order parity mode.
//   EXACT    the same order with the reference's arithmetic: products and a
//            serial f64 sum, f64 update, no FMA contraction, rounded to the
//            storage type on store.  Bit-identical to the reference.
#include <atomic>
#include "hmf_common.cuh"
#include "hmf_internal.h"

#include <type_traits>

namespace hmf {

// ---------------------------------------------------------------------------
// Vectorised per-rating row math shared by HOGWILD and ORDERED.
// ---------------------------------------------------------------------------
template <int K, typename S> struct RowMath {
  using G = Geo<K, S>;
  using ST = Storage<S>;
  using C = typename ST::C;

  __device__ static inline void load(const S* row, int lane_g, C* out) {
#pragma unroll
    for (int v = 0; v < G::NV; ++v) ST::load(row + (v * G::LPR + lane_g) * G::VE, out + v * G::VE);
  }
  __device__ static inline void store(S* row, int lane_g, const C* in) {
#pragma unroll
    for (int v = 0; v < G::NV; ++v) ST::store(row + (v * G::LPR + lane_g) * G::VE, in + v * G::VE);
  }
  __device__ static inline C partial_dot(const C* p, const C* q) {
    C d = C(0);
#pragma unroll
    for (int e = 0; e < G::EPL; ++e) d += p[e] * q[e];
    return d;
  }
  __device__ static inline void update(C* p, C* q, C err, C lr, C ru, C ri) {
#pragma unroll
    for (int e = 0; e < G::EPL; ++e) {
      const C pu = p[e], qv = q[e];
      p[e] = pu + lr * (err * qv - ru * pu);
      q[e] = qv + lr * (err * pu - ri * qv);
    }
  }
  // The same step as deltas (p, q overwritten with lr*(...)), for write-back
  // by vector reductions.
  __device__ static inline void delta(C* p, C* q, C err, C lr, C ru, C ri) {
#pragma unroll
    for (int e = 0; e < G::EPL; ++e) {
      const C pu = p[e], qv = q[e];
      p[e] = lr * (err * qv - ru * pu);
      q[e] = lr * (err * pu - ri * qv);
    }
  }
  __device__ static inline void red(S* row, int lane_g, const C* in) {
#pragma unroll
    for (int v = 0; v < G::NV; ++v) ST::red(row + (v * G::LPR + lane_g) * G::VE, in + v * G::VE);
  }
};

// ILP / block-shape variants of the HOGWILD kernel.  U = ratings a lane group
// keeps in flight per step; WPB = warps per block; MINB = min blocks per SM
// (bounds registers at 65536 / (32 * WPB * MINB)).  The default per (K, S) is
// picked by DefaultVariant; hmf_set_tuning(HMF_TUNE_VARIANT, v) overrides it
// for sweeps.
struct Variant { int u, wpb, minb; };
constexpr Variant kVariants[] = {
    {4, 16, 2}, {2, 16, 2}, {1, 16, 2}, {4, 8, 3}, {2, 8, 4}, {8, 8, 2}, {4, 16, 1}, {2, 32, 1},
};
constexpr int kNumVariants = int(sizeof(kVariants) / sizeof(kVariants[0]));

template <int K, typename S> struct DefaultVariant {
  static constexpr int bytes = Geo<K, S>::EPL * int(sizeof(typename Storage<S>::C));
  // rows of <= 16 bytes per lane: 4 in flight; 32 bytes: 2; more: 1
  static constexpr int index = bytes <= 16 ? 0 : (bytes <= 32 ? 1 : 2);
};

template <typename S> struct ChunkOf { static constexpr int CH = 256; };
template <> struct ChunkOf<double> { static constexpr int CH = 128; };

template <typename S> __host__ __device__ constexpr int stage_bytes() {
  return ChunkOf<S>::CH * (8 + int(sizeof(typename RatingOf<S>::T)));
}
template <typename S> __host__ __device__ constexpr int warp_smem_bytes() {
  return 2 * stage_bytes<S>() + 16;
}

// Per-warp view of one staged chunk.
template <typename S> struct Stage {
  int32_t* rows;
  int32_t* cols;
  typename RatingOf<S>::T* vals;
};

template <typename S> __device__ inline Stage<S> stage_at(unsigned char* wbase, int b) {
  constexpr int CH = ChunkOf<S>::CH;
  unsigned char* p = wbase + b * stage_bytes<S>();
  Stage<S> s;
  s.rows = reinterpret_cast<int32_t*>(p);
  s.cols = reinterpret_cast<int32_t*>(p + CH * 4);
  s.vals = reinterpret_cast<typename RatingOf<S>::T*>(p + CH * 8);
  return s;
}

// Issue the staging of triples [cbeg, cend) into stage buffer `st`.  The
// 16-byte-aligned body goes through cp.async.bulk (complete_tx on `bar`); the
// (<4 element) unaligned tail of the final chunk is copied by plain loads.
template <typename S>
__device__ inline void stage_chunk(const Stage<S>& st, uint64_t* bar, const int32_t* rows,
                                   const int32_t* cols, const typename RatingOf<S>::T* vals,
                                   int64_t cbeg, int64_t cend, bool bulk_ok, int lane) {
  using RT = typename RatingOf<S>::T;
  const int n = int(cend - cbeg);
  const int n_bulk = bulk_ok ? (n & ~3) : 0;
  if (lane == 0) {
    fence_proxy_async();  // order earlier generic reads of this buffer before the async writes
    mbar_arrive_expect_tx(bar, uint32_t(n_bulk) * uint32_t(8 + sizeof(RT)));
    if (n_bulk > 0) {
      bulk_g2s(st.rows, rows + cbeg, n_bulk * 4, bar);
      bulk_g2s(st.cols, cols + cbeg, n_bulk * 4, bar);
      bulk_g2s(st.vals, vals + cbeg, n_bulk * int(sizeof(RT)), bar);
    }
  }
  for (int i = n_bulk + lane; i < n; i += 32) {
    st.rows[i] = __ldg(rows + cbeg + i);
    st.cols[i] = __ldg(cols + cbeg + i);
    st.vals[i] = __ldg(vals + cbeg + i);
  }
}

// ---------------------------------------------------------------------------
// HOGWILD kernel, compile-time K.
// Chunks of CH triples (aligned to 4-element boundaries from a0) are visited
// in a seeded affine permutation (x -> (x*perm_a + perm_b) mod n_chunks), each
// warp taking every TW-th slot; the next chunk is staged while the current one
// is computed.  Pb / Qb are the factor bases biased by -row_base*K and
// -col_base*K so a row address is one wide multiply-add of the staged index.
// ---------------------------------------------------------------------------
template <int K, typename S, int U, int WPB, int MINB, bool ATOMIC>
__global__ void __launch_bounds__(WPB * 32, MINB)
    sgd_hogwild_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const int32_t* __restrict__ rows,
                       const int32_t* __restrict__ cols,
                       const typename RatingOf<S>::T* __restrict__ vals, int64_t start, int64_t stop,
                       typename Storage<S>::C lr, typename Storage<S>::C ru,
                       typename Storage<S>::C ri, uint64_t perm_a, uint64_t perm_b, int bulk_ok) {
  using G = Geo<K, S>;
  using M = RowMath<K, S>;
  using C = typename Storage<S>::C;
  constexpr int CH = ChunkOf<S>::CH;
  constexpr int STEP = G::RPW * U;

  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G::LPR;
  const int lane_g = lane % G::LPR;
  unsigned char* wbase = smem + warp * warp_smem_bytes<S>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + 2 * stage_bytes<S>());
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int64_t a0 = start & ~int64_t(3);
  const int64_t n_chunks = (stop - a0 + CH - 1) / CH;
  const int64_t tw = int64_t(gridDim.x) * WPB;
  const int64_t gw = int64_t(blockIdx.x) * WPB + warp;
  if (gw >= n_chunks) return;

  auto chunk_begin = [&](int64_t x) -> int64_t {
    return a0 + int64_t((uint64_t(x) * perm_a + perm_b) % uint64_t(n_chunks)) * CH;
  };

  {
    const int64_t cbeg = chunk_begin(gw);
    stage_chunk<S>(stage_at<S>(wbase, 0), &bars[0], rows, cols, vals, cbeg, min(cbeg + CH, stop),
                   bulk_ok, lane);
  }

  for (int64_t t = 0;; ++t) {
    const int64_t x = gw + t * tw;
    if (x >= n_chunks) break;
    const int b = int(t & 1);
    const int64_t xn = x + tw;
    if (xn < n_chunks) {
      const int64_t nbeg = chunk_begin(xn);
      stage_chunk<S>(stage_at<S>(wbase, b ^ 1), &bars[b ^ 1], rows, cols, vals, nbeg,
                     min(nbeg + CH, stop), bulk_ok, lane);
    }
    const int64_t cbeg = chunk_begin(x);
    const int lo = int(max(start - cbeg, int64_t(0)));
    const int hi = int(min(cbeg + CH, stop) - cbeg);
    mbar_wait(&bars[b], uint32_t((t >> 1) & 1));
    __syncwarp();
    const Stage<S> st = stage_at<S>(wbase, b);

    for (int base = lo; base < hi; base += STEP) {
      C p[U][G::EPL], q[U][G::EPL], d[U];
      int32_t ui[U], vi[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = base + j * G::RPW + grp;
        const int ii = i < hi ? i : lo;
        ui[j] = i < hi ? st.rows[ii] : -1;
        vi[j] = st.cols[ii];
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (ui[j] >= 0) {
          M::load(Pb + int64_t(ui[j]) * K, lane_g, p[j]);
          M::load(Qb + int64_t(vi[j]) * K, lane_g, q[j]);
        } else {
#pragma unroll
          for (int e = 0; e < G::EPL; ++e) p[j][e] = q[j][e] = C(0);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) d[j] = M::partial_dot(p[j], q[j]);
#pragma unroll
      for (int off = G::LPR / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int j = 0; j < U; ++j) d[j] += __shfl_xor_sync(0xffffffffu, d[j], off);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (ui[j] >= 0) {
          const int i = base + j * G::RPW + grp;
          if constexpr (ATOMIC) {
            M::delta(p[j], q[j], C(st.vals[i]) - d[j], lr, ru, ri);
            M::red(Pb + int64_t(ui[j]) * K, lane_g, p[j]);
            M::red(Qb + int64_t(vi[j]) * K, lane_g, q[j]);
          } else {
            M::update(p[j], q[j], C(st.vals[i]) - d[j], lr, ru, ri);
            M::store(Pb + int64_t(ui[j]) * K, lane_g, p[j]);
            M::store(Qb + int64_t(vi[j]) * K, lane_g, q[j]);
          }
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// HOGWILD kernel, runtime k (any factor count): one rating per warp per step,
// lane l owns elements l, l+32, ...; scalar loads.
// ---------------------------------------------------------------------------
template <typename S, bool ATOMIC>
__global__ void __launch_bounds__(256)
    sgd_hogwild_generic_kernel(S* P, S* Q, const int32_t* __restrict__ rows,
                               const int32_t* __restrict__ cols,
                               const typename RatingOf<S>::T* __restrict__ vals, int64_t start,
                               int64_t stop, int k, typename Storage<S>::C lr,
                               typename Storage<S>::C ru, typename Storage<S>::C ri,
                               int64_t row_base, int64_t col_base) {
  using ST = Storage<S>;
  using C = typename ST::C;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = start + gw; i < stop; i += tw) {
    S* prow = P + (int64_t(rows[i]) - row_base) * k;
    S* qrow = Q + (int64_t(cols[i]) - col_base) * k;
    C d = C(0);
    for (int f = lane; f < k; f += 32) d += ST::load1(prow + f) * ST::load1(qrow + f);
    d = group_sum<32>(d);
    const C err = C(vals[i]) - d;
    for (int f = lane; f < k; f += 32) {
      const C pu = ST::load1(prow + f), qv = ST::load1(qrow + f);
      if constexpr (ATOMIC) {
        ST::red1(prow + f, lr * (err * qv - ru * pu));
        ST::red1(qrow + f, lr * (err * pu - ri * qv));
      } else {
        ST::store1(prow + f, pu + lr * (err * qv - ru * pu));
        ST::store1(qrow + f, qv + lr * (err * pu - ri * qv));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ORDERED kernel: one warp, ratings in the order given by `perm` (offsets
// relative to `start`), same vectorised arithmetic as HOGWILD.
// ---------------------------------------------------------------------------
template <int K, typename S>
__global__ void __launch_bounds__(32)
    sgd_ordered_kernel(S* P, S* Q, const int32_t* __restrict__ rows,
                       const int32_t* __restrict__ cols,
                       const typename RatingOf<S>::T* __restrict__ vals,
                       const int32_t* __restrict__ perm, int64_t start, int64_t n,
                       typename Storage<S>::C lr, typename Storage<S>::C ru,
                       typename Storage<S>::C ri, int64_t row_base, int64_t col_base) {
  using G = Geo<K, S>;
  using M = RowMath<K, S>;
  using C = typename Storage<S>::C;
  const int lane = threadIdx.x & 31;
  const int lane_g = lane % G::LPR;
  const bool active = lane < G::LPR;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = start + perm[t];
    S* prow = P + (int64_t(rows[i]) - row_base) * K;
    S* qrow = Q + (int64_t(cols[i]) - col_base) * K;
    C p[G::EPL], q[G::EPL];
    if (active) {
      M::load(prow, lane_g, p);
      M::load(qrow, lane_g, q);
    } else {
#pragma unroll
      for (int e = 0; e < G::EPL; ++e) p[e] = q[e] = C(0);
    }
    C d = group_sum<G::LPR>(M::partial_dot(p, q));
    if (active) {
      M::update(p, q, C(vals[i]) - d, lr, ru, ri);
      M::store(prow, lane_g, p);
      M::store(qrow, lane_g, q);
    }
    __syncwarp();
  }
}

template <typename S>
__global__ void __launch_bounds__(32)
    sgd_ordered_generic_kernel(S* P, S* Q, const int32_t* __restrict__ rows,
                               const int32_t* __restrict__ cols,
                               const typename RatingOf<S>::T* __restrict__ vals,
                               const int32_t* __restrict__ perm, int64_t start, int64_t n, int k,
                               typename Storage<S>::C lr, typename Storage<S>::C ru,
                               typename Storage<S>::C ri, int64_t row_base, int64_t col_base) {
  using ST = Storage<S>;
  using C = typename ST::C;
  const int lane = threadIdx.x & 31;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = start + perm[t];
    S* prow = P + (int64_t(rows[i]) - row_base) * k;
    S* qrow = Q + (int64_t(cols[i]) - col_base) * k;
    C d = C(0);
    for (int f = lane; f < k; f += 32) d += ST::load1(prow + f) * ST::load1(qrow + f);
    d = group_sum<32>(d);
    const C err = C(vals[i]) - d;
    for (int f = lane; f < k; f += 32) {
      const C pu = ST::load1(prow + f), qv = ST::load1(qrow + f);
      ST::store1(prow + f, pu + lr * (err * qv - ru * pu));
      ST::store1(qrow + f, qv + lr * (err * pu - ri * qv));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// EXACT kernel: reference arithmetic.  numba types f32*f32 as an f32 product
// and promotes it into the f64 accumulator; lr/reg/err are f64, so the update
// is evaluated in f64 and rounded on store (kernels.py:123-131).
// ---------------------------------------------------------------------------
__device__ inline double exact_product(float a, float b) { return double(__fmul_rn(a, b)); }
__device__ inline double exact_product(double a, double b) { return __dmul_rn(a, b); }
__device__ inline float round_to(float, double v) { return __double2float_rn(v); }
__device__ inline double round_to(double, double v) { return v; }

template <typename S>
__global__ void __launch_bounds__(32)
    sgd_exact_kernel(S* P, S* Q, const int32_t* __restrict__ rows,
                     const int32_t* __restrict__ cols,
                     const typename RatingOf<S>::T* __restrict__ vals,
                     const int32_t* __restrict__ perm, int64_t start, int64_t n, int k, double lr,
                     double ru, double ri, int64_t row_base, int64_t col_base) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sp = reinterpret_cast<S*>(smem_raw);
  S* sq = sp + k;
  const int lane = threadIdx.x & 31;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = start + perm[t];
    S* prow = P + (int64_t(rows[i]) - row_base) * k;
    S* qrow = Q + (int64_t(cols[i]) - col_base) * k;
    for (int f = lane; f < k; f += 32) {
      sp[f] = __ldcg(prow + f);
      sq[f] = __ldcg(qrow + f);
    }
    __syncwarp();
    double err = 0.0;
    if (lane == 0) {
      double acc = 0.0;
      for (int f = 0; f < k; ++f) acc = __dadd_rn(acc, exact_product(sp[f], sq[f]));
      err = __dsub_rn(double(vals[i]), acc);
    }
    err = __shfl_sync(0xffffffffu, err, 0);
    for (int f = lane; f < k; f += 32) {
      const double pu = double(sp[f]), qv = double(sq[f]);
      const double np = __dadd_rn(pu, __dmul_rn(lr, __dsub_rn(__dmul_rn(err, qv), __dmul_rn(ru, pu))));
      const double nq = __dadd_rn(qv, __dmul_rn(lr, __dsub_rn(__dmul_rn(err, pu), __dmul_rn(ri, qv))));
      __stcg(prow + f, round_to(S(), np));
      __stcg(qrow + f, round_to(S(), nq));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Host-side launchers.
// ---------------------------------------------------------------------------
static int sm_count() { return device_sm_count(); }

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

static std::atomic<int> g_variant_override{-1};

template <int K, typename S, int U, int WPB, int MINB, bool ATOMIC>
static cudaError_t launch_hogwild_v(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                    const typename RatingOf<S>::T* vals, int64_t start,
                                    int64_t stop, double lr, double ru, double ri, uint64_t seed,
                                    int64_t row_base, int64_t col_base, cudaStream_t stream) {
  using C = typename Storage<S>::C;
  constexpr int CH = ChunkOf<S>::CH;
  auto kern = sgd_hogwild_kernel<K, S, U, WPB, MINB, ATOMIC>;
  const int smem = WPB * warp_smem_bytes<S>();
  int per_sm = 0;
  {
    const cudaError_t e =
        kernel_occupancy(reinterpret_cast<const void*>(kern), WPB * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
  }
  const int64_t a0 = start & ~int64_t(3);
  const int64_t n_chunks = (stop - a0 + CH - 1) / CH;
  const int64_t want = (n_chunks + WPB - 1) / WPB;
  const int64_t cap = int64_t(sm_count()) * per_sm;
  const int64_t grid = want < cap ? want : cap;
  // Seeded affine permutation of chunk slots: multiplier coprime with n_chunks.
  const uint64_t nc = uint64_t(n_chunks);
  uint64_t a = 1, b = 0;
  if (nc > 1) {
    a = 1 + splitmix_finalize(seed + kGolden) % (nc - 1);
    while (gcd_u64(a, nc) != 1) a = a % (nc - 1) + 1;
    b = splitmix_finalize(seed ^ kOrderSalt) % nc;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(cols) |
                         reinterpret_cast<uintptr_t>(vals)) & 15u) == 0;
  kern<<<unsigned(grid), WPB * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols,
                                                   vals, start, stop, C(lr), C(ru), C(ri), a, b,
                                                   aligned ? 1 : 0);
  return cudaGetLastError();
}

template <int K, typename S, int V, bool ATOMIC>
static cudaError_t launch_variant(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                  const typename RatingOf<S>::T* vals, int64_t start, int64_t stop,
                                  double lr, double ru, double ri, uint64_t seed, int64_t row_base,
                                  int64_t col_base, cudaStream_t stream) {
  constexpr Variant v = kVariants[V];
  return launch_hogwild_v<K, S, v.u, v.wpb, v.minb, ATOMIC>(P, Q, rows, cols, vals, start, stop,
                                                            lr, ru, ri, seed, row_base, col_base,
                                                            stream);
}

template <int K, typename S, bool ATOMIC>
static cudaError_t launch_hogwild_k(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                    const typename RatingOf<S>::T* vals, int64_t start,
                                    int64_t stop, double lr, double ru, double ri, uint64_t seed,
                                    int64_t row_base, int64_t col_base, cudaStream_t stream) {
  constexpr int DV = DefaultVariant<K, S>::index;
  // Tuning sweeps cover the fp32 kernels; other storages stay on their default.
  if constexpr (!std::is_same<S, float>::value) {
    return launch_variant<K, S, DV, ATOMIC>(P, Q, rows, cols, vals, start, stop, lr, ru, ri, seed,
                                            row_base, col_base, stream);
  } else {
    switch (g_variant_override.load() < 0 ? DV : g_variant_override.load()) {
#define HMF_VARIANT_CASE(VV)                                                                    \
  case VV:                                                                                      \
    return launch_variant<K, S, VV, ATOMIC>(P, Q, rows, cols, vals, start, stop, lr, ru, ri,    \
                                            seed, row_base, col_base, stream);
      HMF_VARIANT_CASE(0)
      HMF_VARIANT_CASE(1)
      HMF_VARIANT_CASE(2)
      HMF_VARIANT_CASE(3)
      HMF_VARIANT_CASE(4)
      HMF_VARIANT_CASE(5)
      HMF_VARIANT_CASE(6)
      HMF_VARIANT_CASE(7)
#undef HMF_VARIANT_CASE
      default: return cudaErrorInvalidValue;
    }
  }
}

template <typename S, bool ATOMIC>
static cudaError_t launch_hogwild(S* P, S* Q, int k, const int32_t* rows, const int32_t* cols,
                                  const typename RatingOf<S>::T* vals, int64_t start, int64_t stop,
                                  double lr, double ru, double ri, uint64_t seed, int64_t row_base,
                                  int64_t col_base, cudaStream_t stream) {
  const bool aligned_rows =
      ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) == 0;
  if (aligned_rows) {
    switch (k) {
#define HMF_K_CASE(KK)                                                                          \
  case KK:                                                                                      \
    return launch_hogwild_k<KK, S, ATOMIC>(P, Q, rows, cols, vals, start, stop, lr, ru, ri, seed, \
                                           row_base, col_base, stream);
      HMF_K_CASE(32)
      HMF_K_CASE(64)
      HMF_K_CASE(128)
      HMF_K_CASE(256)
#undef HMF_K_CASE
      default: break;
    }
  }
  using C = typename Storage<S>::C;
  const int64_t n = stop - start;
  const int64_t warps = n < int64_t(sm_count()) * 64 ? n : int64_t(sm_count()) * 64;
  const int64_t grid = (warps + 7) / 8;
  sgd_hogwild_generic_kernel<S, ATOMIC><<<unsigned(grid), 256, 0, stream>>>(
      P, Q, rows, cols, vals, start, stop, k, C(lr), C(ru), C(ri), row_base, col_base);
  return cudaGetLastError();
}

template <typename S>
static cudaError_t launch_ordered(S* P, S* Q, int k, const int32_t* rows, const int32_t* cols,
                                  const typename RatingOf<S>::T* vals, const int32_t* perm,
                                  int64_t start, int64_t n, double lr, double ru, double ri,
                                  int64_t row_base, int64_t col_base, cudaStream_t stream) {
  using C = typename Storage<S>::C;
  const bool aligned_rows =
      ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(Q)) & 15u) == 0;
  if (aligned_rows) {
    switch (k) {
#define HMF_ORDERED_CASE(KK)                                                                   \
  case KK:                                                                                     \
    sgd_ordered_kernel<KK, S><<<1, 32, 0, stream>>>(P, Q, rows, cols, vals, perm, start, n,     \
                                                    C(lr), C(ru), C(ri), row_base, col_base); \
    return cudaGetLastError();
      HMF_ORDERED_CASE(32)
      HMF_ORDERED_CASE(64)
      HMF_ORDERED_CASE(128)
      HMF_ORDERED_CASE(256)
#undef HMF_ORDERED_CASE
      default: break;
    }
  }
  sgd_ordered_generic_kernel<S><<<1, 32, 0, stream>>>(P, Q, rows, cols, vals, perm, start, n, k,
                                                      C(lr), C(ru), C(ri), row_base, col_base);
  return cudaGetLastError();
}

template <typename S>
static cudaError_t launch_exact(S* P, S* Q, int k, const int32_t* rows, const int32_t* cols,
                                const typename RatingOf<S>::T* vals, const int32_t* perm,
                                int64_t start, int64_t n, double lr, double ru, double ri,
                                int64_t row_base, int64_t col_base, cudaStream_t stream) {
  const size_t smem = size_t(2) * size_t(k) * sizeof(S);
  if (smem > 48 * 1024) {
    int per_sm = 0;  // sets the shared-memory opt-in on this device
    const cudaError_t e = kernel_occupancy(reinterpret_cast<const void*>(sgd_exact_kernel<S>), 32,
                                           int(smem), &per_sm);
    if (e != cudaSuccess) return e;
  }
  sgd_exact_kernel<S><<<1, 32, smem, stream>>>(P, Q, rows, cols, vals, perm, start, n, k, lr, ru,
                                               ri, row_base, col_base);
  return cudaGetLastError();
}

template <typename S>
int64_t sgd_range_impl(S* P, S* Q, int64_t k, const int32_t* rows, const int32_t* cols,
                       const typename RatingOf<S>::T* vals, int64_t start, int64_t stop, double lr,
                       double ru, double ri, uint64_t seed, int64_t row_base, int64_t col_base,
                       int32_t mode, cudaStream_t stream) {
  const int64_t n = stop - start;
  if (n <= 0) return 0;  // kernels.py:74-76: empty range processes nothing
  if (k < 1 || k > (1 << 20) || start < 0) return set_error(HMF_ERR_ARG, "bad k or start");
  if (!P || !Q || !rows || !cols || !vals) return set_error(HMF_ERR_ARG, "null pointer");
  cudaError_t e = cudaSuccess;
  if (mode == HMF_MODE_HOGWILD) {
    e = launch_hogwild<S, true>(P, Q, int(k), rows, cols, vals, start, stop, lr, ru, ri, seed,
                                row_base, col_base, stream);
  } else if (mode == HMF_MODE_HOGWILD_LWW) {
    e = launch_hogwild<S, false>(P, Q, int(k), rows, cols, vals, start, stop, lr, ru, ri, seed,
                                 row_base, col_base, stream);
  } else if (mode == HMF_MODE_ORDERED || mode == HMF_MODE_EXACT) {
    if (n > INT32_MAX) return set_error(HMF_ERR_ARG, "ordered modes take < 2^31 triples");
    if (mode == HMF_MODE_EXACT && sizeof(S) == 2)
      return set_error(HMF_ERR_UNSUPPORTED, "EXACT mode needs f32 or f64 storage");
    int32_t* perm = nullptr;
    e = cudaMallocAsync(reinterpret_cast<void**>(&perm), size_t(n) * sizeof(int32_t), stream);
    if (e != cudaSuccess) return set_cuda_error(e);
    e = launch_visit_order(n, seed, perm, stream);
    if (e == cudaSuccess) {
      if (mode == HMF_MODE_ORDERED)
        e = launch_ordered<S>(P, Q, int(k), rows, cols, vals, perm, start, n, lr, ru, ri, row_base,
                              col_base, stream);
      else
        e = launch_exact<S>(P, Q, int(k), rows, cols, vals, perm, start, n, lr, ru, ri, row_base,
                            col_base, stream);
    }
    cudaError_t e2 = cudaFreeAsync(perm, stream);
    if (e == cudaSuccess) e = e2;
  } else {
    return set_error(HMF_ERR_ARG, "unknown mode");
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return n;
}

}  // namespace hmf

extern "C" {

int hmf_set_tuning(int32_t key, int32_t value) {
  if (key == HMF_TUNE_VARIANT) {
    if (value < -1 || value >= hmf::kNumVariants)
      return int(hmf::set_error(HMF_ERR_ARG, "variant out of range"));
    hmf::g_variant_override = value;
    return HMF_OK;
  }
  return int(hmf::set_error(HMF_ERR_ARG, "unknown tuning key"));
}

int64_t hmf_sgd_range_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const float* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream) {
  return hmf::sgd_range_impl<float>(user_f, item_f, k, rows, cols, vals, start, stop, lr, reg_user,
                                    reg_item, seed, row_base, col_base, mode,
                                    static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_range_f16(uint16_t* user_f, uint16_t* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const float* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream) {
  return hmf::sgd_range_impl<__half>(reinterpret_cast<__half*>(user_f),
                                     reinterpret_cast<__half*>(item_f), k, rows, cols, vals, start,
                                     stop, lr, reg_user, reg_item, seed, row_base, col_base, mode,
                                     static_cast<cudaStream_t>(stream));
}

int64_t hmf_sgd_range_f64(double* user_f, double* item_f, int64_t k, const int32_t* rows,
                          const int32_t* cols, const double* vals, int64_t start, int64_t stop,
                          double lr, double reg_user, double reg_item, uint64_t seed,
                          int64_t row_base, int64_t col_base, int32_t mode, void* stream) {
  return hmf::sgd_range_impl<double>(user_f, item_f, k, rows, cols, vals, start, stop, lr,
                                     reg_user, reg_item, seed, row_base, col_base, mode,
                                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
