// Run groups over a tile-resident P (Q-band implementation 8).
//
// The chained kernel (qchain.cuh) keeps an item's Q row in registers along
// an item run and moves the user's P row through L2 on every rating (512 B
// read + 512 B written per update at k = 128 fp32), binding on the SM -> L2
// request path.  Here a row tile's P rows stay in shared memory while the
// tile trains.  A first version (round 2's implementation 7, since removed)
// walked item runs one rating per step, each chain changing runs on its own
// every ~4.75 ratings at Netflix density: the warp ran the run-change path
// on more than half of its steps and stalled on the next Q row's L2 load
// (38 instructions per update at 49 % issue, 14.8 G upd/s; profiles/round2/
// s3_ptile_*).
//
// Here the layout hands the kernel whole runs in groups, one run per chain
// of a warp:
//   * inside a row tile the runs (the ratings of one item, in the block's
//     shuffled order) are sorted by length, longest first, and cut into
//     groups of NC = 32 / LPC consecutive runs, so the runs of a group have
//     (nearly) the same length and chain 0 holds the longest; the warp takes
//     groups from a per-tile counter (longest first: the tile's tail is
//     short);
//   * a group is one warp-uniform loop of (longest run) steps: no per-step
//     run-change tests, the item is known per chain (no item ids on the
//     rating stream), only the user id and the rating are broadcast;
//   * groups are software-pipelined two deep: while group g trains, group
//     g+1's Q rows and first batch of ratings load (their run descriptors
//     arrived during g-1) and group g+2's run descriptors load, so neither
//     the dependent descriptor -> row loads nor the L2 latency stall a step;
//   * at a run's end each chain adds its Q change back with vector
//     reductions (red.global.add.v4.f32): no Q update is lost, concurrent
//     runs of one item in other tiles see it at their next load (bounded
//     staleness, data.TILE_RESIDENT_MAX_STALE);
//   * inside a run the visit starts at a seeded rotation (fresh every epoch).
// Chains of a CTA that update one user in the same step race on its P row in
// shared memory (last store wins: the reference's racing lanes,
// workers.py:222-266).  The update arithmetic is the reference's
// (kernels.py:120-131) in fp32, on packed fp32 pairs (FFMA2).
#pragma once

#include "hmf_common.cuh"
#include "lanevec.cuh"

namespace hmf {
namespace qs {

// shared memory for one tile's P rows (the rest of the 227 KB stays free for
// the kernel's static shared memory)
constexpr int kPTileBytes = 208 * 1024;

#ifndef RUNS_SMEM_REDUCE
#define RUNS_SMEM_REDUCE 1
#endif

// Lanes per chain (LPC) and warps per CTA, measured per (k, element size)
// (profiles/round2/s4_k256_cfg.jsonl, s4_chain_cfg.jsonl, s4_ksweep.jsonl):
// 16 elements per lane (k / 16 lanes) for k = 64-256 fp16 and k = 64-128
// fp32 (fp16 k = 64 at 4 lanes: +37 % over 8; fp32 k = 64: +14 %); k = 32
// at 4 lanes; fp32 k = 256 at 8 lanes (32 values per lane, ~190 registers)
// in 8 warps: the reduction is one shared-memory round instead of four
// shuffles, +5.6 % over 16 lanes.  More chains per SM than 128 is faster
// still (k = 32: 2 lanes +12 % fp16, 20 warps +8 % fp32) but trains worse:
// a run's Q change lands at its end, and more runs of one item in flight
// across the CTAs' tiles make those changes staler.  On the narrow
// 2 %-density blocks of test_default_layout_quality_matches_whole_runs
// (fp32 k = 32) the RMSE after 8 epochs goes 0.1222 / 0.1232 / 0.138 / 0.33
// at 16 / 17 / 18 / 20 warps (profiles/round2/s4_wpb_quality.txt).
// Wide (k = 32 only, hmf_qband_opts.runs_wide): 160 chains per SM for fp32
// (20 warps of 4-lane chains), 256 for fp16 (2-lane chains) — the faster
// shapes the staleness bound keeps off narrow blocks.
template <int K, typename S, bool Wide = false> struct RunsCfg {
  static constexpr bool kWide = K >= 256 && sizeof(S) == 4;
  static constexpr bool kMore = Wide && K == 32;
  static constexpr int kLPC = kMore ? (sizeof(S) == 2 ? 2 : 4)
                                    : (sizeof(S) == 2 ? (K <= 64 ? 4 : K / 16)
                                                      : (K >= 128 ? 8 : 4));
  static constexpr int kWPB = kWide ? 8 : (kMore && sizeof(S) == 4 ? 20 : 16);
#ifdef RUNS_EXP_K  // A/B builds (scripts/build_variant.sh): one (k, element size) overridden
  static constexpr bool kExp = K == RUNS_EXP_K && sizeof(S) == RUNS_EXP_S;
  static constexpr int LPC = kExp ? RUNS_EXP_LPC : kLPC;
  static constexpr int WPB = kExp ? RUNS_EXP_WPB : kWPB;
#else
  static constexpr int LPC = kLPC;
  static constexpr int WPB = kWPB;
#endif
};

// rows: int32 user ids (absolute, minus the tile's first row in the kernel)
// or uint16 / uint8 ids relative to the tile (the streamed forms)
template <typename RowT> __device__ inline int tile_row(RowT v, int r0) {
  if constexpr (sizeof(RowT) <= 2) {
    return int(v);
  } else {
    return int(v) - r0;
  }
}

// Row layout of a chain (ChainLay: lane l of the chain holds NV vectors of W
// elements, vector v at element (v * LPC + l) * W) with the vector order
// rotated by the chain index c.  One LDS/STS instruction of a warp touches
// vector v of every chain's row; when a chain's part of it is under 128 bytes
// (fp32 k = 32: 4 lanes x 16 B), unrotated chains would all hit the same half
// of their (128-byte aligned) rows — the same 16 banks, two wavefronts where
// one suffices.  Rotated, chains alternate halves.  P and Q rows use the same
// permutation, so the dot product and the update are unchanged.
template <int K, typename S, int LPC> struct RotLay {
  using B = ChainLay<K, S, LPC>;
  using V = typename B::V;
  static constexpr int EPL = B::EPL, W = B::W, NV = B::NV;
  static_assert((NV & (NV - 1)) == 0, "NV must be a power of two");
  // rotate only where a chain's vector is under a 128-byte line (elsewhere
  // the unrotated offsets are compile-time immediates off one base register)
  static constexpr bool ROT = NV > 1 && LPC * W * int(sizeof(S)) < 128;
  __device__ static int off(int v, int l, int c) {
    return ((ROT ? ((v + c) & (NV - 1)) : v) * LPC + l) * W;
  }
  __device__ static void ldg(const S* row, int l, int c, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::ldg(row + off(v, l, c), o + v * W);
  }
  __device__ static void red(S* row, int l, int c, const float* d) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::red(row + off(v, l, c), d + v * W);
  }
  __device__ static void lds(const S* row, int l, int c, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::lds(row + off(v, l, c), o + v * W);
  }
  __device__ static void sts(S* row, int l, int c, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::sts(row + off(v, l, c), i + v * W);
  }
};

// Rotation of run r's visit, uniform in [0, len): a 32-bit hash of (seed, r)
// scaled by len (the high half of the product).  data.run_rotation restates it.
__device__ __forceinline__ int run_rotation(uint32_t seed32, int r, int len) {
  uint32_t h = uint32_t(r) * 0x9E3779B1u ^ seed32;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return int(__umulhi(h, uint32_t(len)));
}

// A run descriptor: {first rating (offset from rows / vals), length, item,
// run index} — a 16-byte record, one load per chain per group.
template <int K, typename S, int LPC, int WPB, typename RowT>
__global__ void __launch_bounds__(WPB * 32, 1)
    runs_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const RowT* __restrict__ rows,
                const float* __restrict__ vals, const int4* __restrict__ runs,
                const int32_t* __restrict__ tile_run, const int32_t* __restrict__ tile_cut,
                int n_tiles, float lr, float ru, float ri, uint32_t seed32) {
  using L = RotLay<K, S, LPC>;
  constexpr int E = L::EPL;
  constexpr int E2 = E / 2;
  constexpr int NC = 32 / LPC;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char runs_smem[];
  S* tile = reinterpret_cast<S*>(runs_smem);
  __shared__ unsigned next_group;
  // per-warp scratch for the dot-product reduction (kSmemReduce), at 4-8
  // lanes per chain: +2-4 % for fp32; fp16 +1.6 % at 8 lanes (k = 128) but
  // -3.3 % at 4 (k = 64, profiles/round2/s4_f16_reduce_ab.jsonl)
  constexpr bool kSmemReduce =
      RUNS_SMEM_REDUCE && LPC >= 4 && LPC <= 8 && (sizeof(S) == 4 || LPC == 8);
  __shared__ __align__(16) float red_all[kSmemReduce ? WPB * 32 : 4];
  const int lane = threadIdx.x & 31, c = lane / LPC, l = lane % LPC;
  float* red = red_all + (kSmemReduce ? (threadIdx.x >> 5) * 32 : 0);
  const float keep_p = 1.f - lr * ru, keep_q = 1.f - lr * ri;
  const float inv_keep_q = 1.f / keep_q;
  const float2 neg1 = make_float2(-1.f, -1.f);
  // the P tile moves between HBM/L2 and shared memory as one TMA bulk copy
  // each way (cp.async.bulk): one thread issues it, the load completes on an
  // mbarrier, the store drains while the next tile's load waits for it to
  // have read shared memory
  __shared__ __align__(8) uint64_t tile_bar;
  uint32_t tile_phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&tile_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int r0 = tile_cut[t], r1 = tile_cut[t + 1];
    const uint32_t tile_bytes = uint32_t(r1 - r0) * uint32_t(K * sizeof(S));
    if (threadIdx.x == 0) {
      next_group = 0;
      if (tile_bytes) {
        bulk_wait_read_all();  // the previous tile's write-back has read the buffer
        mbar_arrive_expect_tx(&tile_bar, tile_bytes);
        bulk_g2s(tile, Pb + int64_t(r0) * K, tile_bytes, &tile_bar);
      }
    }
    if (tile_bytes) {
      mbar_wait(&tile_bar, tile_phase);
      tile_phase ^= 1u;
    }
    __syncthreads();
    const int run0 = tile_run[t], run1 = tile_run[t + 1];
    const unsigned n_groups = unsigned((run1 - run0 + NC - 1) / NC);

    // stage 0: the descriptor of chain c's run in the warp's next group.  All
    // four words are used (m.w = the run's own index, for its rotation): an
    // unused word would be a dead register the compiler reuses while the
    // 16-byte load is still in flight, stalling on it (write-after-write).
    // m.w < 0: no run; chain 0's m.w < 0 marks the end of the tile for the warp
    auto take_meta = [&](int4& m) {
      unsigned w = 0;
      if (lane == 0) w = atomicAdd(&next_group, 1u);
      w = __shfl_sync(FULL, w, 0);
      m = make_int4(0, 0, 0, -1);
      if (w < n_groups) {
        const int r = run0 + int(w) * NC + c;
        if (r < run1) m = __ldg(runs + r);
      }
    };
    // stage 1: its Q row and first batch (lane l: position l of the rotated run)
    float2 qn[E2];
    int32_t nbu = 0;
    float nbr = 0.f;
    int nrot = 0;
    auto stage_rows = [&](const int4& m) {
      if (m.y > 0) {
        float tq[E];
        L::ldg(Qb + int64_t(m.z) * K, l, c, tq);
#pragma unroll
        for (int e = 0; e < E2; ++e) qn[e] = make_float2(tq[2 * e], tq[2 * e + 1]);
        nrot = run_rotation(seed32, m.w, m.y);
        if (l < m.y) {
          int p = nrot + l;
          if (p >= m.y) p -= m.y;
          nbu = int32_t(__ldg(rows + m.x + p));
          nbr = __ldg(vals + m.x + p);
        }
      }
    };

    int4 m1, m2;     // descriptors of the next two groups
    take_meta(m1);
    stage_rows(m1);
    take_meta(m2);
    bool more = __shfl_sync(FULL, m1.w, 0) >= 0;
    while (more) {
      // group m1 becomes current
      const int beg = m1.x, len = m1.y, item = m1.z, rot = nrot;
      const int steps = __shfl_sync(FULL, len, 0);   // chain 0 holds the longest run
      float2 qs[E2], q0n[E2];                        // q = sq * qs; q0n = -(row as loaded)
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        qs[e] = qn[e];
        q0n[e] = __fmul2_rn(qn[e], neg1);
      }
      // the lanes hold the batch's P-row element offsets (one multiply per
      // lane and batch instead of one per step after the broadcast): +1-2 %
      // at k = 32, 64, 256 and fp16 k = 128, -0.8 % at fp32 k = 128, which
      // keeps the per-step form (profiles/round2/s4_rowoff_ab.jsonl)
      constexpr bool kRowOff = !(K == 128 && sizeof(S) == 4);
      auto rowoff = [&](int32_t v) {
        return kRowOff ? tile_row<RowT>(RowT(v), r0) * K : v;
      };
      int32_t cu = rowoff(nbu);
      float cr = nbr;
      float sq = 1.f, isq = 1.f;
      // the next batch of this run (lane l: position j0 + LPC + l); the
      // group's second batch is requested before the next groups' loads
      int32_t xu = 0;
      float xr = 0.f;
      auto load_batch = [&](int j0) {
        xu = 0;
        xr = 0.f;
        const int pos = j0 + LPC + l;
        if (pos < len) {
          int p = rot + pos;
          if (p >= len) p -= len;
          xu = int32_t(__ldg(rows + beg + p));
          xr = __ldg(vals + beg + p);
        }
      };
      load_batch(0);
      // pipeline: group m2's rows start loading, the one after it is taken
      m1 = m2;
      more = __shfl_sync(FULL, m1.w, 0) >= 0;
      stage_rows(m1);
      take_meta(m2);

      for (int j0 = 0; j0 < steps; j0 += LPC) {
        if (j0 > 0) load_batch(j0);
#pragma unroll
        for (int jj = 0; jj < LPC; ++jj) {
          if (j0 + jj >= steps) break;  // warp-uniform
          const bool act = j0 + jj < len;  // chain-uniform
          const int32_t u = __shfl_sync(FULL, cu, jj, LPC);
          S* prow = kRowOff ? tile + (act ? u : 0)
                            : tile + int64_t(act ? tile_row<RowT>(RowT(u), r0) : 0) * K;
          float2 pc[E2];
          L::lds(prow, l, c, reinterpret_cast<float*>(pc));
          float2 da = make_float2(0.f, 0.f), db = make_float2(0.f, 0.f);
#pragma unroll
          for (int e = 0; e < E2; e += 2) {
            da = __ffma2_rn(pc[e], qs[e], da);
            if (e + 1 < E2) db = __ffma2_rn(pc[e + 1], qs[e + 1], db);
          }
          const float2 ds = __fadd2_rn(da, db);
          // the rating joins the reduction instead of being broadcast: lane jj
          // of the chain holds it, so the chain's sum is p.q - r (q = sq qs)
          float d = fmaf(sq, ds.x + ds.y, l == jj ? -cr : 0.f);
          if constexpr (kSmemReduce) {
            // the chain's LPC partials through shared memory: one 128-byte
            // store for the warp and LPC/4 16-byte broadcast loads per lane
            // (3 wavefronts at LPC = 8, against 3 shuffles of ~1.5); every
            // lane sums them in the same order
            __syncwarp();
            red[lane] = d;
            __syncwarp();
            const float4* src = reinterpret_cast<const float4*>(red + c * LPC);
            float4 s = src[0];
#pragma unroll
            for (int i = 1; i < LPC / 4; ++i) {
              const float4 t = src[i];
              s.x += t.x;
              s.y += t.y;
              s.z += t.z;
              s.w += t.w;
            }
            d = (s.x + s.y) + (s.z + s.w);
          } else {
#pragma unroll
            for (int o = LPC / 2; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
          }
          if (act) {
            const float a = -lr * d;  // lr * (r - p.q)
            const float as = a * sq;
            isq *= inv_keep_q;
            sq *= keep_q;
            const float cq = a * isq;
            // in place: qs' = qs + (a / sq') p, then
            // p' = keep_p p + (a sq) qs = (keep_p - (a sq) cq) p + (a sq) qs'
            const float kq = fmaf(-as, cq, keep_p);
            const float2 as2 = make_float2(as, as), kq2 = make_float2(kq, kq);
            const float2 c2 = make_float2(cq, cq);
#pragma unroll
            for (int e = 0; e < E2; ++e) {
              qs[e] = __ffma2_rn(c2, pc[e], qs[e]);
              pc[e] = __ffma2_rn(as2, qs[e], __fmul2_rn(kq2, pc[e]));
            }
            if constexpr (sizeof(S) == 4 && L::W == 4) {
              const uint32_t a0 = smem_addr(prow);
#pragma unroll
              for (int v = 0; v < L::NV; ++v)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 a0 + uint32_t(L::off(v, l, c)) * 4u),
                             "f"(pc[2 * v].x), "f"(pc[2 * v].y), "f"(pc[2 * v + 1].x),
                             "f"(pc[2 * v + 1].y)
                             : "memory");
            } else {
              L::sts(prow, l, c, reinterpret_cast<const float*>(pc));
            }
          }
        }
        cu = rowoff(xu);
        cr = xr;
        if (sq < 0.25f) {  // keep the scaled row in range on long runs
          const float2 sq2 = make_float2(sq, sq);
#pragma unroll
          for (int e = 0; e < E2; ++e) qs[e] = __fmul2_rn(qs[e], sq2);
          sq = 1.f;
          isq = 1.f;
        }
      }
      // the run's Q change back (vector reductions): q - q0 = sq * qs + q0n
      if (len > 0) {
        float dq[E];
        const float2 sq2 = make_float2(sq, sq);
#pragma unroll
        for (int e = 0; e < E2; ++e) {
          const float2 dd = __ffma2_rn(sq2, qs[e], q0n[e]);
          dq[2 * e] = dd.x;
          dq[2 * e + 1] = dd.y;
        }
        L::red(Qb + int64_t(item) * K, l, c, dq);
      }
    }
    // the chains' shared-memory writes, then the bulk write-back (async
    // proxy) of the tile: every writer fences its generic-proxy stores first
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && tile_bytes) {
      bulk_s2g(Pb + int64_t(r0) * K, tile, tile_bytes);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

}  // namespace qs
}  // namespace hmf
