// Chained item-run kernel (Q-band implementation 4): several independent Q
// chains per warp.
//
// The block's triples are laid out row tile major, then item major
// (data.bucket_qbands), so a (tile, sub-band) bin is a sequence of item runs.
// SGD on one item is a sequential chain (rating i+1 reads the Q row rating i
// wrote); the dot-product reduction (__shfl_xor butterfly) sits on that chain.
// With a whole warp on one rating the chain is 5 shuffle levels long and the
// warp does nothing else meanwhile.  Here a warp is split into NC = 32/LPC
// lane groups ("chains"), each owning its own sub-band and walking it one
// rating per step:
//   * the current item's Q row lives in the chain's registers (fp32, EPL =
//     K/LPC elements per lane); it is written back to Q when the item changes
//     and at the end of the bin — no shared memory at all;
//   * the P row of the next rating is prefetched one step ahead (two register
//     slots, alternated by unrolling the step loop by two);
//   * a chain's triples arrive LPC at a time as one coalesced load per array
//     (lane l holds triple l of the batch) and are broadcast with width-LPC
//     shuffles, the next batch already in flight;
//   * the dot product is reduced over log2(LPC) levels, one shuffle
//     instruction serving all NC chains at once;
//   * P deltas go back by vector reductions (red.global.add.v4.f32), as in the
//     other implementations (other chains and warps may share the user).
// All chains of a warp step together; a chain whose bin is exhausted idles
// (its lanes still join the shuffles).  Sub-band s is owned by chain
// (s mod n_slots) in every row tile, so Q stays race-free across tiles.
// The update is the reference's (kernels.py:120-131) in fp32, refactored as
// a = lr*err:  dP = a*q - (lr*reg_u)*p,  q' = (1 - lr*reg_i)*q + a*p.
#pragma once

#include <map>
#include <mutex>
#include <utility>

#include "hmf_common.cuh"
#include "hmf_internal.h"
#include "lanevec.cuh"

namespace hmf {
namespace qs {

// A K-row spread over the LPC lanes of a chain: EPL = K/LPC elements per
// lane as NV vectors of W elements; vector v of chain lane l starts at element
// (v*LPC + l)*W, so each vector instruction moves LPC*W*sizeof(S) contiguous
// bytes per chain.
template <int K, typename S, int LPC> struct ChainLay {
  static constexpr int NC = 32 / LPC;
  static constexpr int EPL = K / LPC;
  static constexpr int WMAX = 16 / int(sizeof(S));
  static constexpr int W = EPL < WMAX ? EPL : WMAX;
  static constexpr int NV = EPL / W;
  static_assert(K % LPC == 0 && EPL % W == 0, "bad chain layout");
  using V = Vec<S, W>;
  __device__ static int off(int v, int l) { return (v * LPC + l) * W; }
  __device__ static void ldg(const S* row, int l, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::ldg(row + off(v, l), o + v * W);
  }
  __device__ static void stg(S* row, int l, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::stg(row + off(v, l), i + v * W);
  }
  __device__ static void red(S* row, int l, const float* d) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::red(row + off(v, l), d + v * W);
  }
  // the same row in shared memory (storage type, same element interleave)
  __device__ static void lds(const S* row, int l, float* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::lds(row + off(v, l), o + v * W);
  }
  __device__ static void sts(S* row, int l, const float* i) {
#pragma unroll
    for (int v = 0; v < NV; ++v) V::sts(row + off(v, l), i + v * W);
  }
  // storage-typed row kept raw in registers (RW 32-bit words per lane), so a
  // prefetched fp16 row costs half the registers of its fp32 expansion
  static constexpr int VW = W * int(sizeof(S)) / 4;
  static constexpr int RW = NV * VW;
  __device__ static void ldraw(const S* row, int l, uint32_t* o) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const void* p = row + off(v, l);
      if constexpr (VW == 4) {
        const uint4 t = __ldcg(reinterpret_cast<const uint4*>(p));
        o[v * 4] = t.x; o[v * 4 + 1] = t.y; o[v * 4 + 2] = t.z; o[v * 4 + 3] = t.w;
      } else if constexpr (VW == 2) {
        const uint2 t = __ldcg(reinterpret_cast<const uint2*>(p));
        o[v * 2] = t.x; o[v * 2 + 1] = t.y;
      } else {
        o[v] = __ldcg(reinterpret_cast<const unsigned int*>(p));
      }
    }
  }
  __device__ static void cvt(const uint32_t* raw, float* o) {
    if constexpr (sizeof(S) == 4) {
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[e] = __uint_as_float(raw[e]);
    } else {
#pragma unroll
      for (int w = 0; w < RW; ++w) unpack_h2(raw[w], o + 2 * w);
    }
  }
};

// Configurations (hmf_qband_opts.chain_cfg): lanes per chain (about 8 or 16
// fp32 elements per lane, 4..32 lanes), prefetch distance PD in steps, warps
// per CTA and CTAs per SM (register budget).  Configurations 0, 1 and 3 of
// round 1 (16 elements per lane with 1-2 steps ahead; 8 elements with 2
// ahead at 24 warps) were never the fastest at any k and are gone
// (profiles/r02/chain_cfg_by_k.jsonl).
template <int K, int CFG> struct ChainCfg;
template <int K> struct ChainCfg<K, 2> {  // 8 elements/lane, 3 steps ahead, 24 warps/SM
  static constexpr int LPC = (K / 8) < 4 ? 4 : ((K / 8) > 32 ? 32 : (K / 8));
  static constexpr int PD = 3, WPB = 8, MINB = 3;
};
template <int K> struct ChainCfg<K, 4> {  // 16 elements/lane, 4 steps ahead (fp16 rows)
  static constexpr int LPC = (K / 16) < 4 ? 4 : ((K / 16) > 32 ? 32 : (K / 16));
  static constexpr int PD = LPC > 4 ? 4 : LPC - 1, WPB = 16, MINB = 1;
};
template <int K> struct ChainCfg<K, 5> {  // 8 lanes per chain (4 chains), 2 steps ahead
  static constexpr int LPC = K >= 256 ? 16 : 8;
  static constexpr int PD = 2, WPB = 16, MINB = 1;
};
template <int K> struct ChainCfg<K, 6> {  // 8 lanes per chain (4 chains), 4 steps ahead
  static constexpr int LPC = K >= 256 ? 16 : 8;
  static constexpr int PD = 4, WPB = 16, MINB = 1;
};

__device__ inline unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ inline void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Units of work are (tile step i, sub-band s) bins.  Static mode (DYN =
// false): chain g owns sub-bands g, g + n_slots, ... and walks them tile step
// by tile step.  Dynamic mode (DYN = true, `work` = zeroed {counter,
// done[n_sub]}): chains take units in order from a global counter and start
// unit (i, s) once done[s] == i, i.e. once the chain that had (i-1, s)
// released it — Q row ownership moves between chains through
// release/acquire, and load balance no longer depends on the number of
// sub-bands being a multiple of the number of chains.
template <int K, typename S, int LPC, int PD, int WPB, int MINB, bool DYN,
          typename RowT = int32_t, bool PST = false>
__global__ void __launch_bounds__(WPB * 32, MINB)
    qchain_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const RowT* __restrict__ rows,
                  const int32_t* __restrict__ cols, const float* __restrict__ vals,
                  const int64_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_cuts,
                  int n_sub, int n_tiles, const int32_t* __restrict__ tile_row0, float lr,
                  float ru, float ri, uint64_t seed, unsigned* __restrict__ work, int lockstep,
                  int qdelta, int qsync) {
  using L = ChainLay<K, S, LPC>;
  constexpr int NC = L::NC, E = L::EPL, NS = PD + 1;
  static_assert(PD >= 1 && PD < LPC, "prefetch distance must stay within one batch");
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int c = lane / LPC, l = lane % LPC;
  const unsigned cmask = LPC == 32 ? FULL : (((1u << LPC) - 1u) << (c * LPC));
  // global chain id, CTA-minor: consecutive sub-bands land on different SMs,
  // so a block with fewer sub-bands than chains still spreads over the GPU
  const int cg = ((threadIdx.x >> 5) * NC + c) * int(gridDim.x) + int(blockIdx.x);
  const int n_slots = gridDim.x * WPB * NC;
  const float a_ru = lr * ru, keep_q = 1.f - lr * ri;
  const unsigned n_units = unsigned(n_tiles) * unsigned(n_sub);

  // -- per-chain state ------------------------------------------------------
  int ui = 0, us = cg;          // current unit (tile step, sub-band)
  bool done = false;            // no units left for this chain
  bool pend = false;            // unit taken, waiting for its sub-band (dynamic)
  bool have = false;            // a bin is in progress (its Q row to write back)
  bool first = true;            // static mode: no unit taken yet
  int64_t beg = 0;
  int len = 0, nf = 0, nb = 0, rot = 0, x = 0, j = 0, cnt = 0;
  int32_t cu = -1, cv = 0, nu = -1, nv = 0;
  int32_t vbin = 0;  // the bin's item when cols == nullptr (one item per sub-band)
  int32_t tb = 0;    // the bin's tile's first row when rows are tile-relative (tile_row0)
  float cr = 0.f, nr = 0.f;
  uint32_t p[NS][L::RW];
  float q[E];
  int qcur = -1;  // item whose Q row is in q[]
  // qdelta: an item's run may be split over several chains (bins of one item
  // in different sub-bands): each chain works on its own copy of the Q row
  // and adds its change back with vector reductions, the value it loaded
  // kept in shared memory (the reference's lanes race on the staged Q band,
  // workers.py:222-266; reductions lose no update)
  extern __shared__ float q0_smem[];
  float* q0 = q0_smem + ((threadIdx.x >> 5) * NC + c) * K;
  auto q_load = [&](int item) {
    L::ldg(Qb + int64_t(item) * K, l, q);
    if (qdelta) {
#pragma unroll
      for (int v = 0; v < L::NV; ++v)
#pragma unroll
        for (int w = 0; w < L::W; ++w) q0[L::off(v, l) + w] = q[v * L::W + w];
    }
  };
  auto q_store = [&](int item) {
    if (qdelta) {
      float dq[E];
#pragma unroll
      for (int v = 0; v < L::NV; ++v)
#pragma unroll
        for (int w = 0; w < L::W; ++w) dq[v * L::W + w] = q[v * L::W + w] - q0[L::off(v, l) + w];
      L::red(Qb + int64_t(item) * K, l, dq);
    } else {
      L::stg(Qb + int64_t(item) * K, l, q);
    }
  };

  auto bstart = [&](int xx) -> int {
    if (xx >= nf) return nf * LPC;
    int b = xx + rot;
    if (b >= nf) b -= nf;
    return b * LPC;
  };
  auto load_batch = [&](int xx, int32_t& u, int32_t& v, float& r) {
    u = -1;
    if (xx < nb) {
      const int o = bstart(xx) + l;
      if (o < len) {
        u = int32_t(__ldg(rows + beg + o)) + tb;
        v = cols ? __ldg(cols + beg + o) : vbin;
        r = __ldg(vals + beg + o);
      }
    }
  };
  // set up the bin of unit (ui, us): nf full batches of LPC triples visited
  // from a seeded rotation, then the partial batch (if any) last
  auto begin_bin = [&]() {
    const int tile = tile_at(ui, n_tiles, seed);
    const int64_t* sp = sub_ptr + int64_t(tile) * n_sub;
    beg = sp[us];
    len = int(sp[us + 1] - beg);
    if (!cols) vbin = __ldg(sub_cuts + us);
    if (tile_row0) tb = __ldg(tile_row0 + tile);
    nf = len / LPC;
    nb = (len + LPC - 1) / LPC;
    const uint64_t bin = uint64_t(tile) * uint64_t(n_sub) + uint64_t(us);
    rot = nf > 0 ? int(splitmix_finalize(seed + bin * kGolden) % uint64_t(nf)) : 0;
    x = 0;
    j = 0;
    cnt = nf > 0 ? LPC : len;
    load_batch(0, cu, cv, cr);
    load_batch(1, nu, nv, nr);
    qcur = -1;
    have = true;
#pragma unroll
    for (int t = 0; t < PD; ++t) {
      const int32_t u0 = __shfl_sync(cmask, cu, t, LPC);
      if (t < cnt && u0 >= 0) L::ldraw(Pb + int64_t(u0) * K, l, p[t]);
    }
  };
  // the finished bin: Q row back, the unit released (dynamic)
  auto end_bin = [&]() {
    if (qcur >= 0) q_store(qcur);
    qcur = -1;
    have = false;
    if constexpr (DYN) {
      __syncwarp(cmask);
      if (l == 0) {
        __threadfence();
        st_release_u32(work + 1 + us, unsigned(ui + 1));
      }
    }
  };
  // take the next unit (chain-divergent); false when there is none
  auto take = [&]() -> bool {
    if constexpr (DYN) {
      unsigned w = 0;
      if (l == 0) w = atomicAdd(work, 1u);
      w = __shfl_sync(cmask, w, c * LPC);
      if (w >= n_units) return false;
      ui = int(w / unsigned(n_sub));
      us = int(w % unsigned(n_sub));
      pend = true;
      return true;
    } else {
      if (!first) us += n_slots;
      first = false;
      if (us >= n_sub) {
        us = cg;
        ++ui;
      }
      if (ui >= n_tiles || us >= n_sub) return false;
      pend = true;
      return true;
    }
  };
  // start the taken unit if its sub-band is free (never blocks: a chain
  // waiting here must not stall the other chains of its warp, one of which
  // may hold the predecessor unit)
  auto try_start = [&]() -> bool {
    if (DYN && !qdelta) {
      const unsigned f = ld_acquire_u32(work + 1 + us);  // every lane acquires
      if (!__all_sync(cmask, f == unsigned(ui))) return false;
    }
    pend = false;
    begin_bin();
    return true;
  };

  // one rating per active chain: praw holds its P row, pn receives the row of
  // the rating PD steps ahead
  auto step = [&](const uint32_t* praw, uint32_t* pn) {
    const bool act = !done && !pend && x < nb;  // chain-uniform
    const int32_t u = __shfl_sync(FULL, cu, j, LPC);
    const int32_t v = __shfl_sync(FULL, cv, j, LPC);
    const bool ahead_in = j + PD < cnt;
    const int32_t un =
        __shfl_sync(FULL, ahead_in ? cu : nu, ahead_in ? j + PD : j + PD - cnt, LPC);
    if (act && un >= 0) L::ldraw(Pb + int64_t(un) * K, l, pn);
    if (act && v != qcur) {
      if (qcur >= 0) q_store(qcur);
      q_load(v);
      qcur = v;
    }
    float pc[E];
    L::cvt(praw, pc);
    float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
    for (int e = 0; e < E; e += 4) {
      d0 = fmaf(pc[e], q[e], d0);
      if (e + 1 < E) d1 = fmaf(pc[e + 1], q[e + 1], d1);
      if (e + 2 < E) d2 = fmaf(pc[e + 2], q[e + 2], d2);
      if (e + 3 < E) d3 = fmaf(pc[e + 3], q[e + 3], d3);
    }
    // the rating joins the reduction (lane j of the chain holds it) instead
    // of a broadcast shuffle: the chain's sum is p.q - r
    float d = (d0 + d1) + (d2 + d3) - (l == j ? cr : 0.f);
#pragma unroll
    for (int o = LPC / 2; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
    if (act) {
      const float a = -lr * d;  // lr * (r - p.q)
      if constexpr (PST) {
        // the new row stored over the old, as the reference's racing lanes
        // write it (workers.py:222-266): no read-modify-write at L2; a
        // concurrent update of the same user by another chain may be lost
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float pu = pc[e], qv = q[e];
          pc[e] = pu + fmaf(a, qv, -a_ru * pu);
          q[e] = fmaf(a, pu, keep_q * qv);
        }
        L::stg(Pb + int64_t(u) * K, l, pc);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float pu = pc[e], qv = q[e];
          pc[e] = fmaf(a, qv, -a_ru * pu);
          q[e] = fmaf(a, pu, keep_q * qv);
        }
        L::red(Pb + int64_t(u) * K, l, pc);
      }
      if (j + 1 < cnt) {
        ++j;
      } else {
        ++x;
        j = 0;
        cu = nu;
        cv = nv;
        cr = nr;
        load_batch(x + 1, nu, nv, nr);
        cnt = x < nf ? LPC : len - nf * LPC;
      }
    }
  };

  auto advance = [&]() {
    // lockstep: the chains of a warp change bins together (their start-up
    // load latencies overlap) once every one of them has run out
    if (lockstep && !__all_sync(FULL, done || pend || x >= nb)) return;
    while (!done) {
      if (pend) {
        if (!try_start()) break;  // sub-band still busy: retry after the next group
      } else if (x >= nb) {
        if (have) end_bin();
        if (!take()) done = true;
      } else {
        break;  // bin in progress
      }
    }
  };
  advance();
  int group = 0;
  while (__any_sync(FULL, !done)) {
    if (__all_sync(FULL, done || pend)) __nanosleep(256);
#pragma unroll
    for (int t = 0; t < NS; ++t) step(p[t], p[(t + PD) % NS]);
    // Q deltas: every qsync step groups each chain publishes its change and
    // re-reads the row, so chains sharing an item see each other's updates
    // within a bounded window (all chains of the warp at the same step, so
    // their reloads overlap)
    if (qdelta && qsync > 0 && ++group == qsync) {
      group = 0;
      if (!done && !pend && qcur >= 0) {
        q_store(qcur);
        q_load(qcur);
      }
    }
    // chains whose bin ran out move on (bins start at slot 0 of the unrolled
    // group, so the prologue's slots are static)
    advance();
  }
}

// Per-launch options after defaults (hmf_qband_opts, resolved in
// qband_kernels.cu): nothing here is process-global, so concurrent launches
// with different layouts on different streams or threads do not interfere.
struct LaunchOpts {
  int impl;      // 0 (warp per rating), 4, 5 or 6 (chained)
  int cfg;       // chain configuration 2, 4, 5 or 6
  int pstore;    // 1: P rows written back by plain stores (fp32, cfg 5 / 6)
  int qsync;     // implementation 5: ratings between Q publications (0 = item/bin changes)
  int share;     // grid capped at 1/share of the resident CTA slots
  int lockstep;  // chains change bins together: bit 0 static, bit 1 dynamic scheduler
  int wide;      // implementation 8 at k = 32: the wide run-group configuration
};

static inline int grid_share(int cap, int share) {
  const int c = (cap + share - 1) / (share < 1 ? 1 : share);
  return c < 1 ? 1 : c;
}

// Default configuration by k and storage (measured on tiles of at most
// 65 536 users, profiles/r02/small_k_cfg.jsonl, chain_cfg_by_k.jsonl): k = 32
// 4 lanes per chain, 3 steps ahead, 24 warps per SM (cfg 2; 30.6 / 41.9 G
// upd/s fp32 / fp16 vs 28.1 / 32.0 with 16 warps, cfg 4); k = 64 fp32 8
// lanes, 3 ahead, 24 warps (cfg 2; 19.7 vs 18.5), fp16 4 lanes 4 ahead (cfg
// 4); k >= 128: 8 lanes (16 at k = 256), 2 ahead in fp32 (cfg 5, the
// register budget), 4 ahead in fp16 (cfg 6, raw fp16 slots).
static inline int auto_chain_cfg(int k, bool f16) {
  if (k <= 32) return 2;
  if (k <= 64) return f16 ? 4 : 2;
  return f16 ? 6 : 5;
}
static inline bool chain_cfg_ok(int cfg) { return cfg == 2 || (cfg >= 4 && cfg <= 6); }
static inline int chain_lanes(int k, int cfg) {
  if (cfg == 5 || cfg == 6) return k >= 256 ? 16 : 8;
  const int lpc = k / (cfg == 2 ? 8 : 16);
  return lpc < 4 ? 4 : (lpc > 32 ? 32 : lpc);
}

template <int K, typename S, int CFG>
static cudaError_t chain_slots_per_sm_cfg(int* out) {
  using C = ChainCfg<K, CFG>;
  auto kern = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB, false>;
  int per_sm = 0;
  const cudaError_t e =
      kernel_occupancy(reinterpret_cast<const void*>(kern), C::WPB * 32, 0, &per_sm);
  *out = per_sm * C::WPB * (32 / C::LPC);
  return e;
}

template <int K, typename S>
static cudaError_t chain_slots_per_sm(int cfg, int* out) {
  switch (cfg) {
    case 2: return chain_slots_per_sm_cfg<K, S, 2>(out);
    case 4: return chain_slots_per_sm_cfg<K, S, 4>(out);
    case 5: return chain_slots_per_sm_cfg<K, S, 5>(out);
    default: return chain_slots_per_sm_cfg<K, S, 6>(out);
  }
}

// Scratch of the dynamic scheduler ({counter, done[n_sub]}) per (device,
// stream): launches on one stream are ordered, so they can share it.
static cudaError_t chain_work(cudaStream_t stream, size_t words, unsigned** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<unsigned*, size_t>> bufs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto& b = bufs[{dev, stream}];
  if (b.second < words) {
    if (b.first) {
      e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return e;
      cudaFree(b.first);
      b.first = nullptr;
      b.second = 0;
    }
    e = cudaMalloc(reinterpret_cast<void**>(&b.first), words * sizeof(unsigned));
    if (e != cudaSuccess) return e;
    b.second = words;
  }
  *out = b.first;
  return cudaMemsetAsync(b.first, 0, words * sizeof(unsigned), stream);
}

template <int K, typename S, int CFG, typename RowT>
static cudaError_t launch_chain_cfg(S* P, S* Q, const RowT* rows, const int32_t* cols,
                                    const float* vals, const int64_t* sub_ptr,
                                    const int32_t* sub_cuts, int n_sub, int n_tiles,
                                    const int32_t* tile_row0, double lr, double ru, double ri,
                                    uint64_t seed, int64_t row_base, int64_t col_base,
                                    cudaStream_t stream, const LaunchOpts& o) {
  using C = ChainCfg<K, CFG>;
  constexpr int NC = 32 / C::LPC;
  // qdelta 0: whole item runs per sub-band (plain Q stores); 1: bounded
  // staleness (publish and re-read every o.qsync ratings); 2: publish at item
  // and bin changes only (whole runs per sub-band)
  const int qdelta = o.impl == 4 ? 0 : (o.impl == 5 ? 1 : 2);
  auto kstat = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB, false, RowT>;
  auto kdyn = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB, true, RowT>;
  // P write-back by plain stores (the reference's racing lanes): fp32 rows
  // with configurations 5 and 6 only (+19 % at NF k = 128 and 256, +4 % at
  // k = 64; fp16 rows and k = 32 were slower, profiles/r02/pstore*.jsonl);
  // reductions elsewhere
  if constexpr (sizeof(S) == 4 && (CFG == 5 || CFG == 6)) {
    if (o.pstore == 1) {
      kstat = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB, false, RowT, true>;
      kdyn = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB, true, RowT, true>;
    }
  }
  const int smem = qdelta ? C::WPB * NC * K * int(sizeof(float)) : 0;
  int per_sm = 0;
  cudaError_t e =
      kernel_occupancy(reinterpret_cast<const void*>(kstat), C::WPB * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  // a full grid (chains are spread CTA-minor, so even a block with few
  // sub-bands uses every SM); blocks with fewer sub-bands than CTAs need fewer
  const int cap = grid_share(device_sm_count() * per_sm, o.share);
  const int grid = n_sub < cap ? n_sub : cap;
  if (grid <= 0) return cudaSuccess;
  // more sub-bands than chains: units are handed out dynamically (a static
  // split would leave some chains with one sub-band more than others in
  // every tile)
  const bool dyn = int64_t(n_sub) > int64_t(grid) * C::WPB * NC;
  unsigned* work = nullptr;
  if (dyn) {
    e = chain_work(stream, size_t(n_sub) + 1, &work);
    if (e != cudaSuccess) return e;
    e = kernel_occupancy(reinterpret_cast<const void*>(kdyn), C::WPB * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
  }
  auto kern = dyn ? kdyn : kstat;
  const int lockstep = dyn ? (o.lockstep & 2) != 0 : (o.lockstep & 1) != 0;
  const int qsync = qdelta == 1 && o.qsync > 0 ? (o.qsync + C::PD) / (C::PD + 1) : 0;
  kern<<<grid, C::WPB * 32, smem, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                         sub_ptr, sub_cuts, n_sub, n_tiles, tile_row0, float(lr),
                                         float(ru), float(ri), seed, work, lockstep, qdelta,
                                         qsync);
  return cudaGetLastError();
}

// rows: int32 row ids, or uint16 (a row tile's ids relative to its first row:
// 2 bytes per rating on the host stream).  The tile's first row is
// tile_row0[tile] (device, n_tiles entries) or, with tile_row0 == nullptr,
// -row_base for every tile.
template <int K, typename S, typename RowT = int32_t>
static cudaError_t launch_chain(S* P, S* Q, const RowT* rows, const int32_t* cols,
                                const float* vals, const int64_t* sub_ptr,
                                const int32_t* sub_cuts, int n_sub, int n_tiles, double lr,
                                double ru, double ri, uint64_t seed, int64_t row_base,
                                int64_t col_base, cudaStream_t stream, const LaunchOpts& o,
                                const int32_t* tile_row0 = nullptr) {
#define HMF_CHAIN_CFG(CFG)                                                                     \
  return launch_chain_cfg<K, S, CFG, RowT>(P, Q, rows, cols, vals, sub_ptr, sub_cuts, n_sub,  \
                                           n_tiles, tile_row0, lr, ru, ri, seed, row_base,     \
                                           col_base, stream, o)
  switch (o.cfg) {
    case 2: HMF_CHAIN_CFG(2);
    case 4: HMF_CHAIN_CFG(4);
    case 5: HMF_CHAIN_CFG(5);
    case 6: HMF_CHAIN_CFG(6);
    default: return cudaErrorInvalidValue;
  }
#undef HMF_CHAIN_CFG
}

}  // namespace qs
}  // namespace hmf
