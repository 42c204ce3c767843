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

#include "hmf_common.cuh"
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
};

// Configurations (hmf_qband_set_chain_cfg): lanes per chain (about 16 or 8
// fp32 elements per lane, 4..32 lanes), prefetch distance PD in steps,
// warps per CTA and CTAs per SM (register budget).
template <int K, int CFG> struct ChainCfg;
template <int K> struct ChainCfg<K, 0> {  // 16 elements/lane, 1 step ahead
  static constexpr int LPC = (K / 16) < 4 ? 4 : ((K / 16) > 32 ? 32 : (K / 16));
  static constexpr int PD = 1, WPB = 16, MINB = 1;
};
template <int K> struct ChainCfg<K, 1> {  // 16 elements/lane, 2 steps ahead
  static constexpr int LPC = ChainCfg<K, 0>::LPC;
  static constexpr int PD = 2, WPB = 16, MINB = 1;
};
template <int K> struct ChainCfg<K, 2> {  // 8 elements/lane, 3 steps ahead, 24 warps/SM
  static constexpr int LPC = (K / 8) < 4 ? 4 : ((K / 8) > 32 ? 32 : (K / 8));
  static constexpr int PD = 3, WPB = 8, MINB = 3;
};
template <int K> struct ChainCfg<K, 3> {  // 8 elements/lane, 2 steps ahead, 24 warps/SM
  static constexpr int LPC = ChainCfg<K, 2>::LPC;
  static constexpr int PD = 2, WPB = 8, MINB = 3;
};
constexpr int kChainCfgs = 4;

template <int K, typename S, int LPC, int PD, int WPB, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB)
    qchain_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const int32_t* __restrict__ rows,
                  const int32_t* __restrict__ cols, const float* __restrict__ vals,
                  const int64_t* __restrict__ sub_ptr, int n_sub, int n_tiles, float lr, float ru,
                  float ri, uint64_t seed) {
  using L = ChainLay<K, S, LPC>;
  constexpr int NC = L::NC, E = L::EPL, NS = PD + 1;
  static_assert(PD >= 1 && PD < LPC, "prefetch distance must stay within one batch");
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int c = lane / LPC, l = lane % LPC;
  const int gw = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int n_slots = gridDim.x * WPB * NC;
  const float a_ru = lr * ru, keep_q = 1.f - lr * ri;

  for (int ti = 0; ti < n_tiles; ++ti) {
    const int tile = tile_at(ti, n_tiles, seed);
    const int64_t* sp = sub_ptr + int64_t(tile) * n_sub;
    const uint64_t bin0 = uint64_t(tile) * uint64_t(n_sub);
    for (int s0 = gw * NC; s0 < n_sub; s0 += n_slots) {  // warp-uniform
      const int s = s0 + c;
      int64_t beg = 0;
      int len = 0;
      if (s < n_sub) {
        beg = sp[s];
        len = int(sp[s + 1] - beg);
      }
      // nf full batches of LPC triples visited from a seeded rotation, then
      // the partial batch (if any) last
      const int nf = len / LPC;
      const int nb = (len + LPC - 1) / LPC;
      const int rot =
          nf > 0 ? int(splitmix_finalize(seed + (bin0 + uint64_t(s)) * kGolden) % uint64_t(nf))
                 : 0;
      auto bstart = [&](int x) -> int {
        if (x >= nf) return nf * LPC;
        int b = x + rot;
        if (b >= nf) b -= nf;
        return b * LPC;
      };
      auto load_batch = [&](int x, int32_t& u, int32_t& v, float& r) {
        u = -1;
        if (x < nb) {
          const int o = bstart(x) + l;
          if (o < len) {
            u = __ldg(rows + beg + o);
            v = __ldg(cols + beg + o);
            r = __ldg(vals + beg + o);
          }
        }
      };
      int32_t cu, cv = 0, nu, nv = 0;
      float cr = 0.f, nr = 0.f;
      load_batch(0, cu, cv, cr);
      load_batch(1, nu, nv, nr);
      int x = 0, j = 0;
      int cnt = x < nf ? LPC : len - nf * LPC;  // ratings in the current batch
      float p[NS][E], q[E];
      int qcur = -1;  // item whose Q row is in q[]
      // prologue: P rows of ratings 0 .. PD-1 (all in batch 0 when it is full)
#pragma unroll
      for (int t = 0; t < PD; ++t) {
        const int32_t u0 = __shfl_sync(FULL, cu, t, LPC);
        if (t < cnt && u0 >= 0) L::ldg(Pb + int64_t(u0) * K, l, p[t]);
      }
      // one rating per chain: pc holds its P row, pn receives the row of the
      // rating PD steps ahead
      auto step = [&](float* pc, float* pn) {
        const bool act = x < nb;  // chain-uniform
        const int32_t u = __shfl_sync(FULL, cu, j, LPC);
        const int32_t v = __shfl_sync(FULL, cv, j, LPC);
        const float r = __shfl_sync(FULL, cr, j, LPC);
        const bool ahead_in = j + PD < cnt;
        const int32_t un =
            __shfl_sync(FULL, ahead_in ? cu : nu, ahead_in ? j + PD : j + PD - cnt, LPC);
        if (act && un >= 0) L::ldg(Pb + int64_t(un) * K, l, pn);
        if (act && v != qcur) {
          if (qcur >= 0) L::stg(Qb + int64_t(qcur) * K, l, q);
          L::ldg(Qb + int64_t(v) * K, l, q);
          qcur = v;
        }
        float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          d0 = fmaf(pc[e], q[e], d0);
          if (e + 1 < E) d1 = fmaf(pc[e + 1], q[e + 1], d1);
          if (e + 2 < E) d2 = fmaf(pc[e + 2], q[e + 2], d2);
          if (e + 3 < E) d3 = fmaf(pc[e + 3], q[e + 3], d3);
        }
        float d = (d0 + d1) + (d2 + d3);
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
        if (act) {
          const float a = lr * (r - d);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const float pu = pc[e], qv = q[e];
            pc[e] = fmaf(a, qv, -a_ru * pu);
            q[e] = fmaf(a, pu, keep_q * qv);
          }
          L::red(Pb + int64_t(u) * K, l, pc);
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
      while (__any_sync(FULL, x < nb)) {
#pragma unroll
        for (int t = 0; t < NS; ++t) step(p[t], p[(t + PD) % NS]);
      }
      if (qcur >= 0) L::stg(Qb + int64_t(qcur) * K, l, q);
    }
  }
}

static int g_chain_cfg = 1;

template <int K, typename S, int CFG>
static int chain_slots_per_sm_cfg() {
  using C = ChainCfg<K, CFG>;
  auto kern = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, 0);
  return per_sm * C::WPB * (32 / C::LPC);
}

template <int K, typename S>
static int chain_slots_per_sm() {
  switch (g_chain_cfg) {
    case 0: return chain_slots_per_sm_cfg<K, S, 0>();
    case 2: return chain_slots_per_sm_cfg<K, S, 2>();
    case 3: return chain_slots_per_sm_cfg<K, S, 3>();
    default: return chain_slots_per_sm_cfg<K, S, 1>();
  }
}

template <int K, typename S, int CFG>
static cudaError_t launch_chain_cfg(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                    const float* vals, const int64_t* sub_ptr, int n_sub,
                                    int n_tiles, double lr, double ru, double ri, uint64_t seed,
                                    int64_t row_base, int64_t col_base, cudaStream_t stream) {
  using C = ChainCfg<K, CFG>;
  constexpr int NC = 32 / C::LPC;
  auto kern = qchain_kernel<K, S, C::LPC, C::PD, C::WPB, C::MINB>;
  static int per_sm = 0;
  if (per_sm == 0) {
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WPB * 32, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  const int want = (n_sub + C::WPB * NC - 1) / (C::WPB * NC);
  const int cap = device_sm_count() * per_sm;
  const int grid = want < cap ? want : cap;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, C::WPB * 32, 0, stream>>>(P - row_base * K, Q - col_base * K, rows, cols, vals,
                                         sub_ptr, n_sub, n_tiles, float(lr), float(ru), float(ri),
                                         seed);
  return cudaGetLastError();
}

template <int K, typename S>
static cudaError_t launch_chain(S* P, S* Q, const int32_t* rows, const int32_t* cols,
                                const float* vals, const int64_t* sub_ptr, int n_sub, int n_tiles,
                                double lr, double ru, double ri, uint64_t seed, int64_t row_base,
                                int64_t col_base, cudaStream_t stream) {
#define HMF_CHAIN_CFG(CFG)                                                                   \
  return launch_chain_cfg<K, S, CFG>(P, Q, rows, cols, vals, sub_ptr, n_sub, n_tiles, lr, ru, \
                                     ri, seed, row_base, col_base, stream)
  switch (g_chain_cfg) {
    case 0: HMF_CHAIN_CFG(0);
    case 2: HMF_CHAIN_CFG(2);
    case 3: HMF_CHAIN_CFG(3);
    default: HMF_CHAIN_CFG(1);
  }
#undef HMF_CHAIN_CFG
}

}  // namespace qs
}  // namespace hmf
