// Tile-resident P (Q-band implementation 7): both factor rows of an update
// on chip.
//
// The chained kernel (qchain.cuh) keeps the item's Q row in registers along
// an item run and moves the user's P row through L2 on every rating: 512 B
// read + 512 B written per update at k = 128 fp32.  Its ncu profile binds on
// the SM -> L2 request path (l1tex__m_l1tex2xbar_req_cycles_active 86 %: one
// request cycle per written 32-byte sector, ~20 per update), capping it near
// 14 G updates/s.  Here the P rows never leave the SM while they are hot:
//   * the block's users are cut into tiles of at most G rows (G x k x
//     sizeof(S) <= ~208 KB), as many tiles as a multiple of the CTAs; a
//     persistent CTA (one per SM) copies a tile's P rows into shared memory,
//     trains every rating of the tile, and writes the rows back;
//   * inside a tile, ratings are sorted by item (data.bucket_qbands) and cut
//     into item sub-bands ("bins"); lane-group chains take bins from a
//     per-tile counter, walk them one rating per step with the item's Q row
//     in registers, and read / write P rows in shared memory (LDS/STS.128);
//   * Q rows are shared by all CTAs (they train the same items on other
//     tiles): a chain loads the row at the start of a run, keeps the value it
//     loaded, and at the end of the run adds its change back with vector
//     reductions (red.global.add.v4.f32) — no Q update is lost, a concurrent
//     run on the same item sees it at its next load (bounded staleness, as
//     implementation 5).  The next run's Q row is prefetched one step ahead;
//   * P rows in shared memory are the reference's racing lanes
//     (workers.py:222-266): chains of one CTA that update the same user in the
//     same step race (last store wins), as the racing stores of the chained
//     kernel do in L2.
// Per update the SM -> L2 traffic is the Q row per run (load + reduction,
// ~1 KB per run of ~4 ratings at Netflix density) plus the rating; P moves
// twice per tile (load + store), ~10 B per update.  The update arithmetic is
// the reference's (kernels.py:120-131) in fp32, as in qchain.cuh.
#pragma once

#include "hmf_common.cuh"
#include "lanevec.cuh"

namespace hmf {
namespace qs {

// lanes per chain (LPC) and warps per CTA: 8 lanes (16 fp32 elements per lane)
// at k = 64..128, 16 at k = 256, 4 at k = 32
template <int K> struct PTileCfg {
  static constexpr int LPC = K >= 256 ? 16 : (K >= 64 ? 8 : 4);
  static constexpr int WPB = 16;
};
// shared memory for one tile's P rows (the rest of the 227 KB stays free for
// the compiler's static shared memory)
constexpr int kPTileBytes = 208 * 1024;
// bins (item sub-bands) per chain and tile: dynamic hand-out keeps the tile
// barrier's idle tail short
constexpr int kPTileBinsPerChain = 4;

template <int K, typename S, int LPC, int WPB, typename RowT>
__global__ void __launch_bounds__(WPB * 32, 1)
    ptile_kernel(S* __restrict__ Pb, S* __restrict__ Qb, const RowT* __restrict__ rows,
                 const int32_t* __restrict__ cols, const float* __restrict__ vals,
                 const int64_t* __restrict__ sub_ptr, int n_sub, int n_tiles,
                 const int32_t* __restrict__ tile_cut, float lr, float ru, float ri,
                 uint64_t seed) {
  using L = ChainLay<K, S, LPC>;
  constexpr int E = L::EPL;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char ptile_smem[];
  S* tile = reinterpret_cast<S*>(ptile_smem);
  __shared__ unsigned next_bin;
  const int lane = threadIdx.x & 31, c = lane / LPC, l = lane % LPC;
  const unsigned cmask = LPC == 32 ? FULL : (((1u << LPC) - 1u) << (c * LPC));
  const float keep_p = 1.f - lr * ru, keep_q = 1.f - lr * ri;
  const float inv_keep_q = 1.f / keep_q;

  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int r0 = tile_cut[t], r1 = tile_cut[t + 1];
    const int n16 = (r1 - r0) * K * int(sizeof(S)) / 16;
    // 1. the tile's P rows -> shared memory
    {
      const int4* src = reinterpret_cast<const int4*>(Pb + int64_t(r0) * K);
      int4* dst = reinterpret_cast<int4*>(tile);
      for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldcg(src + i);
    }
    if (threadIdx.x == 0) next_bin = 0;
    __syncthreads();

    // 2. the tile's bins, chain by chain.  Each warp step trains one rating
    //    per chain; steps run in batches of LPC ratings (lane m of a chain
    //    holds rating m of the batch), unrolled, so every shuffle reads a
    //    constant lane.
    //    Q in scaled form: the chain holds qs with q = sq * qs, so the decay
    //    q' = (1 - lr*reg_i) q + a p is one FMA per element
    //    (qs += (a / sq') p, sq' = (1 - lr*reg_i) sq); q0 is the row as
    //    loaded, the run's change q - q0 goes back by vector reductions.
    const int64_t* sp = sub_ptr + int64_t(t) * n_sub;
    bool done = false;
    int64_t beg = 0;
    int len = 0, nf = 0, nb = 0, rot = 0, x = 0, cnt = 0;
    int32_t cu = -1, cv = 0, nu = -1, nv = 0;
    float cr = 0.f, nr = 0.f;
    // the row math runs on packed fp32 pairs (FFMA2 / FMUL2: two lanes of
    // fp32 work per instruction, bit-identical to scalar fmaf / fmul)
    constexpr int E2 = E / 2;
    float2 qs[E2], q0[E2], qn[E2];
    float sq = 1.f, isq = 1.f;  // q = sq * qs; isq = 1 / sq
    int qcur = -1, qnext = -1;

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
          u = int32_t(__ldg(rows + beg + o));
          v = __ldg(cols + beg + o);
          r = __ldg(vals + beg + o);
        }
      }
    };
    auto flush_q = [&]() {
      if (qcur >= 0) {
        float dq[E];
        const float2 sq2 = make_float2(sq, sq);
#pragma unroll
        for (int e = 0; e < E2; ++e) {
          const float2 d = __ffma2_rn(sq2, qs[e], make_float2(-q0[e].x, -q0[e].y));
          dq[2 * e] = d.x;
          dq[2 * e + 1] = d.y;
        }
        L::red(Qb + int64_t(qcur) * K, l, dq);
      }
      qcur = -1;
    };
    auto ldq = [&](int32_t v, float2* o) {
      float t[E];
      L::ldg(Qb + int64_t(v) * K, l, t);
#pragma unroll
      for (int e = 0; e < E2; ++e) o[e] = make_float2(t[2 * e], t[2 * e + 1]);
    };
    // take the next bin (chain-divergent); false when the tile has none left
    auto take = [&]() -> bool {
      unsigned w = 0;
      if (l == 0) w = atomicAdd(&next_bin, 1u);
      w = __shfl_sync(cmask, w, c * LPC);
      if (w >= unsigned(n_sub)) return false;
      const int s = int(w);
      beg = sp[s];
      len = int(sp[s + 1] - beg);
      nf = len / LPC;
      nb = (len + LPC - 1) / LPC;
      const uint64_t bin = uint64_t(t) * uint64_t(n_sub) + uint64_t(s);
      rot = nf > 0 ? int(splitmix_finalize(seed + bin * kGolden) % uint64_t(nf)) : 0;
      x = 0;
      cnt = nf > 0 ? LPC : len;
      qnext = -1;
      load_batch(0, cu, cv, cr);
      load_batch(1, nu, nv, nr);
      return true;
    };
    auto advance = [&]() {
      while (!done && x >= nb) {
        flush_q();
        if (!take()) done = true;
      }
    };
    advance();
    while (__any_sync(FULL, !done)) {
#pragma unroll
      for (int jj = 0; jj < LPC; ++jj) {
        const bool act = !done && jj < cnt;  // chain-uniform
        const int32_t u = __shfl_sync(FULL, cu, jj, LPC);
        const int32_t v = __shfl_sync(FULL, cv, jj, LPC);
        const float r = __shfl_sync(FULL, cr, jj, LPC);
        // the next rating (this batch's next lane, or the next batch's first)
        int32_t un = __shfl_sync(FULL, jj + 1 < LPC ? cu : nu, jj + 1 < LPC ? jj + 1 : 0, LPC);
        if (jj + 1 < LPC && jj + 1 >= cnt) un = -1;  // the batch ends here
        const int32_t vn = jj + 1 < LPC ? __shfl_sync(FULL, cv, jj + 1, LPC)
                                        : __shfl_sync(FULL, nv, 0, LPC);
        if (act && v != qcur) {  // a run starts: its Q row, prefetched if possible
          flush_q();
          if (qnext == v) {
#pragma unroll
            for (int e = 0; e < E2; ++e) qs[e] = qn[e];
          } else {
            ldq(v, qs);
          }
#pragma unroll
          for (int e = 0; e < E2; ++e) q0[e] = qs[e];
          sq = 1.f;
          isq = 1.f;
          qcur = v;
          qnext = -1;
        }
        // the run ends after this rating: start loading the next run's row
        if (act && un >= 0 && vn != v && vn != qnext) {
          ldq(vn, qn);
          qnext = vn;
        }
        float2 pc[E2];
        S* prow = tile + int64_t(act ? u - r0 : 0) * K;
        L::lds(prow, l, reinterpret_cast<float*>(pc));
        float2 da = make_float2(0.f, 0.f), db = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < E2; e += 2) {
          da = __ffma2_rn(pc[e], qs[e], da);
          if (e + 1 < E2) db = __ffma2_rn(pc[e + 1], qs[e + 1], db);
        }
        const float2 ds = __fadd2_rn(da, db);
        float d = ds.x + ds.y;
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
        if (act) {
          const float a = lr * fmaf(-sq, d, r);  // lr * (r - p.q)
          const float as = a * sq;                // p' = keep_p p + a q = keep_p p + (a sq) qs
          isq *= inv_keep_q;                      // sq' = keep_q sq
          sq *= keep_q;
          const float c = a * isq;                // qs' = qs + (a / sq') p
          // in place, no temporaries: qs' first, then
          // p' = keep_p p + (a sq) qs = (keep_p - (a sq) c) p + (a sq) qs'
          const float2 as2 = make_float2(as, as);
          const float kq = fmaf(-as, c, keep_p);
          const float2 kq2 = make_float2(kq, kq), c2 = make_float2(c, c);
#pragma unroll
          for (int e = 0; e < E2; ++e) {
            qs[e] = __ffma2_rn(c2, pc[e], qs[e]);
            pc[e] = __ffma2_rn(as2, qs[e], __fmul2_rn(kq2, pc[e]));
          }
          if constexpr (sizeof(S) == 4 && L::W == 4) {
            // fp32 rows: st.shared.v4 straight from the updated pairs
            const uint32_t a0 = smem_addr(prow);
#pragma unroll
            for (int v = 0; v < L::NV; ++v)
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                               a0 + uint32_t(L::off(v, l)) * 4u),
                           "f"(pc[2 * v].x), "f"(pc[2 * v].y), "f"(pc[2 * v + 1].x),
                           "f"(pc[2 * v + 1].y)
                           : "memory");
          } else {
            L::sts(prow, l, reinterpret_cast<const float*>(pc));
          }
        }
      }
      // next batch (chain-divergent from here)
      if (!done) {
        ++x;
        cu = nu;
        cv = nv;
        cr = nr;
        load_batch(x + 1, nu, nv, nr);
        cnt = x < nf ? LPC : len - nf * LPC;
        if (sq < 0.25f && qcur >= 0) {  // keep the scaled row in range on long runs
          const float2 sq2 = make_float2(sq, sq);
#pragma unroll
          for (int e = 0; e < E2; ++e) qs[e] = __fmul2_rn(qs[e], sq2);
          sq = 1.f;
          isq = 1.f;
        }
        advance();
      }
    }
    __syncthreads();
    // 3. the tile's P rows back to global memory
    {
      int4* dst = reinterpret_cast<int4*>(Pb + int64_t(r0) * K);
      const int4* src = reinterpret_cast<const int4*>(tile);
      for (int i = threadIdx.x; i < n16; i += blockDim.x) __stcg(dst + i, src[i]);
    }
    __syncthreads();
  }
}

}  // namespace qs
}  // namespace hmf
