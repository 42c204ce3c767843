// Shared device helpers for libhmf (sm_100a).
//
// Storage traits, 16-byte vector loads/stores of factor rows, the splitmix64
// step used by the reference visit order, and the cp.async.bulk / mbarrier
// wrappers that stage rating triples into shared memory.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace hmf {

// ---------------------------------------------------------------------------
// Storage traits: factor values are stored as S (float, __half or double) and
// computed in C (float for float/__half storage, double for double storage).
// V is one 16-byte vector of S; VE is how many S fit in it.
// ---------------------------------------------------------------------------
template <typename S> struct Storage;

template <> struct Storage<float> {
  using C = float;
  static constexpr int VE = 4;
  __device__ static inline void load(const float* p, C* out) {
    float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
  __device__ static inline void store(float* p, const C* in) {
    __stcg(reinterpret_cast<float4*>(p), make_float4(in[0], in[1], in[2], in[3]));
  }
  __device__ static inline C load1(const float* p) { return __ldcg(p); }
  __device__ static inline void store1(float* p, C v) { __stcg(p, v); }
  // p[0..3] += in[0..3], one vector reduction at L2 (REDG.E.ADD.F32x4)
  __device__ static inline void red(float* p, const C* in) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(in[0]), "f"(in[1]),
                 "f"(in[2]), "f"(in[3])
                 : "memory");
  }
  __device__ static inline void red1(float* p, C v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
  }
};

template <> struct Storage<__half> {
  using C = float;
  static constexpr int VE = 8;
  __device__ static inline void load(const __half* p, C* out) {
    uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(h[i]);
      out[2 * i] = f.x; out[2 * i + 1] = f.y;
    }
  }
  __device__ static inline void store(__half* p, const C* in) {
    uint4 v;
    __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(in[2 * i], in[2 * i + 1]);
    __stcg(reinterpret_cast<uint4*>(p), v);
  }
  __device__ static inline C load1(const __half* p) {
    unsigned short raw = __ldcg(reinterpret_cast<const unsigned short*>(p));
    return __half2float(__ushort_as_half(raw));
  }
  __device__ static inline void store1(__half* p, C v) {
    __stcg(reinterpret_cast<unsigned short*>(p), __half_as_ushort(__float2half_rn(v)));
  }
  // p[0..7] += in[0..7]: one 16-byte vector reduction (REDG.E.ADD.F16x8)
  __device__ static inline void red(__half* p, const C* in) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(in[2 * i], in[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    asm volatile("red.global.add.noftz.v4.f16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
  __device__ static inline void red1(__half* p, C v) {
    asm volatile("red.global.add.noftz.f16 [%0], %1;" ::"l"(p),
                 "h"(__half_as_ushort(__float2half_rn(v)))
                 : "memory");
  }
};

template <> struct Storage<double> {
  using C = double;
  static constexpr int VE = 2;
  __device__ static inline void load(const double* p, C* out) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    out[0] = v.x; out[1] = v.y;
  }
  __device__ static inline void store(double* p, const C* in) {
    __stcg(reinterpret_cast<double2*>(p), make_double2(in[0], in[1]));
  }
  __device__ static inline C load1(const double* p) { return __ldcg(p); }
  __device__ static inline void store1(double* p, C v) { __stcg(p, v); }
  __device__ static inline void red(double* p, const C* in) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(in[0]) : "memory");
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + 1), "d"(in[1]) : "memory");
  }
  __device__ static inline void red1(double* p, C v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
  }
};

// Rating value type paired with each storage type (f64 storage keeps f64
// ratings, the reduced-precision storages keep f32 ratings: 12-byte triples).
template <typename S> struct RatingOf { using T = float; };
template <> struct RatingOf<double> { using T = double; };

// ---------------------------------------------------------------------------
// Row geometry for a compile-time factor count K: a rating is handled by LPR
// lanes (a lane group), each holding NV 16-byte vectors of the P row and of
// the Q row; a warp therefore works on RPW ratings per step.
// ---------------------------------------------------------------------------
template <int K, typename S> struct Geo {
  static constexpr int VE = Storage<S>::VE;
  static constexpr int LPR = (K / VE) < 32 ? (K / VE) : 32;
  static constexpr int NV = K / (VE * LPR);
  static constexpr int RPW = 32 / LPR;
  static constexpr int EPL = NV * VE;  // elements per lane per row
  static_assert(K % VE == 0, "K must be a multiple of the vector width");
  static_assert(LPR * NV * VE == K, "row split must cover K exactly");
};

// Sum over the LPR lanes of an aligned lane group (butterfly, all lanes end
// with the total).
template <int LPR, typename C> __device__ inline C group_sum(C v) {
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// ---------------------------------------------------------------------------
// splitmix64, exactly as the reference visit order uses it
// (hetmf/kernels.py:51-58, state seeded at kernels.py:77).
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixB = 0x94D049BB133111EBull;
constexpr uint64_t kOrderSalt = 0xD1B54A32D192ED03ull;
constexpr int kShuffleWindow = 4096;  // hetmf/kernels.py:24

__host__ __device__ inline uint64_t splitmix_finalize(uint64_t z) {
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}

// z value of the t-th _rand_step call (t >= 1) from initial state s0.
__host__ __device__ inline uint64_t rand_z(uint64_t s0, uint64_t t) {
  return splitmix_finalize(s0 + t * kGolden);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA 1-D) wrappers.
// ---------------------------------------------------------------------------
__device__ inline uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ inline void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ inline void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Copy `bytes` (multiple of 16, both addresses 16-byte aligned) from shared
// to global memory as one bulk-group operation (commit + wait below).
__device__ inline void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ inline void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Prefetch `bytes` (multiple of 16, 16-byte aligned) of global memory into L2.
__device__ inline void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// the committed bulk stores have read their shared-memory source
__device__ inline void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// the committed bulk stores are complete (globally visible)
__device__ inline void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Copy `bytes` (multiple of 16, both addresses 16-byte aligned) from global to
// shared memory, completing on `bar` via complete_tx.
__device__ inline void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

}  // namespace hmf
