// L2 random-row microbenchmark: the memory pattern of the Q-band kernels
// without their arithmetic.  Every warp-instruction touches 4 random rows of
// ROWB bytes (8 lanes x 16 B per row, like a chain of implementation 4) in a
// buffer that fits in L2, and either loads them (ld.global.cg), adds to them
// (red.global.add.v4.f32), or both.  Reports rows/s per mode, the ceiling
// for "P row read + P delta reduction" at a given row size.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_rowbench l2_rowbench.cu
//   ./l2_rowbench [buffer_MB]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// MODE 0 = load, 1 = red, 2 = load + red of the loaded values' negation,
// 3 = f16x2 red, 4 = load + f16x2 red, 5 = store, 6 = load + store of the
// loaded values scaled (the P write-back by plain stores).
// LPR lanes per row; lane l of a row group moves NV = ROWB/(16*LPR) 16-byte
// vectors at byte offsets (v*LPR + l)*16 (the chain layout of qchain.cuh).
template <int MODE, int ROWB, int DEPTH, int LPR>
__global__ void __launch_bounds__(512, 1) rowbench(float* buf, uint32_t n_rows, int iters,
                                                  float* sink) {
  constexpr int NV = ROWB / (16 * LPR);
  const int lane = threadIdx.x & 31;
  const int l = lane % LPR;
  uint32_t seed = (blockIdx.x * blockDim.x + threadIdx.x) / LPR * 7919u + 17u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[DEPTH][NV];
    uint32_t r[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      r[d] = hash32(seed + uint32_t(it * DEPTH + d) * 0x9E3779B9u) % n_rows;
      const float4* p = reinterpret_cast<const float4*>(buf + size_t(r[d]) * (ROWB / 4));
#pragma unroll
      for (int w = 0; w < NV; ++w)
        if (MODE != 1 && MODE != 3 && MODE != 5) v[d][w] = __ldcg(p + w * LPR + l);
    }
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
#pragma unroll
      for (int w = 0; w < NV; ++w) {
        float* p = buf + size_t(r[d]) * (ROWB / 4) + 4 * (w * LPR + l);
        if (MODE == 0) {
          acc += v[d][w].x + v[d][w].y + v[d][w].z + v[d][w].w;
        } else if (MODE >= 5) {
          float4 o = MODE == 6 ? v[d][w] : make_float4(1e-30f, 1e-30f, 1e-30f, 1e-30f);
          if (MODE == 6) { o.x *= 0.999f; o.y *= 0.999f; o.z *= 0.999f; o.w *= 0.999f; }
          __stcg(reinterpret_cast<float4*>(p), o);
        } else if (MODE >= 3) {  // fp16 rows: 8 halves per 16-byte vector
          const unsigned a = MODE == 4 ? (__float_as_uint(v[d][w].x) & 0x00010001u) : 0x00010001u;
          asm volatile("red.global.add.noftz.v4.f16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a),
                       "r"(a), "r"(a), "r"(a)
                       : "memory");
        } else {
          const float a = MODE == 2 ? -1e-30f * v[d][w].x : 1e-30f;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(a),
                       "f"(a), "f"(a)
                       : "memory");
        }
      }
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

// Bulk-reduction mode: each warp adds a ROWB-byte shared-memory row into
// DEPTH random rows per iteration with cp.reduce.async.bulk (the TMA unit),
// optionally loading the rows first (LOAD).  One lane issues; bulk groups are
// drained every iteration.
template <int ROWB, int DEPTH, bool LOAD>
__global__ void __launch_bounds__(512, 1) bulkbench(float* buf, uint32_t n_rows, int iters,
                                                   float* sink) {
  __shared__ __align__(128) float src[16][ROWB / 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < ROWB / 4; i += 32) src[warp][i] = 1e-30f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  uint32_t seed = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 7919u + 17u;
  const uint32_t saddr = static_cast<uint32_t>(__cvta_generic_to_shared(&src[warp][0]));
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) r[d] = hash32(seed + uint32_t(it * DEPTH + d) * 0x9E3779B9u) % n_rows;
    if (LOAD) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(buf + size_t(r[d]) * (ROWB / 4)) + (lane % (ROWB / 16)));
        acc += v.x;
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        float* dst = buf + size_t(r[d]) * (ROWB / 4);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     ::"l"(dst), "r"(saddr), "n"(ROWB) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.f) sink[0] = acc;
}

template <int ROWB, int DEPTH, bool LOAD>
static void run_bulk(float* buf, uint32_t n_rows, float* sink, int sms) {
  const int iters = 400, blocks = sms, threads = 512;
  bulkbench<ROWB, DEPTH, LOAD><<<blocks, threads>>>(buf, n_rows, 4, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bulkbench<ROWB, DEPTH, LOAD><<<blocks, threads>>>(buf, n_rows, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double rows = double(blocks) * threads / 32 * iters * DEPTH;
  printf("{\"mode\": \"%s\", \"row_bytes\": %d, \"depth\": %d, \"lanes_per_row\": 32, "
         "\"rows_per_s\": %.4g, \"GBps_rowbytes\": %.1f}\n",
         LOAD ? "load+bulkred" : "bulkred", ROWB, DEPTH, rows / (ms * 1e-3),
         rows * ROWB / (ms * 1e-3) / 1e9);
}

template <int MODE, int ROWB, int DEPTH, int LPR>
static void run(float* buf, uint32_t n_rows, float* sink, int sms) {
  const int iters = 400;
  const int blocks = sms, threads = 512;
  rowbench<MODE, ROWB, DEPTH, LPR><<<blocks, threads>>>(buf, n_rows, 4, sink);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  rowbench<MODE, ROWB, DEPTH, LPR><<<blocks, threads>>>(buf, n_rows, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double rows = double(blocks) * threads / LPR * iters * DEPTH;
  printf("{\"mode\": \"%s\", \"row_bytes\": %d, \"depth\": %d, \"lanes_per_row\": %d, "
         "\"rows_per_s\": %.4g, \"GBps_rowbytes\": %.1f}\n",
         MODE == 0 ? "load" : MODE == 1 ? "red" : MODE == 2 ? "load+red" : MODE == 3 ? "red_f16x2"
                         : MODE == 4 ? "load+red_f16x2" : MODE == 5 ? "store" : "load+store",
         ROWB, DEPTH, LPR, rows / (ms * 1e-3),
         rows * ROWB / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? size_t(atoi(argv[1])) : 32;
  float* buf;
  float* sink;
  cudaMalloc(&buf, mb << 20);
  cudaMalloc(&sink, 16);
  cudaMemset(buf, 0, mb << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"buffer_MB\": %zu, \"sms\": %d}\n", mb, sms);
#define RUN5(RB, D, LPR)                                         \
  run<0, RB, D, LPR>(buf, uint32_t((mb << 20) / RB), sink, sms); \
  run<1, RB, D, LPR>(buf, uint32_t((mb << 20) / RB), sink, sms); \
  run<2, RB, D, LPR>(buf, uint32_t((mb << 20) / RB), sink, sms); \
  run<3, RB, D, LPR>(buf, uint32_t((mb << 20) / RB), sink, sms); \
  run<4, RB, D, LPR>(buf, uint32_t((mb << 20) / RB), sink, sms);
  // 8 lanes per row (the chain layout), rows of 128 B .. 1 KB
  RUN5(128, 4, 8)
  RUN5(128, 8, 8)
  RUN5(256, 4, 8)
  RUN5(256, 8, 8)
  RUN5(512, 4, 8)
  RUN5(512, 8, 8)
  RUN5(1024, 4, 8)
  // whole-warp rows (the warp-per-rating layout)
  RUN5(512, 4, 32)
  // deeper in-flight windows (the 8-lane chain layout)
  run<2, 512, 16, 8>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run<2, 512, 32, 8>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run<2, 256, 16, 8>(buf, uint32_t((mb << 20) / 256), sink, sms);
  run<4, 256, 16, 8>(buf, uint32_t((mb << 20) / 256), sink, sms);
  run<2, 1024, 8, 8>(buf, uint32_t((mb << 20) / 1024), sink, sms);
  // plain stores, alone and after the load (P write-back by stores)
  run<5, 512, 4, 8>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run<6, 512, 4, 8>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run<6, 512, 8, 8>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run<6, 1024, 4, 8>(buf, uint32_t((mb << 20) / 1024), sink, sms);
  run<6, 1024, 8, 8>(buf, uint32_t((mb << 20) / 1024), sink, sms);
  run<6, 256, 4, 8>(buf, uint32_t((mb << 20) / 256), sink, sms);
  run<6, 256, 8, 8>(buf, uint32_t((mb << 20) / 256), sink, sms);
  // TMA bulk reductions
  run_bulk<512, 4, false>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run_bulk<512, 8, false>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run_bulk<512, 4, true>(buf, uint32_t((mb << 20) / 512), sink, sms);
  run_bulk<512, 8, true>(buf, uint32_t((mb << 20) / 512), sink, sms);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
