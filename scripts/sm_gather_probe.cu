// Per-SM random-row gather bandwidth on B200 (diagnostic, not product code).
// Question: how many SMs does an HBM-bound row gather (512-byte rows at random
// indices, the pool / segment-sum access pattern) need to approach the HBM
// peak?  That decides whether the embedding kernels could run on a small SM
// partition beside the tower's GEMMs (true FWP overlap) or must time-share.
//
// Variants, each on S SMs (one block per SM: the dynamic shared memory request
// keeps a second block off the SM):
//   ldg   : 32 warps, each lane group reads U rows with 128-bit loads (U in flight)
//   bulk  : one thread per warp issues cp.async.bulk of whole rows into a
//           per-warp shared-memory ring (R rows in flight per warp), mbarrier
//           completion; the warp sums the row from shared memory
//   pfl2  : like ldg, but every row of a 32-row chunk is first prefetched into
//           L2 with cp.async.bulk.prefetch.L2 (no registers)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_gather_probe sm_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int D = 128;           // floats per row (512 B)
constexpr int ROWB = D * 4;

__device__ __forceinline__ uint32_t hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return uint32_t(x);
}

template <int U>
__global__ void __launch_bounds__(1024) k_ldg(const float4* __restrict__ tab, int64_t nrows, int64_t per_warp,
                                            float* __restrict__ sink, int pf) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t i0 = 0; i0 < per_warp; i0 += 32) {
    const uint32_t myrow = hash(uint64_t(warp) * 1000003ull + i0 + lane) % uint32_t(nrows);
    if (pf) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tab + int64_t(myrow) * (D / 4)), "r"(ROWB) : "memory");
    for (int t0 = 0; t0 < 32; t0 += U) {
      float4 x[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t r = __shfl_sync(0xffffffffu, myrow, t0 + k);
        x[k] = __ldg(tab + int64_t(r) * (D / 4) + lane);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) { acc.x += x[k].x; acc.y += x[k].y; acc.z += x[k].z; acc.w += x[k].w; }
    }
  }
  if (acc.x == 1234.5f) sink[0] = acc.y + acc.z + acc.w;
}

// bulk: per warp a ring of R rows in shared memory; lane 0 issues the copies
template <int R>
__global__ void __launch_bounds__(1024) k_bulk(const float* __restrict__ tab, int64_t nrows, int64_t per_warp,
                                             float* __restrict__ sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  float* ring = reinterpret_cast<float*>(smem) + size_t(wib) * R * D;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(nw) * R * ROWB) + wib * R;
  if (lane == 0)
    for (int s = 0; s < R; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(bars + s))));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  float acc = 0.f;
  auto issue = [&](int64_t i) {
    const int s = int(i % R);
    const uint32_t r = hash(uint64_t(warp) * 1000003ull + i) % uint32_t(nrows);
    const uint32_t bar = uint32_t(__cvta_generic_to_shared(bars + s));
    const uint32_t dst = uint32_t(__cvta_generic_to_shared(ring + size_t(s) * D));
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(ROWB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(tab + int64_t(r) * D), "r"(ROWB), "r"(bar) : "memory");
  };
  if (lane == 0)
    for (int64_t i = 0; i < R && i < per_warp; ++i) issue(i);
  for (int64_t i = 0; i < per_warp; ++i) {
    const int s = int(i % R);
    const uint32_t bar = uint32_t(__cvta_generic_to_shared(bars + s));
    const uint32_t phase = uint32_t((i / R) & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(bar), "r"(phase) : "memory");
    const float4 v = reinterpret_cast<const float4*>(ring + size_t(s) * D)[lane];
    acc += v.x + v.y + v.z + v.w;
    __syncwarp();
    if (lane == 0 && i + R < per_warp) issue(i + R);
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t nrows = (int64_t(6) << 30) / ROWB;   // 6 GB table
  float* tab;
  float* sink;
  CK(cudaMalloc(&tab, size_t(nrows) * ROWB));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(tab, 0, size_t(nrows) * ROWB));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int smem_hold = 200 * 1024;   // one block per SM
  CK(cudaFuncSetAttribute(k_ldg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_hold));
  CK(cudaFuncSetAttribute(k_ldg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_hold));
  printf("{\"probe\": \"sm_gather\", \"rows_bytes\": %d, \"results\": [\n", ROWB);
  bool first = true;
  for (int S : {8, 16, 32, 48, 64, 96, 148}) {
    if (S > sms) continue;
    for (int variant = 0; variant < 5; ++variant) {
      const int threads = 1024;
      const int64_t per_warp = 4096;
      const int64_t rows = int64_t(S) * (threads / 32) * per_warp;
      auto launch = [&]() -> cudaError_t {
        switch (variant) {
          case 0: k_ldg<4><<<S, threads, smem_hold>>>(reinterpret_cast<float4*>(tab), nrows, per_warp, sink, 0); break;
          case 1: k_ldg<8><<<S, threads, smem_hold>>>(reinterpret_cast<float4*>(tab), nrows, per_warp, sink, 0); break;
          case 2: k_ldg<4><<<S, threads, smem_hold>>>(reinterpret_cast<float4*>(tab), nrows, per_warp, sink, 1); break;
          case 3: {
            const size_t sm = size_t(threads / 32) * 8 * ROWB + size_t(threads / 32) * 8 * 8;
            cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            k_bulk<8><<<S, threads, sm>>>(tab, nrows, per_warp, sink);
            break;
          }
          case 4: {
            const size_t sm = size_t(threads / 32) * 12 * ROWB + size_t(threads / 32) * 12 * 8;
            cudaFuncSetAttribute(k_bulk<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            k_bulk<12><<<S, threads, sm>>>(tab, nrows, per_warp, sink);
            break;
          }
        }
        return cudaGetLastError();
      };
      CK(launch());
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int rep = 0; rep < 3; ++rep) CK(launch());
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double gbs = 3.0 * double(rows) * ROWB / (ms * 1e6);
      const char* names[] = {"ldg_u4", "ldg_u8", "ldg_u4_pfl2", "bulk_ring8", "bulk_ring12"};
      printf("%s {\"sms\": %d, \"variant\": \"%s\", \"gbs\": %.1f, \"gbs_per_sm\": %.1f}", first ? " " : ",\n ", S,
             names[variant], gbs, gbs / S);
      first = false;
    }
  }
  printf("\n]}\n");
  return 0;
}
