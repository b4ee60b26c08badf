// FWP micro-batch partition.
// Sequential mode slices by sample id.  Clustered mode is in cluster.cu.
#include "nest_internal.cuh"

namespace nest {

__global__ void k_schedule_sequential(int B, int N, int32_t* __restrict__ perm,
                                      int32_t* __restrict__ mb_offsets) {
  const int cap = B / N;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) perm[q] = q;
  if (blockIdx.x == 0 && threadIdx.x <= N) mb_offsets[threadIdx.x] = threadIdx.x * cap;
}

void launch_cluster(Ctx& c, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz, int B, int N,
                    int32_t* perm, int32_t* mb_offsets, cudaStream_t st);

void launch_schedule(Ctx& c, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz, int B, int N, int mode,
                     int32_t* perm, int32_t* mb_offsets, cudaStream_t st) {
  if (mode == NEST_SCHED_CLUSTERED && N > 1) {
    launch_cluster(c, keys, bag_offsets, nnz, B, N, perm, mb_offsets, st);
    return;
  }
  int grid = (B + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > 148 * 8) grid = 148 * 8;
  k_schedule_sequential<<<grid, 256, 0, st>>>(B, N, perm, mb_offsets);
  NEST_LAUNCH_CHECK();
}

}  // namespace nest
