// Probe (not product code): NVLink row-copy bandwidth of SM-driven remote
// stores (push) vs remote loads (pull), 512-byte rows at random indices, all
// GPUs exchanging with all others at once.  nvcc -O3 -arch=sm_100a p2p_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void push_rows(const float4* __restrict__ src, float4* const* __restrict__ dst, int ndst,
                          const int* __restrict__ idx, long rows_per_dst) {
  const long nthreads = long(gridDim.x) * blockDim.x;
  const long total = rows_per_dst * ndst * 32;
  for (long t = long(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += nthreads) {
    const long r = t / 32, lane = t % 32;
    const int p = int(r / rows_per_dst);
    const long rr = r % rows_per_dst;
    dst[p][rr * 32 + lane] = src[long(idx[rr]) * 32 + lane];
  }
  __threadfence_system();
}

__global__ void pull_rows(float4* __restrict__ dst, const float4* const* __restrict__ src, int nsrc,
                          const int* __restrict__ idx, long rows_per_src) {
  const long nthreads = long(gridDim.x) * blockDim.x;
  const long total = rows_per_src * nsrc * 32;
  for (long t = long(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += nthreads) {
    const long r = t / 32, lane = t % 32;
    const int p = int(r / rows_per_src);
    const long rr = r % rows_per_src;
    dst[r * 32 + lane] = src[p][long(idx[rr]) * 32 + lane];
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const long rows = 1 << 20;  // rows per peer pair, 512 MB
  std::vector<float4*> buf(n), land(n);
  std::vector<int*> idx(n);
  std::vector<float4**> ptrs(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    for (int e = 0; e < n; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaMalloc(&buf[d], rows * 512 * 2);
    cudaMalloc(&land[d], rows * 512 * (n - 1));
    cudaMalloc(&idx[d], rows * sizeof(int));
    std::vector<int> h(rows);
    for (long i = 0; i < rows; ++i) h[i] = int((i * 2654435761ull) % (2 * rows));
    cudaMemcpy(idx[d], h.data(), rows * sizeof(int), cudaMemcpyHostToDevice);
    cudaMalloc(&ptrs[d], sizeof(float4*) * n);
  }
  for (int mode = 0; mode < 2; ++mode) {
    for (int d = 0; d < n; ++d) {
      std::vector<float4*> p;
      for (int e = 0; e < n; ++e)
        if (e != d) p.push_back(mode == 0 ? land[e] + long(d < e ? d : d - 1) * rows * 32 : buf[e]);
      cudaSetDevice(d);
      cudaMemcpy(ptrs[d], p.data(), sizeof(float4*) * p.size(), cudaMemcpyHostToDevice);
    }
    std::vector<cudaEvent_t> e0(n), e1(n);
    for (int rep = 0; rep < 3; ++rep) {
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
      }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
        cudaEventRecord(e0[d]);
        if (mode == 0)
          push_rows<<<148 * 8, 256>>>(buf[d], ptrs[d], n - 1, idx[d], rows);
        else
          pull_rows<<<148 * 8, 256>>>(land[d], ptrs[d], n - 1, idx[d], rows);
        cudaEventRecord(e1[d]);
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventSynchronize(e1[d]);
        float ms;
        cudaEventElapsedTime(&ms, e0[d], e1[d]);
        worst = ms > worst ? ms : worst;
      }
      const double bytes = double(rows) * 512 * (n - 1);
      if (rep == 2)
        printf("%s: %d GPUs, %.1f MB per GPU to/from %d peers: %.3f ms, %.1f GB/s per GPU per direction\n",
               mode == 0 ? "push (remote stores)" : "pull (remote loads)", n, bytes / 1e6, n - 1, worst,
               bytes / (worst * 1e6));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
