// FWP key-centric sample clustering ("group samples that share
// more sparse keys into the same micro-batch").  The paper gives only the
// objective; this is the round-based parallel greedy of SURVEY §8(c)
// (reading R-CLUSTER), bit-identical to oracle/cluster.py:
//   seeds:  g=0 the largest sample; g>0 the unassigned sample with the least
//           overlap with earlier seeds, then largest, then lowest id;
//   rounds: q_r from the u64 fixed-point x1.25 schedule; snapshot
//           S[s][g] = |keys(s) & union(g)|; for g = 0..N-1 take
//           min(cap - have_g, q_r) unassigned samples by (S desc,
//           size - S asc, id asc); unions grow after the round.
// Layout: distinct keys of a sample are marked by a "first occurrence" flag
// (stable radix sort of (key id, occurrence)), union membership is a per-key
// bit mask, each round is S-kernel -> single-block select -> union update.
// The host knows every round's admission sizes in advance (they depend only on
// B and N), so no host sync is needed.
#include "nest_internal.cuh"

namespace nest {

constexpr int kSelThreads = 1024;
constexpr int kMaxSize = 16383;   // bound on distinct keys per sample (smem histograms)

// occurrence -> sample (thread per bag)
__global__ void k_cl_sample_of(int64_t nbags, int F, const int32_t* __restrict__ bag_off,
                               int32_t* __restrict__ samp) {
  for (int64_t bag = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; bag < nbags;
       bag += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(bag / F);
    for (int j = bag_off[bag]; j < bag_off[bag + 1]; ++j) samp[j] = b;
  }
}

// dense key id of every occurrence (bitmap rank) -> sort key; value = j
__global__ void k_cl_keyid(int64_t nnz, const int64_t* __restrict__ keys, int T, int W,
                           const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_base,
                           const uint32_t* __restrict__ bm, const int32_t* __restrict__ wr, int mark,
                           uint32_t* __restrict__ bm_w, uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                           int32_t* __restrict__ err) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; j0 < nnz; j0 += nth) {
    const int64_t j = j0 + lane;
    uint32_t dom = 0xffffffffu;
    if (j < nnz) {
      const uint64_t key = uint64_t(keys[j]);
      const uint64_t t = key >> kRowBits, row = key & kRowMask;
      if (t < uint64_t(T) && row < uint64_t(__ldg(rows + t))) {
        const uint64_t o = W == 1 ? 0 : row % uint64_t(W);
        const uint64_t lr = W == 1 ? row : row / uint64_t(W);
        dom = uint32_t(__ldg(seg_base + o * T + t) + int64_t(lr));
      } else if (mark) {
        atomicOr(err, kErrKeyRange);
      }
    }
    if (mark) {
      const uint32_t peers = __match_any_sync(0xffffffffu, dom);
      if (dom != 0xffffffffu && (peers & lt) == 0) atomicOr(&bm_w[dom >> 5], 1u << (dom & 31u));
    } else if (j < nnz) {
      kout[j] = dom == 0xffffffffu ? 0u : uint32_t(bit_rank(bm, wr, dom));
      vout[j] = int32_t(j);
    }
  }
}

// after the stable sort by key id: first occurrence of (sample, key) -> cl_u[j] = u, else -1
__global__ void k_cl_first(int64_t nnz, const uint32_t* __restrict__ sk, const int32_t* __restrict__ sv,
                           const int32_t* __restrict__ samp, int32_t* __restrict__ cl_u) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = sk[q];
    const int32_t j = sv[q];
    bool first = q == 0 || sk[q - 1] != u || samp[sv[q - 1]] != samp[j];
    cl_u[j] = first ? int32_t(u) : -1;
  }
}

// warp per sample: size (distinct keys), init assignment
__global__ void k_cl_size(int B, int F, const int32_t* __restrict__ bag_off, const int32_t* __restrict__ cl_u,
                          int32_t* __restrict__ size, int32_t* __restrict__ grp, int32_t* __restrict__ maxsz,
                          int32_t* __restrict__ err) {
  const int lane = lane_id();
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < B; s += nw) {
    const int j0 = bag_off[s * F], j1 = bag_off[(s + 1) * F];
    int n = 0;
    for (int j = j0 + lane; j < j1; j += 32) n += cl_u[j] >= 0;
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) {
      size[s] = n;
      grp[s] = -1;
      if (n > kMaxSize) atomicOr(err, kErrSampleSize);   // rank keys need (smax+1)^2 <= 2^28
      atomicMax(maxsz, min(n, kMaxSize));
    }
  }
}

// seed g: score every unassigned sample, keep the max of
// (maxov - ov) << 42 | size << 21 | (2^21-1 - id)
__global__ void k_cl_seed_score(int B, int F, int g, const int32_t* __restrict__ bag_off,
                                const int32_t* __restrict__ cl_u, const uint32_t* __restrict__ inmask,
                                const int32_t* __restrict__ size, const int32_t* __restrict__ grp,
                                unsigned long long* __restrict__ best) {
  const int lane = lane_id();
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < B; s += nw) {
    if (grp[s] >= 0) continue;
    int ov = 0;
    if (g > 0) {
      const int j0 = bag_off[s * F], j1 = bag_off[(s + 1) * F];
      for (int j = j0 + lane; j < j1; j += 32) {
        const int32_t u = cl_u[j];
        ov += u >= 0 && inmask[u] != 0;
      }
      for (int o = 16; o; o >>= 1) ov += __shfl_xor_sync(0xffffffffu, ov, o);
    }
    if (lane == 0) {
      const unsigned long long sc = (uint64_t(kMaxSize - ov) << 42) | (uint64_t(size[s]) << 21) |
                                    uint64_t((1 << 21) - 1 - int(s));
      atomicMax(best, sc);
    }
  }
}

// apply seed g (one block): grp[s*] = g, union(g) = keys(s*)
__global__ void k_cl_seed_apply(int F, int g, const int32_t* __restrict__ bag_off,
                                const int32_t* __restrict__ cl_u, const unsigned long long* __restrict__ best,
                                uint32_t* __restrict__ inmask, int32_t* __restrict__ grp) {
  const int s = (1 << 21) - 1 - int(*best & ((1ull << 21) - 1));
  if (threadIdx.x == 0) grp[s] = g;
  const int j0 = bag_off[int64_t(s) * F], j1 = bag_off[int64_t(s + 1) * F];
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const int32_t u = cl_u[j];
    if (u >= 0) atomicOr(&inmask[u], 1u << g);
  }
}

constexpr uint32_t kTaken = 0xffffffffu;   // rank key of a sample no longer a candidate

// round snapshot (warp per sample): S = |keys(s) & union(g)| folded into one
// rank key per (g, s), ck = (smax - S) * (smax + 1) + (size - S), so that
// "S desc, size - S asc" is "ck asc"; assigned samples get kTaken.
__global__ void k_cl_S(int B, int F, int N, const int32_t* __restrict__ bag_off,
                       const int32_t* __restrict__ cl_u, const uint32_t* __restrict__ inmask,
                       const int32_t* __restrict__ grp, const int32_t* __restrict__ size,
                       const int32_t* __restrict__ maxsz, uint32_t* __restrict__ ck) {
  const int lane = lane_id();
  const int smax = *maxsz;
  const uint32_t nb = uint32_t(smax) + 1;
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < B; s += nw) {
    if (grp[s] >= 0) {
      if (lane < N) ck[int64_t(lane) * B + s] = kTaken;
      continue;
    }
    const int sz = size[s];
    const int j0 = bag_off[s * F], j1 = bag_off[(s + 1) * F];
    int cnt[NEST_MAX_MICRO_BATCHES] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = j0 + lane; j < j1; j += 32) {
      const int32_t u = cl_u[j];
      if (u < 0) continue;
      const uint32_t m = inmask[u];
#pragma unroll
      for (int g = 0; g < NEST_MAX_MICRO_BATCHES; ++g) cnt[g] += (m >> g) & 1u;
    }
#pragma unroll
    for (int g = 0; g < NEST_MAX_MICRO_BATCHES; ++g) {
      int v = cnt[g];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == g && g < N) ck[int64_t(g) * B + s] = uint32_t(smax - v) * nb + uint32_t(sz - v);
    }
  }
}

struct Takes {
  int32_t v[NEST_MAX_MICRO_BATCHES];
};

// block-wide exclusive scan of one int per thread (1024 threads)
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int& total) {
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int x = ws[lane];
    int xi = warp_incl_scan(x);
    ws[lane] = xi - x;
    if (lane == 31) ws[32] = xi;
  }
  __syncthreads();
  const int r = ws[warp] + inc - v;
  total = ws[32];
  __syncthreads();
  return r;
}

// smallest bin b with cumsum(hist[0..b]) >= k; returns b and the count before b
__device__ void find_bin(const int* hist, int nbins, int k, int* ws, int* out) {
  // each thread owns a contiguous run of bins
  const int per = (nbins + kSelThreads - 1) / kSelThreads;
  const int b0 = threadIdx.x * per;
  int mine = 0;
  for (int b = b0; b < b0 + per && b < nbins; ++b) mine += hist[b];
  int tot;
  const int before = block_excl_scan(mine, ws, tot);
  if (before < k && before + mine >= k) {
    int run = before;
    for (int b = b0; b < b0 + per && b < nbins; ++b) {
      if (run + hist[b] >= k) {
        out[0] = b;
        out[1] = run;
        break;
      }
      run += hist[b];
    }
  }
  __syncthreads();
}

// one round: groups 0..N-1 take their samples in order (single block).
// Group g takes the k samples of least rank key ck (ties: lowest id): a radix
// select on ck finds the threshold T and how many T-ties to take (one
// histogram level when (smax+1)^2 <= kHistBins, else two), then every warp
// walks its own contiguous id range in order, ranking the T-ties by id.
// A sample taken by g is struck from the later groups' keys (ck = kTaken).
constexpr int kHistLog = 14, kHistBins = 1 << kHistLog, kSelUnroll = 8;

__global__ void __launch_bounds__(kSelThreads) k_cl_select(int B, int N, Takes takes,
                                                           const int32_t* __restrict__ maxsz,
                                                           uint32_t* ck, int32_t* __restrict__ grp,
                                                           int32_t* __restrict__ newlist,
                                                           int32_t* __restrict__ nnew) {
  extern __shared__ int hist[];            // [kHistBins]
  __shared__ int ws[33];
  __shared__ int sel[2];
  __shared__ int wcnt[32];
  __shared__ int nnew_s;
  const uint32_t nb = uint32_t(*maxsz) + 1;
  const uint32_t nkeys = nb * nb;          // ck < nb^2 <= 2^28
  int nbits = 0;
  while ((1u << nbits) < nkeys) ++nbits;
  const int lo = nbits > kHistLog ? nbits - kHistLog : 0;
  const int nb1 = lo ? kHistBins : int(nkeys);
  const uint32_t lomask = (1u << lo) - 1u;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const int R = ((B + kSelThreads - 1) / kSelThreads) * 32;   // ids per warp, multiple of 32
  const int w0 = min(B, warp * R), w1 = min(B, w0 + R);
  if (threadIdx.x == 0) nnew_s = 0;
  // warp-aggregated histogram increment (most candidates share a bin)
  auto hist_add = [&](int bin) {
    const uint32_t peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && (peers & lt) == 0) atomicAdd(&hist[bin], __popc(peers));
  };
  // the warp's range in id order, kSelUnroll loads in flight per lane
  auto walk = [&](const uint32_t* ckg, auto&& f) {
    for (int s0 = w0; s0 < w1; s0 += 32 * kSelUnroll) {
      uint32_t v[kSelUnroll];
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u) {
        const int s = s0 + u * 32 + lane;
        v[u] = s < w1 ? ckg[s] : kTaken;
      }
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u)
        if (s0 + u * 32 < w1) f(s0 + u * 32 + lane, v[u]);
    }
  };
  for (int g = 0; g < N; ++g) {
    const int k = takes.v[g];
    if (k <= 0) continue;
    const uint32_t* ckg = ck + int64_t(g) * B;
    // level 1: bins of ck >> lo
    for (int b = threadIdx.x; b < nb1; b += kSelThreads) hist[b] = 0;
    __syncthreads();
    walk(ckg, [&](int, uint32_t c) { hist_add(c != kTaken ? int(c >> lo) : -1); });
    __syncthreads();
    find_bin(hist, nb1, k, ws, sel);
    uint32_t T = uint32_t(sel[0]);
    int kk = k - sel[1];
    int cnt = hist[sel[0]];
    __syncthreads();
    if (lo) {   // level 2: low bits inside the chosen bin
      const uint32_t hi = T;
      for (int b = threadIdx.x; b < (1 << lo); b += kSelThreads) hist[b] = 0;
      __syncthreads();
      walk(ckg, [&](int, uint32_t c) { hist_add(c != kTaken && (c >> lo) == hi ? int(c & lomask) : -1); });
      __syncthreads();
      find_bin(hist, 1 << lo, kk, ws, sel);
      T = (hi << lo) | uint32_t(sel[0]);
      kk -= sel[1];
      cnt = hist[sel[0]];
      __syncthreads();
    }
    const bool partial = kk < cnt;   // only then do the T-ties need ranking by id
    int running = 0;
    if (partial) {
      int n = 0;
      walk(ckg, [&](int, uint32_t c) { n += __popc(__ballot_sync(0xffffffffu, c == T)); });
      if (lane == 0) wcnt[warp] = n;
      __syncthreads();
      for (int w = 0; w < warp; ++w) running += wcnt[w];
    }
    walk(ckg, [&](int s, uint32_t c) {
      const uint32_t tie = __ballot_sync(0xffffffffu, c == T);
      const bool take = c < T || (c == T && (!partial || running + __popc(tie & lt) < kk));
      running += __popc(tie);
      if (take) {
        grp[s] = g;
        for (int g2 = g + 1; g2 < N; ++g2) ck[int64_t(g2) * B + s] = kTaken;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, take);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&nnew_s, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (take) newlist[base + __popc(m & lt)] = s;
    });
    __syncthreads();
  }
  if (threadIdx.x == 0) *nnew = nnew_s;
}

// union(g) grows by the keys of the samples taken this round (warp per sample)
__global__ void k_cl_update(int F, const int32_t* __restrict__ newlist, const int32_t* __restrict__ nnew,
                            const int32_t* __restrict__ bag_off, const int32_t* __restrict__ cl_u,
                            const int32_t* __restrict__ grp, uint32_t* __restrict__ inmask) {
  const int lane = lane_id();
  const int n = *nnew;
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const int s = newlist[i];
    const uint32_t bit = 1u << grp[s];
    const int j0 = bag_off[int64_t(s) * F], j1 = bag_off[int64_t(s + 1) * F];
    for (int j = j0 + lane; j < j1; j += 32) {
      const int32_t u = cl_u[j];
      if (u >= 0 && !(inmask[u] & bit)) atomicOr(&inmask[u], bit);
    }
  }
}

// perm = samples sorted by (group, id); mb_offsets = g * cap (single block)
__global__ void __launch_bounds__(kSelThreads) k_cl_perm(int B, int N, const int32_t* __restrict__ grp,
                                                         int32_t* __restrict__ perm, int32_t* __restrict__ mbo) {
  __shared__ int ws[33];
  const int cap = B / N;
  const int per = (B + kSelThreads - 1) / kSelThreads;
  const int s0 = threadIdx.x * per, s1 = min(B, s0 + per);
  for (int g = 0; g < N; ++g) {
    int mine = 0;
    for (int s = s0; s < s1; ++s) mine += grp[s] == g;
    int tot;
    int r = block_excl_scan(mine, ws, tot);
    for (int s = s0; s < s1; ++s)
      if (grp[s] == g) perm[g * cap + r++] = s;
  }
  if (threadIdx.x <= N) mbo[threadIdx.x] = threadIdx.x * cap;
}

void launch_cluster(Ctx& c, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz, int B, int N,
                    int32_t* perm, int32_t* mb_offsets, cudaStream_t st) {
  NEST_CHECK(B < (1 << 21), NEST_ERR_INVALID, "clustered schedule supports B < 2^21");
  const int F = c.F;
  const int64_t nbags = int64_t(B) * F;
  auto grid = [](int64_t n, int t) {
    int64_t b = (n + t - 1) / t;
    return int(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
  };
  int32_t* samp = c.cl_samp;
  // dense key ids through a presence bitmap over the domain
  NEST_CUDA(cudaMemsetAsync(c.cl_bm, 0, sizeof(uint32_t) * (c.words + 2), st));
  k_cl_keyid<<<grid(nnz, 256), 256, 0, st>>>(nnz, keys, c.T, c.W, c.d_rows, c.d_seg_base, nullptr, nullptr, 1,
                                            c.cl_bm, nullptr, nullptr, c.d_err);
  {
    const uint32_t* bm = c.cl_bm;
    int32_t* wr = c.cl_wr;
    const int64_t nw = c.words + 1;
    scan_exclusive<int32_t>([=] __device__(int64_t i) { return int32_t(__popc(bm[i])); }, nw,
                            [=] __device__(int64_t i, int32_t v) { wr[i] = v; }, c.scan_tmp, st);
  }
  k_cl_keyid<<<grid(nnz, 256), 256, 0, st>>>(nnz, keys, c.T, c.W, c.d_rows, c.d_seg_base, c.cl_bm, c.cl_wr, 0,
                                            nullptr, c.tkey[0], c.tval[0], c.d_err);
  k_cl_sample_of<<<grid(nbags, 256), 256, 0, st>>>(nbags, F, bag_offsets, samp);
  int kbits = 0;
  while ((int64_t(1) << kbits) < c.Kcap) ++kbits;
  radix_sort_pairs(c, c.tkey[0], c.tval[0], c.cl_sk, c.cl_sv, nnz, kbits, st);
  k_cl_first<<<grid(nnz, 256), 256, 0, st>>>(nnz, c.cl_sk, c.cl_sv, samp, c.cl_u);
  NEST_CUDA(cudaMemsetAsync(c.cl_small, 0, sizeof(int64_t) * 4, st));
  int32_t* maxsz = reinterpret_cast<int32_t*>(c.cl_small);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(c.cl_small + 1);
  int32_t* nnew = reinterpret_cast<int32_t*>(c.cl_small + 2);
  k_cl_size<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(B, F, bag_offsets, c.cl_u, c.cl_size, c.cl_grp, maxsz,
                                                        c.d_err);
  NEST_CUDA(cudaMemsetAsync(c.cl_inmask, 0, sizeof(uint32_t) * c.Kcap, st));
  // seeds
  for (int g = 0; g < N; ++g) {
    NEST_CUDA(cudaMemsetAsync(best, 0, sizeof(unsigned long long), st));
    k_cl_seed_score<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(B, F, g, bag_offsets, c.cl_u, c.cl_inmask,
                                                                 c.cl_size, c.cl_grp, best);
    k_cl_seed_apply<<<1, 256, 0, st>>>(F, g, bag_offsets, c.cl_u, best, c.cl_inmask, c.cl_grp);
  }
  // rounds: admission sizes are a function of (B, N) only
  const int cap = B / N;
  std::vector<int64_t> have(N, 1);
  int64_t assigned = N;
  uint64_t Q = uint64_t(1) << 32;
  const size_t smem = sizeof(int) * kHistBins;
  uint32_t* ck = reinterpret_cast<uint32_t*>(c.cl_S);
  static bool attr = false;
  if (!attr) {
    NEST_CUDA(cudaFuncSetAttribute(k_cl_select, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  while (assigned < B) {
    if (Q < (uint64_t(1) << 62)) Q = (5 * Q) / 4;
    const int64_t q = std::max<int64_t>(1, int64_t(Q >> 32));
    Takes tk{};
    for (int g = 0; g < N; ++g) {
      tk.v[g] = int32_t(std::min<int64_t>(cap - have[g], q));
      have[g] += tk.v[g];
      assigned += tk.v[g];
    }
    k_cl_S<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(B, F, N, bag_offsets, c.cl_u, c.cl_inmask, c.cl_grp,
                                                      c.cl_size, maxsz, ck);
    k_cl_select<<<1, kSelThreads, smem, st>>>(B, N, tk, maxsz, ck, c.cl_grp, c.cl_new, nnew);
    k_cl_update<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(F, c.cl_new, nnew, bag_offsets, c.cl_u, c.cl_grp,
                                                           c.cl_inmask);
  }
  k_cl_perm<<<1, kSelThreads, 0, st>>>(B, N, c.cl_grp, perm, mb_offsets);
  NEST_LAUNCH_CHECK();
}

}  // namespace nest
