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

// after the stable sort by key id: first occurrence of (sample, key) -> cl_u[j] = u, else -1;
// kstart[u] = first position of key id u in the sorted occurrences
__global__ void k_cl_first(int64_t nnz, const uint32_t* __restrict__ sk, const int32_t* __restrict__ sv,
                           const int32_t* __restrict__ samp, int32_t* __restrict__ cl_u,
                           int32_t* __restrict__ kstart) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = sk[q];
    const int32_t j = sv[q];
    const bool key_first = q == 0 || sk[q - 1] != u;
    bool first = key_first || samp[sv[q - 1]] != samp[j];
    cl_u[j] = first ? int32_t(u) : -1;
    if (key_first) kstart[u] = int32_t(q);
    if (q == nnz - 1) kstart[u + 1] = int32_t(nnz);
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

// S[g][s] = |keys(s) & union(g)| from scratch (warp per sample), once after
// the seeds; the rounds then maintain it incrementally (k_cl_spread)
__global__ void k_cl_S_full(int B, int F, int N, const int32_t* __restrict__ bag_off,
                            const int32_t* __restrict__ cl_u, const uint32_t* __restrict__ inmask,
                            int32_t* __restrict__ S) {
  const int lane = lane_id();
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < B; s += nw) {
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
      if (lane == g && g < N) S[int64_t(g) * B + s] = v;
    }
  }
}

// round snapshot (thread per sample): S folded into one rank key per (g, s),
// ck = (smax - S) * (smax + 1) + (size - S), so that "S desc, size - S asc"
// is "ck asc"; assigned samples get kTaken.  Also the level-1 histogram of
// every group's candidate keys (bins ck >> lo), warp-aggregated.
__global__ void k_cl_rank(int B, int N, int lo, const int32_t* __restrict__ S, const int32_t* __restrict__ grp,
                          const int32_t* __restrict__ size, const int32_t* __restrict__ maxsz,
                          uint32_t* __restrict__ ck, int32_t* __restrict__ hist, int32_t* __restrict__ err) {
  const int smax = *maxsz;
  const uint32_t nb = uint32_t(smax) + 1;
  const uint32_t lt = lanemask_lt();
  for (int s0 = blockIdx.x * blockDim.x; s0 < B; s0 += gridDim.x * blockDim.x) {
    const int s = s0 + threadIdx.x;
    const bool cand = s < B && grp[s] < 0;
    const int sz = cand ? size[s] : 0;
    for (int g = 0; g < N; ++g) {
      int bin = -1;
      if (s < B) {
        uint32_t key = kTaken;
        if (cand) {
          const int v = S[int64_t(g) * B + s];
          key = uint32_t(smax - v) * nb + uint32_t(sz - v);
          bin = int(key >> lo);
          if (v < 0 || v > sz || bin >= kClHistBins) {   // S out of [0, size]: a bug, never an index
            atomicOr(err, kErrCluster);
            key = kTaken;
            bin = -1;
          }
        }
        ck[int64_t(g) * B + s] = key;
      }
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (bin >= 0 && (peers & lt) == 0) atomicAdd(&hist[g * kClHistBins + bin], __popc(peers));
    }
  }
}

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
// (out[0] = -1 when the histogram holds fewer than k entries)
__device__ void find_bin(const int* hist, int nbins, int k, int* ws, int* out) {
  if (threadIdx.x == 0) out[0] = -1;
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

// One round, group g after group g-1 (multi-block radix select): the
// threshold T of g's k smallest rank keys and how many T-ties (kk) to take,
// lowest ids first, from the level-1 histogram (bins ck >> lo) and, when the
// keys need more than kClHistLog bits, a level-2 histogram of the low bits
// inside the chosen bin; then every block of kClIds ids counts its ties and
// assigns.  A sample taken by g leaves the later groups' histograms and keys.
// sel[g]: {T, kk, partial, b1, kk1}
// level-1 bins of the rank keys: (smax+1)^2 keys, or kClHistBins bins of
// ck >> lo (smax is the batch's, read on the device: the captured round
// sequence is replayed for every batch of the same (B, N, lo))
__device__ __forceinline__ int cl_nb1(const int32_t* maxsz, int lo) {
  const int nb = *maxsz + 1;
  return lo ? kClHistBins : nb * nb;
}

__global__ void __launch_bounds__(kSelThreads) k_cl_find1(int k, const int32_t* __restrict__ maxsz, int lo,
                                                          const int32_t* __restrict__ hist,
                                                          int32_t* __restrict__ sel) {
  __shared__ int ws[33];
  __shared__ int out[2];
  find_bin(hist, cl_nb1(maxsz, lo), k, ws, out);
  if (threadIdx.x == 0) {
    const int b1 = max(out[0], 0), kk1 = out[0] < 0 ? 0 : k - out[1];
    sel[3] = b1;
    sel[4] = kk1;
    if (lo == 0) {
      sel[0] = b1;
      sel[1] = kk1;
      sel[2] = kk1 < hist[b1];
    }
  }
}

__global__ void k_cl_hist2(int B, int lo, const uint32_t* __restrict__ ckg, const int32_t* __restrict__ sel,
                           int32_t* __restrict__ hist2) {
  const uint32_t b1 = uint32_t(sel[3]), lomask = (1u << lo) - 1u;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < B; s += gridDim.x * blockDim.x) {
    const uint32_t c = ckg[s];
    if (c != kTaken && (c >> lo) == b1) atomicAdd(&hist2[c & lomask], 1);
  }
}

// the group's threshold: T, the T-ties to take (kk), whether the tie bin is
// taken partly -- resolved by every block from the histograms (level 1, or
// level 2 inside the bin k_cl_find1 chose)
struct Thr {
  uint32_t T;
  int kk;
  bool partial;
};
__device__ Thr cl_resolve(int k, int nb1, int lo, const int32_t* hist1, const int32_t* hist2,
                          const int32_t* sel, int* ws, int* out, int32_t* err) {
  Thr t;
  const int32_t* h = lo == 0 ? hist1 : hist2;
  const int kk0 = lo == 0 ? k : sel[4];
  find_bin(h, lo == 0 ? nb1 : 1 << lo, kk0, ws, out);
  if (out[0] < 0) {   // fewer candidates than the admission size: a bug, never an index
    if (threadIdx.x == 0) atomicOr(err, kErrCluster);
    t.T = 0;
    t.kk = 0;
    t.partial = true;
    return t;
  }
  t.T = lo == 0 ? uint32_t(out[0]) : (uint32_t(sel[3]) << lo) | uint32_t(out[0]);
  t.kk = kk0 - out[1];
  t.partial = t.kk < h[out[0]];
  return t;
}

// ties of T per block of kClIds ids (only when the tie bin is taken partly)
__global__ void __launch_bounds__(kClIds) k_cl_tiecount(int B, int k, const int32_t* __restrict__ maxsz, int lo,
                                                        const uint32_t* __restrict__ ckg,
                                                        const int32_t* __restrict__ hist1,
                                                        const int32_t* __restrict__ hist2,
                                                        const int32_t* __restrict__ sel, int32_t* __restrict__ bcnt,
                                                        int32_t* __restrict__ err) {
  __shared__ int ws[33];
  __shared__ int out[2];
  const Thr t = cl_resolve(k, cl_nb1(maxsz, lo), lo, hist1, hist2, sel, ws, out, err);
  if (!t.partial) return;
  const int s = blockIdx.x * kClIds + threadIdx.x;
  const int n = __syncthreads_count(s < B && ckg[s] == t.T);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = n;
}

__global__ void __launch_bounds__(kClIds) k_cl_assign(int B, int N, int g, int k, const int32_t* __restrict__ maxsz,
                                                      int lo, uint32_t* ck,
                                                      const int32_t* __restrict__ sel, int32_t* hist,
                                                      const int32_t* __restrict__ hist2,
                                                      const int32_t* __restrict__ bcnt, int32_t* __restrict__ grp,
                                                      int32_t* __restrict__ newlist, int32_t* __restrict__ nnew,
                                                      int32_t* __restrict__ err) {
  __shared__ int ws[33];
  __shared__ int out[2];
  // (hist rows g2 > g change below, row g does not: every block resolves alike)
  const Thr t = cl_resolve(k, cl_nb1(maxsz, lo), lo, hist + g * kClHistBins, hist2, sel, ws, out, err);
  const uint32_t T = t.T;
  const int kk = t.kk;
  const bool partial = t.partial;
  int base = 0;
  if (partial) {   // ties in the blocks before this one
    int part = 0;
    for (int b = threadIdx.x; b < blockIdx.x; b += kClIds) part += bcnt[b];
    int tot;
    block_excl_scan(part, ws, tot);
    base = tot;
  }
  const int s = blockIdx.x * kClIds + threadIdx.x;
  const uint32_t c = s < B ? ck[int64_t(g) * B + s] : kTaken;
  const bool tie = c == T;
  int tot;
  const int rank = base + block_excl_scan(tie ? 1 : 0, ws, tot);
  const bool take = c < T || (tie && (!partial || rank < kk));
  if (take) {
    grp[s] = g;
    for (int g2 = g + 1; g2 < N; ++g2) {
      uint32_t* p2 = ck + int64_t(g2) * B + s;
      atomicSub(&hist[g2 * kClHistBins + (*p2 >> lo)], 1);
      *p2 = kTaken;
    }
  }
  const uint32_t m = __ballot_sync(0xffffffffu, take);
  int at = 0;
  if (lane_id() == 0 && m) at = atomicAdd(nnew, __popc(m));
  at = __shfl_sync(0xffffffffu, at, 0);
  if (take) newlist[at + __popc(m & lanemask_lt())] = s;
}

constexpr int kSpreadChunk = 128;   // occurrences per spread work item

// union(g) grows by the keys of the samples taken this round (warp per
// sample); every (key, group) bit set for the first time is listed as work
// items of <= kSpreadChunk of the key's occurrences: u << 32 | chunk << 3 | g
__global__ void k_cl_update(int F, const int32_t* __restrict__ newlist, const int32_t* __restrict__ nnew,
                            const int32_t* __restrict__ bag_off, const int32_t* __restrict__ cl_u,
                            const int32_t* __restrict__ grp, uint32_t* __restrict__ inmask,
                            const int32_t* __restrict__ kstart, uint64_t* __restrict__ newk,
                            int32_t* __restrict__ nnewk, int64_t ncap, int32_t* __restrict__ err) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int n = *nnew;
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const int s = newlist[i];
    const int g = grp[s];
    const uint32_t bit = 1u << g;
    const int j0 = bag_off[int64_t(s) * F], j1 = bag_off[int64_t(s + 1) * F];
    for (int jb = j0; jb < j1; jb += 32) {
      const int j = jb + lane;
      const int32_t u = j < j1 ? cl_u[j] : -1;
      bool fresh = false;
      if (u >= 0 && !(inmask[u] & bit)) fresh = !(atomicOr(&inmask[u], bit) & bit);
      const int nch = fresh ? (kstart[u + 1] - kstart[u] + kSpreadChunk - 1) / kSpreadChunk : 0;
      const int inc = warp_incl_scan(nch);
      const int tot = __shfl_sync(0xffffffffu, inc, 31);
      int at = 0;
      if (lane == 0 && tot) at = atomicAdd(nnewk, tot);
      at = __shfl_sync(0xffffffffu, at, 0) + inc - nch;
      if (nch && at + nch > ncap) {
        atomicOr(err, kErrCluster);
        continue;
      }
      for (int ch = 0; ch < nch; ++ch)
        newk[at + ch] = (uint64_t(uint32_t(u)) << 32) | (uint64_t(ch) << 3) | uint64_t(g);
    }
  }
}

// S[g][s] += 1 for every unassigned sample s holding a key that joined
// union(g) this round (warp per work item: a chunk of the key's occurrences)
__global__ void k_cl_spread(int B, int64_t ncap, int64_t kcap, const uint64_t* __restrict__ newk,
                            const int32_t* __restrict__ nnewk,
                            const int32_t* __restrict__ kstart, const uint32_t* __restrict__ sk,
                            const int32_t* __restrict__ sv, const int32_t* __restrict__ cl_u,
                            const int32_t* __restrict__ samp, const int32_t* __restrict__ grp,
                            int32_t* __restrict__ S, int32_t* __restrict__ err) {
  const int lane = lane_id();
  const int n = int(min(int64_t(*nnewk), ncap));
  const int64_t nw = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const uint64_t e = newk[i];
    const uint32_t u = uint32_t(e >> 32), g = uint32_t(e) & 7u, ch = uint32_t(e) >> 3;
    const int q0 = kstart[u] + int(ch) * kSpreadChunk;
    const int q1 = min(q0 + kSpreadChunk, kstart[u + 1]);
    if (u >= kcap || q0 < 0 || q1 > kcap) {   // a bug, never an index
      if (lane == 0) atomicOr(err, kErrCluster);
      continue;
    }
    for (int q = q0 + lane; q < q1; q += 32) {
      const int32_t j = sv[q];
      if (cl_u[j] < 0) continue;   // not the sample's first occurrence of u
      const int32_t s = samp[j];
      if (grp[s] < 0) atomicAdd(&S[int64_t(g) * B + s], 1);
    }
  }
}

// perm = samples sorted by (group, id): per block of kClIds ids the count of
// each group, then every block places its members after the earlier blocks'
__global__ void __launch_bounds__(kClIds) k_cl_gcount(int B, int N, const int32_t* __restrict__ grp,
                                                      int32_t* __restrict__ bcnt) {
  const int s = blockIdx.x * kClIds + threadIdx.x;
  const int gs = s < B ? grp[s] : -1;
  for (int g = 0; g < N; ++g) {
    const int n = __syncthreads_count(gs == g);
    if (threadIdx.x == 0) bcnt[blockIdx.x * N + g] = n;
  }
}

__global__ void __launch_bounds__(kClIds) k_cl_perm(int B, int N, const int32_t* __restrict__ grp,
                                                    const int32_t* __restrict__ bcnt, int32_t* __restrict__ perm,
                                                    int32_t* __restrict__ mbo, int32_t* __restrict__ err) {
  __shared__ int ws[33];
  const int cap = B / N;
  const int s = blockIdx.x * kClIds + threadIdx.x;
  const int gs = s < B ? grp[s] : -1;
  for (int g = 0; g < N; ++g) {
    int part = 0;
    for (int b = threadIdx.x; b < blockIdx.x; b += kClIds) part += bcnt[b * N + g];
    int base;
    block_excl_scan(part, ws, base);
    int tot;
    const int r = block_excl_scan(gs == g ? 1 : 0, ws, tot);
    if (gs == g) {
      if (base + r < cap) perm[g * cap + base + r] = s;
      else atomicOr(err, kErrCluster);   // a group over its capacity: a bug, never an index
    }
  }
  if (blockIdx.x == 0 && threadIdx.x <= N) mbo[threadIdx.x] = threadIdx.x * cap;
}

static void cluster_rounds(Ctx& c, int B, int N, int F, int lo, int32_t* maxsz, int32_t* nnew, cudaStream_t st);

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
                                            nullptr, c.rx_aux.tkey[0], c.rx_aux.tval[0], c.d_err);
  k_cl_sample_of<<<grid(nbags, 256), 256, 0, st>>>(nbags, F, bag_offsets, samp);
  int kbits = 0;
  while ((int64_t(1) << kbits) < c.Kcap) ++kbits;
  radix_sort_pairs(c.rx_aux, c.rx_aux.tkey[0], c.rx_aux.tval[0], c.cl_sk, c.cl_sv, nnz, kbits, st);
  k_cl_first<<<grid(nnz, 256), 256, 0, st>>>(nnz, c.cl_sk, c.cl_sv, samp, c.cl_u, c.cl_kstart);
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
  k_cl_S_full<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(B, F, N, bag_offsets, c.cl_u, c.cl_inmask, c.cl_Scnt);
  // the rank keys' histogram split needs smax (one read back on this stream)
  int32_t smax = 0;
  NEST_CUDA(cudaMemcpyAsync(c.cl_hmax, maxsz, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  NEST_CUDA(cudaStreamSynchronize(st));
  smax = *c.cl_hmax;
  const uint32_t nkeys = uint32_t(smax + 1) * uint32_t(smax + 1);
  int nbits = 0;
  while ((1u << nbits) < nkeys) ++nbits;
  const int lo = nbits > kClHistLog ? nbits - kClHistLog : 0;
  // rounds: admission sizes are a function of (B, N) only, every buffer is the
  // library's, so the whole round sequence is captured once per (B, N, lo)
  // into a CUDA graph and replayed (it is ~37 rounds of 3N + 4 launches)
  NEST_CUDA(cudaMemcpyAsync(c.cl_boff, bag_offsets, sizeof(int32_t) * (nbags + 1), cudaMemcpyDeviceToDevice, st));
  const auto gkey = std::make_tuple(B, N, lo);
  auto git = c.cl_graphs.find(gkey);
  if (st == nullptr) {
    cluster_rounds(c, B, N, F, lo, maxsz, nnew, st);   // legacy stream: no capture
  } else if (git == c.cl_graphs.end()) {
    NEST_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cluster_rounds(c, B, N, F, lo, maxsz, nnew, st);
    cudaGraph_t graph = nullptr;
    NEST_CUDA(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec = nullptr;
    NEST_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    git = c.cl_graphs.emplace(gkey, exec).first;
  }
  if (st != nullptr) NEST_CUDA(cudaGraphLaunch(git->second, st));
  const int nblk = (B + kClIds - 1) / kClIds;
  k_cl_gcount<<<nblk, kClIds, 0, st>>>(B, N, c.cl_grp, c.cl_bcnt);
  k_cl_perm<<<nblk, kClIds, 0, st>>>(B, N, c.cl_grp, c.cl_bcnt, perm, mb_offsets, c.d_err);
  NEST_LAUNCH_CHECK();
}

// the admission rounds on library buffers only (captured into a graph)
static void cluster_rounds(Ctx& c, int B, int N, int F, int lo, int32_t* maxsz, int32_t* nnew, cudaStream_t st) {
  int32_t* nnewk = reinterpret_cast<int32_t*>(c.cl_small + 3);
  const int32_t* bag_offsets = c.cl_boff;
  auto grid = [](int64_t n, int t) {
    int64_t b = (n + t - 1) / t;
    return int(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
  };
  const int cap = B / N;
  const int nblk = (B + kClIds - 1) / kClIds;
  std::vector<int64_t> have(N, 1);
  int64_t assigned = N;
  uint64_t Q = uint64_t(1) << 32;
  uint32_t* ck = reinterpret_cast<uint32_t*>(c.cl_S);
  int32_t* hist2 = c.cl_hist + int64_t(N) * kClHistBins;
  while (assigned < B) {
    if (Q < (uint64_t(1) << 62)) Q = (5 * Q) / 4;
    const int64_t q = std::max<int64_t>(1, int64_t(Q >> 32));
    int take[NEST_MAX_MICRO_BATCHES];
    for (int g = 0; g < N; ++g) {
      take[g] = int(std::min<int64_t>(cap - have[g], q));
      have[g] += take[g];
      assigned += take[g];
    }
    NEST_CUDA(cudaMemsetAsync(c.cl_hist, 0, sizeof(int32_t) * kClHistBins * N, st));
    NEST_CUDA(cudaMemsetAsync(nnew, 0, sizeof(int32_t), st));
    k_cl_rank<<<grid(B, 256), 256, 0, st>>>(B, N, lo, c.cl_Scnt, c.cl_grp, c.cl_size, maxsz, ck, c.cl_hist,
                                            c.d_err);
    for (int g = 0; g < N; ++g) {
      if (take[g] <= 0) continue;
      int32_t* sel = c.cl_sel + 8 * g;
      const int32_t* h1 = c.cl_hist + int64_t(g) * kClHistBins;
      if (lo) {
        k_cl_find1<<<1, kSelThreads, 0, st>>>(take[g], maxsz, lo, h1, sel);
        NEST_CUDA(cudaMemsetAsync(hist2, 0, sizeof(int32_t) << lo, st));
        k_cl_hist2<<<grid(B, 256), 256, 0, st>>>(B, lo, ck + int64_t(g) * B, sel, hist2);
      }
      k_cl_tiecount<<<nblk, kClIds, 0, st>>>(B, take[g], maxsz, lo, ck + int64_t(g) * B, h1, hist2, sel, c.cl_bcnt,
                                             c.d_err);
      k_cl_assign<<<nblk, kClIds, 0, st>>>(B, N, g, take[g], maxsz, lo, ck, sel, c.cl_hist, hist2, c.cl_bcnt,
                                           c.cl_grp, c.cl_new, nnew, c.d_err);
    }
    NEST_CUDA(cudaMemsetAsync(nnewk, 0, sizeof(int32_t), st));
    k_cl_update<<<grid(int64_t(B) * 32, 256), 256, 0, st>>>(F, c.cl_new, nnew, bag_offsets, c.cl_u, c.cl_grp,
                                                           c.cl_inmask, c.cl_kstart, c.cl_newk, nnewk,
                                                           c.cl_newk_cap, c.d_err);
    k_cl_spread<<<148 * 8, 256, 0, st>>>(B, c.cl_newk_cap, c.Kcap, c.cl_newk, nnewk, c.cl_kstart, c.cl_sk, c.cl_sv,
                                         c.cl_u, c.cl_samp, c.cl_grp, c.cl_Scnt, c.d_err);
  }
  NEST_LAUNCH_CHECK();
}

}  // namespace nest
