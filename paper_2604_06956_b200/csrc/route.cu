// DBP Key Routing + Embedding Retrieval.
//
// Source side (R1): keys -> owner-major domain index dom(key) =
//   seg_base[owner*T + table] + row div W, owner = row mod W.
// Dedup is a presence bitmap over the domain (a counting sort with 1-bit
// buckets): mark -> per-word popcount prefix -> set bits in ascending order ARE
// the unique keys sorted by (owner, key); the rank of a bit is the inverse.
// This replaces a comparison/radix sort of the K key occurrences by two
// coalesced passes over them plus a pass over a V-bit bitmap that lives in L2
// (13 MB for the DLRM config).  See DESIGN.md "R1 route".
// Owner side (R3): the same on the owner's local domain (= shard row index).
#include "nest_internal.cuh"

namespace nest {

// ---------------------------------------------------------------------------
// radix sort (stable LSD, digits of DB <= kRadixMaxDigit bits): histogram ->
// scan -> ranked scatter.
// ---------------------------------------------------------------------------
template <int DB>
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint32_t* __restrict__ keys,
                                                              int64_t n, int shift,
                                                              uint32_t* __restrict__ hist, int nb) {
  constexpr uint32_t NBIN = 1u << DB;
  __shared__ uint32_t cnt[NBIN];
  for (uint32_t d = threadIdx.x; d < NBIN; d += kRadixThreads) cnt[d] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kRadixTile;
  const uint32_t lt = lanemask_lt();
#pragma unroll 4
  for (int k = 0; k < kRadixItems; ++k) {
    const int64_t i = base + k * kRadixThreads + threadIdx.x;
    const bool v = i < n;
    const uint32_t d = v ? (keys[i] >> shift) & (NBIN - 1) : NBIN;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (v && (peers & lt) == 0) atomicAdd(&cnt[d], __popc(peers));
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < NBIN; d += kRadixThreads) hist[int64_t(d) * nb + blockIdx.x] = cnt[d];
}

template <int DB>
constexpr size_t radix_scatter_smem() {
  return sizeof(uint32_t) * (size_t(kRadixWarps + 2) * (1u << DB) + 2 * size_t(kRadixTile));
}

template <int DB>
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, int64_t n, int shift,
    const uint32_t* __restrict__ offs, int nb, uint32_t* __restrict__ kout,
    int32_t* __restrict__ vout) {
  constexpr uint32_t NBIN = 1u << DB;
  constexpr int DPT = int(NBIN) / kRadixThreads;   // digits owned per thread in the digit scan
  static_assert(DPT >= 1, "at least one digit per thread");
  extern __shared__ uint32_t rsm[];
  uint32_t* wcnt = rsm;                            // [kRadixWarps][NBIN]
  uint32_t* dstart = wcnt + kRadixWarps * NBIN;    // [NBIN]
  uint32_t* gbase = dstart + NBIN;                 // [NBIN]
  uint32_t* skeys = gbase + NBIN;                  // [kRadixTile]
  int32_t* svals = reinterpret_cast<int32_t*>(skeys + kRadixTile);
  __shared__ uint32_t wsum[kRadixWarps];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  for (uint32_t i = threadIdx.x; i < kRadixWarps * NBIN; i += kRadixThreads) wcnt[i] = 0;
  for (uint32_t d = threadIdx.x; d < NBIN; d += kRadixThreads) gbase[d] = offs[int64_t(d) * nb + blockIdx.x];
  __syncthreads();
  // warp w owns the contiguous items [w*512, w*512+512) of the tile, visited
  // in rounds of 32: (warp, round, lane) order == input order -> stable
  const int64_t base = int64_t(blockIdx.x) * kRadixTile + warp * (32 * kRadixItems);
  const uint32_t lt = lanemask_lt();
  uint32_t* wc = wcnt + warp * NBIN;
  uint32_t key[kRadixItems];
  int32_t val[kRadixItems];
  uint32_t lr[kRadixItems];
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const int64_t i = base + k * 32 + lane;
    const bool v = i < n;
    key[k] = v ? kin[i] : 0xffffffffu;
    val[k] = v ? vin[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const bool v = base + k * 32 + lane < n;
    const uint32_t d = v ? (key[k] >> shift) & (NBIN - 1) : NBIN;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = v ? wc[d] : 0u;
    __syncwarp();
    if (v && (peers & lt) == 0) wc[d] = before + __popc(peers);
    __syncwarp();
    lr[k] = before + __popc(peers & lt);
  }
  __syncthreads();
  {
    // thread t owns digits [t*DPT, t*DPT + DPT): per digit an exclusive prefix
    // over the warps, then a block-wide exclusive scan of the digit totals
    uint32_t tot[DPT];
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const uint32_t d = threadIdx.x * DPT + j;
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kRadixWarps; ++w) {
        const uint32_t cc = wcnt[w * NBIN + d];
        wcnt[w * NBIN + d] = run;
        run += cc;
      }
      tot[j] = run;
      mine += run;
    }
    const uint32_t inc = warp_incl_scan(mine);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = lane < kRadixWarps ? wsum[lane] : 0u;
      const uint32_t xi = warp_incl_scan(x);
      if (lane < kRadixWarps) wsum[lane] = xi - x;
    }
    __syncthreads();
    uint32_t start = wsum[warp] + inc - mine;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      dstart[threadIdx.x * DPT + j] = start;
      start += tot[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    if (base + k * 32 + lane < n) {
      const uint32_t d = (key[k] >> shift) & (NBIN - 1);
      const uint32_t s = dstart[d] + wcnt[warp * NBIN + d] + lr[k];
      skeys[s] = key[k];
      svals[s] = val[k];
    }
  }
  __syncthreads();
  const int64_t tb = int64_t(blockIdx.x) * kRadixTile;
  const int nvalid = n - tb < kRadixTile ? int(n - tb) : kRadixTile;
  for (int s = threadIdx.x; s < nvalid; s += kRadixThreads) {
    const uint32_t k2 = skeys[s];
    const uint32_t d = (k2 >> shift) & (NBIN - 1);
    const uint32_t p = gbase[d] + (uint32_t(s) - dstart[d]);
    kout[p] = k2;
    vout[p] = svals[s];
  }
}

// ---------------------------------------------------------------------------
// One-sweep LSD radix (NEST_RADIX=onesweep; not the default, see
// radix_classic below): one histogram pass counts the digits of every
// pass at once (digit counts do not depend on the order), then each pass is a
// single scatter kernel.  Tiles take their index from an atomic counter (so
// every tile a block waits for is already running), rank their items exactly
// as k_radix_scatter does, publish per-digit counts, and find the count of
// their digit in all earlier tiles by decoupled look-back over the tile status
// words (flag | value): no per-pass histogram kernel, no 3-kernel scan.
// Stable: items keep (tile, warp, round, lane) order within a digit.
// ---------------------------------------------------------------------------
constexpr uint32_t kStAgg = 1u << 30, kStInc = 2u << 30, kStVal = (1u << 30) - 1u;

__global__ void __launch_bounds__(kRadixThreads) k_radix_hist_all(const uint32_t* __restrict__ keys, int64_t n,
                                                                  int passes, int db, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t cnt[4 * 256];
  for (int i = threadIdx.x; i < 4 * 256; i += kRadixThreads) cnt[i] = 0;
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  const uint32_t dmask = (1u << db) - 1u;
  for (int64_t i0 = int64_t(blockIdx.x) * kRadixThreads; i0 < n; i0 += int64_t(gridDim.x) * kRadixThreads) {
    const int64_t i = i0 + threadIdx.x;
    const bool v = i < n;
    const uint32_t k = v ? keys[i] : 0u;
    for (int p = 0; p < passes; ++p) {
      const uint32_t d = v ? (k >> (p * db)) & dmask : 0xffffffffu;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (v && (peers & lt) == 0) atomicAdd(&cnt[p * 256 + d], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRadixThreads)
    if (cnt[i]) atomicAdd(&ghist[i], cnt[i]);
}

template <int DB>
__global__ void __launch_bounds__(kRadixThreads) k_radix_onesweep(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, int64_t n, int shift,
    const uint32_t* __restrict__ ghist, uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr,
    uint32_t* __restrict__ kout, int32_t* __restrict__ vout) {
  constexpr uint32_t NBIN = 1u << DB;
  static_assert(NBIN == kRadixThreads, "one digit per thread");
  extern __shared__ uint32_t rsm[];
  uint32_t* wcnt = rsm;                            // [kRadixWarps][NBIN]
  uint32_t* dstart = wcnt + kRadixWarps * NBIN;    // [NBIN]
  uint32_t* gbase = dstart + NBIN;                 // [NBIN]
  uint32_t* skeys = gbase + NBIN;                  // [kRadixTile]
  int32_t* svals = reinterpret_cast<int32_t*>(skeys + kRadixTile);
  __shared__ uint32_t wsum[kRadixWarps], gsum[kRadixWarps];
  __shared__ uint32_t s_tile;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (uint32_t i = threadIdx.x; i < kRadixWarps * NBIN; i += kRadixThreads) wcnt[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = int64_t(tile) * kRadixTile + warp * (32 * kRadixItems);
  const uint32_t lt = lanemask_lt();
  uint32_t* wc = wcnt + warp * NBIN;
  uint32_t key[kRadixItems];
  int32_t val[kRadixItems];
  uint32_t lr[kRadixItems];
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const int64_t i = base + k * 32 + lane;
    const bool v = i < n;
    key[k] = v ? kin[i] : 0xffffffffu;
    val[k] = v ? vin[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const bool v = base + k * 32 + lane < n;
    const uint32_t d = v ? (key[k] >> shift) & (NBIN - 1) : NBIN;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = v ? wc[d] : 0u;
    __syncwarp();
    if (v && (peers & lt) == 0) wc[d] = before + __popc(peers);
    __syncwarp();
    lr[k] = before + __popc(peers & lt);
  }
  __syncthreads();
  // thread t owns digit t: prefix over the warps, the tile's count, the
  // block-wide exclusive scan of the counts (dstart) and of the global counts
  const uint32_t d = threadIdx.x;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) {
    const uint32_t cc = wcnt[w * NBIN + d];
    wcnt[w * NBIN + d] = run;
    run += cc;
  }
  // publish this tile's count of digit d, then look back for the earlier tiles'
  volatile uint32_t* vst = status;
  if (tile == 0) {
    vst[d] = kStInc | run;
  } else {
    vst[int64_t(tile) * NBIN + d] = kStAgg | run;
  }
  const uint32_t g = ghist[d];
  const uint32_t inc = warp_incl_scan(run), ginc = warp_incl_scan(g);
  if (lane == 31) {
    wsum[warp] = inc;
    gsum[warp] = ginc;
  }
  uint32_t excl = 0;
  if (tile > 0) {
    for (int64_t t = int64_t(tile) - 1; t >= 0; --t) {
      uint32_t s;
      do {
        s = vst[t * NBIN + d];
      } while ((s & ~kStVal) == 0);
      excl += s & kStVal;
      if (s & kStInc) break;
    }
    vst[int64_t(tile) * NBIN + d] = kStInc | (excl + run);
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = lane < kRadixWarps ? wsum[lane] : 0u, y = lane < kRadixWarps ? gsum[lane] : 0u;
    const uint32_t xi = warp_incl_scan(x), yi = warp_incl_scan(y);
    if (lane < kRadixWarps) {
      wsum[lane] = xi - x;
      gsum[lane] = yi - y;
    }
  }
  __syncthreads();
  dstart[d] = wsum[warp] + inc - run;
  gbase[d] = gsum[warp] + ginc - g + excl;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    if (base + k * 32 + lane < n) {
      const uint32_t dd = (key[k] >> shift) & (NBIN - 1);
      const uint32_t s = dstart[dd] + wcnt[warp * NBIN + dd] + lr[k];
      skeys[s] = key[k];
      svals[s] = val[k];
    }
  }
  __syncthreads();
  const int64_t tb = int64_t(tile) * kRadixTile;
  const int nvalid = n - tb < kRadixTile ? int(n - tb) : kRadixTile;
  for (int s = threadIdx.x; s < nvalid; s += kRadixThreads) {
    const uint32_t k2 = skeys[s];
    const uint32_t dd = (k2 >> shift) & (NBIN - 1);
    const uint32_t p = gbase[dd] + (uint32_t(s) - dstart[dd]);
    kout[p] = k2;
    vout[p] = svals[s];
  }
}

template <int DB>
static void radix_pass(const RadixScratch& rx, const uint32_t* sk, const int32_t* sv, uint32_t* dk, int32_t* dv,
                       int64_t n, int shift, int nb, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    NEST_CUDA(cudaFuncSetAttribute(k_radix_scatter<DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(radix_scatter_smem<DB>())));
    attr = true;
  }
  k_radix_hist<DB><<<nb, kRadixThreads, 0, st>>>(sk, n, shift, rx.hist, nb);
  uint32_t* h = rx.hist;
  scan_exclusive<uint32_t>([=] __device__(int64_t i) { return h[i]; }, int64_t(1u << DB) * nb,
                           [=] __device__(int64_t i, uint32_t v) { h[i] = v; }, rx.scan_tmp, st);
  k_radix_scatter<DB><<<nb, kRadixThreads, radix_scatter_smem<DB>(), st>>>(sk, sv, n, shift, rx.hist, nb, dk, dv);
  NEST_LAUNCH_CHECK();
}

// digit width of a sort of `bits`-bit keys: the fewest passes of <= kRadixMaxDigit bits
int radix_digit_bits(int bits) {
  if (bits <= 8) return 8;
  const int passes = (bits + kRadixMaxDigit - 1) / kRadixMaxDigit;
  const int db = (bits + passes - 1) / passes;
  return db < 8 ? 8 : db;
}

// stable LSD sort by the 8-bit digits at the given shifts, in order (the
// classic per-pass histogram + scan + scatter)
void radix_sort_pairs_shifts(const RadixScratch& rx, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                             int32_t* vout, int64_t n, const std::vector<int>& shifts, cudaStream_t st) {
  if (n <= 0 || shifts.empty()) return;
  const int nb = radix_blocks(n);
  const uint32_t* sk = kin;
  const int32_t* sv = vin;
  for (size_t p = 0; p < shifts.size(); ++p) {
    uint32_t* dk;
    int32_t* dv;
    if (p + 1 == shifts.size()) {
      dk = kout;
      dv = vout;
    } else {
      const int t = (sk == rx.tkey[0]) ? 1 : 0;
      dk = rx.tkey[t];
      dv = rx.tval[t];
    }
    radix_pass<8>(rx, sk, sv, dk, dv, n, shifts[p], nb, st);
    sk = dk;
    sv = dv;
  }
}

// NEST_RADIX=onesweep: the one-sweep sort above; default: per-pass histogram +
// scan + scatter.  Measured on DLRM W=1 (3.4M pairs, 3 passes): the one-sweep
// form makes the E step slower (1.55 vs 1.50 ms; 128 registers for the
// look-back kernel vs the classic scatter's, and the spin waits share the SMs
// with the window), so it is not the default.
static bool radix_classic() {
  static const bool v = [] {
    const char* e = std::getenv("NEST_RADIX");
    return !(e && std::string(e) == "onesweep");
  }();
  return v;
}

void radix_sort_pairs(const RadixScratch& rx, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                      int32_t* vout, int64_t n, int bits, cudaStream_t st) {
  if (n <= 0) return;
  const int db = radix_digit_bits(bits);
  const int passes = bits <= db ? 1 : (bits + db - 1) / db;
  const int nb = radix_blocks(n);
  if (!radix_classic() && db == 8 && passes <= 4) {
    static bool attr = false;
    if (!attr) {
      NEST_CUDA(cudaFuncSetAttribute(k_radix_onesweep<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(radix_scatter_smem<8>())));
      attr = true;
    }
    uint32_t* ghist = rx.aux;
    uint32_t* ctr = rx.aux + 4 * 256;
    NEST_CUDA(cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * passes * 256, st));
    k_radix_hist_all<<<std::min(nb, 148 * 4), kRadixThreads, 0, st>>>(kin, n, passes, db, ghist);
    const uint32_t* sk = kin;
    const int32_t* sv = vin;
    for (int p = 0; p < passes; ++p) {
      uint32_t* dk;
      int32_t* dv;
      if (p == passes - 1) {
        dk = kout;
        dv = vout;
      } else {
        const int t = (sk == rx.tkey[0]) ? 1 : 0;
        dk = rx.tkey[t];
        dv = rx.tval[t];
      }
      NEST_CUDA(cudaMemsetAsync(rx.hist, 0, sizeof(uint32_t) * 256 * size_t(nb), st));
      NEST_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
      k_radix_onesweep<8><<<nb, kRadixThreads, radix_scatter_smem<8>(), st>>>(sk, sv, n, db * p, ghist + p * 256,
                                                                            rx.hist, ctr, dk, dv);
      NEST_LAUNCH_CHECK();
      sk = dk;
      sv = dv;
    }
    return;
  }
  const uint32_t* sk = kin;
  const int32_t* sv = vin;
  for (int p = 0; p < passes; ++p) {
    uint32_t* dk;
    int32_t* dv;
    if (p == passes - 1) {
      dk = kout;
      dv = vout;
    } else {
      const int t = (sk == rx.tkey[0]) ? 1 : 0;
      dk = rx.tkey[t];
      dv = rx.tval[t];
    }
    static_assert(kRadixMaxDigit == 8, "instantiate radix_pass for the wider digits");
    radix_pass<8>(rx, sk, sv, dk, dv, n, db * p, nb, st);
    sk = dk;
    sv = dv;
  }
}

// ---------------------------------------------------------------------------
// phase A kernels
// ---------------------------------------------------------------------------
inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return int(b);
}

// per sample of the batch (position q in micro-batch order)
__global__ void k_sched_prep(int B, int cap, int F, int pooled, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ bag_off, int32_t* __restrict__ perm_out,
                             int32_t* __restrict__ mb_of, int32_t* __restrict__ samp_base,
                             int32_t* __restrict__ mbnnz) {
  __shared__ int32_t acc[NEST_MAX_MICRO_BATCHES];
  if (threadIdx.x < NEST_MAX_MICRO_BATCHES) acc[threadIdx.x] = 0;
  __syncthreads();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) {
    const int b = perm ? perm[q] : q;
    const int i = q / cap;
    perm_out[q] = b;
    mb_of[b] = i;
    if (pooled) samp_base[b] = (q - i * cap) * F;
    const int len = bag_off[int64_t(b + 1) * F] - bag_off[int64_t(b) * F];
    atomicAdd(&acc[i], len);
  }
  __syncthreads();
  if (threadIdx.x < NEST_MAX_MICRO_BATCHES && acc[threadIdx.x]) atomicAdd(&mbnnz[threadIdx.x], acc[threadIdx.x]);
}

// unpooled: samp_base[perm[q]] = excl[q] - excl[start of q's micro-batch]
__global__ void k_unpooled_base(int B, int cap, const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ excl, int32_t* __restrict__ samp_base) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x)
    samp_base[perm[q]] = excl[q] - excl[(q / cap) * cap];
}

// per bag: occ_mbrow[j] = mb << 28 | output row of occurrence j
template <bool kWarpPerBag>
__global__ void k_expand(int64_t nbags, int F, int pooled, const int32_t* __restrict__ bag_off,
                         const int32_t* __restrict__ mb_of, const int32_t* __restrict__ samp_base,
                         int32_t* __restrict__ occ_mbrow) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  const int64_t step = kWarpPerBag ? nth / 32 : nth;
  for (int64_t bag = kWarpPerBag ? tid / 32 : tid; bag < nbags; bag += step) {
    const int b = int(bag / F), f = int(bag - int64_t(b) * F);
    const int j0 = bag_off[bag], j1 = bag_off[bag + 1];
    const int32_t mbh = mb_of[b] << kMbShift;
    const int32_t sb = samp_base[b];
    const int32_t s0 = bag_off[int64_t(b) * F];
    for (int j = j0 + (kWarpPerBag ? lane_id() : 0); j < j1; j += kWarpPerBag ? 32 : 1)
      occ_mbrow[j] = mbh | (pooled ? sb + f : sb + (j - s0));
  }
}

// per occurrence: domain index + presence bit
__global__ void k_mark(const int64_t* __restrict__ keys, int64_t nnz, int T, int W,
                       const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_base,
                       uint32_t* __restrict__ occ_dom, uint32_t* __restrict__ bm,
                       int32_t* __restrict__ err) {
  const int lane = lane_id();
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
      } else {
        atomicOr(err, kErrKeyRange);
      }
      occ_dom[j] = dom;
      // test before the atomic: Zipf-hot keys find their bit already set
      const uint32_t bit = 1u << (dom & 31u);
      if (dom != 0xffffffffu && !(bm[dom >> 5] & bit)) atomicOr(&bm[dom >> 5], bit);
    }
  }
}

// per bitmap word: emit the set bits in ascending order
__global__ void k_emit(int64_t words, const uint32_t* __restrict__ bm, const int32_t* __restrict__ wr,
                       int T, int W, int nseg, uint32_t mask0, const int64_t* __restrict__ seg_base,
                       int64_t* __restrict__ uniq, uint32_t* __restrict__ mask,
                       int32_t* __restrict__ owner_rows) {
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
       w += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = bm[w];
    if (!x) continue;
    int32_t r = wr[w];
    // segment (owner, table) of the word's first bit: largest s with
    // seg_base[s] <= dom (seg_base[nseg] = V); segments span >= 1 row each,
    // so later bits of the word advance it at most a few steps
    const int64_t dom0 = w * 32 + (__ffs(x) - 1);
    int lo = 0, hi = nseg;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(seg_base + mid) <= dom0) lo = mid; else hi = mid;
    }
    int64_t sb = __ldg(seg_base + lo), se = __ldg(seg_base + lo + 1);
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      const int64_t dom = w * 32 + b;
      while (dom >= se) {
        ++lo;
        sb = se;
        se = __ldg(seg_base + lo + 1);
      }
      const int o = lo / T, t = lo - o * T;
      const int64_t row = (dom - sb) * W + o;
      uniq[r] = (int64_t(t) << kRowBits) | row;
      mask[r] = mask0;
      if (owner_rows) owner_rows[r] = int32_t(dom);
      ++r;
    }
  }
}

// off[o] = rank of the first domain index of owner o (o = 0..W)
__global__ void k_owner_offsets(int W, int T, const int64_t* __restrict__ seg_base,
                                const uint32_t* __restrict__ bm, const int32_t* __restrict__ wr,
                                int32_t* __restrict__ off) {
  const int o = threadIdx.x;
  if (o <= W) off[o] = bit_rank(bm, wr, uint32_t(seg_base[int64_t(o) * T]));
}

// per occurrence: inverse, micro-batch mask, sort key/value
// (one micro-batch: every key's mask is bit 0, written by k_emit; no OR pass)
template <bool kOneMb>
__global__ void k_inverse(int64_t nnz, const uint32_t* __restrict__ occ_dom,
                          const int32_t* __restrict__ occ_mbrow, const uint32_t* __restrict__ bm,
                          const int32_t* __restrict__ wr, int ubits, int32_t* __restrict__ inverse,
                          uint32_t* __restrict__ mask, uint32_t* __restrict__ skey,
                          int32_t* __restrict__ sval) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; j0 < nnz; j0 += nth) {
    const int64_t j = j0 + lane;
    uint32_t u = 0xffffffffu, bit = 0;
    if (j < nnz) {
      const uint32_t dom = occ_dom[j];
      const int32_t mr = occ_mbrow[j];
      const uint32_t mb = uint32_t(mr) >> kMbShift;
      if (dom != 0xffffffffu) {
        u = uint32_t(bit_rank(bm, wr, dom));
        bit = 1u << mb;
      }
      const uint32_t uu = u == 0xffffffffu ? 0u : u;
      inverse[j] = int32_t(uu);
      skey[j] = (mb << ubits) | uu;
      sval[j] = mr & int32_t(kRowFieldMask);
    }
    if (kOneMb) continue;
    const uint32_t peers = __match_any_sync(0xffffffffu, u);
    const uint32_t bits = __reduce_or_sync(peers, bit);
    if (u != 0xffffffffu && (peers & lt) == 0) atomicOr(&mask[u], bits);
  }
}

// per unique key: per (owner, micro-batch) counts
__global__ void k_mb_counts(const int32_t* __restrict__ off, int W, int N,
                            const uint32_t* __restrict__ mask, int32_t* __restrict__ cnt) {
  __shared__ int32_t sc[NEST_MAX_WORLD * NEST_MAX_MICRO_BATCHES];
  __shared__ int32_t soff[NEST_MAX_WORLD + 1];
  for (int i = threadIdx.x; i < W * N; i += blockDim.x) sc[i] = 0;
  for (int i = threadIdx.x; i <= W; i += blockDim.x) soff[i] = off[i];
  __syncthreads();
  const int U = soff[W];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    int o = 0;
    while (o + 1 < W && soff[o + 1] <= u) ++o;
    const uint32_t m = mask[u];
    for (int i = 0; i < N; ++i)
      if ((m >> i) & 1u) atomicAdd(&sc[o * N + i], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W * N; i += blockDim.x)
    if (sc[i]) atomicAdd(&cnt[i], sc[i]);
}

// this rank's row of the count exchange: per owner {U, U_1..U_N, err}
__global__ void k_finalize_counts(int W, int N, int Nc, const int32_t* __restrict__ off,
                                  const int32_t* __restrict__ cnt, const int32_t* __restrict__ err,
                                  int32_t* __restrict__ row) {
  for (int o = threadIdx.x; o < W; o += blockDim.x) {
    int32_t* r = row + int64_t(o) * Nc;
    r[0] = off[o + 1] - off[o];
    for (int i = 0; i < N; ++i) r[1 + i] = cnt[o * N + i];
    r[Nc - 1] = *err;
  }
}

// ---------------------------------------------------------------------------
// phase B (owner side, W > 1)
// ---------------------------------------------------------------------------
__global__ void k_pack(const int32_t* __restrict__ Uptr, const int64_t* __restrict__ uniq,
                       const uint32_t* __restrict__ mask, int64_t* __restrict__ packed) {
  const int U = *Uptr;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x)
    packed[u] = uniq[u] | (int64_t(mask[u]) << 56);
}

// R2 over the exchange window (route_window): this rank's count row stored
// straight into every peer's count area of the slot (same offset)
struct PeerI32 {
  int32_t* p[NEST_MAX_WORLD];
};
__global__ void k_push_counts(int W, int me, const int32_t* __restrict__ row, int n, PeerI32 dst) {
  for (int i = threadIdx.x; i < W * n; i += blockDim.x) {
    const int p = i / n, j = i % n;
    if (p != me) dst.p[p][j] = row[j];
  }
  __threadfence_system();
}

// R2 key All2All over the exchange window: uniq is sorted by owner, so owner
// p's keys are uniq[off[p] .. off[p+1]); each lands at this rank's receive
// offset in p's key area (blockIdx.y = owner; the self part is a local copy)
struct KeyDst {
  int64_t* base[NEST_MAX_WORLD];   // owner p's key area + this rank's receive offset there
  int32_t off[NEST_MAX_WORLD + 1];
};
__global__ void k_pack_push(const int64_t* __restrict__ uniq, const uint32_t* __restrict__ mask, KeyDst kd) {
  const int p = blockIdx.y;
  const int32_t a = kd.off[p], n = kd.off[p + 1] - a;
  int64_t* dst = kd.base[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = uniq[a + i] | (int64_t(mask[a + i]) << 56);
  __threadfence_system();
}

__global__ void k_owner_mark(int64_t R, const int64_t* __restrict__ recv, int T, int W, int rank,
                             const int64_t* __restrict__ rows, const int64_t* __restrict__ lbase,
                             uint32_t* __restrict__ r_ldom, uint32_t* __restrict__ bm,
                             int32_t* __restrict__ err) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; r0 < R; r0 += nth) {
    const int64_t r = r0 + lane;
    uint32_t ld = 0xffffffffu;
    if (r < R) {
      const uint64_t key = uint64_t(recv[r]) & kKeyMask56;
      const uint64_t t = key >> kRowBits, row = key & kRowMask;
      if (t < uint64_t(T) && row < uint64_t(__ldg(rows + t)) && row % uint64_t(W) == uint64_t(rank))
        ld = uint32_t(__ldg(lbase + t) + int64_t(row / uint64_t(W)));
      else
        atomicOr(err, kErrShard);
      r_ldom[r] = ld;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, ld);
    if (ld != 0xffffffffu && (peers & lt) == 0) atomicOr(&bm[ld >> 5], 1u << (ld & 31u));
  }
}

__global__ void k_owner_emit(int64_t words, const uint32_t* __restrict__ bm,
                             const int32_t* __restrict__ wr, int W, int32_t* __restrict__ owner_rows,
                             int32_t* __restrict__ src_tab) {
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
       w += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = bm[w];
    int32_t r = wr[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      owner_rows[r] = int32_t(w * 32 + b);
      for (int s = 0; s < W; ++s) src_tab[int64_t(r) * W + s] = -1;
      ++r;
    }
  }
}

struct Offs64 {
  int32_t v[NEST_MAX_WORLD + 1];
};

__global__ void k_owner_inv(int64_t R, const uint32_t* __restrict__ r_ldom,
                            const uint32_t* __restrict__ bm, const int32_t* __restrict__ wr, int W,
                            Offs64 roff, int32_t* __restrict__ owner_inv, int32_t* __restrict__ src_tab) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < R;
       r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t ld = r_ldom[r];
    if (ld == 0xffffffffu) {
      owner_inv[r] = 0;
      continue;
    }
    const int32_t u = bit_rank(bm, wr, ld);
    owner_inv[r] = u;
    int s = 0;
    while (s + 1 < W && roff.v[s + 1] <= r) ++s;
    src_tab[int64_t(u) * W + s] = int32_t(r);
  }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static int bits_for(int64_t n) {  // bits to represent values in [0, n)
  int b = 0;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

// bitmap popcount prefix: wr[i] = sum_{w<i} popc(bm[w]) for i in [0, nw]; n_out <- total
static void popc_scan(Ctx& c, const uint32_t* bm, int32_t* wr, int64_t nw, int32_t* total_out,
                      cudaStream_t st) {
  scan_exclusive<int32_t>(
      [=] __device__(int64_t i) { return int32_t(__popc(bm[i])); }, nw,
      [=] __device__(int64_t i, int32_t v) {
        wr[i] = v;
        if (total_out && i == nw) *total_out = v;
      },
      c.scan_tmp, st);
}

void route_phase_a(Ctx& c, Slot& s, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz,
                   int B, const int32_t* perm, int N, cudaStream_t st) {
  const int W = c.W, F = c.F, Nc = c.Nmax + 2;
  const bool pooled = c.cfg.pooling == NEST_POOL_SUM;
  s.N = N;
  s.B = B;
  s.cap = B / N;
  // source bitmap: the slot's own bitmap when W == 1 (it doubles as the owner
  // bitmap used by the refresh), the shared transient one otherwise
  uint32_t* bm = W == 1 ? s.obm : c.sbm;
  int32_t* wr = W == 1 ? s.owr : c.swr;
  NEST_CUDA(cudaMemsetAsync(bm, 0, sizeof(uint32_t) * (c.words + 2), st));
  int32_t* xfer = s.xfer;
  int32_t* mbnnz = xfer + int64_t(W) * W * Nc;
  NEST_CUDA(cudaMemsetAsync(mbnnz, 0, sizeof(int32_t) * (c.Nmax + 1), st));
  NEST_CUDA(cudaMemsetAsync(c.d_cnt_scratch, 0, sizeof(int32_t) * W * c.Nmax, st));
  NEST_CUDA(cudaMemcpyAsync(s.bag_off, bag_offsets, sizeof(int32_t) * (int64_t(B) * F + 1),
                            cudaMemcpyDeviceToDevice, st));
  // schedule: micro-batch of every sample and output row bases
  k_sched_prep<<<grid_for(B, 256), 256, 0, st>>>(B, s.cap, F, pooled ? 1 : 0, perm, s.bag_off,
                                                  s.perm, s.mb_of, s.samp_base, mbnnz);
  NEST_LAUNCH_CHECK();
  if (!pooled) {
    const int32_t* bo = s.bag_off;
    const int32_t* pm = s.perm;
    int32_t* tmp = c.samp_scratch;  // scratch [B+1]
    scan_exclusive<int32_t>(
        [=] __device__(int64_t q) {
          const int b = pm[q];
          return bo[int64_t(b + 1) * F] - bo[int64_t(b) * F];
        },
        B, [=] __device__(int64_t q, int32_t v) { tmp[q] = v; }, c.scan_tmp, st);
    k_unpooled_base<<<grid_for(B, 256), 256, 0, st>>>(B, s.cap, s.perm, tmp, s.samp_base);
  }
  const int64_t nbags = int64_t(B) * F;
  const bool long_bags = nbags > 0 && nnz / nbags >= 16;
  if (long_bags)
    k_expand<true><<<grid_for(nbags * 32, 256), 256, 0, st>>>(nbags, F, pooled, s.bag_off, s.mb_of,
                                                               s.samp_base, c.occ_mbrow);
  else
    k_expand<false><<<grid_for(nbags, 256), 256, 0, st>>>(nbags, F, pooled, s.bag_off, s.mb_of,
                                                           s.samp_base, c.occ_mbrow);
  NEST_LAUNCH_CHECK();
  // R1: mark, rank, emit
  k_mark<<<grid_for(nnz, 256), 256, 0, st>>>(keys, nnz, c.T, W, c.d_rows, c.d_seg_base, c.occ_dom, bm,
                                             c.d_err);
  NEST_LAUNCH_CHECK();
  popc_scan(c, bm, wr, c.words + 1, nullptr, st);
  k_emit<<<grid_for(c.words, 256), 256, 0, st>>>(c.words, bm, wr, c.T, W, W * c.T, N == 1 ? 1u : 0u,
                                                 c.d_seg_base,
                                                 s.uniq, s.mask, W == 1 ? s.owner_rows : nullptr);
  k_owner_offsets<<<1, 128, 0, st>>>(W, c.T, c.d_seg_base, bm, wr, s.off);
  s.ubits = bits_for(c.Kcap);
  if (N == 1)
    k_inverse<true><<<grid_for(nnz, 256), 256, 0, st>>>(nnz, c.occ_dom, c.occ_mbrow, bm, wr, s.ubits, s.inverse,
                                                        s.mask, s.rx.tkey[0], s.rx.tval[0]);
  else
    k_inverse<false><<<grid_for(nnz, 256), 256, 0, st>>>(nnz, c.occ_dom, c.occ_mbrow, bm, wr, s.ubits, s.inverse,
                                                         s.mask, s.rx.tkey[0], s.rx.tval[0]);
  k_mb_counts<<<grid_for(c.Kcap, 256, 148 * 4), 256, 0, st>>>(s.off, W, N, s.mask, c.d_cnt_scratch);
  k_finalize_counts<<<1, 64, 0, st>>>(W, N, Nc, s.off, c.d_cnt_scratch, c.d_err,
                                      xfer + int64_t(c.rank) * W * Nc);
  NEST_LAUNCH_CHECK();
  // R2: count exchange (every rank's counts and error flags to every rank)
  if (W > 1 && c.route_window) {
    // over the window: store the row into every peer, flag, wait for theirs
    const int si = slot_index(c, s);
    s.xep = ++c.xepoch;
    PeerI32 dst{};
    for (int p = 0; p < W; ++p) dst.p[p] = c.peer_cnt[si][p] + int64_t(c.rank) * W * Nc;
    k_push_counts<<<1, 256, 0, st>>>(W, c.rank, xfer + int64_t(c.rank) * W * Nc, W * Nc, dst);
    NEST_LAUNCH_CHECK();
    xfer_signal_raw(c, si, XK_CNT, 0, s.xep, st);
    xfer_wait_raw(c, si, XK_CNT, 0, s.xep, st);
  } else if (W > 1) {
    NEST_NCCL(ncclAllGather(xfer + int64_t(c.rank) * W * Nc, xfer, size_t(W) * Nc, ncclInt32,
                            c.comm_aux, st));
  }
  const size_t xbytes = sizeof(int32_t) * (int64_t(W) * W * Nc + c.Nmax + 1);
  NEST_CUDA(cudaMemcpyAsync(s.h_xfer, xfer, xbytes, cudaMemcpyDeviceToHost, st));
  NEST_CUDA(cudaEventRecord(s.ev_sync, st));
}

// The All2All plan of one batch from the gathered counts (pure host; every
// rank sees every rank's counts and error flags, so all ranks take the same
// error / capacity decision).  all: [W][W][Nmax+2], all[s][o] = what source s
// sends to owner o: {U, U_1..U_N, err}.
void exchange_plan(const Ctx& c, int N, const int32_t* all, nest_exchange_plan_t& p) {
  const int W = c.W, Nc = c.Nmax + 2;
  NEST_CHECK(N >= 1 && N <= c.Nmax, NEST_ERR_INVALID, "N out of range");
  auto A = [&](int src, int own, int col) { return int64_t(all[(size_t(src) * W + own) * Nc + col]); };
  int32_t err = 0;
  for (int r = 0; r < W; ++r)
    for (int o = 0; o < W; ++o) {
      err |= int32_t(A(r, o, Nc - 1));
      for (int col = 0; col <= N; ++col)
        NEST_CHECK(A(r, o, col) >= 0, NEST_ERR_INVALID, "negative count");
    }
  if (err & kErrKeyRange) throw Error{NEST_ERR_KEY_RANGE, "key out of range (table >= T or row >= rows[table])"};
  if (err & kErrShard) throw Error{NEST_ERR_SHARD, "owner received a key it does not own"};
  if (err & kErrSampleSize)
    throw Error{NEST_ERR_CAPACITY, "clustered schedule: a sample has more than 16383 distinct keys"};
  if (err & kErrCluster) throw Error{NEST_ERR_CAPACITY, "clustered schedule: an internal bound was exceeded"};
  for (int r = 0; r < W; ++r) {
    int64_t recv = 0, mbrows = 0, mbrecv = 0;
    for (int o = 0; o < W; ++o) {
      recv += A(o, r, 0);
      for (int i = 0; i < N; ++i) {
        mbrows += A(r, o, 1 + i);
        mbrecv += A(o, r, 1 + i);
      }
    }
    if (recv > c.Rcap) throw Error{NEST_ERR_CAPACITY, "owner receives more keys than max_recv_keys"};
    if (mbrows > c.MBcap) throw Error{NEST_ERR_CAPACITY, "micro-batch rows exceed max_mb_rows"};
    if (mbrecv > c.OMBcap) throw Error{NEST_ERR_CAPACITY, "owner micro-batch rows exceed max_owner_mb_rows"};
  }
  p = nest_exchange_plan_t{};
  for (int o = 0; o < W; ++o) p.key_send_off[o + 1] = p.key_send_off[o] + A(c.rank, o, 0);
  for (int r = 0; r < W; ++r) p.key_recv_off[r + 1] = p.key_recv_off[r] + A(r, c.rank, 0);
  p.uniq = p.key_send_off[W];
  p.recv = p.key_recv_off[W];
  for (int i = 0; i < N; ++i) {
    int64_t ui = 0, ri = 0;
    for (int o = 0; o < W; ++o) {
      ui += A(c.rank, o, 1 + i);
      ri += A(o, c.rank, 1 + i);
    }
    p.mb_uniq[i] = ui;
    p.mb_recv[i] = ri;
    p.src_base[i + 1] = p.src_base[i] + ui;
    p.own_base[i + 1] = p.own_base[i] + ri;
  }
}

// after the host sync: plan from the counts, then R1 tail, R2 keys, R3, R4
// after the host sync: the batch's All2All plan from the gathered counts
void route_plan(Ctx& c, Slot& s) {
  const int W = c.W, N = s.N, Nc = c.Nmax + 2;
  s.all.assign(size_t(W) * W * Nc, 0);
  for (size_t i = 0; i < s.all.size(); ++i) s.all[i] = s.h_xfer[i];
  const int32_t* hmbnnz = s.h_xfer + int64_t(W) * W * Nc;
  if (s.h_xfer[int64_t(W) * W * Nc + c.Nmax] & kErrKeyRange)
    throw Error{NEST_ERR_KEY_RANGE, "key out of range (table >= T or row >= rows[table])"};
  nest_exchange_plan_t plan;
  exchange_plan(c, N, s.h_xfer, plan);
  nest_slot_info_t& info = s.info;
  info = nest_slot_info_t{};
  info.num_micro_batches = N;
  info.batch = s.B;
  const int64_t U = plan.uniq, R = plan.recv;
  info.uniq = U;
  info.recv = R;
  s.src_base.assign(plan.src_base, plan.src_base + N + 1);
  s.own_base.assign(plan.own_base, plan.own_base + N + 1);
  s.q0.assign(N + 1, 0);
  int64_t nnz = 0;
  for (int i = 0; i < N; ++i) {
    info.mb_uniq[i] = plan.mb_uniq[i];
    info.mb_recv[i] = plan.mb_recv[i];
    info.mb_nnz[i] = hmbnnz[i];
    info.mb_out_rows[i] = c.cfg.pooling == NEST_POOL_SUM ? int64_t(s.cap) * c.F : hmbnnz[i];
    s.q0[i + 1] = s.q0[i] + hmbnnz[i];
    nnz += hmbnnz[i];
  }
  info.nnz = nnz;
  s.key_soff.assign(plan.key_send_off, plan.key_send_off + W + 1);
  s.key_roff.assign(plan.key_recv_off, plan.key_recv_off + W + 1);
}

// after route_plan: R1 tail, R2 keys, R3, R4 on `st`
void route_phase_b(Ctx& c, Slot& s, cudaStream_t st) {
  const int W = c.W, N = s.N, Nc = c.Nmax + 2, D = c.D;
  const int64_t U = s.info.uniq, R = s.info.recv;

  if (W == 1) {
    // owner == source: the owner-unique keys are the unique keys
    s.n_owner = s.off + 1;
  } else {
    {
      // ---- R2: key All2All (key | mask << 56), grouped send/recv ----
      ProfScope ps(c, ST_KEY_A2A, SK_AUX, st);
      if (c.route_window) {
        // keys stored straight into every owner's key area at this rank's
        // receive offset there (sources in rank order), then flagged
        const int si = slot_index(c, s);
        KeyDst kd{};
        int64_t mx = 1;
        for (int p = 0; p < W; ++p) {
          int64_t roff = 0;
          for (int r = 0; r < c.rank; ++r) roff += s.all[(size_t(r) * W + p) * Nc];
          kd.base[p] = c.peer_key[si][p] + roff;
          kd.off[p] = int32_t(s.key_soff[p]);
          mx = std::max<int64_t>(mx, s.key_soff[p + 1] - s.key_soff[p]);
        }
        kd.off[W] = int32_t(s.key_soff[W]);
        k_pack_push<<<dim3(unsigned(std::min<int64_t>((mx + 255) / 256, 148 * 2)), unsigned(W)), 256, 0, st>>>(
            s.uniq, s.mask, kd);
        NEST_LAUNCH_CHECK();
        xfer_signal_raw(c, si, XK_KEY, 0, s.xep, st);
        xfer_wait_raw(c, si, XK_KEY, 0, s.xep, st);
        ps.launches = 1;
        ps.bytes = 8.0 * double(U - (s.key_soff[c.rank + 1] - s.key_soff[c.rank]));  // off-GPU
      } else {
      k_pack<<<grid_for(c.Kcap, 256, 148 * 8), 256, 0, st>>>(s.off + W, s.uniq, s.mask, c.packed);
      NEST_LAUNCH_CHECK();
      NEST_NCCL(ncclGroupStart());
      for (int p = 0; p < W; ++p) {
        NEST_NCCL(ncclSend(c.packed + s.key_soff[p], size_t(s.key_soff[p + 1] - s.key_soff[p]), ncclInt64,
                           p, c.comm_aux, st));
        NEST_NCCL(ncclRecv(s.recv + s.key_roff[p], size_t(s.key_roff[p + 1] - s.key_roff[p]), ncclInt64,
                           p, c.comm_aux, st));
      }
      NEST_NCCL(ncclGroupEnd());
      ps.bytes = 8.0 * double(U - (s.key_soff[c.rank + 1] - s.key_soff[c.rank]));  // off-GPU
      }
    }
    {
      // ---- R3: owner dedup on the local domain ----
      ProfScope ps(c, ST_OWNER_DEDUP, SK_AUX, st);
      NEST_CUDA(cudaMemsetAsync(s.obm, 0, sizeof(uint32_t) * (c.owords + 2), st));
      if (R > 0)
        k_owner_mark<<<grid_for(R, 256), 256, 0, st>>>(R, s.recv, c.T, W, c.rank, c.d_rows, c.d_lbase,
                                                       c.r_ldom, s.obm, c.d_err);
      popc_scan(c, s.obm, s.owr, c.owords + 1, s.n_owner, st);
      k_owner_emit<<<grid_for(c.owords + 1, 256), 256, 0, st>>>(c.owords + 1, s.obm, s.owr, W,
                                                                s.owner_rows, s.src_tab);
      Offs64 roff{};
      for (int r = 0; r <= W; ++r) roff.v[r] = int32_t(s.key_roff[r]);
      if (R > 0)
        k_owner_inv<<<grid_for(R, 256), 256, 0, st>>>(R, c.r_ldom, s.obm, s.owr, W, roff, s.owner_inv,
                                                      s.src_tab);
      NEST_LAUNCH_CHECK();
      for (int i = 0; i < N; ++i) {
        const int64_t* rk = s.recv;
        int32_t* sp = s.sendpos + int64_t(i) * (c.Rcap + 1);
        scan_exclusive<int32_t>(
            [=] __device__(int64_t r) { return int32_t((uint64_t(rk[r]) >> (56 + i)) & 1u); }, R,
            [=] __device__(int64_t r, int32_t v) { sp[r] = v; }, c.scan_tmp, st);
      }
      ps.launches = 2 * (R > 0) + 3 + 1 + 3 * N;
      if (c.dwb && !s.zero_copy) {
        launch_upd_list(c, s, st);   // the keys the owner's update will touch
        ps.launches += 1;
      }
      ps.bytes = 12.0 * double(R);  // 12 R_o + 8 U_o
      ps.dcount = s.n_owner;
      ps.bpc = 8.0;
    }
  }
  {
    // ---- R4: gather the owned rows from the shard into the slot buffer ----
    // DBP (reading Q8): when the other slot's update is still to
    // come (pipelined: route(t+1) inside window t), its keys K(t) are skipped
    // here and supplied by nest_dbp_refresh from the written-back shard, so
    // this gather never waits for -- nor races -- that update; otherwise the
    // gather follows the other slot's update and reads its written-back rows
    Slot& o = c.slot[&s == &c.slot[0] ? 1 : 0];
    if (s.zero_copy) {
      // no retrieval copy: at W = 1 the window reads the shard in place after
      // the other slot's update (stream order on the compute lane, checked by
      // the lookup), so there is nothing stale to refresh; at W > 1 the
      // owner's rows leave from the shard (early push) and the requesters'
      // copies of the pending update's keys still need the re-push
      s.refresh_pending = c.W > 1 && s.skip_planned && o.routed;
      return;
    }
    const bool skip = s.skip_planned && o.routed;   // decided at nest_route_begin
    if (!skip && o.routed) NEST_CUDA(cudaStreamWaitEvent(st, o.ev_update, 0));
    s.refresh_pending = skip;
    ProfScope ps(c, ST_GATHER, SK_AUX, st);
    launch_gather(c, s, skip ? o.obm : nullptr, st);
    ps.dcount = c.n_refreshed + 2;          // rows copied (U_o minus the skipped ones)
    ps.bpc = 2.0 * c.D * sizeof(float);  // 2 U_o row
  }
  (void)D;
}

// R1 tail: per micro-batch positions of the keys among that micro-batch's
// keys (the pool and the segment-sum of this batch need them; nothing in the
// route does, so nest_route_end issues them after the gather and early push)
void route_positions(Ctx& c, Slot& s, cudaStream_t st) {
  const int N = s.N;
  const int64_t U = s.info.uniq;
  ProfScope ps(c, ST_ROUTE, SK_AUX, st);
  for (int i = 0; i < N; ++i) {
    const uint32_t* mk = s.mask;
    int32_t* pos = s.pos + int64_t(i) * (c.Kcap + 1);
    scan_exclusive<int32_t>([=] __device__(int64_t u) { return int32_t((mk[u] >> i) & 1u); }, U,
                            [=] __device__(int64_t u, int32_t v) { pos[u] = v; }, c.scan_tmp, st);
  }
  ps.launches = 3 * N;
  ps.bytes = double(U) * 4 * (1 + N);   // masks read + N positions written
}

// R1 tail: occurrences sorted by (micro-batch, key) -- the grouping of the
// deterministic segment-sum, first needed by the backward of this batch, so
// it runs after everything the next window's forward waits for
// The key is (mb << ubits) | u with ubits sized for the capacity K (fixed
// before the count sync); after it the batch's U_s is known and u < U_s, so
// only the digits of bits_for(U_s) (+ the micro-batch digit) can differ: e.g.
// gen-rec (K = 67M -> 27 bits, U_s = 5M -> 23 bits) sorts in 3 passes, not 4.
void route_sort(Ctx& c, Slot& s, cudaStream_t st) {
  int mbbits = 0;
  while ((1 << mbbits) < s.N) ++mbbits;
  const int64_t nnz = s.info.nnz;
  ProfScope ps(c, ST_SORT, SK_AUX, st);
  const int ub = std::min(bits_for(std::max<int64_t>(s.info.uniq, 2)), s.ubits);
  int passes;
  if (mbbits == 0) {
    radix_sort_pairs(s.rx, s.rx.tkey[0], s.rx.tval[0], s.skey, s.sval, nnz, ub, st);
    const int db = radix_digit_bits(ub);
    passes = ub <= db ? 1 : (ub + db - 1) / db;
  } else {
    // LSD over the u digits, then the micro-batch digit at ubits (a u digit
    // that also covers micro-batch bits only refines the order of the last
    // pass) -- or, when fewer passes, plain 8-bit digits over the whole
    // (mb << ubits | u) key: the bits between bits(U_s) and ubits are zero, so
    // e.g. DLRM N=2 (u < 2^21, ubits 22) sorts in 3 passes instead of 4
    std::vector<int> shifts;
    for (int sh = 0; sh < ub; sh += kRadixMaxDigit) shifts.push_back(sh);
    shifts.push_back(s.ubits);
    const int total = s.ubits + mbbits;
    if ((total + kRadixMaxDigit - 1) / kRadixMaxDigit < int(shifts.size())) {
      shifts.clear();
      for (int sh = 0; sh < total; sh += kRadixMaxDigit) shifts.push_back(sh);
    }
    radix_sort_pairs_shifts(s.rx, s.rx.tkey[0], s.rx.tval[0], s.skey, s.sval, nnz, shifts, st);
    passes = int(shifts.size());
  }
  ps.launches = nnz > 0 ? 5 * passes : 0;
  ps.bytes = double(nnz) * 16 * passes;   // every pass reads + writes (key, value)
}

}  // namespace nest
