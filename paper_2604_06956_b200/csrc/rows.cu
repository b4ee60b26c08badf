// Row-moving kernels of the hot path.  All are HBM-bound row copies / sums
// over fp32 rows of D floats, moved as 128-bit vectors by lane groups
// (RowGeom<D>): R4 prefetch gather, R6 send gather, R8 pool/expand, R10
// deterministic segment-sum, R12 fused owner reduce + SGD + write-back, R5
// dual-buffer refresh, N10 PRF table init.
#include "nest_internal.cuh"

namespace nest {

#define NEST_DISPATCH_D(dval, ...)                                       \
  switch (dval) {                                                        \
    case 16: { constexpr int D = 16; __VA_ARGS__; } break;               \
    case 32: { constexpr int D = 32; __VA_ARGS__; } break;               \
    case 64: { constexpr int D = 64; __VA_ARGS__; } break;               \
    case 128: { constexpr int D = 128; __VA_ARGS__; } break;             \
    case 256: { constexpr int D = 256; __VA_ARGS__; } break;             \
    default: throw Error{NEST_ERR_INVALID, "unsupported dim"};           \
  }

static inline int blocks_for_rows(int64_t rows, int rows_per_block, int max_blocks = 148 * 8) {
  int64_t b = (rows + rows_per_block - 1) / rows_per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return int(b);
}

constexpr int kRowThreads = 256;

// grid cap of the window's embedding-lane kernels (pool, segment-sum, send),
// which FWP runs concurrently with the dense tower: NEST_EMB_MAX_BLOCKS
static int emb_cap() {
  static int cap = [] {
    const char* e = std::getenv("NEST_EMB_MAX_BLOCKS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 148 * 16;
  }();
  return cap;
}
static inline int emb_blocks(int64_t rows, int rows_per_block) {
  return blocks_for_rows(rows, rows_per_block, emb_cap());
}

// independent segments / bags each lane group walks at once (their index
// chains and row loads overlap; every sum stays in its own sequential order):
// NEST_ROW_ILP = 1 (default), 2 or 4.  Measured on DLRM W=1:
// 2 and 4 are slower -- the extra registers halve occupancy and the random
// 512-byte row reads are bound by DRAM access efficiency, not by latency.
static int row_ilp() {
  static int v = [] {
    const char* e = std::getenv("NEST_ROW_ILP");
    const int x = e ? std::atoi(e) : 1;
    return x == 2 || x == 4 ? x : 1;
  }();
  return v;
}
#define NEST_DISPATCH_ILP(...)                                           \
  switch (row_ilp()) {                                                   \
    case 2: { constexpr int IL = 2; __VA_ARGS__; } break;                \
    case 4: { constexpr int IL = 4; __VA_ARGS__; } break;                \
    default: { constexpr int IL = 1; __VA_ARGS__; } break;               \
  }

// rows in flight per lane group in the streaming kernels: NEST_STREAM_U = 4 (default) or 8
static int stream_u() {
  static const int v = [] {
    const char* e = std::getenv("NEST_STREAM_U");
    return e && std::atoi(e) == 8 ? 8 : 4;
  }();
  return v;
}
// L2 prefetch (cp.async.bulk.prefetch.L2, one per row) of a chunk's rows as
// soon as its indices are known (NEST_PF bit mask: 1 segment-sum, 2 pool).
// Measured on DLRM W=1 (r02, 2 rounds each): pool 0.375 -> 0.327 ms in the E
// step (1.437 -> 1.388 ms), 0.398 -> 0.337 ms in E+T; the segment-sum does not
// gain (0.637 vs 0.645 ms).  Default: pool only.
static int pf_mask() {
  static const int v = [] {
    const char* e = std::getenv("NEST_PF");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
#define NEST_DISPATCH_U(...)                                             \
  if (stream_u() == 8) { constexpr int SU = 8; __VA_ARGS__; }            \
  else { constexpr int SU = 4; __VA_ARGS__; }

// resident blocks to ask of ptxas for a kernel holding IL row vectors per lane
// group in flight: full occupancy (32 registers) for one float4 per lane
template <int D>
constexpr int ilp_min_blocks(int il) {
  return il * RowGeom<D>::VPL <= 1 ? 8 : il * RowGeom<D>::VPL <= 2 ? 4 : 2;
}

// group id / count helpers for grid-stride loops over rows
template <int D>
struct Grp {
  using G = RowGeom<D>;
  int64_t g, ng;  // this group's index, number of groups in the grid
  int l;          // lane within the group
  __device__ Grp() {
    const int lane = lane_id();
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    g = warp * G::GPW + lane / G::L;
    ng = (int64_t(gridDim.x) * blockDim.x >> 5) * G::GPW;
    l = lane % G::L;
  }
  __device__ __forceinline__ int col(int v) const { return (v * G::L + l) * 4; }
};

template <int D>
__device__ __forceinline__ void copy_row(float* __restrict__ dst, const float* __restrict__ src,
                                         const Grp<D>& gp) {
#pragma unroll
  for (int v = 0; v < RowGeom<D>::VPL; ++v) st_f4(dst + gp.col(v), ld_f4(src + gp.col(v)));
}

// ---------------------------------------------------------------------------
// R4: buffer[u] = shard[owner_rows[u]], except the rows of skip_bm (the keys
// the other slot's pending update writes: the dual-buffer refresh copies
// their updated values after that update, so the gather and the update touch
// disjoint shard rows and need no ordering).  Counts the rows copied.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_gather(const float* __restrict__ shard,
                                                        const int32_t* __restrict__ rows,
                                                        const int32_t* __restrict__ n_dev,
                                                        const uint32_t* __restrict__ skip_bm,
                                                        float* __restrict__ out, int32_t* __restrict__ count) {
  Grp<D> gp;
  const int64_t n = *n_dev;
  constexpr int U = 4;
  int32_t local = 0;
  for (int64_t r0 = gp.g * U; r0 < n; r0 += gp.ng * U) {
    int32_t idx[U];
    bool take[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      idx[k] = r0 + k < n ? __ldg(rows + r0 + k) : 0;
      take[k] = r0 + k < n && !(skip_bm && bit_test(skip_bm, uint32_t(idx[k])));
    }
    float4 v[U][RowGeom<D>::VPL];
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < RowGeom<D>::VPL; ++q)
        if (take[k]) v[k][q] = ldg_f4(shard + int64_t(idx[k]) * D + gp.col(q));
#pragma unroll
    for (int k = 0; k < U; ++k) {
#pragma unroll
      for (int q = 0; q < RowGeom<D>::VPL; ++q)
        if (take[k]) st_f4(out + (r0 + k) * D + gp.col(q), v[k][q]);
      if (take[k] && gp.l == 0) ++local;
    }
  }
  if (local) atomicAdd(count, local);
}

void launch_gather(Ctx& c, Slot& s, const uint32_t* skip_bm, cudaStream_t st) {
  NEST_CUDA(cudaMemsetAsync(c.n_refreshed + 2, 0, sizeof(int32_t), st));
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW * 4;
    k_gather<D><<<blocks_for_rows(c.Uocap, rpb, 148 * 16), kRowThreads, 0, st>>>(
        c.shard, s.owner_rows, s.n_owner, skip_bm, s.buffer, c.n_refreshed + 2);
  });
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// R6 (owner, W > 1): send rows of micro-batch mb in (source, key) order
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_send_gather(int64_t R, int mb,
                                                             const int64_t* __restrict__ recv,
                                                             const int32_t* __restrict__ owner_inv,
                                                             const int32_t* __restrict__ sendpos,
                                                             const float* __restrict__ buffer,
                                                             float* __restrict__ out) {
  Grp<D> gp;
  for (int64_t r = gp.g; r < R; r += gp.ng) {
    if (!((uint64_t(__ldg(recv + r)) >> (56 + mb)) & 1u)) continue;
    const int64_t dst = __ldg(sendpos + r);
    const int64_t src = __ldg(owner_inv + r);
    copy_row<D>(out + dst * D, buffer + src * D, gp);
  }
}

void launch_send_gather(Ctx& c, Slot& s, int mb, cudaStream_t st, float* out_rows) {
  const int64_t R = s.info.recv;
  if (R == 0) return;
  float* out = (out_rows ? out_rows : c.own_rows) + s.own_base[mb] * c.D;
  const int32_t* sp = s.sendpos + int64_t(mb) * (c.Rcap + 1);
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    k_send_gather<D><<<emb_blocks(R, rpb), kRowThreads, 0, st>>>(
        R, mb, s.recv, s.owner_inv, sp, s.buffer, out);
  });
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// R8: pool (sum per bag, left to right) or expand (one row per occurrence)
// ---------------------------------------------------------------------------
// IL bags per lane group at once (bags q, q + ng, ...), two rows of each in
// flight per pass, each bag summed left to right
template <int D, bool W1, int IL, typename OutT>
__global__ void __launch_bounds__(kRowThreads, ilp_min_blocks<D>(IL)) k_pool(int64_t nrows, int F,
                                                      const int32_t* __restrict__ perm_mb,
                                                      const int32_t* __restrict__ bag_off,
                                                      const int32_t* __restrict__ inverse,
                                                      const int32_t* __restrict__ pos,
                                                      const float* __restrict__ src,
                                                      OutT* __restrict__ out) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL;
  for (int64_t q0 = gp.g; q0 < nrows; q0 += IL * gp.ng) {
    int j[IL], e[IL];
    int len = 0;
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const int64_t q = q0 + i * gp.ng;
      j[i] = e[i] = 0;
      if (q < nrows) {
        const int p = int(q / F), f = int(q - int64_t(p) * F);
        const int64_t bag = int64_t(__ldg(perm_mb + p)) * F + f;
        j[i] = __ldg(bag_off + bag);
        e[i] = __ldg(bag_off + bag + 1);
        len = max(len, e[i] - j[i]);
      }
    }
    float4 acc[IL][VPL];
#pragma unroll
    for (int i = 0; i < IL; ++i)
#pragma unroll
      for (int v = 0; v < VPL; ++v) acc[i][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int o = 0; o < len; o += 2) {
      int64_t r[IL][2];
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          r[i][t] = -1;
          if (j[i] + o + t < e[i]) {
            const int u = __ldg(inverse + j[i] + o + t);
            r[i][t] = W1 ? u : __ldg(pos + u);
          }
        }
      float4 x[IL][2][VPL];
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (r[i][t] >= 0) x[i][t][v] = ldg_f4(src + r[i][t] * D + gp.col(v));
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (r[i][t] >= 0) acc[i][v] = f4add(acc[i][v], x[i][t][v]);
    }
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const int64_t q = q0 + i * gp.ng;
      if (q < nrows)
#pragma unroll
        for (int v = 0; v < VPL; ++v) st_out4_cs(out + q * D + gp.col(v), acc[i][v]);
    }
  }
}

// unpooled: warp-group per sample of the micro-batch, rows in occurrence order
template <int D, bool W1>
__global__ void __launch_bounds__(kRowThreads) k_expand_rows(int nsamp, int F,
                                                             const int32_t* __restrict__ perm_mb,
                                                             const int32_t* __restrict__ bag_off,
                                                             const int32_t* __restrict__ samp_base,
                                                             const int32_t* __restrict__ inverse,
                                                             const int32_t* __restrict__ pos,
                                                             const float* __restrict__ src,
                                                             float* __restrict__ out) {
  Grp<D> gp;
  for (int64_t p = gp.g; p < nsamp; p += gp.ng) {
    const int b = __ldg(perm_mb + p);
    const int j0 = __ldg(bag_off + int64_t(b) * F), j1 = __ldg(bag_off + int64_t(b + 1) * F);
    const int64_t base = __ldg(samp_base + b);
    for (int j = j0; j < j1; ++j) {
      const int u = __ldg(inverse + j);
      const int64_t i = W1 ? u : __ldg(pos + u);
#pragma unroll
      for (int v = 0; v < RowGeom<D>::VPL; ++v)
        st_f4_cs(out + (base + (j - j0)) * D + gp.col(v), ldg_f4(src + i * D + gp.col(v)));
    }
  }
}

// ---------------------------------------------------------------------------
// Streaming forms of R8 and R10 (default).  A lane group owns a run of
// consecutive items (the occurrences of one sample's bags / a fixed range of
// sorted occurrences): it loads the run's indices with one coalesced load per
// L items, then streams the rows with U loads in flight, flushing a bag /
// segment when the next item belongs to the next one.  The index chain is paid
// once per L items instead of once per bag, and every row load of a batch is
// independent.  Summation order is unchanged for pooling (left to right from
// 0) and fixed for the segment-sum (see k_segsum_range).
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ uint32_t group_mask(const Grp<D>& gp) {
  constexpr int L = RowGeom<D>::L;
  return L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane_id() - gp.l));
}

// R8, pooled: lane group per sample of the micro-batch; bags of a sample are
// contiguous in the batch's CSR, so the sample's occurrences are one run
template <int D, bool W1, int U, typename OutT>
// resident blocks asked of ptxas: 4 (62 registers) measured best at W=1
// (E step 1.43 ms; 5 blocks / 51 registers 1.46, 6 blocks / 40 + spills 1.47)
#ifndef NEST_POOL_STREAM_MINB
#define NEST_POOL_STREAM_MINB 4
#endif
__global__ void __launch_bounds__(kRowThreads, NEST_POOL_STREAM_MINB) k_pool_stream(int64_t nsamp, int F,
                                                             const int32_t* __restrict__ perm_mb,
                                                             const int32_t* __restrict__ bag_off,
                                                             const int32_t* __restrict__ inverse,
                                                             const int32_t* __restrict__ pos,
                                                             const float* __restrict__ src,
                                                             OutT* __restrict__ out, int pf) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  const uint32_t gm = group_mask<D>(gp);
  for (int64_t p = gp.g; p < nsamp; p += gp.ng) {
    const int64_t bag0 = int64_t(__ldg(perm_mb + p)) * F;
    OutT* orow = out + p * F * D;
    int fb = 0;   // first bag of the window of bag ends the lanes hold
    int be = gp.l < F ? __ldg(bag_off + bag0 + gp.l + 1) : INT_MAX;
    const int j0 = __ldg(bag_off + bag0), j1 = __ldg(bag_off + bag0 + F);
    int f = 0;
    int cur_end = __shfl_sync(gm, be, 0, L);
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = j0; c0 < j1; c0 += L) {
      const int n = min(L, j1 - c0);
      int r_l = 0;
      if (gp.l < n) {
        const int u = __ldg(inverse + c0 + gp.l);
        r_l = W1 ? u : __ldg(pos + u);
        if (pf) prefetch_l2(src + int64_t(r_l) * D, D * sizeof(float));
      }
      for (int t0 = 0; t0 < n; t0 += U) {
        float4 x[U][VPL];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int r = __shfl_sync(gm, r_l, (t0 + k) & (L - 1), L);
          if (t0 + k < n)
#pragma unroll
            for (int v = 0; v < VPL; ++v) x[k][v] = ldg_f4(src + int64_t(r) * D + gp.col(v));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          if (t0 + k >= n) break;
          const int j = c0 + t0 + k;
          while (j >= cur_end) {   // bag f is complete (empty bags flush zeros)
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              st_out4_cs(orow + int64_t(f) * D + gp.col(v), acc[v]);
              acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            ++f;
            if (f - fb >= L) {
              fb += L;
              be = fb + gp.l < F ? __ldg(bag_off + bag0 + fb + gp.l + 1) : INT_MAX;
            }
            cur_end = __shfl_sync(gm, be, f - fb, L);
          }
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], x[k][v]);
        }
      }
    }
    for (; f < F; ++f)   // the last bag, then trailing empty bags
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        st_out4_cs(orow + int64_t(f) * D + gp.col(v), acc[v]);
        acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
  }
}

// R8 unpooled, streamed: lane group per sample, the sample's occurrence row
// indices loaded L at a time (coalesced), then U row copies in flight
template <int D, bool W1, int U>
__global__ void __launch_bounds__(kRowThreads) k_expand_stream(int nsamp, int F,
                                                               const int32_t* __restrict__ perm_mb,
                                                               const int32_t* __restrict__ bag_off,
                                                               const int32_t* __restrict__ samp_base,
                                                               const int32_t* __restrict__ inverse,
                                                               const int32_t* __restrict__ pos,
                                                               const float* __restrict__ src,
                                                               float* __restrict__ out) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  const uint32_t gm = group_mask<D>(gp);
  for (int64_t p = gp.g; p < nsamp; p += gp.ng) {
    const int b = __ldg(perm_mb + p);
    const int j0 = __ldg(bag_off + int64_t(b) * F), j1 = __ldg(bag_off + int64_t(b + 1) * F);
    float* orow = out + int64_t(__ldg(samp_base + b) - j0) * D;   // row of occurrence j: orow + j*D
    for (int c0 = j0; c0 < j1; c0 += L) {
      const int n = min(L, j1 - c0);
      int r_l = 0;
      if (gp.l < n) {
        const int u = __ldg(inverse + c0 + gp.l);
        r_l = W1 ? u : __ldg(pos + u);
      }
      for (int t0 = 0; t0 < n; t0 += U) {
        float4 x[U][VPL];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int r = __shfl_sync(gm, r_l, (t0 + k) & (L - 1), L);
          if (t0 + k < n)
#pragma unroll
            for (int v = 0; v < VPL; ++v) x[k][v] = ldg_f4(src + int64_t(r) * D + gp.col(v));
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
          if (t0 + k < n)
#pragma unroll
            for (int v = 0; v < VPL; ++v) st_f4_cs(orow + int64_t(c0 + t0 + k) * D + gp.col(v), x[k][v]);
      }
    }
  }
}

// pooling form: NEST_POOL = stream (default: k_pool_stream, lane group per
// sample) or bag (k_pool, lane group per bag, the r01 kernel)
static bool pool_by_bag() {
  static const bool v = [] {
    const char* e = std::getenv("NEST_POOL");
    return e && std::string(e) == "bag";
  }();
  return v;
}

void launch_pool(Ctx& c, Slot& s, int mb, void* out_v, bool bf16, cudaStream_t st) {
  float* out = reinterpret_cast<float*>(out_v);
  __nv_bfloat16* out_h = reinterpret_cast<__nv_bfloat16*>(out_v);
  // zero-copy (W = 1): the rows come straight from the shard, key u at shard
  // row owner_rows[u] (the non-W1 kernels' indirection); at W > 1 the rows
  // are the received ones either way
  const bool zc = s.zero_copy && c.W == 1;
  const bool w1 = c.W == 1 && !zc;
  const float* src = zc ? c.shard : w1 ? s.buffer : src_rows_of(c, s) + s.src_base[mb] * c.D;
  const int32_t* pos = zc ? s.owner_rows : s.pos + int64_t(mb) * (c.Kcap + 1);
  const int32_t* perm_mb = s.perm + int64_t(mb) * s.cap;
  const int pf = (pf_mask() >> 1) & 1;
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    if (c.cfg.pooling == NEST_POOL_SUM && !pool_by_bag()) {
      NEST_DISPATCH_U({
        if (bf16) {
          if (w1)
            k_pool_stream<D, true, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
                s.cap, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out_h, pf);
          else
            k_pool_stream<D, false, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
                s.cap, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out_h, pf);
        } else {
          if (w1)
            k_pool_stream<D, true, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
                s.cap, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out, pf);
          else
            k_pool_stream<D, false, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
                s.cap, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out, pf);
        }
      });
    } else if (c.cfg.pooling == NEST_POOL_SUM) {
      const int64_t nrows = int64_t(s.cap) * c.F;
      const int grid = emb_blocks(nrows, rpb);
      if (bf16) {
        if (w1)
          k_pool<D, true, 1><<<grid, kRowThreads, 0, st>>>(nrows, c.F, perm_mb, s.bag_off, s.inverse, pos, src,
                                                            out_h);
        else
          k_pool<D, false, 1><<<grid, kRowThreads, 0, st>>>(nrows, c.F, perm_mb, s.bag_off, s.inverse, pos, src,
                                                             out_h);
      } else {
        NEST_DISPATCH_ILP({
          if (w1)
            k_pool<D, true, IL><<<emb_blocks((nrows + IL - 1) / IL, rpb), kRowThreads, 0, st>>>(
                nrows, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out);
          else
            k_pool<D, false, IL><<<emb_blocks((nrows + IL - 1) / IL, rpb), kRowThreads, 0, st>>>(
                nrows, c.F, perm_mb, s.bag_off, s.inverse, pos, src, out);
        });
      }
    } else if (!pool_by_bag()) {
      NEST_DISPATCH_U({
        if (w1)
          k_expand_stream<D, true, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
              s.cap, c.F, perm_mb, s.bag_off, s.samp_base, s.inverse, pos, src, out);
        else
          k_expand_stream<D, false, SU><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
              s.cap, c.F, perm_mb, s.bag_off, s.samp_base, s.inverse, pos, src, out);
      });
    } else {
      if (w1)
        k_expand_rows<D, true><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
            s.cap, c.F, perm_mb, s.bag_off, s.samp_base, s.inverse, pos, src, out);
      else
        k_expand_rows<D, false><<<emb_blocks(s.cap, rpb), kRowThreads, 0, st>>>(
            s.cap, c.F, perm_mb, s.bag_off, s.samp_base, s.inverse, pos, src, out);
    }
  });
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// R10: deterministic segment-sum.  The occurrences of micro-batch mb are
// sorted by unique key (stable, so ascending occurrence order inside a key).
// Segment k (k = pos_mb[u]) sums dout[row] over its occurrences:
//   cold (L <= C): one lane group sums the L rows in order;
//   hot  (L > C): fixed chunks of C rows -> partial rows -> one block sums the
//   partials in a fixed strided order + fixed tree.  No float atomics, so
//   the result is bitwise reproducible run to run.
// ---------------------------------------------------------------------------

__global__ void k_seg_heads(int64_t Ki, const uint32_t* __restrict__ skey, uint32_t umask,
                            const int32_t* __restrict__ pos, int32_t* __restrict__ seg_start,
                            int64_t Ui) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < Ki;
       q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = skey[q] & umask;
    if (q == 0 || (skey[q - 1] & umask) != u) seg_start[pos[u]] = int32_t(q);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) seg_start[Ui] = int32_t(Ki);
}

template <int D>
__device__ __forceinline__ void sum_rows(const int32_t* __restrict__ sval, int64_t q0, int64_t q1,
                                         const float* __restrict__ dout, const Grp<D>& gp,
                                         float4 (&acc)[RowGeom<D>::VPL]) {
  constexpr int VPL = RowGeom<D>::VPL;
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t q = q0;
  for (; q + 3 < q1; q += 4) {
    int32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = __ldg(sval + q + k);
    float4 x[4][VPL];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int v = 0; v < VPL; ++v) x[k][v] = ldg_f4(dout + int64_t(r[k]) * D + gp.col(v));
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], x[k][v]);
  }
  for (; q < q1; ++q) {
    const int32_t r = __ldg(sval + q);
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], ldg_f4(dout + int64_t(r) * D + gp.col(v)));
  }
}

// segment of position p under a PeerRows map, and its destination row
__device__ __forceinline__ int map_seg(const PeerRows& m, int64_t p) {
  int s = 0;
  while (s + 1 < m.n && m.off[s + 1] <= p) ++s;
  return s;
}
__device__ __forceinline__ float* map_row(const PeerRows& m, int64_t p, int D) {
  const int s = map_seg(m, p);
  return m.base[s] + (p - m.off[s]) * D;
}

// owner side of the direct write-back: owner-unique key u is marked iff one
// requester asked for it, in one micro-batch (its gradient is then that
// requester's segment-sum row alone)
__device__ __forceinline__ bool sole_contributor(const int32_t* __restrict__ src_tab, int64_t u, int W,
                                                 const int64_t* __restrict__ recv) {
  int n = 0, r1 = -1;
  for (int s = 0; s < W; ++s) {
    const int32_t r = __ldg(src_tab + u * W + s);
    if (r >= 0) { ++n; r1 = r; }
  }
  return n == 1 && __popc(uint32_t(uint64_t(__ldg(recv + r1)) >> 56)) == 1;
}

// store gradient row k (one float4 per call) or, in fused-SGD mode, apply it:
// shard[owner_rows[k]] = fma(-lr, g, frozen buffer row k)  (Eq. 2)
__device__ __forceinline__ void put_grad(const PeerRows& m, int64_t k, int D, int col, float4 g) {
  if (m.sgd_shard) {
    const int64_t srow = __ldg(m.sgd_rows + k);
    float4 e = ldg_f4((m.sgd_inplace ? m.sgd_shard + srow * D : m.sgd_buffer + k * D) + col);
    e.x = __fmaf_rn(-m.sgd_lr, g.x, e.x);
    e.y = __fmaf_rn(-m.sgd_lr, g.y, e.y);
    e.z = __fmaf_rn(-m.sgd_lr, g.z, e.z);
    e.w = __fmaf_rn(-m.sgd_lr, g.w, e.w);
    st_f4_cs(m.sgd_shard + srow * D + col, e);
  } else if (m.dwb_rows) {
    // W > 1: a sole-contributor key is applied here (Eq. 2 on the received
    // frozen copy) and written back into its owner's shard; any other key's
    // gradient row goes to its owner's receive rows
    const int32_t srow = __ldg(m.dwb_rows + k);
    const int s = map_seg(m, k);
    if (srow >= 0) {
      float4 e = ldg_f4(m.sgd_buffer + k * D + col);
      e.x = __fmaf_rn(-m.sgd_lr, g.x, e.x);
      e.y = __fmaf_rn(-m.sgd_lr, g.y, e.y);
      e.z = __fmaf_rn(-m.sgd_lr, g.z, e.z);
      e.w = __fmaf_rn(-m.sgd_lr, g.w, e.w);
      st_f4(m.dwb_shard[s] + int64_t(srow) * D + col, e);
    } else {
      st_f4(m.base[s] + (k - m.off[s]) * D + col, g);
    }
  } else {
    st_f4(map_row(m, k, D) + col, g);
  }
}

// IL cold segments per lane group at once (k, k + ng, ...), two rows of each
// in flight per pass, each segment summed in occurrence order
// fused one-rank update of key k's gradient row with row-wise AdaGrad: every
// lane of the row's group calls it (converged), `valid` marks a real row
template <int D>
__device__ __forceinline__ void put_row_adagrad(const PeerRows& m, int64_t k, bool valid,
                                                float4 (&acc)[RowGeom<D>::VPL], int l) {
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  const int lane = lane_id();
  const uint32_t gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane - l));
  float sq = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    acc[v] = make_float4(m.ada_gscale * acc[v].x, m.ada_gscale * acc[v].y, m.ada_gscale * acc[v].z,
                         m.ada_gscale * acc[v].w);
    sq = __fmaf_rn(acc[v].x, acc[v].x, sq);
    sq = __fmaf_rn(acc[v].y, acc[v].y, sq);
    sq = __fmaf_rn(acc[v].z, acc[v].z, sq);
    sq = __fmaf_rn(acc[v].w, acc[v].w, sq);
  }
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) sq += __shfl_xor_sync(gmask, sq, o);
  const int64_t srow = valid ? __ldg(m.sgd_rows + k) : 0;
  float mm = 0.f;
  if (valid && l == 0) {
    mm = m.ada_state[srow] + sq * (1.f / float(D));
    m.ada_state[srow] = mm;
  }
  mm = __shfl_sync(gmask, mm, lane - l);
  if (!valid) return;
  const float step = m.sgd_lr / (sqrtf(mm) + m.ada_eps);
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int col = (v * L + l) * 4;
    float4 e = ldg_f4((m.sgd_inplace ? m.sgd_shard + srow * D : m.sgd_buffer + k * D) + col);
    e.x = __fmaf_rn(-step, acc[v].x, e.x);
    e.y = __fmaf_rn(-step, acc[v].y, e.y);
    e.z = __fmaf_rn(-step, acc[v].z, e.z);
    e.w = __fmaf_rn(-step, acc[v].w, e.w);
    st_f4_cs(m.sgd_shard + srow * D + col, e);
  }
}

template <int D, int IL>
__global__ void __launch_bounds__(kRowThreads, ilp_min_blocks<D>(IL)) k_segsum_cold(int64_t Ui, int chunk,
                                                             const int32_t* __restrict__ seg_start,
                                                             const int32_t* __restrict__ sval,
                                                             const float* __restrict__ dout,
                                                             const PeerRows out) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL;
  // warp-uniform trip count (the AdaGrad row reduction shuffles)
  for (int64_t k0 = gp.g; __any_sync(0xffffffffu, k0 < Ui); k0 += IL * gp.ng) {
    int a[IL], b[IL];
    int len = 0;
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const int64_t k = k0 + i * gp.ng;
      a[i] = b[i] = 0;
      if (k < Ui) {
        a[i] = seg_start[k];
        b[i] = seg_start[k + 1];
        if (b[i] - a[i] > chunk) b[i] = a[i] - 1;   // hot: the chunked kernels own it
        len = max(len, b[i] - a[i]);
      }
    }
    float4 acc[IL][VPL];
#pragma unroll
    for (int i = 0; i < IL; ++i)
#pragma unroll
      for (int v = 0; v < VPL; ++v) acc[i][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int o = 0; o < len; o += 2) {
      int32_t r[IL][2];
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t) r[i][t] = a[i] + o + t < b[i] ? __ldg(sval + a[i] + o + t) : -1;
      float4 x[IL][2][VPL];
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (r[i][t] >= 0) x[i][t][v] = ldg_f4(dout + int64_t(r[i][t]) * D + gp.col(v));
#pragma unroll
      for (int i = 0; i < IL; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (r[i][t] >= 0) acc[i][v] = f4add(acc[i][v], x[i][t][v]);
    }
#pragma unroll
    for (int i = 0; i < IL; ++i) {
      const int64_t k = k0 + i * gp.ng;
      const bool valid = k < Ui && b[i] >= a[i];
      if (out.ada) {
        put_row_adagrad<D>(out, k, valid, acc[i], gp.l);
      } else if (valid) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) put_grad(out, k, D, gp.col(v), acc[i][v]);
      }
    }
  }
  if (out.fence) __threadfence_system();
}

template <int D>
__global__ void __launch_bounds__(kRowThreads) k_segsum_hot_chunks(
    int chunk, const int32_t* __restrict__ tot, const int32_t* __restrict__ hot_list,
    const int32_t* __restrict__ hot_ppos, const int32_t* __restrict__ seg_start,
    const int32_t* __restrict__ sval, const float* __restrict__ dout, float* __restrict__ partial) {
  Grp<D> gp;
  const int H = tot[0], P = tot[1];
  for (int64_t cidx = gp.g; cidx < P; cidx += gp.ng) {
    int lo = 0, hi = H;  // largest h with hot_ppos[h] <= cidx
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (hot_ppos[mid] <= cidx) lo = mid; else hi = mid;
    }
    const int k = hot_list[lo];
    const int64_t m = cidx - hot_ppos[lo];
    const int64_t a = seg_start[k] + m * chunk;
    const int64_t e = seg_start[k + 1];
    const int64_t b = e < a + chunk ? e : a + chunk;
    float4 acc[RowGeom<D>::VPL];
    sum_rows<D>(sval, a, b, dout, gp, acc);
#pragma unroll
    for (int v = 0; v < RowGeom<D>::VPL; ++v) st_f4(partial + cidx * D + gp.col(v), acc[v]);
  }
}

template <int D>
__global__ void __launch_bounds__(kRowThreads) k_segsum_hot_final(
    const int32_t* __restrict__ tot, const int32_t* __restrict__ hot_list,
    const int32_t* __restrict__ hot_ppos, const float* __restrict__ partial, const PeerRows out) {
  using G = RowGeom<D>;
  constexpr int NG = (kRowThreads / 32) * G::GPW;  // groups per block
  __shared__ float4 red[NG][G::kVec];
  const int H = tot[0];
  const int lane = lane_id();
  const int grp = (threadIdx.x >> 5) * G::GPW + lane / G::L;
  const int l = lane % G::L;
  for (int h = blockIdx.x; h < H; h += gridDim.x) {
    const int k = hot_list[h];
    const int64_t p0 = hot_ppos[h], np = hot_ppos[h + 1] - p0;
    float4 acc[G::VPL];
#pragma unroll
    for (int v = 0; v < G::VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t m = grp; m < np; m += NG)
#pragma unroll
      for (int v = 0; v < G::VPL; ++v)
        acc[v] = f4add(acc[v], ld_f4(partial + (p0 + m) * D + (v * G::L + l) * 4));
#pragma unroll
    for (int v = 0; v < G::VPL; ++v) red[grp][v * G::L + l] = acc[v];
    __syncthreads();
    if (grp == 0) {
      float4 row[G::VPL];
#pragma unroll
      for (int v = 0; v < G::VPL; ++v) {
        float4 s = red[0][v * G::L + l];
        for (int q = 1; q < NG; ++q) s = f4add(s, red[q][v * G::L + l]);
        row[v] = s;
      }
      if (out.ada) {
        put_row_adagrad<D>(out, k, true, row, l);
      } else {
#pragma unroll
        for (int v = 0; v < G::VPL; ++v) put_grad(out, k, D, (v * G::L + l) * 4, row[v]);
      }
    }
    __syncthreads();
  }
  if (out.fence) __threadfence_system();
}

// R10 over fixed ranges of kSegRange sorted occurrences: range w = [w*R, w*R+R).
// A segment (key) that starts and ends inside a range is summed in occurrence
// order and finished there (stored, or with the fused update applied).  A
// segment cut by range boundaries leaves partial rows: B[w] for its part in the
// range where it starts, A[w'] for its part in each later range; the range
// where it starts lists itself, and k_segsum_fix sums B[w] + A[w+1] + ... in
// range order.  Fixed ranges => a fixed summation order => bitwise
// reproducible, whatever the grid; load balance does not depend on skew.
// L2 eviction hints in k_segsum_range: dout rows evict_last (read once per
// occurrence), frozen rows evict_first (read once)
#ifndef NEST_SEGSUM_L2HINT
#define NEST_SEGSUM_L2HINT 0
#endif
#ifndef NEST_SEG_RANGE
#define NEST_SEG_RANGE 256
#endif
constexpr int kSegRange = NEST_SEG_RANGE;
// c.partial holds Pcap = 2 * Kcap / 32 + 64 rows (api.cu) >= 2 * ceil(K / R) for R >= 32
static_assert(kSegRange >= 32, "NEST_SEG_RANGE must be >= 32 (partial-row capacity)");
// resident 256-thread blocks asked of ptxas for k_segsum_range (2: ~98
// registers, 3: capped at 85)
#ifndef NEST_SEGSUM_RANGE_MINB
#define NEST_SEGSUM_RANGE_MINB 3
#endif

template <int D>
__device__ __forceinline__ void finish_row(const PeerRows& out, int64_t k, float4 (&acc)[RowGeom<D>::VPL],
                                           const Grp<D>& gp) {
  if (out.ada) {
    put_row_adagrad<D>(out, k, true, acc, gp.l);
  } else {
#pragma unroll
    for (int v = 0; v < RowGeom<D>::VPL; ++v) put_grad(out, k, D, gp.col(v), acc[v]);
  }
}

// a finished segment: fused update with the prefetched frozen row (PRE), or
// the store / AdaGrad of finish_row
template <int D, bool PRE>
__device__ __forceinline__ void seg_finish(const PeerRows& out, int32_t k, int32_t srow,
                                           const float4 (&ecur)[RowGeom<D>::VPL], float4 (&g)[RowGeom<D>::VPL],
                                           const Grp<D>& gp) {
  if (PRE) {
#pragma unroll
    for (int v = 0; v < RowGeom<D>::VPL; ++v) {
      float4 e = ecur[v];
      e.x = __fmaf_rn(-out.sgd_lr, g[v].x, e.x);
      e.y = __fmaf_rn(-out.sgd_lr, g[v].y, e.y);
      e.z = __fmaf_rn(-out.sgd_lr, g[v].z, e.z);
      e.w = __fmaf_rn(-out.sgd_lr, g[v].w, e.w);
      st_f4_cs(out.sgd_shard + int64_t(srow) * D + gp.col(v), e);
    }
  } else {
    finish_row<D>(out, k, g, gp);
  }
}

// PRE: fused SGD (W == 1, N == 1, plain SGD) with the frozen rows prefetched
// alongside the gradient row of the segment's first occurrence
template <int D, int U, bool PRE>
__global__ void __launch_bounds__(kRowThreads, NEST_SEGSUM_RANGE_MINB) k_segsum_range(int64_t Ki, const uint32_t* __restrict__ skey,
                                                              uint32_t umask, const int32_t* __restrict__ pos,
                                                              const int32_t* __restrict__ sval,
                                                              const float* __restrict__ dout, const PeerRows out,
                                                              float* __restrict__ partial,
                                                              int32_t* __restrict__ olist,
                                                              int32_t* __restrict__ ocount, int pf) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  const uint32_t gm = group_mask<D>(gp);
  const int64_t nr = (Ki + kSegRange - 1) / kSegRange;
  // L2 policies created once per thread (NEST_SEGSUM_L2HINT builds only)
  const uint64_t pol_el = NEST_SEGSUM_L2HINT ? l2_policy_evict_last() : 0;
  const uint64_t pol_ef = NEST_SEGSUM_L2HINT ? l2_policy_evict_first() : 0;
  for (int64_t w = gp.g; w < nr; w += gp.ng) {
    const int64_t q0 = w * kSegRange, q1 = (q0 + kSegRange < Ki ? q0 + kSegRange : Ki);
    const uint32_t ufirst = __ldg(skey + q0) & umask;
    const bool carry_in = q0 > 0 && (__ldg(skey + q0 - 1) & umask) == ufirst;
    const bool carry_out = q1 < Ki && (__ldg(skey + q1) & umask) == (__ldg(skey + q1 - 1) & umask);
    bool open = carry_in, part_a = carry_in;   // segment open; it started before q0
    int32_t kcur = 0, srow = 0;
    uint32_t uprev = carry_in ? ufirst : 0xffffffffu;
    float4 acc[VPL], ecur[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = ecur[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t c0 = q0; c0 < q1; c0 += L) {
      const int n = int(q1 - c0 < L ? q1 - c0 : L);
      uint32_t u_l = 0xfffffffeu;
      int32_t r_l = 0, k_l = 0, s_l = 0;
      if (gp.l < n) {
        u_l = __ldg(skey + c0 + gp.l) & umask;
        r_l = __ldg(sval + c0 + gp.l);
        if (pf) prefetch_l2(dout + int64_t(r_l) * D, D * sizeof(float));
      }
      uint32_t up = __shfl_up_sync(gm, u_l, 1, L);
      if (gp.l == 0) up = uprev;
      const bool head = gp.l < n && u_l != up;
      if (head) {
        k_l = __ldg(pos + u_l);
        if (PRE) {
          s_l = __ldg(out.sgd_rows + k_l);
          if (pf)
            prefetch_l2(out.sgd_inplace ? out.sgd_shard + int64_t(s_l) * D : out.sgd_buffer + int64_t(k_l) * D,
                        D * sizeof(float));
        }
      }
      const uint32_t heads = __ballot_sync(gm, head) >> (lane_id() - gp.l);
      uprev = __shfl_sync(gm, u_l, n - 1, L);
      for (int t0 = 0; t0 < n; t0 += U) {
        float4 x[U][VPL], ex[U][VPL];
        int32_t kk[U], ss[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int t = t0 + k, sl = t & (L - 1);
          const int32_t r = __shfl_sync(gm, r_l, sl, L);
          kk[k] = __shfl_sync(gm, k_l, sl, L);
          ss[k] = PRE ? __shfl_sync(gm, s_l, sl, L) : 0;
          if (t < n) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              x[k][v] = NEST_SEGSUM_L2HINT ? ldg_f4_hint(dout + int64_t(r) * D + gp.col(v), pol_el)
                                           : ldg_f4(dout + int64_t(r) * D + gp.col(v));
            if (PRE && ((heads >> t) & 1u)) {
              const float* fr = out.sgd_inplace ? out.sgd_shard + int64_t(ss[k]) * D
                                                : out.sgd_buffer + int64_t(kk[k]) * D;
#pragma unroll
              for (int v = 0; v < VPL; ++v)
                ex[k][v] = NEST_SEGSUM_L2HINT ? ldg_f4_hint(fr + gp.col(v), pol_ef) : ldg_f4(fr + gp.col(v));
            }
          }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int t = t0 + k;
          if (t >= n) break;
          if ((heads >> t) & 1u) {
            if (open) {   // the previous segment ends here
              if (part_a) {
#pragma unroll
                for (int v = 0; v < VPL; ++v) st_f4(partial + w * D + gp.col(v), acc[v]);
              } else {
                seg_finish<D, PRE>(out, kcur, srow, ecur, acc, gp);
              }
            }
            open = true;
            part_a = false;
            kcur = kk[k];
            srow = ss[k];
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              if (PRE) ecur[v] = ex[k][v];
              acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], x[k][v]);
        }
      }
    }
    // the segment open at the range end
    if (carry_out || part_a) {
      float* dst = partial + (part_a ? w : nr + w) * D;
#pragma unroll
      for (int v = 0; v < VPL; ++v) st_f4(dst + gp.col(v), acc[v]);
      if (carry_out && !part_a && gp.l == 0) olist[atomicAdd(ocount, 1)] = int32_t(w);
    } else {
      seg_finish<D, PRE>(out, kcur, srow, ecur, acc, gp);
    }
  }
  if (out.fence) __threadfence_system();
}

// last range of the segment that starts in range w and continues past it
__device__ __forceinline__ int64_t seg_last_range(int64_t Ki, const uint32_t* __restrict__ skey, uint32_t umask,
                                                  int64_t w, uint32_t u) {
  const int64_t nr = (Ki + kSegRange - 1) / kSegRange;
  auto through = [&](int64_t r) {   // the segment continues past range r
    return r + 1 < nr && (__ldg(skey + (r + 1) * kSegRange) & umask) == u;
  };
  // through(w) holds (w's carry-out); the last range is the first r > w without it
  int64_t lo = w, hi = w + 1, step = 1;
  while (hi < nr - 1 && through(hi)) {
    lo = hi;
    step <<= 1;
    hi = min(lo + step, nr - 1);
  }
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (through(mid)) lo = mid; else hi = mid;
  }
  return hi;
}

constexpr int kFixWarpMax = 64;   // partials a lane group sums itself; more go to k_segsum_fix_big

// cut segments: B[w] + A[w+1] + ... + A[wb] in range order
template <int D, int U>
__global__ void __launch_bounds__(kRowThreads) k_segsum_fix(int64_t Ki, const uint32_t* __restrict__ skey,
                                                            uint32_t umask, const int32_t* __restrict__ pos,
                                                            const int32_t* __restrict__ olist,
                                                            const int32_t* __restrict__ ocount,
                                                            const float* __restrict__ partial, const PeerRows out,
                                                            int32_t* __restrict__ big, int32_t* __restrict__ nbig) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL;
  const int64_t nr = (Ki + kSegRange - 1) / kSegRange;
  const int n = *ocount;
  for (int64_t e = gp.g; e < n; e += gp.ng) {
    const int64_t w = olist[e];
    const int64_t q1 = ((w + 1) * kSegRange < Ki ? (w + 1) * kSegRange : Ki);
    const uint32_t u = __ldg(skey + q1 - 1) & umask;
    const int64_t wb = seg_last_range(Ki, skey, umask, w, u);
    const int32_t k = __ldg(pos + u);
    if (wb - w + 1 > kFixWarpMax) {
      if (gp.l == 0) {
        const int b = atomicAdd(nbig, 1);
        big[3 * b] = int32_t(w);
        big[3 * b + 1] = int32_t(wb);
        big[3 * b + 2] = k;
      }
      continue;
    }
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = ld_f4(partial + (nr + w) * D + gp.col(v));
    for (int64_t r = w + 1; r <= wb; r += U) {
      float4 x[U][VPL];
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (r + i <= wb)
#pragma unroll
          for (int v = 0; v < VPL; ++v) x[i][v] = ld_f4(partial + (r + i) * D + gp.col(v));
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (r + i <= wb)
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], x[i][v]);
    }
    finish_row<D>(out, k, acc, gp);
  }
  if (out.fence) __threadfence_system();
}

// cut segments with more than kFixWarpMax partials: one block each, groups
// sum strided partials (p = 0: B[w], p >= 1: A[w+p]), then a fixed sequential
// combine of the group sums
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_segsum_fix_big(int64_t Ki, const int32_t* __restrict__ big,
                                                                const int32_t* __restrict__ nbig,
                                                                const float* __restrict__ partial, const PeerRows out) {
  using G = RowGeom<D>;
  constexpr int NG = (kRowThreads / 32) * G::GPW;
  __shared__ float4 red[NG][G::kVec];
  const int64_t nr = (Ki + kSegRange - 1) / kSegRange;
  const int lane = lane_id();
  const int grp = (threadIdx.x >> 5) * G::GPW + lane / G::L;
  const int l = lane % G::L;
  const int nb = *nbig;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t w = big[3 * b], wb = big[3 * b + 1];
    const int32_t k = big[3 * b + 2];
    const int64_t np = wb - w + 1;
    float4 acc[G::VPL];
#pragma unroll
    for (int v = 0; v < G::VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t m = grp; m < np; m += NG) {
      const int64_t prow = m == 0 ? nr + w : w + m;
#pragma unroll
      for (int v = 0; v < G::VPL; ++v) acc[v] = f4add(acc[v], ld_f4(partial + prow * D + (v * G::L + l) * 4));
    }
#pragma unroll
    for (int v = 0; v < G::VPL; ++v) red[grp][v * G::L + l] = acc[v];
    __syncthreads();
    if (grp == 0) {
      float4 row[G::VPL];
#pragma unroll
      for (int v = 0; v < G::VPL; ++v) {
        float4 s = red[0][v * G::L + l];
        for (int q = 1; q < NG; ++q) s = f4add(s, red[q][v * G::L + l]);
        row[v] = s;
      }
      if (out.ada) {
        put_row_adagrad<D>(out, k, true, row, l);
      } else {
#pragma unroll
        for (int v = 0; v < G::VPL; ++v) put_grad(out, k, D, (v * G::L + l) * 4, row[v]);
      }
    }
    __syncthreads();
  }
  if (out.fence) __threadfence_system();
}

// local gradient rows of micro-batch mb (NCCL / CE transports send them)
void launch_segsum(Ctx& c, Slot& s, int mb, const float* dout, cudaStream_t st) {
  PeerRows out{};
  out.base[0] = src_rows_of(c, s) + s.src_base[mb] * c.D;
  out.off[0] = 0;
  out.off[1] = int32_t(s.info.mb_uniq[mb]);
  out.n = 1;
  out.fence = 0;
  launch_segsum_to(c, s, mb, dout, out, st);
}

// R10 + R12 fused for W == 1, N == 1: each key's gradient is its only
// contribution, so the segment-sum applies the SGD update and writes the row
// back directly (no gradient rows stored and re-read)
void launch_segsum_sgd(Ctx& c, Slot& s, const float* dout, const OptStep& opt, cudaStream_t st) {
  PeerRows out{};
  out.base[0] = c.src_rows;
  out.off[0] = 0;
  out.off[1] = int32_t(s.info.mb_uniq[0]);
  out.n = 1;
  out.sgd_buffer = s.buffer;
  out.sgd_inplace = s.zero_copy ? 1 : 0;
  out.sgd_rows = s.owner_rows;
  out.sgd_shard = c.shard;
  out.sgd_lr = opt.lr;
  out.ada = opt.kind == NEST_OPT_ROWWISE_ADAGRAD;
  out.ada_gscale = opt.gscale;
  out.ada_eps = opt.eps;
  out.ada_state = opt.state;
  launch_segsum_to(c, s, 0, dout, out, st);
}

// R6 + R7 fused: the owner's gather writes every requested row straight into
// the requester's receive rows (peer memory over NVLink; own rows locally)
// (direct write-back: src_tab != nullptr -- each row's mark, its shard row
// if the requester is the key's sole contributor else -1, is stored into the
// requester's mark area at the row's index.  stale_bm: the early push skips
// the rows of the pending update's keys -- the skipping gather left them
// stale in the buffer and the re-push after that update sends them anyway.
// Rows stored off-GPU are counted into *sent.)
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_send_push(int64_t R, int mb, const int64_t* __restrict__ recv,
                                                           const int32_t* __restrict__ owner_inv,
                                                           const int32_t* __restrict__ sendpos,
                                                           const float* __restrict__ buffer,
                                                           const int32_t* __restrict__ rowmap,
                                                           const int32_t* __restrict__ src_tab, int W,
                                                           const int32_t* __restrict__ owner_rows,
                                                           const uint32_t* __restrict__ stale_bm, int self,
                                                           int32_t* __restrict__ sent, const PeerRows out) {
  Grp<D> gp;
  int32_t nsent = 0;
  for (int64_t r = gp.g; r < R; r += gp.ng) {
    if (!((uint64_t(__ldg(recv + r)) >> (56 + mb)) & 1u)) continue;
    const int32_t p = __ldg(sendpos + r);
    const int s = map_seg(out, p);
    float* dst = out.base[s] + (p - out.off[s]) * D;
    // the owner's frozen row: its buffer row, or (zero-copy) its shard row
    const int32_t k = __ldg(owner_inv + r);
    const float* src = buffer + int64_t(rowmap ? __ldg(rowmap + k) : k) * D;
    if (src_tab && gp.l == 0)
      out.dwb_dst[s][p - out.off[s]] = sole_contributor(src_tab, k, W, recv) ? __ldg(owner_rows + k) : -1;
    if (stale_bm && bit_test(stale_bm, uint32_t(__ldg(owner_rows + k)))) continue;
    if (gp.l == 0 && s != self) ++nsent;
#pragma unroll
    for (int v = 0; v < RowGeom<D>::VPL; ++v) st_f4(dst + gp.col(v), ldg_f4(src + gp.col(v)));
  }
  if (sent && nsent) atomicAdd(sent, nsent);
  __threadfence_system();
}

// R5 + re-push (early push): for every owner key u of slot p whose shard row
// the active slot wrote back (bit in bm_a), copy the row into p's buffer
// (mb == 0 only) and store it into the receive row of every requester s that
// asked for u in micro-batch mb: src_tab[u][s] = r, row sendpos[r] of s's
// range.  The row is read once for all its requesters.
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_refresh_push(
    const int32_t* __restrict__ n_p, const int32_t* __restrict__ rows_p, const uint32_t* __restrict__ bm_a,
    const float* __restrict__ shard, float* __restrict__ buf_p, const int32_t* __restrict__ src_tab, int W,
    int mb, const int64_t* __restrict__ recv, const int32_t* __restrict__ sendpos, const PeerRows out,
    int32_t* __restrict__ count) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL;
  const int64_t n = *n_p;
  int32_t local = 0;
  for (int64_t u = gp.g; u < n; u += gp.ng) {
    const uint32_t ld = uint32_t(__ldg(rows_p + u));
    if (!bit_test(bm_a, ld)) continue;
    float4 v[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) v[q] = ldg_f4(shard + int64_t(ld) * D + gp.col(q));
    if (mb == 0) {
      if (buf_p)   // zero-copy: the owner has no buffer to refresh, only the requesters' copies
#pragma unroll
        for (int q = 0; q < VPL; ++q) st_f4(buf_p + u * D + gp.col(q), v[q]);
      if (gp.l == 0) ++local;
    }
    for (int s = 0; s < W; ++s) {
      const int32_t r = __ldg(src_tab + u * W + s);
      if (r < 0 || !((uint64_t(__ldg(recv + r)) >> (56 + mb)) & 1u)) continue;
      float* dst = out.base[s] + int64_t(__ldg(sendpos + r) - out.off[s]) * D;
#pragma unroll
      for (int q = 0; q < VPL; ++q) st_f4(dst + gp.col(q), v[q]);
    }
  }
  if (local) atomicAdd(count, local);
  __threadfence_system();
}

// destination map of micro-batch mb's rows: requester p's range of the
// owner's source-major send positions -> p's receive rows of the slot
static PeerRows send_map(Ctx& c, Slot& s, int mb) {
  const int W = c.W, Nc = c.Nmax + 2;
  PeerRows out{};
  int64_t acc = 0;
  for (int p = 0; p < W; ++p) {
    int64_t dst = src_base_at(s, c, p, mb);
    for (int o = 0; o < c.rank; ++o) dst += s.all[(size_t(p) * W + o) * Nc + 1 + mb];
    out.base[p] = peer_src_of(c, s, p) + dst * c.D;
    out.off[p] = int32_t(acc);
    acc += s.all[(size_t(p) * W + c.rank) * Nc + 1 + mb];
  }
  out.off[W] = int32_t(acc);
  out.n = W;
  out.fence = 1;
  if (c.dwb && !s.zero_copy)
    for (int p = 0; p < W; ++p) {
      int64_t dst = src_base_at(s, c, p, mb);
      for (int o = 0; o < c.rank; ++o) dst += s.all[(size_t(p) * W + o) * Nc + 1 + mb];
      out.dwb_dst[p] = peer_dwb_of(c, s, p) + dst;
    }
  return out;
}

void launch_send_push(Ctx& c, Slot& s, int mb, cudaStream_t st, const uint32_t* stale_bm) {
  NEST_CUDA(cudaMemsetAsync(c.n_refreshed + 1, 0, sizeof(int32_t), st));
  const int64_t R = s.info.recv;
  if (R == 0) return;
  const PeerRows out = send_map(c, s, mb);
  const int32_t* sp = s.sendpos + int64_t(mb) * (c.Rcap + 1);
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    const bool marks = c.dwb && !s.zero_copy;
    k_send_push<D><<<emb_blocks(R, rpb), kRowThreads, 0, st>>>(R, mb, s.recv, s.owner_inv, sp,
                                                                s.zero_copy ? c.shard : s.buffer,
                                                                s.zero_copy ? s.owner_rows : nullptr,
                                                                marks ? s.src_tab : nullptr, c.W, s.owner_rows,
                                                                s.zero_copy ? nullptr : stale_bm, c.rank,
                                                                c.n_refreshed + 1, out);
  });
  NEST_LAUNCH_CHECK();
}

void launch_refresh_push(Ctx& c, Slot& a, Slot& p, int mb, cudaStream_t st) {
  if (mb == 0) NEST_CUDA(cudaMemsetAsync(c.n_refreshed, 0, sizeof(int32_t), st));
  if (p.info.recv == 0) return;
  const PeerRows out = send_map(c, p, mb);
  const int32_t* sp = p.sendpos + int64_t(mb) * (c.Rcap + 1);
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    k_refresh_push<D><<<blocks_for_rows(c.Uocap, rpb, 148 * 16), kRowThreads, 0, st>>>(
        p.n_owner, p.owner_rows, a.obm, c.shard, p.zero_copy ? nullptr : p.buffer, p.src_tab, c.W, mb, p.recv,
        sp, out, c.n_refreshed);
  });
  NEST_LAUNCH_CHECK();
}

// segment-sum form: NEST_SEGSUM = range (k_segsum_range + fix-ups) or chunks
// (cold lane groups + hot chunk partials, the r01 kernels); default: range at
// one rank, chunks at W > 1, where the segment-sum stores every key's row into
// a peer's window and the range form measured slower inside the contended
// step (W=4 DLRM: 49.6-50.7 vs 53.6-54.3 M samples/s; W=1: range 0.55 vs
// 0.59 ms serialised, E step 1.50 ms)
static bool segsum_chunks(const Ctx& c) {
  static const int v = [] {
    const char* e = std::getenv("NEST_SEGSUM");
    const std::string s = e ? e : "";
    return s == "chunks" ? 1 : s == "range" ? 0 : -1;
  }();
  return v < 0 ? c.W > 1 : v == 1;
}
// kernels one launch_segsum* call issues for a non-empty micro-batch (profile
// bookkeeping): range form = k_segsum_range + k_segsum_fix + k_segsum_fix_big;
// chunked form = k_seg_heads + 3-kernel scan + cold + hot chunks + hot final
int segsum_launches(const Ctx& c) { return segsum_chunks(c) ? 7 : 3; }
void launch_segsum_to(Ctx& c, Slot& s, int mb, const float* dout, const PeerRows& out, cudaStream_t st) {
  const int64_t Ui = s.info.mb_uniq[mb];
  const int64_t Ki = s.info.mb_nnz[mb];
  if (Ui == 0) return;
  const uint32_t* skey = s.skey + s.q0[mb];
  const int32_t* sval = s.sval + s.q0[mb];
  const int32_t* pos = s.pos + int64_t(mb) * (c.Kcap + 1);
  const uint32_t umask = (1u << s.ubits) - 1u;
  if (!segsum_chunks(c)) {
    // counters: seg_tot[0] = cut segments listed, seg_tot[1] = big ones
    NEST_CUDA(cudaMemsetAsync(c.seg_tot, 0, 2 * sizeof(int32_t), st));
    const int64_t nr = (Ki + kSegRange - 1) / kSegRange;
    const bool pre = out.sgd_shard && !out.ada;
    NEST_DISPATCH_D(c.D, {
      const int gpb = (kRowThreads / 32) * RowGeom<D>::GPW;
      NEST_DISPATCH_U({
        if (pre)
          k_segsum_range<D, SU, true><<<emb_blocks(nr, gpb), kRowThreads, 0, st>>>(
              Ki, skey, umask, pos, sval, dout, out, c.partial, c.hot_list, c.seg_tot, pf_mask() & 1);
        else
          k_segsum_range<D, SU, false><<<emb_blocks(nr, gpb), kRowThreads, 0, st>>>(
              Ki, skey, umask, pos, sval, dout, out, c.partial, c.hot_list, c.seg_tot, pf_mask() & 1);
      });
      k_segsum_fix<D, 4><<<blocks_for_rows(nr / 4 + 1, gpb, 148 * 8), kRowThreads, 0, st>>>(
          Ki, skey, umask, pos, c.hot_list, c.seg_tot, c.partial, out, c.seg_aux, c.seg_tot + 1);
      k_segsum_fix_big<D><<<148, kRowThreads, 0, st>>>(Ki, c.seg_aux, c.seg_tot + 1, c.partial, out);
    });
    NEST_LAUNCH_CHECK();
    return;
  }
  int32_t* seg = c.seg_start;
  k_seg_heads<<<emb_blocks(Ki, 256), 256, 0, st>>>(Ki, skey, umask, pos, seg, Ui);
  // hot-segment bookkeeping: (is_hot, chunks) prefix -> hot_list, hot_ppos
  int32_t* hot_list = c.hot_list;
  int32_t* hot_ppos = c.seg_aux;
  int32_t* tot = c.seg_tot;
  const int chunk = c.seg_chunk;
  scan_exclusive<I2>(
      [=] __device__(int64_t k) {
        const int32_t L = seg[k + 1] - seg[k];
        return L > chunk ? I2(1, (L + chunk - 1) / chunk) : I2(0, 0);
      },
      Ui,
      [=] __device__(int64_t k, I2 v) {
        if (k == Ui) {
          tot[0] = v.a;
          tot[1] = v.b;
          hot_ppos[v.a] = v.b;
        } else if (seg[k + 1] - seg[k] > chunk) {
          hot_list[v.a] = int32_t(k);
          hot_ppos[v.a] = v.b;
        }
      },
      c.scan_tmp_win, st);
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    NEST_DISPATCH_ILP(k_segsum_cold<D, IL><<<emb_blocks((Ui + IL - 1) / IL, rpb), kRowThreads, 0, st>>>(
                          Ui, chunk, seg, sval, dout, out));
    k_segsum_hot_chunks<D><<<std::min(148 * 4, emb_cap()), kRowThreads, 0, st>>>(chunk, tot, hot_list, hot_ppos, seg, sval, dout,
                                                            c.partial);
    k_segsum_hot_final<D><<<std::min(148 * 2, emb_cap()), kRowThreads, 0, st>>>(tot, hot_list, hot_ppos, c.partial, out);
  });
  NEST_LAUNCH_CHECK();
  (void)skey;
}

// ---------------------------------------------------------------------------
// R12: owner reduce over (micro-batch, source) + SGD (Eq. 2) + write-back
// ---------------------------------------------------------------------------
struct MbBases {
  int64_t v[NEST_MAX_MICRO_BATCHES];
};

// (the loop trip count is warp-uniform: row-wise AdaGrad reduces sum g^2
// across the row's lane group with shuffles).  n_done (optional) counts the
// rows moved: contributions read + the frozen row read + the row written.
template <int D, bool W1>
__global__ void __launch_bounds__(kRowThreads) k_reduce_sgd(
    const int32_t* __restrict__ n_dev, int N, int W, const OptStep opt, MbBases base,
    const uint32_t* __restrict__ mask, const int32_t* __restrict__ pos, int64_t pos_stride,
    const int32_t* __restrict__ src_tab, const int64_t* __restrict__ recv,
    const int32_t* __restrict__ sendpos, int64_t sp_stride, const float* __restrict__ rows,
    const int32_t* __restrict__ owner_rows, float* __restrict__ buffer, float* __restrict__ shard,
    const int32_t* __restrict__ list, int32_t* __restrict__ n_done) {
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  const int64_t n = *n_dev;
  const bool ada = opt.kind == NEST_OPT_ROWWISE_ADAGRAD;
  int32_t done = 0;
  for (int64_t q = gp.g; __any_sync(0xffffffffu, q < n); q += gp.ng) {
    // direct write-back (SGD only): only the listed keys (>= 2 contributions)
    const bool act = q < n;
    const int64_t u = list && act ? int64_t(__ldg(list + q)) : q;
    if (act && gp.l == 0) done += 2;
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!act) {
    } else if (W1) {
      const uint32_t m = __ldg(mask + u);
      for (int i = 0; i < N; ++i) {
        if (!((m >> i) & 1u)) continue;
        const int64_t r = base.v[i] + __ldg(pos + i * pos_stride + u);
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], ldg_f4(rows + r * D + gp.col(v)));
        if (gp.l == 0) ++done;
      }
    } else {
      for (int i = 0; i < N; ++i) {
        for (int s = 0; s < W; ++s) {
          const int32_t r = __ldg(src_tab + u * W + s);
          if (r < 0 || !((uint64_t(__ldg(recv + r)) >> (56 + i)) & 1u)) continue;
          const int64_t row = base.v[i] + __ldg(sendpos + i * sp_stride + r);
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4add(acc[v], ldg_f4(rows + row * D + gp.col(v)));
          if (gp.l == 0) ++done;
        }
      }
    }
    // the updated row goes to the shard only (write-back): the
    // dual-buffer refresh reads written-back rows from the shard, so the
    // frozen active buffer is never rewritten (one row of traffic less)
    const int64_t srow = act ? __ldg(owner_rows + u) : 0;
    float step = opt.lr;   // SGD: e = fma(-lr, G, e)
    if (ada) {
      // g = gscale * G; m += mean(g^2) (lane sums in order, then a fixed xor
      // tree over the group's lanes); step = lr / (sqrt(m) + eps)
      float sq = 0.f;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        acc[v] = make_float4(opt.gscale * acc[v].x, opt.gscale * acc[v].y, opt.gscale * acc[v].z,
                             opt.gscale * acc[v].w);
        sq = __fmaf_rn(acc[v].x, acc[v].x, sq);
        sq = __fmaf_rn(acc[v].y, acc[v].y, sq);
        sq = __fmaf_rn(acc[v].z, acc[v].z, sq);
        sq = __fmaf_rn(acc[v].w, acc[v].w, sq);
      }
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      float m = 0.f;
      if (act && gp.l == 0) {
        m = opt.state[srow] + sq * (1.f / float(D));
        opt.state[srow] = m;
      }
      m = __shfl_sync(0xffffffffu, m, lane_id() - gp.l);
      step = opt.lr / (sqrtf(m) + opt.eps);
    }
    if (!act) continue;
    // the frozen row: the slot buffer, or (zero-copy, buffer == nullptr) the
    // shard row itself, read and written once by this lane group
    const float* frozen = buffer ? buffer + u * D : shard + srow * D;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      float4 e = ld_f4(frozen + gp.col(v));
      e.x = __fmaf_rn(-step, acc[v].x, e.x);
      e.y = __fmaf_rn(-step, acc[v].y, e.y);
      e.z = __fmaf_rn(-step, acc[v].z, e.z);
      e.w = __fmaf_rn(-step, acc[v].w, e.w);
      st_f4_cs(shard + srow * D + gp.col(v), e);
    }
  }
  if (n_done && done) atomicAdd(n_done, done);
}

bool dwb_active(const Ctx& c, const Slot& s, const OptStep& opt) {
  return c.dwb && c.W > 1 && !s.zero_copy && opt.kind == NEST_OPT_SGD;
}

// the owner keys with >= 2 contributions (warp-aggregated append; the order
// is irrelevant: every key's update is independent and fixed-order inside)
__global__ void __launch_bounds__(256) k_upd_list(const int32_t* __restrict__ n_owner,
                                                  const int32_t* __restrict__ src_tab, int W,
                                                  const int64_t* __restrict__ recv, int32_t* __restrict__ list,
                                                  int32_t* __restrict__ cnt) {
  const int64_t n = *n_owner;
  const int lane = lane_id();
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; __any_sync(0xffffffffu, u < n);
       u += int64_t(gridDim.x) * blockDim.x) {
    const bool keep = u < n && !sole_contributor(src_tab, u, W, recv);
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    int32_t base = 0;
    if (lane == 0 && m) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) list[base + __popc(m & ((1u << lane) - 1u))] = int32_t(u);
  }
}

void launch_upd_list(Ctx& c, Slot& s, cudaStream_t st) {
  NEST_CUDA(cudaMemsetAsync(s.n_upd, 0, sizeof(int32_t), st));
  k_upd_list<<<148 * 8, 256, 0, st>>>(s.n_owner, s.src_tab, c.W, s.recv, s.upd_list, s.n_upd);
  NEST_LAUNCH_CHECK();
}

// rows moved by the update are counted on the device (c.n_refreshed[3])
void launch_reduce_sgd(Ctx& c, Slot& s, const OptStep& lr, cudaStream_t st) {
  MbBases b{};
  const bool w1 = c.W == 1;
  for (int i = 0; i < s.N; ++i) b.v[i] = w1 ? s.src_base[i] : s.own_base[i];
  int32_t* cnt = c.n_refreshed + 3;
  NEST_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t), st));
  // direct write-back: only the keys with >= 2 contributions (listed by the route)
  const bool dwb = !w1 && dwb_active(c, s, lr);
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    const int grid = blocks_for_rows(c.Uocap, rpb, 148 * 16);
    if (w1)
      k_reduce_sgd<D, true><<<grid, kRowThreads, 0, st>>>(
          s.n_owner, s.N, 1, lr, b, s.mask, s.pos, c.Kcap + 1, nullptr, nullptr, nullptr, 0,
          src_rows_of(c, s), s.owner_rows, s.zero_copy ? nullptr : s.buffer, c.shard, nullptr, cnt);
    else
      k_reduce_sgd<D, false><<<grid, kRowThreads, 0, st>>>(
          dwb ? s.n_upd : s.n_owner, s.N, c.W, lr, b, nullptr, nullptr, 0, s.src_tab, s.recv, s.sendpos,
          c.Rcap + 1, c.own_rows, s.owner_rows, s.zero_copy ? nullptr : s.buffer, c.shard,
          dwb ? s.upd_list : nullptr, cnt);
  });
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// R5: dual-buffer refresh: for every key of the prefetch slot that the active
// slot also holds (bit test in the active slot's owner bitmap), overwrite the
// prefetched row with the updated row.  The update wrote that row back to the
// shard (same bits as the active copy, reading R-REFRESH), so it is copied
// from shard[ldom] -- no rank lookup, no merge of key lists.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_refresh(
    const int32_t* __restrict__ n_p, const int32_t* __restrict__ rows_p,
    const uint32_t* __restrict__ bm_a, const float* __restrict__ shard, float* __restrict__ buf_p,
    int32_t* __restrict__ count) {
  // each lane group tests L keys at once (one coalesced load of their shard
  // rows + one bit test per lane), then copies the hits -- the ~I/U_o
  // fraction that is in the active slot's key set -- U rows in flight
  Grp<D> gp;
  constexpr int VPL = RowGeom<D>::VPL, L = RowGeom<D>::L;
  constexpr int U = 4;
  const uint32_t gm = group_mask<D>(gp);
  const int64_t n = *n_p;
  int32_t local = 0;
  for (int64_t u0 = gp.g * L; u0 < n; u0 += gp.ng * L) {
    const int64_t u = u0 + gp.l;
    const uint32_t ld = u < n ? uint32_t(__ldg(rows_p + u)) : 0u;
    const bool hit = u < n && bit_test(bm_a, ld);
    uint32_t hits = __ballot_sync(gm, hit) >> (lane_id() - gp.l);
    if (gp.l == 0) local += __popc(hits);
    while (hits) {
      int t[U];
      float4 v[U][VPL];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        t[k] = hits ? __ffs(hits) - 1 : -1;
        if (hits) hits &= hits - 1;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t r = __shfl_sync(gm, ld, t[k] < 0 ? 0 : t[k], L);
        if (t[k] >= 0)
#pragma unroll
          for (int q = 0; q < VPL; ++q) v[k][q] = ldg_f4(shard + int64_t(r) * D + gp.col(q));
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (t[k] >= 0)
#pragma unroll
          for (int q = 0; q < VPL; ++q) st_f4(buf_p + (u0 + t[k]) * D + gp.col(q), v[k][q]);
    }
  }
  if (local) atomicAdd(count, local);
}

void launch_refresh(Ctx& c, Slot& a, Slot& p, cudaStream_t st) {
  NEST_CUDA(cudaMemsetAsync(c.n_refreshed, 0, sizeof(int32_t), st));
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW * RowGeom<D>::L;   // keys per block pass
    k_refresh<D><<<blocks_for_rows(c.Uocap, rpb, 148 * 16), kRowThreads, 0, st>>>(
        p.n_owner, p.owner_rows, a.obm, c.shard, p.buffer, c.n_refreshed);
  });
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// N10: PRF initialisation
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float prf_value(uint64_t h1, int j, int mode, float lo, float scale) {
  const uint64_t h = splitmix64(h1 ^ (uint64_t(j) * 0xD1B54A32D192ED03ull));
  if (mode == NEST_INIT_DYADIC) return float(int(h >> 60) - 8) * 0.00390625f;
  if (mode == NEST_INIT_ZERO) return 0.f;
  const float u = float(uint32_t(h >> 40)) * 5.9604644775390625e-08f;  // 2^-24, exact
  return __fmaf_rn(scale, u, lo);
}

__global__ void k_init_tables(int64_t nvec, int D, int T, int W, int rank,
                              const int64_t* __restrict__ lbase, uint64_t seed, int mode, float lo,
                              float scale, float* __restrict__ shard) {
  const int vpr = D / 4;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nvec;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t ld = e / vpr;
    const int c4 = int(e - ld * vpr);
    int lo_t = 0, hi_t = T;  // largest t with lbase[t] <= ld
    while (hi_t - lo_t > 1) {
      const int mid = (lo_t + hi_t) >> 1;
      if (__ldg(lbase + mid) <= ld) lo_t = mid; else hi_t = mid;
    }
    const int64_t row = (ld - __ldg(lbase + lo_t)) * W + rank;
    const uint64_t key = (uint64_t(lo_t) << kRowBits) | uint64_t(row);
    const uint64_t h1 = splitmix64(seed + 0x9E3779B97F4A7C15ull * (key + 1ull));
    float4 v;
    v.x = prf_value(h1, c4 * 4 + 0, mode, lo, scale);
    v.y = prf_value(h1, c4 * 4 + 1, mode, lo, scale);
    v.z = prf_value(h1, c4 * 4 + 2, mode, lo, scale);
    v.w = prf_value(h1, c4 * 4 + 3, mode, lo, scale);
    st_f4_cs(shard + e * 4, v);
  }
}

// zero n floats of device-accessible memory (device or mapped pinned host:
// the optimizer state of a host-tier table)
__global__ void k_zero_f32(float* __restrict__ p, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0.f;
}
void zero_f32(float* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_zero_f32<<<blocks_for_rows(n, 256, 148 * 8), 256, 0, st>>>(p, n);
  NEST_LAUNCH_CHECK();
}

void launch_init_tables(Ctx& c, cudaStream_t st) {
  const int64_t nvec = c.Vo * c.D / 4;
  const float lo = float(-1.0 / std::sqrt(double(c.D)));
  const float scale = float(2.0 / std::sqrt(double(c.D)));
  if (nvec == 0) return;
  k_init_tables<<<148 * 32, 256, 0, st>>>(nvec, c.D, c.T, c.W, c.rank, c.d_lbase, c.cfg.seed,
                                          c.cfg.init_mode, lo, scale, c.shard);
  NEST_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// parity helper: out[i] = shard row of keys[i]
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kRowThreads) k_read_rows(
    int64_t n, const int64_t* __restrict__ keys, int T, int W, int rank,
    const int64_t* __restrict__ rows, const int64_t* __restrict__ lbase,
    const float* __restrict__ shard, float* __restrict__ out, int32_t* __restrict__ err) {
  Grp<D> gp;
  for (int64_t i = gp.g; i < n; i += gp.ng) {
    const uint64_t key = uint64_t(keys[i]);
    const uint64_t t = key >> kRowBits, row = key & kRowMask;
    const bool ok = t < uint64_t(T) && row < uint64_t(rows[t]) && row % uint64_t(W) == uint64_t(rank);
    if (!ok) {
      if (gp.l == 0) atomicOr(err, kErrShard);
#pragma unroll
      for (int v = 0; v < RowGeom<D>::VPL; ++v) st_f4(out + i * D + gp.col(v), make_float4(0, 0, 0, 0));
      continue;
    }
    const int64_t ld = lbase[t] + int64_t(row / uint64_t(W));
    copy_row<D>(out + i * D, shard + ld * D, gp);
  }
}

// parity helper: out[i] = row-wise AdaGrad accumulator of keys[i]'s shard row
__global__ void k_read_state(int64_t n, const int64_t* __restrict__ keys, int T, int W, int rank,
                             const int64_t* __restrict__ rows, const int64_t* __restrict__ lbase,
                             const float* __restrict__ state, float* __restrict__ out, int32_t* __restrict__ err) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = uint64_t(keys[i]);
    const uint64_t t = key >> kRowBits, row = key & kRowMask;
    const bool ok = t < uint64_t(T) && row < uint64_t(rows[t]) && row % uint64_t(W) == uint64_t(rank);
    if (!ok) atomicOr(err, kErrShard);
    out[i] = ok ? state[lbase[t] + int64_t(row / uint64_t(W))] : 0.f;
  }
}

void launch_read_state(Ctx& c, const int64_t* keys, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return;
  k_read_state<<<blocks_for_rows(n, 256), 256, 0, st>>>(n, keys, c.T, c.W, c.rank, c.d_rows, c.d_lbase,
                                                        c.opt_state, out, c.d_err);
  NEST_LAUNCH_CHECK();
}

void launch_read_rows(Ctx& c, const int64_t* keys, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return;
  NEST_DISPATCH_D(c.D, {
    const int rpb = (kRowThreads / 32) * RowGeom<D>::GPW;
    k_read_rows<D><<<blocks_for_rows(n, rpb, 148 * 16), kRowThreads, 0, st>>>(
        n, keys, c.T, c.W, c.rank, c.d_rows, c.d_lbase, c.shard, out, c.d_err);
  });
  NEST_LAUNCH_CHECK();
}

}  // namespace nest
