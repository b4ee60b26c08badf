// Internal header of libnest.so: context layout, device helpers, and the two
// generic building blocks every stage uses -- a 3-phase exclusive scan and a
// stable LSD radix sort of (uint32 key, int32 value) pairs.
//
// Design notes: every hot-path stage is HBM-bound; no
// stage is a dense contraction, so no tensor cores are used here.
#pragma once

#include <cuda_bf16.h>

#include <map>
#include <tuple>
#include <cuda_runtime.h>
#include <nccl.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nest.h"

namespace nest {

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
struct Error {
  nest_status_t code;
  std::string msg;
};

#define NEST_CUDA(call)                                                           \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      throw ::nest::Error{NEST_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

#define NEST_NCCL(call)                                                           \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess)                                                        \
      throw ::nest::Error{NEST_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

#define NEST_CHECK(cond, code, text)                                              \
  do {                                                                            \
    if (!(cond)) throw ::nest::Error{code, text};                                 \
  } while (0)

#define NEST_LAUNCH_CHECK() NEST_CUDA(cudaGetLastError())

// device error bits (OR-ed into ctx->d_err)
enum : int32_t { kErrKeyRange = 1, kErrShard = 2, kErrSampleSize = 4, kErrCluster = 8 };

constexpr int kRowBits = 40;
constexpr uint64_t kRowMask = (uint64_t(1) << kRowBits) - 1;
constexpr uint64_t kKeyMask56 = (uint64_t(1) << 56) - 1;
constexpr int kMbShift = 28;                      // occ_mbrow = mb << 28 | row
constexpr uint32_t kRowFieldMask = (1u << kMbShift) - 1;

// ----------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------
// scratch of one LSD radix sort: ping-pong pairs, per-block digit
// histograms, scan block sums, one-sweep aux words.  Two users run on
// different streams, so each has its own: the clustering schedule (aux
// stream, Ctx::rx_aux) and the occurrence sorts (the sort stream: per-slot
// ping-pong pairs, shared histogram / scan / aux -- one sort at a time there)
struct RadixScratch {
  uint32_t* tkey[2] = {nullptr, nullptr};
  int32_t* tval[2] = {nullptr, nullptr};
  uint32_t* hist = nullptr;
  void* scan_tmp = nullptr;
  uint32_t* aux = nullptr;
};

struct Slot {
  // source side (this rank as requester)
  int64_t* uniq = nullptr;         // [Kcap]
  int32_t* inverse = nullptr;      // [Kcap]
  uint32_t* mask = nullptr;        // [Kcap]
  int32_t* pos = nullptr;          // [Nmax][Kcap+1]
  uint32_t* skey = nullptr;        // [Kcap] sorted (mb << ubits | u)
  RadixScratch rx;                 // the occurrence sort's scratch (rx.tkey[0] / tval[0]: its input)
  int32_t* sval = nullptr;         // [Kcap] sorted dout row of the occurrence
  int32_t* perm = nullptr;         // [Bcap]
  int32_t* bag_off = nullptr;      // [Bcap*F+1]
  int32_t* samp_base = nullptr;    // [Bcap] output row base of each sample in its mb
  int32_t* mb_of = nullptr;        // [Bcap]
  int32_t* off = nullptr;          // [W+1] per-owner offsets into uniq (device)
  int32_t* xfer = nullptr;         // device: all_counts [W][W][Nmax+2] | mbnnz [Nmax] | err [1]
  int32_t* h_xfer = nullptr;       // pinned mirror
  // owner side
  int64_t* recv = nullptr;         // [Rcap] received key | mask << 56 (W>1)
  uint32_t* obm = nullptr;         // owner bitmap over the local domain [owords+1]
  int32_t* owr = nullptr;          // per-word rank [owords+1]
  int32_t* owner_rows = nullptr;   // [Uocap] shard row of each owner-unique key
  int32_t* owner_inv = nullptr;    // [Rcap]
  int32_t* src_tab = nullptr;      // [Uocap][W] received position per source, -1 if none
  int32_t* sendpos = nullptr;      // [Nmax][Rcap+1]
  int32_t* n_owner = nullptr;      // [1] U_o
  // direct write-back (W > 1): the owner keys with >= 2 contributions, the
  // only ones the owner's update touches (any order: keys are independent)
  int32_t* upd_list = nullptr;     // [Uocap]
  int32_t* n_upd = nullptr;        // [1]
  float* buffer = nullptr;         // [Uocap][d] HBM buffer (active / prefetch)
  // host-known plan
  nest_slot_info_t info{};
  int N = 0, B = 0, cap = 0;
  std::vector<int64_t> all;        // [W][W][N+2]
  std::vector<int64_t> src_base, own_base, q0;   // per mb: row bases / sorted-occurrence starts
  std::vector<int64_t> key_soff, key_roff;       // key All2All offsets
  int ubits = 0;
  uint32_t epoch = 0;              // window sequence number (same on every rank)
  uint32_t xep = 0;                // route exchange sequence number of this slot's batch (route_window)
  uint32_t prefetched = 0;         // micro-batches whose embedding All2All is issued
  bool routed = false, updated = false;
  // early push (fused transport, W > 1): the owner pushed every requested row
  // right after the prefetch gather (`early`); the dual-buffer refresh re-pushed
  // the rows the previous window updated (`repushed`)
  bool early = false, repushed = false;
  // the prefetch gather skipped the rows the other slot's pending update
  // writes (K(t) cap K(t+1)); nest_dbp_refresh supplies them
  bool refresh_pending = false;
  bool skip_planned = false;       // nest_route_begin: the other slot's update was not yet issued
  bool zero_copy = false;          // this batch reads / updates the shard in place (no buffer, no refresh)
  cudaEvent_t ev_early = nullptr, ev_repush = nullptr;
  cudaEvent_t ev_sorted = nullptr;  // occurrences sorted (the segment-sum's input)
  cudaEvent_t ev_gather = nullptr, ev_update = nullptr, ev_free = nullptr, ev_emb[NEST_MAX_MICRO_BATCHES] = {},
              ev_grad[NEST_MAX_MICRO_BATCHES] = {}, ev_ready = nullptr, ev_sync = nullptr;
};

// ----------------------------------------------------------------------------
// tracing: CUDA events around every stage (SURVEY §5 tracing), read back by
// nest_profile_read; stage bytes are the algorithmic bytes of SURVEY §8(d)
// ----------------------------------------------------------------------------
enum Stage : int {
  ST_SCHEDULE = 0, ST_ROUTE, ST_SORT, ST_KEY_A2A, ST_OWNER_DEDUP, ST_GATHER, ST_REFRESH,
  ST_SEND_GATHER, ST_EMB_A2A, ST_POOL, ST_TOWER, ST_SEGSUM, ST_GRAD_A2A, ST_UPDATE, ST_TOWER_DW,
  ST_EMB_REPUSH, ST_COUNT
};
enum StreamKind : int { SK_COMPUTE = 0, SK_COMM = 1, SK_AUX = 2 };

struct ProfRec {
  int stage, kind;
  cudaEvent_t e0, e1;
  double bytes;          // fixed part of the algorithmic bytes
  double hbm = -1;       // local-HBM bytes of a transport stage (< 0: same as bytes)
  int cidx;              // index into the pinned device-count ring (-1: none)
  double bytes_per_cnt;  // bytes per unit of that device count
  int launches;
};

struct Profiler {
  bool on = false;
  cudaEvent_t ref = nullptr;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t next_ev = 0;
  int32_t* hcnt = nullptr;   // pinned ring of device counts copied at record time
  int ncnt = 0, cap_cnt = 1 << 16;
  int64_t launches = 0;      // kernels launched while on
  cudaStream_t ref_stream = nullptr;
};

struct Ctx {
  nest_config_t cfg{};
  Profiler prof;
  std::vector<int64_t> rows;       // [T]
  int W = 1, rank = 0, T = 0, D = 0, F = 1, Nmax = 1;
  int64_t Kcap = 0, Bcap = 0, Rcap = 0, Uocap = 0, MBcap = 0, OMBcap = 0, Pcap = 0;
  int64_t V = 0, Vo = 0;           // global / owner domain sizes (rows)
  int64_t words = 0, owords = 0;   // bitmap words
  std::vector<int64_t> seg_base;   // [W*T+1] host copy
  std::vector<int64_t> lbase;      // [T+1]
  // device constants
  int64_t* d_rows = nullptr;       // [T]
  int64_t* d_seg_base = nullptr;   // [W*T+1]
  int64_t* d_lbase = nullptr;      // [T+1]
  float* shard = nullptr;
  float* opt_state = nullptr;      // [Vo] row-wise AdaGrad accumulators (table_mem after the rows)          // [Vo][d]
  // shared transient workspace
  uint32_t* sbm = nullptr;         // source bitmap [words+1] (W>1; W==1 uses slot obm)
  int32_t* swr = nullptr;          // [words+1]
  uint32_t* occ_dom = nullptr;     // [Kcap]
  int32_t* occ_mbrow = nullptr;    // [Kcap]
  uint32_t* tkey[2] = {nullptr, nullptr};  // radix ping-pong [Kcap]
  int32_t* tval[2] = {nullptr, nullptr};
  uint32_t* hist = nullptr;        // [2^kRadixMaxDigit * radix blocks + 2] (one-sweep: tile status words)
  uint32_t* radix_aux = nullptr;   // [kRadixAux] one-sweep: global digit histograms of every pass + tile counter
  RadixScratch rx_aux;             // the clustering schedule's radix sort (aux stream)
  cudaStream_t sort_stream = nullptr;  // library stream (lowest priority): the occurrence sorts
  bool sort_stream_owned = true;
  cudaEvent_t ev_sort_join = nullptr;
  void* scan_tmp = nullptr;        // scan block sums, route-side streams (bytes)
  void* scan_tmp_win = nullptr;    // scan block sums, window-side streams
  int32_t* samp_scratch = nullptr; // [Bcap+1] unpooled sample prefix (route)
  int64_t* packed = nullptr;       // [Kcap] key | mask << 56 (W>1 send buffer)
  uint32_t* r_ldom = nullptr;      // [Rcap]
  int32_t* seg_start = nullptr;    // [Kcap+1]
  int32_t* seg_aux = nullptr;      // [2*(Kcap+1)] hot offsets
  int32_t* hot_list = nullptr;     // [Kcap]
  int32_t* seg_tot = nullptr;      // [4]
  float* partial = nullptr;        // [Pcap][d]
  float* src_rows = nullptr;       // [MBcap][d]
  float* own_rows = nullptr;       // [OMBcap][d] (== src_rows when W == 1)
  int32_t* d_err = nullptr;        // [1]
  int32_t* d_cnt_scratch = nullptr; // [W*(Nmax)] mb counts scratch
  int32_t* n_refreshed = nullptr;  // [4] rows copied by the last refresh | rows re-pushed off-GPU | rows gathered
  // FWP clustering scratch (cluster.cu)
  uint32_t* cl_bm = nullptr;       // [words+2]
  int32_t* cl_wr = nullptr;        // [words+2]
  int32_t* cl_samp = nullptr;      // [Kcap] sample of each occurrence
  uint32_t* cl_sk = nullptr;       // [Kcap]
  int32_t* cl_sv = nullptr;        // [Kcap]
  int32_t* cl_u = nullptr;         // [Kcap] key id of first occurrences in a sample, else -1
  uint32_t* cl_inmask = nullptr;   // [Kcap] groups whose union holds the key
  int32_t* cl_size = nullptr;      // [Bcap]
  int32_t* cl_grp = nullptr;       // [Bcap]
  int32_t* cl_S = nullptr;         // [Nmax][Bcap]
  int32_t* cl_new = nullptr;       // [Bcap]
  int64_t* cl_small = nullptr;     // [4]
  int32_t* cl_hist = nullptr;      // [Nmax + 1][kClHistBins] rank-key histograms (level 1 per group | level 2)
  int32_t* cl_sel = nullptr;       // [Nmax][8] per-group threshold state
  int32_t* cl_bcnt = nullptr;      // [B / kClIds + 1][Nmax] ties / group members per id block
  int32_t* cl_hmax = nullptr;      // pinned: largest distinct-key count of a sample (host copy)
  int32_t* cl_boff = nullptr;      // [Bcap*F+1] library copy of the batch's bag offsets (graph input)
  int32_t* cl_Scnt = nullptr;      // [Nmax][Bcap] S = |keys(s) & union(g)|, maintained incrementally
  int32_t* cl_kstart = nullptr;    // [Kcap+1] first position of each key id in the key-sorted occurrences
  uint64_t* cl_newk = nullptr;     // [cl_newk_cap] (key id, chunk, group) spread work items
  int64_t cl_newk_cap = 0;         // per round: <= K pairs + N*K/128 chunk extras
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> cl_graphs;  // (B, N, lo) -> captured rounds
  Slot slot[2];
  uint32_t epoch = 0;
  // last use of the shared routing scratch (tkey/tval, hist, scan_tmp, occ_*,
  // clustering): every nest_route / nest_fwp_schedule waits for it and
  // records it, whatever stream the caller uses
  cudaEvent_t ev_scratch = nullptr;
  int seg_chunk = 32;              // segment-sum: cold threshold = hot chunk length (>= 32)
  // checked mode (NEST_GUARD=1): guard band offsets in work_mem, device copy, mismatch counter
  bool guard = false;
  std::vector<size_t> guard_offs;
  uint64_t* d_guard_offs = nullptr;
  unsigned long long* d_guard_bad = nullptr;
  char* work_base = nullptr;
  // copy-engine / fused All2All transports (xfer.cu)
  bool xfer_ce = false;            // peer windows mapped (CE or fused mode)
  int a2a_mode = 0;                // A2AMode
  void* xwin = nullptr;            // library-owned, IPC-exported exchange window
  size_t xwin_bytes = 0, xoff_own = 0, xoff_flags = 0;
  uint32_t* xflags = nullptr;      // [2 slots][XK_COUNT kinds][Nmax][W] epoch flags written by peers
  // route exchange over the window (count exchange + key All2All by peer
  // stores; no NCCL): always without NCCL communicators, NEST_ROUTE_XCHG=window otherwise
  bool route_window = false;
  bool connected = false;          // peers' windows mapped (nest_window_connect / NCCL exchange)
  size_t xoff_cnt = 0, xoff_key = 0, xoff_twr = 0, xcnt_stride = 0, xkey_stride = 0;
  uint32_t xepoch = 0;             // route exchanges so far (same sequence on every rank)
  int route_open = -1;             // slot between nest_route_begin and nest_route_end (-1: none)
  cudaStream_t route_stream = nullptr;
  int route_pid = -1;              // its profile record
  std::vector<int32_t*> peer_cnt[2];   // each peer's count area of slot 0 / 1
  std::vector<int64_t*> peer_key[2];   // each peer's received-key area of slot 0 / 1
  // trained tower without NCCL: dW reduce-scatter / all-gather through the
  // window ([2][twr_elems] f32: partial chunks from every rank | summed dW)
  int64_t twr_elems = 0;
  float* twr = nullptr;
  std::vector<float*> peer_twr;
  uint32_t twr_epoch = 0;
  int early_push = 0;              // EarlyPush: embedding rows pushed at route time (fused transport)
  float* send_stage = nullptr;     // [OMBcap][d] early push send rows (copy-engine early push)
  bool grad_ce = false;            // fused transport, gradients by copy engine (NEST_GRAD_PUSH=ce)
  // the prefetch gather skips the pending update's keys (default); 0: the r01
  // ordering, update(t) waits for gather(t+1) (NEST_GATHER_SKIP=0)
  bool gather_skip = true;
  // NEST_ZERO_COPY=1 (W = 1, N = 1, HBM tables): no retrieval copy -- the pool
  // and the fused update read the shard rows in place
  bool zero_copy = false;
  int64_t src_slot_stride = 0;     // floats between the two slots' receive windows (0: shared)
  // direct write-back of sole-contributor keys (W > 1): marks
  // region of the window (int32 per receive row, per slot), every peer's marks
  // and shard; dwb = on for this world (every rank able, NEST_DIRECT_WB != 0)
  bool dwb_wanted = false, dwb = false;
  size_t xoff_dwb = 0;
  int64_t dwb_slot_stride = 0;     // int32s between the two slots' mark areas (0: shared)
  int32_t* dwb_marks = nullptr;
  std::vector<int32_t*> peer_dwb_slot[2];
  std::vector<float*> peer_shard;
  std::vector<void*> peer_shard_map;   // IPC mappings of peers' shard allocations (closed at destroy)
  std::vector<void*> peer_win;
  std::vector<float*> peer_src, peer_own;
  std::vector<float*> peer_src_slot[2];  // each peer's receive rows of slot 0 / 1
  std::vector<uint32_t*> peer_flags;
  ncclComm_t comm = nullptr, comm_aux = nullptr;
  nest_status_t sticky = NEST_OK;
  std::string last_error;
  // tower (cuBLAS), see tower.cu
  void* tower = nullptr;
};

// receive rows of a slot (this rank / peer p's window)
inline int slot_index(const Ctx& c, const Slot& s) { return int(&s - c.slot); }
inline float* src_rows_of(const Ctx& c, const Slot& s) {
  return c.src_rows + slot_index(c, s) * c.src_slot_stride;
}
inline float* peer_src_of(const Ctx& c, const Slot& s, int p) { return c.peer_src_slot[slot_index(c, s)][p]; }
// direct write-back marks of a slot (this rank / peer p's window)
inline int32_t* dwb_of(const Ctx& c, const Slot& s) { return c.dwb_marks + slot_index(c, s) * c.dwb_slot_stride; }
inline int32_t* peer_dwb_of(const Ctx& c, const Slot& s, int p) { return c.peer_dwb_slot[slot_index(c, s)][p]; }

// GPU clustering (cluster.cu): histogram bins of the radix select, ids per
// block of the ordered passes
constexpr int kClHistLog = 14, kClHistBins = 1 << kClHistLog, kClIds = 1024;

// bump allocator over a caller-owned buffer (base == nullptr: size only)
// Checked mode (NEST_GUARD=1): a guard band of kGuardBytes follows every
// buffer; nest_create fills the bands with kGuardWord and nest_check_guards
// counts the words some kernel overwrote (out-of-bounds writes into the
// workspace; compute-sanitizer is not available on the GPU pool)
constexpr size_t kGuardBytes = 256;
constexpr uint32_t kGuardWord = 0xA5C3A5C3u;
struct Carver {
  char* base;
  size_t off = 0;
  std::vector<size_t>* guards = nullptr;   // guard band offsets (checked mode)
  template <class T>
  T* take(int64_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += size_t(std::max<int64_t>(n, 1)) * sizeof(T);
    if (guards) {
      off = (off + 255) & ~size_t(255);
      guards->push_back(off);
      off += kGuardBytes;
    }
    return p;
  }
};

// ----------------------------------------------------------------------------
// small device helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// rank of bit x in a bitmap with per-word exclusive popcount prefix `wr`
__device__ __forceinline__ int32_t bit_rank(const uint32_t* __restrict__ bm,
                                            const int32_t* __restrict__ wr, uint32_t x) {
  const uint32_t w = x >> 5, b = x & 31u;
  return wr[w] + __popc(bm[w] & ((1u << b) - 1u));
}
__device__ __forceinline__ bool bit_test(const uint32_t* __restrict__ bm, uint32_t x) {
  return (bm[x >> 5] >> (x & 31u)) & 1u;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 ldg_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// read-only loads with an L2 eviction priority: evict_last for rows read again
// soon (a bag's dout row, once per occurrence), evict_first for rows read once
__device__ __forceinline__ float4 ldg_f4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// bulk L2 prefetch of `bytes` (multiple of 16, 16-byte aligned) by the TMA
// unit: no registers, no shared memory; the later register loads hit L2
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ float4 ld_f4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st_f4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
// streaming store (evict-first) for write-once outputs
__device__ __forceinline__ void st_f4_cs(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// streaming store of 4 consecutive outputs, fp32 or rounded to bf16 (RN)
__device__ __forceinline__ void st_out4_cs(float* p, float4 v) { st_f4_cs(p, v); }
__device__ __forceinline__ void st_out4_cs(__nv_bfloat16* p, float4 v) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  const uint32_t lo = *reinterpret_cast<const uint32_t*>(&a), hi = *reinterpret_cast<const uint32_t*>(&b);
  asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(lo), "r"(hi) : "memory");
}

// Row geometry for fp32 rows of D floats processed by groups of L lanes, each
// lane owning VPL consecutive float4 chunks strided by L*4 floats.
template <int D>
struct RowGeom {
  static_assert(D % 4 == 0, "dim must be a multiple of 4");
  static constexpr int kVec = D / 4;                       // float4 per row
  static constexpr int L = kVec < 32 ? kVec : 32;          // lanes per row
  static constexpr int VPL = kVec / L;                     // float4 per lane
  static constexpr int GPW = 32 / L;                       // groups (rows) per warp
  static_assert(kVec % L == 0, "row must split evenly over lanes");
};

// ----------------------------------------------------------------------------
// generic exclusive scan (3 phases) over n values produced by a functor
// ----------------------------------------------------------------------------
struct I2 {
  int32_t a, b;
  I2() = default;
  __host__ __device__ I2(int32_t x, int32_t y) : a(x), b(y) {}
  __host__ __device__ I2 operator+(const I2& o) const { return I2(a + o.a, b + o.b); }
};
__device__ __forceinline__ int32_t shfl_up_t(int32_t v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ uint32_t shfl_up_t(uint32_t v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ long long shfl_up_t(long long v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ I2 shfl_up_t(I2 v, int d) {
  return I2(__shfl_up_sync(0xffffffffu, v.a, d), __shfl_up_sync(0xffffffffu, v.b, d));
}
__device__ __forceinline__ int32_t shfl_down_t(int32_t v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ uint32_t shfl_down_t(uint32_t v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ long long shfl_down_t(long long v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ I2 shfl_down_t(I2 v, int d) {
  return I2(__shfl_down_sync(0xffffffffu, v.a, d), __shfl_down_sync(0xffffffffu, v.b, d));
}

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + shfl_down_t(v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = shfl_up_t(v, o);
    if (lane >= o) v = v + n;
  }
  return v;
}

template <typename T, typename In>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(In in, int64_t n, T* block_sums) {
  __shared__ T ws[kScanThreads / 32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  T acc = T();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    if (i < n) acc = acc + in(i);
  }
  acc = warp_reduce_sum(acc);
  if (lane_id() == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T v = threadIdx.x < kScanThreads / 32 ? ws[threadIdx.x] : T();
    v = warp_reduce_sum(v);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
  }
}

// single block: in-place exclusive scan of sums[0..nb), total into sums[nb]
template <typename T>
__global__ void __launch_bounds__(1024) k_scan_block_sums(T* sums, int nb) {
  __shared__ T ws[32];
  __shared__ T carry_s, total_s;
  if (threadIdx.x == 0) carry_s = T();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    T v = i < nb ? sums[i] : T();
    T inc = warp_incl_scan(v);
    T exc = shfl_up_t(inc, 1);
    if (lane == 0) exc = T();
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      T w = ws[lane];
      T wi = warp_incl_scan(w);
      T we = shfl_up_t(wi, 1);
      if (lane == 0) we = T();
      ws[lane] = we;
      if (lane == 31) total_s = wi;
    }
    __syncthreads();
    const T carry = carry_s;
    if (i < nb) sums[i] = carry + ws[warp] + exc;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + total_s;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry_s;
}

template <typename T, typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(In in, int64_t n, const T* offsets,
                                                            int nb, Out out) {
  __shared__ T tile[kScanTile];
  __shared__ T ws[kScanThreads / 32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    tile[k * kScanThreads + threadIdx.x] = i < n ? in(i) : T();
  }
  __syncthreads();
  T loc[kScanItems];
  T s = T();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    loc[k] = s;
    s = s + tile[threadIdx.x * kScanItems + k];
  }
  T inc = warp_incl_scan(s);
  T exc = shfl_up_t(inc, 1);
  if (lane_id() == 0) exc = T();
  if (lane_id() == 31) ws[threadIdx.x >> 5] = inc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T v = threadIdx.x < kScanThreads / 32 ? ws[threadIdx.x] : T();
    T vi = warp_incl_scan(v);
    T ve = shfl_up_t(vi, 1);
    if (threadIdx.x == 0) ve = T();
    if (threadIdx.x < kScanThreads / 32) ws[threadIdx.x] = ve;
  }
  __syncthreads();
  const T off = offsets[blockIdx.x] + ws[threadIdx.x >> 5] + exc;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) tile[threadIdx.x * kScanItems + k] = off + loc[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    if (i < n) out(i, tile[k * kScanThreads + threadIdx.x]);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out(n, offsets[nb]);
}

inline int scan_blocks(int64_t n) { return int(n <= 0 ? 1 : (n + kScanTile - 1) / kScanTile); }

// exclusive scan: out(i, prefix_i) for i in [0, n), out(n, total).
// temp must hold scan_blocks(n) + 1 values of T.
template <typename T, typename In, typename Out>
void scan_exclusive(In in, int64_t n, Out out, void* temp, cudaStream_t st) {
  const int nb = scan_blocks(n);
  T* sums = reinterpret_cast<T*>(temp);
  k_scan_reduce<T, In><<<nb, kScanThreads, 0, st>>>(in, n, sums);
  k_scan_block_sums<T><<<1, 1024, 0, st>>>(sums, nb);
  k_scan_down<T, In, Out><<<nb, kScanThreads, 0, st>>>(in, n, sums, nb, out);
  NEST_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// stable LSD radix sort of (uint32 key, int32 value), 8-bit digits
// ----------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
#ifndef NEST_RADIX_ITEMS
#define NEST_RADIX_ITEMS 8
#endif
constexpr int kRadixItems = NEST_RADIX_ITEMS;   // items per thread (tuning builds: -DNEST_RADIX_ITEMS=...)
constexpr int kRadixTile = kRadixThreads * kRadixItems;   // 2048 (8 items: E step 1.27 vs 1.29 ms at 16, 1.40 at 32)
constexpr int kRadixWarps = kRadixThreads / 32;
// widest digit: 8 bits.  11-bit digits (2 passes for 22-bit keys) measured
// slower on B200: scatter 81 vs 38 us, histogram 34 vs 23 us per pass at
// 3.4M pairs (2 blocks/SM and strided per-block offset reads at 2048 bins)
constexpr int kRadixMaxDigit = 8;

inline int radix_blocks(int64_t n) { return int(n <= 0 ? 1 : (n + kRadixTile - 1) / kRadixTile); }
// one-sweep aux words: 4 passes x 256 global digit counts + tile counter
constexpr int kRadixAux = 4 * 256 + 32;

void radix_sort_pairs_shifts(const RadixScratch& rx, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                             int32_t* vout, int64_t n, const std::vector<int>& shifts, cudaStream_t st);
void radix_sort_pairs(const RadixScratch& rx, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                      int32_t* vout, int64_t n, int bits, cudaStream_t st);
int radix_digit_bits(int bits);

// ----------------------------------------------------------------------------
// stage launchers (route.cu / rows.cu / schedule.cu / tower.cu)
// ----------------------------------------------------------------------------
void route_phase_a(Ctx& c, Slot& s, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz,
                   int B, const int32_t* perm, int N, cudaStream_t st);
void route_plan(Ctx& c, Slot& s);
void route_phase_b(Ctx& c, Slot& s, cudaStream_t st);
void route_sort(Ctx& c, Slot& s, cudaStream_t st);
void route_positions(Ctx& c, Slot& s, cudaStream_t st);
void exchange_plan(const Ctx& c, int N, const int32_t* all, nest_exchange_plan_t& p);
void zero_f32(float* p, int64_t n, cudaStream_t st);
void launch_init_tables(Ctx& c, cudaStream_t st);
void launch_gather(Ctx& c, Slot& s, const uint32_t* skip_bm, cudaStream_t st);
void launch_send_gather(Ctx& c, Slot& s, int mb, cudaStream_t st, float* out_rows = nullptr);
// out: fp32 rows, or bf16 rows (pooled sum only) when bf16
void launch_pool(Ctx& c, Slot& s, int mb, void* out, bool bf16, cudaStream_t st);
void launch_segsum(Ctx& c, Slot& s, int mb, const float* dout, cudaStream_t st);
int segsum_launches(const Ctx& c);
void launch_refresh(Ctx& c, Slot& a, Slot& p, cudaStream_t st);
void launch_read_rows(Ctx& c, const int64_t* keys, int64_t n, float* out, cudaStream_t st);
void launch_schedule(Ctx& c, const int64_t* keys, const int32_t* bag_offsets, int64_t nnz, int B, int N, int mode,
                     int32_t* perm, int32_t* mb_offsets, cudaStream_t st);
// tracing hooks (api.cu); cheap no-ops unless profiling is on
int prof_begin(Ctx& c, int stage, int kind, cudaStream_t st);
void prof_end(Ctx& c, int id, cudaStream_t st, double bytes, const int32_t* dcount = nullptr,
              double bytes_per_cnt = 0.0, int launches = 1) noexcept;
void prof_add_bytes(Ctx& c, int id, double bytes) noexcept;
void prof_set_hbm(Ctx& c, int id, double hbm) noexcept;
void profile_enable(Ctx& c, bool on);
void profile_read(Ctx& c, nest_profile_stage_t* stages, nest_profile_summary_t* sum);
void profile_destroy(Ctx& c);
void guards_fill(Ctx& c, cudaStream_t st);
int64_t guards_check(Ctx& c, cudaStream_t st);
void profile_records(Ctx& c, nest_profile_record_t* out, int64_t cap, int64_t* n);
struct ProfScope {
  Ctx& c;
  int id;
  cudaStream_t st;
  double bytes = 0, bpc = 0;
  double hbm = -1;   // transport stages: local-HBM bytes (bytes = off-GPU bytes)
  const int32_t* dcount = nullptr;
  int launches = 1;
  ProfScope(Ctx& cc, int stage, int kind, cudaStream_t s) : c(cc), id(prof_begin(cc, stage, kind, s)), st(s) {}
  ~ProfScope() {
    prof_end(c, id, st, bytes, dcount, bpc, launches);
    prof_set_hbm(c, id, hbm);
  }
};
// output maps of the fused gather->NVLink-put kernels (rows.cu): position p of
// a micro-batch's (owner- or source-major) row list goes to row
// base[s] + (p - off[s]) with off[s] <= p < off[s+1]
struct PeerRows {
  float* base[NEST_MAX_WORLD];
  int32_t off[NEST_MAX_WORLD + 1];
  int32_t n;          // number of segments (W, or 1 for a purely local map)
  int32_t fence;      // 1: writes go to peer memory (system fence at the end)
  // fused SGD (W == 1, N == 1: every key has exactly one contribution): row k
  // is applied as shard[owner_rows[k]] = fma(-lr, g, buffer[k]) instead of stored
  const float* sgd_buffer;
  const int32_t* sgd_rows;
  float* sgd_shard;
  float sgd_lr;
  // ... or row-wise AdaGrad (ada != 0): g = gscale*G, m += mean(g^2) in
  // state[shard row], shard row = fma(-lr/(sqrt(m)+eps), g, buffer[k])
  int32_t ada;
  float ada_gscale, ada_eps;
  float* ada_state;
  // zero-copy retrieval (W = 1, HBM tables): the frozen row of key k is read
  // from the shard itself (row sgd_rows[k], updated in place) instead of the
  // slot buffer
  int32_t sgd_inplace;
  // direct write-back (W > 1, SGD): dwb_rows[k] >= 0 marks a key whose only
  // contribution is this row -- it is applied to the received frozen copy
  // (sgd_buffer + k*D, lr sgd_lr) and stored at row dwb_rows[k] of the owner's
  // shard (dwb_shard[segment of k]) instead of sent as a gradient row.
  // Owner side (k_send_push): dwb_dst[p] = requester p's mark area, indexed
  // like base[p]
  const int32_t* dwb_rows;
  float* dwb_shard[NEST_MAX_WORLD];
  int32_t* dwb_dst[NEST_MAX_WORLD];
};
enum A2AMode : int { A2A_NCCL = 0, A2A_CE = 1, A2A_FUSED = 2 };
// the update's sparse optimizer step: Eq. 2 SGD (e = fma(-lr, G, e), lr =
// eta/|B|) or row-wise AdaGrad (g = gscale*G; m += mean(g^2);
// e = fma(-lr/(sqrt(m)+eps), g, e); m in state[shard row])
struct OptStep {
  int kind;       // NEST_OPT_SGD / NEST_OPT_ROWWISE_ADAGRAD
  float lr;
  float gscale;
  float eps;
  float* state;
};
void launch_reduce_sgd(Ctx& c, Slot& s, const OptStep& opt, cudaStream_t st);
bool dwb_active(const Ctx& c, const Slot& s, const OptStep& opt);
void launch_upd_list(Ctx& c, Slot& s, cudaStream_t st);
void launch_segsum_sgd(Ctx& c, Slot& s, const float* dout, const OptStep& opt, cudaStream_t st);
void launch_read_state(Ctx& c, const int64_t* keys, int64_t n, float* out, cudaStream_t st);
enum EarlyPush : int { EP_OFF = 0, EP_CE = 1, EP_SM = 2 };
int a2a_mode_wanted(int W);
int64_t src_base_at(const Slot& s, const Ctx& c, int p, int mb);
int64_t own_base_at(const Slot& s, const Ctx& c, int p, int mb);
void launch_send_push(Ctx& c, Slot& s, int mb, cudaStream_t st, const uint32_t* stale_bm = nullptr);
// dual-buffer refresh a -> p fused with the re-push of the refreshed rows to
// every requester of micro-batch mb of slot p (early push)
void launch_refresh_push(Ctx& c, Slot& a, Slot& p, int mb, cudaStream_t st);
void launch_segsum_to(Ctx& c, Slot& s, int mb, const float* dout, const PeerRows& out, cudaStream_t st);
void xfer_signal(Ctx& c, Slot& s, int kind, int mb, cudaStream_t st);
// copy-engine transport (xfer.cu)
bool xfer_wanted(int W);
void xfer_setup(Ctx& c, cudaStream_t st);
void xfer_destroy(Ctx& c);
void xfer_push_emb(Ctx& c, Slot& s, int mb, cudaStream_t st, cudaEvent_t after_self,
                   const float* send_rows = nullptr);
// flag kinds: 0 embedding rows, 1 gradient rows, 2 re-pushed embedding rows
// 3 route counts, 4 route keys (mb 0; route_window), 5 / 6 trained-tower
// reduce-scatter / all-gather (slot 0, mb 0; window AllReduce)
enum XferKind : int { XK_EMB = 0, XK_GRAD = 1, XK_REPUSH = 2, XK_CNT = 3, XK_KEY = 4, XK_TRS = 5, XK_TAG = 6,
                      XK_COUNT = 7 };
constexpr uint64_t kWinMagic = 0x314e495754534e45ull;   // "ENSTWIN1"
void xfer_alloc(Ctx& c, cudaStream_t st);
void xfer_export(const Ctx& c, nest_window_rec_t* r);
void xfer_connect(Ctx& c, const nest_window_rec_t* all);
void xfer_signal_raw(Ctx& c, int slot, int kind, int mb, uint32_t value, cudaStream_t st);
void xfer_wait_raw(Ctx& c, int slot, int kind, int mb, uint32_t value, cudaStream_t st);
void xfer_wait_emb(Ctx& c, Slot& s, int mb, cudaStream_t st, int kind = XK_EMB);
void xfer_push_grad(Ctx& c, Slot& s, int mb, cudaStream_t st);
void xfer_wait_grads(Ctx& c, Slot& s, cudaStream_t st);
void tower_create(Ctx& c);
void tower_destroy(Ctx& c);
// pooled: fp32 rows (cast to bf16 inside) or, with pooled_bf16, bf16 rows read
// in place (they must stay unmodified until the deferred dW GEMMs finish)
double tower_run(Ctx& c, const void* pooled, bool pooled_bf16, int64_t rows, float* dout, cudaStream_t st);
void tower_join(Ctx& c, cudaStream_t st);
void tower_step(Ctx& c, cudaStream_t st);
void tower_set_side(Ctx& c, cudaStream_t st);
void tower_read(Ctx& c, int what, int layer, float* out, cudaStream_t st);

}  // namespace nest
