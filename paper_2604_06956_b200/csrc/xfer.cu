// Copy-engine All2All over NVLink 5 / NVSwitch for the FWP window (R7, R11).
//
// The owner's send rows of a micro-batch are already laid out contiguously per
// requester (R6), and every rank knows every rank's counts after the count
// exchange, so each All2All is W-1 DMA copies straight into the peers'
// receive rows (CUDA IPC mappings of the peers' exchange windows) plus one
// flag per peer written with a stream memory operation after the copies.  The
// receiver's stream waits on its local flags (cuStreamWaitValue32, no kernel,
// no SM).  Copies run on the copy engines, so the overlapped dense compute
// keeps every SM ("eliminates hardware contention between computation
// and communication").
//
// Flags hold the window's epoch (same sequence on every rank), so they never
// need resetting.  Buffer reuse is safe by causality: an owner pushes batch
// t+1's rows only after its update(t), which waited for every requester's
// gradient push of batch t, i.e. after every requester stopped using its rows.
//
// Early push (fused transport; NEST_EARLY_PUSH = sm (default) | ce | 0): the
// owner pushes batch t+1's rows at the end of its route (right after the
// prefetch gather, during window t) into a second receive window, one per
// slot -- by copy engine from a send-staging buffer (ce) or by SM remote
// stores (sm) -- and after update(t) the dual-buffer refresh re-pushes only
// the rows update(t) wrote back (P:363-380's intersection, applied to the
// requesters' copies) from the same kernel that refreshes the owner's buffer.  The same causality argument holds per slot: route(t+1) on the
// owner follows update(t-1) of that slot, after every requester stopped
// reading the slot's window.
#include <cuda.h>

#include <unistd.h>

#include <cstring>

#include "nest_internal.cuh"

namespace nest {

using PFN_wait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_wait g_wait = nullptr;
static PFN_write g_write = nullptr;
static PFN_range g_range = nullptr;

static void load_driver_ops() {
  if (g_wait && g_write) return;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  NEST_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q));
  NEST_CHECK(q == cudaDriverEntryPointSuccess && fn, NEST_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  g_wait = reinterpret_cast<PFN_wait>(fn);
  NEST_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q));
  NEST_CHECK(q == cudaDriverEntryPointSuccess && fn, NEST_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  g_write = reinterpret_cast<PFN_write>(fn);
  // (optional: without it the shard is not exported and direct write-back stays off)
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_range = reinterpret_cast<PFN_range>(fn);
  (void)cudaGetLastError();
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// NEST_A2A = fused (default: gather / segment-sum kernels store straight into
// peer memory), ce (copy engines), nccl (grouped ncclSend/ncclRecv, the baseline)
int a2a_mode_wanted(int W) {
  if (W <= 1) return A2A_NCCL;
  const char* e = std::getenv("NEST_A2A");
  if (e && std::strcmp(e, "nccl") == 0) return A2A_NCCL;
  if (e && std::strcmp(e, "ce") == 0) return A2A_CE;
  return A2A_FUSED;
}
bool xfer_wanted(int W) { return a2a_mode_wanted(W) != A2A_NCCL; }

static int early_push_wanted() {
  const char* e = std::getenv("NEST_EARLY_PUSH");
  if (e && std::strcmp(e, "0") == 0) return EP_OFF;
  if (e && std::strcmp(e, "ce") == 0) return EP_CE;
  return EP_SM;   // measured best at W = 2: sm 4.57, off 4.61, ce 4.92 ms/step
}

// window layout: [src_rows of slot 0 (| slot 1 with early push) MBcap*D f32 |
//                 own_rows OMBcap*D f32 |
//                 route counts [2 slots][W*W*Nc + Nmax + 1] i32 (route_window) |
//                 received keys [2 slots][Rcap] i64 (route_window) |
//                 tower dW exchange [2][n] f32 (trained tower without NCCL) |
//                 direct write-back marks [slot 0 (| slot 1)][MBcap] i32 |
//                 flags [2][XK_COUNT][Nmax][W] u32]
//
// Direct write-back (NEST_DIRECT_WB, default on; fused transport with SM
// pushes, SGD, HBM tables): most keys of a batch have one contributor
// (DLRM at W = 2: 87% of the owner-unique keys come from one source and one
// micro-batch).  For those the owner's reduce would read one gradient row and
// the frozen row and write the shard row; instead the owner's push marks the
// row (its shard index), the requester applies Eq. 2 to its received frozen
// copy -- the same fma on the same operands, so the same bits -- and stores
// the updated row into the owner's shard over NVLink (or locally), and the
// owner's reduce skips the key.  Ordering is unchanged: the owner's update
// (and the refresh / re-push after it) waits for every requester's gradient
// flag, which each requester raises after its segment-sum's stores.
void xfer_alloc(Ctx& c, cudaStream_t st) {
  load_driver_ops();
  c.a2a_mode = a2a_mode_wanted(c.W);
  NEST_CHECK(c.a2a_mode != A2A_NCCL, NEST_ERR_INVALID, "xfer_alloc needs the fused or ce transport");
  c.early_push = c.a2a_mode == A2A_FUSED ? early_push_wanted() : EP_OFF;
  {
    // gradients under the fused transport: segment-sum stores into the
    // owners' windows (sm, default) or local rows + copy-engine DMA (ce)
    const char* g = std::getenv("NEST_GRAD_PUSH");
    c.grad_ce = c.a2a_mode == A2A_FUSED && g && std::strcmp(g, "ce") == 0;
  }
  if (c.early_push == EP_CE)
    NEST_CUDA(cudaMalloc(&c.send_stage, std::max<size_t>(size_t(c.OMBcap) * c.D * sizeof(float), 256)));
  const int Nc = c.Nmax + 2;
  const size_t src1 = align_up(size_t(c.MBcap) * c.D * sizeof(float), 4096);
  const size_t src_b = c.early_push ? 2 * src1 : src1;
  const size_t own_b = align_up(size_t(c.OMBcap) * c.D * sizeof(float), 4096);
  const size_t cnt1 = align_up(sizeof(int32_t) * (size_t(c.W) * c.W * Nc + c.Nmax + 1), 256);
  const size_t key1 = align_up(sizeof(int64_t) * size_t(c.Rcap), 256);
  const size_t cnt_b = c.route_window ? 2 * cnt1 : 0;
  const size_t key_b = c.route_window ? align_up(2 * key1, 4096) : 0;
  const size_t twr_b = align_up(sizeof(float) * 2 * size_t(c.twr_elems), 4096);
  const size_t flg_b = align_up(size_t(2) * XK_COUNT * c.Nmax * c.W * sizeof(uint32_t), 4096);
  {
    const char* e = std::getenv("NEST_DIRECT_WB");
    c.dwb_wanted = !(e && std::strcmp(e, "0") == 0) && c.a2a_mode == A2A_FUSED && !c.grad_ce &&
                   c.early_push != EP_CE && c.cfg.table_location == NEST_TABLE_HBM &&
                   c.cfg.optimizer == NEST_OPT_SGD;
  }
  const size_t dwb1 = align_up(sizeof(int32_t) * size_t(c.MBcap), 4096);
  const size_t dwb_b = c.dwb_wanted ? (c.early_push ? 2 * dwb1 : dwb1) : 0;
  c.dwb_slot_stride = c.early_push ? int64_t(dwb1 / sizeof(int32_t)) : 0;
  c.src_slot_stride = c.early_push ? int64_t(src1 / sizeof(float)) : 0;
  c.xoff_own = src_b;
  c.xoff_cnt = src_b + own_b;
  c.xoff_key = c.xoff_cnt + cnt_b;
  c.xoff_twr = c.xoff_key + key_b;
  c.xoff_dwb = c.xoff_twr + twr_b;
  c.xoff_flags = c.xoff_dwb + dwb_b;
  c.xcnt_stride = cnt1;
  c.xkey_stride = key1;
  c.xwin_bytes = c.xoff_flags + flg_b;
  NEST_CUDA(cudaMalloc(&c.xwin, c.xwin_bytes));
  char* base = reinterpret_cast<char*>(c.xwin);
  NEST_CUDA(cudaMemsetAsync(base + c.xoff_flags, 0, flg_b, st));
  c.src_rows = reinterpret_cast<float*>(base);
  c.own_rows = reinterpret_cast<float*>(base + src_b);
  c.xflags = reinterpret_cast<uint32_t*>(base + c.xoff_flags);
  if (c.route_window) {
    // the count exchange and the key All2All land in the window: peers store
    // their counts / keys straight into this rank's slot areas
    for (int si = 0; si < 2; ++si) {
      c.slot[si].xfer = reinterpret_cast<int32_t*>(base + c.xoff_cnt + si * cnt1);
      c.slot[si].recv = reinterpret_cast<int64_t*>(base + c.xoff_key + si * key1);
    }
  }
  c.twr = c.twr_elems ? reinterpret_cast<float*>(base + c.xoff_twr) : nullptr;
  c.dwb_marks = c.dwb_wanted ? reinterpret_cast<int32_t*>(base + c.xoff_dwb) : nullptr;
}

void xfer_export(const Ctx& c, nest_window_rec_t* r) {
  NEST_CHECK(c.xwin != nullptr, NEST_ERR_INVALID, "no exchange window (world == 1 or NEST_A2A=nccl)");
  std::memset(r, 0, sizeof(*r));
  r->magic = kWinMagic;
  r->pid = int32_t(getpid());
  r->rank = c.rank;
  r->world = c.W;
  int dev = 0;
  NEST_CUDA(cudaGetDevice(&dev));
  r->device = dev;
  r->ptr = reinterpret_cast<uint64_t>(c.xwin);
  cudaIpcMemHandle_t h;
  NEST_CUDA(cudaIpcGetMemHandle(&h, c.xwin));
  static_assert(sizeof(h) <= sizeof(r->ipc), "ipc handle size");
  std::memcpy(r->ipc, &h, sizeof(h));
  r->bytes = c.xwin_bytes;
  r->off_own = c.xoff_own;
  r->off_cnt = c.xoff_cnt;
  r->off_key = c.xoff_key;
  r->off_twr = c.xoff_twr;
  r->off_flags = c.xoff_flags;
  r->src_stride = uint64_t(c.src_slot_stride);
  r->cnt_stride = c.xcnt_stride;
  r->key_stride = c.xkey_stride;
  r->off_dwb = c.xoff_dwb;
  r->dwb_stride = uint64_t(c.dwb_slot_stride);
  r->shard_ptr = reinterpret_cast<uint64_t>(c.shard);
  if (c.dwb_wanted && g_range) {
    // the shard is caller memory (e.g. a block of PyTorch's allocator): export
    // the allocation that holds it, plus the offset
    CUdeviceptr b = 0;
    size_t sz = 0;
    cudaIpcMemHandle_t sh;
    if (g_range(&b, &sz, reinterpret_cast<CUdeviceptr>(c.shard)) == CUDA_SUCCESS &&
        cudaIpcGetMemHandle(&sh, reinterpret_cast<void*>(b)) == cudaSuccess) {
      std::memcpy(r->shard_ipc, &sh, sizeof(sh));
      r->shard_off = reinterpret_cast<uint64_t>(c.shard) - uint64_t(b);
      r->dwb_ok = 1;
    }
    (void)cudaGetLastError();
  }
}

// map every peer's window: the same process (in-process ranks sharing one
// device) uses the raw pointer, another process opens the CUDA IPC handle
void xfer_connect(Ctx& c, const nest_window_rec_t* all) {
  NEST_CHECK(c.xwin != nullptr, NEST_ERR_INVALID, "no exchange window (world == 1 or NEST_A2A=nccl)");
  NEST_CHECK(!c.connected, NEST_ERR_ORDER, "window already connected");
  for (int p = 0; p < c.W; ++p) {
    const nest_window_rec_t& r = all[p];
    NEST_CHECK(r.magic == kWinMagic && r.world == c.W && r.rank == p, NEST_ERR_INVALID,
               "window records must be this world's, in rank order");
    NEST_CHECK(r.bytes == c.xwin_bytes && r.off_flags == c.xoff_flags && r.off_key == c.xoff_key,
               NEST_ERR_INVALID, "peer window geometry differs (every rank needs the same config)");
  }
  NEST_CHECK(all[c.rank].ptr == reinterpret_cast<uint64_t>(c.xwin), NEST_ERR_INVALID,
             "own window record does not match this context");
  c.peer_win.assign(c.W, nullptr);
  c.peer_src.assign(c.W, nullptr);
  c.peer_own.assign(c.W, nullptr);
  c.peer_flags.assign(c.W, nullptr);
  c.peer_twr.assign(c.W, nullptr);
  for (int si = 0; si < 2; ++si) {
    c.peer_src_slot[si].assign(c.W, nullptr);
    c.peer_cnt[si].assign(c.W, nullptr);
    c.peer_key[si].assign(c.W, nullptr);
  }
  const int32_t me_pid = int32_t(getpid());
  for (int p = 0; p < c.W; ++p) {
    const nest_window_rec_t& r = all[p];
    char* base;
    if (p == c.rank) {
      base = reinterpret_cast<char*>(c.xwin);
    } else if (r.pid == me_pid) {
      base = reinterpret_cast<char*>(r.ptr);   // same process: one address space
    } else {
      void* ptr = nullptr;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, r.ipc, sizeof(h));
      NEST_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      base = reinterpret_cast<char*>(ptr);
      c.peer_win[p] = ptr;
    }
    c.peer_src[p] = reinterpret_cast<float*>(base);
    c.peer_src_slot[0][p] = c.peer_src[p];
    c.peer_src_slot[1][p] = c.peer_src[p] + r.src_stride;
    c.peer_own[p] = reinterpret_cast<float*>(base + r.off_own);
    c.peer_flags[p] = reinterpret_cast<uint32_t*>(base + r.off_flags);
    c.peer_twr[p] = reinterpret_cast<float*>(base + r.off_twr);
    for (int si = 0; si < 2; ++si) {
      c.peer_cnt[si][p] = reinterpret_cast<int32_t*>(base + r.off_cnt + si * r.cnt_stride);
      c.peer_key[si][p] = reinterpret_cast<int64_t*>(base + r.off_key + si * r.key_stride);
    }
  }
  // (no barrier needed: the first push happens after the first route's count
  // exchange, which every rank enters after connecting)
  c.xfer_ce = true;
  // direct write-back runs iff every rank can take part
  bool dwb = c.dwb_wanted;
  for (int p = 0; p < c.W; ++p) dwb = dwb && all[p].dwb_ok == 1 && all[p].off_dwb == c.xoff_dwb;
  c.dwb = dwb;
  if (dwb) {
    c.peer_shard.assign(c.W, nullptr);
    for (int si = 0; si < 2; ++si) c.peer_dwb_slot[si].assign(c.W, nullptr);
    for (int p = 0; p < c.W; ++p) {
      const nest_window_rec_t& r = all[p];
      char* base = reinterpret_cast<char*>(c.peer_src[p]);   // window base
      for (int si = 0; si < 2; ++si)
        c.peer_dwb_slot[si][p] = reinterpret_cast<int32_t*>(base + r.off_dwb) + si * int64_t(r.dwb_stride);
      if (p == c.rank) {
        c.peer_shard[p] = c.shard;
      } else if (r.pid == me_pid) {
        c.peer_shard[p] = reinterpret_cast<float*>(r.shard_ptr);
      } else {
        void* ptr = nullptr;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, r.shard_ipc, sizeof(h));
        NEST_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        c.peer_shard_map.push_back(ptr);
        c.peer_shard[p] = reinterpret_cast<float*>(reinterpret_cast<char*>(ptr) + r.shard_off);
      }
    }
  }
  c.connected = true;
}

// NCCL mode: the records travel through the aux communicator
void xfer_setup(Ctx& c, cudaStream_t st) {
  xfer_alloc(c, st);
  nest_window_rec_t mine;
  xfer_export(c, &mine);
  char* dbuf = nullptr;
  const size_t rb = sizeof(nest_window_rec_t);
  NEST_CUDA(cudaMalloc(&dbuf, rb * (c.W + 1)));
  NEST_CUDA(cudaMemcpyAsync(dbuf + rb * c.rank, &mine, rb, cudaMemcpyHostToDevice, st));
  NEST_NCCL(ncclAllGather(dbuf + rb * c.rank, dbuf, rb, ncclUint8, c.comm_aux, st));
  std::vector<nest_window_rec_t> all(c.W);
  NEST_CUDA(cudaMemcpyAsync(all.data(), dbuf, rb * c.W, cudaMemcpyDeviceToHost, st));
  NEST_CUDA(cudaStreamSynchronize(st));
  NEST_CUDA(cudaFree(dbuf));
  xfer_connect(c, all.data());
}

void xfer_destroy(Ctx& c) {
  for (void* p : c.peer_win)
    if (p) cudaIpcCloseMemHandle(p);
  c.peer_win.clear();
  for (void* p : c.peer_shard_map) cudaIpcCloseMemHandle(p);
  c.peer_shard_map.clear();
  if (c.xwin) cudaFree(c.xwin);
  c.xwin = nullptr;
  if (c.send_stage) cudaFree(c.send_stage);
  c.send_stage = nullptr;
}

static inline size_t flag_at(const Ctx& c, int slot, int kind, int mb, int src) {
  return ((size_t(slot) * XK_COUNT + kind) * c.Nmax + mb) * c.W + src;
}
static inline size_t flag_index(const Ctx& c, const Slot& s, int kind, int mb, int src) {
  return flag_at(c, slot_index(c, s), kind, mb, src);
}

// flag (slot, kind, mb) := value in every peer's window, after the work queued on st
void xfer_signal_raw(Ctx& c, int slot, int kind, int mb, uint32_t value, cudaStream_t st) {
  for (int p = 0; p < c.W; ++p) {
    if (p == c.rank) continue;
    CUresult r = g_write(reinterpret_cast<CUstream>(st),
                         reinterpret_cast<CUdeviceptr>(c.peer_flags[p] + flag_at(c, slot, kind, mb, c.rank)),
                         cuuint32_t(value), 0);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
}
// st waits until every peer wrote flag (slot, kind, mb) >= value into this window
void xfer_wait_raw(Ctx& c, int slot, int kind, int mb, uint32_t value, cudaStream_t st) {
  for (int o = 0; o < c.W; ++o) {
    if (o == c.rank) continue;
    CUresult r = g_wait(reinterpret_cast<CUstream>(st),
                        reinterpret_cast<CUdeviceptr>(c.xflags + flag_at(c, slot, kind, mb, o)),
                        cuuint32_t(value), CU_STREAM_WAIT_VALUE_GEQ);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWaitValue32 failed");
  }
}

// rows: [W][W][Nc] counts of the slot; base_of(p, i) = row base of micro-batch
// i in rank p's requester (kind 0) / owner (kind 1) rows
int64_t src_base_at(const Slot& s, const Ctx& c, int p, int mb) {
  const int Nc = c.Nmax + 2;
  int64_t b = 0;
  for (int i = 0; i < mb; ++i)
    for (int o = 0; o < c.W; ++o) b += s.all[(size_t(p) * c.W + o) * Nc + 1 + i];
  return b;
}
int64_t own_base_at(const Slot& s, const Ctx& c, int p, int mb) {
  const int Nc = c.Nmax + 2;
  int64_t b = 0;
  for (int i = 0; i < mb; ++i)
    for (int r = 0; r < c.W; ++r) b += s.all[(size_t(r) * c.W + p) * Nc + 1 + i];
  return b;
}

// R7: owner `rank` pushes micro-batch mb's rows to every requester (on st)
// (self rows first; `after_self` is recorded between the self copy and the
// remote pushes so the local pool does not wait for the outgoing DMA)
void xfer_push_emb(Ctx& c, Slot& s, int mb, cudaStream_t st, cudaEvent_t after_self, const float* send_rows) {
  if (!send_rows) send_rows = c.own_rows;
  const int W = c.W, Nc = c.Nmax + 2, me = c.rank;
  const size_t row = size_t(c.D) * sizeof(float);
  for (int pass = 0; pass < 2; ++pass) {
  int64_t so = s.own_base[mb];
  for (int p = 0; p < W; ++p) {
    const int64_t cnt = s.all[(size_t(p) * W + me) * Nc + 1 + mb];
    if (cnt > 0 && (pass == 0) == (p == me)) {
      int64_t dst = src_base_at(s, c, p, mb);
      for (int o = 0; o < me; ++o) dst += s.all[(size_t(p) * W + o) * Nc + 1 + mb];
      NEST_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(peer_src_of(c, s, p)) + dst * row,
                                reinterpret_cast<const char*>(send_rows) + so * row, cnt * row,
                                cudaMemcpyDeviceToDevice, st));
    }
    so += cnt;
  }
  if (pass == 0) NEST_CUDA(cudaEventRecord(after_self, st));
  }
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    CUresult r = g_write(reinterpret_cast<CUstream>(st),
                         reinterpret_cast<CUdeviceptr>(c.peer_flags[p] + flag_index(c, s, XK_EMB, mb, me)),
                         cuuint32_t(s.epoch), 0);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
}

// epoch flag of (kind, mb) written into every peer after the preceding work
// on st (the fused kernels end with a system-scope fence)
void xfer_signal(Ctx& c, Slot& s, int kind, int mb, cudaStream_t st) {
  for (int p = 0; p < c.W; ++p) {
    if (p == c.rank) continue;
    CUresult r = g_write(reinterpret_cast<CUstream>(st),
                         reinterpret_cast<CUdeviceptr>(c.peer_flags[p] + flag_index(c, s, kind, mb, c.rank)),
                         cuuint32_t(s.epoch), 0);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
}

// the requester's stream waits for every owner's rows of micro-batch mb
// (kind XK_EMB) or for every owner's re-pushed rows (XK_REPUSH)
void xfer_wait_emb(Ctx& c, Slot& s, int mb, cudaStream_t st, int kind) {
  for (int o = 0; o < c.W; ++o) {
    if (o == c.rank) continue;
    CUresult r = g_wait(reinterpret_cast<CUstream>(st),
                        reinterpret_cast<CUdeviceptr>(c.xflags + flag_index(c, s, kind, mb, o)),
                        cuuint32_t(s.epoch), CU_STREAM_WAIT_VALUE_GEQ);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWaitValue32 failed");
  }
}

// R11: requester `rank` pushes micro-batch mb's gradient rows to every owner
void xfer_push_grad(Ctx& c, Slot& s, int mb, cudaStream_t st) {
  const int W = c.W, Nc = c.Nmax + 2, me = c.rank;
  const size_t row = size_t(c.D) * sizeof(float);
  int64_t so = s.src_base[mb];
  for (int p = 0; p < W; ++p) {
    const int64_t cnt = s.all[(size_t(me) * W + p) * Nc + 1 + mb];
    if (cnt > 0) {
      int64_t dst = own_base_at(s, c, p, mb);
      for (int r = 0; r < me; ++r) dst += s.all[(size_t(r) * W + p) * Nc + 1 + mb];
      NEST_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(c.peer_own[p]) + dst * row,
                                reinterpret_cast<const char*>(src_rows_of(c, s)) + so * row, cnt * row,
                                cudaMemcpyDeviceToDevice, st));
    }
    so += cnt;
  }
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    CUresult r = g_write(reinterpret_cast<CUstream>(st),
                         reinterpret_cast<CUdeviceptr>(c.peer_flags[p] + flag_index(c, s, XK_GRAD, mb, me)),
                         cuuint32_t(s.epoch), 0);
    NEST_CHECK(r == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
}

// the owner's stream waits for every requester's gradients of all micro-batches
void xfer_wait_grads(Ctx& c, Slot& s, cudaStream_t st) {
  for (int mb = 0; mb < s.N; ++mb)
    for (int r = 0; r < c.W; ++r) {
      if (r == c.rank) continue;
      CUresult res = g_wait(reinterpret_cast<CUstream>(st),
                            reinterpret_cast<CUdeviceptr>(c.xflags + flag_index(c, s, XK_GRAD, mb, r)),
                            cuuint32_t(s.epoch), CU_STREAM_WAIT_VALUE_GEQ);
      NEST_CHECK(res == CUDA_SUCCESS, NEST_ERR_CUDA, "cuStreamWaitValue32 failed");
    }
}

}  // namespace nest
