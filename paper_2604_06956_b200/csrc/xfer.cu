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

#include <cstring>

#include "nest_internal.cuh"

namespace nest {

using PFN_wait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static PFN_wait g_wait = nullptr;
static PFN_write g_write = nullptr;

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
//                 own_rows OMBcap*D f32 | flags [2][3][Nmax][W] u32]
void xfer_setup(Ctx& c, cudaStream_t st) {
  load_driver_ops();
  c.a2a_mode = a2a_mode_wanted(c.W);
  c.early_push = c.a2a_mode == A2A_FUSED ? early_push_wanted() : EP_OFF;
  {
    // gradients under the fused transport: segment-sum stores into the
    // owners' windows (sm, default) or local rows + copy-engine DMA (ce)
    const char* g = std::getenv("NEST_GRAD_PUSH");
    c.grad_ce = c.a2a_mode == A2A_FUSED && g && std::strcmp(g, "ce") == 0;
  }
  if (c.early_push == EP_CE)
    NEST_CUDA(cudaMalloc(&c.send_stage, std::max<size_t>(size_t(c.OMBcap) * c.D * sizeof(float), 256)));
  const size_t src1 = align_up(size_t(c.MBcap) * c.D * sizeof(float), 4096);
  const size_t src_b = c.early_push ? 2 * src1 : src1;
  const size_t own_b = align_up(size_t(c.OMBcap) * c.D * sizeof(float), 4096);
  const size_t flg_b = align_up(size_t(2) * XK_COUNT * c.Nmax * c.W * sizeof(uint32_t), 4096);
  c.src_slot_stride = c.early_push ? int64_t(src1 / sizeof(float)) : 0;
  c.xwin_bytes = src_b + own_b + flg_b;
  NEST_CUDA(cudaMalloc(&c.xwin, c.xwin_bytes));
  NEST_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(c.xwin) + src_b + own_b, 0, flg_b, st));
  c.xoff_own = src_b;
  c.xoff_flags = src_b + own_b;
  c.src_rows = reinterpret_cast<float*>(c.xwin);
  c.own_rows = reinterpret_cast<float*>(reinterpret_cast<char*>(c.xwin) + src_b);
  c.xflags = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c.xwin) + c.xoff_flags);
  // exchange IPC handles (+ window geometry) through the aux communicator
  struct Rec {
    cudaIpcMemHandle_t h;
    uint64_t own, flags, bytes, src_stride;
  };
  Rec mine{};
  NEST_CUDA(cudaIpcGetMemHandle(&mine.h, c.xwin));
  mine.src_stride = uint64_t(c.src_slot_stride);
  mine.own = c.xoff_own;
  mine.flags = c.xoff_flags;
  mine.bytes = c.xwin_bytes;
  char* dbuf = nullptr;
  NEST_CUDA(cudaMalloc(&dbuf, sizeof(Rec) * (c.W + 1)));
  NEST_CUDA(cudaMemcpyAsync(dbuf + sizeof(Rec) * c.rank, &mine, sizeof(Rec), cudaMemcpyHostToDevice, st));
  NEST_NCCL(ncclAllGather(dbuf + sizeof(Rec) * c.rank, dbuf, sizeof(Rec), ncclUint8, c.comm_aux, st));
  std::vector<Rec> all(c.W);
  NEST_CUDA(cudaMemcpyAsync(all.data(), dbuf, sizeof(Rec) * c.W, cudaMemcpyDeviceToHost, st));
  NEST_CUDA(cudaStreamSynchronize(st));
  NEST_CUDA(cudaFree(dbuf));
  c.peer_win.assign(c.W, nullptr);
  c.peer_src.assign(c.W, nullptr);
  c.peer_own.assign(c.W, nullptr);
  c.peer_flags.assign(c.W, nullptr);
  c.peer_src_slot[0].assign(c.W, nullptr);
  c.peer_src_slot[1].assign(c.W, nullptr);
  for (int p = 0; p < c.W; ++p) {
    char* base;
    if (p == c.rank) {
      base = reinterpret_cast<char*>(c.xwin);
    } else {
      void* ptr = nullptr;
      NEST_CUDA(cudaIpcOpenMemHandle(&ptr, all[p].h, cudaIpcMemLazyEnablePeerAccess));
      base = reinterpret_cast<char*>(ptr);
      c.peer_win[p] = ptr;
    }
    c.peer_src[p] = reinterpret_cast<float*>(base);
    c.peer_src_slot[0][p] = c.peer_src[p];
    c.peer_src_slot[1][p] = c.peer_src[p] + all[p].src_stride;
    c.peer_own[p] = reinterpret_cast<float*>(base + all[p].own);
    c.peer_flags[p] = reinterpret_cast<uint32_t*>(base + all[p].flags);
  }
  // (no barrier needed: the first push happens after the first route's count
  // exchange, a collective every rank enters after this setup)
  c.xfer_ce = true;
}

void xfer_destroy(Ctx& c) {
  for (void* p : c.peer_win)
    if (p) cudaIpcCloseMemHandle(p);
  c.peer_win.clear();
  if (c.xwin) cudaFree(c.xwin);
  c.xwin = nullptr;
  if (c.send_stage) cudaFree(c.send_stage);
  c.send_stage = nullptr;
}

static inline size_t flag_index(const Ctx& c, const Slot& s, int kind, int mb, int src) {
  return ((size_t(slot_index(c, s)) * XK_COUNT + kind) * c.Nmax + mb) * c.W + src;
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
