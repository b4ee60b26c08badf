// C ABI entry points of libnest.so (include/nest.h) and the per-rank runtime:
// configuration checks, workspace carving, NCCL communicators, pipeline-slot
// events, and the stream/event choreography of DBP + FWP (P:363-380,
// P:457-467).
#include <cmath>
#include <cstring>
#include <exception>

#include "nest_internal.cuh"

namespace nest {

static thread_local std::string g_create_error;

// ---------------------------------------------------------------------------
// configuration
// ---------------------------------------------------------------------------
static void derive(Ctx& c, const nest_config_t* cfg) {
  NEST_CHECK(cfg != nullptr, NEST_ERR_INVALID, "null config");
  c.cfg = *cfg;
  c.W = cfg->world;
  c.rank = cfg->rank;
  c.T = cfg->num_tables;
  c.D = cfg->dim;
  c.F = cfg->num_features;
  c.Nmax = cfg->max_micro_batches;
  NEST_CHECK(c.W >= 1 && c.W <= NEST_MAX_WORLD, NEST_ERR_INVALID, "world out of range");
  NEST_CHECK(c.rank >= 0 && c.rank < c.W, NEST_ERR_INVALID, "rank out of range");
  NEST_CHECK(c.T >= 1 && c.T <= NEST_MAX_TABLES, NEST_ERR_INVALID, "num_tables out of range");
  NEST_CHECK(c.D == 16 || c.D == 32 || c.D == 64 || c.D == 128 || c.D == 256, NEST_ERR_INVALID,
             "dim must be one of 16, 32, 64, 128, 256");
  NEST_CHECK(cfg->table_rows != nullptr, NEST_ERR_INVALID, "table_rows is null");
  NEST_CHECK(cfg->pooling == NEST_POOL_SUM || cfg->pooling == NEST_POOL_NONE, NEST_ERR_INVALID,
             "bad pooling");
  NEST_CHECK(c.F >= 1, NEST_ERR_INVALID, "num_features < 1");
  NEST_CHECK(cfg->max_keys >= 1 && cfg->max_keys < (int64_t(1) << kMbShift), NEST_ERR_INVALID,
             "max_keys must be in [1, 2^28)");
  NEST_CHECK(cfg->max_batch >= 1 && cfg->max_batch * c.F < (int64_t(1) << 31), NEST_ERR_INVALID,
             "max_batch out of range");
  NEST_CHECK(c.Nmax >= 1 && c.Nmax <= NEST_MAX_MICRO_BATCHES, NEST_ERR_INVALID,
             "max_micro_batches must be in [1, 8]");
  NEST_CHECK(cfg->init_mode >= 0 && cfg->init_mode <= 2, NEST_ERR_INVALID, "bad init_mode");
  NEST_CHECK(cfg->optimizer == NEST_OPT_SGD || cfg->optimizer == NEST_OPT_ROWWISE_ADAGRAD, NEST_ERR_INVALID,
             "bad optimizer");
  NEST_CHECK(cfg->optimizer == NEST_OPT_SGD || cfg->adagrad_eps >= 0.f, NEST_ERR_INVALID,
             "adagrad_eps must be >= 0");
  NEST_CHECK(cfg->table_location == NEST_TABLE_HBM || cfg->table_location == NEST_TABLE_HOST, NEST_ERR_INVALID,
             "bad table_location");
  NEST_CHECK(cfg->tower_train == 0 || (cfg->tower_train == 1 && cfg->tower_layers > 0), NEST_ERR_INVALID,
             "tower_train needs tower_layers > 0");
  // checked here, before any collective initialisation (tower_create repeats it)
  NEST_CHECK(cfg->tower_layers <= 0 || (cfg->tower_hidden >= 16 && cfg->tower_hidden % 16 == 0),
             NEST_ERR_INVALID, "tower_hidden must be a positive multiple of 16");
  c.rows.assign(cfg->table_rows, cfg->table_rows + c.T);
  for (int t = 0; t < c.T; ++t)
    NEST_CHECK(c.rows[t] >= 1 && c.rows[t] <= int64_t(kRowMask), NEST_ERR_INVALID, "bad table_rows");
  // owner-major domain: segment (o, t) holds the rows of table t owned by o
  c.seg_base.assign(size_t(c.W) * c.T + 1, 0);
  int64_t acc = 0;
  for (int o = 0; o < c.W; ++o)
    for (int t = 0; t < c.T; ++t) {
      c.seg_base[size_t(o) * c.T + t] = acc;
      acc += c.rows[t] > o ? (c.rows[t] - o + c.W - 1) / c.W : 0;
    }
  c.seg_base[size_t(c.W) * c.T] = acc;
  c.V = acc;
  NEST_CHECK(c.V < (int64_t(1) << 31) - 64, NEST_ERR_INVALID, "total rows must be < 2^31");
  c.lbase.assign(c.T + 1, 0);
  const int64_t r0 = c.seg_base[size_t(c.rank) * c.T];
  for (int t = 0; t <= c.T; ++t) c.lbase[t] = c.seg_base[size_t(c.rank) * c.T + t] - r0;
  c.Vo = c.lbase[c.T];
  c.words = (c.V + 31) / 32;
  c.owords = (c.Vo + 31) / 32;
  c.Kcap = cfg->max_keys;
  c.Bcap = cfg->max_batch;
  if (cfg->max_recv_keys > 0)
    c.Rcap = cfg->max_recv_keys;
  else
    c.Rcap = c.W == 1 ? c.Kcap : std::min<int64_t>(2 * c.Kcap, c.W * c.Kcap);
  NEST_CHECK(c.Rcap < (int64_t(1) << 31) - 64, NEST_ERR_INVALID, "max_recv_keys too large");
  // U_o <= R_o <= Rcap and U_o <= shard rows, so this never overflows
  c.Uocap = std::max<int64_t>(1, std::min<int64_t>(c.Rcap, c.Vo));
  c.MBcap = cfg->max_mb_rows > 0 ? cfg->max_mb_rows : c.Kcap;
  if (c.W == 1)
    c.OMBcap = c.MBcap;
  else
    c.OMBcap = cfg->max_owner_mb_rows > 0 ? cfg->max_owner_mb_rows
                                          : (c.Nmax > 1 ? 2 * c.Rcap : c.Rcap);
  c.Pcap = 2 * c.Kcap / 32 + 64;   // partial rows for chunk length >= 32
  if (const char* g = std::getenv("NEST_GUARD")) c.guard = std::atoi(g) != 0;
  if (const char* e = std::getenv("NEST_SEG_CHUNK")) c.seg_chunk = std::max(32, std::atoi(e));
}

size_t tower_workspace_bytes(const Ctx& c);
void tower_bind(Ctx& c, char* mem);

static size_t layout(Ctx& c, char* base) {
  Carver w{base};
  c.guard_offs.clear();
  if (c.guard) w.guards = &c.guard_offs;
  const int64_t K = c.Kcap, B = c.Bcap, R = c.Rcap, Uo = c.Uocap, D = c.D, W = c.W, Nm = c.Nmax;
  const int Nc = c.Nmax + 2;
  int64_t maxn = std::max<int64_t>({c.words + 2, c.owords + 2, K + 2, R + 2, B + 2,
                                    int64_t(1 << kRadixMaxDigit) * radix_blocks(K) + 2});
  const int64_t scan_bytes = (scan_blocks(maxn) + 4) * int64_t(sizeof(I2));
  c.d_rows = w.take<int64_t>(c.T);
  c.d_seg_base = w.take<int64_t>(W * c.T + 1);
  c.d_lbase = w.take<int64_t>(c.T + 1);
  c.sbm = w.take<uint32_t>(c.words + 2);
  c.swr = w.take<int32_t>(c.words + 2);
  c.occ_dom = w.take<uint32_t>(K);
  c.occ_mbrow = w.take<int32_t>(K);
  for (int i = 0; i < 2; ++i) {
    c.tkey[i] = w.take<uint32_t>(K);
    c.tval[i] = w.take<int32_t>(K);
  }
  c.hist = w.take<uint32_t>(int64_t(1 << kRadixMaxDigit) * radix_blocks(K) + 2);
  c.radix_aux = w.take<uint32_t>(kRadixAux);
  c.scan_tmp = w.take<char>(scan_bytes);
  // the clustering sort (aux stream) and the occurrence sorts (sort stream)
  // have separate scratch: they run concurrently
  c.rx_aux.tkey[0] = c.tkey[0];
  c.rx_aux.tkey[1] = c.tkey[1];
  c.rx_aux.tval[0] = c.tval[0];
  c.rx_aux.tval[1] = c.tval[1];
  c.rx_aux.hist = c.hist;
  c.rx_aux.scan_tmp = c.scan_tmp;
  c.rx_aux.aux = c.radix_aux;
  {
    uint32_t* hs = w.take<uint32_t>(int64_t(1 << kRadixMaxDigit) * radix_blocks(K) + 2);
    uint32_t* as = w.take<uint32_t>(kRadixAux);
    char* ss = w.take<char>(scan_bytes);
    for (int si = 0; si < 2; ++si) {
      RadixScratch& rx = c.slot[si].rx;
      for (int i = 0; i < 2; ++i) {
        rx.tkey[i] = w.take<uint32_t>(K);
        rx.tval[i] = w.take<int32_t>(K);
      }
      rx.hist = hs;
      rx.aux = as;
      rx.scan_tmp = ss;
    }
  }
  c.scan_tmp_win = w.take<char>(scan_bytes);
  c.samp_scratch = w.take<int32_t>(B + 2);
  c.packed = w.take<int64_t>(W > 1 ? K : 1);
  c.r_ldom = w.take<uint32_t>(W > 1 ? R : 1);
  c.seg_start = w.take<int32_t>(K + 2);
  c.seg_aux = w.take<int32_t>(K + 2);
  c.hot_list = w.take<int32_t>(K + 1);
  c.seg_tot = w.take<int32_t>(4);
  c.partial = w.take<float>(c.Pcap * D);
  if (xfer_wanted(int(W))) {
    c.src_rows = c.own_rows = nullptr;  // live in the IPC exchange window (xfer_setup)
  } else {
    c.src_rows = w.take<float>(c.MBcap * D);
    c.own_rows = W > 1 ? w.take<float>(c.OMBcap * D) : c.src_rows;
  }
  c.d_err = w.take<int32_t>(4);
  c.d_cnt_scratch = w.take<int32_t>(W * Nm + 1);
  c.n_refreshed = w.take<int32_t>(4);
  if (Nm > 1) {
    c.cl_bm = w.take<uint32_t>(c.words + 2);
    c.cl_wr = w.take<int32_t>(c.words + 2);
    c.cl_samp = w.take<int32_t>(K);
    c.cl_sk = w.take<uint32_t>(K + 1);
    c.cl_sv = w.take<int32_t>(K);
    c.cl_u = w.take<int32_t>(K);
    c.cl_inmask = w.take<uint32_t>(K);
    c.cl_size = w.take<int32_t>(B);
    c.cl_grp = w.take<int32_t>(B);
    c.cl_S = w.take<int32_t>(Nm * B);
    c.cl_new = w.take<int32_t>(B);
    c.cl_small = w.take<int64_t>(4);
    c.cl_hist = w.take<int32_t>(int64_t(Nm + 1) * kClHistBins);
    c.cl_sel = w.take<int32_t>(8 * Nm);
    c.cl_bcnt = w.take<int32_t>(((B + kClIds - 1) / kClIds + 1) * Nm);
    c.cl_boff = w.take<int32_t>(B * c.F + 1);
    c.cl_Scnt = w.take<int32_t>(Nm * B);
    c.cl_kstart = w.take<int32_t>(K + 2);
    // work items per round: fresh (key, group) pairs <= K (keys of the taken
    // samples) plus chunk extras <= N * K / 128 (a key fresh for every group)
    c.cl_newk_cap = K + Nm * (K / 128 + 1) + 64;
    c.cl_newk = w.take<uint64_t>(c.cl_newk_cap);
  }
  for (int si = 0; si < 2; ++si) {
    Slot& s = c.slot[si];
    s.uniq = w.take<int64_t>(K);
    s.inverse = w.take<int32_t>(K);
    s.mask = w.take<uint32_t>(K);
    s.pos = w.take<int32_t>(Nm * (K + 1));
    s.skey = w.take<uint32_t>(K);
    s.sval = w.take<int32_t>(K);
    s.perm = w.take<int32_t>(B);
    s.bag_off = w.take<int32_t>(B * c.F + 1);
    s.samp_base = w.take<int32_t>(B);
    s.mb_of = w.take<int32_t>(B);
    s.off = w.take<int32_t>(W + 1);
    s.xfer = w.take<int32_t>(W * W * Nc + Nm + 1);
    const int64_t ow = W > 1 ? c.owords : c.words;
    s.obm = w.take<uint32_t>(ow + 2);
    s.owr = w.take<int32_t>(ow + 2);
    s.owner_rows = w.take<int32_t>(Uo);
    s.n_owner = w.take<int32_t>(1);
    if (W > 1) {
      s.recv = w.take<int64_t>(R);
      s.owner_inv = w.take<int32_t>(R);
      s.src_tab = w.take<int32_t>(Uo * W);
      s.sendpos = w.take<int32_t>(Nm * (R + 1));
      s.upd_list = w.take<int32_t>(Uo);
      s.n_upd = w.take<int32_t>(1);
    }
    s.buffer = w.take<float>(Uo * D);
  }
  const size_t tw = tower_workspace_bytes(c);
  char* tmem = w.take<char>(int64_t(tw));
  if (base) tower_bind(c, tw ? tmem : nullptr);
  return w.off + 256;
}

// ---------------------------------------------------------------------------
// guard: exceptions -> status codes, sticky device/comm errors
// ---------------------------------------------------------------------------
template <class Fn>
static nest_status_t guard(Ctx* c, Fn&& fn) {
  if (c && c->sticky != NEST_OK) return c->sticky;
  try {
    fn();
    return NEST_OK;
  } catch (const Error& e) {
    if (c) {
      c->last_error = e.msg;
      if (e.code == NEST_ERR_CUDA || e.code == NEST_ERR_NCCL || e.code == NEST_ERR_KEY_RANGE ||
          e.code == NEST_ERR_SHARD)
        c->sticky = e.code;
    } else {
      g_create_error = e.msg;
    }
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what(); else g_create_error = e.what();
    return NEST_ERR_INVALID;
  }
}

static cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

static Slot& slot_of(Ctx& c, int32_t slot) {
  NEST_CHECK(slot == 0 || slot == 1, NEST_ERR_INVALID, "slot must be 0 or 1");
  return c.slot[slot];
}

// grouped send/recv All2Allv of fp32 rows
static void a2a_rows(Ctx& c, const float* send, const std::vector<int64_t>& scnt, float* recv,
                     const std::vector<int64_t>& rcnt, cudaStream_t st) {
  const int W = c.W;
  int64_t so = 0, ro = 0;
  NEST_NCCL(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    NEST_NCCL(ncclSend(send + so * c.D, size_t(scnt[p] * c.D), ncclFloat32, p, c.comm, st));
    NEST_NCCL(ncclRecv(recv + ro * c.D, size_t(rcnt[p] * c.D), ncclFloat32, p, c.comm, st));
    so += scnt[p];
    ro += rcnt[p];
  }
  NEST_NCCL(ncclGroupEnd());
}

// R6 + R7 of micro-batch mb on the comm stream: owner send gather + embedding
// All2All into the requester's receive rows; records ev_emb[mb]
static void lookup_comm(Ctx& c, Slot& s, int mb, cudaStream_t cs, cudaStream_t ms) {
  if (mb == 0 || s.prefetched == 0) {
    // the window starts after everything queued on compute (the refresh) and
    // the slot's gather; later micro-batches only follow the comm chain
    NEST_CUDA(cudaEventRecord(s.ev_ready, cs));
    NEST_CUDA(cudaStreamWaitEvent(ms, s.ev_ready, 0));
    NEST_CUDA(cudaStreamWaitEvent(ms, s.ev_gather, 0));
  }
  const double row = double(c.D) * sizeof(float);
  if (c.a2a_mode == A2A_FUSED) {
    // R6 + R7 in one kernel: gather rows of the frozen buffer and store them
    // straight into every requester's receive rows over NVLink
    {
      ProfScope ps(c, ST_EMB_A2A, SK_COMM, ms);
      launch_send_push(c, s, mb, ms);
      int64_t self = s.all[(size_t(c.rank) * c.W + c.rank) * (c.Nmax + 2) + 1 + mb];
      ps.dcount = c.n_refreshed + 1;   // rows sent off-GPU (counted on the device)
      ps.bpc = row;
      ps.hbm = row * double(s.info.mb_recv[mb] + self);    // rows gathered + rows stored locally
    }
    NEST_CUDA(cudaEventRecord(s.ev_emb[mb], ms));
    xfer_signal(c, s, 0, mb, ms);
    s.prefetched |= 1u << mb;
    return;
  }
  {
    ProfScope ps(c, ST_SEND_GATHER, SK_COMM, ms);
    launch_send_gather(c, s, mb, ms);
    // R_{o,i} buffer rows read + R_{o,i} rows written + 12 B of indices per received key
    ps.bytes = 2.0 * row * double(s.info.mb_recv[mb]) + 12.0 * double(s.info.recv);
  }
  std::vector<int64_t> scnt(c.W), rcnt(c.W);
  const int Nc = c.Nmax + 2;
  for (int p = 0; p < c.W; ++p) {
    scnt[p] = s.all[(size_t(p) * c.W + c.rank) * Nc + 1 + mb];  // owner -> requester p
    rcnt[p] = s.all[(size_t(c.rank) * c.W + p) * Nc + 1 + mb];  // from owner p
  }
  {
    ProfScope ps(c, ST_EMB_A2A, SK_COMM, ms);
    if (c.xfer_ce) {
      xfer_push_emb(c, s, mb, ms, s.ev_emb[mb]);  // records ev_emb after the self rows
    } else {
      a2a_rows(c, c.own_rows + s.own_base[mb] * c.D, scnt, c.src_rows + s.src_base[mb] * c.D, rcnt, ms);
      NEST_CUDA(cudaEventRecord(s.ev_emb[mb], ms));
    }
    ps.launches = 0;
    ps.bytes = row * double(s.info.mb_recv[mb] - scnt[c.rank]);  // rows sent off-GPU
  }
  s.prefetched |= 1u << mb;
}

}  // namespace nest

using namespace nest;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* nest_version(void) { return "nestpipe-b200 0.1 (sm_100a)"; }

nest_status_t nest_get_unique_id(void* uid_out) {
  if (!uid_out) return NEST_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return NEST_ERR_NCCL;
  std::memcpy(uid_out, &id, sizeof(id));
  return NEST_OK;
}

nest_status_t nest_workspace_bytes(const nest_config_t* cfg, size_t* table_bytes, size_t* work_bytes) {
  return guard(nullptr, [&] {
    NEST_CHECK(table_bytes && work_bytes, NEST_ERR_INVALID, "null output");
    Ctx c;
    derive(c, cfg);
    *table_bytes = size_t(std::max<int64_t>(c.Vo, 1)) * c.D * sizeof(float);
    if (cfg->optimizer == NEST_OPT_ROWWISE_ADAGRAD)   // + one fp32 accumulator per row
      *table_bytes += size_t(std::max<int64_t>(c.Vo, 1)) * sizeof(float);
    *work_bytes = layout(c, nullptr);
  });
}

int64_t nest_shard_rows(const nest_config_t* cfg) {
  Ctx c;
  try {
    derive(c, cfg);
  } catch (...) {
    return -1;
  }
  return c.Vo;
}

nest_status_t nest_create(const nest_config_t* cfg, const void* nccl_uids, void* table_mem,
                          void* work_mem, void* stream, nest_ctx_t** out) {
  if (!out) return NEST_ERR_INVALID;
  *out = nullptr;
  Ctx* c = new Ctx();
  nest_status_t st = guard(nullptr, [&] {
    derive(*c, cfg);
    NEST_CHECK(table_mem && work_mem, NEST_ERR_INVALID, "null table_mem / work_mem");
    NEST_CHECK((reinterpret_cast<uintptr_t>(table_mem) & 255) == 0 &&
                   (reinterpret_cast<uintptr_t>(work_mem) & 255) == 0,
               NEST_ERR_INVALID, "memory must be 256-byte aligned");
    {
      // the table tier: device memory (HBM) or pinned host memory reached over
      // PCIe through its UVA device alias (host-DRAM tier, NEXT-3)
      cudaPointerAttributes pa{};
      NEST_CUDA(cudaPointerGetAttributes(&pa, table_mem));
      if (c->cfg.table_location == NEST_TABLE_HOST) {
        NEST_CHECK(pa.type == cudaMemoryTypeHost && pa.devicePointer != nullptr, NEST_ERR_INVALID,
                   "table_location HOST needs pinned, device-mapped host memory");
        c->shard = reinterpret_cast<float*>(pa.devicePointer);
      } else {
        NEST_CHECK(pa.type == cudaMemoryTypeDevice, NEST_ERR_INVALID,
                   "table_location HBM needs device memory (pinned host memory: NEST_TABLE_HOST)");
        c->shard = reinterpret_cast<float*>(table_mem);
      }
    }
    if (const char* e = std::getenv("NEST_GATHER_SKIP")) c->gather_skip = std::atoi(e) != 0;
    if (const char* e = std::getenv("NEST_ZERO_COPY")) c->zero_copy = std::atoi(e) != 0;
    if (c->cfg.optimizer == NEST_OPT_ROWWISE_ADAGRAD) {
      c->opt_state = c->shard + std::max<int64_t>(c->Vo, 1) * c->D;
      zero_f32(c->opt_state, std::max<int64_t>(c->Vo, 1), S(stream));
    }
    layout(*c, reinterpret_cast<char*>(work_mem));
    c->work_base = reinterpret_cast<char*>(work_mem);
    if (c->guard && !c->guard_offs.empty()) {
      const size_t ng = c->guard_offs.size();
      NEST_CUDA(cudaMalloc(&c->d_guard_offs, sizeof(uint64_t) * ng));
      NEST_CUDA(cudaMalloc(&c->d_guard_bad, sizeof(unsigned long long)));
      std::vector<uint64_t> go(c->guard_offs.begin(), c->guard_offs.end());
      NEST_CUDA(cudaMemcpyAsync(c->d_guard_offs, go.data(), sizeof(uint64_t) * ng, cudaMemcpyHostToDevice,
                                S(stream)));
      guards_fill(*c, S(stream));
      NEST_CUDA(cudaStreamSynchronize(S(stream)));
    }
    cudaStream_t st0 = S(stream);
    NEST_CUDA(cudaMemcpyAsync(c->d_rows, c->rows.data(), sizeof(int64_t) * c->T, cudaMemcpyHostToDevice, st0));
    NEST_CUDA(cudaMemcpyAsync(c->d_seg_base, c->seg_base.data(), sizeof(int64_t) * c->seg_base.size(),
                              cudaMemcpyHostToDevice, st0));
    NEST_CUDA(cudaMemcpyAsync(c->d_lbase, c->lbase.data(), sizeof(int64_t) * c->lbase.size(),
                              cudaMemcpyHostToDevice, st0));
    NEST_CUDA(cudaMemsetAsync(c->d_err, 0, sizeof(int32_t) * 4, st0));
    const int Nc = c->Nmax + 2;
    for (int si = 0; si < 2; ++si) {
      Slot& s = c->slot[si];
      NEST_CUDA(cudaMallocHost(&s.h_xfer, sizeof(int32_t) * (int64_t(c->W) * c->W * Nc + c->Nmax + 1)));
      NEST_CUDA(cudaMemsetAsync(s.n_owner, 0, sizeof(int32_t), st0));
      NEST_CUDA(cudaMemsetAsync(s.off, 0, sizeof(int32_t) * (c->W + 1), st0));
      cudaEvent_t* evs[] = {&s.ev_gather, &s.ev_update, &s.ev_free, &s.ev_ready, &s.ev_sync, &s.ev_early,
                            &s.ev_repush, &s.ev_sorted};
      for (auto* e : evs) NEST_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      for (int i = 0; i < NEST_MAX_MICRO_BATCHES; ++i) {
        NEST_CUDA(cudaEventCreateWithFlags(&s.ev_emb[i], cudaEventDisableTiming));
        NEST_CUDA(cudaEventCreateWithFlags(&s.ev_grad[i], cudaEventDisableTiming));
      }
    }
    NEST_CUDA(cudaEventCreateWithFlags(&c->ev_scratch, cudaEventDisableTiming));
    {
      int lo = 0, hi = 0;
      NEST_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      NEST_CUDA(cudaStreamCreateWithPriority(&c->sort_stream, cudaStreamNonBlocking, lo));
      NEST_CUDA(cudaEventCreateWithFlags(&c->ev_sort_join, cudaEventDisableTiming));
    }
    if (c->cl_u) NEST_CUDA(cudaMallocHost(&c->cl_hmax, sizeof(int32_t)));
    NEST_CUDA(cudaStreamSynchronize(st0));
    if (c->W > 1 && c->cfg.tower_train && c->cfg.tower_layers > 0 && nccl_uids == nullptr) {
      // the trained tower's dense AllReduce goes through the window too
      const int64_t H = c->cfg.tower_hidden, L = c->cfg.tower_layers;
      const int64_t n = int64_t(c->F) * c->D * H + (L - 1) * H * H;
      c->twr_elems = (n + c->W - 1) / c->W * c->W;
    }
    if (c->W > 1 && nccl_uids == nullptr) {
      // no NCCL: every exchange over the peer-mapped windows; the caller
      // connects them (nest_window_export / nest_window_connect)
      NEST_CHECK(xfer_wanted(c->W), NEST_ERR_INVALID,
                 "world > 1 without NCCL ids needs the fused or ce transport (NEST_A2A != nccl)");
      c->route_window = true;
      xfer_alloc(*c, st0);
      NEST_CUDA(cudaStreamSynchronize(st0));
    } else if (c->W > 1) {
      ncclUniqueId id0, id1;
      std::memcpy(&id0, nccl_uids, sizeof(id0));
      std::memcpy(&id1, reinterpret_cast<const char*>(nccl_uids) + sizeof(id0), sizeof(id1));
      // bound NCCL's CTAs so the All2Alls leave SMs to the overlapped compute
      // (SURVEY H3); NEST_NCCL_MAX_CTAS overrides
      ncclConfig_t cfg0 = NCCL_CONFIG_INITIALIZER, cfg1 = NCCL_CONFIG_INITIALIZER;
      const char* mc = std::getenv("NEST_NCCL_MAX_CTAS");
      cfg0.maxCTAs = mc ? std::atoi(mc) : 16;
      cfg1.maxCTAs = mc ? std::atoi(mc) : 8;
      NEST_NCCL(ncclCommInitRankConfig(&c->comm, c->W, id0, c->rank, &cfg0));
      NEST_NCCL(ncclCommInitRankConfig(&c->comm_aux, c->W, id1, c->rank, &cfg1));
      if (xfer_wanted(c->W)) {
        // the count exchange and key All2All over the window as well (peer
        // stores + flags; measured equal or better: W=2 E 2.52 vs 2.57 ms,
        // E+T and W=4 tied) -- NEST_ROUTE_XCHG=nccl keeps them on NCCL
        const char* rx = std::getenv("NEST_ROUTE_XCHG");
        c->route_window = !(rx && std::strcmp(rx, "nccl") == 0);
        xfer_setup(*c, st0);
      }
    }
    if (c->cfg.tower_layers > 0) tower_create(*c);
  });
  if (st != NEST_OK) {
    // release whatever was created before the failure (pinned mirrors, events,
    // communicators, the IPC window, the tower): nest_destroy skips null members
    nest_destroy(reinterpret_cast<nest_ctx_t*>(c));
    return st;
  }
  *out = reinterpret_cast<nest_ctx_t*>(c);
  return NEST_OK;
}

nest_status_t nest_window_export(const nest_ctx_t* ctx, nest_window_rec_t* rec) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !rec) return NEST_ERR_INVALID;
  return guard(const_cast<Ctx*>(c), [&] { xfer_export(*c, rec); });
}

nest_status_t nest_window_connect(nest_ctx_t* ctx, const nest_window_rec_t* recs) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !recs) return NEST_ERR_INVALID;
  return guard(c, [&] { xfer_connect(*c, recs); });
}

nest_status_t nest_check_guards(nest_ctx_t* ctx, void* stream, int64_t* bad_words) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !bad_words) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(c->guard, NEST_ERR_INVALID, "context not created in checked mode (NEST_GUARD=1)");
    *bad_words = guards_check(*c, S(stream));
  });
}

nest_status_t nest_destroy(nest_ctx_t* ctx) {
  if (!ctx) return NEST_OK;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  cudaDeviceSynchronize();
  if (c->d_guard_offs) cudaFree(c->d_guard_offs);
  if (c->d_guard_bad) cudaFree(c->d_guard_bad);
  if (c->tower) tower_destroy(*c);
  profile_destroy(*c);
  xfer_destroy(*c);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_aux) ncclCommDestroy(c->comm_aux);
  if (c->ev_scratch) cudaEventDestroy(c->ev_scratch);
  if (c->sort_stream && c->sort_stream_owned) cudaStreamDestroy(c->sort_stream);
  if (c->ev_sort_join) cudaEventDestroy(c->ev_sort_join);
  if (c->cl_hmax) cudaFreeHost(c->cl_hmax);
  for (auto& kv : c->cl_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& s : c->slot) {
    if (s.h_xfer) cudaFreeHost(s.h_xfer);
    cudaEvent_t evs[] = {s.ev_gather, s.ev_update, s.ev_free, s.ev_ready, s.ev_sync, s.ev_early, s.ev_repush,
                         s.ev_sorted};
    for (auto e : evs)
      if (e) cudaEventDestroy(e);
    for (int i = 0; i < NEST_MAX_MICRO_BATCHES; ++i) {
      if (s.ev_emb[i]) cudaEventDestroy(s.ev_emb[i]);
      if (s.ev_grad[i]) cudaEventDestroy(s.ev_grad[i]);
    }
  }
  delete c;
  return NEST_OK;
}

nest_status_t nest_init_tables(nest_ctx_t* ctx, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    launch_init_tables(*c, S(stream));
    if (c->opt_state)   // row-wise AdaGrad accumulators start at 0
      zero_f32(c->opt_state, std::max<int64_t>(c->Vo, 1), S(stream));
  });
}

nest_status_t nest_fwp_schedule(nest_ctx_t* ctx, const int64_t* keys, const int32_t* bag_offsets,
                                int64_t nnz, int32_t B, int32_t N, int32_t mode, int32_t* perm_out,
                                int32_t* mb_offsets_out, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(c->route_open < 0, NEST_ERR_ORDER, "a route is open (nest_route_end first)");
    NEST_CHECK(N >= 1 && N <= c->Nmax, NEST_ERR_INVALID, "N out of range");
    NEST_CHECK(B >= 0 && B <= c->Bcap, NEST_ERR_INVALID, "B out of range");
    NEST_CHECK(B % N == 0, NEST_ERR_DIVISIBILITY, "B mod N != 0");
    NEST_CHECK(mode == NEST_SCHED_SEQUENTIAL || mode == NEST_SCHED_CLUSTERED, NEST_ERR_INVALID, "bad mode");
    NEST_CHECK(perm_out && mb_offsets_out, NEST_ERR_INVALID, "null output");
    NEST_CHECK(mode == NEST_SCHED_SEQUENTIAL || ((keys || nnz == 0) && bag_offsets), NEST_ERR_INVALID,
               "null batch");
    NEST_CHECK(nnz >= 0 && nnz <= c->Kcap, NEST_ERR_CAPACITY, "nnz exceeds max_keys");
    NEST_CHECK(mode == NEST_SCHED_SEQUENTIAL || N == 1 || c->cl_u != nullptr, NEST_ERR_INVALID,
               "clustered schedule needs max_micro_batches > 1");
    NEST_CUDA(cudaStreamWaitEvent(S(stream), c->ev_scratch, 0));
    {
      ProfScope ps(*c, ST_SCHEDULE, SK_AUX, S(stream));
      launch_schedule(*c, keys, bag_offsets, nnz, B, N, mode, perm_out, mb_offsets_out, S(stream));
    }
    NEST_CUDA(cudaEventRecord(c->ev_scratch, S(stream)));
  });
}

nest_status_t nest_route_begin(nest_ctx_t* ctx, int32_t slot, const int64_t* keys, const int32_t* bag_offsets,
                               int64_t nnz, int32_t B, const int32_t* perm, const int32_t* mb_offsets,
                               int32_t N, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    Slot& s = slot_of(*c, slot);
    NEST_CHECK(c->route_open < 0, NEST_ERR_ORDER, "a route is already open (nest_route_end first)");
    NEST_CHECK(N >= 1 && N <= c->Nmax, NEST_ERR_INVALID, "N out of range");
    NEST_CHECK(B >= 1 && B <= c->Bcap, NEST_ERR_INVALID, "B out of range");
    NEST_CHECK(nnz >= 0 && nnz <= c->Kcap, NEST_ERR_CAPACITY, "nnz exceeds max_keys");
    NEST_CHECK(B % N == 0, NEST_ERR_DIVISIBILITY, "B mod N != 0");
    NEST_CHECK(perm != nullptr || N == 1, NEST_ERR_INVALID, "N > 1 needs perm from nest_fwp_schedule");
    NEST_CHECK(bag_offsets != nullptr && (keys != nullptr || nnz == 0), NEST_ERR_INVALID, "null batch");
    NEST_CHECK(c->W == 1 || c->connected || c->comm != nullptr, NEST_ERR_ORDER,
               "exchange windows not connected (nest_window_connect) before the first route");
    (void)mb_offsets;  // micro-batches are equal: mb_offsets[i] = i * B / N
    cudaStream_t st = S(stream);
    s.routed = false;
    // zero-copy retrieval: HBM tables; at W > 1 only with the fused early push
    // (the owner's rows then leave from the shard, refreshed by the re-push)
    s.zero_copy = c->zero_copy && c->cfg.table_location == NEST_TABLE_HBM &&
                  (c->W == 1 || (c->a2a_mode == A2A_FUSED && c->early_push == EP_SM));
    // the pipelined call order (route(t+1) inside window t, before update(t)
    // is issued): the gather will skip K(t) and the refresh supplies it
    {
      Slot& o = c->slot[1 - slot];
      s.skip_planned = c->gather_skip && o.routed && !o.updated;
    }
    // the slot's previous batch must be fully consumed (window + refresh), and
    // its write-back done before this gather reads the shard (reading Q8)
    NEST_CUDA(cudaStreamWaitEvent(st, s.ev_update, 0));
    NEST_CUDA(cudaStreamWaitEvent(st, s.ev_free, 0));
    NEST_CUDA(cudaStreamWaitEvent(st, c->ev_scratch, 0));
    c->route_pid = prof_begin(*c, ST_ROUTE, SK_AUX, st);
    route_phase_a(*c, s, keys, bag_offsets, nnz, B, perm, N, st);
    // phase A kernels (unpooled: + sample-base scan + k_unpooled_base; the
    // window count exchange: + k_push_counts; NCCL kernels are not counted)
    prof_end(*c, c->route_pid, st, 0.0, nullptr, 0.0,
             (c->cfg.pooling == NEST_POOL_SUM ? 11 : 15) + (c->W > 1 && c->route_window ? 1 : 0));
    c->route_open = slot;
    c->route_stream = st;
  });
}

nest_status_t nest_route_end(nest_ctx_t* ctx, int32_t slot) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    Slot& s = slot_of(*c, slot);
    NEST_CHECK(c->route_open == slot, NEST_ERR_ORDER, "nest_route_end without nest_route_begin on this slot");
    c->route_open = -1;
    cudaStream_t st = c->route_stream;
    const int N = s.N;
    NEST_CUDA(cudaEventSynchronize(s.ev_sync));  // the one host sync (All2All sizes)
    route_plan(*c, s);
    // the occurrence sort (needed from this batch's backward on) on the
    // library's lowest-priority stream: it overlaps phase B and the window
    // (its input is phase A's, its scratch this slot's own)
    NEST_CUDA(cudaStreamWaitEvent(c->sort_stream, s.ev_sync, 0));
    route_sort(*c, s, c->sort_stream);
    NEST_CUDA(cudaEventRecord(s.ev_sorted, c->sort_stream));
    route_phase_b(*c, s, st);
    // 12 K + 8 U_s (keys + inverse + uniq)
    prof_add_bytes(*c, c->route_pid, 12.0 * double(s.info.nnz) + 8.0 * double(s.info.uniq));
    s.routed = true;
    s.updated = false;
    s.prefetched = 0;
    s.epoch = ++c->epoch;
    s.early = s.repushed = false;
    if (c->early_push) {
      // early push: every requested row of the prefetch buffer goes to its
      // requester now, overlapping the current window; rows the current
      // window updates are re-pushed by nest_dbp_refresh
      const double row = double(c->D) * sizeof(float);
      for (int mb = 0; mb < N; ++mb) {
        const int64_t self = s.all[(size_t(c->rank) * c->W + c->rank) * (c->Nmax + 2) + 1 + mb];
        if (c->early_push == EP_CE) {
          // send rows gathered locally, then copy-engine DMA per requester
          // (no SM time while the window's kernels run)
          {
            ProfScope ps(*c, ST_SEND_GATHER, SK_AUX, st);
            launch_send_gather(*c, s, mb, st, c->send_stage);
            ps.bytes = 2.0 * row * double(s.info.mb_recv[mb]) + 12.0 * double(s.info.recv);
          }
          ProfScope ps(*c, ST_EMB_A2A, SK_AUX, st);
          xfer_push_emb(*c, s, mb, st, s.ev_emb[mb], c->send_stage);   // signals XK_EMB
          ps.launches = 0;
          ps.bytes = row * double(s.info.mb_recv[mb] - self);  // rows sent off-GPU
          ps.hbm = row * double(s.info.mb_recv[mb] + self);    // staged rows read + self rows stored
        } else {
          ProfScope ps(*c, ST_EMB_A2A, SK_AUX, st);
          // the rows of the pending update's keys are left to the re-push
          launch_send_push(*c, s, mb, st, s.refresh_pending ? c->slot[1 - slot].obm : nullptr);
          ps.dcount = c->n_refreshed + 1;   // rows sent off-GPU (counted on the device)
          ps.bpc = row;
          ps.hbm = row * double(s.info.mb_recv[mb] + self);    // rows gathered + rows stored locally
          xfer_signal(*c, s, XK_EMB, mb, st);
        }
      }
      NEST_CUDA(cudaEventRecord(s.ev_early, st));
      s.early = true;
      s.prefetched = (1u << N) - 1u;
    }
    // the positions last: the early push above does not need them, the
    // lookups of this batch do (ev_gather: "route complete")
    route_positions(*c, s, st);
    NEST_CUDA(cudaEventRecord(s.ev_gather, st));
    NEST_CUDA(cudaEventRecord(c->ev_scratch, st));
  });
}


nest_status_t nest_route(nest_ctx_t* ctx, int32_t slot, const int64_t* keys, const int32_t* bag_offsets,
                         int64_t nnz, int32_t B, const int32_t* perm, const int32_t* mb_offsets,
                         int32_t N, void* stream) {
  const nest_status_t st = nest_route_begin(ctx, slot, keys, bag_offsets, nnz, B, perm, mb_offsets, N, stream);
  return st != NEST_OK ? st : nest_route_end(ctx, slot);
}

nest_status_t nest_dbp_refresh(nest_ctx_t* ctx, int32_t active_slot, int32_t prefetch_slot, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(active_slot != prefetch_slot, NEST_ERR_INVALID, "slots must differ");
    Slot& a = slot_of(*c, active_slot);
    Slot& p = slot_of(*c, prefetch_slot);
    NEST_CHECK(a.routed && p.routed, NEST_ERR_ORDER, "refresh needs both slots routed");
    NEST_CHECK(a.updated, NEST_ERR_ORDER, "refresh before the active slot's update (S:276)");
    cudaStream_t st = S(stream);
    NEST_CUDA(cudaStreamWaitEvent(st, a.ev_update, 0));
    NEST_CUDA(cudaStreamWaitEvent(st, p.ev_gather, 0));
    if (p.zero_copy && c->W == 1) {
      // zero-copy batch: it reads the written-back shard itself, nothing to copy
    } else if (p.early) {
      // the requesters' early copies of the intersection are stale too: the
      // refresh re-pushes exactly those rows (after the early push landed)
      NEST_CUDA(cudaStreamWaitEvent(st, p.ev_early, 0));
      {
        ProfScope ps(*c, ST_EMB_REPUSH, SK_COMPUTE, st);
        for (int mb = 0; mb < p.N; ++mb) launch_refresh_push(*c, a, p, mb, st);
        ps.launches = p.N;   // one k_refresh_push per micro-batch
        // N4 (8 U_o' keys + 2 I rows) + the re-pushed rows (not counted: the
        // requester fan-out of I is known on the device only)
        ps.bytes = 8.0 * double(std::min(p.info.recv, c->Uocap));
        ps.dcount = c->n_refreshed;
        ps.bpc = 2.0 * c->D * sizeof(float);
      }
      for (int mb = 0; mb < p.N; ++mb) xfer_signal(*c, p, XK_REPUSH, mb, st);
      NEST_CUDA(cudaEventRecord(p.ev_repush, st));
      p.repushed = true;
    } else {
      ProfScope ps(*c, ST_REFRESH, SK_COMPUTE, st);
      launch_refresh(*c, a, p, st);
      // 8 (U_o + U_o') key reads + 2 I rows (I counted on the device)
      ps.bytes = 8.0 * double(std::min(p.info.recv, c->Uocap));  // U_o' keys + bit tests
      ps.dcount = c->n_refreshed;
      ps.bpc = 2.0 * c->D * sizeof(float);
    }
    NEST_CUDA(cudaEventRecord(a.ev_free, st));
    p.refresh_pending = false;
  });
}

nest_status_t nest_lookup_prefetch(nest_ctx_t* ctx, int32_t slot, int32_t mb, void* compute, void* comm) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    Slot& s = slot_of(*c, slot);
    NEST_CHECK(s.routed, NEST_ERR_ORDER, "prefetch before route");
    NEST_CHECK(!s.refresh_pending, NEST_ERR_ORDER,
               "dual-buffer refresh pending: nest_dbp_refresh(active, this slot) first (S:276)");
    NEST_CHECK(!s.updated, NEST_ERR_ORDER, "prefetch after the window closed (S:568)");
    NEST_CHECK(mb >= 0 && mb < s.N, NEST_ERR_INVALID, "micro-batch out of range");
    if (s.early) return;   // pushed at route time
    NEST_CHECK(!((s.prefetched >> mb) & 1u), NEST_ERR_ORDER, "micro-batch already prefetched");
    if (c->W > 1) lookup_comm(*c, s, mb, S(compute), S(comm));
  });
}

static nest_status_t lookup_fwd_impl(Ctx* c, int32_t slot, int32_t mb, void* out, bool bf16, void* compute,
                                     void* comm) {
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(!bf16 || c->cfg.pooling == NEST_POOL_SUM, NEST_ERR_INVALID, "bf16 output needs pooling = SUM");
    Slot& s = slot_of(*c, slot);
    NEST_CHECK(s.routed, NEST_ERR_ORDER, "lookup before route");
    NEST_CHECK(!s.refresh_pending, NEST_ERR_ORDER,
               "dual-buffer refresh pending: nest_dbp_refresh(active, this slot) first (S:276)");
    NEST_CHECK(!s.updated, NEST_ERR_ORDER, "lookup after the window closed (S:568)");
    NEST_CHECK(mb >= 0 && mb < s.N, NEST_ERR_INVALID, "micro-batch out of range");
    NEST_CHECK(out != nullptr, NEST_ERR_INVALID, "null out");
    cudaStream_t cs = S(compute), ms = S(comm);
    if (c->W > 1 && s.early) {
      // rows pushed at route time (+ the refresh's re-push) by every owner;
      // ev_gather: the route is complete (the positions come after the push)
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_gather, 0));
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_early, 0));
      xfer_wait_emb(*c, s, mb, cs, XK_EMB);
      if (s.repushed) {
        NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_repush, 0));
        xfer_wait_emb(*c, s, mb, cs, XK_REPUSH);
      }
    } else if (c->W > 1) {
      if (!((s.prefetched >> mb) & 1u)) lookup_comm(*c, s, mb, cs, ms);
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_emb[mb], 0));
      if (c->xfer_ce) xfer_wait_emb(*c, s, mb, cs);   // every owner's rows have landed
    } else if (mb == 0) {
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_gather, 0));
      if (s.zero_copy) {
        // the shard is read in place: after the other slot's update (DBP's
        // staleness-freedom without a buffer, reading Q8)
        Slot& o = c->slot[1 - slot];
        NEST_CHECK(!o.routed || o.updated, NEST_ERR_ORDER,
                   "zero-copy lookup before the previous window's update was issued");
        if (o.routed) NEST_CUDA(cudaStreamWaitEvent(cs, o.ev_update, 0));
      }
    }
    ProfScope ps(*c, ST_POOL, SK_COMPUTE, cs);
    launch_pool(*c, s, mb, out, bf16, cs);
    {
      // U_{s,i} rows + 4 K_i + output rows
      const double row = double(c->D) * sizeof(float);
      ps.bytes = row * double(s.info.mb_uniq[mb]) + 4.0 * double(s.info.mb_nnz[mb]) +
                 (bf16 ? 0.5 : 1.0) * row * double(s.info.mb_out_rows[mb]);
    }
  });
}

nest_status_t nest_lookup_fwd(nest_ctx_t* ctx, int32_t slot, int32_t mb, float* out, void* compute,
                              void* comm) {
  return lookup_fwd_impl(reinterpret_cast<Ctx*>(ctx), slot, mb, out, false, compute, comm);
}

nest_status_t nest_lookup_fwd_bf16(nest_ctx_t* ctx, int32_t slot, int32_t mb, void* out, void* compute,
                                   void* comm) {
  return lookup_fwd_impl(reinterpret_cast<Ctx*>(ctx), slot, mb, out, true, compute, comm);
}

static nest_status_t grad_impl(Ctx* c, int32_t slot, int32_t mb, const float* dout, const OptStep& opt,
                               void* compute, void* comm) {
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(opt.kind == c->cfg.optimizer, NEST_ERR_INVALID,
               "update call does not match the context's optimizer (nest_grad_bwd_update: SGD, "
               "nest_grad_bwd_update_adagrad: row-wise AdaGrad)");
    Slot& s = slot_of(*c, slot);
    NEST_CHECK(s.routed && !s.updated, NEST_ERR_ORDER, "backward outside the window");
    NEST_CHECK(mb >= 0 && mb < s.N, NEST_ERR_INVALID, "micro-batch out of range");
    NEST_CHECK(dout != nullptr || s.info.mb_out_rows[mb] == 0, NEST_ERR_INVALID, "null dout");
    cudaStream_t cs = S(compute), ms = S(comm);
    const double row = double(c->D) * sizeof(float);
    if (mb == 0) {
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_sorted, 0));   // segment-sum input
      NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_gather, 0));   // ... and the key positions
    }
    if (c->W == 1 && s.N == 1) {
      // one rank, one micro-batch: the segment-sum applies Eq. 2 itself (the
      // next slot's gather skipped this slot's rows: no ordering with it,
      // unless NEST_GATHER_SKIP=0)
      if (!c->gather_skip) NEST_CUDA(cudaStreamWaitEvent(cs, c->slot[1 - slot].ev_gather, 0));
      {
        ProfScope ps(*c, ST_SEGSUM, SK_COMPUTE, cs);
        launch_segsum_sgd(*c, s, dout, opt, cs);
        ps.launches = s.info.mb_uniq[0] > 0 ? segsum_launches(*c) : 0;
        // N7 + N8 without the gradient-row round trip: gradient rows read +
        // 4 K + frozen rows read + rows written back
        ps.bytes = row * double(s.info.mb_out_rows[0]) + 4.0 * double(s.info.mb_nnz[0]) +
                   2.0 * row * double(s.info.mb_uniq[0]) +
                   (opt.kind == NEST_OPT_ROWWISE_ADAGRAD ? 8.0 * double(s.info.mb_uniq[0]) : 0.0);
      }
      NEST_CUDA(cudaEventRecord(s.ev_update, cs));
      s.updated = true;
      return;
    }
    const bool fused = c->a2a_mode == A2A_FUSED && !c->grad_ce;
    {
      ProfScope ps(*c, fused ? ST_GRAD_A2A : ST_SEGSUM, SK_COMPUTE, cs);
      if (fused) {
        // R10 + R11 in one pass: each key's gradient row is stored straight
        // into its owner's receive rows (peer memory over NVLink)
        const int W = c->W, Nc = c->Nmax + 2;
        PeerRows out{};
        int64_t acc = 0;
        for (int o = 0; o < W; ++o) {   // owner-major positions of the micro-batch's keys
          int64_t dst = own_base_at(s, *c, o, mb);
          for (int r = 0; r < c->rank; ++r) dst += s.all[(size_t(r) * W + o) * Nc + 1 + mb];
          out.base[o] = c->peer_own[o] + dst * c->D;
          out.off[o] = int32_t(acc);
          acc += s.all[(size_t(c->rank) * W + o) * Nc + 1 + mb];
        }
        out.off[W] = int32_t(acc);
        out.n = W;
        out.fence = 1;
        if (dwb_active(*c, s, opt)) {
          // direct write-back: the owners marked the sole-contributor rows
          out.dwb_rows = dwb_of(*c, s) + s.src_base[mb];
          out.sgd_buffer = src_rows_of(*c, s) + s.src_base[mb] * c->D;
          out.sgd_lr = opt.lr;
          for (int o = 0; o < W; ++o) out.dwb_shard[o] = c->peer_shard[o];
        }
        launch_segsum_to(*c, s, mb, dout, out, cs);
        xfer_signal(*c, s, 1, mb, cs);
      } else {
        launch_segsum(*c, s, mb, dout, cs);
      }
      ps.launches = s.info.mb_uniq[mb] > 0 ? segsum_launches(*c) : 0;
      if (fused) {
        // accounted as the gradient All2All: rows stored off-GPU
        const int64_t self = s.all[(size_t(c->rank) * c->W + c->rank) * (c->Nmax + 2) + 1 + mb];
        ps.bytes = row * double(s.info.mb_uniq[mb] - self);
        // local HBM: the segment-sum's reads (N7: gradient rows + 4 K_i) + rows stored locally
        ps.hbm = row * double(s.info.mb_out_rows[mb]) + 4.0 * double(s.info.mb_nnz[mb]) + row * double(self);
      } else {
        // gradient rows read + 4 K_i + U_{s,i} rows written
        ps.bytes = row * double(s.info.mb_out_rows[mb]) + 4.0 * double(s.info.mb_nnz[mb]) +
                   row * double(s.info.mb_uniq[mb]);
      }
    }
    // SURVEY §8(d) N8 (the update below): sum_i R_{o,i} gradient rows + U_o
    // buffer rows read + U_o rows written back (the survey's third U_o row, the
    // buffer rewrite, is not needed: the refresh copies written-back rows,
    // DESIGN.md §7) -- counted on the device as moved
    if (c->W > 1) {
      NEST_CUDA(cudaEventRecord(s.ev_grad[mb], cs));
      NEST_CUDA(cudaStreamWaitEvent(ms, s.ev_grad[mb], 0));
      std::vector<int64_t> scnt(c->W), rcnt(c->W);
      const int Nc = c->Nmax + 2;
      for (int p = 0; p < c->W; ++p) {
        scnt[p] = s.all[(size_t(c->rank) * c->W + p) * Nc + 1 + mb];  // requester -> owner p
        rcnt[p] = s.all[(size_t(p) * c->W + c->rank) * Nc + 1 + mb];  // from requester p
      }
      if (!fused) {
        ProfScope ps(*c, ST_GRAD_A2A, SK_COMM, ms);
        if (c->xfer_ce)
          xfer_push_grad(*c, s, mb, ms);
        else
          a2a_rows(*c, c->src_rows + s.src_base[mb] * c->D, scnt, c->own_rows + s.own_base[mb] * c->D, rcnt, ms);
        ps.launches = 0;
        ps.bytes = row * double(s.info.mb_uniq[mb] - scnt[c->rank]);  // rows sent off-GPU
        ps.hbm = row * double(s.info.mb_uniq[mb] + scnt[c->rank]);    // rows read + self rows stored
      }
      if (mb == s.N - 1) {
        if (c->xfer_ce) xfer_wait_grads(*c, s, ms);  // every requester's gradients have landed
        if (!c->gather_skip) NEST_CUDA(cudaStreamWaitEvent(ms, c->slot[1 - slot].ev_gather, 0));
        {
          ProfScope ps(*c, ST_UPDATE, SK_COMM, ms);
          launch_reduce_sgd(*c, s, opt, ms);
          // N8 as moved: contributions read + frozen row read + row written
          // (counted on the device; under direct write-back the sole
          // contributors' keys are not touched here), + AdaGrad's accumulator
          ps.bytes = opt.kind == NEST_OPT_ROWWISE_ADAGRAD ? 8.0 * double(std::min(s.info.recv, c->Uocap)) : 0.0;
          ps.dcount = c->n_refreshed + 3;
          ps.bpc = row;
        }
        NEST_CUDA(cudaEventRecord(s.ev_update, ms));
        NEST_CUDA(cudaStreamWaitEvent(cs, s.ev_update, 0));
      }
    } else if (mb == s.N - 1) {
      if (!c->gather_skip) NEST_CUDA(cudaStreamWaitEvent(cs, c->slot[1 - slot].ev_gather, 0));
      {
        ProfScope ps(*c, ST_UPDATE, SK_COMPUTE, cs);
        launch_reduce_sgd(*c, s, opt, cs);
        ps.bytes = opt.kind == NEST_OPT_ROWWISE_ADAGRAD ? 8.0 * double(std::min(s.info.recv, c->Uocap)) : 0.0;
        ps.dcount = c->n_refreshed + 3;   // rows moved (N8), counted on the device
        ps.bpc = row;
      }
      NEST_CUDA(cudaEventRecord(s.ev_update, cs));
    }
    if (mb == s.N - 1) s.updated = true;
  });
}

nest_status_t nest_grad_bwd_update(nest_ctx_t* ctx, int32_t slot, int32_t mb, const float* dout,
                                   float lr_over_B, void* compute, void* comm) {
  const OptStep opt{NEST_OPT_SGD, lr_over_B, 1.f, 0.f, nullptr};
  return grad_impl(reinterpret_cast<Ctx*>(ctx), slot, mb, dout, opt, compute, comm);
}

nest_status_t nest_grad_bwd_update_adagrad(nest_ctx_t* ctx, int32_t slot, int32_t mb, const float* dout,
                                           float grad_scale, float lr, void* compute, void* comm) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  const OptStep opt{NEST_OPT_ROWWISE_ADAGRAD, lr, grad_scale, c->cfg.adagrad_eps, c->opt_state};
  return grad_impl(c, slot, mb, dout, opt, compute, comm);
}

static nest_status_t tower_impl(Ctx* c, const void* pooled, bool bf16, int64_t rows, float* dout, void* stream) {
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(c->tower != nullptr, NEST_ERR_INVALID, "tower_layers == 0");
    NEST_CHECK(rows % c->F == 0, NEST_ERR_INVALID, "rows must be a multiple of F");
    NEST_CHECK(pooled != nullptr && dout != nullptr, NEST_ERR_INVALID, "null pooled / dout");
    ProfScope ps(*c, ST_TOWER, SK_COMPUTE, S(stream));
    ps.bytes = tower_run(*c, pooled, bf16, rows, dout, S(stream));  // FLOPs on this stream
    ps.launches = bf16 ? 0 : 1;  // the cast kernel (the GEMMs are cuBLAS)
  });
}

nest_status_t nest_tower_fwd_bwd(nest_ctx_t* ctx, const float* pooled, int64_t rows, float* dout,
                                 void* stream) {
  return tower_impl(reinterpret_cast<Ctx*>(ctx), pooled, false, rows, dout, stream);
}

nest_status_t nest_tower_fwd_bwd_bf16(nest_ctx_t* ctx, const void* pooled, int64_t rows, float* dout,
                                      void* stream) {
  return tower_impl(reinterpret_cast<Ctx*>(ctx), pooled, true, rows, dout, stream);
}

nest_status_t nest_tower_read(nest_ctx_t* ctx, int32_t what, int32_t layer, float* out, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] { tower_read(*c, what, layer, out, S(stream)); });
}

nest_status_t nest_set_zero_copy(nest_ctx_t* ctx, int32_t on) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] { c->zero_copy = on != 0; });
}

nest_status_t nest_set_streams(nest_ctx_t* ctx, void* sort_stream, void* tower_dw_stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CUDA(cudaDeviceSynchronize());
    if (sort_stream) {
      if (c->sort_stream_owned) NEST_CUDA(cudaStreamDestroy(c->sort_stream));
      c->sort_stream = S(sort_stream);
      c->sort_stream_owned = false;
    }
    if (tower_dw_stream) tower_set_side(*c, S(tower_dw_stream));
  });
}

nest_status_t nest_tower_step(nest_ctx_t* ctx, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] { tower_step(*c, S(stream)); });
}

nest_status_t nest_join(nest_ctx_t* ctx, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    tower_join(*c, S(stream));
    // ... and the occurrence sorts on the library's sort stream
    NEST_CUDA(cudaEventRecord(c->ev_sort_join, c->sort_stream));
    NEST_CUDA(cudaStreamWaitEvent(S(stream), c->ev_sort_join, 0));
  });
}

nest_status_t nest_slot_info(const nest_ctx_t* ctx, int32_t slot, nest_slot_info_t* info) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !info || (slot != 0 && slot != 1)) return NEST_ERR_INVALID;
  *info = c->slot[slot].info;
  info->valid = c->slot[slot].routed ? 1 : 0;
  return NEST_OK;
}

nest_status_t nest_route_view(const nest_ctx_t* ctx, int32_t slot, nest_route_view_t* v) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !v || (slot != 0 && slot != 1)) return NEST_ERR_INVALID;
  const Slot& s = c->slot[slot];
  v->uniq = s.uniq;
  v->inverse = s.inverse;
  v->mask = s.mask;
  v->pos = s.pos;
  v->send_counts = s.xfer + int64_t(c->rank) * c->W * (c->Nmax + 2);
  v->all_counts = s.xfer;
  v->recv_keys = s.recv;
  v->owner_rows = s.owner_rows;
  v->owner_inv = s.owner_inv;
  v->n_owner = s.n_owner;
  v->buffer = s.buffer;
  return NEST_OK;
}

nest_status_t nest_read_rows(nest_ctx_t* ctx, const int64_t* keys, int64_t n, float* out, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(n >= 0 && (n == 0 || (keys && out)), NEST_ERR_INVALID, "bad arguments");
    launch_read_rows(*c, keys, n, out, S(stream));
  });
}

nest_status_t nest_read_state(nest_ctx_t* ctx, const int64_t* keys, int64_t n, float* out, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] {
    NEST_CHECK(c->opt_state != nullptr, NEST_ERR_INVALID, "no optimizer state (SGD context)");
    NEST_CHECK(n >= 0 && (n == 0 || (keys && out)), NEST_ERR_INVALID, "bad arguments");
    launch_read_state(*c, keys, n, out, S(stream));
  });
}

nest_status_t nest_exchange_plan(const nest_config_t* cfg, int32_t N, const int32_t* all_counts,
                                 nest_exchange_plan_t* plan) {
  return guard(nullptr, [&] {
    NEST_CHECK(all_counts && plan, NEST_ERR_INVALID, "null argument");
    Ctx c;
    derive(c, cfg);
    exchange_plan(c, N, all_counts, *plan);
  });
}

nest_status_t nest_profile_enable(nest_ctx_t* ctx, int32_t on) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] { profile_enable(*c, on != 0); });
}

nest_status_t nest_profile_read(nest_ctx_t* ctx, nest_profile_stage_t* stages,
                                nest_profile_summary_t* summary) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return NEST_ERR_INVALID;
  return guard(c, [&] { profile_read(*c, stages, summary); });
}

nest_status_t nest_profile_records(nest_ctx_t* ctx, nest_profile_record_t* out, int64_t cap, int64_t* n) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !n) return NEST_ERR_INVALID;
  return guard(c, [&] { profile_records(*c, out, cap, n); });
}

const char* nest_last_error(const nest_ctx_t* ctx) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  return c ? c->last_error.c_str() : g_create_error.c_str();
}

}  // extern "C"
