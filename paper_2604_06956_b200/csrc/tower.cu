// Stand-in dense tower: the FWP overlap partner, NOT the product (SURVEY R9,
// BASELINE north_star "fixed stand-in dense tower (cuBLAS GEMMs)").
// A fixed L-layer bf16 MLP (identity activations) over the pooled rows of a
// micro-batch viewed as X0 = [B_i, F*d]: forward Y_l = X_{l-1} W_l^T, then a
// fixed top gradient G, backward dW_l = dY_l^T X_{l-1} and dX_{l-1} = dY_l W_l,
// with the input gradient dX_0 written as fp32 `dout`.  GEMMs run on the
// tensor cores through cuBLAS (library GEMMs, allowed for the plain tower).
// Only the dX chain feeds the embedding backward, so by default the dW GEMMs
// run on an internal low-priority stream behind it (overlapping segment-sum,
// update, refresh and the next pool); the next forward waits for them, as it
// would for a dense optimizer step (NEST_TOWER_DEFER_DW=0: all on one stream).
#include <cublasLt.h>
#include <cublas_v2.h>

#include <map>

#include "nest_internal.cuh"

namespace nest {

struct GemmPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo{};
  bool have_algo = false;
};

struct Tower {
  cublasHandle_t h = nullptr;
  cublasLtHandle_t lt = nullptr;
  int32_t sm_target = 0;
  int32_t sm_target_dw = 0;   // the weight-gradient GEMMs (the only transposed-A ones)
  std::map<std::string, struct GemmPlan> plans;
  int L = 0, H = 0, in0 = 0;
  int64_t bmax = 0;
  __nv_bfloat16* w = nullptr;       // weights, layer l at woff[l], [H, in_l] row-major
  std::vector<int64_t> woff;
  __nv_bfloat16* x = nullptr;       // activations X_0..X_{L-1}, X_l at xoff[l] (of the current buffer set)
  std::vector<int64_t> xoff;
  __nv_bfloat16* dy = nullptr;      // dY_l for l = 0..L-2 (layer l's output), [L-1][bmax, H]
  // fixed tower: two activation / dY buffer sets used by alternate calls, so
  // call k's forward overwrites the set of call k-2 and waits only for call
  // k-2's deferred dW GEMMs (they read X and dY), not for call k-1's: the dW
  // GEMMs of one batch overlap the next batch's pool and forward.  A trained
  // tower has one set (its next forward needs the updated weights anyway).
  __nv_bfloat16* xs[2] = {nullptr, nullptr};
  __nv_bfloat16* dys[2] = {nullptr, nullptr};
  int nsets = 1;
  int64_t calls = 0;
  cudaEvent_t ev_dwb[2] = {nullptr, nullptr};
  bool pend_b[2] = {false, false};
  __nv_bfloat16* dw = nullptr;      // [H, max in]
  int acc = 0;                      // micro-batches accumulated into dw32 since the last tower_step
  int64_t acc_rows = 0;             // their rows (the next call's top-gradient offset)
  __nv_bfloat16* gtop = nullptr;    // [bmax, H] fixed top gradient dY_{L-1}
  void* ws = nullptr;               // cuBLASLt workspace of the caller's stream
  void* ws_dw = nullptr;            // ... and of the dW stream
  size_t ws_bytes = 32u << 20;
  bool defer_dw = true;
  cudaStream_t side = nullptr;      // dW GEMMs
  bool side_owned = true;           // false: the caller's stream (nest_set_streams)
  cudaEvent_t ev_dx = nullptr, ev_dw = nullptr;
  bool dw_pending = false;
  char* mem = nullptr;
  // trained tower (NEXT-4): fp32 master weights, per-layer fp32 dW, the dense
  // gradient AllReduce communicator (split from the window's, W > 1)
  bool train = false;
  float lr = 0.f;
  float* w32 = nullptr;
  float* dw32 = nullptr;
  ncclComm_t comm = nullptr;
};

#define NEST_CUBLAS(call)                                                                 \
  do {                                                                                    \
    cublasStatus_t s_ = (call);                                                           \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                      \
      throw ::nest::Error{NEST_ERR_CUDA, std::string(#call) + ": cublas status " + std::to_string(int(s_))}; \
  } while (0)

size_t tower_workspace_bytes(const Ctx& c) {
  const int L = c.cfg.tower_layers, H = c.cfg.tower_hidden;
  if (L <= 0) return 0;
  const int64_t in0 = int64_t(c.F) * c.D, bmax = c.Bcap;
  const int sets = c.cfg.tower_train ? 1 : 2;          // activation / dY buffer sets
  int64_t elems = H * in0 + int64_t(L - 1) * H * H;   // weights
  elems += sets * (bmax * in0 + int64_t(L - 1) * bmax * H);   // activations
  elems += sets * int64_t(std::max(L - 1, 1)) * bmax * H;     // dY of layers 0..L-2 (>= 1: forward scratch)
  elems += int64_t(H) * std::max<int64_t>(H, in0);   // dw
  elems += bmax * H;                                 // top gradient
  const int64_t wel = H * in0 + int64_t(L - 1) * H * H;
  const size_t train = c.cfg.tower_train ? size_t(wel) * 2 * sizeof(float) + 256 : 0;  // w32 + dw32
  return size_t(elems) * 2 + 2 * (32u << 20) + 8 * 256 + train;
}

void tower_bind(Ctx& c, char* mem) {
  if (!mem) return;
  Tower* t = new Tower();
  t->mem = mem;
  c.tower = t;
}

__global__ void k_fill_bf16(__nv_bfloat16* p, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * uint64_t(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const float u = float(uint32_t(z >> 40)) * 5.9604644775390625e-08f;  // [0,1)
    p[i] = __float2bfloat16((2.f * u - 1.f) * scale);
  }
}

__global__ void k_widen_bf16(const __nv_bfloat16* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __bfloat162float(in[i]);
}

// trained tower: w32 -= lr * dW (summed over ranks), bf16 copy for the GEMMs
__global__ void k_dense_sgd(float* __restrict__ w32, __nv_bfloat16* __restrict__ w16,
                            const float* __restrict__ dw, int64_t n, float lr) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float v = __fmaf_rn(-lr, dw[i], w32[i]);
    w32[i] = v;
    w16[i] = __float2bfloat16_rn(v);
  }
}

__global__ void k_cast_bf16(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n4) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<__nv_bfloat162*>(out)[2 * i] = a;
    reinterpret_cast<__nv_bfloat162*>(out)[2 * i + 1] = b;
  }
}

void tower_create(Ctx& c) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  NEST_CHECK(t != nullptr, NEST_ERR_INVALID, "tower memory not bound");
  t->L = c.cfg.tower_layers;
  t->H = c.cfg.tower_hidden;
  NEST_CHECK(t->H >= 16 && t->H % 16 == 0, NEST_ERR_INVALID, "tower_hidden must be a positive multiple of 16");
  t->in0 = c.F * c.D;
  t->bmax = c.Bcap;
  Carver w{t->mem};
  const int L = t->L, H = t->H;
  const int64_t in0 = t->in0, bmax = t->bmax;
  t->woff.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) t->woff[l + 1] = t->woff[l] + int64_t(H) * (l == 0 ? in0 : H);
  t->w = w.take<__nv_bfloat16>(t->woff[L]);
  t->xoff.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) t->xoff[l + 1] = t->xoff[l] + bmax * (l == 0 ? in0 : H);
  t->nsets = c.cfg.tower_train ? 1 : 2;
  for (int b = 0; b < t->nsets; ++b) {
    t->xs[b] = w.take<__nv_bfloat16>(t->xoff[L]);
    t->dys[b] = w.take<__nv_bfloat16>(int64_t(std::max(L - 1, 1)) * bmax * H);
  }
  t->x = t->xs[0];
  t->dy = t->dys[0];
  t->dw = w.take<__nv_bfloat16>(int64_t(H) * std::max<int64_t>(H, in0));
  t->gtop = w.take<__nv_bfloat16>(bmax * H);
  t->ws = w.take<char>(int64_t(t->ws_bytes));
  t->ws_dw = w.take<char>(int64_t(t->ws_bytes));
  t->train = c.cfg.tower_train != 0;
  t->lr = c.cfg.tower_lr;
  if (t->train) {
    t->w32 = w.take<float>(t->woff[L]);
    t->dw32 = w.take<float>(t->woff[L]);
    if (c.W > 1 && c.comm) NEST_NCCL(ncclCommSplit(c.comm, 0, c.rank, &t->comm, nullptr));
    // without NCCL the dense AllReduce runs through the exchange window
    NEST_CHECK(c.W == 1 || c.comm || c.twr, NEST_ERR_INVALID, "trained tower at world > 1 needs NCCL or a window");
  }
  {
    const char* dv = std::getenv("NEST_TOWER_DEFER_DW");
    t->defer_dw = !(dv && std::atoi(dv) == 0);
    int lo = 0, hi = 0;
    NEST_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    NEST_CUDA(cudaStreamCreateWithPriority(&t->side, cudaStreamNonBlocking, lo));   // lowest priority
    NEST_CUDA(cudaEventCreateWithFlags(&t->ev_dx, cudaEventDisableTiming));
    NEST_CUDA(cudaEventCreateWithFlags(&t->ev_dw, cudaEventDisableTiming));
    for (auto& e : t->ev_dwb) NEST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  NEST_CUBLAS(cublasCreate(&t->h));
  NEST_CUBLAS(cublasSetWorkspace(t->h, t->ws, t->ws_bytes));
  NEST_CUBLAS(cublasSetMathMode(t->h, CUBLAS_DEFAULT_MATH));
  // SMs left to the embedding lane (pool / segment-sum / send gather) and the
  // DBP lookahead that run beside the tower: NEST_TOWER_SM_RESERVE,
  // default 24.  W=1 E+T is within noise for 0 / 12 / 24 (19.4-20.3 M
  // samples/s); at W=4, reserve 0 measured 50.6 vs 54.2 M samples/s
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* rv = std::getenv("NEST_TOWER_SM_RESERVE");
    const int reserve = rv ? std::atoi(rv) : 24;
    if (reserve > 0 && reserve < sms) {
      NEST_CUBLAS(cublasSetSmCountTarget(t->h, sms - reserve));
      t->sm_target = sms - reserve;
    }
    // the deferred dW GEMMs run beside the segment-sum, refresh and the next
    // pool: NEST_TOWER_DW_SM_RESERVE (default: the same reserve)
    const char* rd = std::getenv("NEST_TOWER_DW_SM_RESERVE");
    const int reserve_dw = rd ? std::atoi(rd) : reserve;
    t->sm_target_dw = reserve_dw > 0 && reserve_dw < sms ? sms - reserve_dw : 0;
  }
  NEST_CUBLAS(cublasLtCreate(&t->lt));
  for (int l = 0; l < L; ++l) {
    const int64_t fan_in = l == 0 ? in0 : H;
    k_fill_bf16<<<1024, 256>>>(t->w + t->woff[l], int64_t(H) * fan_in, 1000 + l, 1.f / std::sqrt(float(fan_in)));
  }
  k_fill_bf16<<<1024, 256>>>(t->gtop, bmax * H, 77, 1.f / 1024.f);
  if (t->train) k_widen_bf16<<<1024, 256>>>(t->w, t->w32, t->woff[L]);
  NEST_LAUNCH_CHECK();
  NEST_CUDA(cudaDeviceSynchronize());
}

void tower_destroy(Ctx& c) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  if (!t) return;
  if (t->h) cublasDestroy(t->h);
  if (t->comm) ncclCommDestroy(t->comm);
  if (t->side) {
    cudaStreamSynchronize(t->side);
    if (t->side_owned) cudaStreamDestroy(t->side);
  }
  if (t->ev_dx) cudaEventDestroy(t->ev_dx);
  if (t->ev_dw) cudaEventDestroy(t->ev_dw);
  for (auto e : t->ev_dwb)
    if (e) cudaEventDestroy(e);
  for (auto& kv : t->plans) {
    cublasLtMatmulDescDestroy(kv.second.op);
    cublasLtMatrixLayoutDestroy(kv.second.a);
    cublasLtMatrixLayoutDestroy(kv.second.b);
    cublasLtMatrixLayoutDestroy(kv.second.c);
  }
  if (t->lt) cublasLtDestroy(t->lt);
  delete t;
  c.tower = nullptr;
}

// row-major C[M,N] = op(A)[M,K] * op(B)[K,N] through cublasLt.  The first call
// of every shape times the top heuristic algorithms on the real buffers and
// keeps the fastest (one-time autotune; the bench's warm-up absorbs it).

static GemmPlan& plan_for(Tower* t, bool ta, bool tb, int M, int N, int K, int lda, int ldb, int ldc,
                          cudaDataType ctype) {
  const std::string key = std::to_string(ta) + "," + std::to_string(tb) + "," + std::to_string(M) + "," +
                          std::to_string(N) + "," + std::to_string(K) + "," + std::to_string(int(ctype));
  auto it = t->plans.find(key);
  if (it != t->plans.end()) return it->second;
  GemmPlan p;
  NEST_CUBLAS(cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  // column-major view: C^T[N,M] = op(B)^T[N,K] * op(A)^T[K,M]
  const cublasOperation_t oa = tb ? CUBLAS_OP_T : CUBLAS_OP_N, ob = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
  NEST_CUBLAS(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &oa, sizeof(oa)));
  NEST_CUBLAS(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &ob, sizeof(ob)));
  // (ta: the dW GEMMs dY^T X are the only ones with a transposed A)
  const int32_t target = ta ? t->sm_target_dw : t->sm_target;
  if (target > 0)
    NEST_CUBLAS(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_SM_COUNT_TARGET, &target,
                                               sizeof(target)));
  NEST_CUBLAS(cublasLtMatrixLayoutCreate(&p.a, CUDA_R_16BF, oa == CUBLAS_OP_N ? N : K, oa == CUBLAS_OP_N ? K : N, ldb));
  NEST_CUBLAS(cublasLtMatrixLayoutCreate(&p.b, CUDA_R_16BF, ob == CUBLAS_OP_N ? K : M, ob == CUBLAS_OP_N ? M : K, lda));
  NEST_CUBLAS(cublasLtMatrixLayoutCreate(&p.c, ctype, N, M, ldc));
  return t->plans.emplace(key, p).first->second;
}

static void gemm_rm(Tower* t, bool ta, bool tb, int M, int N, int K, const void* A, int lda,
                    const void* B, int ldb, void* C, int ldc, cudaDataType ctype, cudaStream_t st,
                    void* ws, float beta = 0.f) {
  const float alpha = 1.f;
  GemmPlan& p = plan_for(t, ta, tb, M, N, K, lda, ldb, ldc, ctype);
  if (!p.have_algo) {
    cublasLtMatmulPreference_t pref;
    NEST_CUBLAS(cublasLtMatmulPreferenceCreate(&pref));
    NEST_CUBLAS(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &t->ws_bytes,
                                                     sizeof(t->ws_bytes)));
    cublasLtMatmulHeuristicResult_t res[8];
    int n = 0;
    NEST_CUBLAS(cublasLtMatmulAlgoGetHeuristic(t->lt, p.op, p.a, p.b, p.c, p.c, pref, 8, res, &n));
    cublasLtMatmulPreferenceDestroy(pref);
    NEST_CHECK(n > 0, NEST_ERR_CUDA, "no cublasLt algorithm for a tower GEMM");
    // timing runs overwrite C (beta 0); an accumulating call (beta 1) saves C
    // first and restores it after tuning
    const float tune_beta = 0.f;
    void* saved = nullptr;
    const size_t cbytes = size_t(M) * ldc * (ctype == CUDA_R_32F ? 4 : 2);
    if (beta != 0.f) {
      NEST_CUDA(cudaMallocAsync(&saved, cbytes, st));
      NEST_CUDA(cudaMemcpyAsync(saved, C, cbytes, cudaMemcpyDeviceToDevice, st));
    }
    cudaEvent_t e0, e1;
    NEST_CUDA(cudaEventCreate(&e0));
    NEST_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    int bi = 0;
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      bool ok = true;
      for (int rep = 0; rep < 3 && ok; ++rep) {  // warm + 2 timed
        if (rep == 1) cudaEventRecord(e0, st);
        ok = cublasLtMatmul(t->lt, p.op, &alpha, B, p.a, A, p.b, &tune_beta, C, p.c, C, p.c, &res[i].algo, ws,
                            t->ws_bytes, st) == CUBLAS_STATUS_SUCCESS;
      }
      if (!ok) continue;
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) {
        best = ms;
        bi = i;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    NEST_CHECK(best < 1e29f, NEST_ERR_CUDA, "no working cublasLt algorithm for a tower GEMM");
    if (saved) {
      NEST_CUDA(cudaMemcpyAsync(C, saved, cbytes, cudaMemcpyDeviceToDevice, st));
      NEST_CUDA(cudaFreeAsync(saved, st));
    }
    p.algo = res[bi].algo;
    p.have_algo = true;
  }
  NEST_CUBLAS(cublasLtMatmul(t->lt, p.op, &alpha, B, p.a, A, p.b, &beta, C, p.c, C, p.c, &p.algo, ws,
                             t->ws_bytes, st));
}

double tower_run(Ctx& c, const void* pooled, bool pooled_bf16, int64_t rows, float* dout, cudaStream_t st) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  const int64_t bm = rows / c.F;
  if (bm == 0) return 0.0;
  NEST_CHECK(bm <= t->bmax, NEST_ERR_CAPACITY, "tower batch exceeds max_batch");
  const int L = t->L, H = t->H, in0 = t->in0, M = int(bm);
  // buffer set of this call; its previous user's dW GEMMs still read X and dY
  // (trained tower: one set, and the next forward also needs the updated weights)
  const int bset = int(t->calls % t->nsets);
  ++t->calls;
  t->x = t->xs[bset];
  t->dy = t->dys[bset];
  if (t->nsets == 1) {
    if (t->dw_pending) NEST_CUDA(cudaStreamWaitEvent(st, t->ev_dw, 0));
    t->dw_pending = false;
  } else if (t->pend_b[bset]) {
    NEST_CUDA(cudaStreamWaitEvent(st, t->ev_dwb[bset], 0));
    t->pend_b[bset] = false;
  }
  // input of layer l (X_0: the caller's bf16 rows in place, or the cast copy)
  __nv_bfloat16* x0 = pooled_bf16 ? const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(pooled))
                                  : t->x;
  auto X = [&](int l) { return l == 0 ? x0 : t->x + t->xoff[l]; };
  auto W = [&](int l) { return t->w + t->woff[l]; };
  // the fixed top gradient of a row is its position in the window: a trained
  // tower's micro-batches take consecutive slices (rows accumulated since the
  // last tower_step), so N micro-batches see the same top gradient as one
  // full-batch call (sequential schedule); the fixed tower always starts at 0
  const int64_t g0 = t->train ? t->acc_rows : 0;
  NEST_CHECK(g0 + bm <= t->bmax, NEST_ERR_CAPACITY, "tower rows of one window exceed max_batch");
  auto DY = [&](int l) { return l == L - 1 ? t->gtop + g0 * H : t->dy + int64_t(l) * t->bmax * H; };
  auto IN = [&](int l) { return l == 0 ? in0 : H; };
  if (!pooled_bf16) {
    k_cast_bf16<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const float*>(pooled), t->x, bm * in0 / 4);
    NEST_LAUNCH_CHECK();
  }
  // forward: X_{l+1} = X_l W_l^T (the last layer's output is not needed:
  // its gradient is the fixed gtop); the scratch dY_0 takes it
  for (int l = 0; l < L; ++l)
    gemm_rm(t, false, true, M, H, IN(l), X(l), IN(l), W(l), IN(l), l + 1 < L ? X(l + 1) : t->dy, H, CUDA_R_16BF,
            st, t->ws);
  // backward, input-gradient chain: dY_{l-1} = dY_l W_l, dX_0 = dY_0 W_0 (fp32)
  for (int l = L - 1; l >= 1; --l)
    gemm_rm(t, false, false, M, H, H, DY(l), H, W(l), H, DY(l - 1), H, CUDA_R_16BF, st, t->ws);
  gemm_rm(t, false, false, M, in0, H, DY(0), H, W(0), in0, dout, in0, CUDA_R_32F, st, t->ws);
  // weight gradients dW_l = dY_l^T X_l
  cudaStream_t ws = st;
  if (t->defer_dw) {
    NEST_CUDA(cudaEventRecord(t->ev_dx, st));
    NEST_CUDA(cudaStreamWaitEvent(t->side, t->ev_dx, 0));
    ws = t->side;
  }
  const double flops_dw = 2.0 * M * (double(in0) * H + double(L - 1) * H * H);
  {
    ProfScope ps(c, ST_TOWER_DW, SK_AUX, ws);
    // trained tower: the micro-batches of one window accumulate into the fp32
    // dW (beta 0 on the first, 1 after: one gradient per batch, Prop. 2 /
    // Corollary 1 -- every micro-batch sees the same frozen weights); the
    // AllReduce + SGD run once, in tower_step after the window's last tower call
    const float beta = t->acc > 0 ? 1.f : 0.f;
    for (int l = L - 1; l >= 0; --l) {
      if (t->train)   // fp32 dW of every layer, kept for the AllReduce + update
        gemm_rm(t, true, false, H, IN(l), M, DY(l), H, X(l), IN(l), t->dw32 + t->woff[l], IN(l), CUDA_R_32F,
                ws, t->defer_dw ? t->ws_dw : t->ws, beta);
      else
        gemm_rm(t, true, false, H, IN(l), M, DY(l), H, X(l), IN(l), t->dw, IN(l), CUDA_R_16BF, ws,
                t->defer_dw ? t->ws_dw : t->ws);
    }
    if (t->train) {
      ++t->acc;
      t->acc_rows += bm;
    }
    ps.bytes = flops_dw;
    ps.launches = 0;
  }
  if (t->defer_dw) {
    NEST_CUDA(cudaEventRecord(t->ev_dw, t->side));
    t->dw_pending = true;
    NEST_CUDA(cudaEventRecord(t->ev_dwb[bset], t->side));
    t->pend_b[bset] = true;
  }
  return t->defer_dw ? 2.0 * flops_dw : 3.0 * flops_dw;   // FLOPs on `st` (fwd + dX [+ dW])
}

// window AllReduce of the trained tower's dW (no NCCL): chunk p of this
// rank's dW goes to rank p's partial area at row `me`; rank p sums the W
// partial chunks in rank order and stores the sum into every rank's sum area
struct PeerF32 {
  float* p[NEST_MAX_WORLD];
};
__global__ void k_twr_push_rs(const float* __restrict__ dw, int64_t n, int64_t chunk, int me, PeerF32 part) {
  const int p = blockIdx.y;
  float* dst = part.p[p] + int64_t(me) * chunk;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < chunk; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = int64_t(p) * chunk + j;
    dst[j] = g < n ? dw[g] : 0.f;
  }
  __threadfence_system();
}
__global__ void k_twr_reduce_ag(const float* __restrict__ part, int64_t chunk, int W, int me, PeerF32 sum) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < chunk; j += int64_t(gridDim.x) * blockDim.x) {
    float a = 0.f;
    for (int r = 0; r < W; ++r) a += part[int64_t(r) * chunk + j];
    for (int p = 0; p < W; ++p) sum.p[p][int64_t(me) * chunk + j] = a;
  }
  __threadfence_system();
}

// NEXT-4 update, once per batch after its last micro-batch: dense gradients
// summed over the data-parallel ranks (the paper's communication-side
// AllReduce) and SGD on the fp32 master weights + their bf16 copy,
// on the dW stream behind the accumulated dW GEMMs; the next tower call waits
// for it.  No-op for the fixed tower or when nothing was accumulated.
void tower_step(Ctx& c, cudaStream_t st) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  NEST_CHECK(t != nullptr, NEST_ERR_INVALID, "no tower (tower_layers == 0)");
  if (!t->train || t->acc == 0) return;
  cudaStream_t ws = st;
  if (t->defer_dw) {
    // behind the accumulated dW GEMMs on the side stream (ev_dw) and the caller's work
    NEST_CUDA(cudaEventRecord(t->ev_dx, st));
    NEST_CUDA(cudaStreamWaitEvent(t->side, t->ev_dx, 0));
    ws = t->side;
  }
  const int64_t n = t->woff[t->L];
  if (t->comm) {
    NEST_NCCL(ncclAllReduce(t->dw32, t->dw32, size_t(n), ncclFloat32, ncclSum, t->comm, ws));
    k_dense_sgd<<<148 * 4, 256, 0, ws>>>(t->w32, t->w, t->dw32, n, t->lr);
  } else if (c.W > 1) {
    // window AllReduce: reduce-scatter by peer stores (rank r sums chunk r in
    // rank order, so the sum is deterministic), all-gather of the summed
    // chunks, then the same SGD on every replica (bitwise equal replicas)
    const int W = c.W, me = c.rank;
    const int64_t chunk = c.twr_elems / W;
    NEST_CHECK(chunk * W >= n, NEST_ERR_INVALID, "tower window area too small");
    const uint32_t ep = ++c.twr_epoch;
    PeerF32 part{}, sum{};
    for (int p = 0; p < W; ++p) {
      part.p[p] = c.peer_twr[p];
      sum.p[p] = c.peer_twr[p] + c.twr_elems;
    }
    k_twr_push_rs<<<dim3(unsigned(std::min<int64_t>((chunk + 255) / 256, 148)), unsigned(W)), 256, 0, ws>>>(
        t->dw32, n, chunk, me, part);
    NEST_LAUNCH_CHECK();
    xfer_signal_raw(c, 0, XK_TRS, 0, ep, ws);
    xfer_wait_raw(c, 0, XK_TRS, 0, ep, ws);
    k_twr_reduce_ag<<<unsigned(std::min<int64_t>((chunk + 255) / 256, 148 * 2)), 256, 0, ws>>>(
        c.twr, chunk, W, me, sum);
    NEST_LAUNCH_CHECK();
    xfer_signal_raw(c, 0, XK_TAG, 0, ep, ws);
    xfer_wait_raw(c, 0, XK_TAG, 0, ep, ws);
    k_dense_sgd<<<148 * 4, 256, 0, ws>>>(t->w32, t->w, c.twr + c.twr_elems, n, t->lr);
  } else {
    k_dense_sgd<<<148 * 4, 256, 0, ws>>>(t->w32, t->w, t->dw32, n, t->lr);
  }
  NEST_LAUNCH_CHECK();
  t->acc = 0;
  t->acc_rows = 0;
  if (t->defer_dw) {
    NEST_CUDA(cudaEventRecord(t->ev_dw, t->side));
    t->dw_pending = true;
  }
}

void tower_read(Ctx& c, int what, int layer, float* out, cudaStream_t st) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  NEST_CHECK(t != nullptr, NEST_ERR_INVALID, "no tower (tower_layers == 0)");
  NEST_CHECK(out != nullptr, NEST_ERR_INVALID, "null out");
  if (t->dw_pending) NEST_CUDA(cudaStreamWaitEvent(st, t->ev_dw, 0));
  if (what == NEST_TOWER_WEIGHTS) {
    NEST_CHECK(layer >= 0 && layer < t->L, NEST_ERR_INVALID, "tower layer out of range");
    const int64_t n = t->woff[layer + 1] - t->woff[layer];
    if (t->train)
      NEST_CUDA(cudaMemcpyAsync(out, t->w32 + t->woff[layer], sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
    else
      k_widen_bf16<<<256, 256, 0, st>>>(t->w + t->woff[layer], out, n);
  } else if (what == NEST_TOWER_TOP_GRAD) {
    k_widen_bf16<<<256, 256, 0, st>>>(t->gtop, out, t->bmax * t->H);
  } else {
    throw Error{NEST_ERR_INVALID, "bad tower read kind"};
  }
  NEST_LAUNCH_CHECK();
}

// make `st` wait for outstanding dW GEMMs (context teardown / host reads)
// the dW GEMMs on the caller's stream instead of the library's (e.g. one of a
// green context holding the dense lane's SMs)
void tower_set_side(Ctx& c, cudaStream_t st) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  if (!t || !st) return;
  NEST_CUDA(cudaStreamSynchronize(t->side));
  if (t->side_owned) NEST_CUDA(cudaStreamDestroy(t->side));
  t->side = st;
  t->side_owned = false;
}

void tower_join(Ctx& c, cudaStream_t st) {
  Tower* t = reinterpret_cast<Tower*>(c.tower);
  if (t && t->dw_pending) NEST_CUDA(cudaStreamWaitEvent(st, t->ev_dw, 0));
}

}  // namespace nest
