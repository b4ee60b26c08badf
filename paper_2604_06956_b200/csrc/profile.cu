// Native tracing: CUDA events around every stage, a pinned ring for device
// counts known only on the GPU (U_o, refreshed rows), and the exposed-All2All
// interval algebra of SURVEY Q16 (communication "not hidden behind
// dense computation").
#include <algorithm>
#include <cstring>

#include "nest_internal.cuh"

namespace nest {

static_assert(int(ST_COUNT) == int(NEST_PROFILE_STAGES), "stage table out of sync with include/nest.h");
static const char* kStageName[ST_COUNT] = {"schedule", "route", "sort", "key_a2a", "owner_dedup",
                                           "gather", "refresh", "send_gather", "emb_a2a", "pool",
                                           "tower", "segsum", "grad_a2a", "update", "tower_dw",
                                           "emb_repush"};

static cudaEvent_t take_event(Profiler& p) {
  if (p.next_ev == p.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    p.pool.push_back(e);
  }
  return p.pool[p.next_ev++];
}

int prof_begin(Ctx& c, int stage, int kind, cudaStream_t st) {
  Profiler& p = c.prof;
  if (!p.on) return -1;
  ProfRec r{};
  r.stage = stage;
  r.kind = kind;
  r.e0 = take_event(p);
  r.e1 = take_event(p);
  r.cidx = -1;
  if (!r.e0 || !r.e1) return -1;
  cudaEventRecord(r.e0, st);
  p.recs.push_back(r);
  return int(p.recs.size()) - 1;
}

void prof_end(Ctx& c, int id, cudaStream_t st, double bytes, const int32_t* dcount, double bpc,
              int launches) noexcept {
  Profiler& p = c.prof;
  if (id < 0 || id >= int(p.recs.size())) return;
  ProfRec& r = p.recs[id];
  cudaEventRecord(r.e1, st);
  r.bytes += bytes;
  r.bytes_per_cnt = bpc;
  r.launches = launches;
  p.launches += launches;
  if (dcount && p.hcnt && p.ncnt < p.cap_cnt) {
    r.cidx = p.ncnt++;
    cudaMemcpyAsync(p.hcnt + r.cidx, dcount, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  }
}

void prof_add_bytes(Ctx& c, int id, double bytes) noexcept {
  if (id >= 0 && id < int(c.prof.recs.size())) c.prof.recs[id].bytes += bytes;
}

void prof_set_hbm(Ctx& c, int id, double hbm) noexcept {
  if (id >= 0 && id < int(c.prof.recs.size()) && hbm >= 0) c.prof.recs[id].hbm = hbm;
}

void profile_enable(Ctx& c, bool on) {
  Profiler& p = c.prof;
  if (on) {
    NEST_CUDA(cudaDeviceSynchronize());
    if (!p.hcnt) NEST_CUDA(cudaMallocHost(&p.hcnt, sizeof(int32_t) * p.cap_cnt));
    if (!p.ref) NEST_CUDA(cudaEventCreate(&p.ref));
    if (!p.ref_stream) NEST_CUDA(cudaStreamCreateWithFlags(&p.ref_stream, cudaStreamNonBlocking));
    p.recs.clear();
    p.next_ev = 0;
    p.ncnt = 0;
    p.launches = 0;
    NEST_CUDA(cudaEventRecord(p.ref, p.ref_stream));
    NEST_CUDA(cudaStreamSynchronize(p.ref_stream));
    p.on = true;
  } else {
    p.on = false;
  }
}

static double measure(std::vector<std::pair<double, double>> iv) {
  std::sort(iv.begin(), iv.end());
  double tot = 0, cs = -1e300, ce = -1e300;
  for (auto& x : iv) {
    if (x.first > ce) {
      if (ce > cs) tot += ce - cs;
      cs = x.first;
      ce = x.second;
    } else if (x.second > ce) {
      ce = x.second;
    }
  }
  if (ce > cs) tot += ce - cs;
  return tot;
}

// measure of A \ B for interval sets
static double measure_minus(const std::vector<std::pair<double, double>>& A,
                            const std::vector<std::pair<double, double>>& B) {
  std::vector<std::pair<double, double>> AB = A;
  // |A \ B| = |A u B| - |B|
  AB.insert(AB.end(), B.begin(), B.end());
  return measure(AB) - measure(B);
}

void profile_read(Ctx& c, nest_profile_stage_t* stages, nest_profile_summary_t* sum) {
  Profiler& p = c.prof;
  NEST_CUDA(cudaDeviceSynchronize());
  std::vector<nest_profile_stage_t> agg(ST_COUNT);
  for (int s = 0; s < ST_COUNT; ++s) {
    std::memset(&agg[s], 0, sizeof(agg[s]));
    std::strncpy(agg[s].name, kStageName[s], sizeof(agg[s].name) - 1);
    agg[s].stream = -1;
  }
  std::vector<std::pair<double, double>> a2a, comp;
  double t_min = 1e300, t_max = -1e300, a2a_ms = 0;
  for (const ProfRec& r : p.recs) {
    float t0 = 0, t1 = 0;
    NEST_CUDA(cudaEventElapsedTime(&t0, p.ref, r.e0));
    NEST_CUDA(cudaEventElapsedTime(&t1, p.ref, r.e1));
    nest_profile_stage_t& g = agg[r.stage];
    g.stream = r.kind;
    g.records += 1;
    g.launches += r.launches;
    g.ms += double(t1) - double(t0);
    double bytes = r.bytes;
    if (r.cidx >= 0) {
      bytes += r.bytes_per_cnt * double(p.hcnt[r.cidx]);
      g.units += double(p.hcnt[r.cidx]);
    }
    g.bytes += bytes;
    if (r.stage == ST_TOWER || r.stage == ST_TOWER_DW) {
      // FLOPs, not bytes
    } else if (r.stage == ST_EMB_A2A || r.stage == ST_GRAD_A2A || r.stage == ST_KEY_A2A) {
      g.hbm_bytes += r.hbm >= 0 ? r.hbm : 0.0;   // transport stages: `bytes` are off-GPU bytes
    } else {
      g.hbm_bytes += bytes;
    }
    t_min = std::min(t_min, double(t0));
    t_max = std::max(t_max, double(t1));
    if (r.stage == ST_EMB_A2A || r.stage == ST_GRAD_A2A || r.stage == ST_EMB_REPUSH) {
      a2a.emplace_back(t0, t1);
      a2a_ms += double(t1) - double(t0);
    } else if (r.stage == ST_POOL || r.stage == ST_TOWER || r.stage == ST_SEGSUM || r.stage == ST_TOWER_DW) {
      // the compute lane: dense forward/backward of the window
      comp.emplace_back(t0, t1);
    }
  }
  if (stages) std::memcpy(stages, agg.data(), sizeof(nest_profile_stage_t) * ST_COUNT);
  if (sum) {
    sum->span_ms = p.recs.empty() ? 0.0 : t_max - t_min;
    sum->a2a_ms = a2a_ms;
    sum->a2a_union_ms = measure(a2a);
    sum->a2a_exposed_ms = measure_minus(a2a, comp);
    sum->compute_busy_ms = measure(comp);
    sum->launches = p.launches;
  }
}

void profile_records(Ctx& c, nest_profile_record_t* out, int64_t cap, int64_t* n) {
  Profiler& p = c.prof;
  NEST_CUDA(cudaDeviceSynchronize());
  *n = int64_t(p.recs.size());
  if (!out) return;
  for (int64_t i = 0; i < *n && i < cap; ++i) {
    const ProfRec& r = p.recs[size_t(i)];
    float t0 = 0, t1 = 0;
    NEST_CUDA(cudaEventElapsedTime(&t0, p.ref, r.e0));
    NEST_CUDA(cudaEventElapsedTime(&t1, p.ref, r.e1));
    out[i] = nest_profile_record_t{r.stage, r.kind, double(t0), double(t1)};
  }
}

// checked mode: guard bands after every workspace buffer
__global__ void k_guard_fill(char* base, const uint64_t* __restrict__ offs, int64_t n) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    uint32_t* g = reinterpret_cast<uint32_t*>(base + offs[i]);
    for (int j = threadIdx.x; j < int(kGuardBytes / 4); j += blockDim.x) g[j] = kGuardWord;
  }
}
__global__ void k_guard_check(const char* base, const uint64_t* __restrict__ offs, int64_t n,
                              unsigned long long* bad) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t* g = reinterpret_cast<const uint32_t*>(base + offs[i]);
    for (int j = threadIdx.x; j < int(kGuardBytes / 4); j += blockDim.x)
      if (g[j] != kGuardWord) atomicAdd(bad, 1ull);
  }
}
void guards_fill(Ctx& c, cudaStream_t st) {
  k_guard_fill<<<148, 64, 0, st>>>(c.work_base, c.d_guard_offs, int64_t(c.guard_offs.size()));
  NEST_LAUNCH_CHECK();
}
int64_t guards_check(Ctx& c, cudaStream_t st) {
  NEST_CUDA(cudaMemsetAsync(c.d_guard_bad, 0, sizeof(unsigned long long), st));
  k_guard_check<<<148, 64, 0, st>>>(c.work_base, c.d_guard_offs, int64_t(c.guard_offs.size()), c.d_guard_bad);
  NEST_LAUNCH_CHECK();
  unsigned long long h = 0;
  NEST_CUDA(cudaMemcpyAsync(&h, c.d_guard_bad, sizeof(h), cudaMemcpyDeviceToHost, st));
  NEST_CUDA(cudaStreamSynchronize(st));
  return int64_t(h);
}

void profile_destroy(Ctx& c) {
  Profiler& p = c.prof;
  for (auto e : p.pool) cudaEventDestroy(e);
  p.pool.clear();
  if (p.ref) cudaEventDestroy(p.ref);
  if (p.ref_stream) cudaStreamDestroy(p.ref_stream);
  if (p.hcnt) cudaFreeHost(p.hcnt);
  p.ref = nullptr;
  p.ref_stream = nullptr;
  p.hcnt = nullptr;
}

}  // namespace nest
