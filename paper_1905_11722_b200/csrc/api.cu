// api.cu — the extern "C" boundary of libremat_b200.so (include/remat_b200.h).
//
// Host orchestration only: argument validation with the reference's error
// semantics, device buffers, the k-ary budget search.  All per-member, per-pair
// and per-state arithmetic runs in the kernels of family.cu / relax.cu /
// evaluate.cu / simulate.cu; there is no host compute fallback.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace remat {

static thread_local std::string g_last_error;
thread_local cudaStream_t tls_stream = nullptr;

thread_local cudaMemPool_t tls_pool = nullptr;

size_t pool_keep_bytes() {
  static size_t keep = [] {
    const char* e = getenv("REMAT_POOL_KEEP_GB");
    return e ? (size_t)(atof(e) * (1ull << 30)) : kPoolKeepBytes;
  }();
  return keep;
}

cudaMemPool_t prepare_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDevices] = {};
  const int d = dev_slot(device);
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[d]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      cudaDeviceGetDefaultMemPool(&pool, device);  // cannot happen on sm_100; stay usable
    } else {
      unsigned long long keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pools[d] = pool;
  }
  tls_pool = pools[d];
  return pools[d];
}
int sm_count(int device) {
  static std::atomic<int> sms[kMaxDevices] = {};
  const int d = dev_slot(device);
  int v = sms[d].load();
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v < 1)
      v = 148;
    sms[d].store(v);
  }
  return v;
}

static std::atomic<long long> g_launches{0};

void set_error(int code, const std::string& msg) {
  (void)code;
  g_last_error = msg;
}

int fail(int code, const std::string& msg) {
  set_error(code, msg);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? REMAT_ERR_NOMEM : REMAT_ERR_CUDA,
              std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void count_launch(int n) { g_launches += n; }

int Events::create() {
  for (auto& x : e) RM_CUDA(cudaEventCreate(&x));
  return REMAT_OK;
}

void Events::destroy() {
  for (auto& x : e)
    if (x) cudaEventDestroy(x);
}

// Decompose a cost vector into K (mask, coefficient) classes with
// cost[v] = Σ_c coef_c · [v ∈ mask_c], choosing the smaller of value classes
// and bit planes; returns false when both exceed kMaxClasses.
static bool weight_classes(const std::vector<long long>& cost, int n, int Wp,
                           std::vector<u64>& masks, std::vector<long long>& coef) {
  std::map<long long, std::vector<int>> byval;
  for (int v = 0; v < n; v++)
    if (cost[v]) byval[cost[v]].push_back(v);
  int planes = 0;
  long long orall = 0;
  for (int v = 0; v < n; v++) orall |= cost[v];
  for (int b = 0; b < 63; b++) planes += (orall >> b) & 1;
  masks.clear();
  coef.clear();
  if ((int)byval.size() <= planes) {
    if ((int)byval.size() > kMaxClasses) return false;
    for (auto& kv : byval) {
      std::vector<u64> m(Wp, 0);
      for (int v : kv.second) m[v >> 6] |= 1ull << (v & 63);
      masks.insert(masks.end(), m.begin(), m.end());
      coef.push_back(kv.first);
    }
  } else {
    if (planes > kMaxClasses) return false;
    for (int b = 0; b < 63; b++) {
      if (!((orall >> b) & 1)) continue;
      std::vector<u64> m(Wp, 0);
      for (int v = 0; v < n; v++)
        if ((cost[v] >> b) & 1) m[v >> 6] |= 1ull << (v & 63);
      masks.insert(masks.end(), m.begin(), m.end());
      coef.push_back(1LL << b);
    }
  }
  return true;
}

// Classes for both weights at once: (mask, cT, cM) with
// T_v = Σ_{c ∋ v} cT_c and M_v = Σ_{c ∋ v} cM_c.  Either the joint partition
// by (T_v, M_v) value pairs, or the T and M decompositions side by side with
// identical masks merged — whichever has fewer classes (uniform costs: one
// class, so a weighted popcount pair is a single popcount).
static bool joint_classes(const std::vector<long long>& T, const std::vector<long long>& M, int n,
                          int Wp, std::vector<u64>& cls, std::vector<long long>& coef) {
  std::map<std::pair<long long, long long>, std::vector<int>> joint;
  for (int v = 0; v < n; v++)
    if (T[v] || M[v]) joint[{T[v], M[v]}].push_back(v);
  std::vector<u64> mT, mM;
  std::vector<long long> kT, kM;
  const bool okT = weight_classes(T, n, Wp, mT, kT), okM = weight_classes(M, n, Wp, mM, kM);
  // separate form, merging classes with identical masks
  std::vector<std::vector<u64>> sm;
  std::vector<std::pair<long long, long long>> sc;
  auto add = [&](const u64* m, long long ct, long long cm) {
    for (size_t q = 0; q < sm.size(); q++)
      if (std::equal(sm[q].begin(), sm[q].end(), m)) {
        sc[q].first += ct;
        sc[q].second += cm;
        return;
      }
    sm.emplace_back(m, m + Wp);
    sc.push_back({ct, cm});
  };
  if (okT && okM) {
    for (size_t c = 0; c < kT.size(); c++) add(mT.data() + c * Wp, kT[c], 0);
    for (size_t c = 0; c < kM.size(); c++) add(mM.data() + c * Wp, 0, kM[c]);
  }
  cls.clear();
  coef.clear();
  const bool use_joint = (int)joint.size() <= kMaxClasses &&
                         (!(okT && okM) || joint.size() <= sm.size());
  if (use_joint) {
    for (auto& kv : joint) {
      std::vector<u64> m(Wp, 0);
      for (int v : kv.second) m[v >> 6] |= 1ull << (v & 63);
      cls.insert(cls.end(), m.begin(), m.end());
      coef.push_back(kv.first.first);
      coef.push_back(kv.first.second);
    }
    return true;
  }
  if (!(okT && okM) || (int)sm.size() > kMaxClasses) return false;
  for (size_t q = 0; q < sm.size(); q++) {
    cls.insert(cls.end(), sm[q].begin(), sm[q].end());
    coef.push_back(sc[q].first);
    coef.push_back(sc[q].second);
  }
  return true;
}

static int upload(DevBuf<u64>& d, const std::vector<u64>& h, cudaStream_t s) {
  int rc = d.ensure(h.size());
  if (rc < 0) return rc;
  if (!h.empty())
    RM_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
  return REMAT_OK;
}

static int upload(DevBuf<long long>& d, const std::vector<long long>& h, cudaStream_t s) {
  int rc = d.ensure(h.size());
  if (rc < 0) return rc;
  if (!h.empty())
    RM_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
  return REMAT_OK;
}

static int set_device(int dev, cudaStream_t s = nullptr) {
  RM_CUDA(cudaSetDevice(dev));
  prepare_pool(dev);
  tls_stream = s;
  return REMAT_OK;
}

int graph_enter(remat_graph_s* g) { return set_device(g->device, g->stream); }

}  // namespace remat

using namespace remat;

extern "C" {

int remat_abi_version(void) { return REMAT_ABI_VERSION; }

const char* remat_last_error(void) { return g_last_error.c_str(); }

int64_t remat_kernel_launch_count(void) { return g_launches.load(); }

int remat_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *count = c;
  return REMAT_OK;
}

int remat_graph_create(int32_t device, int32_t n, const uint64_t* preds, const uint64_t* succs,
                       const int64_t* compute_costs, const int64_t* memory_costs,
                       remat_graph_t* out) {
  if (!out) return fail(REMAT_ERR_VALUE, "null output pointer");
  *out = nullptr;
  if (!preds || !succs || !compute_costs || !memory_costs)
    return fail(REMAT_ERR_VALUE, "null graph array");
  if (n < 1) return fail(REMAT_ERR_VALUE, "graph must have at least one node");
  const int W = (n + 63) / 64;
  const int Wp = padded_words(W);
  if (Wp < 0 || Wp > kMaxWords)
    return fail(REMAT_ERR_VALUE, "graphs above " + std::to_string(kMaxWords * 64) +
                                     " nodes are not supported by this build");
  long long TV = 0, MV = 0, maxM = 0;
  for (int v = 0; v < n; v++) {
    if (compute_costs[v] < 0) return fail(REMAT_ERR_VALUE, "compute cost must be >= 0");
    if (memory_costs[v] < 1) return fail(REMAT_ERR_VALUE, "memory cost must be >= 1");
    if (__builtin_add_overflow(TV, compute_costs[v], &TV) ||
        __builtin_add_overflow(MV, memory_costs[v], &MV))
      return fail(REMAT_ERR_RANGE, "aggregate node costs exceed the supported integer range");
    maxM = std::max<long long>(maxM, memory_costs[v]);
  }
  if (MV > (1LL << 61))
    return fail(REMAT_ERR_RANGE, "total memory cost must stay below 2^61 (2*M(V) stage bound)");
  int rc = set_device(device);
  if (rc < 0) return rc;
  auto* g = new remat_graph_s();
  g->device = device;
  g->n = n;
  g->W = W;
  g->Wp = Wp;
  g->TV = TV;
  g->MV = MV;
  g->maxM = maxM;
  auto cleanup = [&](int code) {
    if (g->stream) cudaStreamDestroy(g->stream);
    g->ev.destroy();
    delete g;
    return code;
  };
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(REMAT_ERR_CUDA, "cudaStreamCreate failed"));
  tls_stream = g->stream;
  if ((rc = g->ev.create()) < 0) return cleanup(rc);
  std::vector<u64> hp((size_t)n * Wp, 0), hs((size_t)n * Wp, 0);
  for (int v = 0; v < n; v++)
    for (int w = 0; w < W; w++) {
      hp[(size_t)v * Wp + w] = preds[(size_t)v * W + w];
      hs[(size_t)v * Wp + w] = succs[(size_t)v * W + w];
    }
  g->indeg.assign(n, 0);
  g->outdeg.assign(n, 0);
  for (int v = 0; v < n; v++)
    for (int w = 0; w < W; w++) {
      g->indeg[v] += __builtin_popcountll(preds[(size_t)v * W + w]);
      g->outdeg[v] += __builtin_popcountll(succs[(size_t)v * W + w]);
    }
  for (int v = 0; v < n; v++) g->edges += g->outdeg[v];
  g->hT.assign(compute_costs, compute_costs + n);
  g->hM.assign(memory_costs, memory_costs + n);
  g->t_uniform = std::all_of(g->hT.begin(), g->hT.end(), [&](long long t) { return t == g->hT[0]; });
  std::vector<u64> cls;
  std::vector<long long> coef;
  g->cls_enabled = joint_classes(g->hT, g->hM, n, Wp, cls, coef);
  g->K = (int)coef.size() / 2;
  if ((rc = upload(g->preds, hp, g->stream)) < 0 || (rc = upload(g->succs, hs, g->stream)) < 0 ||
      (rc = upload(g->T, g->hT, g->stream)) < 0 || (rc = upload(g->M, g->hM, g->stream)) < 0 ||
      (rc = upload(g->cls, cls, g->stream)) < 0 || (rc = upload(g->coef, coef, g->stream)) < 0)
    return cleanup(rc);
  if (cudaStreamSynchronize(g->stream) != cudaSuccess)
    return cleanup(fail(REMAT_ERR_CUDA, "graph upload failed"));
  *out = g;
  return REMAT_OK;
}

int remat_graph_free(remat_graph_t g) {
  if (!g) return REMAT_OK;
  set_device(g->device, g->stream);
  free_sched_scratch(g);
  g->ev.destroy();
  cudaStream_t s = g->stream;
  delete g;
  if (s) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  tls_stream = nullptr;
  return REMAT_OK;
}

int remat_graph_stream(remat_graph_t g, void** stream) {
  if (!g) return fail(REMAT_ERR_VALUE, "null graph handle");
  *stream = (void*)g->stream;
  return REMAT_OK;
}

int remat_family_create(remat_graph_t g, int32_t kind, int64_t cap, remat_family_t* out) {
  if (!out) return fail(REMAT_ERR_VALUE, "null output pointer");
  *out = nullptr;
  if (!g) return fail(REMAT_ERR_VALUE, "null graph handle");
  if (kind != REMAT_FAMILY_FULL && kind != REMAT_FAMILY_PRUNED)
    return fail(REMAT_ERR_VALUE, "family must be full (0) or pruned (1)");
  if (kind == REMAT_FAMILY_FULL && cap < (int64_t)g->n + 1)
    return fail(REMAT_ERR_VALUE, "cap must be at least n+1 = " + std::to_string(g->n + 1) +
                                     ", got " + std::to_string(cap));
  int rc = set_device(g->device, g->stream);
  if (rc < 0) return rc;
  auto* f = new remat_family_s();
  const long long launches0 = remat_kernel_launch_count();
  rc = build_family(g, kind, cap, f);
  if (rc < 0) {
    cudaStreamSynchronize(g->stream);
    delete f;
    return rc;
  }
  f->timings.kernel_launches = remat_kernel_launch_count() - launches0;
  *out = f;
  return REMAT_OK;
}

int remat_family_size(remat_family_t f, int64_t* size) {
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  *size = f->F;
  return REMAT_OK;
}

int remat_family_masks(remat_family_t f, int64_t start, int64_t count, uint64_t* out) {
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  if (start < 0 || count < 0 || start + count > f->F)
    return fail(REMAT_ERR_VALUE, "family index range out of bounds");
  remat_graph_s* g = f->g;
  int rc = set_device(g->device, g->stream);
  if (rc < 0) return rc;
  const int W = g->W;
  std::vector<u64> tmp((size_t)count);
  for (int w = 0; w < W; w++) {
    if (count)
      RM_CUDA(cudaMemcpyAsync(tmp.data(), f->masks.p + (size_t)w * f->F + start, count * 8,
                              cudaMemcpyDeviceToHost, g->stream));
    RM_CUDA(cudaStreamSynchronize(g->stream));
    for (int64_t i = 0; i < count; i++) out[i * W + w] = tmp[i];
  }
  return REMAT_OK;
}

int remat_family_free(remat_family_t f) {
  if (!f) return REMAT_OK;
  remat_graph_s* g = f->g;
  set_device(g->device, g->stream);
  delete f;
  // return what a large family held beyond the pool's working set
  cudaStreamSynchronize(g->stream);
  cudaMemPoolTrimTo(tls_pool, pool_keep_bytes());
  return REMAT_OK;
}

int remat_family_timings(remat_family_t f, remat_timings* out) {
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  *out = f->timings;
  return REMAT_OK;
}

int remat_family_member_stats(remat_family_t f, int32_t b, int64_t start, int64_t count,
                              int32_t* flen, int32_t* cells, uint64_t* trans, uint64_t* pairs) {
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  if (f->cur_nb < 1) return fail(REMAT_ERR_VALUE, "no solve has run on this family");
  if (b < 0 || b >= f->cur_nb) return fail(REMAT_ERR_VALUE, "budget index out of range");
  if (start < 0 || count < 0 || start + count > f->F)
    return fail(REMAT_ERR_VALUE, "member range out of bounds");
  if (count == 0) return REMAT_OK;
  int rc = set_device(f->g->device, f->g->stream);
  if (rc < 0) return rc;
  cudaStream_t s = f->g->stream;
  const size_t off = (size_t)b * f->F + start;
  if (flen)
    RM_CUDA(cudaMemcpyAsync(flen, f->flen.p + off, 4 * count, cudaMemcpyDeviceToHost, s));
  if (cells)
    RM_CUDA(cudaMemcpyAsync(cells, f->ccount.p + off, 4 * count, cudaMemcpyDeviceToHost, s));
  if (trans)
    RM_CUDA(cudaMemcpyAsync(trans, f->trans.p + off, 8 * count, cudaMemcpyDeviceToHost, s));
  if (pairs)
    RM_CUDA(cudaMemcpyAsync(pairs, f->npairs.p + off, 8 * count, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  return REMAT_OK;
}

int remat_solve(remat_family_t f, const int64_t* budgets, int32_t nb, int32_t objective,
                remat_plan_info* info, uint64_t* chain_masks, uint64_t* cached_masks,
                int64_t* stage_memory) {
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  if (!budgets || !info) return fail(REMAT_ERR_VALUE, "null budget or result array");
  if (nb < 1) return fail(REMAT_ERR_VALUE, "need at least one budget");
  if (objective != REMAT_MINIMIZE && objective != REMAT_MAXIMIZE)
    return fail(REMAT_ERR_VALUE, "objective must be minimize (0) or maximize (1)");
  remat_graph_s* g = f->g;
  int rc = set_device(g->device, g->stream);
  if (rc < 0) return rc;
  std::vector<long long> bs(nb);
  for (int b = 0; b < nb; b++) {
    if (budgets[b] < 0) return fail(REMAT_ERR_VALUE, "budget must be non-negative");
    // every stage needs at most 2·M(V): larger budgets
    // behave identically
    bs[b] = std::min<long long>(budgets[b], 2 * g->MV);
  }
  rc = solve_batch(f, bs, objective, info, (u64*)chain_masks, (u64*)cached_masks,
                   (long long*)stage_memory);
  if (rc < 0) return rc;
  int worst = REMAT_OK;
  for (int b = 0; b < nb; b++) {
    info[b].budget = budgets[b];
    if (info[b].status == REMAT_ERR_INTERNAL) worst = REMAT_ERR_INTERNAL;
  }
  if (worst < 0) return fail(worst, "plan failed the reference self-check (planner.py:206-210)");
  return REMAT_OK;
}

int remat_min_feasible_budget(remat_family_t f, int32_t objective, int32_t probes_per_round,
                              int64_t* b_min, remat_plan_info* info, uint64_t* chain_masks,
                              uint64_t* cached_masks, int64_t* stage_memory,
                              int64_t* probes_run, int64_t* probe_transitions) {
  if (!f || !b_min || !info) return fail(REMAT_ERR_VALUE, "null family handle or output");
  if (objective != REMAT_MINIMIZE && objective != REMAT_MAXIMIZE)
    return fail(REMAT_ERR_VALUE, "objective must be minimize (0) or maximize (1)");
  remat_graph_s* g = f->g;
  int rc = set_device(g->device, g->stream);
  if (rc < 0) return rc;
  const int K = std::max(1, std::min(probes_per_round, 256));
  const int n = g->n, W = g->W;
  const size_t rows = (size_t)(n + 1);
  // feasibility is monotone in the budget; 2·M(V) always admits the
  // single-segment plan and no stage fits below 2·max_v M_v
  long long hi = 2 * g->MV, lo = 2 * g->maxM - 1;
  bool have = false;
  remat_plan_info best{};
  std::vector<uint64_t> bchain(rows * W), bcached(rows * W);
  std::vector<int64_t> bstage(rows);
  long long probes = 0, ptrans = 0;
  std::vector<remat_plan_info> pinfo;
  // a round returns only the probes' figures; the rows of the plan that
  // becomes the new upper bound are fetched from the device alone
  auto take = [&](int idx) -> int {
    best = pinfo[idx];
    have = true;
    return plan_rows(f, idx, (u64*)bchain.data(), (u64*)bcached.data(), (long long*)bstage.data());
  };
  while (hi - lo > 1) {
    std::vector<int64_t> probe;
    for (int k = 1; k <= K; k++) {
      int64_t b = lo + (long long)(((__int128)(hi - lo) * k) / (K + 1));
      if (b > lo && b < hi && (probe.empty() || b != probe.back())) probe.push_back(b);
    }
    if (probe.empty()) probe.push_back(lo + (hi - lo) / 2);
    const int nb = (int)probe.size();
    pinfo.assign(nb, remat_plan_info{});
    rc = remat_solve(f, probe.data(), nb, objective, pinfo.data(), nullptr, nullptr, nullptr);
    if (rc < 0) return rc;
    probes += nb;
    int first_ok = -1;
    for (int b = 0; b < nb; b++) {
      ptrans += pinfo[b].stats.transitions;
      if (pinfo[b].status == REMAT_OK && first_ok < 0) first_ok = b;
    }
    if (first_ok >= 0) {
      hi = probe[first_ok];
      if ((rc = take(first_ok)) < 0) return rc;
      if (first_ok > 0) lo = probe[first_ok - 1];
    } else {
      lo = probe.back();
    }
  }
  if (!have) {
    int64_t b = hi;
    pinfo.assign(1, remat_plan_info{});
    rc = remat_solve(f, &b, 1, objective, pinfo.data(), nullptr, nullptr, nullptr);
    if (rc < 0) return rc;
    probes += 1;
    ptrans += pinfo[0].stats.transitions;
    if (pinfo[0].status != REMAT_OK)
      return fail(REMAT_ERR_INTERNAL, "internal error: single-segment plan must fit 2*M(V)");
    if ((rc = take(0)) < 0) return rc;
  }
  *b_min = hi;
  *info = best;
  if (chain_masks) std::memcpy(chain_masks, bchain.data(), rows * W * 8);
  if (cached_masks) std::memcpy(cached_masks, bcached.data(), rows * W * 8);
  if (stage_memory) std::memcpy(stage_memory, bstage.data(), rows * 8);
  if (probes_run) *probes_run = probes;
  if (probe_transitions) *probe_transitions = ptrans;
  return REMAT_OK;
}

int remat_evaluate(remat_graph_t g, int32_t k, const uint64_t* chain, int64_t* overhead,
                   int64_t* stage_memory, int64_t* peak, int64_t* cached_total,
                   uint64_t* cached_masks) {
  if (!g || !chain || !overhead || !peak || !cached_total)
    return fail(REMAT_ERR_VALUE, "null graph handle or argument");
  const int n = g->n, W = g->W, Wp = g->Wp;
  if (k < 1 || k > n) return fail(REMAT_ERR_VALUE, "chain length must be in [1, n]");
  int rc = set_device(g->device, g->stream);
  if (rc < 0) return rc;
  const size_t rows = (size_t)(n + 1);
  std::vector<u64> hc(rows * Wp, 0);
  for (int s = 0; s < k; s++)
    for (int w = 0; w < W; w++) hc[(size_t)s * Wp + w] = chain[(size_t)s * W + w];
  if ((rc = upload(g->chain_buf, hc, g->stream)) < 0 || (rc = g->int_buf.ensure(2)) < 0 ||
      (rc = g->terms_buf.ensure(rows * 4)) < 0 || (rc = g->bound_buf.ensure(rows * Wp)) < 0 ||
      (rc = g->cached_buf.ensure(rows * Wp)) < 0 || (rc = g->stage_buf.ensure(rows)) < 0 ||
      (rc = g->eval_out.ensure(8)) < 0)
    return rc;
  RM_CUDA(cudaMemcpyAsync(g->int_buf.p, &k, sizeof(int), cudaMemcpyHostToDevice, g->stream));
  rc = evaluate_chains(g, 1, g->chain_buf.p, g->int_buf.p, nullptr, g->stage_buf.p,
                       g->cached_buf.p, g->eval_out.p, g->terms_buf.p, g->bound_buf.p);
  if (rc < 0) return rc;
  long long res[8];
  std::vector<long long> st(rows);
  std::vector<u64> cm(rows * Wp);
  RM_CUDA(cudaMemcpyAsync(res, g->eval_out.p, sizeof res, cudaMemcpyDeviceToHost, g->stream));
  RM_CUDA(cudaMemcpyAsync(st.data(), g->stage_buf.p, rows * 8, cudaMemcpyDeviceToHost, g->stream));
  RM_CUDA(cudaMemcpyAsync(cm.data(), g->cached_buf.p, rows * Wp * 8, cudaMemcpyDeviceToHost,
                          g->stream));
  RM_CUDA(cudaStreamSynchronize(g->stream));
  if (res[0] != REMAT_OK)
    return fail(REMAT_ERR_INTERNAL, "stage-wise overhead disagrees with cache complement");
  *overhead = res[2];
  *peak = res[3];
  *cached_total = res[4];
  for (int s = 0; s < k; s++) {
    if (stage_memory) stage_memory[s] = st[s];
    if (cached_masks)
      for (int w = 0; w < W; w++) cached_masks[(size_t)s * W + w] = cm[(size_t)s * Wp + w];
  }
  return REMAT_OK;
}

int remat_simulate(remat_graph_t g, int32_t nsched, const int64_t* offsets, const int32_t* ops,
                   remat_sim_info* info, int64_t* traces) {
  if (!g || !offsets || !ops || !info) return fail(REMAT_ERR_VALUE, "null graph handle or argument");
  if (nsched < 1) return fail(REMAT_ERR_VALUE, "need at least one schedule");
  if (offsets[0] != 0) return fail(REMAT_ERR_VALUE, "bad schedule offsets");
  // exact event counts per stream (schedule.cu inst_events): F v touches
  // preds+1 refs, B v preds+2+succs, FREE one
  std::vector<int64_t> events(nsched, 0);
  for (int s = 0; s < nsched; s++) {
    if (offsets[s + 1] < offsets[s]) return fail(REMAT_ERR_VALUE, "bad schedule offsets");
    long long e = 0;
    for (long long q = offsets[s]; q < offsets[s + 1]; q++) {
      const int kind = ops[2 * q], v = ops[2 * q + 1];
      if (v < 0 || v >= g->n || kind < 0 || kind > 3) continue;
      e += kind == 0 ? g->indeg[v] + 1 : kind == 1 ? g->indeg[v] + 2 + g->outdeg[v] : 1;
    }
    events[s] = e;
  }
  return remat_schedule_streams(g, nsched, offsets, ops, events.data(), 2, 0, nullptr, nullptr,
                                info, traces);
}

}  // extern "C"
