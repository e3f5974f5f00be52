// shard.cu — level-sharded exact DP across GPUs.
//
// The targets of every heavy level are split into contiguous rank ranges;
// each rank relaxes its share against its full replica of the finished
// levels, then the ranks exchange the finished level IN PLACE: one NCCL group
// of broadcasts per level, rank r the root of its own share, every rank
// receiving straight into its replica's frontier slots, back-pointers and
// per-member records (|frontier|, |cell|, smallest m, Σ|frontier_i|,
// comparable pairs) — no staging copy, no pack or unpack kernel.  A level's
// members (and their frontier slots) are contiguous in family order, so a
// rank's share is one contiguous region per array.  Light levels (less work
// than an exchange costs) are relaxed by every rank in full and batched into
// the cooperative multi-level launch, exactly as on one GPU.  After the last
// level every replica holds the whole table, so reconstruction, figures and
// statistics run unchanged on each rank and every rank returns the same plan
// (bit-identical to one GPU: a target's value does not depend on who computed
// it).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"), so the library has no
// link-time NCCL dependency and shares the copy torch.distributed already
// loaded.  A loopback mode runs G replicas on ONE device with device copies in
// place of the broadcasts — the CI form of the same exchange.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device.cuh"

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

static NcclApi* nccl_api(std::string* why) {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.broadcast = (decltype(api.broadcast))dlsym(h, "ncclBroadcast");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.commAbort = (decltype(api.commAbort))dlsym(h, "ncclCommAbort");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    if (!api.getUniqueId || !api.commInitRank || !api.allGather || !api.broadcast ||
        !api.groupStart || !api.groupEnd || !api.commDestroy) {
      err = "NCCL library lacks the required symbols";
      return;
    }
    api.h = h;
  });
  if (!api.h) {
    if (why) *why = err;
    return nullptr;
  }
  return &api;
}

struct remat_comm_s {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  remat::DevBuf<unsigned long long> flag;  // [world] status words: non-zero once a rank failed
};

// An NCCL call failed on this rank: abort the communicator so the peers'
// pending collectives error out instead of waiting forever, and make the
// handle unusable (remat_comm_free then has nothing left to destroy).
static int comm_abort(remat_comm_s* c, NcclApi* api, ncclResult_t r, const char* what) {
  std::string msg = std::string(what) + ": " + api->errorString(r);
  if (c->comm) {
    if (api->commAbort) api->commAbort(c->comm);
    c->comm = nullptr;
  }
  return remat::fail(REMAT_ERR_CUDA, msg + " (communicator aborted)");
}

namespace remat {

// contiguous share [lo, hi) of `width` targets starting at j0 for `rank`
static inline void part(long long j0, long long width, int world, int rank, long long* lo,
                        long long* hi) {
  *lo = j0 + width * rank / world;
  *hi = j0 + width * (rank + 1) / world;
}

// A batch of word copies (all offsets and lengths are multiples of 4 bytes).
constexpr int kSegs = 48;
struct Segs {
  const unsigned* src[kSegs];
  unsigned* dst[kSegs];
  long long words[kSegs];
  int n;
};

__global__ void k_copy_segs(Segs sg) {
  for (int k = blockIdx.y; k < sg.n; k += gridDim.y) {
    const unsigned* __restrict__ a = sg.src[k];
    unsigned* __restrict__ b = sg.dst[k];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < sg.words[k];
         i += (long long)gridDim.x * blockDim.x)
      b[i] = a[i];
  }
}

struct SegList {
  std::vector<const void*> src;
  std::vector<void*> dst;
  std::vector<long long> bytes;
  void add(const void* s, void* d, long long b) {
    if (b <= 0) return;
    src.push_back(s);
    dst.push_back(d);
    bytes.push_back(b);
  }
  int flush(cudaStream_t st) {
    for (size_t k0 = 0; k0 < src.size(); k0 += kSegs) {
      Segs sg{};
      sg.n = (int)std::min<size_t>(kSegs, src.size() - k0);
      long long mx = 0;
      for (int k = 0; k < sg.n; k++) {
        sg.src[k] = (const unsigned*)src[k0 + k];
        sg.dst[k] = (unsigned*)dst[k0 + k];
        sg.words[k] = bytes[k0 + k] / 4;
        mx = std::max(mx, sg.words[k]);
      }
      const unsigned bx = (unsigned)std::min<long long>(std::max<long long>(1, (mx + 255) / 256), 512);
      k_copy_segs<<<dim3(bx, (unsigned)sg.n), 256, 0, st>>>(sg);
      RM_LAUNCHED();
    }
    src.clear();
    dst.clear();
    bytes.clear();
    return REMAT_OK;
  }
};

// The regions one rank's share [a, b) of a level occupies in a replica, per
// budget: frontier entries and back-pointers (slots foff[a] .. foff[b]), then
// the five per-member records.  The same (offset, bytes) list on every rank.
struct Region {
  size_t off;     // byte offset inside the array
  size_t bytes;
  int array;      // 0 fe, 1 parent, 2 flen, 3 ccount, 4 mmin, 5 trans, 6 npairs
};
static void share_regions(remat_family_s* f, int nb, long long a, long long b,
                          std::vector<Region>& out) {
  out.clear();
  const long long F = f->F;
  const size_t es = f->cur_narrow ? sizeof(EntryN) : sizeof(EntryW);
  const long long e0 = f->h_foff[a], ne = f->h_foff[b] - f->h_foff[a], m = b - a;
  for (int bb = 0; bb < nb; bb++) {
    const size_t slot0 = (size_t)bb * f->slots + e0, mem0 = (size_t)bb * F + a;
    const Region r[] = {{slot0 * es, ne * es, 0}, {slot0 * 4, (size_t)ne * 4, 1},
                        {mem0 * 4, (size_t)m * 4, 2}, {mem0 * 4, (size_t)m * 4, 3},
                        {mem0 * 8, (size_t)m * 8, 4}, {mem0 * 8, (size_t)m * 8, 5},
                        {mem0 * 8, (size_t)m * 8, 6}};
    for (const Region& x : r)
      if (x.bytes) out.push_back(x);
  }
}
static unsigned char* array_base(remat_family_s* f, int array) {
  switch (array) {
    case 0: return f->fe.p;
    case 1: return reinterpret_cast<unsigned char*>(f->parent.p);
    case 2: return reinterpret_cast<unsigned char*>(f->flen.p);
    case 3: return reinterpret_cast<unsigned char*>(f->ccount.p);
    case 4: return reinterpret_cast<unsigned char*>(f->mmin.p);
    case 5: return reinterpret_cast<unsigned char*>(f->trans.p);
    default: return reinterpret_cast<unsigned char*>(f->npairs.p);
  }
}

static int ensure_foff(remat_family_s* f) {
  if ((long long)f->h_foff.size() == f->F + 1) return REMAT_OK;
  f->h_foff.resize(f->F + 1);
  RM_CUDA(cudaMemcpyAsync(f->h_foff.data(), f->foff.p, sizeof(long long) * (f->F + 1),
                          cudaMemcpyDeviceToHost, f->g->stream));
  RM_CUDA(cudaStreamSynchronize(f->g->stream));
  return REMAT_OK;
}

// Budgets back in the caller's units, and the reference's self-check
// (planner.py:206-210) failure surfaced as an error, as remat_solve does.
static int finish_status(remat_plan_info* info, const int64_t* budgets, int nb) {
  int worst = REMAT_OK;
  for (int b = 0; b < nb; b++) {
    info[b].budget = budgets[b];
    if (info[b].status < 0) worst = REMAT_ERR_INTERNAL;
  }
  if (worst < 0) return fail(worst, "plan failed the reference self-check (planner.py:206-210)");
  return REMAT_OK;
}

// Levels whose relaxation is cheaper than an exchange are REPLICATED: every
// rank relaxes the whole level itself (no collective), and runs of them go
// through the cooperative multi-level launch exactly as on one GPU (C5 has
// 517 levels; only the wide upper ones carry enough work to split).  The
// threshold is in (target, predecessor) subset tests per budget batch
// (REMAT_SHARD_REPLICATE overrides it; 0 shards every level).
static long long replicate_tests() {
  const char* e = getenv("REMAT_SHARD_REPLICATE");  // read per solve (tests toggle it)
  return e ? atoll(e) : (4LL << 20);
}

// Relaxes a run of replicated levels (full target ranges) on one replica.
static int relax_run(remat_family_s* f, std::vector<int>& run) {
  int rc = REMAT_OK;
  if (run.size() == 1)
    rc = solve_level(f, run[0], f->level_start[run[0]], f->level_start[run[0] + 1]);
  else if (!run.empty())
    rc = solve_levels(f, run);
  run.clear();
  return rc;
}

static inline bool replicated(remat_family_s* f, int lvl, int nb) {
  const long long j0 = f->level_start[lvl], w = f->level_start[lvl + 1] - j0;
  return w * j0 * nb <= replicate_tests();
}

static int check_same(remat_family_s* a, remat_family_s* b) {
  if (a->F != b->F || a->g->n != b->g->n || a->slots != b->slots || a->narrow != b->narrow)
    return fail(REMAT_ERR_VALUE, "level-sharded replicas must hold the same family");
  return REMAT_OK;
}

}  // namespace remat

using namespace remat;

extern "C" {

int remat_level_partition(int64_t level_start, int64_t width, int32_t world, int32_t rank,
                          int64_t* begin, int64_t* end) {
  if (world < 1 || rank < 0 || rank >= world || width < 0)
    return fail(REMAT_ERR_VALUE, "bad partition arguments");
  long long lo, hi;
  part(level_start, width, world, rank, &lo, &hi);
  *begin = lo;
  *end = hi;
  return REMAT_OK;
}

int remat_comm_unique_id(uint8_t* id) {
  std::string why;
  NcclApi* api = nccl_api(&why);
  if (!api) return fail(REMAT_ERR_CUDA, why);
  ncclUniqueId u;
  ncclResult_t r = api->getUniqueId(&u);
  if (r != ncclSuccess) return fail(REMAT_ERR_CUDA, std::string("ncclGetUniqueId: ") + api->errorString(r));
  static_assert(sizeof(ncclUniqueId) == REMAT_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof u);
  return REMAT_OK;
}

int remat_comm_create(const uint8_t* id, int32_t world, int32_t rank, int32_t device,
                      remat_comm_t* out) {
  if (world < 1 || rank < 0 || rank >= world) return fail(REMAT_ERR_VALUE, "bad world/rank");
  std::string why;
  NcclApi* api = nccl_api(&why);
  if (!api) return fail(REMAT_ERR_CUDA, why);
  RM_CUDA(cudaSetDevice(device));
  auto* c = new remat_comm_s();
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclResult_t r = api->commInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(REMAT_ERR_CUDA, std::string("ncclCommInitRank: ") + api->errorString(r));
  }
  *out = c;
  return REMAT_OK;
}

int remat_comm_free(remat_comm_t c) {
  if (!c) return REMAT_OK;
  NcclApi* api = nccl_api(nullptr);
  cudaSetDevice(c->device);
  if (api && c->comm) api->commDestroy(c->comm);
  delete c;
  return REMAT_OK;
}

int remat_solve_level_sharded(remat_family_t f, remat_comm_t c, const int64_t* budgets,
                              int32_t nb, int32_t objective, remat_plan_info* info,
                              uint64_t* chain_masks, uint64_t* cached_masks,
                              int64_t* stage_memory) {
  if (!c) return fail(REMAT_ERR_VALUE, "null communicator");
  if (!f) return fail(REMAT_ERR_VALUE, "null family handle");
  if (nb < 1) return fail(REMAT_ERR_VALUE, "need at least one budget");
  if (objective != REMAT_MINIMIZE && objective != REMAT_MAXIMIZE)
    return fail(REMAT_ERR_VALUE, "objective must be minimize (0) or maximize (1)");
  remat_graph_s* g = f->g;
  if (g->device != c->device) return fail(REMAT_ERR_VALUE, "family and communicator devices differ");
  RM_CUDA(cudaSetDevice(g->device));
  prepare_pool(g->device);
  tls_stream = g->stream;
  NcclApi* api = nccl_api(nullptr);
  std::vector<long long> bs(nb);
  for (int b = 0; b < nb; b++) {
    if (budgets[b] < 0) return fail(REMAT_ERR_VALUE, "budget must be non-negative");
    bs[b] = std::min<long long>(budgets[b], 2 * g->MV);
  }
  int rc;
  if (!c->comm) return fail(REMAT_ERR_VALUE, "communicator was aborted by an earlier failure");
  if ((rc = ensure_foff(f)) < 0) return rc;
  const char* fx = getenv("REMAT_SHARD_EXCHANGE");
  const bool exchange = c->world > 1 || (fx && fx[0] == '1');
  // one status word per rank, allocated before the level loop (a rank that
  // fails an allocation inside it could not join the remaining collectives)
  int alloc_rc = exchange ? c->flag.ensure(c->world) : REMAT_OK;
  if (c->world > 1) {
    // every rank must hold the same family, solve the same budgets and have
    // its status words: one all-gather of a small header checks it before any
    // level is exchanged
    const int HW = 7;
    long long mine[HW] = {f->F, f->slots, (long long)g->n, (long long)f->narrow, (long long)nb,
                          (long long)objective, (long long)(alloc_rc < 0)};
    for (int b = 0; b < nb; b++) mine[4] = mine[4] * 1000003LL + bs[b];
    unsigned char* sp = nullptr;
    RM_CUDA(cudaMallocFromPoolAsync((void**)&sp, sizeof mine * (c->world + 1), tls_pool, g->stream));
    unsigned char* rp = sp + sizeof mine;
    RM_CUDA(cudaMemcpyAsync(sp, mine, sizeof mine, cudaMemcpyHostToDevice, g->stream));
    ncclResult_t r = api->allGather(sp, rp, sizeof mine, ncclUint8, c->comm, g->stream);
    if (r != ncclSuccess) return comm_abort(c, api, r, "ncclAllGather");
    std::vector<long long> all((size_t)HW * c->world);
    RM_CUDA(cudaMemcpyAsync(all.data(), rp, sizeof mine * c->world, cudaMemcpyDeviceToHost,
                            g->stream));
    RM_CUDA(cudaFreeAsync(sp, g->stream));
    RM_CUDA(cudaStreamSynchronize(g->stream));
    if (alloc_rc < 0) return alloc_rc;
    for (int q = 0; q < c->world; q++) {
      if (all[(size_t)q * HW + 6])
        return fail(REMAT_ERR_NOMEM, "level-sharded rank " + std::to_string(q) +
                                         " could not allocate its status words");
      for (int k = 0; k < HW; k++)
        if (all[(size_t)q * HW + k] != mine[k])
          return fail(REMAT_ERR_VALUE, "level-sharded ranks disagree on the family or budgets (rank " +
                                           std::to_string(q) + ")");
    }
  } else if (alloc_rc < 0) {
    return alloc_rc;
  }
  if ((rc = solve_begin(f, bs, objective)) < 0) return rc;
  if (exchange) RM_CUDA(cudaMemsetAsync(c->flag.p, 0, 8 * c->world, g->stream));
  // A local failure after this point must not strand the peers in a
  // collective: the rank stops computing, raises its status word and keeps
  // joining every level's broadcasts; all ranks fail together at the end.
  int local = REMAT_OK;
  bool flagged = false;
  std::vector<int> run;  // replicated levels waiting for one batched launch
  std::vector<Region> regs;
  for (int lvl = 1; lvl <= g->n; lvl++) {
    const long long j0 = f->level_start[lvl], w = f->level_start[lvl + 1] - j0;
    if (w == 0) continue;
    if (replicated(f, lvl, nb)) {
      run.push_back(lvl);
      continue;
    }
    if (local >= 0) local = relax_run(f, run);
    run.clear();
    long long lo, hi;
    part(j0, w, c->world, c->rank, &lo, &hi);
    if (local >= 0) local = solve_level(f, lvl, lo, hi);
    // a one-rank communicator has nothing to exchange (REMAT_SHARD_EXCHANGE=1
    // still runs the broadcasts: the single-GPU test of the NCCL path)
    if (!exchange) {
      if (local < 0) return local;
      continue;
    }
    if (local < 0 && !flagged) {
      cudaMemsetAsync(c->flag.p + c->rank, 0xFF, 8, g->stream);
      flagged = true;
    }
    // the finished level, in place: rank q is the root of its own share
    ncclResult_t r = api->groupStart();
    for (int q = 0; q < c->world && r == ncclSuccess; q++) {
      long long qlo, qhi;
      part(j0, w, c->world, q, &qlo, &qhi);
      share_regions(f, nb, qlo, qhi, regs);
      for (const Region& x : regs) {
        unsigned char* p = array_base(f, x.array) + x.off;
        if ((r = api->broadcast(p, p, x.bytes, ncclUint8, q, c->comm, g->stream)) != ncclSuccess)
          break;
      }
      if (r == ncclSuccess)
        r = api->broadcast(c->flag.p + q, c->flag.p + q, 8, ncclUint8, q, c->comm, g->stream);
    }
    const ncclResult_t r2 = api->groupEnd();
    if (r != ncclSuccess) return comm_abort(c, api, r, "ncclBroadcast");
    if (r2 != ncclSuccess) return comm_abort(c, api, r2, "ncclGroupEnd");
  }
  if (local >= 0) local = relax_run(f, run);
  if (local < 0) return local;
  if (exchange) {
    std::vector<unsigned long long> st(c->world);
    RM_CUDA(cudaMemcpyAsync(st.data(), c->flag.p, 8 * c->world, cudaMemcpyDeviceToHost, g->stream));
    RM_CUDA(cudaStreamSynchronize(g->stream));
    for (unsigned long long x : st)
      if (x) return fail(REMAT_ERR_CUDA, "a peer rank failed during the level-sharded solve");
  }
  if ((rc = solve_finish(f, info, (u64*)chain_masks, (u64*)cached_masks,
                         (long long*)stage_memory)) < 0)
    return rc;
  return finish_status(info, budgets, nb);
}

int remat_solve_level_sharded_loopback(remat_family_t* fams, int32_t world,
                                       const int64_t* budgets, int32_t nb, int32_t objective,
                                       remat_plan_info* info, uint64_t* chain_masks,
                                       uint64_t* cached_masks, int64_t* stage_memory) {
  if (world < 1 || !fams) return fail(REMAT_ERR_VALUE, "need at least one replica");
  for (int r = 0; r < world; r++)
    if (!fams[r]) return fail(REMAT_ERR_VALUE, "null family handle");
  if (nb < 1) return fail(REMAT_ERR_VALUE, "need at least one budget");
  if (objective != REMAT_MINIMIZE && objective != REMAT_MAXIMIZE)
    return fail(REMAT_ERR_VALUE, "objective must be minimize (0) or maximize (1)");
  remat_family_s* f0 = fams[0];
  remat_graph_s* g = f0->g;
  int rc;
  for (int r = 1; r < world; r++) {
    if ((rc = check_same(f0, fams[r])) < 0) return rc;
    if (fams[r]->g->device != g->device || fams[r]->g->stream != g->stream)
      return fail(REMAT_ERR_VALUE, "loopback replicas must share one graph handle");
  }
  RM_CUDA(cudaSetDevice(g->device));
  prepare_pool(g->device);
  tls_stream = g->stream;
  std::vector<long long> bs(nb);
  for (int b = 0; b < nb; b++) {
    if (budgets[b] < 0) return fail(REMAT_ERR_VALUE, "budget must be non-negative");
    bs[b] = std::min<long long>(budgets[b], 2 * g->MV);
  }
  for (int r = 0; r < world; r++)
    if ((rc = ensure_foff(fams[r])) < 0 || (rc = solve_begin(fams[r], bs, objective)) < 0)
      return rc;
  SegList sl;
  std::vector<Region> regs;
  std::vector<int> run;
  auto flush_run = [&]() {
    int r2 = REMAT_OK;
    for (int r = 0; r < world && r2 >= 0; r++) {
      std::vector<int> copy = run;
      r2 = relax_run(fams[r], copy);
    }
    run.clear();
    return r2;
  };
  for (int lvl = 1; lvl <= g->n; lvl++) {
    const long long j0 = f0->level_start[lvl], w = f0->level_start[lvl + 1] - j0;
    if (w == 0) continue;
    if (replicated(f0, lvl, nb)) {
      run.push_back(lvl);
      continue;
    }
    if ((rc = flush_run()) < 0) return rc;
    for (int r = 0; r < world; r++) {
      long long lo, hi;
      part(j0, w, world, r, &lo, &hi);
      if ((rc = solve_level(fams[r], lvl, lo, hi)) < 0) return rc;
    }
    if (world == 1) continue;
    // the "broadcasts": replica r's share copied straight into every other
    // replica's same regions
    for (int r = 0; r < world; r++) {
      long long lo, hi;
      part(j0, w, world, r, &lo, &hi);
      share_regions(fams[r], nb, lo, hi, regs);
      for (int q = 0; q < world; q++) {
        if (q == r) continue;
        for (const Region& x : regs)
          sl.add(array_base(fams[r], x.array) + x.off, array_base(fams[q], x.array) + x.off,
                 (long long)x.bytes);
      }
    }
    if ((rc = sl.flush(g->stream)) < 0) return rc;
  }
  if ((rc = flush_run()) < 0) return rc;
  // every replica now holds the whole table; finish on each, report replica 0
  std::vector<remat_plan_info> other(nb);
  for (int r = world - 1; r >= 1; r--) {
    if ((rc = solve_finish(fams[r], other.data(), nullptr, nullptr, nullptr)) < 0) return rc;
  }
  if ((rc = solve_finish(f0, info, (u64*)chain_masks, (u64*)cached_masks,
                         (long long*)stage_memory)) < 0)
    return rc;
  for (int b = 0; b < nb; b++) {
    if (world > 1 && (other[b].objective_value != info[b].objective_value ||
                      other[b].stats.transitions != info[b].stats.transitions ||
                      other[b].status != info[b].status))
      return fail(REMAT_ERR_INTERNAL, "level-sharded replicas disagree");
  }
  return finish_status(info, budgets, nb);
}

}  // extern "C"
