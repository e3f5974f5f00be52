// internal.h — shared host/device declarations of libremat_b200.so.
//
// Layout in HBM (see DESIGN.md §Data layout):
//   graph:   preds/succs [n][Wp] u64 (AoS: a node's set is one 8·Wp-byte row),
//            T/M int64[n], weight-class masks [K][Wp]
//   family:  masks/bound SoA [Wp][F] u64 (word w of member i at w*F+i, so a
//            warp reading 32 consecutive members' word w is one coalesced
//            256-byte transaction), per-member int64 scalars ML, TL, Mb, TLnb,
//            base, frontier slot offsets foff[F+1]
//   DP:      per budget b: frontier entries in slots
//            [b*slots + foff[j], b*slots + foff[j+1]) — capacity T(L_j)+1, the
//            dense row length.  Entries are 8 B {t:u32, m:u32} when the packed
//            row key (m << IB | i) fits 32 bits ("narrow", every named config),
//            else 16 B {t:u32, pad, m:i64}; back-pointers live in a parallel
//            int32 array (read only by reconstruction).  Per (budget, member):
//            flen, ccount, mmin (smallest m = last stored entry), trans, npairs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <type_traits>
#include <vector>

#include "../../include/remat_b200.h"

typedef unsigned long long u64;

namespace remat {

constexpr int kMaxWords = 32;        // n <= 2048
constexpr int kMaxClasses = 32;      // weight classes per cost vector
constexpr int kRelaxThreads = 256;
constexpr int kRelaxWarps = kRelaxThreads / 32;

// One non-dominated DP entry (t, m) of a member (DpTable.opt, reference
// planner.py:82-92); the back-pointer (DpTable.parent) is stored apart.
struct __align__(8) EntryN {   // narrow: one LDG.64
  unsigned t;  // accumulated overhead
  unsigned m;  // cached memory
};
struct __align__(16) EntryW {  // wide: one LDG.128 (64-bit t for the sparse-row path)
  unsigned long long t;
  long long m;
};

// Words per set, padded to an instantiated width.
inline int padded_words(int w) {
  static const int kW[] = {1, 2, 3, 4, 6, 8, 9, 12, 16, 24, 32};
  for (int x : kW)
    if (x >= w) return x;
  return -1;
}

template <typename F>
void dispatch_words(int Wp, F&& f) {
  switch (Wp) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 9: f(std::integral_constant<int, 9>{}); break;
    case 12: f(std::integral_constant<int, 12>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    case 24: f(std::integral_constant<int, 24>{}); break;
    case 32: f(std::integral_constant<int, 32>{}); break;
    default: break;
  }
}

struct Status {
  int code = REMAT_OK;
  std::string msg;
  bool ok() const { return code >= 0; }
};

// Facts and one-time setup CUDA keeps per device (SM count, kernel function
// attributes) are cached per device id: one process may drive several GPUs.
constexpr int kMaxDevices = 64;
inline int dev_slot(int device) { return device >= 0 && device < kMaxDevices ? device : 0; }
int sm_count(int device);

void set_error(int code, const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define RM_CUDA(call)                                           \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return ::remat::cuda_fail(_e, #call); \
  } while (0)

#define RM_LAUNCHED()                                               \
  do {                                                              \
    ::remat::count_launch();                                        \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::remat::cuda_fail(_e, "launch"); \
  } while (0)

// ---------------------------------------------------------------------------
// device-side views passed to kernels by value
// ---------------------------------------------------------------------------

struct GraphView {
  int n, Wp;
  const u64* preds;   // [n][Wp]
  const u64* succs;   // [n][Wp]
  const long long* T; // [n]
  const long long* M; // [n]
};

struct FamilyView {
  long long F;
  const u64* masks;  // SoA [Wp][F]
  const u64* bound;  // SoA [Wp][F]
  const long long *ML, *TL, *Mb, *TLnb, *base;
  const long long* foff;  // [F+1]
};

struct ClassView {
  int enabled;                    // 0 -> class path unavailable (> kMaxClasses)
  int K;                          // classes: T(X) = Σ_c coef[c][0]·popc(X ∩ cls_c),
  const u64* cls;                 // [K][Wp]  M(X) = Σ_c coef[c][1]·popc(X ∩ cls_c)
  const long long* coef;          // [K][2]
};

struct DpView {
  long long slots;           // frontier slots per budget
  void* fe;                  // [nb][slots] EntryN or EntryW
  int* parent;               // [nb][slots] family index of the predecessor cell
  int* flen;                 // [nb][F] |frontier|
  int* ccount;               // [nb][F] |cell| (table entries)
  long long* mmin;           // [nb][F] smallest m of the frontier (LLONG_MAX if empty)
  u64* trans;                // [nb][F] Σ |frontier_i| over comparable predecessors
  u64* npairs;               // [nb][F] comparable predecessors (P)
  const long long* budgets;  // [nb] (clamped to 2*M(V))
  int IB;                    // parent-index bits in packed row keys
  int maximize;
};

// ---------------------------------------------------------------------------
// host handles
// ---------------------------------------------------------------------------

// Stream the current API call works on, and the library's PRIVATE memory pool
// of the current device: DevBuf allocations are stream-ordered
// (cudaMallocFromPoolAsync) from a pool whose release threshold is raised so
// freed blocks are reused across solves.  Being private, it never changes the
// behaviour of the device's default pool that other libraries in the process
// (PyTorch's cudaMallocAsync backend, CuPy) allocate from; remat_family_free
// trims it back to pool_keep_bytes() (32 GiB of the 180 GB by default).
extern thread_local cudaStream_t tls_stream;
extern thread_local cudaMemPool_t tls_pool;
constexpr size_t kPoolKeepBytes = size_t(32) << 30;  // REMAT_POOL_KEEP_GB overrides
size_t pool_keep_bytes();
cudaMemPool_t prepare_pool(int device);

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, tls_stream);
    p = nullptr;
    n = 0;
  }
  int ensure(size_t count) {
    if (count <= n && p) return REMAT_OK;
    release();
    size_t c = count ? count : 1;
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), c * sizeof(T), tls_pool,
                                            tls_stream);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return fail(REMAT_ERR_NOMEM, "device allocation of " + std::to_string(c * sizeof(T)) +
                                       " bytes failed: " + cudaGetErrorString(e));
    }
    n = c;
    return REMAT_OK;
  }
};

struct Events {
  cudaEvent_t e[8] = {};
  int create();
  void destroy();
};

}  // namespace remat

struct remat_graph_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int n = 0, W = 0, Wp = 0;
  long long TV = 0, MV = 0, maxM = 0;
  remat::DevBuf<u64> preds, succs;
  remat::DevBuf<long long> T, M;
  // weight classes for the popcount form of T(X) / M(X)
  int cls_enabled = 0, K = 0;
  remat::DevBuf<u64> cls;
  remat::DevBuf<long long> coef;
  std::vector<long long> hT, hM;
  std::vector<int> indeg, outdeg;  // host copies: exact event counts of schedules
  long long edges = 0;
  void* sched = nullptr;           // K7 scratch (schedule.cu), freed with the graph
  int t_uniform = 0;  // every T_v equal: candidates of a warp collide on few row slots
  // evaluate / simulate scratch
  remat::DevBuf<u64> chain_buf, bound_buf, cached_buf;
  remat::DevBuf<long long> terms_buf, eval_out, stage_buf;
  remat::DevBuf<int> int_buf;
  remat::DevBuf<long long> ll_buf;
  remat::DevBuf<int> ops_buf;
  remat::Events ev;

  remat::GraphView view() const {
    return remat::GraphView{n, Wp, preds.p, succs.p, T.p, M.p};
  }
  remat::ClassView classes() const {
    return remat::ClassView{cls_enabled, K, cls.p, coef.p};
  }
};

struct remat_family_s {
  remat_graph_s* g = nullptr;
  int kind = 0;
  long long F = 0;
  int IB = 1;
  remat::DevBuf<u64> masks, bound;              // SoA [Wp][F]
  remat::DevBuf<long long> ML, TL, Mb, TLnb, base, foff;
  long long slots = 0;
  std::vector<long long> level_start;           // [n+2]
  std::vector<long long> h_foff;                // host copy of foff (level sharding)
  std::vector<long long> level_maxR;            // [n+1]
  // DP state for up to nb_cap budgets
  int narrow = 0;                               // 32-bit row keys + 8 B entries
  // sparse-row path (T(V) >= 2^24: a dense overhead row per member no longer
  // fits): cells keyed by their overhead value, at most `hcap` per member
  int sparse = 0, hcap = 0;
  long long fcap = 0;
  remat::DevBuf<int> sparse_err;                // 1: a cell outgrew hcap, 2: a frontier its slots
  remat::DevBuf<u64> sparse_scratch;            // global cells when hcap exceeds shared memory
  remat::DevBuf<unsigned char> fe;
  remat::DevBuf<int> parent, flen, ccount;
  remat::DevBuf<long long> mmin, budgets, results;
  remat::DevBuf<u64> trans, npairs;
  remat::DevBuf<unsigned> ctr;                  // per-tile chunk + done counters (zero)
  remat::DevBuf<unsigned char> levelargs;       // TileArgs of a batched level run
  size_t ctr_cap = 0, grow_cap = 0;             // capacities of ctr / rowscratch (INF rows)
  int grow_key = 0;                             // key size rowscratch was filled for
  remat::DevBuf<u64> rowscratch, chain_out, cached_out;
  remat::DevBuf<long long> stage_out, terms;
  remat::DevBuf<int> chain_idx;
  remat::DevBuf<u64> stage_bound;
  remat_timings timings{};
  // the solve in flight (solve_begin .. solve_finish)
  int cur_nb = 0, cur_objective = 0, cur_narrow = 0;
  long long launches0 = 0, relax_launches = 0;

  remat::DpView dp_view() const {
    return remat::DpView{slots,    fe.p,     parent.p,  flen.p,  ccount.p, mmin.p,
                         trans.p, npairs.p, budgets.p, IB, cur_objective == REMAT_MAXIMIZE};
  }
  remat::FamilyView view() const {
    return remat::FamilyView{F, masks.p, bound.p, ML.p, TL.p, Mb.p, TLnb.p, base.p, foff.p};
  }
};

namespace remat {

// family.cu
int build_family(remat_graph_s* g, int kind, long long cap, remat_family_s* f);
int scan_exclusive(const long long* in, long long* out, long long n, cudaStream_t s,
                   long long* total_host);

// relax.cu: a solve is begin, one call per level (targets [lo, hi) of the
// level), finish; solve_batch runs all levels on one device
int solve_begin(remat_family_s* f, const std::vector<long long>& budgets, int objective);
int solve_level(remat_family_s* f, int lvl, long long lo, long long hi);
int solve_levels(remat_family_s* f, const std::vector<int>& lvls);  // full ranges, batched
// rows (chain, cached, stage memory; n+1 each, unpadded words) of budget b of
// the last solve, still on the device
int plan_rows(remat_family_s* f, int b, u64* chain_masks, u64* cached_masks,
              long long* stage_memory);
int solve_finish(remat_family_s* f, remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                 long long* stage_memory);
int solve_batch(remat_family_s* f, const std::vector<long long>& budgets, int objective,
                remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                long long* stage_memory);

// evaluate.cu: per-stage terms of chains already on device ([nb][n+1][Wp]);
// results [nb][8]: status, k, overhead, peak, cached_total, stagewise, tstar, mfinal
int evaluate_chains(remat_graph_s* g, int nb, const u64* chains, const int* klen,
                    const long long* expect /*[nb][4] tstar,mfinal,budget,check or null*/,
                    long long* stage_mem, u64* cached_masks, long long* results,
                    long long* terms, u64* bounds);

// api.cu: make the graph's device / stream / pool current for this thread
int graph_enter(remat_graph_s* g);

// schedule.cu (K7)
void free_sched_scratch(remat_graph_s* g);

}  // namespace remat
