// family.cu — lower-set families and the per-member precompute (K1, K2, K3).
//
// K1 enumerate_full   replaces lattice.py:59-84 (all_lower_sets) + from_masks 44-47
// K2 closure_family   replaces graph.py:98-107 (closures) + lattice.py:87-93
// K3 member_terms     replaces planner.py:109-115 (boundary, stage_base) plus the
//                     per-member prefix terms of the pair constants
//
// K1 generates level s+1 from level s with the canonical-parent rule (SURVEY
// Appendix A.7): from lower set L emit L ∪ {v} iff v ∉ L, preds(v) ⊆ L and v is
// the largest-index maximal element of L ∪ {v}.  Every lower set is emitted
// exactly once, so no hash/dedup is needed; each level is then ranked by mask
// value, which reproduces the reference order (popcount, mask).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "device.cuh"

namespace remat {

template <int W>
__device__ __forceinline__ u64 pick(const u64 (&a)[W], int q) {
  u64 r = 0;
#pragma unroll
  for (int w = 0; w < W; w++)
    if (w == q) r = a[w];
  return r;
}

template <int W>
__device__ __forceinline__ bool has_bit(const u64 (&a)[W], int v) {
  return (pick<W>(a, v >> 6) >> (v & 63)) & 1ull;
}

// ---------------------------------------------------------------------------
// K1: full lattice, one level at a time
// ---------------------------------------------------------------------------

// Returns for lane's node v whether L ∪ {v} is a canonical child of L; on
// success fills the child's maximal-element set.
template <int W>
__device__ __forceinline__ bool canonical_child(const u64 (&L)[W], const u64 (&X)[W], int v,
                                                const u64* __restrict__ preds, u64 (&cx)[W]) {
  if (has_bit<W>(L, v)) return false;
  const u64* pv = preds + (size_t)v * W;
  u64 missing = 0;
  u64 p[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    p[w] = __ldg(pv + w);
    missing |= p[w] & ~L[w];
  }
  if (missing) return false;
  // highest maximal element of L that stays maximal in L ∪ {v}
  int hb = -1;
#pragma unroll
  for (int w = W - 1; w >= 0; w--) {
    u64 y = X[w] & ~p[w];
    if (hb < 0 && y) hb = w * 64 + 63 - __clzll((long long)y);
  }
  if (v < hb) return false;
#pragma unroll
  for (int w = 0; w < W; w++) cx[w] = (X[w] & ~p[w]) | ((w == (v >> 6)) ? (1ull << (v & 63)) : 0ull);
  return true;
}

#ifndef REMAT_RANK_TASKS
#define REMAT_RANK_TASKS 2
#endif
#ifndef REMAT_RANK_MIN_TILE
#define REMAT_RANK_MIN_TILE 4
#endif
constexpr long long kRankTasks = REMAT_RANK_TASKS;     // ranking tasks per block per level
constexpr long long kRankMinTile = REMAT_RANK_MIN_TILE;  // smallest comparison tile

// (popcount-equal) masks compared as little-endian multi-word integers
template <int W>
__device__ __forceinline__ bool mask_less(const u64* a, const u64* b) {
#pragma unroll
  for (int w = W - 1; w >= 0; w--)
    if (a[w] != b[w]) return a[w] < b[w];
  return false;
}

// ---------------------------------------------------------------------------
// K2: ancestor-closure family
// ---------------------------------------------------------------------------

// closure(v) = {v} ∪ ⋃ closure(preds(v)); preds have smaller indices, so one
// sweep in index order suffices (graph.py:98-107).  One warp, lane q owns word q.
// The closures are read back from shared memory, or (graphs above 1024 nodes,
// whose n·W words exceed it) from the output rows themselves: lane q reads
// only words it wrote.
template <int W>
__global__ void k_closures(const u64* __restrict__ preds, int n, u64* __restrict__ cand,
                           int in_smem) {
  extern __shared__ u64 clo_sm[];  // [n][W]
  u64* clo = in_smem ? clo_sm : cand + 2 * W;
  const int q = threadIdx.x;
  for (int v = 0; v < n; v++) {
    u64 c = (q == (v >> 6)) ? (1ull << (v & 63)) : 0ull;
    for (int w2 = 0; w2 < W; w2++) {
      u64 x = preds[(size_t)v * W + w2];
      while (x) {
        int u = w2 * 64 + __ffsll((long long)x) - 1;
        x &= x - 1;
        if (q < W) c |= clo[u * W + q];
      }
    }
    if (q < W) {
      if (in_smem) clo[v * W + q] = c;
      cand[(size_t)(v + 2) * W + q] = c;
    }
    __syncwarp();
  }
  if (q < W) {
    cand[q] = 0ull;  // ∅
    int lo = q * 64, cnt = n - lo;
    cand[W + q] = cnt >= 64 ? ~0ull : (cnt <= 0 ? 0ull : ((1ull << cnt) - 1));  // V
  }
}

template <int W>
__device__ __forceinline__ int popc_row(const u64* a) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < W; w++) c += __popcll(a[w]);
  return c;
}

// Deduplicate + order the n+2 candidates by (popcount, mask) (from_masks).
// Rows and flags live in shared memory, or — above 1024 nodes — stay in global
// memory (`scratch`: 2N ints).
template <int W>
__global__ void __launch_bounds__(1024) k_pruned_rank(const u64* __restrict__ cand, int N,
                                                      u64* __restrict__ out_rows,
                                                      long long* __restrict__ out_count,
                                                      int* __restrict__ scratch) {
  extern __shared__ u64 sm[];
  const u64* rows = scratch ? cand : sm;  // [N][W]
  int* keep = scratch ? scratch : reinterpret_cast<int*>(sm + (size_t)N * W);
  int* pcs = keep + N;
  if (!scratch)
    for (int e = threadIdx.x; e < N * W; e += blockDim.x) sm[e] = cand[e];
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x) pcs[e] = popc_row<W>(rows + e * W);
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int dup = 0;
    for (int k = 0; k < e && !dup; k++) {
      bool eq = true;
#pragma unroll
      for (int w = 0; w < W; w++) eq &= rows[k * W + w] == rows[e * W + w];
      dup = eq;
    }
    keep[e] = !dup;
  }
  __syncthreads();
  int local = 0;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    if (!keep[e]) continue;
    local++;
    long long rank = 0;
    for (int k = 0; k < N; k++) {
      if (!keep[k]) continue;
      bool less = pcs[k] != pcs[e] ? pcs[k] < pcs[e] : mask_less<W>(rows + k * W, rows + e * W);
      rank += less;
    }
#pragma unroll
    for (int w = 0; w < W; w++) out_rows[rank * W + w] = rows[e * W + w];
  }
  if (local) atomicAdd(reinterpret_cast<unsigned long long*>(out_count), (unsigned long long)local);
}

// ---------------------------------------------------------------------------
// K3: per-member terms
// ---------------------------------------------------------------------------

// One warp per member L (AoS row).  Produces ∂L (SoA), M(L), T(L), M(∂L),
// T(L\∂L) and stage_base = M(δ+(L)\L) + M(δ−(δ+(L)\L)\L)  (planner.py:110-115;
// restricting δ− to successors outside L is exact for lower sets, reference
// tests/test_strategy.py:97-107).
template <int W>
__global__ void k_member_terms(const u64* __restrict__ rows, long long F, GraphView g,
                               u64* __restrict__ bound_soa, long long* __restrict__ ML,
                               long long* __restrict__ TL, long long* __restrict__ Mb,
                               long long* __restrict__ TLnb, long long* __restrict__ base) {
  __shared__ u64 bsh[8][W];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (i >= F) return;
  u64 L[W], dp[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    L[w] = rows[i * W + w];
    dp[w] = 0;
  }
  if (lane < W) bsh[wib][lane] = 0;
  __syncwarp();
  long long ml = 0, tl = 0, mb = 0, tlnb = 0;
  for (int v0 = 0; v0 < g.n; v0 += 32) {
    int v = v0 + lane;
    bool isb = false;
    if (v < g.n && has_bit<W>(L, v)) {
      const u64* sv = g.succs + (size_t)v * W;
      u64 outside = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        u64 s = __ldg(sv + w);
        dp[w] |= s;
        outside |= s & ~L[w];
      }
      long long m = __ldg(g.M + v), t = __ldg(g.T + v);
      ml += m;
      tl += t;
      isb = outside != 0;
      if (isb) mb += m; else tlnb += t;
    }
    unsigned bal = __ballot_sync(kFull, isb);
    if (lane == 0) bsh[wib][v0 >> 6] |= (u64)bal << (v0 & 63);
  }
  ml = warp_sum(ml);
  tl = warp_sum(tl);
  mb = warp_sum(mb);
  tlnb = warp_sum(tlnb);
  u64 D[W], dm[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    D[w] = warp_or(dp[w]) & ~L[w];
    dm[w] = 0;
  }
  long long md = 0;
  for (int v0 = 0; v0 < g.n; v0 += 32) {
    int v = v0 + lane;
    if (v < g.n && has_bit<W>(D, v)) {
      md += __ldg(g.M + v);
      const u64* pv = g.preds + (size_t)v * W;
#pragma unroll
      for (int w = 0; w < W; w++) dm[w] |= __ldg(pv + w);
    }
  }
  md = warp_sum(md);
  u64 E[W];
#pragma unroll
  for (int w = 0; w < W; w++) E[w] = warp_or(dm[w]) & ~L[w];
  long long me = 0;
  for (int v0 = 0; v0 < g.n; v0 += 32) {
    int v = v0 + lane;
    if (v < g.n && has_bit<W>(E, v)) me += __ldg(g.M + v);
  }
  me = warp_sum(me);
  __syncwarp();
  if (lane < W) bound_soa[(size_t)lane * F + i] = bsh[wib][lane];
  if (lane == 0) {
    ML[i] = ml;
    TL[i] = tl;
    Mb[i] = mb;
    TLnb[i] = tlnb;
    base[i] = md + me;
  }
}

template <int W>
__global__ void k_to_soa(const u64* __restrict__ rows, long long F, u64* __restrict__ soa) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F) return;
#pragma unroll
  for (int w = 0; w < W; w++) soa[(size_t)w * F + i] = rows[i * W + w];
}

template <int W>
__global__ void k_popcount_hist(const u64* __restrict__ rows, long long F, long long* hist) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F) return;
  atomicAdd(reinterpret_cast<unsigned long long*>(hist + popc_row<W>(rows + i * W)), 1ull);
}

// frontier capacity of a member: T(L)+1 overhead values, or at most `cap`
// cells on the sparse-row path
__global__ void k_row_len(const long long* __restrict__ TL, long long F, long long* out,
                          long long cap) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < F) out[i] = min(TL[i] + 1, cap);
}

__global__ void k_level_max(const long long* __restrict__ TL, const long long* __restrict__ ls,
                            long long* __restrict__ out, long long cap) {
  __shared__ long long red[32];
  const int s = blockIdx.x;
  long long lo = ls[s], hi = ls[s + 1], mx = 0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) mx = max(mx, min(TL[i] + 1, cap));
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, m));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); k++) mx = max(mx, red[k]);
    out[s] = mx;
  }
}

// ---------------------------------------------------------------------------
// exclusive scan (int64)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(1024) k_scan_block(const long long* __restrict__ in,
                                                     long long* __restrict__ out, long long n,
                                                     long long* __restrict__ sums) {
  __shared__ long long scratch[33];
  long long i = (long long)blockIdx.x * 1024 + threadIdx.x;
  long long v = i < n ? in[i] : 0;
  long long tot;
  long long ex = block_exclusive_sum(v, scratch, &tot);
  if (i < n) out[i] = ex;
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_scan_add(long long* __restrict__ out, long long n,
                           const long long* __restrict__ offs) {
  long long i = (long long)blockIdx.x * 1024 + threadIdx.x;
  if (i < n) out[i] += offs[blockIdx.x];
}

static int scan_rec(const long long* in, long long* out, long long n, cudaStream_t s) {
  long long nb = (n + 1023) / 1024;
  long long* sums = nullptr;
  RM_CUDA(cudaMallocFromPoolAsync(&sums, sizeof(long long) * (nb + 1), tls_pool, s));
  k_scan_block<<<(unsigned)nb, 1024, 0, s>>>(in, out, n, sums);
  RM_LAUNCHED();
  if (nb > 1) {
    long long* soff = nullptr;
    RM_CUDA(cudaMallocFromPoolAsync(&soff, sizeof(long long) * (nb + 1), tls_pool, s));
    int rc = scan_rec(sums, soff, nb, s);
    if (rc < 0) return rc;
    k_scan_add<<<(unsigned)nb, 1024, 0, s>>>(out, n, soff);
    RM_LAUNCHED();
    RM_CUDA(cudaFreeAsync(soff, s));
  }
  RM_CUDA(cudaFreeAsync(sums, s));
  return REMAT_OK;
}

int scan_exclusive(const long long* in, long long* out, long long n, cudaStream_t s,
                   long long* total_host) {
  if (n <= 0) {
    if (total_host) *total_host = 0;
    return REMAT_OK;
  }
  int rc = scan_rec(in, out, n, s);
  if (rc < 0) return rc;
  if (total_host) {
    long long a = 0, b = 0;
    RM_CUDA(cudaMemcpyAsync(&a, out + n - 1, sizeof a, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(&b, in + n - 1, sizeof b, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    *total_host = a + b;
  }
  return REMAT_OK;
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------

// Narrow levels (a few dozen members: the long tails of deep lattices, C5)
// are walked by ONE block with members in shared memory and CTA barriers
// only: a grid barrier plus the L2 round trips of a grid step cost more than
// the whole level's candidate checks.  Block 0 ranks, scatters and expands
// level after level until a level gets wide (or V is reached) and returns the
// level to resume the grid walk at (-1: the lattice overflowed, status set).
// Level k+1 is also written to U[(k+1) % 3], where the grid walk expects it.
template <int W>
__device__ __noinline__ int enum_narrow_run(const u64* __restrict__ preds, int n, long long cap, long long fcap,
                               u64* __restrict__ fam, u64* __restrict__ U, long long ucap,
                               long long* __restrict__ ctr, long long* __restrict__ ls,
                               int* __restrict__ status, int k, long long base, int ncap,
                               long long work_cap, u64* __restrict__ sm) {
  __shared__ int s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = (n + 31) / 32;
  u64* cur = sm;
  u64* nxt = sm + (size_t)ncap * 2 * W;
  long long N = *((volatile long long*)(ctr + k));
  {
    const u64* g = U + (size_t)(k % 3) * ucap * 2 * W;
    for (long long e = tid; e < N * 2 * W; e += blockDim.x) cur[e] = g[e];
  }
  __syncthreads();
  while (true) {
    if (base + N > cap || base + N > fcap) {
      if (tid == 0) status[0] = base + N > cap ? 1 : 2;
      return -1;
    }
    if (tid == 0) ls[k] = base;
    // rank (all masks of a level are distinct) and scatter level k
    if (tid < N) {
      const u64* me = cur + (size_t)tid * 2 * W;
      long long r = 0;
      for (int q = 0; q < N; q++) r += mask_less<W>(cur + (size_t)q * 2 * W, me);
#pragma unroll
      for (int w = 0; w < W; w++) fam[(base + r) * W + w] = me[w];
    }
    if (k == n) {  // V has no children; the grid walk only closes ls
      if (tid == 0) ls[n + 1] = base + N;
      return n + 1;
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    // canonical children of level k
    const long long room = min(min(cap, fcap) - base - N, ucap);
    u64* gn = U + (size_t)((k + 1) % 3) * ucap * 2 * W;
    for (long long task = warp; task < N * nch; task += blockDim.x >> 5) {
      const long long p = task / nch;
      const int v = (int)(task - p * nch) * 32 + lane;
      u64 L[W], X[W], cx[W];
#pragma unroll
      for (int w = 0; w < W; w++) {
        L[w] = cur[p * 2 * W + w];
        X[w] = cur[p * 2 * W + W + w];
      }
      const bool ok = v < n && canonical_child<W>(L, X, v, preds, cx);
      const unsigned bal = __ballot_sync(kFull, ok);
      if (!bal) continue;
      int at0 = 0;
      if (lane == 0) at0 = atomicAdd(&s_cnt, __popc(bal));
      at0 = __shfl_sync(kFull, at0, 0);
      const int at = at0 + __popc(bal & ((1u << lane) - 1));
      if (ok) {
#pragma unroll
        for (int w = 0; w < W; w++) {
          const u64 cl = L[w] | ((w == (v >> 6)) ? (1ull << (v & 63)) : 0ull);
          if (at < room) {
            gn[(size_t)at * 2 * W + w] = cl;
            gn[(size_t)at * 2 * W + W + w] = cx[w];
          }
          if (at < ncap) {
            nxt[(size_t)at * 2 * W + w] = cl;
            nxt[(size_t)at * 2 * W + W + w] = cx[w];
          }
        }
      }
    }
    __syncthreads();
    const long long N1 = s_cnt;
    if (tid == 0) ctr[k + 1] = N1;
    base += N;
    k++;
    u64* t = cur;
    cur = nxt;
    nxt = t;
    N = N1;
    __syncthreads();
    if (N > ncap || N * n > work_cap) {
      if (tid == 0) ls[k] = base;
      return k;  // wide again: the grid walk resumes at level k (in U[k % 3])
    }
  }
}

// K1 as ONE cooperative launch with one grid barrier per level (SURVEY §7
// hard part 5: n = 516 dependent levels at C5).  Level k's members sit
// UNSORTED (mask + maximal-element set) in buffer U[k % 3].  Grid step k runs
// three independent jobs, load-balanced over every block:
//   (a) canonical children of level k, one (member, 32-node chunk) task per
//       warp, appended to U[(k+1) % 3] at atomically reserved positions (the
//       emission order is irrelevant: the level is ranked afterwards);
//   (b) partial ranks of level k: (element tile, comparison tile) tasks of
//       256 x 256 mask comparisons, atomically summed into rank[k % 3]
//       (rank(i) = #{q : mask_q < mask_i}, all masks of a level distinct);
//   (c) scatter of level k-1 into the family at ls[k-1] + rank, using the
//       ranks completed in step k-1.
// Buffers rotate over three slots, so each is written one step after its
// last reader finished.  Runs of narrow levels go to enum_narrow_run (block 0
// alone, the others wait at one grid barrier).
//   ctr[k]    |level k| (ctr[0] = 1: the empty set, pre-set by the host)
//   status[0] 1 when the lattice exceeds `cap` (LatticeTooLargeError), 2 when
//             it exceeds the buffers' capacity `fcap` (< cap): grow and rerun;
//   status[1] the level a narrow run hands back
#ifdef REMAT_ENUM_TRACE
__device__ unsigned long long g_enum_trace[600 * 148 * 4];
extern "C" __attribute__((visibility("default"))) int remat_debug_enum_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_enum_trace, sizeof(g_enum_trace)) == cudaSuccess ? 0 : -1;
}
#endif
template <int W>
__global__ void __launch_bounds__(256) k_enum_all(const u64* __restrict__ preds, int n,
                                                  long long cap, long long fcap,
                                                  u64* __restrict__ fam,
                                                  u64* __restrict__ U, long long ucap,
                                                  unsigned* __restrict__ rank,
                                                  long long* __restrict__ ctr,
                                                  long long* __restrict__ ls,
                                                  int* __restrict__ status, int ncap,
                                                  long long work_cap) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // comparison tile of the ranking step (48 KB static shared memory at most)
  constexpr int kRT = W <= 16 ? 256 : 64;
  __shared__ u64 tile[kRT * W];
  extern __shared__ u64 narrow_sm[];  // [2][ncap][2W]
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * 8;
  const long long gw = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const long long gt = (long long)blockIdx.x * 256 + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * 256;
  const int nch = (n + 31) / 32;
  long long base = 0, prev_base = 0, prevN = 0;  // ls[k], ls[k-1], |level k-1|
  for (int k = 0; k <= n + 1;) {
    long long N = k <= n ? *((volatile long long*)(ctr + k)) : 0;
    if (base + N > cap || base + N > fcap) {  // uniform: every block read the same counters
      if (blockIdx.x == 0 && threadIdx.x == 0) status[0] = base + N > cap ? 1 : 2;
      return;
    }
    const unsigned* rkp = rank + (size_t)((k + 2) % 3) * ucap;
    const u64* prv = U + (size_t)((k + 2) % 3) * ucap * 2 * W;
    if (k <= n && N <= ncap && N * n <= work_cap) {
      // narrow run: finish level k-1's scatter here, block 0 takes over
      for (long long i = gt; i < prevN; i += nthreads) {
        const long long at = prev_base + rkp[i];
        const_cast<unsigned*>(rkp)[i] = 0;
#pragma unroll
        for (int w = 0; w < W; w++) fam[at * W + w] = prv[i * 2 * W + w];
      }
      if (blockIdx.x == 0) {
        const int kr = enum_narrow_run<W>(preds, n, cap, fcap, fam, U, ucap, ctr, ls, status, k,
                                          base, ncap, work_cap, narrow_sm);
        if (threadIdx.x == 0) status[1] = kr;
      }
      grid.sync();
      const int kr = *((volatile int*)(status + 1));
      if (kr < 0) return;
      base = *((volatile long long*)(ls + kr));
      prevN = 0;
      k = kr;
      if (k > n) break;
      continue;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && k <= n) ls[k] = base;
    const u64* cur = U + (size_t)(k % 3) * ucap * 2 * W;   // [N][2W]
    u64* nxt = U + (size_t)((k + 1) % 3) * ucap * 2 * W;
    unsigned* rk = rank + (size_t)(k % 3) * ucap;
    const long long room = min(min(cap, fcap) - base - N, ucap);  // children that fit
#ifdef REMAT_ENUM_TRACE  // per-level phase timestamps (tools/enum_trace.py)
    auto stamp = [&](int ph) {
      if (threadIdx.x == 0 && k < 600) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_enum_trace[((size_t)k * 148 + (blockIdx.x % 148)) * 4 + ph] = t;
      }
    };
    stamp(0);
#endif
    // (c) scatter level k-1, leaving its rank slot zeroed for level k+2
    for (long long i = gt; i < prevN; i += nthreads) {
      const long long at = prev_base + rkp[i];
      const_cast<unsigned*>(rkp)[i] = 0;
#pragma unroll
      for (int w = 0; w < W; w++) fam[at * W + w] = prv[i * 2 * W + w];
    }
#ifdef REMAT_ENUM_TRACE
    stamp(1);
#endif
    // (a) canonical children of level k
    if (k < n)
      for (long long task = gw; task < N * nch; task += nwarps) {
        const long long p = task / nch;
        const int v = (int)(task - p * nch) * 32 + lane;
        u64 L[W], X[W], cx[W];
#pragma unroll
        for (int w = 0; w < W; w++) {
          L[w] = cur[p * 2 * W + w];
          X[w] = cur[p * 2 * W + W + w];
        }
        const bool ok = v < n && canonical_child<W>(L, X, v, preds, cx);
        const unsigned bal = __ballot_sync(kFull, ok);
        if (!bal) continue;
        unsigned long long at0 = 0;
        if (lane == 0)
          at0 = atomicAdd(reinterpret_cast<unsigned long long*>(ctr + k + 1),
                          (unsigned long long)__popc(bal));
        at0 = __shfl_sync(kFull, at0, 0);
        const long long at = (long long)at0 + __popc(bal & ((1u << lane) - 1));
        if (ok && at < room) {
#pragma unroll
          for (int w = 0; w < W; w++) {
            nxt[at * 2 * W + w] = L[w] | ((w == (v >> 6)) ? (1ull << (v & 63)) : 0ull);
            nxt[at * 2 * W + W + w] = cx[w];
          }
        }
      }
#ifdef REMAT_ENUM_TRACE
    stamp(2);
#endif
    // (b) partial ranks of level k over (element tile, comparison tile) tasks
    if (k <= n) {
      // comparison tiles narrow enough for ~2 tasks per block: a level of a
      // few hundred members would otherwise rank on a handful of blocks while
      // the rest wait at the barrier (C5 p=0.2: ranking was 15.8 of the 17.5
      // ms enumeration, 50 us per level on 4 of 148 blocks)
      const long long nt = (N + 255) / 256;
      long long C = kRT;
      while (C > kRankMinTile && nt * ((N + C - 1) / C) < kRankTasks * (long long)gridDim.x) C >>= 1;
      const long long ntc = (N + C - 1) / C;
      // (from the last block down: when the level is narrow the first blocks
      // carry the emission tasks, so ranking runs beside them, not after)
      for (long long task = gridDim.x - 1 - blockIdx.x; task < nt * ntc; task += gridDim.x) {
        const long long it = task / ntc, tt = task - it * ntc;
        const long long i = it * 256 + threadIdx.x, t0 = tt * C;
        const long long c = min(C, N - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < c * W; e += 256) {
          const long long q = e / W;
          tile[e] = cur[(t0 + q) * 2 * W + (e - q * W)];
        }
        __syncthreads();
        if (i < N) {
          u64 me[W];
#pragma unroll
          for (int w = 0; w < W; w++) me[w] = cur[i * 2 * W + w];
          unsigned r = 0;
          for (int q = 0; q < c; q++) r += mask_less<W>(tile + q * W, me);
          if (r) atomicAdd(rk + i, r);
        }
      }
    }
    prev_base = base;
    prevN = k <= n ? N : 0;
    base += N;
#ifdef REMAT_ENUM_TRACE
    __syncthreads();
    stamp(3);
#endif
    grid.sync();
    k++;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ls[n + 1] = base;
}

template <int W>
static int enumerate_full(remat_graph_s* g, long long cap, DevBuf<u64>& fam,
                          std::vector<long long>& level_start) {
  cudaStream_t s = g->stream;
  const int n = g->n;
  // Buffers start at min(cap, 256 K members) and grow 4x (rerun) only when the
  // lattice outgrows them below the cap; the three level buffers hold one
  // level each, and no level is wider than C(n, n/2) nor than the family.
  const long long capn = std::max<long long>(cap, n + 1);
  // (256 K members: every named config fits the first pass; buffers sized for
  // millions of members made every small family build churn ~1 GB of pool
  // memory against the solver's own tables)
  long long fcap = std::min<long long>(capn, 256LL << 10);
  if (const char* e = getenv("REMAT_ENUM_INIT_CAP"))  // test hook for the grow path
    fcap = std::min<long long>(capn, std::max<long long>(n + 1, atoll(e)));
  long double binom = 1;
  for (int i = 1; i <= n / 2; i++) binom = binom * (n - n / 2 + i) / i;
  int rc;
  DevBuf<u64> U;
  DevBuf<unsigned> rank;
  DevBuf<int> status;
  DevBuf<long long> ctr, ls;
  const int num_sms = sm_count(g->device);
  // narrow levels (<= ncap members and <= work_cap candidate checks) run in
  // one block with the level in shared memory (enum_narrow_run)
  const int ncap = (int)std::min<size_t>(96, (40u << 10) / (2 * 2 * W * sizeof(u64)));
  const size_t nsm = (size_t)2 * ncap * 2 * W * sizeof(u64);
  long long work_cap = 1024;  // chain-like levels (DenseNet: 2.1 -> 1.2 ms); C5 keeps the grid walk
  if (const char* e = getenv("REMAT_ENUM_NARROW_WORK"))  // tuning / test hook (0: off)
    work_cap = atoll(e);
  static bool attr[kMaxDevices] = {};
  if (!attr[dev_slot(g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(k_enum_all<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)nsm));
    attr[dev_slot(g->device)] = true;
  }
  int bps = 0;
  RM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_enum_all<W>, 256, nsm));
  if (bps < 1) return fail(REMAT_ERR_CUDA, "enumeration kernel cannot be resident");
  // one block per SM keeps the per-level grid barrier cheap
  const int nblk = num_sms;
  if ((rc = ctr.ensure(n + 2)) < 0 || (rc = ls.ensure(n + 2)) < 0 || (rc = status.ensure(2)) < 0)
    return rc;
  while (true) {
    const long long ucap = (long long)std::min<long double>((long double)fcap, binom + 1);
    if ((rc = fam.ensure((size_t)fcap * W)) < 0 || (rc = U.ensure((size_t)3 * ucap * 2 * W)) < 0 ||
        (rc = rank.ensure((size_t)3 * ucap)) < 0)
      return rc;
    RM_CUDA(cudaMemsetAsync(U.p, 0, sizeof(u64) * 2 * W, s));  // the empty set, no maximal elements
    RM_CUDA(cudaMemsetAsync(rank.p, 0, sizeof(unsigned) * 3 * ucap, s));
    RM_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(long long) * (n + 2), s));
    RM_CUDA(cudaMemsetAsync(status.p, 0, 2 * sizeof(int), s));
    const long long one = 1;
    RM_CUDA(cudaMemcpyAsync(ctr.p, &one, sizeof one, cudaMemcpyHostToDevice, s));
    const u64* preds = g->preds.p;
    u64 *a0 = fam.p, *a1 = U.p;
    long long uc = ucap, fc = fcap;
    unsigned* a2 = rank.p;
    long long *a3 = ctr.p, *a4 = ls.p;
    int* a5 = status.p;
    int nn = n, nc = ncap;
    long long cp = cap, wc = work_cap;
    void* args[] = {(void*)&preds, &nn, &cp, &fc, &a0, &a1, &uc, &a2, &a3, &a4, &a5, &nc, &wc};
    RM_CUDA(cudaLaunchCooperativeKernel((const void*)k_enum_all<W>, dim3(nblk), dim3(256), args,
                                        nsm, s));
    RM_LAUNCHED();
    int st = 0;
    level_start.assign(n + 2, 0);
    RM_CUDA(cudaMemcpyAsync(&st, status.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(level_start.data(), ls.p, sizeof(long long) * (n + 2),
                            cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    if (st == 1)
      return fail(REMAT_ERR_LATTICE, "lattice too large: more than " + std::to_string(cap) +
                                         " lower sets; raise the cap or use the pruned family");
    if (st == 0) return REMAT_OK;
    fcap = std::min<long long>(capn, fcap * 4);  // outgrew the buffers: grow and rerun
  }
}

template <int W>
static int enumerate_pruned(remat_graph_s* g, DevBuf<u64>& fam, long long* Fout) {
  cudaStream_t s = g->stream;
  const int n = g->n, N = n + 2;
  DevBuf<u64> cand;
  DevBuf<long long> cnt;
  int rc;
  if ((rc = cand.ensure((size_t)N * W)) < 0 || (rc = fam.ensure((size_t)N * W)) < 0 ||
      (rc = cnt.ensure(1)) < 0)
    return rc;
  constexpr size_t kSm = 200 << 10;  // dynamic shared memory used at most
  size_t sm1 = sizeof(u64) * n * W;
  const int clo_smem = sm1 <= kSm;
  if (!clo_smem) sm1 = 0;
  RM_CUDA(cudaFuncSetAttribute(k_closures<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(sm1, 1)));
  k_closures<W><<<1, 32, sm1, s>>>(g->preds.p, n, cand.p, clo_smem);
  RM_LAUNCHED();
  size_t sm2 = sizeof(u64) * N * W + 2 * sizeof(int) * N;
  DevBuf<int> scratch;
  if (sm2 > kSm) {
    if ((rc = scratch.ensure((size_t)2 * N)) < 0) return rc;
    sm2 = 0;
  }
  RM_CUDA(cudaFuncSetAttribute(k_pruned_rank<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(sm2, 1)));
  RM_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(long long), s));
  k_pruned_rank<W><<<1, 1024, sm2, s>>>(cand.p, N, fam.p, cnt.p, sm2 ? nullptr : scratch.p);
  RM_LAUNCHED();
  RM_CUDA(cudaMemcpyAsync(Fout, cnt.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  return REMAT_OK;
}

template <int W>
static int build_family_w(remat_graph_s* g, int kind, long long cap, remat_family_s* f) {
  cudaStream_t s = g->stream;
  Events& ev = g->ev;
  RM_CUDA(cudaEventRecord(ev.e[0], s));
  DevBuf<u64> aos;
  int rc;
  long long F = 0;
  if (kind == REMAT_FAMILY_FULL) {
    rc = enumerate_full<W>(g, cap, aos, f->level_start);
    if (rc < 0) return rc;
    F = f->level_start.back();
  } else {
    rc = enumerate_pruned<W>(g, aos, &F);
    if (rc < 0) return rc;
  }
  f->F = F;
  RM_CUDA(cudaEventRecord(ev.e[1], s));
  if ((rc = f->masks.ensure((size_t)F * W)) < 0 || (rc = f->bound.ensure((size_t)F * W)) < 0 ||
      (rc = f->ML.ensure(F)) < 0 || (rc = f->TL.ensure(F)) < 0 || (rc = f->Mb.ensure(F)) < 0 ||
      (rc = f->TLnb.ensure(F)) < 0 || (rc = f->base.ensure(F)) < 0 ||
      (rc = f->foff.ensure(F + 1)) < 0)
    return rc;
  k_to_soa<W><<<(unsigned)((F + 255) / 256), 256, 0, s>>>(aos.p, F, f->masks.p);
  RM_LAUNCHED();
  k_member_terms<W><<<(unsigned)((F + 7) / 8), 256, 0, s>>>(aos.p, F, g->view(), f->bound.p,
                                                            f->ML.p, f->TL.p, f->Mb.p,
                                                            f->TLnb.p, f->base.p);
  RM_LAUNCHED();
  const int n = g->n;
  DevBuf<long long> tmp, lsd, lmax;
  if ((rc = tmp.ensure(std::max<long long>(F, n + 2))) < 0 || (rc = lsd.ensure(n + 2)) < 0 ||
      (rc = lmax.ensure(n + 1)) < 0)
    return rc;
  if (kind == REMAT_FAMILY_PRUNED) {
    RM_CUDA(cudaMemsetAsync(tmp.p, 0, sizeof(long long) * (n + 1), s));
    k_popcount_hist<W><<<(unsigned)((F + 255) / 256), 256, 0, s>>>(aos.p, F, tmp.p);
    RM_LAUNCHED();
    std::vector<long long> hist(n + 1);
    RM_CUDA(cudaMemcpyAsync(hist.data(), tmp.p, sizeof(long long) * (n + 1),
                            cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    f->level_start.assign(n + 2, 0);
    for (int l = 0; l <= n; l++) f->level_start[l + 1] = f->level_start[l] + hist[l];
  }
  RM_CUDA(cudaMemcpyAsync(lsd.p, f->level_start.data(), sizeof(long long) * (n + 2),
                          cudaMemcpyHostToDevice, s));
  const long long rcap = f->sparse ? f->fcap : LLONG_MAX;
  k_level_max<<<n + 1, 256, 0, s>>>(f->TL.p, lsd.p, lmax.p, rcap);
  RM_LAUNCHED();
  k_row_len<<<(unsigned)((F + 255) / 256), 256, 0, s>>>(f->TL.p, F, tmp.p, rcap);
  RM_LAUNCHED();
  long long slots = 0;
  if ((rc = scan_exclusive(tmp.p, f->foff.p, F, s, &slots)) < 0) return rc;
  RM_CUDA(cudaMemcpyAsync(f->foff.p + F, &slots, sizeof(long long), cudaMemcpyHostToDevice, s));
  f->slots = slots;
  f->level_maxR.assign(n + 1, 0);
  RM_CUDA(cudaMemcpyAsync(f->level_maxR.data(), lmax.p, sizeof(long long) * (n + 1),
                          cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaEventRecord(ev.e[2], s));
  RM_CUDA(cudaStreamSynchronize(s));
  float a = 0, b = 0;
  cudaEventElapsedTime(&a, ev.e[0], ev.e[1]);
  cudaEventElapsedTime(&b, ev.e[1], ev.e[2]);
  f->timings.enumerate_ms = a;
  f->timings.precompute_ms = b;
  return REMAT_OK;
}

int build_family(remat_graph_s* g, int kind, long long cap, remat_family_s* f) {
  // The DP keeps a dense overhead row per member (capacity T(L)+1, 32-bit t)
  // while T(V) < 2^24; above that (FLOP-valued compute costs) the cells of a
  // member are keyed by their overhead value instead (relax_sparse.cuh), at
  // most REMAT_SPARSE_CELLS (default 4096) distinct values per member.
  f->sparse = g->TV + 1 > (1LL << 24);
  if (const char* e = getenv("REMAT_FORCE_SPARSE"))  // test hook: the sparse path on any graph
    if (e[0] == '1') f->sparse = 1;
  if (f->sparse) {
    // distinct overhead values per cell (hash capacity, transient per target)
    // and frontier slots per member (persistent)
    const char* e = getenv("REMAT_SPARSE_CELLS");
    const long long h = e ? atoll(e) : (1 << 20);
    int p = 64;
    while (p < h && p < (1 << 22)) p <<= 1;
    f->hcap = p;
    const char* fr = getenv("REMAT_SPARSE_FRONTIER");
    f->fcap = std::max<long long>(2, fr ? atoll(fr) : 4096);
  }
  int rc = fail(REMAT_ERR_VALUE, "unsupported word count");
  f->g = g;
  f->kind = kind;
  dispatch_words(g->Wp, [&](auto wc) {
    constexpr int W = decltype(wc)::value;
    rc = build_family_w<W>(g, kind, cap, f);
  });
  if (rc < 0) return rc;
  // packed row keys (m << IB | parent) need M(V) < 2^(64-IB)
  int ib = 1;
  while ((1LL << ib) < f->F) ib++;
  f->IB = ib;
  if (!f->sparse && (ib >= 62 || (unsigned long long)g->MV >= ((~0ull) >> ib) - 1)) {
    // byte-valued memory costs on a big family: no packed 64-bit key holds
    // (m << IB) | i — the sparse-cell path keeps m and i apart (its frontier
    // slots stay the dense capacities T(L)+1 computed above)
    f->sparse = 1;
    f->hcap = 1 << 20;
    if (const char* e = getenv("REMAT_SPARSE_CELLS")) {
      int p = 64;
      while (p < atoll(e) && p < (1 << 22)) p <<= 1;
      f->hcap = p;
    }
  }
  // 32-bit keys hold (m2 << IB) | i for every m2 <= M(V) strictly below the
  // empty-slot sentinel 0xffffffff
  f->narrow = ((unsigned long long)(g->MV + 1) << ib) < (1ull << 32) && !f->sparse;
  if (const char* e = getenv("REMAT_FORCE_WIDE"))
    if (e[0] == '1') f->narrow = 0;
  return REMAT_OK;
}

}  // namespace remat
