// relax_impl.cuh — kernels and per-width host drivers of the relaxation
// (see relax.cu for the design notes).  Included by the relax_w*.cu
// translation units, each instantiating one bitset width, so the nine
// widths compile in parallel.
#pragma once
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <utility>

#include "device.cuh"

namespace remat {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// resident CTAs of the wide-bitset relaxation kernel (register cap 64; a
// 16-byte spill at W = 9; 3 CTAs at 80 registers measured 1 % slower)
#ifndef REMAT_TILE3_BLOCKS
#define REMAT_TILE3_BLOCKS 4
#endif
constexpr int kTile3MinBlocks = REMAT_TILE3_BLOCKS;
// per-target mask rows in shared memory: wide odd widths padded to an even
// word count, so a row is read with 16-byte loads (two words per LDS.128)
template <int W>
__host__ __device__ constexpr int mask_stride() { return W >= 4 ? (W + 1) & ~1 : W; }
constexpr int kMaxTJ = 32;   // targets per tile at most (one comparable bit each)
constexpr int kTileTJ = 8;   // targets per tile by default (REMAT_TILE_TJ)
constexpr int kRecPerWarp = 256;  // pair-record slots per warp: lanes with records x TJ
constexpr int kDenseLanes = 16;  // lanes with a pair for lane = predecessor constants
constexpr int kSmallF = 4;       // frontier entries kept in registers (small-frontier path)

// One relaxable (predecessor, target) pair of a warp's current group.
struct __align__(16) PairQN {  // narrow: one LDS.128
  int base;       // shared-window byte address of row slot dt_ij of the target (shared rows)
  unsigned cap;   // B − fixed_ij: an entry passes the budget test iff m <= cap
  unsigned kb;    // (dm_ij << IB) | i: key = (m << IB) + kb
  int dtr;        // target row offset in the tile + dt_ij (element index, global rows)
};
struct __align__(16) PairQW {
  long long base;
  long long cap;
  u64 kb;
  int dtr;
  int pad;
};

// A live predecessor of a warp's chunk: its entry for item offset e is at
// ptr + e, its budget-feasible pairs are the records at shared addresses
// [a0, a1) (ready addresses: no index arithmetic per item).
struct __align__(16) PredRec {
  const void* ptr;  // address of the predecessor's entry for item offset 0
  unsigned a0, a1;  // shared-window byte addresses of wq[q0], wq[q1]
};
__device__ __forceinline__ PredRec ld_rec(const PredRec* p) {  // one LDS.128
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  PredRec r;
  r.ptr = reinterpret_cast<const void*>(((unsigned long long)v.y << 32) | v.x);
  r.a0 = v.z;
  r.a1 = v.w;
  return r;
}

template <bool NARROW>
struct Traits;
template <>
struct Traits<true> {
  using Key = unsigned;
  using E = EntryN;
  using Q = PairQN;
  using M = unsigned;
  static constexpr unsigned INF = 0xffffffffu;
  // one LDG.64 per entry (entries of earlier levels are read-only while a
  // level is relaxed, so the non-coherent path is safe)
  template <int MODE = 0>
  static __device__ __forceinline__ void load(const E* p, unsigned& t, unsigned& m) {
    const uint2* q = reinterpret_cast<const uint2*>(p);
    const uint2 v = MODE == 1 ? __ldcg(q) : MODE == 2 ? __ldca(q) : __ldg(q);
    t = v.x;
    m = v.y;
  }
  static __device__ __forceinline__ PairQN lds(const PairQN* p) {  // one LDS.128
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"((unsigned)__cvta_generic_to_shared(p)));
    PairQN q;
    q.base = (int)v.x;
    q.cap = v.y;
    q.kb = v.z;
    q.dtr = (int)v.w;
    return q;
  }
};
template <>
struct Traits<false> {
  using Key = u64;
  using E = EntryW;
  using Q = PairQW;
  using M = long long;
  static constexpr u64 INF = ~0ull;
  template <int MODE = 0>
  static __device__ __forceinline__ void load(const E* p, unsigned& t, long long& m) {
    const longlong2* q = reinterpret_cast<const longlong2*>(p);
    const longlong2 v = MODE == 1 ? __ldcg(q) : MODE == 2 ? __ldca(q) : __ldg(q);
    t = (unsigned)v.x;
    m = v.y;
  }
  static __device__ __forceinline__ PairQW lds(const PairQW* p) { return *p; }
};

// Loads of the DP table being built (frontier entries, |frontier|, smallest m):
//   0  non-coherent path (per-level launches: the table is read-only here)
//   1  L2 only, ld.cg (persistent multi-level kernel: other SMs wrote it)
//   2  L1-cacheable, ld.ca (one CTA per budget walks every level and reads
//      only what it wrote itself, ordered by __syncthreads; chain-like
//      lattices read each predecessor at every later level, so it stays in L1)
template <int MODE, typename T>
__device__ __forceinline__ T ld_dp(const T* p) {
  if constexpr (MODE == 1) return __ldcg(p);
  else if constexpr (MODE == 2) return __ldca(p);
  else return *p;
}

// Shared-memory carve-up of k_relax_tile (host and device agree on it).
struct TileArgs {
  long long jbase;  // first target of this launch
  long long pend;   // end of the predecessor range (= start of the level)
  int width;        // targets in the level
  int TJ;           // targets per tile
  int splits;       // CTAs per tile (they share the tile's predecessor chunks)
  int R;            // row stride (level max T(L)+1)
  int smem_rows;    // rows in shared memory (else in grow)
  int cls;          // weight-class path available
  int rows_pb;      // rows per budget in grow (tiles · TJ)
  void* grow;       // [nb][rows_pb][R] global rows (split / oversized levels)
  unsigned* ctr;    // [nb][ctr_stride] next predecessor chunk of the tile (left zero)
  int tiles;
  int cw;           // predecessors per chunk (<= 32)
  int probe;        // small-frontier path: probe a slot before its RED (uniform T_v)
  int ctr_stride;   // counters per budget: tiles, or the widest level when budgets run
                    // through the levels independently (k_solve_small)
  int qlanes;       // lanes per warp with a pair-record region (>= cw; 32 up to 8 targets)
  int off_tL, off_tB, off_tc, off_tcls, off_bjc, off_coef, off_tacc, off_pairs, off_q, off_qs, off_rows;
  int off_tC;       // [W] intersection of the tile's target sets
  int bytes;
};

template <int W, bool NARROW>
static TileArgs tile_layout(int TJ, int R, int K, bool smem_rows, bool cls) {
  using Key = typename Traits<NARROW>::Key;
  TileArgs a{};
  a.TJ = TJ;
  a.R = R;
  static const int rec_env = [] {  // REMAT_REC_PER_WARP: record slots per warp (A/B)
    const char* e = getenv("REMAT_REC_PER_WARP");
    return e ? std::max(32, atoi(e)) : kRecPerWarp;
  }();
  a.qlanes = std::max(1, std::min(32, rec_env / TJ));
  a.smem_rows = smem_rows;
  a.cls = cls;
  int o = 0;
  auto take = [&](int bytes) {
    int at = o;
    o += (bytes + 15) & ~15;
    return at;
  };
  constexpr int WS = mask_stride<W>();
  a.off_tL = take(TJ * WS * 8);
  a.off_tB = take(TJ * WS * 8);
  a.off_tC = take(W * 8);
  a.off_tc = take(TJ * 4 * 8);
  a.off_tcls = take(TJ * 8);  // per target: path flags, nonzero-word mask
  a.off_bjc = take(cls ? TJ * K * WS * 8 : 0);
  a.off_coef = take(cls ? 2 * K * 8 : 0);
  a.off_tacc = take(TJ * 2 * 8);
  a.off_q = take(kWarps * a.qlanes * TJ * (int)sizeof(typename Traits<NARROW>::Q));
  a.off_qs = take(kWarps * 32 * (16 + 4));
  // a warp's sparse-pair list (<= qlanes·TJ <= 256 u16) lives in its live-
  // predecessor slots (32 x 16 B): the list is consumed before those are
  // written, and the 4 KB saved buys a wider tile at 4 CTAs per SM
  a.off_pairs = a.off_qs;
  a.off_rows = take(smem_rows ? TJ * R * (int)sizeof(Key) : 0);
  a.bytes = o;
  return a;
}

__device__ __forceinline__ void key_min(unsigned* p, unsigned key, bool) {
  if (key < *p) atomicMin(p, key);
}
// sm_100 has no native 64-bit shared-memory min (it lowers to a CAS loop), so
// read first: a losing candidate issues no atomic at all.  Global rows use the
// native 64-bit atomic min.
__device__ __forceinline__ void key_min(u64* p, u64 key, bool smem) {
  if (smem) {
    u64 old = *p;
    while (key < old) {
      u64 prev = atomicCAS(p, old, key);
      if (prev == old) break;
      old = prev;
    }
  } else if (key < *p) {
    atomicMin(p, key);
  }
}

// One candidate into a shared-memory row: row[t2] = min(row[t2], key) if `ok`.
// Every candidate's slot t2 = t + dt_ij <= T(L_j) is inside the row even when
// the budget test fails, so the slot address is always valid.
// Item path (long frontiers): every candidate issues its RED unconditionally
// (INF when it fails the budget test).  A probe-then-predicated-RED costs a
// shared load, a compare and — since ptxas lowers a predicated shared atomic
// to a branch — a reconvergence region per candidate; the bare RED is cheaper
// whenever candidates of a warp step rarely collide on one slot
// (U-Net c=8 relaxation: 17.3 -> 15.5 ms).
__device__ __forceinline__ void red_smem(unsigned a, unsigned key, bool ok) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(a), "r"(ok ? key : 0xffffffffu));
}
// All pairs [a, e) (shared addresses of records) of one item (entry t, m;
// mk = m << IB, t4 = 4t), four
// records per step so four LDS.128 are in flight (U-Net c=8: 4 -> 2 per step
// costs 0.6 %, 1 per step 4 %).
__device__ __forceinline__ PairQN lds_pair(unsigned a) {  // one LDS.128
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  PairQN q;
  q.base = (int)v.x;
  q.cap = v.y;
  q.kb = v.z;
  q.dtr = (int)v.w;
  return q;
}
__device__ __forceinline__ void red_pairs(unsigned a, const unsigned e, unsigned t4, unsigned mk,
                                          unsigned m) {
  for (; a + 48 < e; a += 64) {
    const PairQN p0 = lds_pair(a), p1 = lds_pair(a + 16);
    const PairQN p2 = lds_pair(a + 32), p3 = lds_pair(a + 48);
    red_smem(t4 + (unsigned)p0.base, mk + p0.kb, m <= p0.cap);
    red_smem(t4 + (unsigned)p1.base, mk + p1.kb, m <= p1.cap);
    red_smem(t4 + (unsigned)p2.base, mk + p2.kb, m <= p2.cap);
    red_smem(t4 + (unsigned)p3.base, mk + p3.kb, m <= p3.cap);
  }
  for (; a + 16 < e; a += 32) {
    const PairQN p0 = lds_pair(a), p1 = lds_pair(a + 16);
    red_smem(t4 + (unsigned)p0.base, mk + p0.kb, m <= p0.cap);
    red_smem(t4 + (unsigned)p1.base, mk + p1.kb, m <= p1.cap);
  }
  if (a < e) {
    const PairQN p = lds_pair(a);
    red_smem(t4 + (unsigned)p.base, mk + p.kb, m <= p.cap);
  }
}
// Small-frontier path when every T_v is equal (few distinct slots, the lanes
// of a warp collide on them and same-address REDs serialise): probe first, so
// a losing candidate issues no atomic.
__device__ __forceinline__ void relax_smem(unsigned a, unsigned key, bool ok) {
  asm volatile(
      "{\n\t.reg .pred o, q;\n\t.reg .u32 c;\n\t"
      "ld.shared.u32 c, [%0];\n\t"
      "setp.ne.u32 o, %2, 0;\n\t"
      "setp.lt.and.u32 q, %1, c, o;\n\t"
      "@q red.shared.min.u32 [%0], %1;\n\t}"
      ::"r"(a), "r"(key), "r"((unsigned)ok));
}

template <typename T>
__device__ __forceinline__ T warp_incl_min(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v = o < v ? o : v;
  }
  return v;
}

// K5 for one finished row (one warp): |cell|, the strict prefix-min frontier in
// t order (ascending for minimize, descending for maximize; planner.py:153-161)
// compacted into the member's frontier slot with its back-pointers.
template <typename Key>
__device__ __forceinline__ Key row_ld(const Key* p, bool global) {
  return global ? __ldcg(p) : *p;  // global rows: L2 (other SMs' atomics land there)
}

template <bool NARROW>
__device__ void finalize_row_warp(const typename Traits<NARROW>::Key* row, int Rj,
                                  const DpView& dp, const FamilyView& fv, long long j, int b,
                                  bool global = false) {
  using Key = typename Traits<NARROW>::Key;
  using E = typename Traits<NARROW>::E;
  constexpr Key INF = Traits<NARROW>::INF;
  const int lane = threadIdx.x & 31;
  const long long F = fv.F;
  const int IB = dp.IB;
  const bool mx = dp.maximize;
  const int per = (Rj + 31) / 32;
  const int s0 = min(Rj, lane * per), s1 = min(Rj, s0 + per);
  Key lmin = INF;
  int cells = 0;
  for (int s = s0; s < s1; s++) {
    Key key = row_ld(row + (mx ? Rj - 1 - s : s), global);
    if (key != INF) {
      cells++;
      Key m = key >> IB;
      lmin = m < lmin ? m : lmin;
    }
  }
  Key incl = warp_incl_min(lmin);
  Key pm = __shfl_up_sync(kFull, incl, 1);
  if (lane == 0) pm = INF;
  int nf = 0;
  Key run = pm;
  for (int s = s0; s < s1; s++) {
    Key key = row_ld(row + (mx ? Rj - 1 - s : s), global);
    if (key != INF && (key >> IB) < run) {
      nf++;
      run = key >> IB;
    }
  }
  const int nf_incl = warp_inclusive_sum(nf);
  const int nf_tot = __shfl_sync(kFull, nf_incl, 31);
  const int cells_tot = warp_sum(cells);
  const long long slot0 = (long long)b * dp.slots + fv.foff[j];
  E* out = reinterpret_cast<E*>(dp.fe) + slot0;
  int* par = dp.parent + slot0;
  int pos = nf_incl - nf;
  run = pm;
  const Key pmask = (Key(1) << IB) - 1;
  for (int s = s0; s < s1; s++) {
    const int t = mx ? Rj - 1 - s : s;
    Key key = row_ld(row + t, global);
    if (key != INF && (key >> IB) < run) {
      run = key >> IB;
      E e{};
      e.t = (unsigned)t;
      e.m = run;
      out[pos] = e;
      par[pos] = (int)(key & pmask);
      pos++;
    }
  }
  const Key gmin = __shfl_sync(kFull, incl, 31);
  if (lane == 0) {
    const size_t at = (size_t)b * F + j;
    dp.flen[at] = nf_tot;
    dp.ccount[at] = cells_tot;
    dp.mmin[at] = nf_tot ? (long long)gmin : LLONG_MAX;
  }
}

// K5 for a tile of ONE target (chain-like levels: C1, C3, narrow C5 levels)
// with the whole CTA: each thread scans Rj/256 slots, block scans give the
// prefix-min and the output positions — instead of one warp walking the row
// three times while seven wait at the next barrier (k_solve_small: barrier
// stalls 8.6 per issued instruction on C3).  Called by every thread.
// `scr`: >= 36 u64 of dynamic shared memory free at finalize time (the
// tile's pair-record region: static shared memory here would cost the
// per-level kernels a resident CTA).
template <bool NARROW>
__device__ void finalize_row_block(const typename Traits<NARROW>::Key* row, int Rj,
                                   const DpView& dp, const FamilyView& fv, long long j, int b,
                                   u64* scr) {
  using Key = typename Traits<NARROW>::Key;
  using E = typename Traits<NARROW>::E;
  constexpr Key INF = Traits<NARROW>::INF;
  u64* s_scr = scr;
  u64& s_gmin = scr[35];
  const int tid = threadIdx.x;
  const int IB = dp.IB;
  const bool mx = dp.maximize;
  const int per = (Rj + kThreads - 1) / kThreads;
  const int s0 = min(Rj, tid * per), s1 = min(Rj, s0 + per);
  u64 lmin = ~0ull, cells = 0;
  for (int q = s0; q < s1; q++) {
    const Key key = row[mx ? Rj - 1 - q : q];
    if (key != INF) {
      cells++;
      const u64 m = (u64)(key >> IB);
      lmin = m < lmin ? m : lmin;
    }
  }
  if (tid == 0) s_gmin = ~0ull;
  const u64 pm = block_exclusive_min(lmin, s_scr);
  if (lmin != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(&s_gmin), lmin);
  u64 nf = 0, run = pm;
  for (int q = s0; q < s1; q++) {
    const Key key = row[mx ? Rj - 1 - q : q];
    if (key != INF && (u64)(key >> IB) < run) {
      nf++;
      run = (u64)(key >> IB);
    }
  }
  // one scan for both counts: |frontier| in the high half, |cell| in the low
  u64 both_tot;
  u64 pos = block_exclusive_sum((nf << 32) | cells, s_scr, &both_tot) >> 32;
  const u64 nf_tot = both_tot >> 32, cells_tot = both_tot & 0xffffffffull;
  const long long slot0 = (long long)b * dp.slots + fv.foff[j];
  E* out = reinterpret_cast<E*>(dp.fe) + slot0;
  int* par = dp.parent + slot0;
  const Key pmask = (Key(1) << IB) - 1;
  run = pm;
  for (int q = s0; q < s1; q++) {
    const int t = mx ? Rj - 1 - q : q;
    const Key key = row[t];
    if (key != INF && (u64)(key >> IB) < run) {
      run = (u64)(key >> IB);
      E e{};
      e.t = (unsigned)t;
      e.m = (decltype(e.m))run;
      out[pos] = e;
      par[pos] = (int)(key & pmask);
      pos++;
    }
  }
  if (tid == 0) {
    const size_t at = (size_t)b * fv.F + j;
    dp.flen[at] = (int)nf_tot;
    dp.ccount[at] = (int)cells_tot;
    dp.mmin[at] = nf_tot ? (long long)s_gmin : LLONG_MAX;
  }
}

// K4 (+K5): one (tile, split) "virtual CTA" `vbx` of budget b.  Run either as
// one CTA of k_relax_tile (grid (tiles·splits, nb)) or inside the persistent
// k_relax_levels loop.
// COH: the table being read was written earlier in the SAME launch (persistent
// multi-level kernel) — frontier entries and per-member records are then read
// through L2 (ld.cg), never the non-coherent path.
// Shared-memory set-up of a tile: the targets' sets and scalars, empty rows,
// the weight-class masks.  Reads family constants only, so the persistent
// kernel runs it for the next level before the grid barrier.
__shared__ int s_relax_worked;

template <int W, bool NARROW>
__device__ __forceinline__ void tile_setup(const FamilyView& fv, const ClassView& cv,
                                           const TileArgs& ta, const int vbx, unsigned char* sm) {
  using Key = typename Traits<NARROW>::Key;
  constexpr Key INF = Traits<NARROW>::INF;
  const int tid = threadIdx.x;
  const int TJ = ta.TJ, R = ta.R;
  const long long F = fv.F;
  const long long j0 = ta.jbase + (long long)(vbx / ta.splits) * TJ;
  const int ntj = (int)min((long long)TJ, ta.jbase + ta.width - j0);
  u64* tL = reinterpret_cast<u64*>(sm + ta.off_tL);
  u64* tB = reinterpret_cast<u64*>(sm + ta.off_tB);
  long long* tc = reinterpret_cast<long long*>(sm + ta.off_tc);
  int* tcls = reinterpret_cast<int*>(sm + ta.off_tcls);
  u64* bjc = reinterpret_cast<u64*>(sm + ta.off_bjc);
  long long* tcoef = reinterpret_cast<long long*>(sm + ta.off_coef);
  u64* tacc = reinterpret_cast<u64*>(sm + ta.off_tacc);
  Key* rows = reinterpret_cast<Key*>(sm + ta.off_rows);
  const bool srow = ta.smem_rows;
  if (tid == 0) s_relax_worked = 0;
  constexpr int WS = mask_stride<W>();
  for (int e = tid; e < ntj * WS; e += kThreads) {
    const int jt = e / WS, w = e - jt * WS;
    tL[e] = w < W ? fv.masks[(size_t)w * F + j0 + jt] : 0ull;
    tB[e] = w < W ? fv.bound[(size_t)w * F + j0 + jt] : 0ull;
  }
  for (int jt = tid; jt < ntj; jt += kThreads) {
    const long long j = j0 + jt;
    tc[jt * 4 + 0] = fv.ML[j];
    tc[jt * 4 + 1] = fv.base[j];
    tc[jt * 4 + 2] = fv.TLnb[j];
    tc[jt * 4 + 3] = fv.Mb[j];
    tacc[jt * 2] = 0;
    tacc[jt * 2 + 1] = 0;
  }
  if (srow)
    for (int t = tid; t < ntj * R; t += kThreads) rows[t] = INF;
  __syncthreads();
  if (tid < W) {  // ∩ of the tile's targets: a predecessor inside it precedes all of them
    u64 c = ~0ull;
    for (int jt = 0; jt < ntj; jt++) c &= tL[jt * WS + tid];
    reinterpret_cast<u64*>(sm + ta.off_tC)[tid] = c;
  }
  const int K = cv.K;
  // The pair terms need T and M of L_i ∩ ∂L_j, i.e. T(L_i) − T(L_i ∩ I_j)
  // with I_j = L_j \ ∂L_j the interior.  Wide sets (W >= 4) take, per
  // target, the cheaper mask (deep lattices of dense DAGs: the interior is
  // EMPTY on most levels of C5, so the pair terms need no popcount at all) and
  // visit only its nonzero words; the chosen mask replaces ∂L_j in tB.  Narrow
  // sets keep the boundary (a bit loop over a few nodes on U-Net: the extra
  // set-up was measured +2 % there).  Either way the cheaper method: class
  // popcounts or a bit loop over the mask's nodes.
  if constexpr (W >= 4) {
    for (int jt = tid; jt < ntj; jt += kThreads) {
      int bc = 0, ic = 0;
      unsigned bnz = 0, inz = 0;
      for (int w = 0; w < W; w++) {
        const u64 bw = tB[jt * WS + w], iw = tL[jt * WS + w] & ~bw;
        bc += __popcll(bw);
        ic += __popcll(iw);
        bnz |= (bw != 0 ? 1u : 0u) << w;
        inz |= (iw != 0 ? 1u : 0u) << w;
      }
      auto cost = [&](int bits, unsigned nz) {  // ~warp instructions per pair
        const int cls = ta.cls ? 4 * K * __popc(nz) : INT_MAX;
        return min(cls, 6 * bits);
      };
      const bool interior = cost(ic, inz) < cost(bc, bnz);
      const int bits = interior ? ic : bc;
      const unsigned nz = interior ? inz : bnz;
      if (interior)
        for (int w = 0; w < W; w++) tB[jt * WS + w] = tL[jt * WS + w] & ~tB[jt * WS + w];
      tcls[2 * jt] = (ta.cls && 4 * K * __popc(nz) < 6 * bits ? 1 : 0) | (interior ? 2 : 0);
      tcls[2 * jt + 1] = (int)nz;
    }
    __syncthreads();
  }
  if (ta.cls) {
    for (int e = tid; e < ntj * K * WS; e += kThreads) {
      const int jt = e / (K * WS), r = e - jt * K * WS, c = r / WS, w = r - c * WS;
      bjc[e] = w < W ? tB[jt * WS + w] & cv.cls[c * W + w] : 0ull;
    }
    for (int e = tid; e < 2 * K; e += kThreads) tcoef[e] = cv.coef[e];
  }
  if constexpr (W < 4) {
    for (int jt = tid; jt < ntj; jt += kThreads) {
      int bc = 0;
      for (int w = 0; w < W; w++) bc += __popcll(tB[jt * WS + w]);
      tcls[2 * jt] = ta.cls && K * W < bc;
      tcls[2 * jt + 1] = (1 << W) - 1;
    }
  }
  __syncthreads();
}

template <int W, bool NARROW, bool COH, bool DUAL = false,
          int LDM = !COH ? 0 : (DUAL ? 2 : 1)>
__device__ __forceinline__ void relax_body(const FamilyView& fv, const GraphView& g,
                                           const ClassView& cv, const DpView& dp,
                                           const TileArgs& ta, const int vbx, const int b,
                                           const int nb, unsigned char* sm,
                                           const bool presetup = false) {
  using Key = typename Traits<NARROW>::Key;
  using E = typename Traits<NARROW>::E;
  using Q = typename Traits<NARROW>::Q;
  using MT = typename Traits<NARROW>::M;
  constexpr Key INF = Traits<NARROW>::INF;
  int& s_worked = s_relax_worked;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1;
  const int TJ = ta.TJ, R = ta.R, splits = ta.splits;
  constexpr int WS = mask_stride<W>();
  const long long F = fv.F;
  const int tile = vbx / splits;
  const long long j0 = ta.jbase + (long long)tile * TJ;
  const int ntj = (int)min((long long)TJ, ta.jbase + ta.width - j0);

  u64* tL = reinterpret_cast<u64*>(sm + ta.off_tL);         // [TJ][W]
  u64* tB = reinterpret_cast<u64*>(sm + ta.off_tB);         // [TJ][W]
  long long* tc = reinterpret_cast<long long*>(sm + ta.off_tc);  // [TJ][4]
  int* tcls = reinterpret_cast<int*>(sm + ta.off_tcls);     // [TJ][2]
  u64* bjc = reinterpret_cast<u64*>(sm + ta.off_bjc);       // [TJ][K][W]
  long long* tcoef = reinterpret_cast<long long*>(sm + ta.off_coef);  // [K][2]
  u64* tacc = reinterpret_cast<u64*>(sm + ta.off_tacc);     // [TJ][2]
  unsigned short* wpairs =
      reinterpret_cast<unsigned short*>(sm + ta.off_pairs) + warp * 256;  // aliases wrec
  Q* wq = reinterpret_cast<Q*>(sm + ta.off_q) + warp * ta.qlanes * TJ;  // feasible pairs of a chunk
  const unsigned wq_sa = (unsigned)__cvta_generic_to_shared(wq);
  PredRec* wrec = reinterpret_cast<PredRec*>(sm + ta.off_qs) + warp * 32;  // live predecessors
  int* wpc = reinterpret_cast<int*>(sm + ta.off_qs + kWarps * 32 * 16) + warp * 32;
  Key* grow_t = ta.grow ? reinterpret_cast<Key*>(ta.grow) +
                              ((size_t)b * ta.rows_pb + (size_t)tile * TJ) * R
                        : nullptr;
  Key* rows = ta.smem_rows ? reinterpret_cast<Key*>(sm + ta.off_rows) : grow_t;
  const bool srow = ta.smem_rows;

  if (!presetup) tile_setup<W, NARROW>(fv, cv, ta, vbx, sm);
  const int K = cv.K;

  const long long B = dp.budgets[b];
  const int IB = dp.IB;
  const long long fbase = (long long)b * dp.slots;
  const int* flen_b = dp.flen + (size_t)b * F;
  const long long* mmin_b = dp.mmin + (size_t)b * F;
  const E* fe = reinterpret_cast<const E*>(dp.fe);
  const long long pred_end = ta.pend;
  const int cw = ta.cw;  // predecessors per chunk (32; fewer spreads narrow levels over warps)
  const long long nch = (pred_end + cw - 1) / cw;
  unsigned* ctr = ta.ctr + (size_t)b * ta.ctr_stride + tile;
  u64 my_trans = 0;  // lane = predecessor: its Σ|frontier| over comparable tile targets
  u64 my_pairs = 0;
  bool worked = false;

  // Every CTA of the tile pulls 32-predecessor chunks from the tile's counter,
  // so slices finish together and CTAs of a late wave find nothing left.
  // Pair constants of (predecessor i, tile target jt) -> record q; true iff
  // some frontier entry of i can pass the budget test (cap >= its smallest m).
  // shared-window byte address of the tile rows (shared-row path)
  const unsigned rs_base = srow ? (unsigned)__cvta_generic_to_shared(sm + ta.off_rows) : 0u;
  auto pair_q = [&](const u64 (&Li)[W], long long ii, int jt, long long MLi, long long TLi,
                    long long mmi, Q& q) {
    // weighted popcount of L_i ∩ (∂L_j or I_j) over the mask's nonzero words
    long long ts = 0, ms = 0;
    const int fl = tcls[2 * jt];
    // (narrow sets visit every word: no per-word test)
    const unsigned nz = W >= 4 ? (unsigned)tcls[2 * jt + 1] : (1u << W) - 1;
    if (K == 1 && (fl & 1)) {
      // one weight class (uniform costs, C5): every word, branch-free, with
      // the target's mask words as broadcast shared loads — the general loop
      // below spends most of its issue on per-word branches and the dynamic
      // class-index address arithmetic (C5 p=0.2 relax 153.5 -> 146.6 ms)
      if (nz) {
        const ulonglong2* bj2 = reinterpret_cast<const ulonglong2*>(bjc + (size_t)jt * WS);
        int pc = 0;
#pragma unroll
        for (int w = 0; w < W; w += 2) {
          const ulonglong2 b = bj2[w / 2];  // one LDS.128 (padding word is 0)
          pc += __popcll(Li[w] & b.x);
          if (w + 1 < W) pc += __popcll(Li[w + 1] & b.y);
        }
        ts = tcoef[0] * pc;
        ms = tcoef[1] * pc;
      }
    } else if (fl & 1) {
      const u64* bj = bjc + (size_t)jt * K * WS;
      for (int cc = 0; cc < K; cc++) {
        int pc = 0;
#pragma unroll
        for (int w = 0; w < W; w++)
          if (W < 4 || ((nz >> w) & 1u)) pc += __popcll(Li[w] & bj[cc * WS + w]);
        ts += tcoef[2 * cc] * pc;
        ms += tcoef[2 * cc + 1] * pc;
      }
    } else if (nz) {
#pragma unroll
      for (int w = 0; w < W; w++) {
        if (W >= 4 && !((nz >> w) & 1u)) continue;
        u64 x = Li[w] & tB[jt * WS + w];
        while (x) {
          const int v = w * 64 + __ffsll((long long)x) - 1;
          x &= x - 1;
          ts += __ldg(g.T + v);
          ms += __ldg(g.M + v);
        }
      }
    }
    if (W >= 4 && (fl & 2)) {  // interior mask: T(L_i ∩ ∂L_j) = T(L_i) − T(L_i ∩ I_j)
      ts = TLi - ts;
      ms = MLi - ms;
    }
    const long long fixed = 2 * (tc[jt * 4 + 0] - MLi) + tc[jt * 4 + 1];
    const long long dt = tc[jt * 4 + 2] - TLi + ts;
    const long long dm = tc[jt * 4 + 3] - ms;
    const long long cap = B - fixed;
    q.cap = (MT)max(cap, 0LL);
    q.base = (int)(rs_base + 4u * (unsigned)(jt * R + (int)dt));  // smem byte address of slot dt
    q.kb = (Key)(((u64)dm << IB) | (u64)ii);
    q.dtr = jt * R + (int)dt;
    return cap >= mmi;
  };

  // the first chunk of every warp is static (CTA rank within the tile x warps
  // + warp), later ones come from the counter, offset past the static ones
  const long long nstatic = (long long)splits * kWarps;
  // (the one-CTA-per-budget solver deals its chunks round-robin: a level's
  // few chunks are too even to need balancing, and each counter round trip
  // sits on the level-to-level critical path)
  auto next_chunk = [&](long long ch) {
    if constexpr (DUAL) return ch + nstatic;
    if (nstatic >= nch) return nch;  // the static chunks covered the range
    unsigned got = 0;
    if (lane == 0) got = atomicAdd(ctr, 1u);
    return nstatic + (long long)__shfl_sync(kFull, got, 0);
  };
  for (long long ch = (long long)(vbx - tile * splits) * kWarps + warp; ch < nch;
       ch = next_chunk(ch)) {
    worked = true;
    // lane = predecessor i: its set and scalars in one round of loads.  With
    // chunks of <= 16 predecessors (16-target tiles) the upper half-warp
    // mirrors the lower one and tests the upper half of the tile's targets,
    // so no lane idles in the subset tests; the halves' masks are merged.
    const bool split = cw <= 16 && ntj > 8;  // warp-uniform
    const int pl = split ? (lane & 15) : lane;
    const long long i = ch * cw + pl;
    u64 Li[W];
    int fl = 0;
    long long MLi = 0, TLi = 0, mmi = 0, foffi = 0;
    unsigned mask = 0;
    const bool live = pl < cw && i < pred_end;
#pragma unroll
    for (int w = 0; w < W; w++) Li[w] = live ? __ldg(fv.masks + (size_t)w * F + i) : 0ull;
    // wide sets (deep lattices, C5: nearly every lower predecessor precedes
    // every target): one test against the tile's intersection replaces the
    // per-target tests when it holds for the whole warp (throughput launches
    // only: on the narrow levels of the persistent kernel the extra vote sits
    // on the latency path, C5 p=0.3 +3 %)
    bool allc = false;
    if constexpr (W >= 4 && !COH) {
      const u64* tC = reinterpret_cast<const u64*>(sm + ta.off_tC);
      u64 a = 0;
#pragma unroll
      for (int w = 0; w < W; w++) a |= Li[w] & ~tC[w];
      allc = __all_sync(kFull, a == 0);
    }
    if (live) {
      if (lane == pl) {
        fl = ld_dp<LDM>(flen_b + i);
        mmi = ld_dp<LDM>(mmin_b + i);
        MLi = __ldg(fv.ML + i);
        TLi = __ldg(fv.TL + i);
        foffi = __ldg(fv.foff + i);
      }
      const int j0t = split && lane >= 16 ? 8 : 0;
      const int j1t = split && lane < 16 ? 8 : ntj;
      if (allc) {
        mask = ((j1t >= 32 ? 0u : 1u << j1t) - 1u) & ~((1u << j0t) - 1u);
      } else {
        for (int jt = j0t; jt < j1t; jt++) {
          u64 acc = 0;
          if constexpr (WS > W || (W >= 4 && W % 2 == 0)) {
            const ulonglong2* t2 = reinterpret_cast<const ulonglong2*>(tL + jt * WS);
#pragma unroll
            for (int w = 0; w < W; w += 2) {
              const ulonglong2 t = t2[w / 2];
              acc |= Li[w] & ~t.x;
              if (w + 1 < W) acc |= Li[w + 1] & ~t.y;
            }
          } else {
#pragma unroll
            for (int w = 0; w < W; w++) acc |= Li[w] & ~tL[jt * W + w];
          }
          mask |= (acc == 0 ? 1u : 0u) << jt;
        }
      }
    }
    if (split) {
      mask |= __shfl_xor_sync(kFull, mask, 16);
      if (lane >= 16) mask = 0;
    }
    // statistics on the predecessor side: P and Σ|frontier_i| over the
    // comparable pairs of this lane's predecessor (the totals are what
    // SearchStats needs; a per-target ballot + REDUX per tile target cost
    // ~5 % of the issue slots)
    my_pairs += (u64)__popc(mask);
    my_trans += (u64)__popc(mask) * (u64)fl;
    if (!__any_sync(kFull, mask)) continue;
    // Small frontiers (every predecessor of the chunk has <= kSmallF entries,
    // the uniform-cost regime of deep lattices): each lane keeps its entries
    // in registers and relaxes them into every comparable target directly —
    // no pair records, item mapping or second pass.
    if (__reduce_max_sync(kFull, (unsigned)fl) <= (unsigned)kSmallF) {
      unsigned et[kSmallF];
      MT em[kSmallF];
#pragma unroll
      for (int e = 0; e < kSmallF; e++) {
        et[e] = 0;
        em[e] = 0;
        if (e < fl) Traits<NARROW>::template load<LDM>(fe + (fbase + foffi + e), et[e], em[e]);
      }
      for (int jt = 0; jt < ntj; jt++) {
        const bool bit = (mask >> jt) & 1u;
        if (!bit || fl == 0) continue;
        Q q;
        if (!pair_q(Li, i, jt, MLi, TLi, mmi, q)) continue;
#pragma unroll
        for (int e = 0; e < kSmallF; e++) {
          if (e >= fl) break;
          const Key key = ((Key)em[e] << IB) + (Key)q.kb;
          if constexpr (NARROW) {
            if (srow) {
              if (ta.probe)
                relax_smem((unsigned)q.base + 4u * et[e], key, em[e] <= q.cap);
              else
                red_smem((unsigned)q.base + 4u * et[e], key, em[e] <= q.cap);
              continue;
            }
          }
          if (em[e] <= q.cap) key_min(rows + (et[e] + q.dtr), key, srow);
        }
      }
      continue;
    }
    // per target: statistics, then the pair constants — computed right here
    // (lane = predecessor, no reload) when most lanes hold a pair, else
    // deferred to a compacted list (lane = pair) so sparse targets do not
    // serialise the warp
    Q* myq = wq + lane * TJ;
    int npq = 0;
    const unsigned wantm = fl > 0 ? mask : 0u;
    unsigned sparse = wantm;
    // a target is dense when >= kDenseLanes lanes want it; with chunks of at
    // most kDenseLanes predecessors that means every one of the first 16 lanes,
    // so one REDUX.AND rules the per-target vote out for the whole chunk (the
    // usual case on conv-weighted graphs: 13 % comparable density)
    // (narrow sets only: on the wide-set kernel the extra vote cost C5 0.4 %)
    const bool maybe_dense =
        W >= 4 || cw > kDenseLanes ||
        __reduce_and_sync(kFull, lane < kDenseLanes ? wantm : ~0u) != 0u;
    if (maybe_dense) {
      sparse = 0;
      for (int jt = 0; jt < ntj; jt++) {
        const bool bit = (mask >> jt) & 1u;
        const bool want = bit && fl > 0;
        const unsigned wm = __ballot_sync(kFull, want);
        if (__popc(wm) >= kDenseLanes) {
          if (want) {
            Q q;
            if (pair_q(Li, i, jt, MLi, TLi, mmi, q)) myq[npq++] = q;
          }
        } else if (want) {
          sparse |= 1u << jt;
        }
      }
    }
    wpc[lane] = npq;
    const int scnt = __popc(sparse);
    const int sincl = warp_inclusive_sum(scnt);
    const int nsp = __shfl_sync(kFull, sincl, 31);
    {
      int pos = sincl - scnt;
      unsigned x = sparse;
      while (x) {
        const int jt = __ffs(x) - 1;
        x &= x - 1;
        wpairs[pos++] = (unsigned short)((lane << 5) | jt);
      }
    }
    __syncwarp();
    for (int g0 = 0; g0 < nsp; g0 += 32) {
      if (lane < nsp - g0) {
        const int pr = wpairs[g0 + lane];
        const int jt = pr & 31, pl = pr >> 5;
        const long long ii = ch * cw + pl;
        u64 Lp[W];
#pragma unroll
        for (int w = 0; w < W; w++) Lp[w] = __ldg(fv.masks + (size_t)w * F + ii);
        Q q;
        if (pair_q(Lp, ii, jt, __ldg(fv.ML + ii), __ldg(fv.TL + ii),
                   ld_dp<LDM>(mmin_b + ii), q))
          wq[pl * TJ + atomicAdd(wpc + pl, 1)] = q;
      }
    }
    __syncwarp();
    // items = (predecessor, frontier entry), lane = predecessor again
    const int pc = wpc[lane];
    const int c = pc > 0 ? fl : 0;
    const unsigned has = __ballot_sync(kFull, c > 0);
    if (!has) continue;
    const int iincl = warp_inclusive_sum(c);
    const int tot = __shfl_sync(kFull, iincl, 31);
    const int start = c > 0 ? iincl - c : INT_MAX;
    if (c > 0) {
      PredRec rc;
      rc.ptr = fe + (fbase + foffi - (iincl - c));
      rc.a0 = wq_sa + (unsigned)(lane * TJ * sizeof(Q));
      rc.a1 = rc.a0 + (unsigned)(pc * sizeof(Q));
      wrec[__popc(has & lt)] = rc;
    }
    __syncwarp();
    // Item e belongs to the last live predecessor starting at or before e:
    // per 32-item step one REDUX.OR gathers the predecessor starts inside the
    // step and a popcount ranks each lane among them.  One entry load then
    // feeds every target of that predecessor in the tile (rows are addressed
    // through the shared window directly when they live in shared memory, so
    // each candidate is one ATOMS.MIN).
    const unsigned le = lt | (1u << lane);
    // smem: rows addressed as 32-bit shared-window offsets; global: pointers
    auto relax_items = [&](Key* __restrict__ rw, const unsigned rs, const bool smem) {
      int kbase = -1;
      auto map_step = [&](int r) {  // warp-uniform call
        const unsigned d = (unsigned)(start - r);
        const unsigned smask = __reduce_or_sync(kFull, d < 32u ? 1u << d : 0u);
        const int k = kbase + __popc(smask & le);
        kbase += __popc(smask);
        return k;
      };
      // software-pipelined: the entry of step r+32 is in flight (L2) while
      // the targets of step r are relaxed
      PredRec rec{};
      unsigned t = 0;
      MT m = 0;
      bool v = false;
      {
        const int k = map_step(0);
        v = lane < tot;
        if (v) {
          rec = ld_rec(wrec + k);
          Traits<NARROW>::template load<LDM>(static_cast<const E*>(rec.ptr) + lane, t, m);
        }
      }
      for (int r = 0; r < tot; r += 32) {
        PredRec recn{};
        unsigned tn = 0;
        MT mn = 0;
        bool vn = false;
        if (r + 32 < tot) {
          const int kn = map_step(r + 32);
          vn = r + 32 + lane < tot;
          if (vn) {
            recn = ld_rec(wrec + kn);
            Traits<NARROW>::template load<LDM>(static_cast<const E*>(recn.ptr) + (r + 32 + lane), tn, mn);
          }
        }
        if (v) {
          const Key mk = (Key)m << IB;
          const unsigned t4 = 4u * t;
          bool done = false;
          if constexpr (NARROW) {
            if (smem) {
              red_pairs(rec.a0, rec.a1, t4, mk, m);
              done = true;
            }
          }
          if (!done) {
            const Q* qe = wq + (rec.a1 - wq_sa) / sizeof(Q);
            for (const Q* qp = wq + (rec.a0 - wq_sa) / sizeof(Q); qp < qe; ++qp) {
              const Q p = Traits<NARROW>::lds(qp);
              if (m <= p.cap) key_min(rw + (t + p.dtr), mk + (Key)p.kb, smem);
            }
          }
        }
        rec = recn;
        t = tn;
        m = mn;
        v = vn;
      }
    };
    auto relax_items2 = [&](Key* __restrict__ rw, const unsigned rs, const bool smem) {
      int kbase = -1;
      // 64 items per step, lane owns items 2·lane and 2·lane+1 of the step:
      // two REDUX.OR gather the predecessor starts in each half, popcounts
      // rank both items (warp-uniform call)
      auto map_step = [&](int r, int& k0, int& k1) {
        const unsigned d = (unsigned)(start - r);
        const unsigned lo = __reduce_or_sync(kFull, d < 32u ? 1u << d : 0u);
        const unsigned hi = __reduce_or_sync(kFull, d - 32u < 32u ? 1u << (d - 32u) : 0u);
        const unsigned m0 = (2u << ((2 * lane) & 31)) - 1, m1 = (2u << ((2 * lane + 1) & 31)) - 1;
        const int below = lane < 16 ? 0 : __popc(lo);
        const unsigned half = lane < 16 ? lo : hi;
        k0 = kbase + below + __popc(half & m0);
        k1 = kbase + below + __popc(half & m1);
        kbase += __popc(lo) + __popc(hi);
      };
      struct Item {
        PredRec rec;
        unsigned t;
        MT m;
        bool v;
      };
      auto fetch = [&](int r, Item& x0, Item& x1) {
        int k0, k1;
        map_step(r, k0, k1);
        const int e0 = r + 2 * lane;
        x0.v = e0 < tot;
        x1.v = e0 + 1 < tot;
        if (x0.v) {
          x0.rec = wrec[k0];
          Traits<NARROW>::template load<LDM>(static_cast<const E*>(x0.rec.ptr) + e0, x0.t, x0.m);
        }
        if (x1.v) {
          x1.rec = wrec[k1];
          Traits<NARROW>::template load<LDM>(static_cast<const E*>(x1.rec.ptr) + (e0 + 1), x1.t, x1.m);
        }
      };
      auto relax = [&](const Item& x) {
        const unsigned t = x.t;
        const MT m = x.m;
        const Key mk = (Key)m << IB;
        const unsigned t4 = 4u * t;
        if constexpr (NARROW) {
          if (smem) {
            red_pairs(x.rec.a0, x.rec.a1, t4, mk, m);
            return;
          }
        }
        const Q* qe = wq + (x.rec.a1 - wq_sa) / sizeof(Q);
        for (const Q* qp = wq + (x.rec.a0 - wq_sa) / sizeof(Q); qp < qe; ++qp) {
          const Q p = Traits<NARROW>::lds(qp);
          if (m <= p.cap) key_min(rw + (t + p.dtr), mk + (Key)p.kb, smem);
        }
      };
      // software-pipelined: the two entries of step r+64 are in flight (L2)
      // while the targets of step r are relaxed
      Item a0{}, a1{};
      fetch(0, a0, a1);
      for (int r = 0; r < tot; r += 64) {
        Item b0{}, b1{};
        if (r + 64 < tot) fetch(r + 64, b0, b1);
        if (a0.v) relax(a0);
        if (a1.v) relax(a1);
        a0 = b0;
        a1 = b1;
      }
    };
    // throughput launches relax 32 items per warp step; the one-CTA-per-budget
    // solver (few warps per level, L2-latency bound) takes 64 with two loads
    // in flight per lane
    if constexpr (DUAL) {
      if (srow)
        relax_items2(reinterpret_cast<Key*>(sm + ta.off_rows),
                     (unsigned)__cvta_generic_to_shared(sm + ta.off_rows), true);
      else
        relax_items2(grow_t, 0u, false);
    } else {
      if (srow)
        relax_items(reinterpret_cast<Key*>(sm + ta.off_rows),
                    (unsigned)__cvta_generic_to_shared(sm + ta.off_rows), true);
      else
        relax_items(grow_t, 0u, false);
    }
    __syncwarp();
  }
  if (lane == 0 && worked) s_worked = 1;
  // the tile's totals go to its first target's per-member counters (their
  // sum over the family is the statistic)
  my_trans = warp_sum(my_trans);
  my_pairs = warp_sum(my_pairs);
  if (lane == 0 && (my_pairs | my_trans)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(tacc), my_trans);
    atomicAdd(reinterpret_cast<unsigned long long*>(tacc + 1), my_pairs);
  }
  __syncthreads();
  if (tid < ntj) {
    const size_t at = (size_t)b * F + j0 + tid;
    if (tacc[tid * 2]) atomicAdd(reinterpret_cast<unsigned long long*>(dp.trans + at), tacc[tid * 2]);
    if (tacc[tid * 2 + 1])
      atomicAdd(reinterpret_cast<unsigned long long*>(dp.npairs + at), tacc[tid * 2 + 1]);
  }
  unsigned* done = ctr + (size_t)nb * ta.ctr_stride;  // finished CTAs of the tile
  if (splits == 1 && srow) {
    if (DUAL && ntj == 1)
      finalize_row_block<NARROW>(rows, (int)(fv.TL[j0] + 1), dp, fv, j0, b,
                                 reinterpret_cast<u64*>(sm + ta.off_q));
    else
      for (int jt = warp; jt < ntj; jt += kWarps)
        finalize_row_warp<NARROW>(rows + jt * R, (int)(fv.TL[j0 + jt] + 1), dp,
                                  fv, j0 + jt, b);
    if (tid == 0) *ctr = 0;  // counters are self-resetting for the next level
    return;
  }
  if (srow && s_worked)  // fold this CTA's rows into the tile's global rows
    for (int t = tid; t < ntj * R; t += kThreads) {
      const Key key = rows[t];
      if (key != INF) atomicMin(grow_t + t, key);
    }
  // the last CTA of the tile to finish finalizes its rows and leaves
  // rows and counters as it found them (INF / 0), so no per-level fill,
  // memset or finalize launch is needed
  __shared__ int s_rj[kMaxTJ];
  if (tid < ntj) s_rj[tid] = (int)(fv.TL[j0 + tid] + 1);
  __threadfence();
  __syncthreads();
  if (tid == 0) s_worked = atomicAdd(done, 1u) == (unsigned)(splits - 1);
  __syncthreads();
  if (!s_worked) return;
  __threadfence();
  if (srow) {
    // pull the merged rows into shared memory with independent coalesced
    // loads spread over the whole CTA and finalize from there: a warp
    // scanning its row straight from L2 pays a round trip per group of
    // slots, three times over (C5 p=0.3 relax 8.4 -> 7.5 ms, C1 4.4 -> 4.0 ms)
    for (int e = tid; e < ntj * R; e += kThreads) {
      const int jt = e / R;
      if (e - jt * R < s_rj[jt]) {
        rows[e] = __ldcg(grow_t + e);
        grow_t[e] = INF;
      }
    }
    __syncthreads();
  }
  for (int jt = warp; jt < ntj; jt += kWarps) {
    const int Rj = s_rj[jt];
    if (srow) {
      finalize_row_warp<NARROW>(rows + jt * R, Rj, dp, fv, j0 + jt, b);
      continue;
    }
    Key* gr = grow_t + (size_t)jt * R;
    finalize_row_warp<NARROW>(gr, Rj, dp, fv, j0 + jt, b, true);
    __syncwarp();
    for (int t = lane; t < Rj; t += 32) gr[t] = INF;
  }
  if (tid == 0) {
    *ctr = 0;
    *done = 0;
  }
}

template <int W, bool NARROW>
__global__ void __launch_bounds__(kThreads)
    k_relax_tile(FamilyView fv, GraphView g, ClassView cv, DpView dp, TileArgs ta) {
  extern __shared__ __align__(16) unsigned char sm[];
  relax_body<W, NARROW, false>(fv, g, cv, dp, ta, blockIdx.x, blockIdx.y, gridDim.y, sm);
}

// wide bitsets (W >= 4): register cap for kTile3MinBlocks resident CTAs per SM
template <int W, bool NARROW>
__global__ void __launch_bounds__(kThreads, kTile3MinBlocks)
    k_relax_tile3(FamilyView fv, GraphView g, ClassView cv, DpView dp, TileArgs ta) {
  extern __shared__ __align__(16) unsigned char sm[];
  relax_body<W, NARROW, false>(fv, g, cv, dp, ta, blockIdx.x, blockIdx.y, gridDim.y, sm);
}

template <int W, bool NARROW>
static constexpr auto relax_tile_kernel() {
  if constexpr (W >= 4) return k_relax_tile3<W, NARROW>;
  else return k_relax_tile<W, NARROW>;
}

// A whole small family in ONE launch: one CTA per budget walks every level's
// tiles itself (rows in shared memory, no splits), with only CTA barriers
// between levels — for pruned families and chain-like lattices whose hundreds
// of levels are each far too small for the GPU (C1, C3).
template <int W, bool NARROW>
__global__ void __launch_bounds__(kThreads)
    k_solve_small(FamilyView fv, GraphView g, ClassView cv, DpView dp,
                  const TileArgs* __restrict__ levels, int nlev, int nb) {
  extern __shared__ __align__(16) unsigned char sm[];
  // level plans staged through shared memory one level ahead: the next
  // level's arguments are fetched while this one relaxes, not on the
  // level-to-level critical path
  constexpr int kTaWords = (int)(sizeof(TileArgs) / 4);
  static_assert(sizeof(TileArgs) % 4 == 0, "TileArgs is copied as 32-bit words");
  __shared__ __align__(16) TileArgs s_ta[2];
  const int b = blockIdx.y;
  if (nlev > 0)
    for (int k = threadIdx.x; k < kTaWords; k += kThreads)
      reinterpret_cast<int*>(&s_ta[0])[k] = reinterpret_cast<const int*>(&levels[0])[k];
  __syncthreads();
  for (int l = 0; l < nlev; l++) {
    const TileArgs ta = s_ta[l & 1];
    if (l + 1 < nlev)
      for (int k = threadIdx.x; k < kTaWords; k += kThreads)
        reinterpret_cast<int*>(&s_ta[(l + 1) & 1])[k] = reinterpret_cast<const int*>(&levels[l + 1])[k];
    for (int t = 0; t < ta.tiles; t++) {
      // the next tile / level reads this one (ld.ca, relax_body LDM 2) and
      // reuses its shared memory: the CTA barrier orders both
      relax_body<W, NARROW, true, true>(fv, g, cv, dp, ta, t, b, nb, sm);
      __syncthreads();
    }
  }
}

// Several consecutive small levels in ONE cooperative launch: every block
// walks the (tile, split, budget) virtual CTAs of a level, then a grid barrier
// publishes the level (its tiles were finalized by their last CTA) before the
// next one starts.  Removes the launch + ramp of each of the hundreds of
// narrow levels of deep lattices (C5: 516 levels).
#ifdef REMAT_RELAX_TRACE
__device__ unsigned long long g_relax_trace[600 * 296 * 4];
__device__ int g_relax_trace_meta[600 * 4];
#endif
template <int W, bool NARROW>
__global__ void __launch_bounds__(kThreads)
    k_relax_levels(FamilyView fv, GraphView g, ClassView cv, DpView dp,
                   const TileArgs* __restrict__ levels, int nlev, int nb) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char sm[];
  // the block's first tile of each level is set up between its arrival at
  // the barrier that ends the previous level and the wait (the loads overlap
  // the other blocks' finish)
  bool pre = false;
  if (nlev > 0 && blockIdx.x < levels[0].tiles * levels[0].splits * nb) {
    tile_setup<W, NARROW>(fv, cv, levels[0], blockIdx.x % (levels[0].tiles * levels[0].splits), sm);
    pre = true;
  }
  for (int l = 0; l < nlev; l++) {
    const TileArgs ta = levels[l];
    const int per = ta.tiles * ta.splits;
#ifdef REMAT_RELAX_TRACE
    auto stamp = [&](int ph) {
      if (threadIdx.x == 0 && l < 600 && blockIdx.x < 296) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_relax_trace[((size_t)l * 296 + blockIdx.x) * 4 + ph] = t;
      }
    };
    stamp(0);
#endif
    for (int v = blockIdx.x; v < per * nb; v += gridDim.x) {
      relax_body<W, NARROW, true>(fv, g, cv, dp, ta, v % per, v / per, nb, sm,
                                  pre && v == (int)blockIdx.x);
      __syncthreads();
    }
#ifdef REMAT_RELAX_TRACE
    stamp(1);
#endif
    // split barrier: arrive, set up the next level's first tile, then wait
    auto token = grid.barrier_arrive();
    pre = false;
    if (l + 1 < nlev) {
      const TileArgs& tn = levels[l + 1];
      const int pn = tn.tiles * tn.splits;
      if ((int)blockIdx.x < pn * nb) {
        tile_setup<W, NARROW>(fv, cv, tn, blockIdx.x % pn, sm);
        pre = true;
      }
    }
    grid.barrier_wait(std::move(token));
  }
}

template <typename Key>
__global__ void k_fill(Key* p, size_t n, Key v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

template <bool NARROW>
__global__ void k_dp_init(DpView dp, long long F, int nb) {
  using E = typename Traits<NARROW>::E;
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  E e{};
  e.t = 0;
  e.m = 0;
  reinterpret_cast<E*>(dp.fe)[(long long)b * dp.slots] = e;  // foff[0] == 0: the empty set
  dp.parent[(long long)b * dp.slots] = -1;
  dp.flen[(size_t)b * F] = 1;
  dp.ccount[(size_t)b * F] = 1;
  dp.mmin[(size_t)b * F] = 0;
}

// SearchStats, recomputed from the final table (Appendix A.3).
static __global__ void k_dp_stats(DpView dp, long long F, long long* __restrict__ out) {
  __shared__ long long scr[4][32];
  const int b = blockIdx.x;
  long long sv = 0, te = 0, tr = 0, np = 0;
  for (long long i = threadIdx.x; i < F; i += blockDim.x) {
    sv += dp.flen[(size_t)b * F + i];
    te += dp.ccount[(size_t)b * F + i];
    tr += (long long)dp.trans[(size_t)b * F + i];
    np += (long long)dp.npairs[(size_t)b * F + i];
  }
  sv = warp_sum(sv);
  te = warp_sum(te);
  tr = warp_sum(tr);
  np = warp_sum(np);
  if ((threadIdx.x & 31) == 0) {
    scr[0][threadIdx.x >> 5] = sv;
    scr[1][threadIdx.x >> 5] = te;
    scr[2][threadIdx.x >> 5] = tr;
    scr[3][threadIdx.x >> 5] = np;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); k++) {
      sv += scr[0][k];
      te += scr[1][k];
      tr += scr[2][k];
      np += scr[3][k];
    }
    out[b * 5 + 0] = sv;        // states_visited
    out[b * 5 + 1] = te;        // table_entries
    out[b * 5 + 2] = tr;        // transitions
    out[b * 5 + 3] = te - sv;   // dominated_skipped
    out[b * 5 + 4] = np;        // comparable pairs P
  }
}

// K6: parent walk from (V, t*) back to ∅ (planner.py:180-189), one warp per
// budget.  Each step recomputes dt(parent, j) to recover the parent's t and
// finds that entry in the parent's frontier with a warp-wide ballot.
// expect[b] = {t*, m_final, budget, 1}; klen[b] = k (0 when infeasible,
// -1 on an inconsistent table).
template <int W, bool NARROW>
__global__ void k_reconstruct(FamilyView fv, GraphView g, DpView dp, int n,
                              int* __restrict__ path, u64* __restrict__ chain_out,
                              int* __restrict__ klen, long long* __restrict__ expect) {
  using E = typename Traits<NARROW>::E;
  const int b = blockIdx.x, lane = threadIdx.x;
  const long long F = fv.F;
  const long long fbase = (long long)b * dp.slots;
  const E* fe = reinterpret_cast<const E*>(dp.fe);
  int* pth = path + (size_t)b * (n + 2);
  long long j = F - 1;
  if (dp.flen[(size_t)b * F + j] == 0) {
    if (lane == 0) klen[b] = 0;
    return;
  }
  long long at = fbase + fv.foff[j];
  E cur = fe[at];
  int cpar = dp.parent[at];
  if (lane == 0) {
    expect[b * 4 + 0] = cur.t;
    expect[b * 4 + 1] = (long long)cur.m;
    expect[b * 4 + 2] = dp.budgets[b];
    expect[b * 4 + 3] = 1;
  }
  int len = 0;
  bool bad = false;
  while (true) {
    if (lane == 0) pth[len] = (int)j;
    len++;
    if (j == 0) break;
    if (len > n + 1 || cpar < 0) {
      bad = true;
      break;
    }
    const long long par = cpar;
    long long ts = 0;
    if (lane < W)
      ts = word_weight(fv.masks[(size_t)lane * F + par] & fv.bound[(size_t)lane * F + j], lane,
                       g.T);
    ts = warp_sum(ts);
    const long long dt = fv.TLnb[j] - fv.TL[par] + ts;
    const long long tp = (long long)cur.t - dt;
    const int nfp = dp.flen[(size_t)b * F + par];
    const long long pb = fbase + fv.foff[par];
    bool found = false;
    for (int s0 = 0; s0 < nfp && !found; s0 += 32) {
      int s = s0 + lane;
      bool hit = s < nfp && (long long)fe[pb + s].t == tp;
      unsigned bal = __ballot_sync(kFull, hit);
      if (bal) {
        const long long a2 = pb + s0 + __ffs(bal) - 1;
        cur = fe[a2];
        cpar = dp.parent[a2];
        found = true;
      }
    }
    if (!found) {
      bad = true;
      break;
    }
    j = par;
  }
  __syncwarp();
  if (bad) {
    if (lane == 0) klen[b] = -1;
    return;
  }
  const int k = len - 1;
  for (int s = 0; s < k; s++) {
    int idx = pth[len - 2 - s];
    if (lane < W)
      chain_out[((size_t)b * (n + 1) + s) * W + lane] = fv.masks[(size_t)lane * F + idx];
  }
  if (lane == 0) klen[b] = k;
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------

static constexpr int kSmemLimit = 200 * 1024;  // dynamic shared bytes per CTA
static constexpr int kRowBudget = 64 * 1024;   // tile rows per CTA (4 CTAs/SM)


// The solve in three phases so the level loop can be driven from outside
// (level sharding, shard.cu): begin (buffers + the empty set), one call per
// level for the targets [lo, hi) of that level, finish (reconstruction,
// figures, statistics, copy-out).
template <int W, bool NARROW>
int begin_w(remat_family_s* f, const std::vector<long long>& budgets, int objective) {
  using E = typename Traits<NARROW>::E;
  remat_graph_s* g = f->g;
  cudaStream_t s = g->stream;
  const int nb = (int)budgets.size();
  const int n = g->n;
  const long long F = f->F;
  int rc;
  if ((rc = f->fe.ensure((size_t)nb * f->slots * sizeof(E))) < 0 ||
      (rc = f->parent.ensure((size_t)nb * f->slots)) < 0 ||
      (rc = f->flen.ensure((size_t)nb * F)) < 0 || (rc = f->ccount.ensure((size_t)nb * F)) < 0 ||
      (rc = f->mmin.ensure((size_t)nb * F)) < 0 || (rc = f->trans.ensure((size_t)nb * F)) < 0 ||
      (rc = f->npairs.ensure((size_t)nb * F)) < 0 || (rc = f->budgets.ensure(nb)) < 0 ||
      (rc = f->results.ensure((size_t)nb * 20)) < 0 ||
      (rc = f->chain_out.ensure((size_t)nb * (n + 1) * W)) < 0 ||
      (rc = f->cached_out.ensure((size_t)nb * (n + 1) * W)) < 0 ||
      (rc = f->stage_out.ensure((size_t)nb * (n + 1))) < 0 ||
      (rc = f->chain_idx.ensure((size_t)nb * (n + 2) + nb)) < 0 ||
      (rc = f->terms.ensure((size_t)nb * (n + 1) * 4)) < 0 ||
      (rc = f->stage_bound.ensure((size_t)nb * (n + 1) * W)) < 0)
    return rc;
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev_slot(g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(relax_tile_kernel<W, NARROW>(),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr_set[dev_slot(g->device)] = true;
  }
  f->cur_nb = nb;
  f->cur_objective = objective;
  f->cur_narrow = NARROW;
  f->launches0 = remat_kernel_launch_count();
  f->relax_launches = 0;
  RM_CUDA(cudaMemcpyAsync(f->budgets.p, budgets.data(), sizeof(long long) * nb,
                          cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaEventRecord(g->ev.e[3], s));
  // every per-member array starts zeroed so a level-sharded replica can be
  // filled in any order; trans/npairs are accumulated atomically
  RM_CUDA(cudaMemsetAsync(f->trans.p, 0, sizeof(u64) * nb * F, s));
  RM_CUDA(cudaMemsetAsync(f->npairs.p, 0, sizeof(u64) * nb * F, s));
  RM_CUDA(cudaMemsetAsync(f->flen.p, 0, sizeof(int) * nb * F, s));
  RM_CUDA(cudaMemsetAsync(f->ccount.p, 0, sizeof(int) * nb * F, s));
  if (f->sparse) {
    if ((rc = f->sparse_err.ensure(1)) < 0) return rc;
    RM_CUDA(cudaMemsetAsync(f->sparse_err.p, 0, sizeof(int), s));
  }
  k_dp_init<NARROW><<<(nb + 127) / 128, 128, 0, s>>>(f->dp_view(), F, nb);
  RM_LAUNCHED();
  // per-level scratch for the widest level: tile counters (zero) and global
  // rows (INF); the relaxation kernels leave both as they found them
  using Key = typename Traits<NARROW>::Key;
  long long wmax = 1, rmax = 1;
  for (int l = 1; l <= n; l++) {
    wmax = std::max(wmax, f->level_start[l + 1] - f->level_start[l]);
    rmax = std::max(rmax, f->level_maxR[l]);
  }
  const size_t need_ctr = (size_t)2 * nb * wmax;
  // (rows of the last partial tile: up to 63 past the level for k_relax_wide)
  const size_t need_rows = (size_t)nb * (wmax + 64) * rmax;
  if (need_ctr > f->ctr_cap) {
    if ((rc = f->ctr.ensure(need_ctr)) < 0) return rc;
    f->ctr_cap = need_ctr;
    RM_CUDA(cudaMemsetAsync(f->ctr.p, 0, sizeof(unsigned) * need_ctr, s));
  }
  if (need_rows > f->grow_cap || f->grow_key != (int)sizeof(Key)) {
    if ((rc = f->rowscratch.ensure((need_rows * sizeof(Key) + 7) / 8)) < 0) return rc;
    f->grow_cap = need_rows;
    f->grow_key = (int)sizeof(Key);
    k_fill<Key><<<(unsigned)std::min<size_t>((need_rows + 255) / 256, 4096), 256, 0, s>>>(
        reinterpret_cast<Key*>(f->rowscratch.p), need_rows, Traits<NARROW>::INF);
    RM_LAUNCHED();
  }
  return REMAT_OK;
}

template <int W, bool NARROW>
int plan_level_w(remat_family_s* f, int lvl, long long lo, long long hi, TileArgs& ta,
                        long long max_vctas = 0, bool single_cta = false) {
  using Key = typename Traits<NARROW>::Key;
  remat_graph_s* g = f->g;
  cudaStream_t s = g->stream;
  const int nb = f->cur_nb;
  int rc;
  const DpView dp = f->dp_view();
  const FamilyView fv = f->view();
  const GraphView gv = g->view();
  const ClassView cv = g->classes();
  const int K = cv.K;
  const int num_sms = sm_count(g->device);
  const long long target_ctas = (long long)num_sms * 4;  // resident CTAs at 256 threads
  const long long j0 = f->level_start[lvl];               // predecessors: [0, j0)
  const long long width = hi - lo;
  const int R = (int)f->level_maxR[lvl];
  // targets per tile: as many rows as fit the per-CTA row budget, <= width
  // long frontiers (minimize with varied T_v) take 16 targets per tile with
  // half-width predecessor chunks (records stay 256 per warp): every entry
  // load feeds twice the candidates (U-Net c=8 relax 14.96 -> 14.24 ms);
  // short frontiers keep 8 (C5 p=0.2: 151 -> 170 ms at 16).  Swept 8-32 on
  // the B200 (tools/relax_time.py); REMAT_TILE_TJ overrides.
  static const int tile_tj_env = [] {
    const char* e = getenv("REMAT_TILE_TJ");
    return e ? std::max(1, std::min(kMaxTJ, atoi(e))) : 0;
  }();
  const bool long_frontiers = f->cur_objective == REMAT_MINIMIZE && !g->t_uniform;
  const int tile_tj = tile_tj_env ? tile_tj_env : (long_frontiers ? 2 * kTileTJ : kTileTJ);
  int TJ = (int)std::min<long long>(std::min<long long>(tile_tj, width),
                                    std::max<long long>(1, kRowBudget / ((long long)R * sizeof(Key))));
  const long long nch = (j0 + 31) / 32;
  // fewer targets per tile where the level is too small to give every
  // resident warp a couple of (tile, chunk) tasks
  // (32 tasks per SM and 3 resident-CTA rounds of splits: swept on the B200
  // against 16-64 and 1-8; U-Net relax -2.2 %, C5 p=0.3 -3.6 % vs 64 / 2)
  const long long want = (long long)num_sms * 32;
  while (!single_cta && TJ > 1 && ((width + TJ - 1) / TJ) * nch * nb < want) TJ = (TJ + 1) / 2;
  bool cls = cv.enabled && (long long)TJ * K * W * 8 <= 16 * 1024;
  ta = tile_layout<W, NARROW>(TJ, R, K, true, cls);
  // fewer targets per tile where the shared-memory tile would cost a resident
  // CTA: the register-bound occupancy (4 CTAs/SM at 64 registers) is worth
  // more than two more rows (PSPNet full sweep, rows of 1.4 k slots: 8 -> 6
  // targets kept a third CTA per SM resident, -9 %)
  if (!single_cta) {
    static const int occ_env = [] {  // REMAT_TILE_OCC: resident-CTA target (A/B)
      const char* e = getenv("REMAT_TILE_OCC");
      return e ? std::max(1, atoi(e)) : 0;
    }();
    const int occ = occ_env ? occ_env : (W >= 4 ? kTile3MinBlocks : 4);
    const int per_cta = (228 << 10) / occ - (1 << 10);
    while (TJ > 1 && ta.bytes > per_cta) {
      --TJ;
      cls = cv.enabled && (long long)TJ * K * W * 8 <= 16 * 1024;
      ta = tile_layout<W, NARROW>(TJ, R, K, true, cls);
    }
  }
  if (ta.bytes > kSmemLimit) ta = tile_layout<W, NARROW>(TJ, R, K, false, cls);
  const long long tiles = (width + TJ - 1) / TJ;
  // narrower predecessor chunks where even one target per tile leaves the GPU
  // short of (tile, chunk) tasks (chain-like levels: one target, hundreds of
  // predecessors with long frontiers)
  int cw = ta.qlanes;  // (32 up to 8 targets per tile: records are qlanes x TJ per warp)
  if (!single_cta) {
    // long frontiers (minimize, varied T_v: hundreds of entries per cell)
    // go down to one predecessor per warp, so a chain-like level's items
    // spread over the most CTAs (C1 3.8 -> 3.2 ms); short ones (maximize,
    // uniform T_v) keep >= 4 per chunk
    const int mincw = f->cur_objective == REMAT_MINIMIZE && !g->t_uniform ? 1 : 4;
    while (cw > mincw && tiles * ((j0 + cw - 1) / cw) * nb < want / 4) cw /= 2;
  }
  const long long nchw = (j0 + cw - 1) / cw;
  // split the predecessor scan across CTAs when the level alone cannot fill
  // the GPU (narrow levels near ∅ and V; SURVEY §7 hard part 5)
  long long splits = (3 * target_ctas + tiles * nb - 1) / (tiles * nb);
  if (max_vctas > 0) splits = max_vctas / (tiles * nb);  // persistent: one round per block
  if (single_cta) splits = 1;
  // (rounded up: every chunk of a narrow level is some warp's static first one)
  // (fewer splits — 2-16 chunks per warp at least — measured slower on every
  // config, tools/c5_small.py: the chunks' own latency, not the fold, bounds a
  // narrow level; tools/relax_trace.py)
  splits = std::max(1LL, std::min(splits, (nchw + kWarps - 1) / kWarps));
  ta.jbase = lo;
  ta.pend = j0;
  ta.width = (int)width;
  ta.splits = (int)splits;
  ta.grow = nullptr;
  ta.rows_pb = (int)(tiles * TJ);
  ta.tiles = (int)tiles;
  ta.ctr_stride = (int)tiles;
  ta.cw = std::min(cw, ta.qlanes);  // records: qlanes x TJ slots per warp
  ta.probe = g->t_uniform;
  if (single_cta && f->cur_objective == REMAT_MINIMIZE) {
    // one CTA walks the level: chunks narrow enough that every warp gets some,
    // since a predecessor's items stay with the warp that tested it and
    // minimize frontiers run to hundreds of entries (maximize frontiers hold a
    // few: wide chunks are cheaper there)
    ta.cw = (int)std::max<long long>(4, std::min<long long>(32, j0 / (2 * kWarps)));
    ta.cw = std::min(ta.cw, ta.qlanes);
  }
  ta.ctr = f->ctr.p;  // [nb][tiles] chunk counters + [nb][tiles] done counters, all zero
  if ((size_t)2 * nb * tiles > f->ctr_cap)
    return fail(REMAT_ERR_INTERNAL, "tile counter capacity exceeded");
  if (splits > 1 || !ta.smem_rows) {
    const size_t cells = (size_t)nb * tiles * TJ * R;
    if (cells > f->grow_cap) return fail(REMAT_ERR_INTERNAL, "row scratch capacity exceeded");
    ta.grow = f->rowscratch.p;  // all INF between levels
  }
  return REMAT_OK;
}

}  // namespace remat
#include "relax_pm.cuh"
#include "relax_sparse.cuh"
namespace remat {

// Wide levels of long-frontier (minimize, varied T_v) solves of a budget
// batch go to the predecessor-major cluster kernel (relax_pm.cuh);
// REMAT_PM=0/1 forces it off/on.
template <int W, bool NARROW>
static bool use_pm(remat_family_s* f, long long width) {
  static const int mode = [] {
    const char* e = getenv("REMAT_PM");
    return e ? atoi(e) : -1;
  }();
  if (!NARROW || mode == 0) return false;
  if (mode == 1) return true;
  // measured on the B200 (tools/wd_probe.py): PSPNet 64-budget sweep relax
  // 190 -> 154 ms; single-budget U-Net c=8 14.8 -> 49.9 ms (a batch of one
  // budget leaves the cluster grid too small and every predecessor's entry
  // load exposed) -- so batched sweeps only
  return f->cur_objective == REMAT_MINIMIZE && !f->g->t_uniform && width >= 64 &&
         f->cur_nb >= 8;
}

template <int W, bool NARROW>
int level_w(remat_family_s* f, int lvl, long long lo, long long hi) {
  TileArgs ta;
  if (hi <= lo) return REMAT_OK;
  if constexpr (!NARROW) {
    if (f->sparse) return launch_sparse<W>(f, lvl, lo, hi);
  }
  if constexpr (NARROW) {
    PmArgs pa;
    if (use_pm<W, NARROW>(f, hi - lo) && plan_pm<W>(f, lvl, lo, hi, pa)) return launch_pm<W>(f, pa);
  }
  int rc = plan_level_w<W, NARROW>(f, lvl, lo, hi, ta);
  if (rc < 0) return rc;
  relax_tile_kernel<W, NARROW>()<<<dim3((unsigned)(ta.tiles * ta.splits), (unsigned)f->cur_nb),
                                   kThreads, ta.bytes, f->g->stream>>>(f->view(), f->g->view(), f->g->classes(),
                                                      f->dp_view(), ta);
  RM_LAUNCHED();
  f->relax_launches++;
  return REMAT_OK;
}

// A run of consecutive small levels (full target ranges) as one cooperative
// k_relax_levels launch.
template <int W, bool NARROW>
int levels_w(remat_family_s* f, const std::vector<int>& lvls) {
  std::vector<TileArgs> tas(lvls.size());
  int maxbytes = 0, rc;
  if (f->sparse) {  // sparse cells: one launch per level
    for (int l : lvls)
      if ((rc = level_w<W, NARROW>(f, l, f->level_start[l], f->level_start[l + 1])) < 0) return rc;
    return REMAT_OK;
  }
  static bool attr[kMaxDevices] = {};
  if (!attr[dev_slot(f->g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(k_relax_levels<W, NARROW>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr[dev_slot(f->g->device)] = true;
  }
  const int num_sms0 = sm_count(f->g->device);
  // size the grid from a first plan, then re-plan every level for one round
  for (int pass = 0; pass < 2; pass++) {
    long long grid = 0;
    if (pass == 1) {
      int b0 = 0;
      RM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k_relax_levels<W, NARROW>,
                                                            kThreads, maxbytes));
      grid = (long long)num_sms0 * std::min(std::max(b0, 1), 4);
    }
    maxbytes = 0;
    for (size_t k = 0; k < lvls.size(); k++) {
      const int l = lvls[k];
      if ((rc = plan_level_w<W, NARROW>(f, l, f->level_start[l], f->level_start[l + 1], tas[k],
                                        grid)) < 0)
        return rc;
      maxbytes = std::max(maxbytes, tas[k].bytes);
    }
  }
  int bps = 0;
  RM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_relax_levels<W, NARROW>, kThreads,
                                                        maxbytes));
  if (bps < 1) {  // cannot be co-resident: per-level launches instead
    for (int l : lvls)
      if ((rc = level_w<W, NARROW>(f, l, f->level_start[l], f->level_start[l + 1])) < 0) return rc;
    return REMAT_OK;
  }
  const int num_sms = sm_count(f->g->device);
  cudaStream_t s = f->g->stream;
  if ((rc = f->levelargs.ensure(tas.size() * sizeof(TileArgs))) < 0) return rc;
  RM_CUDA(cudaMemcpyAsync(f->levelargs.p, tas.data(), tas.size() * sizeof(TileArgs),
                          cudaMemcpyHostToDevice, s));
  FamilyView fv = f->view();
  GraphView gv = f->g->view();
  ClassView cv = f->g->classes();
  DpView dp = f->dp_view();
  const TileArgs* la = reinterpret_cast<const TileArgs*>(f->levelargs.p);
  int nl = (int)tas.size(), nb = f->cur_nb;
  void* args[] = {&fv, &gv, &cv, &dp, (void*)&la, &nl, &nb};
  RM_CUDA(cudaLaunchCooperativeKernel((const void*)k_relax_levels<W, NARROW>,
                                      dim3((unsigned)(num_sms * std::min(bps, 4))), dim3(kThreads),
                                      args, (size_t)maxbytes, s));
  RM_LAUNCHED();
  f->relax_launches++;
  return REMAT_OK;
}

// The whole family in one k_solve_small launch (one CTA per budget).  Returns
// 1 without launching when some level's rows do not fit shared memory.
template <int W, bool NARROW>
int small_w(remat_family_s* f) {
  if (f->sparse) return 1;  // sparse cells: the per-level path
  const int n = f->g->n;
  std::vector<TileArgs> tas;
  int maxbytes = 0, rc;
  for (int l = 1; l <= n; l++) {
    const long long j0 = f->level_start[l], j1 = f->level_start[l + 1];
    if (j1 == j0) continue;
    TileArgs ta;
    if ((rc = plan_level_w<W, NARROW>(f, l, j0, j1, ta, 0, true)) < 0) return rc;
    if (!ta.smem_rows) return 1;
    maxbytes = std::max(maxbytes, ta.bytes);
    tas.push_back(ta);
  }
  // budgets walk the levels independently: give each budget its own counters
  int stride = 1;
  for (auto& ta : tas) stride = std::max(stride, ta.tiles);
  for (auto& ta : tas) ta.ctr_stride = stride;
  static bool attr[kMaxDevices] = {};
  if (!attr[dev_slot(f->g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(k_solve_small<W, NARROW>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr[dev_slot(f->g->device)] = true;
  }
  cudaStream_t s = f->g->stream;
  if ((rc = f->levelargs.ensure(tas.size() * sizeof(TileArgs))) < 0) return rc;
  RM_CUDA(cudaMemcpyAsync(f->levelargs.p, tas.data(), tas.size() * sizeof(TileArgs),
                          cudaMemcpyHostToDevice, s));
  k_solve_small<W, NARROW><<<dim3(1, (unsigned)f->cur_nb), kThreads, (size_t)maxbytes, s>>>(
      f->view(), f->g->view(), f->g->classes(), f->dp_view(),
      reinterpret_cast<const TileArgs*>(f->levelargs.p), (int)tas.size(), f->cur_nb);
  RM_LAUNCHED();
  f->relax_launches++;
  return REMAT_OK;
}

template <int W, bool NARROW>
int finish_w(remat_family_s* f, remat_plan_info* info, u64* chain_masks,
                    u64* cached_masks, long long* stage_memory) {
  remat_graph_s* g = f->g;
  cudaStream_t s = g->stream;
  const int nb = f->cur_nb;
  const int n = g->n;
  const long long F = f->F;
  int rc;
  const DpView dp = f->dp_view();
  const FamilyView fv = f->view();
  const GraphView gv = g->view();
  Events& ev = g->ev;
  RM_CUDA(cudaEventRecord(ev.e[4], s));
  long long* expect = f->results.p;           // [nb][4]
  long long* stats = f->results.p + nb * 4;   // [nb][5]
  long long* evres = f->results.p + nb * 9;   // [nb][8]
  int* klen = f->chain_idx.p + (size_t)nb * (n + 2);
  k_reconstruct<W, NARROW><<<nb, 32, 0, s>>>(fv, gv, dp, n, f->chain_idx.p, f->chain_out.p, klen,
                                             expect);
  RM_LAUNCHED();
  if ((rc = evaluate_chains(g, nb, f->chain_out.p, klen, expect, f->stage_out.p,
                            f->cached_out.p, evres, f->terms.p, f->stage_bound.p)) < 0)
    return rc;
  k_dp_stats<<<nb, 1024, 0, s>>>(dp, F, stats);
  RM_LAUNCHED();
  RM_CUDA(cudaEventRecord(ev.e[5], s));
  std::vector<long long> hres((size_t)nb * 17);
  RM_CUDA(cudaMemcpyAsync(hres.data(), f->results.p, sizeof(long long) * nb * 17,
                          cudaMemcpyDeviceToHost, s));
  std::vector<u64> hchain, hcached;
  std::vector<long long> hstage;
  if (chain_masks) hchain.resize((size_t)nb * (n + 1) * W);
  if (cached_masks) hcached.resize((size_t)nb * (n + 1) * W);
  if (stage_memory) hstage.resize((size_t)nb * (n + 1));
  if (chain_masks)
    RM_CUDA(cudaMemcpyAsync(hchain.data(), f->chain_out.p, hchain.size() * 8,
                            cudaMemcpyDeviceToHost, s));
  if (cached_masks)
    RM_CUDA(cudaMemcpyAsync(hcached.data(), f->cached_out.p, hcached.size() * 8,
                            cudaMemcpyDeviceToHost, s));
  if (stage_memory)
    RM_CUDA(cudaMemcpyAsync(hstage.data(), f->stage_out.p, hstage.size() * 8,
                            cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaEventRecord(ev.e[6], s));
  RM_CUDA(cudaStreamSynchronize(s));
  if (f->sparse) {
    int err = 0;
    RM_CUDA(cudaMemcpy(&err, f->sparse_err.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (err == 1)
      return fail(REMAT_ERR_RANGE, "a DP cell holds more than " + std::to_string(f->hcap * 3 / 4) +
                                       " distinct overhead values (sparse-cell capacity); raise "
                                       "REMAT_SPARSE_CELLS");
    if (err)
      return fail(REMAT_ERR_RANGE, "a DP frontier holds more than " + std::to_string(f->fcap) +
                                       " entries (sparse frontier capacity); raise "
                                       "REMAT_SPARSE_FRONTIER");
  }
  float relax_ms = 0, finish_ms = 0, total_ms = 0;
  cudaEventElapsedTime(&relax_ms, ev.e[3], ev.e[4]);
  cudaEventElapsedTime(&finish_ms, ev.e[4], ev.e[5]);
  cudaEventElapsedTime(&total_ms, ev.e[3], ev.e[6]);
  f->timings.relax_ms = relax_ms;
  f->timings.finish_ms = finish_ms;
  f->timings.total_ms = total_ms;
  f->timings.relax_launches = f->relax_launches;
  f->timings.kernel_launches = remat_kernel_launch_count() - f->launches0;

  const int Wu = g->W;
  for (int b = 0; b < nb; b++) {
    remat_plan_info& o = info[b];
    const long long* st = hres.data() + nb * 4 + b * 5;
    const long long* er = hres.data() + nb * 9 + b * 8;
    if (b == 0) f->timings.comparable_pairs = st[4];
    o.stats.states_visited = st[0];
    o.stats.table_entries = st[1];
    o.stats.transitions = st[2];
    o.stats.dominated_skipped = st[3];
    o.k = (int)er[1];
    o.status = (int)er[0];
    o.objective_value = er[2];
    o.overhead = er[2];
    o.peak_memory = er[3];
    o.cached_total = er[4];
    const size_t rows = (size_t)(n + 1);
    if (o.status == REMAT_OK) {
      for (int q = 0; q < o.k; q++)
        for (int w = 0; w < Wu; w++) {
          size_t src = ((size_t)b * rows + q) * W + w, dst = ((size_t)b * rows + q) * Wu + w;
          if (chain_masks) chain_masks[dst] = hchain[src];
          if (cached_masks) cached_masks[dst] = hcached[src];
        }
      if (stage_memory)
        for (int q = 0; q < o.k; q++) stage_memory[b * rows + q] = hstage[b * rows + q];
    }
  }
  return REMAT_OK;
}

}  // namespace remat
