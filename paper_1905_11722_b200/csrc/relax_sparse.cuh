// relax_sparse.cuh — the relaxation with SPARSE cells, for graphs whose total
// compute cost T(V) is too large for a dense overhead row per member
// (T(V) >= 2^24: FLOP-valued compute costs).  Included by relax_impl.cuh.
//
// The reference keeps each DP cell as a dict keyed by the overhead t
// (DpTable, planner.py:82-92), so it has no bound on T.  Here a member's cell
// is keyed by its DISTINCT overhead values, in two passes over the
// candidates of one target j (one CTA per target and budget):
//
//   1. collect: every candidate (t + dt_ij, ·) of every predecessor entry
//      that passes the budget test inserts its overhead t2 into a
//      shared-memory hash set; the set is then compacted and bitonic-sorted —
//      the member's cells in t order (|cell| of the reference, 171-174);
//   2. relax: every candidate again, min-reduced into the row slot of its
//      t2's rank (binary search in the sorted cells): first the smallest m2,
//      then (third pass) the smallest predecessor index i among the
//      candidates with that m2 — the same lexicographic (m2, i) minimum as the
//      dense kernels' packed keys (strict `<` in family order,
//      planner.py:172-175) without their M(V)·2^IB < 2^64 bound.
//
// The frontier (strict prefix-min of m in t order, t descending for maximize,
// planner.py:153-161) then comes out of the ranked row exactly as from a dense
// row, with 64-bit t in the 16-byte entries.  A member may hold at most
// 3/4 · hcap distinct overhead values (REMAT_SPARSE_CELLS, default 2^20; up
// to 8192 the cells live in shared memory, beyond in a global scratch slice
// per CTA) and a frontier of at most REMAT_SPARSE_FRONTIER entries (default
// 4096 slots per member); beyond either the solve fails with a range error
// instead of dropping cells.
// Throughput is not the point of this path: it is the generality fallback
// (every named config runs the dense kernels).

namespace remat {

constexpr u64 kSpEmpty = ~0ull;

struct SpArgs {
  long long jbase, pend, width;
  int H, logH;
  int* err;
  u64* scratch;  // [gridDim.y][gridDim.x][2H] when the cells do not fit shared memory
};

__device__ __forceinline__ void sp_min64(u64* p, u64 key) {  // shared 64-bit min (CAS loop)
  u64 old = *p;
  while (key < old) {
    const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(p), old, key);
    if (prev == old) break;
    old = prev;
  }
}

template <int W>
__global__ void __launch_bounds__(kThreads)
    k_relax_sparse(FamilyView fv, GraphView g, DpView dp, SpArgs sa) {
  extern __shared__ __align__(16) u64 sp_sm[];
  u64* const base = sa.scratch ? sa.scratch + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 3 * sa.H
                               : sp_sm;
  u64* cells = base;          // [H] hash set, then the sorted cell list
  u64* row = base + sa.H;     // [H] ranked row: smallest m2 (scratch for the sort first)
  unsigned* rowi = reinterpret_cast<unsigned*>(base + 2 * sa.H);  // [H] its smallest i
  __shared__ u64 sL[W], sB[W];
  __shared__ long long sc[4];
  __shared__ unsigned long long s_tr, s_np;
  __shared__ int s_n, s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = sa.H;
  const long long F = fv.F;
  const int b = blockIdx.y;
  for (long long task = blockIdx.x; task < sa.width; task += gridDim.x) {
  const long long j = sa.jbase + task;
  __syncthreads();  // the previous target's frontier is written
  if (tid < W) {
    sL[tid] = fv.masks[(size_t)tid * F + j];
    sB[tid] = fv.bound[(size_t)tid * F + j];
  }
  if (tid == 0) {
    sc[0] = fv.ML[j];
    sc[1] = fv.base[j];
    sc[2] = fv.TLnb[j];
    sc[3] = fv.Mb[j];
    s_tr = s_np = 0;
    s_n = 0;
    s_bad = 0;
  }
  for (int e = tid; e < 2 * H + H / 2; e += kThreads) base[e] = kSpEmpty;
  __syncthreads();
  const long long B = dp.budgets[b];
  const long long fbase = (long long)b * dp.slots;
  const int* flen_b = dp.flen + (size_t)b * F;
  const long long* mmin_b = dp.mmin + (size_t)b * F;
  const EntryW* fe = reinterpret_cast<const EntryW*>(dp.fe);
  int n = 0;
  // passes: 0 collect the cells, 1 the smallest m2 per cell, 2 the smallest
  // i among its candidates with that m2 — the lexicographic (m2, i) minimum of
  // the dense kernels' packed keys, without their M(V)·2^IB < 2^64 bound
  for (int pass = 0; pass < 3; pass++) {
    unsigned long long tr = 0, np = 0;
    for (long long i = tid; i < sa.pend; i += kThreads) {
      u64 Li[W];
      u64 out = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        Li[w] = __ldg(fv.masks + (size_t)w * F + i);
        out |= Li[w] & ~sL[w];
      }
      if (out) continue;  // L_i ⊄ L_j
      const int fl = flen_b[i];
      tr += (unsigned)fl;
      np++;
      if (fl == 0) continue;
      long long ts = 0, ms = 0;  // T and M of L_i ∩ ∂L_j
#pragma unroll
      for (int w = 0; w < W; w++) {
        u64 x = Li[w] & sB[w];
        while (x) {
          const int v = w * 64 + __ffsll((long long)x) - 1;
          x &= x - 1;
          ts += __ldg(g.T + v);
          ms += __ldg(g.M + v);
        }
      }
      const long long fixed = 2 * (sc[0] - __ldg(fv.ML + i)) + sc[1];
      const long long dt = sc[2] - __ldg(fv.TL + i) + ts;
      const long long dm = sc[3] - ms;
      const long long cap = B - fixed;
      if (cap < mmin_b[i]) continue;
      const EntryW* src = fe + fbase + fv.foff[i];
      // m falls along the frontier: the passing entries are a suffix
      for (int e = fl - 1; e >= 0; e--) {
        const EntryW x = src[e];
        if (x.m > cap) break;
        const u64 t2 = x.t + (u64)dt;
        if (pass == 0) {
          unsigned h = (unsigned)((t2 * 0x9E3779B97F4A7C15ull) >> (64 - sa.logH));
          for (int probe = 0; probe < H; probe++, h = (h + 1) & (H - 1)) {
            const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(cells + h), kSpEmpty, t2);
            if (old == kSpEmpty) {
              if (atomicAdd(&s_n, 1) >= H * 3 / 4) s_bad = 1;
              break;
            }
            if (old == t2) break;
          }
          if (s_bad) break;
        } else {
          int lo = 0, hi = n;  // first cell >= t2 (it is there: pass 0 inserted it)
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cells[mid] < t2) lo = mid + 1;
            else hi = mid;
          }
          const u64 m2 = (u64)(x.m + dm);
          if (pass == 1) sp_min64(row + lo, m2);
          else if (row[lo] == m2) atomicMin(rowi + lo, (unsigned)i);
        }
      }
    }
    if (pass == 0) {
      atomicAdd(&s_tr, tr);
      atomicAdd(&s_np, np);
    }
    __syncthreads();
    if (pass >= 1) continue;
    if (s_bad) {
      if (tid == 0) atomicExch(sa.err, 1);
      return;  // (uniform: s_bad was read after the barrier)
    }
    // compact the set into row[0, n), bitonic-sort it there, copy back
    n = s_n;
    __syncthreads();
    if (tid == 0) s_n = 0;
    __syncthreads();
    for (int e = tid; e < H; e += kThreads) {
      const u64 v = cells[e];
      if (v != kSpEmpty) row[atomicAdd(&s_n, 1)] = v;
    }
    __syncthreads();
    int P = 1;
    while (P < n) P <<= 1;
    for (int e = n + tid; e < P; e += kThreads) row[e] = kSpEmpty;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int h = k >> 1; h > 0; h >>= 1) {
        for (int e = tid; e < P; e += kThreads) {
          const int l = e ^ h;
          if (l > e) {
            const u64 a = row[e], c = row[l];
            const bool up = (e & k) == 0;
            if ((a > c) == up) {
              row[e] = c;
              row[l] = a;
            }
          }
        }
        __syncthreads();
      }
    for (int e = tid; e < H; e += kThreads) {
      cells[e] = e < n ? row[e] : kSpEmpty;
      row[e] = kSpEmpty;
    }
    __syncthreads();
  }
  // ---- the frontier: strict prefix-min of m over the cells in t order
  // (descending for maximize), one warp, as finalize_row_warp
  if (warp == 0) {
    const bool mx = dp.maximize;
    const int per = (n + 31) / 32;
    const int s0 = min(n, lane * per), s1 = min(n, s0 + per);
    auto at = [&](int s) { return mx ? n - 1 - s : s; };
    u64 lmin = kSpEmpty;
    for (int s = s0; s < s1; s++) {
      const u64 m = row[at(s)];
      lmin = m < lmin ? m : lmin;
    }
    const u64 incl = warp_inclusive_min(lmin);
    u64 pm = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) pm = kSpEmpty;
    int nf = 0;
    u64 run = pm;
    for (int s = s0; s < s1; s++) {
      const u64 m = row[at(s)];
      if (m < run) {
        nf++;
        run = m;
      }
    }
    const int nf_incl = warp_inclusive_sum(nf);
    const int nf_tot = __shfl_sync(kFull, nf_incl, 31);
    if (nf_tot > fv.foff[j + 1] - fv.foff[j]) {  // frontier beyond the member's slots
      if (lane == 0) atomicExch(sa.err, 2);
      continue;
    }
    const long long slot0 = fbase + fv.foff[j];
    EntryW* outp = reinterpret_cast<EntryW*>(dp.fe) + slot0;
    int* par = dp.parent + slot0;
    int pos = nf_incl - nf;
    run = pm;
    for (int s = s0; s < s1; s++) {
      const int r = at(s);
      const u64 m = row[r];
      if (m < run) {
        run = m;
        EntryW x{};
        x.t = cells[r];
        x.m = (long long)m;
        outp[pos] = x;
        par[pos] = (int)rowi[r];
        pos++;
      }
    }
    const u64 gmin = __shfl_sync(kFull, incl, 31);
    if (lane == 0) {
      const size_t a = (size_t)b * F + j;
      dp.flen[a] = nf_tot;
      dp.ccount[a] = n;
      dp.mmin[a] = nf_tot ? (long long)gmin : LLONG_MAX;
      dp.trans[a] += s_tr;
      dp.npairs[a] += s_np;
    }
  }
  }  // targets
}

constexpr int kSpGrid = 1024;       // CTAs per budget of a sparse level launch at most
constexpr int kSpSmemCells = 4096;  // cells held in shared memory (t, m2, i: 80 KB)
constexpr long long kSpScratch = 4LL << 30;  // global cell scratch of one launch at most

template <int W>
static int launch_sparse(remat_family_s* f, int lvl, long long lo, long long hi) {
  static bool attr[kMaxDevices] = {};
  const int H = f->hcap;
  const bool smem = H <= kSpSmemCells;
  const size_t bytes = smem ? (size_t)(2 * H + H / 2) * sizeof(u64) : 0;
  // (at most kSpGrid CTAs in all, and global cells of 16·H bytes per CTA
  // within kSpScratch bytes)
  const long long by_mem = smem ? kSpGrid : std::max<long long>(1, kSpScratch / (16LL * H));
  const long long grid = std::min<long long>(
      hi - lo, std::max<long long>(1, std::min<long long>(kSpGrid, by_mem) / std::max(1, f->cur_nb)));
  if (!attr[dev_slot(f->g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(k_relax_sparse<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit));
    attr[dev_slot(f->g->device)] = true;
  }
  SpArgs sa;
  sa.jbase = lo;
  sa.width = hi - lo;
  sa.pend = f->level_start[lvl];
  sa.scratch = nullptr;
  if (!smem) {
    int rc = f->sparse_scratch.ensure((size_t)f->cur_nb * grid * 3 * H);
    if (rc < 0) return rc;
    sa.scratch = f->sparse_scratch.p;
  }
  sa.H = H;
  sa.logH = 0;
  while ((1 << sa.logH) < H) sa.logH++;
  sa.err = f->sparse_err.p;
  k_relax_sparse<W><<<dim3((unsigned)grid, (unsigned)f->cur_nb), kThreads, bytes,
                      f->g->stream>>>(f->view(), f->g->view(), f->dp_view(), sa);
  RM_LAUNCHED();
  f->relax_launches++;
  return REMAT_OK;
}

}  // namespace remat
