// relax.cu — the DP relaxation as a level-synchronous pull wavefront (K4+K5),
// reconstruction (K6) and the post-hoc search statistics.
//
// Replaces TransitionIndex pair constants (planner.py:117-132), _dp_run
// (planner.py:145-177) and _reconstruct (180-189).
//
// Pull form: for target member j (|L_j| = s) and every
// predecessor i (L_i ⊊ L_j, necessarily |L_i| < s, i.e. i < level_start[s]):
//   candidate (t + dt_ij, m + dm_ij) from every non-dominated entry (t, m) of
//   cell i with m + fixed_ij <= B.
// opt[j][t2] = lexicographic min over (m2, i) — the reference's strict `<`
// push in family order keeps the first (smallest) i among equal m2.  The
// reduction is a 64-bit atomicMin on the packed key (m2 << IB) | i in a
// shared-memory row over t2 ∈ [0, T(L_j)], so it is order-independent and
// deterministic.
//
// Pair constants from per-member prefix terms:
//   fixed_ij = 2(M(L_j) − M(L_i)) + stage_base_j
//   dt_ij    = T(L_j \ ∂L_j) − T(L_i) + T(L_i ∩ ∂L_j)
//   dm_ij    = M(∂L_j) − M(L_i ∩ ∂L_j)
// where the two weighted popcounts of L_i ∩ ∂L_j are either a bit loop over
// the (small) boundary or Σ_c coef_c · popc(L_i ∩ ∂L_j ∩ class_c) over the
// graph's weight classes, whichever is cheaper for this target.
//
// Finalisation (K5) turns the row into the compact frontier (strict prefix-min
// of m in t-ascending order, t-descending for maximize; planner.py:153-161)
// and records |cell|, |frontier| and Σ_i|frontier_i| over comparable i —
// exactly table_entries, states_visited and transitions (Appendix A.3).
#include <algorithm>

#include "device.cuh"

namespace remat {

// One queued predecessor of the current chunk (32 B -> two LDS.128).
constexpr int kWarpMap = 512;  // items per round of a warp's item -> predecessor map

struct __align__(16) QEntry {
  long long foff;  // first frontier entry of the predecessor (budget-offset)
  long long cap;   // B − fixed_ij: an entry passes the budget test iff m <= cap
  long long dm;    // dm_ij
  int dt;          // dt_ij (<= T(V) < 2^24)
  int i;           // predecessor family index
};

// opt[t2] = min(opt[t2], key).  sm_100 has no native 64-bit shared-memory
// min (it lowers to a CAS loop), so read first: a losing candidate issues no
// atomic at all.  Global rows use the native ATOM.MIN.64.
__device__ __forceinline__ void row_min(u64* row, long long t2, u64 key, bool smem) {
  if (smem) {
    u64 old = row[t2];
    while (key < old) {
      u64 prev = atomicCAS(row + t2, old, key);
      if (prev == old) break;
      old = prev;
    }
  } else {
    atomicMin(row + t2, key);
  }
}

// K5 on a finished row: |cell|, the strict prefix-min frontier in t order
// (ascending for minimize, descending for maximize; planner.py:153-161),
// compacted into the member's frontier slot with its back-pointers.
__device__ void finalize_row(const u64* row, long long R, const DpView& dp, const FamilyView& fv,
                             long long j, int b, long long trans_acc, long long pairs_acc,
                             u64* scr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long F = fv.F;
  const int IB = dp.IB;
  const int per = (int)((R + nt - 1) / nt);
  const long long s0 = (long long)tid * per, s1 = min(R, s0 + per);
  const bool mx = dp.maximize;
  u64 lmin = ~0ull;
  unsigned cells = 0;
  for (long long s = s0; s < s1; s++) {
    u64 key = row[mx ? R - 1 - s : s];
    if (key != ~0ull) {
      cells++;
      u64 m = key >> IB;
      lmin = m < lmin ? m : lmin;
    }
  }
  const u64 pm = block_exclusive_min(lmin, scr);
  unsigned nf = 0;
  u64 run = pm;
  for (long long s = s0; s < s1; s++) {
    u64 key = row[mx ? R - 1 - s : s];
    if (key != ~0ull) {
      u64 m = key >> IB;
      if (m < run) {
        nf++;
        run = m;
      }
    }
  }
  u64 tot2;
  u64 ex2 = block_exclusive_sum<u64>(((u64)cells << 32) | nf, scr, &tot2);
  Frontier* out = dp.frontier + (long long)b * dp.slots + fv.foff[j];
  unsigned pos = (unsigned)(ex2 & 0xffffffffu);
  run = pm;
  const u64 pmask = (1ull << IB) - 1;
  for (long long s = s0; s < s1; s++) {
    long long t = mx ? R - 1 - s : s;
    u64 key = row[t];
    if (key != ~0ull) {
      u64 m = key >> IB;
      if (m < run) {
        Frontier f;
        f.m = (long long)m;
        f.t = (unsigned)t;
        f.parent = (int)(key & pmask);
        out[pos++] = f;
        run = m;
      }
    }
  }
  if (tid == 0) {
    dp.flen[(size_t)b * F + j] = (int)(tot2 & 0xffffffffu);
    dp.ccount[(size_t)b * F + j] = (int)(tot2 >> 32);
    dp.trans[(size_t)b * F + j] = trans_acc;
    dp.npairs[(size_t)b * F + j] = (int)pairs_acc;
  }
}

// K4 (+K5 when unsplit).  Grid: (width·splits, nb); CTA (target tj, slice)
// scans the predecessors [slice·P/splits, (slice+1)·P/splits) in 32-member
// chunks.  Warps work independently (no block barrier in the main loop): a
// warp tests 32 predecessors (lane = predecessor), queues the comparable ones
// with a non-empty frontier in its private queue, stamps an item ->
// predecessor map, and relaxes the flattened (predecessor, frontier entry)
// items with its 32 lanes into the CTA's shared row.
template <int W>
__global__ void __launch_bounds__(kRelaxThreads)
    k_relax_level(FamilyView fv, GraphView g, ClassView cv, DpView dp, long long jbase,
                  long long pred_end, int splits, int smem_row, u64* grow, long long grow_stride,
                  long long* part) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ QEntry wq[kRelaxWarps][32];
  __shared__ int wpre[kRelaxWarps][33];
  __shared__ unsigned short wmap[kRelaxWarps][kWarpMap];
  __shared__ u64 scr[33];
  __shared__ long long red[2][kRelaxWarps];
  __shared__ u64 bjc[2 * kMaxClasses * W];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long F = fv.F;
  const int width = gridDim.x / splits;
  const int tj = blockIdx.x / splits, slice = blockIdx.x - tj * splits;
  const long long j = jbase + tj;
  const int b = blockIdx.y;
  u64* grow_j = grow ? grow + ((long long)b * width + tj) * grow_stride : nullptr;
  u64* row = smem_row ? reinterpret_cast<u64*>(smraw) : grow_j;

  u64 Lj[W], Bj[W];
  int bcnt = 0;
#pragma unroll
  for (int w = 0; w < W; w++) {
    Lj[w] = fv.masks[(size_t)w * F + j];
    Bj[w] = fv.bound[(size_t)w * F + j];
    bcnt += __popcll(Bj[w]);
  }
  const long long R = fv.TL[j] + 1;
  const long long MLj = fv.ML[j], basej = fv.base[j], TLnbj = fv.TLnb[j], Mbj = fv.Mb[j];
  const long long B = dp.budgets[b];
  const int IB = dp.IB;
  const int KT = cv.KT, K = cv.KT + cv.KM;
  const bool use_cls = cv.enabled && K * W < bcnt;
  if (use_cls) {
    for (int e = tid; e < K * W; e += kRelaxThreads) {
      int c = e / W, w = e - c * W;
      u64 cls = c < KT ? cv.clsT[c * W + w] : cv.clsM[(c - KT) * W + w];
      bjc[e] = fv.bound[(size_t)w * F + j] & cls;
    }
  }
  if (smem_row)
    for (long long t = tid; t < R; t += kRelaxThreads) row[t] = ~0ull;
  __syncthreads();

  const int* flen_b = dp.flen + (size_t)b * F;
  const long long fbase = (long long)b * dp.slots;
  long long trans_acc = 0, pairs_acc = 0;
  const long long nch = (pred_end + 31) / 32;
  const long long c0 = slice * nch / splits, c1 = (slice + 1) * nch / splits;
  QEntry* q = wq[warp];
  int* qpre = wpre[warp];
  unsigned short* qmap = wmap[warp];

  for (long long ch = c0 + warp; ch < c1; ch += kRelaxWarps) {
    const long long i = ch * 32 + lane;
    int fl = 0;
    bool comparable = false;
    long long fixed = 0, dt = 0, dm = 0;
    if (i < pred_end) {
      u64 Li[W];
      u64 acc = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        Li[w] = __ldg(fv.masks + (size_t)w * F + i);
        acc |= Li[w] & ~Lj[w];
      }
      comparable = acc == 0;
      if (comparable) {
        fl = flen_b[i];
        if (fl > 0) {
          long long ts = 0, ms = 0;
          if (use_cls) {
            for (int c = 0; c < K; c++) {
              int pc = 0;
#pragma unroll
              for (int w = 0; w < W; w++) pc += __popcll(Li[w] & bjc[c * W + w]);
              if (c < KT) ts += __ldg(cv.coefT + c) * pc;
              else ms += __ldg(cv.coefM + c - KT) * pc;
            }
          } else {
#pragma unroll
            for (int w = 0; w < W; w++) {
              u64 x = Li[w] & Bj[w];
              while (x) {
                int v = w * 64 + __ffsll((long long)x) - 1;
                x &= x - 1;
                ts += __ldg(g.T + v);
                ms += __ldg(g.M + v);
              }
            }
          }
          fixed = 2 * (MLj - fv.ML[i]) + basej;
          dt = TLnbj - fv.TL[i] + ts;
          dm = Mbj - ms;
        }
      }
    }
    const unsigned has = __ballot_sync(kFull, fl > 0);
    pairs_acc += __popc(__ballot_sync(kFull, comparable));
    if (!has) continue;
    const int qn = __popc(has);
    const int incl = warp_inclusive_sum(fl);
    const int total = __shfl_sync(kFull, incl, 31);
    trans_acc += total;
    if (fl > 0) {
      const int qp = __popc(has & ((1u << lane) - 1));
      QEntry e;
      e.foff = fbase + fv.foff[i];
      e.cap = B - fixed;
      e.dm = dm;
      e.dt = (int)dt;
      e.i = (int)i;
      q[qp] = e;
      qpre[qp] = incl - fl;
    }
    if (lane == 0) qpre[qn] = total;
    __syncwarp();
    for (int r0 = 0; r0 < total; r0 += kWarpMap) {
      const int r1 = min(total, r0 + kWarpMap);
      if (lane < qn) {
        const int a = max(qpre[lane], r0), z = min(qpre[lane + 1], r1);
        for (int e = a; e < z; e++) qmap[e - r0] = (unsigned short)lane;
      }
      __syncwarp();
#pragma unroll 4
      for (int e = r0 + lane; e < r1; e += 32) {
        const int k = qmap[e - r0];
        const QEntry qe = q[k];
        const Frontier fr = dp.frontier[qe.foff + (e - qpre[k])];
        if (fr.m <= qe.cap) {
          u64 key = ((u64)(fr.m + qe.dm) << IB) | (u64)qe.i;
          row_min(row, (long long)fr.t + qe.dt, key, smem_row);
        }
      }
      __syncwarp();
    }
  }
  // per-CTA totals (trans_acc is warp-uniform; pairs_acc too)
  if (lane == 0) {
    red[0][warp] = trans_acc;
    red[1][warp] = pairs_acc;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kRelaxWarps; w++) {
      trans_acc += red[0][w];
      pairs_acc += red[1][w];
    }
  }
  if (splits == 1 && smem_row) {
    finalize_row(row, R, dp, fv, j, b, trans_acc, pairs_acc, scr);
    return;
  }
  if (smem_row)  // fold this slice's row into the target's global row
    for (long long t = tid; t < R; t += kRelaxThreads) {
      u64 key = row[t];
      if (key != ~0ull) atomicMin(grow_j + t, key);
    }
  if (tid == 0) {
    long long* pp = part + (((long long)b * width + tj) * splits + slice) * 2;
    pp[0] = trans_acc;
    pp[1] = pairs_acc;
  }
}

// K5 for split / global-row levels: one CTA per (target, budget).
__global__ void __launch_bounds__(kRelaxThreads)
    k_finalize_level(FamilyView fv, DpView dp, long long jbase, int width, int splits,
                     const u64* __restrict__ grow, long long grow_stride,
                     const long long* __restrict__ part) {
  __shared__ u64 scr[33];
  const int tj = blockIdx.x, b = blockIdx.y;
  const long long j = jbase + tj;
  long long tr = 0, pr = 0;
  const long long* pp = part + ((long long)b * width + tj) * splits * 2;
  for (int s = 0; s < splits; s++) {
    tr += pp[2 * s];
    pr += pp[2 * s + 1];
  }
  finalize_row(grow + ((long long)b * width + tj) * grow_stride, fv.TL[j] + 1, dp, fv, j, b, tr,
               pr, scr);
}

__global__ void k_dp_init(DpView dp, long long F, int nb) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  Frontier f;
  f.m = 0;
  f.t = 0;
  f.parent = -1;
  dp.frontier[(long long)b * dp.slots] = f;  // foff[0] == 0: the empty set
  dp.flen[(size_t)b * F] = 1;
  dp.ccount[(size_t)b * F] = 1;
  dp.trans[(size_t)b * F] = 0;
  dp.npairs[(size_t)b * F] = 0;
}

// SearchStats, recomputed from the final table (Appendix A.3).
__global__ void k_dp_stats(DpView dp, long long F, long long* __restrict__ out) {
  __shared__ long long scr[4][32];
  const int b = blockIdx.x;
  long long sv = 0, te = 0, tr = 0, np = 0;
  for (long long i = threadIdx.x; i < F; i += blockDim.x) {
    sv += dp.flen[(size_t)b * F + i];
    te += dp.ccount[(size_t)b * F + i];
    tr += dp.trans[(size_t)b * F + i];
    np += dp.npairs[(size_t)b * F + i];
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
template <int W>
__global__ void k_reconstruct(FamilyView fv, GraphView g, DpView dp, int n,
                              int* __restrict__ path, u64* __restrict__ chain_out,
                              int* __restrict__ klen, long long* __restrict__ expect) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const long long F = fv.F;
  const long long fbase = (long long)b * dp.slots;
  int* pth = path + (size_t)b * (n + 2);
  long long j = F - 1;
  if (dp.flen[(size_t)b * F + j] == 0) {
    if (lane == 0) klen[b] = 0;
    return;
  }
  Frontier cur = dp.frontier[fbase + fv.foff[j]];
  if (lane == 0) {
    expect[b * 4 + 0] = cur.t;
    expect[b * 4 + 1] = cur.m;
    expect[b * 4 + 2] = dp.budgets[b];
    expect[b * 4 + 3] = 1;
  }
  int len = 0;
  bool bad = false;
  while (true) {
    if (lane == 0) pth[len] = (int)j;
    len++;
    if (j == 0) break;
    if (len > n + 1 || cur.parent < 0) {
      bad = true;
      break;
    }
    const long long par = cur.parent;
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
      bool hit = s < nfp && (long long)dp.frontier[pb + s].t == tp;
      unsigned bal = __ballot_sync(kFull, hit);
      if (bal) {
        cur = dp.frontier[pb + s0 + __ffs(bal) - 1];
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

static constexpr int kSmemLimit = 200 * 1024;  // dynamic row bytes per CTA

template <int W>
static int solve_w(remat_family_s* f, const std::vector<long long>& budgets, int objective,
                   remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                   long long* stage_memory) {
  remat_graph_s* g = f->g;
  cudaStream_t s = g->stream;
  const int nb = (int)budgets.size();
  const int n = g->n;
  const long long F = f->F;
  int rc;
  if ((rc = f->frontier.ensure((size_t)nb * f->slots)) < 0 ||
      (rc = f->flen.ensure((size_t)nb * F)) < 0 || (rc = f->ccount.ensure((size_t)nb * F)) < 0 ||
      (rc = f->trans.ensure((size_t)nb * F)) < 0 || (rc = f->budgets.ensure(nb)) < 0 ||
      (rc = f->npairs.ensure((size_t)nb * F)) < 0 ||
      (rc = f->results.ensure((size_t)nb * 20)) < 0 ||
      (rc = f->chain_out.ensure((size_t)nb * (n + 1) * W)) < 0 ||
      (rc = f->cached_out.ensure((size_t)nb * (n + 1) * W)) < 0 ||
      (rc = f->stage_out.ensure((size_t)nb * (n + 1))) < 0 ||
      (rc = f->chain_idx.ensure((size_t)nb * (n + 2) + nb)) < 0 ||
      (rc = f->terms.ensure((size_t)nb * (n + 1) * 4)) < 0 ||
      (rc = f->stage_bound.ensure((size_t)nb * (n + 1) * W)) < 0)
    return rc;
  static bool attr_set = false;
  if (!attr_set) {
    RM_CUDA(cudaFuncSetAttribute(k_relax_level<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit));
    attr_set = true;
  }
  DpView dp{f->slots,    f->frontier.p, f->flen.p, f->ccount.p, f->trans.p,
            f->npairs.p, f->budgets.p,  f->IB,     objective == REMAT_MAXIMIZE};
  FamilyView fv = f->view();
  GraphView gv = g->view();
  ClassView cv = g->classes();
  Events& ev = g->ev;
  const long long launches0 = remat_kernel_launch_count();
  RM_CUDA(cudaMemcpyAsync(f->budgets.p, budgets.data(), sizeof(long long) * nb,
                          cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaEventRecord(ev.e[3], s));
  k_dp_init<<<(nb + 127) / 128, 128, 0, s>>>(dp, F, nb);
  RM_LAUNCHED();
  long long relax_launches = 0;
  static int num_sms = 0;
  if (!num_sms) RM_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, g->device));
  const long long target_ctas = (long long)num_sms * 4;  // resident CTAs at 256 threads
  for (int lvl = 1; lvl <= n; lvl++) {
    const long long j0 = f->level_start[lvl], width = f->level_start[lvl + 1] - j0;
    if (width == 0) continue;
    const long long R = f->level_maxR[lvl];
    const bool in_smem = R * 8 <= kSmemLimit;
    const long long nch = (j0 + kRelaxThreads - 1) / kRelaxThreads;
    // split the predecessor scan across CTAs when the level alone cannot fill
    // the GPU (narrow levels near ∅ and V; SURVEY §7 hard part 5)
    long long splits = (target_ctas + width * nb - 1) / (width * nb);
    splits = std::max(1LL, std::min(splits, nch / 2));
    u64* grow = nullptr;
    long long* part = nullptr;
    if (splits > 1 || !in_smem) {
      if ((rc = f->rowscratch.ensure((size_t)width * nb * R)) < 0 ||
          (rc = f->partials.ensure((size_t)width * nb * splits * 2)) < 0)
        return rc;
      grow = f->rowscratch.p;
      part = f->partials.p;
      RM_CUDA(cudaMemsetAsync(grow, 0xff, sizeof(u64) * width * nb * R, s));
    }
    k_relax_level<W><<<dim3((unsigned)(width * splits), (unsigned)nb), kRelaxThreads,
                       in_smem ? (size_t)R * 8 : 0, s>>>(fv, gv, cv, dp, j0, j0, (int)splits,
                                                         in_smem ? 1 : 0, grow, R, part);
    RM_LAUNCHED();
    relax_launches++;
    if (grow) {
      k_finalize_level<<<dim3((unsigned)width, (unsigned)nb), kRelaxThreads, 0, s>>>(
          fv, dp, j0, (int)width, (int)splits, grow, R, part);
      RM_LAUNCHED();
    }
  }
  RM_CUDA(cudaEventRecord(ev.e[4], s));
  long long* expect = f->results.p;           // [nb][4]
  long long* stats = f->results.p + nb * 4;   // [nb][5]
  long long* evres = f->results.p + nb * 9;   // [nb][8]
  int* klen = f->chain_idx.p + (size_t)nb * (n + 2);
  k_reconstruct<W><<<nb, 32, 0, s>>>(fv, gv, dp, n, f->chain_idx.p, f->chain_out.p, klen, expect);
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
  float relax_ms = 0, finish_ms = 0, total_ms = 0;
  cudaEventElapsedTime(&relax_ms, ev.e[3], ev.e[4]);
  cudaEventElapsedTime(&finish_ms, ev.e[4], ev.e[5]);
  cudaEventElapsedTime(&total_ms, ev.e[3], ev.e[6]);
  f->timings.relax_ms = relax_ms;
  f->timings.finish_ms = finish_ms;
  f->timings.total_ms = total_ms;
  f->timings.relax_launches = relax_launches;
  f->timings.kernel_launches = remat_kernel_launch_count() - launches0;

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

int solve_batch(remat_family_s* f, const std::vector<long long>& budgets, int objective,
                remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                long long* stage_memory) {
  int rc = fail(REMAT_ERR_VALUE, "unsupported word count");
  dispatch_words(f->g->Wp, [&](auto wc) {
    constexpr int W = decltype(wc)::value;
    rc = solve_w<W>(f, budgets, objective, info, chain_masks, cached_masks, stage_memory);
  });
  return rc;
}

}  // namespace remat
