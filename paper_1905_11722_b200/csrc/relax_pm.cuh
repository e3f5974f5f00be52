// relax_pm.cuh — the relaxation of WIDE levels with LONG frontiers
// (conv-weighted minimize solves: the U-Net headline, PSPNet sweeps), in a
// predecessor-major form.  Included by relax_impl.cuh.
//
// Same pull semantics as k_relax_tile (relax.cu): the cell of target j is the
// lexicographic min over (m2, i) of candidates (t + dt_ij, m + dm_ij) from
// the frontier entries of every predecessor i ⊊ j that pass m + fixed_ij <= B,
// reduced with an atomic min on the packed key (m2 << IB) | i in the
// target's shared-memory row.  What changes is who does what:
//
//  * a CTA owns up to 32 targets (one bit each in a 32-bit comparable mask),
//    so a predecessor meets ~4x more comparable targets per tile than with
//    8-target tiles;
//  * lane = predecessor for the subset tests and the pair constants, which
//    are compacted into a per-warp record list (16 B each);
//  * then lane = FRONTIER ENTRY: the warp walks its predecessors one at a
//    time, 32 consecutive entries of one predecessor per step (one coalesced
//    load), and every record of that predecessor is one warp-uniform LDS plus
//    one RED per lane.  No per-item predecessor mapping, no divergent pair
//    loops; when a record's cap covers the predecessor's largest m (its first
//    entry) the budget test disappears from the step;
//  * the CTAs that share a tile's predecessor range form a THREAD-BLOCK
//    CLUSTER: at the end their shared-memory rows are min-reduced over
//    distributed shared memory (DSMEM) by the CTA that finalizes each target —
//    no global row scratch, fence or done counter.

namespace remat {

constexpr int kPmMaxTJ = 32;
constexpr int kPmRecCap = 128;  // pair records per warp and round

struct __align__(16) PmRec {
  unsigned base;  // shared byte address of row slot dt_ij of the target
  unsigned cap;   // B − fixed_ij (entries pass iff m <= cap)
  unsigned kb;    // (dm_ij << IB) | i
  unsigned pad;
};

struct PmLayout {
  int off_tL, off_tB, off_tc, off_tcls, off_bjc, off_coef, off_tacc, off_rec, off_rows, bytes;
};

template <int W>
static PmLayout pm_layout(int TJ, int R, int K, bool cls) {
  PmLayout a{};
  int o = 0;
  auto take = [&](int bytes) {
    int at = o;
    o += (bytes + 15) & ~15;
    return at;
  };
  a.off_tL = take(TJ * W * 8);
  a.off_tB = take(TJ * W * 8);
  a.off_tc = take(TJ * 4 * 8);
  a.off_tcls = take(TJ * 4);
  a.off_bjc = take(cls ? TJ * K * W * 8 : 0);
  a.off_coef = take(cls ? 2 * K * 8 : 0);
  a.off_tacc = take(TJ * 2 * 8);
  a.off_rec = take(kWarps * kPmRecCap * (int)sizeof(PmRec));
  a.off_rows = take(TJ * R * 4);
  a.bytes = o;
  return a;
}

struct PmArgs {
  long long jbase, pend;
  int width, TJ, R, tiles, splits, cls, ctr_stride;
  unsigned* ctr;
  PmLayout lay;
};

template <int W>
__global__ void __launch_bounds__(kThreads)
    k_relax_pm(FamilyView fv, GraphView g, ClassView cv, DpView dp, PmArgs pa) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char sm[];
  using Key = unsigned;
  constexpr Key INF = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.y, nb = gridDim.y;
  const int splits = pa.splits;
  const int tile = blockIdx.x / splits, rank = (int)cluster.block_rank();
  const int TJ = pa.TJ, R = pa.R, K = cv.K;
  const long long F = fv.F;
  const long long j0 = pa.jbase + (long long)tile * TJ;
  const int ntj = (int)min((long long)TJ, pa.jbase + pa.width - j0);
  const PmLayout& L = pa.lay;
  u64* tL = reinterpret_cast<u64*>(sm + L.off_tL);
  u64* tB = reinterpret_cast<u64*>(sm + L.off_tB);
  long long* tc = reinterpret_cast<long long*>(sm + L.off_tc);
  int* tcls = reinterpret_cast<int*>(sm + L.off_tcls);
  u64* bjc = reinterpret_cast<u64*>(sm + L.off_bjc);
  long long* tcoef = reinterpret_cast<long long*>(sm + L.off_coef);
  u64* tacc = reinterpret_cast<u64*>(sm + L.off_tacc);
  PmRec* wrec = reinterpret_cast<PmRec*>(sm + L.off_rec) + warp * kPmRecCap;
  Key* rows = reinterpret_cast<Key*>(sm + L.off_rows);
  const unsigned wrec_sa = (unsigned)__cvta_generic_to_shared(wrec);
  const unsigned rows_sa = (unsigned)__cvta_generic_to_shared(rows);

  // ---- tile set-up: target sets and scalars, empty rows, class masks
  for (int e = tid; e < ntj * W; e += kThreads) {
    const int jt = e / W, w = e - jt * W;
    tL[e] = fv.masks[(size_t)w * F + j0 + jt];
    tB[e] = fv.bound[(size_t)w * F + j0 + jt];
  }
  for (int jt = tid; jt < ntj; jt += kThreads) {
    const long long j = j0 + jt;
    tc[jt * 4 + 0] = fv.ML[j];
    tc[jt * 4 + 1] = fv.base[j];
    tc[jt * 4 + 2] = fv.TLnb[j];
    tc[jt * 4 + 3] = fv.Mb[j];
    tacc[jt * 2] = tacc[jt * 2 + 1] = 0;
  }
  for (int t = tid; t < ntj * R; t += kThreads) rows[t] = INF;
  __syncthreads();
  if (pa.cls) {
    for (int e = tid; e < ntj * K * W; e += kThreads) {
      const int jt = e / (K * W), r = e - jt * K * W, c = r / W, w = r - c * W;
      bjc[e] = tB[jt * W + w] & cv.cls[c * W + w];
    }
    for (int e = tid; e < 2 * K; e += kThreads) tcoef[e] = cv.coef[e];
  }
  for (int jt = tid; jt < ntj; jt += kThreads) {
    int bc = 0;
    for (int w = 0; w < W; w++) bc += __popcll(tB[jt * W + w]);
    tcls[jt] = pa.cls && K * W < bc;
  }
  __syncthreads();
  // union of the tile's targets: a predecessor outside it meets no target
  u64 tun[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    u64 x = 0;
    for (int jt = 0; jt < ntj; jt++) x |= tL[jt * W + w];
    tun[w] = x;
  }

  const long long B = dp.budgets[b];
  const int IB = dp.IB;
  const long long fbase = (long long)b * dp.slots;
  const int* flen_b = dp.flen + (size_t)b * F;
  const long long* mmin_b = dp.mmin + (size_t)b * F;
  const EntryN* fe = reinterpret_cast<const EntryN*>(dp.fe);
  const long long nch = (pa.pend + 31) / 32;
  unsigned* ctr = pa.ctr + (size_t)b * pa.ctr_stride + tile;
  u64 my_trans = 0, my_pairs = 0;
  const long long nstatic = (long long)splits * kWarps;
  auto next_chunk = [&](long long ch) {
    if (nstatic >= nch) return nch;
    unsigned got = 0;
    if (lane == 0) got = atomicAdd(ctr, 1u);
    return nstatic + (long long)__shfl_sync(kFull, got, 0);
  };
  for (long long ch = (long long)rank * kWarps + warp; ch < nch; ch = next_chunk(ch)) {
    const long long i = ch * 32 + lane;
    u64 Li[W];
    int fl = 0;
    long long MLi = 0, TLi = 0, mmi = 0, foffi = 0;
    unsigned mask = 0;
    if (i < pa.pend) {
      u64 out = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        Li[w] = __ldg(fv.masks + (size_t)w * F + i);
        out |= Li[w] & ~tun[w];
      }
      if (!out) {
        for (int jt = 0; jt < ntj; jt++) {
          u64 acc = 0;
#pragma unroll
          for (int w = 0; w < W; w++) acc |= Li[w] & ~tL[jt * W + w];
          mask |= (acc == 0 ? 1u : 0u) << jt;
        }
      }
    }
    if (!__any_sync(kFull, mask)) continue;
    if (mask) {
      fl = flen_b[i];
      mmi = mmin_b[i];
      MLi = __ldg(fv.ML + i);
      TLi = __ldg(fv.TL + i);
      foffi = __ldg(fv.foff + i);
    }
    // statistics on the predecessor side (comparable pairs, Σ|frontier|): the
    // tile's totals land on its first target, as in relax_body
    my_pairs += (u64)__popc(mask);
    my_trans += (u64)__popc(mask) * (u64)fl;
    unsigned want = fl > 0 ? mask : 0u;
    // records, in rounds of at most kPmRecCap per warp
    while (__any_sync(kFull, want)) {
      const int c = __popc(want);
      const int incl = warp_inclusive_sum(c);
      // the round takes the lanes whose records fit (a lane has at most 32,
      // so the first lane with records always does)
      const bool mine = c > 0 && incl <= kPmRecCap;
      int pos = incl - c, nrec = 0;
      const int a0 = pos;
      if (mine) {
        unsigned x = want;
        while (x) {
          const int jt = __ffs(x) - 1;
          x &= x - 1;
          long long ts = 0, ms = 0;
          if (tcls[jt]) {
            const u64* bj = bjc + (size_t)jt * K * W;
            for (int cc = 0; cc < K; cc++) {
              int pc = 0;
#pragma unroll
              for (int w = 0; w < W; w++) pc += __popcll(Li[w] & bj[cc * W + w]);
              ts += tcoef[2 * cc] * pc;
              ms += tcoef[2 * cc + 1] * pc;
            }
          } else {
#pragma unroll
            for (int w = 0; w < W; w++) {
              u64 y = Li[w] & tB[jt * W + w];
              while (y) {
                const int v = w * 64 + __ffsll((long long)y) - 1;
                y &= y - 1;
                ts += __ldg(g.T + v);
                ms += __ldg(g.M + v);
              }
            }
          }
          const long long fixed = 2 * (tc[jt * 4 + 0] - MLi) + tc[jt * 4 + 1];
          const long long dt = tc[jt * 4 + 2] - TLi + ts;
          const long long dm = tc[jt * 4 + 3] - ms;
          const long long cap = B - fixed;
          if (cap < mmi) continue;  // no frontier entry of i passes
          PmRec r;
          r.base = rows_sa + 4u * (unsigned)(jt * R + (int)dt);
          r.cap = (unsigned)min(cap, (long long)0xffffffffLL);
          r.kb = (unsigned)(((u64)dm << IB) | (u64)i);
          r.pad = 0;
          wrec[pos + nrec++] = r;
        }
        want = 0;
      }
      __syncwarp();
      // lane = frontier entry: one predecessor of the round at a time
      unsigned live = __ballot_sync(kFull, mine && nrec > 0);
      while (live) {
        const int p = __ffs(live) - 1;
        live &= live - 1;
        const int len = __shfl_sync(kFull, fl, p);
        const long long fo = __shfl_sync(kFull, foffi, p);
        const unsigned ra = wrec_sa + 16u * (unsigned)__shfl_sync(kFull, a0, p);
        const int nr = __shfl_sync(kFull, nrec, p);
        const EntryN* src = fe + (fbase + fo);
        const PmRec* recs = wrec + (ra - wrec_sa) / 16u;
        const unsigned mfirst = src[0].m;  // largest m of the frontier (m falls along it)
        // up to 4 steps (128 entries) of the predecessor in registers, then
        // every record streams its REDs over them: independent atomics, one
        // record load per 128 candidates per lane
        for (int e0 = 0; e0 < len; e0 += 128) {
          unsigned t4[4], mk[4], mm[4];
          bool vv[4];
#pragma unroll
          for (int st = 0; st < 4; st++) {
            const int e = e0 + 32 * st + lane;
            vv[st] = e < len;
            unsigned t = 0, m = 0;
            if (vv[st]) {
              const uint2 v = __ldg(reinterpret_cast<const uint2*>(src + e));
              t = v.x;
              m = v.y;
            }
            t4[st] = 4u * t;
            mk[st] = m << IB;
            mm[st] = m;
          }
          const bool fullblk = e0 + 128 <= len;
          const int nst = min(4, (len - e0 + 31) >> 5);
          for (int r = 0; r < nr; r++) {
            const PmRec q = recs[r];
            if (fullblk && q.cap >= mfirst) {
#pragma unroll
              for (int st = 0; st < 4; st++)
                asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(q.base + t4[st]), "r"(mk[st] + q.kb));
            } else {
#pragma unroll
              for (int st = 0; st < 4; st++)
                if (st < nst) red_smem(q.base + t4[st], mk[st] + q.kb, vv[st] && mm[st] <= q.cap);
            }
          }
        }
      }
      __syncwarp();
    }
  }
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
  // ---- cluster fold over DSMEM: CTA `rank` finalizes targets jt ≡ rank
  cluster.sync();
  for (int jt = rank + splits * warp; jt < ntj; jt += splits * kWarps) {
    const int Rj = (int)(fv.TL[j0 + jt] + 1);
    Key* row = rows + jt * R;
    for (int q = 0; q < splits; q++) {
      if (q == rank) continue;
      const Key* other = cluster.map_shared_rank(row, q);
      for (int t = lane; t < Rj; t += 32) {
        const Key o = other[t];
        if (o < row[t]) row[t] = o;
      }
    }
    __syncwarp();
    finalize_row_warp<true>(row, Rj, dp, fv, j0 + jt, b);
  }
  cluster.sync();  // peers' rows stay alive until every reader is done
  if (rank == 0 && tid == 0) *ctr = 0;  // the tile counter, reset for the next level
}

// Host planning of a pm level; returns false when the level should use the
// tile kernel instead (rows too long for shared memory).
template <int W>
static bool plan_pm(remat_family_s* f, int lvl, long long lo, long long hi, PmArgs& pa) {
  remat_graph_s* g = f->g;
  const ClassView cv = g->classes();
  const int K = cv.K;
  const int R = (int)f->level_maxR[lvl];
  const long long width = hi - lo;
  const long long j0 = f->level_start[lvl];
  const int nb = f->cur_nb;
  static const int row_budget = [] {
    const char* e = getenv("REMAT_PM_ROWS_KB");
    return (e ? atoi(e) : 40) * 1024;
  }();
  int TJ = (int)std::min<long long>(std::min<long long>(kPmMaxTJ, width), row_budget / (R * 4));
  if (TJ < 4) return false;
  bool cls = cv.enabled && (long long)TJ * K * W * 8 <= 16 * 1024;
  pa.lay = pm_layout<W>(TJ, R, K, cls);
  if (pa.lay.bytes > kSmemLimit) return false;
  const long long tiles = (width + TJ - 1) / TJ;
  const int num_sms = sm_count(g->device);
  const int per_sm = std::max(1, (228 << 10) / (pa.lay.bytes + (1 << 10)));
  const long long resident = (long long)num_sms * std::min(per_sm, 8);
  const long long nch = (j0 + 31) / 32;
  int splits = 1;
  static const int max_split = [] {
    const char* e = getenv("REMAT_PM_MAX_SPLIT");
    return e ? atoi(e) : 8;
  }();
  while (splits < max_split && tiles * splits * nb < resident * 3 / 2 &&
         (long long)splits * 2 * kWarps <= nch)
    splits *= 2;
  pa.jbase = lo;
  pa.pend = j0;
  pa.width = (int)width;
  pa.TJ = TJ;
  pa.R = R;
  pa.tiles = (int)tiles;
  pa.splits = splits;
  pa.cls = cls;
  pa.ctr_stride = (int)tiles;
  pa.ctr = f->ctr.p;
  return (size_t)2 * nb * tiles <= f->ctr_cap;
}

template <int W>
static int launch_pm(remat_family_s* f, const PmArgs& pa) {
  static bool attr[kMaxDevices] = {};
  if (!attr[dev_slot(f->g->device)]) {
    RM_CUDA(cudaFuncSetAttribute(k_relax_pm<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemLimit));
    attr[dev_slot(f->g->device)] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(pa.tiles * pa.splits), (unsigned)f->cur_nb);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)pa.lay.bytes;
  cfg.stream = f->g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)pa.splits;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RM_CUDA(cudaLaunchKernelEx(&cfg, k_relax_pm<W>, f->view(), f->g->view(), f->g->classes(),
                             f->dp_view(), pa));
  RM_LAUNCHED();
  f->relax_launches++;
  return REMAT_OK;
}

}  // namespace remat
