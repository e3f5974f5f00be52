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
// reduction is an atomic min on the packed key (m2 << IB) | i in a dense row
// over t2 ∈ [0, T(L_j)], so it is order-independent and deterministic.
//
// Pair constants from per-member prefix terms:
//   fixed_ij = 2(M(L_j) − M(L_i)) + stage_base_j
//   dt_ij    = T(L_j \ ∂L_j) − T(L_i) + T(L_i ∩ ∂L_j)
//   dm_ij    = M(∂L_j) − M(L_i ∩ ∂L_j)
// where the two weighted popcounts of L_i ∩ ∂L_j are either a bit loop over
// the (small) boundary or Σ_c coef_c · popc(L_i ∩ ∂L_j ∩ class_c) over the
// graph's weight classes, whichever is cheaper for this target.
//
// Work decomposition (k_relax_tile): a CTA owns a TILE of TJ consecutive
// targets of one level (their rows live side by side in shared memory) and a
// share of the predecessor range.  A warp tests 32 predecessors against all
// TJ targets (lane = predecessor), turns the comparable (predecessor, target)
// pairs into per-pair constants (lane = pair), then relaxes the flattened
// (pair, frontier entry) items with its 32 lanes.  Pairs of one predecessor
// are adjacent, so a frontier entry fetched for one target is an L1 hit for
// the next: one L2 read of a predecessor's frontier feeds every comparable
// target of the tile (SURVEY §7 hard part 2).  Frontier entries are stored
// with m strictly decreasing, so the budget-feasible ones are a suffix and a
// pair whose cap is below the frontier's smallest m is skipped outright.
//
// Finalisation (K5) turns each row into the compact frontier (strict
// prefix-min of m in t-ascending order, t-descending for maximize;
// planner.py:153-161), one warp per row, and records |cell| and |frontier|;
// with Σ_i|frontier_i| and the comparable-pair counts accumulated during the
// scan these are exactly table_entries, states_visited and transitions
// (Appendix A.3).
//
// The kernels and the per-width drivers live in relax_impl.cuh and are
// instantiated one bitset width per translation unit (relax_w*.cu); this file
// holds the width dispatch and the batch driver.
#include <algorithm>
#include <cstdlib>

#include "relax_decl.h"

namespace remat {

// levels with at most this many (target, predecessor) subset tests are batched
// into one cooperative launch (their work is a fraction of one GPU wave)
static constexpr long long kSmallLevelTests = 2LL << 20;  // swept 1-16 M on the B200
static constexpr long long kSmallLevelPreds = 32LL << 10;
// families up to this size may be solved by one CTA per budget (k_solve_small)
static constexpr long long kSmallFamily = 1100;

template <typename Fn>
static int dispatch_solve(remat_family_s* f, bool narrow, Fn&& fn) {
  int rc = fail(REMAT_ERR_VALUE, "unsupported word count");
  dispatch_words(f->g->Wp, [&](auto wc) {
    constexpr int W = decltype(wc)::value;
    if (narrow) rc = fn(std::integral_constant<int, W>{}, std::true_type{});
    else rc = fn(std::integral_constant<int, W>{}, std::false_type{});
  });
  return rc;
}

int solve_begin(remat_family_s* f, const std::vector<long long>& budgets, int objective) {
  // narrow pair records hold entry offsets within one budget's table as int32
  const bool narrow = f->narrow && f->slots < (1LL << 31);
  return dispatch_solve(f, narrow, [&](auto wc, auto nc) {
    return begin_w<decltype(wc)::value, decltype(nc)::value>(f, budgets, objective);
  });
}

int solve_level(remat_family_s* f, int lvl, long long lo, long long hi) {
  return dispatch_solve(f, f->cur_narrow, [&](auto wc, auto nc) {
    return level_w<decltype(wc)::value, decltype(nc)::value>(f, lvl, lo, hi);
  });
}

int solve_levels(remat_family_s* f, const std::vector<int>& lvls) {
  return dispatch_solve(f, f->cur_narrow, [&](auto wc, auto nc) {
    return levels_w<decltype(wc)::value, decltype(nc)::value>(f, lvls);
  });
}

int solve_small(remat_family_s* f) {
  return dispatch_solve(f, f->cur_narrow, [&](auto wc, auto nc) {
    return small_w<decltype(wc)::value, decltype(nc)::value>(f);
  });
}

int solve_finish(remat_family_s* f, remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                 long long* stage_memory) {
  return dispatch_solve(f, f->cur_narrow, [&](auto wc, auto nc) {
    return finish_w<decltype(wc)::value, decltype(nc)::value>(f, info, chain_masks, cached_masks,
                                                              stage_memory);
  });
}

int plan_rows(remat_family_s* f, int b, u64* chain_masks, u64* cached_masks,
              long long* stage_memory) {
  remat_graph_s* g = f->g;
  const int n = g->n, Wp = g->Wp, Wu = g->W;
  const size_t rows = (size_t)(n + 1);
  std::vector<u64> hc(rows * Wp), hk(rows * Wp);
  cudaStream_t s = g->stream;
  RM_CUDA(cudaMemcpyAsync(hc.data(), f->chain_out.p + (size_t)b * rows * Wp, hc.size() * 8,
                          cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(hk.data(), f->cached_out.p + (size_t)b * rows * Wp, hk.size() * 8,
                          cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(stage_memory, f->stage_out.p + (size_t)b * rows, rows * 8,
                          cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  for (size_t q = 0; q < rows; q++)
    for (int w = 0; w < Wu; w++) {
      chain_masks[q * Wu + w] = hc[q * Wp + w];
      cached_masks[q * Wu + w] = hk[q * Wp + w];
    }
  return REMAT_OK;
}

int solve_batch(remat_family_s* f, const std::vector<long long>& budgets, int objective,
                remat_plan_info* info, u64* chain_masks, u64* cached_masks,
                long long* stage_memory) {
  int rc = solve_begin(f, budgets, objective);
  if (rc < 0) return rc;
  // a small family (pruned families, chain-like lattices) runs whole in one
  // CTA per budget
  static const long long small_family = [] {
    const char* e = getenv("REMAT_SMALL_FAMILY");  // tuning / test hook
    return e ? atoll(e) : kSmallFamily;
  }();
  // one CTA per budget pays off when the batch itself fills the GPU and the
  // frontiers are short (maximize keeps a few entries per cell);
  // a single budget, or long minimize frontiers, spread each level over CTAs
  // unless the batch has a CTA for every SM (C4 pruned 64-budget sweep:
  // one CTA per budget 17.97 ms, per-level launches 16.84 ms)
  static const int force_small = [] {  // REMAT_FORCE_SMALL=1: any batch (A/B hook)
    const char* e = getenv("REMAT_FORCE_SMALL");
    return e ? atoi(e) : 0;
  }();
  const bool small_ok = force_small || (objective == REMAT_MAXIMIZE
                                            ? budgets.size() >= 16
                                            : budgets.size() >= (size_t)sm_count(f->g->device));
  if (f->F <= small_family && small_ok) {
    if ((rc = solve_small(f)) < 0) return rc;
    if (rc == REMAT_OK) return solve_finish(f, info, chain_masks, cached_masks, stage_memory);
  }
  // levels whose subset tests fit one wave of the GPU run back to back in a
  // single cooperative launch; wide levels get their own launch
  std::vector<int> run;
  auto flush = [&]() {
    int r = REMAT_OK;
    if (run.size() == 1)
      r = solve_level(f, run[0], f->level_start[run[0]], f->level_start[run[0] + 1]);
    else if (!run.empty())
      r = solve_levels(f, run);
    run.clear();
    return r;
  };
  for (int lvl = 1; lvl <= f->g->n; lvl++) {
    const long long j0 = f->level_start[lvl], w = f->level_start[lvl + 1] - j0;
    if (w == 0) continue;
    // (a narrow level over a long predecessor range can still carry many
    // frontier entries per pair: those keep their own launch)
    if (w * j0 * (long long)budgets.size() <= kSmallLevelTests && j0 <= kSmallLevelPreds) {
      run.push_back(lvl);
      continue;
    }
    if ((rc = flush()) < 0) return rc;
    if ((rc = solve_level(f, lvl, j0, j0 + w)) < 0) return rc;
  }
  if ((rc = flush()) < 0) return rc;
  return solve_finish(f, info, chain_masks, cached_masks, stage_memory);
}

}  // namespace remat
