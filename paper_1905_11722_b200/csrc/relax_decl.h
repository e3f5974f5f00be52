// relax_decl.h — per-width relaxation drivers, instantiated in relax_w*.cu.
#pragma once
#include "internal.h"

namespace remat {
template <int W, bool NARROW>
int begin_w(remat_family_s* f, const std::vector<long long>& budgets, int objective);
template <int W, bool NARROW>
int level_w(remat_family_s* f, int lvl, long long lo, long long hi);
template <int W, bool NARROW>
int levels_w(remat_family_s* f, const std::vector<int>& lvls);
template <int W, bool NARROW>
int small_w(remat_family_s* f);
template <int W, bool NARROW>
int finish_w(remat_family_s* f, remat_plan_info* info, u64* chain_masks, u64* cached_masks,
             long long* stage_memory);
}  // namespace remat

#define REMAT_INSTANTIATE_RELAX(W)                                                          \
  template int begin_w<W, true>(remat_family_s*, const std::vector<long long>&, int);       \
  template int begin_w<W, false>(remat_family_s*, const std::vector<long long>&, int);      \
  template int level_w<W, true>(remat_family_s*, int, long long, long long);               \
  template int level_w<W, false>(remat_family_s*, int, long long, long long);              \
  template int levels_w<W, true>(remat_family_s*, const std::vector<int>&);                \
  template int levels_w<W, false>(remat_family_s*, const std::vector<int>&);               \
  template int small_w<W, true>(remat_family_s*);                                           \
  template int small_w<W, false>(remat_family_s*);                                          \
  template int finish_w<W, true>(remat_family_s*, remat_plan_info*, u64*, u64*, long long*); \
  template int finish_w<W, false>(remat_family_s*, remat_plan_info*, u64*, u64*, long long*);
