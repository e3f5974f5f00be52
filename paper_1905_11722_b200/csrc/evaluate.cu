// evaluate.cu — strategy figures of a chain (make_sequence + peak_memory,
// reference strategy.py:61-128), on device.
//
// Stage r of the chain L_1 ⊊ … ⊊ L_k (V_r = L_r \ L_{r-1}) needs
//   a_r   = M(∂L_r ∩ V_r)          (what stage r adds to the cache)
//   tt_r  = T(V_r \ ∂L_r)          (its recompute overhead, Eq. 1 stage-wise)
//   seg2  = 2·M(V_r), base_r = M(δ+(L_r)\L_r) + M(δ−(δ+(L_r))\L_r)
// and these are independent per stage: since U_k ∩ V_r = ∂L_r ∩ V_r (SURVEY
// Appendix A.5), M(U_{r-1}) = Σ_{q<r} a_q, so Eq. 2 is a prefix sum.  One warp
// per (stage, chain) computes the terms; one warp per chain scans them and
// re-derives the cache union U_r = ⋃ ∂L_q explicitly, checking both forms of
// Eq. 1 and the cache total like the reference's asserts (strategy.py:100,
// planner.py:206-210).
#include "device.cuh"

namespace remat {

template <int W>
__device__ __forceinline__ bool bit_in(const u64 (&a)[W], int v) {
  u64 r = 0;
#pragma unroll
  for (int w = 0; w < W; w++)
    if (w == (v >> 6)) r = a[w];
  return (r >> (v & 63)) & 1ull;
}

template <int W>
__global__ void k_stage_terms(GraphView g, const u64* __restrict__ chains,
                              const int* __restrict__ klen, long long* __restrict__ terms,
                              u64* __restrict__ bounds) {
  __shared__ u64 bsh[W];
  const int lane = threadIdx.x;
  const int st = blockIdx.x, b = blockIdx.y;
  const int n = g.n;
  if (st >= klen[b]) return;
  const u64* row = chains + ((size_t)b * (n + 1) + st) * W;
  u64 L[W], P[W], dp[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    L[w] = row[w];
    P[w] = st > 0 ? row[w - W] : 0ull;
    dp[w] = 0;
  }
  if (lane < W) bsh[lane] = 0;
  __syncwarp();
  long long a = 0, tt = 0, seg2 = 0;
  for (int v0 = 0; v0 < n; v0 += 32) {
    int v = v0 + lane;
    bool isb = false;
    if (v < n && bit_in<W>(L, v)) {
      const u64* sv = g.succs + (size_t)v * W;
      u64 outside = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        u64 x = __ldg(sv + w);
        dp[w] |= x;
        outside |= x & ~L[w];
      }
      isb = outside != 0;
      if (!bit_in<W>(P, v)) {  // v ∈ V_r
        long long m = __ldg(g.M + v);
        seg2 += 2 * m;
        if (isb) a += m; else tt += __ldg(g.T + v);
      }
    }
    unsigned bal = __ballot_sync(kFull, isb);
    if (lane == 0) bsh[v0 >> 6] |= (u64)bal << (v0 & 63);
  }
  a = warp_sum(a);
  tt = warp_sum(tt);
  seg2 = warp_sum(seg2);
  u64 D[W], dm[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    D[w] = warp_or(dp[w]) & ~L[w];
    dm[w] = 0;
  }
  long long md = 0;
  for (int v0 = 0; v0 < n; v0 += 32) {
    int v = v0 + lane;
    if (v < n && bit_in<W>(D, v)) {
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
  for (int v0 = 0; v0 < n; v0 += 32) {
    int v = v0 + lane;
    if (v < n && bit_in<W>(E, v)) me += __ldg(g.M + v);
  }
  me = warp_sum(me);
  __syncwarp();
  long long* t = terms + ((size_t)b * (n + 1) + st) * 4;
  if (lane == 0) {
    t[0] = a;
    t[1] = tt;
    t[2] = seg2;
    t[3] = md + me;
  }
  if (lane < W) bounds[((size_t)b * (n + 1) + st) * W + lane] = bsh[lane];
}

// results[b][8] = {status, k, overhead, peak, cached_total, stagewise, 0, 0}
template <int W>
__global__ void k_eval_finish(GraphView g, const long long* __restrict__ terms,
                              const u64* __restrict__ bounds, const int* __restrict__ klen,
                              const long long* __restrict__ expect,
                              long long* __restrict__ stage_mem, u64* __restrict__ cached,
                              long long* __restrict__ results) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const int n = g.n;
  const int k = klen[b];
  long long* r = results + (size_t)b * 8;
  if (k <= 0) {
    if (lane == 0) {
      r[0] = k == 0 ? REMAT_INFEASIBLE : REMAT_ERR_INTERNAL;
      r[1] = 0;
      for (int q = 2; q < 8; q++) r[q] = 0;
    }
    return;
  }
  long long cache = 0, peak = 0, stagewise = 0;
  u64 U = 0;
  for (int s = 0; s < k; s++) {
    const long long* t = terms + ((size_t)b * (n + 1) + s) * 4;
    long long mem = cache + t[2] + t[3];
    if (lane == 0) stage_mem[(size_t)b * (n + 1) + s] = mem;
    peak = (s == 0 || mem > peak) ? mem : peak;
    cache += t[0];
    stagewise += t[1];
    if (lane < W) {
      U |= bounds[((size_t)b * (n + 1) + s) * W + lane];
      cached[((size_t)b * (n + 1) + s) * W + lane] = U;
    }
  }
  long long tv = 0, mu = 0;
  if (lane < W) {
    int cnt = n - lane * 64;
    u64 full = cnt >= 64 ? ~0ull : (cnt <= 0 ? 0ull : ((1ull << cnt) - 1));
    tv = word_weight(full & ~U, lane, g.T);
    mu = word_weight(U, lane, g.M);
  }
  tv = warp_sum(tv);
  mu = warp_sum(mu);
  if (lane == 0) {
    long long status = REMAT_OK;
    if (tv != stagewise || mu != cache) status = REMAT_ERR_INTERNAL;  // strategy.py:100
    if (expect && expect[b * 4 + 3]) {
      // planner.py:206-210: overhead == t*, peak <= budget, cached == final[t*]
      if (tv != expect[b * 4 + 0] || cache != expect[b * 4 + 1] || peak > expect[b * 4 + 2])
        status = REMAT_ERR_INTERNAL;
    }
    r[0] = status;
    r[1] = k;
    r[2] = tv;
    r[3] = peak;
    r[4] = cache;
    r[5] = stagewise;
    r[6] = 0;
    r[7] = 0;
  }
}

int evaluate_chains(remat_graph_s* g, int nb, const u64* chains, const int* klen,
                    const long long* expect, long long* stage_mem, u64* cached_masks,
                    long long* results, long long* terms, u64* bounds) {
  int rc = fail(REMAT_ERR_VALUE, "unsupported word count");
  cudaStream_t s = g->stream;
  dispatch_words(g->Wp, [&](auto wc) {
    constexpr int W = decltype(wc)::value;
    rc = REMAT_OK;
    k_stage_terms<W><<<dim3(g->n + 1, nb), 32, 0, s>>>(g->view(), chains, klen, terms, bounds);
    count_launch();
    k_eval_finish<W><<<nb, 32, 0, s>>>(g->view(), terms, bounds, klen, expect, stage_mem,
                                       cached_masks, results);
    count_launch();
  });
  if (rc < 0) return rc;
  RM_CUDA(cudaGetLastError());
  return REMAT_OK;
}

}  // namespace remat
