// simulate.cu — K7, the abstract-memory schedule simulator (reference
// schedule.py:184-254), batched: one warp per schedule, lane q owns word q of
// the live forward / gradient sets, so every dependency check is a W-wide AND
// plus one ballot.  Fault codes (first faulting instruction wins, like the
// reference's raise):
//   1 forward reads non-live fwd   2 forward of a live value   3 >2 forwards
//   4 backward reads non-live fwd  5 backward before a consumer gradient
//   6 duplicate backward           7 double free fwd           8 double free grad
//   9 malformed instruction (kind/node out of range)
#include "device.cuh"

namespace remat {

template <int W>
__global__ void k_simulate(GraphView g, const long long* __restrict__ offs,
                           const int* __restrict__ ops, long long* __restrict__ traces,
                           long long* __restrict__ out) {
  extern __shared__ unsigned char runs[];
  const int s = blockIdx.x, lane = threadIdx.x;
  const int n = g.n;
  for (int v = lane; v < n; v += 32) runs[v] = 0;
  __syncwarp();
  u64 fwd = 0, grad = 0;
  long long mem = 0, peak = 0, total = 0, rec = 0, back = 0;
  int code = 0, ev = -1, ew = -1;
  long long eidx = -1;
  const long long a = offs[s], z = offs[s + 1];
  for (long long idx = a; idx < z; idx++) {
    const int kind = ops[2 * idx], v = ops[2 * idx + 1];
    if (kind < 0 || kind > 3 || v < 0 || v >= n) {
      code = 9;
      ev = v;
      eidx = idx - a;
      break;
    }
    const int q = v >> 6;
    const u64 bit = 1ull << (v & 63);
    const u64 fq = __shfl_sync(kFull, fwd, q), gq = __shfl_sync(kFull, grad, q);
    const long long mv = __ldg(g.M + v);
    if (kind == 0) {
      u64 miss = lane < W ? (__ldg(g.preds + (size_t)v * W + lane) & ~fwd) : 0ull;
      unsigned bal = __ballot_sync(kFull, miss != 0);
      if (bal) {
        int l0 = __ffs(bal) - 1;
        u64 x = __shfl_sync(kFull, miss, l0);
        code = 1; ev = v; ew = l0 * 64 + __ffsll((long long)x) - 1; eidx = idx - a;
        break;
      }
      if (fq & bit) { code = 2; ev = v; eidx = idx - a; break; }
      int r = runs[v] + 1;
      __syncwarp();
      if (lane == 0) runs[v] = (unsigned char)min(r, 3);
      __syncwarp();
      if (r > 2) { code = 3; ev = v; eidx = idx - a; break; }
      long long tv = __ldg(g.T + v);
      if (r == 2) rec += tv;
      total += tv;
      if (lane == q) fwd |= bit;
      mem += mv;
    } else if (kind == 1) {
      u64 need = lane < W ? __ldg(g.preds + (size_t)v * W + lane) : 0ull;
      if (lane == q) need |= bit;
      u64 miss = need & ~fwd;
      unsigned bal = __ballot_sync(kFull, miss != 0);
      if (bal) {
        int l0 = __ffs(bal) - 1;
        u64 x = __shfl_sync(kFull, miss, l0);
        code = 4; ev = v; ew = l0 * 64 + __ffsll((long long)x) - 1; eidx = idx - a;
        break;
      }
      u64 miss2 = lane < W ? (__ldg(g.succs + (size_t)v * W + lane) & ~grad) : 0ull;
      bal = __ballot_sync(kFull, miss2 != 0);
      if (bal) {
        int l0 = __ffs(bal) - 1;
        u64 x = __shfl_sync(kFull, miss2, l0);
        code = 5; ev = v; ew = l0 * 64 + __ffsll((long long)x) - 1; eidx = idx - a;
        break;
      }
      if (gq & bit) { code = 6; ev = v; eidx = idx - a; break; }
      if (lane == q) grad |= bit;
      mem += mv;
      back++;
    } else if (kind == 2) {
      if (!(fq & bit)) { code = 7; ev = v; eidx = idx - a; break; }
      if (lane == q) fwd ^= bit;
      mem -= mv;
    } else {
      if (!(gq & bit)) { code = 8; ev = v; eidx = idx - a; break; }
      if (lane == q) grad ^= bit;
      mem -= mv;
    }
    if (mem > peak) peak = mem;
    if (traces && lane == 0) traces[idx] = mem;
  }
  if (lane == 0) {
    long long* o = out + (size_t)s * 9;
    o[0] = code ? REMAT_ERR_SIM : REMAT_OK;
    o[1] = code;
    o[2] = eidx;
    o[3] = ev;
    o[4] = ew;
    o[5] = peak;
    o[6] = total;
    o[7] = rec;
    o[8] = back;
  }
}

int simulate_batch(remat_graph_s* g, int nsched, const long long* offsets_h, const int* ops_h,
                   long long total, remat_sim_info* info, long long* traces_h) {
  cudaStream_t s = g->stream;
  int rc;
  if ((rc = g->ops_buf.ensure((size_t)2 * total + 2)) < 0 ||
      (rc = g->off_buf.ensure((size_t)nsched + 1)) < 0 ||
      (rc = g->trace_buf.ensure((size_t)total + 1)) < 0 ||
      (rc = g->ll_buf.ensure((size_t)nsched * 9)) < 0)
    return rc;
  RM_CUDA(cudaMemcpyAsync(g->ops_buf.p, ops_h, sizeof(int) * 2 * total, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(g->off_buf.p, offsets_h, sizeof(long long) * (nsched + 1),
                          cudaMemcpyHostToDevice, s));
  rc = fail(REMAT_ERR_VALUE, "unsupported word count");
  dispatch_words(g->Wp, [&](auto wc) {
    constexpr int W = decltype(wc)::value;
    k_simulate<W><<<nsched, 32, (size_t)g->n, s>>>(g->view(), g->off_buf.p, g->ops_buf.p,
                                                    traces_h ? g->trace_buf.p : nullptr,
                                                    g->ll_buf.p);
    count_launch();
    rc = REMAT_OK;
  });
  if (rc < 0) return rc;
  RM_CUDA(cudaGetLastError());
  std::vector<long long> res((size_t)nsched * 9);
  RM_CUDA(cudaMemcpyAsync(res.data(), g->ll_buf.p, sizeof(long long) * nsched * 9,
                          cudaMemcpyDeviceToHost, s));
  if (traces_h && total > 0)
    RM_CUDA(cudaMemcpyAsync(traces_h, g->trace_buf.p, sizeof(long long) * total,
                            cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < nsched; i++) {
    const long long* o = res.data() + (size_t)i * 9;
    remat_sim_info& r = info[i];
    r.status = (int)o[0];
    r.err_code = (int)o[1];
    r.err_index = o[2];
    r.err_v = (int)o[3];
    r.err_w = (int)o[4];
    r.peak_live_memory = o[5];
    r.total_forward_cost = o[6];
    r.recompute_cost = o[7];
    r.backward_count = o[8];
  }
  return REMAT_OK;
}

}  // namespace remat
