// schedule.cu — K7: instruction schedules built, liveness-rewritten and
// simulated on the device, batched over many schedules (one CTA each).
//
// Reference: pkg/src/remat/schedule.py — build_schedule (88-117),
// vanilla_schedule (120-135), liveness_pass (149-181), simulate (184-254).
// Parallel forms:
//
//  * build: the canonical stream is 6k SECTIONS, each one node set emitted in
//    ascending (or, for the backward computes, descending) node order with a
//    fixed instruction kind.  Every section's set is a closed form of the
//    stage sets (segment, ∂L, the stage-entry sets), so the section lengths
//    are popcounts, their exclusive scan places each section, and a node's
//    slot inside its section is the popcount of the section below it.
//  * events: every instruction touches a few value refs (fwd u → u,
//    grad u → n+u): reads, one write ("set"), or one FREE ("clear").  The
//    events are bucketed per ref and ordered by position (counting scatter +
//    rank sort of each ref's short list); one walk per ref annotates each
//    event with the ref's state before it (live, forward-run count, whether a
//    write happened at or before it, whether the next event on the ref is a
//    write or nothing).
//  * liveness: a read/write event closes a live range iff a write of the ref
//    happened at or before it and the ref's next event is a write or nothing
//    — the per-ref segmented max of the reference's last_use bookkeeping.
//    FREEs after instruction p come out in (kind, node) order because every
//    instruction emits its events in ref order.
//  * simulate: every instruction evaluates the reference's checks, in the
//    reference's order, against the annotated state; the first faulting
//    instruction is a block min.  Live memory is an inclusive prefix sum of
//    ±M_v; the peak its max.
//
// Instruction encoding (int32 pairs, as remat_simulate): kind 0 = F, 1 = B,
// 2 = FREE fwd, 3 = FREE grad.
#include "device.cuh"

namespace remat {

constexpr int kSchedThreads = 512;
constexpr int kSchedWarps = kSchedThreads / 32;

enum : unsigned char { EV_READ = 0, EV_SET = 1, EV_CLEAR = 2 };

// ---------------------------------------------------------------------------
// block helpers
// ---------------------------------------------------------------------------

// Exclusive scan of val(i), i in [0, n), into out[i] (out[n] = total); returns
// the total.  `sh` is shared scratch of >= 34 long longs.
template <typename F>
__device__ long long block_scan_to(long long n, F val, long long* out, long long* sh) {
  long long carry = 0;
  for (long long base = 0; base < n; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    const long long v = i < n ? val(i) : 0;
    long long tot;
    const long long ex = block_exclusive_sum<long long>(v, sh, &tot);
    if (i < n) out[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
  __syncthreads();
  return carry;
}

__device__ __forceinline__ int popc64(u64 x) { return __popcll(x); }

// ---------------------------------------------------------------------------
// canonical schedule (build_schedule, schedule.py:88-117)
// ---------------------------------------------------------------------------

struct PlanSets {
  int k;
  const u64 *chain, *seg, *cached;  // [k][Wp]
  u64 *bound, *efwd, *egrad;        // [k][Wp] scratch
};

// Section s of the canonical stream (6k sections):
//   s = 2i, 2i+1 (forward sweep, stage i):  F seg_i ; FREE fwd (seg_i \ ∂L_i)
//   s = 2k + 4j + {0..3} (backward, stage i = k-1-j):
//       F (seg_i \ fwd_live) ; B seg_i (descending) ;
//       FREE fwd (fwd_live ∪ seg_i) \ fwd_target ; FREE grad likewise
// with fwd_live = cached_{k-1} (i = k-1) else entry_fwd_i, grad_live = ∅
// (i = k-1) else entry_grad_i, targets entry_*_{i-1} (∅ for i = 0).
__device__ __forceinline__ u64 section_word(const PlanSets& P, int Wp, int s, int w, int* kind) {
  const int k = P.k;
  if (s < 2 * k) {
    const int i = s >> 1;
    const u64 sg = P.seg[(size_t)i * Wp + w];
    if (!(s & 1)) {
      *kind = 0;
      return sg;
    }
    *kind = 2;
    return sg & ~P.bound[(size_t)i * Wp + w];
  }
  const int j = (s - 2 * k) >> 2, part = (s - 2 * k) & 3;
  const int i = k - 1 - j;
  const u64 sg = P.seg[(size_t)i * Wp + w];
  const u64 fl = i == k - 1 ? P.cached[(size_t)(k - 1) * Wp + w] : P.efwd[(size_t)i * Wp + w];
  switch (part) {
    case 0:
      *kind = 0;
      return sg & ~fl;
    case 1:
      *kind = 1;
      return sg;
    case 2: {
      *kind = 2;
      const u64 ft = i > 0 ? P.efwd[(size_t)(i - 1) * Wp + w] : 0ull;
      return (fl | sg) & ~ft;
    }
    default: {
      *kind = 3;
      const u64 gl = i == k - 1 ? 0ull : P.egrad[(size_t)i * Wp + w];
      const u64 gt = i > 0 ? P.egrad[(size_t)(i - 1) * Wp + w] : 0ull;
      return (gl | sg) & ~gt;
    }
  }
}

// The reference's assert (schedule.py:111): the stage's targets must be live.
__device__ __forceinline__ bool stage_targets_live(const PlanSets& P, int Wp, int i) {
  if (i == 0) return true;
  const int k = P.k;
  bool ok = true;
  for (int w = 0; w < Wp; w++) {
    const u64 sg = P.seg[(size_t)i * Wp + w];
    const u64 fl = (i == k - 1 ? P.cached[(size_t)(k - 1) * Wp + w] : P.efwd[(size_t)i * Wp + w]) | sg;
    const u64 gl = (i == k - 1 ? 0ull : P.egrad[(size_t)i * Wp + w]) | sg;
    ok &= (P.efwd[(size_t)(i - 1) * Wp + w] & ~fl) == 0 && (P.egrad[(size_t)(i - 1) * Wp + w] & ~gl) == 0;
  }
  return ok;
}

struct BuildArgs {
  GraphView g;
  const int* k;              // [nplans]
  const long long* sbase;    // [nplans] first stage row of plan b in the set arrays
  const u64 *chain, *seg, *cached;
  u64 *bound, *efwd, *egrad;  // scratch rows, same indexing
  long long* secoff;         // [Σ(6k+1)] section offsets scratch (plan b at 6·sbase[b] + b)
  int* ops;                  // out: [Σ cap_b][2]
  const long long* obase;    // [nplans] first op slot of plan b
  long long cap;             // op slots per plan
  long long* olen;           // out: [nplans] stream length
  int* status;               // out: [nplans] 0, -1 assert, -2 capacity
};

// One CTA per plan.  Stage sets: warp per stage.  ∂L_i = {v ∈ L : succs(v) ⊄ L},
// δ⁺(L) = ∪_{v∈L} succs(v), entry_grad = δ⁺(L)\L, entry_fwd = U_i ∪ (δ⁻(δ⁺(L))\L)
// (schedule.py:71-85).
__global__ void __launch_bounds__(kSchedThreads) k_build_canonical(BuildArgs A) {
  extern __shared__ u64 smem[];  // [warps][2][Wp]
  __shared__ long long sh[40];
  __shared__ int bad;
  const int b = blockIdx.x, Wp = A.g.Wp, n = A.g.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = A.k[b];
  const size_t r0 = (size_t)A.sbase[b] * Wp;
  PlanSets P{k, A.chain + r0, A.seg + r0, A.cached + r0, A.bound + r0, A.efwd + r0, A.egrad + r0};
  if (threadIdx.x == 0) bad = 0;
  u64* succ = smem + (size_t)warp * 2 * Wp;
  u64* dm = succ + Wp;
  for (int i = warp; i < k; i += kSchedWarps) {
    const u64* L = P.chain + (size_t)i * Wp;
    // ∂L and δ⁺(L): lanes over the nodes of L, 64 at a time
    for (int w = lane; w < Wp; w += 32) succ[w] = dm[w] = 0ull;
    __syncwarp();
    for (int q = 0; q < Wp; q++) {
      const u64 Lq = L[q];
      u64 bword = 0;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int v = q * 64 + h * 32 + lane;
        bool out = false;
        if (v < n && ((Lq >> (h * 32 + lane)) & 1)) {
          const u64* sv = A.g.succs + (size_t)v * Wp;
          for (int w = 0; w < Wp; w++) {
            const u64 x = sv[w];
            if (x) {
              out |= (x & ~L[w]) != 0;
              atomicOr(&succ[w], x);
            }
          }
        }
        const unsigned bal = __ballot_sync(kFull, out);
        bword |= (u64)bal << (h * 32);
      }
      if (lane == 0) P.bound[(size_t)i * Wp + q] = bword;
    }
    __syncwarp();
    // δ⁻(δ⁺(L)): lanes over the nodes of δ⁺(L)
    for (int q = 0; q < Wp; q++) {
      const u64 Sq = succ[q];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int u = q * 64 + h * 32 + lane;
        if (u < n && ((Sq >> (h * 32 + lane)) & 1)) {
          const u64* pu = A.g.preds + (size_t)u * Wp;
          for (int w = 0; w < Wp; w++)
            if (pu[w]) atomicOr(&dm[w], pu[w]);
        }
      }
    }
    __syncwarp();
    for (int w = lane; w < Wp; w += 32) {
      const u64 Lw = L[w];
      P.egrad[(size_t)i * Wp + w] = succ[w] & ~Lw;
      P.efwd[(size_t)i * Wp + w] = P.cached[(size_t)i * Wp + w] | (dm[w] & ~Lw);
    }
    __syncwarp();
  }
  __syncthreads();
  // section lengths + the reference's assert
  const int S = 6 * k;
  long long* off = A.secoff + 6 * A.sbase[b] + b;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    int kind, len = 0;
    for (int w = 0; w < Wp; w++) len += popc64(section_word(P, Wp, s, w, &kind));
    off[s] = len;
    if (s >= 2 * k && ((s - 2 * k) & 3) == 0 && !stage_targets_live(P, Wp, k - 1 - ((s - 2 * k) >> 2)))
      atomicOr(&bad, 1);
  }
  __syncthreads();
  const long long total = block_scan_to(S, [&](long long s) { return off[s]; }, off, sh);
  if (bad || total > A.cap) {
    if (threadIdx.x == 0) {
      A.status[b] = bad ? -1 : -2;
      A.olen[b] = 0;
    }
    return;
  }
  // emission: (section, word) pairs
  int* out = A.ops + 2 * A.obase[b];
  for (long long t = threadIdx.x; t < (long long)S * Wp; t += blockDim.x) {
    const int s = (int)(t / Wp), w = (int)(t % Wp);
    int kind;
    u64 x = section_word(P, Wp, s, w, &kind);
    if (!x) continue;
    long long below = 0;
    for (int q = 0; q < w; q++) below += popc64(section_word(P, Wp, s, q, &kind));
    const long long a = off[s], len = off[s + 1] - off[s];
    while (x) {
      const int bit = __ffsll((long long)x) - 1;
      x &= x - 1;
      const long long pos = kind == 1 ? a + len - 1 - below : a + below;
      out[2 * pos] = kind;
      out[2 * pos + 1] = w * 64 + bit;
      below++;
    }
  }
  if (threadIdx.x == 0) {
    A.status[b] = 0;
    A.olen[b] = total;
  }
}

// ---------------------------------------------------------------------------
// vanilla schedule (schedule.py:120-135)
// ---------------------------------------------------------------------------

// F 0..n-1; for v = n-1..0: B v, then FREE grad u for every u whose smallest
// predecessor is v (u itself when it has none), ascending; FREE fwd 0..n-1.
__global__ void __launch_bounds__(kSchedThreads) k_build_vanilla(GraphView g, u64* groups /*[n][Wp]*/,
                                                                long long* off /*[n+1]*/, int* ops,
                                                                long long* olen) {
  __shared__ long long sh[40];
  const int n = g.n, Wp = g.Wp;
  for (long long t = threadIdx.x; t < (long long)n * Wp; t += blockDim.x) groups[t] = 0ull;
  __syncthreads();
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    int lr = u;
    for (int w = 0; w < Wp; w++) {
      const u64 x = g.preds[(size_t)u * Wp + w];
      if (x) {
        lr = w * 64 + __ffsll((long long)x) - 1;
        break;
      }
    }
    atomicOr(&groups[(size_t)lr * Wp + (u >> 6)], 1ull << (u & 63));
  }
  __syncthreads();
  // backward section j = n-1-v: B v + its group
  const long long tot = block_scan_to(
      n,
      [&](long long j) {
        const int v = n - 1 - (int)j;
        int c = 0;
        for (int w = 0; w < Wp; w++) c += popc64(groups[(size_t)v * Wp + w]);
        return (long long)(1 + c);
      },
      off, sh);
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    ops[2 * v] = 0;
    ops[2 * v + 1] = v;
    const long long tail = n + tot + v;
    ops[2 * tail] = 2;
    ops[2 * tail + 1] = v;
    const long long a = n + off[n - 1 - v];
    ops[2 * a] = 1;
    ops[2 * a + 1] = v;
    long long r = a + 1;
    for (int w = 0; w < Wp; w++) {
      u64 x = groups[(size_t)v * Wp + w];
      while (x) {
        const int bit = __ffsll((long long)x) - 1;
        x &= x - 1;
        ops[2 * r] = 3;
        ops[2 * r + 1] = w * 64 + bit;
        r++;
      }
    }
  }
  if (threadIdx.x == 0) *olen = 2LL * n + tot;
}

// ---------------------------------------------------------------------------
// events (shared by liveness and simulate)
// ---------------------------------------------------------------------------

// Events of instruction (kind, v), in REF order (fwd refs u ∈ [0,n), then
// grad refs n+u): F v: read fwd preds ↑, set fwd v.  B v: read fwd preds ↑,
// read fwd v, set grad v, read grad succs ↑.  FREE fwd/grad v: clear.
// Returns the count; emit(t, ref, type) for t = 0..count-1 when kEmit.
template <bool kEmit, typename E>
__device__ __forceinline__ int inst_events(const GraphView& g, int kind, int v, E emit) {
  const int n = g.n, Wp = g.Wp;
  if (kind < 0 || kind > 3 || v < 0 || v >= n) return 0;
  if (kind >= 2) {
    if constexpr (kEmit) emit(0, kind == 2 ? v : n + v, EV_CLEAR);
    return 1;
  }
  int t = 0;
  const u64* pv = g.preds + (size_t)v * Wp;
  for (int w = 0; w < Wp; w++) {
    u64 x = pv[w];
    if constexpr (!kEmit) {
      t += popc64(x);
    } else {
      while (x) {
        const int bit = __ffsll((long long)x) - 1;
        x &= x - 1;
        emit(t++, w * 64 + bit, EV_READ);
      }
    }
  }
  if (kind == 0) {
    if constexpr (kEmit) emit(t, v, EV_SET);
    return t + 1;
  }
  if constexpr (kEmit) {
    emit(t, v, EV_READ);
    emit(t + 1, n + v, EV_SET);
  }
  t += 2;
  const u64* sv = g.succs + (size_t)v * Wp;
  for (int w = 0; w < Wp; w++) {
    u64 x = sv[w];
    if constexpr (!kEmit) {
      t += popc64(x);
    } else {
      while (x) {
        const int bit = __ffsll((long long)x) - 1;
        x &= x - 1;
        emit(t++, n + w * 64 + bit, EV_READ);
      }
    }
  }
  return t;
}

// Per-schedule scratch, carved from one arena (host and device agree on the
// layout through this struct).
struct EvArena {
  long long L, E;  // instruction and event capacities
  int R;           // refs = 2n
  __host__ __device__ static long long al(long long x) { return (x + 15) & ~15LL; }
  __host__ __device__ long long bytes() const { return off_end(); }
  __host__ __device__ long long off_evoff() const { return 0; }
  __host__ __device__ long long off_refoff() const { return off_evoff() + al(8 * (L + 1)); }
  __host__ __device__ long long off_refcnt() const { return off_refoff() + al(8 * ((long long)R + 1)); }
  __host__ __device__ long long off_pos() const { return off_refcnt() + al(4LL * R); }
  __host__ __device__ long long off_org() const { return off_pos() + al(4 * E); }
  __host__ __device__ long long off_typ() const { return off_org() + al(4 * E); }
  __host__ __device__ long long off_spos() const { return off_typ() + al(E); }
  __host__ __device__ long long off_sorg() const { return off_spos() + al(4 * E); }
  __host__ __device__ long long off_styp() const { return off_sorg() + al(4 * E); }
  __host__ __device__ long long off_ann() const { return off_styp() + al(E); }
  __host__ __device__ long long off_inst() const { return off_ann() + al(4 * E); }
  __host__ __device__ long long off_inst2() const { return off_inst() + al(8 * (L + 1)); }
  __host__ __device__ long long off_cidx() const { return off_inst2() + al(8 * (L + 1)); }
  __host__ __device__ long long off_end() const { return off_cidx() + al(4 * (L + 1)); }
};

struct EvView {
  long long* evoff;  // [L+1] first event of instruction p
  long long* refoff; // [R+1]
  int* refcnt;       // [R] counts, then fill cursors
  int *pos, *org;    // [E] bucketed by ref (unsorted)
  unsigned char* typ;
  int *spos, *sorg;  // [E] bucketed and sorted by position
  unsigned char* styp;
  unsigned* ann;     // [E] by origin: bit0 live before, bit1 next event is set/none,
                     //      bit2 a set at or before, bits 8.. set count up to it
  long long* inst;   // [L+1] per-instruction scratch
  long long* inst2;  // [L+1]
  int* cidx;         // [L+1] compute positions (liveness)
  __device__ EvView(unsigned char* base, const EvArena& a) {
    evoff = (long long*)(base + a.off_evoff());
    refoff = (long long*)(base + a.off_refoff());
    refcnt = (int*)(base + a.off_refcnt());
    pos = (int*)(base + a.off_pos());
    org = (int*)(base + a.off_org());
    typ = base + a.off_typ();
    spos = (int*)(base + a.off_spos());
    sorg = (int*)(base + a.off_sorg());
    styp = base + a.off_styp();
    ann = (unsigned*)(base + a.off_ann());
    inst = (long long*)(base + a.off_inst());
    inst2 = (long long*)(base + a.off_inst2());
    cidx = (int*)(base + a.off_cidx());
  }
};

// Bucket the events of instructions ops[idx(p)], p in [0, L), by ref, order
// each bucket by position, annotate.  Returns false (block-uniform) when the
// events exceed the arena.
template <typename IDX>
__device__ bool build_events(const GraphView& g, const int* ops, long long L, IDX idx,
                             const EvView& V, long long Ecap, long long* sh) {
  const int R = 2 * g.n;
  const long long E = block_scan_to(
      L,
      [&](long long p) {
        const long long q = idx(p);
        return (long long)inst_events<false>(g, ops[2 * q], ops[2 * q + 1], 0);
      },
      V.evoff, sh);
  if (E > Ecap) return false;
  for (int r = threadIdx.x; r < R; r += blockDim.x) V.refcnt[r] = 0;
  __syncthreads();
  for (long long p = threadIdx.x; p < L; p += blockDim.x) {
    const long long q = idx(p);
    inst_events<true>(g, ops[2 * q], ops[2 * q + 1],
                      [&](int, int r, unsigned char) { atomicAdd(&V.refcnt[r], 1); });
  }
  __syncthreads();
  block_scan_to(R, [&](long long r) { return (long long)V.refcnt[r]; }, V.refoff, sh);
  for (int r = threadIdx.x; r < R; r += blockDim.x) V.refcnt[r] = 0;
  __syncthreads();
  for (long long p = threadIdx.x; p < L; p += blockDim.x) {
    const long long q = idx(p);
    const long long e0 = V.evoff[p];
    inst_events<true>(g, ops[2 * q], ops[2 * q + 1], [&](int t, int r, unsigned char ty) {
      const long long slot = V.refoff[r] + atomicAdd(&V.refcnt[r], 1);
      V.pos[slot] = (int)p;
      V.org[slot] = (int)(e0 + t);
      V.typ[slot] = ty;
    });
  }
  __syncthreads();
  // rank sort inside each ref's bucket (positions are distinct within a ref:
  // an instruction touches a ref at most once)
  for (int r = 0; r < R; r++) {
    const long long a = V.refoff[r], z = V.refoff[r + 1];
    for (long long e = a + threadIdx.x; e < z; e += blockDim.x) {
      const int pe = V.pos[e];
      long long rank = 0;
      for (long long f = a; f < z; f++) rank += V.pos[f] < pe;
      V.spos[a + rank] = pe;
      V.sorg[a + rank] = V.org[e];
      V.styp[a + rank] = V.typ[e];
    }
  }
  __syncthreads();
  // one walk per ref
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const long long a = V.refoff[r], z = V.refoff[r + 1];
    unsigned live = 0, runs = 0, seen = 0;
    for (long long e = a; e < z; e++) {
      const unsigned char ty = V.styp[e];
      unsigned an = live;
      if (ty == EV_SET) {
        runs++;
        live = 1;
        seen = 1;
      } else if (ty == EV_CLEAR) {
        live = 0;
      }
      an |= seen << 2;
      an |= min(runs, 255u) << 8;
      V.ann[V.sorg[e]] = an;
    }
    unsigned next_set_or_none = 1;
    for (long long e = z - 1; e >= a; e--) {
      V.ann[V.sorg[e]] |= next_set_or_none << 1;
      next_set_or_none = V.styp[e] == EV_SET;
    }
  }
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------------------
// liveness_pass (schedule.py:149-181)
// ---------------------------------------------------------------------------

struct StreamArgs {
  GraphView g;
  const int* ops;           // input streams [Σ][2]
  const long long* ibase;   // [ns] first op of stream s
  const long long* ilen;    // [ns] its length
  unsigned char* arena;     // [ns] arenas of abytes each
  EvArena ea;
  long long abytes;
  int* out_ops;             // liveness output [Σ cap][2]
  const long long* obase;   // [ns]
  long long ocap;
  long long* olen;          // [ns]
  long long* sim;           // simulate results [ns][9]
  long long* trace;         // [Σ] live memory after each instruction (or null)
  const long long* tbase;   // [ns]
  int* status;              // [ns] 0 ok, -2 capacity
};

__global__ void __launch_bounds__(kSchedThreads) k_liveness(StreamArgs A) {
  __shared__ long long sh[40];
  const int s = blockIdx.x;
  const GraphView g = A.g;
  const int* ops = A.ops + 2 * A.ibase[s];
  const long long Lin = A.ilen[s];
  EvView V(A.arena + (size_t)s * A.abytes, A.ea);
  // compute positions: drop every FREE (schedule.py:158)
  const long long C = block_scan_to(
      Lin, [&](long long q) { return (long long)(ops[2 * q] == 0 || ops[2 * q] == 1); }, V.inst, sh);
  for (long long q = threadIdx.x; q < Lin; q += blockDim.x)
    if (ops[2 * q] == 0 || ops[2 * q] == 1) V.cidx[V.inst[q]] = (int)q;
  __syncthreads();
  if (C > A.ea.L || !build_events(g, ops, C, [&](long long p) { return (long long)V.cidx[p]; }, V,
                                  A.ea.E, sh)) {
    if (threadIdx.x == 0) {
      A.status[s] = -2;
      A.olen[s] = 0;
    }
    return;
  }
  // closes per compute instruction: events that saw a write at or before
  // them and whose next event on the ref is a write or nothing
  const long long total = block_scan_to(
      C,
      [&](long long p) {
        long long c = 0;
        for (long long e = V.evoff[p]; e < V.evoff[p + 1]; e++) c += (V.ann[e] & 6u) == 6u;
        return c;
      },
      V.inst2, sh);
  if (C + total > A.ocap) {
    if (threadIdx.x == 0) {
      A.status[s] = -2;
      A.olen[s] = 0;
    }
    return;
  }
  int* out = A.out_ops + 2 * A.obase[s];
  const int n = g.n;
  for (long long p = threadIdx.x; p < C; p += blockDim.x) {
    const long long q = V.cidx[p];
    long long o = p + V.inst2[p];
    out[2 * o] = ops[2 * q];
    out[2 * o + 1] = ops[2 * q + 1];
    const long long e0 = V.evoff[p];
    inst_events<true>(g, ops[2 * q], ops[2 * q + 1], [&](int t, int r, unsigned char) {
      if ((V.ann[e0 + t] & 6u) == 6u) {
        ++o;
        out[2 * o] = r < n ? 2 : 3;
        out[2 * o + 1] = r < n ? r : r - n;
      }
    });
  }
  if (threadIdx.x == 0) {
    A.status[s] = 0;
    A.olen[s] = C + total;
  }
}

// ---------------------------------------------------------------------------
// simulate (schedule.py:184-254)
// ---------------------------------------------------------------------------

// Fault codes (first faulting instruction wins, like the reference's raise):
//   1 forward reads non-live fwd   2 forward of a live value   3 >2 forwards
//   4 backward reads non-live fwd  5 backward before a consumer gradient
//   6 duplicate backward           7 double free fwd           8 double free grad
//   9 malformed instruction (kind/node out of range)
__device__ __forceinline__ int check_inst(const GraphView& g, int kind, int v, const unsigned* ann,
                                          int* w_out) {
  const int n = g.n, Wp = g.Wp;
  if (kind < 0 || kind > 3 || v < 0 || v >= n) return 9;
  if (kind >= 2) return (ann[0] & 1u) ? 0 : (kind == 2 ? 7 : 8);
  int t = 0;
  const u64* pv = g.preds + (size_t)v * Wp;
  for (int w = 0; w < Wp; w++) {
    u64 x = pv[w];
    while (x) {
      const int bit = __ffsll((long long)x) - 1;
      x &= x - 1;
      if (!(ann[t++] & 1u)) {
        *w_out = w * 64 + bit;
        return kind == 0 ? 1 : 4;
      }
    }
  }
  if (kind == 0) {
    if (ann[t] & 1u) return 2;
    return (ann[t] >> 8) > 2 ? 3 : 0;
  }
  if (!(ann[t] & 1u)) {  // the value of v itself (preds ∪ {v}, v is the largest)
    *w_out = v;
    return 4;
  }
  const unsigned self = ann[t + 1];
  t += 2;
  const u64* sv = g.succs + (size_t)v * Wp;
  for (int w = 0; w < Wp; w++) {
    u64 x = sv[w];
    while (x) {
      const int bit = __ffsll((long long)x) - 1;
      x &= x - 1;
      if (!(ann[t++] & 1u)) {
        *w_out = w * 64 + bit;
        return 5;
      }
    }
  }
  return (self & 1u) ? 6 : 0;
}

// Simulates one stream per CTA: A.ops / ibase / ilen, results in A.sim.
__device__ void simulate_stream(const StreamArgs& A, const int* ops, long long L, const EvView& V,
                                long long* sh, int s) {
  __shared__ unsigned long long first;
  const GraphView g = A.g;
  if (threadIdx.x == 0) first = ~0ull;
  __syncthreads();
  if (!build_events(g, ops, L, [](long long p) { return p; }, V, A.ea.E, sh)) {
    if (threadIdx.x == 0) A.status[s] = -2;
    return;
  }
  long long tf = 0, rc = 0, nb = 0;
  for (long long p = threadIdx.x; p < L; p += blockDim.x) {
    const int kind = ops[2 * p], v = ops[2 * p + 1];
    int w = -1;
    const int code = check_inst(g, kind, v, V.ann + V.evoff[p], &w);
    if (code) {
      atomicMin(&first, ((unsigned long long)p << 8) | (unsigned)code);
      V.inst2[p] = w;
      continue;
    }
    const long long mv = g.M[v];
    V.inst[p] = kind <= 1 ? mv : -mv;
    if (kind == 0) {
      const long long tv = g.T[v];
      tf += tv;
      const unsigned an = V.ann[V.evoff[p + 1] - 1];  // its set event: run count
      if ((an >> 8) == 2) rc += tv;
    } else if (kind == 1) {
      nb++;
    }
  }
  __syncthreads();
  const unsigned long long f = first;
  if (f != ~0ull) {
    if (threadIdx.x == 0) {
      const long long p = (long long)(f >> 8);
      long long* o = A.sim + (size_t)s * 9;
      o[0] = REMAT_ERR_SIM;
      o[1] = (long long)(f & 0xff);
      o[2] = p;
      o[3] = ops[2 * p + 1];
      o[4] = V.inst2[p];
      o[5] = o[6] = o[7] = o[8] = 0;
      A.status[s] = 0;
    }
    return;
  }
  long long tot;
  long long sums[3] = {tf, rc, nb};
  for (int c = 0; c < 3; c++) {
    block_exclusive_sum<long long>(sums[c], sh, &tot);
    sums[c] = tot;
  }
  // live memory: inclusive prefix sum of ±M_v, peak = its max (>= 0)
  long long carry = 0, peak = 0;
  long long* tr = A.trace ? A.trace + A.tbase[s] : nullptr;
  for (long long base = 0; base < L; base += blockDim.x) {
    const long long p = base + threadIdx.x;
    const long long d = p < L ? V.inst[p] : 0;
    long long blk;
    const long long ex = block_exclusive_sum<long long>(d, sh, &blk);
    const long long mem = carry + ex + d;
    if (p < L) {
      if (tr) tr[p] = mem;
      peak = max(peak, mem);
    }
    carry += blk;
  }
  // block max of peak
  for (int m = 16; m > 0; m >>= 1) peak = max(peak, __shfl_xor_sync(kFull, peak, m));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = peak;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long pk = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); q++) pk = max(pk, sh[q]);
    long long* o = A.sim + (size_t)s * 9;
    o[0] = REMAT_OK;
    o[1] = 0;
    o[2] = -1;
    o[3] = -1;
    o[4] = -1;
    o[5] = pk;
    o[6] = sums[0];
    o[7] = sums[1];
    o[8] = sums[2];
    A.status[s] = 0;
  }
}

// simulate the input streams (mode 0) or the liveness outputs (mode 1)
__global__ void __launch_bounds__(kSchedThreads) k_simulate_streams(StreamArgs A, int mode) {
  __shared__ long long sh[40];
  const int s = blockIdx.x;
  if (mode == 1 && A.status[s] != 0) return;
  const int* ops = mode == 0 ? A.ops + 2 * A.ibase[s] : A.out_ops + 2 * A.obase[s];
  const long long L = mode == 0 ? A.ilen[s] : A.olen[s];
  EvView V(A.arena + (size_t)s * A.abytes, A.ea);
  simulate_stream(A, ops, L, V, sh, s);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct SchedScratch {
  DevBuf<int> ops_in, ops_out, ints;
  DevBuf<long long> lls, sim, trace;
  DevBuf<u64> sets;
  DevBuf<unsigned char> arena;
};

static SchedScratch& scratch_of(remat_graph_s* g) {
  if (!g->sched) g->sched = new SchedScratch();
  return *(SchedScratch*)g->sched;
}

void free_sched_scratch(remat_graph_s* g) {
  delete (SchedScratch*)g->sched;
  g->sched = nullptr;
}

static void unpack_sim(const long long* o, remat_sim_info& r) {
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

// Events bound of any stream in which every node appears at most twice as F,
// once as B and three times as FREE (canonical / liveness / vanilla streams).
static long long event_bound(remat_graph_s* g) {
  return 4 * g->edges + 7LL * g->n + 16;
}

// Run liveness (flags & 1) and/or simulate (flags & 2) over `ns` streams that
// are already on the device (ops_d, per-stream base/len on the device).
static int run_streams(remat_graph_s* g, int ns, const int* ops_d, const long long* ibase_d,
                       const long long* ilen_d, long long lcap, long long ecap, int flags,
                       long long ocap, int* out_ops_d, long long* obase_d, long long* olen_d,
                       long long* sim_d, long long* trace_d, const long long* tbase_d,
                       int* status_d, SchedScratch& S) {
  cudaStream_t st = g->stream;
  EvArena ea{std::max(lcap, ocap), ecap, 2 * g->n};
  const long long ab = ea.bytes();
  int rc;
  if ((rc = S.arena.ensure((size_t)ns * ab)) < 0) return rc;
  StreamArgs A{g->view(), ops_d, ibase_d, ilen_d, S.arena.p, ea, ab, out_ops_d, obase_d, ocap,
               olen_d, sim_d, trace_d, tbase_d, status_d};
  if (flags & 1) {
    k_liveness<<<ns, kSchedThreads, 0, st>>>(A);
    RM_LAUNCHED();
  }
  if (flags & 2) {
    k_simulate_streams<<<ns, kSchedThreads, 0, st>>>(A, (flags & 1) ? 1 : 0);
    RM_LAUNCHED();
  }
  return REMAT_OK;
}

}  // namespace remat

using namespace remat;

extern "C" {

int remat_schedule_build(remat_graph_t g, int32_t nplans, const int32_t* k, const uint64_t* chains,
                         const uint64_t* segments, const uint64_t* cached, int32_t flags,
                         int64_t cap, int64_t* offsets, int32_t* ops, int32_t* status,
                         remat_sim_info* info, int64_t* traces) {
  if (!g || !k || !chains || !segments || !cached || !offsets || !ops || !status)
    return fail(REMAT_ERR_VALUE, "null graph handle or argument");
  if (nplans < 1) return fail(REMAT_ERR_VALUE, "need at least one plan");
  if ((flags & 2) && !info) return fail(REMAT_ERR_VALUE, "simulation needs an info array");
  const int n = g->n, W = g->W, Wp = g->Wp;
  int rc = graph_enter(g);
  if (rc < 0) return rc;
  cudaStream_t st = g->stream;
  SchedScratch& S = scratch_of(g);
  std::vector<long long> sbase(nplans), obase(nplans);
  long long rows = 0;
  for (int b = 0; b < nplans; b++) {
    if (k[b] < 1 || k[b] > n) return fail(REMAT_ERR_VALUE, "chain length must be in [1, n]");
    sbase[b] = rows;
    rows += k[b];
    obase[b] = (long long)b * 6 * n;
  }
  const long long per = 6LL * n;  // canonical and liveness streams are <= 6n long
  std::vector<u64> hs((size_t)rows * Wp * 3, 0ull);
  for (long long r = 0; r < rows; r++)
    for (int w = 0; w < W; w++) {
      hs[(size_t)r * Wp + w] = chains[(size_t)r * W + w];
      hs[((size_t)rows + r) * Wp + w] = segments[(size_t)r * W + w];
      hs[((size_t)2 * rows + r) * Wp + w] = cached[(size_t)r * W + w];
    }
  const size_t setw = (size_t)rows * Wp;
  if ((rc = S.sets.ensure(setw * 6)) < 0 || (rc = S.ops_in.ensure((size_t)nplans * per * 2 + 2)) < 0 ||
      (rc = S.ops_out.ensure((size_t)nplans * per * 2 + 2)) < 0 ||
      (rc = S.lls.ensure((size_t)6 * rows + nplans + 5 * (size_t)nplans + 8)) < 0 ||
      (rc = S.ints.ensure((size_t)2 * nplans + nplans + 2)) < 0 ||
      (rc = S.sim.ensure((size_t)nplans * 9)) < 0 ||
      (rc = S.trace.ensure(traces ? (size_t)nplans * per + 1 : 1)) < 0)
    return rc;
  RM_CUDA(cudaMemcpyAsync(S.sets.p, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, st));
  long long* secoff = S.lls.p;
  long long* d_sbase = secoff + 6 * rows + nplans;
  long long* d_obase = d_sbase + nplans;
  long long* d_len0 = d_obase + nplans;   // canonical lengths
  long long* d_len1 = d_len0 + nplans;    // liveness lengths
  int* d_k = S.ints.p;
  int* d_st0 = d_k + nplans;
  int* d_st1 = d_st0 + nplans;
  RM_CUDA(cudaMemcpyAsync(d_sbase, sbase.data(), 8 * nplans, cudaMemcpyHostToDevice, st));
  RM_CUDA(cudaMemcpyAsync(d_obase, obase.data(), 8 * nplans, cudaMemcpyHostToDevice, st));
  RM_CUDA(cudaMemcpyAsync(d_k, k, 4 * nplans, cudaMemcpyHostToDevice, st));
  BuildArgs B{g->view(), d_k, d_sbase, S.sets.p, S.sets.p + setw, S.sets.p + 2 * setw,
              S.sets.p + 3 * setw, S.sets.p + 4 * setw, S.sets.p + 5 * setw, secoff,
              S.ops_in.p, d_obase, per, d_len0, d_st0};
  k_build_canonical<<<nplans, kSchedThreads, (size_t)kSchedWarps * 2 * Wp * 8, st>>>(B);
  RM_LAUNCHED();
  const int* final_ops = S.ops_in.p;
  long long* final_len = d_len0;
  if (flags & 3) {
    if ((rc = run_streams(g, nplans, S.ops_in.p, d_obase, d_len0, per, event_bound(g), flags, per,
                          S.ops_out.p, d_obase, d_len1, S.sim.p, traces ? S.trace.p : nullptr,
                          d_obase, d_st1, S)) < 0)
      return rc;
    if (flags & 1) {
      final_ops = S.ops_out.p;
      final_len = d_len1;
    }
  }
  std::vector<long long> len(nplans);
  std::vector<int> st0(nplans), st1(nplans);
  RM_CUDA(cudaMemcpyAsync(len.data(), final_len, 8 * nplans, cudaMemcpyDeviceToHost, st));
  RM_CUDA(cudaMemcpyAsync(st0.data(), d_st0, 4 * nplans, cudaMemcpyDeviceToHost, st));
  if (flags & 3) RM_CUDA(cudaMemcpyAsync(st1.data(), d_st1, 4 * nplans, cudaMemcpyDeviceToHost, st));
  std::vector<long long> sim((size_t)nplans * 9);
  if (flags & 2)
    RM_CUDA(cudaMemcpyAsync(sim.data(), S.sim.p, 8 * sim.size(), cudaMemcpyDeviceToHost, st));
  RM_CUDA(cudaStreamSynchronize(st));
  offsets[0] = 0;
  for (int b = 0; b < nplans; b++) {
    status[b] = st0[b] == -1 ? REMAT_ERR_INTERNAL : REMAT_OK;
    if (st0[b] == -2 || ((flags & 3) && st1[b] == -2))
      return fail(REMAT_ERR_INTERNAL, "schedule exceeded its 6n-instruction bound");
    offsets[b + 1] = offsets[b] + (st0[b] == 0 ? len[b] : 0);
  }
  if (offsets[nplans] > cap) return fail(REMAT_ERR_VALUE, "ops buffer too small");
  for (int b = 0; b < nplans; b++) {
    const long long m = offsets[b + 1] - offsets[b];
    if (m)
      RM_CUDA(cudaMemcpyAsync(ops + 2 * offsets[b], final_ops + 2 * obase[b], 8 * m,
                              cudaMemcpyDeviceToHost, st));
    if (traces && (flags & 2) && m)
      RM_CUDA(cudaMemcpyAsync(traces + offsets[b], S.trace.p + obase[b], 8 * m,
                              cudaMemcpyDeviceToHost, st));
    if (flags & 2) unpack_sim(sim.data() + (size_t)b * 9, info[b]);
  }
  RM_CUDA(cudaStreamSynchronize(st));
  return REMAT_OK;
}

int remat_schedule_vanilla(remat_graph_t g, int32_t flags, int64_t cap, int64_t* nops,
                           int32_t* ops, remat_sim_info* info, int64_t* traces) {
  if (!g || !nops || !ops) return fail(REMAT_ERR_VALUE, "null graph handle or argument");
  if ((flags & 2) && !info) return fail(REMAT_ERR_VALUE, "simulation needs an info array");
  int rc = graph_enter(g);
  if (rc < 0) return rc;
  cudaStream_t st = g->stream;
  SchedScratch& S = scratch_of(g);
  const int n = g->n, Wp = g->Wp;
  const long long per = 6LL * n;
  if ((rc = S.sets.ensure((size_t)n * Wp)) < 0 || (rc = S.ops_in.ensure((size_t)2 * per + 2)) < 0 ||
      (rc = S.ops_out.ensure((size_t)2 * per + 2)) < 0 || (rc = S.lls.ensure((size_t)n + 16)) < 0 ||
      (rc = S.ints.ensure(4)) < 0 || (rc = S.sim.ensure(9)) < 0 ||
      (rc = S.trace.ensure((size_t)per + 1)) < 0)
    return rc;
  long long* off = S.lls.p;
  long long* d_len0 = off + n + 1;
  long long* d_len1 = d_len0 + 1;
  long long* d_zero = d_len1 + 1;
  RM_CUDA(cudaMemsetAsync(d_zero, 0, 8, st));
  k_build_vanilla<<<1, kSchedThreads, 0, st>>>(g->view(), S.sets.p, off, S.ops_in.p, d_len0);
  RM_LAUNCHED();
  const int* fops = S.ops_in.p;
  long long* flen = d_len0;
  if (flags & 3) {
    if ((rc = run_streams(g, 1, S.ops_in.p, d_zero, d_len0, per, event_bound(g), flags, per,
                          S.ops_out.p, d_zero, d_len1, S.sim.p, traces ? S.trace.p : nullptr,
                          d_zero, S.ints.p, S)) < 0)
      return rc;
    if (flags & 1) {
      fops = S.ops_out.p;
      flen = d_len1;
    }
  }
  long long len = 0;
  int stt = 0;
  long long sim[9];
  RM_CUDA(cudaMemcpyAsync(&len, flen, 8, cudaMemcpyDeviceToHost, st));
  if (flags & 3) RM_CUDA(cudaMemcpyAsync(&stt, S.ints.p, 4, cudaMemcpyDeviceToHost, st));
  if (flags & 2) RM_CUDA(cudaMemcpyAsync(sim, S.sim.p, sizeof sim, cudaMemcpyDeviceToHost, st));
  RM_CUDA(cudaStreamSynchronize(st));
  if (stt == -2) return fail(REMAT_ERR_INTERNAL, "schedule exceeded its 6n-instruction bound");
  if (len > cap) return fail(REMAT_ERR_VALUE, "ops buffer too small");
  *nops = len;
  RM_CUDA(cudaMemcpyAsync(ops, fops, 8 * len, cudaMemcpyDeviceToHost, st));
  if (traces && (flags & 2))
    RM_CUDA(cudaMemcpyAsync(traces, S.trace.p, 8 * len, cudaMemcpyDeviceToHost, st));
  RM_CUDA(cudaStreamSynchronize(st));
  if (flags & 2) unpack_sim(sim, *info);
  return REMAT_OK;
}

// liveness_pass (flags & 1) and/or simulate (flags & 2) of caller streams;
// with both, the liveness outputs are simulated.  events[s] = the exact event
// count of stream s (host-computed from the graph's degrees).
int remat_schedule_streams(remat_graph_t g, int32_t ns, const int64_t* offsets, const int32_t* ops,
                           const int64_t* events, int32_t flags, int64_t cap,
                           int64_t* out_offsets, int32_t* out_ops, remat_sim_info* info,
                           int64_t* traces) {
  if (!g || !offsets || !ops || !events) return fail(REMAT_ERR_VALUE, "null graph handle or argument");
  if (ns < 1) return fail(REMAT_ERR_VALUE, "need at least one schedule");
  if ((flags & 1) && (!out_offsets || !out_ops))
    return fail(REMAT_ERR_VALUE, "liveness needs output arrays");
  if ((flags & 2) && !info) return fail(REMAT_ERR_VALUE, "simulation needs an info array");
  if (!(flags & 3)) return fail(REMAT_ERR_VALUE, "nothing to do");
  int rc = graph_enter(g);
  if (rc < 0) return rc;
  cudaStream_t st = g->stream;
  SchedScratch& S = scratch_of(g);
  const long long total = offsets[ns] - offsets[0];
  if (offsets[0] != 0 || total < 0) return fail(REMAT_ERR_VALUE, "bad schedule offsets");
  long long lmax = 1, emax = 1;
  std::vector<long long> ibase(ns), ilen(ns), obase(ns);
  for (int s = 0; s < ns; s++) {
    ibase[s] = offsets[s];
    ilen[s] = offsets[s + 1] - offsets[s];
    if (ilen[s] < 0) return fail(REMAT_ERR_VALUE, "bad schedule offsets");
    lmax = std::max(lmax, ilen[s]);
    emax = std::max<long long>(emax, events[s]);
  }
  // a liveness output holds the computes plus one FREE per live range:
  // at most twice the input length
  const long long ocap = (flags & 1) ? 2 * lmax : 1;
  for (int s = 0; s < ns; s++) obase[s] = (long long)s * ocap;
  if ((rc = S.ops_in.ensure((size_t)2 * total + 2)) < 0 ||
      (rc = S.ops_out.ensure((size_t)2 * ns * ocap + 2)) < 0 ||
      (rc = S.lls.ensure((size_t)4 * ns + 4)) < 0 || (rc = S.ints.ensure((size_t)ns + 1)) < 0 ||
      (rc = S.sim.ensure((size_t)ns * 9)) < 0 ||
      (rc = S.trace.ensure((size_t)(traces ? std::max(total, (long long)ns * ocap) : 0) + 1)) < 0)
    return rc;
  long long* d_ib = S.lls.p;
  long long* d_il = d_ib + ns;
  long long* d_ob = d_il + ns;
  long long* d_ol = d_ob + ns;
  RM_CUDA(cudaMemcpyAsync(S.ops_in.p, ops, 8 * total, cudaMemcpyHostToDevice, st));
  RM_CUDA(cudaMemcpyAsync(d_ib, ibase.data(), 8 * ns, cudaMemcpyHostToDevice, st));
  RM_CUDA(cudaMemcpyAsync(d_il, ilen.data(), 8 * ns, cudaMemcpyHostToDevice, st));
  RM_CUDA(cudaMemcpyAsync(d_ob, obase.data(), 8 * ns, cudaMemcpyHostToDevice, st));
  // the simulated stream's event bound: the input's, or (liveness first) the
  // same computes with at most as many FREEs as events
  const long long ecap = emax + ((flags & 1) ? lmax : 0) + 16;
  if ((rc = run_streams(g, ns, S.ops_in.p, d_ib, d_il, lmax, ecap, flags, ocap, S.ops_out.p, d_ob,
                        d_ol, S.sim.p, traces ? S.trace.p : nullptr, (flags & 1) ? d_ob : d_ib,
                        S.ints.p, S)) < 0)
    return rc;
  std::vector<long long> olen(ns);
  std::vector<int> stt(ns);
  std::vector<long long> sim((size_t)ns * 9);
  RM_CUDA(cudaMemcpyAsync(stt.data(), S.ints.p, 4 * ns, cudaMemcpyDeviceToHost, st));
  if (flags & 1) RM_CUDA(cudaMemcpyAsync(olen.data(), d_ol, 8 * ns, cudaMemcpyDeviceToHost, st));
  if (flags & 2)
    RM_CUDA(cudaMemcpyAsync(sim.data(), S.sim.p, 8 * sim.size(), cudaMemcpyDeviceToHost, st));
  RM_CUDA(cudaStreamSynchronize(st));
  for (int s = 0; s < ns; s++)
    if (stt[s] == -2) return fail(REMAT_ERR_INTERNAL, "schedule events exceeded their bound");
  if (flags & 1) {
    out_offsets[0] = 0;
    for (int s = 0; s < ns; s++) out_offsets[s + 1] = out_offsets[s] + olen[s];
    if (out_offsets[ns] > cap) return fail(REMAT_ERR_VALUE, "ops buffer too small");
    for (int s = 0; s < ns; s++)
      if (olen[s])
        RM_CUDA(cudaMemcpyAsync(out_ops + 2 * out_offsets[s], S.ops_out.p + 2 * obase[s],
                                8 * olen[s], cudaMemcpyDeviceToHost, st));
  }
  if (traces && (flags & 2)) {
    for (int s = 0; s < ns; s++) {
      const long long m = (flags & 1) ? olen[s] : ilen[s];
      const long long src = (flags & 1) ? obase[s] : ibase[s];
      const long long dst = (flags & 1) ? out_offsets[s] : ibase[s];
      if (m) RM_CUDA(cudaMemcpyAsync(traces + dst, S.trace.p + src, 8 * m, cudaMemcpyDeviceToHost, st));
    }
  }
  RM_CUDA(cudaStreamSynchronize(st));
  if (flags & 2)
    for (int s = 0; s < ns; s++) unpack_sim(sim.data() + (size_t)s * 9, info[s]);
  return REMAT_OK;
}

}  // extern "C"
