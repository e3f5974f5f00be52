/* remat_b200.h — C-ABI of libremat_b200.so, the B200 recomputation-DP solver.
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * Node sets are little-endian uint64 word arrays of W = ceil(n/64) words
 * (bit v of word v/64 = node v), the packed form of the reference's Python-int
 * bitmasks (reference pkg/src/remat/graph.py:20, NodeSet = int).
 *
 * Each entry point replaces a reference function (file:line under
 * /root/reference/pkg/src/remat); the drop-in Python layer that binds them is
 * paper_1905_11722_b200/_native.py (ctypes), see INTEGRATION.md.
 *
 * Status codes: >= 0 success (REMAT_INFEASIBLE is a result, not an error),
 * < 0 error with a message in remat_last_error() (thread-local).
 */
#ifndef REMAT_B200_H
#define REMAT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REMAT_ABI_VERSION 1

#if defined(__GNUC__)
#define REMAT_API __attribute__((visibility("default")))
#else
#define REMAT_API
#endif

enum remat_status {
  REMAT_OK = 0,
  REMAT_INFEASIBLE = 1,      /* PlanResult(feasible=False) planner.py:198-200 */
  REMAT_ERR_VALUE = -1,      /* ValueError (cap < n+1 lattice.py:66-67, bad args) */
  REMAT_ERR_LATTICE = -2,    /* LatticeTooLargeError lattice.py:21-29           */
  REMAT_ERR_CUDA = -3,       /* CUDA runtime failure -> RuntimeError            */
  REMAT_ERR_NOMEM = -4,      /* device allocation failed -> MemoryError         */
  REMAT_ERR_INTERNAL = -5,   /* reference self-check failed planner.py:206-210  */
  REMAT_ERR_RANGE = -6,      /* integer range exceeded -> GraphError            */
  REMAT_ERR_SIM = -7         /* SimulationError schedule.py:184-254             */
};

enum remat_family_kind { REMAT_FAMILY_FULL = 0, REMAT_FAMILY_PRUNED = 1 };
enum remat_objective { REMAT_MINIMIZE = 0, REMAT_MAXIMIZE = 1 };

typedef struct remat_graph_s *remat_graph_t;   /* device-resident DAG          */
typedef struct remat_family_s *remat_family_t; /* lower-set family + precompute */
typedef struct remat_comm_s *remat_comm_t;     /* NCCL communicator (level sharding) */

#define REMAT_COMM_ID_BYTES 128                /* sizeof(ncclUniqueId)        */

typedef struct {
  int64_t states_visited, table_entries, transitions, dominated_skipped;
} remat_stats; /* SearchStats planner.py:61-67 (wall_time_s is host-side) */

typedef struct {
  int32_t status;  /* REMAT_OK, REMAT_INFEASIBLE or REMAT_ERR_INTERNAL        */
  int32_t k;       /* chain length, excluding the empty set                   */
  int64_t budget;  /* the budget as passed (before clamping to 2*M(V))        */
  int64_t objective_value, peak_memory, overhead, cached_total;
  remat_stats stats;
} remat_plan_info;

typedef struct {
  int32_t status;  /* REMAT_OK or REMAT_ERR_SIM                               */
  int32_t err_code;/* 1..8, see paper_1905_11722_b200/schedule.py             */
  int64_t err_index; int32_t err_v, err_w;
  int64_t peak_live_memory, total_forward_cost, recompute_cost, backward_count;
} remat_sim_info;  /* SimulationReport schedule.py:62-68                      */

typedef struct {
  /* device milliseconds of the last family build / solve on the handle,
   * measured with CUDA events on the handle's stream */
  float enumerate_ms, precompute_ms, relax_ms, finish_ms, total_ms;
  int64_t relax_launches;   /* level-relax kernel launches in the last solve   */
  int64_t kernel_launches;  /* all kernels launched by the last call          */
  int64_t comparable_pairs; /* Σ_j |{i : L_i ⊊ L_j}| of the last solve (P)     */
} remat_timings;

REMAT_API int remat_abi_version(void);
REMAT_API const char *remat_last_error(void);
REMAT_API int remat_device_count(int32_t *count);
REMAT_API int64_t remat_kernel_launch_count(void); /* process-wide, monotone           */

/* Upload a graph (replaces ComputationGraph construction, graph.py:60-114;
 * node indexing must already be the reference's topological order). */
REMAT_API int remat_graph_create(int32_t device, int32_t n, const uint64_t *preds,
                       const uint64_t *succs, const int64_t *compute_costs,
                       const int64_t *memory_costs, remat_graph_t *out);
REMAT_API int remat_graph_free(remat_graph_t g);
/* the cudaStream_t the handle's kernels run on (for external event timing) */
REMAT_API int remat_graph_stream(remat_graph_t g, void **stream);

/* all_lower_sets (lattice.py:59-84) or pruned_lower_sets (lattice.py:87-93),
 * plus the per-member half of TransitionIndex (planner.py:104-115). */
REMAT_API int remat_family_create(remat_graph_t g, int32_t kind, int64_t cap,
                        remat_family_t *out);
REMAT_API int remat_family_size(remat_family_t f, int64_t *size);
/* members [start, start+count) in family order (popcount, mask) -> [count][W] */
REMAT_API int remat_family_masks(remat_family_t f, int64_t start, int64_t count,
                       uint64_t *out);
REMAT_API int remat_family_free(remat_family_t f);
REMAT_API int remat_family_timings(remat_family_t f, remat_timings *out);
/* Per-member figures of the last solve's budget `b` for members
 * [start, start+count): |frontier| (SearchStats.states_visited terms), |cell|
 * (table_entries terms), and the transitions (planner.py:164) and
 * comparable-pair counts of the member's LEVEL, accumulated per relaxation
 * tile on the tile's first target (their sum over any run of whole levels is
 * exact; the dense relaxation no longer attributes them per target).
 * Any output may be NULL.  Diagnostics for the per-level work profile. */
REMAT_API int remat_family_member_stats(remat_family_t f, int32_t b, int64_t start,
                                        int64_t count, int32_t *flen, int32_t *cells,
                                        uint64_t *trans, uint64_t *pairs);

/* _plan_with_index (planner.py:192-211) for nb budgets in one batched pass.
 * Optional outputs (NULL to skip), each [nb][n+1][...]:
 *   chain_masks/cached_masks [nb][n+1][W], stage_memory [nb][n+1].        */
REMAT_API int remat_solve(remat_family_t f, const int64_t *budgets, int32_t nb,
                int32_t objective, remat_plan_info *info,
                uint64_t *chain_masks, uint64_t *cached_masks,
                int64_t *stage_memory);

/* min_feasible_budget (planner.py:271-297): same B_min and plan as the
 * reference's binary search, found with batched k-ary probing. */
REMAT_API int remat_min_feasible_budget(remat_family_t f, int32_t objective,
                              int32_t probes_per_round, int64_t *b_min,
                              remat_plan_info *info, uint64_t *chain_masks,
                              uint64_t *cached_masks, int64_t *stage_memory,
                              int64_t *probes_run, int64_t *probe_transitions);

/* make_sequence + peak_memory (strategy.py:61-128) of a caller chain; the
 * chain must already be a valid sequence (validated by the host layer). */
REMAT_API int remat_evaluate(remat_graph_t g, int32_t k, const uint64_t *chain,
                   int64_t *overhead, int64_t *stage_memory, int64_t *peak,
                   int64_t *cached_total, uint64_t *cached_masks);

/* simulate (schedule.py:184-254) for nsched schedules in one launch.
 * ops: [total][2] int32 (kind, node), kind 0 = F, 1 = B, 2 = FREE fwd,
 * 3 = FREE grad; schedule s is ops[offsets[s] .. offsets[s+1]).
 * traces: [total] live memory after each instruction, or NULL. */
REMAT_API int remat_simulate(remat_graph_t g, int32_t nsched, const int64_t *offsets,
                   const int32_t *ops, remat_sim_info *info, int64_t *traces);

/* ---- K7: schedules on the device (schedule.py:88-254) -------------------
 * flags: bit 0 = apply liveness_pass (149-181) to each built stream,
 *        bit 1 = simulate (184-254) the final stream (info[], traces[]).
 * Streams come back concatenated: stream b is ops[offsets[b] .. offsets[b+1])
 * of int32 (kind, node) pairs; `cap` is the ops capacity in instructions. */

/* build_schedule (88-117) for nplans plans: plan b's chain / segments /
 * cached sets (LowerSetSequence fields, strategy.py:40-50) are rows
 * [Σ_{c<b} k[c], +k[b]) of the [Σk][W] arrays.  status[b] = REMAT_OK, or
 * REMAT_ERR_INTERNAL when the reference's assert (schedule.py:111) fails. */
REMAT_API int remat_schedule_build(remat_graph_t g, int32_t nplans, const int32_t *k,
                                   const uint64_t *chains, const uint64_t *segments,
                                   const uint64_t *cached, int32_t flags, int64_t cap,
                                   int64_t *offsets, int32_t *ops, int32_t *status,
                                   remat_sim_info *info, int64_t *traces);
/* vanilla_schedule (120-135); *nops = its length */
REMAT_API int remat_schedule_vanilla(remat_graph_t g, int32_t flags, int64_t cap, int64_t *nops,
                                     int32_t *ops, remat_sim_info *info, int64_t *traces);
/* liveness_pass and/or simulate of caller streams (offsets/ops as
 * remat_simulate); events[s] = Σ over stream s of the refs each instruction
 * touches (F v: |preds|+1, B v: |preds|+2+|succs|, FREE: 1). */
REMAT_API int remat_schedule_streams(remat_graph_t g, int32_t ns, const int64_t *offsets,
                                     const int32_t *ops, const int64_t *events, int32_t flags,
                                     int64_t cap, int64_t *out_offsets, int32_t *out_ops,
                                     remat_sim_info *info, int64_t *traces);

/* ---- level sharding across GPUs (no reference counterpart:
 * the reference is single-threaded) ----------------------
 * The targets of every heavy level of an exact-DP solve are split into
 * contiguous rank ranges; after each such level the ranks exchange the
 * finished frontiers in place (one NCCL group of per-rank broadcasts over
 * NVLink, straight into every replica).  Light levels (fewer than
 * REMAT_SHARD_REPLICATE subset tests, default 4 Mi) are relaxed by every rank
 * in full.  Every rank ends with the whole table and returns the same plan as
 * remat_solve on one GPU.  NCCL is loaded at run time (libnccl.so.2). */
REMAT_API int remat_comm_unique_id(uint8_t *id /* [REMAT_COMM_ID_BYTES] */);
REMAT_API int remat_comm_create(const uint8_t *id, int32_t world, int32_t rank,
                                int32_t device, remat_comm_t *out);
REMAT_API int remat_comm_free(remat_comm_t c);
/* targets [begin, end) of a level [level_start, level_start + width) owned by
 * `rank` (host-only helper, no device needed) */
REMAT_API int remat_level_partition(int64_t level_start, int64_t width, int32_t world,
                                    int32_t rank, int64_t *begin, int64_t *end);
/* remat_solve with the level loop sharded over the communicator's ranks; every
 * rank passes an identical family (same graph, same kind and cap). */
REMAT_API int remat_solve_level_sharded(remat_family_t f, remat_comm_t c,
                                        const int64_t *budgets, int32_t nb,
                                        int32_t objective, remat_plan_info *info,
                                        uint64_t *chain_masks, uint64_t *cached_masks,
                                        int64_t *stage_memory);
/* the same exchange with `world` replicas on ONE device (device copies in
 * place of the broadcasts): the single-GPU test form of level sharding.  The
 * replicas must be families of one graph handle. */
REMAT_API int remat_solve_level_sharded_loopback(remat_family_t *fams, int32_t world,
                                                 const int64_t *budgets, int32_t nb,
                                                 int32_t objective, remat_plan_info *info,
                                                 uint64_t *chain_masks,
                                                 uint64_t *cached_masks,
                                                 int64_t *stage_memory);

#ifdef __cplusplus
}
#endif
#endif
