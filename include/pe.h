/* pe.h — C-ABI of the B200 candidate-evaluation engine for automap
 * (arxiv 2112.02958).  This header is the drop-in boundary: plain C types,
 * caller-owned buffers, status codes instead of exceptions.
 *
 * Every entry point names the reference interface it replaces
 * (REF = /root/reference/proj, SPEC = /root/reference/SPEC.md).  The same
 * structs are used by the CPU parity oracle (oracle/), so a harness can call
 * either implementation through one set of types.
 *
 * Threading: graphs are immutable after creation and may be shared.  One
 * engine per device.  An engine's calls must not run concurrently from
 * several host threads (search is single-threaded); calls on
 * different CUDA streams are accepted and are serialised on the device (each
 * call's stream waits for the previous call's work: they share the engine's
 * arenas, work counters and staging buffers).  Device-mode outputs of a call
 * are complete when its stream reaches the call's last enqueued work.
 */
#ifndef PE_H_
#define PE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PE_MAX_AXES 4  /* mesh axes per program (REF mesh.h:38-48)          */
#define PE_MAX_RANK 4  /* tensor rank bound kMaxRank (REF tensor.h:46)       */

/* Library status codes; the C++ exception hierarchy of REF error.h:25-60
 * maps onto these (the reference CLI maps them to exit codes 1/2/70,
 * SPEC:730). */
typedef enum pe_status {
  PE_OK = 0,
  PE_ERR_PARSE = 1,            /* ParseError(line, col)   error.h:28-39  */
  PE_ERR_VALIDATION = 2,       /* ValidationError         error.h:43-46  */
  PE_ERR_ILLEGAL = 3,          /* IllegalActionError      error.h:49-52  */
  PE_ERR_INVALID_ARGUMENT = 4, /* bad pointer / size at the boundary     */
  PE_ERR_CUDA = 5,             /* CUDA runtime failure                    */
  PE_ERR_NO_DEVICE = 6,        /* no CUDA device: the engine never falls back to CPU */
  PE_ERR_CAPACITY = 7,         /* a per-candidate arena bound was exceeded */
  PE_ERR_INTERNAL = 70         /* InternalError           error.h:57-62  */
} pe_status;

typedef struct pe_error {
  int32_t code;   /* pe_status */
  int32_t line;   /* ParseError position, 1-based; 0 otherwise */
  int32_t column;
  char message[500];
} pe_error;

/* ---- actions (SPEC:484-487 `Action` = TileValue | InferRest | Stop) ---- */
enum {
  PE_ACT_TILE = 0,       /* apply_tile_action(value, dim, axis) then propagate
                            (REF rewrite.cc:61-113, propagate.cc:459-482)      */
  PE_ACT_TILE_GROUP = 1, /* the same on every member of a scope group, one
                            propagate (grouping SPEC:568)            */
  PE_ACT_INFER_REST = 2, /* infer_rest (REF propagate.cc:484-544) over the auto
                            axes; a decision                    */
  PE_ACT_STOP = 3        /* terminal                                           */
};

typedef struct pe_action {
  uint32_t value; /* value index (args [0,A), ops [A,A+N)) or group index */
  uint8_t dim;
  uint8_t axis;   /* mesh axis index in declaration order */
  uint8_t kind;   /* PE_ACT_* */
  uint8_t pad;    /* PE_ACT_FLAG_* */
} pe_action;

/* A TILE action produced by expanding an INFER_REST decision: applied and
 * propagated like any tile action, but not counted as a decision (the
 * INFER_REST marker before it is). */
#define PE_ACT_FLAG_INFERRED 1u
/* An INFER_REST marker whose inferred tile actions follow it (output of
 * pe_infer_rest).  Unexpanded INFER_REST actions are expanded by the entry
 * points: pe_eval_batch (host buffers) and pe_rollout_batch expand every
 * candidate's next one in the same batched evaluation. */
#define PE_ACT_FLAG_EXPANDED 2u

/* ---- per-candidate result record ---- */
enum {
  PE_CAND_OK = 0,
  PE_CAND_ILLEGAL = 1,  /* an action raised IllegalActionError; the state
                           before it is scored, fail_step names the action  */
  PE_CAND_INTERNAL = 2, /* InternalError / ValidationError inside propagate or
                           lowering; no score                               */
  PE_CAND_CAPACITY = 3, /* engine arena bound exceeded (engine only)        */
  PE_CAND_PAUSED = 4    /* internal: an InferRest decision awaiting the
                           host's batched expansion; never returned         */
};

typedef struct pe_result {
  int64_t peak_bytes;       /* peak_liveness            SPEC cost module    */
  int64_t flops;            /* flop_count on local shapes                   */
  int64_t reduction_bytes;  /* comm_cost: sum of all_reduce bytes           */
  int64_t baseline_bytes;   /* max(1, replicated plan peak) used by reward  */
  int64_t ar_bytes[PE_MAX_AXES]; /* collective_stats   REF spmd.cc:405-434 */
  int64_t ag_bytes[PE_MAX_AXES];
  int32_t ar_cnt[PE_MAX_AXES];
  int32_t ag_cnt[PE_MAX_AXES];
  int32_t sbc_cnt[PE_MAX_AXES];
  int32_t n_spmd_ops;       /* ops in the lowered program (REF spmd.h:67)   */
  int32_t n_stuck;          /* stuck nodes of the last propagate            */
  int32_t n_steps;          /* decisions applied (reward's steps term)      */
  int32_t status;           /* PE_CAND_*                                    */
  int32_t fail_step;        /* index of the failing action, or -1           */
  int32_t feasible;         /* peak <= memory budget                        */
  int32_t reserved;         /* 0 */
  int32_t reserved2;        /* 0 (explicit: no uninitialised padding bytes) */
  double runtime_s;         /* runtime_estimate                             */
  double reward;            /* reward in [0,1]                              */
} pe_result;

/* Cost-model constants (SPEC cost module, defaults at SPEC "Default
 * CostParams": 16 GiB, 1e14 flop/s, 1e11 B/s, 1e-6 s, w_mem 0.1, w_comm 1.0,
 * w_steps 0.01). */
typedef struct pe_cost_params {
  int64_t memory_budget_bytes;
  double flops_per_second;
  double bytes_per_second;
  double collective_latency_s;
  double w_mem;
  double w_comm;
  double w_steps;
} pe_cost_params;

/* Search / rollout configuration (SPEC `SearchConfig`). */
typedef struct pe_search_config {
  uint32_t auto_axes_mask; /* bit i = mesh axis i may be searched          */
  uint32_t max_decisions;  /* default 32                                   */
  uint32_t group_scopes;   /* 1 = worklist entries are scope groups        */
  uint32_t episodes;       /* MCTS budget                                  */
  uint64_t seed;
  double uct_c;            /* default 1.414                                */
  uint32_t leaf_batch;     /* leaves evaluated per GPU launch              */
  uint32_t scoped_only;    /* 1 = worklist holds only arguments with a scope
                              (parameters); unscoped inputs are left to manual
                              decisions, as automap's batch axis (PAPER §2.2) */
  uint32_t resurface_stuck; /* 1 = stuck nodes resurface into the worklist
                              (SPEC Worklist: "plus stuck nodes resurfaced by
                              propagation"; REF propagate.cc:412-454): after
                              every decision, the ops of the fixpoint's stuck
                              list join the worklist in discovery order, once
                              each, as TileValue(op result) entries.  Their
                              ordinals follow the static entries:
                              (n_entries + op) * 4 * n_auto + dim * n_auto + ai.
                              Rollouts enumerate legal actions in worklist
                              order (static entries, then resurfaced ones in
                              discovery order).  0 (default) = static worklist */
  const uint32_t* worklist_args; /* optional (NULL = all): the ranker's top-k
                              argument indices (SPEC build_worklist "optionally
                              filtered to ranker top-k").  Static entries are
                              restricted to them: an argument entry is kept when
                              listed, a scope group when any member is listed
                              (a TILE_GROUP action still tiles every member).
                              Read once at engine / oracle setup. */
  uint32_t n_worklist_args;
  uint32_t infer_rest_action; /* 1 = InferRest is a legal action (SPEC
                              legal_actions: "plus InferRest (if any argument
                              untiled)"): legal when some
                              argument is neither sliced nor atomic-wrapped;
                              its ordinal follows every TileValue ordinal
                              (Stop stays last); rollouts draw uniformly over
                              TileValue + InferRest, Stop weight 1 before the
                              first decision and 2 after.  Applying it runs
                              infer_rest (REF propagate.cc:484-544) over the
                              auto axes.  0 (default) = TileValue + Stop. */
} pe_search_config;

void pe_default_cost_params(pe_cost_params* out);
void pe_default_search_config(pe_search_config* out);

/* ---- trace layout (parity; identical for engine and oracle) ----
 * int32 words per candidate:
 *   [0] words used (negative: buffer too small)
 *   [1] n_args, then one spec word per SPMD argument (REF spmd.cc:370-391)
 *   spec word of the returned value
 *   n_stuck, then (op index, reason) pairs (REF propagate.h:28-38)
 *   n_ops, then per SPMD op: head, local_bytes lo, hi, spec word of the op's
 *   final registered DistType, operand buffer indices (arg i -> i, op j -> A+j)
 * head = kind | (axis+1)<<8 | (dim+1)<<12 | n_operands<<16, kind = REF OpKind
 * value (ir.h:31-62).  spec word = per dim (axis+1) in 4 bits (dims 0..3 in
 * bits 0..15) | pending-sum axis mask << 16 | rank << 24.
 */
#define PE_TRACE_KIND_ALL_REDUCE 22
#define PE_TRACE_KIND_ALL_GATHER 23
#define PE_TRACE_KIND_SLICE_BY_COORD 24

/* ---- graph: parse_program + graph compiler ---- */
typedef struct pe_graph pe_graph;

/* Replaces `Program parse_program(std::string_view)` (REF parser.h:28):
 * parses + validates `.pir` text and compiles it into the engine's
 * structure-of-arrays form.  Only untiled (base-dialect) programs are
 * accepted as search roots. */
pe_status pe_graph_create(const char* pir, size_t len, pe_graph** out,
                          pe_error* err);

/* Structured construction: the same graph from arrays instead of text, for
 * a reference-side binding that walks a `partir::Program` (REF ir.h:84-131)
 * directly instead of printing it and re-parsing.  Values
 * are indexed args first, then ops; an op may only use earlier values.  The
 * graph is shape-checked exactly as pe_graph_create's. */
typedef struct pe_arg_desc {
  const char* id;     /* value name (NULL: "a<i>")                        */
  const char* scope;  /* SPEC `scope` attribute, may be NULL              */
  int32_t rank;
  int64_t shape[PE_MAX_RANK];
} pe_arg_desc;

typedef struct pe_op_desc {
  const char* id;           /* value name (NULL: "<i>")                    */
  int32_t kind;             /* REF OpKind value (ir.h:31-62), base dialect */
  int32_t rank;             /* declared result type                        */
  int64_t shape[PE_MAX_RANK];
  int32_t n_operands;
  const int32_t* operands;  /* value indices                               */
  /* dot (REF ir.h DotDims): n_batch / n_contract pairs                    */
  int32_t n_batch, n_contract;
  int32_t lhs_batch[PE_MAX_RANK], rhs_batch[PE_MAX_RANK];
  int32_t lhs_contract[PE_MAX_RANK], rhs_contract[PE_MAX_RANK];
  /* reduce dims / transpose perm / broadcast_in_dim map                   */
  int32_t n_dims;
  int32_t dims[PE_MAX_RANK];
  int64_t start[PE_MAX_RANK], limit[PE_MAX_RANK]; /* slice (rank entries) */
  int32_t dim;              /* concatenate                                 */
  double value;             /* constant                                    */
  const char* scope;        /* may be NULL                                 */
} pe_op_desc;

pe_status pe_graph_create_from_arrays(const char* name, int32_t n_axes,
                                      const char* const* axis_names,
                                      const int64_t* axis_sizes, int32_t n_args,
                                      const pe_arg_desc* args, int32_t n_ops,
                                      const pe_op_desc* ops, int32_t result,
                                      pe_graph** out, pe_error* err);
void pe_graph_destroy(pe_graph* g);
int32_t pe_graph_num_args(const pe_graph* g);
int32_t pe_graph_num_ops(const pe_graph* g);
int32_t pe_graph_num_axes(const pe_graph* g);
int32_t pe_graph_num_operands(const pe_graph* g);
int64_t pe_graph_axis_size(const pe_graph* g, int32_t axis);
/* value index of `%name` (args first, then ops), -1 when absent */
int32_t pe_graph_value_index(const pe_graph* g, const char* name);
int32_t pe_graph_axis_index(const pe_graph* g, const char* name);
/* mesh axis name into buf (declaration order); returns length or -1 */
int32_t pe_graph_axis_name(const pe_graph* g, int32_t axis, char* buf, int32_t cap);
/* value name into buf; returns length or -1 */
int32_t pe_graph_value_name(const pe_graph* g, int32_t value, char* buf,
                            int32_t cap);
/* value rank and dims */
int32_t pe_graph_value_shape(const pe_graph* g, int32_t value, int64_t* dims);
/* argument scope tag (SPEC tensor_ir `scope`); returns length or -1 */
int32_t pe_graph_arg_scope(const pe_graph* g, int32_t arg, char* buf, int32_t cap);
/* scope groups (normalisation SPEC:568) */
int32_t pe_graph_num_groups(const pe_graph* g);
int32_t pe_graph_group_size(const pe_graph* g, int32_t group);
int32_t pe_graph_group_member(const pe_graph* g, int32_t group, int32_t i);

/* ---- engine: one per device ---- */
typedef struct pe_engine pe_engine;

/* Uploads the compiled graph to HBM and sizes the per-candidate arenas.
 * Fails with PE_ERR_NO_DEVICE when no CUDA device is present — there is no
 * CPU fallback. */
pe_status pe_engine_create(const pe_graph* g, const pe_search_config* cfg,
                           const pe_cost_params* cp, int32_t device,
                           pe_engine** out, pe_error* err);
void pe_engine_destroy(pe_engine* e);

#define PE_MEM_DEVICE 1u /* all array arguments are device pointers      */
#define PE_SYNC 2u       /* synchronize the stream before returning       */

/* Batched evaluation: for each candidate c, apply
 * acts[seq_off[c] .. seq_off[c+1]) from the untiled graph — each action is
 * apply_tile_action (REF rewrite.cc:61) followed by propagate
 * (REF propagate.cc:459) — then lower_to_spmd (REF spmd.cc:328),
 * collective_stats (REF spmd.cc:405) and the SPEC cost model.  `trace` may be
 * NULL; otherwise n_cand * trace_words int32 words.  `stream` is a
 * cudaStream_t (NULL = legacy default stream). */
pe_status pe_eval_batch(pe_engine* e, const pe_action* acts,
                        const uint32_t* seq_off, uint32_t n_cand,
                        pe_result* out, int32_t* trace, uint32_t trace_words,
                        uint32_t flags, void* stream, pe_error* err);

/* pe_eval_batch plus per-candidate argument flags (n_cand x A bytes, may be
 * NULL): bit 0 = the argument is sliced (tiled), bit 1 = atomic-wrapped.
 * INFER_REST actions must already be expanded. */
pe_status pe_eval_batch_ex(pe_engine* e, const pe_action* acts,
                           const uint32_t* seq_off, uint32_t n_cand,
                           pe_result* out, int32_t* trace, uint32_t trace_words,
                           uint8_t* argflags, uint32_t flags, void* stream,
                           pe_error* err);

/* infer_rest (REF propagate.cc:484-544, the InferRest action SPEC:522,531)
 * applied to the state reached by `prefix` (host buffers): writes
 * prefix + [INFER_REST marker] + the inferred TILE actions
 * (PE_ACT_FLAG_INFERRED) to `out`.  Each inference round evaluates all
 * (argument x dim x auto axis) trials as one GPU batch. */
pe_status pe_infer_rest(pe_engine* e, const pe_action* prefix, uint32_t n_prefix,
                        pe_action* out, uint32_t cap, uint32_t* n_out,
                        pe_error* err);

/* Leaf-parallel MCTS rollouts (SPEC mcts_search: "uniform-random rollout to
 * terminal"): candidate c first applies its prefix, records the legal
 * TileValue ordinals of that state in legal_out (bitmask of
 * pe_engine_legal_words() uint64 words, may be NULL), then samples actions
 * with the rollout policy (uniform, Stop weight 2 after the first decision,
 * at most max_decisions) from a splitmix64 stream seeded with seeds[c], and
 * scores the terminal state.  acts_out receives the candidate's DECISIONS --
 * the prefix's and the sampled ones; an InferRest decision as its unexpanded
 * marker, its inferred tiles omitted, so replaying the row re-derives them
 * (row stride max_decisions per candidate; entries past a candidate's
 * n_acts_out are unspecified), n_acts_out the count.  With infer_rest_action
 * (or an unexpanded InferRest in a host prefix) a candidate that reaches an
 * InferRest decision pauses; all paused candidates are expanded together
 * (each inference round's trials in one batched evaluation) and resume with
 * their RNG streams advanced by the draws they consumed.  A launch runs 32
 * candidates per warp when it needs every resident lane, fewer otherwise,
 * and one candidate per warp warp-cooperatively. */
pe_status pe_rollout_batch(pe_engine* e, const pe_action* prefix,
                           const uint32_t* prefix_off, const uint64_t* seeds,
                           uint32_t n_cand, pe_action* acts_out,
                           uint32_t* n_acts_out, pe_result* out,
                           uint64_t* legal_out, uint32_t flags, void* stream,
                           pe_error* err);

/* Number of TileValue ordinals: worklist entries x PE_MAX_RANK x auto axes
 * (ordinal = (entry*PE_MAX_RANK + dim)*n_auto + auto-axis rank). */
uint32_t pe_engine_num_ordinals(const pe_engine* e);
uint32_t pe_engine_legal_words(const pe_engine* e);
/* decode an ordinal into an action */
pe_status pe_engine_ordinal_action(const pe_engine* e, uint32_t ordinal,
                                   pe_action* out);
/* replicated plan's peak liveness (reward baseline) */
int64_t pe_engine_baseline_bytes(const pe_engine* e);
/* bytes of the per-candidate arena, and candidate slots per launch */
int64_t pe_engine_arena_bytes(const pe_engine* e);
uint32_t pe_engine_slots(const pe_engine* e);
/* capacities of the tight arena: value slots, loops, front stack, SPMD
 * ops, operand references */
void pe_engine_arena_caps(const pe_engine* e, int32_t* caps5);
/* Measurement: with timing on, every main rollout launch is bracketed by a
 * pair of CUDA events on its stream; pe_engine_kernel_times waits for them,
 * writes the durations (ms) of the launches since the last call and returns
 * their number. */
void pe_engine_set_kernel_timing(pe_engine* e, int32_t on);
uint32_t pe_engine_kernel_times(pe_engine* e, float* ms, uint32_t cap);
/* bytes of the compiled graph image resident in HBM */
int64_t pe_engine_graph_bytes(const pe_engine* e);
/* kernel launches issued by this engine since creation */
uint64_t pe_engine_launch_count(const pe_engine* e);
/* Prefix-trie scheduling: a batch of root rollouts (every
 * prefix empty; in device mode pass prefix = NULL) of at least 8192
 * candidates is evaluated in an order that groups candidates by their first
 * decisions, predicted from the seeds through a trie of legal sets after
 * short decision prefixes (depth 3).  The trie is cached by the engine and
 * grows by one level per call.  Results are unaffected (each candidate is
 * independent; outputs stay in candidate order).  Env PE_SCHED_DEPTH (0 =
 * off) and PE_SCHED_MIN_BATCH override at engine creation.  Returns the
 * number of trie nodes (prefix states probed). */
int64_t pe_engine_sched_nodes(const pe_engine* e);
/* Prefix-state reuse (opt-in): with a snapshot budget > 0
 * (GiB of HBM), the probe that adds a scheduling-trie node also saves the
 * propagated state after the node's decision prefix, and a scheduled root
 * rollout starts from its node's saved state instead of replaying those
 * decisions.  Results are identical; the saved states are computed once and
 * shared by every later call, so this trades per-candidate propagation for
 * state kept across calls -- off by default (budget 0), and bench.py's
 * `value` is measured without it.  Set before the first scheduled call
 * (also env PE_SCHED_SNAP_GB at engine creation). */
pe_status pe_engine_set_state_reuse(pe_engine* e, double budget_gb);

/* Prefix-state cache (incremental leaf evaluation): with a
 * budget > 0 (GiB of HBM), host-mode pe_rollout_batch calls save the
 * propagated state after each candidate's (non-empty, TILE / TILE_GROUP
 * only) prefix, and a later candidate whose prefix extends a cached one
 * starts from that state instead of replaying it -- an MCTS leaf is its
 * parent's state plus one action.  Least-recently-used slots are reused.
 * Results are identical with or without it.  Not used with stuck
 * resurfacing or InferRest actions.  pe_search turns it on (4 GiB) when
 * unset.  Set before the first call that would use it. */
pe_status pe_engine_set_prefix_cache(pe_engine* e, double budget_gb);
/* lookups that started from a cached state, states saved, live entries */
void pe_engine_prefix_cache_stats(const pe_engine* e, uint64_t* hits, uint64_t* saved,
                                  int64_t* entries);

/* ---- state handles (§8(b) pe_state): a propagated partitioning state ----
 * pe_state_create evaluates `acts` (TILE / TILE_GROUP decisions from the
 * untiled graph: apply_tile_action + propagate each, REF rewrite.cc:61,
 * propagate.cc:459) and keeps the propagated state on the device.
 * PE_ERR_ILLEGAL / PE_ERR_INTERNAL when the sequence does not evaluate. */
typedef struct pe_state pe_state;
pe_status pe_state_create(pe_engine* e, const pe_action* acts, uint32_t n, pe_state** out,
                          pe_error* err);
void pe_state_destroy(pe_state* s);
uint32_t pe_state_num_decisions(const pe_state* s);
/* the state's own evaluation (lower_to_spmd + collective_stats + cost) */
pe_status pe_state_result(const pe_state* s, pe_result* out);
/* Per-argument ShardingSpec of the lowered program's arguments and of the
 * returned value as spec words (trace layout above; REF spmd.cc:370-391,
 * mesh.h ShardingSpec), and the stuck list of the last propagate as
 * (op index, reason) pairs (REF propagate.h:28-38).  arg_specs: A words;
 * stuck: 2 * stuck_cap words; any may be NULL. */
pe_status pe_state_specs(const pe_state* s, uint32_t* arg_specs, uint32_t* result_spec,
                         int32_t* stuck, uint32_t stuck_cap, uint32_t* n_stuck, pe_error* err);
/* Incremental evaluation (host buffers): candidate c = parents[c] (NULL =
 * the untiled graph) + acts[seq_off[c] .. seq_off[c+1]) (TILE / TILE_GROUP),
 * each action applied + propagated from the parent's saved state, then
 * lowered and scored: the same result as pe_eval_batch of the parent's
 * decisions followed by the candidate's actions (fail_step indexes that
 * concatenation). */
pe_status pe_eval_from_states(pe_engine* e, const pe_state* const* parents, const pe_action* acts,
                              const uint32_t* seq_off, uint32_t n, pe_result* out, void* stream,
                              pe_error* err);

/* ---- search (SPEC search module: mcts_search / emit_plan) ---- */
#define PE_PLAN_MAX_ACTIONS 64

typedef struct pe_plan {
  pe_action actions[PE_PLAN_MAX_ACTIONS]; /* best terminal action sequence */
  uint32_t n_actions;
  uint32_t episodes;         /* episodes run on this rank                    */
  uint32_t found_at_episode; /* episode (on the winning rank) that found it  */
  uint32_t winner_rank;
  uint64_t seed;
  pe_result result;          /* evaluation of the best plan                  */
} pe_plan;

/* Root-parallel merge hook: replace `values[0..n)` with their element-wise
 * SUM (op 0) or MAX (op 1) over all ranks (an NCCL / gloo all_reduce).
 * Returns 0 on success.  NULL = single rank. */
typedef int (*pe_merge_fn)(void* user, int64_t* values, uint32_t n, int32_t op);

/* Evaluator hook with pe_rollout_batch semantics on host buffers. */
typedef int (*pe_rollout_fn)(void* user, const pe_action* prefix,
                             const uint32_t* prefix_off, const uint64_t* seeds,
                             uint32_t n, pe_action* acts_out, uint32_t* n_acts_out,
                             pe_result* out, uint64_t* legal_out);

typedef struct pe_mcts_params {
  uint32_t n_ordinals;    /* TileValue ordinals; Stop is ordinal n_ordinals  */
  uint32_t max_decisions; /* SPEC default 32                                 */
  uint32_t episodes;      /* budget on this rank                             */
  uint32_t leaf_batch;    /* leaves selected (virtual loss) per evaluation   */
  uint32_t merge_every;   /* episodes between root-statistic merges (0: never) */
  uint32_t rank;
  uint64_t seed;
  double uct_c;           /* SPEC default 1.414                              */
} pe_mcts_params;

/* mcts_search (SPEC search module): UCT selection (ties -> lowest ordinal),
 * lowest-ordinal expansion, uniform rollouts, backpropagation of the reward
 * as 2^-32 fixed point, best terminal plan.  Deterministic for a given
 * (params, evaluator).  `ordinal_actions[k]` decodes ordinal k. */
pe_status pe_mcts_run(const pe_mcts_params* p, pe_rollout_fn eval, void* eval_user,
                      pe_merge_fn merge, void* merge_user,
                      const pe_action* ordinal_actions, pe_plan* out, pe_error* err);

/* mcts_search on this engine: cfg->leaf_batch rollouts per GPU launch. */
pe_status pe_search(pe_engine* e, const pe_search_config* cfg, uint32_t merge_every,
                    uint32_t rank, pe_merge_fn merge, void* merge_user, pe_plan* out,
                    pe_error* err);

/* ---- root-parallel search over NCCL (SURVEY.md §8(b),(e)) ----
 * One tree per GPU (seed + rank, rank = the communicator's); every
 * merge_every episodes the root children's (N, W) int64 statistics are
 * all-reduced (ncclAllReduce SUM on a device buffer), and at the end MAX
 * reductions pick the best plan (ties -> lowest rank); every rank returns it.
 * `comm` is an ncclComm_t (void* here so this header does not need nccl.h);
 * NCCL is resolved at run time from the process (libnccl.so.2). */
pe_status pe_search_multi(pe_engine* e, const pe_search_config* cfg, uint32_t merge_every,
                          void* comm, pe_plan* out, pe_error* err);
/* Helpers for callers without their own NCCL binding: ncclGetUniqueId (128
 * bytes, to broadcast out of band), ncclCommInitRank on `device`, and
 * ncclCommDestroy. */
pe_status pe_nccl_unique_id(uint8_t* out128, pe_error* err);
pe_status pe_nccl_comm_create(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device,
                              void** comm, pe_error* err);
void pe_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* PE_H_ */
