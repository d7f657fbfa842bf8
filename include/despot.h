/*
 * despot.h -- C ABI of libdespot, the B200 (sm_100a) batched leaf expansion
 * of HyP-DESPOT (Cai, Luo, Hsu, Lee, "HyP-DESPOT: A Hybrid Parallel Algorithm
 * for Online Planning under Uncertainty", arXiv 1802.06215).
 *
 * Citations: P:n = line n of PAPER.md (the paper's LaTeX source), S:n = line n
 * of SPEC.md; R<n> = reading n in DESIGN.md §2 (where the paper is silent).
 *
 * The hot path: for every leaf of a batch, the MC_simulation
 * tasks of §III-D2 -- update (replay the last action and keep the
 * parent's scenarios that reach this leaf), expansion over all actions
 * and scenarios (Eq. 9), per-child upper bounds (Eq. 11),
 * default-policy roll-outs to depth D (Eq. 12), the grouping of
 * scenarios into child nodes by observation (Eq. 10) and the
 * one-level Bellman values of Eq. 4.  Many leaves go into one
 * launch (node-level parallelism).
 *
 * Conventions
 *  - Every call returns an int status; 0 = DESPOT_OK.  No C++ exception
 *    crosses the ABI.  On error, despot_last_error() returns a message that
 *    is thread-local and valid until the calling thread's next call.
 *  - A model is immutable after load and may be used from many host threads
 *    at once; each call uses its own device scratch.
 *  - Node arenas live in device memory, are owned by the library and are
 *    immutable once created (their child-key table is written when the node
 *    is expanded), until despot_node_release().
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls that
 *    return outputs are synchronous with respect to those outputs.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one fails with DESPOT_ECUDA.
 */
#ifndef HYP_DESPOT_DESPOT_H
#define HYP_DESPOT_DESPOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DESPOT_ABI_VERSION 2

enum despot_status {
  DESPOT_OK = 0,
  DESPOT_EINVAL = -1,    /* malformed arguments: unknown kind/params, empty or zero-weight
                            belief, leaf depth >= D, unknown child ordinal (its
                            scenario set would be empty), unexpanded parent            */
  DESPOT_EMODEL = -2,    /* step contract violation: action outside [-1, |A|)  */
  DESPOT_ENOMEM = -3,    /* device allocation failed                                  */
  DESPOT_ECAPACITY = -4, /* caller's child_capacity / scen_capacity too small; the
                            needed sizes are in num_children / the n_scen outputs    */
  DESPOT_ECUDA = -5,     /* CUDA error (no device, launch failure, ...)               */
  DESPOT_ENCCL = -6,     /* NCCL unavailable or a collective of the library's
                            communicator failed (the model then enters ESHUTDOWN)     */
  DESPOT_ESHUTDOWN = -7, /* the model entered a failed state after a CUDA error       */
  DESPOT_EHASH = -8      /* two different sparse observation keys shared a 64-bit
                            hash inside one (leaf, action): grouping refused          */
};

/* Thread-local message of the last failing call of this thread. */
const char* despot_last_error(void);
int despot_abi_version(void);

/* ------------------------------------------------------------------------ */
/* Models (DESIGN.md §3 model cards)                   */
/* ------------------------------------------------------------------------ */
typedef struct despot_model despot_model; /* opaque */
typedef uint64_t despot_node;             /* opaque handle of a device node arena */
typedef struct despot_comm despot_comm;   /* opaque: an NCCL communicator the library owns */

typedef struct {
  int device;     /* CUDA device ordinal the model and its nodes live on            */
  int rank;       /* scenario shard of this process: it keeps global ids            */
  int world;      /*   with id % world == rank; world <= 1: no shard */
  uint32_t flags; /* DESPOT_MF_* below                                              */
  despot_comm* comm; /* NULL, or a communicator of `world` ranks (despot_comm_init)
                        whose rank is `rank`: despot_expand_batch then runs the whole
                        sharded batch, its exchange included, in one call            */
  /* Device allocator hooks (both or neither; e.g. torch's caching allocator):
   * node arenas, batch scratch and staging come from dev_alloc(bytes, stream,
   * alloc_ctx) and go back through dev_free(ptr, stream, alloc_ctx), ordered on
   * the call's stream (a prepared batch's persistent scratch excepted).  NULL:
   * cudaMallocAsync / cudaFreeAsync.  dev_alloc returns NULL on failure
   * (ENOMEM).  The hooks must stay valid until despot_model_free returns.   */
  void* (*dev_alloc)(size_t bytes, void* stream, void* ctx);
  void (*dev_free)(void* ptr, void* stream, void* ctx);
  void* alloc_ctx;
} despot_opts;

/* Driving model kernel variant.  Default: chosen per batch -- the factored
 * warp-per-scenario kernel (lanes = pedestrians and the car, within-step
 * parallelism) when the batch has too few (leaf, action, scenario)
 * items to fill the GPU with one thread each, else thread-per-scenario. */
#define DESPOT_MF_UNFACTORED 1u /* always thread per scenario */
#define DESPOT_MF_FACTORED 2u   /* always warp per scenario   */
#define DESPOT_MF_GROUPED 4u    /* a lane group per scenario: lane q owns Philox block q
                                   (the car's word and pedestrians 4q-1 .. 4q+2),
                                   32 / ceil((P+1)/4) scenarios per warp */
#define DESPOT_MF_PAIRED 16u    /* a lane pair per scenario: each lane owns half of a
                                   step's Philox blocks (20 pedestrians: 3 blocks,
                                   11 / 9 pedestrians), 16 scenarios per warp */
#define DESPOT_MF_EXCHANGE 8u   /* with a communicator: run the exchange (pack,
                                   collectives, unpack) even when world == 1 -- the
                                   one-GPU test of the sharded data path */

typedef struct {
  uint32_t num_actions; /* |A|                                                     */
  uint32_t state_words; /* u32 words per scenario state (SoA rows of a node)       */
  uint32_t obs_words;   /* u32 words per observation key                           */
  uint32_t obs_slots;   /* dense observation range incl. TERMINAL; 0 = sparse keys */
  uint32_t max_depth;   /* D, an absolute depth (R3)                                */
  uint32_t elements;    /* factored elements per step                   */
  double gamma;         /* discount                                                 */
  double tail;          /* heuristic l(s) added at depth D (R6)              */
} despot_model_info;

/* kind: "tiger" | "rocksample" | "nav" | "car".  params: "key=value ..." as in
 * the model cards (e.g. "n=15 robots=2 rocks=x:y,... starts=x:y,x:y D=20
 * gamma=0.95").  opts may be NULL (device 0, no sharding).
 * Errors: EINVAL (unknown kind / bad params), ECUDA, ENOMEM. */
int despot_model_load(const char* kind, const char* params, const despot_opts* opts,
                      despot_model** out);
int despot_model_info_get(const despot_model* model, despot_model_info* out);
/* Frees the model and every node still alive.  The model must not be in use. */
int despot_model_free(despot_model* model);

/* ------------------------------------------------------------------------ */
/* Beliefs and nodes                                                        */
/* ------------------------------------------------------------------------ */
/* A belief is K weighted scenarios with their random streams:
 * states_soa [state_words][K] u32 (host), weights [K] f32 > 0 (host), global
 * scenario id = position, stream_seed = the Philox key sigma of phi_t (R13).
 * With world > 1 only ids with id % world == rank are kept on this device.
 * The root has depth 0.  Errors: EINVAL (K == 0, weight <= 0; driving: a car
 * or pedestrian coordinate not finite or beyond |4096| m, outside the model's
 * int16 observation bins, R21), ENOMEM, ECUDA. */
int despot_belief_load(despot_model* model, const uint32_t* states_soa, const float* weights,
                       uint32_t K, uint64_t stream_seed, void* stream, despot_node* root_out);
/* n = scenarios of the node on this device (after the call that created it
 * has returned), depth = Delta of the node. */
int despot_node_info(despot_model* model, despot_node node, uint32_t* n, uint32_t* depth);
/* Copies the node's ids [n], weights [n] and states [state_words][n] to host
 * buffers (any may be NULL).  Synchronous. */
int despot_node_read(despot_model* model, despot_node node, uint32_t* ids, float* weights,
                     uint32_t* states_soa, void* stream);
int despot_node_release(despot_model* model, despot_node node);
/* despot_node_release of n nodes (host array), in order, in one call.  Stops
 * at the first unknown node (EINVAL); the ones before it are released. */
int despot_node_release_many(despot_model* model, const despot_node* nodes, uint32_t n);

/* ------------------------------------------------------------------------ */
/* Batched leaf expansion (the hot path)                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  despot_node parent; /* an expanded node, or the leaf itself when action == -1     */
  int32_t action;     /* last action of the leaf's history; -1: no update step      */
  uint32_t child;     /* child ordinal under (parent, action): first-occurrence
                         order of that expansion (R8)                                */
  uint32_t depth;     /* Delta of the leaf (parent depth + 1, or the node's depth)  */
  uint32_t pad;
} despot_leaf;

/* despot_expansion.flags */
#define DESPOT_X_DEVICE_OUTPUTS 1u  /* all array outputs except `node` are device
                                       pointers (no D2H copies inside the call)     */
#define DESPOT_X_RECORD_SCENARIO 2u /* fill the per-scenario scen_* arrays         */
#define DESPOT_X_TIMING 4u          /* fill phase_ms with CUDA-event times of the
                                       phases, recorded on the call's stream       */
#define DESPOT_X_TIMING_K2 8u       /* only phase_ms[1] (K2), two events: the cheap
                                       form for timing loops (8 events cost ~30 us
                                       of host time per call)                     */
#define DESPOT_X_RESIDENT 32u       /* despot_batch_prepare only (single GPU, no
                                       RECORD), for a batch that finalizes in K2 (few
                                       slots, small L*A) or in the one-kernel wide
                                       finalize (> 32 slots): the scratch's zero
                                       state is set up once at prepare and restored
                                       by the kernels at the end of every run (K2's
                                       last CTA, or each wide-finalize CTA for its
                                       (leaf, action) and the last one for the
                                       counters), which also publishes the status to
                                       mapped host memory: no memset or status D2H
                                       per run.  When every leaf is a node itself
                                       (roots) the leaf table is uploaded once too
                                       and the graph is K2 alone.  A run after an
                                       error sets up again.  Ignored when the batch
                                       does not qualify.                           */
#define DESPOT_X_INDEX_LISTS 16u    /* the paper's update form ("the leaf ...
                                       only contains a set of indexes"): leaf l with
                                       action >= 0 takes the parent positions
                                       index[index_begin[l] .. index_begin[l+1]-1]
                                       (ascending) instead of replay + filter; the
                                       update still replays the action on them and
                                       fails with EINVAL if a position's observation
                                       is not the leaf's key (validation mode; single
                                       call, world == 1)                               */

/* Caller-owned outputs.  Sizes: L leaves, A = |A|, C = child_capacity,
 * S = scen_capacity.  Children of (l, a) are child_begin[l*A+a] ..
 * child_begin[l*A+a+1]-1, in first-occurrence order (R8).  Host outputs that
 * are all page-locked (cudaHostAlloc / cudaHostRegister) are written in place
 * by the kernels (dense keys, <= 4 MB at capacity) or copied into directly;
 * either way they are valid when the call returns. */
typedef struct {
  uint32_t flags;
  despot_node* node;     /* [L] host: new node holding leaf l's scenarios (for
                            action == -1 leaves: the parent itself)                   */
  uint32_t* n_scen;      /* [L] |Phi_l| (all ranks)                                   */
  float* weight;         /* [L] W_l = sum of the leaf's scenario weights              */
  float* act_reward;     /* [L*A] mean step reward  sum_i w_i r_i / W_l  (Eq. 4)      */
  float* act_upper;      /* [L*A] u(b,a) = sum_i w_i (r_i + gamma u_i) / W_l (Eq. 4)  */
  float* act_lower;      /* [L*A] l(b,a) = sum_i w_i (r_i + gamma lambda_i) / W_l     */
  uint32_t* child_begin; /* [L*A+1] CSR offsets                                        */
  uint32_t child_capacity;
  uint32_t* child_count; /* [C] N_c = |Phi_b'|                                         */
  uint32_t* child_first; /* [C] smallest global scenario id of the child               */
  float* child_weight;   /* [C] W_c                                                    */
  float* child_upper;    /* [C] u(b') of Eq. 11                                        */
  float* child_lower;    /* [C] l(b') of Eq. 12                                        */
  uint32_t* child_obs;   /* [C*obs_words] the child's observation key z                */
  /* per scenario, only with DESPOT_X_RECORD_SCENARIO (world == 1), ordered
   * (leaf, action, position in the leaf); S >= A * sum_l n_scen[l]:          */
  uint64_t scen_capacity;
  uint32_t* scen_obs;     /* [S*obs_words] z after the expansion step               */
  float* scen_reward;     /* [S] r                                                   */
  float* scen_upper;      /* [S] u(s') (0 if terminal)                               */
  float* scen_lower;      /* [S] roll-out return lambda (0 if terminal)              */
  uint32_t* scen_len;     /* [S] roll-out length                                     */
  uint64_t* scen_hash;    /* [S] FNV-1a-64 of the roll-out's joint actions           */
  uint32_t* scen_states;  /* [S*state_words] s' after the expansion step             */
  /* host-side results */
  uint64_t scenario_steps; /* out: steps g(s,a,phi) on non-terminal states (this rank) */
  uint32_t num_children;   /* out: total children C used                              */
  uint32_t launches;       /* out: kernels this call launched (begin + end)          */
  /* out with DESPOT_X_TIMING: [0] update (K1), [1] expansion + roll-outs +
   * grouping (K2), [2] child order / CSR / outputs (K3a-c), [3] whole call
   * from the first enqueued operation to the last (device time, ms)          */
  float phase_ms[4];
  uint64_t h2d_bytes;      /* out: bytes this call moved host -> device / device ->  */
  uint64_t d2h_bytes;      /*      host (leaf table -- copied, or read by K1 from the
                              page-locked staging --, status, results -- copied, or
                              written in place --; begin + end)                      */
  /* out, sharded batches run through the model's communicator: */
  float exchange_ms;       /* K4: CUDA-event time of the exchange (collectives and the
                              pack / unpack kernels between them; with DESPOT_X_TIMING) */
  uint32_t exchange_rounds;/* collective rounds issued (a capacity retry adds one)   */
  uint64_t exchange_bytes; /* bytes this rank contributed to the collectives         */
  /* with DESPOT_X_RECORD_SCENARIO: [S] each scenario's child ordinal under its
   * (leaf, action) -- the per-scenario observations' children the paper returns
   * to the host, from which host index lists are built               */
  uint32_t* scen_child;
  /* in, with DESPOT_X_INDEX_LISTS (host arrays): [L+1] offsets, and the parent
   * positions of every leaf (positions in the parent's ascending-id list)     */
  const uint32_t* index_begin;
  const uint32_t* index;
} despot_expansion;

/* Output sizes of a batch before calling it (host only, no device work):
 * *child_capacity = an upper bound of the children C (sum over leaves of
 * A * min(|Phi_parent|, obs_slots); sharded: (local n + 1) * world per parent,
 * which a filtered node may exceed -- the call then fails with ECAPACITY and
 * reports num_children), *scen_capacity = A * sum of the parents' local
 * scenario counts (>= what DESPOT_X_RECORD_SCENARIO writes), *host_bytes =
 * the bytes of every despot_expansion array at those sizes for `flags`
 * (node, n_scen, weight, act_*, child_begin, the child arrays and, with
 * RECORD, the scen_* arrays).  Any output may be NULL.  Errors: EINVAL
 * (unknown node), ECAPACITY (the child bound does not fit in 32 bits). */
int despot_expand_batch_bytes(despot_model* model, const despot_leaf* leaves, uint32_t L, uint32_t flags,
                              uint32_t* child_capacity, uint64_t* scen_capacity, uint64_t* host_bytes);

/* One batch: update (world-local) -> expansion + bounds + roll-outs + grouping
 * -> [exchange] -> child ordering, CSR and outputs.  `leaves` is a host array
 * of L <= 4096 descriptors.  Synchronous.  With world > 1 the model needs a
 * communicator (despot_opts.comm): every rank calls with identical leaves, in
 * the same order, from one host thread per rank (SPMD), and the exchange runs
 * inside the call on `stream` (dense keys -- an all-reduce of
 * the slots any rank used, compacted; sparse keys -- a SUM of the per-action
 * partials and an all-gather of the ranks' child records); without one use
 * the begin/exchange/end form.  Errors: EMODEL (action out of range), EINVAL
 * (see enum), ECAPACITY, EHASH, ENOMEM, ECUDA, ENCCL.  On error outputs are
 * unspecified and nodes created by the call are freed. */
int despot_expand_batch(despot_model* model, const despot_leaf* leaves, uint32_t L,
                        despot_expansion* out, void* stream);

/* Prepared batches (SURVEY §7 hard part 6: launch overhead of small, repeated
 * batches).  despot_batch_prepare validates the leaves, allocates the batch's
 * scratch and staging once, binds `out` (its flags, capacities and array
 * pointers are fixed from here on) and captures the batch's device work --
 * setup copies, K1, K2, K3 and the result copies -- into one CUDA graph.
 * despot_batch_run then allocates the new nodes' arenas, patches the leaf
 * table and launches the graph: every step of the batch runs again, with the
 * host cost of one graph launch.  Each run returns new nodes exactly as
 * despot_expand_batch does.  Single GPU, no RECORD; a run fails with EINVAL if
 * a parent was released.  Runs of one prepared batch must not overlap. */
typedef struct despot_prepared despot_prepared;
int despot_batch_prepare(despot_model* model, const despot_leaf* leaves, uint32_t L, despot_expansion* out,
                         despot_prepared** prepared_out);
int despot_batch_run(despot_prepared* prepared, despot_expansion* out, void* stream);
int despot_batch_prepared_free(despot_prepared* prepared);

/* Multi-GPU scenario sharding driven by the caller, the form
 * for a caller-supplied transport (despot_expand_batch with a communicator is
 * the library-owned form): every rank calls with identical leaves; between
 * begin and end the caller runs the collectives each exchange round names,
 * in place, over the ranks (e.g. NCCL or gloo, ordered after `stream`'s
 * work): SUM over `sums`, MIN over `mins`, and an all-gather over `gather`
 * (world blocks of gather_bytes; this rank's block, at rank * gather_bytes,
 * is filled).  One round for every model: dense keys SUM the exact int64
 * partial block and MIN the first ids; sparse keys (driving) SUM the
 * per-action partials and all-gather the ranks' child records (blocks sized
 * on the host from the leaves alone -- no read-back), merged by exact key in
 * `end`.  `end` then produces identical outputs on every rank, equal to
 * world == 1 bit for bit: the sums are exact int64 fixed-point partials, so
 * nothing depends on the reduction order.  Null pointers / zero sizes: no
 * such collective.  `maxs` is unused since ABI 2 (NULL). */
typedef struct despot_batch despot_batch;
typedef struct {
  int64_t* sums;   /* device [n_sums]  all-reduce SUM (int64)  */
  uint64_t n_sums;
  int32_t* mins;   /* device [n_mins]  all-reduce MIN (int32)  */
  uint64_t n_mins;
  int64_t* maxs;   /* unused (NULL): the ABI 1 MAX round is gone          */
  uint64_t n_maxs;
  void* gather;    /* device [world * gather_bytes]  all-gather (in place) */
  uint64_t gather_bytes;
  uint32_t round;  /* this round's index (0-based)                          */
  uint32_t more;   /* nonzero: call despot_batch_exchange again after this  */
} despot_exchange;
int despot_expand_begin(despot_model* model, const despot_leaf* leaves, uint32_t L,
                        uint32_t flags, void* stream, despot_batch** batch_out);
int despot_batch_exchange(despot_batch* batch, despot_exchange* out);
/* Completes (and frees) the batch; out->flags must equal begin's flags. */
int despot_expand_end(despot_batch* batch, despot_expansion* out, void* stream);
/* Abandons a begun batch (frees it and the nodes it created). */
int despot_batch_abort(despot_batch* batch);

/* Eqs. 11-12 at the node's own depth, e.g. to initialise the root's bounds
 * (R: SURVEY §3.4): weighted means over the node's scenarios of u(s) and of a
 * default-policy roll-out from depth Delta.  per_scen arrays [n] are optional
 * (host; this rank's scenarios).  A sharded model (world > 1) needs its
 * communicator: the means are then over every rank's scenarios (an all-reduce
 * of the exact fixed-point sums; SPMD).  Synchronous.  Errors: EINVAL (sharded
 * without a communicator), ECUDA, ENCCL. */
int despot_rollout_bounds(despot_model* model, despot_node node, float* upper_mean,
                          float* lower_mean, float* per_scen_upper, float* per_scen_lower,
                          void* stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU communicator (SURVEY §8(e) "Bootstrap"): rank 0 creates the NCCL
 * unique id, the caller broadcasts its 128 bytes to every rank over any
 * channel (e.g. a torch.distributed process group), and every rank creates
 * its communicator.  libnccl.so.2 is loaded at run time (the copy the process
 * already has, else $DESPOT_NCCL_LIB, else the loader's search path); a
 * communicator issues its collectives on the batch's stream.               */
/* ------------------------------------------------------------------------ */
/* id_out: 128 bytes.  Errors: ENCCL (no libnccl, or ncclGetUniqueId failed). */
int despot_comm_unique_id(void* id_out);
/* Collective over `world` ranks: every rank calls with the same id.
 * Errors: EINVAL, ECUDA, ENCCL. */
int despot_comm_init(const void* id, int rank, int world, int device, despot_comm** out);
/* The communicator must no longer be in use by any model. */
int despot_comm_destroy(despot_comm* comm);
/* rank / world / NCCL version of a communicator (any output may be NULL). */
int despot_comm_info(const despot_comm* comm, int* rank, int* world, int* nccl_version);

/* ------------------------------------------------------------------------ */
/* Host tree driver (the north star's "thin host driver
 * that coalesces many threads' leaves into one launch")                     */
/* ------------------------------------------------------------------------ */
/* Expansion backend: expands `L` leaves into host arrays of `out` (same
 * contract as despot_expand_batch with host outputs).  libdespot's GPU
 * backend is used by despot_plan; tests plug in the CPU oracle.  With one
 * worker it is called from one thread at a time; with several, two batcher
 * threads may call it concurrently (one waits for its expansion while the
 * other builds the previous batch's children), so the backend must be
 * thread-safe -- libdespot's is.  Returns a despot_status. */
typedef int (*despot_expand_fn)(void* ctx, const despot_leaf* leaves, uint32_t L, despot_expansion* out);
typedef int (*despot_release_fn)(void* ctx, despot_node node);

typedef struct {
  uint32_t num_actions, obs_words, obs_slots, max_depth; /* as despot_model_info       */
  double gamma;
  despot_node root;          /* backend handle of the root belief (depth root_depth) */
  uint32_t root_depth, root_scenarios;
  double root_weight;        /* W_b0                                                  */
  double root_upper, root_lower; /* initial bounds of the root (Eqs. 11-12)          */
  despot_expand_fn expand;
  despot_release_fn release; /* may be NULL                                           */
  void* ctx;
} despot_search_problem;

typedef struct {
  uint32_t workers;       /* CPU search threads                          */
  uint32_t max_batch;     /* leaves per expansion launch                             */
  uint32_t max_inflight;  /* trials a worker may have waiting for expansion          */
  uint32_t batch_wait_us; /* the batcher waits at most this long to fill a batch     */
  uint64_t max_trials;    /* 0 = no limit                                            */
  double time_budget_s;   /* anytime budget; <= 0 = no limit              */
  double xi;              /* WEU target factor (Eq. 6)                               */
  double c_a;             /* PO-UCT exploration scale (Eq. 7)                        */
  double c_o;             /* virtual-loss scale (Eq. 8)                              */
  double target_gap;      /* stop when u(b0) - l(b0) <= target_gap                   */
} despot_search_config;

typedef struct {
  int32_t action;         /* argmax_a l(b0, a), ties by the lowest index     */
  float root_upper, root_lower;
  uint64_t nodes;         /* belief nodes in the tree                                */
  uint64_t expanded;      /* nodes expanded (leaves initialised)                     */
  uint64_t trials;
  uint64_t batches;       /* expansion launches                                      */
  uint32_t max_depth;
  uint32_t pad;
  double seconds;
  uint64_t scenario_steps;
} despot_search_result;

/* One tree node for tests and dumps (pre-order: a node follows its parent). */
typedef struct {
  int32_t parent;         /* index in the dump, -1 for the root                      */
  int32_t action;         /* edge from the parent                                    */
  uint32_t child, depth, n_scen, visits, branch_visits; /* N(b), sum_a N(b, a)      */
  int32_t active;         /* virtual-loss markers still held (0 after a search)      */
  int32_t expanded;
  float weight, upper, lower, upper0, lower0;
} despot_search_node;

/* Anytime parallel DESPOT search from `problem->root`: workers descend with
 * the scenario-based PO-UCT action rule (Eq. 7) and the WEU observation rule
 * with virtual loss (Eqs. 6, 8), hand their leaves to a batcher that expands
 * up to max_batch leaves per backend call, and back up Eq. 4 along each path
 * (lower bounds floored at, upper bounds capped by the initial values).
 * dump (optional, dump_capacity nodes) receives the final tree.  Every node
 * the backend created is released before returning. */
int despot_search(const despot_search_problem* problem, const despot_search_config* config,
                  despot_search_result* result, despot_search_node* dump, uint32_t dump_capacity);

/* despot_search on libdespot's GPU backend: root bounds by
 * despot_rollout_bounds, expansions by despot_expand_batch on `stream`. */
int despot_plan(despot_model* model, despot_node root, const despot_search_config* config,
                despot_search_result* result, void* stream);

/* Raw scenario stream words, for tests of the generator: out[i] = word k of
 * scenario ids[i] at depth t (tag 0), R13.  Host arrays, synchronous. */
int despot_stream_words(despot_model* model, uint64_t stream_seed, const uint32_t* ids,
                        uint32_t n, uint32_t t, uint32_t k, uint32_t* out, void* stream);

/* K0, the measured Philox ceiling (SURVEY §8(d) "Ceilings"): a persistent
 * grid (256-thread CTAs, full occupancy) in which thread g of n_threads draws
 * the Philox4x32-10 blocks ctr = (g, t, 0, 0), t = 1 .. blocks, key = the seed
 * (the R13 addressing of the scenario streams, round keys as a kernel
 * parameter as in K2) and XOR-folds their words.  One warm-up launch, then
 * `reps` launches timed with CUDA events on `stream`: *out_ms = mean ms per
 * launch (n_threads * blocks blocks), *out_checksum = XOR of every word of
 * one launch (tests compare it with the oracle's generator).  Synchronous.
 * Errors: EINVAL (null output, zero sizes), ECUDA. */
int despot_philox_ceiling(despot_model* model, uint64_t stream_seed, uint32_t n_threads, uint32_t blocks,
                          uint32_t reps, void* stream, double* out_ms, uint32_t* out_checksum);

#ifdef __cplusplus
}
#endif
#endif
