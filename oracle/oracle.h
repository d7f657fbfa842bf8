/*
 * oracle.h -- the CPU oracle of HyP-DESPOT's batched leaf expansion.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no source, header, table or constant generator with the CUDA
 * path (paper_1802_06215_b200/csrc); it is written from PAPER.md and the
 * model cards in DESIGN.md.
 *
 * What it computes is DESPOT's serial leaf initialisation (PAPER.md
 * §III-A "Leaf Node Initialization") carried out as the
 * MC_simulation tasks update / expansion / upper bound / roll-out
 * (§III-D2), i.e. Eqs. 9, 11, 12 and the grouping of
 * scenarios by observation behind Eq. 10, plus the one-level
 * Bellman backup of Eq. 4.  Values are accumulated in fp64.
 */
#ifndef HYP_DESPOT_ORACLE_H
#define HYP_DESPOT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_model oracle_model;

typedef struct {
  uint32_t num_actions;   /* |A|                                      */
  uint32_t state_words;   /* u32 words per state                      */
  uint32_t obs_words;     /* u32 words per observation key            */
  uint32_t obs_slots;     /* dense key range incl. TERMINAL, 0=sparse */
  uint32_t max_depth;     /* D (absolute depth, reading C3)           */
  uint32_t elements;      /* factored elements per step   */
  double gamma;           /* discount                                 */
  double tail;            /* l(s) heuristic after depth D     */
} oracle_model_info;

/* Philox4x32-10 (Salmon et al. 2011), the counter-based stream behind the
 * scenario random numbers phi_1, phi_2, .... */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* event threshold T(p) = floor(p * 2^32); an event of probability p fires
 * iff (uint64)u < T(p) (reading C14). */
uint64_t oracle_threshold(double p);

int  oracle_model_load(const char* kind, const char* params, oracle_model** out);
void oracle_model_free(oracle_model* m);
int  oracle_model_info_get(const oracle_model* m, oracle_model_info* out);
const char* oracle_last_error(void);

/* One deterministic step g(s, a, phi_t) (Eq. 9): t is the depth
 * reached by the step (the step from depth t-1 to t draws phi_t). */
int oracle_step(const oracle_model* m, const uint32_t* s, int32_t a, uint32_t id,
                uint32_t t, uint64_t seed, uint32_t* s_out, uint32_t* z_out,
                float* r_out, int32_t* term_out);
/* per-scenario upper bound u(phi) of Eq. 11 (0 for terminal states) */
double oracle_upper(const oracle_model* m, const uint32_t* s);
/* default-policy roll-out of Eq. 12 from state s at absolute depth `depth`,
 * whose last observation is z (NULL: the model's initial observation). */
int oracle_rollout(const oracle_model* m, const uint32_t* s, const uint32_t* z,
                   uint32_t id, uint32_t depth, uint64_t seed, double* ret,
                   uint32_t* len, uint64_t* trace_hash, uint64_t* steps);
/* default policy decision (tests) */
int32_t oracle_default_action(const oracle_model* m, const uint32_t* s, const uint32_t* z,
                              uint64_t memory, uint32_t t);

/* Nodes: a belief is K weighted scenarios with their random streams. */
int64_t oracle_belief_load(oracle_model* m, const uint32_t* states_soa, const float* weights,
                           uint32_t K, uint64_t seed);
int  oracle_node_size(const oracle_model* m, int64_t node, uint32_t* n, uint32_t* depth);
/* copies ids[n], weights[n], states_soa[state_words][n] */
int  oracle_node_read(const oracle_model* m, int64_t node, uint32_t* ids, float* w,
                      uint32_t* states_soa);
int  oracle_node_release(oracle_model* m, int64_t node);

typedef struct {
  int64_t  parent;   /* expanded node (or the leaf itself when action == -1)  */
  int32_t  action;   /* last action of the history, -1: no update step        */
  uint32_t child;    /* child ordinal under (parent, action)                   */
  uint32_t depth;    /* depth Delta of the leaf                                */
  uint32_t pad;
} oracle_leaf;

typedef struct {
  /* per leaf [L] */
  int64_t*  node;          /* new node holding the leaf's scenarios          */
  uint32_t* n_scen;        /* |Phi_l|                                         */
  double*   weight;        /* W_l = sum of weights                            */
  /* per (leaf, action) [L*A] */
  double*   act_reward;    /* r(b,a) = sum w r / W                            */
  double*   act_upper;     /* u(b,a) = sum w (r + gamma u) / W   (Eq. 4)      */
  double*   act_lower;     /* l(b,a) = sum w (r + gamma lambda) / W (Eq. 4)   */
  uint32_t* child_begin;   /* [L*A+1] CSR                                     */
  uint32_t  child_capacity;
  /* per child [C] */
  uint32_t* child_count;
  uint32_t* child_first;   /* smallest global scenario id in the child        */
  double*   child_weight;
  double*   child_upper;   /* Eq. 11 */
  double*   child_lower;   /* Eq. 12 */
  uint32_t* child_obs;     /* [C*obs_words] observation key                   */
  /* per scenario [S], ordered (leaf, action, position) -- nullable */
  uint64_t  scen_capacity;
  uint32_t* scen_obs;      /* [S*obs_words]                                   */
  float*    scen_reward;
  double*   scen_upper;
  double*   scen_lower;
  uint32_t* scen_len;      /* roll-out length                                 */
  uint64_t* scen_hash;     /* FNV-1a of the roll-out action sequence          */
  uint32_t* scen_child;    /* child ordinal                                   */
  uint32_t* scen_states;   /* [S*state_words] s' after the expansion step     */
  uint64_t  scenario_steps;/* out: number of steps on non-terminal states     */
} oracle_expansion;

/* ORACLE_EXPAND: leaves are processed in order; actions with
 * action_mask[a] == 0 are skipped (their outputs are zero, no children). */
int oracle_expand_batch(oracle_model* m, const oracle_leaf* leaves, uint32_t L,
                        const uint8_t* action_mask, oracle_expansion* out);

/* Eqs. 11-12 at a node's own depth (root initialisation). */
int oracle_rollout_bounds(const oracle_model* m, int64_t node, double* upper_mean,
                          double* lower_mean, double* per_scen_upper, double* per_scen_lower);

/* Exact optimal value V*_D of the D-truncated DESPOT on the node's scenarios
 * (brute force over the whole tree; tiny instances only). */
int oracle_brute_force(const oracle_model* m, int64_t node, double* value);
/* Q*_D(b, a) for every action (array of |A|) */
int oracle_brute_force_q(const oracle_model* m, int64_t node, double* q);

#ifdef __cplusplus
}
#endif
#endif
