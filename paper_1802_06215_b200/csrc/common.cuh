// common.cuh -- shared device-side definitions of libdespot (sm_100a).
//
// DevModel is the immutable, host-built description of one model (its
// parameters plus the lookup tables the kernels stage into shared memory).
// Nothing here is shared with oracle/: the CUDA path is an independent
// implementation of the model cards in DESIGN.md §3.
#pragma once
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hd {

constexpr int kGpowN = 256;          // gamma^k table, k < 256 (D <= 250)
constexpr int kRsMaxRocks = 31;
constexpr int kRsMaxN = 32;
constexpr int kRsMaxD2 = 2 * 31 * 31 + 1;
constexpr int kNavMaxN = 16;
constexpr int kNavMaxWords = 7;      // unknown-cell words (n <= 16 -> <= 208 cells)
constexpr int kCarMaxPeds = 31;
constexpr uint32_t kMaxLeaves = 4096;
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;

enum Kind : int32_t { kTiger = 1, kRockSample = 2, kNav = 3, kCar = 4 };

// Dynamic shared memory of every kernel that stages a model: the model's Sm
// struct at offset 0, then the model's variable-size tables
// (DevModel::sm_table_bytes, aligned to 16), then the kernel's own data.
extern __shared__ __align__(16) unsigned char hd_dyn_smem[];

// Programmatic dependent launch (the batch's kernel chain K1 -> K2 -> K3 is
// launched with cudaLaunchAttributeProgrammaticStreamSerialization): a kernel
// lets its successor's CTAs launch as soon as all of its own CTAs have started
// (pdl_trigger), and the successor waits for the predecessor's completion and
// memory (pdl_wait) before it touches anything but the model's constants, so
// launch latency and the successor's prologue (the model's shared-memory
// image) overlap the predecessor.  Both are no-ops on a plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct DevModel {
  int32_t kind;
  uint32_t sm_table_bytes;     // variable-size shared-memory tables after the model's Sm
  uint32_t A, SW, OW, slots, D, terminal_slot, elements;
  double gamma, tail;
  double fx, inv_fx;           // fixed-point scale of the exact reductions
  double gpow[kGpowN];         // gamma^k (host pow, double)
  // tiger
  uint64_t t_listen;
  // rocksample / MARS
  int32_t n, m, R, policy_east;
  int32_t base;                // 5 + m sub-actions per robot
  int8_t rx[32], ry[32];
  int8_t rock_at[kRsMaxN * kRsMaxN];
  uint8_t pos_rock[32];        // default-policy position -> rock index
  uint32_t range_mask[2];      // policy positions handled by robot r
  uint32_t d2max;
  uint32_t sense_thr_m1[kRsMaxD2];  // T(accuracy(d^2)) - 1 (T >= 2^31 > 0)
  // navigation
  int32_t wall_y, gate_x[2], goal_x, goal_y, nav_words;
  uint64_t t_fail, t_flip;
  int32_t nav_unknown;                   // number of unknown cells
  uint32_t nav_known_rows[kNavMaxN + 2];  // padded rows: border + known obstacles
  uint16_t nav_unk_pos[kNavMaxN * kNavMaxN];  // unknown idx -> (x+1) | (y+1) << 8
  // car
  int32_t peds;
  uint64_t t_car_fail;
  float noise_scale;
  float2 car_rot[1021];  // heading-noise rotation (c, s) by byte sum - 510 + 510 (card §3.4)
  // dense models: the kernels' shared-memory image (the model's Sm + its
  // tables) as M::load_sm builds it, made once at model load
  // (k_snapshot_sm); kernels copy it in with 16-byte loads (load_sm_image)
  const uint4* sm_snap;
  uint32_t sm_snap_words;
};

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32->64 products,
// key bumped by the Weyl constants between rounds.  Stream address of
// scenario id at depth t, word k: ctr = (id, t, k >> 2, tag), key = seed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// The Philox key of a batch: either the seed (round keys added on the fly)
// or the ten precomputed round keys passed as a kernel parameter, so that
// the key schedule costs no per-lane instructions (it is read straight from
// the constant bank by the LOP3s).
struct SeedKey {
  uint32_t k0, k1;
};
struct RoundKeys {
  uint32_t k0[10], k1[10];
};
__host__ inline RoundKeys round_keys(uint32_t k0, uint32_t k1) {
  RoundKeys rk;
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    rk.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return rk;
}
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const SeedKey& k) {
  return philox4x32_10(c0, c1, c2, c3, k.k0, k.k1);
}
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const RoundKeys& k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k.k0[r];
    const uint32_t n2 = hi0 ^ c3 ^ k.k1[r];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// NB consecutive blocks of one stream address, ctr = (c0, c1, j, 0) for
// j = 0 .. NB-1 (words 4j .. 4j+3 of scenario c0 at depth c1), computed round
// by round side by side: the blocks' independent multiply/xor chains
// interleave in the instruction stream (in-order issue gets NB-fold
// instruction-level parallelism instead of NB serial chains)
template <int NB, class KeyT>
__device__ __forceinline__ void philox_blocks(uint32_t id, uint32_t t, const KeyT& key, uint4* out) {
  uint32_t c0[NB], c1[NB], c2[NB], c3[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    c0[j] = id;
    c1[j] = t;
    c2[j] = (uint32_t)j;
    c3[j] = 0u;
  }
  uint32_t k0, k1;
  if constexpr (std::is_same<KeyT, SeedKey>::value) {
    k0 = key.k0;
    k1 = key.k1;
  }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t rk0, rk1;
    if constexpr (std::is_same<KeyT, SeedKey>::value) {
      if (r) {
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      rk0 = k0;
      rk1 = k1;
    } else {
      rk0 = key.k0[r];
      rk1 = key.k1[r];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const uint32_t lo0 = 0xD2511F53u * c0[j], hi0 = __umulhi(0xD2511F53u, c0[j]);
      const uint32_t lo1 = 0xCD9E8D57u * c2[j], hi1 = __umulhi(0xCD9E8D57u, c2[j]);
      const uint32_t n0 = hi1 ^ c1[j] ^ rk0;
      const uint32_t n2 = hi0 ^ c3[j] ^ rk1;
      c0[j] = n0;
      c1[j] = lo1;
      c2[j] = n2;
      c3[j] = lo0;
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) out[j] = make_uint4(c0[j], c1[j], c2[j], c3[j]);
}

// event of probability p: (uint64)u < T(p), T(p) = floor(p 2^32) (R14)
__device__ __forceinline__ bool event(uint32_t u, uint64_t T) { return (uint64_t)u < T; }

// ---------------------------------------------------------------------------
// Per-leaf descriptor built by the host for one batch.
// ---------------------------------------------------------------------------
struct LeafDev {
  const uint32_t* p_ids;
  const float* p_w;
  const uint32_t* p_states;  // SoA, row stride p_cap
  const uint32_t* p_keys;    // parent key table [A][p_kcap][OW]
  const uint32_t* p_nchild;  // [A]
  uint32_t p_cap, p_n, p_kcap;
  uint32_t* ids;             // leaf arena (== parent's for action == -1)
  float* w;
  uint32_t* states;
  uint32_t cap;
  uint32_t* keys;            // leaf key table [A][kcap][OW], written at expansion
  uint32_t* nchild;          // [A]
  uint32_t kcap;
  int32_t action;
  uint32_t child, depth;
  uint32_t seed_lo, seed_hi;
  double inv_wroot, wroot;
  const uint32_t* idx;       // DESPOT_X_INDEX_LISTS: the parent positions of the leaf (else null)
  uint32_t idx_n;
};

// error bits of a batch
enum : uint32_t {
  kErrEmptyLeaf = 1u, kErrChildCap = 2u, kErrHash = 4u, kErrScenCap = 8u,
  kErrXOverflow = 16u /* the exchange's packed capacity was too small: dense fallback */,
  kErrCheck = 32u     /* a device self-check failed (HD_CHECKS builds only) */,
  kErrIndexList = 64u /* a host index list names a scenario whose replay is not the leaf's key */
};

// Device self-checks of index and protocol invariants (the self-check build,
// -DHD_CHECKS, libdespot_checked.so; compute-sanitizer is not available on the
// GPU pool): a violated invariant sets kErrCheck in the batch's error word and
// the call fails.  Compiled out of the product build.
#ifdef HD_CHECKS
#define HD_CHECK(errp, cond)              \
  do {                                    \
    if (!(cond)) atomicOr((errp), kErrCheck); \
  } while (0)
#else
#define HD_CHECK(errp, cond) \
  do {                       \
  } while (0)
#endif

// status block of a batch (zeroed per batch; the host reads it back in one copy)
enum : uint32_t {
  kStatErr = 0, kStatChildren = 1, kStatSteps = 2 /* u64: 2-3 */, kStatK1Ticket = 4, kStatK2Ticket = 5,
  kStatK2Tile = 6 /* K2's dynamic tile counter */, kStatXTotal = 7 /* slots in the exchange's union (K4) */,
  kStatK3Done = 8 /* resident batches: K3 CTAs finished (the last one publishes and restores) */,
  kStatWords = 9 /* then n_leaf[L] */
};

struct BatchDev {
  const DevModel* model;
  const LeafDev* leaves;
  const LeafDev* leaves_src;  // the leaf table in page-locked host memory: K1's CTA l copies entry l
                              // into `leaves` first (no H2D copy of the table; null: already there)
  uint32_t L, A, S;          // S = dense slots per (leaf, action) (or per-leaf cap for sparse)
  unsigned long long a_magic;  // floor((2^64 - 1) / A) + 1: x / A = umul64hi(x, a_magic) for x < 2^32
  uint32_t* n_leaf;          // [L] local scenarios per leaf (K1)
  uint32_t* tile_off;        // [L+1] K2 warp tiles prefix
  uint64_t* scen_off;        // [L+1] per-scenario record prefix (A * n)
  int64_t* sums;             // exchange SUM block
  int32_t* mins;             // exchange MIN block
  uint32_t* rank;            // [L*A*S] child ordinal of a slot
  uint32_t* nc;              // [L*A] children per (leaf, action)
  unsigned long long* scan_flags;  // K3b look-back: [0] tile counter, [1 + t] tile t's (flag, prefix)
  uint32_t* status;          // [kStatWords header (kStat*), n_leaf[L]]
  uint32_t fused_k3;         // 1: K2's last CTA runs the small finalize
  uint32_t tile_off_global;  // 1: K2 searches tile_off in global memory (many leaves: the shared
                             // copy would cost a CTA per SM), not a shared copy
  uint32_t k2_prefix;        // 1: K2 forms the tile prefix from n_leaf itself (K1 skips its
                             // last-CTA prefix: dense keys, no per-scenario records)
  uint32_t* hstat;           // resident prepared batch (else null): K2's last CTA publishes the
                             // status here (mapped host memory) and restores the scratch's zero state
  uint32_t* err;
  // outputs (device)
  uint32_t* n_scen;
  float* weight;
  float *act_reward, *act_upper, *act_lower;
  uint32_t* child_begin;
  uint32_t child_capacity;
  uint32_t *child_count, *child_first;
  float *child_weight, *child_upper, *child_lower;
  uint32_t* child_obs;
  uint64_t scen_capacity;
  uint32_t* scen_obs;
  float *scen_reward, *scen_upper, *scen_lower;
  uint32_t* scen_len;
  uint64_t* scen_hash;
  uint32_t* scen_states;
  uint32_t* scen_child;
  // sparse-key scratch
  uint64_t* sp_hash;         // [L*A*S] per-slot key hash (0 = empty)
  uint32_t* sp_item;         // [L*A*S] scenario position holding the slot's key
  uint32_t* sp_keys;         // [L*A*S*OW] per-item observation keys (position-indexed)
};

// K1's prologue: this CTA's leaf descriptor from the host-side table (read
// over the bus once, kept in the device table for K2 and K3)
__device__ __forceinline__ void fetch_leaf(const BatchDev& b) {
  if (!b.leaves_src) return;
  constexpr uint32_t kWords = sizeof(LeafDev) / 4;
  static_assert(sizeof(LeafDev) % 4 == 0, "LeafDev is copied in words");
  const uint32_t* src = reinterpret_cast<const uint32_t*>(b.leaves_src + blockIdx.x);
  uint32_t* dst = reinterpret_cast<uint32_t*>(const_cast<LeafDev*>(b.leaves) + blockIdx.x);
  for (uint32_t k = threadIdx.x; k < kWords; k += blockDim.x) dst[k] = src[k];
  __syncthreads();
}


// layout of the SUM block: W, U, LAMBDA, N per slot; R, Uq, Lq per action; steps
struct SumLayout {
  uint64_t las, la;
  __host__ __device__ uint64_t W(uint64_t i) const { return i; }
  __host__ __device__ uint64_t U(uint64_t i) const { return las + i; }
  __host__ __device__ uint64_t Lm(uint64_t i) const { return 2 * las + i; }
  __host__ __device__ uint64_t N(uint64_t i) const { return 3 * las + i; }
  __host__ __device__ uint64_t Q(uint64_t la_i, int k) const { return 4 * las + 3 * la_i + k; }
  __host__ __device__ uint64_t steps() const { return 4 * las + 3 * la; }
  __host__ __device__ uint64_t total() const { return 4 * las + 3 * la + 1; }
};

// Exact int64 sum over the lanes of `mask` (every lane of mask calls it): the
// value is split into 27 + 27 + 10 bits, each part summed by one REDUX
// (__reduce_add_sync; 32 lanes x (2^27 - 1) < 2^32, the signed top part
// stays far inside int32) and reassembled mod 2^64 -- three warp reductions
// instead of five rounds of two 32-bit shuffles and a 64-bit add.
__device__ __forceinline__ int64_t group_sum64(uint32_t mask, int64_t v) {
  const uint64_t u = (uint64_t)v;
  const uint32_t p0 = (uint32_t)u & 0x7FFFFFFu;
  const uint32_t p1 = (uint32_t)(u >> 27) & 0x7FFFFFFu;
  const uint32_t p2 = (uint32_t)(int32_t)(v >> 54);
  const uint32_t s0 = __reduce_add_sync(mask, p0);
  const uint32_t s1 = __reduce_add_sync(mask, p1);
  const int32_t s2 = (int32_t)__reduce_add_sync(mask, p2);
  return (int64_t)((uint64_t)s0 + ((uint64_t)s1 << 27) + ((uint64_t)(int64_t)s2 << 54));
}
__device__ __forceinline__ int64_t warp_sum64(int64_t v) { return group_sum64(0xffffffffu, v); }

// Fire-and-forget reductions into the batch's global sums (relaxed, device
// scope: what atomicAdd / atomicMin without a used result are).  Through the
// global state space explicitly: on a generic pointer the compiler adds a
// shared-window test and a fallback path around every atomic.
__device__ __forceinline__ void red_add(int64_t* p, int64_t v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_min(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t warp_sum32(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }

// exact fixed-point quantisation of a normalised weighted value
__device__ __forceinline__ int64_t fxq(double v, double fx) { return __double2ll_rn(v * fx); }

}  // namespace hd
