// kernels.cuh -- the batched leaf-expansion kernels (sm_100a), templated on
// the model.  One batch = K1 (update/filter + tile prefix) -> K2
// (expansion + bounds + roll-outs + grouping, fused) -> [exchange] -> K3a
// (child order) -> K3b (CSR scan) -> K3c (outputs).  See DESIGN.md §4.
#pragma once
#include "common.cuh"
#include "finalize.cuh"

namespace hd {

// ---------------------------------------------------------------------------
// The shared-memory image of a dense model (its Sm and tables).  M::load_sm
// derives the tables from the DevModel (divisions, distance and threshold
// look-ups: ~2/3 of an update kernel's instructions); the library runs it
// once per model (k_snapshot_sm) and every kernel then copies the image.
// ---------------------------------------------------------------------------
template <class M>
__device__ __forceinline__ void load_sm_image(typename M::Sm& sm, const DevModel& dm, int tid, int nt) {
  if (const uint4* src = dm.sm_snap) {
    uint4* dst = reinterpret_cast<uint4*>(hd_dyn_smem);
    for (uint32_t i = tid; i < dm.sm_snap_words; i += nt) dst[i] = __ldg(src + i);
  } else {
    M::load_sm(sm, dm, tid, nt);
  }
}
template <class M>
__global__ void __launch_bounds__(256) k_snapshot_sm(const DevModel* dm, uint4* dst, uint32_t words) {
  typename M::Sm& sm = *reinterpret_cast<typename M::Sm*>(hd_dyn_smem);
  M::load_sm(sm, *dm, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint4* s = reinterpret_cast<const uint4*>(hd_dyn_smem);
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = s[i];
}


// ---------------------------------------------------------------------------
// K1: update.  One CTA per leaf: gather the parent's scenarios,
// replay the leaf's last action at depth Delta (drawing phi_Delta), keep those
// whose observation equals the parent's key of child `child`, and compact them
// (order kept) into the leaf arena.  Leaves with action == -1 only publish n.
// ---------------------------------------------------------------------------
template <class M>
__global__ void __launch_bounds__(512) k1_update(BatchDev b) {
  typename M::Sm& sm = *reinterpret_cast<typename M::Sm*>(hd_dyn_smem);
  __shared__ uint32_t warp_cnt[16];
  __shared__ uint32_t s_base;
  pdl_trigger();  // K2 may launch (it waits for this grid before reading)
  fetch_leaf(b);
  const LeafDev& lf = b.leaves[blockIdx.x];
  if (lf.action < 0) {
    if (threadIdx.x == 0) b.n_leaf[blockIdx.x] = lf.p_n;
  } else {
    load_sm_image<M>(sm, *b.model, threadIdx.x, blockDim.x);
    if (threadIdx.x == 0)  // the per-thread scratch after the model's tables (synced below)
      M::bind_scratch((uint32_t)(align16(sizeof(typename M::Sm)) + align16(b.model->sm_table_bytes)));
    const uint32_t nchild = lf.p_nchild[lf.action];
    const bool valid_child = lf.child < nchild;
    const uint32_t key = valid_child ? lf.p_keys[(uint64_t)lf.action * lf.p_kcap + lf.child] : 0xFFFFFFFFu;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t steps = 0;
    // the parent's scenarios (replay + filter), or the host's index list
    // (gather + replay, the replay checked against the leaf's key)
    const uint32_t cnt = lf.idx ? lf.idx_n : lf.p_n;
    for (uint32_t base = 0; base < cnt; base += blockDim.x) {
      const uint32_t j = base + threadIdx.x;
      const uint32_t i = lf.idx ? (j < cnt ? lf.idx[j] : 0u) : j;
      bool keep = false;
      typename M::St s;
      uint32_t id = 0;
      if (j < cnt && valid_child) {
        s = M::load(sm, lf.p_states, lf.p_cap, i);
        id = lf.p_ids[i];
        uint32_t z;
        if (M::terminal(sm, s)) {
          z = M::kTerminalObs;
        } else {
          float r;
          M::step(sm, s, lf.action, id, lf.depth, SeedKey{lf.seed_lo, lf.seed_hi}, z, r);
          ++steps;
        }
        keep = z == key;
        if (lf.idx && !keep) {
          atomicOr(b.err, kErrIndexList);
          keep = true;
        }
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) warp_cnt[wid] = __popc(ballot);
      __syncthreads();
      uint32_t off = s_base;
      for (int w = 0; w < wid; ++w) off += warp_cnt[w];
      off += __popc(ballot & ((1u << lane) - 1u));
      if (keep) {
        HD_CHECK(b.err, off < lf.cap);
        lf.ids[off] = id;
        lf.w[off] = lf.p_w[i];
        M::store(sm, s, lf.states, lf.cap, off);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_cnt[w];
        s_base += tot;
      }
      __syncthreads();
    }
    const uint32_t ws = warp_sum32(steps);
    if (lane == 0 && ws)
      atomicAdd((unsigned long long*)&b.sums[SumLayout{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A}.steps()],
                (unsigned long long)ws);
    if (threadIdx.x == 0) b.n_leaf[blockIdx.x] = s_base;  // may be 0 on a shard
  }
  // K2pre folded in: the last CTA scans the leaf sizes -- unless K2 forms the
  // tile prefix itself (no serial tail on K1)
  if (!b.k2_prefix) last_cta_prefix(b);
}

// ---------------------------------------------------------------------------
// K2 (dense observation keys): one warp per tile of 32 consecutive scenarios
// of one (leaf, action).  Each lane: expansion step (Eq. 9) at depth
// Delta+1, u(s') (Eq. 11), roll-out (Eq. 12), then the warp groups its lanes
// by observation and adds exact int64 fixed-point partial sums of
// (W, U, LAMBDA, N, first) per child slot and (R, Uq, Lq) per action.
// Persistent grid; tiles handed out dynamically (next_tile).
// ---------------------------------------------------------------------------
// UNI_SEED: every leaf of the batch descends from the same belief, so the
// Philox key is a kernel parameter (uniform registers; the key schedule costs
// no per-lane instructions).
#ifndef HD_K2_LANE_RED
#define HD_K2_LANE_RED 1  // 0: the warp always groups its lanes by observation before reducing
#endif
#ifndef HD_K2_LANE_RED_CHUNKS
#define HD_K2_LANE_RED_CHUNKS 16
#endif
constexpr uint32_t kLaneRedChunks = HD_K2_LANE_RED_CHUNKS;  // per-lane reductions up to this many tiles per (leaf, action)
__device__ __forceinline__ uint32_t next_tile(const BatchDev& b, uint32_t nwarps, uint32_t lane) {
  uint32_t t = 0;
  if (lane == 0) t = nwarps + atomicAdd(&b.status[kStatK2Tile], 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}
template <class M, bool RECORD, bool UNI_SEED = false, bool LANE_RED = false>
__global__ void __launch_bounds__(128, M::kMinBlocks) k2_expand_dense(BatchDev b, const RoundKeys rk) {
  typename M::Sm& sm = *reinterpret_cast<typename M::Sm*>(hd_dyn_smem);
  // dynamic shared memory: Sm | tables | tile_off (unless searched in global
  // memory) | the per-thread scratch / the fused finalize's region
  unsigned char* region = hd_dyn_smem + align16(sizeof(typename M::Sm)) + align16(b.model->sm_table_bytes);
  const uint32_t toff_bytes = b.tile_off_global ? 0u : (uint32_t)align16(4 * ((size_t)b.L + 1));
  uint32_t* tile_off_s = reinterpret_cast<uint32_t*>(region);
  const uint32_t* tile_off = b.tile_off_global ? b.tile_off : tile_off_s;
  load_sm_image<M>(sm, *b.model, threadIdx.x, blockDim.x);
  // the per-thread scratch shares the fused finalize's region (used after the tiles)
  if (threadIdx.x == 0) M::bind_scratch((uint32_t)(region - hd_dyn_smem) + toff_bytes);
  pdl_wait();  // K1 complete: tile_off, the leaf arenas
  pdl_trigger();
  __shared__ uint64_t wsum[32];  // block scans: the tile prefix, the fused finalize
  if (b.tile_off_global) {
  } else if (b.k2_prefix) {  // tile_off[l] = sum_{l' < l} A ceil(n_l' / 32), every CTA for itself
    const uint32_t per = (b.L + blockDim.x - 1) / blockDim.x, l0 = threadIdx.x * per;
    auto tiles_of = [&](uint32_t l) { return (uint64_t)b.A * ((__ldcg(&b.n_leaf[l]) + 31u) >> 5); };
    uint64_t tiles = 0;
    for (uint32_t l = l0; l < l0 + per && l < b.L; ++l) tiles += tiles_of(l);
    uint64_t ttot;
    uint64_t tb = block_excl_scan(tiles, wsum, ttot);
    for (uint32_t l = l0; l < l0 + per && l < b.L; ++l) {
      tile_off_s[l] = (uint32_t)tb;
      tb += tiles_of(l);
    }
    if (threadIdx.x == 0) {
      tile_off_s[b.L] = (uint32_t)ttot;
      if (ttot >= 0xFFFFFFFFull && blockIdx.x == 0) atomicOr(b.err, kErrChildCap);
    }
  } else {
    for (uint32_t l = threadIdx.x; l <= b.L; l += blockDim.x) tile_off_s[l] = b.tile_off[l];
  }
  __syncthreads();
  const uint32_t total = tile_off[b.L];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const DevModel& dm = *b.model;
  const double fx = dm.fx, gamma = dm.gamma;
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  uint32_t steps_acc = 0;
  // dynamic tile scheduling: a warp's first tile is its index, every later
  // one comes from a global counter, so the warps finish within about one
  // tile of each other (a static stride leaves the slowest of ~5000 warps'
  // sums of ~100 random tile times ~35% above the mean)
  uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t leaf = 0;  // tile_off[leaf] <= t: a warp's tiles only increase
  for (; t < total; t = next_tile(b, nwarps, lane)) {
    // tile -> (leaf, action, chunk): gallop forward from the previous leaf
    // (the next tile is ~nwarps further, usually in the same or the next
    // leaf), then bisect
    uint32_t step = 1, lo = leaf, hi = leaf + 1;
    while (hi < b.L && tile_off[hi] <= t) {
      lo = hi;
      hi = min(hi + step, b.L);
      step <<= 1;
    }
    while (hi - lo > 1) {  // tile_off[lo] <= t < tile_off[hi] (tile_off[L] = total > t)
      const uint32_t mid = (lo + hi) >> 1;
      if (tile_off[mid] <= t) lo = mid;
      else hi = mid;
    }
    leaf = lo;
    const LeafDev& lf = b.leaves[leaf];
    const uint32_t n = b.n_leaf[leaf];
    const uint32_t chunks = (n + 31) >> 5;
    const uint32_t local = t - tile_off[leaf];
    // chunk-major within the leaf (local = chunk * A + a: consecutive tiles
    // share their 32 scenarios' states), the division by A as a 64-bit
    // multiply-high (exact for 32-bit dividends)
    const uint32_t chunk = b.A > 1 ? (uint32_t)__umul64hi((unsigned long long)local, b.a_magic) : local;
    const uint32_t a = local - chunk * b.A;
    const uint32_t i = chunk * 32 + lane;
    const bool valid = i < n;
    HD_CHECK(b.err, a < b.A && leaf < b.L && (!valid || i < lf.cap));
    uint32_t z = 0xFFFFFFFFu, id = 0;
    int64_t qW = 0, qU = 0, qL = 0, qR = 0, qUq = 0, qLq = 0;
    auto item = [&](const auto& key) {
      typename M::St s = M::load(sm, lf.states, lf.cap, i);
      id = lf.ids[i];
      const double wn = (double)lf.w[i] * lf.inv_wroot;  // normalised weight
      float r = 0.0f;
      bool term;
      if (M::terminal(sm, s)) {  // R7: terminal scenarios stay terminal, reward 0
        z = M::kTerminalObs;
        term = true;
      } else {
        term = M::step(sm, s, (int)a, id, lf.depth + 1, key, z, r);
        ++steps_acc;
      }
      double u = 0.0, lam = 0.0;
      uint32_t len = 0;
      uint64_t h = kFnvOffset;
      if (!term) {
        u = M::upper(sm, s);
        M::template rollout<RECORD>(sm, s, z, id, lf.depth + 1, key, lam, len, h);
        steps_acc += len;
      }
      qW = fxq(wn, fx);
      qU = fxq(wn * u, fx);
      qL = fxq(wn * lam, fx);
      qR = fxq(wn * (double)r, fx);
      qUq = fxq(wn * ((double)r + gamma * u), fx);
      qLq = fxq(wn * ((double)r + gamma * lam), fx);
      if (RECORD) {
        const uint64_t q = b.scen_off[leaf] + (uint64_t)a * n + i;
        if (q < b.scen_capacity) {
          b.scen_obs[q] = z;
          b.scen_reward[q] = r;
          b.scen_upper[q] = (float)u;
          b.scen_lower[q] = (float)lam;
          b.scen_len[q] = len;
          b.scen_hash[q] = h;
          if (b.scen_states) {
            // s' after the expansion step: recompute (the roll-out consumed s)
            typename M::St s2 = M::load(sm, lf.states, lf.cap, i);
            if (!M::terminal(sm, s2)) {
              uint32_t z2;
              float r2;
              M::step(sm, s2, (int)a, id, lf.depth + 1, key, z2, r2);
            }
            // scen_states is [S][SW] (row per scenario): write through a strided view
            uint32_t tmp[16];
            M::store(sm, s2, tmp, 1, 0);
            for (uint32_t k = 0; k < dm.SW; ++k) b.scen_states[q * dm.SW + k] = tmp[k];
          }
        } else {
          atomicOr(b.err, kErrScenCap);
        }
      }
    };
    if (valid) {
      if constexpr (UNI_SEED) item(rk);
      else item(SeedKey{lf.seed_lo, lf.seed_hi});
    }
    // ---- per-action sums (R, Uq, Lq) -----------------------------------
    const uint64_t la = (uint64_t)leaf * b.A + a;
    // (a warp-wide sum: all 32 lanes share these three addresses, and 32-way
    // same-address reductions from every lane measured 1.08 -> 1.58 ms)
    const int64_t sR = warp_sum64(qR), sUq = warp_sum64(qUq), sLq = warp_sum64(qLq);
    if (lane == 0) {
      red_add(&b.sums[lay.Q(la, 0)], sR);
      red_add(&b.sums[lay.Q(la, 1)], sUq);
      red_add(&b.sums[lay.Q(la, 2)], sLq);
    }
    // ---- grouping by observation (Eq. 10) ------------------------------
    // Few tiles per (leaf, action): every lane reduces its exact terms
    // straight into its (leaf, action, observation) slot and the L2's atomic
    // units do the grouping -- the warp's own grouping (the loop below: the
    // distinct observations, a REDUX sum of each group's 64-bit terms in
    // three parts, one leader's reductions) costs ~95 instructions per group,
    // ~3 groups per tile (config 2 K2 1.148 -> 1.078 ms, config 3 63.5 ->
    // 59.9 us).  Many tiles per (leaf, action) (large beliefs, config 5): the
    // warps working at any moment share a few slots, and same-address
    // reductions from every lane serialise in the L2 (config 5 224 -> 509 ms
    // with action-major tiles), so the warp groups first -- unless the leaf
    // has many slots (A x S >= 1024: chunk-major tiles keep the warps in
    // flight on different slots; LANE_RED is chosen per batch on the host).
    // Exact int64 sums: the same result either way.
    uint32_t pending = 0;
    if constexpr (LANE_RED) {
      if (valid) {
        const uint64_t slot = la * b.S + z;
        red_add(&b.sums[lay.W(slot)], qW);
        red_add(&b.sums[lay.U(slot)], qU);
        red_add(&b.sums[lay.Lm(slot)], qL);
        red_add(&b.sums[lay.N(slot)], (int64_t)1);
        red_min(&b.mins[slot], (int32_t)id);
      }
    } else {
      pending = __ballot_sync(0xffffffffu, valid);
    }
    while (pending) {
      const int leader = __ffs(pending) - 1;
      const uint32_t zk = __shfl_sync(0xffffffffu, z, leader);
      const bool in = valid && z == zk;
      const uint32_t gmask = __ballot_sync(0xffffffffu, in);
      pending &= ~gmask;
      if (in) {  // the group's lanes reduce over its mask
        const int64_t gW = group_sum64(gmask, qW), gU = group_sum64(gmask, qU), gL = group_sum64(gmask, qL);
        if ((int)lane == leader) {
          const uint64_t slot = la * b.S + zk;
          HD_CHECK(b.err, zk < b.S && la < (uint64_t)b.L * b.A);
          red_add(&b.sums[lay.W(slot)], gW);
          red_add(&b.sums[lay.U(slot)], gU);
          red_add(&b.sums[lay.Lm(slot)], gL);
          red_add(&b.sums[lay.N(slot)], (int64_t)__popc(gmask));
          red_min(&b.mins[slot], (int32_t)id);  // leader = lowest position = smallest id
        }
      }
    }
  }
  const uint32_t ws = warp_sum32(steps_acc);
  if (lane == 0 && ws) red_add(&b.sums[lay.steps()], (int64_t)ws);
  if (b.fused_k3) {
    // small batch: the last CTA to finish ranks, scans and writes the
    // children (K3) -- one launch per expansion instead of two
    __shared__ bool k2_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      k2_last = atomicAdd(&b.status[kStatK2Ticket], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (k2_last) {
      __threadfence();
      small_finalize_tail(b, region + toff_bytes, wsum);
      if (b.hstat) resident_epilogue(b);
    }
  }
}

// ---------------------------------------------------------------------------
// Roll-out bounds of a node at its own depth (Eqs. 11-12 for the root).
// ---------------------------------------------------------------------------
template <class M>
__global__ void __launch_bounds__(128) k_rollout_bounds(const DevModel* dmp, const uint32_t* ids,
                                                        const float* w, const uint32_t* states,
                                                        uint32_t cap, uint32_t n, uint32_t depth,
                                                        uint32_t k0, uint32_t k1, double inv_wroot,
                                                        float* per_u, float* per_l, int64_t* acc3) {
  typename M::Sm& sm = *reinterpret_cast<typename M::Sm*>(hd_dyn_smem);
  load_sm_image<M>(sm, *dmp, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) M::bind_scratch((uint32_t)(align16(sizeof(typename M::Sm)) + align16(dmp->sm_table_bytes)));
  __syncthreads();
  const double fx = dmp->fx;
  int64_t qW = 0, qU = 0, qL = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    typename M::St s = M::load(sm, states, cap, i);
    double u = 0.0, lam = 0.0;
    if (!M::terminal(sm, s)) {
      u = M::upper(sm, s);
      uint32_t len;
      uint64_t h = kFnvOffset;
      M::template rollout<false>(sm, s, M::initial_obs(sm, s), ids[i], depth, SeedKey{k0, k1}, lam, len, h);
    }
    if (per_u) per_u[i] = (float)u;
    if (per_l) per_l[i] = (float)lam;
    const double wn = (double)w[i] * inv_wroot;
    qW += fxq(wn, fx);
    qU += fxq(wn * u, fx);
    qL += fxq(wn * lam, fx);
  }
  qW = warp_sum64(qW);
  qU = warp_sum64(qU);
  qL = warp_sum64(qL);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long*)&acc3[0], (unsigned long long)qW);
    atomicAdd((unsigned long long*)&acc3[1], (unsigned long long)qU);
    atomicAdd((unsigned long long*)&acc3[2], (unsigned long long)qL);
  }
}

}  // namespace hd
