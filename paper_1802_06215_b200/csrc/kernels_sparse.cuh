// kernels_sparse.cuh -- batched expansion for sparse multi-word observation
// keys (the driving model, card §3.4; |Z| is huge).
//
//   K1s  update/filter with a full-key compare against the parent's key table
//   K2f  expansion + bounds + roll-out, one WARP per (leaf, action, scenario):
//        lane p < P moves pedestrian p, lane 31 the car -- the paper's
//        within-step factoring -- or
//   K2t  the same with one THREAD per (leaf, action, scenario)
//        Both write, per item, the 64-bit key hash, the key words and the
//        exact fixed-point (W, U, LAMBDA) contributions.
//   K3s  one CTA per (leaf, action): group items by hash (first occurrence),
//        verify exact key equality against the group's first item (a 64-bit
//        hash collision is reported, never merged), and add the per-child
//        sums into the same exchange layout the dense path uses.
#pragma once
#include "common.cuh"
#include "model_car.cuh"
#include "finalize.cuh"

namespace hd {

// hash of a key: XOR over words of splitmix64(word ^ (k+1) << 32)
__device__ __forceinline__ uint64_t key_mix(uint32_t w, uint32_t k) {
  uint64_t x = (uint64_t)w ^ ((uint64_t)(k + 1) << 32);
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
constexpr uint32_t kCarTerminalWord0 = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// K1s: update for the car (thread per parent scenario)
// ---------------------------------------------------------------------------
template <class M>
__global__ void __launch_bounds__(256) k1_update_sparse(BatchDev b) {
  __shared__ typename M::Sm sm;
  __shared__ uint32_t warp_cnt[8];
  __shared__ uint32_t s_base;
  pdl_trigger();  // K2 may launch (it waits for this grid before reading)
  fetch_leaf(b);
  const LeafDev& lf = b.leaves[blockIdx.x];
  if (lf.action < 0) {
    if (threadIdx.x == 0) b.n_leaf[blockIdx.x] = lf.p_n;
    last_cta_prefix(b);
    return;  // uniform per CTA
  }
  M::load_sm(sm, *b.model, threadIdx.x, blockDim.x);
  const uint32_t OW = b.model->OW;
  const bool valid_child = lf.child < lf.p_nchild[lf.action];
  const uint32_t* key = lf.p_keys + ((uint64_t)lf.action * lf.p_kcap + lf.child) * OW;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t steps = 0;
  // the parent's scenarios (replay + filter), or the host's index list
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
      bool term = M::terminal(sm, s);
      if (!term) {
        float r;
        term = M::step(sm, s, lf.action, id, lf.depth, SeedKey{lf.seed_lo, lf.seed_hi}, r);
        ++steps;
      }
      if (term) {
        keep = key[0] == kCarTerminalWord0;
        for (uint32_t k = 1; k < OW; ++k) keep = keep && key[k] == 0u;
      } else {
        keep = true;
        M::for_obs_words(sm, s, [&](uint32_t k, uint32_t zk) { keep = keep && zk == key[k]; });
      }
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
  if (threadIdx.x == 0) b.n_leaf[blockIdx.x] = s_base;
  last_cta_prefix(b);
}

// item t -> (leaf, action, position) through the per-scenario prefix
__device__ __forceinline__ uint32_t find_leaf(const uint64_t* off, uint32_t L, uint64_t t) {
  uint32_t lo = 0, hi = L;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= t) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct SparseItemOut {
  uint64_t* hash;    // [Q]
  uint32_t* keys;    // [Q*OW]  (item q's key at keys + q * kstride)
  int64_t* q3;       // [Q*3]  W, U, LAMBDA contributions
  uint32_t kstride;  // words between consecutive keys: OW, or a merged record's size
};

// ---------------------------------------------------------------------------
// K2t: thread per (leaf, action, scenario)
// ---------------------------------------------------------------------------
#ifndef HD_CART_MINB
#define HD_CART_MINB 3  // CTAs of 128 per SM (4: 128 registers with spills, measured slower)
#endif
template <class M, bool RECORD>
// 3 CTAs of 128 per SM: 168 registers, no spills (without the bound ptxas
// may take 181, which leaves 2 CTAs: 0.96 -> 1.25 ms on config 4; 4 CTAs
// spill: 1.06 ms)
__global__ void __launch_bounds__(128, HD_CART_MINB) k2_car_thread(BatchDev b, SparseItemOut io) {
  __shared__ typename M::Sm sm;
  M::load_sm(sm, *b.model, threadIdx.x, blockDim.x);
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  __syncthreads();
  const DevModel& dm = *b.model;
  const uint32_t OW = dm.OW, SW = dm.SW;
  const uint64_t Q = b.scen_off[b.L];
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  uint32_t steps_acc = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Q; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t leaf = find_leaf(b.scen_off, b.L, t);
    const LeafDev& lf = b.leaves[leaf];
    const uint32_t n = b.n_leaf[leaf];
    const uint64_t local = t - b.scen_off[leaf];
    const uint32_t a = (uint32_t)(local / n), i = (uint32_t)(local - (uint64_t)a * n);
    typename M::St s = M::load(sm, lf.states, lf.cap, i);
    const uint32_t id = lf.ids[i];
    const double wn = (double)lf.w[i] * lf.inv_wroot;
    float r = 0.0f;
    bool term = M::terminal(sm, s);
    if (!term) {
      term = M::step(sm, s, (int)a, id, lf.depth + 1, SeedKey{lf.seed_lo, lf.seed_hi}, r);
      ++steps_acc;
    }
    uint64_t hsh = 0;
    auto put = [&](uint32_t k, uint32_t zk) {
      io.keys[t * OW + k] = zk;
      if (RECORD) b.scen_obs[t * OW + k] = zk;
      hsh ^= key_mix(zk, k);
    };
    if (term) {
      for (uint32_t k = 0; k < OW; ++k) put(k, k == 0 ? kCarTerminalWord0 : 0u);
    } else {
      M::for_obs_words(sm, s, put);
    }
    io.hash[t] = hsh;
    if (RECORD && b.scen_states) {
      uint32_t* dst = b.scen_states + t * SW;  // row per scenario: stride-1 view
      M::store(sm, s, dst, 1, 0);
    }
    double u = 0.0, lam = 0.0;
    uint32_t len = 0;
    uint64_t h = kFnvOffset;
    if (!term) {
      u = M::upper(sm, s);
      M::template rollout<RECORD>(sm, s, 0u, id, lf.depth + 1, SeedKey{lf.seed_lo, lf.seed_hi}, lam, len, h);
      steps_acc += len;
    }
    const double fx = dm.fx, gamma = dm.gamma;
    io.q3[3 * t + 0] = fxq(wn, fx);
    io.q3[3 * t + 1] = fxq(wn * u, fx);
    io.q3[3 * t + 2] = fxq(wn * lam, fx);
    const uint64_t la = (uint64_t)leaf * b.A + a;
    red_add(&b.sums[lay.Q(la, 0)], fxq(wn * (double)r, fx));
    red_add(&b.sums[lay.Q(la, 1)], fxq(wn * ((double)r + gamma * u), fx));
    red_add(&b.sums[lay.Q(la, 2)], fxq(wn * ((double)r + gamma * lam), fx));
    if (RECORD) {
      b.scen_reward[t] = r;
      b.scen_upper[t] = (float)u;
      b.scen_lower[t] = (float)lam;
      b.scen_len[t] = len;
      b.scen_hash[t] = h;
    }
  }
  atomicAdd((unsigned long long*)&b.sums[lay.steps()], (unsigned long long)steps_acc);
}

// ---------------------------------------------------------------------------
// K2f: warp per (leaf, action, scenario); lane p < P: pedestrian p, lane 31:
// the car.  Bit-identical to K2t (same operation sequence per element).
// ---------------------------------------------------------------------------
template <bool RECORD>
__global__ void __launch_bounds__(128) k2_car_warp(BatchDev b, SparseItemOut io) {
  __shared__ typename CarThreadT<1>::Sm sm;  // scalar parameters + gamma table
  CarThreadT<1>::load_sm(sm, *b.model, threadIdx.x, blockDim.x);
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  __syncthreads();
  const DevModel& dm = *b.model;
  const uint32_t OW = dm.OW, SW = dm.SW;
  const int P = sm.peds;
  const uint32_t lane = threadIdx.x & 31;
  const bool is_car = lane == 31, is_ped = (int)lane < P;
  const uint32_t word = is_car ? 0u : 1u + lane;  // random word / observation word of this lane
  const uint64_t Q = b.scen_off[b.L];
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  uint32_t steps_acc = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < Q; t += nwarps) {
    const uint32_t leaf = find_leaf(b.scen_off, b.L, t);
    const LeafDev& lf = b.leaves[leaf];
    const uint32_t n = b.n_leaf[leaf];
    const uint64_t local = t - b.scen_off[leaf];
    const uint32_t a0 = (uint32_t)(local / n), i = (uint32_t)(local - (uint64_t)a0 * n);
    const uint32_t id = lf.ids[i];
    const uint32_t cap = lf.cap;
    // element state: car lane (xc, level, term), pedestrian lanes (x, y, goal)
    float xc = __uint_as_float(lf.states[i]);
    const uint32_t w1 = lf.states[cap + i];
    uint32_t level = w1 & 0xFFu;
    bool term = (w1 >> 8) & 1u;
    float px = 0.0f, py = 0.0f;
    uint32_t goal = 0;
    if (is_ped) {
      px = __uint_as_float(lf.states[(4 + 2 * lane) * cap + i]);
      py = __uint_as_float(lf.states[(5 + 2 * lane) * cap + i]);
      goal = (lf.states[(2 + (lane >> 4)) * cap + i] >> (2 * (lane & 15))) & 3u;
    }
    // one factored step g(s, a, phi_t); returns reward, updates term
    auto step = [&](int a, uint32_t tt, float& r) {
      const uint4 wv = philox4x32_10(id, tt, word >> 2, 0u, lf.seed_lo, lf.seed_hi);
      const uint32_t sel = word & 3u;
      const uint32_t u = sel == 0 ? wv.x : sel == 1 ? wv.y : sel == 2 ? wv.z : wv.w;
      // 1. the car (all lanes track it; the car lane's word decides failure)
      const bool fail = __shfl_sync(0xffffffffu, event(u, sm.t_fail) ? 1 : 0, 31) != 0;
      if (!fail) {
        if (a == 1 && level < 4u) level += 1u;
        if (a == 2 && level > 0u) level -= 1u;
      }
      const float v = 0.5f * (float)level;
      xc = xc + v * 0.25f;
      // 2. pedestrians, 3. collision
      bool hit = false;
      if (is_ped) {
        const float2 cs = sm.rot[car_noise_index(u)];
        car_ped_move(px, py, goal, cs.x, cs.y);
        const float dx = px - xc;
        hit = dx * dx + py * py < 1.0f;
      }
      const bool coll = __any_sync(0xffffffffu, hit);
      const bool g = xc >= 20.0f;  // 4. goal
      r = car_reward(a, coll, g, v);
      term = coll || g;
    };
    float r0 = 0.0f;
    const bool was_term = term;
    if (!term) {
      step((int)a0, lf.depth + 1, r0);
      ++steps_acc;
    }
    // key of the child: lane k holds word k (car lane: word 0)
    uint32_t zw = 0;
    if (term) zw = is_car ? kCarTerminalWord0 : 0u;
    else if (is_car) zw = car_bin(xc) | (level << 16);
    else if (is_ped) zw = car_bin(px) | (car_bin(py) << 16);
    uint64_t hk = (is_car || is_ped) ? key_mix(zw, word) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hk ^= __shfl_xor_sync(0xffffffffu, hk, o);
    if (is_car || is_ped) {
      io.keys[t * OW + word] = zw;
      if (RECORD) b.scen_obs[t * OW + word] = zw;
    }
    if (lane == 0) io.hash[t] = hk;
    if (RECORD && b.scen_states) {
      uint32_t* dst = b.scen_states + t * SW;
      if (is_car) {
        dst[0] = __float_as_uint(xc);
        dst[1] = level | ((uint32_t)term << 8);
        dst[2] = lf.states[2 * cap + i];
        dst[3] = lf.states[3 * cap + i];
      }
      if (is_ped) {
        dst[4 + 2 * lane] = __float_as_uint(px);
        dst[5 + 2 * lane] = __float_as_uint(py);
      }
    }
    double u = 0.0, lam = 0.0;
    uint32_t len = 0;
    uint64_t h = kFnvOffset;
    if (!term) {
      int k = (int)ceilf((20.0f - xc) * 2.0f);
      k = k < 1 ? 1 : k;
      u = 100.0 * sm.gpow[k - 1];  // Eq. 11
      // roll-out (Eq. 12): pi0 reads the last observation's bins
      uint32_t tt = lf.depth + 1;
      double acc = 0.0;
      while (tt < sm.D && !term) {
        const int cxb = car_bin_i(xc);
        int gap = 255;
        if (is_ped) {
          const int pxb = car_bin_i(px), pyb = car_bin_i(py);
          if (pxb >= cxb && pyb >= -4 && pyb <= 3) gap = pxb - cxb;
        }
        gap = (int)__reduce_min_sync(0xffffffffu, (uint32_t)gap);
        const int a = car_policy_from_gap(gap);
        if (RECORD) h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
        float r;
        step(a, tt + 1, r);
        acc += sm.gpow[tt - (lf.depth + 1)] * (double)r;
        ++tt;
      }
      if (!term) acc += sm.gpow[tt - (lf.depth + 1)] * sm.tail;
      lam = acc;
      len = tt - (lf.depth + 1);
      steps_acc += len;
    }
    (void)was_term;
    if (lane == 0) {
      const double wn = (double)lf.w[i] * lf.inv_wroot;
      const double fx = dm.fx, gamma = dm.gamma;
      io.q3[3 * t + 0] = fxq(wn, fx);
      io.q3[3 * t + 1] = fxq(wn * u, fx);
      io.q3[3 * t + 2] = fxq(wn * lam, fx);
      const uint64_t la = (uint64_t)leaf * b.A + a0;
      red_add(&b.sums[lay.Q(la, 0)], fxq(wn * (double)r0, fx));
      red_add(&b.sums[lay.Q(la, 1)], fxq(wn * ((double)r0 + gamma * u), fx));
      red_add(&b.sums[lay.Q(la, 2)], fxq(wn * ((double)r0 + gamma * lam), fx));
      if (RECORD) {
        b.scen_reward[t] = r0;
        b.scen_upper[t] = (float)u;
        b.scen_lower[t] = (float)lam;
        b.scen_len[t] = len;
        b.scen_hash[t] = h;
      }
    }
  }
  if (lane == 0) atomicAdd((unsigned long long*)&b.sums[lay.steps()], (unsigned long long)steps_acc);
}

// ---------------------------------------------------------------------------
// K2g: several scenarios per warp (NEXT-3's "packing several small-element
// scenarios per warp"): a group of G = ceil((P + 1) / 4) lanes per
// (leaf, action, scenario), lane q of the group owning Philox block q of the
// step -- the random words 4q .. 4q+3: word 0 is the car's, word 1 + p
// pedestrian p's -- so each lane draws exactly one block per step (as many
// blocks per scenario as the thread kernel) and moves its (up to) four
// pedestrians; the car is tracked by every lane of the group, the failure
// draw comes from lane 0, collisions are a ballot over the group, the
// policy's gap a minimum over the group.  32 / G scenarios per warp (five
// for 20 pedestrians).  Bit-identical to K2t (same operation sequence per
// element).  The group loops run warp-uniformly (shuffles need every lane).
// B > 1: lane q owns B consecutive blocks (words 4Bq .. 4B(q+1)-1), so a group
// has ceil(blocks / B) lanes -- e.g. B = 3 for 20 pedestrians: a lane pair
// per scenario, sixteen scenarios per warp (DESPOT_MF_PAIRED).
// ---------------------------------------------------------------------------
#ifndef HD_CARG_MINB
#define HD_CARG_MINB 6  // 80 registers: the best of 1, 5, 6, 8 CTAs per SM (config 4)
#endif
template <bool RECORD, int B = 1>
__global__ void __launch_bounds__(128, B == 1 ? HD_CARG_MINB : 4) k2_car_group(BatchDev b, SparseItemOut io) {
  constexpr int W = 4 * B;  // words (elements) per lane
  __shared__ typename CarThreadT<1>::Sm sm;  // scalar parameters + gamma table + rotations
  CarThreadT<1>::load_sm(sm, *b.model, threadIdx.x, blockDim.x);
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  __syncthreads();
  const DevModel& dm = *b.model;
  const uint32_t OW = dm.OW, SW = dm.SW;
  const int P = sm.peds;
  const uint32_t NB = (uint32_t)(P + 1 + 3) / 4;                 // Philox blocks per step
  const uint32_t G = (NB + B - 1) / B, GPW = 32 / G;             // lanes per scenario, scenarios per warp
  const uint32_t lane = threadIdx.x & 31, gw = lane / G, q = lane - gw * G;
  const bool in_group = gw < GPW;                 // the last 32 mod G lanes idle
  const uint32_t g0 = gw * G;                     // first lane of the group
  const uint32_t gmask = in_group ? ((G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << g0) : 0u;
  const uint64_t Q = b.scen_off[b.L];
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  const uint64_t wglobal = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  uint32_t steps_acc = 0;
  for (uint64_t base = wglobal * GPW; base < Q; base += nwarps * GPW) {
    const uint64_t t = base + gw;
    const bool valid = in_group && t < Q;
    uint32_t leaf = 0, a0 = 0, i = 0, id = 0, cap = 1;
    const LeafDev* lfp = b.leaves;
    if (valid) {
      leaf = find_leaf(b.scen_off, b.L, t);
      lfp = &b.leaves[leaf];
      const uint32_t n = b.n_leaf[leaf];
      const uint64_t local = t - b.scen_off[leaf];
      a0 = (uint32_t)(local / n);
      i = (uint32_t)(local - (uint64_t)a0 * n);
      id = lfp->ids[i];
      cap = lfp->cap;
    }
    const LeafDev& lf = *lfp;
    // element state: the car (every lane), this lane's pedestrians p = 4q + k - 1
    float xc = 0.0f;
    uint32_t level = 0;
    bool term = true;
    float px[W], py[W];
    uint32_t goal[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
      px[k] = 0.0f;
      py[k] = 0.0f;
      goal[k] = 0u;
    }
    if (valid) {
      xc = __uint_as_float(lf.states[i]);
      const uint32_t w1 = lf.states[cap + i];
      level = w1 & 0xFFu;
      term = (w1 >> 8) & 1u;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int p = (int)(W * q) + k - 1;
        if (p >= 0 && p < P) {
          px[k] = __uint_as_float(lf.states[(4 + 2 * p) * cap + i]);
          py[k] = __uint_as_float(lf.states[(5 + 2 * p) * cap + i]);
          goal[k] = (lf.states[(2 + (p >> 4)) * cap + i] >> (2 * (p & 15))) & 3u;
        }
      }
    }
    // one factored step g(s, a, phi_tt) of this lane's group (active: the
    // group still steps; inactive groups run the shuffles only)
    auto step = [&](bool active, int a, uint32_t tt, float& r) {
      uint32_t ws[W];  // words Wq .. Wq+W-1 (blocks Bq .. Bq+B-1)
#pragma unroll
      for (int bb = 0; bb < B; ++bb) {
        uint4 wv = make_uint4(0u, 0u, 0u, 0u);
        if (B == 1 || B * q + bb < NB) wv = philox4x32_10(id, tt, B * q + (uint32_t)bb, 0u, lf.seed_lo, lf.seed_hi);
        ws[4 * bb] = wv.x;
        ws[4 * bb + 1] = wv.y;
        ws[4 * bb + 2] = wv.z;
        ws[4 * bb + 3] = wv.w;
      }
      // 1. the car: lane 0's word 0 decides the failure
      const int fail0 = event(ws[0], sm.t_fail) ? 1 : 0;
      const bool fail = __shfl_sync(0xffffffffu, fail0, in_group ? g0 : lane) != 0;
      if (active && !fail) {
        if (a == 1 && level < 4u) level += 1u;
        if (a == 2 && level > 0u) level -= 1u;
      }
      const float v = 0.5f * (float)level;
      if (active) xc = xc + v * 0.25f;
      // 2. pedestrians, 3. collision
      bool hit = false;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int p = (int)(W * q) + k - 1;
        if (active && p >= 0 && p < P) {
          const float2 cs = sm.rot[car_noise_index(ws[k])];
          car_ped_move(px[k], py[k], goal[k], cs.x, cs.y);
          const float dx = px[k] - xc;
          hit = hit || (dx * dx + py[k] * py[k] < 1.0f);
        }
      }
      const bool coll = (__ballot_sync(0xffffffffu, hit) & gmask) != 0u;
      const bool g = xc >= 20.0f;  // 4. goal
      r = car_reward(a, coll, g, v);
      if (active) term = coll || g;
    };
    float r0 = 0.0f;
    const bool live0 = valid && !term;
    step(live0, (int)a0, lf.depth + 1, r0);
    if (!live0) r0 = 0.0f;
    if (live0 && q == 0) ++steps_acc;
    // the child's key: this lane's words Wq .. Wq+W-1 (word 0: the car)
    uint64_t hk = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t w = W * q + (uint32_t)k;
      if (valid && w < OW) {
        const int p = (int)w - 1;
        uint32_t zw;
        if (term) zw = w == 0 ? kCarTerminalWord0 : 0u;
        else if (w == 0) zw = car_bin(xc) | (level << 16);
        else zw = car_bin(px[k]) | (car_bin(py[k]) << 16);
        (void)p;
        io.keys[t * OW + w] = zw;
        if (RECORD) b.scen_obs[t * OW + w] = zw;
        hk ^= key_mix(zw, w);
      }
    }
    {  // XOR over the group (the group's lanes in turn)
      uint64_t tot = 0;
      for (uint32_t k = 0; k < G; ++k) tot ^= __shfl_sync(0xffffffffu, hk, in_group ? g0 + k : lane);
      hk = tot;
    }
    if (valid && q == 0) io.hash[t] = hk;
    if (RECORD && valid && b.scen_states) {
      uint32_t* dst = b.scen_states + t * SW;
      if (q == 0) {
        dst[0] = __float_as_uint(xc);
        dst[1] = level | ((uint32_t)term << 8);
        dst[2] = lf.states[2 * cap + i];
        dst[3] = lf.states[3 * cap + i];
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int p = (int)(W * q) + k - 1;
        if (p >= 0 && p < P) {
          dst[4 + 2 * p] = __float_as_uint(px[k]);
          dst[5 + 2 * p] = __float_as_uint(py[k]);
        }
      }
    }
    double u = 0.0, lam = 0.0;
    uint32_t len = 0;
    uint64_t h = kFnvOffset;
    const bool rolled = valid && !term;  // a roll-out from the non-terminal child state
    bool live = rolled;
    if (live) {
      int k = (int)ceilf((20.0f - xc) * 2.0f);
      k = k < 1 ? 1 : k;
      u = 100.0 * sm.gpow[k - 1];  // Eq. 11
    }
    // roll-out (Eq. 12): pi0 reads the last observation's bins
    const uint32_t t0 = lf.depth + 1;
    uint32_t tt = t0;
    double acc = 0.0;
    live = live && tt < sm.D;
    while (__any_sync(0xffffffffu, live)) {
      const int cxb = car_bin_i(xc);
      int gap = 255;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int p = (int)(W * q) + k - 1;
        if (p >= 0 && p < P) {
          const int pxb = car_bin_i(px[k]), pyb = car_bin_i(py[k]);
          if (pxb >= cxb && pyb >= -4 && pyb <= 3 && pxb - cxb < gap) gap = pxb - cxb;
        }
      }
      for (uint32_t k = 0; k < G; ++k) gap = min(gap, __shfl_sync(0xffffffffu, gap, in_group ? g0 + k : lane));
      const int a = car_policy_from_gap(gap);
      if (RECORD && live) h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
      float r;
      step(live, a, tt + 1, r);
      if (live) {
        acc += sm.gpow[tt - t0] * (double)r;
        ++tt;
        live = !term && tt < sm.D;
      }
    }
    if (rolled) {
      if (!term) acc += sm.gpow[tt - t0] * sm.tail;  // reached D non-terminal
      lam = acc;
      len = tt - t0;
    }
    if (valid && q == 0) {
      steps_acc += len;
      const double wn = (double)lf.w[i] * lf.inv_wroot;
      const double fx = dm.fx, gamma = dm.gamma;
      io.q3[3 * t + 0] = fxq(wn, fx);
      io.q3[3 * t + 1] = fxq(wn * u, fx);
      io.q3[3 * t + 2] = fxq(wn * lam, fx);
      const uint64_t la = (uint64_t)leaf * b.A + a0;
      red_add(&b.sums[lay.Q(la, 0)], fxq(wn * (double)r0, fx));
      red_add(&b.sums[lay.Q(la, 1)], fxq(wn * ((double)r0 + gamma * u), fx));
      red_add(&b.sums[lay.Q(la, 2)], fxq(wn * ((double)r0 + gamma * lam), fx));
      if (RECORD) {
        b.scen_reward[t] = r0;
        b.scen_upper[t] = (float)u;
        b.scen_lower[t] = (float)lam;
        b.scen_len[t] = len;
        b.scen_hash[t] = h;
      }
    }
  }
  const uint32_t ws = warp_sum32(steps_acc);
  if (lane == 0 && ws) atomicAdd((unsigned long long*)&b.sums[lay.steps()], (unsigned long long)ws);
}

// ---------------------------------------------------------------------------
// K3s: group the items of one (leaf, action) by key (first occurrence).  An
// open-addressing table in shared memory (2^k >= 2n slots) maps each 64-bit
// key hash to the smallest item position carrying it (atomicMin), so the
// representative of every item is found in O(1) probes; each item's full key
// is then compared with its representative's (a hash collision is an error,
// never a merge), representatives get their ordinal by a block scan in item
// order (= first-occurrence order, R8), and every item adds its exact
// fixed-point contributions to its child's row of the exchange block.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k3_group_sparse(BatchDev b, SparseItemOut io, uint32_t tbits,
                                                       int64_t* xmax) {
  extern __shared__ __align__(16) unsigned char gs_smem[];
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t tsize = 1u << tbits, tmask = tsize - 1u;
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(gs_smem);  // [tsize]
  uint32_t* titem = reinterpret_cast<uint32_t*>(tkey + tsize);              // [tsize]
  const uint64_t la = blockIdx.x;
  const uint32_t leaf = (uint32_t)(la / b.A), a = (uint32_t)(la - (uint64_t)leaf * b.A);
  const uint32_t n = b.n_leaf[leaf];
  const uint64_t q0 = b.scen_off[leaf] + (uint64_t)a * n;
  const uint32_t OW = b.model->OW;
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  const uint64_t base = la * b.S;
  __shared__ uint64_t wsum[32];
  constexpr unsigned long long kEmpty = 0ull;  // hash 0 is remapped to 1
  uint32_t* ord = titem + tsize;  // [n] child ordinal of a representative
  for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x) {
    tkey[s] = kEmpty;
    titem[s] = 0xFFFFFFFFu;
  }
  __syncthreads();
  // 1. insert: slot of the hash, minimum item position per hash
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long h = io.hash[q0 + i];
    h = h ? h : 1ull;
    uint32_t s = (uint32_t)(h ^ (h >> 32)) & tmask;
    for (;;) {
      const unsigned long long prev = atomicCAS(&tkey[s], kEmpty, h);
      if (prev == kEmpty || prev == h) break;
      s = (s + 1u) & tmask;
    }
    atomicMin(&titem[s], i);
  }
  __syncthreads();
  // 2. representative, exact-key check, ordinal of the representatives
  uint32_t run = 0;
  for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const uint32_t i = c0 + threadIdx.x;
    uint32_t is_rep = 0, rep = 0;
    if (i < n) {
      unsigned long long h = io.hash[q0 + i];
      h = h ? h : 1ull;
      uint32_t s = (uint32_t)(h ^ (h >> 32)) & tmask;
      while (tkey[s] != h) s = (s + 1u) & tmask;
      rep = titem[s];
      is_rep = rep == i;
      if (!is_rep) {
        const uint32_t* ki = io.keys + (q0 + i) * OW;
        const uint32_t* kj = io.keys + (q0 + rep) * OW;
        for (uint32_t k = 0; k < OW; ++k)
          if (ki[k] != kj[k]) atomicOr(b.err, kErrHash);
      }
    }
    uint64_t tot;
    const uint64_t before = block_excl_scan(is_rep, wsum, tot);
    if (i < n && is_rep) ord[i] = run + (uint32_t)before;
    run += (uint32_t)tot;
  }
  __syncthreads();
  // 3. exact sums per child
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long h = io.hash[q0 + i];
    h = h ? h : 1ull;
    uint32_t s = (uint32_t)(h ^ (h >> 32)) & tmask;
    while (tkey[s] != h) s = (s + 1u) & tmask;
    const uint32_t rep = titem[s];
    const uint32_t c = ord[rep];
    const uint64_t slot = base + c;
    red_add(&b.sums[lay.W(slot)], io.q3[3 * (q0 + i) + 0]);
    red_add(&b.sums[lay.U(slot)], io.q3[3 * (q0 + i) + 1]);
    red_add(&b.sums[lay.Lm(slot)], io.q3[3 * (q0 + i) + 2]);
    red_add(&b.sums[lay.N(slot)], (int64_t)1);
    if (rep == i) {
      b.mins[slot] = (int32_t)b.leaves[leaf].ids[i];
      b.rank[slot] = c;
      b.sp_item[slot] = (uint32_t)(q0 + i);
    }
  }
  if (threadIdx.x == 0) {
    b.nc[la] = run;
    if (xmax) {  // sharded: this rank's record count and largest child set
      atomicAdd((unsigned long long*)&xmax[0], (unsigned long long)run);
      atomicMax((unsigned long long*)&xmax[1], (unsigned long long)run);
    }
  }
}

// K3c for sparse keys: one CTA per (leaf, action), one thread per child
// (children are already in first-occurrence order)
constexpr uint32_t kWriteSparseThreads = 512;  // a warp per 32 children: one round for ~500 children
__global__ void __launch_bounds__(kWriteSparseThreads) k3_write_sparse(BatchDev b, SparseItemOut io) {
  __shared__ int64_t s_wt[kWriteSparseThreads / 32], s_nt[kWriteSparseThreads / 32];
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t A = b.A;
  const uint64_t LA = (uint64_t)b.L * A;
  const uint64_t la = blockIdx.x;
  const uint32_t leaf = (uint32_t)(la / A), a = (uint32_t)(la - (uint64_t)leaf * A);
  const LeafDev& lf = b.leaves[leaf];
  const DevModel& dm = *b.model;
  const uint32_t OW = dm.OW;
  const SumLayout lay{LA * b.S, LA};
  const uint64_t base = la * b.S;
  const uint32_t cb = b.child_begin[la];
  const uint32_t nc = b.nc[la];
  int64_t wt = 0, nt = 0;
  const uint32_t lane = threadIdx.x & 31, nwc = blockDim.x >> 5;
  // a warp per 32 children: the scalar outputs a lane per child, then the
  // children's keys (OW <= 32 words each) copied a child at a time, a lane
  // per word, so that the key reads and both key writes are contiguous
  for (uint32_t c0 = (threadIdx.x >> 5) * 32; c0 < nc; c0 += nwc * 32) {
    const uint32_t c = c0 + lane;
    uint32_t item = 0;
    if (c < nc) {
      const int64_t N = b.sums[lay.N(base + c)];
      const int64_t W = b.sums[lay.W(base + c)];
      wt += W;
      nt += N;
      item = b.sp_item[base + c];
      const uint32_t oc = cb + c;
      if (oc < b.child_capacity) {
        const double Wd = (double)W;
        b.child_count[oc] = (uint32_t)N;
        b.child_first[oc] = (uint32_t)b.mins[base + c];
        b.child_weight[oc] = (float)(Wd * dm.inv_fx * lf.wroot);
        b.child_upper[oc] = (float)((double)b.sums[lay.U(base + c)] / Wd);
        b.child_lower[oc] = (float)((double)b.sums[lay.Lm(base + c)] / Wd);
      }
    }
    const uint32_t cn = nc - c0 < 32 ? nc - c0 : 32;
    for (uint32_t j0 = 0; j0 < cn; j0 += 16) {  // sixteen children's loads in flight, then their stores
      uint32_t v[16];
#pragma unroll
      for (uint32_t u = 0; u < 16; ++u) {
        const uint32_t j = j0 + u, it = __shfl_sync(0xffffffffu, item, j & 31u);
        v[u] = (j < cn && lane < OW) ? __ldcg(&io.keys[(uint64_t)it * io.kstride + lane]) : 0u;
      }
#pragma unroll
      for (uint32_t u = 0; u < 16; ++u) {
        const uint32_t cj = c0 + j0 + u;
        if (j0 + u < cn && lane < OW) {
          if (cb + cj < b.child_capacity) b.child_obs[(uint64_t)(cb + cj) * OW + lane] = v[u];
          if (cj < lf.kcap) lf.keys[((uint64_t)a * lf.kcap + cj) * OW + lane] = v[u];
        }
      }
    }
  }
  wt = warp_sum64(wt);
  nt = warp_sum64(nt);
  if ((threadIdx.x & 31) == 0) {
    s_wt[threadIdx.x >> 5] = wt;
    s_nt[threadIdx.x >> 5] = nt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) {
      wt += s_wt[w];
      nt += s_nt[w];
    }
    lf.nchild[a] = nc;
    const double Wd = (double)wt;
    b.act_reward[la] = (float)((double)b.sums[lay.Q(la, 0)] / Wd);
    b.act_upper[la] = (float)((double)b.sums[lay.Q(la, 1)] / Wd);
    b.act_lower[la] = (float)((double)b.sums[lay.Q(la, 2)] / Wd);
    if (a == 0) {
      b.n_scen[leaf] = (uint32_t)nt;
      b.weight[leaf] = (float)(Wd * dm.inv_fx * lf.wroot);
      if (nt == 0) atomicOr(b.err, kErrEmptyLeaf);
    }
  }
}

// ---------------------------------------------------------------------------
// Scenario-sharded sparse keys (world > 1).  Every rank groups
// its own scenarios (k3_group_sparse), packs its local children as fixed-size
// records into its block of an all-gather buffer, the caller all-gathers the
// blocks, and every rank merges the same P blocks the same way: records with
// equal keys are one child (exact compare; the 64-bit hash only indexes),
// the child's sums are exact int64 sums, its first id the minimum, and the
// children are ordered by first id -- the world == 1 result, bit for bit.
//
// block of rank r: [nc[L*A] u32 | pad to hdr_pad | records, (leaf, action)-major]
// record: hash u64 | N, W, U, LAMBDA i64 | first i32 | key[OW] u32 (8-aligned)
// ---------------------------------------------------------------------------
constexpr uint32_t kRecN = 8, kRecFirst = 40, kRecKey = 44;
__host__ __device__ inline uint32_t sparse_record_bytes(uint32_t OW) { return (kRecKey + 4 * OW + 7) & ~7u; }

struct PackDev {
  unsigned char* blk;  // this rank's block
  uint32_t hdr_pad, rec_bytes;
  uint32_t* loc_off;   // [L*A] record offset of each (leaf, action)
  uint64_t blk_bytes;  // the block's size (self-checks)
};
// header + record offsets (one CTA)
__global__ void __launch_bounds__(1024) k_pack_sparse_scan(BatchDev b, PackDev p) {
  __shared__ uint64_t wsum[32];
  const uint64_t LA = (uint64_t)b.L * b.A;
  const uint64_t per = (LA + blockDim.x - 1) / blockDim.x, i0 = (uint64_t)threadIdx.x * per;
  uint64_t loc = 0;
  for (uint64_t i = i0; i < i0 + per && i < LA; ++i) loc += b.nc[i];
  uint64_t tot;
  uint64_t run = block_excl_scan(loc, wsum, tot);
  uint32_t* hdr = reinterpret_cast<uint32_t*>(p.blk);
  for (uint64_t i = i0; i < i0 + per && i < LA; ++i) {
    p.loc_off[i] = (uint32_t)run;
    hdr[i] = b.nc[i];
    run += b.nc[i];
  }
}
// records: one CTA per (leaf, action)
__global__ void __launch_bounds__(128) k_pack_sparse(BatchDev b, SparseItemOut io, PackDev p) {
  const uint64_t la = blockIdx.x;
  const uint32_t OW = b.model->OW;
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  const uint64_t base = la * b.S;
  const uint32_t nc = b.nc[la];
  for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
    unsigned char* r = p.blk + p.hdr_pad + (uint64_t)(p.loc_off[la] + c) * p.rec_bytes;
    HD_CHECK(b.err, p.hdr_pad + (uint64_t)(p.loc_off[la] + c + 1) * p.rec_bytes <= p.blk_bytes);
    const uint32_t it = b.sp_item[base + c];
    int64_t* q = reinterpret_cast<int64_t*>(r + kRecN);
    *reinterpret_cast<uint64_t*>(r) = io.hash[it];
    q[0] = b.sums[lay.N(base + c)];
    q[1] = b.sums[lay.W(base + c)];
    q[2] = b.sums[lay.U(base + c)];
    q[3] = b.sums[lay.Lm(base + c)];
    *reinterpret_cast<int32_t*>(r + kRecFirst) = b.mins[base + c];
    uint32_t* key = reinterpret_cast<uint32_t*>(r + kRecKey);
    for (uint32_t k = 0; k < OW; ++k) key[k] = io.keys[(uint64_t)it * OW + k];
  }
}

struct MergeDev {
  const unsigned char* gbuf;  // world blocks
  uint64_t blk;               // bytes per block
  uint32_t hdr_pad, rec_bytes, world;
  uint32_t* offs;             // [world][L*A] record offset of (rank, leaf, action)
};
constexpr uint32_t kMaxMergeWorld = 64;
// per-rank record offsets of every (leaf, action) (one CTA, ranks in turn)
__global__ void __launch_bounds__(1024) k_merge_offsets(BatchDev b, MergeDev g) {
  __shared__ uint64_t wsum[32];
  const uint64_t LA = (uint64_t)b.L * b.A;
  const uint64_t per = (LA + blockDim.x - 1) / blockDim.x, i0 = (uint64_t)threadIdx.x * per;
  for (uint32_t r = 0; r < g.world; ++r) {
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(g.gbuf + r * g.blk);
    uint64_t loc = 0;
    for (uint64_t i = i0; i < i0 + per && i < LA; ++i) loc += hdr[i];
    uint64_t tot;
    uint64_t run = block_excl_scan(loc, wsum, tot);
    for (uint64_t i = i0; i < i0 + per && i < LA; ++i) {
      g.offs[r * LA + i] = (uint32_t)run;
      run += hdr[i];
    }
  }
}
// one CTA per (leaf, action): union of the ranks' records -> global children
// in b.sums/mins/sp_item/nc (b.S = merged row capacity); sp_item holds the
// representative's record index in gbuf units of rec_bytes
__global__ void __launch_bounds__(512) k3_merge_sparse(BatchDev b, MergeDev g, uint32_t tbits) {
  extern __shared__ __align__(16) unsigned char mg_smem[];
  const uint32_t tsize = 1u << tbits, tmask = tsize - 1u;
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(mg_smem);  // [tsize]
  unsigned long long* trep = tkey + tsize;                                     // [tsize] (first << 32 | item)
  __shared__ uint32_t rs[kMaxMergeWorld + 1], nrep;
  const uint64_t LA = (uint64_t)b.L * b.A;
  const uint64_t la = blockIdx.x;
  const uint32_t OW = b.model->OW;
  const SumLayout lay{LA * b.S, LA};
  const uint64_t base = la * b.S;
  if (threadIdx.x == 0) {
    rs[0] = 0;
    for (uint32_t r = 0; r < g.world; ++r)
      rs[r + 1] = rs[r] + reinterpret_cast<const uint32_t*>(g.gbuf + r * g.blk)[la];
    nrep = 0;
  }
  for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x) {
    tkey[s] = 0ull;
    trep[s] = ~0ull;
  }
  __syncthreads();
  const uint32_t n = rs[g.world];
  uint32_t* ord = reinterpret_cast<uint32_t*>(trep + tsize);  // [n] ordinal of a representative
  int32_t* rfirst = reinterpret_cast<int32_t*>(ord + n);      // [n] representatives' first ids
  uint32_t* ritem = reinterpret_cast<uint32_t*>(rfirst + n);  // [n] representatives' items
  auto rec_index = [&](uint32_t i) -> uint64_t {  // global record index of item i
    uint32_t r = 0;
    while (rs[r + 1] <= i) ++r;
    return (r * g.blk + g.hdr_pad) / g.rec_bytes + g.offs[r * LA + la] + (i - rs[r]);
  };
  auto rec = [&](uint64_t gi) {
    HD_CHECK(b.err, (gi + 1) * g.rec_bytes <= g.world * g.blk);
    return g.gbuf + gi * g.rec_bytes;
  };
  auto slot_of = [&](unsigned long long h) {
    uint32_t s = (uint32_t)(h ^ (h >> 32)) & tmask;
    while (tkey[s] != h) s = (s + 1u) & tmask;
    return s;
  };
  // 1. insert: per hash, the item with the smallest first id
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned char* r = rec(rec_index(i));
    unsigned long long h = *reinterpret_cast<const unsigned long long*>(r);
    h = h ? h : 1ull;
    uint32_t s = (uint32_t)(h ^ (h >> 32)) & tmask;
    for (;;) {
      const unsigned long long prev = atomicCAS(&tkey[s], 0ull, h);
      if (prev == 0ull || prev == h) break;
      s = (s + 1u) & tmask;
    }
    const uint32_t first = (uint32_t)*reinterpret_cast<const int32_t*>(r + kRecFirst);
    atomicMin(&trep[s], ((unsigned long long)first << 32) | i);
  }
  __syncthreads();
  // 2. representatives; every other item's key must equal its representative's
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t gi = rec_index(i);
    const unsigned char* r = rec(gi);
    unsigned long long h = *reinterpret_cast<const unsigned long long*>(r);
    const unsigned long long t = trep[slot_of(h ? h : 1ull)];
    const uint32_t rep = (uint32_t)t;
    if (rep == i) {
      const uint32_t j = atomicAdd(&nrep, 1u);
      rfirst[j] = (int32_t)(t >> 32);
      ritem[j] = i;
    } else {
      const uint32_t* ki = reinterpret_cast<const uint32_t*>(r + kRecKey);
      const uint32_t* kj = reinterpret_cast<const uint32_t*>(rec(rec_index(rep)) + kRecKey);
      for (uint32_t k = 0; k < OW; ++k)
        if (ki[k] != kj[k]) atomicOr(b.err, kErrHash);
    }
  }
  __syncthreads();
  // 3. ordinal = number of representatives with a smaller first id (R8)
  const uint32_t nr = nrep;
  for (uint32_t j = threadIdx.x; j < nr; j += blockDim.x) {
    const int32_t f = rfirst[j];
    uint32_t o = 0;
    for (uint32_t q = 0; q < nr; ++q) o += rfirst[q] < f;
    ord[ritem[j]] = o;
  }
  __syncthreads();
  // 4. exact sums per global child
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t gi = rec_index(i);
    const unsigned char* r = rec(gi);
    unsigned long long h = *reinterpret_cast<const unsigned long long*>(r);
    const uint32_t rep = (uint32_t)trep[slot_of(h ? h : 1ull)];
    const uint64_t slot = base + ord[rep];
    const int64_t* q = reinterpret_cast<const int64_t*>(r + kRecN);
    atomicAdd((unsigned long long*)&b.sums[lay.N(slot)], (unsigned long long)q[0]);
    atomicAdd((unsigned long long*)&b.sums[lay.W(slot)], (unsigned long long)q[1]);
    atomicAdd((unsigned long long*)&b.sums[lay.U(slot)], (unsigned long long)q[2]);
    atomicAdd((unsigned long long*)&b.sums[lay.Lm(slot)], (unsigned long long)q[3]);
    if (rep == i) {
      b.mins[slot] = *reinterpret_cast<const int32_t*>(r + kRecFirst);
      b.sp_item[slot] = (uint32_t)gi;
    }
  }
  if (threadIdx.x == 0) b.nc[la] = nr;
}

// ---------------------------------------------------------------------------
// RECORD: each scenario's child ordinal under its (leaf, action) (the
// per-scenario observations' children of P:434), after the finalize.  Dense
// keys: the number of the (leaf, action)'s used slots with a smaller first id
// than the record's slot; sparse keys: the child whose key equals the record's.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k3_scen_child(BatchDev b, uint32_t dense) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint64_t Q = b.scen_off[b.L];
  const uint32_t OW = b.model->OW;
  const uint64_t LA = (uint64_t)b.L * b.A;
  const SumLayout lay{LA * b.S, LA};
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q && q < b.scen_capacity;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t leaf = find_leaf(b.scen_off, b.L, q);
    const uint32_t n = b.n_leaf[leaf];
    const uint32_t a = (uint32_t)((q - b.scen_off[leaf]) / n);
    const uint64_t la = (uint64_t)leaf * b.A + a;
    uint32_t c = 0xFFFFFFFFu;
    if (dense) {
      const uint64_t base = la * b.S;
      const uint32_t z = b.scen_obs[q];
      const int32_t f = b.mins[base + z];
      uint32_t r = 0;
      for (uint32_t s = 0; s < b.S; ++s) r += (b.sums[lay.N(base + s)] != 0 && b.mins[base + s] < f) ? 1u : 0u;
      c = r;
    } else {
      const uint32_t cb = b.child_begin[la], ce = b.child_begin[la + 1];
      for (uint32_t k = cb; k < ce && k < b.child_capacity; ++k) {
        bool eq = true;
        for (uint32_t w = 0; w < OW && eq; ++w) eq = b.child_obs[(uint64_t)k * OW + w] == b.scen_obs[q * OW + w];
        if (eq) {
          c = k - cb;
          break;
        }
      }
    }
    b.scen_child[q] = c;
  }
}

}  // namespace hd
