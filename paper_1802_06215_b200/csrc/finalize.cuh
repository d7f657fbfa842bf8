// finalize.cuh -- K2pre (tile prefix), K3a/K3b/K3c (child order, CSR scan,
// outputs) for dense observation keys.
#pragma once
#include "common.cuh"

namespace hd {

// block-wide exclusive scan of one u64 per thread (blockDim.x <= 1024)
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* wsum, uint64_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t s = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) wsum[lane] = s;
  }
  __syncthreads();
  const uint64_t before = (wid ? wsum[wid - 1] : 0) + x - v;
  total = wsum[nw - 1];
  __syncthreads();
  return before;
}

// per-leaf prefixes: tile_off[l] = sum_{l'<l} A ceil(n_l'/32) (K2 warp tiles),
// scen_off[l] = sum_{l'<l} A n_l' (per-scenario records).  Whole CTA.
__device__ __forceinline__ void leaf_prefix(const BatchDev& b, uint64_t* wsum) {
  const uint32_t per = (b.L + blockDim.x - 1) / blockDim.x;
  const uint32_t l0 = threadIdx.x * per;
  uint64_t tiles = 0, scen = 0;
  for (uint32_t l = l0; l < l0 + per && l < b.L; ++l) {
    const uint64_t n = __ldcg(&b.n_leaf[l]);
    tiles += (uint64_t)b.A * ((n + 31) >> 5);
    scen += (uint64_t)b.A * n;
  }
  uint64_t ttot, stot;
  uint64_t tb = block_excl_scan(tiles, wsum, ttot);
  uint64_t sb = block_excl_scan(scen, wsum, stot);
  for (uint32_t l = l0; l < l0 + per && l < b.L; ++l) {
    b.tile_off[l] = (uint32_t)tb;
    b.scen_off[l] = sb;
    const uint64_t n = __ldcg(&b.n_leaf[l]);
    tb += (uint64_t)b.A * ((n + 31) >> 5);
    sb += (uint64_t)b.A * n;
  }
  if (threadIdx.x == 0) {
    b.tile_off[b.L] = (uint32_t)ttot;
    b.scen_off[b.L] = stot;
    if (ttot >= 0xFFFFFFFFull) atomicOr(b.err, kErrChildCap);
  }
}
__global__ void __launch_bounds__(1024) k2_prefix(BatchDev b) {
  __shared__ uint64_t wsum[32];
  leaf_prefix(b, wsum);
}
// the last CTA of a grid to arrive runs `leaf_prefix` (threadfence reduction)
__device__ __forceinline__ void last_cta_prefix(const BatchDev& b) {
  __shared__ bool am_last;
  __shared__ uint64_t wsum[32];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    am_last = atomicAdd(&b.status[kStatK1Ticket], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    leaf_prefix(b, wsum);
  }
}

// K3a body: child ordinal of each non-empty slot of (leaf, action) la =
// number of non-empty slots with a smaller first id (first occurrence, R8).
// The non-empty slots are compacted first (ballot prefix), so the cost is
// S/32 + c^2/32 per lane for c children instead of S^2/32.
__device__ __forceinline__ void rank_one(const BatchDev& b, uint64_t la, uint32_t lane, int32_t* s_first,
                                         uint32_t* nc_out) {
  const uint32_t S = b.S;
  const uint64_t LA = (uint64_t)b.L * b.A;
  const SumLayout lay{LA * S, LA};
  const uint64_t base = la * S;
  uint32_t* s_slot = reinterpret_cast<uint32_t*>(s_first + S);
  uint32_t cnt = 0;
  for (uint32_t s0 = 0; s0 < S; s0 += 32) {
    const uint32_t s = s0 + lane;
    const bool ne = s < S && __ldcg(&b.sums[lay.N(base + s)]) != 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, ne);
    if (ne) {
      const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
      s_first[pos] = __ldcg(&b.mins[base + s]);
      s_slot[pos] = s;
    }
    cnt += __popc(bal);
  }
  __syncwarp();
  HD_CHECK(b.err, cnt <= S);
  for (uint32_t i = lane; i < cnt; i += 32) {
    const int32_t f = s_first[i];
    uint32_t r = 0;
    for (uint32_t q = 0; q < cnt; ++q) r += s_first[q] < f;
    b.rank[base + s_slot[i]] = r;
  }
  if (lane == 0) *nc_out = cnt;
  __syncwarp();
}
__global__ void __launch_bounds__(128) k3_rank_dense(BatchDev b) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char k3_smem[];
  const uint32_t wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t la = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (la >= (uint64_t)b.L * b.A) return;
  rank_one(b, la, lane, reinterpret_cast<int32_t*>(k3_smem) + (size_t)wid * 2 * b.S, &b.nc[la]);
}

// K3b as a multi-CTA scan with decoupled look-back: each CTA takes the next
// tile of kScanTile counts (an atomic ticket, so every tile it waits on is
// already running), publishes its aggregate, walks back over its
// predecessors' published words until an inclusive prefix, and publishes its
// own inclusive prefix (flag 2).  A (flag, value) pair is one 64-bit word.
constexpr uint32_t kScanTile = 1024;
__global__ void __launch_bounds__(kScanTile) k3_scan_lookback(BatchDev b) {
  __shared__ uint64_t wsum[32];
  __shared__ uint32_t tile_sh;
  __shared__ uint64_t excl_sh;
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kVal = (1ull << 62) - 1;
  const uint64_t LA = (uint64_t)b.L * b.A;
  if (threadIdx.x == 0) tile_sh = (uint32_t)atomicAdd(&b.scan_flags[0], 1ull);
  __syncthreads();
  const uint32_t tile = tile_sh;
  HD_CHECK(b.err, (uint64_t)tile * kScanTile < LA + kScanTile);  // one ticket per CTA
  const uint64_t i = (uint64_t)tile * kScanTile + threadIdx.x;
  const uint32_t v = i < LA ? b.nc[i] : 0u;
  uint64_t tot;
  const uint64_t pre = block_excl_scan(v, wsum, tot);
  unsigned long long* st = b.scan_flags + 1;
  if (threadIdx.x == 0) {
    uint64_t excl = 0;
    if (tile == 0) {
      atomicExch(&st[0], kIncl | tot);
    } else {
      atomicExch(&st[tile], kAgg | tot);
      for (int p = (int)tile - 1;;) {
        HD_CHECK(b.err, p >= 0);  // tile 0 always publishes an inclusive prefix
        const unsigned long long f = atomicAdd(&st[p], 0ull);  // device-scope read
        if (!(f >> 62)) continue;                               // predecessor not published yet
        excl += f & kVal;
        if ((f >> 62) == 2) break;                              // an inclusive prefix: done
        --p;
      }
      atomicExch(&st[tile], kIncl | (excl + tot));
    }
    excl_sh = excl;
  }
  __syncthreads();
  if (i < LA) b.child_begin[i] = (uint32_t)(excl_sh + pre);
  if (threadIdx.x == 0 && (uint64_t)(tile + 1) * kScanTile >= LA) {  // the last tile: totals
    const uint64_t total = excl_sh + tot;
    b.child_begin[LA] = (uint32_t)total;
    if (total > b.child_capacity) atomicOr(b.err, kErrChildCap);
    b.status[1] = (uint32_t)total;
    const uint64_t steps = (uint64_t)__ldcg(&b.sums[SumLayout{LA * b.S, LA}.steps()]);
    b.status[2] = (uint32_t)steps;
    b.status[3] = (uint32_t)(steps >> 32);
  }
}

// K3c body: outputs of (leaf, action) la: Eq. 11/12 child bounds, one-level
// Eq. 4, and the leaf's child-key table
__device__ __forceinline__ void write_one(const BatchDev& b, uint64_t la, uint32_t lane, uint32_t cb, uint32_t nc) {
  const uint32_t S = b.S, A = b.A;
  const uint64_t LA = (uint64_t)b.L * A;
  const uint32_t leaf = (uint32_t)(la / A), a = (uint32_t)(la - (uint64_t)leaf * A);
  const LeafDev& lf = b.leaves[leaf];
  const DevModel& dm = *b.model;
  const SumLayout lay{LA * S, LA};
  const uint64_t base = la * S;
  int64_t wt = 0, nt = 0;
  for (uint32_t s = lane; s < S; s += 32) {
    const int64_t N = __ldcg(&b.sums[lay.N(base + s)]);
    if (!N) continue;
    const int64_t W = __ldcg(&b.sums[lay.W(base + s)]);
    wt += W;
    nt += N;
    const uint32_t rk = b.rank[base + s];
    const uint32_t c = cb + rk;
    HD_CHECK(b.err, rk < nc && rk < S);
    if (c < b.child_capacity) {
      const double Wd = (double)W;
      b.child_count[c] = (uint32_t)N;
      b.child_first[c] = (uint32_t)__ldcg(&b.mins[base + s]);
      b.child_weight[c] = (float)(Wd * dm.inv_fx * lf.wroot);
      b.child_upper[c] = (float)((double)__ldcg(&b.sums[lay.U(base + s)]) / Wd);
      b.child_lower[c] = (float)((double)__ldcg(&b.sums[lay.Lm(base + s)]) / Wd);
      b.child_obs[c] = s;
    }
    if (rk < lf.kcap) lf.keys[(uint64_t)a * lf.kcap + rk] = s;  // key table for later updates
  }
  wt = warp_sum64(wt);
  nt = warp_sum64(nt);
  if (lane == 0) {
    lf.nchild[a] = nc;
    const double Wd = (double)wt;
    b.act_reward[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 0)]) / Wd);
    b.act_upper[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 1)]) / Wd);
    b.act_lower[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 2)]) / Wd);
    if (a == 0) {
      b.n_scen[leaf] = (uint32_t)nt;
      b.weight[leaf] = (float)(Wd * dm.inv_fx * lf.wroot);
      if (nt == 0) atomicOr(b.err, kErrEmptyLeaf);
    }
  }
}
__global__ void __launch_bounds__(128) k3_write_dense(BatchDev b) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t la = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (la >= (uint64_t)b.L * b.A) return;
  write_one(b, la, lane, b.child_begin[la], b.nc[la]);
}
// S rounded up to a power of two: the lanes of one (leaf, action) in the
// lane-per-slot finalize kernels
__host__ __device__ inline uint32_t small_group_width(uint32_t S) {
  uint32_t sp = 1;
  while (sp < S) sp <<= 1;
  return sp;
}

// K3a for few observation slots (S <= 16): only the child count of each
// (leaf, action) -- k3_write_grouped recomputes the ordinals -- a lane per
// slot, 32/S' pairs per warp
__global__ void __launch_bounds__(128) k3_count_grouped(BatchDev b) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t lane = threadIdx.x & 31, S = b.S, LA = b.L * b.A;
  const uint32_t Sp = small_group_width(S);
  const uint32_t j = lane & (Sp - 1), gshift = lane & ~(Sp - 1);
  const uint32_t gbits = Sp == 32 ? 0xffffffffu : (1u << Sp) - 1u;
  const uint32_t la = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / Sp) + lane / Sp;
  if ((la - lane / Sp) >= LA) return;  // warp-uniform
  const SumLayout lay{(uint64_t)LA * S, LA};
  const bool ne = la < LA && j < S && b.sums[lay.N((uint64_t)la * S + j)] != 0;
  const uint32_t gb = (__ballot_sync(0xffffffffu, ne) >> gshift) & gbits;
  if (j == 0 && la < LA) b.nc[la] = __popc(gb);
}

// K3c for few observation slots (S <= 16: RockSample/MARS, Tiger): a lane per
// slot and 32/S' (leaf, action) pairs per warp (S' = S rounded up to a power
// of two), the child ordinals recomputed in registers from the first ids
// (the rank array is not read), every load of a pair issued at once
__global__ void __launch_bounds__(128) k3_write_grouped(BatchDev b) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t lane = threadIdx.x & 31, S = b.S, A = b.A;
  const uint32_t LA = b.L * A;
  const uint32_t Sp = small_group_width(S), G = 32 / Sp;
  const uint32_t j = lane & (Sp - 1), gshift = lane & ~(Sp - 1);
  const uint32_t gbits = Sp == 32 ? 0xffffffffu : (1u << Sp) - 1u;
  const uint32_t la = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G + lane / Sp;
  if ((la - lane / Sp) >= LA) return;  // warp-uniform
  const SumLayout lay{(uint64_t)LA * S, LA};
  const bool v = la < LA && j < S;
  const uint64_t slot = (uint64_t)la * S + j;
  const int64_t N = v ? b.sums[lay.N(slot)] : 0;
  const int64_t W = v ? b.sums[lay.W(slot)] : 0;
  const int64_t U = v ? b.sums[lay.U(slot)] : 0;
  const int64_t Lm = v ? b.sums[lay.Lm(slot)] : 0;
  const int32_t mn = v ? b.mins[slot] : 0;
  const bool q = la < LA && j == 0;
  const int64_t Q0 = q ? b.sums[lay.Q(la, 0)] : 0, Q1 = q ? b.sums[lay.Q(la, 1)] : 0,
                Q2 = q ? b.sums[lay.Q(la, 2)] : 0;
  const uint32_t cb = la < LA ? b.child_begin[la] : 0;
  const bool ne = N != 0;
  const uint32_t gb = (__ballot_sync(0xffffffffu, ne) >> gshift) & gbits;
  uint32_t rk = 0;  // first occurrence (R8): non-empty slots with a smaller first id
  for (uint32_t k = 0; k < Sp; ++k) {
    const int32_t mk = __shfl_sync(0xffffffffu, mn, k, Sp);
    rk += ((gb >> k) & 1u) && mk < mn;
  }
  int64_t wt = W, nt = N;
  for (uint32_t o = Sp >> 1; o; o >>= 1) {
    wt += __shfl_xor_sync(0xffffffffu, wt, o);
    nt += __shfl_xor_sync(0xffffffffu, nt, o);
  }
  if (la >= LA) return;
  const uint32_t leaf = la / A, a = la - leaf * A;
  const LeafDev& lf = b.leaves[leaf];
  const DevModel& dm = *b.model;
  if (ne) {
    const uint32_t c = cb + rk;
    if (c < b.child_capacity) {
      const double Wd = (double)W;
      b.child_count[c] = (uint32_t)N;
      b.child_first[c] = (uint32_t)mn;
      b.child_weight[c] = (float)(Wd * dm.inv_fx * lf.wroot);
      b.child_upper[c] = (float)((double)U / Wd);
      b.child_lower[c] = (float)((double)Lm / Wd);
      b.child_obs[c] = j;
    }
    if (rk < lf.kcap) lf.keys[(uint64_t)a * lf.kcap + rk] = j;  // key table for later updates
  }
  if (j == 0) {
    lf.nchild[a] = __popc(gb);
    const double Wd = (double)wt;
    b.act_reward[la] = (float)((double)Q0 / Wd);
    b.act_upper[la] = (float)((double)Q1 / Wd);
    b.act_lower[la] = (float)((double)Q2 / Wd);
    if (a == 0) {
      b.n_scen[leaf] = (uint32_t)nt;
      b.weight[leaf] = (float)(Wd * dm.inv_fx * lf.wroot);
      if (nt == 0) atomicOr(b.err, kErrEmptyLeaf);
    }
  }
}

// K3c for many observation slots (S > 32: navigation's 257): one CTA per
// (leaf, action), one thread per slot -- a warp per (leaf, action) would walk
// its slots in S/32 dependent rounds
constexpr uint32_t kWideS = 32;
__global__ void __launch_bounds__(256) k3_write_wide(BatchDev b) {
  __shared__ int64_t s_wt[8], s_nt[8];
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t S = b.S, A = b.A;
  const uint64_t LA = (uint64_t)b.L * A, la = blockIdx.x;
  const uint32_t leaf = (uint32_t)(la / A), a = (uint32_t)(la - (uint64_t)leaf * A);
  const LeafDev& lf = b.leaves[leaf];
  const DevModel& dm = *b.model;
  const SumLayout lay{LA * S, LA};
  const uint64_t base = la * S;
  const uint32_t cb = b.child_begin[la];
  int64_t wt = 0, nt = 0;
  for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) {
    const int64_t N = b.sums[lay.N(base + s)];
    if (!N) continue;
    const int64_t W = b.sums[lay.W(base + s)];
    wt += W;
    nt += N;
    const uint32_t rk = b.rank[base + s];
    const uint32_t c = cb + rk;
    if (c < b.child_capacity) {
      const double Wd = (double)W;
      b.child_count[c] = (uint32_t)N;
      b.child_first[c] = (uint32_t)b.mins[base + s];
      b.child_weight[c] = (float)(Wd * dm.inv_fx * lf.wroot);
      b.child_upper[c] = (float)((double)b.sums[lay.U(base + s)] / Wd);
      b.child_lower[c] = (float)((double)b.sums[lay.Lm(base + s)] / Wd);
      b.child_obs[c] = s;
    }
    if (rk < lf.kcap) lf.keys[(uint64_t)a * lf.kcap + rk] = s;  // key table for later updates
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
    lf.nchild[a] = b.nc[la];
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

// K3 for many observation slots (S > 32: navigation's 257) in ONE kernel:
// rank, scan and write of (leaf, action) la per CTA, the CTAs in ticket order
// (la = ticket, so every predecessor a CTA looks back on is already running)
// and the child_begin prefix by decoupled look-back over one (flag, value)
// word per la.  Replaces k3_rank_dense + k3_scan_lookback + k3_write_wide and
// their global rank / count round trips.  Each thread holds its (up to P)
// slots' sums and first id in registers from one round of loads and writes
// their outputs itself.  Dynamic shared memory: 8 S bytes (the compacted
// non-empty slots' first ids and ranks).
constexpr uint32_t kWideFusedThreads = 256;
template <int P>  // ceil(S / 256) slots per thread (S <= 1024)
__global__ void __launch_bounds__(kWideFusedThreads) k3_wide_fused(BatchDev b) {
  extern __shared__ __align__(16) unsigned char k3w_smem[];
  __shared__ uint32_t s_wcnt[kWideFusedThreads / 32], s_ticket, s_cnt;
  __shared__ int64_t s_wt[kWideFusedThreads / 32], s_nt[kWideFusedThreads / 32];
  constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kVal = (1ull << 62) - 1;
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  const uint32_t S = b.S, A = b.A, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr uint32_t NW = kWideFusedThreads / 32;
  const uint64_t LA = (uint64_t)b.L * A;
  int32_t* s_first = reinterpret_cast<int32_t*>(k3w_smem);
  uint32_t* s_rank = reinterpret_cast<uint32_t*>(s_first + S);
  if (threadIdx.x == 0) s_ticket = (uint32_t)atomicAdd(&b.scan_flags[0], 1ull);
  __syncthreads();
  const uint64_t la = s_ticket;
  HD_CHECK(b.err, la < LA);
  const uint32_t leaf = (uint32_t)(la / A), a = (uint32_t)(la - (uint64_t)leaf * A);
  const SumLayout lay{LA * S, LA};
  const uint64_t base = la * S;
  // 1. each thread's slots s = p * 256 + tid, every sum and first id loaded at
  // once (one round trip), then the non-empty ones compacted in slot order
  int64_t N[P], W[P], U[P], Lm[P];
  int32_t mn[P];
  int32_t pos[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint32_t s = p * kWideFusedThreads + threadIdx.x;
    const bool in = s < S;
    N[p] = in ? __ldcg(&b.sums[lay.N(base + s)]) : 0;
    W[p] = in ? __ldcg(&b.sums[lay.W(base + s)]) : 0;
    U[p] = in ? __ldcg(&b.sums[lay.U(base + s)]) : 0;
    Lm[p] = in ? __ldcg(&b.sums[lay.Lm(base + s)]) : 0;
    mn[p] = in ? __ldcg(&b.mins[base + s]) : 0;
  }
  uint32_t cnt = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const bool ne = N[p] != 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, ne);
    if (lane == 0) s_wcnt[wid] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < NW; ++w) {
      before += w < wid ? s_wcnt[w] : 0u;
      tot += s_wcnt[w];
    }
    pos[p] = -1;
    if (ne) {
      pos[p] = (int32_t)(cnt + before + __popc(bal & ((1u << lane) - 1u)));
      s_first[pos[p]] = mn[p];
    }
    cnt += tot;
    __syncthreads();
  }
  HD_CHECK(b.err, cnt <= S);
  unsigned long long* st = b.scan_flags + 1;
  if (threadIdx.x == 0) atomicExch(&st[la], (la == 0 ? kIncl : kAgg) | cnt);  // publish early
  // 2. look-back (warp 0, a window of 32 predecessors per L2 round trip)
  // while the other warps rank
  if (wid == 0) {
    uint64_t excl = 0;
    if (la > 0) {
      int64_t p = (int64_t)la - 1;  // window [p - 31, p], lane j reads p - j
      for (;;) {
        const int64_t q = p - (int64_t)lane;
        const unsigned long long f = q >= 0 ? atomicAdd(&st[q], 0ull) : (kIncl | 0ull);
        // the nearest inclusive prefix in the window
        const uint32_t incl = __ballot_sync(0xffffffffu, (f >> 62) == 2);
        const uint32_t upto = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
        if (__any_sync(0xffffffffu, lane <= upto && !(f >> 62))) continue;  // a predecessor not published yet
        excl += __reduce_add_sync(0xffffffffu, lane <= upto ? (uint32_t)(f & kVal) : 0u);
        if (incl) break;
        p -= 32;
      }
      if (lane == 0) atomicExch(&st[la], kIncl | (excl + cnt));
    }
    if (lane == 0) s_cnt = (uint32_t)excl;
  } else {
    for (uint32_t i = threadIdx.x - 32; i < cnt; i += kWideFusedThreads - 32) {
      const int32_t f = s_first[i];
      uint32_t r = 0;
      for (uint32_t q = 0; q < cnt; ++q) r += s_first[q] < f;
      s_rank[i] = r;  // first occurrence (R8)
    }
  }
  __syncthreads();
  // 3. outputs, by each slot's owner from its registers: Eq. 11/12 child
  // bounds, one-level Eq. 4, the child-key table
  const LeafDev& lf = b.leaves[leaf];
  const DevModel& dm = *b.model;
  const uint32_t cb = s_cnt;  // the exclusive prefix of the child counts
  int64_t wt = 0, nt = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (pos[p] < 0) continue;
    const uint32_t s = p * kWideFusedThreads + threadIdx.x, rk = s_rank[pos[p]];
    HD_CHECK(b.err, rk < cnt);
    wt += W[p];
    nt += N[p];
    const uint32_t c = cb + rk;
    if (c < b.child_capacity) {
      const double Wd = (double)W[p];
      b.child_count[c] = (uint32_t)N[p];
      b.child_first[c] = (uint32_t)mn[p];
      b.child_weight[c] = (float)(Wd * dm.inv_fx * lf.wroot);
      b.child_upper[c] = (float)((double)U[p] / Wd);
      b.child_lower[c] = (float)((double)Lm[p] / Wd);
      b.child_obs[c] = s;
    }
    if (rk < lf.kcap) lf.keys[(uint64_t)a * lf.kcap + rk] = s;  // key table for later updates
  }
  wt = warp_sum64(wt);
  nt = warp_sum64(nt);
  if (lane == 0) {
    s_wt[wid] = wt;
    s_nt[wid] = nt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < NW; ++w) {
      wt += s_wt[w];
      nt += s_nt[w];
    }
    b.child_begin[la] = cb;
    lf.nchild[a] = cnt;
    const double Wd = (double)wt;
    b.act_reward[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 0)]) / Wd);
    b.act_upper[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 1)]) / Wd);
    b.act_lower[la] = (float)((double)__ldcg(&b.sums[lay.Q(la, 2)]) / Wd);
    if (a == 0) {
      b.n_scen[leaf] = (uint32_t)nt;
      b.weight[leaf] = (float)(Wd * dm.inv_fx * lf.wroot);
      if (nt == 0) atomicOr(b.err, kErrEmptyLeaf);
    }
    if (la + 1 == LA) {  // the last pair: totals
      const uint64_t total = (uint64_t)cb + cnt;
      b.child_begin[LA] = (uint32_t)total;
      if (total > b.child_capacity) atomicOr(b.err, kErrChildCap);
      b.status[1] = (uint32_t)total;
      const uint64_t steps = (uint64_t)__ldcg(&b.sums[lay.steps()]);
      b.status[2] = (uint32_t)steps;
      b.status[3] = (uint32_t)(steps >> 32);
    }
  }
  if (b.hstat) {  // resident prepared batch: restore the zero state for the next run
    __syncthreads();  // this pair's sums are read
    for (uint32_t s = threadIdx.x; s < S; s += kWideFusedThreads) {
      b.sums[lay.W(base + s)] = 0;
      b.sums[lay.U(base + s)] = 0;
      b.sums[lay.Lm(base + s)] = 0;
      b.sums[lay.N(base + s)] = 0;
      b.mins[base + s] = 0x7F7F7F7F;
    }
    if (threadIdx.x < 3) b.sums[lay.Q(la, threadIdx.x)] = 0;
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&b.status[kStatK3Done], 1u) == LA - 1;
    }
    __syncthreads();
    if (s_last) {  // every pair is done: publish the status, reset the counters
      __threadfence();
      const uint32_t nst = kStatWords + b.L;
      for (uint32_t i = threadIdx.x; i < nst; i += kWideFusedThreads) b.hstat[i] = __ldcg(&b.status[i]);
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x < kStatWords) b.status[threadIdx.x] = 0u;
      if (threadIdx.x == 0) b.sums[lay.steps()] = 0;
      for (uint64_t i = threadIdx.x; i < LA + 2; i += kWideFusedThreads) b.scan_flags[i] = 0ull;
    }
  }
}
__host__ __device__ inline size_t wide_fused_smem(uint32_t S) { return 8 * (size_t)S; }
constexpr uint32_t kWideFusedMaxS = 4 * kWideFusedThreads;  // P <= 4 register-held slots per thread
constexpr size_t kWideFusedMaxSmem = 96 << 10;

// K3 for small batches (L*A <= kSmallLA, S <= 32): rank, scan and write in
// one CTA -- a kernel of its own, or the tail of K2's last CTA.  The path is
// latency bound (a few L2 round trips per (leaf, action)), so: one lane per
// observation slot, 32/Sp (leaf, action) pairs per warp (Sp = S rounded up
// to a power of two), the loads of kSmallUnroll pairs in flight at once, the
// child ordinals (first occurrence, R8) recomputed in registers from the
// first ids instead of stored, and child_begin scanned in shared memory.
constexpr uint32_t kSmallLA = 4096;
constexpr uint32_t kSmallUnroll = 4;
__host__ __device__ inline size_t small_finalize_smem(uint64_t LA) { return align16(4 * (LA + 1)); }
__device__ __forceinline__ void small_finalize(const BatchDev& b, unsigned char* smem, uint64_t* wsum) {
  const uint32_t wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t S = b.S, A = b.A, LA = b.L * b.A;
  const uint32_t Sp = small_group_width(S), G = 32 / Sp;
  const uint32_t j = lane & (Sp - 1), gshift = lane & ~(Sp - 1);
  const uint32_t gbits = Sp == 32 ? 0xffffffffu : (1u << Sp) - 1u;
  const SumLayout lay{(uint64_t)LA * S, LA};
  const uint32_t stride = nw * G;  // pairs per CTA-wide sweep
  const uint32_t first = wid * G + lane / Sp;
  uint32_t* cb = reinterpret_cast<uint32_t*>(smem);  // [LA + 1]: counts, then offsets
  const double inv_fx = b.model->inv_fx;
  // ---- children per (leaf, action), one-level Eq. 4 ---------------------
  for (uint32_t la0 = first; la0 - lane / Sp < LA; la0 += stride * kSmallUnroll) {
    int64_t n[kSmallUnroll], w[kSmallUnroll], Q[kSmallUnroll][3];
#pragma unroll
    for (uint32_t u = 0; u < kSmallUnroll; ++u) {
      const uint32_t la = la0 + u * stride;
      const bool v = la < LA && j < S;
      n[u] = v ? __ldcg(&b.sums[lay.N((uint64_t)la * S + j)]) : 0;
      w[u] = v ? __ldcg(&b.sums[lay.W((uint64_t)la * S + j)]) : 0;
      const bool q = la < LA && j == 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) Q[u][k] = q ? __ldcg(&b.sums[lay.Q(la, k)]) : 0;
    }
#pragma unroll
    for (uint32_t u = 0; u < kSmallUnroll; ++u) {
      const uint32_t la = la0 + u * stride;
      const uint32_t gb = (__ballot_sync(0xffffffffu, n[u] != 0) >> gshift) & gbits;
      int64_t wt = w[u], nt = n[u];
      for (uint32_t o = Sp >> 1; o; o >>= 1) {
        wt += __shfl_xor_sync(0xffffffffu, wt, o);
        nt += __shfl_xor_sync(0xffffffffu, nt, o);
      }
      if (j == 0 && la < LA) {
        const uint32_t leaf = la / A, a = la - leaf * A;
        const LeafDev& lf = b.leaves[leaf];
        cb[la] = __popc(gb);
        lf.nchild[a] = __popc(gb);
        const double Wd = (double)wt;
        b.act_reward[la] = (float)((double)Q[u][0] / Wd);
        b.act_upper[la] = (float)((double)Q[u][1] / Wd);
        b.act_lower[la] = (float)((double)Q[u][2] / Wd);
        if (a == 0) {
          b.n_scen[leaf] = (uint32_t)nt;
          b.weight[leaf] = (float)(Wd * inv_fx * lf.wroot);
          if (nt == 0) atomicOr(b.err, kErrEmptyLeaf);
        }
      }
    }
  }
  __syncthreads();
  // ---- child_begin: exclusive scan of the counts (in place) -----------
  {
    const uint32_t per = (LA + blockDim.x - 1) / blockDim.x;
    const uint32_t i0 = threadIdx.x * per;
    uint64_t loc = 0;
    for (uint32_t i = i0; i < i0 + per && i < LA; ++i) loc += cb[i];
    uint64_t tot;
    uint64_t run = block_excl_scan(loc, wsum, tot);
    for (uint32_t i = i0; i < i0 + per && i < LA; ++i) {
      const uint32_t c = cb[i];
      cb[i] = (uint32_t)run;
      b.child_begin[i] = (uint32_t)run;
      run += c;
    }
    if (threadIdx.x == 0) {
      cb[LA] = (uint32_t)tot;
      b.child_begin[LA] = (uint32_t)tot;
      if (tot > b.child_capacity) atomicOr(b.err, kErrChildCap);
      b.status[1] = (uint32_t)tot;
      const uint64_t steps = (uint64_t)__ldcg(&b.sums[lay.steps()]);
      b.status[2] = (uint32_t)steps;
      b.status[3] = (uint32_t)(steps >> 32);
    }
  }
  __syncthreads();
  // ---- children: Eq. 11/12 bounds, first ids, key tables --------------
  for (uint32_t la0 = first; la0 - lane / Sp < LA; la0 += stride * kSmallUnroll) {
    int64_t N[kSmallUnroll], W[kSmallUnroll], U[kSmallUnroll], Lm[kSmallUnroll];
    int32_t mn[kSmallUnroll];
#pragma unroll
    for (uint32_t u = 0; u < kSmallUnroll; ++u) {
      const uint32_t la = la0 + u * stride;
      const bool v = la < LA && j < S;
      const uint64_t slot = (uint64_t)la * S + j;
      N[u] = v ? __ldcg(&b.sums[lay.N(slot)]) : 0;
      W[u] = v ? __ldcg(&b.sums[lay.W(slot)]) : 0;
      U[u] = v ? __ldcg(&b.sums[lay.U(slot)]) : 0;
      Lm[u] = v ? __ldcg(&b.sums[lay.Lm(slot)]) : 0;
      mn[u] = v ? __ldcg(&b.mins[slot]) : 0;
    }
#pragma unroll
    for (uint32_t u = 0; u < kSmallUnroll; ++u) {
      const uint32_t la = la0 + u * stride;
      const bool ne = N[u] != 0;
      const uint32_t gb = (__ballot_sync(0xffffffffu, ne) >> gshift) & gbits;
      // ordinal = number of non-empty slots of the pair with a smaller first id
      uint32_t rk = 0;
      for (uint32_t k = 0; k < Sp; ++k) {
        const int32_t mk = __shfl_sync(0xffffffffu, mn[u], k, Sp);
        rk += ((gb >> k) & 1u) && mk < mn[u];
      }
      if (!ne || la >= LA) continue;
      const uint32_t leaf = la / A, a = la - leaf * A;
      const LeafDev& lf = b.leaves[leaf];
      const uint32_t c = cb[la] + rk;
      if (c < b.child_capacity) {
        const double Wd = (double)W[u];
        b.child_count[c] = (uint32_t)N[u];
        b.child_first[c] = (uint32_t)mn[u];
        b.child_weight[c] = (float)(Wd * inv_fx * lf.wroot);
        b.child_upper[c] = (float)((double)U[u] / Wd);
        b.child_lower[c] = (float)((double)Lm[u] / Wd);
        b.child_obs[c] = j;
      }
      if (rk < lf.kcap) lf.keys[(uint64_t)a * lf.kcap + rk] = j;  // key table for later updates
    }
  }
}
// out of line for K2's tail: its registers do not constrain K2's main loop
// (wsum: the caller's 32-word scan scratch, shared with its other scans)
__device__ __noinline__ void small_finalize_tail(const BatchDev& b, unsigned char* smem, uint64_t* wsum) {
  small_finalize(b, smem, wsum);
}
// A resident prepared batch (a graph of one kernel): after
// the fused finalize the last CTA publishes the status block to mapped host
// memory (the host reads it after the stream synchronises: no D2H copy) and
// puts the scratch back into the state the next run starts from (zero sums,
// 0x7F7F7F7F first ids, zero status header; n_leaf and the prefixes are the
// batch's constants), so the graph needs no memset nodes.  Every other CTA
// has finished (it took its ticket after its last tile).
__device__ __noinline__ void resident_epilogue(const BatchDev& b) {
  __syncthreads();  // this CTA's finalize is complete
  const uint32_t nst = kStatWords + b.L;
  for (uint32_t i = threadIdx.x; i < nst; i += blockDim.x) b.hstat[i] = __ldcg(&b.status[i]);
  __threadfence_system();
  __syncthreads();
  const SumLayout lay{(uint64_t)b.L * b.A * b.S, (uint64_t)b.L * b.A};
  const uint64_t ns = lay.total(), nm = lay.las;
  for (uint64_t i = threadIdx.x; i < ns; i += blockDim.x) b.sums[i] = 0;
  for (uint64_t i = threadIdx.x; i < nm; i += blockDim.x) b.mins[i] = 0x7F7F7F7F;
  if (threadIdx.x < kStatWords) b.status[threadIdx.x] = 0u;
}
__global__ void __launch_bounds__(1024) k3_small_dense(BatchDev b) {
  pdl_wait();  // the predecessor complete
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char k3s_smem[];
  __shared__ uint64_t wsum[32];
  small_finalize(b, k3s_smem, wsum);
}

__global__ void k_stream_words(uint32_t k0, uint32_t k1, const uint32_t* ids, uint32_t n, uint32_t t,
                               uint32_t k, uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 w = philox4x32_10(ids[i], t, k >> 2, 0u, k0, k1);
  const uint32_t sel = k & 3u;
  out[i] = sel == 0 ? w.x : sel == 1 ? w.y : sel == 2 ? w.z : w.w;
}

// K0, the measured Philox ceiling (ceiling 2): thread g of the
// grid-stride loop draws the stream blocks (ctr = (g, t, 0, 0), t = 1 ..
// blocks) with the round keys as a kernel parameter -- K2's best case -- and
// XOR-folds every word; one atomicXor per warp keeps the work observable.
__global__ void __launch_bounds__(256) k0_philox(const RoundKeys rk, uint32_t n_threads, uint32_t blocks,
                                                 uint32_t* checksum) {
  uint32_t x = 0;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_threads; g += gridDim.x * blockDim.x) {
    for (uint32_t t = 1; t <= blocks; ++t) {
      const uint4 w = philox(g, t, 0u, 0u, rk);
      x ^= w.x ^ w.y ^ w.z ^ w.w;
    }
  }
  x = __reduce_xor_sync(0xffffffffu, x);
  if ((threadIdx.x & 31) == 0) atomicXor(checksum, x);
}

}  // namespace hd
