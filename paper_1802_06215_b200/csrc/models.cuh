// models.cuh -- device implementations of the dense-observation model cards
// (DESIGN.md §3): Tiger, RockSample / multi-agent RockSample
// and navigation in a partially known map.
//
// Interface of a model M (used by the kernel templates in kernels.cu):
//   M::Sm                 shared-memory copy of the hot tables
//   M::load_sm(sm, dm)    cooperative build of Sm + tables (caller syncs); the
//                         kernels use load_sm_image (a copy of its result)
//   M::St                 per-thread register state; load/store SoA rows
//   M::terminal(sm, s)    terminal flag of a state
//   M::step(...)          g(s, a, phi_t) on a non-terminal state (Eq. 9)
//   M::upper(...)         per-scenario u(s) of Eq. 11 (non-terminal state)
//   M::rollout<TRACE>     default-policy roll-out of Eq. 12 to depth D
#pragma once
#include "common.cuh"

namespace hd {

__device__ __forceinline__ void copy_words(void* dst, const void* src, int bytes, int tid, int nt) {
  const uint32_t* s = static_cast<const uint32_t*>(src);
  uint32_t* d = static_cast<uint32_t*>(dst);
  for (int i = tid; i < bytes / 4; i += nt) d[i] = s[i];
}

// ===========================================================================
// Tiger: state bit0 side, bit1 terminal; 0 LISTEN, 1 OPEN-LEFT, 2 OPEN-RIGHT
// ===========================================================================
struct Tiger {
  static constexpr uint32_t kScratchPerThread = 0;  // no per-thread shared scratch
  static __device__ __forceinline__ void bind_scratch(uint32_t) {}
  static constexpr int kK1Threads = 512;  // K1 block: one round over K = 500 scenarios
  static constexpr int kMinBlocks = 8;  // K2 occupancy target (CTAs of 128 per SM)
  struct Sm {
    uint64_t t_listen;
    uint32_t D;
    double tail;
    double gpow[kGpowN];
  };
  static __device__ void load_sm(Sm& sm, const DevModel& dm, int tid, int nt) {
    if (tid == 0) {
      sm.t_listen = dm.t_listen;
      sm.D = dm.D;
      sm.tail = dm.tail;
    }
    copy_words(sm.gpow, dm.gpow, sizeof(sm.gpow), tid, nt);
  }
  struct St {
    uint32_t s;
  };
  static __device__ __forceinline__ St load(const Sm&, const uint32_t* st, uint32_t cap, uint32_t i) {
    return St{st[i]};
  }
  static __device__ __forceinline__ void store(const Sm&, const St& s, uint32_t* st, uint32_t cap,
                                               uint32_t i) {
    st[i] = s.s;
  }
  static __device__ __forceinline__ bool terminal(const Sm&, const St& s) { return (s.s >> 1) & 1u; }
  static constexpr uint32_t kTerminalObs = 3u;
  static __device__ __forceinline__ bool step_u(const Sm& sm, St& s, int a, uint32_t u0, uint32_t& z,
                                                float& r) {
    const uint32_t side = s.s & 1u;
    if (a == 0) {
      const bool correct = event(u0, sm.t_listen);
      const uint32_t heard = correct ? side : 1u - side;
      r = -1.0f;
      z = 1u + heard;
      return false;
    }
    const uint32_t door = (uint32_t)(a - 1);
    r = (door == side) ? -100.0f : 10.0f;
    s.s = side | 2u;
    z = kTerminalObs;
    return true;
  }
  template <class KeyT>
  static __device__ __forceinline__ bool step(const Sm& sm, St& s, int a, uint32_t id, uint32_t t,
                                              const KeyT& key, uint32_t& z, float& r) {
    const uint4 u = philox(id, t, 0u, 0u, key);
    return step_u(sm, s, a, u.x, z, r);
  }
  static __device__ __forceinline__ double upper(const Sm&, const St&) { return 10.0; }
  static __device__ __forceinline__ uint32_t initial_obs(const Sm&, const St&) { return 0u; }
  template <bool TRACE, class KeyT>
  static __device__ void rollout(const Sm& sm, St s, uint32_t z, uint32_t id, uint32_t t0,
                                 const KeyT& key, double& ret, uint32_t& len, uint64_t& h) {
    double acc = 0.0;
    uint32_t t = t0;
    bool term = false;
    while (t < sm.D && !term) {
      const int a = 0;  // Listen always
      if (TRACE) h = (h ^ (uint64_t)a) * kFnvPrime;
      float r;
      term = step(sm, s, a, id, t + 1, key, z, r);
      acc += sm.gpow[t - t0] * (double)r;
      ++t;
    }
    if (!term) acc += sm.gpow[t - t0] * sm.tail;
    ret = acc;
    len = t - t0;
  }
};

// ===========================================================================
// RockSample(n, m) with R in {1, 2} robots (card §3.2).
// word 0: good-rock mask; word 1: 16 bits per robot (y*n+x, 0xFFFF exited).
// sub-actions: 0 N, 1 S, 2 E, 3 W, 4 SAMPLE, 5+j SENSE j; a = b0 + base*b1.
//
// Device representation: a robot is its cell index, an exited robot the
// pseudo-cell EXIT = n*n whose every action is a no-op.  Every geometric
// question of a step is a shared-memory table lookup built per CTA from the
// layout: the target cell of each move (with the +10 exit through the east
// border as a flag bit), the rock on a cell, the sensing threshold of every
// (cell, rock), and the default policy's move toward each policy position.
// This moves the step's work from the ALU pipe (the kernel's limiter) to the
// load/store pipe, and the pseudo-cell removes the per-robot "exited" selects.
// ===========================================================================
// roll-out pipe balance (ALU vs FMA-heavy), A/B-measured
#ifndef HD_RS_ONE
#define HD_RS_ONE 0
#endif
#ifndef HD_RS_SENSE_LOP
#define HD_RS_SENSE_LOP 1
#endif
#ifndef HD_RS_ROWSEL
#define HD_RS_ROWSEL 1
#endif
#ifndef HD_RS_CELL_SHF
#define HD_RS_CELL_SHF 0
#endif
#ifndef HD_RS_EX_SHF
#define HD_RS_EX_SHF 0
#endif
template <int R>
struct RockSample {
  static constexpr uint32_t kScratchPerThread = 0;  // no per-thread shared scratch
  static __device__ __forceinline__ void bind_scratch(uint32_t) {}
#ifndef HD_RS_MINB
#define HD_RS_MINB 7
#endif
  static constexpr int kMinBlocks = HD_RS_MINB;  // 7: 72 registers, 28 warps per SM (8 / 7 / 6 measured 1.569 / 1.539 / 1.538 ms on config 2)
  static constexpr int kK1Threads = 512;  // K1 block: one round over K = 500 scenarios
  static constexpr int kMaxTable = 16384;  // n*n*m entries of the per-cell rock tables
  struct Sm {
    int32_t n, m, mm, base, ncell, exitc;  // exitc = EXIT pseudo-cell = n*n; mm = max(m, 1)
    uint32_t D;
    uint32_t md;          // the dist table's row stride: mm rounded up to 4 (word loads of 4 rocks)
    uint32_t base_magic;  // ceil(2^32 / base): a / base = umulhi(a, magic) for a < 2^16
    double tail;
    // Default-policy columns: robot r walks its handled rocks in order (x, y, j)
    // through the columns q = qstart[r] .. qstart[r] + k_r - 1, then stays on
    // its sentinel column qstart[r] + k_r (nothing left: E).  A robot only
    // ever marks its current target (GOOD after a GOOD reading; DONE after a
    // BAD reading or a SAMPLE), so the card's per-rock memory is exactly a
    // column index plus one "target known GOOD" bit per robot.
    uint8_t senseb[40];      // column q -> SENSE sub-action 5 + rock(q); a sentinel column -> E
    uint32_t qstart[2];      // first column of robot r
    uint32_t polw;           // columns per cell row of the pol table (m + 2)
    uint32_t one;            // 1, opaque to the compiler: address sums in the roll-out become IMADs
                             // (FMA pipe) instead of IADD3s on the ALU pipe, the loop's limiter
    // byte offsets in hd_dyn_smem of the variable-size tables (sized by n, m, D):
    uint32_t off_act;   // u16 [cell][base]: the effect of sub-action b on a robot at the cell:
                        // bit 0 SENSE (not from EXIT), bit 1 SAMPLE on a rock, bit 2 the +10
                        // exit, bits 3-15 the next cell (EXIT pseudo-cell included)
    uint32_t off_info;  // u32 [cell]: bits 0-4 rock on the cell, bit 5 has a rock; 8-15 x; 16-23 y
    uint32_t off_rock;  // u8  [cell]: 5 + the rock on the cell (0 if none; only read with SAMPLE's flag)
    uint32_t off_thr;   // u32 [cell][mm]: sensing rock j from the cell is correct iff u <= thr
    uint32_t off_pol;   // u8  [cell][m+2]: policy move toward the rock of column q (4 = on it); sentinels
                        // E; row n*n+1 (the SENSE row) holds senseb: the sub-action of a robot whose
                        // target is not known GOOD
    uint32_t off_dist;  // u8  [cell][md]: |x - x_j| + |y - y_j| (255 from EXIT and past m)
    const double* gpow_g;  // gamma^k in the model's global memory (once per roll-out: the tail term)
    uint32_t off_gp10;  // f64 [G + 1]: 10 gamma^k (k < G = max(D, 2n) + 1), then 0.0 (index G: a bad
                        // rock's term in upper())
    uint32_t gzero4;    // G in every byte (the index of gp10's 0.0)
  };
  static __host__ __device__ int gpow_len(int n, uint32_t D) { return (int)(D > (uint32_t)(2 * n) ? D : 2 * n) + 1; }
  static constexpr uint32_t kActSense = 1u, kActSample = 2u, kActExit = 4u, kActShift = 3u;
  // table bytes (host and device agree): pol | act | info | rock | thr | dist | gp | gp10, with the
  // EXIT row (and pol's SENSE row)
  static __host__ __device__ size_t table_bytes(int n, int m, uint32_t D) {
    const size_t c = (size_t)n * n + 1, mm = m > 0 ? (size_t)m : 1, G = (size_t)gpow_len(n, D);
    const size_t md = (mm + 3) & ~size_t(3);
    return align16((c + 1) * (m + 2)) + align16(2 * c * (5 + m)) + align16(4 * c) + align16(c) +
           align16(4 * c * mm) + align16(c * md) + align16(8 * (G + 1));
  }
  static __device__ __forceinline__ uint32_t info(const Sm& sm, int c) {
    return reinterpret_cast<const uint32_t*>(hd_dyn_smem + sm.off_info)[c];
  }
  static __device__ __forceinline__ uint32_t act(const Sm& sm, int c, int sub) {
    return reinterpret_cast<const uint16_t*>(hd_dyn_smem + sm.off_act)[c * sm.base + sub];
  }
  // the threshold of SENSE sub-action `sub` (rock sub - 5) from cell c.  For
  // sub < 5 the index falls on the previous row's entries or, at c = 0, on the
  // rock table in front of the thr table: a harmless value the SENSE flag masks.
  static __device__ __forceinline__ uint32_t thr_sub(const Sm& sm, int c, int sub) {
    return reinterpret_cast<const uint32_t*>(hd_dyn_smem + sm.off_thr)[c * sm.mm + sub - 5];
  }
  static __device__ __forceinline__ uint32_t rock_on(const Sm& sm, int c) { return hd_dyn_smem[sm.off_rock + c]; }
  // the pol table is the first table: its offset is a compile-time constant
  static constexpr uint32_t kOffPol = (uint32_t)align16(sizeof(Sm));
  static __device__ __forceinline__ uint32_t pol(const Sm& sm, int c, int q) {
    return hd_dyn_smem[kOffPol + c * sm.polw + q];
  }
  static __device__ __forceinline__ const uint32_t* dist_row(const Sm& sm, int c) {
    return reinterpret_cast<const uint32_t*>(hd_dyn_smem + sm.off_dist + c * sm.md);
  }
  static __device__ __forceinline__ double gp(const Sm& sm, int k) {
    return sm.gpow_g[k];
  }
  static __device__ __forceinline__ double gp10(const Sm& sm, int k) {
    return reinterpret_cast<const double*>(hd_dyn_smem + sm.off_gp10)[k];
  }
  static __device__ void load_sm(Sm& sm, const DevModel& dm, int tid, int nt) {
    const int n = dm.n, mm = dm.m > 0 ? dm.m : 1, nc = n * n, exitc = nc, G = gpow_len(n, dm.D);
    const int md = (mm + 3) & ~3;
    const uint32_t polw = (uint32_t)dm.m + 2;
    const uint32_t off_pol = kOffPol, off_act = off_pol + (uint32_t)align16((size_t)(nc + 2) * polw),
                   off_info = off_act + (uint32_t)align16(2 * (size_t)(nc + 1) * dm.base),
                   off_rock = off_info + (uint32_t)align16(4 * (size_t)(nc + 1)),
                   off_thr = off_rock + (uint32_t)align16((size_t)(nc + 1)),
                   off_dist = off_thr + (uint32_t)align16(4 * (size_t)(nc + 1) * mm),
                   off_gp10 = off_dist + (uint32_t)align16((size_t)(nc + 1) * md);
    uint16_t* t_act = reinterpret_cast<uint16_t*>(hd_dyn_smem + off_act);
    uint32_t* t_info = reinterpret_cast<uint32_t*>(hd_dyn_smem + off_info);
    uint8_t* t_rock = hd_dyn_smem + off_rock;
    uint32_t* t_thr = reinterpret_cast<uint32_t*>(hd_dyn_smem + off_thr);
    uint8_t* t_pol = hd_dyn_smem + off_pol;
    uint8_t* t_dist = hd_dyn_smem + off_dist;
    double* t_gp10 = reinterpret_cast<double*>(hd_dyn_smem + off_gp10);
    if (tid == 0) {
      sm.off_act = off_act;
      sm.off_info = off_info;
      sm.off_rock = off_rock;
      sm.off_thr = off_thr;
      sm.off_pol = off_pol;
      sm.off_dist = off_dist;
      sm.gpow_g = dm.gpow;
      sm.off_gp10 = off_gp10;
      sm.polw = polw;
      sm.one = 1u;
      sm.n = n;
      sm.m = dm.m;
      sm.mm = mm;
      sm.base = dm.base;
      sm.md = (uint32_t)md;
      sm.gzero4 = (uint32_t)G * 0x01010101u;  // G <= 251
      sm.base_magic = (uint32_t)((0x100000000ull + (uint64_t)dm.base - 1) / (uint64_t)dm.base);
      sm.ncell = nc;
      sm.exitc = exitc;
      sm.D = dm.D;
      sm.tail = dm.tail;
      const uint32_t k0 = (uint32_t)__popc(dm.range_mask[0]);
      sm.qstart[0] = 0;
      sm.qstart[1] = k0 + 1;
    }
    // column q -> policy position (rocks sorted by handling robot, then (x, y, j)) or a sentinel
    const int k0 = __popc(dm.range_mask[0]), k1 = __popc(dm.range_mask[1]);
    auto col_pos = [&](int q) -> int {
      if (q < k0) return q;                       // robot 0's positions 0 .. k0-1
      if (q == k0) return -1;                     // robot 0's sentinel
      if (q - 1 < k0 + k1) return q - 1;          // robot 1's positions k0 .. k0+k1-1
      return -1;                                  // robot 1's sentinel (and unused columns)
    };
    for (int q = tid; q < 40; q += nt) {
      const int p = q < (int)polw ? col_pos(q) : -1;
      sm.senseb[q] = p >= 0 ? (uint8_t)(5 + dm.pos_rock[p]) : (uint8_t)2;
    }
    for (int k = tid; k <= G; k += nt)
      t_gp10[k] = k < G ? 10.0 * dm.gpow[k] : 0.0;  // the product upper() used to form per rock
    for (int e = tid; e < (nc + 1) * md; e += nt) {
      const int c = e / md, j = e - c * md;
      t_dist[e] = (c < nc && j < dm.m) ? (uint8_t)(abs(c % n - dm.rx[j]) + abs(c / n - dm.ry[j])) : (uint8_t)255;
    }
    for (int c = tid; c <= nc; c += nt) {
      uint16_t* row = t_act + (size_t)c * dm.base;
      if (c == exitc) {  // the pseudo-cell: every sub-action is a no-op, no rock
        for (int k = 0; k < dm.base; ++k) row[k] = (uint16_t)(exitc << kActShift);
        t_info[c] = 0;
        t_rock[c] = 0;
        continue;
      }
      const int x = c % n, y = c / n;
      const int8_t rock = dm.rock_at[c];
      const uint32_t sc = (uint32_t)c << kActShift;
      row[0] = (uint16_t)((uint32_t)(y > 0 ? c - n : c) << kActShift);                 // N
      row[1] = (uint16_t)((uint32_t)(y < n - 1 ? c + n : c) << kActShift);             // S
      row[2] = (uint16_t)(x < n - 1 ? (uint32_t)(c + 1) << kActShift
                                    : ((uint32_t)exitc << kActShift) | kActExit);      // E (exit)
      row[3] = (uint16_t)((uint32_t)(x > 0 ? c - 1 : c) << kActShift);                 // W
      row[4] = (uint16_t)(sc | (rock >= 0 ? kActSample : 0u));                         // SAMPLE
      for (int k = 5; k < dm.base; ++k) row[k] = (uint16_t)(sc | kActSense);           // SENSE k - 5
      t_info[c] = (rock >= 0 ? ((uint32_t)rock | 32u) : 0u) | ((uint32_t)x << 8) | ((uint32_t)y << 16);
      t_rock[c] = rock >= 0 ? (uint8_t)(rock + 5) : (uint8_t)0;  // the rock's bit in good << 5
    }
    for (int e = tid; e < (nc + 1) * mm; e += nt) {
      const int c = e / mm, j = e - c * mm;
      uint32_t t = 0;
      if (c < nc && j < dm.m) {
        const int dx = dm.rx[j] - c % n, dy = dm.ry[j] - c / n;
        t = dm.sense_thr_m1[dx * dx + dy * dy];
      }
      t_thr[e] = t;
    }
    for (int e = tid; e < (nc + 2) * (int)polw; e += nt) {
      const int c = e / (int)polw, p = col_pos(e - c * (int)polw);
      uint8_t v = 2;  // E: a sentinel column (nothing left), or the EXIT pseudo-cell
      if (c == nc + 1) {
        v = p >= 0 ? (uint8_t)(5 + dm.pos_rock[p]) : (uint8_t)2;  // the SENSE row
      } else if (c < nc && p >= 0) {
        const int j = dm.pos_rock[p];
        const int dx = dm.rx[j] - c % n, dy = dm.ry[j] - c / n;
        // E if x < tx, W if x > tx, S if y < ty, N if y > ty, on the rock: SAMPLE
        v = (uint8_t)((dx == 0 && dy == 0) ? 4 : dx > 0 ? 2 : dx < 0 ? 3 : dy > 0 ? 1 : 0);
      }
      t_pol[e] = v;
    }
  }
  struct St {
    uint32_t good;
    int32_t cell[R];  // EXIT pseudo-cell once exited
  };
  static __device__ __forceinline__ bool exited(const Sm& sm, const St& s, int r) { return s.cell[r] == sm.exitc; }
  static __device__ __forceinline__ St load(const Sm& sm, const uint32_t* st, uint32_t cap, uint32_t i) {
    St s;
    s.good = st[i];
    const uint32_t pos = st[cap + i];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t c = (pos >> (16 * r)) & 0xFFFFu;
      s.cell[r] = c == 0xFFFFu ? sm.exitc : (int32_t)c;
    }
    return s;
  }
  static __device__ __forceinline__ void store(const Sm& sm, const St& s, uint32_t* st, uint32_t cap,
                                               uint32_t i) {
    uint32_t pos = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) pos |= (exited(sm, s, r) ? 0xFFFFu : (uint32_t)s.cell[r]) << (16 * r);
    st[i] = s.good;
    st[cap + i] = pos;
  }
  // terminal iff every robot has exited
  static __device__ __forceinline__ bool terminal(const Sm& sm, const St& s) {
    bool t = true;
#pragma unroll
    for (int r = 0; r < R; ++r) t = t && exited(sm, s, r);
    return t;
  }
  static constexpr uint32_t kTerminalObs = (R == 1) ? 3u : 9u;

  // one step with per-robot sub-actions b[r] and random words u[r], robots in
  // ascending order.  Branch-free: every lane evaluates the move, sample and
  // sense effects and selects, so roll-out lanes choosing different
  // sub-actions do not diverge.  zrs[r] returns robot r's reading (0 none,
  // 1 GOOD, 2 BAD).  Rewards are integers (exact in fp32).
  static __device__ __forceinline__ bool step_sub(const Sm& sm, St& s, const int* b, const uint32_t* u,
                                                  uint32_t& z, float& rew, uint32_t* zrs = nullptr,
                                                  int* k10 = nullptr, uint32_t* smps = nullptr) {
    int k = 0;  // the step's reward / 10: exits +1, good samples +1, bad samples -1
    uint32_t zsum = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int sub = b[r];
      const int c = s.cell[r];
      // the (cell, sub-action) entry: flags and the next cell (a move's
      // target, itself when blocked or not moving, EXIT through the east border)
      const uint32_t e = act(sm, c, sub);
      // SAMPLE on the current cell's rock
      const uint32_t jr = rock_on(sm, c) - 5u;  // (a cell without a rock: wraps, masked by SAMPLE's flag)
      const uint32_t samp = (e >> 1) & 1u;
      const uint32_t gbit = samp & (s.good >> jr);
      // SENSE rock sub - 5 (evaluated for every lane; masked; none from EXIT);
      // for sub < 5 the shift count wraps and the clamped funnel shift gives 0
      const uint32_t incorrect = u[r] > thr_sub(sm, c, sub) ? 1u : 0u;
      const uint32_t isgood = __funnelshift_rc(s.good, 0u, (uint32_t)sub - 5u) & 1u;
      const uint32_t zr = (e & kActSense) ? 2u - (isgood ^ incorrect) : 0u;  // GOOD (1) iff good == correct
      k += (int)((e >> 2) & 1u) + 2 * (int)gbit - (int)samp;
      s.good &= ~(gbit << jr);
      s.cell[r] = (int)(e >> kActShift);
      if (zrs) zrs[r] = zr;
      if (smps) smps[r] = samp;
      zsum += zr * (r == 0 ? 1u : 3u);
    }
    rew = (float)(10 * k);
    if (k10) *k10 = k;
    const bool term = terminal(sm, s);
    z = term ? kTerminalObs : zsum;
    return term;
  }
  template <class KeyT>
  static __device__ __forceinline__ bool step(const Sm& sm, St& s, int a, uint32_t id, uint32_t t,
                                              const KeyT& key, uint32_t& z, float& r) {
    int b[R];
    int rest = a;
#pragma unroll
    for (int q = 0; q < R; ++q) {  // a < 2^16 (checked at load): exact with the magic
      const int qt = (int)__umulhi((uint32_t)rest, sm.base_magic);
      b[q] = rest - qt * sm.base;
      rest = qt;
    }
    const uint4 w = philox(id, t, 0u, 0u, key);
    const uint32_t u[2] = {w.x, w.y};
    return step_sub(sm, s, b, u, z, r);
  }
  // u(s) = sum_{good j} 10 g^{min_r |r-j|_1} + sum_{r active} 10 g^{n-1-x_r}
  // (per rock: the robots' table distances, the nearest's 10 gamma^d from
  // the premultiplied table; an exited robot's row is 255, never the min
  // while some robot is active -- upper() is only asked of non-terminal states)
  static __device__ __forceinline__ double upper(const Sm& sm, const St& s) {
    // four rocks per word: the robots' byte distances, their byte-wise
    // minimum, a bad rock's byte replaced by G (the table's 0.0 after
    // 10 gamma^(G-1), so it adds +0.0 exactly as a skipped term would); the
    // terms are added in rock order j = 0, 1, ... (padding rocks past m have
    // no good bit: +0.0 too)
    const uint32_t* dr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) dr[r] = dist_row(sm, s.cell[r]);
    const double* g10 = reinterpret_cast<const double*>(hd_dyn_smem + sm.off_gp10);
    double u = 0.0;
    const int nw = (sm.m + 3) >> 2;
    for (int k = 0; k < nw; ++k) {  // uniform trip count, branch-free
      uint32_t mn = dr[0][k];
#pragma unroll
      for (int r = 1; r < R; ++r) mn = __vminu4(mn, dr[r][k]);
      const uint32_t g4 = (s.good >> (4 * k)) & 0xFu;
      const uint32_t gm = ((g4 * 0x00204081u) & 0x01010101u) * 0xFFu;  // 0xFF in the byte of each GOOD rock
      const uint32_t idx = (mn & gm) | (sm.gzero4 & ~gm);
#pragma unroll
      for (int q = 0; q < 4; ++q) u += g10[__byte_perm(idx, 0u, 0x4440u + (uint32_t)q)];
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (!exited(sm, s, r)) u += gp10(sm, sm.n - 1 - (int)((info(sm, s.cell[r]) >> 8) & 0xFFu));
    return u;
  }
  static __device__ __forceinline__ uint32_t initial_obs(const Sm&, const St&) { return 0u; }

  // default policy (card §3.2), branch-free.  Robot r's memory is its column
  // q[r] (its current target rock, or its sentinel) and tg[r] bit 0 (the
  // target read GOOD): a known-GOOD target is approached (the table's move;
  // SAMPLE on it), an unknown one is sensed; at the sentinel: E.  An exited
  // robot's sub-action is immaterial (every action is a no-op at EXIT, the
  // table gives E there, never SAMPLE); TRACE reports E for it.
  // One table read per robot: row = the robot's cell when its target is
  // known GOOD, else the SENSE row.
  template <bool TRACE = false>
  static __device__ __forceinline__ void policy(const Sm& sm, const St& s, const uint32_t* q, const uint32_t* tg,
                                                int* b, uint32_t polw, int sense_row) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = (tg[r] & 1u) ? s.cell[r] : sense_row;
      b[r] = (int)hd_dyn_smem[kOffPol + (uint32_t)row * polw + q[r]];
      if (TRACE && exited(sm, s, r)) b[r] = 2;
    }
  }
  template <bool TRACE, class KeyT>
  static __device__ void rollout_generic(const Sm& sm, St s, uint32_t z, uint32_t id, uint32_t t0,
                                         const KeyT& key, double& ret, uint32_t& len, uint64_t& h) {
    double acc = 0.0;
    uint32_t q[R], tg[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      q[r] = sm.qstart[r];
      tg[r] = 0;
    }
    const double* gpk = reinterpret_cast<const double*>(hd_dyn_smem + sm.off_gp10);  // 10 gamma^(t - t0)
    const uint32_t polw = sm.polw;
    const int sense_row = sm.exitc + 1;
    uint32_t t = t0;
    bool term = false;
    while (t < sm.D && !term) {
      int b[R];
      policy<TRACE>(sm, s, q, tg, b, polw, sense_row);
      if (TRACE) {
        int a = 0, mul = 1;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          a += b[r] * mul;
          mul *= sm.base;
        }
        h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
      }
      const uint4 w = philox(id, t + 1, 0u, 0u, key);
      const uint32_t u[2] = {w.x, w.y};
      float r;
      int k10;
      uint32_t zr[R], smp[R];
      term = step_sub(sm, s, b, u, z, r, zr, &k10, smp);
      // memory: a GOOD reading marks the target GOOD; a BAD reading or a
      // SAMPLE (only ever of the target) marks it DONE: next column
#pragma unroll
      for (int k = 0; k < R; ++k) {
        q[k] += (zr[k] >> 1) | smp[k];
        tg[k] = (tg[k] | zr[k]) & ~smp[k];
      }
      acc = __fma_rn(*gpk++, (double)k10, acc);  // + gamma^(t - t0) r, r = 10 k10
      ++t;
    }
    if (!term) acc = __fma_rn(gp(sm, (int)(t - t0)), sm.tail, acc);
    ret = acc;
    len = t - t0;
  }

  // shared-memory loads at explicit 32-bit shared-space addresses (the
  // roll-out computes its table addresses itself, with IMADs)
  static __device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  static __device__ __forceinline__ uint32_t lds16(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  static __device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  // Eq. 12's roll-out, the ALU-lean form (m <= 27; else rollout_generic, the
  // same card): the roll-out is bound by the ALU pipe, so its bit work is
  // reorganised --
  //   * the good-rock mask is kept as g5 = good << 5, so SENSE sub-action
  //     5 + j and the rock table's 5 + j index it directly;
  //   * every table address is computed with IMADs (an opaque 1 for the unit
  //     strides) on shared-space addresses;
  //   * the flags of an action entry come out through multiply-high
  //     extractions (FMA pipe), the next cell by one;
  //   * the policy row is selected arithmetically (tg in {0, 1});
  //   * the memory update needs no reading code: GOOD = SENSE & x,
  //     BAD = SENSE & ~x with x = (good == correct);
  //   * terminal = no robot left (a live count).
  // It computes exactly the card's step and policy (bit-identical outputs).
  template <bool TRACE, class KeyT>
  static __device__ void rollout(const Sm& sm, St s, uint32_t z, uint32_t id, uint32_t t0,
                                 const KeyT& key, double& ret, uint32_t& len, uint64_t& h) {
    if (sm.m > 27) {  // (uniform) the shifted mask would not fit
      rollout_generic<TRACE>(sm, s, z, id, t0, key, ret, len, h);
      return;
    }
    const uint32_t one = sm.one, polw = sm.polw, base = sm.base, mm = sm.mm;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(hd_dyn_smem);
    const uint32_t a_act = sb + sm.off_act, a_thr = sb + sm.off_thr - 20u, a_rock = sb + sm.off_rock;
    const int sense_row = sm.exitc + 1;
    uint32_t g5 = s.good << 5;
    uint32_t qa[R], tg[R];  // qa: shared address of the robot's column in pol row 0
    int live = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      qa[r] = sb + kOffPol + sm.qstart[r];
      tg[r] = 0;
      live += exited(sm, s, r) ? 0 : 1;
    }
    const double* gpk = reinterpret_cast<const double*>(hd_dyn_smem + sm.off_gp10);  // 10 gamma^(t - t0)
    double acc = 0.0;
    uint32_t t = t0;
    while (t < sm.D && live > 0) {
      const uint4 w = philox(id, t + 1, 0u, 0u, key);
      const uint32_t u[2] = {w.x, w.y};
      int k = 0;  // the step's reward / 10
      int a = 0, mul = 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int c = s.cell[r];
        // pi0: row = the cell when the target is known GOOD, else the SENSE row
#if HD_RS_ROWSEL
        const int row = tg[r] ? c : sense_row;
#else
        const int row = sense_row + (int)tg[r] * (c - sense_row);
#endif
        const uint32_t b = lds8((uint32_t)row * polw + qa[r]);
        if (TRACE) {
          a += (exited(sm, s, r) ? 2 : (int)b) * mul;
          mul *= (int)base;
        }
        const uint32_t e = lds16((uint32_t)c * (2u * base) + (b * 2u + a_act));
        const uint32_t thr = lds32((uint32_t)c * (4u * mm) + (b * 4u + a_thr));  // SENSE rock b - 5
#if HD_RS_ONE
        const uint32_t jr5 = lds8((uint32_t)c * one + a_rock);                 // 5 + the rock on the cell
#else
        const uint32_t jr5 = lds8((uint32_t)c + a_rock);                       // 5 + the rock on the cell
#endif
#if HD_RS_SENSE_LOP
        const uint32_t sense = e & 1u;
#else
        const uint32_t sense = __umulhi(e << 31, 2u);
#endif
        const uint32_t samp = __umulhi(e << 30, 2u);
#if HD_RS_EX_SHF
        const uint32_t ex = (e >> 2) & 1u;
#else
        const uint32_t ex = __umulhi(e << 29, 2u);
#endif
        const uint32_t incorrect = u[r] > thr ? 1u : 0u;
        const uint32_t x = ((g5 >> b) ^ incorrect) & 1u;  // 1: the reading says GOOD
        const uint32_t gbit = (g5 >> jr5) & samp;         // SAMPLE of a good rock
        g5 &= ~(gbit << jr5);                              // it turns bad
        k += (int)ex + 2 * (int)gbit - (int)samp;
        live -= (int)ex;
#if HD_RS_CELL_SHF
        s.cell[r] = (int)(e >> 3);                         // the next cell
#else
        s.cell[r] = (int)__umulhi(e, 1u << 29);           // e >> 3: the next cell
#endif
        // memory: GOOD -> target GOOD; BAD or SAMPLE -> target DONE (next column)
#if HD_RS_ONE
        qa[r] += ((sense & ~x) | samp) * one;
#else
        qa[r] += (sense & ~x) | samp;
#endif
        tg[r] = (tg[r] | (sense & x)) & ~samp;
      }
      if (TRACE) h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
      acc = __fma_rn(*gpk++, (double)k, acc);  // + gamma^(t - t0) r, r = 10 k
      ++t;
    }
    if (live > 0) acc = __fma_rn(gp(sm, (int)(t - t0)), sm.tail, acc);
    ret = acc;
    len = t - t0;
  }
};

// ===========================================================================
// Navigation (card §3.3).  word 0: cell | gate<<8 | terminal<<9;
// words 1..NW: occupancy bits of the unknown cells (row-major order).
// actions 0 STAY, 1..8 = N, NE, E, SE, S, SW, W, NW.
//
// Device representation: when a state is loaded, the thread expands it into
// a padded occupancy grid in shared memory (row y+1, bit x+1 = cell (x, y);
// the border, known obstacles and the closed gate are 1).  A step then reads
// three rows and extracts the 3x3 neighbourhood with shifts.
// ===========================================================================
constexpr int kNavRowStride = 19;      // padded rows (n + 2 <= 18), odd stride
constexpr int kNavMaxThreads = 512;    // largest block of a kernel using Nav (K1: one round over K = 500)

template <int NW>
struct Nav {
#ifndef HD_NAV_MINB
#define HD_NAV_MINB 4
#endif
  static constexpr int kMinBlocks = HD_NAV_MINB;  // 4: 102 registers (5 / 4 / 6 measured 85.3 / 83.2 / 92.0 us on config 3)
  static constexpr int kK1Threads = kNavMaxThreads;  // the per-thread grids are sized for it
  struct Sm {
    int32_t n, wall_y, goal_x, goal_y;
    int32_t gate_x[2];
    int32_t n_unknown;
    uint32_t t_fail, t_flip;  // T(p) < 2^32 (checked at load): an event is u < T
    uint32_t D;
    double tail;
    double rew_d[4];          // step rewards by outcome code (stay, move / failed move, crash, goal), as
    float rew_f[4];           //   the card's fp32 constants and their doubles
    double gpow[kGpowN];
    uint32_t known_rows[kNavMaxN + 2];  // padded rows of the border + known obstacles (gates open)
    uint16_t unk_pos[kNavMaxN * kNavMaxN];  // unknown index -> (x+1) | (y+1) << 8
    uint8_t nb_lut[512];      // 3x3 window bits (row above | row | row below, 3 bits each) -> the
                              //   neighbour occupancy bits N, NE, E, SE, S, SW, W, NW
    uint8_t pol_lut[64];      // pi0: (E, SE, S, SW, W readings) | (t odd) << 5 -> action
  };
  // per-action displacement, 2 bits each (d + 1), actions 0 STAY, 1..8 = N, NE, E, SE, S, SW, W, NW
  static constexpr uint32_t kDX = (1u << 0) | (1u << 2) | (2u << 4) | (2u << 6) | (2u << 8) | (1u << 10) | (0u << 12) |
                                  (0u << 14) | (0u << 16);
  static constexpr uint32_t kDY = (1u << 0) | (0u << 2) | (0u << 4) | (1u << 6) | (2u << 8) | (2u << 10) | (2u << 12) |
                                  (1u << 14) | (0u << 16);
  static __device__ void load_sm(Sm& sm, const DevModel& dm, int tid, int nt) {
    if (tid == 0) {
      sm.n = dm.n;
      sm.wall_y = dm.wall_y;
      sm.goal_x = dm.goal_x;
      sm.goal_y = dm.goal_y;
      sm.gate_x[0] = dm.gate_x[0];
      sm.gate_x[1] = dm.gate_x[1];
      sm.n_unknown = dm.nav_unknown;
      sm.t_fail = (uint32_t)dm.t_fail;
      sm.t_flip = (uint32_t)dm.t_flip;
      sm.D = dm.D;
      sm.tail = dm.tail;
      // stay -0.2, failed move -0.1, crash -1 in place, move -0.1, goal +20
      const float rf[4] = {-0.2f, -0.1f, -1.0f, 20.0f};
      for (int k = 0; k < 4; ++k) {
        sm.rew_f[k] = rf[k];
        sm.rew_d[k] = (double)rf[k];
      }
    }
    for (int i = tid; i < 512; i += nt) {
      const uint32_t up = i & 7u, mid = (i >> 3) & 7u, dn = (i >> 6) & 7u;
      sm.nb_lut[i] = (uint8_t)(((up >> 1) & 1u) | ((up >> 1) & 2u) | (mid & 4u) | ((dn & 4u) << 1) |
                               ((dn & 2u) << 3) | ((dn & 1u) << 5) | ((mid & 1u) << 6) | ((up & 1u) << 7));
    }
    for (int i = tid; i < 64; i += nt) {
      // bits of i: 0 E, 1 SE, 2 S, 3 SW, 4 W read occupied; bit 5: t odd
      const bool odd = (i >> 5) & 1;
      const int cand[5] = {5, 4, 6, odd ? 7 : 3, odd ? 3 : 7};  // S, SE, SW, then E/W by parity
      const int bitof[9] = {-1, -1, -1, 0, 1, 2, 3, 4, -1};       // action -> bit of i
      int a = 0;
      for (int k = 4; k >= 0; --k)
        if (!((i >> bitof[cand[k]]) & 1)) a = cand[k];
      sm.pol_lut[i] = (uint8_t)a;
    }
    copy_words(sm.gpow, dm.gpow, sizeof(sm.gpow), tid, nt);
    copy_words(sm.known_rows, dm.nav_known_rows, sizeof(sm.known_rows), tid, nt);
    copy_words(sm.unk_pos, dm.nav_unk_pos, sizeof(sm.unk_pos), tid, nt);
  }
  // Per-thread scratch in the kernel's dynamic shared memory (each kernel
  // places it after its own data and binds the offset before first use): the
  // scenario's padded occupancy rows, sized by the launching block, not by the
  // largest block of any kernel.
  static constexpr uint32_t kScratchPerThread = 4 * kNavRowStride;
  static __device__ __forceinline__ uint32_t& rows_off() {
    __shared__ uint32_t off;
    return off;
  }
  static __device__ __forceinline__ void bind_scratch(uint32_t off) { rows_off() = off; }  // one thread; caller syncs
  static __device__ __forceinline__ uint32_t* grid() {
    return reinterpret_cast<uint32_t*>(hd_dyn_smem + rows_off()) + threadIdx.x * kNavRowStride;
  }
  struct St {
    int32_t x, y;
    uint32_t gate;
    bool term;
    uint32_t nb;  // occupancy of the 8 neighbours of (x, y) (derived: set by load, kept by step)
    uint32_t occ[NW];
  };
  static __device__ __forceinline__ void build_grid(const Sm& sm, const St& s) {
    uint32_t* g = grid();
    for (int r = 0; r < sm.n + 2; ++r) g[r] = sm.known_rows[r];
    const int closed = sm.gate_x[1 - s.gate];
    g[sm.wall_y + 1] |= 1u << (closed + 1);
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      uint32_t bits = s.occ[k];
      while (bits) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1u;
        const uint32_t pos = sm.unk_pos[32 * k + bit];
        g[pos >> 8] |= 1u << (pos & 0xFFu);
      }
    }
  }
  static __device__ __forceinline__ St load(const Sm& sm, const uint32_t* st, uint32_t cap, uint32_t i) {
    St s;
    const uint32_t w0 = st[i];
    const uint32_t cell = w0 & 0xFFu;
    s.y = (int32_t)(cell / (uint32_t)sm.n);
    s.x = (int32_t)cell - s.y * sm.n;
    s.gate = (w0 >> 8) & 1u;
    s.term = (w0 >> 9) & 1u;
#pragma unroll
    for (int k = 0; k < NW; ++k) s.occ[k] = st[(1 + k) * cap + i];
    build_grid(sm, s);
    s.nb = neighbours(sm, s.x, s.y);
    return s;
  }
  static __device__ __forceinline__ void store(const Sm& sm, const St& s, uint32_t* st, uint32_t cap,
                                               uint32_t i) {
    st[i] = (uint32_t)(s.y * sm.n + s.x) | (s.gate << 8) | ((uint32_t)s.term << 9);
#pragma unroll
    for (int k = 0; k < NW; ++k) st[(1 + k) * cap + i] = s.occ[k];
  }
  static __device__ __forceinline__ bool terminal(const Sm&, const St& s) { return s.term; }
  static constexpr uint32_t kTerminalObs = 0x100u;

  // occupancy of the 8 neighbours of (x, y), bit k = direction k+1
  // (N, NE, E, SE, S, SW, W, NW); off-grid counts as occupied: the 3x3 window
  // of the padded grid through a 512-entry table
  static __device__ __forceinline__ uint32_t neighbours(const Sm& sm, int x, int y) {
    const uint32_t* g = grid();
    const uint32_t up = (g[y] >> x) & 7u, mid = (g[y + 1] >> x) & 7u, dn = (g[y + 2] >> x) & 7u;
    return sm.nb_lut[up | (mid << 3) | (dn << 6)];
  }
  // the nine random words of a step (R13): u[0] move failure, u[1..8] the
  // reading flips N .. NW -- blocks 0 and 1 whole, word 0 of block 2
  struct Words {
    uint4 b0, b1;
    uint32_t w8;
  };
  template <class KeyT>
  static __device__ __forceinline__ Words words(uint32_t id, uint32_t t, const KeyT& key) {
    uint4 b[3];
    philox_blocks<3>(id, t, key, b);  // the three blocks' rounds interleaved
    return Words{b[0], b[1], b[2].x};
  }
  // g(s, a, phi_t) on the step's words, branch-free (integer selects) so that
  // roll-out lanes choosing different actions do not diverge; rcode = the
  // outcome (0 stay, 1 move or failed move, 2 crash, 3 goal), whose reward is
  // the card's constant
  static __device__ __forceinline__ bool step_words(const Sm& sm, St& s, int a, const Words& u, uint32_t t_fail,
                                                    uint32_t t_flip, uint32_t& z, int& rcode) {
    const uint32_t go = a != 0 ? 1u : 0u;                        // not STAY
    const uint32_t fail = go & (u.b0.x < t_fail ? 1u : 0u);      // the attempt fails (0.03)
    const uint32_t occ = ((s.nb << 1) >> a) & 1u;                 // the target cell (carried neighbourhood)
    const uint32_t mv = go & ~fail & ~occ & 1u;
    const int dx = (int)((kDX >> (2 * a)) & 3u) - 1, dy = (int)((kDY >> (2 * a)) & 3u) - 1;
    s.x += (int)mv * dx;
    s.y += (int)mv * dy;
    const uint32_t goal = mv & (s.x == sm.goal_x ? 1u : 0u) & (s.y == sm.goal_y ? 1u : 0u);
    rcode = (int)(go * (1u + (occ & ~fail) + 2u * goal));
    s.term = goal != 0;
    const uint32_t flips = (u.b0.y < t_flip ? 1u : 0u) | (u.b0.z < t_flip ? 2u : 0u) | (u.b0.w < t_flip ? 4u : 0u) |
                           (u.b1.x < t_flip ? 8u : 0u) | (u.b1.y < t_flip ? 16u : 0u) |
                           (u.b1.z < t_flip ? 32u : 0u) | (u.b1.w < t_flip ? 64u : 0u) |
                           (u.w8 < t_flip ? 128u : 0u);
    s.nb = neighbours(sm, s.x, s.y);  // of the new cell: the observation, and the next step's moves
    z = goal ? kTerminalObs : (s.nb ^ flips);
    return goal != 0;
  }
  template <class KeyT>
  static __device__ __forceinline__ bool step(const Sm& sm, St& s, int a, uint32_t id, uint32_t t,
                                              const KeyT& key, uint32_t& z, float& r) {
    int rc;
    const bool term = step_words(sm, s, a, words(id, t, key), sm.t_fail, sm.t_flip, z, rc);
    r = sm.rew_f[rc];
    return term;
  }
  static __device__ __forceinline__ double upper(const Sm& sm, const St& s) {
    const int gx = sm.gate_x[s.gate];
    const int W = sm.wall_y, Gx = sm.goal_x, Gy = sm.goal_y;
    int d;
    if (s.y < W) d = max(abs(s.x - gx), W - s.y) + max(abs(gx - Gx), Gy - W);
    else if (s.y == W) d = max(abs(s.x - Gx), Gy - W);
    else d = max(abs(s.x - Gx), Gy - s.y);
    return 20.0 * sm.gpow[d - 1];
  }
  static __device__ __forceinline__ uint32_t initial_obs(const Sm&, const St&) { return 0u; }
  // pi0: first of [S, SE, SW, t even ? E : W, t even ? W : E] read FREE,
  // else STAY -- one table read (the E..W readings are bits 2..6 of z)
  static __device__ __forceinline__ int policy(const Sm& sm, uint32_t z, uint32_t t) {
    return sm.pol_lut[((z >> 2) & 31u) | ((t & 1u) << 5)];
  }
  template <bool TRACE, class KeyT>
  static __device__ void rollout(const Sm& sm, St s, uint32_t z, uint32_t id, uint32_t t0,
                                 const KeyT& key, double& ret, uint32_t& len, uint64_t& h) {
    double acc = 0.0;
    uint32_t t = t0;
    bool term = false;
    const uint32_t t_fail = sm.t_fail, t_flip = sm.t_flip, D = sm.D;
    const double* gp = sm.gpow - t0;  // gamma^(t - t0)
    // the stream words do not depend on the state: each step draws the next
    // step's words while its own state chain runs (instruction-level
    // parallelism for the latency-bound long roll-outs)
    Words u = words(id, t + 1, key);
    while (t < D && !term) {
      const int a = policy(sm, z, t);
      if (TRACE) h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
      const Words cur = u;
      u = words(id, t + 2, key);
      int rc;
      term = step_words(sm, s, a, cur, t_fail, t_flip, z, rc);
      acc = __fma_rn(gp[t], sm.rew_d[rc], acc);
      ++t;
    }
    if (!term) acc = __fma_rn(gp[t], sm.tail, acc);
    ret = acc;
    len = t - t0;
  }
};

}  // namespace hd
