// model_car.cuh -- driving among pedestrians (card §3.4), the
// sparse-observation model.  Two device implementations of the same card:
//   CarThreadT<P>  one thread per scenario (state in registers)
//   (kernels_car.cuh) one warp per scenario, lane i = pedestrian i, lane 31 =
//   the car: the paper's within-step factoring.
// The library is compiled with -fmad=false and IEEE div/sqrt, so every fp32
// operation below rounds exactly as the card's sequence (R16).
#pragma once
#include "common.cuh"
#include "models.cuh"

namespace hd {

__device__ __forceinline__ uint32_t car_bin(float v) {  // (int16) floor(2 v), as 16 bits
  return ((uint32_t)(int)floorf(2.0f * v)) & 0xFFFFu;
}
__device__ __forceinline__ int car_bin_i(float v) { return (int)(int16_t)(int)floorf(2.0f * v); }

// heading-noise rotation (cos, sin) from one random word: tau = (sum of the
// four bytes - 510) * noise, c = (1 - tau^2)/(1 + tau^2), s = 2 tau/(1 + tau^2).
// The byte sum has 1021 values, so the host evaluates that exact fp32
// sequence once per value (libdespot's own table, built at model load) and the
// kernels look it up in shared memory.
__device__ __forceinline__ int car_noise_index(uint32_t w) {
  return (int)__vsadu4(w, 0u);  // the sum of the four bytes: one VABSDIFF4 instruction
}
// one pedestrian toward goal g with rotation (c, sn), speed 1 m/s, dt 0.25
__device__ __forceinline__ void car_ped_move(float& x, float& y, uint32_t g, float c, float sn) {
  const float gx = (g >= 2u) ? 20.0f : 0.0f;
  const float gy = (g & 1u) ? 10.0f : -10.0f;
  const float dx = gx - x, dy = gy - y;
  const float d2 = dx * dx + dy * dy;
  if (!(d2 < 1e-6f)) {
    const float nrm = sqrtf(d2);
    const float ux = dx / nrm, uy = dy / nrm;
    const float hx = ux * c - uy * sn;
    const float hy = ux * sn + uy * c;
    x = x + 0.25f * hx;
    y = y + 0.25f * hy;
  }
}
__device__ __forceinline__ float car_reward(int a, bool coll, bool goal, float v) {
  float r = -0.1f;
  if (a == 2) r = r + (-0.1f);
  if (coll) r = r + (-1000.0f * (v * v + 0.5f));
  if (goal && !coll) r = r + 100.0f;
  return r;
}
__device__ __forceinline__ int car_policy_from_gap(int gap) { return gap <= 8 ? 2 : gap <= 16 ? 0 : 1; }

// EXACT: the model has exactly MAXP pedestrians (no per-pedestrian runtime
// test of the count)
template <int MAXP, bool EXACT = false>
struct CarThreadT {
  static constexpr int kMaxP = MAXP;
  static constexpr uint32_t kScratchPerThread = 0;  // no per-thread shared scratch
  static __device__ __forceinline__ void bind_scratch(uint32_t) {}
  struct Sm {
    int32_t peds;
    uint64_t t_fail;
    float noise;
    uint32_t D, OW;
    double tail;
    double gpow[kGpowN];
    float2 rot[1021];
  };
  static __device__ void load_sm(Sm& sm, const DevModel& dm, int tid, int nt) {
    if (tid == 0) {
      sm.peds = dm.peds;
      sm.t_fail = dm.t_car_fail;
      sm.noise = dm.noise_scale;
      sm.D = dm.D;
      sm.OW = dm.OW;
      sm.tail = dm.tail;
    }
    copy_words(sm.gpow, dm.gpow, sizeof(sm.gpow), tid, nt);
    copy_words(sm.rot, dm.car_rot, sizeof(sm.rot), tid, nt);
  }
  // gap: pi0's input for this state (the nearest pedestrian ahead in the
  // lane, in bins; 255 = none), maintained by load() and step() as they
  // write the positions, so that policy() needs no pass of its own over them
  struct St {
    float xc;
    uint32_t level;
    bool term;
    uint32_t g0, g1;
    int gap;
    float px[MAXP], py[MAXP];
  };
  // The default policy's view of pedestrian (x, y) from car bin cxb (card
  // §3.4): the nearest pedestrian ahead in the lane, min over {x_bin - cxb :
  // x_bin >= cxb, -4 <= y_bin <= 3} capped at 255, the bins floor(2v).  Kept
  // in float compares, without a conversion per pedestrian: y_bin in -4..3
  // <=> -2 <= y < 2, x_bin >= cxb <=> x >= cxb / 2 (both exact), and the
  // minimum bin is the bin of the minimum x (floor is monotone); gap_end
  // converts once.  Equal to the bins' form for |coordinates| < 2^14, which
  // belief_load guarantees for the driving model (reading R21).
  static __device__ __forceinline__ void gap_min(float& mx, float hcx, float x, float y) {
    if (y >= -2.0f && y < 2.0f && x >= hcx) mx = fminf(mx, x);
  }
  static __device__ __forceinline__ int gap_end(float mx, int cxb) {
    if (!(mx < 3.0e38f)) return 255;
    const int g = car_bin_i(mx) - cxb;
    return g < 255 ? g : 255;
  }
  static __device__ __forceinline__ bool active(const Sm& sm, int p) { return p < MAXP && (EXACT || p < sm.peds); }
  static __device__ __forceinline__ St load(const Sm& sm, const uint32_t* st, uint32_t cap, uint32_t i) {
    St s;
    s.xc = __uint_as_float(st[i]);
    const uint32_t w1 = st[cap + i];
    s.level = w1 & 0xFFu;
    s.term = (w1 >> 8) & 1u;
    s.g0 = st[2 * cap + i];
    s.g1 = st[3 * cap + i];
    const int cxb = car_bin_i(s.xc);
    const float hcx = 0.5f * (float)cxb;
    float mx = 3.4e38f;
#pragma unroll
    for (int p = 0; p < MAXP; ++p) {
      if (active(sm, p)) {
        s.px[p] = __uint_as_float(st[(4 + 2 * p) * cap + i]);
        s.py[p] = __uint_as_float(st[(5 + 2 * p) * cap + i]);
        gap_min(mx, hcx, s.px[p], s.py[p]);
      } else {
        s.px[p] = 0.0f;
        s.py[p] = 0.0f;
      }
    }
    s.gap = gap_end(mx, cxb);
    return s;
  }
  static __device__ __forceinline__ void store(const Sm& sm, const St& s, uint32_t* st, uint32_t cap,
                                               uint32_t i) {
    st[i] = __float_as_uint(s.xc);
    st[cap + i] = s.level | ((uint32_t)s.term << 8);
    st[2 * cap + i] = s.g0;
    st[3 * cap + i] = s.g1;
#pragma unroll
    for (int p = 0; p < MAXP; ++p)
      if (active(sm, p)) {
        st[(4 + 2 * p) * cap + i] = __float_as_uint(s.px[p]);
        st[(5 + 2 * p) * cap + i] = __float_as_uint(s.py[p]);
      }
  }
  static __device__ __forceinline__ bool terminal(const Sm&, const St& s) { return s.term; }
  static __device__ __forceinline__ uint32_t goal(const St& s, int p) {
    return ((p < 16 ? s.g0 : s.g1) >> (2 * (p & 15))) & 3u;
  }
  // f(k, word) for every observation word of a non-terminal state, with
  // compile-time pedestrian indices (no dynamic indexing of the state arrays)
  template <class F>
  static __device__ __forceinline__ void for_obs_words(const Sm& sm, const St& s, F&& f) {
    f(0u, car_bin(s.xc) | (s.level << 16));
#pragma unroll
    for (int p = 0; p < MAXP; ++p)
      if (active(sm, p)) f((uint32_t)(1 + p), car_bin(s.px[p]) | (car_bin(s.py[p]) << 16));
  }
  // observation word k (0: car, 1+i: pedestrian i) of a non-terminal state
  static __device__ __forceinline__ uint32_t obs_word(const St& s, int k) {
    if (k == 0) return car_bin(s.xc) | (s.level << 16);
    float x = 0.0f, y = 0.0f;
#pragma unroll
    for (int p = 0; p < MAXP; ++p)
      if (p == k - 1) {
        x = s.px[p];
        y = s.py[p];
      }
    return car_bin(x) | (car_bin(y) << 16);
  }
  template <class KeyT>
  static __device__ __forceinline__ bool step(const Sm& sm, St& s, int a, uint32_t id, uint32_t t,
                                              const KeyT& key, float& r) {
    // random words are drawn one Philox block at a time (block k = words
    // 4k..4k+3: the car's word 0, then pedestrian p's word 1+p), so only four
    // are live at once; the element order (car, then pedestrians ascending)
    // is the card's
    constexpr int NB = (MAXP + 1 + 3) / 4;
    const uint4 w0 = philox(id, t, 0u, 0u, key);
    if (!event(w0.x, sm.t_fail)) {  // Accelerate / Decelerate fail w.p. 0.01
      if (a == 1 && s.level < 4u) s.level += 1u;
      if (a == 2 && s.level > 0u) s.level -= 1u;
    }
    const float v = 0.5f * (float)s.level;
    s.xc = s.xc + v * 0.25f;
    bool coll = false;
    const int cxb = car_bin_i(s.xc);
    const float hcx = 0.5f * (float)cxb;
    float mx = 3.4e38f;
#pragma unroll
    for (int bk = 0; bk < NB; ++bk) {
      if (4 * bk >= (EXACT ? MAXP : sm.peds) + 1) break;  // uniform
      const uint4 w = bk == 0 ? w0 : philox(id, t, (uint32_t)bk, 0u, key);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int p = 4 * bk + q - 1;  // word 4bk+q belongs to pedestrian 4bk+q-1
        if (p >= 0 && active(sm, p)) {
          const float2 cs = sm.rot[car_noise_index(ws[q])];
          car_ped_move(s.px[p], s.py[p], goal(s, p), cs.x, cs.y);
          const float dx = s.px[p] - s.xc;
          coll = coll || (dx * dx + s.py[p] * s.py[p] < 1.0f);
          gap_min(mx, hcx, s.px[p], s.py[p]);
        }
      }
    }
    s.gap = gap_end(mx, cxb);
    const bool g = s.xc >= 20.0f;
    r = car_reward(a, coll, g, v);
    s.term = coll || g;
    return s.term;
  }
  static __device__ __forceinline__ double upper(const Sm& sm, const St& s) {
    int k = (int)ceilf((20.0f - s.xc) * 2.0f);
    k = k < 1 ? 1 : k;
    return 100.0 * sm.gpow[k - 1];
  }
  // pi0 (card §3.4): from the gap load() / step() formed over this state's
  // positions (the bins of the last observation)
  static __device__ __forceinline__ int policy(const Sm&, const St& s) { return car_policy_from_gap(s.gap); }
  static __device__ __forceinline__ uint32_t initial_obs(const Sm&, const St&) { return 0u; }
  template <bool TRACE, class KeyT>
  static __device__ void rollout(const Sm& sm, St s, uint32_t /*z: bins of s*/, uint32_t id, uint32_t t0,
                                 const KeyT& key, double& ret, uint32_t& len, uint64_t& h) {
    double acc = 0.0;
    uint32_t t = t0;
    bool term = false;
    while (t < sm.D && !term) {
      const int a = policy(sm, s);  // reads only the last observation's bins
      if (TRACE) h = (h ^ (uint64_t)(uint32_t)a) * kFnvPrime;
      float r;
      term = step(sm, s, a, id, t + 1, key, r);
      acc += sm.gpow[t - t0] * (double)r;
      ++t;
    }
    if (!term) acc += sm.gpow[t - t0] * sm.tail;
    ret = acc;
    len = t - t0;
  }
};
using CarThread = CarThreadT<kCarMaxPeds>;

}  // namespace hd
