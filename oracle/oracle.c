/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle of HyP-DESPOT's
 * batched leaf expansion (arXiv 1802.06215).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product
 * path.  Shares nothing with paper_1802_06215_b200/csrc (no header, table,
 * constant generator or helper).  Compiled with -O2 -ffp-contract=off
 * -fno-fast-math so that fp32 model arithmetic is plain IEEE (DESIGN.md
 * reading R16).
 *
 * Citations: P:n = line n of PAPER.md; S:n = line n of SPEC.md; "card" =
 * the model cards of DESIGN.md §3; R<n> = reading n of DESIGN.md §2.
 *
 * Parity status per function (see DESIGN.md §4 for the pins):
 *   philox, thresholds, step/upper/rollout of tiger, rocksample, nav: pinned
 *   (KAT vectors, paper constants, closed forms, brute-force bounds); the
 *   default policies and u(s) of rocksample/MARS and nav by hand-traced
 *   roll-outs, every-branch tables, closed forms and BFS distances
 *   (tests/test_oracle_pins_policy.py).
 *   car: step rewards (time, brake, collision, goal), speed clamp, u(s),
 *   pi0's gap rule, step length and mean heading are pinned by closed-form
 *   single steps (tests/test_oracle_pins.py, card §3.4); the heading noise by
 *   its statistics (mean 0, sd pi/8, reading R21).  Every function is
 *   pinned; the driving constants themselves are PROPOSED (the paper defers
 *   the model to Bai 2015, which is not in the reference).
 */
#include "oracle.h"

/* per-scenario word buffers: state words <= 4 + 2*31 = 66 (driving, 31
 * pedestrians), observation words <= 32 */
#define ORACLE_MAXW 128

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* errors                                                                   */
/* ------------------------------------------------------------------------ */
static __thread char g_err[512];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* oracle_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  Each round multiplies */
/* two counter words by M0, M1 into 64-bit products, the key is bumped by    */
/* the Weyl constants W0, W1 between rounds.                                 */
/* ------------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* phi_t of scenario `id` (reading R13): word k of the scenario's
 * random numbers at depth t is Philox(key=(seed_lo, seed_hi),
 * ctr=(id, t, k/4, tag))[k%4].  Fills nwords words. */
static void draw_words(uint64_t seed, uint32_t id, uint32_t t, uint32_t tag, int nwords,
                       uint32_t* u) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int k = 0; k < nwords; ++k) {
    uint32_t ctr[4] = {id, t, (uint32_t)(k / 4), tag};
    uint32_t block[4];
    oracle_philox4x32_10(ctr, key, block);
    u[k] = block[k % 4];
  }
}

/* T(p) = floor(p * 2^32) (reading R14) */
uint64_t oracle_threshold(double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 4294967296ull;
  return (uint64_t)floor(p * 4294967296.0);
}
static int event(uint32_t u, double p) { return (uint64_t)u < oracle_threshold(p); }

/* ------------------------------------------------------------------------ */
/* models                                                                   */
/* ------------------------------------------------------------------------ */
enum { KIND_TIGER = 1, KIND_RS = 2, KIND_NAV = 3, KIND_CAR = 4 };
enum { NAV_FREE = 0, NAV_OBST = 1, NAV_GATE0 = 2, NAV_GATE1 = 3, NAV_UNKNOWN = 4 };

#define MAX_ROCKS 32
#define MAX_CELLS 1024
#define MAX_PEDS 32

typedef struct {
  uint32_t n, depth;
  uint32_t* ids;
  float* w;
  uint32_t* states; /* AoS: states[i*state_words + k] */
  uint64_t seed;     /* stream seed sigma of the belief the node descends from */
  int expanded;
  uint32_t* nchild;  /* [A] */
  uint32_t** keys;   /* [A] -> nchild[a]*obs_words */
} node_t;

struct oracle_model {
  int kind;
  uint32_t A, SW, OW, slots, D, elements;
  double gamma, tail;
  /* tiger */
  double p_listen;
  /* rocksample / MARS */
  int n, m, R;
  int rx[MAX_ROCKS], ry[MAX_ROCKS];
  int sx[2], sy[2];
  double d0;
  int policy_east;
  int order[2][MAX_ROCKS]; /* rocks handled by robot r, sorted (x, y, j) */
  int norder[2];
  /* navigation */
  int wall_y, gate_x[2], goal_x, goal_y;
  int cell_kind[MAX_CELLS], unk_index[MAX_CELLS], n_unknown;
  double p_fail, p_flip;
  /* car */
  int peds;
  double p_car_fail;
  float noise_scale;
  /* nodes */
  node_t** nodes;
  int64_t n_nodes, cap_nodes;
};

/* ---- params "key=value key=value" ---- */
static const char* find_param(const char* params, const char* key, char* buf, size_t bufsz) {
  size_t kl = strlen(key);
  const char* p = params;
  while (p && *p) {
    while (*p == ' ' || *p == '\t' || *p == '\n') ++p;
    if (!*p) break;
    const char* e = p;
    while (*e && *e != ' ' && *e != '\t' && *e != '\n') ++e;
    if ((size_t)(e - p) > kl && strncmp(p, key, kl) == 0 && p[kl] == '=') {
      size_t vl = (size_t)(e - p) - kl - 1;
      if (vl >= bufsz) vl = bufsz - 1;
      memcpy(buf, p + kl + 1, vl);
      buf[vl] = 0;
      return buf;
    }
    p = e;
  }
  return NULL;
}
static double param_d(const char* params, const char* key, double dflt) {
  char buf[64];
  return find_param(params, key, buf, sizeof buf) ? strtod(buf, NULL) : dflt;
}
static long param_i(const char* params, const char* key, long dflt) {
  char buf[64];
  return find_param(params, key, buf, sizeof buf) ? strtol(buf, NULL, 10) : dflt;
}
/* "x:y,x:y,..." -> count */
static int param_xy(const char* params, const char* key, int* xs, int* ys, int maxn) {
  char buf[4096];
  if (!find_param(params, key, buf, sizeof buf)) return -1;
  int cnt = 0;
  char* p = buf;
  while (*p && cnt < maxn) {
    char* e;
    long x = strtol(p, &e, 10);
    if (*e != ':') return -2;
    long y = strtol(e + 1, &e, 10);
    xs[cnt] = (int)x;
    ys[cnt] = (int)y;
    ++cnt;
    if (*e == ',') ++e;
    else if (*e) return -2;
    p = e;
  }
  return cnt;
}
static int param_list(const char* params, const char* key, int* xs, int maxn) {
  char buf[1024];
  if (!find_param(params, key, buf, sizeof buf)) return -1;
  int cnt = 0;
  char* p = buf;
  while (*p && cnt < maxn) {
    char* e;
    xs[cnt++] = (int)strtol(p, &e, 10);
    if (*e == ',') ++e;
    else if (*e) return -2;
    p = e;
  }
  return cnt;
}

static uint32_t ipow(uint32_t b, uint32_t e) {
  uint32_t r = 1;
  while (e--) r *= b;
  return r;
}

/* ---------------------------- Tiger (card §3.1) ------------------------- */
/* state: bit0 = tiger side (0 left, 1 right), bit1 = terminal.
 * actions: 0 LISTEN, 1 OPEN-LEFT, 2 OPEN-RIGHT.  obs: 1 hear-left,
 * 2 hear-right, 3 TERMINAL.                                                  */
static void tiger_step(const oracle_model* M, const uint32_t* s, int a, const uint32_t* u,
                       uint32_t* s2, uint32_t* z, float* r, int* term) {
  uint32_t side = s[0] & 1u;
  if (a == 0) {
    int correct = event(u[0], M->p_listen);
    uint32_t heard = correct ? side : 1u - side;
    *r = -1.0f;
    s2[0] = side;
    *z = 1u + heard;
    *term = 0;
  } else {
    uint32_t door = (uint32_t)(a - 1); /* 0 left, 1 right */
    *r = (door == side) ? -100.0f : 10.0f;
    s2[0] = side | 2u;
    *z = 3u;
    *term = 1;
  }
}

/* ------------------------ RockSample / MARS (card §3.2) ------------------ */
/* state word 0: good-rock bitmask; word 1: 16 bits per robot, cell y*n+x or
 * 0xFFFF when the robot has exited the map.
 * per-robot sub-actions: 0 N, 1 S, 2 E, 3 W, 4 SAMPLE, 5+j SENSE j.        */
#define RS_EXITED 0xFFFFu
static int rs_rock_at(const oracle_model* M, int x, int y) {
  for (int j = 0; j < M->m; ++j)
    if (M->rx[j] == x && M->ry[j] == y) return j;
  return -1;
}
static int rs_terminal(const oracle_model* M, const uint32_t* s) {
  for (int r = 0; r < M->R; ++r)
    if (((s[1] >> (16 * r)) & 0xFFFFu) != RS_EXITED) return 0;
  return 1;
}
/* sensing accuracy 0.5 (1 + 2^(-d/d0)) ("decreasing exponentially";
 * S:390 curve; reading R17) */
static double rs_sense_accuracy(const oracle_model* M, int d2) {
  return 0.5 * (1.0 + pow(2.0, -sqrt((double)d2) / M->d0));
}
static void rs_step_sub(const oracle_model* M, const uint32_t* s, const int* b, const uint32_t* u,
                        uint32_t* s2, uint32_t* z, float* r, int* term) {
  uint32_t good = s[0];
  uint32_t pos = s[1];
  float reward = 0.0f;
  uint32_t zsum = 0;
  for (int rb = 0; rb < M->R; ++rb) {
    uint32_t cell = (pos >> (16 * rb)) & 0xFFFFu;
    uint32_t zr = 0; /* NONE */
    if (cell != RS_EXITED) {
      int x = (int)(cell % (uint32_t)M->n), y = (int)(cell / (uint32_t)M->n);
      int exited = 0;
      int sub = b[rb];
      if (sub == 0) {
        if (y > 0) y -= 1;
      } else if (sub == 1) {
        if (y < M->n - 1) y += 1;
      } else if (sub == 2) {
        if (x < M->n - 1) x += 1;
        else {
          exited = 1;
          reward = reward + 10.0f; /* "+10 reward upon reaching the east border" P:530 */
        }
      } else if (sub == 3) {
        if (x > 0) x -= 1;
      } else if (sub == 4) {
        int j = rs_rock_at(M, x, y);
        if (j >= 0) {
          if (good & (1u << j)) {
            reward = reward + 10.0f;
            good &= ~(1u << j);      /* sampled rock becomes bad */
          } else {
            reward = reward + (-10.0f);
          }
        }
      } else {
        int j = sub - 5;
        int dx = x - M->rx[j], dy = y - M->ry[j];
        int correct = event(u[rb], rs_sense_accuracy(M, dx * dx + dy * dy));
        int isgood = (good >> j) & 1u;
        zr = (isgood == correct) ? 1u : 2u; /* GOOD : BAD */
      }
      uint32_t field = exited ? RS_EXITED : (uint32_t)(y * M->n + x);
      pos = (pos & ~(0xFFFFu << (16 * rb))) | (field << (16 * rb));
    }
    zsum += zr * ipow(3, (uint32_t)rb);
  }
  s2[0] = good;
  s2[1] = pos;
  *r = reward;
  *term = rs_terminal(M, s2);
  *z = *term ? ipow(3, (uint32_t)M->R) : zsum;
}
static void rs_decode(const oracle_model* M, int a, int* b) {
  int base = 5 + M->m;
  for (int r = 0; r < M->R; ++r) {
    b[r] = a % base;
    a /= base;
  }
}
static int rs_encode(const oracle_model* M, const int* b) {
  int base = 5 + M->m, a = 0, mul = 1;
  for (int r = 0; r < M->R; ++r) {
    a += b[r] * mul;
    mul *= base;
  }
  return a;
}
/* u(s) = sum_{good j} 10 gamma^{min_r dist(r,j)} + sum_r 10 gamma^{n-1-x_r} */
static double rs_upper(const oracle_model* M, const uint32_t* s) {
  if (rs_terminal(M, s)) return 0.0;
  double u = 0.0;
  for (int j = 0; j < M->m; ++j) {
    if (!((s[0] >> j) & 1u)) continue;
    int dmin = 1 << 30;
    for (int r = 0; r < M->R; ++r) {
      uint32_t cell = (s[1] >> (16 * r)) & 0xFFFFu;
      if (cell == RS_EXITED) continue;
      int x = (int)(cell % (uint32_t)M->n), y = (int)(cell / (uint32_t)M->n);
      int d = abs(x - M->rx[j]) + abs(y - M->ry[j]);
      if (d < dmin) dmin = d;
    }
    u += 10.0 * pow(M->gamma, (double)dmin);
  }
  for (int r = 0; r < M->R; ++r) {
    uint32_t cell = (s[1] >> (16 * r)) & 0xFFFFu;
    if (cell == RS_EXITED) continue;
    int x = (int)(cell % (uint32_t)M->n);
    u += 10.0 * pow(M->gamma, (double)(M->n - 1 - x));
  }
  return u;
}
/* default policy (card §3.2): memory holds 2 bits per rock:
 * 0 UNKNOWN, 1 GOOD, 2 DONE.                                                */
static int rs_status(uint64_t mem, int j) { return (int)((mem >> (2 * j)) & 3u); }
static uint64_t rs_set_status(uint64_t mem, int j, int st) {
  mem &= ~(3ull << (2 * j));
  return mem | ((uint64_t)st << (2 * j));
}
static void rs_policy(const oracle_model* M, const uint32_t* s, uint64_t mem, int* b) {
  for (int r = 0; r < M->R; ++r) {
    uint32_t cell = (s[1] >> (16 * r)) & 0xFFFFu;
    if (M->policy_east || cell == RS_EXITED) {
      b[r] = 2;
      continue;
    }
    int x = (int)(cell % (uint32_t)M->n), y = (int)(cell / (uint32_t)M->n);
    int target = -1;
    for (int k = 0; k < M->norder[r]; ++k) {
      int j = M->order[r][k];
      if (rs_status(mem, j) != 2) {
        target = j;
        break;
      }
    }
    if (target < 0) b[r] = 2;
    else if (rs_status(mem, target) == 0) b[r] = 5 + target;
    else if (x == M->rx[target] && y == M->ry[target]) b[r] = 4;
    else if (x < M->rx[target]) b[r] = 2;
    else if (x > M->rx[target]) b[r] = 3;
    else if (y < M->ry[target]) b[r] = 1;
    else b[r] = 0;
  }
}
static uint64_t rs_policy_update(const oracle_model* M, const uint32_t* s, uint64_t mem,
                                 const int* b, uint32_t z) {
  for (int r = 0; r < M->R; ++r) {
    uint32_t zr = (z / ipow(3, (uint32_t)r)) % 3u;
    if (b[r] >= 5) {
      int j = b[r] - 5;
      mem = rs_set_status(mem, j, zr == 1u ? 1 : 2);
    } else if (b[r] == 4) {
      uint32_t cell = (s[1] >> (16 * r)) & 0xFFFFu;
      if (cell != RS_EXITED) {
        int j = rs_rock_at(M, (int)(cell % (uint32_t)M->n), (int)(cell / (uint32_t)M->n));
        if (j >= 0) mem = rs_set_status(mem, j, 2);
      }
    }
  }
  return mem;
}

/* ------------------------ Navigation (card §3.3) ------------------------- */
/* word 0: cell | gate<<8 | terminal<<9; words 1..: unknown-cell occupancy.  */
static const int NAV_DX[9] = {0, 0, 1, 1, 1, 0, -1, -1, -1};
static const int NAV_DY[9] = {0, -1, -1, 0, 1, 1, 1, 0, -1};
static int nav_occupied(const oracle_model* M, const uint32_t* s, int x, int y) {
  if (x < 0 || y < 0 || x >= M->n || y >= M->n) return 1;
  int c = y * M->n + x;
  int kind = M->cell_kind[c];
  uint32_t gate = (s[0] >> 8) & 1u;
  if (kind == NAV_FREE) return 0;
  if (kind == NAV_OBST) return 1;
  if (kind == NAV_GATE0) return gate == 0 ? 0 : 1;
  if (kind == NAV_GATE1) return gate == 1 ? 0 : 1;
  int idx = M->unk_index[c];
  return (int)((s[1 + idx / 32] >> (idx % 32)) & 1u);
}
static void nav_step(const oracle_model* M, const uint32_t* s, int a, const uint32_t* u,
                     uint32_t* s2, uint32_t* z, float* r, int* term) {
  int cell = (int)(s[0] & 0xFFu);
  int x = cell % M->n, y = cell / M->n;
  for (uint32_t k = 0; k < M->SW; ++k) s2[k] = s[k];
  *term = 0;
  if (a == 0) {
    *r = -0.2f; /* "Staying still is discouraged by a small penalty (-0.2)" P:497 */
  } else if (event(u[0], M->p_fail)) {
    *r = -0.1f; /* failed move: robot stays, pays the motion cost (card) */
  } else {
    int tx = x + NAV_DX[a], ty = y + NAV_DY[a];
    if (nav_occupied(M, s, tx, ty)) {
      *r = -1.0f; /* crash penalty (-1), position unchanged */
    } else {
      x = tx;
      y = ty;
      if (x == M->goal_x && y == M->goal_y) {
        *r = 20.0f; /* goal reward (+20), the world terminates */
        *term = 1;
      } else {
        *r = -0.1f; /* motion cost (-0.1) P:497 */
      }
    }
  }
  s2[0] = (uint32_t)(y * M->n + x) | (s[0] & 0x100u) | ((uint32_t)(*term) << 9);
  if (*term) {
    *z = 0x100u;
    return;
  }
  uint32_t obs = 0;
  for (int k = 0; k < 8; ++k) {
    int occ = nav_occupied(M, s2, x + NAV_DX[k + 1], y + NAV_DY[k + 1]);
    int flip = event(u[1 + k], M->p_flip);
    obs |= (uint32_t)(occ ^ flip) << k;
  }
  *z = obs;
}
static int nav_terminal(const uint32_t* s) { return (int)((s[0] >> 9) & 1u); }
static int imax(int a, int b) { return a > b ? a : b; }
/* u = 20 gamma^{d-1}, d = Chebyshev distance to the goal through the gate */
static double nav_upper(const oracle_model* M, const uint32_t* s) {
  if (nav_terminal(s)) return 0.0;
  int cell = (int)(s[0] & 0xFFu);
  int x = cell % M->n, y = cell / M->n;
  int gx = M->gate_x[(s[0] >> 8) & 1u];
  int W = M->wall_y, Gx = M->goal_x, Gy = M->goal_y;
  int d;
  if (y < W) d = imax(abs(x - gx), W - y) + imax(abs(gx - Gx), Gy - W);
  else if (y == W) d = imax(abs(x - Gx), Gy - W);
  else d = imax(abs(x - Gx), Gy - y);
  return 20.0 * pow(M->gamma, (double)(d - 1));
}
/* pi0: first of [S, SE, SW, t even ? E : W, t even ? W : E] read FREE */
static int nav_policy(uint32_t z, uint32_t t) {
  int even = (t % 2u) == 0u;
  int cand[5] = {5, 4, 6, even ? 3 : 7, even ? 7 : 3};
  for (int k = 0; k < 5; ++k)
    if (((z >> (cand[k] - 1)) & 1u) == 0u) return cand[k];
  return 0;
}

/* ------------------------ Driving (card §3.4) ---------------------------- */
/* word 0: car x (f32 bits); word 1: speed level | terminal<<8;
 * words 2,3: pedestrian goals, 2 bits each; words 4+2i, 5+2i: x_i, y_i.     */
static float f_of(uint32_t w) {
  float f;
  memcpy(&f, &w, 4);
  return f;
}
static uint32_t u_of(float f) {
  uint32_t w;
  memcpy(&w, &f, 4);
  return w;
}
static const float CAR_GX[4] = {0.0f, 0.0f, 20.0f, 20.0f};
static const float CAR_GY[4] = {-10.0f, 10.0f, -10.0f, 10.0f};
#define CAR_STEP 0.25f
#define CAR_DT 0.25f
#define CAR_GOAL 20.0f
static int car_terminal(const uint32_t* s) { return (int)((s[1] >> 8) & 1u); }
static uint32_t car_goal(const uint32_t* s, int i) {
  return (s[2 + i / 16] >> (2 * (i % 16))) & 3u;
}
static uint32_t car_bins(float x, float y) {
  int16_t bx = (int16_t)floorf(2.0f * x), by = (int16_t)floorf(2.0f * y);
  return (uint32_t)(uint16_t)bx | ((uint32_t)(uint16_t)by << 16);
}
static void car_observe(const oracle_model* M, const uint32_t* s, uint32_t* z) {
  float xc = f_of(s[0]);
  uint32_t level = s[1] & 0xFFu;
  z[0] = (uint32_t)(uint16_t)(int16_t)floorf(2.0f * xc) | (level << 16);
  for (int i = 0; i < M->peds; ++i) z[1 + i] = car_bins(f_of(s[4 + 2 * i]), f_of(s[5 + 2 * i]));
}
static void car_step(const oracle_model* M, const uint32_t* s, int a, const uint32_t* u,
                     uint32_t* s2, uint32_t* z, float* r, int* term) {
  for (uint32_t k = 0; k < M->SW; ++k) s2[k] = s[k];
  /* 1. the car: Accelerate / Decelerate fail with probability 0.01 */
  uint32_t level = s[1] & 0xFFu;
  if (!event(u[0], M->p_car_fail)) {
    if (a == 1 && level < 4u) level += 1u;
    if (a == 2 && level > 0u) level -= 1u;
  }
  float v = 0.5f * (float)level;
  float xc = f_of(s[0]);
  xc = xc + v * CAR_DT;
  /* 2. pedestrians move toward their goals with heading noise */
  int collision = 0;
  for (int i = 0; i < M->peds; ++i) {
    float x = f_of(s[4 + 2 * i]), y = f_of(s[5 + 2 * i]);
    uint32_t g = car_goal(s, i);
    uint32_t w = u[1 + i];
    int sint = (int)(w & 0xFFu) + (int)((w >> 8) & 0xFFu) + (int)((w >> 16) & 0xFFu) +
               (int)((w >> 24) & 0xFFu) - 510;
    float tau = (float)sint * M->noise_scale;
    float tt = tau * tau;
    float den = 1.0f + tt;
    float c = (1.0f - tt) / den;
    float sn = (tau + tau) / den;
    float dx = CAR_GX[g] - x, dy = CAR_GY[g] - y;
    float d2 = dx * dx + dy * dy;
    if (!(d2 < 1e-6f)) {
      float nrm = sqrtf(d2);
      float ux = dx / nrm, uy = dy / nrm;
      float hx = ux * c - uy * sn;
      float hy = ux * sn + uy * c;
      x = x + CAR_STEP * hx;
      y = y + CAR_STEP * hy;
    }
    s2[4 + 2 * i] = u_of(x);
    s2[5 + 2 * i] = u_of(y);
  }
  /* 3. collision, 4. goal */
  for (int i = 0; i < M->peds; ++i) {
    float dx = f_of(s2[4 + 2 * i]) - xc, y = f_of(s2[5 + 2 * i]);
    if (dx * dx + y * y < 1.0f) collision = 1;
  }
  int goal = xc >= CAR_GOAL;
  float rew = -0.1f;
  if (a == 2) rew = rew + (-0.1f);
  if (collision) rew = rew + (-1000.0f * (v * v + 0.5f));
  if (goal && !collision) rew = rew + 100.0f;
  *term = collision || goal;
  s2[0] = u_of(xc);
  s2[1] = level | ((uint32_t)(*term) << 8);
  *r = rew;
  if (*term) {
    z[0] = 0xFFFFFFFFu;
    for (uint32_t k = 1; k < M->OW; ++k) z[k] = 0;
  } else {
    car_observe(M, s2, z);
  }
}
static double car_upper(const oracle_model* M, const uint32_t* s) {
  if (car_terminal(s)) return 0.0;
  int k = (int)ceilf((CAR_GOAL - f_of(s[0])) * 2.0f);
  if (k < 1) k = 1;
  return 100.0 * pow(M->gamma, (double)(k - 1));
}
static int car_policy(const oracle_model* M, const uint32_t* z) {
  int cxb = (int16_t)(z[0] & 0xFFFFu);
  int gap = 255;
  for (int i = 0; i < M->peds; ++i) {
    int pxb = (int16_t)(z[1 + i] & 0xFFFFu), pyb = (int16_t)(z[1 + i] >> 16);
    if (pxb >= cxb && pyb >= -4 && pyb <= 3 && pxb - cxb < gap) gap = pxb - cxb;
  }
  if (gap <= 8) return 2;  /* DECELERATE */
  if (gap <= 16) return 0; /* MAINTAIN */
  return 1;                /* ACCELERATE */
}

/* ------------------------------------------------------------------------ */
/* generic model interface                                                  */
/* ------------------------------------------------------------------------ */
static int is_terminal(const oracle_model* M, const uint32_t* s) {
  switch (M->kind) {
    case KIND_TIGER: return (int)((s[0] >> 1) & 1u);
    case KIND_RS: return rs_terminal(M, s);
    case KIND_NAV: return nav_terminal(s);
    default: return car_terminal(s);
  }
}
static void terminal_obs(const oracle_model* M, uint32_t* z) {
  for (uint32_t k = 0; k < M->OW; ++k) z[k] = 0;
  if (M->kind == KIND_TIGER) z[0] = 3u;
  else if (M->kind == KIND_RS) z[0] = ipow(3, (uint32_t)M->R);
  else if (M->kind == KIND_NAV) z[0] = 0x100u;
  else z[0] = 0xFFFFFFFFu;
}
static int words_per_step(const oracle_model* M) {
  switch (M->kind) {
    case KIND_TIGER: return 1;
    case KIND_RS: return M->R;
    case KIND_NAV: return 9;
    default: return 1 + M->peds;
  }
}

/* STEP_OR_TERM (reading R7): a terminal state steps to itself with the
 * TERMINAL observation and reward 0, and is not counted as a scenario-step. */
static int step_or_term(const oracle_model* M, const uint32_t* s, int a, uint32_t id, uint32_t t,
                        uint64_t seed, uint32_t* s2, uint32_t* z, float* r, int* term) {
  if (is_terminal(M, s)) {
    for (uint32_t k = 0; k < M->SW; ++k) s2[k] = s[k];
    terminal_obs(M, z);
    *r = 0.0f;
    *term = 1;
    return 0;
  }
  uint32_t u[MAX_PEDS + 9];
  draw_words(seed, id, t, 0, words_per_step(M), u);
  switch (M->kind) {
    case KIND_TIGER: tiger_step(M, s, a, u, s2, z, r, term); break;
    case KIND_RS: {
      int b[2];
      rs_decode(M, a, b);
      rs_step_sub(M, s, b, u, s2, z, r, term);
      break;
    }
    case KIND_NAV: nav_step(M, s, a, u, s2, z, r, term); break;
    default: car_step(M, s, a, u, s2, z, r, term); break;
  }
  return 1;
}

static double upper_of(const oracle_model* M, const uint32_t* s) {
  switch (M->kind) {
    case KIND_TIGER: return is_terminal(M, s) ? 0.0 : 10.0;
    case KIND_RS: return rs_upper(M, s);
    case KIND_NAV: return nav_upper(M, s);
    default: return car_upper(M, s);
  }
}

static void initial_obs(const oracle_model* M, const uint32_t* s, uint32_t* z) {
  for (uint32_t k = 0; k < M->OW; ++k) z[k] = 0;
  if (M->kind == KIND_CAR && !is_terminal(M, s)) car_observe(M, s, z);
}

/* pi0 (card): a function of (policy memory, last observation, the
 * history-determined parts of the state, depth) */
static int policy_action(const oracle_model* M, const uint32_t* s, const uint32_t* z, uint64_t mem,
                         uint32_t t, int* b) {
  switch (M->kind) {
    case KIND_TIGER: return 0; /* Listen always */
    case KIND_RS: rs_policy(M, s, mem, b); return rs_encode(M, b);
    case KIND_NAV: return nav_policy(z[0], t);
    default: return car_policy(M, z);
  }
}

/* ROLLOUT (Eq. 12): follow pi0 from s at absolute
 * depth d0 until terminal or depth D, then add gamma^{D-d0} * tail. */
static void rollout(const oracle_model* M, const uint32_t* s_in, const uint32_t* z_in, uint32_t id,
                    uint32_t d0, uint64_t seed, double* ret_out, uint32_t* len_out,
                    uint64_t* hash_out, uint64_t* steps) {
  uint32_t s[ORACLE_MAXW], s2[ORACLE_MAXW], z[ORACLE_MAXW];
  memcpy(s, s_in, M->SW * 4);
  memcpy(z, z_in, M->OW * 4);
  double ret = 0.0, disc = 1.0;
  uint64_t mem = 0;
  uint32_t t = d0;
  uint64_t h = 0xcbf29ce484222325ull; /* FNV-1a 64 offset basis */
  while (t < M->D && !is_terminal(M, s)) {
    int b[2] = {0, 0};
    int a = policy_action(M, s, z, mem, t, b);
    h = (h ^ (uint64_t)(uint32_t)a) * 0x100000001b3ull; /* FNV-1a 64 prime */
    float r;
    int term;
    *steps += (uint64_t)step_or_term(M, s, a, id, t + 1, seed, s2, z, &r, &term);
    if (M->kind == KIND_RS) mem = rs_policy_update(M, s, mem, b, z[0]);
    memcpy(s, s2, M->SW * 4);
    ret += disc * (double)r;
    disc *= M->gamma;
    t += 1;
  }
  if (!is_terminal(M, s)) ret += disc * M->tail;
  *ret_out = ret;
  *len_out = t - d0;
  *hash_out = h;
}

/* ------------------------------------------------------------------------ */
/* load                                                                     */
/* ------------------------------------------------------------------------ */
int oracle_model_load(const char* kind, const char* params, oracle_model** out) {
  if (!kind || !out) return fail(-1, "null argument");
  if (!params) params = "";
  oracle_model* M = (oracle_model*)calloc(1, sizeof *M);
  M->gamma = param_d(params, "gamma", 0.95);
  M->elements = 1;
  if (!strcmp(kind, "tiger")) {
    M->kind = KIND_TIGER;
    M->A = 3; M->SW = 1; M->OW = 1; M->slots = 4;
    M->D = (uint32_t)param_i(params, "D", 10);
    M->p_listen = param_d(params, "p_listen", 0.85);
    M->tail = 0.0;
  } else if (!strcmp(kind, "rocksample")) {
    M->kind = KIND_RS;
    M->n = (int)param_i(params, "n", 7);
    M->R = (int)param_i(params, "robots", 1);
    M->d0 = param_d(params, "d0", 4.0);
    M->m = param_xy(params, "rocks", M->rx, M->ry, MAX_ROCKS);
    int ns = param_xy(params, "starts", M->sx, M->sy, 2);
    char pol[32];
    M->policy_east = find_param(params, "policy", pol, sizeof pol) && !strcmp(pol, "east");
    if (M->m < 0 || M->m > 31 || M->R < 1 || M->R > 2 || ns != M->R || M->n < 1 ||
        M->n * M->n > 65535) {
      free(M);
      return fail(-1, "rocksample: bad params (need n, robots<=2, rocks<=31, starts)");
    }
    M->A = ipow((uint32_t)(5 + M->m), (uint32_t)M->R);
    M->SW = 2; M->OW = 1; M->slots = ipow(3, (uint32_t)M->R) + 1;
    M->D = (uint32_t)param_i(params, "D", 20);
    M->tail = 0.0;
    M->elements = (uint32_t)M->R;
    /* pi0 rock order: rocks with j mod R == r, sorted by (x, y, j) */
    for (int r = 0; r < M->R; ++r) {
      M->norder[r] = 0;
      for (int j = 0; j < M->m; ++j) {
        if (j % M->R != r) continue;
        int k = M->norder[r]++;
        M->order[r][k] = j;
        while (k > 0) {
          int p = M->order[r][k - 1], q = M->order[r][k];
          int less = (M->rx[q] < M->rx[p]) || (M->rx[q] == M->rx[p] && M->ry[q] < M->ry[p]) ||
                     (M->rx[q] == M->rx[p] && M->ry[q] == M->ry[p] && q < p);
          if (!less) break;
          M->order[r][k - 1] = q;
          M->order[r][k] = p;
          --k;
        }
      }
    }
  } else if (!strcmp(kind, "nav")) {
    M->kind = KIND_NAV;
    M->n = (int)param_i(params, "n", 13);
    M->wall_y = (int)param_i(params, "wall_y", M->n / 2);
    int gates[2];
    if (param_list(params, "gates", gates, 2) != 2) {
      gates[0] = 3;
      gates[1] = 9;
    }
    M->gate_x[0] = gates[0];
    M->gate_x[1] = gates[1];
    int gx[1], gy[1];
    if (param_xy(params, "goal", gx, gy, 1) == 1) {
      M->goal_x = gx[0];
      M->goal_y = gy[0];
    } else {
      M->goal_x = M->n / 2;
      M->goal_y = M->n - 1;
    }
    int lx[64], ly[64];
    int nl = param_xy(params, "landmarks", lx, ly, 64);
    if (nl < 0) nl = 0;
    M->p_fail = param_d(params, "p_fail", 0.03);
    M->p_flip = param_d(params, "p_flip", 0.03);
    if (M->n < 3 || M->n > 16 || M->wall_y <= 0 || M->wall_y >= M->n - 1) {
      free(M);
      return fail(-1, "nav: bad params");
    }
    M->n_unknown = 0;
    for (int y = 0; y < M->n; ++y) {
      for (int x = 0; x < M->n; ++x) {
        int c = y * M->n + x, kindc = NAV_UNKNOWN;
        if (y == 0 || y == M->n - 1) kindc = NAV_FREE;
        else if (y == M->wall_y) kindc = x == M->gate_x[0] ? NAV_GATE0 : x == M->gate_x[1] ? NAV_GATE1 : NAV_OBST;
        else {
          for (int l = 0; l < nl; ++l)
            if (lx[l] == x && ly[l] == y) kindc = NAV_OBST;
        }
        M->cell_kind[c] = kindc;
        M->unk_index[c] = kindc == NAV_UNKNOWN ? M->n_unknown++ : -1;
      }
    }
    M->A = 9; M->SW = 1 + (uint32_t)((M->n_unknown + 31) / 32); M->OW = 1; M->slots = 257;
    M->D = (uint32_t)param_i(params, "D", 90);
    /* tail: value of staying forever, -0.2 / (1 - gamma) (reading R6) */
    M->tail = (double)(-0.2f) / (1.0 - M->gamma);
  } else if (!strcmp(kind, "car")) {
    M->kind = KIND_CAR;
    M->peds = (int)param_i(params, "peds", 20);
    if (M->peds < 1 || M->peds > 31) {
      free(M);
      return fail(-1, "car: 1 <= peds <= 31");
    }
    M->p_car_fail = param_d(params, "p_fail", 0.01);
    M->noise_scale = (float)param_d(params, "noise", 0.001375); /* sd of 2 atan(tau) = pi/8 (card sigma) */
    M->A = 3; M->SW = 4 + 2 * (uint32_t)M->peds; M->OW = 1 + (uint32_t)M->peds; M->slots = 0;
    M->D = (uint32_t)param_i(params, "D", 90);
    M->elements = 1 + (uint32_t)M->peds;
    M->tail = (double)(-0.1f) / (1.0 - M->gamma);
  } else {
    free(M);
    return fail(-1, "unknown model kind");
  }
  if (!(M->gamma > 0.0 && M->gamma < 1.0) || M->D < 1) {
    free(M);
    return fail(-1, "need 0 < gamma < 1 and D >= 1");
  }
  *out = M;
  return 0;
}

static void node_free(node_t* nd, uint32_t A) {
  if (!nd) return;
  free(nd->ids);
  free(nd->w);
  free(nd->states);
  if (nd->keys) {
    for (uint32_t a = 0; a < A; ++a) free(nd->keys[a]);
    free(nd->keys);
  }
  free(nd->nchild);
  free(nd);
}

void oracle_model_free(oracle_model* M) {
  if (!M) return;
  for (int64_t i = 0; i < M->n_nodes; ++i) node_free(M->nodes[i], M->A);
  free(M->nodes);
  free(M);
}

int oracle_model_info_get(const oracle_model* M, oracle_model_info* o) {
  if (!M || !o) return fail(-1, "null argument");
  o->num_actions = M->A;
  o->state_words = M->SW;
  o->obs_words = M->OW;
  o->obs_slots = M->slots;
  o->max_depth = M->D;
  o->elements = M->elements;
  o->gamma = M->gamma;
  o->tail = M->tail;
  return 0;
}

int oracle_step(const oracle_model* M, const uint32_t* s, int32_t a, uint32_t id, uint32_t t,
                uint64_t seed, uint32_t* s_out, uint32_t* z_out, float* r_out, int32_t* term_out) {
  if (a < 0 || (uint32_t)a >= M->A) return fail(-2, "action out of range");
  int term;
  int counted = step_or_term(M, s, a, id, t, seed, s_out, z_out, r_out, &term);
  *term_out = term;
  return counted;
}

double oracle_upper(const oracle_model* M, const uint32_t* s) { return upper_of(M, s); }

int oracle_rollout(const oracle_model* M, const uint32_t* s, const uint32_t* z, uint32_t id,
                   uint32_t depth, uint64_t seed, double* ret, uint32_t* len, uint64_t* hash,
                   uint64_t* steps) {
  uint32_t z0[ORACLE_MAXW];
  if (!z) {
    initial_obs(M, s, z0);
    z = z0;
  }
  uint64_t st = 0;
  rollout(M, s, z, id, depth, seed, ret, len, hash, &st);
  if (steps) *steps = st;
  return 0;
}

int32_t oracle_default_action(const oracle_model* M, const uint32_t* s, const uint32_t* z,
                              uint64_t memory, uint32_t t) {
  int b[2];
  return policy_action(M, s, z, memory, t, b);
}

/* ------------------------------------------------------------------------ */
/* nodes                                                                    */
/* ------------------------------------------------------------------------ */
static int64_t add_node(oracle_model* M, node_t* nd) {
  if (M->n_nodes == M->cap_nodes) {
    M->cap_nodes = M->cap_nodes ? 2 * M->cap_nodes : 64;
    M->nodes = (node_t**)realloc(M->nodes, (size_t)M->cap_nodes * sizeof(node_t*));
  }
  M->nodes[M->n_nodes++] = nd;
  return M->n_nodes; /* handle = index + 1 */
}
static node_t* get_node(const oracle_model* M, int64_t h) {
  if (h < 1 || h > M->n_nodes) return NULL;
  return M->nodes[h - 1];
}
static node_t* new_node(const oracle_model* M, uint32_t n, uint32_t depth) {
  node_t* nd = (node_t*)calloc(1, sizeof *nd);
  nd->n = n;
  nd->depth = depth;
  nd->ids = (uint32_t*)malloc((n ? n : 1) * 4);
  nd->w = (float*)malloc((n ? n : 1) * 4);
  nd->states = (uint32_t*)malloc((size_t)(n ? n : 1) * M->SW * 4);
  return nd;
}

int64_t oracle_belief_load(oracle_model* M, const uint32_t* states_soa, const float* weights,
                           uint32_t K, uint64_t seed) {
  if (K == 0) return fail(-1, "empty belief");
  for (uint32_t i = 0; i < K; ++i)
    if (!(weights[i] > 0.0f)) return fail(-1, "weights must be > 0");
  node_t* nd = new_node(M, K, 0);
  for (uint32_t i = 0; i < K; ++i) {
    nd->ids[i] = i;
    nd->w[i] = weights[i];
    for (uint32_t k = 0; k < M->SW; ++k) nd->states[(size_t)i * M->SW + k] = states_soa[(size_t)k * K + i];
  }
  nd->seed = seed;
  return add_node(M, nd);
}

int oracle_node_size(const oracle_model* M, int64_t h, uint32_t* n, uint32_t* depth) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  if (n) *n = nd->n;
  if (depth) *depth = nd->depth;
  return 0;
}
int oracle_node_read(const oracle_model* M, int64_t h, uint32_t* ids, float* w,
                     uint32_t* states_soa) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  for (uint32_t i = 0; i < nd->n; ++i) {
    if (ids) ids[i] = nd->ids[i];
    if (w) w[i] = nd->w[i];
    if (states_soa)
      for (uint32_t k = 0; k < M->SW; ++k) states_soa[(size_t)k * nd->n + i] = nd->states[(size_t)i * M->SW + k];
  }
  return 0;
}
int oracle_node_release(oracle_model* M, int64_t h) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  node_free(nd, M->A);
  M->nodes[h - 1] = NULL;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* ORACLE_EXPAND                                                            */
/* ------------------------------------------------------------------------ */
static int keys_equal(const uint32_t* a, const uint32_t* b, uint32_t w) {
  for (uint32_t k = 0; k < w; ++k)
    if (a[k] != b[k]) return 0;
  return 1;
}

int oracle_expand_batch(oracle_model* M, const oracle_leaf* leaves, uint32_t L,
                        const uint8_t* action_mask, oracle_expansion* out) {
  const uint32_t A = M->A, SW = M->SW, OW = M->OW;
  uint64_t steps = 0;
  uint32_t nchildren = 0;
  uint64_t scen_pos = 0;
  /* validate all leaves first (errors leave nothing behind) */
  for (uint32_t l = 0; l < L; ++l) {
    const oracle_leaf* lf = &leaves[l];
    node_t* P = get_node(M, lf->parent);
    if (!P) return fail(-1, "leaf: unknown parent node");
    if (lf->action >= (int32_t)A || lf->action < -1) return fail(-2, "leaf: action out of range");
    if (lf->depth >= M->D) return fail(-1, "leaf: depth must be < D");
    if (lf->action >= 0) {
      if (!P->expanded) return fail(-1, "leaf: parent not expanded");
      if (lf->child >= P->nchild[lf->action]) return fail(-1, "leaf: unknown child ordinal");
      if (lf->depth != P->depth + 1) return fail(-1, "leaf: depth != parent depth + 1");
    } else if (lf->depth != P->depth) {
      return fail(-1, "leaf: depth != node depth");
    }
  }
  out->child_begin[0] = 0;
  for (uint32_t l = 0; l < L; ++l) {
    const oracle_leaf* lf = &leaves[l];
    node_t* P = get_node(M, lf->parent);
    const uint64_t seed = P->seed;
    node_t* S;
    int64_t handle;
    if (lf->action < 0) {
      S = P; /* the leaf is the node itself: no update step */
      handle = lf->parent;
    } else {
      /* a1 update: gather the parent's scenarios, replay the last
       * action at depth Delta, keep those whose observation is the child's key */
      const uint32_t* key = P->keys[lf->action] + (size_t)lf->child * OW;
      node_t* tmp = new_node(M, P->n, lf->depth);
      tmp->seed = seed;
      uint32_t kept = 0;
      for (uint32_t i = 0; i < P->n; ++i) {
        uint32_t s2[ORACLE_MAXW], z[ORACLE_MAXW];
        float r;
        int term;
        steps += (uint64_t)step_or_term(M, P->states + (size_t)i * SW, lf->action, P->ids[i],
                                        lf->depth, seed, s2, z, &r, &term);
        if (keys_equal(z, key, OW)) {
          tmp->ids[kept] = P->ids[i];
          tmp->w[kept] = P->w[i];
          memcpy(tmp->states + (size_t)kept * SW, s2, SW * 4);
          ++kept;
        }
      }
      tmp->n = kept;
      if (kept == 0) {
        node_free(tmp, A);
        return fail(-1, "leaf: empty scenario set");
      }
      S = tmp;
      handle = add_node(M, tmp);
    }
    out->node[l] = handle;
    out->n_scen[l] = S->n;
    double W = 0.0;
    for (uint32_t i = 0; i < S->n; ++i) W += (double)S->w[i];
    out->weight[l] = W;
    /* (re)build the key table of the expanded node */
    if (!S->nchild) {
      S->nchild = (uint32_t*)calloc(A, 4);
      S->keys = (uint32_t**)calloc(A, sizeof(uint32_t*));
    }
    S->expanded = 1;
    for (uint32_t a = 0; a < A; ++a) {
      size_t la = (size_t)l * A + a;
      out->act_reward[la] = out->act_upper[la] = out->act_lower[la] = 0.0;
      if (action_mask && !action_mask[a]) {
        out->child_begin[la + 1] = nchildren;
        continue;
      }
      /* a2-a4 per scenario (ascending id), a5 first-occurrence groups */
      double R = 0.0, Uq = 0.0, Lq = 0.0;
      uint32_t ngroups = 0;
      uint32_t* gkey = (uint32_t*)malloc((size_t)S->n * OW * 4);
      uint32_t cbase = nchildren;
      for (uint32_t i = 0; i < S->n; ++i) {
        uint32_t s2[ORACLE_MAXW], z[ORACLE_MAXW];
        float r;
        int term;
        steps += (uint64_t)step_or_term(M, S->states + (size_t)i * SW, (int)a, S->ids[i],
                                        lf->depth + 1, seed, s2, z, &r, &term); /* Eq. 9 */
        double u = term ? 0.0 : upper_of(M, s2);                               /* Eq. 11 */
        double lam = 0.0;
        uint32_t len = 0;
        uint64_t h = 0xcbf29ce484222325ull;
        if (!term) rollout(M, s2, z, S->ids[i], lf->depth + 1, seed, &lam, &len, &h, &steps); /* Eq. 12 */
        uint32_t g;
        for (g = 0; g < ngroups; ++g)
          if (keys_equal(gkey + (size_t)g * OW, z, OW)) break;
        if (g == ngroups) {
          memcpy(gkey + (size_t)g * OW, z, OW * 4);
          ++ngroups;
          uint32_t c = cbase + g;
          if (c >= out->child_capacity) {
            free(gkey);
            return fail(-4, "child capacity exceeded");
          }
          out->child_count[c] = 0;
          out->child_first[c] = S->ids[i];
          out->child_weight[c] = out->child_upper[c] = out->child_lower[c] = 0.0;
          memcpy(out->child_obs + (size_t)c * OW, z, OW * 4);
        }
        uint32_t c = cbase + g;
        double w = (double)S->w[i];
        out->child_count[c] += 1;
        if (S->ids[i] < out->child_first[c]) out->child_first[c] = S->ids[i];
        out->child_weight[c] += w;
        out->child_upper[c] += w * u;
        out->child_lower[c] += w * lam;
        R += w * (double)r;
        Uq += w * ((double)r + M->gamma * u);
        Lq += w * ((double)r + M->gamma * lam);
        if (out->scen_obs && scen_pos < out->scen_capacity) {
          uint64_t q = scen_pos;
          memcpy(out->scen_obs + q * OW, z, OW * 4);
          out->scen_reward[q] = r;
          out->scen_upper[q] = u;
          out->scen_lower[q] = lam;
          out->scen_len[q] = len;
          out->scen_hash[q] = h;
          out->scen_child[q] = g;
          if (out->scen_states) memcpy(out->scen_states + q * SW, s2, SW * 4);
        }
        ++scen_pos;
      }
      /* a6: Eq. 11 / Eq. 12 means per child and the one-level Eq. 4 */
      for (uint32_t g = 0; g < ngroups; ++g) {
        uint32_t c = cbase + g;
        out->child_upper[c] /= out->child_weight[c];
        out->child_lower[c] /= out->child_weight[c];
      }
      out->act_reward[la] = R / W;
      out->act_upper[la] = Uq / W;
      out->act_lower[la] = Lq / W;
      nchildren += ngroups;
      out->child_begin[la + 1] = nchildren;
      /* key table for later update steps of this node's children */
      free(S->keys[a]);
      S->keys[a] = gkey;
      S->nchild[a] = ngroups;
    }
  }
  if (out->scen_obs && scen_pos > out->scen_capacity) return fail(-4, "scenario capacity exceeded");
  out->scenario_steps = steps;
  return 0;
}

int oracle_rollout_bounds(const oracle_model* M, int64_t h, double* upper_mean, double* lower_mean,
                          double* per_u, double* per_l) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  uint64_t seed = nd->seed;
  double W = 0.0, U = 0.0, Lm = 0.0;
  for (uint32_t i = 0; i < nd->n; ++i) {
    const uint32_t* s = nd->states + (size_t)i * M->SW;
    uint32_t z[ORACLE_MAXW];
    initial_obs(M, s, z);
    double u = is_terminal(M, s) ? 0.0 : upper_of(M, s);
    double lam = 0.0;
    uint32_t len;
    uint64_t hh, st = 0;
    if (!is_terminal(M, s)) rollout(M, s, z, nd->ids[i], nd->depth, seed, &lam, &len, &hh, &st);
    double w = (double)nd->w[i];
    W += w;
    U += w * u;
    Lm += w * lam;
    if (per_u) per_u[i] = u;
    if (per_l) per_l[i] = lam;
  }
  *upper_mean = U / W;
  *lower_mean = Lm / W;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* BRUTE_FORCE V*_D: the optimal value of the D-truncated     */
/* DESPOT on the same scenarios and tail, by the Eq. 4 recursion over the    */
/* whole tree with max over actions.                                         */
/* ------------------------------------------------------------------------ */
static double bf_value(const oracle_model* M, uint64_t seed, uint32_t n, const uint32_t* ids,
                       const float* w, const uint32_t* states, uint32_t depth, double* qout);

static double bf_q(const oracle_model* M, uint64_t seed, uint32_t n, const uint32_t* ids,
                   const float* w, const uint32_t* states, uint32_t depth, int a) {
  const uint32_t SW = M->SW, OW = M->OW;
  double W = 0.0, R = 0.0;
  uint32_t* s2 = (uint32_t*)malloc((size_t)n * SW * 4);
  uint32_t* zs = (uint32_t*)malloc((size_t)n * OW * 4);
  uint32_t* done = (uint32_t*)calloc(n, 4);
  for (uint32_t i = 0; i < n; ++i) {
    float r;
    int term;
    step_or_term(M, states + (size_t)i * SW, a, ids[i], depth + 1, seed, s2 + (size_t)i * SW,
                 zs + (size_t)i * OW, &r, &term);
    W += (double)w[i];
    R += (double)w[i] * (double)r;
  }
  double future = 0.0;
  uint32_t* cid = (uint32_t*)malloc(n * 4);
  float* cw = (float*)malloc(n * 4);
  uint32_t* cs = (uint32_t*)malloc((size_t)n * SW * 4);
  for (uint32_t i = 0; i < n; ++i) {
    if (done[i]) continue;
    uint32_t cn = 0;
    double Wc = 0.0;
    for (uint32_t j = i; j < n; ++j) {
      if (done[j] || !keys_equal(zs + (size_t)i * OW, zs + (size_t)j * OW, OW)) continue;
      done[j] = 1;
      cid[cn] = ids[j];
      cw[cn] = w[j];
      memcpy(cs + (size_t)cn * SW, s2 + (size_t)j * SW, SW * 4);
      Wc += (double)w[j];
      ++cn;
    }
    future += (Wc / W) * bf_value(M, seed, cn, cid, cw, cs, depth + 1, NULL);
  }
  free(s2); free(zs); free(done); free(cid); free(cw); free(cs);
  return R / W + M->gamma * future;
}

static double bf_value(const oracle_model* M, uint64_t seed, uint32_t n, const uint32_t* ids,
                       const float* w, const uint32_t* states, uint32_t depth, double* qout) {
  double W = 0.0, T = 0.0;
  int all_term = 1;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t* s = states + (size_t)i * M->SW;
    int term = is_terminal(M, s);
    W += (double)w[i];
    if (!term) {
      all_term = 0;
      T += (double)w[i] * M->tail;
    }
  }
  if (depth >= M->D) return T / W;
  if (all_term) return 0.0;
  double best = -INFINITY;
  for (uint32_t a = 0; a < M->A; ++a) {
    double q = bf_q(M, seed, n, ids, w, states, depth, (int)a);
    if (qout) qout[a] = q;
    if (q > best) best = q;
  }
  return best;
}

int oracle_brute_force(const oracle_model* M, int64_t h, double* value) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  *value = bf_value(M, nd->seed, nd->n, nd->ids, nd->w, nd->states, nd->depth, NULL);
  return 0;
}
int oracle_brute_force_q(const oracle_model* M, int64_t h, double* q) {
  node_t* nd = get_node(M, h);
  if (!nd) return fail(-1, "bad node");
  for (uint32_t a = 0; a < M->A; ++a) q[a] = 0.0;
  if (nd->depth >= M->D) return fail(-1, "node at depth D");
  for (uint32_t a = 0; a < M->A; ++a)
    q[a] = bf_q(M, nd->seed, nd->n, nd->ids, nd->w, nd->states, nd->depth, (int)a);
  return 0;
}
