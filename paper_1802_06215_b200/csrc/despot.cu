// despot.cu -- host side of libdespot: the C ABI of include/despot.h, model
// loading (parameter parsing and lookup tables built from the model cards of
// DESIGN.md §3), node arenas, and the launch sequence of a batch
// (K1 -> K2pre -> K2 -> [exchange] -> K3a -> K3b -> K3c).  Every step of the
// hot path runs in the kernels of kernels.cuh / finalize.cuh.
#include <cuda_runtime.h>

#include <atomic>
#include <type_traits>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/despot.h"
#include "common.cuh"
#include "finalize.cuh"
#include "kernels.cuh"
#include "models.cuh"
#include "model_car.cuh"
#include "kernels_sparse.cuh"
#include "exchange.cuh"
#include "nccl_dl.h"

using namespace hd;

// ===========================================================================
// errors
// ===========================================================================
static thread_local std::string g_err;
static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
extern "C" const char* despot_last_error(void) { return g_err.c_str(); }
extern "C" int despot__set_error(int code, const char* msg) {  // internal (search.cpp)
  g_err = msg ? msg : "";
  return code;
}
extern "C" int despot_abi_version(void) { return DESPOT_ABI_VERSION; }

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      if (e_ == cudaErrorMemoryAllocation) return set_err(DESPOT_ENOMEM, "%s: %s", #call,      \
                                                          cudaGetErrorString(e_));            \
      return set_err(DESPOT_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));                  \
    }                                                                                         \
  } while (0)

// ===========================================================================
// parameter parsing ("key=value key=value"), independent of oracle/
// ===========================================================================
namespace {
bool get_param(const std::string& params, const std::string& key, std::string& val) {
  size_t p = 0;
  while (p < params.size()) {
    while (p < params.size() && isspace((unsigned char)params[p])) ++p;
    size_t e = p;
    while (e < params.size() && !isspace((unsigned char)params[e])) ++e;
    if (e > p) {
      std::string tok = params.substr(p, e - p);
      size_t eq = tok.find('=');
      if (eq != std::string::npos && tok.substr(0, eq) == key) {
        val = tok.substr(eq + 1);
        return true;
      }
    }
    p = e;
  }
  return false;
}
double pd(const std::string& params, const char* key, double dflt) {
  std::string v;
  return get_param(params, key, v) ? strtod(v.c_str(), nullptr) : dflt;
}
long pi(const std::string& params, const char* key, long dflt) {
  std::string v;
  return get_param(params, key, v) ? strtol(v.c_str(), nullptr, 10) : dflt;
}
bool pxy(const std::string& params, const char* key, std::vector<int>& xs, std::vector<int>& ys) {
  std::string v;
  if (!get_param(params, key, v)) return false;
  xs.clear();
  ys.clear();
  const char* p = v.c_str();
  while (*p) {
    char* e;
    long x = strtol(p, &e, 10);
    if (*e != ':') return false;
    long y = strtol(e + 1, &e, 10);
    xs.push_back((int)x);
    ys.push_back((int)y);
    if (*e == ',') ++e;
    else if (*e) return false;
    p = e;
  }
  return true;
}
bool plist(const std::string& params, const char* key, std::vector<int>& xs) {
  std::string v;
  if (!get_param(params, key, v)) return false;
  xs.clear();
  const char* p = v.c_str();
  while (*p) {
    char* e;
    xs.push_back((int)strtol(p, &e, 10));
    if (*e == ',') ++e;
    else if (*e) return false;
    p = e;
  }
  return true;
}
// T(p) = floor(p 2^32), event iff (uint64)u < T (R14)
uint64_t thresh(double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 4294967296ull;
  return (uint64_t)std::floor(p * 4294967296.0);
}
}  // namespace

// ===========================================================================
// model, nodes, batches
// ===========================================================================
constexpr int kBatchEvents = 10;

struct despot_model;
static void dev_free(const despot_model* m, void* p, cudaStream_t st);
struct Block {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  const despot_model* model = nullptr;  // its allocator (despot_opts hooks or stream-ordered)
  ~Block() {
    if (ptr) dev_free(model, ptr, stream);
  }
};

// Host-side trace of one expansion call (env DESPOT_HOST_TRACE=1): the time
// since the call's start at named points, printed to stderr at its end.  A
// diagnostic for the per-call host overhead; off by default (one branch).
struct HostTrace {
  bool on = false;
  int n = 0;
  double t[40];
  const char* name[40];
  static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  void mark(const char* s) {
    if (on && n < 40) {
      t[n] = now_us();
      name[n++] = s;
    }
  }
  void start() {
    static const bool env = getenv("DESPOT_HOST_TRACE") != nullptr;
    on = env;
    n = 0;
    mark("start");
  }
  void dump() {
    if (!on) return;
    fprintf(stderr, "[despot host trace]");
    for (int i = 1; i < n; ++i) fprintf(stderr, " %s=%.1f", name[i], t[i] - t[0]);
    fprintf(stderr, " (us)\n");
  }
};
static thread_local HostTrace g_ht;
// set while despot_batch_prepare captures a batch's device work into a CUDA
// graph: allocations are made outside the stream (cudaMalloc), the new
// arenas are not allocated at all (each run allocates its own and patches
// the leaf table), and the new nodes are templates (not registered)
static thread_local bool g_capture = false;
constexpr uintptr_t kTemplateBase = uintptr_t(1) << 40;  // arena base of a prepared batch's template nodes

struct Node {
  despot_model* model;
  std::shared_ptr<Block> block;
  uint32_t* ids;
  float* w;
  uint32_t* states;
  uint32_t* nchild;
  uint32_t* keys;
  uint32_t cap, kcap;
  uint32_t n;  // local scenarios (host copy, valid once the creating call returned)
  uint32_t gn; // bound on the global scenario count (sizes the sharded sparse key table)
  uint32_t depth;
  uint64_t seed;
  double wroot;
  bool expanded;
};

// An NCCL communicator owned by the library (despot_comm_init).  Collectives
// of one communicator are enqueued under its mutex: the ranks must issue them
// in the same order (SPMD, one host thread per rank and model).
struct despot_comm {
  ncclComm_t c = nullptr;
  int rank = 0, world = 1, device = 0;
  std::mutex mu;
  std::atomic<bool> failed{false};
};

struct despot_model {
  DevModel host;
  DevModel* dev = nullptr;
  std::string kind;
  int device = 0, rank = 0, world = 1;
  uint32_t flags = 0;
  despot_comm* comm = nullptr;
  // device allocator hooks (despot_opts; e.g. torch's caching allocator), else
  // cudaMallocAsync / cudaFreeAsync on the call's stream
  void* (*alloc_fn)(size_t, void*, void*) = nullptr;
  void (*free_fn)(void*, void*, void*) = nullptr;
  void* alloc_ctx = nullptr;
  // packed-exchange capacity (K4, dense keys) in slots per (leaf, action) x 16:
  // raised to 5/4 of the largest union seen, so a capacity retry is rare
  std::atomic<uint32_t> xratio16{64};
  int num_sms = 148;
  std::atomic<bool> failed{false};
  std::mutex mu;
  std::unordered_set<Node*> nodes;
  int k2_occ = 0;
  void* snap = nullptr;  // device copy of the dense model's shared-memory image
};

static void* dev_alloc(const despot_model* m, size_t bytes, cudaStream_t st) {
  if (m && m->alloc_fn) return m->alloc_fn(bytes ? bytes : 1, st, m->alloc_ctx);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes ? bytes : 1, st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
static void dev_free(const despot_model* m, void* p, cudaStream_t st) {
  if (!p) return;
  if (m && m->free_fn) m->free_fn(p, st, m->alloc_ctx);
  else cudaFreeAsync(p, st);
}

struct despot_batch {
  despot_model* model;
  cudaStream_t stream;
  uint32_t L, A, S, flags;
  std::vector<despot_leaf> leaves;
  std::vector<Node*> leaf_node;  // node expanded for each leaf (new or existing)
  std::vector<bool> is_new;
  std::shared_ptr<Block> new_block;
  void* scratch = nullptr;
  BatchDev bd{};
  SparseItemOut io{};
  void* pinned = nullptr;  // leaf-table staging, owned until the batch syncs
  void* stage = nullptr;   // device output staging (host outputs)
  char* hs = nullptr;      // pinned status read-back
  char* hp_out = nullptr;  // pinned output staging
  bool bound = false;      // outputs bound (bind_outputs)
  bool persistent = false; // a prepared batch's (graph-captured) batch: scratch, staging, events kept
  bool k3_fused = false;   // the finalize runs in K2's last CTA
  // resident prepared batch (all leaves are nodes themselves, fused finalize):
  // the graph holds K2 alone; the scratch's zero state and the leaf table are
  // set up once (resident_init) and restored by K2's last CTA, the status
  // arrives in mapped host memory (hmapped); dirty: re-initialise before the
  // next run (after an error)
  bool resident = false, resident_table = false, dirty = false;
  // host outputs all page-locked: the kernels write them in place through
  // their device mapping (no staging, no D2H copies; the bytes still cross
  // the bus inside the call and are counted in d2h)
  bool zc_out = false;
  uint32_t* hmapped = nullptr;
  size_t r_stat = 0, r_zero = 0, r_h2d = 0;  // status offset, bytes zeroed from it, leaf-table bytes
  size_t o_ns = 0, o_w = 0, o_ar = 0, o_au = 0, o_al = 0, o_cb = 0, o_cc = 0, o_cf = 0, o_cw = 0, o_cu = 0,
         o_cl = 0, o_co = 0, o_so = 0;  // staging layout
  bool sparse = false;
  uint64_t n_sums = 0, n_mins = 0;
  // scenario-sharded sparse keys: local grouping, one exchange round (SUM of
  // the per-action partials, all-gather of the ranks' record blocks), merge
  bool sharded_sparse = false;
  bool xlib = false;              // the exchange runs on the model's communicator (in the call)
  uint32_t xround = 0;            // exchange rounds handed out (caller-driven form)
  void* gbuf = nullptr;           // all-gather buffer: world blocks of gblk bytes
  void* mscratch = nullptr;       // merge scratch (offsets, merged sums)
  uint64_t gblk = 0, gn_max = 0;  // block bytes; the largest global scenario count of a leaf
  uint32_t hdr_pad = 0, rec_bytes = 0;
  XDev x{};                       // packed exchange (dense keys, xlib)
  size_t new_bytes = 0;           // bytes of the new arenas of one run
  size_t o_leaves = 0;            // the leaf table's offset in the scratch and the pinned staging
  std::vector<LeafDev> ld;        // the leaf table (a prepared batch patches the new arenas' pointers)
  uint32_t x_rounds = 0;          // collective rounds issued by the library
  uint64_t x_bytes = 0;           // bytes this rank contributed to them
  bool timing = false, timing_k2 = false;  // DESPOT_X_TIMING / DESPOT_X_TIMING_K2 (K2 events only)
  uint32_t launches = 0;  // kernels launched for this batch
  uint64_t h2d = 0, d2h = 0;  // host <-> device bytes copied for this batch
  cudaEvent_t ev[kBatchEvents] = {};  // DESPOT_X_TIMING: 0 call start, 1/2 K1, 3/4 K2, 5/6 K3, 7 end, 8/9 K4
  void mark(int i) {
    // (in a prepared batch's graph capture: external event-record nodes, so
    // every launch of the graph records them)
    if (timing && (!timing_k2 || i == 3 || i == 4))
      cudaEventRecordWithFlags(ev[i], stream, persistent ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
};

namespace {

Node* lookup(despot_model* m, despot_node h) {
  Node* n = reinterpret_cast<Node*>(h);
  std::lock_guard<std::mutex> g(m->mu);
  return m->nodes.count(n) ? n : nullptr;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// bytes of a node arena with capacity cap
size_t node_bytes(const DevModel& dm, uint32_t cap, uint32_t kcap) {
  size_t b = 0;
  b += align256((size_t)cap * 4);                        // ids
  b += align256((size_t)cap * 4);                        // w
  b += align256((size_t)cap * 4 * dm.SW);                // states
  b += align256((size_t)dm.A * 4);                       // nchild
  b += align256((size_t)dm.A * kcap * dm.OW * 4);        // keys
  return b;
}
void carve_node(Node* nd, const DevModel& dm, char*& p) {
  nd->ids = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)nd->cap * 4);
  nd->w = reinterpret_cast<float*>(p);
  p += align256((size_t)nd->cap * 4);
  nd->states = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)nd->cap * 4 * dm.SW);
  nd->nchild = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)dm.A * 4);
  nd->keys = reinterpret_cast<uint32_t*>(p);
  p += align256((size_t)dm.A * nd->kcap * dm.OW * 4);
}
uint32_t key_cap(const DevModel& dm, uint32_t cap) {
  return dm.slots ? dm.slots : (cap ? cap : 1);
}
// key-table capacity of a new child of p: a sharded sparse node keeps the
// keys of the GLOBAL children, bounded by the global scenario count
uint32_t child_kcap(const despot_model* m, const Node* p) {
  return (m->world > 1 && !m->host.slots) ? std::max<uint32_t>(p->gn, 1) : key_cap(m->host, p->cap);
}

// fixed-point scale of the exact reductions: |sum of normalised values| <=
// Vmax <= 2^(61 - shift)
void set_fixed_point(DevModel& dm, double rmax, double umax) {
  const double vmax = (rmax + std::fabs(dm.tail)) * (dm.D + 1) + umax + rmax;
  int shift = 61 - (int)std::ceil(std::log2(vmax));
  if (shift > 52) shift = 52;
  if (shift < 16) shift = 16;
  dm.fx = std::ldexp(1.0, shift);
  dm.inv_fx = std::ldexp(1.0, -shift);
}

int build_model(const char* kind, const std::string& params, DevModel& dm) {
  memset(&dm, 0, sizeof dm);
  dm.gamma = pd(params, "gamma", 0.95);
  dm.elements = 1;
  std::string k(kind);
  double rmax = 0, umax = 0;
  if (k == "tiger") {
    dm.kind = kTiger;
    dm.A = 3; dm.SW = 1; dm.OW = 1; dm.slots = 4; dm.terminal_slot = 3;
    dm.D = (uint32_t)pi(params, "D", 10);
    dm.t_listen = thresh(pd(params, "p_listen", 0.85));
    dm.tail = 0.0;
    rmax = 100; umax = 10;
  } else if (k == "rocksample") {
    dm.kind = kRockSample;
    dm.n = (int)pi(params, "n", 7);
    dm.R = (int)pi(params, "robots", 1);
    const double d0 = pd(params, "d0", 4.0);
    std::vector<int> rx, ry, sx, sy;
    if (!pxy(params, "rocks", rx, ry) || !pxy(params, "starts", sx, sy))
      return set_err(DESPOT_EINVAL, "rocksample: need rocks=x:y,... and starts=x:y,...");
    std::string pol;
    dm.policy_east = get_param(params, "policy", pol) && pol == "east";
    dm.m = (int)rx.size();
    if (dm.R < 1 || dm.R > 2 || (int)sx.size() != dm.R || dm.m > kRsMaxRocks || dm.n < 1 ||
        dm.n > kRsMaxN || dm.n * dm.n * std::max(dm.m, 1) > RockSample<1>::kMaxTable)
      return set_err(DESPOT_EINVAL, "rocksample: need 1<=robots<=2, rocks<=31, n<=32, n*n*rocks<=16384");
    dm.base = 5 + dm.m;
    dm.A = 1;
    for (int r = 0; r < dm.R; ++r) dm.A *= (uint32_t)dm.base;
    dm.SW = 2; dm.OW = 1; dm.slots = (dm.R == 1 ? 3 : 9) + 1; dm.terminal_slot = dm.slots - 1;
    dm.D = (uint32_t)pi(params, "D", 20);
    dm.tail = 0.0;
    dm.elements = (uint32_t)dm.R;
    memset(dm.rock_at, -1, sizeof dm.rock_at);
    for (int j = 0; j < dm.m; ++j) {
      if (rx[j] < 0 || ry[j] < 0 || rx[j] >= dm.n || ry[j] >= dm.n)
        return set_err(DESPOT_EINVAL, "rocksample: rock off the grid");
      if (dm.rock_at[ry[j] * dm.n + rx[j]] >= 0) return set_err(DESPOT_EINVAL, "rocksample: two rocks share a cell");
      dm.rx[j] = (int8_t)rx[j];
      dm.ry[j] = (int8_t)ry[j];
      dm.rock_at[ry[j] * dm.n + rx[j]] = (int8_t)j;
    }
    // sensing accuracy 0.5 (1 + 2^(-d/d0)) (R17): thresholds by d^2
    dm.d2max = (uint32_t)(2 * (dm.n - 1) * (dm.n - 1));
    for (uint32_t d2 = 0; d2 <= dm.d2max; ++d2) {
      const double acc = 0.5 * (1.0 + std::pow(2.0, -std::sqrt((double)d2) / d0));
      const uint64_t T = thresh(acc);
      dm.sense_thr_m1[d2] = (uint32_t)(T - 1);  // T >= 2^31: event iff u <= T - 1
    }
    // default-policy positions: robot r handles rocks j % R == r, sorted (x, y, j)
    int pos = 0;
    for (int r = 0; r < dm.R; ++r) {
      std::vector<int> h;
      for (int j = 0; j < dm.m; ++j)
        if (j % dm.R == r) h.push_back(j);
      for (size_t a = 1; a < h.size(); ++a)
        for (size_t b = a; b > 0; --b) {
          const int p = h[b - 1], q = h[b];
          const bool less = rx[q] < rx[p] || (rx[q] == rx[p] && (ry[q] < ry[p] || (ry[q] == ry[p] && q < p)));
          if (!less) break;
          std::swap(h[b - 1], h[b]);
        }
      uint32_t mask = 0;
      for (int j : h) {
        dm.pos_rock[pos] = (uint8_t)j;
        mask |= 1u << pos;
        ++pos;
      }
      dm.range_mask[r] = dm.policy_east ? 0u : mask;  // always-east test policy: nothing to handle
    }
    rmax = 10.0 * dm.R;
    umax = 10.0 * (dm.m + dm.R);
    dm.sm_table_bytes = (uint32_t)RockSample<1>::table_bytes(dm.n, dm.m, dm.D);
  } else if (k == "nav") {
    dm.kind = kNav;
    dm.n = (int)pi(params, "n", 13);
    dm.wall_y = (int)pi(params, "wall_y", dm.n / 2);
    std::vector<int> gates, gx, gy, lx, ly;
    if (!plist(params, "gates", gates) || gates.size() != 2) gates = {3, 9};
    dm.gate_x[0] = gates[0];
    dm.gate_x[1] = gates[1];
    if (pxy(params, "goal", gx, gy) && gx.size() == 1) {
      dm.goal_x = gx[0];
      dm.goal_y = gy[0];
    } else {
      dm.goal_x = dm.n / 2;
      dm.goal_y = dm.n - 1;
    }
    pxy(params, "landmarks", lx, ly);
    dm.t_fail = thresh(pd(params, "p_fail", 0.03));
    dm.t_flip = thresh(pd(params, "p_flip", 0.03));
    // the device compares 32-bit words with 32-bit thresholds (R14: T < 2^32)
    if (dm.t_fail >= (1ull << 32) || dm.t_flip >= (1ull << 32))
      return set_err(DESPOT_EINVAL, "nav: p_fail and p_flip must be < 1");
    if (dm.n < 3 || dm.n > kNavMaxN || dm.wall_y <= 0 || dm.wall_y >= dm.n - 1)
      return set_err(DESPOT_EINVAL, "nav: need 3 <= n <= 16 and 0 < wall_y < n-1");
    // cell classes: rows 0 and n-1 known free, wall row obstacles except the
    // two gates, landmarks obstacles, everything else unknown (row-major idx)
    std::vector<int> cls(dm.n * dm.n), idx(dm.n * dm.n, -1);
    int nu = 0;
    for (int y = 0; y < dm.n; ++y)
      for (int x = 0; x < dm.n; ++x) {
        int c = 4;  // unknown
        if (y == 0 || y == dm.n - 1) c = 0;
        else if (y == dm.wall_y) c = x == dm.gate_x[0] ? 2 : x == dm.gate_x[1] ? 3 : 1;
        else
          for (size_t l = 0; l < lx.size(); ++l)
            if (lx[l] == x && ly[l] == y) c = 1;
        cls[y * dm.n + x] = c;
        if (c == 4) idx[y * dm.n + x] = nu++;
      }
    dm.nav_words = (nu + 31) / 32;
    if (dm.nav_words > kNavMaxWords || dm.nav_words < 1) return set_err(DESPOT_EINVAL, "nav: unknown cells");
    // padded occupancy rows: row y+1, bit x+1 = cell (x, y); the border is
    // occupied (off-grid counts as occupied), gates are left open here (the
    // closed one is added per scenario on the device)
    dm.nav_unknown = nu;
    for (int r = 0; r < dm.n + 2; ++r) {
      uint32_t row = 0;
      for (int c = 0; c < dm.n + 2; ++c) {
        const int x = c - 1, y = r - 1;
        bool occ = x < 0 || y < 0 || x >= dm.n || y >= dm.n;
        if (!occ) occ = cls[y * dm.n + x] == 1;
        row |= (uint32_t)occ << c;
      }
      dm.nav_known_rows[r] = row;
    }
    for (int y = 0; y < dm.n; ++y)
      for (int x = 0; x < dm.n; ++x)
        if (idx[y * dm.n + x] >= 0) dm.nav_unk_pos[idx[y * dm.n + x]] = (uint16_t)((x + 1) | ((y + 1) << 8));
    dm.A = 9; dm.SW = 1 + (uint32_t)dm.nav_words; dm.OW = 1; dm.slots = 257; dm.terminal_slot = 256;
    dm.D = (uint32_t)pi(params, "D", 90);
    dm.tail = (double)(-0.2f) / (1.0 - dm.gamma);  // stay forever (R6)
    rmax = 20; umax = 20;
  } else if (k == "car") {
    dm.kind = kCar;
    dm.peds = (int)pi(params, "peds", 20);
    if (dm.peds < 1 || dm.peds > kCarMaxPeds) return set_err(DESPOT_EINVAL, "car: 1 <= peds <= 31");
    dm.t_car_fail = thresh(pd(params, "p_fail", 0.01));
    dm.noise_scale = (float)pd(params, "noise", 0.001375);  // heading sd pi/8 (card §3.4)
    dm.A = 3; dm.SW = 4 + 2 * (uint32_t)dm.peds; dm.OW = 1 + (uint32_t)dm.peds; dm.slots = 0;
    dm.terminal_slot = 0;
    dm.D = (uint32_t)pi(params, "D", 90);
    dm.elements = 1 + (uint32_t)dm.peds;
    dm.tail = (double)(-0.1f) / (1.0 - dm.gamma);
    // heading-noise rotations for every byte sum (card §3.4), the card's fp32
    // sequence evaluated here once per value (host fp contraction is off)
    for (int v = 0; v <= 1020; ++v) {
      volatile float tau = (float)(v - 510) * dm.noise_scale;
      volatile float tt = tau * tau;
      volatile float den = 1.0f + tt;
      volatile float c = (1.0f - tt) / den;
      volatile float sn = (tau + tau) / den;
      dm.car_rot[v] = make_float2(c, sn);
    }
    rmax = 1000.0 * 4.5 + 100.2;
    umax = 100;
  } else {
    return set_err(DESPOT_EINVAL, "unknown model kind '%s'", kind);
  }
  if (!(dm.gamma > 0.0 && dm.gamma < 1.0) || dm.D < 1 || dm.D >= (uint32_t)kGpowN - 2)
    return set_err(DESPOT_EINVAL, "need 0 < gamma < 1 and 1 <= D <= 250");
  for (int i = 0; i < kGpowN; ++i) dm.gpow[i] = std::pow(dm.gamma, (double)i);
  set_fixed_point(dm, rmax, umax);
  return DESPOT_OK;
}

// ---------------------------------------------------------------------------
// kernel dispatch over model templates
// ---------------------------------------------------------------------------
template <class F>
int dispatch_dense(const DevModel& dm, F&& f) {
  switch (dm.kind) {
    case kTiger: return f(Tiger{});
    case kRockSample: return dm.R == 1 ? f(RockSample<1>{}) : f(RockSample<2>{});
    case kNav:
      switch (dm.nav_words) {
        case 1: return f(Nav<1>{});
        case 2: return f(Nav<2>{});
        case 3: return f(Nav<3>{});
        case 4: return f(Nav<4>{});
        case 5: return f(Nav<5>{});
        case 6: return f(Nav<6>{});
        default: return f(Nav<7>{});
      }
    default: return set_err(DESPOT_EINVAL, "not a dense-observation model");
  }
}

template <class F>
int dispatch_car(const DevModel& dm, F&& f) {
  // exact instantiations for the studied counts (6 / 12 / 20; 2 for tests)
  switch (dm.peds) {
    case 2: return f(CarThreadT<2, true>{});
    case 6: return f(CarThreadT<6, true>{});
    case 12: return f(CarThreadT<12, true>{});
    case 20: return f(CarThreadT<20, true>{});
    default: break;
  }
  if (dm.peds <= 8) return f(CarThreadT<8>{});
  if (dm.peds <= 20) return f(CarThreadT<20>{});
  return f(CarThreadT<31>{});
}

// Occupancy (CTAs per SM) of a kernel at a dynamic smem size, and the smem
// attribute, cached per (kernel, smem): host calls are not free, and the
// persistent grids must be sized with the launch's real shared memory.
int kernel_occupancy(const void* kern, size_t smem, int block) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  static std::map<const void*, size_t> smem_set;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(kern, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  size_t& cur = smem_set[kern];
  if (smem > std::max<size_t>(cur, 48 << 10)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cur = smem;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
  if (occ < 1) occ = 1;
  cache[key] = occ;
  return occ;
}

// The batch's K2 and K3 kernels can be launched with programmatic stream
// serialization (common.cuh, pdl_wait / pdl_trigger): DESPOT_PDL = bit mask,
// 1 = K2 after K1, 2 = the K3 kernels (default 0: measured no faster).
static int pdl_mask() {
  static const int mk = getenv("DESPOT_PDL") ? atoi(getenv("DESPOT_PDL")) : 0;
  return mk;
}
template <typename... KArgs, typename... Args>
static void launch_pdl(int role, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_mask() & role) ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // errors: check_launch
}

int check_launch(despot_model* m, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    m->failed = true;
    return set_err(DESPOT_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
  }
  return DESPOT_OK;
}

// Pinned host staging buffers.  A batch owns its buffer from the async H2D
// of its leaf table until it has synchronised (end / abort), so concurrent or
// interleaved batches (e.g. the sharded begin/exchange/end form) never share
// one.
class PinnedPool {
 public:
  // power-of-two size classes: a request only reuses a buffer of its own
  // class, so small staging never holds on to the large output buffer
  void* acquire(size_t bytes) {
    size_t sz = 4096;
    while (sz < bytes) sz <<= 1;
    {
      std::lock_guard<std::mutex> g(mu_);
      auto& fl = free_[sz];
      if (!fl.empty()) {
        void* p = fl.back();
        fl.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, sz) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(mu_);
    sizes_[p] = sz;
    return p;
  }
  void release(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu_);
    free_[sizes_[p]].push_back(p);
  }

 private:
  std::mutex mu_;
  std::map<size_t, std::vector<void*>> free_;
  std::unordered_map<void*, size_t> sizes_;
};
// timing events, reused across batches (creating 8 events per call costs more
// than the phases of a small batch)
class EventPool {
 public:
  bool acquire(cudaEvent_t* ev) {
    std::lock_guard<std::mutex> g(mu_);
    for (int i = 0; i < kBatchEvents; ++i) {
      if (!free_.empty()) {
        ev[i] = free_.back();
        free_.pop_back();
      } else if (cudaEventCreate(&ev[i]) != cudaSuccess) {
        return false;
      }
    }
    return true;
  }
  void release(cudaEvent_t* ev) {
    std::lock_guard<std::mutex> g(mu_);
    for (int i = 0; i < kBatchEvents; ++i)
      if (ev[i]) free_.push_back(ev[i]);
  }

 private:
  std::mutex mu_;
  std::vector<cudaEvent_t> free_;
};
EventPool& event_pool() {
  static EventPool* p = new EventPool();
  return *p;
}
PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool();  // never destroyed (process lifetime)
  return *p;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" int despot_model_load(const char* kind, const char* params, const despot_opts* opts,
                                 despot_model** out) {
  if (!kind || !out) return set_err(DESPOT_EINVAL, "null argument");
  std::unique_ptr<despot_model> m(new despot_model());
  int rc = build_model(kind, params ? params : "", m->host);
  if (rc) return rc;
  m->kind = kind;
  if (opts) {
    m->device = opts->device;
    m->rank = opts->rank;
    m->world = opts->world < 1 ? 1 : opts->world;
    m->flags = opts->flags;
    m->comm = opts->comm;
    if ((opts->dev_alloc == nullptr) != (opts->dev_free == nullptr))
      return set_err(DESPOT_EINVAL, "dev_alloc and dev_free come together");
    m->alloc_fn = opts->dev_alloc;
    m->free_fn = opts->dev_free;
    m->alloc_ctx = opts->alloc_ctx;
  }
  if (m->rank < 0 || m->rank >= m->world) return set_err(DESPOT_EINVAL, "rank outside [0, world)");
  // initial capacity of the packed exchange, slots per (leaf, action) x 16 (a
  // library parameter beside the model card's; tests set it low to force the
  // capacity retry)
  m->xratio16 = (uint32_t)std::max<long>(1, pi(params ? params : "", "xratio16", 64));
  if (m->comm && (m->comm->world != m->world || m->comm->rank != m->rank || m->comm->device != m->device))
    return set_err(DESPOT_EINVAL, "communicator (rank %d of %d, device %d) does not match the opts", m->comm->rank,
                   m->comm->world, m->comm->device);
  if (m->world > (int)kMaxMergeWorld) return set_err(DESPOT_EINVAL, "world > %u", kMaxMergeWorld);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(DESPOT_ECUDA, "no CUDA device (libdespot has no CPU fallback)");
  CU(cudaSetDevice(m->device));
  CU(cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, m->device));
  // keep freed stream-ordered memory in the pool (per-batch scratch is reused)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, m->device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  CU(cudaMalloc(&m->dev, sizeof(DevModel)));
  CU(cudaMemcpy(m->dev, &m->host, sizeof(DevModel), cudaMemcpyHostToDevice));
  if (m->host.slots) {  // dense models: the shared-memory image, once (load_sm_image)
    rc = dispatch_dense(m->host, [&](auto mdl) -> int {
      using M = decltype(mdl);
      const size_t bytes = align16(sizeof(typename M::Sm)) + align16(m->host.sm_table_bytes);
      const uint32_t words = (uint32_t)(bytes / 16);
      uint4* snap = nullptr;
      if (cudaMalloc(&snap, bytes) != cudaSuccess) return set_err(DESPOT_ENOMEM, "model image");
      m->snap = snap;
      kernel_occupancy((const void*)k_snapshot_sm<M>, bytes, 256);  // sets the smem attribute if > 48 KB
      k_snapshot_sm<M><<<1, 256, bytes>>>(m->dev, snap, words);
      if (cudaDeviceSynchronize() != cudaSuccess) return set_err(DESPOT_ECUDA, "model image kernel");
      m->host.sm_snap = snap;
      m->host.sm_snap_words = words;
      if (cudaMemcpy(m->dev, &m->host, sizeof(DevModel), cudaMemcpyHostToDevice) != cudaSuccess)
        return set_err(DESPOT_ECUDA, "model copy");
      return DESPOT_OK;
    });
    if (rc) {
      if (m->snap) cudaFree(m->snap);
      cudaFree(m->dev);
      return rc;
    }
  }
  *out = m.release();
  return DESPOT_OK;
}

extern "C" int despot_model_info_get(const despot_model* m, despot_model_info* o) {
  if (!m || !o) return set_err(DESPOT_EINVAL, "null argument");
  o->num_actions = m->host.A;
  o->state_words = m->host.SW;
  o->obs_words = m->host.OW;
  o->obs_slots = m->host.slots;
  o->max_depth = m->host.D;
  o->elements = m->host.elements;
  o->gamma = m->host.gamma;
  o->tail = m->host.tail;
  return DESPOT_OK;
}

extern "C" int despot_model_free(despot_model* m) {
  if (!m) return DESPOT_OK;
  cudaSetDevice(m->device);
  {
    std::lock_guard<std::mutex> g(m->mu);
    for (Node* n : m->nodes) delete n;
    m->nodes.clear();
  }
  cudaDeviceSynchronize();
  if (m->dev) cudaFree(m->dev);
  if (m->snap) cudaFree(m->snap);
  delete m;
  return DESPOT_OK;
}

extern "C" int despot_belief_load(despot_model* m, const uint32_t* states_soa, const float* weights,
                                  uint32_t K, uint64_t seed, void* stream, despot_node* root_out) {
  if (!m || !states_soa || !weights || !root_out) return set_err(DESPOT_EINVAL, "null argument");
  if (m->failed) return set_err(DESPOT_ESHUTDOWN, "model failed earlier");
  if (K == 0) return set_err(DESPOT_EINVAL, "empty belief (S:121)");
  if (K >= 0x7FFFFFFFu) return set_err(DESPOT_EINVAL, "K must be < 2^31");
  const DevModel& dm = m->host;
  double wroot = 0.0;
  for (uint32_t i = 0; i < K; ++i) {
    if (!(weights[i] > 0.0f) || !std::isfinite(weights[i])) return set_err(DESPOT_EINVAL, "weights must be finite and > 0");
    wroot += (double)weights[i];
  }
  if (dm.kind == kCar) {  // positions finite with |v| <= 4096: the bins floor(2v) stay int16 (R21)
    for (uint32_t i = 0; i < K; ++i)
      for (uint32_t k = 0; k < 4 + 2 * (uint32_t)dm.peds; ++k) {
        if (k == 1 || k == 2 || k == 3) continue;
        float v;
        memcpy(&v, &states_soa[(size_t)k * K + i], 4);
        if (!(std::fabs(v) <= 4096.0f)) return set_err(DESPOT_EINVAL, "car: coordinates must be finite, |v| <= 4096");
      }
  }
  // this rank's shard: global ids with id % world == rank
  std::vector<uint32_t> ids;
  for (uint32_t i = (uint32_t)m->rank; i < K; i += (uint32_t)m->world) ids.push_back(i);
  const uint32_t n = (uint32_t)ids.size();
  const uint32_t cap = n ? n : 1;
  std::vector<uint32_t> hbuf((size_t)cap * (2 + dm.SW));
  for (uint32_t i = 0; i < n; ++i) {
    hbuf[i] = ids[i];
    float wv = weights[ids[i]];
    memcpy(&hbuf[cap + i], &wv, 4);
    for (uint32_t k = 0; k < dm.SW; ++k) hbuf[(size_t)(2 + k) * cap + i] = states_soa[(size_t)k * K + ids[i]];
  }
  CU(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  auto blk = std::make_shared<Block>();
  blk->stream = st;
  blk->model = m;
  const uint32_t kcap = (m->world > 1 && !dm.slots) ? std::max<uint32_t>(K, 1) : key_cap(dm, cap);
  if (!(blk->ptr = dev_alloc(m, node_bytes(dm, cap, kcap), st))) return set_err(DESPOT_ENOMEM, "belief arena");
  Node* nd = new Node();
  nd->model = m;
  nd->block = blk;
  nd->cap = cap;
  nd->kcap = kcap;
  nd->gn = K;
  char* p = static_cast<char*>(blk->ptr);
  carve_node(nd, dm, p);
  nd->n = n;
  nd->depth = 0;
  nd->seed = seed;
  nd->wroot = wroot;
  nd->expanded = false;
  int rc = DESPOT_OK;
  if (cudaMemcpyAsync(nd->ids, hbuf.data(), (size_t)cap * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(nd->w, &hbuf[cap], (size_t)cap * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(nd->states, &hbuf[2 * (size_t)cap], (size_t)cap * 4 * dm.SW, cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaMemsetAsync(nd->nchild, 0, (size_t)dm.A * 4, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    rc = set_err(DESPOT_ECUDA, "belief upload failed");
  if (rc) {
    delete nd;
    return rc;
  }
  {
    std::lock_guard<std::mutex> g(m->mu);
    m->nodes.insert(nd);
  }
  *root_out = reinterpret_cast<despot_node>(nd);
  return DESPOT_OK;
}

extern "C" int despot_node_info(despot_model* m, despot_node h, uint32_t* n, uint32_t* depth) {
  Node* nd = m ? lookup(m, h) : nullptr;
  if (!nd) return set_err(DESPOT_EINVAL, "unknown node");
  if (n) *n = nd->n;
  if (depth) *depth = nd->depth;
  return DESPOT_OK;
}

extern "C" int despot_expand_batch_bytes(despot_model* m, const despot_leaf* leaves, uint32_t L, uint32_t flags,
                                         uint32_t* child_capacity, uint64_t* scen_capacity, uint64_t* host_bytes) {
  if (!m || (!leaves && L)) return set_err(DESPOT_EINVAL, "null argument");
  const DevModel& dm = m->host;
  const uint64_t W = (uint64_t)std::max(m->world, 1);
  uint64_t C = 0, S = 0;
  for (uint32_t l = 0; l < L; ++l) {
    Node* p = lookup(m, leaves[l].parent);
    if (!p) return set_err(DESPOT_EINVAL, "leaf %u: unknown node", l);
    // a leaf's scenarios are a subset of its parent's; sharded, only the
    // local count is known: (n + 1) * world bounds the global one for
    // interleaved ids (a filtered node may need more: ECAPACITY says so)
    const uint64_t g = W == 1 ? p->n : ((uint64_t)p->n + 1) * W;
    C += (uint64_t)dm.A * (dm.slots ? std::min<uint64_t>(g, dm.slots) : g);
    S += (uint64_t)dm.A * p->n;
  }
  C = std::max<uint64_t>(C, 1);
  if (C > 0xFFFFFFFFull) return set_err(DESPOT_ECAPACITY, "child bound %llu exceeds 2^32 - 1", (unsigned long long)C);
  const uint64_t LA = (uint64_t)L * dm.A;
  uint64_t bytes = (uint64_t)L * (8 + 4 + 4) + LA * 3 * 4 + (LA + 1) * 4 + C * (4 * 5 + 4 * (uint64_t)dm.OW);
  if (flags & DESPOT_X_RECORD_SCENARIO) bytes += S * (4 * (uint64_t)dm.OW + 4 * 4 + 8 + 4 * (uint64_t)dm.SW);
  if (child_capacity) *child_capacity = (uint32_t)C;
  if (scen_capacity) *scen_capacity = S;
  if (host_bytes) *host_bytes = bytes;
  return DESPOT_OK;
}

extern "C" int despot_node_read(despot_model* m, despot_node h, uint32_t* ids, float* w,
                                uint32_t* states_soa, void* stream) {
  Node* nd = m ? lookup(m, h) : nullptr;
  if (!nd) return set_err(DESPOT_EINVAL, "unknown node");
  CU(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (ids) CU(cudaMemcpyAsync(ids, nd->ids, (size_t)nd->n * 4, cudaMemcpyDeviceToHost, st));
  if (w) CU(cudaMemcpyAsync(w, nd->w, (size_t)nd->n * 4, cudaMemcpyDeviceToHost, st));
  if (states_soa && nd->n)
    CU(cudaMemcpy2DAsync(states_soa, (size_t)nd->n * 4, nd->states, (size_t)nd->cap * 4, (size_t)nd->n * 4,
                         m->host.SW, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return DESPOT_OK;
}

extern "C" int despot_node_release(despot_model* m, despot_node h) {
  if (!m) return set_err(DESPOT_EINVAL, "null model");
  Node* nd = reinterpret_cast<Node*>(h);
  {
    std::lock_guard<std::mutex> g(m->mu);
    if (!m->nodes.erase(nd)) return set_err(DESPOT_EINVAL, "unknown node");
  }
  cudaSetDevice(m->device);
  delete nd;  // the arena block is freed (stream-ordered) with its last node
  return DESPOT_OK;
}

extern "C" int despot_node_release_many(despot_model* m, const despot_node* nodes, uint32_t n) {
  if (!m || (n && !nodes)) return set_err(DESPOT_EINVAL, "null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (int rc = despot_node_release(m, nodes[i])) return rc;
  return DESPOT_OK;
}

// ---------------------------------------------------------------------------
// batches
// ---------------------------------------------------------------------------
static void free_batch(despot_batch* b, bool drop_new_nodes) {
  if (!b) return;
  if (drop_new_nodes) {
    std::lock_guard<std::mutex> g(b->model->mu);
    for (size_t l = 0; l < b->leaf_node.size(); ++l)
      if (b->is_new[l] && b->leaf_node[l]) {
        b->model->nodes.erase(b->leaf_node[l]);
        delete b->leaf_node[l];
        b->leaf_node[l] = nullptr;
      }
  }
  if (b->persistent) {  // a prepared batch: only this run's state goes
    b->new_block.reset();
    for (size_t l = 0; l < b->leaf_node.size(); ++l) b->leaf_node[l] = nullptr;
    return;
  }
  dev_free(b->model, b->scratch, b->stream);
  dev_free(b->model, b->stage, b->stream);
  dev_free(b->model, b->gbuf, b->stream);
  dev_free(b->model, b->mscratch, b->stream);
  if (b->pinned) {
    cudaStreamSynchronize(b->stream);  // the H2D from it must have completed
    pinned_pool().release(b->pinned);
  }
  if (b->timing) event_pool().release(b->ev);
  delete b;
}

static int launch_group_sparse(despot_model* m, despot_batch* b) {
  uint32_t tbits = 1;
  while ((1u << tbits) < 2 * b->S) ++tbits;  // hash table >= 2 n slots
  const size_t smem = 12 * ((size_t)1 << tbits) + 4 * (size_t)b->S;
  kernel_occupancy((const void*)k3_group_sparse, smem, 512);  // sets the smem attribute if > 48 KB
  launch_pdl(2, k3_group_sparse, (unsigned)((uint64_t)b->L * b->A), 512, smem, b->stream, b->bd, b->io, tbits, nullptr);
  ++b->launches;
  return check_launch(m, "K3a(sparse)");
}

static int launch_k2_sparse(despot_model* m, despot_batch* b, bool record) {
  const DevModel& dm = m->host;
  cudaStream_t st = b->stream;
  uint64_t q_bound = 0;
  for (uint32_t l = 0; l < b->L; ++l) q_bound += (uint64_t)dm.A * b->leaf_node[l]->cap;
  b->mark(3);
  // factored (warp per item) when the items cannot fill the SMs one thread
  // each; otherwise thread per item (fewer issue slots per scenario-step)
  // (measured, profiles/r01/peds_sweep.jsonl: the warp kernel wins for >= 12
  // pedestrians at 12k items, the thread kernel everywhere at 96k items and
  // for 6 pedestrians, whose warps would leave 25 of 32 lanes idle)
  // automatic choice (no variant flag), by the items the batch has: thread
  // per scenario when they fill the GPU one thread each; the grouped kernel
  // in between (its packed lane groups beat both others at 8 roots x K = 64,
  // profiles/r01/peds_sweep.jsonl); a warp per scenario for the few-item
  // batches of a tree search (latency: all pedestrians of a step in parallel)
  const bool forced = m->flags & (DESPOT_MF_UNFACTORED | DESPOT_MF_FACTORED | DESPOT_MF_GROUPED | DESPOT_MF_PAIRED);
  // (with <= 8 pedestrians the thread kernel also wins the middle range:
  // 8 roots x K = 64, 6 pedestrians: 0.107 ms vs 0.139 grouped, 0.231 warp)
  const bool big = q_bound >= (uint64_t)m->num_sms * 256 || (dm.peds <= 8 && q_bound >= (uint64_t)m->num_sms * 4),
             tiny = q_bound < (uint64_t)m->num_sms * 4;
  const bool grouped = (m->flags & DESPOT_MF_GROUPED) || (!forced && !big && !tiny);
  const bool unfactored = !grouped && ((m->flags & DESPOT_MF_UNFACTORED) || (!forced && big));
  const bool paired = m->flags & DESPOT_MF_PAIRED;
  if (paired) {  // a lane pair per scenario: lane q owns ceil(blocks / 2) Philox blocks
    const uint32_t NB = ((uint32_t)dm.peds + 4) / 4, Bp = (NB + 1) / 2;
    const uint64_t G = (NB + Bp - 1) / Bp, gpw = 32 / G;
    const uint64_t warps = (q_bound + gpw - 1) / gpw;
    auto pick = [&](auto bc) {
      constexpr int BB = decltype(bc)::value;
      return record ? k2_car_group<true, BB> : k2_car_group<false, BB>;
    };
    auto kern = Bp <= 1 ? pick(std::integral_constant<int, 1>{}) : Bp == 2 ? pick(std::integral_constant<int, 2>{})
                : Bp == 3 ? pick(std::integral_constant<int, 3>{}) : pick(std::integral_constant<int, 4>{});
    const int occ = kernel_occupancy((const void*)kern, 0, 128);
    const uint64_t g = std::min<uint64_t>((warps + 3) / 4, (uint64_t)m->num_sms * occ);
    launch_pdl(1, kern, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
  } else if (grouped) {
    const uint64_t G = ((uint64_t)dm.peds + 4) / 4, gpw = 32 / G;
    const uint64_t warps = (q_bound + gpw - 1) / gpw;
    auto kern = record ? k2_car_group<true> : k2_car_group<false>;
    const int occ = kernel_occupancy((const void*)kern, 0, 128);
    const uint64_t g = std::min<uint64_t>((warps + 3) / 4, (uint64_t)m->num_sms * occ);
    launch_pdl(1, kern, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
  } else if (unfactored) {
    dispatch_car(dm, [&](auto mdl) -> int {
      using M = decltype(mdl);
      const uint64_t g = std::min<uint64_t>((q_bound + 127) / 128, (uint64_t)m->num_sms * 16);
      if (record) launch_pdl(1, k2_car_thread<M, true>, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
      else launch_pdl(1, k2_car_thread<M, false>, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
      return 0;
    });
  } else {
    const uint64_t g = std::min<uint64_t>((q_bound + 3) / 4, (uint64_t)m->num_sms * 16);
    if (record) launch_pdl(1, k2_car_warp<true>, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
    else launch_pdl(1, k2_car_warp<false>, (unsigned)std::max<uint64_t>(g, 1), 128, 0, st, b->bd, b->io);
  }
  b->mark(4);
  ++b->launches;
  return check_launch(m, "K2(car)");
}

static int bind_outputs(despot_batch* b, despot_expansion* out, cudaStream_t st);
static bool outputs_pinned(const despot_expansion* out, uint32_t C);
constexpr uint64_t kZeroCopyMaxBytes = 4ull << 20;

// K3 for many slots as the single fused kernel (dense keys, S > 32, the
// compacted slot arrays within its shared-memory limit)
constexpr uint32_t kTileOffSharedMaxL = 64;  // K2 keeps a shared copy of tile_off up to this many leaves
static bool wide_fused(uint32_t S, bool sparse) {
  return !sparse && S > kWideS && S <= kWideFusedMaxS && wide_fused_smem(S) <= kWideFusedMaxSmem;
}
// look-back words: the tile counter + one per tile (a tile of kScanTile
// (leaf, action) pairs, or one pair in the fused wide kernel) + 1
static uint64_t scan_words(uint64_t LA, uint32_t S, bool sparse) {
  return (wide_fused(S, sparse) ? LA : LA / kScanTile) + 2;
}
static int begin_impl(despot_model* m, const despot_leaf* leaves, uint32_t L, uint32_t flags, void* stream,
                      despot_expansion* bind, despot_batch** out) {
  if (!m || !leaves || !out) return set_err(DESPOT_EINVAL, "null argument");
  if (m->failed) return set_err(DESPOT_ESHUTDOWN, "model failed earlier");
  if (L == 0 || L > kMaxLeaves) return set_err(DESPOT_EINVAL, "need 1 <= L <= %u", kMaxLeaves);
  if ((flags & DESPOT_X_RECORD_SCENARIO) && m->world > 1)
    return set_err(DESPOT_EINVAL, "RECORD_SCENARIO needs world == 1");
  const DevModel& dm = m->host;
  CU(cudaSetDevice(m->device));
  std::unique_ptr<despot_batch> b(new despot_batch());
  b->model = m;
  b->stream = (cudaStream_t)stream;
  b->L = L;
  b->A = dm.A;
  b->S = dm.slots;
  b->sparse = dm.slots == 0;
  // the exchange runs inside the call on the model's communicator (single-call
  // form); DESPOT_MF_EXCHANGE runs it at world 1 too (the one-GPU test of the
  // sharded data path)
  b->xlib = bind && m->comm && (m->world > 1 || (m->flags & DESPOT_MF_EXCHANGE)) &&
            !(flags & DESPOT_X_RECORD_SCENARIO);  // (RECORD batches are world 1: nothing to exchange)
  b->sharded_sparse = b->sparse && (m->world > 1 || b->xlib);
  b->flags = flags;
  b->leaves.assign(leaves, leaves + L);
  b->persistent = g_capture;
  b->timing = flags & (DESPOT_X_TIMING | DESPOT_X_TIMING_K2);
  b->timing_k2 = (flags & DESPOT_X_TIMING_K2) && !(flags & DESPOT_X_TIMING);
  if (b->timing) {
    if (!event_pool().acquire(b->ev)) return set_err(DESPOT_ECUDA, "cudaEventCreate failed");
    b->mark(0);
  }
  b->leaf_node.assign(L, nullptr);
  b->is_new.assign(L, false);
  // validate, size the new arenas
  std::vector<Node*> parent(L);
  size_t new_bytes = 0;
  for (uint32_t l = 0; l < L; ++l) {
    const despot_leaf& lf = leaves[l];
    Node* p = lookup(m, lf.parent);
    if (!p) return set_err(DESPOT_EINVAL, "leaf %u: unknown parent node", l);
    if (lf.action < -1 || lf.action >= (int32_t)dm.A)
      return set_err(DESPOT_EMODEL, "leaf %u: action %d outside [-1, %u)", l, lf.action, dm.A);
    if (lf.depth >= dm.D) return set_err(DESPOT_EINVAL, "leaf %u: depth %u >= D = %u", l, lf.depth, dm.D);
    if (lf.action >= 0) {
      if (!p->expanded) return set_err(DESPOT_EINVAL, "leaf %u: parent not expanded", l);
      if (lf.depth != p->depth + 1) return set_err(DESPOT_EINVAL, "leaf %u: depth != parent depth + 1", l);
      new_bytes += node_bytes(dm, p->cap, child_kcap(m, p));
    } else if (lf.depth != p->depth) {
      return set_err(DESPOT_EINVAL, "leaf %u: depth != node depth", l);
    }
    parent[l] = p;
  }
  // DESPOT_X_INDEX_LISTS (the paper's update form): host lists of
  // parent positions replace the replay + filter (validated here and, per
  // scenario, against the replay in K1)
  const bool ilist = flags & DESPOT_X_INDEX_LISTS;
  uint64_t idx_total = 0;
  if (ilist) {
    if (!bind || !bind->index_begin || !bind->index || m->world > 1)
      return set_err(DESPOT_EINVAL, "index lists need the single-call form, index_begin / index and world == 1");
    if (bind->index_begin[0] != 0) return set_err(DESPOT_EINVAL, "index_begin[0] must be 0");
    for (uint32_t l = 0; l < L; ++l) {
      const uint32_t b0 = bind->index_begin[l], b1 = bind->index_begin[l + 1];
      if (b1 < b0) return set_err(DESPOT_EINVAL, "leaf %u: index_begin decreases", l);
      if (leaves[l].action < 0 && b1 != b0) return set_err(DESPOT_EINVAL, "leaf %u: an index list on a self leaf", l);
      if (leaves[l].action >= 0 && b1 == b0) return set_err(DESPOT_EINVAL, "leaf %u: empty index list", l);
      for (uint32_t k = b0; k < b1; ++k)
        if (bind->index[k] >= parent[l]->n || (k > b0 && bind->index[k] <= bind->index[k - 1]))
          return set_err(DESPOT_EINVAL, "leaf %u: index list not ascending within the parent's %u scenarios", l,
                         parent[l]->n);
    }
    idx_total = bind->index_begin[L];
  }
  uint64_t q_bound = 0;  // sparse: per-item scratch bound sum_l A cap_l
  if (b->sparse) {
    uint32_t smax = 1;
    for (uint32_t l = 0; l < L; ++l) {
      smax = std::max(smax, parent[l]->cap);
      q_bound += (uint64_t)dm.A * parent[l]->cap;
    }
    // the grouping table of k3_group_sparse: 12 B x 2^ceil(log2 2n) + 4n of shared memory
    if (smax > 4096) return set_err(DESPOT_EINVAL, "sparse-key models: at most 4096 scenarios per leaf");
    b->S = smax;
  }
  g_ht.mark("validated");
  cudaStream_t st = b->stream;
  b->new_bytes = new_bytes;
  if (new_bytes && !g_capture) {
    b->new_block = std::make_shared<Block>();
    b->new_block->stream = st;
    b->new_block->model = m;
    if (!(b->new_block->ptr = dev_alloc(m, new_bytes, st))) return set_err(DESPOT_ENOMEM, "new arenas");
  }
  g_ht.mark("arena_alloc");
  // (capture: template nodes carved from a fixed fake base; every run rebases them)
  char* np = b->new_block ? static_cast<char*>(b->new_block->ptr)
                          : (g_capture ? reinterpret_cast<char*>(kTemplateBase) : nullptr);
  std::vector<LeafDev> ld(L);
  for (uint32_t l = 0; l < L; ++l) {
    const despot_leaf& lf = leaves[l];
    Node* p = parent[l];
    Node* nd = p;
    if (lf.action >= 0) {
      nd = new Node();
      nd->model = m;
      nd->block = b->new_block;
      nd->cap = p->cap;
      nd->kcap = child_kcap(m, p);
      nd->gn = p->gn;
      carve_node(nd, dm, np);
      nd->n = 0;
      nd->depth = lf.depth;
      nd->seed = p->seed;
      nd->wroot = p->wroot;
      nd->expanded = false;
      b->is_new[l] = true;
    }
    b->leaf_node[l] = nd;
    LeafDev& d = ld[l];
    d.p_ids = p->ids;
    d.p_w = p->w;
    d.p_states = p->states;
    d.p_keys = p->keys;
    d.p_nchild = p->nchild;
    d.p_cap = p->cap;
    d.p_n = p->n;
    d.p_kcap = p->kcap;
    d.ids = nd->ids;
    d.w = nd->w;
    d.states = nd->states;
    d.cap = nd->cap;
    d.keys = nd->keys;
    d.nchild = nd->nchild;
    d.kcap = nd->kcap;
    d.action = lf.action;
    d.child = lf.child;
    d.depth = lf.depth;
    d.seed_lo = (uint32_t)p->seed;
    d.seed_hi = (uint32_t)(p->seed >> 32);
    d.wroot = p->wroot;
    d.inv_wroot = 1.0 / p->wroot;
  }
  if (!g_capture) {
    std::lock_guard<std::mutex> g(m->mu);
    for (uint32_t l = 0; l < L; ++l)
      if (b->is_new[l]) m->nodes.insert(b->leaf_node[l]);
  }
  b->ld = ld;
  g_ht.mark("leaf_table");
  // scratch: leaves | n_leaf | tile_off | scen_off | sums | mins | rank | nc | err
  const uint64_t LA = (uint64_t)L * dm.A, LAS = LA * b->S;
  const SumLayout lay{LAS, LA};
  b->n_sums = lay.total();
  b->n_mins = LAS;
  size_t off = 0;
  auto take = [&](size_t bytes) {  // 256-byte aligned regions (vector loads need >= 16)
    size_t o = align256(off);
    off = o + align256(bytes);
    return o;
  };
  // status block [err u32 | total children u32 | steps u64 | K1 ticket u32 |
  // pad | n_leaf[L] u32] sits right before the SUM block: one memset zeroes
  // both, one D2H reads it
  const size_t stat_bytes = 4 * kStatWords + 4 * (size_t)L;
  const size_t o_leaves = take(sizeof(LeafDev) * L), o_tile = take(4 * ((size_t)L + 1)),
               o_scen = take(8 * ((size_t)L + 1));
  const size_t o_stat = off;
  off += (stat_bytes + 7) & ~size_t(7);
  // K3b's look-back flags (tile counter + one word per 1024 (leaf, action)
  // pairs), zeroed by the same memset as the status block and the sums
  const size_t o_scan = off;
  off += 8 * scan_words(LA, b->S, b->sparse);
  const size_t o_sums = take(8 * b->n_sums), o_mins = take(4 * b->n_mins), o_rank = take(4 * LAS),
               o_nc = take(4 * LA), o_item = take(b->sparse ? 4 * LAS : 0),
               o_hash = take(8 * q_bound), o_keys = take(4 * q_bound * dm.OW), o_q3 = take(24 * q_bound),
               o_idx = take(4 * idx_total);
  // packed exchange (K4, dense keys): union flags, block counts, packed sums
  // and first ids at the model's capacity hint
  const bool xdense = b->xlib && !b->sparse;
  XDev& x = b->x;
  x.las = LAS;
  x.qn = 3 * LA + 1;
  x.nblk = (uint32_t)((LAS + kXBlk - 1) / kXBlk);
  x.ccap = std::min<uint64_t>(LAS, (LA * m->xratio16.load() + 15) / 16 + 256);
  const size_t o_xflags = take(xdense ? (size_t)x.nblk * kXBlk : 0), o_xcnt = take(xdense ? 4 * (size_t)x.nblk : 0),
               o_xcpk = take(xdense ? 8 * (4 * x.ccap + x.qn) : 0), o_xcmin = take(xdense ? 4 * x.ccap : 0);
  if (g_capture ? cudaMalloc(&b->scratch, off) != cudaSuccess : !(b->scratch = dev_alloc(m, off, st))) {
    free_batch(b.release(), true);
    return set_err(DESPOT_ENOMEM, "batch scratch (%zu bytes)", off);
  }
  g_ht.mark("scratch_alloc");
  char* s = static_cast<char*>(b->scratch);
  BatchDev& bd = b->bd;
  bd.model = m->dev;
  bd.leaves = reinterpret_cast<LeafDev*>(s + o_leaves);
  bd.L = L;
  bd.A = dm.A;
  bd.a_magic = dm.A > 1 ? ~0ull / dm.A + 1 : 0;
  bd.S = b->S;
  bd.status = reinterpret_cast<uint32_t*>(s + o_stat);
  bd.err = bd.status;
  bd.n_leaf = bd.status + kStatWords;
  bd.tile_off = reinterpret_cast<uint32_t*>(s + o_tile);
  bd.scen_off = reinterpret_cast<uint64_t*>(s + o_scen);
  bd.sums = reinterpret_cast<int64_t*>(s + o_sums);
  bd.mins = reinterpret_cast<int32_t*>(s + o_mins);
  bd.rank = reinterpret_cast<uint32_t*>(s + o_rank);
  bd.nc = reinterpret_cast<uint32_t*>(s + o_nc);
  bd.scan_flags = reinterpret_cast<unsigned long long*>(s + o_scan);
  if (b->sparse) {
    bd.sp_item = reinterpret_cast<uint32_t*>(s + o_item);
    b->io.hash = reinterpret_cast<uint64_t*>(s + o_hash);
    b->io.keys = reinterpret_cast<uint32_t*>(s + o_keys);
    b->io.q3 = reinterpret_cast<int64_t*>(s + o_q3);
    b->io.kstride = dm.OW;
  }
  if (xdense) {
    x.flags = reinterpret_cast<uint8_t*>(s + o_xflags);
    x.cnt = reinterpret_cast<uint32_t*>(s + o_xcnt);
    x.cpk = reinterpret_cast<int64_t*>(s + o_xcpk);
    x.cmin = reinterpret_cast<int32_t*>(s + o_xcmin);
  }
  if (b->sharded_sparse) {
    // the record blocks of the all-gather, sized on the host from the leaves
    // alone (identical on every rank): a leaf's local scenarios are at most
    // ceil(K / world) of its root's K (the root shard is the largest node)
    const uint32_t W = (uint32_t)m->world;
    uint64_t rcap = 0;
    for (uint32_t l = 0; l < L; ++l) {
      rcap += (uint64_t)dm.A * ((parent[l]->gn + W - 1) / W);
      b->gn_max = std::max<uint64_t>(b->gn_max, parent[l]->gn);
    }
    b->rec_bytes = sparse_record_bytes(dm.OW);
    b->hdr_pad = (uint32_t)(((4 * LA + b->rec_bytes - 1) / b->rec_bytes) * b->rec_bytes);
    b->gblk = b->hdr_pad + rcap * b->rec_bytes;
    const size_t gbytes = (size_t)W * b->gblk;
    if (!(b->gbuf = dev_alloc(m, gbytes, st)) || !(b->mscratch = dev_alloc(m, 4 * LA, st))) {
      free_batch(b.release(), true);
      return set_err(DESPOT_ENOMEM, "all-gather buffer (%zu bytes)", gbytes);
    }
  }
  // all leaves are nodes themselves (e.g. roots): their sizes are known on the
  // host, so the update kernel and the prefix are skipped and the host ships
  // n, tile and record prefixes with the leaf table in one copy
  bool all_self = true;
  for (uint32_t l = 0; l < L; ++l) all_self = all_self && leaves[l].action < 0;
  const size_t h2d_bytes = all_self ? o_stat + stat_bytes : sizeof(LeafDev) * L;
  // a prepared batch of self leaves that will fuse its finalize: resident
  // (the same rule as k3_fused below, with the outputs bound)
  {
    const uint64_t G = 32 / small_group_width(b->S);
    // the zero state is restored by K2's last CTA (finalize fused into K2) or
    // by the wide finalize's CTAs (many slots); the leaf table is uploaded
    // once only when every leaf is a node itself (no new arenas per run)
    const bool fusable = b->S <= 32 && (uint64_t)L * dm.A <= 4 * G * kSmallUnroll * 2;
    b->resident = g_capture && bind && !ilist && !b->sparse && !xdense && m->world == 1 &&
                  !(flags & DESPOT_X_RECORD_SCENARIO) && (fusable || wide_fused(b->S, false)) &&
                  (bind->flags & DESPOT_X_RESIDENT);
    b->resident_table = b->resident && all_self;
  }
  void* hp = pinned_pool().acquire(std::max<size_t>(h2d_bytes, ilist ? o_idx + 4 * idx_total : 0));
  b->pinned = hp;
  if (ilist)
    for (uint32_t l = 0; l < L; ++l) {
      ld[l].idx = leaves[l].action >= 0 ? reinterpret_cast<const uint32_t*>(s + o_idx) + bind->index_begin[l] : nullptr;
      ld[l].idx_n = bind->index_begin[l + 1] - bind->index_begin[l];
    }
  b->o_leaves = o_leaves;
  int rc = DESPOT_OK;
  if (!hp) rc = set_err(DESPOT_ENOMEM, "pinned staging");
  if (!rc) {
    char* h = static_cast<char*>(hp);
    memcpy(h + o_leaves, ld.data(), sizeof(LeafDev) * L);
    if (all_self) {
      uint32_t* tile = reinterpret_cast<uint32_t*>(h + o_tile);
      uint64_t* scen = reinterpret_cast<uint64_t*>(h + o_scen);
      uint32_t* stat = reinterpret_cast<uint32_t*>(h + o_stat);
      memset(stat, 0, stat_bytes);
      uint64_t tacc = 0, sacc = 0;
      for (uint32_t l = 0; l < L; ++l) {
        const uint32_t n = parent[l]->n;
        stat[kStatWords + l] = n;
        tile[l] = (uint32_t)tacc;
        scen[l] = sacc;
        tacc += (uint64_t)dm.A * ((n + 31) / 32);
        sacc += (uint64_t)dm.A * n;
      }
      tile[L] = (uint32_t)tacc;
      scen[L] = sacc;
    }
    b->r_stat = o_stat;
    b->r_zero = (o_sums - o_stat) + 8 * b->n_sums;
    b->r_h2d = h2d_bytes - o_leaves;
    // when K1 runs, its CTAs read their leaf descriptors straight from the
    // page-locked staging (fetch_leaf): no copy of the table
    bool table_copy = true;
    if (!all_self) {
      LeafDev* dsrc = nullptr;
      if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dsrc), h + o_leaves, 0) == cudaSuccess) {
        bd.leaves_src = dsrc;
        table_copy = false;
      } else {
        cudaGetLastError();
      }
    }
    if (b->resident) {  // set up once, outside the graph (resident_init)
      if (cudaHostAlloc(reinterpret_cast<void**>(&b->hmapped), stat_bytes, cudaHostAllocMapped) != cudaSuccess) {
        b->hmapped = nullptr;
        rc = set_err(DESPOT_ENOMEM, "mapped status block");
      }
      uint32_t* dptr = nullptr;
      if (!rc && cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), b->hmapped, 0) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "mapped status block: device pointer");
      bd.hstat = dptr;
      if (!rc && !b->resident_table && table_copy &&
          cudaMemcpyAsync(s + o_leaves, h + o_leaves, h2d_bytes - o_leaves, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "batch setup copies failed");
    } else if (cudaMemsetAsync(s + o_stat, 0, (o_sums - o_stat) + 8 * b->n_sums, st) != cudaSuccess ||
        cudaMemsetAsync(bd.mins, 0x7F, 4 * b->n_mins, st) != cudaSuccess ||
        (xdense && (size_t)x.nblk * kXBlk > LAS &&
         cudaMemsetAsync(x.flags + LAS, 0, (size_t)x.nblk * kXBlk - LAS, st) != cudaSuccess) ||
        (table_copy &&
         cudaMemcpyAsync(s + o_leaves, h + o_leaves, h2d_bytes - o_leaves, cudaMemcpyHostToDevice, st) != cudaSuccess))
      rc = set_err(DESPOT_ECUDA, "batch setup copies failed");
    if (!b->resident_table) b->h2d += h2d_bytes - o_leaves;
    if (!rc && ilist && idx_total) {
      memcpy(h + o_idx, bind->index, 4 * idx_total);
      if (cudaMemcpyAsync(s + o_idx, h + o_idx, 4 * idx_total, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "index list copy failed");
      b->h2d += 4 * idx_total;
    }
  }
  g_ht.mark("setup_copies");
  // RECORD needs the per-scenario offsets: K1 and K2pre first, then outputs
  // are bound in despot_expand_end (K2 runs there when RECORD is set, since
  // the record pointers arrive with the output struct).
  if (!rc && b->sparse) {
    rc = dispatch_car(dm, [&](auto mdl) -> int {
      using M = decltype(mdl);
      b->mark(1);
      if (!all_self) {
        k1_update_sparse<M><<<L, 256, 0, st>>>(bd);  // + prefix in its last CTA
        ++b->launches;
      }
      b->mark(2);
      return check_launch(m, "K1");
    });
    if (!rc && !(flags & DESPOT_X_RECORD_SCENARIO)) rc = launch_k2_sparse(m, b.get(), false);
    if (!rc && b->sharded_sparse) {  // local grouping now: its records are what the ranks exchange
      b->mark(5);
      rc = launch_group_sparse(m, b.get());
      if (!rc) {  // this rank's records into its block of the all-gather buffer
        PackDev pk{static_cast<unsigned char*>(b->gbuf) + (size_t)m->rank * b->gblk, b->hdr_pad, b->rec_bytes,
                   static_cast<uint32_t*>(b->mscratch), b->gblk};
        k_pack_sparse_scan<<<1, 1024, 0, st>>>(b->bd, pk);
        k_pack_sparse<<<(unsigned)LA, 128, 0, st>>>(b->bd, b->io, pk);
        b->launches += 2;
        rc = check_launch(m, "pack (sharded sparse)");
      }
    }
  } else if (!rc) {
    rc = dispatch_dense(dm, [&](auto mdl) -> int {
      using M = decltype(mdl);
      b->mark(1);
      if (!all_self) {
        const size_t smem1 = align16(sizeof(typename M::Sm)) + align16(dm.sm_table_bytes) +
                             (size_t)M::kScratchPerThread * M::kK1Threads;
        kernel_occupancy((const void*)k1_update<M>, smem1, M::kK1Threads);  // sets the smem attribute if > 48 KB
        // the tile prefix: K2 forms it (no per-scenario records: nothing else
        // reads the prefixes), else K1's last CTA
        // many leaves: K2 searches the tile prefix in global memory (K1's last
        // CTA forms it) -- a shared copy of 4 (L + 1) bytes per CTA would cost
        // MARS its seventh CTA per SM at L = 256
        bd.tile_off_global = L > kTileOffSharedMaxL ? 1u : 0u;
        bd.k2_prefix = ((flags & DESPOT_X_RECORD_SCENARIO) || bd.tile_off_global) ? 0u : 1u;
        k1_update<M><<<L, M::kK1Threads, smem1, st>>>(bd);  // + prefix in its last CTA unless k2_prefix
        ++b->launches;
      }
      b->mark(2);
      return check_launch(m, "K1");
    });
  }
  g_ht.mark("k1");
  // single-call batches bind their outputs now: a small dense batch then runs
  // its finalize in K2's last CTA (no K3 launches)
  if (!rc && bind) {
    despot_batch* raw = b.release();
    if ((rc = bind_outputs(raw, bind, st))) return rc;  // the batch is freed
    b.reset(raw);
    const uint64_t LAd = (uint64_t)L * dm.A;
    // fused only when K2's 4 warps finish it in ~2 sweeps (else the 32-warp
    // k3_small_dense is faster than the launch it saves)
    const uint64_t G = 32 / small_group_width(b->S);
    b->k3_fused = !b->sparse && !(flags & DESPOT_X_RECORD_SCENARIO) && m->world == 1 && !b->xlib && b->S <= 32 &&
                  LAd <= 4 * G * kSmallUnroll * 2;
    b->bd.fused_k3 = b->k3_fused ? 1u : 0u;
  }
  g_ht.mark("bind");
  if (!rc && !b->sparse && !(flags & DESPOT_X_RECORD_SCENARIO)) {
    // K2 now (the exchange block is complete after it)
    rc = dispatch_dense(dm, [&](auto mdl) -> int {
      using M = decltype(mdl);
      // Sm | tables | tile_off | max(the fused finalize's region, the per-thread scratch)
      const size_t smem = align16(sizeof(typename M::Sm)) + align16(dm.sm_table_bytes) +
                          (bd.tile_off_global ? 0 : align16(4 * ((size_t)L + 1))) +
                          std::max<size_t>(b->k3_fused ? small_finalize_smem((uint64_t)L * dm.A) : 0,
                                           (size_t)M::kScratchPerThread * 128);
      bool uni = true;
      for (uint32_t l = 1; l < L; ++l) uni = uni && ld[l].seed_lo == ld[0].seed_lo && ld[l].seed_hi == ld[0].seed_hi;
      // per-lane reductions unless some (leaf, action) spans many tiles (kernels.cuh)
      uint32_t max_chunks = 0;
      for (uint32_t l = 0; l < L; ++l) max_chunks = std::max<uint32_t>(max_chunks, (parent[l]->cap + 31) / 32);
      // (with chunk-major tiles the warps in flight spread over all A x S
      // slots of a leaf: enough of them keep per-lane reductions cheap at any
      // belief size -- config 5 208 -> 198 ms)
      const bool lane_red = HD_K2_LANE_RED && (max_chunks <= kLaneRedChunks || (uint64_t)dm.A * b->S >= 1024);
      auto kern = uni ? (lane_red ? k2_expand_dense<M, false, true, true> : k2_expand_dense<M, false, true, false>)
                      : (lane_red ? k2_expand_dense<M, false, false, true> : k2_expand_dense<M, false, false, false>);
      const int occ = kernel_occupancy((const void*)kern, smem, 128);
      uint64_t tiles_bound = 0;
      for (uint32_t l = 0; l < L; ++l) tiles_bound += (uint64_t)dm.A * ((parent[l]->cap + 31) / 32);
      uint64_t grid = (tiles_bound + 3) / 4;
      const uint64_t maxg = (uint64_t)m->num_sms * occ;
      if (grid > maxg) grid = maxg;
      if (grid < 1) grid = 1;
      b->mark(3);
      launch_pdl(1, kern, (unsigned)grid, 128, smem, st, bd, round_keys(ld[0].seed_lo, ld[0].seed_hi));
      ++b->launches;
      b->mark(4);
      return check_launch(m, "K2");
    });
  }
  if (rc) {
    free_batch(b.release(), true);
    return rc;
  }
  g_ht.mark("k2");
  *out = b.release();
  return DESPOT_OK;
}

extern "C" int despot_expand_begin(despot_model* m, const despot_leaf* leaves, uint32_t L, uint32_t flags,
                                   void* stream, despot_batch** out) {
  return begin_impl(m, leaves, L, flags, stream, nullptr, out);
}

// The one exchange round of a caller-driven sharded batch.  Dense keys: SUM
// of the exact partial block, MIN of the first ids.  Sparse keys: SUM of the
// per-action partials and the step count, all-gather of the record blocks
// (this rank's block was packed in begin).
extern "C" int despot_batch_exchange(despot_batch* b, despot_exchange* out) {
  if (!b || !out) return set_err(DESPOT_EINVAL, "null argument");
  memset(out, 0, sizeof *out);
  const uint64_t LA = (uint64_t)b->L * b->A;
  const SumLayout lay{LA * b->S, LA};
  out->round = b->xround;
  if (b->xround >= 1) return set_err(DESPOT_EINVAL, "exchange: no further round (more == 0)");
  if (!b->sharded_sparse) {
    out->sums = b->bd.sums;
    out->n_sums = b->n_sums;
    out->mins = b->bd.mins;
    out->n_mins = b->n_mins;
  } else {
    out->sums = b->bd.sums + lay.Q(0, 0);  // [L*A][3] per-action partials + the step count
    out->n_sums = 3 * LA + 1;
    out->gather = b->gbuf;
    out->gather_bytes = b->gblk;
  }
  b->xround = 1;
  return DESPOT_OK;
}

static int nccl_err(despot_model* m, despot_comm* c, ncclResult_t r, const char* what) {
  c->failed = true;
  m->failed = true;
  return set_err(DESPOT_ENCCL, "%s: %s", what, nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "?");
}

// The exchange of a sharded batch on the model's communicator, enqueued on the
// batch's stream between K2 (and the sparse local grouping) and K3 -- no host
// round trip.  Dense keys: the packed protocol of exchange.cuh (two rounds);
// sparse keys: one round (SUM of the per-action partials, all-gather of the
// record blocks).
static int lib_exchange(despot_batch* b) {
  despot_model* m = b->model;
  despot_comm* c = m->comm;
  NcclApi& nc = nccl_api();
  if (!nc.ok) return set_err(DESPOT_ENCCL, "%s", nc.err.c_str());
  if (c->failed) return set_err(DESPOT_ESHUTDOWN, "communicator failed earlier");
  cudaStream_t st = b->stream;
  const uint64_t LA = (uint64_t)b->L * b->A;
  const SumLayout lay{LA * b->S, LA};
  std::lock_guard<std::mutex> g(c->mu);
  b->mark(8);
  ncclResult_t r;
  if (b->sharded_sparse) {
    if ((r = nc.GroupStart()) != ncclSuccess) return nccl_err(m, c, r, "ncclGroupStart");
    r = nc.AllReduce(b->bd.sums + lay.Q(0, 0), b->bd.sums + lay.Q(0, 0), 3 * LA + 1, ncclInt64, ncclSum, c->c, st);
    ncclResult_t r2 = nc.AllGather(static_cast<char*>(b->gbuf) + (size_t)m->rank * b->gblk, b->gbuf, b->gblk, ncclUint8,
                                   c->c, st);
    ncclResult_t r3 = nc.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
      return nccl_err(m, c, r != ncclSuccess ? r : r2 != ncclSuccess ? r2 : r3, "sparse exchange");
    b->x_rounds += 1;
    b->x_bytes += 8 * (3 * LA + 1) + b->gblk;
    b->xround = 1;
  } else {
    XDev& x = b->x;
    const unsigned g1 = (unsigned)std::min<uint64_t>((x.las + kXThreads - 1) / kXThreads, (uint64_t)m->num_sms * 8);
    k4_flags<<<std::max(g1, 1u), kXThreads, 0, st>>>(b->bd, x);
    if ((r = nc.AllReduce(x.flags, x.flags, x.las, ncclUint8, ncclSum, c->c, st)) != ncclSuccess)
      return nccl_err(m, c, r, "exchange round A (slot union)");
    k4_count<<<x.nblk, kXThreads, 0, st>>>(x);
    k4_pack<<<x.nblk, kXThreads, 0, st>>>(b->bd, x);
    if ((r = nc.GroupStart()) != ncclSuccess) return nccl_err(m, c, r, "ncclGroupStart");
    r = nc.AllReduce(x.cpk, x.cpk, 4 * x.ccap + x.qn, ncclInt64, ncclSum, c->c, st);
    ncclResult_t r2 = nc.AllReduce(x.cmin, x.cmin, x.ccap, ncclInt32, ncclMin, c->c, st);
    ncclResult_t r3 = nc.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
      return nccl_err(m, c, r != ncclSuccess ? r : r2 != ncclSuccess ? r2 : r3, "exchange round B (packed sums)");
    k4_unpack<<<x.nblk, kXThreads, 0, st>>>(b->bd, x);
    b->launches += 4;
    b->x_rounds += 2;
    b->x_bytes += x.las + 8 * (4 * x.ccap + x.qn) + 4 * x.ccap;
    b->xround = 1;
    if (int rc = check_launch(m, "K4")) return rc;
  }
  b->mark(9);
  return DESPOT_OK;
}

// Capacity fallback of the packed exchange (all ranks see the same union, so
// all of them come here): the dense partial block, untouched by k4_unpack,
// reduced whole.
static int lib_exchange_dense(despot_batch* b) {
  despot_model* m = b->model;
  despot_comm* c = m->comm;
  NcclApi& nc = nccl_api();
  cudaStream_t st = b->stream;
  std::lock_guard<std::mutex> g(c->mu);
  ncclResult_t r = nc.GroupStart();
  if (r != ncclSuccess) return nccl_err(m, c, r, "ncclGroupStart");
  r = nc.AllReduce(b->bd.sums, b->bd.sums, b->n_sums, ncclInt64, ncclSum, c->c, st);
  ncclResult_t r2 = nc.AllReduce(b->bd.mins, b->bd.mins, b->n_mins, ncclInt32, ncclMin, c->c, st);
  ncclResult_t r3 = nc.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
    return nccl_err(m, c, r != ncclSuccess ? r : r2 != ncclSuccess ? r2 : r3, "exchange (dense fallback)");
  b->x_rounds += 1;
  b->x_bytes += 8 * b->n_sums + 4 * b->n_mins;
  return DESPOT_OK;
}

// End of a sharded sparse batch: merge the gathered records into global
// children (b->bd then points at the merged rows, b->io at the records' keys).
static int merge_sparse(despot_model* m, despot_batch* b) {
  if (b->xround != 1) return set_err(DESPOT_EINVAL, "sharded sparse batch: the exchange round was not run");
  cudaStream_t st = b->stream;
  BatchDev& bd = b->bd;
  const uint64_t LA = (uint64_t)b->L * b->A;
  const uint32_t W = (uint32_t)m->world;
  // merged children per (leaf, action) <= the leaf's global scenarios <= its root's K
  const uint64_t nmax = std::max<uint64_t>(1, b->gn_max);
  if (nmax > 4096) return set_err(DESPOT_EINVAL, "sharded sparse merge: more than 4096 children per (leaf, action)");
  const SumLayout old_lay{LA * b->S, LA};
  const uint32_t mS = (uint32_t)nmax;
  const SumLayout lay{LA * mS, LA};
  // merged rows: offsets [W][LA] | sums | mins | sp_item | nc
  size_t off = 0;
  auto take = [&](size_t bytes) {  // 256-byte aligned regions (vector loads need >= 16)
    size_t o = align256(off);
    off = o + align256(bytes);
    return o;
  };
  const size_t o_offs = take(4 * W * LA), o_sums = take(8 * lay.total()), o_mins = take(4 * LA * mS),
               o_item = take(4 * LA * mS), o_nc = take(4 * LA);
  void* ms = nullptr;
  if (!(ms = dev_alloc(m, off, st))) return set_err(DESPOT_ENOMEM, "merge scratch (%zu bytes)", off);
  dev_free(m, b->mscratch, st);  // the pack offsets are no longer needed
  b->mscratch = ms;
  char* s = static_cast<char*>(ms);
  int64_t* nsums = reinterpret_cast<int64_t*>(s + o_sums);
  if (cudaMemsetAsync(nsums, 0, 8 * lay.Q(0, 0), st) != cudaSuccess ||
      cudaMemcpyAsync(nsums + lay.Q(0, 0), bd.sums + old_lay.Q(0, 0), 8 * (3 * LA + 1), cudaMemcpyDeviceToDevice,
                      st) != cudaSuccess ||
      cudaMemsetAsync(s + o_mins, 0x7F, 4 * LA * mS, st) != cudaSuccess)
    return set_err(DESPOT_ECUDA, "merge setup failed");
  bd.sums = nsums;
  bd.mins = reinterpret_cast<int32_t*>(s + o_mins);
  bd.sp_item = reinterpret_cast<uint32_t*>(s + o_item);
  bd.nc = reinterpret_cast<uint32_t*>(s + o_nc);
  bd.S = mS;
  b->S = mS;
  MergeDev g{static_cast<const unsigned char*>(b->gbuf), b->gblk, b->hdr_pad, b->rec_bytes, W,
             reinterpret_cast<uint32_t*>(s + o_offs)};
  k_merge_offsets<<<1, 1024, 0, st>>>(bd, g);
  uint32_t tbits = 1;
  while ((1ull << tbits) < 2 * nmax) ++tbits;
  const size_t smem = 16 * ((size_t)1 << tbits) + 12 * nmax;
  kernel_occupancy((const void*)k3_merge_sparse, smem, 512);  // sets the smem attribute if > 48 KB
  k3_merge_sparse<<<(unsigned)LA, 512, smem, st>>>(bd, g, tbits);
  b->launches += 2;
  b->io.keys = reinterpret_cast<uint32_t*>(static_cast<char*>(b->gbuf) + kRecKey);
  b->io.kstride = b->rec_bytes / 4;
  return check_launch(m, "K3a(merge)");
}

extern "C" int despot_batch_abort(despot_batch* b) {
  if (!b) return DESPOT_OK;
  cudaSetDevice(b->model->device);
  free_batch(b, true);
  return DESPOT_OK;
}

// Binds the caller's outputs (or a device staging block for host outputs) to
// the batch.  On error the batch is freed.
static int bind_outputs(despot_batch* b, despot_expansion* out, cudaStream_t st) {
  despot_model* m = b->model;
  const DevModel& dm = m->host;
  b->stream = st;
  const uint32_t L = b->L;
  const uint64_t LA = (uint64_t)L * dm.A;
  const bool dev_out = out->flags & DESPOT_X_DEVICE_OUTPUTS;
  const bool record = b->flags & DESPOT_X_RECORD_SCENARIO;
  BatchDev& bd = b->bd;
  const uint32_t C = out->child_capacity;
  bd.child_capacity = C;
  bd.scen_capacity = record ? out->scen_capacity : 0;
  if (!out->node || !out->n_scen || !out->weight || !out->act_reward || !out->act_upper || !out->act_lower ||
      !out->child_begin || (C && (!out->child_count || !out->child_first || !out->child_weight ||
                                  !out->child_upper || !out->child_lower || !out->child_obs))) {
    free_batch(b, true);
    return set_err(DESPOT_EINVAL, "missing output arrays");
  }
  if (record && (!out->scen_obs || !out->scen_reward || !out->scen_upper || !out->scen_lower || !out->scen_len ||
                 !out->scen_hash)) {
    free_batch(b, true);
    return set_err(DESPOT_EINVAL, "RECORD_SCENARIO needs the scen_* arrays");
  }
  // output staging (host-output mode) in one allocation
  void*& stage = b->stage;
  size_t so = 0;
  auto take = [&](size_t bytes) {
    size_t o = so;
    so += align256(bytes ? bytes : 4);
    return o;
  };
  const uint64_t S = bd.scen_capacity;
  auto& o_ns = b->o_ns; auto& o_w = b->o_w; auto& o_ar = b->o_ar; auto& o_au = b->o_au; auto& o_al = b->o_al;
  auto& o_cb = b->o_cb; auto& o_cc = b->o_cc; auto& o_cf = b->o_cf; auto& o_cw = b->o_cw; auto& o_cu = b->o_cu;
  auto& o_cl = b->o_cl; auto& o_co = b->o_co; auto& o_so = b->o_so;
  size_t o_sr, o_su, o_sl, o_sn, o_sh, o_ss, o_sc;
  o_ns = take(4 * L), o_w = take(4 * L), o_ar = take(4 * LA), o_au = take(4 * LA),
  o_al = take(4 * LA), o_cb = take(4 * (LA + 1)), o_cc = take(4 * (size_t)C),
  o_cf = take(4 * (size_t)C), o_cw = take(4 * (size_t)C), o_cu = take(4 * (size_t)C),
  o_cl = take(4 * (size_t)C), o_co = take(4 * (size_t)C * dm.OW),
  o_so = take(record ? 4 * S * dm.OW : 0), o_sr = take(record ? 4 * S : 0),
  o_su = take(record ? 4 * S : 0), o_sl = take(record ? 4 * S : 0),
  o_sn = take(record ? 4 * S : 0), o_sh = take(record ? 8 * S : 0),
  o_ss = take(record && out->scen_states ? 4 * S * dm.SW : 0),
  o_sc = take(record && out->scen_child ? 4 * S : 0);
  // page-locked host outputs: bind their device mappings (UVA: the same
  // addresses) and let the kernels write them in place -- for dense keys
  // and outputs of at most kZeroCopyMaxBytes at capacity (the call then has
  // no copy at all and one round trip; measured e2e: config 3 +20 %, while
  // config 2's 2.3 MB and the driving model's 10 MB of children travel
  // faster as bulk copies)
  const uint64_t cap_bytes = 4 * (2 * (uint64_t)L + 4 * LA + 1) + 4 * (uint64_t)C * (5 + dm.OW);
  if (!dev_out && !record && C && !b->sparse && cap_bytes <= kZeroCopyMaxBytes && outputs_pinned(out, C)) {
    void* const hp[] = {out->n_scen, out->weight, out->act_reward, out->act_upper, out->act_lower, out->child_begin,
                        out->child_count, out->child_first, out->child_weight, out->child_upper, out->child_lower,
                        out->child_obs};
    void* dp[12];
    bool ok = true;
    for (int k = 0; k < 12 && ok; ++k) ok = cudaHostGetDevicePointer(&dp[k], hp[k], 0) == cudaSuccess;
    if (ok) {
      b->zc_out = true;
      bd.n_scen = static_cast<uint32_t*>(dp[0]);
      bd.weight = static_cast<float*>(dp[1]);
      bd.act_reward = static_cast<float*>(dp[2]);
      bd.act_upper = static_cast<float*>(dp[3]);
      bd.act_lower = static_cast<float*>(dp[4]);
      bd.child_begin = static_cast<uint32_t*>(dp[5]);
      bd.child_count = static_cast<uint32_t*>(dp[6]);
      bd.child_first = static_cast<uint32_t*>(dp[7]);
      bd.child_weight = static_cast<float*>(dp[8]);
      bd.child_upper = static_cast<float*>(dp[9]);
      bd.child_lower = static_cast<float*>(dp[10]);
      bd.child_obs = static_cast<uint32_t*>(dp[11]);
      bd.scen_obs = nullptr;
      bd.scen_reward = bd.scen_upper = bd.scen_lower = nullptr;
      bd.scen_len = nullptr;
      bd.scen_hash = nullptr;
      bd.scen_states = nullptr;
      bd.scen_child = nullptr;
      b->bound = true;
      return DESPOT_OK;
    }
    cudaGetLastError();
  }
  if (dev_out) {
    bd.n_scen = out->n_scen;
    bd.weight = out->weight;
    bd.act_reward = out->act_reward;
    bd.act_upper = out->act_upper;
    bd.act_lower = out->act_lower;
    bd.child_begin = out->child_begin;
    bd.child_count = out->child_count;
    bd.child_first = out->child_first;
    bd.child_weight = out->child_weight;
    bd.child_upper = out->child_upper;
    bd.child_lower = out->child_lower;
    bd.child_obs = out->child_obs;
    bd.scen_obs = out->scen_obs;
    bd.scen_reward = out->scen_reward;
    bd.scen_upper = out->scen_upper;
    bd.scen_lower = out->scen_lower;
    bd.scen_len = out->scen_len;
    bd.scen_hash = out->scen_hash;
    bd.scen_states = out->scen_states;
    bd.scen_child = record ? out->scen_child : nullptr;
  } else {
    if (b->persistent ? cudaMalloc(&stage, so) != cudaSuccess : !(stage = dev_alloc(b->model, so, st))) {
      free_batch(b, true);
      return set_err(DESPOT_ENOMEM, "output staging (%zu bytes)", so);
    }
    char* p = static_cast<char*>(stage);
    bd.n_scen = reinterpret_cast<uint32_t*>(p + o_ns);
    bd.weight = reinterpret_cast<float*>(p + o_w);
    bd.act_reward = reinterpret_cast<float*>(p + o_ar);
    bd.act_upper = reinterpret_cast<float*>(p + o_au);
    bd.act_lower = reinterpret_cast<float*>(p + o_al);
    bd.child_begin = reinterpret_cast<uint32_t*>(p + o_cb);
    bd.child_count = reinterpret_cast<uint32_t*>(p + o_cc);
    bd.child_first = reinterpret_cast<uint32_t*>(p + o_cf);
    bd.child_weight = reinterpret_cast<float*>(p + o_cw);
    bd.child_upper = reinterpret_cast<float*>(p + o_cu);
    bd.child_lower = reinterpret_cast<float*>(p + o_cl);
    bd.child_obs = reinterpret_cast<uint32_t*>(p + o_co);
    bd.scen_obs = reinterpret_cast<uint32_t*>(p + o_so);
    bd.scen_reward = reinterpret_cast<float*>(p + o_sr);
    bd.scen_upper = reinterpret_cast<float*>(p + o_su);
    bd.scen_lower = reinterpret_cast<float*>(p + o_sl);
    bd.scen_len = reinterpret_cast<uint32_t*>(p + o_sn);
    bd.scen_hash = reinterpret_cast<uint64_t*>(p + o_sh);
    bd.scen_states = (record && out->scen_states) ? reinterpret_cast<uint32_t*>(p + o_ss) : nullptr;
    bd.scen_child = (record && out->scen_child) ? reinterpret_cast<uint32_t*>(p + o_sc) : nullptr;
  }
  b->bound = true;
  return DESPOT_OK;
}

// every host output array of `out` is page-locked (cudaHostAlloc /
// cudaHostRegister): the D2H copies can then go straight into them
static bool outputs_pinned(const despot_expansion* out, uint32_t C) {
  auto pinned = [](const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost;
  };
  const void* head[] = {out->n_scen, out->weight, out->act_reward, out->act_upper, out->act_lower, out->child_begin};
  for (const void* p : head)
    if (!pinned(p)) return false;
  if (C) {
    const void* ch[] = {out->child_count, out->child_first, out->child_weight, out->child_upper, out->child_lower,
                        out->child_obs};
    for (const void* p : ch)
      if (!pinned(p)) return false;
  }
  return true;
}

// Completes a bound batch: [K2 for RECORD] -> K3 (unless fused into K2) ->
// status and outputs to the host -> frees the batch.
// finish_batch modes: the whole completion (the plain call), only the device
// work up to the copies (captured into a prepared batch's graph), or only the
// host side after a prepared batch's graph launch
enum FinishMode { kFinishFull = 0, kFinishEnqueue = 1, kFinishComplete = 2 };
static int finish_batch(despot_batch* b, despot_expansion* out, cudaStream_t st, int mode = kFinishFull) {
  despot_model* m = b->model;
  const DevModel& dm = m->host;
  const uint32_t L = b->L;
  const uint64_t LA = (uint64_t)L * dm.A;
  const bool dev_out = (out->flags & DESPOT_X_DEVICE_OUTPUTS) || b->zc_out;  // (zero-copy: written in place)
  const bool record = b->flags & DESPOT_X_RECORD_SCENARIO;
  BatchDev& bd = b->bd;
  const uint32_t C = out->child_capacity;
  void* stage = b->stage;
  const size_t o_ns = b->o_ns, o_w = b->o_w, o_ar = b->o_ar, o_au = b->o_au, o_al = b->o_al, o_cb = b->o_cb,
               o_cc = b->o_cc, o_cf = b->o_cf, o_cw = b->o_cw, o_cu = b->o_cu, o_cl = b->o_cl, o_co = b->o_co,
               o_so = b->o_so;
  int rc = DESPOT_OK;
  if (mode == kFinishComplete) {
  } else if (record && b->sparse) {
    rc = launch_k2_sparse(m, b, true);
  } else if (record) {
    rc = dispatch_dense(dm, [&](auto mdl) -> int {
      using M = decltype(mdl);
      const size_t smem = align16(sizeof(typename M::Sm)) + align16(dm.sm_table_bytes) +
                          (bd.tile_off_global ? 0 : align16(4 * ((size_t)L + 1))) +
                          (size_t)M::kScratchPerThread * 128;
      auto kern = k2_expand_dense<M, true>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      b->mark(3);
      kern<<<(unsigned)(m->num_sms * 4), 128, smem, st>>>(bd, RoundKeys{});
      ++b->launches;
      b->mark(4);
      return check_launch(m, "K2(record)");
    });
  }
  auto launch_k3 = [&]() -> int {
    int rc = DESPOT_OK;
    const unsigned warps_per_cta = 4;
    const unsigned g3 = (unsigned)((LA + warps_per_cta - 1) / warps_per_cta);
    b->mark(5);
    // small dense batches (few slots): rank + scan + write in one CTA (or in
    // K2's last CTA, already done, when the batch was fused)
    // the single-CTA finalize when its 32 warps cover the pairs in about one
    // sweep; beyond that the multi-CTA kernels win (their launches overlap)
    const bool small_k3 = !b->sparse && b->S <= 32 &&
                          LA <= std::min<uint64_t>(kSmallLA, 32 * (32 / small_group_width(b->S)) * 2);
    if (b->k3_fused) {
    } else if (!rc && wide_fused(b->S, b->sparse)) {
      // many slots: rank + look-back scan + write in one kernel, a CTA per (leaf, action)
      static std::once_flag once;
      std::call_once(once, [] {
        for (auto k : {k3_wide_fused<1>, k3_wide_fused<2>, k3_wide_fused<4>})
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideFusedMaxSmem);
      });
      auto kern = b->S <= kWideFusedThreads       ? k3_wide_fused<1>
                  : b->S <= 2 * kWideFusedThreads ? k3_wide_fused<2>
                                                  : k3_wide_fused<4>;
      launch_pdl(2, kern, (unsigned)LA, kWideFusedThreads, wide_fused_smem(b->S), st, bd);
      ++b->launches;
      rc = check_launch(m, "K3(wide)");
    } else if (!rc && b->sharded_sparse) {
      rc = merge_sparse(m, b);  // the ranks' records -> global children
    } else if (!rc && b->sparse) {
      rc = launch_group_sparse(m, b);
    } else if (!rc && small_k3) {
      // small batch: rank + scan + write in one CTA (one launch instead of three)
      const size_t smem = small_finalize_smem(LA);
      static std::once_flag once;
      std::call_once(once, [] { cudaFuncSetAttribute(k3_small_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10); });
      launch_pdl(2, k3_small_dense, 1, 1024, smem, st, bd);
      ++b->launches;
      rc = check_launch(m, "K3(small)");
    } else if (!rc && b->S <= 16) {  // counts only: k3_write_grouped recomputes the ordinals
      const uint64_t pairs_per_cta = 4 * (32 / small_group_width(b->S));
      launch_pdl(2, k3_count_grouped, (unsigned)((LA + pairs_per_cta - 1) / pairs_per_cta), 128, 0, st, bd);
      ++b->launches;
      rc = check_launch(m, "K3a");
    } else if (!rc) {
      launch_pdl(2, k3_rank_dense, g3, 128, warps_per_cta * b->S * 8, st, bd);
      ++b->launches;
      rc = check_launch(m, "K3a");
    }
    const bool wide1 = wide_fused(b->S, b->sparse);
    if (!rc && !small_k3 && !b->k3_fused && !wide1) {
      launch_pdl(2, k3_scan_lookback, (unsigned)((LA + kScanTile - 1) / kScanTile), kScanTile, 0, st, bd);
      ++b->launches;
      rc = check_launch(m, "K3b");
    }
    if (!rc && b->sparse) {
      launch_pdl(2, k3_write_sparse, (unsigned)LA, kWriteSparseThreads, 0, st, bd, b->io);  // (merged: keys from the gathered records)
      ++b->launches;
      rc = check_launch(m, "K3c(sparse)");
    } else if (!rc && !small_k3 && !wide1) {
      if (b->S > kWideS) {
        launch_pdl(2, k3_write_wide, (unsigned)LA, 256, 0, st, bd);
      } else if (b->S <= 16) {
        const uint64_t pairs_per_cta = 4 * (32 / small_group_width(b->S));
        launch_pdl(2, k3_write_grouped, (unsigned)((LA + pairs_per_cta - 1) / pairs_per_cta), 128, 0, st, bd);
      } else {
        launch_pdl(2, k3_write_dense, g3, 128, 0, st, bd);
      }
      ++b->launches;
      rc = check_launch(m, "K3c");
    }
    if (!rc && record && bd.scen_child) {  // each scenario's child ordinal
      launch_pdl(2, k3_scen_child, (unsigned)m->num_sms * 4, 256, 0, st, bd, b->sparse ? 0u : 1u);
      ++b->launches;
      rc = check_launch(m, "scen_child");
    }
    b->mark(6);
    return rc;
  };
  if (!rc && mode != kFinishComplete) rc = launch_k3();
  g_ht.mark("k3");
  // status block: err | total children | steps | ticket | pad | n_leaf[L]
  const size_t stat_bytes = 4 * kStatWords + 4 * (size_t)L;
  // (a prepared batch keeps its status and output staging: its graph copies into them)
  if (!b->hs) b->hs = static_cast<char*>(pinned_pool().acquire(stat_bytes + 64));
  char* hs = b->hs;
  struct PinGuard {
    despot_batch* b;
    ~PinGuard() {
      if (!b->persistent) {
        pinned_pool().release(b->hs);
        b->hs = nullptr;
      }
    }
  } pin_guard{b};
  if (!rc && !hs) rc = set_err(DESPOT_ENOMEM, "pinned staging");
  // host outputs: the staging block [per-leaf | per-action | CSR | children]
  // goes to one pinned buffer; when it is small (search-sized batches) the
  // whole block travels in this first copy and no second round trip is needed
  char*& hp_out = b->hp_out;
  const size_t head_bytes = o_cc, body_bytes = o_so;
  // page-locked caller buffers: every array is copied straight into them (no
  // staging, no host memcpy); else the head goes through the library's pinned
  // staging (with the whole block when it is small) and the children directly
  // (small blocks: one staging copy beats a dozen small DMA copies)
  const bool small = body_bytes <= (1u << 20);  // every array at capacity in the first round trip
  const bool pinned_out = !dev_out && !record && !small && outputs_pinned(out, C);
  const bool one_copy = small;
  struct PinRelease {
    despot_batch* b;
    ~PinRelease() {
      if (b->hp_out && !b->persistent) {
        pinned_pool().release(b->hp_out);
        b->hp_out = nullptr;
      }
    }
  } pin_out_guard{b};
  auto copy_and_sync = [&](bool enqueue, bool sync) -> int {
    int rc = DESPOT_OK;
    if (enqueue) {
    if (!rc && !b->resident) {  // (resident: K2's last CTA writes it to mapped memory)
      b->d2h += stat_bytes;
      if (cudaMemcpyAsync(hs, bd.status, stat_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "status copy failed");
    }
    if (!rc && pinned_out) {
      const struct {
        void* dst;
        size_t off, bytes;
      } head[] = {{out->n_scen, o_ns, 4 * (size_t)L},  {out->weight, o_w, 4 * (size_t)L},
                  {out->act_reward, o_ar, 4 * LA},     {out->act_upper, o_au, 4 * LA},
                  {out->act_lower, o_al, 4 * LA},      {out->child_begin, o_cb, 4 * (LA + 1)}};
      for (const auto& h : head) b->d2h += h.bytes;
      for (const auto& h : head)
        if (!rc && h.dst && h.bytes &&
            cudaMemcpyAsync(h.dst, static_cast<char*>(stage) + h.off, h.bytes, cudaMemcpyDeviceToHost, st) !=
                cudaSuccess)
          rc = set_err(DESPOT_ECUDA, "output copy failed");
    } else if (!rc && !dev_out) {
      if (!hp_out) hp_out = static_cast<char*>(pinned_pool().acquire(one_copy ? body_bytes : head_bytes));
      if (!hp_out) rc = set_err(DESPOT_ENOMEM, "pinned output staging");
      else if ((b->d2h += one_copy ? body_bytes : head_bytes,
                cudaMemcpyAsync(hp_out, stage, one_copy ? body_bytes : head_bytes, cudaMemcpyDeviceToHost, st)) !=
               cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "output copy failed");
    }
    g_ht.mark("d2h_enqueued");
    b->mark(7);  // end of the call's device work (before the host waits: no extra round trip)
    }
    if (sync && !rc && cudaStreamSynchronize(st) != cudaSuccess) {
      m->failed = true;
      rc = set_err(DESPOT_ECUDA, "batch failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    g_ht.mark("synced");
    return rc;
  };
  if (!rc) rc = copy_and_sync(mode != kFinishComplete, mode != kFinishEnqueue);
  if (mode == kFinishEnqueue) return rc;  // a prepared batch's capture ends here
  if (b->resident) hs = reinterpret_cast<char*>(b->hmapped);  // published by K2's / K3's last CTA
  if (!rc && b->xlib && !b->sparse) {
    // the packed exchange's capacity hint follows the largest union seen (+ 1/4)
    uint32_t T = 0, e0 = 0;
    memcpy(&T, hs + 4 * kStatXTotal, 4);
    memcpy(&e0, hs, 4);
    const uint64_t want = std::min<uint64_t>(((uint64_t)T * 20 + LA - 1) / std::max<uint64_t>(LA, 1), 16ull * b->S);
    uint32_t cur = m->xratio16.load();
    while (want > cur && !m->xratio16.compare_exchange_weak(cur, (uint32_t)want)) {
    }
    if (e0 & kErrXOverflow) {  // every rank saw the same union: the dense fallback, then K3 again
      if (cudaMemsetAsync(bd.err, 0, 4, st) != cudaSuccess ||
          cudaMemsetAsync(bd.scan_flags, 0, 8 * scan_words(LA, b->S, b->sparse), st) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "capacity retry reset failed");
      if (!rc) rc = lib_exchange_dense(b);
      if (!rc) rc = launch_k3();
      if (!rc) rc = copy_and_sync(true, true);
    }
  }
  uint32_t err = 0, nchildren = 0;
  uint64_t steps = 0;
  if (!rc) {
    memcpy(&err, hs, 4);
    memcpy(&nchildren, hs + 4, 4);
    memcpy(&steps, hs + 8, 8);
    out->num_children = nchildren;
    out->scenario_steps = steps;
    out->launches = b->launches;
    if (err & kErrCheck) rc = set_err(DESPOT_ECUDA, "a device self-check failed (HD_CHECKS build)");
    else if (err & kErrIndexList)
      rc = set_err(DESPOT_EINVAL, "an index list names a scenario whose replayed observation is not the leaf's key");
    else if (err & kErrEmptyLeaf) rc = set_err(DESPOT_EINVAL, "a leaf has an empty scenario set (unknown child ordinal)");
    else if (err & kErrHash) rc = set_err(DESPOT_EHASH, "64-bit observation-hash collision");
    else if (err & kErrChildCap)
      rc = set_err(DESPOT_ECAPACITY, "child_capacity %u < %u children", C, nchildren);
    else if (err & kErrScenCap) rc = set_err(DESPOT_ECAPACITY, "scen_capacity too small");
  }
  if (b->resident && (rc || err)) b->dirty = true;  // the device state is not known to be restored
  if (!rc && !dev_out) {
    const uint64_t Cu = nchildren;
    uint64_t Su = 0;
    const uint32_t* nl = reinterpret_cast<const uint32_t*>(hs + 4 * kStatWords);
    for (uint32_t l = 0; l < L; ++l) Su += (uint64_t)dm.A * nl[l];
    struct Part {
      void* dst;
      size_t off, bytes;
    } parts[] = {
        {out->n_scen, o_ns, 4 * (size_t)L},           {out->weight, o_w, 4 * (size_t)L},
        {out->act_reward, o_ar, 4 * LA},              {out->act_upper, o_au, 4 * LA},
        {out->act_lower, o_al, 4 * LA},               {out->child_begin, o_cb, 4 * (LA + 1)},
        {out->child_count, o_cc, 4 * Cu},             {out->child_first, o_cf, 4 * Cu},
        {out->child_weight, o_cw, 4 * Cu},            {out->child_upper, o_cu, 4 * Cu},
        {out->child_lower, o_cl, 4 * Cu},             {out->child_obs, o_co, 4 * Cu * dm.OW},
    };
    if (pinned_out)
      for (int k = 0; k < 6; ++k) parts[k].bytes = 0;  // already in the caller's buffers
    if (!small) {  // second round trip: the used part of each child array, straight to the caller
      for (int k = 6; k < 12; ++k) {
        b->d2h += parts[k].bytes;
        if (parts[k].bytes && cudaMemcpyAsync(parts[k].dst, static_cast<char*>(stage) + parts[k].off,
                                              parts[k].bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
          rc = set_err(DESPOT_ECUDA, "output copy failed");
        parts[k].bytes = 0;  // nothing left to move on the host
      }
    }
    // per-scenario records (validation mode): direct copies
    struct Cp {
      void* dst;
      const void* src;
      size_t bytes;
    } cps[] = {
        {record ? out->scen_obs : nullptr, bd.scen_obs, 4 * Su * dm.OW},
        {record ? out->scen_reward : nullptr, bd.scen_reward, 4 * Su},
        {record ? out->scen_upper : nullptr, bd.scen_upper, 4 * Su},
        {record ? out->scen_lower : nullptr, bd.scen_lower, 4 * Su},
        {record ? out->scen_len : nullptr, bd.scen_len, 4 * Su},
        {record ? out->scen_hash : nullptr, bd.scen_hash, 8 * Su},
        {record ? out->scen_states : nullptr, bd.scen_states, 4 * Su * dm.SW},
        {record ? out->scen_child : nullptr, bd.scen_child, 4 * Su},
    };
    for (auto& c : cps)
      if (!rc && c.dst && c.src && c.bytes &&
          (b->d2h += c.bytes, cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        rc = set_err(DESPOT_ECUDA, "output copy failed");
    if (!rc && (!small || record) && cudaStreamSynchronize(st) != cudaSuccess)
      rc = set_err(DESPOT_ECUDA, "output copy sync failed");
    if (!rc)
      for (auto& p : parts)
        if (p.bytes) memcpy(p.dst, hp_out + p.off, p.bytes);
  }
  out->exchange_ms = 0.0f;
  if (!rc && b->timing) {  // the events are complete: the stream was synchronised
    const int pairs[4][2] = {{1, 2}, {3, 4}, {5, 6}, {0, 7}};
    for (int k = 0; k < 4; ++k) {
      float ms = 0.0f;
      if (!b->timing_k2 || k == 1) cudaEventElapsedTime(&ms, b->ev[pairs[k][0]], b->ev[pairs[k][1]]);
      out->phase_ms[k] = ms;
    }
    if (b->xlib && !b->timing_k2) cudaEventElapsedTime(&out->exchange_ms, b->ev[8], b->ev[9]);
  }
  out->exchange_rounds = b->x_rounds;
  out->exchange_bytes = b->x_bytes;
  if (rc) {
    free_batch(b, true);
    return rc;
  }
  const uint32_t* nl = reinterpret_cast<const uint32_t*>(hs + 4 * kStatWords);
  for (uint32_t l = 0; l < L; ++l) {
    Node* nd = b->leaf_node[l];
    if (b->is_new[l]) nd->n = nl[l];
    nd->expanded = true;
    out->node[l] = reinterpret_cast<despot_node>(nd);
  }
  if (b->zc_out) {  // the outputs the kernels wrote across the bus
    const uint64_t Cu = std::min<uint64_t>(out->num_children, C);
    b->d2h += 4 * (2 * (uint64_t)L + 3 * LA + LA + 1) + 4 * Cu * (5 + dm.OW);
  }
  out->h2d_bytes = b->h2d;
  out->d2h_bytes = b->d2h;
  g_ht.mark("outputs");
  free_batch(b, false);
  g_ht.mark("freed");
  g_ht.dump();
  return DESPOT_OK;
}

extern "C" int despot_expand_end(despot_batch* b, despot_expansion* out, void* stream) {
  if (!b || !out) return set_err(DESPOT_EINVAL, "null argument");
  CU(cudaSetDevice(b->model->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (!b->bound) {
    if (int rc = bind_outputs(b, out, st)) return rc;  // frees the batch on error
  }
  return finish_batch(b, out, st);
}

extern "C" int despot_expand_batch(despot_model* m, const despot_leaf* leaves, uint32_t L,
                                   despot_expansion* out, void* stream) {
  g_ht.start();
  if (!m || !out) return set_err(DESPOT_EINVAL, "null argument");
  if (m->world > 1 && !m->comm)
    return set_err(DESPOT_EINVAL, "world > 1 without a communicator: use despot_expand_begin/exchange/end");
  despot_batch* b = nullptr;
  // outputs are bound before K2 so that small batches finalize in K2's last CTA
  int rc = begin_impl(m, leaves, L, out->flags, stream, out, &b);
  if (rc) return rc;
  if (b->xlib && (rc = lib_exchange(b))) {  // K4: the exchange on the model's communicator
    free_batch(b, true);
    return rc;
  }
  return despot_expand_end(b, out, stream);
}

// ===========================================================================
// prepared batches: one CUDA graph per repeated batch (SURVEY §7 hard part 6)
// ===========================================================================
struct despot_prepared {
  despot_model* m = nullptr;
  despot_batch* b = nullptr;       // persistent: scratch, staging, events, bound outputs
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<Node> tmpl;          // per leaf: the new node's template (arena at kTemplateBase)
  std::vector<despot_leaf> leaves;
  despot_expansion out{};          // the outputs the graph copies into
  uint32_t launches = 0;
  uint64_t h2d = 0, d2h = 0;
};

// a resident batch's starting state: zero status header, n_leaf and the
// prefixes from the host, zero sums, 0x7F first ids, the leaf table
static int resident_init(despot_batch* b, cudaStream_t st) {
  char* s = static_cast<char*>(b->scratch);
  const char* h = static_cast<const char*>(b->pinned);
  if (cudaMemsetAsync(s + b->r_stat, 0, b->r_zero, st) != cudaSuccess ||
      cudaMemsetAsync(b->bd.mins, 0x7F, 4 * b->n_mins, st) != cudaSuccess ||
      (b->resident_table &&
       cudaMemcpyAsync(s + b->o_leaves, h + b->o_leaves, b->r_h2d, cudaMemcpyHostToDevice, st) != cudaSuccess))
    return set_err(DESPOT_ECUDA, "resident batch set-up failed");
  b->dirty = false;
  return DESPOT_OK;
}

static void free_prepared(despot_prepared* p) {
  if (!p) return;
  cudaSetDevice(p->m->device);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (despot_batch* b = p->b) {
    cudaDeviceSynchronize();
    if (b->scratch) cudaFree(b->scratch);
    if (b->stage) cudaFree(b->stage);
    if (b->pinned) pinned_pool().release(b->pinned);
    if (b->hs) pinned_pool().release(b->hs);
    if (b->hp_out) pinned_pool().release(b->hp_out);
    if (b->hmapped) cudaFreeHost(b->hmapped);
    if (b->timing) event_pool().release(b->ev);
    delete b;
  }
  delete p;
}

extern "C" int despot_batch_prepare(despot_model* m, const despot_leaf* leaves, uint32_t L, despot_expansion* out,
                                    despot_prepared** prep) {
  if (!m || !leaves || !out || !prep) return set_err(DESPOT_EINVAL, "null argument");
  if (m->world > 1 || (m->comm && (m->flags & DESPOT_MF_EXCHANGE)))
    return set_err(DESPOT_EINVAL, "prepared batches are single-GPU (world == 1, no exchange)");
  if (out->flags & (DESPOT_X_RECORD_SCENARIO | DESPOT_X_INDEX_LISTS))
    return set_err(DESPOT_EINVAL, "prepared batches do not RECORD or take index lists");
  CU(cudaSetDevice(m->device));
  std::unique_ptr<despot_prepared> p(new despot_prepared());
  p->m = m;
  p->leaves.assign(leaves, leaves + L);
  cudaStream_t cs;
  CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaStreamDestroy(cs);
    return set_err(DESPOT_ECUDA, "cudaStreamBeginCapture failed");
  }
  g_capture = true;
  despot_batch* b = nullptr;
  int rc = begin_impl(m, leaves, L, out->flags, cs, out, &b);
  if (!rc) rc = finish_batch(b, out, cs, kFinishEnqueue);
  g_capture = false;
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (b) {
    p->b = b;  // owned from here (free_prepared releases it)
    for (uint32_t l = 0; l < L; ++l) {
      p->tmpl.push_back(b->is_new[l] ? *b->leaf_node[l] : Node{});
      if (b->is_new[l]) delete b->leaf_node[l];  // templates only: never registered
      b->leaf_node[l] = nullptr;
    }
  }
  p->graph = g;
  if (g && getenv("DESPOT_HOST_TRACE")) {  // the captured nodes, by type
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    fprintf(stderr, "[despot prepared graph] %zu nodes:", nn);
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nd, &t);
      const char* nm = "";
      cudaKernelNodeParams kp;
      if (t == cudaGraphNodeTypeKernel && cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess)
        cudaFuncGetName(&nm, kp.func);
      fprintf(stderr, " %d%s%.40s", (int)t, *nm ? ":" : "", nm);
    }
    fprintf(stderr, "\n");
  }
  if (!rc && (ce != cudaSuccess || !g)) rc = set_err(DESPOT_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
  if (!rc && cudaGraphInstantiate(&p->exec, g, 0) != cudaSuccess)
    rc = set_err(DESPOT_ECUDA, "cudaGraphInstantiate failed");
  if (!rc && b->resident) {
    cudaStream_t is;
    CU(cudaStreamCreateWithFlags(&is, cudaStreamNonBlocking));
    rc = resident_init(b, is);
    if (!rc && cudaStreamSynchronize(is) != cudaSuccess) rc = set_err(DESPOT_ECUDA, "resident batch set-up failed");
    cudaStreamDestroy(is);
  }
  if (rc) {
    cudaGetLastError();
    free_prepared(p.release());
    return rc;
  }
  p->out = *out;
  p->launches = b->launches;
  p->h2d = b->h2d;
  p->d2h = b->d2h;
  *prep = p.release();
  return DESPOT_OK;
}

extern "C" int despot_batch_run(despot_prepared* p, despot_expansion* out, void* stream) {
  if (!p || !out) return set_err(DESPOT_EINVAL, "null argument");
  despot_model* m = p->m;
  despot_batch* b = p->b;
  if (m->failed) return set_err(DESPOT_ESHUTDOWN, "model failed earlier");
  if (out->flags != p->out.flags || out->child_capacity != p->out.child_capacity ||
      out->child_count != p->out.child_count || out->n_scen != p->out.n_scen)
    return set_err(DESPOT_EINVAL, "despot_batch_run: outputs differ from the prepared ones");
  CU(cudaSetDevice(m->device));
  g_ht.start();
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t L = b->L;
  // the parents must still exist (their arenas are in the graph's leaf table)
  for (uint32_t l = 0; l < L; ++l)
    if (!lookup(m, p->leaves[l].parent)) return set_err(DESPOT_EINVAL, "leaf %u: parent released", l);
  // this run's arenas, the nodes, and the leaf table the graph uploads
  b->stream = st;
  if (b->new_bytes) {
    b->new_block = std::make_shared<Block>();
    b->new_block->stream = st;
    b->new_block->model = m;
    if (!(b->new_block->ptr = dev_alloc(m, b->new_bytes, st))) return set_err(DESPOT_ENOMEM, "new arenas");
  }
  const intptr_t shift = b->new_block ? static_cast<char*>(b->new_block->ptr) - reinterpret_cast<char*>(kTemplateBase) : 0;
  auto rebase = [shift](auto* q) { return reinterpret_cast<decltype(q)>(reinterpret_cast<char*>(q) + shift); };
  // the leaf table's arena pointers first (the graph uploads it), the node
  // bookkeeping after the launch, while the GPU runs
  LeafDev* hl = reinterpret_cast<LeafDev*>(static_cast<char*>(b->pinned) + b->o_leaves);
  for (uint32_t l = 0; l < L; ++l) {
    if (p->leaves[l].action < 0) continue;
    const Node& t = p->tmpl[l];
    LeafDev& d = hl[l];
    d.ids = rebase(t.ids);
    d.w = rebase(t.w);
    d.states = rebase(t.states);
    d.keys = rebase(t.keys);
    d.nchild = rebase(t.nchild);
  }
  b->launches = p->launches;
  b->h2d = p->h2d;
  b->d2h = p->d2h;
  if (b->resident && b->dirty) {
    if (int rc = resident_init(b, st)) return rc;
    if (b->resident_table) b->h2d += b->r_h2d;
  }
  g_ht.mark("patched");
  const bool launched = cudaGraphLaunch(p->exec, st) == cudaSuccess;
  g_ht.mark("graph_launched");
  {
    std::lock_guard<std::mutex> g(m->mu);
    for (uint32_t l = 0; l < L; ++l) {
      const despot_leaf& lf = p->leaves[l];
      if (lf.action < 0) {
        b->leaf_node[l] = reinterpret_cast<Node*>(lf.parent);
        b->is_new[l] = false;
        continue;
      }
      Node* nd = new Node(p->tmpl[l]);
      nd->block = b->new_block;
      nd->ids = rebase(nd->ids);
      nd->w = rebase(nd->w);
      nd->states = rebase(nd->states);
      nd->nchild = rebase(nd->nchild);
      nd->keys = rebase(nd->keys);
      m->nodes.insert(nd);
      b->leaf_node[l] = nd;
      b->is_new[l] = true;
    }
  }
  if (!launched) {
    free_batch(b, true);
    return set_err(DESPOT_ECUDA, "cudaGraphLaunch failed");
  }
  return finish_batch(b, out, st, kFinishComplete);
}

extern "C" int despot_batch_prepared_free(despot_prepared* p) {
  free_prepared(p);
  return DESPOT_OK;
}

extern "C" int despot_rollout_bounds(despot_model* m, despot_node h, float* upper_mean, float* lower_mean,
                                     float* per_u, float* per_l, void* stream) {
  Node* nd = m ? lookup(m, h) : nullptr;
  if (!nd) return set_err(DESPOT_EINVAL, "unknown node");
  if (!upper_mean || !lower_mean) return set_err(DESPOT_EINVAL, "null argument");
  if (m->failed) return set_err(DESPOT_ESHUTDOWN, "model failed earlier");
  // a sharded node holds only this rank's scenarios: the means need every rank's sums
  if (m->world > 1 && !m->comm) return set_err(DESPOT_EINVAL, "rollout_bounds: world > 1 without a communicator");
  CU(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  const DevModel& dm = m->host;
  const uint32_t n = nd->n;
  void* scratch = nullptr;
  const size_t bytes = 256 + 8 * (size_t)(n ? n : 1);
  if (!(scratch = dev_alloc(m, bytes, st))) return set_err(DESPOT_ENOMEM, "rollout_bounds scratch");
  int64_t* acc = static_cast<int64_t*>(scratch);
  float* du = reinterpret_cast<float*>(static_cast<char*>(scratch) + 256);
  float* dl = du + (n ? n : 1);
  int rc = DESPOT_OK;
  if (cudaMemsetAsync(acc, 0, 24, st) != cudaSuccess) rc = set_err(DESPOT_ECUDA, "memset");
  if (!rc) {
    auto launch = [&](auto mdl) -> int {
      using M = decltype(mdl);
      const size_t smem = align16(sizeof(typename M::Sm)) + align16(dm.sm_table_bytes) +
                          (size_t)M::kScratchPerThread * 128;
      auto kern = k_rollout_bounds<M>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const unsigned grid = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>((n + 127) / 128, m->num_sms * 8));
      kern<<<grid, 128, smem, st>>>(m->dev, nd->ids, nd->w, nd->states, nd->cap, n, nd->depth,
                                    (uint32_t)nd->seed, (uint32_t)(nd->seed >> 32), 1.0 / nd->wroot, du, dl, acc);
      return check_launch(m, "rollout_bounds");
    };
    if (dm.slots) rc = dispatch_dense(dm, launch);
    else rc = launch(CarThread{});
  }
  if (!rc && m->comm && (m->world > 1 || (m->flags & DESPOT_MF_EXCHANGE))) {  // every rank's exact sums (SPMD)
    NcclApi& nc = nccl_api();
    if (!nc.ok) rc = set_err(DESPOT_ENCCL, "%s", nc.err.c_str());
    if (!rc) {
      std::lock_guard<std::mutex> g(m->comm->mu);
      const ncclResult_t r = nc.AllReduce(acc, acc, 3, ncclInt64, ncclSum, m->comm->c, st);
      if (r != ncclSuccess) rc = nccl_err(m, m->comm, r, "rollout_bounds all-reduce");
    }
  }
  int64_t hacc[3] = {0, 0, 0};
  if (!rc) {
    if (cudaMemcpyAsync(hacc, acc, 24, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        (per_u && n && cudaMemcpyAsync(per_u, du, 4 * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
        (per_l && n && cudaMemcpyAsync(per_l, dl, 4 * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
        cudaStreamSynchronize(st) != cudaSuccess)
      rc = set_err(DESPOT_ECUDA, "rollout_bounds copy failed");
  }
  dev_free(m, scratch, st);
  if (rc) return rc;
  *upper_mean = hacc[0] ? (float)((double)hacc[1] / (double)hacc[0]) : 0.0f;
  *lower_mean = hacc[0] ? (float)((double)hacc[2] / (double)hacc[0]) : 0.0f;
  return DESPOT_OK;
}

extern "C" int despot_stream_words(despot_model* m, uint64_t seed, const uint32_t* ids, uint32_t n, uint32_t t,
                                   uint32_t k, uint32_t* out, void* stream) {
  if (!m || !ids || !out) return set_err(DESPOT_EINVAL, "null argument");
  CU(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) return DESPOT_OK;
  uint32_t* d = nullptr;
  CU(cudaMallocAsync(&d, 8 * (size_t)n, st));
  int rc = DESPOT_OK;
  if (cudaMemcpyAsync(d, ids, 4 * (size_t)n, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = set_err(DESPOT_ECUDA, "copy");
  if (!rc) {
    k_stream_words<<<(n + 255) / 256, 256, 0, st>>>((uint32_t)seed, (uint32_t)(seed >> 32), d, n, t, k, d + n);
    rc = check_launch(m, "stream_words");
  }
  if (!rc && (cudaMemcpyAsync(out, d + n, 4 * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess))
    rc = set_err(DESPOT_ECUDA, "copy back");
  cudaFreeAsync(d, st);
  return rc;
}

extern "C" int despot_philox_ceiling(despot_model* m, uint64_t seed, uint32_t n_threads, uint32_t blocks,
                                     uint32_t reps, void* stream, double* out_ms, uint32_t* out_checksum) {
  if (!m || !out_ms || !out_checksum) return set_err(DESPOT_EINVAL, "null argument");
  if (n_threads == 0 || blocks == 0 || reps == 0) return set_err(DESPOT_EINVAL, "empty K0 launch");
  CU(cudaSetDevice(m->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int occ = kernel_occupancy((const void*)k0_philox, 0, 256);
  const uint64_t full = (uint64_t)m->num_sms * occ;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(full, (n_threads + 255) / 256));
  const RoundKeys rk = round_keys((uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t* d = nullptr;
  CU(cudaMallocAsync(&d, 4 * (size_t)(reps + 1), st));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = DESPOT_OK;
  if (cudaMemsetAsync(d, 0, 4 * (size_t)(reps + 1), st) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
      cudaEventCreate(&e1) != cudaSuccess)
    rc = set_err(DESPOT_ECUDA, "K0 setup");
  if (!rc) {
    k0_philox<<<grid, 256, 0, st>>>(rk, n_threads, blocks, d);  // warm-up
    cudaEventRecord(e0, st);
    for (uint32_t r = 0; r < reps; ++r) k0_philox<<<grid, 256, 0, st>>>(rk, n_threads, blocks, d + 1 + r);
    cudaEventRecord(e1, st);
    rc = check_launch(m, "K0");
  }
  uint32_t cs = 0;
  float ms = 0.0f;
  if (!rc && (cudaMemcpyAsync(&cs, d + 1, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess))
    rc = set_err(DESPOT_ECUDA, "K0 read back");
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFreeAsync(d, st);
  if (rc) return rc;
  *out_ms = (double)ms / reps;
  *out_checksum = cs;
  return DESPOT_OK;
}

// ===========================================================================
// communicator (SURVEY §8(e) "Bootstrap")
// ===========================================================================
extern "C" int despot_comm_unique_id(void* id_out) {
  if (!id_out) return set_err(DESPOT_EINVAL, "null argument");
  NcclApi& nc = nccl_api();
  if (!nc.ok) return set_err(DESPOT_ENCCL, "%s", nc.err.c_str());
  ncclUniqueId id;
  const ncclResult_t r = nc.GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(DESPOT_ENCCL, "ncclGetUniqueId: %s", nc.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id_out, &id, sizeof id);
  return DESPOT_OK;
}

extern "C" int despot_comm_init(const void* id, int rank, int world, int device, despot_comm** out) {
  if (!id || !out) return set_err(DESPOT_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return set_err(DESPOT_EINVAL, "need 0 <= rank < world");
  NcclApi& nc = nccl_api();
  if (!nc.ok) return set_err(DESPOT_ENCCL, "%s", nc.err.c_str());
  CU(cudaSetDevice(device));
  std::unique_ptr<despot_comm> c(new despot_comm());
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  const ncclResult_t r = nc.CommInitRank(&c->c, world, uid, rank);
  if (r != ncclSuccess) return set_err(DESPOT_ENCCL, "ncclCommInitRank: %s", nc.GetErrorString(r));
  c->rank = rank;
  c->world = world;
  c->device = device;
  *out = c.release();
  return DESPOT_OK;
}

extern "C" int despot_comm_destroy(despot_comm* c) {
  if (!c) return DESPOT_OK;
  NcclApi& nc = nccl_api();
  if (nc.ok && c->c) {
    cudaSetDevice(c->device);
    if (c->failed) nc.CommAbort(c->c);
    else nc.CommDestroy(c->c);
  }
  delete c;
  return DESPOT_OK;
}

extern "C" int despot_comm_info(const despot_comm* c, int* rank, int* world, int* nccl_version) {
  if (!c) return set_err(DESPOT_EINVAL, "null argument");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (nccl_version) *nccl_version = nccl_api().version;
  return DESPOT_OK;
}
