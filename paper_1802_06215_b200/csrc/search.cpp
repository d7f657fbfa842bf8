// search.cpp -- host tree driver of libdespot: an anytime parallel DESPOT
// search whose CPU workers coalesce their leaves into batched expansions.
//
//   workers  descend from the root: action by the scenario-based
//                        PO-UCT rule (Eq. 7), observation branch by
//                        the WEU rule with virtual loss (Eqs. 6, 8,
//                        P:355-358); a trial ends at a leaf or when
//                        every WEU is <= 0.
//   batcher              collects the leaves of all workers' trials, expands
//                        up to max_batch of them in ONE backend call
//                        (node-level parallelism), creates the new
//                        children (Eq. 10, done on the CPU as in P:435) and
//                        backs up Eq. 4 along each trial's path.
//
// Readings: weights replace counts (R1); N(b,a) = 0 prefers the
// branch, N(b) = 0 gives no bonus, natural log; the virtual
// loss grows with the number of threads inside the branch; bounds are
// floored / capped by their initial values during backup; a
// node at depth D has the exact value l0 (its roll-out is the tail), so its
// gap is 0; the root action is argmax_a l(b0, a).
// Host-only C++: this file uses libdespot only through include/despot.h.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/despot.h"

// sets the calling thread's despot_last_error message (despot.cu)
extern "C" int despot__set_error(int code, const char* msg);

namespace {

struct TNode;

// A belief node's bounds and counts (every node, expanded or not, is one of
// these; the root's lives in Search).  Children of an expanded node are a
// contiguous array of records; a full TNode exists only once a trial
// descends into the child.
struct TChild {
  float weight = 0.0f;  // W_b'
  uint32_t n_scen = 0;  // |Phi_b'|
  double u0 = 0.0, l0 = 0.0;
  std::atomic<double> upper{0.0}, lower{0.0};
  std::atomic<int> active{0};  // threads inside this branch (virtual loss)
  std::atomic<TNode*> node{nullptr};
  TChild() = default;
  TChild(float w, uint32_t n, double u, double l)
      : weight(w), n_scen(n), u0(u), l0(l), upper(u), lower(l), active(0), node(nullptr) {}
};

// Bump allocator for the child records of a search (all freed with it; a
// TChild needs no destructor): one construction per record instead of a
// zero-initialised array per node and a second pass over it.
class ChildArena {
 public:
  TChild* alloc(size_t n) {
    const size_t bytes = (n ? n : 1) * sizeof(TChild);
    std::lock_guard<std::mutex> g(mu_);
    if (bytes > left_) {
      const size_t chunk = std::max<size_t>(bytes, size_t(32) << 20);
      chunks_.emplace_back(new (std::nothrow) unsigned char[chunk + alignof(TChild)]);
      if (!chunks_.back()) return nullptr;
      uintptr_t p = reinterpret_cast<uintptr_t>(chunks_.back().get());
      p = (p + alignof(TChild) - 1) & ~(uintptr_t)(alignof(TChild) - 1);
      cur_ = reinterpret_cast<unsigned char*>(p);
      left_ = chunk;
    }
    TChild* r = reinterpret_cast<TChild*>(cur_);
    cur_ += bytes;
    left_ -= bytes;
    return r;
  }

 private:
  std::mutex mu_;
  std::vector<std::unique_ptr<unsigned char[]>> chunks_;
  unsigned char* cur_ = nullptr;
  size_t left_ = 0;
};

struct TBranch {
  double reward = 0.0, upper = 0.0, lower = 0.0;  // r(b,a), u(b,a), l(b,a)
  uint32_t visits = 0;                            // N(b,a)
  uint32_t first = 0, count = 0;                  // children: rec[first, first + count)
};

struct TNode {
  TChild* rec = nullptr;  // this node's bounds
  TNode* parent = nullptr;
  int32_t action_in = -1;
  uint32_t child_in = 0;
  uint32_t depth = 0;
  uint32_t visits = 0;     // N(b), under mu
  despot_node handle = 0;  // backend arena once expanded
  enum State { kLeaf, kPending, kExpanded } state = kLeaf;  // under mu
  std::vector<TBranch> branches;                            // [A] once expanded, under mu
  TChild* children = nullptr;                               // all children, action-major (arena)
  uint32_t n_children = 0;
  std::mutex mu;
};

struct Pending {
  TNode* leaf;
  std::vector<TNode*> path;
  std::atomic<uint32_t>* inflight;
};

// The batcher's output arrays, grown on demand and reused across batches.
struct OutBuf {
  size_t L = 0, LA = 0, C = 0, OW = 0;
  std::unique_ptr<despot_node[]> node;
  std::unique_ptr<uint32_t[]> n_scen, child_begin, child_count, child_first, child_obs;
  std::unique_ptr<float[]> weight, ar, au, al, cw, cu, cl;
  void reserve(size_t l, size_t la, size_t c, size_t ow) {
    if (l > L) {
      L = l;
      node.reset(new despot_node[l]);
      n_scen.reset(new uint32_t[l]);
      weight.reset(new float[l]);
    }
    if (la > LA) {
      LA = la;
      child_begin.reset(new uint32_t[la + 1]);
      ar.reset(new float[la]);
      au.reset(new float[la]);
      al.reset(new float[la]);
    }
    if (c > C || ow != OW) {
      C = std::max(c, (size_t)1);
      OW = ow;
      child_count.reset(new uint32_t[C]);
      child_first.reset(new uint32_t[C]);
      child_obs.reset(new uint32_t[C * ow]);
      cw.reset(new float[C]);
      cu.reset(new float[C]);
      cl.reset(new float[C]);
    }
  }
};

struct Search {
  const despot_search_problem& P;
  const despot_search_config& C;
  std::deque<TNode> nodes;  // full nodes (descended into); stable addresses
  std::mutex nodes_mu;
  TChild root_rec;
  TNode* root = nullptr;
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> trials{0}, batches{0}, expanded{0}, steps{0}, records{1};
  std::atomic<uint64_t> done_batches{0};   // batches completed (workers wait on it)
  std::atomic<uint32_t> inflight_total{0};  // leaves queued or being expanded
  std::atomic<uint32_t> max_depth{0};
  std::mutex qmu;
  std::condition_variable qcv;  // batcher wake-up
  std::condition_variable dcv;  // a worker's trial finished expanding
  std::deque<Pending> queue;
  bool workers_done = false;
  uint32_t n_workers = 1;
  uint32_t blocked = 0;  // workers waiting for their in-flight trials (under qmu)
  std::atomic<int> error{0};
  std::string error_msg;
  ChildArena arena;  // the child records of every node (all batchers)
  // batcher time split in ns (DESPOT_SEARCH_TRACE)
  std::atomic<uint64_t> t_call{0}, t_children{0}, t_backup{0}, t_alloc{0}, t_branch{0}, t_rec{0};
  static uint64_t ns(std::chrono::steady_clock::duration d) {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(d).count();
  }

  Search(const despot_search_problem& p, const despot_search_config& c) : P(p), C(c) {}

  TNode* new_node() {
    std::lock_guard<std::mutex> g(nodes_mu);
    nodes.emplace_back();
    return &nodes.back();
  }
  double root_gap() const { return root_rec.upper.load() - root_rec.lower.load(); }

  // Eq. 4 one level: recompute node b's branch a (every branch when a < 0)
  // from its children, then b's bounds as the max over its branches (clamped
  // by the initial bounds).  A trial changes only the children below the
  // branch it took, so the backup along its path recomputes that branch
  // alone: O(A + |children of a|) per node instead of O(all children).
  void backup_node(TNode* b, int32_t a) {
    std::lock_guard<std::mutex> g(b->mu);
    if (b->state != TNode::kExpanded) return;
    const double W = b->rec->weight;
    double bu = -std::numeric_limits<double>::infinity(), bl = bu;
    for (uint32_t k = 0; k < b->branches.size(); ++k) {
      TBranch& br = b->branches[k];
      if (br.count && (a < 0 || (uint32_t)a == k)) {
        double su = 0.0, sl = 0.0;
        for (uint32_t c = br.first; c < br.first + br.count; ++c) {
          const TChild& ch = b->children[c];
          const double f = ch.weight / W;
          su += f * ch.upper.load(std::memory_order_relaxed);
          sl += f * ch.lower.load(std::memory_order_relaxed);
        }
        br.upper = br.reward + P.gamma * su;
        br.lower = br.reward + P.gamma * sl;
      }
      bu = std::max(bu, br.upper);
      bl = std::max(bl, br.lower);
    }
    b->rec->upper.store(std::min(b->rec->u0, bu));
    b->rec->lower.store(std::max(b->rec->l0, bl));
  }
  void backup(const std::vector<TNode*>& path) {
    for (size_t i = path.size(); i-- > 0;) backup_node(path[i], i + 1 < path.size() ? path[i + 1]->action_in : -1);
  }
  static void release_markers(const std::vector<TNode*>& path) {
    for (size_t i = 1; i < path.size(); ++i) path[i]->rec->active.fetch_sub(1);
  }

  // ---------------------------------------------------------------- batcher
  int expand(std::vector<Pending>& batch, OutBuf& ob) {
    const uint32_t L = (uint32_t)batch.size(), A = P.num_actions, OW = P.obs_words;
    std::vector<despot_leaf> leaves(L);
    uint64_t cap = 0;
    for (uint32_t i = 0; i < L; ++i) {
      TNode* b = batch[i].leaf;
      if (b == root) leaves[i] = despot_leaf{P.root, -1, 0, P.root_depth, 0};
      else leaves[i] = despot_leaf{b->parent->handle, b->action_in, b->child_in, b->depth, 0};
      const uint32_t n = b->rec->n_scen ? b->rec->n_scen : 1;
      cap += (uint64_t)A * (P.obs_slots ? std::min(n, P.obs_slots) : n);
    }
    if (cap > 0xFFFFFFFFull) return DESPOT_ECAPACITY;
    // output arrays: the batcher's own grow-only buffers (no per-batch
    // allocation or zero fill; the backend writes every element we read)
    ob.reserve(L, (size_t)L * A, cap, OW);
    despot_node* hnode = ob.node.get();
    uint32_t *n_scen = ob.n_scen.get(), *child_begin = ob.child_begin.get(), *child_count = ob.child_count.get(),
             *child_first = ob.child_first.get(), *child_obs = ob.child_obs.get();
    float *weight = ob.weight.get(), *ar = ob.ar.get(), *au = ob.au.get(), *al = ob.al.get(), *cw = ob.cw.get(),
          *cu = ob.cu.get(), *cl = ob.cl.get();
    despot_expansion out;
    memset(&out, 0, sizeof out);
    out.node = hnode;
    out.n_scen = n_scen;
    out.weight = weight;
    out.act_reward = ar;
    out.act_upper = au;
    out.act_lower = al;
    out.child_begin = child_begin;
    out.child_capacity = (uint32_t)cap;
    out.child_count = child_count;
    out.child_first = child_first;
    out.child_weight = cw;
    out.child_upper = cu;
    out.child_lower = cl;
    out.child_obs = child_obs;
    const auto tc0 = std::chrono::steady_clock::now();
    const int rc = P.expand(P.ctx, leaves.data(), L, &out);
    const auto tc1 = std::chrono::steady_clock::now();
    t_call += ns(tc1 - tc0);
    if (rc != DESPOT_OK) return rc;
    batches.fetch_add(1);
    steps.fetch_add(out.scenario_steps);
    for (uint32_t i = 0; i < L; ++i) {
      TNode* b = batch[i].leaf;
      const uint32_t c0 = child_begin[(size_t)i * A], c1 = child_begin[(size_t)i * A + A];
      const auto ta = std::chrono::steady_clock::now();
      TChild* ch = arena.alloc(c1 - c0);
      if (!ch) return DESPOT_ENOMEM;
      std::vector<TBranch> br(A);
      const auto tb = std::chrono::steady_clock::now();
      t_alloc += ns(tb - ta);
      const bool at_horizon = b->depth + 1 >= P.max_depth;
      for (uint32_t a = 0; a < A; ++a) {
        const size_t la = (size_t)i * A + a;
        br[a].reward = ar[la];
        br[a].upper = au[la];
        br[a].lower = al[la];
        br[a].first = child_begin[la] - c0;
        br[a].count = child_begin[la + 1] - child_begin[la];
      }
      const auto tcc = std::chrono::steady_clock::now();
      t_branch += ns(tcc - tb);
      for (uint32_t c = c0; c < c1; ++c)  // at depth D the value is exactly the tail-based l0: gap 0
        new (&ch[c - c0]) TChild(cw[c], child_count[c], at_horizon ? cl[c] : cu[c], cl[c]);
      records.fetch_add(c1 - c0);
      const auto td = std::chrono::steady_clock::now();
      t_rec += ns(td - tcc);
      {
        std::lock_guard<std::mutex> g(b->mu);
        b->handle = hnode[i];
        if (b->rec->n_scen == 0) b->rec->n_scen = n_scen[i];
        if (b->rec->weight == 0.0f) b->rec->weight = weight[i];
        b->branches = std::move(br);
        b->children = ch;
        b->n_children = c1 - c0;
        b->state = TNode::kExpanded;
      }
      expanded.fetch_add(1);
      uint32_t d = b->depth + 1, m = max_depth.load();
      while (d > m && !max_depth.compare_exchange_weak(m, d)) {
      }
    }
    const auto tc2 = std::chrono::steady_clock::now();
    t_children += ns(tc2 - tc1);
    for (Pending& p : batch) {
      backup(p.path);
      release_markers(p.path);
      if (p.inflight) p.inflight->fetch_sub(1);
      if (p.inflight) inflight_total.fetch_sub(1);
    }
    t_backup += ns(std::chrono::steady_clock::now() - tc2);
    return DESPOT_OK;
  }

  // Batchers take turns: while one waits for its expansion call the other
  // creates the children and backs up the previous batch (the host work and
  // the device work of consecutive batches overlap).
  void batcher() {
    OutBuf ob;
    const uint32_t max_batch = std::max<uint32_t>(1, C.max_batch);
    for (;;) {
      std::vector<Pending> batch;
      {
        std::unique_lock<std::mutex> lk(qmu);
        qcv.wait(lk, [&] { return !queue.empty() || workers_done; });
        if (queue.empty() && workers_done) break;
        // wait for more leaves only while some worker can still produce one
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::microseconds(C.batch_wait_us);
        while (queue.size() < max_batch && blocked < n_workers && !workers_done && !stop.load()) {
          if (qcv.wait_until(lk, deadline) == std::cv_status::timeout) break;
        }
        while (!queue.empty() && batch.size() < max_batch) {
          batch.push_back(std::move(queue.front()));
          queue.pop_front();
        }
      }
      if (batch.empty()) continue;  // the other batcher took the leaves while this one waited
      const int rc = error.load() ? error.load() : expand(batch, ob);
      if (rc != DESPOT_OK) {
        int expected = 0;
        if (error.compare_exchange_strong(expected, rc)) error_msg = despot_last_error();
        stop.store(true);
        for (Pending& p : batch) {  // give the leaves back, release the markers
          {
            std::lock_guard<std::mutex> g(p.leaf->mu);
            p.leaf->state = TNode::kLeaf;
          }
          release_markers(p.path);
          if (p.inflight) p.inflight->fetch_sub(1);
          if (p.inflight) inflight_total.fetch_sub(1);
        }
      }
      {
        std::lock_guard<std::mutex> g(qmu);  // pairs with the workers' dcv wait
        done_batches.fetch_add(1);
      }
      dcv.notify_all();
    }
  }

  // ---------------------------------------------------------------- workers
  // Eq. 7: u(b,a) + c_a sqrt(log(|Phi_b| N(b)) / (|Phi_b| N(b,a)))
  uint32_t choose_action(TNode* b) const {
    const double phi = (double)std::max<uint32_t>(1, b->rec->n_scen);
    const double nb = phi * (double)b->visits;
    uint32_t best = 0;
    double bv = -std::numeric_limits<double>::infinity();
    for (uint32_t a = 0; a < b->branches.size(); ++a) {
      const TBranch& br = b->branches[a];
      double v;
      if (C.c_a > 0.0 && br.visits == 0) v = std::numeric_limits<double>::infinity();
      else if (C.c_a > 0.0 && b->visits > 0)
        v = br.upper + C.c_a * std::sqrt(std::log(nb) / (phi * (double)br.visits));
      else v = br.upper;
      if (v > bv) {
        bv = v;
        best = a;
      }
    }
    return best;
  }

  void worker() {
    std::atomic<uint32_t> inflight{0};
    uint32_t failed = 0;  // consecutive trials that found no leaf
    const uint32_t max_inflight = std::max<uint32_t>(1, C.max_inflight);
    while (!stop.load()) {
      if (inflight.load() >= max_inflight) {
        std::unique_lock<std::mutex> lk(qmu);
        ++blocked;
        qcv.notify_one();  // the batcher need not wait for this worker's next leaf
        dcv.wait(lk, [&] { return inflight.load() < max_inflight || stop.load(); });
        --blocked;
        continue;
      }
      if (C.max_trials && trials.fetch_add(1) >= C.max_trials) {
        stop.store(true);
        break;
      }
      if (!C.max_trials) trials.fetch_add(1);
      std::vector<TNode*> path{root};
      TNode* b = root;
      TNode* leaf = nullptr;
      for (;;) {
        std::unique_lock<std::mutex> lk(b->mu);
        if (b->state == TNode::kLeaf) {
          if (b->depth < P.max_depth) {
            b->state = TNode::kPending;  // claimed: this trial expands it
            leaf = b;
          }
          break;
        }
        if (b->state == TNode::kPending) break;  // another trial is expanding it
        const uint32_t a = choose_action(b);
        b->visits += 1;  // counts bumped on entry
        TBranch& br = b->branches[a];
        br.visits += 1;
        const double gap0 = root_gap();
        TChild* next = nullptr;
        uint32_t next_k = 0;
        double best = 0.0;  // the trial ends unless some WEU > 0
        for (uint32_t k = br.first; k < br.first + br.count; ++k) {
          TChild& c = b->children[k];
          const double gap = c.upper.load(std::memory_order_relaxed) - c.lower.load(std::memory_order_relaxed);
          const double weu = gap - ((double)c.weight / root_rec.weight) * C.xi * gap0;  // Eq. 6
          const double aug = weu - (double)c.active.load() * C.c_o * gap0;              // Eq. 8
          if (aug > best) {
            best = aug;
            next = &c;
            next_k = k;
          }
        }
        if (!next) break;
        TNode* nd = next->node.load();
        if (!nd) {  // first descent into this child: give it a full node
          nd = new_node();
          nd->rec = next;
          nd->parent = b;
          nd->action_in = (int32_t)a;
          nd->child_in = next_k - br.first;
          nd->depth = b->depth + 1;
          next->node.store(nd);
        }
        // the virtual-loss marker (Eq. 8) goes up before the lock is released,
        // so a worker choosing under the same lock right after sees it
        next->active.fetch_add(1);
        lk.unlock();
        path.push_back(nd);
        b = nd;
      }
      if (leaf) {
        failed = 0;
        inflight.fetch_add(1);
        inflight_total.fetch_add(1);
        {
          std::lock_guard<std::mutex> g(qmu);
          queue.push_back(Pending{leaf, std::move(path), &inflight});
        }
        qcv.notify_one();
      } else {
        // no leaf (a pending node or every WEU <= 0): no bound changed, so
        // no backup.  After a second miss in a row the tree will not change
        // until a batch lands: wait for one instead of re-descending (the
        // re-descents would only contend for the node locks).
        release_markers(path);
        if (++failed >= 2 && inflight_total.load() > 0) {
          const uint64_t seen = done_batches.load();
          std::unique_lock<std::mutex> lk(qmu);
          ++blocked;
          qcv.notify_one();
          dcv.wait_for(lk, std::chrono::milliseconds(2),
                       [&] { return done_batches.load() != seen || stop.load(); });
          --blocked;
        }
      }
    }
    // wait for this worker's trials still in the batcher (inflight lives here)
    std::unique_lock<std::mutex> lk(qmu);
    ++blocked;
    qcv.notify_all();
    dcv.wait(lk, [&] { return inflight.load() == 0; });
  }

  // pre-order dump: every belief node (a child record with or without a full node)
  void dump_tree(despot_search_node* out, uint32_t cap, uint32_t& n) const {
    struct Item {
      const TChild* rec;
      const TNode* node;
      int32_t parent, action;
      uint32_t child, depth;
    };
    std::vector<Item> stack{{&root_rec, root, -1, -1, 0, root->depth}};
    while (!stack.empty() && n < cap) {
      const Item it = stack.back();
      stack.pop_back();
      despot_search_node& d = out[n];
      memset(&d, 0, sizeof d);
      d.parent = it.parent;
      d.action = it.action;
      d.child = it.child;
      d.depth = it.depth;
      d.n_scen = it.rec->n_scen;
      d.active = it.rec->active.load();
      d.weight = it.rec->weight;
      d.upper = (float)it.rec->upper.load();
      d.lower = (float)it.rec->lower.load();
      d.upper0 = (float)it.rec->u0;
      d.lower0 = (float)it.rec->l0;
      const TNode* b = it.node;
      if (b) {
        d.visits = b->visits;
        for (const TBranch& br : b->branches) d.branch_visits += br.visits;
        d.expanded = b->state == TNode::kExpanded;
      }
      const int32_t me = (int32_t)n++;
      if (b && b->state == TNode::kExpanded)
        for (int a = (int)b->branches.size() - 1; a >= 0; --a) {
          const TBranch& br = b->branches[a];
          for (int k = (int)br.count - 1; k >= 0; --k) {
            const TChild* c = &b->children[br.first + k];
            stack.push_back({c, c->node.load(), me, a, (uint32_t)k, it.depth + 1});
          }
        }
    }
  }
};

}  // namespace

extern "C" int despot_search(const despot_search_problem* P, const despot_search_config* C,
                             despot_search_result* R, despot_search_node* dump, uint32_t dump_capacity) {
  if (!P || !C || !R || !P->expand || P->num_actions == 0)
    return despot__set_error(DESPOT_EINVAL, "despot_search: null argument or no actions");
  if (P->root_depth >= P->max_depth) return despot__set_error(DESPOT_EINVAL, "despot_search: root depth >= D");
  if (P->root_scenarios == 0) return despot__set_error(DESPOT_EINVAL, "despot_search: root_scenarios == 0");
  const auto t0 = std::chrono::steady_clock::now();
  Search S(*P, *C);
  S.root = S.new_node();
  TNode* root = S.root;
  root->rec = &S.root_rec;
  root->depth = P->root_depth;
  S.root_rec.n_scen = P->root_scenarios;
  S.root_rec.weight = (float)P->root_weight;
  S.root_rec.u0 = P->root_upper;
  S.root_rec.l0 = P->root_lower;
  S.root_rec.upper.store(P->root_upper);
  S.root_rec.lower.store(P->root_lower);
  root->handle = P->root;
  // the root is expanded before any trial (and gives |Phi_b0| and W_b0)
  {
    std::vector<Pending> first{Pending{root, {root}, nullptr}};
    root->state = TNode::kPending;
    OutBuf ob;
    const int rc = S.expand(first, ob);
    if (rc != DESPOT_OK) return rc;
  }
  const uint32_t W = std::max<uint32_t>(1, C->workers);
  S.n_workers = W;
  // two batchers when several workers produce leaves (overlap of host and device work)
  const uint32_t n_batchers = W > 1 ? 2 : 1;
  std::vector<std::thread> batchers;
  for (uint32_t i = 0; i < n_batchers; ++i) batchers.emplace_back([&] { S.batcher(); });
  std::vector<std::thread> workers;
  for (uint32_t i = 0; i < W; ++i) workers.emplace_back([&] { S.worker(); });
  // anytime loop: time budget, trial budget, target gap
  for (;;) {
    if (S.stop.load()) break;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (C->time_budget_s > 0.0 && el >= C->time_budget_s) break;
    if (S.root_gap() <= C->target_gap) break;
    if (C->max_trials == 0 && C->time_budget_s <= 0.0) break;  // no budget at all
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  S.stop.store(true);
  {
    std::lock_guard<std::mutex> g(S.qmu);
  }
  S.dcv.notify_all();
  for (auto& t : workers) t.join();
  {
    std::lock_guard<std::mutex> g(S.qmu);
    S.workers_done = true;
  }
  S.qcv.notify_all();
  for (auto& t : batchers) t.join();
  // result
  R->action = 0;
  double best = -std::numeric_limits<double>::infinity();
  for (uint32_t a = 0; a < root->branches.size(); ++a)
    if (root->branches[a].lower > best) {
      best = root->branches[a].lower;
      R->action = (int32_t)a;
    }
  R->root_upper = (float)S.root_rec.upper.load();
  R->root_lower = (float)S.root_rec.lower.load();
  R->nodes = S.records.load();
  R->expanded = S.expanded.load();
  R->trials = std::min<uint64_t>(S.trials.load(), C->max_trials ? C->max_trials : S.trials.load());
  R->batches = S.batches.load();
  R->max_depth = S.max_depth.load();
  R->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  R->scenario_steps = S.steps.load();
  if (getenv("DESPOT_SEARCH_TRACE"))
    fprintf(stderr, "[despot search] %.3f s: batchers in the expansion call %.3f s, creating children %.3f s, "
                    "backups %.3f s, %llu batches\n",
            R->seconds, 1e-9 * (double)S.t_call.load(), 1e-9 * (double)S.t_children.load(),
            1e-9 * (double)S.t_backup.load(), (unsigned long long)R->batches);
  if (getenv("DESPOT_SEARCH_TRACE"))
    fprintf(stderr, "[despot search]   children: alloc %.3f s, branches %.3f s, records %.3f s\n",
            1e-9 * (double)S.t_alloc.load(), 1e-9 * (double)S.t_branch.load(), 1e-9 * (double)S.t_rec.load());
  if (dump && dump_capacity) {
    uint32_t n = 0;
    S.dump_tree(dump, dump_capacity, n);
  }
  // release the backend arenas this search created (not the caller's root)
  if (P->release)
    for (TNode& b : S.nodes)
      if (&b != root && b.state == TNode::kExpanded && b.handle) P->release(P->ctx, b.handle);
  if (S.error.load()) return despot__set_error(S.error.load(), S.error_msg.c_str());
  return DESPOT_OK;
}

// ---------------------------------------------------------------------------
// despot_plan: the search on libdespot's GPU backend
// ---------------------------------------------------------------------------
namespace {
struct GpuCtx {
  despot_model* model;
  void* stream;
};
int gpu_expand(void* ctx, const despot_leaf* leaves, uint32_t L, despot_expansion* out) {
  GpuCtx* g = static_cast<GpuCtx*>(ctx);
  out->flags = 0;  // host outputs
  return despot_expand_batch(g->model, leaves, L, out, g->stream);
}
int gpu_release(void* ctx, despot_node n) { return despot_node_release(static_cast<GpuCtx*>(ctx)->model, n); }
}  // namespace

extern "C" int despot_plan(despot_model* model, despot_node root, const despot_search_config* config,
                           despot_search_result* result, void* stream) {
  if (!model || !config || !result) return DESPOT_EINVAL;
  despot_model_info info;
  int rc = despot_model_info_get(model, &info);
  if (rc) return rc;
  uint32_t n = 0, depth = 0;
  if ((rc = despot_node_info(model, root, &n, &depth))) return rc;
  float u0 = 0.0f, l0 = 0.0f;
  if ((rc = despot_rollout_bounds(model, root, &u0, &l0, nullptr, nullptr, stream))) return rc;
  GpuCtx ctx{model, stream};
  despot_search_problem P;
  memset(&P, 0, sizeof P);
  P.num_actions = info.num_actions;
  P.obs_words = info.obs_words;
  P.obs_slots = info.obs_slots;
  P.max_depth = info.max_depth;
  P.gamma = info.gamma;
  P.root = root;
  P.root_depth = depth;
  P.root_scenarios = n;  // this device's scenarios (the search is single-GPU)
  P.root_weight = 0.0;
  P.root_upper = u0;
  P.root_lower = l0;
  P.expand = gpu_expand;
  P.release = gpu_release;
  P.ctx = &ctx;
  return despot_search(&P, config, result, nullptr, 0);
}
