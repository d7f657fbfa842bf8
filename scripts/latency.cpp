// latency.cpp -- per-call latency of despot_expand_batch from C (no Python):
// RockSample(7,8), K = 100, the root leaf (BASELINE config 1), host outputs
// and device outputs, on a non-blocking stream.  Build + run (GPU box):
//   g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_1802_06215_b200 -ldespot -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency && /tmp/latency
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "despot.h"

#define OK(x)                                                                 \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_) {                                                                \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, despot_last_error());        \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  const char* params =
      "n=7 robots=1 D=20 gamma=0.95 rocks=2:0,0:1,3:1,6:3,2:4,3:4,5:5,1:6 starts=0:3";
  despot_model* m = nullptr;
  OK(despot_model_load("rocksample", params, nullptr, &m));
  const uint32_t K = 100, A = 13;
  std::vector<uint32_t> st(2 * K);
  std::vector<float> w(K, 1.0f / K);
  std::mt19937 rng(1001);
  for (uint32_t i = 0; i < K; ++i) {
    st[i] = rng() & 0xFFu;
    st[K + i] = 3 * 7 + 0;
  }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  despot_node root;
  OK(despot_belief_load(m, st.data(), w.data(), K, 1001, s, &root));
  despot_leaf leaf{root, -1, 0, 0, 0};
  const uint32_t C = A * 4;
  // host outputs (pinned) and device outputs; mode 2 = device outputs
  // through the two-phase form (begin/end: separate K3, no fusion); modes 3, 4
  // = a prepared batch (despot_batch_prepare: one CUDA graph per run) with
  // host / device outputs; mode 5 = a resident prepared batch
  // (DESPOT_X_RESIDENT: the graph is K2 alone), device outputs
  for (int mode = 0; mode < 6; ++mode) {
    const int dev = mode == 1 || mode == 2 || mode == 4 || mode == 5;
    despot_expansion out;
    memset(&out, 0, sizeof out);
    despot_node node;
    void* buf = nullptr;
    const size_t bytes = 4 * (2 + 3 * A + A + 1 + 6 * C) + 64;
    if (dev) cudaMalloc(&buf, bytes);
    else cudaMallocHost(&buf, bytes);
    char* p = static_cast<char*>(buf);
    auto take = [&](size_t n) {
      char* q = p;
      p += (n + 15) & ~size_t(15);
      return q;
    };
    out.flags = (dev ? DESPOT_X_DEVICE_OUTPUTS : 0) | (mode == 5 ? DESPOT_X_RESIDENT : 0);
    out.node = &node;
    out.n_scen = (uint32_t*)take(4);
    out.weight = (float*)take(4);
    out.act_reward = (float*)take(4 * A);
    out.act_upper = (float*)take(4 * A);
    out.act_lower = (float*)take(4 * A);
    out.child_begin = (uint32_t*)take(4 * (A + 1));
    out.child_capacity = C;
    out.child_count = (uint32_t*)take(4 * C);
    out.child_first = (uint32_t*)take(4 * C);
    out.child_weight = (float*)take(4 * C);
    out.child_upper = (float*)take(4 * C);
    out.child_lower = (float*)take(4 * C);
    out.child_obs = (uint32_t*)take(4 * C);
    despot_prepared* prep = nullptr;
    if (mode >= 3) OK(despot_batch_prepare(m, &leaf, 1, &out, &prep));
    auto call = [&]() -> int {
      if (mode >= 3) return despot_batch_run(prep, &out, s);
      if (mode < 2) return despot_expand_batch(m, &leaf, 1, &out, s);
      despot_batch* b = nullptr;
      if (int rc = despot_expand_begin(m, &leaf, 1, out.flags, s, &b)) return rc;
      return despot_expand_end(b, &out, s);
    };
    for (int i = 0; i < 50; ++i) OK(call());
    const int N = argc > 1 ? atoi(argv[1]) : 2000;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) OK(call());
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / N;
    if (mode < 3) {
      out.flags |= DESPOT_X_TIMING;
      OK(call());
    }
    const char* name[] = {"host", "device", "device-two-phase", "host-prepared-graph", "device-prepared-graph",
                          "device-resident-graph"};
    printf("{\"outputs\": \"%s\", \"us_per_call\": %.2f, \"launches\": %u, \"scenario_steps\": %llu, \"phases_ms\": [%.4f, %.4f, %.4f, %.4f]}\n",
           name[mode], us, out.launches, (unsigned long long)out.scenario_steps, out.phase_ms[0], out.phase_ms[1],
           out.phase_ms[2], out.phase_ms[3]);
    if (prep) despot_batch_prepared_free(prep);
    if (dev) cudaFree(buf);
    else cudaFreeHost(buf);
  }
  despot_model_free(m);
  return 0;
}
