// engine.h — host-side engine of the B200 patched-forward path.
//
// The reference evaluates every (edge, item) patched pass as a full forward
// (DeltaLEngine::delta_l, proj/src/patching.cpp:227-239). This engine keeps
// the reference's semantics bit-for-bit but restructures the work for the
// GPU (SURVEY.md §7 phase 5):
//
//  * policy-major order: edges are grouped by source u (policy_for_edge,
//    pahq.cpp:198-209); the masked clean baseline under p_u is recomputed
//    only from stage(u) (the prefix equals the base-policy run);
//  * suffix recompute: a patch on u->v changes only v and the nodes whose
//    inputs depend on it; everything else is read from the baseline;
//  * receiver inputs are folds over a trie of receivers' present-source
//    lists, so prefixes shared by several receivers (all of them in
//    iteration 1) are summed once, in the reference's ascending order;
//  * all passes of a source group run together, stage by stage, as batched
//    kernels over [edges x items x seq] rows.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <stdexcept>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cqg.h"
#include "kernels.h"

namespace cqg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum NodeKind { kEmbed = 0, kHead = 1, kMlp = 2, kUnembed = 3 };

// ComputationalGraph (model.cpp:166-246)
struct Graph {
  int L = 0, H = 0, D = 0, dk = 0, V = 0, S = 0, mlp = 0;
  int N = 0, E = 0, n_stages = 0, unembed = 0;
  std::vector<int> kind, layer, head, stage;
  std::vector<int> esrc, edst;
  // receivers: one per node except the embed; a head has 3 (q, k, v inputs)
  // under qkv_split (extension, cqg.h)
  int split = 0, NR = 0;
  std::vector<int> recv_node, recv_comp, node_recv, erecv;
  std::vector<std::vector<int>> in_edges;     // per receiver, ascending src
  std::vector<std::vector<int>> stage_nodes;  // ascending index
  int recv(int n, int c) const { return node_recv[n] + (split && kind[n] == kHead ? c : 0); }
  int n_recv(int n) const { return n == 0 ? 0 : (split && kind[n] == kHead ? 3 : 1); }
  explicit Graph(const cqg_config& c);
  int n_mats() const { return 5 + L * (6 + (mlp ? 4 : 0)); }
  int mat(int which, int l) const;  // which: 0 w_e 1 w_pos 2 ln1g 3 ln1b 4 wq 5 wk 6 wv 7 wo
                                    // 8 ln2g 9 ln2b 10 win 11 wout 12 lnfg 13 lnfb 14 wu
  std::vector<int> sweep_order(const std::vector<uint8_t>& mask) const;
};

// PrecisionPolicy (precision_policy.hpp:36-58, model.cpp:52-71)
struct Policy {
  int att = 0, mlp = 1, emb = 2, unemb = 2, mode = 0;
  int th_l = -1, th_h = -1, tm = -1;
  static Policy from(const cqg_policy& p);
  int precision_of(const Graph& g, int node) const;
  int wo_precision(int layer) const { return (th_l >= 0 && th_l == layer) ? 2 : att; }
  bool operator==(const Policy& o) const;
  bool operator<(const Policy& o) const;
};
Policy policy_for_edge(const Graph& g, int e, const Policy& base);  // pahq.cpp:198-209

// Trie over receivers' present-source lists (the structure of sum_inputs).
struct Trie {
  std::vector<int> parent, src;                 // node 0 = root (value 0)
  std::vector<int> rec_in;                      // per receiver (root if no inputs)
  std::vector<std::vector<int>> by_stage;       // trie nodes per stage(src), parents first
  void build(const Graph& g, const uint8_t* mask);
  int size() const { return (int)parent.size(); }
};

struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DeviceBuf() = default;
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
  ~DeviceBuf();
  void ensure(size_t n);  // grow-only
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct Engine;
std::unique_ptr<Engine> make_engine(const cqg_config& cfg, const float* const* mats, int device);

}  // namespace cqg
