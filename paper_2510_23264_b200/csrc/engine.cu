// engine.cu — host orchestration of the patched-forward hot path + C ABI.
// See engine.h for the execution strategy; SURVEY.md §8 for the mapping to
// the reference (proj/src/patching.cpp, model.cpp, acdc.cpp).
#include "engine.h"

#include <dlfcn.h>
#include <nccl.h>

#include <tuple>

#include "gemm_tc.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>

namespace cqg {

static thread_local std::string g_err;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw Error(e_ == cudaErrorMemoryAllocation ? 3 : 2,                                      \
                  std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ") at " +      \
                      __FILE__ + ":" + std::to_string(__LINE__));                               \
  } while (0)

// NCCL is resolved at run time (dlopen of libnccl.so.2) instead of being
// linked: a process that already loaded torch's bundled NCCL reuses that copy,
// and loading libcqg.so never pins an NCCL version torch would then clash with.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!api.AllReduce) throw Error(2, "NCCL (libnccl.so.2) not available");
  return api;
}

#define NK(x)                                                                                  \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess)                                                                     \
      throw Error(2, std::string("NCCL error: ") + cqg::nccl().GetErrorString(r_));                 \
  } while (0)

// ===========================================================================
// Graph / policy / trie
// ===========================================================================
static int node_stage(int kind, int layer, int L) {
  switch (kind) {
    case kEmbed: return 0;
    case kHead: return 1 + 2 * layer;
    case kMlp: return 2 + 2 * layer;
    default: return 1 + 2 * L;
  }
}

Graph::Graph(const cqg_config& c) {
  // ModelConfig::validate (model.cpp:144-155), batch fixed to 1
  if (c.n_layers < 1) throw Error(1, "ModelConfig: n_layers must be >= 1");
  if (c.n_heads < 1) throw Error(1, "ModelConfig: n_heads must be >= 1");
  if (c.d_model < 1 || c.d_k < 1) throw Error(1, "ModelConfig: d_model and d_k must be >= 1");
  if (c.n_heads * c.d_k != c.d_model) throw Error(1, "ModelConfig: n_heads * d_k must equal d_model");
  if (c.vocab < 2) throw Error(1, "ModelConfig: vocab must be >= 2");
  if (c.seq_len < 1) throw Error(1, "ModelConfig: seq_len must be >= 1");
  if (c.has_mlp > 1) throw Error(1, "ModelConfig: has_mlp must be 0 or 1");
  L = (int)c.n_layers, H = (int)c.n_heads, D = (int)c.d_model, dk = (int)c.d_k;
  V = (int)c.vocab, S = (int)c.seq_len, mlp = (int)c.has_mlp;
  // nodes (model.cpp:184-190)
  auto add = [&](int k, int l, int h) {
    kind.push_back(k), layer.push_back(l), head.push_back(h), stage.push_back(node_stage(k, l, L));
  };
  add(kEmbed, -1, -1);
  for (int l = 0; l < L; ++l) {
    for (int h = 0; h < H; ++h) add(kHead, l, h);
    if (mlp) add(kMlp, l, -1);
  }
  add(kUnembed, -1, -1);
  N = (int)kind.size();
  unembed = N - 1;
  n_stages = 2 + 2 * L;
  stage_nodes.resize(n_stages);
  for (int i = 0; i < N; ++i) stage_nodes[stage[i]].push_back(i);
  // receivers: node order, then component (q, k, v of a split head)
  if (c.qkv_split > 1) throw Error(1, "ModelConfig: qkv_split must be 0 or 1");
  split = (int)c.qkv_split;
  node_recv.assign(N, -1);
  for (int j = 1; j < N; ++j) {
    node_recv[j] = (int)recv_node.size();
    for (int q = 0; q < n_recv(j); ++q) recv_node.push_back(j), recv_comp.push_back(q);
  }
  NR = (int)recv_node.size();
  // edges (model.cpp:192-201): for receiver r asc, for i < node(r) asc
  in_edges.resize(NR);
  for (int r = 0; r < NR; ++r) {
    const int j = recv_node[r];
    for (int i = 0; i < j; ++i) {
      if (stage[i] >= stage[j]) continue;
      in_edges[r].push_back((int)esrc.size());
      esrc.push_back(i);
      edst.push_back(j);
      erecv.push_back(r);
    }
  }
  E = (int)esrc.size();
}

int Graph::mat(int which, int l) const {
  const int per = 6 + (mlp ? 4 : 0);
  switch (which) {
    case 0: return 0;
    case 1: return 1;
    case 12: return 2 + L * per;
    case 13: return 3 + L * per;
    case 14: return 4 + L * per;
    default: return 2 + l * per + (which - 2);
  }
}

std::vector<int> Graph::sweep_order(const std::vector<uint8_t>& mask) const {
  // model.cpp:238-246
  std::vector<int> o;
  for (int j = NR - 1; j >= 0; --j)  // receivers desc (= dst desc on the reference's graph)
    for (auto it = in_edges[j].rbegin(); it != in_edges[j].rend(); ++it)
      if (mask[*it]) o.push_back(*it);
  return o;
}

Policy Policy::from(const cqg_policy& p) {
  Policy q;
  q.att = p.attention_default, q.mlp = p.mlp_default, q.emb = p.embed_precision;
  q.unemb = p.unembed_precision, q.mode = p.low_mode;
  q.th_l = p.target_head_layer, q.th_h = p.target_head_layer >= 0 ? p.target_head_head : -1;
  q.tm = p.target_mlp;
  for (int v : {q.att, q.mlp, q.emb, q.unemb})
    if (v < 0 || v > 2) throw Error(1, "policy: precision must be 0 (P8), 1 (P16) or 2 (P32)");
  if (q.mode < 0 || q.mode > 2)
    throw Error(1, "policy: low_mode must be 0 (E4m3), 1 (Rtn4) or 2 (INT8, extension)");
  return q;
}

int Policy::precision_of(const Graph& g, int n) const {
  switch (g.kind[n]) {
    case kEmbed: return emb;
    case kUnembed: return unemb;
    case kHead: return (th_l >= 0 && th_l == g.layer[n] && th_h == g.head[n]) ? 2 : att;
    default: return (tm >= 0 && tm == g.layer[n]) ? 2 : mlp;
  }
}

bool Policy::operator==(const Policy& o) const {
  return att == o.att && mlp == o.mlp && emb == o.emb && unemb == o.unemb && mode == o.mode &&
         th_l == o.th_l && th_h == o.th_h && tm == o.tm;
}
bool Policy::operator<(const Policy& o) const {
  auto t = [](const Policy& p) {
    return std::vector<int>{p.att, p.mlp, p.emb, p.unemb, p.mode, p.th_l, p.th_h, p.tm};
  };
  return t(*this) < t(o);
}

Policy policy_for_edge(const Graph& g, int e, const Policy& base) {
  Policy p = base;
  p.th_l = p.th_h = p.tm = -1;
  const int s = g.esrc[e];
  if (g.kind[s] == kHead) p.th_l = g.layer[s], p.th_h = g.head[s];
  if (g.kind[s] == kMlp) p.tm = g.layer[s];
  return p;
}

void Trie::build(const Graph& g, const uint8_t* mask) {
  parent.assign(1, -1);
  src.assign(1, -1);
  rec_in.assign(g.NR, 0);
  std::map<std::pair<int, int>, int> child;
  for (int w = 0; w < g.NR; ++w) {
    int cur = 0;
    for (int e : g.in_edges[w]) {
      if (mask && !mask[e]) continue;
      const int s = g.esrc[e];
      auto it = child.find({cur, s});
      if (it == child.end()) {
        const int id = (int)parent.size();
        parent.push_back(cur);
        src.push_back(s);
        child[{cur, s}] = id;
        cur = id;
      } else {
        cur = it->second;
      }
    }
    rec_in[w] = cur;
  }
  by_stage.assign(g.n_stages, {});
  for (int t = 1; t < size(); ++t) by_stage[g.stage[src[t]]].push_back(t);
  for (auto& v : by_stage)
    std::sort(v.begin(), v.end(), [&](int a, int b) { return src[a] != src[b] ? src[a] < src[b] : a < b; });
}

// ===========================================================================
// device buffers
// ===========================================================================
DeviceBuf::~DeviceBuf() {
  if (p) cudaFree(p);
}

void DeviceBuf::ensure(size_t n) {
  if (n <= bytes) return;
  if (p) {
    cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  n = (n + 255) & ~size_t(255);
  CK(cudaMalloc(&p, n));
  bytes = n;
}

// ===========================================================================
// Engine
// ===========================================================================
struct Run {  // one evaluation context (a baseline) over nb items
  int nb = 0;
  size_t seg = 0;  // floats per node activation
  DeviceBuf out, trie, logits, lse, prob;  // prob: [nb][V] exp(lp) of the last rows (KL)
  DeviceBuf psum;                           // [nb] sum_v exp(lp_v) (fused unembed + KL)
  DeviceBuf xbp, ebp;                       // logits / exp(lp) zero-padded to 128-column pitch
  std::vector<int8_t> otype;                // OutType of each node's output in `out`
  float* o(int n) const { return out.as<float>() + (size_t)n * seg; }
  float* t(int n) const { return trie.as<float>() + (size_t)n * seg; }
};

struct HeadIO {
  const float* in;  // the head's input (its q input under qkv_split)
  int head;
  float* out;
  int otype;  // OutType the output is stored as
  const float* in_k = nullptr, *in_v = nullptr;  // qkv_split: k / v inputs (null: = in)
  const float* input(int c) const { return c == 1 && in_k ? in_k : (c == 2 && in_v ? in_v : in); }
};
struct SegIO {
  const float* in;
  float* out;
  int otype;
};

struct Engine {
  Graph g;
  int device = 0;
  cudaStream_t st = nullptr;
  std::vector<std::unique_ptr<DeviceBuf>> master;
  std::vector<int64_t> msize;
  std::map<int, std::vector<std::unique_ptr<DeviceBuf>>> img;  // 0 e4m3, 1 bf16, 2 rtn4, 3 int8
  // dataset
  int B = 0, item_off = 0, item_total = 0, metric = 0;
  DeviceBuf d_clean, d_corrupt, d_ans, d_dis;
  std::vector<int> h_ans, h_dis;
  // scratch
  std::map<std::string, std::unique_ptr<DeviceBuf>> pool;
  DeviceBuf zero;
  // job staging
  char* h_stage = nullptr;
  size_t stage_cap = 0, stage_off = 0;
  DeviceBuf d_stage;
  // caches
  Run base_run;                    // masked baseline (per call)
  Run patch_run;                   // full-graph run that supplies patch values
  bool patch_valid = false;
  Policy patch_policy;
  int patch_tokens = -1;           // 0 clean, 1 corrupt
  // per source node (per-edge policies). Invalidation bumps target_gen
  // instead of freeing: the buffers are reused (cudaFree / cudaMalloc of ~150
  // buffers per new dataset cost ~1 s).
  struct TargetVal {
    DeviceBuf buf;
    uint64_t gen = 0;
  };
  std::map<int, TargetVal> target_cache;
  std::map<const float*, std::unique_ptr<DeviceBuf>> wu_pad;  // padded unembed images
  uint64_t target_gen = 1;
  Trie full;
  // comm
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // stats/options
  cqg_stats stats{};
  int64_t opt_exact = 0;
  int64_t opt_packed = 1;
  // BF16 fixups: chunked block kernel (1) or the per-tile kernel (0, default:
  // measured faster, DESIGN.md section 7 "tried")
  int64_t opt_fix_blk = 0;
  int64_t opt_fix_blk_min = 148;
  int64_t opt_kl_fused = 1;  // patched rows: unembed with the KL in its epilogue (no logits)  // ... for launches with at least this many row-tile units
  int64_t opt_fix_cpi = 0;
  int64_t opt_fix_dry = 0;
  int64_t opt_fix_g = 0;  // tile-fixup unit (0: by K, 1 tiles, 2 super-tiles)  // timing experiment (wrong results): fixups without chains  // store E4M3/BF16-rounded node outputs as their codes
  int64_t opt_mem_budget = 0;
  // 1: the patched passes' FP32 unembed on the tensor cores (6-term BF16
  // split) with the KL-level certificate and exact recomputation of flagged
  // rows (KL metric, loss mode). Off by default: on the GPT-2-small workload
  // the certificate rejects every row, because the reference's own FP32
  // logit rounding already moves per-edge KL by ~1e-5 relative (DESIGN.md
  // §4, profiles/r2_unembed_tc_study_gpt2s.json); 0 = exact SIMT logits.
  int64_t opt_unembed_tc = 0;
  int64_t opt_unembed_tol_e9 = 100000;  // certificate tolerance x 1e9 (1e-4 relative KL)

  Engine(const cqg_config& c) : g(c) {}
  ~Engine() {
    if (comm) nccl().CommDestroy(comm);
    if (h_stage) cudaFreeHost(h_stage);
    for (cudaEvent_t ev : stage_ev)
      if (ev) cudaEventDestroy(ev);
    if (st_pf) cudaStreamSynchronize(st_pf), cudaStreamDestroy(st_pf);
    if (st) cudaStreamDestroy(st);
  }

  // host threads for the per-edge plans: a few (the launching thread must
  // keep its core; OpenMP workers spin between regions)
  static int plan_threads() {
    static const int n = std::max(1, std::min(6, omp_get_num_procs() / 4));
    return n;
  }

  // ---- the next group's FP32 slices into L2 on the side stream (a6) ---------
  // HeadBundle (pahq.cpp:21-24, 93-165): the elevated head's W_Q/W_K/W_V
  // column slices (D rows x d_k) and its layer's W_O; an elevated MLP's
  // W_in / W_out. The embed's policy is the base: nothing to fetch.
  cudaStream_t st_pf = nullptr;
  int64_t opt_prefetch = 0;  // measured slower (a6): off by default
  void prefetch_source(int src) {
    if (!opt_prefetch || src < 0 || g.kind[src] == kEmbed || g.kind[src] == kUnembed) return;
    if (!st_pf) CK(cudaStreamCreateWithFlags(&st_pf, cudaStreamNonBlocking));
    PfJob j{};
    const int l = g.layer[src];
    if (g.kind[src] == kHead) {
      const int h = g.head[src];
      if ((g.dk * 4) % 16 == 0 && (g.D * 4) % 16 == 0)
        for (int c = 0; c < 3; ++c) j.col[c] = master[g.mat(4 + c, l)]->as<float>() + h * g.dk;
      j.rows = g.D, j.ld = g.D, j.cols = g.dk;
      j.blk[0] = master[g.mat(7, l)]->p, j.blk_bytes[0] = msize[g.mat(7, l)] * 4;
    } else {
      j.blk[0] = master[g.mat(10, l)]->p, j.blk_bytes[0] = msize[g.mat(10, l)] * 4;
      j.blk[1] = master[g.mat(11, l)]->p, j.blk_bytes[1] = msize[g.mat(11, l)] * 4;
    }
    launch_prefetch_l2(j, st_pf);
    launched();
  }

  size_t segf(int nb) const { return (size_t)nb * g.S * g.D; }

  float* scratch(const std::string& name, size_t floats) {
    auto& b = pool[name];
    if (!b) b = std::make_unique<DeviceBuf>();
    b->ensure(std::max<size_t>(floats, 1) * sizeof(float));
    return b->as<float>();
  }

  const float* zeros(size_t floats) {
    if (zero.bytes < floats * 4) {
      zero.ensure(floats * 4);
      CK(cudaMemsetAsync(zero.p, 0, zero.bytes, st));
    }
    return zero.as<float>();
  }

  // Job arrays travel through a pinned ring. reserve() must be called once per
  // launch with the total bytes of all its arrays so that no later upload of
  // the same launch can wrap (or grow) the ring under an earlier one.
  static size_t up_bytes(size_t n, size_t sz) { return ((std::max<size_t>(n, 1) * sz) + 15) & ~size_t(15); }

  // The staging ring (pinned host + device) of the launches' job lists, in two
  // halves: when one fills, an event marks the end of the work that reads it
  // and the other half is reused once its own event has completed (long
  // done in steady state), so the host never drains the GPU to recycle it.
  double host_blocked_ms = 0;  // host time waiting for the GPU to recycle staging (CQG_HOST_PROF)
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  bool stage_ev_set[2] = {false, false};
  int stage_half = 0;
  void reserve(size_t total) {
    if (2 * total > stage_cap) {
      CK(cudaStreamSynchronize(st));
      if (h_stage) cudaFreeHost(h_stage);
      stage_cap = std::max<size_t>({4 * total, stage_cap * 2, size_t(64) << 20});
      CK(cudaMallocHost(&h_stage, stage_cap));
      d_stage.ensure(stage_cap);
      stage_off = 0, stage_half = 0, stage_ev_set[0] = stage_ev_set[1] = false;
    }
    const size_t half = stage_cap / 2;
    if (stage_off + total > (size_t)(stage_half + 1) * half) {
      if (!stage_ev[0]) {
        CK(cudaEventCreateWithFlags(&stage_ev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&stage_ev[1], cudaEventDisableTiming));
      }
      CK(cudaEventRecord(stage_ev[stage_half], st));
      stage_ev_set[stage_half] = true;
      stage_half ^= 1;
      if (stage_ev_set[stage_half]) {
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaEventSynchronize(stage_ev[stage_half]));
        host_blocked_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      }
      stage_off = (size_t)stage_half * half;
    }
  }

  template <class T>
  T* upload(const std::vector<T>& v) {
    const size_t bytes = up_bytes(v.size(), sizeof(T));
    if (stage_off + bytes > stage_cap) throw Error(2, "internal: staging upload without reserve()");
    if (!v.empty()) std::memcpy(h_stage + stage_off, v.data(), v.size() * sizeof(T));
    CK(cudaMemcpyAsync(d_stage.as<char>() + stage_off, h_stage + stage_off, bytes,
                       cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += (int64_t)bytes;
    T* d = reinterpret_cast<T*>(d_stage.as<char>() + stage_off);
    stage_off += bytes;
    return d;
  }

  void launched(int n = 1) { stats.kernel_launches += n; }

  // ---- per-kernel-class device timing (option "profile") ---------------------
  struct KStat {
    double ms = 0, flops = 0, bytes = 0;
    int64_t launches = 0;
  };
  std::map<std::string, KStat> kprof;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  std::vector<Pending> pending;
  int64_t opt_profile = 0;
  std::string prof_tag;  // "base:" while a baseline run is being computed
  struct Prof {  // RAII region around one launch
    Engine* e;
    Pending p;
    Prof(Engine* en, const char* name, double flops = 0, double bytes = 0) : e(en) {
      e->launched();
      const std::string key = e->prof_tag + name;
      auto& k = e->kprof[key];
      k.launches++, k.flops += flops, k.bytes += bytes;
      if (!e->opt_profile) return;
      p.name = key, p.flops = flops, p.bytes = bytes;
      cudaEventCreate(&p.a);
      cudaEventCreate(&p.b);
      cudaEventRecord(p.a, e->st);
    }
    ~Prof() {
      if (!e->opt_profile) return;
      cudaEventRecord(p.b, e->st);
      e->pending.push_back(p);
    }
  };
  void collect_profile() {
    if (pending.empty()) return;
    cudaStreamSynchronize(st);
    for (auto& p : pending) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.a, p.b);
      kprof[p.name].ms += ms;
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    pending.clear();
  }

  // ---- weights -------------------------------------------------------------
  const float* W(int m, int prec, int mode) {
    if (prec == 2) return master[m]->as<float>();
    const int key = prec == 1 ? 1 : (mode == 0 ? 0 : mode == 1 ? 2 : 3);
    auto& v = img[key];
    if (v.empty()) v.resize(master.size());
    if (!v[m]) {
      v[m] = std::make_unique<DeviceBuf>();
      v[m]->ensure(msize[m] * 4);
      build_image(m, key, v[m]->as<float>());
    }
    return v[m]->as<float>();
  }

  int mat_kind(int m) const {  // returns which-index (see Graph::mat)
    const int per = 6 + (g.mlp ? 4 : 0);
    if (m == 0) return 0;
    if (m == 1) return 1;
    const int n = g.n_mats();
    if (m == n - 3) return 12;
    if (m == n - 2) return 13;
    if (m == n - 1) return 14;
    return 2 + (m - 2) % per;
  }

  void build_image(int m, int key, float* out) {
    const float* in = master[m]->as<float>();
    if (key == 0) launch_quantize(in, out, msize[m], 0, st);
    else if (key == 1) launch_quantize(in, out, msize[m], 1, st);
    else if (key == 3) {
      // INT8 per-channel (extension, oracle/cq_oracle.c int8_matrix): one group
      // per output column; W_O per (head, column) over the head's d_k rows;
      // vectors as one group
      const int w = mat_kind(m);
      const int64_t D = g.D;
      if (w == 7) {
        for (int h = 0; h < g.H; ++h)
          launch_rtn_groups(in + h * g.dk * D, out + h * g.dk * D, g.D, 1, g.dk, 1, g.D, 8, st, 127);
      } else if (w == 2 || w == 3 || w == 8 || w == 9 || w == 12 || w == 13) {
        launch_rtn_groups(in, out, 1, 0, 1, (int)msize[m], (int)msize[m], 8, st, 127);
      } else {
        const int C = w == 10 ? 4 * g.D : (w == 14 ? g.V : g.D);
        const int R = (int)(msize[m] / C);
        launch_rtn_groups(in, out, C, 1, R, 1, C, 8, st, 127);
      }
    } else {
      // quantize_rtn4_matrix (model.cpp:445-469)
      const int w = mat_kind(m);
      if (w == 4 || w == 5 || w == 6)
        launch_rtn_groups(in, out, g.H, g.dk, g.D, g.dk, g.D, 4, st);
      else if (w == 7)
        launch_rtn_groups(in, out, g.H, (int64_t)g.dk * g.D, g.dk, g.D, g.D, 4, st);
      else
        launch_rtn_groups(in, out, 1, 0, 1, (int)msize[m], (int)msize[m], 4, st);
    }
    launched();
  }

  // ---- launch helpers --------------------------------------------------------
  void fold(const std::vector<FoldOp>& ops, const std::vector<FoldProg>& progs, size_t elems) {
    if (progs.empty()) return;
    // algorithmic bytes: every operand read once and every stored value written once
    double words = 0;
    for (const FoldOp& o : ops)
      words += 1.0 + (o.a && o.a != CQG_REG_PREV ? 1.0 : 0.0) + (o.dst ? 1.0 : 0.0);
    reserve(up_bytes(ops.size(), sizeof(FoldOp)) + up_bytes(progs.size(), sizeof(FoldProg)));
    Prof pf(this, "fold", 0, words * 4.0 * (double)elems);
    launch_fold(upload(ops), upload(progs), (int)progs.size(), (int64_t)elems, st);
  }
  void ln(const std::vector<LnJob>& jobs, int l_gamma, int l_beta, int prec) {
    if (jobs.empty()) return;
    int mx = 0;
    double rows = 0;
    for (auto& j : jobs) mx = std::max(mx, j.rows), rows += j.rows;
    reserve(up_bytes(jobs.size(), sizeof(LnJob)));
    Prof pf(this, "layernorm", 0, rows * g.D * 4.0 * 3.0);
    launch_layernorm(upload(jobs), (int)jobs.size(), mx, master[l_gamma]->as<float>(),
                     master[l_beta]->as<float>(), g.D, prec, st);
  }
  void gemm(const std::vector<GemmJob>& jobs, const char* name = "gemm_exact") {
    if (jobs.empty()) return;
    std::vector<int> ts(jobs.size());
    int total = 0;
    double flops = 0;
    bool big = true, wide = g_exact_x2 != 0;
    for (const GemmJob& j : jobs) {
      big = big && j.M >= 128 && j.N >= 128;
      wide = wide && j.M <= 64 && j.N >= 256 && j.epi == 0;
    }
    for (size_t i = 0; i < jobs.size(); ++i) {
      ts[i] = total;
      total += wide  ? gemm_exact_wide_tiles(jobs[i].M, jobs[i].N)
               : big ? gemm_exact_big_tiles(jobs[i].M, jobs[i].N)
                     : gemm_exact_tiles(jobs[i].M, jobs[i].N);
      flops += 2.0 * jobs[i].M * (double)jobs[i].N * jobs[i].K;
    }
    reserve(up_bytes(jobs.size(), sizeof(GemmJob)) + up_bytes(ts.size(), sizeof(int)));
    Prof pf(this, name, flops, 0);
    if (wide) launch_gemm_exact_wide(upload(jobs), upload(ts), (int)jobs.size(), total, st);
    else if (big) launch_gemm_exact_big(upload(jobs), upload(ts), (int)jobs.size(), total, st);
    else launch_gemm_exact(upload(jobs), upload(ts), (int)jobs.size(), total, st);
  }
  // Rtn4 activation groups (one per item), in place
  // P8 under an RTN low mode: Rtn4 (reference) or INT8 (extension). Both run
  // the exact SIMT GEMMs on the FP32 grid values, with an RTN pass over every
  // tensor the reference quantizes (quantize_tensor, kernels.cpp:236-253).
  static bool rtn4(int prec, const Policy& P) { return prec == 0 && P.mode != 0; }
  // Jobs describe one item's [S][cols] tensor (group_off = the item stride).
  // Rtn4: one group per item tensor (the reference's quantize_span of the
  // whole tensor). INT8: one group per row (per-token scales), 8 bits, q <= 127.
  void rtn_act(const std::vector<RtnJob>& jobs, int nb, const Policy& P) {
    if (jobs.empty()) return;
    reserve(up_bytes(jobs.size(), sizeof(RtnJob)));
    if (P.mode == 2) {
      std::vector<RtnJob> rows(jobs);
      for (RtnJob& j : rows) {
        if (j.group_off != (int64_t)j.rows * j.ld) throw Error(2, "internal: INT8 row groups need item-major rows");
        j.group_off = j.ld, j.rows = 1;
      }
      Prof pf(this, "int8_act");
      launch_rtn_rows(upload(rows), (int)rows.size(), nb * g.S, 8, st, 127);
      return;
    }
    Prof pf(this, "rtn4_act");
    launch_rtn_act(upload(jobs), (int)jobs.size(), nb, 4, st);
  }
  void attn(const std::vector<AttnJob>& jobs, int nb) {
    if (jobs.empty()) return;
    reserve(up_bytes(jobs.size(), sizeof(AttnJob)));
    const double S = g.S;
    Prof pf(this, "attention", (double)jobs.size() * nb * 2.0 * g.dk * S * (S + 1), 0);
    launch_attention(upload(jobs), (int)jobs.size(), nb, g.S, g.dk, st);
  }

  void check_policy(const Policy& P) {
    if (P.th_l >= g.L || P.th_h >= g.H || (P.th_l >= 0 && P.th_h < 0))
      throw Error(1, "forward: target head out of range");
    if (P.tm >= 0 && (!g.mlp || P.tm >= g.L)) throw Error(1, "forward: target mlp out of range");
  }

  // ---- tensor-core GEMMs ------------------------------------------------------
  // Packed K-major weight images for the tensor cores (built once per layer
  // from the bit-exact FP32 grid images) and their per-row L2 norms.
  struct PackedB {
    DeviceBuf buf, norm;
    int rows = 0, cols = 0, elem = 0;
  };
  std::map<std::tuple<int, int, int>, std::unique_ptr<PackedB>> packed;
  DeviceBuf fix_mask, fix_tiles, tile_mark, fix_cnt, gelu_lut, fix_items, fix_n;

  // which: 0 QKV [3D x D], 1 W_O [D x D] (per-head K slices), 2 W_in^T [4D x D],
  // 3 W_out^T [D x 4D]
  const PackedB& packedB(int which, int l, int elem, int prec, int mode) {
    auto& p = packed[{which, l, elem}];
    if (p) return *p;
    p = std::make_unique<PackedB>();
    const int D = g.D, esz = elem == kTcBF16 ? 2 : 1;
    p->elem = elem;
    if (which == 0) p->rows = 3 * D, p->cols = D;
    else if (which == 1) p->rows = D, p->cols = D;
    else if (which == 2) p->rows = 4 * D, p->cols = D;
    else p->rows = D, p->cols = 4 * D;
    p->buf.ensure((size_t)p->rows * p->cols * esz);
    const int64_t ld = p->cols;
    if (which == 0) {
      for (int c = 0; c < 3; ++c)
        launch_pack_t(W(g.mat(4 + c, l), prec, mode), D, D, D,
                      p->buf.as<uint8_t>() + (size_t)c * D * D * esz, ld, elem, st);
    } else if (which == 1) {
      launch_pack_t(W(g.mat(7, l), prec, mode), D, D, D, p->buf.p, ld, elem, st);
    } else if (which == 2) {
      launch_pack_t(W(g.mat(10, l), prec, mode), D, 4 * D, 4 * D, p->buf.p, ld, elem, st);
    } else {
      launch_pack_t(W(g.mat(11, l), prec, mode), 4 * D, D, D, p->buf.p, ld, elem, st);
    }
    if (which == 1) {  // norms per head K-slice: [H][D]
      p->norm.ensure((size_t)g.H * D * 4);
      for (int h = 0; h < g.H; ++h)
        launch_rownorm(p->buf.as<uint8_t>(), ld * esz, elem, D, h * g.dk, g.dk,
                       p->norm.as<float>() + (size_t)h * D, st);
    } else {
      p->norm.ensure((size_t)p->rows * 4);
      launch_rownorm(p->buf.as<uint8_t>(), ld * esz, elem, p->rows, 0, p->cols, p->norm.as<float>(), st);
    }
    launched(2);
    return *p;
  }

  bool tc_dims_ok(int K, int elem) const { return (K * (elem == kTcBF16 ? 2 : 1)) % 32 == 0; }

  void gemm_tc(int elem, const void* A, int64_t a_rows, int a_k, const PackedB& B,
               std::vector<TcJob>& jobs, const char* name, const float* a_norm = nullptr,
               const float* a_ss = nullptr, const uint32_t* a_bad = nullptr, float* out_ss = nullptr,
               uint32_t* out_bad = nullptr) {
    if (jobs.empty()) return;
    const int esz = elem == kTcBF16 ? 2 : 1;
    TcLaunch L{};
    if (!tc_make_map(&L.tmA, A, elem, (uint64_t)a_rows, (uint64_t)a_k, (uint64_t)a_k * esz, kTcBM))
      throw Error(2, "cuTensorMapEncodeTiled failed for the A operand");
    if (!tc_make_map(&L.tmB, B.buf.p, elem, (uint64_t)B.rows, (uint64_t)B.cols,
                     (uint64_t)B.cols * esz, kTcBN))
      throw Error(2, "cuTensorMapEncodeTiled failed for the B operand");
    L.A = reinterpret_cast<const uint8_t*>(A);
    L.B = B.buf.as<uint8_t>();
    L.lda = (int64_t)a_k * esz;
    L.ldb = (int64_t)B.cols * esz;
    L.elem = elem;
    L.kappa = 8.0f;
    // fixup columns per work item: adaptive (0) by default; two columns share
    // each A load for long chains (K >= 2048: measured faster on W_out)
    // columns per fixup work item: adaptive (0) by default; two columns share
    // each A load for long chains (K >= 2048: measured faster on W_out)
    L.fix_cpi = opt_fix_cpi ? (int)opt_fix_cpi : (a_k >= 2048 ? 2 : 0);
    L.fix_dry = (int)opt_fix_dry;
    if (!gelu_lut.p) {
      gelu_lut.ensure(65536 * 2);
      launch_gelu_lut(gelu_lut.as<uint16_t>(), st);
      launched();
    }
    L.gelu_lut = gelu_lut.as<uint16_t>();
    L.out_ss = out_ss, L.out_bad = out_bad;
    if (a_norm || a_ss) {  // produced by the kernel that wrote A (fused)
      L.a_norm = a_norm, L.a_ss = a_ss, L.a_bad = a_bad;
    } else {
      float* an = scratch("tc_anorm", (size_t)a_rows);
      Prof pf(this, "rownorm", 0, (double)a_rows * a_k * esz);
      launch_rownorm(L.A, L.lda, elem, (int)a_rows, 0, a_k, an, st);
      L.a_norm = an;
    }
    int total = 0;
    double flops = 0, bytes = 0;
    for (TcJob& j : jobs) {
      j.tile0 = total;
      total += ((j.M + kTcBM - 1) / kTcBM) * ((j.N + kTcBN - 1) / kTcBN);
      flops += 2.0 * j.M * (double)j.N * j.K;
      bytes += (double)j.M * j.N * ((j.out_f32 ? 4 : 0) + (j.out_pack ? esz : 0));
    }
    L.n_jobs = (int)jobs.size();
    L.total_tiles = total;
    L.prec = jobs[0].prec;
    L.epi = jobs[0].epi;
    for (const TcJob& j : jobs)
      if (j.prec != L.prec || j.epi != L.epi) throw Error(2, "internal: mixed epilogues in one TC launch");
    if (!fix_cnt.p) {
      fix_cnt.ensure(32);
      CK(cudaMemsetAsync(fix_cnt.p, 0, 32, st));
    }
    fix_mask.ensure((size_t)total * kFixWords * 4);
    fix_tiles.ensure((size_t)total * 4);
    const size_t had = tile_mark.bytes;
    tile_mark.ensure((size_t)total * 4);
    if (tile_mark.bytes != had) CK(cudaMemsetAsync(tile_mark.p, 0, tile_mark.bytes, st));
    // the tile fixup's units and their item lists (built on the device):
    // 2 x 2-tile super-tiles for short BF16 chains (W_in), else listed tiles
    L.fix_g = opt_fix_g ? (int)opt_fix_g : (elem == kTcBF16 && a_k < 2048 ? 2 : 1);
    std::vector<int4> sts;
    if (L.fix_g == 2) sts = fixup_super_tiles(jobs.data(), (int)jobs.size());
    const size_t units = L.fix_g == 2 ? sts.size() : (size_t)total;
    fix_items.ensure(std::max<size_t>(units, 1) * fix_item_cap(L.fix_g) * 8);
    fix_n.ensure(std::max<size_t>(units, 1) * 4);
    L.fix_items = fix_items.as<uint64_t>();
    L.fix_n = fix_n.as<uint32_t>();
    L.n_fix_st = (int)sts.size();
    L.fix_mask = fix_mask.as<uint32_t>();
    L.fix_tiles = fix_tiles.as<uint32_t>();
    L.tile_mark = tile_mark.as<uint32_t>();
    L.fix_count = fix_cnt.as<uint32_t>();
    uint64_t fixed0 = 0;
    if (opt_profile) {  // flagged-element count (appended by the GEMM epilogue) -> fixup flops
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(&fixed0, fix_cnt.as<uint8_t>() + 8, 8, cudaMemcpyDeviceToHost));
    }
    std::vector<int> tj_map((size_t)total);
    for (size_t j = 0; j < jobs.size(); ++j) {
      const int end = j + 1 < jobs.size() ? jobs[j + 1].tile0 : total;
      for (int t = jobs[j].tile0; t < end; ++t) tj_map[(size_t)t] = (int)j;
    }
    // BF16: the chunked block fixup (gemm_fixup_blk_kernel) when the launch has
    // enough row tiles to fill the GPU; small launches keep the tile fixup
    long row_tiles = 0;
    for (const TcJob& j : jobs)
      row_tiles += (long)((j.M + kTcBM - 1) / kTcBM) * ((j.N + kTcBN - 1) / kTcBN + 5) / 6;
    const bool blk = elem == kTcBF16 && opt_fix_blk && row_tiles >= opt_fix_blk_min;
    std::vector<int4> fb;
    if (blk) {
      fb = fixup_chunks(jobs.data(), (int)jobs.size(), 148);
      if (!tc_make_map_sw32(&L.fxA, A, (uint64_t)a_rows, (uint64_t)a_k, (uint64_t)a_k * esz) ||
          !tc_make_map_sw32(&L.fxB, B.buf.p, (uint64_t)B.rows, (uint64_t)B.cols, (uint64_t)B.cols * esz))
        throw Error(2, "cuTensorMapEncodeTiled failed for the fixup operands");
      L.n_fix_blocks = (int)fb.size();
    }
    reserve(up_bytes(jobs.size(), sizeof(TcJob)) + up_bytes(tj_map.size(), sizeof(int)) +
            (blk ? up_bytes(fb.size(), sizeof(int4)) : 0) + up_bytes(sts.size(), sizeof(int4)));
    const TcJob* dj = upload(jobs);
    L.tile_job = upload(tj_map);
    if (blk) L.fix_blocks = upload(fb);
    L.fix_st = sts.empty() ? nullptr : upload(sts);
    {
      Prof pf(this, elem == kTcBF16 ? (std::string("gemm_tc_bf16_") + name).c_str()
                                    : (std::string("gemm_tc_fp8_") + name).c_str(),
              flops, bytes);
      launch_gemm_tc(L, dj, st);
    }
    const std::string fname = std::string("gemm_fixup_") + name;
    {
      Prof pf(this, fname.c_str());
      if (blk) launch_gemm_fixup_blk(L, dj, st);
      else launch_gemm_fixup(L, dj, st);
    }
    if (opt_profile) {
      uint64_t fixed1 = 0;
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(&fixed1, fix_cnt.as<uint8_t>() + 8, 8, cudaMemcpyDeviceToHost));
      kprof[fname].flops += 2.0 * jobs[0].K * (double)(fixed1 - fixed0);
    }
    launched();  // (the fixup kernel's last CTA resets the tile marks and count)
  }

  // Storage type of node w's output under policy P when the caller accepts
  // packed outputs: the tensor-core W_O (low-precision heads outside the
  // target's layer) and W_out (BF16 / E4M3 MLP) epilogues write the codes.
  int out_type(const Policy& P, int w) const {
    if (opt_exact || !opt_packed) return kOutF32;
    const int k = g.kind[w], l = g.layer[w];
    if (k == kHead) {
      const bool tc = P.att == 0 && P.mode == 0 && tc_dims_ok(g.D, kTcE4M3) && tc_dims_ok(g.dk, kTcE4M3);
      return tc && P.wo_precision(l) == 0 ? kOutE4M3 : kOutF32;
    }
    if (k == kMlp) {
      const int p = P.precision_of(g, w);
      const int elem = p == 1 ? kTcBF16 : kTcE4M3;
      const bool tc = (p == 1 || (p == 0 && P.mode == 0)) && tc_dims_ok(g.D, elem) &&
                      tc_dims_ok(4 * g.D, elem);
      return tc ? (p == 1 ? kOutBF16 : kOutE4M3) : kOutF32;
    }
    return kOutF32;
  }

  // ---- node computations ----------------------------------------------------
  // attention layer (model.cpp:622-718) for a list of (input, head, output)
  // last_only: only row S-1 of each item is consumed downstream (the final
  // layer under a loss metric): K/V still use every row, but the queries,
  // attention, z and W_O run for the last row only and write that row of out.
  void run_heads(int l, const Policy& P, const std::vector<HeadIO>& jobs, int nb,
                 bool last_only = false) {
    if (jobs.empty()) return;
    const int RB = nb * g.S, D = g.D, dk = g.dk, H = g.H;
    const int ZR = last_only ? nb : RB;  // z / W_O rows per job
    const size_t o_off = last_only ? (size_t)(g.S - 1) * D : 0;
    const int o_ld = last_only ? g.S * D : D;
    const size_t SEG = segf(nb);
    const int p_low = P.att;
    // tensor cores for the E4M3 projections of non-target heads
    const bool tc = !opt_exact && p_low == 0 && P.mode == 0 && tc_dims_ok(D, kTcE4M3) &&
                    tc_dims_ok(dk, kTcE4M3);
    // unique inputs over every (head, component): a split head reads its q,
    // k and v projections from (possibly) different inputs
    std::map<const float*, int> uidx;
    std::vector<const float*> uin;
    std::vector<std::array<int, 3>> u_of(jobs.size());
    std::vector<int> xln_of;
    std::vector<char> need_xln;
    for (size_t j = 0; j < jobs.size(); ++j)
      for (int c = 0; c < 3; ++c) {
        const float* in = jobs[j].input(c);
        auto it = uidx.find(in);
        if (it == uidx.end()) {
          it = uidx.emplace(in, (int)uin.size()).first;
          uin.push_back(in);
          need_xln.push_back(0);
        }
        u_of[j][c] = it->second;
        if (P.th_l == l && P.th_h == jobs[j].head) need_xln[it->second] = 1;
      }
    const size_t nu = uin.size();
    xln_of.assign(nu, -1);
    int n_xln = 0;
    for (size_t u = 0; u < nu; ++u)
      if (need_xln[u]) xln_of[u] = n_xln++;
    float* xq = tc ? nullptr : scratch("h_xq", nu * SEG);
    uint8_t* xq8 = tc ? reinterpret_cast<uint8_t*>(scratch("h_xq8", nu * SEG / 4 + 1)) : nullptr;
    float* xln = scratch("h_xln", std::max(n_xln, 1) * SEG);
    float* xnorm = tc ? scratch("h_xnorm", nu * RB) : nullptr;
    std::vector<LnJob> lj;
    for (size_t u = 0; u < nu; ++u)
      lj.push_back({uin[u], xln_of[u] >= 0 ? xln + xln_of[u] * SEG : nullptr,
                    xq ? xq + u * SEG : nullptr, RB, D, xq8 ? xq8 + u * SEG : nullptr, 1,
                    xnorm ? xnorm + u * RB : nullptr});
    const bool r4 = rtn4(p_low, P);  // (tc is off for Rtn4)
    ln(lj, g.mat(2, l), g.mat(3, l), r4 ? 2 : p_low);
    std::vector<RtnJob> rq;
    if (r4)
      for (size_t u = 0; u < nu; ++u) rq.push_back({xq + u * SEG, (int64_t)g.S * D, g.S, D, D, 0});
    rtn_act(rq, nb, P);
    rq.clear();

    // Q/K/V: per unique input a [RB][3D] block (q | k | v, head-major columns)
    const size_t QKV = (size_t)RB * 3 * D;
    // no elevated head in this layer: every Q/K/V value is E4M3-rounded, so
    // the tensor cores store the codes (1 byte) and attention decodes them
    const bool qkv8 = tc && P.th_l != l && dk % 32 == 0 && dk <= 128 && g.S <= 128;  // (the warp attention kernel)
    float* qkv = qkv8 ? nullptr : scratch("h_qkv", nu * QKV);
    uint8_t* qkvb = qkv8 ? reinterpret_cast<uint8_t*>(scratch("h_qkv8", nu * QKV / 4 + 1)) : nullptr;
    std::vector<GemmJob> gj;
    std::vector<TcJob> tj;
    const PackedB* bq = tc ? &packedB(0, l, kTcE4M3, p_low, P.mode) : nullptr;
    for (size_t u = 0; u < nu; ++u) {
      std::vector<std::pair<int, int>> hc;  // (component, non-target head) projections of input u
      for (size_t j = 0; j < jobs.size(); ++j)
        for (int c = 0; c < 3; ++c)
          if (u_of[j][c] == (int)u && !(P.th_l == l && P.th_h == jobs[j].head)) hc.push_back({c, jobs[j].head});
      std::sort(hc.begin(), hc.end());
      hc.erase(std::unique(hc.begin(), hc.end()), hc.end());
      float* blk = qkv8 ? nullptr : qkv + u * QKV;
      uint8_t* blk8 = qkv8 ? qkvb + u * QKV : nullptr;
      if (tc && (int)hc.size() == 3 * H) {
        TcJob t{};
        t.a_row0 = (int)u * RB, t.b_row0 = 0, t.b_k0 = 0, t.M = RB, t.N = 3 * D, t.K = D;
        if (qkv8) t.out_pack = blk8;
        else t.out_f32 = blk;
        t.ldo = 3 * D, t.b_norm = bq->norm.as<float>(), t.prec = p_low;
        tj.push_back(t);
        continue;
      }
      for (const auto& ch : hc) {
          const int c = ch.first, h = ch.second;
          if (tc) {
            TcJob t{};
            t.a_row0 = (int)u * RB, t.b_row0 = c * D + h * dk, t.b_k0 = 0, t.M = RB, t.N = dk, t.K = D;
            if (qkv8) t.out_pack = blk8 + c * D + h * dk;
            else t.out_f32 = blk + c * D + h * dk;
            t.ldo = 3 * D;
            t.b_norm = bq->norm.as<float>() + c * D + h * dk, t.prec = p_low;
            tj.push_back(t);
          } else {
            GemmJob q{};
            q.A = xq + u * SEG, q.B = W(g.mat(4 + c, l), p_low, P.mode) + h * dk;
            q.C = blk + c * D + h * dk;
            q.M = RB, q.N = dk, q.K = D, q.lda = D, q.ldb = D, q.ldc = 3 * D, q.prec = r4 ? 2 : p_low;
            gj.push_back(q);
            if (r4) rq.push_back({q.C, (int64_t)g.S * 3 * D, g.S, dk, 3 * D, 0});
          }
        }
    }
    for (size_t j = 0; j < jobs.size(); ++j) {  // the elevated head: FP32 (model.cpp:665-675)
      const int h = jobs[j].head;
      if (!(P.th_l == l && P.th_h == h)) continue;
      for (int c = 0; c < 3; ++c) {
        GemmJob q{};
        q.A = xln + xln_of[u_of[j][c]] * SEG, q.B = master[g.mat(4 + c, l)]->as<float>() + h * dk;
        q.C = qkv + u_of[j][c] * QKV + c * D + h * dk;
        q.M = RB, q.N = dk, q.K = D, q.lda = D, q.ldb = D, q.ldc = 3 * D, q.prec = 2;
        gj.push_back(q);
      }
    }
    if (tc) gemm_tc(kTcE4M3, xq8, (int64_t)nu * RB, D, *bq, tj, "qkv", xnorm);
    gemm(gj, "gemm_qkv");
    rtn_act(rq, nb, P);
    rq.clear();

    // attention + z (FP32 for the exact W_O, E4M3 bytes for the tensor cores)
    const int wo_prec = P.wo_precision(l);
    const bool tc_wo = tc && wo_prec == 0;
    const size_t per = (size_t)ZR * dk;
    float* z = tc_wo ? nullptr : scratch("h_z", jobs.size() * per);
    uint8_t* z8 = tc_wo ? reinterpret_cast<uint8_t*>(scratch("h_z8", jobs.size() * per / 4 + 1)) : nullptr;
    float* znorm = tc_wo ? scratch("h_znorm", jobs.size() * (size_t)ZR) : nullptr;  // W_O's ||a||
    std::vector<AttnJob> aj;
    for (size_t j = 0; j < jobs.size(); ++j) {
      const int h = jobs[j].head;
      const bool target = P.th_l == l && P.th_h == h;
      AttnJob a{};
      if (qkv8) {
        a.q8 = qkvb + u_of[j][0] * QKV + h * dk;
        a.k8 = qkvb + u_of[j][1] * QKV + D + h * dk;
        a.v8 = qkvb + u_of[j][2] * QKV + 2 * D + h * dk;
      } else {
        a.q = qkv + u_of[j][0] * QKV + h * dk;
        a.k = qkv + u_of[j][1] * QKV + D + h * dk;
        a.v = qkv + u_of[j][2] * QKV + 2 * D + h * dk;
      }
      a.ld = 3 * D;
      a.prec = (target || r4) ? 2 : p_low, a.ldz = dk, a.q0 = last_only ? g.S - 1 : 0;
      a.z = z ? z + j * per : nullptr;
      if (r4 && !target) rq.push_back({a.z, (int64_t)g.S * dk, g.S, dk, dk, 0});
      a.z8 = z8 ? z8 + j * per : nullptr;
      a.znorm = znorm ? znorm + j * (size_t)ZR : nullptr;
      aj.push_back(a);
    }
    attn(aj, nb);
    rtn_act(rq, nb, P);
    rq.clear();
    gj.clear();
    tj.clear();
    if (tc_wo) {
      const PackedB& bo = packedB(1, l, kTcE4M3, wo_prec, P.mode);
      for (size_t j = 0; j < jobs.size(); ++j) {
        const int h = jobs[j].head;
        TcJob t{};
        t.a_row0 = (int)j * ZR, t.b_row0 = 0, t.b_k0 = h * dk, t.M = ZR, t.N = D, t.K = dk;
        if (jobs[j].otype == kOutE4M3) t.out_pack = reinterpret_cast<uint8_t*>(jobs[j].out) + o_off;
        else t.out_f32 = jobs[j].out + o_off;
        t.ldo = o_ld, t.b_norm = bo.norm.as<float>() + (size_t)h * D;
        t.prec = p_low;
        tj.push_back(t);
      }
      gemm_tc(kTcE4M3, z8, (int64_t)jobs.size() * ZR, dk, bo, tj, "wo", znorm);
    } else {
      const float* wo = W(g.mat(7, l), wo_prec, P.mode);
      for (size_t j = 0; j < jobs.size(); ++j) {
        if (jobs[j].otype != kOutF32) throw Error(2, "internal: packed head output on the exact W_O path");
        const int h = jobs[j].head;
        const bool target = P.th_l == l && P.th_h == h;
        GemmJob o{};
        o.A = z + j * per, o.B = wo + (size_t)h * dk * D, o.C = jobs[j].out + o_off;
        o.M = ZR, o.N = D, o.K = dk, o.lda = dk, o.ldb = D, o.ldc = o_ld;
        o.prec = (target || r4) ? 2 : p_low, o.epi = 0;
        gj.push_back(o);
        if (r4 && !target) rq.push_back({o.C, (int64_t)g.S * D, g.S, D, D, 0});
      }
      gemm(gj, "gemm_wo");
      rtn_act(rq, nb, P);
    }
  }

  // MLP (model.cpp:720-739)
  void run_mlp(int l, const Policy& P, const std::vector<SegIO>& jobs, int nb,
               bool last_only = false) {
    if (jobs.empty()) return;
    const int RB = last_only ? nb : nb * g.S, D = g.D;
    const size_t i_off = last_only ? (size_t)(g.S - 1) * D : 0;
    const int i_ld = last_only ? g.S * D : D;
    const size_t SEG = segf(nb);
    const int node = g.stage_nodes[2 + 2 * l][0];
    const int p = P.precision_of(g, node);
    const int elem = p == 1 ? kTcBF16 : kTcE4M3;
    const bool tc = !opt_exact && (p == 1 || (p == 0 && P.mode == 0)) && tc_dims_ok(D, elem) &&
                    tc_dims_ok(4 * D, elem);
    if (tc) {
      const int esz = elem == kTcBF16 ? 2 : 1;
      uint8_t* xqp = reinterpret_cast<uint8_t*>(scratch("m_xqp", jobs.size() * SEG * esz / 4 + 1));
      uint8_t* hidp = reinterpret_cast<uint8_t*>(scratch("m_hidp", jobs.size() * SEG * esz + 1));
      float* xnorm = scratch("m_xnorm", jobs.size() * RB);
      std::vector<LnJob> lj;
      for (size_t j = 0; j < jobs.size(); ++j)
        lj.push_back({jobs[j].in + i_off, nullptr, nullptr, RB, i_ld, xqp + j * RB * D * esz,
                      elem == kTcBF16 ? 2 : 1, xnorm + j * RB});
      ln(lj, g.mat(8, l), g.mat(9, l), p);
      const PackedB& bi = packedB(2, l, elem, p, P.mode);
      const PackedB& bo = packedB(3, l, elem, p, P.mode);
      std::vector<TcJob> t1, t2;
      for (size_t j = 0; j < jobs.size(); ++j) {
        TcJob a{};
        a.a_row0 = (int)j * RB, a.M = RB, a.N = 4 * D, a.K = D;
        a.out_pack = hidp + j * RB * 4 * D * esz, a.ldo = 4 * D, a.b_norm = bi.norm.as<float>();
        a.prec = p, a.epi = 1;
        t1.push_back(a);
        TcJob b{};
        b.a_row0 = (int)j * RB, b.M = RB, b.N = D, b.K = 4 * D;
        if (jobs[j].otype != kOutF32) {
          if (jobs[j].otype != (elem == kTcBF16 ? kOutBF16 : kOutE4M3))
            throw Error(2, "internal: MLP output type does not match its precision");
          b.out_pack = reinterpret_cast<uint8_t*>(jobs[j].out) + i_off * esz;
        } else {
          b.out_f32 = jobs[j].out + i_off;
        }
        b.ldo = i_ld, b.b_norm = bo.norm.as<float>(), b.prec = p;
        t2.push_back(b);
      }
      // the W_in epilogue accumulates the hidden rows' norms for W_out's certificate
      float* hss = scratch("m_hss", 2 * jobs.size() * RB);
      uint32_t* hbad = reinterpret_cast<uint32_t*>(hss + jobs.size() * RB);
      CK(cudaMemsetAsync(hss, 0, sizeof(float) * 2 * jobs.size() * RB, st));
      gemm_tc(elem, xqp, (int64_t)jobs.size() * RB, D, bi, t1, "mlp_in", xnorm, nullptr, nullptr,
              hss, hbad);
      gemm_tc(elem, hidp, (int64_t)jobs.size() * RB, 4 * D, bo, t2, "mlp_out", nullptr, hss, hbad);
      return;
    }
    for (const SegIO& j : jobs)
      if (j.otype != kOutF32) throw Error(2, "internal: packed MLP output on the exact path");
    float* xq = scratch("m_xq", jobs.size() * SEG);
    float* hid = scratch("m_hid", jobs.size() * SEG * 4);
    std::vector<LnJob> lj;
    for (size_t j = 0; j < jobs.size(); ++j) lj.push_back({jobs[j].in + i_off, nullptr, xq + j * SEG, RB, i_ld});
    const bool r4 = rtn4(p, P);
    ln(lj, g.mat(8, l), g.mat(9, l), r4 ? 2 : p);
    std::vector<RtnJob> r0, r1, r2, r3;
    for (size_t j = 0; j < jobs.size() && r4; ++j) {
      const int64_t S = g.S;
      r0.push_back({xq + j * SEG, S * D, g.S, D, D, 0});
      r1.push_back({hid + j * SEG * 4, S * 4 * D, g.S, 4 * D, 4 * D, 0});
      r2.push_back({hid + j * SEG * 4, S * 4 * D, g.S, 4 * D, 4 * D, 1});
      r3.push_back({jobs[j].out, S * D, g.S, D, D, 0});
    }
    rtn_act(r0, nb, P);
    const float* win = W(g.mat(10, l), p, P.mode);
    const float* wout = W(g.mat(11, l), p, P.mode);
    std::vector<GemmJob> g1, g2;
    for (size_t j = 0; j < jobs.size(); ++j) {
      GemmJob a{};
      a.A = xq + j * SEG, a.B = win, a.C = hid + j * SEG * 4;
      a.M = RB, a.N = 4 * D, a.K = D, a.lda = D, a.ldb = 4 * D, a.ldc = 4 * D;
      a.prec = r4 ? 2 : p, a.epi = r4 ? 0 : 1;
      g1.push_back(a);
      GemmJob b{};
      b.A = hid + j * SEG * 4, b.B = wout, b.C = jobs[j].out + i_off;
      b.M = RB, b.N = D, b.K = 4 * D, b.lda = 4 * D, b.ldb = D, b.ldc = i_ld, b.prec = r4 ? 2 : p, b.epi = 0;
      g2.push_back(b);
    }
    gemm(g1, "gemm_mlp_in");
    rtn_act(r1, nb, P);  // round -> GELU -> round (model.cpp:727-731)
    rtn_act(r2, nb, P);
    gemm(g2, "gemm_mlp_out");
    rtn_act(r3, nb, P);
  }

  // unembed (model.cpp:741-753): all_rows=false computes only row S-1 of
  // each item (the only row patched_divergence reads, patching.cpp:155-157).
  void run_unembed(const Policy& P, const std::vector<SegIO>& jobs, int nb, bool all_rows) {
    if (jobs.empty()) return;
    const int rows = all_rows ? nb * g.S : nb, D = g.D, V = g.V;
    const int p = P.unemb;
    if (rtn4(p, P)) {  // group = all S rows of an item: every row is needed
      for (const SegIO& jb : jobs) {
        float* xq = scratch("u_xq", (size_t)nb * g.S * D);
        float* lg = all_rows ? jb.out : scratch("u_lg", (size_t)nb * g.S * V);
        ln({{jb.in, nullptr, xq, nb * g.S, D}}, g.mat(12, 0), g.mat(13, 0), 2);
        rtn_act({{xq, (int64_t)g.S * D, g.S, D, D, 0}}, nb, P);
        GemmJob a{};
        a.A = xq, a.B = W(g.mat(14, 0), p, P.mode), a.C = lg;
        a.M = nb * g.S, a.N = V, a.K = D, a.lda = D, a.ldb = V, a.ldc = V, a.prec = 2;
        gemm({a}, "gemm_unembed");
        rtn_act({{lg, (int64_t)g.S * V, g.S, V, V, 0}}, nb, P);
        if (!all_rows)
          CK(cudaMemcpy2DAsync(jb.out, (size_t)V * 4, lg + (size_t)(g.S - 1) * V, (size_t)g.S * V * 4,
                               (size_t)V * 4, nb, cudaMemcpyDeviceToDevice, st));
      }
      return;
    }
    float* xq = scratch("u_xq", jobs.size() * (size_t)rows * D);
    std::vector<LnJob> lj;
    for (size_t j = 0; j < jobs.size(); ++j)
      lj.push_back({jobs[j].in + (all_rows ? 0 : (size_t)(g.S - 1) * D), nullptr,
                    xq + j * (size_t)rows * D, rows, all_rows ? D : g.S * D});
    ln(lj, g.mat(12, 0), g.mat(13, 0), p);
    // W_u with its row pitch padded to a multiple of 4 floats (one resident
    // copy per image): 16-byte loads in the exact GEMM's B staging
    const float* wu0 = W(g.mat(14, 0), p, P.mode);
    const int ldu = (V + 3) & ~3;
    auto& pad = wu_pad[wu0];
    if (!pad) {
      pad = std::make_unique<DeviceBuf>();
      pad->ensure((size_t)D * ldu * 4);
      CK(cudaMemsetAsync(pad->p, 0, (size_t)D * ldu * 4, st));
      CK(cudaMemcpy2DAsync(pad->p, (size_t)ldu * 4, wu0, (size_t)V * 4, (size_t)V * 4, D,
                           cudaMemcpyDeviceToDevice, st));
    }
    const float* wu = pad->as<float>();
    std::vector<GemmJob> gj;
    bool contiguous = true;  // all segments' logits back to back: one tall GEMM
    for (size_t j = 0; j < jobs.size(); ++j)
      contiguous = contiguous && jobs[j].out == jobs[0].out + j * (size_t)rows * V;
    if (contiguous) {
      GemmJob a{};
      a.A = xq, a.B = wu, a.C = jobs[0].out;
      a.M = rows * (int)jobs.size(), a.N = V, a.K = D, a.lda = D, a.ldb = ldu, a.ldc = V, a.prec = p;
      gj.push_back(a);
    } else {
      for (size_t j = 0; j < jobs.size(); ++j) {
        GemmJob a{};
        a.A = xq + j * (size_t)rows * D, a.B = wu, a.C = jobs[j].out;
        a.M = rows, a.N = V, a.K = D, a.lda = D, a.ldb = ldu, a.ldc = V, a.prec = p, a.epi = 0;
        gj.push_back(a);
      }
    }
    gemm(gj, "gemm_unembed");
  }

  // ---- the patched passes' unembed on the tensor cores --------------------------
  struct Wu6 {
    PackedB b6;  // [V][6D] BF16 split of the FP32 image, + ||w_j|| in b6.norm
  };
  std::map<const float*, std::unique_ptr<Wu6>> wu6;
  DeviceBuf ucnt;  // [0] rows flagged by the current launch, [1] running total of the call
  // K7 + K8 fused (gemm_unembed_kl_kernel): the patched rows' exact unembed
  // writes per-tile KL partials instead of logits; kl_reduce forms the KL.
  bool kl_fused_ok(const Policy& P, bool loss) const {
    return opt_kl_fused && loss && metric == 0 && !unembed_tc_ok(P) && !rtn4(P.unemb, P);
  }
  const double2* run_unembed_kl(const Policy& P, const Run& R, const std::vector<SegIO>& jobs, int nb) {
    const int D = g.D, V = g.V;
    const size_t rows = jobs.size() * (size_t)nb;
    float* xq = scratch("u_xq", rows * D);
    std::vector<LnJob> lj;
    for (size_t j = 0; j < jobs.size(); ++j)
      lj.push_back({jobs[j].in + (size_t)(g.S - 1) * D, nullptr, xq + j * (size_t)nb * D, nb, g.S * D});
    ln(lj, g.mat(12, 0), g.mat(13, 0), P.unemb);
    const int ldu = (V + 3) & ~3;
    const float* wu = wu_padded(W(g.mat(14, 0), P.unemb, P.mode), ldu);
    const int n_ct = unembed_kl_col_tiles(V);
    double2* part = reinterpret_cast<double2*>(scratch("u_klpart", rows * n_ct * 4));
    GemmJob a{};
    a.A = xq, a.B = wu, a.C = nullptr;
    a.M = (int)rows, a.N = V, a.K = D, a.lda = D, a.ldb = ldu, a.ldc = V, a.prec = P.unemb;
    if (!R.xbp.p) throw Error(2, "internal: fused KL without padded baselines");
    KlFuse kf{R.xbp.as<double>(), R.ebp.as<double>(), part, nb, n_ct, n_ct * 128};
    Prof pf(this, "gemm_unembed", 2.0 * (double)rows * V * D, 0);
    launch_gemm_unembed_kl(a, kf, st);
    return part;
  }
  const float* wu_padded(const float* wu0, int ldu) {
    auto& pad = wu_pad[wu0];
    if (!pad) {
      pad = std::make_unique<DeviceBuf>();
      pad->ensure((size_t)g.D * ldu * 4);
      CK(cudaMemsetAsync(pad->p, 0, (size_t)g.D * ldu * 4, st));
      CK(cudaMemcpy2DAsync(pad->p, (size_t)ldu * 4, wu0, (size_t)g.V * 4, (size_t)g.V * 4, g.D,
                           cudaMemcpyDeviceToDevice, st));
    }
    return pad->as<float>();
  }
  bool unembed_tc_ok(const Policy& P) const {
    return opt_unembed_tc && !opt_exact && metric == 0 && P.unemb == 2 && P.mode == 0 &&
           (12 * g.D) % 32 == 0;
  }
  // LN_f -> FP32 rows xq (the exact path's operand, kept for the fallback) ->
  // A6 split + ||a|| -> one tcgen05 GEMM (BF16, FP32 accumulators, no
  // rounding: P32) into the logits. Last rows only (loss metrics).
  struct UnembedTc {
    float* xq = nullptr;
    float* anorm = nullptr;
    const float* wu = nullptr;  // padded FP32 image (the exact fallback's B)
    int ldu = 0;
    const float* wnorm = nullptr;
    int rows = 0;
  };
  UnembedTc run_unembed_tc(const Policy& P, const std::vector<SegIO>& jobs, int nb) {
    const int D = g.D, V = g.V, rows = (int)jobs.size() * nb;
    UnembedTc u;
    u.rows = rows;
    u.xq = scratch("u_xq", (size_t)rows * D);
    std::vector<LnJob> lj;
    for (size_t j = 0; j < jobs.size(); ++j)
      lj.push_back({jobs[j].in + (size_t)(g.S - 1) * D, nullptr, u.xq + j * (size_t)nb * D, nb, g.S * D});
    ln(lj, g.mat(12, 0), g.mat(13, 0), P.unemb);
    const float* wu0 = W(g.mat(14, 0), P.unemb, P.mode);
    auto& w6 = wu6[wu0];
    if (!w6) {
      w6 = std::make_unique<Wu6>();
      w6->b6.rows = V, w6->b6.cols = 6 * D, w6->b6.elem = kTcBF16;
      w6->b6.buf.ensure((size_t)V * 6 * D * 2);
      w6->b6.norm.ensure((size_t)V * 4);
      launch_split_cols(wu0, D, V, w6->b6.buf.as<uint16_t>(), w6->b6.norm.as<float>(), st);
      launched(2);
    }
    u.wnorm = w6->b6.norm.as<float>();
    uint16_t* a6 = reinterpret_cast<uint16_t*>(scratch("u_a6", (size_t)rows * 3 * D));
    u.anorm = scratch("u_anorm", (size_t)rows);
    {
      Prof pf(this, "unembed_split", 0, (double)rows * D * (4.0 + 12.0));
      launch_split_rows(u.xq, rows, D, D, a6, u.anorm, st);
    }
    // the exact fallback's W_u (pitch-padded copy, as run_unembed)
    u.ldu = (V + 3) & ~3;
    auto& pad = wu_pad[wu0];
    if (!pad) {
      pad = std::make_unique<DeviceBuf>();
      pad->ensure((size_t)D * u.ldu * 4);
      CK(cudaMemsetAsync(pad->p, 0, (size_t)D * u.ldu * 4, st));
      CK(cudaMemcpy2DAsync(pad->p, (size_t)u.ldu * 4, wu0, (size_t)V * 4, (size_t)V * 4, D,
                           cudaMemcpyDeviceToDevice, st));
    }
    u.wu = pad->as<float>();
    bool contiguous = true;
    for (size_t j = 0; j < jobs.size(); ++j) contiguous = contiguous && jobs[j].out == jobs[0].out + j * (size_t)nb * V;
    if (!contiguous) throw Error(2, "internal: tensor-core unembed expects contiguous logits");
    std::vector<TcJob> tj(1);
    TcJob& t = tj[0];
    t = TcJob{};
    t.a_row0 = 0, t.b_row0 = 0, t.b_k0 = 0, t.M = rows, t.N = V, t.K = 6 * D;
    t.out_f32 = jobs[0].out, t.ldo = V, t.prec = 2, t.epi = 0;
    gemm_tc(kTcBF16, a6, rows, 6 * D, w6->b6, tj, "unembed", u.anorm);
    return u;
  }

  void run_embed(const Policy& P, const int* d_tok, float* out, int nb) {
    const bool r4 = rtn4(P.emb, P);
    launch_embed(d_tok, W(g.mat(0, 0), P.emb, P.mode), W(g.mat(1, 0), P.emb, P.mode), out, nb, g.S,
                 g.D, r4 ? 2 : P.emb, st);
    launched();
    if (r4) rtn_act({{out, (int64_t)g.S * g.D, g.S, g.D, g.D, 0}}, nb, P);
  }

  // ---- a full (or suffix) forward over a trie: the baseline runs ----------
  void prepare_run(Run& R, const Trie& T, int nb, bool all_rows) {
    R.nb = nb;
    R.seg = segf(nb);
    R.out.ensure((size_t)g.N * R.seg * 4);
    R.trie.ensure((size_t)T.size() * R.seg * 4);
    R.logits.ensure((size_t)(all_rows ? nb * g.S : nb) * g.V * 4);
    R.lse.ensure((size_t)nb * 8);
    R.otype.assign(g.N, kOutF32);
  }

  // node w's input (component c of a split head)
  const float* input_of(const Trie& T, const Run& R, int w, int c = 0) {
    const int r = T.rec_in[g.recv(w, c)];
    return r == 0 ? zeros(R.seg) : R.t(r);
  }
  HeadIO head_io(const Trie& T, const Run& R, int w, float* out, int otype) {
    HeadIO h{input_of(T, R, w), g.head[w], out, otype};
    if (g.split) h.in_k = input_of(T, R, w, 1), h.in_v = input_of(T, R, w, 2);
    return h;
  }

  // loss metrics read only the last position of the logits: the final
  // layer's attention outputs and MLP are then needed at row S-1 only
  // (not under Rtn4, whose per-tensor delta spans every row).
  bool last_rows(int l, const Policy& P, bool loss_only) const {
    return loss_only && l == g.L - 1 && P.mode == 0;
  }

  void forward_run(Run& R, const Trie& T, const Policy& P, const int* d_tok, int sigma0,
                   bool all_rows, int* d_nan, bool loss_only = false) {
    struct Tag {
      std::string& t;
      std::string old;
      Tag(std::string& x) : t(x), old(x) { t = "base:"; }
      ~Tag() { t = old; }
    } tag(prof_tag);
    for (int s = sigma0; s < g.n_stages; ++s) {
      const auto& nodes = g.stage_nodes[s];
      if (nodes.empty()) continue;  // MLP stages of attention-only models
      const int k = g.kind[nodes[0]];
      if (k == kEmbed) {
        run_embed(P, d_tok, R.o(0), R.nb);
        R.otype[0] = kOutF32;
      } else if (k == kHead) {
        std::vector<HeadIO> hj;
        for (int w : nodes) {
          R.otype[w] = (int8_t)out_type(P, w);
          hj.push_back(head_io(T, R, w, R.o(w), R.otype[w]));
        }
        run_heads(g.layer[nodes[0]], P, hj, R.nb, last_rows(g.layer[nodes[0]], P, loss_only));
      } else if (k == kMlp) {
        R.otype[nodes[0]] = (int8_t)out_type(P, nodes[0]);
        run_mlp(g.layer[nodes[0]], P, {{input_of(T, R, nodes[0]), R.o(nodes[0]), R.otype[nodes[0]]}}, R.nb,
                last_rows(g.layer[nodes[0]], P, loss_only));
      } else {
        run_unembed(P, {{input_of(T, R, g.unembed), R.logits.as<float>()}}, R.nb, all_rows);
        if (!all_rows) {
          const bool kl = metric == 0;
          if (kl) R.prob.ensure((size_t)R.nb * g.V * 8), R.psum.ensure((size_t)R.nb * 8);
          launch_lse(R.logits.as<float>(), R.nb, g.V, R.lse.as<double>(), d_nan, st,
                     kl ? R.prob.as<double>() : nullptr, kl ? R.psum.as<double>() : nullptr);
          if (kl && opt_kl_fused) {  // the fused KL's 16-byte-aligned baseline rows
            const int ld = unembed_kl_col_tiles(g.V) * 128;
            R.xbp.ensure((size_t)R.nb * ld * 8), R.ebp.ensure((size_t)R.nb * ld * 8);
            launch_pad_baselines(R.logits.as<float>(), R.prob.as<double>(), R.nb, g.V, ld, R.xbp.as<double>(),
                                 R.ebp.as<double>(), st);
          }
          launched();
        }
      }
      // trie values whose last source is at this stage
      std::vector<FoldOp> ops;
      const float* prev = nullptr;
      for (int t : T.by_stage[s]) {
        const int p = T.parent[t];
        const float* a = p == 0 ? nullptr : R.t(p);
        if (a && a == prev) a = CQG_REG_PREV;
        ops.push_back({a, R.o(T.src[t]), R.t(t), R.otype[T.src[t]]});
        prev = R.t(t);
      }
      if (!ops.empty()) fold(ops, {{0, (int)ops.size()}}, R.seg);
    }
  }

  // ---- patch values (prepare_policy's full-graph runs, patching.cpp:171-185)
  const int* tokens(int which) const { return which == 0 ? d_clean.as<int>() : d_corrupt.as<int>(); }

  void ensure_patch_run(const Policy& base, int which, int* d_nan) {
    if (patch_valid && patch_policy == base && patch_tokens == which) return;
    prepare_run(patch_run, full, B, false);
    forward_run(patch_run, full, base, tokens(which), 0, false, d_nan);
    patch_valid = true;
    patch_policy = base;
    patch_tokens = which;
    ++target_gen;
  }

  // out[s] of the full-graph run under policy_for_edge (target = s)
  const float* patch_value(int s, const Policy& ps, bool per_edge, int* otype) {
    if (!per_edge || g.kind[s] == kEmbed) {
      *otype = patch_run.otype[s];
      return patch_run.o(s);
    }
    *otype = out_type(ps, s);
    auto& c = target_cache[s];
    if (c.gen == target_gen) return c.buf.as<float>();
    c.buf.ensure(patch_run.seg * 4);
    c.gen = target_gen;
    const float* in = input_of(full, patch_run, s);
    if (g.kind[s] == kHead) run_heads(g.layer[s], ps, {head_io(full, patch_run, s, c.buf.as<float>(), *otype)}, B);
    else run_mlp(g.layer[s], ps, {{in, c.buf.as<float>(), *otype}}, B);
    return c.buf.as<float>();
  }

  // ---- the patched passes of one policy group -------------------------------
  struct EdgePlan {
    int e, s, v, sv;
    int r;  // destination receiver (= v's only receiver unless v is a split head)
    const float* pv;
    int pvt;  // OutType of pv
    std::vector<int8_t> nchg, tchg, virt;
    std::vector<int> nslot, tslot;
    int n_slots = 0;
    float* base_ptr = nullptr;  // sval then slots
    float* sval() const { return base_ptr; }
    float* slot(int k, size_t seg) const { return base_ptr + (size_t)(1 + k) * seg; }
  };

  void plan_edge(EdgePlan& P, const Trie& T, bool loss) {
    const int N = g.N, TS = T.size();
    P.nchg.assign(N, 0);
    P.tchg.assign(TS, 0);
    P.virt.assign(TS, 0);
    P.nslot.assign(N, -1);
    P.tslot.assign(TS, -1);
    P.nchg[P.v] = 1;
    const int last = loss ? g.n_stages - 1 : P.sv;
    for (int s = P.sv; s <= last; ++s) {
      if (s > P.sv)
        for (int w : g.stage_nodes[s]) {
          P.nchg[w] = 0;
          for (int c = 0; c < g.n_recv(w); ++c) {  // (a split head: any of q, k, v inputs)
            const int ri = T.rec_in[g.recv(w, c)];
            if (ri != 0 && P.tchg[ri]) P.nchg[w] = 1;
          }
        }
      if (s < last || loss)
        for (int t : T.by_stage[s])
          P.tchg[t] = (P.nchg[T.src[t]] || (T.parent[t] != 0 && P.tchg[T.parent[t]])) ? 1 : 0;
    }
    if (!loss) {  // act_diff: only the destination's output is needed
      std::fill(P.tchg.begin(), P.tchg.end(), 0);
      std::fill(P.nchg.begin(), P.nchg.end(), 0);
      P.nchg[P.v] = 1;
    }
    // consumers of changed trie values
    std::vector<int> ncons(TS, 0), only_child(TS, -1);
    for (int t = 1; t < TS; ++t)
      if (P.tchg[t] && T.parent[t] != 0 && P.tchg[T.parent[t]]) {
        ncons[T.parent[t]]++;
        only_child[T.parent[t]] = t;
      }
    // a changed node's changed inputs are consumed by its kernels (never
    // virtual); its unchanged inputs (other components of a split head) are
    // read from the baseline
    auto changed_inputs = [&](int w, auto&& fn) {
      for (int c = 0; c < g.n_recv(w); ++c) {
        const int ri = T.rec_in[g.recv(w, c)];
        if (ri != 0 && P.tchg[ri]) fn(ri);
      }
    };
    for (int w = 0; w < N; ++w)
      if (P.nchg[w] && g.stage[w] > P.sv) changed_inputs(w, [&](int ri) { ncons[ri] += 2; });
    // program order per stage -> virtual (register-only) values
    for (int s = P.sv; s <= last && loss; ++s) {
      int prev = -1;
      for (int t : T.by_stage[s]) {
        if (!P.tchg[t]) continue;
        if (prev >= 0 && ncons[prev] == 1 && only_child[prev] == t) P.virt[prev] = 1;
        prev = t;
      }
    }
    // liveness over time 2*stage (node compute) / 2*stage+1 (fold)
    struct Val { int def, last, kind, id; };
    std::vector<Val> vals;
    for (int w = 0; w < N; ++w) {
      if (!P.nchg[w] || w == g.unembed) continue;
      vals.push_back({2 * g.stage[w], loss ? 2 * g.stage[w] + 1 : 2 * g.stage[w], 0, w});
    }
    std::vector<int> lastuse(TS, -1);
    for (int t = 1; t < TS; ++t)
      if (P.tchg[t] && T.parent[t] != 0 && P.tchg[T.parent[t]])
        lastuse[T.parent[t]] = std::max(lastuse[T.parent[t]], 2 * g.stage[T.src[t]] + 1);
    for (int w = 0; w < N; ++w)
      if (P.nchg[w] && g.stage[w] > P.sv)
        changed_inputs(w, [&](int ri) { lastuse[ri] = std::max(lastuse[ri], 2 * g.stage[w]); });
    for (int t = 1; t < TS; ++t) {
      if (!P.tchg[t] || P.virt[t]) continue;
      const int def = 2 * g.stage[T.src[t]] + 1;
      vals.push_back({def, std::max(def, lastuse[t]), 1, t});
    }
    std::sort(vals.begin(), vals.end(), [](const Val& a, const Val& b) { return a.def < b.def; });
    std::vector<std::pair<int, int>> busy;  // (last, slot)
    std::vector<int> freel;
    int n = 0;
    for (const Val& x : vals) {
      for (size_t i = 0; i < busy.size();) {
        if (busy[i].first < x.def) {
          freel.push_back(busy[i].second);
          busy[i] = busy.back();
          busy.pop_back();
        } else {
          ++i;
        }
      }
      int sl;
      if (!freel.empty()) {
        sl = freel.back();
        freel.pop_back();
      } else {
        sl = n++;
      }
      busy.push_back({x.last, sl});
      (x.kind == 0 ? P.nslot[x.id] : P.tslot[x.id]) = sl;
    }
    P.n_slots = n;
  }

  // Scores (sum over local items, item order) for the edges of one group.
  void run_passes(const Trie& T, const Policy& P, const Run& R, std::vector<EdgePlan>& plans,
                  bool loss, double* d_d /* [n][nb] */, int* d_nan) {
    const int nb = R.nb;
    const size_t SEG = R.seg;
    const int V = g.V;
    // arena: sval + slots per edge
    size_t total = 0;
    for (auto& p : plans) total += (size_t)(1 + p.n_slots) * SEG;
    float* arena = scratch("p_arena", total);
    size_t off = 0;
    for (auto& p : plans) {
      p.base_ptr = arena + off;
      off += (size_t)(1 + p.n_slots) * SEG;
    }
    // 1) patched receiver inputs: fold along v's source path with s -> pv
    {
      std::vector<FoldOp> ops;
      std::vector<FoldProg> progs;
      for (auto& p : plans) {
        std::vector<int> path;
        for (int t = T.rec_in[p.r]; t != 0; t = T.parent[t]) path.push_back(t);
        std::reverse(path.begin(), path.end());
        size_t k = 0;
        while (k < path.size() && T.src[path[k]] != p.s) ++k;
        if (k == path.size()) throw Error(2, "internal: source missing from receiver path");
        const int b = (int)ops.size();
        for (size_t i = k; i < path.size(); ++i) {
          const int t = path[i];
          const float* a;
          if (i == k) a = T.parent[t] == 0 ? nullptr : R.t(T.parent[t]);
          else a = CQG_REG_PREV;
          const float* bsrc = (i == k) ? p.pv : R.o(T.src[t]);
          ops.push_back({a, bsrc, i + 1 == path.size() ? p.sval() : nullptr,
                         (i == k) ? p.pvt : (int)R.otype[T.src[t]]});
        }
        progs.push_back({b, (int)ops.size()});
      }
      fold(ops, progs, SEG);
    }
    int smin = g.n_stages, smax = 0;
    for (auto& p : plans) smin = std::min(smin, p.sv), smax = std::max(smax, p.sv);
    const int last = loss ? g.n_stages - 1 : smax;
    float* logits = nullptr;
    const double2* klpart = nullptr;  // fused unembed + KL: per-tile partials (no logits)
    UnembedTc utc;  // utc.rows > 0: the logits came from the tensor cores
    std::vector<int> unembed_edges;  // plan indices whose logits were computed
    for (int s = smin; s <= last; ++s) {
      const auto& nodes = g.stage_nodes[s];
      if (nodes.empty()) continue;  // MLP stages of attention-only models
      const int k = g.kind[nodes[0]];
      std::vector<HeadIO> hj;
      std::vector<SegIO> mj;
      std::vector<int> uj;
      for (size_t pi = 0; pi < plans.size(); ++pi) {
        auto& p = plans[pi];
        if (p.sv > s) continue;
        for (int w : nodes) {
          if (!p.nchg[w]) continue;
          // receiver input: the patched sum (the destination receiver), a
          // recomputed trie value, or the baseline's (unchanged component)
          auto rin = [&](int c) -> const float* {
            const int r = g.recv(w, c);
            if (w == p.v && r == p.r) return p.sval();
            const int t = T.rec_in[r];
            if (t != 0 && p.tchg[t]) return p.slot(p.tslot[t], SEG);
            return t == 0 ? zeros(SEG) : R.t(t);
          };
          const float* in = rin(0);
          if (k == kHead) {
            HeadIO h{in, g.head[w], p.slot(p.nslot[w], SEG), out_type(P, w)};
            if (g.split) h.in_k = rin(1), h.in_v = rin(2);
            hj.push_back(h);
          }
          else if (k == kMlp) mj.push_back({in, p.slot(p.nslot[w], SEG), out_type(P, w)});
          else if (k == kUnembed) {
            uj.push_back((int)pi);
            mj.push_back({in, nullptr, kOutF32});
          }
        }
      }
      if (k == kHead) run_heads(g.layer[nodes[0]], P, hj, nb, last_rows(g.layer[nodes[0]], P, loss));
      else if (k == kMlp) run_mlp(g.layer[nodes[0]], P, mj, nb, last_rows(g.layer[nodes[0]], P, loss));
      else if (k == kUnembed && !mj.empty()) {
        const bool all_rows = !loss;
        const size_t rows = all_rows ? (size_t)nb * g.S : (size_t)nb;
        if (kl_fused_ok(P, loss)) {
          klpart = run_unembed_kl(P, R, mj, nb);
        } else {
          logits = scratch("p_logits", mj.size() * rows * V);
          for (size_t j = 0; j < mj.size(); ++j) mj[j].out = logits + j * rows * V;
          if (loss && unembed_tc_ok(P)) {
            utc = run_unembed_tc(P, mj, nb);
            stats.unembed_rows += utc.rows;
          } else {
            run_unembed(P, mj, nb, all_rows);
          }
        }
        unembed_edges = uj;
      }
      if (!loss) {  // act_diff for edges starting here (patching.cpp:249-256)
        std::vector<RmsJob> rj;
        for (size_t pi = 0; pi < plans.size(); ++pi) {
          auto& p = plans[pi];
          if (p.sv != s) continue;
          for (int i = 0; i < nb; ++i) {
            RmsJob r{};
            if (p.v == g.unembed) {
              size_t j = std::find(unembed_edges.begin(), unembed_edges.end(), (int)pi) - unembed_edges.begin();
              const size_t n = (size_t)g.S * V;
              r.a = logits + j * (size_t)nb * n + i * n;
              r.b = R.logits.as<float>() + i * n;
              r.n = (int64_t)n;
            } else {
              const int ta = out_type(P, p.v), tb = R.otype[p.v];
              const size_t off = (size_t)i * g.S * g.D;  // elements
              auto at = [&](const float* base, int t) {
                return reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(base) +
                                                      off * (t == kOutF32 ? 4 : t == kOutBF16 ? 2 : 1));
              };
              r.a = at(p.slot(p.nslot[p.v], SEG), ta), r.atype = ta;
              r.b = at(R.o(p.v), tb), r.btype = tb;
              r.n = (int64_t)g.S * g.D;
            }
            r.out = d_d + pi * nb + i;
            rj.push_back(r);
          }
        }
        if (!rj.empty()) {
          reserve(up_bytes(rj.size(), sizeof(RmsJob)));
          launch_rms(upload(rj), (int)rj.size(), st);
          launched();
        }
        continue;
      }
      // fold: changed trie values whose last source is at this stage
      std::vector<FoldOp> ops;
      std::vector<FoldProg> progs;
      for (auto& p : plans) {
        if (p.sv > s) continue;
        const int b = (int)ops.size();
        const float* prev = nullptr;
        for (int t : T.by_stage[s]) {
          if (!p.tchg[t]) continue;
          const int pa = T.parent[t];
          const float* a;
          if (pa == 0) a = nullptr;
          else if (p.tchg[pa]) a = p.virt[pa] ? CQG_REG_PREV : p.slot(p.tslot[pa], SEG);
          else a = R.t(pa);
          if (a != nullptr && a != CQG_REG_PREV && a == prev) a = CQG_REG_PREV;
          const int sn = T.src[t];
          const float* bsrc = p.nchg[sn] ? p.slot(p.nslot[sn], SEG) : R.o(sn);
          const int bt = p.nchg[sn] ? out_type(P, sn) : (int)R.otype[sn];
          float* dst = p.virt[t] ? nullptr : p.slot(p.tslot[t], SEG);
          ops.push_back({a, bsrc, dst, bt});
          prev = dst;
        }
        if ((int)ops.size() > b) progs.push_back({b, (int)ops.size()});
      }
      fold(ops, progs, SEG);
    }
    if (loss) {
      // zero for edges whose change never reaches the unembed
      CK(cudaMemsetAsync(d_d, 0, sizeof(double) * plans.size() * nb, st));
      if (!unembed_edges.empty()) {
        const int rows = (int)unembed_edges.size() * nb;
        std::vector<int> item_of(rows);
        for (int r = 0; r < rows; ++r) item_of[r] = r % nb;
        bool ident = true;  // every edge's logits computed, in plan order: write in place
        for (size_t j = 0; j < unembed_edges.size(); ++j) ident = ident && unembed_edges[j] == (int)j;
        double* tmp = ident ? d_d : reinterpret_cast<double*>(scratch("p_kl", (size_t)rows * 2));
        reserve(up_bytes(item_of.size(), sizeof(int)));
        {
          std::unique_ptr<Prof> pf(new Prof(this, metric == 0 ? "kl" : "logitdiff", 0, (double)rows * V * 4.0 * 2.0));
          if (klpart) {
            pf.reset();
            Prof pf2(this, "kl_reduce", 0, (double)rows * unembed_kl_col_tiles(V) * 16.0);
            launch_kl_reduce(klpart, rows, unembed_kl_col_tiles(V), R.psum.as<double>(), nb, tmp, d_nan, st);
          } else if (metric == 0 && utc.rows > 0) {
            if (utc.rows != rows) throw Error(2, "internal: tensor-core unembed row count");
            int* cnt = ucnt.as<int>();
            int* list = reinterpret_cast<int*>(scratch("u_list", (size_t)rows));
            const int* d_item = upload(item_of);
            CK(cudaMemsetAsync(cnt, 0, 4, st));
            launch_kl_cert(logits, R.logits.as<float>(), R.lse.as<double>(), d_item, rows, V, tmp, d_nan,
                           R.prob.as<double>(), utc.anorm, utc.wnorm, g.D,
                           (double)opt_unembed_tol_e9 * 1e-9, list, cnt, st);
            pf.reset();  // (the fallback launches are timed under their own names)
            // flagged rows: the reference's exact logits, then their KL
            GemmJob xj{};
            xj.A = utc.xq, xj.B = utc.wu, xj.C = logits;
            xj.N = V, xj.K = g.D, xj.lda = g.D, xj.ldb = utc.ldu, xj.ldc = V, xj.prec = P.unemb;
            {
              Prof pf2(this, "gemm_unembed_exact_rows");
              launch_gemm_exact_rows(xj, list, cnt, st);
            }
            {
              Prof pf3(this, "kl_exact_rows");
              launch_kl_rows(logits, R.logits.as<float>(), R.lse.as<double>(), d_item, V, tmp, d_nan,
                             R.prob.as<double>(), list, cnt, st);
            }
          } else if (metric == 0)
            launch_kl(logits, R.logits.as<float>(), R.lse.as<double>(), upload(item_of), rows, V,
                      tmp, d_nan, st, R.prob.as<double>());
          else
            launch_logitdiff(logits, R.logits.as<float>(), upload(item_of), d_ans.as<int>(),
                             d_dis.as<int>(), rows, V, tmp, d_nan, st);
        }
        for (size_t j = 0; j < unembed_edges.size() && !ident; ++j)
          CK(cudaMemcpyAsync(d_d + (size_t)unembed_edges[j] * nb, tmp + j * nb, sizeof(double) * nb,
                             cudaMemcpyDeviceToDevice, st));
      }
    }
  }

  size_t mem_budget() {
    if (opt_mem_budget > 0) return (size_t)opt_mem_budget;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    return fr / 3;
  }

  size_t edge_bytes(const EdgePlan& p, int nb, bool loss) const {
    const size_t SEG = segf(nb);
    // arena + per-edge scratch of the widest step (heads: xq + qkv + z; mlp: xq + hid; logits:
    // the last row only under loss metrics, patching.cpp:155-157)
    // (fused unembed + KL: per-tile partials, 4 floats per 128 columns)
    const bool fused = loss && opt_kl_fused && metric == 0 && !opt_unembed_tc;
    const size_t lg = fused ? (size_t)nb * unembed_kl_col_tiles(g.V) * 4 : (size_t)nb * (loss ? 1 : g.S) * g.V;
    size_t scratch_b = std::max({SEG + (size_t)g.H * 4 * nb * g.S * g.dk, 5 * SEG, lg});
    return ((size_t)(1 + p.n_slots) * SEG + scratch_b) * 4;
  }

  // ---- public operations ------------------------------------------------------
  void set_dataset(const int* clean, const int* corrupt, const int* ans, const int* dis, int n,
                   int off, int total, int met) {
    // validate_dataset (patching.cpp:64-81)
    if (n < 1) throw Error(1, "validate_dataset: empty dataset");
    if (met != 0 && met != 1) throw Error(1, "metric must be 0 (kl) or 1 (logitdiff)");
    for (int i = 0; i < n; ++i) {
      const std::string at = "validate_dataset: item " + std::to_string(off + i);
      for (int t = 0; t < g.S; ++t) {
        if (clean[i * g.S + t] < 0 || clean[i * g.S + t] >= g.V)
          throw Error(1, at + ": clean token out of range");
        if (corrupt[i * g.S + t] < 0 || corrupt[i * g.S + t] >= g.V)
          throw Error(1, at + ": corrupt token out of range");
      }
      if (ans[i] < 0 || ans[i] >= g.V || dis[i] < 0 || dis[i] >= g.V)
        throw Error(1, at + ": answer tokens out of range");
      if (ans[i] == dis[i]) throw Error(1, at + ": answer equals distractor");
    }
    if (total < n || off < 0 || off + n > total) throw Error(1, "set_dataset: bad shard bounds");
    B = n, item_off = off, item_total = total, metric = met;
    h_ans.assign(ans, ans + n);
    h_dis.assign(dis, dis + n);
    d_clean.ensure((size_t)n * g.S * 4);
    d_corrupt.ensure((size_t)n * g.S * 4);
    d_ans.ensure((size_t)n * 4);
    d_dis.ensure((size_t)n * 4);
    CK(cudaMemcpyAsync(d_clean.p, clean, (size_t)n * g.S * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_corrupt.p, corrupt, (size_t)n * g.S * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_ans.p, ans, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_dis.p, dis, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    patch_valid = false;
    ++target_gen;
  }

  struct EventPair {  // RAII: no leak on the error paths
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
    }
    ~EventPair() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  };

  void score_edges(const uint8_t* mask, const int* edge_ids, int n, const Policy& base_in,
                   bool per_edge, int mode, double* out) {
    auto t0 = std::chrono::steady_clock::now();
    stats = cqg_stats{};
    kprof.clear();
    if (B == 0) throw Error(1, "score_edges: no dataset (call cqg_set_dataset)");
    if (mode != 0 && mode != 1) throw Error(1, "score_mode must be 0 (loss) or 1 (act)");
    check_policy(base_in);
    for (int i = 0; i < n; ++i) {
      if (edge_ids[i] < 0 || edge_ids[i] >= g.E) throw Error(1, "forward: patch references unknown edge");
      if (!mask[edge_ids[i]])
        throw Error(1, "forward: patch references masked edge " + std::to_string(edge_ids[i]));
    }
    // policy_for_edge (pahq.cpp:198-209) resets the base's targets before it
    // elevates the edge's source, so under per-edge policies no scored pass
    // ever runs the base's own target: every shared run (the masked baseline
    // prefix, the full-graph patch run) uses the target-free base.
    Policy base = base_in;
    if (per_edge) base.th_l = base.th_h = base.tm = -1;
    EventPair ev;
    cudaEvent_t ev0 = ev.a, ev1 = ev.b;
    CK(cudaEventRecord(ev0, st));
    const bool loss = mode == 0;
    DeviceBuf& nanbuf = *pool_buf("nan", 4);
    int* d_nan = nanbuf.as<int>();
    CK(cudaMemsetAsync(d_nan, 0, 4, st));
    ucnt.ensure(8);
    CK(cudaMemsetAsync(ucnt.p, 0, 8, st));
    Trie T;
    T.build(g, mask);
    if (full.size() == 0) full.build(g, nullptr);
    const int base_tok = loss ? 0 : 1, patch_tok = loss ? 1 : 0;
    ensure_patch_run(base, patch_tok, d_nan);

    // groups
    std::map<int, std::vector<int>> by_src;  // source -> indices into edge_ids
    for (int i = 0; i < n; ++i) by_src[per_edge ? g.esrc[edge_ids[i]] : -1].push_back(i);
    std::vector<int> order;
    for (auto& kv : by_src) order.push_back(kv.first);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      const int sa = a < 0 ? 0 : g.stage[a], sb = b < 0 ? 0 : g.stage[b];
      return sa != sb ? sa > sb : a > b;
    });
    bool need_all_rows = false;
    if (!loss)
      for (int i = 0; i < n; ++i) need_all_rows |= g.edst[edge_ids[i]] == g.unembed;
    prepare_run(base_run, T, B, need_all_rows);
    auto tb = std::chrono::steady_clock::now();
    forward_run(base_run, T, base, tokens(base_tok), 0, need_all_rows, d_nan, loss);
    double ms_base = 0, ms_pass = 0;
    std::vector<double> sums(n, 0.0);
    // Per-(edge, item) terms of every group land in one device array (row r =
    // the r-th scored edge); a single D2H at the end, so the host plans the
    // next group while the GPU is still running this one (no per-group sync).
    DeviceBuf& dd = *pool_buf("d_scores", sizeof(double) * (size_t)std::max(n, 1) * B);
    std::vector<int> row_edge;  // row -> index into edge_ids
    row_edge.reserve(n);
    for (size_t oi = 0; oi < order.size(); ++oi) {
      const int src = order[oi];
      const auto& idx = by_src[src];
      const Policy P = per_edge ? policy_for_edge(g, edge_ids[idx[0]], base) : base;
      if (per_edge && oi + 1 < order.size()) prefetch_source(order[oi + 1]);
      check_policy(P);
      if (per_edge && !(P == base)) {
        tb = std::chrono::steady_clock::now();
        forward_run(base_run, T, P, tokens(base_tok), g.stage[src], need_all_rows, d_nan, loss);
      } else if (per_edge && src >= 0 && g.kind[src] == kEmbed) {
        forward_run(base_run, T, P, tokens(base_tok), 0, need_all_rows, d_nan, loss);
      }
      if (opt_profile) CK(cudaStreamSynchronize(st));
      auto tp = std::chrono::steady_clock::now();
      ms_base += std::chrono::duration<double, std::milli>(tp - tb).count();
      // plans, batched under the memory budget
      std::vector<EdgePlan> plans(idx.size());
      for (size_t k = 0; k < idx.size(); ++k) {
        const int e = edge_ids[idx[k]];
        plans[k].e = e, plans[k].s = g.esrc[e], plans[k].v = g.edst[e], plans[k].sv = g.stage[g.edst[e]];
        plans[k].r = g.erecv[e];
        plans[k].pv = patch_value(plans[k].s, policy_for_edge(g, e, base), per_edge, &plans[k].pvt);
      }
      // the per-edge plans are independent host work (O(trie) each): on all
      // host threads, so the host keeps ahead of the GPU on small groups
      std::string plan_err;
#pragma omp parallel for schedule(dynamic, 4) num_threads(plan_threads()) if (idx.size() > 32)
      for (long k = 0; k < (long)idx.size(); ++k) {
        try {
          plan_edge(plans[(size_t)k], T, loss);
        } catch (const std::exception& ex) {
#pragma omp critical
          plan_err = ex.what();
        }
      }
      if (!plan_err.empty()) throw Error(2, plan_err);
      std::vector<size_t> ord(idx.size());
      std::iota(ord.begin(), ord.end(), 0);
      std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return plans[a].sv < plans[b].sv; });
      const size_t budget = mem_budget();
      size_t k0 = 0;
      while (k0 < ord.size()) {
        size_t bytes = 0, k1 = k0;
        while (k1 < ord.size() && (k1 == k0 || bytes + edge_bytes(plans[ord[k1]], B, loss) <= budget)) {
          bytes += edge_bytes(plans[ord[k1]], B, loss);
          ++k1;
        }
        std::vector<EdgePlan> batch;
        for (size_t k = k0; k < k1; ++k) batch.push_back(std::move(plans[ord[k]]));
        run_passes(T, P, base_run, batch, loss, dd.as<double>() + row_edge.size() * (size_t)B, d_nan);
        for (size_t k = k0; k < k1; ++k) row_edge.push_back(idx[ord[k]]);
        stats.passes += (int64_t)(k1 - k0) * B;
        k0 = k1;
      }
      if (opt_profile) CK(cudaStreamSynchronize(st));
      tb = std::chrono::steady_clock::now();
      ms_pass += std::chrono::duration<double, std::milli>(tb - tp).count();
    }
    {
      std::vector<double> hd(row_edge.size() * (size_t)B);
      CK(cudaMemcpyAsync(hd.data(), dd.p, sizeof(double) * hd.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      stats.d2h_bytes += (int64_t)(sizeof(double) * hd.size());
      for (size_t r = 0; r < row_edge.size(); ++r) {
        double acc = 0.0;  // delta_l's sequential item sum (patching.cpp:229-238)
        for (int i = 0; i < B; ++i) acc += hd[r * B + i];
        sums[row_edge[r]] = acc;
      }
    }
    int h_nan = 0;
    CK(cudaMemcpyAsync(&h_nan, d_nan, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (comm) {  // any communicator, including a 1-rank one (tests the NCCL path on one GPU)
      // the NaN flag travels with the partial sums (element n), so a NaN on
      // one rank fails the call on every rank instead of leaving the others
      // blocked in the collective
      DeviceBuf& ar = *pool_buf("allreduce", sizeof(double) * (n + 1));
      sums.push_back(h_nan ? 1.0 : 0.0);
      CK(cudaMemcpyAsync(ar.p, sums.data(), sizeof(double) * (n + 1), cudaMemcpyHostToDevice, st));
      NK(nccl().AllReduce(ar.p, ar.p, (size_t)(n + 1), ncclDouble, ncclSum, comm, st));
      CK(cudaMemcpyAsync(sums.data(), ar.p, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      h_nan = sums[n] != 0.0;
      sums.pop_back();
    }
    if (h_nan) throw Error(2, metric == 0 ? "metric_kl: NaN logits" : "metric_logit_diff: NaN logits");
    for (int i = 0; i < n; ++i) out[i] = sums[i] / (double)item_total;
    if (ucnt.p) {  // patched rows whose logits the certificate sent to the exact path
      int c[2] = {0, 0};
      CK(cudaMemcpy(c, ucnt.p, 8, cudaMemcpyDeviceToHost));
      stats.unembed_exact_rows = c[1];
    }
    if (fix_cnt.p) {  // elements recomputed by the exact fixup
      uint64_t c[2] = {0, 0};
      CK(cudaMemcpy(c, fix_cnt.p, 16, cudaMemcpyDeviceToHost));
      stats.fallback_elems = (int64_t)c[1];
      CK(cudaMemsetAsync(fix_cnt.as<uint32_t>() + 2, 0, 8, st));
    }
    stats.ms_baseline = ms_base;
    stats.ms_passes = ms_pass;
    CK(cudaEventRecord(ev1, st));
    CK(cudaEventSynchronize(ev1));
    float dms = 0;
    CK(cudaEventElapsedTime(&dms, ev0, ev1));
    stats.ms_device = dms;
    if (getenv("CQG_HOST_PROF"))  // where the host's time went (diagnostics only)
      fprintf(stderr, "cqg host: baseline phases %.1f ms, pass phases %.1f ms, blocked on staging %.1f ms, device %.1f ms, launches %lld\n",
              ms_base, ms_pass, host_blocked_ms, (double)dms, (long long)stats.kernel_launches);
    host_blocked_ms = 0;
    collect_profile();
    stats.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }

  DeviceBuf* pool_buf(const std::string& name, size_t bytes) {
    auto& b = pool[name];
    if (!b) b = std::make_unique<DeviceBuf>();
    b->ensure(bytes);
    return b.get();
  }

  // Debug forward of one item (model.cpp:556-757) with direct per-receiver
  // folds (independent of the trie planner; used to cross-check it).
  // One item's forward (model.cpp:556-757) with direct per-receiver folds
  // (independent of the trie planner; used to cross-check it). Node outputs
  // go to O ([N][SEG], FP32 outputs: packed types are not requested here),
  // the receiver inputs to I, the logits ([S][V]) to LG. An edge that the mask
  // drops contributes nothing -- unless absent_src is given, in which case it
  // contributes absent_src's output of its source (circuit_stats'
  // "absent edges read the corrupt run", eval.cpp:960-980).
  void forward_item(const int* d_tok, const uint8_t* mask, const Policy& P, int patch_edge,
                    const float* d_patch, float* O, float* I, float* LG, const float* absent_src) {
    const size_t SEG = segf(1);
    auto input = [&](int w, int c = 0) {  // node w's input (component c of a split head)
      w = g.recv(w, c);                    // (I is indexed by receiver)
      std::vector<FoldOp> ops;
      for (int e : g.in_edges[w]) {
        const float* b;
        if (mask && !mask[e]) {
          if (!absent_src) continue;
          b = absent_src + (size_t)g.esrc[e] * SEG;
        } else {
          b = e == patch_edge ? d_patch : O + (size_t)g.esrc[e] * SEG;
        }
        ops.push_back({ops.empty() ? nullptr : CQG_REG_PREV, b, nullptr});
      }
      if (ops.empty()) {
        CK(cudaMemsetAsync(I + (size_t)w * SEG, 0, SEG * 4, st));
      } else {
        ops.back().dst = I + (size_t)w * SEG;
        fold(ops, {{0, (int)ops.size()}}, SEG);
      }
      return (const float*)(I + (size_t)w * SEG);
    };
    for (int s = 0; s < g.n_stages; ++s) {
      const auto& nodes = g.stage_nodes[s];
      if (nodes.empty()) continue;  // MLP stages of attention-only models
      const int k = g.kind[nodes[0]];
      if (k == kEmbed) run_embed(P, d_tok, O, 1);
      else if (k == kHead) {
        std::vector<HeadIO> hj;
        for (int w : nodes) {
          HeadIO h{input(w), g.head[w], O + (size_t)w * SEG, kOutF32};
          if (g.split) h.in_k = input(w, 1), h.in_v = input(w, 2);
          hj.push_back(h);
        }
        run_heads(g.layer[nodes[0]], P, hj, 1);
      } else if (k == kMlp) run_mlp(g.layer[nodes[0]], P, {{input(nodes[0]), O + (size_t)nodes[0] * SEG, kOutF32}}, 1);
      else run_unembed(P, {{input(g.unembed), LG, kOutF32}}, 1, true);
    }
  }

  void forward_single(const int* tok_host, const uint8_t* mask, const Policy& P, int patch_edge,
                      const float* patch_host, float* outs_host) {
    check_policy(P);
    for (int i = 0; i < g.S; ++i)
      if (tok_host[i] < 0 || tok_host[i] >= g.V) throw Error(1, "forward: token id out of range");
    if (patch_edge >= 0) {
      if (patch_edge >= g.E) throw Error(1, "forward: patch references unknown edge");
      if (mask && !mask[patch_edge]) throw Error(1, "forward: patch references masked edge " + std::to_string(patch_edge));
    }
    const size_t SEG = segf(1);
    DeviceBuf& outs = *pool_buf("f_outs", (size_t)g.N * SEG * 4);
    DeviceBuf& ins = *pool_buf("f_ins", (size_t)g.NR * SEG * 4);
    DeviceBuf& lg = *pool_buf("f_logits", (size_t)g.S * g.V * 4);
    DeviceBuf& tk = *pool_buf("f_tok", (size_t)g.S * 4);
    DeviceBuf& pv = *pool_buf("f_patch", SEG * 4);
    CK(cudaMemcpyAsync(tk.p, tok_host, (size_t)g.S * 4, cudaMemcpyHostToDevice, st));
    if (patch_edge >= 0) CK(cudaMemcpyAsync(pv.p, patch_host, SEG * 4, cudaMemcpyHostToDevice, st));
    forward_item(tk.as<int>(), mask, P, patch_edge, pv.as<float>(), outs.as<float>(), ins.as<float>(),
                 lg.as<float>(), nullptr);
    CK(cudaMemcpyAsync(outs_host, outs.p, (size_t)(g.N - 1) * SEG * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(outs_host + (size_t)(g.N - 1) * SEG, lg.p, (size_t)g.S * g.V * 4,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }

  // circuit_stats (eval.cpp:960-985) for the local items at FP32: the clean,
  // corrupt and circuit runs' last-row logit differences. The circuit run
  // keeps the full graph and feeds every absent edge its source's output from
  // the corrupt run.
  void circuit_stats(const uint8_t* mask, double* clean_ld, double* corrupt_ld, double* circuit_ld) {
    if (B == 0) throw Error(1, "circuit_stats: no dataset (call cqg_set_dataset)");
    if (!mask) throw Error(1, "circuit_stats: null mask");
    const Policy P = Policy::from(cqg_policy{2, 2, 2, 2, 0, -1, -1, -1});  // all_fp32
    const size_t SEG = segf(1);
    DeviceBuf& oc = *pool_buf("cs_corr", (size_t)g.N * SEG * 4);
    DeviceBuf& o = *pool_buf("f_outs", (size_t)g.N * SEG * 4);
    DeviceBuf& ins = *pool_buf("f_ins", (size_t)g.NR * SEG * 4);
    DeviceBuf& lg = *pool_buf("f_logits", (size_t)g.S * g.V * 4);
    std::vector<float> row(g.V);
    auto ld = [&](int i) {  // metric_logit_diff of the last row (patching.cpp:140-149)
      CK(cudaMemcpyAsync(row.data(), lg.as<float>() + (size_t)(g.S - 1) * g.V, (size_t)g.V * 4,
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (float x : row)
        if (x != x) throw Error(2, "metric_logit_diff: NaN logits");
      return (double)row[h_ans[i]] - (double)row[h_dis[i]];
    };
    for (int i = 0; i < B; ++i) {
      const int* clean = d_clean.as<int>() + (size_t)i * g.S;
      const int* corr = d_corrupt.as<int>() + (size_t)i * g.S;
      forward_item(corr, nullptr, P, -1, nullptr, oc.as<float>(), ins.as<float>(), lg.as<float>(), nullptr);
      corrupt_ld[i] = ld(i);
      forward_item(clean, nullptr, P, -1, nullptr, o.as<float>(), ins.as<float>(), lg.as<float>(), nullptr);
      clean_ld[i] = ld(i);
      forward_item(clean, mask, P, -1, nullptr, o.as<float>(), ins.as<float>(), lg.as<float>(), oc.as<float>());
      circuit_ld[i] = ld(i);
    }
  }


  // iter0_raw: iteration-1 scores of the full mask's sweep order (after the
  // heads_only filter), already computed -- they do not depend on tau, so a
  // threshold sweep scores them once (roc_sweep below).
  void run_acdc(const cqg_prune& c, int* steps, uint8_t* final_mask, double* last_score, int* n_rec,
                int* rs, int* re, double* rsc, uint8_t* rk, int cap, const double* iter0_raw = nullptr) {
    // PruneConfig::validate (acdc.cpp:14-21)
    if (!(c.tau >= 0.0)) throw Error(1, "PruneConfig: tau must be >= 0");
    if (c.max_steps < 1) throw Error(1, "PruneConfig: max_steps must be >= 1");
    if (!(c.min_change_rate >= 0.0)) throw Error(1, "PruneConfig: min_change_rate must be >= 0");
    if (!(c.act_floor >= 0.0)) throw Error(1, "PruneConfig: act_floor must be >= 0");
    const Policy base = Policy::from(c.base);
    std::vector<uint8_t> mask(g.E, 1);
    std::fill(last_score, last_score + g.E, 0.0);
    int t = 0, k = 0;
    bool keep_going = true;
    do {
      std::vector<int> order = g.sweep_order(mask);
      if (c.heads_only)
        order.erase(std::remove_if(order.begin(), order.end(),
                                   [&](int e) { return g.kind[g.esrc[e]] != kHead; }),
                    order.end());
      if (order.empty()) break;
      std::vector<double> raw(order.size());
      if (t == 0 && iter0_raw)
        std::copy(iter0_raw, iter0_raw + order.size(), raw.begin());
      else
        score_edges(mask.data(), order.data(), (int)order.size(), base, c.per_edge_policy != 0, c.mode,
                    raw.data());
      int removed = 0;
      for (size_t i = 0; i < order.size(); ++i) {
        double s = raw[i];
        if (c.mode == 1 && s < c.act_floor) s = 0.0;
        const bool keep = !(s < c.tau);
        if (k < cap) rs[k] = t, re[k] = order[i], rsc[k] = s, rk[k] = keep ? 1 : 0;
        ++k;
        last_score[order[i]] = s;
        if (!keep) {
          mask[order[i]] = 0;
          ++removed;
        }
      }
      ++t;
      const double change_rate = (double)removed / (double)order.size();
      keep_going = removed > 0 && change_rate > c.min_change_rate;
    } while (t < c.max_steps && std::count(mask.begin(), mask.end(), 1) > 0 && keep_going);
    std::copy(mask.begin(), mask.end(), final_mask);
    *steps = t;
    *n_rec = k;
  }

  std::vector<int> first_order(const cqg_prune& c) const {
    std::vector<int> order = g.sweep_order(std::vector<uint8_t>(g.E, 1));
    if (c.heads_only)
      order.erase(std::remove_if(order.begin(), order.end(),
                                 [&](int e) { return g.kind[g.esrc[e]] != kHead; }),
                  order.end());
    return order;
  }

  // roc_sweep (eval.cpp:1193-1226): run_acdc at every threshold, TPR/FPR of
  // the final mask against the ground truth, AUC (auc_from_points,
  // eval.cpp:1149-1166). Iteration 1 runs on the full mask for every tau, so
  // its scores are computed once and shared; later iterations run per tau.
  double roc_sweep(const cqg_prune& c, const double* taus, int n, const int* gt, int n_gt, double* tpr,
                   double* fpr, int* kept, int* steps) {
    if (n < 1) throw Error(1, "roc_sweep: no thresholds");
    std::vector<uint8_t> is_gt(g.E, 0);
    for (int i = 0; i < n_gt; ++i) {
      if (gt[i] < 0 || gt[i] >= g.E) throw Error(1, "roc_sweep: ground-truth edge out of range");
      is_gt[gt[i]] = 1;
    }
    const int n_pos = (int)std::count(is_gt.begin(), is_gt.end(), 1), n_neg = g.E - n_pos;
    if (n_pos == 0 || n_neg == 0) throw Error(1, "roc_sweep: degenerate ground truth");
    cqg_prune c0 = c;
    c0.tau = taus[0];
    if (!(c0.tau >= 0.0)) throw Error(1, "PruneConfig: tau must be >= 0");
    const std::vector<int> order = first_order(c);
    std::vector<double> raw0(order.size());
    if (!order.empty())
      score_edges(std::vector<uint8_t>(g.E, 1).data(), order.data(), (int)order.size(), Policy::from(c.base),
                  c.per_edge_policy != 0, c.mode, raw0.data());
    std::vector<uint8_t> fm(g.E);
    std::vector<double> ls(g.E);
    struct Pt { double tpr, fpr; };
    std::vector<Pt> pts(n);
    for (int i = 0; i < n; ++i) {
      cqg_prune ci = c;
      ci.tau = taus[i];
      int st = 0, nr = 0;
      run_acdc(ci, &st, fm.data(), ls.data(), &nr, nullptr, nullptr, nullptr, nullptr, 0, raw0.data());
      int tp = 0, fp = 0, k = 0;
      for (int e = 0; e < g.E; ++e) {
        if (!fm[e]) continue;
        ++k;
        (is_gt[e] ? tp : fp) += 1;
      }
      pts[i] = {(double)tp / n_pos, (double)fp / n_neg};
      if (tpr) tpr[i] = pts[i].tpr;
      if (fpr) fpr[i] = pts[i].fpr;
      if (kept) kept[i] = k;
      if (steps) steps[i] = st;
    }
    std::sort(pts.begin(), pts.end(), [](const Pt& a, const Pt& b) {
      return a.fpr != b.fpr ? a.fpr < b.fpr : a.tpr < b.tpr;
    });
    double x = 0.0, y = 0.0, area = 0.0;
    for (const Pt& p : pts) {
      if (p.tpr <= y) continue;
      if (p.fpr > x) {
        area += (p.fpr - x) * y;
        x = p.fpr;
      }
      y = p.tpr;
    }
    return area + (1.0 - x) * y;
  }
};

std::unique_ptr<Engine> make_engine(const cqg_config& cfg, const float* const* mats, int device) {
  auto E = std::make_unique<Engine>(cfg);
  E->device = device;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&E->st, cudaStreamNonBlocking));
  const Graph& g = E->g;
  const int64_t D = g.D, V = g.V, S = g.S;
  for (int m = 0; m < g.n_mats(); ++m) {
    const int w = E->mat_kind(m);
    int64_t n;
    switch (w) {
      case 0: n = V * D; break;
      case 1: n = S * D; break;
      case 2: case 3: case 8: case 9: case 12: case 13: n = D; break;
      case 10: case 11: n = 4 * D * D; break;
      case 14: n = D * V; break;
      default: n = D * D;
    }
    E->msize.push_back(n);
    E->master.push_back(std::make_unique<DeviceBuf>());
    E->master.back()->ensure(n * 4);
    CK(cudaMemcpy(E->master.back()->p, mats[m], n * 4, cudaMemcpyHostToDevice));
  }
  return E;
}

}  // namespace cqg

// ===========================================================================
// C ABI
// ===========================================================================
using cqg::Engine;
using cqg::Error;

struct cqg_ctx {
  std::unique_ptr<Engine> e;
};

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    cqg::g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    cqg::g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    cqg::g_err = e.what();
    return 2;
  }
}

extern "C" {

const char* cqg_last_error(void) { return cqg::g_err.c_str(); }

uint64_t cqg_fnv1a64(const void* data, size_t n) {
  const uint8_t* p = static_cast<const uint8_t*>(data);
  uint64_t h = 14695981039346656037ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

int cqg_create(const cqg_config* cfg, const float* const* mats, int device, cqg_ctx** out) {
  return guarded([&] {
    if (!cfg || !mats || !out) throw Error(1, "cqg_create: null argument");
    auto* c = new cqg_ctx;
    try {
      c->e = cqg::make_engine(*cfg, mats, device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void cqg_destroy(cqg_ctx* ctx) { delete ctx; }

int cqg_set_dataset(cqg_ctx* ctx, const int32_t* clean, const int32_t* corrupt, const int32_t* answer,
                    const int32_t* distractor, int n_items, int item_offset, int item_total, int metric) {
  return guarded([&] {
    if (!ctx) throw Error(1, "null context");
    ctx->e->set_dataset(clean, corrupt, answer, distractor, n_items, item_offset,
                        item_total > 0 ? item_total : n_items, metric);
  });
}

int cqg_get_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    NK(cqg::nccl().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof id);
  });
}

int cqg_init_comm(cqg_ctx* ctx, const void* unique_id, int rank, int world) {
  return guarded([&] {
    if (!ctx) throw Error(1, "null context");
    if (world < 1 || rank < 0 || rank >= world) throw Error(1, "cqg_init_comm: bad rank/world");
    auto& E = *ctx->e;
    E.rank = rank, E.world = world;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    CK(cudaSetDevice(E.device));
    NK(cqg::nccl().CommInitRank(&E.comm, world, id, rank));
  });
}

int cqg_score_edges(cqg_ctx* ctx, const uint8_t* mask, const int32_t* edge_ids, int n,
                    const cqg_policy* base, int per_edge_policy, int score_mode, double* scores_out) {
  return guarded([&] {
    if (!ctx || !mask || (!edge_ids && n > 0) || !base || (!scores_out && n > 0))
      throw Error(1, "cqg_score_edges: null argument");
    CK(cudaSetDevice(ctx->e->device));
    ctx->e->score_edges(mask, edge_ids, n, cqg::Policy::from(*base), per_edge_policy != 0, score_mode,
                        scores_out);
  });
}

int cqg_run_acdc(cqg_ctx* ctx, const cqg_prune* cfg, int* steps, uint8_t* final_mask, double* last_score,
                 int* n_rec, int32_t* rec_step, int32_t* rec_edge, double* rec_score, uint8_t* rec_kept,
                 int rec_cap) {
  return guarded([&] {
    if (!ctx || !cfg) throw Error(1, "cqg_run_acdc: null argument");
    CK(cudaSetDevice(ctx->e->device));
    ctx->e->run_acdc(*cfg, steps, final_mask, last_score, n_rec, rec_step, rec_edge, rec_score,
                     rec_kept, rec_cap);
  });
}

int cqg_roc_sweep(cqg_ctx* ctx, const cqg_prune* cfg, const double* taus, int n_taus,
                  const int32_t* ground_truth, int n_gt, double* tpr, double* fpr, int32_t* kept,
                  int32_t* steps, double* auc) {
  return guarded([&] {
    if (!ctx || !cfg || !taus || (!ground_truth && n_gt > 0) || !auc)
      throw Error(1, "cqg_roc_sweep: null argument");
    CK(cudaSetDevice(ctx->e->device));
    *auc = ctx->e->roc_sweep(*cfg, taus, n_taus, ground_truth, n_gt, tpr, fpr, kept, steps);
  });
}

int cqg_quantize_matrix(cqg_ctx* ctx, int matrix_index, int precision, int low_mode, float* out_host) {
  return guarded([&] {
    if (!ctx) throw Error(1, "null context");
    auto& E = *ctx->e;
    if (matrix_index < 0 || matrix_index >= E.g.n_mats()) throw Error(1, "cqg_quantize_matrix: bad matrix index");
    if (precision < 0 || precision > 2 || low_mode < 0 || low_mode > 2)
      throw Error(1, "cqg_quantize_matrix: bad precision/mode");
    CK(cudaSetDevice(E.device));
    const float* d = E.W(matrix_index, precision, low_mode);
    CK(cudaMemcpyAsync(out_host, d, E.msize[matrix_index] * 4, cudaMemcpyDeviceToHost, E.st));
    CK(cudaStreamSynchronize(E.st));
  });
}

int cqg_forward(cqg_ctx* ctx, const int32_t* tokens, const uint8_t* mask, const cqg_policy* pol,
                int patch_edge, const float* patch_value, float* outs_host) {
  return guarded([&] {
    if (!ctx || !tokens || !pol || !outs_host) throw Error(1, "cqg_forward: null argument");
    CK(cudaSetDevice(ctx->e->device));
    ctx->e->forward_single(tokens, mask, cqg::Policy::from(*pol), patch_edge, patch_value, outs_host);
  });
}

int cqg_circuit_stats(cqg_ctx* ctx, const uint8_t* mask, double* clean_ld, double* corrupt_ld,
                      double* circuit_ld) {
  return guarded([&] {
    if (!ctx || !mask || !clean_ld || !corrupt_ld || !circuit_ld) throw Error(1, "cqg_circuit_stats: null argument");
    CK(cudaSetDevice(ctx->e->device));
    ctx->e->circuit_stats(mask, clean_ld, corrupt_ld, circuit_ld);
  });
}

int cqg_graph_info(const cqg_config* cfg, int* n_nodes, int* n_edges) {
  return guarded([&] {
    cqg::Graph g(*cfg);
    *n_nodes = g.N;
    *n_edges = g.E;
  });
}

int cqg_graph_edge_comp(const cqg_config* cfg, int32_t* comp) {
  return guarded([&] {
    if (!cfg || !comp) throw cqg::Error(1, "cqg_graph_edge_comp: null argument");
    cqg::Graph g(*cfg);
    for (int e = 0; e < g.E; ++e) comp[e] = g.recv_comp[g.erecv[e]];
  });
}

int cqg_graph_edges(const cqg_config* cfg, int32_t* src, int32_t* dst) {
  return guarded([&] {
    cqg::Graph g(*cfg);
    for (int e = 0; e < g.E; ++e) src[e] = g.esrc[e], dst[e] = g.edst[e];
  });
}

int cqg_last_stats(cqg_ctx* ctx, cqg_stats* out) {
  return guarded([&] {
    if (!ctx || !out) throw Error(1, "null argument");
    *out = ctx->e->stats;
  });
}

int cqg_profile_count(cqg_ctx* ctx) { return ctx ? (int)ctx->e->kprof.size() : 0; }

int cqg_profile_entry(cqg_ctx* ctx, int i, char* name64, double* ms, double* flops, double* bytes,
                      int64_t* launches) {
  return guarded([&] {
    if (!ctx || i < 0 || i >= (int)ctx->e->kprof.size()) throw Error(1, "cqg_profile_entry: bad index");
    auto it = ctx->e->kprof.begin();
    std::advance(it, i);
    std::snprintf(name64, 64, "%s", it->first.c_str());
    *ms = it->second.ms, *flops = it->second.flops, *bytes = it->second.bytes;
    *launches = it->second.launches;
  });
}

int cqg_set_option(cqg_ctx* ctx, const char* key, int64_t value) {
  return guarded([&] {
    if (!ctx || !key) throw Error(1, "null argument");
    std::string k(key);
    if (k == "exact") ctx->e->opt_exact = value;
    else if (k == "packed") ctx->e->opt_packed = value;
    else if (k == "fix_cpi") {
      if (value != 0 && value != 1 && value != 2 && value != 4) throw Error(1, "fix_cpi must be 0, 1, 2 or 4");
      ctx->e->opt_fix_cpi = value;
    }
    else if (k == "exact_x2") cqg::g_exact_x2 = (int)value;
    else if (k == "profile") ctx->e->opt_profile = value;
    else if (k == "fix_blk") ctx->e->opt_fix_blk = value;
    else if (k == "fix_blk_min") ctx->e->opt_fix_blk_min = value;
    else if (k == "kl_fused") ctx->e->opt_kl_fused = value;
    else if (k == "fix_dry") ctx->e->opt_fix_dry = value;
    else if (k == "fix_g") {
      if (value < 0 || value > 2) throw Error(1, "fix_g must be 0, 1 or 2");
      ctx->e->opt_fix_g = value;
    }
    else if (k == "prefetch") ctx->e->opt_prefetch = value;
    else if (k == "mem_budget") ctx->e->opt_mem_budget = value;
    else if (k == "unembed_tc") ctx->e->opt_unembed_tc = value;
    else if (k == "unembed_tol_e9") {
      // 0: every row fails the certificate (all logits exact; a test hook)
      if (value < 0) throw Error(1, "unembed_tol_e9 must be >= 0");
      ctx->e->opt_unembed_tol_e9 = value;
    }
    else throw Error(1, "cqg_set_option: unknown key " + k);
  });
}

}  // extern "C"
