// Per-rank executor of one asymmetric-parallel training step.
//
// One process per GPU.  The rank's role (pipeline, stage, TP index, shard
// ranges, samples, PP peers, DP buckets) comes from build_layout (plan.cpp).
// The step is:
//   1F1B over the pipeline's micro-batches (Megatron non-interleaved order;
//   reference prices it as fill + (n-1)*bottleneck, cost_model.cpp:96-111):
//     fwd per layer: RMSNorm -> QKV GEMM (column shard) -> RoPE -> causal
//       attention (batched tcgen05 GEMMs + warp softmax) -> O GEMM (row shard)
//       -> TP allreduce -> RMSNorm -> gate/up GEMM -> SwiGLU -> down GEMM ->
//       TP allreduce;  last stage: final norm, vocab-parallel LM head + CE.
//     bwd mirrors it (dgrad + wgrad GEMMs, TP allreduce of input grads).
//     PP activations / grads move with NCCL send/recv on the world comm.
//   DP: per-tensor scale by (batch_i / global_batch) / multiplicity fused with
//     the bf16 cast, then NCCL allreduce per chunk-matched bucket.
//   AdamW on the fp32 master shard, refreshing the bf16 copy.
// Every kernel is ours (csrc/*.cu); there is no host compute path.
#include "executor.hpp"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>

#include "attention.h"
#include "gemm.h"
#include "kernels.h"
#include "nlohmann/json.hpp"

namespace hexexec {

using ojson = nlohmann::ordered_json;

#define HX_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                      std::to_string(__LINE__) + ")");                                     \
  } while (0)

#define HX_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      throw NcclError(std::string(#x) + ": " + ncclGetErrorString(r_) + " (" __FILE__ ":" + \
                      std::to_string(__LINE__) + ")");                                    \
  } while (0)

ExecConfig parse_exec_config(const std::string& text) {
  ExecConfig c;
  if (text.empty()) return c;
  ojson j = ojson::parse(text, nullptr, false);
  if (j.is_discarded() || !j.is_object()) throw ParseError("exec config: not a JSON object");
  for (auto& [k, v] : j.items()) {
    try {
      if (k == "seed") c.seed = v.get<uint64_t>();
      else if (k == "lr") c.lr = v.get<float>();
      else if (k == "beta1") c.beta1 = v.get<float>();
      else if (k == "beta2") c.beta2 = v.get<float>();
      else if (k == "eps") c.eps = v.get<float>();
      else if (k == "weight_decay") c.weight_decay = v.get<float>();
      else if (k == "sm_cap") c.sm_cap = v.get<std::string>();
      else if (k == "dp_comm_dtype") c.dp_comm_dtype = v.get<std::string>();
      else if (k == "validate_only") c.validate_only = v.get<bool>();
      else if (k == "profile_gemm") c.profile_gemm = v.get<bool>();
      else if (k == "cuda_graph") c.cuda_graph = v.get<bool>();
      else if (k == "attention") c.attention = v.get<std::string>();
      else if (k == "dp_overlap") c.dp_overlap = v.get<bool>();
      else if (k == "gemm_split") c.gemm_split = v.get<bool>();
      else if (k == "recompute") c.recompute = v.get<bool>();
      else if (k == "pp_protocol") c.pp_protocol = v.get<std::string>();
      else if (k == "tp_reduce") c.tp_reduce = v.get<std::string>();
      else if (k == "tp_direction") c.tp_direction = v.get<std::string>();
      else if (k == "graph_gemm_events") c.graph_gemm_events = v.get<bool>();
      else if (k == "fuse_swiglu") c.fuse_swiglu = v.get<bool>();
      else if (k == "wgrad_group") c.wgrad_group = v.get<int>();
      else if (k == "pdl") c.pdl = v.get<bool>();
      else if (k == "tp_pull") c.tp_pull = v.get<std::string>();
      else if (k == "fuse_rope") c.fuse_rope = v.get<bool>();
      else if (k == "pp_dtype") c.pp_dtype = v.get<std::string>();
      else throw ParseError("exec config: unknown key '" + k + "'");
    } catch (const nlohmann::json::exception& e) {
      throw ParseError("exec config: bad value for '" + k + "'");
    }
  }
  if (c.sm_cap != "green" && c.sm_cap != "cta" && c.sm_cap != "none")
    throw ParseError("exec config: sm_cap must be green|cta|none");
  if (c.attention != "fused" && c.attention != "unfused")
    throw ParseError("exec config: attention must be fused|unfused");
  if (c.dp_comm_dtype != "bf16" && c.dp_comm_dtype != "fp32")
    throw ParseError("exec config: dp_comm_dtype must be bf16|fp32");
  if (c.pp_protocol != "direct" && c.pp_protocol != "leader")
    throw ParseError("exec config: pp_protocol must be direct|leader");
  if (c.tp_reduce != "peer" && c.tp_reduce != "nccl")
    throw ParseError("exec config: tp_reduce must be peer|nccl");
  if (c.tp_pull != "sm" && c.tp_pull != "ce")
    throw ParseError("exec config: tp_pull must be sm|ce");
  if (c.pp_dtype != "bf16" && c.pp_dtype != "fp32")
    throw ParseError("exec config: pp_dtype must be bf16|fp32");
  if (c.tp_direction != "auto" && c.tp_direction != "push")
    throw ParseError("exec config: tp_direction must be auto|push");
  return c;
}

namespace {

// bump allocator over one device allocation
class Arena {
 public:
  void reserve(size_t bytes) { total_ += align(bytes); }
  void commit() {
    if (!total_) return;
    cudaError_t e = cudaMalloc(&base_, total_);
    if (e == cudaErrorMemoryAllocation) {
      (void)cudaGetLastError();
      throw Infeasible("plan does not fit this device: rank needs " +
                       std::to_string(total_ >> 20) + " MiB of HBM");
    }
    HX_CUDA(e);
  }
  template <typename T>
  T* take(size_t count) {
    size_t b = align(count * sizeof(T));
    if (used_ + b > total_) throw std::runtime_error("arena overflow");
    T* p = reinterpret_cast<T*>(static_cast<char*>(base_) + used_);
    used_ += b;
    return p;
  }
  void release() {
    if (base_) cudaFree(base_);
    base_ = nullptr;
  }
  size_t total() const { return total_; }

 private:
  static size_t align(size_t b) { return (b + 255) / 256 * 256; }
  void* base_ = nullptr;
  size_t total_ = 0, used_ = 0;
};

struct LayerActs {
  float* x_mid;     // [M, H]
  bf16* xn;         // [M, H]
  float* rstd1;     // [M]
  bf16* qkv;        // [M, 3 d nh]
  bf16* P;          // [mb * nh, S, S]  (unfused attention only)
  float* lse;       // [mb * nh, S]     (fused attention)
  bf16* attn;       // [M, d nh]
  bf16* hn;         // [M, H]
  float* rstd2;     // [M]
  bf16* gu;         // [M, 2 F]
  bf16* act;        // [M, F]
};

struct Slot {
  std::vector<float*> x;  // nl + 1 residual-stream buffers, x[0] = stage input
  std::vector<LayerActs> layers;
  bf16* xf = nullptr;     // last stage: final-norm output
  float* rstdf = nullptr;
  bf16* dlogits = nullptr;
};

struct TensorPtrs {
  float* p32 = nullptr;
  bf16* p16 = nullptr;
  float* g32 = nullptr;
  int64_t rows = 0, cols = 0, row0 = 0, count = 0, offset = 0;
  int spec = -1;
};

}  // namespace

class Executor {
 public:
  Layout L;
  ExecConfig cfg;
  int rank = 0, world = 1, device = 0;
  RankRole role;
  // model shapes for this rank
  int64_t H = 0, S = 0, d = 0, nh = 0, F = 0, Vr = 0, v0 = 0, mb = 0, M = 0, nl = 0;
  int64_t qkvw = 0, kr = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  CUgreenCtx green = nullptr;
  int sm_total = 0, sm_applied = 0;
  std::string sm_mode = "none";
  ncclComm_t world_comm = nullptr;
  std::vector<ncclComm_t> comms;  // per Layout::comm_sets index (null if not a member)
  Arena arena;
  // flat parameter state
  float *P32 = nullptr, *G32 = nullptr, *Mo = nullptr, *Vo = nullptr;
  bf16 *P16 = nullptr, *G16 = nullptr;
  std::map<std::string, TensorPtrs> named;
  // per-layer tensor pointers (local layer index)
  struct LayerW {
    TensorPtrs attn_norm, wqkv, wo, mlp_norm, wgu, wdown;
  };
  std::vector<LayerW> lw;
  TensorPtrs embed, final_norm, lm_head;
  // activations
  std::vector<Slot> slots;
  int n_slots = 0;
  // scratch
  float *scores = nullptr, *dP = nullptr, *logits = nullptr;
  bf16 *dS = nullptr, *ypart = nullptr, *da = nullptr, *dgu = nullptr, *dattn = nullptr,
       *dqkv = nullptr, *dy16 = nullptr;
  float *dx[2] = {nullptr, nullptr}, *ce_scr = nullptr, *loss_acc = nullptr, *loss_host = nullptr;
  bf16* dxb = nullptr;
  float *delta_ = nullptr, *dq_acc_ = nullptr;
  float* gemm_ws_ = nullptr;  // zero between GEMMs (the kernel leaves it zero)
  int* gemm_cnt_ = nullptr;
  float* dg_part_ = nullptr;
  void* embed_keys_ = nullptr;
  LayerActs rc_acts_{};  // recompute: the one shared activation set
  int32_t* tokens = nullptr;
  int32_t* tokens_pinned = nullptr;
  float* idle_loss_ = nullptr;
  // TP exchange over peer memory (tp_reduce = "peer"): local buffer = 2 ring
  // buffers x tp slots x [M, H] bf16 + flags[tp]; peers' buffers IPC-mapped
  uint8_t* xbuf_ = nullptr;
  uint8_t* xpeer_[4] = {nullptr, nullptr, nullptr, nullptr};
  TpPeers tpp_{};
  size_t xflag_off_ = 0;
  unsigned xop_ = 0;
  bool tp_peer_ = false;
  float2* rope_tab_ = nullptr;  // RoPE (cos, sin) [S][d/2] for the QKV epilogue
  int tp_crit_ = -1;  // TP index of the critical (slowest) rank, or -1
  // Weight-gradient grouping (wgrad_group): the operands of the four layer
  // weight-gradient GEMMs (and the LM head's) of G consecutive micro-batches
  // are kept token-concatenated, and one GEMM with K = G*M per weight runs at
  // the group's last backward -- one fp32 store instead of G fp32 reduce-adds
  // of the gradient.  nbuf ring buffers of G micro-batch rows each.
  struct WStash {
    bf16 *act, *hn, *attn, *xn, *dxob, *dgu, *dxmb, *dqkv;
  };
  int64_t wg_ = 1, wg_nbuf_ = 1;
  std::vector<WStash> wst_;      // [nbuf][nl]
  std::vector<bf16*> wst_xf_, wst_dlog_;  // [nbuf]
  int64_t wg_bytes_per_mb() const {
    int64_t w = nl * (3 * F + 4 * H + kr + qkvw);
    if (role.last_stage) w += H + Vr;
    return 2 * M * w;
  }
  WStash& ws(int64_t l, int64_t mbi) { return wst_[size_t(((mbi / wg_) % wg_nbuf_) * nl + l)]; }
  bf16* wrow(bf16* base, int64_t mbi, int64_t width) const { return base + (mbi % wg_) * M * width; }
  bool wg_end(int64_t mbi) const { return mbi % wg_ == wg_ - 1 || mbi == role.n_mb - 1; }
  float* recv_buf = nullptr;  // fwd activations received (fp32 [M,H]) go into slot x[0]
  int64_t step_index = 0;
  // stats
  cudaEvent_t ev_eager_[6] = {}, ev_graph_[6] = {};
  cudaEvent_t* ev = ev_eager_;  // phase events of the mode that ran last
  cudaEvent_t tmr_[2] = {};
  float phase_ms[5] = {0, 0, 0, 0, 0};
  // kernel launches of ours per step; copies_step counts the step's memset /
  // memcpy nodes separately (not kernels)
  int64_t launches_step = 0, launches_total = 0, copies_step = 0;
  int64_t nccl_calls_step = 0;
  float last_loss = 0.f;

  ~Executor() { teardown(); }

  void teardown() {
    // drain the stream and drop the captured graph (it holds NCCL persistent
    // work) before the communicators: destroying a communicator still
    // referenced by a graph exec blocks
    if (stream) cudaStreamSynchronize(stream);
    if (cstream) cudaStreamSynchronize(cstream);
    if (gexec_) cudaGraphExecDestroy(gexec_);
    gexec_ = nullptr;
    for (auto& c : comms)
      if (c) ncclCommFinalize(c);
    if (world_comm) ncclCommFinalize(world_comm);
    for (auto& c : comms)
      if (c) ncclCommDestroy(c);
    comms.clear();
    if (world_comm) ncclCommDestroy(world_comm);
    world_comm = nullptr;
    arena.release();
    for (auto& p : xpeer_)
      if (p) cudaIpcCloseMemHandle(p), p = nullptr;
    if (xbuf_) cudaFree(xbuf_);
    xbuf_ = nullptr;
    if (idle_loss_) cudaFree(idle_loss_);
    idle_loss_ = nullptr;
    if (tokens_pinned) cudaFreeHost(tokens_pinned);
    tokens_pinned = nullptr;
    if (loss_host) cudaFreeHost(loss_host);
    loss_host = nullptr;
    for (auto& e : ev_eager_)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_graph_)
      if (e) cudaEventDestroy(e);
    for (auto& e : tmr_)
      if (e) cudaEventDestroy(e);
    for (auto& r : gemm_pool_) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    gemm_pool_.clear();
    for (auto& e : mark_pool_) cudaEventDestroy(e);
    mark_pool_.clear();
    for (auto& r : graph_recs_) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    graph_recs_.clear();
    graph_shapes_.clear();
    for (auto& m : gmarks_) cudaEventDestroy(m.ev);
    gmarks_.clear();
    if (gexec_) cudaGraphExecDestroy(gexec_);
    gexec_ = nullptr;
    for (auto& g : groups_)
      if (g.ready) cudaEventDestroy(g.ready);
    groups_.clear();
    if (join_ev_) cudaEventDestroy(join_ev_);
    join_ev_ = nullptr;
    if (own_cstream && cstream) cudaStreamDestroy(cstream);
    cstream = nullptr;
    if (own_stream && stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }

  // ------------------------------------------------------------ setup
  void init(const std::string& cj, const std::string& mj, const std::string& pj,
            const std::string& xj, int r, int w, int dev, const void* uid, size_t uid_len) {
    cfg = parse_exec_config(xj);
    L = build_layout(cj, mj, pj);
    if (w != L.world_size)
      throw InvalidArgument("world size " + std::to_string(w) + " does not match the cluster's " +
                            std::to_string(L.world_size) + " devices");
    if (r < 0 || r >= w) throw InvalidArgument("world rank out of range");
    rank = r;
    world = w;
    device = dev;
    role = L.roles[size_t(r)];
    const Model& m = L.model;
    H = m.hidden_dim;
    S = m.seq_len;
    d = m.head_dim();
    if (role.active) {
      nh = role.heads.size();
      F = 64 * role.ffn_chunks.size();
      Vr = 64 * role.vocab_chunks.size();
      v0 = 64 * role.vocab_chunks.begin;
      mb = role.micro_batch;
      M = mb * S;
      if (M > (int64_t(1) << 30))  // 32-bit row indices in the kernels
        throw LimitExceeded("micro_batch * seq_len = " + std::to_string(M) +
                            " tokens exceeds the per micro-batch limit");
      nl = role.layer_count;
      qkvw = 3 * d * nh;
      kr = d * nh;
    }
    // the fused tcgen05 attention kernels cover d = 64 / 128; the plan admits
    // d up to 256 (multiples of 64): those models run the unfused GEMM +
    // softmax attention on the GPU instead of failing at the first step
    if (cfg.attention == "fused" && d != 64 && d != 128) {
      cfg.attention = "unfused";
      attention_note_ = "unfused (fused kernels cover head_dim 64 / 128; head_dim " +
                        std::to_string(d) + ")";
    }
    if (cfg.validate_only) {
      // host-only dry run: size the per-rank arena (no device needed)
      if (role.active) allocate();
      return;
    }

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw CudaError("no CUDA device available (there is no CPU path)");
    HX_CUDA(cudaSetDevice(dev));
    HX_CUDA(cudaDeviceGetAttribute(&sm_total, cudaDevAttrMultiProcessorCount, dev));
    setup_stream();
    gemm_set_pdl(cfg.pdl ? 1 : 0);
    for (auto& e : ev_eager_) HX_CUDA(cudaEventCreate(&e));
    for (auto& e : ev_graph_) HX_CUDA(cudaEventCreate(&e));
    for (auto& e : tmr_) HX_CUDA(cudaEventCreate(&e));
    setup_comms(uid, uid_len);
    if (role.active) {
      allocate();
      setup_tp_exchange();
      init_params();
      build_groups();
      if (!cstream) cfg.dp_overlap = false;
    } else {
      HX_CUDA(cudaMalloc(&idle_loss_, 256));
      loss_acc = idle_loss_;
      HX_CUDA(cudaMallocHost(&loss_host, 64));
    }
    HX_CUDA(cudaStreamSynchronize(stream));
  }

  // SM cap: green context over sm_fraction * SMs (rounded to the driver's split
  // granularity); "cta" caps only the persistent GEMM grid; "none" disables.
  void setup_stream() {
    int want = role.sm_count > 0 ? role.sm_count
                                 : int(std::lround(role.sm_fraction * double(sm_total)));
    want = std::max(1, std::min(want, sm_total));
    sm_applied = sm_total;
    if (cfg.sm_cap == "green" && want < sm_total) {
      if (make_green_stream(want)) {
        sm_mode = "green";
        return;
      }
    }
    HX_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    own_stream = true;
    HX_CUDA(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
    own_cstream = true;
    if ((cfg.sm_cap == "cta" || cfg.sm_cap == "green") && want < sm_total) {
      gemm_set_sm_limit(want);
      sm_applied = want;
      sm_mode = "cta";
    } else {
      gemm_set_sm_limit(0);
    }
  }

  template <typename T>
  static T drv(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<T>(fn);
  }

  bool make_green_stream(int want) {
    auto pGet = drv<PFN_cuDeviceGet>("cuDeviceGet");
    auto pRes = drv<PFN_cuDeviceGetDevResource>("cuDeviceGetDevResource");
    auto pSplit = drv<PFN_cuDevSmResourceSplitByCount>("cuDevSmResourceSplitByCount");
    auto pDesc = drv<PFN_cuDevResourceGenerateDesc>("cuDevResourceGenerateDesc");
    auto pCreate = drv<PFN_cuGreenCtxCreate>("cuGreenCtxCreate");
    auto pStream = drv<PFN_cuGreenCtxStreamCreate>("cuGreenCtxStreamCreate");
    if (!pGet || !pRes || !pSplit || !pDesc || !pCreate || !pStream) return false;
    cudaFree(nullptr);  // make sure the primary context exists
    CUdevice cd;
    if (pGet(&cd, device) != CUDA_SUCCESS) return false;
    CUdevResource all;
    if (pRes(cd, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
    CUdevResource part, rest;
    unsigned int groups = 1;
    if (pSplit(&part, &groups, &all, &rest, 0, unsigned(want)) != CUDA_SUCCESS || groups != 1)
      return false;
    CUdevResourceDesc desc;
    if (pDesc(&desc, &part, 1) != CUDA_SUCCESS) return false;
    if (pCreate(&green, desc, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return false;
    CUstream s;
    if (pStream(&s, green, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return false;
    stream = reinterpret_cast<cudaStream_t>(s);
    own_stream = true;
    CUstream s2;  // comm stream inside the same SM partition
    if (pStream(&s2, green, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) {
      cstream = reinterpret_cast<cudaStream_t>(s2);
      own_cstream = true;
    }
    sm_applied = int(part.sm.smCount);
    gemm_set_sm_limit(sm_applied);
    return true;
  }

  void setup_comms(const void* uid, size_t uid_len) {
    comms.assign(L.comm_sets.size(), nullptr);
    if (world == 1) return;
    if (!uid || uid_len < sizeof(ncclUniqueId))
      throw InvalidArgument("world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    HX_NCCL(ncclCommInitRank(&world_comm, world, id, rank));
    for (size_t i = 0; i < L.comm_sets.size(); ++i) {
      const auto& set = L.comm_sets[i];
      auto it = std::find(set.begin(), set.end(), rank);
      int color = it == set.end() ? NCCL_SPLIT_NOCOLOR : 0;
      int key = it == set.end() ? 0 : int(it - set.begin());
      ncclComm_t c = nullptr;
      HX_NCCL(ncclCommSplit(world_comm, color, key, &c, nullptr));
      comms[i] = c;
    }
  }

  // ------------------------------------------------------------ memory
  void allocate() {
    const int64_t P = role.param_count;
    const bool need_g16 = !L.dp_buckets[size_t(rank)].empty() && cfg.dp_comm_dtype == "bf16";
    n_slots = int(std::min<int64_t>(role.n_mb, role.stage_count - role.stage));
    n_slots = std::max(n_slots, 1);
    // unfused attention keeps S x S probabilities per (sample, head); the fused
    // kernels keep only the per-row log-sum-exp
    const bool fused = cfg.attention == "fused";
    const int64_t SS = fused ? 0 : mb * nh * S * S;
    const int64_t LSE = mb * nh * S;
    // parameters
    arena.reserve(P * 4 * 4);            // P32, G32, M, V
    arena.reserve(P * 2);                // P16
    if (need_g16) arena.reserve(P * 2);  // DP comm buffer
    // activations per slot (with recompute: layer inputs only, plus one
    // shared set of layer activations)
    const int64_t act_sets = cfg.recompute ? 0 : nl;
    auto reserve_acts = [&] {
      arena.reserve(M * H * 4);                  // x_mid
      arena.reserve(M * H * 2 * 2);              // xn, hn
      arena.reserve(M * 4 * 2);                  // rstd1, rstd2
      arena.reserve(M * qkvw * 2);               // qkv
      arena.reserve(SS * 2);                     // P (unfused)
      arena.reserve(LSE * 4);                    // lse (fused)
      arena.reserve(M * kr * 2);                 // attn
      arena.reserve(M * 2 * F * 2 + M * F * 2);  // gu, act
    };
    if (cfg.recompute) reserve_acts();
    for (int s = 0; s < n_slots; ++s) {
      for (int64_t l = 0; l <= nl; ++l) arena.reserve(M * H * 4);
      for (int64_t l = 0; l < act_sets; ++l) reserve_acts();
      if (role.last_stage) {
        arena.reserve(M * H * 2 + M * 4);
        arena.reserve(M * Vr * 2);
      }
    }
    // scratch
    arena.reserve(SS * 4 * 2);  // scores, dP
    arena.reserve(SS * 2);      // dS
    arena.reserve(LSE * 4 + M * kr * 4);  // fused bwd: delta, fp32 dq accumulator
    arena.reserve(M * H * 2);   // ypart
    arena.reserve(M * F * 2 + M * 2 * F * 2 + M * kr * 2 + M * qkvw * 2);
    arena.reserve(M * H * 4 * 2 + M * H * 2 + M * H * 2);  // dx ping-pong, dxb, dy16
    if (role.stage_count > 1 && cfg.pp_dtype == "bf16")
      arena.reserve(3 * M * H * 2);                        // PP bf16 send / recv staging
    if (role.last_stage) {
      arena.reserve(M * Vr * 4);  // logits
      arena.reserve(6 * M * 4);   // CE statistics + row losses
    }
    arena.reserve(256);                                    // loss
    arena.reserve(kGemmWsBytes);                           // GEMM tail-split workspace
    arena.reserve(kGemmWsCounters * 4);
    arena.reserve(size_t(kRmsBwdCtas) * H * 4);             // rmsnorm bwd partial dg rows
    arena.reserve(embed_bwd_scratch_bytes(int(M)));        // embedding bwd sort keys
    arena.reserve(size_t(S) * size_t(d / 2) * 8);          // RoPE (cos, sin) table
    arena.reserve(role.batch * (S + 1) * 4);               // tokens
    // memory tier: the device's memory_gib caps the rank (cost_model.cpp:130-153
    // applies the same per-device budget to its layer-memory estimate)
    const double cap = L.cluster.devices[size_t(role.device)].memory_gib * double(1ull << 30);
    // weight-gradient grouping: as many micro-batches per group as fit
    wg_ = 1;
    wg_nbuf_ = n_slots > 1 ? 2 : 1;
    if (cfg.wgrad_group != 0 && cfg.wgrad_group != 1 && !cfg.recompute && role.n_mb > 1) {
      double budget = cap - double(arena.total() + tp_exchange_bytes()) - double(12ull << 30);
      if (!cfg.validate_only) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
          budget = std::min(budget, double(fr) - double(arena.total() + tp_exchange_bytes()) -
                                        double(6ull << 30));
      }
      const int64_t want = cfg.wgrad_group > 1 ? std::min<int64_t>(cfg.wgrad_group, role.n_mb)
                                               : role.n_mb;
      const int64_t fit = budget > 0 ? int64_t(budget / double(wg_nbuf_ * wg_bytes_per_mb())) : 0;
      int64_t G = std::min(want, fit);
      if (wg_nbuf_ == 2 && G < n_slots - 1) G = 1;
      if (G >= 2) {
        wg_ = G;
        arena.reserve(size_t(wg_nbuf_ * wg_ * wg_bytes_per_mb()) + size_t(wg_nbuf_) * 4096 * 10);
      }
    }
    if (double(arena.total() + tp_exchange_bytes()) > cap)
      throw Infeasible("plan does not fit device '" + L.cluster.devices[size_t(role.device)].id +
                       "': rank needs " + std::to_string((arena.total() + tp_exchange_bytes()) >> 20) +
                       " MiB, memory_gib " +
                       std::to_string(L.cluster.devices[size_t(role.device)].memory_gib));
    if (cfg.validate_only) return;
    arena.commit();

    P32 = arena.take<float>(P);
    G32 = arena.take<float>(P);
    Mo = arena.take<float>(P);
    Vo = arena.take<float>(P);
    P16 = arena.take<bf16>(P);
    if (need_g16) G16 = arena.take<bf16>(P);
    auto take_acts = [&] {
      LayerActs a;
      a.x_mid = arena.take<float>(M * H);
      a.xn = arena.take<bf16>(M * H);
      a.hn = arena.take<bf16>(M * H);
      a.rstd1 = arena.take<float>(M);
      a.rstd2 = arena.take<float>(M);
      a.qkv = arena.take<bf16>(M * qkvw);
      a.P = arena.take<bf16>(SS);
      a.lse = arena.take<float>(LSE);
      a.attn = arena.take<bf16>(M * kr);
      a.gu = arena.take<bf16>(M * 2 * F);
      a.act = arena.take<bf16>(M * F);
      return a;
    };
    if (cfg.recompute) rc_acts_ = take_acts();
    slots.resize(size_t(n_slots));
    for (auto& sl : slots) {
      for (int64_t l = 0; l <= nl; ++l) sl.x.push_back(arena.take<float>(M * H));
      for (int64_t l = 0; l < act_sets; ++l) sl.layers.push_back(take_acts());
      if (role.last_stage) {
        sl.xf = arena.take<bf16>(M * H);
        sl.rstdf = arena.take<float>(M);
        sl.dlogits = arena.take<bf16>(M * Vr);
      }
    }
    scores = arena.take<float>(SS);
    dP = arena.take<float>(SS);
    dS = arena.take<bf16>(SS);
    delta_ = arena.take<float>(LSE);
    dq_acc_ = arena.take<float>(M * kr);
    gemm_ws_ = arena.take<float>(kGemmWsBytes / 4);
    gemm_cnt_ = arena.take<int>(kGemmWsCounters);
    dg_part_ = arena.take<float>(size_t(kRmsBwdCtas) * H);
    embed_keys_ = arena.take<uint8_t>(embed_bwd_scratch_bytes(int(M)));
    rope_tab_ = arena.take<float2>(S * (d / 2));
    k_rope_table(rope_tab_, int(S), int(d), float(L.model.rope_theta), stream);
    ypart = arena.take<bf16>(M * H);
    da = arena.take<bf16>(M * F);
    dgu = arena.take<bf16>(M * 2 * F);
    dattn = arena.take<bf16>(M * kr);
    dqkv = arena.take<bf16>(M * qkvw);
    dx[0] = arena.take<float>(M * H);
    dx[1] = arena.take<float>(M * H);
    dxb = arena.take<bf16>(M * H);
    dy16 = arena.take<bf16>(M * H);
    if (role.stage_count > 1 && cfg.pp_dtype == "bf16") {
      pp_send16_ = arena.take<bf16>(M * H);
      pp_rf16_ = arena.take<bf16>(M * H);
      pp_rb16_ = arena.take<bf16>(M * H);
    }
    if (role.last_stage) {
      logits = arena.take<float>(M * Vr);
      ce_scr = arena.take<float>(6 * M);
    }
    if (wg_ > 1) {
      const int64_t R = wg_ * M;  // token rows per group buffer
      wst_.assign(size_t(wg_nbuf_ * nl), WStash{});
      wst_xf_.assign(size_t(wg_nbuf_), nullptr);
      wst_dlog_.assign(size_t(wg_nbuf_), nullptr);
      for (int64_t b = 0; b < wg_nbuf_; ++b) {
        for (int64_t l = 0; l < nl; ++l) {
          WStash& w = wst_[size_t(b * nl + l)];
          w.act = arena.take<bf16>(R * F);
          w.hn = arena.take<bf16>(R * H);
          w.attn = arena.take<bf16>(R * kr);
          w.xn = arena.take<bf16>(R * H);
          w.dxob = arena.take<bf16>(R * H);
          w.dgu = arena.take<bf16>(R * 2 * F);
          w.dxmb = arena.take<bf16>(R * H);
          w.dqkv = arena.take<bf16>(R * qkvw);
        }
        if (role.last_stage) {
          wst_xf_[size_t(b)] = arena.take<bf16>(R * H);
          wst_dlog_[size_t(b)] = arena.take<bf16>(R * Vr);
        }
      }
    }
    loss_acc = arena.take<float>(32);
    sp_ = reinterpret_cast<StepParams*>(loss_acc + 16);
    HX_CUDA(cudaMemsetAsync(sp_, 0, sizeof(StepParams), stream));
    HX_CUDA(cudaMemsetAsync(gemm_ws_, 0, kGemmWsBytes, stream));
    HX_CUDA(cudaMemsetAsync(gemm_cnt_, 0, kGemmWsCounters * sizeof(int), stream));
    tokens = arena.take<int32_t>(role.batch * (S + 1));
    HX_CUDA(cudaMallocHost(&tokens_pinned, size_t(role.batch * (S + 1)) * 4));
    HX_CUDA(cudaMallocHost(&loss_host, 64));

    // tensor pointers
    lw.assign(size_t(nl), LayerW{});
    for (const auto& rt : role.tensors) {
      const TensorSpec& ts = L.tensors[size_t(rt.spec)];
      TensorPtrs tp;
      tp.p32 = P32 + rt.offset;
      tp.p16 = P16 + rt.offset;
      tp.g32 = G32 + rt.offset;
      tp.rows = rt.rows;
      tp.cols = ts.cols;
      tp.row0 = rt.row0;
      tp.count = rt.rows * ts.cols;
      tp.offset = rt.offset;
      tp.spec = rt.spec;
      named[ts.name] = tp;
      if (ts.layer >= 0) {
        LayerW& w = lw[size_t(ts.layer - role.layer_start)];
        switch (ts.id) {
          case kAttnNorm: w.attn_norm = tp; break;
          case kWqkv: w.wqkv = tp; break;
          case kWo: w.wo = tp; break;
          case kMlpNorm: w.mlp_norm = tp; break;
          case kWgu: w.wgu = tp; break;
          case kWdown: w.wdown = tp; break;
        }
      } else if (ts.id == kEmbed) {
        embed = tp;
      } else if (ts.id == kFinalNorm) {
        final_norm = tp;
      } else if (ts.id == kLmHead) {
        lm_head = tp;
      }
    }
  }

  void init_params() {
    for (const auto& rt : role.tensors) {
      const TensorSpec& ts = L.tensors[size_t(rt.spec)];
      const TensorPtrs& tp = named[ts.name];
      if (ts.id == kAttnNorm || ts.id == kMlpNorm || ts.id == kFinalNorm) {
        k_fill(tp.p32, tp.p16, tp.count, 1.f, stream);
      } else {
        uint64_t seed = mix_seed(cfg.seed, uint64_t(ts.layer + 1), uint64_t(ts.id));
        k_init_normal(tp.p32, tp.p16, tp.count, tp.row0 * tp.cols, seed, stream);
      }
    }
    HX_CUDA(cudaMemsetAsync(Mo, 0, size_t(role.param_count) * 4, stream));
    HX_CUDA(cudaMemsetAsync(Vo, 0, size_t(role.param_count) * 4, stream));
    HX_CUDA(cudaMemsetAsync(G32, 0, size_t(role.param_count) * 4, stream));
    HX_CUDA(cudaGetLastError());
  }

  // ------------------------------------------------------------ helpers
  void kcheck(const char* kind) {
    ++launches_step;
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess)
      throw CudaError(std::string("kernel launch (") + kind + "): " + cudaGetErrorString(e));
    mark(kind);
  }

  // step timeline (profile mode): an event after every operation on the stream;
  // op time = distance to the previous mark (includes any launch gap before it)
  struct Mark {
    cudaEvent_t ev;
    const char* kind;
  };
  std::vector<cudaEvent_t> mark_pool_;
  std::vector<Mark> marks_;
  std::map<std::string, std::pair<double, int64_t>> timeline_;
  // graph timeline (graph_gemm_events): the same marks captured as event
  // nodes for the sampled micro-batch's forward and backward; an op's time is
  // the distance to the previous mark of the same contiguous run
  struct GMark {
    cudaEvent_t ev;
    const char* kind;
    int run;
  };
  std::vector<GMark> gmarks_;
  int gmark_run_ = 0;
  int64_t gmark_last_mb_ = -1;
  bool gmark_last_bwd_ = false;
  bool in_bwd_ = false;
  void mark(const char* kind) {
    if (capturing_ && cfg.graph_gemm_events && cur_mb_ == role.n_mb / 2) {
      if (cur_mb_ != gmark_last_mb_ || in_bwd_ != gmark_last_bwd_ || gmarks_.empty()) {
        ++gmark_run_;  // a new run starts with a reference mark
        gmark_last_mb_ = cur_mb_;
        gmark_last_bwd_ = in_bwd_;
      }
      cudaEvent_t e;
      HX_CUDA(cudaEventCreate(&e));
      HX_CUDA(cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal));
      gmarks_.push_back({e, kind, gmark_run_});
      return;
    }
    if (!cfg.profile_gemm) return;
    if (marks_.size() == mark_pool_.size()) {
      cudaEvent_t e;
      HX_CUDA(cudaEventCreate(&e));
      mark_pool_.push_back(e);
    }
    cudaEvent_t e = mark_pool_[marks_.size()];
    HX_CUDA(cudaEventRecord(e, stream));
    marks_.push_back({e, kind});
  }
  void collect_timeline() {
    timeline_.clear();
    for (size_t i = 1; i < marks_.size(); ++i) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, marks_[i - 1].ev, marks_[i].ev) == cudaSuccess) {
        auto& t = timeline_[marks_[i].kind];
        t.first += ms;
        t.second += 1;
      }
    }
    marks_.clear();
  }

  // GEMM launch; with profile_gemm, each launch is bracketed by CUDA events on
  // the executor stream and its algorithmic FLOPs recorded (kind: 0 = TP
  // linear layer, 1 = attention product, 2 = LM head)
  int gemm_kind_ = 0;
  struct GemmRec {
    cudaEvent_t a, b;
    double flops;
    int kind;
  };
  std::vector<GemmRec> gemm_pool_;
  size_t gemm_used_ = 0;
  double gemm_ms_[3] = {0, 0, 0}, gemm_flops_[3] = {0, 0, 0};
  int64_t gemm_count_[3] = {0, 0, 0};

  // graph_gemm_events: the same event pairs captured into the step graph, so
  // every replay (the bench's timed region) re-times each GEMM in place; read
  // after a sync from the last replay
  // (only the GEMMs of one micro-batch, n_mb / 2, are bracketed: ~2 us per
  // event node would otherwise add ~3% to the step)
  std::vector<GemmRec> graph_recs_;
  std::vector<std::string> graph_shapes_;
  bool capturing_ = false;
  int64_t cur_mb_ = 0;
  double ggemm_ms_[3] = {0, 0, 0}, ggemm_flops_[3] = {0, 0, 0};
  int64_t ggemm_count_[3] = {0, 0, 0};
  void collect_graph_gemm() {
    if (!gexec_ || graph_recs_.empty()) return;
    for (int k = 0; k < 3; ++k) ggemm_ms_[k] = ggemm_flops_[k] = 0, ggemm_count_[k] = 0;
    for (const auto& r : graph_recs_) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
        ggemm_ms_[r.kind] += ms;
        ggemm_flops_[r.kind] += r.flops;
        ggemm_count_[r.kind] += 1;
      }
    }
    (void)cudaGetLastError();
  }

  void gemm(const GemmDesc& gin) {
    GemmDesc g = gin;
    g.split = cfg.gemm_split ? -1 : 0;
    g.ws = gemm_ws_;
    g.ws_bytes = kGemmWsBytes;
    g.ws_cnt = gemm_cnt_;
    g.ws_cnt_n = kGemmWsCounters;
    GemmRec* rec = nullptr;
    if (cfg.profile_gemm) {
      if (gemm_used_ == gemm_pool_.size()) {
        GemmRec r{};
        HX_CUDA(cudaEventCreate(&r.a));
        HX_CUDA(cudaEventCreate(&r.b));
        gemm_pool_.push_back(r);
      }
      rec = &gemm_pool_[gemm_used_++];
      double full = 2.0 * g.M * double(g.N) * g.K * g.nb1 * g.nb2;
      rec->flops = g.causal != kCausalNone ? full * (double(g.M) + 1) / (2.0 * g.M) : full;
      rec->kind = gemm_kind_;
      HX_CUDA(cudaEventRecordWithFlags(rec->a, stream, capturing_ ? cudaEventRecordExternal : 0));
    } else if (capturing_ && cfg.graph_gemm_events && cur_mb_ == role.n_mb / 2) {
      GemmRec r{};
      HX_CUDA(cudaEventCreate(&r.a));
      HX_CUDA(cudaEventCreate(&r.b));
      double full = 2.0 * g.M * double(g.N) * g.K * g.nb1 * g.nb2;
      r.flops = g.causal != kCausalNone ? full * (double(g.M) + 1) / (2.0 * g.M) : full;
      r.kind = gemm_kind_;
      graph_recs_.push_back(r);
      graph_shapes_.push_back(std::to_string(g.M) + "x" + std::to_string(g.N) + "x" +
                              std::to_string(g.K) + (g.A.mn_major ? " A:mn" : " A:k") +
                              (g.B.mn_major ? " B:mn" : " B:k") + (g.beta ? " beta" : "") +
                              (g.npeer ? " peer" + std::to_string(g.npeer) : "") +
                              (g.nb1 * g.nb2 > 1 ? " batch" + std::to_string(g.nb1 * g.nb2) : ""));
      rec = &graph_recs_.back();
      HX_CUDA(cudaEventRecordWithFlags(rec->a, stream, capturing_ ? cudaEventRecordExternal : 0));
    }
    cudaError_t e = gemm_bf16(g, stream);
    if (e != cudaSuccess) throw CudaError(std::string("gemm: ") + cudaGetErrorString(e));
    if (rec) HX_CUDA(cudaEventRecordWithFlags(rec->b, stream, capturing_ ? cudaEventRecordExternal : 0));
    ++launches_step;
    mark(gemm_kind_ == 0 ? "gemm_linear" : gemm_kind_ == 1 ? "gemm_attention" : "gemm_lm_head");
  }

  int64_t steps_since_collect_ = 0;
  void collect_gemm_profile() {
    for (int k = 0; k < 3; ++k) gemm_ms_[k] = gemm_flops_[k] = 0, gemm_count_[k] = 0;
    for (size_t i = 0; i < gemm_used_; ++i) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, gemm_pool_[i].a, gemm_pool_[i].b) == cudaSuccess) {
        gemm_ms_[gemm_pool_[i].kind] += ms;
        gemm_flops_[gemm_pool_[i].kind] += gemm_pool_[i].flops;
        gemm_count_[gemm_pool_[i].kind] += 1;
      }
    }
    gemm_used_ = 0;
  }

  // plain 2D GEMM helper
  GemmDesc g2(int64_t Mm, int64_t Nn, int64_t Kk, const void* A, int amn, int64_t lda,
              const void* B, int bmn, int64_t ldb, void* C, int64_t ldc, int c32) {
    GemmDesc g;
    g.M = int(Mm);
    g.N = int(Nn);
    g.K = int(Kk);
    g.A = {A, amn, lda, 0, 0};
    g.B = {B, bmn, ldb, 0, 0};
    g.C = C;
    g.ldc = ldc;
    g.c_fp32 = c32;
    return g;
  }

  ncclComm_t tp_comm() const {
    int c = L.tp_comm[size_t(rank)];
    return c >= 0 ? comms[size_t(c)] : nullptr;
  }

  void tp_allreduce_bf16(bf16* buf, int64_t n) {
    if (role.tp <= 1) return;
    HX_NCCL(ncclAllReduce(buf, buf, size_t(n), ncclBfloat16, ncclSum, tp_comm(), stream));
    ++nccl_calls_step;
    mark("nccl_tp_allreduce");
  }

  void tp_allreduce_f32(const float* in, float* out, int64_t n, ncclRedOp_t op) {
    if (role.tp <= 1) return;
    HX_NCCL(ncclAllReduce(in, out, size_t(n), ncclFloat32, op, tp_comm(), stream));
    ++nccl_calls_step;
    mark("nccl_tp_allreduce");
  }

  int32_t* tok_of(int64_t mbi) { return tokens + mbi * mb * (S + 1); }

  // ------------------------------------------------------------ TP exchange
  // (tp > kMaxGemmPeers + 1: the GEMM epilogue has no map for more peers; such
  // stages reduce through NCCL)
  bool use_tp_peer() const {
    return role.tp > 1 && role.tp <= kMaxGemmPeers + 1 && cfg.tp_reduce == "peer";
  }
  size_t tp_slot_elems() const { return size_t(M * H); }
  size_t tp_exchange_bytes() const {
    if (!use_tp_peer()) return 0;
    return 2 * size_t(role.tp) * tp_slot_elems() * 2 + 256;
  }

  // exchange buffers: allocate, export (cudaIpc), all-gather the handles over
  // the TP communicator, map every peer's buffer
  void setup_tp_exchange() {
    if (!use_tp_peer()) return;
    ncclComm_t c = tp_comm();
    int me = 0, n = 0;
    HX_NCCL(ncclCommUserRank(c, &me));
    HX_NCCL(ncclCommCount(c, &n));
    if (n != role.tp) throw CudaError("TP communicator size mismatch");
    xflag_off_ = 2 * size_t(role.tp) * tp_slot_elems() * 2;
    HX_CUDA(cudaMalloc(&xbuf_, tp_exchange_bytes()));
    HX_CUDA(cudaMemset(xbuf_ + xflag_off_, 0, 256));
    cudaIpcMemHandle_t h;
    HX_CUDA(cudaIpcGetMemHandle(&h, xbuf_));
    // one record per rank: IPC handle + the SM count actually applied
    struct Rec {
      cudaIpcMemHandle_t h;
      int sms;
      int pad[15];
    };
    Rec mine{};
    mine.h = h;
    mine.sms = sm_applied;
    const size_t hs = sizeof(Rec);
    char* dh = nullptr;
    HX_CUDA(cudaMalloc(&dh, hs * size_t(n)));
    HX_CUDA(cudaMemcpy(dh + hs * size_t(me), &mine, hs, cudaMemcpyHostToDevice));
    HX_NCCL(ncclAllGather(dh + hs * size_t(me), dh, hs, ncclChar, c, stream));
    std::vector<Rec> all(static_cast<size_t>(n));
    HX_CUDA(cudaMemcpyAsync(all.data(), dh, hs * size_t(n), cudaMemcpyDeviceToHost, stream));
    HX_CUDA(cudaStreamSynchronize(stream));
    cudaFree(dh);
    tpp_ = TpPeers{};
    tpp_.tp = n;
    tpp_.me = me;
    tpp_.local = reinterpret_cast<unsigned long long*>(xbuf_ + xflag_off_);
    for (int k = 0; k < n; ++k) {
      if (k == me) continue;
      void* p = nullptr;
      HX_CUDA(cudaIpcOpenMemHandle(&p, all[size_t(k)].h, cudaIpcMemLazyEnablePeerAccess));
      xpeer_[k] = static_cast<uint8_t*>(p);
      tpp_.remote[k] = reinterpret_cast<unsigned long long*>(xpeer_[k] + xflag_off_) + me;
    }
    tp_peer_ = true;
    // Asymmetric direction: the rank with the largest work / SM share (the
    // step's critical path) stores its partial only locally -- the NVLink
    // tail of a peer store would extend its GEMMs -- and the faster ranks,
    // which wait for it anyway, pull it with a copy-engine transfer.  Even
    // stages (no rank >= 5% slower than the next) push symmetrically.
    std::vector<double> ratio;
    for (int k = 0; k < n; ++k) {
      // comm rank k = position in the sorted TP rank set (setup_comms' key)
      const RankRole& q = L.roles[size_t(L.comm_sets[size_t(L.tp_comm[size_t(rank)])][size_t(k)])];
      const double work = double(q.heads.size()) * 4.0 * double(d) * double(H) +
                          double(q.ffn_chunks.size()) * 64.0 * 3.0 * double(H);
      const double share = double(std::max(all[size_t(k)].sms, 1)) / double(std::max(sm_total, 1));
      ratio.push_back(work / share);
    }
    const int crit = int(std::max_element(ratio.begin(), ratio.end()) - ratio.begin());
    double second = 0;
    for (int k = 0; k < n; ++k)
      if (k != crit) second = std::max(second, ratio[size_t(k)]);
    tp_crit_ = ratio[size_t(crit)] >= 1.05 * second ? crit : -1;
    if (cfg.tp_direction == "push") tp_crit_ = -1;
  }

  // slot `src` of ring buffer `b` on TP rank `owner` (owner == me: local)
  bf16* xslot(int owner, unsigned b, int src) {
    uint8_t* base = owner == tpp_.me ? xbuf_ : xpeer_[owner];
    return reinterpret_cast<bf16*>(base) + (size_t(b) * size_t(role.tp) + size_t(src)) * tp_slot_elems();
  }

  // row-parallel partial GEMM: C goes to this rank's slot of the current ring
  // buffer locally and on every peer.  Returns the buffer's slot 0; the
  // consumer sums tp slots (tp_slot_elems apart) after tp_sync().
  const bf16* tp_partial_gemm(GemmDesc g) {
    const unsigned b = xop_ & 1u;
    g.C = xslot(tpp_.me, b, tpp_.me);
    g.npeer = 0;
    if (tpp_.me != tp_crit_)
      for (int k = 0; k < role.tp; ++k)
        if (k != tpp_.me) g.peer_C[g.npeer++] = xslot(k, b, tpp_.me);
    gemm(g);
    return xslot(tpp_.me, b, 0);
  }
  void tp_sync() {
    if (xop_ >= (1u << 24)) throw LimitExceeded("too many TP exchanges per step");
    const unsigned b = xop_ & 1u;
    k_tp_sync(tpp_, sp_, xop_++, stream);
    kcheck("tp_sync");
    if (tp_crit_ >= 0 && tpp_.me != tp_crit_ && !pad_) {
      if (cfg.tp_pull == "ce") {
        HX_CUDA(cudaMemcpyAsync(xslot(tpp_.me, b, tp_crit_), xslot(tp_crit_, b, tp_crit_),
                                tp_slot_elems() * 2, cudaMemcpyDeviceToDevice, stream));
        ++copies_step;
      } else {
        k_peer_copy(xslot(tpp_.me, b, tp_crit_), xslot(tp_crit_, b, tp_crit_),
                    tp_slot_elems() * 2, sm_applied, stream);
        kcheck("tp_pull");
      }
      mark("tp_pull");
    }
  }
  bool pad_ = false;
  std::string attention_note_;

  // ------------------------------------------------------------ forward
  LayerActs& acts(Slot& sl, int64_t l) { return cfg.recompute ? rc_acts_ : sl.layers[size_t(l)]; }

  // recompute = true: re-run for the backward; the layer output (down
  // projection and its TP reduction) is not needed and is skipped
  void layer_fwd(Slot& sl, int64_t l, bool recompute = false) {
    LayerActs& a = acts(sl, l);
    const LayerW& w = lw[size_t(l)];
    if (wg_ > 1) {
      WStash& st = ws(l, cur_mb_);
      a.xn = wrow(st.xn, cur_mb_, H);
      a.hn = wrow(st.hn, cur_mb_, H);
      a.attn = wrow(st.attn, cur_mb_, kr);
      a.act = wrow(st.act, cur_mb_, F);
    }
    float* x_in = sl.x[size_t(l)];
    float* x_out = sl.x[size_t(l + 1)];
    const float eps = float(L.model.norm_eps);
    // attention block
    k_rmsnorm_fwd(x_in, nullptr, nullptr, w.attn_norm.p32, a.xn, a.rstd1, int(M), int(H), eps, stream);
    kcheck("rmsnorm_fwd");
    {
      // QKV projection with RoPE applied in the epilogue (d 64 / 128)
      GemmDesc g = g2(M, qkvw, H, a.xn, 0, H, w.wqkv.p16, 0, H, a.qkv, qkvw, 0);
      const bool fuse = cfg.fuse_rope && (d == 64 || d == 128);
      if (fuse) {
        g.rope = rope_tab_;
        g.rope_d = int(d);
        g.rope_S = int(S);
      }
      gemm(g);
      if (!fuse) {
        k_rope(a.qkv, int(M), int(S), int(nh), int(d), float(L.model.rope_theta), 0, stream);
        kcheck("rope");
      }
    }
    attention_fwd(a);
    if (role.tp == 1) {
      GemmDesc g = g2(M, H, kr, a.attn, 0, kr, w.wo.p16, 1, H, a.x_mid, H, 1);
      g.R = x_in;
      gemm(g);
      k_rmsnorm_fwd(a.x_mid, nullptr, nullptr, w.mlp_norm.p32, a.hn, a.rstd2, int(M), int(H), eps, stream);
      kcheck("rmsnorm_fwd");
    } else if (tp_peer_) {
      const bf16* y = tp_partial_gemm(g2(M, H, kr, a.attn, 0, kr, w.wo.p16, 1, H, nullptr, H, 0));
      tp_sync();
      k_rmsnorm_fwd(x_in, y, a.x_mid, w.mlp_norm.p32, a.hn, a.rstd2, int(M), int(H), eps, stream,
                    role.tp, int64_t(tp_slot_elems()));
      kcheck("rmsnorm_fwd");
    } else {
      gemm(g2(M, H, kr, a.attn, 0, kr, w.wo.p16, 1, H, ypart, H, 0));
      tp_allreduce_bf16(ypart, M * H);
      k_rmsnorm_fwd(x_in, ypart, a.x_mid, w.mlp_norm.p32, a.hn, a.rstd2, int(M), int(H), eps, stream);
      kcheck("rmsnorm_fwd");
    }
    // MLP block: gate-up GEMM with the SwiGLU epilogue (act written from the tile)
    {
      GemmDesc g = g2(M, 2 * F, H, a.hn, 0, H, w.wgu.p16, 0, H, a.gu, 2 * F, 0);
      if (cfg.fuse_swiglu) g.act = a.act;
      gemm(g);
      if (!cfg.fuse_swiglu) {
        k_swiglu_fwd(a.gu, a.act, int(M), int(F), stream);
        kcheck("swiglu_fwd");
      }
    }
    if (recompute) return;
    if (role.tp == 1) {
      GemmDesc g = g2(M, H, F, a.act, 0, F, w.wdown.p16, 1, H, x_out, H, 1);
      g.R = a.x_mid;
      gemm(g);
    } else if (tp_peer_) {
      const bf16* y = tp_partial_gemm(g2(M, H, F, a.act, 0, F, w.wdown.p16, 1, H, nullptr, H, 0));
      tp_sync();
      k_residual_add(a.x_mid, y, x_out, M * H, stream, role.tp, int64_t(tp_slot_elems()));
      kcheck("residual_add");
    } else {
      gemm(g2(M, H, F, a.act, 0, F, w.wdown.p16, 1, H, ypart, H, 0));
      tp_allreduce_bf16(ypart, M * H);
      k_residual_add(a.x_mid, ypart, x_out, M * H, stream);
      kcheck("residual_add");
    }
  }

  // per (sample b, head h): scores = q k^T / sqrt(d) (causal tiles), P = softmax,
  // attn = P v -- batched over z = h + nh * b straight out of the QKV buffer
  void attention_fwd(LayerActs& a) {
    if (cfg.attention == "fused") {
      AttnDesc ad;
      ad.qkv = a.qkv;
      ad.out = a.attn;
      ad.lse = a.lse;
      ad.S = int(S);
      ad.nh = int(nh);
      ad.d = int(d);
      ad.mb = int(mb);
      ad.scale = 1.f / std::sqrt(float(d));
      cudaError_t e = hexexec::attention_fwd(ad, stream);
      if (e != cudaSuccess) throw CudaError(std::string("attention_fwd: ") + cudaGetErrorString(e));
      kcheck("attn_fwd");
      return;
    }
    gemm_kind_ = 1;
    const int64_t SS2 = S * S;
    GemmDesc g;
    g.M = int(S);
    g.N = int(S);
    g.K = int(d);
    g.nb1 = int(nh);
    g.nb2 = int(mb);
    g.A = {a.qkv, 0, qkvw, 3 * d, S * qkvw};
    g.B = {a.qkv + d, 0, qkvw, 3 * d, S * qkvw};
    g.C = scores;
    g.ldc = S;
    g.cbs1 = SS2;
    g.cbs2 = nh * SS2;
    g.c_fp32 = 1;
    g.alpha = 1.f / std::sqrt(float(d));
    g.causal = kCausalSkipUpper;
    gemm(g);
    k_softmax_fwd(scores, a.P, int(S), int(mb * nh), stream);
    kcheck("softmax_fwd");
    GemmDesc o;
    o.M = int(S);
    o.N = int(d);
    o.K = int(S);
    o.nb1 = int(nh);
    o.nb2 = int(mb);
    o.A = {a.P, 0, S, SS2, nh * SS2};
    o.B = {a.qkv + 2 * d, 1, qkvw, 3 * d, S * qkvw};
    o.C = a.attn;
    o.ldc = kr;
    o.cbs1 = d;
    o.cbs2 = S * kr;
    o.causal = kCausalKLower;
    gemm(o);
    gemm_kind_ = 0;
  }

  void head_fwd(Slot& sl, int64_t mbi) {
    const float eps = float(L.model.norm_eps);
    if (wg_ > 1) {
      const size_t b = size_t((mbi / wg_) % wg_nbuf_);
      sl.xf = wrow(wst_xf_[b], mbi, H);
      sl.dlogits = wrow(wst_dlog_[b], mbi, Vr);
    }
    k_rmsnorm_fwd(sl.x[size_t(nl)], nullptr, nullptr, final_norm.p32, sl.xf, sl.rstdf, int(M), int(H), eps, stream);
    kcheck("rmsnorm_fwd");
    gemm_kind_ = 2;
    gemm(g2(M, Vr, H, sl.xf, 0, H, lm_head.p16, 0, H, logits, Vr, 1));
    gemm_kind_ = 0;
    float* lmax = ce_scr;
    float* lsum = ce_scr + M;
    float* st2 = ce_scr + 2 * M;
    float* gmax = ce_scr + 4 * M;
    const int32_t* tk = tok_of(mbi);
    k_ce_stats(logits, int(Vr), int(v0), tk, int(M), int(S), lmax, lsum, st2, stream);
    kcheck("ce_stats");
    if (role.tp > 1) {
      tp_allreduce_f32(lmax, gmax, M, ncclMax);
      k_ce_rescale(lmax, lsum, gmax, st2, int(M), stream);
      kcheck("ce_rescale");
      tp_allreduce_f32(st2, st2, 2 * M, ncclSum);
    } else {
      HX_CUDA(cudaMemcpyAsync(gmax, lmax, size_t(M) * 4, cudaMemcpyDeviceToDevice, stream));
      ++copies_step;
    }
    const float inv_count = 1.f / float(role.batch * S);
    k_ce_finish(logits, int(Vr), int(v0), tk, int(M), int(S), gmax, st2, inv_count, sl.dlogits,
                loss_acc, ce_scr + 5 * M, stream);
    kcheck("ce_finish");
  }

  void forward(int64_t mbi, Slot& sl) {
    cur_mb_ = mbi;
    in_bwd_ = false;
    mark("fwd_begin");
    if (role.first_stage) {
      k_embed_fwd(tok_of(mbi), embed.p32, sl.x[0], int(M), int(S), int(H), stream);
      kcheck("embed_fwd");
    }
    for (int64_t l = 0; l < nl; ++l) layer_fwd(sl, l);
    if (role.last_stage) head_fwd(sl, mbi);
  }

  // ------------------------------------------------------------ backward
  // dxo: fp32 grad of the layer output (+ bf16 copy dxob); writes dx_in/dxb_in
  void layer_bwd(Slot& sl, int64_t l, const float* dxo, const bf16* dxob, float* dxi, bf16* dxib) {
    if (cfg.recompute) layer_fwd(sl, l, true);
    LayerActs& a = acts(sl, l);
    const LayerW& w = lw[size_t(l)];
    const bool first_mb = accum_first_;
    // weight-gradient GEMM operands: this micro-batch's rows (K = M), or with
    // grouping the group's token-concatenated rows at its last micro-batch
    const int64_t mbi = cur_mb_;
    const bool grouped = wg_ > 1;
    const bool do_wgrad = !grouped || wg_end(mbi);
    const int64_t Kw = grouped ? (mbi % wg_ + 1) * M : M;
    const int wbeta = grouped ? (mbi / wg_ > 0 ? 1 : 0) : (first_mb ? 0 : 1);
    WStash* st = grouped ? &ws(l, mbi) : nullptr;
    bf16* dgu_ = grouped ? wrow(st->dgu, mbi, 2 * F) : dgu;
    bf16* dqkv_saved = dqkv;
    if (grouped) dqkv = wrow(st->dqkv, mbi, qkvw);
    auto wgemm = [&](int64_t Mo, const bf16* Ag, int64_t lda_, const bf16* Bg, int64_t ldb_,
                     float* G) {
      GemmDesc g = g2(Mo, H, Kw, Ag, 1, lda_, Bg, 1, ldb_, G, H, 1);
      g.beta = wbeta;
      gemm(g);
    };
    // MLP: down projection
    gemm(g2(M, F, H, dxob, 0, H, w.wdown.p16, 0, H, da, F, 0));
    if (do_wgrad)
      wgemm(F, grouped ? st->act : a.act, F, grouped ? st->dxob : dxob, H, w.wdown.g32);
    k_swiglu_bwd(a.gu, da, dgu_, int(M), int(F), stream);
    kcheck("swiglu_bwd");
    const bf16* dyr = dy16;
    if (tp_peer_)
      dyr = tp_partial_gemm(g2(M, H, 2 * F, dgu_, 0, 2 * F, w.wgu.p16, 1, H, nullptr, H, 0));
    else
      gemm(g2(M, H, 2 * F, dgu_, 0, 2 * F, w.wgu.p16, 1, H, dy16, H, 0));
    if (do_wgrad)
      wgemm(2 * F, grouped ? st->dgu : dgu_, 2 * F, grouped ? st->hn : a.hn, H, w.wgu.g32);
    if (tp_peer_)
      tp_sync();
    else
      tp_allreduce_bf16(dy16, M * H);
    const int ny = tp_peer_ ? int(role.tp) : 1;
    const int64_t ys = int64_t(tp_slot_elems());
    // dx_mid = dx_out + rmsnorm_bwd(dhn);  (reuse dxi as dx_mid storage)
    float* dxm = dxi;
    bf16* dxmb = grouped ? wrow(st->dxmb, mbi, H) : dxib;
    k_rmsnorm_bwd(dyr, nullptr, a.x_mid, a.rstd2, w.mlp_norm.p32, dxo, dxm, dxmb, w.mlp_norm.g32,
                  int(M), int(H), dg_part_, stream, ny, ys);
    kcheck("rmsnorm_bwd");
    // attention: O projection
    gemm(g2(M, kr, H, dxmb, 0, H, w.wo.p16, 0, H, dattn, kr, 0));
    if (do_wgrad)
      wgemm(kr, grouped ? st->attn : a.attn, kr, grouped ? st->dxmb : dxmb, H, w.wo.g32);
    // RoPE backward: fused into the fused attention's dq cast (d 64 / 128)
    if (!attention_bwd(a, cfg.fuse_rope && (d == 64 || d == 128))) {
      k_rope(dqkv, int(M), int(S), int(nh), int(d), float(L.model.rope_theta), 1, stream);
      kcheck("rope");
    }
    if (tp_peer_)
      dyr = tp_partial_gemm(g2(M, H, qkvw, dqkv, 0, qkvw, w.wqkv.p16, 1, H, nullptr, H, 0));
    else
      gemm(g2(M, H, qkvw, dqkv, 0, qkvw, w.wqkv.p16, 1, H, dy16, H, 0));
    if (do_wgrad)
      wgemm(qkvw, grouped ? st->dqkv : dqkv, qkvw, grouped ? st->xn : a.xn, H, w.wqkv.g32);
    if (tp_peer_)
      tp_sync();
    else
      tp_allreduce_bf16(dy16, M * H);
    // dx_in = dx_mid + rmsnorm_bwd(dxn): in place over dx_mid (row-local)
    k_rmsnorm_bwd(dyr, nullptr, sl.x[size_t(l)], a.rstd1, w.attn_norm.p32, dxm, dxi, dxib,
                  w.attn_norm.g32, int(M), int(H), dg_part_, stream, ny, ys);
    kcheck("rmsnorm_bwd");
    dqkv = dqkv_saved;
  }

  // returns true when the RoPE backward was applied (fused path with rope)
  bool attention_bwd(LayerActs& a, bool rope) {
    if (cfg.attention == "fused") {
      AttnBwdDesc ad;
      ad.qkv = a.qkv;
      ad.out = a.attn;
      ad.dout = dattn;
      ad.lse = a.lse;
      ad.delta = delta_;
      ad.dq_acc = dq_acc_;
      ad.dqkv = dqkv;
      ad.S = int(S);
      ad.nh = int(nh);
      ad.d = int(d);
      ad.mb = int(mb);
      ad.scale = 1.f / std::sqrt(float(d));
      if (rope) ad.rope = rope_tab_;
      cudaError_t e = hexexec::attention_bwd(ad, stream);
      if (e != cudaSuccess) throw CudaError(std::string("attention_bwd: ") + cudaGetErrorString(e));
      launches_step += 2;  // delta + dq cast kernels (+ the main kernel below)
      kcheck("attn_bwd");
      return ad.rope != nullptr;
    }
    gemm_kind_ = 1;
    const int64_t SS2 = S * S;
    // dP = dO V^T
    GemmDesc g;
    g.M = int(S);
    g.N = int(S);
    g.K = int(d);
    g.nb1 = int(nh);
    g.nb2 = int(mb);
    g.A = {dattn, 0, kr, d, S * kr};
    g.B = {a.qkv + 2 * d, 0, qkvw, 3 * d, S * qkvw};
    g.C = dP;
    g.ldc = S;
    g.cbs1 = SS2;
    g.cbs2 = nh * SS2;
    g.c_fp32 = 1;
    g.causal = kCausalSkipUpper;
    gemm(g);
    k_softmax_bwd(a.P, dP, dS, 1.f / std::sqrt(float(d)), int(S), int(mb * nh), stream);
    kcheck("softmax_bwd");
    // dQ = dS K
    GemmDesc q;
    q.M = int(S);
    q.N = int(d);
    q.K = int(S);
    q.nb1 = int(nh);
    q.nb2 = int(mb);
    q.A = {dS, 0, S, SS2, nh * SS2};
    q.B = {a.qkv + d, 1, qkvw, 3 * d, S * qkvw};
    q.C = dqkv;
    q.ldc = qkvw;
    q.cbs1 = 3 * d;
    q.cbs2 = S * qkvw;
    q.causal = kCausalKLower;
    gemm(q);
    // dK = dS^T Q
    GemmDesc k = q;
    k.A = {dS, 1, S, SS2, nh * SS2};
    k.B = {a.qkv, 1, qkvw, 3 * d, S * qkvw};
    k.C = dqkv + d;
    k.causal = kCausalKUpper;
    gemm(k);
    // dV = P^T dO
    GemmDesc v = q;
    v.A = {a.P, 1, S, SS2, nh * SS2};
    v.B = {dattn, 1, kr, d, S * kr};
    v.C = dqkv + 2 * d;
    v.causal = kCausalKUpper;
    gemm(v);
    gemm_kind_ = 0;
    return false;
  }

  // backward of one micro-batch; dx_top (fp32) is the grad of the stage output
  // (received), or null on the last stage (starts from dlogits)
  void backward(int64_t mbi, Slot& sl, float* dx_top) {
    cur_mb_ = mbi;
    in_bwd_ = true;
    mark("bwd_begin");
    float* cur = dx[0];
    float* nxt = dx[1];
    bf16* curb = dxb;
    const bool grouped = wg_ > 1;
    if (grouped && nl > 0) curb = wrow(ws(nl - 1, mbi).dxob, mbi, H);
    if (role.last_stage) {
      gemm_kind_ = 2;
      const bf16* dyr = dy16;
      if (tp_peer_)
        dyr = tp_partial_gemm(g2(M, H, Vr, sl.dlogits, 0, Vr, lm_head.p16, 1, H, nullptr, H, 0));
      else
        gemm(g2(M, H, Vr, sl.dlogits, 0, Vr, lm_head.p16, 1, H, dy16, H, 0));
      if (!grouped) {
        GemmDesc g = g2(Vr, H, M, sl.dlogits, 1, Vr, sl.xf, 1, H, lm_head.g32, H, 1);
        g.beta = accum_first_ ? 0 : 1;
        gemm(g);
      } else if (wg_end(mbi)) {
        const size_t b = size_t((mbi / wg_) % wg_nbuf_);
        GemmDesc g = g2(Vr, H, (mbi % wg_ + 1) * M, wst_dlog_[b], 1, Vr, wst_xf_[b], 1, H,
                        lm_head.g32, H, 1);
        g.beta = mbi / wg_ > 0 ? 1 : 0;
        gemm(g);
      }
      gemm_kind_ = 0;
      if (tp_peer_)
        tp_sync();
      else
        tp_allreduce_bf16(dy16, M * H);
      k_rmsnorm_bwd(dyr, nullptr, sl.x[size_t(nl)], sl.rstdf, final_norm.p32, nullptr, cur, curb,
                    final_norm.g32, int(M), int(H), dg_part_, stream, tp_peer_ ? int(role.tp) : 1,
                    int64_t(tp_slot_elems()));
      kcheck("rmsnorm_bwd");
      group_ready(kGroupHead);
    } else {
      HX_CUDA(cudaMemcpyAsync(cur, dx_top, size_t(M * H) * 4, cudaMemcpyDeviceToDevice, stream));
      ++copies_step;
      k_cast_bf16(cur, curb, M * H, stream);
      kcheck("cast_bf16");
    }
    for (int64_t l = nl - 1; l >= 0; --l) {
      // dxi aliases the ping-pong partner; dxb reused in place (row-local ops);
      // with wgrad grouping the bf16 input grad lands in layer l-1's stash row
      bf16* nb = (grouped && l > 0) ? wrow(ws(l - 1, mbi).dxob, mbi, H) : (grouped ? dxb : curb);
      layer_bwd(sl, l, cur, curb, nxt, nb);
      curb = nb;
      std::swap(cur, nxt);
      group_ready(int(role.layer_start + l));
    }
    if (role.first_stage) {
      k_embed_bwd(tok_of(mbi), cur, embed.g32, int(M), int(S), int(H), embed_keys_, stream);
      kcheck("embed_bwd");
      group_ready(kGroupEmbed);
    }
    bwd_out_ = cur;
  }

  // ------------------------------------------------------------ PP comm
  // leader protocol: only tp_index 0 talks to the neighbouring stage (whose
  // first device is the first entry of the send lists), then broadcasts
  bool pp_leader() const { return cfg.pp_protocol == "leader"; }
  // pp_dtype "bf16" (default): the hand-off travels as bf16, the 2-byte payload
  // comm_pp_hop prices (cost_model.cpp:10-13, :59-76); the sender casts its
  // fp32 stage output / input grad into pp_send16_, the receiver lands it in a
  // bf16 staging buffer and widens it into the fp32 destination after the
  // P2P group (and the leader broadcast) completes
  bool pp16() const { return cfg.pp_dtype == "bf16"; }
  void send_to(const std::vector<int>& peers, const float* buf) {
    bool cast = false;
    for (size_t k = 0; k < peers.size(); ++k) {
      if (pp_leader() && (role.tp_index != 0 || k > 0)) break;
      if (pp16()) {
        if (!cast) {
          k_cast_bf16(buf, pp_send16_, M * H, stream);
          kcheck("pp_cast");
          cast = true;
        }
        HX_NCCL(ncclSend(pp_send16_, size_t(M * H), ncclBfloat16, peers[k], world_comm, stream));
      } else {
        HX_NCCL(ncclSend(buf, size_t(M * H), ncclFloat32, peers[k], world_comm, stream));
      }
      ++nccl_calls_step;
    }
  }
  void recv_from(int peer, float* buf, bf16* stage16) {
    if (peer < 0 || (pp_leader() && role.tp_index != 0)) return;
    if (pp16())
      HX_NCCL(ncclRecv(stage16, size_t(M * H), ncclBfloat16, peer, world_comm, stream));
    else
      HX_NCCL(ncclRecv(buf, size_t(M * H), ncclFloat32, peer, world_comm, stream));
    ++nccl_calls_step;
  }
  // leader protocol, after the receive has completed (outside the P2P group).
  // The root is the leader's rank in the TP communicator: that communicator
  // is keyed by position in the sorted rank set (setup_comms), which differs
  // from tp order when a stage lists its devices out of rank order or the
  // cluster's `rank` extension permutes them.
  int leader_comm_rank() const {
    const auto& set = L.comm_sets[size_t(L.tp_comm[size_t(rank)])];
    return int(std::find(set.begin(), set.end(), role.tp_group[0]) - set.begin());
  }
  // after the receive: leader broadcast (leader protocol) and the bf16 -> fp32
  // widening into the destination
  void bcast_in_stage(int peer, float* buf, bf16* stage16) {
    if (peer < 0) return;
    if (pp_leader() && role.tp > 1) {
      if (pp16())
        HX_NCCL(ncclBroadcast(stage16, stage16, size_t(M * H), ncclBfloat16, leader_comm_rank(),
                              tp_comm(), stream));
      else
        HX_NCCL(ncclBroadcast(buf, buf, size_t(M * H), ncclFloat32, leader_comm_rank(),
                              tp_comm(), stream));
      ++nccl_calls_step;
    }
    if (pp16()) {
      k_upcast_bf16(stage16, buf, M * H, stream);
      kcheck("pp_upcast");
    }
  }
  void send_fwd(Slot& sl) { send_to(role.fwd_send_to, sl.x[size_t(nl)]); }
  void recv_fwd(Slot& sl) { recv_from(role.fwd_recv_from, sl.x[0], pp_rf16_); }
  void bcast_fwd(Slot& sl) { bcast_in_stage(role.fwd_recv_from, sl.x[0], pp_rf16_); }
  void send_bwd(const float* g) { send_to(role.bwd_send_to, g); }
  void recv_bwd(float* g) { recv_from(role.bwd_recv_from, g, pp_rb16_); }
  void bcast_bwd(float* g) { bcast_in_stage(role.bwd_recv_from, g, pp_rb16_); }
  bf16 *pp_send16_ = nullptr, *pp_rf16_ = nullptr, *pp_rb16_ = nullptr;

  // ------------------------------------------------------------ step
  bool accum_first_ = true;
  float* bwd_out_ = nullptr;
  float* grad_in_ = nullptr;  // received grad buffer (reuses scores-free scratch)

  void run_pipeline() {
    const int64_t n = role.n_mb;
    const int P = role.stage_count;
    const int j = role.stage;
    const int64_t warm = std::min<int64_t>(P - j - 1, n);
    const int64_t rem = n - warm;
    float* grecv = dx[1];  // grads from the next stage land here before backward copies them
    // we receive into a dedicated region: use ypart-sized fp32? dx[1] is free between
    // backward passes; backward() copies it into dx[0] first.
    auto slot_of = [&](int64_t mbi) -> Slot& { return slots[size_t(mbi % n_slots)]; };
    int64_t next_bwd = 0;
    auto do_bwd = [&](int64_t mbi) {
      accum_first_ = next_bwd == 0;
      last_mb_ = next_bwd == n - 1;
      backward(mbi, slot_of(mbi), grecv);
      ++next_bwd;
    };
    // warm-up forwards
    const bool pp = P > 1;
    for (int64_t i = 0; i < warm; ++i) {
      Slot& sl = slot_of(i);
      recv_fwd(sl);
      bcast_fwd(sl);
      if (pp) mark("nccl_pp");
      forward(i, sl);
      send_fwd(sl);
      if (pp) mark("nccl_pp");
    }
    if (rem > 0) {
      recv_fwd(slot_of(warm));
      bcast_fwd(slot_of(warm));
    }
    if (pp) mark("nccl_pp");
    for (int64_t i = 0; i < rem; ++i) {
      const int64_t f = warm + i;
      Slot& sl = slot_of(f);
      forward(f, sl);
      // send activation + receive the grad for micro-batch i (grouped)
      HX_NCCL(ncclGroupStart());
      send_fwd(sl);
      recv_bwd(grecv);
      HX_NCCL(ncclGroupEnd());
      bcast_bwd(grecv);
      if (pp) mark("nccl_pp");
      do_bwd(i);
      HX_NCCL(ncclGroupStart());
      send_bwd(bwd_out_);
      if (i + 1 < rem) recv_fwd(slot_of(f + 1));
      HX_NCCL(ncclGroupEnd());
      if (i + 1 < rem) bcast_fwd(slot_of(f + 1));
      if (pp) mark("nccl_pp");
    }
    for (int64_t i = rem; i < n; ++i) {
      recv_bwd(grecv);
      bcast_bwd(grecv);
      if (pp) mark("nccl_pp");
      do_bwd(i);
      send_bwd(bwd_out_);
      if (pp) mark("nccl_pp");
    }
  }

  // ------------------------------------------------------------ DP overlap
  // Gradients become final group by group during the backward of the last
  // micro-batch (head, layers descending, embedding).  Each group's DP work --
  // sample-weighted scale + bf16 cast, chunk-matched allreduce, AdamW -- runs
  // on a second stream as soon as the group is final, overlapping the backward
  // of the remaining layers.  Every rank walks the groups in the same global
  // order, so per-communicator call order matches across ranks.
  struct SyncGroup {
    int id = 0;
    std::vector<size_t> tensors;   // indices into role.tensors
    std::vector<DpBucket> buckets;
    cudaEvent_t ready = nullptr;
  };
  std::vector<SyncGroup> groups_;
  cudaStream_t cstream = nullptr;
  bool own_cstream = false;
  cudaEvent_t join_ev_ = nullptr;
  bool last_mb_ = false;

  void build_groups() {
    std::map<int, size_t> idx;
    for (size_t i = 0; i < role.tensors.size(); ++i) {
      const int g = sync_group(L.tensors[size_t(role.tensors[i].spec)]);
      if (!idx.count(g)) {
        idx[g] = groups_.size();
        SyncGroup sg;
        sg.id = g;
        HX_CUDA(cudaEventCreateWithFlags(&sg.ready, cudaEventDisableTiming));
        groups_.push_back(sg);
      }
      groups_[idx[g]].tensors.push_back(i);
    }
    for (const auto& b : L.dp_buckets[size_t(rank)]) groups_[idx.at(b.group)].buckets.push_back(b);
    HX_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
  }

  // enqueue the DP work of one group on stream `s`
  void group_work(const SyncGroup& g, cudaStream_t s) {
    const bool bf = G16 != nullptr;
    for (size_t ti : g.tensors) {
      const RankTensor& rt = role.tensors[ti];
      const int64_t cnt = rt.rows * L.tensors[size_t(rt.spec)].cols;
      if (!covered(rt.offset, cnt)) continue;
      const float sc = float(role.dp_weight / double(rt.multiplicity));
      if (bf)
        k_scale_cast(G32 + rt.offset, G16 + rt.offset, cnt, sc, s);
      else
        k_scale(G32 + rt.offset, cnt, sc, s);
      kcheck("scale");
    }
    if (!g.buckets.empty()) {
      HX_NCCL(ncclGroupStart());
      for (const auto& b : g.buckets) {
        if (bf)
          HX_NCCL(ncclAllReduce(G16 + b.offset, G16 + b.offset, size_t(b.count), ncclBfloat16,
                                ncclSum, comms[size_t(b.comm)], s));
        else
          HX_NCCL(ncclAllReduce(G32 + b.offset, G32 + b.offset, size_t(b.count), ncclFloat32,
                                ncclSum, comms[size_t(b.comm)], s));
        ++nccl_calls_step;
      }
      HX_NCCL(ncclGroupEnd());
    }
    for (size_t ti : g.tensors) {
      const RankTensor& rt = role.tensors[ti];
      const TensorSpec& ts = L.tensors[size_t(rt.spec)];
      const int64_t cnt = rt.rows * ts.cols;
      const float wd = ts.decay ? cfg.weight_decay : 0.f;
      const bool cov = covered(rt.offset, cnt);
      const bf16* g16 = cov && bf ? G16 + rt.offset : nullptr;
      const float* g32 = g16 ? nullptr : G32 + rt.offset;
      const float gscale = cov ? 1.f : float(role.dp_weight / double(rt.multiplicity));
      k_adamw(P32 + rt.offset, P16 + rt.offset, Mo + rt.offset, Vo + rt.offset, g16, g32, cnt,
              gscale, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, wd, 0.f, 0.f, s, sp_);
      kcheck("adamw");
    }
  }

  // group `id` is final on the compute stream: hand it to the comm stream
  void group_ready(int id) {
    if (!cfg.dp_overlap || !last_mb_) return;
    for (auto& g : groups_) {
      if (g.id != id) continue;
      HX_CUDA(cudaEventRecord(g.ready, stream));
      HX_CUDA(cudaStreamWaitEvent(cstream, g.ready, 0));
      group_work(g, cstream);
    }
  }

  void dp_sync_and_update() {
    const auto& buckets = L.dp_buckets[size_t(rank)];
    cudaEventRecordWithFlags(ev[2], stream, capturing_ ? cudaEventRecordExternal : 0);
    const bool bf = G16 != nullptr;
    // 1. weight by samples: scale = (batch_i / global_batch) / multiplicity, fused
    //    with the bf16 cast for tensors that take part in a DP allreduce
    for (const auto& rt : role.tensors) {
      const int64_t cnt = rt.rows * L.tensors[size_t(rt.spec)].cols;
      if (!covered(rt.offset, cnt)) continue;
      const float sc = float(role.dp_weight / double(rt.multiplicity));
      if (bf)
        k_scale_cast(G32 + rt.offset, G16 + rt.offset, cnt, sc, stream);
      else
        k_scale(G32 + rt.offset, cnt, sc, stream);
      kcheck("scale");
    }
    // 2. chunk-matched allreduce, one NCCL call per bucket (grouped)
    if (!buckets.empty()) {
      HX_NCCL(ncclGroupStart());
      for (const auto& b : buckets) {
        if (bf)
          HX_NCCL(ncclAllReduce(G16 + b.offset, G16 + b.offset, size_t(b.count), ncclBfloat16,
                                ncclSum, comms[size_t(b.comm)], stream));
        else
          HX_NCCL(ncclAllReduce(G32 + b.offset, G32 + b.offset, size_t(b.count), ncclFloat32,
                                ncclSum, comms[size_t(b.comm)], stream));
        ++nccl_calls_step;
      }
      HX_NCCL(ncclGroupEnd());
      mark("nccl_dp_allreduce");
    }
    cudaEventRecordWithFlags(ev[3], stream, capturing_ ? cudaEventRecordExternal : 0);
    // 3. AdamW per tensor (weight decay only on matrices)
    const float t = float(step_index + 1);
    const float bc1 = 1.f - std::pow(cfg.beta1, t);
    const float bc2 = 1.f - std::pow(cfg.beta2, t);
    for (const auto& rt : role.tensors) {
      const TensorSpec& ts = L.tensors[size_t(rt.spec)];
      const int64_t cnt = rt.rows * ts.cols;
      const float wd = ts.decay ? cfg.weight_decay : 0.f;
      const bool cov = covered(rt.offset, cnt);
      const bf16* g16 = cov && bf ? G16 + rt.offset : nullptr;
      const float* g32 = g16 ? nullptr : G32 + rt.offset;
      const float gscale = cov ? 1.f : float(role.dp_weight / double(rt.multiplicity));
      k_adamw(P32 + rt.offset, P16 + rt.offset, Mo + rt.offset, Vo + rt.offset, g16, g32, cnt,
              gscale, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, wd, bc1, bc2, stream, sp_);
      kcheck("adamw");
    }
    cudaEventRecordWithFlags(ev[4], stream, capturing_ ? cudaEventRecordExternal : 0);
  }

  // is [off, off+cnt) fully covered by this rank's DP buckets? (buckets never
  // partially cover a tensor unless its shard boundaries differ across pipelines,
  // in which case the uncovered part has a single holder)
  bool covered(int64_t off, int64_t cnt) const {
    int64_t c = 0;
    for (const auto& b : L.dp_buckets[size_t(rank)]) {
      int64_t lo = std::max(off, b.offset), hi = std::min(off + cnt, b.offset + b.count);
      if (hi > lo) c += hi - lo;
    }
    return c == cnt;
  }

  // ------------------------------------------------------------ graph replay
  // After one eager step (NCCL / lazy init warm-up), the whole step -- every
  // kernel, memset, NCCL call and timing event -- is captured once into a CUDA
  // graph and replayed; per-step scalars live in device StepParams.
  cudaGraphExec_t gexec_ = nullptr;
  int64_t graph_launches_ = 0;
  StepParams* sp_ = nullptr;

  void step_enqueue() {
    if (!role.active) {
      // idle device: still joins the world loss reduction (contributes 0)
      HX_CUDA(cudaMemsetAsync(loss_acc, 0, 4, stream));
      finish_loss();
      ++step_index;
      return;
    }
    const bool gen = tokens_from_host_ == nullptr && (role.first_stage || role.last_stage);
    HX_CUDA(cudaMemsetAsync(&sp_->gen_tokens, gen ? 1 : 0, sizeof(int), stream));
    const bool graph = cfg.cuda_graph && !cfg.profile_gemm;
    (void)cudaGetLastError();  // clear non-sticky errors (e.g. a not-ready event query)
    if (graph && gexec_) {
      ev = ev_graph_;
      HX_CUDA(cudaGraphLaunch(gexec_, stream));
      launches_step = graph_launches_;
    } else if (graph && step_index >= 1) {
      ev = ev_graph_;  // the graph owns its own phase events
      HX_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed));
      cudaGraph_t g = nullptr;
      capturing_ = true;
      try {
        enqueue_body();
      } catch (...) {
        capturing_ = false;
        cudaStreamEndCapture(stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      capturing_ = false;
      HX_CUDA(cudaStreamEndCapture(stream, &g));
      cudaError_t e = cudaGraphInstantiate(&gexec_, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) throw CudaError(std::string("graph instantiate: ") + cudaGetErrorString(e));
      graph_launches_ = launches_step;
      HX_CUDA(cudaGraphLaunch(gexec_, stream));
    } else {
      ev = ev_eager_;
      enqueue_body();
    }
    launches_total += launches_step;
    ++step_index;
  }

  void enqueue_body() {
    launches_step = 0;
    copies_step = 0;
    xop_ = 0;
    nccl_calls_step = 0;
    cudaEventRecordWithFlags(ev[0], stream, capturing_ ? cudaEventRecordExternal : 0);
    k_step_tick(sp_, cfg.beta1, cfg.beta2, stream);
    kcheck("step_tick");
    if (role.first_stage || role.last_stage) {
      k_gen_tokens(tokens, role.batch, int(S), role.sample0, cfg.seed, 0,
                   int(L.model.vocab_size), stream, sp_);
      kcheck("gen_tokens");
    }
    HX_CUDA(cudaMemsetAsync(loss_acc, 0, 4, stream));
    ++copies_step;
    // zero the atomically-accumulated grads (norm gains, embedding)
    for (const auto& rt : role.tensors) {
      const TensorSpec& ts = L.tensors[size_t(rt.spec)];
      if (ts.id == kAttnNorm || ts.id == kMlpNorm || ts.id == kFinalNorm || ts.id == kEmbed) {
        HX_CUDA(cudaMemsetAsync(G32 + rt.offset, 0, size_t(rt.rows * ts.cols) * 4, stream));
        ++copies_step;
      }
    }
    mark("prologue");
    cudaEventRecordWithFlags(ev[1], stream, capturing_ ? cudaEventRecordExternal : 0);
    if (cfg.dp_overlap) {
      // fork the comm stream into this step (and into the graph when capturing)
      HX_CUDA(cudaEventRecord(join_ev_, stream));
      HX_CUDA(cudaStreamWaitEvent(cstream, join_ev_, 0));
    }
    run_pipeline();
    // even number of exchanges per step: ring buffer b = op & 1 alternates
    // across the step boundary too (the double-buffer hand-off argument)
    if (tp_peer_ && (xop_ & 1u)) {
      pad_ = true;
      tp_sync();
      pad_ = false;
    }
    if (cfg.dp_overlap) {
      HX_CUDA(cudaEventRecord(join_ev_, cstream));
      HX_CUDA(cudaStreamWaitEvent(stream, join_ev_, 0));
      cudaEventRecordWithFlags(ev[2], stream, capturing_ ? cudaEventRecordExternal : 0);
      cudaEventRecordWithFlags(ev[3], stream, capturing_ ? cudaEventRecordExternal : 0);
      cudaEventRecordWithFlags(ev[4], stream, capturing_ ? cudaEventRecordExternal : 0);
    } else {
      dp_sync_and_update();
    }
    finish_loss();
    cudaEventRecordWithFlags(ev[5], stream, capturing_ ? cudaEventRecordExternal : 0);
  }

  void finish_loss() {
    if (world > 1) {
      HX_NCCL(ncclAllReduce(loss_acc, loss_acc, 1, ncclFloat32, ncclSum, world_comm, stream));
      ++nccl_calls_step;
    }
  }

  cudaStream_t stream_or_default() { return stream; }

  const int32_t* tokens_from_host_ = nullptr;

  void step(const int32_t* host_tokens, size_t n, float* loss_out) {
    if (role.active && host_tokens) {
      const size_t need = size_t(role.batch * (S + 1));
      if (n != need)
        throw InvalidArgument("tokens: expected " + std::to_string(need) + " values for this pipeline");
      std::memcpy(tokens_pinned, host_tokens, need * 4);
      HX_CUDA(cudaMemcpyAsync(tokens, tokens_pinned, need * 4, cudaMemcpyHostToDevice, stream));
    }
    tokens_from_host_ = host_tokens;
    step_enqueue();
    tokens_from_host_ = nullptr;
    HX_CUDA(cudaMemcpyAsync(loss_host, loss_acc, 4, cudaMemcpyDeviceToHost, stream));
    HX_CUDA(cudaStreamSynchronize(stream));
    last_loss = loss_host[0] / float(L.plan.global_batch * S);
    if (role.active) collect_times();
    steps_since_collect_ = 1;
    collect_gemm_profile();
    collect_graph_gemm();
    collect_timeline();
    if (loss_out) *loss_out = last_loss;
  }

  void collect_times() {
    float t;
    if (cudaEventElapsedTime(&t, ev[0], ev[1]) == cudaSuccess) phase_ms[0] = t;
    if (cudaEventElapsedTime(&t, ev[1], ev[2]) == cudaSuccess) phase_ms[1] = t;
    if (cudaEventElapsedTime(&t, ev[2], ev[3]) == cudaSuccess) phase_ms[2] = t;
    if (cudaEventElapsedTime(&t, ev[3], ev[4]) == cudaSuccess) phase_ms[3] = t;
    if (cudaEventElapsedTime(&t, ev[0], ev[5]) == cudaSuccess) phase_ms[4] = t;
    (void)cudaGetLastError();
  }

  std::string stats() const {
    ojson j;
    j["rank"] = rank;
    j["active"] = role.active;
    j["sm_total"] = sm_total;
    j["sm_applied"] = sm_applied;
    j["sm_cap_mode"] = sm_mode;
    j["attention"] = attention_note_.empty() ? cfg.attention : attention_note_;
    j["wgrad_group"] = wg_;
    j["wgrad_group_buffers"] = wg_nbuf_;
    j["tp_reduce"] = tp_peer_ ? (tp_crit_ >= 0 ? "peer(pull from tp rank " + std::to_string(tp_crit_) + ")" : std::string("peer(push)")) : (role.tp > 1 ? std::string("nccl") : std::string("none"));
    j["sm_fraction"] = role.sm_fraction;
    j["arena_bytes"] = arena.total();
    j["activation_slots"] = n_slots;
    j["param_count"] = role.param_count;
    j["steps"] = step_index;
    j["launches_last_step"] = launches_step;
    j["launches_total"] = launches_total;
    j["copy_nodes_last_step"] = copies_step;
    j["nccl_calls_last_step"] = nccl_calls_step;
    j["ms"] = {{"prologue", phase_ms[0]}, {"pipeline", phase_ms[1]}, {"dp_sync", phase_ms[2]},
               {"optimizer", phase_ms[3]}, {"step", phase_ms[4]}};
    j["last_loss"] = last_loss;
    if (cfg.profile_gemm) {
      const char* names[3] = {"tp_linear", "attention", "lm_head"};
      ojson g;
      for (int k = 0; k < 3; ++k)
        g[names[k]] = {{"launches", gemm_count_[k]}, {"ms", gemm_ms_[k]},
                       {"flops", gemm_flops_[k]},
                       {"tflops", gemm_ms_[k] > 0 ? gemm_flops_[k] / gemm_ms_[k] / 1e9 : 0.0}};
      g["steps"] = steps_since_collect_;
      j["gemm_profile"] = g;
      ojson tl;
      for (const auto& [k, v] : timeline_) tl[k] = {{"ms", v.first}, {"ops", v.second}};
      j["timeline_ms"] = tl;
    }
    if (!gmarks_.empty()) {
      std::map<std::string, std::pair<double, int64_t>> t;
      for (size_t i = 1; i < gmarks_.size(); ++i) {
        if (gmarks_[i].run != gmarks_[i - 1].run) continue;
        float ms = 0;
        if (cudaEventElapsedTime(&ms, gmarks_[i - 1].ev, gmarks_[i].ev) != cudaSuccess) continue;
        auto& v = t[gmarks_[i].kind];
        v.first += ms;
        v.second += 1;
      }
      (void)cudaGetLastError();
      ojson tl;
      for (const auto& [k, v] : t) tl[k] = {{"ms", v.first}, {"ops", v.second}};
      j["timeline_graph_one_mb"] = tl;
    }
    if (!graph_recs_.empty()) {
      const char* names[3] = {"tp_linear", "attention", "lm_head"};
      ojson g;
      for (int k = 0; k < 3; ++k)
        g[names[k]] = {{"launches", ggemm_count_[k]}, {"ms", ggemm_ms_[k]},
                       {"flops", ggemm_flops_[k]},
                       {"tflops", ggemm_ms_[k] > 0 ? ggemm_flops_[k] / ggemm_ms_[k] / 1e9 : 0.0}};
      g["steps"] = 1;
      g["micro_batches_sampled"] = 1;
      g["micro_batches"] = role.n_mb;
      g["source"] = "CUDA events captured in the step graph around micro-batch n_mb/2's GEMMs, last replay";
      std::map<std::string, std::tuple<double, double, int64_t>> by;
      for (size_t i = 0; i < graph_recs_.size(); ++i) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, graph_recs_[i].a, graph_recs_[i].b) != cudaSuccess) continue;
        auto& t = by[graph_shapes_[i]];
        std::get<0>(t) += ms;
        std::get<1>(t) += graph_recs_[i].flops;
        std::get<2>(t) += 1;
      }
      (void)cudaGetLastError();
      ojson sh = ojson::array();
      for (const auto& [k, v] : by)
        sh.push_back({{"shape", k}, {"launches", std::get<2>(v)}, {"ms", std::get<0>(v)},
                      {"tflops", std::get<0>(v) > 0 ? std::get<1>(v) / std::get<0>(v) / 1e9 : 0.0}});
      g["shapes"] = sh;
      j["gemm_profile_graph"] = g;
    }
    return j.dump();
  }
};

// ------------------------------------------------------------------ free functions
Executor* make_executor(const std::string& c, const std::string& m, const std::string& p,
                        const std::string& x, int r, int w, int dev, const void* uid,
                        size_t uid_len) {
  auto* e = new Executor();
  try {
    e->init(c, m, p, x, r, w, dev, uid, uid_len);
  } catch (...) {
    delete e;
    throw;
  }
  return e;
}

void executor_step(Executor& e, const int32_t* t, size_t n, float* loss) { e.step(t, n, loss); }

void executor_step_async(Executor& e) {
  e.tokens_from_host_ = nullptr;
  if (e.gemm_used_ == 0) e.steps_since_collect_ = 0;
  e.step_enqueue();
  ++e.steps_since_collect_;
}

void executor_set_profile(Executor& e, bool on) {
  // NCCL work captured in the step graph must not be followed by eager NCCL
  // work on the same communicators (observed to hang): profile before capture
  if (on && e.gexec_ && e.world > 1)
    throw InvalidArgument("profiling must be enabled before the step graph is captured");
  e.cfg.profile_gemm = on;
}

void executor_timer(Executor& e, int stop, float* ms) {
  if (!stop) {
    HX_CUDA(cudaEventRecord(e.tmr_[0], e.stream));
    return;
  }
  HX_CUDA(cudaEventRecord(e.tmr_[1], e.stream));
  HX_CUDA(cudaEventSynchronize(e.tmr_[1]));
  HX_CUDA(cudaEventElapsedTime(ms, e.tmr_[0], e.tmr_[1]));
}

void executor_sync(Executor& e) {
  if (e.stream) HX_CUDA(cudaStreamSynchronize(e.stream));
  HX_CUDA(cudaMemcpy(e.loss_host, e.loss_acc, 4, cudaMemcpyDeviceToHost));
  e.last_loss = e.loss_host[0] / float(e.L.plan.global_batch * e.S);
  if (e.role.active) e.collect_times();
  e.collect_gemm_profile();
  e.collect_graph_gemm();
  e.collect_timeline();
}

float executor_last_loss(Executor& e) { return e.last_loss; }

void executor_synth_tokens(const Executor& e, int64_t step, int32_t* out, size_t n) {
  if (!e.role.active) return;
  const int64_t S1 = e.S + 1;
  if (n != size_t(e.role.batch * S1)) throw InvalidArgument("tokens: wrong buffer size");
  for (int64_t i = 0; i < e.role.batch; ++i) {
    uint64_t base = mix_seed(e.cfg.seed, kTokenTag, uint64_t(step), uint64_t(e.role.sample0 + i));
    for (int64_t p = 0; p < S1; ++p)
      out[i * S1 + p] = int32_t(splitmix64(base + uint64_t(p)) % uint64_t(e.L.model.vocab_size));
  }
}

bool executor_tensor_info(const Executor& e, const std::string& name, int64_t* row0,
                          int64_t* rows, int64_t* cols, int64_t* grows) {
  for (const auto& ts : e.L.tensors) {
    if (ts.name != name) continue;
    *cols = ts.cols;
    *grows = ts.global_rows;
    *row0 = 0;
    *rows = 0;
    auto it = e.named.find(name);
    if (it != e.named.end()) {
      *row0 = it->second.row0;
      *rows = it->second.rows;
    }
    return true;
  }
  return false;
}

void executor_read_tensor(Executor& e, const std::string& name, int which, float* out, size_t n) {
  auto it = e.named.find(name);
  if (it == e.named.end()) throw InvalidArgument("tensor not held by this rank: " + name);
  const TensorPtrs& t = it->second;
  if (n != size_t(t.count)) throw InvalidArgument("read_tensor: wrong element count");
  HX_CUDA(cudaStreamSynchronize(e.stream));
  switch (which) {
    case 0:
      HX_CUDA(cudaMemcpy(out, t.p32, n * 4, cudaMemcpyDeviceToHost));
      break;
    case 1: {
      // the gradient AdamW consumed (DP-reduced, sample-weighted)
      const RankTensor* rt = nullptr;
      for (const auto& r : e.role.tensors)
        if (r.spec == t.spec) rt = &r;
      const bool cov = e.covered(t.offset, t.count);
      if (cov && e.G16) {
        std::vector<uint16_t> tmp(n);
        HX_CUDA(cudaMemcpy(tmp.data(), e.G16 + t.offset, n * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) {
          uint32_t u = uint32_t(tmp[i]) << 16;
          std::memcpy(&out[i], &u, 4);
        }
      } else {
        HX_CUDA(cudaMemcpy(out, t.g32, n * 4, cudaMemcpyDeviceToHost));
        if (!cov) {
          float sc = float(e.role.dp_weight / double(rt ? rt->multiplicity : 1));
          for (size_t i = 0; i < n; ++i) out[i] *= sc;
        }
      }
      break;
    }
    case 2:
      HX_CUDA(cudaMemcpy(out, e.Mo + t.offset, n * 4, cudaMemcpyDeviceToHost));
      break;
    case 3:
      HX_CUDA(cudaMemcpy(out, e.Vo + t.offset, n * 4, cudaMemcpyDeviceToHost));
      break;
    default:
      throw InvalidArgument("read_tensor: which must be 0..3");
  }
}

std::string executor_stats_json(const Executor& e) { return e.stats(); }

// SM placement of this rank's work (tests of the SM cap): what = 0 a probe
// kernel of n CTAs on the executor stream, 1 the same on the comm stream,
// 2 one persistent 4096 x 4096 x 1024 GEMM on
// the executor stream with every CTA logging its %smid (n = its grid, <= n
// entries written).  out receives the SM ids; returns the entries written.
int executor_sm_probe(Executor& e, int what, int* out, int n) {
  if (!e.stream) throw CudaError("executor has no device state (validate_only)");
  if (n <= 0) return 0;
  cudaStream_t s = what == 1 ? (e.cstream ? e.cstream : e.stream) : e.stream;
  int* log = nullptr;
  HX_CUDA(cudaMalloc(&log, size_t(n) * sizeof(int)));
  HX_CUDA(cudaMemsetAsync(log, 0xff, size_t(n) * sizeof(int), s));
  int written = n;
  if (what == 2) {
    if (!e.role.active) {
      cudaFree(log);
      throw InvalidArgument("sm_probe: idle rank holds no GEMM operands");
    }
    // a fixed 4096 x 4096 x 1024 GEMM (256 CTA-pair tiles: every SM the
    // rank may use gets work) on zeroed scratch operands
    const int64_t Mg = 4096, Hh = 4096;
    bf16* a = nullptr;
    float* c = nullptr;
    HX_CUDA(cudaMalloc(&a, size_t(Mg * Hh) * 2));
    HX_CUDA(cudaMalloc(&c, size_t(Mg * Hh) * 4));
    HX_CUDA(cudaMemsetAsync(a, 0, size_t(Mg * Hh) * 2, s));
    GemmDesc g = e.g2(Mg, Hh, 1024, a, 0, 1024, a, 0, 1024, c, Hh, 1);
    gemm_set_smid_log(log);
    cudaError_t err = gemm_bf16(g, s);
    gemm_set_smid_log(nullptr);
    HX_CUDA(err);
    HX_CUDA(cudaStreamSynchronize(s));
    cudaFree(a);
    cudaFree(c);
  } else {
    k_smid_probe(log, n, s);
    HX_CUDA(cudaGetLastError());
  }
  HX_CUDA(cudaMemcpyAsync(out, log, size_t(n) * sizeof(int), cudaMemcpyDeviceToHost, s));
  HX_CUDA(cudaStreamSynchronize(s));
  cudaFree(log);
  if (what == 2) {
    written = 0;
    for (int i = 0; i < n; ++i)
      if (out[i] >= 0) written = i + 1;
  }
  return written;
}

void destroy_executor(Executor* e) { delete e; }

}  // namespace hexexec
