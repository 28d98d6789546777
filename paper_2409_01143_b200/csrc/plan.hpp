// Plan ingestion and integer bookkeeping for the executor (host only).
//
// Data model mirrors the reference (proj/src/types.hpp:58-85): a plan is a
// list of pipelines (DP replicas with their own batch / micro_batch), each a
// list of stages (TP device group + contiguous layer range), plus one DP group
// per layer.  Extensions read from keys the reference parser ignores:
//   model  : num_heads, ffn_dim, vocab_size, rope_theta, norm_eps
//   device : rank (world rank), sm_fraction / sm_count
//   stage  : tp_widths (relative integer weights, one per device)
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hexexec {

// error classes -> hexexec_status at the ABI (same split as the reference's
// proj/src/errors.hpp:9-26, plus CUDA / NCCL)
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidArgument : std::runtime_error { using std::runtime_error::runtime_error; };
struct Infeasible : std::runtime_error { using std::runtime_error::runtime_error; };
struct LimitExceeded : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NcclError : std::runtime_error { using std::runtime_error::runtime_error; };

struct Device {
  std::string id;
  std::string machine;
  double memory_gib = 0;
  double peak_tflops = 0;
  int rank = -1;             // world rank (extension "rank"; default = document order)
  double sm_fraction = 0;    // 0 = derive from peak_tflops / max peak
  int sm_count = 0;          // explicit SM count (extension), overrides fraction
};

struct Cluster {
  std::vector<Device> devices;
  // link matrices as json_io.cpp:149-171 expands them: same machine -> the
  // machine's intra link, else the inter link, then per-pair overrides;
  // bytes/s ("gbps" in the documents means GB/s, json_io.cpp:20) and seconds
  std::vector<std::vector<double>> bandwidth, latency;
  int device_index(const std::string& id) const;
  double max_peak() const;
};

struct Model {
  int64_t num_layers = 0, hidden_dim = 0, seq_len = 0, bytes_per_element = 0;
  int64_t num_heads = 0, ffn_dim = 0, vocab_size = 0;
  double rope_theta = 10000.0, norm_eps = 1e-5;
  int64_t head_dim() const { return hidden_dim / num_heads; }
};

struct Stage {
  std::vector<int> devices;  // cluster device indices
  int tp = 1;
  int layer_start = 0, layer_count = 0;
  std::vector<int64_t> tp_widths;  // empty = equal widths (reference semantics)
};

struct Pipeline {
  std::vector<Stage> stages;
  int64_t batch = 0, micro_batch = 0;
  // reference types.hpp:70-72
  int64_t num_micro_batches() const { return micro_batch > 0 ? batch / micro_batch : 0; }
};

struct DpGroup {
  int layer = 0;
  std::vector<int> members;
};

struct Plan {
  std::vector<Pipeline> pipelines;
  std::vector<DpGroup> dp_groups;
  int64_t global_batch = 0;
};

struct Range {
  int64_t begin = 0, end = 0;
  int64_t size() const { return end - begin; }
};

// global tensor catalogue
enum TensorId : int {
  kEmbed = 0, kAttnNorm = 1, kWqkv = 2, kWo = 3, kMlpNorm = 4, kWgu = 5, kWdown = 6,
  kFinalNorm = 7, kLmHead = 8
};

struct TensorSpec {
  std::string name;
  int layer = -1;  // -1 for embed / final_norm / lm_head
  int id = 0;
  int64_t global_rows = 0, cols = 0;
  bool decay = true;
};

struct RankTensor {
  int spec = -1;           // index into Layout::tensors
  int64_t row0 = 0, rows = 0;
  int64_t offset = 0;      // element offset in the rank's flat parameter buffer
  int multiplicity = 1;    // holders of each element inside this rank's pipeline
};

struct RankRole {
  bool active = false;
  int device = -1;         // cluster device index
  int pipeline = -1, stage = -1, tp_index = 0, tp = 1;
  int layer_start = 0, layer_count = 0;
  bool first_stage = false, last_stage = false;
  Range heads, ffn_chunks, vocab_chunks;  // ffn/vocab in units of 64
  int64_t sample0 = 0, batch = 0, micro_batch = 0, n_mb = 0;
  std::vector<int> tp_group;        // world ranks of the stage, tp order
  int fwd_recv_from = -1, bwd_recv_from = -1;
  std::vector<int> fwd_send_to, bwd_send_to;
  int stage_count = 1;
  double dp_weight = 1.0;           // batch / global_batch
  std::vector<RankTensor> tensors;  // in flat-buffer order
  int64_t param_count = 0;
  double sm_fraction = 1.0;
  int sm_count = 0;
};

// DP sync bucket: a contiguous local range summed over `comm` (a rank set)
struct DpBucket {
  int comm = -1;          // index into Layout::comm_sets
  int64_t offset = 0, count = 0;
  int group = 0;          // sync group (layer index, kGroupEmbed, kGroupHead)
};

// gradients become final in backward order: head, layers descending, embedding
constexpr int kGroupEmbed = -1;
constexpr int kGroupHead = -2;
int sync_group(const TensorSpec& t);

struct ScaleSeg {
  int64_t offset = 0, count = 0;
  float scale = 1.f;
};

struct Layout {
  Cluster cluster;
  Model model;
  Plan plan;
  int world_size = 0;
  std::vector<int> rank_of_device;   // cluster index -> world rank
  std::vector<int> device_of_rank;
  std::vector<TensorSpec> tensors;   // global catalogue
  std::vector<RankRole> roles;       // per world rank
  std::vector<std::vector<int>> comm_sets;  // sorted rank sets (size >= 2)
  std::vector<std::vector<DpBucket>> dp_buckets;  // per world rank
  std::vector<std::vector<ScaleSeg>> dp_scales;   // per world rank
  std::vector<int> tp_comm;          // per world rank: comm set of its TP group or -1
};

// documents -> structures (throw ParseError / InvalidArgument)
Cluster parse_cluster_doc(const std::string& text);
Model parse_model_doc(const std::string& text);
Plan parse_plan_doc(const std::string& text, const Cluster& c, bool* had_dp_groups);

// reference semantics (cost_model.cpp:155-208)
void build_dp_groups(Plan& plan, const Model& m);
void validate_plan(const Plan& plan, const Model& m, const Cluster& c);

// largest-remainder split of `units` by integer weights; ties -> lower index
std::vector<int64_t> largest_remainder(int64_t units, const std::vector<int64_t>& weights);

// everything an executor rank needs; throws on inconsistent inputs
Layout build_layout(const std::string& cluster_json, const std::string& model_json,
                    const std::string& plan_json);

std::string serialize_plan(const Plan& plan, const Cluster& c);
std::string layout_json(const Layout& L);

}  // namespace hexexec
