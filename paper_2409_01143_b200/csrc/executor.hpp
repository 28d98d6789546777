// Per-rank executor of one asymmetric-parallel training step.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace hexexec {

struct ExecConfig {
  uint64_t seed = 0;
  float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.1f;
  std::string sm_cap = "green";       // "green" | "cta" | "none"
  std::string dp_comm_dtype = "bf16"; // "bf16" | "fp32"
  bool validate_only = false;
  bool profile_gemm = false;          // per-GEMM CUDA events (roofline evidence); eager
  bool graph_gemm_events = false;     // per-GEMM CUDA events inside the step graph
  bool fuse_swiglu = true;            // SwiGLU in the gate-up GEMM epilogue
  bool fuse_rope = true;              // RoPE (forward) in the QKV GEMM epilogue
  // weight-gradient GEMMs over G token-concatenated micro-batches: -1 = auto
  // (all micro-batches that fit in memory), 0/1 = per micro-batch, G = force.
  // Off by default: +18-20 % wgrad throughput in isolation
  // (scripts/bench_wgrad_concat.py), but a full-SM B200 is power-capped and
  // the step time stayed flat (100.9 vs 101.0 ms, the clock dropped
  // 1507 -> 1372 MHz) while the stash costs 9-90 GiB per rank
  int wgrad_group = 1;
  // programmatic dependent launch of the GEMMs (prologue overlaps the
  // previous kernel's tail); off: no measurable change on the power-capped
  // step (100.9-101.2 ms either way)
  bool pdl = false;
  bool cuda_graph = true;             // replay the captured step graph (after step 0)
  std::string attention = "fused";    // "fused" (flash, tcgen05) | "unfused" (GEMM+softmax)
  bool dp_overlap = true;             // DP sync + AdamW per layer on a second stream
  // split-K of each GEMM's partial last wave (+3-7% on the affected GEMMs,
  // ~1% of the step); partial sums land in arbitrary order, so it costs
  // run-to-run bitwise determinism and is opt-in
  bool gemm_split = false;
  // activation recompute: keep only each layer's input per
  // micro-batch slot and re-run the layer forward (minus its output GEMM)
  // before the layer backward, into one shared activation set
  bool recompute = false;
  // PP hand-off (cost_model.cpp:59-76): "direct" = every rank of
  // the receiving stage gets its copy from a sender rank; "leader" = the
  // stages' first devices exchange it and the receiving leader broadcasts it
  // over its TP communicator (for links where only leaders are well connected)
  std::string pp_protocol = "direct";
  // PP payload dtype: "bf16" = the 2-byte hand-off comm_pp_hop prices
  // (cost_model.cpp:10-13, :59-76); "fp32" = the residual stream as is
  std::string pp_dtype = "bf16";
  // TP reduction of the row-parallel partials: "peer" = the producing GEMM's
  // epilogue TMA-stores its partial into every TP peer's exchange buffer
  // (IPC-mapped, NVLink) while it runs, a flag handshake orders it, and the
  // consumer (RMSNorm / residual add) sums the slots; "nccl" = ncclAllReduce
  std::string tp_reduce = "peer";
  // "auto": the critical rank of an uneven TP stage does not push (the others
  // pull its partial); "push": every rank pushes
  std::string tp_direction = "auto";
  // how the faster ranks pull the critical rank's partial: "sm" = copy kernel
  // with remote 16-byte loads, "ce" = copy-engine cudaMemcpyAsync; both ~400 GB/s
  // (41 us per 16 MiB slot) and the same step time
  std::string tp_pull = "ce";
};

ExecConfig parse_exec_config(const std::string& text);

class Executor;

Executor* make_executor(const std::string& cluster, const std::string& model,
                                        const std::string& plan, const std::string& cfg,
                                        int world_rank, int world_size, int cuda_device,
                                        const void* uid, size_t uid_len);
void executor_step(Executor& e, const int32_t* tokens_host, size_t n, float* loss_out);
void executor_step_async(Executor& e);
void executor_sync(Executor& e);
// device time between a start (stop=0) and stop (stop=1) mark on the executor stream
void executor_timer(Executor& e, int stop, float* ms);
void executor_set_profile(Executor& e, bool on);
float executor_last_loss(Executor& e);
void executor_synth_tokens(const Executor& e, int64_t step, int32_t* out, size_t n);
bool executor_tensor_info(const Executor& e, const std::string& name, int64_t* row0,
                          int64_t* rows, int64_t* cols, int64_t* grows);
void executor_read_tensor(Executor& e, const std::string& name, int which, float* out,
                          size_t n);
std::string executor_stats_json(const Executor& e);
int executor_sm_probe(Executor& e, int what, int* out, int n);
void destroy_executor(Executor* e);

}  // namespace hexexec
