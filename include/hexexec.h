/* hexexec: B200-native executor for HexiScale's asymmetric-parallel
 * transformer training step.  Consumes the allocation-plan documents that the
 * reference planner emits (hexplan_result_plan_json, reference
 * proj/src/capi.cpp:344-347, serialized by proj/src/report.cpp:25-64; or the
 * CLI's wrapped {"manifest","plan"} form, proj/tools/hexplan_cli.cpp:217-218)
 * together with the reference's cluster and model documents
 * (proj/src/json_io.cpp:80-191).
 *
 * Conventions mirror hexplan.h (reference proj/include/hexplan.h:1-27):
 * opaque handles; every fallible call returns a status and fills an optional
 * NUL-terminated, safely truncated err buffer (capi.cpp:34-39); null
 * arguments give HEXEXEC_ERR_INVALID (capi.cpp:96-99); no exception crosses
 * the ABI (capi.cpp:49-73); strings are malloc'd and released with
 * hexexec_string_free (capi.cpp:41-46, :404).  Tensors are exported into
 * caller-owned buffers.  There is no CPU compute path: step/kernel calls on a
 * host without a CUDA device return HEXEXEC_ERR_CUDA. */
#ifndef HEXEXEC_H
#define HEXEXEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hexexec_status {
  HEXEXEC_OK = 0,
  HEXEXEC_ERR_PARSE = 1,      /* malformed input document (= HEXPLAN_ERR_PARSE) */
  HEXEXEC_ERR_INVALID = 2,    /* argument / plan violates a precondition (= HEXPLAN_ERR_INVALID) */
  HEXEXEC_ERR_INFEASIBLE = 3, /* plan does not fit (memory) (= HEXPLAN_ERR_INFEASIBLE) */
  HEXEXEC_ERR_LIMIT = 4,      /* instance exceeds a hard size limit (= HEXPLAN_ERR_LIMIT) */
  HEXEXEC_ERR_INTERNAL = 5,   /* (= HEXPLAN_ERR_INTERNAL) */
  HEXEXEC_ERR_CUDA = 6,       /* CUDA runtime/driver failure or no device (extension) */
  HEXEXEC_ERR_NCCL = 7        /* NCCL failure (extension) */
} hexexec_status;

typedef struct hexexec_plan hexexec_plan; /* host-only: parsed + validated plan and rank layout */
typedef struct hexexec_ctx hexexec_ctx;   /* one executor rank: device state, comms, step */

/* ---- plan ingestion and bookkeeping (host only, no device needed) ------
 * Replaces: the reference has no plan parser; invariants are
 * validate_plan (proj/src/cost_model.cpp:166-208), DP groups build_dp_groups
 * (:155-164), micro-batch counts PipelinePlan::num_micro_batches
 * (proj/src/types.hpp:70-72).  plan_json may be bare or CLI-wrapped. */
hexexec_status hexexec_plan_parse(const char* cluster_json, const char* model_json,
                                  const char* plan_json, hexexec_plan** out, char* err,
                                  size_t err_len);
/* Re-serialization of the plan in the reference's wire format
 * (report.cpp:25-53, dump(2) + "\n"): byte-identical for reference plans. */
char* hexexec_plan_serialize(const hexexec_plan* p);
/* Full integer layout as JSON: per world rank (pipeline, stage, tp index,
 * head/ffn/vocab shard ranges, sample range), per-pipeline micro-batch map,
 * dp_groups, TP/PP peers, and the chunk-matched DP segment table. */
char* hexexec_plan_layout_json(const hexexec_plan* p);
int hexexec_plan_world_size(const hexexec_plan* p);
/* The reference cost model on this plan (cost_model.cpp:210-258
 * iteration_time, report.cpp:66-93 JSON fields), malloc'd into *report_json.
 * extension = 0: the reference formula (mixed-speed TP stages -> INVALID
 * "mixed-type tensor parallel stage", like the reference); extension = 1:
 * TP stage compute = max_r(w_r/sum(w) * FLOPs / c_r) for uneven tp_widths /
 * mixed device speeds.  Replaces pricing through hexplan's C++ API. */
hexexec_status hexexec_plan_cost(const hexexec_plan* p, double state_multiplier, int extension,
                                 char** report_json, char* err, size_t err_len);
/* MFU in the reference convention (cost_model.cpp:260-265) for a measured
 * step time over this plan's cluster; 0 for a non-positive time. */
double hexexec_plan_mfu(const hexexec_plan* p, double seconds);
void hexexec_plan_free(hexexec_plan* p);

/* ---- NCCL bootstrap ------------------------------------------------------
 * Rank 0 creates the id; the caller distributes the bytes (e.g. through the
 * torch.distributed store) and passes them to hexexec_ctx_create. */
size_t hexexec_unique_id_size(void);
hexexec_status hexexec_unique_id(void* out, size_t out_len, char* err, size_t err_len);

/* ---- executor -------------------------------------------------------------
 * exec_config_json: strict keys (unknown key -> HEXEXEC_ERR_PARSE, like the
 * reference's scheduler config, json_io.cpp:263); defaults in brackets:
 *   seed [0], lr [1e-3], beta1 [0.9], beta2 [0.95], eps [1e-8],
 *   weight_decay [0.1]              AdamW hyper-parameters
 *   sm_cap ["green"|"cta"|"none"]   SM cap of a rank with sm_fraction < 1
 *   dp_comm_dtype ["bf16"|"fp32"]   dtype of the weighted DP allreduce
 *   validate_only [false]           host-only layout + memory sizing
 *   cuda_graph [true]               replay the captured step graph after step 0
 *   attention ["fused"|"unfused"]   tcgen05 flash attention / GEMM + softmax
 *   dp_overlap [true]               DP sync + AdamW per layer on a second stream
 *   recompute [false]               activation recompute
 *   pp_protocol ["direct"|"leader"] PP hand-off
 *   pp_dtype ["bf16"|"fp32"]        PP payload (bf16 = comm_pp_hop's 2 bytes)
 *   tp_reduce ["peer"|"nccl"]       TP partial sums over NVLink peer memory / NCCL
 *   tp_direction ["auto"|"push"]    critical TP rank does not push (auto)
 *   tp_pull ["ce"|"sm"]             copy engine / SM copy for the pull
 *   fuse_swiglu [true]              SwiGLU in the gate-up GEMM epilogue
 *   fuse_rope [true]                RoPE in the QKV epilogue / dq cast
 *   gemm_split [false]              tail-wave split-K (not bitwise reproducible)
 *   wgrad_group [1]                 weight-gradient GEMMs over G micro-batches
 *   pdl [false]                     programmatic dependent launch of the GEMMs
 *   profile_gemm [false]            eager steps with per-GEMM / per-op events
 *   graph_gemm_events [false]       per-GEMM events captured in the step graph
 * world_rank indexes the cluster devices in document order unless devices
 * carry the extension key "rank".  nccl_uid may be NULL when world_size == 1. */
hexexec_status hexexec_ctx_create(const char* cluster_json, const char* model_json,
                                  const char* plan_json, const char* exec_config_json,
                                  int world_rank, int world_size, int cuda_device,
                                  const void* nccl_uid, size_t uid_len, hexexec_ctx** out,
                                  char* err, size_t err_len);
void hexexec_ctx_free(hexexec_ctx* ctx);

/* One training step (fwd + bwd + DP gradient sync + AdamW).
 * tokens_host: this rank's pipeline samples, [batch_i][seq_len + 1] int32
 *   (inputs = [:, :S], targets = [:, 1:]); copied host->device inside the
 *   call.  NULL = synthetic tokens generated on the device from the seed
 *   (the device-resident measurement path).
 * loss_out (optional): global sample-weighted mean loss, read device->host. */
hexexec_status hexexec_step(hexexec_ctx* ctx, const int32_t* tokens_host, size_t n_tokens,
                            float* loss_out, char* err, size_t err_len);
/* Same step without any host<->device traffic (loss stays on the device);
 * returns after the work is enqueued.  hexexec_sync waits for it. */
hexexec_status hexexec_step_async(hexexec_ctx* ctx, char* err, size_t err_len);
hexexec_status hexexec_sync(hexexec_ctx* ctx, char* err, size_t err_len);
hexexec_status hexexec_last_loss(hexexec_ctx* ctx, float* loss_out, char* err, size_t err_len);
/* Profiling mode (on = 1): steps run eagerly (no graph replay) with a CUDA
 * event around every GEMM and after every operation; hexexec_stats_json then
 * reports per-GEMM-class TFLOP/s and a per-kernel-class step timeline. */
hexexec_status hexexec_set_profile(hexexec_ctx* ctx, int on);
/* Device timer on the executor's stream: stop = 0 records the start mark;
 * stop = 1 records the end mark, waits for it and returns the elapsed ms. */
hexexec_status hexexec_timer(hexexec_ctx* ctx, int stop, float* ms_out, char* err,
                             size_t err_len);

/* Synthetic tokens of this rank's pipeline for `step` (host copy of the
 * device generator; the oracle uses the same counter-based RNG). */
hexexec_status hexexec_synth_tokens(const hexexec_ctx* ctx, int64_t step, int32_t* out,
                                    size_t n, char* err, size_t err_len);

/* Tensor names: "embed", "final_norm", "lm_head", "layers.<l>.attn_norm",
 * "layers.<l>.wqkv", "layers.<l>.wo", "layers.<l>.mlp_norm", "layers.<l>.wgu",
 * "layers.<l>.wdown".  Each rank holds rows [row0, row0 + rows) of the global
 * [global_rows, cols] tensor (rows = 0 when the rank does not hold it). */
hexexec_status hexexec_tensor_info(const hexexec_ctx* ctx, const char* name, int64_t* row0,
                                   int64_t* rows, int64_t* cols, int64_t* global_rows);
/* which = 0: fp32 master weights; 1: the DP-reduced gradient fed to AdamW
 * (fp32 view); 2: AdamW m; 3: AdamW v.  n must equal rows * cols. */
hexexec_status hexexec_read_tensor(hexexec_ctx* ctx, const char* name, int which, float* out,
                                   size_t n, char* err, size_t err_len);
/* Per-phase device timings of the last step, kernel-launch counts, memory,
 * SM cap actually applied, communicator sets: JSON, caller frees. */
char* hexexec_stats_json(const hexexec_ctx* ctx);

/* SM placement of this rank's work (evidence for the SM cap of emulated
 * tiers): what = 0 launches n probe CTAs on the executor
 * stream, 1 on its second (DP / comm) stream, 2 runs one persistent GEMM of
 * a fixed 4096 x 4096 x 1024 shape on the executor stream; every CTA writes
 * its %smid into sm_ids (n entries; *written = entries filled).  With an
 * SM-capped rank (green context) every id lies in the rank's partition. */
hexexec_status hexexec_sm_probe(hexexec_ctx* ctx, int what, int* sm_ids, int n, int* written,
                                char* err, size_t err_len);

/* ---- kernel-level entry points (device pointers; used by parity tests) --
 * C[z][m,n] = alpha * sum_k A[z][m,k] * B[z][n,k] (+ C if beta); see
 * csrc/gemm.h.  a_mn/b_mn select MN-major storage; c_fp32 selects fp32 C. */
hexexec_status hexexec_k_gemm(int M, int N, int K, int nb1, int nb2, const void* A, int a_mn,
                              int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* B, int b_mn,
                              int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* C, int64_t ldc,
                              int64_t c_bs1, int64_t c_bs2, int c_fp32, int beta, float alpha,
                              int causal, void* stream);
/* tail split-K of later hexexec_k_gemm calls: split -1 auto, 0 off, >1 force
 * that many k-parts; ws (fp32, ws_bytes) and counters (n ints) must be zeroed
 * device memory, or NULL (then only beta GEMMs without workspace split). */
hexexec_status hexexec_k_gemm_split(int split, float* ws, size_t ws_bytes, int* counters, int n);
/* peer copies for later hexexec_k_gemm calls: every bf16 C tile is also
 * TMA-stored to peers[k] (device pointers with C's layout, e.g. another GPU's
 * buffer reachable over NVLink); n = 0 clears.  At most 3. */
hexexec_status hexexec_k_gemm_peers(void* const* peers, int n);
/* tile raster of every later GEMM (process-wide): bands of group_m M-tiles
 * walked M-fastest (default 8); 0 = N-fastest (tuning / microbenchmarks) */
hexexec_status hexexec_k_gemm_raster(int group_m);
/* SMs the persistent GEMM grid of later launches may occupy (0 = all) */
hexexec_status hexexec_k_gemm_sm_limit(int sms);
/* A-tile multicast of later GEMMs: 2 = clusters of two CTA pairs along N
 * sharing the A tile through TMA multicast, 1 = pairs only (default) */
hexexec_status hexexec_k_gemm_multicast(int mc);
/* 1: choose 128-wide output tiles where they quantise into fewer
 * wave-equivalents than 256-wide ones; 0 (default): 256-wide whenever N >= 256 */
hexexec_status hexexec_k_gemm_tile_auto(int on);
/* fused causal attention over the head-interleaved QKV buffer [mb*S, nh*3*d]:
 * out [mb*S, nh*d] bf16, lse [mb*nh, S] (log2 domain); backward writes
 * dq/dk/dv into dqkv [mb*S, nh*3*d] (delta / dq_acc: fp32 scratch of
 * mb*nh*S and mb*S*nh*d floats). */
/* kernel variants of later attention calls (process-wide; 0 = unchanged):
 * fwd 3 = two query tiles per CTA with P kept in TMEM (default), 2 = the
 * same with P through shared memory, 1 = one tile per CTA; bwd 3 = P^T kept in
 * TMEM + separate dQ epilogue warpgroup (default), 2 = dQ epilogue warpgroup
 * with P^T through shared memory, 1 = softmax warps stream dQ (r01) */
hexexec_status hexexec_k_attn_variant(int fwd, int bwd);
hexexec_status hexexec_k_attn_fwd(const void* qkv, void* out, float* lse, int S, int nh, int d,
                                  int mb, float scale, void* stream);
hexexec_status hexexec_k_attn_bwd(const void* qkv, const void* out, const void* dout,
                                  const float* lse, float* delta, float* dq_acc, void* dqkv, int S,
                                  int nh, int d, int mb, float scale, void* stream);
hexexec_status hexexec_k_rmsnorm_fwd(const float* x, const void* y_bf16, float* xo,
                                     const float* g, void* out_bf16, float* rstd, int M, int H,
                                     float eps, void* stream);
hexexec_status hexexec_k_rmsnorm_bwd(const void* dy_bf16, const float* dy_f32, const float* x,
                                     const float* rstd, const float* g, const float* dres,
                                     float* dx, void* dx_bf16, float* dg, int M, int H,
                                     void* stream);
hexexec_status hexexec_k_rope(void* qkv_bf16, int M, int S, int nh, int d, float theta,
                              int inverse, void* stream);
hexexec_status hexexec_k_softmax_fwd(const float* S, void* P_bf16, int L, int nb, void* stream);
hexexec_status hexexec_k_softmax_bwd(const void* P_bf16, const float* dP, void* dS_bf16,
                                     float scale, int L, int nb, void* stream);
hexexec_status hexexec_k_swiglu_fwd(const void* gu, void* a, int M, int F, void* stream);
hexexec_status hexexec_k_swiglu_bwd(const void* gu, const void* da, void* dgu, int M, int F,
                                    void* stream);
hexexec_status hexexec_k_ce(const float* logits, int Vr, int v0, const int32_t* tok, int M,
                            int S, float inv_count, void* dlogits_bf16, float* loss_acc,
                            float* scratch /* 5*M floats */, void* stream);
hexexec_status hexexec_k_adamw(float* p, void* p_bf16, float* m, float* v, const void* g_bf16,
                               const float* g_f32, int64_t n, float gscale, float lr, float b1,
                               float b2, float eps, float wd, int step, void* stream);
hexexec_status hexexec_k_init_normal(float* out, int64_t n, int64_t offset, uint64_t seed,
                                     void* stream);
hexexec_status hexexec_k_tokens(int32_t* out, int64_t n_samples, int S, int64_t sample0,
                                uint64_t seed, int64_t step, int vocab, void* stream);
hexexec_status hexexec_k_sync(char* err, size_t err_len);

const char* hexexec_version(void);
void hexexec_string_free(char* s);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* HEXEXEC_H */
