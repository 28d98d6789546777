// extern "C" boundary (include/hexexec.h).  Conventions follow the reference
// C ABI proj/src/capi.cpp:34-73: err buffers are always NUL-terminated and
// truncated safely, null arguments -> INVALID, exceptions are translated to
// status codes and never cross the ABI, strings are malloc'd.
#include "hexexec.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "attention.h"
#include "costmodel.hpp"
#include "executor.hpp"
#include "gemm.h"
#include "kernels.h"
#include "plan.hpp"

struct hexexec_plan {
  hexexec::Layout layout;
};
struct hexexec_ctx {
  hexexec::Executor* ex = nullptr;
};

namespace {

void set_err(char* err, size_t err_len, const std::string& msg) {
  if (!err || err_len == 0) return;
  size_t n = msg.size() < err_len - 1 ? msg.size() : err_len - 1;
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

char* dup_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  if (!out) return nullptr;
  std::memcpy(out, s.data(), s.size() + 1);
  return out;
}

template <typename F>
hexexec_status guarded(char* err, size_t err_len, F&& f) {
  try {
    f();
    return HEXEXEC_OK;
  } catch (const hexexec::ParseError& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_PARSE;
  } catch (const hexexec::InvalidArgument& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_INVALID;
  } catch (const hexexec::Infeasible& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_INFEASIBLE;
  } catch (const hexexec::LimitExceeded& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_LIMIT;
  } catch (const hexexec::CudaError& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_CUDA;
  } catch (const hexexec::NcclError& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_NCCL;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return HEXEXEC_ERR_INTERNAL;
  } catch (...) {
    set_err(err, err_len, "unknown error");
    return HEXEXEC_ERR_INTERNAL;
  }
}

hexexec_status cuda_status(cudaError_t e) {
  return e == cudaSuccess ? HEXEXEC_OK : HEXEXEC_ERR_CUDA;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

// ------------------------------------------------------------------ plan
hexexec_status hexexec_plan_parse(const char* cluster_json, const char* model_json,
                                  const char* plan_json, hexexec_plan** out, char* err,
                                  size_t err_len) {
  if (!cluster_json || !model_json || !plan_json || !out) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] {
    auto* p = new hexexec_plan{hexexec::build_layout(cluster_json, model_json, plan_json)};
    *out = p;
  });
}

char* hexexec_plan_serialize(const hexexec_plan* p) {
  if (!p) return nullptr;
  try {
    return dup_string(hexexec::serialize_plan(p->layout.plan, p->layout.cluster));
  } catch (...) {
    return nullptr;
  }
}

char* hexexec_plan_layout_json(const hexexec_plan* p) {
  if (!p) return nullptr;
  try {
    return dup_string(hexexec::layout_json(p->layout));
  } catch (...) {
    return nullptr;
  }
}

int hexexec_plan_world_size(const hexexec_plan* p) { return p ? p->layout.world_size : 0; }

hexexec_status hexexec_plan_cost(const hexexec_plan* p, double state_multiplier, int extension,
                                 char** report_json, char* err, size_t err_len) {
  if (!p || !report_json) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] {
    const hexexec::CostReport r = hexexec::iteration_time(
        p->layout.plan, p->layout.model, p->layout.cluster, state_multiplier, extension != 0);
    char* s = dup_string(hexexec::serialize_report(r, p->layout.cluster));
    if (!s) throw std::bad_alloc();
    *report_json = s;
  });
}

double hexexec_plan_mfu(const hexexec_plan* p, double seconds) {
  if (!p) return 0.0;
  try {
    return hexexec::model_flops_utilization(seconds, p->layout.plan.global_batch, p->layout.model,
                                            p->layout.cluster);
  } catch (...) {
    return 0.0;
  }
}

void hexexec_plan_free(hexexec_plan* p) { delete p; }

// ------------------------------------------------------------------ NCCL id
size_t hexexec_unique_id_size(void) { return sizeof(ncclUniqueId); }

hexexec_status hexexec_unique_id(void* out, size_t out_len, char* err, size_t err_len) {
  if (!out || out_len < sizeof(ncclUniqueId)) {
    set_err(err, err_len, "null argument or buffer too small");
    return HEXEXEC_ERR_INVALID;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    set_err(err, err_len, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    return HEXEXEC_ERR_NCCL;
  }
  std::memcpy(out, &id, sizeof(id));
  return HEXEXEC_OK;
}

// ------------------------------------------------------------------ executor
hexexec_status hexexec_ctx_create(const char* cluster_json, const char* model_json,
                                  const char* plan_json, const char* exec_config_json,
                                  int world_rank, int world_size, int cuda_device,
                                  const void* nccl_uid, size_t uid_len, hexexec_ctx** out,
                                  char* err, size_t err_len) {
  if (!cluster_json || !model_json || !plan_json || !out) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] {
    hexexec::Executor* ex = hexexec::make_executor(
        cluster_json, model_json, plan_json, exec_config_json ? exec_config_json : "",
        world_rank, world_size, cuda_device, nccl_uid, uid_len);
    *out = new hexexec_ctx{ex};
  });
}

void hexexec_ctx_free(hexexec_ctx* ctx) {
  if (!ctx) return;
  try {
    hexexec::destroy_executor(ctx->ex);
  } catch (...) {
  }
  delete ctx;
}

hexexec_status hexexec_step(hexexec_ctx* ctx, const int32_t* tokens_host, size_t n_tokens,
                            float* loss_out, char* err, size_t err_len) {
  if (!ctx || !ctx->ex) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len,
                 [&] { hexexec::executor_step(*ctx->ex, tokens_host, n_tokens, loss_out); });
}

hexexec_status hexexec_step_async(hexexec_ctx* ctx, char* err, size_t err_len) {
  if (!ctx || !ctx->ex) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] { hexexec::executor_step_async(*ctx->ex); });
}

hexexec_status hexexec_sync(hexexec_ctx* ctx, char* err, size_t err_len) {
  if (!ctx || !ctx->ex) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] { hexexec::executor_sync(*ctx->ex); });
}

hexexec_status hexexec_set_profile(hexexec_ctx* ctx, int on) {
  if (!ctx || !ctx->ex) return HEXEXEC_ERR_INVALID;
  return guarded(nullptr, 0, [&] { hexexec::executor_set_profile(*ctx->ex, on != 0); });
}

hexexec_status hexexec_timer(hexexec_ctx* ctx, int stop, float* ms_out, char* err,
                             size_t err_len) {
  if (!ctx || !ctx->ex || (stop && !ms_out)) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] { hexexec::executor_timer(*ctx->ex, stop, ms_out); });
}

hexexec_status hexexec_last_loss(hexexec_ctx* ctx, float* loss_out, char* err, size_t err_len) {
  if (!ctx || !ctx->ex || !loss_out) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] { *loss_out = hexexec::executor_last_loss(*ctx->ex); });
}

hexexec_status hexexec_synth_tokens(const hexexec_ctx* ctx, int64_t step, int32_t* out, size_t n,
                                    char* err, size_t err_len) {
  if (!ctx || !ctx->ex || !out) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len, [&] { hexexec::executor_synth_tokens(*ctx->ex, step, out, n); });
}

hexexec_status hexexec_tensor_info(const hexexec_ctx* ctx, const char* name, int64_t* row0,
                                   int64_t* rows, int64_t* cols, int64_t* global_rows) {
  if (!ctx || !ctx->ex || !name || !row0 || !rows || !cols || !global_rows)
    return HEXEXEC_ERR_INVALID;
  try {
    return hexexec::executor_tensor_info(*ctx->ex, name, row0, rows, cols, global_rows)
               ? HEXEXEC_OK
               : HEXEXEC_ERR_INVALID;
  } catch (...) {
    return HEXEXEC_ERR_INTERNAL;
  }
}

hexexec_status hexexec_read_tensor(hexexec_ctx* ctx, const char* name, int which, float* out,
                                   size_t n, char* err, size_t err_len) {
  if (!ctx || !ctx->ex || !name || !out) {
    set_err(err, err_len, "null argument");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len,
                 [&] { hexexec::executor_read_tensor(*ctx->ex, name, which, out, n); });
}

hexexec_status hexexec_sm_probe(hexexec_ctx* ctx, int what, int* sm_ids, int n, int* written,
                                char* err, size_t err_len) {
  if (!ctx || !ctx->ex || !sm_ids || !written || what < 0 || what > 2) {
    set_err(err, err_len, "null argument or bad probe kind");
    return HEXEXEC_ERR_INVALID;
  }
  return guarded(err, err_len,
                 [&] { *written = hexexec::executor_sm_probe(*ctx->ex, what, sm_ids, n); });
}

char* hexexec_stats_json(const hexexec_ctx* ctx) {
  if (!ctx || !ctx->ex) return nullptr;
  try {
    return dup_string(hexexec::executor_stats_json(*ctx->ex));
  } catch (...) {
    return nullptr;
  }
}

// ------------------------------------------------------------------ kernels
namespace {
struct KSplit {
  int split;
  float* ws;
  size_t ws_bytes;
  int* cnt;
  int n;
};
KSplit g_k_split = {-1, nullptr, 0, nullptr, 0};
// peer copies of C for later hexexec_k_gemm calls (test / microbenchmark)
struct KPeers {
  void* p[hexexec::kMaxGemmPeers] = {nullptr, nullptr, nullptr};
  int n = 0;
} g_k_peers;
}  // namespace

hexexec_status hexexec_k_gemm(int M, int N, int K, int nb1, int nb2, const void* A, int a_mn,
                              int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* B, int b_mn,
                              int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* C, int64_t ldc,
                              int64_t c_bs1, int64_t c_bs2, int c_fp32, int beta, float alpha,
                              int causal, void* stream) {
  hexexec::GemmDesc d;
  d.M = M;
  d.N = N;
  d.K = K;
  d.nb1 = nb1;
  d.nb2 = nb2;
  d.A = {A, a_mn, lda, a_bs1, a_bs2};
  d.B = {B, b_mn, ldb, b_bs1, b_bs2};
  d.C = C;
  d.ldc = ldc;
  d.cbs1 = c_bs1;
  d.cbs2 = c_bs2;
  d.c_fp32 = c_fp32;
  d.beta = beta;
  d.alpha = alpha;
  d.causal = causal;
  d.split = g_k_split.split;
  d.ws = g_k_split.ws;
  d.ws_bytes = g_k_split.ws_bytes;
  d.ws_cnt = g_k_split.cnt;
  d.ws_cnt_n = g_k_split.n;
  d.npeer = g_k_peers.n;
  for (int k = 0; k < g_k_peers.n; ++k) d.peer_C[k] = g_k_peers.p[k];
  return cuda_status(hexexec::gemm_bf16(d, as_stream(stream)));
}

hexexec_status hexexec_k_gemm_tile_auto(int on) {
  hexexec::gemm_set_bn_auto(on);
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_gemm_multicast(int mc) {
  if (mc != 1 && mc != 2) return HEXEXEC_ERR_INVALID;
  hexexec::gemm_set_multicast(mc);
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_gemm_sm_limit(int sms) {
  if (sms < 0) return HEXEXEC_ERR_INVALID;
  hexexec::gemm_set_sm_limit(sms);
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_gemm_raster(int group_m) {
  if (group_m < 0) return HEXEXEC_ERR_INVALID;
  hexexec::gemm_set_group_m(group_m);
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_gemm_peers(void* const* peers, int n) {
  if (n < 0 || n > hexexec::kMaxGemmPeers || (n > 0 && !peers)) return HEXEXEC_ERR_INVALID;
  g_k_peers.n = n;
  for (int k = 0; k < n; ++k) g_k_peers.p[k] = peers[k];
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_gemm_split(int split, float* ws, size_t ws_bytes, int* counters, int n) {
  g_k_split = {split, ws, ws_bytes, counters, n};
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_attn_variant(int fwd, int bwd) {
  if (fwd) hexexec::attention_fwd_variant(fwd);
  if (bwd) hexexec::attention_bwd_variant(bwd);
  return HEXEXEC_OK;
}

hexexec_status hexexec_k_attn_fwd(const void* qkv, void* out, float* lse, int S, int nh, int d,
                                  int mb, float scale, void* stream) {
  hexexec::AttnDesc a;
  a.qkv = static_cast<const __nv_bfloat16*>(qkv);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.lse = lse;
  a.S = S;
  a.nh = nh;
  a.d = d;
  a.mb = mb;
  a.scale = scale;
  return cuda_status(hexexec::attention_fwd(a, as_stream(stream)));
}

hexexec_status hexexec_k_attn_bwd(const void* qkv, const void* out, const void* dout,
                                  const float* lse, float* delta, float* dq_acc, void* dqkv, int S,
                                  int nh, int d, int mb, float scale, void* stream) {
  hexexec::AttnBwdDesc a;
  a.qkv = static_cast<const __nv_bfloat16*>(qkv);
  a.out = static_cast<const __nv_bfloat16*>(out);
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.lse = lse;
  a.delta = delta;
  a.dq_acc = dq_acc;
  a.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  a.S = S;
  a.nh = nh;
  a.d = d;
  a.mb = mb;
  a.scale = scale;
  return cuda_status(hexexec::attention_bwd(a, as_stream(stream)));
}

hexexec_status hexexec_k_rmsnorm_fwd(const float* x, const void* y, float* xo, const float* g,
                                     void* out, float* rstd, int M, int H, float eps,
                                     void* stream) {
  hexexec::k_rmsnorm_fwd(x, static_cast<const hexexec::bf16*>(y), xo, g,
                         static_cast<hexexec::bf16*>(out), rstd, M, H, eps, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_rmsnorm_bwd(const void* dyb, const float* dyf, const float* x,
                                     const float* rstd, const float* g, const float* dres,
                                     float* dx, void* dxb, float* dg, int M, int H,
                                     void* stream) {
  // partial-dg scratch kept across calls, one per device and host thread
  // (grown on demand; kernel test entry only -- the executor passes its own).
  // Calls from one thread on one device are stream-ordered by the caller.
  struct Scratch {
    float* part = nullptr;
    size_t cap = 0;
  };
  static thread_local std::map<int, Scratch> scratch;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HEXEXEC_ERR_CUDA;
  Scratch& sc = scratch[dev];
  const size_t need = size_t(hexexec::kRmsBwdCtas) * size_t(H > 0 ? H : 1) * sizeof(float);
  if (need > sc.cap) {
    if (sc.part) {
      cudaStreamSynchronize(as_stream(stream));  // the old scratch may still be read
      cudaFree(sc.part);
    }
    sc.part = nullptr;
    sc.cap = 0;
    if (cudaMalloc(&sc.part, need) != cudaSuccess) return HEXEXEC_ERR_CUDA;
    sc.cap = need;
  }
  float* part = sc.part;
  hexexec::k_rmsnorm_bwd(static_cast<const hexexec::bf16*>(dyb), dyf, x, rstd, g, dres, dx,
                         static_cast<hexexec::bf16*>(dxb), dg, M, H, part, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_rope(void* qkv, int M, int S, int nh, int d, float theta, int inverse,
                              void* stream) {
  hexexec::k_rope(static_cast<hexexec::bf16*>(qkv), M, S, nh, d, theta, inverse,
                  as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_softmax_fwd(const float* S, void* P, int L, int nb, void* stream) {
  hexexec::k_softmax_fwd(S, static_cast<hexexec::bf16*>(P), L, nb, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_softmax_bwd(const void* P, const float* dP, void* dS, float scale, int L,
                                     int nb, void* stream) {
  hexexec::k_softmax_bwd(static_cast<const hexexec::bf16*>(P), dP,
                         static_cast<hexexec::bf16*>(dS), scale, L, nb, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_swiglu_fwd(const void* gu, void* a, int M, int F, void* stream) {
  hexexec::k_swiglu_fwd(static_cast<const hexexec::bf16*>(gu), static_cast<hexexec::bf16*>(a), M,
                        F, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_swiglu_bwd(const void* gu, const void* da, void* dgu, int M, int F,
                                    void* stream) {
  hexexec::k_swiglu_bwd(static_cast<const hexexec::bf16*>(gu),
                        static_cast<const hexexec::bf16*>(da), static_cast<hexexec::bf16*>(dgu),
                        M, F, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_ce(const float* logits, int Vr, int v0, const int32_t* tok, int M, int S,
                            float inv_count, void* dlogits, float* loss_acc, float* scratch,
                            void* stream) {
  cudaStream_t s = as_stream(stream);
  float* lmax = scratch;
  float* lsum = scratch + M;
  float* st2 = scratch + 2 * M;
  hexexec::k_ce_stats(logits, Vr, v0, tok, M, S, lmax, lsum, st2, s);
  hexexec::k_ce_finish(logits, Vr, v0, tok, M, S, lmax, st2, inv_count,
                       static_cast<hexexec::bf16*>(dlogits), loss_acc, scratch + 4 * M, s);
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_adamw(float* p, void* p16, float* m, float* v, const void* g16,
                               const float* g32, int64_t n, float gscale, float lr, float b1,
                               float b2, float eps, float wd, int step, void* stream) {
  float bc1 = 1.f - std::pow(b1, float(step));
  float bc2 = 1.f - std::pow(b2, float(step));
  hexexec::k_adamw(p, static_cast<hexexec::bf16*>(p16), m, v,
                   static_cast<const hexexec::bf16*>(g16), g32, n, gscale, lr, b1, b2, eps, wd,
                   bc1, bc2, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_init_normal(float* out, int64_t n, int64_t offset, uint64_t seed,
                                     void* stream) {
  hexexec::k_init_normal(out, nullptr, n, offset, seed, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_tokens(int32_t* out, int64_t n_samples, int S, int64_t sample0,
                                uint64_t seed, int64_t step, int vocab, void* stream) {
  hexexec::k_gen_tokens(out, n_samples, S, sample0, seed, step, vocab, as_stream(stream));
  return cuda_status(cudaGetLastError());
}

hexexec_status hexexec_k_sync(char* err, size_t err_len) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_err(err, err_len, cudaGetErrorString(e));
    return HEXEXEC_ERR_CUDA;
  }
  return HEXEXEC_OK;
}

const char* hexexec_version(void) { return "hexexec 0.1.0 (sm_100a)"; }

void hexexec_string_free(char* s) { std::free(s); }

}  // extern "C"
