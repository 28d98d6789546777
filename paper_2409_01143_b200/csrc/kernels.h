// Memory-bound kernels of the training step (sm_100a): init, tokens,
// embedding, RMSNorm, RoPE, causal softmax, SwiGLU, vocab-parallel cross
// entropy, DP gradient scale+cast, AdamW.  RMSNorm runs row bands per CTA
// (the backward through a bulk-copy shared-memory ring); the other row-wise
// ops use a warp or CTA per row; all with 16-byte vector accesses.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hexexec {

using bf16 = __nv_bfloat16;

// ---- counter-based RNG shared with the oracle (oracle/numeric.py) -------
// splitmix64 / mix_seed follow the reference's util.hpp:9-23 exactly.
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b = 0,
                                             uint64_t c = 0) {
  uint64_t h = splitmix64(seed ^ 0x8e12fca87b5d03e1ULL);
  h = splitmix64(h ^ a);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ c);
  return h;
}
// Irwin-Hall(4) normal approximation with std 0.02, bit-reproducible on host
// and device: (sum of four 16-bit lanes - 131070) * 0x1.1bc77ap-21f
__host__ __device__ inline float init_normal(uint64_t tensor_seed, uint64_t idx) {
  uint64_t h = splitmix64(tensor_seed + idx);
  int32_t s = int32_t(h & 0xffff) + int32_t((h >> 16) & 0xffff) + int32_t((h >> 32) & 0xffff) +
              int32_t((h >> 48) & 0xffff) - 131070;
  return float(s) * 0x1.1bc77ap-21f;
}
constexpr uint64_t kTokenTag = 0x746f6b656e73ULL;  // "tokens"

// per-step scalars kept on the device so a captured CUDA graph replays the step
// unchanged: step_tick (first node) advances next_step and derives the AdamW
// bias corrections; gen_tokens is set by a host memset before each launch.
struct StepParams {
  long long next_step;
  long long cur_step;
  float bc1, bc2;
  int gen_tokens;
  int pad;
};
void k_step_tick(StepParams* sp, float b1, float b2, cudaStream_t s);

void k_init_normal(float* master, bf16* copy, long long n, long long global_offset,
                   uint64_t tensor_seed, cudaStream_t s);
void k_fill(float* p, bf16* copy, long long n, float v, cudaStream_t s);
void k_cast_bf16(const float* in, bf16* out, long long n, cudaStream_t s);
void k_upcast_bf16(const bf16* in, float* out, long long n, cudaStream_t s);
// tokens[i][p], i in [0, n_samples), p in [0, S]: sample id = sample0 + i
// sp != null: step and the gen flag come from the device StepParams
void k_gen_tokens(int32_t* tok, long long n_samples, int S, long long sample0, uint64_t seed,
                  long long step, int vocab, cudaStream_t s, const StepParams* sp = nullptr);

// x[m, :] = E[tok(m), :]  (tok row stride S+1)
void k_embed_fwd(const int32_t* tok, const float* E, float* x, int M, int S, int H,
                 cudaStream_t s);
// dE[tok(m), :] += dx[m, :], deterministic (sorted runs, no atomics); token <
// 65536; scratch of embed_bwd_scratch_bytes(M) (M <= 16384: one-CTA bitonic
// sort of 32-bit keys; larger micro-batches: device radix sort of 64-bit keys)
size_t embed_bwd_scratch_bytes(int M);
void k_embed_bwd(const int32_t* tok, const float* dx, float* dE, int M, int S, int H,
                 void* scratch, cudaStream_t s);

// xo = x (+ y[0] + ... + y[ny-1]);  out = bf16(xo * rstd * g);  rstd[m] saved.
// y slots are ys elements apart (TP partial sums, added in slot order).  xo may
// alias x only if y==null.
void k_rmsnorm_fwd(const float* x, const bf16* y, float* xo, const float* g, bf16* out,
                   float* rstd, int M, int H, float eps, cudaStream_t s, int ny = 1,
                   long long ys = 0);
// xo = x + y[0] + ... + y[ny-1] (no norm)
void k_residual_add(const float* x, const bf16* y, float* xo, long long n, cudaStream_t s,
                    int ny = 1, long long ys = 0);
// dx = dres + rmsnorm_bwd(dy);  dx_bf16 optional copy;  dg += sum_m dy*xhat
// dy is bf16 if dy_bf16 != null else fp32 (dy_f32)
// Safe in place (dx == dres): each element is read then written by the same
// thread.  dg_part: fp32 scratch of kRmsBwdCtas * H (per-CTA partial dg rows,
// summed in a fixed order so dg is bitwise reproducible).
constexpr int kRmsBwdCtas = 148;
void k_rmsnorm_bwd(const bf16* dy_bf16, const float* dy_f32, const float* x, const float* rstd,
                   const float* g, const float* dres, float* dx, bf16* dx_bf16, float* dg, int M,
                   int H, float* dg_part, cudaStream_t s, int ny = 1, long long ys = 0);
// (bf16 dy may be ny TP partial slots, ys elements apart, summed in slot order)

// ---- TP exchange over peer memory ---------------------------------------
// Every TP rank owns a flag array flags[tp] (uint64, in its IPC-shared
// exchange buffer).  tp_sync(op): publish epoch(step, op) to flags[me] of every
// peer (release, system scope), then wait until every peer's flag in the local
// array reached it (acquire).  Kernel boundaries order it after the producing
// GEMM (whose TMA stores already reached the peers) and before the consumer.
struct TpPeers {
  unsigned long long* remote[4];  // remote[k] = &flags_of_rank_k[me] (k != me)
  unsigned long long* local;      // this rank's flags[tp]
  int tp, me;
};
void k_tp_sync(const TpPeers& p, const StepParams* sp, unsigned op, cudaStream_t s);
// n CTAs record their %smid into log[0..n) (SM-cap placement evidence)
void k_smid_probe(int* log, int n, cudaStream_t s);
// dst (local) <- src (peer memory), bytes % 16 == 0; grid of 4 CTAs per SM
void k_peer_copy(void* dst, const void* src, size_t bytes, int sms, cudaStream_t s);

// in-place rotary embedding of q and k inside the fused [M, nh*3*d] buffer
// (rotate-half convention); inverse=1 applies the transpose (backward).
void k_rope(bf16* qkv, int M, int S, int nh, int d, float theta, int inverse, cudaStream_t s);
// (cos, sin) table [S][d/2] of the same angles (for the GEMM's RoPE epilogue)
void k_rope_table(float2* tab, int S, int d, float theta, cudaStream_t s);

// causal softmax over fp32 scores [nb][L][L] (already scaled); P bf16 with
// zeros for j > i up to the end of the row's 128-wide tile.
void k_softmax_fwd(const float* S, bf16* P, int L, int nb, cudaStream_t s);
// dS = scale * P * (dP - sum_j P*dP)
void k_softmax_bwd(const bf16* P, const float* dP, bf16* dS, float scale, int L, int nb,
                   cudaStream_t s);

// gu: [M, 2F] chunk-interleaved (64 gate cols, 64 up cols); a: [M, F]
void k_swiglu_fwd(const bf16* gu, bf16* a, int M, int F, cudaStream_t s);
void k_swiglu_bwd(const bf16* gu, const bf16* da, bf16* dgu, int M, int F, cudaStream_t s);

// vocab-parallel CE.  logits [M, Vr] fp32 for global vocab [v0, v0+Vr).
//  stats: lmax[M] (local max), lsum[M] (sum exp(l - lmax)), st2[2M] = {sum, tlogit}
void k_ce_stats(const float* logits, int Vr, int v0, const int32_t* tok, int M, int S,
                float* lmax, float* lsum, float* st2, cudaStream_t s);
// st2[m].sum = lsum[m] * exp(lmax[m] - gmax[m])
void k_ce_rescale(const float* lmax, const float* lsum, const float* gmax, float* st2, int M,
                  cudaStream_t s);
// dlogits = (softmax - onehot) * inv_count (bf16); loss_acc += sum_m (log(sum)+gmax - tlogit)
// (row losses in row_loss[M], summed in a fixed order: reproducible)
void k_ce_finish(const float* logits, int Vr, int v0, const int32_t* tok, int M, int S,
                 const float* gmax, const float* st2, float inv_count, bf16* dlogits,
                 float* loss_acc, float* row_loss, cudaStream_t s);

// DP gradient prep: out = bf16(scale * g)
void k_scale_cast(const float* g, bf16* out, long long n, float scale, cudaStream_t s);
void k_scale(float* g, long long n, float scale, cudaStream_t s);
// AdamW on an fp32 master shard; grad is bf16 (g16) or fp32 (g32) times gscale
void k_adamw(float* p, bf16* p16, float* m, float* v, const bf16* g16, const float* g32,
             long long n, float gscale, float lr, float b1, float b2, float eps, float wd,
             float bc1, float bc2, cudaStream_t s, const StepParams* sp = nullptr);

}  // namespace hexexec
