// Host-side interface of the sm_100a tcgen05 GEMM used for every dense
// contraction of the step (TP column/row GEMMs fwd + dgrad + wgrad, LM head,
// attention score / context products).
//
//   C[z][m, n] = alpha * sum_k A[z][m, k] * B[z][n, k]   (+ C[z][m, n] if beta)
//
// A is logically [M, K], B logically [N, K].  Each is stored either K-major
// (K contiguous, row stride ld) or MN-major (M resp. N contiguous, stride ld
// between consecutive k).  Batch index z = z1 + nb1 * z2 with element strides
// bs1 / bs2, so per-head attention products address the fused QKV buffer in
// place.  Inputs bf16; accumulation fp32 in TMEM; C bf16 or fp32.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hexexec {

struct GemmOperand {
  const void* ptr = nullptr;
  int mn_major = 0;
  long long ld = 0;   // elements between consecutive rows (K-major) / k (MN-major)
  long long bs1 = 0;  // batch strides in elements
  long long bs2 = 0;
};

enum GemmCausal : int {
  kCausalNone = 0,
  kCausalSkipUpper = 1,  // tiles with n0 > m0 + BM - 1 are not computed (nor written)
  kCausalKLower = 2,     // k range limited to [0, min(K, m0 + BM))   (A lower-triangular)
  kCausalKUpper = 3,     // k range limited to [m0, K)                  (A^T of lower-tri)
};

constexpr int kMaxGemmPeers = 3;

struct GemmDesc {
  int M = 0, N = 0, K = 0;
  int nb1 = 1, nb2 = 1;
  GemmOperand A, B;
  void* C = nullptr;
  long long ldc = 0, cbs1 = 0, cbs2 = 0;
  const float* R = nullptr;  // optional fp32 residual, same layout as C: C = alpha*acc + R
  int c_fp32 = 0;  // 1: fp32 output, 0: bf16 output
  int beta = 0;    // 1: C += alpha*acc (fp32 C only)
  float alpha = 1.f;
  int causal = kCausalNone;
  // Split-K of the last, partial wave of tiles (wave quantisation): the
  // leftover tiles are cut into `s` k-ranges spread over all CTA pairs.
  // beta GEMMs without R reduce-add their partials straight into C; the
  // others reduce-add into the fp32 workspace `ws` and the last arriving
  // partial (per-slab counter in `ws_cnt`) finishes the tile.  ws / ws_cnt
  // must be zero on entry and are left zero.  split: -1 auto, 0 off, >1 force.
  float* ws = nullptr;
  size_t ws_bytes = 0;
  int* ws_cnt = nullptr;
  int ws_cnt_n = 0;
  int split = -1;
  // TP peer copies: every C tile is also TMA-stored to peer_C[k] (same layout,
  // bf16, no beta / split; typically IPC-mapped buffers of the other TP ranks
  // so the row-parallel partials cross NVLink while the GEMM still runs)
  void* peer_C[kMaxGemmPeers] = {nullptr, nullptr, nullptr};
  int npeer = 0;
  // SwiGLU epilogue (gate-up projection): C holds [g | u] in 128-column chunk
  // pairs (64 gate, 64 up); act[m, f] = silu(g) * u (bf16, [M, N/2], row
  // stride ld_act or N/2) is written from the same tile.  bf16 C, no beta /
  // split / peers / batch.
  void* act = nullptr;
  long long ld_act = 0;
  // RoPE epilogue (QKV projection, head-interleaved (h, {q,k,v}, d) columns):
  // q and k of every head rotated (rotate-half) with (cos, sin) from
  // rope[(row % rope_S) * rope_d / 2 + i]; d in {64, 128}; bf16 C only
  const float2* rope = nullptr;
  int rope_d = 0, rope_S = 0;
};

// workspace a GemmDesc needs for any split (bytes, counters)
constexpr size_t kGemmWsBytes = size_t(148) * 128 * 256 * 4;
constexpr int kGemmWsCounters = 148 * 8;

// Launch on `stream`.  Returns cudaSuccess or the launch error.  Tensor maps
// are encoded on the host per call (cheap, ~1 us) from the descriptor.
cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t stream);

// number of SMs the GEMM may occupy (0 = all); used for SM-capped ranks
void gemm_set_sm_limit(int sms);
// tests: every CTA of later launches writes its %smid to log[blockIdx.x]
// (null = off); evidence that a capped rank's GEMMs stay in its partition
void gemm_set_smid_log(int* log);
// 0 = auto (CTA pairs when M > 128), 1 / 2 = force single-SM / paired tiles
void gemm_force_cta_group(int cg);
// grouped tile raster: bands of g M-tiles (default 8); 0 = n fastest
void gemm_set_group_m(int g);
// programmatic dependent launch (griddepcontrol.wait after the prologue): 1 = on
void gemm_set_pdl(int on);
// 2: A-tile TMA multicast across two CTA pairs along N (clusters of 4), 1: off
void gemm_set_multicast(int mc);
// 1: 128-wide tiles where they quantise into fewer wave-equivalents (default 0)
void gemm_set_bn_auto(int on);

}  // namespace hexexec
