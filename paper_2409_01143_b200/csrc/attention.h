// Fused causal attention for sm_100a (tcgen05 + TMEM + TMA), reading Q/K/V in
// place from the fused head-interleaved QKV buffer [M = mb*S, nh*3*d]
// (head h: q at column h*3d, k at h*3d+d, v at h*3d+2d) and writing the
// attention output [M, nh*d] (head-major columns).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace hexexec {

struct AttnDesc {
  const __nv_bfloat16* qkv = nullptr;
  __nv_bfloat16* out = nullptr;   // [M, nh*d]
  float* lse = nullptr;           // [mb*nh, S], log2-domain row log-sum-exp of scaled scores
  int S = 0, nh = 0, d = 0, mb = 0;
  float scale = 1.f;              // softmax scale (1/sqrt(d))
};

// forward: out = softmax(scale * q k^T, causal) v ; lse saved for the backward
cudaError_t attention_fwd(const AttnDesc& a, cudaStream_t s);
// 2 (default): two query tiles per CTA with ping-pong softmax warpgroups; 1: one tile
// forward: 3 = P in TMEM (default), 2 = P through shared memory, 1 = one tile / CTA
void attention_fwd_variant(int v);
// backward: 3 = P^T in TMEM + dQ epilogue warpgroup (default), 2 = dQ epilogue
// warpgroup, 1 = the r01 kernel
void attention_bwd_variant(int v);

struct AttnBwdDesc {
  const __nv_bfloat16* qkv = nullptr;
  const __nv_bfloat16* out = nullptr;   // forward output O
  const __nv_bfloat16* dout = nullptr;  // dO [M, nh*d]
  const float* lse = nullptr;
  float* delta = nullptr;               // [mb*nh, S] scratch: rowsum(dO * O)
  float* dq_acc = nullptr;              // [M, nh*d] fp32 scratch (zeroed by the delta pass)
  __nv_bfloat16* dqkv = nullptr;        // [M, nh*3*d]: dq, dk, dv written in place
  int S = 0, nh = 0, d = 0, mb = 0;
  float scale = 1.f;
  // optional RoPE backward fused into the dq cast: (cos, sin) table [S][d/2]
  // of the forward rotation; dq and dk of dqkv come out un-rotated
  const float2* rope = nullptr;
};

// backward: dq, dk, dv of the forward above
cudaError_t attention_bwd(const AttnBwdDesc& a, cudaStream_t s);

}  // namespace hexexec
