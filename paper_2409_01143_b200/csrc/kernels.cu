// Memory-bound kernels of the step (see kernels.h).  All row-wise kernels use
// one warp per row, 16-byte vector accesses where the row width allows, and
// warp-shuffle reductions; elementwise kernels are grid-stride with the grid
// sized to a multiple of the SM count.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hexexec {

namespace {

constexpr int kNumSmsHint = 148;

inline int ew_grid(long long n, int per_thread) {
  long long blocks = (n + 256LL * per_thread - 1) / (256LL * per_thread);
  long long cap = kNumSmsHint * 16LL;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return int(blocks);
}

inline int row_grid(int rows, int warps_per_block) {
  return (rows + warps_per_block - 1) / warps_per_block;
}

__device__ __forceinline__ float bf(bf16 x) { return __bfloat162float(x); }

// ------------------------------------------------------------------ init
__global__ void init_normal_kernel(float* p, bf16* c, long long n, long long off, uint64_t seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float v = init_normal(seed, uint64_t(off + i));
    p[i] = v;
    if (c) c[i] = __float2bfloat16_rn(v);
  }
}

__global__ void fill_kernel(float* p, bf16* c, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    p[i] = v;
    if (c) c[i] = __float2bfloat16_rn(v);
  }
}

__global__ void cast_kernel(const float* in, bf16* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

__global__ void tokens_kernel(int32_t* tok, long long ns, int S1, long long sample0,
                              uint64_t seed, long long step, int vocab, const StepParams* sp) {
  if (sp) {
    if (!sp->gen_tokens) return;
    step = sp->cur_step;
  }
  long long n = ns * S1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long smp = i / S1;
    int pos = int(i % S1);
    uint64_t base = mix_seed(seed, kTokenTag, uint64_t(step), uint64_t(sample0 + smp));
    tok[i] = int32_t(splitmix64(base + uint64_t(pos)) % uint64_t(vocab));
  }
}

// ------------------------------------------------------------------ embedding
__global__ void embed_fwd_kernel(const int32_t* tok, const float* E, float* x, int M, int S,
                                 int H) {
  int row = blockIdx.x;
  if (row >= M) return;
  int t = tok[(row / S) * (S + 1) + row % S];
  const float4* src = reinterpret_cast<const float4*>(E + (long long)t * H);
  float4* dst = reinterpret_cast<float4*>(x + (long long)row * H);
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) dst[i] = src[i];
}

__global__ void embed_bwd_kernel(const int32_t* tok, const float* dx, float* dE, int M, int S,
                                 int H) {
  int row = blockIdx.x;
  if (row >= M) return;
  int t = tok[(row / S) * (S + 1) + row % S];
  float* dst = dE + (long long)t * H;
  const float* src = dx + (long long)row * H;
  for (int i = threadIdx.x; i < H; i += blockDim.x) atomicAdd(dst + i, src[i]);
}

// ------------------------------------------------------------------ rmsnorm
// one warp per row; H % 8 == 0
__global__ void rmsnorm_fwd_kernel(const float* __restrict__ x, const bf16* __restrict__ y,
                                   float* xo, const float* __restrict__ g, bf16* __restrict__ out,
                                   float* __restrict__ rstd, int M, int H, float eps) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= M) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (long long)row * H);
  float4* xor_ = reinterpret_cast<float4*>(xo + (long long)row * H);
  const uint2* yr = y ? reinterpret_cast<const uint2*>(y + (long long)row * H) : nullptr;
  float ss = 0.f;
  for (int i = lane; i < H / 4; i += 32) {
    float4 v = xr[i];
    if (yr) {
      uint2 w = yr[i];
      __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&w.x);
      __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w.y);
      v.x += __low2float(a);
      v.y += __high2float(a);
      v.z += __low2float(b);
      v.w += __high2float(b);
      xor_[i] = v;
    }
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  float r = rsqrtf(ss / float(H) + eps);
  if (lane == 0) rstd[row] = r;
  const float4* src = yr ? reinterpret_cast<const float4*>(xo + (long long)row * H) : xr;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint2* o = reinterpret_cast<uint2*>(out + (long long)row * H);
  for (int i = lane; i < H / 4; i += 32) {
    float4 v = src[i];
    float4 gg = g4[i];
    uint2 w;
    w.x = pack_bf16x2(v.x * r * gg.x, v.y * r * gg.y);
    w.y = pack_bf16x2(v.z * r * gg.z, v.w * r * gg.w);
    o[i] = w;
  }
}

__global__ void residual_add_kernel(const float* x, const bf16* y, float* xo, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    xo[i] = x[i] + bf(y[i]);
}

// RMSNorm backward, two passes:
//   (1) warp per row: c[m] = r^3/H * sum_j dy*g*x
//   (2) column tiles (coalesced float4 columns x 64-row bands):
//       dx = dres + r*dy*g - x*c ;  dg[j] += sum_rows dy*x*r  (register
//       accumulation over the band, one atomic per column per band)
template <bool kDyBf16>
__device__ __forceinline__ float4 load_dy(const bf16* dyb, const float* dyf, long long off) {
  if (kDyBf16) {
    uint2 w = *reinterpret_cast<const uint2*>(dyb + off);
    __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&w.x);
    __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w.y);
    return make_float4(__low2float(a), __high2float(a), __low2float(b), __high2float(b));
  }
  return *reinterpret_cast<const float4*>(dyf + off);
}

template <bool kDyBf16>
__global__ void rmsnorm_bwd_dot_kernel(const bf16* __restrict__ dyb, const float* __restrict__ dyf,
                                       const float* __restrict__ x, const float* __restrict__ rstd,
                                       const float* __restrict__ g, float* __restrict__ coef,
                                       int M, int H) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= M) return;
  const long long base = (long long)row * H;
  float dot = 0.f;
  for (int i = lane * 4; i < H; i += 128) {
    float4 xv = *reinterpret_cast<const float4*>(x + base + i);
    float4 gv = *reinterpret_cast<const float4*>(g + i);
    float4 d = load_dy<kDyBf16>(dyb, dyf, base + i);
    dot += d.x * gv.x * xv.x + d.y * gv.y * xv.y + d.z * gv.z * xv.z + d.w * gv.w * xv.w;
  }
  dot = warp_sum(dot);
  if (lane == 0) {
    const float r = rstd[row];
    coef[row] = dot * r * r * r / float(H);
  }
}

template <bool kDyBf16>
__global__ void rmsnorm_bwd_dx_kernel(const bf16* __restrict__ dyb, const float* __restrict__ dyf,
                                      const float* __restrict__ x, const float* __restrict__ rstd,
                                      const float* __restrict__ coef,
                                      const float* __restrict__ g, const float* __restrict__ dres,
                                      float* __restrict__ dx, bf16* __restrict__ dxb,
                                      float* __restrict__ dg, int M, int H, int band) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (col >= H) return;
  const int r0 = blockIdx.y * band;
  const int r1 = min(M, r0 + band);
  const float4 gv = *reinterpret_cast<const float4*>(g + col);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int row = r0; row < r1; ++row) {
    const long long off = (long long)row * H + col;
    const float r = rstd[row];
    const float c = coef[row];
    float4 xv = *reinterpret_cast<const float4*>(x + off);
    float4 d = load_dy<kDyBf16>(dyb, dyf, off);
    acc.x += d.x * xv.x * r;
    acc.y += d.y * xv.y * r;
    acc.z += d.z * xv.z * r;
    acc.w += d.w * xv.w * r;
    float4 o;
    o.x = r * d.x * gv.x - xv.x * c;
    o.y = r * d.y * gv.y - xv.y * c;
    o.z = r * d.z * gv.z - xv.z * c;
    o.w = r * d.w * gv.w - xv.w * c;
    if (dres) {
      float4 rv = *reinterpret_cast<const float4*>(dres + off);
      o.x += rv.x; o.y += rv.y; o.z += rv.z; o.w += rv.w;
    }
    *reinterpret_cast<float4*>(dx + off) = o;
    if (dxb) {
      uint2 w;
      w.x = pack_bf16x2(o.x, o.y);
      w.y = pack_bf16x2(o.z, o.w);
      *reinterpret_cast<uint2*>(dxb + off) = w;
    }
  }
  atomicAdd(dg + col + 0, acc.x);
  atomicAdd(dg + col + 1, acc.y);
  atomicAdd(dg + col + 2, acc.z);
  atomicAdd(dg + col + 3, acc.w);
}

// ------------------------------------------------------------------ rope
// thread per (row, head, i < d/2) pair, applied to q and k
__device__ __forceinline__ void unpack8(uint4 w, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __low2float(h[k]);
    f[2 * k + 1] = __high2float(h[k]);
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 w;
  w.x = pack_bf16x2(f[0], f[1]);
  w.y = pack_bf16x2(f[2], f[3]);
  w.z = pack_bf16x2(f[4], f[5]);
  w.w = pack_bf16x2(f[6], f[7]);
  return w;
}

// thread per (row, head, q|k, 8 rotation pairs): 16-byte loads of both halves
__global__ void rope_kernel(bf16* qkv, int M, int S, int nh, int d, float theta, int inverse) {
  const int half = d / 2;
  const int g8 = half / 8;
  const float l2t = log2f(theta);
  long long n = (long long)M * nh * 2 * g8;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i8 = int(idx % g8);
    long long t = idx / g8;
    const int part = int(t % 2);
    t /= 2;
    const int h = int(t % nh);
    const int row = int(t / nh);
    const float pos = float(row % S);
    bf16* base = qkv + (long long)row * nh * 3 * d + (long long)h * 3 * d + part * d + i8 * 8;
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(base), a);
    unpack8(*reinterpret_cast<const uint4*>(base + half), b);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i8 * 8 + k;
      const float inv_freq = exp2f(-2.0f * float(i) / float(d) * l2t);
      float sn, cs;
      sincosf(pos * inv_freq, &sn, &cs);
      if (inverse) sn = -sn;
      const float x = a[k], y = b[k];
      a[k] = x * cs - y * sn;
      b[k] = y * cs + x * sn;
    }
    *reinterpret_cast<uint4*>(base) = pack8(a);
    *reinterpret_cast<uint4*>(base + half) = pack8(b);
  }
}

// ------------------------------------------------------------------ softmax
// one warp per row of one (batch) matrix; row i reads S[i, 0..i]
__global__ void softmax_fwd_kernel(const float* __restrict__ S, bf16* __restrict__ P, int L,
                                   long long rows) {
  long long row = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= rows) return;
  int i = int(row % L);
  const float* s = S + row * L;
  bf16* p = P + row * L;
  int n = i + 1;
  float mx = -FLT_MAX;
  for (int j = lane; j < n; j += 32) mx = fmaxf(mx, s[j]);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < n; j += 32) sum += __expf(s[j] - mx);
  sum = warp_sum(sum);
  float inv = 1.f / sum;
  int end = min(L, (i / 128 + 1) * 128);
  for (int j = lane; j < end; j += 32)
    p[j] = __float2bfloat16_rn(j < n ? __expf(s[j] - mx) * inv : 0.f);
}

__global__ void softmax_bwd_kernel(const bf16* __restrict__ P, const float* __restrict__ dP,
                                   bf16* __restrict__ dS, float scale, int L, long long rows) {
  long long row = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= rows) return;
  int i = int(row % L);
  const bf16* p = P + row * L;
  const float* dp = dP + row * L;
  bf16* ds = dS + row * L;
  int n = i + 1;
  float dot = 0.f;
  for (int j = lane; j < n; j += 32) dot += bf(p[j]) * dp[j];
  dot = warp_sum(dot);
  int end = min(L, (i / 128 + 1) * 128);
  for (int j = lane; j < end; j += 32)
    ds[j] = __float2bfloat16_rn(j < n ? scale * bf(p[j]) * (dp[j] - dot) : 0.f);
}

// ------------------------------------------------------------------ swiglu
__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + __expf(-x)); }

// thread per 8 consecutive ffn columns: 16-byte gate / up / out accesses
__global__ void swiglu_fwd_kernel(const bf16* __restrict__ gu, bf16* __restrict__ a, int M,
                                  int F) {
  const long long n = (long long)M * (F / 8);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / (F / 8);
    const int f = int(idx % (F / 8)) * 8;
    const bf16* r = gu + row * 2 * F + (f / 64) * 128 + (f % 64);
    float g[8], u[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(r), g);
    unpack8(*reinterpret_cast<const uint4*>(r + 64), u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoidf_(g[k]) * u[k];
    *reinterpret_cast<uint4*>(a + row * F + f) = pack8(o);
  }
}

__global__ void swiglu_bwd_kernel(const bf16* __restrict__ gu, const bf16* __restrict__ da,
                                  bf16* __restrict__ dgu, int M, int F) {
  const long long n = (long long)M * (F / 8);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / (F / 8);
    const int f = int(idx % (F / 8)) * 8;
    const long long off = row * 2 * F + (f / 64) * 128 + (f % 64);
    float g[8], u[8], d[8], dg[8], du[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + off), g);
    unpack8(*reinterpret_cast<const uint4*>(gu + off + 64), u);
    unpack8(*reinterpret_cast<const uint4*>(da + row * F + f), d);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float sg = sigmoidf_(g[k]);
      dg[k] = d[k] * u[k] * sg * (1.f + g[k] * (1.f - sg));
      du[k] = d[k] * g[k] * sg;
    }
    *reinterpret_cast<uint4*>(dgu + off) = pack8(dg);
    *reinterpret_cast<uint4*>(dgu + off + 64) = pack8(du);
  }
}

// ------------------------------------------------------------------ cross entropy
__device__ __forceinline__ int target_of(const int32_t* tok, int row, int S) {
  return tok[(row / S) * (S + 1) + row % S + 1];
}

// one block (256 threads) per row, online max/sum
__global__ void ce_stats_kernel(const float* __restrict__ logits, int Vr, int v0,
                                const int32_t* __restrict__ tok, int M, int S, float* lmax,
                                float* lsum, float* st2) {
  int row = blockIdx.x;
  const float* l = logits + (long long)row * Vr;
  float mx = -FLT_MAX, sm = 0.f;
  for (int j = threadIdx.x; j < Vr; j += blockDim.x) {
    float v = l[j];
    if (v > mx) {
      sm = sm * __expf(mx - v) + 1.f;
      mx = v;
    } else {
      sm += __expf(v - mx);
    }
  }
  // combine (mx, sm) across the block
  __shared__ float smx[32], ssm[32];
  for (int o = 16; o > 0; o >>= 1) {
    float om = __shfl_xor_sync(0xffffffffu, mx, o);
    float os = __shfl_xor_sync(0xffffffffu, sm, o);
    float nm = fmaxf(mx, om);
    sm = sm * __expf(mx - nm) + os * __expf(om - nm);
    mx = nm;
  }
  int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    smx[w] = mx;
    ssm[w] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -FLT_MAX, s = 0.f;
    for (int i = 0; i < (int)blockDim.x / 32; ++i) {
      float nm = fmaxf(m, smx[i]);
      s = s * __expf(m - nm) + ssm[i] * __expf(smx[i] - nm);
      m = nm;
    }
    lmax[row] = m;
    lsum[row] = s;
    int t = target_of(tok, row, S) - v0;
    st2[2 * row + 1] = (t >= 0 && t < Vr) ? l[t] : 0.f;
    st2[2 * row] = s;  // valid when tp == 1 (gmax == lmax)
  }
}

__global__ void ce_rescale_kernel(const float* lmax, const float* lsum, const float* gmax,
                                  float* st2, int M) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) st2[2 * i] = lsum[i] * __expf(lmax[i] - gmax[i]);
}

__global__ void ce_finish_kernel(const float* __restrict__ logits, int Vr, int v0,
                                 const int32_t* __restrict__ tok, int M, int S,
                                 const float* __restrict__ gmax, const float* __restrict__ st2,
                                 float inv_count, bf16* __restrict__ dl, float* loss_acc) {
  int row = blockIdx.x;
  const float* l = logits + (long long)row * Vr;
  bf16* d = dl + (long long)row * Vr;
  float m = gmax[row];
  float inv_s = 1.f / st2[2 * row];
  int t = target_of(tok, row, S) - v0;
  for (int j = threadIdx.x; j < Vr; j += blockDim.x) {
    float p = __expf(l[j] - m) * inv_s;
    if (j == t) p -= 1.f;
    d[j] = __float2bfloat16_rn(p * inv_count);
  }
  if (threadIdx.x == 0 && v0 == 0) {
    // loss counted once per row, on the rank owning vocab offset 0
    float loss = logf(st2[2 * row]) + m - st2[2 * row + 1];
    atomicAdd(loss_acc, loss);
  }
}

// ------------------------------------------------------------------ DP + optimizer
__global__ void scale_cast_kernel(const float* g, bf16* out, long long n, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(g[i] * scale);
}

__global__ void scale_kernel(float* g, long long n, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    g[i] *= scale;
}

__global__ void adamw_kernel(float* __restrict__ p, bf16* __restrict__ p16, float* __restrict__ m,
                             float* __restrict__ v, const bf16* __restrict__ g16,
                             const float* __restrict__ g32, long long n, float gscale, float lr,
                             float b1, float b2, float eps, float wd, float bc1, float bc2,
                             const StepParams* sp) {
  if (sp) {
    bc1 = sp->bc1;
    bc2 = sp->bc2;
  }
  // 4 elements per thread-iteration: float4 p/m/v, 8-byte bf16 grad / copy
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float gg[4];
    if (g16) {
      uint2 w = __ldcs(reinterpret_cast<const uint2*>(g16) + i);
      __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&w.x);
      __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w.y);
      gg[0] = __low2float(a); gg[1] = __high2float(a); gg[2] = __low2float(b); gg[3] = __high2float(b);
    } else {
      float4 w = __ldcs(reinterpret_cast<const float4*>(g32) + i);
      gg[0] = w.x; gg[1] = w.y; gg[2] = w.z; gg[3] = w.w;
    }
    float4 pm = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* pp = &pm.x;
    float* mp = &mm.x;
    float* vp = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float g = gg[k] * gscale;
      mp[k] = b1 * mp[k] + (1.f - b1) * g;
      vp[k] = b2 * vp[k] + (1.f - b2) * g * g;
      pp[k] = pp[k] - lr * ((mp[k] / bc1) / (sqrtf(vp[k] / bc2) + eps) + wd * pp[k]);
    }
    reinterpret_cast<float4*>(p)[i] = pm;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (p16) {
      uint2 w;
      w.x = pack_bf16x2(pm.x, pm.y);
      w.y = pack_bf16x2(pm.z, pm.w);
      reinterpret_cast<uint2*>(p16)[i] = w;
    }
  }
  // scalar tail (n % 4)
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float g = (g16 ? bf(g16[i]) : g32[i]) * gscale;
    float mi = b1 * m[i] + (1.f - b1) * g;
    float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    float pi = p[i];
    pi = pi - lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * pi);
    p[i] = pi;
    if (p16) p16[i] = __float2bfloat16_rn(pi);
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
void k_init_normal(float* master, bf16* copy, long long n, long long off, uint64_t seed,
                   cudaStream_t s) {
  if (n > 0) init_normal_kernel<<<ew_grid(n, 4), 256, 0, s>>>(master, copy, n, off, seed);
}
void k_fill(float* p, bf16* copy, long long n, float v, cudaStream_t s) {
  if (n > 0) fill_kernel<<<ew_grid(n, 4), 256, 0, s>>>(p, copy, n, v);
}
void k_cast_bf16(const float* in, bf16* out, long long n, cudaStream_t s) {
  if (n > 0) cast_kernel<<<ew_grid(n, 4), 256, 0, s>>>(in, out, n);
}
void k_gen_tokens(int32_t* tok, long long ns, int S, long long sample0, uint64_t seed,
                  long long step, int vocab, cudaStream_t s, const StepParams* sp) {
  long long n = ns * (S + 1);
  if (n > 0)
    tokens_kernel<<<ew_grid(n, 1), 256, 0, s>>>(tok, ns, S + 1, sample0, seed, step, vocab, sp);
}

__global__ void step_tick_kernel(StepParams* sp, float b1, float b2) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    long long s = sp->next_step;
    sp->cur_step = s;
    sp->next_step = s + 1;
    sp->bc1 = 1.f - powf(b1, float(s + 1));
    sp->bc2 = 1.f - powf(b2, float(s + 1));
  }
}

void k_step_tick(StepParams* sp, float b1, float b2, cudaStream_t s) {
  step_tick_kernel<<<1, 32, 0, s>>>(sp, b1, b2);
}
void k_embed_fwd(const int32_t* tok, const float* E, float* x, int M, int S, int H,
                 cudaStream_t s) {
  if (M > 0) embed_fwd_kernel<<<M, 256, 0, s>>>(tok, E, x, M, S, H);
}
void k_embed_bwd(const int32_t* tok, const float* dx, float* dE, int M, int S, int H,
                 cudaStream_t s) {
  if (M > 0) embed_bwd_kernel<<<M, 256, 0, s>>>(tok, dx, dE, M, S, H);
}
void k_rmsnorm_fwd(const float* x, const bf16* y, float* xo, const float* g, bf16* out,
                   float* rstd, int M, int H, float eps, cudaStream_t s) {
  if (M > 0) rmsnorm_fwd_kernel<<<row_grid(M, 8), 256, 0, s>>>(x, y, xo, g, out, rstd, M, H, eps);
}
void k_residual_add(const float* x, const bf16* y, float* xo, long long n, cudaStream_t s) {
  if (n > 0) residual_add_kernel<<<ew_grid(n, 4), 256, 0, s>>>(x, y, xo, n);
}
void k_rmsnorm_bwd(const bf16* dyb, const float* dyf, const float* x, const float* rstd,
                   const float* g, const float* dres, float* dx, bf16* dxb, float* dg, int M,
                   int H, float* coef, cudaStream_t s) {
  if (M <= 0) return;
  const int band = 16;  // rows per block: enough blocks in flight to cover HBM latency
  dim3 g2((H / 4 + 127) / 128, (M + band - 1) / band);
  if (dyb) {
    rmsnorm_bwd_dot_kernel<true><<<row_grid(M, 8), 256, 0, s>>>(dyb, dyf, x, rstd, g, coef, M, H);
    rmsnorm_bwd_dx_kernel<true><<<g2, 128, 0, s>>>(dyb, dyf, x, rstd, coef, g, dres, dx, dxb, dg, M, H, band);
  } else {
    rmsnorm_bwd_dot_kernel<false><<<row_grid(M, 8), 256, 0, s>>>(dyb, dyf, x, rstd, g, coef, M, H);
    rmsnorm_bwd_dx_kernel<false><<<g2, 128, 0, s>>>(dyb, dyf, x, rstd, coef, g, dres, dx, dxb, dg, M, H, band);
  }
}
void k_rope(bf16* qkv, int M, int S, int nh, int d, float theta, int inverse, cudaStream_t s) {
  long long n = (long long)M * nh * (d / 2);
  if (n > 0) rope_kernel<<<ew_grid(n, 4), 256, 0, s>>>(qkv, M, S, nh, d, theta, inverse);
}
void k_softmax_fwd(const float* S, bf16* P, int L, int nb, cudaStream_t s) {
  long long rows = (long long)L * nb;
  if (rows > 0) softmax_fwd_kernel<<<int((rows + 7) / 8), 256, 0, s>>>(S, P, L, rows);
}
void k_softmax_bwd(const bf16* P, const float* dP, bf16* dS, float scale, int L, int nb,
                   cudaStream_t s) {
  long long rows = (long long)L * nb;
  if (rows > 0) softmax_bwd_kernel<<<int((rows + 7) / 8), 256, 0, s>>>(P, dP, dS, scale, L, rows);
}
void k_swiglu_fwd(const bf16* gu, bf16* a, int M, int F, cudaStream_t s) {
  long long n = (long long)M * F;
  if (n > 0) swiglu_fwd_kernel<<<ew_grid(n, 8), 256, 0, s>>>(gu, a, M, F);
}
void k_swiglu_bwd(const bf16* gu, const bf16* da, bf16* dgu, int M, int F, cudaStream_t s) {
  long long n = (long long)M * F;
  if (n > 0) swiglu_bwd_kernel<<<ew_grid(n, 8), 256, 0, s>>>(gu, da, dgu, M, F);
}
void k_ce_stats(const float* logits, int Vr, int v0, const int32_t* tok, int M, int S,
                float* lmax, float* lsum, float* st2, cudaStream_t s) {
  if (M > 0) ce_stats_kernel<<<M, 256, 0, s>>>(logits, Vr, v0, tok, M, S, lmax, lsum, st2);
}
void k_ce_rescale(const float* lmax, const float* lsum, const float* gmax, float* st2, int M,
                  cudaStream_t s) {
  if (M > 0) ce_rescale_kernel<<<(M + 255) / 256, 256, 0, s>>>(lmax, lsum, gmax, st2, M);
}
void k_ce_finish(const float* logits, int Vr, int v0, const int32_t* tok, int M, int S,
                 const float* gmax, const float* st2, float inv_count, bf16* dl,
                 float* loss_acc, cudaStream_t s) {
  if (M > 0)
    ce_finish_kernel<<<M, 256, 0, s>>>(logits, Vr, v0, tok, M, S, gmax, st2, inv_count, dl, loss_acc);
}
void k_scale_cast(const float* g, bf16* out, long long n, float scale, cudaStream_t s) {
  if (n > 0) scale_cast_kernel<<<ew_grid(n, 4), 256, 0, s>>>(g, out, n, scale);
}
void k_scale(float* g, long long n, float scale, cudaStream_t s) {
  if (n > 0) scale_kernel<<<ew_grid(n, 4), 256, 0, s>>>(g, n, scale);
}
void k_adamw(float* p, bf16* p16, float* m, float* v, const bf16* g16, const float* g32,
             long long n, float gscale, float lr, float b1, float b2, float eps, float wd,
             float bc1, float bc2, cudaStream_t s, const StepParams* sp) {
  if (n > 0)
    adamw_kernel<<<ew_grid(n, 4), 256, 0, s>>>(p, p16, m, v, g16, g32, n, gscale, lr, b1, b2, eps,
                                               wd, bc1, bc2, sp);
}

}  // namespace hexexec
