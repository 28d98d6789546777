// Memory-bound kernels of the step (see kernels.h): 16-byte vector accesses
// where the row width allows; RMSNorm as CTA row bands (block reduction per
// row); elementwise kernels grid-stride with the grid sized to a multiple of
// the SM count.  Each kernel's HBM bytes and measured GB/s: scripts/bench_ew.py.
#include <cfloat>

#include <cub/device/device_radix_sort.cuh>

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

// fp32 <-> bf16 conversions (PP hand-off, DP gradient prep): 8 elements per
// thread step, 32-byte fp32 / 16-byte bf16 accesses when both pointers are
// 16-byte aligned (scalar otherwise); out = bf16(scale * in) / in_bf16 * 1
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__global__ void cast_kernel(const float* __restrict__ in, bf16* __restrict__ out, long long n,
                            float scale) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  long long done = 0;
  if (vec) {
    const long long n8 = n / 8;
    for (long long i = t; i < n8; i += stride) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(in) + 2 * i);
      const float4 b = __ldcs(reinterpret_cast<const float4*>(in) + 2 * i + 1);
      uint4 w;
      w.x = pk2(a.x * scale, a.y * scale);
      w.y = pk2(a.z * scale, a.w * scale);
      w.z = pk2(b.x * scale, b.y * scale);
      w.w = pk2(b.z * scale, b.w * scale);
      reinterpret_cast<uint4*>(out)[i] = w;
    }
    done = n8 * 8;
  }
  for (long long i = done + t; i < n; i += stride) out[i] = __float2bfloat16_rn(in[i] * scale);
}
__global__ void upcast_kernel(const bf16* __restrict__ in, float* __restrict__ out, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  long long done = 0;
  if (vec) {
    const long long n8 = n / 8;
    for (long long i = t; i < n8; i += stride) {
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(in) + i);
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
      float f[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        f[2 * k] = __uint_as_float(u[k] << 16);
        f[2 * k + 1] = __uint_as_float(u[k] & 0xffff0000u);
      }
      reinterpret_cast<float4*>(out)[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
      reinterpret_cast<float4*>(out)[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    done = n8 * 8;
  }
  for (long long i = done + t; i < n; i += stride) out[i] = __bfloat162float(in[i]);
}
__global__ void scale_kernel(float* g, long long n, float scale) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long done = 0;
  if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const long long n4 = n / 4;
    for (long long i = t; i < n4; i += stride) {
      float4 v = reinterpret_cast<float4*>(g)[i];
      v.x *= scale;
      v.y *= scale;
      v.z *= scale;
      v.w *= scale;
      reinterpret_cast<float4*>(g)[i] = v;
    }
    done = n4 * 4;
  }
  for (long long i = done + t; i < n; i += stride) g[i] *= scale;
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

// Embedding backward, deterministic: (1) one CTA sorts the micro-batch's
// (token, position) keys in shared memory (bitonic, M <= kEmbedSortMax);
// (2) the CTA at the start of each run of equal tokens sums those rows in
// position order and adds the sum to the token's dE row -- no atomics, so the
// gradient is bitwise reproducible (repeated tokens are common).
constexpr int kEmbedSortMax = 16384;

__global__ void __launch_bounds__(1024) embed_sort_kernel(const int32_t* tok, int M, int S,
                                                          uint32_t* keys) {
  extern __shared__ uint32_t sk[];
  int n = 1;
  while (n < M) n <<= 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    sk[i] = i < M ? (uint32_t(tok[(i / S) * (S + 1) + i % S]) << 16) | uint32_t(i) : 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t a = sk[i], b = sk[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            sk[i] = b;
            sk[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < M; i += blockDim.x) keys[i] = sk[i];
}

__global__ void embed_segsum_kernel(const uint32_t* __restrict__ keys, const float* __restrict__ dx,
                                    float* __restrict__ dE, int M, int H) {
  const int i = blockIdx.x;
  const uint32_t tk = keys[i] >> 16;
  if (i > 0 && (keys[i - 1] >> 16) == tk) return;  // not the start of a run
  int end = i + 1;
  while (end < M && (keys[end] >> 16) == tk) ++end;
  float* dst = dE + (long long)tk * H;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = i; r < end; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(dx + (long long)(keys[r] & 0xffffu) * H + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4 d = *reinterpret_cast<float4*>(dst + c);
    d.x += acc.x; d.y += acc.y; d.z += acc.z; d.w += acc.w;
    *reinterpret_cast<float4*>(dst + c) = d;
  }
}

// Large micro-batches (M > kEmbedSortMax tokens): 64-bit (token << 32 | row)
// keys sorted by a device radix sort (CUB, bits [0, 48): row < 2^32, token <
// 65536), then the same run sums in row order.
__global__ void embed_keys64_kernel(const int32_t* tok, int M, int S, unsigned long long* keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x)
    keys[i] = ((unsigned long long)uint32_t(tok[(long long)(i / S) * (S + 1) + i % S]) << 32) |
              unsigned(i);
}

__global__ void embed_segsum64_kernel(const unsigned long long* __restrict__ keys,
                                      const float* __restrict__ dx, float* __restrict__ dE, int M,
                                      int H) {
  const int i = blockIdx.x;
  const unsigned long long tk = keys[i] >> 32;
  if (i > 0 && (keys[i - 1] >> 32) == tk) return;  // not the start of a run
  int end = i + 1;
  while (end < M && (keys[end] >> 32) == tk) ++end;
  float* dst = dE + (long long)tk * H;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = i; r < end; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(dx + (long long)(keys[r] & 0xffffffffull) * H + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4 d = *reinterpret_cast<float4*>(dst + c);
    d.x += acc.x; d.y += acc.y; d.z += acc.z; d.w += acc.w;
    *reinterpret_cast<float4*>(dst + c) = d;
  }
}

// ------------------------------------------------------------------ rmsnorm
// Row-band kernels: a 256-thread CTA owns whole rows, each thread 8 columns
// per 2048-column chunk (NC chunks cover H), so a row is read from HBM once
// with every load of the row in flight together; the row statistic is a
// block reduction through a double-buffered smem slot (one barrier per row).
constexpr int kNormThreads = 256;
constexpr int kNormChunk = kNormThreads * 8;

__device__ __forceinline__ void load8f(const float* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void store8f(float* p, const float* f) {
  *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
}
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

// sum over the CTA; red is [2][8] floats, parity alternates per row
__device__ __forceinline__ float norm_block_sum(float v, float* red, int parity) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) red[parity * 8 + w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) s += red[parity * 8 + i];
  return s;
}

template <int NC>
__global__ void __launch_bounds__(kNormThreads)
    rmsnorm_fwd_kernel(const float* __restrict__ x, const bf16* __restrict__ y, float* xo,
                       const float* __restrict__ g, bf16* __restrict__ out,
                       float* __restrict__ rstd, int M, int H, float eps, int ny, long long ys) {
  __shared__ float red[16];
  float gr[NC][8];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = c * kNormChunk + threadIdx.x * 8;
    if (col < H) load8f(g + col, gr[c]);
  }
  int parity = 0;
  for (int row = blockIdx.x; row < M; row += gridDim.x, parity ^= 1) {
    const long long base = (long long)row * H;
    float v[NC][8];
    float ss = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int col = c * kNormChunk + threadIdx.x * 8;
      if (col < H) {
        load8f(x + base + col, v[c]);
        if (y) {
          // TP partials (slots in rank order: the same sum on every TP rank)
          for (int j = 0; j < ny; ++j) {
            float t[8];
            unpack8(*reinterpret_cast<const uint4*>(y + j * ys + base + col), t);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[c][k] += t[k];
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) ss += v[c][k] * v[c][k];
      }
    }
    ss = norm_block_sum(ss, red, parity);
    const float r = rsqrtf(ss / float(H) + eps);
    if (threadIdx.x == 0) rstd[row] = r;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int col = c * kNormChunk + threadIdx.x * 8;
      if (col < H) {
        if (y) store8f(xo + base + col, v[c]);
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = v[c][k] * r * gr[c][k];
        *reinterpret_cast<uint4*>(out + base + col) = pack8(o);
      }
    }
  }
}

__global__ void residual_add_kernel(const float* x, const bf16* y, float* xo, long long n, int ny,
                                    long long ys) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float v = x[i];
    for (int j = 0; j < ny; ++j) v += bf(y[j * ys + i]);
    xo[i] = v;
  }
}

// 8 elements per thread (16-byte partial loads, 2 x float4 residual / output)
__global__ void residual_add8_kernel(const float* __restrict__ x, const bf16* __restrict__ y,
                                     float* __restrict__ xo, long long n8, int ny, long long ys) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    float v[8];
    load8f(x + 8 * i, v);
    for (int j = 0; j < ny; ++j) {
      float t[8];
      unpack8(*reinterpret_cast<const uint4*>(y + j * ys + 8 * i), t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] += t[k];
    }
    store8f(xo + 8 * i, v);
  }
}

// RMSNorm backward, one pass; a persistent CTA per SM walks rows
// blockIdx.x, +grid, ... through a ring of shared-memory stages filled by
// 1-D bulk copies (x, dy, dres of one row per stage):
//   c   = r^3/H * sum_j dy*g*x            (block reduction per row)
//   dx  = dres + r*dy*g - x*c
//   dg += sum_rows dy*x*r                 (registers over the CTA's rows, one
//                                          partial row per CTA, summed in CTA
//                                          order by colsum_add_kernel)
// Stage reuse needs no extra barrier: the per-row reduction barrier of row k
// proves every thread has finished row k-1, whose stage is refilled then.
// Thread t owns columns c*2048 + q*1024 + 4t .. +3 (q = 0, 1): conflict-free
// 16-byte shared reads and coalesced global stores.
constexpr int kNormStages = 4;

template <int NC, bool kDyBf16>
__global__ void __launch_bounds__(kNormThreads, NC <= 2 ? 2 : 1)
    rmsnorm_bwd_kernel(const bf16* __restrict__ dyb, const float* __restrict__ dyf,
                       const float* __restrict__ x, const float* __restrict__ rstd,
                       const float* __restrict__ g, const float* dres, float* dx,
                       bf16* __restrict__ dxb, float* __restrict__ dg_part, int M, int H, int nst,
                       int ny, long long ys) {
  extern __shared__ uint8_t nsm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(nsm_raw) + 127) & ~uintptr_t(127));
  __shared__ float red[16];
  __shared__ __align__(8) uint64_t full[kNormStages];
  // dy: ny bf16 TP partial slots (summed in slot order), or one fp32 row
  const uint32_t xb = uint32_t(H) * 4, yb = uint32_t(H) * (kDyBf16 ? 2 * ny : 4);
  const uint32_t rb = dres ? uint32_t(H) * 4 : 0;
  const uint32_t stage_bytes = xb + yb + rb;
  const int G = gridDim.x;
  const int nrows = blockIdx.x < M ? (M - 1 - int(blockIdx.x)) / G + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const long long row = blockIdx.x + (long long)k * G;
    const int s = k % nst;
    uint8_t* st = sm + size_t(s) * stage_bytes;
    mbar_arrive_expect_tx(&full[s], stage_bytes);
    bulk_load_1d(st, x + row * H, xb, &full[s]);
    if (kDyBf16) {
      for (int j = 0; j < ny; ++j)
        bulk_load_1d(st + xb + size_t(j) * H * 2, dyb + j * ys + row * H, uint32_t(H) * 2, &full[s]);
    } else
      bulk_load_1d(st + xb, dyf + row * H, yb, &full[s]);
    if (dres) bulk_load_1d(st + xb + yb, dres + row * H, rb, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < nst && k < nrows; ++k) issue(k);

  float gr[NC][8], acc[NC][8];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = c * kNormChunk + q * (kNormChunk / 2) + threadIdx.x * 4;
      if (col < H) {
        const float4 v = *reinterpret_cast<const float4*>(g + col);
        gr[c][4 * q] = v.x; gr[c][4 * q + 1] = v.y; gr[c][4 * q + 2] = v.z; gr[c][4 * q + 3] = v.w;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[c][4 * q + k] = 0.f;
    }

  float r_next = nrows > 0 ? rstd[blockIdx.x] : 0.f;
  for (int k = 0; k < nrows; ++k) {
    const long long row = blockIdx.x + (long long)k * G;
    const long long base = row * H;
    const float r = r_next;
    if (k + 1 < nrows) r_next = rstd[row + G];  // one row ahead: off the critical path
    const int s = k % nst;
    const uint8_t* st = sm + size_t(s) * stage_bytes;
    const float* sx = reinterpret_cast<const float*>(st);
    const float* sres = reinterpret_cast<const float*>(st + xb + yb);
    mbar_wait(&full[s], uint32_t(k / nst) & 1u);
    float xv[NC][8], dv[NC][8];
    float dot = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = c * kNormChunk + q * (kNormChunk / 2) + threadIdx.x * 4;
        if (col < H) {
          const float4 xx = lds_f4(sx + col);
          float d4[4];
          if (kDyBf16) {
            d4[0] = d4[1] = d4[2] = d4[3] = 0.f;
            for (int j = 0; j < ny; ++j) {
              const uint2 w = lds_u2(st + xb + (size_t(j) * H + size_t(col)) * 2);
              const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&w.x);
              const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
              d4[0] += __low2float(a); d4[1] += __high2float(a);
              d4[2] += __low2float(b); d4[3] += __high2float(b);
            }
          } else {
            const float4 v = lds_f4(st + xb + size_t(col) * 4);
            d4[0] = v.x; d4[1] = v.y; d4[2] = v.z; d4[3] = v.w;
          }
          const float x4[4] = {xx.x, xx.y, xx.z, xx.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            xv[c][4 * q + e] = x4[e];
            dv[c][4 * q + e] = d4[e];
            dot += d4[e] * gr[c][4 * q + e] * x4[e];
            acc[c][4 * q + e] += d4[e] * x4[e] * r;
          }
        }
      }
    dot = norm_block_sum(dot, red, k & 1);
    if (threadIdx.x == 0 && k >= 1 && k - 1 + nst < nrows) issue(k - 1 + nst);
    const float cf = dot * r * r * r / float(H);
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = c * kNormChunk + q * (kNormChunk / 2) + threadIdx.x * 4;
        if (col < H) {
          float o[4];
          if (dres) {
            const float4 v = lds_f4(sres + col);
            o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
          } else {
            o[0] = o[1] = o[2] = o[3] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            o[e] += r * dv[c][4 * q + e] * gr[c][4 * q + e] - xv[c][4 * q + e] * cf;
          *reinterpret_cast<float4*>(dx + base + col) = make_float4(o[0], o[1], o[2], o[3]);
          if (dxb) {
            uint2 w;
            w.x = pack_bf16x2(o[0], o[1]);
            w.y = pack_bf16x2(o[2], o[3]);
            *reinterpret_cast<uint2*>(dxb + base + col) = w;
          }
        }
      }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = c * kNormChunk + q * (kNormChunk / 2) + threadIdx.x * 4;
      if (col < H) {
        *reinterpret_cast<float4*>(dg_part + (long long)blockIdx.x * H + col) =
            make_float4(acc[c][4 * q], acc[c][4 * q + 1], acc[c][4 * q + 2], acc[c][4 * q + 3]);
      }
    }
}

// dg[j] += sum of the CTA partial rows, in a fixed order (deterministic):
// block = 32 columns x 32 row groups; group g sums rows g, g+32, ... then the
// 32 group sums are added in group order
__global__ void __launch_bounds__(1024) colsum_add_kernel(const float* __restrict__ part, int rows,
                                                          int H, float* __restrict__ dg) {
  __shared__ float red[32][33];
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int grp = threadIdx.x >> 5;
  float s = 0.f;
  if (j < H) {
#pragma unroll 4
    for (int r = grp; r < rows; r += 32) s += part[(long long)r * H + j];
  }
  red[grp][threadIdx.x & 31] = s;
  __syncthreads();
  if (grp == 0 && j < H) {
    float t = red[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < 32; ++g) t += red[g][threadIdx.x];
    dg[j] += t;
  }
}

// ------------------------------------------------------------------ rope
// thread per (row, group of kRopeHeads heads, 8 rotation pairs): the 8
// sin/cos pairs are computed once and applied to q and k of every head in
// the group; 16-byte loads of both halves, all loads of the group in flight
constexpr int kRopeHeads = 4;
// (cos, sin) of position p and rotation pair i, the same expressions as below
__global__ void rope_table_kernel(float2* tab, int S, int d, float theta) {
  const int half = d / 2;
  const float l2t = log2f(theta);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < S * half;
       idx += gridDim.x * blockDim.x) {
    const int i = idx % half;
    const float pos = float(idx / half);
    const float inv_freq = exp2f(-2.0f * float(i) / float(d) * l2t);
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    tab[idx] = make_float2(cs, sn);
  }
}
__global__ void rope_kernel(bf16* qkv, int M, int S, int nh, int d, float theta, int inverse) {
  const int half = d / 2;
  const int g8 = half / 8;
  const int ng = (nh + kRopeHeads - 1) / kRopeHeads;
  const float l2t = log2f(theta);
  long long n = (long long)M * ng * g8;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i8 = int(idx % g8);
    long long t = idx / g8;
    const int hg = int(t % ng);
    const int row = int(t / ng);
    const float pos = float(row % S);
    float sn[8], cs[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i8 * 8 + k;
      const float inv_freq = exp2f(-2.0f * float(i) / float(d) * l2t);
      sincosf(pos * inv_freq, &sn[k], &cs[k]);
      if (inverse) sn[k] = -sn[k];
    }
    bf16* rbase = qkv + (long long)row * nh * 3 * d + i8 * 8;
#pragma unroll
    for (int j = 0; j < 2 * kRopeHeads; ++j) {
      const int h = hg * kRopeHeads + j / 2;
      if (h >= nh) break;
      bf16* base = rbase + (long long)h * 3 * d + (j & 1) * d;
      float a[8], b[8];
      unpack8(*reinterpret_cast<const uint4*>(base), a);
      unpack8(*reinterpret_cast<const uint4*>(base + half), b);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // explicit rounding (no FMA contraction): bitwise the same values as
        // the QKV-epilogue and dq-cast rotations (the oracle's float64 tables
        // differ in the last bits; it is compared within tolerance)
        const float x = a[k], y = b[k];
        a[k] = __fsub_rn(__fmul_rn(x, cs[k]), __fmul_rn(y, sn[k]));
        b[k] = __fadd_rn(__fmul_rn(y, cs[k]), __fmul_rn(x, sn[k]));
      }
      *reinterpret_cast<uint4*>(base) = pack8(a);
      *reinterpret_cast<uint4*>(base + half) = pack8(b);
    }
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
  // 8 logits per step (two float4, Vr % 64 == 0): one rescale per 8 values
  const float4* l4 = reinterpret_cast<const float4*>(l);
  for (int j = threadIdx.x; j < Vr / 8; j += blockDim.x) {
    const float4 a = l4[2 * j], b = l4[2 * j + 1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    float m8 = v[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) m8 = fmaxf(m8, v[k]);
    if (m8 > mx) {
      sm *= __expf(mx - m8);
      mx = m8;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) sm += __expf(v[k] - mx);
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
                                 float inv_count, bf16* __restrict__ dl, float* row_loss) {
  int row = blockIdx.x;
  const float* l = logits + (long long)row * Vr;
  bf16* d = dl + (long long)row * Vr;
  float m = gmax[row];
  float inv_s = 1.f / st2[2 * row];
  int t = target_of(tok, row, S) - v0;
  const float4* l4 = reinterpret_cast<const float4*>(l);
  for (int j = threadIdx.x; j < Vr / 4; j += blockDim.x) {
    const float4 a = l4[j];
    float p[4] = {__expf(a.x - m) * inv_s, __expf(a.y - m) * inv_s, __expf(a.z - m) * inv_s,
                  __expf(a.w - m) * inv_s};
    if (t >= 4 * j && t < 4 * j + 4) p[t - 4 * j] -= 1.f;
    uint2 w;
    w.x = pack_bf16x2(p[0] * inv_count, p[1] * inv_count);
    w.y = pack_bf16x2(p[2] * inv_count, p[3] * inv_count);
    *reinterpret_cast<uint2*>(d + 4 * j) = w;
  }
  if (threadIdx.x == 0 && v0 == 0) {
    // loss counted once per row, on the rank owning vocab offset 0
    row_loss[row] = logf(st2[2 * row]) + m - st2[2 * row + 1];
  }
}

// loss_acc += sum of the row losses in a fixed order (one CTA; deterministic)
__global__ void __launch_bounds__(1024) loss_sum_kernel(const float* __restrict__ row_loss, int M,
                                                        float* loss_acc) {
  __shared__ float red[32];
  float acc = 0.f;
  for (int i = threadIdx.x; i < M; i += blockDim.x) acc += row_loss[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = red[threadIdx.x];
    v = warp_sum(v);
    if (threadIdx.x == 0) *loss_acc += v;
  }
}

// ------------------------------------------------------------------ DP + optimizer

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
  if (n > 0) cast_kernel<<<ew_grid(n, 8), 256, 0, s>>>(in, out, n, 1.f);
}
void k_upcast_bf16(const bf16* in, float* out, long long n, cudaStream_t s) {
  if (n > 0) upcast_kernel<<<ew_grid(n, 8), 256, 0, s>>>(in, out, n);
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

// epoch = (step + 1) << 24 | op: strictly increasing over the run, never 0
__global__ void tp_sync_kernel(TpPeers p, const StepParams* sp, unsigned op) {
  const int k = threadIdx.x;
  if (k >= p.tp || k == p.me) return;
  const unsigned long long e = ((unsigned long long)(sp->cur_step + 1) << 24) | op;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.remote[k]), "l"(e) : "memory");
  unsigned long long v = 0;
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.local + k) : "memory");
  } while (v < e);
}
void k_tp_sync(const TpPeers& p, const StepParams* sp, unsigned op, cudaStream_t s) {
  tp_sync_kernel<<<1, 32, 0, s>>>(p, sp, op);
}

// copy of a peer's exchange slot into the local one (the pull of the critical
// TP rank's partial): 16-byte remote loads over NVLink, 4 in flight per thread
__global__ void __launch_bounds__(256) peer_copy_kernel(uint4* __restrict__ dst,
                                                        const uint4* __restrict__ src, long long n16) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcg(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[i + k * stride] = v[k];
  }
  for (; i < n16; i += stride) dst[i] = __ldcg(src + i);
}
void k_peer_copy(void* dst, const void* src, size_t bytes, int sms, cudaStream_t s) {
  const long long n16 = (long long)(bytes / 16);
  if (n16 > 0)
    peer_copy_kernel<<<std::max(1, sms) * 4, 256, 0, s>>>(static_cast<uint4*>(dst),
                                                          static_cast<const uint4*>(src), n16);
}

// SM placement probe: CTA b records its %smid, holding the SM ~spin_ns so
// the grid spreads over every SM the stream's context may use
__global__ void smid_probe_kernel(int* log, long long spin_ns) {
  if (threadIdx.x != 0) return;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  log[blockIdx.x] = int(sm);
  long long t0, t = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < spin_ns);
}
void k_smid_probe(int* log, int n, cudaStream_t s) {
  if (n > 0) smid_probe_kernel<<<n, 32, 0, s>>>(log, 20000);
}

void k_step_tick(StepParams* sp, float b1, float b2, cudaStream_t s) {
  step_tick_kernel<<<1, 32, 0, s>>>(sp, b1, b2);
}
void k_embed_fwd(const int32_t* tok, const float* E, float* x, int M, int S, int H,
                 cudaStream_t s) {
  if (M > 0) embed_fwd_kernel<<<M, 256, 0, s>>>(tok, E, x, M, S, H);
}
size_t embed_bwd_scratch_bytes(int M) {
  if (M <= kEmbedSortMax) return size_t(M) * 4;
  size_t temp = 0;
  if (cub::DeviceRadixSort::SortKeys(nullptr, temp, static_cast<const unsigned long long*>(nullptr),
                                     static_cast<unsigned long long*>(nullptr), M, 0, 48) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    temp = 2 * size_t(M) * 8 + (size_t(1) << 20);  // no device (host-only sizing): upper bound
  }
  return 2 * size_t(M) * 8 + (temp + 255) / 256 * 256;
}
void k_embed_bwd(const int32_t* tok, const float* dx, float* dE, int M, int S, int H,
                 void* scratch, cudaStream_t s) {
  if (M <= 0) return;
  if (M > kEmbedSortMax) {
    auto* kin = static_cast<unsigned long long*>(scratch);
    auto* kout = kin + M;
    size_t temp = embed_bwd_scratch_bytes(M) - 2 * size_t(M) * 8;
    embed_keys64_kernel<<<ew_grid(M, 4), 256, 0, s>>>(tok, M, S, kin);
    cub::DeviceRadixSort::SortKeys(static_cast<void*>(kout + M), temp, kin, kout, M, 0, 48, s);
    embed_segsum64_kernel<<<M, 256, 0, s>>>(kout, dx, dE, M, H);
    return;
  }
  uint32_t* keys = static_cast<uint32_t*>(scratch);
  int n = 1;
  while (n < M) n <<= 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(embed_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kEmbedSortMax * 4);
    attr = true;
  }
  embed_sort_kernel<<<1, 1024, size_t(n) * 4, s>>>(tok, M, S, keys);
  embed_segsum_kernel<<<M, 256, 0, s>>>(keys, dx, dE, M, H);
}
// H <= 4 * 2048 (checked by the executor's model validation)
void k_rmsnorm_fwd(const float* x, const bf16* y, float* xo, const float* g, bf16* out,
                   float* rstd, int M, int H, float eps, cudaStream_t s, int ny, long long ys) {
  if (M <= 0) return;
  // equal row counts per CTA within one resident wave (2048 rows: 1024 CTAs x 2
  // rows rather than 1184 CTAs x 1-2 rows, whose 2-row CTAs form a tail)
  const int per = (M + 148 * 8 - 1) / (148 * 8);
  const int grid = (M + per - 1) / per;
  const int nc = (H + kNormChunk - 1) / kNormChunk;
#define HX_NORM_FWD(NC) \
  rmsnorm_fwd_kernel<NC><<<grid, kNormThreads, 0, s>>>(x, y, xo, g, out, rstd, M, H, eps, ny, ys)
  if (nc <= 1) HX_NORM_FWD(1);
  else if (nc == 2) HX_NORM_FWD(2);
  else if (nc == 3) HX_NORM_FWD(3);
  else HX_NORM_FWD(4);
#undef HX_NORM_FWD
}
void k_residual_add(const float* x, const bf16* y, float* xo, long long n, cudaStream_t s, int ny,
                    long long ys) {
  if (n <= 0) return;
  const bool vec = n % 8 == 0 && ys % 8 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(y) % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(xo) % 16) == 0;
  if (vec)
    residual_add8_kernel<<<ew_grid(n / 8, 1), 256, 0, s>>>(x, y, xo, n / 8, ny, ys);
  else
    residual_add_kernel<<<ew_grid(n, 4), 256, 0, s>>>(x, y, xo, n, ny, ys);
}
void k_rmsnorm_bwd(const bf16* dyb, const float* dyf, const float* x, const float* rstd,
                   const float* g, const float* dres, float* dx, bf16* dxb, float* dg, int M,
                   int H, float* dg_part, cudaStream_t s, int ny, long long ys) {
  if (M <= 0) return;
  if (!dyb) ny = 1;
  // one persistent CTA per SM; each CTA's rows end in one partial dg row
  const int nc = (H + kNormChunk - 1) / kNormChunk;
  const int grid = std::min(M, kRmsBwdCtas);
  const size_t stage = size_t(H) * (4 + (dyb ? 2 * ny : 4) + (dres ? 4 : 0));
  const size_t budget = 200u << 10;
  const int nst = int(std::max<size_t>(1, std::min<size_t>(kNormStages, budget / stage)));
  const size_t smem = stage * nst + 128;
#define HX_NORM_BWD(NC, B)                                                                   \
  do {                                                                                      \
    static bool attr = false;                                                               \
    if (!attr) {                                                                            \
      cudaFuncSetAttribute(rmsnorm_bwd_kernel<NC, B>,                                       \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 210 << 10);         \
      attr = true;                                                                          \
    }                                                                                       \
    rmsnorm_bwd_kernel<NC, B><<<grid, kNormThreads, smem, s>>>(dyb, dyf, x, rstd, g, dres, dx, \
                                                                dxb, dg_part, M, H, nst, ny, ys); \
  } while (0)
#define HX_NORM_BWD_NC(B)       \
  if (nc <= 1) HX_NORM_BWD(1, B); \
  else if (nc == 2) HX_NORM_BWD(2, B); \
  else if (nc == 3) HX_NORM_BWD(3, B); \
  else HX_NORM_BWD(4, B);
  if (dyb) {
    HX_NORM_BWD_NC(true)
  } else {
    HX_NORM_BWD_NC(false)
  }
#undef HX_NORM_BWD_NC
#undef HX_NORM_BWD
  colsum_add_kernel<<<(H + 31) / 32, 1024, 0, s>>>(dg_part, grid, H, dg);
}
void k_rope_table(float2* tab, int S, int d, float theta, cudaStream_t s) {
  const int n = S * (d / 2);
  if (n > 0) rope_table_kernel<<<std::min(1184, (n + 255) / 256), 256, 0, s>>>(tab, S, d, theta);
}
void k_rope(bf16* qkv, int M, int S, int nh, int d, float theta, int inverse, cudaStream_t s) {
  long long n = (long long)M * ((nh + kRopeHeads - 1) / kRopeHeads) * (d / 16);
  if (n > 0) rope_kernel<<<ew_grid(n, 1), 256, 0, s>>>(qkv, M, S, nh, d, theta, inverse);
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
                 float* loss_acc, float* row_loss, cudaStream_t s) {
  if (M <= 0) return;
  ce_finish_kernel<<<M, 256, 0, s>>>(logits, Vr, v0, tok, M, S, gmax, st2, inv_count, dl, row_loss);
  if (v0 == 0) loss_sum_kernel<<<1, 1024, 0, s>>>(row_loss, M, loss_acc);
}
void k_scale_cast(const float* g, bf16* out, long long n, float scale, cudaStream_t s) {
  if (n > 0) cast_kernel<<<ew_grid(n, 8), 256, 0, s>>>(g, out, n, scale);
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
