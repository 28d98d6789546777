// Fused causal attention (flash-style) for sm_100a.
//
// Forward CTA = one (sample, head, 128-query tile).  Warp roles (256 thr):
//   warp 0  TMA producer: Q tile once, then K/V tiles into a 2-slot ring
//   warp 1  MMA issuer:   S_j = Q K_j^T (TMEM, double-buffered), O_j = P_j V_j (TMEM)
//   warp 2  TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4-7 softmax: one thread per query row; online max / sum in fp32,
//            P_j written bf16 into swizzled smem as the A operand of O_j,
//            O accumulated in registers (O = O*alpha + O_j), LSE saved.
// The MMA of S_{j+1} overlaps the softmax of S_j.  Causality: only key tiles
// j <= query tile are visited; the diagonal tile is masked per element.
// Backward: see attn_bwd_kernel below.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <mutex>

#include "attention.h"
#include "common.cuh"

namespace hexexec {

namespace {

constexpr int T = 128;          // query / key tile
constexpr int kThreads = 256;
constexpr uint32_t ATOM = 16384;  // [128 rows][64 bf16] SWIZZLE_128B atom column block

struct AttnParams {
  __nv_bfloat16* out;
  float* lse;
  int S, nh, mb, ldo;
  float scale_log2;
};

template <int D>
struct FwdCfg {
  static constexpr uint32_t TILE = T * D * 2;          // Q / K / V tile bytes
  static constexpr uint32_t P_BYTES = T * T * 2;
  static constexpr uint32_t SMEM = 1024 + TILE * 5 + P_BYTES + 256;
};

HX_DEVICE uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// K-major operand made of 64-column atoms: k-step ks of 16 elements
HX_DEVICE uint64_t kdesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks / 4) * ATOM + (ks % 4) * 32, 16, 1024);
}

// MN-major operand staged as [64-row k block][n atoms of 64][64 k rows x 128 B]
template <int NATOMS>
HX_DEVICE uint64_t mndesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks / 4) * (NATOMS * 8192) + (ks % 4) * 2048, 8192, 1024);
}

// byte offset of 16-byte chunk `kc` (8 bf16 along K) of row r in a K-major
// SWIZZLE_128B operand made of 64-column atoms of [128 rows][128 B]
HX_DEVICE uint32_t kchunk(int r, int kc) {
  return uint32_t((kc / 8) * ATOM + r * 128 + (((kc % 8) ^ (r % 8)) * 16));
}

// 16-byte chunk q of row r in a [32 rows][128 B] SWIZZLE_128B TMA box
HX_DEVICE uint32_t swz128(int r, int q) { return uint32_t(r * 128 + ((q ^ (r % 8)) * 16)); }

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = FwdCfg<D>;
  constexpr int DA = D / 64;  // 64-column atoms across the head dim
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::TILE;          // [2]
  uint8_t* sV = sK + 2 * C::TILE;      // [2]
  uint8_t* sP = sV + 2 * C::TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;    // [2]
  uint64_t* s_empty = bar + 7;   // [2]
  uint64_t* p_full = bar + 9;
  uint64_t* o_full = bar + 10;
  uint64_t* o_empty = bar + 11;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 12);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nqt = p.S / T;
  // heaviest query tiles of every head first (longest-first over the grid)
  const int nz = p.mb * p.nh;
  const int qt = nqt - 1 - int(blockIdx.x / nz);
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int ntiles = qt + 1;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, C::TILE);
      for (int a = 0; a < DA; ++a) tma_load_4d(sQ + a * ATOM, &tmQ, q_full, a * 64, qt * T, h, b);
      for (int j = 0; j < ntiles; ++j) {
        const int slot = j & 1;
        mbar_wait(&kv_empty[slot], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[slot], 2 * C::TILE);
        uint8_t* k = sK + slot * C::TILE;
        uint8_t* v = sV + slot * C::TILE;
        for (int a = 0; a < DA; ++a)
          tma_load_4d(k + a * ATOM, &tmK, &kv_full[slot], a * 64, j * T, h, b);
        for (int kb = 0; kb < 2; ++kb)
          for (int a = 0; a < DA; ++a)
            tma_load_4d(v + kb * (DA * 8192) + a * 8192, &tmV, &kv_full[slot], a * 64,
                        j * T + kb * 64, h, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16(T, T, 0, 0);
      const uint32_t id_o = idesc_bf16(T, D, 0, 1);
      const uint32_t q_addr = smem_u32(sQ);
      const uint32_t p_addr = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int slot = j & 1;
        mbar_wait(&kv_full[slot], (j >> 1) & 1);
        mbar_wait(&s_empty[slot], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + slot * C::TILE);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + uint32_t(slot * T), kdesc(q_addr, ks), kdesc(k_addr, ks), id_s,
                     ks > 0 ? 1u : 0u);
        tc_commit(&s_full[slot]);
      };
      issue_s(0);
      for (int j = 0; j < ntiles; ++j) {
        const int slot = j & 1;
        if (j + 1 < ntiles) issue_s(j + 1);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + slot * C::TILE);
        // O accumulates in TMEM across key tiles (rescaled in place by the
        // softmax warps when their reference max moves)
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + 2 * T, kdesc(p_addr, ks), mndesc<DA>(v_addr, ks), id_o,
                     (j > 0 || ks > 0) ? 1u : 0u);
        tc_commit(o_full);
        tc_commit(&kv_empty[slot]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // query row within the tile
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    // m is a *reference* max: P = 2^(s*c - m) may exceed 1 by up to 2^8; O (in
    // TMEM) and l are rescaled only when some row's max grows past m + 8
    constexpr float kSlack = 8.f;
    float m = -FLT_MAX, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int slot = j & 1;
      const bool diag = j == qt;
      mbar_wait(&s_full[slot], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[T];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t* v = sv + c * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(tbase + lane_off + uint32_t(slot * T + c * 32)));
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[slot]);  // S slot may be overwritten now
      // 8 independent partial maxima (short dependency chains)
      float mx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx[k] = -FLT_MAX;
#pragma unroll
      for (int i = 0; i < T; ++i)
        if (!diag || i <= r) mx[i % 8] = fmaxf(mx[i % 8], __uint_as_float(sv[i]));
      float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      mt *= p.scale_log2;
      // P buffer and O must be released by the previous PV MMA first
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
      }
      if (__any_sync(0xffffffffu, mt > m + kSlack)) {
        const float m_new = fmaxf(m, mt);
        const float alpha = ex2(m - m_new);
        if (j > 0) {
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tbase + lane_off + uint32_t(2 * T + c * 32), v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tbase + lane_off + uint32_t(2 * T + c * 32), v);
          }
          tmem_st_wait();
        }
        l *= alpha;
        m = m_new;
      }
      float lsp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) lsp[k] = 0.f;
#pragma unroll
      for (int q = 0; q < T / 8; ++q) {
        float pr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = q * 8 + k;
          const float e = ex2(fmaf(__uint_as_float(sv[i]), p.scale_log2, -m));
          pr[k] = (!diag || i <= r) ? e : 0.f;
          lsp[k] += pr[k];
        }
        uint4 w;
        w.x = pack_bf16x2(pr[0], pr[1]);
        w.y = pack_bf16x2(pr[2], pr[3]);
        w.z = pack_bf16x2(pr[4], pr[5]);
        w.w = pack_bf16x2(pr[6], pr[7]);
        *reinterpret_cast<uint4*>(sP + kchunk(r, q)) = w;
      }
      l += ((lsp[0] + lsp[1]) + (lsp[2] + lsp[3])) + ((lsp[4] + lsp[5]) + (lsp[6] + lsp[7]));
      tc_fence_before();
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(o_full, (ntiles - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qi = qt * T + r;
    __nv_bfloat16* dst = p.out + ((long long)b * p.S + qi) * p.ldo + (long long)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tbase + lane_off + uint32_t(2 * T + c * 32), v);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        reinterpret_cast<uint4*>(dst)[c * 4 + q] = w;
      }
    }
    p.lse[((long long)b * p.nh + h) * p.S + qi] = m + log2f(l);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// Softmax row pieces, specialised on the diagonal tile so the causal mask
// costs nothing on the other tiles (one thread = one row r of the tile).
template <bool DIAG>
HX_DEVICE float row_max(const uint32_t (&sv)[T], int r) {
  float mx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) mx[k] = -FLT_MAX;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    const float v = __uint_as_float(sv[i]);
    mx[i % 8] = (!DIAG || i <= r) ? fmaxf(mx[i % 8], v) : mx[i % 8];
  }
  return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
}

// P = exp2(s * scale_log2 - m) -> bf16 K-major smem rows; returns the row sum
template <bool DIAG>
HX_DEVICE float exp_store_p(const uint32_t (&sv)[T], int r, float scale_log2, float m,
                            uint8_t* myP) {
  float lsp[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) lsp[k] = 0.f;
#pragma unroll
  for (int q = 0; q < T / 8; ++q) {
    float pv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = q * 8 + k;
      const float e = ex2(fmaf(__uint_as_float(sv[i]), scale_log2, -m));
      pv[k] = (!DIAG || i <= r) ? e : 0.f;
      lsp[k] += pv[k];
    }
    uint4 w;
    w.x = pack_bf16x2(pv[0], pv[1]);
    w.y = pack_bf16x2(pv[2], pv[3]);
    w.z = pack_bf16x2(pv[4], pv[5]);
    w.w = pack_bf16x2(pv[6], pv[7]);
    *reinterpret_cast<uint4*>(myP + kchunk(r, q)) = w;
  }
  return ((lsp[0] + lsp[1]) + (lsp[2] + lsp[3])) + ((lsp[4] + lsp[5]) + (lsp[6] + lsp[7]));
}

// ------------------------------------------------------------------ forward, 2 Q tiles
// CTA = one (sample, head) and the query-tile pair (2t, 2t+1).  Two softmax
// warpgroups (A: warps 4-7, B: warps 8-11) ping-pong: while one computes its
// softmax the tensor core runs the other tile's S or PV product.  K/V tiles
// are loaded once for both query tiles (K double-buffered, V single).
// TMEM: S_A | S_B | O_A | O_B (4 x 128 columns).  Register budget via
// setmaxnreg: the producer/MMA warpgroup drops to 56, softmax warpgroups get 224.
constexpr int kThreads2 = 384;

template <int D>
struct Fwd2Cfg {
  static constexpr uint32_t TILE = T * D * 2;
  static constexpr uint32_t P_BYTES = T * T * 2;
  static constexpr uint32_t SMEM = 1024 + 2 * TILE /*Q*/ + 2 * TILE /*K*/ + TILE /*V*/ +
                                   2 * P_BYTES + 256;
};

template <int D>
__global__ void __launch_bounds__(kThreads2, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Fwd2Cfg<D>;
  constexpr int DA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // [2 tiles]
  uint8_t* sK = sQ + 2 * C::TILE;      // [2 slots]
  uint8_t* sV = sK + 2 * C::TILE;      // [1 slot]
  uint8_t* sP = sV + C::TILE;          // [2 tiles]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * C::P_BYTES);
  uint64_t* q_full = bar;        // Q_A + Q_B
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* k_empty = bar + 3;   // [2]
  uint64_t* v_full = bar + 5;
  uint64_t* v_empty = bar + 6;
  uint64_t* s_full = bar + 7;    // [2 tiles]
  uint64_t* s_empty = bar + 9;   // [2 tiles]
  uint64_t* p_full = bar + 11;   // [2 tiles]
  uint64_t* o_full = bar + 13;   // [2 tiles]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 15);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nqt = p.S / T;
  const int npairs = (nqt + 1) / 2;
  // heaviest pairs of every head first (longest-first over the grid)
  const int nz = p.mb * p.nh;
  const int pr = npairs - 1 - int(blockIdx.x / nz);
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int qa = 2 * pr;                 // query tile of warpgroup A
  const bool has_b = qa + 1 < nqt;       // query tile qa+1 of warpgroup B
  const int nt_a = qa + 1;               // key tiles visited by A / B
  const int nt_b = has_b ? qa + 2 : 0;
  const int nkv = has_b ? nt_b : nt_a;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * C::TILE);
      for (int a = 0; a < DA; ++a) {
        tma_load_4d(sQ + a * ATOM, &tmQ, q_full, a * 64, qa * T, h, b);
        if (has_b) tma_load_4d(sQ + C::TILE + a * ATOM, &tmQ, q_full, a * 64, (qa + 1) * T, h, b);
      }
      for (int j = 0; j < nkv; ++j) {
        const int slot = j & 1;
        mbar_wait(&k_empty[slot], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[slot], C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sK + slot * C::TILE + a * ATOM, &tmK, &k_full[slot], a * 64, j * T, h, b);
        mbar_wait(v_empty, (j & 1) ^ 1);
        mbar_arrive_expect_tx(v_full, C::TILE);
        for (int kb = 0; kb < 2; ++kb)
          for (int a = 0; a < DA; ++a)
            tma_load_4d(sV + kb * (DA * 8192) + a * 8192, &tmV, v_full, a * 64, j * T + kb * 64, h, b);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t id_s = idesc_bf16(T, T, 0, 0);
      const uint32_t id_o = idesc_bf16(T, D, 0, 1);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int g, int j) {  // S_g(j) = Q_g K_j^T
        const int slot = j & 1;
        mbar_wait(&k_full[slot], (j >> 1) & 1);
        mbar_wait(&s_empty[g], (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sQ + g * C::TILE);
        const uint32_t k_addr = smem_u32(sK + slot * C::TILE);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + uint32_t(g * T), kdesc(q_addr, ks), kdesc(k_addr, ks), id_s,
                     ks > 0 ? 1u : 0u);
        tc_commit(&s_full[g]);
      };
      auto issue_o = [&](int g, int j) {  // O_g += P_g(j) V_j
        mbar_wait(&p_full[g], j & 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sP + g * C::P_BYTES);
        const uint32_t v_addr = smem_u32(sV);
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + uint32_t(2 * T + g * T), kdesc(p_addr, ks), mndesc<DA>(v_addr, ks),
                     id_o, (j > 0 || ks > 0) ? 1u : 0u);
        tc_commit(&o_full[g]);
      };
      // S_g(j+1) is issued as soon as warpgroup g has read S_g(j) out of TMEM,
      // so it computes during the softmax of tile j and both warpgroups'
      // softmax run concurrently (latency hiding across the pair)
      if (nt_a > 0) issue_s(0, 0);
      if (has_b) issue_s(1, 0);
      for (int j = 0; j < nkv; ++j) {
        const bool a_on = j < nt_a, b_on = j < nt_b;
        mbar_wait(v_full, j & 1);
        if (a_on) {
          issue_o(0, j);
          if (j + 1 < nt_a) issue_s(0, j + 1);
        }
        if (b_on) {
          issue_o(1, j);
          if (j + 1 < nt_b) issue_s(1, j + 1);
        }
        tc_commit(v_empty);               // V_j consumed once both PV products finish
        tc_commit(&k_empty[j & 1]);       // K_j consumed by both S products
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    const int g = (warp - 4) / 4;  // 0 = A, 1 = B
    const int ew = (warp - 4) % 4;
    const int qt = qa + g;
    const int ntiles = g == 0 ? nt_a : nt_b;
    if (ntiles > 0) {
      const int r = ew * 32 + lane;
      const uint32_t lane_off = uint32_t(ew * 32) << 16;
      const uint32_t s_col = uint32_t(g * T), o_col = uint32_t(2 * T + g * T);
      uint8_t* myP = sP + g * C::P_BYTES;
      constexpr float kSlack = 8.f;
      float m = -FLT_MAX, l = 0.f;
      for (int j = 0; j < ntiles; ++j) {
        const bool diag = j == qt;
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
        uint32_t sv[T];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t* v = sv + c * 32;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(tbase + lane_off + s_col + uint32_t(c * 32)));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[g]);
        float mt = (diag ? row_max<true>(sv, r) : row_max<false>(sv, r)) * p.scale_log2;
        if (j > 0) {  // PV_{j-1} done: P buffer free and O stable
          mbar_wait(&o_full[g], (j - 1) & 1);
          tc_fence_after();
        }
        if (__any_sync(0xffffffffu, mt > m + kSlack)) {
          const float m_new = fmaxf(m, mt);
          const float alpha = ex2(m - m_new);
          if (j > 0) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t v[32];
              tmem_ld_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
              tmem_st_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
            }
            tmem_st_wait();
          }
          l *= alpha;
          m = m_new;
        }
        l += diag ? exp_store_p<true>(sv, r, p.scale_log2, m, myP)
                  : exp_store_p<false>(sv, r, p.scale_log2, m, myP);
        tc_fence_before();
        fence_async_shared();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g]);
      }
      mbar_wait(&o_full[g], (ntiles - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      const int qi = qt * T + r;
      __nv_bfloat16* dst = p.out + ((long long)b * p.S + qi) * p.ldo + (long long)h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          reinterpret_cast<uint4*>(dst)[c * 4 + q] = w;
        }
      }
      p.lse[((long long)b * p.nh + h) * p.S + qi] = m + log2f(l);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// P = exp2(s * scale_log2 - m) packed in place as bf16 pairs: sv[k] holds
// columns (2k, 2k + 1) for k < T / 2 (the TMEM A-operand layout of P);
// returns the row sum of the fp32 values
template <bool DIAG>
HX_DEVICE float exp_pack_p(uint32_t (&sv)[T], int r, float scale_log2, float m) {
  float lsp[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) lsp[k] = 0.f;
#pragma unroll
  for (int k = 0; k < T / 2; ++k) {
    const int i = 2 * k;
    float e0 = ex2(fmaf(__uint_as_float(sv[i]), scale_log2, -m));
    float e1 = ex2(fmaf(__uint_as_float(sv[i + 1]), scale_log2, -m));
    e0 = (!DIAG || i <= r) ? e0 : 0.f;
    e1 = (!DIAG || i + 1 <= r) ? e1 : 0.f;
    lsp[i % 8] += e0;
    lsp[(i + 1) % 8] += e1;
    sv[k] = pack_bf16x2(e0, e1);
  }
  return ((lsp[0] + lsp[1]) + (lsp[2] + lsp[3])) + ((lsp[4] + lsp[5]) + (lsp[6] + lsp[7]));
}

// ------------------------------------------------------------------ forward, v3
// attn_fwd3_kernel with P kept in tensor memory: each softmax thread writes
// its row's P (bf16 pairs) over the S columns it has just read (tcgen05.st),
// and O += P V reads its A operand from TMEM -- P no longer goes through
// shared memory; the freed 64 KB double-buffer V.  S_g(j+1) overwrites those
// columns, so the MMA issuer waits for PV_g(j) (o_full) before issuing it.

template <int D>
struct Fwd3Cfg {
  static constexpr uint32_t TILE = T * D * 2;
  static constexpr uint32_t SMEM = 1024 + 2 * TILE /*Q*/ + 2 * TILE /*K*/ + 2 * TILE /*V*/ + 256;
};

template <int D>
__global__ void __launch_bounds__(kThreads2, 1)
    attn_fwd3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Fwd3Cfg<D>;
  constexpr int DA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // [2 tiles]
  uint8_t* sK = sQ + 2 * C::TILE;      // [2 slots]
  uint8_t* sV = sK + 2 * C::TILE;      // [2 slots]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * C::TILE);
  uint64_t* q_full = bar;        // Q_A + Q_B
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* k_empty = bar + 3;   // [2]
  uint64_t* v_full = bar + 5;    // [2]
  uint64_t* v_empty = bar + 15;  // [2]
  uint64_t* s_full = bar + 7;    // [2 tiles]
  uint64_t* s_empty = bar + 9;   // [2 tiles]
  uint64_t* p_full = bar + 11;   // [2 tiles]
  uint64_t* o_full = bar + 13;   // [2 tiles]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nqt = p.S / T;
  const int npairs = (nqt + 1) / 2;
  // heaviest pairs of every head first (longest-first over the grid)
  const int nz = p.mb * p.nh;
  const int pr = npairs - 1 - int(blockIdx.x / nz);
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int qa = 2 * pr;                 // query tile of warpgroup A
  const bool has_b = qa + 1 < nqt;       // query tile qa+1 of warpgroup B
  const int nt_a = qa + 1;               // key tiles visited by A / B
  const int nt_b = has_b ? qa + 2 : 0;
  const int nkv = has_b ? nt_b : nt_a;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * C::TILE);
      for (int a = 0; a < DA; ++a) {
        tma_load_4d(sQ + a * ATOM, &tmQ, q_full, a * 64, qa * T, h, b);
        if (has_b) tma_load_4d(sQ + C::TILE + a * ATOM, &tmQ, q_full, a * 64, (qa + 1) * T, h, b);
      }
      for (int j = 0; j < nkv; ++j) {
        const int slot = j & 1;
        mbar_wait(&k_empty[slot], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[slot], C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sK + slot * C::TILE + a * ATOM, &tmK, &k_full[slot], a * 64, j * T, h, b);
        mbar_wait(&v_empty[slot], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[slot], C::TILE);
        for (int kb = 0; kb < 2; ++kb)
          for (int a = 0; a < DA; ++a)
            tma_load_4d(sV + slot * C::TILE + kb * (DA * 8192) + a * 8192, &tmV, &v_full[slot],
                        a * 64, j * T + kb * 64, h, b);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t id_s = idesc_bf16(T, T, 0, 0);
      const uint32_t id_o = idesc_bf16(T, D, 0, 1);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int g, int j) {  // S_g(j) = Q_g K_j^T
        const int slot = j & 1;
        mbar_wait(&k_full[slot], (j >> 1) & 1);
        mbar_wait(&s_empty[g], (j & 1) ^ 1);
        // the S_g columns hold P_g(j-1) until PV_g(j-1) has read it
        if (j > 0) mbar_wait(&o_full[g], (j - 1) & 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sQ + g * C::TILE);
        const uint32_t k_addr = smem_u32(sK + slot * C::TILE);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + uint32_t(g * T), kdesc(q_addr, ks), kdesc(k_addr, ks), id_s,
                     ks > 0 ? 1u : 0u);
        tc_commit(&s_full[g]);
      };
      auto issue_o = [&](int g, int j) {  // O_g += P_g(j) V_j, P_g(j) from TMEM
        mbar_wait(&p_full[g], j & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + (j & 1) * C::TILE);
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16_ts(tbase + uint32_t(2 * T + g * T), tbase + uint32_t(g * T + ks * 8),
                        mndesc<DA>(v_addr, ks), id_o, (j > 0 || ks > 0) ? 1u : 0u);
        tc_commit(&o_full[g]);
      };
      // S_g(j+1) is issued as soon as warpgroup g has read S_g(j) out of TMEM,
      // so it computes during the softmax of tile j and both warpgroups'
      // softmax run concurrently (latency hiding across the pair)
      if (nt_a > 0) issue_s(0, 0);
      if (has_b) issue_s(1, 0);
      for (int j = 0; j < nkv; ++j) {
        const bool a_on = j < nt_a, b_on = j < nt_b;
        mbar_wait(&v_full[j & 1], (j >> 1) & 1);
        if (a_on) {
          issue_o(0, j);
          if (j + 1 < nt_a) issue_s(0, j + 1);
        }
        if (b_on) {
          issue_o(1, j);
          if (j + 1 < nt_b) issue_s(1, j + 1);
        }
        tc_commit(&v_empty[j & 1]);       // V_j consumed once both PV products finish
        tc_commit(&k_empty[j & 1]);       // K_j consumed by both S products
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    const int g = (warp - 4) / 4;  // 0 = A, 1 = B
    const int ew = (warp - 4) % 4;
    const int qt = qa + g;
    const int ntiles = g == 0 ? nt_a : nt_b;
    if (ntiles > 0) {
      const int r = ew * 32 + lane;
      const uint32_t lane_off = uint32_t(ew * 32) << 16;
      const uint32_t s_col = uint32_t(g * T), o_col = uint32_t(2 * T + g * T);
      constexpr float kSlack = 8.f;
      float m = -FLT_MAX, l = 0.f;
      for (int j = 0; j < ntiles; ++j) {
        const bool diag = j == qt;
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
        uint32_t sv[T];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t* v = sv + c * 32;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(tbase + lane_off + s_col + uint32_t(c * 32)));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[g]);
        float mt = (diag ? row_max<true>(sv, r) : row_max<false>(sv, r)) * p.scale_log2;
        if (j > 0) {  // PV_{j-1} done: P buffer free and O stable
          mbar_wait(&o_full[g], (j - 1) & 1);
          tc_fence_after();
        }
        if (__any_sync(0xffffffffu, mt > m + kSlack)) {
          const float m_new = fmaxf(m, mt);
          const float alpha = ex2(m - m_new);
          if (j > 0) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t v[32];
              tmem_ld_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
              tmem_st_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
            }
            tmem_st_wait();
          }
          l *= alpha;
          m = m_new;
        }
        l += diag ? exp_pack_p<true>(sv, r, p.scale_log2, m)
                  : exp_pack_p<false>(sv, r, p.scale_log2, m);
        // P (bf16 pairs, K-major) over this row's S columns [0, 64)
        tmem_st_32x32b_x32(tbase + lane_off + s_col, *reinterpret_cast<const uint32_t(*)[32]>(sv));
        tmem_st_32x32b_x32(tbase + lane_off + s_col + 32u,
                           *reinterpret_cast<const uint32_t(*)[32]>(sv + 32));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g]);
      }
      mbar_wait(&o_full[g], (ntiles - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      const int qi = qt * T + r;
      __nv_bfloat16* dst = p.out + ((long long)b * p.S + qi) * p.ldo + (long long)h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + o_col + uint32_t(c * 32), v);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          reinterpret_cast<uint4*>(dst)[c * 4 + q] = w;
        }
      }
      p.lse[((long long)b * p.nh + h) * p.S + qi] = m + log2f(l);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------ backward
// CTA = one (sample, head, 128-key tile kt); loops over query tiles i >= kt.
// Transposed formulation so TMEM rows are keys:
//   S^T = K Q_i^T, dP^T = V dO_i^T                    (TMEM, fp32)
//   P^T = exp2(S^T*scale_log2 - lse_q), dS^T = P^T (dP^T - delta_q) * scale
//   dV += P^T dO_i, dK += dS^T Q_i                    (TMEM accumulators)
//   dQ_i  = dS K  -> TMA reduce-add into an fp32 dq accumulator in HBM
// P^T / dS^T share one bf16 smem buffer (K-major over queries); the same smem
// tiles serve as MN-major operands (LBO = one 64-column atom).
struct BwdParams {
  float* dq_acc;
  const float* lse;
  const float* delta;
  __nv_bfloat16* dqkv;
  int S, nh, mb;
  float scale, scale_log2;
};

template <int D>
struct BwdCfg {
  static constexpr uint32_t TILE = T * D * 2;
  static constexpr uint32_t PDS = T * T * 2;
  static constexpr uint32_t SMEM = 1024 + 6 * TILE + PDS + 2 * T * 4 + 256;
};

// P^T of key row kr over query columns [q0, q0 + 64): pk (S^T in, P^T out,
// kept for the dS pass) and the bf16 copy for the dV product; the causal mask
// only on the diagonal tile
template <bool DIAG>
HX_DEVICE void bwd_p_cols(float (&pk)[T / 2], const float* sLse, float scale_log2, int kr, int q0,
                          uint8_t* sPD) {
#pragma unroll
  for (int q8 = 0; q8 < T / 16; ++q8) {
    const float4 la = *reinterpret_cast<const float4*>(sLse + q0 + q8 * 8);
    const float4 lb = *reinterpret_cast<const float4*>(sLse + q0 + q8 * 8 + 4);
    const float ls[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
    float pr[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int qc = q8 * 8 + k;
      const float e = ex2(fmaf(pk[qc], scale_log2, -ls[k]));
      pr[k] = (DIAG && kr > q0 + qc) ? 0.f : e;
      pk[qc] = pr[k];
    }
    uint4 w;
    w.x = pack_bf16x2(pr[0], pr[1]);
    w.y = pack_bf16x2(pr[2], pr[3]);
    w.z = pack_bf16x2(pr[4], pr[5]);
    w.w = pack_bf16x2(pr[6], pr[7]);
    *reinterpret_cast<uint4*>(sPD + kchunk(kr, q0 / 8 + q8)) = w;
  }
}

template <int NATOMS_UNUSED>
HX_DEVICE uint64_t mnview(uint32_t base, int ks) {
  // K-major tile [atom][128 rows][64] read as MN-major: k = rows, mn = columns
  return umma_desc_sw128(base + ks * 2048, ATOM, 1024);
}

constexpr int kBwdThreads = 384;  // warps 0-3: TMA / MMA / TMEM alloc; 4-11: softmax

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  using C = BwdCfg<D>;
  constexpr int DA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sQ = sV + C::TILE;          // [2]
  uint8_t* sDO = sQ + 2 * C::TILE;     // [2]
  uint8_t* sPD = sDO + 2 * C::TILE;    // P^T / dS^T / dQ staging
  float* sLse = reinterpret_cast<float*>(sPD + C::PDS);
  float* sDel = sLse + T;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sDel + T);
  uint64_t* kv_full = bar;
  uint64_t* qdo_full = bar + 1;    // [2]
  uint64_t* qdo_empty = bar + 3;   // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* dp_full = bar + 6;
  uint64_t* p_full = bar + 7;
  uint64_t* pds_free = bar + 8;
  uint64_t* ds_full = bar + 9;
  uint64_t* dq_full = bar + 10;
  uint64_t* dq_empty = bar + 11;
  uint64_t* dkv_full = bar + 12;
  uint64_t* s_read = bar + 13;     // softmax warps hold S_t in registers
  uint64_t* dq_issued = bar + 14;  // [2] softmax warps have issued their dQ_t reduce-adds
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nt = p.S / T;
  // small kt = most query tiles: every head's kt = 0 first (longest-first)
  const int nz = p.mb * p.nh;
  const int kt = int(blockIdx.x / nz);
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int ntiles = nt - kt;
  // TMEM columns: S^T / dQ [0,128) | dP^T [128,256) | dV [256,256+D) | dK [384, 384+D)
  constexpr uint32_t cS = 0, cP = 128, cV = 256, cK = 384;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    tma_prefetch(&tmDQ);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qdo_full[i], 1);
      mbar_init(&qdo_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 8);
    mbar_init(pds_free, 1);
    mbar_init(ds_full, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    mbar_init(dkv_full, 1);
    mbar_init(s_read, 8);
    mbar_init(&dq_issued[0], 8);
    mbar_init(&dq_issued[1], 8);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
      for (int a = 0; a < DA; ++a) {
        tma_load_4d(sK + a * ATOM, &tmK, kv_full, a * 64, kt * T, h, b);
        tma_load_4d(sV + a * ATOM, &tmV, kv_full, a * 64, kt * T, h, b);
      }
      for (int t = 0; t < ntiles; ++t) {
        const int i = kt + t;
        const int slot = t & 1;
        mbar_wait(&qdo_empty[slot], ((t >> 1) & 1) ^ 1);
        // let the dQ reduce-adds of tile t-2 enter the TMA queue ahead of this
        // tile's 2 x TILE loads (they are on the softmax warps' critical path)
        // (one barrier per slot parity: tile t cannot complete before this load,
        // so a barrier is never two phases ahead of its waiter)
        if (t >= 2) mbar_wait(&dq_issued[slot], ((t - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&qdo_full[slot], 2 * C::TILE);
        for (int a = 0; a < DA; ++a) {
          tma_load_4d(sQ + slot * C::TILE + a * ATOM, &tmQ, &qdo_full[slot], a * 64, i * T, h, b);
          tma_load_4d(sDO + slot * C::TILE + a * ATOM, &tmDO, &qdo_full[slot], a * 64, i * T, h, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_sp = idesc_bf16(T, T, 0, 0);   // K-major x K-major, N = 128 queries
      const uint32_t id_acc = idesc_bf16(T, D, 0, 1);  // A K-major, B MN-major, N = D
      const uint32_t id_dq = idesc_bf16(T, D, 1, 1);   // A MN-major (dS view), B MN-major (K view)
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), pd_addr = smem_u32(sPD);
      mbar_wait(kv_full, 0);
      mbar_wait(&qdo_full[0], 0);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ), ks), id_sp, ks > 0 ? 1u : 0u);
      tc_commit(s_full);
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t & 1;
        const uint32_t q_addr = smem_u32(sQ + slot * C::TILE);
        const uint32_t do_addr = smem_u32(sDO + slot * C::TILE);
        mbar_wait(dq_empty, (t & 1) ^ 1);  // dP region: dQ_{t-1} read out
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + cP, kdesc(v_addr, ks), kdesc(do_addr, ks), id_sp, ks > 0 ? 1u : 0u);
        tc_commit(dp_full);
        mbar_wait(p_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cV, kdesc(pd_addr, ks), mnview<0>(do_addr, ks), id_acc,
                     (t > 0 || ks > 0) ? 1u : 0u);
        tc_commit(pds_free);
        if (t + 1 < ntiles) {
          // S_{t+1} as soon as the softmax warps hold S_t in registers: it runs
          // while they compute dS_t
          const int ns = (t + 1) & 1;
          mbar_wait(&qdo_full[ns], ((t + 1) >> 1) & 1);
          mbar_wait(s_read, t & 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ + ns * C::TILE), ks), id_sp,
                       ks > 0 ? 1u : 0u);
          tc_commit(s_full);
        }
        mbar_wait(ds_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cK, kdesc(pd_addr, ks), mnview<0>(q_addr, ks), id_acc,
                     (t > 0 || ks > 0) ? 1u : 0u);
        // dQ_t into the dP region (dP_t consumed by dS_t): S_{t+1} can be issued
        // at once and overlaps the dQ epilogue of the softmax warps
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cP, mnview<0>(pd_addr, ks), mnview<0>(k_addr, ks), id_dq,
                     ks > 0 ? 1u : 0u);
        tc_commit(dq_full);
        tc_commit(&qdo_empty[slot]);
      }
      tc_commit(dkv_full);
    }
  } else if (warp >= 4) {
    // eight softmax warps, two per SM sub-partition: warp (g, ew) owns TMEM
    // lanes 32*ew.. (key rows) and query columns [64g, 64g+64) of P^T / dS^T,
    // then dQ columns [g*D/2, (g+1)*D/2)
    const int g = (warp - 4) / 4;
    const int ew = (warp - 4) % 4;
    const int tid = threadIdx.x - 128;          // 0..255
    const int kr = ew * 32 + lane;              // key row within the tile (TMEM lane)
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const int q0 = g * (T / 2);                 // first query column of this warp
    uint8_t* stage = sPD + (warp - 4) * 4096;   // dQ staging: [32 rows][32 fp32] per warp
    const long long z0 = ((long long)b * p.nh + h) * p.S + (long long)kt * T;
    const float* stat_src = tid < T ? p.lse : p.delta;
    float* stat_dst = tid < T ? sLse : sDel;
    const int si = tid % T;
    float nstat = stat_src[z0 + si];            // prefetched statistic (lse or delta)
    for (int t = 0; t < ntiles; ++t) {
      const int i = kt + t;
      const bool diag = t == 0;
      const long long zq = ((long long)b * p.nh + h) * p.S + (long long)i * T;
      // this warp's dQ reduce of tile t-1 must have read its staging area (the
      // staging areas overlap other warps' P rows) before anyone writes P_t
      if (lane == 0) bulk_wait_read<0>();
      // per-query statistics of this tile, shared by the eight warps
      asm volatile("bar.sync 1, 256;" ::: "memory");
      stat_dst[si] = nstat;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (t + 1 < ntiles) nstat = stat_src[zq + T + si];
      // P^T (64 query columns), kept in registers for the dS pass
      mbar_wait(s_full, t & 1);
      tc_fence_after();
      uint32_t pu[T / 2];
#pragma unroll
      for (int c = 0; c < 2; ++c)
        tmem_ld_32x32b_x32(tbase + lane_off + cS + uint32_t(q0 + c * 32),
                           *reinterpret_cast<uint32_t(*)[32]>(pu + c * 32));
      tmem_ld_wait();
      float pk[T / 2];
#pragma unroll
      for (int k = 0; k < T / 2; ++k) pk[k] = __uint_as_float(pu[k]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_read);  // S region may take S_{t+1} now
      if (diag)
        bwd_p_cols<true>(pk, sLse, p.scale_log2, kr, q0, sPD);
      else
        bwd_p_cols<false>(pk, sLse, p.scale_log2, kr, q0, sPD);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dS^T (after dV has consumed P^T)
      mbar_wait(dp_full, t & 1);
      mbar_wait(pds_free, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(q0 + c * 32), dv);
        tmem_ld_wait();
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          float ds[8];
          const float4 da = *reinterpret_cast<const float4*>(sDel + q0 + c * 32 + q8 * 8);
          const float4 db = *reinterpret_cast<const float4*>(sDel + q0 + c * 32 + q8 * 8 + 4);
          const float dl[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ds[k] = pk[c * 32 + q8 * 8 + k] * (__uint_as_float(dv[q8 * 8 + k]) - dl[k]) * p.scale;
          uint4 w;
          w.x = pack_bf16x2(ds[0], ds[1]);
          w.y = pack_bf16x2(ds[2], ds[3]);
          w.z = pack_bf16x2(ds[4], ds[5]);
          w.w = pack_bf16x2(ds[6], ds[7]);
          *reinterpret_cast<uint4*>(sPD + kchunk(kr, q0 / 8 + c * 4 + q8)) = w;
        }
      }
      tc_fence_before();
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      // dQ_i partial (TMEM rows = queries) -> staged fp32 -> TMA reduce-add;
      // this warp: D/2 columns in 32-column chunks through a 4 KB stage
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      const int qrow = i * T + ew * 32;  // first query row of this warp's slab
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        const int col = g * (D / 2) + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(col), v);
        tmem_ld_wait();
        if (c > 0) {
          if (lane == 0) bulk_wait_read<0>();  // stage reused by the next chunk
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stage + swz128(lane, q)) =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                          __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_4d(&tmDQ, stage, h * D + col, b * p.S + qrow, 0, 0);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(dq_empty);
        mbar_arrive(&dq_issued[t & 1]);
      }
    }
    if (lane == 0) bulk_wait_all();
    // dK, dV of this key tile -> bf16 into the dqkv buffer (this warp: D/2 columns)
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long row = (long long)b * p.S + kt * T + kr;
    __nv_bfloat16* dst = p.dqkv + row * (3LL * p.nh * D) + (long long)h * 3 * D;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t col0 = part == 0 ? cK : cV;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        const int col = g * (D / 2) + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + col0 + uint32_t(col), v);
        tmem_ld_wait();
        float f[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) f[k] = __uint_as_float(v[k]);
        uint4* o = reinterpret_cast<uint4*>(dst + (part + 1) * D + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(f[8 * q + 0], f[8 * q + 1]);
          w.y = pack_bf16x2(f[8 * q + 2], f[8 * q + 3]);
          w.z = pack_bf16x2(f[8 * q + 4], f[8 * q + 5]);
          w.w = pack_bf16x2(f[8 * q + 6], f[8 * q + 7]);
          o[q] = w;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------ backward, v2
// Same transposed formulation as attn_bwd_kernel; the dQ epilogue moves to its
// own warpgroup so the softmax warps start the next query tile while dQ_t
// streams out (in v1 the eight softmax warps also read dQ_t out of TMEM, staged
// it through the P / dS buffer and issued its TMA reduce-adds -- a serial step
// of every tile):
//   warps 0-3   TMA producer (w0), MMA issuer (w1), TMEM allocator (w2)
//   warps 4-11  P^T, dS^T of each query tile (P values computed in registers
//               while dK_{t-1} / dQ_{t-1} still read the shared P / dS buffer)
//   warps 12-15 dQ_t: TMEM -> registers -> swizzled smem (two 4 KB buffers per
//               warp) -> TMA reduce-add into the fp32 dq accumulator; the dP
//               region (which holds dQ_t) is released after the TMEM loads
// dO is single-buffered: its slot frees once dP_t and dV_t have read it, long
// before dP_{t+1} needs the next tile; that pays for the 32 KB of dQ staging.
// Registers: 128 per thread for every role (512 threads); the softmax warps
// stream S / dP in 32-column chunks and keep P as bf16 pairs (32 registers),
// so they fit without spills; P is computed while dK_{t-1} / dQ_{t-1} still
// read the P / dS buffer and dS is formed from the same bf16 P.
constexpr int kBwd2Threads = 512;

template <int D>
struct Bwd2Cfg {
  static constexpr uint32_t TILE = T * D * 2;
  static constexpr uint32_t PDS = T * T * 2;
  static constexpr uint32_t STG = 4 * 2 * 4096;  // 4 warps x 2 x [32 rows][32 fp32]
  static constexpr uint32_t SMEM = 1024 + 5 * TILE + PDS + STG + 2 * T * 4 + 256;
};

template <int D>
__global__ void __launch_bounds__(kBwd2Threads, 1)
    attn_bwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  using C = Bwd2Cfg<D>;
  constexpr int DA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sQ = sV + C::TILE;        // [2]
  uint8_t* sDO = sQ + 2 * C::TILE;   // [1]
  uint8_t* sPD = sDO + C::TILE;      // P^T / dS^T
  uint8_t* sStg = sPD + C::PDS;      // dQ staging
  float* sLse = reinterpret_cast<float*>(sStg + C::STG);
  float* sDel = sLse + T;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sDel + T);
  uint64_t* kv_full = bar;
  uint64_t* q_full = bar + 1;    // [2]
  uint64_t* q_empty = bar + 3;   // [2] Q_t read by S_t and dK_t
  uint64_t* do_full = bar + 5;
  uint64_t* do_empty = bar + 6;  // dO_t read by dP_t and dV_t
  uint64_t* s_full = bar + 7;
  uint64_t* s_read = bar + 8;    // softmax warps hold S_t in registers
  uint64_t* dp_full = bar + 9;
  uint64_t* p_full = bar + 10;
  uint64_t* pds_free = bar + 11;  // dV_t has read P_t: dS_t may overwrite it
  uint64_t* ds_full = bar + 12;
  uint64_t* pd_free = bar + 13;   // dK_t, dQ_t have read dS_t: P_{t+1} may overwrite it
  uint64_t* dq_full = bar + 14;
  uint64_t* dq_empty = bar + 15;  // dQ_t loaded out of TMEM: dP_{t+1} may overwrite it
  uint64_t* dkv_full = bar + 16;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nt = p.S / T;
  const int nz = p.mb * p.nh;
  const int kt = int(blockIdx.x / nz);  // small kt = most query tiles first
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int ntiles = nt - kt;
  constexpr uint32_t cS = 0, cP = 128, cV = 256, cK = 384;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    tma_prefetch(&tmDQ);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(s_read, 8);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 8);
    mbar_init(pds_free, 1);
    mbar_init(ds_full, 8);
    mbar_init(pd_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(dkv_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp < 4) {
    if (warp == 0 && lane == 0) {
      auto load_q = [&](int t) {
        const int slot = t & 1;
        mbar_wait(&q_empty[slot], ((t >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[slot], C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sQ + slot * C::TILE + a * ATOM, &tmQ, &q_full[slot], a * 64, (kt + t) * T, h, b);
      };
      auto load_do = [&](int t) {
        mbar_wait(do_empty, (t & 1) ^ 1);
        mbar_arrive_expect_tx(do_full, C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sDO + a * ATOM, &tmDO, do_full, a * 64, (kt + t) * T, h, b);
      };
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
      for (int a = 0; a < DA; ++a) {
        tma_load_4d(sK + a * ATOM, &tmK, kv_full, a * 64, kt * T, h, b);
        tma_load_4d(sV + a * ATOM, &tmV, kv_full, a * 64, kt * T, h, b);
      }
      load_q(0);
      load_do(0);
      if (ntiles > 1) load_q(1);
      for (int t = 1; t < ntiles; ++t) {
        load_do(t);                       // after dV_{t-1}
        if (t + 1 < ntiles) load_q(t + 1);  // after dK_{t-1}
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t id_sp = idesc_bf16(T, T, 0, 0);   // K-major x K-major, N = 128 queries
      const uint32_t id_acc = idesc_bf16(T, D, 0, 1);  // A K-major, B MN-major, N = D
      const uint32_t id_dq = idesc_bf16(T, D, 1, 1);   // A MN-major (dS view), B MN-major (K view)
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), pd_addr = smem_u32(sPD);
      const uint32_t do_addr = smem_u32(sDO);
      mbar_wait(kv_full, 0);
      mbar_wait(&q_full[0], 0);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ), ks), id_sp, ks > 0 ? 1u : 0u);
      tc_commit(s_full);
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t & 1;
        const uint32_t q_addr = smem_u32(sQ + slot * C::TILE);
        mbar_wait(do_full, t & 1);
        mbar_wait(dq_empty, (t & 1) ^ 1);  // dQ_{t-1} loaded out of the dP region
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + cP, kdesc(v_addr, ks), kdesc(do_addr, ks), id_sp, ks > 0 ? 1u : 0u);
        tc_commit(dp_full);
        mbar_wait(p_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cV, kdesc(pd_addr, ks), mnview<0>(do_addr, ks), id_acc,
                     (t > 0 || ks > 0) ? 1u : 0u);
        tc_commit(pds_free);
        tc_commit(do_empty);
        if (t + 1 < ntiles) {
          const int ns = (t + 1) & 1;
          mbar_wait(&q_full[ns], ((t + 1) >> 1) & 1);
          mbar_wait(s_read, t & 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ + ns * C::TILE), ks), id_sp,
                       ks > 0 ? 1u : 0u);
          tc_commit(s_full);
        }
        mbar_wait(ds_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cK, kdesc(pd_addr, ks), mnview<0>(q_addr, ks), id_acc,
                     (t > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cP, mnview<0>(pd_addr, ks), mnview<0>(k_addr, ks), id_dq,
                     ks > 0 ? 1u : 0u);
        tc_commit(dq_full);
        tc_commit(&q_empty[slot]);
        tc_commit(pd_free);
      }
      tc_commit(dkv_full);
    }
  } else if (warp < 12) {
    const int g = (warp - 4) / 4;
    const int ew = (warp - 4) % 4;
    const int tid = threadIdx.x - 128;          // 0..255
    const int kr = ew * 32 + lane;              // key row within the tile (TMEM lane)
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const int q0 = g * (T / 2);
    const long long z0 = ((long long)b * p.nh + h) * p.S + (long long)kt * T;
    const float* stat_src = tid < T ? p.lse : p.delta;
    float* stat_dst = tid < T ? sLse : sDel;
    const int si = tid % T;
    float nstat = stat_src[z0 + si];
    for (int t = 0; t < ntiles; ++t) {
      const int i = kt + t;
      const bool diag = t == 0;
      const long long zq = ((long long)b * p.nh + h) * p.S + (long long)i * T;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      sts_f32(stat_dst + si, nstat);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (t + 1 < ntiles) nstat = stat_src[zq + T + si];
      // P^T = exp2(S^T * scale_log2 - lse_q) (causal mask on the diagonal
      // tile), 32 query columns at a time straight into the P / dS buffer once
      // dK / dQ of the previous tile have read it; S_{t+1} may then overwrite
      // the S region.  Register budget: 128 per thread (512-thread CTA).
      mbar_wait(s_full, t & 1);
      tc_fence_after();
      uint32_t pp[T / 4];  // this thread's 64 P values, bf16 pairs
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t su[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cS + uint32_t(q0 + c * 32), su);
        tmem_ld_wait();
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const int qb = q0 + c * 32 + q8 * 8;
          const float4 la = lds_f4(sLse + qb);
          const float4 lb = lds_f4(sLse + qb + 4);
          const float ls[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
          float pr[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float e = ex2(fmaf(__uint_as_float(su[q8 * 8 + k]), p.scale_log2, -ls[k]));
            pr[k] = (diag && kr > qb + k) ? 0.f : e;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) pp[c * 16 + q8 * 4 + k] = pack_bf16x2(pr[2 * k], pr[2 * k + 1]);
        }
      }
      // the S region may take S_{t+1}; the P / dS buffer once dK_{t-1} and
      // dQ_{t-1} have read dS_{t-1} (the P math above overlapped those MMAs)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_read);
      if (t > 0) mbar_wait(pd_free, (t - 1) & 1);
#pragma unroll
      for (int q8 = 0; q8 < 8; ++q8)
        sts_u4(sPD + kchunk(kr, q0 / 8 + q8),
               make_uint4(pp[q8 * 4], pp[q8 * 4 + 1], pp[q8 * 4 + 2], pp[q8 * 4 + 3]));
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dS^T = P^T (dP^T - delta_q) * scale from the bf16 P^T kept in
      // registers, into the buffer after dV has consumed P^T
      mbar_wait(dp_full, t & 1);
      mbar_wait(pds_free, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(q0 + c * 32), dv);
        tmem_ld_wait();
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const int qb = q0 + c * 32 + q8 * 8;
          uint8_t* cell = sPD + kchunk(kr, qb / 8);
          const uint32_t* pu4 = pp + c * 16 + q8 * 4;
          const float4 da = lds_f4(sDel + qb);
          const float4 db = lds_f4(sDel + qb + 4);
          const float dl[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
          float ds[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t u = pu4[k / 2];
            const float pv = __uint_as_float((k & 1) ? (u & 0xffff0000u) : (u << 16));
            ds[k] = pv * (__uint_as_float(dv[q8 * 8 + k]) - dl[k]) * p.scale;
          }
          uint4 w;
          w.x = pack_bf16x2(ds[0], ds[1]);
          w.y = pack_bf16x2(ds[2], ds[3]);
          w.z = pack_bf16x2(ds[4], ds[5]);
          w.w = pack_bf16x2(ds[6], ds[7]);
          sts_u4(cell, w);
        }
      }
      tc_fence_before();
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    // dK, dV of this key tile -> bf16 into the dqkv buffer (this warp: D/2 columns)
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long row = (long long)b * p.S + kt * T + kr;
    __nv_bfloat16* dst = p.dqkv + row * (3LL * p.nh * D) + (long long)h * 3 * D;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t col0 = part == 0 ? cK : cV;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        const int col = g * (D / 2) + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + col0 + uint32_t(col), v);
        tmem_ld_wait();
        uint4* o = reinterpret_cast<uint4*>(dst + (part + 1) * D + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
          w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
          w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
          w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
          o[q] = w;
        }
      }
    }
  } else {
    // dQ epilogue warps: warp 12 + e reads TMEM lanes [32e, 32e + 32) = query rows
    const int ew = warp - 12;
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    uint8_t* base = sStg + ew * 8192;
    int chunk = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int qrow = (kt + t) * T + ew * 32;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c, ++chunk) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(c * 32), v);
        tmem_ld_wait();
        if (c == D / 32 - 1) {  // dQ_t is out of TMEM: the dP region is free
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_empty);
        }
        uint8_t* stg = base + (chunk & 1) * 4096;
        if (chunk >= 2) {
          if (lane == 0) bulk_wait_read<1>();  // this buffer's reduce-add (two chunks ago) has read it
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts_f4(stg + swz128(lane, q),
                 make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_4d(&tmDQ, stg, h * D + c * 32, b * p.S + qrow, 0, 0);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------ backward, v3
// v2 with P^T kept in tensor memory: the softmax warps write P^T (bf16 pairs)
// over the S^T columns they have just read (tcgen05.st), and dV_t = P^T dO_t
// reads its A operand from TMEM.  The shared P / dS buffer then holds only
// dS^T, so dS_t no longer waits for dV_t to finish reading P_t, and P_t no
// longer goes through shared memory.  S_{t+1} is issued once dV_t has
// completed (its commit), since it overwrites the P^T columns.
constexpr int kBwd3Threads = 512;

template <int D>
struct Bwd3Cfg {
  static constexpr uint32_t TILE = T * D * 2;
  static constexpr uint32_t PDS = T * T * 2;
  static constexpr uint32_t STG = 4 * 2 * 4096;  // 4 warps x 2 x [32 rows][32 fp32]
  static constexpr uint32_t SMEM = 1024 + 5 * TILE + PDS + STG + 2 * T * 4 + 256;
};

template <int D>
__global__ void __launch_bounds__(kBwd3Threads, 1)
    attn_bwd3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  using C = Bwd3Cfg<D>;
  constexpr int DA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sQ = sV + C::TILE;        // [2]
  uint8_t* sDO = sQ + 2 * C::TILE;   // [1]
  uint8_t* sPD = sDO + C::TILE;      // P^T / dS^T
  uint8_t* sStg = sPD + C::PDS;      // dQ staging
  float* sLse = reinterpret_cast<float*>(sStg + C::STG);
  float* sDel = sLse + T;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sDel + T);
  uint64_t* kv_full = bar;
  uint64_t* q_full = bar + 1;    // [2]
  uint64_t* q_empty = bar + 3;   // [2] Q_t read by S_t and dK_t
  uint64_t* do_full = bar + 5;
  uint64_t* do_empty = bar + 6;  // dO_t read by dP_t and dV_t
  uint64_t* s_full = bar + 7;
  uint64_t* s_read = bar + 8;    // (unused in v3)
  uint64_t* dp_full = bar + 9;
  uint64_t* p_full = bar + 10;
  uint64_t* pds_free = bar + 11;  // dV_t done: S_{t+1} may overwrite the P^T columns
  uint64_t* ds_full = bar + 12;
  uint64_t* pd_free = bar + 13;   // dK_t, dQ_t have read dS_t: P_{t+1} may overwrite it
  uint64_t* dq_full = bar + 14;
  uint64_t* dq_empty = bar + 15;  // dQ_t loaded out of TMEM: dP_{t+1} may overwrite it
  uint64_t* dkv_full = bar + 16;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int nt = p.S / T;
  const int nz = p.mb * p.nh;
  const int kt = int(blockIdx.x / nz);  // small kt = most query tiles first
  const int zh = int(blockIdx.x % nz);
  const int h = zh % p.nh;
  const int b = zh / p.nh;
  const int ntiles = nt - kt;
  constexpr uint32_t cS = 0, cP = 128, cV = 256, cK = 384;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    tma_prefetch(&tmDQ);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(s_read, 8);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 8);
    mbar_init(pds_free, 1);
    mbar_init(ds_full, 8);
    mbar_init(pd_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(dkv_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp < 4) {
    if (warp == 0 && lane == 0) {
      auto load_q = [&](int t) {
        const int slot = t & 1;
        mbar_wait(&q_empty[slot], ((t >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[slot], C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sQ + slot * C::TILE + a * ATOM, &tmQ, &q_full[slot], a * 64, (kt + t) * T, h, b);
      };
      auto load_do = [&](int t) {
        mbar_wait(do_empty, (t & 1) ^ 1);
        mbar_arrive_expect_tx(do_full, C::TILE);
        for (int a = 0; a < DA; ++a)
          tma_load_4d(sDO + a * ATOM, &tmDO, do_full, a * 64, (kt + t) * T, h, b);
      };
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
      for (int a = 0; a < DA; ++a) {
        tma_load_4d(sK + a * ATOM, &tmK, kv_full, a * 64, kt * T, h, b);
        tma_load_4d(sV + a * ATOM, &tmV, kv_full, a * 64, kt * T, h, b);
      }
      load_q(0);
      load_do(0);
      if (ntiles > 1) load_q(1);
      for (int t = 1; t < ntiles; ++t) {
        load_do(t);                       // after dV_{t-1}
        if (t + 1 < ntiles) load_q(t + 1);  // after dK_{t-1}
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t id_sp = idesc_bf16(T, T, 0, 0);   // K-major x K-major, N = 128 queries
      const uint32_t id_acc = idesc_bf16(T, D, 0, 1);  // A K-major, B MN-major, N = D
      const uint32_t id_dq = idesc_bf16(T, D, 1, 1);   // A MN-major (dS view), B MN-major (K view)
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), pd_addr = smem_u32(sPD);
      const uint32_t do_addr = smem_u32(sDO);
      mbar_wait(kv_full, 0);
      mbar_wait(&q_full[0], 0);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ), ks), id_sp, ks > 0 ? 1u : 0u);
      tc_commit(s_full);
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t & 1;
        const uint32_t q_addr = smem_u32(sQ + slot * C::TILE);
        mbar_wait(do_full, t & 1);
        mbar_wait(dq_empty, (t & 1) ^ 1);  // dQ_{t-1} loaded out of the dP region
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc_mma_f16(tbase + cP, kdesc(v_addr, ks), kdesc(do_addr, ks), id_sp, ks > 0 ? 1u : 0u);
        tc_commit(dp_full);
        mbar_wait(p_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16_ts(tbase + cV, tbase + cS + uint32_t(ks * 8), mnview<0>(do_addr, ks), id_acc,
                        (t > 0 || ks > 0) ? 1u : 0u);
        tc_commit(pds_free);  // dV_t done: the P^T columns may take S_{t+1}
        tc_commit(do_empty);
        if (t + 1 < ntiles) {
          const int ns = (t + 1) & 1;
          mbar_wait(&q_full[ns], ((t + 1) >> 1) & 1);
          mbar_wait(pds_free, t & 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            tc_mma_f16(tbase + cS, kdesc(k_addr, ks), kdesc(smem_u32(sQ + ns * C::TILE), ks), id_sp,
                       ks > 0 ? 1u : 0u);
          tc_commit(s_full);
        }
        mbar_wait(ds_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cK, kdesc(pd_addr, ks), mnview<0>(q_addr, ks), id_acc,
                     (t > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < T / 16; ++ks)
          tc_mma_f16(tbase + cP, mnview<0>(pd_addr, ks), mnview<0>(k_addr, ks), id_dq,
                     ks > 0 ? 1u : 0u);
        tc_commit(dq_full);
        tc_commit(&q_empty[slot]);
        tc_commit(pd_free);
      }
      tc_commit(dkv_full);
    }
  } else if (warp < 12) {
    const int g = (warp - 4) / 4;
    const int ew = (warp - 4) % 4;
    const int tid = threadIdx.x - 128;          // 0..255
    const int kr = ew * 32 + lane;              // key row within the tile (TMEM lane)
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    const int q0 = g * (T / 2);
    const long long z0 = ((long long)b * p.nh + h) * p.S + (long long)kt * T;
    const float* stat_src = tid < T ? p.lse : p.delta;
    float* stat_dst = tid < T ? sLse : sDel;
    const int si = tid % T;
    float nstat = stat_src[z0 + si];
    for (int t = 0; t < ntiles; ++t) {
      const int i = kt + t;
      const bool diag = t == 0;
      const long long zq = ((long long)b * p.nh + h) * p.S + (long long)i * T;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      sts_f32(stat_dst + si, nstat);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (t + 1 < ntiles) nstat = stat_src[zq + T + si];
      // P^T = exp2(S^T * scale_log2 - lse_q) (causal mask on the diagonal
      // tile), 32 query columns at a time straight into the P / dS buffer once
      // dK / dQ of the previous tile have read it; S_{t+1} may then overwrite
      // the S region.  Register budget: 128 per thread (512-thread CTA).
      mbar_wait(s_full, t & 1);
      tc_fence_after();
      uint32_t pp[T / 4];  // this thread's 64 P values, bf16 pairs
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t su[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cS + uint32_t(q0 + c * 32), su);
        tmem_ld_wait();
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const int qb = q0 + c * 32 + q8 * 8;
          const float4 la = lds_f4(sLse + qb);
          const float4 lb = lds_f4(sLse + qb + 4);
          const float ls[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
          float pr[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float e = ex2(fmaf(__uint_as_float(su[q8 * 8 + k]), p.scale_log2, -ls[k]));
            pr[k] = (diag && kr > qb + k) ? 0.f : e;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) pp[c * 16 + q8 * 4 + k] = pack_bf16x2(pr[2 * k], pr[2 * k + 1]);
        }
      }
      // P^T (bf16 pairs, K-major: packed column j = queries 2j, 2j + 1) over
      // the S^T columns [0, 64) once all eight warps have read their S^T
      asm volatile("bar.sync 2, 256;" ::: "memory");
      tmem_st_32x32b_x32(tbase + lane_off + cS + uint32_t(q0 / 2), pp);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dS^T = P^T (dP^T - delta_q) * scale from the bf16 P^T kept in
      // registers, into the (dS-only) buffer once dK_{t-1} / dQ_{t-1} read it
      mbar_wait(dp_full, t & 1);
      if (t > 0) mbar_wait(pd_free, (t - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(q0 + c * 32), dv);
        tmem_ld_wait();
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const int qb = q0 + c * 32 + q8 * 8;
          uint8_t* cell = sPD + kchunk(kr, qb / 8);
          const uint32_t* pu4 = pp + c * 16 + q8 * 4;
          const float4 da = lds_f4(sDel + qb);
          const float4 db = lds_f4(sDel + qb + 4);
          const float dl[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
          float ds[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t u = pu4[k / 2];
            const float pv = __uint_as_float((k & 1) ? (u & 0xffff0000u) : (u << 16));
            ds[k] = pv * (__uint_as_float(dv[q8 * 8 + k]) - dl[k]) * p.scale;
          }
          uint4 w;
          w.x = pack_bf16x2(ds[0], ds[1]);
          w.y = pack_bf16x2(ds[2], ds[3]);
          w.z = pack_bf16x2(ds[4], ds[5]);
          w.w = pack_bf16x2(ds[6], ds[7]);
          sts_u4(cell, w);
        }
      }
      tc_fence_before();
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    // dK, dV of this key tile -> bf16 into the dqkv buffer (this warp: D/2 columns)
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long row = (long long)b * p.S + kt * T + kr;
    __nv_bfloat16* dst = p.dqkv + row * (3LL * p.nh * D) + (long long)h * 3 * D;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t col0 = part == 0 ? cK : cV;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        const int col = g * (D / 2) + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + col0 + uint32_t(col), v);
        tmem_ld_wait();
        uint4* o = reinterpret_cast<uint4*>(dst + (part + 1) * D + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
          w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
          w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
          w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
          o[q] = w;
        }
      }
    }
  } else {
    // dQ epilogue warps: warp 12 + e reads TMEM lanes [32e, 32e + 32) = query rows
    const int ew = warp - 12;
    const uint32_t lane_off = uint32_t(ew * 32) << 16;
    uint8_t* base = sStg + ew * 8192;
    int chunk = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int qrow = (kt + t) * T + ew * 32;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c, ++chunk) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_off + cP + uint32_t(c * 32), v);
        tmem_ld_wait();
        if (c == D / 32 - 1) {  // dQ_t is out of TMEM: the dP region is free
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_empty);
        }
        uint8_t* stg = base + (chunk & 1) * 4096;
        if (chunk >= 2) {
          if (lane == 0) bulk_wait_read<1>();  // this buffer's reduce-add (two chunks ago) has read it
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts_f4(stg + swz128(lane, q),
                 make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_4d(&tmDQ, stg, h * D + c * 32, b * p.S + qrow, 0, 0);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// delta[z][q] = sum_e dO[q, e] * O[q, e]: D/8 consecutive threads per (row,
// head), 16-byte coalesced loads of O and dO, shuffle reduction; the same
// pass zeroes the fp32 dq accumulator (same [M, nh*D] layout) for the
// backward's TMA reduce-adds (no separate memset)
template <int D>
__global__ void attn_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                  const __nv_bfloat16* __restrict__ dout, float* delta,
                                  float* __restrict__ dq_zero, int S, int nh, int mb) {
  constexpr int G = D / 8;  // threads per (row, head): 16 (d 128) or 8 (d 64)
  const long long n = (long long)mb * S * nh * G;
  const int sub = threadIdx.x % G;
  // warp-uniform trip count (the shuffles need every lane of the warp)
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx - threadIdx.x % 32 < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long rh = idx / G;  // row * nh + h
    float acc = 0.f;
    if (idx < n) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(o + rh * D) + sub);
      const uint4 g = __ldcs(reinterpret_cast<const uint4*>(dout + rh * D) + sub);
      // the fp32 dq accumulator has O's layout: zero this thread's 8 elements
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(dq_zero + rh * D)[2 * sub] = z;
      reinterpret_cast<float4*>(dq_zero + rh * D)[2 * sub + 1] = z;
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* pg = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        acc += __low2float(pa[k]) * __low2float(pg[k]) + __high2float(pa[k]) * __high2float(pg[k]);
    }
#pragma unroll
    for (int w = G / 2; w > 0; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
    if (sub == 0 && idx < n) {
      const int h = int(rh % nh);
      const long long row = rh / nh;  // b*S + s
      const int bb = int(row / S), s = int(row % S);
      delta[((long long)bb * nh + h) * S + s] = acc;
    }
  }
}

// dq (fp32 accumulator [M, nh*D]) -> bf16 q slots of dqkv [M, nh*3*D]
template <int D>
__global__ void attn_dq_cast_kernel(const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv,
                                    long long M, int nh) {
  const long long n = M * nh * (D / 8);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = int(idx % (D / 8));
    const long long t = idx / (D / 8);
    const int h = int(t % nh);
    const long long row = t / nh;
    const float4* src = reinterpret_cast<const float4*>(dq + row * nh * D + h * D + c * 8);
    float4 a = src[0], bq = src[1];
    uint4 w;
    w.x = pack_bf16x2(a.x, a.y);
    w.y = pack_bf16x2(a.z, a.w);
    w.z = pack_bf16x2(bq.x, bq.y);
    w.w = pack_bf16x2(bq.z, bq.w);
    *reinterpret_cast<uint4*>(dqkv + row * 3LL * nh * D + (long long)h * 3 * D + c * 8) = w;
  }
}

// dq cast fused with the RoPE backward (inverse rotation) of dq and dk: thread
// per (row, head, 8 rotation pairs).  dq is rounded to bf16 first and dk read
// as bf16, exactly the values the standalone rope kernel would rotate; (cos,
// sin) from the forward epilogue's table tab[pos][D/2], sin negated.
__device__ __forceinline__ void bf16x8_to_f32(uint4 w, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __low2float(h[k]);
    f[2 * k + 1] = __high2float(h[k]);
  }
}
__device__ __forceinline__ uint4 f32x8_to_bf16(const float* f) {
  uint4 w;
  w.x = pack_bf16x2(f[0], f[1]);
  w.y = pack_bf16x2(f[2], f[3]);
  w.z = pack_bf16x2(f[4], f[5]);
  w.w = pack_bf16x2(f[6], f[7]);
  return w;
}
template <int D>
__global__ void attn_dq_cast_rope_kernel(const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv,
                                         const float2* __restrict__ tab, long long M, int S, int nh) {
  constexpr int half = D / 2, g8 = half / 8;
  const long long n = M * nh * g8;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = int(idx % g8);
    const long long t = idx / g8;
    const int h = int(t % nh);
    const long long row = t / nh;
    const float4* tp = reinterpret_cast<const float4*>(tab + (row % S) * half + c * 8);
    float cs[8], sn[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = __ldg(tp + k);
      cs[2 * k] = v.x;
      sn[2 * k] = -v.y;
      cs[2 * k + 1] = v.z;
      sn[2 * k + 1] = -v.w;
    }
    const float* src = dq + row * nh * D + h * D + c * 8;
    __nv_bfloat16* qb = dqkv + row * 3LL * nh * D + (long long)h * 3 * D + c * 8;
    __nv_bfloat16* kb = qb + D;
    float qa[8], qh[8], ka[8], kh[8];
    {
      const float4 a0 = reinterpret_cast<const float4*>(src)[0], a1 = reinterpret_cast<const float4*>(src)[1];
      const float4 b0 = reinterpret_cast<const float4*>(src + half)[0];
      const float4 b1 = reinterpret_cast<const float4*>(src + half)[1];
      const float fa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float fb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        qa[k] = __bfloat162float(__float2bfloat16(fa[k]));
        qh[k] = __bfloat162float(__float2bfloat16(fb[k]));
      }
    }
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(kb), ka);
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(kb + half), kh);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // explicit rounding, as rope_kernel
      float x = qa[k], y = qh[k];
      qa[k] = __fsub_rn(__fmul_rn(x, cs[k]), __fmul_rn(y, sn[k]));
      qh[k] = __fadd_rn(__fmul_rn(y, cs[k]), __fmul_rn(x, sn[k]));
      x = ka[k];
      y = kh[k];
      ka[k] = __fsub_rn(__fmul_rn(x, cs[k]), __fmul_rn(y, sn[k]));
      kh[k] = __fadd_rn(__fmul_rn(y, cs[k]), __fmul_rn(x, sn[k]));
    }
    *reinterpret_cast<uint4*>(qb) = f32x8_to_bf16(qa);
    *reinterpret_cast<uint4*>(qb + half) = f32x8_to_bf16(qh);
    *reinterpret_cast<uint4*>(kb) = f32x8_to_bf16(ka);
    *reinterpret_cast<uint4*>(kb + half) = f32x8_to_bf16(kh);
  }
}

// ------------------------------------------------------------------ host
// 3 = two query tiles per CTA with P in TMEM (default), 2 = the same with P
// through shared memory, 1 = one tile per CTA
int g_fwd_variant = 3;
// 3 = P^T in TMEM + dQ epilogue warpgroup, 2 = dQ epilogue warpgroup,
// 1 = softmax warps stream dQ (r01)
int g_bwd_variant = 3;
PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
std::once_flag g_enc_once;

// 4D bf16 map: element (e, s, h, b) at base + (b*S + s)*row_stride + h*head_stride + e
bool encode(CUtensorMap* map, const void* base, int d, int S, int nh, int mb, long long row_stride,
            long long head_stride, uint32_t box0, uint32_t box1) {
  std::call_once(g_enc_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(d), cuuint64_t(S), cuuint64_t(nh), cuuint64_t(mb)};
  cuuint64_t strides[3] = {cuuint64_t(row_stride * 2), cuuint64_t(head_stride * 2),
                           cuuint64_t(row_stride * 2 * S)};
  cuuint32_t box[4] = {box0, box1, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 [rows, cols] map, box 32 x 32, SWIZZLE_128B (dq accumulator, TMA reduce-add)
bool encode_f32(CUtensorMap* map, float* base, long long cols, long long rows) {
  cuuint64_t dims[4] = {cuuint64_t(cols), cuuint64_t(rows), 1, 1};
  cuuint64_t strides[3] = {cuuint64_t(cols * 4), cuuint64_t(cols * 4 * rows),
                           cuuint64_t(cols * 4 * rows)};
  cuuint32_t box[4] = {32, 32, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_fwd(const AttnDesc& a, cudaStream_t s) {
  using C = FwdCfg<D>;
  using C2 = Fwd2Cfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_fwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(C2::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_fwd3_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Fwd3Cfg<D>::SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long W = 3LL * a.nh * D;
  CUtensorMap q, k, v;
  if (!encode(&q, a.qkv, D, a.S, a.nh, a.mb, W, 3 * D, 64, T) ||
      !encode(&k, a.qkv + D, D, a.S, a.nh, a.mb, W, 3 * D, 64, T) ||
      !encode(&v, a.qkv + 2 * D, D, a.S, a.nh, a.mb, W, 3 * D, 64, 64))
    return cudaErrorInvalidValue;
  AttnParams p;
  p.out = a.out;
  p.lse = a.lse;
  p.S = a.S;
  p.nh = a.nh;
  p.mb = a.mb;
  p.ldo = a.nh * D;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  if (g_fwd_variant == 3) {
    const int grid = ((a.S / T + 1) / 2) * a.nh * a.mb;
    attn_fwd3_kernel<D><<<grid, kThreads2, Fwd3Cfg<D>::SMEM, s>>>(q, k, v, p);
  } else if (g_fwd_variant == 2) {
    const int grid = ((a.S / T + 1) / 2) * a.nh * a.mb;
    attn_fwd2_kernel<D><<<grid, kThreads2, C2::SMEM, s>>>(q, k, v, p);
  } else {
    const int grid = (a.S / T) * a.nh * a.mb;
    attn_fwd_kernel<D><<<grid, kThreads, C::SMEM, s>>>(q, k, v, p);
  }
  return cudaGetLastError();
}

int ew_blocks(long long n) {
  long long b = (n + 255) / 256;
  return int(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

template <int D>
cudaError_t launch_bwd(const AttnBwdDesc& a, cudaStream_t s) {
  using C = BwdCfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_bwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Bwd2Cfg<D>::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_bwd3_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Bwd3Cfg<D>::SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long W = 3LL * a.nh * D;
  const long long M = (long long)a.mb * a.S;
  CUtensorMap q, k, v, dO, dq;
  if (!encode(&q, a.qkv, D, a.S, a.nh, a.mb, W, 3 * D, 64, T) ||
      !encode(&k, a.qkv + D, D, a.S, a.nh, a.mb, W, 3 * D, 64, T) ||
      !encode(&v, a.qkv + 2 * D, D, a.S, a.nh, a.mb, W, 3 * D, 64, T) ||
      !encode(&dO, a.dout, D, a.S, a.nh, a.mb, (long long)a.nh * D, D, 64, T) ||
      !encode_f32(&dq, a.dq_acc, (long long)a.nh * D, M))
    return cudaErrorInvalidValue;
  attn_delta_kernel<D><<<ew_blocks(M * a.nh * (D / 8)), 256, 0, s>>>(a.out, a.dout, a.delta,
                                                                      a.dq_acc, a.S, a.nh, a.mb);
  BwdParams p;
  p.dq_acc = a.dq_acc;
  p.lse = a.lse;
  p.delta = a.delta;
  p.dqkv = a.dqkv;
  p.S = a.S;
  p.nh = a.nh;
  p.mb = a.mb;
  p.scale = a.scale;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  const int grid = (a.S / T) * a.nh * a.mb;
  if (g_bwd_variant == 3)
    attn_bwd3_kernel<D><<<grid, kBwd3Threads, Bwd3Cfg<D>::SMEM, s>>>(q, k, v, dO, dq, p);
  else if (g_bwd_variant == 2)
    attn_bwd2_kernel<D><<<grid, kBwd2Threads, Bwd2Cfg<D>::SMEM, s>>>(q, k, v, dO, dq, p);
  else
    attn_bwd_kernel<D><<<grid, kBwdThreads, C::SMEM, s>>>(q, k, v, dO, dq, p);
  if (a.rope)
    attn_dq_cast_rope_kernel<D><<<ew_blocks(M * a.nh * (D / 16)), 256, 0, s>>>(a.dq_acc, a.dqkv, a.rope,
                                                                              M, a.S, a.nh);
  else
    attn_dq_cast_kernel<D><<<ew_blocks(M * a.nh * (D / 8)), 256, 0, s>>>(a.dq_acc, a.dqkv, M, a.nh);
  return cudaGetLastError();
}

}  // namespace

void attention_fwd_variant(int v) { g_fwd_variant = (v >= 1 && v <= 3) ? v : 3; }
void attention_bwd_variant(int v) { g_bwd_variant = (v >= 1 && v <= 3) ? v : 3; }

cudaError_t attention_fwd(const AttnDesc& a, cudaStream_t s) {
  if (a.S % T != 0 || a.S <= 0) return cudaErrorInvalidValue;
  if (a.d == 128) return launch_fwd<128>(a, s);
  if (a.d == 64) return launch_fwd<64>(a, s);
  return cudaErrorInvalidValue;
}

cudaError_t attention_bwd(const AttnBwdDesc& a, cudaStream_t s) {
  if (a.S % T != 0 || a.S <= 0) return cudaErrorInvalidValue;
  if (a.d == 128) return launch_bwd<128>(a, s);
  if (a.d == 64) return launch_bwd<64>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace hexexec
