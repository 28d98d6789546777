// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
// Roles (256 threads per CTA):  warp 0 = TMA producer (one elected lane),
//                               warp 1 = MMA issuer (one lane, leader CTA only),
//                               warp 2 = TMEM allocator,
//                               warps 4..7 = epilogue (TMEM -> registers -> global).
// CG = 2 runs CTA pairs (cluster of 2, `cta_group::2`): one 256 x BN x 16 UMMA
// per k-step spans both SMs; each CTA stages its 128 rows of A and BN/2 rows of
// B, TMA completion is counted on the leader's mbarrier, the leader issues the
// MMAs and multicasts tcgen05.commit to both CTAs; each CTA's TMEM holds its
// 128 accumulator rows.  CG = 1 is the single-SM variant (M < 256 problems).
// Operands stream through a STAGES-deep smem ring (full/empty mbarriers); the
// fp32 accumulator is double-buffered in TMEM (2 x BN columns) so the
// epilogue of tile t overlaps the mainloop of tile t+1.  SWIZZLE_128B tiles:
// K-major operands as one TMA box [rows][64]; MN-major operands as (rows/64)
// boxes [64 k][64 mn] (canonical MN-major UMMA layout: LBO = 64*128 B between
// MN atoms, SBO = 1024 B between 8-row k groups).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm.h"

namespace hexexec {

namespace {

constexpr int BM = 128;  // rows per CTA
constexpr int BK = 64;
constexpr int kThreads = 256;

struct EpiParams {
  void* C;
  const float* R;
  long long ldc, cbs1, cbs2;
  int M, N, K, nb1, nb2;
  int c_fp32, beta;
  float alpha;
  int causal;
  int m_tiles, n_tiles, num_tiles;
  // split-K of the tail: tiles >= split_first are cut into split_s k-ranges
  int split_first, split_s, num_units;
  int split_direct;  // partials reduce-add straight into C (beta, no R)
  float* ws;         // [split tiles][TM][BN] fp32
  int* ws_cnt;       // per (split tile, 32-row slab)
  int npeer;         // extra copies of every stored C tile (TP peers' buffers)
  int group_m;       // grouped tile raster (M-tiles per band), 0 = n fastest
  int act_mode;      // 1: SwiGLU epilogue, act = silu(g) * u to pm.m[0]
  const float2* rope;  // RoPE epilogue: (cos, sin) table [rope_S][rope_d / 2], or null
  int rope_d, rope_S;
  int mc;            // CTA pairs per cluster along N sharing the A tile (TMA multicast)
  int n_tiles_c;     // cluster tiles along N = ceil(n_tiles / mc)
  int* smid_log;     // tests: CTA b writes its %smid to smid_log[b] (SM-cap placement)
};

// TMA maps of the peer copies of C (IPC-mapped buffers of the other TP ranks,
// reached over NVLink): the epilogue stores each tile to C and to every peer
struct alignas(64) PeerMaps {
  CUtensorMap m[kMaxGemmPeers];
};

template <int BN, int CG>
struct Cfg {
  static constexpr int TM = BM * CG;         // rows per (pair) tile
  static constexpr int BNC = BN / CG;        // B rows staged per CTA
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BNC * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // epilogue staging per epilogue warp: 2 x [32 rows][32 cols] fp32 store buffers
  // (TMA store / reduce-add sources) + 1 buffer for the residual tile (TMA load)
  static constexpr uint32_t EPI_CHUNK = 32 * 32 * 4;
  static constexpr uint32_t EPI_WARP = 3 * EPI_CHUNK;
  static constexpr uint32_t EPI_BYTES = 4 * EPI_WARP;
  // 227 KB opt-in dynamic smem per CTA, minus alignment slack, epilogue, barriers
  static constexpr uint32_t MAIN_BUDGET = 232448u - 1024u - 256u - EPI_BYTES;
  static constexpr int STAGES = int(MAIN_BUDGET / STAGE_BYTES) > 8 ? 8 : int(MAIN_BUDGET / STAGE_BYTES);
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr size_t SMEM =
      1024 /*align slack*/ + size_t(STAGES) * STAGE_BYTES + EPI_BYTES + 256;
};

// byte offset of the 16-byte chunk `chunk` of row `row` inside a [32][row_bytes]
// tile staged for a SWIZZLE_128B (row_bytes 128) / SWIZZLE_64B (row_bytes 64) TMA box
template <int ROW_BYTES>
HX_DEVICE uint32_t swz(int row, int chunk) {
  const uint32_t off = uint32_t(row * ROW_BYTES + chunk * 16);
  constexpr uint32_t mask = ROW_BYTES == 128 ? 7u : 3u;
  return off ^ (((off >> 7) & mask) << 4);
}

template <int TM>
HX_DEVICE bool tile_skipped(const EpiParams& p, int m0, int n0) {
  return p.causal == kCausalSkipUpper && n0 > m0 + TM - 1;
}

template <int TM>
HX_DEVICE void k_range(const EpiParams& p, int m0, int& kb0, int& kb1) {
  int k_begin = 0, k_end = p.K;
  if (p.causal == kCausalKLower) k_end = min(p.K, m0 + TM);
  if (p.causal == kCausalKUpper) k_begin = (m0 / BK) * BK;
  kb0 = k_begin / BK;
  kb1 = (k_end + BK - 1) / BK;
  if (kb1 < kb0) kb1 = kb0;
}

// work unit -> (tile, k part); part -1 = whole tile
HX_DEVICE void decode_unit(const EpiParams& p, int u, int& t, int& part) {
  if (u < p.split_first) {
    t = u;
    part = -1;
  } else {
    const int v = u - p.split_first;
    t = p.split_first + v / p.split_s;
    part = v % p.split_s;
  }
}

template <int TM>
HX_DEVICE void unit_k_range(const EpiParams& p, int m0, int part, int& kb0, int& kb1) {
  k_range<TM>(p, m0, kb0, kb1);
  if (part >= 0) {
    const int len = kb1 - kb0;
    const int a = kb0 + len * part / p.split_s;
    kb1 = kb0 + len * (part + 1) / p.split_s;
    kb0 = a;
  }
}

HX_DEVICE void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// tile t -> (m0, n-tile index, batch coords).  group_m > 0: grouped raster,
// bands of group_m M-tiles walked M-fastest, so one wave of P pairs covers a
// ~group_m x P/group_m block and both operand panels are re-read from L2
// (n-fastest over a wide N would stream every B panel from HBM once per
// M-tile: 8x the B bytes at M = 2048).  group_m = 0: n fastest.
template <int TM>
HX_DEVICE void decode_tile(const EpiParams& p, int t, int& m0, int& nt, int& z1, int& z2) {
  const int per_batch = p.m_tiles * p.n_tiles_c;
  const int z = t / per_batch;
  const int r = t - z * per_batch;
  if (p.group_m > 0) {
    const int per_group = p.group_m * p.n_tiles_c;
    const int g = r / per_group;
    const int first = g * p.group_m;
    const int gm = min(p.group_m, p.m_tiles - first);
    const int q = r - g * per_group;
    m0 = (first + q % gm) * TM;
    nt = q / gm;
  } else {
    nt = r % p.n_tiles_c;
    m0 = (r / p.n_tiles_c) * TM;
  }
  z1 = z % p.nb1;
  z2 = z / p.nb1;
}

// stage a 32-row x 32-col chunk for TMA: fp32 rows of 128 B (SWIZZLE_128B) or
// bf16 rows of 64 B (SWIZZLE_64B); lane = row
HX_DEVICE void stage_chunk(uint8_t* sbuf, const float* v, bool f32, int lane) {
  if (f32) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(sbuf + swz<128>(lane, q)) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
      w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
      *reinterpret_cast<uint4*>(sbuf + swz<64>(lane, q)) = w;
    }
  }
}

// -DHX_GEMM_SLEEP_WAIT: waits with a suspend-time hint; measured: +3 % work per
// clock, -3 % clock under the power cap, same TFLOP/s and GFLOP/J (not used)
#ifdef HX_GEMM_SLEEP_WAIT
#define HX_GEMM_WAIT mbar_wait_sleep
#else
#define HX_GEMM_WAIT mbar_wait
#endif

template <int BN, int A_MN, int B_MN, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                const __grid_constant__ CUtensorMap tmW, const __grid_constant__ PeerMaps pm,
                const EpiParams p) {
  using C = Cfg<BN, CG>;
  constexpr int ST = C::STAGES;
  constexpr int TM = C::TM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * C::A_BYTES;
  uint8_t* sEpi = smem + ST * C::STAGE_BYTES;  // 1024-aligned (stage sizes are multiples of 1 KB)
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + C::EPI_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint64_t* rbar = tempty + 2;    // [4] residual-tile loads, one per epilogue warp
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (p.smid_log != nullptr && threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    p.smid_log[blockIdx.x] = int(sm);
  }
  // cluster = mc CTA pairs along N (pair q owns n-tile mc*nt_c + q); the pair's
  // CTAs are cluster ranks 2q (leader) and 2q+1
  const uint32_t crank_cl = CG == 2 ? cluster_ctarank() : 0;
  const uint32_t crank = crank_cl & 1u;
  const int pair_cl = int(crank_cl >> 1);
  const bool leader = crank == 0;
  // cluster index and count (persistent loop over cluster tiles)
  const int pid = blockIdx.x / (CG * p.mc);
  const int npairs = gridDim.x / (CG * p.mc);

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], p.mc);  // one MMA commit per pair reading the stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * CG);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&rbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 3 && lane == 0) {
    tma_prefetch(&tmC);
    if (p.R) tma_prefetch(&tmR);
  }
  if (warp == 2) {
    if (CG == 2)
      tmem_alloc_2sm<C::TMEM_COLS>(tslot);
    else
      tmem_alloc<C::TMEM_COLS>(tslot);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // programmatic dependent launch: everything above (barriers, TMEM, tensor-map
  // prefetch) overlaps the previous kernel's tail; no global memory is touched
  // before the previous grid has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs of a pair)
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pid; u < p.num_units; u += npairs) {
        int t, part;
        decode_unit(p, u, t, part);
        int m0, nt, z1, z2;
        decode_tile<TM>(p, t, m0, nt, z1, z2);
        nt = nt * p.mc + pair_cl;
        int n0 = nt * BN;
        if (tile_skipped<TM>(p, m0, n0)) continue;
        int kb0, kb1;
        unit_k_range<TM>(p, m0, part, kb0, kb1);
        const int am = m0 + BM * int(crank);      // this CTA's A rows
        const int bn = n0 + C::BNC * int(crank);  // this CTA's B rows
        for (int kb = kb0; kb < kb1; ++kb) {
          HX_GEMM_WAIT(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES * CG);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          int k0 = kb * BK;
          if (CG == 2) {
            if (p.mc == 2) {
              // the A half of this CTA is the same for both pairs: pair 0 loads it
              // into both (multicast), the bytes counted on each pair's leader
              if (pair_cl == 0) {
                const uint16_t mask = uint16_t((1u << crank_cl) | (1u << (crank_cl + 2)));
                if (A_MN) {
#pragma unroll
                  for (int c = 0; c < BM / 64; ++c)
                    tma_load_4d_2sm_mc(a + c * (BK * 128), &tmA, &full[stage], mask, am + c * 64,
                                       k0, z1, z2);
                } else {
                  tma_load_4d_2sm_mc(a, &tmA, &full[stage], mask, k0, am, z1, z2);
                }
              }
            } else if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c)
                tma_load_4d_2sm(a + c * (BK * 128), &tmA, &full[stage], am + c * 64, k0, z1, z2);
            } else {
              tma_load_4d_2sm(a, &tmA, &full[stage], k0, am, z1, z2);
            }
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < C::BNC / 64; ++c)
                tma_load_4d_2sm(b + c * (BK * 128), &tmB, &full[stage], bn + c * 64, k0, z1, z2);
            } else {
              tma_load_4d_2sm(b, &tmB, &full[stage], k0, bn, z1, z2);
            }
          } else {
            if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c)
                tma_load_4d(a + c * (BK * 128), &tmA, &full[stage], am + c * 64, k0, z1, z2);
            } else {
              tma_load_4d(a, &tmA, &full[stage], k0, am, z1, z2);
            }
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < C::BNC / 64; ++c)
                tma_load_4d(b + c * (BK * 128), &tmB, &full[stage], bn + c * 64, k0, z1, z2);
            } else {
              tma_load_4d(b, &tmB, &full[stage], k0, bn, z1, z2);
            }
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA)
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(A_MN) << 15) |
                                 (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) |
                                 (uint32_t(TM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pid; u < p.num_units; u += npairs) {
        int t, part;
        decode_unit(p, u, t, part);
        int m0, nt, z1, z2;
        decode_tile<TM>(p, t, m0, nt, z1, z2);
        nt = nt * p.mc + pair_cl;
        int n0 = nt * BN;
        if (tile_skipped<TM>(p, m0, n0)) continue;
        int kb0, kb1;
        unit_k_range<TM>(p, m0, part, kb0, kb1);
        HX_GEMM_WAIT(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tbase + uint32_t(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          HX_GEMM_WAIT(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            uint64_t ad = A_MN ? umma_desc_sw128(a_addr + ks * 2048, BK * 128, 1024)
                               : umma_desc_sw128(a_addr + ks * 32, 16, 1024);
            uint64_t bd = B_MN ? umma_desc_sw128(b_addr + ks * 2048, BK * 128, 1024)
                               : umma_desc_sw128(b_addr + ks * 32, 16, 1024);
            if (CG == 2)
              tc_mma_f16_2sm(dtm, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
            else
              tc_mma_f16(dtm, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          if (CG == 2)
            tc_commit_2sm_mc(&empty[stage], p.mc == 2 ? uint16_t(0xF) : uint16_t(0x3));
          else
            tc_commit(&empty[stage]);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2)
          tc_commit_2sm_mc(&tfull[acc], uint16_t(0x3u << (2 * pair_cl)));
        else
          tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs; each owns 128 accumulator rows)
    // TMEM -> registers (x alpha, + residual tile loaded by TMA) -> swizzled
    // smem chunk [32 rows][32 cols] -> TMA store (or TMA reduce-add for beta)
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    uint8_t* ebuf = sEpi + ew * C::EPI_WARP;  // two store buffers
    uint8_t* rbuf = ebuf + 2 * C::EPI_CHUNK;  // residual tile
    int acc = 0;
    uint32_t acc_phase = 0, rphase = 0;
    int sb = 0;
    for (int u = pid; u < p.num_units; u += npairs) {
      int t, part;
      decode_unit(p, u, t, part);
      int m0, nt, z1, z2;
      decode_tile<TM>(p, t, m0, nt, z1, z2);
      nt = nt * p.mc + pair_cl;
      int n0 = nt * BN;
      if (tile_skipped<TM>(p, m0, n0)) continue;
      int kb0, kb1;
      unit_k_range<TM>(p, m0, part, kb0, kb1);
      const bool have = kb1 > kb0;
      const bool split = part >= 0;
      const bool to_ws = split && !p.split_direct;  // partial -> workspace
      const bool add_r = p.R && !split;              // a split tile's R is added by its finisher
      const bool f32 = p.c_fp32 || to_ws;
      const int sidx = t - p.split_first;            // split tile index
      const int wrow = sidx * TM + BM * int(crank) + ew * 32;
      HX_GEMM_WAIT(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row0 = m0 + BM * int(crank) + ew * 32;  // this warp's 32-row slab
      if (row0 < p.M && p.act_mode) {
        // SwiGLU epilogue: C columns come in 128-wide (64 gate | 64 up) chunk
        // pairs; per 32-column half: store g and u (bf16) to C and
        // act = silu(g) * u, from the bf16-rounded g and u exactly as
        // swiglu_fwd_kernel computes it, to the act map (pm.m[0], [M, N/2]).
        // Each 4 KB staging buffer holds two bf16 chunks: 3 stores per
        // half, double-buffered over the 3 buffers.
#pragma unroll 1
        for (int c = 0; c < BN; c += 128) {
          if (n0 + c >= p.N) break;
#pragma unroll 1
          for (int h = 0; h < 64; h += 32) {
            uint32_t rg[32], ru[32];
            const uint32_t tcol = tbase + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + c + h);
            tmem_ld_32x32b_x32(tcol, rg);
            tmem_ld_32x32b_x32(tcol + 64, ru);
            tmem_ld_wait();
            float g[32], uu[32], a[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              g[i] = __bfloat162float(__float2bfloat16(__uint_as_float(rg[i]) * p.alpha));
              uu[i] = __bfloat162float(__float2bfloat16(__uint_as_float(ru[i]) * p.alpha));
              a[i] = g[i] * (1.f / (1.f + __expf(-g[i]))) * uu[i];
            }
            // the slot set written now was read by the stores two halves ago
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* b0 = ebuf + sb * (C::EPI_CHUNK / 2);  // slots sb, sb+2, sb+4 (2 KB each)
            uint8_t* b1 = b0 + C::EPI_CHUNK;
            uint8_t* b2 = b1 + C::EPI_CHUNK;
            stage_chunk(b0, g, false, lane);
            stage_chunk(b1, uu, false, lane);
            stage_chunk(b2, a, false, lane);
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmC, b0, n0 + c + h, row0, z1, z2);
              tma_store_4d(&tmC, b1, n0 + c + 64 + h, row0, z1, z2);
              tma_store_4d(&pm.m[0], b2, (n0 + c) / 2 + h, row0, z1, z2);
              bulk_commit();
            }
            sb ^= 1;
          }
        }
      } else if (row0 < p.M && p.rope) {
        // RoPE epilogue (QKV projection): head-interleaved (h, {q, k, v}, d)
        // columns; q and k blocks are rotated (rotate-half, pairs j / j + d/2)
        // from the bf16-rounded values exactly as rope_kernel does, v passes.
        // Position = row % S; angles from the precomputed (cos, sin) table.
        const int dh = p.rope_d, half = dh / 2;
        const float2* trow = p.rope + (long long)((row0 + lane) % p.rope_S) * half;
#pragma unroll 1
        for (int blk = 0; blk < BN; blk += dh) {
          if (n0 + blk >= p.N) break;
          const bool rot = ((n0 + blk) / dh) % 3 != 2;
#pragma unroll 1
          for (int c = 0; c < half; c += 32) {
            uint32_t ra[32], rb[32];
            const uint32_t tcol = tbase + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + blk + c);
            tmem_ld_32x32b_x32(tcol, ra);
            tmem_ld_32x32b_x32(tcol + half, rb);
            tmem_ld_wait();
            float xa[32], xb[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              xa[i] = __bfloat162float(__float2bfloat16(__uint_as_float(ra[i]) * p.alpha));
              xb[i] = __bfloat162float(__float2bfloat16(__uint_as_float(rb[i]) * p.alpha));
            }
            if (rot) {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(trow + c + i));
                const float cs0 = t.x, sn0 = t.y, cs1 = t.z, sn1 = t.w;
                const float x0 = xa[i], y0 = xb[i], x1 = xa[i + 1], y1 = xb[i + 1];
                // explicit rounding, as rope_kernel
                xa[i] = __fsub_rn(__fmul_rn(x0, cs0), __fmul_rn(y0, sn0));
                xb[i] = __fadd_rn(__fmul_rn(y0, cs0), __fmul_rn(x0, sn0));
                xa[i + 1] = __fsub_rn(__fmul_rn(x1, cs1), __fmul_rn(y1, sn1));
                xb[i + 1] = __fadd_rn(__fmul_rn(y1, cs1), __fmul_rn(x1, sn1));
              }
            }
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            uint8_t* b0 = ebuf;
            uint8_t* b1 = ebuf + C::EPI_CHUNK;
            stage_chunk(b0, xa, false, lane);
            stage_chunk(b1, xb, false, lane);
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmC, b0, n0 + blk + c, row0, z1, z2);
              tma_store_4d(&tmC, b1, n0 + blk + half + c, row0, z1, z2);
              bulk_commit();
            }
          }
        }
      } else if (row0 < p.M) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          const int col = n0 + c;
          if (col >= p.N) break;
          if (add_r && lane == 0) {
            mbar_arrive_expect_tx(&rbar[ew], C::EPI_CHUNK);
            tma_load_4d(rbuf, &tmR, &rbar[ew], col, row0, z1, z2);
          }
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + c), r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = have ? __uint_as_float(r[i]) * p.alpha : 0.f;
          if (add_r) {
            mbar_wait(&rbar[ew], rphase);
            rphase ^= 1;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 o = *reinterpret_cast<const float4*>(rbuf + swz<128>(lane, q));
              v[4 * q] += o.x;
              v[4 * q + 1] += o.y;
              v[4 * q + 2] += o.z;
              v[4 * q + 3] += o.w;
            }
          }
          // the buffer written now was the source of the store two chunks ago
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          uint8_t* sbuf = ebuf + sb * C::EPI_CHUNK;
          stage_chunk(sbuf, v, f32, lane);
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            if (to_ws)
              tma_reduce_add_4d(&tmW, sbuf, c, wrow, 0, 0);
            else if (p.beta || split)
              tma_reduce_add_4d(&tmC, sbuf, col, row0, z1, z2);
            else {
              tma_store_4d(&tmC, sbuf, col, row0, z1, z2);
              for (int k = 0; k < p.npeer; ++k) tma_store_4d(&pm.m[k], sbuf, col, row0, z1, z2);
            }
            bulk_commit();
          }
          sb ^= 1;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2)
          mbar_arrive_cluster(&tempty[acc], crank_cl & ~1u);  // the pair leader's MMA waits on both CTAs
        else
          mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (to_ws && row0 < p.M) {
        // publish the partial; the last of the split_s partials of this slab
        // sums the workspace slab into C and leaves slab and counter zero
        int* cnt = p.ws_cnt + sidx * (4 * CG) + int(crank) * 4 + ew;
        int old = 0;
        if (lane == 0) {
          bulk_wait_all();
          fence_proxy_async_global();
          __threadfence();
          old = atomicAdd(cnt, 1);
          if (old == p.split_s - 1) {
            __threadfence();
            fence_proxy_async_global();
          }
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        __syncwarp();
        if (old == p.split_s - 1) {
          // coalesced reads of the workspace slab (lane -> rows lr + 4j, float4
          // column lq), two chunks in flight; transposed through rbuf into the
          // row-per-lane staging layout of the store path
          const int lr = lane >> 3, lq = lane & 7;
          float* wbase = p.ws + (long long)wrow * BN + 4 * lq;
          const int nch = (min(BN, p.N - n0) + 31) / 32;
          float4 cur[8], nxt[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            cur[j] = __ldcg(reinterpret_cast<const float4*>(wbase + (long long)(lr + 4 * j) * BN));
#pragma unroll 1
          for (int ci = 0; ci < nch; ++ci) {
            const int c = ci * 32;
            const int col = n0 + c;
            if (ci + 1 < nch) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                nxt[j] = __ldcg(reinterpret_cast<const float4*>(wbase + (long long)(lr + 4 * j) * BN + c + 32));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              __stcg(reinterpret_cast<float4*>(wbase + (long long)(lr + 4 * j) * BN + c),
                     make_float4(0.f, 0.f, 0.f, 0.f));
            if (p.R && col + 4 * lq < p.N) {
              const float* rs = p.R + (long long)z1 * p.cbs1 + (long long)z2 * p.cbs2 + col + 4 * lq;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int row = row0 + lr + 4 * j;
                if (row < p.M) {
                  const float4 o = __ldcg(reinterpret_cast<const float4*>(rs + (long long)row * p.ldc));
                  cur[j].x += o.x; cur[j].y += o.y; cur[j].z += o.z; cur[j].w += o.w;
                }
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(rbuf + swz<128>(lr + 4 * j, lq)) = cur[j];
            __syncwarp();
            float v[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 o = *reinterpret_cast<const float4*>(rbuf + swz<128>(lane, q));
              v[4 * q] = o.x; v[4 * q + 1] = o.y; v[4 * q + 2] = o.z; v[4 * q + 3] = o.w;
            }
            __syncwarp();
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* sbuf = ebuf + sb * C::EPI_CHUNK;
            stage_chunk(sbuf, v, p.c_fp32, lane);
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              if (p.beta)
                tma_reduce_add_4d(&tmC, sbuf, col, row0, z1, z2);
              else
                tma_store_4d(&tmC, sbuf, col, row0, z1, z2);
              bulk_commit();
            }
            sb ^= 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
          }
          if (lane == 0) atomicExch(cnt, 0);
        }
      }
    }
    if (lane == 0) {
      bulk_wait_all();
      if (p.npeer) {  // peer copies complete and visible before the kernel ends
        fence_proxy_async_global();
        __threadfence_system();
      }
    }
  }

  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_2sm<C::TMEM_COLS>(tbase);
    else
      tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_sm_limit = 0;
int* g_smid_log = nullptr;
int g_num_sms = 0;
int g_force_cg = 0;  // 0 = auto, 1 / 2 = force (tests)
int g_group_m = 8;   // grouped raster band height in M-tiles (0 = n fastest)
int g_pdl = 0;       // launch with programmatic stream serialization
int g_mc = 1;        // 2: A-tile multicast across two CTA pairs (clusters of 4)
// pick 128-wide tiles when they quantise better (off: only nearly empty waves
// qualify, e.g. 2048 x 1024 outputs 645 vs 599 TFLOP/s; a 256 x 128 pair tile
// takes 0.84 of a 256 x 256 one's time)
int g_bn_auto = 0;

cudaError_t load_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  return g_encode ? cudaSuccess : cudaErrorNotSupported;
}

// 4D map over a bf16 operand: dim0 contiguous; box {box0, box1, 1, 1}
bool make_map(CUtensorMap* map, const GemmOperand& op, long long d0, long long d1, int nb1,
              int nb2, uint32_t box0, uint32_t box1) {
  cuuint64_t dims[4] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(nb1), cuuint64_t(nb2)};
  cuuint64_t strides[3] = {cuuint64_t(op.ld * 2), cuuint64_t((op.bs1 ? op.bs1 : 1) * 2),
                           cuuint64_t((op.bs2 ? op.bs2 : 1) * 2)};
  // TMA requires 16-byte aligned strides (unit batch dims get a dummy aligned stride)
  if (nb1 == 1) strides[1] = strides[0] * cuuint64_t(d1);
  if (nb2 == 1) strides[2] = strides[1] * cuuint64_t(nb1);
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 || strides[i] == 0) return false;
  if (reinterpret_cast<uintptr_t>(op.ptr) % 16) return false;
  cuuint32_t box[4] = {box0, box1, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(op.ptr), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 4D map over the output (or residual) matrix: {N, M, nb1, nb2}, box 32 x 32;
// fp32 tiles use SWIZZLE_128B (128-byte rows), bf16 tiles SWIZZLE_64B
bool make_map_c(CUtensorMap* map, void* ptr, int fp32, long long N, long long M, long long ld,
                long long bs1, long long bs2, int nb1, int nb2) {
  const int es = fp32 ? 4 : 2;
  cuuint64_t dims[4] = {cuuint64_t(N), cuuint64_t(M), cuuint64_t(nb1), cuuint64_t(nb2)};
  cuuint64_t strides[3] = {cuuint64_t(ld * es), cuuint64_t((bs1 ? bs1 : 1) * es),
                           cuuint64_t((bs2 ? bs2 : 1) * es)};
  if (nb1 == 1) strides[1] = strides[0] * cuuint64_t(M);
  if (nb2 == 1) strides[2] = strides[1] * cuuint64_t(nb1);
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 || strides[i] == 0) return false;
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return false;
  cuuint32_t box[4] = {32, 32, 1, 1};
  cuuint32_t esd[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        4, ptr, dims, strides, box, esd, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        fp32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int AM, int BMn, int CG>
cudaError_t launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                     const CUtensorMap& mr, const CUtensorMap& mw, const PeerMaps& pm,
                     EpiParams p, int grid, cudaStream_t s) {
  using C = Cfg<BN, CG>;
  static bool attr_done = false;
  auto kern = gemm_kernel<BN, AM, BMn, CG>;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(C::SMEM));
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  if (grid <= 0) return cudaSuccess;
  if (p.mc == 2) {
    // clusters of 4 co-resident at once (GPC packing): one persistent wave
    static int max_cl = 0;
    if (max_cl == 0) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(4 * 64);
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = C::SMEM;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = 4;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) n = 1;
      max_cl = n;
    }
    const int lim = g_sm_limit > 0 ? std::max(1, g_sm_limit / 4) : max_cl;
    grid = std::min(p.num_units, std::min(max_cl, lim)) * 4;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * p.mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mr, mw, pm, p);
}

template <int BN, int CG>
cudaError_t dispatch_major(int am, int bm, const CUtensorMap& ma, const CUtensorMap& mb,
                           const CUtensorMap& mc, const CUtensorMap& mr, const CUtensorMap& mw,
                           const PeerMaps& pm, const EpiParams& p, int grid, cudaStream_t s) {
  if (!am && !bm) return launch_t<BN, 0, 0, CG>(ma, mb, mc, mr, mw, pm, p, grid, s);
  if (!am && bm) return launch_t<BN, 0, 1, CG>(ma, mb, mc, mr, mw, pm, p, grid, s);
  if (am && !bm) return launch_t<BN, 1, 0, CG>(ma, mb, mc, mr, mw, pm, p, grid, s);
  return launch_t<BN, 1, 1, CG>(ma, mb, mc, mr, mw, pm, p, grid, s);
}

// Split of the tail wave: T tiles on P pairs run q = T / P full rounds and a
// last round of r = T % P tiles.  Cutting those r tiles into s k-ranges costs
// ceil(r*s / P) rounds of (1/s + ovh) tile times instead of 1, where ovh is
// the per-part epilogue price measured on B200 (partial reduce-add; plus the
// workspace round trip of the finishing part).  Pick the s (<= 8, >= 4
// k-blocks per part) with the smallest cost; split only if the whole GEMM
// gets >= 4% faster.  Returns 1 when no split pays.
int choose_split(int T, int P, int kblocks, bool direct) {
  const int r = T % P;
  if (r == 0 || P <= 1) return 1;
  const double ovh = direct ? 0.08 : 0.35;
  const int q = T / P;
  int best = 1;
  double best_cost = 1.0;
  for (int s = 2; s <= 8 && kblocks / s >= 4; ++s) {
    const double cost = double((r * s + P - 1) / P) * (1.0 / s + ovh);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  if (best > 1 && (q + best_cost) > 0.96 * (q + 1)) best = 1;
  return best;
}

}  // namespace

void gemm_set_sm_limit(int sms) { g_sm_limit = sms; }
void gemm_set_smid_log(int* log) { g_smid_log = log; }
void gemm_force_cta_group(int cg) { g_force_cg = cg; }
void gemm_set_group_m(int g) { g_group_m = std::max(0, g); }
void gemm_set_pdl(int on) { g_pdl = on ? 1 : 0; }
void gemm_set_multicast(int mc) { g_mc = mc == 2 ? 2 : 1; }
void gemm_set_bn_auto(int on) { g_bn_auto = on ? 1 : 0; }

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t stream) {
  cudaError_t e = load_encode();
  if (e != cudaSuccess) return e;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  if (d.R && !d.c_fp32) return cudaErrorInvalidValue;
  // CTA pairs when M fills 256 rows; tile width 256 for wide outputs, 128
  // otherwise -- or (g_bn_auto) when 128-wide tiles quantise into fewer
  // wave-equivalents: cost = waves x tile time, a 256 x 128 pair tile measured
  // at 0.84 of a 256 x 256 one (2048 x 3072 x 4096: 2 waves of 256-wide tiles
  // 1012 TFLOP/s vs 3 waves of 128-wide 807; A multicast does not change it)
  int CG = d.M > 128 ? 2 : 1;
  if (g_force_cg) CG = g_force_cg;
  int BN = d.N >= 256 ? 256 : 128;
  if (BN == 256 && g_bn_auto && d.causal == kCausalNone) {
    const int sms0 = g_sm_limit > 0 ? std::min(g_sm_limit, g_num_sms) : g_num_sms;
    const long long slots = std::max(1, sms0 / CG);
    const long long mt = (d.M + BM * CG - 1) / (BM * CG), z = (long long)d.nb1 * d.nb2;
    const long long t256 = mt * ((d.N + 255) / 256) * z, t128 = mt * ((d.N + 127) / 128) * z;
    const double c256 = double((t256 + slots - 1) / slots);
    const double c128 = 0.85 * double((t128 + slots - 1) / slots);
    if (c128 < 0.97 * c256) BN = 128;
  }
  const int BNC = BN / CG;
  CUtensorMap ma, mb;
  bool ok;
  if (d.A.mn_major)
    ok = make_map(&ma, d.A, d.M, d.K, d.nb1, d.nb2, 64, BK);
  else
    ok = make_map(&ma, d.A, d.K, d.M, d.nb1, d.nb2, BK, BM);
  if (!ok) return cudaErrorInvalidValue;
  if (d.B.mn_major)
    ok = make_map(&mb, d.B, d.N, d.K, d.nb1, d.nb2, 64, BK);
  else
    ok = make_map(&mb, d.B, d.K, d.N, d.nb1, d.nb2, BK, BNC);
  if (!ok) return cudaErrorInvalidValue;
  EpiParams p;
  p.C = d.C;
  p.R = d.R;
  p.ldc = d.ldc;
  p.cbs1 = d.cbs1;
  p.cbs2 = d.cbs2;
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.nb1 = d.nb1;
  p.nb2 = d.nb2;
  p.c_fp32 = d.c_fp32;
  p.beta = d.beta;
  p.alpha = d.alpha;
  p.causal = d.causal;
  const int TM = BM * CG;
  p.m_tiles = (d.M + TM - 1) / TM;
  p.n_tiles = (d.N + BN - 1) / BN;
  p.num_tiles = p.m_tiles * p.n_tiles * d.nb1 * d.nb2;
  p.group_m = d.causal == kCausalNone ? std::min(p.m_tiles, g_group_m) : 0;
  // A multicast over two CTA pairs along N (dense, paired, >= 2 N tiles)
  p.mc = (g_mc == 2 && CG == 2 && d.causal == kCausalNone && p.n_tiles >= 2) ? 2 : 1;
  p.n_tiles_c = (p.n_tiles + p.mc - 1) / p.mc;
  p.num_tiles = p.m_tiles * p.n_tiles_c * d.nb1 * d.nb2;
  p.smid_log = g_smid_log;
  if (d.beta && !d.c_fp32) return cudaErrorInvalidValue;
  CUtensorMap mc, mr;
  if (!make_map_c(&mc, d.C, d.c_fp32, d.N, d.M, d.ldc, d.cbs1, d.cbs2, d.nb1, d.nb2))
    return cudaErrorInvalidValue;
  if (d.R) {
    if (!make_map_c(&mr, const_cast<float*>(d.R), 1, d.N, d.M, d.ldc, d.cbs1, d.cbs2, d.nb1, d.nb2))
      return cudaErrorInvalidValue;
  } else {
    mr = mc;
  }
  static_assert(sizeof(PeerMaps) == kMaxGemmPeers * sizeof(CUtensorMap), "PeerMaps layout");
  PeerMaps pm;
  p.npeer = d.npeer;
  p.act_mode = d.act ? 1 : 0;
  p.rope = d.rope;
  p.rope_d = d.rope_d;
  p.rope_S = d.rope_S;
  if (d.rope && (d.act || d.npeer || d.beta || d.c_fp32 || d.R || d.nb1 * d.nb2 != 1 ||
                 (d.rope_d != 64 && d.rope_d != 128) || d.N % (3 * d.rope_d) || d.rope_S <= 0))
    return cudaErrorInvalidValue;
  if (d.act && (d.npeer || d.beta || d.c_fp32 || d.R || d.N % 128 || d.nb1 * d.nb2 != 1))
    return cudaErrorInvalidValue;
  if (d.npeer < 0 || d.npeer > kMaxGemmPeers) return cudaErrorInvalidValue;
  if (d.npeer && (d.beta || d.c_fp32)) return cudaErrorInvalidValue;
  for (int k = 0; k < d.npeer; ++k)
    if (!make_map_c(&pm.m[k], d.peer_C[k], 0, d.N, d.M, d.ldc, d.cbs1, d.cbs2, d.nb1, d.nb2))
      return cudaErrorInvalidValue;
  for (int k = d.npeer; k < kMaxGemmPeers; ++k) pm.m[k] = mc;
  if (d.act && !make_map_c(&pm.m[0], d.act, 0, d.N / 2, d.M, d.ld_act ? d.ld_act : d.N / 2, 0, 0, 1, 1))
    return cudaErrorInvalidValue;
  const int sms = g_sm_limit > 0 ? std::min(g_sm_limit, g_num_sms) : g_num_sms;
  const int P = std::max(1, sms / CG);
  // tail split (dense GEMMs only)
  p.split_first = p.num_tiles;
  p.split_s = 1;
  p.num_units = p.num_tiles;
  p.split_direct = 0;
  p.ws = d.ws;
  p.ws_cnt = d.ws_cnt;
  CUtensorMap mw = mc;
  if (d.causal == kCausalNone && d.split != 0 && d.npeer == 0 && !d.act && !d.rope && p.mc == 1 &&
      p.num_tiles > 0) {
    const int kblocks = (d.K + BK - 1) / BK;
    const bool direct = d.beta && !d.R;
    int s = d.split > 1 ? std::min(d.split, std::max(1, kblocks))
                        : choose_split(p.num_tiles, P, kblocks, direct);
    const int r = d.split > 1 ? std::min(p.num_tiles, P) : p.num_tiles % P;
    const int nsplit = r;
    const bool ws_ok = d.ws && d.ws_cnt && size_t(nsplit) * TM * BN * 4 <= d.ws_bytes &&
                       nsplit * 4 * CG <= d.ws_cnt_n &&
                       make_map_c(&mw, d.ws, 1, BN, (long long)nsplit * TM, BN, 0, 0, 1, 1);
    if (s > 1 && r > 0 && (direct || ws_ok)) {
      p.split_first = p.num_tiles - r;
      p.split_s = s;
      p.num_units = p.split_first + r * s;
      p.split_direct = direct ? 1 : 0;
    }
  }
  const int grid = std::min(p.num_units, p.mc == 2 ? P / 2 : P) * CG * p.mc;
  const int am = d.A.mn_major, bmj = d.B.mn_major;
  if (CG == 2) {
    if (BN == 256) return dispatch_major<256, 2>(am, bmj, ma, mb, mc, mr, mw, pm, p, grid, stream);
    return dispatch_major<128, 2>(am, bmj, ma, mb, mc, mr, mw, pm, p, grid, stream);
  }
  if (BN == 256) return dispatch_major<256, 1>(am, bmj, ma, mb, mc, mr, mw, pm, p, grid, stream);
  return dispatch_major<128, 1>(am, bmj, ma, mb, mc, mr, mw, pm, p, grid, stream);
}

}  // namespace hexexec
