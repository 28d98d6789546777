// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
// Roles (256 threads):  warp 0 = TMA producer (one elected lane),
//                       warp 1 = MMA issuer (one elected lane),
//                       warp 2 = TMEM allocator,
//                       warps 4..7 = epilogue (TMEM -> registers -> global).
// Operands stream through a STAGES-deep shared-memory ring (mbarrier
// full/empty pairs); the fp32 accumulator is double-buffered in TMEM
// (2 x BN columns) so the epilogue of tile t overlaps the mainloop of t+1.
// Tile shape 128 x BN x 64, UMMA 128 x BN x 16, SWIZZLE_128B operand tiles.
// K-major operands are loaded as one TMA box [rows][64]; MN-major operands as
// (rows/64) boxes [64 k][64 mn], giving the canonical MN-major UMMA layout
// (LBO = 64*128 B between MN atoms, SBO = 1024 B between 8-row k groups).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm.h"

namespace hexexec {

namespace {

constexpr int BM = 128;
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
};

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN >= 256 ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr size_t SMEM = 1024 /*align slack*/ + size_t(STAGES) * STAGE_BYTES + 256;
};

HX_DEVICE bool tile_skipped(const EpiParams& p, int m0, int n0) {
  return p.causal == kCausalSkipUpper && n0 > m0 + BM - 1;
}

HX_DEVICE void k_range(const EpiParams& p, int m0, int& kb0, int& kb1) {
  int k_begin = 0, k_end = p.K;
  if (p.causal == kCausalKLower) k_end = min(p.K, m0 + BM);
  if (p.causal == kCausalKUpper) k_begin = (m0 / BK) * BK;
  kb0 = k_begin / BK;
  kb1 = (k_end + BK - 1) / BK;
  if (kb1 < kb0) kb1 = kb0;
}

// tile t -> (m0, n-tile index, batch coords); n fastest so CTAs of one wave
// share the A row-panel in L2
HX_DEVICE void decode_tile(const EpiParams& p, int t, int& m0, int& nt, int& z1, int& z2) {
  nt = t % p.n_tiles;
  int r = t / p.n_tiles;
  m0 = (r % p.m_tiles) * BM;
  int z = r / p.m_tiles;
  z1 = z % p.nb1;
  z2 = z / p.nb1;
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const EpiParams p) {
  using C = Cfg<BN>;
  constexpr int ST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * C::STAGE_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int m0, nt, z1, z2;
        decode_tile(p, t, m0, nt, z1, z2);
        int n0 = nt * BN;
        if (tile_skipped(p, m0, n0)) continue;
        int kb0, kb1;
        k_range(p, m0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_4d(a + c * (BK * 128), &tmA, &full[stage], m0 + c * 64, k0, z1, z2);
          } else {
            tma_load_4d(a, &tmA, &full[stage], k0, m0, z1, z2);
          }
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_4d(b + c * (BK * 128), &tmB, &full[stage], n0 + c * 64, k0, z1, z2);
          } else {
            tma_load_4d(b, &tmB, &full[stage], k0, n0, z1, z2);
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(A_MN) << 15) |
                                 (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) |
                                 (uint32_t(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int m0, nt, z1, z2;
        decode_tile(p, t, m0, nt, z1, z2);
        int n0 = nt * BN;
        if (tile_skipped(p, m0, n0)) continue;
        int kb0, kb1;
        k_range(p, m0, kb0, kb1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tbase + uint32_t(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            uint64_t ad = A_MN ? umma_desc_sw128(a_addr + ks * 2048, BK * 128, 1024)
                               : umma_desc_sw128(a_addr + ks * 32, 16, 1024);
            uint64_t bd = B_MN ? umma_desc_sw128(b_addr + ks * 2048, BK * 128, 1024)
                               : umma_desc_sw128(b_addr + ks * 32, 16, 1024);
            tc_mma_f16(dtm, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int m0, nt, z1, z2;
      decode_tile(p, t, m0, nt, z1, z2);
      int n0 = nt * BN;
      if (tile_skipped(p, m0, n0)) continue;
      int kb0, kb1;
      k_range(p, m0, kb0, kb1);
      const bool have = kb1 > kb0;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const long long cbase = z1 * p.cbs1 + z2 * p.cbs2 + (long long)row * p.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + c), r);
        tmem_ld_wait();
        const int col = n0 + c;
        if (row >= p.M || col >= p.N) continue;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = have ? __uint_as_float(r[i]) * p.alpha : 0.f;
        const bool full_chunk = col + 32 <= p.N;
        if (p.c_fp32) {
          float* out = reinterpret_cast<float*>(p.C) + cbase + col;
          const float* res = p.R ? p.R + cbase + col : nullptr;
          if (full_chunk && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
            float4* o4 = reinterpret_cast<float4*>(out);
            // issue every load of the chunk before the first store (no aliasing
            // stalls: 8 independent 16-byte loads in flight per thread)
            if (p.beta || res) {
              float4 o[8];
              const float4* src = p.beta ? o4 : reinterpret_cast<const float4*>(res);
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = __ldcs(src + i);
              if (p.beta && res) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  float4 q = __ldcs(reinterpret_cast<const float4*>(res) + i);
                  o[i].x += q.x; o[i].y += q.y; o[i].z += q.z; o[i].w += q.w;
                }
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                v[4 * i] += o[i].x; v[4 * i + 1] += o[i].y;
                v[4 * i + 2] += o[i].z; v[4 * i + 3] += o[i].w;
              }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
              o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && col + i < p.N; ++i)
              out[i] = (p.beta ? out[i] : 0.f) + (res ? res[i] : 0.f) + v[i];
          }
        } else {
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + cbase + col;
          if (full_chunk && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
            uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint4 w;
              w.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
              w.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
              w.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
              w.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
              o4[i] = w;
            }
          } else {
            for (int i = 0; i < 32 && col + i < p.N; ++i) out[i] = __float2bfloat16_rn(v[i]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_sm_limit = 0;
int g_num_sms = 0;

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

// 4D map over a bf16 operand: dim0 contiguous.  rows_box = box extent on dim1.
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

template <int BN, int AM, int BMn>
cudaError_t launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const EpiParams& p,
                     cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, AM, BMn>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  int sms = g_sm_limit > 0 ? std::min(g_sm_limit, g_num_sms) : g_num_sms;
  int grid = std::min(p.num_tiles, sms);
  if (grid <= 0) return cudaSuccess;
  gemm_kernel<BN, AM, BMn><<<grid, kThreads, C::SMEM, s>>>(ma, mb, p);
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_major(int am, int bm, const CUtensorMap& ma, const CUtensorMap& mb,
                           const EpiParams& p, cudaStream_t s) {
  if (!am && !bm) return launch_t<BN, 0, 0>(ma, mb, p, s);
  if (!am && bm) return launch_t<BN, 0, 1>(ma, mb, p, s);
  if (am && !bm) return launch_t<BN, 1, 0>(ma, mb, p, s);
  return launch_t<BN, 1, 1>(ma, mb, p, s);
}

}  // namespace

void gemm_set_sm_limit(int sms) { g_sm_limit = sms; }

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t stream) {
  cudaError_t e = load_encode();
  if (e != cudaSuccess) return e;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  // tile width: 256 for wide outputs, 128 otherwise (fewer wasted columns on narrow N)
  const int BN = d.N >= 256 ? 256 : 128;
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
    ok = make_map(&mb, d.B, d.K, d.N, d.nb1, d.nb2, BK, BN);
  if (!ok) return cudaErrorInvalidValue;
  EpiParams p;
  p.C = d.C;
  p.R = d.R;
  if (d.R && !d.c_fp32) return cudaErrorInvalidValue;
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
  p.m_tiles = (d.M + BM - 1) / BM;
  p.n_tiles = (d.N + BN - 1) / BN;
  p.num_tiles = p.m_tiles * p.n_tiles * d.nb1 * d.nb2;
  if (BN == 256) return dispatch_major<256>(d.A.mn_major, d.B.mn_major, ma, mb, p, stream);
  return dispatch_major<128>(d.A.mn_major, d.B.mn_major, ma, mb, p, stream);
}

}  // namespace hexexec
