// tc_sa.cu — tensor-core (tcgen05 + TMA) SA kernels for bf16, D = 64 (SATTN_IMPL_TC).
//
// Band-diagonal tiling.  A CTA owns 128 consecutive frames of one
// (batch, head): 4 warps, thread r <-> TMEM lane r <-> row r of the tile.  The
// other operand's rows that any of the 128 rows can touch form one contiguous
// range of 127 + W frames (W = L + R + 1), staged with ONE TMA box (zero-filled
// outside [0, T)) and multiplied densely: S = Q K^T is a 128 x NK tcgen05 MMA
// (NK = 16-rounded 127 + W, e.g. 176 for (32, 8)).  Row r's band is the diagonal
// strip of columns [r, r + W - 1]; warp w only ever reads its 32 rows' strip,
// columns [32w, 32w + CW) with CW = 8-rounded W + 31, from TMEM (tcgen05.ld),
// masks outside the band to -inf before the row max (exact zeros after exp,
// G14), and writes bf16 P (or dS) as the K-major A operand of the second MMA.
//
//  forward  (sa_fwd_tc):   S = Q K^T -> softmax (row max/sum in registers, one thread
//                          per row) -> P -> O = P V (V read MN-major) -> O / l, LSE.
//  backward K1 (sa_bwd_dq_tc, query-major):  delta = rowsum(dO o O); S = Q K^T ->
//                          P = exp(S - LSE); dP = dO V^T (same TMEM columns) ->
//                          dS = P (dP - delta); dQ = scale dS K.
//  backward K2 (sa_bwd_dkdv_tc, key-major):   S^T = K Q^T -> P^T; dP^T = V dO^T ->
//                          dS^T; dV = P^T dO; dK = scale dS^T Q.
// No atomics: every output row is produced by one thread of one CTA -> bitwise
// deterministic (G18).  Operand layouts: TMA tiles are 128-byte rows with the
// 128B swizzle (K-major for Q/K/V/dO as the head-dim-contracted operand, the same
// bytes read MN-major when the frame index is the contraction); thread-written
// P / dS tiles use the no-swizzle 8x16B core-matrix layout.
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "ffma_attn.cuh"
#include "tc_dispatch.h"
#include "tc_ptx.cuh"

namespace sattn {
namespace {

thread_local std::string g_tc_err;
constexpr int kD = 64;
constexpr int kM = 128;          // rows per CTA tile
constexpr int kThreads = 128;

__host__ __device__ constexpr int nk_of(int CW) { return ((96 + CW) + 15) / 16 * 16; }
__host__ __device__ constexpr int tmem_cols_of(int NK) { return NK + 64 <= 256 ? 256 : 512; }

// Write one thread's row (128 rows x NK cols bf16 tile, no-swizzle K-major core-matrix
// layout) from `vals` covering columns [32w, 32w + CW); zeros elsewhere.
template <int CW, int NK>
__device__ __forceinline__ void write_row_interleave(uint8_t* buf, int r, int w, const float* vals) {
  constexpr int SBO = (NK / 8) * 128;
  uint8_t* rowbase = buf + (r >> 3) * SBO + (r & 7) * 16;
#pragma unroll
  for (int j = 0; j < CW / 8; ++j) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(vals[8 * j + 2 * e], vals[8 * j + 2 * e + 1]);
    *reinterpret_cast<uint4*>(rowbase + (4 * w + j) * 128) = v;
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int kc = 0; kc < NK / 8; ++kc)
    if (kc < 4 * w || kc >= 4 * w + CW / 8) *reinterpret_cast<uint4*>(rowbase + kc * 128) = z;
}

// Load columns [32w, 32w + CW) of this warp's 32 TMEM lanes.
template <int CW>
__device__ __forceinline__ void tmem_row_strip(uint32_t tbase, int w, float* v) {
  const uint32_t a = tbase + (uint32_t(32 * w) << 16) + uint32_t(32 * w);
#pragma unroll
  for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(a + 8 * j, v + 8 * j);
}

// Store 64 fp32 accumulators of TMEM row (lane) into a bf16 global row, scaled.
__device__ __forceinline__ void tmem_row64_to_global(uint32_t taddr, float s, bf16* dst, bool store) {
  float v[64];
#pragma unroll
  for (int j = 0; j < 4; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
  tc::tmem_ld_wait();
  if (!store) return;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e] * s, v[8 * j + 2 * e + 1] * s);
    reinterpret_cast<uint4*>(dst)[j] = o;
  }
}

struct TcArgs {
  int T, L, R, BH;
  float scale, scale_log2;
  bf16* O; float* LSE;                           // fwd outputs
  const bf16* Og; const float* LSEin;           // bwd inputs
  bf16* dQ; bf16* dK; bf16* dV; float* delta;    // bwd outputs
};

// ------------------------------------------------------------------------------------------
// forward
// ------------------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__(kThreads, 1)
    sa_fwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, TcArgs a) {
  constexpr int NK = nk_of(CW);
  constexpr int TCOLS = tmem_cols_of(NK);
  constexpr int OCOL = TCOLS == 256 ? NK : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // 128 x 128 B
  uint8_t* sK = sQ + kM * 128;             // NK x 128 B
  uint8_t* sV = sK + NK * 128;             // NK x 128 B
  uint8_t* sP = sV + NK * 128;             // 128 x NK bf16, interleaved
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kM * NK * 2);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * kM, bh = blockIdx.y;
  const int T = a.T, W = a.L + a.R + 1;

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_mbar_init();
  }
  if (w == 0) tc::tmem_alloc(tslot, TCOLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;

  if (tid == 0) {
    tc::mbar_expect_tx(&bars[0], kM * 128 + 2 * NK * 128);
    tc::tma_load_3d(sQ, &tmQ, &bars[0], 0, t0, bh);
    tc::tma_load_3d(sK, &tmK, &bars[0], 0, t0 - a.L, bh);
    tc::tma_load_3d(sV, &tmV, &bars[0], 0, t0 - a.L, bh);
    tc::mbar_wait(&bars[0], 0);
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, NK, 0, 0);
#pragma unroll
    for (int k = 0; k < kD / 16; ++k)
      tc::mma_bf16(tbase, tc::desc_kmajor_sw128(tc::smem_u32(sQ) + 32 * k),
                   tc::desc_kmajor_sw128(tc::smem_u32(sK) + 32 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 0);
  __syncwarp();
  tc::tc_fence_after();

  // softmax over the row's band, in registers
  float s[CW];
  tmem_row_strip<CW>(tbase, w, s);
  tc::tmem_ld_wait();
  const int r = 32 * w + lane;
  const int key0 = t0 - a.L + 32 * w;  // frame of register 0
  float m = neg_inf();
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    const int f = key0 + i;
    const bool v = i >= lane && i < lane + W && f >= 0 && f < T;
    s[i] = v ? s[i] : neg_inf();
    m = fmaxf(m, s[i]);
  }
  const float mref = m == neg_inf() ? 0.f : m;
  float l = 0.f;
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    s[i] = exp2f((s[i] - mref) * a.scale_log2);
    l += s[i];
  }
  write_row_interleave<CW, NK>(sP, r, w, s);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, kD, 0, 1);
    constexpr uint32_t SBO = (NK / 8) * 128;
#pragma unroll
    for (int k = 0; k < NK / 16; ++k)
      tc::mma_bf16(tbase + OCOL, tc::desc_kmajor_interleave(tc::smem_u32(sP) + 256 * k, SBO),
                   tc::desc_mnmajor_sw128(tc::smem_u32(sV) + 2048 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 1);
  __syncwarp();
  tc::tc_fence_after();
  const int t = t0 + r;
  const bool store = t < T;
  tmem_row64_to_global(tbase + (uint32_t(32 * w) << 16) + OCOL, 1.f / l,
                       a.O + ((long long)bh * T + (store ? t : 0)) * kD, store);
  if (store) a.LSE[(long long)bh * T + t] = mref * a.scale + log2f(l) * kLn2;
  tc::tc_fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tbase, TCOLS);
}

// ------------------------------------------------------------------------------------------
// backward K1: delta and dQ (query-major)
// ------------------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__(kThreads, 1)
    sa_bwd_dq_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, TcArgs a) {
  constexpr int NK = nk_of(CW);
  constexpr int TCOLS = tmem_cols_of(NK);
  constexpr int QCOL = TCOLS == 256 ? NK : 256;
  constexpr int R0 = (2 * kM * 128 > kM * NK * 2) ? 2 * kM * 128 : kM * NK * 2;  // [Q | dO] aliased by dS
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + kM * 128;
  uint8_t* sdS = smem;
  uint8_t* sK = smem + ((R0 + 1023) & ~1023);
  uint8_t* sV = sK + NK * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NK * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * kM, bh = blockIdx.y;
  const int T = a.T, W = a.L + a.R + 1;
  const int r = 32 * w + lane, t = t0 + r;
  const bool row_ok = t < T;

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO);
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_mbar_init();
  }
  if (w == 0) tc::tmem_alloc(tslot, TCOLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t lanebase = tbase + (uint32_t(32 * w) << 16);

  if (tid == 0) {
    tc::mbar_expect_tx(&bars[0], 2 * kM * 128 + 2 * NK * 128);
    tc::tma_load_3d(sQ, &tmQ, &bars[0], 0, t0, bh);
    tc::tma_load_3d(sdO, &tmdO, &bars[0], 0, t0, bh);
    tc::tma_load_3d(sK, &tmK, &bars[0], 0, t0 - a.L, bh);
    tc::tma_load_3d(sV, &tmV, &bars[0], 0, t0 - a.L, bh);
  }
  // delta_t = dO_t . O_t  (O from global, dO from the swizzled smem tile once it lands)
  float orow[kD];
  {
    const bf16* op = a.Og + ((long long)bh * T + (row_ok ? t : 0)) * kD;
    load_vec<kD>(orow, op);
  }
  const float lse2 = (row_ok ? a.LSEin[(long long)bh * T + t] : 0.f) * kLog2e;
  tc::mbar_wait(&bars[0], 0);
  float delta = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 raw = *reinterpret_cast<const uint4*>(sdO + r * 128 + ((c ^ (r & 7)) * 16));  // 128B swizzle
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      delta = fmaf(f.x, orow[8 * c + 2 * e], delta);
      delta = fmaf(f.y, orow[8 * c + 2 * e + 1], delta);
    }
  }
  if (row_ok) a.delta[(long long)bh * T + t] = delta;

  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, NK, 0, 0);
#pragma unroll
    for (int k = 0; k < kD / 16; ++k)
      tc::mma_bf16(tbase, tc::desc_kmajor_sw128(tc::smem_u32(sQ) + 32 * k),
                   tc::desc_kmajor_sw128(tc::smem_u32(sK) + 32 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 0);
  __syncwarp();
  tc::tc_fence_after();
  float p[CW];
  tmem_row_strip<CW>(tbase, w, p);
  tc::tmem_ld_wait();
  const int key0 = t0 - a.L + 32 * w;
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    const int f = key0 + i;
    const bool v = i >= lane && i < lane + W && f >= 0 && f < T;
    p[i] = v ? exp2f(p[i] * a.scale_log2 - lse2) : 0.f;
  }
  tc::tc_fence_before();
  __syncthreads();                       // every warp has read S: its columns may be overwritten
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, NK, 0, 0);
#pragma unroll
    for (int k = 0; k < kD / 16; ++k)
      tc::mma_bf16(tbase, tc::desc_kmajor_sw128(tc::smem_u32(sdO) + 32 * k),
                   tc::desc_kmajor_sw128(tc::smem_u32(sV) + 32 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 1);
  __syncwarp();
  tc::tc_fence_after();
  {
    const uint32_t a0 = lanebase + uint32_t(32 * w);
#pragma unroll
    for (int j = 0; j < CW / 8; ++j) {
      float dp[8];
      tc::tmem_ld8(a0 + 8 * j, dp);
      tc::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) p[8 * j + e] = p[8 * j + e] * (dp[e] - delta);
    }
  }
  // dS -> smem (aliases the consumed Q / dO tiles: both MMAs have completed)
  write_row_interleave<CW, NK>(sdS, r, w, p);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, kD, 0, 1);
    constexpr uint32_t SBO = (NK / 8) * 128;
#pragma unroll
    for (int k = 0; k < NK / 16; ++k)
      tc::mma_bf16(tbase + QCOL, tc::desc_kmajor_interleave(tc::smem_u32(sdS) + 256 * k, SBO),
                   tc::desc_mnmajor_sw128(tc::smem_u32(sK) + 2048 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 0);
  __syncwarp();
  tc::tc_fence_after();
  tmem_row64_to_global(lanebase + QCOL, a.scale, a.dQ + ((long long)bh * T + (row_ok ? t : 0)) * kD, row_ok);
  tc::tc_fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tbase, TCOLS);
}

// ------------------------------------------------------------------------------------------
// backward K2: dK, dV (key-major)
// ------------------------------------------------------------------------------------------
template <int CW>
__global__ void __launch_bounds__(kThreads, 1)
    sa_bwd_dkdv_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, TcArgs a) {
  constexpr int NQ = nk_of(CW);
  constexpr int TCOLS = tmem_cols_of(NQ);
  constexpr int R0 = (2 * kM * 128 > kM * NQ * 2) ? 2 * kM * 128 : kM * NQ * 2;  // [K | V] aliased by P^T / dS^T
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + kM * 128;
  uint8_t* sX = smem;                                  // P^T then dS^T
  uint8_t* sQ = smem + ((R0 + 1023) & ~1023);
  uint8_t* sdO = sQ + NQ * 128;
  float* sL2 = reinterpret_cast<float*>(sdO + NQ * 128);
  float* sDel = sL2 + NQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDel + NQ);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int u0 = blockIdx.x * kM, bh = blockIdx.y;
  const int T = a.T, W = a.L + a.R + 1;
  const int r = 32 * w + lane, u = u0 + r;
  const bool row_ok = u < T;
  const int n0 = u0 - a.R;  // query frame of column 0

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO);
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_mbar_init();
  }
  if (w == 0) tc::tmem_alloc(tslot, TCOLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t lanebase = tbase + (uint32_t(32 * w) << 16);

  if (tid == 0) {
    tc::mbar_expect_tx(&bars[0], 2 * kM * 128 + 2 * NQ * 128);
    tc::tma_load_3d(sK, &tmK, &bars[0], 0, u0, bh);
    tc::tma_load_3d(sV, &tmV, &bars[0], 0, u0, bh);
    tc::tma_load_3d(sQ, &tmQ, &bars[0], 0, n0, bh);
    tc::tma_load_3d(sdO, &tmdO, &bars[0], 0, n0, bh);
  }
  for (int j = tid; j < NQ; j += kThreads) {
    const int n = n0 + j;
    const bool ok = n >= 0 && n < T;
    sL2[j] = ok ? a.LSEin[(long long)bh * T + n] * kLog2e : __int_as_float(0x7f800000);
    sDel[j] = ok ? a.delta[(long long)bh * T + n] : 0.f;
  }
  __syncthreads();
  if (tid == 0) {
    tc::mbar_wait(&bars[0], 0);
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, NQ, 0, 0);
#pragma unroll
    for (int k = 0; k < kD / 16; ++k)
      tc::mma_bf16(tbase, tc::desc_kmajor_sw128(tc::smem_u32(sK) + 32 * k),
                   tc::desc_kmajor_sw128(tc::smem_u32(sQ) + 32 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 0);
  __syncwarp();
  tc::tc_fence_after();
  float p[CW];
  tmem_row_strip<CW>(tbase, w, p);
  tc::tmem_ld_wait();
  const int c0 = 32 * w;  // column of register 0
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    const bool v = i >= lane && i < lane + W;   // query n in [u - R, u + L]
    p[i] = v ? exp2f(p[i] * a.scale_log2 - sL2[c0 + i]) : 0.f;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, NQ, 0, 0);
#pragma unroll
    for (int k = 0; k < kD / 16; ++k)
      tc::mma_bf16(tbase, tc::desc_kmajor_sw128(tc::smem_u32(sV) + 32 * k),
                   tc::desc_kmajor_sw128(tc::smem_u32(sdO) + 32 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 1);
  __syncwarp();
  tc::tc_fence_after();
  float ds[CW];
  {
    const uint32_t a0 = lanebase + uint32_t(32 * w);
#pragma unroll
    for (int j = 0; j < CW / 8; ++j) {
      float dp[8];
      tc::tmem_ld8(a0 + 8 * j, dp);
      tc::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) ds[8 * j + e] = p[8 * j + e] * (dp[e] - sDel[c0 + 8 * j + e]);
    }
  }
  // P^T -> smem (aliases the consumed K / V tiles), dV = P^T dO
  write_row_interleave<CW, NQ>(sX, r, w, p);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  constexpr uint32_t SBO = (NQ / 8) * 128;
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, kD, 0, 1);
#pragma unroll
    for (int k = 0; k < NQ / 16; ++k)
      tc::mma_bf16(tbase + 0, tc::desc_kmajor_interleave(tc::smem_u32(sX) + 256 * k, SBO),
                   tc::desc_mnmajor_sw128(tc::smem_u32(sdO) + 2048 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 0);
  // dS^T -> smem (the dV MMA has finished reading P^T), dK = dS^T Q
  write_row_interleave<CW, NQ>(sX, r, w, ds);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc::tc_fence_after();
    constexpr uint32_t id = tc::idesc_bf16(kM, kD, 0, 1);
#pragma unroll
    for (int k = 0; k < NQ / 16; ++k)
      tc::mma_bf16(tbase + 64, tc::desc_kmajor_interleave(tc::smem_u32(sX) + 256 * k, SBO),
                   tc::desc_mnmajor_sw128(tc::smem_u32(sQ) + 2048 * k), id, k > 0);
    tc::mma_commit(&bars[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bars[1], 1);
  __syncwarp();
  tc::tc_fence_after();
  const long long off = ((long long)bh * T + (row_ok ? u : 0)) * kD;
  tmem_row64_to_global(lanebase + 0, 1.f, a.dV + off, row_ok);
  tmem_row64_to_global(lanebase + 64, a.scale, a.dK + off, row_ok);
  tc::tc_fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tbase, TCOLS);
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// [BH][T][64] bf16 viewed as a 3-D tensor (64, T, BH); box (64, rows, 1), 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, int T, int BH, int rows) {
  EncodeTiledFn enc = encoder();
  if (!enc) {
    g_tc_err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)BH};
  cuuint64_t strides[2] = {64 * 2, (cuuint64_t)T * 64 * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

int cw_of(int W) {
  const int need = W + 31;
  const int opts[] = {32, 48, 64, 72, 80, 96, 112, 128, 160};
  for (int c : opts)
    if (c >= need) return c;
  return -1;
}

template <int CW> size_t fwd_smem() { return 1024 + kM * 128 + 2 * nk_of(CW) * 128 + kM * nk_of(CW) * 2 + 64; }
template <int CW> size_t dq_smem() {
  constexpr int NK = nk_of(CW);
  constexpr int R0 = (2 * kM * 128 > kM * NK * 2) ? 2 * kM * 128 : kM * NK * 2;
  return 1024 + ((R0 + 1023) & ~1023) + 2 * NK * 128 + 64;
}
template <int CW> size_t dkdv_smem() {
  constexpr int NQ = nk_of(CW);
  constexpr int R0 = (2 * kM * 128 > kM * NQ * 2) ? 2 * kM * 128 : kM * NQ * 2;
  return 1024 + ((R0 + 1023) & ~1023) + 2 * NQ * 128 + 2 * NQ * 4 + 64;
}

TcArgs tc_args(const AttnArgs& a) {
  TcArgs t{};
  t.T = a.T; t.L = a.L; t.R = a.R; t.BH = a.BH;
  t.scale = a.scale; t.scale_log2 = a.scale_log2;
  t.O = reinterpret_cast<bf16*>(a.Out); t.LSE = a.LSEout;
  t.Og = reinterpret_cast<const bf16*>(a.O); t.LSEin = a.LSE;
  t.dQ = reinterpret_cast<bf16*>(a.dQ); t.dK = reinterpret_cast<bf16*>(a.dK); t.dV = reinterpret_cast<bf16*>(a.dV);
  t.delta = a.delta;
  return t;
}

template <int CW>
sattn_status fwd_launch(const AttnArgs& a, cudaStream_t st) {
  constexpr int NK = nk_of(CW);
  CUtensorMap mq, mk, mv;
  if (!make_map(&mq, a.Q, a.T, a.BH, kM) || !make_map(&mk, a.K, a.T, a.BH, NK) || !make_map(&mv, a.V, a.T, a.BH, NK))
    return SATTN_ECUDA;
  const size_t smem = fwd_smem<CW>();
  cudaFuncSetAttribute(sa_fwd_tc<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((a.T + kM - 1) / kM, a.BH);
  sa_fwd_tc<CW><<<grid, kThreads, smem, st>>>(mq, mk, mv, tc_args(a));
  return SATTN_OK;
}

template <int CW>
sattn_status bwd_launch(const AttnArgs& a, cudaStream_t st) {
  constexpr int NK = nk_of(CW);
  CUtensorMap mq, mk, mv, mdo, mqN, mdoN, mk128, mv128;
  if (!make_map(&mq, a.Q, a.T, a.BH, kM) || !make_map(&mk, a.K, a.T, a.BH, NK) || !make_map(&mv, a.V, a.T, a.BH, NK) ||
      !make_map(&mdo, a.dO, a.T, a.BH, kM) || !make_map(&mqN, a.Q, a.T, a.BH, NK) ||
      !make_map(&mdoN, a.dO, a.T, a.BH, NK) || !make_map(&mk128, a.K, a.T, a.BH, kM) ||
      !make_map(&mv128, a.V, a.T, a.BH, kM))
    return SATTN_ECUDA;
  dim3 grid((a.T + kM - 1) / kM, a.BH);
  const size_t s1 = dq_smem<CW>();
  cudaFuncSetAttribute(sa_bwd_dq_tc<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  sa_bwd_dq_tc<CW><<<grid, kThreads, s1, st>>>(mq, mk, mv, mdo, tc_args(a));
  const size_t s2 = dkdv_smem<CW>();
  cudaFuncSetAttribute(sa_bwd_dkdv_tc<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  sa_bwd_dkdv_tc<CW><<<grid, kThreads, s2, st>>>(mqN, mk128, mv128, mdoN, tc_args(a));
  return SATTN_OK;
}

}  // namespace

bool tc_supported(int dtype, int D, int L, int R, bool llsa) {
  if (llsa || dtype != SATTN_BF16 || D != 64) return false;
  const int W = L + R + 1;
  return W + 31 <= 96;  // backward register budget (p and dS strips); DESIGN.md §5
}

sattn_status tc_forward(const AttnArgs& a, cudaStream_t st) {
  switch (cw_of(a.L + a.R + 1)) {
    case 32: return fwd_launch<32>(a, st);
    case 48: return fwd_launch<48>(a, st);
    case 64: return fwd_launch<64>(a, st);
    case 72: return fwd_launch<72>(a, st);
    case 80: return fwd_launch<80>(a, st);
    case 96: return fwd_launch<96>(a, st);
  }
  g_tc_err = "band too wide for the tensor-core kernels";
  return SATTN_EUNSUPPORTED;
}

sattn_status tc_backward(const AttnArgs& a, cudaStream_t st) {
  switch (cw_of(a.L + a.R + 1)) {
    case 32: return bwd_launch<32>(a, st);
    case 48: return bwd_launch<48>(a, st);
    case 64: return bwd_launch<64>(a, st);
    case 72: return bwd_launch<72>(a, st);
    case 80: return bwd_launch<80>(a, st);
    case 96: return bwd_launch<96>(a, st);
  }
  g_tc_err = "band too wide for the tensor-core kernels";
  return SATTN_EUNSUPPORTED;
}

int tc_backward_launches() { return 2; }
const char* tc_last_error() { return g_tc_err.c_str(); }

}  // namespace sattn
