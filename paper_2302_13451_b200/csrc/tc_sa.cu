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
//  backward K1 (sa_bwd_dq_tc, query-major):  S = Q K^T -> P = exp(S - LSE);
//                          dP = dO V^T (same TMEM columns) -> delta = rowsum(P o dP)
//                          (G26: not dO . O, so the bf16 rounding of O never enters) ->
//                          dS = P (dP - delta); dQ = scale dS K.
//  backward K2 (sa_bwd_dkdv_tc, key-major):   S^T = K Q^T -> P^T; dP^T = V dO^T ->
//                          dS^T; dV = P^T dO; dK = scale dS^T Q.
// No atomics: every output row is produced by one thread of one CTA -> bitwise
// deterministic (G18).  Operand layouts: TMA tiles are 128-byte rows with the
// 128B swizzle (K-major for Q/K/V/dO as the head-dim-contracted operand, the same
// bytes read MN-major when the frame index is the contraction); thread-written
// P / dS tiles use the no-swizzle 8x16B core-matrix layout.
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>
#include <string>

#include "ffma_attn.cuh"
#include "llsa_stair.cuh"
#include "tc_dispatch.h"
#include "tc_ptx.cuh"
#include "host_util.h"

namespace sattn {
namespace {
namespace cg = cooperative_groups;

thread_local std::string g_tc_err;
long long* g_trace = nullptr;  // debug: device buffer [8][64] for CTA 0 phase timestamps
constexpr int kD = 64;
constexpr int kM = 128;          // rows per CTA tile

__host__ __device__ constexpr int nk_of(int CW) { return ((96 + CW) + 15) / 16 * 16; }

struct TcArgs {
  int T, L, R, BH;
  int Tp;                                        // T rounded up to 4: row stride of the padded
                                                 // delta / LSE*log2e workspace rows (16-byte TMA rows)
  float scale, scale_log2;
  bf16* O; float* LSE;                           // fwd outputs
  const bf16* Og; const float* LSEin;           // bwd inputs
  bf16* dQ; bf16* dK; bf16* dV; float* delta;    // bwd outputs
  long long* trace;                              // optional per-phase clock64 trace of CTA 0 (debug)
  int kshift;                                    // keys of query t are frames [t-L-kshift, t+R-kshift]
                                                 // (0 for SA; R-c for LLSA channel c's band, with R := 0)
  float* ws_del; float* ws_l2;                   // padded [BH][Tp] delta / LSE*log2e rows (K1 -> K2)
  const float* ws_dx;                            // padded [BH][Tp] rowsum(P o dP) over slots outside the
                                                 // band (LLSA staircase, from the stair pre-pass); null for SA
  int dq_split;                                  // K1: dQ MMA on bf16 dS hi + lo (LLSA, whose dQ is rounded twice)
  int nch;                                       // K1: channels in one launch (LLSA band pass: C; SA: 1)
  int bcast;                                     // K1: Q is one plane read as every channel (LLSA layer 1)
  int ldp;                                       // stored-band mode: row stride of P [BH][T][ldp] (bf16)
  int ld;                                        // row stride (frames) of the caller's [BH][ld] LSE rows and
                                                 // [BH][ld][64] tensors (= T, or the margined length of a
                                                 // time shard, whose maps start at a row offset)
  // query tiles of this launch per head: kt = kt0 + i + (i >= kt_split ? kt_jump : 0), i < nkt
  // (all tiles: kt0 = 0, nkt = ceil(T/128); a time shard launches interior and edge tiles apart)
  int nkt, kt0, kt_split, kt_jump;
  int Th;                                        // frames per head: row t attends only inside its head
                                                 // [t - t % Th, + Th) (= T, or the head length when a
                                                 // launch packs tiles over the flattened BH*T axis)
  // wide bands (W > 65) as sub-bands of the narrow kernels, accumulated in fp32 (ACC instances):
  // forward (o, m, l) rows merged by log-sum-exp; K1 dQ / K2 dK, dV rows summed; K1 reads the
  // global delta = dO . O from ws_del instead of forming it over its sub-band (G28)
  float *acc_o, *acc_m, *acc_l;                  // [BH][T][64], [BH][T], [BH][T]
  float *acc_dq, *acc_dk, *acc_dv;               // [BH][T][64]
  int acc_first;                                 // first sub-band: store instead of merge / add
};

// r += s * v (or r = s * v when first) for one 64-float fp32 row in global memory
__device__ __forceinline__ void acc_row64(float* row, const float* v, float s, bool first) {
  float4* d = reinterpret_cast<float4*>(row);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    float4 x = first ? make_float4(0.f, 0.f, 0.f, 0.f) : d[c];
    x.x = fmaf(v[4 * c], s, x.x); x.y = fmaf(v[4 * c + 1], s, x.y);
    x.z = fmaf(v[4 * c + 2], s, x.z); x.w = fmaf(v[4 * c + 3], s, x.w);
    d[c] = x;
  }
}

__device__ __forceinline__ int tile_t0(int i, const TcArgs& a) {
  return (a.kt0 + i + (i >= a.kt_split ? a.kt_jump : 0)) * 128;
}

__device__ __forceinline__ void trace_at(long long* tr, int ev, int k) {
  if (tr && blockIdx.x == 0 && k < 64) tr[ev * 64 + k] = clock64();
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// per-CTA [start, end] globaltimer stamps at tr[1024 + 2*cta] (debug); phase events at tr[ev*64 + k], ev < 16
__device__ __forceinline__ void trace_cta(long long* tr, int which) {
  if (tr && threadIdx.x == 0 && blockIdx.x < 256) tr[1024 + 2 * blockIdx.x + which] = gtimer();
}

// ------------------------------------------------------------------------------------------
// forward: persistent, warp-specialised.  One CTA per SM loops over 128-row tiles.
//   warp 0      TMA producer   (Q, K of tile k into QK stage k % NQK)
//   warp 1      MMA issuer     (S(k+1) = Q K^T issued before O(k) = P V, so the tensor
//                               core works on the next tile while softmax runs) and the
//                               V loads: V(k) is fetched into V stage k % NV only once S(k-1)
//                               is issued, so a V stage is held ~TMA latency + softmax, not
//                               for the tile's whole life (more tiles in flight per smem byte)
//   warps 2..9  two softmax + epilogue warpgroups (row r = 32 * (warp % 4) + lane = TMEM lane r)
// TMEM: two buffers of 256 columns (S in [0, NK), O in [NK, NK + 64)); smem: NQK stages of
// Q/K, NV stages of V, two O staging tiles.  mbarriers: full/empty per stage, sfull/ofull/
// pfull/tfree per TMEM buffer.
// ------------------------------------------------------------------------------------------
template <int CW, bool PST = false> struct FwdCfg {
  static constexpr int NK = nk_of(CW);
  static constexpr int QB = kM * 128;
  static constexpr int KB = NK * 128;
  static constexpr int STAGE = QB + 2 * KB;
  static constexpr int QKB = QB + KB;                       // Q/K stage (1024-aligned)
  static constexpr int OB = kM * 128;                       // O staging tile for the TMA store
  // stored-band mode: the band rows go through the O staging tile (a separate band tile would
  // cost a V stage: measured 24.2 vs 22.5 us)
  static constexpr int PSB = 0;
  static constexpr int fits(int nqk, int nv) { return 1024 + nqk * QKB + nv * KB + 2 * OB + 2 * PSB + 256 <= 232448; }
  static constexpr int NQK = fits(3, 3) || fits(3, 2) ? 3 : 2;
  static constexpr int NV = fits(3, 3) ? 3 : 2;
  static constexpr int NS = NQK;
  static constexpr int SMEM = 1024 + NQK * QKB + NV * KB + 2 * OB + 2 * PSB + 256;
  static constexpr int THREADS = 320;   // TMA warp, MMA warp, 2 softmax warpgroups
};

// Softmax of one thread's row strip s[0..CW) (register i <-> key frame key0 + i), valid
// for i in [lo, hi); returns (row max, row sum) and leaves exp2((s - max) * sl2) in s.
template <int CW>
__device__ __forceinline__ void band_softmax(float* s, int lo, int hi, float sl2, float& m_out, float& l_out) {
  float m = neg_inf();
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    s[i] = (i >= lo && i < hi) ? s[i] : neg_inf();
    m = fmaxf(m, s[i]);
  }
  const float mref = m == neg_inf() ? 0.f : m;
  const float mb = mref * sl2;
  float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    s[i] = tc::ex2(fmaf(s[i], sl2, -mb));
    l4[i & 3] += s[i];
  }
  m_out = mref;
  l_out = (l4[0] + l4[1]) + (l4[2] + l4[3]);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Write a thread's bf16 row of an A operand held in TMEM (K-major: lane = row, packed
// column c = elements 2c, 2c+1): the strip s[0..CW) at elements [32*q4, 32*q4 + CW),
// zeros for the rest of [0, NK).  `pa` = TMEM address of (this warp's lane 0, column 0).
// x - bf16(x): the rounding residual, itself rounded to bf16 (x ~= hi + lo to ~2^-17 relative)
__device__ __forceinline__ float bf16_resid(float x) { return x - __bfloat162float(__float2bfloat16_rn(x)); }

template <int CW, int NK, bool LO = false>
__device__ __forceinline__ void tmem_write_row(uint32_t pa, int q4, const float* s) {
  const int c0 = 16 * q4;
#pragma unroll
  for (int j = 0; j < CW / 8; ++j) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = LO ? bf16_resid(s[8 * j + e]) : s[8 * j + e];
    tc::tmem_st4(pa + c0 + 4 * j, pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                 pack_bf16(v[6], v[7]));
  }
  for (int c = 0; c < NK / 2; c += 4)
    if (c < c0 || c >= c0 + CW / 2) tc::tmem_st4(pa + c, 0u, 0u, 0u, 0u);
}

// 64 fp32 values of row r (registers) -> scaled bf16 -> row r of a 128-row x 128-byte tile (128B swizzle)
__device__ __forceinline__ void tmem_row64_to_smem_sw128_regs(const float* v, float sc, uint8_t* tile, int r) {
  const uint32_t row = tc::smem_u32(tile) + r * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    tc::st_shared_v4(row + ((c ^ (r & 7)) << 4),
                     make_uint4(pack_bf16(v[8 * c] * sc, v[8 * c + 1] * sc), pack_bf16(v[8 * c + 2] * sc, v[8 * c + 3] * sc),
                                pack_bf16(v[8 * c + 4] * sc, v[8 * c + 5] * sc), pack_bf16(v[8 * c + 6] * sc, v[8 * c + 7] * sc)));
}

// 64 fp32 TMEM columns of this thread's row -> scaled bf16 -> row r of a 128-row x 128-byte
// smem tile with the 128B swizzle (the layout a SWIZZLE_128B TMA store expects).
__device__ __forceinline__ void tmem_row64_to_smem_sw128(uint32_t taddr, float sc, uint8_t* tile, int r) {
  float v[64];
#pragma unroll
  for (int j = 0; j < 4; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
  tc::tmem_ld_wait();
  const uint32_t row = tc::smem_u32(tile) + r * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    tc::st_shared_v4(row + ((c ^ (r & 7)) << 4),
                     make_uint4(pack_bf16(v[8 * c] * sc, v[8 * c + 1] * sc), pack_bf16(v[8 * c + 2] * sc, v[8 * c + 3] * sc),
                                pack_bf16(v[8 * c + 4] * sc, v[8 * c + 5] * sc), pack_bf16(v[8 * c + 6] * sc, v[8 * c + 7] * sc)));
}

// PST: the stored-band mode (NEXT-4) -- the softmax warpgroup also writes its row of
// a_t (bf16, band layout [BH][T][ldp], zeros outside the clipped window) through the O staging
// tile and a TMA store (tmP: box (ldp, 128, 1)) before the O epilogue.
template <int CW, bool PST = false, bool ACC = false>
__global__ void __launch_bounds__(320, 1)
    sa_fwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
              const __grid_constant__ CUtensorMap tmP, TcArgs a) {
  using C = FwdCfg<CW, PST>;
  constexpr int NK = C::NK, NQK = C::NQK, NV = C::NV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qk0 = smem;                          // [Q | K] x NQK
  uint8_t* v0 = qk0 + NQK * C::QKB;             // V x NV
  uint8_t* obuf0 = v0 + NV * C::KB;
  uint8_t* pbuf0 = obuf0 + 2 * C::OB;           // PST: band staging x 2
  uint64_t* bars = reinterpret_cast<uint64_t*>(pbuf0 + 2 * C::PSB);
  uint64_t* full = bars;            // [NQK] Q/K landed
  uint64_t* empty = full + NQK;     // [NQK] Q/K stage free (S issued and done)
  uint64_t* vfull = empty + NQK;    // [NV]
  uint64_t* vempty = vfull + NV;    // [NV]
  uint64_t* sfull = vempty + NV;    // [2]
  uint64_t* ofull = sfull + 2;      // [2]
  uint64_t* pfull = ofull + 2;      // [2]
  uint64_t* tfree = pfull + 2;      // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, W = a.L + a.R + 1;
  const int ntq = a.nkt;
  const int ntiles = ntq * a.BH;
  const int ntile_me = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  trace_cta(a.trace, 0);

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmK);
    tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmO);
    for (int i = 0; i < NQK; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    for (int i = 0; i < NV; ++i) { tc::mbar_init(&vfull[i], 1); tc::mbar_init(&vempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&ofull[i], 1);
      tc::mbar_init(&pfull[i], 128); tc::mbar_init(&tfree[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // L2 prefetch of the first tiles' boxes while the previous kernel drains (PDL): safe whether or
  // not that kernel writes them (L2 is coherent; only the shared-memory loads must wait)
  if (tid == 0)
    for (int k = 0; k < ntile_me && k < NQK; ++k) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
      tc::tma_prefetch_3d(&tmQ, 0, t0, bh);
      tc::tma_prefetch_3d(&tmK, 0, t0 - a.L, bh);
      tc::tma_prefetch_3d(&tmV, 0, t0 - a.L, bh);
    }
  // everything above overlapped the previous kernel's tail (PDL); its outputs are visible after this
  tc::pdl_wait();
  tc::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < ntile_me; ++k) {
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
        const int st = k % NQK;
        if (k >= NQK) tc::mbar_wait(&empty[st], ((k - NQK) / NQK) & 1);
        uint8_t* sQ = qk0 + st * C::QKB;
        trace_at(a.trace, 0, k);
        tc::mbar_expect_tx(&full[st], C::QKB);
        tc::tma_load_3d(sQ, &tmQ, &full[st], 0, t0, bh);
        tc::tma_load_3d(sQ + C::QB, &tmK, &full[st], 0, t0 - a.L, bh);
        // V(k) into its own ring: the stage frees when PV(k - NV) completes
        const int sv = k % NV;
        if (k >= NV) tc::mbar_wait(&vempty[sv], ((k - NV) / NV) & 1);
        trace_at(a.trace, 9, k);
        tc::mbar_expect_tx(&vfull[sv], C::KB);
        tc::tma_load_3d(v0 + sv * C::KB, &tmV, &vfull[sv], 0, t0 - a.L, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && ntile_me > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(kM, NK, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(kM, kD, 0, 1);
      // Out-of-order issue: S(k) as soon as its stage has landed and TMEM buffer k&1 is free
      // (PV(k-2) issued: tcgen05 ops of one thread execute in issue order, so PV(k-2) reads
      // P(k-2) before S(k) overwrites those columns); PV(k) as soon as softmax(k) has written
      // P(k) and the epilogue of tile k-2 has drained O.  Neither waits behind the other.
      // In-order schedule with blocking waits (mbarrier.try_wait sleeps and wakes ~60 cycles after
      // the arrive; a polling loop pays ~150 cycles per probe):  S(0) S(1) | PV(0) S(2) | PV(1) S(3) ...
      // PV(k) needs P(k) (softmax), the epilogue of tile k-2 (O columns) and V(k); S(k+2) reuses
      // TMEM buffer k&1, whose P(k) the just-issued PV(k) reads first (tcgen05 ops of one thread
      // execute in issue order).
      auto issue_s = [&](int k) {
        tc::mbar_wait(&full[k % NQK], (k / NQK) & 1);
        trace_at(a.trace, 1, k);
        tc::tc_fence_after();
        const uint32_t q = tc::smem_u32(qk0 + (k % NQK) * C::QKB), kk = q + C::QB;
        const uint32_t d = tbase + (k & 1) * 256;
#pragma unroll
        for (int j = 0; j < kD / 16; ++j)
          tc::mma_bf16(d, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(kk + 32 * j), idS, j > 0);
        tc::mma_commit(&sfull[k & 1]);
        tc::mma_commit(&empty[k % NQK]);
        trace_at(a.trace, 2, k);
      };
      issue_s(0);
      if (ntile_me > 1) issue_s(1);
      for (int k = 0; k < ntile_me; ++k) {
        const int b = k & 1, st = k % NV;
        tc::mbar_wait(&pfull[b], (k >> 1) & 1);
        if (k >= 2) tc::mbar_wait(&tfree[b], ((k - 2) >> 1) & 1);
        tc::mbar_wait(&vfull[st], (k / NV) & 1);
        trace_at(a.trace, 3, k);
        tc::tc_fence_after();
        const uint32_t v = tc::smem_u32(v0 + st * C::KB);
        const uint32_t pa = tbase + b * 256;
#pragma unroll
        for (int j = 0; j < NK / 16; ++j)
          tc::mma_bf16_ts(pa + NK, pa + 8 * j, tc::desc_mnmajor_sw128(v + 2048 * j), idO, j > 0);
        tc::mma_commit(&ofull[b]);
        tc::mma_commit(&vempty[st]);
        trace_at(a.trace, 8, k);
        if (k + 2 < ntile_me) issue_s(k + 2);
      }
    }
  } else {
    // two softmax + epilogue warpgroups: warpgroup b = (warp - 2) / 4 owns tiles k with k & 1 == b
    // (TMEM buffer b, O staging tile b); row r = 32 * (warp % 4) + lane = TMEM lane r.
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = (warp & 3) == 2 && lane == 0;   // one thread per warpgroup
    const bool tr = (tid == 64) || (tid == 192);
    uint8_t* ostage = obuf0 + wg * C::OB;
    uint8_t* pstage = ostage;
    for (int k = wg; k < ntile_me; k += 2) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
      const int t = t0 + r;
      const int b = wg;
      const int use = k >> 1;
      tc::mbar_wait(&sfull[b], use & 1);
      if (tr) trace_at(a.trace, 4, k);
      __syncwarp();
      tc::tc_fence_after();
      float s[CW];
      const uint32_t pa = tbase + lanes + b * 256;
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(pa + 32 * q4 + 8 * j, s + 8 * j);
      tc::tmem_ld_wait();
      const int key0 = t0 - a.L + 32 * q4;
      const int hs = t - t % a.Th;              // this row's head: frames [hs, hs + Th)
      float m, l;
      band_softmax<CW>(s, max(lane, hs - key0), min(lane + W, hs + a.Th - key0), a.scale_log2, m, l);
      tmem_write_row<CW, NK>(pa, q4, s);      // P (bf16) over the consumed S columns
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pfull[b]);
      if (tr) trace_at(a.trace, 5, k);
      if constexpr (PST) {   // a_t row -> band staging row r (ld bf16) -> TMA store (rows >= T clipped)
        if (leader) tc::bulk_wait_read0();   // the O store of tile k - 2 has read the staging tile
        tc::named_bar(1 + wg, 128);
        const float inv = 1.f / l;
        const uint32_t prow = tc::smem_u32(pstage) + r * a.ldp * 2;
        // scalar stores (a paired 4-byte variant with odd/even lane selects measured 25.0 vs 22.5 us)
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int j = i - lane;   // band index of register i (zero outside [lo, hi) already)
          if (j >= 0 && j < W) tc::st_shared_u16(prow + 2 * j, __bfloat16_as_ushort(__float2bfloat16_rn(s[i] * inv)));
        }
        for (int j = W; j < a.ldp; ++j) tc::st_shared_u16(prow + 2 * j, 0);
        tc::fence_proxy_async_smem();
        tc::named_bar(1 + wg, 128);
        if (leader) {
          tc::tma_store_3d(&tmP, pstage, 0, t0, bh);
          tc::bulk_commit();
        }
      }
      // epilogue (the other warpgroup runs the next tile's softmax meanwhile)
      tc::mbar_wait(&ofull[b], use & 1);
      if (tr) trace_at(a.trace, 6, k);
      __syncwarp();
      tc::tc_fence_after();
      if constexpr (ACC) {
        // sub-band of a wide band: merge (o, m, l) into the fp32 accumulator rows (log-sum-exp)
        float v[64];
#pragma unroll
        for (int j = 0; j < 4; ++j) tc::tmem_ld16(pa + NK + 16 * j, v + 16 * j);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&tfree[b]);
        if (t < T) {
          const long long row = (long long)bh * T + t;
          const float mn = l > 0.f ? m : neg_inf();          // no valid key in this sub-band: weight 0
          const float mo = a.acc_first ? neg_inf() : a.acc_m[row];
          const float M = fmaxf(mo, mn);
          if (M != neg_inf()) {
            const float wo = a.acc_first ? 0.f : tc::ex2((mo - M) * a.scale_log2);
            const float wn = tc::ex2((mn - M) * a.scale_log2);
            float4* d = reinterpret_cast<float4*>(a.acc_o + row * 64);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              float4 x = a.acc_first ? make_float4(0.f, 0.f, 0.f, 0.f) : d[c];
              x.x = fmaf(v[4 * c], wn, x.x * wo); x.y = fmaf(v[4 * c + 1], wn, x.y * wo);
              x.z = fmaf(v[4 * c + 2], wn, x.z * wo); x.w = fmaf(v[4 * c + 3], wn, x.w * wo);
              d[c] = x;
            }
            a.acc_l[row] = (a.acc_first ? 0.f : a.acc_l[row] * wo) + l * wn;
            a.acc_m[row] = M;
          } else if (a.acc_first) {
            a.acc_m[row] = neg_inf();
            a.acc_l[row] = 0.f;
          }
        }
        if (tr) trace_at(a.trace, 7, k);
        continue;
      }
      if (leader) tc::bulk_wait_read0();        // the previous TMA store has read the staging tile
      tc::named_bar(1 + wg, 128);
      tmem_row64_to_smem_sw128(pa + NK, 1.f / l, ostage, r);
      tc::tc_fence_before();
      tc::mbar_arrive(&tfree[b]);
      if (t < T) a.LSE[(long long)bh * a.ld + t] = m * a.scale + __log2f(l) * kLn2;
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (leader) {
        tc::tma_store_3d(&tmO, ostage, 0, t0, bh);   // rows >= T are clipped by the tensor map
        tc::bulk_commit();
      }
      if (tr) trace_at(a.trace, 7, k);
    }
    if (leader) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
  trace_cta(a.trace, 1);
}

__device__ __forceinline__ float dot8_bf16(uint4 a, uint4 b) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&b);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 u = __bfloat1622float2(x[i]), v = __bfloat1622float2(y[i]);
    s = fmaf(u.x, v.x, s);
    s = fmaf(u.y, v.y, s);
  }
  return s;
}
// 64 fp32 of one row -> bf16 (x sc) -> 128 contiguous bytes in global memory
__device__ __forceinline__ void store_row_bf16(bf16* dst, const float* v, float sc) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    d[c] = make_uint4(pack_bf16(v[8 * c] * sc, v[8 * c + 1] * sc), pack_bf16(v[8 * c + 2] * sc, v[8 * c + 3] * sc),
                      pack_bf16(v[8 * c + 4] * sc, v[8 * c + 5] * sc), pack_bf16(v[8 * c + 6] * sc, v[8 * c + 7] * sc));
}
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) tc::tmem_ld16(taddr + 16 * j, v + 16 * j);
  tc::tmem_ld_wait();
}
// ------------------------------------------------------------------------------------------
// backward K1 (query-major): delta_t = sum_u P_tu dP_tu, dQ_t = scale * sum_u dS_tu K_u.
// Persistent, warp-specialised like the forward.  Per tile (128 queries, TMEM buffer b):
//   MMA  S = Q K^T -> X_b                      WG  P = exp2(S*sl2 - LSE*log2e)   (registers)
//   MMA  dP = dO V^T -> X_b (same columns)     WG  delta = rowsum(P dP) (+ ws_dx);
//                                                  dS = P (dP - delta) -> X_b as packed bf16
//   MMA  dQ = dS K -> Y_b (A = dS from TMEM)   WG  dQ * scale -> smem -> TMA store
// ------------------------------------------------------------------------------------------
template <int CW> struct DqCfg {
  static constexpr int NK = nk_of(CW);
  static constexpr int QB = kM * 128;
  static constexpr int KB = NK * 128;
  static constexpr int STAGE = 2 * QB + 2 * KB;   // Q, dO, K, V (1024-aligned: 128B-swizzle atoms)
  static constexpr int NS = 2;
  static constexpr int SMEM = 1024 + NS * STAGE + 2 * QB + 512;
  static constexpr int THREADS = 320;
};

// PST (stored-band mode): tmQ maps the band P [BH][T][ldp] (box (ldp, 128, 1)) and the tile's
// P rows are staged in the Q slot; no S MMA, no exponentials: the warpgroup reads P from smem.
template <int CW, bool PST = false, bool ACC = false>
__global__ void __launch_bounds__(320, 1)
    sa_bwd_dq_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                 const __grid_constant__ CUtensorMap tmdQ, TcArgs a) {
  using C = DqCfg<CW>;
  constexpr int NK = C::NK, NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage0 = smem;                       // [Q | dO | K | V] per stage
  uint8_t* obuf0 = smem + NS * C::STAGE;        // dQ staging, one per warpgroup
  uint64_t* bars = reinterpret_cast<uint64_t*>(obuf0 + 2 * C::QB);
  uint64_t* full = bars;              // [NS]
  uint64_t* empty = full + NS;        // [NS]
  uint64_t* sfull = empty + NS;       // [2]
  uint64_t* xfree = sfull + 2;        // [2] (128 arrivals)
  uint64_t* dpfull = xfree + 2;       // [2]
  uint64_t* dsfull = dpfull + 2;      // [2] (128)
  uint64_t* dqfull = dsfull + 2;      // [2]
  uint64_t* tfree = dqfull + 2;       // [2] (128)
  // the stage's K region has its own release barrier, so that Q or the band / dO / V (dead once dP
  // is issued and, PST, the warpgroup has read its band rows) are released before the dQ MMA
  // retires K; PST: K also lands on its own barrier (dP does not need it)
  uint64_t* fullK = tfree + 2;        // [NS]
  uint64_t* emptyK = fullK + NS;      // [NS]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(emptyK + NS);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, W = a.L + a.R + 1;
  const int ntq = a.nkt;
  // tiles: (channel c, head bh, query tile) with c slowest; SA has one channel.  LLSA runs every
  // channel's band pass in one launch: channel c's queries see channel-R keys shifted by R - c.
  const int nch = a.nch > 0 ? a.nch : 1;
  const int ntiles = ntq * a.BH * nch;
  const int ntile_me = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int tpc = ntq * a.BH;                            // tiles per channel

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmK); tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO); tc::tma_prefetch_desc(&tmdQ);
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], PST ? 1 + 128 : 1);
      tc::mbar_init(&fullK[i], 1); tc::mbar_init(&emptyK[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&xfree[i], 128); tc::mbar_init(&dpfull[i], 1);
      tc::mbar_init(&dsfull[i], 128); tc::mbar_init(&dqfull[i], 1); tc::mbar_init(&tfree[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // L2 prefetch of the first tiles' boxes while the previous kernel drains (PDL; see the forward)
  if (tid == 0 && nch == 1)
    for (int k = 0; k < ntile_me && k < NS; ++k) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
      tc::tma_prefetch_3d(&tmQ, 0, t0, bh);
      tc::tma_prefetch_3d(&tmdO, 0, t0, bh);
      tc::tma_prefetch_3d(&tmK, 0, t0 - a.L - a.kshift, bh);
      tc::tma_prefetch_3d(&tmV, 0, t0 - a.L - a.kshift, bh);
    }
  // everything above overlapped the previous kernel's tail (PDL); its outputs are visible after this
  tc::pdl_wait();
  tc::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < ntile_me; ++k) {
        const int g0 = blockIdx.x + k * gridDim.x;
        const int c = g0 / tpc, g = g0 % tpc;
        const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
        const int ksh = a.kshift - c;                    // LLSA: R - c (a.kshift = R); SA: 0
        const int st = k % NS;
        uint8_t* b0 = stage0 + st * C::STAGE;
        if (k >= NS) tc::mbar_wait(&empty[st], ((k - NS) / NS) & 1);
        if constexpr (PST) {
          tc::mbar_expect_tx(&full[st], kM * a.ldp * 2 + C::QB + C::KB);
          tc::tma_load_3d(b0, &tmQ, &full[st], 0, t0, bh);
          tc::tma_load_3d(b0 + C::QB, &tmdO, &full[st], 0, t0, bh);
          tc::tma_load_3d(b0 + 2 * C::QB + C::KB, &tmV, &full[st], 0, t0 - a.L - ksh, bh);
          if (k >= NS) tc::mbar_wait(&emptyK[st], ((k - NS) / NS) & 1);
          tc::mbar_expect_tx(&fullK[st], C::KB);
          tc::tma_load_3d(b0 + 2 * C::QB, &tmK, &fullK[st], 0, t0 - a.L - ksh, bh);
          continue;
        } else {
        // Q, dO, V are free once dP is issued (empty); K stays until dQ (emptyK).  S needs K too,
        // so everything lands on `full`, but the Q / dO / V loads no longer wait for the dQ MMA
        tc::mbar_expect_tx(&full[st], 2 * C::QB + 2 * C::KB);
        if (nch > 1) {   // LLSA: [C][BH][T][64] maps
          tc::tma_load_4d(b0, &tmQ, &full[st], 0, t0, bh, a.bcast ? 0 : c);
          tc::tma_load_4d(b0 + C::QB, &tmdO, &full[st], 0, t0, bh, c);
        } else {
          tc::tma_load_3d(b0, &tmQ, &full[st], 0, t0, bh);
          tc::tma_load_3d(b0 + C::QB, &tmdO, &full[st], 0, t0, bh);
        }
        tc::tma_load_3d(b0 + 2 * C::QB + C::KB, &tmV, &full[st], 0, t0 - a.L - ksh, bh);
        if (k >= NS) tc::mbar_wait(&emptyK[st], ((k - NS) / NS) & 1);
        tc::tma_load_3d(b0 + 2 * C::QB, &tmK, &full[st], 0, t0 - a.L - ksh, bh);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(kM, NK, 0, 0);
      constexpr uint32_t idQ = tc::idesc_bf16(kM, kD, 0, 1);
      int ns = 0, ndp = 0, ndq = 0;
      if constexpr (PST) ns = ntile_me;   // no S: dP(k) needs its stage and X_b free (dQ(k-2) issued)
      while (ndq < ntile_me) {
        const uint32_t m = PST ? tc::mbar_test4(tc::smem_u32(&dsfull[ndq & 1]), (ndq >> 1) & 1,
                                                tc::smem_u32(&tfree[ndq & 1]), ((ndq + 2) >> 1) & 1,
                                                tc::smem_u32(&full[ndp % NS]), (ndp / NS) & 1,
                                                tc::smem_u32(&fullK[ndq % NS]), (ndq / NS) & 1)
                               : tc::mbar_test4(tc::smem_u32(&dsfull[ndq & 1]), (ndq >> 1) & 1,
                                          tc::smem_u32(&tfree[ndq & 1]), ((ndq + 2) >> 1) & 1,   // = (ndq-2)>>1 parity
                                          tc::smem_u32(&xfree[ndp & 1]), (ndp >> 1) & 1,
                                          tc::smem_u32(&full[ns % NS]), (ns / NS) & 1);
        if (ndq < ndp && (m & 1) && (ndq < 2 || (m & 2)) && (!PST || (m & 8))) {
          tc::tc_fence_after();
          const int b = ndq & 1, st = ndq % NS;
          const uint32_t x = tbase + b * 256;
          const uint32_t kk = tc::smem_u32(stage0 + st * C::STAGE) + 2 * C::QB;
#pragma unroll
          for (int j = 0; j < NK / 16; ++j)
            tc::mma_bf16_ts(x + NK, x + 8 * j, tc::desc_mnmajor_sw128(kk + 2048 * j), idQ, j > 0);
          if (a.dq_split) {
#pragma unroll
            for (int j = 0; j < NK / 16; ++j)   // + dS_lo K
              tc::mma_bf16_ts(x + NK, x + NK / 2 + 8 * j, tc::desc_mnmajor_sw128(kk + 2048 * j), idQ, true);
          }
          tc::mma_commit(&dqfull[b]);
          tc::mma_commit(&emptyK[st]);
          ++ndq;
          continue;
        }
        if (ndp < ns && (m & 4) && (!PST || ndp < ndq + 2)) {
          tc::tc_fence_after();
          const int b = ndp & 1, st = ndp % NS;
          const uint32_t base = tc::smem_u32(stage0 + st * C::STAGE);
          const uint32_t dO = base + C::QB, v = base + 2 * C::QB + C::KB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(dO + 32 * j), tc::desc_kmajor_sw128(v + 32 * j), idS,
                         j > 0);
          tc::mma_commit(&dpfull[b]);
          tc::mma_commit(&empty[st]);   // Q (or the band) / dO / V: free once S and dP have read them
          ++ndp;
          continue;
        }
        if (!PST && ns < ntile_me && ns < ndq + 2 && (m & 8)) {
          tc::tc_fence_after();
          const int b = ns & 1;
          const uint32_t base = tc::smem_u32(stage0 + (ns % NS) * C::STAGE);
          const uint32_t q = base, kk = base + 2 * C::QB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(kk + 32 * j), idS,
                         j > 0);
          tc::mma_commit(&sfull[b]);
          ++ns;
          continue;
        }
      }
    }
  } else {
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = q4 == 2 && lane == 0;
    uint8_t* ostage = obuf0 + wg * C::QB;
    // LSE (and the staircase rowsum) of this warpgroup's next tile are loaded one tile ahead
    auto row_of = [&](int k, const float* src, int stride, float mul) -> float {
      if (k >= ntile_me || !src) return 0.f;
      const int g0 = blockIdx.x + k * gridDim.x;
      const int c = g0 / tpc, g = g0 % tpc;
      const int t = tile_t0(g % ntq, a) + r;
      return t < T ? src[((long long)c * a.BH + g / ntq) * stride + t] * mul : 0.f;
    };
    float lse_next = PST ? 0.f : row_of(wg, a.LSEin, a.ld, kLog2e), dx_next = row_of(wg, a.ws_dx, a.Tp, 1.f);
    for (int k = wg; k < ntile_me; k += 2) {
      const int g0 = blockIdx.x + k * gridDim.x;
      const int c = g0 / tpc, g = g0 % tpc;
      const int bh = g / ntq, t0 = tile_t0(g % ntq, a);
      const int ksh = a.kshift - c;
      const long long cbh = (long long)c * a.BH + bh;    // row of the [C][BH][Tp] workspaces
      const int t = t0 + r;
      const bool row_ok = t < T;
      const int b = wg, use = k >> 1;
      const float lse2 = lse_next, dx = dx_next;
      if (!PST) lse_next = row_of(k + 2, a.LSEin, a.ld, kLog2e);
      dx_next = row_of(k + 2, a.ws_dx, a.Tp, 1.f);
      const uint32_t x = tbase + lanes + b * 256;
      float p[CW];
      if constexpr (PST) {   // P from the staged band rows: register i <-> band index i - lane
        const int st = k % NS;
        tc::mbar_wait(&full[st], (k / NS) & 1);
        const uint32_t prow = tc::smem_u32(stage0 + st * C::STAGE) + r * a.ldp * 2;
        // band indices (j0, j0 + 1), j0 even, as one 4-byte load: registers (2m, 2m+1) for even
        // lanes, (2m+1, 2m+2) for odd lanes (the staged row is zero beyond W and outside [0, T))
        const bool odd = lane & 1;
        const int jb = -(lane & ~1);
        float nx = 0.f;   // odd lanes: the value for register 2m+2, carried to the next pair
#pragma unroll
        for (int m = 0; m < CW / 2; ++m) {
          const int j0 = 2 * m + jb;
          uint32_t w = 0;
          if (j0 >= 0 && j0 < W) w = tc::ld_shared_u32(prow + 2 * j0);
          const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
          if (odd) { p[2 * m] = nx; p[2 * m + 1] = lo; nx = hi; }
          else { p[2 * m] = lo; p[2 * m + 1] = hi; }
        }
        tc::mbar_arrive(&empty[st]);   // this row of the staged band has been read
      } else {
      // P from S
      tc::mbar_wait(&sfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + 32 * q4 + 8 * j, p + 8 * j);
      tc::tmem_ld_wait();
      const int key0 = t0 - a.L - ksh + 32 * q4;
      {
        const int hs = t - t % a.Th;
        const int lo = max(lane, hs - key0), hi = min(lane + W, hs + a.Th - key0);
#pragma unroll
        for (int i = 0; i < CW; ++i)
          p[i] = (i >= lo && i < hi) ? tc::ex2(fmaf(p[i], a.scale_log2, -lse2)) : 0.f;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      }
      // delta = rowsum(P o dP), then dS from dP
      tc::mbar_wait(&dpfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      // ACC (sub-band of a wide band): the global delta = dO . O, precomputed in ws_del
      float delta = ACC ? (row_ok ? a.ws_del[cbh * a.Tp + t] : 0.f) : dx;
      if constexpr (CW <= 72) {   // dP held in registers
        float dp[CW];
#pragma unroll
        for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + 32 * q4 + 8 * j, dp + 8 * j);
        tc::tmem_ld_wait();
#pragma unroll
        if constexpr (!ACC)
          for (int i = 0; i < CW; ++i) delta = fmaf(p[i], dp[i], delta);
#pragma unroll
        for (int i = 0; i < CW; ++i) p[i] *= dp[i] - delta;
      } else {                    // wide bands: read dP from TMEM twice instead of spilling
#pragma unroll
        for (int j = 0; j < CW / 8; ++j) {
          float dp[8];
          tc::tmem_ld8(x + 32 * q4 + 8 * j, dp);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e) delta = ACC ? delta : fmaf(p[8 * j + e], dp[e], delta);
        }
#pragma unroll
        for (int j = 0; j < CW / 8; ++j) {
          float dp[8];
          tc::tmem_ld8(x + 32 * q4 + 8 * j, dp);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e) p[8 * j + e] *= dp[e] - delta;
        }
      }
      // LLSA: dS as bf16 hi + lo (columns [0, NK/2) and [NK/2, NK), both dead fp32 S/dP by now):
      // the dQ MMA then sees dS to ~2^-17 instead of bf16's 2^-9 (G27: LLSA dQ is rounded twice)
      tmem_write_row<CW, NK>(x, q4, p);
      if (a.dq_split) tmem_write_row<CW, NK, true>(x + NK / 2, q4, p);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&dsfull[b]);
      // padded rows for K2's TMA loads; rows in [T, Tp) get zeros
      if (t < a.Tp) {
        if (!ACC) a.ws_del[cbh * a.Tp + t] = row_ok ? delta : 0.f;
        if (!PST) a.ws_l2[cbh * a.Tp + t] = row_ok ? lse2 : 0.f;
      }
      // dQ epilogue
      tc::mbar_wait(&dqfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      if constexpr (ACC) {
        float v[64];
        tmem_ld64(x + NK, v);
        tc::tc_fence_before();
        tc::mbar_arrive(&tfree[b]);
        if (row_ok) acc_row64(a.acc_dq + ((long long)bh * T + t) * 64, v, a.scale, a.acc_first);
        continue;
      }
      if (leader) tc::bulk_wait_read0();
      tc::named_bar(1 + wg, 128);
      tmem_row64_to_smem_sw128(x + NK, a.scale, ostage, r);
      tc::tc_fence_before();
      tc::mbar_arrive(&tfree[b]);
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (leader) {
        if (nch > 1) tc::tma_store_4d(&tmdQ, ostage, 0, t0, bh, c);
        else tc::tma_store_3d(&tmdQ, ostage, 0, t0, bh);
        tc::bulk_commit();
      }
    }
    if (leader) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// backward K2 (key-major): dV_u = sum_n P_nu dO_n, dK_u = scale * sum_n dS_nu Q_n.
// Per tile (128 keys u0.., queries u0-R .. u0-R+NQ), TMEM X_b double-buffered, dV/dK single:
//   MMA  S^T = K Q^T -> X_b                 WG  P^T = exp2(S^T*sl2 - LSE_n*log2e)
//   MMA  dP^T = V dO^T -> X_b               WG  dS^T = P^T (dP^T - delta_n); P^T, dS^T -> X_b packed
//   MMA  dV = P^T dO, dK = dS^T Q           WG  -> smem -> TMA stores
// ------------------------------------------------------------------------------------------
template <int CW> struct DkvCfg {
  static constexpr int NQ = nk_of(CW);
  static constexpr int KB = kM * 128;
  static constexpr int QB = NQ * 128;
  // K, V, Q, dO, LSE*log2e[NQ], delta[NQ]; 1024-aligned (128B-swizzle atoms)
  // LSE / delta boxes start at a 16-byte-aligned frame (u0 - R rounded down to a multiple of 4)
  // and are padded to 128 bytes: NQ + 3 frames at most are needed
  static constexpr int NQP = (NQ + 3 + 31) / 32 * 32;
  static constexpr int STAGE = (2 * KB + 2 * QB + 2 * NQP * 4 + 1023) / 1024 * 1024;
  static constexpr int NS = 2;
  static constexpr int SMEM = 1024 + NS * STAGE + 4 * KB + 512;
  static constexpr int THREADS = 320;
  // stored-band mode: [P window (NQ rows x PLD bf16) | V | Q | dO | delta] (no K, no LSE)
  static constexpr int PLD = ((CW - 31) + 7) / 8 * 8;
  static constexpr int PB = (NQ * PLD * 2 + 1023) / 1024 * 1024;
  static constexpr int STAGE_P = (PB + KB + 2 * QB + NQP * 4 + 1023) / 1024 * 1024;
  // the stored-band stage is two rings: A = [P window | V | delta] (2 slots, free once dP is
  // issued and dS formed), B = [Q | dO] (3 slots, free once dV / dK are stored: the dV / dK rows
  // are staged in the slot's dead Q / dO tiles, so there are no separate staging tiles)
  static constexpr int STAGE_A = (PB + KB + NQP * 4 + 1023) / 1024 * 1024;
  static constexpr int STAGE_B = 2 * QB;
  static constexpr int NSB = 3;
  static constexpr int SMEM_P = 1024 + NS * STAGE_A + NSB * STAGE_B + 512;
  static_assert(QB >= KB && QB % 1024 == 0, "dV / dK staging in the Q / dO tiles");
};

// PST (stored-band mode): tmK maps the band P [BH][T][ldp] with box (ldp, NQ, 1); the stage is
// [P window | V | Q | dO | delta]; no S MMA, no LSE, no exponentials: the warpgroup reads
// P^T[u][n] = P[n][u - n + L] from the staged rows.
template <int CW, bool PST = false, bool ACC = false>
__global__ void __launch_bounds__(320, 1)
    sa_bwd_dkdv_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                   const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
                   const __grid_constant__ CUtensorMap tmL2, const __grid_constant__ CUtensorMap tmDel, TcArgs a) {
  using C = DkvCfg<CW>;
  constexpr int NQ = C::NQ, NS = C::NS;
  constexpr int DVCOL = 176 <= 256 - 64 ? NQ : 0;   // dV after X_0, dK after X_1
  constexpr int STG = PST ? C::STAGE_A : C::STAGE;
  // PST: ring A [P window | V | delta]; ring B [Q | dO] (OFF_Q / OFF_DO relative to a B slot)
  constexpr int OFF_V = PST ? C::PB : C::KB, OFF_Q = PST ? 0 : OFF_V + C::KB, OFF_DO = OFF_Q + C::QB;
  constexpr int OFF_L2 = PST ? 0 : OFF_DO + C::QB, OFF_DEL = PST ? C::PB + C::KB : OFF_L2 + C::NQP * 4;
  constexpr int NSB = PST ? C::NSB : NS;
  static_assert(NQ + 64 <= 256, "TMEM layout needs NQ <= 192");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage0 = smem;                       // [K | V | Q | dO] (PST: ring A)
  uint8_t* stageB0 = smem + NS * STG;           // PST: ring B
  uint8_t* obuf0 = smem + NS * STG;             // per warpgroup: [dV | dK] staging (not PST)
  uint64_t* bars = reinterpret_cast<uint64_t*>(PST ? stageB0 + NSB * C::STAGE_B : obuf0 + 4 * C::KB);
  uint64_t* full = bars;              // [NS]
  uint64_t* empty = full + NS;        // [NS]
  uint64_t* sfull = empty + NS;       // [2]
  uint64_t* xfree = sfull + 2;        // [2] (128)
  uint64_t* dpfull = xfree + 2;       // [2]
  uint64_t* pdsfull = dpfull + 2;     // [2] (128)
  // dV/dK accumulators are single-buffered but their barriers are per warpgroup: a barrier
  // waited by alternating consumers could be passed a phase early (parity aliasing)
  uint64_t* kvfull = pdsfull + 2;     // [2]
  uint64_t* kvfree = kvfull + 2;      // [2] (128)
  uint64_t* dfull = kvfree + 2;       // [NS] PST: the stage's delta rows landed (K1's output)
  // PST: the stage's Q / dO region has its own barriers: the band window, V and delta (dead once
  // dP is issued and the warpgroup has formed dS) are released before dV / dK retire Q and dO
  uint64_t* fullB = dfull + NS;       // [NSB]
  uint64_t* emptyB = fullB + NSB;     // [NSB]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(emptyB + NSB);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, W = a.L + a.R + 1;
  const int ntq = (T + kM - 1) / kM;
  const int ntiles = ntq * a.BH;
  const int ntile_me = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // K2 walks the tiles in the reverse of K1's order: its first rounds re-read the V / dO / band
  // (or LSE-mode K / V / Q / dO) rows K1 streamed in its last rounds, still resident in L2

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmK); tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO); tc::tma_prefetch_desc(&tmdK); tc::tma_prefetch_desc(&tmdV);
    for (int i = 0; i < NS; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1 + 128); }
    for (int i = 0; i < NSB; ++i) { tc::mbar_init(&fullB[i], 1); tc::mbar_init(&emptyB[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&xfree[i], 128); tc::mbar_init(&dpfull[i], 1);
      tc::mbar_init(&pdsfull[i], 128);
    }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&kvfull[i], 1); tc::mbar_init(&kvfree[i], 128); }
    for (int i = 0; i < NS; ++i) tc::mbar_init(&dfull[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // everything above overlapped the previous kernel's tail (PDL); its outputs are visible after this
  // Only the workspace rows (delta; LSE*log2e in the LSE mode) come from the preceding kernel
  // (K1); K, V, Q, dO and the band were complete before K1 passed its own wait.  So the producer
  // loads those first and waits on K1 (PDL) only before the workspace rows, which land on their
  // own barrier (dfull): the first stages' loads and S / dP MMAs overlap K1's tail.  Safe because
  // K1 executes its griddepcontrol.wait before launch_dependents: K2 cannot start before every
  // kernel ahead of K1 (the forward that wrote P, whatever wrote dO) has completed.  (K1 itself
  // cannot do the same: its predecessor may be the forward that writes the band / LSE it reads.)
  tc::pdl_launch_dependents();
  const uint32_t DV = tbase + DVCOL, DK = tbase + 256 + DVCOL;

  if (warp == 0) {
    if (lane == 0) {
      int nd = 0;   // PST: next tile whose delta rows are to be loaded
      for (int k = 0; k < ntile_me; ++k) {
        const int g = ntiles - 1 - (blockIdx.x + k * gridDim.x);   // reversed order (below)
        const int bh = g / ntq, u0 = (g % ntq) * kM;
        const int st = k % NS;
        uint8_t* b0 = stage0 + st * STG;
        if (k >= NS) tc::mbar_wait(&empty[st], ((k - NS) / NS) & 1);
        trace_at(a.trace, 0, k);
        const int na = (u0 - a.R) & ~3;   // floor to a multiple of 4 (also for negatives)
        if constexpr (PST) {
          tc::mbar_expect_tx(&full[st], NQ * a.ldp * 2 + C::KB);
          tc::tma_load_3d(b0, &tmK, &full[st], 0, u0 - a.R, bh);   // P rows of the query window
          tc::tma_load_3d(b0 + OFF_V, &tmV, &full[st], 0, u0, bh);
          const int sb = k % NSB;
          uint8_t* bb = stageB0 + sb * C::STAGE_B;
          if (k >= NSB) tc::mbar_wait(&emptyB[sb], ((k - NSB) / NSB) & 1);
          tc::mbar_expect_tx(&fullB[sb], 2 * C::QB);
          tc::tma_load_3d(bb + OFF_Q, &tmQ, &fullB[sb], 0, u0 - a.R, bh);
          tc::tma_load_3d(bb + OFF_DO, &tmdO, &fullB[sb], 0, u0 - a.R, bh);
        } else {   // K, V (and the LSE / delta rows) free after dP + dS (empty); Q, dO after dV / dK (emptyB)
          tc::mbar_expect_tx(&full[st], 2 * C::KB + 2 * C::QB);
          tc::tma_load_3d(b0, &tmK, &full[st], 0, u0, bh);
          tc::tma_load_3d(b0 + OFF_V, &tmV, &full[st], 0, u0, bh);
          if (k >= NS) tc::mbar_wait(&emptyB[st], ((k - NS) / NS) & 1);
          tc::tma_load_3d(b0 + OFF_Q, &tmQ, &full[st], 0, u0 - a.R, bh);
          tc::tma_load_3d(b0 + OFF_DO, &tmdO, &full[st], 0, u0 - a.R, bh);
        }
        // workspace rows trail: once the first NS stages' other loads are in flight, wait for K1
        // (PDL) and from then on load each stage's rows right after its other boxes.  LSE*log2e
        // and delta of the NQ query columns (padded rows written by K1; columns outside [0, T)
        // are zero-filled: their Q / dO rows are zero, so they add nothing)
        (void)na;
        if (k + 1 >= NS || k + 1 == ntile_me) {
          if (nd == 0) tc::pdl_wait();   // K1 complete: its rows are visible
          for (; nd <= k; ++nd) {
            const int gd = ntiles - 1 - (blockIdx.x + nd * gridDim.x);   // reversed order (below)
            const int sd = nd % NS, nad = ((gd % ntq) * kM - a.R) & ~3;
            uint8_t* bd = stage0 + sd * STG;
            tc::mbar_expect_tx(&dfull[sd], (PST ? 1 : 2) * C::NQP * 4);
            if (!PST) tc::tma_load_3d(bd + OFF_L2, &tmL2, &dfull[sd], nad, gd / ntq, 0);
            tc::tma_load_3d(bd + OFF_DEL, &tmDel, &dfull[sd], nad, gd / ntq, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(kM, NQ, 0, 0);
      constexpr uint32_t idG = tc::idesc_bf16(kM, kD, 0, 1);
      int ns = 0, ndp = 0, nkv = 0;
      if constexpr (PST) ns = ntile_me;   // no S: dP(k) needs its stage and X_b free (dV/dK(k-2) issued)
      while (nkv < ntile_me) {
        const uint32_t m = PST ? tc::mbar_test4(tc::smem_u32(&pdsfull[nkv & 1]), (nkv >> 1) & 1,
                                                tc::smem_u32(&kvfree[(nkv + 1) & 1]), ((nkv + 3) >> 1) & 1,
                                                tc::smem_u32(&full[ndp % NS]), (ndp / NS) & 1,
                                                tc::smem_u32(&fullB[ndp % NSB]), (ndp / NSB) & 1)
                               : tc::mbar_test4(tc::smem_u32(&pdsfull[nkv & 1]), (nkv >> 1) & 1,
                                          tc::smem_u32(&kvfree[(nkv + 1) & 1]), ((nkv + 3) >> 1) & 1,  // = (nkv-1)>>1 parity
                                          tc::smem_u32(&xfree[ndp & 1]), (ndp >> 1) & 1,
                                          tc::smem_u32(&full[ns % NS]), (ns / NS) & 1);
        if (nkv < ndp && (m & 1) && (nkv < 1 || (m & 2))) {
          tc::tc_fence_after();
          const int b = nkv & 1, st = nkv % NS;
          const uint32_t x = tbase + b * 256;
          const uint32_t base = PST ? tc::smem_u32(stageB0 + (nkv % NSB) * C::STAGE_B) : tc::smem_u32(stage0 + st * STG);
          const uint32_t q = base + OFF_Q, dO = base + OFF_DO;
#pragma unroll
          for (int j = 0; j < NQ / 16; ++j)
            tc::mma_bf16_ts(DV, x + 8 * j, tc::desc_mnmajor_sw128(dO + 2048 * j), idG, j > 0);
#pragma unroll
          for (int j = 0; j < NQ / 16; ++j)
            tc::mma_bf16_ts(DK, x + NQ / 2 + 8 * j, tc::desc_mnmajor_sw128(q + 2048 * j), idG, j > 0);
          tc::mma_commit(&kvfull[b]);
          if (!PST) tc::mma_commit(&emptyB[st]);   // Q, dO (PST: ring B is released after the dV / dK stores)
          ++nkv;
          continue;
        }
        if (ndp < ns && (m & 4) && (!PST || (ndp < nkv + 2 && (m & 8)))) {
          tc::tc_fence_after();
          const int b = ndp & 1, st = ndp % NS;
          const uint32_t base = tc::smem_u32(stage0 + st * STG);
          const uint32_t v = base + OFF_V;
          const uint32_t dO = (PST ? tc::smem_u32(stageB0 + (ndp % NSB) * C::STAGE_B) : base) + OFF_DO;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(v + 32 * j), tc::desc_kmajor_sw128(dO + 32 * j), idS,
                         j > 0);
          tc::mma_commit(&dpfull[b]);
          tc::mma_commit(&empty[st]);   // K (S^T), V: free once S and dP have read them
          ++ndp;
          continue;
        }
        if (!PST && ns < ntile_me && ns < nkv + 2 && (m & 8)) {
          tc::tc_fence_after();
          const int b = ns & 1;
          const uint32_t base = tc::smem_u32(stage0 + (ns % NS) * STG);
          const uint32_t kk = base, q = base + OFF_Q;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(kk + 32 * j), tc::desc_kmajor_sw128(q + 32 * j), idS,
                         j > 0);
          tc::mma_commit(&sfull[b]);
          ++ns;
          continue;
        }
      }
    }
  } else {
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = q4 == 2 && lane == 0;
    uint8_t* ostage = obuf0 + wg * 2 * C::KB;  // [dV | dK] (not PST)
    for (int k = wg; k < ntile_me; k += 2) {
      const int g = ntiles - 1 - (blockIdx.x + k * gridDim.x);   // reversed order (below)
      const int bh = g / ntq, u0 = (g % ntq) * kM;
      const int b = wg, use = k >> 1, st = k % NS;
      const int sh = (u0 - a.R) - ((u0 - a.R) & ~3);   // column 0 sits `sh` floats into the aligned box
      const float* sL2 = reinterpret_cast<const float*>(stage0 + st * STG + OFF_L2) + sh;
      const float* sDel = reinterpret_cast<const float*>(stage0 + st * STG + OFF_DEL) + sh;
      tc::mbar_wait(&full[st], (k / NS) & 1);   // LSE / delta staged by the producer warp
      const bool tr = (tid == 64) || (tid == 192);
      if (tr) trace_at(a.trace, 1, k);
      const uint32_t x = tbase + lanes + b * 256;
      const int c0 = 32 * q4;
      if constexpr (PST) {
        // P^T from the staged band (column i = query u0 - R + c0 + i; band index of key u0 + r is
        // lane - i + W - 1), kept as packed bf16 pairs: the TMEM A operand needs exactly these
        uint32_t pp[CW / 2];
        uint32_t pw = tc::smem_u32(stage0 + st * STG) + (c0 * a.ldp + lane + W - 1) * 2;
        const uint32_t step = 2 * (a.ldp - 1);
#pragma unroll
        for (int m = 0; m < CW / 2; ++m) {
          const int i = 2 * m;
          const uint32_t lo = (i >= lane && i < lane + W) ? tc::ld_shared_u16(pw) : 0u;
          const uint32_t hi = (i + 1 >= lane && i + 1 < lane + W) ? tc::ld_shared_u16(pw + step) : 0u;
          pp[m] = lo | (hi << 16);
          pw += 2 * step;
        }
        if (tr) trace_at(a.trace, 3, k);
        tc::mbar_wait(&dfull[st], (k / NS) & 1);   // delta rows (K1's output)
        tc::mbar_wait(&dpfull[b], use & 1);
        if (tr) trace_at(a.trace, 4, k);
        __syncwarp();
        tc::tc_fence_after();
        float ds[CW];   // (per-chunk waits: one batched wait measured 41.1 -> 41.3 us, more spills)
#pragma unroll
        for (int j = 0; j < CW / 8; ++j) {
          float dp[8];
          tc::tmem_ld8(x + c0 + 8 * j, dp);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const uint32_t w = pp[(8 * j + e) / 2];
            ds[8 * j + e] = __uint_as_float(w << 16) * (dp[e] - sDel[c0 + 8 * j + e]);
            ds[8 * j + e + 1] = __uint_as_float(w & 0xffff0000u) * (dp[e + 1] - sDel[c0 + 8 * j + e + 1]);
          }
        }
        {   // P^T -> packed columns [0, NQ/2) (as tmem_write_row, from the packed pairs)
          const int pc0 = 16 * q4;
#pragma unroll
          for (int j = 0; j < CW / 8; ++j) tc::tmem_st4(x + pc0 + 4 * j, pp[4 * j], pp[4 * j + 1], pp[4 * j + 2], pp[4 * j + 3]);
          for (int c = 0; c < NQ / 2; c += 4)
            if (c < pc0 || c >= pc0 + CW / 2) tc::tmem_st4(x + c, 0u, 0u, 0u, 0u);
        }
        tc::mbar_arrive(&empty[st]);   // this warpgroup's reads of the band window and delta are done
        tmem_write_row<CW, NQ>(x + NQ / 2, q4, ds);      // dS^T -> packed columns [NQ/2, NQ)
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&pdsfull[b]);
      } else {
      float p[CW];
      tc::mbar_wait(&dfull[st], (k / NS) & 1);   // LSE*log2e / delta rows (K1's output)
      tc::mbar_wait(&sfull[b], use & 1);
      if (tr) trace_at(a.trace, 2, k);
      __syncwarp();
      tc::tc_fence_after();
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, p + 8 * j);
      tc::tmem_ld_wait();
      {   // queries of key u = u0 + r inside its head [hs, hs + Th): column i <-> query u0 - R + c0 + i
        const int u = u0 + r, q0 = u0 - a.R + c0;
        const int hs = u - u % a.Th;
        const int lo = max(lane, hs - q0), hi = min(lane + W, hs + a.Th - q0);
#pragma unroll
        for (int i = 0; i < CW; ++i)
          p[i] = (i >= lo && i < hi) ? tc::ex2(fmaf(p[i], a.scale_log2, -sL2[c0 + i])) : 0.f;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      if (tr) trace_at(a.trace, 3, k);
      tc::mbar_wait(&dpfull[b], use & 1);
      if (tr) trace_at(a.trace, 4, k);
      __syncwarp();
      tc::tc_fence_after();
      float ds[CW];   // dP^T strip, all loads in flight before one wait, then dS^T in place
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, ds + 8 * j);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < CW; ++i) ds[i] = p[i] * (ds[i] - sDel[c0 + i]);
      tc::mbar_arrive(&empty[st]);   // this warpgroup's reads of the LSE / delta rows are done
      tmem_write_row<CW, NQ>(x, q4, p);                 // P^T  -> packed columns [0, NQ/2)
      tmem_write_row<CW, NQ>(x + NQ / 2, q4, ds);      // dS^T -> packed columns [NQ/2, NQ)
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pdsfull[b]);
      }
      if (tr) trace_at(a.trace, 5, k);
      // dV / dK epilogue
      tc::mbar_wait(&kvfull[b], use & 1);
      if (tr) trace_at(a.trace, 6, k);
      __syncwarp();
      tc::tc_fence_after();
      if constexpr (ACC) {   // sub-band of a wide band: add into the fp32 dK / dV rows
        // PST: ring B (Q, dO) is dead once dV / dK are done and nothing is staged there
        if (PST && leader) tc::mbar_arrive(&emptyB[k % NSB]);
        float dvr[64], dkr[64];
        tmem_ld64(DV + lanes, dvr);
        tmem_ld64(DK + lanes, dkr);
        tc::tc_fence_before();
        tc::mbar_arrive(&kvfree[b]);
        const int u = u0 + r;
        if (u < T) {
          const long long row = (long long)bh * T + u;
          acc_row64(a.acc_dv + row * 64, dvr, 1.f, a.acc_first);
          acc_row64(a.acc_dk + row * 64, dkr, a.scale, a.acc_first);
        }
        continue;
      }
      if constexpr (PST) {   // dV, dK staged in this tile's ring-B slot (Q, dO dead: the MMAs completed)
        uint8_t* bb = stageB0 + (k % NSB) * C::STAGE_B;
        tmem_row64_to_smem_sw128(DV + lanes, 1.f, bb + OFF_Q, r);
        tmem_row64_to_smem_sw128(DK + lanes, a.scale, bb + OFF_DO, r);
        tc::tc_fence_before();
        tc::mbar_arrive(&kvfree[b]);
        tc::fence_proxy_async_smem();
        tc::named_bar(1 + wg, 128);
        if (leader) {
          tc::tma_store_3d(&tmdV, bb + OFF_Q, 0, u0, bh);
          tc::tma_store_3d(&tmdK, bb + OFF_DO, 0, u0, bh);
          tc::bulk_commit();
          tc::bulk_wait_read0();
          tc::mbar_arrive(&emptyB[k % NSB]);
        }
        continue;
      }
      if (leader) tc::bulk_wait_read0();
      tc::named_bar(1 + wg, 128);
      tmem_row64_to_smem_sw128(DV + lanes, 1.f, ostage, r);
      tmem_row64_to_smem_sw128(DK + lanes, a.scale, ostage + C::KB, r);
      tc::tc_fence_before();
      tc::mbar_arrive(&kvfree[b]);
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (leader) {
        tc::tma_store_3d(&tmdV, ostage, 0, u0, bh);
        tc::tma_store_3d(&tmdK, ostage + C::KB, 0, u0, bh);
        tc::bulk_commit();
      }
      if (tr) trace_at(a.trace, 7, k);
    }
    if (leader) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// backward K2, block-ring variant (the LSE-mode K2 for 49 < W <= 65, whose NQ = 192 window does not
// fit two stages of the kernel above): the key-major kernel with its query window staged as 128-row
// blocks.  A CTA sweeps a contiguous range of key tiles, so consecutive
// tiles' windows [u0 - R, u0 - R + NQ) share a block: each tile loads one new Q block and one
// dO block (not the NQ-row windows), and a 3-slot block ring holds the current tile's two
// blocks plus the next one in flight.  K and V get their own 2-slot rings (released after S
// and dP), LSE*log2e / delta windows a 2-slot ring (released after the dS phase).  The
// NQ-wide MMAs are issued as N = 128 + (NQ - 128) column pieces over the two blocks.
// ------------------------------------------------------------------------------------------
template <int CW> struct DkvRCfg {
  static constexpr int NQ = nk_of(CW);
  static constexpr int NQ2 = NQ - kM;                    // rows taken from the second block
  static constexpr int NB = NQ2 > 0 ? 2 : 1;            // blocks per tile window
  static constexpr int KB = kM * 128;
  static constexpr int BLK = 2 * KB;                    // [Q block | dO block]
  static constexpr int NQP = (NQ + 3 + 31) / 32 * 32;
  static constexpr int RW = 2 * NQP * 4;                // LSE*log2e | delta window
  static constexpr int SMEM = 1024 + 3 * BLK + 2 * KB + 2 * KB + 2 * KB /* staging */ + 2 * RW + 512;
  static constexpr int THREADS = 320;
};

// Block bookkeeping of a CTA's tile sequence (identical in the producer and the MMA issuer):
// tile k's window uses blocks kt and kt+1 of its head; a tile that continues the previous one
// (same head, next key tile) reuses the previous tile's second block as its first.
struct BlkSeq {
  int k, n;          // next tile, next block number to load
  int pbh, pkt, ps;  // previous tile's head, key tile, second block number
  __device__ void init() { k = 0; n = 0; pbh = -1; pkt = -1; ps = -1; }
  // blocks of tile k (global tile g): first f, second s (-1 if NB == 1); new blocks to load in
  // [nl0, nl1); advances to tile k + 1
  __device__ void next(int g, int ntq, int nb, int& f, int& s, int& nl0, int& nl1) {
    const int bh = g / ntq, kt = g % ntq;
    const bool cont = nb == 2 && bh == pbh && kt == pkt + 1;
    nl0 = n;
    if (cont) { f = ps; s = n++; }
    else { f = n++; s = nb == 2 ? n++ : -1; }
    nl1 = n;
    pbh = bh; pkt = kt; ps = s; ++k;
  }
};

template <int CW, bool COOP>
__global__ void __launch_bounds__(320, 1)
    sa_bwd_dkdv_ring_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                        const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
                        const __grid_constant__ CUtensorMap tmL2, const __grid_constant__ CUtensorMap tmDel,
                        TcArgs a) {
  using C = DkvRCfg<CW>;
  constexpr int NQ = C::NQ, NQ2 = C::NQ2, NB = C::NB;
  static_assert(NQ + 64 <= 256 && NQ >= kM && NQ <= 2 * kM, "TMEM layout / two-block window");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* blk0 = smem;                             // [Q | dO] x 3 block slots
  uint8_t* k0 = blk0 + 3 * C::BLK;                  // K x 2
  uint8_t* v0 = k0 + 2 * C::KB;                     // V x 2
  uint8_t* obuf0 = v0 + 2 * C::KB;                  // staging x 2 (one per warpgroup)
  uint8_t* rw0 = obuf0 + 2 * C::KB;                 // LSE / delta windows x 2
  uint64_t* bars = reinterpret_cast<uint64_t*>(rw0 + 2 * C::RW);
  uint64_t* bfull = bars;             // [3]
  uint64_t* bempty = bfull + 3;       // [3]
  uint64_t* kfull = bempty + 3;       // [2]
  uint64_t* kempty = kfull + 2;       // [2]
  uint64_t* vfull = kempty + 2;       // [2]
  uint64_t* vempty = vfull + 2;       // [2]
  uint64_t* rfull = vempty + 2;       // [2]
  uint64_t* rempty = rfull + 2;       // [2] (128)
  uint64_t* sfull = rempty + 2;       // [2]
  uint64_t* xfree = sfull + 2;        // [2] (128)
  uint64_t* dpfull = xfree + 2;       // [2]
  uint64_t* pdsfull = dpfull + 2;     // [2] (128)
  uint64_t* kvfull = pdsfull + 2;     // [2]
  uint64_t* kvfree = kvfull + 2;      // [2] (128)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kvfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, W = a.L + a.R + 1;
  const int ntq = (T + kM - 1) / kM;
  const int ntiles = ntq * a.BH;
  const int G = gridDim.x;
  const int g_begin = (int)((long long)blockIdx.x * ntiles / G);
  const int ntile_me = (int)((long long)(blockIdx.x + 1) * ntiles / G) - g_begin;

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmK); tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO); tc::tma_prefetch_desc(&tmdK); tc::tma_prefetch_desc(&tmdV);
    for (int i = 0; i < 3; ++i) { tc::mbar_init(&bfull[i], 1); tc::mbar_init(&bempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&kfull[i], 1); tc::mbar_init(&kempty[i], 1);
      tc::mbar_init(&vfull[i], 1); tc::mbar_init(&vempty[i], 1);
      constexpr int NW = COOP ? 256 : 128;   // consumers per tile: both warpgroups (COOP) or one
      tc::mbar_init(&rfull[i], 1); tc::mbar_init(&rempty[i], NW);
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&xfree[i], NW); tc::mbar_init(&dpfull[i], 1);
      tc::mbar_init(&pdsfull[i], NW); tc::mbar_init(&kvfull[i], 1); tc::mbar_init(&kvfree[i], NW);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // only the LSE*log2e / delta rows come from K1: the producer waits (PDL) just before loading
  // them (see sa_bwd_dkdv_tc for why this is safe)
  tc::pdl_launch_dependents();
  const uint32_t DV = tbase + NQ, DK = tbase + 256 + NQ;

  if (warp == 0) {
    if (lane == 0) {
      BlkSeq sq;
      sq.init();
      for (int k = 0; k < ntile_me; ++k) {
        const int g = g_begin + k;
        const int bh = g / ntq, kt = g % ntq, u0 = kt * kM;
        int f, s2, nl0, nl1;
        sq.next(g, ntq, NB, f, s2, nl0, nl1);
        trace_at(a.trace, 0, k);
        // new window blocks (block b of this head = frames [128 b - R, 128 b - R + 128))
        for (int n = nl0; n < nl1; ++n) {
          const int sl = n % 3;
          if (n >= 3) tc::mbar_wait(&bempty[sl], ((n / 3) - 1) & 1);
          const int b = (n == f) ? kt : kt + 1;
          uint8_t* d = blk0 + sl * C::BLK;
          tc::mbar_expect_tx(&bfull[sl], C::BLK);
          tc::tma_load_3d(d, &tmQ, &bfull[sl], 0, b * kM - a.R, bh);
          tc::tma_load_3d(d + C::KB, &tmdO, &bfull[sl], 0, b * kM - a.R, bh);
        }
        const int s = k & 1;
        if (k >= 2) tc::mbar_wait(&kempty[s], ((k - 2) >> 1) & 1);
        tc::mbar_expect_tx(&kfull[s], C::KB);
        tc::tma_load_3d(k0 + s * C::KB, &tmK, &kfull[s], 0, u0, bh);
        if (k >= 2) tc::mbar_wait(&vempty[s], ((k - 2) >> 1) & 1);
        tc::mbar_expect_tx(&vfull[s], C::KB);
        tc::tma_load_3d(v0 + s * C::KB, &tmV, &vfull[s], 0, u0, bh);
        if (k == 0) tc::pdl_wait();
        if (k >= 2) tc::mbar_wait(&rempty[s], ((k - 2) >> 1) & 1);
        const int na = (u0 - a.R) & ~3;
        tc::mbar_expect_tx(&rfull[s], C::RW);
        tc::tma_load_3d(rw0 + s * C::RW, &tmL2, &rfull[s], na, bh, 0);
        tc::tma_load_3d(rw0 + s * C::RW + C::NQP * 4, &tmDel, &rfull[s], na, bh, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS1 = tc::idesc_bf16(kM, kM, 0, 0);
      constexpr uint32_t idS2 = tc::idesc_bf16(kM, NQ2 > 0 ? NQ2 : 16, 0, 0);
      constexpr uint32_t idG = tc::idesc_bf16(kM, kD, 0, 1);
      BlkSeq qs, qd, qk;                               // block sequences seen by S, dP, kv
      qs.init(); qd.init(); qk.init();
      int sf = 0, ss = 0, df = 0, ds2 = 0, kf = 0, ks2 = 0, krel2 = 0;   // current tiles' block numbers
      int ns = 0, ndp = 0, nkv = 0;
      auto blk = [&](int n) { return tc::smem_u32(blk0 + (n % 3) * C::BLK); };
      bool s_ready = false, d_ready = false, k_ready = false;            // block numbers fetched
      while (nkv < ntile_me) {
        if (!s_ready && ns < ntile_me) { int a0, a1; qs.next(g_begin + ns, ntq, NB, sf, ss, a0, a1); s_ready = true; }
        if (!d_ready && ndp < ns) { int a0, a1; qd.next(g_begin + ndp, ntq, NB, df, ds2, a0, a1); d_ready = true; }
        if (!k_ready && nkv < ndp) {
          int a0, a1; qk.next(g_begin + nkv, ntq, NB, kf, ks2, a0, a1);
          // the second block is released with this tile unless the next tile continues the head
          const int g = g_begin + nkv, gn = g + 1;
          krel2 = (NB == 2) && !(nkv + 1 < ntile_me && gn / ntq == g / ntq && gn % ntq == g % ntq + 1);
          k_ready = true;
        }
        const uint32_t m = tc::mbar_test4(tc::smem_u32(&pdsfull[nkv & 1]), (nkv >> 1) & 1,
                                          tc::smem_u32(&kvfree[(nkv + 1) & 1]), ((nkv + 3) >> 1) & 1,
                                          tc::smem_u32(&xfree[ndp & 1]), (ndp >> 1) & 1,
                                          tc::smem_u32(&kfull[ns & 1]), (ns >> 1) & 1);
        if (k_ready && nkv < ndp && (m & 1) && (nkv < 1 || (m & 2))) {
          tc::tc_fence_after();
          const int b = nkv & 1;
          const uint32_t x = tbase + b * 256;
          const uint32_t bf = blk(kf), bs = NB == 2 ? blk(ks2) : bf;
#pragma unroll
          for (int j = 0; j < NQ / 16; ++j) {
            const uint32_t dO = (j < kM / 16 ? bf : bs) + C::KB + 2048 * (j % (kM / 16));
            tc::mma_bf16_ts(DV, x + 8 * j, tc::desc_mnmajor_sw128(dO), idG, j > 0);
          }
#pragma unroll
          for (int j = 0; j < NQ / 16; ++j) {
            const uint32_t q = (j < kM / 16 ? bf : bs) + 2048 * (j % (kM / 16));
            tc::mma_bf16_ts(DK, x + NQ / 2 + 8 * j, tc::desc_mnmajor_sw128(q), idG, j > 0);
          }
          tc::mma_commit(&kvfull[b]);
          tc::mma_commit(&bempty[kf % 3]);
          if (krel2) tc::mma_commit(&bempty[ks2 % 3]);
          ++nkv;
          k_ready = false;
          continue;
        }
        if (d_ready && ndp < ns && (m & 4) && tc::mbar_test(tc::smem_u32(&vfull[ndp & 1]), (ndp >> 1) & 1)) {
          tc::tc_fence_after();
          const int b = ndp & 1;
          const uint32_t v = tc::smem_u32(v0 + (ndp & 1) * C::KB);
          const uint32_t dO1 = blk(df) + C::KB, dO2 = (NB == 2 ? blk(ds2) : blk(df)) + C::KB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j) {
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(v + 32 * j), tc::desc_kmajor_sw128(dO1 + 32 * j), idS1,
                         j > 0);
            if (NQ2 > 0)
              tc::mma_bf16(tbase + b * 256 + kM, tc::desc_kmajor_sw128(v + 32 * j), tc::desc_kmajor_sw128(dO2 + 32 * j),
                           idS2, j > 0);
          }
          tc::mma_commit(&dpfull[b]);
          tc::mma_commit(&vempty[ndp & 1]);
          ++ndp;
          d_ready = false;
          continue;
        }
        if (s_ready && ns < ntile_me && ns < nkv + 2 && (m & 8) &&
            tc::mbar_test(tc::smem_u32(&bfull[sf % 3]), (sf / 3) & 1) &&
            (NB == 1 || tc::mbar_test(tc::smem_u32(&bfull[ss % 3]), (ss / 3) & 1))) {
          tc::tc_fence_after();
          const int b = ns & 1;
          const uint32_t kk = tc::smem_u32(k0 + (ns & 1) * C::KB);
          const uint32_t q1 = blk(sf), q2 = NB == 2 ? blk(ss) : q1;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j) {
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(kk + 32 * j), tc::desc_kmajor_sw128(q1 + 32 * j), idS1,
                         j > 0);
            if (NQ2 > 0)
              tc::mma_bf16(tbase + b * 256 + kM, tc::desc_kmajor_sw128(kk + 32 * j), tc::desc_kmajor_sw128(q2 + 32 * j),
                           idS2, j > 0);
          }
          tc::mma_commit(&sfull[b]);
          tc::mma_commit(&kempty[ns & 1]);
          ++ns;
          s_ready = false;
        }
      }
    }
  } else if (COOP) {
    // Both warpgroups work on every tile: warpgroup `half` owns strip chunks [NC0 half, ...) of
    // each row (the two warps of a TMEM lane quadrant split the row), so the P and dS phases take
    // half as long; the dV (half 0) / dK (half 1) epilogue of tile k-1 runs after tile k's dS,
    // while the tensor core works on tile k-1's dV/dK MMAs and on S(k+1).
    const int half = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = q4 == 2 && lane == 0;
    uint8_t* ostage = obuf0 + half * C::KB;
    constexpr int NC = CW / 8, NC0 = (NC + 1) / 2;     // strip chunks, chunks of half 0
    const int c0 = 32 * q4;
    auto epilogue = [&](int kp) {   // dV (half 0) or dK (half 1) rows of tile kp
      const int gp = g_begin + kp;
      const int bhp = gp / ntq, u0p = (gp % ntq) * kM;
      tc::mbar_wait(&kvfull[kp & 1], (kp >> 1) & 1);
      __syncwarp();
      tc::tc_fence_after();
      float v[64];
      tmem_ld64((half ? DK : DV) + lanes, v);
      tc::tc_fence_before();
      tc::mbar_arrive(&kvfree[kp & 1]);
      if (leader) tc::bulk_wait_read0();
      tc::named_bar(1 + half, 128);
      tmem_row64_to_smem_sw128_regs(v, half ? a.scale : 1.f, ostage, r);
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + half, 128);
      if (leader) {
        tc::tma_store_3d(half ? &tmdK : &tmdV, ostage, 0, u0p, bhp);
        tc::bulk_commit();
      }
    };
    // the tile body for one half, with its chunk range known at compile time (no spills)
    auto tile = [&](int k, auto J0c, auto J1c) {
      constexpr int J0 = decltype(J0c)::value, J1 = decltype(J1c)::value, NJ = J1 - J0;
      const int g = g_begin + k;
      const int u0 = (g % ntq) * kM;
      const int b = k & 1, use = k >> 1, s = k & 1;
      const int sh = (u0 - a.R) - ((u0 - a.R) & ~3);
      const float* sL2 = reinterpret_cast<const float*>(rw0 + s * C::RW) + sh + c0 + 8 * J0;
      const float* sDel = sL2 + C::NQP;
      const bool tr = (tid == 64);
      tc::mbar_wait(&rfull[s], (k >> 1) & 1);
      if (tr) trace_at(a.trace, 1, k);
      const uint32_t x = tbase + lanes + b * 256;
      tc::mbar_wait(&sfull[b], use & 1);
      if (tr) trace_at(a.trace, 2, k);
      __syncwarp();
      tc::tc_fence_after();
      float p[8 * NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) tc::tmem_ld8(x + c0 + 8 * (J0 + j), p + 8 * j);
      tc::tmem_ld_wait();
      const int lo = lane - 8 * J0, hi = lane + W - 8 * J0;   // band columns of this row, in local indices
#pragma unroll
      for (int i = 0; i < 8 * NJ; ++i)
        p[i] = (i >= lo && i < hi) ? tc::ex2(fmaf(p[i], a.scale_log2, -sL2[i])) : 0.f;
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      if (tr) trace_at(a.trace, 3, k);
      tc::mbar_wait(&dpfull[b], use & 1);
      if (tr) trace_at(a.trace, 4, k);
      __syncwarp();
      tc::tc_fence_after();
      float ds[8 * NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        float dp[8];
        tc::tmem_ld8(x + c0 + 8 * (J0 + j), dp);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) ds[8 * j + e] = p[8 * j + e] * (dp[e] - sDel[8 * j + e]);
      }
      tc::mbar_arrive(&rempty[s]);
      // the packed P / dS columns overlap the other half's fp32 dP columns: both halves of every
      // row must have read dP first
      tc::tc_fence_before();
      tc::named_bar(3, 256);
      tc::tc_fence_after();
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int pc = 16 * q4 + 4 * (J0 + j);
        tc::tmem_st4(x + pc, pack_bf16(p[8 * j], p[8 * j + 1]), pack_bf16(p[8 * j + 2], p[8 * j + 3]),
                     pack_bf16(p[8 * j + 4], p[8 * j + 5]), pack_bf16(p[8 * j + 6], p[8 * j + 7]));
        tc::tmem_st4(x + NQ / 2 + pc, pack_bf16(ds[8 * j], ds[8 * j + 1]), pack_bf16(ds[8 * j + 2], ds[8 * j + 3]),
                     pack_bf16(ds[8 * j + 4], ds[8 * j + 5]), pack_bf16(ds[8 * j + 6], ds[8 * j + 7]));
      }
      // this half's share of the row's zero columns (half 0 before the strip, half 1 after it)
      {
        const int pc0 = 16 * q4;
        const int zlo = J0 ? pc0 + CW / 2 : 0, zhi = J0 ? NQ / 2 : pc0;
        for (int c = zlo; c < zhi; c += 4) {
          tc::tmem_st4(x + c, 0u, 0u, 0u, 0u);
          tc::tmem_st4(x + NQ / 2 + c, 0u, 0u, 0u, 0u);
        }
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pdsfull[b]);
      if (tr) trace_at(a.trace, 5, k);
      if (k >= 1) epilogue(k - 1);
      if (tr) trace_at(a.trace, 7, k);
    };
    for (int k = 0; k < ntile_me; ++k) {
      if (half) tile(k, std::integral_constant<int, NC0>{}, std::integral_constant<int, NC>{});
      else tile(k, std::integral_constant<int, 0>{}, std::integral_constant<int, NC0>{});
    }
    if (ntile_me > 0) epilogue(ntile_me - 1);
    if (leader) tc::bulk_wait0();
  } else {
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = q4 == 2 && lane == 0;
    uint8_t* ostage = obuf0 + wg * C::KB;
    for (int k = wg; k < ntile_me; k += 2) {
      const int g = g_begin + k;
      const int bh = g / ntq, u0 = (g % ntq) * kM;
      const int b = wg, use = k >> 1, s = k & 1;
      const int sh = (u0 - a.R) - ((u0 - a.R) & ~3);
      const float* sL2 = reinterpret_cast<const float*>(rw0 + s * C::RW) + sh;
      const float* sDel = sL2 + C::NQP;
      tc::mbar_wait(&rfull[s], (k >> 1) & 1);
      const bool tr = (tid == 64) || (tid == 192);
      if (tr) trace_at(a.trace, 1, k);
      const uint32_t x = tbase + lanes + b * 256;
      const int c0 = 32 * q4;
      tc::mbar_wait(&sfull[b], use & 1);
      if (tr) trace_at(a.trace, 2, k);
      __syncwarp();
      tc::tc_fence_after();
      float p[CW];
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, p + 8 * j);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < CW; ++i)
        p[i] = (i >= lane && i < lane + W) ? tc::ex2(fmaf(p[i], a.scale_log2, -sL2[c0 + i])) : 0.f;
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      if (tr) trace_at(a.trace, 3, k);
      tc::mbar_wait(&dpfull[b], use & 1);
      if (tr) trace_at(a.trace, 4, k);
      __syncwarp();
      tc::tc_fence_after();
      float ds[CW];   // dP^T strip, all loads in flight before one wait, then dS^T in place
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, ds + 8 * j);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < CW; ++i) ds[i] = p[i] * (ds[i] - sDel[c0 + i]);
      tc::mbar_arrive(&rempty[s]);                     // LSE / delta window consumed
      tmem_write_row<CW, NQ>(x, q4, p);
      tmem_write_row<CW, NQ>(x + NQ / 2, q4, ds);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pdsfull[b]);
      if (tr) trace_at(a.trace, 5, k);
      // dV then dK through one staging tile (TMA stores)
      tc::mbar_wait(&kvfull[b], use & 1);
      if (tr) trace_at(a.trace, 6, k);
      __syncwarp();
      tc::tc_fence_after();
      float dk[64];
      {
        float dv[64];
        tmem_ld64(DV + lanes, dv);
        tmem_ld64(DK + lanes, dk);
        tc::tc_fence_before();
        tc::mbar_arrive(&kvfree[b]);
        if (leader) tc::bulk_wait_read0();             // the previous tile's dK store has read the tile
        tc::named_bar(1 + wg, 128);
        const uint32_t row = tc::smem_u32(ostage) + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          tc::st_shared_v4(row + ((c ^ (r & 7)) << 4),
                           make_uint4(pack_bf16(dv[8 * c], dv[8 * c + 1]), pack_bf16(dv[8 * c + 2], dv[8 * c + 3]),
                                      pack_bf16(dv[8 * c + 4], dv[8 * c + 5]), pack_bf16(dv[8 * c + 6], dv[8 * c + 7])));
      }
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (leader) {
        tc::tma_store_3d(&tmdV, ostage, 0, u0, bh);
        tc::bulk_commit();
        tc::bulk_wait_read0();
      }
      tc::named_bar(1 + wg, 128);
      {
        const uint32_t row = tc::smem_u32(ostage) + r * 128;
        const float sc = a.scale;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          tc::st_shared_v4(row + ((c ^ (r & 7)) << 4),
                           make_uint4(pack_bf16(dk[8 * c] * sc, dk[8 * c + 1] * sc), pack_bf16(dk[8 * c + 2] * sc, dk[8 * c + 3] * sc),
                                      pack_bf16(dk[8 * c + 4] * sc, dk[8 * c + 5] * sc), pack_bf16(dk[8 * c + 6] * sc, dk[8 * c + 7] * sc)));
      }
      tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (leader) {
        tc::tma_store_3d(&tmdK, ostage, 0, u0, bh);
        tc::bulk_commit();
      }
      if (tr) trace_at(a.trace, 7, k);
    }
    if (leader) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// LLSA backward, band keys (channel R), key-major: for a tile of 128 channel-R keys u, every
// query channel c = 0..R contributes through the band: query (t, c) sees (u, R) iff
// u in [t + c - R - L, t + c - R]  <=>  t in [u + s_c, u + s_c + L],  s_c = R - c
// (Eq. 14 in the horizon form).  Per (tile, c) sub-item, exactly the SA key-major step with
// the query tile shifted by s_c:
//   S^T = K Q_c^T -> P^T (LSE of channel c);  dP^T = V dO_c^T -> dS^T (delta of channel c)
//   dV += P^T dO_c,  dK += dS^T Q_c            accumulated in TMEM over the R+1 channels
// Rings: K/V per key tile (2 stages), Q_c/dO_c/LSE_c/delta_c per sub-item (2 stages).
// ------------------------------------------------------------------------------------------
template <int CW> struct LkvCfg {
  static constexpr int NQ = nk_of(CW);
  static constexpr int KB = kM * 128;
  static constexpr int QB = NQ * 128;
  static constexpr int NQP = (NQ + 3 + 31) / 32 * 32;
  static constexpr int KVSTAGE = 2 * KB;
  static constexpr int QSTAGE = (2 * QB + 2 * NQP * 4 + 1023) / 1024 * 1024;
  static constexpr int NQS = 3;      // sub-item ring depth (dV / dK are staged in the tile's dead K / V)
  static constexpr int SMEM = 1024 + 2 * KVSTAGE + NQS * QSTAGE + 512;
  static_assert(SMEM <= 232448, "LLSA kv pass shared memory");
};

template <int CW>
__global__ void __launch_bounds__(320, 1)
    llsa_bwd_kv_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                   const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
                   const __grid_constant__ CUtensorMap tmL2, const __grid_constant__ CUtensorMap tmDel, TcArgs a,
                   int C, int bcast) {
  using Cf = LkvCfg<CW>;
  constexpr int NQ = Cf::NQ;
  static_assert(NQ + 64 <= 256, "TMEM layout needs NQ <= 192");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NQS = Cf::NQS;
  uint8_t* kv0 = smem;                                   // [K | V] x 2 (then the tile's [dV | dK] staging)
  uint8_t* qs0 = smem + 2 * Cf::KVSTAGE;                 // [Q_c | dO_c | lse2 | delta] x NQS
  uint64_t* bars = reinterpret_cast<uint64_t*>(qs0 + NQS * Cf::QSTAGE);
  uint64_t* kvfull_ld = bars;         // [2] K/V of a tile landed
  uint64_t* kvempty = kvfull_ld + 2;  // [2] K/V stage free (after the tile's dV / dK stores read it)
  uint64_t* qfull = kvempty + 2;      // [NQS]
  uint64_t* qempty = qfull + NQS;     // [NQS]
  uint64_t* sfull = qempty + NQS;     // [2]
  uint64_t* xfree = sfull + 2;        // [2] (128)
  uint64_t* dpfull = xfree + 2;       // [2]
  uint64_t* pdsfull = dpfull + 2;     // [2] (128)
  uint64_t* kvfull = pdsfull + 2;     // [2] dK/dV of a tile accumulated (by tile parity)
  uint64_t* kvfree = kvfull + 2;      // [2] (128) dK/dV drained (by tile parity)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kvfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, L = a.L, R = a.R;
  const int ntq = (T + kM - 1) / kM;
  const int ntiles = ntq * a.BH;
  const int ntile_me = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nsub = ntile_me * C;

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmK); tc::tma_prefetch_desc(&tmV);
    tc::tma_prefetch_desc(&tmdO); tc::tma_prefetch_desc(&tmdK); tc::tma_prefetch_desc(&tmdV);
    for (int i = 0; i < NQS; ++i) { tc::mbar_init(&qfull[i], 1); tc::mbar_init(&qempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&kvfull_ld[i], 1); tc::mbar_init(&kvempty[i], 1);
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&xfree[i], 128); tc::mbar_init(&dpfull[i], 1);
      tc::mbar_init(&pdsfull[i], 128); tc::mbar_init(&kvfull[i], 1); tc::mbar_init(&kvfree[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t DV = tbase + NQ, DK = tbase + 256 + NQ;

  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int kt = 0; kt < ntile_me; ++kt) {
        const int g = ntiles - 1 - (blockIdx.x + kt * gridDim.x);   // reverse of the fused pass order (L2)
        const int bh = g / ntq, u0 = (g % ntq) * kM;
        const int ks = kt & 1;
        if (kt >= 2) tc::mbar_wait(&kvempty[ks], ((kt - 2) >> 1) & 1);
        uint8_t* kvb = kv0 + ks * Cf::KVSTAGE;
        tc::mbar_expect_tx(&kvfull_ld[ks], 2 * Cf::KB);
        tc::tma_load_3d(kvb, &tmK, &kvfull_ld[ks], 0, u0, bh);
        tc::tma_load_3d(kvb + Cf::KB, &tmV, &kvfull_ld[ks], 0, u0, bh);
        for (int c = 0; c < C; ++c, ++k) {
          const int qs = k % NQS;
          if (k >= NQS) tc::mbar_wait(&qempty[qs], ((k - NQS) / NQS) & 1);
          uint8_t* qb = qs0 + qs * Cf::QSTAGE;
          const int n0 = u0 + (R - c);                    // query frame of column 0
          const int na = n0 & ~3;
          tc::mbar_expect_tx(&qfull[qs], 2 * Cf::QB + 2 * Cf::NQP * 4);
          tc::tma_load_4d(qb, &tmQ, &qfull[qs], 0, n0, bh, bcast ? 0 : c);
          tc::tma_load_4d(qb + Cf::QB, &tmdO, &qfull[qs], 0, n0, bh, c);
          tc::tma_load_3d(qb + 2 * Cf::QB, &tmL2, &qfull[qs], na, c * a.BH + bh, 0);
          tc::tma_load_3d(qb + 2 * Cf::QB + Cf::NQP * 4, &tmDel, &qfull[qs], na, c * a.BH + bh, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(kM, NQ, 0, 0);
      constexpr uint32_t idG = tc::idesc_bf16(kM, kD, 0, 1);
      int ns = 0, ndp = 0, nkv = 0;
      while (nkv < nsub) {
        const int kts = ns / C;
        const uint32_t m = tc::mbar_test4(tc::smem_u32(&pdsfull[nkv & 1]), (nkv >> 1) & 1,
                                          tc::smem_u32(&kvfull_ld[kts & 1]), (kts >> 1) & 1,
                                          tc::smem_u32(&xfree[ndp & 1]), (ndp >> 1) & 1,
                                          tc::smem_u32(&qfull[ns % NQS]), (ns / NQS) & 1);
        if (nkv < ndp && (m & 1)) {
          const int kt = nkv / C, c = nkv % C;
          if (c == 0 && kt >= 1 && !tc::mbar_test(tc::smem_u32(&kvfree[(kt - 1) & 1]), ((kt - 1) >> 1) & 1)) {
            // accumulators still being drained by the previous tile's epilogue
          } else {
            tc::tc_fence_after();
            const int b = nkv & 1, qs = nkv % NQS;
            const uint32_t x = tbase + b * 256;
            const uint32_t q = tc::smem_u32(qs0 + qs * Cf::QSTAGE), dO = q + Cf::QB;
#pragma unroll
            for (int j = 0; j < NQ / 16; ++j)
              tc::mma_bf16_ts(DV, x + 8 * j, tc::desc_mnmajor_sw128(dO + 2048 * j), idG, (c > 0) || (j > 0));
#pragma unroll
            for (int j = 0; j < NQ / 16; ++j)
              tc::mma_bf16_ts(DK, x + NQ / 2 + 8 * j, tc::desc_mnmajor_sw128(q + 2048 * j), idG, (c > 0) || (j > 0));
            tc::mma_commit(&qempty[qs]);
            if (c == C - 1) tc::mma_commit(&kvfull[kt & 1]);   // K / V dead: the epilogue stages dV / dK there
            ++nkv;
            continue;
          }
        }
        if (ndp < ns && (m & 4)) {
          tc::tc_fence_after();
          const int b = ndp & 1, kt = ndp / C;
          const uint32_t v = tc::smem_u32(kv0 + (kt & 1) * Cf::KVSTAGE) + Cf::KB;
          const uint32_t dO = tc::smem_u32(qs0 + (ndp % NQS) * Cf::QSTAGE) + Cf::QB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(v + 32 * j), tc::desc_kmajor_sw128(dO + 32 * j), idS,
                         j > 0);
          tc::mma_commit(&dpfull[b]);
          ++ndp;
          continue;
        }
        if (ns < nsub && ns < nkv + 2) {
          const int kt = kts;
          if ((m & 2) && (m & 8)) {
            tc::tc_fence_after();
            const int b = ns & 1;
            const uint32_t kk = tc::smem_u32(kv0 + (kt & 1) * Cf::KVSTAGE);
            const uint32_t q = tc::smem_u32(qs0 + (ns % NQS) * Cf::QSTAGE);
#pragma unroll
            for (int j = 0; j < kD / 16; ++j)
              tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(kk + 32 * j), tc::desc_kmajor_sw128(q + 32 * j), idS,
                           j > 0);
            tc::mma_commit(&sfull[b]);
            ++ns;
          }
        }
      }
    }
  } else {
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    const bool leader = q4 == 2 && lane == 0;
    const int W = L + 1;
    for (int k = wg; k < nsub; k += 2) {
      const int kt = k / C, c = k % C;
      const int g = ntiles - 1 - (blockIdx.x + kt * gridDim.x);
      const int bh = g / ntq, u0 = (g % ntq) * kM;
      const int b = k & 1, use = k >> 1, qs = k % NQS;
      const int n0 = u0 + (R - c);
      const int sh = n0 - (n0 & ~3);
      const float* sL2 = reinterpret_cast<const float*>(qs0 + qs * Cf::QSTAGE + 2 * Cf::QB) + sh;
      const float* sDel = sL2 + Cf::NQP;
      tc::mbar_wait(&qfull[qs], (k / NQS) & 1);
      const uint32_t x = tbase + lanes + b * 256;
      const int c0 = 32 * q4;
      tc::mbar_wait(&sfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      float p[CW];
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, p + 8 * j);
      tc::tmem_ld_wait();
      {   // queries of key u = u0 + r inside its head [hs, hs + Th): column i <-> query n0 + c0 + i
        const int u = u0 + r, qc = n0 + c0;
        const int hs = u - u % a.Th;
        const int lo = max(lane, hs - qc), hi = min(lane + W, hs + a.Th - qc);
#pragma unroll
        for (int i = 0; i < CW; ++i)
          p[i] = (i >= lo && i < hi) ? tc::ex2(fmaf(p[i], a.scale_log2, -sL2[c0 + i])) : 0.f;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      tc::mbar_wait(&dpfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      float ds[CW];   // dP^T strip, all loads in flight before one wait, then dS^T in place
#pragma unroll
      for (int j = 0; j < CW / 8; ++j) tc::tmem_ld8(x + c0 + 8 * j, ds + 8 * j);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < CW; ++i) ds[i] = p[i] * (ds[i] - sDel[c0 + i]);
      tmem_write_row<CW, NQ>(x, q4, p);
      tmem_write_row<CW, NQ>(x + NQ / 2, q4, ds);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pdsfull[b]);
      if (c == C - 1) {
        // dV / dK of the tile (accumulated over the R+1 query channels)
        tc::mbar_wait(&kvfull[kt & 1], (kt >> 1) & 1);
        __syncwarp();
        tc::tc_fence_after();
        uint8_t* ostage = kv0 + (kt & 1) * Cf::KVSTAGE;   // [dV | dK] over the tile's dead [K | V]
        tmem_row64_to_smem_sw128(DV + lanes, 1.f, ostage, r);
        tmem_row64_to_smem_sw128(DK + lanes, a.scale, ostage + Cf::KB, r);
        tc::tc_fence_before();
        tc::mbar_arrive(&kvfree[kt & 1]);
        tc::fence_proxy_async_smem();
        tc::named_bar(1 + wg, 128);
        if (leader) {
          tc::tma_store_3d(&tmdV, ostage, 0, u0, bh);
          tc::tma_store_3d(&tmdK, ostage + Cf::KB, 0, u0, bh);
          tc::bulk_commit();
          tc::bulk_wait_read0();                 // the stores have read the staging: K / V may reload
          tc::mbar_arrive(&kvempty[kt & 1]);
        }
      }
    }
    if (leader) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

static_assert(DqCfg<72>::STAGE % 1024 == 0 && DkvCfg<72>::STAGE % 1024 == 0 && FwdCfg<72>::STAGE % 1024 == 0,
              "smem stages must be 1024-byte aligned");

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
// [BH][T][64] bf16 viewed as a 3-D tensor (64, T, BH); box (64, rows, 1), 128B swizzle.
CUtensorMapL2promotion l2_promo() { return CU_TENSOR_MAP_L2_PROMOTION_L2_256B; }

bool make_map(CUtensorMap* m, const void* base, int T, int BH, int rows, int ld = 0) {
  cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)BH};
  cuuint64_t strides[2] = {64 * 2, (cuuint64_t)(ld > 0 ? ld : T) * 64 * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
  CUresult r = tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, l2_promo());
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

// [C][BH][T][64] bf16 as a 4-D tensor (64, T, BH, C); box (64, rows, 1, 1), 128B swizzle.
bool make_map4(CUtensorMap* m, const void* base, int T, int BH, int C, int rows) {
  cuuint64_t dims[4] = {64, (cuuint64_t)T, (cuuint64_t)BH, (cuuint64_t)C};
  cuuint64_t strides[3] = {128, (cuuint64_t)T * 128, (cuuint64_t)BH * T * 128};
  cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
  CUresult r = tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled (4d) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

// stored band P [BH][T][ldp] bf16 as (ldp, T, BH); box (ldp, rows, 1), no swizzle (row-major
// [rows][ldp] in shared memory); rows outside [0, T) load as zeros and are clipped on store.
// the stored band [BH][T][row] bf16 (row = ldp, or a wider row of which ldp columns from `base` are
// mapped: a sub-band of a wide band); box (ldp, rows, 1), no swizzle
bool make_map_p(CUtensorMap* m, const void* base, int T, int BH, int ldp, int rows, int row = 0, int ld = 0) {
  const int pitch = row > 0 ? row : ldp;   // elements per stored row
  const int frames = ld > 0 ? ld : T;      // rows per head (a time shard's margined length)
  cuuint64_t dims[3] = {(cuuint64_t)ldp, (cuuint64_t)T, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)frames * pitch * 2};
  cuuint32_t box[3] = {(cuuint32_t)ldp, (cuuint32_t)rows, 1};
  CUresult r = tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled (band) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

// padded fp32 workspace rows [BH][Tp] viewed as a 2-D tensor (T, BH); box (rows, 1); no swizzle.
bool make_map_f32_rows(CUtensorMap* m, const void* base, int T, int Tp, int BH, int box) {
  // 3-D view (T, BH, 1) so the load uses the same tensor-tile instruction form as the bf16 tiles
  cuuint64_t dims[3] = {(cuuint64_t)T, (cuuint64_t)BH, 1};
  cuuint64_t strides[2] = {(cuuint64_t)Tp * 4, (cuuint64_t)Tp * 4 * BH};
  cuuint32_t bx[3] = {(cuuint32_t)box, 1, 1};
  CUresult r = tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, bx, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled (f32 rows) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

// Launch with programmatic stream serialization (PDL): the kernel's prologue (barrier init, TMEM
// alloc, descriptor prefetch) overlaps the previous kernel's tail; kernels call pdl_wait() first.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

int cw_of(int W) {
  const int need = W + 31;
  const int opts[] = {32, 48, 64, 72, 80, 96, 112, 128, 160};
  for (int c : opts)
    if (c >= need) return c;
  return -1;
}

TcArgs tc_args(const AttnArgs& a) {
  TcArgs t{};
  t.T = a.T; t.L = a.L; t.R = a.R; t.BH = a.BH;
  t.scale = a.scale; t.scale_log2 = a.scale_log2;
  t.O = reinterpret_cast<bf16*>(a.Out); t.LSE = a.LSEout;
  t.Og = reinterpret_cast<const bf16*>(a.O); t.LSEin = a.LSE;
  t.dQ = reinterpret_cast<bf16*>(a.dQ); t.dK = reinterpret_cast<bf16*>(a.dK); t.dV = reinterpret_cast<bf16*>(a.dV);
  t.delta = a.delta;
  t.Tp = (a.T + 3) & ~3;
  t.trace = g_trace;
  t.kshift = 0;
  t.ws_del = a.delta;
  t.ws_l2 = a.delta + (long long)a.BH * t.Tp;
  t.ldp = a.ldp;
  t.ld = a.ld > 0 ? a.ld : a.T;
  t.Th = a.Th > 0 ? a.Th : a.T;
  const int ntq = (a.T + kM - 1) / kM;
  if (a.nkt > 0) {
    t.nkt = a.nkt; t.kt0 = a.kt0; t.kt_split = a.kt_split; t.kt_jump = a.kt_jump;
  } else {
    t.nkt = ntq; t.kt0 = 0; t.kt_split = ntq; t.kt_jump = 0;
  }
  return t;
}

// Packed tiles.  A full launch over contiguous [BH][T] heads runs on the flattened BH*T frame axis
// as one sequence (BH = 1) whose rows each attend only inside their own head (TcArgs::Th): 128-row
// tiles then straddle head boundaries, and the launch has ceil(BH*T / 128) tiles instead of
// BH * ceil(T / 128).  Base shape (BH = 96, T = 1750): 1313 tiles = 8.87 rounds of 148 SMs instead
// of 1344 = 9.08, i.e. 9 tiles on the busiest CTA instead of 10.  Keys of a neighbouring head in a
// tile's box are masked like frames outside [0, T) were (the stored band holds zeros for them).
// Not for time-shard launches (a row stride or a tile subset) or when packing saves no tile.
AttnArgs flat_view(const AttnArgs& a) {
  const long long tot = (long long)a.BH * a.T;
  if (a.BH <= 1 || a.nkt > 0 || (a.ld > 0 && a.ld != a.T) || a.Th > 0 || tot > (1LL << 30)) return a;
  if ((tot + kM - 1) / kM >= (long long)a.BH * ((a.T + kM - 1) / kM)) return a;
  AttnArgs f = a;
  f.T = (int)tot;
  f.BH = 1;
  f.ld = 0;
  f.Th = a.T;
  return f;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct WideAcc {   // fp32 accumulators of a wide band's sub-band launches (ACC instances)
  float *o, *m, *l, *dq, *dk, *dv;
  int first;
};

template <int CW, bool PST = false, bool ACC = false>
sattn_status fwd_launch(const AttnArgs& a, cudaStream_t st, const WideAcc* wa = nullptr) {
  using C = FwdCfg<CW, PST>;
  TcArgs ta = tc_args(a);
  if (wa) { ta.acc_o = wa->o; ta.acc_m = wa->m; ta.acc_l = wa->l; ta.acc_first = wa->first; }
  CUtensorMap mq, mk, mv, mo, mp;
  if (!make_map(&mq, a.Q, a.T, a.BH, kM, a.ld) || !make_map(&mk, a.K, a.T, a.BH, C::NK, a.ld) ||
      !make_map(&mv, a.V, a.T, a.BH, C::NK, a.ld) || !make_map(&mo, a.Out, a.T, a.BH, kM, a.ld))
    return SATTN_ECUDA;
  if (PST && !make_map_p(&mp, a.P, a.T, a.BH, a.ldp, kM, 0, a.ld)) return SATTN_ECUDA;
  set_smem(sa_fwd_tc<CW, PST, ACC>, C::SMEM);
  const int ntiles = ta.nkt * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  launch_pdl(sa_fwd_tc<CW, PST, ACC>, dim3(grid), dim3(C::THREADS), C::SMEM, st, mq, mk, mv, mo, PST ? mp : mo, ta);
  return SATTN_OK;
}

// phase: bit 0 = K1 (over the launch's query tiles, tc_args), bit 1 = K2 (every key tile).  A time
// shard runs K1 on its interior tiles during the halo exchange, then K1 on the edge tiles and K2.
template <int CW>
sattn_status bwd_launch(const AttnArgs& a, cudaStream_t st, int phase = 3) {
  constexpr int NK = nk_of(CW);
  const int Tp = (a.T + 3) & ~3;
  const float* l2ws = a.delta + (long long)a.BH * Tp;
  // bands too wide for the two-stage K2's shared memory (W > 49: NQ = 192) take the block-ring
  // kernel with the column-split warpgroups (its registers hold half a row)
  constexpr bool wide = DkvCfg<CW>::SMEM > 232448;
  constexpr int NQP = wide ? DkvRCfg<CW>::NQP : DkvCfg<CW>::NQP;
  const int ld = a.ld;
  CUtensorMap mq, mk, mv, mdo, mdq, mqN, mdoN, mk128, mv128, mdk, mdv, ml2, mdel;
  if (!make_map(&mq, a.Q, a.T, a.BH, kM, ld) || !make_map(&mk, a.K, a.T, a.BH, NK, ld) ||
      !make_map(&mv, a.V, a.T, a.BH, NK, ld) || !make_map(&mdo, a.dO, a.T, a.BH, kM, ld) ||
      !make_map(&mdq, a.dQ, a.T, a.BH, kM, ld) || !make_map(&mqN, a.Q, a.T, a.BH, NK, ld) ||
      !make_map(&mdoN, a.dO, a.T, a.BH, NK, ld) || !make_map(&mk128, a.K, a.T, a.BH, kM, ld) ||
      !make_map(&mv128, a.V, a.T, a.BH, kM, ld) || !make_map(&mdk, a.dK, a.T, a.BH, kM, ld) ||
      !make_map(&mdv, a.dV, a.T, a.BH, kM, ld) || !make_map_f32_rows(&ml2, l2ws, a.T, Tp, a.BH, NQP) ||
      !make_map_f32_rows(&mdel, a.delta, a.T, Tp, a.BH, NQP))
    return SATTN_ECUDA;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  if (phase & 1) {
    const TcArgs t1 = tc_args(a);
    const int nt1 = t1.nkt * a.BH;
    set_smem(sa_bwd_dq_tc<CW>, DqCfg<CW>::SMEM);
    launch_pdl(sa_bwd_dq_tc<CW>, dim3(nt1 < num_sms() ? nt1 : num_sms()), dim3(DqCfg<CW>::THREADS), DqCfg<CW>::SMEM,
               st, mq, mk, mv, mdo, mdq, t1);
  }
  if (!(phase & 2)) return SATTN_OK;
  if constexpr (wide) {
    set_smem(sa_bwd_dkdv_ring_tc<CW, true>, DkvRCfg<CW>::SMEM);
    launch_pdl(sa_bwd_dkdv_ring_tc<CW, true>, dim3(grid), dim3(DkvRCfg<CW>::THREADS), DkvRCfg<CW>::SMEM, st, mq,
               mk128, mv128, mdo, mdk, mdv, ml2, mdel, tc_args(a));
  } else {
    set_smem(sa_bwd_dkdv_tc<CW>, DkvCfg<CW>::SMEM);
    launch_pdl(sa_bwd_dkdv_tc<CW>, dim3(grid), dim3(DkvCfg<CW>::THREADS), DkvCfg<CW>::SMEM, st, mqN, mk128, mv128,
               mdoN, mdk, mdv, ml2, mdel, tc_args(a));
  }
  return SATTN_OK;
}

// ------------------------------------------------------------------------------------------
// wide bands (W > 65: NEXT-1, the Fig. 5 sweep to W = 490) on the tensor-core kernels.  The band
// [t - L, t + R] is split into S sub-bands of width <= 49; sub-band j (offsets o_j .. o_j + w_j - 1
// from t - L) is an SA band of its own with (L_j, R_j) = (L - o_j, o_j + w_j - 1 - L), either of
// which may be negative.  Softmax over the union is exact by the log-sum-exp merge of the
// sub-bands' (o, m, l) (forward; the split-K combine), and the gradient is exactly the sum of the
// sub-bands' gradients when each uses the global LSE and delta = dO . O (Eq. 9; G28), so every
// sub-band runs the narrow kernels' ACC instances into fp32 accumulators, then one kernel rounds.
// ------------------------------------------------------------------------------------------
constexpr int kWideSub = 49;   // sub-band width: the two-stage K2's limit

__global__ void wide_delta_kernel(const bf16* dO, const bf16* O, float* del, int T, int Tp, long long nrows) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nrows; i += (long long)gridDim.x * blockDim.x) {
    const long long bh = i / Tp;
    const int t = (int)(i - bh * Tp);
    float s = 0.f;
    if (t < T) {
      const uint4* a = reinterpret_cast<const uint4*>(dO + (bh * T + t) * 64);
      const uint4* b = reinterpret_cast<const uint4*>(O + (bh * T + t) * 64);
#pragma unroll
      for (int c = 0; c < 8; ++c) s += dot8_bf16(a[c], b[c]);
    }
    del[i] = s;
  }
}

__global__ void wide_fwd_finalize(const float* acc_o, const float* acc_m, const float* acc_l, bf16* O, float* LSE,
                                  float scale, long long nrows) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nrows; i += (long long)gridDim.x * blockDim.x) {
    const float l = acc_l[i];
    float v[64];
    const float4* s = reinterpret_cast<const float4*>(acc_o + i * 64);
#pragma unroll
    for (int c = 0; c < 16; ++c) { const float4 x = s[c]; v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w; }
    store_row_bf16(O + i * 64, v, 1.f / l);
    LSE[i] = acc_m[i] * scale + __logf(l);
  }
}

__global__ void f32_to_bf16_kernel(const float* a, bf16* o, long long n8) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 x = reinterpret_cast<const float4*>(a)[2 * i], y = reinterpret_cast<const float4*>(a)[2 * i + 1];
    reinterpret_cast<uint4*>(o)[i] = make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y),
                                                pack_bf16(y.z, y.w));
  }
}

template <int CW>
sattn_status bwd_wide_sub(const AttnArgs& a, cudaStream_t st, const WideAcc& wa) {
  static_assert(DkvCfg<CW>::SMEM <= 232448, "sub-bands use the two-stage K2");
  constexpr int NK = nk_of(CW);
  const int Tp = (a.T + 3) & ~3;
  const float* l2ws = a.delta + (long long)a.BH * Tp;
  constexpr int NQP = DkvCfg<CW>::NQP;
  CUtensorMap mq, mk, mv, mdo, mqN, mdoN, mk128, mv128, ml2, mdel;
  if (!make_map(&mq, a.Q, a.T, a.BH, kM) || !make_map(&mk, a.K, a.T, a.BH, NK) || !make_map(&mv, a.V, a.T, a.BH, NK) ||
      !make_map(&mdo, a.dO, a.T, a.BH, kM) || !make_map(&mqN, a.Q, a.T, a.BH, NK) ||
      !make_map(&mdoN, a.dO, a.T, a.BH, NK) || !make_map(&mk128, a.K, a.T, a.BH, kM) ||
      !make_map(&mv128, a.V, a.T, a.BH, kM) || !make_map_f32_rows(&ml2, l2ws, a.T, Tp, a.BH, NQP) ||
      !make_map_f32_rows(&mdel, a.delta, a.T, Tp, a.BH, NQP))
    return SATTN_ECUDA;
  TcArgs t = tc_args(a);
  t.acc_dq = wa.dq; t.acc_dk = wa.dk; t.acc_dv = wa.dv; t.acc_first = wa.first;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  set_smem(sa_bwd_dq_tc<CW, false, true>, DqCfg<CW>::SMEM);
  launch_pdl(sa_bwd_dq_tc<CW, false, true>, dim3(grid), dim3(DqCfg<CW>::THREADS), DqCfg<CW>::SMEM, st, mq, mk, mv,
             mdo, mq, t);
  set_smem(sa_bwd_dkdv_tc<CW, false, true>, DkvCfg<CW>::SMEM);
  launch_pdl(sa_bwd_dkdv_tc<CW, false, true>, dim3(grid), dim3(DkvCfg<CW>::THREADS), DkvCfg<CW>::SMEM, st, mqN,
             mk128, mv128, mdoN, mk128, mk128, ml2, mdel, t);
  return SATTN_OK;
}

// sub-band j of a band of width W split into S parts: offset and width
void wide_split(int W, int j, int S, int& o, int& w) {
  const int base = (W + S - 1) / S;
  o = j * base;
  w = W - o < base ? W - o : base;
}

// LLSA key-major band pass: dK, dV of channel R's keys accumulated over the C query channels
// (delta and LSE log2e rows from the workspace)
template <int CW>
sattn_status llsa_bwd_kv_launch(const AttnArgs& a0, const bf16* Q, const bf16* dO, const bf16* Kr, const bf16* Vr,
                                bf16* dK, bf16* dV, float* ws_del, float* ws_l2, bool flat, cudaStream_t st) {
  using LC = LkvCfg<CW>;
  const int R = a0.R, C = R + 1;
  const bool bc = a0.in_cs == 0;
  const long long plane = (long long)a0.BH * a0.T * kD;
  // packed tiles (flat: the delta / LSE rows are [C][BH*T rounded to 4], written so by the fused
  // pass): key tiles over the flattened BH*T axis, every query masked to its key's head (Th)
  AttnArgs a = a0;
  if (flat) {
    a.T = a0.BH * a0.T;
    a.BH = 1;
    a.Th = a0.T;
  }
  const int Tp = (a.T + 3) & ~3;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  CUtensorMap mq4, mdo4, mk, mv, mdk, mdv, ml2, mdel;
  if (!make_map4(&mq4, Q, a.T, a.BH, bc ? 1 : C, LC::NQ) || !make_map4(&mdo4, dO, a.T, a.BH, C, LC::NQ) ||
      !make_map(&mk, Kr, a.T, a.BH, kM) || !make_map(&mv, Vr, a.T, a.BH, kM) ||
      !make_map(&mdk, dK + plane * R, a.T, a.BH, kM) || !make_map(&mdv, dV + plane * R, a.T, a.BH, kM) ||
      !make_map_f32_rows(&ml2, ws_l2, a.T, Tp, C * a.BH, LC::NQP) ||
      !make_map_f32_rows(&mdel, ws_del, a.T, Tp, C * a.BH, LC::NQP))
    return SATTN_ECUDA;
  TcArgs t = tc_args(a);
  set_smem(llsa_bwd_kv_tc<CW>, LC::SMEM);
  launch_pdl(llsa_bwd_kv_tc<CW>, dim3(grid), dim3(320), LC::SMEM, st, mq4, mk, mv, mdo4, mdk, mdv, ml2, mdel, t, C,
             bc ? 1 : 0);
  return SATTN_OK;
}

// LLSA backward: band (channel-R keys) on the tensor-core kernels; the rest either in the fused
// horizon-major pass (dense inputs) or, for a broadcast layer-1 input, staircase on mma.sync.
template <int CW>
sattn_status llsa_bwd_launch(const AttnArgs& a, cudaStream_t st, int phase = 3, const int* sub4 = nullptr) {
  constexpr int NK = nk_of(CW);
  using LC = LkvCfg<CW>;
  const int R = a.R, C = R + 1;
  const bool bc = a.in_cs == 0;
  const long long plane = (long long)a.BH * a.T * kD;
  const bf16* Q = reinterpret_cast<const bf16*>(a.Q);
  const bf16* K = reinterpret_cast<const bf16*>(a.K);
  const bf16* V = reinterpret_cast<const bf16*>(a.V);
  const bf16* dO = reinterpret_cast<const bf16*>(a.dO);
  bf16* dQ = reinterpret_cast<bf16*>(a.dQ);
  bf16* dK = reinterpret_cast<bf16*>(a.dK);
  bf16* dV = reinterpret_cast<bf16*>(a.dV);
  const bf16* Kr = K + a.in_cs * R;
  const bf16* Vr = V + a.in_cs * R;
  const int Tp = (a.T + 3) & ~3;
  float* ws_del = a.delta;                          // [C][BH][Tp]
  float* ws_l2 = a.delta + (long long)C * a.BH * Tp;
  float* ws_dx = a.delta + 2LL * C * a.BH * Tp;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  if (tc_llsa_bwd_fused_supported(SATTN_BF16, kD, a.L, R, a.BH, a.T, !bc)) {
    // fused horizon-major pass (tc_llsa.cu): dQ, staircase dK / dV, delta / LSE rows; then the
    // key-major band pass below for channel R's dK / dV
    // packed kv tiles when they save a round's worth of tiles (base shape: 1313 instead of 1344)
    const long long tot = (long long)a.BH * a.T;
    const bool flat = a.BH > 1 && tot <= (1LL << 30) &&
                      (tot + kM - 1) / kM < (long long)a.BH * ((a.T + kM - 1) / kM);
    if (phase & 1) {
      sattn_status r = tc_llsa_bwd_fused(a, ws_del, ws_l2, flat ? 1 : 0, st, sub4);
      if (r != SATTN_OK) {
        g_tc_err = tc_llsa_last_error();
        return r;
      }
    }
    return phase & 2 ? llsa_bwd_kv_launch<CW>(a, Q, dO, Kr, Vr, dK, dV, ws_del, ws_l2, flat, st) : SATTN_OK;
  }
  StairArgs sa{};
  sa.Q = Q; sa.K = K; sa.V = V; sa.dO = dO;
  sa.dQ = dQ; sa.dK = dK; sa.dV = dV;
  sa.del = ws_del; sa.l2 = ws_l2; sa.lse = a.LSE; sa.dx = ws_dx;
  sa.T = a.T; sa.L = a.L; sa.R = R; sa.BH = a.BH; sa.Tp = Tp;
  sa.in_cs = a.in_cs; sa.plane = plane;
  sa.scale = a.scale; sa.scale_log2 = a.scale_log2;
  // horizons run to T - 1 + R (the last staircase keys / queries of channels > 0)
  const dim3 sgrid((a.T + R + kStF - 1) / kStF, a.BH);
  // (0) staircase part of delta = rowsum(P o dP)
  {
    const size_t smem = stair_smem_bytes(R, true);
    set_smem(llsa_bwd_stair<true>, (int)smem);
    llsa_bwd_stair<true><<<sgrid, 256, smem, st>>>(sa);
  }
  // (1) query-major band pass of every channel in one launch: the SA dQ kernel with R := 0 and
  //     channel c's keys shifted by R - c (tiles ordered channel-major)
  {
    set_smem(sa_bwd_dq_tc<CW>, DqCfg<CW>::SMEM);
    CUtensorMap mq, mk, mv, mdo, mdq;
    if (!make_map4(&mq, Q, a.T, a.BH, bc ? 1 : C, kM) || !make_map(&mk, Kr, a.T, a.BH, NK) ||
        !make_map(&mv, Vr, a.T, a.BH, NK) || !make_map4(&mdo, dO, a.T, a.BH, C, kM) ||
        !make_map4(&mdq, dQ, a.T, a.BH, C, kM))
      return SATTN_ECUDA;
    TcArgs t = tc_args(a);
    t.R = 0;
    t.kshift = R;
    t.nch = C;
    t.bcast = bc ? 1 : 0;
    t.LSEin = a.LSE;
    t.ws_del = ws_del;
    t.ws_l2 = ws_l2;
    t.ws_dx = ws_dx;
    t.dq_split = 1;
    const int tiles = (a.T + kM - 1) / kM * a.BH * C;
    launch_pdl(sa_bwd_dq_tc<CW>, dim3(tiles < num_sms() ? tiles : num_sms()), dim3(DqCfg<CW>::THREADS),
               DqCfg<CW>::SMEM, st, mq, mk, mv, mdo, mdq, t);
  }
  // (2) key-major band pass: dK, dV of channel R accumulated over the C query channels
  {
    const sattn_status r = llsa_bwd_kv_launch<CW>(a, Q, dO, Kr, Vr, dK, dV, ws_del, ws_l2, false, st);
    if (r != SATTN_OK) return r;
  }
  // (3) staircase keys and the staircase part of dQ (mma.sync)
  {
    const size_t smem = stair_smem_bytes(R, false);
    set_smem(llsa_bwd_stair<false>, (int)smem);
    llsa_bwd_stair<false><<<sgrid, 256, smem, st>>>(sa);
  }
  return SATTN_OK;
}

}  // namespace

bool tc_wide_supported(int dtype, int D, int L, int R) {
  return dtype == SATTN_BF16 && D == 64 && L + R + 1 > 65 && L + R + 1 <= 4096;
}
int tc_wide_parts(int L, int R) { return (L + R + 1 + kWideSub - 1) / kWideSub; }
size_t tc_wide_fwd_ws(long long BH, long long T) { return (size_t)BH * T * (64 + 2) * sizeof(float); }
size_t tc_wide_bwd_ws(long long BH, long long T) {
  return (size_t)2 * BH * ((T + 3) & ~3LL) * sizeof(float) + (size_t)3 * BH * T * 64 * sizeof(float);
}

sattn_status tc_forward_wide(const AttnArgs& a, void* ws, cudaStream_t st) {
  const int W = a.L + a.R + 1, S = tc_wide_parts(a.L, a.R);
  const long long rows = (long long)a.BH * a.T;
  WideAcc wa{};
  wa.o = static_cast<float*>(ws);
  wa.m = wa.o + rows * 64;
  wa.l = wa.m + rows;
  for (int j = 0; j < S; ++j) {
    int o, w;
    wide_split(W, j, S, o, w);
    AttnArgs aj = a;
    aj.L = a.L - o;
    aj.R = o + w - 1 - a.L;
    wa.first = j == 0;
    sattn_status r;
    switch (cw_of(w)) {
      case 32: r = fwd_launch<32, false, true>(aj, st, &wa); break;
      case 48: r = fwd_launch<48, false, true>(aj, st, &wa); break;
      case 64: r = fwd_launch<64, false, true>(aj, st, &wa); break;
      case 72: r = fwd_launch<72, false, true>(aj, st, &wa); break;
      case 80: r = fwd_launch<80, false, true>(aj, st, &wa); break;
      default: g_tc_err = "wide sub-band"; return SATTN_EUNSUPPORTED;
    }
    if (r != SATTN_OK) return r;
  }
  wide_fwd_finalize<<<4 * num_sms(), 128, 0, st>>>(wa.o, wa.m, wa.l, reinterpret_cast<bf16*>(a.Out), a.LSEout, a.scale,
                                                   rows);
  return SATTN_OK;
}

sattn_status tc_backward_wide(const AttnArgs& a, cudaStream_t st) {
  const int W = a.L + a.R + 1, S = tc_wide_parts(a.L, a.R);
  const long long rows = (long long)a.BH * a.T;
  const int Tp = (a.T + 3) & ~3;
  WideAcc wa{};
  wa.dq = a.delta + 2LL * a.BH * Tp;
  wa.dk = wa.dq + rows * 64;
  wa.dv = wa.dk + rows * 64;
  wide_delta_kernel<<<4 * num_sms(), 256, 0, st>>>(reinterpret_cast<const bf16*>(a.dO), reinterpret_cast<const bf16*>(a.O),
                                                   a.delta, a.T, Tp, (long long)a.BH * Tp);
  for (int j = 0; j < S; ++j) {
    int o, w;
    wide_split(W, j, S, o, w);
    AttnArgs aj = a;
    aj.L = a.L - o;
    aj.R = o + w - 1 - a.L;
    wa.first = j == 0;
    sattn_status r;
    switch (cw_of(w)) {
      case 32: r = bwd_wide_sub<32>(aj, st, wa); break;
      case 48: r = bwd_wide_sub<48>(aj, st, wa); break;
      case 64: r = bwd_wide_sub<64>(aj, st, wa); break;
      case 72: r = bwd_wide_sub<72>(aj, st, wa); break;
      case 80: r = bwd_wide_sub<80>(aj, st, wa); break;
      default: g_tc_err = "wide sub-band"; return SATTN_EUNSUPPORTED;
    }
    if (r != SATTN_OK) return r;
  }
  const long long n8 = rows * 64 / 8;
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dq, reinterpret_cast<bf16*>(a.dQ), n8);
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dk, reinterpret_cast<bf16*>(a.dK), n8);
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dv, reinterpret_cast<bf16*>(a.dV), n8);
  return SATTN_OK;
}

// stored-band mode, wide bands (W > 49): the stored row a_t [0, W) is cut into 48-column sub-bands
// (16-byte aligned column offsets; the last one ends at W, where the row's padding is zero), each
// an SA band of its own with (L_j, R_j) as above whose probabilities are those columns of a_t.
// The gradient is the sum of the sub-bands' gradients with the global delta = dO . O (G28): the
// stored-band K1 / K2 ACC instances accumulate into fp32, then one kernel rounds.
constexpr int kWideSubP = 48;

template <int CW>
sattn_status bwd_p_wide_sub(const AttnArgs& a, int row, cudaStream_t st, const WideAcc& wa) {
  using K2 = DkvCfg<CW>;
  constexpr int NK = nk_of(CW);
  const int Tp = (a.T + 3) & ~3;
  CUtensorMap mp128, mk, mv, mdo, mqN, mpN, mv128, mdoN, mdel;
  if (!make_map_p(&mp128, a.P, a.T, a.BH, a.ldp, kM, row) || !make_map(&mk, a.K, a.T, a.BH, NK) ||
      !make_map(&mv, a.V, a.T, a.BH, NK) || !make_map(&mdo, a.dO, a.T, a.BH, kM) ||
      !make_map(&mqN, a.Q, a.T, a.BH, K2::NQ) || !make_map_p(&mpN, a.P, a.T, a.BH, a.ldp, K2::NQ, row) ||
      !make_map(&mv128, a.V, a.T, a.BH, kM) || !make_map(&mdoN, a.dO, a.T, a.BH, K2::NQ) ||
      !make_map_f32_rows(&mdel, a.delta, a.T, Tp, a.BH, K2::NQP))
    return SATTN_ECUDA;
  TcArgs t = tc_args(a);
  t.acc_dq = wa.dq; t.acc_dk = wa.dk; t.acc_dv = wa.dv; t.acc_first = wa.first;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  set_smem(sa_bwd_dq_tc<CW, true, true>, DqCfg<CW>::SMEM);
  launch_pdl(sa_bwd_dq_tc<CW, true, true>, dim3(grid), dim3(DqCfg<CW>::THREADS), DqCfg<CW>::SMEM, st, mp128, mk, mv,
             mdo, mp128, t);
  set_smem(sa_bwd_dkdv_tc<CW, true, true>, K2::SMEM_P);
  launch_pdl(sa_bwd_dkdv_tc<CW, true, true>, dim3(grid), dim3(K2::THREADS), K2::SMEM_P, st, mqN, mpN, mv128, mdoN,
             mqN, mqN, mdel, mdel, t);
  return SATTN_OK;
}

int tc_wide_p_parts(int L, int R) { return (L + R + 1 + kWideSubP - 1) / kWideSubP; }

sattn_status tc_backward_p_wide(const AttnArgs& a, cudaStream_t st) {
  const int W = a.L + a.R + 1, S = tc_wide_p_parts(a.L, a.R);
  const long long rows = (long long)a.BH * a.T;
  const int Tp = (a.T + 3) & ~3;
  WideAcc wa{};
  wa.dq = a.delta + 2LL * a.BH * Tp;
  wa.dk = wa.dq + rows * 64;
  wa.dv = wa.dk + rows * 64;
  wide_delta_kernel<<<4 * num_sms(), 256, 0, st>>>(reinterpret_cast<const bf16*>(a.dO), reinterpret_cast<const bf16*>(a.O),
                                                   a.delta, a.T, Tp, (long long)a.BH * Tp);
  for (int j = 0; j < S; ++j) {
    const int o = j * kWideSubP, w = W - o < kWideSubP ? W - o : kWideSubP;
    AttnArgs aj = a;
    aj.L = a.L - o;
    aj.R = o + w - 1 - a.L;
    aj.P = reinterpret_cast<bf16*>(a.P) + o;
    aj.ldp = (w + 7) & ~7;
    wa.first = j == 0;
    sattn_status r;
    switch (cw_of(w)) {
      case 32: r = bwd_p_wide_sub<32>(aj, a.ldp, st, wa); break;
      case 48: r = bwd_p_wide_sub<48>(aj, a.ldp, st, wa); break;
      case 64: r = bwd_p_wide_sub<64>(aj, a.ldp, st, wa); break;
      case 72: r = bwd_p_wide_sub<72>(aj, a.ldp, st, wa); break;
      case 80: r = bwd_p_wide_sub<80>(aj, a.ldp, st, wa); break;
      default: g_tc_err = "wide stored-band sub-band"; return SATTN_EUNSUPPORTED;
    }
    if (r != SATTN_OK) return r;
  }
  const long long n8 = rows * 64 / 8;
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dq, reinterpret_cast<bf16*>(a.dQ), n8);
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dk, reinterpret_cast<bf16*>(a.dK), n8);
  f32_to_bf16_kernel<<<4 * num_sms(), 256, 0, st>>>(wa.dv, reinterpret_cast<bf16*>(a.dV), n8);
  return SATTN_OK;
}

bool tc_supported(int dtype, int D, int L, int R, bool llsa, bool backward) {
  if (llsa || dtype != SATTN_BF16 || D != 64) return false;
  const int W = L + R + 1;
  // TMEM (NK + 64 <= 256 per buffer) -> CW <= 96, i.e. W <= 65, forward and backward (the
  // backward takes the block-ring dK/dV kernel beyond CW = 80)
  (void)backward;
  return W + 31 <= 96;
}

sattn_status tc_forward(const AttnArgs& a0, cudaStream_t st) {
  const AttnArgs a = flat_view(a0);
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

sattn_status tc_backward(const AttnArgs& a, cudaStream_t st) { return tc_backward_phase(a, st, 3); }

sattn_status tc_backward_phase(const AttnArgs& a0, cudaStream_t st, int phase) {
  // packed tiles only when one call runs both kernels (K1's delta rows are K2's input layout) and
  // the band takes the two-stage K2 (the block-ring K2 for CW = 96 keeps the per-head tiling)
  const int cw = cw_of(a0.L + a0.R + 1);
  const AttnArgs a = phase == 3 && cw > 0 && cw <= 80 ? flat_view(a0) : a0;
  switch (cw) {
    case 32: return bwd_launch<32>(a, st, phase);
    case 48: return bwd_launch<48>(a, st, phase);
    case 64: return bwd_launch<64>(a, st, phase);
    case 72: return bwd_launch<72>(a, st, phase);
    case 80: return bwd_launch<80>(a, st, phase);
    case 96: return bwd_launch<96>(a, st, phase);
  }
  g_tc_err = "band too wide for the tensor-core kernels";
  return SATTN_EUNSUPPORTED;
}

int tc_backward_launches() { return 2; }
int tc_key_box_rows(int L, int R) { const int cw = cw_of(L + R + 1); return cw > 0 ? nk_of(cw) : -1; }

// ---- stored-band mode (NEXT-4): forward W <= 64 (P staging rows fit the O tile), backward
// W <= 49 (the P window replaces K in the two-stage K2 stage; for W > 41 with one dV/dK
// staging tile per warpgroup)
bool tc_p_supported(int dtype, int D, int L, int R, bool backward) {
  const int W = L + R + 1;
  if (dtype != SATTN_BF16 || D != 64 || L < 0 || R < 0) return false;
  return backward ? cw_of(W) > 0 && cw_of(W) <= 80 : W <= 64;
}

sattn_status tc_forward_p(const AttnArgs& a0, cudaStream_t st) {
  const AttnArgs a = flat_view(a0);
  switch (cw_of(a.L + a.R + 1)) {
    case 32: return fwd_launch<32, true>(a, st);
    case 48: return fwd_launch<48, true>(a, st);
    case 64: return fwd_launch<64, true>(a, st);
    case 72: return fwd_launch<72, true>(a, st);
    case 80: return fwd_launch<80, true>(a, st);
    case 96: return fwd_launch<96, true>(a, st);
  }
  g_tc_err = "band too wide for the tensor-core stored-band forward";
  return SATTN_EUNSUPPORTED;
}

// phase as bwd_launch: bit 0 = K1 over the launch's query tiles, bit 1 = K2 over every key tile
template <int CW>
sattn_status bwd_p_launch(const AttnArgs& a, cudaStream_t st, int phase = 3) {
  using K2 = DkvCfg<CW>;
  static_assert(K2::SMEM_P <= 232448, "stored-band K2 stage");
  constexpr int NK = nk_of(CW);
  const int Tp = (a.T + 3) & ~3;
  const int ld = a.ld;
  CUtensorMap mp128, mk, mv, mdo, mdq, mqN, mpN, mv128, mdoN, mdk, mdv, mdel;
  if (!make_map_p(&mp128, a.P, a.T, a.BH, a.ldp, kM, 0, ld) || !make_map(&mk, a.K, a.T, a.BH, NK, ld) ||
      !make_map(&mv, a.V, a.T, a.BH, NK, ld) || !make_map(&mdo, a.dO, a.T, a.BH, kM, ld) ||
      !make_map(&mdq, a.dQ, a.T, a.BH, kM, ld) || !make_map(&mqN, a.Q, a.T, a.BH, K2::NQ, ld) ||
      !make_map_p(&mpN, a.P, a.T, a.BH, a.ldp, K2::NQ, 0, ld) || !make_map(&mv128, a.V, a.T, a.BH, kM, ld) ||
      !make_map(&mdoN, a.dO, a.T, a.BH, K2::NQ, ld) || !make_map(&mdk, a.dK, a.T, a.BH, kM, ld) ||
      !make_map(&mdv, a.dV, a.T, a.BH, kM, ld) || !make_map_f32_rows(&mdel, a.delta, a.T, Tp, a.BH, K2::NQP))
    return SATTN_ECUDA;
  if (phase & 1) {
    const TcArgs t1 = tc_args(a);
    const int nt1 = t1.nkt * a.BH;
    set_smem(sa_bwd_dq_tc<CW, true>, DqCfg<CW>::SMEM);
    launch_pdl(sa_bwd_dq_tc<CW, true>, dim3(nt1 < num_sms() ? nt1 : num_sms()), dim3(DqCfg<CW>::THREADS),
               DqCfg<CW>::SMEM, st, mp128, mk, mv, mdo, mdq, t1);
  }
  if (!(phase & 2)) return SATTN_OK;
  const int ntiles = (a.T + kM - 1) / kM * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  set_smem(sa_bwd_dkdv_tc<CW, true>, K2::SMEM_P);
  launch_pdl(sa_bwd_dkdv_tc<CW, true>, dim3(grid), dim3(K2::THREADS), K2::SMEM_P, st, mqN, mpN, mv128, mdoN, mdk,
             mdv, mdel, mdel, tc_args(a));
  return SATTN_OK;
}

sattn_status tc_backward_p_phase(const AttnArgs& a0, cudaStream_t st, int phase) {
  const AttnArgs a = phase == 3 ? flat_view(a0) : a0;   // packed tiles: as tc_backward_phase
  switch (cw_of(a.L + a.R + 1)) {
    case 32: return bwd_p_launch<32>(a, st, phase);
    case 48: return bwd_p_launch<48>(a, st, phase);
    case 64: return bwd_p_launch<64>(a, st, phase);
    case 72: return bwd_p_launch<72>(a, st, phase);
    case 80: return bwd_p_launch<80>(a, st, phase);
  }
  g_tc_err = "band too wide for the tensor-core stored-band backward";
  return SATTN_EUNSUPPORTED;
}

sattn_status tc_backward_p(const AttnArgs& a, cudaStream_t st) { return tc_backward_p_phase(a, st, 3); }
size_t tc_backward_ws_bytes() { return 0; }

bool tc_llsa_bwd_supported(int dtype, int D, int L, int R) {
  // band width L+1 on the SA kernels (CW <= 80), staircase staging of 16 + 2R frames x C channels
  return dtype == SATTN_BF16 && D == 64 && R >= 1 && R <= 8 && L + 1 + 31 <= 80;
}

bool tc_llsa_bwd_any_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense) {
  return tc_llsa_bwd_supported(dtype, D, L, R) ||
         (L + 1 + 31 <= 80 && tc_llsa_bwd_fused_supported(dtype, D, L, R, BH, T, dense));
}

sattn_status tc_llsa_backward(const AttnArgs& a, cudaStream_t st) { return tc_llsa_backward_phase(a, st, 3, nullptr); }

sattn_status tc_llsa_backward_phase(const AttnArgs& a, cudaStream_t st, int phase, const int* sub4) {
  if ((phase != 3 || sub4) &&
      !tc_llsa_bwd_fused_supported(SATTN_BF16, kD, a.L, a.R, a.BH, a.T, a.in_cs != 0)) {
    g_tc_err = "LLSA backward phases need the fused horizon-major pass (dense inputs)";
    return SATTN_EUNSUPPORTED;
  }
  switch (cw_of(a.L + 1)) {
    case 32: return llsa_bwd_launch<32>(a, st, phase, sub4);
    case 48: return llsa_bwd_launch<48>(a, st, phase, sub4);
    case 64: return llsa_bwd_launch<64>(a, st, phase, sub4);
    case 72: return llsa_bwd_launch<72>(a, st, phase, sub4);
    case 80: return llsa_bwd_launch<80>(a, st, phase, sub4);
  }
  g_tc_err = "band too wide for the LLSA tensor-core backward";
  return SATTN_EUNSUPPORTED;
}

int tc_llsa_backward_launches(const AttnArgs& a) {
  return tc_llsa_bwd_fused_supported(SATTN_BF16, kD, a.L, a.R, a.BH, a.T, a.in_cs != 0) ? 2 : 4;
}
void tc_set_trace(void* p) { g_trace = static_cast<long long*>(p); }
const char* tc_last_error() { return g_tc_err.c_str(); }

}  // namespace sattn
