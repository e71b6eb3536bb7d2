// tc_llsa.cu — tensor-core LLSA forward (Eq. 14-15 in the horizon form; bf16, D = 64).
//
// Work unit: a horizon tile h in [h0, h0 + 32) of one (batch, head).  Output (t, c) has
// horizon h = t + c (reading G6) and attends
//   band   (u, R) for u in [h-R-L, h-R]      -- channel R, shared by every output of the tile
//   stair  (h-c', c') for c' = 0 .. R-1      -- one key per stair channel, per horizon
// An item is 128 output rows = 4 channels x 32 horizons (row r = 32 * (c % 4) + i): one warp
// per channel, lane = horizon offset i, TMEM lane = row.
//   S_band = Q K_band^T                       tcgen05, M = 128, N = NB = 16-rounded 32 + L
//   s_stair[c'] = q . k_stair[c'][i]           CUDA cores, from the staged stair tiles (smem)
//   softmax over band strip + stair scores     registers (row max / sum)
//   O = [P_band | P_stair] [V_band ; V_stair]   ONE tcgen05 chain, K = NB + 32 R: P_stair is the
//                                              sparse row (entry 32 c' + i per stair block)
//                                              written into TMEM next to P_band
// The band / stair K, V of a horizon tile are staged once (2-stage ring) and reused by the
// ceil(C / 4) items of the tile; Q arrives per item (2-stage ring).  Warp roles as in tc_sa.cu:
// TMA producer, MMA issuer, two softmax / epilogue warpgroups alternating items.
#include <cuda.h>

#include <cstdlib>
#include <string>
#include <utility>

#include "ffma_attn.cuh"
#include "tc_dispatch.h"
#include "tc_ptx.cuh"
#include "host_util.h"
#include "llsa_stair.cuh"

namespace sattn {
namespace {

thread_local std::string g_err;
long long* g_llsa_trace = nullptr;   // debug: device buffer [16][64] for the fused backward's CTA 0
constexpr int kD = 64;
constexpr int kHT = 32;          // horizons per tile
constexpr int kRmax = 8;

struct LlsaArgs {
  int T, L, R, C, BH;
  int bcast;                     // inputs are one plane read as every channel (layer 1)
  int skew;                      // stair K/V and item Q staged by one skewed 4-D box each (see map_skew)
  float scale, scale_log2;
  float* LSE;                    // [C][BH][T]
  bf16* O;                       // [C][BH][T][64] (direct stores of the first tile)
};

template <int NB> struct LCfg {
  static constexpr int BB = NB * 128;                 // band K (or V) tile bytes
  static constexpr int SB = kHT * 128;                // one stair tile (32 rows) bytes
  static constexpr int HSTAGE = 2 * BB + 2 * kRmax * SB;   // K_band, V_band, K_stair[8], V_stair[8]
  static constexpr int QB = 128 * 128;                // item Q tile (128 rows)
  static constexpr int NSQ = 2;
  static constexpr int OB = 128 * 128;                // O staging per warpgroup
  static constexpr int SMEM = 1024 + 2 * HSTAGE + NSQ * QB + 2 * OB + 512;
  static constexpr int PCOLS = (NB + 32 * kRmax) / 2; // packed P columns (<= 160)
  static constexpr int OCOL = 192;                    // O accumulator column within a 256-col buffer
  static_assert(PCOLS <= OCOL, "P region overlaps O");
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int NB>
__global__ void __launch_bounds__(320, 1)
    llsa_fwd_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKb,
                const __grid_constant__ CUtensorMap tmVb, const __grid_constant__ CUtensorMap tmKs,
                const __grid_constant__ CUtensorMap tmVs, const __grid_constant__ CUtensorMap tmO, LlsaArgs a) {
  using Cf = LCfg<NB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* hstage0 = smem;                               // [Kb | Vb | Ks x8 | Vs x8] x 2
  uint8_t* qstage0 = smem + 2 * Cf::HSTAGE;
  uint8_t* obuf0 = qstage0 + Cf::NSQ * Cf::QB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(obuf0 + 2 * Cf::OB);
  uint64_t* hfull = bars;        // [2]
  uint64_t* hempty = hfull + 2;  // [2]
  uint64_t* qfull = hempty + 2;  // [NSQ]
  uint64_t* qempty = qfull + Cf::NSQ;
  uint64_t* sfull = qempty + Cf::NSQ;  // [2]
  uint64_t* pfull = sfull + 2;         // [2] (128)
  uint64_t* ofull = pfull + 2;         // [2]
  uint64_t* tfree = ofull + 2;         // [2] (128)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, L = a.L, R = a.R, C = a.C;
  const int NI = (C + 3) / 4;                            // items per horizon tile
  const int nht = (T + R + kHT - 1) / kHT;               // horizons 0 .. T-1+R
  const int ntiles = nht * a.BH;
  const int ntile_me = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nitems = ntile_me * NI;

  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmKb); tc::tma_prefetch_desc(&tmVb);
    tc::tma_prefetch_desc(&tmKs); tc::tma_prefetch_desc(&tmVs); tc::tma_prefetch_desc(&tmO);
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&hfull[i], 1); tc::mbar_init(&hempty[i], 1); }
    for (int i = 0; i < Cf::NSQ; ++i) { tc::mbar_init(&qfull[i], 1); tc::mbar_init(&qempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&pfull[i], 128);
      tc::mbar_init(&ofull[i], 1); tc::mbar_init(&tfree[i], 128);
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

  auto chan = [&](int c) { return a.bcast ? 0 : c; };   // channel coordinate of an input plane

  if (warp == 0) {
    if (lane == 0) {
      int k = 0;                                          // item counter (Q ring)
      for (int kt = 0; kt < ntile_me; ++kt) {
        const int g = blockIdx.x + kt * gridDim.x;
        const int bh = g / nht, h0 = (g % nht) * kHT;
        const int hs = kt & 1;
        if (kt >= 2) tc::mbar_wait(&hempty[hs], ((kt - 2) >> 1) & 1);
        uint8_t* hb = hstage0 + hs * Cf::HSTAGE;
        tc::mbar_expect_tx(&hfull[hs], 2 * Cf::BB + 2 * R * Cf::SB);
        tc::tma_load_4d(hb, &tmKb, &hfull[hs], 0, h0 - R - L, bh, chan(R));
        tc::tma_load_4d(hb + Cf::BB, &tmVb, &hfull[hs], 0, h0 - R - L, bh, chan(R));
        if (a.skew) {   // rows (h0 - c' + i, c') for all c' < R: one box each for K and V
          tc::tma_load_4d(hb + 2 * Cf::BB, &tmKs, &hfull[hs], 0, h0, 0, bh);
          tc::tma_load_4d(hb + 2 * Cf::BB + kRmax * Cf::SB, &tmVs, &hfull[hs], 0, h0, 0, bh);
        } else {
          for (int cp = 0; cp < R; ++cp) {
            tc::tma_load_4d(hb + 2 * Cf::BB + cp * Cf::SB, &tmKs, &hfull[hs], 0, h0 - cp, bh, chan(cp));
            tc::tma_load_4d(hb + 2 * Cf::BB + (kRmax + cp) * Cf::SB, &tmVs, &hfull[hs], 0, h0 - cp, bh, chan(cp));
          }
        }
        for (int ii = 0; ii < NI; ++ii, ++k) {
          const int qs = k % Cf::NSQ;
          if (k >= Cf::NSQ) tc::mbar_wait(&qempty[qs], ((k - Cf::NSQ) / Cf::NSQ) & 1);
          uint8_t* qb = qstage0 + qs * Cf::QB;
          tc::mbar_expect_tx(&qfull[qs], Cf::QB);
          if (a.skew) {   // rows (h0 - c + i, c) of the item's 4 channels (channels >= C zero-filled)
            tc::tma_load_4d(qb, &tmQ, &qfull[qs], 0, h0, 4 * ii, bh);
            continue;
          }
          for (int w = 0; w < 4; ++w) {
            const int c = 4 * ii + w;
            // channels >= C: a box entirely past the end of the sequence (zero-filled)
            const int f = c < C ? h0 - c : T + 64;
            tc::tma_load_4d(qb + w * kHT * 128, &tmQ, &qfull[qs], 0, f, bh, chan(c < C ? c : 0));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, NB, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, kD, 0, 1);
      const int nstair = 2 * R;                           // 16-row k-steps over the stair V blocks
      int ns = 0, np = 0;
      int kts = 0, nsi = 0;                               // ns / NI, ns % NI (no division in the poll loop)
      while (np < nitems) {
        const uint32_t m = tc::mbar_test4(tc::smem_u32(&hfull[kts & 1]), (kts >> 1) & 1,
                                          tc::smem_u32(&qfull[ns % Cf::NSQ]), (ns / Cf::NSQ) & 1,
                                          tc::smem_u32(&pfull[np & 1]), (np >> 1) & 1,
                                          tc::smem_u32(&tfree[np & 1]), ((np + 2) >> 1) & 1);   // = (np-2)>>1 parity
        if (ns < nitems && ns < np + 2) {
          const int kt = kts, qs = ns % Cf::NSQ;
          if ((m & 1) && (m & 2)) {
            tc::tc_fence_after();
            const uint32_t q = tc::smem_u32(qstage0 + qs * Cf::QB);
            const uint32_t kb = tc::smem_u32(hstage0 + (kt & 1) * Cf::HSTAGE);
            const uint32_t d = tbase + (ns & 1) * 256;
#pragma unroll
            for (int j = 0; j < kD / 16; ++j)
              tc::mma_bf16(d, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(kb + 32 * j), idS, j > 0);
            tc::mma_commit(&sfull[ns & 1]);
            ++ns;
            if (++nsi == NI) { nsi = 0; ++kts; }
            continue;
          }
        }
        if (np < ns && (m & 4) && (np < 2 || (m & 8))) {
          tc::tc_fence_after();
          const int kt = np / NI, b = np & 1;
          const uint32_t hb = tc::smem_u32(hstage0 + (kt & 1) * Cf::HSTAGE);
          const uint32_t vb = hb + Cf::BB, vs = hb + 2 * Cf::BB + kRmax * Cf::SB;
          const uint32_t pa = tbase + b * 256;
          const uint32_t d = pa + Cf::OCOL;
#pragma unroll
          for (int j = 0; j < NB / 16; ++j)
            tc::mma_bf16_ts(d, pa + 8 * j, tc::desc_mnmajor_sw128(vb + 2048 * j), idO, j > 0);
          for (int j = 0; j < nstair; ++j)
            tc::mma_bf16_ts(d, pa + NB / 2 + 8 * j, tc::desc_mnmajor_sw128(vs + 2048 * j), idO, 1);
          tc::mma_commit(&ofull[b]);
          tc::mma_commit(&qempty[np % Cf::NSQ]);
          if (np % NI == NI - 1) tc::mma_commit(&hempty[kt & 1]);   // last item of the tile
          ++np;
        }
      }
    }
  } else {
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const int i = lane;                                  // horizon offset within the tile
    const uint32_t lanes = uint32_t(32 * q4) << 16;
    uint8_t* ostage = obuf0 + wg * Cf::OB + q4 * kHT * 128;   // this warp's 32 staging rows
    for (int k = wg; k < nitems; k += 2) {
      const int kt = k / NI, ii = k % NI, b = k & 1, use = k >> 1, qs = k % Cf::NSQ;
      const int g = blockIdx.x + kt * gridDim.x;
      const int bh = g / nht, h0 = (g % nht) * kHT;
      const int c = 4 * ii + q4;                         // output channel of this warp
      if (c >= C) {
        // padding rows of the last item (C = 9 channels in items of 4): no scores, softmax or
        // epilogue, but the same barrier sequence so the arrivals of consecutive items never mix
        // (their TMEM rows hold garbage that the PV MMA turns into garbage O rows, never stored)
        tc::mbar_wait(&sfull[b], use & 1);
        tc::tc_fence_after();
        tc::tc_fence_before();
        tc::mbar_arrive(&pfull[b]);
        tc::mbar_wait(&ofull[b], use & 1);
        tc::tc_fence_after();
        tc::tc_fence_before();
        tc::mbar_arrive(&tfree[b]);
        continue;
      }
      const int h = h0 + i, t = h - c;
      const uint8_t* hb = hstage0 + (kt & 1) * Cf::HSTAGE;
      tc::mbar_wait(&hfull[kt & 1], (kt >> 1) & 1);
      tc::mbar_wait(&qfull[qs], (k / Cf::NSQ) & 1);
      // ---- stair scores on CUDA cores: q_{t,c} . k_{h-c', c'} (row i of stair tile c')
      float sst[kRmax];
      {
        // q as fp32 pairs; k_stair rows unpacked with shifts (bf16 -> fp32 is a 16-bit shift)
        // and accumulated with packed fp32x2 FMAs (sm_100 FFMA2): the dot products are the
        // WG's largest instruction block (ncu: ~1/3 of the kernel's instructions before)
        float2 q2[kD / 2];
        const uint32_t qrow = tc::smem_u32(qstage0 + qs * Cf::QB) + r * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint4 x = tc::ld_shared_v4(qrow + ((ch ^ (r & 7)) << 4));
          const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            q2[4 * ch + e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
        }
#pragma unroll
        for (int cp = 0; cp < kRmax; ++cp) {
          float2 acc = make_float2(0.f, 0.f);
          if (cp < R) {
            const uint32_t krow = tc::smem_u32(hb + 2 * Cf::BB + cp * Cf::SB) + i * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 x = tc::ld_shared_v4(krow + ((ch ^ (i & 7)) << 4));
              const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                acc = __ffma2_rn(q2[4 * ch + e],
                                 make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u)), acc);
            }
          }
          const int f = h - cp;                           // stair key frame
          sst[cp] = (cp < R && f >= 0 && f < T) ? acc.x + acc.y : neg_inf();
        }
      }
      // ---- band strip from TMEM + joint softmax
      tc::mbar_wait(&sfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      float s[NB];
      const uint32_t pa = tbase + lanes + b * 256;
#pragma unroll
      for (int j = 0; j < NB / 8; ++j) tc::tmem_ld8(pa + 8 * j, s + 8 * j);
      tc::tmem_ld_wait();
      const int key0 = h0 - R - L;                       // frame of band column 0
      const int jlo = max(i, -key0), jhi = min(i + L, T - 1 - key0);   // valid band columns [jlo, jhi]
      float m = neg_inf();
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        s[j] = (j >= jlo && j <= jhi) ? s[j] : neg_inf();
        m = fmaxf(m, s[j]);
      }
#pragma unroll
      for (int cp = 0; cp < kRmax; ++cp) m = fmaxf(m, sst[cp]);
      const float mref = m == neg_inf() ? 0.f : m;
      const float mb = mref * a.scale_log2;
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        s[j] = tc::ex2(fmaf(s[j], a.scale_log2, -mb));
        l += s[j];
      }
#pragma unroll
      for (int cp = 0; cp < kRmax; ++cp) {
        sst[cp] = tc::ex2(fmaf(sst[cp], a.scale_log2, -mb));
        l += sst[cp];
      }
      // ---- P row into TMEM (packed bf16 A operand): band part, then the sparse stair part
#pragma unroll
      for (int j = 0; j < NB / 8; ++j)
        tc::tmem_st4(pa + 4 * j, pack_bf16(s[8 * j], s[8 * j + 1]), pack_bf16(s[8 * j + 2], s[8 * j + 3]),
                     pack_bf16(s[8 * j + 4], s[8 * j + 5]), pack_bf16(s[8 * j + 6], s[8 * j + 7]));
      {
        const int mc = i >> 1;   // packed column of element i (low half if i is even)
#pragma unroll
        for (int cp = 0; cp < kRmax; ++cp) {
          if (cp >= R) break;
          const uint32_t pv = (i & 1) ? pack_bf16(0.f, sst[cp]) : pack_bf16(sst[cp], 0.f);
#pragma unroll
          for (int q4c = 0; q4c < 4; ++q4c) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) w4[e] = (4 * q4c + e == mc) ? pv : 0u;
            tc::tmem_st4(pa + NB / 2 + 16 * cp + 4 * q4c, w4[0], w4[1], w4[2], w4[3]);
          }
        }
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&pfull[b]);
      // ---- epilogue: O / l -> staging -> TMA store of this warp's channel rows
      tc::mbar_wait(&ofull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      if (lane == 0) tc::bulk_wait_read0();
      __syncwarp();
      // a TMA store box may not start before frame 0: the first horizon tile's rows of
      // channels c > 0 (frames h0 - c < 0) are stored directly from registers instead
      const bool direct = h0 - c < 0;
      {
        float v[kD];
#pragma unroll
        for (int j = 0; j < 4; ++j) tc::tmem_ld16(pa + Cf::OCOL + 16 * j, v + 16 * j);
        tc::tmem_ld_wait();
        const float inv = 1.f / l;
        uint4 w8[8];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          w8[ch] = make_uint4(pack_bf16(v[8 * ch] * inv, v[8 * ch + 1] * inv),
                              pack_bf16(v[8 * ch + 2] * inv, v[8 * ch + 3] * inv),
                              pack_bf16(v[8 * ch + 4] * inv, v[8 * ch + 5] * inv),
                              pack_bf16(v[8 * ch + 6] * inv, v[8 * ch + 7] * inv));
        if (direct) {
          if (c < C && t >= 0 && t < T) {
            uint4* dst = reinterpret_cast<uint4*>(a.O + (((long long)c * a.BH + bh) * T + t) * kD);
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) dst[ch] = w8[ch];
          }
        } else {
          const uint32_t row = tc::smem_u32(ostage) + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) tc::st_shared_v4(row + ((ch ^ (lane & 7)) << 4), w8[ch]);
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tfree[b]);
      if (c < C && t >= 0 && t < T) a.LSE[((long long)c * a.BH + bh) * T + t] = mref * a.scale + __log2f(l) * kLn2;
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && c < C && !direct) {
        tc::tma_store_4d(&tmO, ostage, 0, h0 - c, bh, c);   // rows at or past T are clipped
        tc::bulk_commit();
      }
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// LLSA backward, fused horizon-major pass (dense inputs).  Exact gradient of the
// forward above (Eq. 14-16 in the horizon form, reading G8/G9), everything except the band
// keys' dK / dV (channel R, which gather from L+1 horizons and are the key-major llsa_bwd_kv_tc):
//
// Item = HZ horizons x all C channels of one (b, h): row r = c HZ + i <-> output (t, c),
// t = h0 + i - c (so the C rows of a horizon, and therefore every query of its staircase
// keys, sit in one item).  Per item, with TMEM buffer b (256 columns) and stage b:
//   MMA  S   = Q Kb^T -> X_b[0, NB)              WG  stair scores / dP on CUDA cores (FFMA2)
//                                                     P = exp2(S sl2 - LSE log2e) (band + stair)
//   MMA  dP  = dO Vb^T -> X_b[0, NB)             WG  delta = rowsum(P o dP) over band + stair (G26,
//                                                     complete: no pre-pass), dS = P (dP - delta);
//                                                     dS_band -> X_b (packed bf16 A operand);
//                                                     dS_stair, P_stair -> DS, PS (smem, sparse)
//   MMA  dQ  = [dS_band | DS] [Kb ; Ks]   -> X_b[NB, NB+64)     (complete: one rounding)
//        dKs = DS^T Q  (A MN-major)        -> X_b[NB+64, NB+128) (staircase keys: complete)
//        dVs = PS^T dO                     -> X_b[NB+128, NB+192)
//                                             WG  epilogue: dQ, dK_stair, dV_stair rows -> global;
//                                                 delta, LSE log2e rows -> workspace (llsa_bwd_kv_tc)
// DS / PS are [2 K-atoms][128 rows][128 B] K-major SW128 tiles: row r holds its R staircase
// entries at columns c' HZ + i (fixed per row), every other entry stays zero from the start.
// Warp roles as in the forward: TMA producer, MMA issuer, two warpgroups alternating items.
// ------------------------------------------------------------------------------------------
// items of a launch per (b, h): item j = it0 + i + (i >= it_split ? it_jump : 0), i < nit_l (all
// items: it0 = 0, nit_l = ceil((T + R) / HZ), it_split = nit_l, it_jump = 0; a time shard launches
// its interior items during the halo exchange and the edge items after it)
struct ItemSub {
  int it0, nit_l, it_split, it_jump;
};
__host__ __device__ __forceinline__ int item_j(int i, const ItemSub& u) {
  return u.it0 + i + (i >= u.it_split ? u.it_jump : 0);
}
ItemSub all_items(const AttnArgs& a, int HZ) {
  const int n = (a.T + a.R + HZ - 1) / HZ;   // horizons 0 .. T-1+R per (b, h)
  return ItemSub{0, n, n, 0};
}

struct LlsaBwdArgs {
  int T, L, R, C, BH, HZ, Tp;
  ItemSub sub;
  float scale, scale_log2;
  const float* LSE;              // [C][BH][T]
  bf16 *dQ, *dK, *dV;            // [C][BH][T][64]
  float *ws_del, *ws_l2;         // [C][BH][Tp], or [C][Tp] over the flattened BH*T axis (ws_flat)
  int ws_flat;                   // rows for the packed-tile kv pass: index c Tp + bh T + t, Tp = BH*T rounded to 4
  long long* trace;              // debug: per-item phase clock64 stamps of CTA 0 ([16][64]), or null
};

template <int NB, int RM, bool HM = false> struct LBCfg {
  static constexpr int QB = 128 * 128;             // Q / dO item tiles
  static constexpr int KBB = NB * 128;             // band K / V tiles
  static constexpr int SB = 112 * 128;             // stair K / V tiles (rows c' HZ + i, R HZ <= 112)
  static constexpr int STAGE = 2 * QB + 2 * KBB + 2 * SB;
  static constexpr int XB = 2 * 128 * 128;         // DS / PS
  // staircase scores / dP on mma.sync (16 x 8 blocks per horizon) through a per-warpgroup fp32
  // scratch [128][RM] (S, then dP), when it fits; otherwise packed-FFMA2 dot products
  static constexpr bool SMMA = !HM && 1024 + 2 * STAGE + 2 * XB + 2 * 128 * RM * 4 + 128 + 256 <= 232448;
  // both products in one pass through a [2][128][RM] scratch when that fits too (R <= 8)
  static constexpr bool SFUSE = SMMA && 1024 + 2 * STAGE + 2 * XB + 2 * 2 * 128 * RM * 4 + 128 + 256 <= 232448;
  static constexpr int SCR = SMMA ? (SFUSE ? 2 : 1) * 128 * RM * 4 : 0;   // per warpgroup (none for HM)
  static constexpr int SMEM = 1024 + 2 * STAGE + 2 * XB + 2 * SCR + 128 + 256;
  static_assert(NB + 192 <= 256, "TMEM columns per item");
  static_assert(SMEM <= 232448, "shared memory");
};

// byte address of element (row r, column k) of a [2][128][128 B] K-major SW128 tile
__device__ __forceinline__ uint32_t xs_addr(uint32_t base, int r, int k) {
  const int e = k & 63;
  return base + (k >> 6) * 16384 + r * 128 + ((((e >> 3) ^ (r & 7))) << 4) + (e & 7) * 2;
}

__device__ __forceinline__ void tmem_ld64_l(uint32_t addr, float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) tc::tmem_ld16(addr + 16 * j, v + 16 * j);
  tc::tmem_ld_wait();
}
// 64 fp32 values (x sc) -> bf16 row r of a 128-row x 128-byte smem tile with the 128B swizzle
__device__ __forceinline__ void tmem_row64_to_smem_sw128_regs(const float* v, float sc, uint8_t* tile, int r) {
  const uint32_t row = tc::smem_u32(tile) + r * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    tc::st_shared_v4(row + ((c ^ (r & 7)) << 4),
                     make_uint4(pack_bf16(v[8 * c] * sc, v[8 * c + 1] * sc), pack_bf16(v[8 * c + 2] * sc, v[8 * c + 3] * sc),
                                pack_bf16(v[8 * c + 4] * sc, v[8 * c + 5] * sc), pack_bf16(v[8 * c + 6] * sc, v[8 * c + 7] * sc)));
}
// 64 fp32 -> bf16 (x sc) -> 128 contiguous bytes in global memory
__device__ __forceinline__ void store_row64(bf16* dst, const float* v, float sc) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int ch = 0; ch < 8; ++ch)
    d[ch] = make_uint4(pack_bf16(v[8 * ch] * sc, v[8 * ch + 1] * sc), pack_bf16(v[8 * ch + 2] * sc, v[8 * ch + 3] * sc),
                       pack_bf16(v[8 * ch + 4] * sc, v[8 * ch + 5] * sc), pack_bf16(v[8 * ch + 6] * sc, v[8 * ch + 7] * sc));
}

template <int NB, int RM, bool HM>
__global__ void __launch_bounds__(320, 1)
    llsa_bwd_fused_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                      const __grid_constant__ CUtensorMap tmKb, const __grid_constant__ CUtensorMap tmVb,
                      const __grid_constant__ CUtensorMap tmKs, const __grid_constant__ CUtensorMap tmVs,
                      const __grid_constant__ CUtensorMap tmdQ, const __grid_constant__ CUtensorMap tmdK,
                      const __grid_constant__ CUtensorMap tmdV, LlsaBwdArgs a) {
  // HM (horizon-major, R == RM): item rows r = i C + c and staircase keys m = i' RM + c' (the TMA
  // boxes are ordered so), the staircase S / dP as dense tcgen05 products Q Ks^T / dO Vs^T into
  // TMEM [NB, NB + HZ RM) (a row's R entries are the RM contiguous columns of its horizon), instead
  // of per-horizon mma.sync blocks through a shared-memory scratch (the legacy mma.sync rate bound
  // that phase)
  using Cf = LBCfg<NB, RM, HM>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage0 = smem;                                    // [Q | dO | Kb | Vb | Ks | Vs] x 2
  uint8_t* xds = smem + 2 * Cf::STAGE;                       // DS
  uint8_t* xps = xds + Cf::XB;                               // PS
  uint8_t* scr0 = xps + Cf::XB;                              // stair S / dP scratch x 2 warpgroups
  uint8_t* zrow = scr0 + 2 * Cf::SCR;                        // 128 zero bytes (ldmatrix padding rows)
  uint64_t* bars = reinterpret_cast<uint64_t*>(zrow + 128);
  uint64_t* full = bars;           // [2]
  uint64_t* empty = full + 2;      // [2]
  uint64_t* sfull = empty + 2;     // [2]
  uint64_t* xfree = sfull + 2;     // [2] (128)
  uint64_t* dpfull = xfree + 2;    // [2]
  uint64_t* dsfull = dpfull + 2;   // [2] (128)
  uint64_t* done = dsfull + 2;     // [2]
  uint64_t* tfree = done + 2;      // [2] (128)
  uint64_t* xsfree = tfree + 2;    // [1] DS / PS read by the item's MMAs
  uint64_t* emptyA = xsfree + 1;   // [2] the stage's dO / Kb / Vb read by the item's MMAs (not used
                                   //     as epilogue staging: reloaded before the stores finish)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(emptyA + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, L = a.L, R = a.R, C = a.C, HZ = a.HZ;
  const int nit = a.sub.nit_l;                               // items of this launch per (b, h)
  const int nitems = nit * a.BH;
  const int nme = blockIdx.x < nitems ? (nitems - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int qbytes = C * HZ * 128, sbytes = R * HZ * 128;

  // zero the operand tiles once: padding rows / columns that TMA and the warpgroups never write
  for (int o = tid * 16; o < 2 * Cf::STAGE + 2 * Cf::XB + 2 * Cf::SCR + 128; o += 320 * 16)
    *reinterpret_cast<uint4*>(smem + o) = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmdO); tc::tma_prefetch_desc(&tmKb);
    tc::tma_prefetch_desc(&tmVb); tc::tma_prefetch_desc(&tmKs); tc::tma_prefetch_desc(&tmVs);
    for (int i = 0; i < 2; ++i) {
      // the stage is released by the epilogue (after its TMA stores have read the staging rows)
      tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&xfree[i], 128); tc::mbar_init(&dpfull[i], 1);
      tc::mbar_init(&dsfull[i], 128); tc::mbar_init(&done[i], 1); tc::mbar_init(&tfree[i], 128);
    }
    tc::mbar_init(xsfree, 1);
    tc::mbar_init(&emptyA[0], 1); tc::mbar_init(&emptyA[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // L2 prefetch of the first items' boxes while the previous kernel drains (PDL; coherent L2)
  auto prefetch_l2 = [&](int k) {
    if (k >= nme) return;
    const int g = blockIdx.x + k * gridDim.x;
    const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
    tc::tma_prefetch_4d(&tmQ, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
    tc::tma_prefetch_4d(&tmdO, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
    tc::tma_prefetch_4d(&tmKb, 0, h0 - R - L, bh, R);
    tc::tma_prefetch_4d(&tmVb, 0, h0 - R - L, bh, R);
    tc::tma_prefetch_4d(&tmKs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
    tc::tma_prefetch_4d(&tmVs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
  };
  if (tid == 0)
    for (int k = 0; k < 2; ++k) prefetch_l2(k);
  tc::pdl_wait();
  tc::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // L2 prefetch of item k + 2's boxes when item k's loads are issued: its stage frees only after
      // item k's epilogue stores have read it, so the TMA loads then mostly hit L2
      auto prefetch = [&](int k) {
        if (k >= nme) return;
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
        tc::tma_prefetch_4d(&tmQ, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_prefetch_4d(&tmdO, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_prefetch_4d(&tmKb, 0, h0 - R - L, bh, R);
        tc::tma_prefetch_4d(&tmVb, 0, h0 - R - L, bh, R);
        tc::tma_prefetch_4d(&tmKs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_prefetch_4d(&tmVs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
      };
      for (int k = 0; k < nme; ++k) {
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
        const int s = k & 1;
        prefetch(k + 2);
        // dO / Kb / Vb as soon as the previous item on this stage has finished its MMAs; Q / Ks / Vs
        // (the epilogue's staging tiles) once its TMA stores have read them
        if (k >= 2) tc::mbar_wait(&emptyA[s], ((k - 2) >> 1) & 1);
        uint8_t* sb = stage0 + s * Cf::STAGE;
        tc::mbar_expect_tx(&full[s], 2 * qbytes + 2 * Cf::KBB + 2 * sbytes);
        tc::tma_load_4d(sb + Cf::QB, &tmdO, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_load_4d(sb + 2 * Cf::QB, &tmKb, &full[s], 0, h0 - R - L, bh, R);   // band keys (u, R)
        tc::tma_load_4d(sb + 2 * Cf::QB + Cf::KBB, &tmVb, &full[s], 0, h0 - R - L, bh, R);
        if (k >= 2) tc::mbar_wait(&empty[s], ((k - 2) >> 1) & 1);
        tc::tma_load_4d(sb, &tmQ, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);                         // rows (h0+i-c, c)
        tc::tma_load_4d(sb + 2 * Cf::QB + 2 * Cf::KBB, &tmKs, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);   // (h0+i-c', c')
        tc::tma_load_4d(sb + 2 * Cf::QB + 2 * Cf::KBB + Cf::SB, &tmVs, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nme > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, NB, 0, 0);
      constexpr uint32_t idQ = tc::idesc_bf16(128, kD, 0, 1);
      constexpr uint32_t idK = tc::idesc_bf16(128, kD, 1, 1);
      const int nks = (R * HZ + 15) / 16;                    // 16-key steps over the stair keys
      // HM: dense staircase products into [NB, NB + 16 nks) (over item ng - 2's dQ / dK columns:
      // S waits for that item's epilogue instead of the dQ / dK / dV MMAs)
      const uint32_t idSt = tc::idesc_bf16(128, 16 * nks, 0, 0);
      (void)idSt;
      int ns = 0, ndp = 0, ng = 0;
      while (ng < nme) {
        // dQ / dK / dV (ng) overwrite the accumulators of item ng - 2: they wait for its epilogue
        // (tfree); S / dP (ns) only use columns [0, NB) and run during that epilogue
        const uint32_t m = tc::mbar_test4(tc::smem_u32(&dsfull[ng & 1]), (ng >> 1) & 1,
                                          tc::smem_u32(&xfree[ndp & 1]), (ndp >> 1) & 1,
                                          tc::smem_u32(&full[ns & 1]), (ns >> 1) & 1,
                                          HM ? tc::smem_u32(&tfree[ns & 1]) : tc::smem_u32(&tfree[ng & 1]),
                                          HM ? ((ns + 2) >> 1) & 1 : ((ng + 2) >> 1) & 1);
        if (ng < ndp && (m & 1) && (HM || ng < 2 || (m & 8))) {   // dQ, dK_stair, dV_stair of item ng
          tc::tc_fence_after();
          const int b = ng & 1;
          const uint32_t sb = tc::smem_u32(stage0 + b * Cf::STAGE);
          const uint32_t q = sb, dO = sb + Cf::QB, kb = sb + 2 * Cf::QB, ks = kb + 2 * Cf::KBB;
          const uint32_t x = tbase + b * 256;
          const uint32_t ds = tc::smem_u32(xds), ps = tc::smem_u32(xps);
#pragma unroll
          for (int j = 0; j < NB / 16; ++j)
            tc::mma_bf16_ts(x + NB, x + 8 * j, tc::desc_mnmajor_sw128(kb + 2048 * j), idQ, j > 0);
          for (int j = 0; j < nks; ++j)
            tc::mma_bf16(x + NB, tc::desc_kmajor_sw128(ds + (j >> 2) * 16384 + (j & 3) * 32),
                         tc::desc_mnmajor_sw128(ks + 2048 * j), idQ, 1);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            tc::mma_bf16(x + NB + 64, tc::sdesc(ds + 2048 * j, 16384, 1024, 2), tc::desc_mnmajor_sw128(q + 2048 * j),
                         idK, j > 0);
            tc::mma_bf16(x + NB + 128, tc::sdesc(ps + 2048 * j, 16384, 1024, 2),
                         tc::desc_mnmajor_sw128(dO + 2048 * j), idK, j > 0);
          }
          tc::mma_commit(&done[b]);
          tc::mma_commit(xsfree);
          tc::mma_commit(&emptyA[b]);   // dO / Kb / Vb; Q / Ks / Vs are released by the epilogue's stores
          ++ng;
          continue;
        }
        if (ndp < ns && (m & 2)) {   // dP_band of item ndp (S consumed)
          tc::tc_fence_after();
          const int b = ndp & 1;
          const uint32_t sb = tc::smem_u32(stage0 + b * Cf::STAGE);
          const uint32_t dO = sb + Cf::QB, vb = sb + 2 * Cf::QB + Cf::KBB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(dO + 32 * j), tc::desc_kmajor_sw128(vb + 32 * j), idS,
                         j > 0);
          if constexpr (HM) {
            const uint32_t vs = vb + Cf::KBB + Cf::SB;
#pragma unroll
            for (int j = 0; j < kD / 16; ++j)
              tc::mma_bf16(tbase + b * 256 + NB, tc::desc_kmajor_sw128(dO + 32 * j), tc::desc_kmajor_sw128(vs + 32 * j),
                           idSt, j > 0);
          }
          tc::mma_commit(&dpfull[b]);
          ++ndp;
          continue;
        }
        if (ns < nme && ns < ng + 2 && (m & 4) && (!HM || ns < 2 || (m & 8))) {   // S_band of item ns
          tc::tc_fence_after();
          const int b = ns & 1;
          const uint32_t sb = tc::smem_u32(stage0 + b * Cf::STAGE);
          const uint32_t q = sb, kb = sb + 2 * Cf::QB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(kb + 32 * j), idS,
                         j > 0);
          if constexpr (HM) {
            const uint32_t ks = kb + 2 * Cf::KBB;
#pragma unroll
            for (int j = 0; j < kD / 16; ++j)
              tc::mma_bf16(tbase + b * 256 + NB, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(ks + 32 * j),
                           idSt, j > 0);
          }
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
    // output channel / horizon offset of row r (HM: r = i C + c; else r = c HZ + i)
    const int c = HM ? r % C : r / HZ, i = HM ? r / C : r - (r / HZ) * HZ;
    const bool in_item = HM ? i < HZ : c < C;
    // HM: the RM staircase columns of row r are [i RM, i RM + RM) of the stair block; a warp's 32
    // rows span at most KH horizons, read as one warp-uniform window from its first horizon i_lo
    constexpr int KH = 31 / (RM + 1) + 2;
    const int i_lo = HM ? (32 * q4) / C : 0;
    auto stair_cols = [&](uint32_t xcol, float* out) {   // out[c'] = column xcol + i RM + c'
      float v[KH * RM];
#pragma unroll
      for (int j = 0; j < KH * RM / 8; ++j) tc::tmem_ld8(xcol + i_lo * RM + 8 * j, v + 8 * j);
      tc::tmem_ld_wait();
      const int kq = i - i_lo;
#pragma unroll
      for (int cp = 0; cp < RM; ++cp) out[cp] = v[cp];
#pragma unroll
      for (int kk = 1; kk < KH; ++kk)
#pragma unroll
        for (int cp = 0; cp < RM; ++cp) out[cp] = kq == kk ? v[kk * RM + cp] : out[cp];
    };
    (void)stair_cols; (void)i_lo;
    const uint32_t xdsa = tc::smem_u32(xds), xpsa = tc::smem_u32(xps);
    // this row's LSE of item k (loaded one item ahead: the global load's latency is off the chain)
    auto lse_of = [&](int k) -> float {
      if (k >= nme || !in_item) return 0.f;
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / nit, t = item_j(g % nit, a.sub) * HZ + i - c;
      return (t >= 0 && t < T) ? a.LSE[((long long)c * a.BH + bh) * T + t] : 0.f;
    };
    float lse_next = lse_of(wg);
    uint8_t* scr = scr0 + wg * Cf::SCR;                       // [S | dP][128 rows][8] fp32
    const int wq = warp & 3;                                  // warp within the warpgroup
    for (int k = wg; k < nme; k += 2) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
      const int b = wg, use = k >> 1;
      const int h = h0 + i, t = h - c;
      const bool row_ok = in_item && t >= 0 && t < T;
      const long long crow = ((long long)c * a.BH + bh);
      const float lse2 = lse_next * kLog2e;
      lse_next = lse_of(k + 2);
      const uint8_t* sbp = stage0 + b * Cf::STAGE;
      const uint32_t sb = tc::smem_u32(sbp);
#define LTR(ev) do { if (a.trace && blockIdx.x == 0 && r == 0 && k < 64) a.trace[(ev) * 64 + k] = clock64(); } while (0)
      LTR(0);
      tc::mbar_wait(&full[b], use & 1);
      LTR(1);
      float sst[RM], dst[RM];
      if constexpr (HM) {
        // staircase S / dP come from TMEM with the band's (below)
      } else if constexpr (Cf::SMMA) {
        // ---- staircase on mma.sync: horizon ih's blocks S = Q_ih K_ih^T, then dP = dO_ih V_ih^T
        //      (rows c: Q rows c HZ + ih; cols c': stair rows c' HZ + ih; ceil(C/16) x RM/8 blocks of
        //      16 x 8), two horizons per warp iteration, scattered to the scratch rows r = c HZ + ih
        //      and read back per thread (S pass, then dP pass through the same scratch)
        const uint32_t ks = sb + 2 * Cf::QB + 2 * Cf::KBB, vs = ks + Cf::SB;
        const uint32_t za = tc::smem_u32(zrow), sca = tc::smem_u32(scr);
        const int gq = lane >> 2, t4 = lane & 3;
        const int nmb = (C + 15) / 16;
        // SFUSE: one pass computing both products (scratch halves); else S pass, then dP pass
        constexpr int NPASS = Cf::SFUSE ? 1 : 2, NPROD = Cf::SFUSE ? 2 : 1;
        constexpr uint32_t HALF = 128 * RM * 4;
#pragma unroll
        for (int pass = 0; pass < NPASS; ++pass) {
          for (int ih0 = wq; ih0 < HZ; ih0 += 8) {
            for (int mb = 0; mb < nmb; ++mb) {
#pragma unroll
              for (int nb = 0; nb < RM / 8; ++nb) {
                float acc[NPROD][2][4] = {};
                const int am = 16 * mb + (lane & 15), bn = 8 * nb + (lane & 7);
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) {
                  const int ih = ih0 + 4 * u2;
                  const bool hv = ih < HZ;
                  const int arow = (hv && am < C) ? am * HZ + ih : -1, brow = (hv && bn < R) ? bn * HZ + ih : -1;
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    const int ach = 2 * kk + (lane >> 4), bch = 2 * kk + ((lane >> 3) & 1);
                    const uint32_t ao = arow < 0 ? 0u : (uint32_t)(arow * 128 + ((ach ^ (arow & 7)) << 4));
                    const uint32_t bo = brow < 0 ? 0u : (uint32_t)(brow * 128 + ((bch ^ (brow & 7)) << 4));
#pragma unroll
                    for (int pr = 0; pr < NPROD; ++pr) {
                      const int pp = pass + pr;                  // 0: Q . K_stair, 1: dO . V_stair
                      uint32_t af[4], bf[2];
                      ldsm_x4(arow < 0 ? za : sb + pp * Cf::QB + ao, af);
                      ldsm_x2(brow < 0 ? za : (pp ? vs : ks) + bo, bf);
                      mma16816(acc[pr][u2], af, bf);
                    }
                  }
                }
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) {
                  const int ih = ih0 + 4 * u2;
                  if (ih >= HZ) break;
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const int cc = 16 * mb + gq + 8 * (e >> 1), cp = 8 * nb + 2 * t4 + (e & 1);
                    if (cc < C) {
#pragma unroll
                      for (int pr = 0; pr < NPROD; ++pr)
                        tc::st_shared_u32(sca + pr * HALF + (uint32_t)((cc * HZ + ih) * RM + cp) * 4,
                                          __float_as_uint(acc[pr][u2][e]));
                    }
                  }
                }
              }
            }
          }
          tc::named_bar(1 + wg, 128);
          const uint32_t o = sca + (uint32_t)r * RM * 4;
#pragma unroll
          for (int pr = 0; pr < NPROD; ++pr) {
            const int pp = pass + pr;
#pragma unroll
            for (int q = 0; q < RM / 4; ++q) {
              const uint4 s4 = tc::ld_shared_v4(o + pr * HALF + 16 * q);
              const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int cp = 4 * q + e;
                if (pp == 0) {
                  const int f = h - cp;
                  const bool ok = row_ok && cp < R && f >= 0 && f < T;
                  sst[cp] = ok ? tc::ex2(fmaf(__uint_as_float(sv[e]), a.scale_log2, -lse2)) : 0.f;
                } else {
                  dst[cp] = __uint_as_float(sv[e]);
                }
              }
            }
          }
          tc::named_bar(1 + wg, 128);   // the scratch is rewritten (dP pass / next item)
        }
      } else {
      // ---- staircase scores and dP on CUDA cores: key (h - c', c') = stair row c' HZ + i; two
      //      passes (q . k_stair, then dO . v_stair) so one 64-float row is live at a time
      {
        const uint32_t ks = sb + 2 * Cf::QB + 2 * Cf::KBB, vs = ks + Cf::SB;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          float2 q2[kD / 2];
          const uint32_t qrow = sb + pass * Cf::QB + r * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint4 x = tc::ld_shared_v4(qrow + ((ch ^ (r & 7)) << 4));
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              q2[4 * ch + e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
          }
#pragma unroll
          for (int cp = 0; cp < RM; ++cp) {
            float2 acc = make_float2(0.f, 0.f);
            if (cp < R) {
              const int m = cp * HZ + i;
              const uint32_t krow = (pass ? vs : ks) + m * 128;
#pragma unroll
              for (int ch = 0; ch < 8; ++ch) {
                const uint4 x = tc::ld_shared_v4(krow + ((ch ^ (m & 7)) << 4));
                const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  acc = __ffma2_rn(q2[4 * ch + e],
                                   make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u)), acc);
              }
            }
            if (pass == 0) {
              const int f = h - cp;
              const bool ok = row_ok && cp < R && f >= 0 && f < T;
              sst[cp] = ok ? tc::ex2(fmaf(acc.x + acc.y, a.scale_log2, -lse2)) : 0.f;   // P of the stair slot
            } else {
              dst[cp] = acc.x + acc.y;
            }
          }
        }
      }
      }
      LTR(2);
      // ---- band P from S
      tc::mbar_wait(&sfull[b], use & 1);
      LTR(3);
      __syncwarp();
      tc::tc_fence_after();
      float p[NB];
      const uint32_t x = tbase + lanes + b * 256;
      if constexpr (HM) {   // P of the staircase slots (h - c', c'), c' < R (= RM)
        stair_cols(x + NB, sst);
#pragma unroll
        for (int cp = 0; cp < RM; ++cp) {
          const int f = h - cp;
          const bool ok = row_ok && f >= 0 && f < T;
          sst[cp] = ok ? tc::ex2(fmaf(sst[cp], a.scale_log2, -lse2)) : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < NB / 8; ++j) tc::tmem_ld8(x + 8 * j, p + 8 * j);
      tc::tmem_ld_wait();
      {
        const int key0 = h0 - R - L;                       // frame of band column 0
        const int jlo = max(i, -key0), jhi = min(i + L, T - 1 - key0);
#pragma unroll
        for (int j = 0; j < NB; ++j)
          p[j] = (row_ok && j >= jlo && j <= jhi) ? tc::ex2(fmaf(p[j], a.scale_log2, -lse2)) : 0.f;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&xfree[b]);
      LTR(4);
      // ---- dP, delta, dS
      tc::mbar_wait(&dpfull[b], use & 1);
      LTR(5);
      __syncwarp();
      tc::tc_fence_after();
      if constexpr (HM) stair_cols(x + NB, dst);   // staircase dP
      // dP is read from TMEM twice (delta, then dS) instead of being held next to P
      float delta = 0.f;
#pragma unroll
      for (int j = 0; j < NB / 8; ++j) {
        float dp[8];
        tc::tmem_ld8(x + 8 * j, dp);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) delta = fmaf(p[8 * j + e], dp[e], delta);
      }
#pragma unroll
      for (int cp = 0; cp < RM; ++cp) delta = fmaf(sst[cp], dst[cp], delta);
#pragma unroll
      for (int j = 0; j < NB / 8; ++j) {
        float dp[8];
        tc::tmem_ld8(x + 8 * j, dp);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) p[8 * j + e] *= dp[e] - delta;   // dS_band
      }
      // dS_band -> X_b columns [0, NB/2) as the packed bf16 A operand of the dQ MMA
#pragma unroll
      for (int j = 0; j < NB / 8; ++j)
        tc::tmem_st4(x + 4 * j, pack_bf16(p[8 * j], p[8 * j + 1]), pack_bf16(p[8 * j + 2], p[8 * j + 3]),
                     pack_bf16(p[8 * j + 4], p[8 * j + 5]), pack_bf16(p[8 * j + 6], p[8 * j + 7]));
      // staircase dS / P -> DS / PS (row r, columns c' HZ + i); the previous item's MMAs must have
      // read them (one buffer shared by both warpgroups)
      if (k >= 1) tc::mbar_wait(xsfree, (k - 1) & 1);
      if (in_item) {
        if constexpr (HM) {   // the row's RM staircase entries: 16-byte chunks at column i RM
#pragma unroll
          for (int q8 = 0; q8 < RM / 8; ++q8) {
            float d8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) d8[e] = sst[8 * q8 + e] * (dst[8 * q8 + e] - delta);
            const int col = i * RM + 8 * q8;
            tc::st_shared_v4(xs_addr(xdsa, r, col), make_uint4(pack_bf16(d8[0], d8[1]), pack_bf16(d8[2], d8[3]),
                                                              pack_bf16(d8[4], d8[5]), pack_bf16(d8[6], d8[7])));
            const float* p8 = sst + 8 * q8;
            tc::st_shared_v4(xs_addr(xpsa, r, col), make_uint4(pack_bf16(p8[0], p8[1]), pack_bf16(p8[2], p8[3]),
                                                              pack_bf16(p8[4], p8[5]), pack_bf16(p8[6], p8[7])));
          }
        } else {
#pragma unroll
        for (int cp = 0; cp < RM; ++cp) {
          if (cp < R) {
            const float ds = sst[cp] * (dst[cp] - delta);
            tc::st_shared_u16(xs_addr(xdsa, r, cp * HZ + i), __bfloat16_as_ushort(__float2bfloat16_rn(ds)));
            tc::st_shared_u16(xs_addr(xpsa, r, cp * HZ + i), __bfloat16_as_ushort(__float2bfloat16_rn(sst[cp])));
          }
        }
        }
      }
      
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(&dsfull[b]);
      LTR(6);

      // workspace rows for the key-major band pass (padded rows [T, Tp) zero)
      if (row_ok) {
        // per-head rows, or one row per channel over the flattened BH*T axis (padding after the last head)
        const long long w0 = a.ws_flat ? (long long)c * a.Tp + (long long)bh * T : crow * a.Tp;
        const int wend = a.ws_flat ? a.Tp - (a.BH - 1) * T : a.Tp;   // padded end, relative to w0
        a.ws_del[w0 + t] = delta;
        a.ws_l2[w0 + t] = lse2;
        if (t == T - 1 && (!a.ws_flat || bh == a.BH - 1))
          for (int tt = T; tt < wend; ++tt) { a.ws_del[w0 + tt] = 0.f; a.ws_l2[w0 + tt] = 0.f; }
      }
      LTR(7);
      // ---- epilogue: dQ row (t, c); staircase key rows m = r: (u, c'), u = h0 + i' - c'
      tc::mbar_wait(&done[b], use & 1);
      LTR(8);
      __syncwarp();
      tc::tc_fence_after();
      // interior items (every row of the item's skewed boxes inside [0, T)): rows staged in the
      // stage's now-dead Q / Ks / Vs tiles (the layout their TMA loads had) and written by three
      // TMA stores; edge items: direct row stores (a skewed box there would cross into the
      // neighbouring channel planes).  The stage is released once the stores have read it.
      const bool tma_out = h0 >= R && h0 + HZ <= T;
      // staircase key of accumulator row r: (u, cq), u = h0 + iq - cq (HM: r = iq RM + cq)
      const int cq = HM ? r % RM : r / HZ, iq = HM ? r / RM : r - (r / HZ) * HZ, u = h0 + iq - cq;
      const bool key_ok = (HM ? iq < HZ : cq < R) && u >= 0 && u < T;
      const long long krow = ((long long)cq * a.BH + bh) * T + u;
      uint8_t* qst = const_cast<uint8_t*>(sbp);
      uint8_t* kst = qst + 2 * Cf::QB + 2 * Cf::KBB;
      uint8_t* vst = kst + Cf::SB;
      float v[kD];
      tmem_ld64_l(x + NB, v);
      if (tma_out) tmem_row64_to_smem_sw128_regs(v, a.scale, qst, r);
      else if (row_ok) store_row64(a.dQ + (crow * T + t) * kD, v, a.scale);
      tmem_ld64_l(x + NB + 64, v);
      if (tma_out) { if (r < R * HZ) tmem_row64_to_smem_sw128_regs(v, a.scale, kst, r); }
      else if (key_ok) store_row64(a.dK + krow * kD, v, a.scale);
      tmem_ld64_l(x + NB + 128, v);
      if (tma_out) { if (r < R * HZ) tmem_row64_to_smem_sw128_regs(v, 1.f, vst, r); }
      else if (key_ok) store_row64(a.dV + krow * kD, v, 1.f);
      tc::tc_fence_before();
      tc::mbar_arrive(&tfree[b]);
      if (tma_out) tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (r == 0) {
        if (tma_out) {
          tc::tma_store_4d(&tmdQ, qst, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
          tc::tma_store_4d(&tmdK, kst, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
          tc::tma_store_4d(&tmdV, vst, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
          tc::bulk_commit();
          tc::bulk_wait_read0();
        }
        tc::mbar_arrive(&empty[b]);
      }
      
      LTR(9);
#undef LTR
    }
  }
  tc::bulk_wait0();
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// LLSA forward, item form (dense inputs, R <= 8): the same item as the fused backward below —
// HZ horizons x all C channels, row r = c HZ + i <-> output (t, c), t = h0 + i - c — so the
// staircase of a horizon is one 16 x 8 mma.sync block and every row's stair probabilities land
// in a per-warpgroup smem tile read by the PV MMA:
//   MMA  S   = Q Kb^T -> X_b[0, NB)            WG  stair scores (mma.sync per horizon, scratch),
//                                                   band strip from TMEM, joint softmax; P_band ->
//                                                   X_b (packed bf16), P_stair -> PS_wg (smem)
//   MMA  O   = [P_band | PS] [Vb ; Vs] -> X_b[NB, NB + 64)
//                                              WG  O / l, LSE; interior items: O rows staged in
//                                                  the dead Q tile, one skewed TMA store
// ------------------------------------------------------------------------------------------
struct LlsaFwdArgs {
  int T, L, R, C, BH, HZ;
  ItemSub sub;
  float scale, scale_log2;
  float* LSE;                    // [C][BH][T]
  bf16* O;                       // [C][BH][T][64]
};

template <int NB, int RM, bool HM = false> struct LFCfg {
  static constexpr int QB = 128 * 128;
  static constexpr int KBB = NB * 128;
  static constexpr int SB = 112 * 128;
  static constexpr int STAGE = QB + 2 * KBB + 2 * SB;      // Q | Kb | Vb | Ks | Vs
  static constexpr int XB = 2 * 128 * 128;                 // PS (shared by the warpgroups, see below)
  static constexpr int SCR = HM ? 0 : 128 * RM * 4;       // stair scores per warpgroup (mma.sync path)
  // three stages where they fit (the warpgroups otherwise wait on the TMA loads)
  static constexpr int NSTG = 1024 + 3 * STAGE + XB + 2 * SCR + 128 + 256 <= 232448 ? 3 : 2;
  static constexpr int SMEM = 1024 + NSTG * STAGE + XB + 2 * SCR + 128 + 256;
  static_assert(NB + 64 <= 256 && SMEM <= 232448, "TMEM / shared memory");
};

template <int NB, int RM, bool HM>
__global__ void __launch_bounds__(320, 1)
    llsa_fwd_item_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKb,
                     const __grid_constant__ CUtensorMap tmVb, const __grid_constant__ CUtensorMap tmKs,
                     const __grid_constant__ CUtensorMap tmVs, const __grid_constant__ CUtensorMap tmO,
                     LlsaFwdArgs a) {
  // HM (R == RM): horizon-major item rows i C + c and staircase keys i' RM + c' (reordered skewed
  // boxes), the staircase scores as one dense tcgen05 product Q Ks^T into TMEM [NB + 64, NB + 64 +
  // HZ RM) (each row's RM entries are its horizon's contiguous columns), as the fused backward
  using Cf = LFCfg<NB, RM, HM>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage0 = smem;
  constexpr int NSTG = Cf::NSTG;
  uint8_t* xps0 = smem + NSTG * Cf::STAGE;   // P_stair tile, one for both warpgroups
  uint8_t* scr0 = xps0 + Cf::XB;
  uint8_t* zrow = scr0 + 2 * Cf::SCR;
  uint64_t* bars = reinterpret_cast<uint64_t*>(zrow + 128);
  uint64_t* full = bars;          // [NSTG]
  uint64_t* empty = full + NSTG;  // [NSTG] (released by the epilogue leader)
  uint64_t* sfull = empty + NSTG; // [2]
  uint64_t* pfull = sfull + 2;    // [2] (128)
  uint64_t* ofull = pfull + 2;    // [2]
  uint64_t* tfree = ofull + 2;    // [2] (128)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = a.T, L = a.L, R = a.R, C = a.C, HZ = a.HZ;
  const int nit = a.sub.nit_l;                               // items of this launch per (b, h)
  const int nitems = nit * a.BH;
  const int nme = blockIdx.x < nitems ? (nitems - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int qbytes = C * HZ * 128, sbytes = R * HZ * 128;

  for (int o = tid * 16; o < NSTG * Cf::STAGE + Cf::XB + 2 * Cf::SCR + 128; o += 320 * 16)
    *reinterpret_cast<uint4*>(smem + o) = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {
    tc::tma_prefetch_desc(&tmQ); tc::tma_prefetch_desc(&tmKb); tc::tma_prefetch_desc(&tmVb);
    tc::tma_prefetch_desc(&tmKs); tc::tma_prefetch_desc(&tmVs); tc::tma_prefetch_desc(&tmO);
    for (int i = 0; i < NSTG; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sfull[i], 1); tc::mbar_init(&pfull[i], 128);
      tc::mbar_init(&ofull[i], 1); tc::mbar_init(&tfree[i], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  // L2 prefetch of the first items' boxes while the previous kernel drains (PDL; coherent L2)
  auto prefetch_l2 = [&](int k) {
    if (k >= nme) return;
    const int g = blockIdx.x + k * gridDim.x;
    const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
    tc::tma_prefetch_4d(&tmQ, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
    tc::tma_prefetch_4d(&tmKb, 0, h0 - R - L, bh, R);
    tc::tma_prefetch_4d(&tmVb, 0, h0 - R - L, bh, R);
    tc::tma_prefetch_4d(&tmKs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
    tc::tma_prefetch_4d(&tmVs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
  };
  if (tid == 0)
    for (int k = 0; k < 2; ++k) prefetch_l2(k);
  tc::pdl_wait();
  tc::pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      auto prefetch = [&](int k) {
        if (k >= nme) return;
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
        tc::tma_prefetch_4d(&tmQ, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_prefetch_4d(&tmKb, 0, h0 - R - L, bh, R);
        tc::tma_prefetch_4d(&tmVb, 0, h0 - R - L, bh, R);
        tc::tma_prefetch_4d(&tmKs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_prefetch_4d(&tmVs, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
      };
      for (int k = 0; k < nme; ++k) {
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
        const int s = k % NSTG;
        prefetch(k + NSTG);
        if (k >= NSTG) tc::mbar_wait(&empty[s], ((k - NSTG) / NSTG) & 1);
        uint8_t* sb = stage0 + s * Cf::STAGE;
        tc::mbar_expect_tx(&full[s], qbytes + 2 * Cf::KBB + 2 * sbytes);
        tc::tma_load_4d(sb, &tmQ, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_load_4d(sb + Cf::QB, &tmKb, &full[s], 0, h0 - R - L, bh, R);
        tc::tma_load_4d(sb + Cf::QB + Cf::KBB, &tmVb, &full[s], 0, h0 - R - L, bh, R);
        tc::tma_load_4d(sb + Cf::QB + 2 * Cf::KBB, &tmKs, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);
        tc::tma_load_4d(sb + Cf::QB + 2 * Cf::KBB + Cf::SB, &tmVs, &full[s], 0, HM ? 0 : h0, HM ? h0 : 0, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nme > 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, NB, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, kD, 0, 1);
      const int nks = (R * HZ + 15) / 16;
      const uint32_t idSt = tc::idesc_bf16(128, 16 * nks, 0, 0);
      (void)idSt;
      int ns = 0, no = 0;
      while (no < nme) {
        // O(no) overwrites the O columns of item no - 2: it waits for that item's epilogue (tfree);
        // S(ns) only needs its stage and PV(ns - 2) issued ahead of it (in-order execution), so it
        // runs while the warpgroup is still in the epilogue of item ns - 2
        const uint32_t m = tc::mbar_test4(tc::smem_u32(&pfull[no & 1]), (no >> 1) & 1,
                                          tc::smem_u32(&full[ns % NSTG]), (ns / NSTG) & 1,
                                          tc::smem_u32(&tfree[no & 1]), ((no + 2) >> 1) & 1,
                                          tc::smem_u32(&pfull[no & 1]), (no >> 1) & 1);
        if (no < ns && (m & 1) && (no < 2 || (m & 4))) {   // O of item no
          tc::tc_fence_after();
          const int b = no & 1;
          const uint32_t sb = tc::smem_u32(stage0 + (no % NSTG) * Cf::STAGE);
          const uint32_t vb = sb + Cf::QB + Cf::KBB, vs = sb + Cf::QB + 2 * Cf::KBB + Cf::SB;
          const uint32_t x = tbase + b * 256;
          const uint32_t ps = tc::smem_u32(xps0);
#pragma unroll
          for (int j = 0; j < NB / 16; ++j)
            tc::mma_bf16_ts(x + NB, x + 8 * j, tc::desc_mnmajor_sw128(vb + 2048 * j), idO, j > 0);
          for (int j = 0; j < nks; ++j)
            tc::mma_bf16(x + NB, tc::desc_kmajor_sw128(ps + (j >> 2) * 16384 + (j & 3) * 32),
                         tc::desc_mnmajor_sw128(vs + 2048 * j), idO, 1);
          tc::mma_commit(&ofull[b]);
          ++no;
          continue;
        }
        if (ns < nme && ns < no + 2 && (m & 2)) {   // S_band of item ns
          tc::tc_fence_after();
          const int b = ns & 1;
          const uint32_t sb = tc::smem_u32(stage0 + (ns % NSTG) * Cf::STAGE);
          const uint32_t q = sb, kb = sb + Cf::QB;
#pragma unroll
          for (int j = 0; j < kD / 16; ++j)
            tc::mma_bf16(tbase + b * 256, tc::desc_kmajor_sw128(q + 32 * j), tc::desc_kmajor_sw128(kb + 32 * j), idS,
                         j > 0);
          if constexpr (HM) {   // staircase scores, dense: columns [NB + 64, NB + 64 + 16 nks) (beside O)
            const uint32_t ks = kb + 2 * Cf::KBB;
#pragma unroll
            for (int j = 0; j < kD / 16; ++j)
              tc::mma_bf16(tbase + b * 256 + NB + 64, tc::desc_kmajor_sw128(q + 32 * j),
                           tc::desc_kmajor_sw128(ks + 32 * j), idSt, j > 0);
          }
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
    const int c = HM ? r % C : r / HZ, i = HM ? r / C : r - (r / HZ) * HZ;
    const bool in_item = HM ? i < HZ : c < C;
    constexpr int KH = 31 / (RM + 1) + 2;                   // horizons a warp's 32 rows span (HM)
    const int i_lo = HM ? (32 * q4) / C : 0;
    const int wq = warp & 3;
    const uint32_t psa = tc::smem_u32(xps0), sca = tc::smem_u32(scr0 + wg * Cf::SCR);
    const uint32_t za = tc::smem_u32(zrow);
    for (int k = wg; k < nme; k += 2) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / nit, h0 = item_j(g % nit, a.sub) * HZ;
      const int b = wg, use = k >> 1;
      const int h = h0 + i, t = h - c;
      const bool row_ok = in_item && t >= 0 && t < T;
      const int st = k % NSTG;
      uint8_t* sbp = stage0 + st * Cf::STAGE;
      const uint32_t sb = tc::smem_u32(sbp);
      tc::mbar_wait(&full[st], (k / NSTG) & 1);
      // ---- staircase scores S[c][c'] = q_(h-c, c) . k_(h-c', c') on mma.sync: per horizon ceil(C/16)
      //      x RM/8 blocks of 16 x 8 (two horizons per iteration), through the scratch [128][RM]
      //      (HM: from TMEM below)
      if constexpr (!HM) {
        const uint32_t qt = sb, ks = sb + Cf::QB + 2 * Cf::KBB;
        const int gq = lane >> 2, t4 = lane & 3;
        const int nmb = (C + 15) / 16;
        for (int ih0 = wq; ih0 < HZ; ih0 += 8) {
          for (int mb = 0; mb < nmb; ++mb) {
#pragma unroll
            for (int nb = 0; nb < RM / 8; ++nb) {
              float sacc[2][4] = {};
              const int am = 16 * mb + (lane & 15), bn = 8 * nb + (lane & 7);
#pragma unroll
              for (int u2 = 0; u2 < 2; ++u2) {
                const int ih = ih0 + 4 * u2;
                const bool hv = ih < HZ;
                const int arow = (hv && am < C) ? am * HZ + ih : -1, brow = (hv && bn < R) ? bn * HZ + ih : -1;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const int ach = 2 * kk + (lane >> 4), bch = 2 * kk + ((lane >> 3) & 1);
                  const uint32_t ao = arow < 0 ? 0u : (uint32_t)(arow * 128 + ((ach ^ (arow & 7)) << 4));
                  const uint32_t bo = brow < 0 ? 0u : (uint32_t)(brow * 128 + ((bch ^ (brow & 7)) << 4));
                  uint32_t aq[4], bk[2];
                  ldsm_x4(arow < 0 ? za : qt + ao, aq);
                  ldsm_x2(brow < 0 ? za : ks + bo, bk);
                  mma16816(sacc[u2], aq, bk);
                }
              }
#pragma unroll
              for (int u2 = 0; u2 < 2; ++u2) {
                const int ih = ih0 + 4 * u2;
                if (ih >= HZ) break;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int cc = 16 * mb + gq + 8 * (e >> 1), cp = 8 * nb + 2 * t4 + (e & 1);
                  if (cc < C)
                    tc::st_shared_u32(sca + (uint32_t)((cc * HZ + ih) * RM + cp) * 4, __float_as_uint(sacc[u2][e]));
                }
              }
            }
          }
        }
      }
      float sst[RM];
      if constexpr (!HM) {
        tc::named_bar(1 + wg, 128);
        const uint32_t o = sca + (uint32_t)r * RM * 4;
#pragma unroll
        for (int q = 0; q < RM / 4; ++q) {
          const uint4 s4 = tc::ld_shared_v4(o + 16 * q);
          const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int cp = 4 * q + e, f = h - cp;
            sst[cp] = (row_ok && cp < R && f >= 0 && f < T) ? __uint_as_float(sv[e]) : neg_inf();
          }
        }
        tc::named_bar(1 + wg, 128);   // scratch rewritten by this warpgroup's next item
      }
      // ---- band strip + joint softmax
      tc::mbar_wait(&sfull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      float s[NB];
      const uint32_t x = tbase + lanes + b * 256;
      if constexpr (HM) {   // the row's staircase columns: one warp-uniform window of KH horizons + selects
        float v[KH * RM];
#pragma unroll
        for (int j = 0; j < KH * RM / 8; ++j) tc::tmem_ld8(x + NB + 64 + i_lo * RM + 8 * j, v + 8 * j);
        tc::tmem_ld_wait();
        const int kq = i - i_lo;
#pragma unroll
        for (int cp = 0; cp < RM; ++cp) sst[cp] = v[cp];
#pragma unroll
        for (int kk = 1; kk < KH; ++kk)
#pragma unroll
          for (int cp = 0; cp < RM; ++cp) sst[cp] = kq == kk ? v[kk * RM + cp] : sst[cp];
#pragma unroll
        for (int cp = 0; cp < RM; ++cp) {
          const int f = h - cp;
          sst[cp] = (row_ok && f >= 0 && f < T) ? sst[cp] : neg_inf();
        }
      }
#pragma unroll
      for (int j = 0; j < NB / 8; ++j) tc::tmem_ld8(x + 8 * j, s + 8 * j);
      tc::tmem_ld_wait();
      const int key0 = h0 - R - L;
      const int jlo = max(i, -key0), jhi = min(i + L, T - 1 - key0);
      float mx = neg_inf();
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        s[j] = (row_ok && j >= jlo && j <= jhi) ? s[j] : neg_inf();
        mx = fmaxf(mx, s[j]);
      }
#pragma unroll
      for (int cp = 0; cp < RM; ++cp) mx = fmaxf(mx, sst[cp]);
      const float mref = mx == neg_inf() ? 0.f : mx;
      const float mb = mref * a.scale_log2;
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        s[j] = tc::ex2(fmaf(s[j], a.scale_log2, -mb));
        l += s[j];
      }
#pragma unroll
      for (int cp = 0; cp < RM; ++cp) {
        sst[cp] = tc::ex2(fmaf(sst[cp], a.scale_log2, -mb));
        l += sst[cp];
      }
#pragma unroll
      for (int j = 0; j < NB / 8; ++j)
        tc::tmem_st4(x + 4 * j, pack_bf16(s[8 * j], s[8 * j + 1]), pack_bf16(s[8 * j + 2], s[8 * j + 3]),
                     pack_bf16(s[8 * j + 4], s[8 * j + 5]), pack_bf16(s[8 * j + 6], s[8 * j + 7]));
      // P_stair -> PS, shared by the warpgroups: item k - 1's PV MMA (the other warpgroup's) must
      // have read it (every item writes the same positions; the rest stays zero)
      if (k > 0) tc::mbar_wait(&ofull[(k - 1) & 1], ((k - 1) >> 1) & 1);
      if (in_item) {
        if constexpr (HM) {
#pragma unroll
          for (int q8 = 0; q8 < RM / 8; ++q8) {
            const float* p8 = sst + 8 * q8;
            tc::st_shared_v4(xs_addr(psa, r, i * RM + 8 * q8), make_uint4(pack_bf16(p8[0], p8[1]), pack_bf16(p8[2], p8[3]),
                                                                       pack_bf16(p8[4], p8[5]), pack_bf16(p8[6], p8[7])));
          }
        } else {
#pragma unroll
        for (int cp = 0; cp < RM; ++cp)
          if (cp < R) tc::st_shared_u16(xs_addr(psa, r, cp * HZ + i), __bfloat16_as_ushort(__float2bfloat16_rn(sst[cp])));
        }
      }
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(&pfull[b]);
      // ---- epilogue
      tc::mbar_wait(&ofull[b], use & 1);
      __syncwarp();
      tc::tc_fence_after();
      const bool tma_out = h0 >= R && h0 + HZ <= T;
      float v[kD];
      tmem_ld64_l(x + NB, v);
      const float inv = 1.f / l;
      const long long crow = (long long)c * a.BH + bh;
      if (tma_out) tmem_row64_to_smem_sw128_regs(v, inv, sbp, r);
      else if (row_ok) store_row64(a.O + (crow * T + t) * kD, v, inv);
      if (row_ok) a.LSE[crow * T + t] = mref * a.scale + __log2f(l) * kLn2;
      tc::tc_fence_before();
      tc::mbar_arrive(&tfree[b]);
      if (tma_out) tc::fence_proxy_async_smem();
      tc::named_bar(1 + wg, 128);
      if (r == 0) {
        if (tma_out) {
          tc::tma_store_4d(&tmO, sbp, 0, HM ? 0 : h0, HM ? h0 : 0, bh);
          tc::bulk_commit();
          tc::bulk_wait_read0();
        }
        tc::mbar_arrive(&empty[st]);
      }
    }
  }
  tc::bulk_wait0();
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// host
// ------------------------------------------------------------------------------------------
// [C][BH][T][64] bf16 as a 4-D tensor (64, T, BH, C); box (64, rows, 1, 1); 128B swizzle.
bool map4(CUtensorMap* m, const void* base, int T, int BH, int C, int rows) {
  cuuint64_t dims[4] = {64, (cuuint64_t)T, (cuuint64_t)BH, (cuuint64_t)C};
  cuuint64_t strides[3] = {128, (cuuint64_t)T * 128, (cuuint64_t)BH * T * 128};
  cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
  CUresult r = tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (r != CUDA_SUCCESS) {
    g_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
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

// [C][BH][T][64] bf16 viewed so that box row i of channel c is frame y + i - c: dims
// (64, T + R, C, BH) with the channel stride skewed by one frame, (BH T - 1) x 128 B.  One box
// {64, rows, nch, 1} at (0, y, c0, bh) then stages the LLSA staircase diagonal (or an item's
// channel rows) in a single TMA copy.  Coordinates past the frame bounds of the diagonal read
// neighbouring planes (finite data); the kernel masks those slots (P = 0).
bool map_skew(CUtensorMap* m, const void* base, int T, int BH, int C, int R, int rows, int nch) {
  if ((long long)BH * T - 1 < (long long)T + R) return false;
  cuuint64_t dims[4] = {64, (cuuint64_t)(T + R), (cuuint64_t)C, (cuuint64_t)BH};
  cuuint64_t strides[3] = {128, ((cuuint64_t)BH * T - 1) * 128, (cuuint64_t)T * 128};
  cuuint32_t box[4] = {64, (cuuint32_t)rows, (cuuint32_t)nch, 1};
  return tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) == CUDA_SUCCESS;
}

// the skewed map with the channel as the faster box dimension: box (64, nch, rows) lands rows
// i nch + c (horizon-major) instead of c rows + i; element (c, h) is frame h - c of channel c
bool map_hm(CUtensorMap* m, const void* base, int T, int BH, int C, int R, int rows, int nch) {
  if ((long long)BH * T - 1 < (long long)T + R) return false;
  cuuint64_t dims[4] = {64, (cuuint64_t)C, (cuuint64_t)(T + R), (cuuint64_t)BH};
  cuuint64_t strides[3] = {((cuuint64_t)BH * T - 1) * 128, 128, (cuuint64_t)T * 128};
  cuuint32_t box[4] = {64, (cuuint32_t)nch, (cuuint32_t)rows, 1};
  return tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) == CUDA_SUCCESS;
}

template <int NB>
sattn_status launch(const AttnArgs& a, cudaStream_t st) {
  using Cf = LCfg<NB>;
  const int C = a.R + 1;
  const int Cin = a.in_cs == 0 ? 1 : C;
  CUtensorMap mq, mkb, mvb, mks, mvs, mo;
  if (!map4(&mq, a.Q, a.T, a.BH, Cin, kHT) || !map4(&mkb, a.K, a.T, a.BH, Cin, NB) ||
      !map4(&mvb, a.V, a.T, a.BH, Cin, NB) || !map4(&mks, a.K, a.T, a.BH, Cin, kHT) ||
      !map4(&mvs, a.V, a.T, a.BH, Cin, kHT) || !map4(&mo, a.Out, a.T, a.BH, C, kHT))
    return SATTN_ECUDA;
  // skewed single-box staging of the staircase and of each item's Q rows (dense inputs only:
  // a broadcast plane would need a negative channel stride); falls back to per-channel boxes
  bool skew = a.in_cs != 0;
  if (skew) {
    CUtensorMap sq, sk, sv;
    skew = map_skew(&sq, a.Q, a.T, a.BH, C, a.R, kHT, 4) && map_skew(&sk, a.K, a.T, a.BH, C, a.R, kHT, a.R) &&
           map_skew(&sv, a.V, a.T, a.BH, C, a.R, kHT, a.R);
    if (skew) { mq = sq; mks = sk; mvs = sv; }
  }
  LlsaArgs la{};
  la.skew = skew ? 1 : 0;
  la.T = a.T; la.L = a.L; la.R = a.R; la.C = C; la.BH = a.BH;
  la.bcast = a.in_cs == 0;
  la.scale = a.scale; la.scale_log2 = a.scale_log2;
  la.LSE = a.LSEout;
  la.O = reinterpret_cast<bf16*>(a.Out);
  const int nht = (a.T + a.R + kHT - 1) / kHT;
  const int ntiles = nht * a.BH;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  set_smem(llsa_fwd_tc<NB>, Cf::SMEM);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, llsa_fwd_tc<NB>, mq, mkb, mvb, mks, mvs, mo, la);
  return SATTN_OK;
}

// horizons per fused-backward item: all C channels of HZ horizons in <= 128 rows, and the band
// window of the item (HZ + L keys) in NB <= 64 TMEM columns
int fused_hz(int L, int R) {
  const int C = R + 1;
  int hz = 128 / C;
  if (hz > 64 - L) hz = 64 - L;
  if (R * hz > 112) hz = 112 / R;   // the stair tiles hold R HZ <= 112 rows
  return hz;
}

template <int NB, int RM, bool HM = false>
sattn_status bwd_fused_launch(const AttnArgs& a, int HZ, float* ws_del, float* ws_l2, int ws_flat, cudaStream_t st,
                               const ItemSub* sub) {
  using Cf = LBCfg<NB, RM, HM>;
  const int R = a.R, C = R + 1;
  auto mskew = HM ? map_hm : map_skew;
  CUtensorMap mq, mdo, mkb, mvb, mks, mvs, mdq, mdk, mdv;
  if (!mskew(&mq, a.Q, a.T, a.BH, C, R, HZ, C) || !mskew(&mdo, a.dO, a.T, a.BH, C, R, HZ, C) ||
      !map4(&mkb, a.K, a.T, a.BH, C, NB) || !map4(&mvb, a.V, a.T, a.BH, C, NB) ||
      !mskew(&mks, a.K, a.T, a.BH, C, R, HZ, R) || !mskew(&mvs, a.V, a.T, a.BH, C, R, HZ, R) ||
      !mskew(&mdq, a.dQ, a.T, a.BH, C, R, HZ, C) || !mskew(&mdk, a.dK, a.T, a.BH, C, R, HZ, R) ||
      !mskew(&mdv, a.dV, a.T, a.BH, C, R, HZ, R)) {
    g_err = "tensor maps of the fused LLSA backward";
    return SATTN_ECUDA;
  }
  LlsaBwdArgs la{};
  la.T = a.T; la.L = a.L; la.R = R; la.C = C; la.BH = a.BH; la.HZ = HZ; la.Tp = (a.T + 3) & ~3;
  la.scale = a.scale; la.scale_log2 = a.scale_log2;
  la.LSE = a.LSE;
  la.dQ = reinterpret_cast<bf16*>(a.dQ); la.dK = reinterpret_cast<bf16*>(a.dK); la.dV = reinterpret_cast<bf16*>(a.dV);
  la.ws_del = ws_del; la.ws_l2 = ws_l2;
  if (ws_flat) {   // the kv pass runs packed tiles over the flattened BH*T axis (tc_sa.cu)
    la.ws_flat = 1;
    la.Tp = (int)((((long long)a.BH * a.T) + 3) & ~3LL);
  }
  la.trace = g_llsa_trace;
  la.sub = sub ? *sub : all_items(a, HZ);
  const int items = la.sub.nit_l * a.BH;
  if (items == 0) return SATTN_OK;
  const int grid = items < num_sms() ? items : num_sms();
  set_smem(llsa_bwd_fused_tc<NB, RM, HM>, Cf::SMEM);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, llsa_bwd_fused_tc<NB, RM, HM>, mq, mdo, mkb, mvb, mks, mvs, mdq, mdk,
                                           mdv, la);
  if (e != cudaSuccess) {
    g_err = std::string("fused LLSA backward launch: ") + cudaGetErrorString(e);
    return SATTN_ECUDA;
  }
  return SATTN_OK;
}

}  // namespace

template <int NB, int RM, bool HM = false>
sattn_status fwd_item_launch(const AttnArgs& a, int HZ, cudaStream_t st, const ItemSub* sub = nullptr) {
  using Cf = LFCfg<NB, RM, HM>;
  const int R = a.R, C = R + 1;
  auto mskew = HM ? map_hm : map_skew;
  CUtensorMap mq, mkb, mvb, mks, mvs, mo;
  if (!mskew(&mq, a.Q, a.T, a.BH, C, R, HZ, C) || !map4(&mkb, a.K, a.T, a.BH, C, NB) ||
      !map4(&mvb, a.V, a.T, a.BH, C, NB) || !mskew(&mks, a.K, a.T, a.BH, C, R, HZ, R) ||
      !mskew(&mvs, a.V, a.T, a.BH, C, R, HZ, R) || !mskew(&mo, a.Out, a.T, a.BH, C, R, HZ, C)) {
    g_err = "tensor maps of the item-form LLSA forward";
    return SATTN_ECUDA;
  }
  LlsaFwdArgs la{};
  la.T = a.T; la.L = a.L; la.R = R; la.C = C; la.BH = a.BH; la.HZ = HZ;
  la.scale = a.scale; la.scale_log2 = a.scale_log2;
  la.LSE = a.LSEout;
  la.O = reinterpret_cast<bf16*>(a.Out);
  la.sub = sub ? *sub : all_items(a, HZ);
  const int items = la.sub.nit_l * a.BH;
  if (items == 0) return SATTN_OK;
  const int grid = items < num_sms() ? items : num_sms();
  set_smem(llsa_fwd_item_tc<NB, RM, HM>, Cf::SMEM);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, llsa_fwd_item_tc<NB, RM, HM>, mq, mkb, mvb, mks, mvs, mo, la);
  if (e != cudaSuccess) {
    g_err = std::string("item-form LLSA forward launch: ") + cudaGetErrorString(e);
    return SATTN_ECUDA;
  }
  return SATTN_OK;
}

// item form (dense inputs): R <= 16, the item's band window HZ + L in NB <= 64 columns
bool fwd_item_ok(const AttnArgs& a) {
  if (a.in_cs == 0 || a.R < 1 || a.R > 16) return false;
  const int hz = fused_hz(a.L, a.R);
  return hz >= 4 && (long long)a.BH * a.T - 1 >= (long long)a.T + a.R && (hz + a.L + 15) / 16 * 16 <= 64;
}

bool tc_llsa_supported(int dtype, int D, int L, int R) {
  // one warp per channel of a 4-channel item needs >= 2 items per tile (C >= 5); the P row
  // (NB + 32 R packed / 2 <= 192 columns) and the 8 staged stair tiles need R <= 8; the band
  // MMA's N = 16-rounded 32 + L is instantiated for 48 and 64 (1 <= L <= 32)
  return dtype == SATTN_BF16 && D == 64 && R >= 4 && R <= kRmax && L >= 1 && L + 32 <= 64;
}

// item-form forward: horizon-major items with the staircase on tcgen05 when R fills the RM
// staircase columns (R = 8, 16), else the mma.sync staircase
sattn_status fwd_item_dispatch(const AttnArgs& a, int hz, cudaStream_t st, const ItemSub* su) {
  const bool r16 = a.R > 8;
  const int nb = (hz + a.L + 15) / 16 * 16;
  if ((a.R == 8 || a.R == 16) && (hz * a.R) % 16 == 0 && (nb == 48 || nb == 64)) {
    if (nb == 48) return r16 ? fwd_item_launch<48, 16, true>(a, hz, st, su) : fwd_item_launch<48, 8, true>(a, hz, st, su);
    return r16 ? fwd_item_launch<64, 16, true>(a, hz, st, su) : fwd_item_launch<64, 8, true>(a, hz, st, su);
  }
  switch (nb) {
    case 16:
    case 32: return r16 ? fwd_item_launch<32, 16>(a, hz, st, su) : fwd_item_launch<32, 8>(a, hz, st, su);
    case 48: return r16 ? fwd_item_launch<48, 16>(a, hz, st, su) : fwd_item_launch<48, 8>(a, hz, st, su);
    case 64: return r16 ? fwd_item_launch<64, 16>(a, hz, st, su) : fwd_item_launch<64, 8>(a, hz, st, su);
  }
  g_err = "band too wide for the item-form LLSA forward";
  return SATTN_EUNSUPPORTED;
}

// item-form forward over an item subset (sub4 = it0, nit_l, it_split, it_jump per (b, h)); 0 when
// the item form does not apply
int tc_llsa_item_hz(const AttnArgs& a) {
  return fwd_item_ok(a) && tc_llsa_bwd_fused_supported(SATTN_BF16, 64, a.L, a.R, a.BH, a.T, true) ? fused_hz(a.L, a.R)
                                                                                                  : 0;
}

sattn_status tc_llsa_forward_items(const AttnArgs& a, const int* sub4, cudaStream_t st) {
  const int hz = fused_hz(a.L, a.R);
  if (!fwd_item_ok(a)) {
    g_err = "the item-form LLSA forward does not apply";
    return SATTN_EUNSUPPORTED;
  }
  const ItemSub su{sub4[0], sub4[1], sub4[2], sub4[3]};
  return fwd_item_dispatch(a, hz, st, &su);
}

sattn_status tc_llsa_forward(const AttnArgs& a, cudaStream_t st) {
  if (fwd_item_ok(a)) return fwd_item_dispatch(a, fused_hz(a.L, a.R), st, nullptr);
  const int nb = (32 + a.L + 15) / 16 * 16;
  switch (nb) {
    case 48: return launch<48>(a, st);
    case 64: return launch<64>(a, st);
  }
  g_err = "band too wide for the LLSA tensor-core kernel";
  return SATTN_EUNSUPPORTED;
}

// the item form (dense inputs, 1 <= R <= 8) or the 4-channel-item kernel (4 <= R <= 8, L <= 32)
bool tc_llsa_fwd_any_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense) {
  if (tc_llsa_supported(dtype, D, L, R)) return true;
  if (dtype != SATTN_BF16 || D != 64 || !dense || R < 1 || R > 16 || L < 0) return false;
  const int hz = fused_hz(L, R);
  return hz >= 4 && BH * T - 1 >= T + R && (hz + L + 15) / 16 * 16 <= 64;
}

// fused horizon-major LLSA backward (dense inputs): dQ, staircase dK / dV, delta and LSE log2e
// rows; the band keys' dK / dV are llsa_bwd_kv_tc's (tc_sa.cu)
bool tc_llsa_bwd_fused_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense) {
  if (dtype != SATTN_BF16 || D != 64 || !dense || R < 1 || R > 16 || L < 0) return false;
  const int hz = fused_hz(L, R);
  return hz >= 4 && BH * T - 1 >= T + R;
}

sattn_status tc_llsa_bwd_fused(const AttnArgs& a, float* ws_del, float* ws_l2, int ws_flat, cudaStream_t st,
                                 const int* sub4) {
  ItemSub su{};
  const ItemSub* sub = nullptr;
  if (sub4) { su = ItemSub{sub4[0], sub4[1], sub4[2], sub4[3]}; sub = &su; }
  const int HZ = fused_hz(a.L, a.R);
  const int nb = (HZ + a.L + 15) / 16 * 16;
  const bool r16 = a.R > 8;
  // horizon-major items with the staircase on tcgen05 when R fills the RM staircase columns
  if ((a.R == 8 || a.R == 16) && (HZ * a.R) % 16 == 0 && (nb == 48 || nb == 64)) {
    if (nb == 48) return r16 ? bwd_fused_launch<48, 16, true>(a, HZ, ws_del, ws_l2, ws_flat, st, sub)
                             : bwd_fused_launch<48, 8, true>(a, HZ, ws_del, ws_l2, ws_flat, st, sub);
    return r16 ? bwd_fused_launch<64, 16, true>(a, HZ, ws_del, ws_l2, ws_flat, st, sub)
               : bwd_fused_launch<64, 8, true>(a, HZ, ws_del, ws_l2, ws_flat, st, sub);
  }
  switch (nb) {
    case 16:
    case 32: return r16 ? bwd_fused_launch<32, 16>(a, HZ, ws_del, ws_l2, ws_flat, st, sub) : bwd_fused_launch<32, 8>(a, HZ, ws_del, ws_l2, ws_flat, st, sub);
    case 48: return r16 ? bwd_fused_launch<48, 16>(a, HZ, ws_del, ws_l2, ws_flat, st, sub) : bwd_fused_launch<48, 8>(a, HZ, ws_del, ws_l2, ws_flat, st, sub);
    case 64: return r16 ? bwd_fused_launch<64, 16>(a, HZ, ws_del, ws_l2, ws_flat, st, sub) : bwd_fused_launch<64, 8>(a, HZ, ws_del, ws_l2, ws_flat, st, sub);
  }
  g_err = "band too wide for the fused LLSA backward";
  return SATTN_EUNSUPPORTED;
}

const char* tc_llsa_last_error() { return g_err.c_str(); }
void tc_llsa_set_trace(void* p) { g_llsa_trace = static_cast<long long*>(p); }

}  // namespace sattn
