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

namespace sattn {
namespace {

thread_local std::string g_err;
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

}  // namespace

bool tc_llsa_supported(int dtype, int D, int L, int R) {
  // one warp per channel of a 4-channel item needs >= 2 items per tile (C >= 5); the P row
  // (NB + 32 R packed / 2 <= 192 columns) and the 8 staged stair tiles need R <= 8; NB <= 64
  return dtype == SATTN_BF16 && D == 64 && R >= 4 && R <= kRmax && L + 32 <= 64;
}

sattn_status tc_llsa_forward(const AttnArgs& a, cudaStream_t st) {
  const int nb = (32 + a.L + 15) / 16 * 16;
  switch (nb) {
    case 48: return launch<48>(a, st);
    case 64: return launch<64>(a, st);
  }
  g_err = "band too wide for the LLSA tensor-core kernel";
  return SATTN_EUNSUPPORTED;
}

const char* tc_llsa_last_error() { return g_err.c_str(); }

}  // namespace sattn
