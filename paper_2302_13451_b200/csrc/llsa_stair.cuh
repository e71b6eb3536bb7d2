// llsa_stair.cuh — LLSA backward, staircase part: one tiny dense attention gradient per horizon.
//
// The staircase slot (u, c'), c' < R, is attended by exactly the R+1 outputs of horizon
// h = u + c' (Eq. 14, horizon form): (h - c, c), c = 0..R.  So per horizon h the staircase is
// a dense (R+1) x R block:  S = Q_h K_h^T,  dP = dO_h V_h^T  (Q_h / dO_h: rows (h-c, c);
// K_h / V_h: rows (h-c', c')), with P = exp(S*scale - LSE).  Two launches of the same kernel:
//   DX = true  (before the band pass): dx_(h-c, c) = sum_c' P dP, the staircase part of
//              delta = rowsum(P o dP) (G26), written to padded workspace rows for the band pass;
//   DX = false (after it): dS = P (dP - delta) with the full-row delta of the band pass, and
//              dQ_h += scale dS K_h         (added to the band part already in dQ, staged in smem)
//              dK_h  = scale dS^T Q_h,  dV_h = P^T dO_h   (complete: no other horizon touches them)
// Each block is computed by one warp with mma.sync m16n8k16 (bf16 -> fp32): C = R+1 <= 16 rows,
// R <= 8 columns.  A CTA owns 16 horizons of one (b, h); the rows it needs are, per channel c,
// the 16 frames h - c: staged with cp.async into 144-byte rows (channel tiles skewed by 16 B so
// the ldmatrix row gathers across channels are bank-conflict free).
#pragma once
#include "common.cuh"
#include "mma_sync.cuh"

namespace sattn {

constexpr int kStF = 8;           // horizons per CTA
constexpr int kStRS = 144;        // padded row stride (bytes)
constexpr int kStTile = kStF * kStRS + 16;   // one channel's rows (+ skew)

struct StairArgs {
  const bf16 *Q, *K, *V, *dO;     // Q/K/V channel stride in_cs (0 = broadcast), dO dense
  bf16 *dQ, *dK, *dV;             // dense [C][BH][T][64]
  const float *del, *l2;          // padded [C][BH][Tp] (DX = false)
  const float* lse;               // [C][BH][T] forward LSE (DX = true)
  float* dx;                      // padded [C][BH][Tp] staircase rowsum of P o dP (DX = true)
  int T, L, R, BH, Tp;
  long long in_cs, plane;
  float scale, scale_log2;
};

__device__ __forceinline__ float resid(float x) { return x - __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float st_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool DX>
__global__ void __launch_bounds__(256, 3) llsa_bwd_stair(StairArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int R = a.R, C = R + 1, T = a.T;
  const int h0 = blockIdx.x * kStF, bh = blockIdx.y;
  // channel tiles: Q[C], dO[C], K[R], V[R] (+ dQ[C] when DX = false); then a zero row,
  // LSE / delta, per-warp scratch
  uint8_t* sQ = sm;
  uint8_t* sD = sQ + C * kStTile;
  uint8_t* sK = sD + C * kStTile;
  uint8_t* sV = sK + R * kStTile;
  uint8_t* sG = sV + R * kStTile;                      // dQ rows (band part), DX = false
  uint8_t* zrow = sG + (DX ? 0 : C * kStTile);         // 144 zero bytes
  float* sL = reinterpret_cast<float*>(zrow + kStRS);   // [C][16]
  float* sE = sL + C * kStF;                            // [C][16]
  uint8_t* scratch = reinterpret_cast<uint8_t*>(sE + C * kStF);   // per warp: P, dS [16][16] bf16
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- stage: rows h - c of channel c for h in [h0, h0 + 16)  (zero outside [0, T))
  // one warp per (tensor, channel) slot: the slot's plane base and smem tile are computed once,
  // the lanes then cover its 16 rows x 8 16-byte chunks (4 cp.async each)
  const int nslot = (DX ? 2 : 3) * C + 2 * R;
  for (int sl = warp; sl < nslot; sl += blockDim.x >> 5) {
    int tsr, c;
    if (sl < C) { tsr = 0; c = sl; }
    else if (sl < 2 * C) { tsr = 3; c = sl - C; }
    else if (sl < 2 * C + R) { tsr = 1; c = sl - 2 * C; }
    else if (sl < 2 * C + 2 * R) { tsr = 2; c = sl - 2 * C - R; }
    else { tsr = 4; c = sl - 2 * C - 2 * R; }
    const bf16* base = tsr == 0 ? a.Q : tsr == 1 ? a.K : tsr == 2 ? a.V : tsr == 3 ? a.dO : a.dQ;
    const long long cs = tsr >= 3 ? a.plane : a.in_cs;
    const bf16* plane = base + c * cs + (long long)bh * T * 64;
    const uint32_t tile = (uint32_t)__cvta_generic_to_shared(
        (tsr == 0 ? sQ : tsr == 1 ? sK : tsr == 2 ? sV : tsr == 3 ? sD : sG) + c * kStTile);
    const int ch16 = lane & 7;
#pragma unroll
    for (int j = 0; j < kStF / 4; ++j) {
      const int r = (lane >> 3) + 4 * j;
      const int f = h0 + r - c;
      const bool ok = f >= 0 && f < T;
      const bf16* src = plane + (long long)(ok ? f : 0) * 64 + ch16 * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tile + r * kStRS + ch16 * 16), "l"(src),
                   "r"(ok ? 16 : 0)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int idx = tid; idx < C * kStF; idx += blockDim.x) {
    const int c = idx / kStF, r = idx % kStF, f = h0 + r - c;
    const bool ok = f >= 0 && f < T;
    if (DX) {
      sL[idx] = ok ? a.lse[((long long)c * a.BH + bh) * T + f] * 1.4426950408889634f : 0.f;
    } else {
      const long long o = ((long long)c * a.BH + bh) * a.Tp + f;
      sL[idx] = ok ? a.l2[o] : 0.f;
      sE[idx] = ok ? a.del[o] : 0.f;
    }
  }
  if (tid < kStRS / 4) reinterpret_cast<uint32_t*>(zrow)[tid] = 0u;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t zaddr = (uint32_t)__cvta_generic_to_shared(zrow);
  uint8_t* scP = scratch + warp * 2 * 16 * 32;   // [16 rows (c)][16 cols (c')] bf16, 32-byte rows
  uint8_t* scS = scP + 16 * 32;
  const uint32_t scPa = (uint32_t)__cvta_generic_to_shared(scP), scSa = (uint32_t)__cvta_generic_to_shared(scS);
  auto rowaddr = [&](const uint8_t* tile, int c, int nc, int i, int chunk) -> uint32_t {
    return c < nc ? (uint32_t)__cvta_generic_to_shared(tile + c * kStTile + i * kStRS + chunk * 16) : zaddr;
  };

  for (int i = warp; i < kStF; i += 8) {
    const int h = h0 + i;
    // ---- S = Q_h K_h^T and dP = dO_h V_h^T (16 x 8 each; rows c, cols c')
    float s[4] = {0.f, 0.f, 0.f, 0.f}, dp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // A rows m = lane & 15, 16-byte chunk 2 kk + (lane >> 4); B rows n = lane & 7, chunk 2 kk + ((lane >> 3) & 1)
      const int am = lane & 15, ach = 2 * kk + (lane >> 4);
      const int bn = lane & 7, bch = 2 * kk + ((lane >> 3) & 1);
      uint32_t aq[4], ad[4], bk[2], bv[2];
      ldsm_x4(rowaddr(sQ, am, C, i, ach), aq);
      ldsm_x4(rowaddr(sD, am, C, i, ach), ad);
      ldsm_x2(rowaddr(sK, bn, R, i, bch), bk);
      ldsm_x2(rowaddr(sV, bn, R, i, bch), bv);
      mma16816(s, aq, bk);
      mma16816(dp, ad, bv);
    }
    // ---- P, dS (this lane: rows c = g, g + 8; cols c' = 2 t4, 2 t4 + 1)
    float p[4], ds[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = g + 8 * (e >> 1), cp = 2 * t4 + (e & 1);
      const bool ok = c < C && cp < R && h - c >= 0 && h - c < T && h - cp >= 0 && h - cp < T;
      const int cc = c < C ? c : 0;
      p[e] = ok ? st_ex2(s[e] * a.scale_log2 - sL[cc * kStF + i]) : 0.f;
      ds[e] = DX ? 0.f : p[e] * (dp[e] - sE[cc * kStF + i]);
    }
    if (DX) {
      // staircase part of rowsum(P o dP) for rows c = g, g + 8 (reduce over the quad's columns)
      float r0 = fmaf(p[1], dp[1], p[0] * dp[0]), r1 = fmaf(p[3], dp[3], p[2] * dp[2]);
      r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
      r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
      r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
      r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int c = g + 8 * hh, t = h - c;
        if (t4 == 0 && c < C && t >= 0 && t < T) a.dx[((long long)c * a.BH + bh) * a.Tp + t] = hh ? r1 : r0;
      }
      continue;
    }
    // scratch copies (rows c, cols c' < 8; cols 8..15 stay zero) for the transposed products
    *reinterpret_cast<uint32_t*>(scP + g * 32 + 4 * t4) = bf2(p[0], p[1]);
    *reinterpret_cast<uint32_t*>(scP + (g + 8) * 32 + 4 * t4) = bf2(p[2], p[3]);
    *reinterpret_cast<uint32_t*>(scS + g * 32 + 4 * t4) = bf2(ds[0], ds[1]);
    *reinterpret_cast<uint32_t*>(scS + (g + 8) * 32 + 4 * t4) = bf2(ds[2], ds[3]);
    *reinterpret_cast<uint32_t*>(scP + g * 32 + 16 + 4 * t4) = 0u;
    *reinterpret_cast<uint32_t*>(scP + (g + 8) * 32 + 16 + 4 * t4) = 0u;
    *reinterpret_cast<uint32_t*>(scS + g * 32 + 16 + 4 * t4) = 0u;
    *reinterpret_cast<uint32_t*>(scS + (g + 8) * 32 + 16 + 4 * t4) = 0u;
    __syncwarp();
    // ---- dQ_h (16 x 64) = dS (A from the accumulator layout, k = c' < 8) x K_h (rows c')
    {
      // dS as bf16 hi + lo (the band part of dQ is already rounded once: keep this one exact-ish)
      const uint32_t adq[4] = {bf2(ds[0], ds[1]), bf2(ds[2], ds[3]), 0u, 0u};
      const uint32_t adl[4] = {bf2(resid(ds[0]), resid(ds[1])), bf2(resid(ds[2]), resid(ds[3])), 0u, 0u};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t b[2];
        // B = K_h [k = c'][n = d]: rows k = lane & 15 (>= R -> zero row), 16-byte chunk j
        ldsm_x2_t(rowaddr(sK, lane & 15, R, i, j), b);
        mma16816(acc, adq, b);
        mma16816(acc, adl, b);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c = g + 8 * hh, t = h - c;
          if (c < C && t >= 0 && t < T) {   // dQ row (t, c) = row i of channel c's staged tile, in place
            __nv_bfloat162* g2 = reinterpret_cast<__nv_bfloat162*>(sG + c * kStTile + i * kStRS + 16 * j + 4 * t4);
            const float2 cur = __bfloat1622float2(*g2);
            *g2 = __floats2bfloat162_rn(fmaf(acc[2 * hh], a.scale, cur.x), fmaf(acc[2 * hh + 1], a.scale, cur.y));
          }
        }
      }
    }
    // the K_h rows the dQ loop read (ldmatrix, other lanes' rows) are overwritten with dK below
    __syncwarp();
    // ---- dV_h = P^T dO_h and dK_h = scale dS^T Q_h (16 x 64; rows c', k = c)
    {
      uint32_t ap[4], as[4];
      // A = P^T [m = c'][k = c] from the [c][c'] scratch: matrix j = rows c 8(j >> 1).., cols c' 8(j & 1)..
      const int jm = lane >> 3, rr = lane & 7;
      ldsm_x4_t(scPa + (8 * (jm >> 1) + rr) * 32 + 16 * (jm & 1), ap);
      ldsm_x4_t(scSa + (8 * (jm >> 1) + rr) * 32 + 16 * (jm & 1), as);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float dv[4] = {0.f, 0.f, 0.f, 0.f}, dk[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t bd[2], bq[2];
        ldsm_x2_t(rowaddr(sD, lane & 15, C, i, j), bd);   // B = dO_h [k = c][n = d]
        ldsm_x2_t(rowaddr(sQ, lane & 15, C, i, j), bq);   // B = Q_h  [k = c][n = d]
        mma16816(dv, ap, bd);
        mma16816(dk, as, bq);
        const int cp = g;                                 // rows c' = g (rows g + 8 are padding)
        const int u = h - cp;
        if (cp < R && u >= 0 && u < T) {
          // the staircase key (u, c') is horizon h's alone: its K / V rows (row i of tile c', read
          // only by this warp, above) take dK / dV in place
          const int o = cp * kStTile + i * kStRS + 16 * j + 4 * t4;
          *reinterpret_cast<__nv_bfloat162*>(sV + o) = __floats2bfloat162_rn(dv[0], dv[1]);
          *reinterpret_cast<__nv_bfloat162*>(sK + o) = __floats2bfloat162_rn(dk[0] * a.scale, dk[1] * a.scale);
        }
      }
    }
    __syncwarp();
  }
  if (DX) return;
  // ---- write the staged dQ (all channels) and the staircase dK / dV rows: 16-byte stores
  __syncthreads();
  for (int sl = warp; sl < C + 2 * R; sl += blockDim.x >> 5) {
    const int tsr = sl < C ? 0 : sl < C + R ? 1 : 2;
    const int c = tsr == 0 ? sl : tsr == 1 ? sl - C : sl - C - R;
    const uint8_t* tile = (tsr == 0 ? sG : tsr == 1 ? sK : sV) + c * kStTile;
    bf16* plane = (tsr == 0 ? a.dQ : tsr == 1 ? a.dK : a.dV) + c * a.plane + (long long)bh * T * 64;
    const int ch16 = lane & 7;
#pragma unroll
    for (int j = 0; j < kStF / 4; ++j) {
      const int r = (lane >> 3) + 4 * j;
      const int f = h0 + r - c;
      if (f >= 0 && f < T)
        *reinterpret_cast<uint4*>(plane + (long long)f * 64 + ch16 * 8) =
            *reinterpret_cast<const uint4*>(tile + r * kStRS + ch16 * 16);
    }
  }
}

inline size_t stair_smem_bytes(int R, bool dx) {
  const int C = R + 1;
  return (size_t)((dx ? 2 : 3) * C + 2 * R) * kStTile + kStRS + 2 * (size_t)C * kStF * sizeof(float) + 8 * 2 * 16 * 32;
}

}  // namespace sattn
