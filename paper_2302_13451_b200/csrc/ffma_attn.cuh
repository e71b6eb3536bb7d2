// ffma_attn.cuh — CUDA-core (fp32 FFMA) SA / LLSA forward and backward kernels.
//
// These are the any-D / fp32-exact kernel family (SATTN_IMPL_FFMA).  The bf16
// D=64 headline path uses the tcgen05 kernels in tc_sa.cu; DESIGN.md §5 gives
// the roofline argument for which family wins where.
//
// Work decomposition (all three kernels):
//  * a "group" is a lane pair (2g, 2g+1) that owns one query (fwd, dQ) or one key
//    slot (dK/dV) and splits the head dim D in halves (HD = D/2 registers per
//    tensor per thread); partial dot products are combined with one
//    __shfl_xor(…, 1), so both lanes hold the identical score.
//  * a CTA = NW warps = 16*NW consecutive frames of one (channel, batch*head).
//  * the rows every group of the CTA needs from one channel form a contiguous
//    frame range (the "band union"): they are staged in shared memory as fp32
//    in blocks of RB rows (coalesced 16-byte loads) and read by all lanes of a
//    warp at the same address (broadcast), so smem bandwidth never binds.
//    Rows outside a group's own window are computed and masked to -inf before
//    the row max (masked probabilities are exactly 0, G14).
//  * LLSA's staircase slots (Eq. 14's look-ahead keys from channels < R) are a
//    different row per lane; they are read straight from global memory (L1/L2).
//  * softmax is online (running max/sum in the log2 domain, scores prescaled by
//    scale*log2(e)); the backward recomputes P = exp(z - LSE) (no stored P).
//  * no atomics anywhere: every output element is produced by one group in a
//    fixed order, so results are bitwise reproducible run to run (G18).
//
// Windows (Appendix B of SURVEY.md; reading G6 for LLSA):
//  SA   query t:      keys u in [t-L, t+R] of the single channel (Eq. 4).
//  LLSA query (t,c):  h = t+c;  band    (u, R)      u in [h-R-L, h-R]
//                               stair   (h-R+j, R-j) j = 1..R           (Eq. 14)
//  dK/dV gathers:
//  SA   key u:        queries n in [u-R, u+L]                       (Eq. 7 condition, G3)
//  LLSA key (u,R):    queries (h-c, c), h in [u+R, u+R+L], c = 0..R
//  LLSA key (u,c'<R): queries (u+c'-c, c), c = 0..R  (the one horizon h = u+c')
#pragma once
#include "common.cuh"

namespace sattn {

constexpr int kNW = 4;              // warps per CTA
constexpr int kQT = 16 * kNW;       // frames (queries or keys) per CTA
constexpr int kRB = 128;            // staged rows per smem block
constexpr int kCH = 4;              // rows per inner chunk (ILP for the dot chains)

struct AttnArgs {
  const void* Q; const void* K; const void* V;  // inputs, channel stride in_cs (0 = broadcast)
  const void* O; const void* dO;                // backward inputs, dense channel stride out_cs
  const float* LSE;                             // backward input  [C][BH][T]
  void* Out; float* LSEout;                     // forward outputs
  void* dQ; void* dK; void* dV;                 // backward outputs (dense)
  float* delta;                                 // backward workspace [C][BH][T]
  void* P;                                      // SA banded probabilities [BH][T][ldp] (PST kernels)
  int ldp;
  int T, L, R, BH;
  float scale, scale_log2;
  long long in_cs, out_cs;
  // time-shard launches (tensor-core SA only; 0 = defaults): row stride ld (frames) of the
  // [BH][ld][D] tensors and [BH][ld] LSE when it differs from T, and a query-tile subset
  // (see TcArgs in tc_sa.cu)
  int ld;
  int nkt, kt0, kt_split, kt_jump;
  // packed tiles (tensor-core SA, tc_sa.cu flat_view): T is the flattened BH*T frame axis, BH = 1,
  // and Th the frames of one head (every row attends inside its own head); 0 = T
  int Th;
};

template <int D> struct Smem {
  static constexpr int HD = D / 2;
  static constexpr int SD = D + 4;                 // row stride: [half0][4 pad][half1]
  __device__ static int half_off(int half) { return half * (HD + 4); }
};

template <typename E, int D>
__device__ __forceinline__ const E* row_ptr(const void* base, long long cs, int c, int bh, int T, int t) {
  return reinterpret_cast<const E*>(base) + (long long)c * cs + ((long long)bh * T + t) * D;
}

// Stage rows [b0, b0+nr) (all inside [0,T)) of one (channel, bh) plane into smem as fp32.
template <int D, typename E>
__device__ __forceinline__ void stage_rows(float* dst, const E* plane, int b0, int nr) {
  constexpr int HD = D / 2, SD = D + 4;
  if constexpr (D >= 16) {
    constexpr int VE = 16 / sizeof(E);
    constexpr int CPR = D / VE;
    for (int idx = threadIdx.x; idx < nr * CPR; idx += blockDim.x) {
      const int r = idx / CPR, d0 = (idx % CPR) * VE;
      float tmp[VE];
      load_vec<VE>(tmp, plane + (long long)(b0 + r) * D + d0);
      float* o = dst + r * SD + d0 + (d0 >= HD ? 4 : 0);
#pragma unroll
      for (int i = 0; i < VE; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(tmp[i], tmp[i + 1], tmp[i + 2], tmp[i + 3]);
    }
  } else {
    for (int idx = threadIdx.x; idx < nr * D; idx += blockDim.x) {
      const int r = idx / D, d = idx % D;
      dst[r * SD + d + (d >= HD ? 4 : 0)] = to_f(plane[(long long)(b0 + r) * D + d]);
    }
  }
}

template <int N>
__device__ __forceinline__ float dot(const float* a, const float* b) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) s = fmaf(a[i], b[i], s);
  return s;
}

__device__ __forceinline__ float pair_sum(float x) { return x + __shfl_xor_sync(0xffffffffu, x, 1); }

// --------------------------------------------------------------------------------------------
// forward: O, LSE
// --------------------------------------------------------------------------------------------
// PST (SA only, the paper's stored band, NEXT-4 / P:L342): also write a_t into
// P[bh][t][j] = a_{t, t-L+j}, j in [0, ldp), zero outside the clipped window, by a second
// pass over the window once the row's LSE is known.
template <int D, bool LLSA, typename E, bool PST = false>
__global__ void __launch_bounds__(32 * kNW) fwd_ffma(AttnArgs a) {
  constexpr int HD = D / 2, SD = Smem<D>::SD;
  extern __shared__ __align__(16) float smem[];
  float* sK = smem;
  float* sV = smem + kRB * SD;
  const int tid = threadIdx.x, warp = tid >> 5, g = tid >> 1, half = tid & 1;
  const int c = blockIdx.y, bh = blockIdx.z;
  const int T = a.T, L = a.L, R = a.R;
  const int t0 = blockIdx.x * kQT, t = t0 + g;
  const bool active = t < T;
  const int lo_off = LLSA ? c - R - L : -L;
  const int hi_off = LLSA ? c - R : R;
  const int band_ch = LLSA ? R : 0;
  const int hoff = Smem<D>::half_off(half);

  float q[HD], acc[HD];
  load_vec<HD>(q, row_ptr<E, D>(a.Q, a.in_cs, c, bh, T, min(t, T - 1)) + half * HD);
#pragma unroll
  for (int i = 0; i < HD; ++i) { q[i] *= a.scale_log2; acc[i] = 0.f; }
  float m = neg_inf(), l = 0.f;

  const int my_lo = t + lo_off, my_hi = t + hi_off;
  const int tw = t0 + warp * 16;
  const int ulo = max(0, t0 + lo_off), uhi = min(T - 1, t0 + kQT - 1 + hi_off);
  const int wlo = max(0, tw + lo_off), whi = min(T - 1, tw + 15 + hi_off);
  const E* kplane = row_ptr<E, D>(a.K, a.in_cs, band_ch, bh, T, 0);
  const E* vplane = row_ptr<E, D>(a.V, a.in_cs, band_ch, bh, T, 0);

  for (int b0 = ulo; b0 <= uhi; b0 += kRB) {
    const int nr = min(kRB, uhi - b0 + 1);
    __syncthreads();
    stage_rows<D, E>(sK, kplane, b0, nr);
    stage_rows<D, E>(sV, vplane, b0, nr);
    __syncthreads();
    const int r0 = max(b0, wlo), r1 = min(b0 + nr - 1, whi);
    for (int r = r0; r <= r1; r += kCH) {
      float s[kCH];
#pragma unroll
      for (int k = 0; k < kCH; ++k) s[k] = dot<HD>(q, sK + (min(r + k, r1) - b0) * SD + hoff);
#pragma unroll
      for (int k = 0; k < kCH; ++k) {
        s[k] = pair_sum(s[k]);
        const int row = r + k;
        const bool v = row <= r1 && row >= my_lo && row <= my_hi;
        s[k] = v ? s[k] : neg_inf();
      }
      float mc = s[0];
#pragma unroll
      for (int k = 1; k < kCH; ++k) mc = fmaxf(mc, s[k]);
      const float mn = fmaxf(m, mc);
      if (mn != neg_inf()) {
        const float alpha = exp2f(m - mn);
        float p[kCH], ps = 0.f;
#pragma unroll
        for (int k = 0; k < kCH; ++k) { p[k] = exp2f(s[k] - mn); ps += p[k]; }
        l = l * alpha + ps;
#pragma unroll
        for (int i = 0; i < HD; ++i) acc[i] *= alpha;
#pragma unroll
        for (int k = 0; k < kCH; ++k) {
          const float* vr = sV + (min(r + k, r1) - b0) * SD + hoff;
#pragma unroll
          for (int i = 0; i < HD; ++i) acc[i] = fmaf(p[k], vr[i], acc[i]);
        }
        m = mn;
      }
    }
  }
  if constexpr (LLSA) {
    for (int j = 1; j <= R; ++j) {
      const int f = t + c - R + j;
      const bool v = active && f >= 0 && f < T;
      const int fc = min(max(f, 0), T - 1);
      float kk[HD], vv[HD];
      load_vec<HD>(kk, row_ptr<E, D>(a.K, a.in_cs, R - j, bh, T, fc) + half * HD);
      float s = pair_sum(dot<HD>(q, kk));
      s = v ? s : neg_inf();
      const float mn = fmaxf(m, s);
      if (mn != neg_inf()) {
        load_vec<HD>(vv, row_ptr<E, D>(a.V, a.in_cs, R - j, bh, T, fc) + half * HD);
        const float alpha = exp2f(m - mn), p = exp2f(s - mn);
        l = l * alpha + p;
#pragma unroll
        for (int i = 0; i < HD; ++i) acc[i] = fmaf(p, vv[i], acc[i] * alpha);
        m = mn;
      }
    }
  }
  if (active) {
    const float inv = 1.f / l;
#pragma unroll
    for (int i = 0; i < HD; ++i) acc[i] *= inv;
    E* orow = reinterpret_cast<E*>(a.Out) + (long long)c * a.out_cs + ((long long)bh * T + t) * D + half * HD;
    store_vec<HD>(orow, acc);
    if (half == 0) a.LSEout[((long long)c * a.BH + bh) * T + t] = (m + log2f(l)) * kLn2;
  }
  if constexpr (PST && !LLSA) {
    const float lse2 = m + log2f(l);
    E* prow = reinterpret_cast<E*>(a.P) + ((long long)bh * T + t) * a.ldp;
    // entries outside the clipped window (sequence edges, padding j >= W): zero
    if (active)
      for (int j = half; j < a.ldp; j += 2) {
        const int u = t - L + j;
        if (u < 0 || u >= T || j > L + R) prow[j] = from_f<E>(0.f);
      }
    const bool single = uhi - ulo + 1 <= kRB;   // sK still holds the whole union
    for (int b0 = ulo; b0 <= uhi; b0 += kRB) {
      const int nr = min(kRB, uhi - b0 + 1);
      if (!single) {
        __syncthreads();
        stage_rows<D, E>(sK, kplane, b0, nr);
        __syncthreads();
      }
      const int r0 = max(b0, wlo), r1 = min(b0 + nr - 1, whi);
      for (int r = r0; r <= r1; ++r) {
        const float sc = pair_sum(dot<HD>(q, sK + (r - b0) * SD + hoff));
        if (active && half == (r & 1) && r >= my_lo && r <= my_hi) prow[r - my_lo] = from_f<E>(exp2f(sc - lse2));
      }
    }
  }
}

// --------------------------------------------------------------------------------------------
// backward 1 (query-major): delta_t = dO_t . O_t and dQ_t = scale * sum_u dS_tu k_u
// --------------------------------------------------------------------------------------------
// PST (SA only): P_tu read from the stored band a.P instead of exp2(z - LSE) (no q . k)
template <int D, bool LLSA, typename E, bool PST = false>
__global__ void __launch_bounds__(32 * kNW) bwd_dq_ffma(AttnArgs a) {
  constexpr int HD = D / 2, SD = Smem<D>::SD;
  extern __shared__ __align__(16) float smem[];
  float* sK = smem;
  float* sV = smem + kRB * SD;
  const int tid = threadIdx.x, warp = tid >> 5, g = tid >> 1, half = tid & 1;
  const int c = blockIdx.y, bh = blockIdx.z;
  const int T = a.T, L = a.L, R = a.R;
  const int t0 = blockIdx.x * kQT, t = t0 + g;
  const bool active = t < T;
  const int tc = min(t, T - 1);
  const int lo_off = LLSA ? c - R - L : -L;
  const int hi_off = LLSA ? c - R : R;
  const int band_ch = LLSA ? R : 0;
  const int hoff = Smem<D>::half_off(half);

  float q[HD], dout[HD], dq[HD];
  {
    float o[HD];
    load_vec<HD>(q, row_ptr<E, D>(a.Q, a.in_cs, c, bh, T, tc) + half * HD);
    load_vec<HD>(dout, row_ptr<E, D>(a.dO, a.out_cs, c, bh, T, tc) + half * HD);
    load_vec<HD>(o, row_ptr<E, D>(a.O, a.out_cs, c, bh, T, tc) + half * HD);
#pragma unroll
    for (int i = 0; i < HD; ++i) { q[i] *= a.scale_log2; dq[i] = 0.f; }
    const float delta = pair_sum(dot<HD>(dout, o));
    if (active && half == 0) a.delta[((long long)c * a.BH + bh) * T + t] = delta;
    const float lse2 = PST ? 0.f : a.LSE[((long long)c * a.BH + bh) * T + tc] * kLog2e;
    const E* prow = PST ? reinterpret_cast<const E*>(a.P) + ((long long)bh * T + tc) * a.ldp : nullptr;

    const int my_lo = t + lo_off, my_hi = t + hi_off;
    const int tw = t0 + warp * 16;
    const int ulo = max(0, t0 + lo_off), uhi = min(T - 1, t0 + kQT - 1 + hi_off);
    const int wlo = max(0, tw + lo_off), whi = min(T - 1, tw + 15 + hi_off);
    const E* kplane = row_ptr<E, D>(a.K, a.in_cs, band_ch, bh, T, 0);
    const E* vplane = row_ptr<E, D>(a.V, a.in_cs, band_ch, bh, T, 0);

    for (int b0 = ulo; b0 <= uhi; b0 += kRB) {
      const int nr = min(kRB, uhi - b0 + 1);
      __syncthreads();
      stage_rows<D, E>(sK, kplane, b0, nr);
      stage_rows<D, E>(sV, vplane, b0, nr);
      __syncthreads();
      const int r0 = max(b0, wlo), r1 = min(b0 + nr - 1, whi);
      for (int r = r0; r <= r1; r += kCH) {
        float s[kCH], dp[kCH];
#pragma unroll
        for (int k = 0; k < kCH; ++k) {
          const int ro = (min(r + k, r1) - b0) * SD + hoff;
          s[k] = PST ? 0.f : dot<HD>(q, sK + ro);
          dp[k] = dot<HD>(dout, sV + ro);
        }
#pragma unroll
        for (int k = 0; k < kCH; ++k) {
          if (!PST) s[k] = pair_sum(s[k]);
          dp[k] = pair_sum(dp[k]);
          const int row = r + k;
          const bool v = row <= r1 && row >= my_lo && row <= my_hi;
          float p;
          if constexpr (PST) p = v ? to_f(prow[row - my_lo]) : 0.f;
          else p = v ? exp2f(s[k] - lse2) : 0.f;
          const float ds = p * (dp[k] - delta);
          const float* kr = sK + (min(row, r1) - b0) * SD + hoff;
#pragma unroll
          for (int i = 0; i < HD; ++i) dq[i] = fmaf(ds, kr[i], dq[i]);
        }
      }
    }
    if constexpr (LLSA) {
      for (int j = 1; j <= R; ++j) {
        const int f = t + c - R + j;
        const bool v = active && f >= 0 && f < T;
        const int fc = min(max(f, 0), T - 1);
        float kk[HD], vv[HD];
        load_vec<HD>(kk, row_ptr<E, D>(a.K, a.in_cs, R - j, bh, T, fc) + half * HD);
        load_vec<HD>(vv, row_ptr<E, D>(a.V, a.in_cs, R - j, bh, T, fc) + half * HD);
        const float s = pair_sum(dot<HD>(q, kk));
        const float dpv = pair_sum(dot<HD>(dout, vv));
        const float p = v ? exp2f(s - lse2) : 0.f;
        const float ds = p * (dpv - delta);
#pragma unroll
        for (int i = 0; i < HD; ++i) dq[i] = fmaf(ds, kk[i], dq[i]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < HD; ++i) dq[i] *= a.scale;
    E* out = reinterpret_cast<E*>(a.dQ) + (long long)c * a.out_cs + ((long long)bh * T + t) * D + half * HD;
    store_vec<HD>(out, dq);
  }
}

// --------------------------------------------------------------------------------------------
// backward 2 (key-major): dK_u = scale * sum_n dS_nu q_n,  dV_u = sum_n P_nu dO_n
// --------------------------------------------------------------------------------------------
// pst >= 0: P_nu is the stored band value pst (PST kernels), no q . k
template <int D, typename E, bool PST = false>
__device__ __forceinline__ void dkdv_row(const float* qr, const float* dor, float lse2, float delta, bool valid,
                                         const float* k, const float* v, float* dk, float* dv, float scale_log2,
                                         float pst = 0.f) {
  constexpr int HD = D / 2;
  const float dp = pair_sum(dot<HD>(dor, v));
  float p;
  if constexpr (PST) {
    p = valid ? pst : 0.f;
  } else {
    const float sc = pair_sum(dot<HD>(qr, k)) * scale_log2;   // every lane: pair_sum is a shuffle
    p = valid ? exp2f(sc - lse2) : 0.f;
  }
  const float ds = p * (dp - delta);
#pragma unroll
  for (int i = 0; i < HD; ++i) {
    dv[i] = fmaf(p, dor[i], dv[i]);
    dk[i] = fmaf(ds, qr[i], dk[i]);
  }
}

// PST (SA only): P_nu = a.P[n][u - n + L] (the stored band, read along its diagonal)
template <int D, bool LLSA, typename E, bool PST = false>
__global__ void __launch_bounds__(32 * kNW) bwd_dkdv_ffma(AttnArgs a) {
  constexpr int HD = D / 2, SD = Smem<D>::SD;
  extern __shared__ __align__(16) float smem[];
  float* sQ = smem;
  float* sD = smem + kRB * SD;
  float* sL = smem + 2 * kRB * SD;      // lse * log2(e)
  float* sE = sL + kRB;                 // delta
  const int tid = threadIdx.x, warp = tid >> 5, g = tid >> 1, half = tid & 1;
  const int cp = blockIdx.y, bh = blockIdx.z;
  const int T = a.T, L = a.L, R = a.R;
  const int u0 = blockIdx.x * kQT, u = u0 + g;
  const bool active = u < T;
  const int uc = min(u, T - 1);
  const int hoff = Smem<D>::half_off(half);
  const long long lse_plane = (long long)a.BH * T;

  float k[HD], v[HD], dk[HD], dv[HD];
  load_vec<HD>(k, row_ptr<E, D>(a.K, a.in_cs, cp, bh, T, uc) + half * HD);
  load_vec<HD>(v, row_ptr<E, D>(a.V, a.in_cs, cp, bh, T, uc) + half * HD);
#pragma unroll
  for (int i = 0; i < HD; ++i) { dk[i] = 0.f; dv[i] = 0.f; }

  const int uw = u0 + warp * 16;
  // band-union sources: queries of channel qc at frames [u + lo_off, u + hi_off]
  const bool union_mode = !LLSA || cp == R;
  const int nsrc = LLSA ? R + 1 : 1;
  if (union_mode) {
    for (int qc = 0; qc < nsrc; ++qc) {
      const int lo_off = LLSA ? R - qc : -R;
      const int hi_off = LLSA ? R + L - qc : L;
      const int my_lo = u + lo_off, my_hi = u + hi_off;
      const int ulo = max(0, u0 + lo_off), uhi = min(T - 1, u0 + kQT - 1 + hi_off);
      const int wlo = max(0, uw + lo_off), whi = min(T - 1, uw + 15 + hi_off);
      const E* qplane = row_ptr<E, D>(a.Q, a.in_cs, qc, bh, T, 0);
      const E* dplane = row_ptr<E, D>(a.dO, a.out_cs, qc, bh, T, 0);
      const float* lse = a.LSE + qc * lse_plane + (long long)bh * T;
      const float* del = a.delta + qc * lse_plane + (long long)bh * T;
      for (int b0 = ulo; b0 <= uhi; b0 += kRB) {
        const int nr = min(kRB, uhi - b0 + 1);
        __syncthreads();
        stage_rows<D, E>(sQ, qplane, b0, nr);
        stage_rows<D, E>(sD, dplane, b0, nr);
        for (int i = tid; i < nr; i += blockDim.x) {
          if (!PST) sL[i] = lse[b0 + i] * kLog2e;
          sE[i] = del[b0 + i];
        }
        __syncthreads();
        const int r0 = max(b0, wlo), r1 = min(b0 + nr - 1, whi);
        for (int r = r0; r <= r1; ++r) {
          const bool valid = r >= my_lo && r <= my_hi;
          const int ro = (r - b0) * SD + hoff;
          if constexpr (PST) {
            const float pv = valid ? to_f(reinterpret_cast<const E*>(a.P)[((long long)bh * T + r) * a.ldp + (uc - r + L)]) : 0.f;
            dkdv_row<D, E, true>(sQ + ro, sD + ro, 0.f, sE[r - b0], valid, k, v, dk, dv, a.scale_log2, pv);
          } else {
            dkdv_row<D, E>(sQ + ro, sD + ro, sL[r - b0], sE[r - b0], valid, k, v, dk, dv, a.scale_log2);
          }
        }
      }
    }
  } else {
    // staircase key (u, cp < R): the single horizon h = u + cp, queries (h - qc, qc)
    for (int qc = 0; qc <= R; ++qc) {
      const int n = u + cp - qc;
      const bool valid = active && n >= 0 && n < T;
      const int nc = min(max(n, 0), T - 1);
      float qr[HD], dor[HD];
      load_vec<HD>(qr, row_ptr<E, D>(a.Q, a.in_cs, qc, bh, T, nc) + half * HD);
      load_vec<HD>(dor, row_ptr<E, D>(a.dO, a.out_cs, qc, bh, T, nc) + half * HD);
      const float lse2 = a.LSE[qc * lse_plane + (long long)bh * T + nc] * kLog2e;
      const float del = a.delta[qc * lse_plane + (long long)bh * T + nc];
      dkdv_row<D, E>(qr, dor, lse2, del, valid, k, v, dk, dv, a.scale_log2);
    }
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < HD; ++i) dk[i] *= a.scale;
    const long long off = (long long)cp * a.out_cs + ((long long)bh * T + u) * D + half * HD;
    store_vec<HD>(reinterpret_cast<E*>(a.dK) + off, dk);
    store_vec<HD>(reinterpret_cast<E*>(a.dV) + off, dv);
  }
}

template <int D> constexpr size_t fwd_smem_bytes() { return 2u * kRB * (D + 4) * sizeof(float); }
template <int D> constexpr size_t dkdv_smem_bytes() { return (2u * kRB * (D + 4) + 2u * kRB) * sizeof(float); }

}  // namespace sattn
