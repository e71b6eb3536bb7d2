// stream_step.cuh — one incremental LLSA step (infer_llsa) and one
// incremental SA step (infer_sa).
//
// LLSA: one launch runs horizon h through every layer.  CTA = one (batch, head) stream.
// At horizon h each layer computes the R+1 outputs (h-c, c), c = 0..R, which all
// share one window ("the same keys and values of the red vector are used"):
//   slot i in [0, L)      (u = h-R-L+i, channel R): ring of the layer input
//   slot i = L            (u = h-R,     channel R): the current diagonal
//   slot i in [L+1, L+R]  (u = h-R-L+i, channel L+R-i): the current diagonal
// so a (R+1) x (L+R+1) attention per layer; tied Q = K = V = the layer input
// (reading G12), X_{l+1} = (X_l + O_l)/2 rounded exactly like the offline stack
// (O rounded to the storage type first, then the half-sum).  Layer 1's diagonal is
// the last R+1 raw frames (every channel of X_0 equals x).
//
// Latency structure: the layers of a step are sequential, so a step costs n_layers x (one
// layer's dependent phases).  Everything a layer reads that is known at launch — the ring rows
// of every layer (written by earlier steps) — is fetched once, up front, in parallel, into
// shared memory.  Within a layer ONE WARP owns one query row end to end: its query sits in
// registers, lane i scores key i (a 16-byte-vector dot product over a bank-conflict-free row),
// the row softmax is a pair of warp shuffles, and lane d accumulates the value sum of
// dimension d — so a layer has no block-wide barrier except the one that publishes its
// outputs to the next layer.
#pragma once
#include "common.cuh"
#include "mma_sync.cuh"

namespace sattn {

// Shared-memory rows: stride chosen so that the 8 lanes of a 16-byte-load phase hit distinct
// bank groups (stride ≡ 16 bytes mod 128 for D = 64 in either dtype); odd-sized rows fall
// back to scalar loads with a +1 pad.
template <int D, typename T>
struct StreamRow {
  static constexpr bool VEC = (D * sizeof(T)) % 16 == 0;
  static constexpr int N = VEC ? 16 / (int)sizeof(T) : 1;   // elements per vector load
  static constexpr int STRIDE = VEC ? D + N : D + 1;         // elements
};

__device__ __forceinline__ void lds_vec(float* dst, const float* src) {
  const float4 v = *reinterpret_cast<const float4*>(src);
  dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
}
__device__ __forceinline__ void lds_vec(float* dst, const bf16* src) {
  const uint4 raw = *reinterpret_cast<const uint4*>(src);
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(p[j]);
    dst[2 * j] = f.x; dst[2 * j + 1] = f.y;
  }
}

// q . row with four interleaved partial sums (fixed order: deterministic, same as the CUDA-core
// attention kernels' dot products)
template <int D, typename T>
__device__ __forceinline__ float stream_dot(const float (&q)[D], const T* row) {
  using RT = StreamRow<D, T>;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (RT::VEC) {
#pragma unroll
    for (int k = 0; k < D / RT::N; ++k) {
      float v[RT::N];
      lds_vec(v, row + k * RT::N);
#pragma unroll
      for (int j = 0; j < RT::N; ++j) acc[(k * RT::N + j) & 3] = fmaf(q[k * RT::N + j], v[j], acc[(k * RT::N + j) & 3]);
    }
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d & 3] = fmaf(q[d], to_f(row[d]), acc[d & 3]);
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

template <int D, typename T>
__device__ __forceinline__ void load_row_regs(float (&q)[D], const T* row) {
  using RT = StreamRow<D, T>;
  if constexpr (RT::VEC) {
#pragma unroll
    for (int k = 0; k < D / RT::N; ++k) lds_vec(q + k * RT::N, row + k * RT::N);
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) q[d] = to_f(row[d]);
  }
}

// Copy n_rows ring rows (global, T, row length D) into shared rows of StreamRow<D,T>::STRIDE;
// rows whose frame is invalid (src_row returns < 0) are zero-filled.
template <int D, typename T, class SrcRow>
__device__ __forceinline__ void stage_rows(T* dst, const T* ring, int n_rows, SrcRow src_row, int tid, int nt) {
  using RT = StreamRow<D, T>;
  constexpr int PER = RT::VEC ? D / RT::N : D;
  for (int idx = tid; idx < n_rows * PER; idx += nt) {
    const int ch = idx % PER, r = idx / PER;
    const long long sr = src_row(r);
    T* d = dst + (long long)r * RT::STRIDE;
    if constexpr (RT::VEC) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (sr >= 0) v = *reinterpret_cast<const uint4*>(ring + sr * D + ch * RT::N);
      *reinterpret_cast<uint4*>(d + ch * RT::N) = v;
    } else {
      d[ch] = sr >= 0 ? ring[sr * D + ch] : from_f<T>(0.f);
    }
  }
}

__device__ __forceinline__ float warp_max(float m) {
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}
__device__ __forceinline__ float warp_sum(float s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// One warp: softmax weights of query q over window rows [i0, i1] (i0 <= i1; row_of gives each
// row's pointer and kind), normalised into Pw[i].  Then the value sum of lane's dimensions: y[e] for d = lane*E + e (E = D/32 for D = 64, else 1 with
// lanes >= D idle).
template <int D, typename T, class RowF>
__device__ __forceinline__ void warp_attend(const float (&q)[D], int i0, int i1, float scale_log2, float* Pw,
                                            RowF row_of, int lane, float* y) {
  constexpr int E = D >= 64 ? D / 32 : 1;
  // scores (log2 domain), lane i <-> key i
  float m = neg_inf();
  for (int i = i0 + lane; i <= i1; i += 32) {
    const bool ring_row = row_of.is_ring(i);
    const float s = (ring_row ? stream_dot<D, T>(q, row_of.ring(i)) : stream_dot<D, float>(q, row_of.diag(i))) * scale_log2;
    Pw[i] = s;
    m = fmaxf(m, s);
  }
  m = warp_max(m);
  float sum = 0.f;
  for (int i = i0 + lane; i <= i1; i += 32) {
    const float e = exp2f(Pw[i] - m);
    Pw[i] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  const float inv = sum > 0.f ? 1.f / sum : 0.f;
  for (int i = i0 + lane; i <= i1; i += 32) Pw[i] *= inv;
  __syncwarp();
  // value sum: four interleaved partial sums over the window (slot k of the four <-> (i - i0) mod 4)
  float y4[4][E];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int e = 0; e < E; ++e) y4[k][e] = 0.f;
  const int d0 = lane * E;
  auto acc = [&](float (&yk)[E], int i) {
    const float p = Pw[i];
    if (row_of.is_ring(i)) {
      const T* r = row_of.ring(i) + d0;
#pragma unroll
      for (int e = 0; e < E; ++e) yk[e] = fmaf(p, to_f(r[e]), yk[e]);
    } else {
      const float* r = row_of.diag(i) + d0;
#pragma unroll
      for (int e = 0; e < E; ++e) yk[e] = fmaf(p, r[e], yk[e]);
    }
  };
  if (d0 < D) {
    int i = i0;
    for (; i + 3 <= i1; i += 4) {
      acc(y4[0], i); acc(y4[1], i + 1); acc(y4[2], i + 2); acc(y4[3], i + 3);
    }
    if (i <= i1) acc(y4[0], i);
    if (i + 1 <= i1) acc(y4[1], i + 1);
    if (i + 2 <= i1) acc(y4[2], i + 2);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) y[e] = (y4[0][e] + y4[1][e]) + (y4[2][e] + y4[3][e]);
}

struct StreamArgs {
  const void* x_new;   // [BH][D] or nullptr (flush step)
  void* raw;           // [BH][R+1][D], slot = frame mod (R+1)
  void* ring;          // [n_layers][BH][L][D], slot = frame mod L
  void* y_out;         // [BH][D] or nullptr
  long long h, last;   // horizon and last valid frame
  int n_layers, L, R, BH;
  float scale_log2;
  int preload;         // 1: every layer's ring rows are staged into shared memory at the start
};

constexpr int kStreamMaxWarps = 18;   // one warp per LLSA query channel for R <= 17

template <int D, typename T>
struct LLSARows {
  const T* rp;         // this layer's staged ring rows, [L][STRIDE]
  const float* dp;     // the current diagonal, [C][SPD]
  int L, R, SPD;
  __device__ bool is_ring(int i) const { return i < L; }
  __device__ const T* ring(int i) const { return rp + (long long)i * StreamRow<D, T>::STRIDE; }
  __device__ const float* diag(int i) const { return dp + (long long)(i == L ? R : L + R - i) * SPD; }
};

template <int D, typename T>
__global__ void __launch_bounds__(32 * kStreamMaxWarps) llsa_stream_step_kernel(StreamArgs a) {
  using RT = StreamRow<D, T>;
  constexpr int SPD = StreamRow<D, float>::STRIDE;
  constexpr int E = D >= 64 ? D / 32 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = a.L, R = a.R, C = R + 1, W = L + R + 1, Wp = (W + 3) & ~3;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
  float* diag = reinterpret_cast<float*>(smem_raw);   // [C][SPD]
  float* ndiag = diag + C * SPD;                      // [C][SPD]
  float* P = ndiag + C * SPD;                         // [nwarp][Wp]
  T* rings = reinterpret_cast<T*>(P + nwarp * Wp);    // [preload ? n_layers : 1][L][STRIDE]
  const int bh = blockIdx.x;
  const long long h = a.h, last = a.last;
  const long long base = h - R - L;                   // frame of window slot 0
  T* raw = reinterpret_cast<T*>(a.raw) + (long long)bh * C * D;
  const T* ring_g = reinterpret_cast<const T*>(a.ring);
  const int hmL = L > 0 ? (int)(h % L) : 0, hmC = (int)(h % C);
  // ring slot of window slot i < L (frame base + i), -1 if that frame is outside [0, last]
  auto ring_slot = [&](int i) -> int {
    const long long u = base + i;
    if (u < 0 || u > last) return -1;
    const int s = (hmL - R - L + i) % L;
    return s < 0 ? s + L : s;
  };
  if (a.preload && L > 0) {
    stage_rows<D, T>(rings, ring_g, a.n_layers * L, [&](int r) -> long long {
      const int l = r / L, sl = ring_slot(r % L);
      return sl < 0 ? -1 : ((long long)l * a.BH + bh) * L + sl;
    }, tid, nt);
  }
  // layer-1 diagonal: X_0(h - c', c') = x_{h - c'}; x_h goes into its raw slot for later steps
  const T* x = a.x_new ? reinterpret_cast<const T*>(a.x_new) + (long long)bh * D : nullptr;
  for (int idx = tid; idx < C * D; idx += nt) {
    const int cp = idx / D, d = idx % D;
    const long long f = h - cp;
    float v = 0.f;
    if (f >= 0 && f <= last) {
      if (cp == 0 && x) v = to_f(x[d]);
      else { int s = (hmC - cp) % C; s = s < 0 ? s + C : s; v = to_f(raw[s * D + d]); }
    }
    diag[cp * SPD + d] = v;
  }
  if (x)
    for (int d = tid; d < D; d += nt) raw[hmC * D + d] = x[d];
  __syncthreads();
  const int wslot = (h - R >= 0 && h - R <= last && L > 0) ? ring_slot(L) : -1;   // frame h - R
  const int i0 = (int)(base < 0 ? -base : 0);
  const int i1 = (int)(last - base < W - 1 ? last - base : W - 1);
  float* Pw = P + warp * Wp;

  for (int l = 0; l < a.n_layers; ++l) {
    const T* lring = rings;
    if (L > 0) {
      if (a.preload) {
        lring = rings + (long long)l * L * RT::STRIDE;
      } else {
        stage_rows<D, T>(rings, ring_g, L, [&](int r) -> long long {
          const int sl = ring_slot(r);
          return sl < 0 ? -1 : ((long long)l * a.BH + bh) * L + sl;
        }, tid, nt);
        __syncthreads();
      }
      // X_l(h-R, R) joins this layer's ring (its slot held frame h-R-L, already staged)
      if (wslot >= 0) {
        T* ring = reinterpret_cast<T*>(a.ring) + (((long long)l * a.BH + bh) * L + wslot) * D;
        for (int d = tid; d < D; d += nt) ring[d] = from_f<T>(diag[R * SPD + d]);
      }
    }
    const LLSARows<D, T> rows{lring, diag, L, R, SPD};
    for (int c = warp; c < C; c += nwarp) {
      const long long t = h - c;
      float y[E];
#pragma unroll
      for (int e = 0; e < E; ++e) y[e] = 0.f;
      if (t >= 0 && t <= last && i0 <= i1) {
        float q[D];
        load_row_regs<D, float>(q, diag + c * SPD);
        warp_attend<D, T>(q, i0, i1, a.scale_log2, Pw, rows, lane, y);
      }
      const int d0 = lane * E;
      if (d0 < D) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float o = to_f(from_f<T>(y[e]));
          ndiag[c * SPD + d0 + e] = to_f(from_f<T>(0.5f * (diag[c * SPD + d0 + e] + o)));
        }
      }
      __syncwarp();   // Pw is reused by this warp's next row
    }
    __syncthreads();
    float* tmp = diag; diag = ndiag; ndiag = tmp;
  }
  if (a.y_out && h - R >= 0 && h - R <= last) {
    T* y = reinterpret_cast<T*>(a.y_out) + (long long)bh * D;
    for (int d = tid; d < D; d += nt) y[d] = from_f<T>(diag[R * SPD + d]);
  }
}

// launch geometry and shared memory of the LLSA step kernel (preload: every layer's ring rows)
inline int stream_warps(int R) { return R + 1 < kStreamMaxWarps ? R + 1 : kStreamMaxWarps; }
template <int D, typename T>
inline size_t stream_smem_bytes(int L, int R, int n_stage) {
  const int C = R + 1, W = L + R + 1, Wp = (W + 3) & ~3;
  return sizeof(float) * (2 * (size_t)C * StreamRow<D, float>::STRIDE + (size_t)stream_warps(R) * Wp) +
         sizeof(T) * (size_t)n_stage * L * StreamRow<D, T>::STRIDE;
}

// ------------------------------------------------------------------------------------------
// One incremental SA step (infer_sa).  CTA = one (batch, head);
// its four warps stage the rings, then one warp runs the layers.  After frame h arrives, layer l (0-based) computes its output at
// t_l = h - (l+1) R from the window [t_l - L, t_l + R] of its input; the newest window frame
// t_l + R = h - l R is the one the layer below produced in this same step (layer 0: x_h), the
// older ones come from the layer's ring of its last L + R + 1 input frames.
// X_{l+1}(t_l) = (X_l(t_l) + Y_l(t_l)) / 2 (G12), rounded like the offline stack; the stack
// emits X_n(h - n R): latency n R frames.  One query per layer: the warp needs no block barrier.
// ------------------------------------------------------------------------------------------
struct SAStreamArgs {
  const void* x_new;   // [BH][D] or nullptr (flush step)
  void* ring;          // [n_layers][BH][L+R+1][D], slot = frame mod (L+R+1)
  void* y_out;         // [BH][D] or nullptr
  long long h, last;   // step and last valid frame
  int n_layers, L, R, BH;
  float scale_log2;
  int preload;         // 1: every layer's ring rows are staged into shared memory at the start
};

template <int D, typename T>
struct SARows {
  const T* rp;         // this layer's staged window rows 0 .. W-2, [W-1][STRIDE]
  const float* cp;     // window row W-1 (the newest frame)
  int W;
  __device__ bool is_ring(int i) const { return i < W - 1; }
  __device__ const T* ring(int i) const { return rp + (long long)i * StreamRow<D, T>::STRIDE; }
  __device__ const float* diag(int) const { return cp; }
};

constexpr int kSAStreamThreads = 128;

template <int D, typename T>
__global__ void __launch_bounds__(kSAStreamThreads) sa_stream_step_kernel(SAStreamArgs a) {
  using RT = StreamRow<D, T>;
  constexpr int E = D >= 64 ? D / 32 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = a.L, R = a.R, W = L + R + 1, Wp = (W + 3) & ~3, NR = W;
  const int lane = threadIdx.x & 31;
  float* cur = reinterpret_cast<float*>(smem_raw);           // [2][SPD]: newest input frame, double-buffered
  constexpr int SPD = StreamRow<D, float>::STRIDE;
  float* P = cur + 2 * SPD;                                   // [Wp]
  T* rings = reinterpret_cast<T*>(P + Wp);                    // [preload ? n_layers : 1][W-1][STRIDE]
  const int bh = blockIdx.x;
  const long long h = a.h, last = a.last;
  const T* ring_g = reinterpret_cast<const T*>(a.ring);
  // ring slot of frame u = (h mod NR) + (u - h) mod NR: one 64-bit modulo per step
  const int hm = (int)(h % NR);
  auto slot_of = [&](long long u) { int sl = (hm + (int)((u - h) % NR)) % NR; return sl < 0 ? sl + NR : sl; };
  auto window_src = [&](int l, int i) -> long long {   // global ring row of window row i of layer l
    const long long u = h - (long long)(l + 1) * R - L + i;
    return (u >= 0 && u <= last) ? ((long long)l * a.BH + bh) * NR + slot_of(u) : -1;
  };
  // every warp helps stage the rings; then warp 0 alone runs the layers
  if (a.preload && W > 1)
    stage_rows<D, T>(rings, ring_g, a.n_layers * (W - 1), [&](int r) { return window_src(r / (W - 1), r % (W - 1)); },
                     threadIdx.x, blockDim.x);
  bool cur_ok = a.x_new != nullptr && h <= last;
  if (cur_ok) {
    const T* x = reinterpret_cast<const T*>(a.x_new) + (long long)bh * D;
    for (int d = threadIdx.x; d < D; d += blockDim.x) cur[d] = to_f(x[d]);
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  int cb = 0;
  for (int l = 0; l < a.n_layers; ++l) {
    const long long fn = h - (long long)l * R;          // this layer's newest input frame (= cur)
    const long long t = fn - R;                          // the frame it computes
    const bool run = t >= 0 && t <= last;
    const T* lring = rings;
    if (a.preload) {
      lring = rings + (long long)l * (W - 1) * RT::STRIDE;
    } else if (run && W > 1) {
      stage_rows<D, T>(rings, ring_g, W - 1, [&](int i) { return window_src(l, i); }, lane, 32);
      __syncwarp();
    }
    float* c0 = cur + cb * SPD;
    // the newest frame joins the ring (its slot held frame fn - W, outside every window read here)
    if (cur_ok && fn >= 0) {
      T* ring = reinterpret_cast<T*>(a.ring) + (((long long)l * a.BH + bh) * NR + slot_of(fn)) * D;
      for (int d = lane; d < D; d += 32) ring[d] = from_f<T>(c0[d]);
    }
    if (run) {
      const long long base = t - L;
      const int i0 = (int)(base < 0 ? -base : 0);
      const int i1 = (int)(last - base < W - 1 ? last - base : W - 1);
      const SARows<D, T> rows{lring, c0, W};
      float q[D];
      if (L == W - 1) load_row_regs<D, float>(q, c0);
      else load_row_regs<D, T>(q, rows.ring(L));
      float y[E];
      warp_attend<D, T>(q, i0, i1, a.scale_log2, P, rows, lane, y);
      float* c1 = cur + (cb ^ 1) * SPD;
      const int d0 = lane * E;
      if (d0 < D) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float o = to_f(from_f<T>(y[e]));
          const float xq = L == W - 1 ? c0[d0 + e] : to_f(rows.ring(L)[d0 + e]);
          c1[d0 + e] = to_f(from_f<T>(0.5f * (xq + o)));
        }
      }
      cb ^= 1;
    }
    cur_ok = run;
    __syncwarp();
  }
  const long long te = h - (long long)a.n_layers * R;
  if (a.y_out && cur_ok && te >= 0 && te <= last) {
    T* y = reinterpret_cast<T*>(a.y_out) + (long long)bh * D;
    for (int d = lane; d < D; d += 32) y[d] = from_f<T>(cur[cb * SPD + d]);
  }
}

template <int D, typename T>
inline size_t sa_stream_smem_bytes(int L, int R, int n_stage) {
  const int W = L + R + 1, Wp = (W + 3) & ~3;
  return sizeof(float) * (2 * (size_t)StreamRow<D, float>::STRIDE + Wp) +
         sizeof(T) * (size_t)n_stage * (W - 1) * StreamRow<D, T>::STRIDE;
}

// ------------------------------------------------------------------------------------------
// Tensor-core step (bf16, D = 64): both streams on mma.sync, one CTA of kMmaWarps warps per
// (batch, head).
//
// A layer's window is one dense block of rows in shared memory (144-byte rows: ldmatrix
// gathers of 8 consecutive rows are bank-conflict free):
//   LLSA rows 0..L-1   the ring (channel-R frames h-R-L .. h-R-1, staged with cp.async)
//        rows L+j      channel R-j of the current diagonal (frame h-R+j), j = 0..R — the layer
//                      input the layer below produced in this step (layer 0: the raw frames)
//   SA   rows 0..W-2   the ring (frames t-L .. t+R-1, staged with cp.async)
//        row  W-1      the newest input frame (x_h, or the layer below's output of this step)
// rows up to the 16-row padding are zero.  The queries are window rows L.. (LLSA: R+1 rows,
// channel R-m in row L+m; SA: row L), so per layer S = Q K^T is one (16·MT) x Wk block of
// m16n8k16 MMAs, the row softmax runs in the accumulator registers (a row lives in a lane
// quad), P is re-packed in registers as the A operand of O = P V (ldmatrix.trans of the same
// window rows), and the epilogue X_{l+1} = (X_l + O)/2 (both rounded to bf16 as the offline
// stack stores them) lands directly in the next layer's window rows.  Every warp computes S and
// the softmax (24 MMAs at the base band), then O and the epilogue for its own 16 dims: one
// barrier per layer.  The layers' ring rows stream in through NB window buffers, NB-1 layers ahead.
// ------------------------------------------------------------------------------------------
struct StreamMmaArgs {
  const bf16* x_new;   // [BH][64] or nullptr (flush step)
  bf16* raw;           // LLSA: [BH][R+1][64], slot = frame mod (R+1)
  bf16* ring;          // LLSA: [n][BH][L][64] (slot = frame mod L); SA: [n][BH][W][64] (slot = frame mod W)
  bf16* y_out;         // [BH][64] or nullptr
  long long h, last;
  int n_layers, L, R, BH;
  int nrw, nb;         // window rows per buffer (16-padded), number of buffers
  float scale_log2;
};

constexpr int kMmaRowB = 144;   // bytes per window row (64 bf16 + 16 B skew)

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  // wait_group takes an immediate; the buffer count is small
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    default: cp_async_wait<6>(); break;
  }
}

constexpr int kMmaWarps = 4;   // warps per (batch, head): S + softmax on each, O = P V split by dims

__device__ __forceinline__ float fast_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool SA, int NT>
__global__ void __launch_bounds__(32 * kMmaWarps) stream_mma_kernel(StreamMmaArgs a) {
  extern __shared__ __align__(16) uint8_t smem_mma[];
  constexpr int KS = NT / 2;                       // 16-key steps of the PV MMA
  constexpr int DT = 8 / kMmaWarps;                // 8-dim output tiles per warp
  const int L = a.L, R = a.R, C = R + 1, W = L + R + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, tq = lane & 3;
  const int bh = blockIdx.x, NB = a.nb, NRW = a.nrw;
  const long long h = a.h, last = a.last;
  const int n_ring = SA ? W - 1 : L;               // window rows taken from the layer's ring
  const int NRG = SA ? W : L;                      // ring length (slots)
  const int MT = SA ? 1 : (C + 15) / 16;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_mma));
  auto buf_u32 = [&](int l) { return sbase + (uint32_t)((l % NB) * NRW * kMmaRowB); };
  auto buf_ptr = [&](int l) { return smem_mma + (size_t)(l % NB) * NRW * kMmaRowB; };
  const int hmod = NRG > 0 ? (int)(h % NRG) : 0;
  // ring slot of frame u (|u - h| is small): one 64-bit modulo per step
  auto slot_of = [&](long long u) { int s = (hmod + (int)(u - h)) % NRG; return s < 0 ? s + NRG : s; };
  auto frame_of = [&](int l, int i) -> long long {   // frame of window row i of layer l
    return SA ? h - (long long)(l + 1) * R - L + i : h - R - L + i;
  };
  // this thread's 16-byte chunks of a layer's ring rows (n_ring * 8 <= 504): window row, chunk, and
  // the row's frame / ring slot at layer 0 (LLSA: every layer; SA: they move back R per layer)
  constexpr int kMaxChunks = 4;
  int ch_off[kMaxChunks], ch_slot[kMaxChunks];
  long long ch_u[kMaxChunks];
#pragma unroll
  for (int j = 0; j < kMaxChunks; ++j) {
    const int idx = tid + j * 32 * kMmaWarps, r = idx >> 3;
    ch_off[j] = idx < n_ring * 8 ? r * kMmaRowB + 16 * (idx & 7) : -1;
    ch_u[j] = frame_of(0, r);
    ch_slot[j] = NRG > 0 ? slot_of(ch_u[j]) * 64 + 8 * (idx & 7) : 0;   // element offset in the ring
  }
  // one cp.async group per layer and thread (empty past the last layer: the count stays uniform)
  auto issue_layer = [&](int l) {
    if (l < a.n_layers) {
      const bf16* rg = a.ring + ((long long)l * a.BH + bh) * NRG * 64;
      const uint32_t b = buf_u32(l);
      const int shift = SA ? (int)(((long long)l * R) % NRG) * 64 : 0;   // SA: frames move back l R
#pragma unroll
      for (int j = 0; j < kMaxChunks; ++j) {
        if (ch_off[j] < 0) continue;
        const long long u = ch_u[j] - (SA ? (long long)l * R : 0);
        const bool ok = u >= 0 && u <= last;
        int e = ch_slot[j] - shift;
        if (e < 0) e += NRG * 64;
        cp_async16(b + ch_off[j], rg + (ok ? e : 0), ok);
      }
    }
    cp_async_commit();
  };
  for (int l = 0; l < NB - 1; ++l) issue_layer(l);   // the groups of layers 0 .. NB-2

  // zero the padding rows of every buffer (never written afterwards; V rows must be finite)
  for (int b = 0; b < NB; ++b)
    for (int idx = tid; idx < (NRW - W) * 9; idx += 32 * kMmaWarps)
      *reinterpret_cast<uint4*>(smem_mma + (size_t)b * NRW * kMmaRowB + (W + idx / 9) * kMmaRowB + 16 * (idx % 9)) =
          make_uint4(0, 0, 0, 0);
  // layer 0's own rows (4-byte lanes of one warp per row)
  {
    uint8_t* b0 = buf_ptr(0);
    if (SA) {
      if (warp == 0) {
        const bool ok = a.x_new != nullptr && h <= last;
        const uint32_t v = ok ? reinterpret_cast<const uint32_t*>(a.x_new + (long long)bh * 64)[lane] : 0u;
        reinterpret_cast<uint32_t*>(b0 + (W - 1) * kMmaRowB)[lane] = v;
      }
    } else {
      const int hmC = (int)(h % C);
      bf16* raw = a.raw + (long long)bh * C * 64;
      for (int j = warp; j <= R; j += kMmaWarps) {   // row L + j = channel R - j = frame h - (R - j)
        const int cp = R - j;
        const long long f = h - cp;
        uint32_t v = 0u;
        if (f >= 0 && f <= last) {
          if (cp == 0 && a.x_new) v = reinterpret_cast<const uint32_t*>(a.x_new + (long long)bh * 64)[lane];
          else { int sl = (hmC - cp) % C; sl = sl < 0 ? sl + C : sl; v = reinterpret_cast<const uint32_t*>(raw + sl * 64)[lane]; }
        }
        reinterpret_cast<uint32_t*>(b0 + (L + j) * kMmaRowB)[lane] = v;
      }
      __syncthreads();   // every read of the raw ring precedes the write of x_h into its slot
      if (a.x_new && warp == 0)
        reinterpret_cast<uint32_t*>(raw + hmC * 64)[lane] = reinterpret_cast<const uint32_t*>(a.x_new + (long long)bh * 64)[lane];
    }
  }
  bool cur_ok = SA ? (a.x_new != nullptr && h <= last) : true;   // SA: this layer's newest row is a real frame
  cp_async_wait_dyn(NB - 2);
  __syncthreads();

  int mi0 = -1, mi1 = -1;
  uint32_t cmask = 0;   // bit 2 nt + e: key column 8 nt + 2 tq + e is a valid frame
  for (int l = 0; l < a.n_layers; ++l) {
    issue_layer(l + NB - 1);   // into the buffer of layer l - 1, free since the last barrier
    uint8_t* bp = buf_ptr(l);
    const uint32_t bu = buf_u32(l);
    // the ring gains this layer's newest input row (its slot held a frame no later window reads;
    // that frame, if this step reads it, is already staged)
    if (warp == 0) {
      const long long fn = SA ? h - (long long)l * R : h - R;
      const bool wr = SA ? (cur_ok && fn >= 0) : (fn >= 0 && fn <= last && L > 0);
      if (wr) {
        bf16* dst = a.ring + (((long long)l * a.BH + bh) * NRG + slot_of(fn)) * 64;
        reinterpret_cast<uint32_t*>(dst)[lane] = reinterpret_cast<const uint32_t*>(bp + (SA ? W - 1 : L) * kMmaRowB)[lane];
      }
    }
    const long long base = frame_of(l, 0);
    const bool run = SA ? (base + L >= 0 && base + L <= last) : true;
    const int i0 = (int)(base < 0 ? -base : 0);
    const int i1 = (int)(last - base < W - 1 ? last - base : W - 1);
    if (i0 != mi0 || i1 != mi1) {
      mi0 = i0; mi1 = i1; cmask = 0;
#pragma unroll
      for (int k = 0; k < 2 * NT; ++k) {
        const int i = 8 * (k >> 1) + 2 * tq + (k & 1);
        cmask |= (i >= i0 && i <= i1) ? 1u << k : 0u;
      }
    }
    const bool last_layer = l + 1 == a.n_layers;
    uint8_t* nb = buf_ptr(l + 1);
    if (run) {
      for (int mt = 0; mt < MT; ++mt) {
        // Q fragments: window rows L + 16 mt + (0..15), 4 k-steps of 16 dims
        uint32_t qa[4][4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          ldsm_x4(bu + (L + 16 * mt + (lane & 7) + 8 * ((lane >> 3) & 1)) * kMmaRowB + (16 * ks + 8 * (lane >> 4)) * 2, qa[ks]);
        float s[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
          uint32_t kb[8];
          const uint32_t ra = bu + (8 * nt + (lane & 7)) * kMmaRowB + 16 * (lane >> 3);
          ldsm_x4(ra, kb);
          ldsm_x4(ra + 64, kb + 4);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) mma16816(s[nt], qa[ks], kb + 2 * ks);
        }
        // row validity (LLSA: channel R - m's frame; SA: the query row only) and column mask
        uint32_t cm[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          const int m = 16 * mt + g + 8 * hr;
          const bool qv = SA ? m == 0 : (m <= R && h - (R - m) >= 0 && h - (R - m) <= last);
          cm[hr] = qv ? cmask : 0u;
        }
        // row softmax on the raw scores (a row lives in the 4 lanes of a quad); P unnormalised,
        // the 1 / sum is applied to O
        float mx[2] = {neg_inf(), neg_inf()}, inv[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float& v = s[nt][2 * hr + e];
              v = (cm[hr] >> (2 * nt + e)) & 1u ? v : neg_inf();
              mx[hr] = fmaxf(mx[hr], v);
            }
          mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
          mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
          const float mb = mx[hr] == neg_inf() ? 0.f : mx[hr] * a.scale_log2;
          float sum = 0.f;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float& v = s[nt][2 * hr + e];
              v = fast_ex2(fmaf(v, a.scale_log2, -mb));   // exp2(-inf) = 0 for masked entries
              sum += v;
            }
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          inv[hr] = sum > 0.f ? 1.f / sum : 0.f;
        }
        // O = P V over this warp's DT dim tiles: P re-packed from the accumulators as the A
        // operand, V by ldmatrix.trans
        float o[DT][4];
#pragma unroll
        for (int j = 0; j < DT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint32_t pa[4] = {bf2(s[2 * ks][0], s[2 * ks][1]), bf2(s[2 * ks][2], s[2 * ks][3]),
                                  bf2(s[2 * ks + 1][0], s[2 * ks + 1][1]), bf2(s[2 * ks + 1][2], s[2 * ks + 1][3])};
#pragma unroll
          for (int j = 0; j < DT; j += 2) {
            uint32_t vb[4];
            ldsm_x4_t(bu + (16 * ks + 8 * (lane >> 3 & 1) + (lane & 7)) * kMmaRowB + (8 * (DT * warp + j + (lane >> 4))) * 2, vb);
            mma16816(o[j], pa, vb);
            mma16816(o[j + 1], pa, vb + 2);
          }
        }
        // epilogue: X_{l+1} = bf16((X_l + bf16(O)) / 2) into the next window (or the output)
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          const int m = 16 * mt + g + 8 * hr;
          if (SA ? m != 0 : m > R) continue;
#pragma unroll
          for (int j = 0; j < DT; ++j) {
            const int d = 8 * (DT * warp + j) + 2 * tq;
            const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(bp + (L + m) * kMmaRowB + 2 * d));
            const float o0 = __bfloat162float(__float2bfloat16_rn(o[j][2 * hr] * inv[hr]));
            const float o1 = __bfloat162float(__float2bfloat16_rn(o[j][2 * hr + 1] * inv[hr]));
            const __nv_bfloat162 v = __floats2bfloat162_rn(0.5f * (x.x + o0), 0.5f * (x.y + o1));
            if (!last_layer) {
              *reinterpret_cast<__nv_bfloat162*>(nb + (SA ? W - 1 : L + m) * kMmaRowB + 2 * d) = v;
            } else if (m == 0 && a.y_out) {
              const long long te = SA ? base + L : h - R;
              if (te >= 0 && te <= last) *reinterpret_cast<__nv_bfloat162*>(a.y_out + (long long)bh * 64 + d) = v;
            }
          }
        }
      }
    }
    if (SA) cur_ok = run;
    // the next layer: its ring rows (issued NB - 2 layers ago) and this layer's outputs
    cp_async_wait_dyn(NB - 2);
    __syncthreads();
  }
  cp_async_wait<0>();
}

// geometry of the tensor-core step: window rows per buffer, number of buffers, shared memory
inline bool stream_mma_geometry(bool sa, int L, int R, int n_layers, int* nrw, int* nb, int* nt, size_t* smem) {
  const int W = L + R + 1, C = R + 1;
  const int wk = (W + 15) / 16 * 16;
  if (wk > 64 || (!sa && C > 32)) return false;
  const int mt = sa ? 1 : (C + 15) / 16;
  *nt = wk / 8;
  *nrw = wk > L + 16 * mt ? wk : L + 16 * mt;
  const size_t per = (size_t)*nrw * kMmaRowB;
  int b = n_layers < 6 ? n_layers : 6;
  if (b < 2) b = 2;
  while (b > 2 && per * b > 96 * 1024) --b;
  *nb = b;
  *smem = per * b;
  return *smem <= 200 * 1024;
}

}  // namespace sattn
