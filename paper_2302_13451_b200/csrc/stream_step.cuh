// stream_step.cuh — one incremental LLSA step (infer_llsa).
//
// One launch runs horizon h through every layer.  CTA = one (batch, head) stream.
// At horizon h each layer computes the R+1 outputs (h-c, c), c = 0..R, which all
// share one window ("the same keys and values of the red vector are used"):
//   slot i in [0, L]      (u = h-R-L+i, channel R): ring of the layer input (u < h-R)
//                                                    or the current diagonal (u = h-R)
//   slot i in [L+1, L+R]  (u = h-R-L+i, channel L+R-i): the current diagonal
// so a (R+1) x (L+R+1) attention per layer; tied Q = K = V = the layer input
// (reading G12), X_{l+1} = (X_l + O_l)/2 rounded exactly like the offline stack
// (O rounded to the storage type first, then the half-sum).  Layer 1's diagonal is
// the last R+1 raw frames (every channel of X_0 equals x).
#pragma once
#include "common.cuh"

namespace sattn {

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

// Latency structure: the layers of a step are sequential, so the step costs n_layers x (one
// layer's dependent phases).  Everything a layer reads that is known at launch — the ring rows
// of every layer (frames h-R-L .. h-R-1, written by earlier steps) and their slot indices — is
// fetched once, up front, in parallel; a layer then touches only shared memory, and writes its
// one new ring row back without waiting.
template <int D, typename T>
__global__ void __launch_bounds__(256) llsa_stream_step_kernel(StreamArgs a) {
  constexpr int SD = D + 1;
  extern __shared__ float sm[];
  const int C = a.R + 1, W = a.L + a.R + 1;
  const int L = a.L, R = a.R;
  float* win = sm;                    // [W][SD]
  float* diag = win + W * SD;         // [C][SD]
  float* ndiag = diag + C * SD;       // [C][SD]
  float* P = ndiag + C * SD;          // [C][W]
  int* slot = reinterpret_cast<int*>(P + C * W);   // [W] ring slot of window row i < L, -1 if invalid
  int* rslot = slot + W;                             // [C] raw slot of frame h - c', -1 if invalid
  T* rings = reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(rslot + C + 3) & ~uintptr_t(15));  // [n_layers][L][D]
  const int bh = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const long long h = a.h, last = a.last;
  T* raw = reinterpret_cast<T*>(a.raw) + (long long)bh * C * D;

  // slot indices (the only 64-bit modulo work of the step)
  for (int i = tid; i < W; i += nt) {
    const long long u = h - R - L + i;
    slot[i] = (i < L && u >= 0 && u <= last) ? (int)(u % L) : -1;
  }
  for (int cp = tid; cp < C; cp += nt) {
    const long long f = h - cp;
    rslot[cp] = (f >= 0 && f <= last) ? (int)(f % C) : -1;
  }
  // layer-1 diagonal: X_0(h - c', c') = x_{h - c'}
  if (a.x_new) {
    const T* x = reinterpret_cast<const T*>(a.x_new) + (long long)bh * D;
    const int sx = (int)(h % C);
    for (int d = tid; d < D; d += nt) raw[sx * D + d] = x[d];
  }
  __syncthreads();
  if (a.preload && L > 0) {
    // every layer's ring rows, in parallel (16-byte copies when rows are 16-byte multiples)
    constexpr bool VEC = (D * sizeof(T)) % 16 == 0;
    constexpr int PER = VEC ? (int)(D * sizeof(T) / 16) : D;   // chunks (or elements) per row
    const int n = a.n_layers * L * PER;
    for (int idx = tid; idx < n; idx += nt) {
      const int ch = idx % PER, i = (idx / PER) % L, l = idx / (PER * L);
      const int sl = slot[i];
      const T* src = reinterpret_cast<const T*>(a.ring) + (((long long)l * a.BH + bh) * L + (sl < 0 ? 0 : sl)) * D;
      T* dst = rings + ((long long)l * L + i) * D;
      if (VEC) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (sl >= 0) v = reinterpret_cast<const uint4*>(src)[ch];
        reinterpret_cast<uint4*>(dst)[ch] = v;
      } else {
        dst[ch] = sl >= 0 ? src[ch] : from_f<T>(0.f);
      }
    }
  }
  for (int idx = tid; idx < C * D; idx += nt) {
    const int cp = idx / D, d = idx % D;
    diag[cp * SD + d] = rslot[cp] >= 0 ? to_f(raw[rslot[cp] * D + d]) : 0.f;
  }
  __syncthreads();
  const int wslot = (h - R >= 0 && h - R <= last && L > 0) ? (int)((h - R) % L) : -1;

  for (int l = 0; l < a.n_layers; ++l) {
    T* ring = L > 0 ? reinterpret_cast<T*>(a.ring) + ((long long)l * a.BH + bh) * L * D : nullptr;
    const T* lring = rings + (long long)l * L * D;
    // window rows (tied K = V)
    for (int idx = tid; idx < W * D; idx += nt) {
      const int i = idx / D, d = idx % D;
      const long long u = h - R - L + i;
      float x = 0.f;
      if (u >= 0 && u <= last) {
        if (i < L) x = a.preload ? to_f(lring[i * D + d]) : to_f(ring[slot[i] * D + d]);
        else if (i == L) x = diag[R * SD + d];
        else x = diag[(L + R - i) * SD + d];
      }
      win[i * SD + d] = x;
    }
    __syncthreads();
    // scores (log2 domain), masked to -inf for invalid slots / queries
    for (int idx = tid; idx < C * W; idx += nt) {
      const int c = idx / W, i = idx % W;
      const long long u = h - R - L + i, t = h - c;
      float s = neg_inf();
      if (u >= 0 && u <= last && t >= 0 && t <= last) {
        // four independent partial sums: the dependent FMA chain was the step's longest latency
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 16
        for (int d = 0; d < D; ++d) acc[d & 3] = fmaf(diag[c * SD + d], win[i * SD + d], acc[d & 3]);
        s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * a.scale_log2;
      }
      P[c * W + i] = s;
    }
    __syncthreads();
    // softmax per query row: one warp per row
    const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
    for (int c = warp; c < C; c += nwarp) {
      float m = neg_inf();
      for (int i = lane; i < W; i += 32) m = fmaxf(m, P[c * W + i]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float sum = 0.f;
      for (int i = lane; i < W; i += 32) {
        const float e = m == neg_inf() ? 0.f : exp2f(P[c * W + i] - m);
        P[c * W + i] = e;
        sum += e;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float inv = sum > 0.f ? 1.f / sum : 0.f;
      for (int i = lane; i < W; i += 32) P[c * W + i] *= inv;
    }
    __syncthreads();
    // values, block rule, rounding as the offline stack stores them
    for (int idx = tid; idx < C * D; idx += nt) {
      const int c = idx / D, d = idx % D;
      float y4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int i = 0; i < W; ++i) y4[i & 3] = fmaf(P[c * W + i], win[i * SD + d], y4[i & 3]);
      const float y = (y4[0] + y4[1]) + (y4[2] + y4[3]);
      const float o = to_f(from_f<T>(y));
      ndiag[c * SD + d] = to_f(from_f<T>(0.5f * (diag[c * SD + d] + o)));
    }
    __syncthreads();
    // X_l(h-R, R) joins this layer's ring (after every read of the ring above)
    if (wslot >= 0)
      for (int d = tid; d < D; d += nt) ring[wslot * D + d] = from_f<T>(diag[R * SD + d]);
    for (int idx = tid; idx < C * D; idx += nt) diag[(idx / D) * SD + idx % D] = ndiag[(idx / D) * SD + idx % D];
    __syncthreads();
  }
  if (a.y_out && h - R >= 0 && h - R <= last) {
    T* y = reinterpret_cast<T*>(a.y_out) + (long long)bh * D;
    for (int d = tid; d < D; d += nt) y[d] = from_f<T>(diag[R * SD + d]);
  }
}

// shared memory of the step kernel: working set, plus (preload) every layer's ring rows
inline size_t stream_smem_bytes(int D, int L, int R, int n_layers = 0, size_t elem = 4) {
  const int C = R + 1, W = L + R + 1, SD = D + 1;
  const size_t base = sizeof(float) * ((size_t)W * SD + 2 * (size_t)C * SD + (size_t)C * W) + sizeof(int) * (W + C) + 32;
  return base + (size_t)n_layers * L * D * elem;
}

}  // namespace sattn

namespace sattn {

// ------------------------------------------------------------------------------------------
// One incremental SA step (infer_sa).  CTA = one (batch, head).
// After frame h arrives, layer l (0-based) computes its output at t_l = h - (l+1) R from the
// window [t_l - L, t_l + R] of its input; the newest window frame t_l + R = h - l R is the one
// the layer below produced in this same step (layer 0: x_h), the older ones come from the
// layer's ring of its last L + R + 1 input frames.  X_{l+1}(t_l) = (X_l(t_l) + Y_l(t_l)) / 2
// (G12), rounded like the offline stack; the stack emits X_n(h - n R): latency n R frames.
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
__global__ void __launch_bounds__(128) sa_stream_step_kernel(SAStreamArgs a) {
  constexpr int SD = D + 1;
  extern __shared__ float sm[];
  const int L = a.L, R = a.R, W = L + R + 1;
  float* win = sm;                   // [W][SD]
  float* cur = win + W * SD;         // [SD] newest input frame of the current layer
  float* P = cur + SD;               // [W]
  T* rings = reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(P + W + 3) & ~uintptr_t(15));   // [n][W-1][D]
  const int bh = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const long long h = a.h, last = a.last;
  const int NR = W;

  // newest input of layer 0: x_h
  bool cur_ok = a.x_new != nullptr && h <= last;
  if (cur_ok) {
    const T* x = reinterpret_cast<const T*>(a.x_new) + (long long)bh * D;
    for (int d = tid; d < D; d += nt) cur[d] = to_f(x[d]);
  }
  // ring slot of frame u = (h mod NR) + (u - h) mod NR: one 64-bit modulo per step, not per element
  const int hm = (int)(h % NR);
  auto slot_of = [&](long long u) { int sl = (hm + (int)((u - h) % NR)) % NR; return sl < 0 ? sl + NR : sl; };
  // stage every layer's ring rows: window rows i in [0, W-1) of layer l (frames t_l - L + i),
  // 16-byte copies when rows are 16-byte multiples
  if (a.preload) {
    constexpr bool VEC = (D * sizeof(T)) % 16 == 0;
    constexpr int PER = VEC ? (int)(D * sizeof(T) / 16) : D;
    const int n = a.n_layers * (W - 1) * PER;
    for (int idx = tid; idx < n; idx += nt) {
      const int ch = idx % PER, i = (idx / PER) % (W - 1), l = idx / (PER * (W - 1));
      const long long u = h - (long long)(l + 1) * R - L + i;
      const bool ok = u >= 0 && u <= last;
      const T* src = reinterpret_cast<const T*>(a.ring) + (((long long)l * a.BH + bh) * NR + (ok ? slot_of(u) : 0)) * D;
      T* dst = rings + ((long long)l * (W - 1) + i) * D;
      if (VEC) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ok) v = reinterpret_cast<const uint4*>(src)[ch];
        reinterpret_cast<uint4*>(dst)[ch] = v;
      } else {
        dst[ch] = ok ? src[ch] : from_f<T>(0.f);
      }
    }
  }
  __syncthreads();
  for (int l = 0; l < a.n_layers; ++l) {
    T* ring = reinterpret_cast<T*>(a.ring) + ((long long)l * a.BH + bh) * NR * D;
    const long long fn = h - (long long)l * R;          // this layer's newest input frame (= cur)
    const long long t = fn - R;                          // the frame it computes
    const bool run = t >= 0 && t <= last;
    if (run) {
      for (int idx = tid; idx < W * D; idx += nt) {
        const int i = idx / D, d = idx % D;
        const long long u = t - L + i;
        float x = 0.f;
        if (u >= 0 && u <= last) {
          if (i == W - 1) x = cur[d];                    // u = t + R = fn
          else x = a.preload ? to_f(rings[((long long)l * (W - 1) + i) * D + d]) : to_f(ring[slot_of(u) * D + d]);
        }
        win[i * SD + d] = x;
      }
    }
    __syncthreads();
    // the newest frame joins the ring (its slot held frame fn - W, outside every later window)
    if (cur_ok && fn >= 0) {
      const int sl = slot_of(fn);
      for (int d = tid; d < D; d += nt) ring[sl * D + d] = from_f<T>(cur[d]);
    }
    if (run) {
      // scores (log2 domain) of the query X_l(t) = window row L
      for (int i = tid; i < W; i += nt) {
        const long long u = t - L + i;
        float s = neg_inf();
        if (u >= 0 && u <= last) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 16
          for (int d = 0; d < D; ++d) acc[d & 3] = fmaf(win[L * SD + d], win[i * SD + d], acc[d & 3]);
          s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * a.scale_log2;
        }
        P[i] = s;
      }
      __syncthreads();
      if (tid < 32) {
        float m = neg_inf();
        for (int i = tid; i < W; i += 32) m = fmaxf(m, P[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float sum = 0.f;
        for (int i = tid; i < W; i += 32) {
          const float e = exp2f(P[i] - m);
          P[i] = e;
          sum += e;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const float inv = 1.f / sum;
        for (int i = tid; i < W; i += 32) P[i] *= inv;
      }
      __syncthreads();
      // value sum and the block rule; the result is the next layer's newest input frame
      for (int d = tid; d < D; d += nt) {
        float y4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < W; ++i) y4[i & 3] = fmaf(P[i], win[i * SD + d], y4[i & 3]);
        const float o = to_f(from_f<T>((y4[0] + y4[1]) + (y4[2] + y4[3])));
        cur[d] = to_f(from_f<T>(0.5f * (win[L * SD + d] + o)));
      }
    }
    cur_ok = run;
    __syncthreads();
  }
  const long long te = h - (long long)a.n_layers * R;
  if (a.y_out && cur_ok && te >= 0 && te <= last) {
    T* y = reinterpret_cast<T*>(a.y_out) + (long long)bh * D;
    for (int d = tid; d < D; d += nt) y[d] = from_f<T>(cur[d]);
  }
}

inline size_t sa_stream_smem_bytes(int D, int L, int R, int n_layers = 0, size_t elem = 4) {
  const int W = L + R + 1, SD = D + 1;
  return sizeof(float) * ((size_t)W * SD + SD + W) + 32 + (size_t)n_layers * (W - 1) * D * elem;
}

}  // namespace sattn
