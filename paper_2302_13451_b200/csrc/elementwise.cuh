// elementwise.cuh — the stack driver's frame-local block rule (reading G12) and its adjoint:
//   forward   X_{l+1} = (X_l + O_l) / 2            (X_0 broadcast over LLSA channels at l = 0)
//   backward  g = dX_{l+1}/2 + dQ + dK + dV ;  dX_l = g ; dO_{l-1} = g/2
//             and, at l = 0 for LLSA, dX_0 = sum_c g[c]  (adjoint of the duplication)
#pragma once
#include "common.cuh"

namespace sattn {

template <typename T>
__global__ void half_sum_kernel(T* __restrict__ out, const T* __restrict__ a, const T* __restrict__ b,
                                long long n, long long a_plane) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float x = to_f(a[a_plane ? i % a_plane : i]);
    out[i] = from_f<T>(0.5f * (x + to_f(b[i])));
  }
}

template <typename T>
__global__ void scale_kernel(T* __restrict__ out, const T* __restrict__ in, float s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = from_f<T>(s * to_f(in[i]));
}

template <typename T>
__global__ void combine_kernel(T* dX, T* dO_next, const T* dXin, const T* __restrict__ dQ,
                               const T* __restrict__ dK, const T* __restrict__ dV, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float g = 0.5f * to_f(dXin[i]) + to_f(dQ[i]) + to_f(dK[i]) + to_f(dV[i]);
    const T gt = from_f<T>(g);
    dX[i] = gt;
    if (dO_next) dO_next[i] = from_f<T>(0.5f * to_f(gt));
  }
}

template <typename T>
__global__ void combine_chsum_kernel(T* __restrict__ dX0, const T* __restrict__ dXin, const T* __restrict__ dQ,
                                     const T* __restrict__ dK, const T* __restrict__ dV, long long plane, int C) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < plane; i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < C; ++c) {
      const long long j = c * plane + i;
      s += 0.5f * to_f(dXin[j]) + to_f(dQ[j]) + to_f(dK[j]) + to_f(dV[j]);
    }
    dX0[i] = from_f<T>(s);
  }
}

}  // namespace sattn
