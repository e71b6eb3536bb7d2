// sattn_abi.cu — the C ABI of libsattn.so (include/sattn.h): validation, kernel-family
// dispatch, the layer-stack driver and the incremental-stream handle.
#include "sattn.h"

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "elementwise.cuh"
#include "ffma_attn.cuh"
#include "stream_step.cuh"
#include "tc_dispatch.h"
#include "host_util.h"

using namespace sattn;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

sattn_status fail(sattn_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return fail(SATTN_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

sattn_status after_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SATTN_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return SATTN_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t elem_size(int dtype) { return dtype == SATTN_BF16 ? 2 : 4; }

bool supported_D(int64_t D) { return D == 2 || D == 4 || D == 8 || D == 16 || D == 32 || D == 64; }

sattn_status validate(const sattn_desc* d) {
  if (!d) return fail(SATTN_EARG, "desc is NULL");
  if (d->B <= 0 || d->H <= 0 || d->T <= 0 || d->D <= 0)
    return fail(SATTN_EARG, "B,H,T,D must be positive (got %lld,%lld,%lld,%lld)", (long long)d->B,
                (long long)d->H, (long long)d->T, (long long)d->D);
  if (d->L < 0 || d->R < 0) return fail(SATTN_EARG, "L and R must be >= 0 (got %d,%d)", d->L, d->R);
  if (d->dtype != SATTN_F32 && d->dtype != SATTN_BF16) return fail(SATTN_EARG, "unknown dtype %d", d->dtype);
  if (d->impl < SATTN_IMPL_AUTO || d->impl > SATTN_IMPL_TC) return fail(SATTN_EARG, "unknown impl %d", d->impl);
  if (!supported_D(d->D)) return fail(SATTN_EUNSUPPORTED, "D=%lld not supported (2,4,8,16,32,64)", (long long)d->D);
  if (d->B * d->H > 65535) return fail(SATTN_EUNSUPPORTED, "B*H=%lld exceeds 65535", (long long)(d->B * d->H));
  if (d->T > (1LL << 30)) return fail(SATTN_EUNSUPPORTED, "T=%lld too large", (long long)d->T);
  if (d->R + 1 > 65535) return fail(SATTN_EUNSUPPORTED, "R too large");
  if (!(d->scale >= 0.f) || std::isinf(d->scale)) return fail(SATTN_EARG, "scale must be finite and >= 0");
  return SATTN_OK;
}

float eff_scale(const sattn_desc* d) { return d->scale > 0.f ? d->scale : 1.0f / std::sqrt((float)d->D); }

template <int D> using IntC = std::integral_constant<int, D>;

template <class Fn>
sattn_status dispatch(int64_t D, int dtype, bool llsa, Fn&& fn) {
  auto by_t = [&](auto dc) -> sattn_status {
    if (dtype == SATTN_F32)
      return llsa ? fn(dc, std::true_type{}, float{}) : fn(dc, std::false_type{}, float{});
    return llsa ? fn(dc, std::true_type{}, bf16{}) : fn(dc, std::false_type{}, bf16{});
  };
  switch (D) {
    case 2: return by_t(IntC<2>{});
    case 4: return by_t(IntC<4>{});
    case 8: return by_t(IntC<8>{});
    case 16: return by_t(IntC<16>{});
    case 32: return by_t(IntC<32>{});
    case 64: return by_t(IntC<64>{});
  }
  return fail(SATTN_EUNSUPPORTED, "D=%lld", (long long)D);
}

AttnArgs make_args(const sattn_desc* d, bool llsa) {
  AttnArgs a{};
  a.T = (int)d->T;
  a.L = d->L;
  a.R = llsa ? d->R : d->R;
  a.BH = (int)(d->B * d->H);
  a.scale = eff_scale(d);
  a.scale_log2 = a.scale * kLog2e;
  const long long plane = (long long)d->B * d->H * d->T * d->D;
  a.out_cs = plane;
  a.in_cs = (llsa && d->in_broadcast) ? 0 : plane;
  return a;
}


sattn_status ffma_forward(const sattn_desc* d, bool llsa, const AttnArgs& a, cudaStream_t st) {
  const int C = llsa ? d->R + 1 : 1;
  return dispatch(d->D, d->dtype, llsa, [&](auto dc, auto lc, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    constexpr bool LL = decltype(lc)::value;
    using T = decltype(tv);
    const size_t smem = fwd_smem_bytes<D>();
    set_smem(fwd_ffma<D, LL, T>, smem);
    dim3 grid((unsigned)((a.T + kQT - 1) / kQT), (unsigned)C, (unsigned)a.BH);
    fwd_ffma<D, LL, T><<<grid, 32 * kNW, smem, st>>>(a);
    return after_launch("fwd_ffma");
  });
}

sattn_status ffma_backward(const sattn_desc* d, bool llsa, const AttnArgs& a, cudaStream_t st) {
  const int C = llsa ? d->R + 1 : 1;
  return dispatch(d->D, d->dtype, llsa, [&](auto dc, auto lc, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    constexpr bool LL = decltype(lc)::value;
    using T = decltype(tv);
    dim3 grid((unsigned)((a.T + kQT - 1) / kQT), (unsigned)C, (unsigned)a.BH);
    const size_t s1 = fwd_smem_bytes<D>();
    set_smem(bwd_dq_ffma<D, LL, T>, s1);
    bwd_dq_ffma<D, LL, T><<<grid, 32 * kNW, s1, st>>>(a);
    sattn_status r = after_launch("bwd_dq_ffma");
    if (r != SATTN_OK) return r;
    const size_t s2 = dkdv_smem_bytes<D>();
    set_smem(bwd_dkdv_ffma<D, LL, T>, s2);
    bwd_dkdv_ffma<D, LL, T><<<grid, 32 * kNW, s2, st>>>(a);
    return after_launch("bwd_dkdv_ffma");
  });
}

// SA with the stored band (NEXT-4): the PST instances of the CUDA-core kernels
int64_t p_ld(const sattn_desc* d) { return ((int64_t)d->L + d->R + 1 + 7) & ~int64_t(7); }

sattn_status ffma_forward_p(const sattn_desc* d, const AttnArgs& a, cudaStream_t st) {
  return dispatch(d->D, d->dtype, false, [&](auto dc, auto, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    using T = decltype(tv);
    const size_t smem = fwd_smem_bytes<D>();
    set_smem(fwd_ffma<D, false, T, true>, smem);
    dim3 grid((unsigned)((a.T + kQT - 1) / kQT), 1u, (unsigned)a.BH);
    fwd_ffma<D, false, T, true><<<grid, 32 * kNW, smem, st>>>(a);
    return after_launch("fwd_ffma_p");
  });
}

sattn_status ffma_backward_p(const sattn_desc* d, const AttnArgs& a, cudaStream_t st) {
  return dispatch(d->D, d->dtype, false, [&](auto dc, auto, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    using T = decltype(tv);
    dim3 grid((unsigned)((a.T + kQT - 1) / kQT), 1u, (unsigned)a.BH);
    const size_t s1 = fwd_smem_bytes<D>();
    set_smem(bwd_dq_ffma<D, false, T, true>, s1);
    bwd_dq_ffma<D, false, T, true><<<grid, 32 * kNW, s1, st>>>(a);
    sattn_status r = after_launch("bwd_dq_ffma_p");
    if (r != SATTN_OK) return r;
    const size_t s2 = dkdv_smem_bytes<D>();
    set_smem(bwd_dkdv_ffma<D, false, T, true>, s2);
    bwd_dkdv_ffma<D, false, T, true><<<grid, 32 * kNW, s2, st>>>(a);
    return after_launch("bwd_dkdv_ffma_p");
  });
}

bool tc_ok(const sattn_desc* d, bool llsa, bool backward) {
  if (llsa)
    return backward ? tc_llsa_bwd_any_supported(d->dtype, (int)d->D, d->L, d->R, d->B * d->H, d->T, !d->in_broadcast)
                    : tc_llsa_fwd_any_supported(d->dtype, (int)d->D, d->L, d->R, d->B * d->H, d->T, !d->in_broadcast);
  return tc_supported(d->dtype, (int)d->D, d->L, d->R, false, backward);
}

bool use_tc(const sattn_desc* d, bool llsa, bool backward) {
  if (d->impl == SATTN_IMPL_FFMA) return false;
  return tc_ok(d, llsa, backward);
}

sattn_status attn_forward(const sattn_desc* d, bool llsa, const void* Q, const void* K, const void* V, void* O,
                          float* LSE, cudaStream_t st) {
  if (!Q || !K || !V || !O || !LSE) return fail(SATTN_EARG, "NULL tensor pointer");
  if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O) || !aligned16(LSE))
    return fail(SATTN_EARG, "tensor pointers must be 16-byte aligned");
  if (d->impl == SATTN_IMPL_TC && !tc_ok(d, llsa, false))
    return fail(SATTN_EUNSUPPORTED, llsa ? "tensor-core LLSA forward needs bf16, D=64, R <= 8 (4 <= R, L <= 32 for broadcast inputs)"
                                         : "tensor-core SA forward needs bf16, D=64, L+R+1 <= 65");
  AttnArgs a = make_args(d, llsa);
  a.Q = Q; a.K = K; a.V = V; a.Out = O; a.LSEout = LSE;
  if (use_tc(d, llsa, false)) {
    sattn_status r = llsa ? tc_llsa_forward(a, st) : tc_forward(a, st);
    if (r != SATTN_OK) return fail(r, "tc_forward: %s", llsa ? tc_llsa_last_error() : tc_last_error());
    return after_launch(llsa ? "tc_llsa_forward" : "tc_forward");
  }
  return ffma_forward(d, llsa, a, st);
}

bool wide_tc(const sattn_desc* d, bool llsa) {
  return !llsa && d->impl != SATTN_IMPL_FFMA && tc_wide_supported(d->dtype, (int)d->D, d->L, d->R);
}

size_t attn_bwd_ws(const sattn_desc* d, bool llsa) {
  // delta and LSE*log2(e) (+ for LLSA the staircase part of delta), fp32, per channel, rows
  // padded to a multiple of 4 frames (16-byte TMA rows); wide SA bands on tensor cores: + the
  // fp32 dQ / dK / dV accumulators of the sub-band launches
  const size_t C = llsa ? d->R + 1 : 1;
  const size_t Tp = (size_t)((d->T + 3) & ~3LL);
  const size_t rows = (llsa ? 3 : 2) * C * d->B * d->H * Tp * sizeof(float);
  if (wide_tc(d, llsa)) {
    const size_t w = tc_wide_bwd_ws(d->B * d->H, d->T);
    return w > rows ? w : rows;
  }
  return rows;
}

sattn_status attn_backward(const sattn_desc* d, bool llsa, const void* Q, const void* K, const void* V,
                           const void* O, const float* LSE, const void* dO, void* dQ, void* dK, void* dV, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
  if (!Q || !K || !V || !O || !LSE || !dO || !dQ || !dK || !dV || !ws) return fail(SATTN_EARG, "NULL pointer");
  const void* ps[] = {Q, K, V, O, LSE, dO, dQ, dK, dV, ws};
  for (const void* p : ps)
    if (!aligned16(p)) return fail(SATTN_EARG, "pointers must be 16-byte aligned");
  if (ws_bytes < attn_bwd_ws(d, llsa))
    return fail(SATTN_ECONFIG, "workspace %zu < required %zu bytes", ws_bytes, attn_bwd_ws(d, llsa));
  if (d->impl == SATTN_IMPL_TC && !tc_ok(d, llsa, true) && !wide_tc(d, llsa))
    return fail(SATTN_EUNSUPPORTED, llsa ? "tensor-core LLSA backward needs bf16, D=64, L <= 48 and 1 <= R <= 8 (R <= 16 for dense inputs)"
                                         : "tensor-core SA backward needs bf16, D=64, L+R+1 <= 65");
  AttnArgs a = make_args(d, llsa);
  a.Q = Q; a.K = K; a.V = V; a.O = O; a.LSE = LSE; a.dO = dO;
  a.dQ = dQ; a.dK = dK; a.dV = dV; a.delta = static_cast<float*>(ws);
  if (wide_tc(d, llsa)) {
    sattn_status r = tc_backward_wide(a, st);
    if (r != SATTN_OK) return fail(r, "tc_backward_wide: %s", tc_last_error());
    g_launches.fetch_add(4 + 2 * tc_wide_parts(d->L, d->R), std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SATTN_ECUDA, "tc_backward_wide launch: %s", cudaGetErrorString(e));
    return SATTN_OK;
  }
  if (use_tc(d, llsa, true)) {
    sattn_status r = llsa ? tc_llsa_backward(a, st) : tc_backward(a, st);
    if (r != SATTN_OK) return fail(r, "tc_backward: %s", tc_last_error());
    g_launches.fetch_add(llsa ? tc_llsa_backward_launches(a) : tc_backward_launches(), std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SATTN_ECUDA, "tc_backward launch: %s", cudaGetErrorString(e));
    return SATTN_OK;
  }
  return ffma_backward(d, llsa, a, st);
}

template <class T>
sattn_status launch_half_sum(void* out, const void* a, const void* b, long long n, long long a_plane, cudaStream_t st) {
  half_sum_kernel<T><<<1184, 256, 0, st>>>((T*)out, (const T*)a, (const T*)b, n, a_plane);
  return after_launch("half_sum");
}
template <class T>
sattn_status launch_scale(void* out, const void* in, float s, long long n, cudaStream_t st) {
  scale_kernel<T><<<1184, 256, 0, st>>>((T*)out, (const T*)in, s, n);
  return after_launch("scale");
}
template <class T>
sattn_status launch_combine(void* dX, void* dOn, const void* dXin, const void* dQ, const void* dK, const void* dV,
                            long long n, cudaStream_t st) {
  combine_kernel<T><<<1184, 256, 0, st>>>((T*)dX, (T*)dOn, (const T*)dXin, (const T*)dQ, (const T*)dK, (const T*)dV, n);
  return after_launch("combine");
}
template <class T>
sattn_status launch_chsum(void* dX0, const void* dXin, const void* dQ, const void* dK, const void* dV, long long plane,
                          int C, cudaStream_t st) {
  combine_chsum_kernel<T><<<1184, 256, 0, st>>>((T*)dX0, (const T*)dXin, (const T*)dQ, (const T*)dK, (const T*)dV,
                                                plane, C);
  return after_launch("combine_chsum");
}

#define BY_DTYPE(dt, call_f32, call_bf16) ((dt) == SATTN_F32 ? (call_f32) : (call_bf16))

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct StackLayout {
  size_t x0, xl, o, lse, total;  // sizes
  size_t off_x(int l) const { return l == 0 ? 0 : align256(x0) + (size_t)(l - 1) * align256(xl); }
  int n;
  size_t off_o(int l) const { return align256(x0) + (size_t)(n - 1) * align256(xl) + (size_t)l * (align256(o) + align256(lse)); }
  size_t off_lse(int l) const { return off_o(l) + align256(o); }
};

StackLayout stack_layout(const sattn_desc* d, int mode, int n) {
  StackLayout s{};
  const size_t C = mode == SATTN_MODE_LLSA ? d->R + 1 : 1;
  const size_t plane = (size_t)d->B * d->H * d->T * d->D;
  s.n = n;
  s.x0 = plane * elem_size(d->dtype);
  s.xl = C * plane * elem_size(d->dtype);
  s.o = s.xl;
  s.lse = C * d->B * d->H * d->T * sizeof(float);
  s.total = align256(s.x0) + (size_t)(n - 1) * align256(s.xl) + (size_t)n * (align256(s.o) + align256(s.lse));
  return s;
}

}  // namespace

// internal hooks for the other translation units (tshard.cu); declared in internal.h
namespace sattn {
sattn_status set_error(sattn_status st, const char* msg) { return fail(st, "%s", msg); }
sattn_status check_desc(const sattn_desc* d) { return validate(d); }
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
float desc_scale(const sattn_desc* d) { return eff_scale(d); }
}  // namespace sattn

extern "C" {

const char* sattn_last_error(void) { return g_err.c_str(); }
const char* sattn_version(void) { return "sattn 0.1 (sm_100a)"; }
int64_t sattn_launch_count(void) { return g_launches.load(); }
// internal debug hook (not in sattn.h): device buffer of 8 x 64 int64 clock64 stamps of CTA 0
void sattn_debug_trace(void* dev_buf) { tc_set_trace(dev_buf); tc_llsa_set_trace(dev_buf); }

sattn_status sa_forward(const sattn_desc* d, const void* Q, const void* K, const void* V, void* O, float* LSE,
                        void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  return attn_forward(d, false, Q, K, V, O, LSE, (cudaStream_t)stream);
}

size_t sa_backward_workspace(const sattn_desc* d) { return validate(d) == SATTN_OK ? attn_bwd_ws(d, false) : 0; }

size_t sa_forward_workspace(const sattn_desc* d) {
  if (validate(d) != SATTN_OK) return 0;
  return wide_tc(d, false) ? tc_wide_fwd_ws(d->B * d->H, d->T) : 0;
}

sattn_status sa_forward_ws(const sattn_desc* d, const void* Q, const void* K, const void* V, void* O, float* LSE,
                           void* ws, size_t ws_bytes, void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  if (!wide_tc(d, false)) return attn_forward(d, false, Q, K, V, O, LSE, (cudaStream_t)stream);
  if (!Q || !K || !V || !O || !LSE || !ws) return fail(SATTN_EARG, "NULL pointer");
  const void* ps[] = {Q, K, V, O, LSE, ws};
  for (const void* p : ps)
    if (!aligned16(p)) return fail(SATTN_EARG, "pointers must be 16-byte aligned");
  if (ws_bytes < sa_forward_workspace(d))
    return fail(SATTN_ECONFIG, "workspace %zu < required %zu bytes", ws_bytes, sa_forward_workspace(d));
  AttnArgs a = make_args(d, false);
  a.Q = Q; a.K = K; a.V = V; a.Out = O; a.LSEout = LSE;
  r = tc_forward_wide(a, ws, (cudaStream_t)stream);
  if (r != SATTN_OK) return fail(r, "tc_forward_wide: %s", tc_last_error());
  g_launches.fetch_add(1 + tc_wide_parts(d->L, d->R), std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SATTN_ECUDA, "tc_forward_wide launch: %s", cudaGetErrorString(e));
  return SATTN_OK;
}

sattn_status sa_backward(const sattn_desc* d, const void* Q, const void* K, const void* V, const void* O,
                         const float* LSE, const void* dO, void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes,
                         void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  return attn_backward(d, false, Q, K, V, O, LSE, dO, dQ, dK, dV, ws, ws_bytes, (cudaStream_t)stream);
}

sattn_status llsa_forward(const sattn_desc* d, const void* Q, const void* K, const void* V, void* O, float* LSE,
                          void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  return attn_forward(d, true, Q, K, V, O, LSE, (cudaStream_t)stream);
}

size_t llsa_backward_workspace(const sattn_desc* d) { return validate(d) == SATTN_OK ? attn_bwd_ws(d, true) : 0; }

sattn_status llsa_backward(const sattn_desc* d, const void* Q, const void* K, const void* V, const void* O,
                           const float* LSE, const void* dO, void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes,
                           void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  return attn_backward(d, true, Q, K, V, O, LSE, dO, dQ, dK, dV, ws, ws_bytes, (cudaStream_t)stream);
}

int64_t sa_p_ld(const sattn_desc* d) { return validate(d) == SATTN_OK ? p_ld(d) : 0; }

sattn_status sa_forward_p(const sattn_desc* d, const void* Q, const void* K, const void* V, void* O, float* LSE,
                          void* P, void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !LSE || !P) return fail(SATTN_EARG, "NULL tensor pointer");
  if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O) || !aligned16(LSE) || !aligned16(P))
    return fail(SATTN_EARG, "tensor pointers must be 16-byte aligned");
  const bool tc = d->impl != SATTN_IMPL_FFMA && tc_p_supported(d->dtype, (int)d->D, d->L, d->R, false);
  if (d->impl == SATTN_IMPL_TC && !tc)
    return fail(SATTN_EUNSUPPORTED, "tensor-core stored-band forward needs bf16, D=64, L+R+1 <= 64");
  AttnArgs a = make_args(d, false);
  a.Q = Q; a.K = K; a.V = V; a.Out = O; a.LSEout = LSE; a.P = P; a.ldp = (int)p_ld(d);
  if (tc) {
    r = tc_forward_p(a, (cudaStream_t)stream);
    if (r != SATTN_OK) return fail(r, "tc_forward_p: %s", tc_last_error());
    return after_launch("tc_forward_p");
  }
  return ffma_forward_p(d, a, (cudaStream_t)stream);
}

// the stored-band backward of a band too wide for one tensor-core pass (W > 49) runs as sub-bands
bool p_bwd_wide(const sattn_desc* d) {
  const int W = d->L + d->R + 1;
  return d->impl != SATTN_IMPL_FFMA && d->dtype == SATTN_BF16 && d->D == 64 &&
         !tc_p_supported(d->dtype, (int)d->D, d->L, d->R, true) && W > 49 && W <= 4096;
}

size_t sa_backward_p_workspace(const sattn_desc* d) {
  if (validate(d) != SATTN_OK) return 0;
  const size_t n = (size_t)d->B * d->H * ((d->T + 3) & ~3LL) * sizeof(float);
  if (!p_bwd_wide(d)) return n;
  const size_t w = tc_wide_bwd_ws(d->B * d->H, d->T);   // delta rows + fp32 dQ, dK, dV accumulators
  return w > n ? w : n;
}

sattn_status sa_backward_p(const sattn_desc* d, const void* Q, const void* K, const void* V, const void* O,
                           const void* P, const void* dO, void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes,
                           void* stream) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !P || !dO || !dQ || !dK || !dV || !ws) return fail(SATTN_EARG, "NULL pointer");
  const void* ps[] = {Q, K, V, O, P, dO, dQ, dK, dV, ws};
  for (const void* p : ps)
    if (!aligned16(p)) return fail(SATTN_EARG, "pointers must be 16-byte aligned");
  if (ws_bytes < sa_backward_p_workspace(d))
    return fail(SATTN_ECONFIG, "workspace %zu < required %zu bytes", ws_bytes, sa_backward_p_workspace(d));
  const bool tc = d->impl != SATTN_IMPL_FFMA && tc_p_supported(d->dtype, (int)d->D, d->L, d->R, true);
  const bool wide = p_bwd_wide(d);
  if (d->impl == SATTN_IMPL_TC && !tc && !wide)
    return fail(SATTN_EUNSUPPORTED, "tensor-core stored-band backward needs bf16, D=64, L+R+1 <= 4096");
  AttnArgs a = make_args(d, false);
  a.Q = Q; a.K = K; a.V = V; a.O = O; a.dO = dO; a.P = const_cast<void*>(P); a.ldp = (int)p_ld(d);
  a.dQ = dQ; a.dK = dK; a.dV = dV; a.delta = static_cast<float*>(ws);
  if (wide) {
    r = tc_backward_p_wide(a, (cudaStream_t)stream);
    if (r != SATTN_OK) return fail(r, "tc_backward_p_wide: %s", tc_last_error());
    g_launches.fetch_add(1 + 2 * tc_wide_p_parts(d->L, d->R) + 3, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SATTN_ECUDA, "tc_backward_p_wide launch: %s", cudaGetErrorString(e));
    return SATTN_OK;
  }
  if (tc) {
    r = tc_backward_p(a, (cudaStream_t)stream);
    if (r != SATTN_OK) return fail(r, "tc_backward_p: %s", tc_last_error());
    g_launches.fetch_add(2, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SATTN_ECUDA, "tc_backward_p launch: %s", cudaGetErrorString(e));
    return SATTN_OK;
  }
  return ffma_backward_p(d, a, (cudaStream_t)stream);
}

sattn_status sattn_stack_saved_offsets(const sattn_desc* d, int mode, int n_layers, int layer, int64_t* out3) {
  sattn_status r = validate(d);
  if (r != SATTN_OK) return r;
  if (!out3) return fail(SATTN_EARG, "out is NULL");
  if (n_layers < 1 || layer < 0 || layer >= n_layers || (mode != SATTN_MODE_SA && mode != SATTN_MODE_LLSA))
    return fail(SATTN_EARG, "bad mode / n_layers / layer");
  const StackLayout s = stack_layout(d, mode, n_layers);
  out3[0] = (int64_t)s.off_x(layer);
  out3[1] = (int64_t)s.off_o(layer);
  out3[2] = (int64_t)s.off_lse(layer);
  return SATTN_OK;
}

size_t sattn_stack_saved_bytes(const sattn_desc* d, int mode, int n_layers) {
  if (validate(d) != SATTN_OK || n_layers < 1 || (mode != SATTN_MODE_SA && mode != SATTN_MODE_LLSA)) return 0;
  return stack_layout(d, mode, n_layers).total;
}

sattn_status sattn_stack_forward(const sattn_desc* din, int mode, int n, const void* X0, void* saved,
                                 size_t saved_bytes, void* Y, void* stream) {
  sattn_status r = validate(din);
  if (r != SATTN_OK) return r;
  if (mode != SATTN_MODE_SA && mode != SATTN_MODE_LLSA) return fail(SATTN_EARG, "unknown mode %d", mode);
  if (n < 1) return fail(SATTN_EARG, "n_layers must be >= 1");
  if (!X0 || !saved || !Y) return fail(SATTN_EARG, "NULL pointer");
  if (!aligned16(X0) || !aligned16(saved) || !aligned16(Y)) return fail(SATTN_EARG, "pointers must be 16-byte aligned");
  StackLayout s = stack_layout(din, mode, n);
  if (saved_bytes < s.total) return fail(SATTN_ECONFIG, "saved buffer %zu < required %zu", saved_bytes, s.total);
  cudaStream_t st = (cudaStream_t)stream;
  const bool llsa = mode == SATTN_MODE_LLSA;
  const int C = llsa ? din->R + 1 : 1;
  const long long plane = din->B * din->H * din->T * din->D;
  char* base = static_cast<char*>(saved);
  CUDA_TRY(cudaMemcpyAsync(base + s.off_x(0), X0, s.x0, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < n; ++l) {
    sattn_desc d = *din;
    d.in_broadcast = (llsa && l == 0) ? 1 : 0;
    const void* X = base + s.off_x(l);
    void* O = base + s.off_o(l);
    float* LSE = reinterpret_cast<float*>(base + s.off_lse(l));
    r = attn_forward(&d, llsa, X, X, X, O, LSE, st);
    if (r != SATTN_OK) return r;
    void* Xn = (l == n - 1) ? Y : (void*)(base + s.off_x(l + 1));
    const long long a_plane = (llsa && l == 0) ? plane : 0;
    r = BY_DTYPE(d.dtype, launch_half_sum<float>(Xn, X, O, C * plane, a_plane, st),
                 launch_half_sum<bf16>(Xn, X, O, C * plane, a_plane, st));
    if (r != SATTN_OK) return r;
  }
  return SATTN_OK;
}

size_t sattn_stack_workspace(const sattn_desc* d, int mode, int n_layers) {
  if (validate(d) != SATTN_OK || n_layers < 1) return 0;
  const size_t C = mode == SATTN_MODE_LLSA ? d->R + 1 : 1;
  const size_t t = align256(C * d->B * d->H * d->T * d->D * elem_size(d->dtype));
  return 5 * t + align256(attn_bwd_ws(d, mode == SATTN_MODE_LLSA));
}

sattn_status sattn_stack_backward(const sattn_desc* din, int mode, int n, const void* saved, const void* dY,
                                  void* dX0, void* ws, size_t ws_bytes, void* stream) {
  sattn_status r = validate(din);
  if (r != SATTN_OK) return r;
  if (mode != SATTN_MODE_SA && mode != SATTN_MODE_LLSA) return fail(SATTN_EARG, "unknown mode %d", mode);
  if (n < 1) return fail(SATTN_EARG, "n_layers must be >= 1");
  if (!saved || !dY || !dX0 || !ws) return fail(SATTN_EARG, "NULL pointer");
  if (!aligned16(saved) || !aligned16(dY) || !aligned16(dX0) || !aligned16(ws))
    return fail(SATTN_EARG, "pointers must be 16-byte aligned");
  if (ws_bytes < sattn_stack_workspace(din, mode, n)) return fail(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const bool llsa = mode == SATTN_MODE_LLSA;
  const int C = llsa ? din->R + 1 : 1;
  const long long plane = din->B * din->H * din->T * din->D;
  const long long nel = C * plane;
  StackLayout s = stack_layout(din, mode, n);
  const char* base = static_cast<const char*>(saved);
  const size_t tb = align256(nel * elem_size(din->dtype));
  char* w = static_cast<char*>(ws);
  void* dX = w;
  void* dO = w + tb;
  void* dQ = w + 2 * tb;
  void* dK = w + 3 * tb;
  void* dV = w + 4 * tb;
  void* aws = w + 5 * tb;
  const int dt = din->dtype;
  r = BY_DTYPE(dt, launch_scale<float>(dO, dY, 0.5f, nel, st), launch_scale<bf16>(dO, dY, 0.5f, nel, st));
  if (r != SATTN_OK) return r;
  const void* dXin = dY;
  for (int l = n - 1; l >= 0; --l) {
    sattn_desc d = *din;
    d.in_broadcast = (llsa && l == 0) ? 1 : 0;
    const void* X = base + s.off_x(l);
    const void* O = base + s.off_o(l);
    const float* LSE = reinterpret_cast<const float*>(base + s.off_lse(l));
    r = attn_backward(&d, llsa, X, X, X, O, LSE, dO, dQ, dK, dV, aws, attn_bwd_ws(&d, llsa), st);
    if (r != SATTN_OK) return r;
    if (l > 0) {
      r = BY_DTYPE(dt, launch_combine<float>(dX, dO, dXin, dQ, dK, dV, nel, st),
                   launch_combine<bf16>(dX, dO, dXin, dQ, dK, dV, nel, st));
      dXin = dX;
    } else if (llsa) {
      r = BY_DTYPE(dt, launch_chsum<float>(dX0, dXin, dQ, dK, dV, plane, C, st),
                   launch_chsum<bf16>(dX0, dXin, dQ, dK, dV, plane, C, st));
    } else {
      r = BY_DTYPE(dt, launch_combine<float>(dX0, nullptr, dXin, dQ, dK, dV, nel, st),
                   launch_combine<bf16>(dX0, nullptr, dXin, dQ, dK, dV, nel, st));
    }
    if (r != SATTN_OK) return r;
  }
  return SATTN_OK;
}

// ------------------------------------------------------------------------------------------
// incremental stream
// ------------------------------------------------------------------------------------------
}  // extern "C"

struct sattn_stream {
  sattn_desc d;
  int n_layers;
  long long h, n_in;
  bool closed;
  void* raw;
  void* ring;
  int mode;          // SATTN_MODE_LLSA (llsa_stream_*) or SATTN_MODE_SA (sa_stream_*)
};

namespace {
// the tensor-core step (bf16, D = 64, window <= 64 rows): one warp per (batch, head)
sattn_status stream_mma_launch(sattn_stream* s, bool sa, const void* x, void* y, long long h, long long last,
                               cudaStream_t st, bool* launched) {
  *launched = false;
  int nrw = 0, nb = 0, nt = 0;
  size_t smem = 0;
  if (s->d.dtype != SATTN_BF16 || s->d.D != 64 ||
      !stream_mma_geometry(sa, s->d.L, s->d.R, s->n_layers, &nrw, &nb, &nt, &smem))
    return SATTN_OK;
  StreamMmaArgs a{};
  a.x_new = static_cast<const bf16*>(x);
  a.raw = static_cast<bf16*>(s->raw);
  a.ring = static_cast<bf16*>(s->ring);
  a.y_out = static_cast<bf16*>(y);
  a.h = h;
  a.last = last;
  a.n_layers = s->n_layers;
  a.L = s->d.L;
  a.R = s->d.R;
  a.BH = (int)(s->d.B * s->d.H);
  a.nrw = nrw;
  a.nb = nb;
  a.scale_log2 = eff_scale(&s->d) * kLog2e;
  auto go = [&](auto kern) -> sattn_status {
    set_smem(kern, smem);
    kern<<<a.BH, 32 * kMmaWarps, smem, st>>>(a);
    *launched = true;
    return after_launch(sa ? "sa_stream_mma" : "llsa_stream_mma");
  };
  switch (nt) {
    case 2: return sa ? go(stream_mma_kernel<true, 2>) : go(stream_mma_kernel<false, 2>);
    case 4: return sa ? go(stream_mma_kernel<true, 4>) : go(stream_mma_kernel<false, 4>);
    case 6: return sa ? go(stream_mma_kernel<true, 6>) : go(stream_mma_kernel<false, 6>);
    case 8: return sa ? go(stream_mma_kernel<true, 8>) : go(stream_mma_kernel<false, 8>);
  }
  return SATTN_OK;
}

sattn_status stream_launch(sattn_stream* s, const void* x, void* y, long long h, long long last, cudaStream_t st) {
  bool done = false;
  sattn_status r = stream_mma_launch(s, false, x, y, h, last, st, &done);
  if (r != SATTN_OK || done) return r;
  StreamArgs a{};
  a.x_new = x;
  a.raw = s->raw;
  a.ring = s->ring;
  a.y_out = y;
  a.h = h;
  a.last = last;
  a.n_layers = s->n_layers;
  a.L = s->d.L;
  a.R = s->d.R;
  a.BH = (int)(s->d.B * s->d.H);
  a.scale_log2 = eff_scale(&s->d) * kLog2e;
  return dispatch(s->d.D, s->d.dtype, false, [&](auto dc, auto, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    using T = decltype(tv);
    size_t smem = stream_smem_bytes<D, T>(a.L, a.R, a.n_layers);
    a.preload = 1;
    if (smem > 160 * 1024) {   // rings too large to stage at once: each layer stages its own rows
      a.preload = 0;
      smem = stream_smem_bytes<D, T>(a.L, a.R, 1);
    }
    if (smem > 200 * 1024) return fail(SATTN_EUNSUPPORTED, "stream window too large for shared memory");
    set_smem(llsa_stream_step_kernel<D, T>, smem);
    llsa_stream_step_kernel<D, T><<<a.BH, 32 * stream_warps(a.R), smem, st>>>(a);
    return after_launch("llsa_stream_step");
  });
}
sattn_status sa_stream_launch(sattn_stream* s, const void* x, void* y, long long h, long long last, cudaStream_t st) {
  bool done = false;
  sattn_status r = stream_mma_launch(s, true, x, y, h, last, st, &done);
  if (r != SATTN_OK || done) return r;
  SAStreamArgs a{};
  a.x_new = x;
  a.ring = s->ring;
  a.y_out = y;
  a.h = h;
  a.last = last;
  a.n_layers = s->n_layers;
  a.L = s->d.L;
  a.R = s->d.R;
  a.BH = (int)(s->d.B * s->d.H);
  a.scale_log2 = eff_scale(&s->d) * kLog2e;
  return dispatch(s->d.D, s->d.dtype, false, [&](auto dc, auto, auto tv) -> sattn_status {
    constexpr int D = decltype(dc)::value;
    using T = decltype(tv);
    size_t smem = sa_stream_smem_bytes<D, T>(a.L, a.R, a.n_layers);
    a.preload = 1;
    if (smem > 160 * 1024) {
      a.preload = 0;
      smem = sa_stream_smem_bytes<D, T>(a.L, a.R, 1);
    }
    if (smem > 200 * 1024) return fail(SATTN_EUNSUPPORTED, "stream window too large for shared memory");
    set_smem(sa_stream_step_kernel<D, T>, smem);
    sa_stream_step_kernel<D, T><<<a.BH, kSAStreamThreads, smem, st>>>(a);
    return after_launch("sa_stream_step");
  });
}
}  // namespace

extern "C" {

sattn_status sa_stream_create(const sattn_desc* d, int n_layers, sattn_stream** out) {
  if (!out) return fail(SATTN_EARG, "out is NULL");
  *out = nullptr;
  if (!d) return fail(SATTN_EARG, "desc is NULL");
  sattn_desc dd = *d;
  dd.T = 1;
  sattn_status r = validate(&dd);
  if (r != SATTN_OK) return r;
  if (n_layers < 1) return fail(SATTN_EARG, "n_layers must be >= 1");
  sattn_stream* s = new (std::nothrow) sattn_stream{};
  if (!s) return fail(SATTN_ECUDA, "out of host memory");
  s->d = dd;
  s->n_layers = n_layers;
  s->mode = SATTN_MODE_SA;
  const size_t ring_b = (size_t)n_layers * d->B * d->H * (d->L + d->R + 1) * d->D * elem_size(d->dtype);
  cudaError_t e = cudaMalloc(&s->ring, ring_b);
  if (e == cudaSuccess) e = cudaMemset(s->ring, 0, ring_b);
  if (e != cudaSuccess) {
    cudaFree(s->ring);
    delete s;
    return fail(SATTN_ECUDA, "stream state allocation: %s", cudaGetErrorString(e));
  }
  *out = s;
  return SATTN_OK;
}

sattn_status sa_stream_step(sattn_stream* s, const void* x_new, void* y_out, int64_t* out_frame, void* stream) {
  if (!s || !x_new || !y_out) return fail(SATTN_EARG, "NULL pointer");
  if (s->mode != SATTN_MODE_SA) return fail(SATTN_EARG, "not an SA stream handle");
  if (s->closed) return fail(SATTN_ESTATE, "stream already flushed (call sa_stream_reset)");
  const long long h = s->h, lat = (long long)s->n_layers * s->d.R;
  sattn_status r = sa_stream_launch(s, x_new, y_out, h, h, (cudaStream_t)stream);
  if (r != SATTN_OK) return r;
  s->h = h + 1;
  s->n_in = h + 1;
  if (out_frame) *out_frame = h >= lat ? h - lat : -1;
  return SATTN_OK;
}

sattn_status sa_stream_flush(sattn_stream* s, void* y_tail, int32_t* n_out, void* stream) {
  if (!s || !y_tail) return fail(SATTN_EARG, "NULL pointer");
  if (s->mode != SATTN_MODE_SA) return fail(SATTN_EARG, "not an SA stream handle");
  if (s->closed) return fail(SATTN_ESTATE, "stream already flushed");
  s->closed = true;
  const long long T = s->n_in, lat = (long long)s->n_layers * s->d.R;
  const size_t frame_b = s->d.B * s->d.H * s->d.D * elem_size(s->d.dtype);
  int cnt = 0;
  // every step h in [T, T + lat) runs: layers 0..n-2 still compute frames h - (l+1)R for the next
  // layer's ring even when the last layer has nothing to emit yet (h < lat, a stream shorter
  // than the stack's latency); only steps with h >= lat write an output frame
  for (long long h = T; h < T + lat; ++h) {
    const bool emit = h - lat >= 0;
    sattn_status r = sa_stream_launch(s, nullptr, emit ? static_cast<char*>(y_tail) + cnt * frame_b : nullptr, h,
                                      T - 1, (cudaStream_t)stream);
    if (r != SATTN_OK) return r;
    cnt += emit ? 1 : 0;
  }
  if (n_out) *n_out = cnt;
  return SATTN_OK;
}

sattn_status sa_stream_reset(sattn_stream* s) {
  if (!s) return fail(SATTN_EARG, "NULL handle");
  s->h = s->n_in = 0;
  s->closed = false;
  return SATTN_OK;
}

void sa_stream_destroy(sattn_stream* s) {
  if (!s) return;
  cudaFree(s->raw);
  cudaFree(s->ring);
  delete s;
}

sattn_status llsa_stream_create(const sattn_desc* d, int n_layers, sattn_stream** out) {
  if (!out) return fail(SATTN_EARG, "out is NULL");
  *out = nullptr;
  if (!d) return fail(SATTN_EARG, "desc is NULL");
  sattn_desc dd = *d;
  dd.T = 1;
  sattn_status r = validate(&dd);
  if (r != SATTN_OK) return r;
  if (n_layers < 1) return fail(SATTN_EARG, "n_layers must be >= 1");
  sattn_stream* s = new (std::nothrow) sattn_stream{};
  if (!s) return fail(SATTN_ECUDA, "out of host memory");
  s->d = dd;
  s->n_layers = n_layers;
  s->mode = SATTN_MODE_LLSA;
  const size_t es = elem_size(d->dtype);
  const size_t BH = d->B * d->H;
  const size_t raw_b = BH * (d->R + 1) * d->D * es;
  const size_t ring_b = (size_t)n_layers * BH * (d->L > 0 ? d->L : 1) * d->D * es;
  cudaError_t e = cudaMalloc(&s->raw, raw_b);
  if (e == cudaSuccess) e = cudaMalloc(&s->ring, ring_b);
  if (e == cudaSuccess) e = cudaMemset(s->raw, 0, raw_b);
  if (e == cudaSuccess) e = cudaMemset(s->ring, 0, ring_b);
  if (e != cudaSuccess) {
    cudaFree(s->raw);
    cudaFree(s->ring);
    delete s;
    return fail(SATTN_ECUDA, "stream state allocation: %s", cudaGetErrorString(e));
  }
  *out = s;
  return SATTN_OK;
}

sattn_status llsa_stream_step(sattn_stream* s, const void* x_new, void* y_out, int64_t* out_frame, void* stream) {
  if (!s || !x_new || !y_out) return fail(SATTN_EARG, "NULL pointer");
  if (s->mode != SATTN_MODE_LLSA) return fail(SATTN_EARG, "not an LLSA stream handle");
  if (s->closed) return fail(SATTN_ESTATE, "stream already flushed (call llsa_stream_reset)");
  const long long h = s->h;
  sattn_status r = stream_launch(s, x_new, y_out, h, h, (cudaStream_t)stream);
  if (r != SATTN_OK) return r;
  s->h = h + 1;
  s->n_in = h + 1;
  if (out_frame) *out_frame = h >= s->d.R ? h - s->d.R : -1;
  return SATTN_OK;
}

sattn_status llsa_stream_flush(sattn_stream* s, void* y_tail, int32_t* n_out, void* stream) {
  if (!s || !y_tail) return fail(SATTN_EARG, "NULL pointer");
  if (s->mode != SATTN_MODE_LLSA) return fail(SATTN_EARG, "not an LLSA stream handle");
  if (s->closed) return fail(SATTN_ESTATE, "stream already flushed");
  s->closed = true;
  const long long T = s->n_in, R = s->d.R;
  const size_t frame_b = s->d.B * s->d.H * s->d.D * elem_size(s->d.dtype);
  int cnt = 0;
  for (long long h = T; h < T + R; ++h) {
    if (h - R < 0) continue;
    sattn_status r = stream_launch(s, nullptr, static_cast<char*>(y_tail) + cnt * frame_b, h, T - 1, (cudaStream_t)stream);
    if (r != SATTN_OK) return r;
    ++cnt;
  }
  if (n_out) *n_out = cnt;
  return SATTN_OK;
}

sattn_status llsa_stream_reset(sattn_stream* s) {
  if (!s) return fail(SATTN_EARG, "NULL handle");
  s->h = s->n_in = 0;
  s->closed = false;
  return SATTN_OK;
}

void llsa_stream_destroy(sattn_stream* s) {
  if (!s) return;
  cudaFree(s->raw);
  cudaFree(s->ring);
  delete s;
}

}  // extern "C"
