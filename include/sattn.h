/*
 * sattn.h — C ABI of libsattn.so: streaming attention (SA) and low-latency
 * streaming attention (LLSA) of arXiv 2302.13451 on NVIDIA B200 (sm_100a).
 *
 * Citations: P:Lx = line x of the paper text; readings G1..G23 are
 * listed in DESIGN.md §3.  Letters (reading G1): L = look-back (the paper's B),
 * R = look-ahead (the paper's A), B = batch, H = heads, T = frames (N_T),
 * D = head dim (d_k = d_v), C = R + 1 LLSA channels.
 *
 * Conventions (every entry point):
 *  - Tensor pointers are DEVICE pointers owned by the caller, contiguous
 *    row-major, 16-byte aligned.  SA tensors are [B][H][T][D]; LLSA tensors
 *    are channel-major [C][B][H][T][D] (channel c = the version of a frame
 *    computed with c look-ahead frames).  LSE / delta are fp32
 *    [B][H][T] (SA) or [C][B][H][T] (LLSA).
 *  - Element type of Q/K/V/O/dO/dQ/dK/dV/X/Y is desc->dtype (SATTN_F32 or
 *    SATTN_BF16); arithmetic is fp32 (FFMA or tensor-core fp32 accumulate).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Argument
 *    validation is synchronous and returns an error status before anything is
 *    enqueued; execution is asynchronous on `stream`.  Hot calls never
 *    allocate; workspaces are sized by the *_workspace / *_bytes queries.
 *  - No C++ exception crosses this boundary.  On failure the call returns a
 *    non-zero sattn_status and sattn_last_error() (thread-local) describes it.
 *  - Non-finite inputs are not checked on the GPU (NaN propagates).
 *  - LSE is in natural-log units: LSE_t = log sum_{u in window(t)} exp(z_tu),
 *    z_tu = scale * q_t . k_u (Eq. 4).
 */
#ifndef SATTN_H
#define SATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SATTN_OK = 0,
  SATTN_EARG = 1,          /* bad size / pointer / alignment / band */
  SATTN_ESTATE = 2,        /* call not valid in the handle's current state */
  SATTN_ECONFIG = 3,       /* inconsistent configuration (e.g. workspace too small) */
  SATTN_EUNSUPPORTED = 4,  /* valid but not implemented (dtype x D x impl) */
  SATTN_ECUDA = 5,         /* a CUDA runtime/driver call failed */
  SATTN_ENCCL = 6          /* the time-sharded path's exchange failed (NCCL or callback) */
} sattn_status;

enum { SATTN_F32 = 0, SATTN_BF16 = 1 };            /* desc->dtype */
enum { SATTN_MODE_SA = 0, SATTN_MODE_LLSA = 1 };   /* stack mode */
enum {                                             /* desc->impl */
  SATTN_IMPL_AUTO = 0,  /* fastest available kernel family for dtype x D */
  SATTN_IMPL_FFMA = 1,  /* CUDA-core fp32 FFMA kernels (any supported D) */
  SATTN_IMPL_TC = 2     /* tcgen05 tensor-core kernels (bf16, D = 64) */
};

typedef struct {
  int64_t B, H, T, D;      /* batch, heads, frames, head dim (D in {2,4,8,16,32,64}) */
  int32_t L, R;            /* look-back / look-ahead frames, >= 0 (Eq. 4) */
  int32_t dtype;           /* SATTN_F32 | SATTN_BF16 */
  float scale;             /* score scale; 0 -> 1/sqrt(D) (G15) */
  int32_t in_broadcast;    /* LLSA inputs only: 1 -> Q,K,V are a single [B][H][T][D]
                              tensor read as every channel (layer-1 duplication,
                              P:L283, G11); 0 -> dense [C][B][H][T][D] */
  int32_t impl;            /* SATTN_IMPL_* */
} sattn_desc;

/* ---------------- SA: Eq. 4-13 ----------------------------------
 * sa_forward: O_t = sum_{u=t-L}^{t+R} softmax_u(z_tu) V_u, window clipped to
 * [0, T-1] (G2); writes O [B][H][T][D] and LSE [B][H][T].                      */
sattn_status sa_forward(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                        void* O, float* LSE, void* stream);

/* sa_forward_ws: sa_forward with a workspace of >= sa_forward_workspace(desc) bytes (0 when none
 * is needed).  Bands wider than the narrow tensor-core kernels (bf16, D = 64, W = L+R+1 > 65: the
 * paper's Fig. 5 sweep reaches W = 490) then also run on tensor cores: the band is
 * split into ceil(W / 49) sub-bands whose (O, max, sum) rows are merged by log-sum-exp in fp32
 * (exact softmax over the union); sa_forward keeps such bands on the CUDA-core kernels.        */
size_t sa_forward_workspace(const sattn_desc* desc);
sattn_status sa_forward_ws(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                           void* O, float* LSE, void* ws, size_t ws_bytes, void* stream);

/* sa_backward: exact gradients dQ, dK, dV of <dO, O> (Eq. 7-13 with Eq. 7's
 * index condition, G3).  O and LSE must come from sa_forward on the same
 * inputs (not checked: undefined results otherwise).  ws >= sa_backward_workspace(desc)
 * bytes of device memory (holds delta_t = sum_u P_tu dP_tu, fp32, which equals
 * dO_t . O_t for the exact O: the tensor-core path forms it from P and dP (G26),
 * the CUDA-core path from dO and O; wide tensor-core bands (W > 65) take delta = dO . O and
 * sum the sub-bands' gradients in fp32 accumulators also held in ws).  Deterministic (no atomics): bitwise
 * reproducible run to run.                                                    */
size_t sa_backward_workspace(const sattn_desc* desc);
sattn_status sa_backward(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                         const void* O, const float* LSE, const void* dO,
                         void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes, void* stream);

/* ---------------- SA with the stored band (NEXT-4) ----------
 * The paper keeps z_t and a_t as N_T x (A+B+1) matrices; the calls
 * above keep only LSE [B][H][T] and recompute a_t.  These keep a_t instead:
 * sa_p_ld(desc): row stride (elements) of the band, W = L+R+1 rounded up to a
 *   multiple of 8 (16-byte rows); 0 if desc is invalid.
 * sa_forward_p: as sa_forward, and also writes P [B][H][T][ld] (desc->dtype),
 *   P[t][j] = a_{t, t-L+j} (Eq. 5) for j < W, exactly 0 where t-L+j is
 *   outside [0, T-1] (G2) and for j >= W.  Forward on tensor cores for bf16,
 *   D = 64, W <= 64; CUDA cores otherwise (desc->impl = SATTN_IMPL_TC outside
 *   that limit -> SATTN_EUNSUPPORTED).
 * sa_backward_p: gradients of <dO, O> with a_t read from P instead of
 *   recomputed (Eq. 7-13); P must come from sa_forward_p on the same inputs.
 *   Tensor cores for bf16, D = 64: one pass for W <= 49, 48-column sub-bands of
 *   P (gradients summed in fp32) for 49 < W <= 4096; CUDA cores otherwise.
 *   ws >= sa_backward_p_workspace(desc) bytes (delta_t, fp32: sum_j P_tj dP_tj
 *   in the one-pass tensor-core kernels, dO_t . O_t for sub-bands and on CUDA
 *   cores, where O is read; sub-bands also keep fp32 dQ, dK, dV accumulators in
 *   ws).  Deterministic (no atomics).                                         */
int64_t sa_p_ld(const sattn_desc* desc);
sattn_status sa_forward_p(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                          void* O, float* LSE, void* P, void* stream);
size_t sa_backward_p_workspace(const sattn_desc* desc);
sattn_status sa_backward_p(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                           const void* O, const void* P, const void* dO,
                           void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes, void* stream);

/* ---------------- LLSA: Eq. 14-16 -------------------------------
 * Output (t, c) attends the Eq. 14 slots read in the Fig. 3(c) convention (G6):
 * anchor s = t-(R-c); slots (u, R) for u in [s-L, s] and (s+j, R-j), j=1..R,
 * clipped to [0, T-1]; query q_{t,c} (G7).  Q,K,V: [C][B][H][T][D] or, with
 * desc->in_broadcast, one [B][H][T][D] tensor used for every channel.
 * O: [C][B][H][T][D]; LSE: [C][B][H][T].                                      */
sattn_status llsa_forward(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                          void* O, float* LSE, void* stream);

/* llsa_backward: exact gradient (G8/G9).  dQ,dK,dV are always dense
 * [C][B][H][T][D] (gradient per channel slot; with in_broadcast the caller
 * sums over channels).  ws >= llsa_backward_workspace(desc).  Deterministic.  */
size_t llsa_backward_workspace(const sattn_desc* desc);
sattn_status llsa_backward(const sattn_desc* desc, const void* Q, const void* K, const void* V,
                           const void* O, const float* LSE, const void* dO,
                           void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes, void* stream);

/* ---------------- layer-stack driver (reading G12) ---------
 * n_layers tied-QKV layers: Y_l = ATT(X_l, X_l, X_l), X_{l+1} = (X_l + Y_l)/2,
 * ATT = SA (mode SATTN_MODE_SA) or LLSA (SATTN_MODE_LLSA; X_0 duplicated into
 * all channels).  X0: [B][H][T][D].  Y = X_{n}: [B][H][T][D] (SA) or
 * [C][B][H][T][D] (LLSA; designated output = channel R, G10).
 * `saved` (>= sattn_stack_saved_bytes) keeps X_l, O_l, LSE_l for the backward.
 * desc->in_broadcast is ignored (the driver sets it per layer).               */
size_t sattn_stack_saved_bytes(const sattn_desc* desc, int mode, int n_layers);
sattn_status sattn_stack_forward(const sattn_desc* desc, int mode, int n_layers, const void* X0,
                                 void* saved, size_t saved_bytes, void* Y, void* stream);
/* Byte offsets in `saved` of layer l's input X_l (l = 0: [B][H][T][D]; l > 0: [C][B][H][T][D]
 * for LLSA, [B][H][T][D] for SA), its attention output O_l and LSE_l (shaped as the forward
 * calls' outputs) — for inspecting the stack layer by layer (out3 = {X_l, O_l, LSE_l}).       */
sattn_status sattn_stack_saved_offsets(const sattn_desc* desc, int mode, int n_layers, int layer, int64_t* out3);
/* Gradient of <dY, Y> w.r.t. X0 (dY shaped like Y; dX0 [B][H][T][D]).
 * ws >= sattn_stack_workspace(desc, mode, n_layers).                          */
size_t sattn_stack_workspace(const sattn_desc* desc, int mode, int n_layers);
sattn_status sattn_stack_backward(const sattn_desc* desc, int mode, int n_layers, const void* saved,
                                  const void* dY, void* dX0, void* ws, size_t ws_bytes, void* stream);

/* ---------------- incremental LLSA inference (infer_llsa) -------------
 * Library-owned state for n_layers tied-QKV LLSA layers (same block rule as
 * the stack driver): per layer a ring of the channel-R frames of its input for
 * the last L frames, plus the last R+1 raw frames.  desc->T is ignored
 * (unbounded stream).  llsa_stream_step ingests x_new [B][H][D] for frame h
 * (h = number of previous steps), runs horizon h through every layer in one
 * kernel launch and, once h >= R, writes the designated output X_n(h-R, R) to
 * y_out [B][H][D] and sets *out_frame = h-R (else *out_frame = -1; y_out
 * untouched).  llsa_stream_flush ends the stream: it runs the remaining R
 * horizons with windows clipped at the last frame and writes frames
 * T-R..T-1 (those >= 0) to y_tail [R][B][H][D]; *n_out = number written.
 * A handle is single-owner (not thread-safe); create allocates device memory,
 * step/flush never allocate.  out_frame / n_out are host pointers.            */
typedef struct sattn_stream sattn_stream;
sattn_status llsa_stream_create(const sattn_desc* desc, int n_layers, sattn_stream** out);
sattn_status llsa_stream_step(sattn_stream* s, const void* x_new, void* y_out, int64_t* out_frame,
                              void* stream);
sattn_status llsa_stream_flush(sattn_stream* s, void* y_tail, int32_t* n_out, void* stream);
sattn_status llsa_stream_reset(sattn_stream* s);
void llsa_stream_destroy(sattn_stream* s);

/* ---------------- incremental SA inference (infer_sa; NEXT-2) ----------
 * The SA stack of sattn_stack_forward(SATTN_MODE_SA) run frame by frame: layer l
 * can emit frame t only once its input holds t + R, so after frame h arrives
 * layer l computes t = h - (l+1) R and the stack emits X_n(h - n R) — latency
 * n_layers x R frames (Table 3's infer_sa; compare llsa_stream_*).
 * State: per layer a ring of its last L+R+1 input frames.  sa_stream_step
 * ingests x_new [B][H][D] for frame h (one kernel launch for all layers) and,
 * once h >= n_layers R, writes X_n(h - n R) to y_out [B][H][D] and sets
 * *out_frame = h - n R (else -1, y_out untouched).  sa_stream_flush runs the
 * remaining n R steps with windows clipped at the last frame and writes frames
 * T - nR .. T-1 (those >= 0) to y_tail [n R][B][H][D]; *n_out = number written.
 * Ownership and threading as for llsa_stream_*; the handle type is shared and
 * sattn_stream_destroy / llsa_stream_destroy free either kind.                  */
sattn_status sa_stream_create(const sattn_desc* desc, int n_layers, sattn_stream** out);
sattn_status sa_stream_step(sattn_stream* s, const void* x_new, void* y_out, int64_t* out_frame, void* stream);
sattn_status sa_stream_flush(sattn_stream* s, void* y_tail, int32_t* n_out, void* stream);
sattn_status sa_stream_reset(sattn_stream* s);
void sa_stream_destroy(sattn_stream* s);

/* ---------------- time sharding over ranks (Eq. 4) ----
 * One long stream (the hour-long stream) split over ranks by time: rank r owns frames
 * [t0, t0 + T) of every (b, h), shards in rank order.  Eq. 4's window makes O_t depend on
 * K, V over [t-L, t+R] and Eq. 7/13's gathers (G3) make dK_u, dV_u depend on queries
 * [u-R, u+L], so one exchange of boundary frames with the two neighbours per call is exact.
 *
 * MARGINED layout: every tensor of these calls is [B][H][M + T + M][D] (LSE
 * [B][H][M + T + M], fp32) with M = SATTN_TSHARD_MARGIN frames on both sides; the local
 * frames are rows [M, M + T).  The library fills the margins it needs from the neighbours
 * (forward: K, V L+R rows each side, Q R rows left / L right; backward: dO R left / L right)
 * and computes the halo queries' LSE (forward) and delta (backward) itself, so no LSE or
 * delta crosses ranks.  Margin rows the exchange does not write must hold finite values
 * (zero-initialise the buffers once).  The backward must get the same Q, K, V buffers (with
 * the margins the forward filled) and the forward's LSE.  Outputs: local rows of O / LSE /
 * dQ / dK / dV (margin rows of the outputs are scratch).  With t0 a multiple of 128 the local
 * rows are bitwise equal to the unsharded call's on one (b, h) plane per call (a call over
 * several planes packs its 128-row tiles over the flattened B*H*T axis, summing in another
 * order: equal to the parity gate, not bitwise).  Tensor-core path only: bf16, D = 64,
 * L + R + 1 <= 65, L + R <= M; every shard T >= L + R when it has neighbours.
 * The exchange overlaps the tiles whose operands are all local; no host synchronisation.
 * Transport: NCCL (sattn_dist_init: one communicator per process, send/recv to rank +- 1
 * in one group on a library stream) or a caller callback (sattn_dist_init_external). */
#define SATTN_TSHARD_MARGIN 128
typedef struct {
  sattn_desc local;      /* B, H, D, L, R, dtype, scale, impl; T = this rank's frames */
  int64_t t0;            /* global index of this rank's first frame */
  int64_t T_global;      /* frames of the whole stream */
} sattn_tshard_desc;
typedef struct sattn_dist sattn_dist;   /* opaque: communicator, stream, events */
/* callback transport: exchange the four DEVICE buffers with rank-1 (send_left / recv_left) and
 * rank+1 (send_right / recv_right); NULL / 0 where there is no neighbour.  `send_*` are ready
 * once `stream`'s prior work completes; `recv_*` must be filled before later work on `stream`
 * runs (the callback may synchronise).  Return 0 on success. */
typedef int (*sattn_exchange_fn)(void* user, const void* send_left, size_t send_left_bytes, void* recv_left,
                                 size_t recv_left_bytes, const void* send_right, size_t send_right_bytes,
                                 void* recv_right, size_t recv_right_bytes, void* stream);
int64_t sattn_tshard_margin(void);
sattn_status sattn_dist_unique_id(void* id_out /* 128 bytes (ncclUniqueId), host */);
sattn_status sattn_dist_init(int rank, int world, const void* nccl_unique_id, sattn_dist** out);
sattn_status sattn_dist_init_external(int rank, int world, sattn_exchange_fn fn, void* user, sattn_dist** out);
void sattn_dist_destroy(sattn_dist* d);
/* device workspace (bytes) for either call below; 0 if the configuration is invalid */
size_t sa_tsharded_workspace(const sattn_tshard_desc* td, const sattn_dist* d);
sattn_status sa_forward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                 float* LSE, void* ws, size_t ws_bytes, void* stream);
sattn_status sa_backward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                  const void* V, const float* LSE, void* dO, void* dQ, void* dK, void* dV,
                                  void* ws, size_t ws_bytes, void* stream);
/* The stored-band mode (sa_forward_p / sa_backward_p) on the same margined shards, with P margined
 * too: [B][H][M + T + M][sa_p_ld(desc)].  The forward's exchange and overlap are as above and it
 * writes the band rows of the whole slab; the backward exchanges dO only (the halo queries' delta =
 * rowsum(P o dP) is formed from the margins).  Tensor cores, L + R + 1 <= 49.  Same workspace query. */
sattn_status sa_forward_p_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                   float* LSE, void* P, void* ws, size_t ws_bytes, void* stream);
sattn_status sa_backward_p_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                    const void* V, const void* P, void* dO, void* dQ, void* dK, void* dV, void* ws,
                                    size_t ws_bytes, void* stream);
/* host-only: out6 = {hl, hr, slab frames, query tiles, first interior tile, first right-edge tile} */
sattn_status sattn_tshard_geometry(const sattn_tshard_desc* td, int rank, int world, int64_t* out6);

/* Time-sharded LLSA (Eq. 14-16).  Output (t, c) reads frames
 * [t-R-L, t+R] of every channel (horizon t+c: band keys of channel R, staircase keys), and the
 * local dQ/dK/dV also receive from the halo outputs t in [t0-R, t0) and [t1, t1+L+R), whose P
 * and delta are exact when their own windows lie in the slab.  So every tensor of these calls
 * is a contiguous SLAB [C][B][H][hl + T + hr][D] (LSE [C][B][H][hl + T + hr] fp32), hl = hr =
 * llsa_tshard_margin(L, R) = L + 2R where a left / right neighbour exists (else 0), local
 * frames at rows [hl, hl + T).  The forward fills the Q, K, V margins from the neighbours (L+2R
 * rows of every channel) and runs llsa_forward on the slab (halo rows' O, LSE exact, kept for
 * the backward); the backward fills dO's halo rows (R from the left, L+R from the right) and
 * runs llsa_backward on the slab.  Local rows equal the unsharded call's up to summation order;
 * margin rows of outputs are scratch; margin rows the exchange does not write must be finite
 * (zero-initialise once).  The backward must get the forward's Q, K, V, O, LSE slabs.  Dense
 * inputs (in_broadcast = 0); every shard T >= L + 2R when it has neighbours.  On the dense
 * tensor-core path (bf16, D = 64, the item-form kernels) the exchange overlaps the items whose
 * rows are all local (forward: rows [h0-R-L, h0+HZ); backward fused pass: dO rows [h0-R, h0+HZ));
 * the edge items, then the kv pass, follow the halo.  Same transports as SA. */
int64_t llsa_tshard_margin(int32_t L, int32_t R);
size_t llsa_tsharded_workspace(const sattn_tshard_desc* td, const sattn_dist* d);
sattn_status llsa_forward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                   float* LSE, void* ws, size_t ws_bytes, void* stream);
sattn_status llsa_backward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                    const void* V, const void* O, const float* LSE, void* dO, void* dQ, void* dK,
                                    void* dV, void* ws, size_t ws_bytes, void* stream);

/* ---------------- misc ---------------------------------------------------------*/
const char* sattn_last_error(void);      /* thread-local message of the last failure */
const char* sattn_version(void);
/* Number of kernel launches this library has enqueued since load (all threads).
 * Launches replayed from a captured CUDA graph are not re-counted.            */
int64_t sattn_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SATTN_H */
