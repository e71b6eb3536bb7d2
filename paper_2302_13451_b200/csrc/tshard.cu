// tshard.cu — time-sharded SA over ranks: the distributed part of the C ABI.
//
// Rank r owns frames [t0, t0 + T_loc) of every (b, h) of one long stream (the hour-long stream,
// BASELINE configs[4]).  Eq. 4's window makes O_t depend on K, V over [t - L, t + R]
// and Eq. 7/13's gathers (reading G3) make dK_u, dV_u depend on queries n in [u - R, u + L], so
// one exchange of boundary frames with the two neighbours per call is exact.  Every tensor of a
// time-sharded call is MARGINED: [B][H][M + T_loc + M][D] (LSE [B][H][M + T_loc + M]) with
// M = SATTN_TSHARD_MARGIN = 128 frames on both sides, the local frames at rows [M, M + T_loc).
// The kernels run on the slab [M - hl, M + T_loc + hr) (hl = M if a left neighbour exists, else
// 0; hr likewise): the SAME tensor-core kernels as the unsharded call, with tensor maps starting
// at the slab's first row and the margined row stride, so every local frame keeps its 128-frame
// tile offset when t0 is a multiple of 128 (then the local rows are BITWISE equal to the
// unsharded call's: deterministic kernels, identical operands in every tile that touches them).
//
// What is exchanged (rows per side; the paper's letters: L look-back, R look-ahead):
//   forward   K, V: L + R rows each way;  Q: R rows from the left, L rows from the right
//   backward  dO:   R rows from the left, L rows from the right
// Why this set: the backward needs, for the halo queries n in [t0 - R, t0) and [t1, t1 + L) that
// feed local dK / dV, their q_n, dO_n, LSE_n and delta_n.  Instead of shipping LSE_n and delta_n
// (SURVEY §8(e)'s table) this rank recomputes them: the forward's halo tile computes LSE_n from
// the L + R deep K / V margins and the Q margin, the backward's K1 halo tile computes delta_n
// = rowsum(P o dP) (G26) from the same margins and the dO margin.  The backward then needs one
// exchange (dO) before K1's edge tiles and none between K1 and K2.  The K / V / Q margins the
// forward filled must be unchanged when the backward runs (the caller passes the same buffers).
//
// Overlap: the exchange runs on the dist handle's stream while the kernels process the tiles
// whose operand boxes lie inside the local rows (interior tiles); the edge tiles (the halo tiles
// and the tiles whose key boxes reach into a margin) run after it.  No host synchronisation.
//
// Transports: NCCL point-to-point (ncclSend / ncclRecv to rank +- 1 in one group; NVLink between
// GPUs), libnccl.so.2 resolved at sattn_dist_init (the copy torch already loaded, if any); or a
// caller-supplied exchange callback (sattn_dist_init_external: e.g. host-staged gloo for tests on
// one GPU).  Pack / unpack of the strided margins to contiguous messages are one kernel each.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "common.cuh"
#include "ffma_attn.cuh"
#include "host_util.h"
#include "internal.h"
#include "tc_dispatch.h"

using namespace sattn;

namespace {

constexpr int kMargin = SATTN_TSHARD_MARGIN;

// ---------------------------------------------------------------- NCCL, resolved at run time
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok;
};

const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto get = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(get("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(get("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(get("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(get("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(get("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(get("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(get("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(get("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
             api.Recv && api.GetErrorString;
  });
  return api;
}

sattn_status nccl_fail(const char* what, ncclResult_t r) {
  std::string m = std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
  return set_error(SATTN_ENCCL, m.c_str());
}

sattn_status cuda_fail(const char* what, cudaError_t e) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(SATTN_ECUDA, m.c_str());
}

// ------------------------------------------------------------- strided <-> contiguous copies
// A segment moves `heads` blocks of `bytes` (a multiple of 16) from src + h * src_pitch to
// dst + h * dst_pitch.  Pack: strided margins/rows -> a contiguous message; unpack: the reverse.
struct Seg {
  const char* src;
  char* dst;
  long long src_pitch, dst_pitch;
  int bytes, heads;
};
constexpr int kMaxSeg = 8;
struct SegList {
  Seg s[kMaxSeg];
  long long off[kMaxSeg + 1];   // prefix sums of 16-byte chunks
  int n;
};

__global__ void __launch_bounds__(256) copy_segments(SegList L) {
  const long long total = L.off[L.n];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < L.n && i >= L.off[k + 1]) ++k;
    const Seg& s = L.s[k];
    const long long j = i - L.off[k];
    const int per = s.bytes >> 4;
    const long long h = j / per, c = j - h * per;
    const uint4 v = *reinterpret_cast<const uint4*>(s.src + h * s.src_pitch + c * 16);
    *reinterpret_cast<uint4*>(s.dst + h * s.dst_pitch + c * 16) = v;
  }
}

sattn_status run_segments(SegList& L, cudaStream_t st) {
  L.off[0] = 0;
  for (int k = 0; k < L.n; ++k) L.off[k + 1] = L.off[k] + (long long)(L.s[k].bytes >> 4) * L.s[k].heads;
  const long long total = L.off[L.n];
  if (total == 0) return SATTN_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  copy_segments<<<(int)blocks, 256, 0, st>>>(L);
  count_launches(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SATTN_OK : cuda_fail("copy_segments launch", e);
}

// one tensor's halo: `base` = margined buffer (row 0 of head 0), rows of `row_bytes`, pitch
// `ld` rows per head; the left margin needs `need_l` rows from rank-1, the right `need_r` from rank+1
struct HaloT {
  char* base;
  int need_l, need_r;
};

struct Geo {
  long long BH;        // planes (SA: B*H; LLSA: channels x B*H)
  int T_loc, ld, row_bytes;
  bool left, right;
  int first;           // row of the first local frame in a plane (SA: the margin M; LLSA: hl)
};

// message sizes of one exchange (bytes): to / from the left neighbour, to / from the right one
struct Msg {
  size_t send_l, recv_l, send_r, recv_r;
};
Msg msg_sizes(const Geo& g, const HaloT* t, int nt) {
  Msg m{0, 0, 0, 0};
  for (int i = 0; i < nt; ++i) {
    const size_t per = (size_t)g.BH * g.row_bytes;
    if (g.left) { m.send_l += per * t[i].need_r; m.recv_l += per * t[i].need_l; }
    if (g.right) { m.send_r += per * t[i].need_l; m.recv_r += per * t[i].need_r; }
  }
  return m;
}

}  // namespace

struct sattn_dist {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  sattn_exchange_fn fn = nullptr;
  void* user = nullptr;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
};

namespace {

// Enqueue one halo exchange of the tensors t[0..nt) into their margins.  NCCL: on d->cs after
// `st`'s work so far, then d->ev_halo records its completion (the caller waits on it before the
// edge tiles).  External transport: in order on `st`.  ws: [send_l | recv_l | send_r | recv_r].
sattn_status exchange(sattn_dist* d, const Geo& g, const HaloT* t, int nt, char* ws, cudaStream_t st) {
  const Msg m = msg_sizes(g, t, nt);
  char* send_l = ws;
  char* recv_l = send_l + m.send_l;
  char* send_r = recv_l + m.recv_l;
  char* recv_r = send_r + m.send_r;
  const long long pitch = (long long)g.ld * g.row_bytes;
  SegList pack{}, unpack{};
  size_t o_sl = 0, o_rl = 0, o_sr = 0, o_rr = 0;
  for (int i = 0; i < nt; ++i) {
    char* b = t[i].base;
    const long long first = (long long)g.first * g.row_bytes, last = (long long)(g.first + g.T_loc) * g.row_bytes;
    if (g.left) {
      // to rank-1: my first need_r rows (its right margin); from rank-1: my left margin
      pack.s[pack.n++] = Seg{b + first, send_l + o_sl, pitch, (long long)t[i].need_r * g.row_bytes,
                             t[i].need_r * g.row_bytes, (int)g.BH};
      unpack.s[unpack.n++] = Seg{recv_l + o_rl, b + first - (long long)t[i].need_l * g.row_bytes,
                                 (long long)t[i].need_l * g.row_bytes, pitch, t[i].need_l * g.row_bytes, (int)g.BH};
      o_sl += (size_t)g.BH * t[i].need_r * g.row_bytes;
      o_rl += (size_t)g.BH * t[i].need_l * g.row_bytes;
    }
    if (g.right) {
      // to rank+1: my last need_l rows (its left margin); from rank+1: my right margin
      pack.s[pack.n++] = Seg{b + last - (long long)t[i].need_l * g.row_bytes, send_r + o_sr, pitch,
                             (long long)t[i].need_l * g.row_bytes, t[i].need_l * g.row_bytes, (int)g.BH};
      unpack.s[unpack.n++] = Seg{recv_r + o_rr, b + last, (long long)t[i].need_r * g.row_bytes, pitch,
                                 t[i].need_r * g.row_bytes, (int)g.BH};
      o_sr += (size_t)g.BH * t[i].need_l * g.row_bytes;
      o_rr += (size_t)g.BH * t[i].need_r * g.row_bytes;
    }
  }
  // drop empty segments (need 0 rows)
  auto compact = [](SegList& L) {
    int n = 0;
    for (int k = 0; k < L.n; ++k)
      if (L.s[k].bytes > 0) L.s[n++] = L.s[k];
    L.n = n;
  };
  compact(pack);
  compact(unpack);
  if (pack.n == 0 && unpack.n == 0) {
    if (d->comm) {   // nothing to move: still give the caller an event to wait on
      cudaError_t e = cudaEventRecord(d->ev_halo, st);
      if (e != cudaSuccess) return cuda_fail("cudaEventRecord", e);
    }
    return SATTN_OK;
  }
  if (d->comm) {
    cudaError_t e = cudaEventRecord(d->ev_in, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d->cs, d->ev_in, 0);
    if (e != cudaSuccess) return cuda_fail("stream ordering", e);
    sattn_status s = run_segments(pack, d->cs);
    if (s != SATTN_OK) return s;
    const NcclApi& n = nccl();
    ncclResult_t r = n.GroupStart();
    if (r == ncclSuccess && g.left) {
      if (m.send_l) r = n.Send(send_l, m.send_l, ncclUint8, d->rank - 1, d->comm, d->cs);
      if (r == ncclSuccess && m.recv_l) r = n.Recv(recv_l, m.recv_l, ncclUint8, d->rank - 1, d->comm, d->cs);
    }
    if (r == ncclSuccess && g.right) {
      if (m.send_r) r = n.Send(send_r, m.send_r, ncclUint8, d->rank + 1, d->comm, d->cs);
      if (r == ncclSuccess && m.recv_r) r = n.Recv(recv_r, m.recv_r, ncclUint8, d->rank + 1, d->comm, d->cs);
    }
    const ncclResult_t r2 = n.GroupEnd();
    if (r != ncclSuccess) return nccl_fail("halo send/recv", r);
    if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
    s = run_segments(unpack, d->cs);
    if (s != SATTN_OK) return s;
    e = cudaEventRecord(d->ev_halo, d->cs);
    if (e != cudaSuccess) return cuda_fail("cudaEventRecord", e);
    return SATTN_OK;
  }
  sattn_status s = run_segments(pack, st);
  if (s != SATTN_OK) return s;
  const int rc = d->fn(d->user, g.left ? send_l : nullptr, m.send_l, g.left ? recv_l : nullptr, m.recv_l,
                       g.right ? send_r : nullptr, m.send_r, g.right ? recv_r : nullptr, m.recv_r, st);
  if (rc != 0) return set_error(SATTN_ENCCL, "external halo exchange callback failed");
  return run_segments(unpack, st);
}

// Query-tile subsets of the slab (T' = hl + T_loc + hr frames, 128-frame tiles): a tile is an
// EDGE tile if its query rows or its key box [128 kt - L, 128 kt - L + nk) reach into a margin
// that the exchange fills; the rest (interior) only read local rows.  Edge tiles are a prefix
// [0, e0) and a suffix [e1, ntq).
struct Tiles {
  int ntq, e0, e1;
};
Tiles tile_split(int hl, int T_loc, int hr, int L, int nk) {
  Tiles t;
  const int Ts = hl + T_loc + hr;
  t.ntq = (Ts + 127) / 128;
  t.e0 = hl > 0 ? (hl + L + 127) / 128 : 0;                          // 128 kt - L < hl
  t.e1 = t.ntq;
  if (hr > 0) {                                                       // 128 kt - L + nk > hl + T_loc
    const int lim = hl + T_loc + L - nk;                              // kt > lim / 128
    t.e1 = lim < 0 ? 0 : lim / 128 + 1;
  }
  if (t.e0 > t.ntq) t.e0 = t.ntq;
  if (t.e1 < t.e0) t.e1 = t.e0;
  if (t.e1 > t.ntq) t.e1 = t.ntq;
  return t;
}
void set_interior(AttnArgs& a, const Tiles& t) {
  a.kt0 = t.e0; a.nkt = t.e1 - t.e0; a.kt_split = a.nkt; a.kt_jump = 0;
}
void set_edges(AttnArgs& a, const Tiles& t) {
  a.kt0 = 0; a.nkt = t.e0 + (t.ntq - t.e1); a.kt_split = t.e0; a.kt_jump = t.e1 - t.e0;
}

struct Shard {
  Geo g;
  int hl, hr, Ts;
  long long off;   // element offset of the slab's first row in a margined [ld][D] plane
  AttnArgs a;      // slab args (T = Ts, ld, no tile subset yet)
};

sattn_status shard_setup(const sattn_tshard_desc* td, const sattn_dist* d, Shard& s) {
  if (!td || !d) return set_error(SATTN_EARG, "NULL tshard desc or dist handle");
  const sattn_desc& l = td->local;
  sattn_status r = check_desc(&l);
  if (r != SATTN_OK) return r;
  if (l.dtype != SATTN_BF16 || l.D != 64 || l.impl == SATTN_IMPL_FFMA ||
      !tc_supported(l.dtype, (int)l.D, l.L, l.R, false, true))
    return set_error(SATTN_EUNSUPPORTED, "time-sharded SA runs the tensor-core kernels: bf16, D = 64, L + R + 1 <= 65");
  if (l.L + l.R > kMargin) return set_error(SATTN_EUNSUPPORTED, "time sharding needs L + R <= 128 (the margin)");
  if (td->t0 < 0 || td->T_global < td->t0 + l.T) return set_error(SATTN_EARG, "shard [t0, t0 + T) outside [0, T_global)");
  const bool left = td->t0 > 0, right = td->t0 + l.T < td->T_global;
  if (left != (d->rank > 0) || right != (d->rank < d->world - 1))
    return set_error(SATTN_ECONFIG, "shard position does not match the rank (shards must be in rank order)");
  if ((left || right) && l.T < l.L + l.R)
    return set_error(SATTN_ECONFIG, "a shard must hold at least L + R frames for its neighbours' halos");
  s.g.BH = l.B * l.H;
  s.g.T_loc = (int)l.T;
  s.g.ld = (int)l.T + 2 * kMargin;
  s.g.row_bytes = (int)l.D * 2;
  s.g.left = left;
  s.g.right = right;
  s.g.first = kMargin;
  s.hl = left ? kMargin : 0;
  s.hr = right ? kMargin : 0;
  s.Ts = s.hl + (int)l.T + s.hr;
  s.off = (long long)(kMargin - s.hl) * l.D;
  AttnArgs& a = s.a;
  a = AttnArgs{};
  a.T = s.Ts;
  a.ld = s.g.ld;
  a.L = l.L;
  a.R = l.R;
  a.BH = (int)s.g.BH;
  a.scale = desc_scale(&l);
  a.scale_log2 = a.scale * kLog2e;
  a.in_cs = a.out_cs = 0;
  return SATTN_OK;
}

const bf16* at(const void* p, long long off) { return reinterpret_cast<const bf16*>(p) + off; }
bf16* at(void* p, long long off) { return reinterpret_cast<bf16*>(p) + off; }

size_t halo_ws(const Geo& g, const HaloT* t, int nt) {
  const Msg m = msg_sizes(g, t, nt);
  return (m.send_l + m.recv_l + m.send_r + m.recv_r + 255) & ~size_t(255);
}
size_t halo_ws(const Shard& s, const HaloT* t, int nt) { return halo_ws(s.g, t, nt); }
int llsa_tshard_margin_of(int L, int R) { return L + 2 * R; }
int elem_bytes(int dtype) { return dtype == SATTN_BF16 ? 2 : 4; }

void fwd_halos(const Shard& s, const void* Q, const void* K, const void* V, HaloT* t) {
  const int L = s.a.L, R = s.a.R;
  t[0] = HaloT{(char*)K, L + R, L + R};
  t[1] = HaloT{(char*)V, L + R, L + R};
  t[2] = HaloT{(char*)Q, R, L};
}
void bwd_halos(const Shard& s, const void* dO, HaloT* t) { t[0] = HaloT{(char*)dO, s.a.R, s.a.L}; }

size_t bwd_rows_ws(const Shard& s) { return (size_t)2 * s.g.BH * ((s.Ts + 3) & ~3) * sizeof(float); }

// run the compute in two parts around the exchange: interior tiles, then (after the halo) edges
template <class Run>
sattn_status split_run(sattn_dist* d, Shard& s, int nk, cudaStream_t st, bool exchanged, Run&& run) {
  const Tiles tl = tile_split(s.hl, s.g.T_loc, s.hr, s.a.L, nk);
  sattn_status r;
  if (tl.e1 > tl.e0) {
    AttnArgs a = s.a;
    set_interior(a, tl);
    if ((r = run(a, true)) != SATTN_OK) return r;
  }
  if (exchanged && d->comm) {
    cudaError_t e = cudaStreamWaitEvent(st, d->ev_halo, 0);
    if (e != cudaSuccess) return cuda_fail("cudaStreamWaitEvent", e);
  }
  AttnArgs a = s.a;
  set_edges(a, tl);
  if (a.nkt > 0) return run(a, false);
  return SATTN_OK;
}

// ------------------------------------------------------------------------------------------
// Time-sharded LLSA (Eq. 14-16).  Output (t, c) reads the frames
// [t - R - L, t + R] of every channel (its horizon h = t + c: band keys h - R - L .. h - R of
// channel R, staircase keys (h - c', c')), so the local outputs need L + R frames from the left
// and R from the right.  The backward's local dQ, dK, dV also receive from the halo outputs
// (t, c) with t in [t0 - R, t0) and [t1, t1 + L + R) (every output whose window holds a local
// slot); their P and delta are exact when their own windows lie in the slab, i.e. with L + 2R
// frames on each side.  So a rank's tensors are the SLAB [C][B][H][hl + T + hr][D] (hl = L + 2R if
// a left neighbour exists, else 0; hr likewise; local frames at rows [hl, hl + T)), the forward
// exchanges Q, K, V margins of L + 2R rows (every channel) and runs the ordinary LLSA forward on
// the slab (its halo rows' O and LSE are exact), the backward exchanges the halo outputs' dO (R
// rows from the left, L + R from the right) and runs the ordinary LLSA backward on the slab.
// Local rows are exact (equal to the unsharded call's up to summation order); margin rows of the
// outputs are scratch.  Dense inputs only (in_broadcast = 0: a stack's layer 1 duplicates first).
// ------------------------------------------------------------------------------------------
struct LShard {
  Geo g;
  int hl, hr, Ts, C;
  sattn_desc slab;
};

sattn_status lshard_setup(const sattn_tshard_desc* td, const sattn_dist* d, LShard& s) {
  if (!td || !d) return set_error(SATTN_EARG, "NULL tshard desc or dist handle");
  const sattn_desc& l = td->local;
  sattn_status r = check_desc(&l);
  if (r != SATTN_OK) return r;
  if (l.in_broadcast) return set_error(SATTN_EUNSUPPORTED, "time-sharded LLSA takes dense [C][B][H][T][D] inputs");
  if ((l.D * elem_bytes(l.dtype)) % 16 != 0) return set_error(SATTN_EUNSUPPORTED, "rows must be 16-byte multiples");
  if (td->t0 < 0 || td->T_global < td->t0 + l.T) return set_error(SATTN_EARG, "shard [t0, t0 + T) outside [0, T_global)");
  const bool left = td->t0 > 0, right = td->t0 + l.T < td->T_global;
  if (left != (d->rank > 0) || right != (d->rank < d->world - 1))
    return set_error(SATTN_ECONFIG, "shard position does not match the rank (shards must be in rank order)");
  const int mg = llsa_tshard_margin_of(l.L, l.R);
  if ((left || right) && l.T < mg)
    return set_error(SATTN_ECONFIG, "a shard must hold at least L + 2R frames for its neighbours' halos");
  s.C = l.R + 1;
  s.hl = left ? mg : 0;
  s.hr = right ? mg : 0;
  s.Ts = s.hl + (int)l.T + s.hr;
  s.g.BH = (long long)s.C * l.B * l.H;
  s.g.T_loc = (int)l.T;
  s.g.ld = s.Ts;
  s.g.row_bytes = (int)(l.D * elem_bytes(l.dtype));
  s.g.left = left;
  s.g.right = right;
  s.g.first = s.hl;
  s.slab = l;
  s.slab.T = s.Ts;
  return SATTN_OK;
}

// Interior / edge item split of the dense item-form LLSA kernels on a slab (per (b, h), item j =
// horizons [j HZ, j HZ + HZ)): an item reads rows [j HZ - lo, j HZ + HZ - 1] (forward: lo = R + L,
// Q / K / V; backward fused pass: lo = R, the halo-exchanged dO), so it is interior when those rows
// are local or beyond a missing neighbour.  sub = {it0, nit_l, it_split, it_jump} (tc_dispatch.h).
struct ItemSplit {
  int interior[4], edges[4];
};
ItemSplit item_split(const LShard& s, int hz, int lo) {
  const int R = s.slab.R, nit = (s.Ts + R + hz - 1) / hz;
  int ja = s.hl == 0 ? 0 : (s.hl + lo + hz - 1) / hz;
  int jb = nit;
  if (s.hr > 0) {
    const int lim = s.hl + s.g.T_loc - hz;   // j hz + hz - 1 <= hl + T_loc - 1
    jb = lim < 0 ? 0 : lim / hz + 1;
  }
  if (ja > nit) ja = nit;
  if (jb > nit) jb = nit;
  if (jb < ja) jb = ja;
  ItemSplit r;
  const int in[4] = {ja, jb - ja, jb - ja, 0}, ed[4] = {0, ja + (nit - jb), ja, jb - ja};
  for (int i = 0; i < 4; ++i) { r.interior[i] = in[i]; r.edges[i] = ed[i]; }
  return r;
}

// slab args of the dense tensor-core LLSA path ([C][B][H][Ts][D] planes), or false when it does not
// apply (then the caller runs the exchange and the ordinary call)
bool lshard_args(const LShard& s, AttnArgs& a, int& hz) {
  const sattn_desc& l = s.slab;
  if (l.dtype != SATTN_BF16 || l.D != 64 || l.impl == SATTN_IMPL_FFMA || (!s.g.left && !s.g.right)) return false;
  a = AttnArgs{};
  a.T = s.Ts;
  a.L = l.L;
  a.R = l.R;
  a.BH = (int)(l.B * l.H);
  a.scale = desc_scale(&l);
  a.scale_log2 = a.scale * kLog2e;
  a.in_cs = a.out_cs = (long long)a.BH * s.Ts * 64;
  hz = tc_llsa_item_hz(a);
  return hz > 0;
}

}  // namespace

extern "C" {

int64_t sattn_tshard_margin(void) { return kMargin; }

sattn_status sattn_dist_unique_id(void* id_out) {
  if (!id_out) return set_error(SATTN_EARG, "id_out is NULL");
  const NcclApi& n = nccl();
  if (!n.ok) return set_error(SATTN_ENCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  const ncclResult_t r = n.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id_out, &id, sizeof id);
  return SATTN_OK;
}

sattn_status sattn_dist_init(int rank, int world, const void* nccl_unique_id, sattn_dist** out) {
  if (!out) return set_error(SATTN_EARG, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return set_error(SATTN_EARG, "bad rank / world");
  if (world > 1 && !nccl_unique_id) return set_error(SATTN_EARG, "nccl_unique_id is NULL");
  sattn_dist* d = new (std::nothrow) sattn_dist{};
  if (!d) return set_error(SATTN_ECUDA, "out of host memory");
  d->rank = rank;
  d->world = world;
  cudaError_t e = cudaStreamCreateWithFlags(&d->cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    sattn_dist_destroy(d);
    return cuda_fail("dist stream / events", e);
  }
  if (world > 1) {
    const NcclApi& n = nccl();
    if (!n.ok) {
      sattn_dist_destroy(d);
      return set_error(SATTN_ENCCL, "libnccl.so.2 not found");
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    const ncclResult_t r = n.CommInitRank(&d->comm, world, id, rank);
    if (r != ncclSuccess) {
      d->comm = nullptr;
      sattn_dist_destroy(d);
      return nccl_fail("ncclCommInitRank", r);
    }
  }
  *out = d;
  return SATTN_OK;
}

sattn_status sattn_dist_init_external(int rank, int world, sattn_exchange_fn fn, void* user, sattn_dist** out) {
  if (!out) return set_error(SATTN_EARG, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return set_error(SATTN_EARG, "bad rank / world");
  if (!fn) return set_error(SATTN_EARG, "exchange callback is NULL");
  sattn_dist* d = new (std::nothrow) sattn_dist{};
  if (!d) return set_error(SATTN_ECUDA, "out of host memory");
  d->rank = rank;
  d->world = world;
  d->fn = fn;
  d->user = user;
  *out = d;
  return SATTN_OK;
}

void sattn_dist_destroy(sattn_dist* d) {
  if (!d) return;
  if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
  if (d->ev_in) cudaEventDestroy(d->ev_in);
  if (d->ev_halo) cudaEventDestroy(d->ev_halo);
  if (d->cs) cudaStreamDestroy(d->cs);
  delete d;
}

size_t sa_tsharded_workspace(const sattn_tshard_desc* td, const sattn_dist* d) {
  Shard s;
  if (shard_setup(td, d, s) != SATTN_OK) return 0;
  HaloT f[3], b[1];
  fwd_halos(s, nullptr, nullptr, nullptr, f);
  bwd_halos(s, nullptr, b);
  const size_t wf = halo_ws(s, f, 3), wb = halo_ws(s, b, 1) + bwd_rows_ws(s);
  return wf > wb ? wf : wb;
}

sattn_status sa_forward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                 float* LSE, void* ws, size_t ws_bytes, void* stream) {
  Shard s;
  sattn_status r = shard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !LSE) return set_error(SATTN_EARG, "NULL pointer");
  HaloT h[3];
  fwd_halos(s, Q, K, V, h);
  const size_t need = halo_ws(s, h, 3);
  if (need && (!ws || ws_bytes < need)) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  // NCCL: the exchange is enqueued first (on the dist stream) so it overlaps the interior tiles;
  // external transport: interior tiles first, then the (synchronous) exchange on `st`
  const bool ext = d->comm == nullptr;
  if (!ext && (r = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return r;
  s.a.Q = at(Q, s.off); s.a.K = at(K, s.off); s.a.V = at(V, s.off);
  s.a.Out = at(O, s.off);
  s.a.LSEout = LSE + (kMargin - s.hl);
  const int nk = tc_key_box_rows(s.a.L, s.a.R);
  return split_run(d, s, nk, st, true, [&](const AttnArgs& a, bool interior) -> sattn_status {
    sattn_status rr;
    if (!interior && ext && (rr = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return rr;
    if ((rr = tc_forward(a, st)) != SATTN_OK) return set_error(rr, tc_last_error());
    count_launches(1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded forward launch", e);
  });
}

sattn_status sa_backward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                  const void* V, const float* LSE, void* dO, void* dQ, void* dK, void* dV, void* ws,
                                  size_t ws_bytes, void* stream) {
  Shard s;
  sattn_status r = shard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !LSE || !dO || !dQ || !dK || !dV || !ws) return set_error(SATTN_EARG, "NULL pointer");
  HaloT h[1];
  bwd_halos(s, dO, h);
  const size_t nh = halo_ws(s, h, 1), nrows = bwd_rows_ws(s);
  if (ws_bytes < nh + nrows) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const bool ext = d->comm == nullptr;
  if (!ext && (r = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return r;
  s.a.Q = at(Q, s.off); s.a.K = at(K, s.off); s.a.V = at(V, s.off);
  s.a.dO = at(dO, s.off);
  s.a.LSE = LSE + (kMargin - s.hl);
  s.a.dQ = at(dQ, s.off); s.a.dK = at(dK, s.off); s.a.dV = at(dV, s.off);
  s.a.delta = reinterpret_cast<float*>((char*)ws + nh);
  const int nk = tc_key_box_rows(s.a.L, s.a.R);
  r = split_run(d, s, nk, st, true, [&](const AttnArgs& a, bool interior) -> sattn_status {
    sattn_status rr;
    if (!interior && ext && (rr = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return rr;
    if ((rr = tc_backward_phase(a, st, 1)) != SATTN_OK) return set_error(rr, tc_last_error());
    count_launches(1);
    return SATTN_OK;
  });
  if (r != SATTN_OK) return r;
  if ((r = tc_backward_phase(s.a, st, 2)) != SATTN_OK) return set_error(r, tc_last_error());
  count_launches(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded backward launch", e);
}

int64_t llsa_tshard_margin(int32_t L, int32_t R) { return llsa_tshard_margin_of(L, R); }

size_t llsa_tsharded_workspace(const sattn_tshard_desc* td, const sattn_dist* d) {
  LShard s;
  if (lshard_setup(td, d, s) != SATTN_OK) return 0;
  const int mg = llsa_tshard_margin_of(s.slab.L, s.slab.R);
  const HaloT f[3] = {{nullptr, mg, mg}, {nullptr, mg, mg}, {nullptr, mg, mg}};
  const HaloT b[1] = {{nullptr, s.slab.R, s.slab.L + s.slab.R}};
  const size_t wf = halo_ws(s.g, f, 3);
  const size_t wb = halo_ws(s.g, b, 1) + ((llsa_backward_workspace(&s.slab) + 255) & ~size_t(255));
  return wf > wb ? wf : wb;
}

sattn_status llsa_forward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                   float* LSE, void* ws, size_t ws_bytes, void* stream) {
  LShard s;
  sattn_status r = lshard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !LSE) return set_error(SATTN_EARG, "NULL pointer");
  const int mg = llsa_tshard_margin_of(s.slab.L, s.slab.R);
  const HaloT h[3] = {{(char*)Q, mg, mg}, {(char*)K, mg, mg}, {(char*)V, mg, mg}};
  const size_t need = halo_ws(s.g, h, 3);
  if (need && (!ws || ws_bytes < need)) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  AttnArgs a;
  int hz = 0;
  if (lshard_args(s, a, hz)) {
    // the interior items overlap the exchange (NCCL: it runs on the dist stream; a caller transport
    // runs synchronously on `st` after the interior launch), the edge items follow the halo
    a.Q = Q; a.K = K; a.V = V; a.Out = O; a.LSEout = LSE;
    const ItemSplit sp = item_split(s, hz, s.slab.R + s.slab.L);
    const bool ext = d->comm == nullptr;
    if (!ext && (r = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return r;
    if (sp.interior[1] > 0) {
      if ((r = tc_llsa_forward_items(a, sp.interior, st)) != SATTN_OK) return set_error(r, tc_llsa_last_error());
      count_launches(1);
    }
    if (ext && (r = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return r;
    if (!ext) {
      const cudaError_t e = cudaStreamWaitEvent(st, d->ev_halo, 0);
      if (e != cudaSuccess) return cuda_fail("cudaStreamWaitEvent", e);
    }
    if (sp.edges[1] > 0) {
      if ((r = tc_llsa_forward_items(a, sp.edges, st)) != SATTN_OK) return set_error(r, tc_llsa_last_error());
      count_launches(1);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded LLSA forward launch", e);
  }
  if ((r = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return r;
  if (d->comm) {
    const cudaError_t e = cudaStreamWaitEvent(st, d->ev_halo, 0);
    if (e != cudaSuccess) return cuda_fail("cudaStreamWaitEvent", e);
  }
  return llsa_forward(&s.slab, Q, K, V, O, LSE, stream);
}

sattn_status llsa_backward_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                    const void* V, const void* O, const float* LSE, void* dO, void* dQ, void* dK,
                                    void* dV, void* ws, size_t ws_bytes, void* stream) {
  LShard s;
  sattn_status r = lshard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !LSE || !dO || !dQ || !dK || !dV || !ws) return set_error(SATTN_EARG, "NULL pointer");
  const HaloT h[1] = {{(char*)dO, s.slab.R, s.slab.L + s.slab.R}};
  const size_t nh = halo_ws(s.g, h, 1);
  const size_t nb = llsa_backward_workspace(&s.slab);
  if (ws_bytes < nh + nb) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  AttnArgs a;
  int hz = 0;
  if (lshard_args(s, a, hz)) {
    // the fused pass's interior items overlap the dO exchange; its edge items and the kv pass follow
    a.Q = Q; a.K = K; a.V = V; a.O = O; a.LSE = LSE; a.dO = dO;
    a.dQ = dQ; a.dK = dK; a.dV = dV;
    a.delta = reinterpret_cast<float*>((char*)ws + nh);
    const ItemSplit sp = item_split(s, hz, s.slab.R);
    const bool ext = d->comm == nullptr;
    if (!ext && (r = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return r;
    if (sp.interior[1] > 0) {
      if ((r = tc_llsa_backward_phase(a, st, 1, sp.interior)) != SATTN_OK) return set_error(r, tc_last_error());
      count_launches(1);
    }
    if (ext && (r = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return r;
    if (!ext) {
      const cudaError_t e = cudaStreamWaitEvent(st, d->ev_halo, 0);
      if (e != cudaSuccess) return cuda_fail("cudaStreamWaitEvent", e);
    }
    if (sp.edges[1] > 0) {
      if ((r = tc_llsa_backward_phase(a, st, 1, sp.edges)) != SATTN_OK) return set_error(r, tc_last_error());
      count_launches(1);
    }
    if ((r = tc_llsa_backward_phase(a, st, 2, nullptr)) != SATTN_OK) return set_error(r, tc_last_error());
    count_launches(1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded LLSA backward launch", e);
  }
  if ((r = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return r;
  if (d->comm) {
    const cudaError_t e = cudaStreamWaitEvent(st, d->ev_halo, 0);
    if (e != cudaSuccess) return cuda_fail("cudaStreamWaitEvent", e);
  }
  return llsa_backward(&s.slab, Q, K, V, O, LSE, dO, dQ, dK, dV, (char*)ws + nh, ws_bytes - nh, stream);
}

// ------------------------------------------------------------------------------------------
// The stored-band mode (the paper's a_t) on the same margined shards: the forward exchanges
// K, V, Q as above and writes the band rows of the whole slab (the halo rows' a_t are exact for the
// same reason their LSE is); the backward exchanges dO only, K1 forms the halo queries' delta =
// rowsum(P o dP) from the margins (G26), K2 reads the band window.  P is margined like the other
// tensors: [B][H][M + T + M][sa_p_ld(desc)].
// ------------------------------------------------------------------------------------------
sattn_status sa_forward_p_tsharded(const sattn_tshard_desc* td, sattn_dist* d, void* Q, void* K, void* V, void* O,
                                   float* LSE, void* P, void* ws, size_t ws_bytes, void* stream) {
  Shard s;
  sattn_status r = shard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !O || !LSE || !P) return set_error(SATTN_EARG, "NULL pointer");
  if (!tc_p_supported(td->local.dtype, (int)td->local.D, td->local.L, td->local.R, true))
    return set_error(SATTN_EUNSUPPORTED, "time-sharded stored-band SA needs L + R + 1 <= 49");
  HaloT h[3];
  fwd_halos(s, Q, K, V, h);
  const size_t need = halo_ws(s, h, 3);
  if (need && (!ws || ws_bytes < need)) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const bool ext = d->comm == nullptr;
  if (!ext && (r = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return r;
  const int ldp = (s.a.L + s.a.R + 1 + 7) & ~7;
  s.a.Q = at(Q, s.off); s.a.K = at(K, s.off); s.a.V = at(V, s.off);
  s.a.Out = at(O, s.off);
  s.a.LSEout = LSE + (kMargin - s.hl);
  s.a.P = at(P, (long long)(kMargin - s.hl) * ldp);
  s.a.ldp = ldp;
  const int nk = tc_key_box_rows(s.a.L, s.a.R);
  return split_run(d, s, nk, st, true, [&](const AttnArgs& a, bool interior) -> sattn_status {
    sattn_status rr;
    if (!interior && ext && (rr = exchange(d, s.g, h, 3, (char*)ws, st)) != SATTN_OK) return rr;
    if ((rr = tc_forward_p(a, st)) != SATTN_OK) return set_error(rr, tc_last_error());
    count_launches(1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded stored-band forward launch", e);
  });
}

sattn_status sa_backward_p_tsharded(const sattn_tshard_desc* td, sattn_dist* d, const void* Q, const void* K,
                                    const void* V, const void* P, void* dO, void* dQ, void* dK, void* dV, void* ws,
                                    size_t ws_bytes, void* stream) {
  Shard s;
  sattn_status r = shard_setup(td, d, s);
  if (r != SATTN_OK) return r;
  if (!Q || !K || !V || !P || !dO || !dQ || !dK || !dV || !ws) return set_error(SATTN_EARG, "NULL pointer");
  if (!tc_p_supported(td->local.dtype, (int)td->local.D, td->local.L, td->local.R, true))
    return set_error(SATTN_EUNSUPPORTED, "time-sharded stored-band SA needs L + R + 1 <= 49");
  HaloT h[1];
  bwd_halos(s, dO, h);
  const size_t nh = halo_ws(s, h, 1), nrows = bwd_rows_ws(s);
  if (ws_bytes < nh + nrows) return set_error(SATTN_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const bool ext = d->comm == nullptr;
  if (!ext && (r = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return r;
  const int ldp = (s.a.L + s.a.R + 1 + 7) & ~7;
  s.a.Q = at(Q, s.off); s.a.K = at(K, s.off); s.a.V = at(V, s.off);
  s.a.dO = at(dO, s.off);
  s.a.P = const_cast<bf16*>(at(P, (long long)(kMargin - s.hl) * ldp));
  s.a.ldp = ldp;
  s.a.dQ = at(dQ, s.off); s.a.dK = at(dK, s.off); s.a.dV = at(dV, s.off);
  s.a.delta = reinterpret_cast<float*>((char*)ws + nh);
  const int nk = tc_key_box_rows(s.a.L, s.a.R);
  r = split_run(d, s, nk, st, true, [&](const AttnArgs& a, bool interior) -> sattn_status {
    sattn_status rr;
    if (!interior && ext && (rr = exchange(d, s.g, h, 1, (char*)ws, st)) != SATTN_OK) return rr;
    if ((rr = tc_backward_p_phase(a, st, 1)) != SATTN_OK) return set_error(rr, tc_last_error());
    count_launches(1);
    return SATTN_OK;
  });
  if (r != SATTN_OK) return r;
  if ((r = tc_backward_p_phase(s.a, st, 2)) != SATTN_OK) return set_error(r, tc_last_error());
  count_launches(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SATTN_OK : cuda_fail("time-sharded stored-band backward launch", e);
}

// host-only geometry of a shard (for tests and tooling): slab rows and the tile split
sattn_status sattn_tshard_geometry(const sattn_tshard_desc* td, int rank, int world, int64_t* out6) {
  if (!out6) return set_error(SATTN_EARG, "out is NULL");
  sattn_dist d{};
  d.rank = rank;
  d.world = world;
  Shard s;
  sattn_status r = shard_setup(td, &d, s);
  if (r != SATTN_OK) return r;
  const Tiles t = tile_split(s.hl, s.g.T_loc, s.hr, s.a.L, tc_key_box_rows(s.a.L, s.a.R));
  out6[0] = s.hl; out6[1] = s.hr; out6[2] = s.Ts; out6[3] = t.ntq; out6[4] = t.e0; out6[5] = t.e1;
  return SATTN_OK;
}

}  // extern "C"
