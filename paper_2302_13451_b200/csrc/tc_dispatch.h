// tc_dispatch.h — entry points of the tcgen05 (tensor-core) kernel family (tc_sa.cu).
#pragma once
#include <cuda_runtime.h>

#include "sattn.h"

namespace sattn {
struct AttnArgs;
// true when the tensor-core kernels implement this (dtype, D, band, mode)
bool tc_supported(int dtype, int D, int L, int R, bool llsa, bool backward);
sattn_status tc_forward(const AttnArgs& a, cudaStream_t st);
sattn_status tc_backward(const AttnArgs& a, cudaStream_t st);
// phase bit 0: K1 (dQ, delta) over the args' query-tile subset; bit 1: K2 (dK, dV) over every tile
sattn_status tc_backward_phase(const AttnArgs& a, cudaStream_t st, int phase);
int tc_backward_launches();
// wide bands (W > 65) as log-sum-exp-merged sub-bands of the narrow tensor-core kernels
bool tc_wide_supported(int dtype, int D, int L, int R);
int tc_wide_parts(int L, int R);
size_t tc_wide_fwd_ws(long long BH, long long T);
size_t tc_wide_bwd_ws(long long BH, long long T);
sattn_status tc_forward_wide(const AttnArgs& a, void* ws, cudaStream_t st);
sattn_status tc_backward_wide(const AttnArgs& a, cudaStream_t st);
int tc_key_box_rows(int L, int R);   // rows of the K / V box a query tile loads (NK)
size_t tc_backward_ws_bytes();
bool tc_p_supported(int dtype, int D, int L, int R, bool backward);   // stored-band mode (NEXT-4)
// stored-band backward for W > 49: 48-column sub-bands of a_t on the tensor-core kernels (workspace
// tc_wide_bwd_ws; needs O for delta = dO . O)
sattn_status tc_backward_p_wide(const AttnArgs& a, cudaStream_t st);
// the stored-band backward in phases (bit 0: K1 over the launch's query tiles, bit 1: K2), for time shards
sattn_status tc_backward_p_phase(const AttnArgs& a, cudaStream_t st, int phase);
int tc_wide_p_parts(int L, int R);
sattn_status tc_forward_p(const AttnArgs& a, cudaStream_t st);
sattn_status tc_backward_p(const AttnArgs& a, cudaStream_t st);   // SA tensor-core backward: CTA hand-off rows (fused sweep)
const char* tc_last_error();
void tc_set_trace(void* p);  // debug only
// tensor-core LLSA forward (tc_llsa.cu)
bool tc_llsa_supported(int dtype, int D, int L, int R);
bool tc_llsa_fwd_any_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense);
sattn_status tc_llsa_forward(const AttnArgs& a, cudaStream_t st);
const char* tc_llsa_last_error();
void tc_llsa_set_trace(void* p);  // debug only
bool tc_llsa_bwd_supported(int dtype, int D, int L, int R);
sattn_status tc_llsa_backward(const AttnArgs& a, cudaStream_t st);
int tc_llsa_backward_launches(const AttnArgs& a);
bool tc_llsa_bwd_any_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense);
bool tc_llsa_bwd_fused_supported(int dtype, int D, int L, int R, long long BH, long long T, bool dense);
// ws_flat: delta / LSE rows as [C][BH*T rounded to 4] (the packed-tile kv pass) instead of [C][BH][Tp]
// sub4 (or null = all items): it0, nit_l, it_split, it_jump — the items of this launch per (b, h)
sattn_status tc_llsa_bwd_fused(const AttnArgs& a, float* ws_del, float* ws_l2, int ws_flat, cudaStream_t st,
                               const int* sub4 = nullptr);
// time-shard phases of the dense LLSA path: HZ of the item form (0: not available), the item-form
// forward over an item subset, the backward in phases (bit 0: the fused pass over the item subset
// sub4, bit 1: the key-major kv pass); tc_llsa_backward = phases 3 over all items
int tc_llsa_item_hz(const AttnArgs& a);
sattn_status tc_llsa_forward_items(const AttnArgs& a, const int* sub4, cudaStream_t st);
sattn_status tc_llsa_backward_phase(const AttnArgs& a, cudaStream_t st, int phase, const int* sub4);
}  // namespace sattn
