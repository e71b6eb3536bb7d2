// Microbenchmark 3: per-SM TMA box throughput vs number of issuing warps (each with its own ring)
// and swizzle mode.  L2-resident tensor (argv[1] heads x 1792 x 128 B).  Debug aid, not product code.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.b32 %0,1,0,P;\n}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}
// P producer warps (lane 0 each), ring of NS stages per producer; the consumer is the mbarrier wait itself
__global__ void __launch_bounds__(256, 1) ingest(const __grid_constant__ CUtensorMap tm, int rows, int NS, int P, int ntiles_total, int T, long long* cyc, int lanes) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int SB = rows * 128;
  uint64_t* full = (uint64_t*)(sm + P * NS * SB);
  const int w = lanes ? (threadIdx.x < 32 ? threadIdx.x : 99) : (threadIdx.x >> 5);
  const int lane = lanes ? 0 : (threadIdx.x & 31);
  if (threadIdx.x == 0) { for (int i = 0; i < P * NS; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int ntq = T / 128;
  const int me = (ntiles_total - 1 - blockIdx.x) / gridDim.x + 1;
  long long t0 = clock64();
  if (w < P && lane == 0) {
    for (int k = w; k < me; k += P) {
      const int kk = k / P;                 // this producer's k-th tile
      const int st = kk % NS;
      uint64_t* b = &full[w * NS + st];
      if (kk >= NS) while (!try_wait(b, ((kk - NS) / NS) & 1)) {}
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / ntq, r0 = (g % ntq) * 128;
      expect_tx(b, SB);
      tma3(sm + (w * NS + st) * SB, &tm, b, 0, r0, bh);
    }
    // drain
    const int n = (me - w + P - 1) / P;
    for (int kk = (n > NS ? n - NS : 0); kk < n; ++kk) { uint64_t* b = &full[w * NS + kk % NS]; while (!try_wait(b, (kk / NS) & 1)) {} }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

// convergent mode: warp 0's lanes 0..P-1 issue one box each of the same stage (one barrier per stage)
__global__ void __launch_bounds__(256, 1) ingest_conv(const __grid_constant__ CUtensorMap tm, int rows, int NS, int P, int ntiles_total, int T, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int SB = rows * 128;
  uint64_t* full = (uint64_t*)(sm + P * NS * SB);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int ntq = T / 128;
  const int me = (ntiles_total - 1 - blockIdx.x) / gridDim.x + 1;
  const int ngroups = (me + P - 1) / P;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int kk = 0; kk < ngroups; ++kk) {
      const int st = kk % NS;
      uint64_t* b = &full[st];
      if (kk >= NS) while (!try_wait(b, ((kk - NS) / NS) & 1)) {}
      const int nb = min(P, me - kk * P);
      if (lane == 0) expect_tx(b, nb * SB);
      __syncwarp();
      if (lane < nb) {
        const int k = kk * P + lane;
        const int g = blockIdx.x + k * gridDim.x;
        const int bh = g / ntq, r0 = (g % ntq) * 128;
        tma3(sm + (st * P + lane) * SB, &tm, b, 0, r0, bh);
      }
      __syncwarp();
    }
    for (int kk = (ngroups > NS ? ngroups - NS : 0); kk < ngroups; ++kk) { uint64_t* b = &full[kk % NS]; while (!try_wait(b, (kk / NS) & 1)) {} }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  const int BH = argc > 1 ? atoi(argv[1]) : 96, T = 1792;
  size_t bytes = (size_t)BH * T * 128;
  void* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  long long* cyc; cudaMalloc(&cyc, 148 * sizeof(long long));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ntiles = BH * (T / 128);
  for (int lanes : {0, 2}) for (int sw : {1}) for (int rows : {128, 176}) for (int P : {1, 2, 4, 6}) for (int NS : {2}) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)BH};
    cuuint64_t str[2] = {128, (cuuint64_t)T * 128};
    cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    size_t smem = 1024 + (size_t)P * NS * rows * 128 + 512;
    if (smem > 232448) continue;
    cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(ingest_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) { if (lanes == 2) ingest_conv<<<nsm, 256, smem>>>(tm, rows, NS, P, ntiles, T, cyc); else ingest<<<nsm, 256, smem>>>(tm, rows, NS, P, ntiles, T, cyc, lanes); }
    cudaDeviceSynchronize();
    std::vector<long long> h(nsm); cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost);
    double mc = 0; for (auto c : h) mc += c; mc /= nsm;
    double tb = (double)ntiles * rows * 128;
    printf("lanes %d swz %d rows %3d producers %d NS %d: %.1f B/cyc/SM  (%.0f cyc per box per SM) err=%s\n", lanes, sw, rows, P, NS, tb / nsm / mc,
           mc / ((double)ntiles / nsm), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
