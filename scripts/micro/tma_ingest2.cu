// Microbenchmark: TMA ingest rate per SM (bytes/cycle) vs stages in flight and box size.
// Each CTA (one per SM) streams boxes of `rows` x 128 B from a [BH][T][64] bf16 tensor with an
// NS-deep ring; the consumer releases a stage as soon as it lands.  Debug aid, not product code.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.b32 %0,1,0,P;\n}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}

__global__ void __launch_bounds__(64, 1) ingest(const __grid_constant__ CUtensorMap tm, int rows, int NS, int ntiles_total,
                                                 int T, int split, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int SB = rows * 128;
  uint64_t* full = (uint64_t*)(sm + NS * SB);
  uint64_t* empty = full + NS;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ntq = T / 128;
  const int me = (ntiles_total - 1 - blockIdx.x) / gridDim.x + 1;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int k = 0; k < me; ++k) {
      const int g = blockIdx.x + k * gridDim.x;
      const int bh = g / ntq, r0 = (g % ntq) * 128;
      const int st = k % NS;
      if (k >= NS) while (!try_wait(&empty[st], ((k - NS) / NS) & 1)) {}
      expect_tx(&full[st], SB);
      for (int i = 0; i < split; ++i)
        tma3(sm + st * SB + i * (SB / split), &tm, &full[st], 0, r0 + i * (rows / split), bh);
    }
  } else if (threadIdx.x == 32) {
    for (int k = 0; k < me; ++k) {
      const int st = k % NS;
      while (!try_wait(&full[st], (k / NS) & 1)) {}
      arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  const int BH = argc > 1 ? atoi(argv[1]) : 384, T = 1792;   // 4x the bench tensor: 88 MB (DRAM-ish, > L2 after a flush-ish pass)
  size_t bytes = (size_t)BH * T * 128;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ntiles = BH * (T / 128);
  for (int rows : {128, 176, 256}) {
    for (int split : {1, 2}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)BH};
      cuuint64_t str[2] = {128, (cuuint64_t)T * 128};
      cuuint32_t box[3] = {64, (cuuint32_t)(rows / split), 1}, es[3] = {1, 1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int NS : {1, 2, 3, 4, 6}) {
        size_t smem = 1024 + (size_t)NS * rows * 128 + 256;
        if (smem > 232448) continue;
        cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        ingest<<<nsm, 64, smem>>>(tm, rows, NS, ntiles, T, split, cyc);
        cudaEventRecord(e0);
        ingest<<<nsm, 64, smem>>>(tm, rows, NS, ntiles, T, split, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> h(nsm);
        cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost);
        double mc = 0; for (auto c : h) mc += c; mc /= nsm;
        double tb = (double)ntiles * rows * 128;
        printf("rows %3d split %d NS %d: %.1f us  %.2f TB/s  %.1f B/cyc/SM (kernel-avg %.0f cyc)  err=%s\n", rows, split, NS,
               ms * 1e3, tb / (ms * 1e-3) / 1e12, tb / nsm / mc, mc, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
