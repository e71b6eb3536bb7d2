// host_util.h — host-side launch helpers shared by the libsattn.so translation units:
// a per-(pointer, shape, box) cache of TMA tensor maps and a once-per-kernel dynamic shared
// memory opt-in, so an eager (not graph-captured) call does not re-encode its tensor maps or
// re-set kernel attributes every time.  Host only.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

namespace sattn {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn tmap_encoder() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  return fn;
}

// cuTensorMapEncodeTiled through a cache keyed by every argument (the map holds only the address
// and the geometry, never the data, so a hit is exact).  Returns the driver's result.
inline CUresult tmap_encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                            const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                            CUtensorMapSwizzle sw, CUtensorMapL2promotion l2) {
  struct Key {
    int dt, rank, sw, l2;
    const void* base;
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5];
  } k;
  std::memset(&k, 0, sizeof k);
  k.dt = dt; k.rank = rank; k.sw = sw; k.l2 = l2; k.base = base;
  for (int i = 0; i < rank; ++i) { k.dims[i] = dims[i]; k.box[i] = box[i]; }
  for (int i = 0; i + 1 < rank; ++i) k.strides[i] = strides[i];
  const std::string key(reinterpret_cast<const char*>(&k), sizeof k);
  static std::mutex mu;
  static std::unordered_map<std::string, CUtensorMap> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *m = it->second;
      return CUDA_SUCCESS;
    }
  }
  EncodeTiledFn enc = tmap_encoder();
  if (!enc) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, sw, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 16384) cache.clear();
    cache.emplace(key, *m);
  }
  return r;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize once per (device, kernel, size).
inline void set_smem_once(const void* f, int bytes) {
  static std::mutex mu;
  static std::unordered_map<std::string, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::string key(reinterpret_cast<const char*>(&f), sizeof f);
  key.append(reinterpret_cast<const char*>(&dev), sizeof dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done[key] = bytes;
}
template <typename F>
inline void set_smem(F* f, size_t bytes) {
  set_smem_once(reinterpret_cast<const void*>(f), (int)bytes);
}

}  // namespace sattn
