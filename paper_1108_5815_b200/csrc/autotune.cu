// autotune.cu — artificial inputs for the kernel pre-calculation ("All kernels are
// evaluated using artificial coordinates, mass/charges, multipole coefficients").
// A counter-based hash (SplitMix64-style finaliser) so the synthetic set is reproducible.
#include "common.cuh"
#include "kernels.cuh"

__global__ void k_fill_random(float *dst, int64_t n, unsigned seed, float lo, float hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i + 0x9e3779b97f4a7c15ull * (uint64_t)(seed + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const float u = (float)(z >> 40) * (1.0f / 16777216.0f);  // [0, 1)
    dst[i] = lo + (hi - lo) * u;
  }
}

void launch_fill_random(float *dst, int64_t n, unsigned seed, float lo, float hi,
                        cudaStream_t st) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  k_fill_random<<<(int)(b < 1 ? 1 : b), 256, 0, st>>>(dst, n, seed, lo, hi);
}

// ---- per-device one-time setup (common.cuh) ----------------------------------------------------
#include <map>
#include <mutex>
#include <utility>

static std::mutex g_once_mu;

void fmm_smem_optin(const void *func, size_t bytes) {
  if (bytes == 0) return;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_once_mu);
  size_t &have = done[{func, dev}];
  if (have >= bytes) return;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
      cudaSuccess)
    have = bytes;
}

bool fmm_once_per_device(const void *key, bool (*fn)()) {
  static std::map<std::pair<const void *, int>, bool> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_once_mu);
  bool &ok = done[{key, dev}];
  if (!ok) ok = fn();
  return ok;
}

int fmm_resident_blocks(const void *func, int threads, size_t smem) {
  static std::map<std::pair<const void *, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_once_mu);
  int &r = cache[{func, dev}];
  if (!r) {
    int per_sm = 0, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    r = (per_sm > 0 ? per_sm : 1) * nsm;
  }
  return r;
}
