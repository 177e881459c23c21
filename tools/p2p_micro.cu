// p2p_micro.cu — ceiling of the P2P inner loop's instruction mix on the B200: every warp holds 64
// targets (2 per lane, packed) and sweeps a shared-memory tile of sources again and again (no
// global traffic, no list walking), the exact pair code of p2p_core.cuh. Prints pairs/s and the
// fraction of the FP32 peak at 19 flop/pair for several warps-per-SM and slice counts.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1108_5815_b200/csrc/p2p_core.cuh"

template <int S, int U>
__global__ void __launch_bounds__(128) k_micro(int reps, int ns, float4 *out) {
  __shared__ __align__(16) float4 sp[1024];
  for (int j = threadIdx.x; j < ns; j += blockDim.x)
    sp[j] = make_float4(0.001f * j, 0.37f + 0.0007f * j, 0.11f * (j & 7), 1e-3f);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int h = lane % S;
  const float t = 0.5f + 0.01f * lane;
  const f2x tx = pk(-t, -t - 0.003f), ty = pk(-0.2f, -0.21f), tz = pk(-0.3f, -0.33f);
  f2x acc[4] = {0ull, 0ull, 0ull, 0ull};
  for (int r = 0; r < reps; ++r) {
    if (U == 8)
      p2p_tile_rawS8<false, S>(sp, ns, h, tx, ty, tz, acc);
    else
      p2p_tile_rawS<false, S>(sp, ns, h, tx, ty, tz, acc);
  }
  float2 a = upk(acc[0]), b = upk(acc[1]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = make_float4(a.x, a.y, b.x, b.y);
}

template <int S, int U = 4>
void run(int blocks_per_sm, int ns) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * blocks_per_sm, reps = 200;
  float4 *out;
  cudaMalloc(&out, sizeof(float4) * blocks * 128);
  k_micro<S, U><<<blocks, 128>>>(2, ns, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_micro<S, U><<<blocks, 128>>>(reps, ns, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // pair evaluations: per warp 32 lanes x 2 targets x ns / S sources per rep
  const double pairs = (double)blocks * 4 * 64 * ns / S * reps;
  const double peak = nsm * 128 * 2 * 1.965e9;
  printf("{\"U\": %d, \"S\": %d, \"warps_per_sm\": %d, \"ns\": %d, \"ms\": %.3f, \"pairs_per_s\": %.4g, "
         "\"frac_19flop\": %.4f}\n", U, S, 4 * blocks_per_sm, ns, ms, pairs / (ms * 1e-3),
         pairs * 19 / (ms * 1e-3) / peak);
  cudaFree(out);
}

int main() {
  for (int bps : {2, 3, 4, 5, 6, 8}) run<1>(bps, 1024);
  for (int bps : {2, 3, 4, 5, 6, 8}) run<1, 8>(bps, 1024);
  for (int bps : {4, 6}) run<2>(bps, 1024);
  for (int bps : {4, 6}) run<2, 8>(bps, 1024);
  for (int bps : {4}) run<1>(bps, 128);
  return 0;
}
