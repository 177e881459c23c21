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
  // every accumulator reaches the output (else the compiler drops the unused pair arithmetic)
  const float2 a = upk(acc[0]), b = upk(acc[1]), c = upk(acc[2]), d = upk(acc[3]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = make_float4(a.x + a.y, b.x + b.y, c.x + c.y, d.x + d.y);
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

// four targets per lane (two packed pairs), U sources per unrolled step
#ifndef QUAD_MINB
#define QUAD_MINB 4
#endif
template <int S, int U>
__global__ void __launch_bounds__(128, QUAD_MINB) k_micro_quad(int reps, int ns, float4 *out) {
  __shared__ __align__(16) float4 sp[1024];
  for (int j = threadIdx.x; j < ns; j += blockDim.x)
    sp[j] = make_float4(0.001f * j, 0.37f + 0.0007f * j, 0.11f * (j & 7), 1e-3f);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int h = lane % S;
  const float t = 0.5f + 0.01f * lane;
  const f2x tt[6] = {pk(-t, -t - 0.003f), pk(-0.2f, -0.21f), pk(-0.3f, -0.33f),
                     pk(-t - 0.01f, -t - 0.013f), pk(-0.22f, -0.23f), pk(-0.31f, -0.34f)};
  f2x acc[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  for (int r = 0; r < reps; ++r) p2p_tile_quad<false, S, U>(sp, ns, h, tt, acc);
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float2 u = upk(acc[c]), v = upk(acc[4 + c]);
    (&o.x)[c] = u.x + u.y + v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = o;
}

template <int S, int U>
void run_quad(int blocks_per_sm, int ns, int threads = 128) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * blocks_per_sm, reps = 200;
  float4 *out;
  cudaMalloc(&out, sizeof(float4) * blocks * 128);
  k_micro_quad<S, U><<<blocks, 128>>>(2, ns, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_micro_quad<S, U><<<blocks, 128>>>(reps, ns, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double pairs = (double)blocks * 4 * 128 * ns / S * reps;
  const double peak = nsm * 128 * 2 * 1.965e9;
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_micro_quad<S, U>) == cudaSuccess) regs = fa.numRegs;
  printf("{\"quad\": 1, \"U\": %d, \"S\": %d, \"regs\": %d, \"warps_per_sm\": %d, \"ns\": %d, \"ms\": %.3f, "
         "\"pairs_per_s\": %.4g, \"frac_19flop\": %.4f}\n", U, S, regs, 4 * blocks_per_sm, ns, ms,
         pairs / (ms * 1e-3), pairs * 19 / (ms * 1e-3) / peak);
  cudaFree(out);
}

int main() {
  for (int bps : {2, 3, 4, 5, 6, 8}) run_quad<1, 2>(bps, 1024);
  for (int bps : {2, 3, 4, 5, 6, 8}) run_quad<1, 4>(bps, 1024);
  for (int bps : {4, 6}) run_quad<2, 2>(bps, 1024);
  for (int bps : {4}) run_quad<4, 2>(bps, 1024);
  for (int bps : {2, 3, 4, 5, 6, 8}) run<1>(bps, 1024);
  for (int bps : {2, 3, 4, 5, 6, 8}) run<1, 8>(bps, 1024);
  for (int bps : {4, 6}) run<2>(bps, 1024);
  for (int bps : {4, 6}) run<2, 8>(bps, 1024);
  for (int bps : {4}) run<1>(bps, 128);
  return 0;
}
