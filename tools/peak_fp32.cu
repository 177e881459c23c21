// peak_fp32.cu — FP32 CUDA-core ceiling microbenchmark on the B200:
// FFMA (scalar), FFMA2 (packed f32x2) and MUFU.RSQ throughput over all SMs, timed with events,
// plus the clock (clock64 delta / event time). Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
__global__ void k_ffma(float *out, float a, float b, long long *clk) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma2(float *out, float a, float b, long long *clk) {
  float2 x[8];
  for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x + k, threadIdx.x - k);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(x[j], A, B);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND>  // 0 FADD2, 1 FMUL2, 2 mix 5 FFMA2 : 4 FADD2 : 4 FMUL2 (the P2P ratio)
__global__ void k_pk(float *out, float a, float b, long long *clk) {
  float2 x[8];
  for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x + k, threadIdx.x - k);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (KIND == 0) x[j] = __fadd2_rn(x[j], B);
        else if (KIND == 1) x[j] = __fmul2_rn(x[j], A);
        else {
          const int r = (k * 8 + j) % 13;
          x[j] = r < 5 ? __ffma2_rn(x[j], A, B) : r < 9 ? __fadd2_rn(x[j], B) : __fmul2_rn(x[j], A);
        }
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_rsq(float *out, long long *clk) {
  float x0 = threadIdx.x + 1.f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = rsqrtf(x0); x1 = rsqrtf(x1); x2 = rsqrtf(x2); x3 = rsqrtf(x3);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

int main() {
  int dev = 0, nsm = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int blocks = nsm * 4, threads = 512;
  float *out; long long *clk, hclk;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&clk, sizeof(long long));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double res[6][2];
  for (int which = 0; which < 6; ++which) {
    float best = 1e30f; long long bclk = 0;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (which == 0) k_ffma<<<blocks, threads>>>(out, 0.999f, 0.001f, clk);
      else if (which == 1) k_ffma2<<<blocks, threads>>>(out, 0.999f, 0.001f, clk);
      else if (which == 2) k_rsq<<<blocks, threads>>>(out, clk);
      else if (which == 3) k_pk<0><<<blocks, threads>>>(out, 0.999f, 0.001f, clk);
      else if (which == 4) k_pk<1><<<blocks, threads>>>(out, 0.999f, 0.001f, clk);
      else k_pk<2><<<blocks, threads>>>(out, 0.999f, 0.001f, clk);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&hclk, clk, sizeof hclk, cudaMemcpyDeviceToHost);
      if (rep > 0 && ms < best) { best = ms; bclk = hclk; }
    }
    double ops = (double)blocks * threads * ITERS * (which == 0 ? 64 : which == 2 ? 32 : 128);
    double flops = which == 2 ? ops : (which == 3 || which == 4) ? ops : 2.0 * ops;  // lane-ops for 3/4/5
    if (which == 5) flops = ops;  // lane-ops
    res[which][0] = flops / (best * 1e-3) / 1e12;   // TFLOP/s (or T-rsqrt/s)
    res[which][1] = (double)bclk / (best * 1e-3) / 1e6;  // MHz seen by block 0 (approx)
  }
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
         "\"rsqrt_tops\": %.3f, \"fadd2_tlaneops\": %.2f, \"fmul2_tlaneops\": %.2f, "
         "\"p2p_mix_tlaneops\": %.2f, \"fma_lane_peak_tlaneops\": %.2f}\n",
         nsm, clk_khz / 1e3, res[0][0], res[1][0], res[2][0], res[3][0], res[4][0], res[5][0],
         nsm * 128 * clk_khz / 1e9);
  return 0;
}
