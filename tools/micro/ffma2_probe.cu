// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) issue / FLOP throughput: 8 (or 8
// packed) independent dependent chains per thread, 148 x 8 CTAs x 256.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float v[8];
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x * 1e-7f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = fmaf(v[k], a, b);
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 1234.5f) out[blockIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float a, float b) {
  unsigned long long v[8];
  float2 ab = make_float2(a, a), bb = make_float2(b, b);
  const unsigned long long A = *reinterpret_cast<unsigned long long*>(&ab);
  const unsigned long long B = *reinterpret_cast<unsigned long long*>(&bb);
  for (int k = 0; k < 8; ++k) {
    float2 t = make_float2(threadIdx.x * 1e-7f + k, k + 0.5f);
    v[k] = *reinterpret_cast<unsigned long long*>(&t);
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(A), "l"(B));
  float s = 0.f;
  for (int k = 0; k < 8; ++k) {
    float2 t = *reinterpret_cast<float2*>(&v[k]);
    s += t.x + t.y;
  }
  if (s == 1234.5f) out[blockIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * sizeof(float));
  const int iters = 4000, blocks = 148 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pass = 0; pass < 2; ++pass) {
    for (int which = 0; which < 2; ++which) {
      cudaEventRecord(a);
      if (which == 0) k_ffma<<<blocks, 256>>>(out, iters, 0.999999f, 1e-6f);
      else k_ffma2<<<blocks, 256>>>(out, iters, 0.999999f, 1e-6f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double instr = double(blocks) * 256 / 32 * iters * 128;   // warp instructions
      const double flops = double(blocks) * 256 * iters * 128 * 2 * (which ? 2 : 1);
      if (pass) printf("%s: %.3f ms, %.1f TFLOP/s, %.2f warp-instr/clk/SM\n", which ? "FFMA2" : "FFMA ", ms,
                       flops / ms / 1e9, instr / (ms * 1e-3) / 1.965e9 / 148);
    }
  }
  return 0;
}
