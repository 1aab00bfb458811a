// Microbenchmark: K3 snapshot (fp32 copy) variants at 64M / 100M elements.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o snap snapshot_variants.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U, int LOADMODE, int STOREMODE>
__global__ void __launch_bounds__(256) k(const float* __restrict__ src, float* __restrict__ out, size_t nvec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float4* s = reinterpret_cast<const float4*>(src);
  float4* o = reinterpret_cast<float4*>(out);
  for (size_t i0 = tid; i0 < nvec; i0 += stride * U) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        if (LOADMODE == 0) r[u] = __ldcg(s + i);
        else if (LOADMODE == 1) r[u] = __ldg(s + i);
        else r[u] = __ldcs(s + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = i0 + (size_t)u * stride;
      if (i < nvec) {
        if (STOREMODE == 0) o[i] = r[u];
        else if (STOREMODE == 1) __stcs(o + i, r[u]);
        else __stcg(o + i, r[u]);
      }
    }
  }
}

template <int U, int LM, int SM>
void run(const char* name, const float* a, float* b, size_t n, int blocksPerSM, char* flush, size_t fbytes) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t nvec = n / 4;
  size_t want = (nvec + 255) / 256; size_t cap = (size_t)sms * blocksPerSM;
  unsigned grid = (unsigned)(want < cap ? want : cap);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9, tot = 0; int it = 10;
  for (int w = 0; w < 3; ++w) k<U, LM, SM><<<grid, 256>>>(a, b, nvec);
  for (int i = 0; i < it; ++i) {
    cudaMemsetAsync(flush, i, fbytes);
    cudaEventRecord(e0);
    k<U, LM, SM><<<grid, 256>>>(a, b, nvec);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms; if (ms < best) best = ms;
  }
  double gbs = 8.0 * n / (tot / it * 1e-3) / 1e9;
  printf("%-28s n=%zu bps=%d  avg %.1f us  %.0f GB/s  (best %.0f GB/s)\n", name, n, blocksPerSM, tot / it * 1e3, gbs, 8.0 * n / (best * 1e-3) / 1e9);
}

int main() {
  size_t n = 100000000;
  float *a, *b; char* fl; size_t fb = 256u << 20;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&fl, fb);
  cudaMemset(a, 1, n * 4);
  // spin clocks up
  for (int i = 0; i < 200; ++i) k<4, 0, 0><<<1184, 256>>>(a, b, n / 4);
  cudaDeviceSynchronize();
  for (size_t nn : {64000000ul, 100000000ul}) {
    run<4, 0, 0>("cg/default U4", a, b, nn, 8, fl, fb);
    run<4, 0, 1>("cg/cs U4", a, b, nn, 8, fl, fb);
    run<4, 0, 2>("cg/cg U4", a, b, nn, 8, fl, fb);
    run<4, 1, 0>("ldg/default U4", a, b, nn, 8, fl, fb);
    run<4, 2, 1>("cs/cs U4", a, b, nn, 8, fl, fb);
    run<8, 0, 0>("cg/default U8", a, b, nn, 8, fl, fb);
    run<8, 0, 1>("cg/cs U8", a, b, nn, 8, fl, fb);
    run<2, 0, 0>("cg/default U2", a, b, nn, 8, fl, fb);
    run<4, 0, 0>("cg/default U4 bps4", a, b, nn, 4, fl, fb);
    run<8, 0, 0>("cg/default U8 bps4", a, b, nn, 4, fl, fb);
    run<4, 0, 0>("cg/default U4 bps16", a, b, nn, 16, fl, fb);
  }
  // cudaMemcpy reference
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float tot = 0;
  for (int i = 0; i < 10; ++i) { cudaMemsetAsync(fl, i, fb); cudaEventRecord(e0); cudaMemcpyAsync(b, a, n * 4, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms; }
  printf("cudaMemcpyD2D n=%zu avg %.1f us %.0f GB/s\n", n, tot / 10 * 1e3, 8.0 * n / (tot / 10 * 1e-3) / 1e9);
  return 0;
}
