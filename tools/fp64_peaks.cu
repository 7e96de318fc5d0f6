// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync m8n8k4 f64) and DFMA throughput,
// plus the dependent-DMMA latency.  Used to fix the FP64 roofline denominator.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456) out[0] = s;
}

template <typename K>
float time_kernel(K k, int blocks, int threads, double* out, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, iters / 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d  max clock %.0f MHz\n", sms, clk / 1e3);
  double* out; CK(cudaMalloc(&out, 8));
  // DMMA throughput: warps per SM sweep
  for (int wps : {4, 8, 16}) {
    int iters = 20000;
    float ms = time_kernel(dmma_loop<8>, sms, 32 * wps, out, iters);
    double flop = 2.0 * 256 * 8 * double(iters) * sms * wps;
    printf("DMMA m8n8k4 NACC=8 warps/SM=%2d : %.2f TFLOP/s  (%.1f flop/clk/SM at max clk)\n", wps, flop / ms / 1e9,
           flop / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    int iters = 20000;
    float ms = time_kernel(dmma_loop<4>, sms * 2, 256, out, iters);
    double flop = 2.0 * 256 * 4 * double(iters) * sms * 2 * 8;
    printf("DMMA m8n8k4 NACC=4 2x256thr/SM : %.2f TFLOP/s\n", flop / ms / 1e9);
  }
  // dependent latency: 1 warp, 1 accumulator
  {
    int iters = 100000;
    float ms = time_kernel(dmma_loop<1>, 1, 32, out, iters);
    printf("DMMA dependent latency: %.1f ns/op (%.1f clk at max clk)\n", ms * 1e6 / iters, ms * 1e-3 / iters * clk * 1e3);
  }
  for (int wps : {8, 16, 32}) {
    int iters = 20000;
    float ms = time_kernel(dfma_loop<8>, sms, 32 * wps, out, iters);
    double flop = 2.0 * 8 * double(iters) * sms * wps * 32;
    printf("DFMA NACC=8 warps/SM=%2d : %.2f TFLOP/s\n", wps, flop / ms / 1e9);
  }
  // sustained DMMA for ~3 s
  {
    int iters = 20000;
    float ms1 = time_kernel(dmma_loop<8>, sms, 256, out, iters);
    int big = int(iters * (3000.0 / ms1));
    float ms = time_kernel(dmma_loop<8>, sms, 256, out, big);
    double flop = 2.0 * 256 * 8 * double(big) * sms * 8;
    printf("DMMA sustained (%.0f ms): %.2f TFLOP/s\n", ms, flop / ms / 1e9);
  }
  return 0;
}
