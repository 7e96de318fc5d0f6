// Dependent-chain latencies on sm_100a (tool): DFMA, DMUL, LDS.64, rsqrt.approx.f64, bar.sync with 288 threads.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) x = x * 1.0000001;
  long long t2 = clock64();
  int j = threadIdx.x & 1023;
  for (int i = 0; i < 256; ++i) j = idx[j];
  long long t3 = clock64();
  double y = x;
  for (int i = 0; i < 256; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; }
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) __syncthreads();
  long long t5 = clock64();
  double z = 0; for (int i = 0; i < 256; ++i) z = sm[((int)z + i) & 1023] - sm[0] + z * 0.0;
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
    cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256;
  }
  out[threadIdx.x] = x + y + j + z;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 64);
  for (int th : {32, 288}) {
    lat<<<1, th>>>(o, c, 1.0); lat<<<1, th>>>(o, c, 1.0);
    long long h[6]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads=%d: DFMA %lld, DMUL %lld, LDS.32 chain %lld, rsqrt.approx.f64 %lld (+DADD), bar.sync %lld, LDS.64+DADD %lld clk\n",
           th, h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  return 0;
}
