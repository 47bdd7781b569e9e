// FP64 pipe microbenchmark for B200 (sm_100a): throughput of DFMA and of the
// libdevice/IEEE operations the coupled level sampler uses, in thread-ops/s.
// Used once to calibrate the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define ILP 8
template <int OP>
__global__ void bench(double* out, int iters, double seed) {
  double v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = seed + 1e-3 * (threadIdx.x + k) + 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      double x = v[k];
      if (OP == 0) x = fma(x, 0.999999, 1e-7);
      else if (OP == 1) x = 1.0 / x + 0.5;            // div + add
      else if (OP == 2) x = sqrt(x) + 0.25;           // sqrt + add
      else if (OP == 3) x = -log(x) * 0.5 + 0.6;      // log
      else if (OP == 4) { double s, c; sincos(x, &s, &c); x = s * c + 0.7; }
      else if (OP == 5) x = exp(-x) + 0.3;            // exp
      else if (OP == 6) x = -expm1(-x) + 0.3;         // expm1
      else if (OP == 7) x = x * 0.999999;             // dmul
      v[k] = x;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 12345.678) out[0] = s;
}

template <int OP>
double run(const char* name, int iters) {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 grid(sms * 8), block(256);
  bench<OP><<<grid, block>>>(d, 10, 0.1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<OP><<<grid, block>>>(d, iters, 0.1);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(grid.x) * block.x * iters * ILP;
  double rate = ops / (ms * 1e-3);
  printf("%-8s %10.3f ms  %.4e thread-ops/s\n", name, ms, rate);
  cudaFree(d);
  return rate;
}

int main() {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("sms=%d clock_khz=%d\n", sms, clk);
  double fma = run<0>("dfma", 20000);
  printf("dfma lanes/SM/clk at max clock = %.2f\n", fma / (sms * clk * 1e3));
  double r[8];
  r[7] = run<7>("dmul", 20000);
  r[1] = run<1>("div", 2000);
  r[2] = run<2>("sqrt", 2000);
  r[3] = run<3>("log", 1000);
  r[4] = run<4>("sincos", 1000);
  r[5] = run<5>("exp", 1000);
  r[6] = run<6>("expm1", 1000);
  const char* n[] = {"", "div+add", "sqrt+add", "log+2", "sincos+2", "exp+1", "expm1+1", "dmul"};
  for (int i = 1; i < 8; ++i) printf("%-9s ~ %.1f dfma-equivalents\n", n[i], fma / r[i]);
  return 0;
}
