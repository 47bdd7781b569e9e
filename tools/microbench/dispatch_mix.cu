// Dispatch microbenchmark for B200 (sm_100a): does an FP64 warp-instruction
// hold the SMSP's dispatch port for its 2 pipe cycles (16 FP64 lanes per
// SMSP), or can another pipe's instruction issue in the second cycle?
// Streams of independent DFMA, FFMA and LOP3 chains, alone and interleaved,
// at full occupancy; prints warp-instructions issued per SMSP-cycle.
//   model "2-cycle dispatch": DFMA alone 0.5, DFMA+FFMA 1:1 -> 0.667
//   model "1-cycle dispatch": DFMA alone 0.5, DFMA+FFMA 1:1 -> 1.0
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dm tools/microbench/dispatch_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

#define NCH 8
// ND DFMA, NF FFMA, NL LOP3 per chain step (each its own dependent chain)
template <int ND, int NF, int NL>
__global__ void __launch_bounds__(256) mix(double* out, int iters, double seed) {
  double d[NCH];
  float f[NCH];
  unsigned u[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    d[k] = seed + 1e-3 * (threadIdx.x + k);
    f[k] = float(d[k]);
    u[k] = threadIdx.x * 2654435761u + k;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
#pragma unroll
      for (int r = 0; r < ND; ++r) d[k] = fma(d[k], 0.999999, 1e-7);
#pragma unroll
      for (int r = 0; r < NF; ++r) f[k] = fmaf(f[k], 0.999f, 1e-4f);
#pragma unroll
      for (int r = 0; r < NL; ++r) u[k] ^= u[(k + 1) % NCH] & 0x9E3779B9u;  // one LOP3
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += d[k] + f[k] + u[k];
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF, int NL>
void run(const char* name) {
  double* o;
  cudaMalloc(&o, 8);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const dim3 grid(sms * 8), block(256);
  const int iters = 4096;
  mix<ND, NF, NL><<<grid, block>>>(o, 16, 0.1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mix<ND, NF, NL><<<grid, block>>>(o, iters, 0.1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // SM clock under load: taken from the DFMA-only rate assumption is circular,
  // so report raw warp-instr/s per SMSP and the ratio to the DFMA-only run.
  const double warp_instr = double(grid.x) * (block.x / 32) * iters * NCH * (ND + NF + NL);
  const double per_smsp_per_s = warp_instr / (ms * 1e-3) / (sms * 4.0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz (max)
  // (the compiler merges some LOP3s: the SASS census of each loop body gives
  // the exact instruction count; this line assumes ND+NF+NL per chain step)
  printf("%-22s ND=%d NF=%d NL=%d  %.3f ms  nominal %.3f warp-instr/cycle/SMSP at %.0f MHz\n", name,
         ND, NF, NL, ms, per_smsp_per_s / (clk * 1e3), clk / 1e3);
  cudaFree(o);
}

int main() {
  run<1, 0, 0>("DFMA");
  run<0, 1, 0>("FFMA");
  run<0, 0, 1>("LOP3");
  run<1, 1, 0>("DFMA+FFMA 1:1");
  run<1, 2, 0>("DFMA+FFMA 1:2");
  run<1, 0, 1>("DFMA+INT 1:1");
  run<2, 1, 0>("DFMA+FFMA 2:1");
  return 0;
}
