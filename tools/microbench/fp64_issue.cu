// FP64 issue microbenchmark for B200 (sm_100a): what limits K1's FP64-pipe
// utilisation?  Each variant runs a fixed instruction mix over the whole GPU
// (grid = SMs x CTAS_PER_SM CTAs of 256 threads) and prints the FP64-pipe
// utilisation (DFMA/DMUL/DADD lane-ops per SM-cycle / 64) and the issue rate
// (warp-instructions per SMSP-cycle) at the SM clock measured with clock64.
//   * operand form: DFMA with one register operand (the peak probe) vs three
//     register operands (K1's DFMAs: 6 32-bit register reads);
//   * latency hiding: NCH independent chains per thread at 8 warps/SMSP
//     (K1 SE's occupancy: 64 registers, 4 CTAs/SM);
//   * mixes: DFMA + IMAD.WIDE/LOP3 (Philox-like integer work) 1:1, and DFMA
//     chains broken by MUFU.RSQ64H seeds (K1's correctly rounded sqrt).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fi tools/microbench/fp64_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq64h(double x) {  // MUFU.RSQ64H on the high word
  double r;
  asm volatile("{.reg .b32 lo, hi; mov.b64 {lo, hi}, %1; rsqrt.approx.ftz.f64 %0, %1;}"
               : "=d"(r) : "d"(x));
  return r;
}

// KIND 0: d = fma(d, c, c)          (1 register operand)
// KIND 1: d = fma(d, x, y)          (3 register operands, x, y loop-carried per chain)
// KIND 2: KIND 1 + one IMAD.WIDE.U32 + one LOP3 per DFMA (independent integer chain)
// KIND 3: 8 DFMA (KIND 1) then one MUFU.RSQ64H on the chain value
// KIND 4: DMUL d = d * x
template <int KIND, int NCH>
__global__ void __launch_bounds__(256, 4) mix(double* out, long long* cyc, int iters, double seed) {
  double d[NCH], x[NCH], y[NCH];
  unsigned u[NCH], v[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    d[k] = seed + 1e-3 * (threadIdx.x + k);
    x[k] = 0.999999 - 1e-9 * k * threadIdx.x;
    y[k] = 1e-7 + 1e-12 * (k + threadIdx.x);
    u[k] = threadIdx.x * 2654435761u + k;
    v[k] = blockIdx.x ^ k;
  }
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if (KIND == 0) d[k] = fma(d[k], 0.999999, 1e-7);
        else if (KIND == 4) d[k] = d[k] * x[k];
        else if (KIND == 10) d[k] = fma(d[k], x[k], 1e-7);  // 2 register operands + constant
        else if (KIND == 11) {}  // integer only
        else if (KIND == 13) d[k] = fma(d[k], d[k], d[k]) * 0.5;  // one register three times (+DMUL imm)
        else if (KIND == 14) d[k] = fma(d[k], x[k], 0.5);  // 2 registers + immediate
        else if (KIND == 12) {  // IMAD.WIDE only
          const unsigned long long p = (unsigned long long)u[k] * 0xD2511F53u;
          u[k] = unsigned(p >> 32) ^ unsigned(p);
        }
        else d[k] = fma(d[k], x[k], y[k]);
        if (KIND == 2) {
          const unsigned long long p = (unsigned long long)u[k] * 0xD2511F53u;
          u[k] = unsigned(p >> 32) ^ v[k] ^ unsigned(p);
        }
        if (KIND == 5) u[k] = (u[k] * 0xD2511F53u) ^ v[k] ^ (u[k] >> 7);  // IMAD (lo) + LOP3 (+SHF)
        if (KIND == 6) u[k] = __umulhi(u[k], 0xD2511F53u) ^ v[k] ^ u[k];  // IMAD.HI + LOP3
        if (KIND == 7) u[k] = ((u[k] ^ v[k]) & 0x9E3779B9u) ^ (u[k] | v[k]);  // LOP3 only
        if (KIND == 8) u[k] = (u[k] + v[k]) ^ (u[k] << 3);  // IADD3/LEA + LOP3
        if (KIND == 9) {  // FFMA (float chain in u's bits)
          const float f = __uint_as_float(u[k] | 0x3f800000u);
          u[k] = __float_as_uint(fmaf(f, 0.999f, 1e-4f));
        }
      }
    }
    if (KIND == 3) {
#pragma unroll
      for (int k = 0; k < NCH; ++k) d[k] = fma(rsq64h(d[k]), 1e-3, d[k]);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += d[k] + u[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int KIND, int NCH>
void run(const char* name, int ipi /* instructions per iteration per chain (census) */,
         int fp64pi /* FP64-pipe instructions per iteration per chain */) {
  double* o;
  long long* cyc;
  cudaMalloc(&o, 8);
  cudaMalloc(&cyc, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const dim3 grid(sms * 4), block(256);
  const int iters = 2048;
  mix<KIND, NCH><<<grid, block>>>(o, cyc, 16, 0.1);
  cudaMemset(cyc, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  mix<KIND, NCH><<<grid, block>>>(o, cyc, iters, 0.1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double warps_per_smsp = 8.0;  // 4 CTAs x 8 warps / 4 SMSPs
  const double fp64_warp = warps_per_smsp * iters * NCH * fp64pi;
  const double all_warp = warps_per_smsp * iters * NCH * ipi;
  const double mhz = c / (ms * 1e3);
  printf("%-34s NCH=%d  %.3f ms  %5.0f MHz  FP64 pipe %.1f%%  issue %.3f warp-instr/cycle/SMSP\n",
         name, NCH, ms, mhz, 100.0 * 2.0 * fp64_warp / c, all_warp / c);
  cudaFree(o);
  cudaFree(cyc);
}

int main() {
  run<0, 1>("DFMA 1-reg", 8, 8);
  run<0, 2>("DFMA 1-reg", 8, 8);
  run<0, 4>("DFMA 1-reg", 8, 8);
  run<1, 1>("DFMA 3-reg", 8, 8);
  run<1, 2>("DFMA 3-reg", 8, 8);
  run<1, 4>("DFMA 3-reg", 8, 8);
  run<4, 2>("DMUL 2-reg", 8, 8);
  run<4, 4>("DMUL 2-reg", 8, 8);
  run<2, 1>("DFMA 3-reg + IMAD.WIDE+LOP3", 24, 8);
  run<2, 2>("DFMA 3-reg + IMAD.WIDE+LOP3", 24, 8);
  run<2, 4>("DFMA 3-reg + IMAD.WIDE+LOP3", 24, 8);
  run<5, 4>("DFMA 3-reg + IMAD(lo)+LOP3+SHF", 32, 8);
  run<6, 4>("DFMA 3-reg + IMAD.HI+LOP3", 24, 8);
  run<7, 4>("DFMA 3-reg + LOP3 x2", 24, 8);
  run<8, 4>("DFMA 3-reg + IADD+LOP3", 24, 8);
  run<9, 4>("DFMA 3-reg + FFMA+LOP3", 24, 8);
  run<10, 2>("DFMA 2-reg+const", 8, 8);
  run<10, 4>("DFMA 2-reg+const", 8, 8);
  run<12, 4>("IMAD.WIDE + LOP3 only", 16, 0);
  run<13, 4>("DFMA(d,d,d) + DMUL imm", 16, 16);
  run<14, 4>("DFMA 2-reg + imm", 8, 8);
  run<3, 1>("8 DFMA + MUFU.RSQ64H + DFMA", 10, 9);
  run<3, 2>("8 DFMA + MUFU.RSQ64H + DFMA", 10, 9);
  run<3, 4>("8 DFMA + MUFU.RSQ64H + DFMA", 10, 9);
  return 0;
}
