// kernels.h — internal launch interface between the C-ABI host code
// (capi.cpp) and the sm_100a kernels (level_kernels.cu).  Not public.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "ablmc_device.cuh"

#ifndef ABLMC_TILE
#define ABLMC_TILE 256                 // samples per CTA tile (= threads per CTA)
#endif
#define ABLMC_TILES_PER_BLOCK (4096 / ABLMC_TILE)  // 4096 = reference block_size (stats.hpp:100)
#define ABLMC_BLOCKS_PER_SUPER 1024    // 1024 * 4096 = 2^22 = ABLMC_SUPERBLOCK
#define ABLMC_MAX_POLY 14
// per tile / block / super-block count record: {n, failed, cost_steps}
constexpr int kCnt = 3;
#ifndef ABLMC_MINB_SE
#define ABLMC_MINB_SE 4
#endif
#ifndef ABLMC_MINB_GL
#define ABLMC_MINB_GL 3
#endif
#ifndef ABLMC_MINB_PATH
#define ABLMC_MINB_PATH 5
#endif
// samples per thread of the short-path (level 0 / StMC, M <= 4) kernel and
// the unroll of its per-thread sample loop
#ifndef ABLMC_SPT_SHORT
#define ABLMC_SPT_SHORT 4
#endif
#ifndef ABLMC_SPT_UNROLL
#define ABLMC_SPT_UNROLL 1
#endif
#ifndef ABLMC_MINB_BAOAB
#define ABLMC_MINB_BAOAB 3
#endif

// The sample-independent part of a leg's first step from the release state
// (x0, u0) with step h (capi.cu first_step; the device finishes it with the
// sample's normal xi):
//   SE:    u1 = AB + G xi               (AB = (1 - lam h) u0 - dv_dx(u0) h, G = sigma sqrt(h))
//   GL:    u* = D + G xi                (D = e u0, G = sigma sd(lam, h))
//   BAOAB: (x, u, par, nrefl) after the first B and A half-steps and the
//          reflection, then u* = D + G xi' (D = decay u, G = sigma_mid sd_mid).
struct FirstStep {
  double AB, D, G, e;  // e: exp(-lam(x0) h) (GL/BAOAB coarse-noise weight)
  double x, u;
  int par, nrefl;
};

// Everything one launch needs, passed by value (kernel-parameter constant bank).
struct KernelArgs {
  ablmc_dev::DevModel model;
  double x0, u0;
  ablmc_dev::Coef c_x0;     // sde_coeffs(x0): every sample's first-step coefficients (host)
  double h, sqrt_h;         // fine step T/M and sqrt(h)
  double h2, sqrt_h2;       // coarse step 2h and sqrt(2h)
  double h_half, h2_half;   // 0.5*h, 0.5*(2h) (BAOAB half steps)
  int64_t M;                // fine steps (path: steps)
  int64_t first;            // reference `first` (sample index of offset 0)
  int64_t offset;           // offset of this launch's sample 0 from `first`
  int64_t n;                // samples in this launch
  uint32_t k0, k1;          // Philox key of stream (seed, level)
  ablmc_dev::PhiloxKey key; // its 10 round keys
  int signs_on;
  int random_u0;
  int qoi_kind;
  int fast;                 // 1: tame parameters, fast div/sqrt with IEEE recompute on a miss;
                            // 2: same with H == 1 and noise_scale == 1
  int fp32;                 // 1: fp32-state variant (statistical parity only)
  int dim;
  double qa, qb, delta;
  int poly_n;               // r + 2 coefficients
  double poly[ABLMC_MAX_POLY];
  const double* edges;      // device copy of bin edges (binned field)
  double* pos;              // binned field: per-sample (x_f, x_c) of this launch (K1 -> K4)
  // adaptive (non-nested) stepping, coupling.hpp:31-51 / 137-214
  int adaptive;
  double T, x_adapt;
  double h_base;            // T / M: fine base step (coarse base 2 h_base)
  int64_t max_iter;         // pair: 256 ceil(T/h_base) + 256; path: 64 ceil(T/h_base) + 64
  // persistent adaptive sampler (K1P -> K1R -> K1T): per-sample results of
  // this launch, work counters {next sample, redo count}, redo list
  double* ad_y;             // QoI value (scalar kinds)
  long long* ad_steps;      // steps taken, -1 = failed sample
  unsigned long long* ad_ctrl;
  long long* ad_redo;       // samples whose fast path missed (recomputed exactly)
  long long* ad_deep;       // GL/BAOAB pairs with > 64 pending sub-intervals on a leg
                            // (K1D recomputes them with global-memory pending storage);
                            // ad_ctrl = {next sample, redo count, deep count}
  double* ad_scratch;       // K1D: per-thread pending storage, 4 * ABLMC_PEND_DEEP doubles
  // single-pass merge inside the sampler launch: tile -> 4096-sample block ->
  // super-block partials (merge_tail), arrival counters zero between launches
  double* blk_sums;
  long long* blk_cnt;
  double* sb_sums;
  long long* sb_cnt;
  unsigned* arr_blk;
  unsigned* arr_sb;
  int64_t sb_out;           // super-block row of this launch's first super-block
  // (last: the hot fields above keep their parameter-bank offsets, which the
  // level-10 loop's constant loads are scheduled around)
  FirstStep fs[2];          // first fine (h) / coarse (2h) step from (x0, u0), if fs_ok
  int fs_ok;                // 1: fs valid (fixed u0, nothing exceptional in the first step)
};

// K1D geometry and per-thread pending capacity (adaptive_kernels.cu)
#define ABLMC_PEND_DEEP 4096
#define ABLMC_DEEP_THREADS (32 * 64)

struct StateOut {
  double fx, fu, cx, cu;
  int fpar, cpar;
  int fn, cn;
  int ok, steps;             // steps: adaptive steps taken (fine + coarse)
};

cudaError_t launch_level(const KernelArgs& a, int ig, bool coupled, double* tile_sums,
                         long long* tile_cnt, cudaStream_t st);
cudaError_t launch_states(const KernelArgs& a, int ig, bool coupled, const double* xi,
                          StateOut* out, cudaStream_t st);
// adaptive_kernels.cu / binned_kernels.cu (called by launch_level / launch_states)
cudaError_t launch_adaptive_level(const KernelArgs& a, int ig, bool coupled, double* tile_sums,
                                  long long* tile_cnt, cudaStream_t st);
cudaError_t launch_adaptive_states(const KernelArgs& a, int ig, bool coupled, StateOut* out,
                                   cudaStream_t st);
cudaError_t launch_binned(const KernelArgs& a, bool coupled, double* tile_sums,
                          const long long* tile_cnt, cudaStream_t st);
cudaError_t launch_merge_super(int64_t n_sb, int dim, const double* ss, const long long* sc,
                               double* rs, long long* rc, cudaStream_t st);
// collective.cu: pack rows [0, rows) of the super-block partials plus one
// status row into the all-gather send buffer; merge one request's gathered
// rows (all ranks) in global super-block order into the device result.
cudaError_t launch_pack_rows(int64_t rows, int dim, const double* sb_sums, const long long* sb_cnt,
                             double* send, long long status, cudaStream_t st);
cudaError_t launch_merge_gathered(int world, int64_t cap_total, int64_t n_sb, int64_t pbase,
                                  int dim, const double* recv, double* res_sums,
                                  long long* res_cnt, long long* res_status, cudaStream_t st);
cudaError_t upload_log_table();           // Box-Muller log table (ablmc_init), one
cudaError_t upload_log_table_adaptive();  // per translation unit that draws normals
cudaError_t launch_normals(uint32_t k0, uint32_t k1, uint64_t idx, uint64_t kstart, int64_t n,
                           double* out, cudaStream_t st);
// DFMA throughput probe (FP64 lane-ops/s), see ablmc_probe_fp64_rate.
cudaError_t probe_fp64(cudaStream_t st, double* lane_ops_per_s);
// Device self-test of the fast IEEE div/sqrt and the Box-Muller libm kernels:
// out[0..8] = {div checked, div mismatches where ok, div misses, sqrt checked,
// sqrt mismatches where ok, sqrt misses, max ulp log_unit vs libdevice log,
// max |sin - libdevice sin| and |cos - ...| in units of 0.01 * 2^-53}.
cudaError_t launch_selftest(int64_t n, uint64_t seed, unsigned long long* d_out, cudaStream_t st);
