// level_common.cuh — device pieces shared by the level-sampler kernels
// (level_kernels.cu, adaptive_kernels.cu, binned_kernels.cu): the
// uniform-grid sampler, the QoI evaluation and the fixed-tree tile
// reduction.  Internal linkage: each translation unit gets its own copy.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "ablmc_device.cuh"
#include "kernels.h"

namespace {

using namespace ablmc_dev;

#ifndef ABLMC_PEEL_WINDOWS
#define ABLMC_PEEL_WINDOWS 16  // hoisted window 0 for M <= 32 fine steps (GL/BAOAB, reference profile)
#endif
constexpr int kTile = ABLMC_TILE;            // samples per CTA (one per thread)
constexpr int kWarps = kTile / 32;

struct PathOut {
  PState f, c;
  bool ok;
};

// A leg's first step from the release state, finished from its hoisted
// sample-independent part F (KernelArgs::FirstStep, computed on the host with
// this path's IEEE semantics) and the sample's normal xi: the same operations
// on the same values as se_step / gl_step / baoab_step from (x0, u0).  h: the
// step, hh = h/2 (BAOAB), scale: BAOAB's scale_noise_by_parity; BAOAB leaves
// sde_coeffs at the new x in cend.
template <int IG, int PROF, int FAST>
__device__ __forceinline__ bool first_step_finish(PState& s, const FirstStep& F, const Coef& cx0,
                                                  double h, double hh, double xi, bool scale,
                                                  Coef& cend, const DevModel& m, bool& bad) {
  if (IG == kSE) {
    const double u1 = add(F.AB, mul(F.G, xi));
    return reflect_t<FAST>(s, add(s.x, mul(u1, h)), u1, m, bad);
  }
  if (IG == kGL) {
    const double us = add(F.D, mul(F.G, xi));
    const double u1 = sub(us, mul(dv_dx<FAST>(cx0, us, bad), h));
    return reflect_t<FAST>(s, add(s.x, mul(u1, h)), u1, m, bad);
  }
  s = {F.x, F.u, F.par, F.nrefl};
  const double us = add(F.D, mul(F.G, scale ? sgn(s.par, xi) : xi));
  if (!reflect_t<FAST>(s, add(s.x, mul(us, hh)), us, m, bad)) return false;
  cend = coeffs<PROF, FAST>(s.x, m, bad);
  s.u = sub(s.u, mul(dv_dx<FAST>(cend, s.u, bad), hh));
  return true;
}

// Level-0 sample of one step (simulate_path with M = 1 from the fixed
// release state, coupling.hpp:22-29 / 228-244) on the FAST path, for QoIs
// that read the position only: the draw is the cosine half of Philox block 0
// (noise.hpp:60-75; z1 is never used), the step is first_step_finish's with
// the sample-independent part hoisted on the host, and BAOAB's closing B
// half-kick, which changes only the velocity and cannot fail, is skipped.
// Returns x_T; `bad` as in run_sample (the caller recomputes the sample with
// the general path).
template <int IG, int PROF>
__device__ __forceinline__ double level0_x(const KernelArgs& a, uint64_t idx, const Coef& cx0,
                                           bool& bad) {
  uint32_t w[4];
  philox4x32(0u, 0u, uint32_t(idx), uint32_t(idx >> 32), a.key, w);
  double z0, z1;
  box_muller<true>(unit_2p54(w[0], w[1]), unit_2p54(w[2], w[3]), z0, z1);
  (void)z1;
  const FirstStep& F = a.fs[0];
  const DevModel& m = a.model;
  PState s;
  if (IG == kSE) {
    s = {a.x0, a.u0, 1, 0};
    const double u1 = add(F.AB, mul(F.G, z0));
    reflect_fast(s, add(s.x, mul(u1, a.h)), u1, m, bad);
  } else if (IG == kGL) {
    s = {a.x0, a.u0, 1, 0};
    const double us = add(F.D, mul(F.G, z0));
    const double u1 = sub(us, mul(dv_dx<kFastUnit>(cx0, us, bad), a.h));
    reflect_fast(s, add(s.x, mul(u1, a.h)), u1, m, bad);
  } else {
    s = {F.x, F.u, F.par, F.nrefl};
    const double us = add(F.D, mul(F.G, z0));
    reflect_fast(s, add(s.x, mul(us, a.h_half)), us, m, bad);
  }
  return s.x;
}

// simulate_pair (coupling.hpp:64-105) / simulate_path (coupling.hpp:22-29)
// for one sample.  XI: read normals from xi (oracle mode) instead of Philox.
// FAST: fast div/sqrt; returns early with bad = true on any fast-path miss
// (the caller then recomputes the sample with FAST = false).
// SHORT (coupled only): the caller guarantees M == 2 (one window); only that
// path is compiled (the short-path kernel).
template <int IG, int PROF, bool COUPLED, bool XI, int FAST, bool SHORT = false>
__device__ __forceinline__ PathOut run_sample(const KernelArgs& a, uint64_t idx,
                                              const double* __restrict__ xi, bool& bad) {
  const DevModel& m = a.model;
  // sde_coeffs(x0): every path starts at x0, so the first step's (fine and
  // coarse) coefficients are launch constants, evaluated once on the host
  // with the IEEE semantics of this path (capi.cu host_coeffs; the same bits
  // as coeffs<PROF, FAST>(x0) wherever that raises no miss).
  Coef cx0 = a.c_x0;
  cx0.rsu2 = FAST ? recip_fast(cx0.su2) : 0.0;
  PathOut o;
  double u0 = a.u0;
  if (a.random_u0) {
    // Extension D2: u0 ~ N(0, sigma_U(x0)^2) from draw k = M of this stream
    // (disjoint from the step draws 0..M-1), shared by fine and coarse.
    double z0, z1;
    normal_pair(uint64_t(a.M) >> 1, idx, a.key, z0, z1);
    const double z = (a.M & 1) ? z1 : z0;
    u0 = mul(__dsqrt_rn(cx0.su2), z);
  }
  o.f = {a.x0, u0, 1, 0};
  o.c = o.f;
  o.ok = true;
  const double h = a.h, sqrt_h = a.sqrt_h;
  if (!COUPLED) {
    Coef c0 = cx0;  // BAOAB: sde_coeffs at the current x
    double z0 = 0.0, z1 = 0.0;
    // one step; FIRST: at x0 (coefficients cx0)
    auto step = [&](auto first, int64_t k) -> bool {
      constexpr bool FIRST = decltype(first)::value;
      double xi_k;
      if (XI) {
        xi_k = xi[k];
      } else {
        if ((k & 1) == 0) normal_pair(uint64_t(k) >> 1, idx, a.key, z0, z1);
        xi_k = (k & 1) ? z1 : z0;
      }
      if (IG == kSE) {
        return FIRST ? se_update<FAST>(o.f, cx0, h, sqrt_h, xi_k, m, bad)
                     : se_step<PROF, FAST>(o.f, h, sqrt_h, xi_k, m, bad);
      } else if (IG == kGL) {
        double e;
        if (FIRST) {
          double sd;
          ou_terms<FAST>(cx0.lam, h, e, sd, bad);
          return gl_update<FAST>(o.f, cx0, h, xi_k, e, sd, m, bad);
        }
        return gl_step<PROF, FAST>(o.f, h, xi_k, m, e, bad);
      } else {
        int pm;
        return baoab_step<PROF, FAST>(o.f, c0, h, a.h_half, xi_k, false, pm, m, bad);
      }
    };
    if (a.M <= 0) return o;
    bool ok;
    if (a.fs_ok) {  // step 0 from its hoisted sample-independent part
      double xi_0;
      if (XI) {
        xi_0 = xi[0];
      } else {
        normal_pair(0, idx, a.key, z0, z1);
        xi_0 = z0;
      }
      ok = first_step_finish<IG, PROF, FAST>(o.f, a.fs[0], cx0, h, a.h_half, xi_0, false, c0, m,
                                             bad);
    } else {
      ok = step(std::true_type{}, 0);  // step 0 peeled (BAOAB: no difference)
    }
    for (int64_t k = 1; ok && !(FAST && bad) && k < a.M; ++k) ok = step(std::false_type{}, k);
    o.ok = ok;
    return o;
  }
  const double h2 = a.h2, sqrt_h2 = a.sqrt_h2;
  const bool signs = a.signs_on;
  Coef cf = cx0, cc = cx0;  // BAOAB: cached sde_coeffs at the current fine / coarse x
  // (Generating the normals one window ahead was measured 12% slower: the
  // scheduler already overlaps Box-Muller with the window's steps, and the
  // extra live registers cost occupancy.)
  // one window (2 fine steps, 1 coarse step); FIRST: window 0, both legs at x0
  auto window = [&](auto first, int64_t n) -> bool {
    constexpr bool FIRST = decltype(first)::value;
    double xi0, xi1;
    if (XI) {
      xi0 = xi[2 * n];
      xi1 = xi[2 * n + 1];
    } else {
      normal_pair(uint64_t(n), idx, a.key, xi0, xi1);
    }
    bool ok;
    if (IG == kSE) {
      // the coarse coefficients do not depend on the fine steps: issued first
      // so the scheduler can interleave the two chains
      const Coef ccw = FIRST ? cx0 : coeffs<PROF, FAST>(o.c.x, m, bad);
      const int p0 = o.f.par;
      ok = FIRST ? se_update<FAST>(o.f, cx0, h, sqrt_h, xi0, m, bad)
                 : se_step<PROF, FAST>(o.f, h, sqrt_h, xi0, m, bad);
      const int p1 = o.f.par;
      ok = ok && se_step<PROF, FAST>(o.f, h, sqrt_h, xi1, m, bad);
      const int s0 = signs ? p0 : 1, s1 = signs ? p1 : 1, sc = signs ? o.c.par : 1;
      ok = ok && se_update<FAST>(o.c, ccw, h2, sqrt_h2,
                                 coarse_noise_se<FAST>(xi0, xi1, s0, s1, sc, bad), m, bad);
    } else if (IG == kGL) {
      const int p0 = o.f.par;
      double e0, e1, ec;
      if (FIRST) {
        double sd;
        ou_terms<FAST>(cx0.lam, h, e0, sd, bad);
        ok = gl_update<FAST>(o.f, cx0, h, xi0, e0, sd, m, bad);
      } else {
        ok = gl_step<PROF, FAST>(o.f, h, xi0, m, e0, bad);  // e0 = exp(-lam(x_f at window start) h)
      }
      const int p1 = o.f.par;
      ok = ok && gl_step<PROF, FAST>(o.f, h, xi1, m, e1, bad);
      const int s0 = signs ? p0 : 1, s1 = signs ? p1 : 1, sc = signs ? o.c.par : 1;
      const double xic = coarse_noise_gl_e<FAST>(xi0, xi1, e0, s0, s1, sc, bad);
      if (FIRST) {
        double sd;
        ou_terms<FAST>(cx0.lam, h2, ec, sd, bad);
        ok = ok && gl_update<FAST>(o.c, cx0, h2, xic, ec, sd, m, bad);
      } else {
        ok = ok && gl_step<PROF, FAST>(o.c, h2, xic, m, ec, bad);
      }
    } else {
      const double e = ou_decay<FAST>(cf.lam, h, bad);  // lam_fine at the window start
      int pm0, pm1, pmc;
      ok = baoab_step<PROF, FAST>(o.f, cf, h, a.h_half, xi0, false, pm0, m, bad);
      ok = ok && baoab_step<PROF, FAST>(o.f, cf, h, a.h_half, xi1, false, pm1, m, bad);
      const int s0 = signs ? pm0 : 1, s1 = signs ? pm1 : 1;
      ok = ok && baoab_step<PROF, FAST>(o.c, cc, h2, a.h2_half,
                                        coarse_noise_gl_e<FAST>(xi0, xi1, e, s0, s1, 1, bad),
                                        signs, pmc, m, bad);
    }
    return ok;
  };
  const int64_t windows = a.M >> 1;
  // Window 0 with both legs' first steps from the host (first_step_finish).
  // Used for paths of M = 2 fine steps (one window) and, reference profile
  // GL/BAOAB, of M <= 2 ABLMC_PEEL_WINDOWS = 32 (levels 1 and 2-5 when m0 =
  // 1, as in the bench's configs; with the reference's default m0 = 40 every
  // coupled level has M >= 80 and runs the loop).  Longer paths keep the
  // single-body loop: there the hoisting is worth < 2%, and a window peeled
  // in front of the SE loop -- or of the extension profiles' loops -- costs
  // them spills.
  auto window0_hoisted = [&]() -> bool {
    double xi0, xi1;
    if (XI) {
      xi0 = xi[0];
      xi1 = xi[1];
    } else {
      normal_pair(0, idx, a.key, xi0, xi1);
    }
    const int p0 = o.f.par;
    Coef cend;
    bool ok = first_step_finish<IG, PROF, FAST>(o.f, a.fs[0], cx0, h, a.h_half, xi0, false, cend,
                                                m, bad);
    if (IG == kBAOAB) {
      const int pm0 = a.fs[0].par;  // parity at the fine step-0 noise (after its first half)
      int pm1;
      cf = cend;
      ok = ok && baoab_step<PROF, FAST>(o.f, cf, h, a.h_half, xi1, false, pm1, m, bad);
      const int s0 = signs ? pm0 : 1, s1 = signs ? pm1 : 1;
      ok = ok && first_step_finish<IG, PROF, FAST>(
                     o.c, a.fs[1], cx0, h2, a.h2_half,
                     coarse_noise_gl_e<FAST>(xi0, xi1, a.fs[0].e, s0, s1, 1, bad), signs, cc, m,
                     bad);
    } else {
      const int p1 = o.f.par;
      if (IG == kSE) {
        ok = ok && se_step<PROF, FAST>(o.f, h, sqrt_h, xi1, m, bad);
      } else {
        double e1;
        ok = ok && gl_step<PROF, FAST>(o.f, h, xi1, m, e1, bad);
      }
      const int s0 = signs ? p0 : 1, s1 = signs ? p1 : 1, sc = signs ? o.c.par : 1;
      const double xic = IG == kSE ? coarse_noise_se<FAST>(xi0, xi1, s0, s1, sc, bad)
                                   : coarse_noise_gl_e<FAST>(xi0, xi1, a.fs[0].e, s0, s1, sc, bad);
      ok = ok && first_step_finish<IG, PROF, FAST>(o.c, a.fs[1], cx0, h2, a.h2_half, xic, false,
                                                   cend, m, bad);
    }
    return ok;
  };
  if constexpr (SHORT) {  // M = 2: the same branches as below for windows == 1
    if (a.fs_ok) o.ok = window0_hoisted();
    else if (IG != kBAOAB) o.ok = window(std::true_type{}, 0);
    else o.ok = window(std::false_type{}, 0);
    return o;
  }
  constexpr bool kPeelMore = IG != kSE && PROF == kProfileReference;
  if (a.fs_ok && windows == 1) {  // M = 2: the whole sample
    o.ok = window0_hoisted();
    return o;
  }
  if (kPeelMore && a.fs_ok && windows <= ABLMC_PEEL_WINDOWS) {  // 4 <= M <= 32
    bool ok = window0_hoisted();
    for (int64_t n = 1; ok && !(FAST && bad) && n < windows; ++n) ok = window(std::false_type{}, n);
    o.ok = ok;
    return o;
  }
  if (IG != kBAOAB && windows == 1) {
    // M = 2 (level 1 when m0 = 1, the coupled level with the most samples):
    // one window, both legs at x0.  (Peeling window 0 in front of the loop for every
    // level instead costs the SE loop ~200 B of spills.)
    o.ok = window(std::true_type{}, 0);
    return o;
  }
  for (int64_t n = 0; n < windows; ++n) {
    const bool ok = window(std::false_type{}, n);
    if (!ok) o.ok = false;
    if (!ok || (FAST && bad)) break;
  }
  return o;
}

// One sample with IEEE-exact div/sqrt semantics: the fast variant when the
// host certified tame parameters, recomputed with the IEEE variant on a
// fast-path miss.
template <int IG, int PROF, bool COUPLED, bool XI, bool SHORT = false>
__device__ __forceinline__ PathOut sample(const KernelArgs& a, uint64_t idx,
                                          const double* __restrict__ xi) {
  bool bad = false;
  if (a.fast) {
    PathOut o = a.fast == kFastUnit
                    ? run_sample<IG, PROF, COUPLED, XI, kFastUnit, SHORT>(a, idx, xi, bad)
                    : run_sample<IG, PROF, COUPLED, XI, 1, SHORT>(a, idx, xi, bad);
    if (!bad) return o;
    bad = false;
  }
  return run_sample<IG, PROF, COUPLED, XI, 0, SHORT>(a, idx, xi, bad);
}

// ----------------------------------------------------------------- QoI
// qoi.hpp:22-26 Horner, 80-84 g_r.
__device__ __forceinline__ double g_r(double s, const KernelArgs& a) {
  if (s < -1.0) return 1.0;
  if (s > 1.0) return 0.0;
  double acc = 0.0;
  for (int i = a.poly_n; i-- > 0;) acc = add(mul(acc, s), a.poly[i]);
  return acc;
}

// qoi.hpp:171-188 for the scalar kinds.
__device__ __forceinline__ double qoi_scalar(double x, const KernelArgs& a) {
  switch (a.qoi_kind) {
    case 0: return x;
    case 2: return (x >= a.qa && x <= a.qb) ? 1.0 : 0.0;
    case 1: return sub(g_r(__ddiv_rn(sub(x, a.qb), a.delta), a), g_r(__ddiv_rn(sub(x, a.qa), a.delta), a));
    default: return 0.0;
  }
}

// binned_field g-term at edge e (qoi.hpp:157-167): g_r((x - edge[e]) / delta)
// with the pinned values g(edge 0) = 0 and g(edge k) = 1.
__device__ __forceinline__ double g_edge(double x, int e, int k, const double* edges,
                                         const KernelArgs& a) {
  if (e == 0) return 0.0;
  if (e == k) return 1.0;
  return g_r(__ddiv_rn(sub(x, edges[e]), a.delta), a);
}

// Resident CTAs per SM requested from ptxas (register budget 65536 / (256 *
// blocks)); tuned per integrator against spills.  The
// single-path kernels (level 0, StMC: no coarse leg) fit fewer registers.
template <int IG, bool COUPLED = true>
struct MinBlocks {
  static constexpr int value =
      !COUPLED ? ABLMC_MINB_PATH
               : (IG == kSE ? ABLMC_MINB_SE : (IG == kGL ? ABLMC_MINB_GL : ABLMC_MINB_BAOAB));
};

// sum_{i < n} p[i * stride] in index order (the fixed merge order), with the
// loads issued 16 at a time: the merges at the end of a launch are otherwise
// one dependent L2 round trip per partial (a 2^22-sample super-block has 1024
// block partials: ~0.1 ms on the kernel's tail).
__device__ __forceinline__ double ordered_sum(const double* p, int64_t n, int64_t stride) {
  double v = 0.0;
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ldcg(p + (i + k) * stride);
#pragma unroll
    for (int k = 0; k < 16; ++k) v = add(v, x[k]);
  }
  for (; i < n; ++i) v = add(v, __ldcg(p + i * stride));
  return v;
}
__device__ __forceinline__ long long ordered_sum(const long long* p, int64_t n, int64_t stride) {
  long long v = 0;
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    long long x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ldcg(p + (i + k) * stride);
#pragma unroll
    for (int k = 0; k < 16; ++k) v += x[k];
  }
  for (; i < n; ++i) v += __ldcg(p + i * stride);
  return v;
}

// Super-block order: the block partials of a super-block are folded in
// segments of kSeg consecutive blocks (each segment a left fold from 0 in
// block order), and the segment sums are folded in segment order.  One warp
// computes the 32 segments in parallel (merge_tail_warp: ~2 load round trips
// instead of 64 on the launch's tail); one thread per column computes the
// same association sequentially (merge_tail, K4).
constexpr int kSeg = 32;
template <class T>
__device__ __forceinline__ T seg_fold(const T* p, int64_t n, int64_t stride) {
  T v = T(0);
  for (int64_t s0 = 0; s0 < n; s0 += kSeg) {
    const T seg = ordered_sum(p + s0 * stride, min(int64_t(kSeg), n - s0), stride);
    if constexpr (std::is_floating_point<T>::value) v = add(v, seg);
    else v += seg;
  }
  return v;
}
// the same value computed by one warp (all lanes return it)
template <class T>
__device__ __forceinline__ T seg_fold_warp(const T* p, int64_t n, int64_t stride) {
  const int lane = threadIdx.x & 31;
  const int64_t s0 = int64_t(lane) * kSeg;
  T seg = T(0);
  if (s0 < n) seg = ordered_sum(p + s0 * stride, min(int64_t(kSeg), n - s0), stride);
  T v = T(0);
  const int nseg = int((n + kSeg - 1) / kSeg);  // <= 32 (n <= ABLMC_BLOCKS_PER_SUPER)
  for (int l = 0; l < nseg; ++l) {
    const T x = __shfl_sync(0xffffffffu, seg, l);
    if constexpr (std::is_floating_point<T>::value) v = add(v, x);
    else v += x;
  }
  return v;
}
static_assert(ABLMC_BLOCKS_PER_SUPER <= 32 * kSeg, "one warp covers a super-block");

// Per-CTA arrival counter of the tile epilogue (one per CTA; tile_prologue
// zeroes it before any warp can arrive).
__device__ __forceinline__ unsigned& tile_arrivals() {
  __shared__ unsigned s_arrive;
  return s_arrive;
}
__device__ __forceinline__ void tile_prologue() {
  if (threadIdx.x == 0) tile_arrivals() = 0u;
  __syncthreads();
}

// Block / super-block merge of the tile partials, run by ONE warp (the last
// to finish in its CTA) for scalar QoIs (dim2 + kCnt <= 32 values): the last
// tile of a 4096-sample block (arrival counter) sums the block's tile partials
// in tile order, the last block of a 2^22-sample super-block sums the block
// partials in the segment order of seg_fold -- the fixed orders of merge_tail
// below.
// SPT: samples per thread of the launch (a tile covers SPT * kTile samples,
// a 4096-sample block ABLMC_TILES_PER_BLOCK / SPT tiles).
template <int SPT = 1>
__device__ __forceinline__ void merge_tail_warp(const KernelArgs& a, const double* tile_sums,
                                                const long long* tile_cnt, int dim2) {
  constexpr int kTpb = ABLMC_TILES_PER_BLOCK / SPT;
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles = (a.n + SPT * kTile - 1) / (SPT * kTile);
  const int64_t blk = blockIdx.x / kTpb;
  const int64_t t0 = blk * kTpb;
  const int64_t t1 = min(t0 + int64_t(kTpb), n_tiles);
  unsigned last = 0;
  if (lane == 0) {
    __threadfence();  // lane 0 wrote this tile's partial
    last = atomicAdd(a.arr_blk + blk, 1u) == unsigned(t1 - t0 - 1);
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  const int c = lane;
  if (c < dim2) {
    a.blk_sums[blk * dim2 + c] = ordered_sum(tile_sums + t0 * dim2 + c, t1 - t0, dim2);
  } else if (c < dim2 + kCnt) {
    a.blk_cnt[kCnt * blk + (c - dim2)] = ordered_sum(tile_cnt + kCnt * t0 + (c - dim2), t1 - t0, kCnt);
  }
  __threadfence();
  __syncwarp();
  const int64_t n_blk = (n_tiles + kTpb - 1) / kTpb;
  const int64_t sb = blk / ABLMC_BLOCKS_PER_SUPER;
  const int64_t b0 = sb * ABLMC_BLOCKS_PER_SUPER;
  const int64_t b1 = min(b0 + int64_t(ABLMC_BLOCKS_PER_SUPER), n_blk);
  last = 0;
  if (lane == 0) {
    a.arr_blk[blk] = 0u;
    last = atomicAdd(a.arr_sb + sb, 1u) == unsigned(b1 - b0 - 1);
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  const int64_t so = a.sb_out + sb;
  for (int k = 0; k < dim2 + kCnt; ++k) {  // the whole warp per column
    if (k < dim2) {
      const double v = seg_fold_warp(a.blk_sums + b0 * dim2 + k, b1 - b0, int64_t(dim2));
      if (lane == 0) a.sb_sums[so * dim2 + k] = v;
    } else {
      const long long v = seg_fold_warp(a.blk_cnt + kCnt * b0 + (k - dim2), b1 - b0, int64_t(kCnt));
      if (lane == 0) a.sb_cnt[kCnt * so + (k - dim2)] = v;
    }
  }
  if (lane == 0) a.arr_sb[sb] = 0u;
}

// Tile reduction shared by the level kernels: the tile's {sum_y, sum_y2}
// (fixed warp-shuffle tree, then warps in order) of the successful samples'
// QoI values y, and counts {n, failed, cost_steps}.  Binned field: sums come
// from K4, only the counts are reduced here.  No CTA barrier: each warp
// leaves its partial in shared memory and the LAST warp to arrive (shared
// arrival counter, zeroed by tile_prologue) sums the warps in order, writes
// the tile partial and, for scalar QoIs, runs the block/super-block merge;
// the other warps retire at once (at level 0 the barrier was 27% of the
// stalls).
// UNIFORM_STEPS: every successful sample of the tile took `steps` steps (the
// uniform grids), so the counts are two warp votes; otherwise (adaptive) the
// step counts are summed by shuffles.  Integer sums: the same values either way.
// The common tail: per-thread sums (sy, sy2) of the thread's successful
// samples and the warp's counts (cn, cf, cc: warp totals, identical in every
// lane) -> fixed warp-shuffle tree -> warps in order (last warp to arrive)
// -> tile partial at tile blockIdx.x -> block / super-block merge.
template <int SPT = 1>
__device__ __forceinline__ void tile_reduce_sums(const KernelArgs& a, double sy, double sy2,
                                                 long long cn, long long cf, long long cc,
                                                 bool binned, double* __restrict__ tile_sums,
                                                 long long* __restrict__ tile_cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double s_red[kWarps][2];
  __shared__ long long s_cnt[kWarps][kCnt];
  if (!binned) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sy = add(sy, __shfl_down_sync(0xffffffffu, sy, off));
      sy2 = add(sy2, __shfl_down_sync(0xffffffffu, sy2, off));
    }
  }
  unsigned last = 0;
  if (lane == 0) {
    s_red[warp][0] = sy;
    s_red[warp][1] = sy2;
    s_cnt[warp][0] = cn;
    s_cnt[warp][1] = cf;
    s_cnt[warp][2] = cc;
    __threadfence_block();
    last = atomicAdd(&tile_arrivals(), 1u) == unsigned(kWarps - 1);
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  if (lane == 0) {
    __threadfence_block();
    const volatile double* vr = &s_red[0][0];
    const volatile long long* vc = &s_cnt[0][0];
    double ty = 0.0, ty2 = 0.0;
    long long t[kCnt] = {0, 0, 0};
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      ty = add(ty, vr[2 * w]);
      ty2 = add(ty2, vr[2 * w + 1]);
      for (int c = 0; c < kCnt; ++c) t[c] += vc[kCnt * w + c];
    }
    if (!binned) {
      tile_sums[2 * blockIdx.x] = ty;  // dim == 1
      tile_sums[2 * blockIdx.x + 1] = ty2;
    }
    for (int c = 0; c < kCnt; ++c) tile_cnt[kCnt * blockIdx.x + c] = t[c];
  }
  if (!binned) merge_tail_warp<SPT>(a, tile_sums, tile_cnt, 2);
}

// Tile reduction shared by the level kernels: the tile's {sum_y, sum_y2}
// (fixed warp-shuffle tree, then warps in order) of the successful samples'
// QoI values y, and counts {n, failed, cost_steps}.  Binned field: sums come
// from K4, only the counts are reduced here.  No CTA barrier: each warp
// leaves its partial in shared memory and the LAST warp to arrive (shared
// arrival counter, zeroed by tile_prologue) sums the warps in order, writes
// the tile partial and, for scalar QoIs, runs the block/super-block merge;
// the other warps retire at once (at level 0 the barrier was 27% of the
// stalls).
// UNIFORM_STEPS: every successful sample of the tile took `steps` steps (the
// uniform grids), so the counts are two warp votes; otherwise (adaptive) the
// step counts are summed by shuffles.  Integer sums: the same values either way.
template <bool UNIFORM_STEPS>
__device__ __forceinline__ void tile_reduce(const KernelArgs& a, bool active, bool good, double y,
                                            long long steps, bool binned,
                                            double* __restrict__ tile_sums,
                                            long long* __restrict__ tile_cnt) {
  long long cn, cf, cc;
  if (UNIFORM_STEPS) {
    cn = __popc(__ballot_sync(0xffffffffu, good));
    cf = __popc(__ballot_sync(0xffffffffu, active && !good));
    cc = cn * steps;
  } else {
    cn = good ? 1 : 0;
    cf = (active && !good) ? 1 : 0;
    cc = good ? steps : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      cn += __shfl_down_sync(0xffffffffu, cn, off);
      cf += __shfl_down_sync(0xffffffffu, cf, off);
      cc += __shfl_down_sync(0xffffffffu, cc, off);
    }
  }
  const double sy = (!binned && good) ? y : 0.0;
  const double sy2 = (!binned && good) ? mul(y, y) : 0.0;
  tile_reduce_sums<1>(a, sy, sy2, cn, cf, cc, binned, tile_sums, tile_cnt);
}

// Single-pass merge, run by every CTA after its tile partial is written:
// the last CTA of a 4096-sample block (arrival counter) sums the block's
// tile partials in tile order, and the last block of a super-block sums the
// block partials in the segment order of seg_fold -- the same fixed orders as a
// separate tile->block->super-block reduction, without two extra launches.
// Counters reset themselves for the next launch.
// `writers`: threads [0, writers) wrote this CTA's tile partial; only they
// need the fence before the arrival atomic (a fence per warp costs ~100s of
// cycles: at level 0 it was 12% of the kernel's stalls).
__device__ __forceinline__ void merge_tail(const KernelArgs& a, const double* tile_sums,
                                           const long long* tile_cnt, int dim2, int writers = 1) {
  __shared__ int s_last;
  if (int(threadIdx.x) < writers) __threadfence();  // this CTA's tile partial, visible device-wide
  __syncthreads();
  const int64_t n_tiles = (a.n + kTile - 1) / kTile;
  const int64_t blk = blockIdx.x / ABLMC_TILES_PER_BLOCK;
  const int64_t t0 = blk * ABLMC_TILES_PER_BLOCK;
  const int64_t t1 = min(t0 + int64_t(ABLMC_TILES_PER_BLOCK), n_tiles);
  if (threadIdx.x == 0) s_last = atomicAdd(a.arr_blk + blk, 1u) == unsigned(t1 - t0 - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int c = threadIdx.x; c < dim2 + kCnt; c += blockDim.x) {
    if (c < dim2) a.blk_sums[blk * dim2 + c] = ordered_sum(tile_sums + t0 * dim2 + c, t1 - t0, dim2);
    else a.blk_cnt[kCnt * blk + (c - dim2)] = ordered_sum(tile_cnt + kCnt * t0 + (c - dim2), t1 - t0, kCnt);
  }
  __threadfence();
  __syncthreads();
  const int64_t n_blk = (n_tiles + ABLMC_TILES_PER_BLOCK - 1) / ABLMC_TILES_PER_BLOCK;
  const int64_t sb = blk / ABLMC_BLOCKS_PER_SUPER;
  const int64_t b0 = sb * ABLMC_BLOCKS_PER_SUPER;
  const int64_t b1 = min(b0 + int64_t(ABLMC_BLOCKS_PER_SUPER), n_blk);
  if (threadIdx.x == 0) {
    a.arr_blk[blk] = 0u;
    s_last = atomicAdd(a.arr_sb + sb, 1u) == unsigned(b1 - b0 - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t so = a.sb_out + sb;
  for (int c = threadIdx.x; c < dim2 + kCnt; c += blockDim.x) {
    if (c < dim2) a.sb_sums[so * dim2 + c] = seg_fold(a.blk_sums + b0 * dim2 + c, b1 - b0, int64_t(dim2));
    else a.sb_cnt[kCnt * so + (c - dim2)] = seg_fold(a.blk_cnt + kCnt * b0 + (c - dim2), b1 - b0, int64_t(kCnt));
  }
  if (threadIdx.x == 0) a.arr_sb[sb] = 0u;
}

// QoI value of one successful sample (qoi.hpp:171-188; the difference for a
// coupled pair, coupling.hpp:262-268).
template <bool COUPLED>
__device__ __forceinline__ double sample_y(const KernelArgs& a, const PathOut& o) {
  double y = qoi_scalar(o.f.x, a);
  if (COUPLED) y = sub(y, qoi_scalar(o.c.x, a));
  return y;
}

// binned field: the terminal positions for K4 (failed samples as NaN: K4
// skips them).
__device__ __forceinline__ void store_pos(const KernelArgs& a, int64_t j, bool good,
                                          const PathOut& o) {
  a.pos[2 * j] = good ? o.f.x : __longlong_as_double(0x7ff8000000000000LL);
  a.pos[2 * j + 1] = o.c.x;
}

// Tile epilogue of the one-thread-per-sample kernels.
template <bool COUPLED>
__device__ __forceinline__ void tile_epilogue(const KernelArgs& a, int64_t j, bool active,
                                              const PathOut& o, long long steps,
                                              double* __restrict__ tile_sums,
                                              long long* __restrict__ tile_cnt) {
  const bool good = active && o.ok;
  const bool binned = a.qoi_kind == 3;
  if (binned && active) store_pos(a, j, good, o);
  tile_reduce<true>(a, active, good, (!binned && good) ? sample_y<COUPLED>(a, o) : 0.0, steps,
                    binned, tile_sums, tile_cnt);
}

}  // namespace
