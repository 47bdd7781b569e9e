// adaptive_kernels.cu — adaptive (non-nested) stepping, SampleOptions::adaptive
// (coupling.hpp:31-51 simulate_path_adaptive, 137-214 simulate_pair_adaptive;
// SURVEY §8(f) next #4):
//   K1P k_adaptive_persistent  work-queue sampler, one schedule event per
//       loop iteration, per-sample (QoI value, steps) slots
//   K1R k_adaptive_redo        exact recomputation of fast-path misses
//   K1T k_adaptive_tiles       tile partials in the uniform sampler's tree
//   Kst k_states_adaptive      per-sample final states (tests)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <type_traits>

#include "level_common.cuh"

namespace {

// ------------------------------------------------------- adaptive stepping
// SampleOptions::adaptive.  The step sizes are data
// dependent, so every comparison of the reference's schedule (t + h >= T,
// t_next == tau_next, min(h, .)) must see the reference's bits: the FAST
// variant is the same bit-exact fast div/sqrt sequences as the uniform
// sampler (a miss raises `bad` and the sample is recomputed with FAST = 0),
// and sde_coeffs is evaluated once per step and shared by the schedule, the
// pending-noise weights and the step itself.
//
// Sequential NoiseStream::next() (noise.hpp:57): draw k is half of Philox
// block k >> 1.
template <class Key>
struct SeqNoise {
  uint64_t k = 0;
  double z1 = 0.0;
  __device__ __forceinline__ double next(uint64_t idx, const Key& key) {
    double z;
    if ((k & 1) == 0) {
      normal_pair(k >> 1, idx, key, z, z1);
    } else {
      z = z1;
    }
    ++k;
    return z;
  }
};

// The persistent sampler's stream (the same draws in the same order as
// SeqNoise): up to three upcoming normals per lane, refilled one Philox block
// (two normals) at a time in warp-wide batches.  Lanes sit at different
// draws of different samples, so a block generated on demand (SeqNoise: at
// every even draw) ran Philox + Box-Muller on ~44% of the lanes nearly every
// event; here a refill runs only when some lane's buffer is empty, and then
// for every lane holding at most kRefillAt normals (refill_if_any_empty).
#ifndef ABLMC_BUF_NORMALS
#define ABLMC_BUF_NORMALS 3  // buffer capacity: 3 (refill at <= 1) or 4 (refill at <= 2)
#endif
struct BufNoise {
  uint64_t blk;  // next Philox block of the sample's stream
  double q0, q1, q2, q3;
  int n;         // normals buffered (q0 is the next draw)
  static constexpr int kRefillAt = ABLMC_BUF_NORMALS - 2;
  __device__ __forceinline__ void reset() {
    blk = 0;
    n = 0;
  }
  template <class Key>
  __device__ __forceinline__ void refill(uint64_t idx, const Key& key) {  // n <= kRefillAt
    double z0, z1;
    normal_pair(blk, idx, key, z0, z1);
    ++blk;
    if (ABLMC_BUF_NORMALS == 4) q3 = n == 2 ? z1 : q3;
    q2 = n == 1 ? z1 : (n == 2 ? z0 : q2);
    q1 = n == 0 ? z1 : (n == 1 ? z0 : q1);
    q0 = n == 0 ? z0 : q0;
    n += 2;
  }
  template <class Key>
  __device__ __forceinline__ double next(uint64_t, const Key&) {  // n >= 1
    const double z = q0;
    q0 = q1;
    q1 = q2;
    if (ABLMC_BUF_NORMALS == 4) q2 = q3;
    --n;
    return z;
  }
};
// Warp-uniform point of the persistent loop (at most one draw per event).
template <class Key>
__device__ __forceinline__ void refill_if_any_empty(BufNoise& ns, bool live, uint64_t idx,
                                                    const Key& key) {
  if (__any_sync(__activemask(), live && ns.n == 0) && live && ns.n <= BufNoise::kRefillAt)
    ns.refill(idx, key);
}

// timeline.hpp:18-23 — min{h, lambda(x_adapt)/lambda(x) h}
template <int FAST>
__device__ __forceinline__ double adaptive_h(double lam_x, double h, double lam_ref, bool& bad) {
  const double v = mul(Ops<FAST>::div(lam_ref, lam_x, bad), h);
  return (v < h) ? v : h;
}

// coupling.hpp:31-51 — one path of adaptive steps with base size h_base.
template <int IG, int PROF, int FAST>
__device__ __forceinline__ PathOut run_path_adaptive(const KernelArgs& a, uint64_t idx,
                                                     long long& steps, bool& bad) {
  using O = Ops<FAST>;
  const DevModel& m = a.model;
  PathOut o;
  o.f = {a.x0, a.u0, 1, 0};
  o.c = o.f;
  o.ok = true;
  const double T = a.T, hb = a.h_base;
  const double lam_ref = coeffs<PROF, FAST>(a.x_adapt, m, bad).lam;
  SeqNoise<PhiloxKey> ns;
  Coef c = coeffs<PROF, FAST>(a.x0, m, bad);  // sde_coeffs(o.f.x)
  double t = 0.0;
  steps = 0;
  while (t < T) {
    double h = adaptive_h<FAST>(c.lam, hb, lam_ref, bad);
    if (add(t, h) >= T) h = sub(T, t);
    const double xi = ns.next(idx, a.key);
    bool ok;
    if (IG == kSE) {
      ok = se_update<FAST>(o.f, c, h, O::sqrt(h, bad), xi, m, bad);
      c = coeffs<PROF, FAST>(o.f.x, m, bad);
    } else if (IG == kGL) {
      double e, sd;
      ou_terms<FAST>(c.lam, h, e, sd, bad);
      ok = gl_update<FAST>(o.f, c, h, xi, e, sd, m, bad);
      c = coeffs<PROF, FAST>(o.f.x, m, bad);
    } else {
      int pm;
      ok = baoab_step<PROF, FAST>(o.f, c, h, mul(0.5, h), xi, false, pm, m, bad);
    }
    t = (add(t, h) >= T) ? T : add(t, h);
    if (!ok || ++steps > a.max_iter) {
      o.ok = false;
      break;
    }
    if (FAST && bad) break;
  }
  return o;
}

// One leg of the adaptive pair (coupling.hpp:109-129): state, current step
// [t, t_next) of size h_cur, sde_coeffs at the leg's position (constant while
// its sub-intervals are pending), and the running noise increment.
struct ALeg {
  PState s;
  Coef c;         // sde_coeffs(s.x)
  double t, t_next, h_cur;
  double acc;     // SE: sum S_j xi_j sqrt(dtau_j); GL/BAOAB: Horner form of the OU-weighted
                  // sum (used only when more sub-intervals are pending than are stored)
  long long steps;
  int np;         // GL/BAOAB: pending sub-intervals of the current step
  bool done;
};

// GL/BAOAB pending terms (timeline.hpp:86-105): term_r = S_r xi_r sd(lam, dt_r)
// and e_r = exp(-lam dt_r) of each pending sub-interval, so the increment is
// the reference's backward sum acc += term_r damp, damp *= e_r (r = n-1..0),
// bit for bit.  The persistent kernel keeps the first kPend of them per leg
// in shared memory and the next kPendLocal - kPend in local memory (a coarse
// step near the ground can span many fine sub-intervals); the
// one-thread-per-sample kernels keep kPendLocal in local memory.  Beyond
// kPendLocal the Horner form (equal for <= 2 terms, within rounding beyond)
// is used (the persistent FAST kernel hands such samples to K1R first).
#ifndef ABLMC_KPEND
#define ABLMC_KPEND 8
#endif
constexpr int kPend = ABLMC_KPEND;
constexpr int kPendLocal = 64;
struct PendSpill {  // persistent kernel: pending terms kPend .. kPendLocal-1, per leg
  double t[2][kPendLocal - kPend], e[2][kPendLocal - kPend];
};

template <class Term, class Decay>
__device__ __forceinline__ double backward_sum(int n, Term term, Decay decay) {
  double acc = 0.0, damp = 1.0;
  for (int r = n - 1; r >= 0; --r) {
    acc = add(acc, mul(term(r), damp));
    damp = mul(damp, decay(r));
  }
  return acc;
}

struct PendLocal {
  static constexpr int kCap = kPendLocal;
  double t[kPendLocal], e[kPendLocal];
};
// K1D: the same terms in global memory (a per-thread slice of ad_scratch),
// for the rare pairs whose legs exceed kPendLocal; beyond kPendDeep the
// Horner form is the last resort.
constexpr int kPendDeep = ABLMC_PEND_DEEP;
struct PendGlobal {
  static constexpr int kCap = kPendDeep;
  double* t;
  double* e;
};

// coupling.hpp:140-155
template <int FAST>
__device__ __forceinline__ void leg_schedule(ALeg& L, double base, double T, double lam_ref,
                                             bool& bad) {
  double h = adaptive_h<FAST>(L.c.lam, base, lam_ref, bad);
  if (add(L.t, h) >= T) {
    h = sub(T, L.t);
    L.t_next = T;
  } else {
    L.t_next = add(L.t, h);
  }
  L.h_cur = h;
}

// Pending sub-interval (tau, tau + dt) with draw xi and coupling sign S
// (timeline.hpp:75-105 terms).  SE: S xi sqrt(dt), summed forward as the
// reference does.  GL/BAOAB: the term S xi sd(lam, dt) and weight
// exp(-lam dt) are stored for the backward sum at the step (leg_settle);
// the Horner form acc <- acc e + term is kept alongside for overflow.
template <int IG, int FAST, class Pend>
__device__ __forceinline__ void leg_push(ALeg& L, Pend& P, double xi_s, double dt,
                                         double sqrt_dt, bool& bad, bool& deep) {
  if (IG == kSE) {
    L.acc = add(L.acc, mul(xi_s, sqrt_dt));
  } else {
    double e, sd;
    ou_terms<FAST>(L.c.lam, dt, e, sd, bad);
    const double term = mul(xi_s, sd);
    if (L.np < Pend::kCap) {
      P.t[L.np] = term;
      P.e[L.np] = e;
    } else {
      deep = true;
    }
    ++L.np;
    L.acc = add(mul(L.acc, e), term);
  }
}

// the pending increment of a GL/BAOAB leg about to step (register version)
template <int IG, class Pend>
__device__ __forceinline__ void leg_settle(ALeg& L, const Pend& P) {
  if (IG != kSE && L.np >= 3 && L.np <= Pend::kCap)  // <= 2: Horner == backward sum
    L.acc = backward_sum(L.np, [&](int r) { return P.t[r]; }, [&](int r) { return P.e[r]; });
}

// coupling.hpp:158-173 — the leg's step with the equivalent normal of its
// pending increment; sc = the coarse leg's own parity (1 for the fine leg).
template <int IG, int PROF, int FAST>
__device__ __forceinline__ bool leg_take(ALeg& L, bool is_coarse, const DevModel& m, bool& bad) {
  using O = Ops<FAST>;
  const double inc = is_coarse ? sgn(L.s.par, L.acc) : L.acc;
  bool ok;
  if (IG == kSE) {
    const double sqh = O::sqrt(L.h_cur, bad);
    ok = se_update<FAST>(L.s, L.c, L.h_cur, sqh, O::div(inc, sqh, bad), m, bad);
    L.c = coeffs<PROF, FAST>(L.s.x, m, bad);
  } else {
    double e, sd;
    ou_terms<FAST>(L.c.lam, L.h_cur, e, sd, bad);
    const double xi_eq = O::div(inc, sd, bad);
    if (IG == kGL) {
      ok = gl_update<FAST>(L.s, L.c, L.h_cur, xi_eq, e, sd, m, bad);
      L.c = coeffs<PROF, FAST>(L.s.x, m, bad);
    } else {
      int pm;
      ok = baoab_step<PROF, FAST>(L.s, L.c, L.h_cur, mul(0.5, L.h_cur), xi_eq, false, pm, m, bad);
    }
  }
  L.t = L.t_next;
  ++L.steps;
  L.acc = 0.0;
  L.np = 0;
  return ok;
}

// coupling.hpp:137-214 — coupled pair on non-nested adaptive grids.
// DEEP = false: pending terms in local memory; a leg that exceeds kPendLocal
// sets `deep` and ends the sample (its result is discarded: K1D recomputes it
// with DEEP = true and global-memory storage at `scratch`).
template <int IG, int PROF, int FAST, bool DEEP = false>
__device__ __forceinline__ PathOut run_pair_adaptive(const KernelArgs& a, uint64_t idx,
                                                     long long& steps, bool& bad, bool& deep,
                                                     double* scratch = nullptr) {
  using O = Ops<FAST>;
  const DevModel& m = a.model;
  const double T = a.T, hb = a.h_base, hb2 = mul(2.0, a.h_base);
  const double lam_ref = coeffs<PROF, FAST>(a.x_adapt, m, bad).lam;
  ALeg f;
  f.s = {a.x0, a.u0, 1, 0};
  f.c = coeffs<PROF, FAST>(a.x0, m, bad);
  f.t = 0.0;
  f.acc = 0.0;
  f.steps = 0;
  f.np = 0;
  f.done = false;
  ALeg c = f;
  leg_schedule<FAST>(f, hb, T, lam_ref, bad);
  leg_schedule<FAST>(c, hb2, T, lam_ref, bad);
  SeqNoise<PhiloxKey> ns;
  using Pend = typename std::conditional<DEEP, PendGlobal, PendLocal>::type;
  Pend pf, pc;
  if constexpr (DEEP) {
    pf = {scratch, scratch + kPendDeep};
    pc = {scratch + 2 * kPendDeep, scratch + 3 * kPendDeep};
  }
  (void)scratch;
  const bool signs = a.signs_on;
  PathOut o;
  o.ok = true;
  double t = 0.0;
  long long iter = 0;
  while (!f.done || !c.done) {
    const double ta = f.done ? T : f.t_next, tb = c.done ? T : c.t_next;
    const double tau = (tb < ta) ? tb : ta;
    const double dt = sub(tau, t);
    if (dt > 0.0) {
      const double xi = ns.next(idx, a.key);
      const double sqrt_dt = IG == kSE ? O::sqrt(dt, bad) : 0.0;
      const int sf = signs ? f.s.par : 1;
      if (!f.done) leg_push<IG, FAST>(f, pf, xi, dt, sqrt_dt, bad, deep);
      if (!c.done) leg_push<IG, FAST>(c, pc, sgn(sf, xi), dt, sqrt_dt, bad, deep);
      if (!DEEP && deep) break;
    }
    if (!f.done && f.t_next == tau) {
      leg_settle<IG>(f, pf);
      if (!leg_take<IG, PROF, FAST>(f, false, m, bad)) { o.ok = false; break; }
      if (f.t_next >= T) f.done = true;
      else leg_schedule<FAST>(f, hb, T, lam_ref, bad);
    }
    if (!c.done && c.t_next == tau) {
      leg_settle<IG>(c, pc);
      if (!leg_take<IG, PROF, FAST>(c, true, m, bad)) { o.ok = false; break; }
      if (c.t_next >= T) c.done = true;
      else leg_schedule<FAST>(c, hb2, T, lam_ref, bad);
    }
    t = tau;
    if (++iter > a.max_iter) { o.ok = false; break; }
    if (FAST && bad) break;
  }
  o.f = f.s;
  o.c = c.s;
  steps = f.steps + c.steps;
  return o;
}

template <int IG, int PROF, bool COUPLED, int FAST>
__device__ __forceinline__ PathOut run_adaptive(const KernelArgs& a, uint64_t idx,
                                                long long& steps, bool& bad, bool& deep) {
  if (COUPLED) return run_pair_adaptive<IG, PROF, FAST>(a, idx, steps, bad, deep);
  return run_path_adaptive<IG, PROF, FAST>(a, idx, steps, bad);
}

// Fast variant first when the host certified tame parameters; a miss
// recomputes the sample exactly (same policy as sample()).
// deep: a leg exceeded kPendLocal pending sub-intervals (result invalid; the
// caller queues the sample for K1D).
template <int IG, int PROF, bool COUPLED>
__device__ __forceinline__ PathOut sample_adaptive(const KernelArgs& a, uint64_t idx,
                                                   long long& steps, bool& deep) {
  bool bad = false;
  deep = false;
  if (a.fast) {
    PathOut o = a.fast == kFastUnit
                    ? run_adaptive<IG, PROF, COUPLED, kFastUnit>(a, idx, steps, bad, deep)
                    : run_adaptive<IG, PROF, COUPLED, 1>(a, idx, steps, bad, deep);
    if (!bad || deep) return o;
    bad = false;
  }
  return run_adaptive<IG, PROF, COUPLED, 0>(a, idx, steps, bad, deep);
}

// ----------------------------------------- persistent adaptive sampler
// Adaptive samples take data-dependent numbers of steps, so one thread per
// sample leaves most lanes of a warp idle behind its slowest sample (ncu:
// 9.75 of 32 lanes active).  K1P instead runs a fixed grid of resident
// threads, each of which pulls sample indices from a warp-aggregated atomic
// work counter and advances its current sample ONE schedule event per loop
// iteration (one leg step on the pair's merged timeline), starting the next
// sample in the same iteration its previous one ended.  Lanes therefore stay
// busy until the queue drains.  Results go to per-sample slots (QoI value,
// steps), and K1T reduces them in the same fixed 256-sample tile tree as the
// uniform sampler, so the sums do not depend on which thread ran which
// sample.  Fast-path misses are queued and recomputed exactly by K1R.

// Warp-aggregated fetch-and-add: one atomic per group of lanes asking.
__device__ __forceinline__ int64_t grab_sample(unsigned long long* ctr) {
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(mask));
  base = __shfl_sync(mask, base, leader);
  return int64_t(base) + __popc(mask & ((1u << lane) - 1u));
}

template <bool COUPLED>
__device__ __forceinline__ void adaptive_store(const KernelArgs& a, int64_t j, const PathOut& o,
                                               long long steps) {
  if (a.qoi_kind == 3) store_pos(a, j, o.ok, o);
  else a.ad_y[j] = o.ok ? sample_y<COUPLED>(a, o) : 0.0;
  a.ad_steps[j] = o.ok ? steps : -1;
}

// State of one pair in flight.  The fields every event touches for BOTH legs
// (schedule time, pending increment, lambda, parity, done) live in registers
// (LegHot); the rest of a leg (position, velocity, sde_coeffs, step sizes,
// counters) lives in shared memory (LegStore, [field][leg][thread]: no bank
// conflicts) and is loaded only for the leg that steps.  Selecting the
// stepping leg then costs a shared-memory address instead of a select per
// register of both legs, and the register footprint drops by one leg.
// pend_c: the coarse leg still has to step at tau (a coincident grid point:
// the reference steps fine then coarse in the same iteration; here they are
// two consecutive events, in the same order, without a draw).
struct LegHot {
  double t_next, acc, lam;
  int par, np;
  bool done;
};
enum { kColdX, kColdU, kColdSu2, kColdSig, kColdDsu2, kColdRsu2, kColdT, kColdH, kColdN };
// Threads per CTA of the persistent sampler.  Its results go to per-sample
// slots (K1T reduces them in 256-sample tiles), so the CTA size is free: it is
// chosen for the most resident warps at the kernel's register count.
#ifndef ABLMC_AD_THREADS
#define ABLMC_AD_THREADS 256
#endif
constexpr int kAdThreads = ABLMC_AD_THREADS;
struct LegStore {
  double d[kColdN][2][kAdThreads];
  long long steps[2][kAdThreads];
  int nrefl[2][kAdThreads];
  double pt[kPend][2][kAdThreads], pe[kPend][2][kAdThreads];  // GL/BAOAB only (SE launches without)
};
template <int IG>
constexpr size_t leg_store_bytes() {
  return IG == kSE ? offsetof(LegStore, pt) : sizeof(LegStore);
}

struct PairSM {
  LegHot f, c;
  double t, tau;
  long long iter;
  BufNoise ns;
  bool pend_c;
};

__device__ __forceinline__ LegHot leg_hot(const ALeg& L) {
  return {L.t_next, L.acc, L.c.lam, L.s.par, L.np, L.done};
}

__device__ __forceinline__ void leg_store(LegStore& st, int leg, const ALeg& L) {
  const int i = threadIdx.x;
  st.d[kColdX][leg][i] = L.s.x;
  st.d[kColdU][leg][i] = L.s.u;
  st.d[kColdSu2][leg][i] = L.c.su2;
  st.d[kColdSig][leg][i] = L.c.sig;
  st.d[kColdDsu2][leg][i] = L.c.dsu2;
  st.d[kColdRsu2][leg][i] = L.c.rsu2;
  st.d[kColdT][leg][i] = L.t;
  st.d[kColdH][leg][i] = L.h_cur;
  st.steps[leg][i] = L.steps;
  st.nrefl[leg][i] = L.s.nrefl;
}

__device__ __forceinline__ ALeg leg_load(const LegStore& st, int leg, const LegHot& h) {
  const int i = threadIdx.x;
  ALeg L;
  L.s = {st.d[kColdX][leg][i], st.d[kColdU][leg][i], h.par, st.nrefl[leg][i]};
  L.c.su2 = st.d[kColdSu2][leg][i];
  L.c.lam = h.lam;
  L.c.sig = st.d[kColdSig][leg][i];
  L.c.dsu2 = st.d[kColdDsu2][leg][i];
  L.c.rsu2 = st.d[kColdRsu2][leg][i];
  L.t = st.d[kColdT][leg][i];
  L.t_next = h.t_next;
  L.h_cur = st.d[kColdH][leg][i];
  L.acc = h.acc;
  L.steps = st.steps[leg][i];
  L.np = h.np;
  L.done = h.done;
  return L;
}

// pending-increment update on the hot fields (leg_push on LegHot); GL/BAOAB
// terms go to shared memory (overflow: FAST recomputes the sample in K1R)
template <int IG, int FAST>
__device__ __forceinline__ void hot_push(LegHot& L, LegStore& st, PendSpill& sp, int leg,
                                         double xi_s, double dt, double sqrt_dt, bool& bad,
                                         bool& deep) {
  if (IG == kSE) {
    L.acc = add(L.acc, mul(xi_s, sqrt_dt));
  } else {
    double e, sd;
    ou_terms<FAST>(L.lam, dt, e, sd, bad);
    const double term = mul(xi_s, sd);
    if (L.np < kPend) {
      st.pt[L.np][leg][threadIdx.x] = term;
      st.pe[L.np][leg][threadIdx.x] = e;
    } else if (L.np < kPendLocal) {
      sp.t[leg][L.np - kPend] = term;
      sp.e[leg][L.np - kPend] = e;
    } else {
      deep = true;  // the sample goes to K1D
    }
    ++L.np;
    L.acc = add(mul(L.acc, e), term);
  }
}

// One event of simulate_pair_adaptive (coupling.hpp:175-211).  Returns true
// when the sample is finished (both legs at T, or failed).
template <int IG, int PROF, int FAST>
__device__ __forceinline__ bool pair_event(PairSM& S, LegStore& st, PendSpill& sp,
                                           const KernelArgs& a, uint64_t idx, double lam_ref,
                                           bool& ok, bool& bad, bool& deep) {
  using O = Ops<FAST>;
  const double T = a.T;
  bool take_fine;
  if (!S.pend_c) {
    const double ta = S.f.done ? T : S.f.t_next, tb = S.c.done ? T : S.c.t_next;
    S.tau = (tb < ta) ? tb : ta;
    const double dt = sub(S.tau, S.t);
    if (dt > 0.0) {
      const double xi = S.ns.next(idx, a.key);
      const double sqrt_dt = IG == kSE ? O::sqrt(dt, bad) : 0.0;
      const int sf = a.signs_on ? S.f.par : 1;
      if (!S.f.done) hot_push<IG, FAST>(S.f, st, sp, 0, xi, dt, sqrt_dt, bad, deep);
      if (!S.c.done) hot_push<IG, FAST>(S.c, st, sp, 1, sgn(sf, xi), dt, sqrt_dt, bad, deep);
      if (deep) return true;
    }
    take_fine = !S.f.done && S.f.t_next == S.tau;
    S.pend_c = take_fine && !S.c.done && S.c.t_next == S.tau;
  } else {
    take_fine = false;
    S.pend_c = false;
  }
  const int leg = take_fine ? 0 : 1;
  ALeg W = leg_load(st, leg, take_fine ? S.f : S.c);
  // (<= 2 pending terms: the Horner form already equals the backward sum)
  if (IG != kSE && W.np >= 3 && W.np <= kPendLocal) {
    const int i = threadIdx.x;
    W.acc = backward_sum(
        W.np, [&](int r) { return r < kPend ? st.pt[r][leg][i] : sp.t[leg][r - kPend]; },
        [&](int r) { return r < kPend ? st.pe[r][leg][i] : sp.e[leg][r - kPend]; });
  }
  ok = leg_take<IG, PROF, FAST>(W, !take_fine, a.model, bad);
  if (W.t_next >= T) W.done = true;
  else leg_schedule<FAST>(W, take_fine ? a.h_base : mul(2.0, a.h_base), T, lam_ref, bad);
  leg_store(st, leg, W);
  const LegHot hw = leg_hot(W);
  if (take_fine) S.f = hw;
  else S.c = hw;
  if (!S.pend_c) {  // end of the reference's loop iteration
    S.t = S.tau;
    if (++S.iter > a.max_iter) ok = false;
  }
  return !ok || (S.f.done && S.c.done) || (FAST && bad);
}

struct PathSM {
  PState s;
  Coef c;
  double t;
  long long steps;
  BufNoise ns;
};

// One step of simulate_path_adaptive (coupling.hpp:41-49).
template <int IG, int PROF, int FAST>
__device__ __forceinline__ bool path_event(PathSM& S, const KernelArgs& a, uint64_t idx,
                                           double lam_ref, bool& ok, bool& bad) {
  using O = Ops<FAST>;
  const DevModel& m = a.model;
  const double T = a.T;
  double h = adaptive_h<FAST>(S.c.lam, a.h_base, lam_ref, bad);
  if (add(S.t, h) >= T) h = sub(T, S.t);
  const double xi = S.ns.next(idx, a.key);
  if (IG == kSE) {
    ok = se_update<FAST>(S.s, S.c, h, O::sqrt(h, bad), xi, m, bad);
    S.c = coeffs<PROF, FAST>(S.s.x, m, bad);
  } else if (IG == kGL) {
    double e, sd;
    ou_terms<FAST>(S.c.lam, h, e, sd, bad);
    ok = gl_update<FAST>(S.s, S.c, h, xi, e, sd, m, bad);
    S.c = coeffs<PROF, FAST>(S.s.x, m, bad);
  } else {
    int pm;
    ok = baoab_step<PROF, FAST>(S.s, S.c, h, mul(0.5, h), xi, false, pm, m, bad);
  }
  S.t = (add(S.t, h) >= T) ? T : add(S.t, h);
  if (++S.steps > a.max_iter) ok = false;
  return !ok || !(S.t < T) || (FAST && bad);
}

#ifndef ABLMC_MINB_ADAPTIVE
#define ABLMC_MINB_ADAPTIVE 2  // 2 CTAs/SM (<= 128 registers, no spills)
#endif
#ifndef ABLMC_MINB_ADAPTIVE_SE
#define ABLMC_MINB_ADAPTIVE_SE ABLMC_MINB_ADAPTIVE
#endif
template <int IG, int PROF, bool COUPLED, int FAST>
__global__ void __launch_bounds__(kAdThreads, IG == kSE ? ABLMC_MINB_ADAPTIVE_SE : ABLMC_MINB_ADAPTIVE)
    k_adaptive_persistent(const KernelArgs a) {
  const DevModel& m = a.model;
  bool bad = false;
  const double lam_ref = coeffs<PROF, FAST>(a.x_adapt, m, bad).lam;
  // every sample starts from the same state and the same first schedule
  ALeg f0;
  f0.s = {a.x0, a.u0, 1, 0};
  f0.c = coeffs<PROF, FAST>(a.x0, m, bad);
  f0.t = 0.0;
  f0.acc = 0.0;
  f0.steps = 0;
  f0.np = 0;
  f0.done = false;
  ALeg c0 = f0;
  if (COUPLED) {
    leg_schedule<FAST>(f0, a.h_base, a.T, lam_ref, bad);
    leg_schedule<FAST>(c0, mul(2.0, a.h_base), a.T, lam_ref, bad);
  }
  const bool bad0 = bad;
  bool deep = false;
  extern __shared__ double4 ad_smem[];
  LegStore& st = *reinterpret_cast<LegStore*>(ad_smem);  // COUPLED only (dynamic size 0 else)
  PairSM P;
  PendSpill sp;
  PathSM Q;
  auto start = [&]() {
    if (COUPLED) {
      leg_store(st, 0, f0);
      leg_store(st, 1, c0);
      P.f = leg_hot(f0);
      P.c = leg_hot(c0);
      P.t = 0.0;
      P.iter = 0;
      P.ns.reset();
      P.pend_c = false;
    } else {
      Q.s = f0.s;
      Q.c = f0.c;
      Q.t = 0.0;
      Q.steps = 0;
      Q.ns.reset();
    }
    bad = bad0;
    deep = false;
  };
  int64_t j = grab_sample(a.ad_ctrl);
  if (j < a.n) start();
  while (j < a.n) {
    const uint64_t idx = uint64_t(a.first + a.offset + j);
    refill_if_any_empty(COUPLED ? P.ns : Q.ns, true, idx, a.key);
    bool ok = true;
    const bool fin = COUPLED ? pair_event<IG, PROF, FAST>(P, st, sp, a, idx, lam_ref, ok, bad, deep)
                             : path_event<IG, PROF, FAST>(Q, a, idx, lam_ref, ok, bad);
    if (fin) {
      if (deep) {
        a.ad_deep[atomicAdd(a.ad_ctrl + 2, 1ull)] = j;
      } else if (FAST && bad) {
        a.ad_redo[atomicAdd(a.ad_ctrl + 1, 1ull)] = j;
      } else {
        PathOut o;
        long long steps;
        if (COUPLED) {
          const int i = threadIdx.x;
          o.f = {st.d[kColdX][0][i], st.d[kColdU][0][i], P.f.par, st.nrefl[0][i]};
          o.c = {st.d[kColdX][1][i], st.d[kColdU][1][i], P.c.par, st.nrefl[1][i]};
          steps = st.steps[0][i] + st.steps[1][i];
        } else {
          o.f = Q.s;
          o.c = Q.s;
          steps = Q.steps;
        }
        o.ok = ok;
        adaptive_store<COUPLED>(a, j, o, steps);
      }
      j = grab_sample(a.ad_ctrl);
      if (j < a.n) start();
    }
  }
}

// K1R: exact recomputation of the samples whose fast path missed.
template <int IG, int PROF, bool COUPLED>
__global__ void __launch_bounds__(kTile) k_adaptive_redo(const KernelArgs a) {
  const int64_t nr = int64_t(a.ad_ctrl[1]);
  for (int64_t r = int64_t(blockIdx.x) * kTile + threadIdx.x; r < nr;
       r += int64_t(gridDim.x) * kTile) {
    const int64_t j = a.ad_redo[r];
    bool bad = false, deep = false;
    long long steps = 0;
    const PathOut o = run_adaptive<IG, PROF, COUPLED, 0>(a, uint64_t(a.first + a.offset + j),
                                                         steps, bad, deep);
    if (deep) a.ad_deep[atomicAdd(a.ad_ctrl + 2, 1ull)] = j;
    else adaptive_store<COUPLED>(a, j, o, steps);
  }
}

__device__ __forceinline__ StateOut state_out(const PathOut& o, long long steps) {
  StateOut s;
  s.fx = o.f.x;
  s.fu = o.f.u;
  s.fpar = o.f.par;
  s.fn = o.f.nrefl;
  s.cx = o.c.x;
  s.cu = o.c.u;
  s.cpar = o.c.par;
  s.cn = o.c.nrefl;
  s.ok = o.ok ? 1 : 0;
  s.steps = int(steps);
  return s;
}

// K1D: the pairs with more than kPendLocal pending sub-intervals on a leg,
// recomputed exactly with their pending terms in global memory (a slice of
// ad_scratch per thread; ABLMC_DEEP_THREADS threads stride over the list).
// STATES: write the oracle-mode record instead of the per-sample slots.
template <int IG, int PROF, bool STATES>
__global__ void __launch_bounds__(64) k_adaptive_deep(const KernelArgs a, StateOut* __restrict__ out) {
  const int64_t nd = int64_t(a.ad_ctrl[2]);
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double* scratch = a.ad_scratch + tid * 4 * kPendDeep;
  for (int64_t r = tid; r < nd; r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = a.ad_deep[r];
    bool bad = false, deep = false;
    long long steps = 0;
    const PathOut o = run_pair_adaptive<IG, PROF, 0, true>(a, uint64_t(a.first + a.offset + j),
                                                           steps, bad, deep, scratch);
    if (STATES) out[j] = state_out(o, steps);
    else adaptive_store<true>(a, j, o, steps);
  }
}

// K1T: tile partials of the per-sample results (same tree as tile_epilogue).
__global__ void __launch_bounds__(kTile) k_adaptive_tiles(const KernelArgs a,
                                                          double* __restrict__ tile_sums,
                                                          long long* __restrict__ tile_cnt) {
  const int64_t j = int64_t(blockIdx.x) * kTile + threadIdx.x;
  const bool active = j < a.n;
  const bool binned = a.qoi_kind == 3;
  const long long steps = active ? a.ad_steps[j] : 0;
  const bool good = active && steps >= 0;
  tile_prologue();
  tile_reduce<false>(a, active, good, (good && !binned) ? a.ad_y[j] : 0.0, steps, binned,
                     tile_sums, tile_cnt);
}

template <int IG, int PROF, bool COUPLED>
cudaError_t launch_adaptive(const KernelArgs& a, double* tile_sums, long long* tile_cnt,
                            cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.ad_ctrl, 0, 3 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.n + kTile - 1) / kTile;
  const bool fast = a.fast != 0;
  const size_t smem = COUPLED ? leg_store_bytes<IG>() : 0;
  auto run = [&](auto kernel) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kAdThreads, smem);
    const int64_t ctas = (a.n + kAdThreads - 1) / kAdThreads;
    const unsigned grid = unsigned(std::min<int64_t>(ctas, int64_t(sms) * std::max(per_sm, 1)));
    kernel<<<grid, kAdThreads, smem, st>>>(a);
  };
  if (fast && a.fast == kFastUnit) run(k_adaptive_persistent<IG, PROF, COUPLED, kFastUnit>);
  else if (fast) run(k_adaptive_persistent<IG, PROF, COUPLED, 1>);
  else run(k_adaptive_persistent<IG, PROF, COUPLED, 0>);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (fast) {
    k_adaptive_redo<IG, PROF, COUPLED><<<unsigned(sms), kTile, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (COUPLED && IG != kSE) {  // K1D (exits at once when no pair went deep)
    k_adaptive_deep<IG, PROF, false><<<ABLMC_DEEP_THREADS / 64, 64, 0, st>>>(a, nullptr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  k_adaptive_tiles<<<unsigned(tiles), kTile, 0, st>>>(a, tile_sums, tile_cnt);
  return cudaGetLastError();
}

template <int IG, int PROF, bool COUPLED>
__global__ void __launch_bounds__(kTile) k_states_adaptive(const KernelArgs a,
                                                           StateOut* __restrict__ out) {
  const int64_t j = int64_t(blockIdx.x) * kTile + threadIdx.x;
  if (j >= a.n) return;
  long long steps = 0;
  bool deep;
  const PathOut o =
      sample_adaptive<IG, PROF, COUPLED>(a, uint64_t(a.first + a.offset + j), steps, deep);
  if (deep) a.ad_deep[atomicAdd(a.ad_ctrl + 2, 1ull)] = j;  // K1D writes out[j]
  else out[j] = state_out(o, steps);
}

template <int IG, int PROF>
cudaError_t level_t(const KernelArgs& a, bool coupled, double* ts, long long* tc, cudaStream_t st) {
  return coupled ? launch_adaptive<IG, PROF, true>(a, ts, tc, st)
                 : launch_adaptive<IG, PROF, false>(a, ts, tc, st);
}

template <int IG, int PROF>
cudaError_t states_t(const KernelArgs& a, bool coupled, StateOut* out, cudaStream_t st) {
  const dim3 g{unsigned((a.n + kTile - 1) / kTile)};
  cudaError_t e = cudaMemsetAsync(a.ad_ctrl, 0, 3 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (coupled) k_states_adaptive<IG, PROF, true><<<g, kTile, 0, st>>>(a, out);
  else k_states_adaptive<IG, PROF, false><<<g, kTile, 0, st>>>(a, out);
  if ((e = cudaGetLastError()) != cudaSuccess || !coupled || IG == kSE) return e;
  k_adaptive_deep<IG, PROF, true><<<ABLMC_DEEP_THREADS / 64, 64, 0, st>>>(a, out);
  return cudaGetLastError();
}

template <int IG>
cudaError_t level_p(const KernelArgs& a, bool coupled, double* ts, long long* tc, cudaStream_t st) {
  switch (a.model.profile) {
    case kProfileConstant: return level_t<IG, kProfileConstant>(a, coupled, ts, tc, st);
    case kProfileFloored: return level_t<IG, kProfileFloored>(a, coupled, ts, tc, st);
    default: return level_t<IG, kProfileReference>(a, coupled, ts, tc, st);
  }
}

template <int IG>
cudaError_t states_p(const KernelArgs& a, bool coupled, StateOut* out, cudaStream_t st) {
  switch (a.model.profile) {
    case kProfileConstant: return states_t<IG, kProfileConstant>(a, coupled, out, st);
    case kProfileFloored: return states_t<IG, kProfileFloored>(a, coupled, out, st);
    default: return states_t<IG, kProfileReference>(a, coupled, out, st);
  }
}

}  // namespace

cudaError_t upload_log_table_adaptive() { return upload_log_table_here(); }

cudaError_t launch_adaptive_level(const KernelArgs& a, int ig, bool coupled, double* tile_sums,
                                  long long* tile_cnt, cudaStream_t st) {
  switch (ig) {
    case kSE: return level_p<kSE>(a, coupled, tile_sums, tile_cnt, st);
    case kGL: return level_p<kGL>(a, coupled, tile_sums, tile_cnt, st);
    default: return level_p<kBAOAB>(a, coupled, tile_sums, tile_cnt, st);
  }
}

cudaError_t launch_adaptive_states(const KernelArgs& a, int ig, bool coupled, StateOut* out,
                                   cudaStream_t st) {
  switch (ig) {
    case kSE: return states_p<kSE>(a, coupled, out, st);
    case kGL: return states_p<kGL>(a, coupled, out, st);
    default: return states_p<kBAOAB>(a, coupled, out, st);
  }
}
