// collective.cu — device side of the sharded accumulate.
//
// A batch of accumulate requests (one MLMC allocation round: several levels)
// leaves each rank's super-block partials in sb_sums / sb_cnt (merge_tail),
// request q's rows at [pbase_q, pbase_q + own rows).  For the ONE all-gather
// of the batch they are packed into rows of W = 2 dim + 3 doubles (sums, then
// the three int64 counts {n, failed, cost_steps} as bit patterns) followed by
// one status row (this rank's return code), so every rank sends the same
// (cap_total + 1) W doubles.  After the all-gather every rank holds every
// rank's rows and merges them in global super-block order: the fold of the
// reference's block-order merge (stats.hpp:133-135) over the same fixed
// partials, i.e. the same bits as the single-GPU call for any world size.
#include <cuda_runtime.h>

#include <algorithm>

#include "ablmc_device.cuh"
#include "kernels.h"

namespace {

using namespace ablmc_dev;

__global__ void k_pack_rows(int64_t rows, int dim2, const double* __restrict__ sb_sums,
                            const long long* __restrict__ sb_cnt, double* __restrict__ send,
                            long long status) {
  const int64_t W = dim2 + kCnt;
  const int64_t total = (rows + 1) * W;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / W, c = i - r * W;
    double v;
    if (r == rows) v = __longlong_as_double(c == 0 ? status : 0LL);  // status row
    else if (c < dim2) v = sb_sums[r * dim2 + c];
    else v = __longlong_as_double(sb_cnt[r * kCnt + (c - dim2)]);
    send[i] = v;
  }
}

// Rows of rank w for a request of n_sb super-blocks (balanced contiguous
// split, capi.cu shard_range).
__device__ __forceinline__ int64_t rows_of(int64_t n_sb, int w, int world) {
  return n_sb / world + (w < n_sb % world ? 1 : 0);
}

// Device-resident merge of one request's gathered rows, in global
// super-block order (K3 k_merge_super's fold over the same rows): one thread
// per column.  res_status: the first nonzero rank status, else 0.
__global__ void k_merge_gathered(int world, int64_t cap_total, int64_t n_sb, int64_t pbase,
                                 int dim2, const double* __restrict__ recv,
                                 double* __restrict__ res_sums, long long* __restrict__ res_cnt,
                                 long long* __restrict__ res_status) {
  const int64_t W = dim2 + kCnt;
  const int64_t block = (cap_total + 1) * W;
  for (int c = threadIdx.x; c < dim2 + kCnt; c += blockDim.x) {
    double v = 0.0;
    long long n = 0;
    for (int w = 0; w < world; ++w) {
      const double* base = recv + w * block + pbase * W + c;
      const int64_t rw = rows_of(n_sb, w, world);
      for (int64_t r = 0; r < rw; ++r) {
        if (c < dim2) v = add(v, base[r * W]);
        else n += __double_as_longlong(base[r * W]);
      }
    }
    if (c < dim2) res_sums[c] = v;
    else res_cnt[c - dim2] = n;
  }
  if (threadIdx.x == 0) {
    long long st = 0;
    for (int w = 0; w < world && st == 0; ++w)
      st = __double_as_longlong(recv[w * block + cap_total * W]);
    *res_status = st;
  }
}

}  // namespace

cudaError_t launch_pack_rows(int64_t rows, int dim, const double* sb_sums, const long long* sb_cnt,
                             double* send, long long status, cudaStream_t st) {
  const int64_t total = (rows + 1) * (2 * dim + kCnt);
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148));
  k_pack_rows<<<blocks, 256, 0, st>>>(rows, 2 * dim, sb_sums, sb_cnt, send, status);
  return cudaGetLastError();
}

cudaError_t launch_merge_gathered(int world, int64_t cap_total, int64_t n_sb, int64_t pbase,
                                  int dim, const double* recv, double* res_sums,
                                  long long* res_cnt, long long* res_status, cudaStream_t st) {
  const int threads = (2 * dim + kCnt) <= 32 ? 32 : ((2 * dim + kCnt) <= 128 ? 128 : 256);
  k_merge_gathered<<<1, threads, 0, st>>>(world, cap_total, n_sb, pbase, 2 * dim, recv, res_sums,
                                          res_cnt, res_status);
  return cudaGetLastError();
}
