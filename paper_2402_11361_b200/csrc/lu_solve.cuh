// Blocked forward/back substitution with one macro's LU factors, CTA-wide.
#pragma once
#include "common.cuh"

namespace mhdg {

constexpr int TRI_NB = 32;

// In-place y <- U^-1 L^-1 P y for a row-major n x n factor (L unit lower).
// y and tmp are shared-memory vectors of length n; dblk is shared scratch of
// TRI_NB*(TRI_NB+1) doubles.  Row blocks of 32: every warp streams the
// already-solved part of its rows (coalesced along the row), then warp 0
// finishes the 32x32 diagonal triangle out of shared memory.
__device__ void lu_solve_cta(const double* __restrict__ LU, const int* __restrict__ perm, int n,
                             double* y, double* tmp, double* dblk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < n; i += blockDim.x) tmp[i] = y[__ldg(perm + i)];
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) y[i] = tmp[i];
  __syncthreads();

  // forward: unit lower
  for (int b0 = 0; b0 < n; b0 += TRI_NB) {
    const int nb = min(TRI_NB, n - b0);
    for (int rr = warp; rr < nb; rr += nw) {
      const double* a = LU + (size_t)(b0 + rr) * n;
      double acc = 0.0;
      for (int c = lane; c < b0; c += 32) acc += __ldg(a + c) * y[c];
      if (lane < nb) dblk[rr * (TRI_NB + 1) + lane] = __ldg(a + b0 + lane);
      acc = warp_sum(acc);
      if (lane == 0) y[b0 + rr] -= acc;
    }
    __syncthreads();
    if (warp == 0) {
      double yr = lane < nb ? y[b0 + lane] : 0.0;
      for (int j = 0; j < nb - 1; ++j) {
        double yj = __shfl_sync(MHDG_FULL, yr, j);
        if (lane > j && lane < nb) yr -= dblk[lane * (TRI_NB + 1) + j] * yj;
      }
      if (lane < nb) y[b0 + lane] = yr;
    }
    __syncthreads();
  }
  // backward: upper with diagonal
  for (int b1 = n; b1 > 0; b1 -= TRI_NB) {
    const int b0 = max(0, b1 - TRI_NB), nb = b1 - b0;
    for (int rr = warp; rr < nb; rr += nw) {
      const double* a = LU + (size_t)(b0 + rr) * n;
      double acc = 0.0;
      for (int c = b1 + lane; c < n; c += 32) acc += __ldg(a + c) * y[c];
      if (lane < nb) dblk[rr * (TRI_NB + 1) + lane] = __ldg(a + b0 + lane);
      acc = warp_sum(acc);
      if (lane == 0) y[b0 + rr] -= acc;
    }
    __syncthreads();
    if (warp == 0) {
      double yr = lane < nb ? y[b0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        double xj = __shfl_sync(MHDG_FULL, yr, j);
        xj /= dblk[j * (TRI_NB + 1) + j];
        if (lane == j) yr = xj;
        if (lane < j) yr -= dblk[lane * (TRI_NB + 1) + j] * xj;
      }
      if (lane < nb) y[b0 + lane] = yr;
    }
    __syncthreads();
  }
}

}  // namespace mhdg
