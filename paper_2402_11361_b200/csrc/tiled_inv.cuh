// Tiled layout of each macro's explicit Schur-complement inverse S^-1.
//
// The reference keeps S^-1 explicitly (np.linalg.inv, condense.py:62-70) and
// applies it as a batched matvec (condense.py:80-83).  On the device S^-1 is
// stored in the order the streaming apply reads it: row blocks of TI_RB = 64
// rows, each block as consecutive column tiles of TI_CW = 32 columns
// (row-major inside a tile, the last tile narrower), every tile padded to an
// even number of doubles so that one tile is one 16-byte aligned bulk copy
// holding all rows of its block.  A warp that owns rows 8w..8w+7 of a block
// can keep its partial sums in registers across all column tiles: the
// product needs no barrier between tiles.
#pragma once
#include "common.cuh"
#include "packed_lu.cuh"

namespace mhdg {

constexpr int TI_RB = 64;
constexpr int TI_CW = 32;

__host__ __device__ __forceinline__ long long ti_even(long long x) { return x + (x & 1); }

__host__ __device__ inline int ti_nblk(int n) { return (n + TI_RB - 1) / TI_RB; }

__host__ __device__ inline int ti_rows(int n, int b) { return (n - TI_RB * b) < TI_RB ? n - TI_RB * b : TI_RB; }

// doubles of one row block (nb rows x n columns in column tiles)
__host__ __device__ inline long long ti_block_size(int nb, int n) {
  long long o = 0;
  for (int c = 0; c < n; c += TI_CW) o += ti_even((long long)nb * ((n - c) < TI_CW ? n - c : TI_CW));
  return o;
}

__host__ __device__ inline long long ti_size(int n) {
  long long o = 0;
  for (int b = 0; b < ti_nblk(n); ++b) o += ti_block_size(ti_rows(n, b), n);
  return o;
}

// offset of row block b (all blocks before it are full TI_RB rows)
__host__ __device__ inline long long ti_block_off(int n, int b) { return (long long)b * ti_block_size(TI_RB, n); }

// offset of element (r, c) of S^-1
__host__ __device__ __forceinline__ long long ti_idx(int n, int r, int c) {
  const int b = r / TI_RB, rl = r - b * TI_RB, nb = ti_rows(n, b);
  const int j = c / TI_CW, c0 = j * TI_CW, w = (n - c0) < TI_CW ? n - c0 : TI_CW;
  // tiles before j are full width: nb * TI_CW doubles (even)
  return ti_block_off(n, b) + (long long)j * nb * TI_CW + (long long)rl * w + (c - c0);
}

// CTA-wide out = S^-1 v (v, out in shared memory, length n; synchronous loads)
// (packed-LU factors: see factor_solve_cta in local_ops.cuh)
__device__ inline void ti_gemv_cta(const double* __restrict__ F, int n, const double* v, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < n; r += nw) {
    double acc = 0.0;
    for (int c = lane; c < n; c += 32) acc += __ldg(F + ti_idx(n, r, c)) * v[c];
    acc = warp_sum(acc);
    if (lane == 0) out[r] = acc;
  }
  __syncthreads();
}

// out = S^-1 v for macro `mac` with either factor kind (mhdg_factors.kind):
// explicit tiled inverse (GEMV) or packed LU (block triangular solves).
// v is clobbered for the LU kind.  Ends with a CTA barrier.
__device__ inline void factor_solve_cta(const mhdg_factors& fac, int mac, int n, double* v, double* out) {
  if (fac.kind == 1) {
    plu_solve_cta(fac.lu + (size_t)mac * plu_size(n), fac.perm + (size_t)mac * n, n, v, out);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = v[i];
    __syncthreads();
  } else {
    ti_gemv_cta(fac.lu + (size_t)mac * ti_size(n), n, v, out);
  }
}

}  // namespace mhdg
