// Packed LU factor layout consumed by the trace apply.
//
// After LU with partial pivoting (P S = L U, L unit lower), each macro's
// factor is re-laid out in the order the two triangular solves read it, in
// 64-row blocks b = 0..nblk-1 (nb_b rows each):
//   forward  section, b ascending : [ L[b, 0:64b] panel | L_bb strict lower ]
//   backward section, b descending: [ U[b, 64b+nb_b:n] panel | U_bb upper, diagonal stored as 1/U_kk ]
// A panel (nb_b rows x ncol) is stored as consecutive column tiles of
// PLU_TW = 32 columns (the last one narrower); inside a tile the layout is
// column-major (element (r, c) at c * nb_b + r), and the triangles are
// column-major too (column c of L_bb: rows c+1..nb_b-1; of U_bb: rows 0..c).
// So a warp walking a block reads, per column, consecutive rows: one
// coalesced access per column, each lane owning rows of the block.  Every
// tile / triangle is padded to an even number of doubles (16-byte aligned
// pieces).  A block step is a panel GEMV, y_b -= L[b,:b] y_:b, then a
// substitution with the diagonal triangle (column sweeps), and likewise
// backwards.
#pragma once
#include "common.cuh"

namespace mhdg {

constexpr int PLU_NB = 64;
constexpr int PLU_TW = 32;

__host__ __device__ __forceinline__ long long even_ll(long long x) { return x + (x & 1); }

// doubles of a panel of nb rows x ncol columns in column tiles of PLU_TW
__host__ __device__ inline long long plu_panel_size(int nb, int ncol) {
  long long o = 0;
  for (int c = 0; c < ncol; c += PLU_TW) {
    const int w = (ncol - c) < PLU_TW ? ncol - c : PLU_TW;
    o += even_ll((long long)nb * w);
  }
  return o;
}

struct PluOffsets {
  long long fwd_panel, fwd_diag, bwd_panel, bwd_diag;
  int nb, r0, ncol_fwd, ncol_bwd;
};

__host__ __device__ inline int plu_nblk(int n) { return (n + PLU_NB - 1) / PLU_NB; }

// offsets (in doubles, relative to the macro's base) of block b's pieces
__host__ __device__ inline PluOffsets plu_offsets(int n, int b) {
  const int nblk = plu_nblk(n);
  long long o = 0;
  PluOffsets r{};
  for (int k = 0; k < nblk; ++k) {
    const int nb = (n - PLU_NB * k) < PLU_NB ? n - PLU_NB * k : PLU_NB;
    if (k == b) {
      r.fwd_panel = o;
      r.fwd_diag = o + plu_panel_size(nb, PLU_NB * k);
      r.nb = nb;
      r.r0 = PLU_NB * k;
      r.ncol_fwd = PLU_NB * k;
    }
    o += plu_panel_size(nb, PLU_NB * k) + even_ll((long long)nb * (nb - 1) / 2);
  }
  for (int k = nblk - 1; k >= 0; --k) {
    const int nb = (n - PLU_NB * k) < PLU_NB ? n - PLU_NB * k : PLU_NB;
    const int nc = n - PLU_NB * k - nb;
    if (k == b) {
      r.bwd_panel = o;
      r.bwd_diag = o + plu_panel_size(nb, nc);
      r.ncol_bwd = nc;
    }
    o += plu_panel_size(nb, nc) + even_ll((long long)nb * (nb + 1) / 2);
  }
  return r;
}

__host__ __device__ inline long long plu_size(int n) {
  const int nblk = plu_nblk(n);
  long long o = 0;
  for (int k = 0; k < nblk; ++k) {
    const int nb = (n - PLU_NB * k) < PLU_NB ? n - PLU_NB * k : PLU_NB;
    o += plu_panel_size(nb, PLU_NB * k) + even_ll((long long)nb * (nb - 1) / 2);
    o += plu_panel_size(nb, n - PLU_NB * k - nb) + even_ll((long long)nb * (nb + 1) / 2);
  }
  return o;
}

// offset of element (r, c) inside a tiled panel of nb rows x ncol columns
__host__ __device__ __forceinline__ long long plu_panel_idx(int nb, int r, int c) {
  // all tiles before c's are full width (even size nb*PLU_TW); column-major inside a tile
  return (long long)c * nb + r;
}

// column starts of the packed triangles: strict lower (column c: rows c+1..nb-1) and
// upper incl. diagonal (column c: rows 0..c)
__host__ __device__ __forceinline__ int plu_lo_col(int nb, int c) { return c * (nb - 1) - c * (c - 1) / 2; }
__host__ __device__ __forceinline__ int plu_lo(int nb, int r, int c) { return plu_lo_col(nb, c) + (r - c - 1); }
__host__ __device__ __forceinline__ int plu_up(int r, int c) { return c * (c + 1) / 2 + r; }

// CTA-wide in-place y <- U^-1 L^-1 P y with a packed factor (synchronous loads).
// y, t: shared vectors of length n.
__device__ inline void plu_solve_cta(const double* __restrict__ F, const int* __restrict__ perm, int n, double* y,
                                     double* t) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < n; i += blockDim.x) t[i] = y[__ldg(perm + i)];
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) y[i] = t[i];
  __syncthreads();
  const int nblk = plu_nblk(n);
  for (int b = 0; b < nblk; ++b) {
    const PluOffsets o = plu_offsets(n, b);
    for (int r = warp; r < o.nb; r += nw) {
      double acc = 0.0;
      for (int c = lane; c < o.ncol_fwd; c += 32) acc += __ldg(F + o.fwd_panel + plu_panel_idx(o.nb, r, c)) * y[c];
      acc = warp_sum(acc);
      if (lane == 0) y[o.r0 + r] -= acc;
    }
    __syncthreads();
    if (tid == 0) {  // forward substitution with the unit lower diagonal block
      for (int r = 1; r < o.nb; ++r) {
        double acc = y[o.r0 + r];
        for (int c = 0; c < r; ++c) acc -= __ldg(F + o.fwd_diag + plu_lo(o.nb, r, c)) * y[o.r0 + c];
        y[o.r0 + r] = acc;
      }
    }
    __syncthreads();
  }
  for (int b = nblk - 1; b >= 0; --b) {
    const PluOffsets o = plu_offsets(n, b);
    const int c0 = o.r0 + o.nb;
    for (int r = warp; r < o.nb; r += nw) {
      double acc = 0.0;
      for (int c = lane; c < o.ncol_bwd; c += 32)
        acc += __ldg(F + o.bwd_panel + plu_panel_idx(o.nb, r, c)) * y[c0 + c];
      acc = warp_sum(acc);
      if (lane == 0) y[o.r0 + r] -= acc;
    }
    __syncthreads();
    if (tid == 0) {  // backward substitution with the upper diagonal block (1/U_kk stored)
      for (int r = o.nb - 1; r >= 0; --r) {
        double acc = y[o.r0 + r];
        for (int c = r + 1; c < o.nb; ++c) acc -= __ldg(F + o.bwd_diag + plu_up(r, c)) * y[o.r0 + c];
        y[o.r0 + r] = acc * __ldg(F + o.bwd_diag + plu_up(r, r));
      }
    }
    __syncthreads();
  }
}

}  // namespace mhdg
