// Face-block preconditioner (krylov.py:194-238).
//
// k_precond_build: one CTA per skeleton face: B_f = sum over the face's sides
// (flat (mac, lf) order, as np.add.at) of P^T face_trace_trace P, with P the
// side's canonical node permutation (recovered from `gather`); symmetrise,
// Cholesky (PreconditionerError naming the face if not positive definite),
// explicit inverse via L^-T L^-1 as cho_solve(., I) does.
// k_precond_apply: y_f = inv_f v_f, one CTA per face.
#include "common.cuh"

namespace mhdg {

constexpr int PRE_THREADS = 256;

template <int D>
__global__ void __launch_bounds__(PRE_THREADS) k_precond_build(mhdg_disc g, mhdg_blocks b, const double* __restrict__ extra,
                                                               double* inv, int* status, int x_global) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2, NF = D + 1;
  const int f = blockIdx.x, bs = g.Lf * NS, tid = threadIdx.x;
  double* B = sm;            // bs x bs
  // bs x bs Cholesky workspace: shared memory, or (large faces: 3D p = 3 has bs = 140 and
  // 2 bs^2 doubles exceed shared memory) this face's own output block, overwritten last
  double* X = x_global ? inv + (size_t)f * bs * bs : B + bs * bs;
  __shared__ int fail;
  if (tid == 0) fail = 0;
  for (int i = tid; i < bs * bs; i += blockDim.x) B[i] = 0.0;
  __syncthreads();
  // sides in flat (mac, lf) order
  int m0 = g.face_macros[2 * f], m1 = g.face_macros[2 * f + 1];
  int l0 = g.face_locals[2 * f], l1 = g.face_locals[2 * f + 1];
  if (m1 >= 0 && (m1 * NF + l1) < (m0 * NF + l0)) {
    int t = m0; m0 = m1; m1 = t;
    t = l0; l0 = l1; l1 = t;
  }
  for (int side = 0; side < 2; ++side) {
    const int mac = side ? m1 : m0, lf = side ? l1 : l0;
    if (mac < 0) continue;
    const int* gat = g.gather + ((size_t)mac * NF + lf) * bs;
    const double* A = b.face_trace_trace + ((size_t)mac * NF + lf) * bs * bs;
    for (int idx = tid; idx < bs * bs; idx += blockDim.x) {
      const int r = idx / bs, c = idx - r * bs;
      const int pr = gat[r] - f * bs, pc = gat[c] - f * bs;
      B[pr * bs + pc] += A[idx];  // each (pr, pc) hit once per side: no race
    }
    __syncthreads();
  }
  if (extra) {  // the face's other side, held by another rank, already in canonical order
    for (int idx = tid; idx < bs * bs; idx += blockDim.x) B[idx] += extra[(size_t)f * bs * bs + idx];
    __syncthreads();
  }
  for (int idx = tid; idx < bs * bs; idx += blockDim.x) {
    const int r = idx / bs, c = idx - r * bs;
    if (c <= r) {
      const double v = 0.5 * (B[r * bs + c] + B[c * bs + r]);
      X[r * bs + c] = v;  // symmetric part, lower triangle
    }
  }
  __syncthreads();
  // right-looking Cholesky in X (lower)
  for (int j = 0; j < bs; ++j) {
    const double d = X[j * bs + j];
    if (!(d > 0.0)) {
      if (tid == 0) fail = 1;
      break;
    }
    const double ljj = sqrt(d);
    __syncthreads();
    for (int i = j + 1 + tid; i < bs; i += blockDim.x) X[i * bs + j] /= ljj;
    if (tid == 0) X[j * bs + j] = ljj;
    __syncthreads();
    const int w = bs - j - 1;
    for (int idx = tid; idx < w * w; idx += blockDim.x) {
      const int i = j + 1 + idx / w, k = j + 1 + idx % w;
      if (k <= i) X[i * bs + k] -= X[i * bs + j] * X[k * bs + j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) set_status(status, MHDG_ERR_PRECONDITIONER, f, 0, 0.0);
    return;
  }
  // B <- L^-1 (lower) by forward elimination on the identity, all threads per step:
  // step k scales row k by 1 / L_kk, then removes L_ik x row k from the rows below.  Each
  // entry accumulates its terms in the same order (k ascending) and is divided once, as the
  // column-by-column substitution does, so the result is bitwise that of the serial
  // per-column loop -- with bs steps of parallel work instead of one thread per column.
  for (int idx = tid; idx < bs * bs; idx += blockDim.x) {
    const int r = idx / bs, c = idx - r * bs;
    B[idx] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < bs; ++k) {
    const double lkk = X[k * bs + k];
    for (int c = tid; c <= k; c += blockDim.x) B[k * bs + c] = c == k ? 1.0 / lkk : B[k * bs + c] / lkk;
    __syncthreads();
    const int rows = bs - k - 1, cols = k + 1;
    for (int idx = tid; idx < rows * cols; idx += blockDim.x) {
      const int i = k + 1 + idx / cols, c = idx - (idx / cols) * cols;
      B[i * bs + c] -= X[i * bs + k] * B[k * bs + c];
    }
    __syncthreads();
  }
  // inv = L^-T L^-1
  double* out = inv + (size_t)f * bs * bs;
  for (int idx = tid; idx < bs * bs; idx += blockDim.x) {
    const int i = idx / bs, j = idx - i * bs;
    const int k0 = i > j ? i : j;
    double acc = 0.0;
    for (int k = k0; k < bs; ++k) acc += B[k * bs + i] * B[k * bs + j];
    out[idx] = acc;
  }
}

__global__ void __launch_bounds__(PRE_THREADS) k_precond_apply(int bs, const double* __restrict__ inv,
                                                               const double* __restrict__ v, double* __restrict__ y) {
  extern __shared__ double sm[];
  const int f = blockIdx.x;
  for (int i = threadIdx.x; i < bs; i += blockDim.x) sm[i] = v[(size_t)f * bs + i];
  __syncthreads();
  warp_gemv<false>(inv + (size_t)f * bs * bs, bs, bs, sm, sm + bs, 1.0);
  __syncthreads();
  for (int i = threadIdx.x; i < bs; i += blockDim.x) y[(size_t)f * bs + i] = sm[bs + i];
}

// out[i] = P^T face_trace_trace[macs[i], lfs[i]] P in the face's canonical order
template <int D>
__global__ void k_side_blocks(mhdg_disc g, mhdg_blocks b, const int* __restrict__ macs, const int* __restrict__ lfs,
                              int count, double* __restrict__ out) {
  constexpr int NS = D + 2, NF = D + 1;
  const int i = blockIdx.x, bs = g.Lf * NS;
  if (i >= count) return;
  const int mac = macs[i], lf = lfs[i];
  const int* gat = g.gather + ((size_t)mac * NF + lf) * bs;
  const double* A = b.face_trace_trace + ((size_t)mac * NF + lf) * bs * bs;
  const int base = (gat[0] / bs) * bs;  // face id * bs
  for (int idx = threadIdx.x; idx < bs * bs; idx += blockDim.x) {
    const int r = idx / bs, c = idx - r * bs;
    out[(size_t)i * bs * bs + (gat[r] - base) * bs + (gat[c] - base)] = A[idx];
  }
}

template <int D>
int side_blocks(const mhdg_disc& g, const mhdg_blocks& b, const int* macs, const int* lfs, int count, double* out,
                cudaStream_t st) {
  if (count <= 0) return MHDG_OK;
  k_side_blocks<D><<<count, PRE_THREADS, 0, st>>>(g, b, macs, lfs, count, out);
  return launch_ok();
}
template int side_blocks<2>(const mhdg_disc&, const mhdg_blocks&, const int*, const int*, int, double*, cudaStream_t);
template int side_blocks<3>(const mhdg_disc&, const mhdg_blocks&, const int*, const int*, int, double*, cudaStream_t);

template <int D>
int precond_build(const mhdg_disc& g, const mhdg_blocks& b, const double* extra, double* inv, int* status,
                  cudaStream_t st) {
  const int bs = g.Lf * (D + 2);
  size_t bytes = sizeof(double) * 2 * bs * bs;
  const int x_global = bytes > 227 * 1024;
  if (x_global) bytes /= 2;
  if (bytes > 227 * 1024) return MHDG_ERR_CONFIG;
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(k_precond_build<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  tl_begin(TL_PRECOND_BUILD, st);
  k_precond_build<D><<<g.n_faces, PRE_THREADS, bytes, st>>>(g, b, extra, inv, status, x_global);
  tl_end(TL_PRECOND_BUILD, st);
  return launch_ok();
}

int precond_apply(const mhdg_disc& g, const double* inv, const double* v, double* y, cudaStream_t st) {
  const int bs = g.Lf * g.ns;
  tl_begin(TL_PRECOND_APPLY, st);
  k_precond_apply<<<g.n_faces, PRE_THREADS, sizeof(double) * 2 * bs, st>>>(bs, inv, v, y);
  tl_end(TL_PRECOND_APPLY, st);
  return launch_ok();
}

template int precond_build<2>(const mhdg_disc&, const mhdg_blocks&, const double*, double*, int*, cudaStream_t);
template int precond_build<3>(const mhdg_disc&, const mhdg_blocks&, const double*, double*, int*, cudaStream_t);

}  // namespace mhdg
