// Face-block preconditioner (krylov.py:194-238).
//
// One CTA per skeleton face: B_f = sum over the face's sides (flat (mac, lf)
// order, as np.add.at) of P^T face_trace_trace P, with P the side's canonical
// node permutation (recovered from `gather`), symmetrised and inverted
// (PreconditionerError naming the face if not positive definite):
//   k_precond_build_reg (default, face blocks up to 144 dofs): in-place
//     Gauss-Jordan sweep on register tiles, the pivots are the Cholesky pivots;
//   k_precond_build (larger blocks, or mhdg_set_precond_variant(1)): Cholesky in
//     shared memory and the explicit inverse L^-T L^-1 as cho_solve(., I) does.
// k_precond_apply: y_f = inv_f v_f, one CTA per face.
#include "common.cuh"

namespace mhdg {

constexpr int PRE_THREADS = 256;

static int g_precond_variant = 0;
extern "C" void mhdg_set_precond_variant(int v) { g_precond_variant = v; }
static bool precond_shared_build() { return g_precond_variant == 1; }

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
    if (mac < 0 || !b.face_trace_trace) continue;  // no resident blocks: `extra` holds the whole face sum
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

// k_precond_build_reg: the same face block inverted in registers.  The 16 x 16 threads of a
// CTA hold B_f as T x T tiles each (entry (ti + 16 a, tj + 16 b)) and run an in-place
// Gauss-Jordan sweep without pivoting (B_f is symmetric positive definite; the pivots are
// the Cholesky pivots L_kk^2, so the positive-definiteness test is the same): step k
// publishes row k and column k through a double-buffered shared-memory line (one barrier
// per step), then every thread does T^2 FMAs on its registers.  One bs^2 shared-memory
// block stages the coalesced loads into canonical order and the inverse for coalesced
// stores.  bs <= 16 T.
template <int D, int T>
__global__ void __launch_bounds__(PRE_THREADS, T <= 5 ? 3 : 1)
    k_precond_build_reg(mhdg_disc g, mhdg_blocks b, const double* __restrict__ extra, double* __restrict__ inv,
                        int* status) {
  constexpr int NS = D + 2, NF = D + 1, W = 16 * T;
  const int f = blockIdx.x, bs = g.Lf * NS, tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  extern __shared__ double sm[];  // bs x ld staging block: B_f in canonical order, later the inverse
  const int ld = bs | 1;          // odd row stride: the transposed reads are conflict-free
  __shared__ __align__(16) double rowb[2][W], colb[2][W];
  __shared__ int perm[W];
  int m0 = g.face_macros[2 * f], m1 = g.face_macros[2 * f + 1];
  int l0 = g.face_locals[2 * f], l1 = g.face_locals[2 * f + 1];
  if (m1 >= 0 && (m1 * NF + l1) < (m0 * NF + l0)) {  // sides in flat (mac, lf) order, as np.add.at
    int t = m0; m0 = m1; m1 = t;
    t = l0; l0 = l1; l1 = t;
  }
  // coalesced reads of each side's block, scattered into canonical order in shared memory
  bool first = true;
  const float rbs = 1.0f / (float)bs;
  for (int side = 0; side < 2; ++side) {
    const int mac = side ? m1 : m0, lf = side ? l1 : l0;
    if (mac < 0 || !b.face_trace_trace) continue;  // no resident blocks: `extra` holds the whole face sum
    const int* gat = g.gather + ((size_t)mac * NF + lf) * bs;
    const double* As = b.face_trace_trace + ((size_t)mac * NF + lf) * bs * bs;
    __syncthreads();  // the previous side's perm reads and block writes are done
    for (int r = tid; r < bs; r += PRE_THREADS) perm[r] = __ldg(gat + r) - f * bs;
    __syncthreads();
    // the block read linearly, LB loads in flight per thread, then scattered
    constexpr int LB = 12;
    for (int e0 = tid; e0 < bs * bs; e0 += PRE_THREADS * LB) {
      double v[LB];
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int idx = e0 + PRE_THREADS * u;
        v[u] = idx < bs * bs ? __ldg(As + idx) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int idx = e0 + PRE_THREADS * u;
        if (idx < bs * bs) {
          const int r = __float2int_rd(((float)idx + 0.5f) * rbs), c = idx - r * bs;  // exact: idx < 2^15
          double* d = sm + perm[r] * ld + perm[c];
          *d = first ? v[u] : *d + v[u];  // each (pr, pc) hit once per side: no race
        }
      }
    }
    first = false;
  }
  __syncthreads();
  if (extra) {  // the face's other side, held by another rank, already in canonical order
    const double* ex = extra + (size_t)f * bs * bs;
    for (int r = tid >> 5; r < bs; r += PRE_THREADS / 32)
      for (int c = tid & 31; c < bs; c += 32) sm[r * ld + c] = first ? __ldg(ex + r * bs + c) : sm[r * ld + c] + __ldg(ex + r * bs + c);
    __syncthreads();
  }
  double A[T][T];
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int c = 0; c < T; ++c) {
      const int i = ti + 16 * a, j = tj + 16 * c;
      A[a][c] = (i < bs && j < bs) ? 0.5 * (sm[i * ld + j] + sm[j * ld + i]) : 0.0;
    }
  bool bad = false;
#pragma unroll
  for (int ka = 0; ka < T; ++ka) {
    for (int kk = 0; kk < 16; ++kk) {
      const int k = 16 * ka + kk;
      if (k >= bs) break;
      double* rb = rowb[k & 1];
      double* cb = colb[k & 1];
      if (ti == kk) {
#pragma unroll
        for (int c = 0; c < T; ++c) rb[tj + 16 * c] = A[ka][c];
      }
      if (tj == kk) {
#pragma unroll
        for (int a = 0; a < T; ++a) cb[ti + 16 * a] = A[a][ka];
      }
      __syncthreads();
      const double p = rb[k];
      if (!(p > 0.0)) {  // uniform over the CTA
        bad = true;
        break;
      }
      const double ip = 1.0 / p;
      double cc[T], rr[T];
#pragma unroll
      for (int a = 0; a < T; ++a) {
        cc[a] = -cb[ti + 16 * a] * ip;
        rr[a] = rb[tj + 16 * a];
      }
      if (ti == kk) cc[ka] = ip;
      if (tj == kk) rr[ka] = 1.0;
#pragma unroll
      for (int a = 0; a < T; ++a)
#pragma unroll
        for (int c = 0; c < T; ++c) {
          double old = A[a][c];
          if ((a == ka && ti == kk) || (c == ka && tj == kk)) old = 0.0;
          A[a][c] = fma(cc[a], rr[c], old);
        }
    }
    if (bad) break;
  }
  if (bad) {
    if (tid == 0) set_status(status, MHDG_ERR_PRECONDITIONER, f, 0, 0.0);
    return;
  }
  __syncthreads();  // every thread has taken its tile of B_f out of the staging block
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int c = 0; c < T; ++c) {
      const int i = ti + 16 * a, j = tj + 16 * c;
      if (i < bs && j < bs) sm[i * ld + j] = A[a][c];
    }
  __syncthreads();
  double* out = inv + (size_t)f * bs * bs;
  for (int r = tid >> 5; r < bs; r += PRE_THREADS / 32)
    for (int c = tid & 31; c < bs; c += 32) out[r * bs + c] = sm[r * ld + c];
}

template <int D, int T>
static void launch_build_reg(const mhdg_disc& g, const mhdg_blocks& b, const double* extra, double* inv, int* status,
                             cudaStream_t st) {
  const int bs = g.Lf * (D + 2);
  const size_t bytes = sizeof(double) * bs * (bs | 1);
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(k_precond_build_reg<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_precond_build_reg<D, T><<<g.n_faces, PRE_THREADS, bytes, st>>>(g, b, extra, inv, status);
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

// sums[f] += P^T face_trace_trace[mac, lf] P for the sides (mac, lf) of face f with mac in the
// window [mac0, mac0 + count), in flat (mac, lf) order; `b` holds the window's blocks only.
// Windows visited one after the other on a stream leave in sums[f] the same two-term sum
// as k_precond_build forms (a + b is commutative; the first term is added to zero).
template <int D>
__global__ void __launch_bounds__(PRE_THREADS) k_face_sum_window(mhdg_disc g, mhdg_blocks b, int mac0, int count,
                                                                 double* __restrict__ sums) {
  constexpr int NS = D + 2, NF = D + 1;
  const int f = blockIdx.x, bs = g.Lf * NS;
  int m0 = g.face_macros[2 * f], m1 = g.face_macros[2 * f + 1];
  int l0 = g.face_locals[2 * f], l1 = g.face_locals[2 * f + 1];
  if (m1 >= 0 && (m1 * NF + l1) < (m0 * NF + l0)) {
    int t = m0; m0 = m1; m1 = t;
    t = l0; l0 = l1; l1 = t;
  }
  double* out = sums + (size_t)f * bs * bs;
  for (int side = 0; side < 2; ++side) {
    const int mac = side ? m1 : m0, lf = side ? l1 : l0;
    if (mac < mac0 || mac >= mac0 + count) continue;
    const int* gat = g.gather + ((size_t)mac * NF + lf) * bs;
    const double* A = b.face_trace_trace + ((size_t)(mac - mac0) * NF + lf) * bs * bs;
    for (int idx = threadIdx.x; idx < bs * bs; idx += blockDim.x) {
      const int r = idx / bs, c = idx - r * bs;
      out[(gat[r] - f * bs) * bs + (gat[c] - f * bs)] += A[idx];  // each entry hit once per side
    }
    __syncthreads();
  }
}

template <int D>
int face_sum_window(const mhdg_disc& g, const mhdg_blocks& b, int mac0, int count, double* sums, cudaStream_t st) {
  k_face_sum_window<D><<<g.n_faces, PRE_THREADS, 0, st>>>(g, b, mac0, count, sums);
  return launch_ok();
}
template int face_sum_window<2>(const mhdg_disc&, const mhdg_blocks&, int, int, double*, cudaStream_t);
template int face_sum_window<3>(const mhdg_disc&, const mhdg_blocks&, int, int, double*, cudaStream_t);

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
  if (bs <= 144 && !precond_shared_build()) {  // register-tile sweep (no bs^2 shared-memory block)
    tl_begin(TL_PRECOND_BUILD, st);
    if (bs <= 16) launch_build_reg<D, 1>(g, b, extra, inv, status, st);
    else if (bs <= 32) launch_build_reg<D, 2>(g, b, extra, inv, status, st);
    else if (bs <= 48) launch_build_reg<D, 3>(g, b, extra, inv, status, st);
    else if (bs <= 64) launch_build_reg<D, 4>(g, b, extra, inv, status, st);
    else if (bs <= 80) launch_build_reg<D, 5>(g, b, extra, inv, status, st);
    else if (bs <= 112) launch_build_reg<D, 7>(g, b, extra, inv, status, st);
    else launch_build_reg<D, 9>(g, b, extra, inv, status, st);
    tl_end(TL_PRECOND_BUILD, st);
    return launch_ok();
  }
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
