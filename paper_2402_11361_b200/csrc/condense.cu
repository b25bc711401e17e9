// Second-layer static condensation on the device.
//
// k_schur   S = state_state - A_uq A_qq^-1 A_qu   (_schur_correction,
//           condense.py:130-158).  Per sub-element (and face sub-element) the
//           correction is one GEMM  X[(a,s,r), j] = sum_{(q,l)} T1[(a,s,r),(q,l)] VW[(q,l), j]
//           with T1 = sum_k gphys W (the dG/dq stash) and
//           VW[q,l,j] = sum_r inv_jac[r,l] PM[q,r,j], PM = phi M^-1 D (a
//           macro-independent table), scattered into the rows of the
//           sub-element's nodes.
// k_lu      in-place LU with partial pivoting of each macro's S (replaces the
//           reference's np.linalg.inv, condense.py:66-69; FactorizationError on
//           an exactly zero pivot).  Right-looking, 32-column panels in shared
//           memory, 64x64 register-tiled trailing updates.
#include "common.cuh"
#include "local_ops.cuh"
#include "packed_lu.cuh"
#include "tiled_inv.cuh"

namespace mhdg {

constexpr int SCHUR_THREADS = 256;
constexpr int LU_THREADS = 256;
constexpr int LU_NB = 32;

// --------------------------------------------------------------------------
// Schur complement
// --------------------------------------------------------------------------

template <int D>
__global__ void __launch_bounds__(SCHUR_THREADS) k_schur(mhdg_disc g, mhdg_blocks b, double* __restrict__ S) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2, NF = D + 1;
  const Sz sz = make_sz<D>(g);
  const int mac = blockIdx.x, n = sz.n, L = sz.L;
  const double* ij = g.inv_jac + (size_t)mac * D * D;
  double* Sm = S + (size_t)mac * n * n;
  const double* SS = b.state_state + (size_t)mac * n * n;
  for (size_t i = threadIdx.x; i < (size_t)n * n; i += blockDim.x) Sm[i] = SS[i];
  __syncthreads();

  // shared: T1 (rows nloc*NS, k = nq*D) for one r, VW (nq*D x L), ijs
  const int kv = sz.nq * D, kf = sz.nqf * D;
  const int kmax = kv > kf ? kv : kf;
  const int rmax = sz.nloc * NS > sz.nlocf * NS ? sz.nloc * NS : sz.nlocf * NS;
  double* T1 = sm;
  double* VW = T1 + rmax * kmax;

  // ---- volume sub-elements ----
  for (int K = 0; K < sz.n_sub; ++K) {
    // VW[(q,l), j] = sum_r inv_jac[r,l] PM[K,q,r,j]
    for (int idx = threadIdx.x; idx < kv * L; idx += blockDim.x) {
      const int j = idx % L, ql = idx / L, l = ql % D, q = ql / D;
      const double* pm = g.pm_vol + (((size_t)K * sz.nq + q) * D) * L + j;
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) a += __ldg(ij + r * D + l) * __ldg(pm + r * L);
      VW[idx] = a;
    }
    for (int rr = 0; rr < NS; ++rr) {
      // T1[(a,s),(q,l)] = sum_k gphys[q,a,k] W[K,q,k,l,s,rr]
      for (int idx = threadIdx.x; idx < sz.nloc * NS * kv; idx += blockDim.x) {
        const int ql = idx % kv, as = idx / kv, s = as % NS, a = as / NS, l = ql % D, q = ql / D;
        const double* gr = g.grad_ref + (((size_t)K * sz.nq + q) * sz.nloc + a) * D;
        const double* W = b.wdgdq_vol + ((((size_t)mac * sz.n_sub + K) * sz.nq + q) * D * D) * NS * NS;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double gp = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) gp += __ldg(gr + r) * __ldg(ij + r * D + k);
          acc += gp * __ldg(W + ((k * D + l) * NS + s) * NS + rr);
        }
        T1[idx] = acc;
      }
      __syncthreads();
      // S[(conn[a],s), (j,rr)] += sum_{ql} T1[(a,s), ql] VW[ql, j]
      for (int idx = threadIdx.x; idx < sz.nloc * NS * L; idx += blockDim.x) {
        const int j = idx % L, as = idx / L, s = as % NS, a = as / NS;
        const double* t = T1 + as * kv;
        double acc = 0.0;
        for (int k = 0; k < kv; ++k) acc += t[k] * VW[k * L + j];
        const int row = __ldg(g.sub_conn + K * sz.nloc + a) * NS + s;
        Sm[(size_t)row * n + j * NS + rr] += acc;
      }
      __syncthreads();
    }
  }
  // ---- face sub-elements ----
  for (int f = 0; f < NF; ++f) {
    for (int T = 0; T < sz.n_tri; ++T) {
      for (int idx = threadIdx.x; idx < kf * L; idx += blockDim.x) {
        const int j = idx % L, ql = idx / L, l = ql % D, q = ql / D;
        const double* pm = g.pm_face + ((((size_t)f * sz.n_tri + T) * sz.nqf + q) * D) * L + j;
        double a = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) a += __ldg(ij + r * D + l) * __ldg(pm + r * L);
        VW[idx] = a;
      }
      for (int rr = 0; rr < NS; ++rr) {
        for (int idx = threadIdx.x; idx < sz.nlocf * NS * kf; idx += blockDim.x) {
          const int ql = idx % kf, as = idx / kf, s = as % NS, a = as / NS, l = ql % D, q = ql / D;
          const double* W = b.wdgdq_face +
                            ((((size_t)mac * NF + f) * sz.n_tri * sz.nqf + T * sz.nqf + q) * D + l) * NS * NS;
          T1[idx] = __ldg(W + s * NS + rr) * __ldg(g.phi_face + q * sz.nlocf + a);
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < sz.nlocf * NS * L; idx += blockDim.x) {
          const int j = idx % L, as = idx / L, s = as % NS, a = as / NS;
          const double* t = T1 + as * kf;
          double acc = 0.0;
          for (int k = 0; k < kf; ++k) acc += t[k] * VW[k * L + j];
          const int node = __ldg(g.face_vol_nodes + f * sz.Lf + __ldg(g.tri_conn + T * sz.nlocf + a));
          Sm[(size_t)(node * NS + s) * n + j * NS + rr] -= acc;
        }
        __syncthreads();
      }
    }
  }
}

// --------------------------------------------------------------------------
// batched LU with partial pivoting
// --------------------------------------------------------------------------

__device__ __forceinline__ void block_argmax(double v, int i, double* rv, int* ri, double* outv, int* outi) {
  // max |v|, ties -> smallest index (LAPACK idamax semantics)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(MHDG_FULL, v, o);
    int i2 = __shfl_xor_sync(MHDG_FULL, i, o);
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
  if (lane == 0) { rv[warp] = v; ri[warp] = i; }
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? rv[lane] : -1.0;
    i = lane < nw ? ri[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(MHDG_FULL, v, o);
      int i2 = __shfl_xor_sync(MHDG_FULL, i, o);
      if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
    }
    if (lane == 0) { *outv = v; *outi = i; }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(LU_THREADS) k_lu(int n, double* __restrict__ LU, int* __restrict__ perm,
                                                   int* status) {
  extern __shared__ double sm[];
  constexpr int PW = LU_NB + 1;  // padded panel row
  const int mac = blockIdx.x, tid = threadIdx.x;
  double* A = LU + (size_t)mac * n * n;
  int* pm = perm + (size_t)mac * n;
  double* P = sm;                               // n x PW panel
  double* Ut = P + (size_t)n * PW;              // LU_NB x 64 U12 tile
  double* Ar = Ut + LU_NB * 64;                 // LU_NB x 64 staged A12 tile
  double* Li = Ar + LU_NB * 64;                 // LU_NB x PW  L11^-1
  double* red_v = Li + LU_NB * PW;              // 32
  int* red_i = (int*)(red_v + 32);              // 32
  int* piv = red_i + 32;                        // LU_NB
  double* bcast = (double*)(piv + LU_NB + 2);   // 2 (aligned below)
  int* bidx = (int*)(bcast + 2);
  for (int i = tid; i < n; i += blockDim.x) pm[i] = i;
  bool singular = false;

  for (int k0 = 0; k0 < n; k0 += LU_NB) {
    const int nb = min(LU_NB, n - k0), m = n - k0;
    for (int idx = tid; idx < m * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      P[i * PW + c] = A[(size_t)(k0 + i) * n + k0 + c];
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      // pivot search over panel rows j..m-1 of column j
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = j + tid; i < m; i += blockDim.x) {
        const double v = fabs(P[i * PW + j]);
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      block_argmax(best, bi, red_v, red_i, bcast, bidx);
      const int p = *bidx;
      if (tid == 0) piv[j] = p;
      if (*bcast == 0.0) singular = true;
      if (p != j) {
        for (int c = tid; c < nb; c += blockDim.x) {
          const double t = P[j * PW + c];
          P[j * PW + c] = P[p * PW + c];
          P[p * PW + c] = t;
        }
      }
      __syncthreads();
      const double dinv = singular ? 0.0 : 1.0 / P[j * PW + j];
      for (int i = j + 1 + tid; i < m; i += blockDim.x) P[i * PW + j] *= dinv;
      __syncthreads();
      // rank-1 update of the remaining panel columns
      const int w = nb - j - 1;
      if (w > 0) {
        for (int idx = tid; idx < (m - j - 1) * w; idx += blockDim.x) {
          const int i = j + 1 + idx / w, c = j + 1 + idx % w;
          P[i * PW + c] -= P[i * PW + j] * P[j * PW + c];
        }
      }
      __syncthreads();
    }
    // write the panel back; apply the panel's interchanges to the other columns
    for (int idx = tid; idx < m * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      A[(size_t)(k0 + i) * n + k0 + c] = P[i * PW + c];
    }
    for (int j = 0; j < nb; ++j) {
      const int p = piv[j];
      if (p == j) continue;
      const size_t r1 = (size_t)(k0 + j) * n, r2 = (size_t)(k0 + p) * n;
      for (int c = tid; c < n - nb; c += blockDim.x) {
        const int cc = c < k0 ? c : c + nb;
        const double t = A[r1 + cc];
        A[r1 + cc] = A[r2 + cc];
        A[r2 + cc] = t;
      }
      if (tid == 0) {
        const int t = pm[k0 + j];
        pm[k0 + j] = pm[k0 + p];
        pm[k0 + p] = t;
      }
      __syncthreads();
    }
    __syncthreads();
    const int c0 = k0 + nb;
    if (c0 >= n) break;
    // Li = L11^-1 (unit lower), one column per thread
    for (int c = tid; c < LU_NB; c += blockDim.x) {
      for (int i = 0; i < LU_NB; ++i) Li[i * PW + c] = (i == c) ? 1.0 : 0.0;
      for (int i = c + 1; i < nb; ++i) {
        double acc = 0.0;
        for (int k = c; k < i; ++k) acc += P[i * PW + k] * Li[k * PW + c];
        Li[i * PW + c] = -acc;
      }
    }
    __syncthreads();
    // per 64-column tile: U12 = Li A12 (staged in smem), then A22 -= L21 U12
    const int rows = n - c0;
    const int tx = tid & 15, ty = tid >> 4;
    for (int tc = 0; tc < rows; tc += 64) {
      const int wc = min(64, rows - tc);
      for (int idx = tid; idx < LU_NB * 64; idx += blockDim.x) {
        const int r = idx / 64, c = idx % 64;
        Ar[r * 64 + c] = (c < wc && r < nb) ? A[(size_t)(k0 + r) * n + c0 + tc + c] : 0.0;
      }
      __syncthreads();
      for (int idx = tid; idx < LU_NB * 64; idx += blockDim.x) {
        const int r = idx / 64, c = idx % 64;
        double acc = 0.0;
        for (int k = 0; k <= r; ++k) acc += Li[r * PW + k] * Ar[k * 64 + c];
        Ut[r * 64 + c] = acc;
        if (c < wc && r < nb) A[(size_t)(k0 + r) * n + c0 + tc + c] = acc;
      }
      __syncthreads();
      for (int tr = 0; tr < rows; tr += 64) {
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) acc[a][bq] = 0.0;
        for (int k = 0; k < nb; ++k) {
          double lv[4], uv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = tr + ty + 16 * a;
            lv[a] = i < rows ? P[(nb + i) * PW + k] : 0.0;
          }
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) uv[bq] = Ut[k * 64 + tx + 16 * bq];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bq = 0; bq < 4; ++bq) acc[a][bq] += lv[a] * uv[bq];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = tr + ty + 16 * a;
          if (i >= rows) continue;
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) {
            const int c = tx + 16 * bq;
            if (c < wc) A[(size_t)(c0 + i) * n + c0 + tc + c] -= acc[a][bq];
          }
        }
      }
      __syncthreads();
    }
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
}

// --------------------------------------------------------------------------
// pack: factored n x n (scratch) -> packed solve layout with inverted diagonal
// tiles (packed_lu.cuh)
// --------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_pack(int n, const double* __restrict__ F, double* __restrict__ out) {
  extern __shared__ double pk_sm[];
  double(*T)[PLU_NB + 1] = reinterpret_cast<double(*)[PLU_NB + 1]>(pk_sm);
  double(*X)[PLU_NB + 1] = reinterpret_cast<double(*)[PLU_NB + 1]>(pk_sm + PLU_NB * (PLU_NB + 1));
  const int mac = blockIdx.x, tid = threadIdx.x;
  const double* A = F + (size_t)mac * n * n;
  double* O = out + (size_t)mac * plu_size(n);
  const int nblk = plu_nblk(n);
  for (int b = 0; b < nblk; ++b) {
    const PluOffsets o = plu_offsets(n, b);
    const int nb = o.nb, r0 = o.r0;
    for (int idx = tid; idx < nb * o.ncol_fwd; idx += blockDim.x) {
      const int r = idx / o.ncol_fwd, c = idx % o.ncol_fwd;
      O[o.fwd_panel + plu_panel_idx(nb, o.ncol_fwd, r, c)] = A[(size_t)(r0 + r) * n + c];
    }
    for (int idx = tid; idx < nb * o.ncol_bwd; idx += blockDim.x) {
      const int r = idx / o.ncol_bwd, c = idx % o.ncol_bwd;
      O[o.bwd_panel + plu_panel_idx(nb, o.ncol_bwd, r, c)] = A[(size_t)(r0 + r) * n + r0 + nb + c];
    }
    for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
      const int r = idx / nb, c = idx % nb;
      T[r][c] = A[(size_t)(r0 + r) * n + r0 + c];
    }
    __syncthreads();
    if (tid < nb) {  // inverse of the unit lower tile, column tid
      const int c = tid;
      X[c][c] = 1.0;
      for (int i = c + 1; i < nb; ++i) {
        double acc = 0.0;
        for (int k = c; k < i; ++k) acc += T[i][k] * X[k][c];
        X[i][c] = -acc;
      }
    }
    __syncthreads();
    for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
      const int r = idx / nb, c = idx % nb;
      if (c < r) O[o.fwd_diag + plu_lo(r, c)] = X[r][c];
    }
    __syncthreads();
    if (tid < nb) {  // inverse of the upper tile, column tid
      const int c = tid;
      X[c][c] = 1.0 / T[c][c];
      for (int i = c - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int k = i + 1; k <= c; ++k) acc += T[i][k] * X[k][c];
        X[i][c] = -acc / T[i][i];
      }
    }
    __syncthreads();
    for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
      const int r = idx / nb, c = idx % nb;
      if (c >= r) O[o.bwd_diag + plu_up(nb, r, c)] = X[r][c];
    }
    if (tid == 0) {  // zero the even-size padding of the last (narrow) tiles and triangles
      if ((nb * (nb - 1) / 2) & 1) O[o.fwd_diag + nb * (nb - 1) / 2] = 0.0;
      if ((nb * (nb + 1) / 2) & 1) O[o.bwd_diag + nb * (nb + 1) / 2] = 0.0;
      const int wf = o.ncol_fwd % PLU_TW, wb = o.ncol_bwd % PLU_TW;
      if ((nb * wf) & 1) O[o.fwd_diag - 1] = 0.0;
      if ((nb * wb) & 1) O[o.bwd_diag - 1] = 0.0;
    }
    __syncthreads();
  }
}


// --------------------------------------------------------------------------
// batched in-place Gauss-Jordan inversion with partial pivoting
// --------------------------------------------------------------------------
// Replaces np.linalg.inv (LAPACK getrf + getri, condense.py:67) with the same
// 2n^3-flop inverse computed panel by panel: a 32-column panel of all n rows
// is reduced in shared memory (row pivoting, scaling, elimination of every
// other row), which yields the panel's columns of the composite elementary
// transform T; every other column is then updated as A[:, c] += (T - I)[:, panel]
// A_old[panel rows, c] with 64x64 register-tiled rank-32 updates.  Column
// interchanges are undone at the end.  An exactly zero pivot raises
// FactorizationError (np.linalg.inv raises LinAlgError).

constexpr int GJ_NB = 32;

size_t gj_smem_bytes(int n) {
  return sizeof(double) * ((size_t)n * (GJ_NB + 1) + GJ_NB * 64 + 32 + 8) + sizeof(int) * ((size_t)n + 32 + 8) + 64;
}

__global__ void __launch_bounds__(LU_THREADS) k_gj(int n, double* __restrict__ S, int* status) {
  extern __shared__ double sm[];
  constexpr int PW = GJ_NB + 1;
  const int mac = blockIdx.x, tid = threadIdx.x;
  double* A = S + (size_t)mac * n * n;
  double* P = sm;                          // n x PW panel
  double* Bt = P + (size_t)n * PW;         // GJ_NB x 64 tile of the old pivot rows
  double* red_v = Bt + GJ_NB * 64;         // 32
  int* red_i = (int*)(red_v + 32);         // 32
  int* pivg = red_i + 32;                  // n (+ pad)
  double* bcast = (double*)(pivg + n + (n & 1) + 2);
  int* bidx = (int*)(bcast + 2);
  bool singular = false;
  const int tx = tid & 15, ty = tid >> 4;

  for (int k0 = 0; k0 < n; k0 += GJ_NB) {
    const int nb = min(GJ_NB, n - k0);
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      P[i * PW + c] = A[(size_t)i * n + k0 + c];
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      const int k = k0 + j;
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = k + tid; i < n; i += blockDim.x) {
        const double v = fabs(P[i * PW + j]);
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      block_argmax(best, bi, red_v, red_i, bcast, bidx);
      const int p = *bidx;
      if (tid == 0) pivg[k] = p;
      if (*bcast == 0.0) singular = true;
      if (p != k) {
        for (int c = tid; c < nb; c += blockDim.x) {
          const double t = P[k * PW + c];
          P[k * PW + c] = P[p * PW + c];
          P[p * PW + c] = t;
        }
      }
      __syncthreads();
      const double d = singular ? 0.0 : 1.0 / P[k * PW + j];
      // scale the pivot row (its column j becomes d)
      for (int c = tid; c < nb; c += blockDim.x) P[k * PW + c] = (c == j) ? d : P[k * PW + c] * d;
      __syncthreads();
      // eliminate column j from every other row
      for (int idx = tid; idx < n * nb; idx += blockDim.x) {
        const int i = idx / nb, c = idx - i * nb;
        if (i == k) continue;
        const double f = P[i * PW + j];
        if (c == j) continue;
        P[i * PW + c] -= f * P[k * PW + c];
      }
      __syncthreads();
      for (int i = tid; i < n; i += blockDim.x)
        if (i != k) P[i * PW + j] = -P[i * PW + j] * d;
      __syncthreads();
    }
    // interchange the pivot rows in the columns outside the panel
    for (int j = 0; j < nb; ++j) {
      const int k = k0 + j, p = pivg[k];
      if (p != k) {
        for (int c = tid; c < n - nb; c += blockDim.x) {
          const int cc = c < k0 ? c : c + nb;
          const double t = A[(size_t)k * n + cc];
          A[(size_t)k * n + cc] = A[(size_t)p * n + cc];
          A[(size_t)p * n + cc] = t;
        }
      }
      __syncthreads();
    }
    // T - I on the panel
    for (int j = tid; j < nb; j += blockDim.x) P[(k0 + j) * PW + j] -= 1.0;
    __syncthreads();
    // A[:, c] += (T - I)[:, panel] B[:, c] for every column c outside the panel
    const int nrest = n - nb;
    for (int tc = 0; tc < nrest; tc += 64) {
      const int wc = min(64, nrest - tc);
      for (int idx = tid; idx < GJ_NB * 64; idx += blockDim.x) {
        const int r = idx / 64, c = idx % 64;
        const int cc = tc + c < k0 ? tc + c : tc + c + nb;
        Bt[idx] = (c < wc && r < nb) ? A[(size_t)(k0 + r) * n + cc] : 0.0;
      }
      __syncthreads();
      for (int tr = 0; tr < n; tr += 64) {
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) acc[a][bq] = 0.0;
        for (int kk = 0; kk < nb; ++kk) {
          double lv[4], uv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = tr + ty + 16 * a;
            lv[a] = i < n ? P[i * PW + kk] : 0.0;
          }
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) uv[bq] = Bt[kk * 64 + tx + 16 * bq];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bq = 0; bq < 4; ++bq) acc[a][bq] += lv[a] * uv[bq];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = tr + ty + 16 * a;
          if (i >= n) continue;
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) {
            const int c = tx + 16 * bq;
            if (c < wc) {
              const int cc = tc + c < k0 ? tc + c : tc + c + nb;
              A[(size_t)i * n + cc] += acc[a][bq];
            }
          }
        }
      }
      __syncthreads();
    }
    for (int j = tid; j < nb; j += blockDim.x) P[(k0 + j) * PW + j] += 1.0;
    __syncthreads();
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      A[(size_t)i * n + k0 + c] = P[i * PW + c];
    }
    __syncthreads();
  }
  // undo the column interchanges, last pivot first
  for (int k = n - 1; k >= 0; --k) {
    const int p = pivg[k];
    if (p != k) {
      for (int i = tid; i < n; i += blockDim.x) {
        const double t = A[(size_t)i * n + k];
        A[(size_t)i * n + k] = A[(size_t)i * n + p];
        A[(size_t)i * n + p] = t;
      }
    }
    __syncthreads();
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
}

// n x n inverse (scratch) -> tiled layout (tiled_inv.cuh)
__global__ void __launch_bounds__(256) k_pack_inv(int n, const double* __restrict__ F, double* __restrict__ out) {
  const int mac = blockIdx.x;
  const double* A = F + (size_t)mac * n * n;
  double* O = out + (size_t)mac * ti_size(n);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int r = idx / n, c = idx % n;
    O[ti_idx(n, r, c)] = A[idx];
  }
  // zero the even padding of odd-sized tiles
  if (threadIdx.x == 0) {
    for (int b = 0; b < ti_nblk(n); ++b) {
      const int nb = ti_rows(n, b);
      long long o = ti_block_off(n, b);
      for (int c = 0; c < n; c += TI_CW) {
        const int w = (n - c) < TI_CW ? n - c : TI_CW;
        if (((long long)nb * w) & 1) O[o + (long long)nb * w] = 0.0;
        o += ti_even((long long)nb * w);
      }
    }
  }
}

int inv_factor(int n, int n_mac, double* scratch, double* tiled, int* status, cudaStream_t st) {
  const size_t bytes = gj_smem_bytes(n);
  if (bytes > 227 * 1024) return MHDG_ERR_CONFIG;
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_gj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_gj<<<n_mac, LU_THREADS, bytes, st>>>(n, scratch, status);
  int rc = launch_ok();
  if (rc) return rc;
  k_pack_inv<<<n_mac, 256, 0, st>>>(n, scratch, tiled);
  return launch_ok();
}

// --------------------------------------------------------------------------
// host launchers
// --------------------------------------------------------------------------

template <int D>
int schur_matrix(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st) {
  constexpr int NS = D + 2;
  const int kv = g.nq * D, kf = g.nqf * D, kmax = kv > kf ? kv : kf;
  const int rmax = (g.nloc > g.nlocf ? g.nloc : g.nlocf) * NS;
  const size_t bytes = sizeof(double) * ((size_t)rmax * kmax + (size_t)kmax * g.L);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_schur<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_schur<D><<<g.n_mac, SCHUR_THREADS, bytes, st>>>(g, b, S);
  return launch_ok();
}

size_t lu_smem_bytes(int n) {
  return sizeof(double) * ((size_t)n * (LU_NB + 1) + 2 * LU_NB * 64 + LU_NB * (LU_NB + 1) + 32 + 8) + sizeof(int) * (32 + LU_NB + 8) + 64;
}

int lu_factor(int n, int n_mac, double* scratch, double* packed, int* perm, int* status, cudaStream_t st) {
  const size_t bytes = lu_smem_bytes(n);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_lu<<<n_mac, LU_THREADS, bytes, st>>>(n, scratch, perm, status);
  int rc = launch_ok();
  if (rc) return rc;
  const size_t pbytes = sizeof(double) * 2 * PLU_NB * (PLU_NB + 1);
  cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes);
  k_pack<<<n_mac, 256, pbytes, st>>>(n, scratch, packed);
  return launch_ok();
}

template int schur_matrix<2>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template int schur_matrix<3>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);

}  // namespace mhdg
