// Second-layer static condensation on the device.
//
// k_schur_mma  S = state_state - A_uq A_qq^-1 A_qu (_schur_correction,
//              condense.py:130-158) on the FP64 tensor cores; k_schur is the
//              per-macro FFMA fallback (and A/B reference).
// k_gj3        explicit S^-1 (np.linalg.inv, condense.py:62-70) by Gauss-Jordan
//              with partial pivoting, pivots kept in place, DMMA updates;
//              k_pack_inv_rows tiles it for the apply (tiled_inv.cuh).  k_gj2
//              (row interchanges) and k_gj (32-column FFMA panels, any n that
//              fits) are the A/B variant and the large-n fallback.
// k_lu3        batched LU with partial pivoting (pivots in place), packed into
//              block-triangular solve order by k_pack_lu4 (packed_lu.cuh): the
//              MHDG_FACTOR=lu option.
// FactorizationError on an exactly zero pivot.
#include "common.cuh"
#include "dmma.cuh"
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


// S rows of one (face) sub-element += sign * X, X[(a,s),(j,r)] = sum_k T1[r][(a,s)][k] VW[k][j].
// Each thread owns one (a,s) row and 4 consecutive nodes j for all NS components r:
// per k it loads 4 VW and NS T1 values for 4*NS FMAs; the NS*4 outputs are contiguous.
template <int D>
__device__ __forceinline__ void schur_tile_update(const double* T1, const double* VW, int nas, int kk, int L,
                                                  double* Sm, int n, const int* loc, const int* fmap, double sign) {
  constexpr int NS = D + 2;
  const int nj = (L + 3) / 4;
  for (int task = threadIdx.x; task < nas * nj; task += blockDim.x) {
    const int as = task / nj, j0 = (task - as * nj) * 4;
    double acc[4][NS];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < NS; ++r) acc[u][r] = 0.0;
    for (int k = 0; k < kk; ++k) {
      double tv[NS], vw[4];
#pragma unroll
      for (int r = 0; r < NS; ++r) tv[r] = T1[(r * nas + as) * kk + k];
#pragma unroll
      for (int u = 0; u < 4; ++u) vw[u] = (j0 + u < L) ? VW[k * L + j0 + u] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int r = 0; r < NS; ++r) acc[u][r] += tv[r] * vw[u];
    }
    int node = __ldg(loc + as / NS);
    if (fmap) node = __ldg(fmap + node);
    double* out = Sm + (size_t)(node * NS + as % NS) * n + j0 * NS;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < L) {
#pragma unroll
        for (int r = 0; r < NS; ++r) out[u * NS + r] += sign * acc[u][r];
      }
  }
}

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

  // shared: T1[r][(a,s)][(q,l)] for all r, VW[(q,l)][j]
  const int kv = sz.nq * D, kf = sz.nqf * D;
  const int kmax = kv > kf ? kv : kf;
  const int rmax = sz.nloc * NS > sz.nlocf * NS ? sz.nloc * NS : sz.nlocf * NS;
  double* T1 = sm;
  double* VW = T1 + NS * rmax * kmax;

  // ---- volume sub-elements: X[(a,s),(j,r)] = sum_{(q,l)} T1[r][(a,s),(q,l)] VW[(q,l), j] ----
  for (int K = 0; K < sz.n_sub; ++K) {
    for (int idx = threadIdx.x; idx < kv * L; idx += blockDim.x) {
      const int j = idx % L, ql = idx / L, l = ql % D, q = ql / D;
      const double* pm = g.pm_vol + (((size_t)K * sz.nq + q) * D) * L + j;
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) a += __ldg(ij + r * D + l) * __ldg(pm + r * L);
      VW[idx] = a;
    }
    const int nas = sz.nloc * NS;
    for (int idx = threadIdx.x; idx < NS * nas * kv; idx += blockDim.x) {
      const int ql = idx % kv, rest = idx / kv, as = rest % nas, rr = rest / nas;
      const int s = as % NS, a = as / NS, l = ql % D, q = ql / D;
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
    // S[(conn[a],s), (j,rr)] += X, register-tiled: 4 nodes j x NS components per thread
    schur_tile_update<D>(T1, VW, nas, kv, L, Sm, n, g.sub_conn + K * sz.nloc, nullptr, 1.0);
    __syncthreads();
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
      const int nas = sz.nlocf * NS;
      for (int idx = threadIdx.x; idx < NS * nas * kf; idx += blockDim.x) {
        const int ql = idx % kf, rest = idx / kf, as = rest % nas, rr = rest / nas;
        const int s = as % NS, a = as / NS, l = ql % D, q = ql / D;
        const double* W = b.wdgdq_face +
                          ((((size_t)mac * NF + f) * sz.n_tri * sz.nqf + T * sz.nqf + q) * D + l) * NS * NS;
        T1[idx] = __ldg(W + s * NS + rr) * __ldg(g.phi_face + q * sz.nlocf + a);
      }
      __syncthreads();
      schur_tile_update<D>(T1, VW, nas, kf, L, Sm, n, g.tri_conn + T * sz.nlocf, g.face_vol_nodes + f * sz.Lf, -1.0);
      __syncthreads();
    }
  }
}

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


// --------------------------------------------------------------------------
// k_gj2: Gauss-Jordan inverse with 64-column panels and DMMA updates
// --------------------------------------------------------------------------
// Same algorithm as k_gj; the rank-64 update of the columns outside the panel,
// A[:, c] += (T - I)[:, panel] B[:, c], runs on the FP64 tensor cores
// (mma.sync.m8n8k4.f64 -> DMMA) with A-fragments from the shared panel and
// B-fragments from a staged 64x64 tile of the old pivot rows; C tiles are
// read-modify-written from global memory (L2).  The column interchanges are
// not undone here: the pivots go to `piv` and k_pack_inv applies the
// composed column permutation while tiling.

constexpr int GJ2_NB = 64, GJ2_PW = 68, GJ2_TC = 48, GJ2_BS = 52;  // strides chosen for conflict-free DMMA fragments

#ifdef MHDG_STREAM_PROFILE
__device__ unsigned long long g_gjprof[8];
#define GJT(v) long long v = clock64()
#define GJADD(k, v) if (threadIdx.x == 0) atomicAdd(&g_gjprof[k], (unsigned long long)(clock64() - (v)))
extern "C" int mhdg_gj_profile(unsigned long long* out, int reset) {
  if (out) cudaMemcpyFromSymbol(out, g_gjprof, sizeof(g_gjprof));
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_gjprof, z, sizeof(z));
  }
  return 0;
}
#else
#define GJT(v)
#define GJADD(k, v)
#endif


size_t gj2_smem_bytes(int n) {
  return sizeof(double) * ((size_t)n * GJ2_PW + GJ2_NB * GJ2_BS + 32 + 8) + sizeof(int) * (32 + 8) + 64;
}

__global__ void __launch_bounds__(512, 1) k_gj2(int n, double* __restrict__ S, int* __restrict__ piv_out,
                                                 int* status) {
  extern __shared__ double sm[];
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = S + (size_t)mac * n * n;
  int* pivg = piv_out + (size_t)mac * n;
  double* P = sm;                            // n x GJ2_PW panel
  double* Bt = P + (size_t)n * GJ2_PW;       // GJ2_NB x GJ2_TC old pivot rows (row stride GJ2_BS)
  double* red_v = Bt + GJ2_NB * GJ2_BS;      // 32
  int* red_i = (int*)(red_v + 32);           // 32
  double* bcast = (double*)(red_i + 32);     // 2
  int* bidx = (int*)(bcast + 2);
  bool singular = false;

  for (int k0 = 0; k0 < n; k0 += GJ2_NB) {
    const int nb = min(GJ2_NB, n - k0);
    GJT(t0);
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      P[i * GJ2_PW + c] = A[(size_t)i * n + k0 + c];
    }
    __syncthreads();
    GJADD(0, t0);
    // ---- panel: sub-panels of 16 columns; GJ steps inside the sub-panel,
    //      then the sub-panel's transform applied to the other panel columns
    //      with DMMA (C in shared memory) ----
    for (int js = 0; js < nb; js += 16) {
      GJT(t1);
      const int ns = min(16, nb - js);
      const int cl = tid & 15, rg = tid >> 4;  // thread -> (sub-panel column, row group)
      // partial pivot candidates for the next column, one per row group
      __shared__ double cand_v[32];
      __shared__ int cand_i[32];
      constexpr int RPT = 12;  // rows per thread (n <= 32 * RPT = 384)
      const int rbeg = rg * RPT;
      for (int j = js; j < js + ns; ++j) {
        const int k = k0 + j;
        if (warp == 0) {
          double best = -1.0;
          int bi = 0x7fffffff;
          if (j == js) {  // first column of the sub-panel: full scan
            for (int i = k + lane; i < n; i += 32) {
              const double v = fabs(P[i * GJ2_PW + j]);
              if (v > best || (v == best && i < bi)) { best = v; bi = i; }
            }
          } else {  // fused candidates from the previous step's elimination
            best = cand_v[lane];
            bi = cand_i[lane];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(MHDG_FULL, best, o);
            const int i2 = __shfl_xor_sync(MHDG_FULL, bi, o);
            if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
          }
          if (lane == 0) {
            *bidx = bi;
            bcast[0] = best;
            bcast[1] = best == 0.0 ? 0.0 : 1.0 / P[bi * GJ2_PW + j];  // one reciprocal per step
            pivg[k] = bi;
          }
        }
        __syncthreads();
        const int p = *bidx;
        if (bcast[0] == 0.0) singular = true;
        const double d = singular ? 0.0 : bcast[1];
        const int c = js + cl;
        const bool inside = cl < ns;
        const double rowp_c = inside ? P[p * GJ2_PW + c] : 0.0;
        const double rowk_c = inside ? P[k * GJ2_PW + c] : 0.0;
        const double rowk_j = P[k * GJ2_PW + j];
        __syncthreads();  // everyone has read rows k and p before anyone writes
        const bool next_col = (c == j + 1) && (j + 1 < js + ns);
        double cb = -1.0;
        int ci = 0x7fffffff;
        if (inside) {
          const double piv_c = (c == j) ? d : rowp_c * d;  // new row k
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int i = rbeg + q;
            if (i < n && i != k) {
              const double old_i = (i == p) ? rowk_c : P[i * GJ2_PW + c];
              const double old_ij = (i == p) ? rowk_j : P[i * GJ2_PW + j];
              const double nvl = (c == j) ? -old_ij * d : old_i - old_ij * piv_c;
              P[i * GJ2_PW + c] = nvl;
              if (next_col && i > k) {
                const double a = fabs(nvl);
                if (a > cb || (a == cb && i < ci)) { cb = a; ci = i; }
              }
            }
          }
          if (rg == (k / RPT)) P[k * GJ2_PW + c] = piv_c;
          if (next_col && k + 1 < n && rg == ((k + 1) / RPT) && false) {
          }
        }
        if (next_col) {
          cand_v[rg] = cb;
          cand_i[rg] = ci;
        }
        // columns of the panel outside the sub-panel: plain row interchange
        if (p != k)
          for (int cc = tid; cc < GJ2_NB; cc += blockDim.x)
            if (cc < js || cc >= js + ns) {
              const double t = P[k * GJ2_PW + cc];
              P[k * GJ2_PW + cc] = P[p * GJ2_PW + cc];
              P[p * GJ2_PW + cc] = t;
            }
        __syncthreads();
      }
      GJADD(1, t1);
      GJT(t2);
      // other panel columns c (outside [js, js+ns)): P[:, c] += (Ts - I) Bs[:, c]
      for (int idx = tid; idx < 16 * GJ2_NB; idx += blockDim.x) {
        const int r = idx >> 6, c = idx & 63;
        const bool other = (c < js || c >= js + ns) && c < nb && r < ns;
        Bt[r * 68 + c] = other ? P[(k0 + js + r) * GJ2_PW + c] : 0.0;
      }
      __syncthreads();
      for (int r = tid; r < ns; r += blockDim.x) P[(k0 + js + r) * GJ2_PW + js + r] -= 1.0;
      __syncthreads();
      {
        const int g = lane >> 2, t4 = lane & 3;
        // warp -> row band of 8 rows (step 8 * warps); all 8 column tiles of the panel
        for (int r0 = warp * 8; r0 < n; r0 += 8 * (int)(blockDim.x >> 5)) {
          double acc[8][2];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int row = r0 + g, col = 8 * jj + 2 * t4;
            const bool ok = row < n;
            acc[jj][0] = ok ? P[row * GJ2_PW + col] : 0.0;
            acc[jj][1] = ok ? P[row * GJ2_PW + col + 1] : 0.0;
          }
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            const int row = r0 + g;
            const double a = (row < n && kk + t4 < ns) ? P[row * GJ2_PW + js + kk + t4] : 0.0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) dmma_8x8x4(acc[jj][0], acc[jj][1], a, Bt[(kk + t4) * 68 + 8 * jj + g]);
          }
          __syncwarp();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int row = r0 + g, col = 8 * jj + 2 * t4;
            if (row < n) {
              if (col < js || col >= js + ns) P[row * GJ2_PW + col] = acc[jj][0];
              if (col + 1 < js || col + 1 >= js + ns) P[row * GJ2_PW + col + 1] = acc[jj][1];
            }
          }
        }
      }
      __syncthreads();
      for (int r = tid; r < ns; r += blockDim.x) P[(k0 + js + r) * GJ2_PW + js + r] += 1.0;
      __syncthreads();
      GJADD(2, t2);
    }
    GJT(t3);
    // ---- row interchanges outside the panel: the panel's swaps composed into
    //      one permutation (source map, O(n)), applied to the touched rows
    //      through shared memory ----
    {
      int* srcmap = (int*)Bt;          // n
      int* rows = srcmap + n + 1;      // touched rows (<= 2 GJ2_NB)
      double* stage = (double*)(rows + 2 * GJ2_NB + 2 - ((n + 1) & 1));  // 8-byte aligned
      __shared__ int nrows;
      for (int r = tid; r < n; r += blockDim.x) srcmap[r] = r;
      if (tid == 0) nrows = 0;
      __syncthreads();
      if (tid == 0)
        for (int j = 0; j < nb; ++j) {
          const int k = k0 + j, p = pivg[k];
          const int t = srcmap[k];
          srcmap[k] = srcmap[p];
          srcmap[p] = t;
        }
      __syncthreads();
      for (int r = tid; r < n; r += blockDim.x)
        if (srcmap[r] != r) rows[atomicAdd(&nrows, 1)] = r;
      __syncthreads();
      const int m = nrows;
      const int CW = 32;
      for (int c0 = 0; c0 < n - nb && m > 0; c0 += CW) {
        for (int idx = tid; idx < m * CW; idx += blockDim.x) {
          const int q = idx / CW, c = c0 + idx % CW;
          if (c < n - nb) {
            const int cc = c < k0 ? c : c + nb;
            stage[idx] = A[(size_t)srcmap[rows[q]] * n + cc];
          }
        }
        __syncthreads();
        for (int idx = tid; idx < m * CW; idx += blockDim.x) {
          const int q = idx / CW, c = c0 + idx % CW;
          if (c < n - nb) {
            const int cc = c < k0 ? c : c + nb;
            A[(size_t)rows[q] * n + cc] = stage[idx];
          }
        }
        __syncthreads();
      }
    }
    GJADD(3, t3);
    GJT(t_up);
    for (int j = tid; j < nb; j += blockDim.x) P[(k0 + j) * GJ2_PW + j] -= 1.0;  // T - I
    // zero the panel's unused columns so the k-loop can run over a full GJ2_NB
    for (int idx = tid; idx < n * (GJ2_NB - nb); idx += blockDim.x) {
      const int i = idx / (GJ2_NB - nb), c = nb + idx % (GJ2_NB - nb);
      P[i * GJ2_PW + c] = 0.0;
    }
    __syncthreads();
    // ---- update: C += (T - I) B over 64x64 tiles; 16 warps, warp tile 16 x 16,
    //      the next row tile's C prefetched into registers during the DMMAs ----
    const int nrest = n - nb;
    const int wr = (warp / 3) * 16, wc = (warp % 3) * 16;
    const int g = lane >> 2, t4 = lane & 3;
    for (int tc = 0; tc < nrest; tc += GJ2_TC) {
      const int wct = min(GJ2_TC, nrest - tc);
      for (int idx = tid; idx < GJ2_NB * GJ2_TC; idx += blockDim.x) {
        const int r = idx / GJ2_TC, c = idx % GJ2_TC;
        const int cc = tc + c < k0 ? tc + c : tc + c + nb;
        Bt[r * GJ2_BS + c] = (c < wct && r < nb) ? A[(size_t)(k0 + r) * n + cc] : 0.0;
      }
      __syncthreads();
      // 48-column tiles: warps 0..11 own 16x16 sub-tiles of each 64x48 C tile
      if (warp < 12) {
      // global column of this thread's two C columns per 8-wide tile
      int gcol[2][2];
      bool cok[2][2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wc + 8 * jj + 2 * t4 + e;
          cok[jj][e] = col < wct;
          gcol[jj][e] = tc + col < k0 ? tc + col : tc + col + nb;
        }
      double nxt[2][2][2];
      auto load_c = [&](int tr, double (&c)[2][2][2]) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = tr + wr + 8 * i + g;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) c[i][jj][e] = (row < n && cok[jj][e]) ? A[(size_t)row * n + gcol[jj][e]] : 0.0;
        }
      };
      load_c(0, nxt);
      for (int tr = 0; tr < n; tr += 64) {
        double acc[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            acc[i][jj][0] = nxt[i][jj][0];
            acc[i][jj][1] = nxt[i][jj][1];
          }
        if (tr + 64 < n) load_c(tr + 64, nxt);
#pragma unroll 8
        for (int kk = 0; kk < GJ2_NB; kk += 4) {
          double a[2], b[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int row = tr + wr + 8 * i + g;
            a[i] = row < n ? P[row * GJ2_PW + kk + t4] : 0.0;
          }
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) b[jj] = Bt[(kk + t4) * GJ2_BS + wc + 8 * jj + g];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], a[i], b[jj]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = tr + wr + 8 * i + g;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (row < n && cok[jj][e]) A[(size_t)row * n + gcol[jj][e]] = acc[i][jj][e];
        }
      }
      }  // warp < 12
      __syncthreads();
    }
    GJADD(4, t_up);
    GJT(t5);
    for (int j = tid; j < nb; j += blockDim.x) P[(k0 + j) * GJ2_PW + j] += 1.0;
    __syncthreads();
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      A[(size_t)i * n + k0 + c] = P[i * GJ2_PW + c];
    }
    __syncthreads();
    GJADD(5, t5);
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
}

// n x n inverse with pending column interchanges -> tiled layout.  The swaps
// (k <-> piv[k]) applied last-first compose into X[:, j] = A[:, idx[j]].
__global__ void __launch_bounds__(256) k_pack_inv_perm(int n, const double* __restrict__ F, const int* __restrict__ piv,
                                                       double* __restrict__ out) {
  extern __shared__ int idxs[];
  const int mac = blockIdx.x;
  const double* A = F + (size_t)mac * n * n;
  double* O = out + (size_t)mac * ti_size(n);
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) idxs[j] = j;
    for (int k = n - 1; k >= 0; --k) {
      const int p = piv[(size_t)mac * n + k];
      const int t = idxs[k];
      idxs[k] = idxs[p];
      idxs[p] = t;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int r = idx / n, c = idx % n;
    O[ti_idx(n, r, c)] = A[(size_t)r * n + idxs[c]];
  }
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

int inv_factor2(int n, int n_mac, double* scratch, int* piv, double* tiled, int* status, cudaStream_t st) {
  const size_t bytes = gj2_smem_bytes(n);
  if (bytes > 227 * 1024 || n > 384) return -1;  // 12 rows per thread x 32 row groups
  cudaFuncSetAttribute(k_gj2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_gj2<<<n_mac, 512, bytes, st>>>(n, scratch, piv, status);
  int rc = launch_ok();
  if (rc) return rc;
  k_pack_inv_perm<<<n_mac, 256, sizeof(int) * n, st>>>(n, scratch, piv, tiled);
  return launch_ok();
}

// --------------------------------------------------------------------------
// k_gj3: Gauss-Jordan inverse without physical row interchanges
// --------------------------------------------------------------------------
// As k_gj2 (64-column panels in shared memory, 16-column sub-panels, DMMA
// rank-16 / rank-64 updates), but the pivot of logical column k stays in its
// physical row p_k: partial pivoting picks the largest |entry| among the rows
// not yet used as pivots, the rows are never moved, and the identity part of
// the composite transform sits at (p_k, k).  The in-place result M then holds
// (P A)^-1 with row k stored in row p_k, so A^-1[i][j] = M[p_i][pi^-1(j)]
// (k_pack_inv_gather).  This removes the row-interchange passes over the
// matrix; each pivot step is two CTA barriers (every warp reduces the 32
// pivot candidates itself, every thread forms the reciprocal itself).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) k_gj3(int n, double* __restrict__ S, int* __restrict__ piv_out,
                                                 int* status) {
  extern __shared__ double sm[];
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = S + (size_t)mac * n * n;
  int* pivg = piv_out + (size_t)mac * n;
  double* P = sm;                       // n x GJ2_PW panel
  double* Bt = P + (size_t)n * GJ2_PW;  // old pivot rows (row stride GJ2_BS / 68)
  __shared__ double cand_v[32];
  __shared__ int cand_i[32];
  __shared__ int pv[GJ2_NB];            // physical pivot rows of the current panel
  constexpr int RPT = 12;               // rows per thread (n <= 32 * RPT = 384)
  const int cl = tid & 15, rg = tid >> 4, rbeg = rg * RPT;
  unsigned used = 0;                    // bit q: row rbeg + q is a pivot row already
  bool singular = false;

  // candidates for column `col` of P over this thread's unused rows (threads with cl == 0)
  auto scan = [&](int col) {
    if (cl == 0) {
      double cb = -1.0;
      int ci = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = rbeg + q;
        if (i < n && !((used >> q) & 1u)) {
          const double a = fabs(P[i * GJ2_PW + col]);
          if (a > cb) { cb = a; ci = i; }
        }
      }
      cand_v[rg] = cb;
      cand_i[rg] = ci;
    }
  };

  for (int k0 = 0; k0 < n; k0 += GJ2_NB) {
    const int nb = min(GJ2_NB, n - k0);
    GJT(t0);
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, c = idx - i * nb;
      P[i * GJ2_PW + c] = A[(size_t)i * n + k0 + c];
    }
    __syncthreads();
    scan(0);
    __syncthreads();
    GJADD(0, t0);
    for (int js = 0; js < nb; js += 16) {
      GJT(t1);
      const int ns = min(16, nb - js);
      const int c = js + cl;
      const bool inside = cl < ns;
      for (int j = js; j < js + ns; ++j) {
        // pivot: every warp reduces the 32 candidates (lowest row wins ties)
        double best = cand_v[lane];
        int p = cand_i[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double v2 = __shfl_xor_sync(MHDG_FULL, best, o);
          const int i2 = __shfl_xor_sync(MHDG_FULL, p, o);
          if (v2 > best || (v2 == best && i2 < p)) { best = v2; p = i2; }
        }
        if (!(best > 0.0)) singular = true;
        if (singular) p = 0;
        const double piv = P[p * GJ2_PW + j];
        const double d = singular ? 0.0 : 1.0 / piv;
        const double rowp_c = inside ? P[p * GJ2_PW + c] : 0.0;
        double colj[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) colj[q] = (rbeg + q < n) ? P[(rbeg + q) * GJ2_PW + j] : 0.0;
        __syncthreads();  // row p and column j read by everyone before anyone writes
        if (tid == 0) {
          pv[j] = p;
          pivg[k0 + j] = p;
        }
        if (p >= rbeg && p < rbeg + RPT) used |= 1u << (p - rbeg);
        const bool next_col = (c == j + 1) && (j + 1 < js + ns);
        double cb = -1.0;
        int ci = 0x7fffffff;
        if (inside) {
          const double piv_c = (c == j) ? d : rowp_c * d;  // new pivot row
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int i = rbeg + q;
            if (i < n && i != p) {
              const double nvl = (c == j) ? -colj[q] * d : P[i * GJ2_PW + c] - colj[q] * piv_c;
              P[i * GJ2_PW + c] = nvl;
              if (next_col && !((used >> q) & 1u)) {
                const double a = fabs(nvl);
                if (a > cb) { cb = a; ci = i; }
              }
            }
          }
          if (p >= rbeg && p < rbeg + RPT) P[p * GJ2_PW + c] = piv_c;
        }
        if (next_col) {
          cand_v[rg] = cb;
          cand_i[rg] = ci;
        }
        __syncthreads();
      }
      GJADD(1, t1);
      GJT(t2);
      // other panel columns c (outside [js, js+ns)): P[:, c] += (Ts - Es) Bs[:, c], Bs = old pivot rows
      for (int idx = tid; idx < 16 * GJ2_NB; idx += blockDim.x) {
        const int r = idx >> 6, cc = idx & 63;
        const bool other = (cc < js || cc >= js + ns) && cc < nb && r < ns;
        Bt[r * 68 + cc] = other ? P[pv[js + r] * GJ2_PW + cc] : 0.0;
      }
      __syncthreads();
      for (int r = tid; r < ns; r += blockDim.x) P[pv[js + r] * GJ2_PW + js + r] -= 1.0;
      __syncthreads();
      {
        const int g = lane >> 2, t4 = lane & 3;
        for (int r0 = warp * 8; r0 < n; r0 += 8 * (int)(blockDim.x >> 5)) {
          double acc[8][2];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int row = r0 + g, col = 8 * jj + 2 * t4;
            const bool ok = row < n;
            acc[jj][0] = ok ? P[row * GJ2_PW + col] : 0.0;
            acc[jj][1] = ok ? P[row * GJ2_PW + col + 1] : 0.0;
          }
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            const int row = r0 + g;
            const double a = (row < n && kk + t4 < ns) ? P[row * GJ2_PW + js + kk + t4] : 0.0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) dmma_8x8x4(acc[jj][0], acc[jj][1], a, Bt[(kk + t4) * 68 + 8 * jj + g]);
          }
          __syncwarp();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int row = r0 + g, col = 8 * jj + 2 * t4;
            if (row < n) {
              if (col < js || col >= js + ns) P[row * GJ2_PW + col] = acc[jj][0];
              if (col + 1 < js || col + 1 >= js + ns) P[row * GJ2_PW + col + 1] = acc[jj][1];
            }
          }
        }
      }
      __syncthreads();
      for (int r = tid; r < ns; r += blockDim.x) P[pv[js + r] * GJ2_PW + js + r] += 1.0;
      __syncthreads();
      if (js + 16 < nb) {
        scan(js + 16);
        __syncthreads();
      }
      GJADD(2, t2);
    }
    GJT(t_up);
    for (int j = tid; j < nb; j += blockDim.x) P[pv[j] * GJ2_PW + j] -= 1.0;  // T - E
    for (int idx = tid; idx < n * (GJ2_NB - nb); idx += blockDim.x) {
      const int i = idx / (GJ2_NB - nb), cc = nb + idx % (GJ2_NB - nb);
      P[i * GJ2_PW + cc] = 0.0;
    }
    __syncthreads();
    // ---- update of the columns outside the panel: C += (T - E) B, B = old pivot rows.
    //      128 x 48 C passes: warp (wm, wn) owns rows 16 wm.. (two 8-row tiles) of the
    //      3 column tiles 24 wn.. -- 6 independent DMMA accumulators; C of the next
    //      pass and the next chunk's pivot rows are prefetched into registers ----
    const int nrest = n - nb;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t4 = lane & 3;
    constexpr int BPT = GJ2_NB * GJ2_TC / 512;  // pivot-row tile entries per thread
    double bnext[BPT];
    auto load_b = [&](int tc) {
      const int wct = min(GJ2_TC, nrest - tc);
#pragma unroll
      for (int u = 0; u < BPT; ++u) {
        const int idx = tid + 512 * u, r = idx / GJ2_TC, cc0 = idx % GJ2_TC;
        const int cc = tc + cc0 < k0 ? tc + cc0 : tc + cc0 + nb;
        bnext[u] = (cc0 < wct && r < nb) ? A[(size_t)pv[r] * n + cc] : 0.0;
      }
    };
    if (nrest > 0) load_b(0);
    for (int tc = 0; tc < nrest; tc += GJ2_TC) {
      const int wct = min(GJ2_TC, nrest - tc);
#pragma unroll
      for (int u = 0; u < BPT; ++u) {
        const int idx = tid + 512 * u;
        Bt[(idx / GJ2_TC) * GJ2_BS + idx % GJ2_TC] = bnext[u];
      }
      __syncthreads();
      int gcol[3][2];
      bool cok[3][2];
#pragma unroll
      for (int jj = 0; jj < 3; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn * 24 + 8 * jj + 2 * t4 + e;
          cok[jj][e] = col < wct;
          gcol[jj][e] = tc + col < k0 ? tc + col : tc + col + nb;
        }
      auto load_c = [&](int tr, double (&cc)[2][3][2]) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = tr + wm * 16 + 8 * i + g;
#pragma unroll
          for (int jj = 0; jj < 3; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              cc[i][jj][e] = (row < n && cok[jj][e]) ? A[(size_t)row * n + gcol[jj][e]] : 0.0;
        }
      };
      double nx[2][3][2];
      load_c(0, nx);
      if (tc + GJ2_TC < nrest) load_b(tc + GJ2_TC);
      for (int tr = 0; tr < n; tr += 128) {
        double acc[2][3][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) {
            acc[i][jj][0] = nx[i][jj][0];
            acc[i][jj][1] = nx[i][jj][1];
          }
        if (tr + 128 < n) load_c(tr + 128, nx);
        const int row0 = tr + wm * 16 + g;
        if (tr + wm * 16 < n) {
#pragma unroll 4
          for (int kk = 0; kk < GJ2_NB; kk += 4) {
            double a[2], bb[3];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = row0 + 8 * i < n ? P[(row0 + 8 * i) * GJ2_PW + kk + t4] : 0.0;
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) bb[jj] = Bt[(kk + t4) * GJ2_BS + wn * 24 + 8 * jj + g];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int jj = 0; jj < 3; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], a[i], bb[jj]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int row = row0 + 8 * i;
#pragma unroll
            for (int jj = 0; jj < 3; ++jj)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (row < n && cok[jj][e]) A[(size_t)row * n + gcol[jj][e]] = acc[i][jj][e];
          }
        }
      }
      __syncthreads();
    }
    GJADD(4, t_up);
    GJT(t5);
    for (int j = tid; j < nb; j += blockDim.x) P[pv[j] * GJ2_PW + j] += 1.0;
    __syncthreads();
    for (int idx = tid; idx < n * nb; idx += blockDim.x) {
      const int i = idx / nb, cc = idx - i * nb;
      A[(size_t)i * n + k0 + cc] = P[i * GJ2_PW + cc];
    }
    __syncthreads();
    GJADD(5, t5);
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
}

// (P A)^-1 stored with row k in physical row piv[k] -> A^-1 in the tiled layout,
// A^-1[i][j] = M[piv[i]][inv[j]], inv = piv^-1, row by row: each warp stages source row p_i
// in shared memory with coalesced loads and writes the permuted row into its
// 64-row block, one contiguous 32-column tile row per lane group.
__global__ void __launch_bounds__(256) k_pack_inv_rows(int n, const double* __restrict__ F,
                                                       const int* __restrict__ piv, double* __restrict__ out) {
  extern __shared__ double rsm[];
  const int NP = (n + 1) & ~1;
  double* rowbuf = rsm + (threadIdx.x >> 5) * NP;
  int* pp = reinterpret_cast<int*>(rsm + 8 * NP);
  int* inv = pp + n;
  const int mac = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* A = F + (size_t)mac * n * n;
  double* O = out + (size_t)mac * ti_size(n);
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int p = piv[(size_t)mac * n + k];
    pp[k] = p;
    inv[p] = k;
  }
  __syncthreads();
  for (int r = warp; r < n; r += 8) {
    const double* src = A + (size_t)pp[r] * n;
    for (int c = lane; c < n; c += 32) rowbuf[c] = src[c];
    __syncwarp();
    const int b = r / TI_RB, rl = r - b * TI_RB, nb = ti_rows(n, b);
    const long long base = ti_block_off(n, b);
    for (int c = lane; c < n; c += 32) {
      const int j = c / TI_CW, c0 = j * TI_CW, w = (n - c0) < TI_CW ? n - c0 : TI_CW;
      O[base + (long long)j * nb * TI_CW + (long long)rl * w + (c - c0)] = rowbuf[inv[c]];
    }
    __syncwarp();
  }
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

int inv_factor3(int n, int n_mac, double* scratch, int* piv, double* tiled, int* status, cudaStream_t st) {
  const size_t bytes = gj2_smem_bytes(n);
  if (bytes > 227 * 1024 || n > 384) return -1;
  cudaFuncSetAttribute(k_gj3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  tl_begin(TL_FACTOR, st);
  k_gj3<<<n_mac, 512, bytes, st>>>(n, scratch, piv, status);
  tl_end(TL_FACTOR, st);
  int rc = launch_ok();
  if (rc) return rc;
  tl_begin(TL_PACK, st);
  const size_t pb = sizeof(double) * 8 * ((n + 1) & ~1) + sizeof(int) * 2 * n;
  if (pb > 48 * 1024) cudaFuncSetAttribute(k_pack_inv_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pb);
  k_pack_inv_rows<<<n_mac, 256, pb, st>>>(n, scratch, piv, tiled);
  tl_end(TL_PACK, st);
  return launch_ok();
}

// --------------------------------------------------------------------------
// k_schur_mma: the Schur correction on the FP64 tensor cores.
//
// With the geometry folded into the left factor, each (face) sub-element's
// correction is one GEMM against a macro-independent table:
//   X[(a,s,r), j] = sum_{(q,r')} T1'[(a,s,r),(q,r')] PM[(q,r'), j],
//   T1'[(a,s,r),(q,r')] = sum_l inv_jac[r',l] sum_k gphys[q,a,k] W[q][(k,l)][s][r],
//   S[(conn[a], s), (j, r)] += X   (faces: -=, folded into T1').
// One CTA per macro: W and PM staged in shared memory, T1' built there,
// DMMA m8n8k4 tiles whose accumulators start from the S entries they update
// (the read-modify-write of S is the MMA accumulate), sub-elements in the
// reference order so S is deterministic.  Strides make the A (= 4 mod 16) and
// B (= 8 mod 16) fragment loads conflict-free.
// --------------------------------------------------------------------------
// register tiles per dimension: NT column tiles (L <= 8 NT), KS k-steps ((q, r') <= 4 KS);
// the left factor is built for MC rows (a, s, r) at a time
template <int D>
struct SchT {
  static constexpr int NT = D == 2 ? 12 : 5, KS = D == 2 ? 8 : 21, MC = D == 2 ? 160 : 64;
};

template <int D>
struct SchurMmaDims {
  int kv, kf, sA, MV, MF, MVp, LP, nks_v, nks_f;
  __host__ __device__ SchurMmaDims(const mhdg_disc& g) {
    constexpr int NS = D + 2;
    kv = g.nq * D;
    kf = g.nqf * D;
    const int kmax = kv > kf ? kv : kf;
    sA = (kmax + 3) / 4 * 4;
    while (sA % 16 != 4) sA += 4;
    MV = g.nloc * NS * NS;
    MF = g.nlocf * NS * NS;
    const int mmax = MV > MF ? MV : MF;
    MVp = ((mmax < SchT<D>::MC ? mmax : SchT<D>::MC) + 7) / 8 * 8;  // rows of the left-factor buffer
    LP = (g.L + 7) / 8 * 8;
    if (LP % 16 == 0) LP += 8;
    nks_v = (kv + 3) / 4;
    nks_f = (kf + 3) / 4;
  }
  __host__ __device__ size_t smem_doubles(const mhdg_disc& g) const {
    constexpr int NS = D + 2;
    const int kmax = kv > kf ? kv : kf;
    const int nw = g.nq * D * D * NS * NS;
    return (size_t)MVp * sA + (size_t)(kmax + 3) / 4 * 4 * LP + nw + (size_t)g.n_grad_cls * g.nq * g.nloc * D;
  }
};

template <int D>
__global__ void __launch_bounds__(256, 2) k_schur_mma(mhdg_disc g, mhdg_blocks b, double* __restrict__ S) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2, NF = D + 1, NW = D * D * NS * NS;
  const SchurMmaDims<D> dm(g);
  const int mac = blockIdx.x, n = g.L * NS, L = g.L, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = g.nq, nloc = g.nloc, nqf = g.nqf, nlocf = g.nlocf;
  const int kmaxp = ((dm.kv > dm.kf ? dm.kv : dm.kf) + 3) / 4 * 4;
  double* Tp = sm;                                // MVp x sA   (rows (a,s,r), cols (q,r'))
  double* PM = Tp + (size_t)dm.MVp * dm.sA;        // kmaxp x LP (rows (q,r'), cols j)
  double* Wst = PM + (size_t)kmaxp * dm.LP;        // nq x NW (volume) / face stash
  double* gph = Wst + (size_t)nq * NW;             // n_grad_cls x nq x nloc x D
  double* Sm = S + (size_t)mac * n * n;
  double ij[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) ij[a][c] = __ldg(g.inv_jac + (size_t)mac * D * D + a * D + c);

  // S = state_state + corrections without a copy pass: the first volume sub-element
  // touching a node row (smallest K in the node's sorted incidence list) seeds its MMA
  // accumulators from state_state; later touches accumulate onto S.
  const double* SSm = b.state_state + (size_t)mac * n * n;
  // physical gradients per class, zero padding of the GEMM operands
  for (int idx = tid; idx < g.n_grad_cls * nq * nloc * D; idx += blockDim.x) {
    const int k = idx % D, base = idx - k;
    double v = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) v += __ldg(g.grad_cls + base + r) * ij[r][k];
    gph[idx] = v;
  }
  for (int idx = tid; idx < dm.MVp * dm.sA; idx += blockDim.x) Tp[idx] = 0.0;
  for (int idx = tid; idx < kmaxp * dm.LP; idx += blockDim.x) PM[idx] = 0.0;
  __syncthreads();  // S rows visible to every warp before the first accumulate

  const int gq = lane >> 2, t4 = lane & 3;
  // C[M x LP] = Tp[M x 4 nks] PM[4 nks x LP], accumulated into S rows; rows m -> (node, s, r).
  // Per M tile all SCH_NT column tiles of C are loaded from S first (one memory latency per
  // M tile), accumulated by DMMA and stored.
  constexpr int SNT = SchT<D>::NT, SKS = SchT<D>::KS;
  // rows m0 .. m0 + M - 1 of the left factor, held in Tp rows 0 .. M - 1
  auto gemm_into_s = [&](int M, int m0, int nks, auto&& row_node, int Kfirst) {
    const int mtiles = (M + 7) / 8, ntiles = (L + 7) / 8;
    for (int mt = warp; mt < mtiles; mt += 8) {
      const int ml = mt * 8 + gq, m = m0 + ml;
      const bool mok = ml < M;
      const int a = m / (NS * NS), s = (m / NS) % NS, r = m % NS;
      const int node = mok ? row_node(a) : 0;
      const bool first = Kfirst >= 0 && __ldg(g.vn_sub + __ldg(g.vn_ptr + node)) / nloc == Kfirst;
      double* srow = Sm + (size_t)(node * NS + s) * n + r;
      const double* crow = first ? SSm + (size_t)(node * NS + s) * n + r : srow;
      double af[SKS];
#pragma unroll
      for (int ks = 0; ks < SKS; ++ks) af[ks] = ks < nks ? Tp[ml * dm.sA + 4 * ks + t4] : 0.0;
      double c[SNT][2];
#pragma unroll
      for (int nt = 0; nt < SNT; ++nt) {
        const int j0 = nt * 8 + 2 * t4;
        c[nt][0] = (mok && nt < ntiles && j0 < L) ? crow[j0 * NS] : 0.0;
        c[nt][1] = (mok && nt < ntiles && j0 + 1 < L) ? crow[(j0 + 1) * NS] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < SNT; ++nt)
        if (nt < ntiles) {
#pragma unroll
          for (int ks = 0; ks < SKS; ++ks)
            if (ks < nks) dmma_8x8x4(c[nt][0], c[nt][1], af[ks], PM[(4 * ks + t4) * dm.LP + nt * 8 + gq]);
        }
#pragma unroll
      for (int nt = 0; nt < SNT; ++nt) {
        const int j0 = nt * 8 + 2 * t4;
        if (mok && nt < ntiles && j0 < L) srow[j0 * NS] = c[nt][0];
        if (mok && nt < ntiles && j0 + 1 < L) srow[(j0 + 1) * NS] = c[nt][1];
      }
    }
  };

  // The stash of the next (face) sub-element streams in (cp.async) while the GEMMs of the
  // current one run; on arrival the inverse Jacobian is folded into it in place,
  // W'[q][(k, r')][s][r] = sum_l inv_jac[r'][l] W[q][(k, l)][s][r], so a left-factor entry
  // is D products.
  const int nwv = nq * NW, nwf = nqf * D * NS * NS, nstash = g.n_sub + NF * g.n_tri;
  auto stash_src = [&](int i) -> const double* {
    if (i < g.n_sub) return b.wdgdq_vol + ((size_t)mac * g.n_sub + i) * nwv;
    const int fT = i - g.n_sub;  // f * n_tri + T
    return b.wdgdq_face + ((size_t)mac * NF * g.n_tri + fT) * nwf;
  };
  auto prefetch = [&](int i) {
    if (i >= nstash) return;
    const double* src = stash_src(i);
    const int cnt = i < g.n_sub ? nwv : nwf;
    for (int e = tid; e < cnt; e += blockDim.x) cp_async8(Wst + e, src + e, 8);
  };
  auto land_and_fold = [&](int i) {  // wait for stash i, fold inv_jac into it
    cp_async_wait_all();
    __syncthreads();
    const int ngrp = (i < g.n_sub ? nq * D : nqf) * NS * NS;  // (q[, k], s, r) groups
    for (int e = tid; e < ngrp; e += blockDim.x) {
      const int sr = e % (NS * NS), qk = e / (NS * NS);  // qk = q * D + k (volume) or q (face)
      double* w = Wst + (size_t)qk * D * NS * NS + sr;
      double v[D];
#pragma unroll
      for (int l = 0; l < D; ++l) v[l] = w[l * NS * NS];
#pragma unroll
      for (int rp = 0; rp < D; ++rp) {
        double t = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) t += ij[rp][l] * v[l];
        w[rp * NS * NS] = t;
      }
    }
  };

  // ---- volume sub-elements ----
  prefetch(0);
  for (int K = 0; K < g.n_sub; ++K) {
    land_and_fold(K);
    for (int idx = tid; idx < dm.kv * L; idx += blockDim.x) {
      const int j = idx % L, qr = idx / L;
      PM[qr * dm.LP + j] = __ldg(g.pm_vol + ((size_t)K * dm.kv + qr) * L + j);
    }
    __syncthreads();
    const int cls = __ldg(g.grad_cls_of + K);
    for (int m0 = 0; m0 < dm.MV; m0 += dm.MVp) {
      const int mc = min(dm.MVp, dm.MV - m0);
      for (int idx = tid; idx < mc * dm.kv; idx += blockDim.x) {
        const int qr = idx % dm.kv, ml = idx / dm.kv, m = m0 + ml;
        const int q = qr / D, rp = qr % D, a = m / (NS * NS), s = (m / NS) % NS, r = m % NS;
        const double* gp = gph + ((cls * nq + q) * nloc + a) * D;
        const double* w = Wst + q * NW + (rp * NS + s) * NS + r;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) v += gp[k] * w[k * D * NS * NS];
        Tp[ml * dm.sA + qr] = v;
      }
      __syncthreads();
      if (m0 + dm.MVp >= dm.MV) prefetch(K + 1);  // the stash is consumed: overlap the next one
      gemm_into_s(mc, m0, dm.nks_v, [&](int a) { return __ldg(g.sub_conn + K * nloc + a); }, K);
      __syncthreads();
    }
  }
  // ---- face sub-elements (sign folded into T1') ----
  for (int idx = tid; idx < dm.MVp * dm.sA; idx += blockDim.x) Tp[idx] = 0.0;
  for (int idx = tid; idx < kmaxp * dm.LP; idx += blockDim.x) PM[idx] = 0.0;
  for (int f = 0; f < NF; ++f) {
    for (int T = 0; T < g.n_tri; ++T) {
      const int si = g.n_sub + f * g.n_tri + T;
      land_and_fold(si);
      for (int idx = tid; idx < dm.kf * L; idx += blockDim.x) {
        const int j = idx % L, qr = idx / L;
        PM[qr * dm.LP + j] = __ldg(g.pm_face + (((size_t)f * g.n_tri + T) * dm.kf + qr) * L + j);
      }
      __syncthreads();
      for (int m0 = 0; m0 < dm.MF; m0 += dm.MVp) {
        const int mc = min(dm.MVp, dm.MF - m0);
        for (int idx = tid; idx < mc * dm.kf; idx += blockDim.x) {
          const int qr = idx % dm.kf, ml = idx / dm.kf, m = m0 + ml;
          const int q = qr / D, rp = qr % D, a = m / (NS * NS), s = (m / NS) % NS, r = m % NS;
          Tp[ml * dm.sA + qr] = -Wst[((q * D + rp) * NS + s) * NS + r] * __ldg(g.phi_face + q * nlocf + a);
        }
        __syncthreads();
        if (m0 + dm.MVp >= dm.MF) prefetch(si + 1);
        gemm_into_s(mc, m0, dm.nks_f, [&](int a) {
          return __ldg(g.face_vol_nodes + f * g.Lf + __ldg(g.tri_conn + T * nlocf + a));
        }, -1);
        __syncthreads();
      }
    }
  }
}

// --------------------------------------------------------------------------
// k_lu3: batched LU with partial pivoting, pivots kept in place (the
// factorisation the canonical F_cond counts: (2/3) n^3).
// --------------------------------------------------------------------------
// Logical row k of P S = L U lives in physical row piv[k]; columns are never
// permuted.  Per 48-column panel the not-yet-pivoted rows are compacted
// (m = n - k0 rows), so the pivot steps shrink as the factorisation proceeds.
// Inside a panel, 16-column sub-panels are factored by pivot steps (argmax over
// the sub-panel column, multipliers, rank-1 updates of the sub-panel); the
// sub-panel's U rows are then completed on the rest of the panel (16-step
// triangular solve per column) and the other rows updated by a DMMA rank-16
// product.  After the panel: for each 48-column chunk of the columns to its
// right, the pivot rows are staged (A12), turned into U12 = L11^-1 A12 with
// the inverted 16x16 diagonal blocks, written back, and the remaining rows
// updated by a DMMA rank-48 product (C -= L21 U12).  FactorizationError on an
// exactly zero pivot (scipy's lu_factor raises on singular input).
// Panel width NB and CTA size NT are template parameters: NB = 24, NT = 256
// keeps a CTA at ~99 KB of shared memory, so two macros are factored per SM and
// hide each other's pivot-step latency.
template <int NB, int NT>
struct Lu3 {
  static constexpr int PW = NB + 4;               // panel row stride
  static constexpr int TC = 48, BS = 52;           // column chunk of the trailing update, its stride
  static constexpr int NSB = (NB + 15) / 16;       // 16-row diagonal blocks of L11
  static constexpr int NRG = NT / 16;              // row groups
  static constexpr int RPT = (384 + NRG - 1) / NRG;  // compacted rows per thread (n <= 384)
  static constexpr int NW = NT / 32;
  static size_t smem_bytes(int n) {
    return sizeof(double) * ((size_t)n * PW + (size_t)NB * BS + (size_t)NSB * 16 * 17) + sizeof(int) * (3 * (size_t)n + 8);
  }
};

template <int NB, int NT>
__global__ void __launch_bounds__(NT, 2) k_lu3(int n, double* __restrict__ S, int* __restrict__ piv_out, int* status) {
  using C = Lu3<NB, NT>;
  constexpr int PW = C::PW, TC = C::TC, BS = C::BS, RPT = C::RPT, NWp = C::NW;
  extern __shared__ double sm[];
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = S + (size_t)mac * n * n;
  int* pivg = piv_out + (size_t)mac * n;
  double* P = sm;                                   // m x PW: the panel over the compacted rows
  double* Bt = P + (size_t)n * PW;                  // NB x BS: U rows (sub-panel / A12 chunk)
  double* Di = Bt + NB * BS;                        // NSB x 16 x 17: inverted unit-lower diagonal blocks
  int* rows = reinterpret_cast<int*>(Di + C::NSB * 16 * 17);  // n: compacted physical rows
  int* done = rows + n;                                        // n: 1 = pivot row of an earlier panel
  int* ispiv = done + n;                                       // n: compacted row is a pivot of this panel
  __shared__ double cand_v[32];
  __shared__ int cand_i[32];
  __shared__ int ppos[NB];  // compacted positions of this panel's pivots (logical order)
  __shared__ int mrows;
  const int cl = tid & 15, rg = tid >> 4;
  bool singular = false;
  for (int i = tid; i < n; i += NT) done[i] = 0;
  if (tid < 32) {
    cand_v[tid] = -1.0;
    cand_i[tid] = 0x7fffffff;
  }
  __syncthreads();

  for (int k0 = 0; k0 < n; k0 += NB) {
    const int nb = min(NB, n - k0);
    if (tid == 0) {
      int m = 0;
      for (int i = 0; i < n; ++i)
        if (!done[i]) rows[m++] = i;
      mrows = m;
    }
    __syncthreads();
    const int m = mrows;  // = n - k0
    const int rpt = (m + C::NRG - 1) / C::NRG;
    const int rbeg = rg * rpt;
    unsigned piv_here = 0;  // bit q: compacted row rbeg + q pivoted in this panel
    GJT(t0);
    for (int idx = tid; idx < m * nb; idx += NT) {
      const int r = idx / nb, c = idx - r * nb;
      P[r * PW + c] = A[(size_t)rows[r] * n + k0 + c];
    }
    for (int r = tid; r < m; r += NT) ispiv[r] = 0;
    __syncthreads();
    GJADD(0, t0);
    for (int js = 0; js < nb; js += 16) {
      GJT(t1);
      const int ns = min(16, nb - js);
      const int c = js + cl;
      const bool inside = cl < ns;
      if (cl == 0) {  // candidates for the sub-panel's first column
        double cb = -1.0;
        int ci = 0x7fffffff;
        for (int q = 0; q < rpt; ++q) {
          const int r = rbeg + q;
          if (r < m && !((piv_here >> q) & 1u)) {
            const double a = fabs(P[r * PW + js]);
            if (a > cb) { cb = a; ci = r; }
          }
        }
        cand_v[rg] = cb;
        cand_i[rg] = ci;
      }
      __syncthreads();
      for (int j = js; j < js + ns; ++j) {
        double best = cand_v[lane];
        int p = cand_i[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double v2 = __shfl_xor_sync(MHDG_FULL, best, o);
          const int i2 = __shfl_xor_sync(MHDG_FULL, p, o);
          if (v2 > best || (v2 == best && i2 < p)) { best = v2; p = i2; }
        }
        if (!(best > 0.0)) singular = true;
        if (singular) p = 0;
        const double d = singular ? 0.0 : 1.0 / P[p * PW + j];
        const double rowp_c = (inside && c > j) ? P[p * PW + c] : 0.0;
        double colj[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) colj[q] = (q < rpt && rbeg + q < m) ? P[(rbeg + q) * PW + j] : 0.0;
        __syncthreads();  // row p and column j read by everyone before anyone writes
        if (tid == 0) {
          ppos[j] = p;
          ispiv[p] = 1;
          pivg[k0 + j] = rows[p];
        }
        if (p >= rbeg && p < rbeg + rpt) piv_here |= 1u << (p - rbeg);
        const bool next_col = (c == j + 1) && (j + 1 < js + ns);
        double cb = -1.0;
        int ci = 0x7fffffff;
        if (inside && c >= j) {
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int r = rbeg + q;
            if (q < rpt && r < m && !((piv_here >> q) & 1u)) {
              const double l = colj[q] * d;
              const double nv = (c == j) ? l : P[r * PW + c] - l * rowp_c;
              P[r * PW + c] = nv;
              if (next_col) {
                const double a = fabs(nv);
                if (a > cb) { cb = a; ci = r; }
              }
            }
          }
        }
        if (next_col) {
          cand_v[rg] = cb;
          cand_i[rg] = ci;
        }
        __syncthreads();
      }
      GJADD(1, t1);
      GJT(t2);
      const int c0 = js + ns, nrc = nb - c0;  // panel columns right of the sub-panel
      if (nrc > 0) {
        // (a) the sub-panel's U rows on those columns: forward substitution with its unit-lower block
        for (int cc = tid; cc < nrc; cc += NT) {
          for (int k = 1; k < ns; ++k) {
            double v = P[ppos[js + k] * PW + c0 + cc];
            for (int k2 = 0; k2 < k; ++k2) v -= P[ppos[js + k] * PW + js + k2] * P[ppos[js + k2] * PW + c0 + cc];
            P[ppos[js + k] * PW + c0 + cc] = v;
          }
        }
        __syncthreads();
        for (int idx = tid; idx < 16 * NB; idx += NT) {
          const int k = idx / NB, cc = idx % NB;
          Bt[k * BS + cc] = (k < ns && cc < nrc) ? P[ppos[js + k] * PW + c0 + cc] : 0.0;
        }
        __syncthreads();
        // (b) rows not pivoted in this panel: P[r][c0 + cc] -= sum_k L[r][js + k] U[k][cc] (DMMA)
        {
          const int g = lane >> 2, t4 = lane & 3;
          constexpr int NT8 = (NB + 7) / 8;
          const int ntile = (nrc + 7) / 8;
          for (int r0 = warp * 8; r0 < m; r0 += 8 * NWp) {
            const int r = r0 + g;
            const bool upd = r < m && !ispiv[r];
            double acc[NT8][2];
#pragma unroll
            for (int jj = 0; jj < NT8; ++jj) {
              const int col = 8 * jj + 2 * t4;
              acc[jj][0] = (r < m && jj < ntile && col < nrc) ? P[r * PW + c0 + col] : 0.0;
              acc[jj][1] = (r < m && jj < ntile && col + 1 < nrc) ? P[r * PW + c0 + col + 1] : 0.0;
            }
#pragma unroll
            for (int kk = 0; kk < 16; kk += 4) {
              const double a = (r < m && kk + t4 < ns) ? -P[r * PW + js + kk + t4] : 0.0;
#pragma unroll
              for (int jj = 0; jj < NT8; ++jj)
                if (jj < ntile) dmma_8x8x4(acc[jj][0], acc[jj][1], a, Bt[(kk + t4) * BS + 8 * jj + g]);
            }
            __syncwarp();
            if (upd) {
#pragma unroll
              for (int jj = 0; jj < NT8; ++jj) {
                const int col = 8 * jj + 2 * t4;
                if (jj < ntile && col < nrc) P[r * PW + c0 + col] = acc[jj][0];
                if (jj < ntile && col + 1 < nrc) P[r * PW + c0 + col + 1] = acc[jj][1];
              }
            }
          }
        }
        __syncthreads();
      }
      GJADD(2, t2);
    }
    GJT(t_up);
    // ---- inverted unit-lower 16x16 diagonal blocks of L11 (pivot rows, logical order) ----
    const int nsb = (nb + 15) / 16;
    if (tid < 16 * nsb) {
      const int i = tid / 16, cc = tid % 16, b0 = 16 * i, bn = min(16, nb - b0);
      double* X = Di + i * 16 * 17;
      if (cc < bn) {
        X[cc * 17 + cc] = 1.0;
        for (int rr = cc + 1; rr < bn; ++rr) {
          double acc = 0.0;
          for (int k = cc; k < rr; ++k) acc += P[ppos[b0 + rr] * PW + b0 + k] * X[k * 17 + cc];
          X[rr * 17 + cc] = -acc;
        }
        for (int rr = 0; rr < cc; ++rr) X[rr * 17 + cc] = 0.0;
      }
    }
    __syncthreads();
    // ---- columns right of the panel: U12 = L11^-1 A12 per chunk, then C -= L21 U12 ----
    const int nright = n - k0 - nb;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t4 = lane & 3;
    constexpr int RPP = (NT / 64) * 16;       // rows per pass of the trailing product
    constexpr int TPT = (16 * TC + NT - 1) / NT;  // TRSM entries per thread and 16-row block
    for (int tc = 0; tc < nright; tc += TC) {
      GJT(t6);
      const int wct = min(TC, nright - tc), cbase = k0 + nb + tc;
      for (int idx = tid; idx < NB * TC; idx += NT) {
        const int k = idx / TC, cc = idx % TC;
        Bt[k * BS + cc] = (k < nb && cc < wct) ? A[(size_t)rows[ppos[k]] * n + cbase + cc] : 0.0;
      }
      __syncthreads();
      for (int i = 0; i < nsb; ++i) {  // Bt_i = D_i (Bt_i - L[i, <i] Bt_<i)
        const int b0 = 16 * i, bn = min(16, nb - b0);
        double t[TPT];
#pragma unroll
        for (int h = 0; h < TPT; ++h) {
          const int idx = tid + NT * h, k = idx / TC, cc = idx % TC;
          double v = 0.0;
          if (idx < 16 * TC && k < bn) {
            v = Bt[(b0 + k) * BS + cc];
            for (int k2 = 0; k2 < b0; ++k2) v -= P[ppos[b0 + k] * PW + k2] * Bt[k2 * BS + cc];
          }
          t[h] = v;
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < TPT; ++h) {
          const int idx = tid + NT * h, k = idx / TC, cc = idx % TC;
          if (idx < 16 * TC && k < bn) Bt[(b0 + k) * BS + cc] = t[h];
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < TPT; ++h) {
          const int idx = tid + NT * h, k = idx / TC, cc = idx % TC;
          double v = 0.0;
          if (idx < 16 * TC && k < bn)
            for (int k2 = 0; k2 <= k; ++k2) v += Di[i * 16 * 17 + k * 17 + k2] * Bt[(b0 + k2) * BS + cc];
          t[h] = v;
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < TPT; ++h) {
          const int idx = tid + NT * h, k = idx / TC, cc = idx % TC;
          if (idx < 16 * TC && k < bn) Bt[(b0 + k) * BS + cc] = t[h];
        }
        __syncthreads();
      }
      for (int idx = tid; idx < nb * wct; idx += NT) {
        const int k = idx / wct, cc = idx % wct;
        A[(size_t)rows[ppos[k]] * n + cbase + cc] = Bt[k * BS + cc];
      }
      GJADD(6, t6);
      GJT(t7);
      // C -= L21 U12 over the panel's other rows: warp (wm, wn) owns 16 rows x 3 column tiles
      for (int tr = 0; tr < m; tr += RPP) {
        double acc[2][3][2];
        bool upd[2];
        int prow[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = tr + wm * 16 + 8 * i + g;
          upd[i] = r < m && !ispiv[r];
          prow[i] = r < m ? rows[r] : 0;
#pragma unroll
          for (int jj = 0; jj < 3; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = wn * 24 + 8 * jj + 2 * t4 + e;
              acc[i][jj][e] = (upd[i] && col < wct) ? A[(size_t)prow[i] * n + cbase + col] : 0.0;
            }
        }
        if (tr + wm * 16 < m) {
#pragma unroll
          for (int kk = 0; kk < NB; kk += 4) {
            double a[2], bb[3];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = tr + wm * 16 + 8 * i + g;
              a[i] = (r < m && kk + t4 < nb) ? -P[r * PW + kk + t4] : 0.0;
            }
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) bb[jj] = Bt[(kk + t4) * BS + wn * 24 + 8 * jj + g];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int jj = 0; jj < 3; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], a[i], bb[jj]);
          }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jj = 0; jj < 3; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = wn * 24 + 8 * jj + 2 * t4 + e;
              if (upd[i] && col < wct) A[(size_t)prow[i] * n + cbase + col] = acc[i][jj][e];
            }
      }
      __syncthreads();
      GJADD(7, t7);
    }
    GJADD(4, t_up);
    GJT(t5);
    for (int idx = tid; idx < m * nb; idx += NT) {
      const int r = idx / nb, cc = idx - r * nb;
      A[(size_t)rows[r] * n + k0 + cc] = P[r * PW + cc];
    }
    for (int k = tid; k < nb; k += NT) done[rows[ppos[k]]] = 1;
    __syncthreads();
    GJADD(5, t5);
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
}

#ifndef MHDG_LU_NB
#define MHDG_LU_NB 24
#endif
#ifndef MHDG_LU_NT
#define MHDG_LU_NT 256
#endif

// packs an in-place LU (pivot rows in place) into the solve layout (lu.cu)
int pack_lu4(int n, int n_mac, const double* scratch, const int* piv, double* packed, cudaStream_t st);

int lu_factor3(int n, int n_mac, double* scratch, int* piv, double* packed, int* status, cudaStream_t st) {
  using L3 = Lu3<MHDG_LU_NB, MHDG_LU_NT>;
  const size_t bytes = L3::smem_bytes(n);
  if (bytes > 227 * 1024 || n > 384) return -1;
  auto kern = k_lu3<MHDG_LU_NB, MHDG_LU_NT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  tl_begin(TL_FACTOR, st);
  kern<<<n_mac, MHDG_LU_NT, bytes, st>>>(n, scratch, piv, status);
  tl_end(TL_FACTOR, st);
  int rc = launch_ok();
  if (rc) return rc;
  return pack_lu4(n, n_mac, scratch, piv, packed, st);
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

int g_schur_variant = 0;  // 0: k_schur2, 1: k_schur_mma, else per-macro FFMA (A/B knob)
template <int D>
int schur2(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st);

template <int D>
int schur_matrix(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st) {
  constexpr int NS = D + 2;
  const int kv = g.nq * D, kf = g.nqf * D, kmax = kv > kf ? kv : kf;
  const int rmax = (g.nloc > g.nlocf ? g.nloc : g.nlocf) * NS;
  const int n = g.L * NS;
  if (g_schur_variant == 0) {  // stage-pipelined tensor-core kernel (schur.cu)
    const int rc = schur2<D>(g, b, S, st);
    if (rc >= 0) return rc;
  }
  {  // earlier tensor-core kernel when its operands fit
    const SchurMmaDims<D> dm(g);
    const size_t mb = sizeof(double) * dm.smem_doubles(g);
    if (g_schur_variant <= 1 && dm.nks_v <= SchT<D>::KS && dm.nks_f <= SchT<D>::KS &&
        g.L <= 8 * SchT<D>::NT &&
        mb <= 227 * 1024 && g.grad_cls) {
      if (mb > 48 * 1024) cudaFuncSetAttribute(k_schur_mma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mb);
      k_schur_mma<D><<<g.n_mac, 256, mb, st>>>(g, b, S);
      return launch_ok();
    }
  }
  const size_t bytes = sizeof(double) * ((size_t)NS * rmax * kmax + (size_t)kmax * g.L);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_schur<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_schur<D><<<g.n_mac, SCHUR_THREADS, bytes, st>>>(g, b, S);
  return launch_ok();
}

template int schur_matrix<2>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template int schur_matrix<3>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);

}  // namespace mhdg
