// Second-layer static condensation on the device.
//
// schur_matrix  S = state_state - A_uq A_qq^-1 A_qu (_schur_correction,
//               condense.py:130-158): the stage-pipelined FP64 tensor-core
//               kernel k_schur2 (schur.cu) when its stages fit shared memory,
//               else k_schur, the per-macro FFMA kernel for any (d, m, p).
// k_gj3         MHDG_FACTOR=inverse: explicit S^-1 (np.linalg.inv,
//               condense.py:62-70) by Gauss-Jordan with partial pivoting,
//               pivots kept in place, DMMA updates, n <= 384; k_pack_inv_rows
//               tiles it for the apply (tiled_inv.cuh).  k_gj (32-column FFMA
//               panels) covers larger n whose panel fits shared memory.
// The default packed-LU factor kind lives in lu.cu.
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

// The quadrature k = (q, l) extent of a sub-element is processed in chunks of kc so the
// left factor T1 (NS x nloc NS x kc) and VW (kc x L) fit shared memory for any (d, m, p)
// (3D p = 3: nq D = 192); the chunks accumulate into S in a fixed order.
template <int D>
__global__ void __launch_bounds__(SCHUR_THREADS) k_schur(mhdg_disc g, mhdg_blocks b, double* __restrict__ S, int kc) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2, NF = D + 1;
  const Sz sz = make_sz<D>(g);
  const int mac = blockIdx.x, n = sz.n, L = sz.L;
  const double* ij = g.inv_jac + (size_t)mac * D * D;
  double* Sm = S + (size_t)mac * n * n;
  const double* SS = b.state_state + (size_t)mac * n * n;
  for (size_t i = threadIdx.x; i < (size_t)n * n; i += blockDim.x) Sm[i] = SS[i];
  __syncthreads();

  // shared: T1[r][(a,s)][(q,l) chunk] for all r, VW[(q,l) chunk][j]
  const int kv = sz.nq * D, kf = sz.nqf * D;
  const int rmax = sz.nloc * NS > sz.nlocf * NS ? sz.nloc * NS : sz.nlocf * NS;
  double* T1 = sm;
  double* VW = T1 + (size_t)NS * rmax * kc;

  // ---- volume sub-elements: X[(a,s),(j,r)] = sum_{(q,l)} T1[r][(a,s),(q,l)] VW[(q,l), j] ----
  for (int K = 0; K < sz.n_sub; ++K) {
    for (int c0 = 0; c0 < kv; c0 += kc) {
      const int kw = min(kc, kv - c0);
      for (int idx = threadIdx.x; idx < kw * L; idx += blockDim.x) {
        const int j = idx % L, ql = c0 + idx / L, l = ql % D, q = ql / D;
        const double* pm = g.pm_vol + (((size_t)K * sz.nq + q) * D) * L + j;
        double a = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) a += __ldg(ij + r * D + l) * __ldg(pm + r * L);
        VW[idx] = a;
      }
      const int nas = sz.nloc * NS;
      for (int idx = threadIdx.x; idx < NS * nas * kw; idx += blockDim.x) {
        const int ql = c0 + idx % kw, rest = idx / kw, as = rest % nas, rr = rest / nas;
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
      schur_tile_update<D>(T1, VW, nas, kw, L, Sm, n, g.sub_conn + K * sz.nloc, nullptr, 1.0);
      __syncthreads();
    }
  }
  // ---- face sub-elements ----
  for (int f = 0; f < NF; ++f) {
    for (int T = 0; T < sz.n_tri; ++T) {
      for (int c0 = 0; c0 < kf; c0 += kc) {
        const int kw = min(kc, kf - c0);
        for (int idx = threadIdx.x; idx < kw * L; idx += blockDim.x) {
          const int j = idx % L, ql = c0 + idx / L, l = ql % D, q = ql / D;
          const double* pm = g.pm_face + ((((size_t)f * sz.n_tri + T) * sz.nqf + q) * D) * L + j;
          double a = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) a += __ldg(ij + r * D + l) * __ldg(pm + r * L);
          VW[idx] = a;
        }
        const int nas = sz.nlocf * NS;
        for (int idx = threadIdx.x; idx < NS * nas * kw; idx += blockDim.x) {
          const int ql = c0 + idx % kw, rest = idx / kw, as = rest % nas, rr = rest / nas;
          const int s = as % NS, a = as / NS, l = ql % D, q = ql / D;
          const double* W = b.wdgdq_face +
                            ((((size_t)mac * NF + f) * sz.n_tri * sz.nqf + T * sz.nqf + q) * D + l) * NS * NS;
          T1[idx] = __ldg(W + s * NS + rr) * __ldg(g.phi_face + q * sz.nlocf + a);
        }
        __syncthreads();
        schur_tile_update<D>(T1, VW, nas, kw, L, Sm, n, g.tri_conn + T * sz.nlocf, g.face_vol_nodes + f * sz.Lf,
                             -1.0);
        __syncthreads();
      }
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


// --------------------------------------------------------------------------
// k_gj3: Gauss-Jordan inverse without physical row interchanges
// --------------------------------------------------------------------------
// 64-column panels in shared memory, 16-column sub-panels, DMMA rank-16 /
// rank-64 updates (mma.sync.m8n8k4.f64); the pivot of logical column k stays in its
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

int g_schur_variant = 0;  // 0: k_schur2 (default), else the per-macro FFMA kernel (A/B knob)
template <int D>
int schur2(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st);

template <int D>
int schur_matrix(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st) {
  constexpr int NS = D + 2;
  const int kv = g.nq * D, kf = g.nqf * D, kmax = kv > kf ? kv : kf;
  const int rmax = (g.nloc > g.nlocf ? g.nloc : g.nlocf) * NS;
  const int n = g.L * NS;
  if (g_schur_variant == 0) {  // stage-pipelined tensor-core kernel (schur.cu) when its stages fit
    const int rc = schur2<D>(g, b, S, st);
    if (rc >= 0) return rc;
  }
  // k chunk: the whole sub-element when it fits, else the largest that does
  int kc = kmax;
  auto bytes_of = [&](int k) { return sizeof(double) * ((size_t)NS * rmax * k + (size_t)k * g.L); };
  while (kc > 1 && bytes_of(kc) > 227 * 1024) --kc;
  const size_t bytes = bytes_of(kc);
  if (bytes > 227 * 1024) return MHDG_ERR_CONFIG;
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_schur<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_schur<D><<<g.n_mac, SCHUR_THREADS, bytes, st>>>(g, b, S, kc);
  return launch_ok();
}

template int schur_matrix<2>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template int schur_matrix<3>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);

}  // namespace mhdg
