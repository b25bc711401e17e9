// Batched LU with partial pivoting of the condensed local systems S
// (the factorisation the paper's Remark asks for; the
// reference's np.linalg.inv at condense.py:62-70 is getrf + getri, and the
// canonical F_cond of SURVEY 8d counts this getrf part, (2/3) n^3).
//
// k_lu4: one CTA per macro, two CTAs per SM so one macro's pivot chain runs
// under the other's tensor-core updates.  Right-looking, 32-column panels:
//   * the panel (all not-yet-pivoted rows x 32 columns) sits in shared memory
//     (XOR-swizzled rows, conflict-free both row-per-thread and as DMMA
//     A fragments);
//   * it is factored in 16-column sub-panels held in registers, one row per
//     thread: a pivot step is one warp argmax (value and row packed into one
//     64-bit key), one CTA barrier, and register-only row updates; each
//     warp's candidate row is published with its key, so no second barrier
//     is needed to broadcast the pivot row;
//   * between the two sub-panels: a 16-step triangular solve for the pivot
//     rows and a DMMA rank-16 update of the other rows;
//   * trailing update, one 16-column chunk per warp, no CTA barrier:
//     U12 = inv(L11) A12 on DMMA (inv(L11) formed once per panel), U12
//     turned into B fragments with shuffles, then C -= L21 U12 over all
//     remaining rows with C read-modified-written in global memory (L2).
// Pivots stay in place (logical row k = physical row piv[k]; rows are never
// moved), the output contract of k_lu3: k_pack_lu4 packs it for the apply.
// FactorizationError on an exactly zero pivot (scipy's lu_factor / LAPACK
// getrf report singular U).
#include "common.cuh"
#include "dmma.cuh"
#include "packed_lu.cuh"

namespace mhdg {

#ifdef MHDG_STREAM_PROFILE
__device__ unsigned long long g_lu4prof[8];
#define LUT(v) long long v = clock64()
#define LUADD(k, v) if (threadIdx.x == 0) atomicAdd(&g_lu4prof[k], (unsigned long long)(clock64() - (v)))
extern "C" int mhdg_lu4_profile(unsigned long long* out, int reset) {
  if (out) cudaMemcpyFromSymbol(out, g_lu4prof, sizeof(g_lu4prof));
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_lu4prof, z, sizeof(z));
  }
  return 0;
}
#else
#define LUT(v)
#define LUADD(k, v)
#endif

namespace lu4 {
constexpr int SW = 16;       // register sub-panel width
constexpr int CW = 16;       // trailing-update column chunk per warp
constexpr int SWP = SW + 2;  // candidate slot: SW row values, the reciprocal, padding
// panel row stride for panel width NB (= 4 mod 16): conflict-free DMMA A fragments
template <int NB>
constexpr int pstride() { return NB + 4; }

// argmax key: |v| with the low 10 mantissa bits replaced by (1023 - row), so the
// largest key is the largest magnitude, ties (to 2^-42) going to the lowest row (n <= 1024)
constexpr int MAX_N = 1024;
__device__ __forceinline__ unsigned long long pkey(double v, int r) {
  return ((unsigned long long)__double_as_longlong(fabs(v)) & ~0x3FFull) | (unsigned long long)(1023 - r);
}
__device__ __forceinline__ int key_row(unsigned long long k) { return 1023 - (int)(k & 0x3FFull); }

template <int NB, int NT>
size_t smem_bytes(int n) {
  constexpr int NW = NT / 32;
  return sizeof(double) * ((size_t)n * pstride<NB>() + 2 * NW * SWP) + sizeof(unsigned long long) * 2 * NW +
         sizeof(unsigned short) * 2 * (size_t)n + (size_t)n;
}
}  // namespace lu4

// C -= L21 U12 for one 16-column chunk over the m remaining rows (list rl), 16 rows per
// pass with the next three passes' C in flight.  VEC: 16-byte C accesses (full chunk, even n).
#ifndef MHDG_LU_L2MODE
#define MHDG_LU_L2MODE 2
#endif

template <int NB, bool VEC>
__device__ __forceinline__ void trail_pass_loop(double* __restrict__ A, int n, int c0, int cw, int m,
                                                const unsigned short* rl, const double* P, int t4, int g,
                                                const double (&bf)[NB / 4][2], unsigned long long pol) {
  using namespace lu4;
  constexpr int PS = pstride<NB>();
  const int rlast = rl[m - 1];
  auto load = [&](int t, double (&c)[2][2][2], int (&rr)[2], bool (&ok)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ok[h] = t + 8 * h + g < m;
      rr[h] = ok[h] ? rl[t + 8 * h + g] : rlast;
      const double* src = A + (size_t)rr[h] * n + c0 + 2 * t4;
#pragma unroll
      for (int ct = 0; ct < 2; ++ct) {
        if (VEC) {
          const double2 v = ok[h] ? ld_hint(src + 8 * ct, pol) : make_double2(0.0, 0.0);
          c[h][ct][0] = v.x;
          c[h][ct][1] = v.y;
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) c[h][ct][e] = (ok[h] && 8 * ct + 2 * t4 + e < cw) ? src[8 * ct + e] : 0.0;
        }
      }
    }
  };
  auto pass = [&](double (&c)[2][2][2], const int (&rr)[2], const bool (&ok)[2]) {
    const double* pa0 = P + rr[0] * PS + t4;
    const double* pa1 = P + rr[1] * PS + t4;
#pragma unroll
    for (int ks = 0; ks < NB / 4; ++ks) {
      const double a0 = pa0[4 * ks], a1 = pa1[4 * ks];
#pragma unroll
      for (int ct = 0; ct < 2; ++ct) {
        dmma_8x8x4(c[0][ct][0], c[0][ct][1], a0, bf[ks][ct]);
        dmma_8x8x4(c[1][ct][0], c[1][ct][1], a1, bf[ks][ct]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (ok[h]) {
        double* dst = A + (size_t)rr[h] * n + c0 + 2 * t4;
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) {
          if (VEC) {
            st_hint(dst + 8 * ct, make_double2(c[h][ct][0], c[h][ct][1]), pol);
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (8 * ct + 2 * t4 + e < cw) dst[8 * ct + e] = c[h][ct][e];
          }
        }
      }
  };
  // four register stages: C of the next three passes is in flight during a pass
  double s0[2][2][2], s1[2][2][2], s2[2][2][2], s3[2][2][2];
  int r0[2], r1[2], r2[2], r3[2];
  bool o0[2], o1[2], o2[2], o3[2];
  load(0, s0, r0, o0);
  load(16, s1, r1, o1);
  load(32, s2, r2, o2);
  for (int t = 0; t < m; t += 64) {
    load(t + 48, s3, r3, o3);
    pass(s0, r0, o0);
    if (t + 16 >= m) break;
    load(t + 64, s0, r0, o0);
    pass(s1, r1, o1);
    if (t + 32 >= m) break;
    load(t + 80, s1, r1, o1);
    pass(s2, r2, o2);
    if (t + 48 >= m) break;
    load(t + 96, s2, r2, o2);
    pass(s3, r3, o3);
  }
}

template <int NB, int NT, int RPT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_lu4(int n, double* __restrict__ S, int* __restrict__ piv_out,
                                                  int* status, int l2mode, int n_mac) {
  using namespace lu4;
  constexpr int NW = NT / 32, PS = pstride<NB>(), NH = NB / 32;  // NH: 32-column halves of a panel
  extern __shared__ __align__(16) double sm[];
  double* P = sm;                                   // n x PS: the panel, physical rows
  double* cv = P + (size_t)n * PS;                  // [2][NW][SWP] candidate pivot rows
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(cv + 2 * NW * SWP);  // [2][NW] their keys
  unsigned short* npl = reinterpret_cast<unsigned short*>(ck + 2 * NW);  // [2][n] not-yet-pivoted rows
  unsigned char* rflag = reinterpret_cast<unsigned char*>(npl + 2 * n);   // n: 1 = pivot row
  __shared__ int pv[NB];                            // this panel's pivot rows, logical order
  __shared__ int wcnt[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  // grid = n_mac (one macro per CTA) or persistent (fewer CTAs walk the macros: fewer
  // trailing matrices resident at once, so they stay in L2)
#pragma unroll 1
  for (int mac = blockIdx.x; mac < n_mac; mac += gridDim.x) {
  double* A = S + (size_t)mac * n * n;
  int* pivg = piv_out + (size_t)mac * n;
  bool singular = false;
  for (int i = tid; i < n; i += NT) {
    npl[i] = (unsigned short)i;
    rflag[i] = 0;
  }
  int m = n, lb = 0;
  // L2 priority of the trailing-update C traffic: evict_last on the macros with
  // mac % l2mode != 0 (l2mode >= 2), on all (1) or none (0).  The trailing matrices of all
  // resident macros together are about the L2 size and are swept cyclically, so under LRU
  // every macro's lines get evicted; keeping a fraction of the macros resident recovers
  // their hits.
  // final values (the written-back panel, U12) are not read again by the factorisation:
  // evict_first keeps L2 for the trailing matrices (26.2 -> 26.1 ms on one box)
  const unsigned long long pol_final = l2_policy(2);
  const unsigned long long pol = l2_policy(l2mode == 1 || (l2mode >= 2 && mac % l2mode != 0) ? 1 : 0);
  __syncthreads();

  for (int k0 = 0; k0 < n; k0 += NB) {
    const int nb = min(NB, n - k0);
    const unsigned short* np = npl + lb * n;
    LUT(pt0);
    // ---- panel: the m not-yet-pivoted rows, columns k0 .. k0+nb-1 (zero beyond) ----
    if ((n & 1) == 0) {  // 16-byte copies, two rows per warp pass (rows and k0 even)
      for (int i = 2 * warp + (lane >> 4); i < m; i += 2 * NW) {
        const int r = np[i];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = 32 * h + 2 * (lane & 15);
          cp_async16(P + r * PS + c, A + (size_t)r * n + k0 + (c < nb ? c : 0), c < nb ? 16 : 0);
        }
      }
    } else {
      for (int i = warp; i < m; i += NW) {
        const int r = np[i];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = 32 * h + lane;
          cp_async8(P + r * PS + c, A + (size_t)r * n + k0 + (c < nb ? c : 0), c < nb ? 8 : 0);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
    LUADD(0, pt0);

    for (int js = 0; js < nb; js += SW) {
      LUT(pt1);
      double x[RPT][SW];
      bool act[RPT], act0[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = tid + NT * i;
        act[i] = r < n && !rflag[r];
        act0[i] = act[i];
#pragma unroll
        for (int c = 0; c < SW; c += 2) {  // 16-byte loads (PS and js even)
          const double2 v = act[i] ? *reinterpret_cast<const double2*>(P + r * PS + js + c) : make_double2(0.0, 0.0);
          x[i][c] = v.x;
          x[i][c + 1] = v.y;
        }
      }
#pragma unroll
      for (int jj = 0; jj < SW; ++jj) {
        const int j = js + jj;
        if (j >= nb) break;
        // this thread's best row for column j, and its reciprocal (speculative: only the
        // winner's is used; formed here, off the post-barrier path)
        unsigned long long key = 0;
        double xv = 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (act[i]) {
            const unsigned long long kk = pkey(x[i][jj], tid + NT * i);
            if (kk > key) {
              key = kk;
              xv = x[i][jj];
            }
          }
        const double rcp = 1.0 / xv;
        // warp argmax of the 64-bit key: max of the high words, then of the low words among ties
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mh = __reduce_max_sync(MHDG_FULL, hi);
        const unsigned tie = __ballot_sync(MHDG_FULL, hi == mh);
        unsigned ml = 0;
        if (hi == mh) ml = __reduce_max_sync(tie, lo);
        const int par = j & 1;
        const unsigned win = __ballot_sync(MHDG_FULL, hi == mh && lo == ml);
        if (hi == mh && lo == ml) {  // this lane holds the warp's candidate (or none: key 0)
          double* slot = cv + (par * NW + warp) * SWP;
#pragma unroll
          for (int i = 0; i < RPT; ++i)
            if (act[i] && key_row(key) == tid + NT * i) {
#pragma unroll
              for (int c = jj & ~1; c < SW; c += 2)  // from column jj (the pair's first entry is unused)
                *reinterpret_cast<double2*>(slot + c) = make_double2(x[i][c], x[i][c + 1]);
            }
          slot[SW] = rcp;
          if (lane == __ffs(win) - 1) ck[par * NW + warp] = key;
        }
        __syncthreads();
        // CTA argmax over the warps' keys (broadcast loads); the pivot row's warp follows from
        // its index (row r belongs to thread r mod NT)
        unsigned long long best = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const unsigned long long kk = ck[par * NW + w];
          best = kk > best ? kk : best;
        }
        const int p = key_row(best);
        const double* prow = cv + (par * NW + (p % NT) / 32) * SWP;
        // the pivot row from column jj and its reciprocal in 16-byte loads (slots are 16-byte
        // aligned: SWP and the panel region are even); 26.1 -> 25.6 ms at C2
        double pr[SW + 2];
#pragma unroll
        for (int c = jj & ~1; c < SW + 2; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(prow + c);
          pr[c] = v.x;
          pr[c + 1] = v.y;
        }
        const double pd = pr[jj];
        if (pd == 0.0) singular = true;
        const double d = pd == 0.0 ? 0.0 : pr[SW];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          if (!act[i]) continue;
          if (tid + NT * i == p) {
            act[i] = false;  // the pivot row keeps its values: L left of jj, U from jj on
            continue;
          }
          const double l = x[i][jj] * d;
          x[i][jj] = l;
#pragma unroll
          for (int c = jj + 1; c < SW; ++c) x[i][c] -= l * pr[c];
        }
        if (tid == 0) {
          pv[j] = p;
          pivg[k0 + j] = p;
          rflag[p] = 1;
        }
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (act0[i]) {
          const int r = tid + NT * i;
#pragma unroll
          for (int c = 0; c < SW; c += 2)
            *reinterpret_cast<double2*>(P + r * PS + js + c) = make_double2(x[i][c], x[i][c + 1]);
        }
      __syncthreads();
      LUADD(1, pt1);
      LUT(pt2);
      if (js + SW < nb) {
        // (a) U rows of this sub-panel's pivots on the panel's remaining columns
        if (warp == 0) {
          for (int c = js + SW + lane; c < nb; c += 32) {
            double u[SW];
#pragma unroll
            for (int jj = 0; jj < SW; ++jj) {
              const double* pr = P + pv[js + jj] * PS;
              double v = pr[c];
#pragma unroll
              for (int i = 0; i < jj; ++i) v -= pr[js + i] * u[i];
              u[jj] = v;
              P[pv[js + jj] * PS + c] = v;
            }
          }
        }
        __syncthreads();
        // (b) rank-SW DMMA update of the other rows on columns js+SW .. NB-1, 16 at a time
        for (int cg = js + SW; cg < NB; cg += 16) {
          double bf[SW / 4][2];
#pragma unroll
          for (int ks = 0; ks < SW / 4; ++ks)
#pragma unroll
            for (int ct = 0; ct < 2; ++ct) bf[ks][ct] = -P[pv[js + 4 * ks + t4] * PS + cg + 8 * ct + g];
          for (int t = warp * 8; t < m; t += NW * 8) {
            const bool ok = t + g < m;
            const int r = np[ok ? t + g : 0];
            const bool st = ok && !rflag[r];
            double* pr = P + r * PS;
            double c[2][2];
#pragma unroll
            for (int ct = 0; ct < 2; ++ct) {
              const double2 v = *reinterpret_cast<const double2*>(pr + cg + 8 * ct + 2 * t4);
              c[ct][0] = v.x;
              c[ct][1] = v.y;
            }
#pragma unroll
            for (int ks = 0; ks < SW / 4; ++ks) {
              const double a = pr[js + 4 * ks + t4];
#pragma unroll
              for (int ct = 0; ct < 2; ++ct) dmma_8x8x4(c[ct][0], c[ct][1], a, bf[ks][ct]);
            }
            if (st) {
#pragma unroll
              for (int ct = 0; ct < 2; ++ct)
                *reinterpret_cast<double2*>(pr + cg + 8 * ct + 2 * t4) = make_double2(c[ct][0], c[ct][1]);
            }
          }
        }
        __syncthreads();
      }
      LUADD(2, pt2);
    }

    LUT(pt3);
    // ---- write the factored panel back; list of the rows still unpivoted; inv(L11) ----
#pragma unroll 4
    if ((n & 1) == 0) {  // 16-byte stores, two rows per warp pass
      for (int i = 2 * warp + (lane >> 4); i < m; i += 2 * NW) {
        const int r = np[i];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = 32 * h + 2 * (lane & 15);
          if (c < nb)
            st_hint(A + (size_t)r * n + k0 + c, *reinterpret_cast<const double2*>(P + r * PS + c), pol_final);
        }
      }
    } else {
      for (int i = warp; i < m; i += NW) {
        const int r = np[i];
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (32 * h + lane < nb) st_hint1(A + (size_t)r * n + k0 + 32 * h + lane, P[r * PS + 32 * h + lane], pol_final);
      }
    }
    unsigned short* np2 = npl + (lb ^ 1) * n;
    {
      int done_cnt = 0;
      for (int base = 0; base < m; base += NT) {
        const int i = base + tid;
        const bool keep = i < m && !rflag[np[i]];
        const unsigned bal = __ballot_sync(MHDG_FULL, keep);
        if (lane == 0) wcnt[warp] = __popc(bal);
        __syncthreads();
        int off = done_cnt, tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int cw = wcnt[w];
          off += w < warp ? cw : 0;
          tot += cw;
        }
        if (keep) np2[off + __popc(bal & ((1u << lane) - 1u))] = np[i];
        done_cnt += tot;
        __syncthreads();
      }
    }
    {
      // inv(L11): warp w forms columns w, w + NW, ... (lane = rows lane + 32 h), then, once
      // every warp has read L11, stores them over the pivot rows of the panel (written back)
      constexpr int CPW = (NB + NW - 1) / NW;
      double xc[CPW][NH];
#pragma unroll
      for (int cc = 0; cc < CPW; ++cc)
#pragma unroll
        for (int h = 0; h < NH; ++h) xc[cc][h] = (32 * h + lane == warp + NW * cc && 32 * h + lane < nb) ? 1.0 : 0.0;
      int prl[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) prl[h] = 32 * h + lane < nb ? pv[32 * h + lane] : 0;
      for (int k = 0; k < nb - 1; ++k) {
        double lik[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int row = 32 * h + lane;
          lik[h] = (row > k && row < nb) ? P[prl[h] * PS + k] : 0.0;
        }
#pragma unroll
        for (int cc = 0; cc < CPW; ++cc) {
          double src = xc[cc][0];
#pragma unroll
          for (int h = 1; h < NH; ++h) src = (k >> 5) == h ? xc[cc][h] : src;
          const double xk = __shfl_sync(MHDG_FULL, src, k & 31);
#pragma unroll
          for (int h = 0; h < NH; ++h) xc[cc][h] -= lik[h] * xk;
        }
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < NH; ++h)
        if (32 * h + lane < nb) {
#pragma unroll
          for (int cc = 0; cc < CPW; ++cc)
            if (warp + NW * cc < NB) P[prl[h] * PS + warp + NW * cc] = xc[cc][h];
        }
    }
    m -= nb;
    lb ^= 1;
    __syncthreads();
    LUADD(3, pt3);
    LUT(pt4);

    // ---- trailing update, one CW-column chunk per warp (no CTA barrier) ----
    const int ct0 = k0 + nb;
    const int nchunks = (n - ct0 + CW - 1) / CW;
    const double* Lirow[NB / 8];  // inv(L11) row 8 rt + g lives in pivot row pv[8 rt + g]
#pragma unroll
    for (int rt = 0; rt < NB / 8; ++rt) Lirow[rt] = P + pv[8 * rt + g] * PS + t4;
    // Units of work: one chunk per warp, except that the r = nchunks mod NW chunks of the
    // last round are split by rows over NW / r warps each (when that is >= 2), so the
    // warps finish together.  The parts of a split chunk read A12 before a named barrier
    // (ids 1..r); only part 0 then overwrites it with U12.
    const int rlast = nchunks % NW, nparts = rlast > 0 ? NW / rlast : 1;
    const int nfull = nparts >= 2 ? nchunks - rlast : nchunks;
    const int nunits = nfull + (nparts >= 2 ? rlast * nparts : 0);
    for (int un = warp; un < nunits; un += NW) {
      int q = un, part = 0, np_ = 1;
      if (un >= nfull) {
        const int v = un - nfull;
        q = nfull + v / nparts;
        part = v % nparts;
        np_ = nparts;
      }
      const int c0 = ct0 + q * CW, cw = min(CW, n - c0);
      // U12 chunk = inv(L11) A12 (A12 = this panel's pivot rows; nb = NB whenever columns remain)
      double u[NB / 8][2][2];
#pragma unroll
      for (int rt = 0; rt < NB / 8; ++rt)
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) u[rt][ct][0] = u[rt][ct][1] = 0.0;
      {
        double b[NB / 4][2];
#pragma unroll
        for (int ks = 0; ks < NB / 4; ++ks) {
          const double* src = A + (size_t)pv[4 * ks + t4] * n + c0;
#pragma unroll
          for (int ct = 0; ct < 2; ++ct) b[ks][ct] = 8 * ct + g < cw ? src[8 * ct + g] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < NB / 4; ++ks)
#pragma unroll
          for (int rt = 0; rt < NB / 8; ++rt) {
            const double a = Lirow[rt][4 * ks];
#pragma unroll
            for (int ct = 0; ct < 2; ++ct) dmma_8x8x4(u[rt][ct][0], u[rt][ct][1], a, b[ks][ct]);
          }
      }
      __syncwarp();
      if (np_ > 1)  // every part has read A12
        asm volatile("bar.sync %0, %1;" ::"r"(1 + q - nfull), "r"(32 * np_) : "memory");
#pragma unroll
      for (int rt = 0; rt < NB / 8; ++rt) {
        if (part != 0) break;
        double* dst = A + (size_t)pv[8 * rt + g] * n + c0;
#pragma unroll
        for (int ct = 0; ct < 2; ++ct)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * ct + 2 * t4 + e < cw) st_hint1(dst + 8 * ct + 2 * t4 + e, u[rt][ct][e], pol_final);
      }
      // -U12 as B fragments: bf[ks][ct] = -U[4 ks + t4][8 ct + g]
      double bf[NB / 4][2];
      {
        const int src_hi = g >> 1;
#pragma unroll
        for (int ks = 0; ks < NB / 4; ++ks) {
          const int src = (4 * (ks & 1) + t4) * 4 + src_hi;
#pragma unroll
          for (int ct = 0; ct < 2; ++ct) {
            const double v0 = __shfl_sync(MHDG_FULL, u[ks >> 1][ct][0], src);
            const double v1 = __shfl_sync(MHDG_FULL, u[ks >> 1][ct][1], src);
            bf[ks][ct] = -((g & 1) ? v1 : v0);
          }
        }
      }
      // C -= L21 U12 over the remaining rows, 16 rows per pass, next pass's C prefetched
      const int npass = (m + 15) / 16, pb = npass * part / np_, pe = npass * (part + 1) / np_;
      const int mb = 16 * pb, mp = min(m, 16 * pe) - mb;  // this part's rows of the list
      if (mp > 0) {
        if (cw == CW && (n & 1) == 0)
          trail_pass_loop<NB, true>(A, n, c0, cw, mp, np2 + mb, P, t4, g, bf, pol);
        else
          trail_pass_loop<NB, false>(A, n, c0, cw, mp, np2 + mb, P, t4, g, bf, pol);
      }
    }
    LUADD(4, pt4);
    LUT(pt5);
    __syncthreads();
    LUADD(5, pt5);
  }
  if (singular && tid == 0) set_status(status, MHDG_ERR_FACTORIZATION, mac, 0, 0.0);
  __syncthreads();  // the next macro reuses the shared panel and row lists
  }
}

// --------------------------------------------------------------------------
// k_pack_lu4: in-place LU (pivot rows in place) -> the packed solve layout of
// packed_lu.cuh.  One CTA per macro; per 64-row block, every 32-column
// segment of the block's rows is staged in shared memory with coalesced reads
// of the physical rows (the next segment's reads in flight while this one is
// written) and written column-major with coalesced writes: panel tiles, the
// strict lower part of the diagonal block (L_bb) and its upper part (U_bb,
// diagonal stored as 1/U_kk).
// --------------------------------------------------------------------------
namespace pk4 {
constexpr int NT = 256, TS = 33, RPW = PLU_NB / (NT / 32);
}

__global__ void __launch_bounds__(pk4::NT) k_pack_lu4(int n, const double* __restrict__ F,
                                                      const int* __restrict__ piv, double* __restrict__ out) {
  using namespace pk4;
  __shared__ double X[PLU_NB * TS];  // one 64 x 32 segment
  extern __shared__ int pr[];         // n pivot rows
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* A = F + (size_t)mac * n * n;
  double* O = out + (size_t)mac * plu_size(n);
  for (int i = tid; i < n; i += NT) pr[i] = piv[(size_t)mac * n + i];
  __syncthreads();
  const int nblk = plu_nblk(n), nseg = (n + PLU_TW - 1) / PLU_TW;
  const int r = tid & (PLU_NB - 1), grp = tid / PLU_NB;
  constexpr int NG = NT / PLU_NB;
  for (int b = 0; b < nblk; ++b) {
    const PluOffsets o = plu_offsets(n, b);
    const int nb = o.nb, r0 = o.r0;
    double v[RPW];
    auto load = [&](int col) {
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const int rr = warp + (NT / 32) * k;
        v[k] = (rr < nb && col + lane < n) ? A[(size_t)pr[r0 + rr] * n + col + lane] : 0.0;
      }
    };
    load(0);
    for (int sg = 0; sg < nseg; ++sg) {
      const int col = sg * PLU_TW;
      __syncthreads();  // previous segment written out
#pragma unroll
      for (int k = 0; k < RPW; ++k) X[(warp + (NT / 32) * k) * TS + lane] = v[k];
      if (sg + 1 < nseg) load(col + PLU_TW);
      __syncthreads();
      const int w = min(PLU_TW, n - col);
      if (col >= r0 && col < r0 + nb) {  // diagonal block columns
        for (int cc = grp; cc < w && col + cc < r0 + nb; cc += NG) {
          const int c = col - r0 + cc;
          if (r < nb && r > c) O[o.fwd_diag + plu_lo(nb, r, c)] = X[r * TS + cc];
          if (r <= c) O[o.bwd_diag + plu_up(r, c)] = r == c ? 1.0 / X[r * TS + cc] : X[r * TS + cc];
        }
      } else {
        double* dst = col < r0 ? O + o.fwd_panel + (long long)col * nb : O + o.bwd_panel + (long long)(col - r0 - nb) * nb;
        for (int cc = grp; cc < w; cc += NG)
          if (r < nb) dst[cc * nb + r] = X[r * TS + cc];
      }
    }
    if (tid == 0) {  // zero the even-size padding of the last (narrow) tiles and triangles
      if ((nb * (nb - 1) / 2) & 1) O[o.fwd_diag + nb * (nb - 1) / 2] = 0.0;
      if ((nb * (nb + 1) / 2) & 1) O[o.bwd_diag + nb * (nb + 1) / 2] = 0.0;
      const int wf = o.ncol_fwd % PLU_TW, wb = o.ncol_bwd % PLU_TW;
      if ((nb * wf) & 1) O[o.fwd_diag - 1] = 0.0;
      if ((nb * wb) & 1) O[o.bwd_diag - 1] = 0.0;
    }
  }
}

int pack_lu4(int n, int n_mac, const double* scratch, const int* piv, double* packed, cudaStream_t st) {
  const size_t bytes = sizeof(int) * n;
  tl_begin(TL_PACK, st);
  k_pack_lu4<<<n_mac, pk4::NT, bytes, st>>>(n, scratch, piv, packed);
  tl_end(TL_PACK, st);
  return launch_ok();
}



static int g_lu_nb = 32, g_lu_nt = 0, g_lu_l2mode = MHDG_LU_L2MODE, g_lu_grid = 0;
extern "C" void mhdg_set_lu_l2mode(int m) { g_lu_l2mode = m; }
extern "C" void mhdg_set_lu_grid(int ctas) { g_lu_grid = ctas; }
static inline int lu_grid(int n_mac) { return g_lu_grid > 0 && g_lu_grid < n_mac ? g_lu_grid : n_mac; }
// n <= 192 (C3's n = 175 and the smaller C5 combos): CTAs of 32 / 64 / 96 threads (n <= 64 /
// 128 / 192), two rows per thread, 8 / 6 / 4 CTAs per SM -- the factorisation is bound by each
// macro's pivot chain, so more macros in flight per SM (C3: 15.6 -> 13.5 ms; A/B knob)
static int g_lu_small = 2;
extern "C" void mhdg_set_lu_small(int on) { g_lu_small = on; }
extern "C" void mhdg_set_lu_panel(int nb, int threads) {
  g_lu_nb = nb == 64 ? 64 : 32;
  g_lu_nt = threads;
}

template <int NB, int NT, int MINB, int MAXRPT = 2>
static int launch_lu4(int n, int n_mac, double* scratch, int* piv, int* status, cudaStream_t st) {
  if (n > MAXRPT * NT) return -1;
  const size_t bytes = lu4::smem_bytes<NB, NT>(n);
  if (bytes > 227 * 1024) return -1;
  auto kern = n <= NT ? k_lu4<NB, NT, 1, MINB> : n <= 2 * NT || MAXRPT < 3 ? k_lu4<NB, NT, 2, MINB>
                                                                           : k_lu4<NB, NT, MAXRPT, MINB>;
  if (MINB > 1 && MINB * (bytes + 1024) > 228 * 1024) return -1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  tl_begin(TL_FACTOR, st);
  kern<<<lu_grid(n_mac), NT, bytes, st>>>(n, scratch, piv, status, g_lu_l2mode, n_mac);
  tl_end(TL_FACTOR, st);
  return 0;
}

// n > 384 (C5 (m, p) = (2, 3): n = 420): three rows per thread, one CTA per SM (the
// 32-column panel of n rows no longer fits twice into shared memory)
template <int NB, int NT>
static int launch_lu4_large(int n, int n_mac, double* scratch, int* piv, int* status, cudaStream_t st) {
  if (n > 3 * NT || n > lu4::MAX_N) return -1;
  const size_t bytes = lu4::smem_bytes<NB, NT>(n);
  if (bytes > 227 * 1024) return -1;
  auto kern = k_lu4<NB, NT, 3, 1>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  tl_begin(TL_FACTOR, st);
  kern<<<lu_grid(n_mac), NT, bytes, st>>>(n, scratch, piv, status, g_lu_l2mode, n_mac);
  tl_end(TL_FACTOR, st);
  return 0;
}

int lu_max_n() { return 3 * 192; }

int lu_factor4(int n, int n_mac, double* scratch, int* piv, double* packed, int* status, cudaStream_t st) {
  // 32-column panels, two CTAs per SM (one's pivot chain under the other's updates), or
  // 64-column panels, one CTA per SM (half the trailing-update traffic)
#ifndef MHDG_LU4_NT
#define MHDG_LU4_NT 192
#endif
  int rc0 = -1;
  if (g_lu_small && g_lu_nb != 64) {  // smaller CTAs, more macros per SM, while 2 rows per thread cover n
    if (n <= 64) rc0 = launch_lu4<32, 32, 8>(n, n_mac, scratch, piv, status, st);
    else if (n <= 128) rc0 = launch_lu4<32, 64, 6>(n, n_mac, scratch, piv, status, st);
    else if (n <= 192)
      rc0 = g_lu_small == 2 ? launch_lu4<32, 64, 4, 3>(n, n_mac, scratch, piv, status, st)
                            : launch_lu4<32, 96, 4>(n, n_mac, scratch, piv, status, st);
  }
  if (rc0 < 0)
    rc0 = g_lu_nb != 64   ? launch_lu4<32, MHDG_LU4_NT, 2>(n, n_mac, scratch, piv, status, st)
          : g_lu_nt == 384 ? launch_lu4<64, 384, 1>(n, n_mac, scratch, piv, status, st)
                           : launch_lu4<64, 256, 1>(n, n_mac, scratch, piv, status, st);
  if (rc0 < 0) rc0 = launch_lu4_large<32, 192>(n, n_mac, scratch, piv, status, st);
  if (rc0 < 0) return -1;
  int rc = launch_ok();
  if (rc) return rc;
  return pack_lu4(n, n_mac, scratch, piv, packed, st);
}

}  // namespace mhdg
