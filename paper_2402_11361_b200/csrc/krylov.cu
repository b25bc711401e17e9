// Krylov vector kernels (krylov.py:51-191 of the reference), any n, deterministic.
//
// One streaming pass over a block of basis rows V_rows (row stride ldv) and a
// vector w does, by mode:
//   0  dots:          out[i] = V_i . w                       (h = V_j w)
//   1  update + dots: w -= sum_i coef_i V_i, then out[i] = V_i . w
//   2  update + norm: w -= sum_i coef_i V_i, then out[0] = w . w
//   3  combine:       w += sum_i coef_i V_i                  (x += V^T y, Z^T y)
//   4  norm:          out[0] = w . w
// Every CTA owns a contiguous slice of the vector (E elements per thread,
// coalesced), keeps its slice of w in registers between the update and the
// dots (the V rows it re-reads for the dots were just streamed and hit L2), and
// writes one partial per output; the last CTA to finish (threadfence + ticket)
// sums the partials in a fixed tree (lane-strided, then a butterfly), so the
// result depends only on n, never on scheduling.  ICGS (krylov.py:51-58) is
// three passes -- dots; update + dots; update + norm -- the last one's final
// CTA also forming h = h1 + h2 and ||w||: three launches per Arnoldi step and
// V_j streamed three times from HBM (cuBLAS GEMV + norm: four, plus launches).
#include "common.cuh"

namespace mhdg {

constexpr int KV_T = 256;   // threads per CTA
constexpr int KV_E = 4;     // elements per thread
constexpr int KV_SL = KV_T * KV_E;
constexpr int KV_R = 8;     // dot rows per register chunk
constexpr int KV_MAXR = 64; // outputs per pass

static inline int kv_blocks(long long n) {
  const long long nb = (n + KV_SL - 1) / KV_SL;
  return nb < 1 ? 1 : (int)nb;
}

// scratch layout (doubles): [partials nb x 64][h1 64][h2 64][ticket]
struct KvScratch {
  double* partial;
  double* h1;
  double* h2;
  unsigned* ticket;
  __host__ __device__ KvScratch(double* s, int nb) {
    partial = s;
    h1 = s + (size_t)nb * KV_MAXR;
    h2 = h1 + KV_MAXR;
    ticket = reinterpret_cast<unsigned*>(h2 + KV_MAXR);
  }
};

// fixed-order sum of partial[b][i] over b: lane-strided sums, then an xor butterfly
__device__ __forceinline__ double kv_sum_partials(const double* partial, int nb, int i, int lane) {
  double v = 0.0;
  for (int b = lane; b < nb; b += 32) v += __ldcg(partial + (size_t)b * KV_MAXR + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MHDG_FULL, v, o);
  return v;
}

// fin (ICGS pass 3 of mhdg_icgs): dst[0..rows) = h1 + h2, dst[rows] = sqrt(w . w)
template <int MODE>
__global__ void __launch_bounds__(KV_T) k_vec_pass(long long n, int rows, const double* __restrict__ V, long long ldv,
                                                   double* __restrict__ w, const double* __restrict__ coef,
                                                   double* __restrict__ scratch, double* __restrict__ dst, int fin) {
  __shared__ double red[KV_T / 32][KV_R];
  __shared__ double cs[KV_MAXR];
  __shared__ bool last;
  constexpr bool UPD = MODE == 1 || MODE == 2 || MODE == 3;
  constexpr bool DOTS = MODE == 0 || MODE == 1;
  constexpr bool NORM = MODE == 2 || MODE == 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nb = gridDim.x;
  const KvScratch sc(scratch, nb);
  const long long base = (long long)blockIdx.x * KV_SL + tid;
  if (UPD)  // coefficients, zero-padded to a multiple of KV_R rows
    for (int i = tid; i < KV_MAXR; i += KV_T) cs[i] = i < rows ? coef[i] : 0.0;
  double wr[KV_E];
  bool ok[KV_E];
#pragma unroll
  for (int k = 0; k < KV_E; ++k) {
    const long long t = base + (long long)k * KV_T;
    ok[k] = t < n;
    wr[k] = ok[k] ? w[t] : 0.0;
  }
  if (UPD) {
    __syncthreads();
    double s[KV_E];
#pragma unroll
    for (int k = 0; k < KV_E; ++k) s[k] = 0.0;
    for (int i0 = 0; i0 < rows; i0 += KV_R) {  // KV_R rows of loads in flight, then the FMAs in row order
      double vv[KV_R][KV_E];
#pragma unroll
      for (int r = 0; r < KV_R; ++r) {
        const double* vr = V + (long long)(i0 + r) * ldv + base;
#pragma unroll
        for (int k = 0; k < KV_E; ++k) vv[r][k] = (i0 + r < rows && ok[k]) ? vr[(long long)k * KV_T] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < KV_R; ++r)
#pragma unroll
        for (int k = 0; k < KV_E; ++k) s[k] += cs[i0 + r] * vv[r][k];
    }
#pragma unroll
    for (int k = 0; k < KV_E; ++k) {
      wr[k] = MODE == 3 ? wr[k] + s[k] : wr[k] - s[k];
      if (ok[k]) w[base + (long long)k * KV_T] = wr[k];
    }
  }
  if (MODE == 3) return;
  const int nout = DOTS ? rows : 1;
  for (int r0 = 0; r0 < nout; r0 += KV_R) {
    double acc[KV_R];
#pragma unroll
    for (int r = 0; r < KV_R; ++r) acc[r] = 0.0;
    if (NORM) {
#pragma unroll
      for (int k = 0; k < KV_E; ++k) acc[0] += wr[k] * wr[k];
    } else {
#pragma unroll
      for (int r = 0; r < KV_R; ++r) {
        if (r0 + r >= rows) break;
        const double* vr = V + (long long)(r0 + r) * ldv + base;
#pragma unroll
        for (int k = 0; k < KV_E; ++k)
          if (ok[k]) acc[r] += vr[(long long)k * KV_T] * wr[k];
      }
    }
#pragma unroll
    for (int r = 0; r < KV_R; ++r) {
      double v = acc[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MHDG_FULL, v, o);
      if (lane == 0) red[warp][r] = v;
    }
    __syncthreads();
    if (tid < KV_R && r0 + tid < nout) {
      double v = 0.0;
#pragma unroll
      for (int wi = 0; wi < KV_T / 32; ++wi) v += red[wi][tid];
      sc.partial[(size_t)blockIdx.x * KV_MAXR + r0 + tid] = v;
    }
    __syncthreads();
  }
  // the last CTA reduces the partials (fixed order) and re-arms the ticket
  __threadfence();
  if (tid == 0) last = atomicAdd(sc.ticket, 1u) == (unsigned)(nb - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = warp; i < nout; i += KV_T / 32) {
    const double v = kv_sum_partials(sc.partial, nb, i, lane);
    if (lane == 0) {
      if (fin && NORM) {
        dst[rows] = sqrt(v);
      } else {
        dst[i] = v;
      }
    }
  }
  if (fin && NORM)
    for (int i = tid; i < rows; i += KV_T) dst[i] = sc.h1[i] + sc.h2[i];
  if (tid == 0) *sc.ticket = 0u;
}

static int vec_pass(long long n, int rows, const double* V, long long ldv, double* w, const double* coef, int mode,
                    double* out, double* scratch, int fin, cudaStream_t st) {
  if (rows < 0 || rows > KV_MAXR || n < 0) return MHDG_ERR_CONFIG;
  if (n == 0) return MHDG_OK;
  const int nb = kv_blocks(n);
  switch (mode) {
    case 0: k_vec_pass<0><<<nb, KV_T, 0, st>>>(n, rows, V, ldv, w, coef, scratch, out, fin); break;
    case 1: k_vec_pass<1><<<nb, KV_T, 0, st>>>(n, rows, V, ldv, w, coef, scratch, out, fin); break;
    case 2: k_vec_pass<2><<<nb, KV_T, 0, st>>>(n, rows, V, ldv, w, coef, scratch, out, fin); break;
    case 3: k_vec_pass<3><<<nb, KV_T, 0, st>>>(n, rows, V, ldv, w, coef, scratch, out, fin); break;
    case 4: k_vec_pass<4><<<nb, KV_T, 0, st>>>(n, 0, V, ldv, w, coef, scratch, out, fin); break;
    default: return MHDG_ERR_CONFIG;
  }
  return launch_ok();
}

int vec_pass_api(long long n, int rows, const double* V, long long ldv, double* w, const double* coef, int mode,
                 double* out, double* scratch, cudaStream_t st) {
  return vec_pass(n, rows, V, ldv, w, coef, mode, out, scratch, 0, st);
}

int icgs(int n, int j, const double* V, long long ldv, double* w, double* out, double* scratch, cudaStream_t st) {
  const int rows = j + 1;
  if (rows > KV_MAXR - 1) return MHDG_ERR_CONFIG;
  const KvScratch sc(scratch, kv_blocks(n));
  tl_begin(TL_KRYLOV, st);
  int rc = vec_pass(n, rows, V, ldv, w, nullptr, 0, sc.h1, scratch, 0, st);  // h1 = V_j w
  if (!rc) rc = vec_pass(n, rows, V, ldv, w, sc.h1, 1, sc.h2, scratch, 0, st);  // w -= V_j^T h1; h2 = V_j w
  if (!rc) rc = vec_pass(n, rows, V, ldv, w, sc.h2, 2, out, scratch, 1, st);  // w -= V_j^T h2; h, ||w||
  tl_end(TL_KRYLOV, st);
  return rc;
}

long long icgs_scratch_size(int n) { return (long long)kv_blocks(n) * KV_MAXR + 2 * KV_MAXR + 2; }

}  // namespace mhdg
