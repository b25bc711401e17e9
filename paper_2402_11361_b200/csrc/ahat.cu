// Stored local trace operators (the B_A representation of SURVEY §8d / §8f rank 2).
//
// The reference keeps S^-1 and the couplings and applies the condensed operator
// matrix-free (CondensedSchur.apply_trace, condense.py:91-103); its own test
// oracle `dense_trace_operator` (condense.py:269) assembles the same operator
// from the per-macro dense blocks A^{T_i}.  Here those per-macro blocks are
// formed on the device once per condensation and the apply becomes one batched
// GEMV over them plus the usual face reduction:
//   * form: column k of every macro's A^{T_i} is the local apply of the unit
//     trace e_k -- the streamed apply kernels run with an identity gather over a
//     local trace vector, ltr passes -- and is stored column-major per macro
//     (A^T[m][k][t]), one contiguous row per pass;
//   * apply: one CTA per macro, the gathered x_loc in shared memory, thread t
//     owns output row t and walks the columns k with coalesced 8-byte loads
//     (a warp reads 256 contiguous bytes per column), eight loads in flight per
//     thread, partial sums in a fixed order (deterministic).
// HBM bytes per macro-apply: 8 ltr^2 + 12 ltr (B_A = 195 KB at C2, 7.2x fewer
// than B_ref).
#include "common.cuh"

namespace mhdg {

int face_reduce(const mhdg_disc& g, const double* y_loc, const double* add, double add_sign, double* y,
                cudaStream_t st);

__global__ void k_unit_trace(long long total, int ltr, int k, double* __restrict__ x_loc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    x_loc[i] = (i % ltr) == k ? 1.0 : 0.0;
}

__global__ void k_ident(long long total, int* __restrict__ ident) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    ident[i] = (int)i;
}

// A^T[m][k][:] = y_loc[m][:]
__global__ void k_store_col(int n_mac, int ltr, int k, const double* __restrict__ y_loc, double* __restrict__ at) {
  const long long total = (long long)n_mac * ltr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / ltr, t = i - m * ltr;
    at[(m * ltr + k) * ltr + t] = y_loc[i];
  }
}

constexpr int AH_U = 8;  // column loads in flight per thread

__global__ void __launch_bounds__(512) k_ahat_gemv(int n_mac, int ltr, const double* __restrict__ at,
                                                   const int* __restrict__ gather, const double* __restrict__ x,
                                                   double* __restrict__ y_loc) {
  extern __shared__ double xs[];
  const int m = blockIdx.x;
  for (int k = threadIdx.x; k < ltr; k += blockDim.x) xs[k] = __ldg(x + __ldg(gather + (size_t)m * ltr + k));
  __syncthreads();
  const double* a = at + (size_t)m * ltr * ltr;
  for (int t = threadIdx.x; t < ltr; t += blockDim.x) {
    double acc[AH_U];
#pragma unroll
    for (int u = 0; u < AH_U; ++u) acc[u] = 0.0;
    int k = 0;
    for (; k + AH_U <= ltr; k += AH_U) {
      double v[AH_U];
#pragma unroll
      for (int u = 0; u < AH_U; ++u) v[u] = __ldcs(a + (size_t)(k + u) * ltr + t);
#pragma unroll
      for (int u = 0; u < AH_U; ++u) acc[u] += v[u] * xs[k + u];
    }
    for (; k < ltr; ++k) acc[0] += __ldcs(a + (size_t)k * ltr + t) * xs[k];
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < AH_U; ++u) s += acc[u];
    y_loc[(size_t)m * ltr + t] = s;
  }
}

static int ahat_threads(int ltr) {
  int t = (ltr + 31) / 32 * 32;
  return t > 512 ? 512 : t;
}

}  // namespace mhdg

using namespace mhdg;

extern "C" {

int mhdg_apply_trace_local(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* x,
                           double* y_loc, void* st);

int mhdg_ahat_form(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, double* at, double* x_loc,
                   double* y_loc, int* ident, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int ltr = g->nf * g->Lf * g->ns;
  const long long total = (long long)g->n_mac * ltr;
  const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  k_ident<<<blocks, 256, 0, st>>>(total, ident);
  if (launch_ok()) return MHDG_ERR_CUDA;
  mhdg_disc gl = *g;  // the same operator over a local trace vector: identity gather
  gl.gather = ident;
  for (int k = 0; k < ltr; ++k) {
    k_unit_trace<<<blocks, 256, 0, st>>>(total, ltr, k, x_loc);
    if (launch_ok()) return MHDG_ERR_CUDA;
    const int rc = mhdg_apply_trace_local(&gl, b, f, x_loc, y_loc, stream);
    if (rc) return rc;
    k_store_col<<<blocks, 256, 0, st>>>(g->n_mac, ltr, k, y_loc, at);
    if (launch_ok()) return MHDG_ERR_CUDA;
  }
  return MHDG_OK;
}

int mhdg_ahat_apply_local(const mhdg_disc* g, const double* at, const double* x, double* y_loc, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int ltr = g->nf * g->Lf * g->ns;
  const size_t smem = sizeof(double) * (size_t)ltr;
  if (smem > 48 * 1024) return MHDG_ERR_CONFIG;
  tl_begin(TL_APPLY_AHAT, st);
  k_ahat_gemv<<<g->n_mac, ahat_threads(ltr), smem, st>>>(g->n_mac, ltr, at, g->gather, x, y_loc);
  tl_end(TL_APPLY_AHAT, st);
  return launch_ok();
}

int mhdg_ahat_apply(const mhdg_disc* g, const double* at, const double* x, double* y, double* y_loc, void* stream) {
  const int rc = mhdg_ahat_apply_local(g, at, x, y_loc, stream);
  if (rc) return rc;
  tl_begin(TL_FACE_REDUCE, (cudaStream_t)stream);
  const int rc2 = face_reduce(*g, y_loc, nullptr, 0.0, y, (cudaStream_t)stream);
  tl_end(TL_FACE_REDUCE, (cudaStream_t)stream);
  return rc2;
}

}  // extern "C"
