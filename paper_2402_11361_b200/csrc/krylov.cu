// Fused ICGS for the Arnoldi step (krylov.py:51-58 of the reference):
//   h = V_j w; w -= V_j^T h; h2 = V_j w; w -= V_j^T h2; h += h2; hv = ||w||.
// Three passes over V_j instead of four-plus separate GEMV/norm launches: the
// update of each pass is fused with the dots (or norm) of the next, block
// partials are summed in a fixed order by a one-block reduce kernel, so the
// result is deterministic.  out[0..j] = h, out[j+1] = hv.
#include "common.cuh"

namespace mhdg {

constexpr int ICGS_T = 256;
constexpr int ICGS_R = 8;  // V rows per register chunk

// pass 1 (coef == nullptr): partial[b][i] = sum_t V[i][t] w[t]
// pass 2/3: w[t] -= sum_i coef[i] V[i][t], then partial[b][i] = sum_t V[i][t] w_new[t]
//           (pass 3, norm_only: partial[b][0] = sum_t w_new[t]^2)
__global__ void __launch_bounds__(ICGS_T) k_icgs_pass(int n, int rows, const double* __restrict__ V, long long ldv,
                                                      double* __restrict__ w, const double* __restrict__ coef,
                                                      int norm_only, double* __restrict__ partial) {
  __shared__ double red[ICGS_T / 32][ICGS_R];
  __shared__ double cs[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t0 = (long long)blockIdx.x * blockDim.x + tid, stride = (long long)gridDim.x * blockDim.x;
  if (coef)
    for (int i = tid; i < rows; i += blockDim.x) cs[i] = coef[i];
  __syncthreads();
  if (coef) {
    for (long long t = t0; t < n; t += stride) {
      double a = w[t];
      for (int i = 0; i < rows; ++i) a -= cs[i] * V[i * ldv + t];
      w[t] = a;
    }
  }
  const int nout = norm_only ? 1 : rows;
  for (int r0 = 0; r0 < nout; r0 += ICGS_R) {
    double acc[ICGS_R];
#pragma unroll
    for (int k = 0; k < ICGS_R; ++k) acc[k] = 0.0;
    for (long long t = t0; t < n; t += stride) {
      const double wt = w[t];
      if (norm_only) {
        acc[0] += wt * wt;
      } else {
#pragma unroll
        for (int k = 0; k < ICGS_R; ++k)
          if (r0 + k < rows) acc[k] += V[(r0 + k) * ldv + t] * wt;
      }
    }
#pragma unroll
    for (int k = 0; k < ICGS_R; ++k) {
      double v = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MHDG_FULL, v, o);
      if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (tid < ICGS_R && r0 + tid < nout) {
      double v = 0.0;
      for (int wi = 0; wi < ICGS_T / 32; ++wi) v += red[wi][tid];
      partial[(long long)blockIdx.x * 64 + r0 + tid] = v;
    }
    __syncthreads();
  }
}

// out[i] (+)= sum_b partial[b][i] in block order; finalize: out[rows] = sqrt(norm), out[i] = h1 + h2
__global__ void k_icgs_reduce(int nb, int nout, const double* __restrict__ partial, double* __restrict__ dst,
                              const double* __restrict__ add) {
  for (int i = threadIdx.x; i < nout; i += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += partial[(long long)b * 64 + i];
    dst[i] = add ? add[i] + v : v;
  }
}

__global__ void k_icgs_sqrt(double* x) {
  if (threadIdx.x == 0) x[0] = sqrt(x[0]);
}

int icgs(int n, int j, const double* V, long long ldv, double* w, double* out, double* scratch, cudaStream_t st) {
  const int rows = j + 1;
  if (rows > 63) return MHDG_ERR_CONFIG;
  int nb = (int)((n + ICGS_T * 4 - 1) / (ICGS_T * 4));
  if (nb > 1184) nb = 1184;  // 8 blocks per SM on 148 SMs
  if (nb < 1) nb = 1;
  double* partial = scratch;                  // nb x 64
  double* h1 = scratch + (size_t)nb * 64;     // 64
  double* h2 = h1 + 64;                       // 64
  k_icgs_pass<<<nb, ICGS_T, 0, st>>>(n, rows, V, ldv, w, nullptr, 0, partial);
  k_icgs_reduce<<<1, 64, 0, st>>>(nb, rows, partial, h1, nullptr);
  k_icgs_pass<<<nb, ICGS_T, 0, st>>>(n, rows, V, ldv, w, h1, 0, partial);
  k_icgs_reduce<<<1, 64, 0, st>>>(nb, rows, partial, h2, nullptr);
  k_icgs_pass<<<nb, ICGS_T, 0, st>>>(n, rows, V, ldv, w, h2, 1, partial);
  k_icgs_reduce<<<1, 64, 0, st>>>(nb, 1, partial, out + rows, nullptr);
  k_icgs_reduce<<<1, 64, 0, st>>>(1, rows, h2, out, h1);  // h = h1 + h2
  k_icgs_sqrt<<<1, 32, 0, st>>>(out + rows);
  for (int k = 0; k < 8; ++k) launch_ok();
  return cudaPeekAtLastError() == cudaSuccess ? MHDG_OK : MHDG_ERR_CUDA;
}

long long icgs_scratch_size(int n) {
  int nb = (int)((n + ICGS_T * 4 - 1) / (ICGS_T * 4));
  if (nb > 1184) nb = 1184;
  if (nb < 1) nb = 1;
  return (long long)nb * 64 + 128;
}

}  // namespace mhdg
