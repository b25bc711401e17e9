// Slab halo kernels of the multi-GPU path (one process per GPU, macro slabs;
// SURVEY 8e).  The reference has no distributed code; the paper's matvec
// needs communication in its step 4 -- the trace sum of
// _scatter_add (condense.py:48-51) across a slab boundary.
//
// k_halo_gather    buf[i] = src[idx[i]]            (pack a halo message)
// k_halo_scatter   dst[idx[i]] (+)= buf[i]         (unpack; indices unique)
// k_face_reduce_remote
//                  y[i] = y_loc[a] + (y_loc[c] | remote[r] | 0) for the owned
//                  trace dofs: the reverse halo summed inside the face
//                  reduction (a face split across ranks has one local side,
//                  the other side's contribution arrives in `remote`); with at
//                  most two contributions per dof the sum is bitwise the
//                  single-process one whatever the arrival order.
#include "common.cuh"

namespace mhdg {

__global__ void k_halo_gather(long long n, const int* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ buf) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    buf[i] = __ldg(src + __ldg(idx + i));
}

__global__ void k_halo_scatter(long long n, const int* __restrict__ idx, const double* __restrict__ buf,
                               double* __restrict__ dst, int accumulate) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int j = __ldg(idx + i);
    dst[j] = accumulate ? dst[j] + buf[i] : buf[i];
  }
}

__global__ void k_face_reduce_remote(int n_out, const int* __restrict__ src, const double* __restrict__ y_loc,
                                     const int* __restrict__ remote_src, const double* __restrict__ remote,
                                     double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += gridDim.x * blockDim.x) {
    const int a = __ldg(src + 2 * i), c = __ldg(src + 2 * i + 1);
    double v = __ldg(y_loc + a);
    if (c >= 0) {
      v += __ldg(y_loc + c);
    } else if (remote_src) {
      const int r = __ldg(remote_src + i);
      if (r >= 0) v += __ldg(remote + r);
    }
    y[i] = v;
  }
}

static inline int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : (int)b;
}

int halo_gather(long long n, const int* idx, const double* src, double* buf, cudaStream_t st) {
  if (n <= 0) return MHDG_OK;
  tl_begin(TL_HALO, st);
  k_halo_gather<<<grid_for(n), 256, 0, st>>>(n, idx, src, buf);
  tl_end(TL_HALO, st);
  return launch_ok();
}

int halo_scatter(long long n, const int* idx, const double* buf, double* dst, int accumulate, cudaStream_t st) {
  if (n <= 0) return MHDG_OK;
  tl_begin(TL_HALO, st);
  k_halo_scatter<<<grid_for(n), 256, 0, st>>>(n, idx, buf, dst, accumulate);
  tl_end(TL_HALO, st);
  return launch_ok();
}

int face_reduce_remote(const mhdg_disc& g, const double* y_loc, const int* remote_src, const double* remote,
                       int n_out, double* y, cudaStream_t st) {
  if (n_out < 0 || n_out > g.n_trace) return MHDG_ERR_CONFIG;
  if (n_out == 0) return MHDG_OK;
  tl_begin(TL_FACE_REDUCE, st);
  k_face_reduce_remote<<<grid_for(n_out), 256, 0, st>>>(n_out, g.scatter_src, y_loc, remote_src, remote, y);
  tl_end(TL_FACE_REDUCE, st);
  return launch_ok();
}

}  // namespace mhdg
