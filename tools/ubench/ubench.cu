// Microbenchmarks for the FP64 paths on B200 (sm_100a): DMMA latency and
// throughput, DFMA latency, barrier / shuffle / redux / smem-atomic latency.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(int iters, double* out, long long* cyc) {
  double c[CH][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(int iters, double* out, long long* cyc) {
  double x = threadIdx.x, y = 1.0000001;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_bar(int iters, long long* cyc) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_shfl64(int iters, unsigned long long* out, long long* cyc) {
  unsigned long long v = threadIdx.x * 12345ull;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    unsigned long long t = __shfl_xor_sync(0xffffffffu, v, 1);
    v = t > v ? t : v + 1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_redux(int iters, unsigned* out, long long* cyc) {
  unsigned v = threadIdx.x * 7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) v = __reduce_max_sync(0xffffffffu, v) + (threadIdx.x & 1);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_rcp(int iters, double* out, long long* cyc) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = 1.0 / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_satom(int iters, unsigned long long* out, long long* cyc) {
  __shared__ unsigned long long s[4];
  if (threadIdx.x < 4) s[threadIdx.x] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if ((threadIdx.x & 31) == 0) atomicMax(&s[it & 3], (unsigned long long)(it * 131 + threadIdx.x));
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = s[threadIdx.x & 3];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// pointer chase for load latency
__global__ void k_chase(const int* __restrict__ nxt, int iters, int* out, long long* cyc) {
  int p = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) p = nxt[p];
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}

int main() {
  double* dout; long long* cyc; unsigned long long* uout; unsigned* u32; int* iout;
  cudaMalloc(&dout, 1 << 24); cudaMalloc(&cyc, 1 << 16); cudaMalloc(&uout, 1 << 16); cudaMalloc(&u32, 1 << 16);
  cudaMalloc(&iout, 1 << 16);
  long long h[1024];
  const int it = 4096;
  auto rd = [&](int nblk) { cudaDeviceSynchronize(); cudaMemcpy(h, cyc, 8 * nblk, cudaMemcpyDeviceToHost); };
  // DMMA latency: one warp, one chain
  k_dmma<1><<<1, 32>>>(it, dout, cyc); rd(1); printf("DMMA latency (1 chain, 1 warp): %.1f cycles\n", (double)h[0] / it);
  k_dmma<4><<<1, 32>>>(it, dout, cyc); rd(1); printf("DMMA 4 chains, 1 warp: %.1f cycles per DMMA\n", (double)h[0] / it / 4);
  k_dmma<8><<<1, 32>>>(it, dout, cyc); rd(1); printf("DMMA 8 chains, 1 warp: %.1f cycles per DMMA\n", (double)h[0] / it / 8);
  for (int w : {4, 8, 16, 32}) {
    k_dmma<8><<<148, 32 * w>>>(it, dout, cyc); rd(148);
    printf("DMMA 8 chains x %d warps per SM: %.2f cycles per DMMA per SM (%.1f flop/cycle/SM)\n", w,
           (double)h[0] / it / 8 / w, 512.0 * 8 * w * it / h[0]);
  }
  k_dmma<4><<<148, 512>>>(it, dout, cyc); rd(148);
  printf("DMMA 4 chains x 16 warps per SM: %.2f cycles per DMMA per SM\n", (double)h[0] / it / 4 / 16);
  k_dfma<<<1, 32>>>(it, dout, cyc); rd(1); printf("DFMA latency: %.1f\n", (double)h[0] / it);
  for (int t : {256, 512}) { k_bar<<<1, t>>>(it, cyc); rd(1); printf("__syncthreads %d threads: %.1f\n", t, (double)h[0] / it); }
  k_bar<<<296, 256>>>(it, cyc); rd(2); printf("__syncthreads 256 threads, 2 CTAs/SM: %.1f\n", (double)h[0] / it);
  k_shfl64<<<1, 32>>>(it, uout, cyc); rd(1); printf("64-bit shfl + max latency: %.1f\n", (double)h[0] / it);
  k_redux<<<1, 32>>>(it, u32, cyc); rd(1); printf("redux.max latency: %.1f\n", (double)h[0] / it);
  k_rcp<<<1, 32>>>(it, dout, cyc); rd(1); printf("fp64 1/x + 1 latency: %.1f\n", (double)h[0] / it);
  k_satom<<<1, 256>>>(it, uout, cyc); rd(1); printf("8 smem atomicMax u64 + barrier: %.1f\n", (double)h[0] / it);
  // load latency: L2-resident chase (1 MB) and HBM chase (1 GB)
  for (long long bytes : {1LL << 20, 1LL << 30}) {
    const int n = (int)(bytes / 4);
    int* hn = new int[n];
    const int stride = 4099 * 16;
    for (int i = 0; i < n; ++i) hn[i] = (int)(((long long)i + stride) % n);
    int* dn; cudaMalloc(&dn, bytes); cudaMemcpy(dn, hn, bytes, cudaMemcpyHostToDevice);
    k_chase<<<1, 1>>>(dn, 2048, iout, cyc); rd(1); k_chase<<<1, 1>>>(dn, 2048, iout, cyc); rd(1);
    printf("load latency, %lld MB footprint: %.0f cycles\n", bytes >> 20, (double)h[0] / 2048);
    cudaFree(dn); delete[] hn;
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
