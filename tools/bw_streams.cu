// Micro-benchmark: HBM bandwidth of a kernel that reads R and writes W
// separate arrays (one double each per point, grid-stride, coalesced), the
// access pattern of the BL / SS work-array fills (R ~ 10 / 3 inputs, W = 54 /
// 9 outputs).  Answers whether many concurrent write streams, rather than
// the fills' own latency, bound them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_streams tools/bw_streams.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void k(const double* __restrict__ in, double* __restrict__ out, long n) {
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += __ldg(in + r * n + t);
#pragma unroll
    for (int w = 0; w < W; ++w) out[w * n + t] = s + w;
  }
}

template <int R, int W>
void run(double* in, double* out, long n, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<R, W><<<blocks, threads>>>(in, out, n);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k<R, W><<<blocks, threads>>>(in, out, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)(R + W) * n * 8 * reps;
  printf("R=%2d W=%2d blocks=%6d threads=%4d: %7.1f GB/s  (%.3f ms per launch)\n", R, W, blocks,
         threads, bytes / (ms / 1e3) / 1e9, ms / reps);
}

int main() {
  const long n = 134217728L / 4;   // 32 Mi points per array (256 MiB)
  double *in, *out;
  if (cudaMalloc(&in, 10 * n * 8) || cudaMalloc(&out, 54 * n * 8)) { printf("oom\n"); return 1; }
  cudaMemset(in, 0, 10 * n * 8);
  for (int bpsm : {4, 8, 16}) {
    const int blocks = 148 * bpsm;
    run<1, 1>(in, out, n, blocks, 256);
    run<3, 9>(in, out, n, blocks, 256);
    run<10, 18>(in, out, n, blocks, 256);
    run<10, 36>(in, out, n, blocks, 256);
    run<10, 54>(in, out, n, blocks, 256);
    run<0, 54>(in, out, n, blocks, 256);
  }
  return 0;
}
