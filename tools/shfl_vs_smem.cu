// Microbenchmark: warp-shuffle vs shared-memory throughput per SM on B200, and
// whether they share a datapath (both in one loop).
#include <cstdio>
template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters) {
  __shared__ double sm[8][256 * 2];
  const int t = threadIdx.x;
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = t * 1.0 + j; sm[j][t] = x[j]; sm[j][t + 256] = x[j]; }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0 || MODE == 2) x[j] = __shfl_xor_sync(0xffffffffu, x[j], 1 + (j & 15)) + 1.0;
      if (MODE == 1 || MODE == 2) {
        double2 v = reinterpret_cast<double2*>(&sm[j][0])[(t + it + j) & 255];
        x[j] += v.x + v.y;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * 256 + t] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 8, iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, 256>>>(out, iters);
      if (mode == 1) k<1><<<blocks, 256>>>(out, iters);
      if (mode == 2) k<2><<<blocks, 256>>>(out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double warp_ops = (double)blocks * 8 * iters * 8;  // warps * iters * 8 per iter
      double clk = ms * 1e-3 * 1.965e9;
      if (rep) printf("mode %d (%s): %.3f ms, %.3f warp-ops/clk/SM (shfl.f64 = 2 SHFL; lds.128 = 4 wavefronts)\n",
                      mode, mode == 0 ? "shfl f64" : mode == 1 ? "lds.128" : "both", ms, warp_ops / clk / 148);
    }
  }
  return 0;
}
