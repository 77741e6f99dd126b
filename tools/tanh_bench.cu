// latency/throughput and accuracy of FP64 tanh variants with 4 independent evaluations per thread, 256 threads
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tanh_bench.bin tools/tanh_bench.cu
#include <cstdio>
#include <cmath>
#include "../paper_2510_11023_b200/csrc/pf_device.cuh"
__device__ __forceinline__ double tanh_exp(double u) {
  const double a = fabs(u);
  const double t = expm1(-2.0 * a);     // in (-1, 0]
  const double r = -t / (2.0 + t);
  return copysign(r, u);
}
template <int V>
__global__ void k(double* out, int reps, long long* cyc) {
  double u0 = 0.001 * threadIdx.x - 0.1, u1 = u0 + 0.3, u2 = u0 - 0.7, u3 = u0 + 1.1;
  double s = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double a, b, c, d;
    if (V == 0) { a = tanh(u0); b = tanh(u1); c = tanh(u2); d = tanh(u3); }
    else if (V == 1) { a = tanh_exp(u0); b = tanh_exp(u1); c = tanh_exp(u2); d = tanh_exp(u3); }
    else { a = pf::tanh_abs(u0); b = pf::tanh_abs(u1); c = pf::tanh_abs(u2); d = pf::tanh_abs(u3); }
    s += a + b + c + d;
    u0 += 1e-9 * a; u1 += 1e-9 * b; u2 += 1e-9 * c; u3 += 1e-9 * d;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_acc(double* maxabs, double* maxrcp) {
  // |tanh_abs - tanh| over u in [-30, 30] and a few tiny / huge arguments; rcp_fast vs 1/a
  double m = 0, mr = 0;
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < 6000000; i += blockDim.x * gridDim.x) {
    const double u = -30.0 + 1e-5 * i;
    m = fmax(m, fabs(pf::tanh_abs(u) - tanh(u)));
    const double a = 1.0 + 1e-3 * i;
    mr = fmax(mr, fabs(pf::rcp_fast(a) - 1.0 / a) * a);
  }
  const double sp[] = {0.0, -0.0, 1e-300, -1e-20, 1e-9, 700.0, -1e300, 1e308};
  for (double u : sp) m = fmax(m, fabs(pf::tanh_abs(u) - tanh(u)));
  atomicMax((unsigned long long*)maxabs, __double_as_longlong(m));   // positive doubles order as integers
  atomicMax((unsigned long long*)maxrcp, __double_as_longlong(mr));
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 64 * 256); cudaMalloc(&c, 8 * 64);
  long long h[64];
  k<0><<<64, 256>>>(o, 100, c); k<0><<<64, 256>>>(o, 1000, c); cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("CUDA tanh  : %.1f cycles per 4 evaluations (256 threads/SM)\n", h[0] / 1000.0);
  k<1><<<64, 256>>>(o, 1000, c); cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("expm1 tanh : %.1f cycles per 4 evaluations\n", h[0] / 1000.0);
  k<2><<<64, 256>>>(o, 1000, c); cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tanh_abs   : %.1f cycles per 4 evaluations\n", h[0] / 1000.0);
  double* m; cudaMalloc(&m, 16); cudaMemset(m, 0, 16);
  k_acc<<<148, 256>>>(m, m + 1);
  double hm[2]; cudaMemcpy(hm, m, 16, cudaMemcpyDeviceToHost);
  printf("max |tanh_abs - tanh| = %.3e   max rel |rcp_fast - 1/a| = %.3e   (%s)\n", hm[0], hm[1], cudaGetErrorString(cudaDeviceSynchronize()));
}
