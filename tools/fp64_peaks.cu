// FP64 peak microbenchmarks on sm_100a: DFMA pipe, DMMA (mma.sync f64), cuBLAS DGEMM,
// plus __syncthreads round-trip latency for a 256/512-thread CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  // m8n8k4 f64: A 8x4 (1 reg/thread), B 4x8 (1 reg), C/D 8x8 (2 regs)
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  // m16n8k16 f64 (sm_90+ shape): A 8 regs, B 4 regs, C 4 regs
  double a[8], b[4], c[4][4];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = threadIdx.x * 1e-3 + t;
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = 1.0 - t * 1e-4;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int t = 0; t < 4; ++t) c[u][t] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int t = 0; t < 4; ++t) s += c[u][t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void sync_kernel(double* out, int iters, long long* cycles) {
  __shared__ double buf[1024];
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[threadIdx.x] = acc;
    __syncthreads();
    acc += buf[(threadIdx.x + 1) % blockDim.x];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096, threads = 512, blocks = sms * 4;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (threads / 32) * blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    dmma16_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * (threads / 32) * blocks;
    printf("DMMA m16n8k16: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  // cuBLAS DGEMM
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {1024, 2048, 4096, 8192}) {
    double *A, *B, *C; cudaMalloc(&A, 8.0 * n * n); cudaMalloc(&B, 8.0 * n * n); cudaMalloc(&C, 8.0 * n * n);
    cudaMemset(A, 0, 8.0 * n * n); cudaMemset(B, 0, 8.0 * n * n);
    double al = 1, be = 0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
    cudaDeviceSynchronize();
    int reps = n >= 4096 ? 5 : 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("cuBLAS DGEMM n=%d: %.2f TFLOP/s\n", n, 2.0 * n * n * (double)n * reps / ms / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // batched small DGEMM (64 x 512x512x1024) like the dense Galerkin assembly
  {
    int M = 512, Q = 1024, bs = 64;
    double *A, *C; cudaMalloc(&A, 8.0 * Q * M * bs); cudaMalloc(&C, 8.0 * M * M * bs);
    cudaMemset(A, 0, 8.0 * Q * M * bs);
    double al = 1, be = 0;
    for (int r = 0; r < 6; ++r) {
      if (r == 1) cudaEventRecord(e0);
      cublasDgemmStridedBatched(h, CUBLAS_OP_T, CUBLAS_OP_N, M, M, Q, &al, A, Q, (long long)Q * M, A, Q, (long long)Q * M, &be, C, M, (long long)M * M, bs);
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("cuBLAS batched 64x(512x512x1024): %.2f TFLOP/s, %.3f ms each\n", 2.0 * M * M * (double)Q * bs * 5 / ms / 1e9, ms / 5);
  }
  // sync latency
  long long* cyc; cudaMalloc(&cyc, sizeof(long long) * 1024);
  for (int threads : {128, 256, 512, 1024}) {
    int iters = 10000;
    sync_kernel<<<64, threads>>>(out, iters, cyc);
    long long hc[64]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    printf("syncthreads pair, %d threads, 64 CTAs: %.1f cycles per (2 syncs + smem)\n", threads, (double)hc[0] / iters);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
