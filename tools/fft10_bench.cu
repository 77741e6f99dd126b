// Microbenchmarks behind the round-2 FFT-pass changes of the config-3 sweep:
//  (1) DFMA issue rate per SM sub-partition for warps with 32 / 16 / 8 active lanes
//  (2) the Q = 1024 inverse -> pointwise -> forward pass chain (apply_k's shape) with the
//      radix-8 butterflies on 4 full warps (threads 0..127) or on 8 half warps (16 lanes each)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/fft10_bench.bin tools/fft10_bench.cu
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2510_11023_b200/csrc/pf_sine1d.cuh"
using namespace pf;

template <int ACTIVE, int CHAINS>
__global__ void k_dfma(int reps, long long* cyc, double* sink) {
  double a[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  if ((threadIdx.x & 31) < ACTIVE) {
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) a[i] = fma(a[i], m, c);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += a[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// radix-8 pass with the butterflies on 8 half warps
template <bool INV, int NS, int TWO, int MODE>
__device__ __forceinline__ void r8_pass10m(const cd* __restrict__ a, cd* __restrict__ b, const cd* __restrict__ tw) {
  const int tid = threadIdx.x;
  const int j = MODE == 0 ? tid : ((tid >> 5) * 16 + (tid & 15));
  const bool on = MODE == 0 ? tid < 128 : (tid & 31) < 16;
  if (on) {
    const int k = j & (NS - 1);
    cd v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = a[sw10(j + t * 128)];
    if (NS > 1) {
      cd w1 = tw[TWO + k], w4 = tw[TWO + NS + k];
      if (INV) {
        w1.y = -w1.y;
        w4.y = -w4.y;
      }
      const cd w2 = cmul(w1, w1), w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
      v[1] = cmul(v[1], w1);
      v[2] = cmul(v[2], w2);
      v[3] = cmul(v[3], w3);
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], w5);
      v[6] = cmul(v[6], w6);
      v[7] = cmul(v[7], w7);
    }
    dft8<INV>(v);
    const int base = ((j - k) << 3) + k;
#pragma unroll
    for (int m = 0; m < 8; ++m) b[sw10(base + m * NS)] = v[m];
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_pair(const cd* twg, int reps, long long* cyc, double* sink) {
  extern __shared__ __align__(16) char sm[];
  cd* tw = reinterpret_cast<cd*>(sm);
  cd* A = tw + T10_SIZE;
  cd* B = A + 1024;
  double* dq = reinterpret_cast<double*>(B + 1024);
  for (int j = threadIdx.x; j < T10_SIZE; j += 256) tw[j] = twg[j];
  for (int j = threadIdx.x; j < 1024; j += 256) {
    A[sw10(j)] = {1.0 / (j + 1), 0.5};
    dq[j] = 1.0 / 1024 + 1e-6 * j;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    r8_pass10m<true, 1, 0, MODE>(A, B, tw);
    __syncthreads();
    r8_pass10m<true, 8, T10_R8_8, MODE>(B, A, tw);
    __syncthreads();
    r4_pass10<true, 64, T10_R4_64>(A, B, tw);
    __syncthreads();
    cd v[4];
    last_inv10(B, tw, v);
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = {0.0, dq[threadIdx.x + 256 * q] * (0.5 * v[q].y)};
    first_fwd10(v, A);
    __syncthreads();
    r4_pass10<false, 4, T10_R4_4>(A, B, tw);
    __syncthreads();
    r8_pass10m<false, 16, T10_R8_16, MODE>(B, A, tw);
    __syncthreads();
    r8_pass10m<false, 128, T10_R8_128, MODE>(A, B, tw);
    __syncthreads();
    // keep magnitudes bounded: scale into A
    for (int j = threadIdx.x; j < 1024; j += 256) {
      const cd z = B[sw10(j)];
      A[sw10(j)] = {z.x * 1e-3, z.y * 1e-3};
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x] = A[5].x;
  }
}

template <int ACTIVE, int CHAINS>
void run_dfma(int nthreads) {
  long long* d_c;
  cudaMalloc(&d_c, 8 * 64);
  double* d_s;
  cudaMalloc(&d_s, 8 * 64 * 1024);
  const int reps = 4000;
  k_dfma<ACTIVE, CHAINS><<<64, nthreads>>>(10, d_c, d_s);
  k_dfma<ACTIVE, CHAINS><<<64, nthreads>>>(reps, d_c, d_s);
  long long c[64];
  cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
  const int wps = nthreads / 128;  // warps per sub-partition
  printf("DFMA active=%2d chains=%2d warps/SMSP=%d : %.2f cycles per warp-DFMA per SMSP\n", ACTIVE, CHAINS, wps,
         (double)c[0] / ((double)reps * CHAINS * wps));
  cudaFree(d_c);
  cudaFree(d_s);
}

template <int MODE>
void run_pair(const cd* d_tw) {
  long long* d_c;
  cudaMalloc(&d_c, 8 * 64);
  double* d_s;
  cudaMalloc(&d_s, 8 * 64);
  size_t smem = sizeof(cd) * (T10_SIZE + 2048) + 8 * 1024;
  cudaFuncSetAttribute(k_pair<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 2000;
  k_pair<MODE><<<64, 256, smem>>>(d_tw, 10, d_c, d_s);
  k_pair<MODE><<<64, 256, smem>>>(d_tw, reps, d_c, d_s);
  long long c[64];
  cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
  double s;
  cudaMemcpy(&s, d_s, 8, cudaMemcpyDeviceToHost);
  printf("pair chain MODE=%d : %.1f cycles per inverse+forward pair (sink %.6e)\n", MODE, (double)c[0] / reps, s);
}

int main() {
  run_dfma<32, 8>(128);
  run_dfma<16, 8>(128);
  run_dfma<8, 8>(128);
  run_dfma<32, 8>(256);
  run_dfma<16, 8>(256);
  run_dfma<32, 1>(128);
  run_dfma<16, 1>(128);
  // twiddle table (any unit-modulus values time the same; use the real ones' shape)
  std::vector<cd> tw(T10_SIZE);
  for (int i = 0; i < T10_SIZE; ++i) {
    const double a = -2 * M_PI * i / 1024.0;
    tw[i] = {cos(a), sin(a)};
  }
  cd* d_tw;
  cudaMalloc(&d_tw, sizeof(cd) * T10_SIZE);
  cudaMemcpy(d_tw, tw.data(), sizeof(cd) * T10_SIZE, cudaMemcpyHostToDevice);
  run_pair<0>(d_tw);
  run_pair<1>(d_tw);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
