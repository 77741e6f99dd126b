// Microbenchmark of the in-smem FP64 FFT core: cycles per length-Q FFT for one
// CTA (the fine-sweep kernel's latency-bound regime), plus __syncthreads cost.
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2510_11023_b200/csrc/pf_sine1d.cuh"
using namespace pf;

template <int LG, int NT>
__global__ void k_fft(const cd* twg, int reps, long long* cyc, double* sink) {
  extern __shared__ __align__(16) char sm[];
  constexpr int Q = 1 << LG;
  constexpr int TW = tw_table_size(LG);
  cd* tw = reinterpret_cast<cd*>(sm);
  cd* A = tw + TW;
  cd* B = A + Q;
  for (int j = threadIdx.x; j < TW; j += NT) tw[j] = twg[j];
  for (int j = threadIdx.x; j < Q; j += NT) A[sw(j)] = {1.0 / (j + 1), 0.5};
  __syncthreads();
  long long t0 = clock64();
  cd* a = A; cd* b = B;
  for (int r = 0; r < reps; ++r) {
    cd* R = fft_stockham<LG, NT, false>(a, b, tw);
    cd* O = (R == a) ? b : a;
    a = R; b = O;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; sink[blockIdx.x] = a[1].x; }
}

template <int NT>
__global__ void k_bar(int reps, long long* cyc) {
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) bar<NT>();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int LG, int NT>
void run(const char* name) {
  const int Q = 1 << LG, TW = tw_table_size(LG);
  std::vector<cd> tw(TW > 0 ? TW : 1);
  int off = 0;
  for (int p = 1, ns = 4; p < LG / 2; ++p, ns *= 4) {
    for (int r = 1; r <= 3; ++r)
      for (int k = 0; k < ns; ++k) { double a = -2 * M_PI * r * k / (4.0 * ns); tw[off + (r - 1) * ns + k] = {cos(a), sin(a)}; }
    off += 3 * ns;
  }
  if (LG & 1) { int ns = 1 << (LG - 1); for (int k = 0; k < ns; ++k) { double a = -2 * M_PI * k / (2.0 * ns); tw[off + k] = {cos(a), sin(a)}; } }
  cd* d_tw; cudaMalloc(&d_tw, sizeof(cd) * tw.size()); cudaMemcpy(d_tw, tw.data(), sizeof(cd) * tw.size(), cudaMemcpyHostToDevice);
  long long* d_c; cudaMalloc(&d_c, 8 * 64); double* d_s; cudaMalloc(&d_s, 8 * 64);
  size_t smem = sizeof(cd) * (TW + 2 * Q);
  cudaFuncSetAttribute(k_fft<LG, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int reps = 2000;
  k_fft<LG, NT><<<64, NT, smem>>>(d_tw, 10, d_c, d_s);
  k_fft<LG, NT><<<64, NT, smem>>>(d_tw, reps, d_c, d_s);
  long long c[64]; cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-24s Q=%5d NT=%4d : %8.1f cycles per FFT (%d passes)\n", name, Q, NT, (double)c[0] / reps, LG / 2 + (LG & 1));
}

int main() {
  run<6, 32>("fft");
  run<7, 32>("fft");
  run<8, 64>("fft");
  run<9, 128>("fft");
  run<10, 256>("fft");
  run<10, 128>("fft");
  run<11, 256>("fft");
  long long* d_c; cudaMalloc(&d_c, 8 * 64); long long c[64];
  k_bar<256><<<64, 256>>>(10000, d_c); cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
  printf("__syncthreads (256 thr): %.1f cycles\n", c[0] / 10000.0);
  k_bar<128><<<64, 128>>>(10000, d_c); cudaMemcpy(c, d_c, sizeof(c), cudaMemcpyDeviceToHost);
  printf("__syncthreads (128 thr): %.1f cycles\n", c[0] / 10000.0);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
