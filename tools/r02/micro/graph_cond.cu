// Cost of conditional graph nodes on this pool: NODES x [k, IF{ k, WHILE(ITERS){5 k} }, k]
// vs the same kernels as a flat graph and as plain stream launches.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__global__ void work(int* v) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(v + 1, 1); }
__global__ void setw(cudaGraphConditionalHandle h, int* v, int iters) {
  int c = v[0]; cudaGraphSetConditional(h, c < iters ? 1u : 0u); v[0] = c + 1;
}
__global__ void setif(cudaGraphConditionalHandle h, int* v) { v[0] = 0; cudaGraphSetConditional(h, 1u); }
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
int main(int argc, char** argv) {
  const int NODES = 128, ITERS = argc > 1 ? atoi(argv[1]) : 3, GRID = 64;
  cudaStream_t s[3];
  for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  int* d; CK(cudaMalloc(&d, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // conditional graph
  CK(cudaStreamBeginCapture(s[0], cudaStreamCaptureModeRelaxed));
  for (int n = 0; n < NODES; ++n) {
    work<<<GRID, 256, 0, s[0]>>>(d);
    cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
    CK(cudaStreamGetCaptureInfo(s[0], &st, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle hi; CK(cudaGraphConditionalHandleCreate(&hi, g, 0, 0));
    setif<<<1, 1, 0, s[0]>>>(hi, d);
    CK(cudaStreamGetCaptureInfo(s[0], &st, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional; p.conditional.handle = hi;
    p.conditional.type = cudaGraphCondTypeIf; p.conditional.size = 1;
    cudaGraphNode_t node; CK(cudaGraphAddNode(&node, g, deps, nd, &p));
    CK(cudaStreamUpdateCaptureDependencies(s[0], &node, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(s[1], p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    work<<<GRID, 256, 0, s[1]>>>(d);
    CK(cudaStreamGetCaptureInfo(s[1], &st, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle hw; CK(cudaGraphConditionalHandleCreate(&hw, g, 0, 0));
    setw<<<1, 1, 0, s[1]>>>(hw, d, ITERS);
    CK(cudaStreamGetCaptureInfo(s[1], &st, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams q = {}; q.type = cudaGraphNodeTypeConditional; q.conditional.handle = hw;
    q.conditional.type = cudaGraphCondTypeWhile; q.conditional.size = 1;
    cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, deps, nd, &q));
    CK(cudaStreamUpdateCaptureDependencies(s[1], &wn, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(s[2], q.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < 5; ++i) work<<<GRID, 256, 0, s[2]>>>(d);
    setw<<<1, 1, 0, s[2]>>>(hw, d, ITERS);
    cudaGraph_t b; CK(cudaStreamEndCapture(s[2], &b));
    CK(cudaStreamEndCapture(s[1], &b));
    work<<<GRID, 256, 0, s[0]>>>(d);
  }
  cudaGraph_t g; CK(cudaStreamEndCapture(s[0], &g));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  // flat graph: the same kernel count unrolled
  CK(cudaStreamBeginCapture(s[0], cudaStreamCaptureModeRelaxed));
  for (int n = 0; n < NODES; ++n) {
    work<<<GRID, 256, 0, s[0]>>>(d); work<<<GRID, 256, 0, s[0]>>>(d);
    for (int i = 0; i < ITERS; ++i) for (int j = 0; j < 5; ++j) work<<<GRID, 256, 0, s[0]>>>(d);
    work<<<GRID, 256, 0, s[0]>>>(d);
  }
  cudaGraph_t gf; CK(cudaStreamEndCapture(s[0], &gf));
  cudaGraphExec_t exf; CK(cudaGraphInstantiate(&exf, gf, 0));
  for (int rep = 0; rep < 3; ++rep) {
    float ms[3];
    cudaEventRecord(e0, s[0]); CK(cudaGraphLaunch(ex, s[0])); cudaEventRecord(e1, s[0]); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms[0], e0, e1);
    cudaEventRecord(e0, s[0]); CK(cudaGraphLaunch(exf, s[0])); cudaEventRecord(e1, s[0]); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms[1], e0, e1);
    cudaEventRecord(e0, s[0]);
    for (int n = 0; n < NODES; ++n) {
      work<<<GRID, 256, 0, s[0]>>>(d); work<<<GRID, 256, 0, s[0]>>>(d);
      for (int i = 0; i < ITERS; ++i) for (int j = 0; j < 5; ++j) work<<<GRID, 256, 0, s[0]>>>(d);
      work<<<GRID, 256, 0, s[0]>>>(d);
    }
    cudaEventRecord(e1, s[0]); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms[2], e0, e1);
    int kernels = NODES * (3 + 5 * ITERS);
    printf("iters %d: conditional graph %.3f ms (%.2f us/kernel), flat graph %.3f ms (%.2f), stream %.3f ms (%.2f)\n",
           ITERS, ms[0], 1e3 * ms[0] / kernels, ms[1], 1e3 * ms[1] / kernels, ms[2], 1e3 * ms[2] / kernels);
  }
  return 0;
}
