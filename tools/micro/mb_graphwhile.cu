#include <cuda_runtime.h>
#include <cstdio>
__global__ void ctl(cudaGraphConditionalHandle h, int* c, int n) {
  int k = c[0]; c[0] = k + 1;
  cudaGraphSetConditional(h, (k + 1 < n) ? 1u : 0u);
}
__global__ void work(int* c) { atomicAdd(c + 1, 1); }
int main() {
  int* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) { printf("handle fail\n"); return 1; }
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  if (e != cudaSuccess) { printf("add node %s\n", cudaGetErrorString(e)); return 1; }
  cudaGraph_t body = p.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) { printf("capture %s\n", cudaGetErrorString(e)); return 1; }
  work<<<1, 32, 0, s>>>(d);
  ctl<<<1, 1, 0, s>>>(h, d, 10);
  e = cudaStreamEndCapture(s, &body);
  if (e != cudaSuccess) { printf("end capture %s\n", cudaGetErrorString(e)); return 1; }
  cudaGraphExec_t x; e = cudaGraphInstantiate(&x, g, 0);
  if (e != cudaSuccess) { printf("inst %s\n", cudaGetErrorString(e)); return 1; }
  cudaGraphLaunch(x, s); cudaStreamSynchronize(s);
  int h2[2]; cudaMemcpy(h2, d, 8, cudaMemcpyDeviceToHost);
  printf("iters %d work %d err %s\n", h2[0], h2[1], cudaGetErrorString(cudaGetLastError()));
}
