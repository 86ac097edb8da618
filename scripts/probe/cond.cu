#include <cstdio>
#include <cuda_runtime.h>
__global__ void setc(cudaGraphConditionalHandle h, int* ctr, int limit) {
  int v = ++*ctr;
  cudaGraphSetConditional(h, v < limit ? 1u : 0u);
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {cudaGraphNodeTypeConditional};
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node; cudaGraphAddNode(&node, g, nullptr, 0, &p);
  cudaGraph_t body = p.conditional.phGraph_out[0];
  int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  setc<<<1,1,0,s>>>(h, ctr, 7);
  cudaGraph_t out; cudaStreamEndCapture(s, &out);
  cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int h_ctr; cudaMemcpy(&h_ctr, ctr, 4, cudaMemcpyDeviceToHost);
  printf("instantiate %s, iterations %d (expect 7), err %s\n", cudaGetErrorString(e), h_ctr, cudaGetErrorString(cudaGetLastError()));
}
