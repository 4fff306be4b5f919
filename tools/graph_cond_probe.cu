// Probe: a CUDA-graph WHILE node whose body holds two nested IF nodes, all conditions set
// from device code (the device-resident LM loop of lm_capi.inc relies on this).
// Expected output: "while 10, if-a 5, if-b 4".
#include <cuda_runtime.h>
#include <cstdio>
__global__ void ctl(cudaGraphConditionalHandle hw, cudaGraphConditionalHandle ha, cudaGraphConditionalHandle hb, int* c) {
  const int v = ++c[0];
  cudaGraphSetConditional(ha, v % 2);
  cudaGraphSetConditional(hb, v % 3 == 0 ? 1 : 0);
  cudaGraphSetConditional(hw, v < 10 ? 1 : 0);
}
__global__ void inc(int* c) { ++*c; }
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
static int add_cond(cudaGraph_t g, cudaGraphNode_t* deps, int nd, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType t,
                    cudaGraphNode_t* node, cudaGraph_t* body) {
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = t; p.conditional.size = 1;
  CK(cudaGraphAddNode(node, g, deps, nd, &p));
  *body = p.conditional.phGraph_out[0];
  return 0;
}
int main() {
  int* c; CK(cudaMalloc(&c, 16)); CK(cudaMemset(c, 0, 16));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw, ha, hb;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNode_t wn; cudaGraph_t body;
  if (add_cond(g, nullptr, 0, hw, cudaGraphCondTypeWhile, &wn, &body)) return 1;
  CK(cudaGraphConditionalHandleCreate(&ha, body, 0, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&hb, body, 0, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  inc<<<1, 1, 0, s>>>(c + 1);
  ctl<<<1, 1, 0, s>>>(hw, ha, hb, c);
  CK(cudaStreamEndCapture(s, &body));
  size_t n = 0; CK(cudaGraphGetNodes(body, nullptr, &n));
  cudaGraphNode_t nodes[8]; CK(cudaGraphGetNodes(body, nodes, &n));
  cudaGraphNode_t an, bn; cudaGraph_t ab, bb;
  if (add_cond(body, &nodes[n - 1], 1, ha, cudaGraphCondTypeIf, &an, &ab)) return 1;
  if (add_cond(body, &an, 1, hb, cudaGraphCondTypeIf, &bn, &bb)) return 1;
  CK(cudaStreamBeginCaptureToGraph(s, ab, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  inc<<<1, 1, 0, s>>>(c + 2);
  CK(cudaStreamEndCapture(s, &ab));
  CK(cudaStreamBeginCaptureToGraph(s, bb, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  inc<<<1, 1, 0, s>>>(c + 3);
  CK(cudaStreamEndCapture(s, &bb));
  cudaGraphExec_t x; CK(cudaGraphInstantiate(&x, g, 0));
  CK(cudaGraphLaunch(x, s)); CK(cudaStreamSynchronize(s));
  int h[4]; CK(cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost));
  printf("while %d, if-a %d, if-b %d\n", h[1], h[2], h[3]);
  return 0;
}
