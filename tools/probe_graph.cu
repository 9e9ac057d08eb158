// probe: which conditional-graph construction does this driver accept?
#include <cuda_runtime.h>
#include <cstdio>
__global__ void kset(cudaGraphConditionalHandle h, int* cnt, int use) {
  if (threadIdx.x == 0) { int c = atomicAdd(cnt, 1); if (use) cudaGraphSetConditional(h, c < 3 ? 1 : 0); }
}
__global__ void kplain(int* cnt) { if (threadIdx.x == 0) atomicAdd(cnt, 100); }
#define P(x) do { cudaError_t e = (x); printf("%-60s -> %s\n", #x, cudaGetErrorString(e)); } while (0)
int main() { setvbuf(stdout, NULL, _IONBF, 0);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* cnt; cudaMalloc(&cnt, 4);
  for (int variant = 1; variant < 4; ++variant) {
    printf("--- variant %d\n", variant);
    cudaMemset(cnt, 0, 4);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    P(cudaGraphConditionalHandleCreate(&h, g, variant == 2 ? 1 : 0, cudaGraphCondAssignDefault));
    // upstream kernel (captured)
    P(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    kset<<<1, 32, 0, s>>>(h, cnt, variant == 1 || variant == 3);
    cudaGraph_t tmp; P(cudaStreamEndCapture(s, &tmp));
    if (variant != 0) {
      size_t nn = 0; cudaGraphGetNodes(g, nullptr, &nn);
      cudaGraphNode_t nodes[8]; cudaGraphGetNodes(g, nodes, &nn);
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
      cudaGraphNode_t cn; P(cudaGraphAddNode(&cn, g, nodes, nn, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      if (variant == 3) {
        // add body kernel via explicit node API
        cudaKernelNodeParams kp = {}; void* args[] = {&h, &cnt, &variant};
        int use = 1; void* args2[] = {&h, &cnt, &use};
        kp.func = (void*)kset; kp.gridDim = dim3(1); kp.blockDim = dim3(32); kp.kernelParams = args2;
        cudaGraphNode_t kn; P(cudaGraphAddKernelNode(&kn, body, nullptr, 0, &kp));
      } else {
        P(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        kset<<<1, 32, 0, s>>>(h, cnt, 1);
        cudaGraph_t tmp2; P(cudaStreamEndCapture(s, &tmp2));
      }
    }
    cudaGraphExec_t ge; P(cudaGraphInstantiate(&ge, g, 0));
    P(cudaGraphLaunch(ge, s)); P(cudaStreamSynchronize(s));
    int hv; cudaMemcpy(&hv, cnt, 4, cudaMemcpyDeviceToHost); printf("count=%d\n", hv);
  }
  return 0;
}
