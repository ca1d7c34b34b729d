#include <cuda_runtime.h>
#include <stdio.h>
__global__ void k_step(cudaGraphConditionalHandle h, int *k, int n) {
    int v = ++(*k);
    cudaGraphSetConditional(h, v < n ? 1u : 0u);
}
int main() {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle hd;
    cudaGraphConditionalHandleCreate(&hd, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = hd; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t node; cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t s; cudaStreamCreate(&s);
    int *k; cudaMalloc(&k, 4); cudaMemset(k, 0, 4);
    cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    k_step<<<1,1,0,s>>>(hd, k, 10);
    cudaStreamEndCapture(s, &body);
    cudaGraphExec_t ex; cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
    int hk; cudaMemcpy(&hk, k, 4, cudaMemcpyDeviceToHost);
    printf("k=%d err=%s\n", hk, cudaGetErrorString(cudaGetLastError()));
}
