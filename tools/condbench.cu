// Microbenchmark: cost of one conditional-WHILE iteration in a CUDA graph
// (device-side body relaunch) vs the same kernels unrolled in a plain graph.
// The body is K dependent tiny kernels; the last one decrements a counter and
// sets the loop condition, like the GMRES inner loop's update kernel.
//   condbench [iters] [kernels-per-body]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1); } } while (0)

__global__ void k_work(int* c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(c + 1, 1);
}
__global__ void k_last(int* c, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const int left = --c[0];
        cudaGraphSetConditional(h, left > 0 ? 1u : 0u);
    }
}
__global__ void k_last_plain(int* c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) --c[0];
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? std::atoi(argv[1]) : 1000;
    const int kper = argc > 2 ? std::atoi(argv[2]) : 8;
    int* c;
    CK(cudaMalloc(&c, 8));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // conditional WHILE graph
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
    for (int k = 0; k < kper - 1; ++k) k_work<<<1, 32, 0, st>>>(c);
    k_last<<<1, 32, 0, st>>>(c, h);
    CK(cudaStreamEndCapture(st, &body));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    // plain unrolled graph of the same kernels
    cudaGraph_t gp;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < iters; ++i) {
        for (int k = 0; k < kper - 1; ++k) k_work<<<1, 32, 0, st>>>(c);
        k_last_plain<<<1, 32, 0, st>>>(c);
    }
    CK(cudaStreamEndCapture(st, &gp));
    cudaGraphExec_t gpe;
    CK(cudaGraphInstantiate(&gpe, gp, 0));
    for (int rep = 0; rep < 3; ++rep) {
        int init[2] = {iters, 0};
        CK(cudaMemcpy(c, init, 8, cudaMemcpyHostToDevice));
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms_c = 0;
        CK(cudaEventElapsedTime(&ms_c, e0, e1));
        CK(cudaMemcpy(c, init, 8, cudaMemcpyHostToDevice));
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(gpe, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms_p = 0;
        CK(cudaEventElapsedTime(&ms_p, e0, e1));
        std::printf("%d iterations x %d kernels: conditional %.2f us/iter, unrolled %.2f us/iter, "
                    "WHILE overhead %.2f us/iter\n", iters, kper, 1000.0 * ms_c / iters,
                    1000.0 * ms_p / iters, 1000.0 * (ms_c - ms_p) / iters);
    }
    return 0;
}
