// Microbenchmark: chains of dependent 7-point DIA smoothing kernels
//   y = x + wd * (r - A x)
// launched three ways inside one CUDA graph:
//   mode 0  plain stream order (full kernel boundary between links)
//   mode 1  programmatic launch + griddepcontrol.wait (prologue overlap only)
//   mode 2  programmatic launch + per-CTA completion flags: a CTA waits only
//           for the producer CTAs whose rows its stencil reads, so the next
//           link runs in the previous link's tail
// usage: flowbench [links] [reps]  -> one line per (n, mode): us per link
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1); } } while (0)

constexpr int kT = 256;

struct Flow {
    const unsigned* dep;   // producer flags (per producer CTA) or null
    unsigned* out;         // this kernel's flags
    const unsigned* seqp;  // expected flag value
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kT) k_smooth(int n, int w, const double* __restrict__ vals,
                                               const double* x, const double* __restrict__ r,
                                               const double* __restrict__ wd, double* y, Flow f) {
    if (MODE == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int i = blockIdx.x * kT + threadIdx.x;
    const int off[7] = {-w - 1, -w, -1, 0, 1, w, w + 1};
    double v[7];
    const int ii = min(i, n - 1);
#pragma unroll
    for (int d = 0; d < 7; ++d) v[d] = __ldg(vals + static_cast<long long>(d) * n + ii);
    if (MODE == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned seq = 0;
    if (MODE == 2) {
        // the chain's first link waits for its (normal) predecessor; every
        // link reads the expected flag value before letting dependents launch
        if (!f.dep) asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seq) : "l"(f.seqp) : "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (f.dep) {
            const int nb = (n + kT - 1) / kT;
            const int lo = max(0, static_cast<int>(blockIdx.x) * kT - w - 1) / kT;
            const int hi = min(nb - 1, (static_cast<int>(blockIdx.x) * kT + kT - 1 + w + 1) / kT);
            for (int p = lo + threadIdx.x; p <= hi; p += kT)
                while (ld_acquire(f.dep + p) != seq) __nanosleep(20);
        }
        __syncthreads();
    }
    if (i < n) {
        double s = 0.0;
#pragma unroll
        for (int d = 0; d < 7; ++d) {
            const int c = min(max(i + off[d], 0), n - 1);
            s += v[d] * x[c];
        }
        y[i] = x[i] + wd[i] * (r[i] - s);
    }
    if (MODE == 2) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_relaxed(f.out + blockIdx.x, seq);
        }
    }
}

__global__ void k_bump(unsigned* seq) { *seq += 1; }

template <int MODE>
void launch(int n, int w, const double* vals, const double* x, const double* r, const double* wd, double* y,
            Flow f, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((n + kT - 1) / kT);
    cfg.blockDim = dim3(kT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = MODE >= 1 ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_smooth<MODE>, n, w, vals, x, r, wd, y, f));
}

int main(int argc, char** argv) {
    const int links = argc > 1 ? std::atoi(argv[1]) : 40;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
    const int sizes[] = {1046529, 174847, 19494, 2205};
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    unsigned* seq;
    CK(cudaMalloc(&seq, 4));
    CK(cudaMemset(seq, 0, 4));
    std::vector<double> ref_out;
    for (int n : sizes) {
        int w = 1;
        while ((w + 1) * (w + 1) <= n) ++w;
        const int nb = (n + kT - 1) / kT;
        std::vector<double> hv(7LL * n), hx(n), hr(n), hw(n);
        for (long long k = 0; k < 7LL * n; ++k) hv[k] = (k % 7 == 3) ? 4.0 : -0.5 + 0.01 * (k % 5);
        for (int i = 0; i < n; ++i) {
            hx[i] = std::sin(0.37 * i) + 0.5;
            hr[i] = std::cos(0.11 * i);
            hw[i] = 0.6 / 4.0;
        }
        double *vals, *r, *wd, *b[3];
        CK(cudaMalloc(&vals, 8 * hv.size()));
        CK(cudaMalloc(&r, 8LL * n));
        CK(cudaMalloc(&wd, 8LL * n));
        for (auto& p : b) CK(cudaMalloc(&p, 8LL * n));
        CK(cudaMemcpy(vals, hv.data(), 8 * hv.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(r, hr.data(), 8LL * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wd, hw.data(), 8LL * n, cudaMemcpyHostToDevice));
        unsigned* flags;
        CK(cudaMalloc(&flags, 4LL * nb * links));
        CK(cudaMemset(flags, 0, 4LL * nb * links));
        for (int mode = 0; mode < 3; ++mode) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            k_bump<<<1, 1, 0, st>>>(seq);
            for (int k = 0; k < links; ++k) {
                Flow f{k ? flags + static_cast<long long>(k - 1) * nb : nullptr, flags + static_cast<long long>(k) * nb, seq};
                const double* x = b[k % 3];
                double* y = b[(k + 1) % 3];
                if (mode == 0) launch<0>(n, w, vals, x, r, wd, y, f, st);
                if (mode == 1) launch<1>(n, w, vals, x, r, wd, y, f, st);
                if (mode == 2) launch<2>(n, w, vals, x, r, wd, y, f, st);
            }
            CK(cudaStreamEndCapture(st, &g));
            cudaGraphExec_t ge;
            CK(cudaGraphInstantiate(&ge, g, 0));
            for (auto p : b) CK(cudaMemcpy(p, hx.data(), 8LL * n, cudaMemcpyHostToDevice));
            for (int q = 0; q < 3; ++q) CK(cudaGraphLaunch(ge, st));
            CK(cudaStreamSynchronize(st));
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, st));
            for (int q = 0; q < reps; ++q) CK(cudaGraphLaunch(ge, st));
            CK(cudaEventRecord(e1, st));
            CK(cudaStreamSynchronize(st));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::vector<double> out(n);
            CK(cudaMemcpy(out.data(), b[links % 3], 8LL * n, cudaMemcpyDeviceToHost));
            if (mode == 0) ref_out = out;
            bool same = out == ref_out;
            const double us = 1000.0 * ms / reps / links;
            const double gbs = (7.0 * 8 + 4 * 8) * n / (us * 1e-6) / 1e9;
            std::printf("n=%8d mode=%d  %7.2f us/link  %7.1f GB/s  %s\n", n, mode, us, gbs,
                        same ? "bit-identical" : "MISMATCH");
            CK(cudaGraphExecDestroy(ge));
            CK(cudaGraphDestroy(g));
        }
        cudaFree(vals); cudaFree(r); cudaFree(wd); cudaFree(flags);
        for (auto p : b) cudaFree(p);
    }
    return 0;
}
