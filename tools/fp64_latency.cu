// Microbenchmark: dependent-chain latency of DADD / DMUL / LDS on one warp
// (clock64 around 4096 dependent operations).  nvcc -arch=sm_100a -O3 --fmad=false
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
    __syncthreads();
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x - b;            // dependent DADD chain
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) y = y * b;            // dependent DMUL chain
    long long t2 = clock64();
    int idx = threadIdx.x & 1023;
    double z = 0.0;
    for (int i = 0; i < n; ++i) {                     // dependent LDS chain
        z += sm[idx];
        idx = (idx + static_cast<int>(z)) & 1023;
    }
    long long t3 = clock64();
    float f = static_cast<float>(a);
    for (int i = 0; i < n; ++i) f = f - static_cast<float>(b);  // FADD chain
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    }
    out[threadIdx.x] = x + y + z + f;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 4 * 8);
    for (int w : {32, 128, 1024}) {
        k<<<1, w>>>(out, cyc, 1.0, 1e-7, 4096);
        cudaDeviceSynchronize();
        printf("threads %4d: DADD %.1f  DMUL %.1f  LDS+DADD+cvt chain %.1f  FADD %.1f cycles/op\n", w,
               cyc[0] / 4096.0, cyc[1] / 4096.0, cyc[2] / 4096.0, cyc[3] / 4096.0);
    }
    return 0;
}
