// Shared device-side definitions for the B200 IRK solve phase.
//
// Numerics contract (what makes device == oracle bit-for-bit):
//   * every kernel is compiled with --fmad=false, so a*b+c is a rounded
//     multiply followed by a rounded add, exactly like the x86-64 oracle
//     (no FMA without -march) and the reference (proj/CMakeLists.txt:7-9);
//   * every sparse row sum is sequential in CSR column order starting from
//     0.0, the order of the reference spmv (csr.cpp:108-113);
//   * every reduction (dot, nrm2) uses the fixed tree defined by
//     kChunk / kRedThreads below, independent of grid size; the C oracle
//     (oracle/irk_oracle.c: red_chunk/red_final) emulates the same tree.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace irkb {
namespace dev {

constexpr int kRedThreads = 256;            // threads per reduction CTA
constexpr int kRedPerThread = 16;           // elements per thread per chunk
constexpr int kChunk = kRedThreads * kRedPerThread;  // 4096 elements
constexpr int kMaxStages = 7;
constexpr int kMaxRestart = 512;            // device Hessenberg capacity

// A vector that may live in a GMRES basis slot chosen at run time:
//   address = base + (slot ? (*slot + slot_add) * stride : 0) + offset
// Lets one captured CUDA graph serve every GMRES iteration (the iteration
// index is read from device memory, never baked into the graph).
struct VecRef {
    double* base;
    const int* slot;
    long long stride;
    int slot_add;
    long long offset;
    __host__ __device__ double* get() const {
        long long o = offset;
        if (slot) o += static_cast<long long>(*slot + slot_add) * stride;
        return base + o;
    }
};

inline VecRef plain(double* p) { return VecRef{p, nullptr, 0, 0, 0}; }
inline VecRef plain(const double* p) { return plain(const_cast<double*>(p)); }

#ifdef __CUDACC__
// Hypotenuse with one scaling, identical to oracle/irk_oracle.c:hyp().
__device__ __forceinline__ double hyp(double a, double b) {
    a = fabs(a);
    b = fabs(b);
    const double mx = a > b ? a : b, mn = a > b ? b : a;
    if (mx == 0.0) return 0.0;
    const double r = mn / mx;
    return mx * sqrt(1.0 + r * r);
}
#endif

}  // namespace dev
}  // namespace irkb

#define IRK_CUDA_CHECK(expr)                                                     \
    do {                                                                         \
        cudaError_t e__ = (expr);                                                \
        if (e__ != cudaSuccess)                                                  \
            throw ::irkb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e__)); \
    } while (0)

namespace irkb {

// Makes `device` current for the scope and restores the caller's device on
// exit, so that a solver on one GPU never changes (or depends on) the device
// the calling thread has selected (torch.cuda.set_device, another solver).
class DeviceScope {
public:
    explicit DeviceScope(int device) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        if (prev_ != device) {
            IRK_CUDA_CHECK(cudaSetDevice(device));
            set_ = true;
        }
    }
    ~DeviceScope() {
        if (set_ && prev_ >= 0) cudaSetDevice(prev_);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;

private:
    int prev_ = -1;
    bool set_ = false;
};

}  // namespace irkb
