// Single-launch coarse tail of the V-cycle (levels >= Lc) on one thread-block
// cluster.  See coarse_tail.cu.
#pragma once

#include "kernels.cuh"

namespace irkb {
namespace dev {

constexpr int kMaxTailLevels = 8;

struct TailCsr {
    const int* ptr = nullptr;
    const int* idx = nullptr;
    const void* val = nullptr;
    const double* tab = nullptr;
    int vf = kF64;
};

struct TailLevel {
    int n = 0;
    TailCsr A, P, R;       // P, R absent on the coarsest level
    const double* wd = nullptr;
    double* r = nullptr;   // rhs (levels > 0 of the tail)
    double* z = nullptr;   // solution (levels > 0 of the tail)
    double* t = nullptr;   // residual / prolongated iterate
};

struct TailArgs {
    int nlev = 0;          // tail levels including the coarsest
    TailLevel lv[kMaxTailLevels];
    const double* cinv = nullptr;
    int nc = 0;
    VecRef r0{};           // rhs of the first tail level
    VecRef z0{};           // solution of the first tail level
};

// 0 / -1 when cluster launches are unavailable.
int coarse_tail_cluster_size();
// cluster <= 1: one CTA (bottom solver); > 1: one 16-CTA cluster.
void coarse_tail(const TailArgs& a, int cluster, cudaStream_t st);

}  // namespace dev
}  // namespace irkb
