// Fused coarse-level V-cycle kernels (see amg_fused.cu).
#pragma once

#include "coarse_tail.cuh"
#include "kernels.cuh"

namespace irkb {
namespace dev {

// One coarse level l (CSR operators) for the fused down / up kernels.
struct FusedLevel {
    int n = 0;                 // rows of A_l
    int nrc = 0;               // rows of A_{l+1}
    TailCsr A, P, R;
    const double* wd = nullptr;
    VecRef r{};                // level rhs
    VecRef z{};                // level solution (up)
    double* rc = nullptr;        // next level rhs (down: written)
    const double* zc = nullptr;  // next level solution (up: read)
    // down on the level above the coarsest: the last CTA applies the dense
    // coarse inverse, zcw = cinv rc (nc x nc), counter elects that CTA
    const double* cinv = nullptr;
    int nc = 0;
    double* zcw = nullptr;
    unsigned* counter = nullptr;
};

void amg_down_fused(const FusedLevel& v, cudaStream_t st);
void amg_up_fused(const FusedLevel& v, cudaStream_t st);

}  // namespace dev
}  // namespace irkb
