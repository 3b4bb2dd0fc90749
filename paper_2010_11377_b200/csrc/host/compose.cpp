// Composed V-cycle operators (setup only).
//
// One damped-Jacobi V(1,1) level of the reference cycle (amg.cpp:144-168) is
//     z  = W r                       pre-smoothing from the zero iterate
//     t  = r - A z
//     rc = R t                       restriction
//     zc = cycle(rc)
//     z += P zc                      prolongation
//     z += W (r - A z)               post-smoothing
// with W = omega * D^-1.  Both legs are fixed linear maps of (r, zc):
//     rc = G r,          G = R (I - A W)
//     z  = S r + Q zc,   S = W (I - A W) + W,   Q = P - W (A P)
// On the GPU the recursive form is four dependent kernels per level (residual,
// restriction, prolongation, smoother), each a full-grid launch with its own
// dependent-load chain; the composed form is two (`r_{l+1} = G_l r_l` going
// down, `z_l = [S_l Q_l] [r_l; z_{l+1}]` coming up) and moves fewer bytes on
// the fine level (t and the prolongated iterate are never written).  Same
// operator as the recursive cycle, different rounding -- the same trade as
// the dense coarsest inverse and the dense tail operator (tail.cpp); the
// oracle applies the same G and U in the device's row-sum order, so
// device == oracle stays bit-exact, and the composed cycle is pinned to the
// reference's amg_vcycle at 1e-12 (tests/test_oracle_vs_ref.py).
//
// Every product below is a rounded multiply and every sum a rounded add in a
// fixed order (matmul / add of sparse.cpp), so the operators are reproducible
// bit for bit from the hierarchy.
#include <array>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <set>
#include <vector>

#include "setup.hpp"

namespace irkb {

namespace {

// Lanes per row of a composed operator: about `per_lane` entries per lane
// (IRK_LT_PER_LANE10 tenths, default 6.0), a power of two <= 32.
int lanes_for(const Csr& A) {
    const char* v = std::getenv("IRK_LT_PER_LANE10");
    const double per_lane = 0.1 * (v ? std::atoi(v) : 60);
    const double avg = A.rows ? static_cast<double>(A.nnz()) / A.rows : 0.0;
    int g = 1;
    while (g < 32 && per_lane * g < avg) g *= 2;
    return g;
}

// True when the square operator S has exactly 7 distinct diagonals (the P1
// stencil of the structured fine grid) and at most 256 distinct row stencils
// (tuples of the 7 fp64 bit patterns, absent entries = 0.0): the device then
// stores S as one class byte per row, and the up leg is summed sequentially,
// one thread per row (k_up_cls).
bool stencil7_classes(const Csr& S) {
    int offs[8];
    int nd = 0;
    for (int i = 0; i < S.rows; ++i)
        for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k) {
            const int o = S.idx[k] - i;
            int q = 0;
            while (q < nd && offs[q] != o) ++q;
            if (q == nd) {
                if (nd == 7) return false;
                offs[nd++] = o;
            }
        }
    if (nd != 7) return false;
    std::set<std::array<uint64_t, 7>> seen;
    for (int i = 0; i < S.rows; ++i) {
        std::array<uint64_t, 7> t{};
        for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k) {
            const int o = S.idx[k] - i;
            int q = 0;
            while (offs[q] != o) ++q;
            std::memcpy(&t[q], &S.val[k], sizeof(uint64_t));
        }
        seen.insert(t);
        if (seen.size() > 256) return false;
    }
    return true;
}

}  // namespace

bool compose_enabled() {
    const char* v = std::getenv("IRK_COMPOSE");
    return !(v && std::atoi(v) == 0);
}

void attach_composed(Hierarchy& h) {
    for (AmgLevel& lev : h.levels) {
        lev.G = Csr{};
        lev.U = Csr{};
        lev.g_lanes = lev.u_lanes = 1;
    }
    const AmgParams& p = h.params;
    if (!compose_enabled() || p.smoother != 0 || p.pre_sweeps != 1 || p.post_sweeps != 1) return;
    const int L = h.n_levels();
    // levels at or below the dense tail are never visited by the device cycle
    const int end = h.tail_from > 0 ? h.tail_from : L - 1;
    for (int l = 0; l < end; ++l) {
        AmgLevel& lev = h.levels[l];
        const Csr& A = lev.A;
        const int n = A.rows;
        std::vector<double> wd(n);
        for (int i = 0; i < n; ++i) wd[i] = p.jacobi_weight * lev.inv_diag[i];
        // E = I - A W on A's pattern (A stores its diagonal)
        Csr E = A;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i)
            for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
                const int j = A.idx[k];
                const double aw = A.val[k] * wd[j];
                E.val[k] = j == i ? 1.0 - aw : -aw;
            }
        lev.G = matmul(lev.R, E);
        // S = W E + W on A's pattern
        Csr S = E;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i)
            for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
                const double we = wd[i] * E.val[k];
                S.val[k] = A.idx[k] == i ? we + wd[i] : we;
            }
        // Q = P - W (A P)
        Csr AP = matmul(A, lev.P);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i)
            for (int k = AP.ptr[i]; k < AP.ptr[i + 1]; ++k) AP.val[k] = wd[i] * AP.val[k];
        const Csr Q = add(1.0, lev.P, -1.0, AP);
        // U = [S | Q]: Q's columns follow S's n columns
        Csr& U = lev.U;
        U.rows = n;
        U.cols = n + Q.cols;
        U.ptr.assign(n + 1, 0);
        for (int i = 0; i < n; ++i)
            U.ptr[i + 1] = U.ptr[i] + (S.ptr[i + 1] - S.ptr[i]) + (Q.ptr[i + 1] - Q.ptr[i]);
        U.idx.resize(U.ptr[n]);
        U.val.resize(U.ptr[n]);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            int o = U.ptr[i];
            for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k, ++o) {
                U.idx[o] = S.idx[k];
                U.val[o] = S.val[k];
            }
            for (int k = Q.ptr[i]; k < Q.ptr[i + 1]; ++k, ++o) {
                U.idx[o] = n + Q.idx[k];
                U.val[o] = Q.val[k];
            }
        }
        lev.g_lanes = lanes_for(lev.G);
        lev.u_lanes = stencil7_classes(S) ? 1 : lanes_for(U);
    }
}

}  // namespace irkb
