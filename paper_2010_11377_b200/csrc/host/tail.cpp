// Dense operator of the coarse V-cycle tail (setup only).
//
// The V-cycle below a level l (its smoothing, restriction, the coarser
// levels and the coarsest solve, amg.cpp:144-168) is a fixed linear map
// r_l -> z_l.  On the coarse levels it is pure latency on the GPU: at C2,
// levels 3..5 (2205 / 347 / 52 rows) are ~10 dependent launches per V-cycle
// moving < 2 MB.  When n_l is small the map is stored as a dense n_l x n_l
// matrix B_l (columns B_l e_k, computed here by running the tail V-cycle on
// the unit vectors) and the device applies it in ONE bandwidth-bound matvec
// (k_tail_mv).  Same operator as the recursive cycle, different rounding --
// the same trade as the dense coarsest inverse in place of the reference's
// sparse LU (amg.cpp:150); the oracle applies the same B_l in the device's
// summation order, so device == oracle stays bit-exact.
#include <cstdlib>
#include <vector>

#include "setup.hpp"

namespace irkb {
namespace {

// One smoothing sweep on level `lev` (amg.cpp:115-142): damped Jacobi, or
// Gauss-Seidel forward / backward in CSR column order.
void sweep(const AmgLevel& lev, const AmgParams& p, const double* r, std::vector<double>& z,
           bool backward, std::vector<double>& az) {
    const Csr& A = lev.A;
    const int n = A.rows;
    if (p.smoother == 0) {
        spmv(A, z.data(), az.data());
        const double w = p.jacobi_weight;
        for (int i = 0; i < n; ++i) z[i] += w * lev.inv_diag[i] * (r[i] - az[i]);
        return;
    }
    auto row = [&](int i) {
        double s = r[i];
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
            if (A.idx[k] != i) s -= A.val[k] * z[A.idx[k]];
        z[i] = s * lev.inv_diag[i];
    };
    if (!backward)
        for (int i = 0; i < n; ++i) row(i);
    else
        for (int i = n - 1; i >= 0; --i) row(i);
}

void vcycle_from(const Hierarchy& h, int l, const double* r, std::vector<double>& z) {
    const AmgLevel& lev = h.levels[l];
    const int n = lev.A.rows;
    z.assign(n, 0.0);
    if (l == h.n_levels() - 1) {
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += h.coarse_inverse[static_cast<size_t>(i) * n + j] * r[j];
            z[i] = s;
        }
        return;
    }
    std::vector<double> az(n);
    for (int s = 0; s < h.params.pre_sweeps; ++s) sweep(lev, h.params, r, z, false, az);
    spmv(lev.A, z.data(), az.data());
    for (int i = 0; i < n; ++i) az[i] = r[i] - az[i];
    std::vector<double> rc(lev.R.rows), zc;
    spmv(lev.R, az.data(), rc.data());
    vcycle_from(h, l + 1, rc.data(), zc);
    std::vector<double> corr(n);
    spmv(lev.P, zc.data(), corr.data());
    for (int i = 0; i < n; ++i) z[i] += corr[i];
    for (int s = 0; s < h.params.post_sweeps; ++s) sweep(lev, h.params, r, z, true, az);
}

}  // namespace

int tail_max_rows(const AmgParams& p) {
    const char* v = std::getenv("IRK_TAIL_MAX");
    // recursive levels (Gauss-Seidel, V(pre,post) != V(1,1), IRK_COMPOSE=0) cost
    // 4+ dependent launches each: the tail starts at <= 3300 rows (B_l <= ~87
    // MB); composed levels cost two cheap launches, so there the matvec only
    // pays below 1500 rows (C2: 2205^2 -> 347^2; profiles/r2/ab_composed_vcycle.txt)
    const bool composed = compose_enabled() && p.smoother == 0 && p.pre_sweeps == 1 && p.post_sweeps == 1;
    const int n = v ? std::atoi(v) : composed ? 1500 : 3300;
    return n < 6000 ? n : 6000;             // k_tail_mv stages r in 48 KB of shared memory
}

void attach_tail(Hierarchy& h, int max_n) {
    h.tail_from = -1;
    h.tail_ld = 0;
    h.tail.clear();
    const int L = h.n_levels();
    // the first level >= 1 small enough; the coarsest alone is the dense
    // inverse already (coarse_inverse), so the tail must span >= 2 levels
    int from = -1;
    for (int l = 1; l < L - 1; ++l)
        if (h.levels[l].A.rows <= max_n) {
            from = l;
            break;
        }
    if (from < 0) return;
    const int n = h.levels[from].A.rows;
    const int ld = (n + 1) / 2 * 2;  // even row stride: 16-byte aligned double2 rows
    h.tail.assign(static_cast<size_t>(n) * ld, 0.0);
#pragma omp parallel
    {
        std::vector<double> e(n, 0.0), z;
#pragma omp for schedule(dynamic, 16)
        for (int k = 0; k < n; ++k) {
            e[k] = 1.0;
            vcycle_from(h, from, e.data(), z);
            e[k] = 0.0;
            for (int i = 0; i < n; ++i) h.tail[static_cast<size_t>(i) * ld + k] = z[i];
        }
    }
    h.tail_from = from;
    h.tail_ld = ld;
}

}  // namespace irkb
