// Host setup of the IRK stage system: the inputs the device solve phase is
// built from.  Everything here runs once per problem/preconditioner and is
// outside the timed solve (SURVEY.md §8d "Unit of work").
//
//  * P1 finite elements on the structured SW-NE triangulation: heat
//    (mass + stiffness) and the double-glazing SUPG pair, with strong
//    Dirichlet elimination and lifting
//    (reference: mesh.cpp:17-51, fem.cpp:139-164, 174-304, 315-379).
//  * Butcher tables (Radau IIA s=1..7, Lobatto IIIC s=2..5), pivot-free LDU
//    and the preconditioner coefficient kinds (butcher.cpp:29-101, 190-288).
//  * Smoothed-aggregation AMG setup with the reference's coarsening
//    (amg.cpp:15-227), plus the dense inverse of the coarsest operator used
//    by the device coarse solve.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "sparse.hpp"

namespace irkb {

// ------------------------------------------------------------------ FE
struct Problem {
    Csr M, K;                  // free-dof mass and stiffness (K = F)
    std::vector<double> f_lift;  // (K g) on the free dofs
    std::vector<std::array<double, 2>> coords;  // free-dof coordinates
    int cells = 0;
};

// Heat u_t = Δu on [0,1]^2, zero Dirichlet, no forcing.
Problem make_heat_problem(int cells);
// Double glazing on [-1,1]^2 with `cells` cells per side, P1 SUPG, East = 1
// (study.cpp:215-249 with manufactured = false).
Problem make_double_glazing_problem(int cells, double eps);
// u0 = sin(pi x) sin(pi y) + U[-amp, amp] at free nodes; noise from a
// splitmix64 stream seeded with `seed` (project-defined, shared by every arm).
std::vector<double> heat_initial(const Problem& p, double noise_amp,
                                 unsigned long long seed);

// ------------------------------------------------------------------ Butcher
enum class Scheme { RadauIIA = 0, LobattoIIIC = 1 };
enum class CoeffKind { Jacobi = 0, GaussSeidelLower = 1, UpperFactor = 2,
                       LowerFactor = 3, Custom = 4 };
enum class Structure { Diagonal = 0, Lower = 1, Upper = 2 };

struct Tableau {
    int s = 0, q = 0;
    std::vector<double> A, b, c;  // A row-major s*s
};
Tableau radau_iia(int s);
Tableau lobatto_iiic(int s);
Tableau make_tableau(Scheme scheme, int s);

struct Ldu {
    std::vector<double> L, D, U;
};
Ldu ldu_factorize(int s, const std::vector<double>& A);

struct Coeff {
    std::vector<double> At;  // row-major s*s
    Structure structure = Structure::Diagonal;
};
Coeff precond_coeff(const Tableau& t, CoeffKind kind);
Coeff custom_coeff(int s, const std::vector<double>& At);
// read_coeff_file (butcher.cpp:300-313): "s" then s*s row-major values,
// whitespace separated, parsed with the same stream extraction; IoError on a
// missing file, a bad stage count or truncated data.  Returns At, sets s.
std::vector<double> read_coeff_file(const std::string& path, int& s);
// make_coeff (study.cpp:269-282): precond_coeff for the built-in kinds; for
// Custom, read_coeff_file(custom_path), its size checked against t.s, then
// custom_coeff.
Coeff make_coeff(const Tableau& t, CoeffKind kind, const std::string& custom_path);

// ------------------------------------------------------------------ AMG
struct AmgParams {
    double theta = 0.25;
    int pre_sweeps = 1, post_sweeps = 1;
    int smoother = 0;  // 0 damped Jacobi (the only device smoother)
    double jacobi_weight = 2.0 / 3.0;
    double prolongation_weight = 4.0 / 3.0;
    int prolongation_steps = 1;
    int max_coarse = 64;
    int max_levels = 10;
};

struct AmgLevel {
    Csr A;
    std::vector<double> inv_diag;
    Csr P, R;  // empty on the coarsest level
    // Composed Jacobi V(1,1) legs (compose.cpp): r_{l+1} = G r_l going down,
    // z_l = U [r_l; z_{l+1}] coming up (U = [S | Q], Q's columns offset by
    // A.rows); empty when the level is not composed.
    Csr G, U;
    // Row-sum association of G and U (part of their definition, shared with
    // the oracle): L lanes, lane q adds the row's entries q, q+L, q+2L, ...
    // in order from 0.0, then the lanes are folded by the xor butterfly
    // L/2, ..., 1.  L = 1 is the sequential CSR row sum.
    int g_lanes = 1, u_lanes = 1;
};

struct Hierarchy {
    std::vector<AmgLevel> levels;
    std::vector<double> coarse_inverse;  // dense row-major n_L x n_L
    AmgParams params;
    // Dense operator of the V-cycle below level tail_from (tail.cpp): row-major
    // n x tail_ld (n = levels[tail_from].A.rows, tail_ld = n rounded up to
    // even); tail_from = -1 when no level is small enough.
    int tail_from = -1, tail_ld = 0;
    std::vector<double> tail;
    int n_levels() const { return static_cast<int>(levels.size()); }
};

Hierarchy amg_setup(const Csr& A, const AmgParams& p);
// Attaches the dense tail operator B_l for the first level l >= 1 (above the
// coarsest) with at most max_n rows (tail.cpp); amg_setup and
// amg_setup_device call it with tail_max_rows(params) (IRK_TAIL_MAX; default 1500
// rows for composed hierarchies, 3300 for recursive ones;
// 0 disables).
void attach_tail(Hierarchy& h, int max_n);
int tail_max_rows(const AmgParams& p);
bool compose_enabled();  // IRK_COMPOSE != 0
// Attaches the composed operators G_l, U_l of every level above the tail (or
// the coarsest level) for damped-Jacobi V(1,1) hierarchies (compose.cpp);
// amg_setup and amg_setup_device call it after attach_tail.  IRK_COMPOSE=0
// in the environment disables it.
void attach_composed(Hierarchy& h);
// Dense inverse of the coarsest operator (Gauss-Jordan, partial pivoting).
std::vector<double> dense_inverse_host(const Csr& A);

// Distinct diagonal coefficients by exact equality (stage.cpp:85-97):
// block j uses hierarchy solver_of_block[j], built for distinct[k].
void distinct_diagonals(int s, const std::vector<double>& At,
                        std::vector<int>& solver_of_block,
                        std::vector<double>& distinct);

}  // namespace irkb
