// Drop-in demo: one IRK step of the heat problem assembled
// with the reference's own API, solved by the reference's irk_step (CPU) and
// by the adapter irk_step_b200 (B200 through the C ABI), on the same inputs.
// Exit code 0 iff the iteration counts agree within 1 and u_{n+1} agrees to
// 1e-9 relative L2 (the BASELINE bar).   usage: irk_b200_demo [cells] [s]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "irkprec/butcher.hpp"
#include "irkprec/fem.hpp"
#include "irkprec/irk.hpp"
#include "irkprec/mesh.hpp"
#include "irkprec/stage.hpp"

namespace irkprec {
IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg);
}

int main(int argc, char** argv) {
    using namespace irkprec;
    const int cells = argc > 1 ? std::atoi(argv[1]) : 256;
    const int s = argc > 2 ? std::atoi(argv[2]) : 3;
    const double ht = 1e-3;
    const Mesh2D mesh = build_structured_mesh(Domain::UnitSquare, cells);
    const FemSpace space = make_space(mesh, 1);
    EliminatedSystem e = eliminate_dirichlet(assemble_mass(space), assemble_diffusion(space, 1.0), space, {});
    LinearParabolicSystem sys;
    sys.M = std::make_shared<const CsrMatrix>(std::move(e.M_ff));
    sys.F = std::make_shared<const CsrMatrix>(std::move(e.F_ff));
    const int n = sys.n();
    std::vector<double> u(n);
    for (int i = 0; i < n; ++i) u[i] = std::sin(0.37 * i) * 0.5 + 0.5;  // any u_n
    const ButcherTable table = make_radau_iia(s);
    BlockPreconditioner P(sys.M, sys.F, precond_coeff(table, CoeffKind::LowerFactor), ht,
                          SubsolverKind::AmgVcycle);
    GmresConfig cfg;  // right, 1e-8, 500 (the adapter restarts at 50, as BASELINE)
    const IrkStepResult dev = irk_step_b200(sys, table, ht, 0.0, u, &P, cfg);
    const IrkStepResult ref = irk_step(sys, table, ht, 0.0, u, &P, cfg);
    double num = 0.0, den = 0.0;
    for (int i = 0; i < n; ++i) {
        num += (dev.u_next[i] - ref.u_next[i]) * (dev.u_next[i] - ref.u_next[i]);
        den += ref.u_next[i] * ref.u_next[i];
    }
    const double rel = std::sqrt(num / den);
    std::printf("heat %d^2 Radau IIA s=%d: device %d iterations (%.3f ms), reference %d iterations (%.3f s), "
                "u_next rel L2 %.3e\n", cells, s, dev.report.iterations, 1e3 * dev.report.solve_seconds,
                ref.report.iterations, ref.report.solve_seconds, rel);
    const bool ok = std::abs(dev.report.iterations - ref.report.iterations) <= 1 && rel <= 1e-9 &&
                    dev.report.converged;
    return ok ? 0 : 1;
}
