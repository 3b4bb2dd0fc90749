// Drop-in demo: one IRK step of the heat problem assembled
// with the reference's own API, solved by the reference's irk_step (CPU) and
// by the adapter irk_step_b200 (B200 through the C ABI), on the same inputs.
// Exit code 0 iff the iteration counts agree within 1 and u_{n+1} agrees to
// 1e-9 relative L2 (the BASELINE bar).
//   usage: irk_b200_demo [cells] [s] [heat|dg]
// dg: the double-glazing problem (P1 SUPG, eps 0.005, East wall = 1, so the
// Dirichlet lift f_lift is non-zero; study.cpp:215-249 without forcing).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
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
TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg);
}

int main(int argc, char** argv) {
    using namespace irkprec;
    const int cells = argc > 1 ? std::atoi(argv[1]) : 256;
    const int s = argc > 2 ? std::atoi(argv[2]) : 3;
    const bool dg = argc > 3 && std::string(argv[3]) == "dg";
    const double ht = dg ? 1e-2 : 1e-3;
    LinearParabolicSystem sys;
    if (dg) {
        const Mesh2D mesh = build_structured_mesh(Domain::BiUnitSquare, cells);
        const FemSpace space = make_space(mesh, 1);
        SupgMatrices supg = assemble_advection_supg(space, make_double_glazing_wind(), 0.005);
        WallValues walls;
        walls.east = 1.0;
        EliminatedSystem e = eliminate_dirichlet(supg.M, supg.F, space, walls);
        sys.M = std::make_shared<const CsrMatrix>(std::move(e.M_ff));
        sys.F = std::make_shared<const CsrMatrix>(std::move(e.F_ff));
        sys.f_lift = std::move(e.f_lift);
    } else {
        const Mesh2D mesh = build_structured_mesh(Domain::UnitSquare, cells);
        const FemSpace space = make_space(mesh, 1);
        EliminatedSystem e = eliminate_dirichlet(assemble_mass(space), assemble_diffusion(space, 1.0), space, {});
        sys.M = std::make_shared<const CsrMatrix>(std::move(e.M_ff));
        sys.F = std::make_shared<const CsrMatrix>(std::move(e.F_ff));
    }
    const int n = sys.n();
    std::vector<double> u(n, 0.0);
    if (!dg)
        for (int i = 0; i < n; ++i) u[i] = std::sin(0.37 * i) * 0.5 + 0.5;  // any u_n (dg: u0 = 0)
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
    std::printf("%s %d^2 Radau IIA s=%d: device %d iterations (%.3f ms), reference %d iterations (%.3f s), "
                "u_next rel L2 %.3e\n", dg ? "double glazing" : "heat", cells, s, dev.report.iterations, 1e3 * dev.report.solve_seconds,
                ref.report.iterations, ref.report.solve_seconds, rel);
    bool ok = std::abs(dev.report.iterations - ref.report.iterations) <= 1 && rel <= 1e-9 &&
              dev.report.converged;
    // integrate: 3.5 steps of ht (a truncated last step, so the factory is
    // consulted twice), device-resident vs the reference's loop
    const PrecondFactory factory = [&](double h) {
        return std::make_shared<const BlockPreconditioner>(sys.M, sys.F, precond_coeff(table, CoeffKind::LowerFactor),
                                                           h, SubsolverKind::AmgVcycle);
    };
    const double t_final = 3.5 * ht;
    const TrajectorySummary td = integrate_b200(sys, table, u, t_final, ht, factory, cfg);
    const TrajectorySummary tr = integrate(sys, table, u, t_final, ht, factory, cfg);
    num = den = 0.0;
    for (int i = 0; i < n; ++i) {
        num += (td.u_final[i] - tr.u_final[i]) * (td.u_final[i] - tr.u_final[i]);
        den += tr.u_final[i] * tr.u_final[i];
    }
    const double trel = std::sqrt(num / den);
    std::printf("integrate to %.4g: device %d steps (t %.6g), reference %d steps (t %.6g); iterations", t_final,
                td.steps, td.t_final, tr.steps, tr.t_final);
    bool its_ok = td.steps == tr.steps;
    for (int k = 0; k < td.steps && k < tr.steps; ++k) {
        std::printf(" %d/%d", td.reports[k].iterations, tr.reports[k].iterations);
        its_ok = its_ok && std::abs(td.reports[k].iterations - tr.reports[k].iterations) <= 1;
    }
    std::printf("; u_final rel L2 %.3e\n", trel);
    ok = ok && its_ok && trel <= 1e-9 && td.t_final == tr.t_final && td.all_converged;
    return ok ? 0 : 1;
}
