// Drop-in demo: IRK steps of problems assembled with the
// reference's own API, solved by the reference's irk_step (CPU) and by the
// adapter irk_step_b200 (B200 through the C ABI), on the same inputs.
//
//   irk_b200_demo [cells] [s] [heat|dg] [LD|GSL|DU|J] [restart]
//       one step + a 3.5-step integrate; restart 0 (default) = full GMRES,
//       the reference's semantics.  Exit code 0 iff the iteration counts
//       agree within 1 and u_{n+1} agrees to 1e-9 relative L2 (the BASELINE
//       bar).  Prints "iterations device/reference" for the tests.
//   irk_b200_demo study
//       the reference study's run_cell pattern (study.cpp:294-332, 446, 495):
//       Butcher table and BlockPreconditioner are locals of nested loops over
//       meshes, s and preconditioner kinds, so their addresses repeat from
//       cell to cell with the same ht; every cell must still match.
// dg: the double-glazing problem (P1 SUPG, eps 0.005, East wall = 1, so the
// Dirichlet lift f_lift is non-zero; study.cpp:215-249 without forcing).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "irk_b200.hpp"
#include "irkprec/butcher.hpp"
#include "irkprec/fem.hpp"
#include "irkprec/irk.hpp"
#include "irkprec/mesh.hpp"
#include "irkprec/stage.hpp"

using namespace irkprec;

namespace {

LinearParabolicSystem make_system(int cells, bool dg) {
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
        EliminatedSystem e =
            eliminate_dirichlet(assemble_mass(space), assemble_diffusion(space, 1.0), space, {});
        sys.M = std::make_shared<const CsrMatrix>(std::move(e.M_ff));
        sys.F = std::make_shared<const CsrMatrix>(std::move(e.F_ff));
    }
    return sys;
}

std::vector<double> initial(int n, bool dg) {
    std::vector<double> u(n, 0.0);
    if (!dg)
        for (int i = 0; i < n; ++i) u[i] = std::sin(0.37 * i) * 0.5 + 0.5;  // any u_n (dg: u0 = 0)
    return u;
}

CoeffKind kind_of(const std::string& k) {
    if (k == "J") return CoeffKind::Jacobi;
    if (k == "GSL") return CoeffKind::GaussSeidelLower;
    if (k == "DU") return CoeffKind::UpperFactor;
    return CoeffKind::LowerFactor;
}

double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / den);
}

// One step through the adapter and through the reference; true if within the bar.
bool compare_step(const char* label, const LinearParabolicSystem& sys, const ButcherTable& table,
                  double ht, const std::vector<double>& u, const BlockPreconditioner& P,
                  const GmresConfig& cfg, const B200Options& opt) {
    const IrkStepResult dev = irk_step_b200(sys, table, ht, 0.0, u, &P, cfg, opt);
    const IrkStepResult ref = irk_step(sys, table, ht, 0.0, u, &P, cfg);
    const double rel = rel_l2(dev.u_next, ref.u_next);
    std::printf("%s: iterations device/reference %d/%d (%.3f ms / %.3f s), converged %d/%d, "
                "u_next rel L2 %.3e\n",
                label, dev.report.iterations, ref.report.iterations, 1e3 * dev.report.solve_seconds,
                ref.report.solve_seconds, dev.report.converged, ref.report.converged, rel);
    return std::abs(dev.report.iterations - ref.report.iterations) <= 1 && rel <= 1e-9 &&
           dev.report.converged == ref.report.converged;
}

// run_cell (study.cpp:294-332) as the study drives it: locals reused per cell.
int study() {
    bool ok = true;
    const char* kinds[] = {"LD", "DU", "GSL", "J"};
    for (int cells : {32, 48}) {
        const LinearParabolicSystem sys = make_system(cells, false);
        const std::vector<double> u = initial(sys.n(), false);
        for (int s = 2; s <= 3; ++s) {
            const ButcherTable table = make_radau_iia(s);  // study.cpp:446
            for (const char* k : kinds) {
                const BlockPreconditioner P(sys.M, sys.F, precond_coeff(table, kind_of(k)), 1e-3,
                                            SubsolverKind::AmgVcycle);  // run_cell's local P
                char label[96];
                std::snprintf(label, sizeof label, "study heat %d^2 Radau s=%d %s", cells, s, k);
                ok = compare_step(label, sys, table, 1e-3, u, P, GmresConfig{}, B200Options{}) && ok;
            }
        }
    }
    // A preconditioner built with non-default AmgParams needs them passed:
    // the adapter must refuse to solve with a different hierarchy.
    {
        const LinearParabolicSystem sys = make_system(32, false);
        const ButcherTable table = make_radau_iia(2);
        AmgParams strong;
        strong.max_coarse = 200;
        const BlockPreconditioner P(sys.M, sys.F, precond_coeff(table, CoeffKind::LowerFactor), 1e-3,
                                    SubsolverKind::AmgVcycle, strong);
        bool refused = false;
        try {
            irk_step_b200(sys, table, 1e-3, 0.0, initial(sys.n(), false), &P, GmresConfig{});
        } catch (const std::invalid_argument& e) {
            refused = true;
            std::printf("mismatched AmgParams refused: %s\n", e.what());
        }
        B200Options opt;
        opt.amg = strong;
        ok = refused && compare_step("heat 32^2 max_coarse 200 (AmgParams passed)", sys, table, 1e-3,
                                     initial(sys.n(), false), P, GmresConfig{}, opt) && ok;
    }
    // The study driver's own subsolve cycle (ExperimentConfig::amg,
    // study.hpp:44-47: Gauss-Seidel V(4,4), two prolongator smoothing steps)
    // and the Custom kind read from a coefficient file (make_coeff,
    // study.cpp:269-282), as run_cell builds them.
    {
        AmgParams study_amg;
        study_amg.pre_sweeps = 4;
        study_amg.post_sweeps = 4;
        study_amg.smoother = AmgSmoother::GaussSeidel;
        study_amg.prolongation_steps = 2;
        B200Options opt;
        opt.amg = study_amg;
        for (bool dg : {false, true}) {
            const LinearParabolicSystem sys = make_system(48, dg);
            const ButcherTable table = make_radau_iia(3);
            const double ht = dg ? 1e-2 : 1e-3;
            const BlockPreconditioner P(sys.M, sys.F, precond_coeff(table, CoeffKind::LowerFactor), ht,
                                        SubsolverKind::AmgVcycle, study_amg);
            ok = compare_step(dg ? "study cycle GS V(4,4) x2, double glazing 48^2 s=3 LD"
                                 : "study cycle GS V(4,4) x2, heat 48^2 s=3 LD",
                              sys, table, ht, initial(sys.n(), dg), P, GmresConfig{}, opt) && ok;
        }
        const char* path = "irk_b200_demo_coeff.txt";
        {
            std::FILE* f = std::fopen(path, "w");
            std::fprintf(f, "3\n0.9 0 0\n0.31 0.7 0\n-0.12 0.25 1.1\n");
            std::fclose(f);
        }
        const LinearParabolicSystem sys = make_system(48, false);
        const ButcherTable table = make_radau_iia(3);
        const BlockPreconditioner P(sys.M, sys.F, custom_coeff(read_coeff_file(path)), 1e-3,
                                    SubsolverKind::AmgVcycle);
        std::remove(path);
        ok = compare_step("custom coefficient file, heat 48^2 s=3", sys, table, 1e-3,
                          initial(sys.n(), false), P, GmresConfig{}, B200Options{}) && ok;
    }
    irk_b200_release();
    std::printf("study %s\n", ok ? "ok" : "FAILED");
    return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "study") return study();
    const int cells = argc > 1 ? std::atoi(argv[1]) : 256;
    const int s = argc > 2 ? std::atoi(argv[2]) : 3;
    const bool dg = argc > 3 && std::string(argv[3]) == "dg";
    const std::string kind = argc > 4 ? argv[4] : "LD";
    B200Options opt;
    opt.restart = argc > 5 ? std::atoi(argv[5]) : 0;
    const double ht = dg ? 1e-2 : 1e-3;
    const LinearParabolicSystem sys = make_system(cells, dg);
    const std::vector<double> u = initial(sys.n(), dg);
    const ButcherTable table = make_radau_iia(s);
    BlockPreconditioner P(sys.M, sys.F, precond_coeff(table, kind_of(kind)), ht, SubsolverKind::AmgVcycle);
    GmresConfig cfg;  // right, 1e-8, 500: the reference's defaults
    char label[96];
    std::snprintf(label, sizeof label, "%s %d^2 Radau IIA s=%d %s restart %d", dg ? "double glazing" : "heat",
                  cells, s, kind.c_str(), opt.restart);
    bool ok = compare_step(label, sys, table, ht, u, P, cfg, opt);
    // integrate: 3.5 steps of ht (a truncated last step, so the factory is
    // consulted twice), device-resident vs the reference's loop
    const PrecondFactory factory = [&](double h) {
        return std::make_shared<const BlockPreconditioner>(sys.M, sys.F, precond_coeff(table, kind_of(kind)), h,
                                                           SubsolverKind::AmgVcycle);
    };
    const double t_final = 3.5 * ht;
    const TrajectorySummary td = integrate_b200(sys, table, u, t_final, ht, factory, cfg, opt);
    const TrajectorySummary tr = integrate(sys, table, u, t_final, ht, factory, cfg);
    const double trel = rel_l2(td.u_final, tr.u_final);
    std::printf("integrate to %.4g: device %d steps (t %.6g), reference %d steps (t %.6g); iterations", t_final,
                td.steps, td.t_final, tr.steps, tr.t_final);
    bool its_ok = td.steps == tr.steps;
    for (int k = 0; k < td.steps && k < tr.steps; ++k) {
        std::printf(" %d/%d", td.reports[k].iterations, tr.reports[k].iterations);
        its_ok = its_ok && std::abs(td.reports[k].iterations - tr.reports[k].iterations) <= 1;
    }
    std::printf("; u_final rel L2 %.3e\n", trel);
    ok = ok && its_ok && trel <= 1e-9 && td.t_final == tr.t_final && td.all_converged;
    irk_b200_release();
    return ok ? 0 : 1;
}
