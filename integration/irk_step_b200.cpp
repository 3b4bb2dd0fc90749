// Reference-side adapter: irkprec::irk_step's signature
// (irk.hpp:36-39) forwarding to the B200 C ABI (include/irkdev.h).  This is
// the code a maintainer adds to irkprec; it includes the reference's own
// headers and is compiled against them here (integration/Makefile) so the
// drop-in is checked, not only described.  Named irk_step_b200 so that the
// demo can run it beside the reference's irk_step in one binary.
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "irkdev.h"
#include "irkprec/irk.hpp"
#include "irkprec/stage.hpp"

namespace irkprec {
namespace {

[[noreturn]] void rethrow(int st) {
    const std::string m = irk_last_error();
    if (st == IRK_EINVAL) throw std::invalid_argument(m);
    if (st == IRK_ESINGULAR) throw SingularError(m);
    if (st == IRK_ENUMERICAL) throw NumericalError(m);
    throw std::runtime_error(m);  // IRK_ECUDA / IRK_EUNSUPPORTED / internal
}

irk_csr view(const CsrMatrix& A) {
    return irk_csr{A.n_rows, A.n_cols, A.nnz(), A.row_ptr.data(), A.col_idx.data(), A.vals.data()};
}

int forward_forcing(double t, double* out, int n, void* user) {
    const Vec f = (*static_cast<const std::function<Vec(double)>*>(user))(t);
    if (static_cast<int>(f.size()) != n) return 1;
    std::copy(f.begin(), f.end(), out);
    return 0;
}

}  // namespace

IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg) {
    require(P != nullptr, "irk_step (B200): needs a preconditioner");
    require(static_cast<int>(u_n.size()) == sys.n(), "irk_step: u_n size mismatch");
    // one device solver per (preconditioner, table, step size); uploaded once
    static thread_local std::map<std::pair<const BlockPreconditioner*, const void*>, std::pair<double, irkdev*>>
        cache;
    auto& entry = cache[{P, &table}];
    if (!entry.second || entry.first != ht) {
        if (entry.second) irkdev_destroy(entry.second);
        entry.second = nullptr;
        const irk_csr M = view(*sys.M), K = view(*sys.F);
        irk_amg_params amg;
        irk_amg_params_default(&amg);  // library-default AmgParams (amg.hpp:14-29)
        const PrecondCoeff& c = P->coeff();
        irkdev* d = nullptr;
        if (int st = irkdev_create(&M, &K, table.s, table.A.values.data(), table.b.data(),
                                   c.Atilde.values.data(), static_cast<int>(c.structure), ht, &amg,
                                   /*n_hier=*/0, nullptr, /*device=*/0, &d))
            rethrow(st);
        entry = {ht, d};
    }
    irk_gmres_cfg g{cfg.side == PrecondSide::Left ? 0 : 1, cfg.rel_tol, cfg.max_iter, /*restart=*/50};
    IrkStepResult out;
    out.u_next.resize(u_n.size());
    std::vector<double> hist(cfg.max_iter + 1);
    irk_report rep;
    const double* lift = sys.f_lift.empty() ? nullptr : sys.f_lift.data();
    if (int st = irkdev_step_forced(entry.second, u_n.data(), lift, t_n, table.c.data(),
                                    sys.forcing ? forward_forcing : nullptr,
                                    const_cast<std::function<Vec(double)>*>(&sys.forcing), &g,
                                    out.u_next.data(), nullptr, &rep, hist.data()))
        rethrow(st);
    out.report.iterations = rep.iterations;
    out.report.history.assign(hist.begin(), hist.begin() + rep.history_len);
    out.report.final_rel_residual = rep.final_rel_residual;
    out.report.true_rel_residual = rep.true_rel_residual;
    out.report.converged = rep.converged != 0;
    out.report.solve_seconds = rep.solve_seconds;
    return out;
}

namespace {

// What the PrecondFactory callback needs: the system, the table, the
// reference's factory, and ownership of what it produced.
struct IntegrateCtx {
    const LinearParabolicSystem* sys;
    const ButcherTable* table;
    const PrecondFactory* make;
    std::vector<std::shared_ptr<const BlockPreconditioner>> keep;
    std::vector<irkdev*> made;
    std::string err;
};

// One device solver for step size h from the reference's factory.
irkdev* make_device(double h, void* user) {
    IntegrateCtx& c = *static_cast<IntegrateCtx*>(user);
    auto P = (*c.make)(h);
    const irk_csr M = view(*c.sys->M), K = view(*c.sys->F);
    irk_amg_params amg;
    irk_amg_params_default(&amg);
    const PrecondCoeff& pc = P->coeff();
    irkdev* d = nullptr;
    if (irkdev_create(&M, &K, c.table->s, c.table->A.values.data(), c.table->b.data(),
                      pc.Atilde.values.data(), static_cast<int>(pc.structure), h, &amg, 0, nullptr, 0,
                      &d) != IRK_OK) {
        c.err = irk_last_error();
        return nullptr;
    }
    c.keep.push_back(std::move(P));
    c.made.push_back(d);
    return d;
}

}  // namespace

// integrate (irk.hpp:54-58) on the device: u stays in HBM across the steps;
// the PrecondFactory is consulted exactly when the reference consults it (the
// first step size and a truncated last step), each preconditioner it returns
// becoming one device solver.
TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg) {
    require(static_cast<int>(u0.size()) == sys.n(), "integrate: u0 size mismatch");
    IntegrateCtx ctx{&sys, &table, &make_precond, {}, {}, {}};
    irkdev* first = make_device(ht, &ctx);
    if (!first) throw std::runtime_error(ctx.err);
    int nsteps = 0;
    if (int st = irk_integrate_steps(t_final, ht, &nsteps)) rethrow(st);
    irk_gmres_cfg g{cfg.side == PrecondSide::Left ? 0 : 1, cfg.rel_tol, cfg.max_iter, /*restart=*/50};
    TrajectorySummary out;
    out.u_final.resize(u0.size());
    std::vector<irk_report> reps(nsteps);
    std::vector<double> hist(static_cast<size_t>(nsteps) * (cfg.max_iter + 1));
    int steps = 0, all = 0;
    double t_out = 0.0;
    const double* lift = sys.f_lift.empty() ? nullptr : sys.f_lift.data();
    const int st = irkdev_integrate(first, make_device, &ctx, u0.data(), lift, table.c.data(),
                                    sys.forcing ? forward_forcing : nullptr,
                                    const_cast<std::function<Vec(double)>*>(&sys.forcing), t_final, ht, &g,
                                    out.u_final.data(), reps.data(), nsteps, hist.data(), &steps, &t_out, &all);
    for (irkdev* d : ctx.made) irkdev_destroy(d);
    if (st) rethrow(st);
    out.t_final = t_out;
    out.steps = steps;
    out.all_converged = all != 0;
    for (int k = 0; k < steps; ++k) {
        SolveReport r;
        r.iterations = reps[k].iterations;
        const double* h0 = hist.data() + static_cast<size_t>(k) * (cfg.max_iter + 1);
        r.history.assign(h0, h0 + reps[k].history_len);
        r.final_rel_residual = reps[k].final_rel_residual;
        r.true_rel_residual = reps[k].true_rel_residual;
        r.converged = reps[k].converged != 0;
        r.solve_seconds = reps[k].solve_seconds;
        out.reports.push_back(std::move(r));
    }
    return out;
}

}  // namespace irkprec
