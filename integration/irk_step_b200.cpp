// Reference-side adapter: irkprec::irk_step's signature
// (irk.hpp:36-39) forwarding to the B200 C ABI (include/irkdev.h).  This is
// the code a maintainer adds to irkprec; it includes the reference's own
// headers and is compiled against them here (integration/Makefile) so the
// drop-in is checked, not only described.  Named irk_step_b200 so that the
// demo can run it beside the reference's irk_step in one binary.
#include <functional>
#include <map>
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

}  // namespace irkprec
