// Reference-side adapter: irkprec::irk_step's signature
// (irk.hpp:36-39) forwarding to the B200 C ABI (include/irkdev.h).  This is
// the code a maintainer adds to irkprec; it includes the reference's own
// headers and is compiled against them here (integration/Makefile) so the
// drop-in is checked, not only described.  Named irk_step_b200 so that the
// demo can run it beside the reference's irk_step in one binary.
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "irk_b200.hpp"
#include "irkdev.h"
#include "irkprec/amg.hpp"
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

namespace {

// Device solvers, reused across calls on identical inputs.  The key is the
// CONTENT of everything that defines the device solver -- table A, b, c;
// P's Atilde, structure and subsolver; ht; the AmgParams; the device -- plus
// the identity of the (immutable, shared_ptr-owned) M and F, which every
// entry pins by holding their shared_ptrs, so a freed matrix's address can
// never alias a cached one.  A small LRU bounds device memory (a C2 solver
// holds ~2.6 GB): IRK_B200_CACHE entries, default 4.
struct SolverKey {
    const CsrMatrix* M;
    const CsrMatrix* F;
    std::vector<double> nums;  // A, b, c, Atilde, ht, AmgParams (doubles)
    std::vector<int> ints;     // s, structure, subsolver, AmgParams (ints), device
    bool operator==(const SolverKey& o) const {
        return M == o.M && F == o.F && ints == o.ints && nums.size() == o.nums.size() &&
               std::memcmp(nums.data(), o.nums.data(), sizeof(double) * nums.size()) == 0;
    }
};

struct CacheEntry {
    SolverKey key;
    std::shared_ptr<const CsrMatrix> M, F;  // pinned: keeps the key's addresses unique
    irkdev* d = nullptr;
};

struct SolverCache {
    std::list<CacheEntry> lru;  // most recent first
    ~SolverCache() { clear(); }
    void clear() {
        for (CacheEntry& e : lru) irkdev_destroy(e.d);
        lru.clear();
    }
    static std::size_t capacity() {
        const char* v = std::getenv("IRK_B200_CACHE");
        const long c = v ? std::strtol(v, nullptr, 10) : 4;
        return c < 1 ? 1 : static_cast<std::size_t>(c);
    }
};

SolverCache& solver_cache() {
    static thread_local SolverCache c;
    return c;
}

SolverKey make_key(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                   const BlockPreconditioner& P, const B200Options& opt) {
    SolverKey k{sys.M.get(), sys.F.get(), {}, {}};
    const PrecondCoeff& c = P.coeff();
    k.nums.insert(k.nums.end(), table.A.values.begin(), table.A.values.end());
    k.nums.insert(k.nums.end(), table.b.begin(), table.b.end());
    k.nums.insert(k.nums.end(), table.c.begin(), table.c.end());
    k.nums.insert(k.nums.end(), c.Atilde.values.begin(), c.Atilde.values.end());
    const AmgParams& a = opt.amg;
    k.nums.insert(k.nums.end(), {ht, a.theta, a.jacobi_weight, a.prolongation_weight});
    k.ints = {table.s, static_cast<int>(c.structure), static_cast<int>(P.subsolver()), a.pre_sweeps,
              a.post_sweeps, static_cast<int>(a.smoother), a.prolongation_steps, a.max_coarse,
              a.max_levels, opt.device};
    return k;
}

irk_amg_params to_c(const AmgParams& a) {
    irk_amg_params p;
    irk_amg_params_default(&p);
    p.theta = a.theta;
    p.pre_sweeps = a.pre_sweeps;
    p.post_sweeps = a.post_sweeps;
    p.smoother = a.smoother == AmgSmoother::GaussSeidel ? 1 : 0;
    p.jacobi_weight = a.jacobi_weight;
    p.prolongation_weight = a.prolongation_weight;
    p.prolongation_steps = a.prolongation_steps;
    p.max_coarse = a.max_coarse;
    p.max_levels = a.max_levels;
    return p;
}

// The device hierarchies must be the ones P built (same AmgParams): level
// count, level sizes and operator complexity per distinct subsolver.
void check_hierarchies(irkdev* d, const BlockPreconditioner& P) {
    int n_hier = 0;
    if (int st = irkdev_info(d, nullptr, nullptr, &n_hier, nullptr, nullptr)) rethrow(st);
    const std::vector<AmgStats>& ref = P.hierarchy_stats();
    bool same = static_cast<int>(ref.size()) == n_hier;
    for (int k = 0; same && k < n_hier; ++k) {
        const int nl = irkdev_num_levels(d, k);
        same = nl == ref[k].levels && static_cast<int>(ref[k].sizes.size()) == nl;
        double nnz = 0.0, nnz0 = 0.0;
        for (int l = 0; same && l < nl; ++l) {
            int n = 0, nA = 0, nP = 0, nR = 0;
            if (int st = irkdev_level_info(d, k, l, &n, &nA, &nP, &nR, nullptr)) rethrow(st);
            same = n == ref[k].sizes[l];
            nnz += nA;
            if (l == 0) nnz0 = nA;
        }
        same = same && nnz / nnz0 == ref[k].operator_complexity;
    }
    if (!same)
        throw std::invalid_argument(
            "irk_step (B200): the device AMG hierarchies differ from the preconditioner's; "
            "pass the AmgParams P was built with in B200Options::amg");
}

irkdev* device_solver(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                      const BlockPreconditioner& P, const B200Options& opt) {
    SolverCache& cache = solver_cache();
    SolverKey key = make_key(sys, table, ht, P, opt);
    for (auto it = cache.lru.begin(); it != cache.lru.end(); ++it)
        if (it->key == key) {
            cache.lru.splice(cache.lru.begin(), cache.lru, it);
            return it->d;
        }
    const irk_csr M = view(*sys.M), K = view(*sys.F);
    const irk_amg_params amg = to_c(opt.amg);
    const PrecondCoeff& c = P.coeff();
    irkdev* d = nullptr;
    if (int st = irkdev_create(&M, &K, table.s, table.A.values.data(), table.b.data(),
                               c.Atilde.values.data(), static_cast<int>(c.structure), ht, &amg,
                               /*n_hier=*/0, nullptr, opt.device, &d))
        rethrow(st);
    try {
        check_hierarchies(d, P);
    } catch (...) {
        irkdev_destroy(d);
        throw;
    }
    while (cache.lru.size() >= SolverCache::capacity()) {
        irkdev_destroy(cache.lru.back().d);
        cache.lru.pop_back();
    }
    cache.lru.push_front(CacheEntry{std::move(key), sys.M, sys.F, d});
    return d;
}

}  // namespace

// Releases every cached device solver of the calling thread.
void irk_b200_release() { solver_cache().clear(); }

IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg, const B200Options& opt) {
    require(P != nullptr, "irk_step (B200): needs a preconditioner");
    require(static_cast<int>(u_n.size()) == sys.n(), "irk_step: u_n size mismatch");
    require(P->stages() == table.s && P->block_size() == sys.n(),
            "irk_step (B200): preconditioner does not match the system");
    if (P->subsolver() != SubsolverKind::AmgVcycle)
        throw std::invalid_argument("irk_step (B200): only the AmgVcycle subsolver runs on the device "
                                    "(ExactLU is the reference's analysis path)");
    irkdev* d = device_solver(sys, table, ht, *P, opt);
    irk_gmres_cfg g{cfg.side == PrecondSide::Left ? 0 : 1, cfg.rel_tol, cfg.max_iter, opt.restart};
    IrkStepResult out;
    out.u_next.resize(u_n.size());
    std::vector<double> hist(cfg.max_iter + 1);
    irk_report rep;
    const double* lift = sys.f_lift.empty() ? nullptr : sys.f_lift.data();
    if (int st = irkdev_step_forced(d, u_n.data(), lift, t_n, table.c.data(),
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

// The reference's exact signature (irk.hpp:36-39): full GMRES, library-default
// AmgParams, device 0.
IrkStepResult irk_step_b200(const LinearParabolicSystem& sys, const ButcherTable& table, double ht,
                            double t_n, std::span<const double> u_n, const BlockPreconditioner* P,
                            const GmresConfig& cfg) {
    return irk_step_b200(sys, table, ht, t_n, u_n, P, cfg, B200Options{});
}

namespace {

// What the PrecondFactory callback needs: the system, the table, the
// reference's factory, and ownership of what it produced.
struct IntegrateCtx {
    const LinearParabolicSystem* sys;
    const ButcherTable* table;
    const PrecondFactory* make;
    B200Options opt;
    std::vector<std::shared_ptr<const BlockPreconditioner>> keep;
    std::vector<irkdev*> made;
    std::string err;
};

// One device solver for step size h from the reference's factory.
irkdev* make_device(double h, void* user) {
    IntegrateCtx& c = *static_cast<IntegrateCtx*>(user);
    irkdev* d = nullptr;
    try {
        auto P = (*c.make)(h);
        if (P->subsolver() != SubsolverKind::AmgVcycle)
            throw std::invalid_argument("integrate (B200): only the AmgVcycle subsolver runs on the device");
        const irk_csr M = view(*c.sys->M), K = view(*c.sys->F);
        const irk_amg_params amg = to_c(c.opt.amg);
        const PrecondCoeff& pc = P->coeff();
        if (int st = irkdev_create(&M, &K, c.table->s, c.table->A.values.data(), c.table->b.data(),
                                   pc.Atilde.values.data(), static_cast<int>(pc.structure), h, &amg, 0,
                                   nullptr, c.opt.device, &d))
            rethrow(st);
        c.made.push_back(d);
        check_hierarchies(d, *P);
        c.keep.push_back(std::move(P));
    } catch (const std::exception& e) {
        c.err = e.what();
        return nullptr;
    }
    return d;
}

}  // namespace

// integrate (irk.hpp:54-58) on the device: u stays in HBM across the steps;
// the PrecondFactory is consulted exactly when the reference consults it (the
// first step size and a truncated last step), each preconditioner it returns
// becoming one device solver.
TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg,
                                 const B200Options& opt) {
    require(static_cast<int>(u0.size()) == sys.n(), "integrate: u0 size mismatch");
    IntegrateCtx ctx{&sys, &table, &make_precond, opt, {}, {}, {}};
    irkdev* first = make_device(ht, &ctx);
    if (!first) {
        for (irkdev* d : ctx.made) irkdev_destroy(d);
        throw std::runtime_error(ctx.err);
    }
    int nsteps = 0;
    if (int st = irk_integrate_steps(t_final, ht, &nsteps)) rethrow(st);
    irk_gmres_cfg g{cfg.side == PrecondSide::Left ? 0 : 1, cfg.rel_tol, cfg.max_iter, opt.restart};
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

TrajectorySummary integrate_b200(const LinearParabolicSystem& sys, const ButcherTable& table,
                                 std::span<const double> u0, double t_final, double ht,
                                 const PrecondFactory& make_precond, const GmresConfig& cfg) {
    return integrate_b200(sys, table, u0, t_final, ht, make_precond, cfg, B200Options{});
}

}  // namespace irkprec
