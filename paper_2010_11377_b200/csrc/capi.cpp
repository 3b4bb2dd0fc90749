// C ABI (include/irkdev.h): exception -> status mapping and thin marshalling.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/irkdev.h"
#include "device/amg_device.hpp"
#include "device/solver.hpp"
#include "host/mmio.hpp"
#include "host/setup.hpp"

struct irk_problem {
    irkb::Problem p;
};
struct irk_hierarchy {
    irkb::Hierarchy h;
};
struct irkdev {
    std::unique_ptr<irkb::DeviceSolver> s;
};
struct irk_matrix {
    irkb::Csr a;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return IRK_OK;
    } catch (const irkb::InvalidArgument& e) {
        g_err = e.what();
        return IRK_EINVAL;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return IRK_EINVAL;
    } catch (const irkb::SingularError& e) {
        g_err = e.what();
        return IRK_ESINGULAR;
    } catch (const irkb::NumericalError& e) {
        g_err = e.what();
        return IRK_ENUMERICAL;
    } catch (const irkb::CudaError& e) {
        g_err = e.what();
        return IRK_ECUDA;
    } catch (const irkb::Unsupported& e) {
        g_err = e.what();
        return IRK_EUNSUPPORTED;
    } catch (const irkb::IoError& e) {
        g_err = e.what();
        return IRK_EIO;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return IRK_EINTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return IRK_EINTERNAL;
    }
}

irkb::Csr to_csr(const irk_csr* v) {
    irkb::check(v && v->row_ptr && v->n_rows >= 0 && v->n_cols >= 0, "csr: null or negative view");
    irkb::Csr A;
    A.rows = v->n_rows;
    A.cols = v->n_cols;
    A.ptr.assign(v->row_ptr, v->row_ptr + v->n_rows + 1);
    irkb::check(A.ptr.back() == v->nnz, "csr: row_ptr[n] != nnz");
    A.idx.assign(v->col_idx, v->col_idx + v->nnz);
    A.val.assign(v->vals, v->vals + v->nnz);
    A.validate();
    return A;
}

void view(const irkb::Csr& A, irk_csr* out) {
    out->n_rows = A.rows;
    out->n_cols = A.cols;
    out->nnz = A.nnz();
    out->row_ptr = A.ptr.data();
    out->col_idx = A.idx.data();
    out->vals = A.val.data();
}

irkb::AmgParams to_params(const irk_amg_params* p) {
    irkb::AmgParams q;
    if (!p) return q;
    q.theta = p->theta;
    q.pre_sweeps = p->pre_sweeps;
    q.post_sweeps = p->post_sweeps;
    q.smoother = p->smoother;
    q.jacobi_weight = p->jacobi_weight;
    q.prolongation_weight = p->prolongation_weight;
    q.prolongation_steps = p->prolongation_steps;
    q.max_coarse = p->max_coarse;
    q.max_levels = p->max_levels;
    return q;
}

void fill_report(const irkb::SolveReport& r, double setup, irk_report* rep, double* history) {
    if (rep) {
        rep->iterations = r.iterations;
        rep->cycles = r.cycles;
        rep->n_reorth = r.n_reorth;
        rep->converged = r.converged;
        rep->final_rel_residual = r.final_rel;
        rep->true_rel_residual = r.true_rel;
        rep->solve_seconds = r.solve_seconds;
        rep->setup_seconds = setup;
        rep->history_len = static_cast<int>(r.history.size());
    }
    if (history) std::memcpy(history, r.history.data(), sizeof(double) * r.history.size());
}

// The reference time loop's step sizes (irk.cpp:85-99): ht repeated, the
// last one truncated to land on t_final.
std::vector<double> integrate_plan(double t_final, double ht) {
    std::vector<double> plan;
    double t = 0.0;
    while (t < t_final - 1e-14 * t_final) {
        double step = ht;
        if (t + step > t_final) step = t_final - t;
        plan.push_back(step);
        t += step;
    }
    return plan;
}

irkb::GmresConfig to_cfg(const irk_gmres_cfg* c) {
    irkb::GmresConfig g;
    if (c) {
        g.side = c->side;
        g.rel_tol = c->rel_tol;
        g.max_iter = c->max_iter;
        g.restart = c->restart;
    }
    return g;
}

template <class F>
void with_device_vectors(irkdev* d, const double* in, long long nin, double* out, long long nout,
                         F&& f) {
    irkb::DeviceScope on(d->s->device());
    irkb::DevBuf a(sizeof(double) * nin), b(sizeof(double) * nout);
    IRK_CUDA_CHECK(cudaMemcpy(a.as<double>(), in, sizeof(double) * nin, cudaMemcpyHostToDevice));
    f(a.as<double>(), b.as<double>());
    IRK_CUDA_CHECK(cudaMemcpy(out, b.as<double>(), sizeof(double) * nout, cudaMemcpyDeviceToHost));
}

}  // namespace

extern "C" {

const char* irk_last_error(void) { return g_err.c_str(); }

void irk_amg_params_default(irk_amg_params* p) {
    const irkb::AmgParams d;
    p->theta = d.theta;
    p->pre_sweeps = d.pre_sweeps;
    p->post_sweeps = d.post_sweeps;
    p->smoother = d.smoother;
    p->jacobi_weight = d.jacobi_weight;
    p->prolongation_weight = d.prolongation_weight;
    p->prolongation_steps = d.prolongation_steps;
    p->max_coarse = d.max_coarse;
    p->max_levels = d.max_levels;
}

void irk_gmres_cfg_default(irk_gmres_cfg* c) {
    c->side = 1;
    c->rel_tol = 1e-8;
    c->max_iter = 500;
    c->restart = 0;  // full GMRES, the reference (gmres.hpp:20)
}

int irk_problem_heat(int cells, irk_problem** out) {
    return guard([&] { *out = new irk_problem{irkb::make_heat_problem(cells)}; });
}

int irk_problem_double_glazing(int cells, double eps, irk_problem** out) {
    return guard([&] { *out = new irk_problem{irkb::make_double_glazing_problem(cells, eps)}; });
}

int irk_problem_n(const irk_problem* p) { return p->p.M.rows; }

int irk_problem_matrix(const irk_problem* p, int which, irk_csr* out) {
    return guard([&] {
        irkb::check(which == 0 || which == 1, "problem matrix: which must be 0 (M) or 1 (K)");
        view(which == 0 ? p->p.M : p->p.K, out);
    });
}

const double* irk_problem_lift(const irk_problem* p) { return p->p.f_lift.data(); }

int irk_problem_initial(const irk_problem* p, double noise, unsigned long long seed, double* u0) {
    return guard([&] {
        const std::vector<double> u = irkb::heat_initial(p->p, noise, seed);
        std::memcpy(u0, u.data(), sizeof(double) * u.size());
    });
}

void irk_problem_free(irk_problem* p) { delete p; }

int irk_tableau(int scheme, int s, double* A, double* b, double* c, int* q) {
    return guard([&] {
        irkb::check(scheme == 0 || scheme == 1, "tableau: scheme must be 0 (Radau IIA) or 1 (Lobatto IIIC)");
        const irkb::Tableau t = irkb::make_tableau(static_cast<irkb::Scheme>(scheme), s);
        std::memcpy(A, t.A.data(), sizeof(double) * s * s);
        std::memcpy(b, t.b.data(), sizeof(double) * s);
        std::memcpy(c, t.c.data(), sizeof(double) * s);
        if (q) *q = t.q;
    });
}

int irk_ldu(int s, const double* A, double* L, double* D, double* U) {
    return guard([&] {
        irkb::check(s >= 1, "ldu_factorize: s >= 1");
        const irkb::Ldu f = irkb::ldu_factorize(s, std::vector<double>(A, A + s * s));
        std::memcpy(L, f.L.data(), sizeof(double) * s * s);
        std::memcpy(D, f.D.data(), sizeof(double) * s);
        std::memcpy(U, f.U.data(), sizeof(double) * s * s);
    });
}

int irk_precond_coeff(int scheme, int s, int kind, double* Atilde, int* structure) {
    return guard([&] {
        irkb::check(kind >= 0 && kind <= 4, "precond_coeff: unknown kind");
        const irkb::Tableau t = irkb::make_tableau(static_cast<irkb::Scheme>(scheme), s);
        const irkb::Coeff c = irkb::precond_coeff(t, static_cast<irkb::CoeffKind>(kind));
        std::memcpy(Atilde, c.At.data(), sizeof(double) * s * s);
        *structure = static_cast<int>(c.structure);
    });
}

int irk_custom_coeff(int s, const double* Atilde, int* structure) {
    return guard([&] {
        const irkb::Coeff c = irkb::custom_coeff(s, std::vector<double>(Atilde, Atilde + s * s));
        *structure = static_cast<int>(c.structure);
    });
}

int irk_read_coeff_file(const char* path, int cap, int* s, double* Atilde) {
    return guard([&] {
        irkb::check(path != nullptr, "read_coeff_file: null path");
        int ns = 0;
        const std::vector<double> At = irkb::read_coeff_file(path, ns);
        *s = ns;
        irkb::check(Atilde == nullptr || cap >= ns * ns, "read_coeff_file: output buffer too small");
        if (Atilde) std::memcpy(Atilde, At.data(), sizeof(double) * At.size());
    });
}

int irk_make_coeff(int scheme, int s, int kind, const char* custom_path, double* Atilde,
                   int* structure) {
    return guard([&] {
        irkb::check(kind >= 0 && kind <= 4, "make_coeff: unknown kind");
        const irkb::Tableau t = irkb::make_tableau(static_cast<irkb::Scheme>(scheme), s);
        const irkb::Coeff c = irkb::make_coeff(t, static_cast<irkb::CoeffKind>(kind),
                                               custom_path ? custom_path : "");
        std::memcpy(Atilde, c.At.data(), sizeof(double) * s * s);
        *structure = static_cast<int>(c.structure);
    });
}

int irk_amg_setup(const irk_csr* A, const irk_amg_params* p, irk_hierarchy** out) {
    return guard([&] { *out = new irk_hierarchy{irkb::amg_setup(to_csr(A), to_params(p))}; });
}

int irk_amg_setup_device(const irk_csr* A, const irk_amg_params* p, int device, irk_hierarchy** out) {
    return guard([&] { *out = new irk_hierarchy{irkb::amg_setup_device(to_csr(A), to_params(p), device)}; });
}

int irk_hierarchy_levels(const irk_hierarchy* h) { return h->h.n_levels(); }

int irk_hierarchy_level(const irk_hierarchy* h, int level, int which, irk_csr* out) {
    return guard([&] {
        irkb::check(level >= 0 && level < h->h.n_levels(), "hierarchy: level out of range");
        const irkb::AmgLevel& L = h->h.levels[level];
        irkb::check(which >= 0 && which <= 4, "hierarchy: which must be 0..4");
        view(which == 0 ? L.A : which == 1 ? L.P : which == 2 ? L.R : which == 3 ? L.G : L.U, out);
    });
}

int irk_hierarchy_compose_lanes(const irk_hierarchy* h, int level, int* g_lanes, int* u_lanes) {
    return guard([&] {
        irkb::check(level >= 0 && level < h->h.n_levels(), "hierarchy: level out of range");
        *g_lanes = h->h.levels[level].g_lanes;
        *u_lanes = h->h.levels[level].u_lanes;
    });
}

const double* irk_hierarchy_inv_diag(const irk_hierarchy* h, int level) {
    return h->h.levels[level].inv_diag.data();
}

const double* irk_hierarchy_coarse_inverse(const irk_hierarchy* h, int* n) {
    *n = h->h.levels.back().A.rows;
    return h->h.coarse_inverse.data();
}

const double* irk_hierarchy_tail(const irk_hierarchy* h, int* from, int* n, int* ld) {
    const irkb::Hierarchy& H = h->h;
    *from = H.tail_from;
    *n = H.tail_from > 0 ? H.levels[H.tail_from].A.rows : 0;
    *ld = H.tail_ld;
    return H.tail_from > 0 ? H.tail.data() : nullptr;
}

void irk_hierarchy_free(irk_hierarchy* h) { delete h; }

int irk_mm_write(const irk_csr* A, const char* path) {
    return guard([&] {
        irkb::check(path != nullptr, "matrix market: null path");
        irkb::write_matrix_market(to_csr(A), path);
    });
}

int irk_mm_read(const char* path, irk_matrix** out) {
    return guard([&] {
        irkb::check(path != nullptr, "matrix market: null path");
        *out = new irk_matrix{irkb::read_matrix_market(path)};
    });
}

int irk_matrix_view(const irk_matrix* m, irk_csr* out) {
    return guard([&] { view(m->a, out); });
}

void irk_matrix_free(irk_matrix* m) { delete m; }

namespace {
int put_text(const std::string& t, char* buf, int cap) {
    irkb::check(buf != nullptr && cap > static_cast<int>(t.size()), "csv: buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return static_cast<int>(t.size());
}
}  // namespace

int irk_csv_header(char* buf, int cap) {
    return guard([&] { put_text(irkb::csv_header(), buf, cap); });
}

int irk_csv_row(int scheme, int s, int hx_inv, double ht, int n_free, int kind, int side,
                int subsolver, double iterations, double true_residual, double rel_error,
                double seconds, int failed, char* buf, int cap) {
    return guard([&] {
        irkb::CsvCell c;
        c.scheme = scheme;
        c.s = s;
        c.hx_inv = hx_inv;
        c.ht = ht;
        c.n_free = n_free;
        c.kind = kind;
        c.side = side;
        c.subsolver = subsolver;
        c.iterations = iterations;
        c.true_residual = true_residual;
        c.rel_error = rel_error;
        c.seconds = seconds;
        c.failed = failed != 0;
        put_text(irkb::csv_row(c), buf, cap);
    });
}

int irkdev_create(const irk_csr* M, const irk_csr* K, int s, const double* A, const double* b,
                  const double* Atilde, int structure, double ht, const irk_amg_params* amg,
                  int n_hier, const irk_hierarchy* const* hiers, int device, irkdev** out) {
    return guard([&] {
        irkb::check(s >= 1 && s <= 7, "device solver: s must be in 1..7");
        irkb::check(structure >= 0 && structure <= 2, "device solver: bad coefficient structure");
        const irkb::Csr Mc = to_csr(M), Kc = to_csr(K);
        std::vector<double> Av(A, A + s * s), bv(b, b + s), Atv(Atilde, Atilde + s * s);
        irkb::custom_coeff(s, Atv);  // validates structure / nonzero diagonal
        std::vector<irkb::Hierarchy> hv;
        for (int k = 0; k < n_hier; ++k) hv.push_back(hiers[k]->h);
        const irkb::AmgParams prm = to_params(amg);
        auto* d = new irkdev;
        try {
            d->s = std::make_unique<irkb::DeviceSolver>(Mc, Kc, s, Av, bv, Atv,
                                                        static_cast<irkb::Structure>(structure), ht,
                                                        prm, std::move(hv), device);
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

void irkdev_destroy(irkdev* d) { delete d; }

int irkdev_info(const irkdev* d, int* n, int* s, int* n_hier, int* sob, double* setup) {
    return guard([&] {
        if (n) *n = d->s->n();
        if (s) *s = d->s->s();
        if (n_hier) *n_hier = static_cast<int>(d->s->hierarchies().size());
        if (sob)
            for (int j = 0; j < d->s->s(); ++j) sob[j] = d->s->solver_of_block()[j];
        if (setup) *setup = d->s->setup_seconds();
    });
}

int irkdev_hierarchy(const irkdev* d, int k, irk_hierarchy** out) {
    return guard([&] {
        const auto& hs = d->s->hierarchies();
        irkb::check(k >= 0 && k < static_cast<int>(hs.size()), "hierarchy: index out of range");
        *out = new irk_hierarchy{hs[k]};
    });
}

int irkdev_num_levels(const irkdev* d, int k) {
    return d->s->hierarchies().at(k).n_levels();
}

int irkdev_level_info(const irkdev* d, int k, int l, int* n, int* nnz_A, int* nnz_P, int* nnz_R,
                      int* fmt_A) {
    return guard([&] {
        const irkb::Hierarchy& h = d->s->hierarchies().at(k);
        irkb::check(l >= 0 && l < h.n_levels(), "level_info: level out of range");
        const irkb::AmgLevel& L = h.levels[l];
        *n = L.A.rows;
        *nnz_A = L.A.nnz();
        *nnz_P = L.P.nnz();
        *nnz_R = L.R.nnz();
        if (fmt_A) *fmt_A = l == 0 ? d->s->matrix_format(1) : 0;
    });
}

int irk_set_option(const char* name, long long value) {
    return guard([&] {
        irkb::check(name != nullptr, "set_option: name is null");
        irkb::dev::set_option(name, value);
    });
}

int irkdev_level_value_format(const irkdev* d, int k, int l, int* vf) {
    return guard([&] { *vf = d->s->level_value_format(k, l); });
}

int irkdev_step(irkdev* d, const double* u_n, const double* f_lift, const irk_gmres_cfg* cfg,
                double* u_next, double* k_out, irk_report* rep, double* history) {
    return guard([&] {
        const irkb::SolveReport r = d->s->step_host(u_n, f_lift, to_cfg(cfg), u_next, k_out);
        fill_report(r, d->s->setup_seconds(), rep, history);
    });
}

int irkdev_step_device(irkdev* d, const double* u_n, const double* f_lift,
                       const irk_gmres_cfg* cfg, double* u_next, double* k_out, irk_report* rep) {
    return guard([&] {
        const irkb::SolveReport r = d->s->step(u_n, f_lift, to_cfg(cfg), u_next, k_out);
        fill_report(r, d->s->setup_seconds(), rep, nullptr);
    });
}

int irkdev_step_forced(irkdev* d, const double* u_n, const double* f_lift, double t_n,
                       const double* c, irk_forcing_fn forcing, void* forcing_user,
                       const irk_gmres_cfg* cfg, double* u_next, double* k_out, irk_report* rep,
                       double* history) {
    return guard([&] {
        std::vector<double> fv;
        if (forcing) {
            irkb::check(c != nullptr, "stage_rhs: forcing needs the stage nodes c");
            const int n = d->s->n(), s = d->s->s();
            fv.resize(static_cast<size_t>(s) * n);
            for (int i = 0; i < s; ++i)
                irkb::check(forcing(t_n + c[i] * d->s->ht(), fv.data() + static_cast<size_t>(i) * n, n,
                                    forcing_user) == 0,
                            "stage_rhs: forcing callback failed");
        }
        const irkb::SolveReport r = d->s->step_host(u_n, f_lift, to_cfg(cfg), u_next, k_out,
                                                    forcing ? fv.data() : nullptr);
        fill_report(r, d->s->setup_seconds(), rep, history);
    });
}

int irk_integrate_steps(double t_final, double ht, int* steps) {
    return guard([&] {
        irkb::check(ht > 0.0, "integrate: ht must be positive");
        irkb::check(t_final >= 0.0, "integrate: t_final must be nonnegative");
        *steps = static_cast<int>(integrate_plan(t_final, ht).size());
    });
}

int irkdev_integrate(irkdev* d, irkdev_factory_fn make, void* make_user, const double* u0,
                     const double* f_lift, const double* c, irk_forcing_fn forcing,
                     void* forcing_user, double t_final, double ht, const irk_gmres_cfg* cfg,
                     double* u_final, irk_report* reports, int cap, double* histories,
                     int* steps, double* t_out, int* all_converged) {
    return guard([&] {
        irkb::check(ht > 0.0, "integrate: ht must be positive");
        irkb::check(t_final >= 0.0, "integrate: t_final must be nonnegative");
        irkb::check(d->s->ht() == ht, "integrate: the solver was built for a different ht");
        const std::vector<double> plan = integrate_plan(t_final, ht);
        irkb::check(static_cast<long long>(plan.size()) <= cap, "integrate: reports capacity too small");
        const irkb::GmresConfig g = to_cfg(cfg);
        const size_t hl = static_cast<size_t>(g.max_iter) + 1;
        irkdev* cur = d;
        double t = 0.0;
        bool conv = true;
        cur->s->load_u(u0);
        size_t k = 0;
        while (k < plan.size()) {
            if (plan[k] != cur->s->ht()) {  // step size changed: make_precond(step), irk.cpp:89-92
                irkb::check(make != nullptr, "integrate: step size changed and no factory was given");
                irkdev* nd = make(plan[k], make_user);
                irkb::check(nd != nullptr && nd->s, "integrate: factory returned no solver");
                irkb::check(nd->s->ht() == plan[k], "integrate: factory solver has the wrong ht");
                irkb::check(nd->s->n() == cur->s->n() && nd->s->s() == cur->s->s(),
                            "integrate: factory solver has the wrong size");
                nd->s->load_u(cur->s->state());
                cur = nd;
            }
            size_t run = 0;
            while (k + run < plan.size() && plan[k + run] == cur->s->ht()) ++run;
            const std::vector<irkb::SolveReport> reps = cur->s->run_segment(
                static_cast<int>(run), &t, f_lift, forcing, forcing_user, c, g, histories != nullptr);
            for (size_t q = 0; q < run; ++q) {
                fill_report(reps[q], cur->s->setup_seconds(), reports + k + q,
                            histories ? histories + hl * (k + q) : nullptr);
                conv = conv && reps[q].converged;
            }
            k += run;
        }
        cur->s->store_u(u_final);
        if (steps) *steps = static_cast<int>(plan.size());
        if (t_out) *t_out = t;
        if (all_converged) *all_converged = conv ? 1 : 0;
    });
}


int irkdev_stage_apply(irkdev* d, const double* v, double* y) {
    return guard([&] {
        const long long N = d->s->sN();
        with_device_vectors(d, v, N, y, N, [&](double* a, double* b) { d->s->stage_apply(a, b); });
    });
}

int irkdev_precond_apply(irkdev* d, const double* v, double* w) {
    return guard([&] {
        const long long N = d->s->sN();
        with_device_vectors(d, v, N, w, N, [&](double* a, double* b) { d->s->precond_apply(a, b); });
    });
}

int irkdev_vcycle(irkdev* d, int k, const double* r, double* z) {
    return guard([&] {
        const long long n = d->s->n();
        with_device_vectors(d, r, n, z, n, [&](double* a, double* b) { d->s->vcycle(k, a, b); });
    });
}

int irkdev_dot(irkdev* d, const double* x, const double* y, long long n, double* out) {
    return guard([&] {
        irkb::DeviceScope on(d->s->device());
        irkb::DevBuf a(sizeof(double) * n), b(sizeof(double) * n);
        IRK_CUDA_CHECK(cudaMemcpy(a.as<double>(), x, sizeof(double) * n, cudaMemcpyHostToDevice));
        IRK_CUDA_CHECK(cudaMemcpy(b.as<double>(), y, sizeof(double) * n, cudaMemcpyHostToDevice));
        *out = d->s->dot(a.as<double>(), b.as<double>(), n);
    });
}

int irkdev_time_kernel(irkdev* d, int which, int reps, double* ms) {
    return guard([&] { *ms = d->s->time_kernel(which, reps); });
}

int irkdev_last_timed_bytes(const irkdev* d, double* bytes) {
    return guard([&] { *bytes = d->s->last_timed_bytes(); });
}

int irkdev_launch_counts(const irkdev* d, int* c) {
    return guard([&] {
        const auto& v = d->s->launch_counts();
        for (int i = 0; i < 4; ++i) c[i] = v[i];
    });
}

int irkdev_model_bytes(const irkdev* d, double* out) {
    return guard([&] {
        const auto& t = d->s->model_bytes();
        const double v[8] = {t[0].fixed, t[1].fixed, t[1].per_j, t[2].fixed, t[2].per_j, t[3].fixed, 0.0, 0.0};
        for (int i = 0; i < 8; ++i) out[i] = v[i];
    });
}

int irkdev_stream(const irkdev* d, void** stream) {
    return guard([&] { *stream = static_cast<void*>(d->s->stream()); });
}

int irkdev_graph_info(const irkdev* d, int* lpi, int* mode) {
    return guard([&] {
        if (lpi) *lpi = d->s->launches_per_iteration();
        if (mode) *mode = d->s->graph_mode();
    });
}

}  // extern "C"
