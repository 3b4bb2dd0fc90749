// Device-resident IRK stage-system solver: the B200 replacement for the
// reference's irk_step -> gmres -> {StageOperator, BlockPreconditioner ->
// amg_vcycle} call stack (SURVEY.md §3 stack B).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdlib>
#include <deque>
#include <cstdint>
#include <memory>
#include <vector>

#include "../host/setup.hpp"
#include "kernels.cuh"

namespace irkb {


// Owns one device allocation.
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t bytes);
    ~DevBuf();
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T> T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

struct GmresConfig {
    int side = 1;        // 1 right, 0 left (delayed CGS2 only)
    double rel_tol = 1e-8;
    int max_iter = 500;
    int restart = 50;    // 0 = full GMRES (restart = max_iter)
};

struct SolveReport {
    int iterations = 0, cycles = 0, n_reorth = 0, converged = 0;
    double final_rel = 0.0, true_rel = 0.0;
    double solve_seconds = 0.0;
    std::vector<double> history;
};

struct DevLevel {
    int n = 0;
    dev::Mat A, P, R;
    dev::Mat G, U;                // composed V(1,1) legs (compose.cpp); G.rows == 0: recursive level
    dev::Mat US, UQ;              // up leg of a 7-point level: S as row classes, Q as SELL-32
    bool up_cls = false;          // (U itself is then not stored)
    double* wd = nullptr;         // omega * D^-1
    double* r = nullptr;          // level rhs (levels >= 1)
    double* z = nullptr;          // level solution (levels >= 1)
    double* t = nullptr;          // residual / prolongated iterate
    double* u = nullptr;          // post-sweep ping-pong
    double* zp = nullptr;         // pre-smoothed iterate (pre > 1 only)
    double* zr = nullptr;         // wd .* r, written by the restriction (levels >= 1)
    dev::GsSweep gsf, gsb;        // Gauss-Seidel schedules (forward / backward sweeps)
};

struct DevHier {
    std::vector<DevLevel> lv;
    double* cinv = nullptr;
    int nc = 0;
    AmgParams prm;
    int bot_from = -1;    // first level handled by the single-CTA bottom kernel
    dev::BotDesc bot;
    int tail_from = -1;   // first level replaced by the dense tail operator
    int tail_ld = 0;
    double* tail = nullptr;
};

class DeviceSolver {
public:
    // Builds (or takes) one AMG hierarchy per distinct diagonal of At and
    // uploads everything.  `hiers` may be empty (built here with `amg`).
    DeviceSolver(const Csr& M, const Csr& K, int s, const std::vector<double>& A,
                 const std::vector<double>& b, const std::vector<double>& At, Structure st,
                 double ht, const AmgParams& amg, std::vector<Hierarchy> hiers, int device);
    ~DeviceSolver();

    int n() const { return n_; }
    int device() const { return device_; }
    int s() const { return s_; }
    long long sN() const { return sN_; }
    cudaStream_t stream() const { return st_; }
    const std::vector<Hierarchy>& hierarchies() const { return hier_host_; }
    const std::vector<int>& solver_of_block() const { return sob_; }
    double setup_seconds() const { return setup_seconds_; }
    bool fused_stage_op() const { return fused_op_; }
    int matrix_format(int which) const;
    int level_value_format(int k, int l) const {
        check(k >= 0 && k < static_cast<int>(hier_.size()), "level_value_format: hierarchy out of range");
        check(l >= 0 && l < static_cast<int>(hier_[k].lv.size()), "level_value_format: level out of range");
        return hier_[k].lv[l].A.vf;
    }  // 0 M, 1 K -> 0 CSR, 1 DIA

    // Device-pointer entry points (enqueue + synchronise).
    void stage_apply(const double* v, double* y);
    void precond_apply(const double* v, double* w);
    void vcycle(int k, const double* r, double* z);
    double dot(const double* x, const double* y, long long n);
    // forcing (may be null): s*n stage-major values forcing(t_n + c_i ht)
    // (irk.cpp:24-30), host or device pointer.
    SolveReport step(const double* u, const double* lift, const GmresConfig& cfg, double* u_next,
                     double* k_out, const double* forcing = nullptr);
    // Host-pointer step: H2D of u (and lift), D2H of u_next (and K).
    SolveReport step_host(const double* u, const double* lift, const GmresConfig& cfg,
                          double* u_next, double* k_out, const double* forcing = nullptr);

    // Device-resident trajectory segment (irk.cpp:85-99 for a run of steps of
    // this solver's ht): u stays in HBM between steps; the host only
    // evaluates the forcing (double-buffered pinned staging, overlapped with
    // the previous step) and collects the reports once at the end.
    // load_u copies u0 (host or device) into the solver's state vector.
    using ForcingFn = int (*)(double t, double* out, int n, void* user);
    void load_u(const double* u0);
    const double* state() const { return u_; }
    // Runs nsteps steps from time *t (advanced in place as t += ht, the
    // reference's accumulation); c: the tableau's stage nodes (s values).
    std::vector<SolveReport> run_segment(int nsteps, double* t, const double* lift,
                                         ForcingFn forcing, void* user, const double* c,
                                         const GmresConfig& cfg, bool want_history);
    void store_u(double* dst);  // u -> dst (host or device), synchronises
    double ht() const { return ht_; }

    // Timing hooks for the roofline (bench.py): launches `reps` applications
    // of the named hot kernel between CUDA events on the solver's stream and
    // returns the mean milliseconds per launch.  which: 0 stage operator,
    // 1 fine-level smoother SpMV, 2 preconditioner apply, 3 V-cycle, 4.. V-cycle
    // below level which-3, 100+j GMRES block-dot at inner index j, 20/21 empty-
    // kernel launch floor (graph / stream), 60+2l(+1) Gauss-Seidel forward
    // (backward) sweep of hierarchy 0 at level l.
    // 7 / 8: the composed level-0 down / up leg of hierarchy 0 alone.
    double time_kernel(int which, int reps);
    // algorithmic bytes (stored formats) of one application of the phase last
    // timed through the generic path (which < 20)
    double last_timed_bytes() const { return last_timed_bytes_; }
    int launches_per_iteration() const { return launches_per_iter_; }
    const std::array<int, 4>& launch_counts() const { return launch_counts_; }
    // Algorithmic bytes per phase (pre, cycle, iteration, post) of the last
    // recorded step graph, each as fixed + per_j * j (dev::Tally).
    const std::array<dev::Tally, 4>& model_bytes() const { return tally_; }
    int graph_mode() const { return graph_mode_; }

private:
    // tree_lanes: 0 format by heuristics; 1 SELL-32 (sequential row sums);
    // >= 2 CSR with lane-tree row sums (composed operators)
    dev::Mat upload(const Csr& A, bool allow_dia, double omega, int tree_lanes = 0);
    // Row-signature storage (dev::kRowSig) of a composed operator; `split` > 0:
    // columns >= split address the second operand.  False when the rows do
    // not repeat (general operators): the caller keeps the CSR form.
    bool upload_rowsig(const Csr& A, int lanes, int split, dev::Mat& m);
    // U = [S | Q] of a 7-point level as row classes + SELL-32 (false: not that shape)
    bool upload_up_cls(const Csr& U, int n, dev::Mat& S, dev::Mat& Q);
    void build_bottom(DevHier& dh, const Hierarchy& h);
    // DIA row classes (dev::kCls) for one operator or a pair sharing a pattern
    bool to_row_classes(std::vector<dev::Mat*> mats, const std::vector<const std::vector<double>*>& vals,
                        double omega);
    // codes_out (optional): when the values are dictionary codes and code +
    // column fit one 32-bit word, the codes are returned instead of uploaded
    // and m.pk_shift is set; the caller packs them with pack_codes (kP8)
    void upload_values(dev::Mat& m, const std::vector<double>& vals, double omega,
                       std::vector<unsigned>* codes_out = nullptr);
    void pack_codes(dev::Mat& m, std::vector<int>& idx, const std::vector<unsigned>& codes);
    template <class T> const T* upload_array(const std::vector<T>& h);
    double* alloc(size_t count);
    void* raw_alloc(size_t bytes);
    void record_vcycle(int k, dev::VecRef r, dev::VecRef z, int first = 0);
    void record_vcycle_gs(int k, dev::VecRef r, dev::VecRef z, int first);
    dev::GsSweep upload_gs(const Csr& A, const std::vector<double>& inv_diag, bool backward);
    void record_precond(dev::VecRef v, dev::VecRef w);
    void record_stage_op(dev::VecRef z, dev::VecRef y);
    void record_iteration();
    void ensure_gmres(int restart, int max_iter);
    void build_graph(bool lift, bool forcing, int restart, int max_iter, double rtol,
                     bool use_cond);
    int prepare(const GmresConfig& cfg, bool lift, bool forcing);  // -> max_iter
    void launch_solve();  // enqueue one step (graph mode) / run it (host-driven)
    static SolveReport report_from(const dev::GmresCtl& c, const double* hist, int max_iter);

    int n_ = 0, s_ = 0;
    long long sN_ = 0, stride_ = 0;
    int device_ = 0;
    cudaStream_t st_ = nullptr;
    struct Branches {                    // block-Jacobi V-cycle branches
        std::vector<cudaStream_t> st;    // index 0 unused (the recording stream)
        std::vector<cudaEvent_t> ev;     // [0] fork, [k] join of branch k
    };
    std::deque<Branches> branch_sets_;   // one set per concurrently open capture
    std::vector<DevBuf> bufs_;

    dev::Mat M_, K_;
    bool fused_op_ = false;
    dev::StageCoef coef_{};
    std::vector<double> At_, hb_;
    Structure structure_ = Structure::Diagonal;
    double ht_ = 0.0;
    std::vector<int> sob_;
    std::vector<Hierarchy> hier_host_;
    std::vector<DevHier> hier_;
    double setup_seconds_ = 0.0;
    // work vectors
    double *rhs_ = nullptr, *fw_ = nullptr;  // fw_: s * n
    double *u_ = nullptr, *lift_ = nullptr, *unext_ = nullptr, *ku_ = nullptr;
    double* forcing_ = nullptr;  // s * n, allocated on first forced step
    double *b_ = nullptr, *x_ = nullptr, *r_ = nullptr, *ax_ = nullptr;
    double *red_part_ = nullptr, *red_out_ = nullptr;
    unsigned* red_cnt_ = nullptr;
    // GMRES
    int cap_restart_ = 0, cap_iter_ = 0;
    dev::GmresBufs gb_{};
    DevBuf V_, Z_, H_, hist_, part_, ctl_, cnt_;
    dev::GmresCtl* ctl_host_ = nullptr;  // pinned
    double* hist_host_ = nullptr;        // pinned
    // graph cache
    cudaGraphExec_t exec_ = nullptr;
    cudaGraphExec_t exec_iter_ = nullptr, exec_pre_ = nullptr, exec_cb_ = nullptr,
                    exec_ce_ = nullptr, exec_post_ = nullptr;
    int graph_mode_ = -1;  // 1 conditional nodes, 0 host-driven loop
    bool g_lift_ = false, g_forcing_ = false;
    int g_restart_ = -1, g_iter_ = -1;
    unsigned g_opt_gen_ = ~0u;  // dev::option_generation() the graphs were recorded with
    double g_rtol_ = -1.0;
    int launches_per_iter_ = 0;
    std::array<dev::Tally, 4> tally_{};
    std::array<int, 4> launch_counts_{};
    bool compress_values_ = true;
    int ortho_ = 1;  // 1 DCGS2 (default), 0 CGS + conditional second pass
    int side_ = 1, g_side_ = -1;  // GMRES preconditioning side (1 right, 0 left)
    // the next recorded V-cycle's first kernel follows a late-trigger kernel
    // (a sweep) and may be launched programmatically (IRK_PDL_FINE)
    bool vc_pdl_first_ = false;
    double last_timed_bytes_ = 0.0;
    bool pack_sell_ = false;  // upload(): pack the next SELL operator's codes (the up leg's Q part)
};

}  // namespace irkb
