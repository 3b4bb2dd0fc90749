/* irkdev.h -- C ABI of the B200-native IRK stage-system solve phase.
 *
 * Drop-in boundary for the reference's C++ solver interface (irkprec):
 * plain pointers and sizes, no torch or C++ types.  Every entry point
 * returns an irk_status; the message of the last failure on the calling
 * thread is irk_last_error().  Error classes map 1:1 onto the reference's
 * exceptions (common.hpp:16-41): IRK_EINVAL <-> std::invalid_argument
 * (require, common.hpp:39-41), IRK_ESINGULAR <-> SingularError,
 * IRK_ENUMERICAL <-> NumericalError.  GMRES non-convergence is NOT an error:
 * it is reported in irk_report.converged (gmres.hpp:45-48).
 *
 * The library has no CPU fallback: device entry points fail with IRK_ECUDA
 * when no CUDA device is present.
 */
#ifndef IRKDEV_H
#define IRKDEV_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IRK_OK = 0,
    IRK_EINVAL = 1,       /* std::invalid_argument (common.hpp:39-41)     */
    IRK_ESINGULAR = 2,    /* SingularError (common.hpp:16-24)             */
    IRK_ENUMERICAL = 3,   /* NumericalError (common.hpp:28-37)            */
    IRK_ECUDA = 4,        /* CUDA runtime failure / no device             */
    IRK_EUNSUPPORTED = 5, /* valid reference option not run on the device */
    IRK_EIO = 6,          /* std::runtime_error of file I/O / parsing
                             (butcher.cpp:300-313, csr.cpp:240-290)      */
    IRK_EINTERNAL = 9
} irk_status;

const char* irk_last_error(void);

/* CSR view (csr.hpp:15-32): int32 row_ptr[n_rows+1], col_idx[nnz],
 * fp64 vals[nnz]; columns strictly increasing within a row. */
typedef struct {
    int n_rows, n_cols, nnz;
    const int* row_ptr;
    const int* col_idx;
    const double* vals;
} irk_csr;

/* AmgParams (amg.hpp:14-29). smoother: 0 damped Jacobi (device), 1 GS. */
typedef struct {
    double theta;
    int pre_sweeps, post_sweeps, smoother;
    double jacobi_weight, prolongation_weight;
    int prolongation_steps, max_coarse, max_levels;
} irk_amg_params;
/* library-default AmgParams{} (amg.hpp:14-29): theta 0.25, V(1,1) damped
 * Jacobi with omega 2/3, prolongation weight 4/3 x 1 step, max_coarse 64. */
void irk_amg_params_default(irk_amg_params* p);

/* GmresConfig (gmres.hpp:17-21) plus the restart length of GMRES(m);
 * restart = 0 means full GMRES (the reference's behaviour). side: 1 right. */
typedef struct {
    int side;
    double rel_tol;
    int max_iter;
    int restart;
} irk_gmres_cfg;
/* GmresConfig{} (gmres.hpp:17-21) plus the restart length: right, 1e-8, 500,
 * restart = 0 -- full GMRES, the reference's behaviour (BASELINE's GMRES(50)
 * sets restart = 50). */
void irk_gmres_cfg_default(irk_gmres_cfg* c);

/* SolveReport (gmres.hpp:23-38) without the history vector, which is
 * copied into a caller buffer. */
typedef struct {
    int iterations, cycles, n_reorth, converged;
    double final_rel_residual, true_rel_residual;
    double solve_seconds, setup_seconds;
    int history_len;
} irk_report;

/* ------------------------------------------------------ host setup ---- */
typedef struct irk_problem irk_problem;
/* Heat u_t = lap u on [0,1]^2, P1, zero Dirichlet, no forcing
 * (study.cpp:190-211 minus the manufactured forcing). */
int irk_problem_heat(int cells, irk_problem** out);
/* Double glazing on [-1,1]^2, cells per side, P1 SUPG, East wall = 1
 * (study.cpp:215-249, manufactured = false). */
int irk_problem_double_glazing(int cells, double eps, irk_problem** out);
int irk_problem_n(const irk_problem* p);
/* which: 0 M (mass), 1 K (stiffness / SUPG operator, the reference's F). */
int irk_problem_matrix(const irk_problem* p, int which, irk_csr* out);
const double* irk_problem_lift(const irk_problem* p);
/* u0 = sin(pi x) sin(pi y) + U[-noise, noise] (splitmix64(seed)). */
int irk_problem_initial(const irk_problem* p, double noise, unsigned long long seed, double* u0);
void irk_problem_free(irk_problem* p);

/* scheme: 0 Radau IIA (s=1..7), 1 Lobatto IIIC (s=2..5)
 * (butcher.hpp:31-40). A row-major s*s. */
int irk_tableau(int scheme, int s, double* A, double* b, double* c, int* q);
/* A = L diag(D) U (butcher.hpp:49-58). */
int irk_ldu(int s, const double* A, double* L, double* D, double* U);
/* kind: 0 Jacobi, 1 GSL, 2 DU, 3 LD (butcher.hpp:55-61).
 * structure out: 0 diagonal, 1 lower, 2 upper. */
int irk_precond_coeff(int scheme, int s, int kind, double* Atilde, int* structure);
/* custom_coeff (butcher.hpp:71-73): validates and infers the structure. */
int irk_custom_coeff(int s, const double* Atilde, int* structure);
/* read_coeff_file (butcher.cpp:300-313): the stage count then s*s row-major
 * values; *s is set, Atilde (cap >= s*s doubles, or NULL to query s) gets
 * the matrix.  IRK_EIO: cannot open / bad stage count / truncated data. */
int irk_read_coeff_file(const char* path, int cap, int* s, double* Atilde);
/* make_coeff (study.cpp:269-282): kinds 0-3 as irk_precond_coeff; kind 4
 * (custom) reads custom_path (IRK_EINVAL when NULL/empty or when its size is
 * not s), then custom_coeff validates it and infers the structure. */
int irk_make_coeff(int scheme, int s, int kind, const char* custom_path, double* Atilde,
                   int* structure);

typedef struct irk_hierarchy irk_hierarchy;
/* amg_setup (amg.hpp:52): the reference's smoothed-aggregation coarsening. */
int irk_amg_setup(const irk_csr* A, const irk_amg_params* p, irk_hierarchy** out);
/* amg_setup on the GPU `device` (amg.cpp:172-227): strength
 * graph, rho estimate, prolongator smoothing, R = P^T and the Galerkin
 * products run on the device, the greedy aggregation passes on the host.
 * Bit-identical to irk_amg_setup; IRK_ECUDA without a GPU (no fallback). */
int irk_amg_setup_device(const irk_csr* A, const irk_amg_params* p, int device, irk_hierarchy** out);
int irk_hierarchy_levels(const irk_hierarchy* h);
/* which: 0 A, 1 P, 2 R (amg.hpp:35-40); 3 G, 4 U: the composed V(1,1) legs
 * r_{l+1} = G r_l and z_l = U [r_l; z_{l+1}] the device cycle applies on the
 * levels above the tail (csrc/host/compose.cpp; 0 rows when not composed). */
int irk_hierarchy_level(const irk_hierarchy* h, int level, int which, irk_csr* out);
/* Row-sum association of the composed legs of `level`: L lanes per row (lane
 * q adds entries q, q+L, ... in order, then an xor butterfly over the lanes);
 * 1 = the sequential CSR row sum. */
int irk_hierarchy_compose_lanes(const irk_hierarchy* h, int level, int* g_lanes, int* u_lanes);
const double* irk_hierarchy_inv_diag(const irk_hierarchy* h, int level);
const double* irk_hierarchy_coarse_inverse(const irk_hierarchy* h, int* n);
/* The dense V-cycle tail operator attached by the setup (NULL if none):
 * *from = first level it replaces, B row-major n x *ld with n = rows of that
 * level (see csrc/host/tail.cpp). */
const double* irk_hierarchy_tail(const irk_hierarchy* h, int* from, int* n, int* ld);
void irk_hierarchy_free(irk_hierarchy* h);

/* ------------------------------------------------------ on-disk formats */
/* MatrixMarket coordinate files (csr.cpp:240-290): write_matrix_market
 * ("general", 1-based, %.17g) and read_matrix_market (general or symmetric,
 * duplicates summed); the read matrix is owned by the handle. */
typedef struct irk_matrix irk_matrix;
int irk_mm_write(const irk_csr* A, const char* path);
int irk_mm_read(const char* path, irk_matrix** out);
int irk_matrix_view(const irk_matrix* m, irk_csr* out);
void irk_matrix_free(irk_matrix* m);
/* Study CSV (study.cpp:334-360): header and one row, NUL-terminated into
 * buf (cap bytes).  scheme 0 radau_iia / 1 lobatto_iiic / 2 custom; kind as
 * irk_precond_coeff (4 custom); side 1 right / 0 left; subsolver 0 amg / 1 lu;
 * failed != 0 writes the reference's "failed" row. */
int irk_csv_header(char* buf, int cap);
int irk_csv_row(int scheme, int s, int hx_inv, double ht, int n_free, int kind, int side,
                int subsolver, double iterations, double true_residual, double rel_error,
                double seconds, int failed, char* buf, int cap);

/* ------------------------------------------------------ device solver - */
typedef struct irkdev irkdev;

/* BlockPreconditioner + StageOperator on the device
 * (stage.hpp:56-59, stage.hpp:21-23).  A, b: Butcher matrix/weights;
 * Atilde: preconditioner coefficients with `structure`.  When
 * n_hier == 0 the hierarchies are built here (one per distinct Atilde_jj,
 * stage.cpp:85-106); otherwise hiers[k] is used for the k-th distinct
 * diagonal in first-appearance order. */
int irkdev_create(const irk_csr* M, const irk_csr* K, int s, const double* A, const double* b,
                  const double* Atilde, int structure, double ht, const irk_amg_params* amg,
                  int n_hier, const irk_hierarchy* const* hiers, int device, irkdev** out);
void irkdev_destroy(irkdev* d);
int irkdev_info(const irkdev* d, int* n, int* s, int* n_hier, int* solver_of_block,
                double* setup_seconds);
/* hierarchy k, level l: sizes for the roofline byte model. */
int irkdev_level_info(const irkdev* d, int k, int l, int* n, int* nnz_A, int* nnz_P,
                      int* nnz_R, int* fmt_A);
/* A copy of hierarchy k as the solver built and uploaded it (its distinct
 * diagonal block's amg_setup, stage.cpp:85-106); free with irk_hierarchy_free.
 * Lets a caller pin the device setup against the reference's amg_setup. */
int irkdev_hierarchy(const irkdev* d, int k, irk_hierarchy** out);
int irkdev_num_levels(const irkdev* d, int k);
/* Stored value format of hierarchy k's level-l operator on the device:
 * 0 fp64, 1 u8 codes, 2 u16 codes, 3 DIA row classes (roofline byte counts). */
int irkdev_level_value_format(const irkdev* d, int k, int l, int* vf);
/* Tuning switch override (same names as the IRK_* environment variables);
 * solvers re-record their graphs on the next step.  For same-process A/B runs. */
int irk_set_option(const char* name, long long value);

/* irk_step (irk.hpp:36-39): host pointers.  f_lift may be NULL (zero),
 * k_out may be NULL; history (max_iter+1 doubles) may be NULL. */
int irkdev_step(irkdev* d, const double* u_n, const double* f_lift, const irk_gmres_cfg* cfg,
                double* u_next, double* k_out, irk_report* rep, double* history);
/* Same with DEVICE pointers (inputs already resident in HBM). */
int irkdev_step_device(irkdev* d, const double* d_u_n, const double* d_f_lift,
                       const irk_gmres_cfg* cfg, double* d_u_next, double* d_k_out,
                       irk_report* rep);

/* Forcing (irk.hpp:19, std::function<Vec(double)>): write the forcing at time
 * t into out[0..n); return 0 on success (nonzero -> IRK_EINVAL). */
typedef int (*irk_forcing_fn)(double t, double* out, int n, void* user);

/* irk_step at time t_n with forcing (stage_rhs, irk.cpp:9-33): block i of the
 * right-hand side gets forcing(t_n + c_i ht), evaluated on the host.  c: the
 * tableau's s stage nodes.  forcing may be NULL (then c may be NULL). */
int irkdev_step_forced(irkdev* d, const double* u_n, const double* f_lift, double t_n,
                       const double* c, irk_forcing_fn forcing, void* forcing_user,
                       const irk_gmres_cfg* cfg, double* u_next, double* k_out, irk_report* rep,
                       double* history);

/* PrecondFactory (irk.hpp:51-52): a solver for step size ht.  Handles it
 * returns stay owned by the caller (destroy them after integrate returns). */
typedef irkdev* (*irkdev_factory_fn)(double ht, void* user);

/* Number of steps integrate takes for (t_final, ht): the reference loop
 * (irk.cpp:85-99) including a truncated last step. */
int irk_integrate_steps(double t_final, double ht, int* steps);

/* integrate (irk.hpp:55-59, irk.cpp:70-102), device-resident: u stays in HBM
 * across steps, the host evaluates only the forcing (overlapped with the
 * previous step) and reads the reports once.  d is the solver for ht (the
 * reference's first make_precond(ht)); make is consulted when the step size
 * changes (the truncated last step) and may be NULL when no step changes
 * size.  u0, f_lift, u_final: host pointers (f_lift may be NULL).  reports:
 * cap entries, histories: NULL or cap * (max_iter + 1) doubles (per-step
 * residual histories).  Outputs: *steps, *t_out (the accumulated time) and
 * *all_converged. */
int irkdev_integrate(irkdev* d, irkdev_factory_fn make, void* make_user, const double* u0,
                     const double* f_lift, const double* c, irk_forcing_fn forcing,
                     void* forcing_user, double t_final, double ht, const irk_gmres_cfg* cfg,
                     double* u_final, irk_report* reports, int cap, double* histories,
                     int* steps, double* t_out, int* all_converged);

/* Kernel-level entry points, host pointers (parity tests):
 * StageOperator::apply (stage.cpp:28-44), BlockPreconditioner::apply
 * (stage.cpp:138-182), amg_vcycle for hierarchy k (amg.cpp:229-237). */
int irkdev_stage_apply(irkdev* d, const double* v, double* y);
int irkdev_precond_apply(irkdev* d, const double* v, double* w);
int irkdev_vcycle(irkdev* d, int k, const double* r, double* z);
/* Deterministic device dot (the GMRES reduction tree), host pointers. */
int irkdev_dot(irkdev* d, const double* x, const double* y, long long n, double* out);

/* Roofline hook: mean ms per launch of a hot kernel, CUDA events on the
 * solver stream.  which: 0 stage operator, 1 fine smoother SpMV,
 * 2 preconditioner apply, 3 V-cycle, 4+l V-cycle below level l+1,
 * 7 / 8 the composed level-0 down / up leg of hierarchy 0 alone,
 * 100+j GMRES block-dot at inner index j, 20 / 21 empty-kernel launch
 * floor in a graph / on the stream. */
int irkdev_time_kernel(irkdev* d, int which, int reps, double* ms);
/* Algorithmic bytes (operands once, in their stored formats) of one
 * application of the phase last timed with which < 20. */
int irkdev_last_timed_bytes(const irkdev* d, double* bytes);
/* Kernel launches per GMRES iteration in the captured graph body, and the
 * graph mode (1 conditional WHILE nodes, 0 host-driven). */
int irkdev_graph_info(const irkdev* d, int* launches_per_iteration, int* graph_mode);
/* Kernel launches of the captured step graph per phase: [0] once per step
 * before the GMRES loop, [1] per restart cycle, [2] per Arnoldi iteration,
 * [3] once per step after the loop. */
int irkdev_launch_counts(const irkdev* d, int* counts4);
/* Algorithmic HBM bytes of the captured step graph (the roofline numerator:
 * every kernel's operands read once and results written once, in their stored
 * formats): out8 = {pre, cycle, cycle_per_m, iteration, iteration_per_j,
 * post, 0, 0}; a step of cycles c_k (m_k columns) and iterations j moves
 * pre + post + sum_k (cycle + m_k cycle_per_m) + sum_j (iteration + j
 * iteration_per_j) bytes. */
int irkdev_model_bytes(const irkdev* d, double* out8);
/* The solver's CUDA stream (cudaStream_t) for event timing by the caller. */
int irkdev_stream(const irkdev* d, void** stream);

#ifdef __cplusplus
}
#endif
#endif
