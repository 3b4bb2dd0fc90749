/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the IRK solve phase.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this (as the checker).  The product never links it.  See irk_oracle.c. */
#ifndef IRK_ORACLE_H
#define IRK_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int rows, cols;
    const int* ptr;
    const int* idx;
    const double* val;
} or_csr;

typedef struct {
    int nlev;
    const or_csr* A;             /* nlev */
    const or_csr* P;             /* nlev - 1 */
    const or_csr* R;             /* nlev - 1 */
    const double* const* inv_diag; /* nlev */
    const double* cinv;          /* dense nc x nc inverse of A[nlev-1] */
    int nc;
    double omega;
    int pre, post;
    /* dense V-cycle tail operator (the product's setup, csrc/host/tail.cpp):
     * levels >= tail_from are z = B r, B row-major n x tail_ld; -1 = none */
    int tail_from, tail_ld;
    const double* tail;
    int smoother;      /* 0 damped Jacobi, 1 Gauss-Seidel (amg.cpp:125-140) */
    /* composed Jacobi V(1,1) legs (the product's setup, csrc/host/compose.cpp):
     * on a level l with G[l].rows > 0 the cycle is r_{l+1} = G_l r_l going
     * down and z_l = U_l [r_l; z_{l+1}] coming up; NULL = recursive form */
    const or_csr* G;   /* nlev - 1 */
    const or_csr* U;   /* nlev - 1 */
    /* row-sum association of G[l], U[l] (part of their definition): L lanes,
     * lane q adds entries q, q+L, ... of the row in order from 0.0, then the
     * xor butterfly L/2, ..., 1 folds the lanes; 1 = sequential */
    const int* g_lanes;
    const int* u_lanes;
} or_hier;

typedef struct {
    int n, s;
    or_csr M, K;
    const double* A;   /* s*s Butcher matrix */
    const double* b;   /* s weights */
    double ht;
    const double* At;  /* s*s preconditioner coefficients */
    int structure;     /* 0 diagonal, 1 lower, 2 upper */
    int nh;
    const or_hier* h;
    const int* sob;    /* solver_of_block[s] */
} or_sys;

void or_spmv(const or_csr* A, const double* x, double* y);
double or_dot(const double* x, const double* y, long n);
void or_vcycle(const or_hier* h, const double* r, double* z);
void or_stage_apply(const or_sys* S, const double* v, double* y);
void or_precond_apply(const or_sys* S, const double* v, double* w);

typedef struct {
    int iterations, cycles, n_reorth, converged;
    double true_rel, final_rel;
    double seconds;
} or_report;

/* 1 (default): delayed CGS2 (the device's scheme); 0: CGS + conditional
 * second pass (the device's former scheme, IRK_ORTHO=cgs2). */
void or_set_ortho(int scheme);

/* One IRK step: rhs, GMRES(restart) (right preconditioning, the scheme of
 * or_set_ortho, flexible basis), u_next.  hist gets
 * max_iter+1 entries (may be NULL). */
int or_irk_step(const or_sys* S, const double* u, const double* lift, double rtol,
                int restart, int max_iter, double* u_next, double* K, or_report* rep,
                double* hist);
/* Same with a forcing term (forcing = s*n stage-major values of
 * forcing(t_n + c_q ht), irk.cpp:24-30, or NULL) and the preconditioning
 * side (1 right, 0 left: delayed CGS2 only, returns -1 otherwise). */
int or_irk_step_f(const or_sys* S, const double* u, const double* lift, const double* forcing,
                  int side, double rtol, int restart, int max_iter, double* u_next, double* K,
                  or_report* rep, double* hist);

#ifdef __cplusplus
}
#endif
#endif
