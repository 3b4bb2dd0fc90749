/* TEST INFRASTRUCTURE ONLY -- CPU restatement ("oracle") of the IRK solve
 * phase of irkprec, used by tests/ (as the checker), __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg.  The product path never links or calls it.
 *
 * Parity is pinned two ways:
 *   1. against the reference itself compiled in place (oracle/_ref, built by
 *      oracle/Makefile from /root/reference/proj/src): stage apply, V-cycle,
 *      preconditioner apply and whole IRK steps, tests/test_oracle_vs_ref.py;
 *   2. against the reference's own known-answer tests restated in
 *      tests/test_kat.py (test_blocksolve.cpp, test_amg.cpp KATs).
 *
 * Restated algorithms (reference file:line):
 *   or_spmv           csr.cpp:102-114       sequential row sums
 *   or_stage_apply    stage.cpp:28-44       s F-products, s M-products, s^2 axpys
 *   or_vcycle         amg.cpp:115-168, 229-237  V(pre,post) damped Jacobi or
 *                     Gauss-Seidel (forward pre-sweeps, backward post-sweeps)
 *   or_precond_apply  stage.cpp:138-182     diagonal / forward / backward sweeps
 *   or_irk_step(_f)   irk.cpp:9-68, gmres.cpp:14-142 with the documented
 *                     deviations of the B200 path: GMRES(m) restarts,
 *                     delayed CGS2 (default) or classical Gram-Schmidt with
 *                     the reference's 0.7071 second-pass rule (gmres.cpp:84),
 *                     a flexible basis (x = Z y, which equals P^-1 V y by
 *                     linearity), dense coarse inverse.
 *
 * Floating-point order mirrors the device kernels exactly (compiled with
 * -ffp-contract=off; device with --fmad=false), including the fixed
 * reduction tree of paper_2010_11377_b200/csrc/device/common.cuh, so the
 * device result is expected to be bit-identical to this file's. */
#include "irk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define RED_T 256
#define RED_PT 16
#define CHUNK (RED_T * RED_PT)

/* ------------------------------------------------------------ reductions */
/* Warp shuffle-down tree on 32 lanes (lane 0 result). */
static double warp_tree(double* a) {
    for (int off = 16; off > 0; off >>= 1)
        for (int i = 0; i < off; ++i) a[i] = a[i] + a[i + off];
    return a[0];
}

/* 256 per-thread values -> block sum: per-warp trees, then warps in order. */
static double block_sum(double* t) {
    double w[8];
    for (int k = 0; k < 8; ++k) w[k] = warp_tree(t + 32 * k);
    double r = w[0];
    for (int k = 1; k < 8; ++k) r += w[k];
    return r;
}

static double chunk_partial(const double* x, const double* y, long n, long c) {
    double t[RED_T];
    for (int th = 0; th < RED_T; ++th) {
        double acc = 0.0;
        for (int u = 0; u < RED_PT / 2; ++u)
            for (int e = 0; e < 2; ++e) {
                const long k = c * CHUNK + (long)u * 2 * RED_T + 2 * th + e;
                const double xv = k < n ? x[k] : 0.0, yv = k < n ? y[k] : 0.0;
                acc += xv * yv;
            }
        t[th] = acc;
    }
    return block_sum(t);
}

static double final_sum(const double* part, long nch) {
    double t[RED_T];
    for (int th = 0; th < RED_T; ++th) {
        double acc = 0.0;
        for (long p = th; p < nch; p += RED_T) acc += part[p];
        t[th] = acc;
    }
    return block_sum(t);
}

double or_dot(const double* x, const double* y, long n) {
    long nch = (n + CHUNK - 1) / CHUNK;
    if (nch < 1) nch = 1;
    double* part = (double*)malloc(sizeof(double) * nch);
#pragma omp parallel for schedule(static)
    for (long c = 0; c < nch; ++c) part[c] = chunk_partial(x, y, n, c);
    const double r = final_sum(part, nch);
    free(part);
    return r;
}

/* ------------------------------------------------------------ sparse */
void or_spmv(const or_csr* A, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A->rows; ++i) {
        double s = 0.0;
        for (int k = A->ptr[i]; k < A->ptr[i + 1]; ++k) s += A->val[k] * x[A->idx[k]];
        y[i] = s;
    }
}

/* y_i = e(s_i) for s = A x with x = wd.*r (implicit) or x (plain). */
enum { EPI_PLAIN, EPI_RESID, EPI_SMOOTH, EPI_PROLONG };

static void spmv_epi(const or_csr* A, const double* x, const double* r, const double* wd,
                     const double* zb, int implicit_x, int epi, double* y) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A->rows; ++i) {
        double s = 0.0;
        for (int k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
            const int c = A->idx[k];
            const double xv = implicit_x ? wd[c] * r[c] : x[c];
            s += A->val[k] * xv;
        }
        double out = s;
        if (epi == EPI_RESID) out = r[i] - s;
        else if (epi == EPI_SMOOTH) out = x[i] + wd[i] * (r[i] - s);
        else if (epi == EPI_PROLONG) out = (zb ? zb[i] : wd[i] * r[i]) + s;
        y[i] = out;
    }
}

/* y = A x with the lane-tree row sum of the composed operators
 * (k_spmv_lt, kernels.cu): lane q of L adds the products of entries q, q+L,
 * ... in order from 0.0; the lanes are folded by the xor butterfly. */
static void spmv_lanes(const or_csr* A, int L, const double* x, double* y) {
    if (L <= 1) {
        or_spmv(A, x, y);
        return;
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A->rows; ++i) {
        double p[32], q[32];
        const int lo = A->ptr[i], len = A->ptr[i + 1] - lo;
        for (int l = 0; l < L; ++l) {
            double acc = 0.0;
            for (int k = l; k < len; k += L) acc = acc + A->val[lo + k] * x[A->idx[lo + k]];
            p[l] = acc;
        }
        for (int o = L / 2; o > 0; o >>= 1) {
            for (int l = 0; l < L; ++l) q[l] = p[l] + p[l ^ o];
            memcpy(p, q, sizeof(double) * L);
        }
        y[i] = p[0];
    }
}

/* ------------------------------------------------------------ V-cycle */
/* z = B r in k_tail_mv's order (kernels.cu, kTailWarps = 4): per row, 128
 * thread partials -- thread t adds the pairs p = t, t+128, ... (B[2p] r[2p],
 * then B[2p+1] r[2p+1] when 2p+1 < n) from 0.0 -- each warp of 32 folded by
 * the xor butterfly 16, 8, 4, 2, 1, and the 4 warp sums added in order. */
static void tail_mv(int n, int ld, const double* B, const double* r, double* z) {
    enum { W = 4, S = 32 * W };
    const int np = (n + 1) / 2;
    for (int i = 0; i < n; ++i) {
        const double* b = B + (long)i * ld;
        double ws[W];
        for (int w = 0; w < W; ++w) {
            double lane[32], nxt[32];
            for (int l = 0; l < 32; ++l) {
                double acc = 0.0;
                for (int p = 32 * w + l; p < np; p += S) {
                    acc = acc + b[2 * p] * r[2 * p];
                    if (2 * p + 1 < n) acc = acc + b[2 * p + 1] * r[2 * p + 1];
                }
                lane[l] = acc;
            }
            for (int o = 16; o > 0; o >>= 1) {
                for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ o];
                memcpy(lane, nxt, sizeof lane);
            }
            ws[w] = lane[0];
        }
        double sum = ws[0];
        for (int w = 1; w < W; ++w) sum = sum + ws[w];
        z[i] = sum;
    }
}

/* Gauss-Seidel sweep in place, CSR column order, the diagonal skipped
 * (amg.cpp:125-140). */
static void gs_sweep(const or_csr* A, const double* dinv, const double* r, double* z,
                     int backward) {
    const int n = A->rows;
    for (int t = 0; t < n; ++t) {
        const int i = backward ? n - 1 - t : t;
        double s = r[i];
        for (int k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
            if (A->idx[k] != i) s -= A->val[k] * z[A->idx[k]];
        z[i] = s * dinv[i];
    }
}

static void vcycle_level(const or_hier* h, double** wd, int l, const double* r, double* z);

/* amg.cpp:144-168 with the Gauss-Seidel smoother: the reference's order. */
static void vcycle_level_gs(const or_hier* h, double** wd, int l, const double* r, double* z) {
    const or_csr* A = &h->A[l];
    const int n = A->rows;
    const int nc = h->A[l + 1].rows;
    double* t = (double*)malloc(sizeof(double) * n);
    double* rc = (double*)malloc(sizeof(double) * nc);
    double* zc = (double*)malloc(sizeof(double) * nc);
    for (int i = 0; i < n; ++i) z[i] = 0.0;
    for (int sw = 0; sw < h->pre; ++sw) gs_sweep(A, h->inv_diag[l], r, z, 0);
    spmv_epi(A, z, r, NULL, NULL, 0, EPI_RESID, t);
    or_spmv(&h->R[l], t, rc);
    vcycle_level(h, wd, l + 1, rc, zc);
    spmv_epi(&h->P[l], zc, r, NULL, z, 0, EPI_PROLONG, t);
    memcpy(z, t, sizeof(double) * n);
    for (int sw = 0; sw < h->post; ++sw) gs_sweep(A, h->inv_diag[l], r, z, 1);
    free(t);
    free(rc);
    free(zc);
}

static void vcycle_level(const or_hier* h, double** wd, int l, const double* r, double* z) {
    const or_csr* A = &h->A[l];
    const int n = A->rows;
    if (h->tail && l == h->tail_from) {
        tail_mv(n, h->tail_ld, h->tail, r, z);
        return;
    }
    if (l == h->nlev - 1) {
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += h->cinv[(long)i * n + j] * r[j];
            z[i] = s;
        }
        return;
    }
    if (h->smoother) {
        vcycle_level_gs(h, wd, l, r, z);
        return;
    }
    const int nc = h->A[l + 1].rows;
    if (h->G && h->U && h->G[l].rows > 0 && h->pre == 1 && h->post == 1) {
        /* composed level (the device's record_vcycle, solver.cu): the down
         * leg and the up leg are one sparse product each, every row summed
         * with the operator's lane tree; the up leg's operand is
         * [r_l; z_{l+1}] */
        double* x = (double*)malloc(sizeof(double) * (n + nc));
        double* rc2 = (double*)malloc(sizeof(double) * nc);
        memcpy(x, r, sizeof(double) * n);
        spmv_lanes(&h->G[l], h->g_lanes ? h->g_lanes[l] : 1, r, rc2);
        vcycle_level(h, wd, l + 1, rc2, x + n);
        spmv_lanes(&h->U[l], h->u_lanes ? h->u_lanes[l] : 1, x, z);
        free(x);
        free(rc2);
        return;
    }
    double* t = (double*)malloc(sizeof(double) * n);
    double* zp = NULL;
    double* rc = (double*)malloc(sizeof(double) * nc);
    double* zc = (double*)malloc(sizeof(double) * nc);
    if (h->pre > 1) {
        /* first sweep from z = 0 gives wd.*r, then pre-1 Jacobi sweeps */
        zp = (double*)malloc(sizeof(double) * n);
        double* tmp = (double*)malloc(sizeof(double) * n);
        for (int i = 0; i < n; ++i) zp[i] = wd[l][i] * r[i];
        for (int sw = 1; sw < h->pre; ++sw) {
            spmv_epi(A, zp, r, wd[l], NULL, 0, EPI_SMOOTH, tmp);
            memcpy(zp, tmp, sizeof(double) * n);
        }
        free(tmp);
        spmv_epi(A, zp, r, wd[l], NULL, 0, EPI_RESID, t);
    } else {
        spmv_epi(A, NULL, r, wd[l], NULL, 1, EPI_RESID, t);
    }
    or_spmv(&h->R[l], t, rc);
    vcycle_level(h, wd, l + 1, rc, zc);
    /* z = zp + P zc, then post-smoothing sweeps */
    spmv_epi(&h->P[l], zc, r, wd[l], zp, 0, EPI_PROLONG, t);
    double* cur = t;
    double* nxt = z;
    for (int sw = 0; sw < h->post; ++sw) {
        spmv_epi(A, cur, r, wd[l], NULL, 0, EPI_SMOOTH, nxt);
        double* sv = cur;
        cur = nxt;
        nxt = sv;
    }
    if (cur != z) memcpy(z, cur, sizeof(double) * n);
    free(t);
    free(zp);
    free(rc);
    free(zc);
}

void or_vcycle(const or_hier* h, const double* r, double* z) {
    double** wd = (double**)malloc(sizeof(double*) * h->nlev);
    for (int l = 0; l < h->nlev; ++l) {
        const int n = h->A[l].rows;
        wd[l] = (double*)malloc(sizeof(double) * n);
        for (int i = 0; i < n; ++i) wd[l][i] = h->omega * h->inv_diag[l][i];
    }
    vcycle_level(h, wd, 0, r, z);
    for (int l = 0; l < h->nlev; ++l) free(wd[l]);
    free(wd);
}

/* ------------------------------------------------------------ stage system */
void or_stage_apply(const or_sys* S, const double* v, double* y) {
    const int n = S->n, s = S->s;
    double* Fv = (double*)malloc(sizeof(double) * (size_t)s * n);
    for (int j = 0; j < s; ++j) or_spmv(&S->K, v + (size_t)j * n, Fv + (size_t)j * n);
    for (int i = 0; i < s; ++i) {
        double* yi = y + (size_t)i * n;
        or_spmv(&S->M, v + (size_t)i * n, yi);
        for (int j = 0; j < s; ++j) {
            const double c = S->ht * S->A[i * s + j];
            const double* f = Fv + (size_t)j * n;
            for (int k = 0; k < n; ++k) yi[k] = yi[k] + c * f[k];
        }
    }
    free(Fv);
}

void or_precond_apply(const or_sys* S, const double* v, double* w) {
    const int n = S->n, s = S->s;
    double* Fw = (double*)malloc(sizeof(double) * (size_t)s * n);
    double* rhs = (double*)malloc(sizeof(double) * n);
    for (int q = 0; q < s; ++q) {
        const int j = S->structure == 2 ? s - 1 - q : q;
        const double* in = v + (size_t)j * n;
        if (S->structure != 0 && q > 0) {
            const int prev = S->structure == 2 ? j + 1 : j - 1;
            or_spmv(&S->K, w + (size_t)prev * n, Fw + (size_t)prev * n);
            const int k0 = S->structure == 2 ? j + 1 : 0;
            const int k1 = S->structure == 2 ? s : j;
            memcpy(rhs, in, sizeof(double) * n);
            for (int k = k0; k < k1; ++k) {
                const double a = S->At[j * s + k];
                if (a == 0.0) continue;
                const double e = -S->ht * a;
                const double* f = Fw + (size_t)k * n;
                for (int i = 0; i < n; ++i) rhs[i] = rhs[i] + e * f[i];
            }
            in = rhs;
        }
        or_vcycle(&S->h[S->sob[j]], in, w + (size_t)j * n);
    }
    free(Fw);
    free(rhs);
}

/* ------------------------------------------------------------ GMRES(m) */
/* Orthogonalisation scheme: 1 = delayed classical Gram-Schmidt with
 * re-orthogonalisation (DCGS2, the device default), 0 = CGS with the
 * reference's conditional second pass (gmres.cpp:84-90). */
static int g_ortho = 1;
void or_set_ortho(int scheme) { g_ortho = scheme; }

static double hyp(double a, double b) {
    a = fabs(a);
    b = fabs(b);
    const double mx = a > b ? a : b, mn = a > b ? b : a;
    if (mx == 0.0) return 0.0;
    const double r = mn / mx;
    return mx * sqrt(1.0 + r * r);
}

/* Rotates column `col` (entries 0..j+1, j = its index) into triangular form
 * with the stored rotations, adds rotation j and updates g (gmres.cpp:93-112). */
static void givens_column(double* col, int j, double* cs, double* sn, double* g) {
    for (int i = 0; i < j; ++i) {
        const double t = cs[i] * col[i] + sn[i] * col[i + 1];
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
        col[i] = t;
    }
    const double denom = hyp(col[j], col[j + 1]);
    double c = 1.0, sv = 0.0;
    if (denom > 0.0) {
        c = col[j] / denom;
        sv = col[j + 1] / denom;
    }
    cs[j] = c;
    sn[j] = sv;
    col[j] = denom;
    col[j + 1] = 0.0;
    g[j + 1] = -sv * g[j];
    g[j] = c * g[j];
}

/* One restart cycle of GMRES with delayed classical Gram-Schmidt
 * re-orthogonalisation (DCGS2; Bielich, Langou, Thomas, Swirydowicz,
 * Yamazaki, Boman 2022).  Slot j of V holds the once-orthogonalised,
 * unnormalised vector vt_j until iteration j re-orthogonalises it against
 * v_0..v_{j-1} in the same pass that projects w = A P^-1 vt_j:
 *   block-dot : s_i = v_i.vt_j, p_i = v_i.w (i < j), sig = vt_j.vt_j, pi = vt_j.w
 *   scalars   : alpha = sqrt(sig - sum s_i^2); column j-1 += s, h_{j,j-1} = alpha
 *               (finalised, rotated, residual recorded); h_jj = (pi - s.p)/alpha
 *   update    : v_j = (vt_j - sum s_i v_i)/alpha;  w' = w - sum p_i v_i - h_jj v_j
 * so each iteration streams the basis twice instead of four times.  The stop
 * test after iteration j uses the first-pass column with h_{j+1,j} = ||w'||;
 * the last column is finalised by one more block-dot at the end of the cycle.
 * Mirrors paper_2010_11377_b200/csrc/device/kernels.cu (k_dgs_*) bit for bit. */
/* side 1 (right): w = A P^-1 vt_j, Z_j = P^-1 vt_j.  side 0 (left,
 * gmres.cpp:69-71): w = P^-1 (A vt_j), Z_j = vt_j (scratch: N doubles); the
 * base r is then P^-1 r_k and its norm (alpha at j = 0) fixes the cycle's
 * tolerance rtol ||P^-1 b|| / ||P^-1 r_k|| (*hnorm = ||P^-1 b|| in cycle 0). */
static void dcgs2_cycle(const or_sys* S, long N, int R, int budget, double* V, double* Z,
                        double* H, double* g, double* cs, double* sn, double* s_, double* p_,
                        const double* r, double* hnorm, double* beta_io, double tol_c, int cycles,
                        int* total, int* m_out, int* stop_out, double* final_rel, double* hist,
                        int side, double rtol, double* scratch, double* zs) {
    double beta = *beta_io;
    memcpy(V, r, sizeof(double) * N); /* vt_0 = r, unnormalised */
    int j = 0, stop = 0;
    double* col = (double*)malloc(sizeof(double) * (R + 2));
    while (1) {
        double* vt = V + (long)j * N;
        double* w = V + (long)(j + 1) * N;
        if (side == 0) {
            memcpy(Z + (long)j * N, vt, sizeof(double) * N);
            or_stage_apply(S, vt, scratch);
            or_precond_apply(S, scratch, w);
        } else {
            or_precond_apply(S, vt, Z + (long)j * N);
            or_stage_apply(S, Z + (long)j * N, w);
        }
        for (int i = 0; i < j; ++i) {
            s_[i] = or_dot(V + (long)i * N, vt, N);
            p_[i] = or_dot(V + (long)i * N, w, N);
        }
        const double sig = or_dot(vt, vt, N);
        const double pi = or_dot(vt, w, N);
        double ss = 0.0, sp = 0.0;
        for (int i = 0; i < j; ++i) ss += s_[i] * s_[i];
        for (int i = 0; i < j; ++i) sp += s_[i] * p_[i];
        const double a2 = sig - ss;
        const double alpha = a2 > 0.0 ? sqrt(a2) : 0.0;
        if (j == 0) {
            beta = alpha;
            g[0] = beta;
            if (side == 0) {
                if (cycles == 0) {
                    *hnorm = alpha;
                    tol_c = rtol;
                } else {
                    tol_c = rtol * *hnorm / alpha;
                }
            }
        } else {
            double* hc = H + (long)(j - 1) * (R + 1);
            for (int i = 0; i < j; ++i) hc[i] = hc[i] + s_[i];
            hc[j] = alpha;
            givens_column(hc, j - 1, cs, sn, g);
            *total += 1;
            const double res_rel = fabs(g[j]) / beta;
            const double hv = cycles == 0 ? res_rel : res_rel * beta / *hnorm;
            if (hist) hist[*total] = hv;
            *final_rel = hv;
        }
        const double hjj = alpha > 0.0 ? (pi - sp) / alpha : 0.0;
        const double inv = alpha > 0.0 ? 1.0 / alpha : 0.0;
        /* column j (input Z_j = P^-1 vt_j) stored for the unit input: / alpha;
         * the next direction is stored / alpha as well, x uses y_j / alpha_j */
        double* hcj = H + (long)j * (R + 1);
        for (int i = 0; i < j; ++i) hcj[i] = p_[i] * inv;
        hcj[j] = hjj * inv;
        zs[j] = inv;
        for (long k = 0; k < N; ++k) {
            double v = vt[k], ww = w[k];
            for (int i = 0; i < j; ++i) {
                const double vi = V[(long)i * N + k];
                v = v - s_[i] * vi;
                ww = ww - p_[i] * vi;
            }
            v = v * inv;
            ww = (ww - hjj * v) * inv;
            vt[k] = v;
            w[k] = ww;
        }
        const double wn = sqrt(or_dot(w, w, N));
        /* provisional test on the first-pass column */
        for (int i = 0; i <= j; ++i) col[i] = hcj[i];
        col[j + 1] = wn;
        {
            double gj = g[j], gn;
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * col[i] + sn[i] * col[i + 1];
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
                col[i] = t;
            }
            const double denom = hyp(col[j], col[j + 1]);
            const double sv = denom > 0.0 ? col[j + 1] / denom : 0.0;
            gn = -sv * gj;
            const double res_prov = fabs(gn) / beta;
            const int bad = !(res_prov == res_prov) || !(wn == wn) || !(alpha == alpha);
            if (res_prov <= tol_c) stop = 1;
            else if (wn <= 1e-14 * beta || bad || alpha == 0.0) stop = 2;
            else if (j + 1 >= budget) stop = 3;
            else stop = 0;
        }
        if (stop) break;
        j += 1;
    }
    /* finalise column j against the fully orthogonal v_0..v_j */
    {
        double* w = V + (long)(j + 1) * N;
        for (int i = 0; i <= j; ++i) s_[i] = or_dot(V + (long)i * N, w, N);
        const double sig = or_dot(w, w, N);
        double ss = 0.0;
        for (int i = 0; i <= j; ++i) ss += s_[i] * s_[i];
        const double a2 = sig - ss;
        const double alpha = a2 > 0.0 ? sqrt(a2) : 0.0;
        double* hc = H + (long)j * (R + 1);
        for (int i = 0; i <= j; ++i) hc[i] = hc[i] + s_[i];
        hc[j + 1] = alpha;
        givens_column(hc, j, cs, sn, g);
        *total += 1;
        const double res_rel = fabs(g[j + 1]) / beta;
        const double hv = cycles == 0 ? res_rel : res_rel * beta / *hnorm;
        if (hist) hist[*total] = hv;
        *final_rel = hv;
        if (stop == 1 && !(res_rel <= tol_c)) stop = 3; /* provisional pass, final fail: restart */
        /* converged = final residual <= tol (gmres.cpp:139), also after a breakdown */
        if ((stop == 3 || stop == 2) && res_rel <= tol_c) stop = 1;
    }
    free(col);
    *m_out = j + 1;
    *stop_out = stop;
    *beta_io = beta;
}

int or_irk_step(const or_sys* S, const double* u, const double* lift, double rtol, int restart,
                int max_iter, double* u_next, double* K, or_report* rep, double* hist) {
    return or_irk_step_f(S, u, lift, NULL, 1, rtol, restart, max_iter, u_next, K, rep, hist);
}

int or_irk_step_f(const or_sys* S, const double* u, const double* lift, const double* forcing,
                  int side, double rtol, int restart, int max_iter, double* u_next, double* K,
                  or_report* rep, double* hist) {
    if (side == 0 && g_ortho != 1) return -1; /* left runs with delayed CGS2 only */
    struct timespec ts0, ts1;
    clock_gettime(CLOCK_MONOTONIC, &ts0);
    const int n = S->n, s = S->s;
    const long N = (long)s * n;
    if (restart <= 0 || restart > max_iter) restart = max_iter;
    const int R = restart;
    double* b = (double*)malloc(sizeof(double) * N);
    double* x = (double*)calloc(N, sizeof(double));
    double* r = (double*)malloc(sizeof(double) * N);
    double* ax = (double*)malloc(sizeof(double) * N);
    double* V = (double*)malloc(sizeof(double) * N * (R + 1));
    double* Z = (double*)malloc(sizeof(double) * N * (R > 0 ? R : 1));
    double* H = (double*)calloc((size_t)(R > 0 ? R : 1) * (R + 1), sizeof(double));
    double* g = (double*)calloc(R + 1, sizeof(double));
    double* cs = (double*)calloc(R + 1, sizeof(double));
    double* sn = (double*)calloc(R + 1, sizeof(double));
    double* h = (double*)calloc(R + 2, sizeof(double));
    double* cc = (double*)calloc(R + 2, sizeof(double));
    double* y = (double*)calloc(R + 1, sizeof(double));
    double* zs = (double*)calloc(R + 1, sizeof(double)); /* DCGS2 column scales */
    double* ys = (double*)calloc(R + 1, sizeof(double));

    /* stage right-hand side (irk.cpp:9-33): blk = -(F u + lift), then
     * blk += 1.0 * forcing(t_n + c_q ht) (forcing: s*n stage-major, or NULL) */
    {
        double* ku = (double*)malloc(sizeof(double) * n);
        or_spmv(&S->K, u, ku);
        for (int i = 0; i < n; ++i) {
            double f = ku[i];
            if (lift) f = f + lift[i];
            for (int q = 0; q < s; ++q) {
                const long k = (long)q * n + i;
                b[k] = forcing ? -f + forcing[k] : -f;
            }
        }
        free(ku);
    }
    memcpy(r, b, sizeof(double) * N);
    const double bnorm = sqrt(or_dot(b, b, N));
    double hnorm = bnorm; /* history / tolerance base (left: ||P^-1 b||, set in cycle 0) */
    double* base = side == 0 ? (double*)malloc(sizeof(double) * N) : NULL;
    int total = 0, cycles = 0, nre = 0, converged = 0, stop = 0;
    double beta = bnorm, tol_c = rtol, final_rel = 1.0, true_rel = 0.0;
    if (hist) hist[0] = 1.0;
    if (bnorm == 0.0) {
        converged = 1;
        final_rel = 0.0;
        if (hist) hist[0] = 0.0;
    } else {
        int budget = R < max_iter ? R : max_iter;
        double inv = 1.0 / bnorm;
        while (budget > 0) {
            int j = 0, m = 0;
            stop = 0;
            if (g_ortho == 1) {
                if (side == 0) or_precond_apply(S, r, base); /* left: base P^-1 r_k */
                dcgs2_cycle(S, N, R, budget, V, Z, H, g, cs, sn, h, cc, side == 0 ? base : r,
                            &hnorm, &beta, tol_c, cycles, &total, &m, &stop, &final_rel, hist,
                            side, rtol, ax, zs);
                nre += m;
                goto cycle_end;
            }
            for (long k = 0; k < N; ++k) V[k] = r[k] * inv;
            g[0] = beta;
            while (1) {
                double* vj = V + (long)j * N;
                double* zj = Z + (long)j * N;
                double* w = V + (long)(j + 1) * N;
                or_precond_apply(S, vj, zj);
                or_stage_apply(S, zj, w);
                for (int i = 0; i <= j; ++i) h[i] = or_dot(V + (long)i * N, w, N);
                const double before = sqrt(or_dot(w, w, N));
                for (long k = 0; k < N; ++k) {
                    double t = w[k];
                    for (int i = 0; i <= j; ++i) t = t - h[i] * V[(long)i * N + k];
                    w[k] = t;
                }
                double hnext = sqrt(or_dot(w, w, N));
                if (hnext < 0.70710678118654752 * before) {
                    for (int i = 0; i <= j; ++i) cc[i] = or_dot(V + (long)i * N, w, N);
                    for (long k = 0; k < N; ++k) {
                        double t = w[k];
                        for (int i = 0; i <= j; ++i) t = t - cc[i] * V[(long)i * N + k];
                        w[k] = t;
                    }
                    for (int i = 0; i <= j; ++i) h[i] = h[i] + cc[i];
                    hnext = sqrt(or_dot(w, w, N));
                    nre += 1;
                }
                /* Givens (gmres.cpp:93-112) */
                h[j + 1] = hnext;
                for (int i = 0; i < j; ++i) {
                    const double t = cs[i] * h[i] + sn[i] * h[i + 1];
                    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
                    h[i] = t;
                }
                const double denom = hyp(h[j], h[j + 1]);
                double c = 1.0, sv = 0.0;
                if (denom > 0.0) {
                    c = h[j] / denom;
                    sv = h[j + 1] / denom;
                }
                cs[j] = c;
                sn[j] = sv;
                h[j] = denom;
                h[j + 1] = 0.0;
                g[j + 1] = -sv * g[j];
                g[j] = c * g[j];
                for (int i = 0; i <= j + 1; ++i) H[(long)j * (R + 1) + i] = h[i];
                total += 1;
                m = j + 1;
                const double res_rel = fabs(g[j + 1]) / beta;
                const double hv = cycles == 0 ? res_rel : res_rel * beta / hnorm;
                if (hist) hist[total] = hv;
                final_rel = hv;
                const int bad = !(res_rel == res_rel) || !(hnext == hnext);
                if (res_rel <= tol_c) stop = 1;
                else if (hnext <= 1e-14 * beta || bad) stop = 2;
                else if (j + 1 >= budget) stop = 3;
                else stop = 0;
                if (stop) break;
                const double hinv = 1.0 / hnext;
                for (long k = 0; k < N; ++k) w[k] = w[k] * hinv;
                j += 1;
            }
        cycle_end:
            /* y = H^-1 g, x += Z y (gmres.cpp:126-132, flexible form) */
            for (int i = m - 1; i >= 0; --i) {
                double acc = g[i];
                for (int k = i + 1; k < m; ++k) acc -= H[(long)k * (R + 1) + i] * y[k];
                y[i] = acc / H[(long)i * (R + 1) + i];
            }
            for (int i = 0; i < m; ++i) ys[i] = g_ortho == 1 ? y[i] * zs[i] : y[i];
            for (long k = 0; k < N; ++k) {
                double t = x[k];
                for (int i = 0; i < m; ++i) t = t + ys[i] * Z[(long)i * N + k];
                x[k] = t;
            }
            or_stage_apply(S, x, ax);
            for (long k = 0; k < N; ++k) r[k] = b[k] - ax[k];
            const double rn = sqrt(or_dot(r, r, N));
            cycles += 1;
            true_rel = rn / bnorm;
            if (stop == 1 || stop == 2 || total >= max_iter || rn == 0.0) {
                converged = stop == 1;
                break;
            }
            (void)inv;
            beta = rn;
            tol_c = rtol * bnorm / rn;
            const int left = max_iter - total;
            budget = R < left ? R : left;
            inv = 1.0 / rn;
        }
    }
    /* u_{n+1} = u_n + ht sum_i b_i K_i (irk.cpp:59-65) */
    double hb[7];
    for (int q = 0; q < s; ++q) hb[q] = S->ht * S->b[q];
    for (int i = 0; i < n; ++i) {
        double acc = u[i];
        for (int q = 0; q < s; ++q) acc = acc + hb[q] * x[(long)q * n + i];
        u_next[i] = acc;
    }
    if (K) memcpy(K, x, sizeof(double) * N);
    clock_gettime(CLOCK_MONOTONIC, &ts1);
    if (rep) {
        rep->iterations = total;
        rep->cycles = cycles;
        rep->n_reorth = nre;
        rep->converged = converged;
        rep->true_rel = true_rel;
        rep->final_rel = final_rel;
        rep->seconds = (ts1.tv_sec - ts0.tv_sec) + 1e-9 * (ts1.tv_nsec - ts0.tv_nsec);
    }
    free(b); free(x); free(r); free(ax); free(V); free(Z); free(H); free(base);
    free(g); free(cs); free(sn); free(h); free(cc); free(y); free(zs); free(ys);
    return 0;
}
