// Kernel interface of the B200 IRK solve phase (fp64, HBM-bound, CUDA cores).
// Each launcher enqueues on the given stream; none synchronises.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace irkb {
namespace dev {

constexpr int kMaxDiags = 16;
constexpr int kRsQ = 1 << 30;  // RSIG offset flag: second operand

// Device matrix formats.  Both keep the reference's per-row summation order
// (column-ascending, sequential), so results are bit-identical to a CSR row
// sum:
//   DIA  -- a few constant diagonals (the fine-level FE stencils: M, K and
//           every fine-level A); entries stored diagonal-major, no indices.
//   SELL -- SELL-32: slices of 32 consecutive rows padded to the slice's
//           longest row, stored column-major inside the slice, so a warp
//           streams one slice fully coalesced with one thread per row
//           (short rows: the prolongators).
//   CSRV -- plain CSR, G lanes per row (long rows: restrictions and the
//           Galerkin coarse operators).
// Values are fp64 or, when the matrix has few distinct values, uint8 /
// uint16 codes into an exact fp64 dictionary (lossless; e.g. 3 distinct
// values in the fine-level stencils, 14 in the fine prolongator).
//   RSIG -- row signatures (composed operators on structured grids): rows
//           whose column offsets (relative to the row's first column; for a
//           split operand relative to the first column of each half) and
//           fp64 values are identical share one signature, stored once; a
//           row is its signature id and its base column(s).  Lossless; the
//           row sums keep the lane-tree order of the CSR form.
enum MatFmt { kSell = 0, kDia = 1, kCsrVec = 2, kRowSig = 3 };
// kCls (DIA with 7 diagonals only): one u8 row class per row; rows of one
// class have the identical stencil, stored once in tab[class * nd + d]
// (lossless: a class is a distinct tuple of fp64 bit patterns).  On the
// uniform P1 grid nearly every row is interior, so a row costs one byte and
// one coalesced load instead of nd codes.
// kP8 (composed operators with value codes): the dictionary code rides in the
// top bits of the column index word (Mat::pk_shift = 32 - code bits; the
// columns fit below), one 4-byte load per entry and no separate value stream.
enum ValFmt { kF64 = 0, kU8 = 1, kU16 = 2, kCls = 3, kP8 = 4 };

struct Mat {
    int fmt = kSell;
    int vf = kF64;
    int rows = 0, cols = 0, nnz = 0;
    // SELL-32
    const int* sptr = nullptr;  // slice offsets (entries), rows/32 + 1
    const int* idx = nullptr;   // column per stored entry (SELL / CSR)
    // CSR-vector: G lanes per row load the row at once; the row sum is then
    // accumulated in column order through warp shuffles
    const int* ptr = nullptr;   // row offsets, rows + 1
    int lanes = 1;
    // lane-tree row sums (the composed V-cycle operators, compose.cpp): each
    // of the `lanes` lanes adds its strided entries in order, then an xor
    // butterfly folds the lanes (k_spmv_lt) -- part of the operator's
    // definition, restated by the oracle.  0: not a lane-tree operator; else the
    // entries staged per lane and row by the pipelined kernel (4..6, a tuning
    // hint: about the 95th percentile row length / lanes)
    int tree = 0;
    int pk_shift = 24;  // kP8: column = word & (2^pk_shift - 1), code = word >> pk_shift
    // RSIG: per row the signature id and base columns; per signature its
    // length and `rs_w` slots of (offset, value); an offset with kRsQ set is
    // relative to base1 and addresses the second operand (x2) of a split product
    const unsigned short* rs_sig = nullptr;
    const int* rs_base0 = nullptr;
    const int* rs_base1 = nullptr;
    const int* rs_len = nullptr;
    const int* rs_off = nullptr;
    const double* rs_val = nullptr;
    int rs_w = 0, rs_n = 0;
    // values (both formats): f64 / u8 / u16 per stored entry
    const void* val = nullptr;
    const double* tab = nullptr;  // code dictionary (vf != kF64)
    int ntab = 0;
    int tab_smem = 0;             // u8: stage the dictionaries in shared memory per CTA
    // DIA
    int nd = 0;
    int off[kMaxDiags] = {};
    int diag0 = -1;                 // slot of offset 0
    long long dstride = 0;          // entries per stored diagonal (>= rows, multiple of 4)
    const double* wdtab = nullptr;  // omega / diagonal value per code (DIA, u8)
    // kCls hierarchy operators: per class, omega / a_cc of each diagonal's
    // partner row (0 where the coefficient is 0), so wd .* r needs no
    // neighbour class lookups
    const double* nbwd = nullptr;
    // kCls: the most frequent class (the interior stencil of a uniform grid)
    // also travels in the kernel parameters -- a warp whose rows all have it
    // takes its stencil, partner omega / a_cc and omega / a_ii from the
    // constant bank instead of 15 class-table loads per row
    int dom = -1;
    double dom_tab[7] = {};
    double dom_nbwd[7] = {};
    double dom_wd = 0.0;
    size_t bytes = 0;               // device bytes of the stored operator
};

// x operand of an SpMV: either a plain vector or the implicit Jacobi
// pre-smoothed iterate wd .* r (never materialised).
// kXSplit (SELL / CSR-vector only): the operand is the concatenation
// [x (split entries); x2] of two vectors -- the composed up leg
// z_l = [S_l Q_l] [r_l; z_{l+1}] (csrc/host/compose.cpp).
enum XMode { kXPlain = 0, kXWdR = 1, kXSplit = 2 };
// Row epilogue applied to s = (A x)_i.
enum Epi {
    kEPlain = 0,    // y = s
    kEResid = 1,    // y = r - s
    kESmooth = 2,   // y = x + wd*(r - s)        (Jacobi sweep, x = input)
    kEProlong = 3,  // y = zb + s,  zb = wd .* r (implicit) or a vector
};

struct SpmvArgs {
    VecRef x{};                  // plain x (kXPlain)
    VecRef x2{};                 // kXSplit: columns >= split read x2[col - split]
    int split = 0;
    VecRef r{};                  // residual / rhs vector
    const double* wd = nullptr;  // omega * D^-1
    const double* zb = nullptr;  // prolong base (nullptr -> wd .* r)
    VecRef y{};
    // optional second output y2 = wd2 .* y (a restriction also writes the
    // next level's pre-smoothed iterate wd .* r, so that level's residual
    // gathers one vector instead of two)
    double* y2 = nullptr;
    const double* wd2 = nullptr;
    // programmatic launch with the trigger at the END of each thread's work
    // (set by spmv() inside a set_pdl_late scope): the dependent grid's
    // launch overlaps this grid's last wave instead of taking its slots
    int late = 0;
};

// Algorithmic-bytes tally (the roofline's numerator): while a
// tally is open on this thread, every launcher adds the bytes its kernel must
// move -- each array it reads or writes once, in its STORED format (row
// classes, u8/u16 codes, SELL/CSR indices) -- as fixed + per_j * j, where j is
// the Arnoldi index (iteration kernels) or the cycle length m (cycle end).
struct Tally {
    double fixed = 0.0, per_j = 0.0;
};
void tally_open(Tally* t);
void tally_close();
// Bytes of one pass over the stored operator (values, indices, row structure).
double mat_bytes(const Mat& A);

// Programmatic dependent launch, opt-in via IRK_PDL=1.
bool pdl_enabled();
// Programmatic launch for the kernels recorded while the scope is on (the
// latency-bound coarse AMG levels, IRK_PDL_COARSE).
void set_pdl_scope(bool on);
// Kernels recorded while on are launched programmatically with the late
// trigger (SpmvArgs::late): the many-wave level-0/1 SpMVs (IRK_PDL_FINE).
void set_pdl_late(bool on);

void spmv(const Mat& A, int xmode, int epi, const SpmvArgs& a, cudaStream_t st);
// Composed up leg on a 7-point fine level: y = S x + Q x2, S stored as DIA row
// classes and Q as SELL-32, one thread per row, the row summed sequentially
// (S's diagonals in ascending offset order, then Q's entries in column order
// -- the CSR order of U = [S | Q]).
void up_cls(const Mat& S, const Mat& Q, const SpmvArgs& a, cudaStream_t st);

// Tuning switches: a runtime override (irk_set_option) or the environment
// variable of the same name, else `dflt`.  Read when a graph is recorded;
// every override bumps option_generation() so solvers re-record.
long long option(const char* name, long long dflt);
// diagnostic: last DCGS2 block-dot tail timestamps (builds with -DIRK_DGS_PROF)
void dgs_prof_read(long long* out);
void set_option(const char* name, long long value);
unsigned option_generation();

// Stage operator y_i = M z_i + sum_j c_ij K z_j (c = ht*A), M/K sharing one
// DIA pattern; one pass over both value arrays for all s stage vectors.
struct StageCoef {
    int s;
    double c[kMaxStages * kMaxStages];
};
void stage_op_dia(const Mat& M, const Mat& K, const StageCoef& c, VecRef z,
                  VecRef y, int n, cudaStream_t st);

// Block-substitution sweep, fused for DIA K:
//   fresh = K w;  store_fresh (optional) = fresh;
//   out = v + sum_t coef_t * term_t  (terms in the given order; the term
//   flagged `fresh` uses the value just computed).
struct SweepTerms {
    int nt;
    double coef[kMaxStages];
    const double* buf[kMaxStages];  // nullptr marks the fresh term
};
void sweep_dia(const Mat& K, VecRef w, VecRef v, const SweepTerms& t,
               double* store_fresh, VecRef out, int n, cudaStream_t st);
// Generic element-wise combine (used with a CSR K): out = v + sum coef*buf.
void combine(VecRef v, const SweepTerms& t, VecRef out, int n, cudaStream_t st);
// y += alpha * x, element-wise (rounded multiply then add).
void axpy(double alpha, const double* x, VecRef y, int n, cudaStream_t st);

// z = B r with the dense V-cycle tail operator (n x ld row-major, ld even;
// tail.cpp): one launch in place of the cycle below the tail level.
void tail_mv(int n, int ld, const double* B, const double* r, double* z, cudaStream_t st);
// Coarsest-level solve z = Ainv r (dense row-major inverse).
void dense_mv(int n, const double* Ainv, VecRef r, VecRef z, cudaStream_t st);

// Bottom of a V-cycle in one CTA (levels b..L-1 of a hierarchy whose
// operators fit in shared memory): residual, restriction, dense coarse solve,
// prolongation and smoothing with barriers between phases.  The operators are
// packed once into a blob (CSR, u16 column indices, fp64 values, 16-byte
// aligned arrays; offsets below are byte offsets into it) that the CTA copies
// to shared memory before waiting on its predecessor.
constexpr int kMaxBot = 4;
struct BotLevel {
    int n;
    int a_sell;               // A_l stored as SELL-32 (a_ptr = slice offsets, a_len = row lengths)
    int a_len;
    int a_ptr, a_idx, a_val;  // A_l
    int p_ptr, p_idx, p_val;  // P_l (n x n_{l+1})
    int r_ptr, r_idx, r_val;  // R_l (n_{l+1} x n)
    int wd;                   // omega / a_ii
};
struct BotDesc {
    const char* blob = nullptr;
    int bytes = 0;            // blob bytes (multiple of 16)
    int nl = 0;               // smoothed levels in the kernel (the dense one excluded)
    BotLevel lv[kMaxBot];
    int nc = 0, cinv = 0;     // coarsest size, dense inverse offset
    int vec = 0;              // smem offset of the level vectors
    int vr[kMaxBot + 1], vt[kMaxBot + 1], vz[kMaxBot + 1];  // per-level vector offsets
    int smem = 0;             // dynamic smem bytes
    long long* prof = nullptr; // optional phase timestamps (globaltimer ns, 16 slots)
};
void bottom_cycle(const BotDesc& d, const double* r_in, double* z_out, cudaStream_t st);
// Gauss-Seidel sweep (amg.cpp:125-140) of one level, level-scheduled: the
// rows are grouped by dependency depth (row i after every row j it reads
// updated: j < i forward, j > i backward) and stored in that order, the
// depths cut into chunks of <= kGsRows rows and <= kGsEnt padded entries
// (rows of one chunk are independent).  Per schedule position q:
// hdr[q] = {i, off-diagonal entries}, dinv[q] = 1 / a_ii; a chunk's entries
// are column-major (entry k of its row q at chunk base + k * rows + q,
// padded to the chunk's longest row; per row in CSR column order, the
// diagonal dropped as the reference skips it), each with its value and two
// static codes:
//   ref  (the gather)  -(2c+1): the not-yet-updated value of column c, else 0
//   sref (the sweep)   0 .. kGsRing-1: an updated value still in the
//                      kernel's ring of the last kGsRing computed rows (slot
//                      = position mod kGsRing); kGsRing: the gathered product
//                      (the ring's constant 1.0 slot); -(c+2): an updated
//                      value too old for the ring (zout[c]; `far` sweeps).
constexpr int kGsRows = 256, kGsEnt = 2048, kGsRing = 4096;
struct GsSweep {
    const int2* hdr = nullptr;   // n, schedule order
    const int* ref = nullptr;    // nnz gather codes
    const int* sref = nullptr;   // nnz sweep codes
    const double* val = nullptr; // nnz values
    const double* dinv = nullptr;
    const int* cptr = nullptr;   // nch + 1 chunk position offsets
    const int* ceptr = nullptr;  // nch + 1 chunk entry offsets (padded, rows x width)
    double* rs = nullptr;        // n: r in schedule order (written by the gather)
    double* ps = nullptr;        // nnz: the gathered entry operands
    int nch = 0, n = 0;
    int far = 0;                 // some operands older than the ring
    long long nnz = 0;           // stored (padded) entries
    long long* prof = nullptr;   // diagnostic: per-chunk phase clocks (time_kernel, IRK_GS_PROF)
};
// zout_i = (r_i - sum_{j != i} a_ij z_j) / a_ii in CSR column order, with z_j
// the updated value for j before i in sweep order and zin_j otherwise
// (zin == nullptr: the zero iterate of a cycle's first sweep).  zin and zout
// are different vectors (ping-pong), which gives exactly the in-place
// reference sweep.  Two launches: a parallel gather (r in schedule order;
// each not-yet-updated operand multiplied by its value -- the same rounded
// product the row sum subtracts) and the single-CTA sweep.
void gs_sweep(const GsSweep& S, bool backward, VecRef r, const double* zin, VecRef zout,
              cudaStream_t st);
// z = wd .* r (first Jacobi sweep from a zero iterate, amg.cpp:119-124).
void wd_times_r(int n, const double* wd, VecRef r, double* z, cudaStream_t st);

// b_q = -(K u + lift) + forcing_q for every stage q (irk.cpp:9-33); lift and
// forcing (s*n, stage-major) may be null.
void stage_rhs_finish(const double* ku, const double* lift, const double* forcing, double* b,
                      int n, int s, cudaStream_t st);
// u_next = u + sum_i hb_i x_i (irk.cpp:59-65).
void irk_update(const double* u, const double* x, const double* hb, int n, int s,
                double* u_next, cudaStream_t st);

// ------------------------------------------------------------------ GMRES
// Control block shared by every GMRES kernel (device memory).
struct GmresCtl {
    int j;          // inner iteration index within the cycle
    int j_next;
    int budget;
    int total;      // iterations so far
    int cycles;
    int stop;       // 0 continue, 1 converged, 2 breakdown, 3 budget
    int done;
    int converged;
    int reorth;     // current iteration re-orthogonalises
    int n_reorth;
    int restart, max_iter;
    int m;          // columns of the last cycle
    int bad;        // non-finite scalar seen
    double rel_tol, bnorm, beta, tol_c, inv, before, after, hnext;
    double final_rel, true_rel;
    double g[kMaxRestart + 1];
    double cs[kMaxRestart];
    double sn[kMaxRestart];
    double hcol[kMaxRestart + 2];
    double y[kMaxRestart];
    // delayed CGS2 (DCGS2) scalars of the current iteration
    double sv[kMaxRestart + 1];  // s_i = v_i . vt_j   (re-orthogonalisation of vt_j)
    double pv[kMaxRestart + 1];  // p_i = v_i . w      (projections of w)
    double hjj, inv_alpha;
    double zscale[kMaxRestart];  // DCGS2: x += sum_j y_j zscale_j Z_j (1 for CGS2)
    int ortho;                   // 1 DCGS2, 0 CGS + conditional second pass
    int side;                    // 1 right (flexible Z basis), 0 left (gmres.cpp:41-46, 69-71)
    double hnorm;                // history / tolerance base: ||b|| (right), ||P^-1 b|| (left)
};

struct GmresBufs {
    GmresCtl* ctl;
    double* H;          // (restart) columns of (restart+1)
    double* hist;       // max_iter + 1
    double* partials;   // (kMaxRestart + 2) * nchunks
    unsigned* counters; // one per reduction kernel
    double* V;          // (restart + 1) * sN
    double* Z;          // restart * sN
    long long sN;
    int nchunks;
    cudaGraphConditionalHandle h_inner;
    cudaGraphConditionalHandle h_outer;
    int use_cond;       // 1 when running inside conditional graph nodes
    int cap;            // restart capacity (sizes the DCGS2 reduction buffers)
};

// b -> r copy and ||b||; initialises the control block (bnorm == 0 ends the
// solve: x = 0).
void gm_init(const GmresBufs& g, const double* b, double* r, double rel_tol,
             int restart, int max_iter, int ortho, int side, cudaStream_t st);
// y = x for the basis slot x resolves to (sN values).
void copy_ref(VecRef x, VecRef y, long long n, cudaStream_t st);
// V_0 = r / beta, g_0 = beta, j = 0 (start of a restart cycle).
void gm_cycle_begin(const GmresBufs& g, const double* r, cudaStream_t st);
// h = V_{0..j}^T w and ||w||  (pass 1), or c = V^T w (pass 2, if reorth).
void gm_blockdot(const GmresBufs& g, int pass, cudaStream_t st);
// w -= V h (pass 1) / w -= V c, h += c (pass 2), ||w||, scalar tail.
void gm_update(const GmresBufs& g, int pass, cudaStream_t st);
// Delayed CGS2 (the default orthogonalisation): one fused block-dot
// (s = V_{j-1}^T vt_j, p = V_{j-1}^T w, vt_j.vt_j, vt_j.w; finalises column
// j-1) and one fused update (v_j, w') per iteration; `finalize` runs the
// cycle-end block-dot that completes the last column.
void gm_dgs_dot(const GmresBufs& g, int finalize, cudaStream_t st);
void gm_dgs_update(const GmresBufs& g, cudaStream_t st);
// V_{j+1} = w / h_{j+1,j} if continuing; advance j; set loop condition.
void gm_normalize(const GmresBufs& g, cudaStream_t st);
// y = H^-1 g (1 thread) then x += Z y.
void gm_solution(const GmresBufs& g, double* x, cudaStream_t st);
// r = b - Ax, beta = ||r||, restart decision.
void gm_residual(const GmresBufs& g, const double* b, const double* ax, double* r,
                 cudaStream_t st);

// Standalone deterministic dot (same tree) for tests: out[0] = x.y.
void dot(const double* x, const double* y, long long n, double* partials,
         unsigned* counter, double* out, cudaStream_t st);

}  // namespace dev
}  // namespace irkb
