/* awg_cuda.h — C ABI of the B200-native AWG-PCG hot path.
 *
 * One opaque context owns all device memory and one CUDA stream; it is used
 * from one host thread at a time (the reference is single-threaded and its
 * applies are const after setup).  Plain pointers and sizes
 * only; no CUDA or C++ types cross this boundary.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/proj/):
 *   awg_set_matrix      SparseSymMatrix (include/awg/sparse.hpp:12-21); the
 *                       read_matrix_market product (src/sparse.cpp:89-119)
 *   awg_set_partition   Partition + build_pou + check_minimal_overlap
 *                       (include/awg/partition.hpp:14-41; src/partition.cpp:94-156;
 *                       validation as in src/harness.cpp:85-91)
 *   awg_setup           ProblemContext::ProblemContext / h2 / second_coarse
 *                       (src/harness.cpp:100-124): Splitting (src/splitting.cpp:86-105),
 *                       build_coarse (src/coarse.cpp:113-154), build_w
 *                       (src/preconditioner.cpp:84-128), AwgPreconditioner ctor (:130-147)
 *   awg_load_factors    the same products taken from an external factorization
 *                       (apply-parity protocol)
 *   awg_apply           ApplyFn (include/awg/operators.hpp:8) for spmv (src/sparse.cpp:49-56),
 *                       Splitting::apply_Aminus/apply_Aplus (src/splitting.cpp:119-147),
 *                       OneLevel::apply (src/preconditioner.cpp:32-57), coarse_correct
 *                       (src/coarse.cpp:156-166), TwoLevel::apply (src/preconditioner.cpp:64-82),
 *                       AwgPreconditioner::second_correct/apply/apply_pi3(_transpose)
 *                       (src/preconditioner.cpp:149-221)
 *   awg_pcg             pcg (include/awg/krylov.hpp:34-36; src/krylov.cpp:36-124) with
 *                       apply_a = spmv and apply_h = H3 (src/harness.cpp:137-139)
 *   awg_query / awg_get_*   SolveReport fields and the report quantities of
 *                       src/harness.cpp:151-204 (subdomain sizes, n^s_-, coarse dim/rank,
 *                       W inner iterations, ...)
 *
 * Return codes mirror the reference's exceptions: AWG_E_NOT_SPD carries the
 * pivot index (NotSpdError, include/awg/dense.hpp:58-63; awg_last_error_index),
 * AWG_E_BREAKDOWN and AWG_E_NO_CONVERGENCE are the std::runtime_error paths of
 * pcg/build_w, AWG_E_OVERLAP the minimal-overlap check, AWG_E_ARG the
 * std::invalid_argument paths. */
#ifndef AWG_CUDA_H_
#define AWG_CUDA_H_

#ifdef __cplusplus
extern "C" {
#endif

enum awg_status {
  AWG_OK = 0,
  AWG_E_ARG = 1,            /* std::invalid_argument */
  AWG_E_CUDA = 2,           /* device failure (no CPU fallback exists) */
  AWG_E_NOT_SPD = 3,        /* NotSpdError(pivot) */
  AWG_E_BREAKDOWN = 4,      /* pcg: <p,Ap> <= 0 or <r,Hr> <= 0 */
  AWG_E_NO_CONVERGENCE = 5, /* build_w inner PCG / eigensolver */
  AWG_E_OVERLAP = 6,        /* minimal overlap violated / uncovered dof */
  AWG_E_STATE = 7           /* call order (e.g. apply before setup) */
};

enum awg_op {
  AWG_OP_A = 0,      /* y = A x                          spmv */
  AWG_OP_AMINUS = 1, /* y = A- x                         Splitting::apply_Aminus */
  AWG_OP_APLUS = 2,  /* y = A+ x                         Splitting::apply_Aplus */
  AWG_OP_H1 = 3,     /* one-level NN                      OneLevel::apply */
  AWG_OP_Q = 4,      /* Z K0^+ Z^T x                      coarse_correct */
  AWG_OP_QW = 5,     /* W KW^+ W^T x                      second_correct */
  AWG_OP_H2 = 6,     /* two-level                         TwoLevel::apply */
  AWG_OP_H3 = 7,     /* AWG (mode from the config)        AwgPreconditioner::apply */
  AWG_OP_PI3 = 8,    /* x - W KW^+ W^T A x                apply_pi3 */
  AWG_OP_PI3T = 9    /* x - A W KW^+ W^T x                apply_pi3_transpose */
};

enum awg_ptr_kind { AWG_PTR_HOST = 0, AWG_PTR_DEVICE = 1 };

/* PreconditionerConfig (include/awg/preconditioner.hpp:21-31) plus the
 * selection / semantics switches of SURVEY.md §8d and §7. */
typedef struct awg_config {
  int one_level;      /* 0 AS, 1 AS_PLUS, 2 NN (OneLevelKind; NN is the measured path) */
  int composition;    /* 0 ADDITIVE, 1 HYBRID */
  int use_coarse;     /* 0/1 */
  double tau_sharp;   /* NN threshold, (0,1) */
  double tau_flat;    /* AS_PLUS / AS threshold, > 1 */
  int fixed_k;        /* > 0: fixed-k GenEO rule k_s = max(k, n_nonpos(s)) + cluster closing */
  int awg_mode;       /* 0 NONE, 1 AD, 2 HYB, 3 INEX (AwgMode) */
  double w_rtol;      /* inner PCG tolerance for W (default 1e-10) */
  int w_maxit_factor; /* inner maxit = factor * n (default 10) */
  int rrf_semantics;  /* 0: reference pivoted factor (dense.cpp:299-346, swap of stale
                         upper values included); 1: exact pivoted Cholesky */
  int lu_semantics;   /* INEX core solve: 0 reference lu_solve (dense.cpp:395-410), 1 exact */
} awg_config;

/* Setup products from an external factorization (row-major nothing: every
 * dense block is column-major with leading dimension = its row count). */
typedef struct awg_factors {
  const double* lam;          /* sum n_s: eigenvalues of B^s, ascending, snapped */
  const double* V;            /* sum n_s^2: eigenvectors of B^s, column-major per s */
  const int* n_nonpos;        /* N */
  const int* n_zero;          /* N */
  const int* ks;              /* N: coarse columns per subdomain */
  const double* Y;            /* sum n_s k_s: GenEO vectors (MB-normalised), col-major per s */
  int r0;                     /* rank of K0 */
  const int* k0_retained;     /* r0 */
  const double* k0_l11;       /* r0 x r0 lower, col-major */
  int n_minus;                /* columns of W */
  const double* W;            /* n x n_minus col-major */
  const double* neg_weights;  /* n_minus: -lambda > 0 per column (INEX core) */
  const double* v_minus;      /* n x n_minus col-major (INEX core) */
  int rw;                     /* rank of KW */
  const int* kw_retained;     /* rw */
  const double* kw_l11;       /* rw x rw lower, col-major */
} awg_factors;

/* SolveReport (include/awg/krylov.hpp:14-28), scalar part. */
typedef struct awg_solve_report {
  int iterations;
  int converged;
  double final_relative_residual;
  double recurrence_residual_at_exit;
  double ritz_min;
  double ritz_max;
  double kappa_estimate;
  double solve_ms;  /* device time of the solve (CUDA events) */
} awg_solve_report;

typedef struct awg_stats {
  int n, nnz, n_sub;
  int n0;          /* coarse dimension #V0 */
  int r0;          /* retained rank of K0 */
  int n_minus;     /* n_- */
  int rw;          /* retained rank of KW */
  long long sum_ns;     /* sum n_s */
  long long sum_ns2;    /* sum n_s^2 (V^s entries) */
  long long sum_ns_ks;  /* block-sparse Z entries */
  long long sum_ns_ms;  /* sum n_s * n_nonpos(s) */
  long long sum_ns_qs;  /* sum n_s * n_neg(s) */
  double t_setup_ms[8]; /* splitting, pencils, coarse, w, misc... (see awg_setup) */
  int w_inner_total;    /* sum of inner PCG iterations of build_w */
  int w_batches;        /* block passes of the batched W build (continuous batching) */
  int nn_single_pass;   /* 1: the NN local solve streams V^s once per apply (k_nn_fused) */
  int nn_static_split;  /* 1: k_nn_fused runs equal static byte shares per CTA (no work queue) */
  int coarse_az;        /* 1: the hybrid H2's post-solve half uses the precomputed A Z (option coarse_az) */
} awg_stats;

int awg_create(struct awg_ctx** ctx, int device);
void awg_destroy(struct awg_ctx* ctx);
const char* awg_last_error(const struct awg_ctx* ctx);
int awg_last_error_index(const struct awg_ctx* ctx);

int awg_set_matrix(struct awg_ctx* ctx, int n, const int* row_offsets, const int* col_indices,
                   const double* values);
/* offsets: N+1 (int64), indices: sorted, duplicate-free global dofs per subdomain */
int awg_set_partition(struct awg_ctx* ctx, int n_sub, const long long* offsets, const int* indices);

/* GPU-side problem assembly, an alternative to
 * awg_set_matrix / awg_set_partition for the benchmark generators:
 *   awg_assemble_fd         cell-centred 5-point (dims 2) / 7-point (dims 3) diffusion
 *                           with harmonic face coefficients; shape = cells per
 *                           axis, cell_coef lexicographic (x fastest), host memory
 *   awg_assemble_elasticity Q1 plane strain, h = 1 (assemble, src/fem.cpp:99-162, with the
 *                           element formula of fem.cpp:53-97 and TripletBuilder's summation
 *                           order, src/sparse.cpp:19-47); element row ey uses material
 *                           (ey / layer_thickness) % n_materials; load = body force (2);
 *                           the assembled rhs is awg_get_array(16)
 *   awg_partition_owner     Omega^s = disjoint owners grown by `overlap` rings of matrix-graph
 *                           closure (src/partition.cpp:79-90), computed on the device
 *   awg_partition_boxes     the same with box owners of the assembled grid / mesh nodes
 * Built on the device, then installed exactly as awg_set_matrix / awg_set_partition
 * would (same validation, same errors). */
int awg_assemble_fd(struct awg_ctx* ctx, int dims, const int* shape, const double* cell_coef);
int awg_assemble_elasticity(struct awg_ctx* ctx, int nodes_x, int nodes_y, int layer_thickness, int n_materials,
                            const double* young, const double* poisson, const double* load);
int awg_partition_owner(struct awg_ctx* ctx, const int* owner, int n_sub, int overlap);
int awg_partition_boxes(struct awg_ctx* ctx, const int* boxes, int overlap);

/* Experiment switches for tests and profiles (no reference counterpart; the
 * product defaults are frozen in the library and no environment variable is
 * read).  Names: pdl, nn_two_pass, fused_cpb, fused_hold, fused_prefetch,
 * fused_static, fused_static_cols, pcg_adaptive, pdl_local, pdl_early,
 * rows_group, w_split, fused_nbuf, fused_chunks, fused_reserve,
 * fused_min_cols, fused_tail, synth_nm, dgemm_variant, coarse_neg, verbose,
 * wbuild_cublas, setup_cusolver (1: cuSOLVER eigensolvers / Cholesky in the
 * setup instead of the hand-written ones, for A/B checks).  Unknown names return AWG_E_ARG. */
int awg_set_option(struct awg_ctx* ctx, const char* name, long long value);

int awg_setup(struct awg_ctx* ctx, const awg_config* cfg);

/* rank_revealing_sym_factor (src/dense.cpp:299-346; RankRevealingFactor,
 * include/awg/dense.hpp:78-89) on a caller-supplied symmetric n x n G
 * (column-major, host): the device pivoted factor that awg_setup runs on
 * Z^T A+ Z (coarse.cpp:145-152) and W^T A W (preconditioner.cpp:119-126),
 * exposed so its retained set can be checked directly.  exact = 0: the
 * reference's semantics (stale-upper swap), 1: exact pivoted Cholesky.
 * Writes rank r, retained[r] (pivot order) and l11[r*r] (lower, column-major;
 * caller sizes both for r = n). */
int awg_pivoted_factor(struct awg_ctx* ctx, int n, const double* G, int exact, int* rank, int* retained,
                       double* l11);
int awg_load_factors(struct awg_ctx* ctx, const awg_config* cfg, const awg_factors* f);

int awg_apply(struct awg_ctx* ctx, int op, const double* x, double* y, int ptr_kind);
/* rank_revealing_solve (src/dense.cpp:348-366) with the factor awg_setup built:
 * which = 0 K0 (dimension n0, coarse.cpp:156-166), 1 KW (n_minus,
 * preconditioner.cpp:149-159); b and x host vectors of that dimension. */
int awg_coarse_solve(struct awg_ctx* ctx, int which, const double* b, double* x);
int awg_pcg(struct awg_ctx* ctx, const double* b, double* x, double rtol, int maxit, int ptr_kind,
            awg_solve_report* report);

int awg_query(struct awg_ctx* ctx, awg_stats* stats);
/* History of the last awg_pcg: residuals (relative, recursive), Lanczos
 * diagonal / off-diagonal; returns the number of entries written. */
int awg_get_history(struct awg_ctx* ctx, int which /*0 resid,1 diag,2 offdiag*/, double* out, int cap);
/* Setup products (for parity checks / reports).  which:
 *  0 lam (sum n_s)   1 n_nonpos (N, int)   2 n_zero (N, int)  3 ks (N, int)
 *  4 pencil eigenvalues (sum n_s)          5 multiplicity (n, int)
 *  6 k0_retained (r0, int)  7 k0_l11 (r0*r0)  8 kw_retained (rw, int)  9 kw_l11 (rw*rw)
 *  10 W (n*n_minus)  11 neg_weights (n_minus)  12 w_inner_iterations (n_minus, int)
 *  13 Y (sum n_s k_s)  14 V (sum n_s^2)  15 eps_zero (N)  16 assembled rhs (n)
 *  17 row_offsets (n+1, int)  18 col_indices (nnz, int)  19 values (nnz)
 *  20 partition offsets (N+1, int)  21 partition indices (sum n_s, int) */
int awg_get_array(struct awg_ctx* ctx, int which, void* out, long long cap_elems, long long* n_elems);

/* Kernel launches issued by this context since creation (product kernels only). */
long long awg_launch_count(const struct awg_ctx* ctx);
/* Device time (ms) of the last apply loop: runs op `reps` times on device buffers. */
int awg_time_apply(struct awg_ctx* ctx, int op, int reps, double* ms_per_apply);
/* Device time (ms per launch, CUDA events on the context stream) of one hot
 * kernel launched `reps` times back to back: 0 batched NN GEMV^T (V^s^T x),
 * 1 batched NN GEMV (V^s u), 2 CSR SpMV, 3 W^T x, 4 W c, 5 single-pass NN
 * local solve (V^s streamed once).  Also returns the
 * algorithmic bytes one launch must move (operands read once, results written). */
int awg_time_kernel(struct awg_ctx* ctx, int which, int reps, double* ms_per_launch, double* bytes_per_launch);
/* In-kernel launch timer of the single-pass local solve (%globaltimer, first
 * CTA start to last CTA end, accumulated over every launch, graphs included):
 * total ms and launch count since the last reset. */
int awg_kernel_timer(struct awg_ctx* ctx, int reset, double* ms_total, long long* launches);
/* Benchmark hook: synthetic local factors (V^s filled on the device with
 * pseudo-random values, n_nonpos = m_per_sub zero modes, no coarse spaces) so
 * the local-solve kernels can be timed at full scale without the setup. */
int awg_synthetic_factors(struct awg_ctx* ctx, int m_per_sub, unsigned long long seed);
/* Benchmark / check hook of the setup's grouped FP64 tensor-core GEMM
 * (dgemm.cu; the W build's block one-level P^s X^s, preconditioner.cpp:97-113):
 * `count` column-major products C = A B (A m x k, B k x n; with transpose_a,
 * C = A^T B with A stored k x m — the W^T A W assembly), seeded pseudo-random
 * values, in one grouped launch, timed over `reps` launches and checked against
 * cuBLAS DGEMM on the same operands.  out[0] max |C - C_cublas| / max |C_cublas|,
 * out[1] ms per grouped launch, out[2] ms for the same products as `count`
 * cuBLAS calls, out[3] grouped TFLOP/s, out[4] cuBLAS TFLOP/s. */
/* Check / benchmark hook of the setup's batched symmetric eigensolver (eig.cu,
 * the dense_sym_eig of dense.cpp:117-209 for B^s and the GenEO pencils):
 * `count` seeded symmetric matrices of order n (kind 0 random, 1 the 5-point
 * Laplacian of a sqrt(n) x sqrt(n) grid with repeated eigenvalues, 2 graded
 * spectrum), checked against cuSOLVER Dsyevd on the same matrices.
 * out[0] max eigenvalue error / ||A||, out[1] max residual ||A z - w z|| / ||A||,
 * out[2] max |Z^T Z - I|, out[3] ms for the batch, out[4] cuSOLVER ms. */
int awg_bench_eig(struct awg_ctx* ctx, int n, int count, int kind, unsigned long long seed, double* out);
int awg_bench_dgemm(struct awg_ctx* ctx, int m, int n, int k, int count, int transpose_a, int reps, double* out);

#ifdef __cplusplus
}
#endif

#endif /* AWG_CUDA_H_ */
