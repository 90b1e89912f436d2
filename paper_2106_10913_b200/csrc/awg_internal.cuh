// Internal declarations of the B200-native AWG-PCG library (not part of the
// C ABI).  Device data layout (HBM), per context:
//
//   CSR A            rp[n+1] int32, ci[nnz] int32, va[nnz] f64    (sparse.hpp:12-21)
//   Partition        pidx[P] int32 (P = sum n_s, subdomains concatenated, each sorted),
//                    poff[N+1] int64; psub[P] subdomain of entry p
//   POU              ds[P] = 1/mu(pidx[p])  (partition.cpp:94-108)
//   Owner lists      own_off[n+1], own_pos[P]: entries p with pidx[p] == i in
//                    ascending s — the deterministic prolongation order of
//                    OneLevel::apply (preconditioner.cpp:37-55)
//   V^s              column-major, leading dimension ld_s = round_up(n_s, 4) (32-byte
//                    aligned columns, zero padding rows), block offsets voff[s]
//   lam              [P] eigenvalues of B^s, ascending, snapped (splitting.cpp:64-84)
//   A- modes         list of (s, k, -lambda_k) for k < n_nonpos(s), lambda_k != 0
//   Z (block sparse) Y_s column-major with the same ld_s, offsets yoff[s]; column
//                    j of Z = R^s^T Y_s(:, j - koff[s]) (coarse.cpp:136-141)
//   K0, KW           retained index lists and the inverse of the l11 factor (lower,
//                    r x r column-major) — the triangular solves of
//                    rank_revealing_solve (dense.cpp:348-366) become two triangular
//                    matrix-vector products
//   W                n x n_minus column-major, leading dimension round_up(n, 4)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/awg_cuda.h"

namespace awgb {

struct AwgError : std::runtime_error {
  int code;
  int index;
  AwgError(int c, const std::string& m, int idx = -1) : std::runtime_error(m), code(c), index(idx) {}
};

#define AWG_CUDA(x)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      throw ::awgb::AwgError(AWG_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw AwgError(AWG_E_CUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e));
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute of a
// kernel: remember what was set per (kernel, device) so a context on another
// GPU of the same process raises it there too.
inline void ensure_dyn_smem(const void* func, size_t bytes) {
  static std::map<std::pair<const void*, int>, size_t> done;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  AWG_CUDA(cudaGetDevice(&dev));
  size_t& have = done[{func, dev}];
  if (bytes > have) {
    AWG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    have = bytes;
  }
}

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  DArr() = default;
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  ~DArr() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) AWG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void zero(cudaStream_t s) {
    if (n) AWG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) AWG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  std::vector<T> download(cudaStream_t s) const {
    std::vector<T> h(n);
    if (n) AWG_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    AWG_CUDA(cudaStreamSynchronize(s));
    return h;
  }
};

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

struct Ctx;
int w_chunks(const Ctx& c);  // column chunks of the W c GEMV (enough CTAs for small n)

// Work items of the batched NN local solve.
struct GemvTTask {  // columns [j0, j1) of V^s
  int s, j0, j1, pad;
};
struct GemvTask {  // rows [i0, i0 + rows) x columns [j0, j1) of V^s, partial slot kc
  int s, i0, j0, j1, kc, pad;
};

// Work lists of one batched local solve (GEMV^T tasks, split GEMV tasks, column
// chunks per subdomain).
struct LocalPlan {
  DArr<GemvTTask> tT;
  DArr<GemvTask> t;
  DArr<int> nkc;
  int cols_max = 0;
  int kcmax = 1;
  // single-pass variant (k_nn_fused): column ranges per CTA, their chunk counts
  bool fused = false;
  DArr<GemvTask> tf;
  DArr<int> cta_off;    // static split (AWG_FUSED_STATIC): tasks of CTA b are [cta_off[b], cta_off[b + 1])
  int static_grid = 0;
  DArr<int> nkc_f;
  int kcmax_f = 1;
  DArr<int2> own_nkc, own_nkc_f;  // per owner entry: (p, nkc / nkc_f of its subdomain)
};

// Owner-list entries resolved once per factor load, so the prolongation kernels
// walk two dependent loads per dof (own_off, entry) instead of five
// (own_off, own_pos, psub, per-subdomain offsets, data).  OwnEnt: the block of
// subdomain s = psub[own_pos[q]] seen from that dof (column-major block, its
// leading dimension and the coefficient range of s); the int2 form for the
// local-solve partials: (p, chunk count of s).
struct OwnEnt {
  long long mbase;  // moff[s] + (p - poff[s])
  int L, q0, q1, pad;
};

// Grouped FP64 tensor-core GEMM (dgemm.cu): C = A B for a list of column-major
// problems in one launch (one CTA per 128 x 128 output tile of any problem).
struct GemmDesc {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
  int sub;    // 0: C = A B;  1: C = C - A B
  int lower;  // 1: only tiles that touch the lower triangle (m >= n) are computed
};
struct GemmTile {
  int prob, m0, n0, pad;
};
struct Ctx;
struct GroupedGemm {
  DArr<GemmDesc> desc;
  DArr<GemmTile> tiles;
  int ntiles = 0;
  bool ta = false;  // C = A^T B (A stored K x M, column-major)
  double flops = 0.0;
  // validates and uploads the tile list; transpose_a: every problem is C = A^T B
  void set(Ctx& c, const std::vector<GemmDesc>& probs, bool transpose_a = false);
  void run(Ctx& c) const;                                 // on c.stream
};

// Block-sparse GEMV^T plan (k_bs_gemvT): one CTA per (subdomain, 512-row
// chunk) over the subdomains that own columns; partials per (column, chunk),
// summed in chunk order by the last CTA of each subdomain.
constexpr int kBsRows = 512;  // rows per CTA (256 threads x 2)
struct BsPlan {
  DArr<int> ts, tc;  // task -> subdomain, chunk
  DArr<int> nch;     // chunks per subdomain
  DArr<int> cnt;     // CTAs finished per subdomain (reset by the last one)
  DArr<double> part; // columns x maxch
  int ntask = 0, maxch = 1;
  int ncg = 1;       // column groups of 8 (grid.y): the most columns of any subdomain / 8
};

// Triangular coarse factor with retained pivots (RankRevealingFactor,
// dense.hpp:81-86), stored as the inverse of l11.
struct CoarseFactor {
  int dim = 0;   // original dimension (n0 or n_minus)
  int rank = 0;  // r
  DArr<int> retained;
  DArr<double> linv;   // r x r, column-major, lower
  DArr<double> kinv;   // L^-T L^-1 (r x r, symmetric): K^+ on the retained pivots
  DArr<int> pos;       // dim: position among the retained pivots, -1 if dropped
  std::vector<int> h_retained;
  std::vector<double> h_l11;  // r x r, as produced (for exports)
  void clear() {
    dim = rank = 0;
    retained.release();
    linv.release();
    kinv.release();
    pos.release();
    h_retained.clear();
    h_l11.clear();
  }
};

// PCG state in device memory; every iteration kernel is gated on `done`.
struct PcgState {
  double bnorm, rz, pq, alpha, beta, relres, true_rel, alpha_prev, beta_prev;
  double final_rel, rec_exit, rtol;
  int it, maxit, done, converged, past_rtol, need_true, error, force_true;
};

enum PcgError { PCG_OK = 0, PCG_BAD_OPERATOR = 1, PCG_BAD_PRECOND = 2 };

// The PCG's <r, z> fused into the last kernel of the preconditioner apply
// (k_prolong_sum's combine epilogue) when that kernel writes z.
struct RzFuse {
  PcgState* st = nullptr;
  const double* r = nullptr;
  const double* z = nullptr;
  double* part = nullptr;
  unsigned* count = nullptr;
};

struct Ctx;

// ---- launchers (kernels.cu) -------------------------------------------------
namespace k {
void spmv(Ctx& c, const double* x, double* y, int mode, const double* add, const double* sub, const int* gate);
void gather(Ctx& c, const double* x, const double* scale, double* xs, const int* gate);
void prolong(Ctx& c, const double* w, double* y, const int* gate);
void h1(Ctx& c, const double* x, double* y, const int* gate);         // one-level NN
void nn_gemvT(Ctx& c, const double* x, const int* gate);               // uh = mask(1/lam) V^T D R x
void nn_gemv(Ctx& c, const int* gate);                                 // part = V uh (column chunks)
void nn_prolong(Ctx& c, double* y, const int* gate);                   // y = sum_s R^T D sum_kc part
void nn_fused(Ctx& c, const double* x, const int* gate);               // single pass over V^s into part
void aminus(Ctx& c, const double* x, double* y, const int* gate);     // y = A- x
// mode 1: y = A+ x;  mode 2: y = sub - A+ x  (A- prolongation fused into the SpMV)
// neg_ready: neg_c already holds the A- dots of x (from coarse_q_neg)
void aplus(Ctx& c, const double* x, double* y, int mode, const double* sub, const int* gate, bool neg_ready = false);
bool coarse_q_neg(Ctx& c, const double* x, double* y, const int* gate);  // Q x and the A- dots of Q x
void build_coarse_neg(Ctx& c);  // M2 = M1 K+ (A- dots of the retained coarse columns), after K0 is set
void build_az(Ctx& c);          // A Z on ring-extended supports + the combined dots plan, after build_coarse_neg
// y = ((hp - Z K+ Z^T A+ hp) + corr) [+ extra] without forming A+ hp (needs c.az_on)
void coarse_q_combine_az(Ctx& c, const double* hp, double* y, const double* corr, const double* extra,
                         cudaEvent_t wait_before_combine, const int* gate);
void coarse_q(Ctx& c, const double* x, double* y, const int* gate);   // y = Z K0+ Z^T x
// y = ((a - Z K0+ Z^T x) + d) [+ e] in one epilogue (a == nullptr: y = Z K0+ Z^T x);
// the stream waits on `wait_before_combine` (if set) before the combining kernel
void coarse_q_combine(Ctx& c, const double* x, double* y, const double* a, const double* d, const double* e,
                      cudaEvent_t wait_before_combine, const int* gate);
void second_q(Ctx& c, const double* x, double* y, const int* gate);   // y = W KW+ W^T x
void second_q_coef(Ctx& c, const double* x, const int* gate);         // c.cw second half = KW+ W^T x
void second_q_apply(Ctx& c, double* y, const int* gate);              // y = W (c.cw second half)
void inex_q(Ctx& c, const double* x, double* y, const int* gate);     // y = W core^-1 W^T x
void axpby(Ctx& c, int n, const double* a, const double* b, const double* d, double* y, int mode, const int* gate);
void rr_solve(Ctx& c, const CoarseFactor& f, const double* b, double* x, const int* gate);
// L^-1 of the r x r lower factor l, K^+ = L^-T L^-1 and the retained positions
void coarse_inverse(Ctx& c, const double* l, CoarseFactor& f);
void zT(Ctx& c, const double* x, double* out, const int* gate);  // out = Z^T x (n0)
void wT(Ctx& c, const double* x, double* out, const int* gate);  // out = W^T x (n_minus)
void w_apply_public(Ctx& c, const double* coef, double* y, const int* gate);  // y = W coef
void scatter_col(Ctx& c, int s, const double* col, double* z);  // z[Omega^s] = col (z pre-zeroed)
void owner_tables(Ctx& c);  // ent_neg, ent_z and the plans' own_nkc (after the factors and plans)
}  // namespace k

// ---- the context --------------------------------------------------------------
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // concurrent branch (second coarse correction of H3,ad)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_mid = nullptr;  // main stream past the local solve (split W branch)
  int w_split = -1;              // AD W branch split around the local solve: -1 automatic, 0 off, 1 on
  std::string err;
  int err_index = -1;
  long long launches = 0;
  int sm_count = 148;

  // problem
  int n = 0, nnz = 0, N = 0;
  long long P = 0;  // sum n_s
  std::vector<int> h_rp, h_ci;
  std::vector<double> h_va;
  std::vector<long long> h_poff;
  std::vector<int> h_pidx, h_mult, h_ns, h_ld;
  DArr<int> rp, ci;
  DArr<double> va;
  DArr<int> pidx, psub, own_off, own_pos, mult;
  DArr<long long> poff;
  DArr<double> ds;
  DArr<int> emult;  // multiplicity of each stored entry (splitting.cpp:20-33)

  // local factors
  bool have_factors = false;
  std::vector<int> h_m, h_nzero, h_ks;
  std::vector<long long> h_voff, h_yoff;
  std::vector<double> h_lam, h_eps, h_plam;
  std::vector<double> h_plam2;  // AS: pencil_as2 spectrum (h_plam holds pencil_as1)
  std::vector<int> h_ks_as1;    // AS: columns per subdomain taken from pencil_as1
  DArr<int> ns, ld, msz;
  DArr<long long> voff;
  DArr<double> V, lam;
  DArr<double> rlam;  // 1 / lambda for lambda > 0 (single-pass local solve), else 0
  int rows_per_gemv = 512;
  int gemv_cols = 1024;  // column chunk of the split GEMV
  int one_level = 2;     // OneLevelKind of the configuration: 0 AS, 1 AS_PLUS, 2 NN
  bool use_fused = true; // single-pass NN local solve (option nn_two_pass=1 disables)
  // single-pass tuning (env AWG_FUSED_CPB / AWG_FUSED_NBUF / AWG_FUSED_CHUNKS; 0 = automatic)
  bool use_priority = true;  // main stream high priority, W branch low
  bool use_pdl = true;       // programmatic dependent launch on the solve path
  // GPU-side assembly (assemble.cu): -1 external matrix, 0 cell grid, 1 Q1 mesh
  int asm_kind = -1, asm_dims = 0, asm_shape[3] = {0, 0, 0};
  std::vector<double> h_rhs_asm;  // assembled right-hand side (elasticity body force)
  DArr<unsigned long long> fused_timer;  // k_nn_fused launch timer (see kernels.cu)
  int fused_reserve = 0;
  int fused_min_cols = 128, fused_tail_pct = 0;  // single-pass task sizes (columns), guided tail share  // SMs the single-pass kernel leaves free (for the concurrent W branch)
  int fused_cpb = 0, fused_nbuf = 0, fused_chunks_per_sm = 8;  // 0: automatic
  int pdl_early = 0;        // coarse-chain kernels release their dependents at entry (option pdl_early=1; measured neutral)
  int rows_group = 0;       // lanes per dof of the block-sparse prolongations (0: automatic)
  bool pdl_local = true;     // early trigger into the single-pass local solve + its pre-wait prologue (option pdl_local=0 off)
  int trigger_next = 0;     // set around the launch that precedes the local solve
  bool pcg_adaptive = true;  // host batch sizes from the convergence rate (option pcg_adaptive=0: doubling only)
  bool fused_static = true;  // equal byte shares per CTA instead of the atomic queue (option fused_static=0 off)
  bool fused_prefetch = true;  // next task's first steps issued during the current one (option fused_prefetch=0 off)
  bool fused_hold = true;  // column values kept in registers across the step's reduction (option fused_hold=0 off)
  BsPlan bs_neg, bs_z;   // A- dots (V^s columns k < n_nonpos), Z^T x (Y_s blocks)
  DArr<OwnEnt> ent_neg, ent_z;  // owner entries into V^s (A- modes) and Y_s (Z columns)
  DArr<double> m2t;  // (K+ M1^T): r0 x n_neg column-major; M1(q, jj) = A- dot q of coarse column retained[jj]
  // A Z on ring-extended supports (k::build_az): the post-solve half of the hybrid H2
  // needs Z^T A+ hp = (A Z)^T hp + M1^T (V-^T R hp); both dot families run as ONE
  // block-sparse GEMV^T over 2N "subdomains" (s < N: V-^s on Omega^s, s >= N: (A Z)_s on
  // E_s = Omega^s + one graph ring), and the M1 term rides in the coarse solve (m2)
  bool az_on = false;
  BsPlan bs_az;
  DArr<int> az_ns, az_ld, az_pidx, az_coff, az_ccol;
  DArr<long long> az_poff, az_moff;  // az_moff: element offsets from V.p (the AZ blocks live in AZ)
  DArr<double> AZ, az_out;           // az_out: [unweighted A- dots (nneg); (A Z)^T x (n0)]
  DArr<double> m2;                   // M1 K+ (n_neg x r0 column-major): m2t transposed
  LocalPlan plan_nn;     // V^s with the eigenvalue mask (NN)
  LocalPlan plan_as;     // U^s = L^-T, triangular (AS / AS+)
  DArr<double> U;        // AS / AS+ local factors, same layout as V
  DArr<double> wpart_nn; // kcmax x P partial sums
  DArr<int> fused_queue; // work counter of the persistent single-pass kernel

  // A- modes
  int nneg = 0;
  DArr<int> neg_s, neg_k, negoff;
  DArr<double> neg_w, neg_c;

  // coarse space
  int n0 = 0;
  DArr<long long> yoff;
  DArr<double> Y;
  DArr<int> zcol_s, zcol_loc, koff;
  CoarseFactor k0;

  // second coarse space
  int nm = 0;
  int ldw = 0;
  DArr<double> W, neg_weights, vminus;
  CoarseFactor kw;
  std::vector<int> h_w_inner;
  std::vector<double> h_neg_weights;
  // INEX core: LU of Lambda^-1 - V-^T W (dense.cpp:368-393)
  DArr<double> core_lu;
  DArr<int> core_perm;
  int lu_semantics = 0;

  // configuration
  awg_config cfg{};
  double t_setup_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int w_batches = 0;

  // work buffers
  DArr<double> xs, uh, wl;                          // P each
  DArr<double> t0, t1, t2, t3, t4, t5, t6, t7, t8;  // n each
  DArr<double> cz;  // coarse (K0) scratch
  DArr<double> cw;  // second coarse (KW) scratch (may run concurrently)
  DArr<double> wpart;                               // split-K partials of W^T x
  DArr<double> wpart2;                              // column-chunk partials of W c
  DArr<double> red;                                 // reduction partials
  DArr<unsigned> red_count;

  // pcg
  RzFuse rz_fuse;         // armed by run_pcg around the preconditioner apply it captures
  bool rz_fused = false;   // set when an apply consumed rz_fuse
  DArr<double> pp2;        // second search-direction buffer (p formed inside the SpMV)
  DArr<PcgState> pcg;
  DArr<int> pcg_flag;
  std::map<int, cudaGraphExec_t> graphs;  // one PCG iteration per operator pair
  std::map<int, long long> graph_launches;
  void invalidate_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
    graph_launches.clear();
  }
  ~Ctx() { invalidate_graphs(); }
  DArr<double> px, pr, pz, pp, pq, pb, pt;
  DArr<double> hist_res, hist_diag, hist_off;
  int hist_cap = 0;
  std::vector<double> h_hist_res, h_hist_diag, h_hist_off;

  // experiment switches set through awg_set_option (tests / profiles only;
  // the product defaults are the literals at each use)
  std::map<std::string, long long> opts;
  long long opt(const char* name, long long dflt) const {
    auto it = opts.find(name);
    return it == opts.end() ? dflt : it->second;
  }
  void alloc_work();  // also invalidates cached graphs
  void fail(int code, const std::string& m, int idx = -1) { throw AwgError(code, m, idx); }
};

// Programmatic dependent launch: every solve-path kernel is launched with
// programmatic stream serialization, so it is scheduled while its predecessor
// drains and waits in pdl_wait() (griddepcontrol.wait, first statement of
// every such kernel, before it reads or writes anything the predecessor
// touches).  Captured into the per-iteration CUDA graph as programmatic edges.
// No kernel triggers its dependents early (griddepcontrol.launch_dependents):
// measured on c2, waiting successor CTAs then crowd the running grid
// (1,797 vs 1,875 applies/s); the implicit trigger at grid exit hides the
// launch gap alone (+2.4% over no PDL).  One exception: the A+ SpMV right
// before the single-pass local solve triggers early, and the local solve
// issues its first (constant) V^s copies before its griddepcontrol.wait
// (option pdl_local; H3 apply 0.475 -> 0.467 ms at c2, profiles/r01f/knobs_pdl_local_c2.json).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// CSR row product  sum_k va[k] x[ci[k]]  in ascending k with separately
// rounded multiply and add — bit-identical to the reference build of
// sparse.cpp:49-56 (GCC emits vmulsd + vaddsd there).  The row's loads are
// issued in groups of 8 ahead of the dependent add chain (the plain loop
// stalls on every add before it can issue the next load).  P(j) supplies the
// vector entry (x[j], or p formed on the fly).
template <class P>
__device__ __forceinline__ double csr_row(const int* __restrict__ ci, const double* __restrict__ va, int k0, int k1,
                                          P xv) {
  double acc = 0.0;
  for (int k = k0; k < k1; k += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (k + u < k1) ? __dmul_rn(va[k + u], xv(ci[k + u])) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k + u < k1) acc = __dadd_rn(acc, t[u]);
  }
  return acc;
}

template <typename... P, typename... A>
inline void launch(Ctx& c, void (*kern)(P...), dim3 grid, dim3 block, size_t smem, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c.use_pdl ? 1 : 0;
  AWG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

// ---- operators (ops.cu) -------------------------------------------------------
void op_apply(Ctx& c, int op, const double* x, double* y, const int* gate);
void run_pcg(Ctx& c, const double* b_dev, double rtol, int maxit, awg_solve_report* rep,
             int op_a = AWG_OP_A, int op_h = AWG_OP_H3);
void finalize_factors(Ctx& c);  // task lists, A- modes, inverses, work buffers
// GPU-side problem assembly (assemble.cu)
void assemble_fd(Ctx& c, int dims, const int* shape, const double* coef, std::vector<int>& rp, std::vector<int>& ci,
                 std::vector<double>& va);
void assemble_elasticity(Ctx& c, int nodes_x, int nodes_y, int layer, int nmat, const double* young,
                         const double* poisson, const double* load, std::vector<int>& rp, std::vector<int>& ci,
                         std::vector<double>& va, std::vector<double>& b);
void partition_closure(Ctx& c, const std::vector<int>& owner, int nsub, int rings, std::vector<long long>& off,
                       std::vector<int>& idx);
// dgemm.cu: grouped DMMA GEMM vs cuBLAS on seeded operands (awg_bench_dgemm)
void bench_grouped_dgemm(Ctx& c, int m, int n, int k, int count, bool transpose_a, int reps, double* out);
void build_core(Ctx& c);        // INEX core LU
void run_setup(Ctx& c, const awg_config& cfg);  // setup.cu
// batched dense symmetric eigensolver (eig.cu): A (n x n, ld, lower; destroyed),
// w (n eigenvalues, ascending), Z (n x nvec eigenvectors of the nvec smallest, ldz)
struct SyevJob {
  double* A;
  int n, ld;
  double* w;
  double* Z;
  int ldz, nvec;
};
// pick(q, w): after the eigenvalues of problem q are known (host copy, ascending),
// the number of eigenvectors it needs (<= its nvec); null: nvec as given
void eig_batched(Ctx& c, const std::vector<SyevJob>& jobs,
                 const std::function<int(int, const double*)>& pick);  // on c.stream
void eig_check(Ctx& c, int n, int count, int kind, unsigned long long seed, double* out);  // awg_bench_eig
// batched Cholesky + block triangular solves (chol.cu), all on c.stream
struct CholJob {
  double* A;  // n x n, ld (lower; the factor L on return)
  int n, ld;
};
struct CholBatch {
  std::vector<CholJob> jobs;
  int nmax = 0, npan = 0;
  DArr<double> di, dit;  // inverted 64 x 64 diagonal blocks and their transposes
  DArr<int> info;
  void factor(Ctx& c, const std::vector<CholJob>& jobs);  // AWG_E_NOT_SPD with the pivot index
  void solve_lower(Ctx& c, const std::vector<double*>& B, const std::vector<int>& ldb, const std::vector<int>& nrhs);
  void solve_upper_t(Ctx& c, const std::vector<double*>& B, const std::vector<int>& ldb, const std::vector<int>& nrhs);
  void reduce_pencil(Ctx& c, const std::vector<double*>& MA, const std::vector<double*>& T);  // MA <- sym(L^-1 MA L^-T)
  void inverse_transpose(Ctx& c, const std::vector<double*>& U, const std::vector<double*>& T);  // U <- L^-T
};
void pivoted_factor_of(Ctx& c, int n, const double* G_host, int exact, CoarseFactor& f);  // setup.cu
void build_local_cholesky(Ctx& c);              // setup.cu: AS / AS+ factors U^s = L^-T
// wbuild.cu: batched inner PCGs for W (modes = (s, k) list, ascending)
void build_w_batched(Ctx& c, struct cublasContext* h, const std::vector<std::pair<int, int>>& modes, int maxit,
                     double rtol, std::vector<int>& iters, int max_block);

}  // namespace awgb

struct awg_ctx {
  awgb::Ctx c;
};
