/*
 * khb200 -- C-ABI of the B200-native Fast-Diagonalization space-time solver.
 *
 * Every entry point replaces one piece of the reference's FD hot path
 * (reference package `kronheat`, pkg/src/kronheat/):
 *
 *   kh_analyze ................ sparse_direct.analyze          sparse_direct.py:112-152
 *                               (called once per solve from solvers.py:379 _union_symbolic)
 *   kh_plan_create ............ per-shift matrix build K = Mc + lam*Ac   solvers.py:378, :384
 *   kh_plan_factor ............ sparse_direct.factorize (SuperLU zgstrf) sparse_direct.py:155-188,
 *                               batched over the shifts of the loop at solvers.py:383-393
 *   kh_plan_pivot_check ....... pivot guard |U_ii| >= 1e-13 max|a|      sparse_direct.py:182-187
 *   kh_plan_solve ............. sparse_direct.solve (SuperLU zgstrs)    sparse_direct.py:191-209
 *   kh_plan_factor_solve ...... factorize + solve of one shift batch with the forward sweep fused
 *                               into the factorization (the first FD application, solvers.py:383-393)
 *   kh_dgemm .................. modal transforms (zgemm)                solvers.py:368-372, :397-400
 *   kh_plan_residual .......... residual / kron_apply_right             solvers.py:428-440, dense.py:264-286
 *   kh_plan_residual_dd, kh_dgemm_dd, kh_csr_pair_residual_dd
 *                               the same residual in compensated arithmetic (refinement at c4)
 *   kh_sumsq .................. norms of _discard_imaginary              solvers.py:406-413
 *   kh_dgemm_rowscatter ....... multi-GPU back transform fused with the scatter of its
 *   kh_sum_parts                reduce-scatter (solvers.py:397-400 per rank)
 *   kh_ipc_handle/open/close .. peer-memory mapping of the receive slots (one process per GPU)
 *   kh_ht_assemble ............ temporal H_T matrices A_t, M_t, C_t     temporal.py:98-151, :300-329
 *   kh_ht_workspace_bytes       (P1 hats as the reference; P2 Lagrange basis for config c5)
 *
 * Conventions: plain pointers and 64-bit sizes, column-major matrices,
 * caller-owned buffers. Pointers documented "device" must be CUDA device
 * memory of the plan's device; "host" pointers are ordinary host memory.
 * `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 * every device call is stream-ordered and asynchronous unless noted.
 * Every call returns a kh status (0 = OK); kh_last_error() gives the detail
 * of the last failure on the calling thread.
 *
 * Status -> reference exception (pkg/src/kronheat/errors.py):
 *   KH_ERR_DIMENSION  -> DimensionMismatch
 *   KH_ERR_SINGULAR   -> SingularMatrix
 *   KH_ERR_INVALID    -> UsageError
 *   KH_ERR_CUDA, KH_ERR_NOMEM -> DeviceError (new class derived from KronheatError)
 * Threading: distinct plans may be used from distinct threads; one plan is
 * not re-entrant. One process per GPU for multi-GPU runs.
 */
#ifndef KHB200_H
#define KHB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KH_OK 0
#define KH_ERR_DIMENSION 1
#define KH_ERR_SINGULAR 2
#define KH_ERR_INVALID 3
#define KH_ERR_CUDA 4
#define KH_ERR_NOMEM 5

typedef struct kh_symbolic kh_symbolic;
typedef struct kh_plan kh_plan;

typedef struct {
  int64_t n;             /* matrix dimension */
  int64_t nnz;           /* entries of the analyzed (symmetrized) CSR pattern */
  int64_t n_fronts;      /* supernodal fronts of the dissection tree */
  int64_t max_front;     /* largest front order m = p + q */
  int64_t max_pivots;    /* largest pivot block p */
  int64_t depth;         /* tree depth (levels = depth + 1) */
  int64_t factor_nnz;    /* entries of L incl. diagonal (complex) */
  int64_t panel_entries; /* complex entries of retained factor storage per shift */
  int64_t upd_entries;   /* complex entries of update buffers per in-flight shift */
  int64_t leaf_size;
  double flops;          /* real flops per shift of the complex LDL^T (8 per complex FMA) */
} kh_symbolic_stats;

int kh_version(void);
/* Number of kernels the library has launched so far in this process. */
int64_t kh_launch_count(void);
const char* kh_status_string(int status);
const char* kh_last_error(void);

/* Symbolic analysis (host). `indptr`/`indices`: host CSR of a square,
 * structurally symmetric pattern (duplicates and self loops allowed).
 * `leaf_size` <= 0 selects the default. */
int kh_analyze(int64_t n, const int64_t* indptr, const int64_t* indices, int32_t leaf_size, kh_symbolic** out);
/* kh_analyze of the union of two patterns (the FD path analyzes M_x + A_x:
 * solvers.py:216-223, _union_symbolic) without forming the sum on the host
 * first; rows are merged in parallel. */
int kh_analyze_union(int64_t n, const int64_t* indptr1, const int64_t* indices1, const int64_t* indptr2,
                     const int64_t* indices2, int32_t leaf_size, kh_symbolic** out);
int kh_symbolic_stats_get(const kh_symbolic* s, kh_symbolic_stats* out);
/* perm[k] = original index eliminated k-th (host array of n). */
int kh_symbolic_perm(const kh_symbolic* s, int64_t* perm);
/* Per-front arrays (host, n_fronts each; any may be NULL). */
int kh_symbolic_fronts(const kh_symbolic* s, int64_t* first, int32_t* npiv, int32_t* nupd, int32_t* parent,
                       int32_t* depth);
/* The analyzed CSR (host, n + 1 and stats.nnz entries): the input pattern
 * symmetrized (A | A^T) with the full diagonal, rows sorted, no duplicates.
 * Value arrays for kh_plan_create are aligned to it (kh_align_values). */
int kh_symbolic_pattern(const kh_symbolic* s, int64_t* indptr, int64_t* indices);
/* Concatenated update-row lists (permuted positions), sum of nupd entries. */
int kh_symbolic_rows(const kh_symbolic* s, int64_t* rows);
void kh_symbolic_free(kh_symbolic* s);
/* Host: scatter the values of a canonical n x n CSR (sorted, no duplicates)
 * onto a canonical pattern (pat_*) that contains it (out: one double per
 * pattern entry, zero where absent). Returns KH_ERR_DIMENSION if the matrix
 * has an entry outside the pattern. This is the per-shift matrix build
 * K = Mc + lam*Ac of solvers.py:384 moved ahead of the loop: M and A are
 * aligned once and the shift is applied on the device. */
int kh_align_values(int64_t n, const int64_t* pat_indptr, const int64_t* pat_indices, const int64_t* indptr,
                    const int64_t* indices, const double* vals, double* out);

/* Numeric plan on `device`: uploads the analysis and the value arrays of the
 * two matrices M and A (host, aligned with the analyzed CSR `indptr/indices`,
 * which must be the pattern given to kh_analyze). The plan factors shifted
 * matrices M + lambda A. It allocates factor storage for `factor_slots`
 * shifts and work space for up to `max_batch` shifts per call. All device
 * memory of the plan is carved from one workspace: `workspace` (device, at
 * least kh_plan_bytes() bytes, caller-owned, e.g. from a caching allocator)
 * or, if NULL, one cudaMalloc owned by the plan. */
int kh_plan_create(const kh_symbolic* s, int device, const int64_t* indptr, const int64_t* indices,
                   const double* m_vals, const double* a_vals, int64_t max_batch, int64_t factor_slots,
                   void* workspace, int64_t workspace_bytes, kh_plan** out);
/* Exact workspace size of a plan (no allocation). */
int kh_plan_bytes(const kh_symbolic* s, int64_t max_batch, int64_t factor_slots, int64_t* bytes);
int kh_plan_set_values(kh_plan* plan, const double* m_vals, const double* a_vals);
/* Factor M + lambda_s A for s < nshift into slots slot0.. ; `lambda_ri` is a
 * host array of nshift (re, im) pairs. nshift <= max_batch. */
int kh_plan_factor(kh_plan* plan, int64_t slot0, int64_t nshift, const double* lambda_ri, void* stream);
/* Synchronizes `stream`; returns KH_ERR_SINGULAR if some shift has a pivot
 * |d| < rel_threshold * max|a_ij| (or a non-finite pivot). `first_bad`
 * (may be NULL) receives the first offending shift index or -1;
 * `worst_ratio` (may be NULL) the smallest |d|/max|a|. */
int kh_plan_pivot_check(kh_plan* plan, int64_t slot0, int64_t nshift, double rel_threshold, void* stream,
                        int64_t* first_bad, double* worst_ratio);
/* Solve (M + lambda_s A) x_s = b_s with the factors in slots slot0.. .
 * Device arrays; column s of b/x at b_re + s*ldb. b_im/x_im may be NULL
 * (real rhs / discard imaginary part). nshift <= max_batch. */
int kh_plan_solve(kh_plan* plan, int64_t slot0, int64_t nshift, const double* b_re, const double* b_im,
                  int64_t ldb, double* x_re, double* x_im, int64_t ldx, void* stream);
/* kh_plan_factor + kh_plan_solve in one pass: the forward sweep runs inside
 * the shared-memory factorization kernels (each front's rhs segment sits
 * beside it in shared memory and is swept after its LDL^T) and beside the
 * large fronts' Schur kernels, so the factors are read back only once, by the
 * backward sweep. Same arguments and results as the two calls (rounding
 * aside). */
int kh_plan_factor_solve(kh_plan* plan, int64_t slot0, int64_t nshift, const double* lambda_ri, const double* b_re,
                         const double* b_im, int64_t ldb, double* x_re, double* x_im, int64_t ldx, void* stream);
/* The two halves of kh_plan_factor_solve: factorization + forward sweep
 * (the result stays in the plan's solve work space), then the backward sweep
 * of the same batch; nothing else may use the plan in between. */
int kh_plan_factor_fwd(kh_plan* plan, int64_t slot0, int64_t nshift, const double* lambda_ri, const double* b_re,
                       const double* b_im, int64_t ldb, void* stream);
int kh_plan_solve_bwd(kh_plan* plan, int64_t slot0, int64_t nshift, double* x_re, double* x_im, int64_t ldx,
                      void* stream);
/* Per-level timing of the factorization (measurement aid for the per-level
 * roofline): with timing on, the next factorizations record CUDA events at
 * every level boundary on the caller's stream; kh_plan_level_times waits for
 * the last one and returns the milliseconds of each level of the most recent
 * factorization, indexed by tree depth (0 = root), n_levels = depth + 1. */
/* Device address of the retained factor storage (slot-major, panel_total
 * complex entries per slot; front panels column-major m x p in front order)
 * for diagnostics and tests. */
int kh_plan_factor_storage(const kh_plan* plan, void** panels, int64_t* panel_total);
int kh_plan_set_level_timing(kh_plan* plan, int32_t on);
int kh_plan_level_times(kh_plan* plan, float* ms, int32_t n_levels);
/* R = F - (M Y[:, :nt] + A Y[:, nt:2nt]) on the plan's CSR (device arrays);
 * R may be NULL. norms2 (device, 2 doubles) receives ||R||_F^2, ||F||_F^2. */
int kh_plan_residual(kh_plan* plan, int64_t nt, const double* Y, int64_t ldy, const double* F, int64_t ldf,
                     double* R, int64_t ldr, double* norms2, void* stream);
/* norms2 (device, 2 doubles) = (|| |F| + |M_x| |Y1| + |A_x| |Y2| ||^2, ||F||^2): the
 * magnitude of the terms the residual cancels, whose eps multiple is the
 * rounding floor of evaluating kh_plan_residual in fp64 (decides when
 * refinement needs the compensated residual). Same Y / F layout. */
int kh_plan_residual_scale(kh_plan* plan, int64_t nt, const double* Y, int64_t ldy, const double* F, int64_t ldf,
                           double* norms2, void* stream);
/* Compensated variant of kh_plan_residual (refinement at fine meshes, where the
 * fp64 evaluation of f - K u floors the residual): Y2 = U M_t^T given as the
 * unevaluated sum Y2hi + Y2lo (kh_dgemm_dd), Y1 = U A_t^T in fp64 (ld ldy1);
 * R = F - (M_x Y1 + A_x Y2) accumulated with error-free products and sums,
 * rounded once. Replaces the same reference lines as kh_plan_residual. */
int kh_plan_residual_dd(kh_plan* plan, int64_t nt, const double* Y1, int64_t ldy1, const double* Y2hi,
                        const double* Y2lo, int64_t ldy2, const double* F, int64_t ldf, double* R, int64_t ldr,
                        double* norms2, void* stream);
void kh_plan_free(kh_plan* plan);

/* C = alpha A B + beta C, fp64, column-major, device arrays (DMMA GEMM). */
int kh_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
             int64_t ldb, double beta, double* C, int64_t ldc, void* stream);
/* Plan-free residual on a device CSR (indptr n+1, indices/m_vals/a_vals nnz):
 * same contract as kh_plan_residual. */
int kh_csr_pair_residual(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                         const double* m_vals, const double* a_vals, const double* Y, int64_t ldy,
                         const double* F, int64_t ldf, double* R, int64_t ldr, double* norms2, void* stream);
/* C_hi + C_lo = A B (m x n, K = k, column-major device arrays) with compensated
 * products and sums (Dot2): the temporal product U M_t^T of the compensated
 * residual. */
int kh_dgemm_dd(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                double* C_hi, double* C_lo, int64_t ldc, void* stream);
/* Plan-free kh_plan_residual_dd on a device CSR. */
int kh_csr_pair_residual_dd(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                            const double* m_vals, const double* a_vals, const double* Y1, int64_t ldy1,
                            const double* Y2hi, const double* Y2lo, int64_t ldy2, const double* F, int64_t ldf,
                            double* R, int64_t ldr, double* norms2, void* stream);
/* y += alpha x over n device doubles (refinement update of a row shard). */
int kh_daxpy(int64_t n, double alpha, const double* x, double* y, void* stream);
/* out (device, 1 double) = sum_i x_i^2 over n device doubles. */
int kh_sumsq(const double* x, int64_t n, double* out, void* stream);
/* Multi-GPU back transform (one process per GPU). C = A B (m x n, K = k,
 * device arrays, column-major), with row r written to part c = r / rows_per_part
 * at dst[c] + (r - c rows_per_part) + j ld_dst, where `dst` is a DEVICE array of
 * `parts` pointers, typically peer-mapped receive slots of the other ranks
 * (kh_ipc_open): each finished tile goes straight over NVLink to the rank that
 * owns its rows, fusing the GEMM with the scatter of a reduce-scatter. */
int kh_dgemm_rowscatter(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* const* dst, int32_t parts, int64_t rows_per_part, int64_t ld_dst, void* stream);
/* out[e] = sum_{c < parts} slots[c part_elems + e] in slot order (deterministic
 * reduction of the received partial sums; device arrays). */
int kh_sum_parts(int32_t parts, const double* slots, int64_t part_elems, double* out, void* stream);
/* CUDA IPC: `handle` is 64 opaque bytes (host) naming the allocation that
 * contains dev_ptr; `offset` receives dev_ptr's byte offset inside it.
 * kh_ipc_open maps another process's allocation into this process (peer
 * access enabled) and returns its base: add the sender's offset. */
int kh_ipc_handle(const void* dev_ptr, void* handle, int64_t* offset);
int kh_ipc_open(const void* handle, void** dev_ptr);
int kh_ipc_close(void* dev_ptr);
/* Temporal H_T matrices (reference temporal.py:300-329) of the P1 (degree 1)
 * or P2 (degree 2) basis on the partition `nodes` (device, n_cells + 1
 * doubles, nodes[0] = 0, T = nodes[n_cells]), truncated at j_max. Outputs
 * (device, column-major, overwritten): A and M (nr x nr), C (nr x n_cells),
 * nr = degree * n_cells; A is the full product (the caller mirrors its lower
 * triangle like the reference's dsyrk). `workspace`: device, at least
 * kh_ht_workspace_bytes(). */
int kh_ht_workspace_bytes(int32_t degree, int64_t n_cells, int64_t* bytes);
int kh_ht_assemble(int32_t degree, int64_t n_cells, const double* nodes, int64_t j_max, double* A, double* M,
                   double* C, void* workspace, int64_t workspace_bytes, void* stream);
int kh_set_device(int device);
int kh_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KHB200_H */
