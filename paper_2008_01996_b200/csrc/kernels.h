// Internal launcher interfaces shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

struct KhDevFront {
  int64_t first;
  int32_t p, q;
  int64_t panel_off, upd_off, rupd_off;
  int64_t orig_begin, orig_end;
  int64_t rows_begin;  // urows / relind of this front
  int64_t cmap_begin;  // pull map over the parent's rows (see symbolic.h)
  int32_t child_begin, child_end;
  int32_t depth, pad;
};

// Update (Schur complement) blocks are stored packed: the lower triangle of
// the q x q block column by column, entry (i, j), i >= j, at kh_upk(q, i, j)
// (one contiguous q(q+1)/2 array per front: a single bulk copy moves it).
__host__ __device__ inline int64_t kh_upk(int q, int i, int j) { return i + (int64_t)j * (2 * q - j - 1) / 2; }
// 32-bit form for q < 46341 (every front here; kh_analyze caps local offsets at 2^31)
__host__ __device__ inline int kh_upk32(int q, int i, int j) { return i + j * (2 * q - j - 1) / 2; }

// Packed block-column layout of a fused front (m <= 128) in shared memory:
// the 8-column block b stores rows 8b..m-1 with leading dimension
// roundup8(m - 8b) + 2 (2 mod 8 in 16-byte units: conflict-free DMMA
// fragment loads). Entry (r, c), r >= c, sits at kh_packed_col_base(m, c) + r.
__host__ __device__ constexpr int kh_packed_ld(int m, int b) { return ((m - 8 * b + 7) / 8) * 8 + 2; }
// (closed forms: block b has leading dimension 8 (ceil(m/8) - b) + 2)
__host__ __device__ constexpr int kh_packed_elems(int m) {
  const int M8 = (m + 7) / 8;
  return 32 * M8 * (M8 + 1) + 16 * M8;
}
__host__ __device__ constexpr int kh_packed_col_base(int m, int c) {
  const int M8 = (m + 7) / 8, b = c >> 3;
  return 64 * b * M8 - 32 * b * (b - 1) + 16 * b + (c & 7) * kh_packed_ld(m, b) - 8 * b;
}

// A child as its parent's assembly needs it (parallel to child_list).
struct KhKid {
  int64_t upd_off, rows_begin, rupd_off, cmap_begin;
  int32_t q, pad;
};

struct KhTree {  // device pointers shared by every level kernel
  const KhDevFront* fronts;
  // fronts in level-launch order (level_fronts), with the front index in
  // `pad`, and the children's records: one dependent load each instead of
  // level_fronts -> fronts and child_list -> fronts
  const KhDevFront* lf_fronts;
  const int32_t* lf_base;
  const KhKid* kids;
  const int32_t* child_list;
  const int32_t* relind;
  const int32_t* cmap;
  const int64_t* urows;
  const int64_t* orig_src;
  const int32_t* orig_dst;  // panel offset (r + c*m); packed offset for fused fronts
  const double* mv;  // M values aligned with the analyzed CSR
  const double* av;  // A values aligned with the analyzed CSR
  const double* om;  // M values in front-original order: om[e] = mv[orig_src[e]]
  const double* oa;  // A values in front-original order
  int32_t nf;
  int64_t n;
  int64_t panel_total;
};

cudaError_t kh_launch_dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                            cudaStream_t stream);

// C = A B with row r written to dst[r / rp] (row r % rp, ld ldd): fused GEMM +
// scatter into peer receive slots; and the ordered sum of g slots.
cudaError_t kh_launch_dgemm_batched(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                                    int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta, double* C,
                                    int64_t ldc, int64_t sC, int32_t batch, cudaStream_t stream);
cudaError_t kh_launch_dgemm_rowscatter(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                                       const double* B, int64_t ldb, double* const* dst, int64_t rp, int64_t ldd,
                                       cudaStream_t stream);
cudaError_t kh_launch_sum_parts(int32_t g, const double* parts, int64_t len, double* out, cudaStream_t stream);

// mid_panel > 0: every front of the launch has a lower panel of at most
// mid_panel entries and m <= mid_m, small enough for the bulk-copy staged
// kernels on a wide level (0: the level kernels).
cudaError_t kh_launch_fwd_level(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                int32_t max_m, const double2* panels, double2* y, double2* ru_cur,
                                int64_t ru_stride_cur, const double2* ru_child, int64_t ru_stride_child,
                                cudaStream_t stream, int32_t mid_panel = 0, int32_t mid_m = 0, int32_t lvl_m = 0);
// Level-synchronous kernels for the large fronts (see frontal.cu). Tasks are
// (front, index) int32 pairs; schur tasks are (front, tile row, tile col).
#ifndef KH_ASM_CHUNK_DEF
#define KH_ASM_CHUNK_DEF 512
#endif
constexpr int KH_ASM_CHUNK = KH_ASM_CHUNK_DEF;
cudaError_t kh_launch_big_assemble(const KhTree& T, const int32_t* tasks, int32_t ntasks, int32_t batch,
                                   const double2* lam, double2* panels, const double2* upd_child,
                                   int64_t upd_stride_child, cudaStream_t stream);
cudaError_t kh_launch_schur(const KhTree& T, const int32_t* tasks, int32_t ntasks, int32_t batch,
                            const double2* panels, double2* upd_cur, int64_t upd_stride_cur, const double2* upd_child,
                            int64_t upd_stride_child, cudaStream_t stream);
// Warp-per-front solves for fronts with m <= 64.
cudaError_t kh_launch_fwd_small(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                const double2* panels, double2* y, double2* ru_cur, int64_t ru_stride_cur,
                                const double2* ru_child, int64_t ru_stride_child, int32_t max_panel,
                                cudaStream_t stream, int32_t max_m = 64);
// max_panel: largest lower-panel entry count p m - p (p - 1) / 2 among the fronts
// (sizes the shared-memory staging of the bulk-copy variant)
cudaError_t kh_launch_bwd_small(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                const double2* panels, double2* y, int32_t max_panel, cudaStream_t stream,
                                int32_t max_m = 64);
cudaError_t kh_launch_bwd_level(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                int32_t max_p, int32_t max_m, const double2* panels, double2* y,
                                cudaStream_t stream, int32_t mid_panel = 0, int32_t mid_m = 0, int32_t lvl_m = 0);
cudaError_t kh_launch_gather_rhs(int64_t n, int32_t batch, const int64_t* perm, const double* g_re,
                                 const double* g_im, int64_t ldg, double2* y, cudaStream_t stream);
cudaError_t kh_launch_scatter_sol(int64_t n, int32_t batch, const int64_t* perm, const double2* y,
                                  double* z_re, double* z_im, int64_t ldz, cudaStream_t stream);
cudaError_t kh_launch_shift_absmax_nnz(const double* mv, const double* av, int64_t nnz, int32_t batch,
                                       const double2* lam, double* part, int32_t nblk, cudaStream_t stream);
cudaError_t kh_launch_rowreduce(const double* in, int64_t len, int32_t rows, int op, double* out,
                                cudaStream_t stream);
cudaError_t kh_launch_pair_residual(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                    const double* mv, const double* av, const double* Y, int64_t ldy,
                                    const double* F, int64_t ldf, double* R, int64_t ldr, double* part,
                                    int32_t nblk, cudaStream_t stream);
// ||(|f| + |M_x| |Y1| + |A_x| |Y2|)||^2 and ||f||^2 (the scale of the terms the
// fp64 residual cancels: its evaluation floor is ~eps times that norm).
cudaError_t kh_launch_residual_scale(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                     const double* mv, const double* av, const double* Y, int64_t ldy,
                                     const double* F, int64_t ldf, double* part, int32_t nblk, cudaStream_t stream);
// Compensated (double-double) residual pieces (residual.cu).
cudaError_t kh_launch_dgemm_dd(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                               int64_t ldb, double* Chi, double* Clo, int64_t ldc, cudaStream_t stream);
cudaError_t kh_launch_pair_residual_dd(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                       const double* mv, const double* av, const double* Y1, int64_t ldy1,
                                       const double* Y2h, const double* Y2l, int64_t ldy2, const double* F,
                                       int64_t ldf, double* R, int64_t ldr, double* part, int32_t nblk,
                                       cudaStream_t stream);
cudaError_t kh_launch_sumsq(const double* x, int64_t n, double* part, int32_t nblk, cudaStream_t stream);
cudaError_t kh_launch_daxpy(int64_t n, double alpha, const double* x, double* y, cudaStream_t stream);
// Shared-memory DMMA factorization of fronts with m <= ms (ms = 32, 48 or 64).
// Fused forward solve of the factor kernels (kh_plan_factor_fwd): y holds the
// gathered rhs of the batch; rhs updates go through the level buffers of the
// solve (ru_cur: this level, ru_child: the children's level).
struct KhFwd {
  double2* y;
  double2* ru_cur;
  int64_t ru_stride_cur;
  const double2* ru_child;
  int64_t ru_stride_child;
};
cudaError_t kh_launch_factor_small(int ms, const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                   const double2* lam, double2* panels, double2* upd_cur, int64_t upd_stride_cur,
                                   const double2* upd_child, int64_t upd_stride_child, double* minpiv,
                                   cudaStream_t stream, const KhFwd* fwd = nullptr);

// Large fronts (frontal.cu), per 64-pivot super-block at column c0: pivot-block
// LDL^T writing the block's DMMA B image (tasks: front, scratch offset), the
// blocked TRSM of the rows below by 8-row warps (tasks: front, row, offset),
// the right-looking update of the later pivot columns (tasks: front, row, col).
// super-block width: 48 with the register-resident pivot kernel
// (KH_PIVOT_WARP, default), 64 with the shared-memory one
#ifndef KH_PIVOT_WARP
#define KH_PIVOT_WARP 1
#endif
__host__ __device__ constexpr int kh_piv_max() { return KH_PIVOT_WARP ? 48 : 64; }
cudaError_t kh_launch_pivot_warp(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                 double2* panels, double* minpiv, double2* img, int64_t img_stride,
                                 cudaStream_t stream);
cudaError_t kh_launch_pivot_block(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                 double2* panels, double* minpiv, double2* img, int64_t img_stride,
                                 cudaStream_t stream);
cudaError_t kh_launch_panel_solve(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                  double2* panels, const double2* img, int64_t img_stride, cudaStream_t stream);
cudaError_t kh_launch_panel_update(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                   double2* panels, cudaStream_t stream);
// Register-resident warp-per-(front, shift) factorization of the fronts with
// m <= 8 mt (warpfront.cu; mt = 4, 5 or 6): wdst[e] is the slot of original e
// in the CTA's dense originals image (kh_warp_front_slot).
int kh_warp_front_slot(int32_t m, int32_t p, int32_t r, int32_t c);
cudaError_t kh_launch_warp_front(int mt, const KhTree& T, const int32_t* level_fronts, int32_t nlev,
                                 int32_t batch, const double2* lam, double2* panels, double2* upd_cur,
                                 int64_t upd_stride_cur, const double2* upd_child, int64_t upd_stride_child,
                                 double* minpiv, const int32_t* wdst, cudaStream_t stream);

// om[e] = mv[src[e]], oa[e] = av[src[e]] (values in the order the fronts read them).
cudaError_t kh_launch_gather_orig(int64_t n_orig, const int64_t* src, const double* mv, const double* av, double* om,
                                  double* oa, cudaStream_t stream);

// Counts every kernel launch made by the library (kh_launch_count in the ABI).
void kh_note_launch();

// Dynamic shared memory above 48 KB: the opt-in attribute is per device, so it
// is cached per (kernel, current device) and raised when a larger size comes.
cudaError_t kh_smem_optin(const void* kernel, int bytes);

// Temporal H_T assembly (temporal.cu).
namespace kh_ht {
int splits(int nr);
int chunk(int nr);
int64_t workspace_doubles(int nr, int n_cells, int jc);
cudaError_t assemble(int degree, int n_cells, const double* d_nodes, double T, int64_t j_max, int jc, double* A,
                     double* M, double* C, double* ws, cudaStream_t st);
}  // namespace kh_ht
