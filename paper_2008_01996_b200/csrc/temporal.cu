// Temporal H_T matrices on the GPU: the truncated
// sine series of reference temporal.py:98-151, 300-329 (P1 hats) and of the
// P2 Lagrange basis (p2.py), for graded or uniform partitions of (0, T):
//
//   A = 1/2 sum_j theta_j a_j a_j^T,  M = sum_j a_j b_j^T,  C = sum_j a_j d_j^T
//
// over frequencies theta_j = pi (j + 1/2), j = 0..j_max. Per chunk of JC
// frequencies (descending j, like the reference's accumulation order):
//   1. ht_coeff_kernel writes the coefficient panels -- (a sqrt(theta/2)) and
//      a with the basis index fastest (GEMM "A" operands), and
//      (a sqrt(theta/2)), b and d with the frequency fastest (GEMM "B"
//      operands) -- each from sincospi of (j + 1/2) t_i / T (exact argument
//      reduction; the node values are recomputed per basis function, which is
//      cheap next to the GEMMs);
//   2. three batched DMMA GEMMs (dgemm.cu) over S split-K slices write S
//      partial products each (S chosen to fill the 148 SMs);
//   3. ht_accumulate_kernel adds the S partials to A, M, C in slice order
//      (deterministic).
// Work per chunk: 2 N_r^2 JC flops each for A and M, 2 N_r N_c JC for C
// (N_r = basis functions, N_c = cells): DMMA-bound.
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

struct NodeTrig {
  double s, c;
};

KH_DEV NodeTrig trig(const double* nodes, int i, double jh, double T) {
  NodeTrig r;
  sincospi(jh * (nodes[i] / T), &r.s, &r.c);
  return r;
}

// Coefficients of basis function `row` at frequency index j (jh = j + 1/2).
// out[0] = a, out[1] = b (cosine integral), out[2] = d of cell `row` (when
// row < n_cells).
template <int DEG>
KH_DEV void coeffs(const double* nodes, int n_cells, int row, double jh, double T, double out[3]) {
  const double theta = kPi * jh;
  const double w = theta / T;
  const double sign = (((int64_t)(jh - 0.5)) & 1) ? -1.0 : 1.0;
  if (DEG == 1) {
    // hat at node row+1: cells row (rising) and row+1 (falling)
    const int l = row;
    NodeTrig t0 = trig(nodes, l, jh, T), t1 = trig(nodes, l + 1, jh, T);
    const double h0 = nodes[l + 1] - nodes[l];
    double bs = (t1.s - t0.s) / h0, bc = (t1.c - t0.c) / h0;
    if (l + 1 < n_cells) {
      NodeTrig t2 = trig(nodes, l + 2, jh, T);
      const double h1 = nodes[l + 2] - nodes[l + 1];
      bs -= (t2.s - t1.s) / h1;
      bc -= (t2.c - t1.c) / h1;
    }
    out[0] = bs * (2.0 * T / (theta * theta));
    out[1] = bc * (T * T / (theta * theta));
    if (l == n_cells - 1) out[1] += sign * T / theta;
    out[2] = (t1.s - t0.s) * (T / theta);
  } else {
    // P2: row 2c = midpoint of cell c (L1), row 2c+1 = vertex t_{c+1}
    // (L2 of cell c + L0 of cell c+1)
    const int c = row >> 1;
    const bool mid = (row & 1) == 0;
    double si = 0.0, ci = 0.0;
    auto cell = [&](int cc, double dl, double dr, double d2) {
      NodeTrig ta = trig(nodes, cc, jh, T), tb = trig(nodes, cc + 1, jh, T);
      const double h = nodes[cc + 1] - nodes[cc];
      const double ih = 1.0 / h, ih2 = ih * ih;
      const double qs = (dr * tb.s - dl * ta.s) * ih, qc = (dr * tb.c - dl * ta.c) * ih;
      const double q2 = d2 * ih2;
      si += (qs / w + q2 * (tb.c - ta.c) / (w * w)) / w;
      ci += (qc / w - q2 * (tb.s - ta.s) / (w * w)) / w;
    };
    if (mid) {
      cell(c, 4.0, -4.0, -8.0);
    } else {
      cell(c, -1.0, 3.0, 4.0);
      if (c + 1 < n_cells) cell(c + 1, -3.0, 1.0, 4.0);
    }
    out[0] = si * (2.0 / T);
    out[1] = ci;
    if (row == 2 * n_cells - 1) out[1] += sign * T / theta;
    out[2] = 0.0;
    if (row < n_cells) {
      NodeTrig ta = trig(nodes, row, jh, T), tb = trig(nodes, row + 1, jh, T);
      out[2] = (tb.s - ta.s) * (T / theta);
    }
  }
}

// ROWS layout: element (row, k) at row + k * nr (basis index fastest): writes
// wa_r, a_r. COLS layout: element (k, row) at k + row * jc (frequency
// fastest): writes wa_c, b_c, d_c. Frequencies beyond j_end are zero.
template <int DEG, bool ROWS>
__global__ void __launch_bounds__(256) ht_coeff_kernel(const double* __restrict__ nodes, int n_cells, int nr, double T,
                                                       int64_t j0, int jc, int64_t j_end, double* __restrict__ o0,
                                                       double* __restrict__ o1, double* __restrict__ o2) {
  const int64_t total = (int64_t)nr * jc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int row, k;
    if (ROWS) {
      row = (int)(e % nr);
      k = (int)(e / nr);
    } else {
      k = (int)(e % jc);
      row = (int)(e / jc);
    }
    const int64_t j = j0 + k;
    double v[3] = {0.0, 0.0, 0.0};
    double wa = 0.0;
    if (j < j_end) {
      const double jh = (double)j + 0.5;
      coeffs<DEG>(nodes, n_cells, row, jh, T, v);
      wa = v[0] * sqrt(0.5 * kPi * jh);
    }
    if (ROWS) {
      o0[e] = wa;
      o1[e] = v[0];
    } else {
      o0[e] = wa;
      o1[e] = v[1];
      if (row < n_cells) o2[(int64_t)row * jc + k] = v[2];
    }
  }
}

// dst[e] += sum_{s < S} parts[s * len + e]
__global__ void ht_accumulate_kernel(int32_t S, const double* __restrict__ parts, int64_t len, double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int32_t s = 0; s < S; ++s) acc += parts[(int64_t)s * len + e];
    dst[e] += acc;
  }
}

int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? b : 148 * 16);
}

}  // namespace

namespace kh_ht {

int splits(int nr) {
  const int64_t ctas = ((nr + 127) / 128) * (int64_t)((nr + 63) / 64);
  int64_t s = (2 * 148 + ctas - 1) / ctas;
  return (int)(s < 1 ? 1 : (s > 64 ? 64 : s));
}

// chunk length: S slices of a multiple of 16 frequencies, ~8192 in total
int chunk(int nr) {
  const int S = splits(nr);
  int ks = (8192 / S + 15) / 16 * 16;
  return S * (ks < 16 ? 16 : ks);
}

int64_t workspace_doubles(int nr, int n_cells, int jc) {
  const int S = splits(nr);
  return (int64_t)jc * (4 * (int64_t)nr + n_cells) + (int64_t)S * (2 * (int64_t)nr * nr + (int64_t)nr * n_cells);
}

// A, M: nr x nr, C: nr x n_cells, column-major device buffers, overwritten.
cudaError_t assemble(int degree, int n_cells, const double* d_nodes, double T, int64_t j_max, int jc, double* A,
                     double* M, double* C, double* ws, cudaStream_t st) {
  const int nr = degree * n_cells;
  const int S = splits(nr);
  const int ks = jc / S;  // slice length (jc is a multiple of 16 * S)
  double* wa_r = ws;
  double* a_r = wa_r + (int64_t)nr * jc;
  double* wa_c = a_r + (int64_t)nr * jc;
  double* b_c = wa_c + (int64_t)nr * jc;
  double* d_c = b_c + (int64_t)nr * jc;
  double* pA = d_c + (int64_t)n_cells * jc;
  double* pM = pA + (int64_t)S * nr * nr;
  double* pC = pM + (int64_t)S * nr * nr;
  cudaError_t e;
  if ((e = cudaMemsetAsync(A, 0, sizeof(double) * nr * nr, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(M, 0, sizeof(double) * nr * nr, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(C, 0, sizeof(double) * nr * n_cells, st)) != cudaSuccess) return e;
  const int64_t j_end = j_max + 1;
  const int64_t top = (j_max / jc) * jc;
  const int nb = blocks_for((int64_t)nr * jc);
  for (int64_t j0 = top; j0 >= 0; j0 -= jc) {
    if (degree == 1) {
      ht_coeff_kernel<1, true><<<nb, 256, 0, st>>>(d_nodes, n_cells, nr, T, j0, jc, j_end, wa_r, a_r, nullptr);
      ht_coeff_kernel<1, false><<<nb, 256, 0, st>>>(d_nodes, n_cells, nr, T, j0, jc, j_end, wa_c, b_c, d_c);
    } else {
      ht_coeff_kernel<2, true><<<nb, 256, 0, st>>>(d_nodes, n_cells, nr, T, j0, jc, j_end, wa_r, a_r, nullptr);
      ht_coeff_kernel<2, false><<<nb, 256, 0, st>>>(d_nodes, n_cells, nr, T, j0, jc, j_end, wa_c, b_c, d_c);
    }
    kh_note_launch();
    kh_note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // slice s covers chunk columns [s ks, (s+1) ks)
    if ((e = kh_launch_dgemm_batched(nr, nr, ks, 1.0, wa_r, nr, (int64_t)nr * ks, wa_c, jc, ks, 0.0, pA, nr,
                                     (int64_t)nr * nr, S, st)) != cudaSuccess)
      return e;
    if ((e = kh_launch_dgemm_batched(nr, nr, ks, 1.0, a_r, nr, (int64_t)nr * ks, b_c, jc, ks, 0.0, pM, nr,
                                     (int64_t)nr * nr, S, st)) != cudaSuccess)
      return e;
    if ((e = kh_launch_dgemm_batched(nr, n_cells, ks, 1.0, a_r, nr, (int64_t)nr * ks, d_c, jc, ks, 0.0, pC, nr,
                                     (int64_t)nr * n_cells, S, st)) != cudaSuccess)
      return e;
    ht_accumulate_kernel<<<blocks_for((int64_t)nr * nr), 256, 0, st>>>(S, pA, (int64_t)nr * nr, A);
    ht_accumulate_kernel<<<blocks_for((int64_t)nr * nr), 256, 0, st>>>(S, pM, (int64_t)nr * nr, M);
    ht_accumulate_kernel<<<blocks_for((int64_t)nr * n_cells), 256, 0, st>>>(S, pC, (int64_t)nr * n_cells, C);
    kh_note_launch();
    kh_note_launch();
    kh_note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace kh_ht
