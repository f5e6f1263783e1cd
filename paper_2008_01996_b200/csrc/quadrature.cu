// Space-time quadrature on the GPU: the RHS
// projection of reference fem.py:267-297 and the error norms of
// fem.py:358-418, for P1 triangles x temporal cells.
//
// This file is a template compiled at run time with NVRTC
// (quadrature_gpu.py): the user's fields arrive as C expressions in x, y, t
// through the macros KH_F (right-hand side), KH_U, KH_UX, KH_UY, KH_UT
// (exact solution, gradient, time derivative); the quadrature tables
// (triangle rule, per-cell time panels) are kernel arguments, the same rules
// as the host code (fem.triangle_rule, fem._time_panels).
//
// project_rhs_kernel: one thread per (triangle, cell), cell index fastest
//   (coalesced writes of the n_tri x n_cells result):
//   out[tri, ell] = 2 sum_panels w_q sum_i w_i f(x_i, y_i, t_ell + h q).
// error_norms_kernel: one thread per triangle looping over all cells and
//   time panels; writes the triangle's (L2^2, H1^2) partial sums, which the
//   host reduces in a fixed order (deterministic).
#ifndef KH_PI
#define KH_PI 3.141592653589793238462643383279502884
#endif

#define KH_MAXQ 64  // spatial quadrature points held per thread

extern "C" __global__ void project_rhs_kernel(const double* __restrict__ verts, const long long* __restrict__ tris,
                                              long long n_tri, const double* __restrict__ nodes, int n_cells,
                                              const double* __restrict__ pts, const double* __restrict__ wts, int nq,
                                              const double* __restrict__ tq0, const double* __restrict__ tw0, int nt0,
                                              const double* __restrict__ tq1, const double* __restrict__ tw1, int nt1,
                                              double* __restrict__ out) {
  const long long total = n_tri * (long long)n_cells;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long tri = e / n_cells;
    const int ell = (int)(e - tri * n_cells);
    const long long a = tris[3 * tri], b = tris[3 * tri + 1], c = tris[3 * tri + 2];
    const double ax = verts[2 * a], ay = verts[2 * a + 1];
    const double bx = verts[2 * b], by = verts[2 * b + 1];
    const double cx = verts[2 * c], cy = verts[2 * c + 1];
    const double t0 = nodes[ell], h = nodes[ell + 1] - t0;
    const double* tq = ell == 0 ? tq0 : tq1;
    const double* tw = ell == 0 ? tw0 : tw1;
    const int ntq = ell == 0 ? nt0 : nt1;
    double acc = 0.0;
    for (int iq = 0; iq < ntq; ++iq) {
      const double t = t0 + h * tq[iq];
      double s = 0.0;
      for (int i = 0; i < nq; ++i) {
        const double l1 = pts[2 * i], l2 = pts[2 * i + 1], l0 = 1.0 - l1 - l2;
        const double x = l0 * ax + l1 * bx + l2 * cx;
        const double y = l0 * ay + l1 * by + l2 * cy;
        s += (KH_F) * wts[i];
      }
      acc += tw[iq] * s;
    }
    out[e] = 2.0 * acc;
  }
}

// coeffs: n_vertices x (n_cells + 1) row-major, column 0 = t_0 (zeros)
extern "C" __global__ void error_norms_kernel(const double* __restrict__ verts, const long long* __restrict__ tris,
                                              long long n_tri, const double* __restrict__ nodes, int n_cells,
                                              const double* __restrict__ pts, const double* __restrict__ wts, int nq,
                                              const double* __restrict__ tq0, const double* __restrict__ tw0, int nt0,
                                              const double* __restrict__ tq1, const double* __restrict__ tw1, int nt1,
                                              const double* __restrict__ coeffs, double* __restrict__ part) {
  for (long long tri = blockIdx.x * (long long)blockDim.x + threadIdx.x; tri < n_tri;
       tri += (long long)gridDim.x * blockDim.x) {
    const long long v[3] = {tris[3 * tri], tris[3 * tri + 1], tris[3 * tri + 2]};
    const double px[3] = {verts[2 * v[0]], verts[2 * v[1]], verts[2 * v[2]]};
    const double py[3] = {verts[2 * v[0] + 1], verts[2 * v[1] + 1], verts[2 * v[2] + 1]};
    // P1 geometry (fem._geometry): gradients of the barycentric coordinates
    const double bb[3] = {py[1] - py[2], py[2] - py[0], py[0] - py[1]};
    const double cc[3] = {px[2] - px[1], px[0] - px[2], px[1] - px[0]};
    const double two_area = bb[0] * cc[1] - bb[1] * cc[0];
    const double area = 0.5 * two_area;
    double gx[3], gy[3];
    for (int k = 0; k < 3; ++k) {
      gx[k] = bb[k] / two_area;
      gy[k] = cc[k] / two_area;
    }
    double l2 = 0.0, h1 = 0.0;
    for (int ell = 0; ell < n_cells; ++ell) {
      const double t0 = nodes[ell], h = nodes[ell + 1] - t0;
      double clo[3], chi[3], cdt[3];
      for (int k = 0; k < 3; ++k) {
        clo[k] = coeffs[v[k] * (n_cells + 1) + ell];
        chi[k] = coeffs[v[k] * (n_cells + 1) + ell + 1];
        cdt[k] = (chi[k] - clo[k]) / h;
      }
      const double* tq = ell == 0 ? tq0 : tq1;
      const double* tw = ell == 0 ? tw0 : tw1;
      const int ntq = ell == 0 ? nt0 : nt1;
      for (int iq = 0; iq < ntq; ++iq) {
        const double q = tq[iq];
        const double t = t0 + h * q;
        double c[3];
        for (int k = 0; k < 3; ++k) c[k] = (1.0 - q) * clo[k] + q * chi[k];
        const double ghx = c[0] * gx[0] + c[1] * gx[1] + c[2] * gx[2];
        const double ghy = c[0] * gy[0] + c[1] * gy[1] + c[2] * gy[2];
        double sl2 = 0.0, sh1 = 0.0;
        for (int i = 0; i < nq; ++i) {
          const double l1 = pts[2 * i], l2b = pts[2 * i + 1], l0 = 1.0 - l1 - l2b;
          const double x = l0 * px[0] + l1 * px[1] + l2b * px[2];
          const double y = l0 * py[0] + l1 * py[1] + l2b * py[2];
          const double uh = c[0] * l0 + c[1] * l1 + c[2] * l2b;
          const double duh = cdt[0] * l0 + cdt[1] * l1 + cdt[2] * l2b;
          const double w = 2.0 * area * wts[i];
          const double e = (KH_U) - uh;
          const double ed = (KH_UT) - duh;
          const double e1 = (KH_UX) - ghx, e2 = (KH_UY) - ghy;
          sl2 += w * e * e;
          sh1 += w * (ed * ed + e1 * e1 + e2 * e2);
        }
        const double wt = tw[iq] * h;
        l2 += wt * sl2;
        h1 += wt * sh1;
      }
    }
    part[2 * tri] = l2;
    part[2 * tri + 1] = h1;
  }
}
