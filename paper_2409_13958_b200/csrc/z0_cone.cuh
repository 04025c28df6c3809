// Exact element integrals of the Z0 near-field correction, host + device, fp64.
//
// For an observer o and a tetrahedron T with linear basis phi_i:
//   A_m    = int_T phi_m(r) / |o - r| dV
//   B_km   = int_T phi_k(r) phi_m(r) (o - r) / |o - r|^3 dV
// via the signed cone decomposition from o,
//   int_T g dV = sum_F h_F int_F dA(y) int_0^1 t^2 g(o + t (y - o)) dt,
// h_F = signed distance from o to the plane of face F (positive on the inner side).  With
// phi(o + t(y-o)) = a + t b (a = phi(o), b = phi(y) - phi(o)) the radial integrals are exact:
//   A : t^2 * phi_m / (t |y-o|)               -> (a_m/6 + phi_m(y)/3) / |y-o|
//   B : t^2 * phi_k phi_m (-t(y-o))/(t^3|y-o|^3) -> -(a_k a_m + (a_k b_m + a_m b_k)/2 + b_k b_m/3) (y-o)/|y-o|^3
// leaving smooth face integrals, evaluated with collapsed Gauss rules (n = 4, 6, 8 chosen by
// the size/distance ratio) on adaptively subdivided triangles (iterative, explicit stack).
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define ZC_HD __host__ __device__
#else
#define ZC_HD
#endif

namespace pmfem {

struct TriRules {              // collapsed n x n Gauss on the reference triangle, n = 4, 6, 8, 12
  double l0[260], l1[260], l2[260], w[260];
  double split;                // a face piece is subdivided while size > split * distance bound
  double thr0, thr1, thr2;     // rule by size / distance: <= thr0 -> 4x4, <= thr1 -> 6x6,
                               // <= thr2 -> 8x8, else 12x12
  int off[4], cnt[4];
};
ZC_HD inline int tri_rule(const TriRules& R, double ratio) {
  return ratio <= R.thr0 ? 0 : (ratio <= R.thr1 ? 1 : (ratio <= R.thr2 ? 2 : 3));
}

// host: fill the three rules (Gauss-Legendre nodes on [0,1] by Newton iteration)
void build_tri_rules(TriRules& R);

ZC_HD inline double zc_dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// A sub-triangle of a face (F0, F1, F2) in dyadic barycentric form: vertex k is
// F0 + (u_k E1 + v_k E2) / 2^depth with E1 = F1 - F0, E2 = F2 - F0 (exact for depth <= 7).
struct DTri { short u[3], v[3], depth, pad; };
ZC_HD inline DTri dtri_root() {
  DTri t;
  t.u[0] = 0; t.v[0] = 0; t.u[1] = 1; t.v[1] = 0; t.u[2] = 0; t.v[2] = 1; t.depth = 0; t.pad = 0;
  return t;
}
ZC_HD inline void dtri_vertices(const double* F0, const double* E1, const double* E2, const DTri& t, double V[3][3]) {
  const double s = 1.0 / (double)(1 << t.depth);
  for (int k = 0; k < 3; ++k)
    for (int x = 0; x < 3; ++x) V[k][x] = F0[x] + ((double)t.u[k] * E1[x] + (double)t.v[k] * E2[x]) * s;
}
// the 4 children (corner 0, corner 1, corner 2, centre) in the order of the round-1 subdivision
ZC_HD inline void dtri_children(const DTri& t, DTri* c) {
  short U[3], Vv[3], mu[3], mv[3];
  for (int k = 0; k < 3; ++k) { U[k] = 2 * t.u[k]; Vv[k] = 2 * t.v[k]; }
  // midpoints m01, m02, m12
  mu[0] = t.u[0] + t.u[1]; mv[0] = t.v[0] + t.v[1];
  mu[1] = t.u[0] + t.u[2]; mv[1] = t.v[0] + t.v[2];
  mu[2] = t.u[1] + t.u[2]; mv[2] = t.v[1] + t.v[2];
  const short cu[4][3] = {{U[0], mu[0], mu[1]}, {mu[0], U[1], mu[2]}, {mu[1], mu[2], U[2]}, {mu[2], mu[1], mu[0]}};
  const short cv[4][3] = {{Vv[0], mv[0], mv[1]}, {mv[0], Vv[1], mv[2]}, {mv[1], mv[2], Vv[2]}, {mv[2], mv[1], mv[0]}};
  for (int i = 0; i < 4; ++i) {
    for (int k = 0; k < 3; ++k) { c[i].u[k] = cu[i][k]; c[i].v[k] = cv[i][k]; }
    c[i].depth = t.depth + 1;
    c[i].pad = 0;
  }
}
// size (longest edge) and the distance lower bound max(|h|, |centroid - o| - circumradius)
ZC_HD inline void dtri_measure(const double V[3][3], const double* o, double h, double& size, double& dest) {
  double cen[3], e01[3], e02[3], e12[3];
  for (int x = 0; x < 3; ++x) {
    cen[x] = (V[0][x] + V[1][x] + V[2][x]) / 3.0;
    e01[x] = V[1][x] - V[0][x]; e02[x] = V[2][x] - V[0][x]; e12[x] = V[2][x] - V[1][x];
  }
  size = sqrt(fmax(zc_dot(e01, e01), fmax(zc_dot(e02, e02), zc_dot(e12, e12))));
  double rc = 0;
  for (int k = 0; k < 3; ++k) {
    const double d[3] = {V[k][0] - cen[0], V[k][1] - cen[1], V[k][2] - cen[2]};
    rc = fmax(rc, sqrt(zc_dot(d, d)));
  }
  const double dc[3] = {cen[0] - o[0], cen[1] - o[1], cen[2] - o[2]};
  dest = fmax(fabs(h), sqrt(zc_dot(dc, dc)) - rc);
}

struct ConeIntegrator {
  double P[4][3], g[4][3], c[4];     // phi_i(r) = c_i + g_i . r
  double o[3], a[4];
  double A[4], B[4][4][3];
  const TriRules* R;
  long long npts = 0;                // quadrature points evaluated (cost diagnostics)

  ZC_HD double phi(int i, const double* r) const { return c[i] + zc_dot(g[i], r); }

  ZC_HD void quad(const double* V0, const double* V1, const double* V2, double h, double size, double dest) {
    double e01[3], e02[3];
    for (int x = 0; x < 3; ++x) { e01[x] = V1[x] - V0[x]; e02[x] = V2[x] - V0[x]; }
    const double cr[3] = {e01[1] * e02[2] - e01[2] * e02[1], e01[2] * e02[0] - e01[0] * e02[2],
                          e01[0] * e02[1] - e01[1] * e02[0]};
    const double area2 = sqrt(zc_dot(cr, cr));
    const double ratio = size / dest;
    const int r = tri_rule(*R, ratio);
    npts += R->cnt[r];
    for (int q = R->off[r]; q < R->off[r] + R->cnt[r]; ++q) {
      double y[3];
      for (int x = 0; x < 3; ++x) y[x] = R->l0[q] * V0[x] + R->l1[q] * V1[x] + R->l2[q] * V2[x];
      const double Rv[3] = {y[0] - o[0], y[1] - o[1], y[2] - o[2]};
      const double inv = 1.0 / sqrt(zc_dot(Rv, Rv));
      const double inv3 = inv * inv * inv;
      const double w = R->w[q] * area2 * h;
      double py[4], b[4];
      for (int i = 0; i < 4; ++i) { py[i] = phi(i, y); b[i] = py[i] - a[i]; }
      for (int m = 0; m < 4; ++m) A[m] += w * (a[m] / 6.0 + py[m] / 3.0) * inv;
      for (int k = 0; k < 4; ++k)
        for (int m = k; m < 4; ++m) {
          const double s = -w * (a[k] * a[m] + 0.5 * (a[k] * b[m] + a[m] * b[k]) + b[k] * b[m] / 3.0) * inv3;
          for (int x = 0; x < 3; ++x) B[k][m][x] += s * Rv[x];
        }
    }
  }

  // adaptive face integral: split into 4 while size > split * dest (distance lower bound),
  // depth <= 7; sub-triangles in dyadic barycentric form (DTri, shared with the GPU's
  // breadth-first version in z0_gpu.cu: the same leaves, the same vertex arithmetic).  The
  // depth-first stack never overflows (3 per level + 4 <= 24 for depth < 7), so the leaf set does
  // not depend on the traversal order.
  ZC_HD void face(const double* F0, const double* F1, const double* F2, double h) {
    double E1[3], E2[3];
    for (int x = 0; x < 3; ++x) { E1[x] = F1[x] - F0[x]; E2[x] = F2[x] - F0[x]; }
    DTri stack[24];
    int top = 1;
    stack[0] = dtri_root();
    while (top > 0) {
      const DTri T = stack[--top];
      double V[3][3], size, dest;
      dtri_vertices(F0, E1, E2, T, V);
      dtri_measure(V, o, h, size, dest);
      if (size > R->split * dest && T.depth < 7) {
        dtri_children(T, stack + top);
        top += 4;
        continue;
      }
      quad(V[0], V[1], V[2], h, size, dest);
    }
  }

  // va >= 0: o is vertex va of T (only the opposite face has h != 0)
  ZC_HD void run(int va) {
    for (int i = 0; i < 4; ++i) {
      A[i] = 0;
      for (int j = 0; j < 4; ++j)
        for (int x = 0; x < 3; ++x) B[i][j][x] = 0;
    }
    for (int i = 0; i < 4; ++i) c[i] = 1.0 - zc_dot(g[i], P[i]);
    for (int i = 0; i < 4; ++i) a[i] = (va >= 0) ? (i == va ? 1.0 : 0.0) : phi(i, o);
    for (int j = 0; j < 4; ++j) {
      if (va >= 0 && j != va) continue;
      const double gn = sqrt(zc_dot(g[j], g[j]));
      const double h = a[j] / gn;            // phi_j(o) = |g_j| h_j
      if (fabs(h) * gn < 1e-14) continue;
      face(P[(j + 1) % 4], P[(j + 2) % 4], P[(j + 3) % 4], h);
    }
    for (int k = 0; k < 4; ++k)
      for (int m = 0; m < k; ++m)
        for (int x = 0; x < 3; ++x) B[k][m][x] = B[m][k][x];
  }
};

// element gradients from vertex coordinates: grad phi_i = rows of J^-1 (J cols = P_i - P_0)
ZC_HD inline void tet_grads(const double P[4][3], double g[4][3]) {
  double e[3][3];
  for (int k = 0; k < 3; ++k)
    for (int x = 0; x < 3; ++x) e[k][x] = P[k + 1][x] - P[0][x];
  auto cross = [](const double* u, const double* v, double* w) {
    w[0] = u[1] * v[2] - u[2] * v[1]; w[1] = u[2] * v[0] - u[0] * v[2]; w[2] = u[0] * v[1] - u[1] * v[0];
  };
  cross(e[1], e[2], g[1]);
  cross(e[2], e[0], g[2]);
  cross(e[0], e[1], g[3]);
  const double det = zc_dot(e[0], g[1]);
  for (int k = 1; k < 4; ++k)
    for (int x = 0; x < 3; ++x) g[k][x] /= det;
  for (int x = 0; x < 3; ++x) g[0][x] = -(g[1][x] + g[2][x] + g[3][x]);
}

}  // namespace pmfem
