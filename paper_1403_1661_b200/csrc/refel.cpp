// refel.cpp -- reference-element builder of the product path.
//
// Operators of the nodal DG discretisation (P:81 Warp & Blend Lagrange basis,
// triangle cubature, Gauss edge quadrature; P:651 P, Pr, Ps "pre multiplied
// with cubature integration weights"; P:691 lift L^g; P:716 Gauss
// interpolation), built from the orthonormal Dubiner basis
//   psi_ij(r,s) = sqrt2 Phat_i^{(0,0)}(a) Phat_j^{(2i+1,0)}(b) (1-b)^i,
//   a = 2(1+r)/(1-s) - 1, b = s,
// and Gauss rules obtained as eigenvalues of the Jacobi matrix (Sturm
// bisection, Golub-Welsch weights).  Readings: cubature = the
// symmetric degree-2N rule (A2', the paper's "integration order 2N" from
// Cools' rules) for N <= 5; Ng = N+1 Gauss points per face.
#include <algorithm>
#include <cmath>

#include "host.hpp"

namespace swe {

namespace {

// Jacobi-matrix recurrence coefficients (monic) for weight (1-x)^al (1+x)^be.
void jacobi_recurrence(int n, double al, double be, std::vector<double> &a, std::vector<double> &b, double &mu0) {
  a.assign(n, 0.0);
  b.assign(n, 0.0);  // b[0] unused
  for (int k = 0; k < n; k++) {
    double s = 2.0 * k + al + be;
    if (k == 0)
      a[k] = (be - al) / (al + be + 2.0);
    else
      a[k] = (be * be - al * al) / (s * (s + 2.0));
    if (k >= 1) {
      double num = 4.0 * k * (k + al) * (k + be) * (k + al + be);
      double den = s * s * (s + 1.0) * (s - 1.0);
      b[k] = num / den;
    }
  }
  mu0 = std::pow(2.0, al + be + 1.0) * std::tgamma(al + 1.0) * std::tgamma(be + 1.0) / std::tgamma(al + be + 2.0);
}

// Orthonormal polynomials phat_0..phat_{n} at x (and derivatives) from the recurrence.
void orthonormal_values(int n, const std::vector<double> &a, const std::vector<double> &b, double mu0, double x,
                        std::vector<double> &p, std::vector<double> &dp) {
  p.assign(n + 1, 0.0);
  dp.assign(n + 1, 0.0);
  p[0] = 1.0 / std::sqrt(mu0);
  for (int k = 0; k < n; k++) {
    double sb1 = std::sqrt(b[k + 1]);
    double prev = k > 0 ? p[k - 1] : 0.0, dprev = k > 0 ? dp[k - 1] : 0.0;
    double sbk = k > 0 ? std::sqrt(b[k]) : 0.0;
    p[k + 1] = ((x - a[k]) * p[k] - sbk * prev) / sb1;
    dp[k + 1] = ((x - a[k]) * dp[k] + p[k] - sbk * dprev) / sb1;
  }
}

// n-point Gauss rule for weight (1-x)^al (1+x)^be: eigenvalues of the
// symmetric tridiagonal Jacobi matrix by Sturm-sequence bisection, one Newton
// polish on phat_n, weights w_i = 1 / sum_k phat_k(x_i)^2 (Christoffel numbers).
void gauss_rule(int n, double al, double be, std::vector<double> &x, std::vector<double> &w) {
  std::vector<double> a, b;
  double mu0;
  jacobi_recurrence(n + 1, al, be, a, b, mu0);
  auto count_below = [&](double t) {
    int c = 0;
    double q = a[0] - t;
    if (q < 0) c++;
    for (int i = 1; i < n; i++) {
      double qq = q != 0.0 ? q : 1e-300;
      q = a[i] - t - b[i] / qq;
      if (q < 0) c++;
    }
    return c;
  };
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 0; k < n; k++) {
    double lo = -1.0, hi = 1.0;
    for (int it = 0; it < 200 && hi - lo > 0; it++) {
      double mid = 0.5 * (lo + hi);
      if (mid == lo || mid == hi) break;
      if (count_below(mid) > k)
        hi = mid;
      else
        lo = mid;
    }
    double xk = 0.5 * (lo + hi);
    std::vector<double> p, dp;
    for (int it = 0; it < 2; it++) {
      orthonormal_values(n, a, b, mu0, xk, p, dp);
      if (dp[n] != 0.0) xk -= p[n] / dp[n];
    }
    orthonormal_values(n, a, b, mu0, xk, p, dp);
    double sum = 0.0;
    for (int j = 0; j < n; j++) sum += p[j] * p[j];
    x[k] = xk;
    w[k] = 1.0 / sum;
  }
}

// Orthonormal Jacobi polynomial Phat_n^{(al,be)} and derivative at x.
void jacobi_phat(int n, double al, double be, double x, double &v, double &dv) {
  std::vector<double> a, b, p, dp;
  double mu0;
  jacobi_recurrence(n + 1, al, be, a, b, mu0);
  orthonormal_values(n, a, b, mu0, x, p, dp);
  v = p[n];
  dv = dp[n];
}

// Dubiner basis value and (r,s)-gradient.
void dubiner(int i, int j, double r, double s, double &f, double &fr, double &fs) {
  double a = (s != 1.0) ? 2.0 * (1.0 + r) / (1.0 - s) - 1.0 : -1.0;
  double b = s;
  double A, dA, Bj, dBj;
  jacobi_phat(i, 0.0, 0.0, a, A, dA);
  jacobi_phat(j, 2.0 * i + 1.0, 0.0, b, Bj, dBj);
  const double sq2 = std::sqrt(2.0);
  double om = 1.0 - b;
  double omi = std::pow(om, i), omi1 = i > 0 ? std::pow(om, i - 1) : 0.0;
  f = sq2 * A * Bj * omi;
  // d/dr = 2/(1-b) d/da ; d/ds = (1+a)/(1-b) d/da + d/db
  fr = i > 0 ? 2.0 * sq2 * dA * Bj * omi1 : 0.0;
  double dfa_over = i > 0 ? sq2 * (1.0 + a) * dA * Bj * omi1 : 0.0;
  double dfb = sq2 * A * (dBj * omi - (i > 0 ? i * Bj * omi1 : 0.0));
  fs = dfa_over + dfb;
}

DMat vandermonde(int N, const std::vector<double> &r, const std::vector<double> &s, int which) {
  int Np = (N + 1) * (N + 2) / 2;
  DMat V((int)r.size(), Np);
  for (size_t p = 0; p < r.size(); p++) {
    int m = 0;
    for (int i = 0; i <= N; i++)
      for (int j = 0; j <= N - i; j++) {
        double f, fr, fs;
        dubiner(i, j, r[p], s[p], f, fr, fs);
        V((int)p, m++) = which == 0 ? f : (which == 1 ? fr : fs);
      }
  }
  return V;
}

DMat mul(const DMat &A, const DMat &B) {
  DMat C(A.rows, B.cols);
  for (int i = 0; i < A.rows; i++)
    for (int k = 0; k < A.cols; k++) {
      double aik = A(i, k);
      for (int j = 0; j < B.cols; j++) C(i, j) += aik * B(k, j);
    }
  return C;
}

DMat transpose(const DMat &A) {
  DMat T(A.cols, A.rows);
  for (int i = 0; i < A.rows; i++)
    for (int j = 0; j < A.cols; j++) T(j, i) = A(i, j);
  return T;
}

// LU with partial pivoting, then column-by-column solves.
bool invert(const DMat &A, DMat &Ainv) {
  int n = A.rows;
  DMat LU = A;
  std::vector<int> piv(n);
  for (int i = 0; i < n; i++) piv[i] = i;
  for (int k = 0; k < n; k++) {
    int p = k;
    for (int i = k + 1; i < n; i++)
      if (std::fabs(LU(i, k)) > std::fabs(LU(p, k))) p = i;
    if (LU(p, k) == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < n; j++) std::swap(LU(k, j), LU(p, j));
      std::swap(piv[k], piv[p]);
    }
    for (int i = k + 1; i < n; i++) {
      LU(i, k) /= LU(k, k);
      for (int j = k + 1; j < n; j++) LU(i, j) -= LU(i, k) * LU(k, j);
    }
  }
  Ainv = DMat(n, n);
  std::vector<double> y(n);
  for (int c = 0; c < n; c++) {
    for (int i = 0; i < n; i++) {
      double v = (piv[i] == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; j++) v -= LU(i, j) * y[j];
      y[i] = v;
    }
    for (int i = n - 1; i >= 0; i--) {
      double v = y[i];
      for (int j = i + 1; j < n; j++) v -= LU(i, j) * Ainv(j, c);
      Ainv(i, c) = v / LU(i, i);
    }
  }
  return true;
}

// Warp & Blend (Hesthaven-Warburton): warp of the 1D equispaced -> LGL map,
// evaluated through the Legendre Vandermonde system of the equispaced points.
std::vector<double> warp_factor(int N, const std::vector<double> &rout) {
  std::vector<double> lgl(N + 1), req(N + 1), xi, wi;
  lgl[0] = -1.0;
  lgl[N] = 1.0;
  if (N > 1) {
    gauss_rule(N - 1, 1.0, 1.0, xi, wi);  // interior LGL points = Gauss-Jacobi(1,1)
    for (int k = 0; k < N - 1; k++) lgl[k + 1] = xi[k];
  }
  for (int k = 0; k <= N; k++) req[k] = -1.0 + 2.0 * k / N;
  DMat Veq(N + 1, N + 1), Veqinv;
  for (int i = 0; i <= N; i++)
    for (int k = 0; k <= N; k++) {
      double v, dv;
      jacobi_phat(k, 0.0, 0.0, req[i], v, dv);
      Veq(i, k) = v;
    }
  invert(Veq, Veqinv);
  std::vector<double> out(rout.size());
  for (size_t p = 0; p < rout.size(); p++) {
    // l_i(r) = sum_k Veqinv(k, i) P_k(r)
    std::vector<double> Pk(N + 1);
    for (int k = 0; k <= N; k++) {
      double v, dv;
      jacobi_phat(k, 0.0, 0.0, rout[p], v, dv);
      Pk[k] = v;
    }
    double w = 0.0;
    for (int i = 0; i <= N; i++) {
      double li = 0.0;
      for (int k = 0; k <= N; k++) li += Veqinv(k, i) * Pk[k];
      w += li * (lgl[i] - req[i]);
    }
    double r = rout[p];
    out[p] = (std::fabs(r) < 1.0 - 1e-10) ? w / (1.0 - r * r) : 0.0;
  }
  return out;
}

void nodes2d(int N, std::vector<double> &r, std::vector<double> &s) {
  static const double alpopt[15] = {0.0000, 0.0000, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
                                    1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258};
  const double alpha = alpopt[N - 1];
  const double pi = std::acos(-1.0), sq3 = std::sqrt(3.0);
  int Np = (N + 1) * (N + 2) / 2;
  std::vector<double> L1(Np), L2(Np), L3(Np);
  int k = 0;
  for (int n = 1; n <= N + 1; n++)
    for (int m = 1; m <= N + 2 - n; m++) {
      L1[k] = (n - 1.0) / N;
      L3[k] = (m - 1.0) / N;
      L2[k] = 1.0 - L1[k] - L3[k];
      k++;
    }
  std::vector<double> d1(Np), d2(Np), d3(Np);
  for (int i = 0; i < Np; i++) {
    d1[i] = L3[i] - L2[i];
    d2[i] = L1[i] - L3[i];
    d3[i] = L2[i] - L1[i];
  }
  std::vector<double> w1 = warp_factor(N, d1), w2 = warp_factor(N, d2), w3 = warp_factor(N, d3);
  r.assign(Np, 0.0);
  s.assign(Np, 0.0);
  for (int i = 0; i < Np; i++) {
    double x = -L2[i] + L3[i], y = (-L2[i] - L3[i] + 2.0 * L1[i]) / sq3;
    double W1 = 4.0 * L2[i] * L3[i] * w1[i] * (1.0 + (alpha * L1[i]) * (alpha * L1[i]));
    double W2 = 4.0 * L1[i] * L3[i] * w2[i] * (1.0 + (alpha * L2[i]) * (alpha * L2[i]));
    double W3 = 4.0 * L1[i] * L2[i] * w3[i] * (1.0 + (alpha * L3[i]) * (alpha * L3[i]));
    x += W1 + std::cos(2.0 * pi / 3.0) * W2 + std::cos(4.0 * pi / 3.0) * W3;
    y += std::sin(2.0 * pi / 3.0) * W2 + std::sin(4.0 * pi / 3.0) * W3;
    double l1 = (sq3 * y + 1.0) / 3.0, l2 = (-3.0 * x - sq3 * y + 2.0) / 6.0, l3 = (3.0 * x - sq3 * y + 2.0) / 6.0;
    r[i] = -l2 + l3 - l1;
    s[i] = -l2 - l3 + l1;
  }
}

// Symmetric degree-2N triangle cubature ("cubature rules for triangles",
// P:108-110 "integration order 10" at N = 5; reading A2').  Orbit structure and
// 15-digit starting values from Dunavant (1985), Tables for degrees 2-10;
// the rule is the Newton root of the orthonormal moment equations
//   sum_i w_i psi_k(r_i, s_i) = int_T psi_k = sqrt(2) delta_k0,  deg psi_k <= 2N,
// with the analytic Jacobian through the Dubiner gradients.  Point order:
// orbits in table order; a point is a permutation of the orbit's barycentric
// triple t = (a, b, c) (S21: b = c = (1-a)/2; S111: c = 1-a-b), barycentric
// l_k = t[perm[k]], (r, s) = l0 (-1,-1) + l1 (1,-1) + l2 (-1,1).
struct SymOrbit {
  int npts;  // 1, 3 or 6
  double w, a, b;
};

bool dunavant_start(int N, std::vector<SymOrbit> &orb) {
  static const SymOrbit d2[] = {{3, 1.0 / 3.0, 2.0 / 3.0, 0.0}};
  static const SymOrbit d4[] = {{3, 0.223381589678011, 0.108103018168070, 0.0},
                                {3, 0.109951743655322, 0.816847572980459, 0.0}};
  static const SymOrbit d6[] = {{3, 0.116786275726379, 0.501426509658179, 0.0},
                                {3, 0.050844906370207, 0.873821971016996, 0.0},
                                {6, 0.082851075618374, 0.053145049844817, 0.310352451033784}};
  static const SymOrbit d8[] = {{1, 0.144315607677787, 0.0, 0.0},
                                {3, 0.095091634267285, 0.081414823414554, 0.0},
                                {3, 0.103217370534718, 0.658861384496480, 0.0},
                                {3, 0.032458497623198, 0.898905543365938, 0.0},
                                {6, 0.027230314174435, 0.008394777409958, 0.263112829634638}};
  static const SymOrbit d10[] = {{1, 0.090817990382754, 0.0, 0.0},
                                 {3, 0.036725957756467, 0.028844733232685, 0.0},
                                 {3, 0.045321059435528, 0.781036849029926, 0.0},
                                 {6, 0.072757916845420, 0.141707219414880, 0.307939838764121},
                                 {6, 0.028327242531057, 0.025003534762686, 0.246672560639903},
                                 {6, 0.009421666963733, 0.009540815400299, 0.066803251012200}};
  const SymOrbit *t = nullptr;
  size_t n = 0;
  switch (N) {
    case 1: t = d2, n = 1; break;
    case 2: t = d4, n = 2; break;
    case 3: t = d6, n = 3; break;
    case 4: t = d8, n = 5; break;
    case 5: t = d10, n = 6; break;
    default: return false;
  }
  orb.assign(t, t + n);
  return true;
}

// perm tables: barycentric slot k takes orbit coordinate perm[k] (0 = a, 1 = b, 2 = c)
const int kPerm3[3][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}};
const int kPerm6[6][3] = {{0, 1, 2}, {1, 2, 0}, {2, 0, 1}, {1, 0, 2}, {2, 1, 0}, {0, 2, 1}};

// Points, weights and d(r,s)/d(a,b) of every point of the orbits.
void expand_orbits(const std::vector<SymOrbit> &orb, std::vector<double> &r, std::vector<double> &s,
                   std::vector<double> &w, std::vector<double> &drda, std::vector<double> &dsda,
                   std::vector<double> &drdb, std::vector<double> &dsdb) {
  r.clear(), s.clear(), w.clear(), drda.clear(), dsda.clear(), drdb.clear(), dsdb.clear();
  const double vr[3] = {-1.0, 1.0, -1.0}, vs[3] = {-1.0, -1.0, 1.0};
  for (const SymOrbit &o : orb) {
    for (int p = 0; p < o.npts; p++) {
      double l[3], la[3], lb[3];
      for (int k = 0; k < 3; k++) {
        int c = o.npts == 1 ? -1 : (o.npts == 3 ? kPerm3[p][k] : kPerm6[p][k]);
        if (c < 0) {
          l[k] = 1.0 / 3.0, la[k] = 0.0, lb[k] = 0.0;
        } else if (o.npts == 3) {
          l[k] = c == 0 ? o.a : 0.5 * (1.0 - o.a);
          la[k] = c == 0 ? 1.0 : -0.5;
          lb[k] = 0.0;
        } else {
          l[k] = c == 0 ? o.a : (c == 1 ? o.b : 1.0 - o.a - o.b);
          la[k] = c == 0 ? 1.0 : (c == 1 ? 0.0 : -1.0);
          lb[k] = c == 1 ? 1.0 : (c == 0 ? 0.0 : -1.0);
        }
      }
      double rr = 0, ss = 0, ra = 0, sa = 0, rb = 0, sb = 0;
      for (int k = 0; k < 3; k++) {
        rr += l[k] * vr[k], ss += l[k] * vs[k];
        ra += la[k] * vr[k], sa += la[k] * vs[k];
        rb += lb[k] * vr[k], sb += lb[k] * vs[k];
      }
      r.push_back(rr), s.push_back(ss), w.push_back(2.0 * o.w);
      drda.push_back(ra), dsda.push_back(sa), drdb.push_back(rb), dsdb.push_back(sb);
    }
  }
}

bool symmetric_cubature(int N, std::vector<double> &rc, std::vector<double> &sc, std::vector<double> &wc) {
  std::vector<SymOrbit> orb;
  if (!dunavant_start(N, orb)) return false;
  const int deg = 2 * N, nmom = (deg + 1) * (deg + 2) / 2;
  int nunk = 0;
  for (const SymOrbit &o : orb) nunk += o.npts == 1 ? 1 : (o.npts == 3 ? 2 : 3);
  std::vector<double> r, s, w, ra, sa, rb, sb;
  for (int it = 0; it < 8; it++) {
    expand_orbits(orb, r, s, w, ra, sa, rb, sb);
    const int np = (int)w.size();
    DMat F = vandermonde(deg, r, s, 0), Fr = vandermonde(deg, r, s, 1), Fs = vandermonde(deg, r, s, 2);
    DMat J(nmom, nunk);
    std::vector<double> res(nmom, 0.0);
    for (int k = 0; k < nmom; k++) res[k] = k == 0 ? -std::sqrt(2.0) : 0.0;
    int p0 = 0, u = 0;
    for (const SymOrbit &o : orb) {
      for (int p = p0; p < p0 + o.npts; p++)
        for (int k = 0; k < nmom; k++) {
          res[k] += w[p] * F(p, k);
          J(k, u) += 2.0 * F(p, k);  // d/d(table weight); point weight = 2 w
          if (o.npts >= 3) J(k, u + 1) += w[p] * (Fr(p, k) * ra[p] + Fs(p, k) * sa[p]);
          if (o.npts == 6) J(k, u + 2) += w[p] * (Fr(p, k) * rb[p] + Fs(p, k) * sb[p]);
        }
      p0 += o.npts;
      u += o.npts == 1 ? 1 : (o.npts == 3 ? 2 : 3);
    }
    (void)np;
    // least-squares step: (J^T J) d = J^T res
    DMat Jt = transpose(J), JtJ = mul(Jt, J), JtJinv;
    if (!invert(JtJ, JtJinv)) return false;
    std::vector<double> g(nunk, 0.0), d(nunk, 0.0);
    for (int i = 0; i < nunk; i++)
      for (int k = 0; k < nmom; k++) g[i] += Jt(i, k) * res[k];
    for (int i = 0; i < nunk; i++)
      for (int j = 0; j < nunk; j++) d[i] += JtJinv(i, j) * g[j];
    u = 0;
    for (SymOrbit &o : orb) {
      o.w -= d[u++];
      if (o.npts >= 3) o.a -= d[u++];
      if (o.npts == 6) o.b -= d[u++];
    }
  }
  expand_orbits(orb, r, s, w, ra, sa, rb, sb);
  DMat F = vandermonde(deg, r, s, 0);
  double worst = 0.0;
  for (int k = 0; k < nmom; k++) {
    double acc = k == 0 ? -std::sqrt(2.0) : 0.0;
    for (size_t p = 0; p < w.size(); p++) acc += w[p] * F((int)p, k);
    worst = std::max(worst, std::fabs(acc));
  }
  if (!(worst < 1e-14)) return false;
  rc = r, sc = s, wc = w;
  return true;
}

}  // namespace

bool build_refops(int N, RefOps &o, std::string *err) {
  if (N < 1 || N > 8) {
    if (err) *err = "order out of range";
    return false;
  }
  o.N = N;
  o.Np = (N + 1) * (N + 2) / 2;
  o.Nfp = N + 1;
  o.Ng = N + 1;
  const int q = N + 1, Np = o.Np;
  nodes2d(N, o.r, o.s);
  o.V = vandermonde(N, o.r, o.s, 0);
  if (!invert(o.V, o.Vinv)) {
    if (err) *err = "singular Vandermonde";
    return false;
  }
  o.Dr = mul(vandermonde(N, o.r, o.s, 1), o.Vinv);
  o.Ds = mul(vandermonde(N, o.r, o.s, 2), o.Vinv);
  DMat MrefInv = mul(o.V, transpose(o.V));  // (V V^T) = Mref^{-1} for an orthonormal basis
  invert(MrefInv, o.Mref);

  // cubature (A2'): symmetric degree 2N for N <= 5, else collapsed
  // Gauss-Legendre (a) x Gauss-Jacobi(1,0) (b), r = (1+a)(1-b)/2 - 1, s = b
  o.rc.clear();
  o.sc.clear();
  o.wc.clear();
  if (N <= 5) {
    if (!symmetric_cubature(N, o.rc, o.sc, o.wc)) {
      if (err) *err = "symmetric cubature did not converge";
      return false;
    }
  } else {
    std::vector<double> xa, wa, xb, wb;
    gauss_rule(q, 0.0, 0.0, xa, wa);
    gauss_rule(q, 1.0, 0.0, xb, wb);
    for (int jb = 0; jb < q; jb++)
      for (int ia = 0; ia < q; ia++) {
        o.rc.push_back(0.5 * (1.0 + xa[ia]) * (1.0 - xb[jb]) - 1.0);
        o.sc.push_back(xb[jb]);
        o.wc.push_back(0.5 * wa[ia] * wb[jb]);
      }
  }
  o.Nc = (int)o.wc.size();
  gauss_rule(o.Ng, 0.0, 0.0, o.tg, o.wg);

  std::vector<double> rg, sg;
  const double vr[3] = {-1.0, 1.0, -1.0}, vs[3] = {-1.0, -1.0, 1.0};
  for (int f = 0; f < 3; f++)
    for (int j = 0; j < o.Ng; j++) {
      double t = o.tg[j];
      rg.push_back(0.5 * (1.0 - t) * vr[f] + 0.5 * (1.0 + t) * vr[(f + 1) % 3]);
      sg.push_back(0.5 * (1.0 - t) * vs[f] + 0.5 * (1.0 + t) * vs[(f + 1) % 3]);
    }

  o.Ic = mul(vandermonde(N, o.rc, o.sc, 0), o.Vinv);
  o.IcDr = mul(o.Ic, o.Dr);
  o.IcDs = mul(o.Ic, o.Ds);
  o.Ig = mul(vandermonde(N, rg, sg, 0), o.Vinv);

  DMat IcW(o.Nc, Np), IcDrW(o.Nc, Np), IcDsW(o.Nc, Np), IgW(3 * o.Ng, Np);
  for (int c = 0; c < o.Nc; c++)
    for (int i = 0; i < Np; i++) {
      IcW(c, i) = o.wc[c] * o.Ic(c, i);
      IcDrW(c, i) = o.wc[c] * o.IcDr(c, i);
      IcDsW(c, i) = o.wc[c] * o.IcDs(c, i);
    }
  for (int g = 0; g < 3 * o.Ng; g++)
    for (int i = 0; i < Np; i++) IgW(g, i) = o.wg[g % o.Ng] * o.Ig(g, i);
  o.P = mul(MrefInv, transpose(IcW));
  o.Pr = mul(MrefInv, transpose(IcDrW));
  o.Ps = mul(MrefInv, transpose(IcDsW));
  o.Lg = mul(MrefInv, transpose(IgW));

  o.wmean.assign(Np, 0.0);
  for (int c = 0; c < o.Nc; c++)
    for (int i = 0; i < Np; i++) o.wmean[i] += o.wc[c] * o.Ic(c, i);

  // face nodes in counter-clockwise order along each face
  o.Fmask.assign(3 * o.Nfp, -1);
  const double tol = 1e-10;
  for (int f = 0; f < 3; f++) {
    std::vector<std::pair<double, int>> fn;
    for (int i = 0; i < Np; i++) {
      double r = o.r[i], s = o.s[i];
      if (f == 0 && std::fabs(s + 1.0) < tol) fn.push_back({r, i});
      if (f == 1 && std::fabs(r + s) < tol) fn.push_back({s, i});
      if (f == 2 && std::fabs(r + 1.0) < tol) fn.push_back({-s, i});
    }
    if ((int)fn.size() != o.Nfp) {
      if (err) *err = "face node count mismatch";
      return false;
    }
    std::sort(fn.begin(), fn.end());
    for (int k = 0; k < o.Nfp; k++) o.Fmask[f * o.Nfp + k] = fn[k].second;
  }
  // 1D interpolation face nodes -> Gauss points; all three faces carry the
  // same (symmetric) node distribution in their own parameter t in [-1,1].
  std::vector<double> tn(o.Nfp);
  for (int k = 0; k < o.Nfp; k++) tn[k] = o.r[o.Fmask[k]];
  for (int f = 1; f < 3; f++)
    for (int k = 0; k < o.Nfp; k++) {
      int i = o.Fmask[f * o.Nfp + k];
      double t = (f == 1) ? o.s[i] : -o.s[i];
      if (std::fabs(t - tn[k]) > 1e-13 || std::fabs(tn[k] + tn[o.Nfp - 1 - k]) > 1e-13) {
        if (err) *err = "face nodes not symmetric";
        return false;
      }
    }
  o.Ig1 = DMat(o.Ng, o.Nfp);
  for (int j = 0; j < o.Ng; j++)
    for (int k = 0; k < o.Nfp; k++) {
      double l = 1.0;
      for (int m = 0; m < o.Nfp; m++)
        if (m != k) l *= (o.tg[j] - tn[m]) / (tn[k] - tn[m]);
      o.Ig1(j, k) = l;
    }

  // P1 projection: Dubiner modes (0,0)->0, (0,1)->1, (1,0)->N+1; vertex values
  const int modes[3] = {0, 1, N + 1};
  std::vector<double> vrr = {-1.0, 1.0, -1.0}, vss = {-1.0, -1.0, 1.0};
  DMat Vv = vandermonde(N, vrr, vss, 0);
  o.Pv = DMat(3, Np);
  for (int v = 0; v < 3; v++)
    for (int i = 0; i < Np; i++) {
      double acc = 0.0;
      for (int m : modes) acc += Vv(v, m) * o.Vinv(m, i);
      o.Pv(v, i) = acc;
    }
  return true;
}

}  // namespace swe
