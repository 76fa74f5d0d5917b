// oracle/refel.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Reference-element construction, P:81 ("Lagrange polynomials with Warp &
// Blend interpolation nodes ... cubature rules for triangles ... Gauss
// quadrature rules"), P:651 (P, Pr, Ps "projection matrices that are pre
// multiplied with cubature integration weights"), P:691 (lift L^g).
// Readings: SURVEY §8(c) O1-O3, A2' (symmetric degree-2N cubature for N <= 5,
// collapsed Gauss-Jacobi above; Ng = N+1 Gauss points per edge), A8 (HW alpha table).
//
// Everything here is computed in long double (x87 80-bit) and rounded to
// double once at the end: the tensor-Legendre basis L_p(r)L_q(s) is
// ill-conditioned on the triangle and extended precision keeps the final
// operators accurate to double round-off.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "oracle.hpp"

namespace orc {

typedef long double LD;

template <class T>
struct TMat {
  int rows = 0, cols = 0;
  std::vector<T> v;
  TMat() {}
  TMat(int r, int c) : rows(r), cols(c), v((size_t)r * (size_t)c, T(0)) {}
  T &operator()(int i, int j) { return v[(size_t)i * cols + j]; }
  T operator()(int i, int j) const { return v[(size_t)i * cols + j]; }
};
typedef TMat<LD> LMat;

template <class M>
static M t_matmul(const M &A, const M &B) {
  M C(A.rows, B.cols);
  for (int i = 0; i < A.rows; i++)
    for (int j = 0; j < B.cols; j++) {
      auto acc = A(0, 0) * 0;
      for (int k = 0; k < A.cols; k++) acc += A(i, k) * B(k, j);
      C(i, j) = acc;
    }
  return C;
}

// Gauss-Jordan elimination with partial pivoting on [A | I].
template <class M>
static M t_inverse(const M &A) {
  int n = A.rows;
  M a = A, inv(n, n);
  for (int i = 0; i < n; i++) inv(i, i) = 1;
  for (int col = 0; col < n; col++) {
    int piv = col;
    for (int i = col + 1; i < n; i++)
      if (std::fabs(a(i, col)) > std::fabs(a(piv, col))) piv = i;
    if (a(piv, col) == 0) throw std::runtime_error("singular matrix");
    for (int j = 0; j < n; j++) {
      std::swap(a(col, j), a(piv, j));
      std::swap(inv(col, j), inv(piv, j));
    }
    auto d = a(col, col);
    for (int j = 0; j < n; j++) {
      a(col, j) /= d;
      inv(col, j) /= d;
    }
    for (int i = 0; i < n; i++) {
      if (i == col) continue;
      auto f = a(i, col);
      if (f == 0) continue;
      for (int j = 0; j < n; j++) {
        a(i, j) -= f * a(col, j);
        inv(i, j) -= f * inv(col, j);
      }
    }
  }
  return inv;
}

Mat matmul(const Mat &A, const Mat &B) {
  Mat C(A.rows, B.cols);
  for (int i = 0; i < A.rows; i++)
    for (int j = 0; j < B.cols; j++) {
      double acc = 0.0;
      for (int k = 0; k < A.cols; k++) acc += A(i, k) * B(k, j);
      C(i, j) = acc;
    }
  return C;
}
Mat transpose(const Mat &A) {
  Mat T(A.cols, A.rows);
  for (int i = 0; i < A.rows; i++)
    for (int j = 0; j < A.cols; j++) T(j, i) = A(i, j);
  return T;
}
Mat inverse(const Mat &A) {
  LMat L(A.rows, A.cols);
  for (size_t i = 0; i < A.v.size(); i++) L.v[i] = A.v[i];
  LMat I = t_inverse(L);
  Mat M(A.rows, A.cols);
  for (size_t i = 0; i < M.v.size(); i++) M.v[i] = (double)I.v[i];
  return M;
}
static Mat to_double(const LMat &A) {
  Mat M(A.rows, A.cols);
  for (size_t i = 0; i < A.v.size(); i++) M.v[i] = (double)A.v[i];
  return M;
}
static std::vector<double> to_double(const std::vector<LD> &a) { return std::vector<double>(a.begin(), a.end()); }

// ---------------------------------------------------------------- 1D polynomials
// Bonnet recurrence (n+1) L_{n+1} = (2n+1) x L_n - n L_{n-1}.
template <class T>
static T t_legendre(int n, T x) {
  if (n == 0) return T(1);
  T a = 1, b = x;
  for (int k = 1; k < n; k++) {
    T c = ((T(2) * k + 1) * x * b - T(k) * a) / T(k + 1);
    a = b;
    b = c;
  }
  return b;
}
// L'_{n+1} = L'_{n-1} + (2n+1) L_n.
template <class T>
static T t_legendre_deriv(int n, T x) {
  if (n == 0) return T(0);
  T dm1 = 0, d = 1;  // L'_0, L'_1
  for (int k = 1; k < n; k++) {
    T dn = dm1 + (T(2) * k + 1) * t_legendre<T>(k, x);
    dm1 = d;
    d = dn;
  }
  return d;
}
double legendre(int n, double x) { return t_legendre<double>(n, x); }
double legendre_deriv(int n, double x) { return t_legendre_deriv<double>(n, x); }

static const LD kPiL = 3.141592653589793238462643383279502884L;

template <class T>
static void sort_rule(std::vector<T> &x, std::vector<T> &w) {
  std::vector<size_t> idx(x.size());
  for (size_t k = 0; k < idx.size(); k++) idx[k] = k;
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return x[a] < x[b]; });
  std::vector<T> xs(x.size()), ws(w.size());
  for (size_t k = 0; k < idx.size(); k++) {
    xs[k] = x[idx[k]];
    ws[k] = w[idx[k]];
  }
  x = xs;
  w = ws;
}

// Gauss-Legendre: Newton on L_q from the classical cosine guesses;
// w = 2 / ((1-x^2) L_q'(x)^2).
static void ld_gauss_legendre(int q, std::vector<LD> &x, std::vector<LD> &w) {
  x.assign(q, 0);
  w.assign(q, 0);
  for (int k = 0; k < q; k++) {
    LD xk = -std::cos(kPiL * (k + 0.75L) / (q + 0.5L));
    for (int it = 0; it < 100; it++) {
      LD dx = t_legendre<LD>(q, xk) / t_legendre_deriv<LD>(q, xk);
      xk -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
    LD dp = t_legendre_deriv<LD>(q, xk);
    x[k] = xk;
    w[k] = 2 / ((1 - xk * xk) * dp * dp);
  }
  sort_rule(x, w);
}

// Unnormalised Jacobi P_n^{(a,b)}(x) by the standard three-term recurrence.
static LD jacobi(int n, LD a, LD b, LD x) {
  if (n == 0) return 1;
  LD p0 = 1, p1 = 0.5L * ((a + b + 2) * x + (a - b));
  for (int k = 2; k <= n; k++) {
    LD c = 2.0L * k + a + b;
    LD a1 = 2.0L * k * (k + a + b) * (c - 2);
    LD a2 = (c - 1) * (a * a - b * b);
    LD a3 = (c - 2) * (c - 1) * c;
    LD a4 = 2.0L * (k + a - 1) * (k + b - 1) * c;
    LD p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}
// d/dx P_n^{(a,b)} = (n+a+b+1)/2 P_{n-1}^{(a+1,b+1)}
static LD jacobi_deriv(int n, LD a, LD b, LD x) {
  if (n == 0) return 0;
  return 0.5L * (n + a + b + 1) * jacobi(n - 1, a + 1, b + 1, x);
}

// Gauss-Jacobi rule for weight (1-x)^1 (1+x)^0: roots of P_q^{(1,0)} by Newton
// with deflation; w_i = 4 / ((1-x_i^2) P_q'(x_i)^2).
static void ld_gauss_jacobi10(int q, std::vector<LD> &x, std::vector<LD> &w) {
  x.assign(q, 0);
  w.assign(q, 0);
  for (int k = 0; k < q; k++) {
    LD xk = -std::cos((2.0L * k + 1) * kPiL / (2.0L * q));
    if (k > 0) xk = 0.5L * (xk + x[k - 1]);
    for (int it = 0; it < 200; it++) {
      LD p = jacobi(q, 1, 0, xk), dp = jacobi_deriv(q, 1, 0, xk);
      LD defl = 0;
      for (int j = 0; j < k; j++) defl += 1 / (xk - x[j]);
      LD dx = p / (dp - p * defl);
      xk -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
    x[k] = xk;
    LD dp = jacobi_deriv(q, 1, 0, xk);
    w[k] = 4 / ((1 - xk * xk) * dp * dp);
  }
  sort_rule(x, w);
}

// Legendre-Gauss-Lobatto points: roots of L_{N+1} - L_{N-1} (= c (x^2-1) L_N'),
// Newton from Chebyshev-Gauss-Lobatto guesses; derivative (2N+1) L_N.
static void ld_lobatto(int N, std::vector<LD> &x) {
  x.assign(N + 1, 0);
  for (int i = 0; i <= N; i++) {
    LD xi = -std::cos(kPiL * i / N);
    if (i > 0 && i < N) {
      for (int it = 0; it < 200; it++) {
        LD f = t_legendre<LD>(N + 1, xi) - t_legendre<LD>(N - 1, xi);
        LD df = (2.0L * N + 1) * t_legendre<LD>(N, xi);
        LD dx = f / df;
        xi -= dx;
        if (std::fabs(dx) < 1e-19L) break;
      }
    }
    x[i] = xi;
  }
  x[0] = -1;
  x[N] = 1;
}

void gauss_legendre(int q, std::vector<double> &x, std::vector<double> &w) {
  std::vector<LD> X, W;
  ld_gauss_legendre(q, X, W);
  x = to_double(X);
  w = to_double(W);
}
void gauss_jacobi10(int q, std::vector<double> &x, std::vector<double> &w) {
  std::vector<LD> X, W;
  ld_gauss_jacobi10(q, X, W);
  x = to_double(X);
  w = to_double(W);
}
void lobatto_points(int N, std::vector<double> &x) {
  std::vector<LD> X;
  ld_lobatto(N, X);
  x = to_double(X);
}

// ---------------------------------------------------------------- Warp & Blend nodes
// P:81 cites hesthaven2008nodal. Equilateral-triangle construction: equispaced
// barycentric lattice, warped along each edge by the 1D map equispaced -> LGL,
// warp(r) = sum_i (x_LGL,i - x_eq,i) l_i^eq(r) / (1 - r^2) with l^eq the
// equispaced Lagrange polynomials, blended with 4 L_a L_b (1 + (alpha L_c)^2),
// then mapped to (r,s).  Node order: rows of constant s upward, r increasing.
static LD warp_factor(int N, LD rout) {
  std::vector<LD> lgl;
  ld_lobatto(N, lgl);
  LD w = 0;
  for (int i = 0; i <= N; i++) {
    LD req_i = -1 + 2.0L * i / N;
    LD li = 1;
    for (int j = 0; j <= N; j++) {
      if (j == i) continue;
      LD req_j = -1 + 2.0L * j / N;
      li *= (rout - req_j) / (req_i - req_j);
    }
    w += (lgl[i] - req_i) * li;
  }
  if (std::fabs(rout) < 1 - 1e-10L) return w / (1 - rout * rout);
  return 0;
}

static void ld_nodes(int N, std::vector<LD> &r, std::vector<LD> &s) {
  static const LD alpopt[15] = {0.0000L, 0.0000L, 1.4152L, 0.1001L, 0.2751L, 0.9800L, 1.0999L, 1.2832L,
                                1.3648L, 1.4773L, 1.4959L, 1.5743L, 1.5770L, 1.6223L, 1.6258L};
  LD alpha = (N < 16) ? alpopt[N - 1] : 5.0L / 3.0L;
  int Np = (N + 1) * (N + 2) / 2;
  r.assign(Np, 0);
  s.assign(Np, 0);
  const LD sq3 = std::sqrt((LD)3);
  int sk = 0;
  for (int n = 0; n <= N; n++) {
    for (int m = 0; m <= N - n; m++) {
      LD L1 = (LD)n / N, L3 = (LD)m / N, L2 = 1 - L1 - L3;
      LD x = -L2 + L3, y = (-L2 - L3 + 2 * L1) / sq3;
      LD b1 = 4 * L2 * L3, b2 = 4 * L1 * L3, b3 = 4 * L1 * L2;
      LD w1 = b1 * warp_factor(N, L3 - L2) * (1 + (alpha * L1) * (alpha * L1));
      LD w2 = b2 * warp_factor(N, L1 - L3) * (1 + (alpha * L2) * (alpha * L2));
      LD w3 = b3 * warp_factor(N, L2 - L1) * (1 + (alpha * L3) * (alpha * L3));
      x += w1 + std::cos(2 * kPiL / 3) * w2 + std::cos(4 * kPiL / 3) * w3;
      y += std::sin(2 * kPiL / 3) * w2 + std::sin(4 * kPiL / 3) * w3;
      // equilateral (x,y) -> reference (r,s) through barycentric coordinates
      LD l1 = (sq3 * y + 1) / 3;
      LD l2 = (-3 * x - sq3 * y + 2) / 6;
      LD l3 = (3 * x - sq3 * y + 2) / 6;
      r[sk] = -l2 + l3 - l1;
      s[sk] = -l2 - l3 + l1;
      sk++;
    }
  }
}

void warp_blend_nodes(int N, std::vector<double> &r, std::vector<double> &s) {
  std::vector<LD> R, S;
  ld_nodes(N, R, S);
  r = to_double(R);
  s = to_double(S);
}

// ---------------------------------------------------------------- basis L_p(r) L_q(s), p+q <= N
// which: 0 value, 1 d/dr, 2 d/ds
static LMat vandermonde(int N, const std::vector<LD> &r, const std::vector<LD> &s, int which) {
  int Np = (N + 1) * (N + 2) / 2;
  LMat V((int)r.size(), Np);
  for (size_t i = 0; i < r.size(); i++) {
    int k = 0;
    for (int p = 0; p <= N; p++)
      for (int q = 0; q <= N - p; q++) {
        LD a = which == 1 ? t_legendre_deriv<LD>(p, r[i]) : t_legendre<LD>(p, r[i]);
        LD b = which == 2 ? t_legendre_deriv<LD>(q, s[i]) : t_legendre<LD>(q, s[i]);
        V((int)i, k++) = a * b;
      }
  }
  return V;
}

Mat interp_matrix(const RefElement &re, const std::vector<double> &r, const std::vector<double> &s) {
  std::vector<LD> R(r.begin(), r.end()), S(s.begin(), s.end()), Rn, Sn;
  ld_nodes(re.N, Rn, Sn);
  LMat Vinv = t_inverse(vandermonde(re.N, Rn, Sn, 0));
  return to_double(t_matmul(vandermonde(re.N, R, S, 0), Vinv));
}

// ---------------------------------------------------------------- cubature
// P:81 "The volume integrals are computed using cubature rules for triangles
// [Cools]"; P:108-110 (Fig. 1): polynomial order 5 with "integration order 10",
// i.e. a symmetric rule of degree 2N.  Reading A2': for N <= 5 the
// fully symmetric rules of Dunavant (1985, IJNME 21:1129, Tables; also listed
// in Cools' encyclopedia) -- 3, 6, 12, 16, 25 points for degrees 2, 4, 6, 8, 10.
// The tabulated 15-digit values are only the starting point: the rule is the
// root of its moment equations, refined here in long double by Gauss-Newton on
// "sum_i w_i r_i^a s_i^b = int_T r^a s^b for all a+b <= 2N".
// Orbits (barycentric (l1,l2,l3) -> (r,s) = l1 v0 + l2 v1 + l3 v2):
//   S3  : centroid;
//   S21 : (a,b,b),(b,a,b),(b,b,a) with b = (1-a)/2;
//   S111: (a,b,c),(b,c,a),(c,a,b),(b,a,c),(c,b,a),(a,c,b) with c = 1-a-b.
// Points are listed orbit by orbit in table order, weights scaled to area 2.
struct Orbit {
  int type;           // 1 = S3, 3 = S21, 6 = S111
  LD w, a, b;         // weight (sum over all points = 1 in the table) and coordinates
};

static std::vector<Orbit> dunavant_table(int N) {
  switch (N) {
    case 1: return {{3, 1.0L / 3.0L, 2.0L / 3.0L, 0}};
    case 2: return {{3, 0.223381589678011L, 0.108103018168070L, 0},
                    {3, 0.109951743655322L, 0.816847572980459L, 0}};
    case 3: return {{3, 0.116786275726379L, 0.501426509658179L, 0},
                    {3, 0.050844906370207L, 0.873821971016996L, 0},
                    {6, 0.082851075618374L, 0.053145049844817L, 0.310352451033784L}};
    case 4: return {{1, 0.144315607677787L, 0, 0},
                    {3, 0.095091634267285L, 0.081414823414554L, 0},
                    {3, 0.103217370534718L, 0.658861384496480L, 0},
                    {3, 0.032458497623198L, 0.898905543365938L, 0},
                    {6, 0.027230314174435L, 0.008394777409958L, 0.263112829634638L}};
    case 5: return {{1, 0.090817990382754L, 0, 0},
                    {3, 0.036725957756467L, 0.028844733232685L, 0},
                    {3, 0.045321059435528L, 0.781036849029926L, 0},
                    {6, 0.072757916845420L, 0.141707219414880L, 0.307939838764121L},
                    {6, 0.028327242531057L, 0.025003534762686L, 0.246672560639903L},
                    {6, 0.009421666963733L, 0.009540815400299L, 0.066803251012200L}};
    default: return {};
  }
}

static void orbit_points(const std::vector<Orbit> &orb, std::vector<LD> &r, std::vector<LD> &s, std::vector<LD> &w) {
  r.clear();
  s.clear();
  w.clear();
  auto push = [&](LD l1, LD l2, LD l3, LD wt) {
    r.push_back(-l1 + l2 - l3);
    s.push_back(-l1 - l2 + l3);
    w.push_back(2 * wt);
  };
  for (const Orbit &o : orb) {
    if (o.type == 1) {
      push(1.0L / 3, 1.0L / 3, 1.0L / 3, o.w);
    } else if (o.type == 3) {
      LD a = o.a, b = (1 - o.a) / 2;
      push(a, b, b, o.w);
      push(b, a, b, o.w);
      push(b, b, a, o.w);
    } else {
      LD a = o.a, b = o.b, c = 1 - o.a - o.b;
      push(a, b, c, o.w);
      push(b, c, a, o.w);
      push(c, a, b, o.w);
      push(b, a, c, o.w);
      push(c, b, a, o.w);
      push(a, c, b, o.w);
    }
  }
}

// int_T r^a s^b over T = {r,s >= -1, r+s <= 0}: with r = 2x-1, s = 2y-1 on the
// unit simplex, int x^i y^j = i! j! / (i+j+2)!.
static LD tri_monomial(int a, int b) {
  auto fact = [](int n) { LD f = 1; for (int k = 2; k <= n; k++) f *= k; return f; };
  auto binom = [&](int n, int k) { return fact(n) / (fact(k) * fact(n - k)); };
  LD acc = 0;
  for (int i = 0; i <= a; i++)
    for (int j = 0; j <= b; j++) {
      LD sign = ((a - i + b - j) % 2) ? -1 : 1;
      acc += sign * binom(a, i) * binom(b, j) * std::pow(2.0L, i + j) * fact(i) * fact(j) / fact(i + j + 2);
    }
  return 4 * acc;
}

static bool ld_symmetric_rule(int N, std::vector<LD> &rc, std::vector<LD> &sc, std::vector<LD> &wc) {
  std::vector<Orbit> orb = dunavant_table(N);
  if (orb.empty()) return false;
  const int deg = 2 * N;
  // unknown vector theta: per orbit w, then a (S21, S111), then b (S111)
  auto pack = [&](const std::vector<Orbit> &o) {
    std::vector<LD> t;
    for (const Orbit &x : o) {
      t.push_back(x.w);
      if (x.type >= 3) t.push_back(x.a);
      if (x.type == 6) t.push_back(x.b);
    }
    return t;
  };
  auto unpack = [&](const std::vector<LD> &t) {
    std::vector<Orbit> o = orb;
    size_t k = 0;
    for (Orbit &x : o) {
      x.w = t[k++];
      if (x.type >= 3) x.a = t[k++];
      if (x.type == 6) x.b = t[k++];
    }
    return o;
  };
  std::vector<std::pair<int, int>> mono;
  std::vector<LD> exact;
  for (int a = 0; a <= deg; a++)
    for (int b = 0; a + b <= deg; b++) {
      mono.push_back({a, b});
      exact.push_back(tri_monomial(a, b));
    }
  auto residual = [&](const std::vector<LD> &t) {
    std::vector<LD> r, s, w, res(mono.size());
    orbit_points(unpack(t), r, s, w);
    for (size_t m = 0; m < mono.size(); m++) {
      LD acc = 0;
      for (size_t i = 0; i < w.size(); i++)
        acc += w[i] * std::pow(r[i], (LD)mono[m].first) * std::pow(s[i], (LD)mono[m].second);
      res[m] = acc - exact[m];
    }
    return res;
  };
  std::vector<LD> theta = pack(orb);
  const int n = (int)theta.size(), m = (int)mono.size();
  for (int it = 0; it < 12; it++) {
    std::vector<LD> r0 = residual(theta);
    LMat J(m, n);
    for (int j = 0; j < n; j++) {  // central differences in long double
      const LD h = 1e-7L;
      std::vector<LD> tp = theta, tm = theta;
      tp[j] += h;
      tm[j] -= h;
      std::vector<LD> rp = residual(tp), rm = residual(tm);
      for (int i = 0; i < m; i++) J(i, j) = (rp[i] - rm[i]) / (2 * h);
    }
    LMat JtJ(n, n), Jtr(n, 1);
    for (int a = 0; a < n; a++) {
      for (int b = 0; b < n; b++) {
        LD acc = 0;
        for (int i = 0; i < m; i++) acc += J(i, a) * J(i, b);
        JtJ(a, b) = acc;
      }
      LD acc = 0;
      for (int i = 0; i < m; i++) acc += J(i, a) * r0[i];
      Jtr(a, 0) = acc;
    }
    LMat d = t_matmul(t_inverse(JtJ), Jtr);
    for (int j = 0; j < n; j++) theta[j] -= d(j, 0);
  }
  LD worst = 0;
  for (LD v : residual(theta)) worst = std::max(worst, std::fabs(v));
  if (!(worst < 1e-16L)) throw std::runtime_error("symmetric cubature: Newton did not converge");
  orbit_points(unpack(theta), rc, sc, wc);
  return true;
}

void build_refel(int N, RefElement &re) {
  re.N = N;
  re.Np = (N + 1) * (N + 2) / 2;
  re.Nfp = N + 1;
  re.Ng = N + 1;
  int q = N + 1, Np = re.Np;
  std::vector<LD> r, s;
  ld_nodes(N, r, s);
  re.r = to_double(r);
  re.s = to_double(s);

  LMat V = vandermonde(N, r, s, 0);
  LMat Vinv = t_inverse(V);
  LMat Dr = t_matmul(vandermonde(N, r, s, 1), Vinv);
  LMat Ds = t_matmul(vandermonde(N, r, s, 2), Vinv);
  re.V = to_double(V);
  re.Vinv = to_double(Vinv);
  re.Dr = to_double(Dr);
  re.Ds = to_double(Ds);

  // Volume cubature (reading A2'): the symmetric degree-2N rule for N <= 5;
  // above that (no tabulated rule here) the collapsed (Stroud) rule
  // r = (1+a)(1-b)/2 - 1, s = b, dr ds = (1-b)/2 da db, Gauss-Legendre in a,
  // Gauss-Jacobi(1,0) in b, exact to degree 2q-1 = 2N+1.
  std::vector<LD> rc, sc, wc;
  if (!ld_symmetric_rule(N, rc, sc, wc)) {
    std::vector<LD> xa, wa, xb, wb;
    ld_gauss_legendre(q, xa, wa);
    ld_gauss_jacobi10(q, xb, wb);
    for (int j = 0; j < q; j++)
      for (int i = 0; i < q; i++) {
        rc.push_back(0.5L * (1 + xa[i]) * (1 - xb[j]) - 1);
        sc.push_back(xb[j]);
        wc.push_back(0.5L * wa[i] * wb[j]);
      }
  }
  re.Ncub = (int)wc.size();
  re.rc = to_double(rc);
  re.sc = to_double(sc);
  re.wc = to_double(wc);

  // Edges: face f runs v_f -> v_{f+1}, v0=(-1,-1), v1=(1,-1), v2=(-1,1);
  // point at parameter t: v_f (1-t)/2 + v_{f+1} (1+t)/2.
  std::vector<LD> tg, wg, rg, sg;
  ld_gauss_legendre(re.Ng, tg, wg);
  re.tg = to_double(tg);
  re.wg = to_double(wg);
  const LD vr[3] = {-1, 1, -1}, vs[3] = {-1, -1, 1};
  for (int f = 0; f < 3; f++)
    for (int j = 0; j < re.Ng; j++) {
      LD t = tg[j];
      int a = f, b = (f + 1) % 3;
      rg.push_back(0.5L * (1 - t) * vr[a] + 0.5L * (1 + t) * vr[b]);
      sg.push_back(0.5L * (1 - t) * vs[a] + 0.5L * (1 + t) * vs[b]);
    }
  re.rg = to_double(rg);
  re.sg = to_double(sg);

  LMat Ic = t_matmul(vandermonde(N, rc, sc, 0), Vinv);
  LMat Ig = t_matmul(vandermonde(N, rg, sg, 0), Vinv);
  re.Ic = to_double(Ic);
  re.Ig = to_double(Ig);

  // Mref_ij = int l_i l_j = sum_c w_c Ic_ci Ic_cj (exact: degree 2N <= the rule's strength)
  LMat Mref(Np, Np);
  for (int i = 0; i < Np; i++)
    for (int j = 0; j < Np; j++) {
      LD acc = 0;
      for (int c = 0; c < re.Ncub; c++) acc += wc[c] * Ic(c, i) * Ic(c, j);
      Mref(i, j) = acc;
    }
  re.Mref = to_double(Mref);
  LMat Minv = t_inverse(Mref);

  // P = M^-1 Ic^T W, Pr = M^-1 (Ic Dr)^T W, Ps = M^-1 (Ic Ds)^T W
  LMat IcDr = t_matmul(Ic, Dr), IcDs = t_matmul(Ic, Ds);
  LMat IcTW(Np, re.Ncub), IcDrTW(Np, re.Ncub), IcDsTW(Np, re.Ncub);
  for (int i = 0; i < Np; i++)
    for (int c = 0; c < re.Ncub; c++) {
      IcTW(i, c) = Ic(c, i) * wc[c];
      IcDrTW(i, c) = IcDr(c, i) * wc[c];
      IcDsTW(i, c) = IcDs(c, i) * wc[c];
    }
  re.P = to_double(t_matmul(Minv, IcTW));
  re.Pr = to_double(t_matmul(Minv, IcDrTW));
  re.Ps = to_double(t_matmul(Minv, IcDsTW));

  // L^g = M^-1 Ig^T W_g
  LMat IgTW(Np, 3 * re.Ng);
  for (int i = 0; i < Np; i++)
    for (int g = 0; g < 3 * re.Ng; g++) IgTW(i, g) = Ig(g, i) * wg[g % re.Ng];
  re.Lg = to_double(t_matmul(Minv, IgTW));

  re.wmean.assign(Np, 0.0);
  for (int i = 0; i < Np; i++) {
    LD acc = 0;
    for (int j = 0; j < Np; j++) acc += Mref(i, j);
    re.wmean[i] = (double)acc;
  }
}

}  // namespace orc
