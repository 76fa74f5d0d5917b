// oracle/mrab.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Multi-rate Adams-Bashforth, P:127 (level l steps with 2^{l-1} dt_min),
// P:130-147 (Alg. 1), P:174-191 (Alg. 2: limiters after every update).
// Reading A17: recursive slowest-first order
//   Advance(l, t) = { update level l from t to t + dt_l with R evaluated at t;
//                     if l > 1: Advance(l-1, t); Advance(l-1, t + dt_{l-1}) }
// with coarser neighbours read mid-step through the AB3 dense output, so that
// R(Q^{n+(nstep-s)/Nsteps(l)}) of Alg. 1 is evaluated at a time-consistent
// state.  Reading A18: per-level Euler -> AB2 -> AB3 start-up ramp.
#include <algorithm>
#include <cassert>
#include <cmath>

#include "oracle.hpp"

namespace orc {

// Adams-Bashforth weights with m history values ("3rd order
// Adams-Bashforth"; ramp A18).
void ab_coeffs(int m, double a[3]) {
  a[0] = a[1] = a[2] = 0.0;
  if (m <= 1) {
    a[0] = 1.0;
  } else if (m == 2) {
    a[0] = 1.5;
    a[1] = -0.5;
  } else {
    a[0] = 23.0 / 12.0;
    a[1] = -16.0 / 12.0;
    a[2] = 5.0 / 12.0;
  }
}

// Dense output: integral over [0, theta] of the Lagrange interpolant of the
// history R(0), R(-1), R(-2) (times in units of the level step):
//   l0 = (tau+1)(tau+2)/2, l1 = -tau(tau+2), l2 = tau(tau+1)/2
//   -> b0 = th^3/6 + 3th^2/4 + th, b1 = -th^3/3 - th^2, b2 = th^3/6 + th^2/4
// (m = 2: b0 = th + th^2/2, b1 = -th^2/2; m = 1: b0 = th).  b(1) = AB weights.
void dense_coeffs(int m, double th, double b[3]) {
  b[0] = b[1] = b[2] = 0.0;
  double t2 = th * th, t3 = t2 * th;
  if (m <= 1) {
    b[0] = th;
  } else if (m == 2) {
    b[0] = th + 0.5 * t2;
    b[1] = -0.5 * t2;
  } else {
    b[0] = t3 / 6.0 + 0.75 * t2 + th;
    b[1] = -t3 / 3.0 - t2;
    b[2] = t3 / 6.0 + 0.25 * t2;
  }
}

void Mrab::init(int K_, int ndof_, int L_, double dt_, const std::vector<int> &level_) {
  K = K_;
  ndof = ndof_;
  L = L_;
  dt = dt_;
  level = level_;
  elems.assign(L + 1, std::vector<int>());
  for (int e = 0; e < K; e++) elems[level[e]].push_back(e);
  Q.resize((size_t)K * ndof, 0.0);
  Qs.assign((size_t)K * ndof, 0.0);
  for (int s = 0; s < 3; s++) Rh[s].assign((size_t)K * ndof, 0.0);
  for (int l = 0; l < 17; l++) {
    kcount[l] = 0;
    tick_s[l] = 0;
    t_e[l] = 0;
  }
  tick = 0;
}

void Mrab::state_at(int n, long t, double *out) const {
  int c = level[n];
  const double *q = &Q[(size_t)n * ndof];
  if (coupling == 1 || t_e[c] == t) {  // latest committed (variant) / synchronised neighbour
    for (int i = 0; i < ndof; i++) out[i] = q[i];
    return;
  }
  // coarser neighbour in the middle of its step [tick_s, t_e)
  assert(tick_s[c] <= t && t < t_e[c]);
  const double *qs = &Qs[(size_t)n * ndof];
  if (t == tick_s[c]) {
    for (int i = 0; i < ndof; i++) out[i] = qs[i];
    return;
  }
  long step = t_e[c] - tick_s[c];
  double theta = (double)(t - tick_s[c]) / (double)step;
  int m = std::min(kcount[c], 3);
  double b[3];
  dense_coeffs(m, theta, b);
  double h = std::ldexp(dt, c - 1);
  for (int i = 0; i < ndof; i++) {
    double acc = 0.0;
    for (int s = 0; s < m; s++) {
      int slot = ((kcount[c] - 1 - s) % 3 + 3) % 3;
      acc += b[s] * Rh[slot][(size_t)n * ndof + i];
    }
    out[i] = qs[i] + h * acc;
  }
}

void Mrab::update_level(int l, long t) {
  const std::vector<int> &E = elems[l];
  std::vector<double> Rnew(E.size() * (size_t)ndof);
#pragma omp parallel for schedule(dynamic, 64)
  for (long idx = 0; idx < (long)E.size(); idx++) rhs(E[idx], t, &Rnew[(size_t)idx * ndof]);

  int k = kcount[l];
  int m = std::min(k + 1, 3);
  double a[3];
  ab_coeffs(m, a);
  double h = std::ldexp(dt, l - 1);
  for (size_t idx = 0; idx < E.size(); idx++) {
    int e = E[idx];
    size_t o = (size_t)e * ndof;
    for (int i = 0; i < ndof; i++) Rh[k % 3][o + i] = Rnew[idx * ndof + i];
    for (int i = 0; i < ndof; i++) {
      double acc = 0.0;
      for (int s = 0; s < m; s++) acc += a[s] * Rh[(k - s) % 3][o + i];
      Qs[o + i] = Q[o + i];
      Q[o + i] = Q[o + i] + h * acc;
    }
  }
  kcount[l] = k + 1;
  tick_s[l] = t;
  t_e[l] = t + (1L << (l - 1));
  if (post) post(l, E);
}

void Mrab::advance(int l, long t) {
  update_level(l, t);
  if (l > 1) {
    advance(l - 1, t);
    advance(l - 1, t + (1L << (l - 2)));
  }
}

void Mrab::macro_step() {
  if (coupling == 1) {  // Alg. 1 as printed: for l = L..1, for s = 0..Nsteps(l)-1
    for (int l = L; l >= 1; l--)
      for (long s = 0; s < (1L << (L - l)); s++) update_level(l, tick + s * (1L << (l - 1)));
  } else {
    advance(L, tick);
  }
  tick += 1L << (L - 1);
}

}  // namespace orc
