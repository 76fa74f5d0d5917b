// oracle/swe.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// The shallow-water system on top of the generic MRAB driver:
//   * RHS R = N + S  (P:82-87 Eq. ode; P:641-651 volume, P:685-691 surface)
//     with the well-balanced LLF flux and the Xing-Shu split
//     source (reading A3);
//   * positivity-preserving limiter M Pi (Alg. 3; O10);
//   * characteristic TVB limiter of Cockburn-Shu with the positivity fix
//     Eq. modified_TVB (O11);
//   * level binning (Eq. cfl + grouping rule; A19);
//   * diagnostics (O12).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "oracle.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

static const int NPMAX = 45, NCMAX = 81, NGMAX = 9;

struct TvbEdge {
  int pj = 0, pk = 0;        // the two neighbour slots (faces of e) used for edge i
  double aj = 0, ak = 0;     // m_i - b0 = aj (b_j - b0) + ak (b_k - b0), clamped >= 0
  double dx = 0, dy = 0;     // unit direction (m_i - b0)/|m_i - b0|
};

struct Swe {
  RefElement re;
  Mesh mesh;
  Params prm;
  double g = 9.81;
  int N = 0, Np = 0, K = 0, Ng = 0, Ncub = 0;
  std::vector<double> B;    // K*Np
  // Dirichlet boundary data (reading A7''): the nodal state [e][field][node] whose trace is the ghost state
  // on the element's Dirichlet faces (and whose cell mean is their TVB ghost mean); empty = not set
  std::vector<double> Qbnd;
  std::vector<double> Q0;   // unlimited state as passed to set_state (for binning)
  Mrab mr;                  // holds the state in mr.Q, element-major [e][field][node]
  bool have_state = false, scheduled = false;
  double sched_dt = 0;
  double t_base = 0;  // simulated time carried across swe_regroup (P:149 regrouping)
  int sched_L = 0;
  std::vector<int> dry;
  std::vector<TvbEdge> tvb;  // K*3
  Mat M1inv;                 // inverse P1 Gram matrix on the reference triangle
  long n_pp = 0, n_dry = 0, n_tvb = 0;
  long n_posfix = 0;  // Eq. modified_TVB applications (min vertex of the TVB-limited h below h0)
  long n_tvb_cw = 0;  // TVB replacements in the component-wise branch (mean depth below h_char, A14)
  double injected = 0;
  std::string err;

  double vel(double h, double m) const;
  void flux(double hm, double hum, double hvm, double bm, double hp, double hup, double hvp, double bp,
            double nx, double ny, double out[3]) const;
  void rhs(int e, const std::function<void(int, double *)> &nbr, const double *q, double *R) const;
  void means(const double *q, double qb[3]) const;
  void p1_coeffs(const double *qf, double d[3]) const;
  void pp(int e, double *q, const unsigned char *rec);
  void tvb_apply(const std::vector<int> &E, const unsigned char *rec);
  void limit(const std::vector<int> &E);
  // Decision replay: a log of the product path's limiter decisions, one record of K bytes per
  // limiter application (Alg. 2 line 1, then every level update), element order of the caller; bits
  // 1 Alg. 3 triggered, 2 dry branch, 4 TVB replaced, 8 Eq. modified_TVB applied, 0xFF not updated.  Where
  // this oracle's own decision sits within kReplayMargin (relative) of its threshold, it adopts the
  // logged decision (n_adopted); a disagreement farther from the threshold is counted in n_mismatch.
  std::vector<unsigned char> replay;
  long replay_n = 0, replay_u = 0;
  long n_adopted = 0, n_mismatch = 0;
  bool decide(bool own, double margin, const unsigned char *rec, int e, unsigned bit);
  void build_tvb_geometry();
  void bin_levels(int L, std::vector<int> &lev) const;
  // Dirichlet faces present but no boundary state given
  bool missing_bnd() const {
    if (!Qbnd.empty()) return false;
    for (signed char t : mesh.bc)
      if (t == 2) return true;
    return false;
  }
};

// A4: continuous desingularised velocity  u = sqrt2 h+ m / sqrt(h+^4 + max(h+^4, eps_u^4)).
// Expression pinned (the product path evaluates it identically for binning).
// Reading A4': eps_u defaults to 1000 h0.  With eps_u = h0 the Alg. 3 limiter
// leaves O(h0) vertex depths carrying O(mean) momentum, |u| grows past the
// fixed CFL speed and the wet/dry Thacker run diverges (measured: eps_u =
// h0, 10 h0, 100 h0 all blow up within 80 steps on C3 at H = 200 m; 1000 h0
// is stable with round-off mass drift).
double Swe::vel(double h, double m) const {
  double hp = std::max(h, 0.0);
  double h2 = hp * hp, h4 = h2 * h2;
  double e2 = prm.eps_u * prm.eps_u, e4 = e2 * e2;
  return (std::sqrt(2.0) * hp * m) / std::sqrt(h4 + std::max(h4, e4));
}

// Well-balanced LLF flux at one Gauss point, own (minus) side total
// (reading A3/A5/A6):
//   h*+- = max(0, h+- + B+- - max(B+, B-)),  Q*+- = (h*, h* u+-, h* v+-)
//   Fhat = 1/2 (Fn(Q*-) + Fn(Q*+)) - lam/2 (Q*+ - Q*-),
//   lam  = max(|u_n-| + sqrt(g h*-), |u_n+| + sqrt(g h*+))
//   own total = Fhat + (0, g/2 ((h-)^2 - (h*-)^2 - (B-)^2) n)
// The -(g/2)(B-)^2 n term is the boundary part of the split source (A3).
void Swe::flux(double hm, double hum, double hvm, double bm, double hp, double hup, double hvp, double bp,
               double nx, double ny, double out[3]) const {
  double um = vel(hm, hum), vm = vel(hm, hvm);
  double up = vel(hp, hup), vp = vel(hp, hvp);
  double Bmax = std::max(bm, bp);
  double hsm = std::max(0.0, hm + bm - Bmax);
  double hsp = std::max(0.0, hp + bp - Bmax);
  double unm = um * nx + vm * ny, unp = up * nx + vp * ny;
  double lam = std::max(std::fabs(unm) + std::sqrt(g * hsm), std::fabs(unp) + std::sqrt(g * hsp));
  double FM[3] = {hsm * unm, hsm * um * unm + 0.5 * g * hsm * hsm * nx, hsm * vm * unm + 0.5 * g * hsm * hsm * ny};
  double FP[3] = {hsp * unp, hsp * up * unp + 0.5 * g * hsp * hsp * nx, hsp * vp * unp + 0.5 * g * hsp * hsp * ny};
  double QM[3] = {hsm, hsm * um, hsm * vm};
  double QP[3] = {hsp, hsp * up, hsp * vp};
  for (int k = 0; k < 3; k++) out[k] = 0.5 * (FM[k] + FP[k]) - 0.5 * lam * (QP[k] - QM[k]);
  double corr = 0.5 * g * (hm * hm - hsm * hsm - bm * bm);
  out[1] += corr * nx;
  out[2] += corr * ny;
}

// R(Q) for element e (P:643-645 N = Pr cF1 + Ps cF2 + P cS; P:687-689 S = -L^g F_n^*).
// q = own state [3][Np]; nbr(n, out) returns a neighbour's nodal state at the
// evaluation time (MRAB driver: committed, start-of-step or dense output).
void Swe::rhs(int e, const std::function<void(int, double *)> &nbr, const double *q, double *R) const {
  const double *b = &B[(size_t)e * Np];
  double rx = mesh.rx[e], ry = mesh.ry[e], sx = mesh.sx[e], sy = mesh.sy[e], J = mesh.J[e];

  // nodal bathymetry gradient (chain rule) -- O6
  double bxn[NPMAX], byn[NPMAX];
  for (int i = 0; i < Np; i++) {
    double br = 0, bs = 0;
    for (int j = 0; j < Np; j++) {
      br += re.Dr(i, j) * b[j];
      bs += re.Ds(i, j) * b[j];
    }
    bxn[i] = rx * br + sx * bs;
    byn[i] = ry * br + sy * bs;
  }

  // volume: interpolate to cubature points, fluxes and split source there
  double cF1[3][NCMAX], cF2[3][NCMAX], cS[3][NCMAX];
  for (int c = 0; c < Ncub; c++) {
    double hc = 0, huc = 0, hvc = 0, bc = 0, bxc = 0, byc = 0;
    for (int i = 0; i < Np; i++) {
      double w = re.Ic(c, i);
      hc += w * q[i];
      huc += w * q[Np + i];
      hvc += w * q[2 * Np + i];
      bc += w * b[i];
      bxc += w * bxn[i];
      byc += w * byn[i];
    }
    double u = vel(hc, huc), v = vel(hc, hvc);
    double p = 0.5 * g * (hc * hc - bc * bc);  // split pressure g/2 (h^2 - B^2)
    double F[3] = {huc, huc * u + p, huc * v};
    double G[3] = {hvc, hvc * u, hvc * v + p};
    double S[3] = {0.0, -g * (hc + bc) * bxc, -g * (hc + bc) * byc};
    for (int k = 0; k < 3; k++) {
      cF1[k][c] = rx * F[k] + ry * G[k];
      cF2[k][c] = sx * F[k] + sy * G[k];
      cS[k][c] = S[k];
    }
  }
  for (int k = 0; k < 3; k++)
    for (int i = 0; i < Np; i++) {
      double acc = 0;
      for (int c = 0; c < Ncub; c++) acc += re.Pr(i, c) * cF1[k][c] + re.Ps(i, c) * cF2[k][c] + re.P(i, c) * cS[k][c];
      R[k * Np + i] = acc;
    }

  // surface: traces Q^g = I_g Q on both sides, numerical flux, lift
  double qg[3][3 * NGMAX], bg[3 * NGMAX], fl[3][3 * NGMAX];
  for (int gp = 0; gp < 3 * Ng; gp++) {
    double a[4] = {0, 0, 0, 0};
    for (int i = 0; i < Np; i++) {
      double w = re.Ig(gp, i);
      a[0] += w * q[i];
      a[1] += w * q[Np + i];
      a[2] += w * q[2 * Np + i];
      a[3] += w * b[i];
    }
    qg[0][gp] = a[0];
    qg[1][gp] = a[1];
    qg[2][gp] = a[2];
    bg[gp] = a[3];
  }
  double qn[3 * NPMAX];
  for (int f = 0; f < 3; f++) {
    int n = mesh.EToE[3 * (size_t)e + f], nf = mesh.EToF[3 * (size_t)e + f];
    bool bnd = (n == e && nf == f);
    const int tag = bnd && !mesh.bc.empty() ? mesh.bc[3 * (size_t)e + f] : 0;
    bool outflow = tag == 1, dirichlet = tag == 2;
    bool wall = bnd && !outflow && !dirichlet;
    double nx = mesh.nx[3 * (size_t)e + f], ny = mesh.ny[3 * (size_t)e + f];
    double scale = mesh.sJ[3 * (size_t)e + f] / J;
    if (!bnd) nbr(n, qn);
    const double *bn = &B[(size_t)n * Np];
    for (int j = 0; j < Ng; j++) {
      int gm = f * Ng + j;
      double hm = qg[0][gm], hum = qg[1][gm], hvm = qg[2][gm], bm = bg[gm];
      double hp, hup, hvp, bp;
      if (wall) {  // reflective wall ghost (A7): mirror the normal momentum
        double mn = hum * nx + hvm * ny;
        hp = hm;
        bp = bm;
        hup = hum - 2.0 * mn * nx;
        hvp = hvm - 2.0 * mn * ny;
      } else if (outflow) {  // transmissive ghost (A7'): the interior trace itself
        hp = hm;
        bp = bm;
        hup = hum;
        hvp = hvm;
      } else if (dirichlet) {  // Dirichlet ghost (A7''): the trace of the prescribed state, B+ = B-
        double a[3] = {0, 0, 0};
        const double *qd = &Qbnd[(size_t)e * 3 * Np];
        for (int i = 0; i < Np; i++) {
          double w = re.Ig(gm, i);
          a[0] += w * qd[i];
          a[1] += w * qd[Np + i];
          a[2] += w * qd[2 * Np + i];
        }
        hp = a[0];
        hup = a[1];
        hvp = a[2];
        bp = bm;
      } else {  // neighbour's Gauss points run in the opposite direction
        int gpn = nf * Ng + (Ng - 1 - j);
        double a[4] = {0, 0, 0, 0};
        for (int i = 0; i < Np; i++) {
          double w = re.Ig(gpn, i);
          a[0] += w * qn[i];
          a[1] += w * qn[Np + i];
          a[2] += w * qn[2 * Np + i];
          a[3] += w * bn[i];
        }
        hp = a[0];
        hup = a[1];
        hvp = a[2];
        bp = a[3];
      }
      double F[3];
      flux(hm, hum, hvm, bm, hp, hup, hvp, bp, nx, ny, F);
      for (int k = 0; k < 3; k++) fl[k][gm] = scale * F[k];
    }
  }
  for (int k = 0; k < 3; k++)
    for (int i = 0; i < Np; i++) {
      double acc = 0;
      for (int gp = 0; gp < 3 * Ng; gp++) acc += re.Lg(i, gp) * fl[k][gp];
      R[k * Np + i] -= acc;
    }
}

// cell mean of each field: 1/2 sum_i w_i q_i, w = Mref 1 (reference area 2)
void Swe::means(const double *q, double qb[3]) const {
  for (int k = 0; k < 3; k++) {
    double acc = 0;
    for (int i = 0; i < Np; i++) acc += re.wmean[i] * q[k * Np + i];
    qb[k] = 0.5 * acc;
  }
}

// L2 projection of one field onto P1 = span{1, r, s} (Pi_1), by its
// definition: Gram system with exact cubature.  Returns d with q1 = d0 + d1 r + d2 s.
void Swe::p1_coeffs(const double *qf, double d[3]) const {
  double rhs[3] = {0, 0, 0};
  for (int c = 0; c < Ncub; c++) {
    double qc = 0;
    for (int i = 0; i < Np; i++) qc += re.Ic(c, i) * qf[i];
    double phi[3] = {1.0, re.rc[c], re.sc[c]};
    for (int a = 0; a < 3; a++) rhs[a] += re.wc[c] * qc * phi[a];
  }
  for (int a = 0; a < 3; a++) d[a] = M1inv(a, 0) * rhs[0] + M1inv(a, 1) * rhs[1] + M1inv(a, 2) * rhs[2];
}

// Decision of a discontinuous branch (A26 replay): own = this oracle's decision, margin = its signed
// distance to the threshold relative to the threshold's scale.  Without a replay log: own.
static const double kReplayMargin = 1e-9;
bool Swe::decide(bool own, double margin, const unsigned char *rec, int e, unsigned bit) {
  if (!rec || rec[e] == 0xFF) return own;
  const bool logged = (rec[e] & bit) != 0;
  if (logged == own) return own;
  if (std::fabs(margin) < kReplayMargin) {
#pragma omp atomic
    n_adopted++;
    return logged;
  }
#pragma omp atomic
  n_mismatch++;
  return own;
}

// Alg. 3, reading O10 / A10-A13.
// Reading A11': both comparisons of Alg. 3 use a relative tie band tau = 1e-10,
//   trigger  <=>  h_min <= eps (1 + tau),   dry  <=>  hbar < h0 (1 + tau).
// The dry branch itself writes h = h0 exactly, i.e. ON the threshold; without
// the band the next update's decisions for such elements are decided by the
// last bit of the cell mean (measured: the GPU and this oracle disagree on
// 666 of 2458 triggers in the first Thacker step).
static const double kTieBand = 1e-10;
void Swe::pp(int e, double *q, const unsigned char *rec) {
  double hmin = q[0];
  for (int i = 1; i < Np; i++) hmin = std::min(hmin, q[i]);
  const double trig_at = prm.eps * (1.0 + kTieBand);
  if (!decide(!(hmin > trig_at), (trig_at - hmin) / trig_at, rec, e, 1)) {
    dry[e] = 0;
    return;
  }
  double qb[3];
  means(q, qb);
  double d[3][3];
  for (int k = 0; k < 3; k++) p1_coeffs(q + k * Np, d[k]);
#pragma omp atomic
  n_pp++;
  const double dry_at = prm.h0 * (1.0 + kTieBand);
  if (decide(qb[0] < dry_at, (dry_at - qb[0]) / dry_at, rec, e, 2)) {  // dry element: h = h0, hu = hv = 0 (not conservative, A13)
    for (int i = 0; i < Np; i++) {
      q[i] = prm.h0;
      q[Np + i] = 0.0;
      q[2 * Np + i] = 0.0;
    }
    double inj = (prm.h0 - qb[0]) * 2.0 * mesh.J[e];
#pragma omp atomic
    injected += inj;
#pragma omp atomic
    n_dry++;
    dry[e] = 1;
    return;
  }
  // min of the linear height over the three vertices
  const double vr[3] = {-1, 1, -1}, vs[3] = {-1, -1, 1};
  double h1min = std::numeric_limits<double>::infinity();
  for (int v = 0; v < 3; v++) h1min = std::min(h1min, d[0][0] + d[0][1] * vr[v] + d[0][2] * vs[v]);
  double theta = 1.0;
  if (qb[0] - h1min > 0.0) theta = std::min(1.0, (qb[0] - prm.h0) / (qb[0] - h1min));
  for (int k = 0; k < 3; k++)
    for (int i = 0; i < Np; i++) {
      double q1 = d[k][0] + d[k][1] * re.r[i] + d[k][2] * re.s[i];
      q[k * Np + i] = qb[k] + theta * (q1 - qb[k]);
    }
  dry[e] = 0;
}

// Static TVB geometry (Cockburn-Shu 1998): for edge i with midpoint m_i,
// m_i - b0 = a_j (b_j - b0) + a_k (b_k - b0) with pair (i,i+1) tried before
// (i,i+2); accept when both a >= -1e-12, else the pair with the larger min(a);
// clamp a >= 0.  Wall ghost barycentre = b0 reflected across the edge; a
// neighbour across a periodic face is translated by (own face midpoint -
// neighbour face midpoint).
void Swe::build_tvb_geometry() {
  tvb.assign(3 * (size_t)K, TvbEdge());
  std::vector<double> bx(K), by(K);
  for (int e = 0; e < K; e++) {
    const int *v = &mesh.EToV[3 * (size_t)e];
    bx[e] = (mesh.vx[v[0]] + mesh.vx[v[1]] + mesh.vx[v[2]]) / 3.0;
    by[e] = (mesh.vy[v[0]] + mesh.vy[v[1]] + mesh.vy[v[2]]) / 3.0;
  }
  auto midpoint = [&](int e, int f, double &x, double &y) {
    const int *v = &mesh.EToV[3 * (size_t)e];
    int a = v[f], b = v[(f + 1) % 3];
    x = 0.5 * (mesh.vx[a] + mesh.vx[b]);
    y = 0.5 * (mesh.vy[a] + mesh.vy[b]);
  };
  for (int e = 0; e < K; e++) {
    double nbx[3], nby[3];
    for (int f = 0; f < 3; f++) {
      int n = mesh.EToE[3 * (size_t)e + f], nf = mesh.EToF[3 * (size_t)e + f];
      double mx, my;
      midpoint(e, f, mx, my);
      if (n == e && nf == f) {
        double nx = mesh.nx[3 * (size_t)e + f], ny = mesh.ny[3 * (size_t)e + f];
        double dist = (bx[e] - mx) * nx + (by[e] - my) * ny;
        nbx[f] = bx[e] - 2.0 * dist * nx;
        nby[f] = by[e] - 2.0 * dist * ny;
      } else {
        double mnx, mny;
        midpoint(n, nf, mnx, mny);
        nbx[f] = bx[n] + (mx - mnx);
        nby[f] = by[n] + (my - mny);
      }
    }
    for (int i = 0; i < 3; i++) {
      double mx, my;
      midpoint(e, i, mx, my);
      double tx = mx - bx[e], ty = my - by[e];
      TvbEdge &te = tvb[3 * (size_t)e + i];
      double len = std::sqrt(tx * tx + ty * ty);
      te.dx = tx / len;
      te.dy = ty / len;
      int cand[2][2] = {{i, (i + 1) % 3}, {i, (i + 2) % 3}};
      double best = -std::numeric_limits<double>::infinity();
      int chosen = -1;
      double ca[2][2];
      for (int p = 0; p < 2; p++) {
        int j = cand[p][0], k = cand[p][1];
        double djx = nbx[j] - bx[e], djy = nby[j] - by[e];
        double dkx = nbx[k] - bx[e], dky = nby[k] - by[e];
        double det = djx * dky - djy * dkx;
        if (det == 0.0) {
          ca[p][0] = ca[p][1] = -std::numeric_limits<double>::infinity();
          continue;
        }
        ca[p][0] = (tx * dky - ty * dkx) / det;
        ca[p][1] = (djx * ty - djy * tx) / det;
        if (chosen < 0 && ca[p][0] >= -1e-12 && ca[p][1] >= -1e-12) chosen = p;
      }
      if (chosen < 0) {
        for (int p = 0; p < 2; p++) {
          double mn = std::min(ca[p][0], ca[p][1]);
          if (mn > best) {
            best = mn;
            chosen = p;
          }
        }
      }
      te.pj = cand[chosen][0];
      te.pk = cand[chosen][1];
      te.aj = std::max(0.0, ca[chosen][0]);
      te.ak = std::max(0.0, ca[chosen][1]);
    }
  }
}

// TVB-modified minmod (Cockburn-Shu): a if |a| <= M Hk^2 (thr), else minmod(a, b).
// Returns true when the first argument was returned.
static bool mbar(double A, double Bv, double thr, double *out) {
  if (std::fabs(A) <= thr) {
    *out = A;
    return true;
  }
  if (A > 0 && Bv > 0) {
    *out = A <= Bv ? A : Bv;
    return A <= Bv;
  }
  if (A < 0 && Bv < 0) {
    *out = A >= Bv ? A : Bv;
    return A >= Bv;
  }
  *out = 0.0;
  return false;
}

// Cockburn-Shu rebalancing so that the three midpoint offsets sum to zero
// (mean preserved): pos = sum max(0,D), neg = sum max(0,-D),
// Dhat = min(1,neg/pos) max(0,D) - min(1,pos/neg) max(0,-D); zero if pos or neg is 0.
static void rebalance(const double D[3], double Dh[3]) {
  double pos = 0, neg = 0;
  for (int i = 0; i < 3; i++) {
    pos += std::max(0.0, D[i]);
    neg += std::max(0.0, -D[i]);
  }
  if (pos != 0.0 && neg != 0.0) {
    double tp = std::min(1.0, neg / pos), tm = std::min(1.0, pos / neg);
    for (int i = 0; i < 3; i++) Dh[i] = tp * std::max(0.0, D[i]) - tm * std::max(0.0, -D[i]);
  } else {
    for (int i = 0; i < 3; i++) Dh[i] = 0.0;
  }
}

// Eq. modified_TVB, reading A15: a linear function with midpoint
// offsets D has vertex values hb + (-D_i + D_j + D_k) (i = face opposite the
// vertex).  If the smallest is below h0:
//   theta = clamp((hb + Dbar - h0) / (Dbar - min(-D_i + D_j + D_k)), 0, 1),
//   Dt_i = Dbar + theta (D_i - Dbar),  Dbar = avg(D).
// fire: < 0 decide by the formula (smallest vertex below h0), 0 / 1 forced (decision replay, A26);
// margin (optional): (smallest vertex - h0) / h0.
static bool posfix(const double D[3], double hb, double h0, double out[3], int force = -1, double *margin = nullptr) {
  double Dbar = (D[0] + D[1] + D[2]) / 3.0;
  double combo_min = std::numeric_limits<double>::infinity();
  for (int i = 0; i < 3; i++) combo_min = std::min(combo_min, -D[i] + D[(i + 1) % 3] + D[(i + 2) % 3]);
  double o[3] = {D[0], D[1], D[2]};
  if (margin) *margin = (hb + combo_min - h0) / h0;
  const bool fire = force < 0 ? hb + combo_min < h0 : force == 1;
  if (fire) {
    double den = Dbar - combo_min;
    double th = den > 0.0 ? (hb + Dbar - h0) / den : 0.0;
    th = std::min(1.0, std::max(0.0, th));
    for (int i = 0; i < 3; i++) o[i] = Dbar + th * (D[i] - Dbar);
  }
  for (int i = 0; i < 3; i++) out[i] = o[i];
  return fire;
}

// Eigenvectors of the normal flux Jacobian along n at the mean state (h, u, v),
// c = sqrt(g h): R columns (1, u - c nx, v - c ny), (0, -ny, nx), (1, u + c nx, v + c ny),
// L = R^{-1}.  Identity (component-wise limiting) when h < h_char (A14).
static void char_matrices(double g, double h, double u, double v, double nx, double ny, double h_char,
                          double Lm[3][3], double Rm[3][3]) {
  if (h >= h_char) {
    double c = std::sqrt(g * h), un = u * nx + v * ny;
    double R_[3][3] = {{1.0, 0.0, 1.0}, {u - c * nx, -ny, u + c * nx}, {v - c * ny, nx, v + c * ny}};
    double L_[3][3] = {{(un + c) / (2.0 * c), -nx / (2.0 * c), -ny / (2.0 * c)},
                       {ny * u - nx * v, -ny, nx},
                       {(c - un) / (2.0 * c), nx / (2.0 * c), ny / (2.0 * c)}};
    std::memcpy(Lm, L_, sizeof(L_));
    std::memcpy(Rm, R_, sizeof(R_));
  } else {
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) Lm[a][b] = Rm[a][b] = (a == b) ? 1.0 : 0.0;
  }
}

// TVB (reading O11/A14-A16/A20) on the elements E, using the
// cell means of the current state of every element (same-level neighbours are
// post-PP values of this update).
void Swe::tvb_apply(const std::vector<int> &E, const unsigned char *rec) {
  if (!prm.use_tvb) return;
  const int ndof = 3 * Np;
  std::vector<double> mean(3 * (size_t)K);
  for (int e = 0; e < K; e++) means(&mr.Q[(size_t)e * ndof], &mean[3 * (size_t)e]);
  std::vector<double> out(E.size() * (size_t)ndof);
  std::vector<char> changed(E.size(), 0), fixed(E.size(), 0), cw(E.size(), 0);
  const double h_char = prm.h_char;
  const double mref[3][2] = {{0.0, -1.0}, {0.0, 0.0}, {-1.0, 0.0}};  // reference edge midpoints
#pragma omp parallel for schedule(dynamic, 64)
  for (long idx = 0; idx < (long)E.size(); idx++) {
    int e = E[idx];
    if (dry[e]) continue;
    bool near_dry = false;
    for (int f = 0; f < 3; f++) {
      int n = mesh.EToE[3 * (size_t)e + f];
      if (dry[n]) near_dry = true;
    }
    if (near_dry) continue;
    const double *q = &mr.Q[(size_t)e * ndof];
    const double *qb = &mean[3 * (size_t)e];
    double d[3][3];
    for (int k = 0; k < 3; k++) p1_coeffs(q + k * Np, d[k]);
    double hb = qb[0];
    double ub = vel(hb, qb[1]), vb = vel(hb, qb[2]);
    double Hk = mesh.Hk[e];
    double thr = prm.tvb_M * Hk * Hk;
    bool all_first = true;
    double Delta[3][3];  // [field][edge]
    for (int i = 0; i < 3; i++) {
      const TvbEdge &te = tvb[3 * (size_t)e + i];
      double ut[3], du[3];
      for (int k = 0; k < 3; k++) ut[k] = d[k][0] + d[k][1] * mref[i][0] + d[k][2] * mref[i][1] - qb[k];
      double nm[2][3];
      int slots[2] = {te.pj, te.pk};
      for (int p = 0; p < 2; p++) {
        int f = slots[p];
        int n = mesh.EToE[3 * (size_t)e + f], nf = mesh.EToF[3 * (size_t)e + f];
        const int tag = (n == e && nf == f && !mesh.bc.empty()) ? mesh.bc[3 * (size_t)e + f] : 0;
        if (tag == 1) {  // outflow ghost mean
          for (int k = 0; k < 3; k++) nm[p][k] = qb[k];
        } else if (tag == 2) {  // Dirichlet ghost mean: the cell mean of the prescribed state (A7'')
          means(&Qbnd[(size_t)e * 3 * Np], nm[p]);
        } else if (n == e && nf == f) {  // wall ghost mean
          double nx = mesh.nx[3 * (size_t)e + f], ny = mesh.ny[3 * (size_t)e + f];
          double mn = qb[1] * nx + qb[2] * ny;
          nm[p][0] = qb[0];
          nm[p][1] = qb[1] - 2.0 * mn * nx;
          nm[p][2] = qb[2] - 2.0 * mn * ny;
        } else {
          for (int k = 0; k < 3; k++) nm[p][k] = mean[3 * (size_t)n + k];
        }
      }
      for (int k = 0; k < 3; k++) du[k] = te.aj * (nm[0][k] - qb[k]) + te.ak * (nm[1][k] - qb[k]);
      // characteristic variables along the edge direction at the mean state
      double Lm[3][3], Rm[3][3];
      char_matrices(g, hb, ub, vb, te.dx, te.dy, h_char, Lm, Rm);
      double wa[3], wb[3], lim[3];
      for (int a = 0; a < 3; a++) {
        wa[a] = Lm[a][0] * ut[0] + Lm[a][1] * ut[1] + Lm[a][2] * ut[2];
        wb[a] = prm.tvb_nu * (Lm[a][0] * du[0] + Lm[a][1] * du[1] + Lm[a][2] * du[2]);
      }
      for (int a = 0; a < 3; a++)
        if (!mbar(wa[a], wb[a], thr, &lim[a])) all_first = false;
      for (int k = 0; k < 3; k++) Delta[k][i] = Rm[k][0] * lim[0] + Rm[k][1] * lim[1] + Rm[k][2] * lim[2];
    }
    if (rec && rec[e] != 0xFF && ((rec[e] & 4) != 0) == all_first) {  // TVB decision differs from the log
#pragma omp atomic
      n_mismatch++;
    }
    if (all_first) continue;  // P1 part unchanged: keep the full P^N polynomial
    double Dh[3][3];
    for (int k = 0; k < 3; k++) rebalance(Delta[k], Dh[k]);
    {
      double D0[3] = {Dh[0][0], Dh[0][1], Dh[0][2]}, mg = 0.0, tmp[3];
      const bool own = posfix(D0, hb, prm.h0, tmp, -1, &mg);
      const bool fire = decide(own, mg, rec, e, 8);
      fixed[idx] = posfix(D0, hb, prm.h0, Dh[0], fire ? 1 : 0) ? 1 : 0;
    }
    cw[idx] = hb < h_char ? 1 : 0;
    // replace by the limited P1 function q = qb + sum_i D_i phi_i, phi_i = 1 - 2 lambda_{(i+2)%3}
    double *o = &out[(size_t)idx * ndof];
    for (int nd = 0; nd < Np; nd++) {
      double lam[3] = {-0.5 * (re.r[nd] + re.s[nd]), 0.5 * (1.0 + re.r[nd]), 0.5 * (1.0 + re.s[nd])};
      for (int k = 0; k < 3; k++) {
        double acc = qb[k];
        for (int i = 0; i < 3; i++) acc += Dh[k][i] * (1.0 - 2.0 * lam[(i + 2) % 3]);
        o[k * Np + nd] = acc;
      }
    }
    changed[idx] = 1;
  }
  for (size_t idx = 0; idx < E.size(); idx++)
    if (changed[idx]) {
      std::memcpy(&mr.Q[(size_t)E[idx] * ndof], &out[idx * ndof], sizeof(double) * ndof);
      n_tvb++;
      n_posfix += fixed[idx];
      n_tvb_cw += cw[idx];
    }
}

// Lambda Pi M Pi (Alg. 2 line 5) on the elements E.
void Swe::limit(const std::vector<int> &E) {
  const int ndof = 3 * Np;
  const unsigned char *rec = replay_u < replay_n ? &replay[(size_t)replay_u * K] : nullptr;
  replay_u++;
  if (prm.use_pp) {
#pragma omp parallel for schedule(dynamic, 64)
    for (long idx = 0; idx < (long)E.size(); idx++) pp(E[idx], &mr.Q[(size_t)E[idx] * ndof], rec);
  }
  tvb_apply(E, rec);
}

// Level binning (reading A19): from the unlimited state passed to set_state.
void Swe::bin_levels(int L, std::vector<int> &lev) const {
  std::vector<double> r(K);
  double rmin = std::numeric_limits<double>::infinity();
  for (int e = 0; e < K; e++) {
    double amax = 0.0;
    for (int i = 0; i < Np; i++) {
      double h = Q0[(size_t)e * 3 * Np + i];
      double u = vel(h, Q0[(size_t)e * 3 * Np + Np + i]);
      double v = vel(h, Q0[(size_t)e * 3 * Np + 2 * Np + i]);
      double hp = std::max(h, 0.0);
      double a = std::sqrt(u * u + v * v) + std::sqrt(g * hp);
      amax = std::max(amax, a);
    }
    double ae = std::max(prm.a_floor, amax);
    r[e] = ae > 0.0 ? mesh.Hk[e] / ae : std::numeric_limits<double>::infinity();
    rmin = std::min(rmin, r[e]);
  }
  lev.assign(K, 1);
  for (int e = 0; e < K; e++) {
    int l = 1;
    for (int k = 1; k < L; k++)
      if (r[e] >= std::ldexp(rmin, k)) l = k + 1;
    lev[e] = l;
  }
}

}  // namespace orc

// =============================================================== C API (ctypes)
using namespace orc;

extern "C" {

typedef struct {
  double h0, eps, tvb_M, tvb_nu, a_floor, eps_u, h_char;
  int use_pp, use_tvb;
  int mrab_coupling;
} orc_params;

typedef struct {
  double t, mass, injected_mass, min_h;
  long n_pp, n_dry, n_tvb;
  int K, Np, nlevels;
  int level_count[16];
  long n_posfix, n_tvb_cw;
  long n_adopted, n_mismatch;
} orc_info;

int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

// Reference-element export for the operator pins.
int orc_refel_sizes(int N, int *out) {
  if (N < 1 || N > 8) return -3;
  out[0] = (N + 1) * (N + 2) / 2;
  out[1] = N + 1;
  RefElement re;
  build_refel(N, re);
  out[2] = re.Ncub;
  out[3] = N + 1;
  return 0;
}
int orc_refel_get(int N, const char *name, double *out) {
  if (N < 1 || N > 8) return -3;
  RefElement re;
  build_refel(N, re);
  std::string n(name);
  auto put = [&](const std::vector<double> &v) { std::copy(v.begin(), v.end(), out); };
  if (n == "r") put(re.r);
  else if (n == "s") put(re.s);
  else if (n == "rc") put(re.rc);
  else if (n == "sc") put(re.sc);
  else if (n == "wc") put(re.wc);
  else if (n == "tg") put(re.tg);
  else if (n == "wg") put(re.wg);
  else if (n == "rg") put(re.rg);
  else if (n == "sg") put(re.sg);
  else if (n == "wmean") put(re.wmean);
  else if (n == "Dr") put(re.Dr.v);
  else if (n == "Ds") put(re.Ds.v);
  else if (n == "Mref") put(re.Mref.v);
  else if (n == "Ic") put(re.Ic.v);
  else if (n == "Ig") put(re.Ig.v);
  else if (n == "P") put(re.P.v);
  else if (n == "Pr") put(re.Pr.v);
  else if (n == "Ps") put(re.Ps.v);
  else if (n == "Lg") put(re.Lg.v);
  else return -1;
  return 0;
}
int orc_quad(int which, int q, double *x, double *w) {
  std::vector<double> X, W;
  if (which == 0) gauss_legendre(q, X, W);
  else if (which == 1) gauss_jacobi10(q, X, W);
  else if (which == 2) {
    lobatto_points(q, X);
    W.assign(X.size(), 0.0);
  } else return -1;
  std::copy(X.begin(), X.end(), x);
  std::copy(W.begin(), W.end(), w);
  return 0;
}

void *orc_create(int nverts, const double *vx, const double *vy, int K, const int *etov, const int *vper,
                 const double *B, int N, double g, const orc_params *p, int *err, char *msg, int msglen) {
  *err = 0;
  if (N < 1 || N > 8) {
    *err = -3;
    return nullptr;
  }
  Swe *s = new Swe();
  std::string m;
  int rc = build_mesh(nverts, vx, vy, K, etov, vper, s->mesh, &m);
  if (rc) {
    *err = rc;
    if (msg && msglen > 0) {
      std::strncpy(msg, m.c_str(), msglen - 1);
      msg[msglen - 1] = 0;
    }
    delete s;
    return nullptr;
  }
  build_refel(N, s->re);
  s->N = N;
  s->Np = s->re.Np;
  s->Ng = s->re.Ng;
  s->Ncub = s->re.Ncub;
  s->K = K;
  s->g = g;
  if (p) {
    s->prm.h0 = p->h0 > 0 ? p->h0 : 1e-6;
    s->prm.eps = p->eps > 0 ? p->eps : s->prm.h0;
    s->prm.tvb_M = p->tvb_M;
    s->prm.tvb_nu = p->tvb_nu > 0 ? p->tvb_nu : 1.5;
    s->prm.a_floor = p->a_floor;
    s->prm.eps_u = p->eps_u > 0 ? p->eps_u : 1000.0 * s->prm.h0;  // reading A4'
    s->prm.h_char = p->h_char > 0 ? p->h_char : 10.0 * s->prm.h0;
    s->prm.use_pp = p->use_pp;
    s->prm.use_tvb = p->use_tvb;
    s->prm.mrab_coupling = p->mrab_coupling;
  } else {
    s->prm.eps = s->prm.h0;
    s->prm.eps_u = 1000.0 * s->prm.h0;
    s->prm.h_char = 10.0 * s->prm.h0;
  }
  s->B.assign(B, B + (size_t)K * s->Np);
  s->dry.assign(K, 0);
  // P1 Gram matrix on the reference triangle, by exact cubature
  Mat M1(3, 3);
  for (int c = 0; c < s->Ncub; c++) {
    double phi[3] = {1.0, s->re.rc[c], s->re.sc[c]};
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) M1(a, b) += s->re.wc[c] * phi[a] * phi[b];
  }
  s->M1inv = inverse(M1);
  s->build_tvb_geometry();
  std::vector<int> lev(K, 1);
  s->mr.init(K, 3 * s->Np, 1, 0.0, lev);
  s->mr.coupling = s->prm.mrab_coupling;
  return s;
}

// caller layout: h[e*Np + i]; internal: Q[(e*3 + field)*Np + i]
int orc_set_state(void *hnd, const double *h, const double *hu, const double *hv) {
  Swe *s = (Swe *)hnd;
  if (s->missing_bnd()) return -4;  // the initial TVB needs the Dirichlet ghost means
  int K = s->K, Np = s->Np;
  s->Q0.assign((size_t)K * 3 * Np, 0.0);
  for (int e = 0; e < K; e++)
    for (int i = 0; i < Np; i++) {
      s->Q0[((size_t)e * 3 + 0) * Np + i] = h[(size_t)e * Np + i];
      s->Q0[((size_t)e * 3 + 1) * Np + i] = hu[(size_t)e * Np + i];
      s->Q0[((size_t)e * 3 + 2) * Np + i] = hv[(size_t)e * Np + i];
    }
  std::vector<int> lev(K, 1);
  s->mr.init(K, 3 * Np, 1, 0.0, lev);
  s->mr.Q = s->Q0;
  s->dry.assign(K, 0);
  s->n_pp = s->n_dry = s->n_tvb = s->n_posfix = s->n_tvb_cw = 0;
  s->replay_u = 0;
  s->injected = 0;
  s->have_state = true;
  s->scheduled = false;
  s->t_base = 0;
  // Alg. 2 line 1: Q^0 = Lambda Pi M Pi (Pi_H Q^0) on every element
  std::vector<int> all(K);
  for (int e = 0; e < K; e++) all[e] = e;
  s->limit(all);
  return 0;
}

int orc_step(void *hnd, double dt, int nlevels) {
  Swe *s = (Swe *)hnd;
  if (!s->have_state || s->missing_bnd()) return -4;
  if (!(dt > 0) || !std::isfinite(dt) || nlevels < 1 || nlevels > 8) return -1;
  if (!s->scheduled) {
    std::vector<int> lev;
    s->bin_levels(nlevels, lev);
    std::vector<double> Q = s->mr.Q;
    s->mr.init(s->K, 3 * s->Np, nlevels, dt, lev);
    s->mr.Q = Q;
    s->mr.rhs = [s](int e, long t, double *R) {
      auto nbr = [s, t](int n, double *out) { s->mr.state_at(n, t, out); };
      s->rhs(e, nbr, &s->mr.Q[(size_t)e * 3 * s->Np], R);
    };
    s->mr.post = [s](int, const std::vector<int> &E) { s->limit(E); };
    s->scheduled = true;
    s->sched_dt = dt;
    s->sched_L = nlevels;
  } else if (dt != s->sched_dt || nlevels != s->sched_L) {
    return -5;
  }
  s->mr.macro_step();
  for (double v : s->mr.Q)
    if (!std::isfinite(v)) return -6;
  return 0;
}

// Level regrouping ("elements can be regrouped after every few time steps"; SURVEY
// NEXT-4): the current state becomes the state of a fresh swe_set_state -- levels re-binned at
// the next step from it, Alg. 2 line 1 applied to it, AB ramp and counters restarted -- while the
// simulated time continues.
// Boundary tags (reading A7'): an unmatched face whose two vertices are both tagged 1 is a
// transmissive outflow boundary (ghost state = interior trace); every other unmatched face stays a
// reflective wall.  vbc = NULL: all walls.
int orc_set_boundary(void *hnd, const signed char *vbc) {
  Swe *s = (Swe *)hnd;
  s->mesh.bc.assign((size_t)3 * s->K, 0);
  if (!vbc) return 0;
  for (int e = 0; e < s->K; e++)
    for (int f = 0; f < 3; f++) {
      const size_t i = 3 * (size_t)e + f;
      if (s->mesh.EToE[i] != e || s->mesh.EToF[i] != f) continue;
      const int a = s->mesh.EToV[3 * (size_t)e + f], b = s->mesh.EToV[3 * (size_t)e + (f + 1) % 3];
      // both vertices tagged: the face takes the smaller tag (1 outflow, 2 Dirichlet); otherwise a wall
      s->mesh.bc[i] = (vbc[a] >= 1 && vbc[b] >= 1) ? (signed char)std::min<int>(std::min<int>(vbc[a], vbc[b]), 2) : 0;
    }
  return 0;
}

// Dirichlet boundary data (reading A7''): caller layout [e*Np + i]; kept until replaced.
int orc_set_boundary_state(void *hnd, const double *h, const double *hu, const double *hv) {
  Swe *s = (Swe *)hnd;
  const int K = s->K, Np = s->Np;
  s->Qbnd.assign((size_t)K * 3 * Np, 0.0);
  for (int e = 0; e < K; e++)
    for (int i = 0; i < Np; i++) {
      s->Qbnd[((size_t)e * 3 + 0) * Np + i] = h[(size_t)e * Np + i];
      s->Qbnd[((size_t)e * 3 + 1) * Np + i] = hu[(size_t)e * Np + i];
      s->Qbnd[((size_t)e * 3 + 2) * Np + i] = hv[(size_t)e * Np + i];
    }
  return 0;
}

int orc_get_state(void *hnd, double *h, double *hu, double *hv);
int orc_regroup(void *hnd) {
  Swe *s = (Swe *)hnd;
  if (!s->have_state) return -4;
  const double t = s->t_base + (s->scheduled ? s->sched_dt * (double)s->mr.tick : 0.0);
  const size_t KNp = (size_t)s->K * s->Np;
  std::vector<double> h(KNp), hu(KNp), hv(KNp);
  orc_get_state(hnd, h.data(), hu.data(), hv.data());
  orc_set_state(hnd, h.data(), hu.data(), hv.data());
  s->t_base = t;
  return 0;
}

int orc_get_state(void *hnd, double *h, double *hu, double *hv) {
  Swe *s = (Swe *)hnd;
  if (!s->have_state) return -4;
  int K = s->K, Np = s->Np;
  for (int e = 0; e < K; e++)
    for (int i = 0; i < Np; i++) {
      h[(size_t)e * Np + i] = s->mr.Q[((size_t)e * 3 + 0) * Np + i];
      hu[(size_t)e * Np + i] = s->mr.Q[((size_t)e * 3 + 1) * Np + i];
      hv[(size_t)e * Np + i] = s->mr.Q[((size_t)e * 3 + 2) * Np + i];
    }
  return 0;
}

int orc_get_levels(void *hnd, int *level) {
  Swe *s = (Swe *)hnd;
  if (!s->scheduled) return -4;
  for (int e = 0; e < s->K; e++) level[e] = s->mr.level[e];
  return 0;
}

// levels without stepping (for the bit-exact binning test)
int orc_bin_levels(void *hnd, int nlevels, int *level) {
  Swe *s = (Swe *)hnd;
  if (!s->have_state) return -4;
  std::vector<int> lev;
  s->bin_levels(nlevels, lev);
  std::copy(lev.begin(), lev.end(), level);
  return 0;
}

int orc_get_connectivity(void *hnd, int *etoe, signed char *etof) {
  Swe *s = (Swe *)hnd;
  for (size_t i = 0; i < 3 * (size_t)s->K; i++) {
    etoe[i] = s->mesh.EToE[i];
    etof[i] = (signed char)s->mesh.EToF[i];
  }
  return 0;
}

int orc_get_geometry(void *hnd, double *J, double *Hk, int *nflipped) {
  Swe *s = (Swe *)hnd;
  for (int e = 0; e < s->K; e++) {
    J[e] = s->mesh.J[e];
    Hk[e] = s->mesh.Hk[e];
  }
  *nflipped = s->mesh.nflipped;
  return 0;
}

int orc_get_tvb_geometry(void *hnd, int *pairs, double *alphas) {
  Swe *s = (Swe *)hnd;
  for (size_t i = 0; i < 3 * (size_t)s->K; i++) {
    pairs[2 * i] = s->tvb[i].pj;
    pairs[2 * i + 1] = s->tvb[i].pk;
    alphas[2 * i] = s->tvb[i].aj;
    alphas[2 * i + 1] = s->tvb[i].ak;
  }
  return 0;
}

int orc_nodes(void *hnd, double *x, double *y) {
  Swe *s = (Swe *)hnd;
  for (int e = 0; e < s->K; e++) {
    const int *v = &s->mesh.EToV[3 * (size_t)e];
    double x1 = s->mesh.vx[v[0]], x2 = s->mesh.vx[v[1]], x3 = s->mesh.vx[v[2]];
    double y1 = s->mesh.vy[v[0]], y2 = s->mesh.vy[v[1]], y3 = s->mesh.vy[v[2]];
    for (int i = 0; i < s->Np; i++) {
      double r = s->re.r[i], ss = s->re.s[i];
      x[(size_t)e * s->Np + i] = -0.5 * (r + ss) * x1 + 0.5 * (1.0 + r) * x2 + 0.5 * (1.0 + ss) * x3;
      y[(size_t)e * s->Np + i] = -0.5 * (r + ss) * y1 + 0.5 * (1.0 + r) * y2 + 0.5 * (1.0 + ss) * y3;
    }
  }
  return 0;
}

// Single-rate RHS of a given (unlimited) state, every neighbour synchronised.
int orc_rhs(void *hnd, const double *h, const double *hu, const double *hv, double *Rh_, double *Rhu, double *Rhv) {
  Swe *s = (Swe *)hnd;
  if (s->missing_bnd()) return -4;
  int K = s->K, Np = s->Np;
  std::vector<double> Q((size_t)K * 3 * Np);
  for (int e = 0; e < K; e++)
    for (int i = 0; i < Np; i++) {
      Q[((size_t)e * 3 + 0) * Np + i] = h[(size_t)e * Np + i];
      Q[((size_t)e * 3 + 1) * Np + i] = hu[(size_t)e * Np + i];
      Q[((size_t)e * 3 + 2) * Np + i] = hv[(size_t)e * Np + i];
    }
#pragma omp parallel for
  for (int e = 0; e < K; e++) {
    double R[3 * NPMAX];
    auto nbr = [&](int n, double *out) { std::memcpy(out, &Q[(size_t)n * 3 * Np], sizeof(double) * 3 * Np); };
    s->rhs(e, nbr, &Q[(size_t)e * 3 * Np], R);
    for (int i = 0; i < Np; i++) {
      Rh_[(size_t)e * Np + i] = R[i];
      Rhu[(size_t)e * Np + i] = R[Np + i];
      Rhv[(size_t)e * Np + i] = R[2 * Np + i];
    }
  }
  return 0;
}

// Apply PP (+TVB) to a given state once (limiter pins); returns dry flags.
int orc_limit(void *hnd, double *h, double *hu, double *hv, int *dry) {
  Swe *s = (Swe *)hnd;
  int rc = orc_set_state(hnd, h, hu, hv);
  if (rc) return rc;
  orc_get_state(hnd, h, hu, hv);
  for (int e = 0; e < s->K; e++) dry[e] = s->dry[e];
  return 0;
}

int orc_get_info(void *hnd, orc_info *info) {
  Swe *s = (Swe *)hnd;
  std::memset(info, 0, sizeof(*info));
  info->K = s->K;
  info->Np = s->Np;
  info->nlevels = s->scheduled ? s->sched_L : 0;
  info->t = s->t_base + (s->scheduled ? s->sched_dt * (double)s->mr.tick : 0.0);
  double mass = 0, minh = std::numeric_limits<double>::infinity();
  for (int e = 0; e < s->K; e++) {
    const double *q = &s->mr.Q[(size_t)e * 3 * s->Np];
    double acc = 0;
    for (int i = 0; i < s->Np; i++) {
      acc += s->re.wmean[i] * q[i];
      minh = std::min(minh, q[i]);
    }
    mass += s->mesh.J[e] * acc;
    if (s->scheduled) info->level_count[s->mr.level[e] - 1]++;
  }
  info->mass = mass;
  info->min_h = minh;
  info->injected_mass = s->injected;
  info->n_pp = s->n_pp;
  info->n_dry = s->n_dry;
  info->n_tvb = s->n_tvb;
  info->n_posfix = s->n_posfix;
  info->n_tvb_cw = s->n_tvb_cw;
  info->n_adopted = s->n_adopted;
  info->n_mismatch = s->n_mismatch;
  return 0;
}

// ---- small pure functions exported for the pins
double orc_vel(double h, double m, double eps_u) {
  Swe s;
  s.prm.eps_u = eps_u;
  return s.vel(h, m);
}
void orc_flux(double g, double eps_u, const double *qm, double bm, const double *qp, double bp, double nx, double ny,
              double *out) {
  Swe s;
  s.g = g;
  s.prm.eps_u = eps_u;
  s.flux(qm[0], qm[1], qm[2], bm, qp[0], qp[1], qp[2], bp, nx, ny, out);
}
// Decision replay: log of nrec records of K bytes (see Swe::replay), consumed one record per
// limiter application from the next orc_set_state on.  nrec = 0 switches replay off.
int orc_set_replay(void *hnd, const unsigned char *log, long nrec) {
  Swe *s = (Swe *)hnd;
  s->replay.assign(log, log + (size_t)nrec * s->K);
  s->replay_n = nrec;
  s->replay_u = 0;
  s->n_adopted = s->n_mismatch = 0;
  return 0;
}

int orc_mbar(double a, double b, double thr, double *out) { return mbar(a, b, thr, out) ? 1 : 0; }
void orc_rebalance(const double *D, double *out) { rebalance(D, out); }
int orc_posfix(const double *D, double hb, double h0, double *out) { return posfix(D, hb, h0, out) ? 1 : 0; }
void orc_char(double g, double h, double u, double v, double nx, double ny, double *L, double *R) {
  double Lm[3][3], Rm[3][3];
  char_matrices(g, h, u, v, nx, ny, 0.0, Lm, Rm);
  std::memcpy(L, Lm, sizeof(Lm));
  std::memcpy(R, Rm, sizeof(Rm));
}

void orc_destroy(void *hnd) { delete (Swe *)hnd; }

// Linear toy ODE  dy_e/dt = sum_j A_ej y_j(t)  integrated by the same MRAB
// driver (order pins).  seed0/seed1 (optional): exact R at
// t0 - 2 dt_l and t0 - dt_l for each element's level (exact AB history).
int orc_toy_mrab(int K, const double *A, const int *level, const double *y0, double dt, int L, int nsteps,
                 const double *seed0, const double *seed1, double *yout, int coupling) {
  Mrab mr;
  mr.coupling = coupling;
  std::vector<int> lev(level, level + K);
  mr.init(K, 1, L, dt, lev);
  for (int e = 0; e < K; e++) mr.Q[e] = y0[e];
  mr.rhs = [&](int e, long t, double *R) {
    double acc = 0;
    for (int j = 0; j < K; j++) {
      double a = A[(size_t)e * K + j];
      if (a == 0.0) continue;
      double yj;
      mr.state_at(j, t, &yj);
      acc += a * yj;
    }
    R[0] = acc;
  };
  if (seed0 && seed1) {
    for (int l = 1; l <= L; l++) {
      mr.kcount[l] = 2;
      mr.tick_s[l] = -(1L << (l - 1));
      mr.t_e[l] = 0;
    }
    for (int e = 0; e < K; e++) {
      mr.Rh[0][e] = seed0[e];
      mr.Rh[1][e] = seed1[e];
    }
  }
  for (int n = 0; n < nsteps; n++) mr.macro_step();
  for (int e = 0; e < K; e++) yout[e] = mr.Q[e];
  return 0;
}

}  // extern "C"
