// oracle/oracle.hpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the method of
// arXiv:1403.1661 ("GPU accelerated discontinuous Galerkin methods for shallow
// water equations", PAPER.md), written from the paper and SURVEY.md §8(c).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load it.  It shares no code, header, table or
// helper with the CUDA product path in paper_1403_1661_b200/.
//
// Citation shorthand: P:n = /root/reference/PAPER.md line n.
//
// Deliberately different construction from the product path: the oracle uses
// a tensor-Legendre basis L_p(r)L_q(s) (p+q<=N) for every polynomial operation
// and defines mass matrix / projections by cubature sums (their plain
// definitions), while the product path builds the orthonormal Dubiner basis.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- linear algebra
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> v;
  Mat() {}
  Mat(int r, int c) : rows(r), cols(c), v((size_t)r * (size_t)c, 0.0) {}
  double &operator()(int i, int j) { return v[(size_t)i * cols + j]; }
  double operator()(int i, int j) const { return v[(size_t)i * cols + j]; }
};
Mat matmul(const Mat &A, const Mat &B);
Mat transpose(const Mat &A);
Mat inverse(const Mat &A);  // Gauss-Jordan, partial pivoting; throws on singular

// ---------------------------------------------------------------- 1D polynomials / rules
double legendre(int n, double x);        // L_n, L_n(1) = 1
double legendre_deriv(int n, double x);  // L_n'
void gauss_legendre(int q, std::vector<double> &x, std::vector<double> &w);
void gauss_jacobi10(int q, std::vector<double> &x, std::vector<double> &w);  // weight (1-x)
void lobatto_points(int N, std::vector<double> &x);                           // N+1 LGL points

// ---------------------------------------------------------------- reference element
struct RefElement {
  int N = 0, Np = 0, Nfp = 0, Ncub = 0, Ng = 0;
  std::vector<double> r, s;        // Warp & Blend nodes, HW Nodes2D order
  std::vector<double> rc, sc, wc;  // triangle cubature (collapsed Gauss-Jacobi)
  std::vector<double> tg, wg;      // 1D Gauss-Legendre on [-1,1]
  std::vector<double> rg, sg;      // 3*Ng face Gauss points, face-major, CCW along each face
  Mat V, Vinv;                     // tensor-Legendre Vandermonde at the nodes
  Mat Dr, Ds;                      // nodal differentiation
  Mat Mref;                        // reference mass matrix  (int l_i l_j)
  Mat Ic, Ig;                      // nodes -> cubature points, nodes -> face Gauss points
  Mat P, Pr, Ps, Lg;               // P:651 projections, P:691 lift
  std::vector<double> wmean;       // Mref * 1 (int l_i), sums to 2
};
void warp_blend_nodes(int N, std::vector<double> &r, std::vector<double> &s);
void build_refel(int N, RefElement &re);
Mat interp_matrix(const RefElement &re, const std::vector<double> &r, const std::vector<double> &s);

// ---------------------------------------------------------------- mesh
struct Mesh {
  int K = 0, nflipped = 0;
  std::vector<double> vx, vy;
  std::vector<int> EToV;          // K*3, counter-clockwise after orientation fix
  std::vector<int> EToE, EToF;    // K*3, boundary: self reference
  std::vector<double> J, rx, ry, sx, sy, area, Hk;
  std::vector<double> nx, ny, sJ;  // K*3, face f = v_f -> v_{f+1}
  std::vector<signed char> bc;     // K*3, boundary faces: 0 reflective wall, 1 transmissive outflow (A7')
};
// returns 0, or -2 (mesh error) with msg filled
int build_mesh(int nverts, const double *vx, const double *vy, int K, const int *etov,
               const int *vper, Mesh &m, std::string *msg);

// ---------------------------------------------------------------- parameters
struct Params {
  double h0 = 1e-6, eps = 0, tvb_M = 0, tvb_nu = 1.5, a_floor = 0, eps_u = 0, h_char = 0;
  int use_pp = 1, use_tvb = 1;
  int mrab_coupling = 0;  // 0: reading A17 (recursive, dense output); 1: Alg. 1 printed order, latest committed
};

// ---------------------------------------------------------------- MRAB driver (Alg. 1)
// Generic over the right-hand side so the same scheduling code is exercised by
// the SWE system and by the linear toy ODE used for the order pins.
struct Mrab {
  int K = 0, ndof = 0, L = 1;
  double dt = 0;
  std::vector<int> level;                     // 1..L per element
  std::vector<std::vector<int>> elems;        // elems[l] = elements of level l
  std::vector<double> Q, Qs, Rh[3];           // K*ndof each
  int kcount[17] = {0};                       // updates done by level l
  long tick_s[17] = {0};                      // tick at which level l's current step started
  long t_e[17] = {0};                         // tick of level l's committed state
  long tick = 0;                              // macro-step start, in units of dt
  // 0: recursive slowest-first order with AB3 dense output (reading A17);
  // 1: Alg. 1's printed loop nest (levels descending, substeps inner) with every
  //    neighbour read at its latest committed value (SPEC's reading; first order at level interfaces)
  int coupling = 0;
  // R(e) at `tick`, may call state_at() for any element
  std::function<void(int e, long tick, double *R)> rhs;
  // hook applied after the AB update of level l (limiters, Alg. 2)
  std::function<void(int l, const std::vector<int> &elems)> post;

  void init(int K, int ndof, int L, double dt, const std::vector<int> &level);
  // value of element n at time `t` (ticks): committed, start-of-step, or AB3 dense output
  void state_at(int n, long t, double *out) const;
  void update_level(int l, long t);
  void advance(int l, long t);
  void macro_step();
};
void ab_coeffs(int m, double alpha[3]);
void dense_coeffs(int m, double theta, double beta[3]);

}  // namespace orc
