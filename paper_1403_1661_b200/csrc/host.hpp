// host.hpp -- host-side builders of the product path (reference element,
// mesh/connectivity, static TVB geometry, MRAB level binning, element order).
// Independent of oracle/ (no shared code); cross-checked against it by tests.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace swe {

constexpr int kMaxOrder = 5;  // device kernels are instantiated for N = 1..5

// Row-major dense matrix.
struct DMat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  DMat() {}
  DMat(int r, int c) : rows(r), cols(c), a((size_t)r * c, 0.0) {}
  double &operator()(int i, int j) { return a[(size_t)i * cols + j]; }
  double operator()(int i, int j) const { return a[(size_t)i * cols + j]; }
};

// Reference-element operators.
struct RefOps {
  int N = 0, Np = 0, Nfp = 0, Ng = 0, Nc = 0;
  std::vector<double> r, s;         // Warp & Blend nodes
  std::vector<double> rc, sc, wc;   // collapsed Gauss-Jacobi cubature, strength 2N+1
  std::vector<double> tg, wg;       // Gauss-Legendre, Ng = N+1 per face
  DMat V, Vinv, Dr, Ds, Mref;
  DMat Ic, IcDr, IcDs;              // Nc x Np
  DMat P, Pr, Ps;                   // Np x Nc
  DMat Ig, Lg;                      // 3Ng x Np, Np x 3Ng
  DMat Ig1;                         // Ng x Nfp: face nodes (CCW) -> face Gauss points
  DMat Pv;                          // 3 x Np: vertex values of the L2 projection onto P1
  std::vector<double> wmean;        // int l_i (sums to 2)
  std::vector<int> Fmask;           // 3 x Nfp, face nodes in CCW order along each face
};
bool build_refops(int N, RefOps &ops, std::string *err);

// Mesh after orientation fix, with connectivity (caller element order).
struct HostMesh {
  int K = 0, nv = 0, nflipped = 0;
  std::vector<double> vx, vy;
  std::vector<int32_t> etov;   // K*3 counter-clockwise
  std::vector<int32_t> etoe;   // K*3
  std::vector<int8_t> etof;    // K*3
  std::vector<double> hk;      // incircle diameter
  std::vector<int8_t> bc;      // K*3: boundary faces 0 reflective wall, 1 transmissive outflow (A7'), 2 Dirichlet (A7'')
};
// Outflow tags from vertex tags (swe_mesh.vbc, NULL = all walls).
void apply_boundary_tags(HostMesh &m, const int8_t *vbc);
// returns 0 or SWE_ERR_MESH (-2)
int build_mesh(int nverts, const double *vx, const double *vy, int K, const int32_t *etov,
               const int32_t *vper, HostMesh &m, std::string *err);

// Static Cockburn-Shu geometry per element edge (caller order): neighbour
// slots (j,k) and alphas with m_i - b0 = a_j (b_j - b0) + a_k (b_k - b0).
struct TvbGeom {
  std::vector<int8_t> pj, pk;     // K*3
  std::vector<double> aj, ak;     // K*3
};
void build_tvb_geometry(const HostMesh &m, TvbGeom &t);

// Wave-speed pieces shared by host binning and the device a_e kernel.
double desing_velocity(double h, double m, double e4);
// a_e = max(a_floor, max_nodes |u| + sqrt(g max(h,0))), caller layout [K][Np]
void element_speeds(int K, int Np, double g, double eps_u, double a_floor, const double *h, const double *hu,
                    const double *hv, double *ae);
// level = 1 + max{k in [0,L-1] : Hk/a_e >= 2^k r_min}  (reading A19)
void bin_levels(int K, const double *hk, const double *ae, int L, int32_t *level);
// same with a given (global, all-rank) r_min
void bin_levels_rmin(int K, const double *hk, const double *ae, int L, double rmin, int32_t *level);

// Internal element order: level-major, Morton order of the barycentres within a level.
void element_order(const HostMesh &m, const int32_t *level, std::vector<int32_t> &order);

}  // namespace swe

namespace swe {

// Partition of a (sub-)mesh among ranks.  Every element of the
// given mesh carries a global id and an owner rank.  Owned elements are the
// ones with owner == rank; ghosts are the non-owned face neighbours of owned
// elements; every other element is dropped.  Send list to peer q: owned
// elements with a ghost neighbour owned by q; receive list from q: ghosts owned
// by q.  Both sides order their lists by global id, so rank r's send list to q
// equals q's receive list from r element by element.
struct HaloPlan {
  std::vector<int32_t> owned, ghosts;   // element indices of the given mesh
  std::vector<int32_t> peers;           // peer ranks, ascending
  std::vector<std::vector<int32_t>> send, recv;  // per peer: element indices of the given mesh, by gid
};
void build_halo_plan(const HostMesh &m, const int64_t *gid, const int32_t *owner, int rank, HaloPlan &plan);

}  // namespace swe
