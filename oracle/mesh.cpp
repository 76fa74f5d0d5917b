// oracle/mesh.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Conforming triangulation ("non-overlapping, conforming triangles"),
// face connectivity and affine geometry.  Readings: SURVEY §8(c) O4 (Hk =
// incircle diameter 4A/perimeter, expression pinned for bit-exact level
// binning), O5 (faces keyed by the sorted pair of canonical vertex ids;
// unmatched faces are walls with self reference; >2 owners is an error).
#include <cmath>
#include <map>
#include <utility>

#include "oracle.hpp"

namespace orc {

int build_mesh(int nverts, const double *vx, const double *vy, int K, const int *etov,
               const int *vper, Mesh &m, std::string *msg) {
  m.K = K;
  m.vx.assign(vx, vx + nverts);
  m.vy.assign(vy, vy + nverts);
  m.EToV.assign(etov, etov + 3 * (size_t)K);
  m.nflipped = 0;
  for (int e = 0; e < K; e++) {
    int *v = &m.EToV[3 * (size_t)e];
    for (int k = 0; k < 3; k++)
      if (v[k] < 0 || v[k] >= nverts) {
        if (msg) *msg = "vertex index out of range in element " + std::to_string(e);
        return -2;
      }
    if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2]) {
      if (msg) *msg = "repeated vertex in element " + std::to_string(e);
      return -2;
    }
    double x1 = vx[v[0]], x2 = vx[v[1]], x3 = vx[v[2]];
    double y1 = vy[v[0]], y2 = vy[v[1]], y3 = vy[v[2]];
    double A = 0.5 * ((x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1));
    if (A == 0.0) {
      if (msg) *msg = "zero-area element " + std::to_string(e);
      return -2;
    }
    if (A < 0.0) {  // clockwise: swap v1 and v2
      int t = v[1];
      v[1] = v[2];
      v[2] = t;
      m.nflipped++;
    }
  }

  // connectivity: key = sorted pair of canonical vertex ids
  std::map<std::pair<int, int>, std::vector<std::pair<int, int>>> faces;
  for (int e = 0; e < K; e++)
    for (int f = 0; f < 3; f++) {
      int a = m.EToV[3 * (size_t)e + f], b = m.EToV[3 * (size_t)e + (f + 1) % 3];
      if (vper) {
        a = vper[a];
        b = vper[b];
      }
      std::pair<int, int> key(std::min(a, b), std::max(a, b));
      faces[key].push_back(std::make_pair(e, f));
    }
  m.EToE.assign(3 * (size_t)K, 0);
  m.EToF.assign(3 * (size_t)K, 0);
  for (int e = 0; e < K; e++)
    for (int f = 0; f < 3; f++) {
      m.EToE[3 * (size_t)e + f] = e;
      m.EToF[3 * (size_t)e + f] = f;
    }
  for (auto &kv : faces) {
    if (kv.second.size() > 2) {
      if (msg) *msg = "face shared by more than two elements";
      return -2;
    }
    if (kv.second.size() == 2) {
      auto p = kv.second[0], q = kv.second[1];
      m.EToE[3 * (size_t)p.first + p.second] = q.first;
      m.EToF[3 * (size_t)p.first + p.second] = q.second;
      m.EToE[3 * (size_t)q.first + q.second] = p.first;
      m.EToF[3 * (size_t)q.first + q.second] = p.second;
    }
  }

  // affine geometry: x = -(r+s)/2 x1 + (1+r)/2 x2 + (1+s)/2 x3
  m.J.assign(K, 0);
  m.rx.assign(K, 0);
  m.ry.assign(K, 0);
  m.sx.assign(K, 0);
  m.sy.assign(K, 0);
  m.area.assign(K, 0);
  m.Hk.assign(K, 0);
  m.nx.assign(3 * (size_t)K, 0);
  m.ny.assign(3 * (size_t)K, 0);
  m.sJ.assign(3 * (size_t)K, 0);
  for (int e = 0; e < K; e++) {
    const int *v = &m.EToV[3 * (size_t)e];
    double x1 = vx[v[0]], x2 = vx[v[1]], x3 = vx[v[2]];
    double y1 = vy[v[0]], y2 = vy[v[1]], y3 = vy[v[2]];
    double xr = 0.5 * (x2 - x1), xs = 0.5 * (x3 - x1), yr = 0.5 * (y2 - y1), ys = 0.5 * (y3 - y1);
    double J = xr * ys - xs * yr;
    m.J[e] = J;
    m.rx[e] = ys / J;
    m.ry[e] = -xs / J;
    m.sx[e] = -yr / J;
    m.sy[e] = xr / J;
    // pinned expressions: A and Hk = 4A / (l01 + l12 + l20)
    double A = 0.5 * ((x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1));
    double X[3] = {x1, x2, x3}, Y[3] = {y1, y2, y3}, len[3];
    for (int f = 0; f < 3; f++) {
      double dx = X[(f + 1) % 3] - X[f], dy = Y[(f + 1) % 3] - Y[f];
      len[f] = std::sqrt(dx * dx + dy * dy);
      m.nx[3 * (size_t)e + f] = dy / len[f];
      m.ny[3 * (size_t)e + f] = -dx / len[f];
      m.sJ[3 * (size_t)e + f] = 0.5 * len[f];
    }
    m.area[e] = A;
    m.Hk[e] = (4.0 * A) / ((len[0] + len[1]) + len[2]);
  }
  return 0;
}

}  // namespace orc
