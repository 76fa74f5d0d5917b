// solver.cu -- context, MRAB scheduler and C ABI (include/swe.h) of the
// B200-native DG shallow-water solver.  Device work: kernels.cuh (hot path)
// plus the setup / permutation / diagnostics kernels below.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/swe.h"
#include "host.hpp"
#include "kernels.cuh"

namespace swe {

// NVTX ranges (header-only NVTX3: no-ops unless a profiler injects itself) around the host driver's phases
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
static const char *kLevelRange[9] = {"update L0", "update L1", "update L2", "update L3", "update L4",
                                     "update L5", "update L6", "update L7", "update L8"};

// ------------------------------------------------------------------ setup kernels
// a_e of every element from the staged caller-layout state, with IEEE
// round-to-nearest intrinsics (no FMA contraction), bit-identical to the host
// expression of element_speeds() (reading A19).
__global__ void k_speeds(int K, int Np, double g, double e4, double a_floor, const double *h, const double *hu,
                         const double *hv, double *ae) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  const double sq2 = 1.4142135623730951;  // == sqrt(2.0) correctly rounded
  double amax = 0.0;
  for (int i = 0; i < Np; i++) {
    size_t k = (size_t)e * Np + i;
    double hh = h[k];
    double hp = hh > 0.0 ? hh : 0.0;
    double h2 = __dmul_rn(hp, hp), h4 = __dmul_rn(h2, h2);
    double den = __dsqrt_rn(__dadd_rn(h4, h4 > e4 ? h4 : e4));
    double num = __dmul_rn(sq2, hp);
    double u = __ddiv_rn(__dmul_rn(num, hu[k]), den), v = __ddiv_rn(__dmul_rn(num, hv[k]), den);
    double a = __dadd_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v))), __dsqrt_rn(__dmul_rn(g, hp)));
    amax = a > amax ? a : amax;
  }
  ae[e] = a_floor > amax ? a_floor : amax;
}

// Level binning on the device, bit-identical to the host bin_levels_rmin() (reading A19):
// r_e = Hk_e / a_e (IEEE division; +inf when a_e = 0), r_min = min_e r_e,
// level_e = 1 + max{k < L : r_e >= 2^k r_min}.  Hk is the host's own array (uploaded once).
// Positive doubles (and +inf) order like their bit patterns, so r_min is an atomicMin on the bits.
__global__ void k_rmin(int K, const double *hk, const double *ae, unsigned long long *rmin_bits) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double r = inf;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K; e += gridDim.x * blockDim.x) {
    const double re = ae[e] > 0.0 ? __ddiv_rn(hk[e], ae[e]) : inf;
    r = re < r ? re : r;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_xor_sync(0xffffffffu, r, o);
    r = q < r ? q : r;
  }
  if ((threadIdx.x & 31) == 0) atomicMin(rmin_bits, (unsigned long long)__double_as_longlong(r));
}
__global__ void k_levels(int K, const double *hk, const double *ae, const double *rmin_p, int L, int32_t *level,
                         const int32_t *resident, int *changed) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const double r = ae[e] > 0.0 ? __ddiv_rn(hk[e], ae[e]) : inf, rmin = *rmin_p;
  int l = 1;
  for (int k = 1; k < L; k++)
    if (r >= ldexp(rmin, k)) l = k + 1;
  level[e] = l;
  if (resident && resident[e] != l) atomicOr(changed, 1);
}

// caller layout [K][Np] (3 arrays) -> internal element-blocked [K/32][3][Np][32] in internal order
// Through a shared tile, as k_gather_tile: each caller row (Np consecutive doubles) is read by consecutive lanes,
// each element-blocked row written by consecutive lanes.  Launch: blocks of kScatterTile threads, dynamic shared
// memory kScatterTile * Np doubles.
constexpr int kScatterTile = 128;
template <typename T>
__global__ void __launch_bounds__(kScatterTile) k_scatter_state(int K, int Np, const int *orig, const double *h,
                                                                const double *hu, const double *hv, T *Q) {
  extern __shared__ double tile[];  // [kScatterTile][Np]
  __shared__ int src_of[kScatterTile];
  const int k0 = (int)blockIdx.x * kScatterTile, n = min(kScatterTile, K - k0);
  if ((int)threadIdx.x < n) src_of[threadIdx.x] = orig[k0 + (int)threadIdx.x];
  __syncthreads();
  const double *ins[3] = {h, hu, hv};
  for (int f = 0; f < 3; f++) {
    for (int idx = (int)threadIdx.x; idx < n * Np; idx += kScatterTile) {  // row-contiguous reads: node fastest
      const int el = idx / Np, node = idx % Np;
      tile[idx] = ins[f][(size_t)src_of[el] * Np + node];
    }
    __syncthreads();
    for (int idx = (int)threadIdx.x; idx < n * Np; idx += kScatterTile) {  // coalesced writes: element fastest
      const int el = idx % n, node = idx / n;
      Q[eb_at(k0 + el, f * Np + node, 3 * Np)] = (T)tile[el * Np + node];
    }
    __syncthreads();
  }
}

// cell means of a T-typed element-blocked nodal state ([K/32][3 Np][32]) -> [K/32][3][32], wm2 = mean weights
template <typename T>
__global__ void k_cell_means(int K, int Np, const T *Q, const double *wm2, T *means) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  for (int f = 0; f < 3; f++) {
    double m = 0.0;
    for (int i = 0; i < Np; i++) m = fma(wm2[i], (double)Q[eb_at(e, f * Np + i, 3 * Np)], m);
    means[eb_at(e, f, 3)] = (T)m;
  }
}

// K1 geometry table: the metric terms and face normals K1 would derive from the
// vertices, with the same expressions.
template <typename T>
__global__ void k_geo(int K, const double *V, T *geo) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  const double X[3] = {V[e], V[K + e], V[2 * (size_t)K + e]};
  const double Y[3] = {V[3 * (size_t)K + e], V[4 * (size_t)K + e], V[5 * (size_t)K + e]};
  const double xr = 0.5 * (X[1] - X[0]), xs = 0.5 * (X[2] - X[0]), yr = 0.5 * (Y[1] - Y[0]), ys = 0.5 * (Y[2] - Y[0]);
  const double J = xr * ys - xs * yr;
  const double rJ = 1.0 / J;
  T *G = geo + eb_base(e, kGeoRows);  // element-blocked [K/32][14][32]
  G[0] = (T)(ys * rJ);
  G[kEB] = (T)(-xs * rJ);
  G[2 * kEB] = (T)(-yr * rJ);
  G[3 * kEB] = (T)(xr * rJ);
  G[4 * kEB] = (T)J;
  for (int f = 0; f < 3; f++) {
    const int f1 = f == 2 ? 0 : f + 1;
    const double dx = X[f1] - X[f], dy = Y[f1] - Y[f];
    const double len = sqrt(dx * dx + dy * dy);
    G[(5 + 3 * f) * kEB] = (T)(dy / len);
    G[(6 + 3 * f) * kEB] = (T)(-dx / len);
    G[(7 + 3 * f) * kEB] = (T)(0.5 * len * rJ);
  }
}

// Static TVB geometry of every element (P:224-253 limiter stencil): Hk = 4A / perimeter
// (level-binning geometry) and the unit vectors from the centroid to the three edge midpoints,
// with the exact expressions K2 used when it derived them per launch.
template <typename T>
__global__ void k_tvb_geo(int K, const double *V, T *tgeo) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  const double XV[3] = {V[e], V[K + e], V[2 * (size_t)K + e]};
  const double YV[3] = {V[3 * (size_t)K + e], V[4 * (size_t)K + e], V[5 * (size_t)K + e]};
  const double A = 0.5 * ((XV[1] - XV[0]) * (YV[2] - YV[0]) - (XV[2] - XV[0]) * (YV[1] - YV[0]));
  double len[3];
  for (int f = 0; f < 3; f++) {
    const double dx = XV[(f + 1) % 3] - XV[f], dy = YV[(f + 1) % 3] - YV[f];
    len[f] = sqrt(dx * dx + dy * dy);
  }
  tgeo[eb_at(e, 0, 7)] = (T)((4.0 * A) / ((len[0] + len[1]) + len[2]));  // element-blocked [K/32][7][32]
  const double bx = (XV[0] + XV[1] + XV[2]) / 3.0, by = (YV[0] + YV[1] + YV[2]) / 3.0;
  for (int i = 0; i < 3; i++) {
    const double mx = 0.5 * (XV[i] + XV[(i + 1) % 3]), my = 0.5 * (YV[i] + YV[(i + 1) % 3]);
    const double tx = mx - bx, ty = my - by;
    const double tl = sqrt(tx * tx + ty * ty);
    tgeo[eb_at(e, 1 + 2 * i, 7)] = (T)(tx / tl);
    tgeo[eb_at(e, 2 + 2 * i, 7)] = (T)(ty / tl);
  }
}

template <typename T>
__global__ void k_scatter_field(int K, int Np, const int *orig, const double *src, T *dst) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  size_t e = (size_t)orig[k];
  for (int i = 0; i < Np; i++) dst[eb_at(k, i, Np)] = (T)src[e * Np + i];  // element-blocked [K/32][Np][32]
}

// internal committed state (parity per level) -> caller layout
struct GatherParams {
  int K, Np, nlev, off[9], par[8];  // K = elements to process (owned), Kstride = array stride
  int Kstride;
  const int *orig;
  const void *Q;  // T-typed internal state
  double *h, *hu, *hv;
};
// Caller-layout read-back through a shared tile: a block reads kGatherTile consecutive internal elements' nodes
// coalesced from the element-blocked state and writes each element's Np consecutive doubles with consecutive lanes
// (the one-thread-per-element gather below scattered 8-byte stores over 32 caller rows per instruction).
constexpr int kGatherTile = 128;
template <typename T>
__global__ void __launch_bounds__(kGatherTile) k_gather_tile(const __grid_constant__ GatherParams p) {
  extern __shared__ double tile[];  // [kGatherTile][Np]
  __shared__ int par_of[kGatherTile], dst_of[kGatherTile];
  const int k0 = (int)blockIdx.x * kGatherTile, n = min(kGatherTile, p.K - k0), Np = p.Np;
  const size_t K = p.Kstride;
  if ((int)threadIdx.x < n) {
    const int k = k0 + (int)threadIdx.x;
    int c = 0;
    for (int l = 1; l < p.nlev; l++) c += (k >= p.off[l]) ? 1 : 0;
    par_of[threadIdx.x] = p.par[c];
    dst_of[threadIdx.x] = p.orig[k];
  }
  __syncthreads();
  double *outs[3] = {p.h, p.hu, p.hv};
  for (int f = 0; f < 3; f++) {
    for (int idx = (int)threadIdx.x; idx < n * Np; idx += kGatherTile) {  // coalesced reads: element fastest
      const int el = idx % n, node = idx / n, k = k0 + el;
      const T *Q = (const T *)p.Q + (size_t)par_of[el] * 3 * Np * eb_pad(K);
      tile[el * Np + node] = (double)Q[eb_at(k, f * Np + node, 3 * Np)];
    }
    __syncthreads();
    double *out = outs[f];
    for (int idx = (int)threadIdx.x; idx < n * Np; idx += kGatherTile) {  // row-contiguous writes: node fastest
      const int el = idx / Np, node = idx % Np;
      out[(size_t)dst_of[el] * Np + node] = tile[idx];
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void k_gather_state(const __grid_constant__ GatherParams p) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p.K) return;
  int c = 0;
  for (int l = 1; l < p.nlev; l++) c += (k >= p.off[l]) ? 1 : 0;
  const size_t K = p.Kstride;
  const T *Q = (const T *)p.Q + (size_t)p.par[c] * 3 * p.Np * eb_pad(K) + eb_base(k, 3 * p.Np);
  size_t e = (size_t)p.orig[k];
  for (int i = 0; i < p.Np; i++) {
    p.h[e * p.Np + i] = (double)Q[(size_t)i * kEB];
    p.hu[e * p.Np + i] = (double)Q[(size_t)(p.Np + i) * kEB];
    p.hv[e * p.Np + i] = (double)Q[(size_t)(2 * p.Np + i) * kEB];
  }
}

// mass and min h per block -> partials[2*block]
template <typename T>
__global__ void k_diag(const __grid_constant__ GatherParams p, const double *V, const double *wm2,
                       double *partials) {
  __shared__ double smass[256], smin[256];
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  double mass = 0.0, mn = 1e300;
  if (k < p.K) {
    int c = 0;
    for (int l = 1; l < p.nlev; l++) c += (k >= p.off[l]) ? 1 : 0;
    const size_t K = p.Kstride;
    const T *Q = (const T *)p.Q + (size_t)p.par[c] * 3 * p.Np * eb_pad(K) + eb_base(k, 3 * p.Np);
    double x0 = V[k], x1 = V[K + k], x2 = V[2 * K + k], y0 = V[3 * K + k], y1 = V[4 * K + k], y2 = V[5 * K + k];
    double J = 0.25 * ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0));
    double acc = 0.0;
    for (int i = 0; i < p.Np; i++) {
      double h = (double)Q[(size_t)i * kEB];
      acc += wm2[i] * h;
      mn = fmin(mn, h);
    }
    mass = 2.0 * J * acc;
  }
  smass[threadIdx.x] = mass;
  smin[threadIdx.x] = mn;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      smass[threadIdx.x] += smass[threadIdx.x + s];
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = smass[0];
    partials[2 * blockIdx.x + 1] = smin[0];
  }
}

// ------------------------------------------------------------------ context
struct Ctx;

// Exchange table of one phase (A: elements, B: element faces) and one direction.  Entries of a level
// are contiguous in the index arrays ([level][peer] order, each peer's list in the order both ranks
// agree on); the BUFFER layout is [level][peer] for receives and [peer][level] for sends, so that the
// sender's segment for (level l, receiver) starts at base[peer] + (the receiver's own counts of the
// levels below l) -- what a receiver needs to read a peer's send buffer directly (CUDA-IPC transport).
struct XTable {
  std::vector<int> cnt;   // [(L+1) * npeer]  (level 1..L)
  std::vector<int> off;   // buffer position (entries) of segment (level, peer)
  std::vector<int> loff;  // index-array range of level l: [loff[l-1], loff[l])
  std::vector<int> base;  // sends: first buffer position of peer i's block ([peer][level] layout)
  int total = 0;
  int didx = 0, ddst = -1;  // offsets of this table's entry and destination arrays in the device block
};

struct Ctx {
  std::string err;
  int N = 0, Np = 0, device = 0;
  int Kin = 0;   // elements of the mesh given to swe_create
  int K = 0;     // local elements (owned + ghosts)
  int kown = 0;  // owned elements
  int rank = 0, nranks = 1;
  double g = 9.81;
  swe_params prm;
  bool f32 = false;  // FP32 variant (swe_params.precision == 32): T = float for the state and kernels
  size_t esz = 8;    // bytes per element of the T-typed arrays
  cudaStream_t stream = 0;
  RefOps ops;
  HostMesh mesh;  // given mesh, with connectivity
  TvbGeom tvb;
  std::vector<int64_t> gid;
  std::vector<int32_t> owner;
  HaloPlan plan;  // peers / send / recv lists (given-mesh indices)
  // transport
  ncclComm_t comm = nullptr;
  std::vector<Ctx *> group;  // in-process peers (local transport), indexed by rank
  // device
  double *dQ = nullptr, *dR = nullptr, *dB = nullptr, *dV = nullptr, *dMeans = nullptr, *dUT = nullptr;
  double *dTalpha = nullptr, *dTgeo = nullptr, *dGeo = nullptr, *dAe = nullptr, *dStage = nullptr, *dInjected = nullptr, *dWm2 = nullptr;
  double *dBcaller = nullptr, *dPartials = nullptr, *dOpsG = nullptr, *dOpsGf = nullptr, *dRmin = nullptr;
  int *dK2list = nullptr;             // K2_LIST: elements K1 hands to K2 (single rank)
  unsigned int *dK2cnt = nullptr;     // [2] list lengths
  long k2u = 0;                       // list-mode updates so far (the slot of an update is k2u & 1)
  double *dGather = nullptr;             // caller-layout state for swe_get_state (allocated on first use)
  double *dSnap[2] = {nullptr, nullptr};  // swe_get_state_async snapshot buffers (allocated on first use)
  cudaStream_t ostream = nullptr;         // swe_get_state_async device->host copies
  cudaEvent_t oevG[2] = {nullptr, nullptr}, oevC[2] = {nullptr, nullptr};  // snapshot gathered / copied
  long nsnap = 0;                         // swe_get_state_async calls so far
  double *dBndStage = nullptr;           // Dirichlet boundary state, caller layout [3][Kin][Np] (A7'')
  double *dQbnd = nullptr, *dBmean = nullptr;  // ... in the internal layout, and its cell means
  bool bnd_set = false;
  long n_dirichlet = 0;                  // Dirichlet faces of the given mesh (counted at swe_create)
  double *dHk = nullptr;                 // host Hk (caller order), for the device binning
  int32_t *dLev = nullptr, *dLevRes = nullptr;  // binned levels; levels of the resident layout
  int *dFlag = nullptr;
  bool levres_ok = false;  // dLevRes holds the levels of the resident layout
  double *dXsBuf = nullptr, *dXrBuf = nullptr;
  int *dE2E = nullptr, *dTcode = nullptr, *dOrig = nullptr, *dXidx = nullptr;
  size_t capS = 0, capR = 0;  // exchange buffer capacities (T values): max over the two phases' payloads
  // phase entry lists per peer (given-mesh codes: A element, B (element << 2) | face), in the agreed order
  std::vector<std::vector<int64_t>> sendA, recvA, sendB, recvB;
  unsigned char *dDry = nullptr;
  unsigned char *dDec = nullptr;            // decision log of the update in flight (record_decisions, A26)
  std::vector<unsigned char> declog;        // host log: ndec records of Kin bytes (caller order)
  long ndec = 0;
  unsigned long long *dCounters = nullptr;
  unsigned long long *hCounters = nullptr;  // pinned
  double *hInjected = nullptr;              // pinned
  // state / schedule
  bool have_state = false, materialized = false, scheduled = false;
  bool layout_valid = false;  // internal order + static tables match c->level / c->L
  double dt = 0.0;
  double t_base = 0.0;  // simulated time carried across swe_regroup
  int L = 1;
  std::vector<int32_t> level;  // given-mesh order
  std::vector<int32_t> order;  // internal k -> given-mesh e (owned first, then ghosts)
  int off[9] = {0}, goff[9] = {0};
  XTable xs[2], xr[2];  // [phase]: 0 = A (means, dry flags; element entries), 1 = B (face traces)
  int bnd[9] = {0};      // owned level l: boundary elements [off[l-1], bnd[l]), interior [bnd[l], off[l])
  long xcount = 0;       // exchanges done (identical on every rank: the schedule is global)
  // CUDA-IPC transport (SURVEY 8(e) NVLink peer memory): every rank's exchange block is mapped by every
  // other rank; a receiver copies its segments straight out of the sender's send slot
  bool ipc = false;
  char *ipcBlock = nullptr;     // own block: header (flags, r_min words), send slots 0 and 1
  size_t ipcSlotBytes = 0;
  std::vector<char *> ipcPeer;  // [nranks]: mapped blocks of the other ranks (nullptr for self)
  std::vector<size_t> ipcPeerSlot;  // [nranks]: their send-slot sizes (ranks' send volumes differ)
  std::vector<long> ipcBaseA, ipcBaseB;  // [peer index]: the peer's send-layout base of its block for me
  long rcount = 0;              // r_min reductions done (IPC)
  cudaStream_t cstream = nullptr;          // communication stream (multi-rank overlap)
  cudaEvent_t xev[4] = {nullptr, nullptr, nullptr, nullptr};
  int kcount[9] = {0}, par[9] = {0};
  long tick_s[9] = {0}, t_e[9] = {0};
  long tick = 0;
  long n_updates = 0;
  std::vector<std::pair<int, long>> schedule;  // (level, tick offset) of one macro step
  StepParams cur;  // parameters of the update in flight
  // CUDA graphs of whole macro steps (single rank): the launch sequence repeats with period 6 after the
  // AB ramp (ring slot mod 3, Q parity mod 2), so each distinct parameter sequence is captured once
  struct StepGraph {
    std::vector<StepParams> seq;
    long kmod = 0;  // multi-rank: exchange count mod 4 at the step start (the flag values baked into the graph)
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<StepGraph> graphs;
  bool use_graphs = true;
  cudaStream_t gstream = nullptr;          // private non-blocking stream: graphs are captured and replayed here
  cudaEvent_t gev0 = nullptr, gev1 = nullptr;  // order gstream after / before the caller's stream
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev;      // (start, stop) pairs recorded this macro step
  std::vector<int> evwhich;         // kernel (0 K1, 1 K2) of each pair
  std::vector<cudaEvent_t> evpool;  // created once, reused
  size_t evnext = 0;
  double prof_ms[2] = {0, 0}, prof_bytes[2] = {0, 0};
  long prof_launch[2] = {0, 0};
  bool alloc_ok = true;

  void *dalloc(size_t bytes) {
    void *p = nullptr;
    if (bytes == 0) bytes = 8;
    if (prm.dev_alloc) {
      p = prm.dev_alloc(bytes, (void *)stream, prm.alloc_user);
    } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
      p = nullptr;
    }
    if (!p) alloc_ok = false;
    return p;
  }
  void dfree(void *p) {
    if (!p) return;
    if (prm.dev_free)
      prm.dev_free(p, (void *)stream, prm.alloc_user);
    else
      cudaFree(p);
  }
};

// sum of one counter over its kSlots (host copy)
static unsigned long long counter(const Ctx *c, int which) {
  unsigned long long s = 0;
  for (int i = 0; i < kSlots; i++) s += c->hCounters[which * kSlots + i];
  return s;
}

static int cuda_fail(Ctx *c, cudaError_t e, const char *where) {
  c->err = std::string(where) + ": " + cudaGetErrorString(e);
  return SWE_ERR_CUDA;
}
#define CK(call)                                          \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(c, _e, #call); \
  } while (0)
#define NK(call)                                                           \
  do {                                                                     \
    ncclResult_t _r = (call);                                              \
    if (_r != ncclSuccess) {                                               \
      c->err = std::string(#call) + ": " + ncclGetErrorString(_r);         \
      return SWE_ERR_NCCL;                                                 \
    }                                                                      \
  } while (0)

template <int N, typename T>
static void fill_ops(const RefOps &o, Ops<N, T> &h) {
  constexpr int Np = Ops<N>::Np;
  for (int i = 0; i < Np; i++) {
    h.wm2[i] = (T)(0.5 * o.wmean[i]);
    for (int v = 0; v < 3; v++) h.Pv[v][i] = (T)o.Pv(v, i);
    h.lam[i][0] = (T)(-0.5 * (o.r[i] + o.s[i]));
    h.lam[i][1] = (T)(0.5 * (1.0 + o.r[i]));
    h.lam[i][2] = (T)(0.5 * (1.0 + o.s[i]));
  }
}

template <int N>
static cudaError_t upload_ops(const RefOps &o) {
  if (o.Nc != Ops<N>::Nc || o.Np != Ops<N>::Np) return cudaErrorInvalidValue;  // host rule and kernel template disagree
  Ops<N> h;
  Ops<N, float> hf;
  fill_ops<N, double>(o, h);
  fill_ops<N, float>(o, hf);
  const void *syms[5] = {&c_ops1, &c_ops2, &c_ops3, &c_ops4, &c_ops5};
  const void *symfs[5] = {&c_opsf1, &c_opsf2, &c_opsf3, &c_opsf4, &c_opsf5};
  const void *sym = syms[N - 1], *symf = symfs[N - 1];
  cudaError_t e = cudaMemcpyToSymbol(sym, &h, sizeof(h));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(symf, &hf, sizeof(hf));
}

template <int N>
static std::vector<double> smem_ops(const RefOps &o) {
  using SO = SmemOps<N>;
  std::vector<double> v(SO::total, 0.0);
  for (int c = 0; c < SO::Nc; c++)
    for (int i = 0; i < SO::Np; i++) {
      v[SO::Ic + c * SO::NpP + i] = o.Ic(c, i);
      v[SO::IcDr + c * SO::NpP + i] = o.IcDr(c, i);
      v[SO::IcDs + c * SO::NpP + i] = o.IcDs(c, i);
      v[SO::PrT + c * SO::NpP + i] = o.Pr(i, c);
      v[SO::PsT + c * SO::NpP + i] = o.Ps(i, c);
      v[SO::PT + c * SO::NpP + i] = o.P(i, c);
    }
  for (int g = 0; g < 3 * SO::Ng; g++)
    for (int i = 0; i < SO::Np; i++) v[SO::LgT + g * SO::NpP + i] = o.Lg(i, g);
  for (int j = 0; j < SO::Ng; j++)
    for (int k = 0; k < SO::Nfp; k++) v[SO::Ig1 + j * SO::NfpP + k] = o.Ig1(j, k);
  // DMMA fragments (K1_MMA)
  const DMat *icops[3] = {&o.Ic, &o.IcDr, &o.IcDs}, *pops[3] = {&o.Pr, &o.Ps, &o.P};
  for (int op = 0; op < 3; op++)
    for (int ks = 0; ks < SO::NKN; ks++)
      for (int nt = 0; nt < SO::NTP; nt++)
        for (int l = 0; l < 32; l++) {
          // column j = l / 4 of n-tile nt carries point 4 (2 nt + (j & 1)) + (j >> 1): lane l of the accumulator
          // (columns 2 (l % 4) + i) then holds exactly the points 4 ks + l % 4, ks = 2 nt + i, that its projection
          // A fragments need, so no shuffles are required between the two contractions
          const int j = l / 4, pt = 4 * (2 * nt + (j & 1)) + (j >> 1), node = 4 * ks + l % 4;
          v[SO::FIc + ((op * SO::NKN + ks) * SO::NTP + nt) * 32 + l] =
              (pt < SO::Nc && node < SO::Np) ? (*icops[op])(pt, node) : 0.0;
        }
  for (int op = 0; op < 3; op++)
    for (int ks = 0; ks < SO::NKP; ks++)
      for (int nt = 0; nt < SO::NTN; nt++)
        for (int l = 0; l < 32; l++) {
          const int node = 8 * nt + l / 4, pt = 4 * ks + l % 4;
          v[SO::FP + ((op * SO::NKP + ks) * SO::NTN + nt) * 32 + l] =
              (pt < SO::Nc && node < SO::Np) ? (*pops[op])(node, pt) : 0.0;
        }
  // lift fragments (k_rhs_update_mma2)
  v.resize(SO::total2, 0.0);
  for (int ks = 0; ks < SO::NKL / 4; ks++)
    for (int nt = 0; nt < SO::NTN; nt++)
      for (int l = 0; l < 32; l++) {
        const int node = 8 * nt + l / 4, gp = 4 * ks + l % 4;
        v[SO::FL + (ks * SO::NTN + nt) * 32 + l] = (node < SO::Np && gp < 3 * SO::Ng) ? -o.Lg(node, gp) : 0.0;
      }
  return v;
}
static std::vector<double> smem_ops_any(const RefOps &o) {
  switch (o.N) {
    case 1: return smem_ops<1>(o);
    case 2: return smem_ops<2>(o);
    case 3: return smem_ops<3>(o);
    case 4: return smem_ops<4>(o);
    case 5: return smem_ops<5>(o);
  }
  return {};
}

static cudaError_t upload_ops_any(const RefOps &o) {
  switch (o.N) {
    case 1: return upload_ops<1>(o);
    case 2: return upload_ops<2>(o);
    case 3: return upload_ops<3>(o);
    case 4: return upload_ops<4>(o);
    case 5: return upload_ops<5>(o);
  }
  return cudaErrorInvalidValue;
}

// Launch with programmatic stream serialization (K1_PDL): the kernel may start while the previous kernel in the
// stream drains; it calls griddep_wait() before reading anything that kernel wrote.
template <typename P>
static void launch_pdl(void (*kern)(P), int grid, int block, size_t smem, cudaStream_t s, const P &p) {
#if K1_PDL
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
#else
  kern<<<grid, block, smem, s>>>(p);
#endif
}

template <int N, bool INIT, typename T>
static void launch_k1(const StepParamsT<T> &p, cudaStream_t s) {
  int n = p.k1 - p.k0;
  if (n <= 0) return;
  size_t smem = INIT ? 0 : (size_t)k1_ops_bytes<N, T>();
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_rhs_update<N, INIT, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = (n + K1_BLOCK - 1) / K1_BLOCK;
  if constexpr (!INIT && N >= K1_MMA_MIN_N && sizeof(T) == 8) {  // FP64 tensor path: volume term and lift on DMMA (FP32: scalar path)
    const size_t smem2 = mma2_smem_bytes<N>();
    if (smem2 > 48 * 1024)
      cudaFuncSetAttribute(k_rhs_update_mma2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    constexpr int bs = mma2_block<N>();
    int grid = (n + bs - 1) / bs;
    if constexpr (N >= K1_MMA2_PERSIST) {  // persistent grid: SMs x resident blocks
      static int resident[6] = {0, 0, 0, 0, 0, 0};  // per order (one device per process)
      if (!resident[N]) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rhs_update_mma2<N>, bs, smem2);
        resident[N] = std::max(1, sms * per_sm);
      }
      grid = std::min(grid, resident[N]);
    }
    launch_pdl(k_rhs_update_mma2<N>, grid, bs, smem2, s, reinterpret_cast<const StepParams &>(p));
    return;
  }
#if K1_CARVEOUT >= 0
  // shared-memory carveout hint (percent of the maximum): the blocks need ~17 KB per SM, the rest is L1 for the
  // own-state re-reads and the neighbour gathers
  cudaFuncSetAttribute(k_rhs_update<N, INIT, T>, cudaFuncAttributePreferredSharedMemoryCarveout, K1_CARVEOUT);
#endif
  if (INIT)
    k_rhs_update<N, INIT, T><<<grid, K1_BLOCK, smem, s>>>(p);
  else
    launch_pdl(k_rhs_update<N, INIT, T>, grid, K1_BLOCK, smem, s, p);
}
template <int N, typename T>
static void launch_k2(const StepParamsT<T> &p, cudaStream_t s) {
  int n = p.k1 - p.k0;
  if (n <= 0) return;
#if K2_CARVEOUT >= 0
  cudaFuncSetAttribute(k_tvb<N, T>, cudaFuncAttributePreferredSharedMemoryCarveout, K2_CARVEOUT);
#endif
  if (p.k2list) {  // K2_LIST: a grid-stride pass over the list K1 built (its length is known on the device only)
    launch_pdl(k_tvb_list<N, T>, std::min((n + K2_BLOCK - 1) / K2_BLOCK, K2_LIST_GRID), K2_BLOCK, 0, s, p);
    return;
  }
  launch_pdl(k_tvb<N, T>, (n + K2_BLOCK - 1) / K2_BLOCK, K2_BLOCK, 0, s, p);
}
template <typename T>
static void launch_t(int which, bool init, int N, const StepParamsT<T> &p, cudaStream_t s) {
  if (which == 0) {
    switch (N) {
      case 1: init ? launch_k1<1, true, T>(p, s) : launch_k1<1, false, T>(p, s); break;
      case 2: init ? launch_k1<2, true, T>(p, s) : launch_k1<2, false, T>(p, s); break;
      case 3: init ? launch_k1<3, true, T>(p, s) : launch_k1<3, false, T>(p, s); break;
      case 4: init ? launch_k1<4, true, T>(p, s) : launch_k1<4, false, T>(p, s); break;
      case 5: init ? launch_k1<5, true, T>(p, s) : launch_k1<5, false, T>(p, s); break;
    }
  } else {
    switch (N) {
      case 1: launch_k2<1, T>(p, s); break;
      case 2: launch_k2<2, T>(p, s); break;
      case 3: launch_k2<3, T>(p, s); break;
      case 4: launch_k2<4, T>(p, s); break;
      case 5: launch_k2<5, T>(p, s); break;
    }
  }
}

// The host builds every update's parameters in double; the FP32 variant gets a
// copy with float scalars and its float-typed device arrays.
static StepParamsT<float> to_f32(const StepParams &d) {
  StepParamsT<float> f;
  std::memset(&f, 0, sizeof(f));
  f.k0 = d.k0, f.k1 = d.k1, f.K = d.K;
  f.Q = (float *)d.Q, f.R = (float *)d.R, f.B = (const float *)d.B, f.V = d.V, f.E2E = d.E2E, f.tcode = d.tcode;
  f.talpha = (const float *)d.talpha, f.geo = (const float *)d.geo, f.tgeo = (const float *)d.tgeo;
  f.means = (float *)d.means, f.dry = d.dry, f.UT = (float *)d.UT;
  f.own_par = d.own_par, f.write_par = d.write_par, f.write_slot = d.write_slot, f.nab = d.nab;
  for (int i = 0; i < 3; i++) f.ab_slot[i] = d.ab_slot[i], f.ab[i] = (float)d.ab[i];
  f.nlev = d.nlev, f.kown = d.kown;
  for (int l = 0; l <= 8; l++) f.off[l] = d.off[l], f.goff[l] = d.goff[l];
  for (int l = 0; l < 8; l++) {
    f.lev[l].par = d.lev[l].par, f.lev[l].dense = d.lev[l].dense, f.lev[l].nterm = d.lev[l].nterm;
    for (int s = 0; s < 3; s++) f.lev[l].slot[s] = d.lev[l].slot[s], f.lev[l].beta[s] = (float)d.lev[l].beta[s];
  }
  f.g = (float)d.g, f.h0 = (float)d.h0, f.eps = (float)d.eps, f.e4 = (float)d.e4;
  f.tvb_M = (float)d.tvb_M, f.tvb_nu = (float)d.tvb_nu, f.h_char = (float)d.h_char;
  f.use_pp = d.use_pp, f.use_tvb = d.use_tvb;
  f.counters = d.counters, f.injected = d.injected, f.opsG = (const float *)d.opsG, f.dec = d.dec;
  f.Qbnd = (const float *)d.Qbnd, f.bmean = (const float *)d.bmean;
  f.k2list = d.k2list, f.k2cnt = d.k2cnt, f.k2slot = d.k2slot;
  return f;
}

static void launch(int which, bool init, int N, const StepParams &p, cudaStream_t s, bool f32) {
  if (f32)
    launch_t<float>(which, init, N, to_f32(p), s);
  else
    launch_t<double>(which, init, N, p, s);
}

// algorithmic bytes per element update
static double k1_bytes(int N, int nab, bool tvb, size_t esz) {
  int Np = (N + 1) * (N + 2) / 2, Nfp = N + 1;
  double d = 3 * Np /*Q r*/ + 3 * Np /*Q w*/ + 3 * Np /*R w*/ + 3 * Np * (nab - 1) /*R r*/ + Np /*B*/ +
             9 * Nfp /*nbr Q faces*/ + 3 * Nfp /*nbr B faces*/ + 14 /*geometry table*/ + 3 /*means w*/ + (tvb ? 9 : 0);
  return (double)esz * d + 12.0 /*E2E*/ + 1.0 /*dry flag*/;
}
// own means, 3 neighbours' means, P1 midpoint data, alphas, static geometry (tgeo); E2E, pair code, 4 dry flags
static double k2_bytes(size_t esz) { return (double)esz * (3 + 9 + 9 + 6 + 7) + 12.0 + 4.0 + 4.0; }

static StepParams base_params(Ctx *c) {
  StepParams p;
  std::memset(&p, 0, sizeof(p));
  p.K = c->K;
  p.Q = c->dQ;
  p.R = c->dR;
  p.B = c->dB;
  p.V = c->dV;
  p.E2E = c->dE2E;
  p.tcode = c->dTcode;
  p.talpha = c->dTalpha;
  p.tgeo = c->dTgeo;
  p.geo = c->dGeo;
  p.means = c->dMeans;
  p.dry = c->dDry;
  p.UT = c->dUT;
  p.g = c->g;
  p.h0 = c->prm.h0;
  p.eps = c->prm.eps;
  double e2 = c->prm.eps_u * c->prm.eps_u;
  p.e4 = e2 * e2;
  p.tvb_M = c->prm.tvb_M;
  p.tvb_nu = c->prm.tvb_nu;
  p.h_char = c->prm.h_char;
  p.use_pp = c->prm.use_pp;
  p.use_tvb = c->prm.use_tvb;
  p.counters = c->dCounters;
  p.injected = c->dInjected;
  p.dec = c->dDec;
  p.Qbnd = c->dQbnd;
  p.bmean = c->dBmean;
  p.opsG = c->f32 ? c->dOpsGf : c->dOpsG;
  p.nlev = c->L;
  p.kown = c->kown;
  for (int l = 0; l <= 8; l++) {
    p.off[l] = c->off[l];
    p.goff[l] = c->goff[l];
  }
  return p;
}

static void build_entry_lists(Ctx *c);
static int alloc_state(Ctx *c) {
  if (c->dQ) return SWE_OK;
  size_t K = c->K, Np = c->Np, Kin = c->Kin;
  const size_t es = c->esz;  // T-typed arrays
  const size_t Kp = eb_pad(K);  // element-blocked arrays: whole blocks of kEB elements
  c->dQ = (double *)c->dalloc(es * 2 * 3 * Np * Kp);
  c->dR = (double *)c->dalloc(es * 3 * 3 * Np * Kp);
  c->dB = (double *)c->dalloc(es * Np * Kp);
  c->dV = (double *)c->dalloc(sizeof(double) * 6 * K);
  c->dMeans = (double *)c->dalloc(es * 3 * Kp);
  c->dUT = (double *)c->dalloc(es * 9 * Kp);
  c->dTalpha = (double *)c->dalloc(es * 6 * Kp);
  c->dTgeo = (double *)c->dalloc(es * 7 * Kp);
  c->dGeo = (double *)c->dalloc(es * kGeoRows * Kp);
  c->dAe = (double *)c->dalloc(sizeof(double) * Kin);
  c->dStage = (double *)c->dalloc(sizeof(double) * 3 * Np * Kin);
  c->dE2E = (int *)c->dalloc(sizeof(int) * 3 * Kp);
  c->dTcode = (int *)c->dalloc(sizeof(int) * K);
  c->dOrig = (int *)c->dalloc(sizeof(int) * K);
  c->dDry = (unsigned char *)c->dalloc((size_t)4 * K);  // [K][4] dry words (kernels.cuh store_dry)
  if (c->prm.record_decisions) c->dDec = (unsigned char *)c->dalloc(K);
  c->dPartials = (double *)c->dalloc(sizeof(double) * 2 * ((K + 255) / 256));
  c->dRmin = (double *)c->dalloc(sizeof(double));
  c->dK2list = (int *)c->dalloc(sizeof(int) * K);
  c->dK2cnt = (unsigned int *)c->dalloc(sizeof(unsigned int) * 2);
  // exchange entry lists (level-independent) and buffer capacities
  build_entry_lists(c);
  size_t nsA = 0, nrA = 0, nsB = 0, nrB = 0;
  for (auto &v : c->sendA) nsA += v.size();
  for (auto &v : c->recvA) nrA += v.size();
  for (auto &v : c->sendB) nsB += v.size();
  for (auto &v : c->recvB) nrB += v.size();
  const size_t Nfp = (size_t)c->N + 1;
  c->capS = std::max((size_t)4 * nsA, 6 * Nfp * nsB) + 8;
  c->capR = std::max((size_t)4 * nrA, 6 * Nfp * nrB) + 8;
  c->dXsBuf = (double *)c->dalloc(es * c->capS);
  c->dXrBuf = (double *)c->dalloc(es * c->capR);
  if (!c->alloc_ok) {
    c->err = "device allocation failed";
    return SWE_ERR_NOMEM;
  }
  return SWE_OK;
}

// ------------------------------------------------------------------ halo exchange tables
// Entry lists of both phases, per peer, in the order both ranks derive independently:
//   phase A: the halo plan's element lists (global-id order);
//   phase B: the faces of those elements that border the other rank -- sends: faces of my boundary
//            elements whose neighbour the peer owns; receives: faces of the peer's ghosts whose neighbour
//            I own -- per element ordered by the global id of the element across the face.
static void face_entries(const Ctx *c, const std::vector<int32_t> &elems, int other, std::vector<int64_t> &out) {
  out.clear();
  for (int e : elems) {
    int fs[3], n = 0;
    for (int f = 0; f < 3; f++) {
      const int nb = c->mesh.etoe[(size_t)3 * e + f];
      if (nb != e && c->owner[nb] == other) fs[n++] = f;
    }
    std::sort(fs, fs + n, [&](int a, int b) {
      const int64_t ga = c->gid[c->mesh.etoe[(size_t)3 * e + a]], gb = c->gid[c->mesh.etoe[(size_t)3 * e + b]];
      return ga != gb ? ga < gb : a < b;
    });
    for (int j = 0; j < n; j++) out.push_back(((int64_t)e << 2) | fs[j]);
  }
}
static void build_entry_lists(Ctx *c) {
  const size_t np = c->plan.peers.size();
  c->sendA.assign(np, {});
  c->recvA.assign(np, {});
  c->sendB.assign(np, {});
  c->recvB.assign(np, {});
  for (size_t i = 0; i < np; i++) {
    c->sendA[i].assign(c->plan.send[i].begin(), c->plan.send[i].end());
    c->recvA[i].assign(c->plan.recv[i].begin(), c->plan.recv[i].end());
    face_entries(c, c->plan.send[i], c->plan.peers[i], c->sendB[i]);
    face_entries(c, c->plan.recv[i], c->rank, c->recvB[i]);
  }
}

// Table of one phase and direction for the current internal order (inv: given -> internal index).
// Appends the entry array (internal codes, [level][peer] order) and, for sends, the destination array to
// `blk`, recording their offsets in t.didx / t.ddst.
static void build_xtable(Ctx *c, const std::vector<std::vector<int64_t>> &lists, bool faces, bool send,
                         const std::vector<int32_t> &inv, XTable &t, std::vector<int> &blk) {
  const int np = (int)lists.size(), L = c->L, NP = std::max(np, 1);
  auto elem = [&](int64_t code) { return (int)(faces ? code >> 2 : code); };
  t.cnt.assign((size_t)(L + 1) * NP, 0);
  t.off.assign((size_t)(L + 1) * NP, 0);
  t.loff.assign(L + 2, 0);
  t.base.assign(np + 1, 0);
  for (int i = 0; i < np; i++)
    for (int64_t code : lists[i]) t.cnt[(size_t)c->level[elem(code)] * NP + i]++;
  for (int i = 0; i < np; i++) t.base[i + 1] = t.base[i] + (int)lists[i].size();
  if (send) {
    for (int i = 0; i < np; i++) {
      int o = t.base[i];
      for (int l = 1; l <= L; l++) {
        t.off[(size_t)l * NP + i] = o;
        o += t.cnt[(size_t)l * NP + i];
      }
    }
  } else {
    int o = 0;
    for (int l = 1; l <= L; l++)
      for (int i = 0; i < np; i++) {
        t.off[(size_t)l * NP + i] = o;
        o += t.cnt[(size_t)l * NP + i];
      }
  }
  std::vector<int> idx, dst;
  for (int l = 1; l <= L; l++) {
    t.loff[l - 1] = (int)idx.size();
    for (int i = 0; i < np; i++) {
      int j = 0;
      for (int64_t code : lists[i]) {
        const int e = elem(code);
        if (c->level[e] != l) continue;
        idx.push_back(faces ? (inv[e] << 2) | (int)(code & 3) : inv[e]);
        dst.push_back(t.off[(size_t)l * NP + i] + j++);
      }
    }
  }
  t.loff[L] = (int)idx.size();
  t.total = (int)idx.size();
  t.didx = (int)blk.size();
  blk.insert(blk.end(), idx.begin(), idx.end());
  t.ddst = -1;
  if (send) {
    t.ddst = (int)blk.size();
    blk.insert(blk.end(), dst.begin(), dst.end());
  }
}

// ------------------------------------------------------------------ halo exchange (pack / transfer / unpack)
static int payload(Ctx *c, int phase) { return phase == 0 ? 4 : 6 * (c->N + 1); }
constexpr size_t kIpcHdr = 256;  // IPC block header: u64 flag[2] @0, u64 rflag[2] @16, double rmin[2] @32

// send buffer of exchange k: the IPC block's slot (k mod 2) -- a peer may still be reading slot k-1 -- or
// the plain device buffer (NCCL, in-process)
static char *send_buf(Ctx *c, long k) {
  if (c->ipc) return c->ipcBlock + kIpcHdr + (size_t)(k & 1) * c->ipcSlotBytes;
  return (char *)c->dXsBuf;
}

static void halo_launch(Ctx *c, bool pack, int phase, int a, int b, int par, int slot, cudaStream_t s, char *buf,
                        const XTable &t) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    HaloParamsT<T> h;
    std::memset(&h, 0, sizeof(h));
    h.n = b - a;
    h.K = c->K;
    h.N = c->N;
    h.Np = c->Np;
    h.Nfp = c->N + 1;
    h.phase = phase;
    h.par = par;
    h.slot = slot;
    h.idx = c->dXidx + t.didx + a;
    h.dst = pack ? c->dXidx + t.ddst + a : nullptr;
    h.buf = pack ? (T *)buf : (T *)buf + (size_t)payload(c, phase) * a;
    h.Q = (T *)c->dQ;
    h.R = (T *)c->dR;
    h.means = (T *)c->dMeans;
    h.dry = c->dDry;
    h.kown = c->kown;
    h.E2E = c->dE2E;
    if (pack)
      k_halo_pack<T><<<(h.n + 127) / 128, 128, 0, s>>>(h);
    else
      k_halo_unpack<T><<<(h.n + 127) / 128, 128, 0, s>>>(h);
  };
  if (c->f32)
    run(float{});
  else
    run(double{});
}

// lvl = 0: all levels (initial exchange), else one level
static int xpack(Ctx *c, int phase, int lvl, int par, int slot, cudaStream_t s, long k) {
  if (c->plan.peers.empty()) return SWE_OK;
  const XTable &t = c->xs[phase];
  int a = lvl == 0 ? 0 : t.loff[lvl - 1], b = lvl == 0 ? t.total : t.loff[lvl];
  if (b <= a) return SWE_OK;
  halo_launch(c, true, phase, a, b, par, slot, s, send_buf(c, k), t);
  CK(cudaGetLastError());
  return SWE_OK;
}

static int xunpack(Ctx *c, int phase, int lvl, int par, int slot, cudaStream_t s) {
  if (c->plan.peers.empty()) return SWE_OK;
  const XTable &t = c->xr[phase];
  int a = lvl == 0 ? 0 : t.loff[lvl - 1], b = lvl == 0 ? t.total : t.loff[lvl];
  if (b <= a) return SWE_OK;
  halo_launch(c, false, phase, a, b, par, slot, s, (char *)c->dXrBuf, t);
  CK(cudaGetLastError());
  return SWE_OK;
}

// ---- stream memory operations (driver API, resolved at run time: the library does not link libcuda)
typedef CUresult (*PfnWait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PfnWrite64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static PfnWait64 g_wait64 = nullptr;
static PfnWrite64 g_write64 = nullptr;
static unsigned g_wait_flush = 0;
static int memops_init(Ctx *c) {
  if (g_wait64 && g_write64) return SWE_OK;
  cudaDriverEntryPointQueryResult q1, q2;
  void *f1 = nullptr, *f2 = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f1, cudaEnableDefault, &q1) != cudaSuccess || !f1 ||
      cudaGetDriverEntryPoint("cuStreamWriteValue64", &f2, cudaEnableDefault, &q2) != cudaSuccess || !f2) {
    c->err = "stream memory operations (cuStreamWaitValue64) unavailable";
    return SWE_ERR_CUDA;
  }
  int flush = 0;
  cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, c->device);
  g_wait_flush = flush ? (unsigned)CU_STREAM_WAIT_VALUE_FLUSH : 0u;
  g_wait64 = (PfnWait64)f1;
  g_write64 = (PfnWrite64)f2;
  return SWE_OK;
}
// flag value of exchange k in the parity word k mod 2.  A rank writes value(k+2) into that word only after
// it has waited for every peer's value(k+1), which each peer writes after its own wait on value(k) has
// passed: an equality wait can therefore never miss its value, and it only needs value(k) != value(k-2).
// Values cycle with period 4, so a captured macro step (2 exchanges per update, 2 (2^L - 1) per step) replays
// with the same values every other step (CUDA graphs, graph_step).
static cuuint64_t flag_value(long k) { return (cuuint64_t)(k & 3) + 1; }

// transfer of exchange k (NCCL point-to-point, in-process peers, or CUDA IPC), enqueued on stream s
static int xtransfer(Ctx *c, int phase, int lvl, cudaStream_t s, long k) {
  const int np = (int)c->plan.peers.size();
  if (np == 0) return SWE_OK;
  const int P = payload(c, phase);
  const XTable &xs = c->xs[phase], &xr = c->xr[phase];
  const int l0 = lvl == 0 ? 1 : lvl, l1 = lvl == 0 ? c->L : lvl;
  if (c->ipc) {
    const int sl = (int)(k & 1);
    const cuuint64_t v = flag_value(k);
    if (g_write64((CUstream)s, (CUdeviceptr)(c->ipcBlock + 8 * sl), v, 0) != CUDA_SUCCESS) {
      c->err = "cuStreamWriteValue64 failed";
      return SWE_ERR_CUDA;
    }
    for (int i = 0; i < np; i++) {
      char *pb = c->ipcPeer[c->plan.peers[i]];
      if (g_wait64((CUstream)s, (CUdeviceptr)(pb + 8 * sl), v, CU_STREAM_WAIT_VALUE_EQ | g_wait_flush) !=
          CUDA_SUCCESS) {
        c->err = "cuStreamWaitValue64 failed";
        return SWE_ERR_CUDA;
      }
      const char *src = pb + kIpcHdr + (size_t)sl * c->ipcPeerSlot[c->plan.peers[i]];
      long so = phase == 0 ? c->ipcBaseA[i] : c->ipcBaseB[i];
      for (int l = 1; l <= c->L; l++) {
        const int rc = xr.cnt[(size_t)l * np + i];
        if (l >= l0 && l <= l1 && rc > 0)
          CK(cudaMemcpyAsync((char *)c->dXrBuf + c->esz * P * xr.off[(size_t)l * np + i], src + c->esz * P * so,
                             c->esz * P * rc, cudaMemcpyDeviceToDevice, s));
        so += rc;
      }
    }
    return SWE_OK;
  }
  if (c->comm) {
    NK(ncclGroupStart());
    for (int i = 0; i < np; i++) {
      for (int l = l0; l <= l1; l++) {
        int so = xs.off[(size_t)l * np + i], sc = xs.cnt[(size_t)l * np + i];
        int ro = xr.off[(size_t)l * np + i], rc = xr.cnt[(size_t)l * np + i];
        const ncclDataType_t dt = c->f32 ? ncclFloat : ncclDouble;
        char *sb = (char *)c->dXsBuf, *rb = (char *)c->dXrBuf;
        if (sc > 0) NK(ncclSend(sb + c->esz * P * so, (size_t)P * sc, dt, c->plan.peers[i], c->comm, s));
        if (rc > 0) NK(ncclRecv(rb + c->esz * P * ro, (size_t)P * rc, dt, c->plan.peers[i], c->comm, s));
      }
    }
    NK(ncclGroupEnd());
    return SWE_OK;
  }
  if (!c->group.empty()) {  // in-process peers on one device: copy out of the peer's send buffer
    for (int i = 0; i < np; i++) {
      Ctx *q = c->group[c->plan.peers[i]];
      if (!q) {
        c->err = "in-process group member destroyed";
        return SWE_ERR_STATE;
      }
      int qi = -1;
      for (size_t j = 0; j < q->plan.peers.size(); j++)
        if (q->plan.peers[j] == c->rank) qi = (int)j;
      if (qi < 0) {
        c->err = "halo plan mismatch between in-process peers";
        return SWE_ERR_STATE;
      }
      const int qnp = (int)q->plan.peers.size();
      const XTable &qs = q->xs[phase];
      for (int l = l0; l <= l1; l++) {
        int ro = xr.off[(size_t)l * np + i], rc = xr.cnt[(size_t)l * np + i];
        int so = qs.off[(size_t)l * qnp + qi], sc = qs.cnt[(size_t)l * qnp + qi];
        if (rc != sc) {
          c->err = "halo exchange size mismatch";
          return SWE_ERR_STATE;
        }
        if (rc > 0)
          CK(cudaMemcpyAsync((char *)c->dXrBuf + c->esz * P * ro, (char *)q->dXsBuf + c->esz * P * so, c->esz * P * rc,
                             cudaMemcpyDeviceToDevice, s));
      }
    }
    return SWE_OK;
  }
  c->err = "ranks > 1 without a transport (swe_ipc_open, nccl_id, or swe_link_group)";
  return SWE_ERR_NCCL;
}

// Element order for a subset: level-major, Morton within a level (owned elements).
static void order_subset(const HostMesh &m, const std::vector<int32_t> &levels, const std::vector<int32_t> &subset,
                         std::vector<int32_t> &out) {
  std::vector<int32_t> all;
  element_order(m, levels.data(), all);  // global level-major Morton order
  std::vector<char> in(m.K, 0);
  for (int e : subset) in[e] = 1;
  out.clear();
  for (int e : all)
    if (in[e]) out.push_back(e);
}

// Build the internal order for `levels` (given-mesh order), upload static data,
// scatter the staged unlimited state, reset the MRAB schedule.  The initial
// limiting (Alg. 2 line 1) is applied by init_limit_* (group-aware).
static int materialize_state(Ctx *c);
static void clear_graphs(Ctx *c);
static int materialize(Ctx *c, const std::vector<int32_t> &levels, int L) {
  const int K = c->K;
  // The layout (internal order, connectivity, geometry, exchange tables) depends only on the
  // levels: a new state that bins to the resident levels reuses it and only scatters the state.
  if (c->layout_valid && c->L == L && c->level == levels) return materialize_state(c);
  c->layout_valid = false;
  clear_graphs(c);
  c->level = levels;
  c->L = L;
  std::vector<int32_t> owned_sorted, ghosts_sorted;
  order_subset(c->mesh, levels, c->plan.owned, owned_sorted);
  // boundary-first within each level (SURVEY 8(e) overlap): elements with a ghost neighbour (the phase-A
  // send lists) lead their level, so a level update can launch them first and exchange their results
  // while the interior elements compute.  Single rank: no boundary, order unchanged.
  std::vector<char> isb(c->Kin, 0);
  for (auto &lst : c->plan.send)
    for (int e : lst) isb[e] = 1;
  std::stable_sort(owned_sorted.begin(), owned_sorted.end(), [&](int a, int b) {
    if (levels[a] != levels[b]) return levels[a] < levels[b];
    return isb[a] > isb[b];
  });
  ghosts_sorted = c->plan.ghosts;
  std::stable_sort(ghosts_sorted.begin(), ghosts_sorted.end(), [&](int a, int b) {
    if (levels[a] != levels[b]) return levels[a] < levels[b];
    return c->gid[a] < c->gid[b];
  });
  c->order = owned_sorted;
  c->order.insert(c->order.end(), ghosts_sorted.begin(), ghosts_sorted.end());
  if ((int)c->order.size() != K) {
    c->err = "local element count mismatch";
    return SWE_ERR_STATE;
  }
  for (int k = 1; k < c->kown; k++)
    if (levels[c->order[k]] < levels[c->order[k - 1]]) {
      c->err = "internal element order is not level-major";
      return SWE_ERR_SCHEDULE;
    }
  std::vector<int32_t> inv(c->Kin, -1);
  for (int k = 0; k < K; k++) inv[c->order[k]] = k;
  // level offsets (owned, then ghosts)
  for (int l = 0; l <= 8; l++) {
    c->off[l] = c->kown;
    c->goff[l] = K;
  }
  {
    std::vector<int> co(10, 0), cg(10, 0);
    for (int k = 0; k < c->kown; k++) co[levels[c->order[k]]]++;
    for (int k = c->kown; k < K; k++) cg[levels[c->order[k]]]++;
    int ao = 0, ag = c->kown;
    for (int l = 1; l <= L; l++) {
      c->off[l - 1] = ao;
      c->goff[l - 1] = ag;
      ao += co[l];
      ag += cg[l];
    }
    for (int l = 1; l <= 8; l++) {
      int k = c->off[l - 1];
      const int k1 = l <= L ? c->off[l] : c->kown;
      while (k < k1 && isb[c->order[k]]) k++;
      c->bnd[l] = k;
    }
  }
  // E2E and the TVB alphas are element-blocked ([K/32][rows][32], kernels.cuh), V and TC are [rows][K]
  std::vector<double> V((size_t)6 * K, 0.0), TA((size_t)6 * eb_pad(K), 0.0);
  std::vector<int> E2E((size_t)3 * eb_pad(K), 0), TC(K, 0);
  for (int k = 0; k < K; k++) {
    int e = c->order[k];
    const int32_t *v = &c->mesh.etov[(size_t)3 * e];
    for (int j = 0; j < 3; j++) {
      V[(size_t)j * K + k] = c->mesh.vx[v[j]];
      V[(size_t)(3 + j) * K + k] = c->mesh.vy[v[j]];
    }
    int code = 0;
    for (int f = 0; f < 3; f++) {
      int n = c->mesh.etoe[(size_t)3 * e + f], nf = c->mesh.etof[(size_t)3 * e + f];
      if (k < c->kown) {
        if (inv[n] < 0) {
          c->err = "owned element with a neighbour outside the local set";
          return SWE_ERR_MESH;
        }
        // boundary faces are self references (n == e) with face code f for a reflective wall, 3 for a
        // transmissive outflow face (A7') and (f + 1) mod 3 for a Dirichlet face (A7'')
        const int tag = (n == e && nf == f) ? c->mesh.bc[(size_t)3 * e + f] : 0;
        E2E[eb_at(k, f, 3)] = (inv[n] << 2) | (tag == 1 ? 3 : (tag == 2 ? (f + 1) % 3 : nf));
      } else {  // ghosts are never launched; their rows name their local neighbours (halo unpack A uses them)
        E2E[eb_at(k, f, 3)] = (n != e && inv[n] >= 0) ? (inv[n] << 2) | nf : (k << 2) | f;
      }
      size_t s = (size_t)3 * e + f;
      code |= (c->tvb.pj[s] & 3) << (4 * f);
      code |= (c->tvb.pk[s] & 3) << (4 * f + 2);
      TA[eb_at(k, 2 * f, 6)] = c->tvb.aj[s];
      TA[eb_at(k, 2 * f + 1, 6)] = c->tvb.ak[s];
    }
    TC[k] = code;
  }
  std::vector<int> xblk;
  build_xtable(c, c->sendA, false, true, inv, c->xs[0], xblk);
  build_xtable(c, c->recvA, false, false, inv, c->xr[0], xblk);
  build_xtable(c, c->sendB, true, true, inv, c->xs[1], xblk);
  build_xtable(c, c->recvB, true, false, inv, c->xr[1], xblk);
  c->dfree(c->dXidx);
  c->dXidx = (int *)c->dalloc(sizeof(int) * std::max<size_t>(xblk.size(), 1));
  if (!c->dXidx) {
    c->alloc_ok = true;
    c->err = "device allocation failed (exchange tables)";
    return SWE_ERR_NOMEM;
  }
  CK(cudaMemcpyAsync(c->dV, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, c->stream));
  std::vector<float> TAf;
  if (c->f32) {
    TAf.assign(TA.begin(), TA.end());
    CK(cudaMemcpyAsync(c->dTalpha, TAf.data(), sizeof(float) * TAf.size(), cudaMemcpyHostToDevice, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->dTalpha, TA.data(), sizeof(double) * TA.size(), cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaMemcpyAsync(c->dE2E, E2E.data(), sizeof(int) * E2E.size(), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dTcode, TC.data(), sizeof(int) * TC.size(), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dOrig, c->order.data(), sizeof(int) * K, cudaMemcpyHostToDevice, c->stream));
  if (!xblk.empty())
    CK(cudaMemcpyAsync(c->dXidx, xblk.data(), sizeof(int) * xblk.size(), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));  // host vectors above are released on return
  int nb = (K + 127) / 128;
  if (c->f32) {
    k_scatter_field<float><<<nb, 128, 0, c->stream>>>(K, c->Np, c->dOrig, c->dBcaller, (float *)c->dB);
    k_tvb_geo<float><<<nb, 128, 0, c->stream>>>(K, c->dV, (float *)c->dTgeo);
    k_geo<float><<<nb, 128, 0, c->stream>>>(K, c->dV, (float *)c->dGeo);
  } else {
    k_scatter_field<double><<<nb, 128, 0, c->stream>>>(K, c->Np, c->dOrig, c->dBcaller, c->dB);
    k_tvb_geo<double><<<nb, 128, 0, c->stream>>>(K, c->dV, c->dTgeo);
    k_geo<double><<<nb, 128, 0, c->stream>>>(K, c->dV, c->dGeo);
  }
  CK(cudaGetLastError());
  c->layout_valid = true;
  return materialize_state(c);
}

// Dirichlet boundary state (A7''): staged caller layout -> internal layout + cell means
static int scatter_bnd(Ctx *c) {
  if (!c->bnd_set || !c->layout_valid) return SWE_OK;
  const int K = c->K, nb = (K + 127) / 128;
  const size_t KNp = (size_t)c->Kin * c->Np;
  double *st = c->dBndStage;
  if (c->f32) {
    k_scatter_state<float><<<(K + kScatterTile - 1) / kScatterTile, kScatterTile, sizeof(double) * kScatterTile * c->Np, c->stream>>>(K, c->Np, c->dOrig, st, st + KNp, st + 2 * KNp, (float *)c->dQbnd);
    k_cell_means<float><<<nb, 128, 0, c->stream>>>(K, c->Np, (const float *)c->dQbnd, c->dWm2, (float *)c->dBmean);
  } else {
    k_scatter_state<double><<<(K + kScatterTile - 1) / kScatterTile, kScatterTile, sizeof(double) * kScatterTile * c->Np, c->stream>>>(K, c->Np, c->dOrig, st, st + KNp, st + 2 * KNp, c->dQbnd);
    k_cell_means<double><<<nb, 128, 0, c->stream>>>(K, c->Np, c->dQbnd, c->dWm2, c->dBmean);
  }
  CK(cudaGetLastError());
  return SWE_OK;
}

// Dirichlet faces present but no boundary state given
static int check_bnd(Ctx *c) {
  if (c->bnd_set || c->n_dirichlet == 0) return SWE_OK;
  c->err = "the mesh has Dirichlet faces (vbc = 2) but swe_set_boundary_state was not called";
  return SWE_ERR_STATE;
}

// State part of materialize: the staged caller-order state into the internal order, fresh
// dry flags, counters, AB ramp and clocks.
static int materialize_state(Ctx *c) {
  const int K = c->K;
  const size_t KNp = (size_t)c->Kin * c->Np;
  if (c->f32)
    k_scatter_state<float><<<(K + kScatterTile - 1) / kScatterTile, kScatterTile, sizeof(double) * kScatterTile * c->Np, c->stream>>>(K, c->Np, c->dOrig, c->dStage, c->dStage + KNp,
                                                      c->dStage + 2 * KNp, (float *)c->dQ);
  else
    k_scatter_state<double><<<(K + kScatterTile - 1) / kScatterTile, kScatterTile, sizeof(double) * kScatterTile * c->Np, c->stream>>>(K, c->Np, c->dOrig, c->dStage, c->dStage + KNp,
                                                       c->dStage + 2 * KNp, c->dQ);
  CK(cudaGetLastError());
  if (int rc = scatter_bnd(c)) return rc;
  CK(cudaMemsetAsync(c->dDry, 0, (size_t)4 * K, c->stream));
  CK(cudaMemsetAsync(c->dK2cnt, 0, sizeof(unsigned int) * 2, c->stream));
  c->k2u = 0;
  CK(cudaMemsetAsync(c->dCounters, 0, sizeof(unsigned long long) * kCounters * kSlots, c->stream));
  CK(cudaMemsetAsync(c->dInjected, 0, sizeof(double) * kSlots, c->stream));
  c->n_updates = 0;
  for (int l = 0; l <= 8; l++) {
    c->kcount[l] = 0;
    c->par[l] = 0;
    c->tick_s[l] = 0;
    c->t_e[l] = 0;
  }
  c->tick = 0;
  c->materialized = true;
  return SWE_OK;
}

// recursive slowest-first macro step (reading A17):
// S(l, t) = [(l, t)] + S(l-1, t) + S(l-1, t + 2^(l-2))
// Alg. 1's loop nest as printed, the mrab_coupling = 1 variant: for l = L..1, substeps inner.
static void build_schedule_printed(int L, std::vector<std::pair<int, long>> &out) {
  for (int l = L; l >= 1; l--)
    for (long s = 0; s < (1L << (L - l)); s++) out.push_back({l, s * (1L << (l - 1))});
}

static void build_schedule(int l, long t, std::vector<std::pair<int, long>> &out) {
  out.push_back({l, t});
  if (l > 1) {
    build_schedule(l - 1, t, out);
    build_schedule(l - 1, t + (1L << (l - 2)), out);
  }
}

static void ab_weights(int m, double a[3]) {
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
// integral over [0, theta] of the quadratic interpolant of R(0), R(-1), R(-2)
static void dense_weights(int m, double th, double b[3]) {
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

// Parameters of update (l, t) for one context (MRAB bookkeeping, reading A17).
static StepParams update_params(Ctx *c, int l, long t) {
  StepParams p = base_params(c);
  p.k0 = c->off[l - 1];
  p.k1 = c->off[l];
  if (K2_LIST && c->nranks <= 1 && c->group.size() <= 1 && c->prm.use_tvb && p.k1 > p.k0) {
    // K2 over the list of the update's non-quiet, non-dry elements that K1 appends to
    p.k2list = c->dK2list;
    p.k2cnt = c->dK2cnt;
    p.k2slot = (int)(c->k2u++ & 1);
  }
  const double dtl = std::ldexp(c->dt, l - 1);
  const int k = c->kcount[l];
  const int m = std::min(k + 1, 3);
  double a[3];
  ab_weights(m, a);
  p.own_par = c->par[l];
  p.write_par = 1 - c->par[l];
  p.write_slot = k % 3;
  p.nab = m;
  for (int s = 0; s < 3; s++) {
    p.ab[s] = a[s] * dtl;
    p.ab_slot[s] = ((k - s) % 3 + 3) % 3;
  }
  for (int cl = 1; cl <= c->L; cl++) {
    LevelTab &T = p.lev[cl - 1];
    if (c->prm.mrab_coupling == 1 || c->t_e[cl] == t) {  // latest committed (variant) / synchronised
      T.par = c->par[cl];
      T.dense = 0;
    } else {  // coarser level in the middle of its step
      T.par = 1 - c->par[cl];
      long step = c->t_e[cl] - c->tick_s[cl];
      double theta = (double)(t - c->tick_s[cl]) / (double)step;
      if (t == c->tick_s[cl]) {
        T.dense = 0;
      } else {
        T.dense = 1;
        T.nterm = std::min(c->kcount[cl], 3);
        double b[3];
        dense_weights(T.nterm, theta, b);
        double dtc = std::ldexp(c->dt, cl - 1);
        for (int s = 0; s < 3; s++) {
          T.beta[s] = b[s] * dtc;
          T.slot[s] = ((c->kcount[cl] - 1 - s) % 3 + 3) % 3;
        }
      }
    }
  }
  return p;
}

static void launch_timed(Ctx *c, int which, const StepParams &p, cudaStream_t s = nullptr) {
  const int nel = p.k1 - p.k0;
  if (nel <= 0) return;
  if (!s) s = c->stream;
  if (c->prof) {
    while (c->evpool.size() < c->evnext + 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->evpool.push_back(e);
    }
    cudaEvent_t e0 = c->evpool[c->evnext], e1 = c->evpool[c->evnext + 1];
    c->evnext += 2;
    cudaEventRecord(e0, s);
    launch(which, false, c->N, p, s, c->f32);
    cudaEventRecord(e1, s);
    c->ev.push_back(e0);
    c->ev.push_back(e1);
    c->evwhich.push_back(which);
    c->prof_bytes[which] += (which == 0 ? k1_bytes(c->N, p.nab, c->prm.use_tvb, c->esz) : k2_bytes(c->esz)) * nel;
    c->prof_launch[which]++;
  } else {
    launch(which, false, c->N, p, s, c->f32);
  }
}

static void collect_profile(Ctx *c) {
  // events come in (start, stop) pairs, in launch order
  for (size_t i = 0; i + 1 < c->ev.size(); i += 2) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]);
    c->prof_ms[c->evwhich[i / 2]] += ms;
  }
  c->ev.clear();
  c->evwhich.clear();
  c->evnext = 0;
}

static void clear_graphs(Ctx *c) {
  for (auto &g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
}

// MRAB bookkeeping after an update of level l at tick t (shared by the eager and the graph paths)
static void commit_update(Ctx *c, int l, long t, const StepParams &p) {
  c->n_updates += p.k1 - p.k0;
  c->par[l] ^= 1;
  c->kcount[l] = c->kcount[l] + 1;
  c->tick_s[l] = t;
  c->t_e[l] = t + (1L << (l - 1));
}

// One macro step of a single-rank context through a cached CUDA graph: the parameters of every
// update are computed first (with the bookkeeping); an identical sequence replays its graph,
// a new one is captured (up to kMaxGraphs) and launched.
constexpr size_t kMaxGraphs = 12;

// parameters of the next macro step, with its bookkeeping applied to c
static std::vector<StepParams> next_step_params(Ctx *c) {
  std::vector<StepParams> seq;
  seq.reserve(c->schedule.size());
  for (auto &st : c->schedule) {
    const long t = c->tick + st.second;
    seq.push_back(update_params(c, st.first, t));
    commit_update(c, st.first, t, seq.back());
  }
  return seq;
}

static long step_kmod(const Ctx *c, long k0) { return c->nranks > 1 ? (k0 & 3) : 0; }

static Ctx::StepGraph *find_graph(Ctx *c, const std::vector<StepParams> &seq, long kmod) {
  for (auto &g : c->graphs)
    if (g.kmod == kmod && g.seq.size() == seq.size() &&
        std::memcmp(g.seq.data(), seq.data(), sizeof(StepParams) * seq.size()) == 0)
      return &g;
  return nullptr;
}

static int enqueue_rank_update(Ctx *c, const StepParams &p, int l, long k, cudaStream_t S);
static int ensure_comm_stream(Ctx *c);

// The launches of one macro step (no bookkeeping) on stream S: single rank K1 + K2 per update; a rank of a
// CUDA-IPC partition the overlapped sequence of rank_update with exchanges k0, k0 + 1, ...
static int enqueue_step(Ctx *c, const std::vector<StepParams> &seq, long k0, cudaStream_t S) {
  if (c->nranks <= 1) {
    for (const StepParams &p : seq)
      if (p.k1 > p.k0) {
        launch(0, false, c->N, p, S, c->f32);
        if (c->prm.use_tvb) launch(1, false, c->N, p, S, c->f32);
      }
    return SWE_OK;
  }
  for (size_t i = 0; i < seq.size(); i++)
    if (int rc = enqueue_rank_update(c, seq[i], c->schedule[i].first, k0 + 2 * (long)i, S)) return rc;
  return SWE_OK;
}

static int capture_graph(Ctx *c, std::vector<StepParams> seq, long k0) {
  CK(cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeThreadLocal));
  const int erc = enqueue_step(c, seq, k0, c->gstream);
  cudaGraph_t graph = nullptr;
  const cudaError_t le = cudaGetLastError();
  const cudaError_t ee = cudaStreamEndCapture(c->gstream, &graph);  // always ends the capture
  if (erc || le != cudaSuccess || ee != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    if (erc) return erc;
    return cuda_fail(c, le != cudaSuccess ? le : ee, "graph capture");
  }
  Ctx::StepGraph g;
  g.seq = std::move(seq);
  g.kmod = step_kmod(c, k0);
  cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
  c->graphs.push_back(std::move(g));
  return SWE_OK;
}

static bool ramp_done(const Ctx *c) {
  for (int l = 1; l <= c->L; l++)
    if (c->off[l] > c->off[l - 1] && c->kcount[l] < 2) return false;
  return true;
}

static int graph_step(Ctx *c) {
  Nvtx range("macro step: CUDA graph");
  if (!c->gstream) {
    CK(cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->gev0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->gev1, cudaEventDisableTiming));
  }
  if (c->nranks > 1)
    if (int rc = ensure_comm_stream(c)) return rc;
  const bool after_ramp = ramp_done(c);
  const long k0 = c->xcount, kstep = c->nranks > 1 ? 2 * (long)c->schedule.size() : 0;
  std::vector<StepParams> seq = next_step_params(c);
  c->cur = seq.back();
  c->xcount += kstep;
  Ctx::StepGraph *g = find_graph(c, seq, step_kmod(c, k0));
  if (!g) {
    if (c->graphs.size() >= kMaxGraphs)  // cache full: launch eagerly
      return enqueue_step(c, seq, k0, c->stream);
    if (int rc = capture_graph(c, seq, k0)) return rc;
    g = &c->graphs.back();
    if (after_ramp) {
      // the launch sequence is periodic (ring slot mod 3, parity mod 2): capture the next five
      // phases now, on a copy of the bookkeeping, so that later steps only replay
      const int par[9] = {c->par[0], c->par[1], c->par[2], c->par[3], c->par[4], c->par[5], c->par[6], c->par[7],
                          c->par[8]};
      int kc[9];
      long ts[9], te[9];
      for (int l = 0; l <= 8; l++) kc[l] = c->kcount[l], ts[l] = c->tick_s[l], te[l] = c->t_e[l];
      const long tick = c->tick, nup = c->n_updates, k2u = c->k2u;
      for (int k = 0; k < 5 && c->graphs.size() < kMaxGraphs; k++) {
        c->tick += 1L << (c->L - 1);
        std::vector<StepParams> s2 = next_step_params(c);
        const long k2 = k0 + (k + 1) * kstep;
        if (!find_graph(c, s2, step_kmod(c, k2)))
          if (int rc = capture_graph(c, std::move(s2), k2)) return rc;
      }
      for (int l = 0; l <= 8; l++) c->par[l] = par[l], c->kcount[l] = kc[l], c->tick_s[l] = ts[l], c->t_e[l] = te[l];
      c->tick = tick;
      c->n_updates = nup;
      c->k2u = k2u;
      g = find_graph(c, seq, step_kmod(c, k0));
    }
  }
  CK(cudaEventRecord(c->gev0, c->stream));  // the step starts after the caller's prior work
  CK(cudaStreamWaitEvent(c->gstream, c->gev0, 0));
  CK(cudaGraphLaunch(g->exec, c->gstream));
  CK(cudaEventRecord(c->gev1, c->gstream));  // and the caller's later work waits for the step
  CK(cudaStreamWaitEvent(c->stream, c->gev1, 0));
  return SWE_OK;
}

// Append one decision record (A26) for the owned internal range [k0, k1) of the limiter application just
// launched (stream-synchronising; record_decisions is a debug mode).
static int record_dec(Ctx *c, int k0, int k1) {
  if (!c->dDec) return SWE_OK;
  std::vector<unsigned char> d((size_t)std::max(0, k1 - k0));
  if (k1 > k0) CK(cudaMemcpyAsync(d.data(), c->dDec + k0, (size_t)(k1 - k0), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const size_t base = c->declog.size();
  c->declog.resize(base + (size_t)c->Kin, 0xFF);
  for (int k = k0; k < k1; k++) c->declog[base + (size_t)c->order[k]] = d[(size_t)(k - k0)];
  c->ndec++;
  return SWE_OK;
}

// One halo exchange of `phase` for every context of the group, on each context's stream: pack into the send
// buffer of exchange k, transfer, unpack (in-process contexts share one stream, so every pack precedes
// every transfer).
static int group_exchange(std::vector<Ctx *> &G, int phase, int lvl, int par, int slot) {
  Nvtx range(phase == 0 ? "halo A (means, dry)" : "halo B (face traces)");
  std::vector<long> ks;
  for (Ctx *c : G) ks.push_back(c->xcount++);
  for (size_t i = 0; i < G.size(); i++)
    if (int rc = xpack(G[i], phase, lvl, par, slot, G[i]->stream, ks[i])) return rc;
  for (size_t i = 0; i < G.size(); i++)
    if (int rc = xtransfer(G[i], phase, lvl, G[i]->stream, ks[i])) return rc;
  for (Ctx *c : G)
    if (int rc = xunpack(c, phase, lvl, par, slot, c->stream)) return rc;
  return SWE_OK;
}

// One MRAB update of level l at tick t for every context of an in-process group (one stream), with the
// two halo exchanges: A (means, dry; after K1) and B (face traces of Q and the R slot; after K2).
static int group_update(std::vector<Ctx *> &G, int l, long t) {
  Nvtx range(kLevelRange[l]);
  for (Ctx *c : G) {
    c->cur = update_params(c, l, t);
    launch_timed(c, 0, c->cur);
  }
  if (int rc = group_exchange(G, 0, l, 0, 0)) return rc;
  for (Ctx *c : G)
    if (c->prm.use_tvb) launch_timed(c, 1, c->cur);
  if (int rc = group_exchange(G, 1, l, G[0]->cur.write_par, G[0]->cur.write_slot)) return rc;
  for (Ctx *c : G)
    if (int rc = record_dec(c, c->cur.k0, c->cur.k1)) return rc;
  for (Ctx *c : G) commit_update(c, l, t, c->cur);
  return SWE_OK;
}

static int ensure_comm_stream(Ctx *c) {
  if (c->cstream) return SWE_OK;
  CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
  for (auto &e : c->xev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SWE_OK;
}

// One MRAB update of level l at tick t of a rank of a multi-process partition (CUDA-IPC or NCCL
// transport), with the exchanges on the communication stream overlapping interior work:
//   compute: K1(boundary) | pack A |  K1(interior)  | wait A | K2(boundary) | pack B |  K2(interior)  | wait B
//   comm:                         | exchange A     |                               | exchange B     |
// Interior elements have no ghost neighbour, so K1(interior) does not read what exchange B of the previous
// update delivers, and neither interior kernel touches a ghost.
// The launches of one such update on compute stream S (eager: the context's stream; graph capture: the capture
// stream), exchanges k and k + 1.
static int enqueue_rank_update(Ctx *c, const StepParams &p, int l, long k, cudaStream_t S) {
  if (int rc = ensure_comm_stream(c)) return rc;
  StepParams pb = p, pi = p;
  pb.k1 = c->bnd[l];
  pi.k0 = c->bnd[l];
  cudaStream_t X = c->cstream;
  launch_timed(c, 0, pb, S);
  if (int rc = xpack(c, 0, l, 0, 0, S, k)) return rc;
  CK(cudaEventRecord(c->xev[0], S));
  CK(cudaStreamWaitEvent(X, c->xev[0], 0));
  if (int rc = xtransfer(c, 0, l, X, k)) return rc;
  if (int rc = xunpack(c, 0, l, 0, 0, X)) return rc;
  CK(cudaEventRecord(c->xev[1], X));
  launch_timed(c, 0, pi, S);
  CK(cudaStreamWaitEvent(S, c->xev[1], 0));
  if (c->prm.use_tvb) launch_timed(c, 1, pb, S);
  k++;
  if (int rc = xpack(c, 1, l, p.write_par, p.write_slot, S, k)) return rc;
  CK(cudaEventRecord(c->xev[2], S));
  CK(cudaStreamWaitEvent(X, c->xev[2], 0));
  if (int rc = xtransfer(c, 1, l, X, k)) return rc;
  if (int rc = xunpack(c, 1, l, p.write_par, p.write_slot, X)) return rc;
  CK(cudaEventRecord(c->xev[3], X));
  if (c->prm.use_tvb) launch_timed(c, 1, pi, S);
  CK(cudaStreamWaitEvent(S, c->xev[3], 0));
  return SWE_OK;
}

static int rank_update(Ctx *c, int l, long t) {
  Nvtx range(kLevelRange[l]);
  const StepParams p = update_params(c, l, t);
  c->cur = p;
  if (int rc = enqueue_rank_update(c, p, l, c->xcount, c->stream)) return rc;
  c->xcount += 2;
  if (int rc = record_dec(c, p.k0, p.k1)) return rc;
  commit_update(c, l, t, p);
  return SWE_OK;
}

// Alg. 2 line 1 on every owned element, then the full halo exchange.
static int group_init_limit(std::vector<Ctx *> &G) {
  for (Ctx *c : G) {  // the initial limiting is the first record of the decision log (A26)
    c->declog.clear();
    c->ndec = 0;
  }
  for (Ctx *c : G) {
    StepParams p = base_params(c);
    p.k0 = 0;
    p.k1 = c->kown;
    p.own_par = 0;
    p.write_par = 0;
    c->cur = p;
    launch(0, true, c->N, p, c->stream, c->f32);
    CK(cudaGetLastError());
  }
  if (int rc = group_exchange(G, 0, 0, 0, 0)) return rc;
  for (Ctx *c : G)
    if (c->prm.use_tvb) launch(1, false, c->N, c->cur, c->stream, c->f32);
  if (int rc = group_exchange(G, 1, 0, 0, -1)) return rc;
  for (Ctx *c : G)
    if (int rc = record_dec(c, 0, c->kown)) return rc;
  return SWE_OK;
}

// Global minimum of r_min over every rank through the IPC blocks (the r_min words have their own flag
// pair, counted per binning: a rank can be at most one binning ahead of any other).
static int ipc_rmin(Ctx *c) {
  const long n = c->rcount++;
  const int sl = (int)(n & 1);
  const cuuint64_t v = (cuuint64_t)n + 1;
  cudaStream_t S = c->stream;
  CK(cudaMemcpyAsync(c->ipcBlock + 32 + 8 * sl, c->dRmin, sizeof(double), cudaMemcpyDeviceToDevice, S));
  if (g_write64((CUstream)S, (CUdeviceptr)(c->ipcBlock + 16 + 8 * sl), v, 0) != CUDA_SUCCESS) {
    c->err = "cuStreamWriteValue64 failed";
    return SWE_ERR_CUDA;
  }
  std::vector<double> r((size_t)c->nranks, std::numeric_limits<double>::infinity());
  for (int q = 0; q < c->nranks; q++) {
    char *pb = q == c->rank ? c->ipcBlock : c->ipcPeer[q];
    if (q != c->rank &&
        g_wait64((CUstream)S, (CUdeviceptr)(pb + 16 + 8 * sl), v, CU_STREAM_WAIT_VALUE_GEQ | g_wait_flush) !=
            CUDA_SUCCESS) {
      c->err = "cuStreamWaitValue64 failed";
      return SWE_ERR_CUDA;
    }
    CK(cudaMemcpyAsync(&r[q], pb + 32 + 8 * sl, sizeof(double), cudaMemcpyDeviceToHost, S));
  }
  CK(cudaStreamSynchronize(S));
  double m = r[0];
  for (double x : r) m = std::min(m, x);
  CK(cudaMemcpyAsync(c->dRmin, &m, sizeof(double), cudaMemcpyHostToDevice, S));
  CK(cudaStreamSynchronize(S));
  return SWE_OK;
}

// r_min over all ranks (levels are global, reading A19)
static int group_bin(std::vector<Ctx *> &G, int nlevels) {
  Nvtx range("level binning + initial limiting");
  // r_min on the device, reduced over the group's contexts and over NCCL ranks
  const double inf = std::numeric_limits<double>::infinity();
  double rmin = inf;
  for (Ctx *c : G) {
    const unsigned long long infbits = 0x7ff0000000000000ULL;
    CK(cudaMemcpyAsync(c->dRmin, &infbits, sizeof(infbits), cudaMemcpyHostToDevice, c->stream));
    k_rmin<<<std::min((c->Kin + 255) / 256, 4 * 148), 256, 0, c->stream>>>(c->Kin, c->dHk, c->dAe,
                                                                          (unsigned long long *)c->dRmin);
    CK(cudaGetLastError());
    if (G.size() == 1 && c->comm)  // global minimum across NCCL ranks
      NK(ncclAllReduce(c->dRmin, c->dRmin, 1, ncclDouble, ncclMin, c->comm, c->stream));
    if (G.size() == 1 && c->ipc)  // across CUDA-IPC ranks
      if (int rc = ipc_rmin(c)) return rc;
    double r = inf;
    CK(cudaMemcpyAsync(&r, c->dRmin, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    rmin = std::min(rmin, r);
  }
  for (Ctx *c : G) {
    // levels on the device; the host needs them only when they differ from the resident layout's
    const bool cmp = c->layout_valid && c->levres_ok && c->L == nlevels;
    int changed = 0;
    CK(cudaMemcpyAsync(c->dRmin, &rmin, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->dFlag, 0, sizeof(int), c->stream));
    k_levels<<<(c->Kin + 255) / 256, 256, 0, c->stream>>>(c->Kin, c->dHk, c->dAe, c->dRmin, nlevels, c->dLev,
                                                         cmp ? c->dLevRes : nullptr, c->dFlag);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&changed, c->dFlag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (cmp && !changed) {  // same levels: keep the layout, scatter the new state
      if (int rc = materialize(c, c->level, nlevels)) return rc;
    } else {
      std::vector<int32_t> lev(c->Kin, 1);
      CK(cudaMemcpyAsync(lev.data(), c->dLev, sizeof(int32_t) * c->Kin, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (int rc = materialize(c, lev, nlevels)) return rc;
      CK(cudaMemcpyAsync(c->dLevRes, c->dLev, sizeof(int32_t) * c->Kin, cudaMemcpyDeviceToDevice, c->stream));
      c->levres_ok = true;
    }
  }
  return group_init_limit(G);
}

static int group_step(std::vector<Ctx *> &G, double dt, int nlevels) {
  Nvtx range("swe_step (macro step)");
  for (Ctx *c : G)
    if (int rc = check_bnd(c)) return rc;
  for (Ctx *c : G) {
    if (!c->have_state) {
      c->err = "swe_step before swe_set_state";
      return SWE_ERR_STATE;
    }
    if (!(dt > 0) || !std::isfinite(dt) || nlevels < 1 || nlevels > 8) {
      c->err = "invalid dt or nlevels";
      return SWE_ERR_ARG;
    }
  }
  if (!G[0]->scheduled) {
    if (int rc = group_bin(G, nlevels)) return rc;
    for (Ctx *c : G) {
      c->scheduled = true;
      c->dt = dt;
      c->L = nlevels;
      c->schedule.clear();
      if (c->prm.mrab_coupling == 1)
        build_schedule_printed(nlevels, c->schedule);
      else
        build_schedule(nlevels, 0, c->schedule);
    }
  } else {
    for (Ctx *c : G)
      if (dt != c->dt || nlevels != c->L) {
        c->err = "(dt, nlevels) differ from the first swe_step (levels are fixed, P:149)";
        return SWE_ERR_SCHEDULE;
      }
  }
  Ctx *c0 = G[0];
  if (G.size() == 1 && (c0->nranks <= 1 || c0->ipc) && !c0->prof && c0->use_graphs && !c0->dDec) {
    if (int rc = graph_step(c0)) return rc;
  } else if (G.size() == 1 && c0->nranks > 1 && (c0->ipc || c0->comm)) {
    for (auto &st : c0->schedule)
      if (int rc = rank_update(c0, st.first, c0->tick + st.second)) return rc;
  } else {
    for (auto &st : c0->schedule)
      if (int rc = group_update(G, st.first, c0->tick + st.second)) return rc;
  }
  for (Ctx *c : G) {
    c->tick += 1L << (c->L - 1);
    Ctx *c_ = c;
    {
      Ctx *c = c_;
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(c->hCounters, c->dCounters, sizeof(unsigned long long) * kCounters * kSlots, cudaMemcpyDeviceToHost,
                         c->stream));
    }
  }
  for (Ctx *c : G) {
    CK(cudaStreamSynchronize(c->stream));
    if (c->prof) collect_profile(c);
    if (counter(c, 3) != 0) {
      c->err = "non-finite values produced";
      return SWE_ERR_NONFINITE;
    }
  }
  return SWE_OK;
}

static int ensure_materialized_group(std::vector<Ctx *> &G) {
  for (Ctx *c : G)
    if (int rc = check_bnd(c)) return rc;
  bool need = false;
  for (Ctx *c : G) need = need || !c->materialized;
  if (!need) return SWE_OK;
  for (Ctx *c : G) {
    std::vector<int32_t> ones(c->Kin, 1);
    c->levres_ok = false;
    if (int rc = materialize(c, ones, 1)) return rc;
  }
  return group_init_limit(G);
}

static std::vector<Ctx *> group_of(Ctx *c) {
  if (c->group.empty()) return {c};
  return c->group;
}

static GatherParams gather_params(Ctx *c, double *h, double *hu, double *hv) {
  GatherParams g;
  std::memset(&g, 0, sizeof(g));
  g.K = c->kown;  // owned elements only
  g.Np = c->Np;
  g.nlev = c->L;
  for (int l = 0; l <= 8; l++) g.off[l] = c->off[l];
  for (int l = 1; l <= 8; l++) g.par[l - 1] = c->par[l];
  g.Kstride = c->K;
  g.orig = c->dOrig;
  g.Q = c->dQ;
  g.h = h;
  g.hu = hu;
  g.hv = hv;
  return g;
}

}  // namespace swe

using namespace swe;

struct swe_ctx {
  Ctx c;
};

extern "C" {

static void fill_defaults(swe_params &p, const swe_params *in) {
  std::memset(&p, 0, sizeof(p));
  if (in) {
    p = *in;
  } else {
    p.use_pp = 1;
    p.use_tvb = 1;
  }
  if (!(p.h0 > 0)) p.h0 = 1e-6;
  if (!(p.eps > 0)) p.eps = p.h0;
  if (!(p.tvb_nu > 0)) p.tvb_nu = 1.5;
  if (!(p.eps_u > 0)) p.eps_u = 1000.0 * p.h0;
  if (!(p.h_char > 0)) p.h_char = 10.0 * p.h0;
  if (p.a_floor < 0) p.a_floor = 0;
  if (p.tvb_M < 0) p.tvb_M = 0;
  if (p.nranks < 1) p.nranks = 1;
}

int swe_nodes(const swe_mesh *mesh, int N, double *x, double *y) {
  if (!mesh || !x || !y || !mesh->etov || !mesh->vx || !mesh->vy || mesh->nelems <= 0) return SWE_ERR_ARG;
  if (N < 1 || N > 8) return SWE_ERR_ORDER;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  RefOps o;
  if (!build_refops(N, o, &err)) return SWE_ERR_ORDER;
  for (int e = 0; e < m.K; e++) {
    const int32_t *v = &m.etov[(size_t)3 * e];
    double x1 = m.vx[v[0]], x2 = m.vx[v[1]], x3 = m.vx[v[2]], y1 = m.vy[v[0]], y2 = m.vy[v[1]], y3 = m.vy[v[2]];
    for (int i = 0; i < o.Np; i++) {
      double r = o.r[i], s = o.s[i];
      x[(size_t)e * o.Np + i] = -0.5 * (r + s) * x1 + 0.5 * (1.0 + r) * x2 + 0.5 * (1.0 + s) * x3;
      y[(size_t)e * o.Np + i] = -0.5 * (r + s) * y1 + 0.5 * (1.0 + r) * y2 + 0.5 * (1.0 + s) * y3;
    }
  }
  return SWE_OK;
}

int swe_nccl_unique_id(void *id128) {
  if (!id128) return SWE_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SWE_ERR_NCCL;
  std::memcpy(id128, &id, sizeof(id));
  return SWE_OK;
}

int swe_create(const swe_mesh *mesh, const double *B, int N, double g, const swe_params *params, swe_ctx **out) {
  if (!out) return SWE_ERR_ARG;
  *out = nullptr;
  if (!mesh || !B || !mesh->etov || !mesh->vx || !mesh->vy || mesh->nelems <= 0 || mesh->nverts <= 0 || !(g > 0))
    return SWE_ERR_ARG;
  if (N < 1 || N > kMaxOrder) return SWE_ERR_ORDER;
  swe_ctx *h = new swe_ctx();
  Ctx *c = &h->c;
  fill_defaults(c->prm, params);
  c->N = N;
  c->Np = (N + 1) * (N + 2) / 2;
  c->Kin = mesh->nelems;
  c->g = g;
  c->device = c->prm.device;
  c->stream = (cudaStream_t)c->prm.stream;
  c->rank = c->prm.rank;
  c->nranks = c->prm.nranks;
  auto fail = [&](int rc) {
    swe_destroy(h);
    return rc;
  };
  if (c->prm.mrab_coupling != 0 && c->prm.mrab_coupling != 1) {
    c->err = "mrab_coupling must be 0 or 1";
    return fail(SWE_ERR_ARG);
  }
  if (c->prm.precision != 0 && c->prm.precision != 32 && c->prm.precision != 64) {
    c->err = "precision must be 32 or 64";
    return fail(SWE_ERR_ARG);
  }
  c->f32 = c->prm.precision == 32;
  c->esz = c->f32 ? sizeof(float) : sizeof(double);
  if (c->rank < 0 || c->rank >= c->nranks) return fail(SWE_ERR_ARG);
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, c->mesh, &c->err);
  if (rc) return fail(rc);
  apply_boundary_tags(c->mesh, mesh->vbc);
  for (int8_t t : c->mesh.bc) c->n_dirichlet += t == 2 ? 1 : 0;
  if (!build_refops(N, c->ops, &c->err)) return fail(SWE_ERR_ORDER);
  for (int f = 0; f < 3; f++)
    for (int k = 0; k < c->ops.Nfp; k++)
      if (c->ops.Fmask[f * c->ops.Nfp + k] != fmask(N, f, k)) {
        c->err = "face node table mismatch";
        return fail(SWE_ERR_ORDER);
      }
  build_tvb_geometry(c->mesh, c->tvb);
  // ownership (every element owned by this rank when no partition is given)
  c->gid.resize(c->Kin);
  c->owner.assign(c->Kin, c->rank);
  for (int e = 0; e < c->Kin; e++) c->gid[e] = c->prm.gid ? c->prm.gid[e] : e;
  if (c->prm.owner) {
    for (int e = 0; e < c->Kin; e++) {
      if (c->prm.owner[e] < 0 || c->prm.owner[e] >= c->nranks) {
        c->err = "owner rank out of range";
        return fail(SWE_ERR_ARG);
      }
      c->owner[e] = c->prm.owner[e];
    }
  }
  build_halo_plan(c->mesh, c->gid.data(), c->owner.data(), c->rank, c->plan);
  c->kown = (int)c->plan.owned.size();
  c->K = c->kown + (int)c->plan.ghosts.size();
  if (c->kown == 0) {
    c->err = "rank owns no element";
    return fail(SWE_ERR_MESH);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    c->err = "no CUDA device";
    cudaGetLastError();
    return fail(SWE_ERR_CUDA);
  }
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(SWE_ERR_CUDA);
  if (upload_ops_any(c->ops) != cudaSuccess) return fail(SWE_ERR_CUDA);
  rc = alloc_state(c);
  if (rc) return fail(rc);
  c->dBcaller = (double *)c->dalloc(sizeof(double) * (size_t)c->Kin * c->Np);
  c->dWm2 = (double *)c->dalloc(sizeof(double) * c->Np);
  c->dHk = (double *)c->dalloc(sizeof(double) * c->Kin);
  c->dLev = (int32_t *)c->dalloc(sizeof(int32_t) * c->Kin);
  c->dLevRes = (int32_t *)c->dalloc(sizeof(int32_t) * c->Kin);
  c->dFlag = (int *)c->dalloc(sizeof(int));
  std::vector<double> sops = smem_ops_any(c->ops);
  c->dOpsG = (double *)c->dalloc(sizeof(double) * sops.size());
  std::vector<float> sopsf(sops.begin(), sops.end());
  c->dOpsGf = (double *)c->dalloc(sizeof(float) * sopsf.size());
  c->dCounters = (unsigned long long *)c->dalloc(sizeof(unsigned long long) * kCounters * kSlots);
  c->dInjected = (double *)c->dalloc(sizeof(double) * kSlots);
  if (!c->alloc_ok) return fail(SWE_ERR_NOMEM);
  if (cudaMallocHost(&c->hCounters, sizeof(unsigned long long) * kCounters * kSlots) != cudaSuccess) return fail(SWE_ERR_CUDA);
  if (cudaMallocHost(&c->hInjected, sizeof(double) * kSlots) != cudaSuccess) return fail(SWE_ERR_CUDA);
  std::vector<double> wm2(c->Np);
  for (int i = 0; i < c->Np; i++) wm2[i] = 0.5 * c->ops.wmean[i];
  if (cudaMemcpyAsync(c->dBcaller, B, sizeof(double) * (size_t)c->Kin * c->Np, cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess ||
      cudaMemcpyAsync(c->dWm2, wm2.data(), sizeof(double) * c->Np, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(c->dHk, c->mesh.hk.data(), sizeof(double) * c->Kin, cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess ||
      cudaMemcpyAsync(c->dOpsG, sops.data(), sizeof(double) * sops.size(), cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess ||
      cudaMemcpyAsync(c->dOpsGf, sopsf.data(), sizeof(float) * sopsf.size(), cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess ||
      cudaMemsetAsync(c->dCounters, 0, sizeof(unsigned long long) * kCounters * kSlots, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->dInjected, 0, sizeof(double) * kSlots, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->err = "initial upload failed";
    return fail(SWE_ERR_CUDA);
  }
  if (c->nranks > 1 && c->prm.nccl_id) {
    ncclUniqueId id;
    std::memcpy(&id, c->prm.nccl_id, sizeof(id));
    if (ncclCommInitRank(&c->comm, c->nranks, id, c->rank) != ncclSuccess) {
      c->err = "ncclCommInitRank failed";
      c->comm = nullptr;
      return fail(SWE_ERR_NCCL);
    }
  }
  *out = h;
  return SWE_OK;
}

int swe_set_state(swe_ctx *h, const double *hh, const double *hu, const double *hv) {
  if (!h || !hh || !hu || !hv) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  const size_t KNp = (size_t)c->Kin * c->Np;
  CK(cudaMemcpyAsync(c->dStage, hh, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dStage + KNp, hu, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dStage + 2 * KNp, hv, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  double e2 = c->prm.eps_u * c->prm.eps_u, e4 = e2 * e2;
  k_speeds<<<(c->Kin + 127) / 128, 128, 0, c->stream>>>(c->Kin, c->Np, c->g, e4, c->prm.a_floor, c->dStage,
                                                         c->dStage + KNp, c->dStage + 2 * KNp, c->dAe);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(c->dCounters, 0, sizeof(unsigned long long) * kCounters * kSlots, c->stream));
  CK(cudaMemsetAsync(c->dInjected, 0, sizeof(double) * kSlots, c->stream));
  c->have_state = true;
  c->materialized = false;
  c->scheduled = false;
  c->n_updates = 0;
  c->tick = 0;
  c->t_base = 0.0;
  c->declog.clear();
  c->ndec = 0;
  return SWE_OK;
}

int swe_set_boundary_state(swe_ctx *h, const double *hh, const double *hu, const double *hv) {
  if (!h || !hh || !hu || !hv) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  const size_t KNp = (size_t)c->Kin * c->Np;
  if (!c->dBndStage) {
    c->dBndStage = (double *)c->dalloc(sizeof(double) * 3 * KNp);
    c->dQbnd = (double *)c->dalloc(c->esz * 3 * c->Np * eb_pad((size_t)c->K));
    c->dBmean = (double *)c->dalloc(c->esz * 3 * eb_pad((size_t)c->K));
    if (!c->alloc_ok) {
      c->alloc_ok = true;
      c->err = "swe_set_boundary_state: device allocation failed";
      return SWE_ERR_NOMEM;
    }
  }
  CK(cudaMemcpyAsync(c->dBndStage, hh, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dBndStage + KNp, hu, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->dBndStage + 2 * KNp, hv, sizeof(double) * KNp, cudaMemcpyHostToDevice, c->stream));
  c->bnd_set = true;
  return scatter_bnd(c);
}

int swe_step(swe_ctx *h, double dt, int nlevels) {
  if (!h) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->group.empty()) {
    c->err = "context is linked to an in-process group: use swe_step_group";
    return SWE_ERR_STATE;
  }
  std::vector<Ctx *> G = {c};
  return group_step(G, dt, nlevels);
}

int swe_link_group(swe_ctx **ctxs, int n) {
  if (!ctxs || n < 1) return SWE_ERR_ARG;
  std::vector<Ctx *> G(n, nullptr);
  for (int i = 0; i < n; i++) {
    if (!ctxs[i]) return SWE_ERR_ARG;
    Ctx *c = &ctxs[i]->c;
    if (c->nranks != n || c->rank < 0 || c->rank >= n || G[c->rank]) return SWE_ERR_ARG;
    if (c->stream != ctxs[0]->c.stream || c->device != ctxs[0]->c.device) return SWE_ERR_ARG;
    G[c->rank] = c;
  }
  for (Ctx *c : G) c->group = G;
  return SWE_OK;
}

int swe_step_group(swe_ctx **ctxs, int n, double dt, int nlevels) {
  if (!ctxs || n < 1 || !ctxs[0]) return SWE_ERR_ARG;
  Ctx *c0 = &ctxs[0]->c;
  if ((int)c0->group.size() != n) {
    c0->err = "contexts are not linked (swe_link_group)";
    return SWE_ERR_STATE;
  }
  std::vector<Ctx *> G = c0->group;
  return group_step(G, dt, nlevels);
}

int swe_regroup(swe_ctx *h) {
  if (!h) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->have_state) return SWE_ERR_STATE;
  if (c->nranks > 1) {
    c->err = "swe_regroup: single-rank contexts only";
    return SWE_ERR_ARG;
  }
  if (!c->materialized) return SWE_OK;  // nothing stepped since swe_set_state: the staged state stands
  // current state -> staging (caller order), then the swe_set_state path from there
  const size_t KNp = (size_t)c->Kin * c->Np;
  GatherParams g = gather_params(c, c->dStage, c->dStage + KNp, c->dStage + 2 * KNp);
  if (c->f32)
    k_gather_state<float><<<(c->kown + 127) / 128, 128, 0, c->stream>>>(g);
  else
    k_gather_state<double><<<(c->kown + 127) / 128, 128, 0, c->stream>>>(g);
  CK(cudaGetLastError());
  const double t = c->t_base + (c->scheduled ? c->dt * (double)c->tick : 0.0);
  double e2 = c->prm.eps_u * c->prm.eps_u, e4 = e2 * e2;
  k_speeds<<<(c->Kin + 127) / 128, 128, 0, c->stream>>>(c->Kin, c->Np, c->g, e4, c->prm.a_floor, c->dStage,
                                                         c->dStage + KNp, c->dStage + 2 * KNp, c->dAe);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(c->dCounters, 0, sizeof(unsigned long long) * kCounters * kSlots, c->stream));
  CK(cudaMemsetAsync(c->dInjected, 0, sizeof(double) * kSlots, c->stream));
  c->materialized = false;
  c->scheduled = false;
  c->n_updates = 0;
  c->tick = 0;
  c->t_base = t;
  c->declog.clear();
  c->ndec = 0;
  return SWE_OK;
}

int swe_get_state(swe_ctx *h, double *hh, double *hu, double *hv) {
  if (!h || !hh || !hu || !hv) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->have_state) return SWE_ERR_STATE;
  std::vector<Ctx *> G = group_of(c);
  for (Ctx *q : G)
    if (!q->have_state) return SWE_ERR_STATE;
  int rc = ensure_materialized_group(G);
  if (rc) return rc;
  const size_t KNp = (size_t)c->Kin * c->Np;
  if (!c->dGather) {
    c->dGather = (double *)c->dalloc(sizeof(double) * 3 * KNp);
    if (!c->dGather) {
      c->alloc_ok = true;  // a later call may retry
      c->err = "swe_get_state: device allocation failed";
      return SWE_ERR_NOMEM;
    }
  }
  double *tmp = c->dGather;
  GatherParams g = gather_params(c, tmp, tmp + KNp, tmp + 2 * KNp);
  if (c->f32)
    k_gather_tile<float><<<(c->kown + kGatherTile - 1) / kGatherTile, kGatherTile, sizeof(double) * kGatherTile * c->Np, c->stream>>>(g);
  else
    k_gather_tile<double><<<(c->kown + kGatherTile - 1) / kGatherTile, kGatherTile, sizeof(double) * kGatherTile * c->Np, c->stream>>>(g);
  cudaError_t e = cudaGetLastError();
  if (c->kown == c->Kin) {  // every element owned: straight copies
    if (e == cudaSuccess) e = cudaMemcpyAsync(hh, tmp, sizeof(double) * KNp, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hu, tmp + KNp, sizeof(double) * KNp, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hv, tmp + 2 * KNp, sizeof(double) * KNp, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  } else {  // only owned rows are written
    std::vector<double> buf(3 * KNp);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(buf.data(), tmp, sizeof(double) * 3 * KNp, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) {
      double *outs[3] = {hh, hu, hv};
      for (int k = 0; k < c->kown; k++) {
        size_t o = (size_t)c->order[k] * c->Np;
        for (int f = 0; f < 3; f++) std::memcpy(outs[f] + o, &buf[f * KNp + o], sizeof(double) * c->Np);
      }
    }
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "swe_get_state");
  return SWE_OK;
}

int swe_get_state_async(swe_ctx *h, double *hh, double *hu, double *hv) {
  if (!h || !hh || !hu || !hv) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->have_state) return SWE_ERR_STATE;
  if (c->nranks > 1 || !c->group.empty() || c->kown != c->Kin) return swe_get_state(h, hh, hu, hv);
  std::vector<Ctx *> G = {c};
  if (int rc = ensure_materialized_group(G)) return rc;
  const size_t KNp = (size_t)c->Kin * c->Np;
  const int i = (int)(c->nsnap & 1);
  if (!c->ostream) {
    CK(cudaStreamCreateWithFlags(&c->ostream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; k++) {
      CK(cudaEventCreateWithFlags(&c->oevG[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->oevC[k], cudaEventDisableTiming));
    }
  }
  if (!c->dSnap[i]) {
    c->dSnap[i] = (double *)c->dalloc(sizeof(double) * 3 * KNp);
    if (!c->dSnap[i]) {
      c->alloc_ok = true;  // a later call may retry
      c->err = "swe_get_state_async: device allocation failed";
      return SWE_ERR_NOMEM;
    }
  }
  double *tmp = c->dSnap[i];
  if (c->nsnap >= 2) CK(cudaStreamWaitEvent(c->stream, c->oevC[i], 0));  // the buffer's previous copy is done
  GatherParams g = gather_params(c, tmp, tmp + KNp, tmp + 2 * KNp);
  if (c->f32)
    k_gather_tile<float><<<(c->kown + kGatherTile - 1) / kGatherTile, kGatherTile, sizeof(double) * kGatherTile * c->Np, c->stream>>>(g);
  else
    k_gather_tile<double><<<(c->kown + kGatherTile - 1) / kGatherTile, kGatherTile, sizeof(double) * kGatherTile * c->Np, c->stream>>>(g);
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->oevG[i], c->stream));
  CK(cudaStreamWaitEvent(c->ostream, c->oevG[i], 0));
  double *outs[3] = {hh, hu, hv};
  for (int f = 0; f < 3; f++)
    CK(cudaMemcpyAsync(outs[f], tmp + (size_t)f * KNp, sizeof(double) * KNp, cudaMemcpyDeviceToHost, c->ostream));
  CK(cudaEventRecord(c->oevC[i], c->ostream));
  c->nsnap++;
  return SWE_OK;
}

int swe_wait_state(swe_ctx *h) {
  if (!h) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (c->ostream) CK(cudaStreamSynchronize(c->ostream));
  return SWE_OK;
}

void swe_destroy(swe_ctx *h) {
  if (!h) return;
  Ctx *c = &h->c;
  if (c->stream || c->dQ) cudaStreamSynchronize(c->stream);
  if (c->ostream) {
    cudaStreamSynchronize(c->ostream);
    cudaStreamDestroy(c->ostream);
    for (int k = 0; k < 2; k++) {
      if (c->oevG[k]) cudaEventDestroy(c->oevG[k]);
      if (c->oevC[k]) cudaEventDestroy(c->oevC[k]);
    }
  }
  if (c->cstream) {
    cudaStreamSynchronize(c->cstream);
    cudaStreamDestroy(c->cstream);
  }
  for (cudaEvent_t e : c->xev)
    if (e) cudaEventDestroy(e);
  for (char *pb : c->ipcPeer)
    if (pb) cudaIpcCloseMemHandle(pb);
  if (c->ipcBlock) cudaFree(c->ipcBlock);
  if (c->comm) ncclCommDestroy(c->comm);
  // destroying one member unlinks the whole in-process group: the survivors become unlinked
  // contexts (their next step reports the missing transport instead of touching a freed peer)
  const std::vector<Ctx *> members = c->group;
  for (Ctx *q : members)
    if (q && q != c) q->group.clear();
  void *ptrs[] = {c->dQ,       c->dR,     c->dB,    c->dV,        c->dMeans,   c->dUT,    c->dTalpha, c->dTgeo, c->dGeo,
                  c->dAe,      c->dStage, c->dInjected, c->dWm2,  c->dBcaller, c->dPartials, c->dOpsG, c->dOpsGf, c->dHk, c->dLev, c->dLevRes, c->dFlag,
                  c->dRmin,    c->dXsBuf, c->dXrBuf, c->dE2E,     c->dTcode,   c->dOrig,  c->dXidx,
                  c->dDry,   c->dCounters, c->dGather, c->dDec, c->dBndStage, c->dQbnd, c->dBmean, c->dK2list, c->dK2cnt,
                  c->dSnap[0], c->dSnap[1]};
  clear_graphs(c);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  if (c->gev0) cudaEventDestroy(c->gev0);
  if (c->gev1) cudaEventDestroy(c->gev1);
  for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
  for (void *p : ptrs) c->dfree(p);
  if (c->hCounters) cudaFreeHost(c->hCounters);
  if (c->hInjected) cudaFreeHost(c->hInjected);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  delete h;
}

int swe_get_levels(swe_ctx *h, int32_t *level) {
  if (!h || !level) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->scheduled) return SWE_ERR_STATE;
  std::copy(c->level.begin(), c->level.end(), level);
  return SWE_OK;
}

int swe_get_connectivity(const swe_ctx *h, int32_t *etoe, int8_t *etof) {
  if (!h || !etoe || !etof) return SWE_ERR_ARG;
  const Ctx *c = &h->c;
  std::copy(c->mesh.etoe.begin(), c->mesh.etoe.end(), etoe);
  std::copy(c->mesh.etof.begin(), c->mesh.etof.end(), etof);
  return SWE_OK;
}

int swe_get_info(swe_ctx *h, swe_info *info) {
  if (!h || !info) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  std::memset(info, 0, sizeof(*info));
  info->K = c->kown;
  info->Np = c->Np;
  info->N = c->N;
  info->nflipped = c->mesh.nflipped;
  info->nlevels = c->scheduled ? c->L : 0;
  info->t = c->t_base + (c->scheduled ? c->dt * (double)c->tick : 0.0);
  info->n_updates = c->n_updates;
  if (c->scheduled)
    for (int l = 1; l <= c->L; l++) info->level_count[l - 1] = c->off[l] - c->off[l - 1];
  if (!c->have_state) return SWE_OK;
  std::vector<Ctx *> G = group_of(c);
  int rc = ensure_materialized_group(G);
  if (rc) return rc;
  int nb = (c->kown + 255) / 256;
  GatherParams g = gather_params(c, nullptr, nullptr, nullptr);
  if (c->f32)
    k_diag<float><<<nb, 256, 0, c->stream>>>(g, c->dV, c->dWm2, c->dPartials);
  else
    k_diag<double><<<nb, 256, 0, c->stream>>>(g, c->dV, c->dWm2, c->dPartials);
  std::vector<double> part(2 * (size_t)nb);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(part.data(), c->dPartials, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->hCounters, c->dCounters, sizeof(unsigned long long) * kCounters * kSlots, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->hInjected, c->dInjected, sizeof(double) * kSlots, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  double mass = 0.0, mn = 1e300;
  for (int b = 0; b < nb; b++) {
    mass += part[2 * b];
    mn = std::min(mn, part[2 * b + 1]);
  }
  info->mass = mass;
  info->min_h = mn;
  double inj = 0.0;
  for (int i = 0; i < kSlots; i++) inj += c->hInjected[i];
  info->injected_mass = inj;
  info->n_pp = (int64_t)counter(c, 0);
  info->n_dry = (int64_t)counter(c, 1);
  info->n_tvb = (int64_t)counter(c, 2);
  info->n_posfix = (int64_t)counter(c, 4);
  info->n_tvb_cw = (int64_t)counter(c, 5);
  return SWE_OK;
}

const char *swe_last_error(const swe_ctx *h) { return h ? h->c.err.c_str() : "null context"; }

// ---- CUDA-IPC transport: exchange-block handles
namespace {
struct IpcBlobHdr {
  uint32_t magic, version;
  int32_t rank, nranks;
  uint64_t slot_bytes;
  cudaIpcMemHandle_t handle;
};  // followed by int64 baseA[nranks], baseB[nranks]
constexpr uint32_t kIpcMagic = 0x53574531u;  // "SWE1"
size_t ipc_blob_bytes(int nranks) { return sizeof(IpcBlobHdr) + 2 * sizeof(int64_t) * (size_t)nranks; }
}  // namespace

int swe_ipc_handle(swe_ctx *h, void *blob, size_t *bytes) {
  if (!h || !bytes) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  const size_t need = ipc_blob_bytes(c->nranks);
  if (!blob) {
    *bytes = need;
    return SWE_OK;
  }
  if (*bytes < need) return SWE_ERR_ARG;
  if (c->nranks <= 1) {
    c->err = "swe_ipc_handle: single-rank context";
    return SWE_ERR_ARG;
  }
  if (!c->ipcBlock) {  // plain cudaMalloc (IPC-exportable), not the caller's allocator
    c->ipcSlotBytes = (c->esz * c->capS + 255) / 256 * 256;
    void *p = nullptr;
    CK(cudaMalloc(&p, kIpcHdr + 2 * c->ipcSlotBytes));
    c->ipcBlock = (char *)p;
    CK(cudaMemset(c->ipcBlock, 0, kIpcHdr));
  }
  IpcBlobHdr hd;
  std::memset(&hd, 0, sizeof(hd));
  hd.magic = kIpcMagic;
  hd.version = 1;
  hd.rank = c->rank;
  hd.nranks = c->nranks;
  hd.slot_bytes = c->ipcSlotBytes;
  CK(cudaIpcGetMemHandle(&hd.handle, c->ipcBlock));
  std::vector<int64_t> base((size_t)2 * c->nranks, -1);
  int64_t oa = 0, ob = 0;
  for (size_t i = 0; i < c->plan.peers.size(); i++) {  // send layout [peer][level]: peer i's block start
    base[(size_t)c->plan.peers[i]] = oa;
    base[(size_t)c->nranks + c->plan.peers[i]] = ob;
    oa += (int64_t)c->sendA[i].size();
    ob += (int64_t)c->sendB[i].size();
  }
  std::memcpy(blob, &hd, sizeof(hd));
  std::memcpy((char *)blob + sizeof(hd), base.data(), sizeof(int64_t) * base.size());
  *bytes = need;
  return SWE_OK;
}

int swe_ipc_open(swe_ctx *h, const void *blobs) {
  if (!h || !blobs) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->ipcBlock) {
    c->err = "swe_ipc_open before swe_ipc_handle";
    return SWE_ERR_STATE;
  }
  if (int rc = memops_init(c)) return rc;
  const size_t bb = ipc_blob_bytes(c->nranks);
  c->ipcPeer.assign((size_t)c->nranks, nullptr);
  c->ipcPeerSlot.assign((size_t)c->nranks, 0);
  c->ipcBaseA.assign(c->plan.peers.size(), 0);
  c->ipcBaseB.assign(c->plan.peers.size(), 0);
  for (int q = 0; q < c->nranks; q++) {
    const char *b = (const char *)blobs + bb * (size_t)q;
    IpcBlobHdr hd;
    std::memcpy(&hd, b, sizeof(hd));
    if (hd.magic != kIpcMagic || hd.version != 1 || hd.rank != q || hd.nranks != c->nranks) {
      c->err = "swe_ipc_open: blob " + std::to_string(q) + " is not rank " + std::to_string(q) + "'s handle";
      return SWE_ERR_ARG;
    }
    const int64_t *base = (const int64_t *)(b + sizeof(hd));
    bool peer = false;
    for (size_t i = 0; i < c->plan.peers.size(); i++)
      if (c->plan.peers[i] == q) {
        peer = true;
        c->ipcBaseA[i] = base[c->rank];
        c->ipcBaseB[i] = base[c->nranks + c->rank];
      }
    if (peer != (base[c->rank] >= 0)) {
      c->err = "swe_ipc_open: halo plans of ranks " + std::to_string(c->rank) + " and " + std::to_string(q) + " disagree";
      return SWE_ERR_MESH;
    }
    c->ipcPeerSlot[(size_t)q] = (size_t)hd.slot_bytes;
    if (q == c->rank) continue;
    void *p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, hd.handle, cudaIpcMemLazyEnablePeerAccess));
    c->ipcPeer[(size_t)q] = (char *)p;
  }
  c->ipc = true;
  return SWE_OK;
}

int swe_get_decisions(swe_ctx *h, uint8_t *log, int64_t *nrec) {
  if (!h || !nrec) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  if (!c->prm.record_decisions) {
    c->err = "swe_get_decisions: record_decisions is off";
    return SWE_ERR_STATE;
  }
  if (!log) {
    *nrec = c->ndec;
    return SWE_OK;
  }
  const int64_t n = std::max<int64_t>(0, std::min<int64_t>(*nrec, c->ndec));
  std::memcpy(log, c->declog.data(), (size_t)n * (size_t)c->Kin);
  *nrec = n;
  return SWE_OK;
}

int swe_profile(swe_ctx *h, int on) {
  if (!h) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  c->prof = on != 0;
  if (on) {
    c->prof_ms[0] = c->prof_ms[1] = 0;
    c->prof_bytes[0] = c->prof_bytes[1] = 0;
    c->prof_launch[0] = c->prof_launch[1] = 0;
  }
  return SWE_OK;
}

int swe_profile_read(swe_ctx *h, double *times_ms, int64_t *launches, double *bytes) {
  if (!h) return SWE_ERR_ARG;
  Ctx *c = &h->c;
  for (int i = 0; i < 2; i++) {
    if (times_ms) times_ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_launch[i];
    if (bytes) bytes[i] = c->prof_bytes[i];
  }
  return SWE_OK;
}

int swe_host_halo_plan(const swe_mesh *mesh, const int64_t *gid, const int32_t *owner, int rank, int32_t *counts,
                       int32_t *peers, int64_t *send_gids, int64_t *recv_gids) {
  if (!mesh || !owner || !counts) return SWE_ERR_ARG;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  std::vector<int64_t> g(m.K);
  for (int e = 0; e < m.K; e++) g[e] = gid ? gid[e] : e;
  HaloPlan plan;
  build_halo_plan(m, g.data(), owner, rank, plan);
  int np = (int)plan.peers.size();
  counts[0] = (int32_t)plan.owned.size();
  counts[1] = (int32_t)plan.ghosts.size();
  counts[2] = np;
  size_t ns = 0, nr = 0;
  for (int i = 0; i < np; i++) {
    if (peers) peers[3 * i] = plan.peers[i];
    if (peers) peers[3 * i + 1] = (int32_t)plan.send[i].size();
    if (peers) peers[3 * i + 2] = (int32_t)plan.recv[i].size();
    for (int e : plan.send[i])
      if (send_gids) send_gids[ns++] = g[e];
    for (int e : plan.recv[i])
      if (recv_gids) recv_gids[nr++] = g[e];
  }
  return SWE_OK;
}

// ------------------------------------------------------------------ host-only builders
int swe_host_refel(int N, const char *name, double *out, int32_t *rows, int32_t *cols) {
  if (!name) return SWE_ERR_ARG;
  RefOps o;
  std::string err;
  if (!build_refops(N, o, &err)) return SWE_ERR_ORDER;
  std::string n(name);
  std::vector<double> v;
  int r = 0, cc = 1;
  auto vec = [&](const std::vector<double> &a) {
    v = a;
    r = (int)a.size();
    cc = 1;
  };
  auto mat = [&](const DMat &m) {
    v = m.a;
    r = m.rows;
    cc = m.cols;
  };
  if (n == "r") vec(o.r);
  else if (n == "s") vec(o.s);
  else if (n == "rc") vec(o.rc);
  else if (n == "sc") vec(o.sc);
  else if (n == "wc") vec(o.wc);
  else if (n == "tg") vec(o.tg);
  else if (n == "wg") vec(o.wg);
  else if (n == "wmean") vec(o.wmean);
  else if (n == "Dr") mat(o.Dr);
  else if (n == "Ds") mat(o.Ds);
  else if (n == "Mref") mat(o.Mref);
  else if (n == "Ic") mat(o.Ic);
  else if (n == "Ig") mat(o.Ig);
  else if (n == "P") mat(o.P);
  else if (n == "Pr") mat(o.Pr);
  else if (n == "Ps") mat(o.Ps);
  else if (n == "Lg") mat(o.Lg);
  else if (n == "Pv") mat(o.Pv);
  else if (n == "Ig1") mat(o.Ig1);
  else return SWE_ERR_ARG;
  if (rows) *rows = r;
  if (cols) *cols = cc;
  if (out) std::copy(v.begin(), v.end(), out);
  return SWE_OK;
}

int swe_host_connectivity(const swe_mesh *mesh, int32_t *etoe, int8_t *etof, int32_t *nflipped) {
  if (!mesh || !etoe || !etof) return SWE_ERR_ARG;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  std::copy(m.etoe.begin(), m.etoe.end(), etoe);
  std::copy(m.etof.begin(), m.etof.end(), etof);
  if (nflipped) *nflipped = m.nflipped;
  return SWE_OK;
}

int swe_host_hk(const swe_mesh *mesh, double *hk) {
  if (!mesh || !hk) return SWE_ERR_ARG;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  std::copy(m.hk.begin(), m.hk.end(), hk);
  return SWE_OK;
}

int swe_host_levels(const swe_mesh *mesh, int N, double g, const double *h, const double *hu, const double *hv,
                    const swe_params *params, int nlevels, int32_t *level) {
  if (!mesh || !h || !hu || !hv || !level || nlevels < 1 || nlevels > 8) return SWE_ERR_ARG;
  if (N < 1 || N > 8) return SWE_ERR_ORDER;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  swe_params p;
  fill_defaults(p, params);
  int Np = (N + 1) * (N + 2) / 2;
  std::vector<double> ae(m.K);
  element_speeds(m.K, Np, g, p.eps_u, p.a_floor, h, hu, hv, ae.data());
  bin_levels(m.K, m.hk.data(), ae.data(), nlevels, level);
  return SWE_OK;
}

int swe_host_tvb_geometry(const swe_mesh *mesh, int32_t *pairs, double *alphas) {
  if (!mesh || !pairs || !alphas) return SWE_ERR_ARG;
  HostMesh m;
  std::string err;
  int rc = build_mesh(mesh->nverts, mesh->vx, mesh->vy, mesh->nelems, mesh->etov, mesh->vperiodic, m, &err);
  if (rc) return rc;
  TvbGeom t;
  build_tvb_geometry(m, t);
  for (size_t i = 0; i < (size_t)3 * m.K; i++) {
    pairs[2 * i] = t.pj[i];
    pairs[2 * i + 1] = t.pk[i];
    alphas[2 * i] = t.aj[i];
    alphas[2 * i + 1] = t.ak[i];
  }
  return SWE_OK;
}

}  // extern "C"
