/* include/swe.h -- C ABI of the B200-native DG shallow-water solver.
 *
 * Implements the data-parallel hot path of arXiv:1403.1661 (PAPER.md, cited
 * as P:n = line n): the nodal discontinuous-Galerkin right-hand side of the
 * 2D shallow water equations on unstructured triangles (Eqs. 1-6:
 * volume term N(Q) = Pr cF1 + Ps cF2 + P cS; surface term
 * S = -L^g F*_n; well-balanced Lax-Friedrichs flux),
 * advanced by multi-rate Adams-Bashforth local time stepping (P:115-147,
 * Alg. 1) with the positivity-preserving limiter M Pi (Alg. 3) and
 * the TVB limiter Lambda Pi after every update (Alg. 2).
 * The readings of the paper that this library implements are listed in
 * DESIGN.md ("Readings").
 *
 * Conventions (all calls):
 *   - Every pointer argument is HOST memory owned by the caller.  Inputs are
 *     copied during the call and never retained; outputs are written before
 *     the call returns.
 *   - Nodal arrays are [element][node] in the caller's element order, node
 *     order = Hesthaven-Warburton Nodes2D of the element AFTER the orientation
 *     fix (rows of constant s from s = -1 upward, r increasing in a row;
 *     N = 2: (-1,-1),(0,-1),(1,-1),(-1,0),(0,0),(-1,1)), reference triangle
 *     (-1,-1),(1,-1),(-1,1), face f runs vertex f -> vertex (f+1)%3.
 *     swe_nodes() returns the physical coordinates of those nodes.
 *   - Clockwise triangles are re-oriented by swapping their 2nd and 3rd
 *     vertex (counted in swe_info.nflipped).
 *   - Errors are negative return codes; nothing aborts.  The message of the
 *     last error of a context is available from swe_last_error().
 *   - A context is not thread-safe; distinct contexts are independent.
 *   - Arithmetic is IEEE binary64 throughout (device and host), unless swe_params.precision
 *     selects the FP32 variant for the device state and kernels.
 */
#ifndef SWE_H
#define SWE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SWE_OK = 0,
  SWE_ERR_ARG = -1,       /* invalid argument (NULL, size, dt <= 0, nlevels out of [1,8]) */
  SWE_ERR_MESH = -2,      /* vertex index out of range, zero-area element, face with > 2 owners */
  SWE_ERR_ORDER = -3,     /* polynomial order outside the supported range [1, 5] (order 5 with integration order 10) */
  SWE_ERR_STATE = -4,     /* swe_step / swe_get_state before swe_set_state */
  SWE_ERR_SCHEDULE = -5,  /* (dt, nlevels) differ from the first swe_step after swe_set_state */
  SWE_ERR_NONFINITE = -6, /* NaN/Inf produced; the state is left as computed */
  SWE_ERR_CUDA = -7,      /* CUDA runtime error, or no device */
  SWE_ERR_NCCL = -8,      /* reserved for the multi-GPU exchange */
  SWE_ERR_NOMEM = -9      /* device allocation failed */
};

typedef struct swe_ctx swe_ctx;

/* Conforming triangulation.  Faces are matched on the sorted pair of
 * canonical vertex ids vperiodic[v] (identity when NULL), which is how
 * periodic partners are expressed.  Unmatched faces are reflective walls. */
typedef struct {
  int32_t nverts;
  const double *vx, *vy;      /* [nverts] */
  int32_t nelems;
  const int32_t *etov;        /* [nelems*3], 0-based vertex indices */
  const int32_t *vperiodic;   /* [nverts] or NULL */
  /* Boundary tags [nverts] or NULL: an unmatched face whose two vertices are both tagged (>= 1) takes
   * the smaller tag -- 1: transmissive outflow (reading A7': ghost state = interior trace, TVB ghost
   * mean = own mean), 2: Dirichlet (reading A7'': swe_set_boundary_state); every other unmatched face
   * is a reflective wall. */
  const int8_t *vbc;
} swe_mesh;

/* Parameters; a zero-initialised struct (or NULL) selects the defaults. */
typedef struct {
  double h0;       /* dry threshold of Alg. 3, default 1e-6 */
  double eps;      /* Alg. 3 trigger: limit when min nodal h <= eps, default h0 */
  double tvb_M;    /* TVB constant M, threshold M*Hk^2 (default 0 = TVD minmod) */
  double tvb_nu;   /* Cockburn-Shu nu, default 1.5 */
  double a_floor;  /* lower bound of the wave speed used for level binning, default 0 */
  double eps_u;    /* velocity desingularisation scale, default 1000*h0 (A4') */
  double h_char;   /* below this mean depth TVB limits component-wise, default 10*h0 */
  int32_t use_pp;  /* apply M Pi (Alg. 3); fields are used as given (NULL params => both on) */
  int32_t use_tvb; /* apply Lambda Pi */
  int32_t device;  /* CUDA device ordinal */
  void *stream;    /* cudaStream_t for all work (e.g. torch.cuda.current_stream()), NULL = legacy default */
  /* optional device allocator (e.g. the torch caching allocator); NULL => cudaMalloc/cudaFree */
  void *(*dev_alloc)(size_t bytes, void *stream, void *user);
  void (*dev_free)(void *ptr, void *stream, void *user);
  void *alloc_user;
  /* Multi-GPU (element partition).  nranks <= 1: single rank, every
   * element owned.  Otherwise every element of the given mesh carries an owner
   * rank (owner[nelems]) and a global id (gid[nelems], NULL => the index; gids
   * must agree across ranks for the elements the ranks share).  Each rank
   * advances the elements it owns; the non-owned face neighbours of owned
   * elements are ghosts refreshed by halo exchanges after every level update;
   * elements that are neither are ignored.  Transport: NCCL when nccl_id
   * (128-byte ncclUniqueId, same on all ranks, see swe_nccl_unique_id) is set;
   * otherwise several contexts of one process are linked with swe_link_group
   * and advanced with swe_step_group. */
  int32_t rank, nranks;
  const int32_t *owner;
  const int64_t *gid;
  const void *nccl_id;
  /* Arithmetic precision of the device state and kernels: 64 (or 0, default) = IEEE binary64; 32 = the
   * FP32 variant: state, history and kernels in binary32, host arrays still double,
   * level binning still from the binary64 input (bit-exact); parity target 1e-5 against the FP64 oracle
   * (DESIGN.md).  Other values: SWE_ERR_ARG. */
  int32_t precision;
  /* MRAB inter-level coupling: 0 (default) = reading A17, recursive slowest-first order with coarser
   * neighbours read mid-step through the AB3 dense output (third order); 1 = Alg. 1's loop nest as
   * printed (levels descending, substeps inner) with every neighbour at its latest committed
   * value (SPEC's reading, first order at level interfaces, kept for comparison). */
  int32_t mrab_coupling;
  /* Decision log for oracle replay (debug): nonzero => every limiter application (Alg. 2
   * line 1, then every level update) appends one record of nelems bytes to a host log, read with
   * swe_get_decisions.  Forces eager launches (no CUDA graphs) and one stream sync per update. */
  int32_t record_decisions;
} swe_params;

typedef struct {
  double t;              /* simulated time (sum of macro steps) */
  double mass;           /* sum_e J_e int h (current state) */
  double injected_mass;  /* mass added by the dry branch of Alg. 3 since swe_set_state */
  double min_h;          /* minimum nodal h */
  int64_t n_pp;          /* Alg. 3 triggers (h_min <= eps) */
  int64_t n_dry;         /* Alg. 3 dry-branch applications */
  int64_t n_tvb;         /* elements replaced by the TVB limiter */
  int64_t n_updates;     /* element updates (sum over launched levels) */
  int32_t K, Np, N, nlevels, nflipped;
  int32_t level_count[8];
  int64_t n_posfix;      /* TVB-replaced elements whose h needed Eq. modified_TVB (a P1 vertex below h0) */
  int64_t n_tvb_cw;      /* TVB-replaced elements limited component-wise (mean depth below h_char, A14) */
} swe_info;

/* ------------------------------------------------------------ solver */

/* Physical coordinates of the nodes of every element, [nelems*Np] each.
 * Host only (no device needed).  Returns SWE_OK or SWE_ERR_MESH/ORDER/ARG. */
int swe_nodes(const swe_mesh *mesh, int N, double *x, double *y);

/* Build a solver for order N in [1,5], gravity g > 0, nodal bathymetry B
 * ([nelems*Np], P^N per element).  Host builder (reference element, mesh
 * connectivity, geometry) + device upload.  On failure *out = NULL. */
int swe_create(const swe_mesh *mesh, const double *B, int N, double g, const swe_params *params,
               swe_ctx **out);

/* Set the nodal state (h, hu, hv), each [nelems*Np].  Resets time, the AB
 * start-up ramp, the counters and the level schedule; the limiters of Alg. 2
 * line 1 (Q^0 = Lambda Pi M Pi Q^0) are applied lazily by the next
 * swe_step / swe_get_state.  Levels are binned from this unlimited state. */
int swe_set_state(swe_ctx *ctx, const double *h, const double *hu, const double *hv);

/* One MRAB macro step of length 2^(nlevels-1)*dt (level l steps with
 * 2^(l-1) dt; dt is the finest level's step).  The first call after
 * swe_set_state bins the levels (Eq. cfl) and fixes them for the
 * run; later calls with another (dt, nlevels) fail with
 * SWE_ERR_SCHEDULE.  Synchronises the stream once to check for NaN/Inf. */
int swe_step(swe_ctx *ctx, double dt, int nlevels);

/* Copy the current state to the host, caller order, [nelems*Np] each. */
int swe_get_state(swe_ctx *ctx, double *h, double *hu, double *hv);

/* Output while the run goes on: enqueue a copy of the current state (the state after every call made so far) into
 * h, hu, hv ([nelems*Np] each, caller order) and return without waiting.  The state is first gathered on the device
 * into one of two context-owned snapshot buffers (3*nelems*Np doubles each, allocated on first use); the device->host
 * copy then runs on a separate copy stream, so the next swe_step computes while it crosses PCIe.  The host buffers
 * belong to the library until swe_wait_state returns: their contents are undefined before, and they must stay
 * allocated.  Pinned (page-locked) buffers are needed for the overlap; pageable ones give a correct, synchronous
 * copy.  With two snapshots in flight, the next call first waits (on the device) for the older one's copy.
 * Contexts of a multi-rank or in-process partition take the synchronous swe_get_state path. */
int swe_get_state_async(swe_ctx *ctx, double *h, double *hu, double *hv);

/* Wait until every swe_get_state_async copy of this context has reached the host. */
int swe_wait_state(swe_ctx *ctx);

/* Dirichlet boundary data (reading A7''; P:355 sets "Dirichlet boundary conditions ... to the exact
 * solution").  A boundary face whose two vertices are both tagged 2 in swe_mesh.vbc is a Dirichlet face:
 * its ghost state is the trace of the nodal state given here ([nelems*Np] each, caller layout; only the
 * face nodes of elements with Dirichlet faces are used), with B+ = B-, and its TVB ghost mean is that
 * state's cell mean.  The data stay until the next call (call it between swe_step calls to follow a
 * time-dependent boundary; it is held constant during a macro step).  swe_step / swe_get_state return
 * SWE_ERR_STATE while a mesh with Dirichlet faces has no boundary state. */
int swe_set_boundary_state(swe_ctx *ctx, const double *h, const double *hu, const double *hv);

/* Level regrouping ("elements can be regrouped after every few time steps"):
 * the current state becomes the state of a fresh swe_set_state -- levels re-binned at the next
 * swe_step (which may use a new dt and nlevels), Alg. 2 line 1 applied to it, AB ramp and counters
 * restarted -- while swe_info.t continues.  Single-rank contexts (nranks <= 1) only: SWE_ERR_ARG
 * otherwise; SWE_ERR_STATE before swe_set_state. */
int swe_regroup(swe_ctx *ctx);

void swe_destroy(swe_ctx *ctx); /* NULL-safe; frees all device memory */

/* ------------------------------------------------------------ multi-rank */
/* A fresh NCCL unique id (128 bytes) for swe_params.nccl_id; call on one rank and broadcast. */
int swe_nccl_unique_id(void *id128);
/* Link n contexts of this process (ranks 0..n-1 of one partition, same device and stream) so that
 * swe_step_group advances them together with in-process halo copies (one-GPU validation of the
 * partitioned path).  swe_get_state / swe_get_info of a linked context materialise the group. */
int swe_link_group(swe_ctx **ctxs, int n);
int swe_step_group(swe_ctx **ctxs, int n, double dt, int nlevels);

/* CUDA-IPC transport (NVLink peer memory; also two or more ranks sharing one GPU, where NCCL
 * refuses to run).  Every rank of an nranks > 1 partition exports its exchange block (a cudaMalloc'ed
 * header with the exchange flags plus two send slots) and maps every other rank's.  An exchange is then:
 * pack into the own send slot (exchange count mod 2), cuStreamWriteValue64 of the own flag, and per
 * neighbour cuStreamWaitValue64 on its flag followed by a device copy of the neighbour's segment straight
 * out of its send slot (peer reads over NVLink).  r_min for the level binning is reduced over all ranks the
 * same way.
 *   swe_ipc_handle: blob = NULL -> *bytes = blob size; else writes this rank's blob (device handle, send
 *                   layout offsets).  Call on every rank, gather the blobs in rank order (e.g. with
 *                   torch.distributed.all_gather_object), then
 *   swe_ipc_open:   blobs = nranks blobs of that size, rank order; maps the peers' blocks and selects the
 *                   IPC transport for swe_step.  SWE_ERR_MESH if two ranks' halo plans disagree. */
int swe_ipc_handle(swe_ctx *ctx, void *blob, size_t *bytes);
int swe_ipc_open(swe_ctx *ctx, const void *blobs);

/* ------------------------------------------------------------ introspection */
/* Decision log (swe_params.record_decisions): nrec records of nelems bytes, caller element
 * order, one per limiter application since swe_set_state: bit 1 Alg. 3 triggered, 2 dry branch
 * (P:206), 4 replaced by the TVB limiter, 8 Eq. modified_TVB applied; 0xFF = element
 * not updated by that application (other level, or not owned).  log = NULL: *nrec receives the record
 * count; otherwise min(*nrec, count) records are copied and *nrec is set to that number.
 * SWE_ERR_STATE if recording is off. */
int swe_get_decisions(swe_ctx *ctx, uint8_t *log, int64_t *nrec);
int swe_get_levels(swe_ctx *ctx, int32_t *level);                       /* [nelems], 1..nlevels */
int swe_get_connectivity(const swe_ctx *ctx, int32_t *etoe, int8_t *etof); /* [nelems*3], boundary = self */
int swe_get_info(swe_ctx *ctx, swe_info *info);
const char *swe_last_error(const swe_ctx *ctx);

/* Per-kernel device time accumulated with CUDA events on the context stream
 * while profiling is on: times_ms[0] = K1 (RHS + AB update + PP), [1] = K2
 * (TVB); launches[] likewise; bytes[] = algorithmic bytes moved (DESIGN.md
 * roofline model).  swe_profile(ctx, 1) resets and starts, 0 stops. */
int swe_profile(swe_ctx *ctx, int on);
int swe_profile_read(swe_ctx *ctx, double *times_ms, int64_t *launches, double *bytes);

/* ------------------------------------------------------------ host-only builders (no device) */
/* Reference-element operator by name ("r","s","Dr","Ds","Mref","Ic","Ig","P","Pr","Ps","Lg",
 * "rc","sc","wc","tg","wg","wmean","Pv","Ig1"); rows/cols receive the shape, out may be NULL. */
int swe_host_refel(int N, const char *name, double *out, int32_t *rows, int32_t *cols);
/* Connectivity of a mesh exactly as swe_create builds it. */
int swe_host_connectivity(const swe_mesh *mesh, int32_t *etoe, int8_t *etof, int32_t *nflipped);
/* Element characteristic length Hk = 4A / perimeter (incircle diameter). */
int swe_host_hk(const swe_mesh *mesh, double *hk);
/* Level binning of a nodal state exactly as the first swe_step does it. */
int swe_host_levels(const swe_mesh *mesh, int N, double g, const double *h, const double *hu, const double *hv,
                    const swe_params *params, int nlevels, int32_t *level);
/* Static TVB geometry: pairs[K*3*2] (neighbour face slots used for edge i), alphas[K*3*2]. */
int swe_host_tvb_geometry(const swe_mesh *mesh, int32_t *pairs, double *alphas);
/* Halo plan of `rank`: counts = {owned, ghosts, npeers}; peers[3*i] = peer rank, [3*i+1] = send count,
 * [3*i+2] = receive count; send_gids / recv_gids: the lists concatenated in peer order (gid order
 * within a peer).  Any output pointer except counts may be NULL (query sizes first). */
int swe_host_halo_plan(const swe_mesh *mesh, const int64_t *gid, const int32_t *owner, int rank, int32_t *counts,
                       int32_t *peers, int64_t *send_gids, int64_t *recv_gids);

#ifdef __cplusplus
}
#endif

#endif /* SWE_H */
