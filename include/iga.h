/*
 * iga.h -- C ABI of libiga: Galerkin residual / Jacobian assembly on tensor-product
 * B-spline / NURBS spaces, B200 (sm_100a) fp64 CUDA.  arXiv:1305.4452 ("PetIGA").
 *
 * The four calls follow the paper's statement of the problem:
 *   iga_space_create   -- an IGA space: dim, degree, knots, continuity (periodic
 *                         unclamping, Alg. 1), control points and weights
 *                         (NURBS, eqs. rational), dofs per node
 *   iga_csr_pattern    -- the CSR nonzero pattern from the knot vectors (Alg. 3, P:468-484;
 *                         "preallocation is crucial for efficient matrix assembly" P:444-446)
 *   iga_form_residual  -- FormVector, Alg. 4
 *   iga_form_jacobian  -- the matrix analogue, J = a dR/dUdot + b dR/dU
 *                         (generalized-alpha Newton matrix)
 *
 * Conventions:
 *  - Plain pointers only.  "device" = CUDA device memory on the space's device (allocated
 *    by the caller, e.g. with torch); "host" = ordinary host memory.
 *  - Numbering: node (i0,i1,i2) of the unique (periodic-identified) functions has flat index
 *    (i0*n1 + i1)*n2 + i2 (last parametric axis fastest); global dof = node*dof + component.
 *  - Vectors (U, Udot, F) are owned-rows-only in that order (single GPU: all rows).
 *  - CSR: row_ptr int64 [nrows+1] (config 5 has 4.19e9 nonzeros > 2^31), col_idx int32 [nnz]
 *    global dof indices, ascending within each row; csr_val fp64 [nnz].
 *  - Every call that takes a cudaStream_t (passed as void*) is asynchronous on that stream
 *    and allocates no device memory (iga_gmres and iga_form_jacobian_host excepted, see
 *    there).  Buffers must stay alive
 *    until the stream reaches them.
 *  - Errors: every call returns an iga_status; iga_last_error() gives a thread-local message.
 *    Argument / knot / continuity validation is synchronous.  Device-side conditions
 *    (detJ <= 0, SURVEY A-7; non-finite integrand) set a device flag that
 *    iga_space_check() reports after a stream synchronisation.
 *  - There is no CPU fallback: without a usable CUDA device every call fails with
 *    IGA_ERR_CUDA.
 */
#ifndef IGA_H
#define IGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IGA_OK = 0,
    IGA_ERR_PARAM = 1,        /* bad argument / unsupported combination                 */
    IGA_ERR_DOMAIN = 2,       /* knots not non-decreasing, continuity out of range, ...  */
    IGA_ERR_SINGULAR_MAP = 3, /* detJ <= 0 at a quadrature point (A-7)                   */
    IGA_ERR_PATTERN = 4,      /* a contribution outside the Alg. 3 pattern (debug)       */
    IGA_ERR_NONFINITE = 5,    /* non-finite residual / Jacobian coefficient              */
    IGA_ERR_CUDA = 6,
    IGA_ERR_COMM = 7,
    IGA_ERR_NOMEM = 8,
    IGA_ERR_STATE = 9
} iga_status;

typedef struct iga_space_s *iga_space;    /* opaque, library-owned */

typedef enum { IGA_GEOM_PARAMETRIC = 0, IGA_GEOM_NURBS = 1 } iga_geom;

typedef struct {
    int dim;                       /* 2 or 3 (parametric dim = spatial dim); 1 => IGA_ERR_PARAM */
    int degree[3];                 /* p_d in [1,3]; the form calls need one p on every axis in
                                      this build (IGA_ERR_PARAM otherwise)                       */
    int n_knots[3];                /* knots on axis d                                          */
    const double *knots[3];        /* host; OPEN (clamped) knot vectors, non-decreasing        */
    int periodic[3];               /* 1 => unclamp axis d with Alg. 1 for C^k periodicity      */
    int periodic_continuity[3];    /* k_d in [0, p_d-1] (read only when periodic)              */
    int dof;                       /* m dofs per node, 1..4                                    */
    int quad[3];                   /* Gauss points per dimension: 0 or p_d+1 (A-6); any other
                                      count => IGA_ERR_PARAM in this build                       */
    int geometry;                  /* iga_geom: PARAMETRIC => x = xi (knots carry coordinates)  */
    const double *ctrl;            /* host [n0][n1][n2][dim] Euclidean control points (NURBS)  */
    const double *weights;         /* host [n0][n1][n2] projective weights > 0, NULL => 1      */
    /* ctrl / weights live on the OPEN function grid, n_d = n_knots[d] - degree[d] - 1.  On a
     * periodic axis they are the clamped net of a C^k-periodic geometry: the library unclamps
     * every line with Alg. 2 in homogeneous coordinates (w x, w) and keeps the
     * n_d - (k+1) unique points; if the last k+1 unclamped points of a line do not repeat its
     * first k+1 (within 1e-10 relative) the geometry is not periodic: IGA_ERR_DOMAIN. */
} iga_space_desc;

/* Box decomposition of the element grid over ranks ("partitioning of the
 * [parametric] domain").  NULL => one rank owns everything.
 * procs[d] ranks along axis d, rank = (r0*p1+r1)*p2+r2; elements of axis d split as
 * b_r = floor(N r / P); a function belongs to the rank owning the last element of
 * its support (SURVEY A-9), so every rank's touched-but-not-owned ("halo") functions sit just
 * above its owned range and belong to its upper neighbours.  Each rank needs >= p elements per
 * partitioned axis (IGA_ERR_PARAM otherwise).
 * transport: IGA_XPORT_NCCL -- one process per GPU; nccl_id is an ncclUniqueId (from
 *            iga_nccl_unique_id on one rank, broadcast by the caller) identical on all ranks;
 *            iga_form_* then run the ghost / halo exchanges with NCCL send/recv on the stream.
 *            IGA_XPORT_LOCAL -- all ranks' spaces live in this process (one GPU; tests): the
 *            forms go through iga_form_*_group, exchanges are device copies. */
enum { IGA_XPORT_NCCL = 0, IGA_XPORT_LOCAL = 1 };
typedef struct {
    int rank;
    int nranks;
    int procs[3];
    int transport;
    unsigned char nccl_id[128];
} iga_dist;

/* One message of the halo-row exchange (the ghost-U exchange is the same list reversed):
 * subbox = bits (axis 0 = 4, axis 1 = 2, axis 2 = 1) of the axes on which the box is the halo
 * layer; box_lo/box_n = the box in the touched-box (send) or owned-box (receive) local indices
 * of the reporting rank; rows = nodes * dof; values = CSR values of those full rows. */
typedef struct {
    int peer;
    int subbox;
    int64_t rows;
    int64_t values;
    int box_lo[3];
    int box_n[3];
} iga_msg;

/* Host only -- needs no GPU and allocates nothing on a device: the decomposition seen by rank
 * dist->rank (owned function box [own_lo, own_hi), element box [el_lo, el_hi), touched box
 * extent ext_n = owned + halo per axis) and its messages: `send` = its halo rows to their
 * owners, `recv` = partial rows from its lower neighbours.  Up to max_msgs of each are
 * written; *nsend / *nrecv give the full counts (at most 7 each). */
iga_status iga_dist_plan(const iga_space_desc *desc, const iga_dist *dist, int64_t own_lo[3],
                         int64_t own_hi[3], int64_t el_lo[3], int64_t el_hi[3], int64_t ext_n[3],
                         int max_msgs, iga_msg *send, int *nsend, iga_msg *recv, int *nrecv);

/* A fresh ncclUniqueId (128 bytes) for IGA_XPORT_NCCL (dlopen's libnccl.so.2). */
iga_status iga_nccl_unique_id(unsigned char out[128]);

/* Create a space on CUDA device `device`.  Copies all host inputs.  Builds the per-axis
 * quadrature rule (Gauss-Legendre, A-6), the 1D basis tables at the Gauss points (kernel K1)
 * and the per-axis Alg. 3 stencils.  Returns IGA_ERR_DOMAIN for invalid knots. */
iga_status iga_space_create(const iga_space_desc *desc, const iga_dist *dist, int device,
                            iga_space *out);
iga_status iga_space_destroy(iga_space s);

/* Sizes (host outputs; any pointer may be NULL):
 *   ndof_global  -- total dofs;  nrows_owned -- rows this rank owns;  nnz_owned -- nonzeros
 *   in those rows;  nqp_local -- quadrature points of this rank's elements;
 *   owned_lo/hi[3] -- owned node box [lo,hi) per axis;  elem_lo/hi[3] -- element box. */
iga_status iga_space_info(iga_space s, int64_t *ndof_global, int64_t *nrows_owned,
                          int64_t *nnz_owned, int64_t *nqp_local, int64_t owned_lo[3],
                          int64_t owned_hi[3], int64_t elem_lo[3], int64_t elem_hi[3]);

/* CSR pattern of the owned rows (kernel K2): Alg. 3 per axis x tensor product x dof blocks,
 * sorted ascending.  row_ptr: device int64[nrows_owned+1] (starts at 0); col_idx: device
 * int32[nnz_owned].  stream: cudaStream_t. */
iga_status iga_csr_pattern(iga_space s, int64_t *row_ptr, int32_t *col_idx, void *stream);

/* Physics (the paper's "user integrand", is a closed set here) */
typedef enum {
    IGA_PHYS_LAPLACE = 0,        /* p = [kappa, sigma, source_id]; m = 1                      */
    IGA_PHYS_CAHN_HILLIARD = 1,  /* p = [theta, alpha]; m = 1; needs Hessians      */
    IGA_PHYS_NEOHOOKE = 2,       /* p = [lambda, mu]; m = 3, dim 3                 */
    IGA_PHYS_NS_VMS = 3,         /* p = [nu, dt, C_t, C_I]; m = 4, dim 3, parametric*/
    IGA_PHYS_NSK = 4             /* p = [a, b, R, theta, mu_bar, lambda_bar, lambda]; m = 3 (rho, u),
                                    dim 2, Navier-Stokes-Korteweg */
} iga_phys_kind;

typedef struct {
    int kind;
    double p[8];
} iga_phys;

/* Residual R(U, Udot) (Alg. 4).  U, Udot: device fp64 [nrows_owned] (the owned box, node-major,
 * dof innermost; = all dofs on a single rank) -- Udot may be NULL (=> 0).  F: device fp64
 * [nrows_owned], overwritten.  Multi-rank (IGA_XPORT_NCCL): collective over all ranks (every
 * rank calls with its owned vectors); the ghost-U and halo exchanges run on `stream`. */
iga_status iga_form_residual(iga_space s, const iga_phys *phys, const double *U,
                             const double *Udot, double *F, void *stream);

/* Jacobian J = a dR/dUdot + b dR/dU into csr_val (device fp64 [nnz_owned], overwritten, in
 * the order of iga_csr_pattern); if F is non-NULL the residual is formed in the same pass. */
iga_status iga_form_jacobian(iga_space s, const iga_phys *phys, double a, double b,
                             const double *U, const double *Udot, double *csr_val, double *F,
                             void *stream);

/* Host-buffer variant (end-to-end path): copies U/Udot host->device, forms J (and F if
 * F_host != NULL) and copies csr_val / F back, all on `stream`; returns after the stream
 * synchronises.  Host buffers should be pinned for full PCIe bandwidth.
 * On 3D spaces with uniform knots along axis 0 the elements are assembled in slabs along axis 0
 * (option "hb_slabs", default 32; 0 = one launch) and each node layer's CSR rows are copied back
 * on a second stream as soon as the last element touching the layer is assembled, so the copy
 * of the values overlaps the assembly.
 * Device memory: the first call allocates the device staging buffers (2 ndof + nnz + nrows
 * doubles: 34 GB for config 5) and keeps them with the space (freed by iga_space_destroy);
 * IGA_ERR_NOMEM if that allocation fails.  Single-rank spaces only (IGA_ERR_STATE otherwise). */
iga_status iga_form_jacobian_host(iga_space s, const iga_phys *phys, double a, double b,
                                  const double *U_host, const double *Udot_host,
                                  double *csr_val_host, double *F_host, void *stream);

/* In-process multi-rank forms (IGA_XPORT_LOCAL): spaces[k] must be rank k of the same
 * decomposition, all on one device; U[k], Udot[k] (NULL entries allowed for Udot when all are
 * NULL), csr_val[k], F[k] are that rank's owned vectors / values (device).  Ranks' kernels run
 * one after another on `stream`, the exchanges are device copies between their buffers. */
iga_status iga_form_jacobian_group(int n, const iga_space *spaces, const iga_phys *phys, double a,
                                   double b, const double *const *U, const double *const *Udot,
                                   double *const *csr_val, double *const *F, void *stream);
iga_status iga_form_residual_group(int n, const iga_space *spaces, const iga_phys *phys,
                                   const double *const *U, const double *const *Udot,
                                   double *const *F, void *stream);

/* Basis evaluation at the quadrature points -- Alg. 4's "Basis(G_e, x_q)" extended to
 * the third spatial derivatives the paper derives for higher-order PDEs on mapped geometry:
 * (dddrational) P:248-255, the inverse-map derivatives P:316-340, (dspatial)-(dddspatial)
 * P:309-315.  For every element of this rank (element box, C order, last axis fastest), every
 * local function A of the element (C order) and every Gauss point q of the element (C order):
 *   out[((e * nen + A) * ncomp + c) * nq + q],  nen = prod(p_d+1), nq = prod(quad_d),
 *   components c: R_A; R_{A,i} (order >= 1); R_{A,ij} (order >= 2, i-major); R_{A,ijk} (order 3),
 *   ncomp = 1 + d + d^2 + d^3 (truncated at `order`).
 * out: device fp64, caller-allocated.  order in [0, 3]; IGA_ERR_PARAM otherwise.  A point with
 * detJ <= 0 sets the device flag (iga_space_check -> IGA_ERR_SINGULAR_MAP). */
iga_status iga_basis_eval(iga_space s, int order, double *out, void *stream);

/* Linear solve with the assembled Jacobian -- the Newton step's J dU = -F of the paper's
 * solver protocol (§5: "30 GMRES iterations per Newton iteration", "block Jacobi
 * ... ILU(0) ... in each block").  Right-preconditioned restarted GMRES(restart) (Saad-Schultz,
 * cited P:872), classical Gram-Schmidt applied twice, Givens rotations; stops when the
 * preconditioned-Krylov residual estimate |g_{j+1}| <= rtol * ||b|| or after maxit total
 * iterations.  Preconditioner `precond`: 0 none, 1 point Jacobi (diag), 2 block Jacobi with ILU(0)
 * (Saad's IKJ ILU(0), no fill) in each diagonal block of `block_rows` consecutive rows (0 -> 32;
 * reading A-28: the GPU's blocks are row runs, not one per process).  Entries outside the block
 * are not part of the preconditioner.
 * row_ptr/col_idx/val: this space's CSR (iga_csr_pattern + iga_form_jacobian), device, sorted
 * columns, every row holding its diagonal.  b (rhs) and x (initial guess in, solution out):
 * device fp64 of nrows_owned.  Workspace ((2 restart + 3) n doubles + the packed preconditioner,
 * or nnz doubles for blocks > 64 rows) is allocated on first use, kept with the space for later
 * calls and freed by iga_space_destroy; the call synchronises `stream`.
 * iters (total iterations) / relres (TRUE ||b - A x|| / ||b|| of the returned x) may be NULL.
 * Multi-rank spaces (box decomposition): with IGA_XPORT_NCCL every rank calls iga_gmres with
 * its owned rows (global column indices, as iga_csr_pattern returns them); in-process
 * (IGA_XPORT_LOCAL) ranks call iga_gmres_group.  The distributed solve exchanges a ghost layer
 * of width p of x per SpMV, all-reduces the Gram-Schmidt dots, and factors block-Jacobi ILU(0)
 * on each rank's owned-owned block (the paper's "one block per process", cut into block_rows
 * runs); it supports the fixed budget only (rtol = 0, IGA_ERR_PARAM otherwise) and restart <= 62.
 * IGA_ERR_NOMEM if the workspace does not fit. */
typedef struct {
    int restart;    /* m, Krylov dimension per cycle (paper: 30) */
    int maxit;      /* total iteration cap (paper: 30 per Newton step) */
    double rtol;    /* relative tolerance on ||b - A x|| / ||b|| */
    int precond;    /* 0 none, 1 Jacobi, 2 block-Jacobi ILU(0) */
    int block_rows; /* rows per block-Jacobi block (precond 2); 0 -> 32 */
} iga_krylov;
iga_status iga_gmres(iga_space s, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                     const double *b, double *x, const iga_krylov *opt, int *iters, double *relres,
                     void *stream);
/* Host only (no GPU): the distributed solve's ghost-exchange plan of rank dist->rank.  The
 * extended box (owned box + `ghost` = p layers on each side of the partitioned axes) has extent
 * ext_n; messages are boxes of it in node units (box_lo / box_n), `rows` = nodes * dof values,
 * `subbox` = ((o0+1)*3 + (o1+1))*3 + (o2+1) for the neighbour offset o in {-1,0,1}^3, `values` = 0.
 * send[k]: this rank's owned slab on side o, to the rank at coordinate + o, ascending o;
 * recv[k]: its ghost layer on side o, from the rank at coordinate + o, descending o (the order a
 * grouped NCCL exchange pairs repeated peers in).  Up to max_msgs each; counts in nsend / nrecv. */
iga_status iga_krylov_plan(const iga_space_desc *desc, const iga_dist *dist, int64_t own_lo[3],
                           int64_t own_hi[3], int64_t ext_n[3], int64_t ghost[3], int max_msgs,
                           iga_msg *send, int *nsend, iga_msg *recv, int *nrecv);

/* All n in-process ranks (IGA_XPORT_LOCAL spaces, rank k = spaces[k]) solve together on one
 * stream; per-rank arrays as for iga_gmres; iters / relres are global. */
iga_status iga_gmres_group(int n, const iga_space *spaces, const int64_t *const *row_ptr,
                           const int32_t *const *col_idx, const double *const *val,
                           const double *const *b, double *const *x, const iga_krylov *opt,
                           int *iters, double *relres, void *stream);

/* One generalized-alpha time step with a fixed-budget Newton loop -- eq. (ga) of P:697-709 with
 * the rho_inf parametrisation of P:719-723 (am = (3 - rho)/(2 (1 + rho)), af = 1/(1 + rho),
 * gamma = 1/2 + am - af), Newton on Udot_{n+1} from the constant-U predictor
 * U_{n+1} = U_n, Udot_{n+1} = (gamma - 1)/gamma Udot_n (reading A-29), and the §5 protocol
 * (P:866-876): exactly `newton_its` iterations, each
 *     assemble R(U_{n+af}, Udot_{n+am}) and J = am dR/dUdot + af gamma dt dR/dU (iga_form_jacobian),
 *     solve J dx = R with iga_gmres(krylov) from x = 0,   Udot_{n+1} -= dx,  U_{n+1} -= gamma dt dx.
 * No convergence test (the paper's fixed budget: 2 Newton x 30 GMRES).  row_ptr/col_idx: this
 * space's pattern; val: caller's device buffer of nnz doubles (holds the last Jacobian on
 * return).  U, Udot: device, all rows; in: step n, out: step n+1.  Physics time-step parameters
 * (e.g. NS-VMS p[1] = dt) are the caller's to keep consistent with opt->dt.  stats (may be NULL):
 * ||R|| at each Newton iterate and each solve's iterations / true relative residual.
 * Multi-rank: IGA_XPORT_NCCL ranks each call iga_alpha_step with their owned vectors (the forms
 * and the distributed GMRES exchange internally; the fixed GMRES budget rtol = 0 is required);
 * in-process ranks call iga_alpha_step_group.  newton_its in [1, 8]; 0 <= rho_inf <= 1; dt > 0
 * (IGA_ERR_PARAM otherwise).
 * Stage vectors (6 n doubles) are kept with the space; the call synchronises `stream`. */
typedef struct {
    double rho_inf;
    double dt;
    int newton_its;     /* paper: 2 */
    iga_krylov krylov;  /* paper: GMRES, 30 iterations, block-Jacobi ILU(0) */
} iga_alpha;
typedef struct {
    double res_norm[8];       /* ||R(U_{n+af}, Udot_{n+am})|| at Newton iterate k */
    int gmres_its[8];
    double gmres_relres[8];
} iga_step_stats;
iga_status iga_alpha_step(iga_space s, const iga_phys *phys, const iga_alpha *opt, const int64_t *row_ptr,
                          const int32_t *col_idx, double *val, double *U, double *Udot,
                          iga_step_stats *stats, void *stream);
iga_status iga_alpha_step_group(int n, const iga_space *spaces, const iga_phys *phys, const iga_alpha *opt,
                                const int64_t *const *row_ptr, const int32_t *const *col_idx,
                                double *const *val, double *const *U, double *const *Udot,
                                iga_step_stats *stats, void *stream);

/* Synchronises `stream` and reports (then clears) the device error flag of the last form
 * call: IGA_OK, IGA_ERR_SINGULAR_MAP or IGA_ERR_NONFINITE. */
iga_status iga_space_check(iga_space s, void *stream);

/* Tuning / testing options: "split" = 1 forces the generic two-kernel path (pointwise kernel +
 * contraction kernel through an HBM workspace) instead of the fused kernels; "general" = 1
 * disables the uniform-table fast paths (per-element tables always read from memory); 0
 * restores the default.  Returns IGA_ERR_PARAM for an unknown key. */
iga_status iga_space_set_option(iga_space s, const char *key, long long value);

/* Number of kernel launches the last form / pattern call issued (for the bench's gpu_launches). */
int iga_last_launch_count(iga_space s);

/* Kernel-level timing hook (bench only).  When enabled, every kernel a call launches is
 * bracketed by CUDA events recorded on that call's stream.  iga_profile_read synchronises the
 * recorded events and returns, per kernel name (up to `max` names of < 32 chars), the number
 * of launches and the summed device time in ms since the last reset; returns the count of
 * names, or -1 on error. */
iga_status iga_profile_enable(iga_space s, int on);
iga_status iga_profile_reset(iga_space s);
int iga_profile_read(iga_space s, int max, char *names /* [max][32] */, int *launches, double *ms);

/* Diagnostics (K8): measured ceilings on this device.  which: 0 DFMA flop/s, 1 DMMA
 * (mma.sync m8n8k4 f64) flop/s, 2 DFMA+DMMA mixed flop/s, 3/4/5 fp64 red.add per second with
 * 32/4/1 lanes per contiguous group into a `param`-double (default 26 MB) array, 6 store
 * bytes/s, 7 shared-memory fp64 atomics/s, 8/10 bulk reductions (96/384 B) per second, 9 fp64
 * red.add/s in the config-5 lane pattern, 11/12 warp-level 128-bit broadcast loads per second
 * (4 distinct addresses per warp, shared memory / L1-resident global).  Returns < 0 on error. */
double iga_microbench(int device, int which, long long param);

const char *iga_last_error(void);
const char *iga_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IGA_H */
