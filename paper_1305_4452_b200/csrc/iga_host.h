// iga_host.h -- host-side state of an IGA space (libiga internals).
#pragma once
#include <string>
#include <vector>

#include "iga_internal.cuh"

namespace iga {
// per-axis host data (space.cu axis_host): everything about one parametric axis, including the
// box decomposition of its elements over all P rank coordinates
struct AxisHost {
    int p = 0, nel = 0, nu = 0, nfun = 0, nq = 0, periodic = 0, colmax = 1, uniform = 1;
    std::vector<double> U, hpar, qx, qw;
    std::vector<int> first, rowW, cols, pos, suplo, supcnt, posd;
    std::vector<int> el_lo, el_hi, own_lo, own_hi, halo;   // [P] per rank coordinate
};
iga_status axis_host(const iga_space_desc *d, int a, int P, AxisHost &H);
struct DistState;   // dist.cu: multi-rank buffers, exchange plan, transport
int dist_transport(const DistState *D);
}  // namespace iga

struct iga_space_s {
    int device = 0;
    iga::SpaceDev dev{};                 // device view (pointers into `allocs`)
    int dim = 0, dof = 1, geom = 0, weighted = 0, mode = 0;
    int p[3] = {0, 0, 0}, nel[3] = {1, 1, 1}, nu[3] = {1, 1, 1}, nq[3] = {1, 1, 1}, nfun[3] = {1, 1, 1};
    int periodic[3] = {0, 0, 0};
    std::vector<double> U[3];            // unclamped knot vectors
    std::vector<int> rowW[3];            // per axis stencil widths [nu]
    std::vector<int> cols[3];            // per axis column lists [nu][colmax]
    int colmax[3] = {1, 1, 1};
    // distribution (box decomposition)
    int rank = 0, nranks = 1, procs[3] = {1, 1, 1}, rcoord[3] = {0, 0, 0};
    int own_lo[3] = {0, 0, 0}, own_hi[3] = {1, 1, 1};
    int halo[3] = {0, 0, 0};             // halo functions per axis (touched, owned by the upper neighbour)
    long long Th[3] = {0, 0, 0};
    iga::AxisHost part[3];
    iga::DistState *dist = nullptr;
    // unclamped knot vectors on the device (third-order basis evaluation only; deliberately not in
    // SpaceDev, whose size the fused kernels' register allocation turned out to be sensitive to)
    const double *dknots[3] = {nullptr, nullptr, nullptr};
    double *hb_U = nullptr, *hb_Ud = nullptr, *hb_val = nullptr, *hb_F = nullptr;   // host-buffer path staging
    int hb_slabs = 32;                   // host path: element slabs along axis 0 whose finished rows are
                                         // copied back while later slabs assemble (option "hb_slabs", 0 = off)
    cudaStream_t hb_copy = nullptr;      // host path: device-to-host copy stream
    std::vector<cudaEvent_t> hb_ev;      // host path: one event per slab
    int el_lo[3] = {0, 0, 0}, el_hi[3] = {1, 1, 1};
    long long ndof_global = 0, nrows_owned = 0, nnz_owned = 0, nqp_local = 0, nel_local = 0;
    // device allocations owned by the space
    std::vector<void *> allocs;
    double *work = nullptr;              // per-batch quadrature-point coefficient workspace
    size_t work_bytes = 0;
    int *errflag = nullptr;
    int last_launches = 0;
    int force_split = 0;
    int force_general = 0;
    int bw_opt = 0;                      // 3D element-order block width override (0: from the L2 size)
    int skip_zero = 0;                   // dist.cu: the caller zeroed the outputs (sub-box launches)
    int last_occupancy = 0;
    int dbg = 0;                         // experiment bits (bench A/B only; results invalid when set)
    // per axis: all elements share the same 1D tables / weights / span length (uniform knots,
    // translation invariance; equal to 1e-13 relative) -> element-0 copies (host)
    int tab_uniform[3] = {0, 0, 0};
    std::vector<double> tab0[3], qw0[3];
    double hp0[3] = {1.0, 1.0, 1.0};
    // iga_gmres workspace (solver.cu): [0] Krylov vectors, [1] preconditioner; kept until destroy;
    // iga_alpha_step: [2] its stage vectors
    void *gm_buf[3] = {nullptr, nullptr, nullptr};
    int gm_host_ctrl = 0;                // option "gmres_host": host-side Arnoldi control even at rtol = 0
    size_t gm_cap[3] = {0, 0, 0};
    // distributed-GMRES workspace (gmres_group): the k-th allocation of a solve reuses slot k when
    // it is large enough, so repeated solves (one per Newton iteration) do not cudaMalloc/Free
    std::vector<std::pair<void *, size_t>> dr_cache;
    // kernel timing hook (iga_profile_*)
    struct ProfRec { const char *name; cudaEvent_t a, b; };
    bool prof_on = false;
    std::vector<ProfRec> prof_pending;
    std::vector<cudaEvent_t> prof_pool;
    std::vector<std::string> prof_names;
    std::vector<int> prof_count;
    std::vector<double> prof_ms;
};

namespace iga {
// bracket one kernel launch with events when profiling is on
struct ProfScope {
    iga_space_s *s;
    const char *name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(iga_space_s *s_, const char *n, cudaStream_t st_);
    ~ProfScope();
};
void set_error(const std::string &msg);
iga_status launch_form(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                       const double *Udot, double *csr_val, double *F, cudaStream_t st);
// launch_form over the element sub-box [lo, hi) of this rank's element box, outputs not zeroed
iga_status launch_form_box(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                           const double *Udot, double *csr_val, double *F, cudaStream_t st, const int lo[3],
                           const int hi[3]);
void k_zero_vec(double *p, long long n, cudaStream_t st, int nsm);
void k_zero_pair(double *p, long long n, double *q, long long m, cudaStream_t st, int nsm);   // p and/or q may be null
iga_status launch_fused2d(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                          const double *Ud, double *val, double *F, cudaStream_t st, int nsm);
iga_status launch_fused2dm(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                           const double *Ud, double *val, double *F, cudaStream_t st, int nsm);
iga_status launch_fused3d(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                          const double *Ud, double *val, double *F, cudaStream_t st, int nsm);
iga_status launch_pattern(iga_space_s *s, int64_t *row_ptr, int32_t *col_idx, cudaStream_t st);
iga_status launch_basis3(iga_space_s *s, int order, double *out, cudaStream_t st);   // basis3.cu
iga_status gmres_solve(iga_space_s *s, const int64_t *rp, const int32_t *ci, const double *a, const double *b, double *x,
                       const iga_krylov *opt, int *iters, double *relres, cudaStream_t st);        // solver.cu
iga_status alpha_step(iga_space_s *s, const iga_phys *phys, const iga_alpha *opt, const int64_t *rp, const int32_t *ci,
                      double *val, double *U, double *Udot, iga_step_stats *stats, cudaStream_t st);  // solver.cu
iga_status krylov_plan_host(const iga_space_desc *d, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                            int64_t ext_n[3], int64_t ghost[3], int max_msgs, iga_msg *send, int *nsend, iga_msg *recv,
                            int *nrecv);                                                               // solver.cu
iga_status alpha_step_group(int nr, iga_space_s *const *sp, const iga_phys *phys, const iga_alpha *opt,
                            const int64_t *const *rp, const int32_t *const *ci, double *const *val, double *const *U,
                            double *const *Udot, iga_step_stats *stats, cudaStream_t st);              // solver.cu
iga_status check_phys(iga_space_s *s, const iga_phys *phys);                                          // space.cu
iga_status form_one(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U, const double *Ud,
                    double *val, double *F, cudaStream_t st);                                         // space.cu
// dist.cu
iga_status dist_setup(iga_space_s *s, const iga_dist *dist);
iga_status dist_allreduce_sum(iga_space_s *s, double *buf, size_t n, cudaStream_t st);
iga_status dist_sendrecv(iga_space_s *s, int ns, const int *speer, const double *const *sbuf, const long long *scount,
                         int nr, const int *rpeer, double *const *rbuf, const long long *rcount, cudaStream_t st);
iga_status gmres_group(int nr, iga_space_s *const *sp, const int64_t *const *rp, const int32_t *const *ci,
                       const double *const *a, const double *const *b, double *const *x, const iga_krylov *opt,
                       int *iters, double *relres, cudaStream_t st);                              // solver.cu
void dist_destroy(iga_space_s *s);
iga_status dist_form(iga_space_s **sp, int n, const iga_phys *ph, double a, double b, const double *const *U,
                     const double *const *Ud, double *const *val, double *const *F, cudaStream_t st);
iga_status nccl_unique_id(unsigned char out[128]);
iga_status dist_plan_host(const iga_space_desc *d, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                          int64_t el_lo[3], int64_t el_hi[3], int64_t ext_n[3], int max_msgs, iga_msg *send,
                          int *nsend, iga_msg *recv, int *nrecv);
}  // namespace iga
