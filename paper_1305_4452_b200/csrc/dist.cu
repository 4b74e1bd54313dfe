// dist.cu -- multi-rank assembly: box decomposition of the element grid,
// ghost-U exchange before the kernels and the off-rank row exchange after them.
//
// The paper's PETSc design (P:552-559 ghost values, "off-process cache" + MatAssembly)
// becomes, per rank:
//   * a touched box = owned functions + `halo` functions above them on each partitioned axis
//     (A-9 ownership puts every touched-but-not-owned function on the upper side);
//   * U, Udot gathered into the touched box: owned part copied from the caller's vector, the
//     halo sub-boxes received from their owners (ghost exchange, one message per upper peer);
//   * the assembly kernels write owned rows straight into the caller's CSR and halo rows into a
//     library buffer laid out as 2^d - 1 sub-boxes, each a closed-form CSR of full rows
//     (iga_internal.cuh row_start) -- so each sub-box IS the message to its owner;
//   * the owner receives the sub-box and adds it row by row into its CSR (kernel K5, one warp per
//     row, contiguous coalesced adds) and the residual halo into its F.
// Transport: NCCL send/recv (dlopen'ed libnccl.so.2, the one torch already loaded) in one group
// per exchange on the caller's stream, or -- for spaces of several ranks living in one process
// (tests on one GPU) -- stream-ordered device copies between the ranks' buffers (iga_*_group).
#include <dlfcn.h>

#include <cstring>
#include <string>
#include <vector>

#include "iga_host.h"

namespace iga {

// ---- NCCL entry points (dlopen; ABI types of nccl.h) ----------------------------------------
struct NcclUid { char internal[128]; };
typedef void *ncclComm_t;
struct NcclApi {
    bool ok = false;
    int (*GetUniqueId)(NcclUid *) = nullptr;
    int (*CommInitRank)(ncclComm_t *, int, NcclUid, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
};
constexpr int NCCL_FLOAT64 = 8;

static NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.GetUniqueId = (int (*)(NcclUid *))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (int (*)(ncclComm_t *, int, NcclUid, int))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
    api.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
    api.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
    api.Send = (int (*)(const void *, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclSend");
    api.Recv = (int (*)(void *, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclRecv");
    api.GetErrorString = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
    api.AllReduce = (int (*)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
             api.Recv;
    return api;
}

// ---- exchange plan ------------------------------------------------------------------------
// One message per (peer, sub-box s), s != 0 with bit (2 - a) set <=> the halo layer on axis a.
//  up   message: this rank -> owner of its halo sub-box s (rank coordinate c + s); carries the
//                halo rows (matrix) and halo residual; the ghost U for that sub-box comes back
//                along it.  box = this rank's touched-box region of sub-box s.
//  down message: the mirror image, from the rank at c - s; box = the first h layers of this
//                rank's owned box on the s axes (h = the sender's halo count), full owned range
//                on the others.
struct Msg {
    int peer, sub;
    int lo[3], n[3];          // box in this rank's touched-box local indices
    long long Tb[3];          // box totals of the per-axis Alg. 3 widths
    long long rows_nodes;     // prod n
    long long nval;           // CSR values (full rows) = m^2 prod Tb
    long long val_off;        // offset in the halo buffer (up) or the receive buffer (down)
    long long vec_off;        // offset in nodes*m units in the vector message buffers
};

struct DistState {
    int transport = 0;
    ncclComm_t comm = nullptr;
    // element sub-boxes: blo[a] = first element of the rank's box touching a halo function along
    // axis a (= el_hi without a halo); the upper slabs are computed first, the interior overlaps
    // the halo-row exchange (which runs on `side`)
    int blo[3] = {0, 0, 0};
    cudaStream_t side = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_xchg = nullptr;
    std::vector<Msg> up, down;
    long long ext_nodes = 0, halo_vals = 0, recv_vals = 0, up_vec = 0, down_vec = 0;
    double *Uext = nullptr, *Udext = nullptr, *Fext = nullptr;
    double *halo = nullptr, *recv = nullptr;
    double *ghost_send = nullptr, *ghost_recv = nullptr;   // [U | Udot] boxes, down / up messages
    double *fh_send = nullptr, *fh_recv = nullptr;         // residual halo, up / down messages
    std::vector<void *> allocs;
};

int dist_transport(const DistState *D) { return D->transport; }

static int coord_rank(const int procs[3], const int c[3]) { return (c[0] * procs[1] + c[1]) * procs[2] + c[2]; }

// Build the message lists of rank `rank` from the per-axis partitions (host only; shared by
// iga_space_create and the GPU-free iga_dist_plan).
static void build_plan(const AxisHost part[3], int dim, int m, const int procs[3], const int rc[3],
                       std::vector<Msg> &up, std::vector<Msg> &down, long long hbase[8], long long &halo_vals,
                       long long &recv_vals, long long &up_vec, long long &down_vec) {
    up.clear();
    down.clear();
    halo_vals = recv_vals = up_vec = down_vec = 0;
    for (int s = 0; s < 8; s++) hbase[s] = 0;
    auto wsum = [&](int a, int g0, int cnt) {      // sum of Alg. 3 widths of functions g0 .. g0+cnt-1 (mod nu)
        long long t = 0;
        for (int k = 0; k < cnt; k++) t += part[a].rowW[(g0 + k) % part[a].nu];
        return t;
    };
    for (int s = 1; s < 8; s++) {
        int sb[3] = {(s >> 2) & 1, (s >> 1) & 1, s & 1};
        bool valid = true;
        for (int a = dim; a < 3; a++)
            if (sb[a]) valid = false;
        if (!valid) continue;
        // ---- up: my halo sub-box s -> its owner ----
        {
            Msg u{};
            u.sub = s;
            int pc[3];
            long long nval = (long long)m * m, nodes = 1;
            for (int a = 0; a < 3; a++) {
                const AxisHost &H = part[a];
                const int c = rc[a];
                if (a >= dim) { u.lo[a] = 0; u.n[a] = 1; u.Tb[a] = 1; pc[a] = 0; continue; }
                const int nown = H.own_hi[c] - H.own_lo[c];
                if (sb[a]) {
                    u.lo[a] = nown; u.n[a] = H.halo[c];
                    u.Tb[a] = wsum(a, H.own_hi[c] % H.nu, H.halo[c]);
                    pc[a] = (c + 1) % procs[a];
                } else {
                    u.lo[a] = 0; u.n[a] = nown;
                    u.Tb[a] = wsum(a, H.own_lo[c], nown);
                    pc[a] = c;
                }
                nval *= u.Tb[a];
                nodes *= u.n[a];
            }
            hbase[s] = halo_vals;
            if (nodes > 0) {
                u.peer = coord_rank(procs, pc);
                u.rows_nodes = nodes;
                u.nval = nval;
                u.val_off = halo_vals;
                u.vec_off = up_vec;
                halo_vals += nval;
                up_vec += nodes * m;
                up.push_back(u);
            }
        }
        // ---- down: the sub-box s of my lower neighbour -> me ----
        {
            Msg dn{};
            dn.sub = s;
            int pc[3];
            long long nval = (long long)m * m, nodes = 1;
            bool exists = true;
            for (int a = 0; a < 3; a++) {
                const AxisHost &H = part[a];
                const int c = rc[a];
                dn.lo[a] = 0;
                if (a >= dim) { dn.n[a] = 1; dn.Tb[a] = 1; pc[a] = 0; continue; }
                const int nown = H.own_hi[c] - H.own_lo[c];
                if (sb[a]) {
                    int cl = c - 1;
                    if (cl < 0) {
                        if (H.periodic) cl += procs[a];
                        else exists = false;
                    }
                    const int h = exists ? H.halo[cl] : 0;
                    dn.n[a] = h;
                    dn.Tb[a] = wsum(a, H.own_lo[c], h);
                    pc[a] = exists ? cl : 0;
                } else {
                    dn.n[a] = nown;
                    dn.Tb[a] = wsum(a, H.own_lo[c], nown);
                    pc[a] = c;
                }
                nval *= dn.Tb[a];
                nodes *= dn.n[a];
            }
            if (exists && nodes > 0) {
                dn.peer = coord_rank(procs, pc);
                dn.rows_nodes = nodes;
                dn.nval = nval;
                dn.val_off = recv_vals;
                dn.vec_off = down_vec;
                recv_vals += nval;
                down_vec += nodes * m;
                down.push_back(dn);
            }
        }
    }
}

// ---- kernels ----------------------------------------------------------------------------------
// box copy between an array laid out as [d0][d1][d2][m] (strided) and a contiguous box
// [n0][n1][n2][m]: mode 0 contig = strided, 1 strided = contig, 2 strided += contig
__global__ void k_box(double *__restrict__ strided, int d1, int d2, int lo0, int lo1, int lo2, int n0, int n1, int n2,
                      int m, double *__restrict__ contig, int mode) {
    const long long tot = (long long)n0 * n1 * n2 * m;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        long long r = t;
        const int i = (int)(r % m); r /= m;
        const int b2 = (int)(r % n2); r /= n2;
        const int b1 = (int)(r % n1);
        const int b0 = (int)(r / n1);
        const long long si = ((((long long)(lo0 + b0) * d1) + lo1 + b1) * d2 + lo2 + b2) * m + i;
        if (mode == 0) contig[t] = strided[si];
        else if (mode == 1) strided[si] = contig[t];
        else strided[si] += contig[t];
    }
}

struct K5Box {
    int n[3];
    long long Tb[3];
    long long off;
};

// K5: add a received sub-box of full CSR rows into the owner's rows, one warp per row.
// Both sides use the same closed form (row-major over the box, component innermost, entries in
// the row's Alg. 3 order), the destination with the owner's owned-box prefix sums.
__global__ void k_halo_add(SpaceDev s, int m, K5Box b, const double *__restrict__ recv, double *__restrict__ val) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nrows = (long long)b.n[0] * b.n[1] * b.n[2] * m;
    if (warp >= nrows) return;
    long long r = warp;
    const int i = (int)(r % m); r /= m;
    const int l2 = (int)(r % b.n[2]); r /= b.n[2];
    const int l1 = (int)(r % b.n[1]);
    const int l0 = (int)(r / b.n[1]);
    const int l[3] = {l0, l1, l2};
    long long S[3];
    int W[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const AxisDev &ax = s.ax[a];
        int g = ax.own_lo + l[a];
        if (g >= ax.nu) g -= ax.nu;
        S[a] = ax.lS[l[a]];
        W[a] = ax.rowW[g];
    }
    const long long Wn = (long long)W[0] * W[1] * W[2];
    const long long mm = (long long)m * m;
    const long long src = b.off + mm * (S[0] * b.Tb[1] * b.Tb[2] + W[0] * S[1] * b.Tb[2] + (long long)W[0] * W[1] * S[2])
                          + (long long)i * Wn * m;
    const long long dst = mm * (S[0] * s.ax[1].T * s.ax[2].T + W[0] * S[1] * s.ax[2].T + (long long)W[0] * W[1] * S[2])
                          + (long long)i * Wn * m;
    for (long long k = lane; k < Wn * m; k += 32) val[dst + k] += recv[src + k];
}

static void box_launch(double *strided, const int dims[3], const int lo[3], const int n[3], int m, double *contig,
                       int mode, cudaStream_t st) {
    const long long tot = (long long)n[0] * n[1] * n[2] * m;
    if (tot <= 0) return;
    const long long blocks = std::min<long long>((tot + 255) / 256, 148 * 8);
    k_box<<<(unsigned)blocks, 256, 0, st>>>(strided, dims[1], dims[2], lo[0], lo[1], lo[2], n[0], n[1], n[2], m, contig,
                                           mode);
}

// ---- setup / teardown ---------------------------------------------------------------------------
static iga_status dmalloc(DistState *D, double **p, long long n) {
    void *ptr = nullptr;
    if (cudaMalloc(&ptr, (size_t)std::max<long long>(n, 1) * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaMalloc (multi-rank buffers) failed");
        return IGA_ERR_NOMEM;
    }
    D->allocs.push_back(ptr);
    *p = (double *)ptr;
    return IGA_OK;
}

void dist_destroy(iga_space_s *s) {
    if (!s->dist) return;
    DistState *D = s->dist;
    if (D->comm && nccl().ok) nccl().CommDestroy(D->comm);
    if (D->ev_pack) cudaEventDestroy(D->ev_pack);
    if (D->ev_xchg) cudaEventDestroy(D->ev_xchg);
    if (D->side) cudaStreamDestroy(D->side);
    for (void *p : D->allocs) cudaFree(p);
    delete D;
    s->dist = nullptr;
}

iga_status dist_setup(iga_space_s *s, const iga_dist *dist) {
    DistState *D = new DistState();
    s->dist = D;
    D->transport = dist->transport;
    const int m = s->dof;
    build_plan(s->part, s->dim, m, s->procs, s->rcoord, D->up, D->down, s->dev.hbase, D->halo_vals, D->recv_vals,
               D->up_vec, D->down_vec);
    D->ext_nodes = 1;
    for (int a = 0; a < 3; a++) D->ext_nodes *= s->dev.ax[a].x_n;
    iga_status st;
    if ((st = dmalloc(D, &D->Uext, D->ext_nodes * m)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->Udext, D->ext_nodes * m)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->Fext, D->ext_nodes * m)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->halo, D->halo_vals)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->recv, D->recv_vals)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->ghost_send, 2 * D->down_vec)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->ghost_recv, 2 * D->up_vec)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->fh_send, D->up_vec)) != IGA_OK) return st;
    if ((st = dmalloc(D, &D->fh_recv, D->down_vec)) != IGA_OK) return st;
    s->dev.halo = D->halo;
    for (int a = 0; a < 3; a++) {
        const AxisHost &H = s->part[a];
        int b = s->el_hi[a];
        if (a < s->dim && s->halo[a] > 0) {
            const int n_own = s->own_hi[a] - s->own_lo[a];
            for (int e = s->el_hi[a] - 1; e >= s->el_lo[a]; e--) {
                bool touches = false;
                for (int al = 0; al <= H.p; al++) {
                    int l = (H.first[e] + al) % H.nu - s->own_lo[a];
                    if (l < 0) l += H.nu;
                    if (l >= n_own) touches = true;
                }
                if (!touches) break;
                b = e;
            }
        }
        D->blo[a] = b;
    }
    if (cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D->ev_xchg, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        set_error("multi-rank stream / event creation failed");
        return IGA_ERR_CUDA;
    }
    if (D->transport == IGA_XPORT_NCCL) {
        NcclApi &api = nccl();
        if (!api.ok) { set_error("libnccl.so.2 not loadable (multi-rank needs NCCL)"); return IGA_ERR_COMM; }
        NcclUid uid;
        std::memcpy(uid.internal, dist->nccl_id, 128);
        const int r = api.CommInitRank(&D->comm, s->nranks, uid, s->rank);
        if (r != 0) {
            D->comm = nullptr;
            set_error(std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "error"));
            return IGA_ERR_COMM;
        }
    }
    return IGA_OK;
}

// ---- phases ---------------------------------------------------------------------------------------
static void ext_dims(const iga_space_s *s, int d[3]) {
    for (int a = 0; a < 3; a++) d[a] = s->dev.ax[a].x_n;
}
static void own_dims(const iga_space_s *s, int d[3]) {
    for (int a = 0; a < 3; a++) d[a] = s->dev.ax[a].n_own;
}

// owned U -> touched box; pack the ghost boxes my lower neighbours need
static void phase_ghost_pack(iga_space_s *s, const double *U, const double *Ud, cudaStream_t st) {
    DistState *D = s->dist;
    const int m = s->dof;
    int ed[3], od[3], z[3] = {0, 0, 0};
    ext_dims(s, ed);
    own_dims(s, od);
    ProfScope ps(s, "k_box", st);
    box_launch(D->Uext, ed, z, od, m, const_cast<double *>(U), 1, st);
    if (Ud) box_launch(D->Udext, ed, z, od, m, const_cast<double *>(Ud), 1, st);
    for (const Msg &g : D->down) {
        const long long c = g.rows_nodes * m;
        box_launch(const_cast<double *>(U), od, g.lo, g.n, m, D->ghost_send + 2 * g.vec_off, 0, st);
        if (Ud) box_launch(const_cast<double *>(Ud), od, g.lo, g.n, m, D->ghost_send + 2 * g.vec_off + c, 0, st);
    }
}

static void phase_ghost_unpack(iga_space_s *s, bool has_ud, cudaStream_t st) {
    DistState *D = s->dist;
    const int m = s->dof;
    int ed[3];
    ext_dims(s, ed);
    ProfScope ps(s, "k_box", st);
    for (const Msg &u : D->up) {
        const long long c = u.rows_nodes * m;
        box_launch(D->Uext, ed, u.lo, u.n, m, D->ghost_recv + 2 * u.vec_off, 1, st);
        if (has_ud) box_launch(D->Udext, ed, u.lo, u.n, m, D->ghost_recv + 2 * u.vec_off + c, 1, st);
    }
}

static void phase_halo_pack(iga_space_s *s, bool has_F, cudaStream_t st) {
    DistState *D = s->dist;
    if (!has_F) return;
    const int m = s->dof;
    int ed[3];
    ext_dims(s, ed);
    ProfScope ps(s, "k_box", st);
    for (const Msg &u : D->up) box_launch(D->Fext, ed, u.lo, u.n, m, D->fh_send + u.vec_off, 0, st);
}

static void phase_halo_add(iga_space_s *s, double *val, double *F, cudaStream_t st) {
    DistState *D = s->dist;
    const int m = s->dof;
    int ed[3], od[3], z[3] = {0, 0, 0};
    ext_dims(s, ed);
    own_dims(s, od);
    if (F) {
        ProfScope ps(s, "k_box", st);
        box_launch(D->Fext, ed, z, od, m, F, 0, st);          // owned part of the touched-box residual
        for (const Msg &g : D->down) box_launch(F, od, g.lo, g.n, m, D->fh_recv + g.vec_off, 2, st);
    }
    if (val) {
        ProfScope ps(s, "k_halo_add", st);
        for (const Msg &g : D->down) {
            K5Box b;
            for (int a = 0; a < 3; a++) { b.n[a] = g.n[a]; b.Tb[a] = g.Tb[a]; }
            b.off = g.val_off;
            const long long rows = g.rows_nodes * m;
            k_halo_add<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(s->dev, m, b, D->recv, val);
        }
    }
}

// ---- transport ----------------------------------------------------------------------------------
enum { XCHG_GHOST = 0, XCHG_HALO = 1 };

static const Msg *find_msg(const std::vector<Msg> &v, int peer, int sub) {
    for (const Msg &x : v)
        if (x.peer == peer && x.sub == sub) return &x;
    return nullptr;
}

static iga_status exchange(iga_space_s **sp, int n, int which, bool has_ud, bool has_val, bool has_F, cudaStream_t st) {
    const int m = sp[0]->dof;
    if (sp[0]->dist->transport == IGA_XPORT_NCCL) {
        iga_space_s *s = sp[0];
        DistState *D = s->dist;
        NcclApi &api = nccl();
        int r = api.GroupStart();
        if (which == XCHG_GHOST) {
            for (const Msg &g : D->down) {
                const long long c = g.rows_nodes * m * (has_ud ? 2 : 1);
                if (!r) r = api.Send(D->ghost_send + 2 * g.vec_off, (size_t)c, NCCL_FLOAT64, g.peer, D->comm, st);
            }
            for (const Msg &u : D->up) {
                const long long c = u.rows_nodes * m * (has_ud ? 2 : 1);
                if (!r) r = api.Recv(D->ghost_recv + 2 * u.vec_off, (size_t)c, NCCL_FLOAT64, u.peer, D->comm, st);
            }
        } else {
            for (const Msg &u : D->up) {
                if (has_val && !r) r = api.Send(D->halo + u.val_off, (size_t)u.nval, NCCL_FLOAT64, u.peer, D->comm, st);
                if (has_F && !r) r = api.Send(D->fh_send + u.vec_off, (size_t)(u.rows_nodes * m), NCCL_FLOAT64, u.peer, D->comm, st);
            }
            for (const Msg &g : D->down) {
                if (has_val && !r) r = api.Recv(D->recv + g.val_off, (size_t)g.nval, NCCL_FLOAT64, g.peer, D->comm, st);
                if (has_F && !r) r = api.Recv(D->fh_recv + g.vec_off, (size_t)(g.rows_nodes * m), NCCL_FLOAT64, g.peer, D->comm, st);
            }
        }
        const int r2 = api.GroupEnd();
        if (r || r2) {
            set_error(std::string("NCCL exchange: ") + (api.GetErrorString ? api.GetErrorString(r ? r : r2) : "error"));
            return IGA_ERR_COMM;
        }
        s->last_launches += 1;
        return IGA_OK;
    }
    // in-process transport: every rank's space is in sp[0..n) (indexed by rank)
    for (int k = 0; k < n; k++) {
        iga_space_s *s = sp[k];
        DistState *D = s->dist;
        if (which == XCHG_GHOST) {
            for (const Msg &u : D->up) {
                const Msg *g = find_msg(sp[u.peer]->dist->down, s->rank, u.sub);
                if (!g || g->rows_nodes != u.rows_nodes) { set_error("ghost plan mismatch"); return IGA_ERR_STATE; }
                const long long c = u.rows_nodes * m * (has_ud ? 2 : 1);
                cudaMemcpyAsync(D->ghost_recv + 2 * u.vec_off, sp[u.peer]->dist->ghost_send + 2 * g->vec_off,
                                c * sizeof(double), cudaMemcpyDeviceToDevice, st);
            }
        } else {
            for (const Msg &g : D->down) {
                const Msg *u = find_msg(sp[g.peer]->dist->up, s->rank, g.sub);
                if (!u || u->nval != g.nval || u->rows_nodes != g.rows_nodes) { set_error("halo plan mismatch"); return IGA_ERR_STATE; }
                if (has_val)
                    cudaMemcpyAsync(D->recv + g.val_off, sp[g.peer]->dist->halo + u->val_off, g.nval * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st);
                if (has_F)
                    cudaMemcpyAsync(D->fh_recv + g.vec_off, sp[g.peer]->dist->fh_send + u->vec_off,
                                    g.rows_nodes * m * sizeof(double), cudaMemcpyDeviceToDevice, st);
            }
        }
    }
    return IGA_OK;
}

// ---- the multi-rank form call ---------------------------------------------------------------------
// Schedule per rank (caller's stream st; NCCL halo exchange on the rank's side stream):
//   zero outputs | pack ghost U -> ghost exchange -> unpack | upper slabs (elements touching halo
//   rows) -> pack halo residual -> [halo-row exchange on `side` || interior elements on st] ->
//   K5 adds.  The interior never touches halo rows or ghost functions, so the largest message
//   (full halo rows) travels while most of the elements are integrated.
// sp[k], U[k], ... for the n ranks this call drives: n = 1 with NCCL (one process per GPU), or all
// ranks of an in-process group (exchanges = device copies, everything on st).  val[k] == nullptr
// => residual only.
static void sub_boxes(const iga_space_s *s, int lo[4][3], int hi[4][3]) {
    const int *L = s->el_lo, *H = s->el_hi, *B = s->dist->blo;
    // 0..2: upper slabs along axes 0, 1, 2 (disjoint); 3: interior
    for (int k = 0; k < 4; k++)
        for (int d = 0; d < 3; d++) { lo[k][d] = L[d]; hi[k][d] = H[d]; }
    lo[0][0] = B[0];
    hi[1][0] = B[0]; lo[1][1] = B[1];
    hi[2][0] = B[0]; hi[2][1] = B[1]; lo[2][2] = B[2];
    hi[3][0] = B[0]; hi[3][1] = B[1]; hi[3][2] = B[2];
}

iga_status dist_form(iga_space_s **sp, int n, const iga_phys *ph, double a, double b, const double *const *U,
                     const double *const *Ud, double *const *val, double *const *F, cudaStream_t st) {
    const bool has_ud = Ud[0] != nullptr, has_val = val[0] != nullptr, has_F = F[0] != nullptr;
    const bool nccl_x = sp[0]->dist->transport == IGA_XPORT_NCCL;
    int launches[64] = {0};
    for (int k = 0; k < n; k++) {
        iga_space_s *s = sp[k];
        DistState *D = s->dist;
        {
            ProfScope ps(s, "k_zero", st);
            k_zero_pair(has_val ? val[k] : nullptr, has_val ? s->nnz_owned : 0, has_F ? D->Fext : nullptr,
                        has_F ? D->ext_nodes * s->dof : 0, st, 148);
            if (has_val && D->halo_vals) k_zero_vec(D->halo, D->halo_vals, st, 148);
        }
        phase_ghost_pack(s, U[k], Ud[k], st);
    }
    iga_status r = exchange(sp, n, XCHG_GHOST, has_ud, has_val, has_F, st);
    if (r != IGA_OK) return r;
    int lo[64][4][3], hi[64][4][3];
    for (int k = 0; k < n; k++) {
        iga_space_s *s = sp[k];
        DistState *D = s->dist;
        phase_ghost_unpack(s, has_ud, st);
        sub_boxes(s, lo[k % 64], hi[k % 64]);
        for (int j = 0; j < 3; j++) {
            r = launch_form_box(s, ph, a, b, D->Uext, has_ud ? D->Udext : nullptr, val[k], has_F ? D->Fext : nullptr, st,
                                lo[k % 64][j], hi[k % 64][j]);
            if (r != IGA_OK) return r;
            launches[k % 64] += s->last_launches;
        }
        phase_halo_pack(s, has_F, st);
    }
    if (nccl_x) {
        // halo rows leave on the side stream while the interior is integrated on st
        DistState *D = sp[0]->dist;
        cudaEventRecord(D->ev_pack, st);
        cudaStreamWaitEvent(D->side, D->ev_pack, 0);
        r = exchange(sp, n, XCHG_HALO, has_ud, has_val, has_F, D->side);
        if (r != IGA_OK) return r;
        cudaEventRecord(D->ev_xchg, D->side);
    } else {
        r = exchange(sp, n, XCHG_HALO, has_ud, has_val, has_F, st);
        if (r != IGA_OK) return r;
    }
    for (int k = 0; k < n; k++) {
        iga_space_s *s = sp[k];
        DistState *D = s->dist;
        r = launch_form_box(s, ph, a, b, D->Uext, has_ud ? D->Udext : nullptr, val[k], has_F ? D->Fext : nullptr, st,
                            lo[k % 64][3], hi[k % 64][3]);
        if (r != IGA_OK) return r;
        launches[k % 64] += s->last_launches;
    }
    if (nccl_x) cudaStreamWaitEvent(st, sp[0]->dist->ev_xchg, 0);
    for (int k = 0; k < n; k++) {
        phase_halo_add(sp[k], val[k], F[k], st);
        sp[k]->last_launches = launches[k % 64];
    }
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("multi-rank form: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

iga_status nccl_unique_id(unsigned char out[128]) {
    NcclApi &api = nccl();
    if (!api.ok) { set_error("libnccl.so.2 not loadable"); return IGA_ERR_COMM; }
    NcclUid uid;
    const int r = api.GetUniqueId(&uid);
    if (r != 0) { set_error("ncclGetUniqueId failed"); return IGA_ERR_COMM; }
    std::memcpy(out, uid.internal, 128);
    return IGA_OK;
}

// host-only plan (iga_dist_plan)
iga_status dist_plan_host(const iga_space_desc *d, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                          int64_t el_lo[3], int64_t el_hi[3], int64_t ext_n[3], int max_msgs, iga_msg *send,
                          int *nsend, iga_msg *recv, int *nrecv) {
    if (!d || !dist) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (d->dim < 2 || d->dim > 3 || d->dof < 1 || d->dof > 4) { set_error("dim 2..3, dof 1..4"); return IGA_ERR_PARAM; }
    int procs[3] = {1, 1, 1}, rc[3] = {0, 0, 0}, prod = 1;
    for (int a = 0; a < 3; a++) {
        procs[a] = a < d->dim ? std::max(1, dist->procs[a]) : 1;
        prod *= procs[a];
    }
    if (prod != dist->nranks || dist->rank < 0 || dist->rank >= dist->nranks) {
        set_error("iga_dist: procs product must equal nranks and 0 <= rank < nranks");
        return IGA_ERR_PARAM;
    }
    int r = dist->rank;
    rc[2] = r % procs[2]; r /= procs[2];
    rc[1] = r % procs[1]; r /= procs[1];
    rc[0] = r;
    AxisHost part[3];
    for (int a = 0; a < 3; a++) {
        if (a >= d->dim) {
            AxisHost &H = part[a];
            H.p = 0; H.nel = 1; H.nu = 1; H.nfun = 1; H.nq = 1;
            H.rowW = {1};
            H.el_lo = {0}; H.el_hi = {1}; H.own_lo = {0}; H.own_hi = {1}; H.halo = {0};
            continue;
        }
        iga_status st = axis_host(d, a, procs[a], part[a]);
        if (st != IGA_OK) return st;
    }
    std::vector<Msg> up, down;
    long long hb[8], hv, rv, uv, dv;
    build_plan(part, d->dim, d->dof, procs, rc, up, down, hb, hv, rv, uv, dv);
    for (int a = 0; a < 3; a++) {
        const AxisHost &H = part[a];
        const int c = rc[a];
        if (own_lo) own_lo[a] = H.own_lo[c];
        if (own_hi) own_hi[a] = H.own_hi[c];
        if (el_lo) el_lo[a] = H.el_lo[c];
        if (el_hi) el_hi[a] = H.el_hi[c];
        if (ext_n) ext_n[a] = H.own_hi[c] - H.own_lo[c] + H.halo[c];
    }
    auto put = [&](const std::vector<Msg> &v, iga_msg *out, int *cnt) {
        if (cnt) *cnt = (int)v.size();
        for (int k = 0; k < (int)v.size() && k < max_msgs && out; k++) {
            out[k].peer = v[k].peer;
            out[k].subbox = v[k].sub;
            out[k].rows = v[k].rows_nodes * d->dof;
            out[k].values = v[k].nval;
            for (int a = 0; a < 3; a++) {
                out[k].box_lo[a] = v[k].lo[a];
                out[k].box_n[a] = v[k].n[a];
            }
        }
    };
    put(up, send, nsend);
    put(down, recv, nrecv);
    return IGA_OK;
}

// ---- collectives for the distributed Krylov solve (solver.cu) ---------------------------------
// sum-all-reduce of n doubles in place on `st` (NCCL transport)
iga_status dist_allreduce_sum(iga_space_s *s, double *buf, size_t n, cudaStream_t st) {
    NcclApi &api = nccl();
    if (!s->dist || !s->dist->comm || !api.ok || !api.AllReduce) { set_error("allreduce: no NCCL communicator"); return IGA_ERR_COMM; }
    const int r = api.AllReduce(buf, buf, n, NCCL_FLOAT64, 0 /* ncclSum */, s->dist->comm, st);
    if (r) { set_error("ncclAllReduce failed"); return IGA_ERR_COMM; }
    return IGA_OK;
}

// grouped point-to-point exchange: sends in the given order, receives in the given order
iga_status dist_sendrecv(iga_space_s *s, int ns, const int *speer, const double *const *sbuf, const long long *scount,
                         int nr, const int *rpeer, double *const *rbuf, const long long *rcount, cudaStream_t st) {
    NcclApi &api = nccl();
    if (!s->dist || !s->dist->comm || !api.ok) { set_error("sendrecv: no NCCL communicator"); return IGA_ERR_COMM; }
    int r = api.GroupStart();
    for (int k = 0; k < ns && !r; k++) r = api.Send(sbuf[k], (size_t)scount[k], NCCL_FLOAT64, speer[k], s->dist->comm, st);
    for (int k = 0; k < nr && !r; k++) r = api.Recv(rbuf[k], (size_t)rcount[k], NCCL_FLOAT64, rpeer[k], s->dist->comm, st);
    const int r2 = api.GroupEnd();
    if (r || r2) { set_error("NCCL send/recv failed"); return IGA_ERR_COMM; }
    return IGA_OK;
}

}  // namespace iga
