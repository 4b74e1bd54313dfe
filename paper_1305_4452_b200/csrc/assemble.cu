// assemble.cu -- residual / Jacobian assembly kernels (Alg. 4) for sm_100a, fp64.
//
// Two kernels per batch of elements:
//   K3a  k_point     one thread per (element, quadrature point): 1D tables -> tensor-product
//                    kinds -> rational basis and isoparametric push-forward
//                    (folded into the map T) -> fields U_e -> physics -> the compact
//                    coefficient lists r~ and D~ written to the HBM workspace (SoA, coalesced).
//   K3b  k_contract  one CTA per element: stages the element's 1D tables and coefficients in
//                    shared memory, contracts  K_e = w_A w_B sum_q P(A,q)^T D~(q) P(B,q)
//                    (rank form, compile-time sparse), F_e likewise, and scatter-adds the
//                    dense element blocks into the CSR values / F at positions computed in
//                    closed form from the per-axis Alg. 3 stencils (no search).
// DESIGN.md documents the data layout and the roofline of each kernel.
#include <cstdio>
#include <type_traits>

#include "iga_host.h"
#include "kinds.cuh"
#include "physics.cuh"
#include "pointwise.cuh"

namespace iga {


__device__ __forceinline__ void elem_coords(const SpaceDev &s, long long el, int e[3]) {
    const int n1 = s.ax[1].el_hi - s.ax[1].el_lo, n2 = s.ax[2].el_hi - s.ax[2].el_lo;
    e[2] = s.ax[2].el_lo + (int)(el % n2);
    el /= n2;
    e[1] = s.ax[1].el_lo + (int)(el % n1);
    el /= n1;
    e[0] = s.ax[0].el_lo + (int)el;
}

// ============================================================================================
// K3a: pointwise kernel
// ============================================================================================
struct GlobalNodes {
    static constexpr bool PREMUL = false;
    const SpaceDev *s;
    const double *U, *Ud;
    long long node[64];      // global node (geometry: control points, weights)
    long long lnode[64];     // touched-box node (fields U, Udot)
    int M;
    __device__ double u(int A, int m) const { return __ldg(U + lnode[A] * M + m); }
    __device__ double ud(int A, int m) const { return __ldg(Ud + lnode[A] * M + m); }
    __device__ bool has_ud() const { return Ud != nullptr; }
    __device__ double w(int A) const { return s->wts ? __ldg(s->wts + node[A]) : 1.0; }
    __device__ double x(int A, int i) const { return __ldg(s->ctrl + node[A] * s->dim + i); }
};

template <int DIM, int P, class PH, int MODE, bool JAC>
__global__ void __launch_bounds__(128)
k_point(SpaceDev s, Prm prm, double a, double b, const double *__restrict__ U, const double *__restrict__ Ud,
        double *__restrict__ Dt, double *__restrict__ Rt, long long e0, int nb, long long ldq) {
    constexpr int NQ1 = P + 1, NP1 = P + 1;
    constexpr int NQ = ipow(NQ1, DIM), NEN = ipow(NP1, DIM);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nb * NQ) return;
    const int q = (int)(t % NQ);
    int e[3];
    elem_coords(s, e0 + t / NQ, e);
    int qd[3] = {0, 0, 0};
    {
        int r = q;
#pragma unroll
        for (int d = DIM - 1; d >= 0; d--) { qd[d] = r % NQ1; r /= NQ1; }
    }
    double v[DIM][3][NP1];
    double wq = 1.0, xq[DIM], hp[DIM];
    int first[DIM];
#pragma unroll
    for (int d = 0; d < DIM; d++) {
        const double *tp = s.ax[d].tab + (size_t)(e[d] * NQ1 + qd[d]) * 3 * NP1;
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int aa = 0; aa < NP1; aa++) v[d][k][aa] = __ldg(tp + k * NP1 + aa);
        wq *= __ldg(s.ax[d].qw + e[d] * NQ1 + qd[d]);
        xq[d] = __ldg(s.ax[d].qx + e[d] * NQ1 + qd[d]);
        hp[d] = __ldg(s.ax[d].hpar + e[d]);
        first[d] = __ldg(s.ax[d].first + e[d]);
    }
    GlobalNodes nodes;
    nodes.s = &s;
    nodes.U = U;
    nodes.Ud = Ud;
    nodes.M = PH::M;
    for (int A = 0; A < NEN; A++) {
        int g[3] = {0, 0, 0};
        int r = A;
        for (int d = DIM - 1; d >= 0; d--) {
            g[d] = first[d] + r % NP1;
            r /= NP1;
            if (g[d] >= s.ax[d].nu) g[d] -= s.ax[d].nu;
        }
        nodes.node[A] = node_index(s, g[0], g[1], g[2]);
        nodes.lnode[A] = local_node(s, g[0], g[1], g[2]);
    }
    const int bad = pointwise_qp<DIM, P, PH, MODE, JAC>(s, prm, a, b, v, wq, xq, hp, nodes, Dt + t, ldq,
                                                        Rt ? Rt + t : nullptr, ldq);
    if (bad) atomicOr(s.errflag, bad);
}

// ============================================================================================
// K3b: contraction + scatter kernel (one CTA per element)
// ============================================================================================
template <int DIM, int P, class PH, int MODE, bool JAC>
__global__ void __launch_bounds__(256)
k_contract(SpaceDev s, const double *__restrict__ Dt, const double *__restrict__ Rt, long long e0, long long ldq,
           double *__restrict__ val, double *__restrict__ Fout) {
    using L = Lists<PH, DIM, MODE>;
    using KS = typename L::KS;
    constexpr int M = PH::M, NQ1 = P + 1, NP1 = P + 1;
    constexpr int NQ = ipow(NQ1, DIM), NEN = ipow(NP1, DIM);
    constexpr int NC = KS::NC;
    __shared__ double tabs[DIM][NQ1][3][NP1];
    __shared__ double *rowP[NEN];               // CSR row of (A, i = 0): owned -> val, halo -> halo buffer
    __shared__ long long rowL[NEN];             // touched-box node of A (F layout)
    __shared__ double sA[NEN];
    __shared__ int Wn[NEN], W1n[NEN], W2n[NEN];
    __shared__ int posT[DIM][NP1][NP1];
    extern __shared__ double dyn[];
    double *Ds = dyn;                                   // [NE][NQ]
    double *Rs = dyn + (JAC ? L::NE * NQ : 0);          // [NR][NQ]

    int e[3];
    elem_coords(s, e0 + blockIdx.x, e);
    const long long qbase = (long long)blockIdx.x * NQ;
    const int tid = threadIdx.x;
    for (int idx = tid; idx < DIM * NQ1 * 3 * NP1; idx += blockDim.x) {
        const int d = idx / (NQ1 * 3 * NP1), rest = idx % (NQ1 * 3 * NP1);
        (&tabs[0][0][0][0])[idx] = s.ax[d].tab[(size_t)e[d] * NQ1 * 3 * NP1 + rest];
    }
    for (int idx = tid; idx < DIM * NP1 * NP1; idx += blockDim.x) {
        const int d = idx / (NP1 * NP1), rest = idx % (NP1 * NP1);
        (&posT[0][0][0])[idx] = s.ax[d].pos[(size_t)e[d] * NP1 * NP1 + rest];
    }
    if (JAC)
        for (int idx = tid; idx < L::NE * NQ; idx += blockDim.x)
            Ds[idx] = Dt[(idx / NQ) * ldq + qbase + idx % NQ];
    if (Fout)
        for (int idx = tid; idx < L::NR * NQ; idx += blockDim.x)
            Rs[idx] = Rt[(idx / NQ) * ldq + qbase + idx % NQ];
    for (int A = tid; A < NEN; A += blockDim.x) {
        int aa[3] = {0, 0, 0};
        int r = A;
        for (int d = DIM - 1; d >= 0; d--) { aa[d] = r % NP1; r /= NP1; }
        int g[3] = {0, 0, 0}, Wd[3] = {1, 1, 1};
        for (int d = 0; d < DIM; d++) {
            g[d] = s.ax[d].first[e[d]] + aa[d];
            if (g[d] >= s.ax[d].nu) g[d] -= s.ax[d].nu;
            Wd[d] = s.ax[d].rowW[g[d]];
        }
        int Wtot = 1;
        rowP[A] = val ? row_start(s, val, g[0], g[1], g[2], 0, M, &Wtot) : nullptr;
        Wn[A] = Wd[0] * Wd[1] * Wd[2];
        W1n[A] = Wd[1];
        W2n[A] = Wd[2];
        rowL[A] = local_node(s, g[0], g[1], g[2]) * M;
        sA[A] = (MODE == MODE_NURBS && s.wts) ? s.wts[node_index(s, g[0], g[1], g[2])] : 1.0;
    }
    __syncthreads();

    // ---- residual: thread per test function A --------------------------------------------
    if (Fout) {
        for (int A = tid; A < NEN; A += blockDim.x) {
            int aa[3] = {0, 0, 0};
            int r = A;
#pragma unroll
            for (int d = DIM - 1; d >= 0; d--) { aa[d] = r % NP1; r /= NP1; }
            double acc[M];
#pragma unroll
            for (int i = 0; i < M; i++) acc[i] = 0.0;
#pragma unroll 1
            for (int q = 0; q < NQ; q++) {
                int qd[3] = {0, 0, 0};
                int rq = q;
#pragma unroll
                for (int d = DIM - 1; d >= 0; d--) { qd[d] = rq % NQ1; rq /= NQ1; }
                double v[DIM][3][NP1];
#pragma unroll
                for (int d = 0; d < DIM; d++)
#pragma unroll
                    for (int k = 0; k < 3; k++)
#pragma unroll
                        for (int x = 0; x < NP1; x++) v[d][k][x] = tabs[d][qd[d]][k][x];
                static_for<L::NR>([&](auto RR) {
                    constexpr int rr = decltype(RR)::value;
                    constexpr int c = L::R.c[rr], i = L::R.i[rr];
                    acc[i] += kind_value<KS, DIM, c, NP1>(v, aa) * Rs[rr * NQ + q];
                });
            }
#pragma unroll
            for (int i = 0; i < M; i++) atomicAdd(Fout + rowL[A] + i, sA[A] * acc[i]);
        }
    }

    // ---- Jacobian: thread per (A, B) pair ---------------------------------------------------
    if constexpr (JAC) {
        for (int idx = tid; idx < NEN * NEN; idx += blockDim.x) {
            const int A = idx / NEN, B = idx % NEN;
            int aa[3] = {0, 0, 0}, bb[3] = {0, 0, 0};
            {
                int r = A, r2 = B;
#pragma unroll
                for (int d = DIM - 1; d >= 0; d--) { aa[d] = r % NP1; r /= NP1; bb[d] = r2 % NP1; r2 /= NP1; }
            }
            double K[M][M];
#pragma unroll
            for (int i = 0; i < M; i++)
#pragma unroll
                for (int j = 0; j < M; j++) K[i][j] = 0.0;
#pragma unroll 1
            for (int q = 0; q < NQ; q++) {
                int qd[3] = {0, 0, 0};
                int rq = q;
#pragma unroll
                for (int d = DIM - 1; d >= 0; d--) { qd[d] = rq % NQ1; rq /= NQ1; }
                double va[DIM][3][NP1];
#pragma unroll
                for (int d = 0; d < DIM; d++)
#pragma unroll
                    for (int k = 0; k < 3; k++)
#pragma unroll
                        for (int x = 0; x < NP1; x++) va[d][k][x] = tabs[d][qd[d]][k][x];
                double PA[NC], PB[NC];
                static_for<NC>([&](auto C) {
                    constexpr int c = decltype(C)::value;
                    if constexpr (L::test_used(c)) PA[c] = kind_value<KS, DIM, c, NP1>(va, aa);
                    else PA[c] = 0.0;
                    if constexpr (L::trial_used(c)) PB[c] = kind_value<KS, DIM, c, NP1>(va, bb);
                    else PB[c] = 0.0;
                });
                static_for<L::NE>([&](auto E) {
                    constexpr int ee = decltype(E)::value;
                    constexpr int i = L::E.i[ee], j = L::E.j[ee], c = L::E.c[ee], c2 = L::E.c2[ee];
                    K[i][j] += PA[c] * Ds[ee * NQ + q] * PB[c2];
                });
            }
            int pos[3] = {0, 0, 0};
#pragma unroll
            for (int d = 0; d < DIM; d++) pos[d] = posT[d][aa[d]][bb[d]];
            const long long off = ((long long)(pos[0] * W1n[A] + pos[1]) * W2n[A] + pos[2]) * M;
            const double sc = sA[A] * sA[B];
#pragma unroll
            for (int i = 0; i < M; i++) {
                double *dst = rowP[A] + (long long)i * Wn[A] * M + off;
#pragma unroll
                for (int j = 0; j < M; j++) atomicAdd(dst + j, sc * K[i][j]);
            }
        }
    }
}

__global__ void k_zero(double *__restrict__ p, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) p[k] = 0.0;
}

// two arrays in one launch (CSR values + residual): 16-byte stores where aligned
__global__ void k_zero2(double *__restrict__ p, long long n, double *__restrict__ q, long long m) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n2 = ((reinterpret_cast<uintptr_t>(p) & 15) == 0) ? n / 2 : 0;
    for (long long k = t0; k < n2; k += stride) reinterpret_cast<double2 *>(p)[k] = make_double2(0.0, 0.0);
    for (long long k = 2 * n2 + t0; k < n; k += stride) p[k] = 0.0;
    for (long long k = t0; k < m; k += stride) q[k] = 0.0;
}

void k_zero_pair(double *p, long long n, double *q, long long m, cudaStream_t st, int nsm) {
    if (!p) { p = q; n = m; q = nullptr; m = 0; }
    if (!q) m = 0;
    if (n <= 0 && m <= 0) return;
    long long blocks = (std::max(n / 2, m) + 255) / 256;
    const long long cap = (long long)nsm * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_zero2<<<(unsigned)blocks, 256, 0, st>>>(p, n, q, m);
}

void k_zero_vec(double *p, long long n, cudaStream_t st, int nsm) {
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    const long long cap = (long long)nsm * 16;
    if (blocks > cap) blocks = cap;
    k_zero<<<(unsigned)blocks, 256, 0, st>>>(p, n);
}

static int zero_launch(iga_space_s *s, double *p, long long n, cudaStream_t st, int nsm) {
    if (n <= 0) return 0;
    ProfScope ps(s, "k_zero", st);
    k_zero_vec(p, n, st, nsm);
    return 1;
}

// ============================================================================================
// host launcher
// ============================================================================================
template <int DIM, int P, class PH, int MODE>
static iga_status run_form(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                           const double *Ud, double *val, double *F, cudaStream_t st) {
    using L = Lists<PH, DIM, MODE>;
    constexpr int NQ = ipow(P + 1, DIM);
    const bool jac = val != nullptr;
    Prm prm;
    for (int i = 0; i < 8; i++) prm.p[i] = phys->p[i];
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    int launches = 0;
    if (jac && !s->skip_zero) launches += zero_launch(s, val, s->nnz_owned, st, nsm);
    if (F && !s->skip_zero) launches += zero_launch(s, F, s->nrows_owned, st, nsm);
    const size_t per_el = (size_t)NQ * ((jac ? L::NE : 0) + (F ? L::NR : 0)) * sizeof(double);
    long long nb_max = per_el ? (long long)(s->work_bytes / per_el) : s->nel_local;
    if (nb_max < 1) { set_error("workspace too small"); return IGA_ERR_NOMEM; }
    if (nb_max > s->nel_local) nb_max = s->nel_local;
    nb_max = std::min<long long>(nb_max, (1LL << 31) / NQ - 1);
    const size_t dsm = (size_t)NQ * ((jac ? L::NE : 0) + L::NR) * sizeof(double);
    {   // per-device attribute: set on the current device before every launch
        cudaError_t ce;
        if (jac) ce = cudaFuncSetAttribute(k_contract<DIM, P, PH, MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        else ce = cudaFuncSetAttribute(k_contract<DIM, P, PH, MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (ce != cudaSuccess) { set_error(cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    }
    double *Dt = s->work;
    for (long long e0 = 0; e0 < s->nel_local; e0 += nb_max) {
        const int nb = (int)std::min<long long>(nb_max, s->nel_local - e0);
        const long long ldq = (long long)nb * NQ;
        double *Rt = F ? Dt + (jac ? (size_t)L::NE * ldq : 0) : nullptr;
        const long long nthr = (long long)nb * NQ;
        const unsigned gA = (unsigned)((nthr + 127) / 128);
        if (jac) {
            { ProfScope ps(s, "k_point", st);
              k_point<DIM, P, PH, MODE, true><<<gA, 128, 0, st>>>(s->dev, prm, a, b, U, Ud, Dt, Rt, e0, nb, ldq); }
            { ProfScope ps(s, "k_contract", st);
              k_contract<DIM, P, PH, MODE, true><<<nb, 256, dsm, st>>>(s->dev, Dt, Rt, e0, ldq, val, F); }
        } else {
            { ProfScope ps(s, "k_point", st);
              k_point<DIM, P, PH, MODE, false><<<gA, 128, 0, st>>>(s->dev, prm, a, b, U, Ud, Dt, Rt, e0, nb, ldq); }
            { ProfScope ps(s, "k_contract", st);
              k_contract<DIM, P, PH, MODE, false><<<nb, 256, dsm, st>>>(s->dev, Dt, Rt, e0, ldq, val, F); }
        }
        launches += 2;
    }
    s->last_launches = launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("kernel launch: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

template <int DIM, int P, class PH>
static iga_status dispatch_mode(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                                const double *Ud, double *val, double *F, cudaStream_t st) {
    if (s->mode == MODE_PARAM) return run_form<DIM, P, PH, MODE_PARAM>(s, ph, a, b, U, Ud, val, F, st);
    if constexpr (std::is_same<PH, PhysNSVMS>::value || std::is_same<PH, PhysNSK>::value) {
        set_error("NS_VMS / NSK support parametric geometry with unit weights only");
        return IGA_ERR_PARAM;
    } else {
        return run_form<DIM, P, PH, MODE_NURBS>(s, ph, a, b, U, Ud, val, F, st);
    }
}

template <int DIM, class PH>
static iga_status dispatch_p(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                             const double *Ud, double *val, double *F, cudaStream_t st) {
    const int p = s->p[0];
    switch (p) {
    case 1: return dispatch_mode<DIM, 1, PH>(s, ph, a, b, U, Ud, val, F, st);
    case 2: return dispatch_mode<DIM, 2, PH>(s, ph, a, b, U, Ud, val, F, st);
    case 3: return dispatch_mode<DIM, 3, PH>(s, ph, a, b, U, Ud, val, F, st);
    default: break;
    }
    set_error("degree must be 1, 2 or 3 (equal on all axes) in this build");
    return IGA_ERR_PARAM;
}

iga_status launch_form(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                       const double *Ud, double *val, double *F, cudaStream_t st) {
    if (!s->force_split) {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
        iga_status fs = launch_fused2d(s, ph, a, b, U, Ud, val, F, st, nsm);
        if (fs != IGA_ERR_STATE) return fs;
        fs = launch_fused3d(s, ph, a, b, U, Ud, val, F, st, nsm);
        if (fs != IGA_ERR_STATE) return fs;
        fs = launch_fused2dm(s, ph, a, b, U, Ud, val, F, st, nsm);
        if (fs != IGA_ERR_STATE) return fs;
    }
    for (int d = 1; d < s->dim; d++)
        if (s->p[d] != s->p[0]) { set_error("degree must be equal on all axes in this build"); return IGA_ERR_PARAM; }
    for (int d = 0; d < s->dim; d++)
        if (s->nq[d] != s->p[d] + 1) { set_error("quad must be p+1 in this build"); return IGA_ERR_PARAM; }
    switch (ph->kind) {
    case IGA_PHYS_LAPLACE:
        if (s->dof != 1) break;
        if (s->dim == 2) return dispatch_p<2, PhysLaplace>(s, ph, a, b, U, Ud, val, F, st);
        if (s->dim == 3) return dispatch_p<3, PhysLaplace>(s, ph, a, b, U, Ud, val, F, st);
        break;
    case IGA_PHYS_CAHN_HILLIARD:
        if (s->dof != 1) break;
        if (s->dim == 2) return dispatch_p<2, PhysCahnHilliard>(s, ph, a, b, U, Ud, val, F, st);
        if (s->dim == 3) return dispatch_p<3, PhysCahnHilliard>(s, ph, a, b, U, Ud, val, F, st);
        break;
    case IGA_PHYS_NEOHOOKE:
        if (s->dof != 3 || s->dim != 3) break;
        return dispatch_p<3, PhysNeoHooke>(s, ph, a, b, U, Ud, val, F, st);
    case IGA_PHYS_NS_VMS:
        if (s->dof != 4 || s->dim != 3) break;
        return dispatch_p<3, PhysNSVMS>(s, ph, a, b, U, Ud, val, F, st);
    case IGA_PHYS_NSK:
        if (s->dof != 3 || s->dim != 2) break;
        return dispatch_p<2, PhysNSK>(s, ph, a, b, U, Ud, val, F, st);
    default:
        set_error("unknown physics kind");
        return IGA_ERR_PARAM;
    }
    set_error("physics / dim / dof combination not supported");
    return IGA_ERR_PARAM;
}

// Element sub-box launch (multi-rank schedule, dist.cu): the kernels take their element range
// from the space (SpaceDev axes, el_lo/el_hi, nel_local), so the sub-box is swapped in for the
// launch and restored; the outputs are not zeroed (the caller zeroes them once per form).
iga_status launch_form_box(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                           const double *Ud, double *val, double *F, cudaStream_t st, const int lo[3],
                           const int hi[3]) {
    long long nel = 1, nqp = 1;
    for (int d = 0; d < 3; d++) {
        if (hi[d] <= lo[d]) return IGA_OK;            // empty box
        nel *= hi[d] - lo[d];
        nqp *= (long long)(hi[d] - lo[d]) * s->nq[d];
    }
    int sl[3], sh[3];
    const long long snel = s->nel_local, snqp = s->nqp_local;
    for (int d = 0; d < 3; d++) {
        sl[d] = s->el_lo[d]; sh[d] = s->el_hi[d];
        s->el_lo[d] = s->dev.ax[d].el_lo = lo[d];
        s->el_hi[d] = s->dev.ax[d].el_hi = hi[d];
    }
    s->nel_local = nel;
    s->nqp_local = nqp;
    const int skip = s->skip_zero;
    s->skip_zero = 1;
    iga_status r = launch_form(s, ph, a, b, U, Ud, val, F, st);
    s->skip_zero = skip;
    s->nel_local = snel;
    s->nqp_local = snqp;
    for (int d = 0; d < 3; d++) {
        s->el_lo[d] = s->dev.ax[d].el_lo = sl[d];
        s->el_hi[d] = s->dev.ax[d].el_hi = sh[d];
    }
    return r;
}

}  // namespace iga
