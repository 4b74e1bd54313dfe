// iga_internal.cuh -- device-side data layout of an IGA space (libiga internals).
//
// HBM layout: everything per axis is a few KB (1D tables, spans,
// Alg. 3 stencils); the only large arrays are the caller's CSR (row_ptr/col_idx/val), the
// vectors, and the per-batch quadrature-point coefficient workspace.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/iga.h"

namespace iga {

constexpr int MAXP = 3;          // degrees 1..3 in this build
constexpr int MAXD = 3;

enum Mode { MODE_PARAM = 0, MODE_NURBS = 1 };   // x = xi, unit weights  |  rational / mapped

// One parametric axis (device pointers).
struct AxisDev {
    int p;            // degree
    int nel;          // elements (nonzero spans) on this axis (global)
    int nu;           // unique functions (periodic identification, SURVEY A-8)
    int nq;           // Gauss points per element
    const double *tab;        // [nel][nq][3][p+1]  N, N', N'' of the span's p+1 functions
    const double *qw;         // [nel][nq]  Gauss weight * (h_e / 2)
    const double *qx;         // [nel][nq]  parametric coordinate of the Gauss point
    const double *hpar;       // [nel]      span length h_e
    const int *first;         // [nel]      first (unwrapped) function index of the span = s - p
    const int *pos;           // [nel][p+1][p+1] position of function beta in row alpha's columns
    const int *rowW;          // [nu]       Alg. 3 stencil width (columns per row, per axis)
    const long long *rowS;    // [nu]       exclusive prefix of rowW over the OWNED range
    const int *cols;          // [nu][colmax] sorted, wrapped column lists
    int colmax;
    long long T;              // sum of rowW over the owned range
    int own_lo, own_hi;       // owned function range [lo, hi)
    int el_lo, el_hi;         // this rank's element range [lo, hi)
    const int *suplo;         // [nu] first element of the (cyclic) support of function g
    const int *supcnt;        // [nu] number of elements in that support
    const int *posd;          // [nu][2p+1] position of column g+delta in row g's list, or -1
    int uniform;              // first[e+1] == first[e] + 1 for all e (simple interior knots)
    int first0;               // first[0] (uniform: first[e] = first0 + e)
    int uni_lo, uni_hi;       // elements [uni_lo, uni_hi) share the middle element's 1D tables
    // touched box of this rank (box decomposition): local index l = g - own_lo
    // (mod nu) in [0, x_n); l < n_own are owned functions, the next x_n - n_own are the halo
    // (owned by the upper neighbour).  Single rank: own_lo = 0, n_own = x_n = nu.
    int n_own, x_n;
    const long long *lS;      // [x_n] prefix of rowW restarting at the owned/halo boundary
    long long Th;             // sum of rowW over the halo segment
};

struct SpaceDev {
    int dim, dof, mode;
    int weighted;             // weights present (rational basis)
    int geom;                 // iga_geom
    AxisDev ax[MAXD];
    const double *ctrl;       // [nnodes][dim]   (NURBS geometry)
    const double *wts;        // [nnodes]        (or nullptr)
    long long nnodes;
    int *errflag;             // device error flag (bit 0: detJ<=0, bit 1: non-finite)
    unsigned long long *wq;   // element work counter of the persistent 3D kernel (zeroed per launch)
    // multi-rank: CSR rows of halo functions (sub-box id s != 0, bit d-1-a set = halo on axis a)
    // accumulate into the library's halo buffer at hbase[s]; owned rows (s = 0) into csr_val
    double *halo;
    long long hbase[8];
};

// local (touched-box) index of unique function g on an axis
__host__ __device__ inline int local_fn(const AxisDev &ax, int g) {
    int l = g - ax.own_lo;
    if (l < 0) l += ax.nu;
    return l;
}

// node index in the touched box (the layout of U / Udot / F inside the kernels; equal to the
// global node index on a single rank)
__host__ __device__ inline long long local_node(const SpaceDev &s, int g0, int g1, int g2) {
    return ((long long)local_fn(s.ax[0], g0) * s.ax[1].x_n + local_fn(s.ax[1], g1)) * s.ax[2].x_n + local_fn(s.ax[2], g2);
}

// CSR row of functions (g0, g1, g2), component i: pointer to its first value and its width W
// (nodes).  Closed form over the touched box:
//   start = m^2 (S0 T1 T2 + W0 S1 T2 + W0 W1 S2) + i W m,  T_a = owned or halo segment total.
__device__ inline double *row_start(const SpaceDev &s, double *val, int g0, int g1, int g2, int i, int m,
                                    int *W_out = nullptr) {
    const int g[3] = {g0, g1, g2};
    long long S[3], T[3];
    int W[3], sub = 0;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const AxisDev &ax = s.ax[a];
        const int l = local_fn(ax, g[a]);
        const int seg = l >= ax.n_own;
        sub = sub * 2 + seg;
        S[a] = ax.lS[l];
        T[a] = seg ? ax.Th : ax.T;
        W[a] = ax.rowW[g[a]];
    }
    const long long Wn = (long long)W[0] * W[1] * W[2];
    if (W_out) *W_out = (int)Wn;
    double *base = sub ? s.halo + s.hbase[sub] : val;
    return base + (long long)m * m * (S[0] * T[1] * T[2] + W[0] * S[1] * T[2] + (long long)W[0] * W[1] * S[2])
           + (long long)i * Wn * m;
}

__host__ __device__ inline long long node_index(const SpaceDev &s, int g0, int g1, int g2) {
    return ((long long)g0 * s.ax[1].nu + g1) * s.ax[2].nu + g2;
}

// out-of-line copy for register-critical kernels (keeps the address arithmetic out of their
// register allocation)
static __device__ __noinline__ double *row_start_ni(const SpaceDev &s, double *val, int g0, int g1, int g2, int m,
                                                    int *W_out) {
    return row_start(s, val, g0, g1, g2, 0, m, W_out);
}

}  // namespace iga
