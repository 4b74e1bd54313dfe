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
};

__host__ __device__ inline long long node_index(const SpaceDev &s, int g0, int g1, int g2) {
    return ((long long)g0 * s.ax[1].nu + g1) * s.ax[2].nu + g2;
}

}  // namespace iga
