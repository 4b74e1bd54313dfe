// space.cu -- libiga space setup (host orchestration + kernels K1 basis tables, K2 CSR pattern)
// and the extern "C" entry points declared in include/iga.h.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "iga_host.h"

namespace iga {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

static cudaEvent_t prof_event(iga_space_s *s) {
    if (!s->prof_pool.empty()) {
        cudaEvent_t e = s->prof_pool.back();
        s->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(iga_space_s *s_, const char *n, cudaStream_t st_) : s(s_), name(n), st(st_) {
    if (!s->prof_on) return;
    a = prof_event(s);
    b = prof_event(s);
    cudaEventRecord(a, st);
}

ProfScope::~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    s->prof_pending.push_back({name, a, b});
}

static void prof_collect(iga_space_s *s) {
    for (auto &r : s->prof_pending) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        size_t k = 0;
        for (; k < s->prof_names.size(); k++)
            if (s->prof_names[k] == r.name) break;
        if (k == s->prof_names.size()) {
            s->prof_names.push_back(r.name);
            s->prof_count.push_back(0);
            s->prof_ms.push_back(0.0);
        }
        s->prof_count[k] += 1;
        s->prof_ms[k] += ms;
        s->prof_pool.push_back(r.a);
        s->prof_pool.push_back(r.b);
    }
    s->prof_pending.clear();
}

#define CUDA_TRY(x)                                                                   \
    do {                                                                              \
        cudaError_t _e = (x);                                                         \
        if (_e != cudaSuccess) {                                                      \
            set_error(std::string(#x) + ": " + cudaGetErrorString(_e));               \
            return IGA_ERR_CUDA;                                                      \
        }                                                                             \
    } while (0)

// ------------------------------------------------------------------------------------------
// K1: univariate basis N, N', N'' of the p+1 functions of a span at a point, by the triangular
// in-span scheme (the "more computationally efficient algorithm" P:191-193 points to): the
// upper triangle of ndu holds the degree-by-degree basis values, the lower triangle the knot
// differences, from which the derivatives follow by the recurrence on the a[][] coefficients.
// ------------------------------------------------------------------------------------------
__device__ void span_basis_ders(int span, double xi, int p, const double *U, double out[3][MAXP + 1]) {
    double ndu[MAXP + 1][MAXP + 1], left[MAXP + 1], right[MAXP + 1];
    ndu[0][0] = 1.0;
    for (int j = 1; j <= p; j++) {
        left[j] = xi - U[span + 1 - j];
        right[j] = U[span + j] - xi;
        double saved = 0.0;
        for (int r = 0; r < j; r++) {
            ndu[j][r] = right[r + 1] + left[j - r];
            const double tmp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        ndu[j][j] = saved;
    }
    for (int r = 0; r <= p; r++) {
        out[0][r] = ndu[r][p];
        out[1][r] = 0.0;
        out[2][r] = 0.0;
    }
    const int nd = p < 2 ? p : 2;
    double a[2][MAXP + 1];
    for (int r = 0; r <= p; r++) {
        int s1 = 0, s2 = 1;
        a[0][0] = 1.0;
        for (int k = 1; k <= nd; k++) {
            double d = 0.0;
            const int rk = r - k, pk = p - k;
            if (r >= k) {
                a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
                d = a[s2][0] * ndu[rk][pk];
            }
            const int j1 = (rk >= -1) ? 1 : -rk;
            const int j2 = (r - 1 <= pk) ? k - 1 : p - r;
            for (int j = j1; j <= j2; j++) {
                a[s2][j] = (a[s1][j] - a[s1][j - 1]) / ndu[pk + 1][rk + j];
                d += a[s2][j] * ndu[rk + j][pk];
            }
            if (r <= pk) {
                a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
                d += a[s2][k] * ndu[r][pk];
            }
            out[k][r] = d;
            const int t = s1; s1 = s2; s2 = t;
        }
    }
    double f = p;
    for (int k = 1; k <= nd; k++) {
        for (int r = 0; r <= p; r++) out[k][r] *= f;
        f *= (p - k);
    }
}

__global__ void k_tables(int nel, int nq, int p, const double *__restrict__ U, const int *__restrict__ first,
                         const double *__restrict__ qx, double *__restrict__ tab) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nel * nq) return;
    const int e = t / nq;
    double out[3][MAXP + 1];
    span_basis_ders(first[e] + p, qx[t], p, U, out);
    for (int k = 0; k < 3; k++)
        for (int a = 0; a <= p; a++) tab[(size_t)t * 3 * (p + 1) + k * (p + 1) + a] = out[k][a];
}

// ------------------------------------------------------------------------------------------
// K2: CSR pattern, one warp per owned row.  row r = (local node, component i);
//   row start = m^2 (S0 T1 T2 + W0 S1 T2 + W0 W1 S2) + i W m   (separable prefix sums)
//   entry t = ((c0 W1 + c1) W2 + c2) m + j  ->  column node(cols0[c0], cols1[c1], cols2[c2]) m + j
// ------------------------------------------------------------------------------------------
__global__ void k_pattern(SpaceDev s, long long nrows, long long nnz, long long *__restrict__ row_ptr,
                          int *__restrict__ col_idx) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nrows) return;
    const int m = s.dof;
    long long r = warp;
    const int i = (int)(r % m);
    r /= m;
    const int n1o = s.ax[1].own_hi - s.ax[1].own_lo, n2o = s.ax[2].own_hi - s.ax[2].own_lo;
    const int g2 = s.ax[2].own_lo + (int)(r % n2o);
    r /= n2o;
    const int g1 = s.ax[1].own_lo + (int)(r % n1o);
    r /= n1o;
    const int g0 = s.ax[0].own_lo + (int)r;
    const int W0 = s.ax[0].rowW[g0], W1 = s.ax[1].rowW[g1], W2 = s.ax[2].rowW[g2];
    const long long S0 = s.ax[0].rowS[g0], S1 = s.ax[1].rowS[g1], S2 = s.ax[2].rowS[g2];
    const long long T1 = s.ax[1].T, T2 = s.ax[2].T;
    const long long W = (long long)W0 * W1 * W2;
    const long long start = (long long)m * m * (S0 * T1 * T2 + W0 * S1 * T2 + (long long)W0 * W1 * S2) + i * W * m;
    if (lane == 0) {
        row_ptr[warp] = start;
        if (warp == nrows - 1) row_ptr[nrows] = nnz;
    }
    const int *c0 = s.ax[0].cols + (size_t)g0 * s.ax[0].colmax;
    const int *c1 = s.ax[1].cols + (size_t)g1 * s.ax[1].colmax;
    const int *c2 = s.ax[2].cols + (size_t)g2 * s.ax[2].colmax;
    const int nu1 = s.ax[1].nu, nu2 = s.ax[2].nu;
    const long long len = W * m;
    for (long long t = lane; t < len; t += 32) {
        long long u = t;
        const int j = (int)(u % m);
        u /= m;
        const int k2 = (int)(u % W2);
        u /= W2;
        const int k1 = (int)(u % W1);
        const int k0 = (int)(u / W1);
        const long long node = ((long long)c0[k0] * nu1 + c1[k1]) * nu2 + c2[k2];
        col_idx[start + t] = (int)(node * m + j);
    }
}

iga_status launch_pattern(iga_space_s *s, int64_t *row_ptr, int32_t *col_idx, cudaStream_t st) {
    const long long nrows = s->nrows_owned;
    if (nrows == 0) return IGA_OK;
    const long long threads = nrows * 32;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    {
        ProfScope ps(s, "k_pattern", st);
        k_pattern<<<blocks, 256, 0, st>>>(s->dev, nrows, s->nnz_owned, (long long *)row_ptr, col_idx);
    }
    CUDA_TRY(cudaGetLastError());
    s->last_launches = 1;
    return IGA_OK;
}

// ------------------------------------------------------------------------------------------
// host setup helpers
// ------------------------------------------------------------------------------------------
// Alg. 1: unclamp U (n+1 functions, degree p) for C^k periodicity, in place.
static void unclamp(std::vector<double> &U, int p, int k) {
    const int n = (int)U.size() - p - 2;
    const int m = n + p + 1;
    for (int i = 0; i <= k; i++) {
        U[k - i] = U[p] - U[n + 1] + U[n - i];
        U[m - k + i] = U[n + 1] - U[p] + U[p + i + 1];
    }
}

// Gauss-Legendre nodes/weights on [-1,1] (A-6), Newton on the three-term recurrence in double.
static void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    const double pi = 3.14159265358979323846;
    for (int i = 1; i <= n; i++) {
        double z = std::cos(pi * (i - 0.25) / (n + 0.5));
        double dp = 1.0;
        for (int it = 0; it < 100; it++) {
            double p0 = 1.0, p1 = z;
            for (int k = 2; k <= n; k++) {
                const double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = (n == 1) ? 1.0 : n * (p0 - z * p1) / (1.0 - z * z);
            const double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) <= 1e-17) break;
        }
        double p0 = 1.0, p1 = z;
        for (int k = 2; k <= n; k++) {
            const double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        dp = (n == 1) ? 1.0 : n * (p0 - z * p1) / (1.0 - z * z);
        x[n - i] = z;
        w[n - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

template <class T>
static iga_status dalloc(iga_space_s *s, T **p, size_t count) {
    void *ptr = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&ptr, count * sizeof(T));
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return IGA_ERR_NOMEM;
    }
    s->allocs.push_back(ptr);
    *p = (T *)ptr;
    return IGA_OK;
}

template <class T>
static iga_status upload(iga_space_s *s, T **p, const std::vector<T> &h) {
    iga_status st = dalloc(s, p, h.size());
    if (st != IGA_OK) return st;
    if (!h.empty()) CUDA_TRY(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return IGA_OK;
}

static void free_space(iga_space_s *s) {
    if (!s) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    prof_collect(s);
    dist_destroy(s);
    for (cudaEvent_t e : s->prof_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : s->hb_ev) cudaEventDestroy(e);
    if (s->hb_copy) cudaStreamDestroy(s->hb_copy);
    for (void *p : s->allocs) cudaFree(p);
    for (void *p : s->gm_buf) if (p) cudaFree(p);
    for (auto &c : s->dr_cache) if (c.first) cudaFree(c.first);
    cudaSetDevice(prev);
    delete s;
}


// ------------------------------------------------------------------------------------------
// Alg. 2 ("UnclampCurve"): unclamp one line of n+1 homogeneous control points (h
// doubles each, `st` doubles apart) for C^k periodicity, given a copy of the axis' OPEN knots;
// left end (knots, then points), right end likewise.  Then geometry_unique() applies it to every
// line of every periodic axis of the open control net, requires the last k+1 points of each line
// to repeat its first k+1 (the periodic identification) and keeps the nu unique ones.
// ------------------------------------------------------------------------------------------
static void unclamp_line(std::vector<double> U, int p, int k, double *P, int h, long long st) {
    const int n = (int)U.size() - p - 2, m = n + p + 1;
    for (int i = 0; i <= k; i++) U[k - i] = U[p] - U[n + 1] + U[n - i];
    for (int i = p - k - 1; i <= p - 2; i++)
        for (int j = i; j >= 0; j--) {
            const double al = (U[p] - U[p + j - i - 1]) / (U[p + j + 1] - U[p + j - i - 1]);
            double *a = P + j * st, *b = P + (j + 1) * st;
            for (int c = 0; c < h; c++) a[c] = (a[c] - al * b[c]) / (1.0 - al);
        }
    for (int i = 0; i <= k; i++) U[m - k + i] = U[n + 1] - U[p] + U[p + i + 1];
    for (int i = p - k - 1; i <= p - 2; i++)
        for (int j = i; j >= 0; j--) {
            const double al = (U[n + 1] - U[n - j]) / (U[n - j + i + 2] - U[n - j]);
            double *a = P + (n - j) * st, *b = P + (n - j - 1) * st;
            for (int c = 0; c < h; c++) a[c] = (a[c] - (1.0 - al) * b[c]) / al;
        }
}

static iga_status geometry_unique(const iga_space_desc *d, const int *nfun, const int *nu, std::vector<double> &ctrl,
                                  std::vector<double> &wts) {
    const int dim = d->dim, h = dim + 1;
    long long nopen = 1, nuniq = 1;
    for (int a = 0; a < dim; a++) { nopen *= nfun[a]; nuniq *= nu[a]; }
    std::vector<double> P((size_t)nopen * h);
    for (long long q = 0; q < nopen; q++) {
        const double w = d->weights ? d->weights[q] : 1.0;
        if (!(w > 0.0)) { set_error("weights must be > 0"); return IGA_ERR_DOMAIN; }
        for (int c = 0; c < dim; c++) P[q * h + c] = (d->ctrl ? d->ctrl[q * dim + c] : 0.0) * w;
        P[q * h + dim] = w;
    }
    long long pstride[3] = {1, 1, 1};          // point stride per axis on the open grid
    for (int a = dim - 2; a >= 0; a--) pstride[a] = pstride[a + 1] * nfun[a + 1];
    for (int a = 0; a < dim; a++) {
        if (!d->periodic[a]) continue;
        const int p = d->degree[a], k = d->periodic_continuity[a];
        const std::vector<double> U0(d->knots[a], d->knots[a] + d->n_knots[a]);
        for (long long q = 0; q < nopen; q++) {
            if ((q / pstride[a]) % nfun[a] != 0) continue;       // one line per base point
            double *line = P.data() + q * h;
            unclamp_line(U0, p, k, line, h, pstride[a] * h);
            for (int g = 0; g <= k; g++)
                for (int c = 0; c < h; c++) {
                    const double x0 = line[g * pstride[a] * h + c], x1 = line[(nu[a] + g) * pstride[a] * h + c];
                    if (std::fabs(x0 - x1) > 1e-10 * (1.0 + std::fabs(x0))) {
                        set_error("geometry on a periodic axis is not C^k periodic: Alg. 2 leaves its wrapped "
                                  "control points distinct");
                        return IGA_ERR_DOMAIN;
                    }
                }
        }
    }
    ctrl.assign(d->ctrl ? (size_t)nuniq * dim : 0, 0.0);
    wts.assign(d->weights ? (size_t)nuniq : 0, 0.0);
    for (long long u = 0; u < nuniq; u++) {
        long long rem = u, q = 0;
        int ui[3] = {0, 0, 0};
        for (int a = dim - 1; a >= 0; a--) { ui[a] = (int)(rem % nu[a]); rem /= nu[a]; }
        for (int a = 0; a < dim; a++) q = q * nfun[a] + ui[a];
        const double w = P[q * h + dim];
        if (d->ctrl)
            for (int c = 0; c < dim; c++) ctrl[u * dim + c] = P[q * h + c] / w;
        if (d->weights) wts[u] = w;
    }
    return IGA_OK;
}

// ------------------------------------------------------------------------------------------
// per-axis host setup (no CUDA): knots (Alg. 1 unclamping), elements, Gauss rule, Alg. 3
// stencils, supports, and the box decomposition of the axis over P rank coordinates
// (b_r = floor(N r / P)) with DOF ownership A-9 (owner of a function = owner of the
// last element of its support).  Touched-but-not-owned functions ("halo") must be the next
// `halo` functions after the owned range, owned by coordinate c+1 (mod P on periodic axes):
// true for uniform knots with >= p elements per rank; anything else is rejected.
// ------------------------------------------------------------------------------------------
iga_status axis_host(const iga_space_desc *d, int a, int P, AxisHost &H) {
    const int p = d->degree[a];
    if (p < 1 || p > MAXP) { set_error("degree must be 1..3"); return IGA_ERR_PARAM; }
    const int nk = d->n_knots[a];
    if (nk < 2 * (p + 1) || !d->knots[a]) { set_error("too few knots"); return IGA_ERR_DOMAIN; }
    std::vector<double> U(d->knots[a], d->knots[a] + nk);
    for (int i = 0; i + 1 < nk; i++)
        if (!(U[i] <= U[i + 1])) { set_error("knots must be non-decreasing"); return IGA_ERR_DOMAIN; }
    const int nfun = nk - p - 1;
    int nu = nfun;
    H.periodic = d->periodic[a] ? 1 : 0;
    if (H.periodic) {
        const int k = d->periodic_continuity[a];
        if (k < 0 || k > p - 1) { set_error("periodic continuity must be in [0, p-1]"); return IGA_ERR_DOMAIN; }
        unclamp(U, p, k);
        nu = nfun - (k + 1);
    }
    // elements: nonzero spans inside [U_p, U_nfun]
    std::vector<int> first;
    std::vector<double> hpar;
    for (int sp = p; sp < nfun; sp++)
        if (U[sp] < U[sp + 1]) { first.push_back(sp - p); hpar.push_back(U[sp + 1] - U[sp]); }
    const int nel = (int)first.size();
    if (H.periodic && nu < 2 * p + 1) { set_error("periodic axis needs >= 2p+1 functions"); return IGA_ERR_DOMAIN; }
    const int nq = d->quad[a] > 0 ? d->quad[a] : p + 1;
    std::vector<double> gx, gw;
    gauss_legendre(nq, gx, gw);
    std::vector<double> qx((size_t)nel * nq), qw((size_t)nel * nq);
    for (int e = 0; e < nel; e++) {
        const double lo = U[first[e] + p], hi = U[first[e] + p + 1];
        for (int q = 0; q < nq; q++) {
            qx[(size_t)e * nq + q] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx[q];
            qw[(size_t)e * nq + q] = gw[q] * 0.5 * (hi - lo);
        }
    }
    // Alg. 3 on every representative i of each unique function, wrapped mod nu
    std::vector<std::vector<int>> colset(nu);
    for (int i = 0; i < nfun; i++) {
        int k = i;
        while (k + 1 < nk && U[k] == U[k + 1]) k++;
        const int l = k - p;
        k = i + p + 1;
        while (k - 1 >= 0 && U[k] == U[k - 1]) k--;
        const int r = k - 1;
        auto &cs = colset[i % nu];
        for (int j = l; j <= r; j++) cs.push_back(((j % nu) + nu) % nu);
    }
    int colmax = 1;
    std::vector<int> rowW(nu);
    for (int g = 0; g < nu; g++) {
        auto &cs = colset[g];
        std::sort(cs.begin(), cs.end());
        cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
        rowW[g] = (int)cs.size();
        colmax = std::max(colmax, rowW[g]);
    }
    std::vector<int> cols((size_t)nu * colmax, 0);
    for (int g = 0; g < nu; g++) std::copy(colset[g].begin(), colset[g].end(), cols.begin() + (size_t)g * colmax);
    // per element: position of column function beta in row function alpha's list
    std::vector<int> pos((size_t)nel * (p + 1) * (p + 1));
    for (int e = 0; e < nel; e++)
        for (int al = 0; al <= p; al++)
            for (int be = 0; be <= p; be++) {
                const int ga = (first[e] + al) % nu, gb = (first[e] + be) % nu;
                const auto &cs = colset[ga];
                pos[((size_t)e * (p + 1) + al) * (p + 1) + be] = (int)(std::lower_bound(cs.begin(), cs.end(), gb) - cs.begin());
            }
    // ownership (A-9)
    std::vector<int> last_el(nu, -1);
    for (int e = 0; e < nel; e++)
        for (int al = 0; al <= p; al++) {
            const int i = first[e] + al;
            if (i < nu) last_el[i] = std::max(last_el[i], e);     // representative i = g
        }
    for (int g = 0; g < nu; g++)
        if (last_el[g] < 0) last_el[g] = nel - 1;
    if (P < 1 || P > nel) { set_error("more ranks than elements on an axis"); return IGA_ERR_PARAM; }
    H.el_lo.assign(P, 0); H.el_hi.assign(P, 0); H.own_lo.assign(P, 0); H.own_hi.assign(P, 0); H.halo.assign(P, 0);
    for (int c = 0; c < P; c++) {
        const int el_lo = (int)((long long)nel * c / P), el_hi = (int)((long long)nel * (c + 1) / P);
        int own_lo = nu, own_hi = 0, cnt = 0;
        for (int g = 0; g < nu; g++)
            if (last_el[g] >= el_lo && last_el[g] < el_hi) { own_lo = std::min(own_lo, g); own_hi = std::max(own_hi, g + 1); cnt++; }
        if (own_hi <= own_lo || cnt != own_hi - own_lo) { set_error("rank owns no (or a non-contiguous set of) functions on an axis"); return IGA_ERR_PARAM; }
        H.el_lo[c] = el_lo; H.el_hi[c] = el_hi; H.own_lo[c] = own_lo; H.own_hi[c] = own_hi;
    }
    for (int c = 0; c < P; c++) {
        // touched functions of coordinate c's elements
        std::vector<char> touched(nu, 0);
        for (int e = H.el_lo[c]; e < H.el_hi[c]; e++)
            for (int al = 0; al <= p; al++) touched[(first[e] + al) % nu] = 1;
        int nt = 0;
        for (int g = 0; g < nu; g++) nt += touched[g];
        const int n_own = H.own_hi[c] - H.own_lo[c];
        const int h = nt - n_own;
        bool ok = h >= 0 && (P > 1 || h == 0);
        for (int l = 0; ok && l < nt; l++) ok = touched[(H.own_lo[c] + l) % nu] != 0;
        if (ok && h > 0) {
            const int cn = H.periodic ? (c + 1) % P : c + 1;
            ok = cn < P && cn != c && (H.own_lo[cn] == H.own_hi[c] % nu) && (H.own_hi[cn] - H.own_lo[cn] >= h);
        }
        if (!ok) { set_error("box decomposition: a rank's halo is not owned by its upper neighbour (too many ranks for this axis?)"); return IGA_ERR_PARAM; }
        H.halo[c] = h;
    }
    // cyclic support [suplo, suplo+supcnt) of each unique function, and delta positions
    std::vector<int> suplo(nu, 0), supcnt(nu, 0), posd((size_t)nu * (2 * p + 1), -1);
    {
        std::vector<std::vector<int>> sup(nu);
        for (int e = 0; e < nel; e++)
            for (int al = 0; al <= p; al++) sup[(first[e] + al) % nu].push_back(e);
        for (int g = 0; g < nu; g++) {
            auto &v = sup[g];
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            const int c = (int)v.size();
            int lo = c ? v[0] : 0;
            // cyclic start: the element whose predecessor (mod nel) is not in the support
            for (int k = 0; k < c; k++) {
                const int prev = (v[k] - 1 + nel) % nel;
                if (!std::binary_search(v.begin(), v.end(), prev)) { lo = v[k]; break; }
            }
            suplo[g] = lo;
            supcnt[g] = c;
            for (int dl = -p; dl <= p; dl++) {
                if (!H.periodic && (g + dl < 0 || g + dl >= nu)) continue;   // no wrap on open axes
                const int col = (((g + dl) % nu) + nu) % nu;
                const auto &cs = colset[g];
                auto it = std::lower_bound(cs.begin(), cs.end(), col);
                if (it != cs.end() && *it == col) posd[(size_t)g * (2 * p + 1) + dl + p] = (int)(it - cs.begin());
            }
        }
    }
    int uniform = 1;
    for (int e = 0; e + 1 < nel; e++)
        if (first[e + 1] != first[e] + 1) uniform = 0;
    H.p = p; H.nel = nel; H.nu = nu; H.nfun = nfun; H.nq = nq; H.colmax = colmax; H.uniform = uniform;
    H.U = std::move(U); H.first = std::move(first); H.hpar = std::move(hpar); H.qx = std::move(qx); H.qw = std::move(qw);
    H.rowW = std::move(rowW); H.cols = std::move(cols); H.pos = std::move(pos);
    H.suplo = std::move(suplo); H.supcnt = std::move(supcnt); H.posd = std::move(posd);
    return IGA_OK;
}

static iga_status create(const iga_space_desc *d, const iga_dist *dist, int device, iga_space *out) {
    if (!d || !out) { set_error("null argument"); return IGA_ERR_PARAM; }
    *out = nullptr;
    if (d->dim < 2 || d->dim > 3) { set_error("dim must be 2 or 3 in this build"); return IGA_ERR_PARAM; }
    if (d->dof < 1 || d->dof > 4) { set_error("dof must be 1..4"); return IGA_ERR_PARAM; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_error("no CUDA device (libiga has no CPU fallback)");
        return IGA_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) { set_error("bad device ordinal"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    CUDA_TRY(cudaSetDevice(device));
    iga_space_s *s = new iga_space_s();
    s->device = device;
    s->dim = d->dim;
    s->dof = d->dof;
    s->geom = d->geometry;
    s->weighted = d->weights != nullptr;
    s->mode = (d->geometry == IGA_GEOM_NURBS || d->weights) ? MODE_NURBS : MODE_PARAM;
    if (d->geometry == IGA_GEOM_NURBS && !d->ctrl) { delete s; set_error("NURBS geometry needs ctrl"); return IGA_ERR_PARAM; }
    // distribution
    if (dist) {
        s->rank = dist->rank;
        s->nranks = dist->nranks;
        int prod = 1;
        for (int a = 0; a < 3; a++) {
            s->procs[a] = a < d->dim ? std::max(1, dist->procs[a]) : 1;
            prod *= s->procs[a];
        }
        if (prod != s->nranks || s->rank < 0 || s->rank >= s->nranks) {
            delete s;
            set_error("iga_dist: procs product must equal nranks and 0 <= rank < nranks");
            return IGA_ERR_PARAM;
        }
        int r = s->rank;
        s->rcoord[2] = r % s->procs[2]; r /= s->procs[2];
        s->rcoord[1] = r % s->procs[1]; r /= s->procs[1];
        s->rcoord[0] = r;
    }
    iga_status st = IGA_OK;
    long long nnodes = 1, nrows_nodes = 1;
    s->dev.ctrl = nullptr;
    s->dev.wts = nullptr;
    for (int a = 0; a < 3; a++) {
        AxisDev &ax = s->dev.ax[a];
        if (a >= d->dim) {
            // trivial axis: one element, one function, one point
            s->p[a] = 0; s->nel[a] = 1; s->nu[a] = 1; s->nq[a] = 1; s->nfun[a] = 1;
            s->rowW[a] = {1};
            s->cols[a] = {0};
            s->colmax[a] = 1;
            ax.p = 0; ax.nel = 1; ax.nu = 1; ax.nq = 1;
            std::vector<double> one = {1.0, 0.0, 0.0}, w1 = {1.0}, x0 = {0.0}, h1 = {1.0};
            std::vector<int> z = {0}, one_i = {1}, zc = {0};
            std::vector<long long> zl = {0};
            if ((st = upload(s, (double **)&ax.tab, one)) != IGA_OK) goto fail;
            if ((st = upload(s, (double **)&ax.qw, w1)) != IGA_OK) goto fail;
            if ((st = upload(s, (double **)&ax.qx, x0)) != IGA_OK) goto fail;
            if ((st = upload(s, (double **)&ax.hpar, h1)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.first, z)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.pos, z)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.rowW, one_i)) != IGA_OK) goto fail;
            if ((st = upload(s, (long long **)&ax.rowS, zl)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.cols, zc)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.suplo, z)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.supcnt, one_i)) != IGA_OK) goto fail;
            if ((st = upload(s, (int **)&ax.posd, z)) != IGA_OK) goto fail;
            if ((st = upload(s, (long long **)&ax.lS, zl)) != IGA_OK) goto fail;
            if ((st = upload(s, (double **)&s->dknots[a], x0)) != IGA_OK) goto fail;
            ax.n_own = 1; ax.x_n = 1; ax.Th = 0;
            ax.uni_lo = 0; ax.uni_hi = 1;
            ax.uniform = 1;
            ax.first0 = 0;
            ax.colmax = 1; ax.T = 1; ax.own_lo = 0; ax.own_hi = 1; ax.el_lo = 0; ax.el_hi = 1;
            s->own_lo[a] = 0; s->own_hi[a] = 1; s->el_lo[a] = 0; s->el_hi[a] = 1;
            continue;
        }
        AxisHost H;
        if ((st = axis_host(d, a, s->procs[a], H)) != IGA_OK) goto fail;
        const int p = H.p, nel = H.nel, nu = H.nu, nfun = H.nfun, nq = H.nq;
        const int rc = s->rcoord[a];
        const int el_lo = H.el_lo[rc], el_hi = H.el_hi[rc], own_lo = H.own_lo[rc], own_hi = H.own_hi[rc];
        const int halo = H.halo[rc], n_own = own_hi - own_lo;
        std::vector<double> &U = H.U, &qx = H.qx, &qw = H.qw, &hpar = H.hpar;
        std::vector<int> &first = H.first, &rowW = H.rowW, &cols = H.cols, &pos = H.pos;
        std::vector<int> &suplo = H.suplo, &supcnt = H.supcnt, &posd = H.posd;
        const int colmax = H.colmax, uniform = H.uniform;
        s->periodic[a] = H.periodic;
        // closed-form CSR row starts over the touched box: prefix sums of the Alg. 3 widths,
        // restarting at the owned / halo segment boundary (local index l = g - own_lo mod nu)
        std::vector<long long> rowS(nu, 0), lS(n_own + halo + 1, 0);
        long long T = 0, Th = 0;
        for (int g = own_lo; g < own_hi; g++) { rowS[g] = T; T += rowW[g]; }
        for (int l = 0; l < n_own; l++) lS[l] = rowS[own_lo + l];
        for (int l = n_own; l < n_own + halo; l++) { lS[l] = Th; Th += rowW[(own_lo + l) % nu]; }
        s->halo[a] = halo;
        s->Th[a] = Th;
        s->part[a] = H;
        s->p[a] = p; s->nel[a] = nel; s->nu[a] = nu; s->nq[a] = nq; s->nfun[a] = nfun;
        s->U[a] = U; s->rowW[a] = rowW; s->cols[a] = cols; s->colmax[a] = colmax;
        s->own_lo[a] = own_lo; s->own_hi[a] = own_hi; s->el_lo[a] = el_lo; s->el_hi[a] = el_hi;
        ax.p = p; ax.nel = nel; ax.nu = nu; ax.nq = nq; ax.colmax = colmax; ax.T = T;
        ax.own_lo = own_lo; ax.own_hi = own_hi; ax.el_lo = el_lo; ax.el_hi = el_hi;
        double *dU = nullptr;
        double *dtab = nullptr;
        if ((st = upload(s, &dU, U)) != IGA_OK) goto fail;
        s->dknots[a] = dU;
        if ((st = upload(s, (double **)&ax.qw, qw)) != IGA_OK) goto fail;
        if ((st = upload(s, (double **)&ax.qx, qx)) != IGA_OK) goto fail;
        if ((st = upload(s, (double **)&ax.hpar, hpar)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.first, first)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.pos, pos)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.rowW, rowW)) != IGA_OK) goto fail;
        if ((st = upload(s, (long long **)&ax.rowS, rowS)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.cols, cols)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.suplo, suplo)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.supcnt, supcnt)) != IGA_OK) goto fail;
        if ((st = upload(s, (int **)&ax.posd, posd)) != IGA_OK) goto fail;
        if ((st = upload(s, (long long **)&ax.lS, lS)) != IGA_OK) goto fail;
        ax.n_own = n_own; ax.x_n = n_own + halo; ax.Th = Th;
        ax.uniform = uniform;
        ax.first0 = first.empty() ? 0 : first[0];
        if ((st = dalloc(s, &dtab, (size_t)nel * nq * 3 * (p + 1))) != IGA_OK) goto fail;
        {
            const int nt = nel * nq;
            k_tables<<<(nt + 127) / 128, 128>>>(nel, nq, p, dU, ax.first, ax.qx, dtab);
            cudaError_t ce = cudaGetLastError();
            if (ce != cudaSuccess) { st = IGA_ERR_CUDA; set_error(cudaGetErrorString(ce)); goto fail; }
        }
        ax.tab = dtab;
        {
            // uniform-table detection: the maximal run of elements around the middle one whose 1D
            // tables, Gauss weights and span lengths equal the middle element's (all of them on
            // periodic / uniform knots; all but p at each end on open uniform knots).  The fused
            // kernels' fast path uses the middle element's tables for elements of that run.
            std::vector<double> ht((size_t)nel * nq * 3 * (p + 1));
            CUDA_TRY(cudaMemcpy(ht.data(), dtab, ht.size() * sizeof(double), cudaMemcpyDeviceToHost));
            const size_t per = (size_t)nq * 3 * (p + 1);
            const int em = nel / 2;
            double mx = 0.0;
            for (size_t k = 0; k < per; k++) mx = std::max(mx, std::fabs(ht[em * per + k]));
            auto same = [&](int e) {
                for (size_t k = 0; k < per; k++)
                    if (std::fabs(ht[e * per + k] - ht[em * per + k]) > 1e-13 * mx) return false;
                // spans of a uniform vector on [a, b] agree only to ~n ulp(b) / h in fp64 (config 5 on
                // [0, 2 pi]: 1.8e-14 relative), so the weights and span lengths are compared to 1e-13:
                // the middle element's values then differ from an element's own by < 1e-13
                // relative, two orders below the 1e-11 parity bar
                for (int q = 0; q < nq; q++)
                    if (std::fabs(qw[(size_t)e * nq + q] - qw[(size_t)em * nq + q]) > 1e-13 * std::fabs(qw[(size_t)em * nq + q]))
                        return false;
                return std::fabs(hpar[e] - hpar[em]) <= 1e-13 * hpar[em];
            };
            int ilo = em, ihi = em + 1;
            while (ilo > 0 && same(ilo - 1)) ilo--;
            while (ihi < nel && same(ihi)) ihi++;
            const bool uni = ilo == 0 && ihi == nel;
            ax.uni_lo = ilo;
            ax.uni_hi = ihi;
            s->tab0[a].assign(ht.begin() + em * per, ht.begin() + (em + 1) * per);
            s->qw0[a].assign(qw.begin() + (size_t)em * nq, qw.begin() + (size_t)(em + 1) * nq);
            s->hp0[a] = hpar[em];
            s->tab_uniform[a] = uni ? 1 : 0;
        }
        nnodes *= nu;
        nrows_nodes *= (own_hi - own_lo);
    }
    {
        s->dev.dim = s->dim;
        s->dev.dof = s->dof;
        s->dev.mode = s->mode;
        s->dev.weighted = s->weighted;
        s->dev.geom = s->geom;
        s->dev.nnodes = nnodes;
        const int m = s->dof;
        s->ndof_global = nnodes * m;
        s->nrows_owned = nrows_nodes * m;
        long long Tprod = 1;
        for (int a = 0; a < 3; a++) Tprod *= s->dev.ax[a].T;
        s->nnz_owned = Tprod * m * m;
        s->nel_local = 1;
        s->nqp_local = 1;
        for (int a = 0; a < 3; a++) {
            s->nel_local *= (s->el_hi[a] - s->el_lo[a]);
            s->nqp_local *= (long long)(s->el_hi[a] - s->el_lo[a]) * s->nq[a];
        }
        if (d->geometry == IGA_GEOM_NURBS || d->weights) {
            // control net / weights: given on the OPEN function grid; periodic axes unclamped
            // with Alg. 2 and reduced to the unique functions
            std::vector<double> c, w;
            if ((st = geometry_unique(d, s->nfun, s->nu, c, w)) != IGA_OK) goto fail;
            if (d->geometry == IGA_GEOM_NURBS && (st = upload(s, (double **)&s->dev.ctrl, c)) != IGA_OK) goto fail;
            if (d->weights && (st = upload(s, (double **)&s->dev.wts, w)) != IGA_OK) goto fail;
        }
        if ((st = dalloc(s, &s->errflag, 1)) != IGA_OK) goto fail;
        CUDA_TRY(cudaMemset(s->errflag, 0, sizeof(int)));
        s->dev.errflag = s->errflag;
        if ((st = dalloc(s, &s->dev.wq, 1)) != IGA_OK) goto fail;
        if (s->nranks > 1 && (st = dist_setup(s, dist)) != IGA_OK) goto fail;
        // quadrature-point coefficient workspace: <= 4 GiB, sized to the local element count
        size_t want = (size_t)s->nqp_local * 512 * sizeof(double);
        const size_t cap = (size_t)4 << 30;
        s->work_bytes = std::min(want, cap);
        s->work_bytes = std::max<size_t>(s->work_bytes, 1 << 20);
        if ((st = dalloc(s, (char **)&s->work, s->work_bytes)) != IGA_OK) goto fail;
        CUDA_TRY(cudaDeviceSynchronize());
    }
    cudaSetDevice(prev);
    *out = s;
    return IGA_OK;
fail:
    free_space(s);
    cudaSetDevice(prev);
    return st;
}

}  // namespace iga

using namespace iga;

iga_status iga::check_phys(iga_space s, const iga_phys *phys) {
    if (!s || !phys) { set_error("null argument"); return IGA_ERR_PARAM; }
    return IGA_OK;
}

// single-space form: one rank, or one rank of an NCCL decomposition
iga_status iga::form_one(iga_space s, const iga_phys *phys, double a, double b, const double *U, const double *Ud,
                           double *val, double *F, cudaStream_t st) {
    if (s->nranks > 1) {
        if (!s->dist || dist_transport(s->dist) != IGA_XPORT_NCCL) {
            set_error("IGA_XPORT_LOCAL spaces form through iga_form_*_group");
            return IGA_ERR_STATE;
        }
        return dist_form(&s, 1, phys, a, b, &U, &Ud, &val, &F, st);
    }
    return launch_form(s, phys, a, b, U, Ud, val, F, st);
}


extern "C" {

const char *iga_last_error(void) { return g_err.c_str(); }
const char *iga_version(void) { return "libiga 0.1 (sm_100a, fp64)"; }

iga_status iga_space_create(const iga_space_desc *desc, const iga_dist *dist, int device, iga_space *out) {
    return create(desc, dist, device, out);
}

iga_status iga_space_destroy(iga_space s) {
    free_space(s);
    return IGA_OK;
}

iga_status iga_space_info(iga_space s, int64_t *ndof_global, int64_t *nrows_owned, int64_t *nnz_owned,
                          int64_t *nqp_local, int64_t owned_lo[3], int64_t owned_hi[3], int64_t elem_lo[3],
                          int64_t elem_hi[3]) {
    if (!s) { set_error("null space"); return IGA_ERR_PARAM; }
    if (ndof_global) *ndof_global = s->ndof_global;
    if (nrows_owned) *nrows_owned = s->nrows_owned;
    if (nnz_owned) *nnz_owned = s->nnz_owned;
    if (nqp_local) *nqp_local = s->nqp_local;
    for (int a = 0; a < 3; a++) {
        if (owned_lo) owned_lo[a] = s->own_lo[a];
        if (owned_hi) owned_hi[a] = s->own_hi[a];
        if (elem_lo) elem_lo[a] = s->el_lo[a];
        if (elem_hi) elem_hi[a] = s->el_hi[a];
    }
    return IGA_OK;
}

iga_status iga_csr_pattern(iga_space s, int64_t *row_ptr, int32_t *col_idx, void *stream) {
    if (!s || !row_ptr || !col_idx) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (s->ndof_global > 0x7fffffffLL) { set_error("global dof count exceeds int32 column indices"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    iga_status st = launch_pattern(s, row_ptr, col_idx, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

static iga_status form_group(int n, const iga_space *spaces, const iga_phys *phys, double a, double b,
                             const double *const *U, const double *const *Ud, double *const *val, double *const *F,
                             cudaStream_t st) {
    if (n < 1 || n > 64 || !spaces || !phys || !U) { set_error("bad group arguments"); return IGA_ERR_PARAM; }
    std::vector<iga_space_s *> sp(n);
    for (int k = 0; k < n; k++) {
        sp[k] = spaces[k];
        if (!sp[k] || sp[k]->nranks != n || sp[k]->rank != k || sp[k]->device != sp[0]->device) {
            set_error("group: spaces[k] must be rank k of an n-rank decomposition on one device");
            return IGA_ERR_PARAM;
        }
        if (n > 1 && (!sp[k]->dist || dist_transport(sp[k]->dist) != IGA_XPORT_LOCAL)) {
            set_error("group forms need IGA_XPORT_LOCAL spaces");
            return IGA_ERR_STATE;
        }
    }
    std::vector<const double *> Ud0(n, nullptr);
    std::vector<double *> v0(n, nullptr), F0(n, nullptr);
    if (n == 1) return launch_form(sp[0], phys, a, b, U[0], Ud ? Ud[0] : nullptr, val ? val[0] : nullptr,
                                   F ? F[0] : nullptr, st);
    return dist_form(sp.data(), n, phys, a, b, U, Ud ? Ud : Ud0.data(), val ? val : v0.data(), F ? F : F0.data(), st);
}

iga_status iga_form_residual(iga_space s, const iga_phys *phys, const double *U, const double *Udot, double *F,
                             void *stream) {
    iga_status st = check_phys(s, phys);
    if (st != IGA_OK) return st;
    if (!U || !F) { set_error("U and F are required"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    st = form_one(s, phys, 0.0, 0.0, U, Udot, nullptr, F, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_form_jacobian(iga_space s, const iga_phys *phys, double a, double b, const double *U,
                             const double *Udot, double *csr_val, double *F, void *stream) {
    iga_status st = check_phys(s, phys);
    if (st != IGA_OK) return st;
    if (!U || !csr_val) { set_error("U and csr_val are required"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    st = form_one(s, phys, a, b, U, Udot, csr_val, F, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

// Host-buffer path, pipelined (3D, uniform axis 0): the outputs are zeroed once, the elements
// are assembled in slabs along axis 0, and the CSR rows of every node layer go back to the host
// on a second stream as soon as the last element touching that layer has been assembled (its
// slab's event), so the device-to-host copy of the values -- 33.6 GB for config 5, longer than
// the assembly itself -- runs under the assembly of the later slabs.  A layer g0's rows are one
// contiguous range of the CSR values: offset m^2 S0(g0) T1 T2, length m^2 W0(g0) T1 T2 (the
// closed-form row start, single rank).  Layer completion comes from the Alg. 1
// element -> function map (uniform: element e touches first0 + e + k, k = 0..p, mod nu), so on a
// periodic axis the first p layers (also touched by the last elements) go last.
static iga_status form_host_pipelined(iga_space_s *s, const iga_phys *phys, double a, double b, const double *dU,
                                      const double *dUd, double *dV, double *dF, double *val_h, double *F_h,
                                      cudaStream_t cs) {
    const int lo0 = s->el_lo[0], ne0 = s->el_hi[0] - lo0, nu0 = s->nu[0], p0 = s->p[0], m = s->dof;
    const int nsl = std::min(s->hb_slabs, ne0);
    const AxisDev &ax0 = s->dev.ax[0];
    std::vector<int> done(nu0, -1);                       // slab after which layer g is complete
    std::vector<int> bnd(nsl + 1);                        // slab j = elements [bnd[j], bnd[j+1])
    for (int j = 0; j <= nsl; j++) bnd[j] = (int)((long long)j * ne0 / nsl);
    for (int e = 0, sl = 0; e < ne0; e++) {
        while (e >= bnd[sl + 1]) sl++;
        for (int k = 0; k <= p0; k++) {
            int g = ax0.first0 + lo0 + e + k;
            g %= nu0;
            done[g] = std::max(done[g], sl);
        }
    }
    for (int g = 0; g < nu0; g++) if (done[g] < 0) done[g] = nsl - 1;   // (every function has support)
    long long T1 = 0, T2 = 0;
    for (int w : s->rowW[1]) T1 += w;
    for (int w : s->rowW[2]) T2 += w;
    const long long per = (long long)m * m * T1 * T2;     // values per unit of axis-0 width
    std::vector<long long> S0(nu0 + 1, 0);
    for (int g = 0; g < nu0; g++) S0[g + 1] = S0[g] + (long long)s->rowW[0][g] * per;
    cudaError_t ce = cudaSuccess;
    if (!s->hb_copy) ce = cudaStreamCreateWithFlags(&s->hb_copy, cudaStreamNonBlocking);
    while (ce == cudaSuccess && (int)s->hb_ev.size() < nsl + 1) {
        cudaEvent_t ev;
        ce = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (ce == cudaSuccess) s->hb_ev.push_back(ev);
    }
    if (ce != cudaSuccess) { set_error(std::string("host pipeline: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    k_zero_pair(dV, s->nnz_owned, dF, dF ? s->nrows_owned : 0, cs, nsm);
    int launches = 1;
    iga_status st = IGA_OK;
    for (int j = 0; j < nsl && st == IGA_OK; j++) {
        int lo[3], hi[3];
        for (int d = 0; d < 3; d++) { lo[d] = s->el_lo[d]; hi[d] = s->el_hi[d]; }
        lo[0] = lo0 + bnd[j];
        hi[0] = lo0 + bnd[j + 1];
        st = launch_form_box(s, phys, a, b, dU, dUd, dV, dF, cs, lo, hi);
        launches += s->last_launches;
        if (st != IGA_OK) break;
        ce = cudaEventRecord(s->hb_ev[j], cs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s->hb_copy, s->hb_ev[j], 0);
        for (int g = 0; g < nu0 && ce == cudaSuccess;) {     // contiguous runs of layers done after slab j
            if (done[g] != j) { g++; continue; }
            int h = g;
            while (h < nu0 && done[h] == j) h++;
            ce = cudaMemcpyAsync(val_h + S0[g], dV + S0[g], (size_t)(S0[h] - S0[g]) * sizeof(double),
                                 cudaMemcpyDeviceToHost, s->hb_copy);
            g = h;
        }
        if (ce != cudaSuccess) break;
    }
    if (st == IGA_OK && ce == cudaSuccess && F_h) {
        ce = cudaEventRecord(s->hb_ev[nsl], cs);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s->hb_copy, s->hb_ev[nsl], 0);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(F_h, dF, (size_t)s->nrows_owned * sizeof(double), cudaMemcpyDeviceToHost, s->hb_copy);
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s->hb_copy);
    s->last_launches = launches;
    if (ce != cudaSuccess) { set_error(std::string("host pipeline: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return st;
}

iga_status iga_form_jacobian_host(iga_space s, const iga_phys *phys, double a, double b, const double *U_host,
                                  const double *Udot_host, double *csr_val_host, double *F_host, void *stream) {
    iga_status st = check_phys(s, phys);
    if (st != IGA_OK) return st;
    if (!U_host || !csr_val_host) { set_error("U and csr_val are required"); return IGA_ERR_PARAM; }
    if (s->nranks > 1) { set_error("the host-buffer variant is single-rank"); return IGA_ERR_STATE; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    cudaStream_t cs = (cudaStream_t)stream;
    const size_t nU = (size_t)s->ndof_global, nF = (size_t)s->nrows_owned, nz = (size_t)s->nnz_owned;
    // device staging buffers of the host-buffer path: allocated on first use, kept by the space
    cudaError_t ce = cudaSuccess;
    if (!s->hb_U) {
        double *p4[4] = {nullptr, nullptr, nullptr, nullptr};
        const size_t sz[4] = {nU, nU, nz, nF};
        for (int k = 0; k < 4 && ce == cudaSuccess; k++) {
            ce = cudaMalloc(&p4[k], std::max<size_t>(sz[k], 1) * sizeof(double));
            if (ce == cudaSuccess) s->allocs.push_back(p4[k]);
        }
        if (ce != cudaSuccess) { cudaGetLastError(); cudaSetDevice(prev); set_error("host-path staging allocation failed"); return IGA_ERR_NOMEM; }
        s->hb_U = p4[0]; s->hb_Ud = p4[1]; s->hb_val = p4[2]; s->hb_F = p4[3];
    }
    double *dU = s->hb_U, *dUd = Udot_host ? s->hb_Ud : nullptr, *dV = s->hb_val, *dF = F_host ? s->hb_F : nullptr;
    ce = cudaMemcpyAsync(dU, U_host, nU * sizeof(double), cudaMemcpyHostToDevice, cs);
    if (ce == cudaSuccess && Udot_host) ce = cudaMemcpyAsync(dUd, Udot_host, nU * sizeof(double), cudaMemcpyHostToDevice, cs);
    const int ne0 = s->el_hi[0] - s->el_lo[0];
    const bool pipe = s->hb_slabs > 1 && s->dim == 3 && s->dev.ax[0].uniform && ne0 >= 2 * s->hb_slabs && !s->force_split;
    if (ce == cudaSuccess && pipe) {
        st = form_host_pipelined(s, phys, a, b, dU, dUd, dV, dF, csr_val_host, F_host, cs);
    } else if (ce == cudaSuccess) {
        st = launch_form(s, phys, a, b, dU, dUd, dV, dF, cs);
        const int nl = s->last_launches;
        if (st == IGA_OK) ce = cudaMemcpyAsync(csr_val_host, dV, nz * sizeof(double), cudaMemcpyDeviceToHost, cs);
        if (st == IGA_OK && ce == cudaSuccess && F_host)
            ce = cudaMemcpyAsync(F_host, dF, nF * sizeof(double), cudaMemcpyDeviceToHost, cs);
        s->last_launches = nl;
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(cs);
    cudaSetDevice(prev);
    if (ce != cudaSuccess) { set_error(cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return st;
}

iga_status iga_space_check(iga_space s, void *stream) {
    if (!s) { set_error("null space"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    int flag = 0;
    cudaError_t ce = cudaStreamSynchronize((cudaStream_t)stream);
    if (ce == cudaSuccess) ce = cudaMemcpy(&flag, s->errflag, sizeof(int), cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess) ce = cudaMemset(s->errflag, 0, sizeof(int));
    cudaSetDevice(prev);
    if (ce != cudaSuccess) { set_error(cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    if (flag & 1) { set_error("detJ <= 0 at a quadrature point"); return IGA_ERR_SINGULAR_MAP; }
    if (flag & 2) { set_error("non-finite coefficient"); return IGA_ERR_NONFINITE; }
    return IGA_OK;
}

int iga_last_launch_count(iga_space s) { return s ? s->last_launches : 0; }

iga_status iga_form_jacobian_group(int n, const iga_space *spaces, const iga_phys *phys, double a, double b,
                                   const double *const *U, const double *const *Udot, double *const *csr_val,
                                   double *const *F, void *stream) {
    if (!csr_val) { set_error("csr_val is required"); return IGA_ERR_PARAM; }
    if (n < 1 || !spaces || !spaces[0]) { set_error("bad group arguments"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(spaces[0]->device);
    iga_status st = form_group(n, spaces, phys, a, b, U, Udot, csr_val, F, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_form_residual_group(int n, const iga_space *spaces, const iga_phys *phys, const double *const *U,
                                   const double *const *Udot, double *const *F, void *stream) {
    if (!F) { set_error("F is required"); return IGA_ERR_PARAM; }
    if (n < 1 || !spaces || !spaces[0]) { set_error("bad group arguments"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(spaces[0]->device);
    iga_status st = form_group(n, spaces, phys, 0.0, 0.0, U, Udot, nullptr, F, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_dist_plan(const iga_space_desc *desc, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                         int64_t el_lo[3], int64_t el_hi[3], int64_t ext_n[3], int max_msgs, iga_msg *send, int *nsend,
                         iga_msg *recv, int *nrecv) {
    return dist_plan_host(desc, dist, own_lo, own_hi, el_lo, el_hi, ext_n, max_msgs, send, nsend, recv, nrecv);
}

iga_status iga_krylov_plan(const iga_space_desc *desc, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                           int64_t ext_n[3], int64_t ghost[3], int max_msgs, iga_msg *send, int *nsend, iga_msg *recv,
                           int *nrecv) {
    return krylov_plan_host(desc, dist, own_lo, own_hi, ext_n, ghost, max_msgs, send, nsend, recv, nrecv);
}

iga_status iga_basis_eval(iga_space s, int order, double *out, void *stream) {
    if (!s || !out) { set_error("null argument"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    iga_status st = launch_basis3(s, order, out, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_gmres(iga_space s, const int64_t *row_ptr, const int32_t *col_idx, const double *val, const double *b,
                     double *x, const iga_krylov *opt, int *iters, double *relres, void *stream) {
    if (!s || !row_ptr || !col_idx || !val || !b || !x || !opt) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (opt->precond < 0 || opt->precond > 2 || opt->restart < 1 || opt->maxit < 0 || !(opt->rtol >= 0.0)) {
        set_error("gmres: bad options");
        return IGA_ERR_PARAM;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    iga_status st = gmres_solve(s, row_ptr, col_idx, val, b, x, opt, iters, relres, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_gmres_group(int n, const iga_space *spaces, const int64_t *const *row_ptr, const int32_t *const *col_idx,
                           const double *const *val, const double *const *b, double *const *x, const iga_krylov *opt,
                           int *iters, double *relres, void *stream) {
    if (n < 1 || n > 64 || !spaces || !row_ptr || !col_idx || !val || !b || !x || !opt) {
        set_error("bad group arguments");
        return IGA_ERR_PARAM;
    }
    if (opt->precond < 0 || opt->precond > 2 || opt->restart < 1 || opt->maxit < 0) { set_error("gmres: bad options"); return IGA_ERR_PARAM; }
    std::vector<iga_space_s *> sp(n);
    for (int k = 0; k < n; k++) {
        sp[k] = spaces[k];
        if (!sp[k] || sp[k]->nranks != n || sp[k]->rank != k || sp[k]->device != sp[0]->device) {
            set_error("group: spaces[k] must be rank k of an n-rank decomposition on one device");
            return IGA_ERR_PARAM;
        }
        if (n > 1 && (!sp[k]->dist || dist_transport(sp[k]->dist) != IGA_XPORT_LOCAL)) {
            set_error("group solves need IGA_XPORT_LOCAL spaces");
            return IGA_ERR_STATE;
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(sp[0]->device);
    iga_status st = gmres_group(n, sp.data(), row_ptr, col_idx, val, b, x, opt, iters, relres, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_alpha_step_group(int n, const iga_space *spaces, const iga_phys *phys, const iga_alpha *opt,
                                const int64_t *const *row_ptr, const int32_t *const *col_idx, double *const *val,
                                double *const *U, double *const *Udot, iga_step_stats *stats, void *stream) {
    if (n < 1 || n > 64 || !spaces || !opt || !row_ptr || !col_idx || !val || !U || !Udot) { set_error("bad group arguments"); return IGA_ERR_PARAM; }
    iga_status st = check_phys(spaces[0], phys);
    if (st != IGA_OK) return st;
    if (opt->newton_its < 1 || opt->newton_its > 8 || !(opt->dt > 0.0) || !(opt->rho_inf >= 0.0 && opt->rho_inf <= 1.0) ||
        opt->krylov.precond < 0 || opt->krylov.precond > 2 || opt->krylov.restart < 1 || opt->krylov.maxit < 0) {
        set_error("alpha_step: bad options");
        return IGA_ERR_PARAM;
    }
    std::vector<iga_space_s *> sp(n);
    for (int k = 0; k < n; k++) {
        sp[k] = spaces[k];
        if (!sp[k] || sp[k]->nranks != n || sp[k]->rank != k || sp[k]->device != sp[0]->device) {
            set_error("group: spaces[k] must be rank k of an n-rank decomposition on one device");
            return IGA_ERR_PARAM;
        }
        if (n > 1 && (!sp[k]->dist || dist_transport(sp[k]->dist) != IGA_XPORT_LOCAL)) {
            set_error("group steps need IGA_XPORT_LOCAL spaces");
            return IGA_ERR_STATE;
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(sp[0]->device);
    st = alpha_step_group(n, sp.data(), phys, opt, row_ptr, col_idx, val, U, Udot, stats, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_alpha_step(iga_space s, const iga_phys *phys, const iga_alpha *opt, const int64_t *row_ptr,
                          const int32_t *col_idx, double *val, double *U, double *Udot, iga_step_stats *stats,
                          void *stream) {
    iga_status st = check_phys(s, phys);
    if (st != IGA_OK) return st;
    if (!opt || !row_ptr || !col_idx || !val || !U || !Udot) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (opt->newton_its < 1 || opt->newton_its > 8 || !(opt->dt > 0.0) || !(opt->rho_inf >= 0.0 && opt->rho_inf <= 1.0) ||
        opt->krylov.precond < 0 || opt->krylov.precond > 2 || opt->krylov.restart < 1 || opt->krylov.maxit < 0) {
        set_error("alpha_step: bad options");
        return IGA_ERR_PARAM;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    st = alpha_step(s, phys, opt, row_ptr, col_idx, val, U, Udot, stats, (cudaStream_t)stream);
    cudaSetDevice(prev);
    return st;
}

iga_status iga_nccl_unique_id(unsigned char out[128]) {
    if (!out) { set_error("null argument"); return IGA_ERR_PARAM; }
    return nccl_unique_id(out);
}

iga_status iga_space_set_option(iga_space s, const char *key, long long value) {
    if (!s || !key) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (std::strcmp(key, "split") == 0) { s->force_split = value != 0; return IGA_OK; }
    if (std::strcmp(key, "general") == 0) { s->force_general = value != 0; return IGA_OK; }
    if (std::strcmp(key, "dbg") == 0) { s->dbg = (int)value; return IGA_OK; }
    if (std::strcmp(key, "bw") == 0) { s->bw_opt = (int)value; return IGA_OK; }
    if (std::strcmp(key, "hb_slabs") == 0) { s->hb_slabs = (int)std::max<long long>(0, value); return IGA_OK; }
    if (std::strcmp(key, "gmres_host") == 0) { s->gm_host_ctrl = value != 0; return IGA_OK; }
    set_error(std::string("unknown option ") + key);
    return IGA_ERR_PARAM;
}

iga_status iga_profile_enable(iga_space s, int on) {
    if (!s) { set_error("null space"); return IGA_ERR_PARAM; }
    s->prof_on = on != 0;
    return IGA_OK;
}

iga_status iga_profile_reset(iga_space s) {
    if (!s) { set_error("null space"); return IGA_ERR_PARAM; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    prof_collect(s);
    s->prof_names.clear();
    s->prof_count.clear();
    s->prof_ms.clear();
    cudaSetDevice(prev);
    return IGA_OK;
}

int iga_profile_read(iga_space s, int max, char *names, int *launches, double *ms) {
    if (!s) { set_error("null space"); return -1; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    prof_collect(s);
    cudaSetDevice(prev);
    const int n = (int)s->prof_names.size();
    for (int k = 0; k < n && k < max; k++) {
        if (names) {
            std::strncpy(names + 32 * k, s->prof_names[k].c_str(), 31);
            names[32 * k + 31] = 0;
        }
        if (launches) launches[k] = s->prof_count[k];
        if (ms) ms[k] = s->prof_ms[k];
    }
    return n;
}

}  // extern "C"
