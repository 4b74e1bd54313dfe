/*
 * oracle/oracle.c -- the CPU ORACLE for Galerkin residual / Jacobian assembly on
 * tensor-product B-spline / NURBS spaces (arXiv:1305.4452, "PetIGA").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1305_4452_b200/, include/iga.h) never links, imports or calls it, and this
 * file includes nothing from there: the two share no code, headers or tables.
 *
 * Plain, slow, obviously-correct fp64 C.  Every function cites the passage of
 * /root/reference/PAPER.md ("P:line", section / equation / algorithm) it follows;
 * where the paper is silent the SURVEY.md §8(c) reading (A-n) is cited and repeated
 * in DESIGN.md.  There is no blocking, fusion or reordering beyond the definitions:
 *   - periodic spaces: Alg. 1 on the knots; geometry on a periodic axis is
 *     given as a clamped net and unclamped with Alg. 2,
 *   - univariate basis: the literal Cox-de Boor recursion of P:184-190 (not the
 *     triangular in-span scheme), derivatives by the textbook recursion (A5),
 *   - tensor product P:196-203, rational basis eqs. (rational),(drational),(ddrational)
 *     P:211, isoparametric map P:268-278, inverse map (derividentity)
 *     P:292 as a matrix inverse (A-5), inverse-map second derivative P:316-327,
 *     push-forward (dspatial),(ddspatial) P:309-310,
 *   - integrands per SURVEY Appendix A, each Jacobian entry as the literal
 *     linearisation of the residual at that quadrature point,
 *   - element integration per Alg. 4: F_e += F_q J_q w_q, dense K_e,
 *   - assembly "dense-then-CSR": a dense global matrix (tiny spaces) or complete rows
 *     of a row subset scattered by binary search into the Alg. 3 pattern,
 *     with every touched entry required to lie in that pattern.
 *
 * Readings without a paper value: the Cahn-Hilliard mobility and chemical potential (A-10) and
 * the VMS stabilisation (A-14).  They are pinned to values computed independently of this file
 * (SURVEY Appendices A and C: G, tau_M, tau_C at config 5; M, mu' and the term-group diagonal
 * magnitudes at config 3) by tests/test_oracle_state_pins.py, which also shows that seeded
 * mutations of these formulas fail the pins; the weak forms around them are pinned to the
 * paper's strong forms (test_oracle_ch_strong.py, test_oracle_vms_consistency.py, and the NSK
 * strong-form test in test_oracle_nsk.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXD 3
#define ORC_MAXP 4
#define ORC_MAXEN 125 /* (ORC_MAXP+1)^3 */
#define ORC_MAXM 4

enum { ORC_LAPLACE = 0, ORC_CAHN_HILLIARD = 1, ORC_NEOHOOKE = 2, ORC_NS_VMS = 3, ORC_NSK = 4 };
enum { ORC_PARAMETRIC = 0, ORC_NURBS = 1 };

/* ------------------------------------------------------------------------------------ */
/* Alg. 1: unclamp a knot vector for C^k periodicity, in place.              */
/* U has m+1 = n+p+2 entries (n+1 basis functions).                                      */
/* ------------------------------------------------------------------------------------ */
void orc_unclamp_knots(int n, int p, int k, double *U)
{
    int m = n + p + 1;
    for (int i = 0; i <= k; i++) {
        U[k - i] = U[p] - U[n + 1] + U[n - i];
        U[m - k + i] = U[n + 1] - U[p] + U[p + i + 1];
    }
}

/* ------------------------------------------------------------------------------------ */
/* Alg. 2 ("UnclampCurve"): unclamp the knot vector U and the n+1 homogeneous  */
/* control points of a curve for C^k periodicity, in place, in the paper's loop order.   */
/* Point j is Pw[j*stride .. j*stride+h-1] (h = dim+1 homogeneous coordinates).  The     */
/* pseudocode's stray '}' after the first double loop is a garble; the structure is two  */
/* (knots, points) passes, left end then right end (the NURBS book's A12.1 shape).        */
/* ------------------------------------------------------------------------------------ */
void orc_unclamp_curve(int n, int p, int k, double *U, double *Pw, int h, long stride)
{
    int m = n + p + 1;
    for (int i = 0; i <= k; i++) /* unclamp at left end */
        U[k - i] = U[p] - U[n + 1] + U[n - i];
    for (int i = p - k - 1; i <= p - 2; i++)
        for (int j = i; j >= 0; j--) {
            double alpha = (U[p] - U[p + j - i - 1]) / (U[p + j + 1] - U[p + j - i - 1]);
            for (int c = 0; c < h; c++)
                Pw[j * stride + c] = (Pw[j * stride + c] - alpha * Pw[(j + 1) * stride + c]) / (1.0 - alpha);
        }
    for (int i = 0; i <= k; i++) /* unclamp at right end */
        U[m - k + i] = U[n + 1] - U[p] + U[p + i + 1];
    for (int i = p - k - 1; i <= p - 2; i++)
        for (int j = i; j >= 0; j--) {
            double alpha = (U[n + 1] - U[n - j]) / (U[n - j + i + 2] - U[n - j]);
            for (int c = 0; c < h; c++)
                Pw[(n - j) * stride + c] = (Pw[(n - j) * stride + c] - (1.0 - alpha) * Pw[(n - j - 1) * stride + c]) / alpha;
        }
}

/* ------------------------------------------------------------------------------------ */
/* Alg. 3: leftmost / rightmost basis indices interacting with basis i.      */
/* nk = number of knots (bounds guard only; the paper's loops assume it).                */
/* ------------------------------------------------------------------------------------ */
void orc_basis_stencil(int i, int p, const double *U, int nk, int *l, int *r)
{
    int k = i;
    while (k + 1 < nk && U[k] == U[k + 1]) k++;
    *l = k - p;
    k = i + p + 1;
    while (k - 1 >= 0 && U[k] == U[k - 1]) k--;
    *r = k - 1;
}

/* ------------------------------------------------------------------------------------ */
/* Cox-de Boor recursion, literal; 0/0 := 0 (reading A-1).                    */
/* ------------------------------------------------------------------------------------ */
double orc_coxdeboor(int i, int p, const double *U, double xi)
{
    if (p == 0) return (U[i] <= xi && xi < U[i + 1]) ? 1.0 : 0.0;
    double left = 0.0, right = 0.0;
    double d1 = U[i + p] - U[i];
    double d2 = U[i + p + 1] - U[i + 1];
    if (d1 != 0.0) left = (xi - U[i]) / d1 * orc_coxdeboor(i, p - 1, U, xi);
    if (d2 != 0.0) right = (U[i + p + 1] - xi) / d2 * orc_coxdeboor(i + 1, p - 1, U, xi);
    return left + right;
}

/* k-th derivative: the textbook derivative of the recursion (A5, implied by P:218-224):
 *   N^{(k)}_{i,p} = p/(U_{i+p}-U_i) N^{(k-1)}_{i,p-1} - p/(U_{i+p+1}-U_{i+1}) N^{(k-1)}_{i+1,p-1} */
double orc_coxdeboor_deriv(int i, int p, const double *U, double xi, int k)
{
    if (k == 0) return orc_coxdeboor(i, p, U, xi);
    if (p == 0) return 0.0;
    double left = 0.0, right = 0.0;
    double d1 = U[i + p] - U[i];
    double d2 = U[i + p + 1] - U[i + 1];
    if (d1 != 0.0) left = p / d1 * orc_coxdeboor_deriv(i, p - 1, U, xi, k - 1);
    if (d2 != 0.0) right = p / d2 * orc_coxdeboor_deriv(i + 1, p - 1, U, xi, k - 1);
    return left - right;
}

/* ------------------------------------------------------------------------------------ */
/* Gauss-Legendre rule on [-1,1] (Alg. 4 "Quadrature(q)"; rule unstated -> A-6).  */
/* Newton on P_n in long double from cosine guesses; w = 2/((1-x^2) P_n'(x)^2).          */
/* Nodes ascending.                                                                       */
/* ------------------------------------------------------------------------------------ */
void orc_gauss_legendre(int n, double *x, double *w)
{
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int i = 0; i < n; i++) {
        long double z = cosl(pi * (i + 0.75L) / (n + 0.5L));
        long double dp = 1.0L;
        for (int it = 0; it < 200; it++) {
            long double p0 = 1.0L, p1 = z;
            for (int j = 2; j <= n; j++) {
                long double p2 = ((2.0L * j - 1.0L) * z * p1 - (j - 1.0L) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = (n == 1) ? 1.0L : n * (z * p1 - p0) / (z * z - 1.0L);
            long double dz = p1 / dp;
            z -= dz;
            if (fabsl(dz) < 1e-30L) break;
        }
        {   /* derivative at the converged root */
            long double p0 = 1.0L, p1 = z;
            for (int j = 2; j <= n; j++) {
                long double p2 = ((2.0L * j - 1.0L) * z * p1 - (j - 1.0L) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = (n == 1) ? 1.0L : n * (z * p1 - p0) / (z * z - 1.0L);
        }
        x[n - 1 - i] = (double)z;
        w[n - 1 - i] = (double)(2.0L / ((1.0L - z * z) * dp * dp));
    }
}

/* ------------------------------------------------------------------------------------ */
/* The space: one NURBS patch, elements = nonzero knot spans.     */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int dim, dof, geom;
    int p[ORC_MAXD], nk[ORC_MAXD];
    double *U[ORC_MAXD];            /* knot vectors (unclamped by Alg. 1 when periodic) */
    int periodic[ORC_MAXD], cont[ORC_MAXD];
    int nfun[ORC_MAXD];             /* functions in the (unwrapped) knot vector          */
    int nu[ORC_MAXD];               /* unique (global) functions; i -> i mod nu (A-8)    */
    int nel[ORC_MAXD];
    int *span[ORC_MAXD];            /* element -> span index                             */
    int nq[ORC_MAXD];
    double gx[ORC_MAXD][16], gw[ORC_MAXD][16];
    int64_t nnodes;
    double *ctrl;                   /* [nnodes][dim] Euclidean, NURBS only               */
    double *wts;                    /* [nnodes] or NULL (=1)                             */
    /* per axis: columns of each global function (Alg. 3, wrapped, sorted, unique) */
    int *colcnt[ORC_MAXD];
    int *cols[ORC_MAXD];            /* [nu][colmax] */
    int colmax[ORC_MAXD];
} orc_space;

static int cmp_int(const void *a, const void *b)
{
    int x = *(const int *)a, y = *(const int *)b;
    return (x > y) - (x < y);
}

void orc_space_free(orc_space *s)
{
    if (!s) return;
    for (int d = 0; d < ORC_MAXD; d++) {
        free(s->U[d]);
        free(s->span[d]);
        free(s->colcnt[d]);
        free(s->cols[d]);
    }
    free(s->ctrl);
    free(s->wts);
    free(s);
}

/* knots: concatenated open knot vectors; nk[d] knots on axis d. Returns NULL on bad input. */
orc_space *orc_space_new(int dim, const int *p, const int *nk, const double *knots,
                         const int *periodic, const int *cont, int dof, const int *quad,
                         int geom, const double *ctrl, const double *wts)
{
    if (dim < 1 || dim > 3 || dof < 1 || dof > ORC_MAXM) return NULL;
    orc_space *s = (orc_space *)calloc(1, sizeof(orc_space));
    s->dim = dim;
    s->dof = dof;
    s->geom = geom;
    const double *kp = knots;
    s->nnodes = 1;
    for (int d = 0; d < dim; d++) {
        s->p[d] = p[d];
        s->nk[d] = nk[d];
        if (p[d] < 1 || p[d] > ORC_MAXP) { orc_space_free(s); return NULL; }
        s->U[d] = (double *)malloc(sizeof(double) * nk[d]);
        memcpy(s->U[d], kp, sizeof(double) * nk[d]);
        kp += nk[d];
        s->nfun[d] = nk[d] - p[d] - 1;
        s->periodic[d] = periodic ? periodic[d] : 0;
        s->cont[d] = cont ? cont[d] : p[d] - 1;
        if (s->periodic[d]) {
            /* Alg. 1 with n+1 = nfun functions */
            orc_unclamp_knots(s->nfun[d] - 1, p[d], s->cont[d], s->U[d]);
            s->nu[d] = s->nfun[d] - (s->cont[d] + 1);
        } else {
            s->nu[d] = s->nfun[d];
        }
        /* elements: nonzero spans inside [U_p, U_nfun] */
        s->span[d] = (int *)malloc(sizeof(int) * nk[d]);
        s->nel[d] = 0;
        for (int sp = p[d]; sp < s->nfun[d]; sp++)
            if (s->U[d][sp] < s->U[d][sp + 1]) s->span[d][s->nel[d]++] = sp;
        s->nq[d] = (quad && quad[d] > 0) ? quad[d] : p[d] + 1;
        if (s->nq[d] > 16) { orc_space_free(s); return NULL; }
        orc_gauss_legendre(s->nq[d], s->gx[d], s->gw[d]);
        s->nnodes *= s->nu[d];

        /* per-axis pattern from Alg. 3 on every representative i of each global g (A-8) */
        int nu = s->nu[d];
        int cap = 0;
        int *tl = (int *)malloc(sizeof(int) * s->nfun[d]);
        int *tr = (int *)malloc(sizeof(int) * s->nfun[d]);
        for (int i = 0; i < s->nfun[d]; i++) {
            orc_basis_stencil(i, p[d], s->U[d], nk[d], &tl[i], &tr[i]);
            if (tr[i] - tl[i] + 1 > cap) cap = tr[i] - tl[i] + 1;
        }
        cap *= (s->nfun[d] + nu - 1) / nu; /* representatives per g */
        s->colmax[d] = cap;
        s->colcnt[d] = (int *)calloc(nu, sizeof(int));
        s->cols[d] = (int *)malloc(sizeof(int) * (size_t)nu * cap);
        for (int g = 0; g < nu; g++) {
            int *c = s->cols[d] + (size_t)g * cap;
            int cnt = 0;
            for (int i = g; i < s->nfun[d]; i += nu)
                for (int j = tl[i]; j <= tr[i]; j++) c[cnt++] = ((j % nu) + nu) % nu;
            qsort(c, cnt, sizeof(int), cmp_int);
            int u = 0;
            for (int t = 0; t < cnt; t++)
                if (u == 0 || c[u - 1] != c[t]) c[u++] = c[t];
            s->colcnt[d][g] = u;
        }
        free(tl);
        free(tr);
    }
    for (int d = dim; d < ORC_MAXD; d++) {
        s->p[d] = 0; s->nfun[d] = 1; s->nu[d] = 1; s->nel[d] = 1; s->nq[d] = 1;
        s->gx[d][0] = 0.0; s->gw[d][0] = 1.0;
        s->span[d] = (int *)calloc(1, sizeof(int));
        s->colcnt[d] = (int *)calloc(1, sizeof(int)); s->colcnt[d][0] = 1;
        s->cols[d] = (int *)calloc(1, sizeof(int)); s->colmax[d] = 1;
    }
    if (geom == ORC_NURBS && !ctrl) { orc_space_free(s); return NULL; }
    if (ctrl || wts) {
        /* geometry data is given on the OPEN function grid (nfun per axis).  On periodic axes the
         * clamped net is unclamped with Alg. 2 in homogeneous coordinates (w x, w), line by line,
         * and the last k+1 points -- the wrapped copies of the first k+1 on a C^k-periodic
         * geometry -- must coincide with them (else the description is invalid); the unique
         * nu points are kept. */
        int h = dim + 1;
        long nopen = 1;
        for (int d = 0; d < dim; d++) nopen *= s->nfun[d];
        double *Pw = (double *)malloc(sizeof(double) * nopen * h);
        for (long q = 0; q < nopen; q++) {
            double wq = wts ? wts[q] : 1.0;
            for (int c = 0; c < dim; c++) Pw[q * h + c] = (ctrl ? ctrl[q * dim + c] : 0.0) * wq;
            Pw[q * h + dim] = wq;
        }
        long str[ORC_MAXD];
        long acc = h;
        for (int d = dim - 1; d >= 0; d--) { str[d] = acc; acc *= s->nfun[d]; }
        int bad = 0;
        const double *kq = knots;
        for (int d = 0; d < dim; d++) {
            if (s->periodic[d]) {
                int nf = s->nfun[d], k = s->cont[d];
                double *Uc = (double *)malloc(sizeof(double) * nk[d]);
                for (long q = 0; q < nopen; q++) {
                    long coord = (q / (str[d] / h)) % nf;
                    if (coord != 0) continue;             /* one line per base point */
                    memcpy(Uc, kq, sizeof(double) * nk[d]);
                    orc_unclamp_curve(nf - 1, p[d], k, Uc, Pw + q * h, h, str[d]);
                    for (int g = 0; g <= k; g++)
                        for (int c = 0; c < h; c++) {
                            double a0 = Pw[q * h + g * str[d] + c], a1 = Pw[q * h + (s->nu[d] + g) * str[d] + c];
                            if (fabs(a0 - a1) > 1e-10 * (1.0 + fabs(a0))) bad = 1;
                        }
                }
                free(Uc);
            }
            kq += nk[d];
        }
        if (bad) { free(Pw); orc_space_free(s); return NULL; }
        if (ctrl) s->ctrl = (double *)malloc(sizeof(double) * s->nnodes * dim);
        if (wts) s->wts = (double *)malloc(sizeof(double) * s->nnodes);
        for (long u = 0; u < s->nnodes; u++) {
            /* unique node u (C order over nu) -> open-grid index */
            long rem = u, q = 0;
            long ui[ORC_MAXD];
            for (int d = dim - 1; d >= 0; d--) { ui[d] = rem % s->nu[d]; rem /= s->nu[d]; }
            for (int d = 0; d < dim; d++) q = q * s->nfun[d] + ui[d];
            double wq = Pw[q * h + dim];
            if (ctrl) for (int c = 0; c < dim; c++) s->ctrl[u * dim + c] = Pw[q * h + c] / wq;
            if (wts) s->wts[u] = wq;
        }
        free(Pw);
    }
    return s;
}

int64_t orc_ndof(const orc_space *s) { return s->nnodes * s->dof; }

void orc_space_info(const orc_space *s, int *nu, int *nel, int *nq, int *nfun)
{
    for (int d = 0; d < ORC_MAXD; d++) {
        nu[d] = s->nu[d]; nel[d] = s->nel[d]; nq[d] = s->nq[d]; nfun[d] = s->nfun[d];
    }
}

/* unclamped knot vector of axis d (for tests) */
void orc_space_knots(const orc_space *s, int d, double *out)
{
    memcpy(out, s->U[d], sizeof(double) * s->nk[d]);
}

/* ------------------------------------------------------------------------------------ */
/* Pattern rows: Alg. 3 per axis x tensor product x dof blocks; sorted.       */
/* rowlen[r] always written; cols (if non-NULL) gets the concatenated rows.              */
/* ------------------------------------------------------------------------------------ */
static void node_to_ijk(const orc_space *s, int64_t node, int g[3])
{
    g[2] = (int)(node % s->nu[2]); node /= s->nu[2];
    g[1] = (int)(node % s->nu[1]); node /= s->nu[1];
    g[0] = (int)node;
}

int64_t orc_pattern_rows(const orc_space *s, int64_t nrows, const int64_t *rows,
                         int64_t *rowlen, int32_t *cols)
{
    int64_t total = 0;
    int m = s->dof;
    for (int64_t t = 0; t < nrows; t++) {
        int64_t node = rows[t] / m;
        int g[3];
        node_to_ijk(s, node, g);
        int n0 = s->colcnt[0][g[0]], n1 = s->colcnt[1][g[1]], n2 = s->colcnt[2][g[2]];
        const int *c0 = s->cols[0] + (size_t)g[0] * s->colmax[0];
        const int *c1 = s->cols[1] + (size_t)g[1] * s->colmax[1];
        const int *c2 = s->cols[2] + (size_t)g[2] * s->colmax[2];
        int64_t len = (int64_t)n0 * n1 * n2 * m;
        rowlen[t] = len;
        if (cols) {
            int32_t *o = cols + total;
            for (int a = 0; a < n0; a++)
                for (int b = 0; b < n1; b++)
                    for (int c = 0; c < n2; c++) {
                        int64_t cn = ((int64_t)c0[a] * s->nu[1] + c1[b]) * s->nu[2] + c2[c];
                        for (int j = 0; j < m; j++) *o++ = (int32_t)(cn * m + j);
                    }
        }
        total += len;
    }
    return total;
}

/* ------------------------------------------------------------------------------------ */
/* Quadrature-point evaluation: Basis(G_e, x_q) of Alg. 4.                        */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int nen;
    int64_t node[ORC_MAXEN];              /* global node of local function A            */
    double R[ORC_MAXEN];                  /* R_A                                        */
    double dR[ORC_MAXEN][3];              /* R_{A,i}  spatial (dspatial)                */
    double ddR[ORC_MAXEN][3][3];          /* R_{A,ij} spatial (ddspatial)               */
    double x[3];                          /* physical point                            */
    double detJ, dV;                      /* detJ and detJ * w_q                       */
    double dxi_dx[3][3];                  /* xi_{alpha,i}                              */
    double hpar[3];                       /* parametric element lengths                */
} orc_qp;

/* 3x3 (or dim x dim) inverse by cofactors (A-5: matrix inverse of x_{i,alpha}); returns det */
static double inverse(int dim, double A[3][3], double Ai[3][3])
{
    double det;
    if (dim == 1) {
        det = A[0][0];
        Ai[0][0] = 1.0 / det;
    } else if (dim == 2) {
        det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
        Ai[0][0] = A[1][1] / det;
        Ai[0][1] = -A[0][1] / det;
        Ai[1][0] = -A[1][0] / det;
        Ai[1][1] = A[0][0] / det;
    } else {
        det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1])
            - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0])
            + A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
        Ai[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / det;
        Ai[0][1] = -(A[0][1] * A[2][2] - A[0][2] * A[2][1]) / det;
        Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
        Ai[1][0] = -(A[1][0] * A[2][2] - A[1][2] * A[2][0]) / det;
        Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
        Ai[1][2] = -(A[0][0] * A[1][2] - A[0][2] * A[1][0]) / det;
        Ai[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / det;
        Ai[2][1] = -(A[0][0] * A[2][1] - A[0][1] * A[2][0]) / det;
        Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    }
    return det;
}

/* Evaluate the basis at the parametric point xi[] inside element (e0,e1,e2).
 * wq = the product of the (mapped) quadrature weights, or 1 for a plain point evaluation. */
static int eval_point(const orc_space *s, const int e[3], const double xi[3], double wq, orc_qp *Q)
{
    int dim = s->dim;
    /* univariate N, N', N'' of the p+1 functions of each span (literal recursion) */
    double Nv[3][ORC_MAXP + 1][3];
    int first[3];
    for (int d = 0; d < 3; d++) {
        if (d >= dim) { Nv[d][0][0] = 1.0; Nv[d][0][1] = 0.0; Nv[d][0][2] = 0.0; first[d] = 0; continue; }
        int sp = s->span[d][e[d]];
        first[d] = sp - s->p[d];
        for (int a = 0; a <= s->p[d]; a++)
            for (int k = 0; k < 3; k++)
                Nv[d][a][k] = orc_coxdeboor_deriv(first[d] + a, s->p[d], s->U[d], xi[d], k);
        Q->hpar[d] = s->U[d][sp + 1] - s->U[d][sp];
    }
    int n1 = s->p[1] + 1, n2 = s->p[2] + 1, n0 = s->p[0] + 1;
    if (dim < 2) n1 = 1;
    if (dim < 3) n2 = 1;
    Q->nen = n0 * n1 * n2;
    /* tensor product M_A, M_{A,alpha}, M_{A,alpha beta}, A = (a0*n1+a1)*n2+a2 */
    static __thread double M[ORC_MAXEN], dM[ORC_MAXEN][3], ddM[ORC_MAXEN][3][3], wA[ORC_MAXEN];
    for (int a0 = 0; a0 < n0; a0++)
        for (int a1 = 0; a1 < n1; a1++)
            for (int a2 = 0; a2 < n2; a2++) {
                int A = (a0 * n1 + a1) * n2 + a2;
                int aa[3] = {a0, a1, a2};
                int g[3];
                for (int d = 0; d < 3; d++) g[d] = (first[d] + aa[d]) % s->nu[d];
                Q->node[A] = ((int64_t)g[0] * s->nu[1] + g[1]) * s->nu[2] + g[2];
                M[A] = Nv[0][a0][0] * Nv[1][a1][0] * Nv[2][a2][0];
                for (int al = 0; al < 3; al++) {
                    double v = 1.0;
                    for (int d = 0; d < 3; d++) v *= Nv[d][aa[d]][d == al ? 1 : 0];
                    dM[A][al] = v;
                    for (int be = 0; be < 3; be++) {
                        double u = 1.0;
                        for (int d = 0; d < 3; d++) {
                            int k = (d == al) + (d == be);
                            u *= Nv[d][aa[d]][k];
                        }
                        ddM[A][al][be] = u;
                    }
                }
                wA[A] = s->wts ? s->wts[Q->node[A]] : 1.0;
            }
    /* rational basis: w, w_{,alpha}, w_{,alpha beta}, eqs. (rational) P:211,
     * (drational) P:234, (ddrational) P:245 */
    double w = 0.0, dw[3] = {0, 0, 0}, ddw[3][3] = {{0}};
    for (int A = 0; A < Q->nen; A++) {
        w += wA[A] * M[A];
        for (int al = 0; al < 3; al++) {
            dw[al] += wA[A] * dM[A][al];
            for (int be = 0; be < 3; be++) ddw[al][be] += wA[A] * ddM[A][al][be];
        }
    }
    static __thread double Rp[ORC_MAXEN][3], Rpp[ORC_MAXEN][3][3];
    for (int A = 0; A < Q->nen; A++) {
        Q->R[A] = wA[A] * M[A] / w;
        for (int al = 0; al < dim; al++) Rp[A][al] = (wA[A] * dM[A][al] - Q->R[A] * dw[al]) / w;
        for (int al = 0; al < dim; al++)
            for (int be = 0; be < dim; be++)
                Rpp[A][al][be] = (wA[A] * ddM[A][al][be] - Q->R[A] * ddw[al][be]
                                  - Rp[A][be] * dw[al] - Rp[A][al] * dw[be]) / w;
    }
    /* isoparametric map x = sum x_B R_B, x_{i,alpha}, x_{i,alpha beta} */
    double X[3] = {0, 0, 0}, Xa[3][3] = {{0}}, Xab[3][3][3] = {{{0}}};
    if (s->geom == ORC_NURBS) {
        for (int B = 0; B < Q->nen; B++)
            for (int i = 0; i < dim; i++) {
                double xb = s->ctrl[Q->node[B] * dim + i];
                X[i] += xb * Q->R[B];
                for (int al = 0; al < dim; al++) {
                    Xa[i][al] += xb * Rp[B][al];
                    for (int be = 0; be < dim; be++) Xab[i][al][be] += xb * Rpp[B][al][be];
                }
            }
    } else {
        for (int i = 0; i < dim; i++) {   /* parametric: x = xi */
            X[i] = xi[i];
            Xa[i][i] = 1.0;
        }
    }
    /* inverse map xi_{alpha,i} = (x_{i,alpha})^{-1} (identity P:287, derividentity P:292, A-5) */
    double Xi[3][3] = {{0}};
    double det = inverse(dim, Xa, Xi);
    if (!(det > 0.0)) return -1; /* A-7: orientation with detJ > 0 asserted */
    /* xi_{nu,n l} = - x_{m,eps mu} xi_{eps,n} xi_{mu,l} xi_{nu,m} */
    double Xi2[3][3][3] = {{{0}}};
    for (int nu_ = 0; nu_ < dim; nu_++)
        for (int n = 0; n < dim; n++)
            for (int l = 0; l < dim; l++) {
                double v = 0.0;
                for (int m = 0; m < dim; m++)
                    for (int ep = 0; ep < dim; ep++)
                        for (int mu = 0; mu < dim; mu++)
                            v -= Xab[m][ep][mu] * Xi[ep][n] * Xi[mu][l] * Xi[nu_][m];
                Xi2[nu_][n][l] = v;
            }
    /* push-forward: (dspatial) P:309, (ddspatial) P:310 */
    for (int A = 0; A < Q->nen; A++) {
        for (int i = 0; i < 3; i++) {
            Q->dR[A][i] = 0.0;
            for (int j = 0; j < 3; j++) Q->ddR[A][i][j] = 0.0;
        }
        for (int i = 0; i < dim; i++) {
            double v = 0.0;
            for (int al = 0; al < dim; al++) v += Rp[A][al] * Xi[al][i];
            Q->dR[A][i] = v;
            for (int j = 0; j < dim; j++) {
                double u = 0.0;
                for (int al = 0; al < dim; al++)
                    for (int be = 0; be < dim; be++) u += Rpp[A][al][be] * Xi[al][i] * Xi[be][j];
                for (int al = 0; al < dim; al++) u += Rp[A][al] * Xi2[al][i][j];
                Q->ddR[A][i][j] = u;
            }
        }
    }
    for (int i = 0; i < 3; i++) {
        Q->x[i] = X[i];
        for (int j = 0; j < 3; j++) Q->dxi_dx[i][j] = (i < dim && j < dim) ? Xi[i][j] : 0.0;
    }
    Q->detJ = det;
    Q->dV = det * wq;
    return 0;
}

/* Public point evaluation for tests: element e[], parametric point xi[].  Outputs per local
 * function A (nen of them): R, dR[3], ddR[9], node; and x[3], detJ. Returns nen or <0. */
int orc_eval_point(const orc_space *s, const int *e, const double *xi, double *R, double *dR,
                   double *ddR, int64_t *node, double *x, double *detJ)
{
    orc_qp Q;
    int ee[3] = {0, 0, 0};
    double xx[3] = {0, 0, 0};
    for (int d = 0; d < s->dim; d++) { ee[d] = e[d]; xx[d] = xi[d]; }
    if (eval_point(s, ee, xx, 1.0, &Q) < 0) return -1;
    for (int A = 0; A < Q.nen; A++) {
        R[A] = Q.R[A];
        node[A] = Q.node[A];
        for (int i = 0; i < 3; i++) {
            dR[A * 3 + i] = Q.dR[A][i];
            for (int j = 0; j < 3; j++) ddR[A * 9 + i * 3 + j] = Q.ddR[A][i][j];
        }
    }
    for (int i = 0; i < 3; i++) x[i] = Q.x[i];
    *detJ = Q.detJ;
    return Q.nen;
}

/* ------------------------------------------------------------------------------------ */
/* Third-order basis: every spatial derivative of R_A up to order 3 at */
/* one point, written out in the paper's order and notation:                               */
/*   N and its first three derivatives by the derivative recursion (A5), tensor product     */
/*   M_{A,abg}; w, w_{,a}, w_{,ab}, w_{,abg}; R_A ... R_{A,abg} by  */
/*   (rational) P:211, (drational) P:234, (ddrational) P:245, (dddrational) P:248-255;      */
/*   x_{m,a}, x_{m,ab}, x_{m,abg} = sum_B x_B R_{B,...} (isoparametric map P:265-278);        */
/*   xi_{a,i} (A-5), xi_{n,nl}, xi_{n,nlo};                  */
/*   R_{A,i}, R_{A,ij}, R_{A,ijk} by (dspatial), (ddspatial), (dddspatial) P:309-315.        */
/* Output per local function A: R[A], d1[A][3], d2[A][3][3], d3[A][3][3][3] (unused dims 0). */
/* ------------------------------------------------------------------------------------ */
int orc_eval_point3(const orc_space *s, const int *e_in, const double *xi_in, double *R, double *d1, double *d2,
                    double *d3, int64_t *node, double *x, double *detJ)
{
    int dim = s->dim;
    int e[3] = {0, 0, 0};
    double xi[3] = {0, 0, 0};
    for (int d = 0; d < dim; d++) { e[d] = e_in[d]; xi[d] = xi_in[d]; }
    double Nv[3][ORC_MAXP + 1][4];
    int first[3];
    for (int d = 0; d < 3; d++) {
        if (d >= dim) { Nv[d][0][0] = 1.0; Nv[d][0][1] = Nv[d][0][2] = Nv[d][0][3] = 0.0; first[d] = 0; continue; }
        int sp = s->span[d][e[d]];
        first[d] = sp - s->p[d];
        for (int a = 0; a <= s->p[d]; a++)
            for (int k = 0; k < 4; k++) Nv[d][a][k] = orc_coxdeboor_deriv(first[d] + a, s->p[d], s->U[d], xi[d], k);
    }
    int n0 = s->p[0] + 1, n1 = dim > 1 ? s->p[1] + 1 : 1, n2 = dim > 2 ? s->p[2] + 1 : 1;
    int nen = n0 * n1 * n2;
    static __thread double M[ORC_MAXEN], M1[ORC_MAXEN][3], M2[ORC_MAXEN][3][3], M3[ORC_MAXEN][3][3][3], wA[ORC_MAXEN];
    for (int A = 0; A < nen; A++) {
        int aa[3] = {A / (n1 * n2), (A / n2) % n1, A % n2};
        int g[3];
        for (int d = 0; d < 3; d++) g[d] = (first[d] + aa[d]) % s->nu[d];
        node[A] = ((int64_t)g[0] * s->nu[1] + g[1]) * s->nu[2] + g[2];
        wA[A] = s->wts ? s->wts[node[A]] : 1.0;
        M[A] = Nv[0][aa[0]][0] * Nv[1][aa[1]][0] * Nv[2][aa[2]][0];
        for (int al = 0; al < 3; al++)
            for (int be = 0; be < 3; be++)
                for (int ga = 0; ga < 3; ga++) {
                    double v1 = 1.0, v2 = 1.0, v3 = 1.0;
                    for (int d = 0; d < 3; d++) {
                        int k1 = (d == al), k2 = k1 + (d == be), k3 = k2 + (d == ga);
                        v1 *= (k1 < 4) ? Nv[d][aa[d]][k1] : 0.0;
                        v2 *= (k2 < 4) ? Nv[d][aa[d]][k2] : 0.0;
                        v3 *= (k3 < 4) ? Nv[d][aa[d]][k3] : 0.0;
                    }
                    M1[A][al] = v1;
                    M2[A][al][be] = v2;
                    M3[A][al][be][ga] = v3;
                }
    }
    /* weight function and its derivatives */
    double w = 0.0, w1[3] = {0}, w2[3][3] = {{0}}, w3[3][3][3] = {{{0}}};
    for (int A = 0; A < nen; A++) {
        w += wA[A] * M[A];
        for (int al = 0; al < 3; al++) {
            w1[al] += wA[A] * M1[A][al];
            for (int be = 0; be < 3; be++) {
                w2[al][be] += wA[A] * M2[A][al][be];
                for (int ga = 0; ga < 3; ga++) w3[al][be][ga] += wA[A] * M3[A][al][be][ga];
            }
        }
    }
    /* rational basis and parametric derivatives */
    static __thread double Rp1[ORC_MAXEN][3], Rp2[ORC_MAXEN][3][3], Rp3[ORC_MAXEN][3][3][3];
    for (int A = 0; A < nen; A++) {
        R[A] = wA[A] * M[A] / w;
        for (int al = 0; al < dim; al++) Rp1[A][al] = (wA[A] * M1[A][al] - R[A] * w1[al]) / w;
        for (int al = 0; al < dim; al++)
            for (int be = 0; be < dim; be++)
                Rp2[A][al][be] = (wA[A] * M2[A][al][be] - R[A] * w2[al][be] - Rp1[A][be] * w1[al] - Rp1[A][al] * w1[be]) / w;
        for (int al = 0; al < dim; al++)
            for (int be = 0; be < dim; be++)
                for (int ga = 0; ga < dim; ga++)
                    Rp3[A][al][be][ga] = (wA[A] * M3[A][al][be][ga] - R[A] * w3[al][be][ga]) / w
                                         - (Rp1[A][al] * w2[be][ga] + Rp1[A][be] * w2[al][ga] + Rp1[A][ga] * w2[al][be]) / w
                                         - (Rp2[A][be][ga] * w1[al] + Rp2[A][al][ga] * w1[be] + Rp2[A][al][be] * w1[ga]) / w;
    }
    /* isoparametric map and its parametric derivatives up to third order */
    double X[3] = {0}, X1[3][3] = {{0}}, X2[3][3][3] = {{{0}}}, X3[3][3][3][3] = {{{{0}}}};
    if (s->geom == ORC_NURBS) {
        for (int B = 0; B < nen; B++)
            for (int m = 0; m < dim; m++) {
                double xb = s->ctrl[node[B] * dim + m];
                X[m] += xb * R[B];
                for (int al = 0; al < dim; al++) {
                    X1[m][al] += xb * Rp1[B][al];
                    for (int be = 0; be < dim; be++) {
                        X2[m][al][be] += xb * Rp2[B][al][be];
                        for (int ga = 0; ga < dim; ga++) X3[m][al][be][ga] += xb * Rp3[B][al][be][ga];
                    }
                }
            }
    } else {
        for (int m = 0; m < dim; m++) { X[m] = xi[m]; X1[m][m] = 1.0; }
    }
    double Xi[3][3] = {{0}};
    double det = inverse(dim, X1, Xi);
    if (!(det > 0.0)) return -1;
    /* xi_{nu,nl} = - x_{m,eps mu} xi_{eps,n} xi_{mu,l} xi_{nu,m} */
    double Xi2[3][3][3] = {{{0}}};
    for (int nu_ = 0; nu_ < dim; nu_++)
        for (int n = 0; n < dim; n++)
            for (int l = 0; l < dim; l++) {
                double v = 0.0;
                for (int m = 0; m < dim; m++)
                    for (int ep = 0; ep < dim; ep++)
                        for (int mu = 0; mu < dim; mu++) v -= X2[m][ep][mu] * Xi[ep][n] * Xi[mu][l] * Xi[nu_][m];
                Xi2[nu_][n][l] = v;
            }
    /* xi_{nu,nlo} = - x_{m,eps mu om} xi_{eps,n} xi_{mu,l} xi_{nu,m} xi_{om,o}
     *              - x_{m,eps mu} (xi_{eps,no} xi_{mu,l} xi_{nu,m} + xi_{eps,n} xi_{mu,lo} xi_{nu,m}
     *                              + xi_{eps,n} xi_{mu,l} xi_{nu,mo}) */
    double Xi3[3][3][3][3] = {{{{0}}}};
    for (int nu_ = 0; nu_ < dim; nu_++)
        for (int n = 0; n < dim; n++)
            for (int l = 0; l < dim; l++)
                for (int o = 0; o < dim; o++) {
                    double v = 0.0;
                    for (int m = 0; m < dim; m++)
                        for (int ep = 0; ep < dim; ep++)
                            for (int mu = 0; mu < dim; mu++) {
                                for (int om = 0; om < dim; om++)
                                    v -= X3[m][ep][mu][om] * Xi[ep][n] * Xi[mu][l] * Xi[nu_][m] * Xi[om][o];
                                v -= X2[m][ep][mu] * (Xi2[ep][n][o] * Xi[mu][l] * Xi[nu_][m] + Xi[ep][n] * Xi2[mu][l][o] * Xi[nu_][m]
                                                      + Xi[ep][n] * Xi[mu][l] * Xi2[nu_][m][o]);
                            }
                    Xi3[nu_][n][l][o] = v;
                }
    /* push-forward (dspatial) P:309, (ddspatial) P:310, (dddspatial) P:311-315 */
    for (int A = 0; A < nen; A++) {
        for (int i = 0; i < 3; i++) {
            double v1 = 0.0;
            if (i < dim)
                for (int al = 0; al < dim; al++) v1 += Rp1[A][al] * Xi[al][i];
            d1[A * 3 + i] = v1;
            for (int j = 0; j < 3; j++) {
                double v2 = 0.0;
                if (i < dim && j < dim) {
                    for (int al = 0; al < dim; al++)
                        for (int be = 0; be < dim; be++) v2 += Rp2[A][al][be] * Xi[al][i] * Xi[be][j];
                    for (int al = 0; al < dim; al++) v2 += Rp1[A][al] * Xi2[al][i][j];
                }
                d2[(A * 3 + i) * 3 + j] = v2;
                for (int k = 0; k < 3; k++) {
                    double v3 = 0.0;
                    if (i < dim && j < dim && k < dim) {
                        for (int al = 0; al < dim; al++)
                            for (int be = 0; be < dim; be++) {
                                for (int ga = 0; ga < dim; ga++) v3 += Rp3[A][al][be][ga] * Xi[al][i] * Xi[be][j] * Xi[ga][k];
                                v3 += Rp2[A][al][be] * (Xi[al][i] * Xi2[be][j][k] + Xi[be][j] * Xi2[al][i][k] + Xi[be][k] * Xi2[al][i][j]);
                            }
                        for (int al = 0; al < dim; al++) v3 += Rp1[A][al] * Xi3[al][i][j][k];
                    }
                    d3[((A * 3 + i) * 3 + j) * 3 + k] = v3;
                }
            }
        }
    }
    for (int i = 0; i < 3; i++) x[i] = X[i];
    *detJ = det;
    return nen;
}

/* ------------------------------------------------------------------------------------ */
/* Fields at the quadrature point from U_e (Alg. 4).                      */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    double u[ORC_MAXM], du[ORC_MAXM][3], lap[ORC_MAXM], ut[ORC_MAXM];
} orc_fields;

static void eval_fields(const orc_space *s, const orc_qp *Q, const double *U, const double *Udot,
                        orc_fields *f)
{
    int m = s->dof, dim = s->dim;
    memset(f, 0, sizeof(*f));
    for (int A = 0; A < Q->nen; A++)
        for (int c = 0; c < m; c++) {
            double uA = U[Q->node[A] * m + c];
            double vA = Udot ? Udot[Q->node[A] * m + c] : 0.0;
            f->u[c] += uA * Q->R[A];
            f->ut[c] += vA * Q->R[A];
            for (int i = 0; i < dim; i++) {
                f->du[c][i] += uA * Q->dR[A][i];
                f->lap[c] += uA * Q->ddR[A][i][i];
            }
        }
}

/* ------------------------------------------------------------------------------------ */
/* Integrands (the paper leaves them to the user).          */
/* res(A) -> r[c]  (times dV by the caller);  jac(A,B) -> K[i][j] (times dV by caller).   */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int kind, dim, m;
    const double *prm;
    double a, b;
    /* CH */
    double M, Mp, Mpp, mup, mupp;
    /* NH */
    double F[3][3], S[3][3], P[3][3], Ci[3][3], J, AA[3][3][3][3];
    /* VMS */
    double tauM, tauC, rM[3], rC, up[3], pp, G[3][3], gg;
    /* NSK */
    double pv, dpv;
} orc_pt;

/* LAPLACE: R_A = int kappa grad N_A . grad u + sigma N_A u - N_A f; J_AB = b int (...)  */
static double laplace_source(const orc_pt *P, const orc_qp *Q)
{
    if ((int)P->prm[2] == 1) {
        const double pi = 3.14159265358979323846;
        return 2.0 * pi * pi * sin(pi * Q->x[0]) * sin(pi * Q->x[1]);
    }
    return 0.0;
}

/* Cahn-Hilliard (readings A-10, A-11): M = c(1-c),
 * mu' = 3 alpha (1/(2 theta c(1-c)) - 2), mu'' = 3 alpha (2c-1)/(2 theta c^2 (1-c)^2) */
static void ch_setup(orc_pt *P, const orc_fields *f)
{
    double th = P->prm[0], al = P->prm[1];
    double c = f->u[0];
    P->M = c * (1.0 - c);
    P->Mp = 1.0 - 2.0 * c;
    P->Mpp = -2.0;
    P->mup = 3.0 * al * (1.0 / (2.0 * th * c * (1.0 - c)) - 2.0);
    P->mupp = 3.0 * al * (2.0 * c - 1.0) / (2.0 * th * c * c * (1.0 - c) * (1.0 - c));
}

/* Neo-Hookean (A-12, A-13): F = I + grad u, C = F^T F, J = det F,
 * S = lambda/2 (J^2-1) C^{-1} + mu (I - C^{-1}), P = F S */
static void nh_setup(orc_pt *P, const orc_fields *f)
{
    double lam = P->prm[0], mu = P->prm[1];
    double C[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) P->F[i][j] = (i == j ? 1.0 : 0.0) + f->du[i][j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            C[i][j] = 0.0;
            for (int k = 0; k < 3; k++) C[i][j] += P->F[k][i] * P->F[k][j];
        }
    double Fi[3][3];
    P->J = inverse(3, P->F, Fi);
    inverse(3, C, P->Ci);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++)
            P->S[i][j] = lam / 2.0 * (P->J * P->J - 1.0) * P->Ci[i][j]
                       + mu * ((i == j ? 1.0 : 0.0) - P->Ci[i][j]);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            P->P[i][j] = 0.0;
            for (int k = 0; k < 3; k++) P->P[i][j] += P->F[i][k] * P->S[k][j];
        }
}

/* C_IJKL = lambda J^2 Ci_IJ Ci_KL + (mu - lambda (J^2-1)/2)(Ci_IK Ci_JL + Ci_IL Ci_JK) */
static double nh_CC(const orc_pt *P, int I, int J, int K, int L)
{
    double lam = P->prm[0], mu = P->prm[1];
    return lam * P->J * P->J * P->Ci[I][J] * P->Ci[K][L]
         + (mu - lam * (P->J * P->J - 1.0) / 2.0) * (P->Ci[I][K] * P->Ci[J][L] + P->Ci[I][L] * P->Ci[J][K]);
}

/* AA_aIbJ = delta_ab S_IJ + F_aK C_KILJ F_bL, once per point */
static void nh_tangent(orc_pt *P)
{
    for (int a = 0; a < 3; a++)
        for (int I = 0; I < 3; I++)
            for (int bb = 0; bb < 3; bb++)
                for (int J = 0; J < 3; J++) {
                    double AA = (a == bb ? P->S[I][J] : 0.0);
                    for (int Kk = 0; Kk < 3; Kk++)
                        for (int L = 0; L < 3; L++)
                            AA += P->F[a][Kk] * nh_CC(P, Kk, I, L, J) * P->F[bb][L];
                    P->AA[a][I][bb][J] = AA;
                }
}

/* RBVMS (readings A-14, A-15). prm = [nu, dt, C_t, C_I].
 * G_ij = sum_k dxihat_k/dx_i dxihat_k/dx_j, dxihat_k/dx_i = (2/h_k) xi_{k,i};
 * tau_M = (C_t/dt^2 + u.G u + C_I nu^2 G:G)^{-1/2}, tau_C = 1/(tau_M g.g). */
static void vms_tau(orc_pt *P, const orc_qp *Q, const orc_fields *ftau)
{
    double nu = P->prm[0], dt = P->prm[1], Ct = P->prm[2], CI = P->prm[3];
    double D[3][3], G[3][3], g[3];
    for (int k = 0; k < 3; k++)
        for (int i = 0; i < 3; i++) D[k][i] = 2.0 / Q->hpar[k] * Q->dxi_dx[k][i];
    for (int i = 0; i < 3; i++) {
        g[i] = 0.0;
        for (int k = 0; k < 3; k++) g[i] += D[k][i];
        for (int j = 0; j < 3; j++) {
            G[i][j] = 0.0;
            for (int k = 0; k < 3; k++) G[i][j] += D[k][i] * D[k][j];
        }
    }
    double uGu = 0.0, GG = 0.0, gg = 0.0;
    for (int i = 0; i < 3; i++) {
        gg += g[i] * g[i];
        for (int j = 0; j < 3; j++) {
            uGu += ftau->u[i] * G[i][j] * ftau->u[j];
            GG += G[i][j] * G[i][j];
        }
    }
    P->tauM = 1.0 / sqrt(Ct / (dt * dt) + uGu + CI * nu * nu * GG);
    P->tauC = 1.0 / (P->tauM * gg);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) P->G[i][j] = G[i][j];
    P->gg = gg;
}

static void vms_setup(orc_pt *P, const orc_fields *f)
{
    double nu = P->prm[0];
    /* r_M,i = udot_i + u_k u_{i,k} + p_{,i} - nu lap u_i ; r_C = u_{k,k} */
    P->rC = 0.0;
    for (int i = 0; i < 3; i++) {
        double conv = 0.0;
        for (int k = 0; k < 3; k++) conv += f->u[k] * f->du[i][k];
        P->rM[i] = f->ut[i] + conv + f->du[3][i] - nu * f->lap[i];
        P->rC += f->du[i][i];
    }
    for (int i = 0; i < 3; i++) P->up[i] = -P->tauM * P->rM[i];
    P->pp = -P->tauC * P->rC;
}

/* Navier-Stokes-Korteweg, readings A-25..A-27:
 * unknowns (rho, u_1..u_d) per node; prm = [a, b, R, theta, mu_bar, lambda_bar, lambda].
 * van der Waals pressure p = R b rho theta / (b - rho) - a rho^2, p' = R b^2 theta/(b-rho)^2 - 2 a rho.
 * Weak form of the strong form P:780-782 on a periodic domain (boundary terms vanish):
 *   R^C_A    = N_A rho_t - N_{A,j} rho u_j
 *   R^M_{Ai} = N_A (rho_t u_i + rho u_{i,t}) + N_{A,j} (-rho u_i u_j - p delta_ij + tau_ij + zeta_ij)
 *   tau  = mu_bar (grad u + grad u^T) + lambda_bar (div u) I
 *   zeta = lambda (rho lap rho + |grad rho|^2 / 2) I - lambda grad rho (x) grad rho */
static void nsk_setup(orc_pt *P, const orc_fields *f)
{
    const double av = P->prm[0], bv = P->prm[1], Rg = P->prm[2], th = P->prm[3];
    double rho = f->u[0];
    P->pv = Rg * bv * rho * th / (bv - rho) - av * rho * rho;
    P->dpv = Rg * bv * bv * th / ((bv - rho) * (bv - rho)) - 2.0 * av * rho;
}

/* NSK residual at a point for test function values (N, dN): r[0..dim] */
static void nsk_residual(const orc_pt *P, const orc_fields *f, double N, const double *dN, double *r)
{
    int dim = P->dim;
    const double mub = P->prm[4], lamb = P->prm[5], lam = P->prm[6];
    double rho = f->u[0], rhot = f->ut[0];
    double div = 0.0, g2 = 0.0;
    for (int k = 0; k < dim; k++) { div += f->du[1 + k][k]; g2 += f->du[0][k] * f->du[0][k]; }
    double v = N * rhot;
    for (int j = 0; j < dim; j++) v -= dN[j] * rho * f->u[1 + j];
    r[0] = v;
    for (int i = 0; i < dim; i++) {
        double w = N * (rhot * f->u[1 + i] + rho * f->ut[1 + i]);
        for (int j = 0; j < dim; j++) {
            double sig = -rho * f->u[1 + i] * f->u[1 + j];
            double tau = mub * (f->du[1 + i][j] + f->du[1 + j][i]);
            double zeta = -lam * f->du[0][i] * f->du[0][j];
            if (i == j) {
                sig -= P->pv;
                tau += lamb * div;
                zeta += lam * (rho * f->lap[0] + 0.5 * g2);
            }
            w += dN[j] * (sig + tau + zeta);
        }
        r[1 + i] = w;
    }
}

static void residual_at(const orc_pt *P, const orc_qp *Q, const orc_fields *f, int A, double *r)
{
    int dim = P->dim;
    const double *dN = Q->dR[A];
    double N = Q->R[A];
    switch (P->kind) {
    case ORC_LAPLACE: {
        double kap = P->prm[0], sig = P->prm[1];
        double gg = 0.0;
        for (int i = 0; i < dim; i++) gg += dN[i] * f->du[0][i];
        r[0] = kap * gg + sig * N * f->u[0] - N * laplace_source(P, Q);
        break;
    }
    case ORC_CAHN_HILLIARD: {
        /* R_A = N_A cdot + M mu' gradN.gradc + M' (gradN.gradc) lap c + M lapN lap c  (A-11) */
        double gNc = 0.0, lapN = 0.0;
        for (int i = 0; i < dim; i++) { gNc += dN[i] * f->du[0][i]; lapN += Q->ddR[A][i][i]; }
        double lc = f->lap[0];
        r[0] = N * f->ut[0] + P->M * P->mup * gNc + P->Mp * gNc * lc + P->M * lapN * lc;
        break;
    }
    case ORC_NEOHOOKE: {
        /* R_{Aa} = N_{A,J} P_{aJ} (A-12) */
        for (int a = 0; a < 3; a++) {
            double v = 0.0;
            for (int J = 0; J < 3; J++) v += dN[J] * P->P[a][J];
            r[a] = v;
        }
        break;
    }
    case ORC_NSK:
        nsk_residual(P, f, N, dN, r);
        break;
    case ORC_NS_VMS: {
        double nu = P->prm[0];
        /* momentum (Appendix A) */
        for (int i = 0; i < 3; i++) {
            double v = N * f->ut[i];
            for (int k = 0; k < 3; k++) {
                v += -dN[k] * f->u[k] * f->u[i];
                v += nu * dN[k] * (f->du[i][k] + f->du[k][i]);
            }
            v += -dN[i] * f->u[3];
            double uN = 0.0;
            for (int k = 0; k < 3; k++) uN += f->u[k] * dN[k];
            v += -uN * P->up[i];
            v += -dN[i] * P->pp;
            for (int k = 0; k < 3; k++) v += N * P->up[k] * f->du[i][k];
            for (int k = 0; k < 3; k++) v += -dN[k] * P->up[i] * P->up[k];
            r[i] = v;
        }
        /* continuity */
        {
            double v = 0.0;
            for (int k = 0; k < 3; k++) v += N * f->du[k][k] - dN[k] * P->up[k];
            r[3] = v;
        }
        break;
    }
    }
}

/* Jacobian block K[i][j] of test (A,i), trial (B,j): J = a dR/dUdot + b dR/dU (A-16),
 * each part the literal linearisation of residual_at() in the direction N_B e_j. */
static void jacobian_at(const orc_pt *P, const orc_qp *Q, const orc_fields *f, int A, int B, double *K)
{
    int dim = P->dim, m = P->m;
    const double *dNA = Q->dR[A], *dNB = Q->dR[B];
    double NA = Q->R[A], NB = Q->R[B];
    double lapA = 0.0, lapB = 0.0;
    for (int i = 0; i < dim; i++) { lapA += Q->ddR[A][i][i]; lapB += Q->ddR[B][i][i]; }
    switch (P->kind) {
    case ORC_LAPLACE: {
        double kap = P->prm[0], sig = P->prm[1];
        double gg = 0.0;
        for (int i = 0; i < dim; i++) gg += dNA[i] * dNB[i];
        K[0] = P->b * (kap * gg + sig * NA * NB);
        break;
    }
    case ORC_CAHN_HILLIARD: {
        double gNc = 0.0, gNdc = 0.0;
        for (int i = 0; i < dim; i++) { gNc += dNA[i] * f->du[0][i]; gNdc += dNA[i] * dNB[i]; }
        double lc = f->lap[0];
        /* delta c = N_B, delta grad c = grad N_B, delta lap c = lap N_B */
        double dM = P->Mp * NB, dmup = P->mupp * NB, dMp = P->Mpp * NB;
        double dR = (dM * P->mup + P->M * dmup) * gNc + P->M * P->mup * gNdc
                  + dMp * gNc * lc + P->Mp * gNdc * lc + P->Mp * gNc * lapB
                  + dM * lapA * lc + P->M * lapA * lapB;
        K[0] = P->a * NA * NB + P->b * dR;
        break;
    }
    case ORC_NEOHOOKE: {
        /* K_(Aa)(Bb) = b N_{A,I} AA_{aIbJ} N_{B,J}, AA_aIbJ = delta_ab S_IJ + F_aK C_KILJ F_bL */
        for (int a = 0; a < 3; a++)
            for (int bb = 0; bb < 3; bb++) {
                double v = 0.0;
                for (int I = 0; I < 3; I++)
                    for (int J = 0; J < 3; J++) v += dNA[I] * P->AA[a][I][bb][J] * dNB[J];
                K[a * 3 + bb] = P->b * v;
            }
        break;
    }
    case ORC_NSK: {
        const double mub = P->prm[4], lamb = P->prm[5], lam = P->prm[6];
        double rho = f->u[0], rhot = f->ut[0];
        double g2 = 0.0;
        for (int k = 0; k < dim; k++) g2 += f->du[0][k] * f->du[0][k];
        for (int j = 0; j < m; j++) {
            double res[2][ORC_MAXM];
            for (int part = 0; part < 2; part++) {
                /* perturbation of the fields in the direction N_B e_j */
                double drho = 0.0, drhot = 0.0, dgrho[3] = {0, 0, 0}, dlrho = 0.0;
                double du[3] = {0, 0, 0}, dut[3] = {0, 0, 0}, dgu[3][3] = {{0}};
                if (part == 0) {
                    if (j == 0) drhot = NB; else dut[j - 1] = NB;
                } else if (j == 0) {
                    drho = NB;
                    for (int k = 0; k < dim; k++) dgrho[k] = dNB[k];
                    dlrho = lapB;
                } else {
                    du[j - 1] = NB;
                    for (int k = 0; k < dim; k++) dgu[j - 1][k] = dNB[k];
                }
                double ddiv = 0.0, dg2 = 0.0;
                for (int k = 0; k < dim; k++) { ddiv += dgu[k][k]; dg2 += 2.0 * f->du[0][k] * dgrho[k]; }
                double v = NA * drhot;
                for (int l = 0; l < dim; l++) v -= dNA[l] * (drho * f->u[1 + l] + rho * du[l]);
                res[part][0] = v;
                for (int i = 0; i < dim; i++) {
                    double w = NA * (drhot * f->u[1 + i] + rhot * du[i] + drho * f->ut[1 + i] + rho * dut[i]);
                    for (int l = 0; l < dim; l++) {
                        double dsig = -(drho * f->u[1 + i] * f->u[1 + l] + rho * du[i] * f->u[1 + l] + rho * f->u[1 + i] * du[l]);
                        double dtau = mub * (dgu[i][l] + dgu[l][i]);
                        double dzeta = -lam * (dgrho[i] * f->du[0][l] + f->du[0][i] * dgrho[l]);
                        if (i == l) {
                            dsig -= P->dpv * drho;
                            dtau += lamb * ddiv;
                            dzeta += lam * (drho * f->lap[0] + rho * dlrho + 0.5 * dg2);
                        }
                        w += dNA[l] * (dsig + dtau + dzeta);
                    }
                    res[part][1 + i] = w;
                }
            }
            for (int i = 0; i < m; i++) K[i * m + j] = P->a * res[0][i] + P->b * res[1][i];
        }
        break;
    }
    case ORC_NS_VMS: {
        double nu = P->prm[0];
        for (int j = 0; j < 4; j++) {
            double res[2][4];
            for (int part = 0; part < 2; part++) {  /* part 0: d/dUdot, part 1: d/dU */
                double du[3] = {0, 0, 0}, dgu[3][3] = {{0}}, dlap[3] = {0, 0, 0}, dp = 0.0, dgp[3] = {0, 0, 0};
                double dut[3] = {0, 0, 0};
                if (part == 0) {
                    if (j < 3) dut[j] = NB;
                } else if (j < 3) {
                    du[j] = NB;
                    for (int k = 0; k < 3; k++) dgu[j][k] = dNB[k];
                    dlap[j] = lapB;
                } else {
                    dp = NB;
                    for (int k = 0; k < 3; k++) dgp[k] = dNB[k];
                }
                /* tau frozen (A-15) */
                double drM[3], drC = 0.0, dup[3];
                for (int i = 0; i < 3; i++) {
                    double v = dut[i] + dgp[i] - nu * dlap[i];
                    for (int k = 0; k < 3; k++) v += du[k] * f->du[i][k] + f->u[k] * dgu[i][k];
                    drM[i] = v;
                    drC += dgu[i][i];
                }
                for (int i = 0; i < 3; i++) dup[i] = -P->tauM * drM[i];
                double dpp = -P->tauC * drC;
                double uN = 0.0, duN = 0.0;
                for (int k = 0; k < 3; k++) { uN += f->u[k] * dNA[k]; duN += du[k] * dNA[k]; }
                for (int i = 0; i < 3; i++) {
                    double v = NA * dut[i];
                    for (int k = 0; k < 3; k++) {
                        v += -dNA[k] * (du[k] * f->u[i] + f->u[k] * du[i]);
                        v += nu * dNA[k] * (dgu[i][k] + dgu[k][i]);
                    }
                    v += -dNA[i] * dp;
                    v += -duN * P->up[i] - uN * dup[i];
                    v += -dNA[i] * dpp;
                    for (int k = 0; k < 3; k++) v += NA * (dup[k] * f->du[i][k] + P->up[k] * dgu[i][k]);
                    for (int k = 0; k < 3; k++) v += -dNA[k] * (dup[i] * P->up[k] + P->up[i] * dup[k]);
                    res[part][i] = v;
                }
                {
                    double v = 0.0;
                    for (int k = 0; k < 3; k++) v += NA * dgu[k][k] - dNA[k] * dup[k];
                    res[part][3] = v;
                }
            }
            for (int i = 0; i < 4; i++) K[i * m + j] = P->a * res[0][i] + P->b * res[1][i];
        }
        break;
    }
    }
}

static int phys_dof(int kind)
{
    switch (kind) {
    case ORC_LAPLACE: case ORC_CAHN_HILLIARD: return 1;
    case ORC_NEOHOOKE: return 3;
    case ORC_NS_VMS: return 4;
    }
    return -1;
}

static int phys_dof_dim(int kind, int dim) { return kind == ORC_NSK ? 1 + dim : phys_dof(kind); }

/* ------------------------------------------------------------------------------------ */
/* Element integration (Alg. 4 lines P:599-604): dense K_e and F_e.                       */
/* Ke is (nen*m)^2 row-major with row = A*m+i, col = B*m+j.  Utau: state for the frozen   */
/* VMS tau (NULL => U).  Returns 0, or <0 on detJ <= 0.                                   */
/* ------------------------------------------------------------------------------------ */
static int element_integrate(const orc_space *s, int kind, const double *prm, double a, double b,
                             const double *U, const double *Udot, const double *Utau,
                             const int e[3], int want_K, const unsigned char *rowmask,
                             double *Ke, double *Fe, orc_qp *Qlast)
{
    int m = s->dof, dim = s->dim;
    orc_qp Q;
    int nen = 0;
    int nq0 = s->nq[0], nq1 = s->nq[1], nq2 = s->nq[2];
    for (int q0 = 0; q0 < nq0; q0++)
        for (int q1 = 0; q1 < nq1; q1++)
            for (int q2 = 0; q2 < nq2; q2++) {
                int qq[3] = {q0, q1, q2};
                double xi[3] = {0, 0, 0}, wq = 1.0;
                for (int d = 0; d < dim; d++) {
                    int sp = s->span[d][e[d]];
                    double lo = s->U[d][sp], hi = s->U[d][sp + 1];
                    xi[d] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * s->gx[d][qq[d]];
                    wq *= s->gw[d][qq[d]] * 0.5 * (hi - lo);
                }
                if (eval_point(s, e, xi, wq, &Q) < 0) return -1;
                if (nen == 0) {
                    nen = Q.nen;
                    if (Ke) memset(Ke, 0, sizeof(double) * (size_t)nen * m * nen * m);
                    if (Fe) memset(Fe, 0, sizeof(double) * (size_t)nen * m);
                }
                orc_fields f, ftau;
                eval_fields(s, &Q, U, Udot, &f);
                orc_pt P;
                memset(&P, 0, sizeof(P));
                P.kind = kind; P.dim = dim; P.m = m; P.prm = prm; P.a = a; P.b = b;
                if (kind == ORC_CAHN_HILLIARD) ch_setup(&P, &f);
                if (kind == ORC_NSK) nsk_setup(&P, &f);
                if (kind == ORC_NEOHOOKE) { nh_setup(&P, &f); if (want_K) nh_tangent(&P); }
                if (kind == ORC_NS_VMS) {
                    if (Utau) { eval_fields(s, &Q, Utau, Udot, &ftau); vms_tau(&P, &Q, &ftau); }
                    else vms_tau(&P, &Q, &f);
                    vms_setup(&P, &f);
                }
                for (int A = 0; A < nen; A++) {
                    if (rowmask && !rowmask[A]) continue;
                    if (Fe) {
                        double r[ORC_MAXM];
                        residual_at(&P, &Q, &f, A, r);
                        for (int i = 0; i < m; i++) Fe[A * m + i] += r[i] * Q.dV;   /* F_e += F_q J_q w_q */
                    }
                    if (want_K && Ke)
                        for (int B = 0; B < nen; B++) {
                            double Kb[ORC_MAXM * ORC_MAXM];
                            jacobian_at(&P, &Q, &f, A, B, Kb);
                            for (int i = 0; i < m; i++)
                                for (int j = 0; j < m; j++)
                                    Ke[(size_t)(A * m + i) * nen * m + B * m + j] += Kb[i * m + j] * Q.dV;
                        }
                }
            }
    if (Qlast) *Qlast = Q;
    return nen;
}

/* Point state of the integrand at parametric point xi[] of element e[] (tests only: it exposes
 * the reading-dependent constitutive quantities so that tests/test_oracle_state_pins.py can pin
 * them to the independently computed values of SURVEY Appendices A and C).  Same call sequence
 * as element_integrate: eval_point, eval_fields, *_setup.  out[] by kind:
 *   ORC_NS_VMS:        tauM, tauC, G[3][3] (row-major), g.g, u'[3], p'       (16 doubles)
 *   ORC_CAHN_HILLIARD: M, M', M'', mu', mu''                                  (5 doubles)
 * Returns the number of doubles written, or <0. */
int orc_point_state(const orc_space *s, int kind, const double *prm, const double *U, const double *Udot,
                    const int *e_in, const double *xi_in, double *out)
{
    orc_qp Q;
    int e[3] = {0, 0, 0};
    double xi[3] = {0, 0, 0};
    for (int d = 0; d < s->dim; d++) { e[d] = e_in[d]; xi[d] = xi_in[d]; }
    if (eval_point(s, e, xi, 1.0, &Q) < 0) return -1;
    orc_fields f;
    eval_fields(s, &Q, U, Udot, &f);
    orc_pt P;
    memset(&P, 0, sizeof(P));
    P.kind = kind; P.dim = s->dim; P.m = s->dof; P.prm = prm;
    if (kind == ORC_NS_VMS) {
        if (s->dim != 3 || s->dof != 4) return -3;
        vms_tau(&P, &Q, &f);
        vms_setup(&P, &f);
        out[0] = P.tauM;
        out[1] = P.tauC;
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) out[2 + 3 * i + j] = P.G[i][j];
        out[11] = P.gg;
        for (int i = 0; i < 3; i++) out[12 + i] = P.up[i];
        out[15] = P.pp;
        return 16;
    }
    if (kind == ORC_CAHN_HILLIARD) {
        if (s->dof != 1) return -3;
        ch_setup(&P, &f);
        out[0] = P.M; out[1] = P.Mp; out[2] = P.Mpp; out[3] = P.mup; out[4] = P.mupp;
        return 5;
    }
    return -2;
}

/* Dense element matrix / vector of element (e0,e1,e2) (for tests). nodes[] gets the nen
 * global nodes. Returns nen or <0. */
int orc_element(const orc_space *s, int kind, const double *prm, double a, double b,
                const double *U, const double *Udot, const double *Utau, const int *e,
                double *Ke, double *Fe, int64_t *nodes)
{
    if (phys_dof_dim(kind, s->dim) != s->dof) return -3;
    int ee[3] = {0, 0, 0};
    for (int d = 0; d < s->dim; d++) ee[d] = e[d];
    orc_qp Q;
    int nen = element_integrate(s, kind, prm, a, b, U, Udot, Utau, ee, Ke != NULL, NULL, Ke, Fe, &Q);
    if (nen < 0) return nen;
    for (int A = 0; A < nen; A++) nodes[A] = Q.node[A];
    return nen;
}

/* ------------------------------------------------------------------------------------ */
/* Dense global assembly (tiny spaces; O-8 "literal reading"): K (ndof x ndof row-major),  */
/* touched[] marks entries any element contributed to; F the residual (Alg. 4). */
/* ------------------------------------------------------------------------------------ */
int orc_assemble_dense(const orc_space *s, int kind, const double *prm, double a, double b,
                       const double *U, const double *Udot, const double *Utau,
                       double *K, unsigned char *touched, double *F)
{
    if (phys_dof_dim(kind, s->dim) != s->dof) return -3;
    int m = s->dof;
    int64_t nd = orc_ndof(s);
    if (K) memset(K, 0, sizeof(double) * (size_t)nd * nd);
    if (touched) memset(touched, 0, (size_t)nd * nd);
    if (F) memset(F, 0, sizeof(double) * (size_t)nd);
    double *Ke = (double *)malloc(sizeof(double) * ORC_MAXEN * ORC_MAXM * ORC_MAXEN * ORC_MAXM);
    double *Fe = (double *)malloc(sizeof(double) * ORC_MAXEN * ORC_MAXM);
    for (int e0 = 0; e0 < s->nel[0]; e0++)
        for (int e1 = 0; e1 < s->nel[1]; e1++)
            for (int e2 = 0; e2 < s->nel[2]; e2++) {
                int e[3] = {e0, e1, e2};
                orc_qp Q;
                int nen = element_integrate(s, kind, prm, a, b, U, Udot, Utau, e, K != NULL, NULL,
                                            Ke, Fe, &Q);
                if (nen < 0) { free(Ke); free(Fe); return nen; }
                for (int A = 0; A < nen; A++)
                    for (int i = 0; i < m; i++) {
                        int64_t row = Q.node[A] * m + i;
                        if (F) F[row] += Fe[A * m + i];      /* F_e -> F */
                        if (K)
                            for (int B = 0; B < nen; B++)
                                for (int j = 0; j < m; j++) {
                                    int64_t col = Q.node[B] * m + j;
                                    K[row * nd + col] += Ke[(size_t)(A * m + i) * nen * m + B * m + j];
                                    if (touched) touched[row * nd + col] = 1;
                                }
                    }
            }
    free(Ke);
    free(Fe);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Complete rows of a row subset (O-10): visit every element in the union of the supports */
/* of the rows' nodes, accumulate only rows in S, scatter by binary search into the       */
/* Alg. 3 pattern given by (rowptr, cols) (from orc_pattern_rows).  Every contribution    */
/* must land inside the pattern (else returns -2).  rows must be sorted ascending.        */
/* vals (nnz) / F (nrows) may be NULL.  touched (nnz, may be NULL) marks hit entries.     */
/* Returns the number of elements visited.                                                */
/* ------------------------------------------------------------------------------------ */
static int64_t find_row(const int64_t *rows, int64_t n, int64_t r)
{
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (rows[mid] == r) return mid;
        if (rows[mid] < r) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static int64_t find_col(const int32_t *c, int64_t n, int64_t col)
{
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (c[mid] == col) return mid;
        if (c[mid] < col) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

int64_t orc_assemble_rows(const orc_space *s, int kind, const double *prm, double a, double b,
                          const double *U, const double *Udot, const double *Utau,
                          int64_t nrows, const int64_t *rows, const int64_t *rowptr,
                          const int32_t *cols, double *vals, double *F, unsigned char *touched)
{
    if (phys_dof_dim(kind, s->dim) != s->dof) return -3;
    int m = s->dof;
    int dim = s->dim;
    /* elements touching each global function, per axis */
    int64_t nel_tot = (int64_t)s->nel[0] * s->nel[1] * s->nel[2];
    unsigned char *visit = (unsigned char *)calloc((size_t)nel_tot, 1);
    int *elist[3], *ecnt[3], emax[3];
    for (int d = 0; d < 3; d++) {
        int nu = s->nu[d];
        emax[d] = (d < dim) ? (s->p[d] + 1) * ((s->nfun[d] + nu - 1) / nu + 1) : 1;
        elist[d] = (int *)malloc(sizeof(int) * (size_t)nu * emax[d]);
        ecnt[d] = (int *)calloc(nu, sizeof(int));
        for (int e = 0; e < s->nel[d]; e++) {
            int first = (d < dim) ? s->span[d][e] - s->p[d] : 0;
            int np1 = (d < dim) ? s->p[d] + 1 : 1;
            for (int t = 0; t < np1; t++) {
                int g = (first + t) % nu;
                int dup = 0;
                for (int u = 0; u < ecnt[d][g]; u++) if (elist[d][(size_t)g * emax[d] + u] == e) dup = 1;
                if (!dup) elist[d][(size_t)g * emax[d] + ecnt[d][g]++] = e;
            }
        }
    }
    for (int64_t t = 0; t < nrows; t++) {
        int g[3];
        node_to_ijk(s, rows[t] / m, g);
        for (int x = 0; x < ecnt[0][g[0]]; x++)
            for (int y = 0; y < ecnt[1][g[1]]; y++)
                for (int z = 0; z < ecnt[2][g[2]]; z++) {
                    int64_t e = ((int64_t)elist[0][(size_t)g[0] * emax[0] + x] * s->nel[1]
                                 + elist[1][(size_t)g[1] * emax[1] + y]) * s->nel[2]
                                + elist[2][(size_t)g[2] * emax[2] + z];
                    visit[e] = 1;
                }
    }
    if (vals) memset(vals, 0, sizeof(double) * (size_t)rowptr[nrows]);
    if (touched) memset(touched, 0, (size_t)rowptr[nrows]);
    if (F) memset(F, 0, sizeof(double) * (size_t)nrows);
    double *Ke = (double *)malloc(sizeof(double) * ORC_MAXEN * ORC_MAXM * ORC_MAXEN * ORC_MAXM);
    double *Fe = (double *)malloc(sizeof(double) * ORC_MAXEN * ORC_MAXM);
    int64_t nvisit = 0, status = 0;
    for (int64_t e = 0; e < nel_tot && status == 0; e++) {
        if (!visit[e]) continue;
        nvisit++;
        int ee[3] = {(int)(e / ((int64_t)s->nel[1] * s->nel[2])), (int)((e / s->nel[2]) % s->nel[1]),
                     (int)(e % s->nel[2])};
        /* which local functions have at least one row in S */
        unsigned char mask[ORC_MAXEN];
        int64_t slot[ORC_MAXEN][ORC_MAXM];
        {
            orc_qp Q0;
            int nen0 = 1;
            for (int d = 0; d < dim; d++) nen0 *= s->p[d] + 1;
            /* node numbers of the element's functions (same mapping as eval_point) */
            int n1 = dim > 1 ? s->p[1] + 1 : 1, n2 = dim > 2 ? s->p[2] + 1 : 1;
            for (int A = 0; A < nen0; A++) {
                int aa[3] = {A / (n1 * n2), (A / n2) % n1, A % n2};
                int gg[3];
                for (int d = 0; d < 3; d++) {
                    int first = (d < dim) ? s->span[d][ee[d]] - s->p[d] : 0;
                    gg[d] = (first + aa[d]) % s->nu[d];
                }
                Q0.node[A] = ((int64_t)gg[0] * s->nu[1] + gg[1]) * s->nu[2] + gg[2];
                mask[A] = 0;
                for (int i = 0; i < m; i++) {
                    slot[A][i] = find_row(rows, nrows, Q0.node[A] * m + i);
                    if (slot[A][i] >= 0) mask[A] = 1;
                }
            }
        }
        orc_qp Q;
        int nen = element_integrate(s, kind, prm, a, b, U, Udot, Utau, ee, vals != NULL, mask, Ke, Fe, &Q);
        if (nen < 0) { status = nen; break; }
        for (int A = 0; A < nen; A++) {
            if (!mask[A]) continue;
            for (int i = 0; i < m; i++) {
                int64_t sl = slot[A][i];
                if (sl < 0) continue;
                if (F) F[sl] += Fe[A * m + i];
                if (vals || touched) {
                    const int32_t *rc = cols + rowptr[sl];
                    int64_t rl = rowptr[sl + 1] - rowptr[sl];
                    for (int B = 0; B < nen; B++)
                        for (int j = 0; j < m; j++) {
                            int64_t pos = find_col(rc, rl, Q.node[B] * m + j);
                            if (pos < 0) { status = -2; continue; }   /* outside Alg. 3 pattern */
                            if (vals) vals[rowptr[sl] + pos] += Ke[(size_t)(A * m + i) * nen * m + B * m + j];
                            if (touched) touched[rowptr[sl] + pos] = 1;
                        }
                }
            }
        }
    }
    free(Ke);
    free(Fe);
    free(visit);
    for (int d = 0; d < 3; d++) { free(elist[d]); free(ecnt[d]); }
    return status < 0 ? status : nvisit;
}
