// kinds.cuh -- compile-time description of the basis "kinds" the contraction works on, and of
// the compact (structurally nonzero) coefficient lists derived from a physics' D / r masks.
//
// MODE_PARAM (x = xi, unit weights): contraction kinds ARE the spatial kinds
//   {N, dN/dxi_0.., lap N}; lap N = sum_alpha d2N/dxi_alpha^2 is a sum of separable terms.
// MODE_NURBS (rational basis and/or mapped geometry): contraction kinds are the PARAMETRIC
//   B-spline kinds {M, M_,alpha, M_,alpha beta (alpha<=beta)}, each one separable tensor
//   product; rational basis (eqs. rational/drational/ddrational) and the
//   push-forward (dspatial/ddspatial P:309-310) are folded into the per-point coefficients
//   through a linear map T (spatial kind k <- parametric kind c), so that
//       B_k(A,q) = w_A * sum_c T_kc(q) P_c(A,q).
#pragma once
#include <utility>

#include "iga_internal.cuh"

namespace iga {

constexpr int MAXE = 448;   // max compact D entries
constexpr int MAXR = 64;    // max compact r entries

template <int DIM, int MODE, bool HESS>
struct KindSet {
    static constexpr int NKS = 1 + DIM + (HESS ? 1 : 0);                        // spatial kinds
    static constexpr int NH = DIM * (DIM + 1) / 2;                              // Hessian pairs
    static constexpr int NC = MODE == MODE_PARAM ? NKS : 1 + DIM + (HESS ? NH : 0);
    // Hessian pair index h -> (alpha, beta), alpha <= beta, row-major upper triangle
    static constexpr int hal(int h) {
        int t = 0;
        for (int al = 0; al < DIM; al++)
            for (int be = al; be < DIM; be++) {
                if (t == h) return al;
                t++;
            }
        return -1;
    }
    static constexpr int hbe(int h) {
        int t = 0;
        for (int al = 0; al < DIM; al++)
            for (int be = al; be < DIM; be++) {
                if (t == h) return be;
                t++;
            }
        return -1;
    }
    static constexpr int hidx(int al, int be) {
        if (al > be) { int t = al; al = be; be = t; }
        int t = 0;
        for (int a = 0; a < DIM; a++)
            for (int b = a; b < DIM; b++) {
                if (a == al && b == be) return t;
                t++;
            }
        return -1;
    }
    // number of separable terms of contraction kind c
    static constexpr int nterms(int c) {
        return (MODE == MODE_PARAM && HESS && c == 1 + DIM) ? DIM : 1;
    }
    // derivative order on axis d of term t of contraction kind c
    static constexpr int ord(int c, int t, int d) {
        if (c == 0) return 0;
        if (c <= DIM) return (d == c - 1) ? 1 : 0;
        if (MODE == MODE_PARAM) return (d == t) ? 2 : 0;     // lap = sum of pure second derivatives
        const int h = c - 1 - DIM;
        return (d == hal(h) ? 1 : 0) + (d == hbe(h) ? 1 : 0);
    }
    // structural dependence of spatial kind k on contraction kind c (the T map)
    static constexpr bool tmask(int k, int c) {
        if (MODE == MODE_PARAM) return k == c;
        if (k == 0) return c == 0;
        if (k <= DIM) return c <= DIM;
        return true;   // lap depends on everything
    }
};

template <class PH, int DIM, int MODE>
struct Lists {
    using KS = KindSet<DIM, MODE, PH::HESS>;
    static constexpr int M = PH::M;
    static constexpr int NKS = KS::NKS;
    static constexpr int NC = KS::NC;
    static constexpr bool cmask(int c, int i, int c2, int j) {
        for (int k = 0; k < NKS; k++)
            for (int k2 = 0; k2 < NKS; k2++)
                if (KS::tmask(k, c) && KS::tmask(k2, c2) && PH::template dmask<DIM>(k, i, k2, j)) return true;
        return false;
    }
    static constexpr bool crmask(int c, int i) {
        for (int k = 0; k < NKS; k++)
            if (KS::tmask(k, c) && PH::rmask(k, i)) return true;
        return false;
    }
    struct EList { int n; int c[MAXE], i[MAXE], c2[MAXE], j[MAXE]; };
    struct RList { int n; int c[MAXR], i[MAXR]; };
    static constexpr EList make_e() {
        EList L{};
        L.n = 0;
        for (int c = 0; c < NC; c++)
            for (int i = 0; i < M; i++)
                for (int c2 = 0; c2 < NC; c2++)
                    for (int j = 0; j < M; j++)
                        if (cmask(c, i, c2, j)) {
                            L.c[L.n] = c; L.i[L.n] = i; L.c2[L.n] = c2; L.j[L.n] = j; L.n++;
                        }
        return L;
    }
    static constexpr RList make_r() {
        RList L{};
        L.n = 0;
        for (int c = 0; c < NC; c++)
            for (int i = 0; i < M; i++)
                if (crmask(c, i)) { L.c[L.n] = c; L.i[L.n] = i; L.n++; }
        return L;
    }
    // the same entries ordered by (i, j, c, c2): one contiguous run per component pair
    static constexpr EList make_eij() {
        EList L{};
        L.n = 0;
        for (int i = 0; i < M; i++)
            for (int j = 0; j < M; j++)
                for (int c = 0; c < NC; c++)
                    for (int c2 = 0; c2 < NC; c2++)
                        if (cmask(c, i, c2, j)) {
                            L.c[L.n] = c; L.i[L.n] = i; L.c2[L.n] = c2; L.j[L.n] = j; L.n++;
                        }
        return L;
    }
    static constexpr EList E = make_e();
    static constexpr EList EIJ = make_eij();
    static constexpr int eij_start(int i, int j) {
        for (int e = 0; e < EIJ.n; e++)
            if (EIJ.i[e] == i && EIJ.j[e] == j) return e;
        return EIJ.n;
    }
    static constexpr int eij_count(int i, int j) {
        int n = 0;
        for (int e = 0; e < EIJ.n; e++)
            if (EIJ.i[e] == i && EIJ.j[e] == j) n++;
        return n;
    }
    // position of entry ee (in E order) within EIJ
    static constexpr int eij_of(int ee) {
        for (int e = 0; e < EIJ.n; e++)
            if (EIJ.i[e] == E.i[ee] && EIJ.j[e] == E.j[ee] && EIJ.c[e] == E.c[ee] && EIJ.c2[e] == E.c2[ee]) return e;
        return -1;
    }
    // is (c, i) a test row of some entry with trial component j
    static constexpr bool test_used_ij(int c, int i, int j) {
        for (int e = 0; e < EIJ.n; e++)
            if (EIJ.c[e] == c && EIJ.i[e] == i && EIJ.j[e] == j) return true;
        return false;
    }
    static constexpr RList R = make_r();
    static constexpr int NE = E.n;
    static constexpr int NR = R.n;
    // is contraction kind c used as a test / trial kind at all
    static constexpr bool test_used(int c) {
        for (int e = 0; e < NE; e++) if (E.c[e] == c) return true;
        for (int r = 0; r < NR; r++) if (R.c[r] == c) return true;
        return false;
    }
    static constexpr bool trial_used(int c) {
        for (int e = 0; e < NE; e++) if (E.c2[e] == c) return true;
        return false;
    }
    static_assert(NE <= MAXE && NR <= MAXR, "coefficient list too long");
    // dense per-(i,j) blocks over the union of test kinds (TK) and trial kinds (QK)
    static constexpr int NTK = [] { int n = 0; for (int c = 0; c < NC; c++) if (test_used(c)) n++; return n; }();
    static constexpr int NQK = [] { int n = 0; for (int c = 0; c < NC; c++) if (trial_used(c)) n++; return n; }();
    static constexpr int tk(int t) { int n = 0; for (int c = 0; c < NC; c++) if (test_used(c)) { if (n == t) return c; n++; } return -1; }
    static constexpr int qk(int t) { int n = 0; for (int c = 0; c < NC; c++) if (trial_used(c)) { if (n == t) return c; n++; } return -1; }
    static constexpr int tk_of(int c) { int n = 0; for (int x = 0; x < NC; x++) if (test_used(x)) { if (x == c) return n; n++; } return -1; }
    static constexpr int qk_of(int c) { int n = 0; for (int x = 0; x < NC; x++) if (trial_used(x)) { if (x == c) return n; n++; } return -1; }
};

// compile-time loop
template <typename F, int... Is>
__host__ __device__ __forceinline__ void static_for_impl(F &&f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F>
__host__ __device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

}  // namespace iga
