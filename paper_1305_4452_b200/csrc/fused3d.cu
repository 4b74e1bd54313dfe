// fused3d.cu -- K3/K4 for 3D parametric spaces (configs 4, 5, 8): one fused kernel per call.
//
// Persistent CTAs (two per SM, so that one CTA's latency-bound point phase overlaps the other's
// FP64-bound contraction) walk the element grid; per element a CTA runs Alg. 4 in
// phases separated by __syncthreads, everything staged in shared memory:
//   1. stage the element's 1D tables, Gauss weights, node numbers, U_e, CSR row starts and the
//      column-offset table colOff[A][B] (closed forms of the per-axis Alg. 3 tables);
//   2. field kinds at every point  Phi[q][m][k] = sum_A U_Am P_k(A,q)  (thread per (q, m));
//   3. per point: physics state + residual coefficients r~ (thread per q);
//   4. Jacobian coefficients: warp-uniform trial column (k2, j), lane = q -> dense per-(i,j)
//      blocks D[q][i,j][test kind][trial kind];
//   5. test-side sum factorisation: thread = (trial function B, trial component j), one pass per
//      test component i: H(q) = D_(i,j)(q) P(B,q), then the contraction over q2, q1, q0 with the
//      1D tables (729 FMA per column for p = 2 instead of 19683 for the rank form); the column is
//      added straight into the CSR values with red.global.add.f64 -- consecutive threads hold
//      consecutive (B, j), i.e. contiguous runs of a CSR row (coalesced);
//   6. F_e[A, i] (thread per (A, i)).
// On uniform meshes (all elements share the 1D tables -- translation invariance of uniform
// B-splines) the test-side tables travel as a __grid_constant__ parameter: immediates in the
// unrolled contraction.
#include <cstdio>
#include <type_traits>

#include "iga_host.h"
#include "pointwise.cuh"

#ifndef IGA_Q1U
#define IGA_Q1U 1   // experiments: unroll factor of the contraction's q1 loop
#endif
#ifndef IGA_HOIST
#define IGA_HOIST 1  // trial 1D values hoisted out of the contraction loops (see tsf_column_3d)
#endif
#ifndef IGA_TAIL
#define IGA_TAIL 1   // split the partial last pass of column tasks over q0 sub-ranges
#endif
#ifndef IGA_DYN
#define IGA_DYN 1    // dynamic element order through a global counter (see the element loop)
#endif
#ifndef IGA_PREF
#define IGA_PREF 1   // next element claimed at the start of the current one (counter latency hidden)
#endif
#ifndef IGA_UFIRST
#define IGA_UFIRST 1  // staging: U_e / Udot_e loads issued before the table / position items (config 8 140.9 -> 138.0 ms, config 5 132.85 -> 132.2 ms)
#endif
#ifndef IGA_RS3
#define IGA_RS3 1    // row starts computed by warps 1.. during phase 3 (uniform knots; one barrier per element fewer)
#endif
#ifndef IGA_BAL
#define IGA_BAL 1   // column tasks dealt round-robin over all threads (phase 5, non-symmetric forms)
#endif

namespace iga {

template <int P>
struct UniTab {
    double t[3][P + 1][3][P + 1];   // [axis][q][k][a]
    double qw[3][P + 1];
    double hp[3];
};

// leading doubles of PH::State that the Jacobian coefficients (dcol) read; 0 => the whole state
template <class PH, class = void> struct PhysJState { static constexpr int value = 0; };
template <class PH> struct PhysJState<PH, std::void_t<decltype(PH::JSTATE)>> { static constexpr int value = PH::JSTATE; };

// ---- fully sum-factorised contraction (FS): compile-time tables ----
// K_IJ[A, B] = sum_q sum_(t,k) P_t(A,q) D_IJ,tk(q) P_k(B,q) with every kind a sum of separable
// terms prod_d T_d[q_d][o_d][a_d] is contracted one axis at a time for test AND trial functions:
//   stage 1 (axis 2):  X1_G[q0 q1][a2 b2] = sum_(tau,kap in G) sum_q2 T2[q2][o2 tau][a2] T2[q2][o2 kap][b2] D_IJ,t(tau)k(kap)(q)
//   stage 2+3 (axes 1, 0):  K_IJ[A, B] = sum_G sum_q0 TT0_G[q0][a0 b0] sum_q1 T1[q1][o1 ta][a1] T1[q1][o1 ka][b1] X1_G[q0 q1][a2 b2]
// where a group G = (test class ta, trial class ka) collects the terms by their (axis-0, axis-1)
// derivative orders.  Every loaded coefficient then feeds 3-9 FMAs held in registers (the
// test-side column form reads the whole D block once per column and point: 1 FMA per load).
template <class L>
struct FsMeta {
    using KS = typename L::KS;
    static constexpr int M = L::M;
    struct Term { int k, o0, o1, o2; };           // kind index (t or kq) and derivative orders
    struct Terms { int n; Term t[16]; };
    static constexpr Terms make_terms(bool test) {
        Terms T{};
        const int nk = test ? L::NTK : L::NQK;
        for (int k = 0; k < nk; k++) {
            const int c = test ? L::tk(k) : L::qk(k);
            for (int s = 0; s < KS::nterms(c); s++) {
                T.t[T.n].k = k;
                T.t[T.n].o0 = KS::ord(c, s, 0);
                T.t[T.n].o1 = KS::ord(c, s, 1);
                T.t[T.n].o2 = KS::ord(c, s, 2);
                T.n++;
            }
        }
        return T;
    }
    static constexpr Terms TT = make_terms(true), QT = make_terms(false);
    struct Cls { int n; int o0[16], o1[16]; };
    static constexpr Cls make_cls(const Terms &T) {
        Cls C{};
        for (int i = 0; i < T.n; i++) {
            bool seen = false;
            for (int c = 0; c < C.n; c++) seen = seen || (C.o0[c] == T.t[i].o0 && C.o1[c] == T.t[i].o1);
            if (!seen) { C.o0[C.n] = T.t[i].o0; C.o1[C.n] = T.t[i].o1; C.n++; }
        }
        return C;
    }
    static constexpr Cls TA = make_cls(TT), KA = make_cls(QT);
    static constexpr int NTA = TA.n, NKA = KA.n, NG = NTA * NKA;
    static constexpr int cls(const Cls &C, int o0, int o1) {
        for (int c = 0; c < C.n; c++) if (C.o0[c] == o0 && C.o1[c] == o1) return c;
        return -1;
    }
    // combos (test term, trial term) of group g = ta * NKA + ka
    static constexpr int ncombo(int g) {
        int n = 0;
        for (int a = 0; a < TT.n; a++)
            for (int b = 0; b < QT.n; b++)
                if (cls(TA, TT.t[a].o0, TT.t[a].o1) == g / NKA && cls(KA, QT.t[b].o0, QT.t[b].o1) == g % NKA) n++;
        return n;
    }
    static constexpr int combo(int g, int c, bool test) {
        int n = 0;
        for (int a = 0; a < TT.n; a++)
            for (int b = 0; b < QT.n; b++)
                if (cls(TA, TT.t[a].o0, TT.t[a].o1) == g / NKA && cls(KA, QT.t[b].o0, QT.t[b].o1) == g % NKA) {
                    if (n == c) return test ? a : b;
                    n++;
                }
        return -1;
    }
    static constexpr int MAXC = [] { int m = 1; for (int g = 0; g < NG; g++) m = ncombo(g) > m ? ncombo(g) : m; return m; }();
    static constexpr int cbase(int g) { int n = 0; for (int x = 0; x < g; x++) n += ncombo(x); return n; }
    static constexpr int NCMB = cbase(NG);              // all (test term, trial term) combos
    // axis-0 order pairs (o0 test, o0 trial): stage 3 sums the groups of one pair first
    struct O0P { int n; int a[16], b[16]; };
    static constexpr O0P make_o0p() {
        O0P P{};
        for (int g = 0; g < NG; g++) {
            const int a = TA.o0[g / NKA], b = KA.o0[g % NKA];
            bool seen = false;
            for (int p = 0; p < P.n; p++) seen = seen || (P.a[p] == a && P.b[p] == b);
            if (!seen) { P.a[P.n] = a; P.b[P.n] = b; P.n++; }
        }
        return P;
    }
    static constexpr O0P PO = make_o0p();
    static constexpr int NO0P = PO.n;
    static constexpr bool in_o0p(int g, int p) { return TA.o0[g / NKA] == PO.a[p] && KA.o0[g % NKA] == PO.b[p]; }
    // compact coefficient index of (i, j, contraction kind c, c2) in the (i, j, c, c2)-ordered list
    static constexpr int eij(int i, int j, int c, int c2) {
        for (int e = 0; e < L::EIJ.n; e++)
            if (L::EIJ.i[e] == i && L::EIJ.j[e] == j && L::EIJ.c[e] == c && L::EIJ.c2[e] == c2) return e;
        return -1;
    }
};

// FS stage-1 coefficient offsets per (I, J) and combo (__grid_constant__); a structurally zero
// coefficient points at a zero slot of every point's row, so one copy of the stage-1 code serves
// all 16 blocks with the same work per warp
template <int NIJ, int NCMB, int NOFF4 = 1>
struct alignas(4) FsTab {
    unsigned char off[NIJ][(NCMB + 3) / 4 * 4];   // stage 1: rows padded to whole words
    unsigned char off4[NOFF4];                     // phase 4: [kq][j][i][t] compact index or 255
};
#ifndef IGA_FS_BS1
#define IGA_FS_BS1 5   // FS loop: the barrier protecting X1 sits inside stage 1, after the arithmetic of its
                       // first IGA_FS_BS1 groups (held in registers; 5 = the first test class) and before
                       // their stores: the coefficient loads and a third of the stage overlap the wait for
                       // the slowest stage-2+3 warp.  Config 5 A/B: 0: 136.45, 1: 134.95, 3: 135.3,
                       // 5: 134.6, 8: 136.6 ms
#endif
#ifndef IGA_FS_ALL
#define IGA_FS_ALL 1   // FS stage 1: all coefficient loads of a block issued before the classes
#endif
#ifndef IGA_FS_P4
#define IGA_FS_P4 1   // FS phase 4: one code copy per trial kind, component j = warp at run time
#endif
#ifndef IGA_FS_TK
#define IGA_FS_TK 1   // stage-1 offsets indexed by (test kind, trial kind): the Laplacian's three trial
                      // terms share one coefficient, loaded once
#endif

#if IGA_FS_BS1 && !IGA_FS_TK
#error "IGA_FS_BS1 needs the IGA_FS_TK form of stage 1"
#endif
// FS is used for the uniform-table kernels whose CTA has one warp per trial component.  On for
// VMS (m = 4, 128 threads).  Neo-Hooke (m = 3) has uniform tables only on periodic meshes (config
// 4 is open: never reached, untested); 3D Cahn-Hilliard (m = 1): A/B config 8 149.9 vs 140.8 ms,
// the column form is kept.  Also tried: X1 in two passes for three CTAs per SM, and
// stage 1 over balanced group sets with the structural zeros skipped -- both slower.
#ifndef IGA_FS_NH
#define IGA_FS_NH 0
#endif
#ifndef IGA_FS_CH
#define IGA_FS_CH 0
#endif
template <class PH> struct FsOk {
    static constexpr bool value = PH::M == 4 || (PH::M == 3 && IGA_FS_NH) || (PH::M == 1 && IGA_FS_CH);
};

template <int P, class PH, bool FS = false>
struct F3 {
    static constexpr bool FSC = FS && P == 2;                  // FS contraction + compact D
    static constexpr int M = PH::M;
    static constexpr int NP1 = P + 1, NQ1 = P + 1, NQ = NQ1 * NQ1 * NQ1, NEN = NP1 * NP1 * NP1;
    static constexpr int NCOMBO = M * M;
    static constexpr int NT = ((NEN * M + 31) / 32) * 32;       // one thread per (B, j): 128 (m=4), 96 (m=3)
    static constexpr int NWARP = NT / 32;
    using L = Lists<PH, 3, MODE_PARAM>;
    using KS = typename L::KS;
    static constexpr int NKS = KS::NKS, NC = KS::NC, NR = L::NR, NTK = L::NTK, NQK = L::NQK;
    static constexpr int DB = (NTK * NQK + 1) / 2 * 2;        // dense block per (i, j), padded even
    // q stride: dense blocks (+2: spread smem banks); FS: the compact (i, j, c, c2) list, odd
    // stride so that the 9 (q0, q1) rows a stage-1 warp reads fall in distinct bank pairs
    static constexpr int DQS = FSC ? ((L::EIJ.n + 1) | 1) : NCOMBO * DB + 2;
    static constexpr int ZSLOT = L::EIJ.n;                   // FS: zero coefficient slot per point
    using State = typename PH::template State<3>;
    static constexpr int STD = (sizeof(State) + 7) / 8;      // doubles per state
    // symmetric element Jacobian (hyperelastic tangent, major symmetry): contract blocks I <= J
#ifndef IGA_NH_SYM
#define IGA_NH_SYM 1
#endif
    static constexpr bool SYMJ = std::is_same<PH, PhysNeoHooke>::value && IGA_NH_SYM;
    // resident CTAs per SM the register budget is sized for (m = 3: 96 threads -> 3 CTAs; m = 1:
    // one-warp CTAs (27 trial functions), 8 per SM)
#ifndef IGA_VMS_MINB
#define IGA_VMS_MINB 2
#endif
#ifndef IGA_NH_MINB
#define IGA_NH_MINB 3
#endif
#ifndef IGA_NH_HOIST
#define IGA_NH_HOIST 0
#endif
    static constexpr int MINB = M == 1 ? 8 : M == 3 ? IGA_NH_MINB : IGA_VMS_MINB;
    // doubles of the per-point state that the Jacobian coefficients read (the leading members;
    // VMS keeps its residual coefficients rN, rG after them): only these go to shared memory
    static constexpr int STJ = PhysJState<PH>::value > 0 ? PhysJState<PH>::value : STD;
    // shared-memory carve-up (in doubles).  Everything that dies before the coefficient blocks are
    // built (field kinds Phi, U_e, Udot_e, residual coefficients, node numbers) overlays the D
    // region: the element's residual F_e is formed before phase 4 for that reason.  VMS fits three
    // CTAs per SM this way (<= 75 KB each).
    static constexpr int O_TAB = 0;                          // [3][NQ1][3][NP1]
    static constexpr int O_QW = O_TAB + 3 * NQ1 * 3 * NP1;   // [3][NQ1]
    static constexpr int O_QX = O_QW + 3 * NQ1;              // [3][NQ1]
    static constexpr int O_HP = O_QX + 3 * NQ1;              // [4]
    static constexpr int O_ST = O_HP + 4;                    // [NQ][STJ]
    static constexpr int O_DV = O_ST + NQ * STJ;             // [NQ]
    static constexpr int O_D = (O_DV + NQ + 1) / 2 * 2;      // [NQ][DQS]  (16-byte aligned)
    static constexpr int O_PHI = O_D;                        // [NQ][M][NKS+1]     } overlay D
    static constexpr int O_U = O_PHI + NQ * M * (NKS + 1);   // [NEN][M]            } (dead before
    static constexpr int O_UD = O_U + NEN * M;               // [NEN][M]            }  phase 4)
    static constexpr int O_RA = O_UD + NEN * M;              // [NR][NQ]            }
    static constexpr int O_NDA = O_RA + NR * NQ;             // long long [NEN]     }
    // FS (IGA_NB3): R and the node numbers overlay the stage-1 output X1 instead of D (X1 is
    // first written after phase 4), so phase 4 needs no barrier after the residual F_e
#ifndef IGA_NB3
#define IGA_NB3 1
#endif
    static constexpr bool RX1 = FSC && IGA_NB3;
    static constexpr int OVL = (RX1 ? O_RA : O_NDA + NEN) - O_D;   // overlay extent
    static constexpr int O_RS = O_D + (NQ * DQS > OVL ? NQ * DQS : OVL);   // long long [NEN*M] row starts
#ifndef IGA_PBS
#define IGA_PBS 0
#endif
    // trial values P_k(B, q) of every (function, point, trial kind) in shared memory (uniform
    // tables only: identical for every element, built once per CTA) instead of per column
    // (A/B: slower at 2 CTAs/SM, and it does not fit three)
    static constexpr bool PBS = IGA_PBS && M == 4;
    static constexpr int O_PB = O_RS + NEN * M;              // [NQ][NQK][NEN]
    // FS stage-1 output X1[J][G][q0 q1][a2 b2] of one test component I; J stride = 4 mod 16
    // doubles so that a stage-2 warp (lanes J fastest, then a2 b2) reads distinct bank pairs
    static constexpr int X1G = NQ1 * NQ1 * NP1 * NP1;
    static constexpr int xjs() {
        if constexpr (FSC) {
            const int n = FsMeta<L>::NG * X1G;
            return n + ((4 - n) % 16 + 16) % 16;
        } else return 0;
    }
    static constexpr int XJS = xjs();
    static constexpr int O_X1 = O_PB + (PBS ? NQ * NQK * NEN : 0);
    static constexpr int O_R = RX1 ? O_X1 : O_RA;
    static constexpr int O_ND = RX1 ? O_X1 + NR * NQ : O_NDA;
    static constexpr int ncmb() {
        if constexpr (FSC) return IGA_FS_TK ? NTK * NQK : FsMeta<L>::NCMB;
        else return 1;
    }
    using FT = FsTab<FSC ? M * M : 1, ncmb(), FSC ? NQK * M * M * NTK : 1>;
    static constexpr size_t SMEM = (size_t)(O_X1 + M * XJS) * sizeof(double);
    // residual only: no coefficient blocks -- row starts (unused) right after the overlay
    static constexpr int O_RS_RES = O_ND + NEN;
    static constexpr size_t SMEM_RES = (size_t)(O_RS_RES + NEN * M) * sizeof(double);
    static_assert(NQ * M * (NKS + 1) <= NQ * DQS, "Phi must fit in the D region");
    static_assert(!RX1 || NR * NQ + NEN <= M * XJS, "R and the node numbers must fit the X1 region");
};

// test-side sum factorisation in 3D of one column (trial function B = (b0,b1,b2), pair ij):
//   Kc[A] = sum_q sum_{tk,qk} P_tk(A,q) D[q][ij][tk][qk] P_qk(B,q)
// Trial values P_qk(B,q) are formed on the fly from the lane's 1D values (smem table).
template <class F, bool UNI, int P>
__device__ __forceinline__ void tsf_column_3d(double (&Kc)[F::NEN], const double *__restrict__ Dsm, int ij,
                                              int b0, int b1, int b2, const double *__restrict__ tab,
                                              const UniTab<P> &ut, const double *__restrict__ pbS,
                                              int q0lo = 0, int q0hi = F::NQ1) {
    using L = typename F::L;
    using KS = typename F::KS;
    constexpr int NP1 = F::NP1, NQ1 = F::NQ1, NEN = F::NEN, NTK = F::NTK, NQK = F::NQK, DB = F::DB;
    // Neo-Hooke runs 3 CTAs/SM at the 168-register cap: hoisting spills there (A/B +6 %)
    constexpr int HOIST = F::M == 3 ? IGA_NH_HOIST : IGA_HOIST;
    auto T = [&](int d, int q, int k, int a) -> double {
        if constexpr (UNI) return ut.t[d][q][k][a];
        else return tab[((d * NQ1 + q) * 3 + k) * NP1 + a];
    };
    auto TS = [&](int d, int q, int k, int a) -> double { return tab[((d * NQ1 + q) * 3 + k) * NP1 + a]; };
    constexpr auto used01 = [](int o0, int o1) {
        for (int t = 0; t < NTK; t++) {
            const int c = L::tk(t);
            for (int s = 0; s < KS::nterms(c); s++)
                if (KS::ord(c, s, 0) == o0 && KS::ord(c, s, 1) == o1) return true;
        }
        return false;
    };
    constexpr auto used0 = [](int o0) {
        for (int t = 0; t < NTK; t++) {
            const int c = L::tk(t);
            for (int s = 0; s < KS::nterms(c); s++)
                if (KS::ord(c, s, 0) == o0) return true;
        }
        return false;
    };
#pragma unroll
    for (int A = 0; A < NEN; A++) Kc[A] = 0.0;
    // trial 1D values of this column along axis 1 for every q1, loaded once (HOIST >= 1:
    // the per-iteration loads at the head of the rolled q1 loop were the kernel's largest
    // single stall, ncu r02a) and along axis 2 (HOIST >= 2)
    double n1all[HOIST >= 1 ? NQ1 : 1][3], n2all[HOIST >= 2 ? NQ1 : 1][3];
    if constexpr (HOIST >= 1) {
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
            for (int k = 0; k < 3; k++) n1all[q][k] = TS(1, q, k, b1);
    }
    if constexpr (HOIST >= 2) {
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
            for (int k = 0; k < 3; k++) n2all[q][k] = TS(2, q, k, b2);
    }
#pragma unroll 1
    for (int q0 = q0lo; q0 < q0hi; q0++) {   // a q0 sub-range: partial column (tail split)
        double n0[3];
#pragma unroll
        for (int k = 0; k < 3; k++) n0[k] = TS(0, q0, k, b0);
        double Tt[3][NP1][NP1];
#pragma unroll
        for (int o = 0; o < 3; o++)
#pragma unroll
            for (int x = 0; x < NP1; x++)
#pragma unroll
                for (int y = 0; y < NP1; y++) Tt[o][x][y] = 0.0;
        // q1 loop rolled: unrolled, VMS spills at 255 registers and Neo-Hooke (168-register cap of
        // 3 CTAs/SM) misses in the instruction cache (A/B: 208 vs 216 ms, 10.1 vs 10.6 ms)
        constexpr int kQ1U = IGA_Q1U;
#pragma unroll kQ1U
        for (int q1 = 0; q1 < NQ1; q1++) {
            double n1[3];
            if constexpr (HOIST >= 1) {
                // q1 is a rolled loop index: select from registers without local-memory indexing
#pragma unroll
                for (int k = 0; k < 3; k++) n1[k] = q1 == 0 ? n1all[0][k] : (q1 == 1 ? n1all[1][k] : n1all[NQ1 - 1][k]);
            } else {
#pragma unroll
                for (int k = 0; k < 3; k++) n1[k] = TS(1, q1, k, b1);
            }
            // trial 2D products n0[o0] n1[o1] once per (q0, q1) (unused orders are dead code)
            double n01[3][3];
#pragma unroll
            for (int o0 = 0; o0 < 3; o0++)
#pragma unroll
                for (int o1 = 0; o1 < 3; o1++) n01[o0][o1] = n0[o0] * n1[o1];
            double S[3][3][NP1];
#pragma unroll
            for (int o = 0; o < 3; o++)
#pragma unroll
                for (int o2 = 0; o2 < 3; o2++)
#pragma unroll
                    for (int x = 0; x < NP1; x++) S[o][o2][x] = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < NQ1; q2++) {
                const int q = (q0 * NQ1 + q1) * NQ1 + q2;
                double n2[3];
                if constexpr (HOIST >= 2) {
#pragma unroll
                    for (int k = 0; k < 3; k++) n2[k] = n2all[q2][k];
                } else if constexpr (!(UNI && F::PBS)) {
#pragma unroll
                    for (int k = 0; k < 3; k++) n2[k] = TS(2, q2, k, b2);
                }
                double pb[NQK];
                if constexpr (UNI && F::PBS) {
#pragma unroll
                    for (int kq = 0; kq < NQK; kq++) pb[kq] = pbS[(q * NQK + kq) * NEN + (b0 * NP1 + b1) * NP1 + b2];
                } else {
                static_for<NQK>([&](auto K) {
                    constexpr int kq = decltype(K)::value;
                    constexpr int c = L::qk(kq);
                    double v = 0.0;
                    static_for<KS::nterms(c)>([&](auto TT) {
                        constexpr int s = decltype(TT)::value;
                        v += n01[KS::ord(c, s, 0)][KS::ord(c, s, 1)] * n2[KS::ord(c, s, 2)];
                    });
                    pb[kq] = v;
                });
                }
                // H[t] = sum_k D[k][t] pb[k]: block rows (trial kind k) streamed 16 bytes at a time
                const double2 *Dq2 = reinterpret_cast<const double2 *>(Dsm + q * F::DQS + ij * DB);
                double H[NTK];
#pragma unroll
                for (int t = 0; t < NTK; t++) H[t] = 0.0;
#pragma unroll
                for (int x = 0; x < DB / 2; x++) {
                    const double2 v2 = Dq2[x];
                    const int e0 = 2 * x, e1 = 2 * x + 1;
                    if (e0 < NTK * NQK) H[e0 % NTK] += v2.x * pb[e0 / NTK];
                    if (e1 < NTK * NQK) H[e1 % NTK] += v2.y * pb[e1 / NTK];
                }
                static_for<NTK>([&](auto TK) {
                    constexpr int t = decltype(TK)::value;
                    constexpr int c = L::tk(t);
                    static_for<KS::nterms(c)>([&](auto TT) {
                        constexpr int s = decltype(TT)::value;
                        constexpr int o0 = KS::ord(c, s, 0), o1 = KS::ord(c, s, 1), o2 = KS::ord(c, s, 2);
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) S[o0][o1][a2] += H[t] * T(2, q2, o2, a2);
                    });
                });
            }
            static_for<3>([&](auto O0) {
                constexpr int o0 = decltype(O0)::value;
                static_for<3>([&](auto O1) {
                    constexpr int o1 = decltype(O1)::value;
                    if constexpr (used01(o0, o1)) {
#pragma unroll
                        for (int a1 = 0; a1 < NP1; a1++) {
                            const double t1 = T(1, q1, o1, a1);
#pragma unroll
                            for (int a2 = 0; a2 < NP1; a2++) Tt[o0][a1][a2] += t1 * S[o0][o1][a2];
                        }
                    }
                });
            });
        }
        static_for<3>([&](auto O0) {
            constexpr int o0 = decltype(O0)::value;
            if constexpr (used0(o0)) {
#pragma unroll
                for (int a0 = 0; a0 < NP1; a0++) {
                    const double t0 = T(0, q0, o0, a0);
#pragma unroll
                    for (int a1 = 0; a1 < NP1; a1++)
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) Kc[(a0 * NP1 + a1) * NP1 + a2] += t0 * Tt[o0][a1][a2];
                }
            }
        });
    }
}

// FS stage 1 (axis 2) for test component I and trial component J = warp: lane = (q0 q1, a2),
// 3 accumulators (b2) per group G; the coefficient of combo c of block (I, J) sits at offset
// ft.off[I M + J][c] of every point's compact row (the zero slot if it is structurally zero).
//   X1[J][G][q0 q1][a2 b2] = sum_(tau, kap in G) sum_q2 T2[q2][o2 tau][a2] T2[q2][o2 kap][b2] D_IJ(q)
// Every loaded coefficient feeds one DMUL and three DFMAs.
template <class F, int P>
__device__ __forceinline__ void fs_stage1(int I, int J, const double *__restrict__ sD, const double *__restrict__ sTab,
                                          double *__restrict__ sX1, const UniTab<P> &ut, const typename F::FT &ft,
                                          int lane_, bool bar = false) {
    using FM = FsMeta<typename F::L>;
    constexpr int NQ1 = F::NQ1, NP1 = F::NP1, NQQ = NQ1 * NQ1, NAB = NP1 * NP1;
#if IGA_FS_BS1
    // every lane runs the stage (idle lanes on lane 0's operands, stores predicated) so that the
    // CTA barrier protecting X1 can sit between the first group's arithmetic and its stores
    const bool act = lane_ < NQQ * NP1;
    const int lane = act ? lane_ : 0;
#else
    const int lane = lane_;
    constexpr bool act = true;
    if (lane >= NQQ * NP1) return;
#endif
    const int q01 = lane / NP1, a2 = lane - q01 * NP1;
    double t2a[NQ1][3];                                  // test values on axis 2 (unused orders are dead)
#pragma unroll
    for (int q2 = 0; q2 < NQ1; q2++)
#pragma unroll
        for (int o = 0; o < 3; o++) t2a[q2][o] = sTab[((2 * NQ1 + q2) * 3 + o) * NP1 + a2];
    const double *Dq = sD + q01 * NQ1 * F::DQS;
    const unsigned char *off = ft.off[I * F::M + J];
    double *dst = sX1 + J * F::XJS + q01 * NAB + a2 * NP1;
#if IGA_FS_TK
    // per test class: each (test term, trial kind) coefficient at the three q2 loaded once into
    // registers (the Laplacian's three trial terms share it), then the class's groups
#if IGA_FS_ALL
    // all of the block's coefficients issued up front (60 loads for VMS), then the classes
    double dv[FM::TT.n][F::NQK][NQ1];
    static_for<FM::TT.n>([&](auto TU) {
        constexpr int tu = decltype(TU)::value;
        static_for<F::NQK>([&](auto KQ) {
            constexpr int kq = decltype(KQ)::value;
            const int e = off[FM::TT.t[tu].k * F::NQK + kq];
#pragma unroll
            for (int q2 = 0; q2 < NQ1; q2++) dv[tu][kq][q2] = Dq[q2 * F::DQS + e];
        });
    });
#endif
#if IGA_FS_BS1
    static_assert(IGA_FS_BS1 <= FM::NG, "IGA_FS_BS1: groups held before the barrier");
    double hold[IGA_FS_BS1][NP1];
#endif
    static_for<FM::NTA>([&](auto TAC) {
        constexpr int ta = decltype(TAC)::value;
#if !IGA_FS_ALL
        double dv[FM::TT.n][F::NQK][NQ1];
        static_for<FM::TT.n>([&](auto TU) {
            constexpr int tu = decltype(TU)::value;
            if constexpr (FM::cls(FM::TA, FM::TT.t[tu].o0, FM::TT.t[tu].o1) == ta) {
                static_for<F::NQK>([&](auto KQ) {
                    constexpr int kq = decltype(KQ)::value;
                    const int e = off[FM::TT.t[tu].k * F::NQK + kq];
#pragma unroll
                    for (int q2 = 0; q2 < NQ1; q2++) dv[tu][kq][q2] = Dq[q2 * F::DQS + e];
                });
            }
        });
#endif
        static_for<FM::NKA>([&](auto KAC) {
            constexpr int g = ta * FM::NKA + decltype(KAC)::value;
            double acc[NP1];
#pragma unroll
            for (int b2 = 0; b2 < NP1; b2++) acc[b2] = 0.0;
            // every (test term, trial term) pair of the class pair is a combo (structural zeros
            // read the zero slot): per trial term, sum over the test terms first
            static_for<FM::QT.n>([&](auto KB) {
                constexpr int kb = decltype(KB)::value;
                if constexpr (FM::cls(FM::KA, FM::QT.t[kb].o0, FM::QT.t[kb].o1) == decltype(KAC)::value) {
                    constexpr int ok = FM::QT.t[kb].o2, kq = FM::QT.t[kb].k;
#pragma unroll
                    for (int q2 = 0; q2 < NQ1; q2++) {
                        double y = 0.0;
                        static_for<FM::TT.n>([&](auto TU) {
                            constexpr int tu = decltype(TU)::value;
                            if constexpr (FM::cls(FM::TA, FM::TT.t[tu].o0, FM::TT.t[tu].o1) == ta)
                                y += dv[tu][kq][q2] * t2a[q2][FM::TT.t[tu].o2];
                        });
#pragma unroll
                        for (int b2 = 0; b2 < NP1; b2++) acc[b2] += y * ut.t[2][q2][ok][b2];
                    }
                }
            });
#if IGA_FS_BS1
            // the first IGA_FS_BS1 groups are held in registers until the barrier
            if constexpr (g < IGA_FS_BS1) {
#pragma unroll
                for (int b2 = 0; b2 < NP1; b2++) hold[g][b2] = acc[b2];
                if constexpr (g == IGA_FS_BS1 - 1) {
                    if (bar) __syncthreads();            // all stage-2+3 reads of the previous X1 are done
                    if (act) {
#pragma unroll
                        for (int h = 0; h < IGA_FS_BS1; h++)
#pragma unroll
                            for (int b2 = 0; b2 < NP1; b2++) dst[h * NQQ * NAB + b2] = hold[h][b2];
                    }
                }
            } else
#endif
            if (act) {
#pragma unroll
                for (int b2 = 0; b2 < NP1; b2++) dst[g * NQQ * NAB + b2] = acc[b2];
            }
        });
    });
    (void)FM::NCMB;
#else
    static_for<FM::NG>([&](auto GG) {
        constexpr int g = decltype(GG)::value;
        double acc[NP1];
#pragma unroll
        for (int b2 = 0; b2 < NP1; b2++) acc[b2] = 0.0;
        static_for<FM::ncombo(g)>([&](auto CC) {
            constexpr int c = decltype(CC)::value;
            constexpr int ta = FM::combo(g, c, true), kb = FM::combo(g, c, false);
            constexpr int ot = FM::TT.t[ta].o2, ok = FM::QT.t[kb].o2;
            const int e = off[IGA_FS_TK ? FM::TT.t[ta].k * F::NQK + FM::QT.t[kb].k : FM::cbase(g) + c];
#pragma unroll
            for (int q2 = 0; q2 < NQ1; q2++) {
                const double x = Dq[q2 * F::DQS + e] * t2a[q2][ot];
#pragma unroll
                for (int b2 = 0; b2 < NP1; b2++) acc[b2] += x * ut.t[2][q2][ok][b2];
            }
        });
#pragma unroll
        for (int b2 = 0; b2 < NP1; b2++) dst[g * NQQ * NAB + b2] = acc[b2];
    });
#endif
}

// FS stages 2 + 3 (axes 1 and 0) for test component I: task (J, a2 b2, a1), J fastest (4
// consecutive lanes fill one 32-byte sector of a CSR row), K[a0][b0][b1] in registers:
//   z_p[b1]    = sum_(G in p) sum_q1 T1[q1][o1 ta][a1] T1[q1][o1 ka][b1] X1_G[q0 q1][a2 b2]
//   y_oa[b0 b1] = sum_(p: test o0 = oa) T0[q0][o0 trial p][b0] z_p[b1]
//   K[a0 b0 b1] += T0[q0][oa][a0] y_oa[b0 b1]          (per q0)
// then each value is added into its CSR position with red.global.add.f64.
template <class F, int P>
__device__ __forceinline__ void fs_stage23(int I, int tid, const double *__restrict__ sX1, const double *__restrict__ sTab,
                                           const int *sPosE, const int *sW, const long long *sRS, double *__restrict__ val,
                                           const UniTab<P> &ut, int dbg) {
    using FM = FsMeta<typename F::L>;
    constexpr int M = F::M, NQ1 = F::NQ1, NP1 = F::NP1, NQQ = NQ1 * NQ1, NAB = NP1 * NP1, NKA = FM::NKA;
#pragma unroll 1
    for (int task = tid; task < M * NAB * NP1; task += F::NT) {
        const int J = task % M, r = task / M, ab2 = r % NAB, a1 = r / NAB;
        const int a2 = ab2 / NP1, b2 = ab2 - a2 * NP1;
        double t1a[NQ1][3];                              // test values on axis 1 (unused orders are dead)
#pragma unroll
        for (int q1 = 0; q1 < NQ1; q1++)
#pragma unroll
            for (int o = 0; o < 3; o++) t1a[q1][o] = sTab[((1 * NQ1 + q1) * 3 + o) * NP1 + a1];
        double K[NP1][NP1][NP1];
#pragma unroll
        for (int x = 0; x < NP1 * NP1 * NP1; x++) (&K[0][0][0])[x] = 0.0;
        const double *X = sX1 + J * F::XJS + ab2;
        static_for<NQ1>([&](auto Q0) {
            constexpr int q0 = decltype(Q0)::value;
            static_for<3>([&](auto OA) {                   // test derivative order on axis 0
                constexpr int oa = decltype(OA)::value;
                constexpr bool used = [] { for (int p = 0; p < FM::NO0P; p++) if (FM::PO.a[p] == oa) return true; return false; }();
                if constexpr (used) {
                    double y[NP1][NP1];
#pragma unroll
                    for (int x = 0; x < NP1 * NP1; x++) (&y[0][0])[x] = 0.0;
                    static_for<FM::NO0P>([&](auto PP) {
                        constexpr int pp = decltype(PP)::value;
                        if constexpr (FM::PO.a[pp] == oa) {
                            double z[NP1];
#pragma unroll
                            for (int b1 = 0; b1 < NP1; b1++) z[b1] = 0.0;
                            // per trial class of this pair and q1: the test classes (with their
                            // axis-1 test value) summed before the trial table
                            static_for<NKA>([&](auto KAC) {
                                constexpr int ka = decltype(KAC)::value;
                                if constexpr (FM::KA.o0[ka] == FM::PO.b[pp]) {
                                    constexpr int ob1 = FM::KA.o1[ka];
#pragma unroll
                                    for (int q1 = 0; q1 < NQ1; q1++) {
                                        double x = 0.0;
                                        static_for<FM::NTA>([&](auto TAC) {
                                            constexpr int ta = decltype(TAC)::value;
                                            if constexpr (FM::TA.o0[ta] == oa) {
                                                constexpr int g = ta * NKA + ka, oa1 = FM::TA.o1[ta];
                                                x += X[(g * NQQ + q0 * NQ1 + q1) * NAB] * t1a[q1][oa1];
                                            }
                                        });
#pragma unroll
                                        for (int b1 = 0; b1 < NP1; b1++) z[b1] += x * ut.t[1][q1][ob1][b1];
                                    }
                                }
                            });
                            constexpr int ob0 = FM::PO.b[pp];
#pragma unroll
                            for (int b0 = 0; b0 < NP1; b0++)
#pragma unroll
                                for (int b1 = 0; b1 < NP1; b1++) y[b0][b1] += ut.t[0][q0][ob0][b0] * z[b1];
                        }
                    });
#pragma unroll
                    for (int a0 = 0; a0 < NP1; a0++)
#pragma unroll
                        for (int x = 0; x < NP1 * NP1; x++) (&K[a0][0][0])[x] += ut.t[0][q0][oa][a0] * (&y[0][0])[x];
                }
            });
        });
        if (!(dbg & 2)) {
            // CSR position of (A, B) in row (A, I): ((pos0 W1 + pos1) W2 + pos2) nodes
            const int W1a = sW[NP1 + a1], W2a = sW[2 * NP1 + a2];
            const int P2ab = sPosE[2 * NP1 * NP1 + a2 * NP1 + b2];
            int P1b[NP1];
#pragma unroll
            for (int b1 = 0; b1 < NP1; b1++) P1b[b1] = sPosE[NP1 * NP1 + a1 * NP1 + b1];
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) {
                const long long rs = sRS[((a0 * NP1 + a1) * NP1 + a2) * M + I] + J;
#pragma unroll
                for (int b0 = 0; b0 < NP1; b0++) {
                    const int p0 = sPosE[a0 * NP1 + b0];
#pragma unroll
                    for (int b1 = 0; b1 < NP1; b1++) {
                        const int co = (p0 * W1a + P1b[b1]) * W2a + P2ab;
                        atomicAdd(val + rs + (long long)co * M, K[a0][b0][b1]);
                    }
                }
            }
        } else {
            double sum = 0.0;
#pragma unroll
            for (int x = 0; x < NP1 * NP1 * NP1; x++) sum += (&K[0][0][0])[x];
            if (sum == 1.2345e300) val[0] = sum;
        }
    }
}

#ifndef IGA_FS
#define IGA_FS 1    // fully sum-factorised contraction for the uniform-table VMS Jacobian (0: column form)
#endif
template <int P, class PH, bool JAC, bool UNI>
using F3K = F3<P, PH, JAC && UNI && FsOk<PH>::value && IGA_FS>;

template <int P, class PH, bool JAC, bool UNI>
__global__ void __launch_bounds__(F3<P, PH>::NT, JAC ? F3<P, PH>::MINB : (F3<P, PH>::M == 1 ? 16 : 8))   // residual-only: A/B 4 -> 8 = -15 % / -12 % (configs 4 / 5); m = 1: 16 (-10 %)
k_fused3d(SpaceDev s, Prm prm, double a, double b, const double *__restrict__ U, const double *__restrict__ Ud,
          double *__restrict__ val, double *__restrict__ Fout, long long nelem, const __grid_constant__ UniTab<P> ut,
          const __grid_constant__ typename F3K<P, PH, JAC, UNI>::FT ft, int dbg, int bw) {
    using F = F3K<P, PH, JAC, UNI>;
    constexpr int NTH = F::NT, NWP = F::NWARP;
    using L = typename F::L;
    using KS = typename F::KS;
    using State = typename F::State;
    constexpr int M = F::M, NP1 = F::NP1, NQ1 = F::NQ1, NQ = F::NQ, NEN = F::NEN;
    constexpr int NKS = F::NKS, NR = F::NR, NTK = F::NTK, NQK = F::NQK, DB = F::DB;
    extern __shared__ __align__(16) double sm[];
    double *sU = sm + F::O_U, *sUd = sm + F::O_UD, *sTab = sm + F::O_TAB, *sQW = sm + F::O_QW, *sQX = sm + F::O_QX;
    double *sHP = sm + F::O_HP, *sPhi = sm + F::O_PHI, *sDV = sm + F::O_DV, *sR = sm + F::O_R, *sD = sm + F::O_D;
    double *sStd = sm + F::O_ST;                             // [NQ][STJ] leading state doubles
    // [NEN*M] CSR row (A, i): offset of its first value from `val`, in doubles.  Halo rows live in
    // the halo buffer; their offsets are taken in the flat 64-bit address space (both arrays are
    // 8-byte aligned) so the scatter below addresses everything from the uniform `val` register.
    long long *sRS = reinterpret_cast<long long *>(sm + (JAC ? F::O_RS : F::O_RS_RES));
    long long *sNode = reinterpret_cast<long long *>(sm + F::O_ND); // [NEN] touched-box node (overlays D)
    __shared__ int sG[3 * NP1], sW[3 * NP1], sPosE[3 * NP1 * NP1], sSeg[3 * NP1];
    __shared__ long long sS[3 * NP1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int errbits = 0;
    const int n0 = s.ax[0].el_hi - s.ax[0].el_lo, n1 = s.ax[1].el_hi - s.ax[1].el_lo, n2 = s.ax[2].el_hi - s.ax[2].el_lo;
    auto TB = [&](int d, int q, int k, int aa) -> double {
        if constexpr (UNI) return ut.t[d][q][k][aa];
        else return sTab[((d * NQ1 + q) * 3 + k) * NP1 + aa];
    };

    const bool uni_knots = s.ax[0].uniform && s.ax[1].uniform && s.ax[2].uniform;
    if constexpr (JAC && UNI && F::PBS) {
        // P_k(B, q) = sum over the separable terms of kind k of T0 T1 T2 (the element-independent
        // uniform tables), once per CTA; read per column in the contraction
        double *pbS = sm + F::O_PB;
        for (int i = tid; i < NQ * NQK * NEN; i += NTH) {
            const int B = i % NEN, kq = (i / NEN) % NQK, q = i / (NEN * NQK);
            const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
            const int b0 = B / (NP1 * NP1), b1 = (B / NP1) % NP1, b2 = B % NP1;
            double v = 0.0;
            static_for<NQK>([&](auto K) {
                constexpr int kk = decltype(K)::value;
                constexpr int c = L::qk(kk);
                if (kk == kq) {
                    static_for<KS::nterms(c)>([&](auto TT) {
                        constexpr int t = decltype(TT)::value;
                        v += ut.t[0][q0][KS::ord(c, t, 0)][b0] * ut.t[1][q1][KS::ord(c, t, 1)][b1] *
                             ut.t[2][q2][KS::ord(c, t, 2)][b2];
                    });
                }
            });
            pbS[i] = v;
        }
        __syncthreads();
    }
    // Dynamic element order (IGA_DYN): after its first element a CTA takes the next unprocessed one
    // from a global counter, so all CTAs stay on consecutive elements of the L2-blocked order and
    // the CSR rows they add into stay L2-resident (a static stride lets the 296 CTAs drift apart by
    // hundreds of pencils over ~7000 elements each: DRAM traffic was independent of bw, 5.8-6.8x
    // the algorithmic bytes).
    __shared__ long long sEl;
    // IGA_PREF on the FS kernel only (3D Cahn-Hilliard: A/B 147.0 vs 140.8 ms with it)
    constexpr bool PREF = IGA_PREF && F::FSC;
    long long nxt = 0;
    for (long long el = blockIdx.x; el < nelem;) {
        // IGA_PREF: claim the next element now; the counter's round trip overlaps this element
        if (IGA_DYN && PREF && tid == 0) nxt = (long long)gridDim.x + (long long)atomicAdd(s.wq, 1ULL);
        // L2-blocked element order: pencils along axis 2, swept over axis 0 inside blocks of `bw`
        // pencils along axis 1, so the CSR rows an element layer leaves half-accumulated are
        // still in L2 when the next layer adds to them (the red.add scatter then reads each
        // row from HBM about once)
        int e[3];
        {
            const long long r = el / n2;
            e[2] = s.ax[2].el_lo + (int)(el - r * n2);
            const long long blk = (long long)n0 * bw;
            const int e1b = (int)(r / blk);
            const int bwe = min(bw, n1 - e1b * bw);
            const int rem = (int)(r - e1b * blk);
            e[0] = s.ax[0].el_lo + rem / bwe;
            e[1] = s.ax[1].el_lo + e1b * bw + rem % bwe;
        }
        auto EL = [&](int d) { return d == 0 ? e[0] : (d == 1 ? e[1] : e[2]); };   // no local-memory indexing
        // ---- 1. stage: tables, per-axis function data, position tables, and (uniform knots:
        //         first[e] = first0 + e, no dependent load) U_e -- one global round trip ----
#if IGA_UFIRST
        // the U_e / Udot_e loads are issued first, into registers, and stored after the loop: the
        // loop's own global loads (positions, row widths, segment prefixes) share their round trip
        // instead of preceding it
        static_assert(NEN * M <= NTH, "one U_e entry per thread");
        const int nU1 = 0;
        const bool uld = uni_knots && tid < NEN * M;
        double pu = 0.0, pud = 0.0;
        if (uld) {
            const int A = tid / M, m = tid - A * M;
            int g[3];
#pragma unroll
            for (int d = 0; d < 3; d++) {
                const int aa = d == 0 ? A / (NP1 * NP1) : d == 1 ? (A / NP1) % NP1 : A % NP1;
                g[d] = s.ax[d].first0 + EL(d) + aa;
                if (g[d] >= s.ax[d].nu) g[d] -= s.ax[d].nu;
            }
            const long long node = local_node(s, g[0], g[1], g[2]);
            pu = U[node * M + m];
            pud = Ud ? Ud[node * M + m] : 0.0;
        }
#else
        const int nU1 = uni_knots ? NEN * M : 0;
#endif
        for (int i = tid; i < 3 * NQ1 * 3 * NP1 + 6 * NQ1 + 3 + 3 * NP1 + 3 * NP1 * NP1 + nU1; i += NTH) {
            int k = i;
            if (k < 3 * NQ1 * 3 * NP1) {
                const int d = k / (NQ1 * 3 * NP1), r = k % (NQ1 * 3 * NP1);
                if constexpr (UNI) sTab[k] = (&ut.t[0][0][0][0])[k];
                else sTab[k] = s.ax[d].tab[(size_t)EL(d) * NQ1 * 3 * NP1 + r];
                continue;
            }
            k -= 3 * NQ1 * 3 * NP1;
            if (k < 6 * NQ1) {
                const int w = k / (3 * NQ1), r = k % (3 * NQ1), d = r / NQ1, q = r % NQ1;
                if (w == 0) {
                    if constexpr (UNI) sQW[r] = ut.qw[d][q];
                    else sQW[r] = s.ax[d].qw[(size_t)EL(d) * NQ1 + q];
                } else sQX[r] = s.ax[d].qx[(size_t)EL(d) * NQ1 + q];
                continue;
            }
            k -= 6 * NQ1;
            if (k < 3) {
                if constexpr (UNI) sHP[k] = ut.hp[k];
                else sHP[k] = s.ax[k].hpar[EL(k)];
                continue;
            }
            k -= 3;
            if (k < 3 * NP1 * NP1) {
                const int d = k / (NP1 * NP1);
                sPosE[k] = s.ax[d].pos[(size_t)EL(d) * NP1 * NP1 + k % (NP1 * NP1)];
                continue;
            }
            k -= 3 * NP1 * NP1;
            if (k >= 3 * NP1) {
                k -= 3 * NP1;
                const int A = k / M, m = k - A * M;
                int g[3];
#pragma unroll
                for (int d = 0; d < 3; d++) {
                    const int aa = d == 0 ? A / (NP1 * NP1) : d == 1 ? (A / NP1) % NP1 : A % NP1;
                    g[d] = s.ax[d].first0 + EL(d) + aa;
                    if (g[d] >= s.ax[d].nu) g[d] -= s.ax[d].nu;
                }
                const long long node = local_node(s, g[0], g[1], g[2]);
                sU[k] = U[node * M + m];
                sUd[k] = Ud ? Ud[node * M + m] : 0.0;
                continue;
            }
            {
                const int d = k / NP1, aa = k % NP1;
                int g = (s.ax[d].uniform ? s.ax[d].first0 + EL(d) : s.ax[d].first[EL(d)]) + aa;
                if (g >= s.ax[d].nu) g -= s.ax[d].nu;
                sG[k] = g;
                sW[k] = s.ax[d].rowW[g];
                const int l = local_fn(s.ax[d], g);
                sS[k] = s.ax[d].lS[l];
                sSeg[k] = l >= s.ax[d].n_own;
            }
        }
#if IGA_UFIRST
        if (uld) {
            sU[tid] = pu;
            sUd[tid] = pud;
        }
#endif
        __syncthreads();
        // node numbers and closed-form row starts (and U_e on non-uniform knots).  IGA_RS3 with
        // uniform knots: nothing before phase 3b reads them, so warps 1.. compute them during
        // phase 3 (whose 27 points occupy warp 0 only) and the barrier after this pass is dropped
        constexpr bool RS3 = IGA_RS3 && NTH > 32;
        auto row_starts = [&](int i0, int stride) {
            for (int i = i0; i < NEN * M; i += stride) {
                {
                    const int k = i, A = k / M, m = k - A * M;
                    const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
                    const long long node = local_node(s, sG[a0], sG[NP1 + a1], sG[2 * NP1 + a2]);
                    if (!uni_knots) {
                        sU[k] = U[node * M + m];
                        sUd[k] = Ud ? Ud[node * M + m] : 0.0;
                    }
                    if (m == 0) {
                        // closed-form row start (iga_internal.cuh row_start) from the staged
                        // per-axis segment prefixes
                        sNode[A] = node;
                        const int s0 = sSeg[a0], s1 = sSeg[NP1 + a1], s2 = sSeg[2 * NP1 + a2];
                        const long long T1 = s1 ? s.ax[1].Th : s.ax[1].T, T2 = s2 ? s.ax[2].Th : s.ax[2].T;
                        const long long W0 = sW[a0], W1 = sW[NP1 + a1], W2 = sW[2 * NP1 + a2];
                        const int sub = (s0 * 2 + s1) * 2 + s2;
                        long long base = (long long)M * M * (sS[a0] * T1 * T2 + W0 * sS[NP1 + a1] * T2 + W0 * W1 * sS[2 * NP1 + a2]);
                        if (sub) base += ((long long)(uintptr_t)(s.halo + s.hbase[sub]) - (long long)(uintptr_t)val) / 8;
                        const long long Wn = W0 * W1 * W2;
#pragma unroll
                        for (int ii = 0; ii < M; ii++) sRS[A * M + ii] = base + ii * Wn * M;
                    }
                }
            }
        };
        if (!(RS3 && uni_knots)) {
            row_starts(tid, NTH);
            __syncthreads();
        }

        // ---- 2. field kinds per (q, m), sum factorised over the element's functions:
        //         Phi_k(q) = sum_a0 T0 (sum_a1 T1 (sum_a2 T2 U)) per separable term of kind k ----
        for (int task = (dbg & 4) ? NQ * M : tid; task < NQ * M; task += NTH) {
            const int q = task / M, m = task % M;
            const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
            double v0[3][NP1], v1[3][NP1], v2[3][NP1];
#pragma unroll
            for (int k = 0; k < 3; k++)
#pragma unroll
                for (int x = 0; x < NP1; x++) {
                    v0[k][x] = sTab[((0 * NQ1 + q0) * 3 + k) * NP1 + x];
                    v1[k][x] = sTab[((1 * NQ1 + q1) * 3 + k) * NP1 + x];
                    v2[k][x] = sTab[((2 * NQ1 + q2) * 3 + k) * NP1 + x];
                }
            // stage a2: s2[a0][a1][o2] (and the Udot value, order 0 only)
            double s2[NP1][NP1][3], d2[NP1][NP1];
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++)
#pragma unroll
                for (int a1 = 0; a1 < NP1; a1++) {
                    double u[NP1];
#pragma unroll
                    for (int a2 = 0; a2 < NP1; a2++) u[a2] = sU[((a0 * NP1 + a1) * NP1 + a2) * M + m];
#pragma unroll
                    for (int o = 0; o < 3; o++) {
                        double t = 0.0;
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) t += v2[o][a2] * u[a2];
                        s2[a0][a1][o] = t;
                    }
                    double t = 0.0;
                    if constexpr (PH::UDOT) {
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) t += v2[0][a2] * sUd[((a0 * NP1 + a1) * NP1 + a2) * M + m];
                    }
                    d2[a0][a1] = t;
                }
            // stage a1: s1[a0][o1][o2] (unused order pairs are dead code)
            double s1[NP1][3][3], d1[NP1];
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) {
#pragma unroll
                for (int o1 = 0; o1 < 3; o1++)
#pragma unroll
                    for (int o2 = 0; o2 < 3; o2++) {
                        double t = 0.0;
#pragma unroll
                        for (int a1 = 0; a1 < NP1; a1++) t += v1[o1][a1] * s2[a0][a1][o2];
                        s1[a0][o1][o2] = t;
                    }
                double t = 0.0;
#pragma unroll
                for (int a1 = 0; a1 < NP1; a1++) t += v1[0][a1] * d2[a0][a1];
                d1[a0] = t;
            }
            double *dst = sPhi + (q * M + m) * (NKS + 1);
            static_for<NKS>([&](auto K) {
                constexpr int k = decltype(K)::value;
                double pv = 0.0;
                static_for<KS::nterms(k)>([&](auto TT) {
                    constexpr int t = decltype(TT)::value;
                    constexpr int o0 = KS::ord(k, t, 0), o1 = KS::ord(k, t, 1), o2 = KS::ord(k, t, 2);
#pragma unroll
                    for (int a0 = 0; a0 < NP1; a0++) pv += v0[o0][a0] * s1[a0][o1][o2];
                });
                dst[k] = pv;
            });
            double pt = 0.0;
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) pt += v0[0][a0] * d1[a0];
            dst[NKS] = pt;
        }
        __syncthreads();

        // ---- 3. per-point state + residual coefficients ----
        if (RS3 && uni_knots && tid >= 32) row_starts(tid - 32, NTH - 32);
        if (tid < NQ && !(dbg & 8)) {
            const int q = tid;
            const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
            Fields<3, M> Fq;
#pragma unroll
            for (int m = 0; m < M; m++) {
                const double *ph = sPhi + (q * M + m) * (NKS + 1);
                Fq.u[m] = ph[0];
#pragma unroll
                for (int i = 0; i < 3; i++) Fq.gu[m][i] = ph[1 + i];
                Fq.lu[m] = PH::HESS ? ph[NKS - 1] : 0.0;
                Fq.ut[m] = ph[NKS];
            }
            const int qq[3] = {q0, q1, q2};
#pragma unroll
            for (int i = 0; i < 3; i++) {
                Fq.x[i] = sQX[i * NQ1 + qq[i]];
                Fq.hpar[i] = sHP[i];
#pragma unroll
                for (int j = 0; j < 3; j++) Fq.dxi[i][j] = (i == j) ? 1.0 : 0.0;
            }
            const double dV = sQW[q0] * sQW[NQ1 + q1] * sQW[2 * NQ1 + q2];
            State st;
            PH::template prepare<3>(prm.p, Fq, st);
            {
                const double *src = reinterpret_cast<const double *>(&st);
#pragma unroll
                for (int k = 0; k < F::STJ; k++) sStd[q * F::STJ + k] = src[k];
            }
            sDV[q] = dV;
            if (Fout) {
                double r[NKS * M];
                PH::template residual<3>(st, r);
                double chk = 0.0;
                static_for<NR>([&](auto RR) {
                    constexpr int rr = decltype(RR)::value;
                    constexpr int c = L::R.c[rr], i = L::R.i[rr];
                    const double v = r[c * M + i] * dV;
                    chk += v;
                    sR[rr * NQ + q] = v;
                });
                if (!isfinite(chk)) errbits |= 2;
            }
        }
        __syncthreads();

        // ---- 3b. residual F_e[A, i] (formed before phase 4: R and the node numbers overlay D):
        //         warp = component i (warp-uniform), lane = A; sum factorised per test kind:
        //         sum_q0 T0 (sum_q1 T1 (sum_q2 T2 r(q))) ----
        if (Fout && warp < M && lane < NEN && !(dbg & 32)) {
            const int A = lane;
            const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
            double t0[NQ1][3], t1[NQ1][3], t2[NQ1][3];
#pragma unroll
            for (int q = 0; q < NQ1; q++)
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    t0[q][k] = sTab[((0 * NQ1 + q) * 3 + k) * NP1 + a0];
                    t1[q][k] = sTab[((1 * NQ1 + q) * 3 + k) * NP1 + a1];
                    t2[q][k] = sTab[((2 * NQ1 + q) * 3 + k) * NP1 + a2];
                }
            // residual kinds common to all components (r~ entry rr = rbase(c) + i): one code copy
            // with I = warp at run time (IGA_FS_P4), else one copy per component
            constexpr bool RUNI = [] {
                for (int c = 0; c < KS::NC; c++) {
                    int n = 0;
                    for (int i = 0; i < M; i++) n += L::crmask(c, i);
                    if (n != 0 && n != M) return false;
                }
                for (int r = 0; r < NR; r++) {
                    int base = 0;
                    for (int c = 0; c < L::R.c[r]; c++) base += L::crmask(c, 0) ? M : 0;
                    if (r != base + L::R.i[r]) return false;
                }
                return true;
            }();
            if constexpr (RUNI && IGA_FS_P4 && F::FSC) {
                const int I = warp;
                double acc = 0.0;
                static_for<KS::NC>([&](auto CC) {
                    constexpr int c = decltype(CC)::value;
                    if constexpr (L::crmask(c, 0)) {
                        constexpr int rb = [] { int b = 0; for (int x = 0; x < c; x++) b += L::crmask(x, 0) ? M : 0; return b; }();
                        const double *Rr = sR + (rb + I) * NQ;
                        static_for<KS::nterms(c)>([&](auto TT) {
                            constexpr int t = decltype(TT)::value;
                            constexpr int o0 = KS::ord(c, t, 0), o1 = KS::ord(c, t, 1), o2 = KS::ord(c, t, 2);
#pragma unroll
                            for (int q0 = 0; q0 < NQ1; q0++) {
                                double s1 = 0.0;
#pragma unroll
                                for (int q1 = 0; q1 < NQ1; q1++) {
                                    double s2 = 0.0;
#pragma unroll
                                    for (int q2 = 0; q2 < NQ1; q2++) s2 += t2[q2][o2] * Rr[(q0 * NQ1 + q1) * NQ1 + q2];
                                    s1 += t1[q1][o1] * s2;
                                }
                                acc += t0[q0][o0] * s1;
                            }
                        });
                    }
                });
                atomicAdd(Fout + sNode[A] * M + I, acc);
            } else
            static_for<M>([&](auto II) {
                constexpr int I = decltype(II)::value;
                if (warp == I) {
                    double acc = 0.0;
                    static_for<NR>([&](auto RR) {
                        constexpr int rr = decltype(RR)::value;
                        constexpr int c = L::R.c[rr];
                        if constexpr (L::R.i[rr] == I) {
                            static_for<KS::nterms(c)>([&](auto TT) {
                                constexpr int t = decltype(TT)::value;
                                constexpr int o0 = KS::ord(c, t, 0), o1 = KS::ord(c, t, 1), o2 = KS::ord(c, t, 2);
#pragma unroll
                                for (int q0 = 0; q0 < NQ1; q0++) {
                                    double s1 = 0.0;
#pragma unroll
                                    for (int q1 = 0; q1 < NQ1; q1++) {
                                        double s2 = 0.0;
#pragma unroll
                                        for (int q2 = 0; q2 < NQ1; q2++)
                                            s2 += t2[q2][o2] * sR[rr * NQ + (q0 * NQ1 + q1) * NQ1 + q2];
                                        s1 += t1[q1][o1] * s2;
                                    }
                                    acc += t0[q0][o0] * s1;
                                }
                            });
                        }
                    });
                    atomicAdd(Fout + sNode[A] * M + I, acc);
                }
            });
        }
        if constexpr (JAC && !F::RX1) __syncthreads();   // F_e read R / sNode: both overlay D

        // ---- 4. Jacobian coefficients: warp-uniform trial column (k2 = qk(kq), j), lane = q ----
        if constexpr (JAC) {
            if constexpr (F::FSC) {
                if (tid < NQ) sD[tid * F::DQS + F::ZSLOT] = 0.0;   // FS zero slot (the region overlays phase 2-3 data)
            }
            // warp w owns the columns kj = w, w + NWARP, ...: the state stays in registers
            if (lane < NQ && !(dbg & 16)) {
                const int q = lane;
                State st;
                {
                    double *dst = reinterpret_cast<double *>(&st);
#pragma unroll
                    for (int k = 0; k < F::STJ; k++) dst[k] = sStd[q * F::STJ + k];
                }
                const double dV = sDV[q];
                double chk = 0.0;
                if constexpr (F::FSC && IGA_FS_P4) {
                    // warp w computes the columns (kq, j = w) of every trial kind kq (M == NWARP)
                    const int j = warp;
                    static_for<NQK>([&](auto KQ) {
                        constexpr int kq = decltype(KQ)::value;
                        double col[NKS * M];
                        PH::template dcol_j<3, L::qk(kq)>(st, j, a, b, col);
                        const unsigned char *o4 = ft.off4 + (kq * M + j) * M * NTK;
                        static_for<M>([&](auto II) {
                            constexpr int i = decltype(II)::value;
                            static_for<NTK>([&](auto TK) {
                                constexpr int t = decltype(TK)::value;
                                const int e = o4[i * NTK + t];
                                if (e != 255) {
                                    const double v = col[L::tk(t) * M + i] * dV;
                                    chk += v;
                                    sD[q * F::DQS + e] = v;
                                }
                            });
                        });
                    });
                    if (!isfinite(chk)) errbits |= 2;
                } else {
                    static_for<NQK * M>([&](auto KJ) {
                        constexpr int kq = decltype(KJ)::value / M, j = decltype(KJ)::value % M;
                        constexpr int k2 = L::qk(kq);
                        if (warp == decltype(KJ)::value % NWP) {
                            double col[NKS * M];
                            PH::template dcol<3>(st, k2, j, a, b, col);
                            if constexpr (F::FSC) {
                                // compact list: only the structurally nonzero (i, j, t, k) entries
                                static_for<M>([&](auto II) {
                                    constexpr int i = decltype(II)::value;
                                    static_for<NTK>([&](auto TK) {
                                        constexpr int t = decltype(TK)::value;
                                        constexpr int e = FsMeta<L>::eij(i, j, L::tk(t), k2);
                                        if constexpr (e >= 0) {
                                            const double v = col[L::tk(t) * M + i] * dV;
                                            chk += v;
                                            sD[q * F::DQS + e] = v;
                                        }
                                    });
                                });
                            } else {
#pragma unroll
                            for (int i = 0; i < M; i++) {
                                // block layout [trial kind k][test kind t]: this column's NTK entries
                                // are contiguous (16-byte stores when NTK is even)
                                double *dst = sD + q * F::DQS + (i * M + j) * DB + kq * NTK;
                                double v[NTK];
                                static_for<NTK>([&](auto TK) {
                                    constexpr int t = decltype(TK)::value;
                                    v[t] = col[L::tk(t) * M + i] * dV;
                                    chk += v[t];
                                });
                                if constexpr (NTK % 2 == 0 && (NTK * 8) % 16 == 0) {
#pragma unroll
                                    for (int t = 0; t < NTK; t += 2)
                                        *reinterpret_cast<double2 *>(dst + t) = make_double2(v[t], v[t + 1]);
                                } else {
#pragma unroll
                                    for (int t = 0; t < NTK; t++) dst[t] = v[t];
                                }
                            }
                            }
                        }
                    });
                    if (!isfinite(chk)) errbits |= 2;
                }
            }
            __syncthreads();

            if constexpr (F::FSC) {
                // ---- 5 (FS). fully sum-factorised contraction, one test component I at a time:
                //      stage 1 per (I, J = warp) compiled with its exact coefficient structure ----
                static_assert(F::NWARP == M, "FS stage 1 maps warp = trial component J");
                using FM = FsMeta<L>;
                double *sX1 = sm + F::O_X1;
#pragma unroll 1
                for (int I = 0; I < M; I++) {
#if IGA_FS_BS1
                    fs_stage1<F, P>(I, warp, sD, sTab, sX1, ut, ft, lane, I > 0);
                    __syncthreads();
                    fs_stage23<F, P>(I, tid, sX1, sTab, sPosE, sW, sRS, val, ut, dbg);
                    if (I + 1 == M && !PREF) __syncthreads();  // the last one: the end-of-element barrier
#else
                    fs_stage1<F, P>(I, warp, sD, sTab, sX1, ut, ft, lane);
                    __syncthreads();
                    fs_stage23<F, P>(I, tid, sX1, sTab, sPosE, sW, sRS, val, ut, dbg);
                    if (I + 1 < M || !PREF) __syncthreads();   // the last one: the end-of-element barrier
#endif
                }
            } else
            // ---- 5. test-side sum factorisation + coalesced emission ----
            // Non-symmetric forms: the NEN*M*M column tasks (I, B, J) (J fastest: 4 consecutive
            // lanes write one 32-byte sector of a CSR row) are dealt round-robin over all NT
            // threads -- 432 tasks on 128 threads = 14 warp-passes instead of 4 passes of the
            // 108 (B, J) threads on 4 warps (16 warp-passes, the last warp 12/32 lanes busy).
            if constexpr (!F::SYMJ && IGA_BAL) {
                // The last NCOL mod NT columns (a partial pass: 48 of 432 for VMS) are split in two
                // q0 sub-ranges on two threads each (partial columns, both added with red.add): the
                // tail takes 2/3 of a column time instead of a whole one while the rest of the
                // CTA waits at the barrier (IGA_TAIL=0: whole tail columns).
                constexpr int NCOL = NEN * M * M, NFULL = NCOL / NTH * NTH, NTAIL = NCOL - NFULL;
                constexpr bool SPLIT = IGA_TAIL && NTAIL > 0 && 2 * NTAIL <= NTH && NQ1 >= 2;
#pragma unroll 1
                for (int cc = tid; cc < (SPLIT ? NFULL + 2 * NTAIL : NCOL); cc += NTH) {
                    int c = cc, q0lo = 0, q0hi = NQ1;
                    if (SPLIT && cc >= NFULL) {
                        const int h = (cc - NFULL) / NTAIL;                 // 0: q0 < NQ1-1, 1: last slab
                        c = NFULL + (cc - NFULL) - h * NTAIL;
                        q0lo = h ? NQ1 - 1 : 0;
                        q0hi = h ? NQ1 : NQ1 - 1;
                    }
                    const int I = c / (NEN * M), r = c - I * (NEN * M), B = r / M, J = r - B * M;
                    const int b0 = B / (NP1 * NP1), b1 = (B / NP1) % NP1, b2 = B % NP1;
                    double Kc[NEN];
                    if (!(dbg & 1)) tsf_column_3d<F, UNI, P>(Kc, sD, I * M + J, b0, b1, b2, sTab, ut, sm + F::O_PB, q0lo, q0hi);
                    else {
#pragma unroll
                        for (int A = 0; A < NEN; A++) Kc[A] = sD[A * 7 + J];
                    }
                    if (!(dbg & 2)) {
                        int P0[NP1], P1[NP1], P2[NP1], W1[NP1], W2[NP1];
#pragma unroll
                        for (int x = 0; x < NP1; x++) {
                            P0[x] = sPosE[x * NP1 + b0];
                            P1[x] = sPosE[NP1 * NP1 + x * NP1 + b1];
                            P2[x] = sPosE[2 * NP1 * NP1 + x * NP1 + b2];
                            W1[x] = sW[NP1 + x];
                            W2[x] = sW[2 * NP1 + x];
                        }
#pragma unroll
                        for (int A = 0; A < NEN; A++) {
                            const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
                            const int co = (P0[a0] * W1[a1] + P1[a1]) * W2[a2] + P2[a2];
                            atomicAdd(val + sRS[A * M + I] + (long long)co * M + J, Kc[A]);
                        }
                    } else {
                        double sum = 0.0;
#pragma unroll
                        for (int A = 0; A < NEN; A++) sum += Kc[A];
                        if (sum == 1.2345e300) val[0] = sum;
                    }
                }
            } else if (tid < NEN * M) {
                const int B = tid / M, T = tid - B * M;
                const int b0 = B / (NP1 * NP1), b1 = (B / NP1) % NP1, b2 = B % NP1;
                // Symmetric tangents (hyperelasticity: major symmetry of A_aIbJ, A-12): only the
                // M(M+1)/2 blocks I <= J are contracted, (M+1)/2 per thread, and block (J, I) is
                // written as the transpose.  Otherwise thread (B, J) does blocks (0..M-1, J).
                constexpr bool SYMJ = F::SYMJ;
                constexpr int NPAIR = SYMJ ? (M + 1) / 2 : M;
#pragma unroll 1
                for (int pi = 0; pi < NPAIR; pi++) {
                    int I, J;
                    if constexpr (SYMJ) {
                        const int k = T * NPAIR + pi;                  // k-th pair of the upper triangle
                        I = 0;
                        J = k;
                        while (J >= M - I) { J -= M - I; I++; }       // row I holds pairs (I, I..M-1)
                        J += I;
                        if (I >= M) break;                            // odd M*(M+1)/2 remainder
                    } else {
                        I = pi;
                        J = T;
                    }
                    double Kc[NEN];
                    if (!(dbg & 1)) tsf_column_3d<F, UNI, P>(Kc, sD, I * M + J, b0, b1, b2, sTab, ut, sm + F::O_PB);
                    else {
#pragma unroll
                        for (int A = 0; A < NEN; A++) Kc[A] = sD[A * 7 + J];
                    }
                    if (!(dbg & 2)) {
                        // column offset of (A, B) in row A: closed form of the per-axis Alg. 3
                        // positions, ((pos0 W1 + pos1) W2 + pos2) (in nodes)
                        int P0[NP1], P1[NP1], P2[NP1], W1[NP1], W2[NP1];
#pragma unroll
                        for (int x = 0; x < NP1; x++) {
                            P0[x] = sPosE[x * NP1 + b0];
                            P1[x] = sPosE[NP1 * NP1 + x * NP1 + b1];
                            P2[x] = sPosE[2 * NP1 * NP1 + x * NP1 + b2];
                            W1[x] = sW[NP1 + x];
                            W2[x] = sW[2 * NP1 + x];
                        }
#pragma unroll
                        for (int A = 0; A < NEN; A++) {
                            const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
                            const int co = (P0[a0] * W1[a1] + P1[a1]) * W2[a2] + P2[a2];
                            atomicAdd(val + sRS[A * M + I] + (long long)co * M + J, Kc[A]);
                        }
                        if (SYMJ && I != J) {
                            // transpose: row (B, J), column (A, I); positions of A in row B
                            const int W1B = sW[NP1 + b1], W2B = sW[2 * NP1 + b2];
#pragma unroll
                            for (int x = 0; x < NP1; x++) {
                                P0[x] = sPosE[b0 * NP1 + x];
                                P1[x] = sPosE[NP1 * NP1 + b1 * NP1 + x];
                                P2[x] = sPosE[2 * NP1 * NP1 + b2 * NP1 + x];
                            }
                            const long long rowB = sRS[B * M + J] + I;
#pragma unroll
                            for (int A = 0; A < NEN; A++) {
                                const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
                                const int co = (P0[a0] * W1B + P1[a1]) * W2B + P2[a2];
                                atomicAdd(val + rowB + (long long)co * M, Kc[A]);
                            }
                        }
                    } else {
                        double sum = 0.0;
#pragma unroll
                        for (int A = 0; A < NEN; A++) sum += Kc[A];
                        if (sum == 1.2345e300) val[0] = sum;
                    }
                }
            }
        }
        if constexpr (IGA_DYN) {
            if (tid == 0) sEl = PREF ? nxt : (long long)gridDim.x + (long long)atomicAdd(s.wq, 1ULL);
            __syncthreads();
            el = sEl;
        } else {
            __syncthreads();
            el += gridDim.x;
        }
    }
    if (errbits) atomicOr(s.errflag, errbits);
}

template <int P, class PH, bool UNI>
static iga_status run_fused3d(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                              const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    using FF = F3K<P, PH, true, UNI>;
    using FR = F3K<P, PH, false, UNI>;
    Prm prm;
    for (int i = 0; i < 8; i++) prm.p[i] = phys->p[i];
    UniTab<P> ut{};
    if (UNI)
        for (int d = 0; d < 3; d++) {
            for (int i = 0; i < (P + 1) * 3 * (P + 1); i++) (&ut.t[d][0][0][0])[i] = s->tab0[d][i];
            for (int q = 0; q <= P; q++) ut.qw[d][q] = s->qw0[d][q];
            ut.hp[d] = s->hp0[d];
        }
    typename FF::FT ft{};
    typename FR::FT ftr{};
    if constexpr (FF::FSC) {
        using L = typename FF::L;
        using FM = FsMeta<L>;
        static_assert(FF::DQS <= 255, "compact offsets must fit a byte");
        for (int I = 0; I < FF::M; I++)
            for (int J = 0; J < FF::M; J++)
                for (int g = 0; g < FM::NG; g++)
                    for (int c = 0; c < FM::ncombo(g); c++) {
                        const int t = FM::TT.t[FM::combo(g, c, true)].k, kq = FM::QT.t[FM::combo(g, c, false)].k;
                        const int e = FM::eij(I, J, L::tk(t), L::qk(kq));
                        ft.off[I * FF::M + J][IGA_FS_TK ? t * FF::NQK + kq : FM::cbase(g) + c] = (unsigned char)(e < 0 ? FF::ZSLOT : e);
                    }
        for (int kq = 0; kq < FF::NQK; kq++)
            for (int j = 0; j < FF::M; j++)
                for (int i = 0; i < FF::M; i++)
                    for (int t = 0; t < FF::NTK; t++) {
                        const int e = FM::eij(i, j, L::tk(t), L::qk(kq));
                        ft.off4[((kq * FF::M + j) * FF::M + i) * FF::NTK + t] = (unsigned char)(e < 0 ? 255 : e);
                    }
    }
    const bool jac = val != nullptr;
    const bool jac_ = val != nullptr;
    const size_t smem = jac_ ? FF::SMEM : FR::SMEM_RES;
    {   // per-device attribute: set on the current device before every launch
        cudaError_t ce = jac ? cudaFuncSetAttribute(k_fused3d<P, PH, true, UNI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(k_fused3d<P, PH, false, UNI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce != cudaSuccess) { set_error(std::string("fused3d smem: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    }
    int occ = 1;
    if (jac) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused3d<P, PH, true, UNI>, FF::NT, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused3d<P, PH, false, UNI>, FF::NT, smem);
    occ = std::max(occ, 1);
    const long long nel = s->nel_local;
    const int grid = (int)std::min<long long>(nel, (long long)nsm * occ);
    int launches = 0;
    if ((jac || F) && !s->skip_zero) {
        ProfScope ps(s, "k_zero", st);
        k_zero_pair(val, jac ? s->nnz_owned : 0, F, F ? s->nrows_owned : 0, st, nsm);
        launches++;
    }
    {
        ProfScope ps(s, "k_fused3d", st);
        // block width: ~3 element layers of a block's rows (values, m^2 (2p+1)^3 per node) in half the L2
        const int ne1 = s->el_hi[1] - s->el_lo[1], ne2 = s->el_hi[2] - s->el_lo[2];
        const double row_bytes = 8.0 * FF::M * FF::M * (2 * P + 1) * (2 * P + 1) * (2 * P + 1);
        int bw = (int)(60e6 / (3.0 * (ne2 + P) * row_bytes)) - P;
        if (s->bw_opt > 0) bw = s->bw_opt;
        bw = std::max(1, std::min(bw, ne1));
        if (IGA_DYN) {
            cudaError_t me = cudaMemsetAsync(s->dev.wq, 0, sizeof(unsigned long long), st);
            if (me != cudaSuccess) { set_error(std::string("fused3d counter: ") + cudaGetErrorString(me)); return IGA_ERR_CUDA; }
        }
        if (jac) k_fused3d<P, PH, true, UNI><<<grid, FF::NT, smem, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel, ut, ft, s->dbg, bw);
        else k_fused3d<P, PH, false, UNI><<<grid, FF::NT, smem, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel, ut, ftr, s->dbg, bw);
        launches++;
    }
    s->last_launches = launches;
    s->last_occupancy = occ;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("fused3d launch: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

iga_status launch_fused3d(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                          const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    if (s->dim != 3 || s->mode != MODE_PARAM) return IGA_ERR_STATE;
    if (s->p[0] != 2 || s->p[1] != 2 || s->p[2] != 2) return IGA_ERR_STATE;
    const bool uni = s->tab_uniform[0] && s->tab_uniform[1] && s->tab_uniform[2] && !s->force_general;
    if (ph->kind == IGA_PHYS_NS_VMS && s->dof == 4)
        return uni ? run_fused3d<2, PhysNSVMS, true>(s, ph, a, b, U, Ud, val, F, st, nsm)
                   : run_fused3d<2, PhysNSVMS, false>(s, ph, a, b, U, Ud, val, F, st, nsm);
    if (ph->kind == IGA_PHYS_NEOHOOKE && s->dof == 3)
        return uni ? run_fused3d<2, PhysNeoHooke, true>(s, ph, a, b, U, Ud, val, F, st, nsm)
                   : run_fused3d<2, PhysNeoHooke, false>(s, ph, a, b, U, Ud, val, F, st, nsm);
    if (ph->kind == IGA_PHYS_CAHN_HILLIARD && s->dof == 1)      // 3D CH
        return uni ? run_fused3d<2, PhysCahnHilliard, true>(s, ph, a, b, U, Ud, val, F, st, nsm)
                   : run_fused3d<2, PhysCahnHilliard, false>(s, ph, a, b, U, Ud, val, F, st, nsm);
    return IGA_ERR_STATE;
}

}  // namespace iga
