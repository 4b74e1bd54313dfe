// fused2d.cu -- K4/K3 for 2D scalar spaces (configs 1-3): one fused kernel per call.
//
// A CTA owns a tile of TE0 x TE1 elements (persistent over tiles).  Per element, a group of
// NEN lanes (16 for p=3, 9 for p=2) runs Alg. 4 for all its quadrature points at once:
//   lane q  -> pointwise_qp (tables -> kinds -> rational/geometry -> fields -> physics), the
//              compact coefficients D~ / r~ for its point go to a per-group shared scratch;
//   lane B  -> test-side sum factorisation of column B of the element matrix
//              K_e[A,B] = w_A w_B sum_q P(A,q)^T D~(q) P(B,q): H(q) = D~(q) P(B,q), then the
//              contraction over q1 (per q0) and over q0, using the 1D tables only;
//   lane A  -> F_e[A].
// Column B of the element block is added straight into the caller's CSR rows with
// red.global.add.f64 (rows pre-zeroed by k_zero; a shared-memory row image was measured slower:
// an fp64 shared atomicAdd is a CAS loop on sm_100a).  The CSR position of
// (row A, column B) is a closed form of the per-node row starts and the per-axis Alg. 3 stencil
// positions staged once per tile, so no kernel searches col_idx.
#include <cstdio>

#include "iga_host.h"
#include "pointwise.cuh"

namespace iga {

template <int P> struct Tile2 {
    static constexpr int TE0 = 16;
    // TE1 = the widest tile along axis 1 (shared-memory layout); the launch picks the actual
    // width te1 <= TE1 so that the tile count fills the SMs in whole rounds (wave quantisation)
    static constexpr int TE1 = P == 2 ? 36 : 32;
    // 12 warps (168 registers, no spills with the direct scatter; measured best for p = 2 and 3)
#ifndef IGA_NW2
#define IGA_NW2 12
#endif
#ifndef IGA_NW3
#define IGA_NW3 12
#endif
    static constexpr int NWARP = P == 2 ? IGA_NW2 : IGA_NW3;
    static constexpr int NB0 = TE0 + P, NB1 = TE1 + P;      // touched node box (uniform knots)
    static constexpr int NSL = (2 * P + 1) * (2 * P + 1);   // stencil slots per row
};

// element's nodes in the tile box: local function A = (a0, a1) -> box index base + a0*NB1 + a1
template <int NP1, int NB1>
struct SmemNodes2 {
    static constexpr bool PREMUL = true;     // tile staging stores w u, w udot, w x (NURBS)
    const double *pu, *pud, *pw, *px0, *px1;
    int base;
    bool hud;
    __device__ __forceinline__ int idx(int A) const { return base + (A / NP1) * NB1 + A % NP1; }
    __device__ __forceinline__ double u(int A, int) const { return pu[idx(A)]; }
    __device__ __forceinline__ double ud(int A, int) const { return pud[idx(A)]; }
    __device__ __forceinline__ bool has_ud() const { return hud; }
    __device__ __forceinline__ double w(int A) const { return pw ? pw[idx(A)] : 1.0; }
    __device__ __forceinline__ double x(int A, int i) const { return i == 0 ? px0[idx(A)] : px1[idx(A)]; }
};

// uniform knots: every element shares the 1D tables (translation invariance of uniform
// B-splines); they travel as a __grid_constant__ parameter so the unrolled test-side
// contraction reads them as constant-bank operands instead of shared-memory loads
template <int P>
struct UniTab2 {
    double t[2][P + 1][3][P + 1];   // [axis][q][k][a]
};

// test-side sum factorisation of one column (trial function (b0,b1)) in 2D
template <class L, class KS, int P, bool UNI>
__device__ __forceinline__ void tsf_column_2d(double (&Kc)[(P + 1) * (P + 1)], const double *__restrict__ Dg,
                                              const double *__restrict__ tb0, const double *__restrict__ tb1,
                                              int b0, int b1, const UniTab2<P> &ut) {
    constexpr int NP1 = P + 1, NQ1 = P + 1, NQ = NQ1 * NQ1, NC = KS::NC;
    auto T0 = [&](int q, int k, int a) -> double {
        if constexpr (UNI) return ut.t[0][q][k][a];
        else return tb0[(q * 3 + k) * NP1 + a];
    };
    auto T1 = [&](int q, int k, int a) -> double {
        if constexpr (UNI) return ut.t[1][q][k][a];
        else return tb1[(q * 3 + k) * NP1 + a];
    };
    // tb_d layout: [q][k][a]
#pragma unroll
    for (int A = 0; A < NP1 * NP1; A++) Kc[A] = 0.0;
    // the q0 loop rolled (smaller code; A/B -1.5 % config 2, -1.7 % config 3; rolling q1 too: +17 %)
#pragma unroll 1
    for (int q0 = 0; q0 < NQ1; q0++) {
        double S[3][NP1];
#pragma unroll
        for (int o = 0; o < 3; o++)
#pragma unroll
            for (int a = 0; a < NP1; a++) S[o][a] = 0.0;
        double vb0[3];
#pragma unroll
        for (int k = 0; k < 3; k++) vb0[k] = tb0[(q0 * 3 + k) * NP1 + b0];
#pragma unroll
        for (int q1 = 0; q1 < NQ1; q1++) {
            const int q = q0 * NQ1 + q1;
            double vb1[3];
#pragma unroll
            for (int k = 0; k < 3; k++) vb1[k] = tb1[(q1 * 3 + k) * NP1 + b1];
            double Pb[NC], H[NC];
            static_for<NC>([&](auto C) {
                constexpr int c = decltype(C)::value;
                H[c] = 0.0;
                Pb[c] = 0.0;
                if constexpr (L::trial_used(c)) {
                    static_for<KS::nterms(c)>([&](auto T) {
                        constexpr int t = decltype(T)::value;
                        Pb[c] += vb0[KS::ord(c, t, 0)] * vb1[KS::ord(c, t, 1)];
                    });
                }
            });
            static_for<L::NE>([&](auto E) {
                constexpr int e = decltype(E)::value;
                constexpr int c = L::E.c[e], c2 = L::E.c2[e];
                H[c] += Dg[e * NQ + q] * Pb[c2];
            });
            // stage 1: contract q1 into tracks keyed by the axis-0 derivative order
            static_for<NC>([&](auto C) {
                constexpr int c = decltype(C)::value;
                if constexpr (L::test_used(c)) {
                    static_for<KS::nterms(c)>([&](auto T) {
                        constexpr int t = decltype(T)::value;
                        constexpr int o0 = KS::ord(c, t, 0), o1 = KS::ord(c, t, 1);
#pragma unroll
                        for (int a1 = 0; a1 < NP1; a1++) S[o0][a1] += H[c] * T1(q1, o1, a1);
                    });
                }
            });
        }
        // stage 2: contract q0
#pragma unroll
        for (int o0 = 0; o0 < 3; o0++) {
            bool used = false;
            static_for<NC>([&](auto C) {
                constexpr int c = decltype(C)::value;
                if constexpr (L::test_used(c)) {
                    static_for<KS::nterms(c)>([&](auto T) {
                        constexpr int t = decltype(T)::value;
                        if (KS::ord(c, t, 0) == o0) used = true;
                    });
                }
            });
            if (!used) continue;
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) {
                const double n0 = T0(q0, o0, a0);
#pragma unroll
                for (int a1 = 0; a1 < NP1; a1++) Kc[a0 * NP1 + a1] += n0 * S[o0][a1];
            }
        }
    }
}

// UNI: 0 general tables, 1 uniform runs checked per element, 2 every element uniform
#ifndef IGA_DBG
#define IGA_DBG 0      // 1: honour the dbg phase-skip bits (A/B timing builds only)
#endif

template <int P, class PH, int MODE, bool JAC, int UNI>
// residual-only parametric launches: 2 CTAs per SM (A/B: config 3 residual -6 %; NURBS slower)
__global__ void __launch_bounds__(32 * Tile2<P>::NWARP, (!JAC && MODE == MODE_PARAM) ? 2 : 1)
k_fused2d(SpaceDev s, Prm prm, double a, double b, const double *__restrict__ U, const double *__restrict__ Ud,
          double *__restrict__ val, double *__restrict__ Fout, int ntile0, int ntile1, int te1, int dbg_,
          const __grid_constant__ UniTab2<P> ut) {
    const int dbg = IGA_DBG ? dbg_ : 0;
    using L = Lists<PH, 2, MODE>;
    using KS = typename L::KS;
    using TL = Tile2<P>;
    constexpr int NP1 = P + 1, NQ1 = P + 1, NQ = NQ1 * NQ1, NEN = NP1 * NP1;
    constexpr int G = NEN;                  // lanes per element group
    constexpr int GPW = 32 / G;             // groups per warp
    constexpr int NWARP = TL::NWARP, NGRP = NWARP * GPW;
    constexpr int NB0 = TL::NB0, NB1 = TL::NB1, NBN = NB0 * NB1, NSL = TL::NSL, W2 = 2 * P + 1;
    constexpr int NE = L::NE, NR = L::NR;
    // group scratch per point: coefficients D~ (Jacobian) and r~; for p = 3 also room for the
    // sum-factorised homogeneous sums (residual-only launches need it beyond r~)
    constexpr int SFN = (P == 3 || MODE == MODE_NURBS)
                            ? (NP1 * NQ1 * ((MODE == MODE_NURBS ? 3 : 0) + 1 + (PH::UDOT ? 1 : 0)) * 3 + NQ - 1) / NQ : 0;
    constexpr int SCR = JAC ? NE + NR : (NR > SFN ? NR : SFN);

    extern __shared__ __align__(16) double sm[];
    double *nU = sm, *nUd = nU + NBN, *nw = nUd + NBN, *nx0 = nw + NBN, *nx1 = nx0 + NBN;
    double *tb = nx1 + NBN;                             // [2][TE][NQ1][3][NP1]
    double *qwb = tb + 2 * TL::TE1 * NQ1 * 3 * NP1;      // [2][TE][NQ1]  weights
    double *qxb = qwb + 2 * TL::TE1 * NQ1;              // [2][TE][NQ1]  coordinates
    double *hpb = qxb + 2 * TL::TE1 * NQ1;              // [2][TE]
    double *scr = hpb + 2 * TL::TE1;                    // [NGRP][SCR][NQ]
    // scatter metadata of the tile's rows (computed once per node, not per entry)
    // group scratch stride: p = 3 pads one double so the two groups of a warp (whose lanes all
    // read their own group's coefficient at the same offset) hit different banks
    constexpr int GSTR = SCR * NQ + (P == 3 ? 1 : 0);
    long long *rowOff = reinterpret_cast<long long *>(scr + (size_t)NGRP * GSTR);   // [NBN] CSR row start - val
    long long *fIdx = rowOff + NBN;                         // [NBN] residual entry of the node
    int *rowW1 = reinterpret_cast<int *>(fIdx + NBN);       // [NBN] Alg. 3 width along axis 1
    int *pd0 = rowW1 + NBN;                                 // [NB0][W2] position of column g0+delta in row g0
    int *pd1 = pd0 + NB0 * W2;                              // [NB1][W2]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp_in_warp = lane / G, t = lane % G;
    const bool lane_ok = grp_in_warp < GPW;
    const int grp = warp * GPW + (lane_ok ? grp_in_warp : 0);
    double *gs = scr + (size_t)grp * GSTR;
    const AxisDev &A0 = s.ax[0], &A1 = s.ax[1];
    int errbits = 0;

    for (int tile = blockIdx.x; tile < ntile0 * ntile1; tile += gridDim.x) {
        const int T0 = tile / ntile1, T1 = tile % ntile1;
        const int e0lo = A0.el_lo + T0 * TL::TE0, e1lo = A1.el_lo + T1 * te1;
        const int ne0 = min(TL::TE0, A0.el_hi - e0lo), ne1 = min(te1, A1.el_hi - e1lo);
        const int F00 = A0.first[e0lo], F01 = A1.first[e1lo];
        const int nb0 = ne0 + P, nb1 = ne1 + P;
        // ---- stage the tile: node data, scatter metadata, tables ----
        for (int i = (dbg & 16) ? NBN : tid; i < NBN; i += blockDim.x) {
            const int l0 = i / NB1, l1 = i % NB1;
            if (l0 < nb0 && l1 < nb1) {
                int g0 = F00 + l0, g1 = F01 + l1;
                if (g0 >= A0.nu) g0 -= A0.nu;
                if (g1 >= A1.nu) g1 -= A1.nu;
                const long long node = (long long)g0 * A1.nu + g1;             // geometry: global
                const long long lnode = local_node(s, g0, g1, 0);               // fields: touched box
                fIdx[i] = lnode;
                // homogeneous (weighted) node data for the rational basis, staged once per tile
                const double wn = (MODE == MODE_NURBS && s.wts) ? s.wts[node] : 1.0;
                nU[i] = wn * U[lnode];
                nUd[i] = Ud ? wn * Ud[lnode] : 0.0;
                nw[i] = wn;
                if (s.geom == IGA_GEOM_NURBS) {
                    nx0[i] = wn * s.ctrl[node * 2];
                    nx1[i] = wn * s.ctrl[node * 2 + 1];
                }
                if (JAC) {
                    // closed-form CSR row start over the touched box (row_start with m = 1 and a
                    // trivial axis 2); halo rows as offsets from val in the flat address space
                    const int m0 = local_fn(A0, g0), m1 = local_fn(A1, g1);
                    const int sg0 = m0 >= A0.n_own, sg1 = m1 >= A1.n_own;
                    long long off = A0.lS[m0] * (sg1 ? A1.Th : A1.T) + (long long)A0.rowW[g0] * A1.lS[m1];
                    if (sg0 | sg1)
                        off += ((long long)(uintptr_t)(s.halo + s.hbase[(sg0 * 2 + sg1) * 2]) - (long long)(uintptr_t)val) / 8;
                    rowOff[i] = off;
                    rowW1[i] = A1.rowW[g1];
                }
            }
        }
        if (JAC) {
            for (int i = tid; i < (NB0 + NB1) * W2; i += blockDim.x) {
                const int d = i >= NB0 * W2, k = d ? i - NB0 * W2 : i;
                const int l = k / W2, dl = k % W2;
                const AxisDev &ax = d ? A1 : A0;
                int g = (d ? F01 : F00) + l;
                if (g >= ax.nu) g -= ax.nu;
                pd0[i] = (l < (d ? nb1 : nb0)) ? ax.posd[g * W2 + dl] : -1;
            }
        }
        for (int i = (dbg & 16) ? 1 << 30 : tid; i < 2 * TL::TE1 * NQ1 * 3 * NP1; i += blockDim.x) {
            const int d = i / (TL::TE1 * NQ1 * 3 * NP1), r = i % (TL::TE1 * NQ1 * 3 * NP1);
            const int el = r / (NQ1 * 3 * NP1);
            const int elo = d == 0 ? e0lo : e1lo, ne = d == 0 ? ne0 : ne1;
            if (el < ne) tb[i] = s.ax[d].tab[(size_t)(elo + el) * NQ1 * 3 * NP1 + r % (NQ1 * 3 * NP1)];
        }
        for (int i = (dbg & 16) ? 1 << 30 : tid; i < 2 * TL::TE1 * NQ1; i += blockDim.x) {
            const int d = i / (TL::TE1 * NQ1), r = i % (TL::TE1 * NQ1);
            const int el = r / NQ1;
            const int elo = d == 0 ? e0lo : e1lo, ne = d == 0 ? ne0 : ne1;
            if (el < ne) {
                qwb[i] = s.ax[d].qw[(size_t)(elo + el) * NQ1 + r % NQ1];
                qxb[i] = s.ax[d].qx[(size_t)(elo + el) * NQ1 + r % NQ1];
            }
        }
        for (int i = (dbg & 16) ? 1 << 30 : tid; i < 2 * TL::TE1; i += blockDim.x) {
            const int d = i / TL::TE1, el = i % TL::TE1;
            const int elo = d == 0 ? e0lo : e1lo, ne = d == 0 ? ne0 : ne1;
            if (el < ne) hpb[i] = s.ax[d].hpar[elo + el];
        }
        __syncthreads();

        // ---- element loop: one group of G lanes per element ----
        const int nel_tile = ne0 * ne1;
        for (int base = 0; base < nel_tile; base += NGRP) {
            const int el = base + grp;
            const bool act = lane_ok && el < nel_tile;
            const int le0 = act ? el / ne1 : 0, le1 = act ? el % ne1 : 0;
            // local node offsets of the element's functions within the tile box
            // (uniform knots, checked at launch: first[e] = first0 + e)
            const int fo0 = le0, fo1 = le1;
            const double *tb0 = tb + (size_t)(0 * TL::TE1 + le0) * NQ1 * 3 * NP1;
            const double *tb1 = tb + (size_t)(1 * TL::TE1 + le1) * NQ1 * 3 * NP1;
            // (0) the point's homogeneous sums (w, w x, w u, w udot and their kinds), sum factorised
            //     over the element's functions by the lane group: stage 1, lane (a0, q1):
            //     S1[f][o1][a0][q1] = sum_a1 T1(q1, o1, a1) f(a0, a1), into the group scratch (lane-
            //     contiguous: no bank conflicts);
            //     stage 2, lane (q0, q1): S[f][o0][o1] = sum_a0 T0(q0, o0, a0) S1[a0][q1][f][o1]
            //     (2 (p+1)^3 FMA per field and order pair instead of (p+1)^4 per point)
            constexpr int NFW = MODE == MODE_NURBS ? 3 : 0;               // w, w x0, w x1
            constexpr int NF = NFW + 1 + (PH::UDOT ? 1 : 0);              // + w u (+ w udot)
            // p = 3 always; p = 2 only for residual-only NURBS launches (A/B: p = 2 Jacobian and the
            // parametric residual are slower with it)
            constexpr bool SFP = (P == 3 || (!JAC && MODE == MODE_NURBS)) && NP1 == NQ1 && NP1 * NQ1 * NF * 3 <= SCR * NQ;
            constexpr int NPRE = KS::NC * (1 + 2 + 1) + 1;
            if constexpr (SFP) {
                double pre[NPRE];
                const int base_n = fo0 * NB1 + fo1;
                constexpr auto used = [](int o0, int o1) {
                    for (int c = 0; c < KS::NC; c++)
                        for (int tt = 0; tt < KS::nterms(c); tt++)
                            if (KS::ord(c, tt, 0) == o0 && KS::ord(c, tt, 1) == o1) return true;
                    return o0 == 0 && o1 == 0;
                };
                constexpr auto used1 = [](int o1) {
                    for (int o0 = 0; o0 < 3; o0++)
                        for (int c = 0; c < KS::NC; c++)
                            for (int tt = 0; tt < KS::nterms(c); tt++)
                                if (KS::ord(c, tt, 0) == o0 && KS::ord(c, tt, 1) == o1) return true;
                    return o1 == 0;
                };
                const double *fsrc[5] = {nw, nx0, nx1, nU, nUd};
                if (act && !(dbg & 4)) {
                    const int a0 = t / NQ1, q1 = t % NQ1;
                    double fv[NF][NP1];
#pragma unroll
                    for (int f = 0; f < NF; f++)
#pragma unroll
                        for (int a1 = 0; a1 < NP1; a1++) fv[f][a1] = fsrc[NFW ? f : f + 3][base_n + a0 * NB1 + a1];
                    static_for<3>([&](auto O1) {
                        constexpr int o1 = decltype(O1)::value;
                        if constexpr (used1(o1)) {
                            double t1[NP1];
#pragma unroll
                            for (int a1 = 0; a1 < NP1; a1++) t1[a1] = tb1[(q1 * 3 + o1) * NP1 + a1];
#pragma unroll
                            for (int f = 0; f < NF; f++) {
                                double acc = 0.0;
#pragma unroll
                                for (int a1 = 0; a1 < NP1; a1++) acc += t1[a1] * fv[f][a1];
                                gs[((f * 3 + o1) * NP1 + a0) * NQ1 + q1] = acc;
                            }
                        }
                    });
                }
                __syncwarp();
                if (act && !(dbg & 4)) {
                    const int q0 = t / NQ1, q1 = t % NQ1;
                    double S[NF][3][3];
                    static_for<3>([&](auto O0) {
                        constexpr int o0 = decltype(O0)::value;
                        static_for<3>([&](auto O1) {
                            constexpr int o1 = decltype(O1)::value;
                            if constexpr (used(o0, o1)) {
#pragma unroll
                                for (int f = 0; f < NF; f++) {
                                    double acc = 0.0;
#pragma unroll
                                    for (int a0 = 0; a0 < NP1; a0++)
                                        acc += tb0[(q0 * 3 + o0) * NP1 + a0] * gs[((f * 3 + o1) * NP1 + a0) * NQ1 + q1];
                                    S[f][o0][o1] = acc;
                                }
                            }
                        });
                    });
                    // kinds: sum of the kind's separable terms; pre = [W][X0][X1][Phi][Phit]
                    static_for<KS::NC>([&](auto C) {
                        constexpr int c = decltype(C)::value;
                        double kv[NF];
#pragma unroll
                        for (int f = 0; f < NF; f++) kv[f] = 0.0;
                        static_for<KS::nterms(c)>([&](auto TT) {
                            constexpr int tt = decltype(TT)::value;
#pragma unroll
                            for (int f = 0; f < NF; f++) kv[f] += S[f][KS::ord(c, tt, 0)][KS::ord(c, tt, 1)];
                        });
                        pre[c] = NFW ? kv[0] : 1.0;
                        pre[KS::NC + c] = NFW ? kv[1] : 0.0;
                        pre[2 * KS::NC + c] = NFW ? kv[2] : 0.0;
                        pre[3 * KS::NC + c] = kv[NFW];
                    });
                    pre[4 * KS::NC] = PH::UDOT ? S[NF - 1][0][0] : 0.0;
                }
                __syncwarp();                    // S1 consumed before pointwise_qp writes the scratch
            if (act) {
                // (1) pointwise at quadrature point q = t
                const int q0 = t / NQ1, q1 = t % NQ1;
                double v[2][3][NP1];
#pragma unroll
                for (int k = 0; k < 3; k++)
#pragma unroll
                    for (int x = 0; x < NP1; x++) {
                        v[0][k][x] = tb0[(q0 * 3 + k) * NP1 + x];
                        v[1][k][x] = tb1[(q1 * 3 + k) * NP1 + x];
                    }
                const double wq = qwb[le0 * NQ1 + q0] * qwb[TL::TE1 * NQ1 + le1 * NQ1 + q1];
                const double xq[2] = {qxb[le0 * NQ1 + q0], qxb[TL::TE1 * NQ1 + le1 * NQ1 + q1]};
                const double hp[2] = {hpb[le0], hpb[TL::TE1 + le1]};
                SmemNodes2<NP1, NB1> nodes;
                nodes.pu = nU; nodes.pud = nUd; nodes.pw = s.wts ? nw : nullptr; nodes.px0 = nx0; nodes.px1 = nx1;
                nodes.hud = Ud != nullptr;
                nodes.base = base_n;
                if (!(dbg & 4))          // dbg bits skip phases (A/B timing only; results invalid)
                    errbits |= pointwise_qp<2, P, PH, MODE, JAC, SmemNodes2<NP1, NB1>, true, SFP>(
                        s, prm, a, b, v, wq, xq, hp, nodes, JAC ? gs + t : nullptr, NQ,
                        Fout ? gs + (JAC ? NE * NQ : 0) + t : nullptr, NQ, pre);
            }
            } else {
            if (act) {
                // (1) pointwise at quadrature point q = t
                const int q0 = t / NQ1, q1 = t % NQ1;
                double v[2][3][NP1];
#pragma unroll
                for (int k = 0; k < 3; k++)
#pragma unroll
                    for (int x = 0; x < NP1; x++) {
                        v[0][k][x] = tb0[(q0 * 3 + k) * NP1 + x];
                        v[1][k][x] = tb1[(q1 * 3 + k) * NP1 + x];
                    }
                const double wq = qwb[le0 * NQ1 + q0] * qwb[TL::TE1 * NQ1 + le1 * NQ1 + q1];
                const double xq[2] = {qxb[le0 * NQ1 + q0], qxb[TL::TE1 * NQ1 + le1 * NQ1 + q1]};
                const double hp[2] = {hpb[le0], hpb[TL::TE1 + le1]};
                SmemNodes2<NP1, NB1> nodes;
                nodes.pu = nU; nodes.pud = nUd; nodes.pw = s.wts ? nw : nullptr; nodes.px0 = nx0; nodes.px1 = nx1;
                nodes.hud = Ud != nullptr;
                nodes.base = fo0 * NB1 + fo1;
                if (!(dbg & 4))          // dbg bits skip phases (A/B timing only; results invalid)
                    errbits |= pointwise_qp<2, P, PH, MODE, JAC, SmemNodes2<NP1, NB1>, true>(
                        s, prm, a, b, v, wq, xq, hp, nodes, JAC ? gs + t : nullptr, NQ,
                        Fout ? gs + (JAC ? NE * NQ : 0) + t : nullptr, NQ);
            }
            }
            __syncwarp();
            if (act) {
                const int c0 = t / NP1, c1 = t % NP1;          // this lane's local function (A or B)
                const int nidx = (fo0 + c0) * NB1 + fo1 + c1;
                const double sw = s.wts ? nw[nidx] : 1.0;
                // (2) residual F_e[A], A = t
                if (Fout && !(dbg & 8)) {
                    // sum factorised per separable term: sum_q0 T0[o0](a0) sum_q1 T1[o1](a1) r(q0, q1)
                    const double *Rg = gs + (JAC ? NE * NQ : 0);
                    double t0[NQ1][3], t1[NQ1][3];
#pragma unroll
                    for (int q = 0; q < NQ1; q++)
#pragma unroll
                        for (int k = 0; k < 3; k++) {
                            t0[q][k] = tb0[(q * 3 + k) * NP1 + c0];
                            t1[q][k] = tb1[(q * 3 + k) * NP1 + c1];
                        }
                    double acc = 0.0;
                    static_for<NR>([&](auto RR) {
                        constexpr int rr = decltype(RR)::value;
                        constexpr int c = L::R.c[rr];
                        static_for<KS::nterms(c)>([&](auto TT) {
                            constexpr int tt = decltype(TT)::value;
                            constexpr int o0 = KS::ord(c, tt, 0), o1 = KS::ord(c, tt, 1);
#pragma unroll
                            for (int q0 = 0; q0 < NQ1; q0++) {
                                double s1 = 0.0;
#pragma unroll
                                for (int q1 = 0; q1 < NQ1; q1++) s1 += t1[q1][o1] * Rg[rr * NQ + q0 * NQ1 + q1];
                                acc += t0[q0][o0] * s1;
                            }
                        });
                    });
                    atomicAdd(Fout + fIdx[nidx], sw * acc);           // red.global (no return value)
                }
                // (3) Jacobian column B = t
                if constexpr (JAC) {
                    double Kc[NEN];
                    // elements inside both axes' uniform runs take the constant-operand tables
                    const int ge0 = e0lo + le0, ge1 = e1lo + le1;
                    if (dbg & 1) {
#pragma unroll
                        for (int A = 0; A < NEN; A++) Kc[A] = gs[A];
                    } else if constexpr (UNI == 2)
                        tsf_column_2d<L, KS, P, true>(Kc, gs, tb0, tb1, c0, c1, ut);
                    else if (UNI == 1 && ge0 >= A0.uni_lo && ge0 < A0.uni_hi && ge1 >= A1.uni_lo && ge1 < A1.uni_hi)
                        tsf_column_2d<L, KS, P, true>(Kc, gs, tb0, tb1, c0, c1, ut);
                    else
                        tsf_column_2d<L, KS, P, false>(Kc, gs, tb0, tb1, c0, c1, ut);
                    // column B of the element block straight into the CSR rows with red.global.add
                    // (fire-and-forget; rows of a tile stay L2-resident): entry (A, B) at
                    // rowOff(A) + pos0(a0 -> b0) W1(A) + pos1(a1 -> b1)
#pragma unroll
                    for (int A = 0; A < NEN; A++) {
                        if (dbg & 2) { if (Kc[A] == 1.2345e300) val[0] = 0.0; continue; }
                        const int a0 = A / NP1, a1 = A % NP1;
                        const int ridx = (fo0 + a0) * NB1 + fo1 + a1;
                        const double sa = s.wts ? nw[ridx] : 1.0;
                        const int p0 = pd0[(fo0 + a0) * W2 + c0 - a0 + P], p1 = pd1[(fo1 + a1) * W2 + c1 - a1 + P];
                        atomicAdd(val + rowOff[ridx] + (long long)p0 * rowW1[ridx] + p1, sa * sw * Kc[A]);
                    }
                }
            }
            __syncwarp();
        }
        __syncthreads();
    }
    if (errbits) atomicOr(s.errflag, errbits);
}

template <int P, class PH, int MODE>
static size_t fused2d_smem(bool jac) {
    using L = Lists<PH, 2, MODE>;
    using TL = Tile2<P>;
    constexpr int NQ1 = P + 1, NP1 = P + 1, NQ = NQ1 * NQ1;
    constexpr int NGRP = TL::NWARP * (32 / (NP1 * NP1));
    constexpr int SFN = (P == 3 || MODE == MODE_NURBS)
                            ? (NP1 * NQ1 * ((MODE == MODE_NURBS ? 3 : 0) + 1 + (PH::UDOT ? 1 : 0)) * 3 + NQ - 1) / NQ : 0;
    const int NBN = TL::NB0 * TL::NB1;
    size_t n = 5 * (size_t)NBN + 2 * TL::TE1 * NQ1 * 3 * NP1 + 4 * TL::TE1 * NQ1
               + 2 * TL::TE1 + (size_t)NGRP * ((jac ? L::NE + L::NR : std::max(L::NR, SFN)) * NQ + (P == 3 ? 1 : 0));
    // scatter metadata: rowOff, fIdx (8 B) + rowW1 (4 B) per node, posd tables
    return n * sizeof(double) + (size_t)NBN * 20 + (size_t)(TL::NB0 + TL::NB1) * (2 * P + 1) * sizeof(int);
}

template <int P, class PH, int MODE, bool JAC, int UNI>
static iga_status launch_k2(iga_space_s *s, const Prm &prm, double a, double b, const double *U, const double *Ud,
                            double *val, double *F, int ne0, int ne1, const UniTab2<P> &ut, cudaStream_t st, int nsm) {
    using TL = Tile2<P>;
    constexpr int NT = 32 * TL::NWARP;
    const size_t smem = fused2d_smem<P, PH, MODE>(JAC);
    {   // the opt-in is a per-device attribute: set it on the current device before every launch
        cudaError_t ce = cudaFuncSetAttribute(k_fused2d<P, PH, MODE, JAC, UNI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem);
        if (ce != cudaSuccess) { set_error(std::string("fused2d smem: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2d<P, PH, MODE, JAC, UNI>, NT, smem);
    occ = std::max(occ, 1);
    // tile width along axis 1: fewest whole rounds of the persistent CTAs times the per-tile work
    // (te1 + P node columns), ties to the wider tile
    const int nt0 = (ne0 + TL::TE0 - 1) / TL::TE0, slots = nsm * occ;
    int te1 = TL::TE1;
    long long best = -1;
    for (int w = TL::TE1; w >= std::max(4, TL::TE1 / 2); w--) {
        const long long nt = (long long)nt0 * ((ne1 + w - 1) / w);
        const long long cost = ((nt + slots - 1) / slots) * (w + P);
        if (best < 0 || cost < best) { best = cost; te1 = w; }
    }
    const int nt1 = (ne1 + te1 - 1) / te1;
    const int grid = (int)std::min<long long>((long long)nt0 * nt1, slots);
    ProfScope ps(s, "k_fused2d", st);
    k_fused2d<P, PH, MODE, JAC, UNI><<<grid, NT, smem, st>>>(s->dev, prm, a, b, U, Ud, val, F, nt0, nt1, te1, s->dbg, ut);
    return IGA_OK;
}

template <int P, class PH, int MODE>
iga_status run_fused2d(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U, const double *Ud,
                       double *val, double *F, cudaStream_t st, int nsm) {
    using TL = Tile2<P>;
    Prm prm;
    for (int i = 0; i < 8; i++) prm.p[i] = phys->p[i];
    const bool jac = val != nullptr;
    const int ne0 = s->el_hi[0] - s->el_lo[0], ne1 = s->el_hi[1] - s->el_lo[1];
    // fast path whenever both axes have a uniform run (all elements on periodic knots, all but p at
    // each end on open uniform knots); the kernel checks each element against the runs
    const bool runs = s->dev.ax[0].uni_hi > s->dev.ax[0].uni_lo && s->dev.ax[1].uni_hi > s->dev.ax[1].uni_lo;
    const int uni = s->force_general ? 0 : (s->tab_uniform[0] && s->tab_uniform[1]) ? 2 : runs ? 1 : 0;
    UniTab2<P> ut{};
    if (uni)
        for (int d = 0; d < 2; d++)
            for (int i = 0; i < (P + 1) * 3 * (P + 1); i++) (&ut.t[d][0][0][0])[i] = s->tab0[d][i];
    int launches = 0;
    if ((F || jac) && !s->skip_zero) {
        // CSR values (rows not complete inside one element receive red.add) and residual, one launch
        ProfScope ps(s, "k_zero", st);
        k_zero_pair(val, jac ? s->nnz_owned : 0, F, F ? s->nrows_owned : 0, st, nsm);
        launches++;
    }
    iga_status r;
    if (jac) r = uni == 2 ? launch_k2<P, PH, MODE, true, 2>(s, prm, a, b, U, Ud, val, F, ne0, ne1, ut, st, nsm)
               : uni == 1 ? launch_k2<P, PH, MODE, true, 1>(s, prm, a, b, U, Ud, val, F, ne0, ne1, ut, st, nsm)
                          : launch_k2<P, PH, MODE, true, 0>(s, prm, a, b, U, Ud, val, F, ne0, ne1, ut, st, nsm);
    else r = launch_k2<P, PH, MODE, false, 0>(s, prm, a, b, U, Ud, val, F, ne0, ne1, ut, st, nsm);
    if (r != IGA_OK) return r;
    launches++;
    s->last_launches = launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("fused2d launch: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

// dispatch: returns IGA_ERR_STATE if the fused 2D path does not apply (caller falls back)
iga_status launch_fused2d(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                          const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    if (s->dim != 2 || s->dof != 1) return IGA_ERR_STATE;
    if (!s->dev.ax[0].uniform || !s->dev.ax[1].uniform) return IGA_ERR_STATE;
    if (s->p[0] != s->p[1]) return IGA_ERR_STATE;
    const int p = s->p[0];
    const bool nurbs = s->mode == MODE_NURBS;
    if (ph->kind == IGA_PHYS_LAPLACE) {
        if (p == 2) return nurbs ? run_fused2d<2, PhysLaplace, MODE_NURBS>(s, ph, a, b, U, Ud, val, F, st, nsm)
                                 : run_fused2d<2, PhysLaplace, MODE_PARAM>(s, ph, a, b, U, Ud, val, F, st, nsm);
        if (p == 3) return nurbs ? run_fused2d<3, PhysLaplace, MODE_NURBS>(s, ph, a, b, U, Ud, val, F, st, nsm)
                                 : run_fused2d<3, PhysLaplace, MODE_PARAM>(s, ph, a, b, U, Ud, val, F, st, nsm);
    }
    if (ph->kind == IGA_PHYS_CAHN_HILLIARD) {
        if (p == 2) return nurbs ? run_fused2d<2, PhysCahnHilliard, MODE_NURBS>(s, ph, a, b, U, Ud, val, F, st, nsm)
                                 : run_fused2d<2, PhysCahnHilliard, MODE_PARAM>(s, ph, a, b, U, Ud, val, F, st, nsm);
        if (p == 3) return nurbs ? run_fused2d<3, PhysCahnHilliard, MODE_NURBS>(s, ph, a, b, U, Ud, val, F, st, nsm)
                                 : run_fused2d<3, PhysCahnHilliard, MODE_PARAM>(s, ph, a, b, U, Ud, val, F, st, nsm);
    }
    return IGA_ERR_STATE;
}

}  // namespace iga
