// fused2dm.cu -- K3/K4 for 2D parametric spaces with several dofs per node (Navier-Stokes-Korteweg,
// SURVEY §8(f) rank 4): one WARP per element, four independent warps per CTA (warp-level
// synchronisation only), Alg. 4 in phases inside the warp's shared-memory slice:
//   1. stage U_e, Udot_e, the element's 1D tables, Gauss data, Alg. 3 positions and row starts;
//   2. field kinds Phi[q][m][k], sum factorised over the element's functions (lane = (q, m));
//   3. per point physics state and residual coefficients (lane = q);
//   4. Jacobian coefficient columns, warp-uniform trial column (k2, j), lane = q, into dense
//      per-(i, j) blocks D[q][i,j][trial kind][test kind];
//   5. test-side sum factorisation (lane = (B, j), loop over i) -> red.global.add straight into
//      the CSR rows (closed-form positions);
//   6. F_e sum factorised (lane = (A, i)).
// The 3D kernel (fused3d.cu) uses a CTA per element; in 2D an element's work fits one warp.
#include "iga_host.h"
#include "pointwise.cuh"

namespace iga {

template <int P, class PH>
struct F2M {
    static constexpr int M = PH::M;
    static constexpr int NP1 = P + 1, NQ1 = P + 1, NQ = NQ1 * NQ1, NEN = NP1 * NP1;
    static constexpr int WARPS = 4;                                   // elements in flight per CTA
    using L = Lists<PH, 2, MODE_PARAM>;
    using KS = typename L::KS;
    static constexpr int NKS = KS::NKS, NR = L::NR, NTK = L::NTK, NQK = L::NQK;
    static constexpr int DB = NTK * NQK;                              // dense block [trial kind][test kind]
    static constexpr int DQS = M * M * DB + 1;                        // q stride (odd: spread banks)
    using State = typename PH::template State<2>;
    static constexpr int STD = (sizeof(State) + 7) / 8;
    // per-warp slice (doubles)
    static constexpr int O_U = 0;                                     // [NEN][M]
    static constexpr int O_UD = O_U + NEN * M;                        // [NEN][M]
    static constexpr int O_TAB = O_UD + NEN * M;                      // [2][NQ1][3][NP1]
    static constexpr int O_QW = O_TAB + 2 * NQ1 * 3 * NP1;            // [2][NQ1]
    static constexpr int O_QX = O_QW + 2 * NQ1;                       // [2][NQ1]
    static constexpr int O_HP = O_QX + 2 * NQ1;                       // [2]
    static constexpr int O_PHI = O_HP + 2;                            // [NQ][M][NKS+1]
    static constexpr int O_ST = O_PHI + NQ * M * (NKS + 1);           // [NQ][STD]
    static constexpr int O_DV = O_ST + NQ * STD;                      // [NQ]
    static constexpr int O_R = O_DV + NQ;                             // [NR][NQ]
    static constexpr int O_D = O_R + NR * NQ;                         // [NQ][DQS]
    static constexpr int O_RS = O_D + NQ * DQS;                       // long long [NEN*M]
    static constexpr int O_ND = O_RS + NEN * M;                       // long long [NEN]
    static constexpr int O_POS = O_ND + NEN;                          // int [2][NP1][NP1] (packed)
    static constexpr int O_W = O_POS + (2 * NP1 * NP1 + 1) / 2;       // int [2][NP1] (packed)
    static constexpr int SLICE = O_W + (2 * NP1 + 1) / 2 + 1;
    static constexpr size_t SMEM = (size_t)WARPS * SLICE * sizeof(double);
    static_assert(NEN * M <= 32 && NQ * M <= 32 && NQ <= 32, "one warp per element");
};

template <int P, class PH, bool JAC>
__global__ void __launch_bounds__(32 * F2M<P, PH>::WARPS)
k_fused2dm(SpaceDev s, Prm prm, double a, double b, const double *__restrict__ U, const double *__restrict__ Ud,
           double *__restrict__ val, double *__restrict__ Fout, long long nelem) {
    using F = F2M<P, PH>;
    using L = typename F::L;
    using KS = typename F::KS;
    using State = typename F::State;
    constexpr int M = F::M, NP1 = F::NP1, NQ1 = F::NQ1, NQ = F::NQ, NEN = F::NEN;
    constexpr int NKS = F::NKS, NR = F::NR, NTK = F::NTK, NQK = F::NQK, DB = F::DB;
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double *W = sm + (size_t)wid * F::SLICE;
    double *sU = W + F::O_U, *sUd = W + F::O_UD, *sTab = W + F::O_TAB, *sQW = W + F::O_QW, *sQX = W + F::O_QX;
    double *sHP = W + F::O_HP, *sPhi = W + F::O_PHI, *sDV = W + F::O_DV, *sR = W + F::O_R, *sD = W + F::O_D;
    State *sSt = reinterpret_cast<State *>(W + F::O_ST);
    long long *sRS = reinterpret_cast<long long *>(W + F::O_RS);
    long long *sNode = reinterpret_cast<long long *>(W + F::O_ND);
    int *sPos = reinterpret_cast<int *>(W + F::O_POS), *sWd = reinterpret_cast<int *>(W + F::O_W);
    const AxisDev &A0 = s.ax[0], &A1 = s.ax[1];
    const int n1 = A1.el_hi - A1.el_lo;
    int errbits = 0;
    auto T = [&](int d, int q, int k, int aa) -> double { return sTab[((d * NQ1 + q) * 3 + k) * NP1 + aa]; };

    for (long long el = (long long)blockIdx.x * F::WARPS + wid; el < nelem; el += (long long)gridDim.x * F::WARPS) {
        const int e0 = A0.el_lo + (int)(el / n1), e1 = A1.el_lo + (int)(el % n1);
        const int ee[2] = {e0, e1};
        // ---- 1. stage ----
        for (int i = lane; i < 2 * NQ1 * 3 * NP1 + 4 * NQ1 + 2 + 2 * NP1 * NP1 + 2 * NP1; i += 32) {
            int k = i;
            if (k < 2 * NQ1 * 3 * NP1) {
                const int d = k / (NQ1 * 3 * NP1);
                sTab[k] = s.ax[d].tab[(size_t)ee[d] * NQ1 * 3 * NP1 + k % (NQ1 * 3 * NP1)];
                continue;
            }
            k -= 2 * NQ1 * 3 * NP1;
            if (k < 4 * NQ1) {
                const int w = k / (2 * NQ1), r = k % (2 * NQ1), d = r / NQ1, q = r % NQ1;
                if (w == 0) sQW[r] = s.ax[d].qw[(size_t)ee[d] * NQ1 + q];
                else sQX[r] = s.ax[d].qx[(size_t)ee[d] * NQ1 + q];
                continue;
            }
            k -= 4 * NQ1;
            if (k < 2) { sHP[k] = s.ax[k].hpar[ee[k]]; continue; }
            k -= 2;
            if (k < 2 * NP1 * NP1) {
                const int d = k / (NP1 * NP1);
                sPos[k] = s.ax[d].pos[(size_t)ee[d] * NP1 * NP1 + k % (NP1 * NP1)];
                continue;
            }
            k -= 2 * NP1 * NP1;
            {
                const int d = k / NP1, aa = k % NP1;
                int g = s.ax[d].first[ee[d]] + aa;
                if (g >= s.ax[d].nu) g -= s.ax[d].nu;
                sWd[k] = s.ax[d].rowW[g];
            }
        }
        for (int k = lane; k < NEN * M; k += 32) {
            const int A = k / M, m = k - A * M, a0 = A / NP1, a1 = A % NP1;
            int g0 = A0.first[e0] + a0, g1 = A1.first[e1] + a1;
            if (g0 >= A0.nu) g0 -= A0.nu;
            if (g1 >= A1.nu) g1 -= A1.nu;
            const long long node = local_node(s, g0, g1, 0);
            sU[k] = U[node * M + m];
            sUd[k] = Ud ? Ud[node * M + m] : 0.0;
            if (m == 0) sNode[A] = node;
            if (JAC) sRS[k] = row_start(s, val, g0, g1, 0, m, M) - val;
        }
        __syncwarp();
        // ---- 2. field kinds (lane = (q, m)), sum factorised ----
        if (lane < NQ * M) {
            const int q = lane / M, m = lane - q * M, q0 = q / NQ1, q1 = q % NQ1;
            double s1[NP1][3], d1[NP1];
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) {
#pragma unroll
                for (int o = 0; o < 3; o++) {
                    double t = 0.0;
#pragma unroll
                    for (int a1 = 0; a1 < NP1; a1++) t += T(1, q1, o, a1) * sU[(a0 * NP1 + a1) * M + m];
                    s1[a0][o] = t;
                }
                double t = 0.0;
                if constexpr (PH::UDOT) {
#pragma unroll
                    for (int a1 = 0; a1 < NP1; a1++) t += T(1, q1, 0, a1) * sUd[(a0 * NP1 + a1) * M + m];
                }
                d1[a0] = t;
            }
            double *dst = sPhi + (q * M + m) * (NKS + 1);
            static_for<NKS>([&](auto K) {
                constexpr int k = decltype(K)::value;
                double pv = 0.0;
                static_for<KS::nterms(k)>([&](auto TT) {
                    constexpr int t = decltype(TT)::value;
                    constexpr int o0 = KS::ord(k, t, 0), o1 = KS::ord(k, t, 1);
#pragma unroll
                    for (int a0 = 0; a0 < NP1; a0++) pv += T(0, q0, o0, a0) * s1[a0][o1];
                });
                dst[k] = pv;
            });
            double pt = 0.0;
#pragma unroll
            for (int a0 = 0; a0 < NP1; a0++) pt += T(0, q0, 0, a0) * d1[a0];
            dst[NKS] = pt;
        }
        __syncwarp();
        // ---- 3. physics per point (lane = q) ----
        if (lane < NQ) {
            const int q = lane, q0 = q / NQ1, q1 = q % NQ1;
            Fields<2, M> Fq;
#pragma unroll
            for (int m = 0; m < M; m++) {
                const double *ph = sPhi + (q * M + m) * (NKS + 1);
                Fq.u[m] = ph[0];
                Fq.gu[m][0] = ph[1];
                Fq.gu[m][1] = ph[2];
                Fq.lu[m] = PH::HESS ? ph[NKS - 1] : 0.0;
                Fq.ut[m] = ph[NKS];
            }
            const int qq[2] = {q0, q1};
#pragma unroll
            for (int i = 0; i < 2; i++) {
                Fq.x[i] = sQX[i * NQ1 + qq[i]];
                Fq.hpar[i] = sHP[i];
#pragma unroll
                for (int j = 0; j < 2; j++) Fq.dxi[i][j] = (i == j) ? 1.0 : 0.0;
            }
            const double dV = sQW[q0] * sQW[NQ1 + q1];
            State st;
            PH::template prepare<2>(prm.p, Fq, st);
            sSt[q] = st;
            sDV[q] = dV;
            if (Fout) {
                double r[NKS * M];
                PH::template residual<2>(st, r);
                double chk = 0.0;
                static_for<NR>([&](auto RR) {
                    constexpr int rr = decltype(RR)::value;
                    const double v = r[L::R.c[rr] * M + L::R.i[rr]] * dV;
                    chk += v;
                    sR[rr * NQ + q] = v;
                });
                if (!isfinite(chk)) errbits |= 2;
            }
        }
        __syncwarp();
        if constexpr (JAC) {
            // ---- 4. coefficient columns (warp-uniform trial column (kq, j), lane = q) ----
            if (lane < NQ) {
                const int q = lane;
                const State st = sSt[q];
                const double dV = sDV[q];
                double chk = 0.0;
                static_for<NQK * M>([&](auto KJ) {
                    constexpr int kq = decltype(KJ)::value / M, j = decltype(KJ)::value % M;
                    double col[NKS * M];
                    PH::template dcol<2>(st, L::qk(kq), j, a, b, col);
#pragma unroll
                    for (int i = 0; i < M; i++) {
                        double *dst = sD + q * F::DQS + (i * M + j) * DB + kq * NTK;
                        static_for<NTK>([&](auto TK) {
                            constexpr int t = decltype(TK)::value;
                            const double v = col[L::tk(t) * M + i] * dV;
                            chk += v;
                            dst[t] = v;
                        });
                    }
                });
                if (!isfinite(chk)) errbits |= 2;
            }
            __syncwarp();
            // ---- 5. test-side sum factorisation, lane = (B, J), loop over test component I ----
            if (lane < NEN * M) {
                const int B = lane / M, J = lane - B * M, b0 = B / NP1, b1 = B % NP1;
#pragma unroll 1
                for (int I = 0; I < M; I++) {
                    double Kc[NEN];
#pragma unroll
                    for (int A = 0; A < NEN; A++) Kc[A] = 0.0;
                    const double *Db = sD + (I * M + J) * DB;
#pragma unroll
                    for (int q0 = 0; q0 < NQ1; q0++) {
                        double S[3][NP1];
#pragma unroll
                        for (int o = 0; o < 3; o++)
#pragma unroll
                            for (int x = 0; x < NP1; x++) S[o][x] = 0.0;
#pragma unroll
                        for (int q1 = 0; q1 < NQ1; q1++) {
                            const int q = q0 * NQ1 + q1;
                            double pb[NQK];
                            static_for<NQK>([&](auto K) {
                                constexpr int kq = decltype(K)::value;
                                constexpr int c = L::qk(kq);
                                double v = 0.0;
                                static_for<KS::nterms(c)>([&](auto TT) {
                                    constexpr int t = decltype(TT)::value;
                                    v += T(0, q0, KS::ord(c, t, 0), b0) * T(1, q1, KS::ord(c, t, 1), b1);
                                });
                                pb[kq] = v;
                            });
                            double H[NTK];
#pragma unroll
                            for (int t = 0; t < NTK; t++) H[t] = 0.0;
                            const double *Dq = Db + q * F::DQS;
#pragma unroll
                            for (int kq = 0; kq < NQK; kq++)
#pragma unroll
                                for (int t = 0; t < NTK; t++) H[t] += Dq[kq * NTK + t] * pb[kq];
                            static_for<NTK>([&](auto TK) {
                                constexpr int t = decltype(TK)::value;
                                constexpr int c = L::tk(t);
                                static_for<KS::nterms(c)>([&](auto TT) {
                                    constexpr int tt = decltype(TT)::value;
                                    constexpr int o0 = KS::ord(c, tt, 0), o1 = KS::ord(c, tt, 1);
#pragma unroll
                                    for (int a1 = 0; a1 < NP1; a1++) S[o0][a1] += H[t] * T(1, q1, o1, a1);
                                });
                            });
                        }
#pragma unroll
                        for (int o0 = 0; o0 < 3; o0++)
#pragma unroll
                            for (int a0 = 0; a0 < NP1; a0++) {
                                const double t0 = T(0, q0, o0, a0);
#pragma unroll
                                for (int a1 = 0; a1 < NP1; a1++) Kc[a0 * NP1 + a1] += t0 * S[o0][a1];
                            }
                    }
                    // entry (A, B) of row A: ((pos0 W1(A) + pos1)) nodes into the row
#pragma unroll
                    for (int A = 0; A < NEN; A++) {
                        const int a0 = A / NP1, a1 = A % NP1;
                        const int co = sPos[a0 * NP1 + b0] * sWd[NP1 + a1] + sPos[NP1 * NP1 + a1 * NP1 + b1];
                        atomicAdd(val + sRS[A * M + I] + (long long)co * M + J, Kc[A]);
                    }
                }
            }
        }
        // ---- 6. residual F_e[A, i], lane = (A, i), sum factorised per test term ----
        if (Fout && lane < NEN * M) {
            const int A = lane / M, Ii = lane - A * M, a0 = A / NP1, a1 = A % NP1;
            double acc = 0.0;
            static_for<NR>([&](auto RR) {
                constexpr int rr = decltype(RR)::value;
                constexpr int c = L::R.c[rr], ri = L::R.i[rr];
                if (ri == Ii) {
                    static_for<KS::nterms(c)>([&](auto TT) {
                        constexpr int tt = decltype(TT)::value;
                        constexpr int o0 = KS::ord(c, tt, 0), o1 = KS::ord(c, tt, 1);
#pragma unroll
                        for (int q0 = 0; q0 < NQ1; q0++) {
                            double s1 = 0.0;
#pragma unroll
                            for (int q1 = 0; q1 < NQ1; q1++) s1 += T(1, q1, o1, a1) * sR[rr * NQ + q0 * NQ1 + q1];
                            acc += T(0, q0, o0, a0) * s1;
                        }
                    });
                }
            });
            atomicAdd(Fout + sNode[A] * M + Ii, acc);
        }
        __syncwarp();
    }
    if (errbits) atomicOr(s.errflag, errbits);
}

template <int P, class PH>
static iga_status run_fused2dm(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                               const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    using FF = F2M<P, PH>;
    Prm prm;
    for (int i = 0; i < 8; i++) prm.p[i] = phys->p[i];
    const bool jac = val != nullptr;
    {   // per-device attribute: set on the current device before every launch
        cudaError_t ce = jac ? cudaFuncSetAttribute(k_fused2dm<P, PH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FF::SMEM)
                             : cudaFuncSetAttribute(k_fused2dm<P, PH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FF::SMEM);
        if (ce != cudaSuccess) { set_error(std::string("fused2dm smem: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    }
    int occ = 1;
    if (jac) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2dm<P, PH, true>, 32 * FF::WARPS, FF::SMEM);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2dm<P, PH, false>, 32 * FF::WARPS, FF::SMEM);
    occ = std::max(occ, 1);
    const long long nel = s->nel_local;
    const int grid = (int)std::min<long long>((nel + FF::WARPS - 1) / FF::WARPS, (long long)nsm * occ);
    int launches = 0;
    if ((jac || F) && !s->skip_zero) {
        ProfScope ps(s, "k_zero", st);
        k_zero_pair(val, jac ? s->nnz_owned : 0, F, F ? s->nrows_owned : 0, st, nsm);
        launches++;
    }
    {
        ProfScope ps(s, "k_fused2dm", st);
        if (jac) k_fused2dm<P, PH, true><<<grid, 32 * FF::WARPS, FF::SMEM, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel);
        else k_fused2dm<P, PH, false><<<grid, 32 * FF::WARPS, FF::SMEM, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel);
        launches++;
    }
    s->last_launches = launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("fused2dm launch: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

// dispatch: IGA_ERR_STATE when this path does not apply (the caller falls back)
iga_status launch_fused2dm(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                           const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    if (s->dim != 2 || s->mode != MODE_PARAM || s->p[0] != 2 || s->p[1] != 2) return IGA_ERR_STATE;
    if (ph->kind == IGA_PHYS_NSK && s->dof == 3) return run_fused2dm<2, PhysNSK>(s, ph, a, b, U, Ud, val, F, st, nsm);
    return IGA_ERR_STATE;
}

}  // namespace iga
