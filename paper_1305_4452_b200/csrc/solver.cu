// solver.cu -- Newton-Krylov linear solve around the assembly (the paper's
// §5 protocol: "30 GMRES iterations per Newton iteration", "block Jacobi ... ILU(0)
// ... in each block").  Right-preconditioned restarted GMRES(m) (Saad 1986, cited P:872) with
// classical Gram-Schmidt and DGKS selective reorthogonalisation (one multi-dot and one fused
// multi-axpy + normalise kernel per pass instead of j dependent dot products), Givens rotations
// on the host.  Preconditioner: block
// Jacobi with ILU(0) in each block.  Reading A-28: on one GPU "one block per process"
// would serialise the triangular solves, so the blocks are contiguous runs of `block_rows` rows
// (default 32): one thread each over packed in-block entries for blocks <= 64 rows, one warp each
// over the CSR otherwise (the factor and the solves are sequential over a block's rows).  All vector work runs in the kernels below; the host only does the (m+1) x m
// Hessenberg least-squares update.
#include <array>
#include <cmath>
#include <cstddef>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "iga_host.h"

namespace iga {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// out[k] += sum_i V[k][i] w[i] for k < nk (V rows of length ld); block partial sums + fp64 atomics
__global__ void k_multidot(long long n, int nk, const double *__restrict__ V, long long ld, const double *__restrict__ w,
                           double *__restrict__ out, const int *__restrict__ gate = nullptr) {
    constexpr int KC = 8;                       // vectors per sweep over w (16: slower, 50 vs 34 us)
    __shared__ double part[8][KC + 1];
    if (gate && !*gate) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int k0 = 0; k0 < nk; k0 += KC) {
        const int kc = min(KC, nk - k0);
        double acc[KC];
#pragma unroll
        for (int k = 0; k < KC; k++) acc[k] = 0.0;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
            const double wi = w[i];
#pragma unroll
            for (int k = 0; k < KC; k++)
                if (k < kc) acc[k] += V[(k0 + k) * ld + i] * wi;
        }
#pragma unroll
        for (int k = 0; k < KC; k++) {
            if (k < kc) {
                const double v = warp_sum(acc[k]);
                if (lane == 0) part[wid][k] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x < kc) {
            double s = 0.0;
            for (int q = 0; q < (int)(blockDim.x >> 5); q++) s += part[q][threadIdx.x];
            atomicAdd(out + k0 + threadIdx.x, s);
        }
        __syncthreads();
    }
}

// w = (w - sum_k V[k] h[k]) * scale
__global__ void k_multiaxpy(long long n, int nk, const double *__restrict__ V, long long ld, const double *__restrict__ h,
                            double *w, double scale, const double *__restrict__ dscale = nullptr,
                            const int *__restrict__ gate = nullptr) {
    if (gate && !*gate) return;
    if (dscale) scale = *dscale;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double s = w[i];
        for (int k = 0; k < nk; k++) s -= h[k] * V[k * ld + i];
        w[i] = s * scale;
    }
}

// y = alpha x + beta y
__global__ void k_axpby(long long n, double alpha, const double *__restrict__ x, double beta, double *__restrict__ y) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = alpha * x[i] + beta * y[i];
}

// position of the diagonal entry of every row (-1 if absent)
__global__ void k_diagpos(long long n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, int64_t *__restrict__ dp) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long lo = rp[i], hi = rp[i + 1] - 1, pos = -1;
    while (lo <= hi) {
        const long long mid = (lo + hi) >> 1;
        if (ci[mid] == i) { pos = mid; break; }
        if (ci[mid] < i) lo = mid + 1; else hi = mid - 1;
    }
    dp[i] = pos;
}

__device__ __forceinline__ long long find_col(const int64_t *rp, const int32_t *ci, long long row, int col) {
    long long lo = rp[row], hi = rp[row + 1] - 1;
    while (lo <= hi) {
        const long long mid = (lo + hi) >> 1;
        const int c = ci[mid];
        if (c == col) return mid;
        if (c < col) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

// ILU(0) of each diagonal block [r0, r0+B) (IKJ variant, Saad's ILU(0)): warp per block, rows in
// order, for each lower entry k of the row (ascending): l_ik = a_ik / u_kk, then a_ij -= l_ik u_kj
// for the row's entries j > k (lanes), u_kj found by binary search in row k.  Entries whose column
// leaves the block are not part of the preconditioner.
__global__ void k_ilu0(long long n, int B, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                       const int64_t *__restrict__ dp, double *__restrict__ lu) {
    const long long blk = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long r0 = blk * B;
    if (r0 >= n) return;
    const long long r1 = min(n, r0 + B);
    for (long long i = r0; i < r1; i++) {
        const long long pb = rp[i], pe = rp[i + 1];
        for (long long p = pb; p < pe; p++) {
            const int k = ci[p];
            if (k >= i) break;
            if (k < r0) continue;
            double lik = 0.0;
            if (lane == 0) lik = lu[p] / lu[dp[k]];
            lik = __shfl_sync(0xffffffffu, lik, 0);
            __syncwarp();
            if (lane == 0) lu[p] = lik;
            for (long long q = p + 1 + lane; q < pe; q += 32) {
                const int j = ci[q];
                if (j >= r1) continue;
                const long long kq = find_col(rp, ci, k, j);
                if (kq >= 0) lu[q] -= lik * lu[kq];
            }
            __syncwarp();
        }
    }
}

// z = (LU)^{-1} r per block: forward (unit L) then backward (U), warp per block
__global__ void k_ilu0_solve(long long n, int B, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                             const int64_t *__restrict__ dp, const double *__restrict__ lu, const double *__restrict__ r,
                             double *__restrict__ z) {
    const long long blk = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long r0 = blk * B;
    if (r0 >= n) return;
    const long long r1 = min(n, r0 + B);
    for (long long i = r0; i < r1; i++) {
        double s = 0.0;
        for (long long p = rp[i] + lane; p < dp[i]; p += 32) {
            const int k = ci[p];
            if (k >= r0) s += lu[p] * z[k];
        }
        s = warp_sum(s);
        if (lane == 0) z[i] = r[i] - s;
        __syncwarp();
    }
    for (long long i = r1 - 1; i >= r0; i--) {
        double s = 0.0;
        for (long long p = dp[i] + 1 + lane; p < rp[i + 1]; p += 32) {
            const int j = ci[p];
            if (j < r1) s += lu[p] * z[j];
        }
        s = warp_sum(s);
        if (lane == 0) z[i] = (z[i] - s) / lu[dp[i]];
        __syncwarp();
    }
}

// Same solve for blocks of <= 1024 rows, latency-hidden: the block's z lives in shared memory and
// the rows are taken in groups of G whose (independent) row-pointer / first-chunk / rhs loads are
// all issued before the group's sequential dependency chain runs out of shared memory.
constexpr int ILU_G = 8;
__global__ void __launch_bounds__(128) k_ilu0_solve_g(long long n, int B, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ ci, const int64_t *__restrict__ dp,
                                                      const double *__restrict__ lu, const double *__restrict__ r,
                                                      double *__restrict__ z) {
    extern __shared__ double zsm[];
    const long long blk = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    double *zs = zsm + (threadIdx.x >> 5) * B;
    const long long r0 = blk * B;
    if (r0 >= n) return;
    const int nb = (int)min((long long)B, n - r0);
    for (int i0 = 0; i0 < nb; i0 += ILU_G) {
        long long pb[ILU_G], pd[ILU_G];
        double rr[ILU_G], lc[ILU_G];
        int kc[ILU_G];
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            const long long i = r0 + min(i0 + g, nb - 1);
            pb[g] = rp[i];
            pd[g] = dp[i];
            rr[g] = r[i];
        }
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            const long long p = pb[g] + lane;
            kc[g] = -1;
            lc[g] = 0.0;
            if (p < pd[g]) { kc[g] = (int)(ci[p] - r0); lc[g] = lu[p]; }
        }
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            if (i0 + g < nb) {
                double s = kc[g] >= 0 ? lc[g] * zs[kc[g]] : 0.0;
                for (long long p = pb[g] + 32 + lane; p < pd[g]; p += 32) {
                    const long long k = ci[p] - r0;
                    if (k >= 0) s += lu[p] * zs[k];
                }
                s = warp_sum(s);
                if (lane == 0) zs[i0 + g] = rr[g] - s;
                __syncwarp();
            }
        }
    }
    for (int i0 = nb - 1; i0 >= 0; i0 -= ILU_G) {
        long long pd[ILU_G], pe[ILU_G];
        double dv[ILU_G], lc[ILU_G];
        int jc[ILU_G];
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            const long long i = r0 + max(i0 - g, 0);
            pd[g] = dp[i];
            pe[g] = rp[i + 1];
        }
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            const long long p = pd[g] + 1 + lane;
            dv[g] = lu[pd[g]];
            jc[g] = -1;
            lc[g] = 0.0;
            if (p < pe[g]) {
                const long long j = ci[p] - r0;
                if (j < nb) { jc[g] = (int)j; lc[g] = lu[p]; }
            }
        }
#pragma unroll
        for (int g = 0; g < ILU_G; g++) {
            if (i0 - g >= 0) {
                double s = jc[g] >= 0 ? lc[g] * zs[jc[g]] : 0.0;
                for (long long p = pd[g] + 33 + lane; p < pe[g]; p += 32) {
                    const long long j = ci[p] - r0;
                    if (j < nb) s += lu[p] * zs[j];
                }
                s = warp_sum(s);
                if (lane == 0) zs[i0 - g] = (zs[i0 - g] - s) / dv[g];
                __syncwarp();
            }
        }
    }
    for (int i = lane; i < nb; i += 32) z[r0 + i] = zs[i];
}

// ---- small-block path (block_rows <= 64, the default): one THREAD per block ------------------
// The preconditioner only ever uses a block's in-block entries, so after the pattern is known they
// are packed once per solve into slot-major arrays -- value, 8-bit column offset inside the block --
// indexed ((il * W + slot) * nblk + blk): consecutive lanes (= consecutive blocks) read consecutive
// words, and no load of the solve depends on data (no row_ptr / diag-position chains).  Padding
// slots hold value 0 and offset 0.  The factor (IKJ ILU(0), as k_ilu0) and the triangular solves
// then run as one sequential chain per thread, the block's z in a padded shared-memory row.
constexpr int TPB_MAXB = 64, TPB_MAXW = 16, TPB_CTA = 64;

__device__ __forceinline__ long long ell_at(int il, int s, int W, long long nblk, long long blk) {
    return ((long long)il * W + s) * nblk + blk;
}

// in-block lower / upper entry counts of every row -> maxima (wmax[0], wmax[1])
__global__ void k_ell_count(long long n, int B, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            const int64_t *__restrict__ dp, int *__restrict__ wmax) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int nl = 0, nu = 0;
    if (i < n) {
        const long long r0 = (i / B) * B, r1 = min(n, r0 + B);
        for (long long p = rp[i]; p < dp[i]; p++) nl += ci[p] >= r0;
        for (long long p = dp[i] + 1; p < rp[i + 1]; p++) nu += ci[p] < r1;
    }
    nl = __reduce_max_sync(0xffffffffu, nl);
    nu = __reduce_max_sync(0xffffffffu, nu);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(wmax, nl);
        atomicMax(wmax + 1, nu);
    }
}

// pack the in-block entries of A (rows >= n of the ragged last block: empty, D = 1)
__global__ void k_ell_pack(long long n, int B, long long nblk, const int64_t *__restrict__ rp,
                           const int32_t *__restrict__ ci, const int64_t *__restrict__ dp, const double *__restrict__ a,
                           int WL, int WU, double *__restrict__ Lv, uint8_t *__restrict__ Lc, double *__restrict__ Uv,
                           uint8_t *__restrict__ Uc, double *__restrict__ D) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nblk * B) return;
    const long long blk = g / B;
    const int il = (int)(g % B);
    const long long r0 = blk * B, r1 = min(n, r0 + B);
    int sl = 0, su = 0;
    if (g < n) {
        for (long long p = rp[g]; p < dp[g]; p++)
            if (ci[p] >= r0) {
                Lv[ell_at(il, sl, WL, nblk, blk)] = a[p];
                Lc[ell_at(il, sl, WL, nblk, blk)] = (uint8_t)(ci[p] - r0);
                sl++;
            }
        for (long long p = dp[g] + 1; p < rp[g + 1]; p++)
            if (ci[p] < r1) {
                Uv[ell_at(il, su, WU, nblk, blk)] = a[p];
                Uc[ell_at(il, su, WU, nblk, blk)] = (uint8_t)(ci[p] - r0);
                su++;
            }
        D[(long long)il * nblk + blk] = a[dp[g]];
    } else {
        D[(long long)il * nblk + blk] = 1.0;
    }
    for (; sl < WL; sl++) { Lv[ell_at(il, sl, WL, nblk, blk)] = 0.0; Lc[ell_at(il, sl, WL, nblk, blk)] = 0; }
    for (; su < WU; su++) { Uv[ell_at(il, su, WU, nblk, blk)] = 0.0; Uc[ell_at(il, su, WU, nblk, blk)] = 0; }
}

// ILU(0) in place on the packed block, thread per block, row il held in local arrays.  Padding
// lower slots act as k = 0 with a_ik = 0, so l = 0 and they change nothing; padding upper slots
// (offset 0) never match a column j > k >= 0.
__global__ void k_ell_ilu0(long long nblk, int B, int WL, int WU, double *__restrict__ Lv, const uint8_t *__restrict__ Lc,
                           double *__restrict__ Uv, const uint8_t *__restrict__ Uc, double *__restrict__ D) {
    const long long blk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (blk >= nblk) return;
    double lv[TPB_MAXW], uv[TPB_MAXW];
    int lc[TPB_MAXW], uc[TPB_MAXW];
    for (int il = 0; il < B; il++) {
        for (int t = 0; t < WL; t++) { lv[t] = Lv[ell_at(il, t, WL, nblk, blk)]; lc[t] = Lc[ell_at(il, t, WL, nblk, blk)]; }
        for (int t = 0; t < WU; t++) { uv[t] = Uv[ell_at(il, t, WU, nblk, blk)]; uc[t] = Uc[ell_at(il, t, WU, nblk, blk)]; }
        double d = D[(long long)il * nblk + blk];
        for (int t = 0; t < WL; t++) {
            const int k = lc[t];
            const double l = lv[t] / D[(long long)k * nblk + blk];
            lv[t] = l;
            if (l == 0.0) continue;
            for (int s = 0; s < WU; s++) {
                const double ukj = Uv[ell_at(k, s, WU, nblk, blk)];
                const int j = Uc[ell_at(k, s, WU, nblk, blk)];
                if (j <= k) continue;                           // padding
                if (j == il) d -= l * ukj;
                else if (j < il) {
                    for (int t2 = t + 1; t2 < WL; t2++)
                        if (lc[t2] == j) { lv[t2] -= l * ukj; break; }
                } else {
                    for (int t2 = 0; t2 < WU; t2++)
                        if (uc[t2] == j) { uv[t2] -= l * ukj; break; }
                }
            }
        }
        for (int t = 0; t < WL; t++) Lv[ell_at(il, t, WL, nblk, blk)] = lv[t];
        for (int t = 0; t < WU; t++) Uv[ell_at(il, t, WU, nblk, blk)] = uv[t];
        D[(long long)il * nblk + blk] = d;
    }
}

// W = padded slot count (2, 4, 8, 16).  Rows go in chunks of PF whose slot loads (independent of
// the chain) are issued one chunk ahead (double-buffered registers), so the chain of chunk c runs
// out of shared memory while the loads of chunk c+1 are in flight.
template <int W, int PF>
struct EllChunk {
    double v[PF][W], d[PF];
    int k[PF][W];
};

template <int W, int PF, bool LOWER>
__device__ __forceinline__ void ell_load(EllChunk<W, PF> &C, int c0, int B, long long nblk, long long blk,
                                         const double *__restrict__ V, const uint8_t *__restrict__ K,
                                         const double *__restrict__ D) {
#pragma unroll
    for (int q = 0; q < PF; q++) {
        const int il = LOWER ? min(c0 + q, B - 1) : max(c0 - q, 0);
        if (!LOWER) C.d[q] = D[(long long)il * nblk + blk];
#pragma unroll
        for (int t = 0; t < W; t++) {
            C.v[q][t] = V[ell_at(il, t, W, nblk, blk)];
            C.k[q][t] = K[ell_at(il, t, W, nblk, blk)];
        }
    }
}

template <int W, int PF, bool LOWER>
__device__ __forceinline__ void ell_chain(const EllChunk<W, PF> &C, int c0, int B, double *my) {
#pragma unroll
    for (int q = 0; q < PF; q++) {
        const int il = LOWER ? c0 + q : c0 - q;
        if (LOWER ? il < B : il >= 0) {
            double acc = my[il];
#pragma unroll
            for (int t = 0; t < W; t++) acc -= C.v[q][t] * my[C.k[q][t]];
            my[il] = LOWER ? acc : acc / C.d[q];
        }
    }
}

template <int W>
__global__ void __launch_bounds__(TPB_CTA) k_ell_solve(long long n, int B, long long nblk, const double *__restrict__ Lv,
                                                       const uint8_t *__restrict__ Lc, const double *__restrict__ Uv,
                                                       const uint8_t *__restrict__ Uc, const double *__restrict__ D,
                                                       const double *__restrict__ r, double *__restrict__ z) {
    constexpr int PF = W >= 16 ? 1 : 16 / W;
    extern __shared__ double zsm[];
    const int tid = threadIdx.x, ld = B + 1;
    const long long cta_r0 = (long long)blockIdx.x * TPB_CTA * B;
    for (int idx = tid; idx < TPB_CTA * B; idx += TPB_CTA) {
        const long long g = cta_r0 + idx;
        zsm[(idx / B) * ld + idx % B] = g < n ? r[g] : 0.0;
    }
    __syncthreads();
    const long long blk = (long long)blockIdx.x * TPB_CTA + tid;
    if (blk < nblk) {
        double *my = zsm + tid * ld;
        EllChunk<W, PF> A, Bq;
        ell_load<W, PF, true>(A, 0, B, nblk, blk, Lv, Lc, D);
        for (int c = 0; c < B; c += 2 * PF) {
            ell_load<W, PF, true>(Bq, c + PF, B, nblk, blk, Lv, Lc, D);
            ell_chain<W, PF, true>(A, c, B, my);
            ell_load<W, PF, true>(A, c + 2 * PF, B, nblk, blk, Lv, Lc, D);
            ell_chain<W, PF, true>(Bq, c + PF, B, my);
        }
        ell_load<W, PF, false>(A, B - 1, B, nblk, blk, Uv, Uc, D);
        for (int c = B - 1; c >= 0; c -= 2 * PF) {
            ell_load<W, PF, false>(Bq, c - PF, B, nblk, blk, Uv, Uc, D);
            ell_chain<W, PF, false>(A, c, B, my);
            ell_load<W, PF, false>(A, c - 2 * PF, B, nblk, blk, Uv, Uc, D);
            ell_chain<W, PF, false>(Bq, c - PF, B, my);
        }
    }
    __syncthreads();
    for (int idx = tid; idx < TPB_CTA * B; idx += TPB_CTA) {
        const long long g = cta_r0 + idx;
        if (g < n) z[g] = zsm[(idx / B) * ld + idx % B];
    }
}

// y = A x (or bsub - A x) for short rows, CSR-stream: a CTA takes SP_R consecutive rows, streams
// their nonzeros contiguously (coalesced a / col_idx loads, many in flight per thread) into
// shared-memory products, then one thread per row sums its range.  Blocks whose nonzeros exceed
// SP_CAP fall back to one warp per row.
constexpr int SP_R = 128, SP_CAP = 4096;
__global__ void __launch_bounds__(SP_R) k_spmv_stream(long long n, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ ci, const double *__restrict__ a,
                                                      const double *__restrict__ x, double *__restrict__ y,
                                                      const double *__restrict__ bsub) {
    __shared__ double prod[SP_CAP];
    __shared__ long long srp[SP_R + 1];
    const long long row0 = (long long)blockIdx.x * SP_R;
    const int nr = (int)min((long long)SP_R, n - row0);
    for (int i = threadIdx.x; i <= nr; i += SP_R) srp[i] = rp[row0 + i];
    __syncthreads();
    const long long p0 = srp[0], cnt = srp[nr] - p0;
    if (cnt <= SP_CAP) {
#pragma unroll 4
        for (int k = threadIdx.x; k < cnt; k += SP_R) prod[k] = __ldcs(a + p0 + k) * __ldg(x + __ldcs(ci + p0 + k));
        __syncthreads();
        if (threadIdx.x < nr) {
            const int r = threadIdx.x;
            double s = 0.0;
            for (long long k = srp[r] - p0; k < srp[r + 1] - p0; k++) s += prod[k];
            y[row0 + r] = bsub ? bsub[row0 + r] - s : s;
        }
    } else {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int r = wid; r < nr; r += SP_R / 32) {
            double s = 0.0;
            for (long long p = srp[r] + lane; p < srp[r + 1]; p += 32) s += a[p] * __ldg(x + ci[p]);
            s = warp_sum(s);
            if (lane == 0) y[row0 + r] = bsub ? bsub[row0 + r] - s : s;
        }
    }
}

// y = A x with LPR lanes per row (short IGA rows: 4-16 lanes keep the warp's lanes busy)
// (bsub != NULL: y = bsub - A x, the residual)
template <int LPR>
__global__ void k_spmv_sw(long long n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                          const double *__restrict__ a, const double *__restrict__ x, double *__restrict__ y,
                          const double *__restrict__ bsub) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long row = t / LPR;
    const int sub = (int)(t % LPR);
    double s = 0.0;
    if (row < n)
        for (long long p = rp[row] + sub; p < rp[row + 1]; p += LPR) s += a[p] * __ldg(x + ci[p]);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (row < n && sub == 0) y[row] = bsub ? bsub[row] - s : s;
}

// z = D^{-1} r
__global__ void k_jacobi(long long n, const int64_t *__restrict__ dp, const double *__restrict__ a, const double *__restrict__ r,
                         double *__restrict__ z) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        z[i] = r[i] / a[dp[i]];
}

// ---- device-driven Arnoldi control (fixed iteration budget, rtol = 0: the paper's protocol) ----
// The decisions the host makes per iteration in the general path -- DGKS second pass, |h_{j+1}|,
// the Givens update of the Hessenberg column -- are taken by one thread on the device, so a cycle
// is a stream of launches with no host round trip.  Layout of the control block (doubles):
// hbuf[m+2] (multi-dot target), hvec[m+1] (this pass's coefficients), H[(m+1) m], cs[m], sn[m],
// g[m+1], yneg[m], then ArnCtl.
struct ArnCtl {
    double scale, res, beta;
    int need2, jstop;
};
struct ArnLayout {
    int m;
    __host__ __device__ size_t hbuf() const { return 0; }
    __host__ __device__ size_t hvec() const { return m + 2; }
    __host__ __device__ size_t H() const { return 2 * m + 3; }
    __host__ __device__ size_t cs() const { return H() + (size_t)(m + 1) * m; }
    __host__ __device__ size_t sn() const { return cs() + m; }
    __host__ __device__ size_t g() const { return sn() + m; }
    __host__ __device__ size_t yneg() const { return g() + m + 1; }
    __host__ __device__ size_t ctl() const { return (yneg() + m + 1) / 2 * 2; }
    __host__ __device__ size_t total() const { return ctl() + 8; }
};

__global__ void k_arn_start(ArnLayout Lo, double *base) {
    double *hb = base + Lo.hbuf(), *g = base + Lo.g();
    ArnCtl *c = reinterpret_cast<ArnCtl *>(base + Lo.ctl());
    const double beta = sqrt(fmax(hb[0], 0.0));
    hb[0] = 0.0;
    g[0] = beta;
    for (int i = 1; i <= Lo.m; i++) g[i] = 0.0;
    c->beta = beta;
    c->scale = beta > 0.0 ? 1.0 / beta : 1.0;
    c->res = beta;
    // beta = 0: the start vector already solves the system; no column is used, so the update
    // y is 0 (not -0/0) and x stays as it is
    c->jstop = beta > 0.0 ? Lo.m : 0;
    c->need2 = 1;
}

// one warp: lanes load / reduce the column in parallel, lane 0 runs the short sequential part
// (previous rotations, new rotation) out of shared memory
__global__ void __launch_bounds__(32) k_arn_ctrl(ArnLayout Lo, double *base, int j, int pass) {
    const int m = Lo.m, lane = threadIdx.x;
    double *hb = base + Lo.hbuf(), *hv = base + Lo.hvec(), *H = base + Lo.H(), *cs = base + Lo.cs(),
           *sn = base + Lo.sn(), *g = base + Lo.g();
    ArnCtl *c = reinterpret_cast<ArnCtl *>(base + Lo.ctl());
    __shared__ double col[64], scs[64], ssn[64];
    __shared__ int last_s;
    if (pass == 1 && !c->need2) return;
    double hh = 0.0;
    for (int i = lane; i <= j; i += 32) {
        const double h = hb[i];
        hv[i] = h;
        hh += h * h;
        col[i] = (pass == 0 ? 0.0 : H[(size_t)i * m + j]) + h;
        if (i < j) { scs[i] = cs[i]; ssn[i] = sn[i]; }
    }
    hh = warp_sum(hh);
    const double ww = hb[j + 1], nrm2 = ww - hh;
    __syncwarp();
    for (int i = lane; i <= j + 1; i += 32) hb[i] = 0.0;
    if (lane == 0) {
        const bool last = pass == 1 || nrm2 > 0.5 * ww;
        if (pass == 0) c->need2 = last ? 0 : 1;          // gates the second pass's three launches
        c->scale = 1.0;
        last_s = last;
        if (last) {
            const double hj1 = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
            if (hj1 > 0.0) c->scale = 1.0 / hj1;
            for (int i = 0; i < j; i++) {
                const double a0 = col[i], a1 = col[i + 1];
                col[i] = scs[i] * a0 + ssn[i] * a1;
                col[i + 1] = -ssn[i] * a0 + scs[i] * a1;
            }
            const double hjj = col[j], den = hypot(hjj, hj1);
            cs[j] = den > 0.0 ? hjj / den : 1.0;
            sn[j] = den > 0.0 ? hj1 / den : 0.0;
            col[j] = den;
            const double gj = g[j];
            g[j + 1] = -sn[j] * gj;
            g[j] = cs[j] * gj;
            if (c->jstop == m || c->jstop > j) c->res = fabs(g[j + 1]);
            if (hj1 == 0.0 && c->jstop > j + 1) c->jstop = j + 1;   // lucky breakdown: later columns unused
        }
    }
    __syncwarp();
    for (int i = lane; i <= j; i += 32) H[(size_t)i * m + j] = col[i];
}

// y = R^{-1} g over the first min(jmax, jstop) columns; yneg = -y, zero beyond
__global__ void __launch_bounds__(256) k_arn_solve(ArnLayout Lo, double *base, int jmax) {
    const int m = Lo.m;
    const double *H = base + Lo.H(), *g = base + Lo.g();
    double *yn = base + Lo.yneg();
    const ArnCtl *c = reinterpret_cast<const ArnCtl *>(base + Lo.ctl());
    __shared__ double sH[64 * 64], sy[64];
    const int j = min(jmax, c->jstop);
    for (int t = threadIdx.x; t < j * j; t += blockDim.x) sH[t] = H[(size_t)(t / j) * m + t % j];
    for (int t = threadIdx.x; t < j; t += blockDim.x) sy[t] = g[t];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = j - 1; i >= 0; i--) {                 // sy = -y
            double t = sy[i];
            for (int k = i + 1; k < j; k++) t += sH[i * j + k] * sy[k];
            const double d = sH[i * j + i];
            sy[i] = d != 0.0 ? -t / d : 0.0;                // zero pivot (exact breakdown): drop the direction
        }
    __syncthreads();
    for (int t = threadIdx.x; t < jmax; t += blockDim.x) yn[t] = t < j ? sy[t] : 0.0;
}

// device buffer `slot` of the space's solver workspace, grown to >= bytes (contents not kept)
static void *ws_ensure(iga_space_s *s, int slot, size_t bytes) {
    if (s->gm_cap[slot] < bytes) {
        if (s->gm_buf[slot]) cudaFree(s->gm_buf[slot]);
        s->gm_buf[slot] = nullptr;
        s->gm_cap[slot] = 0;
        if (cudaMalloc(&s->gm_buf[slot], bytes) != cudaSuccess) { cudaGetLastError(); s->gm_buf[slot] = nullptr; return nullptr; }
        s->gm_cap[slot] = bytes;
    }
    return s->gm_buf[slot];
}

iga_status gmres_solve(iga_space_s *s, const int64_t *rp, const int32_t *ci, const double *a, const double *b, double *x,
                       const iga_krylov *opt, int *iters_out, double *relres_out, cudaStream_t st) {
    const long long n = s->nrows_owned, nnz = s->nnz_owned;
    const int m = std::max(1, opt->restart), maxit = std::max(0, opt->maxit);
    const int B = opt->block_rows > 0 ? opt->block_rows : 32;
    if (s->nranks > 1) {
        if (!s->dist || dist_transport(s->dist) != IGA_XPORT_NCCL) {
            set_error("gmres: in-process (IGA_XPORT_LOCAL) ranks solve through iga_gmres_group");
            return IGA_ERR_STATE;
        }
        return gmres_group(1, &s, &rp, &ci, &a, &b, &x, opt, iters_out, relres_out, st);
    }
    // workspace, cached on the space (gm_buf): [0] V[m+1][n], Z[m][n], w[n], dp[n], h[2(m+1)];
    // [1] the preconditioner (packed blocks or the CSR copy of the ILU factor)
    auto ensure = [&](int slot, size_t bytes) { return ws_ensure(s, slot, bytes); };
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t szV = al(sizeof(double) * (size_t)(m + 1) * n), szZ = al(sizeof(double) * (size_t)m * n),
                 szw = al(sizeof(double) * (size_t)n), szdp = al(sizeof(int64_t) * (size_t)n),
                 szh = al(sizeof(double) * std::max<size_t>(2 * (size_t)(m + 1), ArnLayout{m}.total()));
    char *base = (char *)ensure(0, szV + szZ + szw + szdp + szh);
    if (!base) { set_error("gmres workspace"); return IGA_ERR_NOMEM; }
    double *V = (double *)base, *Z = (double *)(base + szV), *w = (double *)(base + szV + szZ);
    int64_t *dp = (int64_t *)(base + szV + szZ + szw);
    double *dh = (double *)(base + szV + szZ + szw + szdp);
    double *lu = nullptr, *Lv = nullptr, *Uv = nullptr, *Dd = nullptr;
    uint8_t *Lc = nullptr, *Uc = nullptr;
    cudaError_t ce = cudaSuccess;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    const unsigned gv = (unsigned)std::min<long long>((n + 255) / 256, (long long)nsm * 8);
    const long long avg = n > 0 ? nnz / n : 0;
    const int lpr = avg <= 12 ? 4 : avg <= 40 ? 8 : avg <= 96 ? 16 : 32;
    const unsigned grow = (unsigned)((n * lpr + 255) / 256);
    const bool stream_spmv = avg <= SP_CAP / SP_R && !s->gm_host_ctrl;   // mean row fits the stream tile
    auto spmv = [&](const double *xin, double *yout, const double *bsub) {
        if (stream_spmv) k_spmv_stream<<<(unsigned)((n + SP_R - 1) / SP_R), SP_R, 0, st>>>(n, rp, ci, a, xin, yout, bsub);
        else if (lpr == 4) k_spmv_sw<4><<<grow, 256, 0, st>>>(n, rp, ci, a, xin, yout, bsub);
        else if (lpr == 8) k_spmv_sw<8><<<grow, 256, 0, st>>>(n, rp, ci, a, xin, yout, bsub);
        else if (lpr == 16) k_spmv_sw<16><<<grow, 256, 0, st>>>(n, rp, ci, a, xin, yout, bsub);
        else k_spmv_sw<32><<<grow, 256, 0, st>>>(n, rp, ci, a, xin, yout, bsub);
    };
    const unsigned gblk = (unsigned)((((n + B - 1) / B) * 32 + 127) / 128);
    int launches = 0;
    k_diagpos<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, rp, ci, dp);
    launches++;
    // block-Jacobi ILU(0): packed thread-per-block path for small blocks, CSR warp path otherwise
    const long long nblk = (n + B - 1) / B;
    bool ell = false;
    int WL = 0, WU = 0;
    if (opt->precond == 2 && B <= TPB_MAXB && n > 0) {
        int wm[2] = {0, 0};
        cudaMemsetAsync(dh, 0, 2 * sizeof(int), st);
        k_ell_count<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, B, rp, ci, dp, (int *)dh);
        launches++;
        cudaMemcpyAsync(wm, dh, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const int wmax = std::max(wm[0], wm[1]);
        WL = WU = wmax <= 2 ? 2 : wmax <= 4 ? 4 : wmax <= 8 ? 8 : 16;       // padded slot count
        if (wmax <= TPB_MAXW) {
            const size_t rows = (size_t)nblk * B;
            const size_t sv = al(sizeof(double) * rows * WL), sd = al(sizeof(double) * rows), sc = al(rows * WL);
            char *pb = (char *)ensure(1, 2 * sv + sd + 2 * sc);
            if (!pb) { set_error("gmres workspace"); return IGA_ERR_NOMEM; }
            Lv = (double *)pb;
            Uv = (double *)(pb + sv);
            Dd = (double *)(pb + 2 * sv);
            Lc = (uint8_t *)(pb + 2 * sv + sd);
            Uc = (uint8_t *)(pb + 2 * sv + sd + sc);
            k_ell_pack<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(n, B, nblk, rp, ci, dp, a, WL, WU, Lv, Lc, Uv, Uc, Dd);
            k_ell_ilu0<<<(unsigned)((nblk + 63) / 64), 64, 0, st>>>(nblk, B, WL, WU, Lv, Lc, Uv, Uc, Dd);
            launches += 2;
            ell = true;
        }
    }
    if (opt->precond == 2 && !ell) {
        lu = (double *)ensure(1, sizeof(double) * (size_t)nnz);
        if (!lu) { set_error("gmres workspace"); return IGA_ERR_NOMEM; }
        cudaMemcpyAsync(lu, a, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice, st);
        k_ilu0<<<gblk, 128, 0, st>>>(n, B, rp, ci, dp, lu);
        launches++;
    }
    const unsigned gell = (unsigned)((nblk + TPB_CTA - 1) / TPB_CTA);
    const size_t smell = sizeof(double) * (size_t)TPB_CTA * (B + 1);
    auto precond = [&](const double *r, double *z) {
        if (ell && WL == 2) k_ell_solve<2><<<gell, TPB_CTA, smell, st>>>(n, B, nblk, Lv, Lc, Uv, Uc, Dd, r, z);
        else if (ell && WL == 4) k_ell_solve<4><<<gell, TPB_CTA, smell, st>>>(n, B, nblk, Lv, Lc, Uv, Uc, Dd, r, z);
        else if (ell && WL == 8) k_ell_solve<8><<<gell, TPB_CTA, smell, st>>>(n, B, nblk, Lv, Lc, Uv, Uc, Dd, r, z);
        else if (ell) k_ell_solve<16><<<gell, TPB_CTA, smell, st>>>(n, B, nblk, Lv, Lc, Uv, Uc, Dd, r, z);
        else if (opt->precond == 2 && B <= 1024) k_ilu0_solve_g<<<gblk, 128, 4 * B * sizeof(double), st>>>(n, B, rp, ci, dp, lu, r, z);
        else if (opt->precond == 2) k_ilu0_solve<<<gblk, 128, 0, st>>>(n, B, rp, ci, dp, lu, r, z);
        else if (opt->precond == 1) k_jacobi<<<gv, 256, 0, st>>>(n, dp, a, r, z);
        else cudaMemcpyAsync(z, r, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st);
        launches++;
    };
    auto norm2 = [&](const double *v) -> double {
        cudaMemsetAsync(dh, 0, sizeof(double), st);
        k_multidot<<<gv, 256, 0, st>>>(n, 1, v, n, v, dh);
        launches++;
        double h = 0.0;
        cudaMemcpyAsync(&h, dh, sizeof(double), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        return std::sqrt(h);
    };
    const double bnorm = norm2(b);
    if (opt->rtol == 0.0 && !s->gm_host_ctrl && m <= 62) {   // (k_arn_* stage <= 64 entries in smem)
        // fixed budget: device-driven cycles, one host synchronisation at the end
        const ArnLayout Lo{m};
        int *need2 = reinterpret_cast<int *>(reinterpret_cast<ArnCtl *>(dh + Lo.ctl())) + 6;   // ArnCtl::need2
        const double *dscale = dh + Lo.ctl();                                                   // ArnCtl::scale
        static_assert(offsetof(ArnCtl, need2) == 24 && offsetof(ArnCtl, scale) == 0, "ArnCtl layout");
        cudaMemsetAsync(dh, 0, sizeof(double) * Lo.total(), st);
        int it = 0;
        while (it < maxit && bnorm > 0.0) {
            spmv(x, V, b);
            k_multidot<<<gv, 256, 0, st>>>(n, 1, V, n, V, dh);
            k_arn_start<<<1, 1, 0, st>>>(Lo, dh);
            k_multiaxpy<<<gv, 256, 0, st>>>(n, 0, V, n, dh, V, 1.0, dscale);
            launches += 4;
            const int jm = std::min(m, maxit - it);
            for (int j = 0; j < jm; j++) {
                double *vj1 = V + (size_t)(j + 1) * n;
                precond(V + (size_t)j * n, Z + (size_t)j * n);
                spmv(Z + (size_t)j * n, vj1, nullptr);
                for (int pass = 0; pass < 2; pass++) {
                    k_multidot<<<gv, 256, 0, st>>>(n, j + 2, V, n, vj1, dh, pass ? need2 : nullptr);
                    k_arn_ctrl<<<1, 32, 0, st>>>(Lo, dh, j, pass);
                    k_multiaxpy<<<gv, 256, 0, st>>>(n, j + 1, V, n, dh + Lo.hvec(), vj1, 1.0, dscale,
                                                    pass ? need2 : nullptr);
                }
                launches += 7;
            }
            k_arn_solve<<<1, 256, 0, st>>>(Lo, dh, jm);
            k_multiaxpy<<<gv, 256, 0, st>>>(n, jm, Z, n, dh + Lo.yneg(), x, 1.0);
            launches += 2;
            it += jm;
        }
        spmv(x, w, b);
        launches++;
        const double res = norm2(w);
        s->last_launches = launches;
        if (iters_out) *iters_out = it;
        if (relres_out) *relres_out = res / (bnorm > 0.0 ? bnorm : 1.0);
        ce = cudaGetLastError();
        if (ce != cudaSuccess) { set_error(std::string("gmres: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
        return IGA_OK;
    }
    const double target = opt->rtol * (bnorm > 0.0 ? bnorm : 1.0);
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), hcol(m + 1), y(m);
    int it = 0;
    double res = 0.0;
    std::vector<double> hp(m + 2), ny(m);
    while (true) {
        // r = b - A x -> V[0]
        spmv(x, V, b);
        launches++;
        const double beta = norm2(V);
        res = beta;
        if (beta <= target || it >= maxit) break;
        k_axpby<<<gv, 256, 0, st>>>(n, 1.0 / beta, V, 0.0, V);
        launches++;
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int j = 0;
        for (; j < m && it < maxit; j++, it++) {
            double *vj1 = V + (size_t)(j + 1) * n;
            precond(V + (size_t)j * n, Z + (size_t)j * n);
            spmv(Z + (size_t)j * n, vj1, nullptr);            // w, in place of v_{j+1}
            launches++;
            // classical Gram-Schmidt with DGKS selective reorthogonalisation: one multi-dot gives
            // V_j^T w and w.w; ||w - V_j h||^2 = w.w - h.h when V_j is orthonormal; a second pass
            // only when that loses more than half of w.w (eta = 1/sqrt 2).  The final pass
            // normalises v_{j+1} in the same sweep.
            std::fill(hcol.begin(), hcol.end(), 0.0);
            double hj1 = 0.0;
            for (int pass = 0; pass < 2; pass++) {
                cudaMemsetAsync(dh, 0, sizeof(double) * (size_t)(j + 2), st);
                k_multidot<<<gv, 256, 0, st>>>(n, j + 2, V, n, vj1, dh);
                launches++;
                cudaMemcpyAsync(hp.data(), dh, sizeof(double) * (size_t)(j + 2), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                double hh = 0.0;
                for (int i = 0; i <= j; i++) { hh += hp[i] * hp[i]; hcol[i] += hp[i]; }
                const double ww = hp[j + 1], nrm2 = ww - hh;
                const bool last = pass == 1 || nrm2 > 0.5 * ww;
                double scale = 1.0;
                if (last) {
                    hj1 = nrm2 > 0.0 ? std::sqrt(nrm2) : 0.0;
                    if (hj1 > 0.0) scale = 1.0 / hj1;
                }
                k_multiaxpy<<<gv, 256, 0, st>>>(n, j + 1, V, n, dh, vj1, scale);
                launches++;
                if (last) break;
            }
            hcol[j + 1] = hj1;
            // Givens
            for (int i = 0; i < j; i++) {
                const double t = cs[i] * hcol[i] + sn[i] * hcol[i + 1];
                hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1];
                hcol[i] = t;
            }
            const double den = std::hypot(hcol[j], hcol[j + 1]);
            cs[j] = den > 0.0 ? hcol[j] / den : 1.0;
            sn[j] = den > 0.0 ? hcol[j + 1] / den : 0.0;
            hcol[j] = den;
            hcol[j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            for (int i = 0; i <= j; i++) H[(size_t)i * m + j] = hcol[i];
            res = std::fabs(g[j + 1]);
            if (res <= target || hj1 == 0.0) { j++; it++; break; }
        }
        // y = R^{-1} g, x += Z y (one multi-axpy with -y)
        for (int i = j - 1; i >= 0; i--) {
            double t = g[i];
            for (int k = i + 1; k < j; k++) t -= H[(size_t)i * m + k] * y[k];
            y[i] = t / H[(size_t)i * m + i];
        }
        for (int k = 0; k < j; k++) ny[k] = -y[k];
        if (j > 0) {
            cudaMemcpyAsync(dh, ny.data(), sizeof(double) * (size_t)j, cudaMemcpyHostToDevice, st);
            k_multiaxpy<<<gv, 256, 0, st>>>(n, j, Z, n, dh, x, 1.0);
            launches++;
        }
        if (res <= target || it >= maxit) {
            // true residual of the final iterate
            spmv(x, w, b);
            launches++;
            res = norm2(w);
            break;
        }
    }
    s->last_launches = launches;
    if (iters_out) *iters_out = it;
    if (relres_out) *relres_out = res / (bnorm > 0.0 ? bnorm : 1.0);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("gmres: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

// ---- generalized-alpha step (eq. (ga)) with the §5 fixed Newton budget ----------
// predictor: U1 = U, Ud1 = c Ud
__global__ void k_ga_predict(long long n, const double *__restrict__ U, const double *__restrict__ Ud, double c,
                             double *__restrict__ U1, double *__restrict__ Ud1) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        U1[i] = U[i];
        Ud1[i] = c * Ud[i];
    }
}

// stage values: Ua = U + af (U1 - U), Uda = Ud + am (Ud1 - Ud)
__global__ void k_ga_stage(long long n, const double *__restrict__ U, const double *__restrict__ Ud,
                           const double *__restrict__ U1, const double *__restrict__ Ud1, double af, double am,
                           double *__restrict__ Ua, double *__restrict__ Uda) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        Ua[i] = U[i] + af * (U1[i] - U[i]);
        Uda[i] = Ud[i] + am * (Ud1[i] - Ud[i]);
    }
}

// Newton update: Ud1 -= dx, U1 -= gdt dx
__global__ void k_ga_update(long long n, const double *__restrict__ dx, double gdt, double *__restrict__ U1,
                            double *__restrict__ Ud1) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        Ud1[i] -= dx[i];
        U1[i] -= gdt * dx[i];
    }
}

__global__ void k_sum_ranks(int nr, double *const *bufs, int cnt);

// all ranks of a decomposition (in-process: nr = nranks; NCCL: nr = 1, this process's rank; one
// rank: the plain step)
iga_status alpha_step_group(int nr, iga_space_s *const *sp, const iga_phys *phys, const iga_alpha *opt,
                            const int64_t *const *rp, const int32_t *const *ci, double *const *val, double *const *U,
                            double *const *Udot, iga_step_stats *stats, cudaStream_t st) {
    const double rho = opt->rho_inf, dt = opt->dt;
    const double am = 0.5 * (3.0 - rho) / (1.0 + rho), af = 1.0 / (1.0 + rho), gamma = 0.5 + am - af;
    const bool multi = sp[0]->nranks > 1;
    const bool local = !multi || dist_transport(sp[0]->dist) == IGA_XPORT_LOCAL;
    if (multi && opt->krylov.rtol != 0.0) { set_error("alpha_step: multi-rank steps use the fixed GMRES budget (rtol = 0)"); return IGA_ERR_PARAM; }
    std::vector<double *> U1(nr), Ud1(nr), Ua(nr), Uda(nr), R(nr), dx(nr), dn(nr);
    std::vector<long long> n(nr);
    for (int r = 0; r < nr; r++) {
        n[r] = sp[r]->nrows_owned;
        const size_t vb = ((sizeof(double) * (size_t)n[r] + 255) & ~(size_t)255);
        char *base = (char *)ws_ensure(sp[r], 2, 6 * vb + 256);
        if (!base) { set_error("alpha_step workspace"); return IGA_ERR_NOMEM; }
        U1[r] = (double *)base; Ud1[r] = (double *)(base + vb); Ua[r] = (double *)(base + 2 * vb);
        Uda[r] = (double *)(base + 3 * vb); R[r] = (double *)(base + 4 * vb); dx[r] = (double *)(base + 5 * vb);
        dn[r] = (double *)(base + 6 * vb);
    }
    double **dptrs = nullptr;
    if (local && nr > 1) {
        if (cudaMalloc(&dptrs, sizeof(double *) * nr) != cudaSuccess) { cudaGetLastError(); set_error("alpha_step ptrs"); return IGA_ERR_NOMEM; }
        cudaMemcpyAsync(dptrs, dn.data(), sizeof(double *) * nr, cudaMemcpyHostToDevice, st);
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, sp[0]->device);
    auto gv = [&](long long m_) { return (unsigned)std::max<long long>(1, std::min<long long>((m_ + 255) / 256, (long long)nsm * 8)); };
    int launches = 0;
    iga_status e = IGA_OK;
    if (stats) *stats = iga_step_stats{};
    for (int r = 0; r < nr; r++) k_ga_predict<<<gv(n[r]), 256, 0, st>>>(n[r], U[r], Udot[r], (gamma - 1.0) / gamma, U1[r], Ud1[r]);
    launches += nr;
    for (int k = 0; k < opt->newton_its && e == IGA_OK; k++) {
        for (int r = 0; r < nr; r++) k_ga_stage<<<gv(n[r]), 256, 0, st>>>(n[r], U[r], Udot[r], U1[r], Ud1[r], af, am, Ua[r], Uda[r]);
        launches += nr;
        if (!multi) e = form_one(sp[0], phys, am, af * gamma * dt, Ua[0], Uda[0], val[0], R[0], st);
        else {
            std::vector<const double *> ua(Ua.begin(), Ua.end()), uda(Uda.begin(), Uda.end());
            std::vector<iga_space_s *> spv(sp, sp + nr);
            e = dist_form(spv.data(), nr, phys, am, af * gamma * dt, ua.data(), uda.data(), val, R.data(), st);
        }
        if (e != IGA_OK) break;
        launches += sp[0]->last_launches;
        if (stats) {
            double r2 = 0.0;
            for (int r = 0; r < nr; r++) {
                cudaMemsetAsync(dn[r], 0, sizeof(double), st);
                k_multidot<<<gv(n[r]), 256, 0, st>>>(n[r], 1, R[r], n[r], R[r], dn[r]);
            }
            if (multi && local) k_sum_ranks<<<1, 64, 0, st>>>(nr, dptrs, 1);
            else if (multi && (e = dist_allreduce_sum(sp[0], dn[0], 1, st)) != IGA_OK) break;
            cudaMemcpyAsync(&r2, dn[0], sizeof(double), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            stats->res_norm[k] = std::sqrt(r2);
        }
        for (int r = 0; r < nr; r++) cudaMemsetAsync(dx[r], 0, sizeof(double) * (size_t)n[r], st);
        int its = 0;
        double rr = 0.0;
        if (!multi) e = gmres_solve(sp[0], rp[0], ci[0], val[0], R[0], dx[0], &opt->krylov, &its, &rr, st);
        else {
            std::vector<const double *> vv(val, val + nr), bb(R.begin(), R.end());
            e = gmres_group(nr, sp, rp, ci, vv.data(), bb.data(), dx.data(), &opt->krylov, &its, &rr, st);
        }
        if (e != IGA_OK) break;
        if (stats) {
            stats->gmres_its[k] = its;
            stats->gmres_relres[k] = rr;
        }
        for (int r = 0; r < nr; r++) k_ga_update<<<gv(n[r]), 256, 0, st>>>(n[r], dx[r], gamma * dt, U1[r], Ud1[r]);
        launches += nr;
    }
    if (e == IGA_OK)
        for (int r = 0; r < nr; r++) {
            cudaMemcpyAsync(U[r], U1[r], sizeof(double) * (size_t)n[r], cudaMemcpyDeviceToDevice, st);
            cudaMemcpyAsync(Udot[r], Ud1[r], sizeof(double) * (size_t)n[r], cudaMemcpyDeviceToDevice, st);
        }
    cudaStreamSynchronize(st);
    if (dptrs) cudaFree(dptrs);
    if (e != IGA_OK) return e;
    sp[0]->last_launches = launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("alpha_step: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

iga_status alpha_step(iga_space_s *s, const iga_phys *phys, const iga_alpha *opt, const int64_t *rp, const int32_t *ci,
                      double *val, double *U, double *Udot, iga_step_stats *stats, cudaStream_t st) {
    if (s->nranks > 1 && (!s->dist || dist_transport(s->dist) != IGA_XPORT_NCCL)) {
        set_error("alpha_step: in-process (IGA_XPORT_LOCAL) ranks step through iga_alpha_step_group");
        return IGA_ERR_STATE;
    }
    return alpha_step_group(1, &s, phys, opt, &rp, &ci, &val, &U, &Udot, stats, st);
}


// ============================================================================================
// Distributed GMRES over the box decomposition (SURVEY §8(e) x §8(f) rank 2): every rank holds
// its owned rows; the SpMV needs x on a ghost layer of width p around the owned box on the
// partitioned axes (the Alg. 3 stencil reaches p functions either way), exchanged per SpMV as
// box messages (one per neighbour offset in {-1,0,1}^d); the Gram-Schmidt dots are all-reduced
// (NCCL: ncclAllReduce on the stream; in-process ranks: a device sum over the ranks' buffers);
// block Jacobi ILU(0) runs on each rank's owned-owned block only -- the paper's "one block per
// process", cut into runs of block_rows rows as on one rank (reading A-28).  Fixed
// iteration budget only (rtol = 0, the §5 protocol): the Arnoldi control runs on the device.
// ============================================================================================
struct DPlan {
    int dim, m;
    int E[3], G[3], N[3], lo[3], nu[3], part[3];
};

__device__ __forceinline__ void dplan_coords(const DPlan &P, long long node, int g[3]) {
    long long r = node;
    for (int a = P.dim - 1; a >= 0; a--) { g[a] = (int)(r % P.nu[a]); r /= P.nu[a]; }
    for (int a = P.dim; a < 3; a++) g[a] = 0;
}

// column (global dof) -> ext-box index; *own = owned-box local index or -1
__device__ __forceinline__ long long dplan_ext(const DPlan &P, int col, long long *own) {
    const long long node = col / P.m;
    const int comp = col - (int)node * P.m;
    int g[3];
    dplan_coords(P, node, g);
    long long e = 0, o = 0;
    bool owned = true;
    for (int a = 0; a < 3; a++) {
        int l;
        if (a >= P.dim) l = 0;
        else if (P.part[a]) {
            int d = g[a] - P.lo[a];
            if (d < -P.G[a]) d += P.nu[a];
            else if (d >= P.N[a] + P.G[a]) d -= P.nu[a];
            l = d + P.G[a];
            owned = owned && d >= 0 && d < P.N[a];
            o = o * P.N[a] + d;
        } else {
            l = g[a];
            o = o * P.N[a] + g[a];
        }
        e = e * P.E[a] + l;
    }
    *own = owned ? o * P.m + comp : -1;
    return e * P.m + comp;
}

__global__ void k_dplan_lci(DPlan P, long long nnz, const int32_t *__restrict__ ci, int32_t *__restrict__ lci) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (long long)gridDim.x * blockDim.x) {
        long long own;
        lci[p] = (int32_t)dplan_ext(P, ci[p], &own);
    }
}

__global__ void k_dplan_own_count(DPlan P, long long n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                  int64_t *__restrict__ cnt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long c = 0;
    for (long long p = rp[i]; p < rp[i + 1]; p++) {
        long long own;
        dplan_ext(P, ci[p], &own);
        c += own >= 0;
    }
    cnt[i + 1] = c;
    if (i == 0) cnt[0] = 0;
}

__global__ void k_dplan_own_fill(DPlan P, long long n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                 const double *__restrict__ a, const int64_t *__restrict__ orp, int32_t *__restrict__ oci,
                                 double *__restrict__ oval) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long q = orp[i];
    for (long long p = rp[i]; p < rp[i + 1]; p++) {
        long long own;
        dplan_ext(P, ci[p], &own);
        if (own >= 0) { oci[q] = (int32_t)own; oval[q] = a[p]; q++; }
    }
}

// owned vector (owned-box C order, dof innermost) <-> ext box interior
__global__ void k_dplan_scatter(DPlan P, long long n, const double *__restrict__ x, double *__restrict__ xe) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        long long node = r / P.m;
        const int comp = (int)(r - node * P.m);
        int o[3] = {0, 0, 0};
        for (int a = P.dim - 1; a >= 0; a--) { o[a] = (int)(node % P.N[a]); node /= P.N[a]; }
        long long e = 0;
        for (int a = 0; a < 3; a++) e = e * P.E[a] + (a < P.dim ? o[a] + (P.part[a] ? P.G[a] : 0) : 0);
        xe[e * P.m + comp] = x[r];
    }
}

// box [lo, lo+bn) of the ext vector <-> contiguous buffer (node C order, dof innermost)
struct DBox { int lo[3], n[3]; };
__global__ void k_dplan_box(DPlan P, DBox B, double *__restrict__ xe, double *__restrict__ buf, int unpack) {
    const long long cnt = (long long)B.n[0] * B.n[1] * B.n[2] * P.m;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += (long long)gridDim.x * blockDim.x) {
        long long node = k / P.m;
        const int comp = (int)(k - node * P.m);
        const int b2 = (int)(node % B.n[2]);
        node /= B.n[2];
        const int b1 = (int)(node % B.n[1]);
        const int b0 = (int)(node / B.n[1]);
        const long long e = (((long long)(B.lo[0] + b0) * P.E[1] + (B.lo[1] + b1)) * P.E[2] + (B.lo[2] + b2)) * P.m + comp;
        if (unpack) xe[e] = buf[k];
        else buf[k] = xe[e];
    }
}

// in-process ranks: out[r][i] = sum_q in[q][i] for every rank r
__global__ void k_sum_ranks(int nr, double *const *bufs, int cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    double s = 0.0;
    for (int r = 0; r < nr; r++) s += bufs[r][i];
    for (int r = 0; r < nr; r++) bufs[r][i] = s;
}

struct DMsg {
    int peer, o[3];
    DBox box;
    long long off, cnt;
};

struct DRank {
    iga_space_s *s = nullptr;
    const int64_t *rp = nullptr;
    const int32_t *ci = nullptr;
    const double *a = nullptr, *b = nullptr;
    double *x = nullptr;
    long long n = 0, nnz = 0, next = 0, onnz = 0;
    DPlan P{};
    std::vector<DMsg> snd, rcv;
    long long sn = 0, rn = 0;
    int32_t *lci = nullptr, *oci = nullptr;
    int64_t *orp = nullptr, *dp = nullptr;
    double *oval = nullptr, *xe = nullptr, *sbuf = nullptr, *rbuf = nullptr, *V = nullptr, *Z = nullptr, *w = nullptr,
           *dh = nullptr, *lu = nullptr, *Lv = nullptr, *Uv = nullptr, *Dd = nullptr;
    uint8_t *Lc = nullptr, *Uc = nullptr;
    int W = 0;
    bool ell = false;
    size_t nalloc = 0;   // allocations of this solve; slot k of s->dr_cache backs the k-th one
    template <class T> T *alloc(size_t count) {
        const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
        auto &c = s->dr_cache;
        if (c.size() <= nalloc) c.resize(nalloc + 1, {nullptr, 0});
        auto &slot = c[nalloc++];
        if (slot.second < bytes) {
            if (slot.first) cudaFree(slot.first);
            slot = {nullptr, 0};
            void *p = nullptr;
            if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
            slot = {p, bytes};
        }
        return (T *)slot.first;
    }
};

// host-only: the ghost-exchange messages of the rank at coordinate rc (no GPU; also behind the
// GPU-free iga_krylov_plan).  Sends (ascending offset) carry this rank's owned slab on side o to
// the neighbour at rc + o; receives (descending offset) fill the ghost layer on side o.
static void dplan_messages(const DPlan &P, const int procs[3], const int rc[3], const int per[3],
                           std::vector<DMsg> &snd, std::vector<DMsg> &rcv, long long &sn, long long &rn) {
    std::vector<std::array<int, 3>> offs;
    for (int o0 = -1; o0 <= 1; o0++)
        for (int o1 = -1; o1 <= 1; o1++)
            for (int o2 = -1; o2 <= 1; o2++) {
                const int o[3] = {o0, o1, o2};
                bool ok = !(o0 == 0 && o1 == 0 && o2 == 0);
                for (int a = 0; a < 3 && ok; a++)
                    if (o[a] && !P.part[a]) ok = false;
                if (ok) offs.push_back({o0, o1, o2});
            }
    snd.clear();
    rcv.clear();
    sn = rn = 0;
    auto peer_of = [&](const int o[3], int &peer) {
        int c[3];
        for (int a = 0; a < 3; a++) {
            c[a] = rc[a] + o[a];
            if (c[a] < 0 || c[a] >= procs[a]) {
                if (!per[a]) return false;
                c[a] = (c[a] + procs[a]) % procs[a];
            }
        }
        peer = (c[0] * procs[1] + c[1]) * procs[2] + c[2];
        return true;
    };
    for (size_t k = 0; k < offs.size(); k++) {
        const int *o = offs[k].data();
        DMsg M{};
        if (!peer_of(o, M.peer)) continue;
        for (int a = 0; a < 3; a++) {
            M.o[a] = o[a];
            M.box.lo[a] = o[a] > 0 ? P.G[a] + P.N[a] - P.G[a] : P.G[a];
            M.box.n[a] = o[a] ? P.G[a] : P.N[a];
        }
        M.cnt = (long long)M.box.n[0] * M.box.n[1] * M.box.n[2] * P.m;
        M.off = sn;
        sn += M.cnt;
        snd.push_back(M);
    }
    for (size_t kk = offs.size(); kk-- > 0;) {
        const int *o = offs[kk].data();
        DMsg M{};
        if (!peer_of(o, M.peer)) continue;
        for (int a = 0; a < 3; a++) {
            M.o[a] = o[a];
            M.box.lo[a] = o[a] < 0 ? 0 : o[a] > 0 ? P.G[a] + P.N[a] : P.G[a];
            M.box.n[a] = o[a] ? P.G[a] : P.N[a];
        }
        M.cnt = (long long)M.box.n[0] * M.box.n[1] * M.box.n[2] * P.m;
        M.off = rn;
        rn += M.cnt;
        rcv.push_back(M);
    }
}

static void dplan_build(DRank &R) {
    iga_space_s *s = R.s;
    DPlan &P = R.P;
    P.dim = s->dim;
    P.m = s->dof;
    int per[3] = {0, 0, 0};
    for (int a = 0; a < 3; a++) {
        P.nu[a] = a < s->dim ? s->nu[a] : 1;
        P.part[a] = a < s->dim && s->procs[a] > 1;
        P.lo[a] = a < s->dim ? s->own_lo[a] : 0;
        P.N[a] = a < s->dim ? s->own_hi[a] - s->own_lo[a] : 1;
        P.G[a] = P.part[a] ? s->p[a] : 0;
        P.E[a] = P.part[a] ? P.N[a] + 2 * P.G[a] : P.N[a];
        per[a] = a < s->dim && s->periodic[a];
    }
    R.next = (long long)P.E[0] * P.E[1] * P.E[2] * P.m;
    dplan_messages(P, s->procs, s->rcoord, per, R.snd, R.rcv, R.sn, R.rn);
}

// GPU-free: the distributed-solve plan of one rank from the space description
iga_status krylov_plan_host(const iga_space_desc *d, const iga_dist *dist, int64_t own_lo[3], int64_t own_hi[3],
                            int64_t ext_n[3], int64_t ghost[3], int max_msgs, iga_msg *send, int *nsend, iga_msg *recv,
                            int *nrecv) {
    if (!d || !dist) { set_error("null argument"); return IGA_ERR_PARAM; }
    if (d->dim < 2 || d->dim > 3 || d->dof < 1 || d->dof > 4) { set_error("dim 2..3, dof 1..4"); return IGA_ERR_PARAM; }
    int procs[3] = {1, 1, 1}, rc[3] = {0, 0, 0}, per[3] = {0, 0, 0}, prod = 1;
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
    DPlan P{};
    P.dim = d->dim;
    P.m = d->dof;
    for (int a = 0; a < 3; a++) {
        if (a >= d->dim) { P.nu[a] = 1; P.N[a] = 1; P.E[a] = 1; continue; }
        AxisHost H;
        iga_status st = axis_host(d, a, procs[a], H);
        if (st != IGA_OK) return st;
        P.nu[a] = H.nu;
        P.part[a] = procs[a] > 1;
        P.lo[a] = H.own_lo[rc[a]];
        P.N[a] = H.own_hi[rc[a]] - H.own_lo[rc[a]];
        P.G[a] = P.part[a] ? H.p : 0;
        P.E[a] = P.part[a] ? P.N[a] + 2 * P.G[a] : P.N[a];
        per[a] = H.periodic;
        if (own_lo) own_lo[a] = H.own_lo[rc[a]];
        if (own_hi) own_hi[a] = H.own_hi[rc[a]];
    }
    for (int a = 0; a < 3; a++) {
        if (a >= d->dim) { if (own_lo) own_lo[a] = 0; if (own_hi) own_hi[a] = 1; }
        if (ext_n) ext_n[a] = P.E[a];
        if (ghost) ghost[a] = P.G[a];
    }
    std::vector<DMsg> snd, rcv;
    long long sn, rn;
    dplan_messages(P, procs, rc, per, snd, rcv, sn, rn);
    auto put = [&](const std::vector<DMsg> &L, iga_msg *out, int *cnt) {
        if (cnt) *cnt = (int)L.size();
        for (int k = 0; k < (int)L.size() && k < max_msgs && out; k++) {
            out[k].peer = L[k].peer;
            out[k].subbox = ((L[k].o[0] + 1) * 3 + (L[k].o[1] + 1)) * 3 + (L[k].o[2] + 1);
            out[k].rows = L[k].cnt;
            out[k].values = 0;
            for (int a = 0; a < 3; a++) { out[k].box_lo[a] = L[k].box.lo[a]; out[k].box_n[a] = L[k].box.n[a]; }
        }
    };
    put(snd, send, nsend);
    put(rcv, recv, nrecv);
    return IGA_OK;
}

iga_status gmres_group(int nr, iga_space_s *const *sp, const int64_t *const *rp, const int32_t *const *ci,
                       const double *const *a, const double *const *b, double *const *x, const iga_krylov *opt,
                       int *iters_out, double *relres_out, cudaStream_t st) {
    if (opt->rtol != 0.0) { set_error("distributed gmres: fixed iteration budget only (rtol = 0)"); return IGA_ERR_PARAM; }
    const int m = std::max(1, opt->restart), maxit = std::max(0, opt->maxit);
    if (m > 62) { set_error("distributed gmres: restart <= 62"); return IGA_ERR_PARAM; }
    const int B = opt->block_rows > 0 ? opt->block_rows : 32;
    const bool local = nr > 1 || sp[0]->nranks == 1 || dist_transport(sp[0]->dist) == IGA_XPORT_LOCAL;
    if (!local && nr != 1) { set_error("distributed gmres: one NCCL rank per process"); return IGA_ERR_PARAM; }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, sp[0]->device);
    std::vector<DRank> R(nr);
    const ArnLayout Lo{m};
    // ---- setup ----
    for (int r = 0; r < nr; r++) {
        DRank &D = R[r];
        D.s = sp[r];
        D.rp = rp[r]; D.ci = ci[r]; D.a = a[r]; D.b = b[r]; D.x = x[r];
        D.n = D.s->nrows_owned;
        D.nnz = D.s->nnz_owned;
        dplan_build(D);
        D.lci = D.alloc<int32_t>(D.nnz);
        D.orp = D.alloc<int64_t>(D.n + 1);
        D.dp = D.alloc<int64_t>(D.n);
        D.xe = D.alloc<double>(D.next);
        D.sbuf = D.alloc<double>(D.sn);
        D.rbuf = D.alloc<double>(D.rn);
        D.V = D.alloc<double>((size_t)(m + 1) * D.n);
        D.Z = D.alloc<double>((size_t)m * D.n);
        D.w = D.alloc<double>(D.n);
        D.dh = D.alloc<double>(Lo.total());
        if (!D.lci || !D.orp || !D.dp || !D.xe || !D.sbuf || !D.rbuf || !D.V || !D.Z || !D.w || !D.dh) {
            set_error("distributed gmres workspace");
            return IGA_ERR_NOMEM;
        }
        const unsigned gn = (unsigned)std::max<long long>(1, (D.n + 255) / 256);
        k_dplan_lci<<<(unsigned)std::min<long long>((D.nnz + 255) / 256, (long long)nsm * 16), 256, 0, st>>>(D.P, D.nnz, D.ci, D.lci);
        k_dplan_own_count<<<gn, 256, 0, st>>>(D.P, D.n, D.rp, D.ci, D.orp);
        size_t tmp = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tmp, D.orp, D.orp, (int)(D.n + 1), st);
        void *tbuf = D.alloc<char>(tmp);
        cub::DeviceScan::InclusiveSum(tbuf, tmp, D.orp, D.orp, (int)(D.n + 1), st);
        cudaMemcpyAsync(&D.onnz, D.orp + D.n, sizeof(long long), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        D.oci = D.alloc<int32_t>(D.onnz);
        D.oval = D.alloc<double>(D.onnz);
        if (!D.oci || !D.oval) { set_error("distributed gmres workspace"); return IGA_ERR_NOMEM; }
        k_dplan_own_fill<<<gn, 256, 0, st>>>(D.P, D.n, D.rp, D.ci, D.a, D.orp, D.oci, D.oval);
        k_diagpos<<<gn, 256, 0, st>>>(D.n, D.orp, D.oci, D.dp);
        // block-Jacobi ILU(0) of the owned-owned block (as gmres_solve)
        const long long nblk = (D.n + B - 1) / B;
        if (opt->precond == 2) {
            int wm[2] = {0, 0};
            cudaMemsetAsync(D.dh, 0, 2 * sizeof(int), st);
            k_ell_count<<<gn, 256, 0, st>>>(D.n, B, D.orp, D.oci, D.dp, (int *)D.dh);
            cudaMemcpyAsync(wm, D.dh, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            const int wmax = std::max(wm[0], wm[1]);
            if (B <= TPB_MAXB && wmax <= TPB_MAXW) {
                D.W = wmax <= 2 ? 2 : wmax <= 4 ? 4 : wmax <= 8 ? 8 : 16;
                const size_t rows = (size_t)nblk * B;
                D.Lv = D.alloc<double>(rows * D.W); D.Uv = D.alloc<double>(rows * D.W); D.Dd = D.alloc<double>(rows);
                D.Lc = D.alloc<uint8_t>(rows * D.W); D.Uc = D.alloc<uint8_t>(rows * D.W);
                if (!D.Lv || !D.Uv || !D.Dd || !D.Lc || !D.Uc) { set_error("distributed gmres workspace"); return IGA_ERR_NOMEM; }
                k_ell_pack<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(D.n, B, nblk, D.orp, D.oci, D.dp, D.oval, D.W, D.W,
                                                                            D.Lv, D.Lc, D.Uv, D.Uc, D.Dd);
                k_ell_ilu0<<<(unsigned)((nblk + 63) / 64), 64, 0, st>>>(nblk, B, D.W, D.W, D.Lv, D.Lc, D.Uv, D.Uc, D.Dd);
                D.ell = true;
            } else {
                D.lu = D.alloc<double>(D.onnz);
                if (!D.lu) { set_error("distributed gmres workspace"); return IGA_ERR_NOMEM; }
                cudaMemcpyAsync(D.lu, D.oval, sizeof(double) * (size_t)D.onnz, cudaMemcpyDeviceToDevice, st);
                k_ilu0<<<(unsigned)(((nblk * 32) + 127) / 128), 128, 0, st>>>(D.n, B, D.orp, D.oci, D.dp, D.lu);
            }
        }
        cudaMemsetAsync(D.xe, 0, sizeof(double) * (size_t)D.next, st);
    }
    // pointer table for the in-process all-reduce
    std::vector<double *> hptrs(nr);
    for (int r = 0; r < nr; r++) hptrs[r] = R[r].dh;
    double **dptrs = R[0].alloc<double *>(nr);
    if (!dptrs) { set_error("gmres ptrs"); return IGA_ERR_NOMEM; }
    cudaMemcpyAsync(dptrs, hptrs.data(), sizeof(double *) * nr, cudaMemcpyHostToDevice, st);
    auto allreduce = [&](int cnt) -> iga_status {
        if (local) {
            if (nr > 1) k_sum_ranks<<<(cnt + 63) / 64, 64, 0, st>>>(nr, dptrs, cnt);
            return IGA_OK;
        }
        return dist_allreduce_sum(R[0].s, R[0].dh, (size_t)cnt, st);
    };
    // ghost exchange of the ext vectors (after the owned interiors are current)
    auto exchange = [&]() -> iga_status {
        for (int r = 0; r < nr; r++)
            for (const DMsg &M : R[r].snd)
                k_dplan_box<<<(unsigned)std::max<long long>(1, std::min<long long>((M.cnt + 255) / 256, (long long)nsm * 4)), 256, 0, st>>>(
                    R[r].P, M.box, R[r].xe, R[r].sbuf + M.off, 0);
        if (local) {
            // rank r's receive for offset o from peer q = the send of q for offset -o to r
            std::vector<std::vector<int>> used(nr);
            for (int r = 0; r < nr; r++) used[r].assign(R[r].snd.size(), 0);
            for (int r = 0; r < nr; r++)
                for (const DMsg &M : R[r].rcv) {
                    const DRank &Q = R[M.peer];
                    int found = -1;
                    for (size_t k = 0; k < Q.snd.size(); k++) {
                        const DMsg &S = Q.snd[k];
                        if (S.peer == r && S.o[0] == -M.o[0] && S.o[1] == -M.o[1] && S.o[2] == -M.o[2]) { found = (int)k; break; }
                    }
                    if (found < 0 || Q.snd[found].cnt != M.cnt) { set_error("distributed gmres: inconsistent ghost plan"); return IGA_ERR_STATE; }
                    cudaMemcpyAsync(R[r].rbuf + M.off, Q.sbuf + Q.snd[found].off, sizeof(double) * (size_t)M.cnt,
                                    cudaMemcpyDeviceToDevice, st);
                }
        } else {
            DRank &D = R[0];
            std::vector<int> sp_(D.snd.size()), rp_(D.rcv.size());
            std::vector<const double *> sb(D.snd.size());
            std::vector<double *> rb(D.rcv.size());
            std::vector<long long> sc(D.snd.size()), rc(D.rcv.size());
            for (size_t k = 0; k < D.snd.size(); k++) { sp_[k] = D.snd[k].peer; sb[k] = D.sbuf + D.snd[k].off; sc[k] = D.snd[k].cnt; }
            for (size_t k = 0; k < D.rcv.size(); k++) { rp_[k] = D.rcv[k].peer; rb[k] = D.rbuf + D.rcv[k].off; rc[k] = D.rcv[k].cnt; }
            iga_status e = dist_sendrecv(D.s, (int)sp_.size(), sp_.data(), sb.data(), sc.data(), (int)rp_.size(), rp_.data(),
                                         rb.data(), rc.data(), st);
            if (e != IGA_OK) return e;
        }
        for (int r = 0; r < nr; r++)
            for (const DMsg &M : R[r].rcv)
                k_dplan_box<<<(unsigned)std::max<long long>(1, std::min<long long>((M.cnt + 255) / 256, (long long)nsm * 4)), 256, 0, st>>>(
                    R[r].P, M.box, R[r].xe, R[r].rbuf + M.off, 1);
        return IGA_OK;
    };
    // y_r = (bsub_r -) A_r x_r for every rank
    auto spmv_all = [&](const std::vector<const double *> &xs, const std::vector<double *> &ys,
                        const std::vector<const double *> &bs) -> iga_status {
        for (int r = 0; r < nr; r++)
            k_dplan_scatter<<<(unsigned)std::max<long long>(1, std::min<long long>((R[r].n + 255) / 256, (long long)nsm * 8)), 256, 0, st>>>(
                R[r].P, R[r].n, xs[r], R[r].xe);
        iga_status e = exchange();
        if (e != IGA_OK) return e;
        for (int r = 0; r < nr; r++)
            k_spmv_stream<<<(unsigned)std::max<long long>(1, (R[r].n + SP_R - 1) / SP_R), SP_R, 0, st>>>(
                R[r].n, R[r].rp, R[r].lci, R[r].a, R[r].xe, ys[r], bs[r]);
        return IGA_OK;
    };
    auto gv_of = [&](long long n) { return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)nsm * 8)); };
    auto precond = [&](int r, const double *in, double *out) {
        DRank &D = R[r];
        const long long nblk = (D.n + B - 1) / B;
        const unsigned gell = (unsigned)((nblk + TPB_CTA - 1) / TPB_CTA);
        const size_t smell = sizeof(double) * (size_t)TPB_CTA * (B + 1);
        const unsigned gblk = (unsigned)(((nblk * 32) + 127) / 128);
        if (opt->precond == 2 && D.ell) {
            if (D.W == 2) k_ell_solve<2><<<gell, TPB_CTA, smell, st>>>(D.n, B, nblk, D.Lv, D.Lc, D.Uv, D.Uc, D.Dd, in, out);
            else if (D.W == 4) k_ell_solve<4><<<gell, TPB_CTA, smell, st>>>(D.n, B, nblk, D.Lv, D.Lc, D.Uv, D.Uc, D.Dd, in, out);
            else if (D.W == 8) k_ell_solve<8><<<gell, TPB_CTA, smell, st>>>(D.n, B, nblk, D.Lv, D.Lc, D.Uv, D.Uc, D.Dd, in, out);
            else k_ell_solve<16><<<gell, TPB_CTA, smell, st>>>(D.n, B, nblk, D.Lv, D.Lc, D.Uv, D.Uc, D.Dd, in, out);
        } else if (opt->precond == 2 && B <= 1024) {
            k_ilu0_solve_g<<<gblk, 128, 4 * B * sizeof(double), st>>>(D.n, B, D.orp, D.oci, D.dp, D.lu, in, out);
        } else if (opt->precond == 2) {
            k_ilu0_solve<<<gblk, 128, 0, st>>>(D.n, B, D.orp, D.oci, D.dp, D.lu, in, out);
        } else if (opt->precond == 1) {
            k_jacobi<<<gv_of(D.n), 256, 0, st>>>(D.n, D.dp, D.oval, in, out);
        } else {
            cudaMemcpyAsync(out, in, sizeof(double) * (size_t)D.n, cudaMemcpyDeviceToDevice, st);
        }
    };
    auto norm2_all = [&](const std::vector<const double *> &vs) -> double {
        for (int r = 0; r < nr; r++) {
            cudaMemsetAsync(R[r].dh, 0, sizeof(double), st);
            k_multidot<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, 1, vs[r], R[r].n, vs[r], R[r].dh);
        }
        allreduce(1);
        double h = 0.0;
        cudaMemcpyAsync(&h, R[0].dh, sizeof(double), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        return std::sqrt(h);
    };
    std::vector<const double *> bvec(nr), xvec(nr), wvec(nr), V0c(nr);
    std::vector<double *> V0(nr), wv(nr);
    for (int r = 0; r < nr; r++) { bvec[r] = R[r].b; xvec[r] = R[r].x; V0[r] = R[r].V; V0c[r] = R[r].V; wv[r] = R[r].w; wvec[r] = R[r].w; }
    const double bnorm = norm2_all(bvec);
    for (int r = 0; r < nr; r++) cudaMemsetAsync(R[r].dh, 0, sizeof(double) * Lo.total(), st);
    int it = 0;
    iga_status e = IGA_OK;
    while (it < maxit && bnorm > 0.0) {
        if ((e = spmv_all(xvec, V0, bvec)) != IGA_OK) return e;
        for (int r = 0; r < nr; r++) k_multidot<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, 1, R[r].V, R[r].n, R[r].V, R[r].dh);
        if ((e = allreduce(1)) != IGA_OK) return e;
        for (int r = 0; r < nr; r++) {
            k_arn_start<<<1, 1, 0, st>>>(Lo, R[r].dh);
            k_multiaxpy<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, 0, R[r].V, R[r].n, R[r].dh, R[r].V, 1.0, R[r].dh + Lo.ctl());
        }
        const int jm = std::min(m, maxit - it);
        for (int j = 0; j < jm; j++) {
            std::vector<const double *> zj(nr);
            std::vector<double *> vj1(nr);
            for (int r = 0; r < nr; r++) {
                precond(r, R[r].V + (size_t)j * R[r].n, R[r].Z + (size_t)j * R[r].n);
                zj[r] = R[r].Z + (size_t)j * R[r].n;
                vj1[r] = R[r].V + (size_t)(j + 1) * R[r].n;
            }
            std::vector<const double *> nob(nr, nullptr);
            if ((e = spmv_all(zj, vj1, nob)) != IGA_OK) return e;
            for (int pass = 0; pass < 2; pass++) {
                for (int r = 0; r < nr; r++) {
                    int *need2 = &reinterpret_cast<ArnCtl *>(R[r].dh + Lo.ctl())->need2;
                    k_multidot<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, j + 2, R[r].V, R[r].n, vj1[r], R[r].dh, pass ? need2 : nullptr);
                }
                if ((e = allreduce(j + 2)) != IGA_OK) return e;
                for (int r = 0; r < nr; r++) {
                    int *need2 = &reinterpret_cast<ArnCtl *>(R[r].dh + Lo.ctl())->need2;
                    k_arn_ctrl<<<1, 32, 0, st>>>(Lo, R[r].dh, j, pass);
                    k_multiaxpy<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, j + 1, R[r].V, R[r].n, R[r].dh + Lo.hvec(), vj1[r], 1.0,
                                                                R[r].dh + Lo.ctl(), pass ? need2 : nullptr);
                }
            }
        }
        for (int r = 0; r < nr; r++) {
            k_arn_solve<<<1, 256, 0, st>>>(Lo, R[r].dh, jm);
            k_multiaxpy<<<gv_of(R[r].n), 256, 0, st>>>(R[r].n, jm, R[r].Z, R[r].n, R[r].dh + Lo.yneg(), R[r].x, 1.0);
        }
        it += jm;
    }
    if ((e = spmv_all(xvec, wv, bvec)) != IGA_OK) return e;
    const double res = norm2_all(wvec);
    if (iters_out) *iters_out = it;
    if (relres_out) *relres_out = res / (bnorm > 0.0 ? bnorm : 1.0);
    cudaStreamSynchronize(st);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("distributed gmres: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

}  // namespace iga
