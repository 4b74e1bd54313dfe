// microbench.cu -- K8: measured ceilings that set the roofline denominators and the design
// choices of DESIGN.md (FP64 DFMA vs DMMA peak, L2 fp64 reduction throughput, store bandwidth).
// Exposed as iga_microbench(); used by bench.py (peak_measured) and tests/test_microbench.py.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/iga.h"

namespace {

constexpr int ITERS = 2048;

__global__ void k_dfma(double *out, double seed) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double m = 1.0000001, c = 1e-9;
#pragma unroll 16
    for (int i = 0; i < ITERS; i++) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;
}

// D(8x8) += A(8x4) B(4x8), fp64 tensor-core path (mma.sync, the only FP64 MMA on sm_100a)
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, double seed) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
    const double a = seed + threadIdx.x * 1e-3, b = 1e-3;
#pragma unroll 4
    for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

// even warps DFMA, odd warps DMMA: do the two FP64 paths add up?
__global__ void k_mixed(double *out, double seed) {
    const int w = threadIdx.x >> 5;
    if (w & 1) {
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
        const double a = seed + threadIdx.x * 1e-3, b = 1e-3;
#pragma unroll 4
        for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
            for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], a, b);
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
        if (s == 12345.678) out[0] = s;
    } else {
        double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
               a6 = a0 + 6, a7 = a0 + 7;
        const double m = 1.0000001, cc = 1e-9;
#pragma unroll 16
        for (int i = 0; i < ITERS; i++) {
            a0 = fma(a0, m, cc); a1 = fma(a1, m, cc); a2 = fma(a2, m, cc); a3 = fma(a3, m, cc);
            a4 = fma(a4, m, cc); a5 = fma(a5, m, cc); a6 = fma(a6, m, cc); a7 = fma(a7, m, cc);
        }
        const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
        if (s == 12345.678) out[0] = s;
    }
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

// each warp: `reps` x (32 lanes add to `group`-consecutive doubles at random aligned spots)
__global__ void k_red(double *arr, long long n, int group, int reps) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nslots = n / group;
    for (int r = 0; r < reps; r++) {
        const uint32_t h = hash32((uint32_t)(warp * 977 + r * 131 + (lane / group) * 7919));
        const long long slot = h % nslots;
        atomicAdd(arr + slot * group + (lane % group), 1.0);
    }
}

// config-5-like lane pattern: 27 lanes = 9 runs of 3 entries with stride 4 doubles
__global__ void k_red_c5(double *arr, long long n, int reps) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane >= 27) return;
    const int run = lane / 3, k = lane % 3;
    for (int r = 0; r < reps; r++) {
        const uint32_t h = hash32((uint32_t)(warp * 977 + r * 131));
        const long long base = (long long)(h % (uint32_t)((n - 4096) / 32)) * 32;
        atomicAdd(arr + base + run * 500 / 8 * 8 + k * 4, 1.0);
    }
}

// TMA bulk reductions (cp.reduce.async.bulk .add.f64) of `seg`-byte segments from smem
__global__ void k_bulkred(double *arr, long long n, int seg, int reps) {
    __shared__ __align__(128) double sm[32 * 16];
    for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) sm[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm + (threadIdx.x >> 5) * 16);
    const long long nseg = n / 4 - 64;
    if (lane == 0) {
        for (int r = 0; r < reps; r++) {
            const uint32_t h = hash32((uint32_t)(warp * 977 + r * 131));
            double *dst = arr + (long long)(h % (uint32_t)nseg) * 4;
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                         :: "l"(dst), "r"(sa), "r"(seg) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void k_store(double2 *arr, long long n2) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
        arr[i] = make_double2(1.0, 2.0);
}

__global__ void k_smem_atomic(double *out, int reps) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0.0;
    __syncthreads();
    for (int r = 0; r < reps; r++) atomicAdd(&buf[(threadIdx.x * 33 + r * 97) & 4095], 1.0);
    __syncthreads();
    if (threadIdx.x == 0 && buf[0] == -1.0) out[0] = buf[1];
}

// Broadcast 128-bit loads, the 3D contraction's coefficient pattern: lanes (B, J) = (lane / 4,
// lane % 4) read block J's double2 (4 distinct conflict-free 16-byte addresses per warp
// instruction), 10 loads feeding 20 independent DFMAs per iteration.  V = 0: shared memory,
// 1: global (L1-resident).  Shows that a warp-uniform 128-bit load costs 4 data-pipe wavefronts
// from either memory.
template <int V>
__global__ void __launch_bounds__(128, 4) k_bcast(const double2 *g, double *out, int iters) {
    __shared__ double2 sm[4 * 42 * 12];
    const int tid = threadIdx.x, J = tid & 3;
    const double2 *gb = g + (size_t)blockIdx.x * 4 * 42 * 12;
    for (int i = tid; i < 4 * 42 * 12; i += blockDim.x) sm[i] = gb[i];
    __syncthreads();
    double acc[20];
#pragma unroll
    for (int i = 0; i < 20; i++) acc[i] = 0.0;
    const double pb[5] = {1.0 + tid, 2.0, 3.0, 4.0, 5.0};
    for (int it = 0; it < iters; it++) {
        const int base = ((it % 12) * 4 + J) * 42;   // 42 double2 per block: J offsets in distinct banks
#pragma unroll
        for (int x = 0; x < 10; x++) {
            const double2 v = V == 0 ? sm[base + x] : gb[base + x];
            acc[2 * x] += v.x * pb[(2 * x) % 5];
            acc[2 * x + 1] += v.y * pb[(2 * x + 1) % 5];
        }
    }
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 20; i++) t += acc[i];
    out[blockIdx.x * blockDim.x + tid] = t;
}

}  // namespace

extern "C" double iga_microbench(int device, int which, long long param) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    double *buf = nullptr;
    const long long n = param > 0 ? param : (26LL << 20) / 8;   // default 26 MB (config-2 CSR size)
    if (cudaMalloc(&buf, (size_t)n * sizeof(double) + 256) != cudaSuccess) { cudaSetDevice(prev); return -1.0; }
    cudaMemset(buf, 0, (size_t)n * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double work = 0.0;
    float ms = 0.f;
    const int blocks = nsm * 8, thr = 256;
    for (int pass = 0; pass < 2; pass++) {   // pass 0 warms up
        cudaEventRecord(a);
        switch (which) {
        case 0:   // DFMA flop/s
            k_dfma<<<blocks, thr>>>(buf, 1.0);
            work = 2.0 * 8 * ITERS * (double)blocks * thr;
            break;
        case 1:   // DMMA flop/s (m8n8k4: 2*256 flop per warp instruction)
            k_dmma<<<blocks, thr>>>(buf, 1.0);
            work = 2.0 * 256 * 8 * (ITERS / 4) * (double)blocks * (thr / 32);
            break;
        case 2:   // mixed: total flop/s
            k_mixed<<<blocks, thr>>>(buf, 1.0);
            work = (2.0 * 8 * ITERS * (thr / 2) + 2.0 * 256 * 8 * (ITERS / 4) * (thr / 64)) * (double)blocks;
            break;
        case 3: case 4: case 5: {   // fp64 red.add: lanes per contiguous group = 32 / 4 / 1
            const int group = which == 3 ? 32 : (which == 4 ? 4 : 1);
            const int reps = 64;
            k_red<<<blocks * 4, thr>>>(buf, n, group, reps);
            work = (double)blocks * 4 * thr * reps;      // atomic adds
            break;
        }
        case 6:   // store bandwidth, bytes/s
            k_store<<<blocks, thr>>>((double2 *)buf, n / 2);
            work = 16.0 * (n / 2);
            break;
        case 7:   // shared-memory fp64 atomics / s
            k_smem_atomic<<<blocks, thr>>>(buf, 256);
            work = (double)blocks * thr * 256;
            break;
        case 8:   // bulk reductions of 96 B per op: ops/s (x12 = fp64 adds/s)
            k_bulkred<<<blocks, thr>>>(buf, n, 96, 64);
            work = (double)blocks * (thr / 32) * 64;
            break;
        case 9:   // config-5 lane pattern red.add: adds/s
            k_red_c5<<<blocks * 4, thr>>>(buf, n, 64);
            work = (double)blocks * 4 * (thr / 32) * 27 * 64;
            break;
        case 11: case 12: {   // broadcast 128-bit loads (shared / L1-resident global): warp-loads/s
            const int grid = nsm * 4, iters = 1 << 14;
            const size_t need = (size_t)grid * 4 * 42 * 12 * 2;   // doubles
            if ((size_t)n < need) { work = 0.0; break; }
            if (which == 11) k_bcast<0><<<grid, 128>>>((const double2 *)buf, buf + need, iters);
            else k_bcast<1><<<grid, 128>>>((const double2 *)buf, buf + need, iters);
            work = (double)grid * 4 * iters * 10;
            break;
        }
        case 10:  // bulk reductions of 384 B per op
            k_bulkred<<<blocks, thr>>>(buf, n, 384, 64);
            work = (double)blocks * (thr / 32) * 64;
            break;
        default:
            work = 0.0;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaSetDevice(prev);
    if (e != cudaSuccess || ms <= 0.f) return -1.0;
    return work / (ms * 1e-3);
}
