// kernels.cu -- hand-written sm_100a FP64 kernels of one Newton-Raphson iteration.
//
// Layout: a *task tile* is 32 scenarios = the 32 lanes of a
// warp.  Per-bus tapes are element-major [bus][bpad] (lane-contiguous, 256 B
// per warp access); the A / LU / b tapes are tile-major [tile][slot][32], so a
// CTA owning one tile streams a contiguous region.  Scenarios are independent,
// so every kernel is one CTA per tile and no grid-wide synchronization exists.
//
//   npm_kernel       compute_npm + convergence (Alg. 1)
//   jacobian_kernel  update_jacobian into the A tape via the static lookup
//                    (signs per SURVEY App. B)
//   lu_kernel        refactorize_batch / execute_schedule (
//                    Alg. 2/3): columns in level order, warps of the CTA take
//                    columns round-robin and wait on per-warp progress counters
//                    (dependency-driven, so later columns start early -- Alg. 3
//                    stage 2 -- without grid or level barriers)
//   fsbs_kernel      fs_bs_batch: pull-style rows, same
//                    progress-counter scheduling, no atomics
//   vupdate_kernel   update_voltage + unit phasor refresh
#include "../../include/gbnr.h"
#include "kernels.hpp"
#include "numerics.cuh"

namespace gbnr {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double nan_as_inf_abs(double v) {
    double a = fabs(v);
    return isnan(a) ? INFINITY : a;
}

// Per-warp progress counters: prog[w] = number of schedule entries warp w has
// finished.  Entry at schedule position p belongs to warp p % NW, rank p / NW.
template <int NW>
__device__ __forceinline__ void wait_done(const int* prog, int pos) {
    const int ow = pos % NW, rk = pos / NW;
    const volatile int* f = prog + ow;
    if (*f <= rk) {
        while (*f <= rk) {
        }
    }
    __threadfence_block();  // acquire: order the data loads after the flag
}

__device__ __forceinline__ void signal_done(int* prog, int warp, int value, int lane) {
    __threadfence_block();  // release: every lane's stores before the flag
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile int*>(prog + warp) = value;
}

// ---------------------------------------------------------------------------
// init: unit phasors, task state, tile activity
// ---------------------------------------------------------------------------
__global__ void init_kernel(DevView v) {
    const int tile = blockIdx.x, lane = threadIdx.x & 31;
    const int t = tile * kTile + lane;
    const bool real = t < v.n_tasks;
    for (int bus = threadIdx.x >> 5; bus < v.n; bus += blockDim.x >> 5) {
        const size_t o = size_t(bus) * v.bpad + t;
        const double vm = real ? v.vm_in[o] : 1.0, va = real ? v.va_in[o] : 0.0;
        v.vm[o] = vm;
        v.va[o] = va;
        double s, c;
        gb_sincos(va, &s, &c);
        v.s[o] = s;
        v.c[o] = c;
    }
    if (threadIdx.x < 32) {
        v.status[t] = real ? GBNR_DIVERGED : -1;
        v.iters[t] = 0;
        v.active[t] = real ? 1 : 0;
        v.flag[t] = 0;
        v.maxmis[t] = real ? INFINITY : 0.0;
        const int cnt = __popc(__ballot_sync(kFull, real));
        if (lane == 0) v.tile_active[tile] = cnt;
    }
}

// ---------------------------------------------------------------------------
// NPM + convergence.  Warp w of the tile's CTA sweeps Ybus rows w, w+NW, ...
// (row-level parallelism); lane = task.
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32, 3) npm_kernel(DevView v, int it) {
    __shared__ double red[NW][32];
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (v.tile_active[tile] == 0) return;
    const int t = tile * kTile + lane;
    const size_t bp = v.bpad;
    double* bt = v.b + size_t(tile) * v.nJ * kTile + lane;
    double nrm = 0.0;
    for (int ri = warp; ri < v.n_rows; ri += NW) {
        const int r = v.rows[ri];
        double ire = 0.0, iim = 0.0;
        const int q1 = v.yp[r + 1];
        for (int q = v.yp[r]; q < q1; ++q) {
            const int k = v.yi[q];
            const double vmk = v.vm[k * bp + t];
            acc_current(v.yre[q], v.yim[q], vmk * v.c[k * bp + t], vmk * v.s[k * bp + t], ire, iim);
        }
        const double vmr = v.vm[r * bp + t];
        const double vre = vmr * v.c[r * bp + t], vim = vmr * v.s[r * bp + t];
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        const double fp = P - v.p0[size_t(r) * v.s_ld + size_t(t) * v.s_inc];
        bt[size_t(v.brow_p[r]) * kTile] = fp;
        nrm = fmax(nrm, nan_as_inf_abs(fp));
        const int bq = v.brow_q[r];
        if (bq >= 0) {
            const double fq = Q - v.q0[size_t(r) * v.s_ld + size_t(t) * v.s_inc];
            bt[size_t(bq) * kTile] = fq;
            nrm = fmax(nrm, nan_as_inf_abs(fq));
        }
    }
    red[warp][lane] = nrm;
    __syncthreads();
    if (warp == 0) {
        double m = red[0][lane];
#pragma unroll
        for (int w = 1; w < NW; ++w) m = fmax(m, red[w][lane]);
        bool act = v.active[t] != 0;
        if (act) {
            v.maxmis[t] = m;
            if (m < v.tol) {
                v.status[t] = GBNR_CONVERGED;
                v.iters[t] = it;
                v.active[t] = 0;
                act = false;
            } else if (it >= v.max_iter) {
                v.status[t] = GBNR_DIVERGED;
                v.iters[t] = v.max_iter;
                v.active[t] = 0;
                act = false;
            }
        }
        const int cnt = __popc(__ballot_sync(kFull, act));
        if (lane == 0) {
            v.tile_active[tile] = cnt;
            if (cnt) {
                atomicAdd(v.active_count + it, cnt);       // active tasks after iteration it
                atomicAdd(v.active_count + 32 + it, 1);    // tiles with work left
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Jacobian -> A tape (J nonzeros in LU slot order; fill slots are implicit).
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32, 3) jacobian_kernel(DevView v) {
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (v.tile_active[tile] == 0) return;
    const int t = tile * kTile + lane;
    const bool act = v.active[t] != 0;
    const size_t bp = v.bpad;
    double* at = v.A + size_t(tile) * v.nA * kTile + lane;
    for (int ri = warp; ri < v.n_rows; ri += NW) {
        const int r = v.rows[ri];
        const int q0 = v.yp[r], q1 = v.yp[r + 1];
        double ire = 0.0, iim = 0.0;
        for (int q = q0; q < q1; ++q) {
            const int k = v.yi[q];
            const double vmk = v.vm[k * bp + t];
            acc_current(v.yre[q], v.yim[q], vmk * v.c[k * bp + t], vmk * v.s[k * bp + t], ire, iim);
        }
        const double vmr = v.vm[r * bp + t];
        const double vre = vmr * v.c[r * bp + t], vim = vmr * v.s[r * bp + t];
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        for (int q = q0; q < q1; ++q) {
            const int k = v.yi[q];
            const double ck = v.c[k * bp + t], sk = v.s[k * bp + t], vmk = v.vm[k * bp + t];
            double zre, zim, j[4];
            jac_z(v.yre[q], v.yim[q], vre, vim, ck, sk, zre, zim);
            jac_entries(k == r, zre, zim, vmk, ck, sk, ire, iim, P, Q, j);
            const int4 l = *reinterpret_cast<const int4*>(v.lk + 4 * size_t(q));
            if (act) {
                if (l.x >= 0) at[size_t(l.x) * kTile] = j[0];
                if (l.y >= 0) at[size_t(l.y) * kTile] = j[1];
                if (l.z >= 0) at[size_t(l.z) * kTile] = j[2];
                if (l.w >= 0) at[size_t(l.w) * kTile] = j[3];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Batched LU refactorization (Alg. 2 operation order per column; Alg. 3-style
// dependency-driven column parallelism inside the tile's CTA).
// ---------------------------------------------------------------------------
// Wait until every schedule position in `pos` (one per lane, -1 = none) is
// done; the 32 checks run in parallel across the warp.
template <int NW>
__device__ __forceinline__ void wait_all(const int* prog, int pos) {
    const volatile int* pv = prog;
    bool ok = pos < 0 || pv[pos % NW] > pos / NW;
    while (!__all_sync(kFull, ok)) ok = pos < 0 || pv[pos % NW] > pos / NW;
}

// One column of Alg. 2 for the 32 tasks of the tile.  x is the working column
// (shared memory when it fits, else the LU tape in place); the function is
// inlined at two call sites so each keeps a concrete address space.
// Metadata is read warp-coalesced (32 records per load) and broadcast with
// shuffles, so no per-update load sits on the dependency chain.
template <int NW>
__device__ __forceinline__ bool factor_column(const DevView& v, double* x, const double* __restrict__ a,
                                              double* lut, double* out, const int* prog, int len,
                                              int dp, int dep0, int ndep, int u0, int nu,
                                              double stol, int lane, long long* st) {
    long long t0 = st ? clock64() : 0;
    // A(:, j): contiguous in the A tape (fill slots hold zeros), 8 loads in flight
    for (int z0 = 0; z0 < len; z0 += 8) {
        double av[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) av[q] = z0 + q < len ? a[(z0 + q) * kTile] : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (z0 + q < len) x[(z0 + q) * kTile] = av[q];
    }
    long long t1 = 0;
    if (st) {
        __syncwarp();
        t1 = clock64();
        st[0] += t1 - t0;
    }
    // every U dependency column must be final before its L(:, k) is read
    for (int b = 0; b < ndep; b += 32)
        wait_all<NW>(prog, b + lane < ndep ? __ldg(v.dep_wait + dep0 + b + lane) : -1);
    __threadfence_block();
    long long t2 = 0;
    if (st) {
        t2 = clock64();
        st[1] += t2 - t1;
    }
    // VMAD stream in Alg. 2 order: x[dst] -= x[k] * L(i, k)
    const int2* up = reinterpret_cast<const int2*>(v.upd) + u0;
    int2 rec = lane < nu ? __ldg(up + lane) : make_int2(0, 0);
    for (int c = 0; c < nu; c += 32) {
        const int2 rnext = c + 32 + lane < nu ? __ldg(up + c + 32 + lane) : make_int2(0, 0);
        const int m = min(32, nu - c);
        double l[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int ls = __shfl_sync(kFull, rec.x, q);
            l[q] = q < m ? lut[size_t(ls) * kTile] : 0.0;
        }
        for (int g = 0; g < m; g += 8) {
            double ln[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int qq = g + 8 + q;
                const int ls = __shfl_sync(kFull, rec.x, qq & 31);
                ln[q] = qq < m ? lut[size_t(ls) * kTile] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int dk = __shfl_sync(kFull, rec.y, (g + q) & 31);
                if (g + q < m) {
                    const int dst = dk & 0xffff, kp = dk >> 16;
                    x[dst * kTile] = fma(-x[kp * kTile], l[q], x[dst * kTile]);
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) l[q] = ln[q];
        }
        rec = rnext;
    }
    long long t3 = 0;
    if (st) {
        __syncwarp();
        t3 = clock64();
        st[2] += t3 - t2;
    }
    // pivot check and normalization L = x * (1 / pivot)
    const double piv = x[dp * kTile];
    double cmax = 0.0;
    for (int z = 0; z < len; ++z) cmax = fmax(cmax, fabs(x[z * kTile]));
    const bool flagged = isfinite(cmax) && (piv == 0.0 || fabs(piv) < stol * cmax);
    const double inv = 1.0 / piv;
    for (int z = 0; z < len; ++z) {
        const double xv = x[z * kTile];
        out[z * kTile] = z > dp ? xv * inv : xv;
    }
    if (st) {
        __syncwarp();
        st[3] += clock64() - t3;
    }
    return flagged;
}

template <int NW, int CAP>
__global__ void __launch_bounds__(NW * 32, (NW <= 8 ? 3 : 1)) lu_kernel(DevView v) {
    extern __shared__ double xs_all[];  // [NW][CAP][32]
    __shared__ int prog[NW];
    __shared__ unsigned flags[NW];
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (v.tile_active[tile] == 0) return;
    if (threadIdx.x < NW) prog[threadIdx.x] = 0;
    __syncthreads();
    const int t = tile * kTile + lane;
    const double* __restrict__ at = v.A + size_t(tile) * v.nA * kTile + lane;
    double* lut = v.LU + size_t(tile) * v.nnzLU * kTile + lane;
    double* xs = xs_all + size_t(warp) * CAP * kTile + lane;
    const double stol = v.singular_tol;
    const int4* ci = reinterpret_cast<const int4*>(v.col);
    bool flagged = false;
    int done = 0;
    long long stv[4] = {0, 0, 0, 0};
    long long* st = v.lu_stats ? stv : nullptr;
    int4 c0 = make_int4(0, 0, 0, 0), c1 = make_int4(0, 0, 0, 0);
    if (warp < v.nJ) {
        const int j = __ldg(v.lu_sched + warp);
        c0 = __ldg(ci + 2 * j);
        c1 = __ldg(ci + 2 * j + 1);
    }
    for (int p = warp; p < v.nJ; p += NW) {
        int4 n0 = c0, n1 = c1;  // prefetch the next column's record
        if (p + NW < v.nJ) {
            const int jn = __ldg(v.lu_sched + p + NW);
            n0 = __ldg(ci + 2 * jn);
            n1 = __ldg(ci + 2 * jn + 1);
        }
        const int s0 = c0.x, len = c0.y & 0xffff, dp = c0.y >> 16;
        double* col = lut + size_t(s0) * kTile;
        if (CAP > 0 && len <= CAP)
            flagged |= factor_column<NW>(v, xs, at + size_t(s0) * kTile, lut, col, prog, len, dp, c0.z,
                                         c0.w, c1.x, c1.y, stol, lane, st);
        else
            flagged |= factor_column<NW>(v, col, at + size_t(s0) * kTile, lut, col, prog, len, dp, c0.z,
                                         c0.w, c1.x, c1.y, stol, lane, st);
        ++done;
        signal_done(prog, warp, done, lane);
        c0 = n0;
        c1 = n1;
    }
    if (st && lane == 0)
        for (int q = 0; q < 4; ++q) v.lu_stats[(size_t(tile) * NW + warp) * 4 + q] = stv[q];
    // any warp may flag the task; combine through shared memory
    const unsigned fb = __ballot_sync(kFull, flagged);
    if (lane == 0) flags[warp] = fb;
    __syncthreads();
    if (warp == 0) {
        unsigned all = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) all |= flags[w];
        v.flag[t] = (all >> lane) & 1u;
    }
}

// ---------------------------------------------------------------------------
// Forward / backward substitution, pull-style rows with progress counters.
// Per row: the entry records are read warp-coalesced, the LU loads of the
// first 8 entries are issued before the dependency check (which runs on all
// entries in parallel), then b/x loads and the in-order fma chain.
// ---------------------------------------------------------------------------
template <int NW, bool BACK>
__device__ __forceinline__ void tri_solve(const DevView& v, const int32_t* sched,
                                          const RowInfo* rinfo, const RowEnt* ent,
                                          const double* __restrict__ lut, double* bt, int* prog,
                                          int warp, int lane) {
    const int4* rif = reinterpret_cast<const int4*>(rinfo);
    const int4* enf = reinterpret_cast<const int4*>(ent);
    int done = 0;
    int i = warp < v.nJ ? __ldg(sched + warp) : 0;
    int4 ri = warp < v.nJ ? __ldg(rif + i) : make_int4(0, 0, 0, 0);
    for (int p = warp; p < v.nJ; p += NW) {
        int inext = i;
        int4 rnext = ri;
        if (p + NW < v.nJ) {
            inext = __ldg(sched + p + NW);
            rnext = __ldg(rif + inext);
        }
        const int e0 = ri.x, ne = ri.y;
        double acc = bt[size_t(i) * kTile];
        for (int c = 0; c < ne; c += 32) {
            const int4 en = c + lane < ne ? __ldg(enf + e0 + c + lane) : make_int4(0, 0, -1, 0);
            const int m = min(32, ne - c);
            wait_all<NW>(prog, en.z);
            __threadfence_block();
            constexpr int G = NW <= 8 ? 8 : (NW <= 16 ? 4 : 2);
            for (int g = 0; g < m; g += G) {
                double l[G], xb[G];
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const int sl = __shfl_sync(kFull, en.x, (g + q) & 31);
                    const int k = __shfl_sync(kFull, en.y, (g + q) & 31);
                    l[q] = g + q < m ? lut[size_t(sl) * kTile] : 0.0;
                    xb[q] = g + q < m ? bt[size_t(k) * kTile] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < G; ++q)
                    if (g + q < m) acc = fma(-l[q], xb[q], acc);
            }
        }
        if (BACK) acc = acc / lut[size_t(ri.z) * kTile];
        bt[size_t(i) * kTile] = acc;
        ++done;
        signal_done(prog, warp, done, lane);
        i = inext;
        ri = rnext;
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, (NW <= 16 ? 3 : 1)) fsbs_kernel(DevView v, int it) {
    __shared__ int prog[NW];
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (v.tile_active[tile] == 0) return;
    const int t = tile * kTile + lane;
    if (warp == 0 && v.active[t] && v.flag[t]) {  // frozen pivot collapsed
        v.status[t] = GBNR_SINGULAR;
        v.iters[t] = it;
        v.active[t] = 0;
    }
    if (threadIdx.x < NW) prog[threadIdx.x] = 0;
    __syncthreads();
    const double* __restrict__ lut = v.LU + size_t(tile) * v.nnzLU * kTile + lane;
    double* bt = v.b + size_t(tile) * v.nJ * kTile + lane;
    tri_solve<NW, false>(v, v.fs_sched, v.lrow, v.lent, lut, bt, prog, warp, lane);
    __syncthreads();
    if (threadIdx.x < NW) prog[threadIdx.x] = 0;
    __syncthreads();
    tri_solve<NW, true>(v, v.bs_sched, v.urow, v.uent, lut, bt, prog, warp, lane);
}



// ---------------------------------------------------------------------------
// V update for active tasks: va -= dtheta, vm -= d|V|; refresh (cos, sin).
// Block = 8 warps = 8 buses of one tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) vupdate_kernel(DevView v) {
    const int tile = blockIdx.y, lane = threadIdx.x & 31;
    const int bus = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (bus >= v.n || v.tile_active[tile] == 0) return;
    const int t = tile * kTile + lane;
    if (!v.active[t]) return;
    const int zt = v.zcol_t[bus];
    if (zt < 0) return;
    const double* bt = v.b + size_t(tile) * v.nJ * kTile + lane;
    const size_t o = size_t(bus) * v.bpad + t;
    const double va = v.va[o] - bt[size_t(zt) * kTile];
    v.va[o] = va;
    const int zv = v.zcol_v[bus];
    if (zv >= 0) v.vm[o] = v.vm[o] - bt[size_t(zv) * kTile];
    double s, c;
    gb_sincos(va, &s, &c);
    v.s[o] = s;
    v.c[o] = c;
}

__global__ void broadcast_kernel(double* dst, const double* src, int32_t n, int32_t bpad) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < size_t(n) * bpad) dst[i] = src[i / bpad];
}

template <int NW, int CAP>
void set_lu_smem() {
    cudaFuncSetAttribute(lu_kernel<NW, CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         NW * CAP * kTile * int(sizeof(double)));
    cudaFuncSetAttribute(lu_kernel<NW, CAP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

}  // namespace

size_t lu_smem_bytes(const LaunchCfg& c) { return size_t(c.lu_warps) * c.lu_cap * kTile * sizeof(double); }

void configure_kernels(const LaunchCfg& c) {
    (void)c;
    set_lu_smem<4, 32>();
    set_lu_smem<8, 32>();
    set_lu_smem<8, 16>();
    set_lu_smem<8, 0>();
    set_lu_smem<16, 16>();
    set_lu_smem<16, 0>();
}

void launch_init(const DevView& v, cudaStream_t st) { init_kernel<<<v.n_tiles, 256, 0, st>>>(v); }

void launch_npm(const DevView& v, const LaunchCfg& c, int it, cudaStream_t st) {
    if (c.row_warps == 8)
        npm_kernel<8><<<v.n_tiles, 8 * 32, 0, st>>>(v, it);
    else
        npm_kernel<16><<<v.n_tiles, 16 * 32, 0, st>>>(v, it);
}

void launch_jacobian(const DevView& v, const LaunchCfg& c, cudaStream_t st) {
    if (c.row_warps == 8)
        jacobian_kernel<8><<<v.n_tiles, 8 * 32, 0, st>>>(v);
    else
        jacobian_kernel<16><<<v.n_tiles, 16 * 32, 0, st>>>(v);
}

void launch_lu(const DevView& v, const LaunchCfg& c, cudaStream_t st) {
    const size_t sm = lu_smem_bytes(c);
    const int w = c.lu_warps, cap = c.lu_cap;
    if (w == 4 && cap == 32)
        lu_kernel<4, 32><<<v.n_tiles, 4 * 32, sm, st>>>(v);
    else if (w == 8 && cap == 16)
        lu_kernel<8, 16><<<v.n_tiles, 8 * 32, sm, st>>>(v);
    else if (w == 8 && cap == 0)
        lu_kernel<8, 0><<<v.n_tiles, 8 * 32, 0, st>>>(v);
    else if (w == 16 && cap == 16)
        lu_kernel<16, 16><<<v.n_tiles, 16 * 32, sm, st>>>(v);
    else if (w == 16 && cap == 0)
        lu_kernel<16, 0><<<v.n_tiles, 16 * 32, 0, st>>>(v);
    else
        lu_kernel<8, 32><<<v.n_tiles, 8 * 32, 8 * 32 * kTile * sizeof(double), st>>>(v);
}

void launch_fsbs(const DevView& v, const LaunchCfg& c, int it, cudaStream_t st) {
    if (c.fs_warps == 8)
        fsbs_kernel<8><<<v.n_tiles, 8 * 32, 0, st>>>(v, it);
    else if (c.fs_warps == 32)
        fsbs_kernel<32><<<v.n_tiles, 32 * 32, 0, st>>>(v, it);
    else
        fsbs_kernel<16><<<v.n_tiles, 16 * 32, 0, st>>>(v, it);
}

void launch_vupdate(const DevView& v, cudaStream_t st) {
    dim3 grid((v.n + 7) / 8, v.n_tiles);
    vupdate_kernel<<<grid, 256, 0, st>>>(v);
}

void launch_broadcast(double* dst, const double* src, int32_t n, int32_t bpad, cudaStream_t st) {
    const size_t tot = size_t(n) * bpad;
    broadcast_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(dst, src, n, bpad);
}

}  // namespace gbnr
