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
#include <cuda/atomic>

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
__device__ __forceinline__ void wait_done(int* prog, int pos) {
    const int ow = pos % NW, rk = pos / NW;
    cuda::atomic_ref<int, cuda::thread_scope_block> a(prog[ow]);
    while (a.load(cuda::memory_order_acquire) <= rk) {
    }
}

__device__ __forceinline__ void signal_done(int* prog, int warp, int value, int lane) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
        cuda::atomic_ref<int, cuda::thread_scope_block> a(prog[warp]);
        a.store(value, cuda::memory_order_release);
    }
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
        if (!real) {
            v.vm[o] = 1.0;
            v.va[o] = 0.0;
        }
        double s, c;
        gb_sincos(v.va[o], &s, &c);
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
__global__ void __launch_bounds__(NW * 32) npm_kernel(DevView v, int it) {
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
            if (cnt) atomicAdd(v.active_count + it, cnt);
        }
    }
}

// ---------------------------------------------------------------------------
// Jacobian -> A tape (J nonzeros in LU slot order; fill slots are implicit).
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32) jacobian_kernel(DevView v) {
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
template <int NW, int CAP>
__global__ void __launch_bounds__(NW * 32) lu_kernel(DevView v) {
    extern __shared__ double xs_all[];  // [NW][CAP][32]
    __shared__ int prog[NW];
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (v.tile_active[tile] == 0) return;
    if (threadIdx.x < NW) prog[threadIdx.x] = 0;
    __syncthreads();
    const int t = tile * kTile + lane;
    const double* __restrict__ at = v.A + size_t(tile) * v.nA * kTile + lane;
    double* lut = v.LU + size_t(tile) * v.nnzLU * kTile + lane;
    double* xs = xs_all + size_t(warp) * CAP * kTile + lane;
    const double stol = v.singular_tol;
    bool flagged = false;
    int done = 0;
    for (int p = warp; p < v.nJ; p += NW) {
        const int j = v.lu_sched[p];
        const ColInfo ci = v.col[j];
        const int len = ci.len_dp & 0xffff, dp = ci.len_dp >> 16;
        double* x = len <= CAP ? xs : lut + size_t(ci.s0) * kTile;
        // gather A(:, j); fill positions start at zero (Alg. 3 preamble)
        for (int z = 0; z < len; ++z) {
            const int a = v.aidx[ci.s0 + z];
            x[z * kTile] = a >= 0 ? at[size_t(a) * kTile] : 0.0;
        }
        // x(L rows) -= x(k) * L(:, k) for the U dependencies k, ascending
        const int d1 = ci.dep0 + ci.ndep;
        for (int d = ci.dep0; d < d1; ++d) {
            const DepInfo di = v.dep[d];
            wait_done<NW>(prog, di.wait);
            const int cnt = di.cnt_pos & 0xffff;
            const double xk = x[(di.cnt_pos >> 16) * kTile];
            const double* lk = lut + size_t(di.lstart) * kTile;
            const uint16_t* dst = v.upd + di.upd0;
            int z = 0;
            for (; z + 4 <= cnt; z += 4) {
                const double l0 = lk[(z + 0) * kTile], l1 = lk[(z + 1) * kTile];
                const double l2 = lk[(z + 2) * kTile], l3 = lk[(z + 3) * kTile];
                const int e0 = dst[z], e1 = dst[z + 1], e2 = dst[z + 2], e3 = dst[z + 3];
                x[e0 * kTile] = fma(-xk, l0, x[e0 * kTile]);
                x[e1 * kTile] = fma(-xk, l1, x[e1 * kTile]);
                x[e2 * kTile] = fma(-xk, l2, x[e2 * kTile]);
                x[e3 * kTile] = fma(-xk, l3, x[e3 * kTile]);
            }
            for (; z < cnt; ++z) {
                const int e = dst[z];
                x[e * kTile] = fma(-xk, lk[z * kTile], x[e * kTile]);
            }
        }
        // pivot check and normalization L = x / pivot
        const double piv = x[dp * kTile];
        double cmax = 0.0;
        for (int z = 0; z < len; ++z) cmax = fmax(cmax, fabs(x[z * kTile]));
        if (isfinite(cmax) && (piv == 0.0 || fabs(piv) < stol * cmax)) flagged = true;
        const double inv = 1.0 / piv;
        double* out = lut + size_t(ci.s0) * kTile;
        for (int z = 0; z < len; ++z) {
            const double xv = x[z * kTile];
            out[z * kTile] = z > dp ? xv * inv : xv;
        }
        ++done;
        signal_done(prog, warp, done, lane);
    }
    // any warp may flag the task; combine through shared memory
    __shared__ unsigned flags[NW];
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
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32) fsbs_kernel(DevView v, int it) {
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
    int done = 0;
    for (int p = warp; p < v.nJ; p += NW) {
        const int i = v.fs_sched[p];
        const RowInfo ri = v.lrow[i];
        double acc = bt[size_t(i) * kTile];
        for (int e = ri.e0; e < ri.e0 + ri.ne; ++e) {
            const RowEnt en = v.lent[e];
            wait_done<NW>(prog, en.wait);
            acc = fma(-lut[size_t(en.slot) * kTile], bt[size_t(en.k) * kTile], acc);
        }
        bt[size_t(i) * kTile] = acc;
        ++done;
        signal_done(prog, warp, done, lane);
    }
    __syncthreads();
    if (threadIdx.x < NW) prog[threadIdx.x] = 0;
    __syncthreads();
    done = 0;
    for (int p = warp; p < v.nJ; p += NW) {
        const int i = v.bs_sched[p];
        const RowInfo ri = v.urow[i];
        double acc = bt[size_t(i) * kTile];
        for (int e = ri.e0; e < ri.e0 + ri.ne; ++e) {
            const RowEnt en = v.uent[e];
            wait_done<NW>(prog, en.wait);
            acc = fma(-lut[size_t(en.slot) * kTile], bt[size_t(en.k) * kTile], acc);
        }
        bt[size_t(i) * kTile] = acc / lut[size_t(ri.diag) * kTile];
        ++done;
        signal_done(prog, warp, done, lane);
    }
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
}

}  // namespace

size_t lu_smem_bytes(const LaunchCfg& c) { return size_t(c.lu_warps) * c.lu_cap * kTile * sizeof(double); }

void configure_kernels(const LaunchCfg& c) {
    (void)c;
    set_lu_smem<4, 32>();
    set_lu_smem<8, 32>();
    set_lu_smem<16, 32>();
    set_lu_smem<8, 16>();
    set_lu_smem<16, 16>();
    set_lu_smem<8, 64>();
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
    if (c.lu_warps == 4 && c.lu_cap == 32)
        lu_kernel<4, 32><<<v.n_tiles, 4 * 32, sm, st>>>(v);
    else if (c.lu_warps == 16 && c.lu_cap == 32)
        lu_kernel<16, 32><<<v.n_tiles, 16 * 32, sm, st>>>(v);
    else if (c.lu_warps == 8 && c.lu_cap == 16)
        lu_kernel<8, 16><<<v.n_tiles, 8 * 32, sm, st>>>(v);
    else if (c.lu_warps == 16 && c.lu_cap == 16)
        lu_kernel<16, 16><<<v.n_tiles, 16 * 32, sm, st>>>(v);
    else if (c.lu_warps == 8 && c.lu_cap == 64)
        lu_kernel<8, 64><<<v.n_tiles, 8 * 32, sm, st>>>(v);
    else
        lu_kernel<8, 32><<<v.n_tiles, 8 * 32, lu_smem_bytes(LaunchCfg{8, c.row_warps, 32}), st>>>(v);
}

void launch_fsbs(const DevView& v, const LaunchCfg& c, int it, cudaStream_t st) {
    if (c.lu_warps == 4)
        fsbs_kernel<4><<<v.n_tiles, 4 * 32, 0, st>>>(v, it);
    else if (c.lu_warps == 16)
        fsbs_kernel<16><<<v.n_tiles, 16 * 32, 0, st>>>(v, it);
    else
        fsbs_kernel<8><<<v.n_tiles, 8 * 32, 0, st>>>(v, it);
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
