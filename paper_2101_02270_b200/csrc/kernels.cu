// kernels.cu -- hand-written sm_100a FP64 kernels of one Newton-Raphson iteration.
//
// Layout.  Voltage / injection / right-hand-side tapes are
// element-major, exactly the reference's BatchTape (batch_tape.hpp:6-9):
// value(elem, task) at elem * bpad + task, bpad = 32 * n_tiles.  The two
// [nnzLU]-slot tapes (A = Jacobian in LU slot order, LU = factors) are
// *tile-blocked*: value(slot, task) at (tile * nnzLU + slot) * 32 + lane, so a
// column of one tile is one contiguous run (one TMA bulk copy).  A *tile* is the
// 32 tasks of one warp, one lane per task.
//
//   npm_kernel<JAC> / conv_kernel  compute_npm + convergence (
//                              Alg. 1) fused with update_jacobian into the A tape via the
//                              static lookup (signs per
//                              SURVEY App. B): one sweep computes the currents for both
//   lu_walk_kernel<FS>         refactorize_batch (Alg. 2 operation order)
//                              fused with the forward substitution:
//                              one warp walks one tile through every column (walk.hpp)
//   bs_walk_kernel             backward substitution, one warp per tile, rows in reverse
//   vupdate_kernel             update_voltage + unit phasor refresh
// Scenarios are independent, so no kernel ever needs a grid-wide barrier.
#include "../../include/gbnr.h"
#include "kernels.hpp"
#include "numerics.cuh"

#include <algorithm>

namespace gbnr {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double nan_as_inf_abs(double v) {
    const double a = fabs(v);
    return isnan(a) ? INFINITY : a;
}

// ---------------------------------------------------------------------------
// init: working voltages from the staged inputs, unit phasors, task state
// grid (ceil(n/32), n_super), block 256: warp = tile, 32 buses per block
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) init_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.y * kSuper + warp;
    if (tile >= v.n_tiles) return;
    const int t = tile * v.tw + min(lane, v.tw - 1);
    const bool real = t < v.n_tasks;
    const int b1 = min(v.n, int(blockIdx.x + 1) * 32);
    for (int bus = blockIdx.x * 32; bus < b1; ++bus) {
        const size_t o = size_t(bus) * v.bpad + t;
        const size_t vi = size_t(bus) * v.vin_ld + size_t(real ? t : 0) * v.vin_inc;
        const double vm = real ? v.vm_in[vi] : 1.0, va = real ? v.va_in[vi] : 0.0;
        v.vm[o] = vm;
        v.va[o] = va;
        double s, c;
        gb_sincos(va, &s, &c);
        v.s[o] = s;
        v.c[o] = c;
    }
    if (blockIdx.x == 0 && lane < v.tw) {
        v.status[t] = real ? GBNR_DIVERGED : -1;
        v.iters[t] = 0;
        v.active[t] = real ? 1 : 0;
        v.flag[t] = 0;
        v.maxmis[t] = real ? INFINITY : 0.0;
        v.mis_prev[t] = INFINITY;
        v.jskip[t] = 0;
        v.norm_bits[t] = 0ull;
        if (t == 0) *v.it_dev = 0;
    }
    if (blockIdx.x == 0) {
        const int cnt = __popc(__ballot_sync(kFull, real && lane < v.tw));
        if (lane == 0) v.tile_active[tile] = cnt;
    }
}

// ---------------------------------------------------------------------------
// NPM (Alg. 1, row-level parallelism PAPER.md:183): block (row chunk, super-tile),
// each warp sweeps the chunk's Ybus rows for its tile; partial max-norms merge
// with an exact integer atomicMax on the (non-negative) IEEE bits.
// ---------------------------------------------------------------------------
// JMODE: 0 no Jacobian; 1 speculative (active tasks not predicted to converge at
// this check); 2 the tasks mode 1 skipped that are still active; 3 every active task
enum { kJacNone = 0, kJacSpec = 1, kJacFix = 2, kJacAll = 3 };

// Predicted to converge at this check: quadratic convergence extrapolated from
// the last two checks, |F_k| ~ |F_k-1|^3 / |F_k-2|^2 < tol.  Only decides where
// the Jacobian is computed; a wrong guess costs a kJacFix launch, never a result.
__device__ __forceinline__ bool predict_converged(const DevView& v, int t) {
    if (v.jpolicy != 0) return v.jpolicy == 2;  // never / always deferred
    const double n1 = v.maxmis[t], n2 = v.mis_prev[t];
    return isfinite(n2) && n1 * n1 * n1 < v.tol * n2 * n2;
}

// TW_: the tile width as a compile-time constant (8 / 16 / 24 / 32: no register
// for it under the 5-blocks-per-SM budget), 0 = read from the view.
// Warps cover 32 consecutive tasks whatever the tile width (the element-major
// tapes are task-contiguous); the Jacobian / F stores go to each task's lane of
// its tile's A block.  Lanes past the batch shadow its last task (duplicate
// stores of equal values).
#ifndef GBNR_NPM_BATCH
#define GBNR_NPM_BATCH 2  // neighbours whose loads are issued together in the current sweep (A/B: profiles/r02j)
#endif
// The sweep's A-tape stores (F and J, read back only by the next LU walk) and
// injection loads stream past L2 (evict-first), so the gathered voltages of the
// task group being swept stay L2-resident
#ifndef GBNR_NPM_PLAIN
#define NPM_ST(p, x) __stcs((p), (x))
#define NPM_LDS(p) __ldcs(p)
#else
#define NPM_ST(p, x) (*(p) = (x))
#define NPM_LDS(p) __ldg(p)
#endif
#ifndef GBNR_NPM_MINB
#define GBNR_NPM_MINB 5   // resident blocks per SM the register budget is sized for
#endif
#ifndef GBNR_JSKIP_LANE
#define GBNR_JSKIP_LANE 0
#endif
template <bool NPM, int JMODE, int TW_>
__global__ void __launch_bounds__(256, GBNR_NPM_MINB) npm_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = blockIdx.y * kSuper + warp;  // group of 32 tasks
    if (g * 32 >= v.n_tasks) return;
    const int t = min(g * 32 + lane, v.n_tasks - 1);
    if (!__any_sync(kFull, v.active[t] != 0)) return;  // every task of the group has finished
    const int TW = TW_ ? TW_ : v.tw;
    const size_t bp = v.bpad;
    double* a_t = v.A + size_t(t / TW) * v.tstride + (t % TW);  // tile-blocked A tape
    const size_t yt = size_t(t) * v.y_inc;  // this task's Ybus value set
    bool act = JMODE != kJacNone && v.active[t] != 0;
    if (JMODE == kJacSpec) {
        // skipped per warp: only when every active task of the 32 is predicted to
        // converge.  A lane skipping alone would leave holes in the warp's J stores,
        // and the partial sectors cost their L2 fills from HBM (+1.5 GB, +1.8 ms in
        // the sweep where some tasks converge; profiles/r02jj)
#if GBNR_JSKIP_LANE
        const bool skip = act && predict_converged(v, t);
#else
        const bool all_pred = __all_sync(kFull, !act || predict_converged(v, t));  // every lane votes
        const bool skip = act && all_pred;
#endif
        act = act && !skip;
        if (blockIdx.x == 0) v.jskip[t] = skip;
    } else if (JMODE == kJacFix) {
        act = act && v.jskip[t] != 0;
    }
#if !GBNR_JSKIP_LANE
    // a warp that builds J stores it in every lane, for finished and skipped tasks
    // too (their A rows are dead, or rebuilt bit-identically by the fix launch), so
    // its stores fill whole sectors
    if (JMODE != kJacNone) act = __any_sync(kFull, act);
#endif
    if (JMODE != kJacNone && blockIdx.x == 0) v.flag[t] = 0;  // pivot flags of the coming refactorization
    if (!NPM && !__any_sync(kFull, act)) return;
    double nrm = 0.0;
    const int r1 = min(v.n_rows, int(blockIdx.x + 1) * kRowChunk);
    for (int ri = blockIdx.x * kRowChunk; ri < r1; ++ri) {
        const int r = __ldg(v.rows + ri);
        const int q0 = __ldg(v.yp + r), q1 = __ldg(v.yp + r + 1);
        double ire = 0.0, iim = 0.0;
        int q = q0;
#if GBNR_NPM_BATCH > 1
        constexpr int NB = GBNR_NPM_BATCH;
        for (; q + NB <= q1; q += NB) {  // NB neighbours' loads in flight, then the CSR-order sums
            int kk[NB];
            double gm[NB], gc[NB], gs[NB], gr[NB], gi[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) kk[u] = __ldg(v.yi + q + u);
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                gm[u] = __ldg(v.vm + kk[u] * bp + t);
                gc[u] = __ldg(v.c + kk[u] * bp + t);
                gs[u] = __ldg(v.s + kk[u] * bp + t);
                gr[u] = __ldg(v.yre + size_t(q + u) * v.y_ld + yt);
                gi[u] = __ldg(v.yim + size_t(q + u) * v.y_ld + yt);
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) acc_current(gr[u], gi[u], gm[u] * gc[u], gm[u] * gs[u], ire, iim);
        }
#endif
        for (; q < q1; ++q) {
            const int k = __ldg(v.yi + q);
            const double vmk = __ldg(v.vm + k * bp + t);
            acc_current(__ldg(v.yre + size_t(q) * v.y_ld + yt), __ldg(v.yim + size_t(q) * v.y_ld + yt), vmk * __ldg(v.c + k * bp + t),
                        vmk * __ldg(v.s + k * bp + t), ire, iim);
        }
        const double vmr = __ldg(v.vm + r * bp + t);
        const double vre = vmr * __ldg(v.c + r * bp + t), vim = vmr * __ldg(v.s + r * bp + t);
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        if (NPM) {
            const size_t ts = size_t(t) * v.s_inc;
            const double fp = P - NPM_LDS(v.p0 + size_t(r) * v.s_ld + ts);
            NPM_ST(a_t + size_t(__ldg(v.fslot_p + r)) * TW, fp);  // F beside its A column
            nrm = fmax(nrm, nan_as_inf_abs(fp));
            const int fq_slot = __ldg(v.fslot_q + r);
            if (fq_slot >= 0) {
                const double fq = Q - NPM_LDS(v.q0 + size_t(r) * v.s_ld + ts);
                NPM_ST(a_t + size_t(fq_slot) * TW, fq);
                nrm = fmax(nrm, nan_as_inf_abs(fq));
            }
        }
        if (JMODE != kJacNone && act) {
#ifdef GBNR_NPM_JUNROLL
#pragma unroll 2
#endif
            for (int q = q0; q < q1; ++q) {
                const int k = __ldg(v.yi + q);
                const double ck = __ldg(v.c + k * bp + t), sk = __ldg(v.s + k * bp + t), vmk = __ldg(v.vm + k * bp + t);
                double zre, zim, j[4];
                jac_z(__ldg(v.yre + size_t(q) * v.y_ld + yt), __ldg(v.yim + size_t(q) * v.y_ld + yt), vre, vim, ck, sk, zre, zim);
                jac_entries(k == r, zre, zim, vmk, ck, sk, ire, iim, P, Q, j);
                const int4 l = __ldg(reinterpret_cast<const int4*>(v.lk) + q);
                if (l.x >= 0) NPM_ST(a_t + size_t(l.x) * TW, j[0]);
                if (l.y >= 0) NPM_ST(a_t + size_t(l.y) * TW, j[1]);
                if (l.z >= 0) NPM_ST(a_t + size_t(l.z) * TW, j[2]);
                if (l.w >= 0) NPM_ST(a_t + size_t(l.w) * TW, j[3]);
            }
        }
    }
    if (NPM) atomicMax(v.norm_bits + t, static_cast<unsigned long long>(__double_as_longlong(nrm)));
}

// Convergence / status per task (MATPOWER iteration convention).
__global__ void __launch_bounds__(256) conv_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * kSuper + warp;
    if (tile >= v.n_tiles) return;
    const bool in = lane < v.tw;  // lanes >= tw shadow lane tw - 1: counted once
    const int t = tile * v.tw + min(lane, v.tw - 1);
    const int it = *v.it_dev;
    const double m = __longlong_as_double(static_cast<long long>(v.norm_bits[t]));
    // shadow lanes only read: the real lane owns every write of task t
    bool act = in && v.tile_active[tile] != 0 && v.active[t] != 0;
    if (in) v.norm_bits[t] = 0ull;
    if (act) {
        if (it == 0) v.mis0[t] = m;
        v.mis_prev[t] = v.maxmis[t];
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
    const int nj = __popc(__ballot_sync(kFull, act && v.jskip[t] != 0));
    if (lane == 0) {
        v.tile_active[tile] = cnt;
        if (cnt) {
            atomicAdd(v.active_count + it, cnt);     // active tasks after iteration it
            atomicAdd(v.active_count + 32 + it, 1);  // tiles with work left
        }
        if (nj) atomicAdd(v.active_count + 96 + it, nj);  // still active, Jacobian skipped
    }
}

// Iteration bump; publishes this iteration's counters to mapped host memory (a
// kernel store over PCIe, not a DMA copy that would queue behind bulk D2H
// traffic of a pipelined neighbouring batch).
__global__ void bump_kernel(DevView v) {
    const int it = *v.it_dev;
    volatile int32_t* h = v.h_counts;
    h[it] = v.active_count[it];
    h[32 + it] = v.active_count[32 + it];
    h[96 + it] = v.active_count[96 + it];
    __threadfence_system();
    *v.it_dev = it + 1;
}

// Final per-status task counts -> mapped host memory.
__global__ void status_count_kernel(DevView v) {
    __shared__ int c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < v.n_tasks; t += blockDim.x) {
        const int s = v.status[t];
        atomicAdd(&c[(s >= 0 && s <= 3) ? s : 2], 1);
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        volatile int32_t* h = v.h_counts;
        h[64 + threadIdx.x] = c[threadIdx.x];
    }
    __threadfence_system();
}


// ---------------------------------------------------------------------------
// Tile walks (walk.hpp).  One warp = one tile = one CTA.  Shared memory is a
// ring of step blocks plus a staging ring, filled by cp.async.bulk (TMA) copies
// that complete on mbarriers (expect_tx).  Lane 0 issues the host-planned ops
// as the warp passes their events; every lane computes its own task.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// A value the compiler must keep (or spill) instead of re-deriving it: the walk
// loops run at the 80-register cap, where ptxas otherwise rematerialises the
// tile's tape pointers and shared addresses from SR_CTAID / SR_TID / SR_CgaCtaId
// reads at every record dispatch.
#ifndef GBNR_OPAQUE
#define GBNR_OPAQUE 1
#endif
#ifndef GBNR_LANE_SHFL
#define GBNR_LANE_SHFL 1  // the LU walk's lane id through a shuffle (profiles/r02pp_lane_shfl.log)
#endif
__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
#if GBNR_OPAQUE
    asm volatile("mov.b32 %0, %0;\n" : "+r"(x));
#endif
    return x;
}
template <class T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
#if GBNR_OPAQUE
    asm volatile("mov.b64 %0, %0;\n" : "+l"(p));
#endif
    return p;
}
// Shared row address of the low / high 16-bit row index of a packed word
// (PRMT / SHF, then one shift-add for the power-of-two row sizes); RB = bytes per
// row = tile width x 8
__device__ __forceinline__ unsigned row_lo(unsigned base, int32_t w, unsigned RB) {
    return base + __byte_perm(unsigned(w), 0u, 0x4410) * RB;
}
__device__ __forceinline__ unsigned row_hi(unsigned base, int32_t w, unsigned RB) {
    return base + __byte_perm(unsigned(w), 0u, 0x4432) * RB;
}
// 32-bit shared-window accesses of the walk rows (no generic-address arithmetic)
__device__ __forceinline__ double lds(unsigned a) {
    double r;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void sts(unsigned a, double x) {
    asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try_s(unsigned a, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_s(unsigned a, unsigned parity) {
    if (mbar_try_s(a, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_s(a, parity)) {
        if (clock64() - t0 > (1ll << 33)) __trap();
    }
}
// Bounded wait: a plan bug must fail loudly (trap -> CUDA error), never hang the GPU.
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    if (mbar_try(b, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try(b, parity)) {
        if (clock64() - t0 > (1ll << 33)) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// generic-proxy writes -> later async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// The walk's program is a word stream (walk.hpp kRec*) paged through shared
// memory by TMA; every lane reads the same words (smem broadcast).
constexpr int kWalkBars = 32;   // op i completes on barrier i % 32
constexpr int kWalkPages = 2;   // resident program pages

struct Prog {
    double* R;                  // smem rows [ring_rows + stage_rows][32]
    int32_t* pg;                // smem pages [kWalkPages][page_words]
    unsigned long long* bar;    // op barriers [kWalkBars]
    unsigned long long* pbar;   // page barriers [kWalkPages]
    const int32_t* gs;          // stream in global memory
    const int32_t* cur;         // next record
    const char* tb;             // this tile's tape block: A, LU, b rows (256 B each)
    int32_t tape_rows;          // rows per tape: tape t starts at row t * tape_rows
    int W, n_pages, page;
    int once_tape;              // tape whose copies the walk reads exactly once: L2 evict-first
    unsigned Rs, bars;          // shared-window addresses of R and bar (kept, not re-derived)
};

// Debug timeline (GBNR_DBG & 4): kernel start (-1), phase barrier (0), end (1).
#ifdef GBNR_TRACE
__device__ __noinline__ void walk_trace_print(int tile, int warp, int what) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    printf("[walk] tile %d warp %d %s at %llu ns\n", tile, warp,
           what < 0 ? "start" : (what == 0 ? "reached sync" : "done"), t);
}
#endif
__device__ __forceinline__ void walk_trace(const DevView& v, int tile, int warp, int lane, int what) {
#ifdef GBNR_TRACE  // make GBNR_TRACE=1: compiled out of production builds (no call frame)
    if ((v.dbg & 4) && lane == 0 && (tile == 0 || tile == v.n_tiles - 1)) walk_trace_print(tile, warp, what);
#endif
}

// Walker time breakdown (make GBNR_PROF=1, GBNR_DBG & 8): clock64 deltas per
// record category, summed over tiles per (phase, warp) into DevView::prof.
#ifdef GBNR_PROF
#define PROF_DECL long long pf_t = clock64(), pf[12] = {0}; int pf_ph = 0;
#define PROF_MARK(c) { const long long now_ = clock64(); pf[c] += now_ - pf_t; pf_t = now_; }
#define PROF_CNT(c) { pf[c] += 1; }
#define PROF_FLUSH                                                                          \
    if (v.prof && lane == 0) {                                                              \
        for (int i_ = 0; i_ < 12; ++i_)                                                     \
            if (warp < 8) atomicAdd(v.prof + (size_t(pf_ph) * 8 + warp) * 16 + i_, (unsigned long long)pf[i_]); \
        for (int i_ = 0; i_ < 12; ++i_) pf[i_] = 0;                                         \
    }
#else
#define PROF_DECL
#define PROF_MARK(c)
#define PROF_CNT(c)
#define PROF_FLUSH
#endif

// Shared memory of a walk CTA: [rows][32] doubles shared by the walkers (each
// phase's plan gives every walker a disjoint share), then per walker its
// program pages and its op / page mbarriers.
__device__ __forceinline__ void prog_begin(const DevView& v, const WalkView& w, Prog& P, int tile, int warp,
                                           int lane) {
    extern __shared__ __align__(128) unsigned char walk_smem[];
    P.R = reinterpret_cast<double*>(walk_smem);
    unsigned char* mine = walk_smem + size_t(w.rows) * size_t(w.tw) * 8 +
                          size_t(warp) * (size_t(kWalkPages) * w.page_words * 4 + (kWalkBars + kWalkPages) * 8);
    P.pg = reinterpret_cast<int32_t*>(mine);
    P.bar = reinterpret_cast<unsigned long long*>(mine + size_t(kWalkPages) * w.page_words * 4);
    P.pbar = P.bar + kWalkBars;
    P.Rs = opaque_u32(smem_u32(P.R));
    P.bars = opaque_u32(smem_u32(P.bar));
    P.W = w.page_words;
    P.gs = w.stream + size_t(w.wpage0[warp]) * P.W;
    P.n_pages = w.wpage0[warp + 1] - w.wpage0[warp];
    P.page = 0;
    P.cur = P.pg;
    P.tb = reinterpret_cast<const char*>(v.A + size_t(tile) * v.tstride);
    P.tape_rows = v.tape_rows;
    P.once_tape = w.once_tape;
    mbar_init(P.bar + lane, 1);
    if (lane < kWalkPages) mbar_init(P.pbar + lane, 1);
    __syncwarp();  // every lane's barrier is initialised before lane 0 arms the page barriers
    if (lane == 0) {
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int p = 0; p < kWalkPages && p < P.n_pages; ++p) {
            mbar_expect_tx(P.pbar + p, unsigned(P.W) * 4u);
            bulk_g2s(P.pg + p * P.W, P.gs + size_t(p) * P.W, unsigned(P.W) * 4u, P.pbar + p);
        }
    }
    __syncwarp();
    mbar_wait(P.pbar, 0);
}

__device__ __forceinline__ void prog_next_page(Prog& P, int lane) {
    __syncwarp();
    const int slot = P.page & (kWalkPages - 1);
    if (lane == 0 && P.page + kWalkPages < P.n_pages) {
        fence_proxy_async_smem();
        mbar_expect_tx(P.pbar + slot, unsigned(P.W) * 4u);
        bulk_g2s(P.pg + slot * P.W, P.gs + size_t(P.page + kWalkPages) * P.W, unsigned(P.W) * 4u, P.pbar + slot);
    }
    ++P.page;
    const int ns = P.page & (kWalkPages - 1);
    P.cur = P.pg + ns * P.W;
    mbar_wait(P.pbar + ns, unsigned((P.page / kWalkPages) & 1));
}

// kRecIssue: lane 0 arms the op's barrier and issues its bulk copies.
__device__ __forceinline__ int prog_issue(const DevView& v, Prog& P, const int32_t* r, int lane, unsigned RB) {
    const int ncopy = (r[0] >> 4) & 0xfff;
    fence_proxy_async_smem();  // this lane's smem accesses before the async overwrite
    const unsigned ubar = P.bars + unsigned(r[1] & (kWalkBars - 1)) * 8u;
    __syncwarp();
    if (lane == 0)  // rows -> bytes
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(ubar), "r"(unsigned(r[2]) * RB)
                     : "memory");
    // one copy per lane; a copy may complete before lane 0's arrive.expect_tx (the
    // barrier's tx-count dips below zero, its phase cannot complete without the arrive)
    const unsigned rbase = P.Rs;
    for (int i = lane; i < ncopy; i += 32) {
        const int32_t c = r[3 + 2 * i], slot = r[4 + 2 * i];
        const unsigned rows = (unsigned(c) >> 2) & 1023u, smem = unsigned(c) >> 12;
        const char* src = P.tb + size_t(unsigned((c & 3) * P.tape_rows + slot)) * RB;
        if ((c & 3) == P.once_tape) {  // the walk reads this tape once: evict first from L2
            asm volatile(
                "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
                " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}\n" ::"r"(
                    rbase + smem * RB),
                "l"(src), "r"(rows * RB), "r"(ubar)
                : "memory");
            continue;
        }
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                rbase + smem * RB),
            "l"(src), "r"(rows * RB), "r"(ubar)
            : "memory");
    }
    return 3 + 2 * ncopy;
}

__device__ __forceinline__ void prog_wait(const Prog& P, int op) {
    mbar_wait_s(P.bars + unsigned(op & (kWalkBars - 1)) * 8u, unsigned((op / kWalkBars) & 1));
}

// Forward walk: Alg. 2 column by column (+ forward substitution when FS).
// Shared rows are addressed as 32-bit shared-window offsets: row r of this
// lane at R0 + r * 256.
// TW_: the tile width as a compile-time constant (8 / 16 / 24 / 32), 0 = from the view.
template <bool FS, int TW_>
__global__ void __launch_bounds__(32 * kLuWarps, 3) lu_walk_kernel(DevView v, WalkView w) {
    const unsigned tid = opaque_u32(threadIdx.x);
    const int tile = int(opaque_u32(blockIdx.x)), warp = int(tid >> 5);
#if GBNR_LANE_SHFL
    const int lane = __shfl_sync(kFull, int(tid & 31u), int(tid & 31u));  // a register ptxas cannot re-derive
#else
    const int lane = int(tid & 31u);
#endif
    if (tile >= v.n_tiles || v.tile_active[tile] == 0) return;
    Prog P;
    walk_trace(v, tile, warp, lane, -1);
    prog_begin(v, w, P, tile, warp, lane);
    const int TW = TW_ ? TW_ : v.tw, le = min(lane, TW - 1);  // lanes >= tw shadow lane tw - 1
    double* lu_t = opaque_ptr(v.LU + size_t(tile) * v.tstride + le);
    const double stol = v.singular_tol;
    const unsigned RB = unsigned(TW) * 8u;  // bytes per shared / tape row
    const unsigned R0 = P.Rs + unsigned(le) * 8u;
    bool flagged = false;
    unsigned xs = R0;  // this step's block
    int len = 0, dp = 0, lslot = 0, brow = 0;  // brow: slot of y_m in the backward block
    double acc_y = 0.0;
    // global forms (walk.hpp kRec*G): the step's block as a generic pointer (shared
    // rows or this walker's global scratch), and the running column maximum
    double* xg = nullptr;
    double gmax = 0.0;
    int32_t h = P.cur[0];  // header of the next record, loaded one record ahead
    PROF_DECL
    for (;;) {
        const int32_t* r = P.cur;
        const int type = h & 15;
        if (__builtin_expect(type == kRecDep2, 1)) {
            // supernode pair k, k+1: x[kpos2] -= m1 L(k+1,k) gives m2; then every
            // other row gets k's update, then k+1's (the oracle's order per element)
            const int op = (h >> 4) - 1;
            const int w1 = r[1], w2 = r[2], w3 = r[3], w4 = r[4], w5 = r[5];
            const int fs2 = w5 & 0xffff, op2 = int(unsigned(w5) >> 16) - 1;
            const int nrows = w2 & 0xffff;
            const int n4 = (nrows + 3) & ~3;
            h = r[6 + (n4 >> 1)];
            PROF_MARK(5)
            if (op >= 0) prog_wait(P, op);
            if (op2 >= 0) prog_wait(P, op2);
            PROF_MARK(1)
            PROF_CNT(10)
            const unsigned s1 = R0 + (unsigned(w2) >> 16) * RB, s2 = R0 + unsigned(w3 & 0xffff) * RB;
            const int fs1 = int(unsigned(w3) >> 16);
            double fl1 = 0.0, fy1 = 0.0, fl2 = 0.0, fy2 = 0.0;
            if (FS && fs1 != 0xffff) {
                fl1 = lds(s1 + unsigned(fs1) * RB);
                fy1 = lds(R0 + unsigned(w4 & 0xffff) * RB);
            }
            if (FS && fs2 != 0xffff) {
                fl2 = lds(s2 + unsigned(fs2) * RB);
                fy2 = lds(R0 + (unsigned(w4) >> 16) * RB);
            }
            const double m1 = lds(xs + unsigned(w1 & 0xffff) * RB);
            const unsigned p2 = xs + (unsigned(w1) >> 16) * RB;
            const double m2 = fma(-m1, lds(s1), lds(p2));
            sts(p2, m2);
            const int32_t* dw = r + 6;
            const int last = nrows - 1;
#pragma unroll 1
            for (int q = 0; q < nrows; q += 4) {
                const int32_t v0 = dw[q >> 1], v1 = dw[(q >> 1) + 1];
                const unsigned d0 = row_lo(xs, v0, RB), d1 = row_hi(xs, v0, RB);
                const unsigned d2 = row_lo(xs, v1, RB), d3 = row_hi(xs, v1, RB);
                const int q1 = min(q + 1, last), q2 = min(q + 2, last), q3 = min(q + 3, last);
                const double a0 = lds(s1 + unsigned(q + 1) * RB), a1 = lds(s1 + unsigned(q1 + 1) * RB);
                const double a2 = lds(s1 + unsigned(q2 + 1) * RB), a3 = lds(s1 + unsigned(q3 + 1) * RB);
                const double b0 = lds(s2 + unsigned(q) * RB), b1 = lds(s2 + unsigned(q1) * RB);
                const double b2 = lds(s2 + unsigned(q2) * RB), b3 = lds(s2 + unsigned(q3) * RB);
                double x0 = lds(d0), x1 = lds(d1), x2 = lds(d2), x3 = lds(d3);
                x0 = fma(-m2, b0, fma(-m1, a0, x0));
                x1 = fma(-m2, b1, fma(-m1, a1, x1));
                x2 = fma(-m2, b2, fma(-m1, a2, x2));
                x3 = fma(-m2, b3, fma(-m1, a3, x3));
                sts(d0, x0);
                sts(d1, x1);
                sts(d2, x2);
                sts(d3, x3);
            }
            if (FS) {
                if (fs1 != 0xffff) acc_y = fma(-fl1, fy1, acc_y);
                if (fs2 != 0xffff) acc_y = fma(-fl2, fy2, acc_y);
            }
            P.cur += 6 + (n4 >> 1);
            PROF_MARK(5)
        } else if (__builtin_expect(type == kRecDep, 1)) {
            const int op = (h >> 4) - 1;
            const int kpos_fs = r[1], nrows = r[2] & 0xffff, src_row = int(unsigned(r[2]) >> 16);
            const int ysrc = r[3];
            const int n4 = (nrows + 3) & ~3;  // destinations padded with the scratch row len
            h = r[4 + (n4 >> 1)];
            PROF_MARK(4)
            if (op >= 0) prog_wait(P, op);
            PROF_MARK(1)
            PROF_CNT(9)
            const unsigned src = R0 + unsigned(src_row) * RB;
            // forward-substitution operands first: they live in other blocks than
            // the x being updated, so their latency hides under the update
            const int fspos = int(unsigned(kpos_fs) >> 16);
            double fl = 0.0, fy = 0.0;
            if (FS && fspos != 0xffff) {
                fl = lds(src + unsigned(fspos) * RB);
                fy = lds(R0 + unsigned(ysrc) * RB);
            }
            if (nrows > 0) {
                const double mult = lds(xs + unsigned(kpos_fs & 0xffff) * RB);
                const int32_t* dw = r + 4;
                int q = 0;
#pragma unroll 1
                for (; q + 8 <= nrows; q += 8) {  // eight independent rows in flight
                    const int32_t w0 = dw[q >> 1], w1 = dw[(q >> 1) + 1], w2 = dw[(q >> 1) + 2],
                                  w3 = dw[(q >> 1) + 3];
                    const unsigned d0 = row_lo(xs, w0, RB), d1 = row_hi(xs, w0, RB);
                    const unsigned d2 = row_lo(xs, w1, RB), d3 = row_hi(xs, w1, RB);
                    const unsigned d4 = row_lo(xs, w2, RB), d5 = row_hi(xs, w2, RB);
                    const unsigned d6 = row_lo(xs, w3, RB), d7 = row_hi(xs, w3, RB);
                    const unsigned sq = src + unsigned(q) * RB;
                    double l[8], a[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) l[u] = lds(sq + unsigned(u) * RB);
                    a[0] = lds(d0);
                    a[1] = lds(d1);
                    a[2] = lds(d2);
                    a[3] = lds(d3);
                    a[4] = lds(d4);
                    a[5] = lds(d5);
                    a[6] = lds(d6);
                    a[7] = lds(d7);
#pragma unroll
                    for (int u = 0; u < 8; ++u) a[u] = fma(-mult, l[u], a[u]);
                    sts(d0, a[0]);
                    sts(d1, a[1]);
                    sts(d2, a[2]);
                    sts(d3, a[3]);
                    sts(d4, a[4]);
                    sts(d5, a[5]);
                    sts(d6, a[6]);
                    sts(d7, a[7]);
                }
#pragma unroll 1
                for (; q < nrows; q += 4) {
                    // whole groups of 4: padding rows re-read the last L row and
                    // land in the scratch row
                    const int32_t w0 = dw[q >> 1], w1 = dw[(q >> 1) + 1];
                    const unsigned d0 = row_lo(xs, w0, RB), d1 = row_hi(xs, w0, RB);
                    const unsigned d2 = row_lo(xs, w1, RB), d3 = row_hi(xs, w1, RB);
                    const unsigned sq = src + unsigned(q) * RB;
                    const int last = nrows - 1;
                    const double l0 = lds(sq), l1 = lds(src + unsigned(min(q + 1, last)) * RB);
                    const double l2 = lds(src + unsigned(min(q + 2, last)) * RB);
                    const double l3 = lds(src + unsigned(min(q + 3, last)) * RB);
                    double a0 = lds(d0), a1 = lds(d1), a2 = lds(d2), a3 = lds(d3);
                    a0 = fma(-mult, l0, a0);
                    a1 = fma(-mult, l1, a1);
                    a2 = fma(-mult, l2, a2);
                    a3 = fma(-mult, l3, a3);
                    sts(d0, a0);
                    sts(d1, a1);
                    sts(d2, a2);
                    sts(d3, a3);
                }
            }
            if (FS && fspos != 0xffff) acc_y = fma(-fl, fy, acc_y);
            P.cur += 4 + (n4 >> 1);
            PROF_MARK(4)
        } else if (__builtin_expect(type == kRecIssue, 1)) {
            P.cur += prog_issue(v, P, r, lane, RB);
            h = P.cur[0];
            PROF_MARK(7)
            PROF_CNT(11)
        } else if (type == kRecStep) {
            const int ring = r[1] & 0xffff;
            len = int(unsigned(r[1]) >> 16);
            dp = r[2];
            lslot = r[3];
            brow = r[4];
            const int op = r[5];
            h = r[6];
            P.cur += 6;
            PROF_MARK(8)
            prog_wait(P, op);
            PROF_MARK(0)
            PROF_CNT(3)
            xs = R0 + unsigned(ring) * RB;
            xg = P.R + size_t(ring) * TW + le;
            acc_y = FS ? lds(xs + unsigned(len) * RB) : 0.0;
        } else if (type == kRecEnd) {
            h = r[1 + dp];
            // normalization L = x * (1 / pivot) and the U scatter, with the
            // pivot check's column maximum folded into the same
            // passes over x (max |x| is exact in any order)
            const double piv = lds(xs + unsigned(dp) * RB);
            const double inv = 1.0 / piv;
            double c0 = fabs(piv), c1 = 0.0;
            double* lcol = lu_t + ptrdiff_t(lslot - dp - 1) * TW;  // L row z of x at lcol[z], y at lcol[len]
            int z = dp + 1;
            for (; z + 2 <= len; z += 2) {
                const double x0 = lds(xs + unsigned(z) * RB), x1 = lds(xs + unsigned(z + 1) * RB);
                c0 = fmax(c0, fabs(x0));
                c1 = fmax(c1, fabs(x1));
                const double l0 = x0 * inv, l1 = x1 * inv;
                sts(xs + unsigned(z) * RB, l0);
                sts(xs + unsigned(z + 1) * RB, l1);
                lcol[size_t(z) * TW] = l0;
                lcol[size_t(z + 1) * TW] = l1;
            }
            if (z < len) {
                const double x0 = lds(xs + unsigned(z) * RB);
                c0 = fmax(c0, fabs(x0));
                const double l0 = x0 * inv;
                sts(xs + unsigned(z) * RB, l0);
                lcol[size_t(z) * TW] = l0;
            }
            z = 0;
            for (; z + 4 <= dp; z += 4) {  // U part -> its row-major slots
                const int32_t s0 = r[1 + z], s1 = r[2 + z], s2 = r[3 + z], s3 = r[4 + z];
                const double u0 = lds(xs + unsigned(z) * RB), u1 = lds(xs + unsigned(z + 1) * RB),
                             u2 = lds(xs + unsigned(z + 2) * RB), u3 = lds(xs + unsigned(z + 3) * RB);
                c0 = fmax(c0, fabs(u0));
                c1 = fmax(c1, fabs(u1));
                c0 = fmax(c0, fabs(u2));
                c1 = fmax(c1, fabs(u3));
                lu_t[size_t(s0) * TW] = u0;
                lu_t[size_t(s1) * TW] = u1;
                lu_t[size_t(s2) * TW] = u2;
                lu_t[size_t(s3) * TW] = u3;
            }
            for (; z < dp; ++z) {
                const double u0 = lds(xs + unsigned(z) * RB);
                c0 = fmax(c0, fabs(u0));
                lu_t[size_t(r[1 + z]) * TW] = u0;
            }
            const double cmax = fmax(c0, c1);
            flagged |= isfinite(cmax) && (piv == 0.0 || fabs(piv) < stol * cmax);
            lu_t[size_t(brow + 1) * TW] = piv;  // U(m,m) closing the backward block
            if (FS) {  // y_m after the L rows (forward re-fetches) and in the backward block
                sts(xs + unsigned(len) * RB, acc_y);
                lcol[size_t(len) * TW] = acc_y;
                lu_t[size_t(brow) * TW] = acc_y;
            }
            fence_proxy_async_global();  // later TMA re-fetches of this column see it
            P.cur += 1 + dp;
            PROF_MARK(6)
        } else if (type == kRecPage) {
            PROF_MARK(8)
            prog_next_page(P, lane);
            h = P.cur[0];
            PROF_MARK(2)
        } else if (type == kRecDepG) {
            // a dependency read from global memory (L(:,k) and y_k in the LU tape)
            const int op = (h >> 4) - 1;
            const int kpos_fs = r[1], nrows = r[2], slot = r[3], nl = r[4];
            h = r[5 + ((nrows + 1) >> 1)];
            if (op >= 0) prog_wait(P, op);
            const double* src = lu_t + size_t(slot) * TW;
            const int fspos = int(unsigned(kpos_fs) >> 16);
            if (nrows > 0) {
                const double mult = xg[size_t(kpos_fs & 0xffff) * TW];
                const int32_t* dw = r + 5;
                int q = 0;
#pragma unroll 1
                for (; q + 8 <= nrows; q += 8) {  // 16 independent loads in flight per group
                    int d[8];
                    double l[8], a[8];
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const int32_t wq = dw[(q + u) >> 1];
                        d[u] = wq & 0xffff;
                        d[u + 1] = int(unsigned(wq) >> 16);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) l[u] = src[size_t(q + u) * TW];
#pragma unroll
                    for (int u = 0; u < 8; ++u) a[u] = xg[size_t(d[u]) * TW];
#pragma unroll
                    for (int u = 0; u < 8; ++u) xg[size_t(d[u]) * TW] = fma(-mult, l[u], a[u]);
                }
                for (; q < nrows; ++q) {
                    const int32_t wq = dw[q >> 1];
                    const int d = (q & 1) ? int(unsigned(wq) >> 16) : (wq & 0xffff);
                    xg[size_t(d) * TW] = fma(-mult, src[size_t(q) * TW], xg[size_t(d) * TW]);
                }
            }
            if (FS && fspos != 0xffff) acc_y = fma(-src[size_t(fspos) * TW], src[size_t(nl) * TW], acc_y);
            P.cur += 5 + ((nrows + 1) >> 1);
        } else if (type == kRecStepG) {
            // a column too large for the pool: A rows + F into this walker's scratch
            len = r[1] & 0xffff;
            dp = int(unsigned(r[1]) >> 16);
            const int a0 = r[2];
            lslot = r[3];
            brow = r[4];
            h = r[5];
            P.cur += 5;
            xg = v.scratch + (size_t(tile) * kLuWarps + warp) * size_t(v.scratch_rows) * TW + le;
            const double* at = v.A + size_t(tile) * v.tstride + le + size_t(a0) * TW;
            int z = 0;
#pragma unroll 1
            for (; z + 8 <= len + 1; z += 8) {  // loads grouped ahead of the stores
                double a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = at[size_t(z + u) * TW];
#pragma unroll
                for (int u = 0; u < 8; ++u) xg[size_t(z + u) * TW] = a[u];
            }
            for (; z <= len; ++z) xg[size_t(z) * TW] = at[size_t(z) * TW];
            acc_y = FS ? xg[size_t(len) * TW] : 0.0;
            gmax = 0.0;
        } else if (type == kRecEndU) {
            // U entries z0 .. z0+cnt-1 of a global step -> their row-major slots
            const int cnt = (h >> 4) & 0xfffff, z0 = r[1];
            h = r[2 + cnt];
            int i = 0;
#pragma unroll 1
            for (; i + 8 <= cnt; i += 8) {
                double u[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) u[k] = xg[size_t(z0 + i + k) * TW];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    gmax = fmax(gmax, fabs(u[k]));
                    lu_t[size_t(r[2 + i + k]) * TW] = u[k];
                }
            }
            for (; i < cnt; ++i) {
                const double u = xg[size_t(z0 + i) * TW];
                gmax = fmax(gmax, fabs(u));
                lu_t[size_t(r[2 + i]) * TW] = u;
            }
            P.cur += 2 + cnt;
        } else if (type == kRecEndG) {
            // END of a global step (the U part went out in kRecEndU records)
            h = r[1];
            const double piv = xg[size_t(dp) * TW];
            const double inv = 1.0 / piv;
            double c0 = fmax(gmax, fabs(piv));
            double* lcol = lu_t + ptrdiff_t(lslot - dp - 1) * TW;
            int z = dp + 1;
#pragma unroll 1
            for (; z + 8 <= len; z += 8) {
                double x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = xg[size_t(z + k) * TW];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    c0 = fmax(c0, fabs(x[k]));
                    lcol[size_t(z + k) * TW] = x[k] * inv;
                }
            }
            for (; z < len; ++z) {
                const double x0 = xg[size_t(z) * TW];
                c0 = fmax(c0, fabs(x0));
                lcol[size_t(z) * TW] = x0 * inv;
            }
            flagged |= isfinite(c0) && (piv == 0.0 || fabs(piv) < stol * c0);
            lu_t[size_t(brow + 1) * TW] = piv;
            if (FS) {
                lcol[size_t(len) * TW] = acc_y;
                lu_t[size_t(brow) * TW] = acc_y;
            }
            fence_proxy_async_global();  // later TMA re-fetches of this column see it
            P.cur += 1;
        } else if (type == kRecSync) {
            walk_trace(v, tile, warp, lane, 0);
            PROF_MARK(8)
            __syncthreads();  // phase boundary: every walker's columns are written and fenced
            PROF_MARK(3)
            PROF_FLUSH
#ifdef GBNR_PROF
            ++pf_ph;
#endif
            P.cur += 1;
            h = P.cur[0];
        } else {
            walk_trace(v, tile, warp, lane, 1);
            PROF_MARK(8)
            PROF_FLUSH
            break;
        }
    }
    if (flagged && v.active[tile * TW + le]) v.flag[tile * TW + le] = 1;
}

// Backward walk: x_i = (y_i - sum_k U(i,k) x_k) / U(i,i), k descending.
// up to kBsWarps walkers, three CTAs per SM
template <int TW_>
__global__ void __launch_bounds__(32 * kBsWarps, 3) bs_walk_kernel(DevView v, WalkView w) {
    const int tile = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (tile >= v.n_tiles || v.tile_active[tile] == 0) return;
    Prog P;
    walk_trace(v, tile, warp, lane, -1);
    prog_begin(v, w, P, tile, warp, lane);
    const int TW = TW_ ? TW_ : v.tw, le = min(lane, TW - 1);  // lanes >= tw shadow lane tw - 1
    double* b_t = v.b + size_t(tile) * v.tstride + le;
    const double* lu_t = v.LU + size_t(tile) * v.tstride + le;
    const unsigned RB = unsigned(TW) * 8u;
    const unsigned R0 = P.Rs + unsigned(le) * 8u;
    unsigned blk = R0, e = R0;  // this step's block; its next U entry
    const double *blk_g = lu_t, *e_g = lu_t;  // a global step's row block in the LU tape
    int ne = 0, brow = 0;
    double acc = 0.0;
    int32_t h = P.cur[0];  // header of the next record, loaded one record ahead
    for (;;) {
        const int32_t* r = P.cur;
        const int type = h & 15;
        if (__builtin_expect(type == kRecDepN, 1)) {
            const int op = (h >> 4) - 1;
            const int n = r[1];
            h = r[2 + ((n + 1) >> 1)];
            if (op >= 0) prog_wait(P, op);
            const int32_t* yw = r + 2;
            int i = 0;
            for (; i + 2 <= n; i += 2) {  // acc -= U(i,k) x_k, k descending (operand loads paired)
                const int32_t w2 = yw[i >> 1];
                const double u0 = lds(e), x0 = lds(row_lo(R0, w2, RB)), u1 = lds(e + RB), x1 = lds(row_hi(R0, w2, RB));
                acc = fma(-u0, x0, acc);
                acc = fma(-u1, x1, acc);
                e += 2 * RB;
            }
            if (i < n) {
                acc = fma(-lds(e), lds(row_lo(R0, yw[i >> 1], RB)), acc);
                e += RB;
            }
            P.cur += 2 + ((n + 1) >> 1);
        } else if (__builtin_expect(type == kRecIssue, 1)) {
            const int len = prog_issue(v, P, r, lane, RB);
            P.cur += len;
            h = P.cur[0];
        } else if (type == kRecStep) {
            const int ring = r[1] & 0xffff;
            ne = int(unsigned(r[1]) >> 16);
            brow = r[4];
            const int op = r[5];
            h = r[6];
            P.cur += 6;
            prog_wait(P, op);
            blk = R0 + unsigned(ring) * RB;
            e = blk;
            acc = lds(blk + unsigned(ne) * RB);
        } else if (type == kRecEnd) {
            h = r[1];
            const double xi = acc / lds(blk + unsigned(ne + 1) * RB);
            sts(blk + unsigned(ne) * RB, xi);
            b_t[size_t(brow) * TW] = xi;
            fence_proxy_async_global();
            P.cur += 1;
        } else if (type == kRecPage) {
            prog_next_page(P, lane);
            h = P.cur[0];
        } else if (type == kRecPair) {
            // two independent rows A, B: their dependency chains interleave (each
            // accumulator sees its own row's operations in the unpaired order)
            const int nA = (h >> 4) & 0xfff, nw = (h >> 16) & 0xff;
            const int32_t wa = r[1], wb = r[2], bra = r[3], brb = r[4], ops = r[5], nB = r[6];
            const int32_t* ya = r + 7 + nw;
            const int32_t* yb = ya + ((nA + 1) >> 1);
            h = yb[(nB + 1) >> 1];
            if ((ops & 0xffff) != 0) prog_wait(P, (ops & 0xffff) - 1);
            if ((unsigned(ops) >> 16) != 0) prog_wait(P, int(unsigned(ops) >> 16) - 1);
            for (int i = 0; i < nw; ++i) prog_wait(P, r[7 + i] - 1);
            const unsigned ba = R0 + unsigned(wa & 0xffff) * RB, bb = R0 + unsigned(wb & 0xffff) * RB;
            const unsigned nea = unsigned(wa) >> 16, neb = unsigned(wb) >> 16;
            double acca = lds(ba + nea * RB), accb = lds(bb + neb * RB);
            unsigned ea = ba, eb = bb;
            const int m = min(nA, nB);
            int i = 0;
#pragma unroll 1
            for (; i < m; ++i) {
                const int32_t pa = ya[i >> 1], pb = yb[i >> 1];
                const double xa = lds((i & 1) ? row_hi(R0, pa, RB) : row_lo(R0, pa, RB));
                const double xb = lds((i & 1) ? row_hi(R0, pb, RB) : row_lo(R0, pb, RB));
                const double ua = lds(ea), ub = lds(eb);
                acca = fma(-ua, xa, acca);
                accb = fma(-ub, xb, accb);
                ea += RB;
                eb += RB;
            }
            for (int j = i; j < nA; ++j) {
                const int32_t pa = ya[j >> 1];
                acca = fma(-lds(ea), lds((j & 1) ? row_hi(R0, pa, RB) : row_lo(R0, pa, RB)), acca);
                ea += RB;
            }
            for (int j = i; j < nB; ++j) {
                const int32_t pb = yb[j >> 1];
                accb = fma(-lds(eb), lds((j & 1) ? row_hi(R0, pb, RB) : row_lo(R0, pb, RB)), accb);
                eb += RB;
            }
            const double xa = acca / lds(ba + (nea + 1) * RB), xb = accb / lds(bb + (neb + 1) * RB);
            sts(ba + nea * RB, xa);
            sts(bb + neb * RB, xb);
            b_t[size_t(bra) * TW] = xa;
            b_t[size_t(brb) * TW] = xb;
            fence_proxy_async_global();
            P.cur = yb + ((nB + 1) >> 1);
        } else if (type == kRecStepG) {
            // a row too long for the pool: its block read in place from the LU tape
            ne = r[1];
            blk_g = e_g = lu_t + size_t(r[2]) * TW;
            brow = r[3];
            h = r[4];
            P.cur += 4;
            acc = blk_g[size_t(ne) * TW];
        } else if (type == kRecDepNG) {
            const int n = (h >> 4) & 0xfffff;
            h = r[1 + n];
            int i = 0;
#pragma unroll 1
            for (; i + 8 <= n; i += 8) {  // acc -= U(i,k) x_k, k descending, x_k from the b tape
                double u[8], x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    u[k] = e_g[size_t(k) * TW];
                    x[k] = b_t[size_t(r[1 + i + k]) * TW];
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = fma(-u[k], x[k], acc);
                e_g += 8 * TW;
            }
            for (; i < n; ++i) {
                acc = fma(-e_g[0], b_t[size_t(r[1 + i]) * TW], acc);
                e_g += TW;
            }
            P.cur += 1 + n;
        } else if (type == kRecEndG) {
            h = r[1];
            b_t[size_t(brow) * TW] = acc / blk_g[size_t(ne + 1) * TW];
            fence_proxy_async_global();
            P.cur += 1;
        } else if (type == kRecSync) {
            walk_trace(v, tile, warp, lane, 0);
            __syncthreads();  // phase boundary: every walker's columns are written and fenced
            P.cur += 1;
            h = P.cur[0];
        } else {
            walk_trace(v, tile, warp, lane, 1);
            break;
        }
    }
}

// ---------------------------------------------------------------------------
// V update for active tasks: va -= dtheta, vm -= d|V|; refresh (cos, sin).
// block (32-bus chunk, super-tile), warp = tile.
// ---------------------------------------------------------------------------
#ifndef GBNR_VUP_BATCH
#define GBNR_VUP_BATCH 8  // buses per load batch (A/B: profiles/r02ff)
#endif
template <int TW_>
__global__ void __launch_bounds__(256) vupdate_kernel(DevView v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = (blockIdx.y * kSuper + warp) * 32 + lane;  // 32 consecutive tasks per warp
    const bool in = t < v.n_tasks;
    bool upd = in && v.active[t];
    if (upd && v.flag[t]) {  // frozen pivot collapsed: stop, never update V
        if (blockIdx.x == 0) {
            v.status[t] = GBNR_SINGULAR;
            v.iters[t] = *v.it_dev;
            v.active[t] = 0;
        }
        upd = false;
    }
    // Lanes of finished tasks in a warp that updates rewrite their unchanged values
    // (x - 0.0 == x; cos / sin recomputed from the angle, as every writer of the
    // tapes does), so the warp's stores fill whole sectors instead of leaving
    // holes that L2 fills from HBM
    if (!__any_sync(kFull, upd) || !in) return;
    const int TW = TW_ ? TW_ : v.tw;
    const size_t bp = v.bpad;
    const double* b_t = v.b + size_t(t / TW) * v.tstride + (t % TW);  // tile-blocked b tape
    const int b0 = blockIdx.x * 32, b1 = min(v.n, b0 + 32);
    // VB buses' loads in flight per warp before their updates (the loop is
    // latency-bound at one bus per round trip otherwise)
    constexpr int VB = GBNR_VUP_BATCH;
    for (int bus = b0; bus < b1; bus += VB) {
        int zt[VB], zv[VB];
        double va[VB], vm[VB], dt[VB], dv[VB];
#pragma unroll
        for (int u = 0; u < VB; ++u) {
            const bool in = bus + u < b1;
            zt[u] = in ? __ldg(v.zcol_t + bus + u) : -1;
            zv[u] = in ? __ldg(v.zcol_v + bus + u) : -1;
        }
#pragma unroll
        for (int u = 0; u < VB; ++u) {
            const size_t o = size_t(bus + u) * bp + t;
            if (zt[u] >= 0) {
                va[u] = v.va[o];
                dt[u] = upd ? b_t[size_t(zt[u]) * TW] : 0.0;
            }
            if (zt[u] >= 0 && zv[u] >= 0) {
                vm[u] = v.vm[o];
                dv[u] = upd ? b_t[size_t(zv[u]) * TW] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < VB; ++u) {
            if (zt[u] < 0) continue;
            const size_t o = size_t(bus + u) * bp + t;
            const double a = va[u] - dt[u];
            v.va[o] = a;
            if (zv[u] >= 0) v.vm[o] = vm[u] - dv[u];
            double s, c;
            gb_sincos(a, &s, &c);
            v.s[o] = s;
            v.c[o] = c;
        }
    }
}

// calc_branch_flows on the solved voltages: block (32-branch
// chunk, super-tile), warp = tile; outputs [n_branch][n_tasks] packed.
__global__ void __launch_bounds__(256) flows_kernel(DevView v, int32_t nb, const int32_t* bf, const int32_t* bt,
                                                    const double* adm, const int32_t* outage, double* sfr,
                                                    double* sfi, double* str, double* sti) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.y * kSuper + warp;
    if (tile >= v.n_tiles) return;
    const int t = tile * v.tw + lane;
    if (lane >= v.tw || t >= v.n_tasks) return;
    const size_t bp = v.bpad, T = size_t(v.n_tasks);
    const int out = outage ? outage[t] : -1;
    const int k1 = min(nb, int(blockIdx.x + 1) * 32);
    for (int k = blockIdx.x * 32; k < k1; ++k) {
        const size_t o = size_t(k) * T + t;
        if (k == out) {
            sfr[o] = sfi[o] = str[o] = sti[o] = 0.0;
            continue;
        }
        const int f = __ldg(bf + k), to = __ldg(bt + k);
        const double vmf = v.vm[f * bp + t], vmt = v.vm[to * bp + t];
        // unit phasors from the angles (the same gb_sincos that fills the c / s tapes,
        // so voltages written back from the host -- second chance -- need no c / s)
        double sf, cf, st, ct;
        gb_sincos(v.va[f * bp + t], &sf, &cf);
        gb_sincos(v.va[to * bp + t], &st, &ct);
        const double vfr = vmf * cf, vfi = vmf * sf;
        const double vtr = vmt * ct, vti = vmt * st;
        const double* a = adm + size_t(8) * k;
        double P, Q;
        branch_end_flow(__ldg(a), __ldg(a + 1), __ldg(a + 2), __ldg(a + 3), vfr, vfi, vtr, vti, vfr, vfi, P, Q);
        sfr[o] = P;
        sfi[o] = Q;
        branch_end_flow(__ldg(a + 4), __ldg(a + 5), __ldg(a + 6), __ldg(a + 7), vfr, vfi, vtr, vti, vtr, vti, P, Q);
        str[o] = P;
        sti[o] = Q;
    }
}

// [n][bpad] -> [n][n_tasks] (packed for a single linear D2H copy)
__global__ void pack_kernel(double* __restrict__ dst, const double* __restrict__ src, int32_t n, int32_t n_tasks,
                            int32_t bpad) {
    const size_t tot = size_t(n) * n_tasks;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < tot; i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / size_t(n_tasks), t = i - r * size_t(n_tasks);
        dst[i] = src[r * size_t(bpad) + t];
    }
}

__global__ void broadcast_kernel(double* dst, const double* src, int32_t n, int32_t bpad) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < size_t(n) * bpad) dst[i] = src[i / bpad];
}

unsigned n_super(const DevView& v) { return unsigned((v.n_tiles + kSuper - 1) / kSuper); }
// blocks of 8 warps x 32 consecutive tasks (NPM, V update)
unsigned n_groups8(const DevView& v) { return unsigned((v.n_tasks + 32 * kSuper - 1) / (32 * kSuper)); }

}  // namespace

size_t walk_smem_bytes(const WalkView& w) {
    return size_t(w.rows) * size_t(w.tw) * 8 +
           size_t(w.walkers) * (size_t(kWalkPages) * w.page_words * 4 + size_t(kWalkBars + kWalkPages) * 8);
}

template <class K>
void configure_walk(K k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

template <int TW_>
void configure_width() {
    configure_walk(lu_walk_kernel<true, TW_>);
    configure_walk(lu_walk_kernel<false, TW_>);
    configure_walk(bs_walk_kernel<TW_>);
}

void configure_kernels() {
    configure_width<0>();
    configure_width<8>();
    configure_width<16>();
    configure_width<24>();
    configure_width<32>();
}

int bs_ctas_per_sm(size_t smem, int threads) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, bs_walk_kernel<32>, threads, smem) != cudaSuccess) return 0;
    return n;
}

int walk_ctas_per_sm(size_t smem, int threads) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lu_walk_kernel<true, 32>, threads, smem) != cudaSuccess)
        return 0;
    return n;
}

void launch_init(const DevView& v, cudaStream_t st) {
    init_kernel<<<dim3(unsigned((v.n + 31) / 32), n_super(v)), 256, 0, st>>>(v);
}

template <bool NPM, int JMODE>
void launch_npm_tw(const DevView& v, dim3 grid, cudaStream_t st) {
    switch (v.tw) {
        case 8: npm_kernel<NPM, JMODE, 8><<<grid, 256, 0, st>>>(v); break;
        case 16: npm_kernel<NPM, JMODE, 16><<<grid, 256, 0, st>>>(v); break;
        case 24: npm_kernel<NPM, JMODE, 24><<<grid, 256, 0, st>>>(v); break;
        case 32: npm_kernel<NPM, JMODE, 32><<<grid, 256, 0, st>>>(v); break;
        default: npm_kernel<NPM, JMODE, 0><<<grid, 256, 0, st>>>(v); break;
    }
}

void launch_npm(const DevView& v, bool jac, cudaStream_t st) {
    const dim3 grid(unsigned((v.n_rows + kRowChunk - 1) / kRowChunk), n_groups8(v));
    if (jac)
        launch_npm_tw<true, kJacSpec>(v, grid, st);
    else
        launch_npm_tw<true, kJacNone>(v, grid, st);
    conv_kernel<<<n_super(v), 256, 0, st>>>(v);
    bump_kernel<<<1, 1, 0, st>>>(v);
}

void launch_status_count(const DevView& v, cudaStream_t st) { status_count_kernel<<<1, 1024, 0, st>>>(v); }

void launch_jacobian(const DevView& v, bool all, cudaStream_t st) {
    const dim3 grid(unsigned((v.n_rows + kRowChunk - 1) / kRowChunk), n_groups8(v));
    if (all)
        launch_npm_tw<false, kJacAll>(v, grid, st);
    else
        launch_npm_tw<false, kJacFix>(v, grid, st);
}

template <int TW_>
void launch_lu_tw(const DevView& v, const WalkView& w, bool fs, cudaStream_t st) {
    const size_t smem = walk_smem_bytes(w);
    const unsigned threads = unsigned(32 * w.walkers);
    if (fs)
        lu_walk_kernel<true, TW_><<<unsigned(v.n_tiles), threads, smem, st>>>(v, w);
    else
        lu_walk_kernel<false, TW_><<<unsigned(v.n_tiles), threads, smem, st>>>(v, w);
}

void launch_lu_walk(const DevView& v, const WalkView& w, bool fs, cudaStream_t st) {
    switch (v.tw) {
        case 8: launch_lu_tw<8>(v, w, fs, st); break;
        case 16: launch_lu_tw<16>(v, w, fs, st); break;
        case 24: launch_lu_tw<24>(v, w, fs, st); break;
        case 32: launch_lu_tw<32>(v, w, fs, st); break;
        default: launch_lu_tw<0>(v, w, fs, st); break;
    }
}

void launch_bs_walk(const DevView& v, const WalkView& w, cudaStream_t st) {
    const dim3 grid(unsigned(v.n_tiles)), block(unsigned(32 * w.walkers));
    const size_t smem = walk_smem_bytes(w);
    switch (v.tw) {
        case 8: bs_walk_kernel<8><<<grid, block, smem, st>>>(v, w); break;
        case 16: bs_walk_kernel<16><<<grid, block, smem, st>>>(v, w); break;
        case 24: bs_walk_kernel<24><<<grid, block, smem, st>>>(v, w); break;
        case 32: bs_walk_kernel<32><<<grid, block, smem, st>>>(v, w); break;
        default: bs_walk_kernel<0><<<grid, block, smem, st>>>(v, w); break;
    }
}

void launch_vupdate(const DevView& v, cudaStream_t st) {
    const dim3 grid(unsigned((v.n + 31) / 32), n_groups8(v));
    switch (v.tw) {
        case 8: vupdate_kernel<8><<<grid, 256, 0, st>>>(v); break;
        case 16: vupdate_kernel<16><<<grid, 256, 0, st>>>(v); break;
        case 24: vupdate_kernel<24><<<grid, 256, 0, st>>>(v); break;
        case 32: vupdate_kernel<32><<<grid, 256, 0, st>>>(v); break;
        default: vupdate_kernel<0><<<grid, 256, 0, st>>>(v); break;
    }
}

void launch_flows(const DevView& v, int32_t nb, const int32_t* bf, const int32_t* bt, const double* adm,
                  const int32_t* outage, double* sfr, double* sfi, double* str, double* sti, cudaStream_t st) {
    flows_kernel<<<dim3(unsigned((nb + 31) / 32), n_super(v)), 256, 0, st>>>(v, nb, bf, bt, adm, outage, sfr, sfi,
                                                                          str, sti);
}

void launch_pack(double* dst, const double* src, int32_t n, int32_t n_tasks, int32_t bpad, cudaStream_t st) {
    pack_kernel<<<148 * 8, 256, 0, st>>>(dst, src, n, n_tasks, bpad);
}

void launch_broadcast(double* dst, const double* src, int32_t n, int32_t bpad, cudaStream_t st) {
    const size_t tot = size_t(n) * bpad;
    broadcast_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(dst, src, n, bpad);
}

}  // namespace gbnr
