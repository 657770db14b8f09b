// plan.cu -- the gbnr_plan object and the extern "C" boundary (include/gbnr.h).
//
// A plan owns the frozen symbolic state (symbolic.cpp) replicated on its
// device, the per-batch tapes, one CUDA stream and pinned scratch.  The Newton
// loop is driven from the host: one launch per kernel per iteration, and one
// 4-byte device->host read of the active-task count per iteration to stop as
// soon as every task has finished (PAPER.md:193 checked convergence on the
// CPU; here the check itself runs on the device, only the count comes back).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <atomic>
#include <chrono>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gbnr.h"
#include "kernels.hpp"
#include "symbolic.hpp"

using gbnr::Error;

namespace {

thread_local std::string g_err;

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw Error(GBNR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return GBNR_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return GBNR_ECONFIG;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GBNR_ECONFIG;
    }
}

// Device memory is stream-ordered (cudaMallocAsync / cudaFreeAsync on the plan's
// stream): a plan freeing its buffers never synchronizes the device, so the
// concurrent second-chance plans of one solve do not serialize each other.
template <class T>
T* dev_upload(std::vector<void*>& owned, const std::vector<T>& h, cudaStream_t st) {
    T* d = nullptr;
    const size_t bytes = std::max<size_t>(h.size(), 1) * sizeof(T);
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes, st));
    owned.push_back(d);
    if (!h.empty()) CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return d;
}

enum Phase { kNpm = 0, kJac, kLu, kFsbs, kVupd, kPhases };

}  // namespace

// gbnr_plan_create with `sub`: a second-chance / re-derivation plan (no LU-only walk)
static int create_plan(int32_t n_bus, const int32_t* indptr, const int32_t* indices, const double* y_re,
                       const double* y_im, int32_t ref, const int32_t* pv, int32_t n_pv, const int32_t* pq,
                       int32_t n_pq, const double* vm0, const double* va0, const gbnr_options* opt, gbnr_plan** out,
                       bool sub);

struct gbnr_plan {
    gbnr::Symbolic sym;
    std::vector<int32_t> in_pv, in_pq;  // creation inputs kept for second-chance re-plans
    gbnr::LuLayout lay;
    // The walk programs depend on the tile width only through each walker's row
    // budget (a row is one value per task of a tile): one set per tile width,
    // planned on first use (tile width).
    struct TileWalks {
        int32_t tw = gbnr::kTile;
        gbnr::WalkSet wf, wl, wb;        // forward LU+FS, LU-only, backward walks
        gbnr::WalkView vf{}, vl{}, vb{};
    };
    std::vector<std::unique_ptr<TileWalks>> walks;
    TileWalks* cur = nullptr;    // the walks of the staged batch's tile width
    gbnr::WalkConfig wcfg;       // planning configuration (row bytes set per width)
    int32_t n_sm = 148, ctas_per_sm = 3;
    gbnr_options opt{};
    bool on_device = false;
    cudaStream_t stream = nullptr;
    // batch pipeline (gbnr_solve_batches): copy streams, a second input set and
    // two result sets, so batch i+1's H2D and batch i-1's D2H overlap batch i
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    std::vector<void*> pipe;
    size_t pipe_lanes = 0;
    double *p0_set[2] = {nullptr, nullptr}, *q0_set[2] = {nullptr, nullptr};
    double *out_vm[2] = {nullptr, nullptr}, *out_va[2] = {nullptr, nullptr}, *out_mm[2] = {nullptr, nullptr};
    int32_t *out_it[2] = {nullptr, nullptr}, *out_st[2] = {nullptr, nullptr};
    cudaEvent_t ev_in[2] = {}, ev_free_in[2] = {}, ev_res[2] = {}, ev_out[2] = {};
    // pinned staging of the small per-task results (a D2H into pageable memory
    // would block the host until the copy stream drains)
    int32_t *h_it[2] = {nullptr, nullptr}, *h_st[2] = {nullptr, nullptr};
    double* h_mm[2] = {nullptr, nullptr};
    std::vector<void*> owned;     // structure buffers
    double* d_scratch = nullptr;  // [n] staging for broadcast sets
    std::vector<void*> batch;     // per-batch tapes
    size_t cap_lanes = 0;         // allocated task slots (tiles x tile width)
    int32_t cap_scratch = 0;      // allocated global-step scratch rows per walker
    size_t a_bytes = 0;           // A + LU + b tape bytes
    int32_t a_tw = 0;             // tile width whose Jacobian slots the A tape holds (0: all zero)
    size_t batch_bytes = 0, pipe_bytes = 0;  // device bytes held by the batch tapes / the pipeline
    std::vector<double> y_host_re, y_host_im;       // the plan's shared Ybus values (host copy)
    std::vector<std::unique_ptr<gbnr_plan>> peers;  // device plans 2..n_devices (gbnr_options.n_devices)
    bool sub_plan = false;         // a second-chance / re-derivation plan: no LU-only walk
    bool whole_on_device = false;  // the device state holds every task of the last solve
    double *p0_own = nullptr, *q0_own = nullptr;  // [n][bpad] injections owned by the plan
    bool staged = false;
    bool solved = false;  // device voltages hold a finished solve
    gbnr::DevView v{};
    int32_t* h_count = nullptr;   // pinned, mapped (device writes counters here)
    double timing[24] = {0};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // profiling: an event pair per phase, recorded without host syncs and
    // resolved once at the end of the solve
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_used;  // (phase, first event index)

    template <class T>
    T* dev_upload_s(const std::vector<T>& h) {
        return dev_upload(owned, h, stream);
    }
    void* dmalloc(size_t bytes) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), stream));
        return p;
    }
    void dfree(void* p) {
        if (p) cudaFreeAsync(p, stream);
    }

    ~gbnr_plan() {
        if (!on_device) return;
        cudaSetDevice(opt.device);
        if (stream) cudaStreamSynchronize(stream);
        for (void* p : batch) dfree(p);
        for (void* p : owned) dfree(p);
        if (h_count) cudaFreeHost(h_count);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
        for (void* q : pipe) dfree(q);
        dfree(y_task_re);
        dfree(y_task_im);
        if (stream) cudaStreamSynchronize(stream);
        for (int i = 0; i < 2; ++i) {
            for (cudaEvent_t e : {ev_in[i], ev_free_in[i], ev_res[i], ev_out[i]})
                if (e) cudaEventDestroy(e);
            if (h_it[i]) cudaFreeHost(h_it[i]);
            if (h_st[i]) cudaFreeHost(h_st[i]);
            if (h_mm[i]) cudaFreeHost(h_mm[i]);
        }
        if (s_h2d) cudaStreamDestroy(s_h2d);
        if (s_d2h) cudaStreamDestroy(s_d2h);
        if (stream) cudaStreamDestroy(stream);
    }

    void upload_structure() {
        CK(cudaSetDevice(opt.device));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t* e : {&ev_in[i], &ev_free_in[i], &ev_res[i], &ev_out[i]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CK(cudaHostAlloc(&h_count, sizeof(int32_t) * 128, cudaHostAllocMapped));
        {
            void* dp = nullptr;
            CK(cudaHostGetDevicePointer(&dp, h_count, 0));
            v.h_counts = static_cast<int32_t*>(dp);
        }
        CK(cudaEventCreate(&ev0));
        CK(cudaEventCreate(&ev1));
        gbnr::configure_kernels();
        const gbnr::Symbolic& s = sym;
        d_scratch = static_cast<double*>(dmalloc(size_t(s.n) * sizeof(double)));
        owned.push_back(d_scratch);
        v.n = s.n;
        v.nJ = s.nJ;
        v.nnzY = s.nnzY;
        v.n_rows = static_cast<int32_t>(s.rows.size());
        v.nnzLU = static_cast<int32_t>(s.nnzLU);
        v.yp = dev_upload_s(s.yp);
        v.yi = dev_upload_s(s.yi);
        v.rows = dev_upload_s(s.rows);
        v.brow_p = dev_upload_s(s.brow_p);
        v.brow_q = dev_upload_s(s.brow_q);
        {
            // A-tape slots (walk.hpp LuLayout): CCS entry z of column j at z + j,
            // F_m right after column m
            std::vector<int32_t> col_of(s.nnzLU);
            for (int32_t j = 0; j < s.nJ; ++j)
                for (int32_t z = s.cp[j]; z < s.cp[j + 1]; ++z) col_of[z] = j;
            std::vector<int32_t> lk(s.lk.size()), fp(s.brow_p.size()), fq(s.brow_q.size());
            for (size_t i = 0; i < lk.size(); ++i) lk[i] = s.lk[i] >= 0 ? gbnr::a_slot(s.lk[i], col_of[s.lk[i]]) : -1;
            auto fslot = [&](int32_t m) { return m >= 0 ? gbnr::a_slot(s.cp[m + 1], m) : -1; };
            for (size_t r = 0; r < fp.size(); ++r) fp[r] = fslot(s.brow_p[r]);
            for (size_t r = 0; r < fq.size(); ++r) fq[r] = fslot(s.brow_q[r]);
            v.lk = dev_upload_s(lk);
            v.fslot_p = dev_upload_s(fp);
            v.fslot_q = dev_upload_s(fq);
            v.tape_rows = lay.rows;
        }
        {
            // dx_k sits at b-tape row nJ-1-k (walk.hpp: the backward walk's
            // descending dependencies then re-fetch ascending rows and merge)
            std::vector<int32_t> zt(s.zcol_t), zv(s.zcol_v);
            for (int32_t& z : zt) z = z >= 0 ? s.nJ - 1 - z : -1;
            for (int32_t& z : zv) z = z >= 0 ? s.nJ - 1 - z : -1;
            v.zcol_t = dev_upload_s(zt);
            v.zcol_v = dev_upload_s(zv);
        }
        int32_t* itd = nullptr;
        itd = static_cast<int32_t*>(dmalloc(sizeof(int32_t)));
        owned.push_back(itd);
        v.it_dev = itd;
        if (const char* d = std::getenv("GBNR_DBG")) v.dbg = std::atoi(d);
#ifdef GBNR_PROF
        if (v.dbg & 8) {
            v.prof = static_cast<unsigned long long*>(dmalloc(4 * 8 * 16 * sizeof(unsigned long long)));
            owned.push_back(v.prof);
        }
#endif
        CK(cudaStreamSynchronize(stream));
        v.tol = opt.tol;
        v.singular_tol = opt.singular_tol;
        v.max_iter = opt.max_iter;
        v.jpolicy = opt.jacobian;
    }

    gbnr::WalkView upload_walk(const gbnr::WalkSet& w, int32_t tw) {
        gbnr::WalkView x{};
        x.stream = dev_upload_s(w.stream);
        x.walkers = w.walkers;
        x.page_words = w.page_words;
        x.rows = w.rows;
        x.tw = tw;
        if (w.walkers < 1 || w.walkers > 16) throw Error(GBNR_ECONFIG, "1..16 walkers per tile");
        for (int32_t i = 0; i <= w.walkers; ++i) x.wpage0[i] = w.wpage0[i];
        if (w.barriers != 32 || w.pages != 2) throw Error(GBNR_ECONFIG, "walk kernels use 32 barriers, 2 pages");
        if (w.row_bytes != tw * 8 || gbnr::walk_smem_bytes(x) != w.smem_bytes())
            throw Error(GBNR_ECONFIG, "walk smem layout mismatch");
        if (gbnr::walk_smem_bytes(x) > 227 * 1024)
            throw Error(GBNR_ECONFIG, "walk needs more shared memory than a B200 CTA has");
        return x;
    }

    // Walkers of the backward walk (at most kBsWarps; GBNR_BS_WALKERS overrides).
    int32_t bs_walkers() const {
        int32_t k = std::min(gbnr::kBsWarps, std::max(opt.walkers, 1) == 8 ? gbnr::kBsWarps : opt.walkers);
        if (const char* e = std::getenv("GBNR_BS_WALKERS")) k = std::atoi(e);
        return std::max(1, std::min(k, gbnr::kBsWarps));
    }

    // The walks of tile width tw, planned (and on a device plan uploaded) on first
    // use.  On the device the row budget shrinks until ctas_per_sm walk CTAs really
    // co-reside on an SM.
    TileWalks* walks_for(int32_t tw) {
        for (auto& w : walks)
            if (w->tw == tw) return w.get();
        auto tws = std::make_unique<TileWalks>();
        tws->tw = tw;
        gbnr::WalkConfig wc = wcfg;
        wc.row_bytes = tw * 8;
        // the three programs are independent: planned on three host threads
        auto build = [&] {
            std::exception_ptr e1, e2;
            std::thread tl([&] {
                try {
                    if (!sub_plan) tws->wl = gbnr::build_forward_walk(sym, lay, false, wc);
                } catch (...) {
                    e1 = std::current_exception();
                }
            });
            std::thread tb([&] {
                try {
                    gbnr::WalkConfig wcb = wc;
                    wcb.walkers = bs_walkers();
                    if (const char* e = std::getenv("GBNR_BS_STAGE_FRAC")) wcb.stage_frac = std::atof(e);
                    tws->wb = gbnr::build_backward_walk(sym, lay, wcb);
                } catch (...) {
                    e2 = std::current_exception();
                }
            });
            std::exception_ptr e0;
            try {
                tws->wf = gbnr::build_forward_walk(sym, lay, true, wc);
            } catch (...) {
                e0 = std::current_exception();
            }
            tl.join();
            tb.join();
            for (auto& e : {e0, e1, e2})
                if (e) std::rethrow_exception(e);
        };
        build();
        if (on_device) {
            CK(cudaSetDevice(opt.device));
            while ((gbnr::walk_ctas_per_sm(tws->wf.smem_bytes(), 32 * tws->wf.walkers) < ctas_per_sm ||
                    gbnr::bs_ctas_per_sm(tws->wb.smem_bytes(), 32 * tws->wb.walkers) < ctas_per_sm) &&
                   wc.smem_budget > 65536) {
                wc.smem_budget -= 1024;
                build();
            }
            tws->vf = upload_walk(tws->wf, tw);
            if (!sub_plan) tws->vl = upload_walk(tws->wl, tw);
            tws->vb = upload_walk(tws->wb, tw);
            set_once_tapes(*tws);
            CK(cudaStreamSynchronize(stream));
        }
        walks.push_back(std::move(tws));
        return walks.back().get();
    }

    // L2 policy of the walk copies: the forward walks read each A-tape block once,
    // so those copies are evict-first (room for the LU columns they re-fetch and
    // the U rows the backward walk reads next).  Within the box noise so far
    // (profiles/r02z_l2_hints.log); GBNR_ONCE_TAPE_LU / _BS override (-1: none).
    static void set_once_tapes(TileWalks& t) {
        t.vf.once_tape = t.vl.once_tape = gbnr::kTapeA;
        t.vb.once_tape = -1;
        if (const char* e = std::getenv("GBNR_ONCE_TAPE_BS")) t.vb.once_tape = std::atoi(e);
        if (const char* e = std::getenv("GBNR_ONCE_TAPE_LU")) t.vf.once_tape = t.vl.once_tape = std::atoi(e);
    }

    // A copy of another device plan's walks (same programs), uploaded here.
    void adopt_walks(const TileWalks& src) {
        auto tws = std::make_unique<TileWalks>();
        tws->tw = src.tw;
        tws->wf = src.wf;
        tws->wl = src.wl;
        tws->wb = src.wb;
        CK(cudaSetDevice(opt.device));
        tws->vf = upload_walk(tws->wf, src.tw);
        if (!sub_plan) tws->vl = upload_walk(tws->wl, src.tw);
        tws->vb = upload_walk(tws->wb, src.tw);
        set_once_tapes(*tws);
        CK(cudaStreamSynchronize(stream));
        walks.push_back(std::move(tws));
    }

    // Tile width of a batch of T tasks.  The LU walk's time is its busiest SM's:
    // the number of tiles that SM hosts and the shared-memory rows each walker
    // gets.  32 lanes while every SM hosts at most two full-width tiles (or the
    // batch needs three anyway); in between, 24 lanes put at most three tiles on
    // every SM -- the busiest SM hosts no more tiles than with 32 lanes, and every
    // walker gets a third more rows (profiles/r02h_tile_width.log: LU walk -7% at
    // 10k tasks).  gbnr_options.tile_width / GBNR_TW override.
    int32_t choose_tw(int32_t T) const {
        int32_t tw = opt.tile_width;
        if (const char* e = std::getenv("GBNR_TW")) tw = std::atoi(e);
        if (tw > 0) return std::min(gbnr::kTile, std::max(2, tw + (tw & 1)));
        const int64_t sm = n_sm;
        if (int64_t(T) > sm * 2 * gbnr::kTile && int64_t(T) <= sm * ctas_per_sm * 24 && ctas_per_sm >= 3) return 24;
        return gbnr::kTile;
    }

    // the plan's shared Ybus value set (one for every task)
    const double *y_shared_re = nullptr, *y_shared_im = nullptr;
    // per-task value sets (N-1 contingencies), [nnzY][n_tasks] as the caller lays them out
    double *y_task_re = nullptr, *y_task_im = nullptr;
    size_t y_task_cap = 0;

    void set_ybus(const double* re, const double* im) {
        y_host_re.assign(re, re + sym.nnzY);
        y_host_im.assign(im, im + sym.nnzY);
        v.yre = y_shared_re = dev_upload_s(y_host_re);
        v.yim = y_shared_im = dev_upload_s(y_host_im);
        v.y_ld = 1;
        v.y_inc = 0;
    }

    // Ybus values for the next solve: NULL = the plan's shared set; otherwise the
    // caller's set(s) are staged into a per-call buffer (one shared set, y_inc = 0,
    // or one per task, [nnzY][n_tasks]) and the plan's own set is never touched.
    // ld_y > 0: per-task sets, columns [0, n_tasks) of a host array [nnzY][ld_y]
    // (a slice of a larger batch; the caller offsets the pointers)
    void stage_ybus(const double* y_re, const double* y_im, int32_t n_ysets, int32_t n_tasks, int64_t ld_y = 0) {
        if (ld_y > 0 && y_re && y_im) {
            const size_t bytes = size_t(sym.nnzY) * size_t(n_tasks) * 8;
            ensure_ytask(bytes);
            for (auto [dst, src] : {std::pair{y_task_re, y_re}, {y_task_im, y_im}})
                CK(cudaMemcpy2DAsync(dst, size_t(n_tasks) * 8, src, size_t(ld_y) * 8, size_t(n_tasks) * 8,
                                     size_t(sym.nnzY), cudaMemcpyHostToDevice, stream));
            v.yre = y_task_re;
            v.yim = y_task_im;
            v.y_ld = n_tasks;
            v.y_inc = 1;
            return;
        }
        if (!y_re || !y_im) {
            if (n_ysets != 1) throw Error(GBNR_ECONFIG, "per-task Ybus sets need y_re and y_im");
            v.yre = y_shared_re;
            v.yim = y_shared_im;
            v.y_ld = 1;
            v.y_inc = 0;
            return;
        }
        const bool shared = n_ysets == 1 || n_tasks == 1;
        if (!shared && n_ysets != n_tasks) throw Error(GBNR_ECONFIG, "n_ysets must be 1 or n_tasks");
        const size_t sets = shared ? 1 : size_t(n_tasks);
        const size_t bytes = size_t(sym.nnzY) * sets * 8;
        ensure_ytask(bytes);
        CK(cudaMemcpyAsync(y_task_re, y_re, bytes, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(y_task_im, y_im, bytes, cudaMemcpyHostToDevice, stream));
        v.yre = y_task_re;
        v.yim = y_task_im;
        v.y_ld = shared ? 1 : n_tasks;
        v.y_inc = shared ? 0 : 1;
    }

    void ensure_ytask(size_t bytes) {
        if (bytes <= y_task_cap) return;
        CK(cudaStreamSynchronize(stream));
        dfree(y_task_re);
        dfree(y_task_im);
        y_task_re = y_task_im = nullptr;
        y_task_cap = 0;
        y_task_re = static_cast<double*>(dmalloc(bytes));
        y_task_im = static_cast<double*>(dmalloc(bytes));
        CK(cudaStreamSynchronize(stream));
        y_task_cap = bytes;
    }

    // Device bytes one task of a solve needs: its lane of the A / LU / b blocks, of
    // the [n][bpad] voltage / injection tapes, per-task state, walk scratch, and its
    // Ybus set when the batch has per-task sets.
    size_t bytes_per_task(bool per_task_y) const {
        int32_t scr = 0;
        for (const auto& w : walks) scr = std::max({scr, w->wf.scratch_rows, w->wl.scratch_rows});
        size_t b = (2 * size_t(lay.rows) + size_t(sym.nJ)) * 8 + 8 * size_t(sym.n) * 8 + 64 + size_t(8) * scr * 8;
        if (per_task_y) b += 2 * size_t(sym.nnzY) * 8;
        return b;
    }

    // Tasks one launch of this plan can hold: gbnr_options.chunk_tasks, else what
    // the free device memory (plus what this plan already holds) allows, keeping a
    // reserve for the second-chance re-plans and the driver.
    int32_t chunk_capacity(bool per_task_y) {
        if (opt.chunk_tasks > 0) return opt.chunk_tasks;
        CK(cudaSetDevice(opt.device));
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const size_t held = batch_bytes + pipe_bytes + y_task_cap;
        const size_t reserve = (size_t(4) << 30) + total_b / 50;
        const size_t avail = free_b + held > reserve ? free_b + held - reserve : 0;
        const size_t tasks = avail / bytes_per_task(per_task_y) / gbnr::kTile * gbnr::kTile;
        return int32_t(std::max<size_t>(gbnr::kTile, std::min<size_t>(tasks, size_t(1) << 30)));
    }

    // Device tapes for `lanes` = n_tiles x tile width task slots.  Every buffer is
    // sized by lanes, so one allocation serves any tile width; the tile geometry
    // (tstride, the LU / b offsets) is set per batch by set_geometry.
    void ensure_capacity(size_t lanes, int32_t scratch_rows) {
        if (lanes <= cap_lanes && scratch_rows <= cap_scratch) return;
        CK(cudaStreamSynchronize(stream));
        for (void* p : batch) dfree(p);
        batch.clear();
        lanes = std::max(lanes, cap_lanes);
        scratch_rows = std::max(scratch_rows, cap_scratch);
        batch_bytes = 0;
        auto alloc = [&](size_t bytes) {
            void* p = dmalloc(bytes);
            batch.push_back(p);
            batch_bytes += bytes;
            return p;
        };
        const size_t nb = size_t(sym.n) * lanes * sizeof(double);
        v.vm = static_cast<double*>(alloc(nb));
        v.va = static_cast<double*>(alloc(nb));
        v.vm_in = static_cast<double*>(alloc(nb));
        v.va_in = static_cast<double*>(alloc(nb));
        v.c = static_cast<double*>(alloc(nb));
        v.s = static_cast<double*>(alloc(nb));
        // the plan's own injection tapes; the batch pipeline points v.p0 / v.q0 at
        // its input sets for the duration of gbnr_solve_batches only
        v.p0 = p0_own = static_cast<double*>(alloc(nb));
        v.q0 = q0_own = static_cast<double*>(alloc(nb));
        // one block per tile: A, LU and b rows adjacent, so a walk copy's source is
        // tile base + (tape * tape_rows + slot) rows
        a_bytes = (2 * size_t(v.tape_rows) + size_t(v.nJ)) * lanes * sizeof(double);
        v.A = static_cast<double*>(alloc(a_bytes));
        // fill slots of the A tape are never written by the Jacobian kernel and
        // must read zero (re-zeroed when the tile width changes, set_geometry)
        CK(cudaMemsetAsync(v.A, 0, a_bytes, stream));
        a_tw = 0;
        v.status = static_cast<int32_t*>(alloc(lanes * sizeof(int32_t)));
        v.iters = static_cast<int32_t*>(alloc(lanes * sizeof(int32_t)));
        v.active = static_cast<uint8_t*>(alloc(lanes));
        v.flag = static_cast<uint8_t*>(alloc(lanes));
        v.maxmis = static_cast<double*>(alloc(lanes * sizeof(double)));
        v.mis_prev = static_cast<double*>(alloc(lanes * sizeof(double)));
        v.mis0 = static_cast<double*>(alloc(lanes * sizeof(double)));
        v.jskip = static_cast<uint8_t*>(alloc(lanes));
        v.norm_bits = static_cast<unsigned long long*>(alloc(lanes * sizeof(unsigned long long)));
        v.tile_active = static_cast<int32_t*>(alloc(lanes * sizeof(int32_t)));  // >= tiles at any width
        // global scratch of the forward walks' global steps (columns too large for
        // a walker's shared-memory pool), 8 walkers per tile
        v.scratch = scratch_rows > 0 ? static_cast<double*>(alloc(lanes * gbnr::kLuWarps * size_t(scratch_rows) * 8))
                                     : nullptr;
        v.active_count = static_cast<int32_t*>(alloc(128 * sizeof(int32_t)));
        cap_lanes = lanes;
        cap_scratch = scratch_rows;
        CK(cudaStreamSynchronize(stream));  // stream-ordered allocations ready for every stream
    }

    // Tile geometry of a batch of n_tasks tasks at tile width tw (its walks current).
    void set_geometry(int32_t n_tasks, int32_t tw) {
        cur = walks_for(tw);
        const int32_t n_tiles = (n_tasks + tw - 1) / tw;
        const int32_t scr = std::max(cur->wf.scratch_rows, cur->wl.scratch_rows);
        ensure_capacity(size_t(n_tiles) * tw, scr);
        if (a_tw != 0 && a_tw != tw) CK(cudaMemsetAsync(v.A, 0, a_bytes, stream));  // J slots move with tw
        a_tw = tw;
        v.tw = tw;
        v.n_tiles = n_tiles;
        v.bpad = n_tiles * tw;
        v.n_tasks = n_tasks;
        v.tstride = (2 * size_t(v.tape_rows) + size_t(v.nJ)) * size_t(tw);
        v.LU = v.A + size_t(v.tape_rows) * tw;
        v.b = v.LU + size_t(v.tape_rows) * tw;
        v.scratch_rows = scr;
    }

    // Element-major host [n][sets] -> device [n][bpad] (broadcast when sets == 1).
    void put_tape(double* dst, const double* src, int32_t sets, int32_t n_tasks) {
        const size_t bpad = size_t(v.bpad);
        if (sets == n_tasks && n_tasks > 1) {
            CK(cudaMemcpy2DAsync(dst, bpad * sizeof(double), src, size_t(n_tasks) * sizeof(double),
                                 size_t(n_tasks) * sizeof(double), sym.n, cudaMemcpyHostToDevice,
                                 stream));
        } else {
            CK(cudaMemcpyAsync(d_scratch, src, size_t(sym.n) * sizeof(double), cudaMemcpyHostToDevice,
                               stream));
            gbnr::launch_broadcast(dst, d_scratch, sym.n, int32_t(bpad), stream);
            CK(cudaGetLastError());
        }
    }

    // ld_s / ld_v > 0: the injections / start voltages are per task, columns
    // [0, n_tasks) of host arrays [n][ld] (a slice of a larger batch; the caller
    // offsets the pointers; n_ssets / n_vsets are then ignored)
    void stage(int32_t n_tasks, const double* p0, const double* q0, int32_t n_ssets,
               const double* vm0, const double* va0, int32_t n_vsets, int64_t ld_s = 0, int64_t ld_v = 0) {
        if (!on_device) throw Error(GBNR_ECONFIG, "host-only plan (device = -1) cannot solve");
        if (n_tasks <= 0) throw Error(GBNR_ECONFIG, "n_tasks must be positive");
        if (ld_s > 0) n_ssets = n_tasks;
        if (ld_v > 0) n_vsets = n_tasks;
        if ((n_ssets != 0 && n_ssets != 1 && n_ssets != n_tasks) || (n_vsets != 1 && n_vsets != n_tasks))
            throw Error(GBNR_ECONFIG, "set counts must be 1 or n_tasks");
        // host [n][ld] columns [0, n_tasks) -> device [n][n_tasks], one linear copy when unsliced
        auto h2d_cols = [&](const double* dst, const double* src, int64_t ld) {
            const size_t w = size_t(n_tasks) * 8;
            if (ld <= 0 || ld == n_tasks)
                CK(cudaMemcpyAsync(const_cast<double*>(dst), src, size_t(sym.n) * w, cudaMemcpyHostToDevice, stream));
            else
                CK(cudaMemcpy2DAsync(const_cast<double*>(dst), w, src, size_t(ld) * 8, w, size_t(sym.n),
                                     cudaMemcpyHostToDevice, stream));
        };
        CK(cudaSetDevice(opt.device));
        set_geometry(n_tasks, choose_tw(n_tasks));
        // start voltages as given: [n] shared or [n][n_tasks], one linear copy each
        // (init_kernel reads them through vin_ld / vin_inc)
        const bool vshared = n_vsets == 1 && ld_v <= 0;
        if (vshared) {
            const size_t vbytes = size_t(sym.n) * sizeof(double);
            CK(cudaMemcpyAsync(const_cast<double*>(v.vm_in), vm0, vbytes, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(const_cast<double*>(v.va_in), va0, vbytes, cudaMemcpyHostToDevice, stream));
        } else {
            h2d_cols(v.vm_in, vm0, ld_v);
            h2d_cols(v.va_in, va0, ld_v);
        }
        v.vin_ld = vshared ? 1 : n_tasks;
        v.vin_inc = vshared ? 0 : 1;
        if (n_ssets != 0) {
            v.p0 = p0_own;
            v.q0 = q0_own;
        }
        if (n_ssets == 0) {
            // injections are placed by the caller (batch pipeline)
        } else if (ld_s > 0) {
            h2d_cols(v.p0, p0, ld_s);
            h2d_cols(v.q0, q0, ld_s);
            v.s_ld = n_tasks;
            v.s_inc = 1;
        } else if (n_ssets == 1 && n_tasks > 1) {
            CK(cudaMemcpyAsync(const_cast<double*>(v.p0), p0, size_t(sym.n) * sizeof(double),
                               cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(const_cast<double*>(v.q0), q0, size_t(sym.n) * sizeof(double),
                               cudaMemcpyHostToDevice, stream));
            v.s_ld = 1;
            v.s_inc = 0;
        } else if (n_ssets == n_tasks && n_tasks > 1) {
            // the host layout [n][n_tasks] as is: one linear copy per array (a
            // pitched copy into [n][bpad] runs the DMA engines row by row)
            const size_t bytes = size_t(sym.n) * size_t(n_tasks) * sizeof(double);
            CK(cudaMemcpyAsync(const_cast<double*>(v.p0), p0, bytes, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(const_cast<double*>(v.q0), q0, bytes, cudaMemcpyHostToDevice, stream));
            v.s_ld = n_tasks;
            v.s_inc = 1;
        } else {
            put_tape(const_cast<double*>(v.p0), p0, n_ssets, n_tasks);
            put_tape(const_cast<double*>(v.q0), q0, n_ssets, n_tasks);
            v.s_ld = v.bpad;
            v.s_inc = 1;
        }
        staged = true;
        whole_on_device = true;
    }

    void timed(int phase, const std::function<void()>& launch) {
        if (!opt.profile) {
            launch();
            return;
        }
        const size_t k = 2 * ev_used.size();
        while (ev_pool.size() < k + 2) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        CK(cudaEventRecord(ev_pool[k], stream));
        launch();
        CK(cudaEventRecord(ev_pool[k + 1], stream));
        ev_used.emplace_back(phase, int(k));
    }

    void resolve_profile() {
        for (const auto& [phase, k] : ev_used) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev_pool[k], ev_pool[k + 1]));
            timing[phase] += ms;
            timing[6 + phase] += 1.0;
        }
        ev_used.clear();
    }

    // LU refactorization fused with the forward substitution, then the
    // backward substitution: one launch each (tile walks, walk.hpp)
    void launch_lu_all() { gbnr::launch_lu_walk(v, cur->vf, true, stream); }
    void launch_fsbs_all() { gbnr::launch_bs_walk(v, cur->vb, stream); }

    static int launches_per_iteration() { return 6; }  // lu+fs, bs, vupd, npm+jac, conv, bump

    // One batched Newton solve of the staged tasks.  finish: also the second chance
    // of flagged tasks (and, inside gbnr_solve, the re-derivation decision);
    // solve_general finishes chunks itself.
    void run(bool finish = true) {
        if (!staged) throw Error(GBNR_ECONFIG, "gbnr_run before gbnr_stage");
        CK(cudaSetDevice(opt.device));
        std::memset(timing, 0, sizeof timing);
        ev_used.clear();
        CK(cudaEventRecord(ev0, stream));
        CK(cudaMemsetAsync(v.active_count, 0, 128 * sizeof(int32_t), stream));
        gbnr::launch_init(v, stream);
        CK(cudaGetLastError());
        timed(kNpm, [&] { gbnr::launch_npm(v, opt.max_iter > 0, stream); });
        int it_done = 0, jac_fix = 0;
        for (int it = 1; it <= opt.max_iter; ++it) {
            CK(cudaStreamSynchronize(stream));  // the bump kernel published active_count[it-1]
            const volatile int32_t* hc = h_count;
            if (hc[it - 1] == 0) break;
            if (hc[96 + it - 1] > 0) {  // mispredicted convergence: those tasks' Jacobian
                timed(kJac, [&] { gbnr::launch_jacobian(v, false, stream); });
                ++jac_fix;
            }
            timed(kLu, [&] { launch_lu_all(); });
            timed(kFsbs, [&] { launch_fsbs_all(); });
            timed(kVupd, [&] { gbnr::launch_vupdate(v, stream); });
            timed(kNpm, [&] { gbnr::launch_npm(v, it < opt.max_iter, stream); });
            CK(cudaGetLastError());
            it_done = it;
        }
        CK(cudaEventRecord(ev1, stream));
        gbnr::launch_status_count(v, stream);
        CK(cudaStreamSynchronize(stream));
        double tiles = 0, tasks = 0;
        for (int it = 1; it <= it_done; ++it) {
            tiles += h_count[32 + it - 1];
            tasks += h_count[it - 1];
        }
        timing[14] = tiles;
        timing[15] = tasks;
        first_flagged = h_count[66] > 0 ? flagged_at_first_solve() : 0;
        if (finish && opt.second_chance && h_count[66] > 0) second_chance();
        count_statuses();
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev0, ev1));
        resolve_profile();
        timing[5] = ms;
        timing[12] = it_done;
        timing[13] = v.n_tasks;
        timing[19] = double(launches_per_iteration()) * it_done + 4 + jac_fix;  // kernels launched
        solved = true;
    }

    // second_chance_refactorize (open question :436): a task
    // whose frozen pivot collapsed (status singular after `it` linear solves) is
    // re-planned alone -- a fresh threshold-pivoting factorization at its current
    // voltages, kept for the rest of its Newton loop -- and continues on the GPU
    // with the remaining budget max_iter - (it - 1).  Its results replace the
    // task's column of the batch state; status GBNR_FALLBACK_CONVERGED if it
    // converges, else the re-run's status.  A fresh factorization that is itself
    // singular leaves the task singular.  Host orchestration only: the re-run uses
    // the same kernels (oracle/pyoracle.py OraclePlan._second_chance is the checker).
    int32_t first_flagged = 0;  // tasks of the last run flagged at their first linear solve

    // converged (incl. second chance), diverged, singular; [20] the second-chance subset
    void count_statuses() {
        timing[16] = h_count[64] + h_count[67];
        timing[17] = h_count[65];
        timing[18] = h_count[66];
        timing[20] = h_count[67];
    }

    int32_t flagged_at_first_solve() {
        const int32_t nt = v.n_tasks;
        std::vector<int32_t> st(nt), it(nt);
        CK(cudaMemcpyAsync(st.data(), v.status, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(it.data(), v.iters, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        int32_t c = 0;
        for (int32_t t = 0; t < nt; ++t) c += st[t] == GBNR_SINGULAR && it[t] == 1;
        return c;
    }

    // ---- second chance -------------------------------
    // Every flagged task gets a fresh threshold-pivoting factorization at its
    // current voltages and continues on this GPU with its remaining budget
    // max_iter - (it - 1).  A re-plan is a host symbolic analysis plus walk plans
    // (about 0.3 s at synth9241), so: first one fresh plan from the flagged task
    // with the largest mismatch at its failure (its own voltages and Ybus values;
    // first of the largest) solves every flagged task in one batch -- flags that
    // share a cause are done after one re-plan; the tasks its pivots do not carry
    // (they collapse again) then each get their own fresh plan, concurrently.
    // Status 3 on convergence, else the re-run's status; a task whose own fresh
    // factorization is singular stays singular (oracle/pyoracle.py
    // OraclePlan._second_chance restates the same rule).
    struct Chance {
        int32_t t = 0, it = 0;
        std::vector<double> vm, va, yr, yi, pp, qq;  // the task's state at the failure
        double mm_fail = 0.0;
        bool done = false, ran = false;
        int32_t status = GBNR_SINGULAR, iters = 0;
        double mm = 0.0;
        std::vector<double> vm_out, va_out;
    };

    // options of a second-chance plan: one chance, one device
    gbnr_options chance_options() const {
        gbnr_options o = opt;
        o.second_chance = 0;
        o.profile = 0;
        o.n_devices = 1;
        o.chunk_tasks = 0;
        return o;
    }

    // Solve the chances `grp` (budget b) through the fresh plan `sp` in one batch; a
    // task that does not collapse again -- or the plan's own representative `self`,
    // whatever becomes of it -- takes the re-run's results.
    void run_chances(gbnr_plan& sp, std::vector<Chance>& work, const std::vector<int32_t>& grp, int32_t b,
                     bool per_y, int32_t self) {
        const int32_t n = sym.n, nY = sym.nnzY, m = int32_t(grp.size());
        std::vector<double> P(size_t(n) * m), Q(P.size()), VM(P.size()), VA(P.size());
        std::vector<double> YR(per_y ? size_t(nY) * m : 0), YI(YR.size());
        for (int32_t j = 0; j < m; ++j) {
            const Chance& c = work[grp[j]];
            for (int32_t q = 0; q < n; ++q) {
                P[size_t(q) * m + j] = c.pp[q];
                Q[size_t(q) * m + j] = c.qq[q];
                VM[size_t(q) * m + j] = c.vm[q];
                VA[size_t(q) * m + j] = c.va[q];
            }
            if (per_y)
                for (int32_t q = 0; q < nY; ++q) {
                    YR[size_t(q) * m + j] = c.yr[q];
                    YI[size_t(q) * m + j] = c.yi[q];
                }
        }
        std::vector<double> ovm(P.size()), ova(P.size()), omm(m);
        std::vector<int32_t> oit(m), ost(m);
        sp.opt.max_iter = b;
        sp.v.max_iter = b;
        const SolveIn in{m, per_y ? YR.data() : nullptr, per_y ? YI.data() : nullptr, per_y ? m : 1,
                         P.data(), Q.data(), m, VM.data(), VA.data(), m};
        const SolveOut out{ovm.data(), ova.data(), oit.data(), nullptr, ost.data(), omm.data()};
        sp.solve_general(in, out, false);
        for (int32_t j = 0; j < m; ++j) {
            Chance& c = work[grp[j]];
            if (ost[j] == GBNR_SINGULAR && grp[j] != self) continue;  // not carried: its own plan next
            c.done = c.ran = true;
            c.status = ost[j] == GBNR_CONVERGED ? GBNR_FALLBACK_CONVERGED : ost[j];
            c.iters = c.it - 1 + oit[j];
            c.mm = omm[j];
            c.vm_out.resize(n);
            c.va_out.resize(n);
            for (int32_t q = 0; q < n; ++q) {
                c.vm_out[q] = ovm[size_t(q) * m + j];
                c.va_out[q] = ova[size_t(q) * m + j];
            }
        }
    }

    void second_chance() {
        CK(cudaSetDevice(opt.device));
        const int32_t nt = v.n_tasks, n = sym.n, nY = sym.nnzY;
        std::vector<int32_t> st(nt), it(nt);
        std::vector<double> mmf(nt);
        CK(cudaMemcpyAsync(st.data(), v.status, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(it.data(), v.iters, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(mmf.data(), v.maxmis, size_t(nt) * 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        std::vector<Chance> work;
        const size_t bp = size_t(v.bpad);
        auto column = [&](std::vector<double>& dst, const double* src, size_t pitch, int32_t rows) {
            dst.resize(size_t(rows));
            CK(cudaMemcpy2DAsync(dst.data(), 8, src, pitch * 8, 8, size_t(rows), cudaMemcpyDeviceToHost, stream));
        };
        for (int32_t t = 0; t < nt; ++t) {
            if (st[t] != GBNR_SINGULAR || opt.max_iter - (it[t] - 1) < 1) continue;
            Chance c;
            c.t = t;
            c.it = it[t];
            c.mm_fail = mmf[t];
            column(c.vm, v.vm + t, bp, n);
            column(c.va, v.va + t, bp, n);
            column(c.yr, v.yre + size_t(t) * v.y_inc, size_t(v.y_ld), nY);
            column(c.yi, v.yim + size_t(t) * v.y_inc, size_t(v.y_ld), nY);
            column(c.pp, v.p0 + size_t(t) * v.s_inc, size_t(v.s_ld), n);
            column(c.qq, v.q0 + size_t(t) * v.s_inc, size_t(v.s_ld), n);
            work.push_back(std::move(c));
        }
        CK(cudaStreamSynchronize(stream));
        if (work.empty()) return;
        const bool per_y = v.y_inc != 0;
        // round 1: the representative's fresh plan for every flagged task, in one batch
        // per remaining budget
        int32_t w = 0;  // largest mismatch at failure, first of the largest
        for (int32_t i = 1; i < int32_t(work.size()); ++i)
            if (work[i].mm_fail > work[w].mm_fail) w = i;
        gbnr_plan* sub = nullptr;
        const gbnr_options co = chance_options();
        {
            const Chance& rep = work[w];
            const int rc = create_plan(n, sym.yp.data(), sym.yi.data(), rep.yr.data(), rep.yi.data(), sym.ref,
                                       in_pv.data(), int32_t(in_pv.size()), in_pq.data(), int32_t(in_pq.size()),
                                       rep.vm.data(), rep.va.data(), &co, &sub, true);
            if (rc == GBNR_ESINGULAR) {
                work[w].done = true;  // no fresh factorization: the representative stays failed
                sub = nullptr;
            } else if (rc != GBNR_OK) {
                throw Error(rc, std::string("second chance: ") + gbnr_last_error());
            }
        }
        if (sub) {
            std::unique_ptr<gbnr_plan, void (*)(gbnr_plan*)> guard(sub, gbnr_plan_destroy);
            std::vector<int32_t> budgets;
            for (const Chance& c : work) budgets.push_back(opt.max_iter - (c.it - 1));
            std::sort(budgets.begin(), budgets.end());
            budgets.erase(std::unique(budgets.begin(), budgets.end()), budgets.end());
            for (int32_t b : budgets) {
                std::vector<int32_t> grp;
                for (int32_t i = 0; i < int32_t(work.size()); ++i)
                    if (opt.max_iter - (work[i].it - 1) == b) grp.push_back(i);
                run_chances(*sub, work, grp, b, per_y, w);
            }
            work[w].done = true;
        }
        // the tasks the representative's pivots did not carry: each its own fresh
        // plan, concurrently (host threads, one plan and stream each)
        std::vector<int32_t> rest;
        for (int32_t i = 0; i < int32_t(work.size()); ++i)
            if (!work[i].done) rest.push_back(i);
        if (!rest.empty()) {
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            const size_t per_plan = bytes_per_task(false) * gbnr::kTile + (size_t(64) << 20);
            const size_t by_mem = free_b > (size_t(1) << 30) ? (free_b - (size_t(1) << 30)) / per_plan : 1;
            const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
            const size_t W = std::max<size_t>(1, std::min({rest.size(), size_t(std::min(hw, 16u)), by_mem}));
            std::atomic<size_t> next{0};
            std::vector<std::exception_ptr> errs(W);
            auto worker = [&](size_t wk) {
                try {
                    for (size_t j; (j = next.fetch_add(1)) < rest.size();) {
                        Chance& c = work[rest[j]];
                        gbnr_plan* own = nullptr;
                        const int rc = create_plan(n, sym.yp.data(), sym.yi.data(), c.yr.data(), c.yi.data(),
                                                   sym.ref, in_pv.data(), int32_t(in_pv.size()), in_pq.data(),
                                                   int32_t(in_pq.size()), c.vm.data(), c.va.data(),
                                                   &co, &own, true);
                        if (rc == GBNR_ESINGULAR) continue;  // the task stays failed
                        if (rc != GBNR_OK) throw Error(rc, std::string("second chance: ") + gbnr_last_error());
                        std::unique_ptr<gbnr_plan, void (*)(gbnr_plan*)> g(own, gbnr_plan_destroy);
                        run_chances(*own, work, {rest[j]}, opt.max_iter - (c.it - 1), per_y, rest[j]);
                    }
                } catch (...) {
                    errs[wk] = std::current_exception();
                    next = rest.size();
                }
            };
            std::vector<std::thread> pool;
            for (size_t wk = 1; wk < W; ++wk) pool.emplace_back(worker, wk);
            worker(0);
            for (auto& th : pool) th.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        }
        // results -> this batch's device state (statuses, iterations, mismatch, V)
        CK(cudaSetDevice(opt.device));
        for (const Chance& c : work) {
            if (!c.ran) continue;
            const int32_t t = c.t;
            CK(cudaMemcpy(v.status + t, &c.status, 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(v.iters + t, &c.iters, 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(v.maxmis + t, &c.mm, 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy2D(v.vm + t, bp * 8, c.vm_out.data(), 8, 8, size_t(n), cudaMemcpyHostToDevice));
            CK(cudaMemcpy2D(v.va + t, bp * 8, c.va_out.data(), 8, 8, size_t(n), cudaMemcpyHostToDevice));
        }
        gbnr::launch_status_count(v, stream);
        CK(cudaStreamSynchronize(stream));
    }

    // ---- gbnr_solve: shards over devices, chunks, re-derivation ----------------
    struct SolveIn {
        int32_t n_tasks;
        const double *y_re, *y_im;
        int32_t n_ysets;
        const double *p0, *q0;
        int32_t n_ssets;
        const double *vm0, *va0;
        int32_t n_vsets;
    };
    struct SolveOut {
        double *vm, *va;
        int32_t* it;
        uint8_t* conv;
        int32_t* st;
        double* mm;
    };

    // timing of one run -> a running total ([5] total device ms and counts add up,
    // [12] Newton iterations is the maximum)
    static void add_timing(double* acc, const double* t) {
        for (int i = 0; i < 24; ++i) acc[i] = i == 12 ? std::max(acc[i], t[i]) : acc[i] + t[i];
    }

    // Tasks [t0, t0 + T) of `in` on this device plan, in chunks of at most
    // chunk_capacity() tasks; results into the same columns of `out`; per-task
    // mismatch at V0 into mis0 and the count of tasks flagged at their first
    // linear solve (the re-derivation rule) into *first.
    void solve_slice(const SolveIn& in, const SolveOut& out, int32_t t0, int32_t T, double* mis0, int64_t* first,
                     double* acc) {
        CK(cudaSetDevice(opt.device));
        const int64_t N = in.n_tasks;
        const bool per_y = in.y_re && in.n_ysets > 1, per_s = in.n_ssets > 1, per_v = in.n_vsets > 1;
        const int32_t cap = chunk_capacity(per_y);
        const int32_t nch = (T + cap - 1) / cap;
        const bool sliced = T != N || nch > 1;
        for (int32_t ch = 0; ch < nch; ++ch) {
            const int32_t a = t0 + int32_t(int64_t(T) * ch / nch), b = t0 + int32_t(int64_t(T) * (ch + 1) / nch);
            const int32_t m = b - a;
            if (sliced) {
                stage_ybus(per_y ? in.y_re + a : in.y_re, per_y ? in.y_im + a : in.y_im, per_y ? m : 1, m,
                           per_y ? N : 0);
                stage(m, per_s ? in.p0 + a : in.p0, per_s ? in.q0 + a : in.q0, 1, per_v ? in.vm0 + a : in.vm0,
                      per_v ? in.va0 + a : in.va0, 1, per_s ? N : 0, per_v ? N : 0);
            } else {
                stage_ybus(in.y_re, in.y_im, in.n_ysets, m);
                stage(m, in.p0, in.q0, in.n_ssets, in.vm0, in.va0, in.n_vsets);
            }
            run(false);
            *first += first_flagged;
            CK(cudaMemcpy(mis0 + a, v.mis0, size_t(m) * 8, cudaMemcpyDeviceToHost));
            if (opt.second_chance && h_count[66] > 0) second_chance();
            count_statuses();
            add_timing(acc, timing);
            auto at = [&](auto* p) { return p ? p + a : p; };
            fetch(at(out.vm), at(out.va), at(out.it), at(out.conv), at(out.st), at(out.mm), sliced ? N : 0);
        }
        whole_on_device = !sliced;
    }

    void solve_general(const SolveIn& in, const SolveOut& out, bool allow_rd) {
        const int32_t N = in.n_tasks;
        if (N <= 0) throw Error(GBNR_ECONFIG, "n_tasks must be positive");
        if ((in.n_ssets != 1 && in.n_ssets != N) || (in.n_vsets != 1 && in.n_vsets != N))
            throw Error(GBNR_ECONFIG, "set counts must be 1 or n_tasks");
        if (in.y_re && in.y_im && in.n_ysets != 1 && in.n_ysets != N)
            throw Error(GBNR_ECONFIG, "n_ysets must be 1 or n_tasks");
        if ((!in.y_re || !in.y_im) && in.n_ysets != 1) throw Error(GBNR_ECONFIG, "per-task Ybus sets need y_re and y_im");
        std::vector<gbnr_plan*> dev{this};
        for (auto& q : peers) dev.push_back(q.get());
        const size_t D = dev.size();
        std::vector<double> mis0(size_t(N), 0.0);
        std::vector<int64_t> first(D, 0);
        std::vector<std::array<double, 24>> acc(D);
        std::vector<std::exception_ptr> errs(D);
        auto shard = [&](size_t d) {
            try {
                acc[d].fill(0.0);
                const int32_t a = int32_t(int64_t(N) * int64_t(d) / int64_t(D));
                const int32_t b = int32_t(int64_t(N) * int64_t(d + 1) / int64_t(D));
                if (b > a) dev[d]->solve_slice(in, out, a, b - a, mis0.data(), &first[d], acc[d].data());
            } catch (...) {
                errs[d] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (size_t d = 1; d < D; ++d) th.emplace_back(shard, d);
        shard(0);
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        // shards ran concurrently: the job's device time is the slowest shard's
        double agg[24] = {0};
        for (size_t d = 0; d < D; ++d) {
            const double ms = agg[5];
            add_timing(agg, acc[d].data());
            agg[5] = std::max(ms, acc[d][5]);
        }
        agg[13] = N;
        std::memcpy(timing, agg, sizeof timing);
        if (D > 1) whole_on_device = false;
        int64_t ff = 0;
        for (int64_t f : first) ff += f;
        if (allow_rd && opt.second_chance && ff * 20 > N) rederive(in, out, mis0);
    }

    // Representative re-derivation (SPEC.md DESIGN DECISIONS): the frozen pivot
    // order failed for more than 5% of the tasks at their first solve -> solve the
    // batch again, once, from a plan whose pivots come from the task with the worst
    // mismatch at V0 (its V0 and Ybus values).  A representative that is itself
    // singular keeps the first results (their second chances are done).
    void rederive(const SolveIn& in, const SolveOut& out, const std::vector<double>& mis0) {
        const int32_t N = in.n_tasks, n = sym.n, nY = sym.nnzY;
        int32_t w = 0;
        for (int32_t t = 1; t < N; ++t)
            if (mis0[t] > mis0[w]) w = t;  // first of the largest
        std::vector<double> vm(n), va(n), yr(nY), yi(nY);
        const int32_t vw = in.n_vsets == 1 ? 0 : w;
        for (int32_t b = 0; b < n; ++b) {
            vm[b] = in.vm0[size_t(b) * in.n_vsets + vw];
            va[b] = in.va0[size_t(b) * in.n_vsets + vw];
        }
        if (in.y_re && in.y_im) {
            const int32_t yw = in.n_ysets == 1 ? 0 : w;
            for (int32_t q = 0; q < nY; ++q) {
                yr[q] = in.y_re[size_t(q) * in.n_ysets + yw];
                yi[q] = in.y_im[size_t(q) * in.n_ysets + yw];
            }
        } else {
            yr = y_host_re;
            yi = y_host_im;
        }
        gbnr_plan* alt = nullptr;
        const int rc = create_plan(n, sym.yp.data(), sym.yi.data(), yr.data(), yi.data(), sym.ref, in_pv.data(),
                                   int32_t(in_pv.size()), in_pq.data(), int32_t(in_pq.size()), vm.data(), va.data(),
                                   &opt, &alt, false);
        if (rc == GBNR_ESINGULAR) return;
        if (rc != GBNR_OK) throw Error(rc, std::string("re-derivation: ") + gbnr_last_error());
        std::unique_ptr<gbnr_plan, void (*)(gbnr_plan*)> guard(alt, gbnr_plan_destroy);
        alt->solve_general(in, out, false);
        std::memcpy(timing, alt->timing, sizeof timing);
        timing[21] = 1;  // restarted from a re-derived representative
        whole_on_device = false;
        if (alt->whole_on_device && peers.empty()) {
            // device state for gbnr_branch_flows: the restarted solve's voltages
            CK(cudaSetDevice(opt.device));
            const size_t nb = size_t(n) * size_t(v.bpad) * 8;
            for (auto [dst, src] : {std::pair{v.vm, alt->v.vm}, {v.va, alt->v.va}})
                CK(cudaMemcpy(dst, src, nb, cudaMemcpyDeviceToDevice));
            const size_t nt = size_t(v.n_tasks);
            CK(cudaMemcpy(v.status, alt->v.status, nt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(v.iters, alt->v.iters, nt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(v.maxmis, alt->v.maxmis, nt * 8, cudaMemcpyDeviceToDevice));
            whole_on_device = true;
        }
    }

    void ensure_pipe(size_t lanes) {
        if (lanes <= pipe_lanes) return;
        CK(cudaDeviceSynchronize());
        for (void* q : pipe) dfree(q);
        pipe.clear();
        const size_t nb = size_t(sym.n) * lanes * sizeof(double);
        const size_t tb = lanes;
        pipe_bytes = 0;
        auto alloc = [&](size_t bytes) {
            void* q = dmalloc(bytes);
            pipe.push_back(q);
            pipe_bytes += bytes;
            return q;
        };
        for (int i = 0; i < 2; ++i) {
            if (h_it[i]) cudaFreeHost(h_it[i]);
            if (h_st[i]) cudaFreeHost(h_st[i]);
            if (h_mm[i]) cudaFreeHost(h_mm[i]);
            CK(cudaMallocHost(&h_it[i], tb * sizeof(int32_t)));
            CK(cudaMallocHost(&h_st[i], tb * sizeof(int32_t)));
            CK(cudaMallocHost(&h_mm[i], tb * sizeof(double)));
            p0_set[i] = static_cast<double*>(alloc(nb));
            q0_set[i] = static_cast<double*>(alloc(nb));
            out_vm[i] = static_cast<double*>(alloc(nb));
            out_va[i] = static_cast<double*>(alloc(nb));
            out_mm[i] = static_cast<double*>(alloc(tb * sizeof(double)));
            out_it[i] = static_cast<int32_t*>(alloc(tb * sizeof(int32_t)));
            out_st[i] = static_cast<int32_t*>(alloc(tb * sizeof(int32_t)));
        }
        pipe_lanes = lanes;
        CK(cudaStreamSynchronize(stream));  // the copy streams use these buffers next
    }

    // Pipelined sequence of batches (all of n_tasks tasks, injections per task,
    // start voltages shared): H2D of batch i+1 (copy stream) and D2H of batch
    // i-1 (second copy stream) run while batch i solves.  Results per batch as
    // in gbnr_solve.
    void solve_batches(int32_t n_batches, int32_t n_tasks, const double* const* p0s, const double* const* q0s,
                       const double* vm0, const double* va0, double* const* vms, double* const* vas,
                       int32_t* const* its, uint8_t* const* convs, int32_t* const* sts, double* const* mms) {
        if (n_batches <= 0) return;
        // whatever happens, the plan's own injection tapes are the staged ones afterwards
        struct Restore {
            gbnr_plan* p;
            ~Restore() {
                p->v.p0 = p->p0_own;
                p->v.q0 = p->q0_own;
            }
        } restore{this};
        const size_t ntt = size_t(n_tasks);
        // batch j's small results: pinned staging -> the caller's arrays
        auto unstage_small = [&](int32_t j) {
            const int set = j & 1;
            CK(cudaEventSynchronize(ev_out[set]));
            if (its && its[j]) std::memcpy(its[j], h_it[set], ntt * 4);
            if (sts && sts[j]) std::memcpy(sts[j], h_st[set], ntt * 4);
            if (mms && mms[j]) std::memcpy(mms[j], h_mm[set], ntt * 8);
            if (convs && convs[j])
                for (size_t t = 0; t < ntt; ++t)
                    convs[j][t] = h_st[set][t] == GBNR_CONVERGED || h_st[set][t] == GBNR_FALLBACK_CONVERGED;
        };
        // geometry, the plan's Ybus and the shared start voltages (injections come per batch below)
        stage_ybus(nullptr, nullptr, 1, n_tasks);
        stage(n_tasks, nullptr, nullptr, 0, vm0, va0, 1);
        CK(cudaStreamSynchronize(stream));
        ensure_pipe(size_t(v.bpad));
        const size_t nt = size_t(n_tasks), row = nt * sizeof(double);
        const size_t bytes = size_t(sym.n) * row;  // host layout [n][n_tasks], copied linearly
        auto issue_h2d = [&](int32_t j) {
            const int set = j & 1;
            if (j >= 2) CK(cudaStreamWaitEvent(s_h2d, ev_free_in[set], 0));
            CK(cudaMemcpyAsync(p0_set[set], p0s[j], bytes, cudaMemcpyHostToDevice, s_h2d));
            CK(cudaMemcpyAsync(q0_set[set], q0s[j], bytes, cudaMemcpyHostToDevice, s_h2d));
            CK(cudaEventRecord(ev_in[set], s_h2d));
        };
        issue_h2d(0);
        for (int32_t i = 0; i < n_batches; ++i) {
            const int set = i & 1;
            if (i + 1 < n_batches) issue_h2d(i + 1);
            CK(cudaStreamWaitEvent(stream, ev_in[set], 0));
            v.p0 = p0_set[set];
            v.q0 = q0_set[set];
            v.s_ld = n_tasks;
            v.s_inc = 1;
            run();
            CK(cudaEventRecord(ev_free_in[set], stream));
            if (i >= 2) CK(cudaStreamWaitEvent(stream, ev_out[set], 0));
            // pack [n][bpad] -> [n][n_tasks] on the device so the D2H is one linear copy
            gbnr::launch_pack(out_vm[set], v.vm, sym.n, n_tasks, v.bpad, stream);
            gbnr::launch_pack(out_va[set], v.va, sym.n, n_tasks, v.bpad, stream);
            CK(cudaMemcpyAsync(out_it[set], v.iters, nt * 4, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(out_st[set], v.status, nt * 4, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(out_mm[set], v.maxmis, nt * 8, cudaMemcpyDeviceToDevice, stream));
            CK(cudaEventRecord(ev_res[set], stream));
            CK(cudaStreamWaitEvent(s_d2h, ev_res[set], 0));
            if (vms[i]) CK(cudaMemcpyAsync(vms[i], out_vm[set], bytes, cudaMemcpyDeviceToHost, s_d2h));
            if (vas[i]) CK(cudaMemcpyAsync(vas[i], out_va[set], bytes, cudaMemcpyDeviceToHost, s_d2h));
            if (i >= 2) unstage_small(i - 2);  // its pinned staging set is reused now
            CK(cudaMemcpyAsync(h_it[set], out_it[set], nt * 4, cudaMemcpyDeviceToHost, s_d2h));
            CK(cudaMemcpyAsync(h_st[set], out_st[set], nt * 4, cudaMemcpyDeviceToHost, s_d2h));
            CK(cudaMemcpyAsync(h_mm[set], out_mm[set], nt * 8, cudaMemcpyDeviceToHost, s_d2h));
            CK(cudaEventRecord(ev_out[set], s_d2h));
        }
        CK(cudaStreamSynchronize(s_d2h));
        CK(cudaStreamSynchronize(s_h2d));
        for (int32_t i = std::max(0, n_batches - 2); i < n_batches; ++i) unstage_small(i);
        staged = false;  // the device tapes no longer hold a staged batch
    }

    // Results to the host.  ld > 0: vm / va go to columns [0, n_tasks) of host
    // arrays [n][ld] (a slice of a larger batch; the caller offsets the pointers).
    void fetch(double* vm, double* va, int32_t* iters, uint8_t* conv, int32_t* status,
               double* maxmis, int64_t ld = 0) {
        CK(cudaSetDevice(opt.device));
        const int32_t nt = v.n_tasks;
        const size_t row = size_t(nt) * 8;
        // pack [n][bpad] -> [n][n_tasks] on the device into the phasor tapes (free
        // after a solve: the next run recomputes them, flows read the angles), then
        // one linear (or pitched, for a slice) D2H each
        auto d2h = [&](double* dst, double* packed, const double* src) {
            gbnr::launch_pack(packed, src, sym.n, nt, v.bpad, stream);
            if (ld <= 0 || ld == nt)
                CK(cudaMemcpyAsync(dst, packed, size_t(sym.n) * row, cudaMemcpyDeviceToHost, stream));
            else
                CK(cudaMemcpy2DAsync(dst, size_t(ld) * 8, packed, row, row, size_t(sym.n), cudaMemcpyDeviceToHost,
                                     stream));
        };
        if (vm) d2h(vm, v.c, v.vm);
        if (va) d2h(va, v.s, v.va);
        std::vector<int32_t> st(nt);
        CK(cudaMemcpyAsync(st.data(), v.status, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        if (iters) CK(cudaMemcpyAsync(iters, v.iters, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
        if (maxmis) CK(cudaMemcpyAsync(maxmis, v.maxmis, size_t(nt) * 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (status) std::memcpy(status, st.data(), size_t(nt) * 4);
        if (conv)
            for (int32_t t = 0; t < nt; ++t) conv[t] = st[t] == GBNR_CONVERGED || st[t] == GBNR_FALLBACK_CONVERGED;
    }

    // calc_branch_flows on the voltages of the last solve (device-resident)
    void branch_flows(int32_t nb, const int32_t* bf, const int32_t* bt, const double* adm, const int32_t* outage,
                      double* sfr, double* sfi, double* str, double* sti) {
        if (!solved) throw Error(GBNR_ECONFIG, "gbnr_branch_flows before a solve");
        if (!whole_on_device)
            throw Error(GBNR_ECONFIG, "the last solve was sharded over devices or chunked: the device does not hold "
                                      "every task's voltages (solve with n_devices = 1 and a batch that fits)");
        CK(cudaSetDevice(opt.device));
        const size_t T = size_t(v.n_tasks), out_bytes = size_t(nb) * T * 8;
        std::vector<void*> tmp;
        auto up = [&](const void* h, size_t bytes) {
            void* d = dmalloc(bytes);
            tmp.push_back(d);
            if (h) CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
            return d;
        };
        try {
            auto* dbf = static_cast<const int32_t*>(up(bf, size_t(nb) * 4));
            auto* dbt = static_cast<const int32_t*>(up(bt, size_t(nb) * 4));
            auto* dadm = static_cast<const double*>(up(adm, size_t(nb) * 64));
            auto* dout = outage ? static_cast<const int32_t*>(up(outage, T * 4)) : nullptr;
            double* o[4];
            for (auto& q : o) q = static_cast<double*>(up(nullptr, out_bytes));
            gbnr::launch_flows(v, nb, dbf, dbt, dadm, dout, o[0], o[1], o[2], o[3], stream);
            CK(cudaGetLastError());
            double* h[4] = {sfr, sfi, str, sti};
            for (int i = 0; i < 4; ++i)
                if (h[i]) CK(cudaMemcpyAsync(h[i], o[i], out_bytes, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
        } catch (...) {
            for (void* q : tmp) dfree(q);
            throw;
        }
        for (void* q : tmp) dfree(q);
    }

    // walker time breakdown of the launches since the last reset (GBNR_PROF builds)
    void prof_report(const char* what) {
        if (!v.prof) return;
        std::vector<unsigned long long> h(4 * 8 * 16);
        CK(cudaMemcpy(h.data(), v.prof, h.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemset(v.prof, 0, h.size() * 8));
        static const char* cat[12] = {"stepwait", "depwait", "page", "sync", "dep", "dep2", "end", "issue",
                                      "other", "n_dep", "n_dep2", "n_issue"};
        std::fprintf(stderr, "[prof %s] per phase: cycles summed over tiles, per walker warp\n", what);
        for (int ph = 0; ph < 4; ++ph)
            for (int w = 0; w < 8; ++w) {
                const unsigned long long* c = h.data() + (ph * 8 + w) * 16;
                unsigned long long tot = 0;
                for (int i = 0; i < 9; ++i) tot += c[i];
                if (!tot) continue;
                std::fprintf(stderr, "ph%d w%d tot %.3g:", ph, w, double(tot));
                for (int i = 0; i < 12; ++i)
                    std::fprintf(stderr, " %s=%.3g", cat[i], i < 9 ? double(c[i]) / double(tot) : double(c[i]));
                std::fprintf(stderr, "\n");
            }
    }

    void refactor(int32_t reps, double* lu_out, uint8_t* flags_out, double* ms_out) {
        if (!staged) throw Error(GBNR_ECONFIG, "gbnr_refactor before gbnr_stage");
        CK(cudaSetDevice(opt.device));
        gbnr::launch_init(v, stream);
        gbnr::launch_jacobian(v, true, stream);
        CK(cudaGetLastError());
        gbnr::launch_lu_walk(v, cur->vl, false, stream);  // warm-up
        if (v.prof) {
            CK(cudaStreamSynchronize(stream));
            CK(cudaMemset(v.prof, 0, 4 * 8 * 16 * 8));
        }
        CK(cudaEventRecord(ev0, stream));
        for (int32_t r = 0; r < reps; ++r) gbnr::launch_lu_walk(v, cur->vl, false, stream);
        CK(cudaEventRecord(ev1, stream));
        CK(cudaGetLastError());
        CK(cudaEventSynchronize(ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev0, ev1));
        if (ms_out) *ms_out = reps > 0 ? ms / reps : 0.0;
        prof_report("refactor");
        const int32_t nt = v.n_tasks;
        if (flags_out) CK(cudaMemcpy(flags_out, v.flag, size_t(nt), cudaMemcpyDeviceToHost));
        if (lu_out) {
            // tile-blocked tape -> element-major CCS order [nnzLU][n_tasks]
            const size_t TW = size_t(v.tw), z = size_t(v.nnzLU), tr = size_t(v.tape_rows) * TW;
            std::vector<double> tape(size_t(v.n_tiles) * tr);  // the LU part of every tile's block
            CK(cudaMemcpy2D(tape.data(), tr * 8, v.LU, v.tstride * 8, tr * 8, size_t(v.n_tiles),
                            cudaMemcpyDeviceToHost));
            for (size_t c = 0; c < z; ++c) {
                const size_t ts = size_t(lay.tape_of_ccs[c]);
                for (int32_t t = 0; t < nt; ++t)
                    lu_out[c * nt + t] = tape[size_t(t) / TW * tr + ts * TW + size_t(t) % TW];
            }
        }
    }
};

extern "C" {

void gbnr_default_options(gbnr_options* o) {
    std::memset(o, 0, sizeof *o);
    o->tol = 1e-8;
    o->max_iter = 10;
    o->pivot_tol = 1e-3;
    o->singular_tol = 1e-14;
    o->device = 0;
    o->ring_rows = 0;
    o->profile = 0;
    o->stage_rows = 0;
    o->prefetch = 8;
    o->headroom = 1;
    o->walkers = 8;
    o->jacobian = 0;
    o->second_chance = 1;
    o->n_devices = 1;
    o->device_step = 1;
    o->chunk_tasks = 0;
    o->tile_width = 0;
}

const char* gbnr_last_error(void) { return g_err.c_str(); }

const char* gbnr_version(void) { return "gbnr 0.1 sm_100a"; }

int gbnr_build_ybus(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                    const double* r, const double* x, const double* b, const double* tap,
                    const double* shift_deg, const uint8_t* in_service, const double* gs,
                    const double* bs, double base_mva, int32_t* indptr, int32_t* indices,
                    int32_t* diag, double* y_re, double* y_im, int32_t* nnz_out) {
    return guarded([&] {
        const gbnr::YbusCsr y = gbnr::build_ybus(n_bus, n_branch, from, to, r, x, b, tap, shift_deg,
                                                 in_service, gs, bs, base_mva);
        std::memcpy(indptr, y.indptr.data(), y.indptr.size() * 4);
        std::memcpy(indices, y.indices.data(), y.indices.size() * 4);
        std::memcpy(diag, y.diag.data(), y.diag.size() * 4);
        std::memcpy(y_re, y.re.data(), y.re.size() * 8);
        std::memcpy(y_im, y.im.data(), y.im.size() * 8);
        *nnz_out = static_cast<int32_t>(y.indices.size());
    });
}

int gbnr_contingency_values(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                            const double* r, const double* x, const double* b, const double* tap,
                            const double* shift_deg, const uint8_t* in_service, const double* gs,
                            const double* bs, double base_mva, const int32_t* outage_branch, int32_t n_tasks,
                            double* y_re, double* y_im, uint8_t* islanded) {
    return guarded([&] {
        if (n_tasks <= 0) throw Error(GBNR_ECONFIG, "n_tasks must be positive");
        const gbnr::YbusCsr y = gbnr::build_ybus(n_bus, n_branch, from, to, r, x, b, tap, shift_deg,
                                                 in_service, gs, bs, base_mva);
        gbnr::contingency_values(y, n_branch, from, to, in_service, outage_branch, n_tasks, y_re, y_im,
                                 islanded);
    });
}

int gbnr_branch_admittances(int32_t n_bus, int32_t n_branch, const int32_t* from, const int32_t* to,
                            const double* r, const double* x, const double* b, const double* tap,
                            const double* shift_deg, const uint8_t* in_service, const double* gs,
                            const double* bs, double base_mva, double* adm) {
    return guarded([&] {
        const gbnr::YbusCsr y = gbnr::build_ybus(n_bus, n_branch, from, to, r, x, b, tap, shift_deg,
                                                 in_service, gs, bs, base_mva);
        std::memcpy(adm, y.adm.data(), y.adm.size() * sizeof(double));
    });
}

int gbnr_branch_flows(gbnr_plan* p, int32_t n_branch, const int32_t* from, const int32_t* to,
                      const double* adm, const int32_t* outage_branch, double* sf_re, double* sf_im,
                      double* st_re, double* st_im) {
    return guarded([&] {
        if (!p->on_device) throw Error(GBNR_ECONFIG, "host-only plan (device = -1) has no voltages");
        for (int32_t k = 0; k < n_branch; ++k)
            if (from[k] < 0 || from[k] >= p->sym.n || to[k] < 0 || to[k] >= p->sym.n)
                throw Error(GBNR_ESTRUCT, "branch endpoint out of range");
        p->branch_flows(n_branch, from, to, adm, outage_branch, sf_re, sf_im, st_re, st_im);
    });
}

int gbnr_amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix, int32_t* fwd) {
    return guarded([&] {
        const std::vector<int32_t> f = gbnr::amd_order(n, col_ptr, row_ix);
        std::memcpy(fwd, f.data(), size_t(n) * 4);
    });
}

}  // extern "C"

static int create_plan(int32_t n_bus, const int32_t* indptr, const int32_t* indices, const double* y_re,
                       const double* y_im, int32_t ref, const int32_t* pv, int32_t n_pv, const int32_t* pq,
                       int32_t n_pq, const double* vm0, const double* va0, const gbnr_options* opt, gbnr_plan** out,
                       bool sub) {
    *out = nullptr;
    gbnr_plan* p = new (std::nothrow) gbnr_plan();
    if (!p) {
        g_err = "host out of memory";
        return GBNR_ECONFIG;
    }
    const int rc = guarded([&] {
        if (opt)
            p->opt = *opt;
        else
            gbnr_default_options(&p->opt);
        if (!(p->opt.tol > 0.0) || p->opt.max_iter < 1 || p->opt.max_iter > 30)
            throw Error(GBNR_ECONFIG, "need tol > 0 and 1 <= max_iter <= 30");
        if (p->opt.ring_rows < 0 || p->opt.stage_rows < 0 || p->opt.prefetch < 0 || p->opt.headroom < 0 ||
            p->opt.walkers < 0 || p->opt.walkers > gbnr::kLuWarps)
            throw Error(GBNR_ECONFIG, "negative walk parameter");
        if (p->opt.jacobian < 0 || p->opt.jacobian > 2) throw Error(GBNR_ECONFIG, "jacobian policy must be 0, 1 or 2");
        if (p->opt.second_chance < 0) throw Error(GBNR_ECONFIG, "second_chance must be >= 0");
        if (p->opt.n_devices < 0 || p->opt.n_devices > 64 || p->opt.device_step < 0 || p->opt.chunk_tasks < 0)
            throw Error(GBNR_ECONFIG, "need 0 <= n_devices <= 64, device_step >= 0, chunk_tasks >= 0");
        if (p->opt.tile_width < 0 || p->opt.tile_width > gbnr::kTile || (p->opt.tile_width & 1))
            throw Error(GBNR_ECONFIG, "tile_width must be 0 (automatic) or even in 2..32");
        p->sub_plan = sub;
        const auto t0 = std::chrono::steady_clock::now();
        p->sym.analyze(n_bus, indptr, indices, y_re, y_im, ref, pv, n_pv, pq, n_pq, vm0, va0,
                       p->opt.pivot_tol);
        p->in_pv.assign(pv, pv + n_pv);
        p->in_pq.assign(pq, pq + n_pq);
        p->lay = gbnr::build_lu_layout(p->sym);
        const auto t1 = std::chrono::steady_clock::now();
        gbnr::WalkConfig wc;
        if (p->opt.ring_rows) wc.ring_rows = p->opt.ring_rows;
        if (p->opt.stage_rows) wc.stage_rows = p->opt.stage_rows;
        if (p->opt.prefetch) wc.prefetch = p->opt.prefetch;
        if (p->opt.headroom) wc.headroom = p->opt.headroom;
        if (p->opt.walkers) wc.walkers = p->opt.walkers;
        if (const char* e = std::getenv("GBNR_STAGE_FRAC")) wc.stage_frac = std::atof(e);
        if (const char* e = std::getenv("GBNR_STAGE_FRAC_UP")) wc.stage_frac_up = std::atof(e);
        if (const char* e = std::getenv("GBNR_PAGE_WORDS")) wc.page_words = std::atoi(e);
        if (const char* e = std::getenv("GBNR_UNIFIED")) wc.unified = std::atoi(e) != 0;  // 0: split plans
        if (const char* e = std::getenv("GBNR_PAIRS")) wc.pairs = std::atoi(e) != 0;      // 0: no row pairs
        if (const char* e = std::getenv("GBNR_SMEM_BUDGET")) wc.smem_budget = std::atoi(e);
        if (const char* e = std::getenv("GBNR_BALANCE")) wc.balance = std::atof(e);
        // tests: also move blocks larger than this share of a walker's pool to global memory
        if (const char* e = std::getenv("GBNR_GLOBAL_FRAC")) wc.global_frac = std::atof(e);
        if (const char* e = std::getenv("GBNR_LEVELS")) {  // e.g. "8,8,4,2,1"
            for (const char* q = e; *q;) {
                wc.levels.push_back(std::atoi(q));
                while (*q && *q != ',') ++q;
                if (*q == ',') ++q;
            }
            if (wc.levels.empty() || wc.levels.front() != wc.walkers || wc.levels.back() != 1)
                throw Error(GBNR_ECONFIG, "GBNR_LEVELS must start at the walker count and end at 1");
        }
        p->wcfg = wc;
        if (const char* e = std::getenv("GBNR_CTAS")) p->ctas_per_sm = std::max(1, std::atoi(e));
        if (p->opt.device < 0) {
            p->cur = p->walks_for(gbnr::kTile);  // host-only plan: the full-width programs (inspection, tests)
            if (std::getenv("GBNR_PLAN_TIMING"))
                std::fprintf(stderr, "[plan] analysis %.1f ms, walks %.1f ms\n",
                             std::chrono::duration<double, std::milli>(t1 - t0).count(),
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
        } else {
            int ndev = 0;
            CK(cudaGetDeviceCount(&ndev));
            if (p->opt.device >= ndev) throw Error(GBNR_ECUDA, "CUDA device ordinal out of range");
            CK(cudaSetDevice(p->opt.device));
            CK(cudaDeviceGetAttribute(&p->n_sm, cudaDevAttrMultiProcessorCount, p->opt.device));
            gbnr::configure_kernels();
            p->on_device = true;
            p->upload_structure();
            p->set_ybus(y_re, y_im);
            p->cur = p->walks_for(gbnr::kTile);
            // n_devices > 1: the same frozen symbolic state and walk programs on
            // devices device + i * device_step, one plan each
            const int32_t nd = std::max(1, p->opt.n_devices);
            for (int32_t i = 1; i < nd; ++i) {
                const int32_t d = p->opt.device + i * p->opt.device_step;
                if (d >= ndev) throw Error(GBNR_ECUDA, "n_devices: CUDA device ordinal out of range");
                auto q = std::make_unique<gbnr_plan>();
                q->sym = p->sym;
                q->in_pv = p->in_pv;
                q->in_pq = p->in_pq;
                q->lay = p->lay;
                q->wcfg = p->wcfg;
                q->ctas_per_sm = p->ctas_per_sm;
                q->opt = p->opt;
                q->opt.device = d;
                q->opt.n_devices = 1;
                q->sub_plan = sub;
                CK(cudaSetDevice(d));
                CK(cudaDeviceGetAttribute(&q->n_sm, cudaDevAttrMultiProcessorCount, d));
                gbnr::configure_kernels();
                q->on_device = true;
                q->upload_structure();
                q->set_ybus(y_re, y_im);
                for (const auto& w : p->walks) q->adopt_walks(*w);
                q->cur = q->walks.front().get();
                p->peers.push_back(std::move(q));
            }
            CK(cudaSetDevice(p->opt.device));
        }
    });
    if (rc != GBNR_OK) {
        delete p;
        return rc;
    }
    *out = p;
    return GBNR_OK;
}

extern "C" {

int gbnr_plan_create(int32_t n_bus, const int32_t* indptr, const int32_t* indices,
                     const double* y_re, const double* y_im, int32_t ref, const int32_t* pv,
                     int32_t n_pv, const int32_t* pq, int32_t n_pq, const double* vm0,
                     const double* va0, const gbnr_options* opt, gbnr_plan** out) {
    return create_plan(n_bus, indptr, indices, y_re, y_im, ref, pv, n_pv, pq, n_pq, vm0, va0, opt, out, false);
}

void gbnr_plan_destroy(gbnr_plan* plan) { delete plan; }

int gbnr_plan_stats(const gbnr_plan* p, int64_t* o) {
    return guarded([&] {
        const gbnr::Symbolic& s = p->sym;
        const int64_t vals[16] = {s.nJ,         s.nnzJ,      s.nnzLU,     s.nnzL,
                                  s.nnzU,       s.D,         2 * s.D + s.nnzL, s.levels_lu,
                                  s.levels_fs,  s.levels_bs, s.offdiag_piv, s.npvpq,
                                  s.nnzLU - s.nnzJ, s.max_col, s.max_udeps, s.nnzY};
        std::memcpy(o, vals, sizeof vals);
    });
}

int gbnr_plan_export(const gbnr_plan* p, int32_t* row_fwd, int32_t* col_fwd, int32_t* col_ptr,
                     int32_t* row_ix, int32_t* level) {
    return guarded([&] {
        const gbnr::Symbolic& s = p->sym;
        if (row_fwd) std::memcpy(row_fwd, s.row_fwd.data(), size_t(s.nJ) * 4);
        if (col_fwd) std::memcpy(col_fwd, s.col_fwd.data(), size_t(s.nJ) * 4);
        if (col_ptr) std::memcpy(col_ptr, s.cp.data(), size_t(s.nJ + 1) * 4);
        if (row_ix) std::memcpy(row_ix, s.ri.data(), size_t(s.nnzLU) * 4);
        if (level) std::memcpy(level, s.level.data(), size_t(s.nJ) * 4);
    });
}

int gbnr_stage(gbnr_plan* p, int32_t n_tasks, const double* p0, const double* q0, int32_t n_ssets,
               const double* vm0, const double* va0, int32_t n_vsets) {
    return guarded([&] {
        if (n_ssets < 1) throw Error(GBNR_ECONFIG, "n_ssets must be 1 or n_tasks");
        if (p->on_device) p->stage_ybus(nullptr, nullptr, 1, n_tasks);  // the plan's shared set
        p->stage(n_tasks, p0, q0, n_ssets, vm0, va0, n_vsets);
    });
}

int gbnr_run(gbnr_plan* p) {
    return guarded([&] { p->run(); });
}

int gbnr_fetch(gbnr_plan* p, double* vm_out, double* va_out, int32_t* iterations_out,
               uint8_t* converged_out, int32_t* status_out, double* max_mismatch_out) {
    return guarded([&] {
        if (!p->staged) throw Error(GBNR_ECONFIG, "gbnr_fetch before gbnr_stage");
        p->fetch(vm_out, va_out, iterations_out, converged_out, status_out, max_mismatch_out);
    });
}

int gbnr_solve(gbnr_plan* p, int32_t n_tasks, const double* y_re, const double* y_im,
               int32_t n_ysets, const double* p0, const double* q0, int32_t n_ssets,
               const double* vm0, const double* va0, int32_t n_vsets, double* vm_out,
               double* va_out, int32_t* iterations_out, uint8_t* converged_out,
               int32_t* status_out, double* max_mismatch_out) {
    return guarded([&] {
        if (!p->on_device) throw Error(GBNR_ECONFIG, "host-only plan (device = -1) cannot solve");
        const gbnr_plan::SolveIn in{n_tasks, y_re, y_im, n_ysets, p0, q0, n_ssets, vm0, va0, n_vsets};
        const gbnr_plan::SolveOut out{vm_out, va_out, iterations_out, converged_out, status_out, max_mismatch_out};
        // N-1 batches (per-task Ybus sets): islanded tasks dominate the flags, no re-derivation
        p->solve_general(in, out, !y_re || n_ysets == 1);
        p->solved = true;
    });
}

int gbnr_solve_batches(gbnr_plan* p, int32_t n_batches, int32_t n_tasks, const double* const* p0,
                       const double* const* q0, const double* vm0, const double* va0, double* const* vm_out,
                       double* const* va_out, int32_t* const* iterations_out, uint8_t* const* converged_out,
                       int32_t* const* status_out, double* const* max_mismatch_out) {
    return guarded([&] {
        for (int32_t i = 0; i < n_batches; ++i)
            if (!p0 || !q0 || !p0[i] || !q0[i]) throw Error(GBNR_ECONFIG, "every batch needs p0 and q0");
        if (p->peers.empty()) {
            p->solve_batches(n_batches, n_tasks, p0, q0, vm0, va0, vm_out, va_out, iterations_out, converged_out,
                             status_out, max_mismatch_out);
            return;
        }
        // n_devices > 1: batches dealt round-robin, each device pipelines its own
        // share from its own host thread
        std::vector<gbnr_plan*> dev{p};
        for (auto& q : p->peers) dev.push_back(q.get());
        const size_t D = dev.size();
        std::vector<std::exception_ptr> errs(D);
        auto pick = [&](auto* const* a, size_t d) {
            std::vector<std::remove_const_t<std::remove_pointer_t<decltype(a)>>> o;
            for (int32_t j = int32_t(d); j < n_batches; j += int32_t(D)) o.push_back(a ? a[j] : nullptr);
            return o;
        };
        auto shard = [&](size_t d) {
            try {
                auto P = pick(p0, d);
                auto Q = pick(q0, d);
                auto VM = pick(vm_out, d);
                auto VA = pick(va_out, d);
                auto IT = pick(iterations_out, d);
                auto CV = pick(converged_out, d);
                auto ST = pick(status_out, d);
                auto MM = pick(max_mismatch_out, d);
                if (!P.empty())
                    dev[d]->solve_batches(int32_t(P.size()), n_tasks, P.data(), Q.data(), vm0, va0, VM.data(),
                                          VA.data(), IT.data(), CV.data(), ST.data(), MM.data());
            } catch (...) {
                errs[d] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (size_t d = 1; d < D; ++d) th.emplace_back(shard, d);
        shard(0);
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

int gbnr_last_timing(const gbnr_plan* p, double* out) {
    return guarded([&] { std::memcpy(out, p->timing, sizeof p->timing); });
}

static const gbnr::WalkSet& pick_walk(const gbnr_plan* p, int32_t which) {
    if (which == 0) return p->cur->wf;
    if (which == 1) return p->cur->wl;
    if (which == 2) return p->cur->wb;
    throw Error(GBNR_ECONFIG, "walk index must be 0, 1 or 2");
}

int gbnr_walk_info(const gbnr_plan* p, int32_t which, int64_t* o) {
    return guarded([&] {
        const gbnr::WalkSet& w = pick_walk(p, which);
        const int64_t vals[20] = {w.steps, w.walkers, w.phases, w.rows, w.page_words, w.pages,
                                  w.barriers, int64_t(w.stream.size()), w.events, w.ring_dep_rows,
                                  w.fetched_rows, w.n_ops, w.n_copies, int64_t(w.smem_bytes()),
                                  w.parts.empty() ? 0 : w.parts[0].ring_rows,
                                  w.parts.empty() ? 0 : w.parts[0].stage_rows,
                                  w.global_steps, w.global_deps, w.scratch_rows, 0};
        std::memcpy(o, vals, sizeof vals);
    });
}

int gbnr_walk_export(const gbnr_plan* p, int32_t which, int32_t part, void* dst) {
    return guarded([&] {
        const gbnr::WalkSet& w = pick_walk(p, which);
        auto put = [&](const auto& vec) {
            if (!vec.empty()) std::memcpy(dst, vec.data(), vec.size() * sizeof(vec[0]));
        };
        switch (part) {
            case 0: put(w.stream); break;
            case 1: put(w.wpage0); break;
            case 2: put(w.owner); break;
            case 3: put(p->lay.tape_of_ccs); break;
            case 4: put(p->lay.lslot); break;
            case 5: put(p->lay.ucrs0); break;
            default: throw Error(GBNR_ECONFIG, "walk part must be 0..5");
        }
    });
}

int gbnr_refactor(gbnr_plan* p, int32_t reps, double* lu_out, uint8_t* flags_out, double* ms_out) {
    return guarded([&] { p->refactor(reps, lu_out, flags_out, ms_out); });
}

}  // extern "C"
