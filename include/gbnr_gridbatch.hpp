// gbnr_gridbatch.hpp -- the reference-side adapter.
//
// What a maintainer of the reference (gridbatch, header-only C++20) adds next to
// SPEC's `newton` module so that `nr_solve_batch` runs on
// libgbnr.so.  It uses only the reference's own types -- GridCase (grid.hpp:60),
// YbusModel / build_ybus (grid.hpp:188-243), ProfileBatch / assemble_profiles
// (grid.hpp:290-344), BatchTape (batch_tape.hpp:20-56), the error taxonomy
// (core.hpp:33-65) -- and the plain C ABI of gbnr.h.  The reference does not
// define NrConfig / TaskStatus / TaskResult yet; they
// are declared here as SPEC states them.  tests/test_integration_adapter.py
// compiles this header against /root/reference/proj/include and runs it.
#pragma once

#include <cstdint>
#include <vector>

#include "gbnr.h"
#include "gridbatch/batch_tape.hpp"
#include "gridbatch/core.hpp"
#include "gridbatch/grid.hpp"

namespace gridbatch {

struct NrConfig {
    real_t tol = 1e-8;
    int32_t max_iter = 10;
};

enum class TaskStatus { converged, diverged, singular, fallback_converged, islanded };

struct TaskResult {
    TaskStatus status = TaskStatus::diverged;
    int32_t iterations = 0;
    real_t max_mismatch = 0.0;
    std::vector<real_t> vm, va;
};

// core.hpp:32-65 taxonomy for a non-zero gbnr return code
[[noreturn]] inline void gbnr_throw(int rc) {
    const char* msg = gbnr_last_error();
    switch (rc) {
        case GBNR_EPARSE: throw ParseError(msg);
        case GBNR_ESTRUCT: throw StructuralError(msg);
        case GBNR_ESINGULAR: throw SingularError(msg);
        default: throw ConfigError(msg);  // GBNR_ECONFIG, GBNR_ECUDA
    }
}

// SPEC.md:392-400 `initialize`: the symbolic analysis and the device plan.
class GbnrSymbolic {
public:
    GbnrSymbolic(const GridCase& gc, const ProfileBatch& pb, const NrConfig& cfg, int device) {
        const YbusModel y = build_ybus(gc);  // grid.hpp:208
        std::vector<double> yre(y.base_values.size()), yim(y.base_values.size());
        for (size_t s = 0; s < yre.size(); ++s) {
            yre[s] = y.base_values[s].real();
            yim[s] = y.base_values[s].imag();
        }
        gbnr_options o;
        gbnr_default_options(&o);
        o.tol = cfg.tol;
        o.max_iter = cfg.max_iter;
        o.device = device;
        n_bus_ = gc.n_bus();
        const int rc = gbnr_plan_create(gc.n_bus(), y.pattern.row_ptr.data(), y.pattern.col_ix.data(), yre.data(),
                                        yim.data(), gc.slack_bus, gc.pv_buses.data(),
                                        static_cast<int32_t>(gc.pv_buses.size()), gc.pq_buses.data(),
                                        static_cast<int32_t>(gc.pq_buses.size()), pb.vm_start.data(),
                                        pb.va_start.data(), &o, &plan_);
        if (rc != GBNR_OK) gbnr_throw(rc);
    }
    GbnrSymbolic(const GbnrSymbolic&) = delete;
    GbnrSymbolic& operator=(const GbnrSymbolic&) = delete;
    ~GbnrSymbolic() { gbnr_plan_destroy(plan_); }

    gbnr_plan* plan() const { return plan_; }
    index_t n_bus() const { return n_bus_; }

private:
    gbnr_plan* plan_ = nullptr;
    index_t n_bus_ = 0;
};

// per-task results; per-task numerical trouble goes to the
// status, never to an exception (core.hpp:33-34).
inline std::vector<TaskResult> nr_solve_batch_gbnr(GbnrSymbolic& s, const ProfileBatch& pb) {
    const index_t n = s.n_bus(), T = pb.n_tasks;
    std::vector<double> vm(size_t(n) * T), va(size_t(n) * T), mis(T);
    std::vector<int32_t> it(T), st(T);
    std::vector<uint8_t> ok(T);
    // BatchTape is element-major with the task innermost -- gbnr's layout, no transpose
    const int rc = gbnr_solve(s.plan(), T, nullptr, nullptr, 1, pb.p0.data(), pb.q0.data(), pb.n_sets,
                              pb.vm_start.data(), pb.va_start.data(), 1, vm.data(), va.data(), it.data(),
                              ok.data(), st.data(), mis.data());
    if (rc != GBNR_OK) gbnr_throw(rc);
    std::vector<TaskResult> out(T);
    for (index_t t = 0; t < T; ++t) {
        TaskResult& r = out[t];
        r.status = st[t] == GBNR_CONVERGED            ? TaskStatus::converged
                   : st[t] == GBNR_FALLBACK_CONVERGED ? TaskStatus::fallback_converged
                   : st[t] == GBNR_SINGULAR           ? TaskStatus::singular
                                                      : TaskStatus::diverged;
        r.iterations = it[t];
        r.max_mismatch = mis[t];
        r.vm.resize(n);
        r.va.resize(n);
        for (index_t b = 0; b < n; ++b) {
            r.vm[b] = vm[size_t(b) * T + t];
            r.va[b] = va[size_t(b) * T + t];
        }
    }
    return out;
}

}  // namespace gridbatch
