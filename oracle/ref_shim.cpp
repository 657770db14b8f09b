// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim that compiles the reference's own header-only C++20
// substrate (/root/reference/proj/include/gridbatch/*.hpp, read in place, never
// copied) into oracle/_ref/libgbref.so, so the parity suite can run the
// reference itself on the same inputs:
//   * parse_case            case_io.hpp:345-351 (MATPOWER subset :150-240, JSON :246)
//   * build_ybus            grid.hpp:208-243 (branch_admittance :195-206)
//   * assemble_profiles     grid.hpp:299-344 (P0/Q0 :326-327, V0 rule :331-342)
//   * amd_order             amd.hpp:29-157
//   * crs_from_coordinates  sparse.hpp:146-181, crs_to_ccs_pattern :194-220,
//     build_scatter_lookup  sparse.hpp:237-267
// The reference has no Newton-Raphson / LU code; those parts
// of the oracle are the C restatement in oracle/oracle.c.
//
// Built by oracle/Makefile (target ref) only where /root/reference exists.

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gridbatch/amd.hpp"
#include "gridbatch/case_io.hpp"
#include "gridbatch/grid.hpp"
#include "gridbatch/sparse.hpp"

using namespace gridbatch;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const StructuralError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 3;
    } catch (const SingularError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Parsed case handle.
void* ref_parse_case(const char* text, int* rc) {
    GridCase* out = nullptr;
    *rc = guarded([&] { out = new GridCase(parse_case(text)); });
    return out;
}

void ref_free_case(void* h) { delete static_cast<GridCase*>(h); }

// dims: n_bus, n_branch, slack, n_pv, n_pq, nnz(Ybus)
int ref_case_dims(void* h, int64_t* dims) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const YbusModel y = build_ybus(gc);
        dims[0] = gc.n_bus();
        dims[1] = gc.n_branch();
        dims[2] = gc.slack_bus;
        dims[3] = static_cast<int64_t>(gc.pv_buses.size());
        dims[4] = static_cast<int64_t>(gc.pq_buses.size());
        dims[5] = y.pattern.nnz();
    });
}

int ref_case_sets(void* h, int32_t* pv, int32_t* pq) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        std::memcpy(pv, gc.pv_buses.data(), gc.pv_buses.size() * sizeof(int32_t));
        std::memcpy(pq, gc.pq_buses.data(), gc.pq_buses.size() * sizeof(int32_t));
    });
}

int ref_build_ybus(void* h, int32_t* indptr, int32_t* indices, int32_t* diag, double* yre,
                   double* yim) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const YbusModel y = build_ybus(gc);
        std::memcpy(indptr, y.pattern.row_ptr.data(), y.pattern.row_ptr.size() * sizeof(int32_t));
        std::memcpy(indices, y.pattern.col_ix.data(), y.pattern.col_ix.size() * sizeof(int32_t));
        std::memcpy(diag, y.pattern.diag_ptr.data(), y.pattern.diag_ptr.size() * sizeof(int32_t));
        for (size_t s = 0; s < y.base_values.size(); ++s) {
            yre[s] = y.base_values[s].real();
            yim[s] = y.base_values[s].imag();
        }
    });
}

// Profiles for an explicit per-set load table (p_mw/q_mvar [n_bus][n_sets]).
// Outputs p0,q0 [n_bus][n_sets]; vm_start, va_start, vm_setpoint [n_bus].
int ref_profiles(void* h, int32_t n_tasks, int32_t n_sets, const double* p_mw,
                 const double* q_mvar, double* p0, double* q0, double* vm_start,
                 double* va_start, double* vm_set) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const size_t n = static_cast<size_t>(gc.n_bus());
        ScenarioTable sc;
        sc.n_tasks = n_tasks;
        sc.n_sets = n_sets;
        sc.p_mw.assign(p_mw, p_mw + n * n_sets);
        sc.q_mvar.assign(q_mvar, q_mvar + n * n_sets);
        const ProfileBatch pb = assemble_profiles(gc, sc);
        std::memcpy(p0, pb.p0.data(), n * n_sets * sizeof(double));
        std::memcpy(q0, pb.q0.data(), n * n_sets * sizeof(double));
        std::memcpy(vm_start, pb.vm_start.data(), n * sizeof(double));
        std::memcpy(va_start, pb.va_start.data(), n * sizeof(double));
        std::memcpy(vm_set, pb.vm_setpoint.data(), n * sizeof(double));
    });
}

// Case loads as the reference reads them (MW / MVAr), for building scenario tables.
int ref_case_loads(void* h, double* p_mw, double* q_mvar) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const ScenarioTable sc = case_scenario(gc, 1);
        std::memcpy(p_mw, sc.p_mw.data(), sc.p_mw.size() * sizeof(double));
        std::memcpy(q_mvar, sc.q_mvar.data(), sc.q_mvar.size() * sizeof(double));
    });
}

// ybus_values_with_outage (grid.hpp:245-255) for one branch, and the islanding
// pre-check outage_islands_grid (grid.hpp:257-261).
int ref_ybus_outage(void* h, int32_t branch, double* yre, double* yim, int32_t* islands) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const YbusModel y = build_ybus(gc);
        const std::vector<cplx> v = ybus_values_with_outage(y, branch);
        for (size_t s = 0; s < v.size(); ++s) {
            yre[s] = v[s].real();
            yim[s] = v[s].imag();
        }
        *islands = outage_islands_grid(gc, branch) ? 1 : 0;
    });
}

// parse_scenario_csv (case_io.hpp:368-447): per-task bus loads [bus][n_tasks];
// call with p_mw = nullptr first to get n_tasks.
int ref_parse_scenario(void* h, const char* text, int32_t* n_tasks, double* p_mw, double* q_mvar) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const ScenarioTable sc = parse_scenario_csv(text, gc);
        *n_tasks = sc.n_tasks;
        if (p_mw) std::memcpy(p_mw, sc.p_mw.data(), sc.p_mw.size() * sizeof(double));
        if (q_mvar) std::memcpy(q_mvar, sc.q_mvar.data(), sc.q_mvar.size() * sizeof(double));
    });
}

// parse_outage_list (case_io.hpp:449-471); call with out = nullptr for the count.
int ref_parse_outages(void* h, const char* text, int32_t* n, int32_t* out) {
    return guarded([&] {
        const GridCase& gc = *static_cast<GridCase*>(h);
        const std::vector<index_t> o = parse_outage_list(text, gc);
        *n = static_cast<int32_t>(o.size());
        if (out)
            for (size_t i = 0; i < o.size(); ++i) out[i] = static_cast<int32_t>(o[i]);
    });
}

// amd_order on a square CCS pattern; writes forward[old] = new.
int ref_amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix, int32_t* fwd) {
    return guarded([&] {
        SparseCcs p;
        p.n_rows = p.n_cols = n;
        p.col_ptr.assign(col_ptr, col_ptr + n + 1);
        p.row_ix.assign(row_ix, row_ix + col_ptr[n]);
        const Permutation perm = amd_order(p);
        std::memcpy(fwd, perm.forward.data(), n * sizeof(int32_t));
    });
}

// crs_from_coordinates: returns nnz; row_ptr [n_rows+1], col_ix [cap], diag [n_rows].
int ref_crs_from_coords(int32_t n_rows, int32_t n_cols, int32_t n_entries, const int32_t* rows,
                        const int32_t* cols, int32_t cap, int32_t* row_ptr, int32_t* col_ix,
                        int32_t* diag, int32_t* nnz_out) {
    return guarded([&] {
        std::vector<std::pair<index_t, index_t>> e;
        for (int32_t i = 0; i < n_entries; ++i) e.emplace_back(rows[i], cols[i]);
        const SparseCrs m = crs_from_coordinates(n_rows, n_cols, std::move(e));
        *nnz_out = m.nnz();
        if (m.nnz() > cap) throw ConfigError("capacity too small");
        std::memcpy(row_ptr, m.row_ptr.data(), m.row_ptr.size() * sizeof(int32_t));
        std::memcpy(col_ix, m.col_ix.data(), m.col_ix.size() * sizeof(int32_t));
        if (!m.diag_ptr.empty())
            std::memcpy(diag, m.diag_ptr.data(), m.diag_ptr.size() * sizeof(int32_t));
    });
}

// crs_to_ccs_pattern: col_ptr [n_cols+1], row_ix [nnz], map [nnz].
int ref_crs_to_ccs(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_ix,
                   int32_t* col_ptr, int32_t* row_ix, int32_t* map) {
    return guarded([&] {
        SparseCrs m;
        m.n_rows = n_rows;
        m.n_cols = n_cols;
        m.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
        m.col_ix.assign(col_ix, col_ix + row_ptr[n_rows]);
        const CcsConversion c = crs_to_ccs_pattern(m);
        std::memcpy(col_ptr, c.ccs.col_ptr.data(), c.ccs.col_ptr.size() * sizeof(int32_t));
        std::memcpy(row_ix, c.ccs.row_ix.data(), c.ccs.row_ix.size() * sizeof(int32_t));
        std::memcpy(map, c.crs_to_ccs.data(), c.crs_to_ccs.size() * sizeof(int32_t));
    });
}

// build_scatter_lookup from a square CRS source into the CCS conversion of
// `target_crs` under (perm_row, perm_col); row_map/col_map filter (-1 = drop).
int ref_scatter_lookup(int32_t n, const int32_t* src_row_ptr, const int32_t* src_col_ix,
                       const int32_t* perm_row_fwd, const int32_t* perm_col_fwd, int32_t nt,
                       const int32_t* tgt_col_ptr, const int32_t* tgt_row_ix,
                       const int32_t* row_map, const int32_t* col_map, int32_t* lookup) {
    return guarded([&] {
        SparseCrs s;
        s.n_rows = s.n_cols = n;
        s.row_ptr.assign(src_row_ptr, src_row_ptr + n + 1);
        s.col_ix.assign(src_col_ix, src_col_ix + src_row_ptr[n]);
        SparseCcs t;
        t.n_rows = t.n_cols = nt;
        t.col_ptr.assign(tgt_col_ptr, tgt_col_ptr + nt + 1);
        t.row_ix.assign(tgt_row_ix, tgt_row_ix + tgt_col_ptr[nt]);
        const Permutation pr = Permutation::from_forward({perm_row_fwd, perm_row_fwd + nt});
        const Permutation pc = Permutation::from_forward({perm_col_fwd, perm_col_fwd + nt});
        const ScatterLookup lk = build_scatter_lookup(
            s, pr, pc, t, std::span<const index_t>(row_map, n), std::span<const index_t>(col_map, n));
        std::memcpy(lookup, lk.target_positions.data(), lk.target_positions.size() * sizeof(int32_t));
    });
}

}  // extern "C"
