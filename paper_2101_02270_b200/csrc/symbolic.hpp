// symbolic.hpp -- one-time host analysis (C++) for the batched NR solver.
//
// Everything here runs once per plan, single-threaded, and produces the frozen
// structures every task shares read-only (sparse.hpp:1-7):
//   * Ybus (grid.hpp:195-243)                         build_ybus
//   * reduced Jacobian pattern      Symbolic::analyze
//   * AMD ordering (amd.hpp:29-157)                    amd_order
//   * left-looking Gilbert-Peierls factorization with threshold partial
//     pivoting on the representative task -> frozen L+U
//     pattern, row/col permutations (Eq. 3)
//   * scatter lookup Ybus slot x quadrant -> A slot (sparse.hpp:237-267 shape)
//   * level schedule counters; the execution plan of the
//     refactorization and the triangular solves is walk.hpp
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gbnr {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct YbusCsr {
    int32_t n = 0;
    std::vector<int32_t> indptr, indices, diag;
    std::vector<double> re, im;
    std::vector<int32_t> slot;  // [4 * n_branch] slots of (ff, ft, tf, tt)
    std::vector<double> adm;    // [8 * n_branch] (re, im) of the branch's (ff, ft, tf, tt)
};

YbusCsr build_ybus(int32_t n_bus, int32_t n_branch, const int32_t* f, const int32_t* t,
                   const double* r, const double* x, const double* b, const double* tap,
                   const double* shift_deg, const uint8_t* on, const double* gs, const double* bs,
                   double base_mva);

std::vector<int32_t> amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix);

// N-1 value sets (element-major [nnzY][n_tasks]) and islanding flags per task;
// outage[task] = branch index, or -1 for the base case.
void contingency_values(const YbusCsr& y, int32_t n_branch, const int32_t* from, const int32_t* to,
                        const uint8_t* in_service, const int32_t* outage, int32_t n_tasks, double* y_re,
                        double* y_im, uint8_t* islanded);

struct Symbolic {
    // inputs
    int32_t n = 0, ref = 0, npv = 0, npq = 0, npvpq = 0, nJ = 0, nnzY = 0;
    std::vector<int32_t> yp, yi;
    std::vector<int32_t> jth, jvm;  // bus -> J index of theta / |V| unknown (-1)
    // J / LU structure
    int64_t nnzJ = 0, nnzLU = 0, nnzL = 0, nnzU = 0, D = 0, offdiag_piv = 0;
    int32_t max_col = 0, max_udeps = 0, levels_lu = 0, levels_fs = 0, levels_bs = 0;
    std::vector<int32_t> row_fwd, col_fwd;  // J row/col -> LU row/col
    std::vector<int32_t> cp, ri, dpos;      // LU CCS in pivot numbering
    std::vector<int32_t> aidx;              // LU slot -> rank among J-fed slots (-1 = fill)
    std::vector<int32_t> lk;                // [4*nnzY] Ybus slot x {Pth,Pvm,Qth,Qvm} -> LU slot
    std::vector<int32_t> level;             // LU level per column
    // NPM / J row list (non-slack buses) and per-bus b / z positions
    std::vector<int32_t> rows;            // non-slack buses, ascending
    std::vector<int32_t> brow_p, brow_q;  // bus -> LU row of its P / Q equation (-1)
    std::vector<int32_t> zcol_t, zcol_v;  // bus -> LU col of its theta / |V| unknown (-1)

    void analyze(int32_t n_bus, const int32_t* indptr, const int32_t* indices, const double* y_re,
                 const double* y_im, int32_t ref, const int32_t* pv, int32_t n_pv,
                 const int32_t* pq, int32_t n_pq, const double* vm0, const double* va0,
                 double pivot_tol);
};

}  // namespace gbnr
