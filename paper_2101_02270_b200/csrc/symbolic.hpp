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
//   * refactorization program (U deps ascending + L destinations, Alg. 2)
//   * sync-free schedules for LU, FS and BS (level order)
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
};

YbusCsr build_ybus(int32_t n_bus, int32_t n_branch, const int32_t* f, const int32_t* t,
                   const double* r, const double* x, const double* b, const double* tap,
                   const double* shift_deg, const uint8_t* on, const double* gs, const double* bs,
                   double base_mva);

std::vector<int32_t> amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix);

// Per-column record of the refactorization program (32 B, two uniform loads).
struct ColInfo {
    int32_t s0;      // first LU slot of the column
    int32_t len_dp;  // len | (diag position << 16)
    int32_t dep0;    // first entry in dep_wait
    int32_t ndep;    // number of U dependencies (ascending row order)
    int32_t u0;      // first update record
    int32_t nu;      // number of update records (= sum of |L(:,k)| over the deps)
    int32_t pad0, pad1;
};
// One VMAD element update of Alg. 2: x[dst] -= x[kpos] * LU[lslot], records of
// a column in dependency-ascending order (the sequential operation order).
struct Upd {
    int32_t lslot;     // LU slot of L(i, k)
    int32_t dst_kpos;  // position of row i in the column | (position of row k << 16)
};
// Per-row record for the pull-style triangular solves.
struct RowInfo {
    int32_t e0;    // first entry in the row list
    int32_t ne;    // number of entries
    int32_t diag;  // LU slot of the diagonal (BS); unused for FS
    int32_t pad;
};
struct RowEnt {
    int32_t slot;  // LU slot of L(i,k) / U(i,k)
    int32_t k;     // column index k (b/x position)
    int32_t wait;  // schedule position of row k
    int32_t pad;
};

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
    // refactorization program + schedule
    std::vector<ColInfo> col;
    std::vector<int32_t> dep_wait;  // schedule position of each U dependency column
    std::vector<Upd> upd;
    std::vector<int32_t> lu_sched;  // schedule position -> column
    // FS / BS
    std::vector<RowInfo> lrow, urow;
    std::vector<RowEnt> lent, uent;
    std::vector<int32_t> fs_sched, bs_sched;
    // level pointers into the schedules and the bulk / sync-free split levels
    std::vector<int32_t> lu_lvl_ptr, fs_lvl_ptr, bs_lvl_ptr;
    std::vector<int32_t> lu_lvl_maxlen;  // longest column per LU level
    // per level, columns split by working-set size: short (len <= short_cap) run in
    // the pipelined kernel, long ones in the large-working-set kernel
    int32_t short_cap = 24;
    std::vector<int32_t> lu_short, lu_short_ptr, lu_long, lu_long_ptr, lu_long_maxlen, lu_short_maxlen;
    int32_t bulk_min = 32, lu_split = 0, fs_split = 0, bs_split = 0;
    // NPM / J row list (non-slack buses) and per-bus b / z positions
    std::vector<int32_t> rows;            // non-slack buses, ascending
    std::vector<int32_t> brow_p, brow_q;  // bus -> LU row of its P / Q equation (-1)
    std::vector<int32_t> zcol_t, zcol_v;  // bus -> LU col of its theta / |V| unknown (-1)

    void analyze(int32_t n_bus, const int32_t* indptr, const int32_t* indices, const double* y_re,
                 const double* y_im, int32_t ref, const int32_t* pv, int32_t n_pv,
                 const int32_t* pq, int32_t n_pq, const double* vm0, const double* va0,
                 double pivot_tol, int32_t bulk_min_entries);
};

}  // namespace gbnr
