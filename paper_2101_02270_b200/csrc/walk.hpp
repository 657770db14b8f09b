// walk.hpp -- tile-owned sequential walks over the frozen LU (host plans).
//
// The level-scheduled refactorization of PAPER.md Alg. 3 / SPEC.md:319-327
// launches once per level and reads every L(:,k) from HBM once per dependent
// column.  On B200 the batch is only ~313 tiles of 32 scenarios, so instead
// each tile is walked by ONE warp through all columns in elimination order
// (a topological order of the column DAG, so Alg. 2's per-element operation
// order is unchanged and results stay bit-identical):
//
//   * forward walk  = refactorize_batch fused with the
//                     forward substitution of fs_bs_batch:
//                     at column m the dependencies k ascending are exactly
//                     the columns whose L(:,k) holds L(m,k) (structurally
//                     symmetric J), so y_m = b_m - sum_k L(m,k) y_k rides along;
//   * backward walk = the backward substitution, rows in reverse order over a
//                     row-major copy of U written by the forward walk.
//
// Shared memory holds a ring of recently produced column blocks and a staging
// ring; all global->shared movement is cp.async.bulk (TMA) into mbarrier-
// tracked slots.  The plan below is the complete, static program of those
// copies: which step's data lives where in shared memory, which dependency is
// still resident in the ring (most are: AMD puts a column's dependencies just
// before it) and which must be re-fetched, and after which consumer event each
// copy may be issued.  It is computed once per plan on the host, shared by all
// tiles, and verified by a host simulation before it is ever launched.
#pragma once

#include <cstdint>
#include <vector>

#include "symbolic.hpp"

namespace gbnr {

enum : int32_t { kTapeA = 0, kTapeLU = 1, kTapeB = 2 };

// One step (LU column / BS row).
struct WStep {
    int32_t ring;    // smem row of the step's block
    int32_t len_dp;  // forward: len | dp << 16; backward: number of U entries
    int32_t dep0;    // first WDep
    int32_t ndep;    // number of WDep
    int32_t lslot;   // LU-tape slot of the first L row (L rows, then y)
    int32_t ut0;     // forward: first index into the U-scatter list (dp entries)
    int32_t op;      // op carrying the block
    int32_t brow;    // b-tape row of the step (LU row / column index)
    int32_t global = 0;  // block in global memory (too large for the walker's pool)
    int32_t gslot = 0;   // global step: A-tape slot of the column (fwd) / LU-tape slot of the row (bwd)
};
// One dependency of a step.  32 B.
struct WDep {
    int32_t kpos_fs;  // forward: kpos | fspos << 16 (0xffff = none)
    int32_t nrows;    // forward: rows of L(:,k) applied (0 = FS-only)
    int32_t src;      // smem row of L(:,k) (forward) / of nothing (backward)
    int32_t ysrc;     // smem row of y_k (forward) / x_k (backward)
    int32_t u0;       // forward: first destination record
    int32_t op;       // op to wait on, -1 = resident in the ring
    int32_t global;   // source read from global memory (too large to stage)
    int32_t gslot;    // global source: LU-tape slot of L(:,k) (fwd) / b-tape row of x_k (bwd)
    int32_t gnl;      // global source (fwd): rows of L(:,k) (y_k follows them)
    int32_t prod = -1;  // producing step of this walker's program (-1: earlier phase / walker)
};
// One TMA bulk copy: nrows rows of tape `tape` from slot/row `slot` (a row is one
// value per task of a tile: tile width x 8 bytes).
struct WCopy {
    int32_t tape_rows;  // tape | nrows << 8
    int32_t slot;
    int32_t smem;       // destination smem row
    int32_t pad;
};
struct WOp {
    int32_t after;  // issue once the consumer has passed this event (-1 = prologue)
    int32_t ncopy;
    int32_t bytes;  // expect_tx total in rows (the kernel multiplies by its row bytes)
    int32_t c0;     // first copy in Walk::copies
};

struct WalkConfig {
    int32_t walkers = 8;          // K: warps per tile walking disjoint etree subtrees
    int32_t smem_budget = 76800;  // bytes per CTA: three tiles per SM (228 KB - 3 x 1 KB reserved)
    int32_t row_bytes = 256;      // bytes per shared / tape row: tile width x 8
    int32_t ring_rows = 0;        // per-walker ring override (0 = from the budget)
    int32_t stage_rows = 0;       // per-walker staging override (0 = from the budget)
    int32_t barriers = 32;        // mbarriers per walker (op i uses barrier i % 32)
    int32_t prefetch = 8;         // steps an op may run ahead of its consumer
    int32_t headroom = 1;         // ring residency margin (steps) before an overwrite
    int32_t page_words = 128;     // program-stream page (grown to the longest record)
    int32_t pages = 2;            // program-stream pages resident per walker
    double balance = 1.5;         // split subtrees heavier than total / (walkers * balance)
    double stage_frac = 0.45;     // staging share of a walker's rows (split plan; the
                                  // subtree partition sizes columns against it too)
    double stage_frac_up = 0.3;   // staging share above level 0 (< 0: stage_frac)
    double global_frac = 0.0;     // > 0: also stage in global memory every block larger than
                                  // this share of the pool and every fetch larger than half
                                  // of it (tests; columns that cannot be planned in shared
                                  // memory go global regardless)
    std::vector<int32_t> levels;  // walkers per level (empty: walkers, walkers/2, ..., 1)
    bool pairs = true;            // backward: independent consecutive rows in one kRecPair
    bool unified = true;          // blocks and fetches share one pool (plan_unified;
                                  // the split ring / staging plan where it is infeasible)
};

// The device program of a walk: per walker one int32 word stream the warp
// interprets in order, streamed through shared memory in pages by TMA.
// Records (word 0 low 4 bits = type) never straddle a page; kRecPage moves to
// the next page, kRecSync is a CTA barrier between phases.
enum : int32_t {
    kRecIssue = 1,  // 1 | ncopy << 4, op, bytes, {tape | rows << 2 | smem << 12, slot} x ncopy
    kRecStep = 2,   // 2 | ndep << 4, ring | len << 16 (fwd) / ring | ne << 16 (bwd), dp, lslot, brow, op
    kRecDep = 3,    // fwd: 3 | (op + 1) << 4, kpos_fs, nrows | src << 16, ysrc, dst u16 pairs
                    // bwd: 3 | (op + 1) << 4, ysrc
    kRecEnd = 4,    // 4 | dp << 4, U-CRS tape slots [dp] (fwd)
    kRecPage = 5,
    kRecDone = 6,
    kRecSync = 7,
    // fwd: two dependencies k, k+1 of one supernode (L(:,k) = {k+1} u L(:,k+1)),
    // applied in one pass over x: 8 | (op + 1) << 4, kpos1 | kpos2 << 16,
    // nrows2 | src1 << 16, src2 | fspos1 << 16, ysrc1 | ysrc2 << 16, fspos2 | (op2 + 1) << 16,
    // dst u16 pairs of L(:,k+1) (padded to 4)
    kRecDep2 = 8,
    // bwd: n consecutive dependencies, only the first may wait:
    // 9 | (op + 1) << 4, n, ysrc u16 pairs
    kRecDepN = 9,
    // Global-memory forms for columns / rows too large for a walker's pool (the
    // same operation order per element, data in the tile's global scratch / tapes):
    // fwd: 10 | ndep << 4, len | dp << 16, A slot, lslot, brow       (column -> scratch)
    // bwd: 10 | ndep << 4, ne, LU slot of the row block, brow
    kRecStepG = 10,
    // fwd: 11 | (op + 1) << 4, kpos_fs, nrows, src, nl, dst u16 pairs (padded to 2);
    //      src < 0: L(:,k) at LU-tape slot -src-1 (y_k nl rows further), else a shared
    //      row (y_k at src + nl); x = the step's block (shared or scratch).  A dependency
    //      may continue in further records (kpos only, no FS role).
    kRecDepG = 11,
    kRecEndG = 12,   // fwd: 12 (normalise the L part, flag, y); bwd: 12
    // fwd: 13 | cnt << 4, z0, U-CRS slots [cnt]: scatter U entries z0.. of a global step
    kRecEndU = 13,
    // bwd: 14 | n << 4, b-tape rows of x_k [n] (global row block, x_k from the b tape)
    kRecDepNG = 14,
    // bwd: two consecutive independent rows A, B in one record (their dependency
    // chains interleave; every op they wait for is issued before it):
    // 15 | nA << 4 | nw << 16, ringA | neA << 16, ringB | neB << 16, browA, browB,
    // (opA + 1) | (opB + 1) << 16, nB, (dep op + 1) x nw, ysrc u16 pairs of A, of B
    kRecPair = 15,
};
constexpr int32_t kMaxPageWords = 256;  // longer records are split (global forms)

// One verified single-walker program (one walker in one phase).
struct Walk {
    int32_t ring_base = 0, ring_rows = 0, stage_rows = 0, barriers = 0, n_steps = 0;
    int32_t global_steps = 0, global_deps = 0, scratch_rows = 0;
    std::vector<WStep> step;
    std::vector<WDep> dep;
    std::vector<uint16_t> dst;  // forward: destination position per applied L row
    std::vector<WOp> op;
    std::vector<WCopy> copies;
    std::vector<int32_t> ut;    // forward: U-part CCS slot -> U-CRS tape slot (by step)
    int64_t events = 0, ring_dep_rows = 0, fetched_rows = 0, block_rows = 0;
};

// All walkers of one tile, all phases: what a kernel launch runs.
struct WalkSet {
    int32_t walkers = 1, phases = 1, rows = 0, page_words = 0, pages = 0, barriers = 0, row_bytes = 256;
    std::vector<Walk> parts;        // [phase * walkers + w]
    std::vector<int32_t> stream;    // every walker's pages, walker-major
    std::vector<int32_t> wpage0;    // [walkers + 1] first page of each walker
    std::vector<int32_t> owner;     // column / row -> level * 16 + walker
    int64_t steps = 0, events = 0, ring_dep_rows = 0, fetched_rows = 0, n_ops = 0, n_copies = 0;
    int64_t global_steps = 0, global_deps = 0;
    int32_t scratch_rows = 0;       // per-tile global scratch rows (forward global steps)
    size_t smem_bytes() const {
        return size_t(rows) * size_t(row_bytes) +
               size_t(walkers) * (size_t(pages) * page_words * 4 + size_t(barriers + pages) * 8);
    }
};

// LU tape layout of the walks: the L+diag part of every column contiguous
// (column-major, diagonal first) followed by U row-major (each row's entries in
// descending column order, the backward walk's consumption order).
// Tape layouts (rows of 256 B = 32 lanes), each sized so one walk copy moves a
// whole block:
//   A tape  column m: its CCS entries, then F_m           (slots cp[m] + m ...)
//   LU tape column k: L rows, then y_k                     (lslot[k] ...)
//           row i:    U entries (k descending), y_i, U(i,i) (ucrs0[i] ...)
// so a step block, a re-fetched dependency (L rows + y) and a backward block
// are one contiguous copy each, and the dependencies k, k+1 re-fetched side by
// side merge into one copy.
struct LuLayout {
    std::vector<int32_t> lslot;        // [nJ] slot of the first L row of column k
    std::vector<int32_t> ucrs0;        // [nJ+1] first U-CRS slot of row i (then y_i, U(i,i))
    std::vector<int32_t> tape_of_ccs;  // [nnzLU] CCS slot -> tape slot
    int32_t rows = 0;                  // LU tape rows: nnzLU + 2 nJ
};
// A tape slot of CCS entry z of column j / of F_m
inline int32_t a_slot(int32_t z, int32_t j) { return z + j; }

LuLayout build_lu_layout(const Symbolic& s);
// Columns -> (level, walker) by splitting the elimination tree into whole
// subtrees that fit a walker's shared-memory share, level by level with
// halving walker counts; false if dependencies would cross walkers
// (unsymmetric pivoting), in which case one walker is used.
bool partition_levels(const Symbolic& s, const WalkConfig& cfg, const std::vector<int32_t>& lvl_walkers,
                      const std::vector<int32_t>& ring_w, const std::vector<int32_t>& stage_w, bool backward,
                      std::vector<int32_t>& level, std::vector<int32_t>& bin);
WalkSet build_forward_walk(const Symbolic& s, const LuLayout& lay, bool with_fs, const WalkConfig& cfg);
WalkSet build_backward_walk(const Symbolic& s, const LuLayout& lay, const WalkConfig& cfg);

}  // namespace gbnr
