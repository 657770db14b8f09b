// symbolic.cpp -- one-time host analysis for the batched NR solver (see symbolic.hpp).
#include "symbolic.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <functional>
#include <numbers>
#include <queue>
#include <utility>

#include "numerics.cuh"

namespace gbnr {

namespace {

using cplx = std::complex<double>;

// Sorted, de-duplicated CRS pattern from packed (row * n_cols + col) keys.
void crs_from_keys(int32_t n_rows, int32_t n_cols, std::vector<int64_t>& keys,
                   std::vector<int32_t>& rp, std::vector<int32_t>& ci) {
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    rp.assign(static_cast<size_t>(n_rows) + 1, 0);
    ci.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        rp[keys[i] / n_cols + 1]++;
        ci[i] = static_cast<int32_t>(keys[i] % n_cols);
    }
    for (int32_t r = 0; r < n_rows; ++r) rp[r + 1] += rp[r];
}

int32_t find_sorted(const std::vector<int32_t>& idx, int32_t lo, int32_t hi, int32_t key) {
    auto first = idx.begin() + lo, last = idx.begin() + hi;
    auto it = std::lower_bound(first, last, key);
    return (it != last && *it == key) ? static_cast<int32_t>(it - idx.begin()) : -1;
}

}  // namespace

// ---------------------------------------------------------------------------
// Ybus with the MATPOWER branch model; std::complex arithmetic so the values
// round exactly like grid.hpp:195-243.
// ---------------------------------------------------------------------------
YbusCsr build_ybus(int32_t n, int32_t nbr, const int32_t* f, const int32_t* t, const double* r,
                   const double* x, const double* b, const double* tap, const double* shift_deg,
                   const uint8_t* on, const double* gs, const double* bs, double base_mva) {
    if (n <= 0) throw Error(3, "n_bus must be positive");
    std::vector<int64_t> keys;
    keys.reserve(2 * static_cast<size_t>(nbr) + n);
    for (int32_t k = 0; k < nbr; ++k) {
        if (f[k] < 0 || f[k] >= n || t[k] < 0 || t[k] >= n)
            throw Error(2, "branch " + std::to_string(k) + " endpoint out of range");
        keys.push_back(int64_t(f[k]) * n + t[k]);
        keys.push_back(int64_t(t[k]) * n + f[k]);
    }
    for (int32_t i = 0; i < n; ++i) keys.push_back(int64_t(i) * n + i);
    YbusCsr y;
    y.n = n;
    crs_from_keys(n, n, keys, y.indptr, y.indices);
    const size_t nnz = y.indices.size();
    std::vector<cplx> v(nnz, cplx(0.0, 0.0));
    y.diag.resize(n);
    for (int32_t i = 0; i < n; ++i) y.diag[i] = find_sorted(y.indices, y.indptr[i], y.indptr[i + 1], i);
    y.slot.resize(4 * static_cast<size_t>(nbr));
    y.adm.resize(8 * static_cast<size_t>(nbr));
    for (int32_t k = 0; k < nbr; ++k) {
        cplx ff(0.0, 0.0), ft(0.0, 0.0), tf(0.0, 0.0), tt(0.0, 0.0);
        if (on[k]) {
            const cplx ys = 1.0 / cplx(r[k], x[k]);
            const cplx ysh(0.0, b[k] / 2.0);
            const cplx tc = std::polar(tap[k], shift_deg[k] * std::numbers::pi_v<double> / 180.0);
            tt = ys + ysh;
            ff = (ys + ysh) / (tap[k] * tap[k]);
            ft = -ys / std::conj(tc);
            tf = -ys / tc;
        }
        const int32_t sl[4] = {y.diag[f[k]], find_sorted(y.indices, y.indptr[f[k]], y.indptr[f[k] + 1], t[k]),
                               find_sorted(y.indices, y.indptr[t[k]], y.indptr[t[k] + 1], f[k]), y.diag[t[k]]};
        const cplx a[4] = {ff, ft, tf, tt};
        for (int q = 0; q < 4; ++q) {
            v[sl[q]] += a[q];
            y.slot[4 * size_t(k) + q] = sl[q];
            y.adm[8 * size_t(k) + 2 * q] = a[q].real();
            y.adm[8 * size_t(k) + 2 * q + 1] = a[q].imag();
        }
    }
    for (int32_t i = 0; i < n; ++i) v[y.diag[i]] += cplx(gs[i], bs[i]) / base_mva;
    y.re.resize(nnz);
    y.im.resize(nnz);
    for (size_t s = 0; s < nnz; ++s) {
        y.re[s] = v[s].real();
        y.im[s] = v[s].imag();
    }
    return y;
}

// ---------------------------------------------------------------------------
// N-1 contingency value sets on the fixed pattern: ybus_values_with_outage
// (grid.hpp:245-255) -- the outaged branch's four contributions subtracted from
// the base values, complex arithmetic as the reference -- and the islanding
// pre-check outage_islands_grid (grid.hpp:257-261): an in-service branch whose
// removal disconnects the grid is a bridge (one Tarjan pass, parallel branches
// counted as distinct edges).
// ---------------------------------------------------------------------------
void contingency_values(const YbusCsr& y, int32_t nbr, const int32_t* f, const int32_t* t, const uint8_t* on,
                        const int32_t* outage, int32_t n_tasks, double* y_re, double* y_im, uint8_t* islanded) {
    const int32_t n = y.n;
    const size_t nnz = y.indices.size(), T = size_t(n_tasks);
    // bridges of the in-service branch graph
    std::vector<uint8_t> bridge(nbr, 0);
    {
        std::vector<std::vector<std::pair<int32_t, int32_t>>> adj(n);  // (neighbour, branch)
        for (int32_t k = 0; k < nbr; ++k)
            if (on[k] && f[k] != t[k]) {
                adj[f[k]].emplace_back(t[k], k);
                adj[t[k]].emplace_back(f[k], k);
            }
        std::vector<int32_t> disc(n, -1), low(n, 0), it(n, 0), via(n, -1), stack;
        int32_t timer = 0;
        for (int32_t root = 0; root < n; ++root) {
            if (disc[root] >= 0) continue;
            disc[root] = low[root] = timer++;
            stack.push_back(root);
            while (!stack.empty()) {  // iterative DFS (grids are deep)
                const int32_t u = stack.back();
                if (it[u] < int32_t(adj[u].size())) {
                    const auto [w, k] = adj[u][it[u]++];
                    if (k == via[u]) continue;
                    if (disc[w] < 0) {
                        disc[w] = low[w] = timer++;
                        via[w] = k;
                        stack.push_back(w);
                    } else {
                        low[u] = std::min(low[u], disc[w]);
                    }
                } else {
                    stack.pop_back();
                    if (!stack.empty()) {
                        const int32_t p = stack.back();
                        low[p] = std::min(low[p], low[u]);
                        if (low[u] > disc[p]) bridge[via[u]] = 1;
                    }
                }
            }
        }
    }
    for (size_t task = 0; task < T; ++task) {
        const int32_t k = outage[task];
        if (k >= nbr) throw Error(2, "outage branch out of range");
        for (size_t q = 0; q < nnz; ++q) {
            y_re[q * T + task] = y.re[q];
            y_im[q * T + task] = y.im[q];
        }
        if (islanded) islanded[task] = k >= 0 && on[k] && bridge[k];
        if (k < 0 || !on[k]) continue;  // no outage / out-of-service branch: the base values
        for (int c = 0; c < 4; ++c) {
            const size_t q = size_t(y.slot[4 * size_t(k) + c]);
            const cplx v = cplx(y.re[q], y.im[q]) - cplx(y.adm[8 * size_t(k) + 2 * c], y.adm[8 * size_t(k) + 2 * c + 1]);
            y_re[q * T + task] = v.real();
            y_im[q * T + task] = v.imag();
        }
    }
}

// ---------------------------------------------------------------------------
// Approximate minimum degree, same semantics as amd.hpp:29-157 (quotient
// graph, the three-way approximate external degree bound, no supervariables,
// minimum (degree, index) pivot).  Min-heap with lazy invalidation.
// ---------------------------------------------------------------------------
std::vector<int32_t> amd_order(int32_t n, const int32_t* col_ptr, const int32_t* row_ix) {
    std::vector<int32_t> fwd(static_cast<size_t>(n));
    if (n == 0) return fwd;
    std::vector<std::vector<int32_t>> A(n), E(n), Le(n);
    for (int32_t c = 0; c < n; ++c)
        for (int32_t p = col_ptr[c]; p < col_ptr[c + 1]; ++p) {
            const int32_t r = row_ix[p];
            if (r == c) continue;
            A[c].push_back(r);
            A[r].push_back(c);
        }
    std::vector<int32_t> deg(n), mark(n, 0), w(n, 0);
    std::vector<uint8_t> dead(n, 0), elem(n, 0);
    using Key = std::pair<int32_t, int32_t>;
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> pq;
    for (int32_t i = 0; i < n; ++i) {
        std::sort(A[i].begin(), A[i].end());
        A[i].erase(std::unique(A[i].begin(), A[i].end()), A[i].end());
        deg[i] = static_cast<int32_t>(A[i].size());
        pq.emplace(deg[i], i);
    }
    int32_t tag = 0;
    std::vector<int32_t> lp;
    for (int32_t k = 0; k < n; ++k) {
        int32_t p;
        for (;;) {
            const Key top = pq.top();
            pq.pop();
            p = top.second;
            if (!dead[p] && deg[p] == top.first) break;
        }
        dead[p] = 1;
        fwd[p] = k;
        ++tag;
        lp.clear();
        mark[p] = tag;
        auto take = [&](int32_t v) {
            if (dead[v] || mark[v] == tag) return;
            mark[v] = tag;
            lp.push_back(v);
        };
        for (int32_t v : A[p]) take(v);
        for (int32_t e : E[p]) {
            if (!elem[e]) continue;
            for (int32_t v : Le[e]) take(v);
            elem[e] = 0;
            Le[e].clear();
        }
        std::sort(lp.begin(), lp.end());
        for (int32_t i : lp)
            for (int32_t e : E[i]) {
                if (!elem[e]) continue;
                if (mark[e] != tag) {
                    mark[e] = tag;
                    std::erase_if(Le[e], [&](int32_t v) { return dead[v] != 0; });
                    w[e] = static_cast<int32_t>(Le[e].size());
                }
                --w[e];
            }
        const int32_t alive = n - k - 1;
        const int32_t grow = static_cast<int32_t>(lp.size()) - 1;
        for (int32_t i : lp) {
            std::erase_if(A[i], [&](int32_t v) { return v == p || dead[v] || mark[v] == tag; });
            int32_t esum = 0;
            std::erase_if(E[i], [&](int32_t e) {
                if (!elem[e]) return true;
                esum += std::max(w[e], 0);
                return false;
            });
            E[i].push_back(p);
            int32_t d = std::min({alive, deg[i] + grow,
                                  static_cast<int32_t>(A[i].size()) + grow + esum});
            d = std::max(d, 0);
            deg[i] = d;
            pq.emplace(d, i);
        }
        A[p].clear();
        E[p].clear();
        elem[p] = 1;
        Le[p] = lp;
    }
    return fwd;
}

// ---------------------------------------------------------------------------
// Symbolic::analyze
// ---------------------------------------------------------------------------
void Symbolic::analyze(int32_t n_bus, const int32_t* indptr, const int32_t* indices,
                       const double* y_re, const double* y_im, int32_t ref_bus, const int32_t* pv,
                       int32_t n_pv, const int32_t* pq, int32_t n_pq, const double* vm0,
                       const double* va0, double pivot_tol) {
    n = n_bus;
    ref = ref_bus;
    npv = n_pv;
    npq = n_pq;
    npvpq = npv + npq;
    nJ = npv + 2 * npq;
    if (n <= 0 || ref < 0 || ref >= n) throw Error(3, "bad n_bus / ref");
    if (indptr[0] != 0) throw Error(2, "Ybus indptr[0] != 0");
    nnzY = indptr[n];
    yp.assign(indptr, indptr + n + 1);
    yi.assign(indices, indices + nnzY);
    for (int32_t r = 0; r < n; ++r) {
        if (yp[r] > yp[r + 1]) throw Error(2, "Ybus indptr not monotone");
        bool has_diag = false;
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            if (yi[q] < 0 || yi[q] >= n) throw Error(2, "Ybus column index out of range");
            if (q > yp[r] && yi[q] <= yi[q - 1]) throw Error(2, "Ybus columns not strictly increasing");
            has_diag |= yi[q] == r;
        }
        if (!has_diag) throw Error(2, "Ybus row " + std::to_string(r) + " lacks a structural diagonal");
    }
    jth.assign(n, -1);
    jvm.assign(n, -1);
    for (int32_t i = 0; i < npv; ++i) {
        if (pv[i] < 0 || pv[i] >= n || jth[pv[i]] >= 0) throw Error(2, "bad pv index");
        jth[pv[i]] = i;
    }
    for (int32_t i = 0; i < npq; ++i) {
        if (pq[i] < 0 || pq[i] >= n || jth[pq[i]] >= 0) throw Error(2, "bad pq index");
        jth[pq[i]] = npv + i;
        jvm[pq[i]] = npvpq + i;
    }
    if (jth[ref] >= 0 || npvpq != n - 1) throw Error(2, "pv / pq / ref must partition the buses");

    // ---- reduced Jacobian pattern: 4 Ybus-shaped blocks, filtered ----
    std::vector<int64_t> keys;
    keys.reserve(4 * static_cast<size_t>(nnzY) + nJ);
    for (int32_t r = 0; r < n; ++r)
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            const int32_t k = yi[q];
            const int32_t rr[2] = {jth[r], jvm[r]}, cc[2] = {jth[k], jvm[k]};
            for (int a = 0; a < 2; ++a)
                for (int c = 0; c < 2; ++c)
                    if (rr[a] >= 0 && cc[c] >= 0) keys.push_back(int64_t(rr[a]) * nJ + cc[c]);
        }
    for (int32_t i = 0; i < nJ; ++i) keys.push_back(int64_t(i) * nJ + i);
    std::vector<int32_t> jp, ji;
    crs_from_keys(nJ, nJ, keys, jp, ji);
    nnzJ = static_cast<int64_t>(ji.size());
    // CCS of J (transpose) with crs -> ccs slot map
    std::vector<int32_t> jcp(nJ + 1, 0), jri(ji.size()), j2c(ji.size());
    for (int32_t c : ji) jcp[c + 1]++;
    for (int32_t c = 0; c < nJ; ++c) jcp[c + 1] += jcp[c];
    {
        std::vector<int32_t> nx(jcp.begin(), jcp.end() - 1);
        for (int32_t r = 0; r < nJ; ++r)
            for (int32_t s = jp[r]; s < jp[r + 1]; ++s) {
                const int32_t slot = nx[ji[s]]++;
                jri[slot] = r;
                j2c[s] = slot;
            }
    }
    // quadrant -> J CRS slot
    std::vector<int32_t> jslot(4 * static_cast<size_t>(nnzY), -1);
    for (int32_t r = 0; r < n; ++r)
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            const int32_t k = yi[q];
            const int32_t rr[2] = {jth[r], jvm[r]}, cc[2] = {jth[k], jvm[k]};
            for (int a = 0; a < 2; ++a)
                for (int c = 0; c < 2; ++c)
                    if (rr[a] >= 0 && cc[c] >= 0)
                        jslot[4 * size_t(q) + 2 * a + c] = find_sorted(ji, jp[rr[a]], jp[rr[a] + 1], cc[c]);
        }

    // ---- ordering ----
    col_fwd = amd_order(nJ, jcp.data(), jri.data());
    std::vector<int32_t> amd_inv(nJ);
    for (int32_t i = 0; i < nJ; ++i) amd_inv[col_fwd[i]] = i;

    // ---- representative Jacobian values (task 0 at V0), CCS order ----
    std::vector<double> c0(n), s0(n);
    for (int32_t i = 0; i < n; ++i) gb_sincos(va0[i], &s0[i], &c0[i]);
    std::vector<double> jval(ji.size(), 0.0);
    for (int32_t r = 0; r < n; ++r) {
        if (r == ref) continue;
        double ire = 0.0, iim = 0.0;
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            const int32_t k = yi[q];
            acc_current(y_re[q], y_im[q], vm0[k] * c0[k], vm0[k] * s0[k], ire, iim);
        }
        const double vre = vm0[r] * c0[r], vim = vm0[r] * s0[r];
        double P, Q;
        injection(vre, vim, ire, iim, P, Q);
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            const int32_t k = yi[q];
            double zre, zim, jv[4];
            jac_z(y_re[q], y_im[q], vre, vim, c0[k], s0[k], zre, zim);
            jac_entries(k == r, zre, zim, vm0[k], c0[k], s0[k], ire, iim, P, Q, jv);
            for (int a = 0; a < 4; ++a) {
                const int32_t js = jslot[4 * size_t(q) + a];
                if (js >= 0) jval[j2c[js]] = jv[a];
            }
        }
    }

    // ---- left-looking G-P with threshold partial pivoting ----
    // L columns are kept with J-row ids until every row has a pivot position;
    // numeric updates run in ascending pivot order (a topological order of L),
    // the same canonical order the oracle and the refactorization use.
    std::vector<int32_t> pinv(nJ, -1);
    std::vector<std::vector<int32_t>> Lr(nJ), Ur(nJ);
    std::vector<std::vector<double>> Lv(nJ);
    std::vector<double> x(nJ, 0.0);
    std::vector<int32_t> seen(nJ, -1), reach;
    std::vector<std::pair<int32_t, int32_t>> piv_rows;
    reach.reserve(nJ);
    offdiag_piv = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        const int32_t colj = amd_inv[k];
        reach.clear();
        for (int32_t q = jcp[colj]; q < jcp[colj + 1]; ++q)
            if (seen[jri[q]] != k) {
                seen[jri[q]] = k;
                reach.push_back(jri[q]);
            }
        for (size_t h = 0; h < reach.size(); ++h) {
            const int32_t i = reach[h];
            if (pinv[i] < 0) continue;
            for (int32_t v : Lr[pinv[i]])
                if (seen[v] != k) {
                    seen[v] = k;
                    reach.push_back(v);
                }
        }
        for (int32_t i : reach) x[i] = 0.0;
        for (int32_t q = jcp[colj]; q < jcp[colj + 1]; ++q) x[jri[q]] = jval[q];
        piv_rows.clear();
        for (int32_t i : reach)
            if (pinv[i] >= 0) piv_rows.emplace_back(pinv[i], i);
        std::sort(piv_rows.begin(), piv_rows.end());
        for (const auto& [j, row] : piv_rows) {
            const double xj = x[row];
            for (size_t z = 0; z < Lr[j].size(); ++z) x[Lr[j][z]] = fma(-xj, Lv[j][z], x[Lr[j][z]]);
            Ur[k].push_back(row);
        }
        int32_t ipiv = -1;
        double amax = -1.0;
        for (int32_t i : reach) {
            if (pinv[i] >= 0) continue;
            const double a = std::fabs(x[i]);
            if (a > amax || (a == amax && ipiv >= 0 && i < ipiv)) {
                amax = a;
                ipiv = i;
            }
        }
        if (ipiv < 0) throw Error(2, "structurally singular Jacobian column " + std::to_string(k));
        if (!(amax > 0.0)) throw Error(4, "numerically singular pivot in column " + std::to_string(k));
        const int32_t idiag = amd_inv[k];
        if (pinv[idiag] < 0 && seen[idiag] == k && std::fabs(x[idiag]) >= pivot_tol * amax) ipiv = idiag;
        if (ipiv != idiag) ++offdiag_piv;
        const double piv = x[ipiv];
        pinv[ipiv] = k;
        for (int32_t i : reach) {
            if (pinv[i] >= 0) continue;
            Lr[k].push_back(i);
            Lv[k].push_back(x[i] / piv);
        }
    }
    row_fwd = pinv;

    // ---- frozen LU pattern in pivot numbering ----
    cp.assign(nJ + 1, 0);
    for (int32_t k = 0; k < nJ; ++k) cp[k + 1] = cp[k] + int32_t(Ur[k].size() + 1 + Lr[k].size());
    nnzLU = cp[nJ];
    ri.resize(nnzLU);
    dpos.resize(nJ);
    nnzL = nnzU = 0;
    max_col = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        int32_t* dst = ri.data() + cp[k];
        int32_t m = 0;
        for (int32_t v : Ur[k]) dst[m++] = pinv[v];
        dst[m++] = k;
        for (int32_t v : Lr[k]) dst[m++] = pinv[v];
        std::sort(dst, dst + m);
        dpos[k] = cp[k] + int32_t(std::find(dst, dst + m, k) - dst);
        nnzU += Ur[k].size();
        nnzL += Lr[k].size();
        max_col = std::max(max_col, m);
    }
    if (max_col >= 65536) throw Error(3, "LU column longer than 65535 entries");

    // ---- lookup: Ybus slot quadrant -> LU slot of the A tape (fill slots are never
    //      written and stay zero); aidx marks the J-fed slots (-1 = fill) ----
    std::vector<int32_t> jslot_to_lu(ji.size(), -1);
    for (int32_t r = 0; r < nJ; ++r)
        for (int32_t s = jp[r]; s < jp[r + 1]; ++s) {
            const int32_t ar = row_fwd[r], ac = col_fwd[ji[s]];
            const int32_t slot = find_sorted(ri, cp[ac], cp[ac + 1], ar);
            if (slot < 0) throw Error(2, "Jacobian entry missing from the frozen LU pattern");
            jslot_to_lu[s] = slot;
        }
    aidx.assign(nnzLU, -1);
    for (int32_t s : jslot_to_lu) aidx[s] = 0;
    int32_t na = 0;
    for (int64_t s = 0; s < nnzLU; ++s)
        if (aidx[s] == 0) aidx[s] = na++;
    lk.assign(4 * static_cast<size_t>(nnzY), -1);
    for (size_t q = 0; q < jslot.size(); ++q)
        if (jslot[q] >= 0) lk[q] = jslot_to_lu[jslot[q]];

    // ---- levels ----
    level.assign(nJ, 0);
    std::vector<int32_t> fl(nJ, 0), bl(nJ, 0);
    levels_lu = levels_fs = levels_bs = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        int32_t l = 0;
        for (int32_t z = cp[k]; z < dpos[k]; ++z) l = std::max(l, level[ri[z]] + 1);
        level[k] = l;
        levels_lu = std::max(levels_lu, l + 1);
        levels_fs = std::max(levels_fs, fl[k] + 1);
        for (int32_t z = dpos[k] + 1; z < cp[k + 1]; ++z) fl[ri[z]] = std::max(fl[ri[z]], fl[k] + 1);
    }
    for (int32_t k = nJ - 1; k >= 0; --k) {
        levels_bs = std::max(levels_bs, bl[k] + 1);
        for (int32_t z = cp[k]; z < dpos[k]; ++z) bl[ri[z]] = std::max(bl[ri[z]], bl[k] + 1);
    }
    // ---- VMAD count D = sum over U dependencies k of |L(:,k)| ----
    D = 0;
    max_udeps = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        max_udeps = std::max(max_udeps, dpos[k] - cp[k]);
        for (int32_t z = cp[k]; z < dpos[k]; ++z) {
            const int32_t j = ri[z];
            D += cp[j + 1] - dpos[j] - 1;
        }
    }

    // ---- NPM / J row list, b rows and z columns per bus ----
    rows.clear();
    brow_p.assign(n, -1);
    brow_q.assign(n, -1);
    zcol_t.assign(n, -1);
    zcol_v.assign(n, -1);
    // Row order of the NPM / Jacobian sweeps: reverse Cuthill-McKee on the Ybus
    // graph, so a block's 32 consecutive rows share neighbours and the
    // neighbours' voltage rows are re-read from L2 (results do not depend on
    // it: rows are independent and the max-norm is order-free).
    std::vector<int32_t> order;
    {
        std::vector<uint8_t> seen(n, 0);
        std::vector<int32_t> deg(n);
        for (int32_t i = 0; i < n; ++i) deg[i] = yp[i + 1] - yp[i];
        std::vector<int32_t> by_deg(n);
        for (int32_t i = 0; i < n; ++i) by_deg[i] = i;
        std::stable_sort(by_deg.begin(), by_deg.end(), [&](int32_t a, int32_t b) { return deg[a] < deg[b]; });
        for (int32_t start : by_deg) {
            if (seen[start]) continue;
            size_t head = order.size();
            order.push_back(start);
            seen[start] = 1;
            while (head < order.size()) {
                const int32_t u = order[head++];
                const size_t first = order.size();
                for (int32_t q = yp[u]; q < yp[u + 1]; ++q)
                    if (!seen[yi[q]]) {
                        seen[yi[q]] = 1;
                        order.push_back(yi[q]);
                    }
                std::stable_sort(order.begin() + first, order.end(),
                                 [&](int32_t a, int32_t b) { return deg[a] < deg[b]; });
            }
        }
        std::reverse(order.begin(), order.end());
    }
    for (int32_t b : order) {
        if (b == ref) continue;
        rows.push_back(b);
    }
    for (int32_t b = 0; b < n; ++b) {
        if (b == ref) continue;
        brow_p[b] = row_fwd[jth[b]];
        zcol_t[b] = col_fwd[jth[b]];
        if (jvm[b] >= 0) {
            brow_q[b] = row_fwd[jvm[b]];
            zcol_v[b] = col_fwd[jvm[b]];
        }
    }
}

}  // namespace gbnr
