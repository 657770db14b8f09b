// walk.cpp -- host planner of the tile-owned LU/FS and BS walks (see walk.hpp).
#include "walk.hpp"

#include <algorithm>
#include <deque>
#include <limits>
#include <queue>
#include <string>

namespace gbnr {

namespace {

constexpr int32_t kInf = std::numeric_limits<int32_t>::max();

WCopy copy(int32_t tape, int32_t slot, int32_t rows, int32_t smem_rel) {
    return WCopy{tape | (rows << 8), slot, smem_rel, 0};
}
int32_t copy_rows(const WCopy& c) { return c.tape_rows >> 8; }

// What a step loads into its own ring block, and what each dependency needs.
struct DepIn {
    int32_t producer;        // producing step of the same program, -1 = external
                             // (an earlier phase / another walker: always re-fetched)
    int32_t ring_src = -1;   // rows relative to the producer's block
    int32_t ring_ysrc = -1;
    std::vector<WCopy> fetch;  // copies relative to a staging allocation
    int32_t fetch_rows = 0;
    int32_t stage_src = -1, stage_ysrc = -1;
    bool global = false;       // read from global memory, never staged
    WDep rec{};                // payload fields (kpos_fs, nrows, u0, gslot, gnl)
};
struct StepIn {
    int32_t blk_rows = 0;
    std::vector<WCopy> copies;  // smem relative to the block
    std::vector<DepIn> deps;
    bool global = false;        // block in global memory (scratch / the LU tape)
    int32_t global_rows = 0;    // forward: scratch rows a global block needs
    WStep rec{};                // payload fields (len_dp, lslot, ut0, brow, gslot)
};
// A walker's program before planning: its steps and their payload arrays.
struct Program {
    std::vector<StepIn> steps;
    std::vector<uint16_t> dst;
    std::vector<int32_t> ut;
};

struct PlanCfg {
    int32_t ring_base, ring_rows, stage_rows, barriers, prefetch, headroom, max_copies;
};

// Allocate rows [cur, cur+n) in a ring of `cap` rows; skip to the start when
// the request does not fit before the end (TMA copies must be contiguous).
int32_t ring_alloc(int32_t& cur, int32_t n, int32_t cap) {
    if (cur + n > cap) cur = 0;
    const int32_t at = cur;
    cur += n;
    return at;
}

// Plan one walker's program over its shared-memory share; op indices local.
Walk plan(std::vector<StepIn>& steps, const PlanCfg& cfg) {
    const int32_t T = static_cast<int32_t>(steps.size());
    Walk w;
    w.ring_base = cfg.ring_base;
    w.ring_rows = cfg.ring_rows;
    w.stage_rows = cfg.stage_rows;
    w.barriers = cfg.barriers;
    w.n_steps = T;
    const int32_t XR = w.ring_rows, SR = w.stage_rows, NB = w.barriers, RB = cfg.ring_base;
    for (const StepIn& s : steps) {
        if (s.blk_rows > XR) throw Error(3, "walk block larger than the walker's ring");
        for (const DepIn& d : s.deps)
            if (d.fetch_rows > SR) throw Error(3, "walk fetch larger than the walker's staging ring");
    }

    // 1. ring placement and first overwriter of every block
    std::vector<int32_t> ring(T), ovw(T, kInf);
    std::vector<std::vector<int32_t>> ovl(T);
    {
        int32_t cur = 0;
        std::deque<int32_t> live;
        for (int32_t t = 0; t < T; ++t) {
            ring[t] = ring_alloc(cur, steps[t].blk_rows, XR);
            const int32_t a = ring[t], b = a + steps[t].blk_rows;
            std::deque<int32_t> keep;
            for (int32_t c : live) {
                const int32_t ca = ring[c], cb = ca + steps[c].blk_rows;
                if (ca < b && a < cb && steps[t].blk_rows > 0 && steps[c].blk_rows > 0) {
                    ovw[c] = t;
                    ovl[t].push_back(c);
                } else {
                    keep.push_back(c);
                }
            }
            keep.push_back(t);
            live.swap(keep);
        }
    }
    // 2. ring residency of every dependency; last ring reader of every block
    std::vector<int32_t> lastuser(T);
    for (int32_t t = 0; t < T; ++t) lastuser[t] = t;
    std::vector<std::vector<char>> resident(T);
    for (int32_t t = 0; t < T; ++t) {
        resident[t].resize(steps[t].deps.size());
        for (size_t d = 0; d < steps[t].deps.size(); ++d) {
            const DepIn& di = steps[t].deps[d];
            if (di.producer >= t) throw Error(3, "walk dependency is not earlier in the walk");
            const bool res = !di.global && di.producer >= 0 && !steps[di.producer].global &&
                             (ovw[di.producer] == kInf || t + cfg.headroom < ovw[di.producer]);
            resident[t][d] = res;
            if (res) lastuser[di.producer] = std::max(lastuser[di.producer], t);
        }
    }
    // 3. consumer events: one after every dependency, one when the step is done
    std::vector<int64_t> ev0(T + 1);
    int64_t e = 0;
    for (int32_t t = 0; t < T; ++t) {
        ev0[t] = e;
        e += int64_t(steps[t].deps.size()) + 1;
    }
    ev0[T] = e;
    w.events = e;
    if (e >= kInf) throw Error(3, "walk too long");
    auto ev_dep = [&](int32_t t, size_t d) { return int32_t(ev0[t] + int64_t(d)); };
    auto ev_done = [&](int32_t t) { return t < 0 ? -1 : int32_t(ev0[t + 1] - 1); };

    // 4. ops in consumption order with their issue events.  One op per step
    //    carries the step's block AND every re-fetched dependency whose staging
    //    region fits beside the others (a "chunk"); a step whose fetches exceed
    //    the staging ring (or a page's copy limit) continues in further chunks,
    //    each waited on at its first dependency.
    struct Live {
        int32_t a, b, release;
    };
    std::deque<Live> stage_live;
    int32_t scur = 0;
    std::vector<int32_t> release;      // per op: event after which its mbarrier may be re-armed
    std::vector<int32_t> tag_of_copy;  // content tag per copy (verification)
    std::vector<int32_t> dep_tag0(T + 1, 0);  // tag of dependency (t, d) = T + dep_tag0[t] + d
    for (int32_t t = 0; t < T; ++t) dep_tag0[t + 1] = dep_tag0[t] + int32_t(steps[t].deps.size());
    std::vector<int32_t> tag_producer(dep_tag0[T], -1), op_of_tag(dep_tag0[T], kInf);
    for (int32_t t = 0; t < T; ++t)
        for (size_t d = 0; d < steps[t].deps.size(); ++d) tag_producer[dep_tag0[t] + d] = steps[t].deps[d].producer;
    struct Chunk {
        std::vector<WCopy> cps;
        std::vector<int32_t> tags;
        int32_t after = -1, consume = -1, rel = -1, lo = kInf, hi = -1;  // staging span
    };
    auto push_chunk = [&](Chunk& c) {
        const int32_t s = static_cast<int32_t>(w.op.size());
        int32_t after = c.after;
        if (s >= NB) after = std::max(after, release[s - NB]);
        if (s > 0) after = std::max(after, w.op[s - 1].after);
        if (after > c.consume) throw Error(3, "walk plan infeasible (shared-memory rings too small)");
        WOp o{};
        o.after = after;
        o.ncopy = static_cast<int32_t>(c.cps.size());
        o.c0 = static_cast<int32_t>(w.copies.size());
        for (size_t i = 0; i < c.cps.size(); ++i) {
            o.bytes += copy_rows(c.cps[i]);
            w.copies.push_back(c.cps[i]);
            tag_of_copy.push_back(c.tags[i]);
            if (c.tags[i] >= T) op_of_tag[c.tags[i] - T] = s;
        }
        w.op.push_back(o);
        release.push_back(c.rel);
        return s;
    };
    for (int32_t t = 0; t < T; ++t) {
        StepIn& si = steps[t];
        WStep rec = si.rec;
        rec.ring = RB + ring[t];
        rec.dep0 = static_cast<int32_t>(w.dep.size());
        rec.ndep = static_cast<int32_t>(si.deps.size());
        w.block_rows += si.blk_rows;
        Chunk ch;
        ch.after = ev_done(t - cfg.prefetch - 1);
        for (int32_t c : ovl[t]) ch.after = std::max(ch.after, ev_done(std::max(c, lastuser[c])));
        ch.consume = ev_done(t - 1);
        ch.rel = int32_t(ev0[t]);  // barrier free once the step-start wait has passed
        for (WCopy c : si.copies) {
            c.smem += RB + ring[t];
            ch.cps.push_back(c);
            ch.tags.push_back(t);
        }
        bool first_chunk = true;
        std::vector<size_t> chunk_deps;  // deps (indices into w.dep) of the open chunk
        auto close_chunk = [&]() {
            if (ch.cps.empty() && first_chunk) {  // a global step with nothing staged: no op
                rec.op = -1;
                first_chunk = false;
                return;
            }
            const int32_t op = push_chunk(ch);
            if (first_chunk)
                rec.op = op;
            else
                w.dep[chunk_deps.front()].op = op;  // waited on at its first dependency
            first_chunk = false;
            chunk_deps.clear();
        };
        if (si.global) {
            ++w.global_steps;
            w.scratch_rows = std::max(w.scratch_rows, si.global_rows);
        }
        for (size_t d = 0; d < si.deps.size(); ++d) {
            DepIn& di = si.deps[d];
            WDep dr = di.rec;
            dr.prod = di.producer;
            dr.op = -1;
            if (di.global) {
                dr.src = dr.ysrc = -1;
                dr.global = 1;
                ++w.global_deps;
                w.dep.push_back(dr);
                continue;
            }
            if (resident[t][d]) {
                dr.src = di.ring_src >= 0 ? RB + ring[di.producer] + di.ring_src : -1;
                dr.ysrc = di.ring_ysrc >= 0 ? RB + ring[di.producer] + di.ring_ysrc : -1;
                w.ring_dep_rows += di.fetch_rows;
                w.dep.push_back(dr);
                continue;
            }
            if (di.fetch_rows <= 0) throw Error(3, "walk dependency with nothing to fetch");
            int32_t cur = scur;
            const int32_t at = XR + ring_alloc(cur, di.fetch_rows, SR);
            // a region overlapping this chunk's own staging span, or too many
            // copies for one program record, starts a new chunk
            const bool clash = ch.hi >= 0 && at < ch.hi && ch.lo < at + di.fetch_rows;
            if (clash || int32_t(ch.cps.size() + di.fetch.size()) > cfg.max_copies) {
                close_chunk();
                ch = Chunk{};
                ch.after = ev_done(t - cfg.prefetch - 1);
                ch.consume = d == 0 ? ev_done(t - 1) : ev_dep(t, d - 1);
                ch.rel = ev_dep(t, d);
            }
            scur = cur;
            ch.lo = std::min(ch.lo, at);
            ch.hi = std::max(ch.hi, at + di.fetch_rows);
            if (di.producer >= 0) ch.after = std::max(ch.after, ev_done(di.producer));
            std::deque<Live> keep;
            for (const Live& l : stage_live) {
                if (l.a < at + di.fetch_rows && at < l.b)
                    ch.after = std::max(ch.after, l.release);
                else
                    keep.push_back(l);
            }
            keep.push_back(Live{at, at + di.fetch_rows, ev_dep(t, d)});
            stage_live.swap(keep);
            for (WCopy c : di.fetch) {
                c.smem += RB + at;
                ch.cps.push_back(c);
                ch.tags.push_back(T + dep_tag0[t] + int32_t(d));
            }
            dr.src = di.stage_src >= 0 ? RB + at + di.stage_src : -1;
            dr.ysrc = di.stage_ysrc >= 0 ? RB + at + di.stage_ysrc : -1;
            w.fetched_rows += di.fetch_rows;
            chunk_deps.push_back(w.dep.size());
            w.dep.push_back(dr);
        }
        close_chunk();
        w.step.push_back(rec);
    }

    // 5. independent verification: replay the consumer's events, issue ops at
    //    their events and check that no shared-memory row is overwritten while
    //    its content is still to be read, that every op is issued before it is
    //    waited on, that every read finds the content it expects, and that
    //    every fetch of produced data follows its producer.
    {
        const int32_t rows = XR + SR;
        const int32_t n_tags = T + dep_tag0[T];
        std::vector<int32_t> need(n_tags, -1);  // last event reading each content tag
        for (int32_t t = 0; t < T; ++t) {
            need[t] = std::max(need[t], ev_done(t));
            for (int32_t d = 0; d < w.step[t].ndep; ++d) {
                if (steps[t].deps[d].global) continue;
                const int32_t p = steps[t].deps[d].producer;
                const int32_t g = resident[t][d] ? p : T + dep_tag0[t] + d;
                need[g] = std::max(need[g], ev_dep(t, d));
            }
        }
        std::vector<int32_t> row_tag(rows, -1);
        size_t next = 0;
        auto issue_upto = [&](int32_t ev) {
            while (next < w.op.size() && w.op[next].after <= ev) {
                const WOp& o = w.op[next];
                for (int32_t i = 0; i < o.ncopy; ++i) {
                    const WCopy& c = w.copies[o.c0 + i];
                    const int32_t a = c.smem - RB, n = copy_rows(c), g = tag_of_copy[o.c0 + i];
                    if (a < 0 || a + n > rows) throw Error(3, "walk copy outside the walker's shared memory");
                    for (int32_t r = a; r < a + n; ++r) {
                        if (row_tag[r] >= 0 && need[row_tag[r]] > ev)
                            throw Error(3, "walk plan overwrites live shared memory (row " +
                                               std::to_string(r) + ")");
                        row_tag[r] = g;
                    }
                    if (g >= T) {  // a re-fetch of produced data: its producer must be done
                        const int32_t p = tag_producer[g - T];
                        if (p >= 0 && ev < ev_done(p))
                            throw Error(3, "walk fetch issued before its producer finished");
                    }
                }
                ++next;
            }
        };
        auto expect = [&](int32_t row, int32_t g) {
            if (row >= 0 && row_tag[row - RB] != g) throw Error(3, "walk reads content that is not there");
        };
        issue_upto(-1);
        int32_t waited = -1;
        for (int32_t t = 0; t < T; ++t) {
            const WStep& st = w.step[t];
            if (st.op >= 0 && size_t(st.op) >= next) throw Error(3, "walk waits on an unissued op");
            if (!steps[t].global) {
                if (st.op < 0) throw Error(3, "walk step block without an op");
                waited = std::max(waited, st.op);
                expect(st.ring, t);
            }
            for (int32_t d = 0; d < st.ndep; ++d) {
                const WDep& dr = w.dep[st.dep0 + d];
                if (dr.global) {
                    issue_upto(ev_dep(t, d));
                    continue;
                }
                if (dr.op >= 0) {
                    if (size_t(dr.op) >= next) throw Error(3, "walk waits on an unissued fetch");
                    waited = std::max(waited, dr.op);
                }
                const int32_t p = steps[t].deps[d].producer;
                const int32_t g = resident[t][d] ? p : T + dep_tag0[t] + d;
                expect(dr.src, g);
                expect(dr.ysrc, g);
                if (!resident[t][d] && op_of_tag[g - T] > waited)
                    throw Error(3, "walk reads a fetch it never waited for");
                issue_upto(ev_dep(t, d));
            }
            issue_upto(ev_done(t));
        }
        if (next != w.op.size()) throw Error(3, "walk ops left unissued");
    }
    return w;
}

// Unified-pool variant of plan(): the step blocks and the re-fetched
// dependencies share one circular pool of ring + staging rows, allocated in
// consumption order, so a step with few fetches prefetches its successors'
// blocks further ahead and a step with many fetches borrows block rows.  A
// dependency stays resident while its producer's block is intact.  Every
// overlap with live rows becomes an issue constraint; an overlap that would
// make the op late (or hit the step's own block or its chunk) moves the
// allocation past that region.  Same verification as plan().
Walk plan_unified(std::vector<StepIn>& steps, const PlanCfg& cfg) {
    const int32_t T = static_cast<int32_t>(steps.size());
    Walk w;
    w.ring_base = cfg.ring_base;
    w.ring_rows = cfg.ring_rows;
    w.stage_rows = cfg.stage_rows;
    w.barriers = cfg.barriers;
    w.n_steps = T;
    const int32_t XR = w.ring_rows, SR = w.stage_rows, NB = w.barriers, RB = cfg.ring_base;
    const int32_t PR = XR + SR;
    for (const StepIn& st : steps) {
        if (st.blk_rows > PR) throw Error(3, "walk block larger than the walker's pool");
        for (const DepIn& d : st.deps)
            if (d.fetch_rows > PR) throw Error(3, "walk fetch larger than the walker's pool");
    }
    std::vector<int64_t> ev0(T + 1);
    int64_t e = 0;
    for (int32_t t = 0; t < T; ++t) {
        ev0[t] = e;
        e += int64_t(steps[t].deps.size()) + 1;
    }
    ev0[T] = e;
    w.events = e;
    if (e >= kInf) throw Error(3, "walk too long");
    auto ev_dep = [&](int32_t t, size_t d) { return int32_t(ev0[t] + int64_t(d)); };
    auto ev_done = [&](int32_t t) { return t < 0 ? -1 : int32_t(ev0[t + 1] - 1); };

    struct Reg {
        int32_t a, b, release, block;  // block: producing step, -1 = a fetch
    };
    std::vector<Reg> live;
    std::vector<int32_t> ring(T, 0);
    std::vector<char> intact(T, 0);
    std::vector<std::vector<char>> resident(T);
    int32_t cur = 0;
    // place n rows: returns the row or -1; `after` gets the overlapped releases
    auto place = [&](int32_t n, int32_t consume, int32_t lo, int32_t hi, int32_t self_block, int32_t& after) {
        int32_t at = cur;
        for (int32_t tries = 0; tries < 2 * PR + 2; ++tries) {
            if (at + n > PR) at = 0;
            bool ok = true;
            int32_t aft = -1, skip_to = at + 1;
            for (const Reg& r : live) {
                if (r.a < at + n && at < r.b) {
                    if (r.release > consume || (self_block >= 0 && r.block == self_block)) {
                        ok = false;
                        skip_to = std::max(skip_to, r.b);
                    } else {
                        aft = std::max(aft, r.release);
                    }
                }
            }
            if (ok && hi >= 0 && at < hi && lo < at + n) {  // the open chunk's own rows
                ok = false;
                skip_to = std::max(skip_to, hi);
            }
            if (ok) {
                after = aft;
                return at;
            }
            at = skip_to;
        }
        return int32_t(-1);
    };
    auto occupy = [&](int32_t at, int32_t n, int32_t release, int32_t block) {
        std::vector<Reg> keep;
        for (const Reg& r : live) {
            if (r.a < at + n && at < r.b) {
                if (r.block >= 0) intact[r.block] = 0;
            } else {
                keep.push_back(r);
            }
        }
        keep.push_back(Reg{at, at + n, release, block});
        live.swap(keep);
        cur = at + n;
    };

    std::vector<int32_t> release;
    std::vector<int32_t> tag_of_copy;
    std::vector<int32_t> dep_tag0(T + 1, 0);
    for (int32_t t = 0; t < T; ++t) dep_tag0[t + 1] = dep_tag0[t] + int32_t(steps[t].deps.size());
    std::vector<int32_t> tag_producer(dep_tag0[T], -1), op_of_tag(dep_tag0[T], kInf);
    for (int32_t t = 0; t < T; ++t)
        for (size_t d = 0; d < steps[t].deps.size(); ++d) tag_producer[dep_tag0[t] + d] = steps[t].deps[d].producer;
    struct Chunk {
        std::vector<WCopy> cps;
        std::vector<int32_t> tags;
        int32_t after = -1, consume = -1, rel = -1, lo = kInf, hi = -1;
    };
    auto push_chunk = [&](Chunk& c) {
        const int32_t s = static_cast<int32_t>(w.op.size());
        int32_t after = c.after;
        if (s >= NB) after = std::max(after, release[s - NB]);
        if (s > 0) after = std::max(after, w.op[s - 1].after);
        if (after > c.consume) throw Error(3, "walk plan infeasible (shared-memory pool too small)");
        WOp o{};
        o.after = after;
        o.ncopy = static_cast<int32_t>(c.cps.size());
        o.c0 = static_cast<int32_t>(w.copies.size());
        for (size_t i = 0; i < c.cps.size(); ++i) {
            o.bytes += copy_rows(c.cps[i]);
            w.copies.push_back(c.cps[i]);
            tag_of_copy.push_back(c.tags[i]);
            if (c.tags[i] >= T) op_of_tag[c.tags[i] - T] = s;
        }
        w.op.push_back(o);
        release.push_back(c.rel);
        return s;
    };
    for (int32_t t = 0; t < T; ++t) {
        StepIn& si = steps[t];
        WStep rec = si.rec;
        Chunk ch;
        ch.consume = ev_done(t - 1);
        ch.rel = int32_t(ev0[t]);
        // the block goes where it leaves a contiguous gap for the step's largest
        // fetch (a block in the middle of the pool fragments it): the FIFO
        // position first, then either end
        int32_t need = 0;
        for (const DepIn& di : si.deps) need = std::max(need, di.fetch_rows);
        int32_t aft = -1, at = -1;
        if (si.global) {  // nothing of the step in the pool (its deps are global too)
            WStep grec = si.rec;
            grec.ring = 0;
            grec.op = -1;
            grec.dep0 = static_cast<int32_t>(w.dep.size());
            grec.ndep = static_cast<int32_t>(si.deps.size());
            resident[t].assign(si.deps.size(), 0);
            ++w.global_steps;
            w.scratch_rows = std::max(w.scratch_rows, si.global_rows);
            for (const DepIn& di : si.deps) {
                if (!di.global) throw Error(3, "walk: a global step with a staged dependency");
                WDep dr = di.rec;
            dr.prod = di.producer;
                dr.op = -1;
                dr.src = dr.ysrc = -1;
                dr.global = 1;
                ++w.global_deps;
                w.dep.push_back(dr);
            }
            w.step.push_back(grec);
            continue;
        }
        // producers this step could read from the pool (still intact)
        std::vector<int32_t> prods;
        for (const DepIn& di : si.deps)
            if (di.producer >= 0 && intact[di.producer]) prods.push_back(di.producer);
        auto hits_prod = [&](int32_t pos) {
            for (const Reg& r : live)
                if (r.block >= 0 && r.a < pos + si.blk_rows && pos < r.b &&
                    std::find(prods.begin(), prods.end(), r.block) != prods.end())
                    return true;
            return false;
        };
        int score_best = -1;
        for (int32_t cand : {cur, 0, PR - si.blk_rows}) {
            const int32_t keep_cur = cur;
            cur = cand;
            int32_t a2 = -1;
            const int32_t pos = place(si.blk_rows, ch.consume, 0, -1, -1, a2);
            cur = keep_cur;
            if (pos < 0) continue;
            const bool gap = std::max(pos, PR - pos - si.blk_rows) >= need;
            const int score = (gap ? 2 : 0) + (hits_prod(pos) ? 0 : 1);
            if (score > score_best) {
                score_best = score;
                at = pos;
                aft = a2;
            }
            if (score == 3) break;
        }
        if (at < 0) throw Error(3, "walk plan infeasible (no pool rows for a block)");
        occupy(at, si.blk_rows, ev_done(t), t);
        intact[t] = 1;
        ring[t] = at;
        ch.after = std::max(ev_done(t - cfg.prefetch - 1), aft);
        rec.ring = RB + at;
        rec.dep0 = static_cast<int32_t>(w.dep.size());
        rec.ndep = static_cast<int32_t>(si.deps.size());
        w.block_rows += si.blk_rows;
        for (WCopy c : si.copies) {
            c.smem += RB + at;
            ch.cps.push_back(c);
            ch.tags.push_back(t);
        }
        bool first_chunk = true;
        std::vector<size_t> chunk_deps;
        auto close_chunk = [&]() {
            const int32_t op = push_chunk(ch);
            if (first_chunk)
                rec.op = op;
            else
                w.dep[chunk_deps.front()].op = op;
            first_chunk = false;
            chunk_deps.clear();
        };
        resident[t].assign(si.deps.size(), 0);
        for (size_t d = 0; d < si.deps.size(); ++d) {
            DepIn& di = si.deps[d];
            WDep dr = di.rec;
            dr.prod = di.producer;
            dr.op = -1;
            const int32_t pr = di.producer;
            if (di.global) {
                dr.src = dr.ysrc = -1;
                dr.global = 1;
                ++w.global_deps;
                w.dep.push_back(dr);
                continue;
            }
            if (pr >= 0 && intact[pr] && (di.ring_src >= 0 || di.ring_ysrc >= 0)) {
                resident[t][d] = 1;
                for (Reg& r : live)
                    if (r.block == pr) r.release = std::max(r.release, ev_dep(t, d));
                dr.src = di.ring_src >= 0 ? RB + ring[pr] + di.ring_src : -1;
                dr.ysrc = di.ring_ysrc >= 0 ? RB + ring[pr] + di.ring_ysrc : -1;
                w.ring_dep_rows += di.fetch_rows;
                w.dep.push_back(dr);
                continue;
            }
            if (di.fetch_rows <= 0) throw Error(3, "walk dependency with nothing to fetch");
            int32_t faft = -1;
            int32_t fat = int32_t(int(ch.cps.size() + di.fetch.size()) <= cfg.max_copies
                                      ? place(di.fetch_rows, ch.consume, ch.lo, ch.hi, t, faft) : -1);
            if (fat < 0) {  // a new chunk, waited on at this dependency
                close_chunk();
                ch = Chunk{};
                ch.after = ev_done(t - cfg.prefetch - 1);
                ch.consume = d == 0 ? ev_done(t - 1) : ev_dep(t, d - 1);
                ch.rel = ev_dep(t, d);
                fat = place(di.fetch_rows, ch.consume, 0, -1, t, faft);
                if (fat < 0) throw Error(3, "walk plan infeasible (no pool rows for a fetch)");
            }
            occupy(fat, di.fetch_rows, ev_dep(t, d), -1);
            ch.after = std::max(ch.after, faft);
            if (pr >= 0) ch.after = std::max(ch.after, ev_done(pr));
            ch.lo = std::min(ch.lo, fat);
            ch.hi = std::max(ch.hi, fat + di.fetch_rows);
            for (WCopy c : di.fetch) {
                c.smem += RB + fat;
                ch.cps.push_back(c);
                ch.tags.push_back(T + dep_tag0[t] + int32_t(d));
            }
            dr.src = di.stage_src >= 0 ? RB + fat + di.stage_src : -1;
            dr.ysrc = di.stage_ysrc >= 0 ? RB + fat + di.stage_ysrc : -1;
            w.fetched_rows += di.fetch_rows;
            chunk_deps.push_back(w.dep.size());
            w.dep.push_back(dr);
        }
        close_chunk();
        w.step.push_back(rec);
    }

    // 5. independent verification: replay the consumer's events, issue ops at
    //    their events and check that no shared-memory row is overwritten while
    //    its content is still to be read, that every op is issued before it is
    //    waited on, that every read finds the content it expects, and that
    //    every fetch of produced data follows its producer.
    {
        const int32_t rows = XR + SR;
        const int32_t n_tags = T + dep_tag0[T];
        std::vector<int32_t> need(n_tags, -1);  // last event reading each content tag
        for (int32_t t = 0; t < T; ++t) {
            need[t] = std::max(need[t], ev_done(t));
            for (int32_t d = 0; d < w.step[t].ndep; ++d) {
                if (steps[t].deps[d].global) continue;
                const int32_t p = steps[t].deps[d].producer;
                const int32_t g = resident[t][d] ? p : T + dep_tag0[t] + d;
                need[g] = std::max(need[g], ev_dep(t, d));
            }
        }
        std::vector<int32_t> row_tag(rows, -1);
        size_t next = 0;
        auto issue_upto = [&](int32_t ev) {
            while (next < w.op.size() && w.op[next].after <= ev) {
                const WOp& o = w.op[next];
                for (int32_t i = 0; i < o.ncopy; ++i) {
                    const WCopy& c = w.copies[o.c0 + i];
                    const int32_t a = c.smem - RB, n = copy_rows(c), g = tag_of_copy[o.c0 + i];
                    if (a < 0 || a + n > rows) throw Error(3, "walk copy outside the walker's shared memory");
                    for (int32_t r = a; r < a + n; ++r) {
                        if (row_tag[r] >= 0 && need[row_tag[r]] > ev)
                            throw Error(3, "walk plan overwrites live shared memory (row " +
                                               std::to_string(r) + ")");
                        row_tag[r] = g;
                    }
                    if (g >= T) {  // a re-fetch of produced data: its producer must be done
                        const int32_t p = tag_producer[g - T];
                        if (p >= 0 && ev < ev_done(p))
                            throw Error(3, "walk fetch issued before its producer finished");
                    }
                }
                ++next;
            }
        };
        auto expect = [&](int32_t row, int32_t g) {
            if (row >= 0 && row_tag[row - RB] != g) throw Error(3, "walk reads content that is not there");
        };
        issue_upto(-1);
        int32_t waited = -1;
        for (int32_t t = 0; t < T; ++t) {
            const WStep& st = w.step[t];
            if (st.op >= 0 && size_t(st.op) >= next) throw Error(3, "walk waits on an unissued op");
            if (!steps[t].global) {
                if (st.op < 0) throw Error(3, "walk step block without an op");
                waited = std::max(waited, st.op);
                expect(st.ring, t);
            }
            for (int32_t d = 0; d < st.ndep; ++d) {
                const WDep& dr = w.dep[st.dep0 + d];
                if (dr.global) {
                    issue_upto(ev_dep(t, d));
                    continue;
                }
                if (dr.op >= 0) {
                    if (size_t(dr.op) >= next) throw Error(3, "walk waits on an unissued fetch");
                    waited = std::max(waited, dr.op);
                }
                const int32_t p = steps[t].deps[d].producer;
                const int32_t g = resident[t][d] ? p : T + dep_tag0[t] + d;
                expect(dr.src, g);
                expect(dr.ysrc, g);
                if (!resident[t][d] && op_of_tag[g - T] > waited)
                    throw Error(3, "walk reads a fetch it never waited for");
                issue_upto(ev_dep(t, d));
            }
            issue_upto(ev_done(t));
        }
        if (next != w.op.size()) throw Error(3, "walk ops left unissued");
    }
    return w;
}

// Program-stream writer of one walker: pads to the next page whenever a record
// would straddle one.
struct Emitter {
    std::vector<int32_t> st;
    int32_t W;
    void emit(const std::vector<int32_t>& rec) {
        if (int32_t(rec.size()) > W - 1) throw Error(3, "walk record longer than a program page");
        const int32_t used = int32_t(st.size() % size_t(W));
        if (used + int32_t(rec.size()) > W - 1) {
            st.push_back(kRecPage);
            while (st.size() % size_t(W)) st.push_back(0);
        }
        st.insert(st.end(), rec.begin(), rec.end());
    }
    void finish() {
        emit({kRecDone});
        while (st.size() % size_t(W)) st.push_back(0);
    }
};

// Two consecutive forward dependencies k, k+1 of one step form a supernode
// pair when L(:,k) is row k+1 followed by exactly the rows of L(:,k+1) (so the
// destinations of k are kpos(k+1) then those of k+1).  Every x element still
// sees k's update before k+1's.
bool pairable(const Walk& w, const WDep& e, const WDep& f, int64_t ev_e, int32_t op_base, int32_t W) {
    if (e.global || f.global) return false;
    if (6 + ((f.nrows + 3) & ~3) / 2 > W - 1) return false;  // the pair record must fit a page
    if (e.nrows <= 0 || f.nrows < 0 || e.nrows != f.nrows + 1) return false;
    // a second wait is hoisted to the pair's start: its op must already be issued
    // there (issue event before e's) and its number must fit the record
    if (f.op >= 0 && (w.op[f.op].after >= ev_e || op_base + f.op + 1 >= 65536)) return false;
    if ((f.kpos_fs & 0xffff) == 0xffff || f.nrows == 0) return false;
    if (int32_t(w.dst[e.u0]) != (f.kpos_fs & 0xffff)) return false;
    for (int32_t r = 0; r < f.nrows; ++r)
        if (w.dst[e.u0 + 1 + r] != w.dst[f.u0 + r]) return false;
    return e.ysrc < 65536 && f.ysrc < 65536 && f.src < 65536;
}

// Serialise one verified program: prologue issues, then per step: STEP,
// (DEP, ISSUE*) per dependency, END, ISSUE* -- each ISSUE right after the
// consumer event it waits for.  Op numbers continue at op_base (barrier parity
// runs on across phases).
void encode(Emitter& em, const Walk& w, bool forward, int32_t op_base, bool pairs) {
    size_t next = 0;
    auto issue_upto = [&](int64_t ev) {
        while (next < w.op.size() && w.op[next].after <= ev) {
            const WOp& o = w.op[next];
            // copies that continue each other in the tape and in shared memory
            // (dependencies k, k+1 staged side by side) travel as one
            std::vector<WCopy> cps;
            for (int32_t i = 0; i < o.ncopy; ++i) {
                const WCopy& c = w.copies[o.c0 + i];
                if (!cps.empty()) {
                    WCopy& p = cps.back();
                    const int32_t pr = p.tape_rows >> 8, cr = c.tape_rows >> 8;
                    if ((p.tape_rows & 0xff) == (c.tape_rows & 0xff) && c.slot == p.slot + pr &&
                        c.smem == p.smem + pr && pr + cr < 1024) {
                        p.tape_rows = (p.tape_rows & 0xff) | ((pr + cr) << 8);
                        continue;
                    }
                }
                cps.push_back(c);
            }
            std::vector<int32_t> rec{kRecIssue | (int32_t(cps.size()) << 4), op_base + int32_t(next), o.bytes};
            for (const WCopy& c : cps) {
                const int32_t tape = c.tape_rows & 0xff, rows = c.tape_rows >> 8;
                if (rows >= 1024 || c.smem >= (1 << 20)) throw Error(3, "walk copy too large to encode");
                rec.push_back(tape | (rows << 2) | (c.smem << 12));
                rec.push_back(c.slot);
            }
            em.emit(rec);
            ++next;
        }
    };
    auto opn = [&](int32_t op) { return op >= 0 ? op_base + op : -1; };
    const int32_t W = em.W;
    // a global-source dependency in records of at most W - 1 words: rows split
    // into chunks (each re-reads the multiplier; only the first carries the FS role)
    auto emit_dep_global = [&](const WDep& e, int32_t len) {
        (void)len;
        const int32_t max_rows = 2 * (W - 1 - 5);
        int32_t q0 = 0;
        bool first = true;
        do {
            const int32_t n = std::min(e.nrows - q0, max_rows);
            const int32_t kpos = e.kpos_fs & 0xffff;
            const int32_t fs = first ? int32_t(unsigned(e.kpos_fs) >> 16) : 0xffff;
            std::vector<int32_t> rec{kRecDepG | ((first ? opn(e.op) + 1 : 0) << 4), kpos | (fs << 16), n,
                                     e.gslot + q0, e.gnl - q0};
            for (int32_t r = 0; r < n; r += 2) {
                const int32_t a = int32_t(w.dst[e.u0 + q0 + r]);
                const int32_t b = r + 1 < n ? int32_t(w.dst[e.u0 + q0 + r + 1]) : 0;
                rec.push_back(a | (b << 16));
            }
            em.emit(rec);
            q0 += n;
            first = false;
        } while (q0 < e.nrows);
    };
    issue_upto(-1);
    int64_t ev = 0;
    // backward: two consecutive rows travel as one kRecPair when the second does not
    // depend on the first, every op either waits for is already issued, and the
    // record fits a page (their copy issues follow the pair)
    auto pair_record = [&](const WStep& a, const WStep& b, int32_t t) -> std::vector<int32_t> {
        if (forward || a.global || b.global || !pairs) return {};
        const int32_t nA = a.ndep, nB = b.ndep;
        if (nA >= 4096 || nB >= 65536) return {};
        std::vector<int32_t> waits;
        auto ready = [&](int32_t op) { return op < 0 || (size_t(op) < next && opn(op) + 1 < 65536); };
        if (!ready(a.op) || !ready(b.op)) return {};
        for (const WStep* st : {&a, &b})
            for (int32_t d = 0; d < st->ndep; ++d) {
                const WDep& e = w.dep[st->dep0 + d];
                if (st == &b && e.prod == t) return {};  // B needs A's x
                if (e.global || e.ysrc >= 65536 || !ready(e.op)) return {};
                if (e.op >= 0 && std::find(waits.begin(), waits.end(), opn(e.op) + 1) == waits.end())
                    waits.push_back(opn(e.op) + 1);
            }
        const int32_t len = 7 + int32_t(waits.size()) + (nA + 1) / 2 + (nB + 1) / 2;
        if (len > W - 1 || waits.size() >= 256) return {};
        std::vector<int32_t> rec{kRecPair | (nA << 4) | (int32_t(waits.size()) << 16), a.ring | (a.len_dp << 16),
                                 b.ring | (b.len_dp << 16), a.brow, b.brow, (opn(a.op) + 1) | ((opn(b.op) + 1) << 16),
                                 nB};
        rec.insert(rec.end(), waits.begin(), waits.end());
        for (const WStep* st : {&a, &b})
            for (int32_t i = 0; i < st->ndep; i += 2) {
                const int32_t lo = w.dep[st->dep0 + i].ysrc;
                const int32_t hi = i + 1 < st->ndep ? w.dep[st->dep0 + i + 1].ysrc : 0;
                rec.push_back(lo | (hi << 16));
            }
        return rec;
    };
    for (int32_t t = 0; t < int32_t(w.step.size()); ++t) {
        const WStep& s = w.step[t];
        if (t + 1 < int32_t(w.step.size())) {
            std::vector<int32_t> rec = pair_record(s, w.step[t + 1], t);
            if (!rec.empty()) {
                em.emit(rec);
                const int32_t evs = s.ndep + 1 + w.step[t + 1].ndep + 1;
                for (int32_t i = 0; i < evs; ++i) issue_upto(ev++);
                ++t;
                continue;
            }
        }
        if (forward) {
            const int32_t len = s.len_dp & 0xffff, dp = s.len_dp >> 16;
            if (s.global) {
                em.emit({kRecStepG | (s.ndep << 4), len | (dp << 16), s.gslot, s.lslot, s.brow});
                for (int32_t d = 0; d < s.ndep; ++d) {
                    emit_dep_global(w.dep[s.dep0 + d], len);
                    issue_upto(ev++);
                }
                for (int32_t z0 = 0; z0 < dp; z0 += W - 3) {  // the U part -> its row-major slots
                    const int32_t cnt = std::min(dp - z0, W - 3);
                    std::vector<int32_t> rec{kRecEndU | (cnt << 4), z0};
                    for (int32_t z = z0; z < z0 + cnt; ++z) rec.push_back(w.ut[s.ut0 + z]);
                    em.emit(rec);
                }
                em.emit({kRecEndG});
                issue_upto(ev++);
                continue;
            }
            em.emit({kRecStep | (s.ndep << 4), s.ring | (len << 16), dp, s.lslot, s.brow, opn(s.op)});
            for (int32_t d = 0; d < s.ndep; ++d) {
                const WDep& e = w.dep[s.dep0 + d];
                if (e.global) {
                    emit_dep_global(e, len);
                    issue_upto(ev++);
                    continue;
                }
                if (e.src >= 65536 || e.nrows >= 65536) throw Error(3, "walk dependency too large to encode");
                if (d + 1 < s.ndep && pairable(w, e, w.dep[s.dep0 + d + 1], ev, op_base, W)) {
                    // supernode pair: dep k's rows are row k+1 (x position kpos2) then
                    // exactly dep k+1's rows; one pass applies both in order
                    const WDep& f = w.dep[s.dep0 + d + 1];
                    const int32_t kpos1 = e.kpos_fs & 0xffff, fs1 = int32_t(unsigned(e.kpos_fs) >> 16);
                    const int32_t kpos2 = f.kpos_fs & 0xffff, fs2 = int32_t(unsigned(f.kpos_fs) >> 16);
                    std::vector<int32_t> rec{kRecDep2 | ((opn(e.op) + 1) << 4), kpos1 | (kpos2 << 16),
                                             f.nrows | (std::max(e.src, 0) << 16), std::max(f.src, 0) | (fs1 << 16),
                                             (std::max(e.ysrc, 0) & 0xffff) | (std::max(f.ysrc, 0) << 16),
                                             fs2 | ((opn(f.op) + 1) << 16)};
                    const int32_t n4 = (f.nrows + 3) & ~3;
                    auto dst = [&](int32_t r) { return r < f.nrows ? int32_t(w.dst[f.u0 + r]) : len; };
                    for (int32_t r = 0; r < n4; r += 2) rec.push_back(dst(r) | (dst(r + 1) << 16));
                    em.emit(rec);
                    issue_upto(ev++);
                    issue_upto(ev++);
                    ++d;
                    continue;
                }
                std::vector<int32_t> rec{kRecDep | ((opn(e.op) + 1) << 4), e.kpos_fs,
                                         e.nrows | (std::max(e.src, 0) << 16), e.ysrc};
                // destinations padded to a multiple of 4 with the block's spare
                // row `len` (dead between STEP and END), so the kernel runs whole
                // 4-row groups without tails
                const int32_t n4 = (e.nrows + 3) & ~3;
                auto dst = [&](int32_t r) { return r < e.nrows ? int32_t(w.dst[e.u0 + r]) : len; };
                for (int32_t r = 0; r < n4; r += 2) rec.push_back(dst(r) | (dst(r + 1) << 16));
                em.emit(rec);
                issue_upto(ev++);
            }
            std::vector<int32_t> end{kRecEnd | (dp << 4)};
            for (int32_t z = 0; z < dp; ++z) end.push_back(w.ut[s.ut0 + z]);
            em.emit(end);
            issue_upto(ev++);
        } else if (s.global) {
            // a row block read in place from the LU tape, x_k from the b tape
            em.emit({kRecStepG | (s.ndep << 4), s.len_dp, s.gslot, s.brow});
            for (int32_t d = 0; d < s.ndep;) {
                const int32_t n = std::min(s.ndep - d, W - 2);
                std::vector<int32_t> rec{kRecDepNG | (n << 4)};
                for (int32_t i = 0; i < n; ++i) rec.push_back(w.dep[s.dep0 + d + i].gslot);
                em.emit(rec);
                for (int32_t i = 0; i < n; ++i) issue_upto(ev++);
                d += n;
            }
            em.emit({kRecEndG});
            issue_upto(ev++);
        } else {
            em.emit({kRecStep | (s.ndep << 4), s.ring | (s.len_dp << 16), 0, s.lslot, s.brow, opn(s.op)});
            // runs of dependencies that need no wait of their own travel in one
            // record (their copy issues follow the run)
            const int32_t max_run = 2 * (em.W - 4);
            for (int32_t d = 0; d < s.ndep;) {
                int32_t n = 1;
                while (d + n < s.ndep && n < max_run && w.dep[s.dep0 + d + n].op < 0) ++n;
                std::vector<int32_t> rec{kRecDepN | ((opn(w.dep[s.dep0 + d].op) + 1) << 4), n};
                for (int32_t i = 0; i < n; i += 2) {
                    const int32_t lo = w.dep[s.dep0 + d + i].ysrc;
                    const int32_t hi = i + 1 < n ? w.dep[s.dep0 + d + i + 1].ysrc : 0;
                    if (lo >= 65536 || hi >= 65536) throw Error(3, "walk dependency too large to encode");
                    rec.push_back(lo | (hi << 16));
                }
                em.emit(rec);
                for (int32_t i = 0; i < n; ++i) issue_upto(ev++);
                d += n;
            }
            em.emit({kRecEnd});
            issue_upto(ev++);
        }
    }
    if (next != w.op.size()) throw Error(3, "walk stream left ops unissued");
}

// Elimination tree of the frozen pattern: parent(k) = first L row of column k.
std::vector<int32_t> etree_parent(const Symbolic& s) {
    std::vector<int32_t> parent(s.nJ, -1);
    for (int32_t k = 0; k < s.nJ; ++k)
        if (s.dpos[k] + 1 < s.cp[k + 1]) parent[k] = s.ri[s.dpos[k] + 1];
    return parent;
}

// Shared-memory geometry of a launch: page size from the longest possible
// record, then the rows left in the CTA budget.
struct Geometry {
    int32_t W = 0, rows = 0;
};
Geometry geometry(const Symbolic& s, const WalkConfig& cfg, int32_t walkers) {
    int32_t longest = 8;
    for (int32_t k = 0; k < s.nJ; ++k) {
        longest = std::max(longest, 2 + (s.dpos[k] - s.cp[k]));           // END
        longest = std::max(longest, 6 + (s.cp[k + 1] - s.dpos[k]) / 2);  // DEP (rows padded to 4)
    }
    // longer records than a page of kMaxPageWords go global (their forms split)
    const int32_t W = std::min(std::max(cfg.page_words, 4 * ((longest + 1 + 3) / 4)), kMaxPageWords);
    const int64_t fixed = int64_t(walkers) * (int64_t(cfg.pages) * W * 4 + int64_t(cfg.barriers + cfg.pages) * 8);
    const int64_t rows = (int64_t(cfg.smem_budget) - fixed) / cfg.row_bytes;
    return Geometry{W, int32_t(std::max<int64_t>(rows, 0))};
}

// Per-walker ring / staging split of a share of rows.
void split_share(const WalkConfig& cfg, int32_t share, int32_t& ring, int32_t& stage, int32_t level = 0) {
    const double frac = level > 0 && cfg.stage_frac_up >= 0.0 ? cfg.stage_frac_up : cfg.stage_frac;
    stage = cfg.stage_rows ? cfg.stage_rows : int32_t(share * frac);
    ring = cfg.ring_rows ? cfg.ring_rows : share - stage;
}

struct Phase {
    std::vector<std::vector<int32_t>> lists;  // per walker: steps (column / row ids) in walk order
};

// Global-memory fallback: blocks larger than gb rows (and every dependency of
// such a step) and fetches larger than gf rows are read from global memory
// instead of staged; so are records that would not fit a program page.  The
// per-element operation order is unchanged, only where the operands live.
void apply_global(Program& pr, int32_t gb, int32_t gf, int32_t W, bool forward) {
    for (StepIn& si : pr.steps) {
        const int32_t dp = forward ? (si.rec.len_dp >> 16) : 0;
        if (si.blk_rows > gb || (forward && 1 + dp > W - 1)) {
            si.global = true;
            si.global_rows = forward ? si.blk_rows : 0;
            si.blk_rows = 0;
            si.copies.clear();
            si.rec.global = 1;
        }
        for (DepIn& di : si.deps) {
            const int32_t n4 = (di.rec.nrows + 3) & ~3;
            if (si.global || di.fetch_rows > gf || (forward && 4 + n4 / 2 > W - 1)) {
                di.global = true;
                di.fetch.clear();
                di.fetch_rows = 0;
                di.ring_src = di.ring_ysrc = -1;
                di.rec.global = 1;
            }
        }
    }
}

// Plan one walker's program: shared memory only if it fits, else with the
// largest blocks / fetches moved to global memory, halving the limits until the
// plan is feasible (everything global always is: no copies at all).
Walk plan_walker(const Program& base, const PlanCfg& pc, const WalkConfig& cfg, int32_t W, bool forward) {
    const int32_t PR = pc.ring_rows + pc.stage_rows;
    int32_t gb = kInf, gf = kInf;
    if (cfg.global_frac > 0.0) {
        gb = std::max(1, int32_t(cfg.global_frac * PR));
        gf = std::max(1, gb / 2);
    }
    for (;;) {
        Program pr = base;
        apply_global(pr, gb, gf, W, forward);
        if (cfg.unified) {
            try {
                return plan_unified(pr.steps, pc);
            } catch (const Error&) {  // infeasible: the split ring / staging plan
            }
        }
        try {
            return plan(pr.steps, pc);
        } catch (const Error&) {
            if (gb == 0) throw;
        }
        gb = gb == kInf ? PR / 2 : gb / 2;
        gf = gb / 2;
    }
}

// Plan and encode every (phase, walker) program of a walk set.
template <class MakeProgram>
WalkSet assemble(const WalkConfig& cfg, int32_t walkers, const Geometry& g, const std::vector<Phase>& phases,
                 bool forward, MakeProgram&& make_program) {
    WalkSet ws;
    ws.walkers = walkers;
    ws.phases = static_cast<int32_t>(phases.size());
    ws.page_words = g.W;
    ws.pages = cfg.pages;
    ws.barriers = cfg.barriers;
    ws.rows = g.rows;
    ws.row_bytes = cfg.row_bytes;
    std::vector<Emitter> em(walkers, Emitter{{}, g.W});
    std::vector<int32_t> op_base(walkers, 0);
    for (size_t ph = 0; ph < phases.size(); ++ph) {
        int32_t active = 0;
        for (const auto& l : phases[ph].lists) active += !l.empty();
        const int32_t share = active > 0 ? g.rows / active : g.rows;
        int32_t slot = 0;
        for (int32_t w = 0; w < walkers; ++w) {
            const std::vector<int32_t>& list = phases[ph].lists[w];
            Walk part;
            if (!list.empty()) {
                PlanCfg pc{};
                pc.ring_base = slot * share;
                split_share(cfg, share, pc.ring_rows, pc.stage_rows, int32_t(ph));
                if (pc.ring_rows + pc.stage_rows > share) throw Error(3, "walk ring overrides exceed the CTA budget");
                pc.barriers = cfg.barriers;
                pc.prefetch = cfg.prefetch;
                pc.headroom = cfg.headroom;
                pc.max_copies = (g.W - 5) / 2;
                Program pr = make_program(list);
                part = plan_walker(pr, pc, cfg, g.W, forward);
                part.dst = std::move(pr.dst);
                part.ut = std::move(pr.ut);
                encode(em[w], part, forward, op_base[w], cfg.pairs);
                op_base[w] += static_cast<int32_t>(part.op.size());
                ++slot;
            }
            ws.steps += part.n_steps;
            ws.events += part.events;
            ws.ring_dep_rows += part.ring_dep_rows;
            ws.fetched_rows += part.fetched_rows;
            ws.n_ops += int64_t(part.op.size());
            ws.n_copies += int64_t(part.copies.size());
            ws.global_steps += part.global_steps;
            ws.global_deps += part.global_deps;
            ws.scratch_rows = std::max(ws.scratch_rows, part.scratch_rows);
            ws.parts.push_back(std::move(part));
        }
        if (ph + 1 < phases.size())
            for (auto& e : em) e.emit({kRecSync});
    }
    ws.wpage0.assign(walkers + 1, 0);
    for (int32_t w = 0; w < walkers; ++w) {
        em[w].finish();
        ws.wpage0[w + 1] = ws.wpage0[w] + int32_t(em[w].st.size() / size_t(g.W));
        ws.stream.insert(ws.stream.end(), em[w].st.begin(), em[w].st.end());
    }
    if (ws.smem_bytes() > size_t(cfg.smem_budget)) throw Error(3, "walk exceeds its shared-memory budget");
    return ws;
}

// Phase lists from the level / bin assignment: forward = level 0 (most
// walkers) first, backward = the last level (the serial top) first.
std::vector<Phase> make_phases(const std::vector<int32_t>& level, const std::vector<int32_t>& bin, int32_t K,
                               int32_t levels, bool forward) {
    const int32_t n = static_cast<int32_t>(level.size());
    std::vector<Phase> by_level(levels);
    for (auto& p : by_level) p.lists.resize(K);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t c = forward ? i : n - 1 - i;
        by_level[level[c]].lists[bin[c]].push_back(c);
    }
    std::vector<Phase> ph;
    for (int32_t l = 0; l < levels; ++l) {
        Phase& p = by_level[forward ? l : levels - 1 - l];
        bool any = false;
        for (const auto& x : p.lists) any |= !x.empty();
        if (any) ph.push_back(std::move(p));
    }
    return ph;
}

struct Schedule {
    int32_t K = 1, levels = 1;
    std::vector<int32_t> lvl_walkers, level, bin;
};

// Walkers per level halve until one walks the remaining top alone.
Schedule choose_schedule(const Symbolic& s, const WalkConfig& cfg, Geometry& g, bool backward) {
    Schedule sc;
    sc.K = std::max(1, std::min(cfg.walkers, 16));
    for (;;) {
        g = geometry(s, cfg, sc.K);
        sc.lvl_walkers.clear();
        if (!cfg.levels.empty() && sc.K == cfg.walkers) {
            sc.lvl_walkers = cfg.levels;  // explicit walkers per level (experiments)
        } else {
            for (int32_t k = sc.K; k > 1; k /= 2) sc.lvl_walkers.push_back(k);
            sc.lvl_walkers.push_back(1);
        }
        sc.levels = static_cast<int32_t>(sc.lvl_walkers.size());
        std::vector<int32_t> ring(sc.levels), stage(sc.levels);
        for (int32_t l = 0; l < sc.levels; ++l) split_share(cfg, g.rows / sc.lvl_walkers[l], ring[l], stage[l], l);
        if (partition_levels(s, cfg, sc.lvl_walkers, ring, stage, backward, sc.level, sc.bin)) return sc;
        if (sc.K == 1) throw Error(3, "walk schedule failed with one walker");
        sc.K = 1;  // dependencies cross subtrees: one walker
    }
}

}  // namespace

LuLayout build_lu_layout(const Symbolic& s) {
    const int32_t nJ = s.nJ;
    LuLayout lay;
    lay.lslot.resize(nJ);
    int32_t at = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        lay.lslot[k] = at;
        at += s.cp[k + 1] - s.dpos[k];  // L rows, y_k
    }
    // U rows: entries (k descending) of row i
    std::vector<int32_t> cnt(nJ, 0);
    for (int32_t k = 0; k < nJ; ++k)
        for (int32_t z = s.cp[k]; z < s.dpos[k]; ++z) cnt[s.ri[z]]++;
    lay.ucrs0.assign(nJ + 1, 0);
    lay.ucrs0[0] = at;
    for (int32_t i = 0; i < nJ; ++i) lay.ucrs0[i + 1] = lay.ucrs0[i] + cnt[i] + 2;  // U row, y_i, U(i,i)
    lay.rows = lay.ucrs0[nJ];
    if (lay.rows != s.nnzLU + 2 * nJ) throw Error(2, "LU layout does not cover the pattern");
    lay.tape_of_ccs.assign(s.nnzLU, -1);
    std::vector<int32_t> fill(nJ, 0);
    for (int32_t k = nJ - 1; k >= 0; --k)  // descending k within each row
        for (int32_t z = s.cp[k]; z < s.dpos[k]; ++z) {
            const int32_t i = s.ri[z];
            lay.tape_of_ccs[z] = lay.ucrs0[i] + fill[i]++;
        }
    for (int32_t k = 0; k < nJ; ++k) {
        lay.tape_of_ccs[s.dpos[k]] = lay.ucrs0[k + 1] - 1;  // U(k,k) closes row k's block
        for (int32_t z = s.dpos[k] + 1; z < s.cp[k + 1]; ++z) lay.tape_of_ccs[z] = lay.lslot[k] + (z - s.dpos[k] - 1);
    }
    return lay;
}

// Subtree-to-walker mapping (proportional mapping on the elimination tree),
// level by level: at level l, peel the heaviest subtrees of the still
// unassigned (top) forest -- and any subtree holding a column too big for a
// walker's share at that level -- back into the top, then deal the remaining
// whole subtrees to that level's walkers, heaviest first onto the lightest.
// The last level (one walker) takes whatever is left.  Returns false if some
// dependency would cross walkers (possible only with unsymmetric pivoting).
bool partition_levels(const Symbolic& s, const WalkConfig& cfg, const std::vector<int32_t>& lvl_walkers,
                      const std::vector<int32_t>& ring_w, const std::vector<int32_t>& stage_w, bool backward,
                      std::vector<int32_t>& level, std::vector<int32_t>& bin) {
    const int32_t nJ = s.nJ, L = static_cast<int32_t>(lvl_walkers.size());
    level.assign(nJ, -1);
    bin.assign(nJ, 0);
    const std::vector<int32_t> parent = etree_parent(s);
    std::vector<double> work(nJ);
    std::vector<int32_t> blk(nJ), fetch(nJ), urow(nJ, 0);
    std::vector<std::vector<int32_t>> children(nJ);
    for (int32_t k = 0; k < nJ; ++k)
        for (int32_t z = s.cp[k]; z < s.dpos[k]; ++z) urow[s.ri[z]]++;
    for (int32_t k = 0; k < nJ; ++k) {
        if (parent[k] >= 0 && parent[k] <= k) return false;
        if (!backward) {  // column k of the LU walk: its A block, its L(:,k) + y fetch
            double wk = 60.0 + (s.cp[k + 1] - s.cp[k]);
            for (int32_t z = s.cp[k]; z < s.dpos[k]; ++z) {
                const int32_t j = s.ri[z];
                wk += 12.0 + (s.cp[j + 1] - s.dpos[j] - 1);
            }
            work[k] = wk;
            blk[k] = s.cp[k + 1] - s.cp[k] + 1;
            fetch[k] = s.cp[k + 1] - s.dpos[k];
        } else {  // row k of the backward walk: its U row + y + diagonal, single x rows
            work[k] = 40.0 + 10.0 * urow[k];
            blk[k] = urow[k] + 2;
            fetch[k] = 1;
        }
        if (parent[k] >= 0) children[parent[k]].push_back(k);
    }
    for (int32_t l = 0; l < L; ++l) {
        const int32_t K = lvl_walkers[l];
        if (l == L - 1 || K == 1) {
            for (int32_t k = 0; k < nJ; ++k)
                if (level[k] < 0) level[k] = l, bin[k] = 0;
            break;
        }
        // subtree sums over the unassigned forest (parent > child: one pass)
        std::vector<double> sub(nJ, 0.0);
        std::vector<int32_t> smax_blk(nJ, 0), smax_fetch(nJ, 0);
        double total = 0.0;
        for (int32_t k = 0; k < nJ; ++k) {
            if (level[k] >= 0) continue;
            sub[k] += work[k];
            smax_blk[k] = std::max(smax_blk[k], blk[k]);
            smax_fetch[k] = std::max(smax_fetch[k], fetch[k]);
            total += work[k];
            const int32_t p = parent[k];
            if (p >= 0 && level[p] < 0) {
                sub[p] += sub[k];
                smax_blk[p] = std::max(smax_blk[p], smax_blk[k]);
                smax_fetch[p] = std::max(smax_fetch[p], smax_fetch[k]);
            }
        }
        const double thr = total / (K * cfg.balance);
        std::priority_queue<std::pair<double, int32_t>> heap;
        for (int32_t k = 0; k < nJ; ++k)
            if (level[k] < 0 && (parent[k] < 0 || level[parent[k]] >= 0)) heap.emplace(sub[k], k);
        std::vector<std::pair<double, int32_t>> keep;
        while (!heap.empty()) {
            const auto [wt, r] = heap.top();
            heap.pop();
            if (wt > thr || smax_blk[r] > ring_w[l] || smax_fetch[r] > stage_w[l]) {
                for (int32_t c : children[r])
                    if (level[c] < 0) heap.emplace(sub[c], c);  // r stays in the top
            } else {
                keep.emplace_back(wt, r);
            }
        }
        std::sort(keep.begin(), keep.end(), std::greater<>());
        std::vector<double> load(K, 0.0);
        for (const auto& [wt, r] : keep) {
            const int32_t b = int32_t(std::min_element(load.begin(), load.end()) - load.begin());
            load[b] += wt;
            std::vector<int32_t> st{r};
            while (!st.empty()) {
                const int32_t u = st.back();
                st.pop_back();
                level[u] = l;
                bin[u] = b;
                for (int32_t c : children[u])
                    if (level[c] < 0) st.push_back(c);
            }
        }
    }
    // every dependency must be finished before its consumer runs: a column's U
    // rows (its dependencies) lie in an earlier level or in the same (level,
    // bin); its L rows (its consumers) in a later level or the same (level, bin)
    for (int32_t j = 0; j < nJ; ++j)
        for (int32_t z = s.cp[j]; z < s.cp[j + 1]; ++z) {
            const int32_t k = s.ri[z];
            if (k == j) continue;
            const bool same = level[k] == level[j] && bin[k] == bin[j];
            if (k < j && !(same || level[k] < level[j])) return false;
            if (k > j && !(same || level[k] > level[j])) return false;
        }
    return true;
}

// Forward walk: column m of Alg. 2 (+ row m of the forward substitution).
// Block of column m: its A rows (len) [+ the b row, replaced by y_m].
// Dependencies, ascending k: the union of the U pattern of column m (LU
// updates) and the L pattern of row m (FS terms).
WalkSet build_forward_walk(const Symbolic& s, const LuLayout& lay, bool with_fs, const WalkConfig& cfg) {
    const int32_t nJ = s.nJ;
    std::vector<std::vector<int32_t>> lrow(nJ);  // k with L(m,k) != 0, ascending
    if (with_fs)
        for (int32_t k = 0; k < nJ; ++k)
            for (int32_t z = s.dpos[k] + 1; z < s.cp[k + 1]; ++z) lrow[s.ri[z]].push_back(k);
    Geometry g;
    const Schedule sc = choose_schedule(s, cfg, g, false);
    const std::vector<Phase> phases = make_phases(sc.level, sc.bin, sc.K, sc.levels, true);
    std::vector<int32_t> posmap(nJ, -1), local(nJ, -1);
    auto make_program = [&](const std::vector<int32_t>& list) {
        for (size_t i = 0; i < list.size(); ++i) local[list[i]] = int32_t(i);
        Program pr;
        pr.steps.resize(list.size());
        for (size_t i = 0; i < list.size(); ++i) {
            const int32_t m = list[i];
            const int32_t c0 = s.cp[m], len = s.cp[m + 1] - c0, dp = s.dpos[m] - c0;
            StepIn& si = pr.steps[i];
            si.blk_rows = len + 1;  // row len: b / y (FS), the update padding's scratch row
            si.copies.push_back(copy(kTapeA, a_slot(c0, m), len + 1, 0));  // column + F_m
            si.rec.len_dp = len | (dp << 16);
            si.rec.lslot = lay.lslot[m];
            si.rec.ut0 = static_cast<int32_t>(pr.ut.size());
            si.rec.brow = lay.ucrs0[m + 1] - 2;  // y_m, U(m,m) of the backward block
            si.rec.gslot = a_slot(c0, m);        // the column in the A tape (global form)
            for (int32_t z = c0; z < s.dpos[m]; ++z) pr.ut.push_back(lay.tape_of_ccs[z]);
            for (int32_t z = c0; z < c0 + len; ++z) posmap[s.ri[z]] = z - c0;
            std::vector<int32_t> ks;
            for (int32_t z = c0; z < s.dpos[m]; ++z) ks.push_back(s.ri[z]);
            ks.insert(ks.end(), lrow[m].begin(), lrow[m].end());
            std::sort(ks.begin(), ks.end());
            ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
            for (int32_t k : ks) {
                DepIn di;
                di.producer = local[k] >= 0 && local[k] < int32_t(i) ? local[k] : -1;
                const int32_t lk0 = s.dpos[k] + 1, nl = s.cp[k + 1] - lk0;  // L(:,k) rows
                if (nl == 0) throw Error(2, "walk dependency on an empty L column");
                const int32_t kpos = posmap[k];
                const bool upd = kpos >= 0 && kpos < dp;
                int32_t fspos = 0xffff;
                if (with_fs) {
                    const int32_t* b = s.ri.data() + lk0;
                    const int32_t* f = std::lower_bound(b, b + nl, m);
                    if (f != b + nl && *f == m) fspos = int32_t(f - b);
                }
                if (!upd && fspos == 0xffff) throw Error(2, "walk dependency without a role");
                di.rec.kpos_fs = (upd ? kpos : 0xffff) | (fspos << 16);
                di.rec.nrows = upd ? nl : 0;
                di.rec.u0 = static_cast<int32_t>(pr.dst.size());
                if (upd)
                    for (int32_t zz = lk0; zz < lk0 + nl; ++zz) {
                        const int32_t d = posmap[s.ri[zz]];
                        if (d < 0) throw Error(2, "frozen LU pattern is not closed");
                        pr.dst.push_back(static_cast<uint16_t>(d));
                    }
                const int32_t klen = s.cp[k + 1] - s.cp[k], kdp = s.dpos[k] - s.cp[k];
                di.ring_src = kdp + 1;
                di.ring_ysrc = with_fs ? klen : -1;
                di.rec.gslot = lay.lslot[k];  // L(:,k) then y_k in the LU tape (global form)
                di.rec.gnl = nl;
                di.fetch.push_back(copy(kTapeLU, lay.lslot[k], with_fs ? nl + 1 : nl, 0));  // L rows (+ y_k)
                di.stage_src = 0;
                di.fetch_rows = nl;
                if (with_fs) {
                    di.stage_ysrc = nl;
                    di.fetch_rows = nl + 1;
                }
                si.deps.push_back(std::move(di));
            }
            for (int32_t z = c0; z < c0 + len; ++z) posmap[s.ri[z]] = -1;
        }
        for (int32_t c : list) local[c] = -1;
        return pr;
    };
    WalkSet ws = assemble(cfg, sc.K, g, phases, true, make_program);
    ws.owner.resize(nJ);
    for (int32_t c = 0; c < nJ; ++c) ws.owner[c] = sc.level[c] * 16 + sc.bin[c];
    return ws;
}

// Backward walk: rows i = nJ-1 .. 0.  Block of row i: its U entries (CRS,
// descending k), the y_i row (replaced by x_i) and the diagonal U(i,i).
// Dependencies: x_k for every U(i,k), descending k.
WalkSet build_backward_walk(const Symbolic& s, const LuLayout& lay, const WalkConfig& cfg) {
    const int32_t nJ = s.nJ;
    std::vector<std::vector<int32_t>> urow(nJ);  // k descending
    for (int32_t k = nJ - 1; k >= 0; --k)
        for (int32_t z = s.cp[k]; z < s.dpos[k]; ++z) urow[s.ri[z]].push_back(k);
    Geometry g;
    const Schedule sc = choose_schedule(s, cfg, g, true);
    std::vector<Phase> phases = make_phases(sc.level, sc.bin, sc.K, sc.levels, false);
    std::vector<int32_t> local(nJ, -1);
    if (cfg.pairs) {
        // zip: after each row, pull forward the first of the next 32 rows that needs
        // neither that row nor any other row not yet walked, so consecutive rows are
        // independent as often as possible (encode pairs them into kRecPair records).
        // Any such order is a topological order of the row DAG.
        std::vector<char> out(nJ, 0);
        for (Phase& ph : phases)
            for (std::vector<int32_t>& list : ph.lists) {
                for (size_t t = 0; t < list.size(); ++t) local[list[t]] = int32_t(t);
                auto ready = [&](int32_t r, int32_t without) {
                    for (int32_t k : urow[r])
                        if (local[k] >= 0 && (!out[k] || k == without)) return false;
                    return true;
                };
                std::vector<int32_t> zipped;
                zipped.reserve(list.size());
                std::vector<char> taken(list.size(), 0);
                size_t head = 0;
                while (zipped.size() < list.size()) {
                    while (taken[head]) ++head;
                    const int32_t a = list[head];
                    taken[head] = 1;
                    zipped.push_back(a);
                    out[a] = 1;
                    for (size_t j = head + 1, seen = 0; j < list.size() && seen < 32; ++j) {
                        if (taken[j]) continue;
                        ++seen;
                        if (ready(list[j], a)) {
                            taken[j] = 1;
                            zipped.push_back(list[j]);
                            out[list[j]] = 1;
                            break;
                        }
                    }
                }
                for (int32_t c : list) {
                    local[c] = -1;
                    out[c] = 0;
                }
                list.swap(zipped);
            }
    }
    auto make_program = [&](const std::vector<int32_t>& list) {
        for (size_t t = 0; t < list.size(); ++t) local[list[t]] = int32_t(t);
        Program pr;
        pr.steps.resize(list.size());
        for (size_t t = 0; t < list.size(); ++t) {
            const int32_t i = list[t];
            const int32_t ne = static_cast<int32_t>(urow[i].size());
            StepIn& si = pr.steps[t];
            si.blk_rows = ne + 2;
            si.copies.push_back(copy(kTapeLU, lay.ucrs0[i], ne + 2, 0));  // U row, y_i, U(i,i)
            si.rec.len_dp = ne;
            si.rec.lslot = lay.lslot[i];
            si.rec.brow = nJ - 1 - i;  // x_i's b-tape row: descending k re-fetches ascending rows
            si.rec.gslot = lay.ucrs0[i];  // the row block in the LU tape (global form)
            for (int32_t k : urow[i]) {
                DepIn di;
                di.producer = local[k] >= 0 && local[k] < int32_t(t) ? local[k] : -1;
                di.ring_ysrc = static_cast<int32_t>(urow[k].size());
                di.fetch.push_back(copy(kTapeB, nJ - 1 - k, 1, 0));
                di.rec.gslot = nJ - 1 - k;  // x_k's b-tape row (global form)
                di.stage_ysrc = 0;
                di.fetch_rows = 1;
                si.deps.push_back(std::move(di));
            }
        }
        for (int32_t c : list) local[c] = -1;
        return pr;
    };
    WalkSet ws = assemble(cfg, sc.K, g, phases, false, make_program);
    ws.owner.resize(nJ);
    for (int32_t c = 0; c < nJ; ++c) ws.owner[c] = sc.level[c] * 16 + sc.bin[c];
    return ws;
}

}  // namespace gbnr
