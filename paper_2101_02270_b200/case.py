"""Grid case model and MATPOWER-subset parser (host side, numpy).

Mirrors the reference's grid_model module so that callers build exactly the
inputs the reference pipeline builds:

* ``parse_matpower``  -- case_io.hpp:150-240 (tokenizer :55-103, tables :113-135,
  bus typing rule :228-236), then ``finalize`` = grid.hpp:123-173.
* ``GridCase.profiles`` -- grid.hpp:290-344 ``assemble_profiles`` (P0/Q0 :326-327,
  the V0 warm-start rule :331-342, first in-service gen regulates :319).
* ``GridCase.ybus`` -- grid.hpp:208-243 ``build_ybus``; computed by the C++ host
  library (``gbnr_build_ybus``) so complex division rounds exactly like the
  reference's ``std::complex`` code.

Internal bus numbering is file order (grid.hpp:125-129); angles are radians
internally and degrees at the file boundary.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SLACK, PV, PQ = 3, 2, 1


class CaseError(ValueError):
    """Parse (code 1) or structural (code 2) error, mirroring core.hpp:32-65."""

    def __init__(self, msg: str, code: int = 1, line: int = -1):
        super().__init__(msg if line < 0 else f"{msg} (line {line})")
        self.code = code
        self.line = line


@dataclass
class GridCase:
    base_mva: float
    bus_id: np.ndarray      # int64 [n] external ids
    bus_kind: np.ndarray    # int8 [n] 3 slack / 2 pv / 1 pq (after the typing rule)
    pd: np.ndarray          # MW
    qd: np.ndarray          # MVAr
    gs: np.ndarray
    bs: np.ndarray
    vm_init: np.ndarray
    va_init: np.ndarray     # degrees
    base_kv: np.ndarray
    br_f: np.ndarray        # internal from bus
    br_t: np.ndarray        # internal to bus
    br_r: np.ndarray
    br_x: np.ndarray
    br_b: np.ndarray
    br_tap: np.ndarray
    br_shift: np.ndarray    # degrees
    br_on: np.ndarray       # uint8
    br_rate: np.ndarray
    gen_bus: np.ndarray     # internal bus
    gen_p: np.ndarray       # MW
    gen_vm: np.ndarray
    gen_on: np.ndarray      # uint8
    slack: int = 0
    pv: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pq: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    @property
    def n_bus(self) -> int:
        return int(self.bus_id.shape[0])

    @property
    def n_branch(self) -> int:
        return int(self.br_f.shape[0])

    # ------------------------------------------------------------------ Ybus
    def ybus(self):
        """(indptr, indices, diag_ptr, y_re, y_im) -- grid.hpp:208-243."""
        from . import solver

        return solver.build_ybus(self)

    # -------------------------------------------------------------- profiles
    def gen_injection(self) -> tuple[np.ndarray, np.ndarray]:
        """Per-bus in-service generator P (MW) and regulated |V| (grid.hpp:309-320)."""
        n = self.n_bus
        gen_p = np.zeros(n)
        gen_vm = np.zeros(n)
        for g in range(self.gen_bus.shape[0]):
            if not self.gen_on[g]:
                continue
            b = int(self.gen_bus[g])
            gen_p[b] += self.gen_p[g]
            if gen_vm[b] == 0.0:
                gen_vm[b] = self.gen_vm[g]
        return gen_p, gen_vm

    def v_start(self) -> tuple[np.ndarray, np.ndarray]:
        """(vm_start, va_start[rad]) per grid.hpp:331-342 (warm start from the file)."""
        _, gen_vm = self.gen_injection()
        regulated = self.bus_kind != PQ
        vm_set = np.where(regulated & (gen_vm > 0.0), gen_vm, self.vm_init)
        vm0 = np.where(regulated, vm_set, self.vm_init).astype(np.float64)
        va0 = self.va_init * math.pi / 180.0  # core.hpp deg_to_rad: deg * pi / 180
        return vm0, va0.astype(np.float64)

    def profiles(self, p_mw: np.ndarray, q_mvar: np.ndarray,
                 gen_scale: np.ndarray | None = None):
        """Specified injections for load tables [n_bus][n_sets] (MW / MVAr).

        Returns (p0, q0) [n_bus][n_sets] in p.u.: P0 = (Pg - Pd)/base, Q0 = -Qd/base
        (grid.hpp:326-327). ``gen_scale`` ([n_bus][n_sets] or None) multiplies the
        per-bus generator P before the subtraction (Monte-Carlo load/PV mode).
        """
        gen_p, _ = self.gen_injection()
        p_mw = np.asarray(p_mw, np.float64)
        q_mvar = np.asarray(q_mvar, np.float64)
        if p_mw.ndim == 1:
            p_mw = p_mw[:, None]
            q_mvar = q_mvar[:, None]
        g = gen_p[:, None] if gen_scale is None else gen_p[:, None] * gen_scale
        p0 = (g - p_mw) / self.base_mva
        q0 = -q_mvar / self.base_mva
        return p0, q0


# ---------------------------------------------------------------------------
# MATPOWER subset tokenizer / parser (case_io.hpp:55-240)
# ---------------------------------------------------------------------------

def _tokens(text: str):
    line = 1
    cur = []
    out = []
    i = 0
    n = len(text)
    while i < n:
        ch = text[i]
        if ch == "%":
            if cur:
                out.append(("".join(cur), line)); cur = []
            while i < n and text[i] != "\n":
                i += 1
            line += 1
            i += 1
            continue
        if ch == "\n":
            if cur:
                out.append(("".join(cur), line)); cur = []
            line += 1
        elif ch.isspace() or ch == ",":
            if cur:
                out.append(("".join(cur), line)); cur = []
        elif ch in "[];=":
            if cur:
                out.append(("".join(cur), line)); cur = []
            out.append((ch, line))
        else:
            cur.append(ch)
        i += 1
    if cur:
        out.append(("".join(cur), line))
    return out


def _number(tok: str, line: int) -> float:
    # std::from_chars semantics: no leading '+', no '_' separators, nan/inf allowed.
    try:
        if tok == "" or tok[0] == "+" or "_" in tok or tok.strip() != tok:
            raise ValueError
        return float(tok)
    except ValueError:
        raise CaseError(f"malformed numeric field '{tok}'", 1, line) from None


def _is_field(tok: str, name: str) -> bool:
    if tok == name:
        return True
    dot = tok.rfind(".")
    return dot >= 0 and tok[dot + 1:] == name


def _matrix(toks, pos):
    if pos >= len(toks) or toks[pos][0] != "=":
        raise CaseError("expected '=' after table name", 1, toks[pos][1] if pos < len(toks) else -1)
    pos += 1
    if pos >= len(toks) or toks[pos][0] != "[":
        raise CaseError("expected '[' to open table", 1, toks[pos][1] if pos < len(toks) else -1)
    start_line = toks[pos][1]
    pos += 1
    rows, row = [], []
    while pos < len(toks):
        t, ln = toks[pos]
        pos += 1
        if t == "]":
            if row:
                rows.append(row)
            return rows, start_line, pos
        if t == ";":
            if row:
                rows.append(row)
            row = []
            continue
        row.append(_number(t, ln))
    raise CaseError("unterminated table", 1, start_line)


def parse_matpower(text: str) -> GridCase:
    toks = _tokens(text)
    base = None
    bus_t = gen_t = br_t = None
    pos = 0
    while pos < len(toks):
        t, ln = toks[pos]
        pos += 1
        if _is_field(t, "baseMVA"):
            if pos >= len(toks) or toks[pos][0] != "=":
                raise CaseError("expected '=' after baseMVA", 1, ln)
            pos += 1
            if pos >= len(toks):
                raise CaseError("missing baseMVA value", 1, ln)
            base = _number(*toks[pos]); pos += 1
            if pos < len(toks) and toks[pos][0] == ";":
                pos += 1
        elif _is_field(t, "bus"):
            bus_t = _matrix(toks, pos); pos = bus_t[2]
        elif _is_field(t, "gen"):
            gen_t = _matrix(toks, pos); pos = gen_t[2]
        elif _is_field(t, "branch"):
            br_t = _matrix(toks, pos); pos = br_t[2]
    if base is None:
        raise CaseError("missing baseMVA")
    if bus_t is None:
        raise CaseError("missing bus table")
    if br_t is None:
        raise CaseError("missing branch table")

    bus_rows, bus_line, _ = bus_t
    for r in bus_rows:
        if len(r) < 10:
            raise CaseError(f"bus row needs >= 10 columns, got {len(r)}", 1, bus_line)
        if int(r[1]) not in (1, 2, 3):
            raise CaseError(f"unsupported bus type {int(r[1])} (isolated buses are rejected)", 1, bus_line)
    gens = []
    if gen_t is not None:
        for r in gen_t[0]:
            if len(r) < 8:
                raise CaseError(f"gen row needs >= 8 columns, got {len(r)}", 1, gen_t[1])
            gens.append((int(r[0]), r[1], r[5], r[7] > 0.0))
    brs = []
    for r in br_t[0]:
        if len(r) < 11:
            raise CaseError(f"branch row needs >= 11 columns, got {len(r)}", 1, br_t[1])
        brs.append((int(r[0]), int(r[1]), r[2], r[3], r[4], r[5],
                    1.0 if r[8] == 0.0 else r[8], r[9], r[10] > 0.0))

    ids = np.array([int(r[0]) for r in bus_rows], np.int64)
    kind = np.array([int(r[1]) for r in bus_rows], np.int8)
    # bus typing rule (case_io.hpp:228-236)
    has_gen = {g[0] for g in gens if g[3]}
    for i in range(len(ids)):
        if kind[i] != SLACK:
            kind[i] = PV if int(ids[i]) in has_gen else PQ

    col = lambda k: np.array([r[k] for r in bus_rows], np.float64)
    gc = GridCase(
        base_mva=float(base), bus_id=ids, bus_kind=kind,
        pd=col(2), qd=col(3), gs=col(4), bs=col(5), vm_init=col(7), va_init=col(8), base_kv=col(9),
        br_f=np.zeros(len(brs), np.int32), br_t=np.zeros(len(brs), np.int32),
        br_r=np.array([b[2] for b in brs], np.float64), br_x=np.array([b[3] for b in brs], np.float64),
        br_b=np.array([b[4] for b in brs], np.float64), br_tap=np.array([b[6] for b in brs], np.float64),
        br_shift=np.array([b[7] for b in brs], np.float64),
        br_on=np.array([1 if b[8] else 0 for b in brs], np.uint8),
        br_rate=np.array([b[5] for b in brs], np.float64),
        gen_bus=np.zeros(len(gens), np.int32), gen_p=np.array([g[1] for g in gens], np.float64),
        gen_vm=np.array([g[2] for g in gens], np.float64),
        gen_on=np.array([1 if g[3] else 0 for g in gens], np.uint8),
    )
    _finalize(gc, [(b[0], b[1]) for b in brs], [g[0] for g in gens])
    return gc


def _finalize(gc: GridCase, br_ext, gen_ext) -> None:
    """grid.hpp:123-173 -- numbering, index sets, structural validation."""
    index = {}
    for i, bid in enumerate(gc.bus_id.tolist()):
        if bid in index:
            raise CaseError(f"duplicate bus id {bid}", 2)
        index[bid] = i

    def internal(ext):
        if ext not in index:
            raise CaseError(f"unknown bus id {ext}", 2)
        return index[ext]

    slack = [i for i in range(gc.n_bus) if gc.bus_kind[i] == SLACK]
    if len(slack) > 1:
        raise CaseError("duplicate slack bus", 2)
    if not slack:
        raise CaseError("no slack bus", 2)
    for i in range(gc.n_bus):
        if gc.vm_init[i] <= 0.0:
            raise CaseError(f"vm_init must be positive at bus {int(gc.bus_id[i])}", 2)
    gc.slack = slack[0]
    gc.pv = np.array([i for i in range(gc.n_bus) if gc.bus_kind[i] == PV], np.int32)
    gc.pq = np.array([i for i in range(gc.n_bus) if gc.bus_kind[i] == PQ], np.int32)
    for b, (f, t) in enumerate(br_ext):
        gc.br_f[b] = internal(f)
        gc.br_t[b] = internal(t)
        if gc.br_f[b] == gc.br_t[b]:
            raise CaseError(f"branch {b} is a self loop", 2)
        if gc.br_r[b] == 0.0 and gc.br_x[b] == 0.0:
            raise CaseError(f"branch {b} has zero impedance", 2)
        if gc.br_tap[b] <= 0.0:
            raise CaseError(f"branch {b} has tap <= 0", 2)
    for g, ext in enumerate(gen_ext):
        gc.gen_bus[g] = internal(ext)
        if gc.gen_on[g] and gc.bus_kind[gc.gen_bus[g]] == PQ:
            raise CaseError(f"bus {ext} has an in-service generator but kind pq", 2)
    # single island over in-service branches (grid.hpp:92-116)
    adj = [[] for _ in range(gc.n_bus)]
    for b in range(gc.n_branch):
        if gc.br_on[b]:
            adj[gc.br_f[b]].append(int(gc.br_t[b]))
            adj[gc.br_t[b]].append(int(gc.br_f[b]))
    seen = np.zeros(gc.n_bus, bool)
    seen[gc.slack] = True
    stack = [gc.slack]
    while stack:
        u = stack.pop()
        for v in adj[u]:
            if not seen[v]:
                seen[v] = True
                stack.append(v)
    if not seen.all():
        raise CaseError("disconnected island in base case", 2)


# ---------------------------------------------------------------------------
# Scenario and outage files (case_io.hpp:363-471)
# ---------------------------------------------------------------------------

def _internal_bus(gc: GridCase, bus_id: int) -> int:
    """GridCase::internal_bus (grid.hpp:76-81): unknown id -> structural error."""
    hit = np.nonzero(gc.bus_id == bus_id)[0]
    if hit.size == 0:
        raise CaseError(f"unknown bus id {bus_id}", 2)
    return int(hit[0])


def parse_scenario_csv(text: str, gc: GridCase):
    """parse_scenario_csv (case_io.hpp:368-447).  Header ``bus:<id>:p,bus:<id>:q,...``,
    one row per task; the named columns replace those bus loads (MW / MVAr), the
    other buses keep the case loads.  Returns (p_mw, q_mvar) [n_bus][n_tasks];
    malformed input raises CaseError (code 1 parse / 2 unknown bus) with the line."""
    lines = text.split("\n")
    if text == "" or not lines:
        raise CaseError("empty scenario file")

    def split(s):
        return s.replace("\r", "").split(",")

    cols = []
    for h in split(lines[0]):
        if len(h) < 7 or not h.startswith("bus:"):
            raise CaseError(f"bad scenario column '{h}'", 1, 1)
        second = h.find(":", 4)
        if second < 0:
            raise CaseError(f"bad scenario column '{h}'", 1, 1)
        id_str, fld = h[4:second], h[second + 1:]
        if fld not in ("p", "q"):
            raise CaseError(f"scenario column must end in :p or :q, got '{h}'", 1, 1)
        # std::from_chars(int): optional '-', decimal digits, whole token
        body = id_str[1:] if id_str.startswith("-") else id_str
        if not body.isdigit() or not body.isascii():
            raise CaseError(f"bad bus id in column '{h}'", 1, 1)
        cols.append((_internal_bus(gc, int(id_str)), fld == "p"))
    rows = []
    for ln, line in enumerate(lines[1:], start=2):
        if line.strip(" \t\n\v\f\r") == "":
            continue
        cells = split(line)
        if len(cells) != len(cols):
            raise CaseError(f"scenario row has {len(cells)} cells, header has {len(cols)}", 1, ln)
        rows.append([_number(c, ln) for c in cells])
    if not rows:
        raise CaseError("scenario file has no task rows")
    T = len(rows)
    p = np.repeat(gc.pd[:, None].astype(np.float64), T, axis=1)
    q = np.repeat(gc.qd[:, None].astype(np.float64), T, axis=1)
    for t, r in enumerate(rows):
        for (bus, is_p), val in zip(cols, r):
            (p if is_p else q)[bus, t] = val
    return p, q


def parse_outage_list(text: str, gc: GridCase) -> np.ndarray:
    """parse_outage_list (case_io.hpp:449-471): one 0-based branch index per token,
    '#' starts a comment; out-of-range or non-integral indices and an empty list
    are parse errors.  Returns int32 branch indices in file order."""
    out = []
    for ln, line in enumerate(text.split("\n"), start=1):
        line = line.split("#", 1)[0]
        for tok in line.split():
            v = _number(tok, ln)
            idx = int(v) if math.isfinite(v) else -1
            if idx < 0 or idx >= gc.n_branch or float(idx) != v:
                raise CaseError(f"branch index out of range: {tok}", 1, ln)
            out.append(idx)
    if not out:
        raise CaseError("outage list is empty")
    return np.asarray(out, np.int32)


def load_case(path: str) -> GridCase:
    with open(path, "r") as fh:
        return parse_matpower(fh.read())


def write_matpower(gc: GridCase, name: str = "case") -> str:
    """Serialize back to the MATPOWER subset (round-trips through parse_matpower)."""
    lines = [f"function mpc = {name}", "mpc.version = '2';", f"mpc.baseMVA = {gc.base_mva!r};", "",
             "%% bus data", "mpc.bus = ["]
    for i in range(gc.n_bus):
        lines.append("\t" + "\t".join(repr(float(v)) if not float(v).is_integer() else str(int(v)) for v in (
            gc.bus_id[i], gc.bus_kind[i], gc.pd[i], gc.qd[i], gc.gs[i], gc.bs[i], 1,
            gc.vm_init[i], gc.va_init[i], gc.base_kv[i], 1, 1.1, 0.9)) + ";")
    lines += ["];", "", "%% generator data", "mpc.gen = ["]
    for g in range(gc.gen_bus.shape[0]):
        lines.append("\t" + "\t".join(repr(float(v)) if not float(v).is_integer() else str(int(v)) for v in (
            gc.bus_id[gc.gen_bus[g]], gc.gen_p[g], 0, 0, 0, gc.gen_vm[g], gc.base_mva,
            int(gc.gen_on[g]), 0, 0)) + ";")
    lines += ["];", "", "%% branch data", "mpc.branch = ["]
    for b in range(gc.n_branch):
        tap = gc.br_tap[b]
        lines.append("\t" + "\t".join(repr(float(v)) if not float(v).is_integer() else str(int(v)) for v in (
            gc.bus_id[gc.br_f[b]], gc.bus_id[gc.br_t[b]], gc.br_r[b], gc.br_x[b], gc.br_b[b],
            gc.br_rate[b], 0, 0, 0 if tap == 1.0 else tap, gc.br_shift[b], int(gc.br_on[b]))) + ";")
    lines += ["];", ""]
    return "\n".join(lines)
