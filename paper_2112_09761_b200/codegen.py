"""PlanForest -> CUDA C++ for sm_100a (one specialised kernel per forest).

The generated kernel is a persistent, warp-per-task-group DFS: every warp
repeatedly grabs a chunk of tasks from a device counter, decodes them into
groups that share v1 (consecutive edge tasks of one CSR row), and runs the
forest's nested loops with all set operations warp-cooperative
(``g2m_device.cuh``). The loop nest, the level expressions, the per-pattern
bounds, the injectivity filter and the terminal actions are all compile-time
constants of the kernel -- this is the B200 analog of the reference's
``emit_source`` (plan.py:334-347) pseudocode, executed instead of printed.

Semantics follow the reference executor exactly (executor.py:113-325):

* node evaluation and per-pattern cuts            executor.py:218-273
* count terminal ``|S ∩ [0, v_b)| - hits``        executor.py:161-202
* binomial terminal ``C(n, t)``                   executor.py:204-216
* edge task level-2 filter ``bound None or dst < src``  executor.py:297-325
* vertex task entry                               executor.py:284-295

Kernel-level optimisation (counts unchanged): an iterating node whose
children are count-only leaves that intersect with ``N(v_L)`` is lowered to a
*flattened* pass -- the 32 lanes share the concatenated neighbour lists of up
to 32 candidates (load-balanced regardless of list lengths) and probe the
loop-invariant lists, which are staged in shared memory when they fit.
Candidates whose list is much longer than the invariant lists are routed to
the generic stream-the-shorter path instead (the reference's own size rule,
setops.py:35-50).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

from .plan import (BINOMIAL_COUNT, EDGE_PARALLEL, EMIT_COUNT, EMIT_MATCH,
                   PlanForest, PlanNode, SetExpr, iter_nodes)

KERNEL_NAME = "g2m_plan_kernel"

# Per-warp shared-memory layout (u32 words) of the flattened-pass metadata.
_FL_WORDS = 32 * 4 + 32 * 2          # end, v, mask, spare + u64 offsets
_FL_CNT_PIDS = 8                     # binomial per-owner counters per child


@dataclass
class GeneratedKernel:
    source: str
    name: str
    num_patterns: int
    num_slots: int
    granularity: int          # 0 edge, 1 vertex
    max_level: int
    labeled: bool
    list_mode: bool
    smem_slot_cap: int        # 0 = global slots
    warps_per_block: int
    warp_words: int           # per-warp dynamic shared memory (u32 words)
    pattern_ids: list[str] = field(default_factory=list)
    hw_levels: int = 0        # buffered nesting depth (high-water slots)

    @property
    def smem_bytes(self) -> int:
        return self.warps_per_block * self.warp_words * 4

    @property
    def key(self) -> str:
        return hashlib.sha1(self.source.encode()).hexdigest()[:16]


class _Out:
    def __init__(self):
        self.lines: list[str] = []
        self.ind = 1

    def __call__(self, text: str = "") -> None:
        for ln in text.split("\n"):
            self.lines.append(("    " * self.ind + ln) if ln else "")

    def push(self, text: str) -> None:
        self(text)
        self.ind += 1

    def pop(self, text: str = "}") -> None:
        self.ind -= 1
        self(text)


def _is_count(action: str) -> bool:
    return action in (EMIT_COUNT, BINOMIAL_COUNT)


class _Gen:
    def __init__(self, forest: PlanForest, labeled: bool, list_mode: bool,
                 smem_slot_cap: int, warps_per_block: int, stage_words: int,
                 flatten: bool, instrument: bool = False, frontier: str | None = None):
        self.f = forest
        self.frontier = frontier         # None | "expand" | "consume"
        self.l3_ids: dict[int, int] = {}  # id(level-3 iterating node) -> item node id
        self.instrument = instrument
        self.labeled = labeled
        self.list_mode = list_mode
        self.smem_cap = smem_slot_cap
        self.wpb = warps_per_block
        self.stage_words = stage_words
        self.flatten = flatten and not list_mode and not instrument
        if not list_mode:
            forest = _as_counting(forest)
            self.f = forest
        self.pids = forest.pattern_ids
        if len(self.pids) > 32:
            raise ValueError("at most 32 patterns per fused forest")
        self.pidx = {p: i for i, p in enumerate(self.pids)}
        self.kmax = max(pl.depth for pl in forest.plans.values())
        self.edge = forest.parallel_granularity == EDGE_PARALLEL
        self.o = _Out()
        self.uid = 0
        # which neighbourhoods / buffers are referenced anywhere
        self.nbr_used: set[int] = set()
        for root in forest.roots:
            for n in iter_nodes(root):
                e = n.expr
                if e.base[0] == "nbr":
                    self.nbr_used.add(e.base[1])
                self.nbr_used.update(e.intersect)
                self.nbr_used.update(e.subtract)
        self.num_slots = 0
        self.hw_levels = 0
        self.stage_used = False
        self.fl_used = False
        if frontier is not None:
            if not self.edge or list_mode or instrument or labeled:
                raise ValueError("frontier kernels need an unlabeled edge-parallel count forest")
            for root in forest.roots:
                for c in root.children:
                    for gc in c.children:
                        if _iterates(gc, False):
                            self.l3_ids[id(gc)] = len(self.l3_ids)

    # -- helpers ------------------------------------------------------------

    def fresh(self, stem: str) -> str:
        self.uid += 1
        return f"{stem}{self.uid}"

    def mask_of(self, pids) -> int:
        m = 0
        for p in pids:
            m |= 1 << self.pidx[p]
        return m

    def label_args(self, expr: SetExpr) -> tuple[str, str]:
        if self.labeled and expr.label is not None:
            return "a.labels", f"{int(expr.label)}u"
        return "(const u32*)nullptr", "0u"

    def is_view(self, expr: SetExpr) -> bool:
        return (not expr.intersect and not expr.subtract
                and (expr.label is None or not self.labeled))

    def lists(self, expr: SetExpr, skip_level: int | None = None):
        """(intersect-side lists, subtract lists) as (ptr, len, is_global)."""
        inter, sub = [], []
        kind, j = expr.base[0], (expr.base[1] if len(expr.base) > 1 else None)
        if kind == "nbr":
            if j != skip_level:
                inter.append((f"nb{j}p", f"nb{j}n", True))
        elif kind == "buf":
            inter.append((f"s{j}p", f"s{j}n", self.smem_cap == 0))
        for i in expr.intersect:
            if i != skip_level:
                inter.append((f"nb{i}p", f"nb{i}n", True))
        for i in expr.subtract:
            sub.append((f"nb{i}p", f"nb{i}n", True))
        return inter, sub

    def ex_decl(self, level: int) -> str:
        """Exclusion array {v1..v_{level-1}} (injectivity, executor.py:161-169,258-264)."""
        vs = ", ".join(f"v{l}" for l in range(1, level))
        return f"const u32 ex[{level - 1}] = {{{vs}}};"

    def bind_level(self, level: int, var: str) -> None:
        o = self.o
        o(f"const u32 v{level} = {var};")
        if level in self.nbr_used:
            o(f"const u64 nb{level}o = __ldg(a.off + v{level});")
            o(f"const u32* nb{level}p = a.nbr + nb{level}o;")
            o(f"const u32 nb{level}n = (u32)(__ldg(a.off + v{level} + 1) - nb{level}o);")

    def acc_add(self, pid: str, action: str, tail: int, nexpr: str) -> None:
        p = self.pidx[pid]
        if action == EMIT_COUNT:
            self.o(f"g2m_acc(acc{p}, (u64)({nexpr}), a.counts + {2 * p});")
        else:
            self.o(f"g2m_acc_binom(acc{p}, (u64)({nexpr}), {tail}, a.counts + {2 * p});")

    def balg_stmt(self, expr: SetExpr, count_bound: str | None, full_eval: bool,
                  cond: str | None = None) -> None:
        """Instrumentation: add the reference's bytes of _eval / _eval_count."""
        inter, sub = self.lists(expr)
        lp = [x[0] for x in inter + sub]
        ln = [x[1] for x in inter + sub]
        nb = 1 if expr.base[0] == "nbr" else 0
        o = self.o
        o.push(f"if ({cond}) {{" if cond else "{")
        o(f"const u32* bl[{len(lp)}] = {{{', '.join(lp)}}};")
        o(f"const u32 bn[{len(ln)}] = {{{', '.join(ln)}}};")
        if full_eval:
            o(f"balg += g2m_balg_eval(bl, bn, {len(inter) - 1}, {len(sub)}, {nb});")
        else:
            o(f"balg += g2m_balg_evalcount(bl, bn, {len(inter) - 1}, {len(sub)}, {nb}, {count_bound});")
        o.pop()

    # -- leaf terminals (not iterated): _eval_count -----------------------------

    def bound_groups(self, node: PlanNode, pids):
        groups: dict[int | None, list[str]] = {}
        for pid in pids:
            groups.setdefault(node.bounds[pid], []).append(pid)
        return groups

    def emit_leaf(self, node: PlanNode, mask: str) -> None:
        o = self.o
        L = node.level
        count_pids = [p for p in sorted(node.actions) if _is_count(node.actions[p][0])]
        if not count_pids:
            return
        inter, sub = self.lists(node.expr)
        lp = [x[0] for x in inter + sub]
        ln = [x[1] for x in inter + sub]
        labp, labv = self.label_args(node.expr)
        if self.instrument:
            full = self.labeled and node.expr.label is not None
            for pid in count_pids:
                b = node.bounds[pid]
                self.balg_stmt(node.expr, f"v{b}" if b is not None else "G2M_NOBOUND", full,
                               cond=f"{mask} & {1 << self.pidx[pid]}u")
        for b, group in self.bound_groups(node, count_pids).items():
            gm = self.mask_of(group)
            o.push(f"if ({mask} & {gm}u) {{")
            o(f"const u32* lp[{len(lp)}] = {{{', '.join(lp)}}};")
            o(f"u32 ln[{len(ln)}] = {{{', '.join(ln)}}};")
            o(self.ex_decl(L))
            bexpr = f"v{b}" if b is not None else "G2M_NOBOUND"
            o(f"const u32 n = g2m_count<{len(inter)}, {len(lp)}, {L - 1}>(lp, ln, {bexpr}, ex, {labp}, {labv});")
            for pid in group:
                act, tail = node.actions[pid]
                if len(group) > 1:
                    o.push(f"if ({mask} & {1 << self.pidx[pid]}u) {{")
                    self.acc_add(pid, act, tail, "n")
                    o.pop()
                else:
                    self.acc_add(pid, act, tail, "n")
            o.pop()

    # -- flattened leaf pass -------------------------------------------------

    def flattenable(self, child: PlanNode, L: int) -> bool:
        if child.children:
            return False
        if any(not _is_count(a) for a, _ in child.actions.values()):
            return False
        if not child.actions:
            return False
        e = child.expr
        on_base = e.base == ("nbr", L)
        if not (on_base or L in e.intersect):
            return False
        if any(a == BINOMIAL_COUNT for a, _ in child.actions.values()) \
                and len(child.actions) > _FL_CNT_PIDS:
            return False
        return True

    def emit_flat(self, child: PlanNode, L: int, cand_p: str, cand_n: str,
                  am_expr: str) -> None:
        """Flattened pass over candidates cand_p[0:cand_n) at level L for
        the leaf `child` (level L+1). am_expr: per-lane C expression for the
        candidate's active mask given `ci` (index) and `cx` (vertex)."""
        o = self.o
        self.fl_used = True
        C = L + 1
        inter, sub = self.lists(child.expr, skip_level=L)
        count_pids = [p for p in sorted(child.actions)]
        binom = [p for p in count_pids if child.actions[p][0] == BINOMIAL_COUNT]
        labp, labv = self.label_args(child.expr)
        o.push("{")
        o(f"// flattened: {child.expr.render()} over v{L} candidates")
        # loop-invariant lists: hash the ones that fit into the warp's shared
        # staging area (membership ~1.5 shared loads); the rest keep a
        # binary search in global memory
        fixed = inter + sub
        names = []
        for idx, (p, n, is_g) in enumerate(fixed):
            fp, fn = f"fp{idx}", f"fn{idx}"
            o(f"const u32* {fp} = {p}; const u32 {fn} = {n};")
            names.append((fp, fn))
        ninter = len(inter)
        hashed = []
        if fixed and self.stage_words > 0:
            self.stage_used = True
            o("u32 stw = 0;")
            for idx in range(len(fixed)):
                fp, fn = names[idx]
                o(f"u32 hl{idx} = {fn} > 8u ? g2m_hlog({fn}) : 0u; u32 ho{idx} = 0;")
                o(f"if (hl{idx} && (1u << hl{idx}) <= {self.stage_words}u - stw) "
                  f"{{ ho{idx} = stw; stw += 1u << hl{idx}; "
                  f"g2m_hset_build(stage + ho{idx}, hl{idx}, {fp}, {fn}); }} else hl{idx} = 0;")
                hashed.append(idx)
        if ninter:
            o(f"u32 fmin = fn0;")
            for idx in range(1, ninter):
                o(f"fmin = min(fmin, fn{idx});")
            o("const u32 heavy_at = 4u * fmin + 128u;")
        for p in count_pids:
            o(f"u64 pa{self.pidx[p]} = 0;")
        o.push(f"for (u32 cb = 0; cb < {cand_n}; cb += 32) {{")
        o("const u32 ci = cb + lane;")
        o(f"bool cv = ci < {cand_n};")
        o(f"const u32 cx = cv ? {cand_p}[ci] : 0u;")
        for l in range(1, L):
            o(f"cv = cv && cx != v{l};")
        o(f"u32 am = cv ? (u32)({am_expr}) : 0u;")
        o("u64 ro = 0; u32 rn = 0;")
        o("if (am) { ro = __ldg(a.off + cx); rn = (u32)(__ldg(a.off + cx + 1) - ro); }")
        if ninter:
            o("const bool heavy = am && rn > heavy_at;")
            o("u32 hm = __ballot_sync(G2M_FULL, heavy);")
            o("if (heavy) rn = 0;")
        o("const u32 incl = g2m_scan_incl(rn);")
        o("const u32 tot = __shfl_sync(G2M_FULL, incl, 31);")
        o("fl_end[lane] = incl; fl_v[lane] = cx; fl_m[lane] = am; fl_off[lane] = ro;")
        for bi, p in enumerate(binom):
            o(f"fl_cnt[{bi} * 32 + lane] = 0;")
        o("__syncwarp();")
        o("u32 ow = 0;")
        o.push("for (u32 e = lane; e < tot; e += 32) {")
        o("while (fl_end[ow] <= e) ++ow;")
        o("const u32 st = ow ? fl_end[ow - 1] : 0u;")
        o("const u32 x = __ldg(a.nbr + fl_off[ow] + (e - st));")
        o("const u32 vo = fl_v[ow];")
        conds = ["x != vo"] + [f"x != v{l}" for l in range(1, L)]
        o(f"bool ok = {' && '.join(conds)};")
        for idx in range(len(fixed)):
            fp, fn = names[idx]
            search = "g2m_has_g" if fixed[idx][2] else "g2m_has"
            test = (f"(hl{idx} ? g2m_hset_has(stage + ho{idx}, hl{idx}, x) : {search}({fp}, {fn}, x))"
                    if idx in hashed else f"{search}({fp}, {fn}, x)")
            o(f"ok = ok && {'' if idx < ninter else '!'}{test};")
        if labp != "(const u32*)nullptr":
            o(f"ok = ok && __ldg(a.labels + x) == {labv};")
        o.push("if (ok) {")
        o("const u32 mo = fl_m[ow];")
        for p in count_pids:
            pi = self.pidx[p]
            b = child.bounds[p]
            cond = f"((mo >> {pi}) & 1u)"
            if b is not None:
                cond += f" && x < {'vo' if b == L else f'v{b}'}"
            if p in binom:
                bi = binom.index(p)
                o(f"if ({cond}) atomicAdd(&fl_cnt[{bi} * 32 + ow], 1u);")
            else:
                o(f"if ({cond}) ++pa{pi};")
        o.pop()
        o.pop()
        o("__syncwarp();")
        for bi, p in enumerate(binom):
            pi = self.pidx[p]
            tail = child.actions[p][1]
            o(f"if ((am >> {pi}) & 1u) pa{pi} += (u64)g2m_binom(fl_cnt[{bi} * 32 + lane], {tail});")
        o("__syncwarp();")
        if ninter:
            # heavy candidates: generic stream-the-shorter path
            o.push("while (hm) {")
            o("const int hj = __ffs(hm) - 1; hm &= hm - 1;")
            o(f"const u32 hmask = __shfl_sync(G2M_FULL, am, hj);")
            o.push("{")
            self.bind_level(L, "__shfl_sync(G2M_FULL, cx, hj)")
            # the generic leaf reads lists named nb{i}/s{j}; loop-invariant
            # staged copies are only an optimisation, so use the originals
            self.emit_leaf(child, "hmask")
            o.pop()
            o.pop()
        o.pop()
        for p in count_pids:
            pi = self.pidx[p]
            if p in binom:
                # per-lane u64 partial of binomials can be large: reduce carefully
                o(f"{{ const u64 w = g2m_wsum(pa{pi}); g2m_acc(acc{pi}, w, a.counts + {2 * pi}); }}")
            else:
                o(f"{{ const u64 w = g2m_wsum(pa{pi}); g2m_acc(acc{pi}, w, a.counts + {2 * pi}); }}")
        o.pop()

    # -- iterating node (exec_node) ---------------------------------------------

    def emit_node(self, node: PlanNode, mask: str, slot_depth: int, buf_depth: int) -> None:
        o = self.o
        L = node.level
        emitters = [p for p in node.actions if node.actions[p][0] == EMIT_MATCH] \
            if self.list_mode else []
        if not node.children and not emitters:
            self.emit_leaf(node, mask)
            return
        o.push(f"{{ // level {L}: S{L} = {node.expr.render()}  [{', '.join(node.members)}]")
        # ---- the level's candidate set
        if self.is_view(node.expr):
            kind, j = node.expr.base
            src = f"nb{j}" if kind == "nbr" else f"s{j}"
            o(f"const u32* s{L}p = {src}p; const u32 s{L}n = {src}n;")
            child_slot = slot_depth
        else:
            inter, sub = self.lists(node.expr)
            lp = [x[0] for x in inter + sub]
            ln = [x[1] for x in inter + sub]
            labp, labv = self.label_args(node.expr)
            self.num_slots = max(self.num_slots, slot_depth + 1)
            o(f"u32* s{L}p = SLOT({slot_depth});")
            o(f"u32 s{L}n;")
            o.push("{")
            o(f"const u32* lp[{len(lp)}] = {{{', '.join(lp)}}};")
            o(f"u32 ln[{len(ln)}] = {{{', '.join(ln)}}};")
            o(f"s{L}n = g2m_materialize<{len(inter)}, {len(lp)}>(lp, ln, {labp}, {labv}, s{L}p);")
            o.pop()
            child_slot = slot_depth + 1
        if self.instrument:
            self.balg_stmt(node.expr, None, True)
        child_buf = buf_depth
        if node.buffered:
            self.hw_levels = max(self.hw_levels, buf_depth + 1)
            if buf_depth < 8:
                o(f"hw{buf_depth} = max(hw{buf_depth}, s{L}n);")
            child_buf = buf_depth + 1
        # ---- terminals applied at this node from the set (_count_from_set);
        # a consume pass already had them applied by its expand pass
        cpids = [p for p in sorted(node.actions) if _is_count(node.actions[p][0])]
        if self.frontier == "consume" and L == 3:
            cpids = []
        for b, group in self.bound_groups(node, cpids).items():
            gm = self.mask_of(group)
            o.push(f"if ({mask} & {gm}u) {{")
            o(self.ex_decl(L))
            if b is None:
                o(f"const u32 cut = s{L}n;")
                o(f"const u32 n = cut - g2m_hits<{L - 1}>(s{L}p, cut, G2M_NOBOUND, ex);")
            else:
                o(f"const u32 cut = g2m_wlb(s{L}p, s{L}n, v{b});")
                o(f"const u32 n = cut - g2m_hits<{L - 1}>(s{L}p, cut, v{b}, ex);")
            for pid in group:
                act, tail = node.actions[pid]
                o.push(f"if ({mask} & {1 << self.pidx[pid]}u) {{")
                self.acc_add(pid, act, tail, "n")
                o.pop()
            o.pop()
        # ---- per-pattern cuts (executor.py:241-253)
        participants = set(emitters)
        for c in node.children:
            participants.update(c.members)
        part_mask = self.mask_of(participants)
        groups = self.bound_groups(node, sorted(participants))
        o.push(f"if ({mask} & {part_mask}u) {{")
        cut_names = {}
        o("u32 maxcut = 0;")
        for gi, (b, group) in enumerate(sorted(groups.items(), key=lambda kv: (kv[0] is None, kv[0] or 0))):
            cn = f"cut{L}_{gi}"
            cut_names[b] = (cn, self.mask_of(group))
            if b is None:
                o(f"const u32 {cn} = s{L}n;")
            else:
                o(f"const u32 {cn} = g2m_wlb(s{L}p, s{L}n, v{b});")
            o(f"if ({mask} & {self.mask_of(group)}u) maxcut = max(maxcut, {cn});")
        if self.instrument:
            o("balg += 4ull * maxcut;")

        def mask_at(idx_var: str) -> str:
            parts = []
            for b, (cn, gm) in cut_names.items():
                if b is None:
                    parts.append(f"{gm}u")
                else:
                    parts.append(f"(({idx_var}) < {cn} ? {gm}u : 0u)")
            return f"({mask} & ({' | '.join(parts)}))"

        if self.frontier == "expand" and L == 3:
            # bounded-frontier BFS: the level-3 candidates become work items
            # of `fchunk` candidates each, (v1, v2, node, first index)
            nid = self.l3_ids[id(node)]
            o.push("if (maxcut) {")
            o("const u32 nit = (maxcut + a.fchunk - 1u) / a.fchunk;")
            o("u64 fb = 0;")
            o("if (lane == 0) fb = atomicAdd(a.frontier_n, (u64)nit);")
            o("fb = __shfl_sync(G2M_FULL, fb, 0);")
            o.push("for (u32 q = lane; q < nit; q += 32) {")
            o(f"if (fb + q < a.frontier_cap) a.frontier[fb + q] = G2MItem{{v1, v2, {nid}u, q * a.fchunk}};")
            o.pop()
            o.pop()
            o.pop()
            o.pop()
            return
        lo, hi = "0u", "maxcut"
        if self.frontier == "consume" and L == 3:
            o("const u32 flo = min(item.lo, maxcut), fhi = min(item.lo + a.fchunk, maxcut);")
            lo, hi = "flo", "fhi"
        flat, loop_children = [], []
        for c in node.children:
            if self.flatten and self.flattenable(c, L):
                flat.append(c)
            else:
                loop_children.append(c)
        for c in flat:
            cm = self.mask_of(c.members)
            o.push(f"if ({mask} & {cm}u) {{")
            if lo == "0u":
                self.emit_flat(c, L, f"s{L}p", "maxcut", f"{mask_at('ci')} & {cm}u")
            else:
                self.emit_flat(c, L, f"(s{L}p + {lo})", f"({hi} - {lo})",
                               f"{mask_at(f'(ci + {lo})')} & {cm}u")
            o.pop()
        if loop_children or emitters:
            o.push(f"for (u32 idx = {lo}; idx < {hi}; ++idx) {{")
            o(f"const u32 cand = s{L}p[idx];")
            skip = " || ".join(f"cand == v{l}" for l in range(1, L))
            o(f"if ({skip}) continue;")
            o(f"const u32 m{L} = {mask_at('idx')};")
            self.bind_level(L, "cand")
            for p in emitters:
                self.emit_match(p, L, f"m{L}")
            for c in loop_children:
                cm = self.mask_of(c.members)
                o.push(f"if (m{L} & {cm}u) {{")
                o(f"const u32 m{L}c = m{L} & {cm}u;")
                self.emit_node(c, f"m{L}c", child_slot, child_buf)
                o.pop()
            o.pop()
        o.pop()
        o.pop()

    def emit_match(self, pid: str, level: int, mask: str) -> None:
        o = self.o
        p = self.pidx[pid]
        o.push(f"if ({mask} & {1 << p}u) {{")
        o(f"++acc{p};")
        o.push("if (a.list_pass) {")
        o("const u64 w = mcur++;")
        o.push("if (lane == 0) {")
        width = self.kmax + 1
        o(f"u32* dst = a.match_buf + w * {width}ull;")
        o(f"dst[0] = {p}u;")
        for l in range(1, self.kmax + 1):
            o(f"dst[{l}] = {f'v{l}' if l <= level else '0u'};")
        o.pop()
        o.pop("} else { ++mcur; }")
        o.pop()

    # -- task entry -------------------------------------------------------------

    def emit_edge_group(self) -> None:
        """Body for a task group (v1, v2s[0:n2)) -- run_edge_task (executor.py:297-325)."""
        o = self.o
        if self.instrument:
            o("balg += 8ull * n2;")
        for root in self.f.roots:
            if root.expr.label is not None and self.labeled:
                o.push(f"if (__ldg(a.labels + v1) == {int(root.expr.label)}u) {{")
            else:
                o.push("{")
            for c in root.children:
                self.emit_level2_edge(c)
            o.pop()

    def emit_level2_edge(self, c: PlanNode) -> None:
        o = self.o
        members = self.mask_of(c.members)
        unbounded = self.mask_of([p for p in c.members if c.bounds[p] is None])
        lab = c.expr.label if (self.labeled and c.expr.label is not None) else None
        # per-task active mask (executor.py:309-311)
        am = f"({unbounded}u | (cx < v1 ? {members}u : 0u))"
        if lab is not None:
            am = f"((__ldg(a.labels + cx) == {int(lab)}u) ? {am} : 0u)"
        o.push(f"{{ // level 2: {c.expr.render()}  [{', '.join(c.members)}]")
        flat, loop_children = [], []
        for gc in c.children:
            if self.flatten and self.flattenable(gc, 2) and not self.list_mode:
                flat.append(gc)
            else:
                loop_children.append(gc)
        term = [p for p in sorted(c.actions)]
        # level-2 count terminals: +1 per active task (count via a lane-parallel pass)
        cnt_terms = [p for p in term if c.actions[p][0] == EMIT_COUNT]
        if cnt_terms:
            o.push("{")
            for p in cnt_terms:
                o(f"u32 t{self.pidx[p]} = 0;")
            o.push("for (u32 cb = 0; cb < n2; cb += 32) {")
            o("const u32 ci = cb + lane; const bool cv = ci < n2;")
            o("const u32 cx = cv ? v2s[ci] : 0u;")
            o(f"const u32 amx = cv ? (u32){am} : 0u;")
            for p in cnt_terms:
                pi = self.pidx[p]
                o(f"t{pi} += __popc(__ballot_sync(G2M_FULL, (amx >> {pi}) & 1u));")
            o.pop()
            for p in cnt_terms:
                pi = self.pidx[p]
                o(f"g2m_acc(acc{pi}, (u64)t{pi}, a.counts + {2 * pi});")
            o.pop()
        for gc in flat:
            cm = self.mask_of(gc.members)
            self.emit_flat(gc, 2, "v2s", "n2", f"{am} & {cm}u")
        emit_terms = [p for p in term if c.actions[p][0] == EMIT_MATCH] if self.list_mode else []
        if loop_children or emit_terms:
            o.push("for (u32 ti = 0; ti < n2; ++ti) {")
            o("const u32 cx = v2s[ti];")
            o(f"const u32 m2 = (u32){am};")
            o.push("if (m2) {")
            self.bind_level(2, "cx")
            for p in emit_terms:
                self.emit_match(p, 2, "m2")
            for gc in loop_children:
                cm = self.mask_of(gc.members)
                o.push(f"if (m2 & {cm}u) {{")
                o(f"const u32 m2c = m2 & {cm}u;")
                self.emit_node(gc, "m2c", 0, 0)
                o.pop()
            o.pop()
            o.pop()
        o.pop()

    def emit_consume_item(self) -> None:
        """Consume pass of the bounded-frontier BFS: one item = (v1, v2,
        level-3 node, first candidate index); re-evaluate that node's set and
        run its subtree for candidates [lo, lo + fchunk)."""
        o = self.o
        o("const u32 cx = item.v2;")
        o.push("switch (item.node) {")
        for root in self.f.roots:
            for c in root.children:
                members = self.mask_of(c.members)
                unbounded = self.mask_of([p for p in c.members if c.bounds[p] is None])
                for gc in c.children:
                    if id(gc) not in self.l3_ids:
                        continue
                    o.push(f"case {self.l3_ids[id(gc)]}u: {{")
                    o(f"const u32 m2 = (u32)({unbounded}u | (cx < v1 ? {members}u : 0u));")
                    self.bind_level(2, "cx")
                    cm = self.mask_of(gc.members)
                    o.push(f"if (m2 & {cm}u) {{")
                    o(f"const u32 m2c = m2 & {cm}u;")
                    self.emit_node(gc, "m2c", 0, 0)
                    o.pop()
                    o("break;")
                    o.pop()
        o.pop()

    def emit_vertex_task(self) -> None:
        """run_vertex_task (executor.py:284-295)."""
        o = self.o
        if self.instrument:
            o("balg += 4;")
        for root in self.f.roots:
            if root.expr.label is not None and self.labeled:
                o.push(f"if (__ldg(a.labels + v1) == {int(root.expr.label)}u) {{")
            else:
                o.push("{")
            rm = self.mask_of(root.members)
            for c in root.children:
                cm = self.mask_of(c.members) & rm
                o.push("{")
                o(f"const u32 m1c = {cm}u;")
                self.emit_node(c, "m1c", 0, 0)
                o.pop()
            o.pop()

    # -- whole kernel -------------------------------------------------------------

    def generate(self) -> GeneratedKernel:
        o = self.o
        body_mark = len(o.lines)
        o.ind = 4
        if self.frontier == "consume":
            self.emit_consume_item()
        elif self.edge:
            self.emit_edge_group()
        else:
            self.emit_vertex_task()
        body = o.lines[body_mark:]
        del o.lines[body_mark:]

        npat = len(self.pids)
        slot_words = self.num_slots * self.smem_cap if self.smem_cap else 0
        fl_words = (_FL_WORDS + _FL_CNT_PIDS * 32) if self.fl_used else 0
        stage_words = self.stage_words if self.stage_used else 0
        warp_words = max(4, (slot_words + fl_words + stage_words + 3) // 4 * 4)
        src = []
        w = src.append
        w("// generated by paper_2112_09761_b200.codegen -- do not edit")
        for root in self.f.roots:
            for n in iter_nodes(root):
                w(f"// L{n.level} {n.expr.render()} members={list(n.members)} "
                  f"bounds={ {k: v for k, v in sorted(n.bounds.items())} } "
                  f"actions={ {k: v for k, v in sorted(n.actions.items())} }")
        w('#include "g2m_device.cuh"')
        w(f"#define NPAT {npat}")
        w(f"#define WARP_WORDS {warp_words}")
        w(f"#define WPB {self.wpb}")
        if self.smem_cap:
            w(f"#define SLOT(d) (wsm + (d) * {self.smem_cap}u)")
        else:
            w(f"#define SLOT(d) (a.scratch + (gwarp * {max(self.num_slots, 1)}ull + (d)) * a.slot_cap)")
        w(f'extern "C" __global__ void __launch_bounds__(WPB * 32) {KERNEL_NAME}(const G2MArgs a) {{')
        w("    extern __shared__ __align__(16) u32 g2m_smem[];")
        w("    const u32 lane = g2m_lane();")
        w("    u32* wsm = g2m_smem + (threadIdx.x >> 5) * WARP_WORDS;")
        w("    const u64 gwarp = (u64)blockIdx.x * WPB + (threadIdx.x >> 5);")
        w("    (void)wsm; (void)gwarp;")
        if self.fl_used:
            base = slot_words
            w(f"    u32* fl_end = wsm + {base};")
            w(f"    u32* fl_v = wsm + {base + 32};")
            w(f"    u32* fl_m = wsm + {base + 64};")
            w(f"    u64* fl_off = (u64*)(wsm + {base + 128});")
            w(f"    u32* fl_cnt = wsm + {base + _FL_WORDS};")
        if self.stage_used:
            w(f"    u32* stage = wsm + {slot_words + fl_words};")
        for p in range(npat):
            w(f"    u64 acc{p} = 0;")
        for d in range(min(self.hw_levels, 8)):
            w(f"    u32 hw{d} = 0;")
        if self.list_mode:
            w("    u64 mcur = 0;")
        if self.instrument:
            w("    u64 balg = 0;")
        w("    u64 row_hint = 0; bool have_hint = false;")
        w("    for (;;) {")
        w("        u64 t0 = 0;")
        w("        if (lane == 0) t0 = atomicAdd(a.next, a.grab);")
        w("        t0 = __shfl_sync(G2M_FULL, t0, 0);")
        w("        if (t0 >= a.ntasks) break;")
        w("        const u64 t1 = min(t0 + a.grab, a.ntasks);")
        w("        have_hint = false;")
        w("        for (u64 t = t0; t < t1;) {")
        if self.frontier == "consume":
            w("            const G2MItem item = a.frontier[t];")
            w("            t += 1;")
            w("            {")
            w("                " + self._bind1_text().replace("v1_", "item.v1"))
        elif self.edge:
            w("            u32 v1_; const u32* v2s; u32 n2; const u64 tgrp = t;")
            w("            if (a.source == 1) {")
            w("                v1_ = __ldg(a.t_src + t); v2s = a.t_dst + t;")
            w("                u64 run = 1;")
            w("                while (t + run < t1) {")
            w("                    const u64 q = t + run + lane;")
            w("                    const bool same = q < t1 && __ldg(a.t_src + q) == v1_;")
            w("                    const u32 bm = __ballot_sync(G2M_FULL, !same);")
            w("                    if (bm) { run += __ffs(bm) - 1; break; }")
            w("                    run += 32;")
            w("                }")
            w("                n2 = (u32)run;")
            w("            } else {")
            w("                const u64 g = g2m_global_task(a, t);")
            w("                const u64 crun = g2m_contig_run(a, t, t1);")
            w("                const u64 row = have_hint ? g2m_row_from(a.task_off, a.nv, row_hint, g)")
            w("                                          : g2m_row_of(a.task_off, a.nv, g);")
            w("                row_hint = row; have_hint = (a.source == 0);")
            w("                const u64 tb = __ldg(a.task_off + row);")
            w("                const u64 te = __ldg(a.task_off + row + 1);")
            w("                const u64 run = min(crun, te - g);")
            w("                v1_ = (u32)row; v2s = a.nbr + __ldg(a.off + row) + (g - tb); n2 = (u32)run;")
            w("            }")
            if self.list_mode:
                w("            n2 = 1;")
            w("            t += n2;")
            w("            {")
            if self.list_mode:
                w("                mcur = a.list_pass ? a.task_match[tgrp - a.task_base] : 0ull;")
            w("                " + self._bind1_text())
        else:
            w("            u32 v1_;")
            w("            const u64 tgrp = t;")
            w("            if (a.source == 2) v1_ = __ldg(a.t_src + t);")
            w("            else v1_ = (u32)g2m_global_task(a, t);")
            w("            t += 1;")
            w("            {")
            if self.list_mode:
                w("                mcur = a.list_pass ? a.task_match[tgrp - a.task_base] : 0ull;")
            w("                " + self._bind1_text())
        src.extend(body)
        if self.list_mode:
            w("                if (!a.list_pass && lane == 0) a.task_match[tgrp - a.task_base] = mcur;")
        w("            }")
        w("        }")
        w("    }")
        for p in range(npat):
            w(f"    if (lane == 0) g2m_add128(a.counts + {2 * p}, acc{p}, 0);")
        for d in range(min(self.hw_levels, 8)):
            w(f"    if (lane == 0 && hw{d}) atomicMax(a.stats + 1 + {d}, (u64)hw{d});")
        if self.instrument:
            w("    if (lane == 0) g2m_add128(a.stats + 9, balg, 0);")
        w("}")
        return GeneratedKernel(
            source="\n".join(src) + "\n", name=KERNEL_NAME, num_patterns=npat,
            num_slots=self.num_slots, granularity=0 if self.edge else 1,
            max_level=self.kmax, labeled=self.labeled, list_mode=self.list_mode,
            smem_slot_cap=self.smem_cap, warps_per_block=self.wpb,
            warp_words=warp_words, pattern_ids=list(self.pids),
            hw_levels=self.hw_levels)

    def _bind1_text(self) -> str:
        if 1 in self.nbr_used:
            return ("const u32 v1 = v1_; const u64 nb1o = __ldg(a.off + v1); "
                    "const u32* nb1p = a.nbr + nb1o; "
                    "const u32 nb1n = (u32)(__ldg(a.off + v1 + 1) - nb1o);")
        return "const u32 v1 = v1_;"


def _iterates(node: PlanNode, list_mode: bool) -> bool:
    return bool(node.children) or (list_mode and any(a == EMIT_MATCH for a, _ in node.actions.values()))


def frontier_nodes(forest: PlanForest) -> int:
    """Level-3 iterating nodes of an edge-parallel forest: the node ids of
    the bounded-frontier BFS items (0 = nothing to split, DFS only)."""
    if forest.parallel_granularity != EDGE_PARALLEL:
        return 0
    return sum(1 for root in forest.roots for c in root.children for gc in c.children
               if _iterates(gc, False))


def _as_counting(forest: PlanForest) -> PlanForest:
    """Count-only view of a forest: an EMIT_MATCH terminal without a sink
    just counts its candidates (executor.py:275-280 with sink=None), which is
    exactly an EMIT_COUNT terminal over the same set and bound."""
    def conv(n: PlanNode) -> PlanNode:
        acts = {p: ((EMIT_COUNT, 0) if a == EMIT_MATCH else (a, t))
                for p, (a, t) in n.actions.items()}
        return PlanNode(level=n.level, expr=n.expr, members=n.members, bounds=dict(n.bounds),
                        actions=acts, buffered=n.buffered,
                        children=tuple(conv(c) for c in n.children))
    return PlanForest(roots=tuple(conv(r) for r in forest.roots), plans=forest.plans,
                      parallel_granularity=forest.parallel_granularity,
                      uses_orientation=forest.uses_orientation,
                      num_buffers=forest.num_buffers)


def slots_needed(forest: PlanForest, labeled: bool) -> int:
    """Materialised-set nesting depth of a forest (per-warp slot count)."""
    def view(e: SetExpr) -> bool:
        return not e.intersect and not e.subtract and (e.label is None or not labeled)

    def walk(node: PlanNode, depth: int, top: bool) -> int:
        iterates = bool(node.children) or any(a == EMIT_MATCH for a, _ in node.actions.values())
        here = depth
        if iterates and not top and not view(node.expr):
            here = depth + 1
        best = here
        for c in node.children:
            best = max(best, walk(c, here, False))
        return best

    edge = forest.parallel_granularity == EDGE_PARALLEL
    best = 0
    for root in forest.roots:
        for c in root.children:
            if edge:
                for gc in c.children:
                    best = max(best, walk(gc, 0, False))
            else:
                best = max(best, walk(c, 0, False))
    return best


def generate(forest: PlanForest, *, labeled: bool = False, list_mode: bool = False,
             smem_slot_cap: int = 0, warps_per_block: int = 8, stage_words: int = 1024,
             flatten: bool = True, instrument: bool = False,
             frontier: str | None = None) -> GeneratedKernel:
    """Emit the CUDA source of one plan forest. ``smem_slot_cap`` > 0 keeps
    materialised sets in shared memory (capacity in u32 per slot); 0 puts
    them in per-warp global scratch. ``frontier`` = "expand" / "consume"
    emits the two passes of the bounded-frontier BFS runtime: expand runs
    levels 1-3 (terminals included) and writes the level-3 candidates as
    work items; consume runs levels >= 4 for one item per task."""
    return _Gen(forest, labeled, list_mode, smem_slot_cap, warps_per_block,
                stage_words, flatten, instrument, frontier).generate()
