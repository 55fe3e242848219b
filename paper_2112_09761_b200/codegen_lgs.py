"""Hub-rooted SearchPlan -> bitmap local-graph-search (LGS) kernel for sm_100a.

The reference runs every hub-rooted plan (the first matched vertex -- and,
for edge tasks, the second -- adjacent to all others) inside a per-task
*local graph* (``_LocalRunner`` / ``run_dfs_lgs``, executor.py:415-599;
``build_local_graph`` setops.py:101-142; bitmap helpers setops.py:145-173;
the paper's LGS, "generalizes and automates it for all
hub patterns"). This module lowers such a plan to one CUDA kernel with the
same entry point and argument block as the generated plan kernel
(``g2m_plan_kernel(G2MArgs)``), so ``g2m_run`` / ``g2m_list`` drive it
unchanged -- count mode, and list mode with the exact reference order.

Per task (one warp):

* anchor ``A`` = N(v1) (vertex tasks) or N(v1) ∩ N(v2) (edge tasks), sorted,
  renamed to local ids 0..n-1 (ascending ids, as the reference's LocalGraph);
* local rows ``R[i]`` = bitmap of A ∩ N(A[i]) -- built only when a level
  references a non-anchored level (``needs_rows``, executor.py:432-435) --
  by probing the concatenated out-lists of A against a shared-memory hash
  of A, all 32 lanes busy whatever the list lengths;
* the start level's set is the whole anchor; each later level is
  base & R[..] & ~R[..] over W = ncap/64 words, with the bound vertices'
  bits cleared (``_clear_bound_bits`` :483-492) and the symmetry bound as a
  mask below a local id (``_bound_mask`` :474-481); terminals popcount,
  C(popcount, t), or emit the tuples of the set bits in ascending order.

The start level's candidates are dealt to the lanes in rounds of 32; each
lane runs its candidate's subtree in registers (bit loops, no warp
collectives). In the list write pass a lane first counts its subtree, a
warp scan turns counts into offsets, and the lane re-runs the subtree
writing its tuples there -- so per task the tuples come out in the
reference's DFS order (candidate order, then depth-first).

Rows live in shared memory while the anchor bound ``ncap`` (the graph's
maximum degree rounded up to a multiple of 64) is at most SMEM_NCAP,
otherwise in a per-warp global (L2-resident) slab.
"""
from __future__ import annotations

from .codegen import GeneratedKernel, KERNEL_NAME, _Out
from .plan import BINOMIAL_COUNT, DESCEND, EDGE_PARALLEL, EMIT_COUNT, EMIT_MATCH, SearchPlan

SMEM_NCAP = 256


def lgs_ncap(max_degree: int) -> int:
    """Anchor capacity: the maximum degree rounded up to a power of two >= 64
    (every anchor is a subset of one neighbour list)."""
    nc = 64
    while nc < max_degree:
        nc *= 2
    return nc


def anchored_levels(plan: SearchPlan) -> tuple[int, ...]:
    return (1, 2) if plan.parallel_granularity == EDGE_PARALLEL else (1,)


def needs_rows(plan: SearchPlan) -> bool:
    anch = anchored_levels(plan)
    start = len(anch) + 1
    return any(ref not in anch for lv in plan.levels[start - 1:] for ref in lv.expr.referenced_levels())


def check_plan(plan: SearchPlan) -> None:
    """The reference's structural preconditions (executor.py:415-599)."""
    anch = anchored_levels(plan)
    for lv in plan.levels[len(anch):]:
        if any(j in anch for j in lv.expr.subtract):
            raise ValueError("hub level in a difference term")


class _LgsGen:
    def __init__(self, plan: SearchPlan, list_mode: bool, ncap: int, wpb: int, max_degree: int):
        check_plan(plan)
        self.p = plan
        self.list_mode = list_mode
        self.nc = ncap
        self.W = ncap // 64
        self.wpb = wpb
        self.edge = plan.parallel_granularity == EDGE_PARALLEL
        self.anch = anchored_levels(plan)
        self.S = len(self.anch) + 1
        self.K = plan.depth
        self.rows = needs_rows(plan)
        self.smem = ncap <= SMEM_NCAP
        # per-warp words: R [nc][W] u64 | A [nc] | HK, HV [2nc] each | FL 96
        self.words = (2 * ncap * self.W if self.rows else 0) + ncap + (4 * ncap if self.rows else 0) + 96
        self.max_degree = max(1, max_degree)
        self.o = _Out()

    # -- helpers ----------------------------------------------------------------
    def bind(self, l: int) -> str:
        """Global id bound at level l."""
        if l in self.anch:
            return f"v{l}"
        return f"A[l{l}]"

    def words_for(self, lv, dst: str) -> None:
        """dst[W] = the level's set before clears/bounds (_words_for :457-472)."""
        o, W = self.o, self.W
        e = lv.expr
        kind, j = e.base[0], (e.base[1] if len(e.base) > 1 else None)
        o(f"u64 {dst}[W];")
        o("#pragma unroll")
        o.push("for (int q = 0; q < W; ++q) {")
        if kind == "buf":
            src = "envS[q]" if j == self.S else f"env{j}[q]"
            o(f"{dst}[q] = {src};")
        elif kind == "nbr" and j not in self.anch:
            o(f"{dst}[q] = R[l{j} * W + q];")
        else:           # anchored base (or universe): the whole anchor
            o(f"{dst}[q] = full[q];")
        for i in e.intersect:
            if i not in self.anch:
                o(f"{dst}[q] &= R[l{i} * W + q];")
        for s in e.subtract:
            o(f"{dst}[q] &= ~R[l{s} * W + q];")
        o.pop()

    def clear_bits(self, dst: str, level: int) -> None:
        """_clear_bound_bits (:483-492): anchored vertices present in A, and
        every non-anchored level below."""
        o = self.o
        for l in range(1, level):
            if l in self.anch:
                o(f"if (in{l}) g2m_lgs_clear({dst}, p{l});")
            else:
                o(f"g2m_lgs_clear({dst}, l{l});")

    def cutoff(self, lv) -> str:
        b = lv.bound
        if b is None:
            return "n"
        return f"p{b}" if b in self.anch else f"l{b}"

    def visible(self, src: str, dst: str, cut: str) -> None:
        o = self.o
        o(f"u64 {dst}[W];")
        o("#pragma unroll")
        o(f"for (int q = 0; q < W; ++q) {dst}[q] = {src}[q] & g2m_lgs_below(q, {cut});")

    def popc(self, v: str) -> str:
        return f"g2m_lgs_popc<W>({v})"

    def emit_tuple(self, level: int, off: str) -> None:
        o = self.o
        width = self.K + 1
        o(f"u32* dst = a.match_buf + ({off}) * {width}ull;")
        o("dst[0] = 0u;")
        for l in range(1, self.K + 1):
            o(f"dst[{l}] = {self.bind(l) if l <= level else '0u'};")

    # -- lane-level subtree (levels S+1 .. K) -------------------------------------
    def lane_level(self, L: int) -> None:
        """Level L for one lane; adds matches to c (u128 counts) and, in the
        write pass, writes them at mo++."""
        o = self.o
        lv = self.p.levels[L - 1]
        o.push(f"{{ // level {L}: {lv.expr.render()} bound={lv.bound} {lv.action}")
        self.words_for(lv, f"w{L}")
        self.clear_bits(f"w{L}", L)
        if lv.buffer_slot is not None:
            o(f"u64 env{L}[W];")
            o("#pragma unroll")
            o(f"for (int q = 0; q < W; ++q) env{L}[q] = w{L}[q];")
        self.visible(f"w{L}", f"s{L}", self.cutoff(lv))
        if lv.action == EMIT_COUNT:
            o(f"c += {self.popc(f's{L}')};")
        elif lv.action == BINOMIAL_COUNT:
            o(f"c += g2m_binom({self.popc(f's{L}')}, {int(lv.tail)});")
        else:
            o("#pragma unroll 1")
            o.push("for (int q = 0; q < W; ++q) {")
            o(f"u64 bits = g2m_lgs_get(s{L}, q);")
            o.push("while (bits) {")
            o(f"const u32 l{L} = (u32)q * 64u + (u32)(__ffsll((long long)bits) - 1);")
            o("bits &= bits - 1;")
            if lv.action == EMIT_MATCH:
                if self.list_mode:
                    o.push("if (emit) {")
                    self.emit_tuple(L, "mo")
                    o("++mo;")
                    o.pop()
                o("c += 1;")
            else:
                o(f"(void)l{L};")
                self.lane_level(L + 1)
            o.pop()
            o.pop()
        o.pop()

    # -- kernel -----------------------------------------------------------------
    def generate(self) -> GeneratedKernel:
        o = self.o
        nc, W, S, K = self.nc, self.W, self.S, self.K
        lv_s = self.p.levels[S - 1]
        src = []
        w = src.append
        w("// generated by paper_2112_09761_b200.codegen_lgs -- do not edit")
        w(f"// LGS plan {self.p.pattern_id}: anchored levels {self.anch}, start level {S}, depth {K}, "
          f"rows {'yes' if self.rows else 'no'}, ncap {nc}, {'shared' if self.smem else 'global'} rows")
        for lv in self.p.levels:
            w(f"// L{lv.level} {lv.expr.render()} bound={lv.bound} slot={lv.buffer_slot} {lv.action} t={lv.tail}")
        w('#include "g2m_device.cuh"')
        w(f"#define W {W}")
        w(f"#define NC {nc}u")
        w(f"#define WPB {self.wpb}")
        w(f"#define WARP_WORDS {self.words if self.smem else 4}")
        ns = -(-self.words // self.max_degree) + 1
        ns += ns & 1                     # even: 8-byte aligned per-warp slabs
        w(f"#define NSLOTS {ns}ull")
        w("__device__ __forceinline__ u64 g2m_lgs_below(int q, u32 c) {")
        w("    const u32 w0 = c >> 6;")
        w("    return (u32)q < w0 ? ~0ull : ((u32)q == w0 ? ((1ull << (c & 63u)) - 1ull) : 0ull);")
        w("}")
        w("template <int NW> __device__ __forceinline__ u64 g2m_lgs_popc(const u64 (&v)[NW]) {")
        w("    u64 c = 0;")
        w("#pragma unroll")
        w("    for (int q = 0; q < NW; ++q) c += (u64)__popcll(v[q]);")
        w("    return c;")
        w("}")
        w("// word q / clear bit b of a W-word set held in registers (unrolled selects:")
        w("// a dynamic index would move the array to local memory)")
        w("__device__ __forceinline__ u64 g2m_lgs_get(const u64 (&v)[W], int q) {")
        w("    u64 r = 0;")
        w("#pragma unroll")
        w("    for (int i = 0; i < W; ++i) r = i == q ? v[i] : r;")
        w("    return r;")
        w("}")
        w("__device__ __forceinline__ void g2m_lgs_clear(u64 (&v)[W], u32 b) {")
        w("#pragma unroll")
        w("    for (int i = 0; i < W; ++i) if ((u32)i == (b >> 6)) v[i] &= ~(1ull << (b & 63u));")
        w("}")
        w("// i-th set bit (0-based) of v[W]")
        w("__device__ __forceinline__ u32 g2m_lgs_nth(const u64 (&v)[W], u32 i) {")
        w("    u32 res = 0u;")
        w("    bool done = false;")
        w("#pragma unroll")
        w("    for (int q = 0; q < W; ++q) {")
        w("        const u32 pc = (u32)__popcll(v[q]);")
        w("        if (!done && i < pc) {")
        w("            u64 b = v[q];")
        w("            for (u32 r = 0; r < i; ++r) b &= b - 1;")
        w("            res = (u32)q * 64u + (u32)(__ffsll((long long)b) - 1);")
        w("            done = true;")
        w("        } else if (!done) {")
        w("            i -= pc;")
        w("        }")
        w("    }")
        w("    return res;")
        w("}")
        w(f'extern "C" __global__ void __launch_bounds__(WPB * 32) {KERNEL_NAME}(const G2MArgs a) {{')
        w("    extern __shared__ __align__(16) u32 g2m_smem[];")
        w("    const u32 lane = g2m_lane();")
        w("    const u64 gwarp = (u64)blockIdx.x * WPB + (threadIdx.x >> 5);")
        if self.smem:
            w("    u32* wsm = g2m_smem + (threadIdx.x >> 5) * WARP_WORDS;")
        else:
            w("    u32* wsm = a.scratch + gwarp * NSLOTS * a.slot_cap;")
        w("    (void)gwarp;")
        off = 0
        if self.rows:
            w("    u64* R = (u64*)wsm;")
            off += 2 * nc * W
        w(f"    u32* A = wsm + {off};")
        off += nc
        if self.rows:
            w(f"    u32* HK = wsm + {off};")
            w(f"    u32* HV = wsm + {off + 2 * nc};")
            off += 4 * nc
        w(f"    u32* FLE = wsm + {off};")
        w(f"    u64* FLB = (u64*)(wsm + {off + 32});")
        w("    (void)FLE; (void)FLB;")
        w("    unsigned __int128 acc = 0;")
        w("    for (;;) {")
        w("        u64 t0 = 0;")
        w("        if (lane == 0) t0 = atomicAdd(a.next, a.grab);")
        w("        t0 = __shfl_sync(G2M_FULL, t0, 0);")
        w("        if (t0 >= a.ntasks) break;")
        w("        const u64 t1 = min(t0 + a.grab, a.ntasks);")
        w("        for (u64 t = t0; t < t1; ++t) {")
        o.ind = 3
        self.task_body()
        src.extend(o.lines)
        w("        }")
        w("    }")
        w("    const u64 lo = (u64)acc, hi = (u64)(acc >> 64);")
        w("    if (lo | hi) g2m_add128(a.counts, lo, hi);")
        w("}")
        gen = GeneratedKernel(
            source="\n".join(src) + "\n", name=KERNEL_NAME, num_patterns=1,
            num_slots=0 if self.smem else ns, granularity=0 if self.edge else 1, max_level=K,
            labeled=False, list_mode=self.list_mode, smem_slot_cap=0,
            warps_per_block=self.wpb, warp_words=self.words if self.smem else 4,
            pattern_ids=[self.p.pattern_id], hw_levels=0)
        return gen

    def task_body(self) -> None:
        o = self.o
        S, K = self.S, self.K
        lm = self.list_mode
        # ---- decode the task (executor.py:284-325)
        if self.edge:
            o("u32 v1, v2;")
            o.push("if (a.source == 1) {")
            o("v1 = __ldg(a.t_src + t); v2 = __ldg(a.t_dst + t);")
            o.pop("} else {")
            o.ind += 1
            o("const u64 g = g2m_global_task(a, t);")
            o("const u64 row = g2m_row_of(a.task_off, a.nv, g);")
            o("v1 = (u32)row; v2 = __ldg(a.nbr + __ldg(a.off + row) + (g - __ldg(a.task_off + row)));")
            o.pop()
        else:
            o("const u32 v1 = a.source == 2 ? __ldg(a.t_src + t) : (u32)g2m_global_task(a, t);")
        if lm:
            o("u64 mcur = a.list_pass ? a.task_match[t - a.task_base] : 0ull;")
            o("u64 tcount = 0;")
        o.push("do {")
        if self.edge and self.p.levels[1].bound is not None:
            o("if (!(v2 < v1)) break;   // run_dfs_lgs level-2 filter (executor.py:576-580)")
        # ---- anchor
        o("const u64 o1 = __ldg(a.off + v1); const u32 n1 = (u32)(__ldg(a.off + v1 + 1) - o1);")
        if self.edge:
            o("const u64 o2 = __ldg(a.off + v2); const u32 n2 = (u32)(__ldg(a.off + v2 + 1) - o2);")
            o("const u32* lp[2] = {a.nbr + o1, a.nbr + o2}; u32 ln[2] = {n1, n2};")
            o("const u32 n = g2m_materialize<2, 2>(lp, ln, nullptr, 0u, A);")
        else:
            o("const u32 n = n1;")
            o("g2m_stage(a.nbr + o1, n, A);")
        o("if (n == 0u) break;")
        # anchored positions (searchsorted left) and presence
        for l in self.anch:
            o(f"const u32 p{l} = g2m_lb(A, n, v{l}); const bool in{l} = p{l} < n && A[p{l}] == v{l};")
            o(f"(void)in{l};")
        # ---- local rows (build_local_graph)
        if self.rows:
            self.emit_rows()
        # ---- start level (warp-uniform)
        lv = self.p.levels[S - 1]
        o(f"// start level {S}: {lv.expr.render()} bound={lv.bound} {lv.action}")
        o("u64 full[W];")
        o("#pragma unroll")
        o("for (int q = 0; q < W; ++q) full[q] = g2m_lgs_below(q, n);")
        o("u64 envS[W];")
        o("#pragma unroll")
        o("for (int q = 0; q < W; ++q) envS[q] = full[q];")
        self.clear_bits("envS", S)
        self.visible("envS", "sS", self.cutoff(lv))
        o("const u32 ncand = (u32)g2m_lgs_popc<W>(sS);")
        if lv.action == EMIT_COUNT:
            o("if (lane == 0) acc += ncand;")
            if lm:
                o("tcount += ncand;")
        elif lv.action == BINOMIAL_COUNT:
            o(f"if (lane == 0) acc += g2m_binom(ncand, {int(lv.tail)});")
        elif lv.action == EMIT_MATCH:
            o("if (lane == 0) acc += ncand;")
            if lm:
                o("tcount += ncand;")
                o.push("if (a.list_pass) {")
                o.push("for (u32 r0 = 0; r0 < ncand; r0 += 32) {")
                o(f"const u32 j = r0 + lane;")
                o.push("if (j < ncand) {")
                o(f"const u32 l{S} = g2m_lgs_nth(sS, j);")
                self.emit_tuple(S, "mcur + j")
                o.pop()
                o.pop()
                o.pop()
        else:
            # lanes take the start level's candidates in rounds of 32
            o("const u64 mbase = " + ("mcur" if lm else "0ull") + ";")
            o("u64 carry = 0;")
            o.push("for (u32 r0 = 0; r0 < ncand; r0 += 32) {")
            o("const u32 j = r0 + lane;")
            o("const bool has = j < ncand;")
            o(f"const u32 l{S} = has ? g2m_lgs_nth(sS, j) : 0u;")
            o("unsigned __int128 c = 0;")
            o("u64 mo = 0; const bool emit = false; (void)mo; (void)emit;")
            o.push("if (has) {")
            self.lane_level(S + 1)
            o.pop()
            if lm:
                o("const u64 cc = (u64)c;")
                o("const u64 incl = g2m_scan_incl64(cc);")
                o.push("if (a.list_pass && has && cc) {")
                o("u64 mo = mbase + carry + incl - cc; const bool emit = true; unsigned __int128 c = 0;")
                self.lane_level(S + 1)
                o("(void)c;")
                o.pop()
                o("carry += __shfl_sync(G2M_FULL, incl, 31);")
                o("acc += cc;")
            else:
                o("acc += c;")
            o.pop()
            if lm:
                o("tcount += carry;")
        o.pop("} while (0);")
        if lm:
            o("if (!a.list_pass && lane == 0) a.task_match[t - a.task_base] = tcount;")

    def emit_rows(self) -> None:
        """R[i] = bitmap of A ∩ N(A[i]) (setops.build_local_graph :124-142):
        the out-lists of 32 rows at a time concatenated over the lanes, each
        element looked up in a hash map of A (local id or empty)."""
        o = self.o
        o("const u32 hl = g2m_hlog(n);")
        o("g2m_hmap_build(HK, HV, hl, A, n, lane, 32);")
        o("for (u32 x = lane; x < n * W; x += 32) R[x] = 0ull;")
        o("__syncwarp();")
        o.push("for (u32 i0 = 0; i0 < n; i0 += 32) {")
        o("const u32 i = i0 + lane;")
        o("u64 ro = 0; u32 rn = 0;")
        o("if (i < n) { const u32 y = A[i]; ro = __ldg(a.off + y); rn = (u32)(__ldg(a.off + y + 1) - ro); }")
        o("const u32 incl = g2m_scan_incl(rn);")
        o("const u32 tot = __shfl_sync(G2M_FULL, incl, 31);")
        o("FLE[lane] = incl; FLB[lane] = ro - (u64)(incl - rn);")
        o("__syncwarp();")
        o("u32 ow = 0;")
        o.push("for (u32 e = lane; e < tot; e += 32) {")
        o("while (FLE[ow] <= e) ++ow;")
        o("const u32 x = __ldg(a.nbr + FLB[ow] + e);")
        o("const u32 pos = g2m_hmap_get(HK, HV, hl, x);")
        o("if (pos != G2M_EMPTY) atomicOr((u32*)(R + (u64)(i0 + ow) * W) + (pos >> 5), 1u << (pos & 31u));")
        o.pop()
        o("__syncwarp();")
        o.pop()


def generate_lgs(plan: SearchPlan, *, list_mode: bool, max_degree: int, wpb: int = 4) -> GeneratedKernel:
    nc = lgs_ncap(max_degree)
    return _LgsGen(plan, list_mode, nc, wpb, max_degree).generate()
