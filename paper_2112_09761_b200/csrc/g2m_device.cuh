// g2m_device.cuh -- device primitives shared by every generated plan kernel.
//
// Included (as an in-memory NVRTC header) by the CUDA source that codegen.py
// emits for a PlanForest, and by g2m.cu for the fixed kernels.  Everything is
// warp-centric: one warp owns one task group at a time, set operations are
// warp-cooperative (lanes stream one operand, binary-search the others,
// __ballot_sync/__popc compact or count), and every sorted list is a
// (pointer, length) view into the CSR or into a per-warp slot.
//
// Reference semantics reproduced here (pkg/src/patminer/):
//   sorted-set kernels            setops.py:21-90
//   count terminal with bound and
//   injectivity discount          executor.py:161-194, 204-216
//   per-pattern cuts / DFS loop   executor.py:239-273
//   edge / vertex task entry      executor.py:284-325
//   implicit task lists           graph.py:255-286
#pragma once

typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;

#define G2M_FULL 0xffffffffu

// Does this partition own source r? Chunked round-robin over sources:
// chunk = r / rr_chunk, or with the workload estimator (wpre = exclusive
// prefix of per-source estimated work) chunk = wpre[r] / wchunk, i.e.
// consecutive sources of equal estimated work.
__device__ __forceinline__ bool g2m_owns(u64 r, u64 rr_chunk, u32 parts, u32 part, const u64* wpre, u64 wchunk) {
    if (wpre) return ((wpre[r] / wchunk) % parts) == part;
    return !rr_chunk || ((r / rr_chunk) % parts) == part;
}

// Bounded-frontier BFS work item: level-3 candidates [lo, lo + fchunk) of
// level-3 node `node` under the edge task (v1, v2).
struct G2MItem {
    u32 v1, v2, node, lo;
};

// Layout shared with the host (g2m.cu). Plain old data only.
struct G2MArgs {
    const u64* off;         // CSR row offsets [nv+1]
    const u32* nbr;         // CSR neighbour ids
    const u32* labels;      // vertex labels or nullptr
    u64 nv;
    // --- task source ---
    int kind;               // 0 edge, 1 vertex
    int source;             // 0 implicit, 1 explicit pairs, 2 explicit vertices, 3 index
    const u64* task_off;    // implicit edge tasks: per-row task offsets [nv+1]
    const u32* t_src;       // explicit pairs src / explicit vertices
    const u32* t_dst;       // explicit pairs dst
    const u64* t_index;     // index source: implicit task indices
    u64 ntasks;             // tasks this launch iterates (local numbering)
    u64 total_implicit;     // size of the implicit list
    u64 rr_chunk;           // 0 or chunked round-robin partition of the implicit list
    u32 rr_parts, rr_part;
    u64 grab;               // tasks per dynamic work grab
    u64* next;              // work counter
    u64* counts;            // 2 words (lo, hi) per pattern
    u64* stats;             // [0] active tasks, [1..8] slot high water, [9,10] alg bytes
    u32* scratch;           // global per-warp slots (when not in shared memory)
    u64 slot_cap;           // u32 entries per slot
    // --- list mode ---
    u32* match_buf;         // tuples, k words each
    u64 match_cap;          // tuples that fit
    u64* match_count;       // tuples written (count pass: per-task counts)
    u64* task_match;        // list pass: per-task first-tuple index; count pass: per-task counts
    u64 task_base;          // first local task of this list batch
    u64 task_end;           // one past the last local task of this batch
    int list_pass;          // 0 count pass, 1 write pass
    int reserved;
    // --- bounded-frontier BFS (level-3 frontier items: v1, v2, node, lo) ---
    G2MItem* frontier;      // expand: item output; consume: item input
    u64 frontier_cap;       // items that fit (expand)
    u64* frontier_n;        // items produced (expand, may exceed cap)
    u32 fchunk;             // level-3 candidates per item
    u32 reserved2;
};

__device__ __forceinline__ u32 g2m_lane() { return threadIdx.x & 31u; }
__device__ __forceinline__ u32 g2m_lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T g2m_ld(const T* p) { return __ldg(p); }

// ---------------------------------------------------------------------------
// Searches
// ---------------------------------------------------------------------------

// Per-lane lower_bound in a sorted list (generic pointer: global or shared).
__device__ __forceinline__ u32 g2m_lb(const u32* p, u32 n, u32 key) {
    u32 lo = 0;
    while (n > 0) {
        u32 half = n >> 1;
        if (p[lo + half] < key) { lo += half + 1; n -= half + 1; }
        else n = half;
    }
    return lo;
}

// Per-lane membership test (setops.contains, setops.py:87-90).
__device__ __forceinline__ bool g2m_has(const u32* p, u32 n, u32 key) {
    u32 lo = 0;
    while (n > 1) {
        u32 half = n >> 1;
        lo = (p[lo + half] <= key) ? lo + half : lo;
        n -= half;
    }
    return n == 1 && p[lo] == key;
}

// Same, through the read-only path; p must be global.
__device__ __forceinline__ bool g2m_has_g(const u32* p, u32 n, u32 key) {
    u32 lo = 0;
    while (n > 1) {
        u32 half = n >> 1;
        lo = (__ldg(p + lo + half) <= key) ? lo + half : lo;
        n -= half;
    }
    return n == 1 && __ldg(p + lo) == key;
}

// Warp-cooperative lower_bound: 32-ary search, all lanes get the answer
// (setops.bound_list's searchsorted, setops.py:21-23).
__device__ __forceinline__ u32 g2m_wlb(const u32* p, u32 n, u32 key) {
    const u32 lane = g2m_lane();
    u32 lo = 0, hi = n;
    while (hi - lo > 32) {
        u32 seg = (hi - lo + 31) >> 5;
        u32 q = lo + lane * seg;
        bool lt = (q < hi) && (p[q] < key);
        u32 c = __popc(__ballot_sync(G2M_FULL, lt));
        if (c == 0) return lo;
        u32 nlo = lo + (c - 1) * seg + 1;
        u32 nhi = lo + c * seg;
        lo = nlo;
        hi = nhi < hi ? nhi : hi;
    }
    bool lt = (lo + lane < hi) && (p[lo + lane] < key);
    return lo + __popc(__ballot_sync(G2M_FULL, lt));
}

// Row of global implicit task index g: largest r with task_off[r] <= g
// (task_off is non-decreasing, task_off[0] == 0, g < task_off[nv]).
__device__ __forceinline__ u64 g2m_row_of(const u64* to, u64 nv, u64 g) {
    const u32 lane = g2m_lane();
    u64 lo = 0, hi = nv;   // answer in [lo, hi)
    while (hi - lo > 32) {
        u64 seg = (hi - lo + 31) >> 5;
        u64 q = lo + (u64)lane * seg;
        bool le = (q < hi) && (__ldg(to + q) <= g);
        u32 c = __popc(__ballot_sync(G2M_FULL, le));
        // lanes 0..c-1 satisfied; answer in [lo+(c-1)seg, lo+c*seg)
        u64 nlo = lo + (u64)(c - 1) * seg;
        u64 nhi = lo + (u64)c * seg;
        lo = nlo;
        hi = nhi < hi ? nhi : hi;
    }
    bool le = (lo + lane < hi) && (__ldg(to + lo + lane) <= g);
    return lo + __popc(__ballot_sync(G2M_FULL, le)) - 1;
}

// Next row at or after `from` that contains g (fast path for walking rows).
__device__ __forceinline__ u64 g2m_row_from(const u64* to, u64 nv, u64 from, u64 g) {
    const u32 lane = g2m_lane();
    u64 r = from + lane;
    // row r contains g iff to[r] <= g < to[r+1]
    bool past = (r + 1 <= nv) && (__ldg(to + r + 1) <= g);
    u32 m = __ballot_sync(G2M_FULL, !past);
    if (m) return from + (__ffs(m) - 1);
    return g2m_row_of(to, nv, g);
}

// ---------------------------------------------------------------------------
// Counters
// ---------------------------------------------------------------------------

// 128-bit global accumulation as (lo, hi) u64 words.
__device__ __forceinline__ void g2m_add128(u64* c, u64 lo, u64 hi) {
    if (lo) {
        u64 old = atomicAdd(c, lo);
        if (old + lo < old) hi += 1;
    }
    if (hi) atomicAdd(c + 1, hi);
}

// Warp-local u64 accumulator with overflow spill into the 128-bit counter.
__device__ __forceinline__ void g2m_acc(u64& acc, u64 x, u64* c) {
    u64 s = acc + x;
    if (s < acc) {          // wrapped: spill the old value
        if (g2m_lane() == 0) g2m_add128(c, acc, 0);
        s = x;
    }
    acc = s;
}

__device__ __forceinline__ u64 g2m_wsum(u64 v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(G2M_FULL, v, o);
    return v;
}

// C(n, t) in 128 bits (t <= 8): product/division stays exact because each
// partial product C(n, i) is an integer.
__device__ __forceinline__ unsigned __int128 g2m_binom(u64 n, int t) {
    if ((u64)t > n) return 0;
    unsigned __int128 r = 1;
    for (int i = 1; i <= t; ++i) r = r * (unsigned __int128)(n - t + i) / (unsigned __int128)i;
    return r;
}

__device__ __forceinline__ void g2m_acc_binom(u64& acc, u64 n, int t, u64* c) {
    if (t == 2) {
        u64 v = (n < 2) ? 0ull : (n * (n - 1)) >> 1;   // n < 2^32
        g2m_acc(acc, v, c);
        return;
    }
    unsigned __int128 v = g2m_binom(n, t);
    if ((v >> 64) == 0) g2m_acc(acc, (u64)v, c);
    else if (g2m_lane() == 0) g2m_add128(c, (u64)v, (u64)(v >> 64));
}

// ---------------------------------------------------------------------------
// Task decoding (graph.py:255-286, executor.py:284-325)
// ---------------------------------------------------------------------------

// Local (per-launch) task number -> global implicit index.
__device__ __forceinline__ u64 g2m_global_task(const G2MArgs& a, u64 t) {
    if (a.source == 3) return __ldg(a.t_index + t);
    if (a.rr_chunk == 0) return t;
    u64 q = t / a.rr_chunk, r = t - q * a.rr_chunk;
    return (q * a.rr_parts + a.rr_part) * a.rr_chunk + r;
}

// Longest run starting at local task t (bounded by t_end) that stays on one
// row and inside one contiguous stretch of the implicit list.
__device__ __forceinline__ u64 g2m_contig_run(const G2MArgs& a, u64 t, u64 t_end) {
    if (a.source == 3) return 1;
    if (a.rr_chunk == 0) return t_end - t;
    u64 r = t % a.rr_chunk;
    u64 left = a.rr_chunk - r;
    return (t_end - t) < left ? (t_end - t) : left;
}

// Slot-space helpers for implicit edge tasks: row v holds tasks
// [task_off[v], task_off[v+1]); its j-th task is (v, nbr[off[v] + j]).

// ---------------------------------------------------------------------------
// Set expressions  S = L0 & L1 & ... & L(NI-1) - L(NI) - ... - L(NL-1)
// (SetExpr, plan.py:26-60; _eval / _eval_count, executor.py:124-194).
// The shortest intersect-side list is streamed lane-parallel, every other
// list is binary-searched; any stream choice yields the same sorted set.
// ---------------------------------------------------------------------------

#define G2M_NOBOUND 0xffffffffu

template <int NI, int NL>
__device__ __forceinline__ void g2m_pick_stream(const u32* (&lp)[NL], u32 (&ln)[NL]) {
#pragma unroll
    for (int i = 1; i < NI; ++i) {
        if (ln[i] < ln[0]) {
            const u32* tp = lp[0]; lp[0] = lp[i]; lp[i] = tp;
            u32 tn = ln[0]; ln[0] = ln[i]; ln[i] = tn;
        }
    }
}

template <int NI, int NL>
__device__ __forceinline__ bool g2m_pass(const u32* (&lp)[NL], u32 (&ln)[NL], u32 x) {
    bool ok = true;
#pragma unroll
    for (int j = 1; j < NI; ++j) ok = ok && g2m_has(lp[j], ln[j], x);
#pragma unroll
    for (int j = NI; j < NL; ++j) ok = ok && !g2m_has(lp[j], ln[j], x);
    return ok;
}

// |S ∩ [0, bound) \ ex|  -- the count terminal: the reference subtracts the
// bound vertices that are members below the bound (_bound_hits); excluding
// them from the stream is the same quantity.
template <int NI, int NL, int NE>
__device__ __forceinline__ u32 g2m_count(const u32* (&lp)[NL], u32 (&ln)[NL], u32 bound,
                                         const u32 (&ex)[NE], const u32* labels, u32 label) {
    const u32 lane = g2m_lane();
    g2m_pick_stream<NI, NL>(lp, ln);
    const u32* sp = lp[0];
    u32 sn = ln[0];
    if (bound != G2M_NOBOUND) sn = g2m_wlb(sp, sn, bound);
    u32 cnt = 0;
    for (u32 b = 0; b < sn; b += 32) {
        u32 i = b + lane;
        bool ok = i < sn;
        u32 x = ok ? sp[i] : 0u;
#pragma unroll
        for (int e = 0; e < NE; ++e) ok = ok && (x != ex[e]);
        ok = ok && g2m_pass<NI, NL>(lp, ln, x);
        if (labels) ok = ok && (__ldg(labels + x) == label);
        cnt += __popc(__ballot_sync(G2M_FULL, ok));
    }
    return cnt;
}

// Materialise S (full set: no bound, no exclusion -- executor.py:227-237)
// into `out`, preserving ascending order. Returns |S|.
template <int NI, int NL>
__device__ __forceinline__ u32 g2m_materialize(const u32* (&lp)[NL], u32 (&ln)[NL],
                                               const u32* labels, u32 label, u32* out) {
    const u32 lane = g2m_lane();
    __syncwarp();          // lanes may still read out's previous contents (racecheck WAR)
    g2m_pick_stream<NI, NL>(lp, ln);
    const u32* sp = lp[0];
    const u32 sn = ln[0];
    u32 w = 0;
    for (u32 b = 0; b < sn; b += 32) {
        u32 i = b + lane;
        bool ok = i < sn;
        u32 x = ok ? sp[i] : 0u;
        ok = ok && g2m_pass<NI, NL>(lp, ln, x);
        if (labels) ok = ok && (__ldg(labels + x) == label);
        u32 m = __ballot_sync(G2M_FULL, ok);
        if (ok) out[w + __popc(m & g2m_lanemask_lt())] = x;
        w += __popc(m);
    }
    __syncwarp();
    return w;
}

// Number of excluded (bound) vertices present in S[0, cut): the reference's
// _bound_hits on a materialised set (_count_from_set, executor.py:196-202).
template <int NE>
__device__ __forceinline__ u32 g2m_hits(const u32* sp, u32 cut, u32 bound, const u32 (&ex)[NE]) {
    const u32 lane = g2m_lane();
    bool hit = false;
#pragma unroll
    for (int e = 0; e < NE; ++e)
        if (lane == (u32)e) hit = (ex[e] < bound) && g2m_has(sp, cut, ex[e]);
    return __popc(__ballot_sync(G2M_FULL, hit));
}

// Stage a list into shared memory (coalesced copy), returns the smem view.
__device__ __forceinline__ const u32* g2m_stage(const u32* src, u32 n, u32* dst) {
    const u32 lane = g2m_lane();
    __syncwarp();          // previous readers of dst are done (racecheck WAR)
    for (u32 i = lane; i < n; i += 32) dst[i] = __ldg(src + i);
    __syncwarp();
    return dst;
}

__device__ __forceinline__ u32 g2m_scan_incl(u32 x) {
    const u32 lane = g2m_lane();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(G2M_FULL, x, o);
        if (lane >= (u32)o) x += y;
    }
    return x;
}

__device__ __forceinline__ u64 g2m_scan_incl64(u64 x) {
    const u32 lane = g2m_lane();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(G2M_FULL, x, o);
        if (lane >= (u32)o) x += y;
    }
    return x;
}

// ---------------------------------------------------------------------------
// Instrumentation: SURVEY.md 8(d) algorithmic bytes of the REFERENCE plan
// (4*(|a|+|b|) per set op as the reference executor passes its operands,
// 16 per _term call, 4 per DESCEND candidate, 8 / 4 per edge / vertex
// task). Only compiled into instrumented kernels, which run once outside
// any timed region to produce the roofline numerator.
// ---------------------------------------------------------------------------

// |L0 ∩ .. ∩ L(ni-1) - L(ni) - .. - L(nl-1) ∩ [0, bound)| with runtime arity.
__device__ __noinline__ u32 g2m_count_rt(const u32* const* lp, const u32* ln, int ni, int nl,
                                         u32 bound) {
    const u32 lane = g2m_lane();
    int s = 0;
    for (int i = 1; i < ni; ++i) if (ln[i] < ln[s]) s = i;
    const u32* sp = lp[s];
    u32 sn = ln[s];
    if (bound != G2M_NOBOUND) sn = g2m_wlb(sp, sn, bound);
    u32 cnt = 0;
    for (u32 b = 0; b < sn; b += 32) {
        u32 i = b + lane;
        bool ok = i < sn;
        u32 x = ok ? sp[i] : 0u;
        for (int j = 0; j < ni && ok; ++j) if (j != s) ok = g2m_has(lp[j], ln[j], x);
        for (int j = ni; j < nl && ok; ++j) ok = !g2m_has(lp[j], ln[j], x);
        cnt += __popc(__ballot_sync(G2M_FULL, ok));
    }
    return cnt;
}

// Bytes of _eval(expr) (executor.py:124-140): base (+16 when a neighbour
// list), intersect terms sorted by length (stable) each +16 when sorted and
// 4*(|s|+|t|) when applied, then subtract terms +16 and 4*(|s|+|t|).
// lp/ln: [base, intersect terms..., subtract terms...].
__device__ __noinline__ u64 g2m_balg_eval(const u32* const* lp_in, const u32* ln_in, int ni_terms,
                                          int ns, int base_is_nbr) {
    const u32* lp[9];
    u32 ln[9];
    int ord[8];
    for (int q = 0; q < ni_terms; ++q) ord[q] = q;
    for (int q = 1; q < ni_terms; ++q) {          // stable insertion sort by length
        int x = ord[q], r = q - 1;
        while (r >= 0 && ln_in[1 + ord[r]] > ln_in[1 + x]) { ord[r + 1] = ord[r]; --r; }
        ord[r + 1] = x;
    }
    u64 b = base_is_nbr ? 16 : 0;
    b += 16ull * (u64)ni_terms;
    lp[0] = lp_in[0];
    ln[0] = ln_in[0];
    u64 cur = ln_in[0];
    int n = 1;
    for (int q = 0; q < ni_terms; ++q) {
        const int t = 1 + ord[q];
        b += 4ull * (cur + ln_in[t]);
        lp[n] = lp_in[t];
        ln[n] = ln_in[t];
        ++n;
        cur = g2m_count_rt(lp, ln, n, n, G2M_NOBOUND);
    }
    for (int q = 0; q < ns; ++q) {
        const int t = 1 + ni_terms + q;
        b += 16 + 4ull * (cur + ln_in[t]);
        lp[n] = lp_in[t];
        ln[n] = ln_in[t];
        ++n;
        cur = g2m_count_rt(lp, ln, 1 + ni_terms, n, G2M_NOBOUND);
    }
    return b;
}

// Bytes of _eval_count (executor.py:171-194) without a label filter: base
// (+16 if a neighbour list) cut by the bound, then the ops in expression
// order (intersections, then subtractions), each +16 and 4*(|s|+|t|).
__device__ __noinline__ u64 g2m_balg_evalcount(const u32* const* lp_in, const u32* ln_in,
                                               int ni_terms, int ns, int base_is_nbr, u32 bound) {
    const u32* lp[9];
    u32 ln[9];
    u64 b = base_is_nbr ? 16 : 0;
    lp[0] = lp_in[0];
    ln[0] = ln_in[0];
    u64 cur = (bound != G2M_NOBOUND) ? g2m_wlb(lp_in[0], ln_in[0], bound) : ln_in[0];
    const int nops = ni_terms + ns;
    int n = 1;
    for (int q = 0; q < nops; ++q) {
        const int t = 1 + q;
        b += 16 + 4ull * (cur + ln_in[t]);
        lp[n] = lp_in[t];
        ln[n] = ln_in[t];
        ++n;
        if (q + 1 < nops) {
            const int ni = (q < ni_terms) ? n : 1 + ni_terms;
            cur = g2m_count_rt(lp, ln, ni, n, bound);
        }
    }
    return b;
}

// ---------------------------------------------------------------------------
// Shared-memory hash sets / maps for loop-invariant lists (open addressing,
// linear probing, load <= 1/2). Membership then costs ~1.5 shared loads
// instead of log2(n) dependent probes. Vertex id 0xffffffff marks empty
// slots (ids are < 2^32 - 1: GCSR graphs have |V| <= 2^32 - 1).
// ---------------------------------------------------------------------------

#define G2M_EMPTY 0xffffffffu

__device__ __forceinline__ u32 g2m_hslot(u32 x, u32 logcap) {
    return (x * 0x9E3779B1u) >> (32u - logcap);
}

// Smallest logcap with 2n <= 2^logcap (>= 1).
__device__ __forceinline__ u32 g2m_hlog(u32 n) {
    u32 l = 1;
    while ((1u << l) < 2u * n) ++l;
    return l;
}

// Warp-cooperative build of a set over src[0, n) (src global or shared).
__device__ __forceinline__ void g2m_hset_build(u32* keys, u32 logcap, const u32* src, u32 n) {
    const u32 lane = g2m_lane();
    const u32 cap = 1u << logcap;
    for (u32 i = lane; i < cap; i += 32) keys[i] = G2M_EMPTY;
    __syncwarp();
    for (u32 i = lane; i < n; i += 32) {
        const u32 x = src[i];
        u32 h = g2m_hslot(x, logcap);
        while (atomicCAS(&keys[h], G2M_EMPTY, x) != G2M_EMPTY) h = (h + 1) & (cap - 1);
    }
    __syncwarp();
}

__device__ __forceinline__ bool g2m_hset_has(const u32* keys, u32 logcap, u32 x) {
    const u32 mask = (1u << logcap) - 1u;
    u32 h = g2m_hslot(x, logcap);
    for (;;) {
        const u32 k = keys[h];
        if (k == x) return true;
        if (k == G2M_EMPTY) return false;
        h = (h + 1) & mask;
    }
}

// Map variant: vals[slot] = position of the key in src (local id).
__device__ __forceinline__ void g2m_hmap_build(u32* keys, u32* vals, u32 logcap, const u32* src, u32 n,
                                               u32 tid, u32 nthreads) {
    const u32 cap = 1u << logcap;
    for (u32 i = tid; i < cap; i += nthreads) keys[i] = G2M_EMPTY;
    if (nthreads == 32) __syncwarp(); else __syncthreads();
    for (u32 i = tid; i < n; i += nthreads) {
        const u32 x = src[i];
        u32 h = g2m_hslot(x, logcap);
        while (atomicCAS(&keys[h], G2M_EMPTY, x) != G2M_EMPTY) h = (h + 1) & (cap - 1);
        vals[h] = i;
    }
    if (nthreads == 32) __syncwarp(); else __syncthreads();
}

__device__ __forceinline__ u32 g2m_hmap_get(const u32* keys, const u32* vals, u32 logcap, u32 x) {
    const u32 mask = (1u << logcap) - 1u;
    u32 h = g2m_hslot(x, logcap);
    for (;;) {
        const u32 k = keys[h];
        if (k == x) return vals[h];
        if (k == G2M_EMPTY) return G2M_EMPTY;
        h = (h + 1) & mask;
    }
}

// ---------------------------------------------------------------------------
// 1-D bulk copies (TMA engine: cp.async.bulk, SASS UBLKCP) global -> shared,
// completion tracked by a shared-memory mbarrier (transaction bytes).
// Global source and shared destination must be 16-byte aligned and the size
// a multiple of 16: g2m_bulk_list copies the 16-byte-aligned superset of a
// u32 list and returns the list's first element's offset in the copy.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 g2m_smem_addr(const void* p) {
    return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void g2m_mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(g2m_smem_addr(bar)), "r"(count) : "memory");
}

// make initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void g2m_fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// this thread's arrival + the bytes the barrier's phase must also see land
__device__ __forceinline__ void g2m_mbar_arrive_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(g2m_smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void g2m_bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            g2m_smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(g2m_smem_addr(bar))
        : "memory");
}

// wait for the barrier phase with parity `phase` to complete (all threads
// that read the copied data call it; try_wait suspends in hardware)
__device__ __forceinline__ void g2m_mbar_wait(u64* bar, u32 phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W%=;\n}" ::"r"(g2m_smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// Bytes of the aligned copy of list [p, p + n) and the list's offset (u32
// elements) inside it. 16-byte granules: head = (p & 15) / 4 elements.
__device__ __forceinline__ u32 g2m_bulk_span(const u32* p, u32 n, u32* head) {
    const unsigned long long a = (unsigned long long)p;
    const unsigned long long a0 = a & ~15ull;
    const unsigned long long a1 = (a + 4ull * n + 15ull) & ~15ull;
    *head = (u32)((a - a0) >> 2);
    return (u32)(a1 - a0);
}

// One thread: arm `bar` with the copy's bytes and issue it; dst must hold
// g2m_bulk_span bytes (16-byte aligned). Returns the list's offset in dst.
__device__ __forceinline__ u32 g2m_bulk_list(u32* dst, const u32* p, u32 n, u64* bar) {
    u32 head;
    const u32 bytes = g2m_bulk_span(p, n, &head);
    g2m_mbar_arrive_tx(bar, bytes);
    g2m_bulk_g2s(dst, (const void*)((unsigned long long)p & ~15ull), bytes, bar);
    return head;
}
