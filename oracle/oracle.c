/*
 * oracle.c -- CPU restatement of the reference executor, TEST INFRASTRUCTURE
 * ONLY. Used by tests/ (parity checker), __graft_entry__.smoke() (checker)
 * and bench.py's cpu_baseline / --impl reference leg. Never part of the
 * product path (paper_2112_09761_b200 does not import or link it).
 *
 * Reference: /root/reference/pkg/src/patminer/executor.py (patminer 0.1.0),
 * a pure Python + numpy package (no native reference to compile). Each
 * function below restates one reference function:
 *
 *   term / eval_set      _TreeRunner._term / _eval        executor.py:124-140
 *   member / bound_hits  _member / _bound_hits            executor.py:142-169
 *   eval_count           _eval_count                      executor.py:171-194
 *   count_from_set       _count_from_set                  executor.py:196-202
 *   apply_terminals      _apply_terminals                 executor.py:204-216
 *   exec_node            exec_node                        executor.py:218-273
 *   run_vertex_task      run_vertex_task                  executor.py:284-295
 *   run_edge_task        run_edge_task                    executor.py:297-325
 *   set kernels          setops.intersect/difference/...  setops.py:21-90
 *
 * Besides the per-pattern counts it accumulates the SURVEY.md 8(d)
 * "algorithmic bytes" exactly as the instrumented reference does:
 * 4*(|a|+|b|) per intersect/difference call (operands as passed),
 * 16 per _term call outside _member, 4 per DESCEND candidate
 * (executor.py:257), 8 per edge task, 4 per vertex task.
 *
 * Counts are 128-bit (the reference uses Python ints).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define MAXL 9          /* levels 1..8 */
#define MAXP 32
#define MAXC 24

enum { B_UNIVERSE = 0, B_NBR = 1, B_BUF = 2 };
enum { A_NONE = 0, A_COUNT = 1, A_BINOM = 2, A_MATCH = 3 };

typedef struct {
    int level;
    int base_kind, base_ref;
    int ni, inter[MAXL];
    int ns, sub[MAXL];
    int label;                 /* -1 none */
    int buffered;
    int nchild, child[MAXC];
    uint32_t members;
    int bound[MAXP];           /* -1 none */
    int action[MAXP];
    int tail[MAXP];
} onode;

typedef struct {
    const uint64_t* off;
    const uint32_t* nbr;
    const uint32_t* labels;
    uint64_t nv;
    const onode* nodes;
    int nnodes;
    const int* roots;
    int nroots;
    int npat;
    uint64_t cap;              /* max degree (set capacity) */
} oracle_ctx;

typedef struct {
    const oracle_ctx* c;
    uint32_t bind[MAXL];
    uint32_t* lvl[MAXL];       /* per-level set storage (s of the node at that level) */
    uint32_t* tmp[4];
    const uint32_t* env[MAXL]; /* buffered sets by level */
    uint64_t envn[MAXL];
    u128 counts[MAXP];
    u128 bytes;
    /* list output (single thread only) */
    uint32_t* mout;
    uint64_t mcap, mcount;
    int width;
} worker;

/* ---- set kernels (setops.py:21-90); results are set-semantics exact ---- */

static uint64_t lower_bound(const uint32_t* a, uint64_t n, uint32_t y) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < y) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static int contains(const uint32_t* a, uint64_t n, uint32_t x) {
    uint64_t i = lower_bound(a, n, x);
    return i < n && a[i] == x;
}

/* out may alias a (written index never passes read index) */
static uint64_t intersect(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
    uint64_t i = 0, j = 0, k = 0;
    if (na > nb) { const uint32_t* t = a; a = b; b = t; uint64_t tn = na; na = nb; nb = tn; }
    if (nb >= 4 * na) {
        for (i = 0; i < na; ++i)
            if (contains(b, nb, a[i])) out[k++] = a[i];
        return k;
    }
    while (i < na && j < nb) {
        if (a[i] == b[j]) { out[k++] = a[i]; ++i; ++j; }
        else if (a[i] < b[j]) ++i;
        else ++j;
    }
    return k;
}

static uint64_t intersect_count(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
    uint64_t i, k = 0;
    if (na > nb) { const uint32_t* t = a; a = b; b = t; uint64_t tn = na; na = nb; nb = tn; }
    for (i = 0; i < na; ++i) k += (uint64_t)contains(b, nb, a[i]);
    return k;
}

static uint64_t difference(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* out) {
    uint64_t i, k = 0;
    for (i = 0; i < na; ++i)
        if (!contains(b, nb, a[i])) out[k++] = a[i];
    return k;
}

static uint64_t difference_count(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
    uint64_t i, k = 0;
    for (i = 0; i < na; ++i) k += (uint64_t)!contains(b, nb, a[i]);
    return k;
}

/* ---- _TreeRunner restatement ---- */

static inline void term(worker* w, int j, const uint32_t** p, uint64_t* n, int counted) {
    const oracle_ctx* c = w->c;
    uint32_t v = w->bind[j];
    *p = c->nbr + c->off[v];
    *n = c->off[v + 1] - c->off[v];
    if (counted) w->bytes += 16;
}

static int cmp_len(const void* x, const void* y) {
    const uint64_t* a = (const uint64_t*)x;
    const uint64_t* b = (const uint64_t*)y;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return a[1] < b[1] ? -1 : (a[1] > b[1]);
}

/* _eval (executor.py:124-140): result written into `out` (capacity cap).
 * Intermediate results ping-pong between `out` and tmp[2] (no aliasing). */
static uint64_t eval_set(worker* w, const onode* nd, uint32_t* out) {
    const oracle_ctx* c = w->c;
    const uint32_t* s;
    uint64_t sn;
    uint32_t* pp[2] = {out, w->tmp[2]};
    int nxt = 0;
    if (nd->base_kind == B_NBR) term(w, nd->base_ref, &s, &sn, 1);
    else { s = w->env[nd->base_ref]; sn = w->envn[nd->base_ref]; }
    if (nd->ni) {
        /* sorted((self._term(j) for j in intersect), key=len): stable by length */
        uint64_t order[MAXL][2];
        for (int q = 0; q < nd->ni; ++q) {
            const uint32_t* tp; uint64_t tn;
            term(w, nd->inter[q], &tp, &tn, 1);
            order[q][0] = tn;
            order[q][1] = (uint64_t)q;
        }
        qsort(order, (size_t)nd->ni, sizeof(order[0]), cmp_len);
        for (int q = 0; q < nd->ni; ++q) {
            const uint32_t* tp; uint64_t tn;
            term(w, nd->inter[order[q][1]], &tp, &tn, 0);
            w->bytes += 4 * (u128)(sn + tn);
            uint32_t* dst = pp[nxt]; nxt ^= 1;
            sn = intersect(s, sn, tp, tn, dst);
            s = dst;
        }
    }
    for (int q = 0; q < nd->ns; ++q) {
        const uint32_t* tp; uint64_t tn;
        term(w, nd->sub[q], &tp, &tn, 1);
        w->bytes += 4 * (u128)(sn + tn);
        uint32_t* dst = pp[nxt]; nxt ^= 1;
        sn = difference(s, sn, tp, tn, dst);
        s = dst;
    }
    if (nd->label >= 0 && c->labels) {
        uint32_t* dst = pp[nxt]; nxt ^= 1;
        uint64_t k = 0;
        for (uint64_t i = 0; i < sn; ++i)
            if (c->labels[s[i]] == (uint32_t)nd->label) dst[k++] = s[i];
        sn = k;
        s = dst;
    }
    if (s != out) memmove(out, s, sn * sizeof(uint32_t));
    return sn;
}

/* _member (executor.py:142-159): no byte accounting (injectivity check). */
static int member(worker* w, const onode* nd, uint32_t v) {
    const oracle_ctx* c = w->c;
    const uint32_t* p; uint64_t n;
    if (nd->base_kind == B_NBR) { term(w, nd->base_ref, &p, &n, 0); if (!contains(p, n, v)) return 0; }
    else if (!contains(w->env[nd->base_ref], w->envn[nd->base_ref], v)) return 0;
    for (int q = 0; q < nd->ni; ++q) { term(w, nd->inter[q], &p, &n, 0); if (!contains(p, n, v)) return 0; }
    for (int q = 0; q < nd->ns; ++q) { term(w, nd->sub[q], &p, &n, 0); if (contains(p, n, v)) return 0; }
    if (nd->label >= 0 && c->labels && c->labels[v] != (uint32_t)nd->label) return 0;
    return 1;
}

static uint64_t bound_hits(worker* w, const onode* nd, int level, int has_bound, uint32_t bv) {
    uint64_t hits = 0;
    for (int l = 1; l < level; ++l) {
        uint32_t v = w->bind[l];
        if (has_bound && v >= bv) continue;
        hits += (uint64_t)member(w, nd, v);
    }
    return hits;
}

/* _eval_count (executor.py:171-194) */
static uint64_t eval_count(worker* w, const onode* nd, int level, int bound) {
    const oracle_ctx* c = w->c;
    int hb = bound >= 0;
    uint32_t bv = hb ? w->bind[bound] : 0;
    uint64_t n;
    if (nd->label >= 0 && c->labels) {
        uint32_t* s = w->tmp[0];
        uint64_t sn = eval_set(w, nd, s);
        if (hb) sn = lower_bound(s, sn, bv);
        n = sn;
    } else {
        const uint32_t* s; uint64_t sn;
        if (nd->base_kind == B_NBR) term(w, nd->base_ref, &s, &sn, 1);
        else { s = w->env[nd->base_ref]; sn = w->envn[nd->base_ref]; }
        if (hb) sn = lower_bound(s, sn, bv);
        int nops = nd->ni + nd->ns;
        if (nops == 0) {
            n = sn;
        } else {
            uint32_t* pp[2] = {w->tmp[1], w->tmp[3]};
            int nxt = 0;
            for (int q = 0; q < nops; ++q) {
                int is_i = q < nd->ni;
                int j = is_i ? nd->inter[q] : nd->sub[q - nd->ni];
                const uint32_t* tp; uint64_t tn;
                term(w, j, &tp, &tn, 1);
                w->bytes += 4 * (u128)(sn + tn);
                if (q + 1 < nops) {
                    uint32_t* buf = pp[nxt]; nxt ^= 1;
                    sn = is_i ? intersect(s, sn, tp, tn, buf) : difference(s, sn, tp, tn, buf);
                    s = buf;
                } else {
                    sn = is_i ? intersect_count(s, sn, tp, tn) : difference_count(s, sn, tp, tn);
                }
            }
            n = sn;
        }
    }
    return n - bound_hits(w, nd, level, hb, bv);
}

static u128 binom(uint64_t n, int t) {
    if ((uint64_t)t > n) return 0;
    u128 r = 1;
    for (int i = 1; i <= t; ++i) r = r * (u128)(n - (uint64_t)t + (uint64_t)i) / (u128)i;
    return r;
}

static void apply_terminals(worker* w, const onode* nd, uint32_t active, const uint32_t* s, uint64_t sn,
                            int have_set) {
    for (int p = 0; p < w->c->npat; ++p) {
        int a = nd->action[p];
        if (!((active >> p) & 1u) || a == A_NONE || a == A_MATCH) continue;
        uint64_t n;
        int b = nd->bound[p];
        if (have_set) {
            uint32_t bv = b >= 0 ? w->bind[b] : 0;
            uint64_t k = b >= 0 ? lower_bound(s, sn, bv) : sn;
            n = k - bound_hits(w, nd, nd->level, b >= 0, bv);
        } else {
            n = eval_count(w, nd, nd->level, b);
        }
        if (a == A_COUNT) w->counts[p] += n;
        else w->counts[p] += binom(n, nd->tail[p]);
    }
}

static void emit(worker* w, int p, int level) {
    w->counts[p] += 1;
    if (w->mout && w->mcount < w->mcap) {
        uint32_t* dst = w->mout + w->mcount * (uint64_t)w->width;
        dst[0] = (uint32_t)p;
        for (int l = 1; l < w->width; ++l) dst[l] = l <= level ? w->bind[l] : 0u;
    }
    if (w->mout) w->mcount++;
}

static void exec_node(worker* w, const onode* nd, uint32_t active) {
    const oracle_ctx* c = w->c;
    const int level = nd->level;
    uint32_t emitters = 0;
    for (int p = 0; p < c->npat; ++p)
        if (nd->action[p] == A_MATCH && ((active >> p) & 1u)) emitters |= 1u << p;
    if (!nd->nchild && !emitters) {
        apply_terminals(w, nd, active, NULL, 0, 0);
        return;
    }
    uint32_t* s = w->lvl[level];
    uint64_t sn = eval_set(w, nd, s);
    if (nd->buffered) { w->env[level] = s; w->envn[level] = sn; }
    apply_terminals(w, nd, active, s, sn, 1);
    uint32_t part = emitters;
    for (int q = 0; q < nd->nchild; ++q) part |= c->nodes[nd->child[q]].members & active;
    if (!part) return;
    uint64_t cut[MAXP];
    uint64_t maxcut = 0;
    for (int p = 0; p < c->npat; ++p) {
        if (!((part >> p) & 1u)) continue;
        int b = nd->bound[p];
        cut[p] = b < 0 ? sn : lower_bound(s, sn, w->bind[b]);
        if (cut[p] > maxcut) maxcut = cut[p];
    }
    for (uint64_t idx = 0; idx < maxcut; ++idx) {
        w->bytes += 4;
        uint32_t v = s[idx];
        int skip = 0;
        for (int l = 1; l < level; ++l) if (w->bind[l] == v) { skip = 1; break; }
        if (skip) continue;
        w->bind[level] = v;
        for (int p = 0; p < c->npat; ++p)
            if (((emitters >> p) & 1u) && idx < cut[p]) emit(w, p, level);
        for (int q = 0; q < nd->nchild; ++q) {
            const onode* ch = &c->nodes[nd->child[q]];
            uint32_t ca = 0;
            for (int p = 0; p < c->npat; ++p)
                if (((ch->members & active) >> p & 1u) && idx < cut[p]) ca |= 1u << p;
            if (ca) exec_node(w, ch, ca);
        }
    }
}

static void run_vertex_task(worker* w, uint32_t v) {
    const oracle_ctx* c = w->c;
    w->bytes += 4;
    for (int r = 0; r < c->nroots; ++r) {
        const onode* root = &c->nodes[c->roots[r]];
        if (root->label >= 0 && c->labels && c->labels[v] != (uint32_t)root->label) continue;
        w->bind[1] = v;
        for (int q = 0; q < root->nchild; ++q) {
            const onode* ch = &c->nodes[root->child[q]];
            uint32_t ca = root->members & ch->members;
            if (ca) exec_node(w, ch, ca);
        }
    }
}

static void run_edge_task(worker* w, uint32_t src, uint32_t dst) {
    const oracle_ctx* c = w->c;
    w->bytes += 8;
    for (int r = 0; r < c->nroots; ++r) {
        const onode* root = &c->nodes[c->roots[r]];
        if (root->label >= 0 && c->labels && c->labels[src] != (uint32_t)root->label) continue;
        w->bind[1] = src;
        for (int q = 0; q < root->nchild; ++q) {
            const onode* ch = &c->nodes[root->child[q]];
            if (ch->label >= 0 && c->labels && c->labels[dst] != (uint32_t)ch->label) continue;
            uint32_t active = 0;
            for (int p = 0; p < c->npat; ++p)
                if (((ch->members >> p) & 1u) && (ch->bound[p] < 0 || dst < src)) active |= 1u << p;
            if (!active) continue;
            w->bind[2] = dst;
            for (int p = 0; p < c->npat; ++p) {
                if (!((active >> p) & 1u)) continue;
                if (ch->action[p] == A_MATCH) emit(w, p, 2);
                else if (ch->action[p] == A_COUNT) w->counts[p] += 1;
            }
            for (int g = 0; g < ch->nchild; ++g) {
                const onode* gc = &c->nodes[ch->child[g]];
                uint32_t ga = active & gc->members;
                if (ga) exec_node(w, gc, ga);
            }
        }
    }
}

/* ---- driver ---- */

typedef struct {
    const oracle_ctx* c;
    int edge;
    const int64_t* tasks;
    uint64_t lo, hi;
    worker w;
    int rc;
} job;

static int worker_init(worker* w, const oracle_ctx* c) {
    memset(w, 0, sizeof(*w));
    w->c = c;
    uint64_t cap = c->cap + 1;
    for (int l = 0; l < MAXL; ++l) {
        w->lvl[l] = (uint32_t*)malloc(cap * sizeof(uint32_t));
        if (!w->lvl[l]) return -1;
    }
    for (int t = 0; t < 4; ++t) {
        w->tmp[t] = (uint32_t*)malloc(cap * sizeof(uint32_t));
        if (!w->tmp[t]) return -1;
    }
    return 0;
}

static void worker_free(worker* w) {
    for (int l = 0; l < MAXL; ++l) free(w->lvl[l]);
    for (int t = 0; t < 4; ++t) free(w->tmp[t]);
}

static void* run_job(void* arg) {
    job* j = (job*)arg;
    for (uint64_t t = j->lo; t < j->hi; ++t) {
        if (j->edge) run_edge_task(&j->w, (uint32_t)j->tasks[2 * t], (uint32_t)j->tasks[2 * t + 1]);
        else run_vertex_task(&j->w, (uint32_t)j->tasks[t]);
    }
    return NULL;
}

/*
 * Run a serialized plan forest over explicit tasks.
 * nodes: array of onode (layout shared with oracle.py), roots: node indices.
 * edge != 0: tasks are (src,dst) int64 pairs; else int64 vertex ids.
 * counts: 2 words (lo, hi) per pattern. bytes: 2 words (lo, hi).
 * match_out (optional, forces 1 thread): (pid, v1..v_{width-1}) tuples.
 * Returns 0 on success, -1 on allocation failure.
 */
int oracle_run(const uint64_t* off, const uint32_t* nbr, const uint32_t* labels, uint64_t nv,
               uint64_t max_degree, const onode* nodes, int nnodes, const int* roots, int nroots,
               int npat, int edge, const int64_t* tasks, uint64_t ntasks, int nthreads,
               uint64_t* counts, uint64_t* bytes, uint32_t* match_out, uint64_t match_cap,
               int width, uint64_t* match_count) {
    oracle_ctx c = {off, nbr, labels, nv, nodes, nnodes, roots, nroots, npat, max_degree};
    if (nthreads < 1) nthreads = 1;
    if (match_out) nthreads = 1;
    if ((uint64_t)nthreads > ntasks) nthreads = ntasks ? (int)ntasks : 1;
    job* jobs = (job*)calloc((size_t)nthreads, sizeof(job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) return -1;
    uint64_t per = ntasks / (uint64_t)nthreads, extra = ntasks % (uint64_t)nthreads, start = 0;
    int rc = 0;
    for (int i = 0; i < nthreads; ++i) {
        jobs[i].c = &c;
        jobs[i].edge = edge;
        jobs[i].tasks = tasks;
        jobs[i].lo = start;
        start += per + ((uint64_t)i < extra ? 1 : 0);
        jobs[i].hi = start;
        if (worker_init(&jobs[i].w, &c)) rc = -1;
        jobs[i].w.mout = match_out;
        jobs[i].w.mcap = match_cap;
        jobs[i].w.width = width;
    }
    if (rc == 0) {
        for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, run_job, &jobs[i]);
        run_job(&jobs[0]);
        for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
        u128 tb = 0;
        for (int p = 0; p < npat; ++p) {
            u128 s = 0;
            for (int i = 0; i < nthreads; ++i) s += jobs[i].w.counts[p];
            counts[2 * p] = (uint64_t)s;
            counts[2 * p + 1] = (uint64_t)(s >> 64);
        }
        for (int i = 0; i < nthreads; ++i) tb += jobs[i].w.bytes;
        bytes[0] = (uint64_t)tb;
        bytes[1] = (uint64_t)(tb >> 64);
        if (match_count) *match_count = jobs[0].w.mcount;
    }
    for (int i = 0; i < nthreads; ++i) worker_free(&jobs[i].w);
    free(jobs);
    free(th);
    return rc;
}

int oracle_node_size(void) { return (int)sizeof(onode); }
