/*
 * g2m.h -- C ABI of libg2m.so, the B200 (sm_100a) pattern-mining engine.
 *
 * This is the drop-in boundary behind the reference package's execution
 * operators.  Every entry point uses plain pointers and fixed-width integers
 * (no torch / numpy / C++ types), returns a status code and leaves a
 * thread-local message in g2m_last_error() on failure.
 *
 * Reference interfaces replaced (paths relative to the reference package
 * pkg/src/patminer/):
 *
 *   g2m_graph_create        Graph(row_offsets, neighbors, labels, oriented)
 *                            graph.py:38-61 -- host CSR (u64 offsets,
 *                            u32 ids) becomes a device-resident replica.
 *   g2m_graph_from_edges    from_edges(edges, num_vertices, labels)
 *                            graph.py:116-142 -- drop self loops,
 *                            symmetrise, dedup, CSR, on the device.
 *   g2m_graph_orient        orient(g) graph.py:204-221 -- keep u->v iff
 *                            (deg_u,u) < (deg_v,v), on the device.
 *   g2m_graph_download      host view of a device graph (Graph arrays).
 *   g2m_kernel_compile      the "codegen" step: the CUDA source emitted for
 *                            one PlanForest (plan.py:205-301; analog of
 *                            emit_source plan.py:334-347) is compiled with
 *                            NVRTC for sm_100a.
 *   g2m_run                 run_dfs(g, forest, tasks, cfg, sink=None)
 *                            executor.py:339-408 (count terminals) and
 *                            run_dfs_lgs executor.py:526-599; one call per
 *                            device -- scheduler.run_on_devices
 *                            (scheduler.py:207-239) issues one per GPU.
 *   g2m_run_bfs             run_dfs through the bounded-frontier BFS
 *                            runtime (same counts; DFS/BFS chooser in
 *                            executor.choose_search).
 *   g2m_list                run_dfs(..., sink) list mode: matches are
 *                            produced on the device in exact reference
 *                            order (task order, then DFS order) and handed
 *                            to the host in batches (executor.py:275-280).
 *   g2m_cycle4_count        run_dfs for the count-mode 4-cycle plan
 *                            (executor.py:339-408 over plan.py:110-174):
 *                            same count, wedge-aggregation kernels.
 *   g2m_diamond_count       run_dfs for the count-mode diamond plan with
 *                            the counting rewrite (executor.py:204-216):
 *                            same count, edge triangle-support kernels.
 *   g2m_setop_batch         setops.intersect/intersect_count/difference/
 *                            difference_count (setops.py:35-84) as a
 *                            batched device call (kernel-library parity).
 *
 * Status codes map onto the reference's exceptions:
 *   G2M_OK 0, G2M_EUSAGE 1 -> ValueError, G2M_EBUDGET 2 -> BudgetError,
 *   G2M_ECUDA 3 -> RuntimeError, G2M_STOPPED 4 -> RunResult.stopped_early.
 */
#ifndef G2M_H
#define G2M_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define G2M_ABI_VERSION 7

#define G2M_OK 0
#define G2M_EUSAGE 1
#define G2M_EBUDGET 2
#define G2M_ECUDA 3
#define G2M_STOPPED 4

/* Task kinds (executor.py:284-325). */
#define G2M_TASKS_EDGE 0
#define G2M_TASKS_VERTEX 1

/* Task sources. IMPLICIT: the default task list of run_dfs/run_job
 * (graph.py:270-286 all_edge_tasks / reduced src>dst, or arange(|V|)),
 * generated on the device in the reference's order.  PAIRS: an explicit
 * EdgeTaskList.edges int64 (m,2) array.  VERTICES: explicit int64 vertex
 * ids.  INDEX: int64 indices into the IMPLICIT list (Schedule queues,
 * scheduler.py:27-105). */
#define G2M_SRC_IMPLICIT 0
#define G2M_SRC_PAIRS 1
#define G2M_SRC_VERTICES 2
#define G2M_SRC_INDEX 3

typedef struct g2m_graph g2m_graph;
typedef struct g2m_kernel g2m_kernel;

typedef struct g2m_graph_info {
    uint64_t num_vertices;
    uint64_t num_slots;     /* directed CSR entries == Graph.num_edges */
    uint64_t max_degree;    /* Graph.max_degree (out-degree if oriented) */
    int32_t oriented;
    int32_t labeled;
    int32_t device;
    int32_t reserved;
    uint64_t sum_degree_sq; /* Σ_v degree(v)^2 (frontier bound of the BFS runtime) */
} g2m_graph_info;

typedef struct g2m_task_spec {
    int32_t kind;           /* G2M_TASKS_EDGE / G2M_TASKS_VERTEX */
    int32_t source;         /* G2M_SRC_* */
    int32_t reduced;        /* IMPLICIT/INDEX edge lists: only src > dst */
    int32_t weighted;       /* source-partitioned kernels (g2m_clique_count,
                               g2m_cycle4_count): 1 = the chunks of the
                               round-robin are runs of consecutive sources of
                               equal ESTIMATED work (the pattern-aware
                               workload estimator, PAPER.md:1256-1262,
                               1309-1322), rr_chunk = sources per chunk on
                               average (c = alpha * y); 0 = rr_chunk sources
                               per chunk */
    const int64_t* data;    /* host array for PAIRS (2*count) / VERTICES / INDEX */
    uint64_t count;         /* entries in data (ignored for IMPLICIT) */
    uint64_t rr_chunk;      /* IMPLICIT only: 0 = whole list, else chunked
                               round-robin partition (scheduler.py:77-94) */
    uint32_t rr_parts;
    uint32_t rr_part;
} g2m_task_spec;

typedef struct g2m_kernel_meta {
    int32_t num_patterns;   /* counters, in forest.pattern_ids order */
    int32_t num_slots;      /* materialised-set slots per warp */
    int32_t granularity;    /* G2M_TASKS_EDGE / G2M_TASKS_VERTEX */
    int32_t max_level;      /* deepest plan level */
    int32_t needs_labels;
    int32_t list_mode;      /* kernel emits matches */
    int32_t smem_slot_cap;  /* >0: slots live in shared memory with this
                               many u32 entries each; 0: global scratch */
    int32_t warps_per_block;
    int32_t instrumented;   /* kernel accumulates algorithmic bytes */
    int32_t warp_words;     /* dynamic shared memory per warp (u32 words) */
    int32_t reserved[6];
} g2m_kernel_meta;

typedef struct g2m_run_config {
    int32_t blocks;         /* 0 = SM count x occupancy */
    int32_t reserved0;
    uint64_t chunk;         /* tasks per dynamic work grab, 0 = auto */
    uint64_t scratch_budget;/* bytes for per-warp global slots, 0 = auto */
    int32_t time_kernel;    /* record kernel time with CUDA events */
    int32_t reserved[5];
} g2m_run_config;

typedef struct g2m_run_stats {
    uint64_t tasks;             /* tasks in the list handed to the kernel */
    uint64_t tasks_active;      /* tasks passing the level-2 filter */
    uint64_t warps;             /* resident warps launched */
    uint64_t alg_bytes_lo;      /* SURVEY 8(d) algorithmic bytes (instrumented kernels) */
    uint64_t alg_bytes_hi;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t high_water[8];     /* max materialised size per slot */
    double kernel_ms;           /* CUDA-event time of the mining kernel(s) */
    double total_ms;            /* wall time of the whole call */
    double device_ms;           /* CUDA-event time of all device work of the call
                                   after task upload: counter reset, kernel(s),
                                   result copy-back */
    uint64_t launches;          /* kernels of libg2m launched by the call */
} g2m_run_stats;

/* Match callback for g2m_list: `n` tuples of `k` vertex ids (level order),
 * all for pattern index `pid`. Return nonzero to stop (sink -> True). */
typedef int (*g2m_match_cb)(void* user, int32_t pid, int32_t k, uint64_t n,
                            const uint32_t* tuples);

const char* g2m_last_error(void);
int32_t g2m_abi_version(void);
int g2m_device_count(int32_t* out);

int g2m_graph_create(int32_t device, const uint64_t* row_offsets, uint64_t num_vertices,
                     const uint32_t* neighbors, uint64_t num_slots,
                     const uint32_t* labels_or_null, int32_t oriented, g2m_graph** out);
int g2m_graph_from_edges(int32_t device, const int64_t* edges, uint64_t num_pairs,
                         uint64_t num_vertices, const uint32_t* labels_or_null,
                         g2m_graph** out);
/* R-MAT graph built on the device (SURVEY A.6 process: per edge and bit one
 * uniform draw picks the quadrant with probabilities a, b, c, 1-a-b-c; then
 * from_edges semantics). The uniforms come from a counter-based hash of
 * (seed, edge, bit), not numpy's stream: for graphs too large for a host
 * generator (scale >= 25, BASELINE config C5). */
int g2m_graph_rmat(int32_t device, int32_t scale, int32_t edgefactor, uint64_t seed, double a, double b,
                   double c, g2m_graph** out);
int g2m_graph_orient(const g2m_graph* g, g2m_graph** out);
int g2m_graph_replicate(const g2m_graph* g, int32_t device, g2m_graph** out);
int g2m_graph_info_get(const g2m_graph* g, g2m_graph_info* info);
int g2m_graph_download(const g2m_graph* g, uint64_t* row_offsets, uint32_t* neighbors,
                       uint32_t* labels_or_null);
int g2m_graph_destroy(g2m_graph* g);
/* The (degree, id) rank relabelling of g as a new graph (same orientation):
 * the id space of g2m_clique_count / g2m_cycle4_count. Relabelling it again
 * is the identity, so vertex partitions of it mean the same source sets for
 * the specialised kernels and for g2m_run (full-scale parity). Counts of
 * every pattern are invariant under the renaming (graph.py:224-238). */
int g2m_graph_rank_copy(const g2m_graph* g, g2m_graph** out);
/* Algorithmic work of the specialised kernels on g (bench roofline):
 * family 0 = bitmap k-clique on an oriented graph (rank space, with the hub
 * core the kernels use; 2 = the same without the core), 1 = 4-cycle wedges on
 * a symmetric graph. out[0]
 * operand bytes, out[1] probed ids / wedges, out[2] core bit tests (0) /
 * counter updates (1), out[3] sources with work (see g2m.cu). */
int g2m_kernel_work(const g2m_graph* g, int32_t family, uint64_t* out);
/* len(EdgeTaskList.implicit(g, reduced=True)) (graph.py:270-286): slots with
 * dst < src, counted on the device (cached with the reduced task offsets). */
int g2m_graph_reduced_tasks(const g2m_graph* g, uint64_t* out);
/* Hub-pattern vertex partition (replaces scheduler.partition_vertices_for_hub,
 * scheduler.py:125-163): the owned range [lo, hi) plus its 1-hop closure as
 * the induced subgraph, ids renamed in ascending global order, built on the
 * device. *num_local = its vertex count; the owned vertices are the local
 * ids [*first_owned, *first_owned + hi - lo). g2m_graph_local_ids copies the
 * local -> global map (num_local u32) of such a part. */
int g2m_graph_hub_part(const g2m_graph* g, uint64_t lo, uint64_t hi, g2m_graph** out,
                       uint64_t* num_local, uint64_t* first_owned);
int g2m_graph_local_ids(const g2m_graph* g, uint32_t* local_to_global);

/* Bounded-BFS frequent subgraph mining, device side of fsm.run_bounded_bfs
 * (replaces the level loop body of fsm.py:107-210; the canonical forms,
 * the support / filter callbacks and the result dictionaries stay on the
 * host). A g2m_fsm holds one BFS level: subgraphs of l edges (l <= 7) as
 * rows (edges u64 u << 32 | v ascending, 7 per row; vertices u32 ascending,
 * 8 per row; vertex count u8).
 *   create   level 1: every edge u < w of a labeled graph with ok[u], ok[w]
 *            (ok = label-frequency pruning, null = all)          fsm.py:135-146
 *   rows     copy the rows out (subgraph_filter hook)
 *   keep     keep the rows with keep[r] != 0
 *   quick    group rows by quick pattern (fsm.py:40-47): *nq groups;
 *   quick_records  12 u32 per group: k | l << 8, labels[8], position pairs
 *            (6 bits each, (min << 3 | max), ascending) as a u64
 *   domains  canonical id, position maps per group (host canonical forms,
 *            fsm.py:50-80) -> unique (canon << 36 | position << 32 | vertex)
 *            domain keys, their (canon << 4 | position) run lengths (the
 *            domain sizes, fsm.py:158-170) and the unique parent << 32 |
 *            child pattern pairs (fsm.py:171-175)
 *   results  copy run keys / lengths, domain keys, parent-child pairs
 *   extend   rows of patterns with kept[canon] grow by one adjacent edge,
 *            new edge sets deduplicated with their parent patterns
 *            (fsm.py:178-203) */
typedef struct g2m_fsm g2m_fsm;
int g2m_fsm_create(const g2m_graph* g, const uint8_t* ok_or_null, g2m_fsm** out, uint64_t* nrows);
int g2m_fsm_destroy(g2m_fsm* f);
int g2m_fsm_rows(const g2m_fsm* f, uint64_t* edges, uint32_t* verts, uint8_t* nverts);
int g2m_fsm_keep(g2m_fsm* f, const uint8_t* keep, uint64_t* nrows);
int g2m_fsm_quick(g2m_fsm* f, uint64_t* nq);
int g2m_fsm_quick_records(const g2m_fsm* f, uint32_t* out);
int g2m_fsm_domains(g2m_fsm* f, const uint32_t* canon, const uint32_t* nmaps, const uint32_t* map_off,
                    const uint8_t* maps, uint64_t maps_bytes, uint64_t* ndom, uint64_t* nruns, uint64_t* npc);
int g2m_fsm_results(const g2m_fsm* f, uint64_t* run_keys, uint64_t* run_len, uint64_t* dom_keys,
                    uint64_t* pc_pairs);
int g2m_fsm_extend(g2m_fsm* f, const uint8_t* kept, uint32_t ncanon, uint64_t* nrows);

int g2m_kernel_compile(const char* cuda_source, const char* kernel_name,
                       const char* const* header_sources, const char* const* header_names,
                       int32_t num_headers, const g2m_kernel_meta* meta, g2m_kernel** out);
int g2m_kernel_get_meta(const g2m_kernel* k, g2m_kernel_meta* meta);
int g2m_kernel_destroy(g2m_kernel* k);

int g2m_run(const g2m_kernel* k, const g2m_graph* g, const g2m_task_spec* tasks,
            const g2m_run_config* cfg, uint64_t* counts_lo_hi, g2m_run_stats* stats);
int g2m_list(const g2m_kernel* k, const g2m_graph* g, const g2m_task_spec* tasks,
             const g2m_run_config* cfg, g2m_match_cb cb, void* user,
             uint64_t* counts_lo_hi, g2m_run_stats* stats);

/* Bounded-frontier BFS runtime (run_dfs semantics, executor.py:339-408;
 * the level-synchronous extension of PAPER.md Alg. 2 / test_executor.py:
 * 203-235 restricted to the first three levels). `expand` and `consume` are
 * the two frontier kernels of one edge-parallel count forest (codegen
 * frontier="expand"/"consume"). Tasks are processed in blocks; each block's
 * level-3 candidates become work items of `chunk` candidates that the
 * consume kernel finishes depth-first, so hub edges are split across warps.
 * The item buffer is at most `frontier_bytes` (0: a quarter of free HBM);
 * a block that overflows it is halved and redone. stats->high_water[6] =
 * blocks, [7] = peak items. Counts equal g2m_run's. */
int g2m_run_bfs(const g2m_kernel* expand, const g2m_kernel* consume, const g2m_graph* g,
                const g2m_task_spec* tasks, const g2m_run_config* cfg, uint32_t chunk,
                uint64_t frontier_bytes, uint64_t* counts_lo_hi, g2m_run_stats* stats);

/* k-clique count (3 <= k <= 5) on an ORIENTED graph with the bitmap
 * local-graph kernels (one local DAG per source vertex; setops.py:101-173,
 * executor.py:415-523). `part` (optional, kind VERTEX, source IMPLICIT with
 * rr_chunk/rr_parts/rr_part) restricts the sources to a chunked round-robin
 * share. Sources whose out-degree exceeds the bitmap tiers (> 1024) are
 * counted by `fallback`, the generated plan kernel of the same k-clique
 * plan, over their edge tasks. counts_lo_hi receives (lo, hi). */
int g2m_clique_count(const g2m_graph* g, int32_t k, const g2m_task_spec* part,
                     const g2m_kernel* fallback, const g2m_run_config* cfg,
                     uint64_t* counts_lo_hi, g2m_run_stats* stats);

/* 4-cycle count of a SYMMETRIC (unoriented) graph: the count-mode result of
 * subgraph_listing(g, 4-cycle) (apps.py:291-297; plan PAPER.md §A.2),
 * computed by wedge aggregation on the (degree, id) rank relabelling
 * (cycle4_kernels.cuh). `part` (optional, IMPLICIT with rr_chunk/rr_parts/
 * rr_part) restricts the highest-ranked cycle vertex to a chunked round-robin
 * share. counts_lo_hi receives (lo, hi). */
int g2m_cycle4_count(const g2m_graph* g, const g2m_task_spec* part, const g2m_run_config* cfg,
                     uint64_t* counts_lo_hi, g2m_run_stats* stats);

/* Diamond count of a SYMMETRIC graph: the count-mode result of
 * subgraph_listing(g, diamond) with the counting rewrite (apps.py:133-150,
 * plan.py:177-198), Σ over edges of C(common neighbours, 2), from per-edge
 * triangle support accumulated by the bitmap triangle kernels on the
 * degree-oriented rank-space DAG. Single device (support is not additive
 * over task partitions). counts_lo_hi receives (lo, hi). */
int g2m_diamond_count(const g2m_graph* g, const g2m_run_config* cfg, uint64_t* counts_lo_hi,
                      g2m_run_stats* stats);

/* The two halves of g2m_diamond_count for a multi-GPU run, where per-edge
 * support is NOT additive over a source split but IS additive as an array:
 * g2m_diamond_support adds into `tsup` (device memory of g's device,
 * *num_slots u32, zeroed by the caller) the support contributions of the
 * triangles whose DAG source is in `part` (chunked round-robin share, as for
 * g2m_clique_count; null = all). With tsup == NULL it only builds the
 * oriented rank-space copy and reports *num_slots. After an all-reduce (sum)
 * of tsup over the ranks, g2m_support_choose2 gives Σ C(tsup[s], 2) over a
 * slot share [lo, hi), additive over the ranks' shares. Replaces the
 * edge-parallel plan kernel of run_on_devices for the diamond plan
 * (scheduler.py:207-239, plan.py:177-198). */
int g2m_diamond_support(const g2m_graph* g, const g2m_task_spec* part, uint32_t* tsup,
                        uint64_t* num_slots, g2m_run_stats* stats);
int g2m_support_choose2(const g2m_graph* g, const uint32_t* tsup, uint64_t lo, uint64_t hi,
                        uint64_t* counts_lo_hi, g2m_run_stats* stats);

/* Batched sorted-set kernels (setops.py:35-84). Lists are concatenated u32
 * arrays addressed by u64 offsets; op: 0 intersect, 1 intersect_count,
 * 2 difference, 3 difference_count. bound[i] < 0 means "no bound".
 * Outputs: out_count[i]; for materialising ops the elements at
 * out_values[out_offsets[i] ...] (out_offsets sized by |a|). */
int g2m_setop_batch(int32_t device, int32_t op, uint64_t num_cases,
                    const uint32_t* a_values, const uint64_t* a_offsets,
                    const uint32_t* b_values, const uint64_t* b_offsets,
                    const int64_t* bounds, uint64_t* out_count, uint32_t* out_values);

#ifdef __cplusplus
}
#endif

#endif /* G2M_H */
