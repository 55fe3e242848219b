// g2m.cu -- libg2m.so: C ABI (include/g2m.h) of the B200 pattern-mining engine.
//
// Owns device graphs (CSR replicas), the NVRTC compiler for generated plan
// kernels, task-list preparation, kernel launch and result collection.
// Fixed (non-generated) kernels live here too: orientation, reduced-task
// offsets, CSR construction, task conversion, batched set operations.
#include "g2m.h"
#include "g2m_device.cuh"
#include "clique_kernels.cuh"
#include "cycle4_kernels.cuh"
#include "fsm_kernels.cuh"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <cub/cub.cuh>
#include <thrust/execution_policy.h>
#include <thrust/scan.h>
#include <thrust/sort.h>
#include <thrust/unique.h>
#include <thrust/reduce.h>
#include <thrust/iterator/constant_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define G2M_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(G2M_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Driver API entry points, resolved through the runtime so the library
// loads on hosts without libcuda.so (the build container) and binds to the
// driver only when a GPU is actually used.
struct Drv {
    CUresult (*ModuleLoadData)(CUmodule*, const void*);
    CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*);
    CUresult (*ModuleUnload)(CUmodule);
    CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
    CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t);
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             unsigned, CUstream, void**, void**);
    CUresult (*GetErrorString)(CUresult, const char**);
    bool ok = false;
};
static Drv g_drv;
static std::mutex g_drv_mu;

static int drv_init() {
    std::lock_guard<std::mutex> lk(g_drv_mu);
    if (g_drv.ok) return 0;
    struct { const char* name; void** slot; } tab[] = {
        {"cuModuleLoadData", (void**)&g_drv.ModuleLoadData},
        {"cuModuleGetFunction", (void**)&g_drv.ModuleGetFunction},
        {"cuModuleUnload", (void**)&g_drv.ModuleUnload},
        {"cuFuncSetAttribute", (void**)&g_drv.FuncSetAttribute},
        {"cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&g_drv.OccupancyMaxActiveBlocksPerMultiprocessor},
        {"cuLaunchKernel", (void**)&g_drv.LaunchKernel},
        {"cuGetErrorString", (void**)&g_drv.GetErrorString},
    };
    for (auto& t : tab) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(t.name, t.slot, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !*t.slot)
            return -1;
    }
    g_drv.ok = true;
    return 0;
}

#define G2M_CU(call)                                                                    \
    do {                                                                                \
        if (drv_init()) return fail(G2M_ECUDA, "CUDA driver entry points unavailable"); \
        CUresult r_ = g_drv.call;                                                       \
        if (r_ != CUDA_SUCCESS) {                                                       \
            const char* s_ = nullptr;                                                   \
            g_drv.GetErrorString(r_, &s_);                                              \
            return fail(G2M_ECUDA, std::string(#call) + ": " + (s_ ? s_ : "?"));        \
        }                                                                               \
    } while (0)

#define G2M_TRY(call)               \
    do {                            \
        int rc_ = (call);           \
        if (rc_ != G2M_OK) return rc_; \
    } while (0)

using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------

// Allocations are stream-ordered (cudaMallocAsync / cudaFreeAsync) on the
// stream of the device the current API call works on (set by dev_state), from
// the device's memory pool with no release threshold: graphs created and freed
// call after call reuse pooled memory instead of cudaMalloc/cudaFree round trips.
static thread_local cudaStream_t t_alloc_stream = nullptr;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    int ensure(size_t n) {
        if (n <= bytes && p) return G2M_OK;
        release();
        if (n == 0) n = 16;
        s = t_alloc_stream;
        // +16 B: 1-D bulk copies (g2m_bulk_list) read the 16-byte-aligned
        // superset of a list, up to 12 bytes past the last element
        cudaError_t e = s ? cudaMallocAsync(&p, n + 16, s) : cudaMalloc(&p, n + 16);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(G2M_ECUDA, std::string("cudaMalloc(") + std::to_string(n) +
                                       "): " + cudaGetErrorString(e));
        }
        bytes = n;
        return G2M_OK;
    }
    void release() {
        if (p) {
            if (s) cudaFreeAsync(p, s);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return reinterpret_cast<T*>(p); }
    void swap_with(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(s, o.s);
    }
};

// Per-device reusable workspace (one run at a time per device).
struct DevState {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
    DevBuf counters;    // next, counts, stats
    DevBuf scratch;     // per-warp slots
    DevBuf tasks_a, tasks_b, task_match, matches, cub_tmp;
    DevBuf gr_slab;             // rows of the clique tiers that keep them in L2
    DevBuf core_bits;           // hub core of graph core_gid (see ensure_core)
    uint64_t core_gid = 0;
    uint32_t core_lo = 0, core_T = 0;
    int sms = 0;
    uint64_t launches = 0;   // kernels of ours launched on this device (g2m_run_stats.launches)
    DevBuf tmp1, tmp2, tmp3; // grow-only scratch of the preprocessing passes (rank relabelling)
    DevBuf frontier;         // BFS level-3 frontier items (grow-only)
    DevBuf c4slab;           // 4-cycle staging slabs, one per block
    DevBuf hubs;             // [0] = count, then the hub rows of a row pass (rows longer than kHubRow)
    DevBuf mids;             // a second row list (rank-space rows: the CTA-sorted ones)
    // side streams: independent kernel tiers run concurrently so one tier's
    // tail overlaps the next tier's work (fork/join through events)
    static constexpr int kSide = 8;
    cudaStream_t side[kSide] = {};
    cudaEvent_t evfork = nullptr, evjoin[kSide] = {};
};

static std::mutex g_dev_mu;
static std::map<int, std::unique_ptr<DevState>> g_devs;

// Grow-only scratch of the O(E) preprocessing passes (graph build, rank
// relabelling) can reach tens of GB at RMAT-27 (a radix sort of 4.3e9 keys):
// hand it back to the pool once the pass is done.
static void trim_scratch(DevState* st) {
    const size_t big = (size_t)1 << 30;
    if (st->cub_tmp.bytes > big) st->cub_tmp.release();
    if (st->tmp1.bytes > big) st->tmp1.release();
    if (st->tmp2.bytes > big) st->tmp2.release();
    if (st->tmp3.bytes > big) st->tmp3.release();
}

static int dev_state(int dev, DevState** out) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_devs.find(dev);
    if (it == g_devs.end()) {
        G2M_CUDA(cudaSetDevice(dev));
        G2M_CUDA(cudaFree(0));
        auto st = std::make_unique<DevState>();
        G2M_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
        G2M_CUDA(cudaEventCreate(&st->ev0));
        G2M_CUDA(cudaEventCreate(&st->ev1));
        G2M_CUDA(cudaEventCreate(&st->evs0));
        G2M_CUDA(cudaEventCreate(&st->evs1));
        G2M_CUDA(cudaEventCreateWithFlags(&st->evfork, cudaEventDisableTiming));
        for (int i = 0; i < DevState::kSide; ++i) {
            G2M_CUDA(cudaStreamCreateWithFlags(&st->side[i], cudaStreamNonBlocking));
            G2M_CUDA(cudaEventCreateWithFlags(&st->evjoin[i], cudaEventDisableTiming));
        }
        G2M_CUDA(cudaDeviceGetAttribute(&st->sms, cudaDevAttrMultiProcessorCount, dev));
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
        it = g_devs.emplace(dev, std::move(st)).first;
    }
    *out = it->second.get();
    t_alloc_stream = (*out)->stream;
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// graph
// ---------------------------------------------------------------------------

static std::atomic<uint64_t> g_graph_ids{1};

struct g2m_graph {
    const uint64_t gid = g_graph_ids.fetch_add(1);   // identity for per-device caches
    int dev = 0;
    uint64_t nv = 0, slots = 0, maxdeg = 0, sumsq = 0;
    int oriented = 0;
    DevBuf off, nbr, labels;
    std::mutex mu;
    DevBuf red_off;          // reduced (src > dst) task offsets, lazily built
    uint64_t red_total = 0;
    bool has_red = false;
    // the same graph relabelled by its (degree, id) order, lazily built
    DevBuf rk_off, rk_nbr;
    bool has_rank = false;
    // oriented graphs built by g2m_graph_orient: the undirected degree of every
    // vertex (the orientation's key), so the rank order needs no in-degree pass
    DevBuf symdeg;
    uint64_t symdeg_max = 0;
    // symmetric graphs uploaded by g2m_graph_create: the orientation's degree
    // table and keep bits (+ per-word counts), computed on a side stream as
    // the neighbour chunks land (under the PCIe copy)
    DevBuf pre_deg, pre_keep, pre_wcnt;
    bool pre_ready = false;
    uint64_t rk_deg1 = 0;    // ranks [0, rk_deg1) have degree <= 1
    // oriented graphs: rank-space rows holding a column <= their row, i.e. DAG
    // edges against the (degree, id) order (an input oriented some other way)
    uint64_t rk_down = 0;
    // symmetric graphs: degree orientation, lazily built (diamond support)
    std::unique_ptr<g2m_graph> oriented_copy;
    // workload estimator: exclusive prefix of per-source estimated work in
    // rank space (wpre[nv] = total), for the last (kernel family, k) asked
    DevBuf wpre;
    int wpre_key = -1;
    uint64_t wpre_total = 0, wpre_sources = 0;
    // hub partitions (g2m_graph_hub_part): local -> global ids, and the local
    // id of the first owned vertex (owned vertices are consecutive)
    DevBuf l2g;
    uint64_t part_first = 0, part_owned = 0;
    // oriented graphs: the hub core lives in the device state (one per device,
    // rebuilt when another graph uses it: no per-graph GB-sized allocations)
};

// out[0] = max degree, out[1] = Σ degree² (the BFS frontier bound, executor.choose_search)
__global__ void k_max_degree(const u64* off, u64 nv, u64* out) {
    u64 best = 0, sq = 0;
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x) {
        const u64 d = off[v + 1] - off[v];
        best = max(best, d);
        sq += d * d;
    }
    for (int o = 16; o; o >>= 1) {
        best = max(best, __shfl_xor_sync(G2M_FULL, best, o));
        sq += __shfl_xor_sync(G2M_FULL, sq, o);
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
    if ((threadIdx.x & 31) == 0 && sq) atomicAdd(out + 1, sq);
}

static int grid_for(DevState* st, uint64_t n, int threads) {
    uint64_t want = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)st->sms * 16;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (int)want;
}

static int finish_graph(g2m_graph* g, DevState* st) {
    DevBuf tmp;
    G2M_TRY(tmp.ensure(16));
    G2M_CUDA(cudaMemsetAsync(tmp.p, 0, 16, st->stream));
    if (g->nv) {
        k_max_degree<<<grid_for(st, g->nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nv, tmp.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    uint64_t h[2] = {0, 0};
    G2M_CUDA(cudaMemcpyAsync(h, tmp.p, 16, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    g->maxdeg = h[0];
    g->sumsq = h[1];
    return G2M_OK;
}

extern "C" const char* g2m_last_error(void) { return g_err.c_str(); }
extern "C" int32_t g2m_abi_version(void) { return G2M_ABI_VERSION; }

extern "C" int g2m_device_count(int32_t* out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = 0;
        return fail(G2M_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *out = n;
    return G2M_OK;
}

static int upload_symmetric_pipelined(g2m_graph* g, DevState* st, const uint64_t* off_h, const uint32_t* nbr_h);

extern "C" int g2m_graph_create(int32_t device, const uint64_t* row_offsets, uint64_t num_vertices,
                                const uint32_t* neighbors, uint64_t num_slots,
                                const uint32_t* labels, int32_t oriented, g2m_graph** out) {
    if (!out) return fail(G2M_EUSAGE, "null output handle");
    if (!row_offsets && num_vertices) return fail(G2M_EUSAGE, "null row_offsets");
    DevState* st;
    G2M_TRY(dev_state(device, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(device));
    auto g = std::make_unique<g2m_graph>();
    g->dev = device;
    g->nv = num_vertices;
    g->slots = num_slots;
    g->oriented = oriented ? 1 : 0;
    G2M_TRY(g->off.ensure((num_vertices + 1) * 8));
    G2M_TRY(g->nbr.ensure(std::max<uint64_t>(num_slots, 1) * 4));
    const bool pipe = !oriented && num_vertices && num_slots && row_offsets &&
                      !(getenv("G2M_UPLOAD_PIPE") && atoi(getenv("G2M_UPLOAD_PIPE")) == 0);
    if (pipe) {
        G2M_TRY(upload_symmetric_pipelined(g.get(), st, row_offsets, neighbors));
    } else {
        if (row_offsets)
            G2M_CUDA(cudaMemcpyAsync(g->off.p, row_offsets, (num_vertices + 1) * 8, cudaMemcpyHostToDevice,
                                     st->stream));
        else
            G2M_CUDA(cudaMemsetAsync(g->off.p, 0, 8, st->stream));
        if (num_slots)
            G2M_CUDA(cudaMemcpyAsync(g->nbr.p, neighbors, num_slots * 4, cudaMemcpyHostToDevice, st->stream));
    }
    if (labels) {
        G2M_TRY(g->labels.ensure(std::max<uint64_t>(num_vertices, 1) * 4));
        if (num_vertices)
            G2M_CUDA(cudaMemcpyAsync(g->labels.p, labels, num_vertices * 4, cudaMemcpyHostToDevice, st->stream));
    }
    G2M_TRY(finish_graph(g.get(), st));
    *out = g.release();
    return G2M_OK;
}

extern "C" int g2m_graph_info_get(const g2m_graph* g, g2m_graph_info* info) {
    if (!g || !info) return fail(G2M_EUSAGE, "null argument");
    info->num_vertices = g->nv;
    info->num_slots = g->slots;
    info->max_degree = g->maxdeg;
    info->oriented = g->oriented;
    info->labeled = g->labels.p ? 1 : 0;
    info->device = g->dev;
    info->reserved = 0;
    info->sum_degree_sq = g->sumsq;
    return G2M_OK;
}

extern "C" int g2m_graph_download(const g2m_graph* g, uint64_t* row_offsets, uint32_t* neighbors,
                                  uint32_t* labels) {
    if (!g) return fail(G2M_EUSAGE, "null graph");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    if (row_offsets)
        G2M_CUDA(cudaMemcpyAsync(row_offsets, g->off.p, (g->nv + 1) * 8, cudaMemcpyDeviceToHost, st->stream));
    if (neighbors && g->slots)
        G2M_CUDA(cudaMemcpyAsync(neighbors, g->nbr.p, g->slots * 4, cudaMemcpyDeviceToHost, st->stream));
    if (labels && g->labels.p && g->nv)
        G2M_CUDA(cudaMemcpyAsync(labels, g->labels.p, g->nv * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

extern "C" int g2m_graph_destroy(g2m_graph* g) {
    if (!g) return G2M_OK;
    cudaSetDevice(g->dev);
    delete g;
    return G2M_OK;
}

// ---- orientation (graph.py:204-221): keep u->w iff (deg u, u) < (deg w, w)

// Degrees as u32 (a 4-byte L2-resident lookup per slot instead of two
// random 8-byte offset loads).
__global__ void k_degrees(const u64* off, u64 nv, u32* deg) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x)
        deg[v] = (u32)(off[v + 1] - off[v]);
}

__device__ __forceinline__ bool orient_keep(u32 du, u32 u, u32 dw, u32 w) {
    return du < dw || (du == dw && u < w);
}

// Row passes run one warp per row. Rows longer than kHubRow (the hubs of a
// skewed graph: up to ~10^6 slots) would serialise the whole pass on one
// warp, so the warp pass appends them to a list and a second kernel gives
// each hub a 1024-thread block.
constexpr u32 kHubRow = 2048;
constexpr int kHubThreads = 1024;

__device__ __forceinline__ void push_hub(u32* hubs, u32 u) {
    hubs[1 + atomicAdd(hubs, 1u)] = u;
}

// List of the rows longer than min_row: at most slots / (min_row + 1) of them.
static int hub_list(DevState* st, uint64_t slots, u32 min_row, u32** out) {
    G2M_TRY(st->hubs.ensure((slots / (min_row + 1) + 2) * 4));
    G2M_CUDA(cudaMemsetAsync(st->hubs.p, 0, 4, st->stream));
    *out = st->hubs.as<u32>();
    return G2M_OK;
}

static int hub_grid(DevState* st, uint64_t slots) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(slots / kHubRow + 1, (uint64_t)st->sms * 2));
}

static int exclusive_scan_u64(DevState* st, const u64* in, u64* out, uint64_t n) {
    // out has n+1 entries; out[0] = 0, out[i+1] = sum in[0..i]
    G2M_CUDA(cudaMemsetAsync(out, 0, 8, st->stream));
    if (n == 0) return G2M_OK;
    size_t tmp = 0;
    G2M_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, (int64_t)n, st->stream));
    G2M_TRY(st->cub_tmp.ensure(tmp));
    G2M_CUDA(cub::DeviceScan::InclusiveSum(st->cub_tmp.p, tmp, in, out + 1, (int64_t)n, st->stream));
    return G2M_OK;
}

// ---- slot-parallel row passes (orientation, rank relabelling) -------------
// A CTA takes a tile of kTileSlots consecutive CSR slots and first recovers
// every slot's row in shared memory: the row of the tile's first slot by one
// binary search over the offsets, each row starting inside the tile marked
// at its first slot, then a block-wide running max. The passes then stream
// the slots coalesced, with no warp walking rows one by one (a 32-row group
// of hubs used to queue on one warp) and no hub lists.
constexpr int kTileThreads = 256;
constexpr u32 kTileSlots = 4096;

__device__ __forceinline__ u64 row_of_slot(const u64* off, u64 nv, u64 s) {
    u64 lo = 0, n = nv + 1;   // largest r with off[r] <= s (off[0] = 0)
    while (n > 0) {
        const u64 half = n >> 1;
        if (__ldg(off + lo + half) <= s) {
            lo += half + 1;
            n -= half + 1;
        } else {
            n = half;
        }
    }
    return lo - 1;
}

// map[p] = row of slot S0 + p, p < S1 - S0; scr: kTileThreads / 32 words.
// Each warp scans its own kTileSlots / 8 segment, carried in from the max
// over the earlier segments: four block barriers per tile (a running max in
// 16 block-wide passes took 34; keep pass -8 %, rank tiles 0.76 -> 0.71 ms).
__device__ __forceinline__ void tile_rowmap(const u64* off, u64 nv, u64 S0, u64 S1, u32* map, u32* scr,
                                            u64* s_r) {
    const u32 t = threadIdx.x, lane = g2m_lane(), w = t >> 5;
    if (t == 0) s_r[0] = row_of_slot(off, nv, S0);
    if (t == 32) s_r[1] = row_of_slot(off, nv, S1 - 1);
    for (u32 p = t; p < kTileSlots; p += kTileThreads) map[p] = 0;
    __syncthreads();
    const u64 r0 = s_r[0], r1 = s_r[1];
    if (t == 0) map[0] = (u32)r0;
    // rows r0 < r <= r1 start inside the tile (off[r0 + 1] > S0); an empty
    // row shares its start with the next row, the larger id wins
    for (u64 r = r0 + 1 + t; r <= r1; r += kTileThreads) atomicMax(map + (__ldg(off + r) - S0), (u32)r);
    __syncthreads();
    constexpr u32 SEG = kTileSlots / (kTileThreads / 32);
    u32 mx = 0;
    for (u32 j = w * SEG + lane; j < (w + 1) * SEG; j += 32) mx = max(mx, map[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(G2M_FULL, mx, o));
    if (lane == 0) scr[w] = mx;
    __syncthreads();
    u32 carry = 0;
    for (u32 q = 0; q < w; ++q) carry = max(carry, scr[q]);
    for (u32 j = w * SEG; j < (w + 1) * SEG; j += 32) {
        u32 incl = map[j + lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(G2M_FULL, incl, o);
            if (lane >= (u32)o) incl = max(incl, y);
        }
        incl = max(incl, carry);
        map[j + lane] = incl;
        carry = __shfl_sync(G2M_FULL, incl, 31);
    }
    __syncthreads();
}

// keep bit of every slot of a symmetric CSR (word s >> 5 = slots 32w ..),
// and the word's popcount
__global__ void __launch_bounds__(kTileThreads)
k_orient_keep_tiles(const u64* off, const u32* nbr, const u32* deg, u64 nv, u64 slots, u32* keep, u64* wcnt,
                    u64 tile0, u64 tile1) {
    __shared__ u32 map[kTileSlots];
    __shared__ u32 scr[kTileThreads / 32];
    __shared__ u64 s_r[2];
    const u32 lane = g2m_lane();
    for (u64 tile = tile0 + blockIdx.x; tile < tile1 && tile * kTileSlots < slots; tile += gridDim.x) {
        const u64 S0 = tile * kTileSlots, S1 = min(S0 + kTileSlots, slots);
        tile_rowmap(off, nv, S0, S1, map, scr, s_r);
        for (u32 p = threadIdx.x; p < kTileSlots; p += kTileThreads) {
            const u64 s = S0 + p;
            bool k = false;
            if (s < S1) {
                const u32 u = map[p], x = __ldg(nbr + s);
                k = orient_keep(__ldg(deg + u), u, __ldg(deg + x), x);
            }
            const u32 m = __ballot_sync(G2M_FULL, k);
            if (lane == 0 && s < S1) {
                keep[s >> 5] = m;
                wcnt[s >> 5] = __popc(m);
            }
        }
        __syncthreads();
    }
}

// noff[u] = kept slots before off[u], u in [0, nv]
__global__ void k_orient_offsets(const u64* off, u64 nv, const u32* keep, const u64* wpre, u64* noff) {
    for (u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x; u <= nv; u += (u64)gridDim.x * blockDim.x) {
        const u64 s = off[u], w = s >> 5;
        const u32 b = (u32)(s & 31u);
        noff[u] = wpre[w] + (b ? (u64)__popc(keep[w] & ((1u << b) - 1u)) : 0ull);
    }
}

// ordered compaction of the kept slots (a warp per keep word)
__global__ void k_orient_fill_slots(const u32* __restrict__ nbr, u64 slots, const u32* __restrict__ keep,
                                    const u64* __restrict__ wpre, u32* __restrict__ out) {
    const u32 lane = g2m_lane();
    const u64 words = (slots + 31) >> 5;
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    constexpr int B = 4;   // keep words per warp in flight
    for (u64 w0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; w0 < words; w0 += B * nw) {
        u32 m[B], x[B];
        u64 base[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const u64 w = w0 + q * nw;
            m[q] = w < words ? __ldg(keep + w) : 0u;
            base[q] = w < words ? __ldg(wpre + w) : 0ull;
            x[q] = ((m[q] >> lane) & 1u) ? __ldg(nbr + (w << 5) + lane) : 0u;
        }
#pragma unroll
        for (int q = 0; q < B; ++q)
            if ((m[q] >> lane) & 1u) out[base[q] + __popc(m[q] & g2m_lanemask_lt())] = x[q];
    }
}

// Upload of a symmetric CSR with the orientation's first pass under the copy:
// the offsets first, then the neighbours in up to 8 tile-aligned chunks on
// the main stream; a side stream computes the degree table once the offsets
// are in, then the keep bits of each chunk's tiles as it lands (rows may
// span chunks: a tile only reads its own slots, and the offsets are all in).
static int upload_symmetric_pipelined(g2m_graph* g, DevState* st, const uint64_t* off_h, const uint32_t* nbr_h) {
    const u64 nv = g->nv, slots = g->slots;
    const u64 words = (slots + 31) >> 5, tiles = (slots + kTileSlots - 1) / kTileSlots;
    G2M_TRY(g->pre_deg.ensure(std::max<u64>(nv, 1) * 4));
    G2M_TRY(g->pre_keep.ensure(std::max<u64>(words, 1) * 4));
    G2M_TRY(g->pre_wcnt.ensure(std::max<u64>(words, 1) * 8));
    cudaStream_t cs = st->side[0];
    const u64 per = std::max<u64>((tiles + 7) / 8, 1);
    const int nchunks = (int)((tiles + per - 1) / per);
    std::vector<cudaEvent_t> ev(nchunks + 2, nullptr);
    for (auto& e : ev) G2M_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    G2M_CUDA(cudaMemcpyAsync(g->off.p, off_h, (nv + 1) * 8, cudaMemcpyHostToDevice, st->stream));
    G2M_CUDA(cudaEventRecord(ev[0], st->stream));
    G2M_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
    ++st->launches;
    k_degrees<<<grid_for(st, nv, 256), 256, 0, cs>>>(g->off.as<u64>(), nv, g->pre_deg.as<u32>());
    for (int c = 0; c < nchunks; ++c) {
        const u64 t0 = (u64)c * per, t1 = std::min<u64>(tiles, t0 + per);
        const u64 a = t0 * kTileSlots, b = std::min<u64>(slots, t1 * kTileSlots);
        G2M_CUDA(cudaMemcpyAsync(g->nbr.as<u32>() + a, nbr_h + a, (b - a) * 4, cudaMemcpyHostToDevice, st->stream));
        G2M_CUDA(cudaEventRecord(ev[1 + c], st->stream));
        G2M_CUDA(cudaStreamWaitEvent(cs, ev[1 + c], 0));
        ++st->launches;
        k_orient_keep_tiles<<<(int)std::min<u64>(t1 - t0, (u64)st->sms * 8), kTileThreads, 0, cs>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), g->pre_deg.as<u32>(), nv, slots, g->pre_keep.as<u32>(),
            g->pre_wcnt.as<u64>(), t0, t1);
    }
    G2M_CUDA(cudaGetLastError());
    G2M_CUDA(cudaEventRecord(ev[nchunks + 1], cs));
    G2M_CUDA(cudaStreamWaitEvent(st->stream, ev[nchunks + 1], 0));
    for (auto& e : ev) cudaEventDestroy(e);   // released once the recorded work completes
    g->pre_ready = true;
    return G2M_OK;
}

static int orient_impl(const g2m_graph* g, DevState* st, g2m_graph** out) {
    auto o = std::make_unique<g2m_graph>();
    o->dev = g->dev;
    o->nv = g->nv;
    o->oriented = 1;
    const bool dbg = getenv("G2M_DEBUG") != nullptr;
    auto tr = Clock::now();
    auto phase = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(st->stream);
        fprintf(stderr, "[g2m] orient %s: %.2f ms\n", what, ms_since(tr));
        tr = Clock::now();
    };
    G2M_TRY(o->off.ensure((g->nv + 1) * 8));
    DevBuf& deg = o->symdeg;   // kept: the rank order of the oriented graph reuses it
    o->symdeg_max = g->maxdeg;
    G2M_TRY(deg.ensure(std::max<uint64_t>(g->nv, 1) * 4));
    // slot-parallel: keep bits per 32-slot word, their exclusive prefix, the new
    // offsets from the prefix at each row start, an ordered compaction
    // (RMAT-22: 1.1 ms, against 2.5 ms for warp-per-row count and fill passes)
    const u64 words = (g->slots + 31) >> 5;
    DevBuf keepbuf;
    G2M_TRY(st->tmp3.ensure((words + 1) * 8));
    u64* wpre = st->tmp3.as<u64>();
    const u32* keep;
    const u64* wcnt;
    if (g->pre_ready) {   // computed under the upload (upload_symmetric_pipelined)
        G2M_CUDA(cudaMemcpyAsync(deg.p, g->pre_deg.p, std::max<u64>(g->nv, 1) * 4, cudaMemcpyDeviceToDevice,
                                 st->stream));
        keep = g->pre_keep.as<u32>();
        wcnt = g->pre_wcnt.as<u64>();
    } else {
        G2M_TRY(keepbuf.ensure(std::max<u64>(words, 1) * 4));
        G2M_TRY(st->tmp1.ensure(std::max<u64>(words, 1) * 8));
        u64* wc = st->tmp1.as<u64>();
        ++st->launches;
        k_degrees<<<grid_for(st, g->nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nv, deg.as<u32>());
        if (g->slots) {
            ++st->launches;
            const u64 tiles = (g->slots + kTileSlots - 1) / kTileSlots;
            k_orient_keep_tiles<<<(int)std::min<u64>(tiles, (u64)st->sms * 8), kTileThreads, 0, st->stream>>>(
                g->off.as<u64>(), g->nbr.as<u32>(), deg.as<u32>(), g->nv, g->slots, keepbuf.as<u32>(), wc, 0,
                tiles);
        }
        keep = keepbuf.as<u32>();
        wcnt = wc;
    }
    G2M_CUDA(cudaGetLastError());
    phase("degrees+keep");
    G2M_TRY(exclusive_scan_u64(st, wcnt, wpre, words));
    ++st->launches;
    k_orient_offsets<<<grid_for(st, g->nv + 1, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nv, keep, wpre,
                                                                            o->off.as<u64>());
    G2M_CUDA(cudaGetLastError());
    G2M_CUDA(cudaMemcpyAsync(&o->slots, o->off.as<u64>() + g->nv, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    phase("scan+offsets");
    G2M_TRY(o->nbr.ensure(std::max<uint64_t>(o->slots, 1) * 4));
    if (words) {
        ++st->launches;
        k_orient_fill_slots<<<grid_for(st, words * 32, 256), 256, 0, st->stream>>>(
            g->nbr.as<u32>(), g->slots, keep, wpre, o->nbr.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    if (g->labels.p) {
        G2M_TRY(o->labels.ensure(std::max<uint64_t>(g->nv, 1) * 4));
        G2M_CUDA(cudaMemcpyAsync(o->labels.p, g->labels.p, g->nv * 4, cudaMemcpyDeviceToDevice, st->stream));
    }
    phase("fill");
    G2M_TRY(finish_graph(o.get(), st));
    phase("max degree");
    *out = o.release();
    return G2M_OK;
}

extern "C" int g2m_graph_orient(const g2m_graph* g, g2m_graph** out) {
    if (!g || !out) return fail(G2M_EUSAGE, "null argument");
    if (g->oriented) return fail(G2M_EUSAGE, "graph is already oriented");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    return orient_impl(g, st, out);
}

// ---- hub-pattern vertex partitioning (scheduler.py:125-163)
// Part [lo, hi) of the vertex range plus its 1-hop closure, as the induced
// subgraph with ids renamed in ascending global order: every search rooted
// at an owned vertex of a hub pattern (all others adjacent to the root)
// stays inside the part. Built on the device: mark, scan, gather rows.

__global__ void k_hub_mark(const u64* off, const u32* nbr, u64 lo, u64 hi, u32* flag) {
    const u64 s0 = off[lo], s1 = off[hi];
    for (u64 v = lo + blockIdx.x * (u64)blockDim.x + threadIdx.x; v < hi; v += (u64)gridDim.x * blockDim.x)
        flag[v] = 1u;
    for (u64 s = s0 + blockIdx.x * (u64)blockDim.x + threadIdx.x; s < s1; s += (u64)gridDim.x * blockDim.x)
        flag[nbr[s]] = 1u;
}

// g2l = exclusive scan of flag (u64); l2g[g2l[v]] = v for flagged v
__global__ void k_hub_l2g(const u32* flag, const u64* g2l, u64 nv, u32* l2g) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x)
        if (flag[v]) l2g[g2l[v]] = (u32)v;
}

// one warp per local vertex: kept neighbours (count pass) or their local ids
// in order (fill pass, ballot compaction)
template <bool FILL>
__global__ void k_hub_rows(const u64* off, const u32* nbr, const u32* flag, const u64* g2l, const u32* l2g,
                           u64 nsub, u64* cnt, const u64* soff, u32* snbr) {
    const u32 lane = g2m_lane();
    for (u64 x = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; x < nsub;
         x += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u32 v = l2g[x];
        const u64 b = off[v], e = off[v + 1];
        u64 pos = FILL ? soff[x] : 0;
        u64 c = 0;
        for (u64 s0 = b; s0 < e; s0 += 32) {
            const u64 s = s0 + lane;
            u32 w = 0;
            bool keep = false;
            if (s < e) {
                w = nbr[s];
                keep = flag[w] != 0u;
            }
            const u32 m = __ballot_sync(G2M_FULL, keep);
            if (FILL && keep) snbr[pos + __popc(m & g2m_lanemask_lt())] = (u32)g2l[w];
            pos += __popc(m);
            c += __popc(m);
        }
        if (!FILL && lane == 0) cnt[x] = c;
    }
}

__global__ void k_gather_u32(const u32* src, const u32* idx, u64 n, u32* dst) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

__global__ void k_u32_to_u64(const u32* a, u64 n, u64* b) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        b[i] = a[i];
}

extern "C" int g2m_graph_hub_part(const g2m_graph* g, uint64_t lo, uint64_t hi, g2m_graph** out,
                                  uint64_t* num_local, uint64_t* first_owned) {
    if (!g || !out || !num_local || !first_owned) return fail(G2M_EUSAGE, "null argument");
    if (lo > hi || hi > g->nv) return fail(G2M_EUSAGE, "owned range outside the vertex range");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    const u64 nv = g->nv;
    auto o = std::make_unique<g2m_graph>();
    o->dev = g->dev;
    o->oriented = g->oriented;
    DevBuf flag, flag64, g2l, cnt;
    G2M_TRY(flag.ensure(std::max<u64>(nv, 1) * 4));
    G2M_TRY(flag64.ensure(std::max<u64>(nv, 1) * 8));
    G2M_TRY(g2l.ensure((nv + 1) * 8));
    G2M_CUDA(cudaMemsetAsync(flag.p, 0, std::max<u64>(nv, 1) * 4, st->stream));
    if (hi > lo) {
        ++st->launches;
        k_hub_mark<<<grid_for(st, std::max<u64>(hi - lo, 1) * 8, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), lo, hi, flag.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    if (nv) {
        ++st->launches;
        k_u32_to_u64<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(flag.as<u32>(), nv, flag64.as<u64>());
    }
    G2M_TRY(exclusive_scan_u64(st, flag64.as<u64>(), g2l.as<u64>(), nv));
    u64 nsub = 0;
    G2M_CUDA(cudaMemcpyAsync(&nsub, g2l.as<u64>() + nv, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    o->nv = nsub;
    G2M_TRY(o->l2g.ensure(std::max<u64>(nsub, 1) * 4));
    G2M_TRY(o->off.ensure((nsub + 1) * 8));
    G2M_TRY(cnt.ensure(std::max<u64>(nsub, 1) * 8));
    if (nv) {
        ++st->launches;
        k_hub_l2g<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(flag.as<u32>(), g2l.as<u64>(), nv, o->l2g.as<u32>());
    }
    if (nsub) {
        ++st->launches;
        k_hub_rows<false><<<grid_for(st, nsub * 32, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), flag.as<u32>(), g2l.as<u64>(), o->l2g.as<u32>(), nsub,
            cnt.as<u64>(), nullptr, nullptr);
        G2M_CUDA(cudaGetLastError());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), o->off.as<u64>(), nsub));
    G2M_CUDA(cudaMemcpyAsync(&o->slots, o->off.as<u64>() + nsub, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    G2M_TRY(o->nbr.ensure(std::max<u64>(o->slots, 1) * 4));
    if (nsub) {
        ++st->launches;
        k_hub_rows<true><<<grid_for(st, nsub * 32, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), flag.as<u32>(), g2l.as<u64>(), o->l2g.as<u32>(), nsub, nullptr,
            o->off.as<u64>(), o->nbr.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    if (g->labels.p) {
        G2M_TRY(o->labels.ensure(std::max<u64>(nsub, 1) * 4));
        if (nsub) {
            ++st->launches;
            k_gather_u32<<<grid_for(st, nsub, 256), 256, 0, st->stream>>>(g->labels.as<u32>(), o->l2g.as<u32>(),
                                                                          nsub, o->labels.as<u32>());
        }
    }
    u64 first = 0;
    if (hi > lo) G2M_CUDA(cudaMemcpyAsync(&first, g2l.as<u64>() + lo, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    G2M_TRY(finish_graph(o.get(), st));
    o->part_first = first;
    o->part_owned = hi - lo;
    *num_local = nsub;
    *first_owned = first;
    *out = o.release();
    return G2M_OK;
}

extern "C" int g2m_graph_local_ids(const g2m_graph* g, uint32_t* local_to_global) {
    if (!g || !local_to_global) return fail(G2M_EUSAGE, "null argument");
    if (!g->l2g.p) return fail(G2M_EUSAGE, "graph is not a hub partition");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    if (g->nv)
        G2M_CUDA(cudaMemcpyAsync(local_to_global, g->l2g.p, g->nv * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

extern "C" int g2m_graph_replicate(const g2m_graph* g, int32_t device, g2m_graph** out) {
    if (!g || !out) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(device, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(device));
    auto o = std::make_unique<g2m_graph>();
    o->dev = device;
    o->nv = g->nv;
    o->slots = g->slots;
    o->maxdeg = g->maxdeg;
    o->sumsq = g->sumsq;
    o->oriented = g->oriented;
    G2M_TRY(o->off.ensure((g->nv + 1) * 8));
    G2M_TRY(o->nbr.ensure(std::max<uint64_t>(g->slots, 1) * 4));
    // peer copy over NVLink (staged through the host when peers are not accessible)
    G2M_CUDA(cudaMemcpyPeerAsync(o->off.p, device, g->off.p, g->dev, (g->nv + 1) * 8, st->stream));
    if (g->slots)
        G2M_CUDA(cudaMemcpyPeerAsync(o->nbr.p, device, g->nbr.p, g->dev, g->slots * 4, st->stream));
    if (g->labels.p) {
        G2M_TRY(o->labels.ensure(std::max<uint64_t>(g->nv, 1) * 4));
        G2M_CUDA(cudaMemcpyPeerAsync(o->labels.p, device, g->labels.p, g->dev, g->nv * 4, st->stream));
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    *out = o.release();
    return G2M_OK;
}

// ---- CSR construction on the device (graph.py:116-142)

// Both directions of every non-loop edge as keys u*n+v (warp-aggregated appends).
__device__ __forceinline__ void emit_pair_keys(u64 u, u64 v, bool ok, u64 n, u64* keys, u64* nkeys) {
    const u32 m = __ballot_sync(__activemask(), ok);
    if (!m) return;
    const u32 lane = g2m_lane();
    const u32 leader = __ffs(m) - 1;
    u64 base = 0;
    if (lane == leader) base = atomicAdd(nkeys, 2ull * __popc(m));
    base = __shfl_sync(__activemask(), base, leader);
    if (ok) {
        const u64 slot = base + 2ull * __popc(m & g2m_lanemask_lt());
        keys[slot] = u * n + v;
        keys[slot + 1] = v * n + u;
    }
}

__global__ void k_edge_keys(const i64* edges, u64 m, u64 n, u64* keys, u64* nkeys) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    const u64 m32 = (m + 31) & ~(u64)31;   // whole warps iterate together
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m32; i += stride) {
        u64 u = 0, v = 0;
        if (i < m) { u = (u64)edges[2 * i]; v = (u64)edges[2 * i + 1]; }
        emit_pair_keys(u, v, i < m && u != v, n, keys, nkeys);
    }
}

// R-MAT edges (Graph500 quadrant probabilities a, b, c, d = 1-a-b-c), one
// counter-based uniform per (edge, bit): the same process as SURVEY A.6 with
// a device RNG instead of numpy's stream (graphs of scale >= 25 do not fit a
// host-side generator).
__device__ __forceinline__ double rmat_uniform(u64 seed, u64 i, u32 bit) {
    u64 z = seed * 0x9E3779B97F4A7C15ull + i * 0xD1B54A32D192ED03ull + (u64)bit * 0xABC98388FB8FAC03ull;
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_rmat_keys(u64 m, int scale, u64 seed, double a, double b, double c, u64 n, u64* keys,
                            u64* nkeys) {
    const u64 stride = (u64)gridDim.x * blockDim.x;
    const u64 m32 = (m + 31) & ~(u64)31;
    const double ab = a + b, abc = a + b + c;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m32; i += stride) {
        u64 u = 0, v = 0;
        if (i < m)
            for (int bit = 0; bit < scale; ++bit) {
                const double r = rmat_uniform(seed, i, bit);
                u |= (u64)(r >= ab) << bit;
                v |= (u64)((r >= a && r < ab) || r >= abc) << bit;
            }
        emit_pair_keys(u, v, i < m && u != v, n, keys, nkeys);
    }
}

__global__ void k_keys_to_csr(const u64* keys, u64 nk, u64 n, u32* nbr, u64* cnt) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nk; i += (u64)gridDim.x * blockDim.x) {
        u64 k = keys[i];
        u64 s = k / n;
        nbr[i] = (u32)(k - s * n);
        atomicAdd(cnt + s, 1ull);
    }
}

// Sorted, deduplicated keys -> CSR graph (graph.py:116-142: symmetric, no
// self loops, no duplicates, rows ascending).
static int keys_to_graph(DevState* st, int device, uint64_t n, DevBuf& keys, DevBuf& keys2, DevBuf& nk,
                         uint64_t nkeys, const uint32_t* labels, g2m_graph** out) {
    int nbits = 0;
    while (nbits < 33 && (n >> nbits)) ++nbits;
    int end_bit = std::max(1, std::min(64, 2 * nbits));
    uint64_t nuniq = 0;
    if (nkeys) {
        size_t tmp = 0;
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.as<u64>(), keys2.as<u64>(), (int64_t)nkeys, 0,
                                                end_bit, st->stream));
        G2M_TRY(st->cub_tmp.ensure(tmp));
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(st->cub_tmp.p, tmp, keys.as<u64>(), keys2.as<u64>(), (int64_t)nkeys,
                                                0, end_bit, st->stream));
        size_t tmp2 = 0;
        G2M_CUDA(cub::DeviceSelect::Unique(nullptr, tmp2, keys2.as<u64>(), keys.as<u64>(), nk.as<u64>() + 1,
                                           (int64_t)nkeys, st->stream));
        G2M_TRY(st->cub_tmp.ensure(tmp2));
        G2M_CUDA(cub::DeviceSelect::Unique(st->cub_tmp.p, tmp2, keys2.as<u64>(), keys.as<u64>(), nk.as<u64>() + 1,
                                           (int64_t)nkeys, st->stream));
        G2M_CUDA(cudaMemcpyAsync(&nuniq, nk.as<u64>() + 1, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
    }
    keys2.release();
    if (nuniq > 0xffffffffull * 4) return fail(G2M_EUSAGE, "graph too large");
    auto g = std::make_unique<g2m_graph>();
    g->dev = device;
    g->nv = n;
    g->slots = nuniq;
    DevBuf cnt;
    G2M_TRY(cnt.ensure(std::max<uint64_t>(n, 1) * 8));
    G2M_CUDA(cudaMemsetAsync(cnt.p, 0, std::max<uint64_t>(n, 1) * 8, st->stream));
    G2M_TRY(g->off.ensure((n + 1) * 8));
    G2M_TRY(g->nbr.ensure(std::max<uint64_t>(nuniq, 1) * 4));
    if (nuniq) {
        k_keys_to_csr<<<grid_for(st, nuniq, 256), 256, 0, st->stream>>>(keys.as<u64>(), nuniq, n, g->nbr.as<u32>(),
                                                                          cnt.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), g->off.as<u64>(), n));
    if (labels) {
        G2M_TRY(g->labels.ensure(std::max<uint64_t>(n, 1) * 4));
        if (n) G2M_CUDA(cudaMemcpyAsync(g->labels.p, labels, n * 4, cudaMemcpyHostToDevice, st->stream));
    }
    G2M_TRY(finish_graph(g.get(), st));
    trim_scratch(st);
    *out = g.release();
    return G2M_OK;
}

extern "C" int g2m_graph_from_edges(int32_t device, const int64_t* edges, uint64_t m,
                                    uint64_t num_vertices, const uint32_t* labels, g2m_graph** out) {
    if (!out) return fail(G2M_EUSAGE, "null output handle");
    DevState* st;
    G2M_TRY(dev_state(device, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(device));
    const uint64_t n = num_vertices;
    DevBuf din, keys, keys2, nk;
    G2M_TRY(din.ensure(std::max<uint64_t>(m, 1) * 16));
    G2M_TRY(keys.ensure(std::max<uint64_t>(2 * m, 1) * 8));
    G2M_TRY(keys2.ensure(std::max<uint64_t>(2 * m, 1) * 8));
    G2M_TRY(nk.ensure(16));
    G2M_CUDA(cudaMemsetAsync(nk.p, 0, 16, st->stream));
    if (m) {
        G2M_CUDA(cudaMemcpyAsync(din.p, edges, m * 16, cudaMemcpyHostToDevice, st->stream));
        ++st->launches;
        k_edge_keys<<<grid_for(st, m, 256), 256, 0, st->stream>>>(din.as<i64>(), m, n, keys.as<u64>(), nk.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    uint64_t nkeys = 0;
    G2M_CUDA(cudaMemcpyAsync(&nkeys, nk.p, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    din.release();
    return keys_to_graph(st, device, n, keys, keys2, nk, nkeys, labels, out);
}

extern "C" int g2m_graph_rmat(int32_t device, int32_t scale, int32_t edgefactor, uint64_t seed, double a,
                              double b, double c, g2m_graph** out) {
    if (!out) return fail(G2M_EUSAGE, "null output handle");
    if (scale < 1 || scale > 31 || edgefactor < 1) return fail(G2M_EUSAGE, "bad R-MAT scale / edge factor");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1) return fail(G2M_EUSAGE, "bad R-MAT probabilities");
    DevState* st;
    G2M_TRY(dev_state(device, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(device));
    const uint64_t n = (uint64_t)1 << scale;
    const uint64_t m = (uint64_t)edgefactor << scale;
    DevBuf keys, keys2, nk;
    G2M_TRY(keys.ensure(2 * m * 8));
    G2M_TRY(keys2.ensure(2 * m * 8));
    G2M_TRY(nk.ensure(16));
    G2M_CUDA(cudaMemsetAsync(nk.p, 0, 16, st->stream));
    ++st->launches;
    k_rmat_keys<<<st->sms * 16, 256, 0, st->stream>>>(m, scale, seed, a, b, c, n, keys.as<u64>(), nk.as<u64>());
    G2M_CUDA(cudaGetLastError());
    uint64_t nkeys = 0;
    G2M_CUDA(cudaMemcpyAsync(&nkeys, nk.p, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return keys_to_graph(st, device, n, keys, keys2, nk, nkeys, nullptr, out);
}

// ---- reduced edge-task offsets: row v holds |N(v) ∩ [0, v)| tasks (graph.py:275-286)

__global__ void k_red_count(const u64* off, const u32* nbr, u64 nv, u64* cnt) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x) {
        u64 b = off[v], e = off[v + 1];
        cnt[v] = g2m_lb(nbr + b, (u32)(e - b), (u32)v);
    }
}

static int ensure_reduced(const g2m_graph* cg, DevState* st) {
    g2m_graph* g = const_cast<g2m_graph*>(cg);
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->has_red) return G2M_OK;
    G2M_TRY(g->red_off.ensure((g->nv + 1) * 8));
    DevBuf cnt;
    G2M_TRY(cnt.ensure(std::max<uint64_t>(g->nv, 1) * 8));
    if (g->nv) {
        ++st->launches;
        k_red_count<<<grid_for(st, g->nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nbr.as<u32>(), g->nv, cnt.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), g->red_off.as<u64>(), g->nv));
    G2M_CUDA(cudaMemcpyAsync(&g->red_total, g->red_off.as<u64>() + g->nv, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    g->has_red = true;
    return G2M_OK;
}

// ---- rank-space DAG (derived, oriented graphs only)
//
// The oriented graph keeps u->v iff (deg_u, u) < (deg_v, v) (graph.py:204-221).
// Relabelling every vertex by its position in that order (its *rank*) turns
// the DAG into "edges point to larger ids", with the high-degree vertices at
// the top of the id range. Counts are invariant under the renaming
// (SURVEY 7.3-3); what changes is locality: N+(u) of a source in the
// bitmap-LGS tiers spans a narrow id window, so a direct-address bitmap of
// that window in shared memory replaces hashing (clique_kernels.cuh).
// deg_v = d+(v) + d-(v) on the oriented graph (each undirected edge is kept
// once), so the order is recomputed exactly without the undirected graph.
// Symmetric graphs get the same relabelling with deg_v = row length
// (cycle4_kernels.cuh).

__global__ void k_rank_indeg(const u32* nbr, u64 slots, u32* indeg) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < slots; i += (u64)gridDim.x * blockDim.x)
        atomicAdd(indeg + __ldg(nbr + i), 1u);
}

__global__ void k_rank_keys(const u64* off, const u32* indeg, u64 nv, u64* keys) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x)
        keys[v] = ((off[v + 1] - off[v] + (u64)indeg[v]) << 32) | v;
}

__global__ void k_rank_keys_sym(const u32* deg, u64 nv, u64* keys) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x)
        keys[v] = ((u64)deg[v] << 32) | v;
}

__global__ void k_count_deg_le1(const u64* keys, u64 nv, u64* out) {
    u64 c = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nv; i += (u64)gridDim.x * blockDim.x)
        c += (keys[i] >> 32) <= 1 ? 1 : 0;
    c = g2m_wsum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_rank_scatter(const u64* off, const u64* sorted, u64 nv, u32* rank, u64* rdeg) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nv; i += (u64)gridDim.x * blockDim.x) {
        const u32 v = (u32)sorted[i];
        rank[v] = (u32)i;
        rdeg[i] = off[v + 1] - off[v];
    }
}

// (new row << rb | new column) per slot (ids < 2^rb); one radix sort puts
// every row's columns in ascending order.
__global__ void k_rank_keys64(const u64* off, const u32* nbr, u64 nv, const u32* rank, int rb, u64* keys,
                              u32* hubs) {
    const u32 lane = g2m_lane();
    for (u64 v = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; v < nv;
         v += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 b = off[v], e = off[v + 1];
        if (b == e) continue;
        if (e - b > kHubRow) {
            if (lane == 0) push_hub(hubs, (u32)v);
            continue;
        }
        const u64 hi = (u64)rank[v] << rb;
        for (u64 i = b + lane; i < e; i += 32) keys[i] = hi | __ldg(rank + __ldg(nbr + i));
    }
}

__global__ void __launch_bounds__(kHubThreads)
k_rank_keys64_hubs(const u64* off, const u32* nbr, const u32* rank, int rb, u64* keys, const u32* hubs) {
    const u32 nh = hubs[0];
    for (u32 h = blockIdx.x; h < nh; h += gridDim.x) {
        const u32 v = hubs[1 + h];
        const u64 b = off[v], e = off[v + 1];
        const u64 hi = (u64)rank[v] << rb;
        for (u64 i = b + threadIdx.x; i < e; i += kHubThreads) keys[i] = hi | __ldg(rank + __ldg(nbr + i));
    }
}

// ---- rank-space rows (replaces the global key sort) -------------------------
// Row r = rank[v] of the rank-space CSR holds rank[w] for w in N(v), sorted.
// Short rows inside a slot tile are placed by counting (k_rank_fill_tiles),
// rows up to 512 slots sorted in a warp's registers (k_rank_fill_warp*),
// longer ones by one 256-thread CTA per row in shared memory (<=
// kRowSortBlock); graphs with longer rows take the global key sort. RMAT-22
// (32 M slots): 4.1 ms with a warp walking 32 rows of up to 1024 slots, 2.2 ms
// with rows > 128 on CTAs, 1.9 ms now (tiles 0.75, warps 0.44 + 0.24, CTAs).
constexpr u32 kRowSortBlock = 8192;

// Bitonic sort of s[0, P) (P a power of two) by `nt` threads with index t;
// sync() separates the stages.
template <typename Sync>
__device__ __forceinline__ void bitonic_smem(u32* s, u32 P, u32 t, u32 nt, Sync&& sync) {
    for (u32 k = 2; k <= P; k <<= 1)
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            for (u32 i = t; i < P / 2; i += nt) {
                const u32 lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));   // i-th pair (lo, lo ^ j)
                const u32 hi = lo | j;
                const u32 a = s[lo], b = s[hi];
                const bool asc = (lo & k) == 0;
                if ((a > b) == asc) { s[lo] = b; s[hi] = a; }
            }
            sync();
        }
}

// Rank-space rows by slot tiles: each CTA recovers its tile's rows (tile_rowmap),
// gathers rank[nbr[s]] into shared memory, and places every slot of a row that
// lies wholly inside the tile and has at most kTileRowMax slots at its rank
// within the row (a count over the row in shared memory, no sort). The other
// rows go on a list, pushed by the tile holding their first slot: rows of at
// most kWarpRowMax slots to a warp each (k_rank_fill_warp), longer ones to a
// CTA each (k_rank_fill_hubs).
constexpr u32 kTileRowMax = 32;
constexpr u32 kWarpRowMax = 256;
__global__ void __launch_bounds__(kTileThreads)
k_rank_fill_tiles(const u64* __restrict__ off, const u32* __restrict__ nbr, u64 nv, u64 slots,
                  const u32* __restrict__ rank, const u64* __restrict__ rk_off, u32* __restrict__ rk_nbr) {
    __shared__ u32 map[kTileSlots];
    __shared__ u32 val[kTileSlots];
    __shared__ u32 scr[kTileThreads / 32];
    __shared__ u64 s_r[2];
    constexpr u32 B = 4;   // slots per thread in flight
    for (u64 tile = blockIdx.x; tile * kTileSlots < slots; tile += gridDim.x) {
        const u64 S0 = tile * kTileSlots, S1 = min(S0 + kTileSlots, slots);
        const u32 n = (u32)(S1 - S0);
        tile_rowmap(off, nv, S0, S1, map, scr, s_r);
        for (u32 p0 = threadIdx.x; p0 < n; p0 += B * kTileThreads) {
            u32 x[B];
#pragma unroll
            for (u32 q = 0; q < B; ++q) {
                const u32 p = p0 + q * kTileThreads;
                x[q] = p < n ? __ldg(nbr + S0 + p) : 0u;
            }
#pragma unroll
            for (u32 q = 0; q < B; ++q) {
                const u32 p = p0 + q * kTileThreads;
                if (p < n) val[p] = __ldg(rank + x[q]);
            }
        }
        __syncthreads();
        for (u32 p0 = threadIdx.x; p0 < n; p0 += B * kTileThreads) {
            u32 u[B];
            u64 b[B], e[B];
#pragma unroll
            for (u32 q = 0; q < B; ++q) {
                const u32 p = p0 + q * kTileThreads;
                u[q] = p < n ? map[p] : 0u;
                b[q] = __ldg(off + u[q]);
                e[q] = __ldg(off + u[q] + 1);
            }
            u64 dst[B];
#pragma unroll
            for (u32 q = 0; q < B; ++q) {
                const u32 p = p0 + q * kTileThreads;
                const bool in = p < n && b[q] >= S0 && e[q] <= S1 && e[q] - b[q] <= kTileRowMax;
                dst[q] = in ? __ldg(rk_off + __ldg(rank + u[q])) : ~0ull;
            }
#pragma unroll
            for (u32 q = 0; q < B; ++q) {
                const u32 p = p0 + q * kTileThreads;
                if (p >= n) continue;
                if (dst[q] != ~0ull) {
                    const u32 v = val[p], a = (u32)(b[q] - S0), L = (u32)(e[q] - b[q]);
                    u32 c = 0;
                    for (u32 t = 0; t < L; ++t) c += val[a + t] < v ? 1u : 0u;
                    rk_nbr[dst[q] + c] = v;
                }
            }
        }
        __syncthreads();
    }
}

// The rows the tiles leave (longer than kTileRowMax, or across a tile edge):
// rows of at most kWarpRowMax slots on one list, the rest on another
// (warp-aggregated appends).
__global__ void k_rank_classify(const u64* __restrict__ off, u64 nv, u32* __restrict__ wrows,
                                u32* __restrict__ crows) {
    const u32 lane = g2m_lane();
    for (u64 v0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; v0 < nv;
         v0 += (u64)gridDim.x * blockDim.x) {
        const u64 v = v0 + lane;
        u64 d = 0;
        bool tile = true;
        if (v < nv) {
            const u64 b = off[v], e = off[v + 1];
            d = e - b;
            tile = d == 0 || (d <= kTileRowMax && b / kTileSlots == (e - 1) / kTileSlots);
        }
        const bool w = !tile && d <= kWarpRowMax, c = !tile && d > kWarpRowMax;
        const u32 mw = __ballot_sync(G2M_FULL, w), mc = __ballot_sync(G2M_FULL, c);
        u32 bw = 0, bc = 0;
        if (lane == 0) {
            if (mw) bw = atomicAdd(wrows, (u32)__popc(mw));
            if (mc) bc = atomicAdd(crows, (u32)__popc(mc));
        }
        bw = __shfl_sync(G2M_FULL, bw, 0);
        bc = __shfl_sync(G2M_FULL, bc, 0);
        if (w) wrows[1 + bw + __popc(mw & g2m_lanemask_lt())] = (u32)v;
        if (c) crows[1 + bc + __popc(mc & g2m_lanemask_lt())] = (u32)v;
    }
}

// Bitonic sort of 32 * E values held E per lane (element lane * E + q in v[q]):
// partners below E are in the same lane, the others one shuffle away.
template <int E>
__device__ __forceinline__ void warp_bitonic(u32 (&v)[E], u32 lane) {
    constexpr u32 P = 32u * E;
#pragma unroll
    for (u32 k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            if (j >= (u32)E) {
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    const u32 i = lane * E + q;
                    const u32 y = __shfl_xor_sync(G2M_FULL, v[q], j / E);
                    const bool asc = (i & k) == 0, lower = (i & j) == 0;
                    v[q] = (lower == asc) ? min(v[q], y) : max(v[q], y);
                }
            } else {
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    const int q2 = q ^ (int)j;
                    if (q2 > q) {
                        const bool asc = ((lane * E + q) & k) == 0;
                        const u32 a = v[q], c = v[q2];
                        const bool sw = asc ? (a > c) : (a < c);
                        v[q] = sw ? c : a;
                        v[q2] = sw ? a : c;
                    }
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ void warp_row_sort(const u32* __restrict__ src, u32 d, const u32* __restrict__ rank,
                                              u32* __restrict__ out, u32 lane) {
    u32 x[E], v[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
        const u32 i = lane * E + q;
        x[q] = i < d ? __ldg(src + i) : 0u;
    }
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = lane * E + q < d ? __ldg(rank + x[q]) : 0xffffffffu;
    warp_bitonic<E>(v, lane);
#pragma unroll
    for (int q = 0; q < E; ++q)
        if (lane * E + q < d) out[lane * E + q] = v[q];
}

// Listed rows of at most kWarpRowMax slots, a warp each, sorted in registers.
__global__ void __launch_bounds__(256)
k_rank_fill_warp(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ rank,
                 const u64* __restrict__ rk_off, u32* __restrict__ rk_nbr, const u32* __restrict__ rows) {
    const u32 lane = g2m_lane();
    const u32 nr = rows[0];
    for (u32 h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < nr; h += (gridDim.x * blockDim.x) >> 5) {
        const u32 v = rows[1 + h];
        const u64 b = __ldg(off + v);
        const u32 d = (u32)(__ldg(off + v + 1) - b);
        u32* out = rk_nbr + __ldg(rk_off + __ldg(rank + v));
        const u32* src = nbr + b;
        if (d <= 32) warp_row_sort<1>(src, d, rank, out, lane);
        else if (d <= 64) warp_row_sort<2>(src, d, rank, out, lane);
        else if (d <= 128) warp_row_sort<4>(src, d, rank, out, lane);
        else warp_row_sort<8>(src, d, rank, out, lane);   // d <= kWarpRowMax
    }
}

// Listed rows of 32 * E / 2 < d <= 32 * E, a warp each (the register file
// holds the row: E = 16).
template <int E>
__global__ void __launch_bounds__(128)
k_rank_fill_warp_big(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ rank,
                     const u64* __restrict__ rk_off, u32* __restrict__ rk_nbr, const u32* __restrict__ rows) {
    const u32 lane = g2m_lane();
    const u32 nr = rows[0];
    for (u32 h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < nr; h += (gridDim.x * blockDim.x) >> 5) {
        const u32 v = rows[1 + h];
        const u64 b = __ldg(off + v);
        const u32 d = (u32)(__ldg(off + v + 1) - b);
        if (d <= 16u * E || d > 32u * E) continue;
        warp_row_sort<E>(nbr + b, d, rank, rk_nbr + __ldg(rk_off + __ldg(rank + v)), lane);
    }
}

// Listed rows longer than min_d, one 256-thread CTA per row (several CTAs per SM).
constexpr int kRankFillThreads = 256;
__global__ void __launch_bounds__(kRankFillThreads)
k_rank_fill_hubs(const u64* off, const u32* nbr, const u32* rank, const u64* rk_off, u32* rk_nbr, const u32* hubs,
                 u32 min_d) {
    constexpr u32 kHubThreads = kRankFillThreads;
    __shared__ u32 sb[kRowSortBlock];
    const u32 nh = hubs[0];
    for (u32 h = blockIdx.x; h < nh; h += gridDim.x) {
        const u32 v = hubs[1 + h];
        const u64 b = off[v];
        const u32 d = (u32)(off[v + 1] - b);   // <= kRowSortBlock (host check)
        if (d <= min_d) continue;
        u32* out = rk_nbr + rk_off[rank[v]];
        const u32 P = 1u << (32 - __clz(d - 1));
        for (u32 i = threadIdx.x; i < P; i += kHubThreads) sb[i] = i < d ? __ldg(rank + __ldg(nbr + b + i)) : 0xffffffffu;
        __syncthreads();
        bitonic_smem(sb, P, threadIdx.x, kHubThreads, [] { __syncthreads(); });
        for (u32 i = threadIdx.x; i < d; i += kHubThreads) out[i] = sb[i];
        __syncthreads();
    }
}

// Rows are ascending, so a row points against the order iff its first column
// is not above the row.
__global__ void k_rank_down_rows(const u64* off, const u32* nbr, u64 nv, u64* out) {
    u64 c = 0;
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < nv; r += (u64)gridDim.x * blockDim.x) {
        const u64 b = off[r];
        if (off[r + 1] > b && (u64)__ldg(nbr + b) <= r) ++c;
    }
    c = g2m_wsum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_low_bits(const u64* keys, u64 n, int rb, u32* out) {
    const u64 mask = ((u64)1 << rb) - 1;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = (u32)(keys[i] & mask);
}

static int ensure_rank(const g2m_graph* cg, DevState* st) {
    g2m_graph* g = const_cast<g2m_graph*>(cg);
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->has_rank) return G2M_OK;
    const u64 nv = g->nv, slots = g->slots;
    const bool dbg = getenv("G2M_DEBUG") != nullptr;
    auto tr = Clock::now();
    auto phase = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(st->stream);
        fprintf(stderr, "[g2m] rank build %s: %.2f ms\n", what, ms_since(tr));
        tr = Clock::now();
    };
    G2M_TRY(g->rk_off.ensure((nv + 1) * 8));
    G2M_TRY(g->rk_nbr.ensure(std::max<u64>(slots, 1) * 4));
    DevBuf indeg, keys, sorted, rank, rdeg;
    G2M_TRY(indeg.ensure(std::max<u64>(nv, 1) * 4));
    G2M_TRY(keys.ensure(std::max<u64>(nv, 1) * 8));
    G2M_TRY(sorted.ensure(std::max<u64>(nv, 1) * 8));
    G2M_TRY(rank.ensure(std::max<u64>(nv, 1) * 4));
    G2M_TRY(rdeg.ensure(std::max<u64>(nv, 1) * 8));
    // an oriented graph from g2m_graph_orient carries the undirected degrees its
    // orientation used (no in-degree atomics); others: deg = d+ + d- (symmetric
    // graphs: the row length)
    const bool sym = g->oriented && g->symdeg.p && !getenv("G2M_RANK_INDEG");
    if (!sym) G2M_CUDA(cudaMemsetAsync(indeg.p, 0, std::max<u64>(nv, 1) * 4, st->stream));
    if (nv) {
        if (slots && g->oriented && !sym) {
            ++st->launches;
            k_rank_indeg<<<grid_for(st, slots, 256), 256, 0, st->stream>>>(g->nbr.as<u32>(), slots, indeg.as<u32>());
        }
        ++st->launches;
        if (sym)
            k_rank_keys_sym<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->symdeg.as<u32>(), nv, keys.as<u64>());
        else
            k_rank_keys<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), indeg.as<u32>(), nv,
                                                                        keys.as<u64>());
        G2M_CUDA(cudaGetLastError());
        const u64 dmax = sym ? g->symdeg_max : 2 * std::max<u64>(slots, 1);
        int hi = 32;
        while (hi < 64 && ((u64)1 << (hi - 32)) <= dmax) ++hi;   // degree < 2^(hi-32)
        size_t tb = 0;
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<u64>(), sorted.as<u64>(), (int64_t)nv, 0, hi,
                                                st->stream));
        G2M_TRY(st->cub_tmp.ensure(tb));
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(st->cub_tmp.p, tb, keys.as<u64>(), sorted.as<u64>(), (int64_t)nv, 0,
                                                hi, st->stream));
        ++st->launches;
        k_rank_scatter<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), sorted.as<u64>(), nv,
                                                                       rank.as<u32>(), rdeg.as<u64>());
        G2M_CUDA(cudaGetLastError());
        u64* d1 = (u64*)indeg.p;    // indeg is no longer needed
        G2M_CUDA(cudaMemsetAsync(d1, 0, 8, st->stream));
        ++st->launches;
        k_count_deg_le1<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(sorted.as<u64>(), nv, d1);
        G2M_CUDA(cudaMemcpyAsync(&g->rk_deg1, d1, 8, cudaMemcpyDeviceToHost, st->stream));
    }
    phase("keys+sort+scatter");
    G2M_TRY(exclusive_scan_u64(st, rdeg.as<u64>(), g->rk_off.as<u64>(), nv));
    // rows of at most kRowSortBlock (oriented graphs; symmetric graphs without
    // hubs) are written in place and sorted per row; otherwise one global key
    // sort (a segmented sort leaves a 10^6-slot hub row to one CTA)
    // (a slot-parallel gather into the rank-space rows + cub::DeviceSegmentedSort
    // measured 0.5 + 8.3 ms on RMAT-22 against 2.2 ms for the per-row fill below)
    if (nv && slots && g->maxdeg <= kRowSortBlock && !getenv("G2M_RANK_RADIX")) {
        const u64 tiles = (slots + kTileSlots - 1) / kTileSlots;
        // lists: [0] = count, then rows; at most one row per tile crosses its edge
        G2M_TRY(st->hubs.ensure((slots / (kTileRowMax + 1) + tiles + 2) * 4));
        G2M_TRY(st->mids.ensure((slots / (kWarpRowMax + 1) + tiles + 2) * 4));
        u32* wrows = st->hubs.as<u32>();
        u32* crows = st->mids.as<u32>();
        G2M_CUDA(cudaMemsetAsync(wrows, 0, 4, st->stream));
        G2M_CUDA(cudaMemsetAsync(crows, 0, 4, st->stream));
        ++st->launches;
        k_rank_classify<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), nv, wrows, crows);
        G2M_CUDA(cudaGetLastError());
        // disjoint rows; on five side streams they ran no faster (2.08 vs 1.98 ms
        // RMAT-22: the tile pass fills every SM first)
        const u64* o = g->off.as<u64>();
        const u32* nb = g->nbr.as<u32>();
        const u32* rk = rank.as<u32>();
        const u64* ro = g->rk_off.as<u64>();
        u32* rn = g->rk_nbr.as<u32>();
        st->launches += 4;
        k_rank_fill_tiles<<<(int)std::min<u64>(tiles, (u64)st->sms * 7), kTileThreads, 0, st->stream>>>(
            o, nb, nv, slots, rk, ro, rn);
        k_rank_fill_warp<<<st->sms * 8, 256, 0, st->stream>>>(o, nb, rk, ro, rn, wrows);
        k_rank_fill_warp_big<16><<<st->sms * 4, 128, 0, st->stream>>>(o, nb, rk, ro, rn, crows);
        // rows > 512: one CTA each (a warp with 32 values per lane measured 0.06 ms
        // slower at RMAT-22: 165 registers, 12 % warps active, i-cache misses)
        k_rank_fill_hubs<<<st->sms * 6, kRankFillThreads, 0, st->stream>>>(o, nb, rk, ro, rn, crows, 512u);
        G2M_CUDA(cudaGetLastError());
    } else if (nv && slots) {
        int rb = 1;
        while (rb < 32 && ((u64)1 << rb) < nv) ++rb;
        G2M_TRY(st->tmp1.ensure(slots * 8));   // grow-only device scratch, no malloc per call
        G2M_TRY(st->tmp2.ensure(slots * 8));
        u64* k64 = st->tmp1.as<u64>();
        u64* s64 = st->tmp2.as<u64>();
        u32* hubs = nullptr;
        G2M_TRY(hub_list(st, slots, kHubRow, &hubs));
        st->launches += 2;
        k_rank_keys64<<<grid_for(st, nv * 32, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nbr.as<u32>(), nv,
                                                                            rank.as<u32>(), rb, k64, hubs);
        k_rank_keys64_hubs<<<hub_grid(st, slots), kHubThreads, 0, st->stream>>>(g->off.as<u64>(), g->nbr.as<u32>(),
                                                                                rank.as<u32>(), rb, k64, hubs);
        G2M_CUDA(cudaGetLastError());
        phase("scan+keys");
        size_t tb2 = 0;
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, k64, s64, (int64_t)slots, 0, 2 * rb, st->stream));
        G2M_TRY(st->cub_tmp.ensure(tb2));
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(st->cub_tmp.p, tb2, k64, s64, (int64_t)slots, 0, 2 * rb, st->stream));
        ++st->launches;
        k_low_bits<<<grid_for(st, slots, 256), 256, 0, st->stream>>>(s64, slots, rb, g->rk_nbr.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    if (nv && slots && g->oriented) {
        G2M_TRY(st->tmp2.ensure(8));
        u64* dn = st->tmp2.as<u64>();
        G2M_CUDA(cudaMemsetAsync(dn, 0, 8, st->stream));
        ++st->launches;
        k_rank_down_rows<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->rk_off.as<u64>(), g->rk_nbr.as<u32>(), nv,
                                                                          dn);
        G2M_CUDA(cudaGetLastError());
        G2M_CUDA(cudaMemcpyAsync(&g->rk_down, dn, 8, cudaMemcpyDeviceToHost, st->stream));
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    phase("rows");
    trim_scratch(st);
    g->has_rank = true;
    return G2M_OK;
}

// The hub core of an oriented graph's rank-space DAG: the top T = 2^G2M_PAIR_CORE
// ranks as a packed bit matrix (built once, cached). Default 17 (1 GB):
// RMAT-22 TC 27.8 -> 17.6 ms, 4-clique 53.2 -> 34.9 ms with the CTA-tier core
// rows (profiles/r02/core_ab.txt, ctacore_ab.txt); 0 = off.
static g2m_clique::HubCore ensure_core(const g2m_graph* cg, DevState* st) {
    g2m_graph* g = const_cast<g2m_graph*>(cg);
    g2m_clique::HubCore hc{nullptr, 0, 0};
    const char* e = getenv("G2M_PAIR_CORE");
    const int lg = e ? atoi(e) : 17;
    if (lg <= 0 || !g->oriented || !g->has_rank || g->rk_down || g->nv < 2) return hc;
    const u64 T = std::min<u64>((u64)1 << std::min(lg, 20), g->nv);
    if (st->core_gid != g->gid || st->core_T != T) {
        const u64 q = (T - 1) >> 5, r = (T - 1) & 31u;
        const u64 words = 16ull * q * (q + 1) + r * (q + 1) + 1;
        if (st->core_bits.ensure(words * 4) != G2M_OK) { cudaGetLastError(); st->core_gid = 0; return hc; }
        cudaMemsetAsync(st->core_bits.p, 0, words * 4, st->stream);
        st->core_lo = (uint32_t)(g->nv - T);
        ++st->launches;
        g2m_clique::k_core_build<<<grid_for(st, T * 32, 256), 256, 0, st->stream>>>(
            g->rk_off.as<u64>(), g->rk_nbr.as<u32>(), g->nv, st->core_lo, (u32)T, st->core_bits.as<u32>());
        if (cudaGetLastError() != cudaSuccess) { st->core_gid = 0; return hc; }
        st->core_T = (uint32_t)T;
        st->core_gid = g->gid;
    }
    hc.bits = st->core_bits.as<u32>();
    hc.lo = st->core_lo;
    hc.T = st->core_T;
    return hc;
}

extern "C" int g2m_graph_reduced_tasks(const g2m_graph* g, uint64_t* out) {
    if (!g || !out) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    G2M_TRY(ensure_reduced(g, st));
    *out = g->red_total;
    return G2M_OK;
}

// ---- the specialised kernels' own algorithmic work (bench roofline) ---------
// out[0] = operand bytes the algorithm must read at least once (the CSR words
// and offsets it consumes; served by L2 or HBM), out[1] = the unit count the
// cost is linear in, out[2] = updates of counters (4 B read-modify-write
// each), out[3] = sources with work.
//   family 0, k-clique on an oriented graph (bitmap local graphs): per source u
//     the offsets and N+(u), then for each v in N+(u) its offsets and N+(v)
//     (the local-graph probes): 16 n + 20 m + 4 Σ_v d-(v) d+(v);
//     out[1] = Σ_v d-(v) d+(v) (probed ids).
//   family 1, 4-cycle on a symmetric graph (wedge aggregation, rank space):
//     per top vertex r its offsets and N<(r), per v in N<(r) its offsets and
//     the wedge ends N(v) ∩ [lo_x, r): 16 n + 20 Σ_r l(r) + 4 W; out[1] = W
//     wedges, out[2] = W counter increments.
__global__ void k_work_clique(const u64* off, const u32* nbr, u64 nv, const u32* indeg, u64* out) {
    u64 probes = 0, src = 0;
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x) {
        const u64 d = off[v + 1] - off[v];
        probes += d * (u64)indeg[v];
        src += d ? 1 : 0;
    }
    probes = g2m_wsum(probes);
    src = g2m_wsum(src);
    if ((threadIdx.x & 31) == 0) {
        if (probes) atomicAdd(out, probes);
        if (src) atomicAdd(out + 1, src);
    }
}

__global__ void k_work_c4(const u64* off, const u32* nbr, u64 nv, u32 lo_x, u64* out) {
    const u32 lane = g2m_lane();
    u64 w = 0, lsum = 0, src = 0;
    for (u64 r = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; r < nv;
         r += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 b = off[r];
        const u32 d = (u32)(off[r + 1] - b);
        const u32 l1 = g2m_wlb(nbr + b, d, (u32)r);
        if (l1 < 2) continue;
        for (u32 i = lane; i < l1; i += 32) {
            const u32 v = __ldg(nbr + b + i);
            const u64 ro = __ldg(off + v);
            const u32 dv = (u32)(__ldg(off + v + 1) - ro);
            const u32 s0 = g2m_lb(nbr + ro, dv, lo_x), e1 = g2m_lb(nbr + ro, dv, (u32)r);
            w += e1 > s0 ? e1 - s0 : 0;
        }
        if (lane == 0) {
            lsum += l1;
            ++src;
        }
    }
    w = g2m_wsum(w);
    if (lane == 0) {
        if (w) atomicAdd(out, w);
        if (lsum) atomicAdd(out + 1, lsum);
        if (src) atomicAdd(out + 2, src);
    }
}

// family 0 with the hub core (rank space): per source u, its offsets and
// N+(u); per member v = A[i] outside the core its offsets and N+(v), per member
// in the core one 4-byte core word per later member (the bit tests).
// out: [0] bytes beyond the per-source 16 + 4d, [1] probed ids, [2] core bit tests.
__global__ void k_work_clique_core(const u64* off, const u32* nbr, u64 nv, u32 core_lo, int core_on, u64* out) {
    const u32 lane = g2m_lane();
    u64 bytes = 0, probes = 0, bits = 0, src = 0;
    for (u64 u = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; u < nv;
         u += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 b = off[u];
        const u32 d = (u32)(off[u + 1] - b);
        if (d && lane == 0) ++src;
        for (u32 i = lane; i < d; i += 32) {
            const u32 v = __ldg(nbr + b + i);
            if (core_on && v >= core_lo) {
                bits += d - 1 - i;
                bytes += 4ull * (d - 1 - i);
            } else {
                const u64 dv = __ldg(off + v + 1) - __ldg(off + v);
                probes += dv;
                bytes += 16 + 4 * dv;
            }
        }
    }
    bytes = g2m_wsum(bytes);
    probes = g2m_wsum(probes);
    bits = g2m_wsum(bits);
    src = g2m_wsum(src);
    if (lane == 0) {
        if (bytes) atomicAdd(out, bytes);
        if (probes) atomicAdd(out + 1, probes);
        if (bits) atomicAdd(out + 2, bits);
        if (src) atomicAdd(out + 3, src);
    }
}

extern "C" int g2m_kernel_work(const g2m_graph* g, int32_t family, uint64_t* out) {
    if (!g || !out) return fail(G2M_EUSAGE, "null argument");
    // family 2 = family 0 without the hub core (the diamond support tiers probe every list)
    const bool no_core = family == 2;
    if (family == 2) family = 0;
    if (family == 0 && !g->oriented) return fail(G2M_EUSAGE, "clique work needs an oriented graph");
    if (family == 1 && g->oriented) return fail(G2M_EUSAGE, "4-cycle work needs a symmetric graph");
    if (family != 0 && family != 1) return fail(G2M_EUSAGE, "unknown kernel family");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    const u64 nv = g->nv;
    DevBuf acc, indeg;
    G2M_TRY(acc.ensure(4 * 8));
    G2M_CUDA(cudaMemsetAsync(acc.p, 0, 4 * 8, st->stream));
    uint64_t h[4] = {0, 0, 0, 0};
    if (family == 0 && !g->rk_down) {
        // the kernels' own work, in rank space with the hub core they use
        G2M_TRY(ensure_rank(g, st));
        const g2m_clique::HubCore hc = no_core ? g2m_clique::HubCore{nullptr, 0, 0} : ensure_core(g, st);
        if (nv) {
            ++st->launches;
            k_work_clique_core<<<grid_for(st, nv * 32, 256), 256, 0, st->stream>>>(
                g->rk_off.as<u64>(), g->rk_nbr.as<u32>(), nv, hc.lo, hc.bits ? 1 : 0, acc.as<u64>());
            G2M_CUDA(cudaGetLastError());
        }
        G2M_CUDA(cudaMemcpyAsync(h, acc.p, 32, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        out[0] = 16 * nv + 4 * g->slots + h[0];
        out[1] = h[1];
        out[2] = h[2];
        out[3] = h[3];
        return G2M_OK;
    }
    if (family == 0) {
        G2M_TRY(indeg.ensure(std::max<u64>(nv, 1) * 4));
        G2M_CUDA(cudaMemsetAsync(indeg.p, 0, std::max<u64>(nv, 1) * 4, st->stream));
        if (g->slots) {
            ++st->launches;
            k_rank_indeg<<<grid_for(st, g->slots, 256), 256, 0, st->stream>>>(g->nbr.as<u32>(), g->slots,
                                                                                indeg.as<u32>());
        }
        if (nv) {
            ++st->launches;
            k_work_clique<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nbr.as<u32>(), nv,
                                                                            indeg.as<u32>(), acc.as<u64>());
        }
        G2M_CUDA(cudaGetLastError());
        G2M_CUDA(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        out[1] = h[0];
        out[0] = 16 * nv + 20 * g->slots + 4 * h[0];
        out[2] = 0;
        out[3] = h[1];
        return G2M_OK;
    }
    G2M_TRY(ensure_rank(g, st));
    if (nv) {
        ++st->launches;
        k_work_c4<<<grid_for(st, nv * 32, 256), 256, 0, st->stream>>>(g->rk_off.as<u64>(), g->rk_nbr.as<u32>(), nv,
                                                                        (u32)g->rk_deg1, acc.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    G2M_CUDA(cudaMemcpyAsync(h, acc.p, 24, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    out[1] = h[0];
    out[0] = 16 * nv + 20 * h[1] + 4 * h[0];
    out[2] = h[0];
    out[3] = h[2];
    return G2M_OK;
}

// The (degree, id) rank relabelling as a graph of its own (same orientation
// flag): the id space the bitmap-LGS and wedge kernels work in. Relabelling
// it again is the identity, so a chunked round-robin share of its vertices is
// the same source set for those kernels and for the generated plan kernel
// (bench parity at full scale).
extern "C" int g2m_graph_rank_copy(const g2m_graph* g, g2m_graph** out) {
    if (!g || !out) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    G2M_TRY(ensure_rank(g, st));
    auto r = std::make_unique<g2m_graph>();
    r->dev = g->dev;
    r->nv = g->nv;
    r->slots = g->slots;
    r->oriented = g->oriented;
    G2M_TRY(r->off.ensure((g->nv + 1) * 8));
    G2M_TRY(r->nbr.ensure(std::max<u64>(g->slots, 1) * 4));
    G2M_CUDA(cudaMemcpyAsync(r->off.p, g->rk_off.p, (g->nv + 1) * 8, cudaMemcpyDeviceToDevice, st->stream));
    if (g->slots)
        G2M_CUDA(cudaMemcpyAsync(r->nbr.p, g->rk_nbr.p, g->slots * 4, cudaMemcpyDeviceToDevice, st->stream));
    G2M_TRY(finish_graph(r.get(), st));
    *out = r.release();
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// kernels: NVRTC
// ---------------------------------------------------------------------------

struct g2m_kernel {
    g2m_kernel_meta meta;
    std::string name;
    std::vector<char> cubin;
    std::mutex mu;
    std::map<int, std::pair<CUmodule, CUfunction>> mods;
    std::map<int, int> occ;   // blocks per SM per device
};

extern "C" int g2m_kernel_compile(const char* src, const char* name, const char* const* hsrc,
                                  const char* const* hnames, int32_t nh, const g2m_kernel_meta* meta,
                                  g2m_kernel** out) {
    if (!src || !name || !meta || !out) return fail(G2M_EUSAGE, "null argument");
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, src, "g2m_plan.cu", nh, hsrc, hnames);
    if (r != NVRTC_SUCCESS) return fail(G2M_ECUDA, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                          "-default-device", "--device-int128"};
    r = nvrtcCompileProgram(prog, 5, opts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        nvrtcDestroyProgram(&prog);
        return fail(G2M_ECUDA, "NVRTC compile failed:\n" + log);
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    auto k = std::make_unique<g2m_kernel>();
    k->cubin.resize(n);
    nvrtcGetCUBIN(prog, k->cubin.data());
    nvrtcDestroyProgram(&prog);
    k->meta = *meta;
    k->name = name;
    *out = k.release();
    return G2M_OK;
}

extern "C" int g2m_kernel_get_meta(const g2m_kernel* k, g2m_kernel_meta* meta) {
    if (!k || !meta) return fail(G2M_EUSAGE, "null argument");
    *meta = k->meta;
    return G2M_OK;
}

extern "C" int g2m_kernel_destroy(g2m_kernel* k) {
    if (!k) return G2M_OK;
    for (auto& kv : k->mods) {
        cudaSetDevice(kv.first);
        if (g_drv.ok) g_drv.ModuleUnload(kv.second.first);
    }
    delete k;
    return G2M_OK;
}

static int kernel_fn(const g2m_kernel* ck, int dev, DevState* st, CUfunction* fn, int* blocks_per_sm) {
    g2m_kernel* k = const_cast<g2m_kernel*>(ck);
    std::lock_guard<std::mutex> lk(k->mu);
    auto it = k->mods.find(dev);
    if (it == k->mods.end()) {
        CUmodule mod;
        CUfunction f;
        G2M_CU(ModuleLoadData(&mod, k->cubin.data()));
        G2M_CU(ModuleGetFunction(&f, mod, k->name.c_str()));
        const int threads = k->meta.warps_per_block * 32;
        const size_t smem = (size_t)k->meta.warps_per_block * (size_t)k->meta.warp_words * 4;
        if (smem > 48 * 1024)
            G2M_CU(FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem));
        int occ = 0;
        G2M_CU(OccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, threads, smem));
        if (occ < 1) return fail(G2M_ECUDA, "generated kernel cannot be resident (shared memory / registers)");
        k->occ[dev] = occ;
        it = k->mods.emplace(dev, std::make_pair(mod, f)).first;
    }
    *fn = it->second.second;
    *blocks_per_sm = k->occ[dev];
    (void)st;
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// task preparation
// ---------------------------------------------------------------------------

__global__ void k_pairs_u32(const i64* pairs, u64 m, u32* src, u32* dst) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        src[i] = (u32)pairs[2 * i];
        dst[i] = (u32)pairs[2 * i + 1];
    }
}

__global__ void k_i64_u32(const i64* in, u64 m, u32* out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        out[i] = (u32)in[i];
}

struct Prepared {
    G2MArgs a;
    uint64_t h2d = 0;
};

static uint64_t rr_local_count(uint64_t total, uint64_t c, uint32_t parts, uint32_t part) {
    if (c == 0) return total;
    uint64_t nch = (total + c - 1) / c;
    if (part >= nch) return 0;
    uint64_t mine = (nch - part + parts - 1) / parts;   // chunks part, part+parts, ...
    uint64_t last = part + (mine - 1) * parts;          // index of my last chunk
    uint64_t last_size = std::min<uint64_t>(c, total - last * c);
    return (mine - 1) * c + last_size;
}

static int prepare_tasks(const g2m_kernel* k, const g2m_graph* g, const g2m_task_spec* ts,
                         DevState* st, Prepared* P) {
    G2MArgs& a = P->a;
    std::memset(&a, 0, sizeof(a));
    a.off = g->off.as<u64>();
    a.nbr = g->nbr.as<u32>();
    a.labels = g->labels.as<u32>();
    a.nv = g->nv;
    a.kind = ts->kind;
    a.source = ts->source;
    if (ts->kind != k->meta.granularity)
        return fail(G2M_EUSAGE, ts->kind == G2M_TASKS_EDGE ? "edge tasks supplied to a vertex-parallel forest"
                                                           : "vertex tasks supplied to an edge-parallel forest");
    const bool edge = ts->kind == G2M_TASKS_EDGE;
    if (edge && (ts->source == G2M_SRC_IMPLICIT || ts->source == G2M_SRC_INDEX)) {
        if (ts->reduced) {
            G2M_TRY(ensure_reduced(g, st));
            a.task_off = g->red_off.as<u64>();
            a.total_implicit = g->red_total;
        } else {
            a.task_off = g->off.as<u64>();
            a.total_implicit = g->slots;
        }
    } else if (!edge) {
        a.total_implicit = g->nv;
    }
    switch (ts->source) {
    case G2M_SRC_IMPLICIT:
        if (ts->rr_chunk && ts->rr_parts == 0) return fail(G2M_EUSAGE, "rr_parts must be positive");
        a.rr_chunk = ts->rr_chunk;
        a.rr_parts = ts->rr_parts;
        a.rr_part = ts->rr_part;
        a.ntasks = rr_local_count(a.total_implicit, ts->rr_chunk, ts->rr_parts, ts->rr_part);
        break;
    case G2M_SRC_PAIRS: {
        if (!edge) return fail(G2M_EUSAGE, "edge tasks supplied to a vertex-parallel forest");
        a.ntasks = ts->count;
        G2M_TRY(st->tasks_a.ensure(std::max<uint64_t>(ts->count, 1) * 16));
        G2M_TRY(st->tasks_b.ensure(std::max<uint64_t>(ts->count, 1) * 8));
        if (ts->count) {
            G2M_CUDA(cudaMemcpyAsync(st->tasks_a.p, ts->data, ts->count * 16, cudaMemcpyHostToDevice, st->stream));
            ++st->launches;
            k_pairs_u32<<<grid_for(st, ts->count, 256), 256, 0, st->stream>>>(
                st->tasks_a.as<i64>(), ts->count, st->tasks_b.as<u32>(), st->tasks_b.as<u32>() + ts->count);
            G2M_CUDA(cudaGetLastError());
        }
        a.t_src = st->tasks_b.as<u32>();
        a.t_dst = st->tasks_b.as<u32>() + ts->count;
        P->h2d += ts->count * 16;
        break;
    }
    case G2M_SRC_VERTICES: {
        if (edge) return fail(G2M_EUSAGE, "vertex tasks supplied to an edge-parallel forest");
        a.ntasks = ts->count;
        G2M_TRY(st->tasks_a.ensure(std::max<uint64_t>(ts->count, 1) * 8));
        G2M_TRY(st->tasks_b.ensure(std::max<uint64_t>(ts->count, 1) * 4));
        if (ts->count) {
            G2M_CUDA(cudaMemcpyAsync(st->tasks_a.p, ts->data, ts->count * 8, cudaMemcpyHostToDevice, st->stream));
            ++st->launches;
            k_i64_u32<<<grid_for(st, ts->count, 256), 256, 0, st->stream>>>(st->tasks_a.as<i64>(), ts->count,
                                                                               st->tasks_b.as<u32>());
            G2M_CUDA(cudaGetLastError());
        }
        a.t_src = st->tasks_b.as<u32>();
        P->h2d += ts->count * 8;
        break;
    }
    case G2M_SRC_INDEX: {
        a.ntasks = ts->count;
        G2M_TRY(st->tasks_a.ensure(std::max<uint64_t>(ts->count, 1) * 8));
        if (ts->count)
            G2M_CUDA(cudaMemcpyAsync(st->tasks_a.p, ts->data, ts->count * 8, cudaMemcpyHostToDevice, st->stream));
        a.t_index = st->tasks_a.as<u64>();
        P->h2d += ts->count * 8;
        break;
    }
    default:
        return fail(G2M_EUSAGE, "unknown task source");
    }
    return G2M_OK;
}

// counters layout (u64 words): [0] next, [1..] counts (2 per pattern), then stats[16]
static const int kStatsWords = 16;

static int launch(const g2m_kernel* k, const g2m_graph* g, DevState* st, G2MArgs& a,
                  const g2m_run_config* cfg, uint64_t task_lo, uint64_t task_hi, double* kernel_ms,
                  uint64_t* warps_out) {
    CUfunction fn;
    int occ = 0;
    G2M_TRY(kernel_fn(k, g->dev, st, &fn, &occ));
    const int wpb = k->meta.warps_per_block;
    const size_t smem = (size_t)wpb * (size_t)k->meta.warp_words * 4;
    int blocks = (cfg && cfg->blocks > 0) ? cfg->blocks : st->sms * occ;
    // global slot scratch: warps x slots x slot_cap u32
    const uint64_t nslots = (uint64_t)std::max(k->meta.num_slots, 0);
    if (nslots && k->meta.smem_slot_cap == 0) {
        const uint64_t cap = std::max<uint64_t>(g->maxdeg, 1);
        uint64_t budget = (cfg && cfg->scratch_budget) ? cfg->scratch_budget : (uint64_t)24 << 30;
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        budget = std::min<uint64_t>(budget, free_b > ((size_t)2 << 30) ? free_b - ((size_t)2 << 30) : free_b / 2);
        uint64_t per_block = (uint64_t)wpb * nslots * cap * 4;
        uint64_t max_blocks = budget / std::max<uint64_t>(per_block, 1);
        if (max_blocks < 1) return fail(G2M_EBUDGET, "device memory cannot hold one block's slots");
        if ((uint64_t)blocks > max_blocks) blocks = (int)max_blocks;
        G2M_TRY(st->scratch.ensure((uint64_t)blocks * per_block));
        a.scratch = st->scratch.as<u32>();
        a.slot_cap = cap;
    }
    const uint64_t ntask = task_hi - task_lo;
    uint64_t grab = (cfg && cfg->chunk) ? cfg->chunk : 0;
    if (grab == 0) {
        uint64_t warps = (uint64_t)blocks * wpb;
        grab = ntask / (warps * 16);
        if (a.kind == G2M_TASKS_EDGE) grab = std::max<uint64_t>(grab, 1);
        grab = std::min<uint64_t>(std::max<uint64_t>(grab, 1), 256);
        if (k->meta.list_mode) grab = 1;
    }
    a.grab = grab;
    u64* ctr = st->counters.as<u64>();
    a.next = ctr;
    a.counts = ctr + 1;
    a.stats = ctr + 1 + 2 * std::max(k->meta.num_patterns, 1);
    G2M_CUDA(cudaMemcpyAsync(ctr, &task_lo, 8, cudaMemcpyHostToDevice, st->stream));
    a.ntasks = task_hi;
    void* params[] = {&a};
    if (warps_out) *warps_out = (uint64_t)blocks * wpb;
    G2M_CUDA(cudaEventRecord(st->ev0, st->stream));
    if (ntask) ++st->launches;
    if (ntask) G2M_CU(LaunchKernel(fn, blocks, 1, 1, wpb * 32, 1, 1, (unsigned)smem, (CUstream)st->stream, params, nullptr));
    G2M_CUDA(cudaEventRecord(st->ev1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->ev1));
    G2M_CUDA(cudaGetLastError());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, st->ev0, st->ev1);
    if (kernel_ms) *kernel_ms += ms;
    return G2M_OK;
}

static int reset_counters(const g2m_kernel* k, DevState* st) {
    const size_t words = 1 + 2 * (size_t)std::max(k->meta.num_patterns, 1) + kStatsWords;
    G2M_TRY(st->counters.ensure(words * 8));
    G2M_CUDA(cudaMemsetAsync(st->counters.p, 0, words * 8, st->stream));
    return G2M_OK;
}

static int collect(const g2m_kernel* k, DevState* st, uint64_t* counts, g2m_run_stats* stats) {
    const int np = std::max(k->meta.num_patterns, 1);
    const size_t words = 1 + 2 * (size_t)np + kStatsWords;
    std::vector<uint64_t> h(words);
    G2M_CUDA(cudaMemcpyAsync(h.data(), st->counters.p, words * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    if (counts)
        for (int i = 0; i < 2 * k->meta.num_patterns; ++i) counts[i] = h[1 + i];
    if (stats) {
        const uint64_t* s = h.data() + 1 + 2 * np;
        stats->tasks_active = s[0];
        for (int i = 0; i < 8; ++i) stats->high_water[i] = s[1 + i];
        stats->alg_bytes_lo = s[9];
        stats->alg_bytes_hi = s[10];
        stats->d2h_bytes += words * 8;
    }
    return G2M_OK;
}

extern "C" int g2m_run(const g2m_kernel* k, const g2m_graph* g, const g2m_task_spec* ts,
                       const g2m_run_config* cfg, uint64_t* counts, g2m_run_stats* stats) {
    if (!k || !g || !ts) return fail(G2M_EUSAGE, "null argument");
    auto t0 = Clock::now();
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    if (k->meta.needs_labels && !g->labels.p) return fail(G2M_EUSAGE, "kernel compiled for a labeled graph");
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    Prepared P;
    G2M_TRY(prepare_tasks(k, g, ts, st, &P));
    G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
    G2M_TRY(reset_counters(k, st));
    S->tasks = P.a.ntasks;
    G2MArgs a = P.a;
    G2M_TRY(launch(k, g, st, a, cfg, 0, a.ntasks, &S->kernel_ms, &S->warps));
    G2M_TRY(collect(k, st, counts, S));
    G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->evs1));
    {
        float dm = 0.f;
        cudaEventElapsedTime(&dm, st->evs0, st->evs1);
        S->device_ms = dm;
    }
    S->h2d_bytes += P.h2d;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

// Bounded-frontier BFS: per block of tasks, the expand kernel runs levels
// 1-3 (their terminals included) and writes the level-3 candidates as work
// items of `chunk` candidates; the consume kernel runs levels >= 4 over the
// items. A block whose frontier overflows the buffer is halved and redone
// (its partial counts are discarded), so the frontier is bounded by
// `frontier_bytes` whatever the graph.
extern "C" int g2m_run_bfs(const g2m_kernel* ke, const g2m_kernel* kc, const g2m_graph* g,
                           const g2m_task_spec* ts, const g2m_run_config* cfg, uint32_t chunk,
                           uint64_t frontier_bytes, uint64_t* counts, g2m_run_stats* stats) {
    if (!ke || !kc || !g || !ts) return fail(G2M_EUSAGE, "null argument");
    if (ke->meta.num_patterns != kc->meta.num_patterns) return fail(G2M_EUSAGE, "expand/consume kernels differ");
    if (chunk == 0) return fail(G2M_EUSAGE, "frontier chunk must be positive");
    auto t0 = Clock::now();
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    Prepared P;
    G2M_TRY(prepare_tasks(ke, g, ts, st, &P));
    const uint64_t nt = P.a.ntasks;
    S->tasks = nt;
    const int np = std::max(ke->meta.num_patterns, 1);
    std::vector<unsigned __int128> tot(np, 0);
    size_t fr = 0, tb = 0;
    cudaMemGetInfo(&fr, &tb);
    uint64_t fbytes = frontier_bytes ? frontier_bytes : (uint64_t)fr / 4;
    fbytes = std::min<uint64_t>(fbytes, (uint64_t)fr / 2);
    const uint64_t cap = std::max<uint64_t>(fbytes / sizeof(G2MItem), 64);
    DevBuf& items = st->frontier;   // grow-only, kept across calls
    DevBuf fn;
    G2M_TRY(items.ensure(cap * sizeof(G2MItem)));
    G2M_TRY(fn.ensure(8));
    G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
    uint64_t lo = 0, block = nt, peak = 0, blocks = 0;
    std::vector<uint64_t> h(2 * np);
    while (lo < nt) {
        const uint64_t hi = std::min(nt, lo + block);
        // expand levels 1-3 of tasks [lo, hi)
        G2M_TRY(reset_counters(ke, st));
        G2M_CUDA(cudaMemsetAsync(fn.p, 0, 8, st->stream));
        G2MArgs a = P.a;
        a.frontier = items.as<G2MItem>();
        a.frontier_cap = cap;
        a.frontier_n = fn.as<u64>();
        a.fchunk = chunk;
        G2M_TRY(launch(ke, g, st, a, cfg, lo, hi, &S->kernel_ms, &S->warps));
        uint64_t nitems = 0;
        G2M_CUDA(cudaMemcpyAsync(&nitems, fn.p, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        if (nitems > cap) {   // frontier overflow: redo a smaller block
            if (hi - lo == 1) return fail(G2M_EBUDGET, "one task's level-3 frontier exceeds the frontier buffer");
            block = std::max<uint64_t>(1, (hi - lo) / 2);
            continue;
        }
        G2M_TRY(collect(ke, st, h.data(), nullptr));
        for (int p = 0; p < ke->meta.num_patterns; ++p)
            tot[p] += ((unsigned __int128)h[2 * p + 1] << 64) | h[2 * p];
        peak = std::max(peak, nitems);
        ++blocks;
        // consume levels >= 4 of the block's items
        if (nitems) {
            G2M_TRY(reset_counters(kc, st));
            G2MArgs b;
            std::memset(&b, 0, sizeof(b));
            b.off = g->off.as<u64>();
            b.nbr = g->nbr.as<u32>();
            b.labels = g->labels.as<u32>();
            b.nv = g->nv;
            b.kind = G2M_TASKS_EDGE;
            b.frontier = items.as<G2MItem>();
            b.frontier_cap = cap;
            b.fchunk = chunk;
            G2M_TRY(launch(kc, g, st, b, cfg, 0, nitems, &S->kernel_ms, nullptr));
            G2M_TRY(collect(kc, st, h.data(), nullptr));
            for (int p = 0; p < kc->meta.num_patterns; ++p)
                tot[p] += ((unsigned __int128)h[2 * p + 1] << 64) | h[2 * p];
        }
        lo = hi;
    }
    for (int p = 0; p < ke->meta.num_patterns; ++p) {
        counts[2 * p] = (uint64_t)tot[p];
        counts[2 * p + 1] = (uint64_t)(tot[p] >> 64);
    }
    G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->evs1));
    float dm = 0.f;
    cudaEventElapsedTime(&dm, st->evs0, st->evs1);
    S->device_ms = dm;
    S->high_water[6] = blocks;
    S->high_water[7] = peak;
    S->h2d_bytes += P.h2d;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

// List mode: a counting pass sizes every task's match stream, then batches
// of whole tasks are re-run writing tuples at exact offsets, so the host sees
// matches in reference order (task order, then DFS order).
extern "C" int g2m_list(const g2m_kernel* k, const g2m_graph* g, const g2m_task_spec* ts,
                        const g2m_run_config* cfg, g2m_match_cb cb, void* user, uint64_t* counts,
                        g2m_run_stats* stats) {
    if (!k || !g || !ts || !cb) return fail(G2M_EUSAGE, "null argument");
    if (!k->meta.list_mode) return fail(G2M_EUSAGE, "kernel was not generated for list mode");
    auto t0 = Clock::now();
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    Prepared P;
    G2M_TRY(prepare_tasks(k, g, ts, st, &P));
    const uint64_t nt = P.a.ntasks;
    S->tasks = nt;
    // pass 1: per-task match counts
    G2M_TRY(reset_counters(k, st));
    G2M_TRY(st->task_match.ensure(std::max<uint64_t>(nt, 1) * 8));
    G2M_CUDA(cudaMemsetAsync(st->task_match.p, 0, std::max<uint64_t>(nt, 1) * 8, st->stream));
    G2MArgs a = P.a;
    a.task_match = st->task_match.as<u64>();
    a.task_base = 0;
    a.list_pass = 0;
    G2M_TRY(launch(k, g, st, a, cfg, 0, nt, &S->kernel_ms, &S->warps));
    std::vector<uint64_t> per(nt);
    if (nt) G2M_CUDA(cudaMemcpyAsync(per.data(), st->task_match.p, nt * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_TRY(collect(k, st, counts, S));
    S->d2h_bytes += nt * 8;
    const int width = k->meta.max_level + 1;
    const uint64_t cap = std::max<uint64_t>(1, ((uint64_t)64 << 20) / (width * 4));
    G2M_TRY(st->matches.ensure(cap * width * 4));
    std::vector<uint32_t> host;
    std::vector<uint64_t> offs;
    uint64_t t = 0;
    int stopped = 0;
    std::vector<uint64_t> delivered(std::max(k->meta.num_patterns, 1), 0);
    while (t < nt && !stopped) {
        // batch [t, e) with total matches <= cap (at least one task)
        uint64_t e = t, tot = 0;
        offs.clear();
        while (e < nt && (e == t || tot + per[e] <= cap)) {
            offs.push_back(tot);
            tot += per[e];
            ++e;
        }
        if (tot == 0) { t = e; continue; }
        if (tot > cap) {
            G2M_TRY(st->matches.ensure(tot * width * 4));
        }
        G2M_CUDA(cudaMemcpyAsync(st->task_match.p, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, st->stream));
        G2M_TRY(reset_counters(k, st));
        G2MArgs b = P.a;
        b.task_match = st->task_match.as<u64>();
        b.task_base = t;
        b.list_pass = 1;
        b.match_buf = st->matches.as<u32>();
        b.match_cap = tot;
        G2M_TRY(launch(k, g, st, b, cfg, t, e, &S->kernel_ms, nullptr));
        host.resize(tot * width);
        G2M_CUDA(cudaMemcpyAsync(host.data(), st->matches.p, tot * width * 4, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        S->d2h_bytes += tot * width * 4;
        // hand over in order; runs of one pattern id per callback
        uint64_t i = 0;
        while (i < tot && !stopped) {
            uint32_t pid = host[i * width];
            uint64_t j = i + 1;
            while (j < tot && host[j * width] == pid) ++j;
            // deliver one at a time so a stop lands on the exact match
            for (uint64_t q = i; q < j; ++q) {
                delivered[pid] += 1;
                int r = cb(user, (int32_t)pid, width - 1, 1, host.data() + q * width + 1);
                if (r) { stopped = 1; break; }
            }
            i = j;
        }
        t = e;
    }
    if (stopped && counts) {
        for (int p = 0; p < k->meta.num_patterns; ++p) {
            counts[2 * p] = delivered[p];
            counts[2 * p + 1] = 0;
        }
    }
    S->h2d_bytes += P.h2d;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return stopped ? G2M_STOPPED : G2M_OK;
}

// ---------------------------------------------------------------------------
// k-clique via bitmap local graphs
// ---------------------------------------------------------------------------

__global__ void k_heavy_len(const u64* off, const u32* verts, u64 n, u64* len) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u32 v = verts[i];
        len[i] = off[v + 1] - off[v];
    }
}

__global__ void k_heavy_fill(const u64* off, const u32* verts, u64 n, const u64* pos, u64* idx) {
    // one warp per heavy vertex: its slot range [off[v], off[v+1]) as task indices
    const u32 lane = g2m_lane();
    for (u64 i = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u32 v = verts[i];
        const u64 b = off[v], e = off[v + 1];
        for (u64 s = b + lane; s < e; s += 32) idx[pos[i] + (s - b)] = s;
    }
}

// Source classes of k_clique_bucket: 8 pair tier (d <= 64 by default), 1 warp tier,
// 2..5 CTA tiers W = 2..16, 7 CTA tier W = 64 (k = 3) / 32 (rows in L2),
// 6 generic plan kernel.
static const int kClasses = 9;

// Sources up to this out-degree go to the pair tier (G2M_PAIR_MAXD, 0 = off).
static u64 pair_maxd() {
    static const u64 v = [] {
        const char* e = getenv("G2M_PAIR_MAXD");
        return e ? std::min<u64>(strtoull(e, nullptr, 10), 64) : (u64)64;
    }();
    return v;
}

// k = 3, 4 take the pair tier further (G2M_PAIR_MAXD3, <= 128; two-word rows for k = 4).
static u64 pair_maxd3() {
    static const u64 v = [] {
        const char* e = getenv("G2M_PAIR_MAXD3");
        return e ? std::min<u64>(strtoull(e, nullptr, 10), 128) : (u64)128;
    }();
    return v;
}

// Triangle counting (no rows) takes the pair tier furthest (G2M_PAIR_MAXD_TC,
// <= 256): to 128 while the CTA tiers' id windows fit their shared-memory
// bitmaps, to 256 on graphs large enough that they do not (> 2^24 vertices).
static u64 pair_maxd_tc(u64 nv) {
    if (const char* e = getenv("G2M_PAIR_MAXD_TC")) return std::min<u64>(strtoull(e, nullptr, 10), 256);
    return nv > ((u64)1 << 24) ? 256 : 128;
}

template <int K, bool SUP = false>
static int clique_launch_all(const u64* off, const u32* nbr, DevState* st, const u32* lists, u64 stride,
                             const uint64_t* sizes, const uint32_t* spans, u64* ctr, double* kms,
                             u32* tsup = nullptr, g2m_clique::HubCore core = g2m_clique::HubCore{nullptr, 0, 0}) {
    using namespace g2m_clique;
    u64* count = ctr;        // (lo, hi)
    u64* next = ctr + 2;     // one work counter per launch
    int slot = 0;
    const bool dbg = getenv("G2M_DEBUG") != nullptr;
    // The tiers are independent (own work counter, atomic 128-bit count), so
    // they run on the side streams concurrently: a persistent tier's blocks
    // retire as its queue drains and the next tier's blocks take the SMs, so
    // tails overlap instead of draining the GPU between launches. The mining
    // time is the fork -> join span on the main stream. G2M_DEBUG or
    // G2M_SERIAL_TIERS serialise them with one timed launch each.
    // Measured (RMAT-22, r02b): concurrent tiers cost k = 3/4 5-12 % (each
    // tier already fills the GPU; co-resident blocks of two tiers halve the
    // occupancy each was sized for) and gain k = 5 3 % (its W=16 tier runs
    // 1 CTA/SM for 589 ms and the small tiers fill the gaps). Default: one
    // stream without host syncs for k <= 4 (each tier starts as the previous
    // drains), two side streams for k = 5. G2M_TIER_STREAMS=n overrides.
    const bool serial = dbg || getenv("G2M_SERIAL_TIERS") != nullptr;
    const char* ts = getenv("G2M_TIER_STREAMS");
    const int want_streams = ts ? std::max(1, atoi(ts)) : (K == 5 ? 2 : 1);
    const bool one_stream = want_streams == 1;
    const int nstreams = std::min(want_streams, (int)DevState::kSide);
    int nside = 0;
    if constexpr (K == 5) {
        // G2M_CL5_BIG=0: rows with 128 < |R_i| <= 256 stay on the per-warp path
        const u32 big = getenv("G2M_CL5_BIG") ? (u32)atoi(getenv("G2M_CL5_BIG")) : 0u;
        G2M_CUDA(cudaMemcpyToSymbolAsync(g2m_clique::g_cl5_big, &big, 4, 0, cudaMemcpyHostToDevice, st->stream));
    }
    G2M_CUDA(cudaEventRecord(st->ev0, st->stream));
    auto timed = [&](auto&& fn) -> int {
        if (!serial && one_stream) {
            fn(st->stream);
            G2M_CUDA(cudaGetLastError());
            return G2M_OK;
        }
        if (!serial) {
            // ordered after everything on the main stream so far (incl. allocations)
            cudaStream_t s = st->side[nside % nstreams];
            G2M_CUDA(cudaEventRecord(st->evfork, st->stream));
            G2M_CUDA(cudaStreamWaitEvent(s, st->evfork, 0));
            fn(s);
            G2M_CUDA(cudaGetLastError());
            ++nside;
            return G2M_OK;
        }
        cudaEvent_t a = nullptr;
        G2M_CUDA(cudaEventCreate(&a));
        G2M_CUDA(cudaEventRecord(a, st->stream));
        fn(st->stream);
        G2M_CUDA(cudaGetLastError());
        G2M_CUDA(cudaEventRecord(st->ev1, st->stream));
        G2M_CUDA(cudaEventSynchronize(st->ev1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, st->ev1);
        cudaEventDestroy(a);
        if (dbg) fprintf(stderr, "[g2m]   launch %d: %.3f ms\n", slot, ms);
        return G2M_OK;
    };
    auto join = [&]() -> int {
        for (int i = 0; i < std::min(nside, nstreams); ++i) {
            G2M_CUDA(cudaEventRecord(st->evjoin[i], st->side[i]));
            G2M_CUDA(cudaStreamWaitEvent(st->stream, st->evjoin[i], 0));
        }
        G2M_CUDA(cudaEventRecord(st->ev1, st->stream));
        G2M_CUDA(cudaEventSynchronize(st->ev1));
        float ms = 0.f;
        G2M_CUDA(cudaEventElapsedTime(&ms, st->ev0, st->ev1));
        *kms += ms;
        return G2M_OK;
    };
    // G2M_CTA_CORE=0: the CTA tiers probe hub-core rows instead of reading the core bits
    const g2m_clique::HubCore cta_core =
        (getenv("G2M_CTA_CORE") && atoi(getenv("G2M_CTA_CORE")) == 0) ? g2m_clique::HubCore{nullptr, 0, 0} : core;
    int max_smem = 0;
    G2M_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
    int sm_smem = 0;
    G2M_CUDA(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0));
    DevBuf& slab = st->gr_slab;   // global rows of the GR tier (grow-only, per device)
    // G2M_DIRECT_MAX: widest window (bits) for the direct bitmap (tests force
    // the two-level window / hash paths with small values)
    const u32 direct_max = getenv("G2M_DIRECT_MAX") ? (u32)strtoul(getenv("G2M_DIRECT_MAX"), nullptr, 10)
                                                     : 0xffffffffu;
    auto cta = [&](auto wtag, auto nwtag, auto grtag, int cls, int want_ctas) -> int {
        constexpr int W = decltype(wtag)::value;
        constexpr int NW = decltype(nwtag)::value;
        constexpr bool GR = decltype(grtag)::value;
        if (!sizes[cls]) return G2M_OK;
        // window bitmap: as wide as the widest source of the class needs, within
        // the shared memory left at `want_ctas` blocks per SM
        const size_t base = cta_smem_bytes(K, W, NW, 0, GR, SUP);
        const size_t per_block = std::min<size_t>((size_t)max_smem, (size_t)sm_smem / want_ctas - 2048);
        u32 bmw = 0;
        if (per_block > base + 64) bmw = (u32)std::min<size_t>((per_block - base) / 6, ((size_t)spans[cls] + 31) / 32);
        bmw &= ~1u;
        const size_t smem = cta_smem_bytes(K, W, NW, bmw, GR, SUP);
        auto kern = k_clique_cta<K, W, NW, GR, SUP>;
        G2M_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem));
        // a handful of huge sources (the L2-row tier) would leave most SMs idle:
        // split their counting over several blocks each (k > 3)
        const u32 split = (GR && K > 3) ? (u32)std::max<u64>(1, std::min<u64>(32, (u64)st->sms / sizes[cls])) : 1u;
        const u64 items = sizes[cls] * split;
        const u64 grid = std::min<u64>(items, (u64)st->sms * std::max(occ, 1));
        u64* grows = nullptr;
        if (GR) {
            G2M_TRY(slab.ensure(grid * cta_row_words(K, W, NW) * 8));
            grows = slab.as<u64>();
        }
        if (dbg)
            fprintf(stderr, "[g2m] clique k=%d class %d: %llu sources, W=%d NW=%d%s, window<=%u bits, bitmap %u bits, smem %zu, %d CTA/SM\n",
                    K, cls, (unsigned long long)sizes[cls], W, NW, GR ? " (rows in L2)" : "", spans[cls], bmw * 32, smem, occ);
        G2M_TRY(timed([&](cudaStream_t ss) {
            ++st->launches;
            kern<<<(unsigned)grid, NW * 32, smem, ss>>>(off, nbr, lists + (u64)cls * stride, sizes[cls],
                                                                 next + slot, count, bmw, grows, tsup, split,
                                                                 direct_max, cta_core);
        }));
        ++slot;
        return G2M_OK;
    };
    using std::integral_constant;
    using F = std::false_type;
    // heaviest sources first (longest-processing-time order): the tiers with
    // few, large local graphs start at once and the fine-grained tiers fill
    // the SMs their tails leave idle
    if constexpr (K == 3)
        G2M_TRY(cta(integral_constant<int, 64>{}, integral_constant<int, 32>{}, F{}, 7, 1));
    else
        G2M_TRY(cta(integral_constant<int, 32>{}, integral_constant<int, 16>{}, std::true_type{}, 7, 1));
    // one block per SM (the 139 KB of rows allow no second): as many warps as the
    // per-warp candidate lists leave room for
    if constexpr (K == 4)
        G2M_TRY(cta(integral_constant<int, 16>{}, integral_constant<int, 32>{}, F{}, 5, 1));
    else if constexpr (K == 5)
        G2M_TRY(cta(integral_constant<int, 16>{}, integral_constant<int, 24>{}, F{}, 5, 1));
    else   // k = 3: no rows; two blocks per SM, windows beyond the bitmap go two-level
        G2M_TRY(cta(integral_constant<int, 16>{}, integral_constant<int, 16>{}, F{}, 5, 2));
    G2M_TRY(cta(integral_constant<int, 8>{}, integral_constant<int, 16>{}, F{}, 4, 2));
    G2M_TRY(cta(integral_constant<int, 4>{}, integral_constant<int, 16>{}, F{}, 3, 3));
    G2M_TRY(cta(integral_constant<int, 2>{}, integral_constant<int, 16>{}, F{}, 2, 2));
    // G2M_PAIR_BULK=1|2: the staged pair tier (TMA bulk copies of the searched
    // lists; 1: 2 x 512-element buffers per warp, 2: 2 x 1088)
    const int pair_bulk = getenv("G2M_PAIR_BULK") ? atoi(getenv("G2M_PAIR_BULK")) : 0;
    auto bulk_pairs = [&](auto kern, size_t per_warp, int wpb) -> int {
        const size_t smem = per_warp * wpb;
        G2M_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, wpb * 32, smem));
        const u64 grab = std::max<u64>(1, std::min<u64>(16, sizes[8] / ((u64)st->sms * 64 * wpb)));
        if (dbg)
            fprintf(stderr, "[g2m] clique k=%d staged pair tier: %llu sources, %zu B smem per warp, %d CTA/SM\n",
                    K, (unsigned long long)sizes[8], per_warp, occ);
        G2M_TRY(timed([&](cudaStream_t ss) {
            ++st->launches;
            kern<<<st->sms * std::max(occ, 1), wpb * 32, smem, ss>>>(off, nbr, lists + 8 * stride, sizes[8],
                                                                     next + slot, grab, count);
        }));
        ++slot;
        return G2M_OK;
    };
    if (kClasses > 8 && sizes[8] && pair_bulk) {
        constexpr int WPB = 4;
        constexpr int MAXD = K == 3 ? 256 : (K == 4 ? 128 : 64);
        if (pair_bulk == 2)
            G2M_TRY(bulk_pairs(k_clique_pairs_bulk<K, WPB, MAXD, 1088>, sizeof(PairBulkSmem<K, MAXD, 1088>), WPB));
        else
            G2M_TRY(bulk_pairs(k_clique_pairs_bulk<K, WPB, MAXD, 512>, sizeof(PairBulkSmem<K, MAXD, 512>), WPB));
    } else if (kClasses > 8 && sizes[8]) {
        constexpr int WPB = 8;
        u64 grab = std::max<u64>(1, std::min<u64>(16, sizes[8] / ((u64)st->sms * 64 * WPB)));
        // G2M_PAIR_PU: pair tests (core-word loads) in flight per lane per step
        const int pu = getenv("G2M_PAIR_PU") ? atoi(getenv("G2M_PAIR_PU")) : 1;
        G2M_TRY(timed([&](cudaStream_t ss) {
            ++st->launches;
            constexpr int MX = K == 3 ? 256 : (K == 4 ? 128 : 64);
            if (pu >= 4)
                k_clique_pairs<K, WPB, MX, 4><<<st->sms * 8, WPB * 32, 0, ss>>>(
                    off, nbr, lists + 8 * stride, sizes[8], next + slot, grab, count, core);
            else if (pu == 2)
                k_clique_pairs<K, WPB, MX, 2><<<st->sms * 8, WPB * 32, 0, ss>>>(
                    off, nbr, lists + 8 * stride, sizes[8], next + slot, grab, count, core);
            else
                k_clique_pairs<K, WPB, MX, 1><<<st->sms * 8, WPB * 32, 0, ss>>>(
                    off, nbr, lists + 8 * stride, sizes[8], next + slot, grab, count, core);
        }));
        ++slot;
    }
    if (sizes[1]) {
        constexpr int WPB = 8;
        u64 grab = std::max<u64>(1, std::min<u64>(8, sizes[1] / ((u64)st->sms * 64 * WPB)));
        G2M_TRY(timed([&](cudaStream_t ss) {
            ++st->launches;
            k_clique_warp<K, WPB, SUP><<<st->sms * 8, WPB * 32, 0, ss>>>(
                off, nbr, lists + 1 * stride, sizes[1], next + slot, grab, count, tsup);
        }));
        ++slot;
    }
    return join();
}

// ---- pattern-aware workload estimator ----
// Per source vertex of the rank-space graph, the estimated work of its
// search, one warp per source:
//   k-clique (bitmap LGS): Σ_{v ∈ N+(u)} d+(v) (the local-graph probes) +
//                          d+(u) * ceil(d+(u)/32) * (k - 2) (row words per level)
//   4-cycle (wedges):      Σ_{v ∈ N(r), v < r} d(v) (the wedge bound of r)
// The partition deals runs of consecutive sources of equal estimated work
// round-robin (g2m_owns), so a chunk of hub sources is as heavy as a chunk
// of thousands of leaves.
__global__ void k_source_cost(const u64* off, const u32* nbr, u64 nv, int kind, int k, u64* cost, u64* nz) {
    const u32 lane = g2m_lane();
    u64 cnt = 0;
    for (u64 r = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; r < nv;
         r += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 b = off[r];
        const u32 d = (u32)(off[r + 1] - b);
        const u32 l = kind == 0 ? d : g2m_wlb(nbr + b, d, (u32)r);
        u64 w = 0;
        if (l >= (kind == 0 ? (u32)(k - 1) : 2u)) {
            for (u32 i = lane; i < l; i += 32) {
                const u32 v = __ldg(nbr + b + i);
                w += __ldg(off + v + 1) - __ldg(off + v);
            }
            w = g2m_wsum(w);
            if (kind == 0) w += (u64)d * ((d + 31) / 32) * (u64)(k - 2);
        }
        if (lane == 0) {
            cost[r] = w;
            cnt += w ? 1 : 0;
        }
    }
    if (lane == 0 && cnt) atomicAdd(nz, cnt);
}

// wpre/wchunk for a weighted partition `part` of the rank-space graph g
// (kind 0 clique of size k, 1 4-cycle); nullptr/0 when not weighted.
static int source_weights(const g2m_graph* cg, DevState* st, const g2m_task_spec* part, int kind, int k,
                          const u64** wpre, u64* wchunk) {
    *wpre = nullptr;
    *wchunk = 0;
    if (!part || !part->weighted || !part->rr_chunk) return G2M_OK;
    g2m_graph* g = const_cast<g2m_graph*>(cg);
    const u64 nv = g->nv;
    const int key = kind * 16 + k;
    if (g->wpre_key != key) {
        G2M_TRY(g->wpre.ensure((nv + 1) * 8));
        G2M_TRY(st->tmp2.ensure((nv + 1) * 8 + 8));
        u64* cost = st->tmp2.as<u64>();
        u64* nz = cost + nv + 1;
        G2M_CUDA(cudaMemsetAsync(cost, 0, (nv + 1) * 8 + 8, st->stream));
        if (nv) {
            ++st->launches;
            k_source_cost<<<grid_for(st, nv * 32, 256), 256, 0, st->stream>>>(g->rk_off.as<u64>(), g->rk_nbr.as<u32>(),
                                                                                 nv, kind, k, cost, nz);
            G2M_CUDA(cudaGetLastError());
        }
        G2M_TRY(exclusive_scan_u64(st, cost, g->wpre.as<u64>(), nv));
        uint64_t h[2] = {0, 0};
        G2M_CUDA(cudaMemcpyAsync(h, g->wpre.as<u64>() + nv, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaMemcpyAsync(h + 1, nz, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        g->wpre_total = h[0];
        g->wpre_sources = h[1];
        g->wpre_key = key;
    }
    // as many chunks as chunks of rr_chunk sources there are (c = alpha * y),
    // each carrying an equal share of the estimated work
    const u64 nchunks = std::max<u64>(1, g->wpre_sources / part->rr_chunk);
    *wchunk = std::max<u64>(1, (g->wpre_total + nchunks - 1) / nchunks);
    *wpre = g->wpre.as<u64>();
    return G2M_OK;
}

static int clique_impl(const g2m_graph* g, int32_t k, const g2m_task_spec* part, const g2m_kernel* fallback,
                       const g2m_run_config* cfg, uint64_t* counts, g2m_run_stats* stats, DevState* st);

extern "C" int g2m_clique_count(const g2m_graph* g, int32_t k, const g2m_task_spec* part,
                                const g2m_kernel* fallback, const g2m_run_config* cfg,
                                uint64_t* counts, g2m_run_stats* stats) {
    if (!g || !counts) return fail(G2M_EUSAGE, "null argument");
    if (!g->oriented) return fail(G2M_EUSAGE, "plan orientation does not match the graph");
    if (k < 3 || k > 5) return fail(G2M_EUSAGE, "bitmap clique kernels cover 3 <= k <= 5");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    return clique_impl(g, k, part, fallback, cfg, counts, stats, st);
}

// g2m_clique_count with the device lock held
static int clique_impl(const g2m_graph* g, int32_t k, const g2m_task_spec* part, const g2m_kernel* fallback,
                       const g2m_run_config* cfg, uint64_t* counts, g2m_run_stats* stats, DevState* st) {
    auto t0 = Clock::now();
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    u64 rr_chunk = 0;
    u32 parts = 1, pt = 0;
    if (part && part->rr_chunk) {
        if (part->rr_parts == 0) return fail(G2M_EUSAGE, "rr_parts must be positive");
        rr_chunk = part->rr_chunk;
        parts = part->rr_parts;
        pt = part->rr_part;
    }
    // the kernels run on the rank-space copy of the DAG (built once per graph)
    G2M_TRY(ensure_rank(g, st));
    const u64* off = g->rk_off.as<u64>();
    const u32* nbr = g->rk_nbr.as<u32>();
    const u64* wpre = nullptr;
    u64 wchunk = 0;
    G2M_TRY(source_weights(g, st, part, 0, k, &wpre, &wchunk));
    const bool dbgc = getenv("G2M_DEBUG") != nullptr;
    auto tc0 = Clock::now();
    const g2m_clique::HubCore core = ensure_core(g, st);
    if (dbgc) {
        cudaStreamSynchronize(st->stream);
        fprintf(stderr, "[g2m] hub core: %.2f ms (setup since call start %.2f ms)\n", ms_since(tc0), ms_since(t0));
    }
    G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
    // counters: ctr[8..9] count (lo, hi), ctr[10..] one work counter per launch
    G2M_TRY(st->counters.ensure(32 * 8));
    u64* ctr = st->counters.as<u64>();
    G2M_CUDA(cudaMemsetAsync(ctr, 0, 32 * 8, st->stream));
    const u64 stride = std::max<u64>(g->nv, 1);
    G2M_TRY(st->tasks_b.ensure((u64)kClasses * stride * 4));
    G2M_TRY(st->tasks_a.ensure(kClasses * 8 + kClasses * 4));
    u64* dsizes = st->tasks_a.as<u64>();
    u32* dspans = (u32*)(dsizes + kClasses);
    G2M_CUDA(cudaMemsetAsync(dsizes, 0, kClasses * 12, st->stream));
    if (g->nv) {
        ++st->launches;
        // a DAG not oriented by (degree, id) (Graph(..., oriented=True) from another
        // orientation) breaks the tiers' "edges point up" invariant: every source
        // then takes the generated plan kernel (max_cta_d = 0)
        g2m_clique::k_clique_bucket<<<grid_for(st, g->nv, 256), 256, 0, st->stream>>>(
            off, nbr, g->nv, k - 1, g->rk_down ? 0 : (k == 3 ? 4096 : 2048),
            k == 3 ? pair_maxd_tc(g->nv) : (k == 4 ? pair_maxd3() : pair_maxd()), rr_chunk, parts, pt, wpre,
            wchunk, st->tasks_b.as<u32>(),
            stride, dsizes, dspans);
        G2M_CUDA(cudaGetLastError());
    }
    uint64_t sizes[kClasses];
    uint32_t spans[kClasses];
    G2M_CUDA(cudaMemcpyAsync(sizes, dsizes, kClasses * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaMemcpyAsync(spans, dspans, kClasses * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    const u32* lists = st->tasks_b.as<u32>();
    if (getenv("G2M_DEBUG"))
        fprintf(stderr, "[g2m] clique k=%d buckets: pairs %llu warp<=64:%llu 128:%llu 256:%llu 512:%llu 1024:%llu 4096:%llu generic:%llu\n",
                k, (unsigned long long)sizes[8], (unsigned long long)sizes[1], (unsigned long long)sizes[2], (unsigned long long)sizes[3],
                (unsigned long long)sizes[4], (unsigned long long)sizes[5], (unsigned long long)sizes[7],
                (unsigned long long)sizes[6]);
    {
        u64* blk = ctr + 8;
        int rc;
        switch (k) {
        case 3: rc = clique_launch_all<3>(off, nbr, st, lists, stride, sizes, spans, blk, &S->kernel_ms, nullptr, core); break;
        case 4: rc = clique_launch_all<4>(off, nbr, st, lists, stride, sizes, spans, blk, &S->kernel_ms, nullptr, core); break;
        default: rc = clique_launch_all<5>(off, nbr, st, lists, stride, sizes, spans, blk, &S->kernel_ms, nullptr, core); break;
        }
        if (rc != G2M_OK) return rc;
    }
    uint64_t h[2] = {0, 0};
    G2M_CUDA(cudaMemcpyAsync(h, ctr + 8, 16, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    unsigned __int128 total = ((unsigned __int128)h[1] << 64) | h[0];
    S->tasks = 0;
    for (int c = 1; c < kClasses; ++c) S->tasks += sizes[c];
    // sources beyond the bitmap tiers: the generated plan kernel over their edge tasks
    if (sizes[6]) {
        if (!fallback) return fail(G2M_EUSAGE, "sources beyond the bitmap tiers need a fallback kernel");
        const u64 nh = sizes[6];
        DevBuf lens, pos, idx;
        G2M_TRY(lens.ensure(nh * 8));
        G2M_TRY(pos.ensure((nh + 1) * 8));
        ++st->launches;
        k_heavy_len<<<grid_for(st, nh, 256), 256, 0, st->stream>>>(off, lists + 6 * stride, nh, lens.as<u64>());
        G2M_CUDA(cudaGetLastError());
        G2M_TRY(exclusive_scan_u64(st, lens.as<u64>(), pos.as<u64>(), nh));
        uint64_t ntask = 0;
        G2M_CUDA(cudaMemcpyAsync(&ntask, pos.as<u64>() + nh, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        G2M_TRY(idx.ensure(std::max<uint64_t>(ntask, 1) * 8));
        ++st->launches;
        k_heavy_fill<<<grid_for(st, nh * 32, 256), 256, 0, st->stream>>>(off, lists + 6 * stride, nh,
                                                                          pos.as<u64>(), idx.as<u64>());
        G2M_CUDA(cudaGetLastError());
        G2M_TRY(reset_counters(fallback, st));
        G2MArgs a;
        std::memset(&a, 0, sizeof(a));
        a.off = off;
        a.nbr = nbr;
        a.nv = g->nv;
        a.kind = G2M_TASKS_EDGE;
        a.source = G2M_SRC_INDEX;
        a.task_off = off;
        a.total_implicit = g->slots;
        a.t_index = idx.as<u64>();
        a.ntasks = ntask;
        G2M_TRY(launch(fallback, g, st, a, cfg, 0, ntask, &S->kernel_ms, nullptr));
        uint64_t fc[2] = {0, 0};
        G2M_TRY(collect(fallback, st, fc, nullptr));
        total += ((unsigned __int128)fc[1] << 64) | fc[0];
    }
    counts[0] = (uint64_t)total;
    counts[1] = (uint64_t)(total >> 64);
    G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->evs1));
    float dm = 0.f;
    cudaEventElapsedTime(&dm, st->evs0, st->evs1);
    S->device_ms = dm;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// diamond count from per-edge triangle support
// ---------------------------------------------------------------------------
// Edge-induced diamonds = Σ over edges {u, v} of C(|N(u) ∩ N(v)|, 2): the
// count the reference's counting rewrite evaluates per edge task
// (plan.py:177-198, executor.py:204-216). |N(u) ∩ N(v)| is the number of
// triangles on the edge, accumulated by the bitmap triangle kernels over the
// rank-space DAG of the degree orientation (one support counter per DAG edge).

// Triangle support of every edge of the degree-oriented rank-space DAG of a
// symmetric graph, from the triangles whose DAG source is in `part` (all when
// null), added into tsup (og->slots u32 per rank-space slot). Builds the
// oriented copy and its rank relabelling once per graph. Device lock held.
static int diamond_support_impl(const g2m_graph* g, const g2m_task_spec* part, u32* tsup, g2m_run_stats* S,
                                DevState* st, const g2m_graph** og_out) {
    g2m_graph* gm = const_cast<g2m_graph*>(g);
    {
        std::lock_guard<std::mutex> glk(gm->mu);
        if (!gm->oriented_copy) {
            g2m_graph* o = nullptr;
            G2M_TRY(orient_impl(g, st, &o));
            gm->oriented_copy.reset(o);
        }
    }
    const g2m_graph* og = gm->oriented_copy.get();
    *og_out = og;
    G2M_TRY(ensure_rank(og, st));
    if (!tsup) return G2M_OK;
    u64 rr_chunk = 0;
    u32 parts = 1, pt = 0;
    if (part && part->rr_chunk) {
        if (part->rr_parts == 0) return fail(G2M_EUSAGE, "rr_parts must be positive");
        rr_chunk = part->rr_chunk;
        parts = part->rr_parts;
        pt = part->rr_part;
    }
    const u64* off = og->rk_off.as<u64>();
    const u32* nbr = og->rk_nbr.as<u32>();
    const u64* wpre = nullptr;
    u64 wchunk = 0;
    G2M_TRY(source_weights(og, st, part, 0, 3, &wpre, &wchunk));
    G2M_TRY(st->counters.ensure(32 * 8));
    u64* ctr = st->counters.as<u64>();
    G2M_CUDA(cudaMemsetAsync(ctr, 0, 32 * 8, st->stream));
    const u64 stride = std::max<u64>(og->nv, 1);
    G2M_TRY(st->tasks_b.ensure((u64)kClasses * stride * 4));
    G2M_TRY(st->tasks_a.ensure(kClasses * 8 + kClasses * 4));
    u64* dsizes = st->tasks_a.as<u64>();
    u32* dspans = (u32*)(dsizes + kClasses);
    G2M_CUDA(cudaMemsetAsync(dsizes, 0, kClasses * 12, st->stream));
    if (og->nv) {
        ++st->launches;
        g2m_clique::k_clique_bucket<<<grid_for(st, og->nv, 256), 256, 0, st->stream>>>(
            off, nbr, og->nv, 2, 4096, 0, rr_chunk, parts, pt, wpre, wchunk, st->tasks_b.as<u32>(), stride, dsizes,
            dspans);
        G2M_CUDA(cudaGetLastError());
    }
    uint64_t sizes[kClasses];
    uint32_t spans[kClasses];
    G2M_CUDA(cudaMemcpyAsync(sizes, dsizes, kClasses * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaMemcpyAsync(spans, dspans, kClasses * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    if (sizes[6]) return fail(G2M_EUSAGE, "diamond support kernels cover out-degrees <= 4096");
    G2M_TRY((clique_launch_all<3, true>(off, nbr, st, st->tasks_b.as<u32>(), stride, sizes, spans, ctr + 8,
                                         &S->kernel_ms, tsup)));
    S->tasks = 0;
    for (int c = 1; c < kClasses; ++c) S->tasks += sizes[c];
    return G2M_OK;
}

// Σ C(tsup[s], 2) over slots [lo, hi) into ctr (lo, hi), timed into kms.
static int support_choose2(DevState* st, const u32* tsup, u64 lo, u64 hi, u64* ctr, double* kms) {
    G2M_CUDA(cudaEventRecord(st->ev0, st->stream));
    if (hi > lo) {
        ++st->launches;
        g2m_clique::k_sum_choose2<<<grid_for(st, hi - lo, 256), 256, 0, st->stream>>>(tsup + lo, hi - lo, ctr);
        G2M_CUDA(cudaGetLastError());
    }
    G2M_CUDA(cudaEventRecord(st->ev1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, st->ev0, st->ev1);
    *kms += ms;
    return G2M_OK;
}

extern "C" int g2m_diamond_count(const g2m_graph* g, const g2m_run_config* cfg, uint64_t* counts,
                                 g2m_run_stats* stats) {
    (void)cfg;
    if (!g || !counts) return fail(G2M_EUSAGE, "null argument");
    if (g->oriented) return fail(G2M_EUSAGE, "plan orientation does not match the graph");
    auto t0 = Clock::now();
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    const g2m_graph* og = nullptr;
    G2M_TRY(diamond_support_impl(g, nullptr, nullptr, S, st, &og));   // oriented copy + rank (untimed)
    G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
    DevBuf& tsup = st->tmp1;   // grow-only scratch (the rank build that also uses it is done)
    G2M_TRY(tsup.ensure(std::max<u64>(og->slots, 1) * 4));
    G2M_CUDA(cudaMemsetAsync(tsup.p, 0, std::max<u64>(og->slots, 1) * 4, st->stream));
    G2M_TRY(diamond_support_impl(g, nullptr, tsup.as<u32>(), S, st, &og));
    u64* ctr = st->counters.as<u64>();
    G2M_TRY(support_choose2(st, tsup.as<u32>(), 0, og->slots, ctr + 16, &S->kernel_ms));
    uint64_t h[2] = {0, 0};
    G2M_CUDA(cudaMemcpyAsync(h, ctr + 16, 16, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->evs1));
    counts[0] = h[0];
    counts[1] = h[1];
    float dm = 0.f;
    cudaEventElapsedTime(&dm, st->evs0, st->evs1);
    S->device_ms = dm;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

extern "C" int g2m_diamond_support(const g2m_graph* g, const g2m_task_spec* part, uint32_t* tsup,
                                   uint64_t* num_slots, g2m_run_stats* stats) {
    if (!g || !num_slots) return fail(G2M_EUSAGE, "null argument");
    if (g->oriented) return fail(G2M_EUSAGE, "diamond support needs the symmetric graph");
    auto t0 = Clock::now();
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    const g2m_graph* og = nullptr;
    G2M_TRY(diamond_support_impl(g, part, nullptr, S, st, &og));
    *num_slots = og->slots;
    if (tsup) {
        G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
        G2M_TRY(diamond_support_impl(g, part, tsup, S, st, &og));
        G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
        G2M_CUDA(cudaEventSynchronize(st->evs1));
        float dm = 0.f;
        cudaEventElapsedTime(&dm, st->evs0, st->evs1);
        S->device_ms = dm;
    }
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

extern "C" int g2m_support_choose2(const g2m_graph* g, const uint32_t* tsup, uint64_t lo, uint64_t hi,
                                   uint64_t* counts, g2m_run_stats* stats) {
    if (!g || !tsup || !counts) return fail(G2M_EUSAGE, "null argument");
    if (lo > hi) return fail(G2M_EUSAGE, "lo > hi");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    const g2m_graph* og = g->oriented ? g : const_cast<g2m_graph*>(g)->oriented_copy.get();
    if (!og || hi > og->slots) return fail(G2M_EUSAGE, "slot range beyond the support array");
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    G2M_TRY(st->counters.ensure(32 * 8));
    u64* ctr = st->counters.as<u64>();
    G2M_CUDA(cudaMemsetAsync(ctr + 16, 0, 16, st->stream));
    G2M_TRY(support_choose2(st, tsup, lo, hi, ctr + 16, &S->kernel_ms));
    G2M_CUDA(cudaMemcpy(counts, ctr + 16, 16, cudaMemcpyDeviceToHost));
    S->device_ms = S->kernel_ms;
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// 4-cycle count by wedge aggregation (cycle4_kernels.cuh)
// ---------------------------------------------------------------------------

static int cycle4_impl(const g2m_graph* g, const g2m_task_spec* part, uint64_t* counts, g2m_run_stats* stats,
                       DevState* st);

extern "C" int g2m_cycle4_count(const g2m_graph* g, const g2m_task_spec* part, const g2m_run_config* cfg,
                                uint64_t* counts, g2m_run_stats* stats) {
    (void)cfg;
    if (!g || !counts) return fail(G2M_EUSAGE, "null argument");
    if (g->oriented) return fail(G2M_EUSAGE, "plan orientation does not match the graph");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    return cycle4_impl(g, part, counts, stats, st);
}

// g2m_cycle4_count with the device lock held
static int cycle4_impl(const g2m_graph* g, const g2m_task_spec* part, uint64_t* counts, g2m_run_stats* stats,
                       DevState* st) {
    auto t0 = Clock::now();
    g2m_run_stats local{};
    g2m_run_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    const uint64_t l0 = st->launches;
    u64 rr_chunk = 0;
    u32 parts = 1, pt = 0;
    if (part && part->rr_chunk) {
        if (part->rr_parts == 0) return fail(G2M_EUSAGE, "rr_parts must be positive");
        rr_chunk = part->rr_chunk;
        parts = part->rr_parts;
        pt = part->rr_part;
    }
    G2M_TRY(ensure_rank(g, st));
    const u64* off = g->rk_off.as<u64>();
    const u32* nbr = g->rk_nbr.as<u32>();
    const u64 nv = g->nv;
    const u32 lo_x = (u32)g->rk_deg1;
    const u64* wpre = nullptr;
    u64 wchunk = 0;
    G2M_TRY(source_weights(g, st, part, 1, 4, &wpre, &wchunk));
    const bool dbg = getenv("G2M_DEBUG") != nullptr;
    constexpr int NW = 16;
    // tier 3 setup: bucket array in shared memory, staging slab per block
    int max_smem = 0;
    G2M_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->dev));
    const u32 nbmax = (u32)((nv >> g2m_c4::kBucketBits) + 2 + 3) & ~3u;   // keeps the u64 scratch aligned
    const size_t stage_smem = g2m_c4::stage_smem_bytes(NW, nbmax);
    // coarse-bucket staging (k_c4_stage2, 32 warps) unless G2M_C4_FINE selects the 1024-id buckets
    // Fine buckets while every block's open write cursors (one 32 B sector per
    // bucket) fit a quarter of L2 together; beyond that the scatter thrashes
    // L2 and the coarse buckets win (RMAT-24: 2.63 -> 1.55 s).
    int l2 = 0;
    G2M_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->dev));
    bool coarse = (u64)nbmax * 32 * st->sms > (u64)l2 / 4;
    if (const char* e = getenv("G2M_C4_FINE")) coarse = atoi(e) == 0;
    constexpr int NW2 = 32;
    const u32 nbmax2 = (u32)((nv >> g2m_c4::kCoarseBits) + 2 + 3) & ~3u;
    const size_t stage2_smem = g2m_c4::stage2_smem_bytes(NW2, nbmax2);
    const bool tier3 = (coarse ? stage2_smem : stage_smem) <= (size_t)max_smem;
    // wedges per v1 staged (64 MB slab per block). 64M was measured too:
    // RMAT-25 6.59 -> 6.48 s, but RMAT-27 58 -> 85 s (the moved top vertices
    // have 4096 coarse buckets each; the staged tier's per-bucket barriers
    // dominate them), so 16M.
    u64 stage_cap = tier3 ? ((u64)16 << 20) : 0;
    if (const char* e = getenv("G2M_C4_STAGE_CAP")) stage_cap = tier3 ? strtoull(e, nullptr, 10) : 0;
    G2M_CUDA(cudaEventRecord(st->evs0, st->stream));
    G2M_TRY(st->counters.ensure(32 * 8));
    u64* ctr = st->counters.as<u64>();
    G2M_CUDA(cudaMemsetAsync(ctr, 0, 32 * 8, st->stream));
    const u64 stride = std::max<u64>(nv, 1);
    // lists/lows: classes 0..4 x nv u32 each; wkeys (class 3 sort keys) + sorted copy
    G2M_TRY(st->tasks_b.ensure(10 * stride * 4));
    G2M_TRY(st->matches.ensure(2 * stride * 8));
    G2M_TRY(st->tasks_a.ensure(16 * 8));
    u32* lists = st->tasks_b.as<u32>();
    u32* lows = lists + 5 * stride;
    u64* wkeys = st->matches.as<u64>();
    u64* wsorted = wkeys + stride;
    u64* dsizes = st->tasks_a.as<u64>();
    G2M_CUDA(cudaMemsetAsync(dsizes, 0, 16 * 8, st->stream));
    if (nv) {
        ++st->launches;
        g2m_c4::k_c4_bucket<<<grid_for(st, nv * 32, 256), 256, 0, st->stream>>>(
            off, nbr, nv, rr_chunk, parts, pt, wpre, wchunk, stage_cap, lists, lows, wkeys, stride, dsizes);
        G2M_CUDA(cudaGetLastError());
    }
    uint64_t sizes[10];
    G2M_CUDA(cudaMemcpyAsync(sizes, dsizes, 10 * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    if (dbg)
        fprintf(stderr, "[g2m] cycle4: warp %llu, cta %llu, staged %llu, grid %llu sources (lo_x %u); "
                        "wedge bounds %llu %llu %llu %llu\n",
                (unsigned long long)sizes[1], (unsigned long long)sizes[2], (unsigned long long)sizes[3],
                (unsigned long long)sizes[4], lo_x, (unsigned long long)sizes[6], (unsigned long long)sizes[7],
                (unsigned long long)sizes[8], (unsigned long long)sizes[9]);
    // the staged tier runs its largest wedge fans first
    if (sizes[3]) {
        size_t tb = 0;
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, wkeys, wsorted, (int64_t)sizes[3], 0, 64, st->stream));
        G2M_TRY(st->cub_tmp.ensure(tb));
        G2M_CUDA(cub::DeviceRadixSort::SortKeys(st->cub_tmp.p, tb, wkeys, wsorted, (int64_t)sizes[3], 0, 64,
                                                st->stream));
        ++st->launches;
        g2m_c4::k_c4_unpack<<<grid_for(st, sizes[3], 256), 256, 0, st->stream>>>(
            wsorted, sizes[3], off, nbr, lists + 3 * stride, lows + 3 * stride);
        G2M_CUDA(cudaGetLastError());
    }
    u64* count = ctr + 8;
    u64* next = ctr + 10;
    int slot = 0;
    auto timed = [&](auto&& fn) -> int {
        G2M_CUDA(cudaEventRecord(st->ev0, st->stream));
        if constexpr (std::is_same_v<decltype(fn()), int>) {
            G2M_TRY(fn());
        } else {
            fn();
        }
        G2M_CUDA(cudaGetLastError());
        G2M_CUDA(cudaEventRecord(st->ev1, st->stream));
        G2M_CUDA(cudaEventSynchronize(st->ev1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, st->ev0, st->ev1);
        S->kernel_ms += ms;
        if (dbg) fprintf(stderr, "[g2m]   cycle4 launch %d: %.3f ms\n", slot, ms);
        ++slot;
        return G2M_OK;
    };
    if (sizes[1]) {
        constexpr int WPB = 4;     // 4 x 8.4 KB of static shared memory
        auto kern = g2m_c4::k_c4_warp<WPB>;
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WPB * 32, 0));
        G2M_TRY(timed([&] {
            ++st->launches;
            kern<<<st->sms * std::max(occ, 1), WPB * 32, 0, st->stream>>>(off, nbr, lists + stride, lows + stride,
                                                                           sizes[1], next + 0, count, lo_x);
        }));
    }
    if (sizes[2]) {
        const u32 cap = 16384;
        const size_t smem = (size_t)2 * cap * 4 + (size_t)NW * 96 * 4;
        auto kern = g2m_c4::k_c4_cta<NW>;
        G2M_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem));
        const u64 grid = std::min<u64>(sizes[2], (u64)st->sms * std::max(occ, 1));
        G2M_TRY(timed([&] {
            ++st->launches;
            kern<<<(unsigned)grid, NW * 32, smem, st->stream>>>(off, nbr, lists + 2 * stride, lows + 2 * stride,
                                                                 sizes[2], next + 1, count, cap, lo_x);
        }));
    }
    if (sizes[3] && coarse) {
        // G2M_C4_ROUNDS=0: every bucket counted by the whole CTA (two barriers each)
        const u32 rounds = getenv("G2M_C4_ROUNDS") ? (u32)atoi(getenv("G2M_C4_ROUNDS")) : 1u;
        G2M_CUDA(cudaMemcpyToSymbolAsync(g2m_c4::g_c4_rounds, &rounds, 4, 0, cudaMemcpyHostToDevice, st->stream));
        auto kern = g2m_c4::k_c4_stage2<NW2>;
        G2M_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage2_smem));
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW2 * 32, stage2_smem));
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        u64 grid = std::min<u64>(sizes[3], (u64)st->sms * std::max(occ, 1));
        grid = std::min<u64>(grid, std::max<u64>(1, (fr + st->c4slab.bytes) / 4 / (stage_cap * 4)));
        G2M_TRY(st->c4slab.ensure(grid * stage_cap * 4));
        G2M_TRY(timed([&] {
            ++st->launches;
            kern<<<(unsigned)grid, NW2 * 32, stage2_smem, st->stream>>>(off, nbr, lists + 3 * stride,
                                                                         lows + 3 * stride, sizes[3], next + 2, count,
                                                                         st->c4slab.as<u32>(), stage_cap, nbmax2, lo_x);
        }));
    } else if (sizes[3]) {
        auto kern = g2m_c4::k_c4_stage<NW>;
        G2M_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_smem));
        int occ = 0;
        G2M_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, stage_smem));
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        u64 grid = std::min<u64>(sizes[3], (u64)st->sms * std::max(occ, 1));
        grid = std::min<u64>(grid, std::max<u64>(1, (fr + st->c4slab.bytes) / 4 / (stage_cap * 4)));
        G2M_TRY(st->c4slab.ensure(grid * stage_cap * 4));
        G2M_TRY(timed([&] {
            ++st->launches;
            kern<<<(unsigned)grid, NW * 32, stage_smem, st->stream>>>(off, nbr, lists + 3 * stride, lows + 3 * stride,
                                                                       sizes[3], next + 2, count, st->c4slab.as<u32>(),
                                                                       stage_cap, nbmax, lo_x);
        }));
    }
    if (sizes[4]) {
        // one v1 at a time on the whole grid, its wedges flattened over all
        // warps; counters shared by the grid for one id range per pass
        // (G2M_C4_RANGE ids, default 2^24 = 64 MB of counters: L2-resident)
        std::vector<u32> gv(sizes[4]), gl(sizes[4]);
        G2M_CUDA(cudaMemcpyAsync(gv.data(), lists + 4 * stride, sizes[4] * 4, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaMemcpyAsync(gl.data(), lows + 4 * stride, sizes[4] * 4, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        u32 lmax = 0;
        for (u32 l : gl) lmax = std::max(lmax, l);
        // Fire-and-forget increments + a C(c,2) sweep per range (G2M_C4_RED=0:
        // increments returning the old count, then a memset). RMAT-25 grid tier
        // 3.80 -> 3.15 s (profiles/r02/c4_grid_ab.txt).
        const bool red = !(getenv("G2M_C4_RED") && atoi(getenv("G2M_C4_RED")) == 0);
        u64 range = (u64)1 << 24;
        if (const char* e = getenv("G2M_C4_RANGE")) range = std::max<u64>(1024, strtoull(e, nullptr, 10));
        range = std::min<u64>(range, stride);
        G2M_TRY(st->tmp1.ensure(range * 4 + 64));
        G2M_TRY(st->tmp2.ensure((u64)lmax * 24 + 64));
        u32* dense = st->tmp1.as<u32>();
        u64* rn = st->tmp2.as<u64>();
        u64* rb = rn + lmax;
        u64* re = rb + lmax;
        u64* gctr = ctr + 12;
        size_t tb = 0;
        G2M_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, rn, re, (int64_t)lmax, st->stream));
        G2M_TRY(st->cub_tmp.ensure(tb));
        G2M_CUDA(cudaMemsetAsync(dense, 0, range * 4, st->stream));
        u64 passes = 0;
        G2M_TRY(timed([&]() -> int {
            for (u64 q = 0; q < sizes[4]; ++q) {
                const u32 r1 = gv[q], l1 = gl[q];
                for (u64 lo = lo_x; lo < r1; lo += range) {
                    const u32 hi = (u32)std::min<u64>(r1, lo + range);
                    ++passes;
                    ++st->launches;
                    g2m_c4::k_c4_rows<<<grid_for(st, l1, 256), 256, 0, st->stream>>>(off, nbr, r1, l1, (u32)lo, hi,
                                                                                       rn, rb);
                    size_t t2 = tb;
                    G2M_CUDA(cub::DeviceScan::InclusiveSum(st->cub_tmp.p, t2, rn, re, (int64_t)l1, st->stream));
                    ++st->launches;
                    g2m_c4::k_c4_base<<<grid_for(st, l1, 256), 256, 0, st->stream>>>(l1, rn, rb, re);
                    G2M_CUDA(cudaMemsetAsync(gctr, 0, 8, st->stream));
                    ++st->launches;
                    if (red) {
                        g2m_c4::k_c4_grid<true><<<st->sms * 4, 512, 0, st->stream>>>(nbr, l1, rn, rb, re, gctr,
                                                                                   dense, (u32)lo, count);
                        ++st->launches;
                        g2m_c4::k_c4_sweep<<<grid_for(st, (hi - lo) / 4 + 1, 256), 256, 0, st->stream>>>(
                            dense, hi - lo, count);
                        G2M_CUDA(cudaGetLastError());
                    } else {
                        g2m_c4::k_c4_grid<false><<<st->sms * 4, 512, 0, st->stream>>>(nbr, l1, rn, rb, re, gctr,
                                                                                    dense, (u32)lo, count);
                        G2M_CUDA(cudaGetLastError());
                        G2M_CUDA(cudaMemsetAsync(dense, 0, (size_t)(hi - lo) * 4, st->stream));
                    }
                }
            }
            return G2M_OK;
        }));
        if (dbg) fprintf(stderr, "[g2m] cycle4 grid tier: %llu sources, %llu range passes of <= %llu ids\n",
                         (unsigned long long)sizes[4], (unsigned long long)passes, (unsigned long long)range);
    }
    uint64_t h[2] = {0, 0};
    G2M_CUDA(cudaMemcpyAsync(h, count, 16, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaEventRecord(st->evs1, st->stream));
    G2M_CUDA(cudaEventSynchronize(st->evs1));
    counts[0] = h[0];
    counts[1] = h[1];
    S->tasks = sizes[1] + sizes[2] + sizes[3] + sizes[4];
    float dm = 0.f;
    cudaEventElapsedTime(&dm, st->evs0, st->evs1);
    S->device_ms = dm;
    S->launches = st->launches - l0;
    S->total_ms = ms_since(t0);
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// batched set operations (setops.py:35-84)
// ---------------------------------------------------------------------------

__global__ void k_setops(int op, u64 ncase, const u32* av, const u64* ao, const u32* bv, const u64* bo,
                         const i64* bounds, u64* out_n, u32* out_v) {
    const u32 lane = g2m_lane();
    for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c < ncase;
         c += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u32* a = av + ao[c];
        u32 na = (u32)(ao[c + 1] - ao[c]);
        const u32* b = bv + bo[c];
        u32 nb = (u32)(bo[c + 1] - bo[c]);
        const i64 bd = bounds[c];
        if (bd >= 0) {
            u32 y = bd > 0xffffffffll ? 0xffffffffu : (u32)bd;
            na = g2m_wlb(a, na, y);
            if (op < 2) nb = g2m_wlb(b, nb, y);   // bound_list on both for intersections
        }
        const u32 ex[1] = {G2M_NOBOUND};
        u32 n = 0;
        if (op == 0 || op == 1) {
            const u32* lp[2] = {a, b};
            u32 ln[2] = {na, nb};
            if (op == 0) n = g2m_materialize<2, 2>(lp, ln, nullptr, 0u, out_v + ao[c]);
            else n = g2m_count<2, 2, 1>(lp, ln, G2M_NOBOUND, ex, nullptr, 0u);
        } else {
            const u32* lp[2] = {a, b};
            u32 ln[2] = {na, nb};
            if (op == 2) n = g2m_materialize<1, 2>(lp, ln, nullptr, 0u, out_v + ao[c]);
            else n = g2m_count<1, 2, 1>(lp, ln, G2M_NOBOUND, ex, nullptr, 0u);
        }
        if (lane == 0) out_n[c] = n;
    }
}

extern "C" int g2m_setop_batch(int32_t device, int32_t op, uint64_t nc, const uint32_t* av,
                               const uint64_t* ao, const uint32_t* bv, const uint64_t* bo,
                               const int64_t* bounds, uint64_t* out_n, uint32_t* out_v) {
    if (op < 0 || op > 3) return fail(G2M_EUSAGE, "unknown set operation");
    if (nc == 0) return G2M_OK;
    DevState* st;
    G2M_TRY(dev_state(device, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(device));
    const uint64_t na = ao[nc], nb = bo[nc];
    DevBuf dav, dao, dbv, dbo, dbd, dn, dv;
    G2M_TRY(dav.ensure(std::max<uint64_t>(na, 1) * 4));
    G2M_TRY(dbv.ensure(std::max<uint64_t>(nb, 1) * 4));
    G2M_TRY(dao.ensure((nc + 1) * 8));
    G2M_TRY(dbo.ensure((nc + 1) * 8));
    G2M_TRY(dbd.ensure(nc * 8));
    G2M_TRY(dn.ensure(nc * 8));
    G2M_TRY(dv.ensure(std::max<uint64_t>(na, 1) * 4));
    if (na) G2M_CUDA(cudaMemcpyAsync(dav.p, av, na * 4, cudaMemcpyHostToDevice, st->stream));
    if (nb) G2M_CUDA(cudaMemcpyAsync(dbv.p, bv, nb * 4, cudaMemcpyHostToDevice, st->stream));
    G2M_CUDA(cudaMemcpyAsync(dao.p, ao, (nc + 1) * 8, cudaMemcpyHostToDevice, st->stream));
    G2M_CUDA(cudaMemcpyAsync(dbo.p, bo, (nc + 1) * 8, cudaMemcpyHostToDevice, st->stream));
    G2M_CUDA(cudaMemcpyAsync(dbd.p, bounds, nc * 8, cudaMemcpyHostToDevice, st->stream));
    k_setops<<<grid_for(st, nc * 32, 256), 256, 0, st->stream>>>(op, nc, dav.as<u32>(), dao.as<u64>(), dbv.as<u32>(),
                                                                 dbo.as<u64>(), dbd.as<i64>(), dn.as<u64>(), dv.as<u32>());
    G2M_CUDA(cudaGetLastError());
    G2M_CUDA(cudaMemcpyAsync(out_n, dn.p, nc * 8, cudaMemcpyDeviceToHost, st->stream));
    if (out_v && (op == 0 || op == 2) && na)
        G2M_CUDA(cudaMemcpyAsync(out_v, dv.p, na * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

// ---------------------------------------------------------------------------
// bounded-BFS frequent subgraph mining (fsm.py:107-210), device side; the
// level loop, canonical forms and the support / filter callbacks stay in
// Python (paper_2112_09761_b200/fsm.py)
// ---------------------------------------------------------------------------

struct g2m_fsm {
    const g2m_graph* g = nullptr;
    int l = 1;                       // edges per subgraph at this level
    u64 n = 0;                       // rows
    DevBuf ok;                       // allowed vertices (u8) or empty
    DevBuf redges, rverts, rnv;      // rows
    DevBuf par_off, par;             // per row: parent patterns (previous level's canonical ids)
    DevBuf rec, qid, first;          // quick records, quick id per row, first row per quick id
    u64 nq = 0;
    DevBuf canon, nmaps, map_off, maps;
    DevBuf dom;                      // unique domain keys
    u64 ndom = 0;
    DevBuf runs_cp, runs_n;          // (canon, position) runs of dom
    u64 nruns = 0;
    DevBuf pc;                       // unique parent -> child pairs
    u64 npc = 0;
};

static auto thrust_on(DevState* st) { return thrust::cuda::par.on(st->stream); }

static int fsm_alloc_rows(g2m_fsm* f, u64 n) {
    G2M_TRY(f->redges.ensure(std::max<u64>(n, 1) * g2m_fsmk::kFsmE * 8));
    G2M_TRY(f->rverts.ensure(std::max<u64>(n, 1) * g2m_fsmk::kFsmV * 4));
    G2M_TRY(f->rnv.ensure(std::max<u64>(n, 1)));
    G2M_TRY(f->par_off.ensure((n + 1) * 4));
    return G2M_OK;
}

extern "C" int g2m_fsm_create(const g2m_graph* g, const uint8_t* ok, g2m_fsm** out, uint64_t* nrows) {
    if (!g || !out || !nrows) return fail(G2M_EUSAGE, "null argument");
    if (!g->labels.p) return fail(G2M_EUSAGE, "frequent subgraph mining requires a labeled graph");
    DevState* st;
    G2M_TRY(dev_state(g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(g->dev));
    auto f = std::make_unique<g2m_fsm>();
    f->g = g;
    const u64 nv = g->nv;
    const unsigned char* okp = nullptr;
    if (ok) {
        G2M_TRY(f->ok.ensure(std::max<u64>(nv, 1)));
        if (nv) G2M_CUDA(cudaMemcpyAsync(f->ok.p, ok, nv, cudaMemcpyHostToDevice, st->stream));
        okp = f->ok.as<unsigned char>();
    }
    DevBuf cnt, pos;
    G2M_TRY(cnt.ensure(std::max<u64>(nv, 1) * 8));
    G2M_TRY(pos.ensure((nv + 1) * 8));
    if (nv) {
        ++st->launches;
        g2m_fsmk::k_fsm_l1_count<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(g->off.as<u64>(), g->nbr.as<u32>(), nv,
                                                                               okp, cnt.as<u64>());
        G2M_CUDA(cudaGetLastError());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), pos.as<u64>(), nv));
    u64 n = 0;
    G2M_CUDA(cudaMemcpyAsync(&n, pos.as<u64>() + nv, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    G2M_TRY(fsm_alloc_rows(f.get(), n));
    G2M_CUDA(cudaMemsetAsync(f->redges.p, 0, std::max<u64>(n, 1) * g2m_fsmk::kFsmE * 8, st->stream));
    G2M_CUDA(cudaMemsetAsync(f->rverts.p, 0, std::max<u64>(n, 1) * g2m_fsmk::kFsmV * 4, st->stream));
    G2M_CUDA(cudaMemsetAsync(f->par_off.p, 0, (n + 1) * 4, st->stream));
    if (nv) {
        ++st->launches;
        g2m_fsmk::k_fsm_l1_fill<<<grid_for(st, nv, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), nv, okp, pos.as<u64>(), f->redges.as<u64>(), f->rverts.as<u32>(),
            f->rnv.as<unsigned char>());
        G2M_CUDA(cudaGetLastError());
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    f->n = n;
    f->l = 1;
    *nrows = n;
    *out = f.release();
    return G2M_OK;
}

extern "C" int g2m_fsm_destroy(g2m_fsm* f) {
    if (!f) return G2M_OK;
    cudaSetDevice(f->g->dev);
    delete f;
    return G2M_OK;
}

extern "C" int g2m_fsm_rows(const g2m_fsm* f, uint64_t* edges, uint32_t* verts, uint8_t* nverts) {
    if (!f) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    if (f->n) {
        if (edges) G2M_CUDA(cudaMemcpyAsync(edges, f->redges.p, f->n * g2m_fsmk::kFsmE * 8, cudaMemcpyDeviceToHost, st->stream));
        if (verts) G2M_CUDA(cudaMemcpyAsync(verts, f->rverts.p, f->n * g2m_fsmk::kFsmV * 4, cudaMemcpyDeviceToHost, st->stream));
        if (nverts) G2M_CUDA(cudaMemcpyAsync(nverts, f->rnv.p, f->n, cudaMemcpyDeviceToHost, st->stream));
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

__global__ void k_fsm_compact(const u64* redges, const u32* rverts, const unsigned char* rnv, const u32* par_off,
                              const u32* par, const unsigned char* keep, const u64* pos, const u64* ppos, u64 n,
                              u64* oe, u32* ov, unsigned char* onv, u32* opoff, u32* opar) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        if (!keep[r]) continue;
        const u64 p = pos[r];
        for (int t = 0; t < g2m_fsmk::kFsmE; ++t) oe[p * g2m_fsmk::kFsmE + t] = redges[r * g2m_fsmk::kFsmE + t];
        for (int t = 0; t < g2m_fsmk::kFsmV; ++t) ov[p * g2m_fsmk::kFsmV + t] = rverts[r * g2m_fsmk::kFsmV + t];
        onv[p] = rnv[r];
        u64 q = ppos[r];
        opoff[p] = (u32)q;
        for (u32 j = par_off[r]; j < par_off[r + 1]; ++j) opar[q++] = par[j];
    }
}

// keep the rows with keep[r] != 0 (the subgraph_filter hook, fsm.py:140-146, 196-197)
extern "C" int g2m_fsm_keep(g2m_fsm* f, const uint8_t* keep, uint64_t* nrows) {
    if (!f || !keep || !nrows) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    const u64 n = f->n;
    std::vector<uint32_t> hpo(n + 1, 0);
    if (n) G2M_CUDA(cudaMemcpyAsync(hpo.data(), f->par_off.p, (n + 1) * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    std::vector<uint64_t> pos(n + 1, 0), ppos(n + 1, 0);
    for (u64 r = 0; r < n; ++r) {
        pos[r + 1] = pos[r] + (keep[r] ? 1 : 0);
        ppos[r + 1] = ppos[r] + (keep[r] ? (hpo[r + 1] - hpo[r]) : 0);
    }
    const u64 m = pos[n];
    DevBuf dk, dpos, dppos;
    G2M_TRY(dk.ensure(std::max<u64>(n, 1)));
    G2M_TRY(dpos.ensure((n + 1) * 8));
    G2M_TRY(dppos.ensure((n + 1) * 8));
    if (n) {
        G2M_CUDA(cudaMemcpyAsync(dk.p, keep, n, cudaMemcpyHostToDevice, st->stream));
        G2M_CUDA(cudaMemcpyAsync(dpos.p, pos.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st->stream));
        G2M_CUDA(cudaMemcpyAsync(dppos.p, ppos.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st->stream));
    }
    auto o = std::make_unique<g2m_fsm>();
    G2M_TRY(fsm_alloc_rows(o.get(), m));
    G2M_CUDA(cudaMemsetAsync(o->redges.p, 0, std::max<u64>(m, 1) * g2m_fsmk::kFsmE * 8, st->stream));
    G2M_TRY(o->par.ensure(std::max<u64>(ppos[n], 1) * 4));
    if (n) {
        ++st->launches;
        k_fsm_compact<<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            f->redges.as<u64>(), f->rverts.as<u32>(), f->rnv.as<unsigned char>(), f->par_off.as<u32>(),
            f->par.p ? f->par.as<u32>() : nullptr, dk.as<unsigned char>(), dpos.as<u64>(), dppos.as<u64>(), n,
            o->redges.as<u64>(), o->rverts.as<u32>(), o->rnv.as<unsigned char>(), o->par_off.as<u32>(),
            o->par.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    const uint32_t tail = (uint32_t)ppos[n];
    G2M_CUDA(cudaMemcpyAsync(o->par_off.as<u32>() + m, &tail, 4, cudaMemcpyHostToDevice, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    f->redges.swap_with(o->redges);
    f->rverts.swap_with(o->rverts);
    f->rnv.swap_with(o->rnv);
    f->par_off.swap_with(o->par_off);
    f->par.swap_with(o->par);
    f->n = m;
    *nrows = m;
    return G2M_OK;
}

// group the rows by quick pattern (fsm.py:40-47); *nq distinct quick patterns
extern "C" int g2m_fsm_quick(g2m_fsm* f, uint64_t* nq) {
    if (!f || !nq) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    const u64 n = f->n;
    G2M_TRY(f->rec.ensure(std::max<u64>(n, 1) * g2m_fsmk::kRec * 4));
    G2M_TRY(f->qid.ensure(std::max<u64>(n, 1) * 4));
    DevBuf hash, rows, head, grp, err;
    G2M_TRY(hash.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(rows.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(head.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(grp.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(err.ensure(4));
    G2M_CUDA(cudaMemsetAsync(err.p, 0, 4, st->stream));
    u64 groups = 0;
    if (n) {
        ++st->launches;
        g2m_fsmk::k_fsm_quick<<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            f->redges.as<u64>(), f->rverts.as<u32>(), f->rnv.as<unsigned char>(), n, f->l, f->g->labels.as<u32>(),
            f->rec.as<u32>(), hash.as<u64>(), rows.as<u64>());
        G2M_CUDA(cudaGetLastError());
        auto pol = thrust_on(st);
        u64* hp = hash.as<u64>();
        u64* rp = rows.as<u64>();
        thrust::sort_by_key(pol, hp, hp + n, rp);
        u64* hd = head.as<u64>();
        thrust::transform(pol, thrust::counting_iterator<u64>(0), thrust::counting_iterator<u64>(n), hd,
                          [hp] __device__(u64 i) -> u64 { return (i == 0 || hp[i] != hp[i - 1]) ? 1ull : 0ull; });
        u64* gp = grp.as<u64>();
        thrust::inclusive_scan(pol, hd, hd + n, gp);
        G2M_CUDA(cudaMemcpyAsync(&groups, gp + n - 1, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        G2M_TRY(f->first.ensure(std::max<u64>(groups, 1) * 8));
        u64* fp = f->first.as<u64>();
        u32* qp = f->qid.as<u32>();
        thrust::for_each(pol, thrust::counting_iterator<u64>(0), thrust::counting_iterator<u64>(n),
                         [=] __device__(u64 i) {
                             const u64 g = gp[i] - 1;
                             qp[rp[i]] = (u32)g;
                             if (hd[i]) fp[g] = rp[i];
                         });
        ++st->launches;
        g2m_fsmk::k_fsm_check<<<grid_for(st, n, 256), 256, 0, st->stream>>>(rp, n, f->rec.as<u32>(), fp, qp,
                                                                            err.as<u32>());
        G2M_CUDA(cudaGetLastError());
    }
    uint32_t e = 0;
    G2M_CUDA(cudaMemcpyAsync(&e, err.p, 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    if (e) return fail(G2M_ECUDA, "quick-pattern hash collision");
    f->nq = groups;
    *nq = groups;
    return G2M_OK;
}

__global__ void k_fsm_gather_rec(const u32* rec, const u64* first, u64 nq, u32* out) {
    for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < nq; q += (u64)gridDim.x * blockDim.x)
        for (int w = 0; w < g2m_fsmk::kRec; ++w) out[q * g2m_fsmk::kRec + w] = rec[first[q] * g2m_fsmk::kRec + w];
}

// the quick record of every group (12 u32 each: k | l << 8, labels[8], position pairs u64)
extern "C" int g2m_fsm_quick_records(const g2m_fsm* f, uint32_t* out) {
    if (!f || !out) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    if (!f->nq) return G2M_OK;
    DevBuf tmp;
    G2M_TRY(tmp.ensure(f->nq * g2m_fsmk::kRec * 4));
    ++st->launches;
    k_fsm_gather_rec<<<grid_for(st, f->nq, 256), 256, 0, st->stream>>>(f->rec.as<u32>(), f->first.as<u64>(), f->nq,
                                                                         tmp.as<u32>());
    G2M_CUDA(cudaMemcpyAsync(out, tmp.p, f->nq * g2m_fsmk::kRec * 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

// domains (fsm.py:158-166): canonical id and position maps per quick pattern
// from the host; unique (canon, position, vertex) keys, their (canon, position)
// run lengths (domain sizes), and the parent -> child pattern pairs
extern "C" int g2m_fsm_domains(g2m_fsm* f, const uint32_t* canon, const uint32_t* nmaps, const uint32_t* map_off,
                               const uint8_t* maps, uint64_t maps_bytes, uint64_t* ndom, uint64_t* nruns,
                               uint64_t* npc) {
    if (!f || !canon || !nmaps || !map_off || !ndom || !nruns || !npc) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    const u64 n = f->n, nq = f->nq;
    G2M_TRY(f->canon.ensure(std::max<u64>(nq, 1) * 4));
    G2M_TRY(f->nmaps.ensure(std::max<u64>(nq, 1) * 4));
    G2M_TRY(f->map_off.ensure(std::max<u64>(nq, 1) * 4));
    G2M_TRY(f->maps.ensure(std::max<u64>(maps_bytes, 1)));
    if (nq) {
        G2M_CUDA(cudaMemcpyAsync(f->canon.p, canon, nq * 4, cudaMemcpyHostToDevice, st->stream));
        G2M_CUDA(cudaMemcpyAsync(f->nmaps.p, nmaps, nq * 4, cudaMemcpyHostToDevice, st->stream));
        G2M_CUDA(cudaMemcpyAsync(f->map_off.p, map_off, nq * 4, cudaMemcpyHostToDevice, st->stream));
    }
    if (maps_bytes) G2M_CUDA(cudaMemcpyAsync(f->maps.p, maps, maps_bytes, cudaMemcpyHostToDevice, st->stream));
    DevBuf cnt, pos;
    G2M_TRY(cnt.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(pos.ensure((n + 1) * 8));
    if (n) {
        ++st->launches;
        g2m_fsmk::k_fsm_dom_count<<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            f->qid.as<u32>(), f->nmaps.as<u32>(), f->rnv.as<unsigned char>(), n, cnt.as<u64>());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), pos.as<u64>(), n));
    u64 nk = 0;
    G2M_CUDA(cudaMemcpyAsync(&nk, pos.as<u64>() + n, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    G2M_TRY(f->dom.ensure(std::max<u64>(nk, 1) * 8));
    auto pol = thrust_on(st);
    u64 nu = 0;
    if (n) {
        ++st->launches;
        g2m_fsmk::k_fsm_dom_fill<<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            f->qid.as<u32>(), f->canon.as<u32>(), f->nmaps.as<u32>(), f->map_off.as<u32>(),
            f->maps.as<unsigned char>(), f->rverts.as<u32>(), f->rnv.as<unsigned char>(), n, pos.as<u64>(),
            f->dom.as<u64>());
        G2M_CUDA(cudaGetLastError());
        u64* dp = f->dom.as<u64>();
        thrust::sort(pol, dp, dp + nk);
        nu = (u64)(thrust::unique(pol, dp, dp + nk) - dp);
    }
    // runs of (canon, position) = key >> 32
    G2M_TRY(f->runs_cp.ensure(std::max<u64>(nu, 1) * 8));
    G2M_TRY(f->runs_n.ensure(std::max<u64>(nu, 1) * 8));
    u64 nr = 0;
    if (nu) {
        u64* dp = f->dom.as<u64>();
        auto hi = thrust::make_transform_iterator(dp, [] __device__(u64 k) -> u64 { return k >> 32; });
        auto ends = thrust::reduce_by_key(pol, hi, hi + nu, thrust::constant_iterator<u64>(1), f->runs_cp.as<u64>(),
                                          f->runs_n.as<u64>());
        nr = (u64)(ends.first - f->runs_cp.as<u64>());
    }
    // parent -> child pairs
    uint32_t npar = 0;
    if (n) G2M_CUDA(cudaMemcpyAsync(&npar, f->par_off.as<u32>() + n, 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    G2M_TRY(f->pc.ensure(std::max<u64>(npar, 1) * 8));
    u64 np = 0;
    if (npar) {
        ++st->launches;
        g2m_fsmk::k_fsm_pc<<<grid_for(st, n, 256), 256, 0, st->stream>>>(f->qid.as<u32>(), f->canon.as<u32>(),
                                                                          f->par_off.as<u32>(), f->par.as<u32>(), n,
                                                                          f->pc.as<u64>());
        G2M_CUDA(cudaGetLastError());
        u64* pp = f->pc.as<u64>();
        thrust::sort(pol, pp, pp + npar);
        np = (u64)(thrust::unique(pol, pp, pp + npar) - pp);
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    f->ndom = nu;
    f->nruns = nr;
    f->npc = np;
    *ndom = nu;
    *nruns = nr;
    *npc = np;
    return G2M_OK;
}

// copies: run keys (canon << 4 | position) and lengths, unique domain keys,
// parent -> child pairs (parent << 32 | child); any pointer may be null
extern "C" int g2m_fsm_results(const g2m_fsm* f, uint64_t* run_keys, uint64_t* run_len, uint64_t* dom_keys,
                               uint64_t* pc_pairs) {
    if (!f) return fail(G2M_EUSAGE, "null argument");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    if (run_keys && f->nruns) G2M_CUDA(cudaMemcpyAsync(run_keys, f->runs_cp.p, f->nruns * 8, cudaMemcpyDeviceToHost, st->stream));
    if (run_len && f->nruns) G2M_CUDA(cudaMemcpyAsync(run_len, f->runs_n.p, f->nruns * 8, cudaMemcpyDeviceToHost, st->stream));
    if (dom_keys && f->ndom) G2M_CUDA(cudaMemcpyAsync(dom_keys, f->dom.p, f->ndom * 8, cudaMemcpyDeviceToHost, st->stream));
    if (pc_pairs && f->npc) G2M_CUDA(cudaMemcpyAsync(pc_pairs, f->pc.p, f->npc * 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    return G2M_OK;
}

// next level (fsm.py:178-203): rows of the patterns with kept[canon] != 0 grow
// one edge; new edge sets deduplicated, each with its parent patterns
extern "C" int g2m_fsm_extend(g2m_fsm* f, const uint8_t* kept, uint32_t ncanon, uint64_t* nrows) {
    if (!f || !kept || !nrows) return fail(G2M_EUSAGE, "null argument");
    if (f->l + 1 > g2m_fsmk::kFsmE) return fail(G2M_EUSAGE, "max_edges beyond 7 is not supported");
    DevState* st;
    G2M_TRY(dev_state(f->g->dev, &st));
    std::lock_guard<std::mutex> lk(st->mu);
    G2M_CUDA(cudaSetDevice(f->g->dev));
    const u64 n = f->n;
    const int l = f->l;
    DevBuf dk, cnt, pos;
    G2M_TRY(dk.ensure(std::max<u32>(ncanon, 1)));
    if (ncanon) G2M_CUDA(cudaMemcpyAsync(dk.p, kept, ncanon, cudaMemcpyHostToDevice, st->stream));
    G2M_TRY(cnt.ensure(std::max<u64>(n, 1) * 8));
    G2M_TRY(pos.ensure((n + 1) * 8));
    const unsigned char* okp = f->ok.p ? f->ok.as<unsigned char>() : nullptr;
    const g2m_graph* g = f->g;
    if (n) {
        ++st->launches;
        g2m_fsmk::k_fsm_extend<false><<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), okp, f->redges.as<u64>(), f->rverts.as<u32>(),
            f->rnv.as<unsigned char>(), f->qid.as<u32>(), f->canon.as<u32>(), dk.as<unsigned char>(), n, l,
            cnt.as<u64>(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
        G2M_CUDA(cudaGetLastError());
    }
    G2M_TRY(exclusive_scan_u64(st, cnt.as<u64>(), pos.as<u64>(), n));
    u64 m = 0;
    G2M_CUDA(cudaMemcpyAsync(&m, pos.as<u64>() + n, 8, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    DevBuf ce, cv, cnv, cpar, ch, cid, head, grp, gp, err;
    G2M_TRY(ce.ensure(std::max<u64>(m, 1) * g2m_fsmk::kFsmE * 8));
    G2M_TRY(cv.ensure(std::max<u64>(m, 1) * g2m_fsmk::kFsmV * 4));
    G2M_TRY(cnv.ensure(std::max<u64>(m, 1)));
    G2M_TRY(cpar.ensure(std::max<u64>(m, 1) * 4));
    G2M_TRY(ch.ensure(std::max<u64>(m, 1) * 8));
    G2M_TRY(cid.ensure(std::max<u64>(m, 1) * 8));
    G2M_TRY(head.ensure(std::max<u64>(m, 1) * 4));
    G2M_TRY(grp.ensure(std::max<u64>(m, 1) * 8));
    G2M_TRY(gp.ensure(std::max<u64>(m, 1) * 8));
    G2M_TRY(err.ensure(4));
    G2M_CUDA(cudaMemsetAsync(err.p, 0, 4, st->stream));
    G2M_CUDA(cudaMemsetAsync(ce.p, 0, std::max<u64>(m, 1) * g2m_fsmk::kFsmE * 8, st->stream));
    G2M_CUDA(cudaMemsetAsync(cv.p, 0, std::max<u64>(m, 1) * g2m_fsmk::kFsmV * 4, st->stream));
    u64 groups = 0;
    auto pol = thrust_on(st);
    if (m) {
        ++st->launches;
        g2m_fsmk::k_fsm_extend<true><<<grid_for(st, n, 256), 256, 0, st->stream>>>(
            g->off.as<u64>(), g->nbr.as<u32>(), okp, f->redges.as<u64>(), f->rverts.as<u32>(),
            f->rnv.as<unsigned char>(), f->qid.as<u32>(), f->canon.as<u32>(), dk.as<unsigned char>(), n, l, nullptr,
            pos.as<u64>(), ce.as<u64>(), cv.as<u32>(), cnv.as<unsigned char>(), cpar.as<u32>(), ch.as<u64>(),
            cid.as<u64>());
        G2M_CUDA(cudaGetLastError());
        // sort by (hash, then edge words) so equal edge sets are adjacent
        u64* hp = ch.as<u64>();
        u64* ip = cid.as<u64>();
        thrust::sort_by_key(pol, hp, hp + m, ip);
        ++st->launches;
        g2m_fsmk::k_fsm_cand_heads<<<grid_for(st, m, 256), 256, 0, st->stream>>>(hp, ip, m, ce.as<u64>(), l,
                                                                                 head.as<u32>(), err.as<u32>());
        G2M_CUDA(cudaGetLastError());
        u32* hd = head.as<u32>();
        u64* gg = grp.as<u64>();
        thrust::transform(pol, hd, hd + m, gg, [] __device__(u32 h) -> u64 { return (u64)h; });
        thrust::inclusive_scan(pol, gg, gg + m, gg);
        G2M_CUDA(cudaMemcpyAsync(&groups, gg + m - 1, 8, cudaMemcpyDeviceToHost, st->stream));
        G2M_CUDA(cudaStreamSynchronize(st->stream));
        thrust::transform(pol, gg, gg + m, gg, [] __device__(u64 x) -> u64 { return x - 1; });
    }
    uint32_t e = 0;
    G2M_CUDA(cudaMemcpyAsync(&e, err.p, 4, cudaMemcpyDeviceToHost, st->stream));
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    if (e) return fail(G2M_ECUDA, "subgraph edge-set hash collision");
    auto o = std::make_unique<g2m_fsm>();
    G2M_TRY(fsm_alloc_rows(o.get(), groups));
    G2M_CUDA(cudaMemsetAsync(o->redges.p, 0, std::max<u64>(groups, 1) * g2m_fsmk::kFsmE * 8, st->stream));
    G2M_CUDA(cudaMemsetAsync(o->rverts.p, 0, std::max<u64>(groups, 1) * g2m_fsmk::kFsmV * 4, st->stream));
    u64 npairs = 0;
    if (m) {
        ++st->launches;
        g2m_fsmk::k_fsm_next<<<grid_for(st, m, 256), 256, 0, st->stream>>>(
            cid.as<u64>(), grp.as<u64>(), m, head.as<u32>(), ce.as<u64>(), cv.as<u32>(), cnv.as<unsigned char>(),
            cpar.as<u32>(), o->redges.as<u64>(), o->rverts.as<u32>(), o->rnv.as<unsigned char>(), gp.as<u64>());
        G2M_CUDA(cudaGetLastError());
        u64* pp = gp.as<u64>();
        thrust::sort(pol, pp, pp + m);
        npairs = (u64)(thrust::unique(pol, pp, pp + m) - pp);
    }
    // parents per new row: counts of (group, parent) pairs per group -> offsets
    G2M_TRY(o->par.ensure(std::max<u64>(npairs, 1) * 4));
    DevBuf pcnt;
    G2M_TRY(pcnt.ensure(std::max<u64>(groups, 1) * 4));
    G2M_CUDA(cudaMemsetAsync(pcnt.p, 0, std::max<u64>(groups, 1) * 4, st->stream));
    G2M_CUDA(cudaMemsetAsync(o->par_off.p, 0, (groups + 1) * 4, st->stream));
    if (npairs) {
        u64* pp = gp.as<u64>();
        u32* pc = pcnt.as<u32>();
        u32* pr = o->par.as<u32>();
        thrust::for_each(pol, thrust::counting_iterator<u64>(0), thrust::counting_iterator<u64>(npairs),
                         [=] __device__(u64 i) {
                             atomicAdd(pc + (pp[i] >> 32), 1u);
                             pr[i] = (u32)pp[i];
                         });
        thrust::exclusive_scan(pol, pc, pc + groups, o->par_off.as<u32>());
        const uint32_t tail = (uint32_t)npairs;
        G2M_CUDA(cudaMemcpyAsync(o->par_off.as<u32>() + groups, &tail, 4, cudaMemcpyHostToDevice, st->stream));
    }
    G2M_CUDA(cudaStreamSynchronize(st->stream));
    f->redges.swap_with(o->redges);
    f->rverts.swap_with(o->rverts);
    f->rnv.swap_with(o->rnv);
    f->par_off.swap_with(o->par_off);
    f->par.swap_with(o->par);
    f->n = groups;
    f->l = l + 1;
    f->nq = 0;
    *nrows = groups;
    return G2M_OK;
}
