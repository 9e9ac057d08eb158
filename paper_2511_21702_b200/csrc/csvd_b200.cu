// csvd_b200: C ABI (include/csvd_b200.h) over the B200 step kernel (kernels.cuh).
//
// One step = one CUDA-graph replay of [H2D config (+h)] -> k_step (persistent,
// cooperative) [-> D2H result].  All control flow (waves, fallback chain,
// full-vocabulary fallback) is decided on the device inside k_step.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/csvd_b200.h"
#include "headstep.cuh"

// permute rows on device: dst[pos] = src[perm[pos]]
__global__ void k_permute_rows(const char *src, char *dst, const long long *perm, long long V, long long row_bytes) {
    for (long long pos = blockIdx.x; pos < V; pos += gridDim.x) {
        const char *s = src + perm[pos] * row_bytes;
        char *t = dst + pos * row_bytes;
        if ((row_bytes & 15) == 0) {  // 16-byte rows: vector copies
            for (long long b = threadIdx.x * 16; b < row_bytes; b += blockDim.x * 16)
                *reinterpret_cast<uint4 *>(t + b) = *reinterpret_cast<const uint4 *>(s + b);
        } else if ((row_bytes & 3) == 0) {  // odd d: rows are only 4-byte aligned
            for (long long b = threadIdx.x * 4; b < row_bytes; b += blockDim.x * 4)
                *reinterpret_cast<unsigned *>(t + b) = *reinterpret_cast<const unsigned *>(s + b);
        } else {
            for (long long b = threadIdx.x; b < row_bytes; b += blockDim.x) t[b] = s[b];
        }
    }
}

// L2 flush for benchmarking: stream-read a buffer larger than L2 (clean
// lines: nothing to write back when the next step allocates)
__global__ void k_l2_flush(const uint4 *buf, size_t n, unsigned *sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;  // keep the loads alive
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef void (*kern_t)(Dev);

// A batch lane: one query's step running on its own slice of the GPU (a
// cooperative grid of ~148/B CTAs) concurrently with the other lanes.  Lanes
// share every read-only table / index buffer (W rows and centroids are read
// through the shared L2) and own their per-step workspaces.
struct Lane {
    Dev D{};
    Dev Dh{};  // the same lane publishing into mapped host memory (host-API batches)
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
};

struct csvd_ctx {
    int device = 0;
    Dev D{};
    std::string err;
    cudaStream_t stream = nullptr;
    std::vector<void *> dev_allocs;
    void *k_buffers[4] = {};  // K-dependent: dense candidate lists, cluster top-k summaries
    kern_t kern = nullptr;
    kern_t kdense = nullptr;  // standalone full-vocabulary GEMV (regular plans)
    int dense_grid = 0;
    size_t dense_smem = 0;
    int grid = 0;
    int grid_cap = 0;  // the grid the K-dependent buffers were sized for
    int nsm = 0;
    size_t smem = 0;
    csvd_config *d_cfg = nullptr;
    double *d_h = nullptr;
    double *h_pin = nullptr;
    double *h_map = nullptr;  // mapped pinned query: the host-API head graph reads it in place (zero-copy)
    bool h_zero_copy = false;
    // pinned staging configs, one per kind of graph that reads one at execution
    // time (step/shard: cfg_pin; batch: cfg_pin_b; dense/bounds: cfg_pin_fixed)
    csvd_config *cfg_pin = nullptr, *cfg_pin_b = nullptr, *cfg_pin_fixed = nullptr;
    csvd_config cfg_dev{};   // the config currently resident in d_cfg
    bool cfg_valid = false;
    csvd_result *res_pin = nullptr;
    long long *ids_pin = nullptr;
    double *logits_pin = nullptr;
    cudaGraphExec_t g_step = nullptr, g_host = nullptr, g_bounds = nullptr, g_dense = nullptr;
    // head step (headstep.cuh): [h2d] -> k_head -> IF(undecided) k_step
    void (*khead)(Dev) = nullptr;
    cudaGraphExec_t g_step_head = nullptr, g_host_head = nullptr;
    // the device head graph reads h where the caller keeps it: its kernel
    // node's Dev.h is updated in the executable graph (a host-side call) when
    // the caller's pointer changes, instead of a device-to-device copy node
    cudaGraph_t g_step_head_src = nullptr;
    cudaGraphNode_t g_step_head_node = nullptr;
    const double *g_step_head_h = nullptr;
    // zero-copy host results (csvd_step_host): mapped pinned buffers + flag
    csvd_result *res_map = nullptr;
    long long *ids_map = nullptr;
    double *logits_map = nullptr;
    Dev Dhost{};
    int direct = 0;
    void *flush_buf = nullptr;
    int64_t first_chunk = 0;
    std::vector<int2> wleaves, bleaves;
    std::vector<short> wprog, bprog;
    // shard contexts
    bool shard = false;
    std::vector<uint8_t> owned;      // [C]
    std::vector<int> order_h, cum_h;  // staging for csvd_shard_open
    std::vector<long long> sids_h;
    std::vector<double> slog_h, sum_h;
    std::vector<long long> local_tokens;  // owned token ids, ascending
    // batch lanes (decode_step over a batch of queries)
    std::vector<Lane> lanes;
    std::vector<void *> lane_allocs;
    int lane_grid = 0, lane_K = 0;
    double *d_H = nullptr;                 // [lanes, d]
    csvd_result *d_res_all = nullptr;      // [lanes]
    double *H_pin = nullptr;
    csvd_result *res_pin_b = nullptr;
    long long *ids_pin_b = nullptr;
    double *logits_pin_b = nullptr;
    cudaEvent_t fork = nullptr;
    double **d_Uraw_l = nullptr, **d_dots_l = nullptr;  // [lanes] per-lane bound outputs
    kern_t kgroup = nullptr;                      // grouped lanes kernel (one launch per batch)
    kern_t kgroup_head = nullptr;                 // grouped head-step lanes (head-eligible configs)
    LaneWS *d_lanes = nullptr, *d_lanes_host = nullptr;
    void (*kbb)(Dev, const double *, int, double *const *, double *const *, csvd_result *, int) = nullptr;
    size_t kbb_smem = 0;
    int kbb_gq = 0;
    bool kbb2 = false;  // k_bbatch (chain-per-lane batched dots) instead of k_bounds_batch
    int kbb2_kq = 0;
    size_t kbb2_smem = 0;
    cudaGraphExec_t g_batch = nullptr;
    int g_batch_B = 0, g_batch_host = 0, g_batch_head = 0;
    int last_launches = 0;  // kernels launched by the last entry point (csvd_last_launches)
    csvd_result *res_map_b = nullptr;  // [lanes] mapped
    long long *ids_map_b = nullptr;    // [lanes, V] mapped
    double *logits_map_b = nullptr;    // [lanes, V] mapped
};

static int fail(csvd_ctx *c, int code, const std::string &msg) {
    if (c) c->err = msg;
    return code;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(ctx, CSVD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

// numpy pairwise tree enumeration (oracle/pairwise.c restatement)
static void pw_enumerate(int off, int n, std::vector<int2> &leaves, std::vector<short> &prog, bool &balanced) {
    if (n <= 128) {
        prog.push_back((short)leaves.size());
        leaves.push_back(make_int2(off, n));
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    if (n2 * 2 != n) balanced = false;
    pw_enumerate(off, n2, leaves, prog, balanced);
    pw_enumerate(off + n2, n - n2, leaves, prog, balanced);
    prog.push_back(-1);
}

static void make_plan(int n, PwPlan &pl, std::vector<int2> &leaves, std::vector<short> &prog) {
    memset(&pl, 0, sizeof(pl));
    pl.n = n;
    leaves.clear();
    prog.clear();
    bool balanced = true;
    pw_enumerate(0, n, leaves, prog, balanced);
    const int nl = (int)leaves.size();
    const int L = leaves[0].y;
    bool equal = true;
    for (auto &lf : leaves) equal = equal && (lf.y == L);
    const bool pow2 = (nl & (nl - 1)) == 0;
    if (balanced && equal && pow2 && L % 8 == 0 && L >= 8 && nl >= 4 && nl <= 128) {
        pl.regular = 1;
        pl.leaf_len = L;
        pl.steps = L / 8;
        if (nl >= 32) {
            pl.cpl = 8;
            pl.q = nl / 32;
        } else {
            pl.cpl = 8 / (32 / nl);
            pl.q = 1;
        }
    }
    pl.nleaf = nl;
    pl.nprog = (int)prog.size();
}

template <typename T>
static int dalloc(csvd_ctx *ctx, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
    if (e != cudaSuccess) return fail(ctx, CSVD_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ctx->dev_allocs.push_back(q);
    *p = reinterpret_cast<T *>(q);
    return 0;
}

template <typename T>
static int dupload(csvd_ctx *ctx, T **p, const T *src, size_t count) {
    int rc = dalloc(ctx, p, count);
    if (rc) return rc;
    CK(cudaMemcpy(*p, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return 0;
}

// --- kernel instantiation per (weight dtype, W plan, bounds plan) ----------
// (instantiated in kinst.cu, one translation unit per dtype / plan)
#define CSVD_EXTERN_K(ET, CPL, Q)                                  \
    extern template __global__ void k_step<ET, CPL, Q, CPL, Q>(const __grid_constant__ Dev); \
    extern template __global__ void k_step<ET, CPL, Q, 0, 0>(const __grid_constant__ Dev);   \
    extern template __global__ void k_dense_gemv<ET, CPL, Q>(const __grid_constant__ Dev);   \
    extern template __global__ void k_step<ET, CPL, Q, CPL, Q, true>(const __grid_constant__ Dev);
#define CSVD_EXTERN_ET(ET) \
    CSVD_EXTERN_K(ET, 8, 1) CSVD_EXTERN_K(ET, 8, 2) CSVD_EXTERN_K(ET, 8, 4) \
    CSVD_EXTERN_K(ET, 4, 1) CSVD_EXTERN_K(ET, 2, 1) CSVD_EXTERN_K(ET, 1, 1)
CSVD_EXTERN_ET(float)
CSVD_EXTERN_ET(uint16_t)
#define CSVD_EXTERN_HEADL(ET) \
    extern template __global__ void k_head_lanes<ET, 1>(const __grid_constant__ Dev); \
    extern template __global__ void k_head_lanes<ET, 2>(const __grid_constant__ Dev); \
    extern template __global__ void k_head_lanes<ET, 4>(const __grid_constant__ Dev);
CSVD_EXTERN_HEADL(float)
CSVD_EXTERN_HEADL(uint16_t)
#define CSVD_EXTERN_HEAD(ET) \
    extern template __global__ void k_head<ET, 1>(const __grid_constant__ Dev); \
    extern template __global__ void k_head<ET, 2>(const __grid_constant__ Dev); \
    extern template __global__ void k_head<ET, 4>(const __grid_constant__ Dev);
CSVD_EXTERN_HEAD(float)
CSVD_EXTERN_HEAD(uint16_t)
typedef void (*khead_t)(Dev);
template <typename ET>
static khead_t pick_head_t(const PwPlan &wp) {
    switch (wp.q) {
        case 1: return k_head<ET, 1>;
        case 2: return k_head<ET, 2>;
        default: return k_head<ET, 4>;
    }
}
// the head step needs a regular 8-chain plan shared by W rows and centroids
// (every d = 32 * 2^m * L with L % 8 == 0; not bias-augmented d + 1)
static khead_t pick_head(const Dev &D) {
    if (getenv("CSVD_NO_HEAD")) return nullptr;
    if (!D.wplan.regular || D.wplan.cpl != 8 || D.wplan.n != D.bplan.n || D.mode == CSVD_MODE_BIAS_AUGMENTED)
        return nullptr;
    return D.wdtype == CSVD_W_BF16 ? pick_head_t<uint16_t>(D.wplan) : pick_head_t<float>(D.wplan);
}
template <typename ET>
static kern_t pick_head_lanes_t(const PwPlan &wp) {
    switch (wp.q) {
        case 1: return k_head_lanes<ET, 1>;
        case 2: return k_head_lanes<ET, 2>;
        default: return k_head_lanes<ET, 4>;
    }
}
static kern_t pick_head_lanes(const Dev &D) {
    if (getenv("CSVD_NO_HEAD") || getenv("CSVD_NO_HEAD_LANES")) return nullptr;
    if (!D.wplan.regular || D.wplan.cpl != 8 || D.wplan.n != D.bplan.n || D.mode == CSVD_MODE_BIAS_AUGMENTED)
        return nullptr;
    return D.wdtype == CSVD_W_BF16 ? pick_head_lanes_t<uint16_t>(D.wplan) : pick_head_lanes_t<float>(D.wplan);
}
// configs the head step can decide (everything else goes straight to k_step)
static bool head_config(const csvd_config *cfg) {
    return cfg->variant == CSVD_VARIANT_INCREMENTAL && cfg->first_wave_tokens <= 0 && cfg->k <= KH;
}
extern template __global__ void k_step<float, 0, 0, 0, 0>(const __grid_constant__ Dev);
extern template __global__ void k_step<uint16_t, 0, 0, 0, 0>(const __grid_constant__ Dev);
template <typename ET, int CPL, int Q>
static kern_t pick_b(bool same) {
    if (same) return k_step<ET, CPL, Q, CPL, Q>;
    return k_step<ET, CPL, Q, 0, 0>;  // separate bounds plan: generic (bias-augmented d+1)
}
template <typename ET>
static kern_t pick_w(const PwPlan &wp, const PwPlan &bp) {
    const bool same = (wp.n == bp.n);
    if (!wp.regular) return k_step<ET, 0, 0, 0, 0>;
    switch (wp.cpl * 8 + wp.q) {
        case 8 * 8 + 1: return pick_b<ET, 8, 1>(same);
        case 8 * 8 + 2: return pick_b<ET, 8, 2>(same);
        case 8 * 8 + 4: return pick_b<ET, 8, 4>(same);
        case 4 * 8 + 1: return pick_b<ET, 4, 1>(same);
        case 2 * 8 + 1: return pick_b<ET, 2, 1>(same);
        default: return pick_b<ET, 1, 1>(same);
    }
}
template <typename ET>
static kern_t pick_dense_t(const PwPlan &wp) {
    if (!wp.regular) return nullptr;
    switch (wp.cpl * 8 + wp.q) {
        case 8 * 8 + 1: return k_dense_gemv<ET, 8, 1>;
        case 8 * 8 + 2: return k_dense_gemv<ET, 8, 2>;
        case 8 * 8 + 4: return k_dense_gemv<ET, 8, 4>;
        case 4 * 8 + 1: return k_dense_gemv<ET, 4, 1>;
        case 2 * 8 + 1: return k_dense_gemv<ET, 2, 1>;
        default: return k_dense_gemv<ET, 1, 1>;
    }
}
static kern_t pick_dense(const Dev &D) {
    return D.wdtype == CSVD_W_BF16 ? pick_dense_t<uint16_t>(D.wplan) : pick_dense_t<float>(D.wplan);
}
template <typename ET>
static kern_t pick_grouped_t(const PwPlan &wp, const PwPlan &bp) {
    if (!wp.regular || wp.n != bp.n) return nullptr;
    switch (wp.cpl * 8 + wp.q) {
        case 8 * 8 + 1: return k_step<ET, 8, 1, 8, 1, true>;
        case 8 * 8 + 2: return k_step<ET, 8, 2, 8, 2, true>;
        case 8 * 8 + 4: return k_step<ET, 8, 4, 8, 4, true>;
        case 4 * 8 + 1: return k_step<ET, 4, 1, 4, 1, true>;
        case 2 * 8 + 1: return k_step<ET, 2, 1, 2, 1, true>;
        default: return k_step<ET, 1, 1, 1, 1, true>;
    }
}
static kern_t pick_grouped(const Dev &D) {
    return D.wdtype == CSVD_W_BF16 ? pick_grouped_t<uint16_t>(D.wplan, D.bplan)
                                   : pick_grouped_t<float>(D.wplan, D.bplan);
}
static kern_t pick_kernel(const Dev &D) {
    return D.wdtype == CSVD_W_BF16 ? pick_w<uint16_t>(D.wplan, D.bplan) : pick_w<float>(D.wplan, D.bplan);
}

// shared-memory layout (doubles): hs_w | hs_b? | generic scratch? | ordering | chunk scratch.
// Pure function of (D, K): the K-dependent part is the chunk scratch (2 running
// top-k lists + chunk * K cluster lists).  When even chunk = 1 does not fit in
// 227 KB, those lists move to global memory (per CTA, D.klists): any k <= V
// is accepted, as in the reference (decode.py:104-115).
struct SmemPlan {
    size_t bytes;
    int hs_off_b, scratch_off, ord_off, sum_off, chunk;
    bool klists_global;
};
static SmemPlan plan_smem(const Dev &D, int K) {
    SmemPlan p{};
    const bool same = D.wplan.n == D.bplan.n;
    size_t off = pw_hs_size(D.wplan);
    off = (off + 1) & ~(size_t)1;
    p.hs_off_b = 0;
    if (!same) {
        p.hs_off_b = (int)off;
        off += pw_hs_size(D.bplan);
        off = (off + 1) & ~(size_t)1;
    }
    p.scratch_off = (int)off;
    if (!D.wplan.regular || !D.bplan.regular) off += WARPS * (CSVD_MAX_LEAVES / 4);
    p.ord_off = (int)off;
    // the per-CTA ordering (sort keys, U, Uo, lrh; order, cum)
    off += ord_doubles(D.C, D.Cp);
    off = (off + 1) & ~(size_t)1;
    p.sum_off = (int)off;
    const size_t budget = (227 * 1024) / 8;
    const size_t fixed = 9 * CHUNK;
    int chunk = CHUNK;
    while (chunk > 1 && off + fixed + 2 * (size_t)K + (size_t)chunk * K > budget) chunk >>= 1;
    if (off + fixed + 2 * (size_t)K + (size_t)chunk * K <= budget) {
        p.klists_global = false;
        off += fixed + 2 * (size_t)K + (size_t)chunk * K;
    } else {
        p.klists_global = true;  // lists in global memory (L2-resident at these sizes)
        chunk = CHUNK;
        off += fixed;
    }
    p.chunk = chunk;
    p.bytes = 8 * off;
    return p;
}
// doubles of global K-list scratch per CTA (klists_global plans)
static size_t klist_stride(const SmemPlan &p, int K) { return 2 * (size_t)K + (size_t)p.chunk * K; }

static void layout_smem(csvd_ctx *ctx) {
    Dev &D = ctx->D;
    const SmemPlan p = plan_smem(D, D.K);
    D.hs_off_b = p.hs_off_b;
    D.scratch_off = p.scratch_off;
    D.ord_off = p.ord_off;
    D.sum_off = p.sum_off;
    D.chunk = p.chunk;
    ctx->smem = p.bytes;
}

// K-dependent device buffers: dense candidate lists [grid*WARPS, K], the shard
// aggregate, and (large K) the per-CTA global K-lists.  Allocated into
// temporaries first: on failure the context keeps its previous, consistent K.
static int alloc_k(csvd_ctx *ctx, int K) {
    Dev &D = ctx->D;
    const SmemPlan pl = plan_smem(D, K);
    // per-CTA / per-warp buffers are sized for the current grid, which is then
    // a cap: configure() never grows the grid past it (a smaller plan for a new
    // K could otherwise raise the occupancy above what the buffers hold)
    const int grid = ctx->grid;
    void *nb[4] = {};
    const size_t sizes[3] = {sizeof(double) * (size_t)grid * WARPS * K + 16,
                             sizeof(double) * (CSVD_SH_TOPK + (size_t)K) + 16,
                             pl.klists_global ? sizeof(double) * (size_t)grid * klist_stride(pl, K) + 16 : 0};
    for (int i = 0; i < 3; ++i) {
        if (!sizes[i]) continue;
        cudaError_t e = cudaMalloc(&nb[i], sizes[i]);
        if (e != cudaSuccess) {
            for (int j = 0; j < i; ++j)
                if (nb[j]) cudaFree(nb[j]);
            return fail(ctx, CSVD_ENOMEM, std::string("cudaMalloc (k workspace): ") + cudaGetErrorString(e));
        }
    }
    for (int i = 0; i < 4; ++i)
        if (ctx->k_buffers[i]) cudaFree(ctx->k_buffers[i]);
    for (int i = 0; i < 4; ++i) ctx->k_buffers[i] = nb[i];
    D.cand = (double *)nb[0];
    D.shard_out = (double *)nb[1];
    D.klists = (double *)nb[2];
    D.klist_stride = pl.klists_global ? klist_stride(pl, K) : 0;
    D.K = K;
    ctx->grid_cap = grid;
    return 0;
}

// grid: every SM, as many CTAs as fit (cooperative launch requires residency)
static int configure(csvd_ctx *ctx) {
    Dev &D = ctx->D;
    layout_smem(ctx);
    ctx->kern = pick_kernel(D);
    if (ctx->smem > 227 * 1024) return fail(ctx, CSVD_ECONFIG, "shared memory plan exceeds 227 KB (C or d too large)");
    CK(cudaFuncSetAttribute((const void *)ctx->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->kern, THREADS, ctx->smem));
    if (occ < 1) return fail(ctx, CSVD_ECONFIG, "step kernel does not fit on an SM");
    ctx->grid = ctx->nsm * occ;
    if (ctx->grid_cap > 0 && ctx->grid > ctx->grid_cap) ctx->grid = ctx->grid_cap;
    D.nblocks = ctx->grid;
    ctx->kdense = getenv("CSVD_DENSE_PERSISTENT") ? nullptr : pick_dense(D);
    ctx->khead = ctx->shard ? nullptr : pick_head(D);
    if (ctx->khead) {
        CK(cudaFuncSetAttribute((const void *)ctx->khead, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem));
        int occh = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occh, ctx->khead, THREADS, ctx->smem));
        if (occh * ctx->nsm < ctx->grid) ctx->khead = nullptr;  // must co-reside like k_step
    }
    // L2 bulk prefetch policy (measured: prefetching rows ahead in the dense GEMV
    // causes re-reads and costs 25%; CSVD_DENSE_PD / CSVD_PF override)
    D.dense_pd = getenv("CSVD_DENSE_PD") ? atoi(getenv("CSVD_DENSE_PD")) : 0;
    // 4: the head step's row CTAs prefetch their W rows into L2 (measured no gain: off); 1 / 2: older
    // prefetch points of the general step (no measurable gain either way)
    D.pf_mask = getenv("CSVD_PF") ? atoi(getenv("CSVD_PF")) : 0;
    if (ctx->kdense) {
        ctx->dense_smem = sizeof(double) * (size_t)pw_hs_size(D.wplan);
        CK(cudaFuncSetAttribute((const void *)ctx->kdense, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ctx->dense_smem));
        int occ2 = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, ctx->kdense, THREADS, ctx->dense_smem));
        ctx->dense_grid = ctx->nsm * (occ2 > 0 ? occ2 : 1);
    }
    if ((long long)D.C > (long long)MAX_PER_WARP * ctx->grid * WARPS)
        return fail(ctx, CSVD_ECONFIG, "too many clusters for the resident grid");
    return 0;
}

static int launch(csvd_ctx *ctx, int mode, cudaStream_t s, bool host_map = false) {
    Dev D = host_map ? ctx->Dhost : ctx->D;
    D.launch_mode = mode;
    if (mode == LAUNCH_DENSE && ctx->kdense && !ctx->shard) {  // standalone GEMV: no k-th / top-k needed
        ctx->kdense<<<ctx->dense_grid, THREADS, ctx->dense_smem, s>>>(D);
        CK(cudaGetLastError());
        return 0;
    }
    void *args[] = {&D};
    CK(cudaLaunchCooperativeKernel((const void *)ctx->kern, dim3(ctx->grid), dim3(THREADS), args, ctx->smem, s));
    return 0;
}

static int capture(csvd_ctx *ctx, int mode, bool host_io, cudaGraphExec_t *out) {
    cudaStream_t s = ctx->stream;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    if (host_io) CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    // step graphs carry no config upload: the config is uploaded only when it
    // changes (sync_cfg), so an unchanged config costs no copy node per step
    if (mode != LAUNCH_STEP)
        CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin_fixed, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    // host I/O: the kernel itself writes the result into mapped host memory
    int rc = launch(ctx, mode, s, host_io);
    if (rc) {
        cudaStreamEndCapture(s, &g);
        return rc;
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(out, g, 0));
    CK(cudaGraphDestroy(g));
    return 0;
}

// [h2d h] -> k_head (which runs the general step itself when the head cannot
// decide): one kernel node per step
static int capture_head(csvd_ctx *ctx, bool host_io, cudaGraphExec_t *out) {
    cudaStream_t s = ctx->stream;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    Dev D = host_io ? ctx->Dhost : ctx->D;
    if (host_io && ctx->h_zero_copy) {  // the kernel stages h straight from mapped host memory
        void *p = nullptr;
        CK(cudaHostGetDevicePointer(&p, ctx->h_map, 0));
        D.h = (const double *)p;
    } else if (host_io) {
        CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    }
    D.launch_mode = LAUNCH_STEP;
    void *args[] = {&D};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)ctx->khead, dim3(ctx->grid), dim3(THREADS), args,
                                                ctx->smem, s);
    cudaError_t e2 = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess || e2 != cudaSuccess) {
        if (e2 == cudaSuccess) cudaGraphDestroy(g);
        return fail(ctx, CSVD_ECUDA, std::string("head graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
    }
    e = cudaGraphInstantiate(out, g, 0);
    if (e == cudaSuccess && !host_io) {  // keep the source graph: its kernel node addresses the exec's
        size_t n = 1;
        cudaGraphNode_t node = nullptr;
        if (cudaGraphGetNodes(g, &node, &n) == cudaSuccess && n == 1) {
            if (ctx->g_step_head_src) cudaGraphDestroy(ctx->g_step_head_src);
            ctx->g_step_head_src = g;
            ctx->g_step_head_node = node;
            ctx->g_step_head_h = D.h;
            return 0;
        }
    }
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(ctx, CSVD_ECUDA, std::string("head graph instantiate: ") + cudaGetErrorString(e));
    return 0;
}

static void drop_head_src(csvd_ctx *ctx) {
    if (ctx->g_step_head_src) cudaGraphDestroy(ctx->g_step_head_src);
    ctx->g_step_head_src = nullptr;
    ctx->g_step_head_node = nullptr;
    ctx->g_step_head_h = nullptr;
}

// Point the device head graph's kernel at h (no copy node); false: not possible
static bool head_graph_set_h(csvd_ctx *ctx, const double *h) {
    if (!ctx->g_step_head || !ctx->g_step_head_node) return false;
    if (h == ctx->g_step_head_h) return true;
    cudaKernelNodeParams kp{};
    if (cudaGraphKernelNodeGetParams(ctx->g_step_head_node, &kp) != cudaSuccess || !kp.kernelParams) return false;
    Dev D = *reinterpret_cast<Dev *>(kp.kernelParams[0]);
    D.h = h;
    void *args[] = {&D};
    kp.kernelParams = args;
    if (cudaGraphExecKernelNodeSetParams(ctx->g_step_head, ctx->g_step_head_node, &kp) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    ctx->g_step_head_h = h;
    return true;
}

static int build_graphs(csvd_ctx *ctx) {
    {  // the host-API variant of the per-step Dev: mapped result buffers
        Dev &H = ctx->Dhost;
        H = ctx->D;
        void *p = nullptr;
        CK(cudaHostGetDevicePointer(&p, ctx->res_map, 0));
        H.res_host = (csvd_result *)p;
        CK(cudaHostGetDevicePointer(&p, ctx->ids_map, 0));
        H.ids_host = (long long *)p;
        CK(cudaHostGetDevicePointer(&p, ctx->logits_map, 0));
        H.logits_host = (double *)p;
    }
    for (cudaGraphExec_t *g : {&ctx->g_step, &ctx->g_host, &ctx->g_bounds, &ctx->g_dense, &ctx->g_step_head,
                               &ctx->g_host_head}) {
        if (*g) cudaGraphExecDestroy(*g);
        *g = nullptr;
    }
    drop_head_src(ctx);
    int rc;
    if (ctx->D.W) {
        if ((rc = capture(ctx, LAUNCH_STEP, false, &ctx->g_step))) return rc;
        if ((rc = capture(ctx, LAUNCH_STEP, true, &ctx->g_host))) return rc;
        if ((rc = capture(ctx, LAUNCH_DENSE, false, &ctx->g_dense))) return rc;
        if (ctx->khead) {
            if ((rc = capture_head(ctx, false, &ctx->g_step_head))) return rc;
            if ((rc = capture_head(ctx, true, &ctx->g_host_head))) return rc;
        }
    }
    if ((rc = capture(ctx, LAUNCH_BOUNDS, false, &ctx->g_bounds))) return rc;
    return 0;
}

static int check_cfg(csvd_ctx *ctx, const csvd_config *cfg);
static void fixed_cfg(csvd_config *cfg, long long V, int slack_f32);

static void free_lanes(csvd_ctx *ctx) {
    if (ctx->g_batch) cudaGraphExecDestroy(ctx->g_batch);
    ctx->g_batch = nullptr;
    ctx->g_batch_B = 0;
    for (Lane &l : ctx->lanes) {
        if (l.stream) cudaStreamDestroy(l.stream);
        if (l.done) cudaEventDestroy(l.done);
    }
    ctx->lanes.clear();
    for (void *p : ctx->lane_allocs) cudaFree(p);
    ctx->lane_allocs.clear();
    if (ctx->H_pin) cudaFreeHost(ctx->H_pin);
    if (ctx->res_pin_b) cudaFreeHost(ctx->res_pin_b);
    if (ctx->ids_pin_b) cudaFreeHost(ctx->ids_pin_b);
    if (ctx->logits_pin_b) cudaFreeHost(ctx->logits_pin_b);
    for (void *p : {(void *)ctx->res_map_b, (void *)ctx->ids_map_b, (void *)ctx->logits_map_b})
        if (p) cudaFreeHost(p);
    ctx->res_map_b = nullptr;
    ctx->ids_map_b = nullptr;
    ctx->logits_map_b = nullptr;
    ctx->H_pin = nullptr;
    ctx->res_pin_b = nullptr;
    ctx->ids_pin_b = nullptr;
    ctx->logits_pin_b = nullptr;
    ctx->lane_grid = 0;
}

template <typename T>
static int lalloc(csvd_ctx *ctx, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
    if (e != cudaSuccess) return fail(ctx, CSVD_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ctx->lane_allocs.push_back(q);
    *p = reinterpret_cast<T *>(q);
    return 0;
}

#define LANE_MIN_G 1  // CTAs per batch lane at least (4 measured no better for c4 / c5: the
                      // lanes' rows are not the large-batch bottleneck)
// B lanes, each a full per-step workspace and a grid of max(LANE_MIN_G, grid / B) CTAs
static int ensure_lanes(csvd_ctx *ctx, int B) {
    const Dev &D0 = ctx->D;
    // CTAs per lane: the grid split B ways, but at least LANE_MIN_G (large
    // batches then run in sub-batches of grid / G lanes, one launch each)
    const int G = std::min(ctx->grid, std::max(ctx->grid / B, std::min(LANE_MIN_G, ctx->grid)));
    if ((int)ctx->lanes.size() == B && ctx->lane_grid == G && ctx->lane_K == D0.K) return 0;
    free_lanes(ctx);
    const int C = D0.C, V = D0.V, K = D0.K;
    int rc;
    if ((rc = lalloc(ctx, &ctx->d_H, (size_t)B * D0.d))) return rc;
    if ((rc = lalloc(ctx, &ctx->d_res_all, (size_t)B))) return rc;
    CK(cudaMemset(ctx->d_res_all, 0, sizeof(csvd_result) * B));
    const int first = (int)ctx->first_chunk;
    CK(cudaHostAlloc(&ctx->H_pin, sizeof(double) * B * D0.d, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->res_pin_b, sizeof(csvd_result) * B, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->ids_pin_b, sizeof(long long) * B * first, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->logits_pin_b, sizeof(double) * B * first, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->res_map_b, sizeof(csvd_result) * B, cudaHostAllocMapped));
    CK(cudaHostAlloc(&ctx->ids_map_b, sizeof(long long) * B * (size_t)V, cudaHostAllocMapped));
    CK(cudaHostAlloc(&ctx->logits_map_b, sizeof(double) * B * (size_t)V, cudaHostAllocMapped));
    ctx->lanes.resize(B);
    for (int b = 0; b < B; ++b) {
        Lane &l = ctx->lanes[b];
        Dev L = D0;  // shared read-only table / index data, own workspaces
        L.h = ctx->d_H + (size_t)b * D0.d;
        L.res = ctx->d_res_all + b;
        const SmemPlan pl = plan_smem(D0, K);
        L.klists = nullptr;
        L.klist_stride = pl.klists_global ? klist_stride(pl, K) : 0;
        if ((rc = lalloc(ctx, &L.U, C)) || (rc = lalloc(ctx, &L.Uraw, C)) || (rc = lalloc(ctx, &L.dots, C)) ||
            (rc = lalloc(ctx, &L.order_g, C)) || (rc = lalloc(ctx, &L.cum_g, C + 1)) ||
            (rc = lalloc(ctx, &L.S_logits, (size_t)V)) || (rc = lalloc(ctx, &L.S_ids, (size_t)V)) ||
            (rc = lalloc(ctx, &L.st, 1)) || (rc = lalloc(ctx, &L.bar, 4)) ||
            (rc = lalloc(ctx, &L.cand, (size_t)G * WARPS * K)) ||
            (rc = lalloc(ctx, &L.shard_out, (size_t)CSVD_SH_TOPK + K)) ||
            (pl.klists_global && (rc = lalloc(ctx, &L.klists, (size_t)G * L.klist_stride))))
            return rc;
        CK(cudaMemset(L.bar, 0, 16));
        CK(cudaMemset(L.st, 0, sizeof(ScanState)));
        if ((rc = lalloc(ctx, &L.hcnt, (size_t)HW_TOTAL_INTS)) || (rc = lalloc(ctx, &L.bar64, 4))) return rc;
        CK(cudaMemset(L.hcnt, 0, sizeof(int) * HW_TOTAL_INTS));
        CK(cudaMemset(L.bar64, 0, 32));
        L.nblocks = G;
        L.gsum = nullptr;  // distributed wave summaries: single-step contexts only
        L.dbg = b == 0 ? D0.dbg : nullptr;  // debug timestamps follow lane 0
        L.res_host = nullptr;
        L.ids_host = nullptr;
        L.logits_host = nullptr;
        l.D = L;
        {
            Dev Hl = L;
            void *p = nullptr;
            CK(cudaHostGetDevicePointer(&p, ctx->res_map_b + b, 0));
            Hl.res_host = (csvd_result *)p;
            CK(cudaHostGetDevicePointer(&p, ctx->ids_map_b + (size_t)b * V, 0));
            Hl.ids_host = (long long *)p;
            CK(cudaHostGetDevicePointer(&p, ctx->logits_map_b + (size_t)b * V, 0));
            Hl.logits_host = (double *)p;
            l.Dh = Hl;
        }
        CK(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
    }
    if (!ctx->fork) CK(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
    // shared batched bounds: regular bound plans (d = 2^m leaves of L % 8 == 0)
    ctx->kbb = nullptr;
    if (D0.bplan.regular && D0.bplan.cpl == 8 && D0.mode != CSVD_MODE_BIAS_AUGMENTED) {
        const bool pair = getenv("CSVD_KBB_PAIR") ? atoi(getenv("CSVD_KBB_PAIR")) != 0 : D0.C > ctx->grid * WARPS;
        switch (D0.bplan.q) {
            // two clusters per warp task (half the shared-memory reads of h) when
            // the clusters outnumber the warps; else one cluster x 6 queries
            case 1: ctx->kbb = pair ? k_bounds_batch<1, 2> : k_bounds_batch<1, 1>; break;
            case 2: ctx->kbb = pair ? k_bounds_batch<2, 2> : k_bounds_batch<2, 1>; break;
            case 4: ctx->kbb = pair ? k_bounds_batch<4, 2> : k_bounds_batch<4, 1>; break;
        }
    }
    if (ctx->kbb) {
        std::vector<double *> ur(B), dt(B);
        for (int b = 0; b < B; ++b) {
            ur[b] = ctx->lanes[b].D.Uraw;
            dt[b] = ctx->lanes[b].D.dots;
            ctx->lanes[b].D.pre_bounds = 1;
            ctx->lanes[b].Dh.pre_bounds = 1;  // the host-I/O twin of the lane too
        }
        if ((rc = lalloc(ctx, &ctx->d_Uraw_l, B)) || (rc = lalloc(ctx, &ctx->d_dots_l, B))) return rc;
        CK(cudaMemcpy(ctx->d_Uraw_l, ur.data(), sizeof(double *) * B, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_dots_l, dt.data(), sizeof(double *) * B, cudaMemcpyHostToDevice));
        const size_t hsb = sizeof(double) * (size_t)((pw_hs_size(D0.bplan) + 1) & ~1);
        ctx->kbb_gq = (int)std::min<size_t>(BQN1, (227 * 1024 - 64) / hsb);
        if (const char *e = getenv("CSVD_KBB_GQ"))  // queries per pass cap (<= 3: two-cluster path)
            ctx->kbb_gq = std::max(1, std::min(ctx->kbb_gq, atoi(e)));
        ctx->kbb_smem = hsb * ctx->kbb_gq;
        CK(cudaFuncSetAttribute((const void *)ctx->kbb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ctx->kbb_smem));
        // chain-per-lane form (k_bbatch): 4 <= NL <= 64 leaves (the slice tree's depth)
        const int NL = D0.d / D0.bplan.leaf_len;
        const int NS = NL / 4;
        ctx->kbb2_kq = KBQ;
        while (ctx->kbb2_kq > 0 && kbb2_smem_bytes(ctx->kbb2_kq, D0.d, NS) > 227 * 1024) --ctx->kbb2_kq;
        ctx->kbb2 = getenv("CSVD_KBB_NEW") && NL >= 4 && NL <= 64 && (NL & (NL - 1)) == 0 && ctx->kbb2_kq >= 1;
        if (ctx->kbb2) {
            ctx->kbb2_smem = kbb2_smem_bytes(ctx->kbb2_kq, D0.d, NS);
            CK(cudaFuncSetAttribute((const void *)k_bbatch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ctx->kbb2_smem));
        }
    }
    {  // per-lane workspace tables for the grouped launch
        auto ws = [](const Dev &L) {
            LaneWS w{};
            w.h = L.h;
            w.U = L.U;
            w.Uraw = L.Uraw;
            w.dots = L.dots;
            w.order_g = L.order_g;
            w.cum_g = L.cum_g;
            w.S_logits = L.S_logits;
            w.S_ids = L.S_ids;
            w.st = L.st;
            w.res = L.res;
            w.bar = L.bar;
            w.cand = L.cand;
            w.klists = L.klists;
            w.shard_out = L.shard_out;
            w.res_host = L.res_host;
            w.ids_host = L.ids_host;
            w.logits_host = L.logits_host;
            w.hcnt = L.hcnt;
            w.bar64 = L.bar64;
            return w;
        };
        std::vector<LaneWS> td(B), th(B);
        for (int b = 0; b < B; ++b) {
            td[b] = ws(ctx->lanes[b].D);
            th[b] = ws(ctx->lanes[b].Dh);
        }
        if ((rc = lalloc(ctx, &ctx->d_lanes, B)) || (rc = lalloc(ctx, &ctx->d_lanes_host, B))) return rc;
        CK(cudaMemcpy(ctx->d_lanes, td.data(), sizeof(LaneWS) * B, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_lanes_host, th.data(), sizeof(LaneWS) * B, cudaMemcpyHostToDevice));
        const int LB = std::min(B, ctx->grid / G);  // lanes per launch
        ctx->kgroup = getenv("CSVD_LANES_FORKED") ? nullptr : pick_grouped(D0);
        ctx->kgroup_head = (ctx->kgroup && ctx->kbb) ? pick_head_lanes(D0) : nullptr;
        if (ctx->kgroup_head) {
            CK(cudaFuncSetAttribute((const void *)ctx->kgroup_head, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ctx->smem));
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->kgroup_head, THREADS, ctx->smem));
            if (occ * ctx->nsm < LB * G) ctx->kgroup_head = nullptr;
        }
        if (ctx->kgroup) {
            CK(cudaFuncSetAttribute((const void *)ctx->kgroup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ctx->smem));
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->kgroup, THREADS, ctx->smem));
            if (occ * ctx->nsm < LB * G) ctx->kgroup = nullptr;
        }
    }
    ctx->lane_grid = G;
    ctx->lane_K = K;
    return 0;
}

// the batch graph: [H2D H, cfg] -> fork -> B lane kernels -> join [-> D2H results + first chunks]
static int capture_batch(csvd_ctx *ctx, int B, bool host_io, bool head) {
    if (ctx->g_batch) cudaGraphExecDestroy(ctx->g_batch);
    ctx->g_batch = nullptr;
    cudaStream_t s = ctx->stream;
    cudaGraph_t g;
    const Dev &D0 = ctx->D;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    if (host_io)
        CK(cudaMemcpyAsync(ctx->d_H, ctx->H_pin, sizeof(double) * B * D0.d, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin_b, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    if (ctx->kbb && ctx->kbb2) {  // all B dot vectors at once: clusters x queries register blocks
        const int ng = (B + ctx->kbb2_kq - 1) / ctx->kbb2_kq;
        k_bbatch<<<ctx->nsm, THREADS, ctx->kbb2_smem, s>>>(D0, ctx->d_H, B, ctx->d_dots_l, ctx->kbb2_kq, ng);
        CK(cudaGetLastError());
    } else if (ctx->kbb) {  // all B bounds vectors at once, each centroid row read once per 4 queries
        ctx->kbb<<<ctx->grid, THREADS, ctx->kbb_smem, s>>>(D0, ctx->d_H, B, ctx->d_Uraw_l, ctx->d_dots_l,
                                                           ctx->d_res_all, ctx->kbb_gq);
        CK(cudaGetLastError());
    }
    if (ctx->kgroup) {  // every lane in one cooperative launch of B x G CTAs
        Dev Dg = host_io ? ctx->lanes[0].Dh : ctx->lanes[0].D;
        Dg.launch_mode = LAUNCH_STEP;
        Dg.lanes = host_io ? ctx->d_lanes_host : ctx->d_lanes;
        const kern_t kl = (head && ctx->kgroup_head) ? ctx->kgroup_head : ctx->kgroup;
        const LaneWS *base = Dg.lanes;
        const int LB = ctx->grid / ctx->lane_grid;  // lanes per launch (sub-batches for large B)
        for (int first = 0; first < B; first += LB) {
            const int n = std::min(LB, B - first);
            Dg.lanes = base + first;
            void *args[] = {&Dg};
            CK(cudaLaunchCooperativeKernel((const void *)kl, dim3(n * ctx->lane_grid), dim3(THREADS), args,
                                           ctx->smem, s));
        }
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ctx->g_batch, g, 0));
        CK(cudaGraphDestroy(g));
        ctx->g_batch_B = B;
        ctx->g_batch_host = host_io ? 1 : 0;
        ctx->g_batch_head = head ? 1 : 0;
        return 0;
    }
    CK(cudaEventRecord(ctx->fork, s));
    for (int b = 0; b < B; ++b) {
        Lane &l = ctx->lanes[b];
        CK(cudaStreamWaitEvent(l.stream, ctx->fork, 0));
        Dev Dl = host_io ? l.Dh : l.D;  // host I/O: each lane publishes into mapped memory
        Dl.launch_mode = LAUNCH_STEP;
        void *args[] = {&Dl};
        CK(cudaLaunchCooperativeKernel((const void *)ctx->kern, dim3(ctx->lane_grid), dim3(THREADS), args, ctx->smem,
                                       l.stream));
        CK(cudaEventRecord(l.done, l.stream));
        CK(cudaStreamWaitEvent(s, l.done, 0));
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ctx->g_batch, g, 0));
    CK(cudaGraphDestroy(g));
    ctx->g_batch_B = B;
    ctx->g_batch_host = host_io ? 1 : 0;
    ctx->g_batch_head = head ? 1 : 0;
    return 0;
}

// Rewrite a pinned staging config that queued graphs' memcpy nodes read at
// execution time: wait for the streams first when the contents change (an
// earlier asynchronous replay must still see the config it was issued with).
static int stage_pinned_cfg(csvd_ctx *ctx, csvd_config *pin, const csvd_config &cfg, cudaStream_t s) {
    if (memcmp(pin, &cfg, sizeof cfg) == 0) return 0;
    CK(cudaStreamSynchronize(s));
    if (s != ctx->stream) CK(cudaStreamSynchronize(ctx->stream));
    *pin = cfg;
    return 0;
}

static int batch_prepare(csvd_ctx *ctx, int B, const csvd_config *cfg, bool host_io, cudaStream_t s) {
    if (ctx) ctx->cfg_valid = false;  // this path writes its own config into d_cfg
    if (B < 1 || B > 1024) return fail(ctx, CSVD_ECONFIG, "batch size must be in [1, 1024]");
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    if ((rc = ensure_lanes(ctx, B))) return rc;
    if ((rc = stage_pinned_cfg(ctx, ctx->cfg_pin_b, *cfg, s))) return rc;
    const bool head = ctx->kgroup_head && head_config(cfg);
    if (!ctx->g_batch || ctx->g_batch_B != B || ctx->g_batch_host != (host_io ? 1 : 0) ||
        ctx->g_batch_head != (head ? 1 : 0))
        if ((rc = capture_batch(ctx, B, host_io, head))) return rc;
    return 0;
}

extern "C" int csvd_step_batch_device(csvd_ctx *ctx, int32_t B, const double *H_dev, const csvd_config *cfg,
                                      void *stream) {
    if (!ctx || !cfg || !H_dev) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    int rc = batch_prepare(ctx, B, cfg, false, s);
    if (rc) return rc;
    if (H_dev != ctx->d_H)
        CK(cudaMemcpyAsync(ctx->d_H, H_dev, sizeof(double) * B * ctx->D.d, cudaMemcpyDeviceToDevice, s));
    CK(cudaGraphLaunch(ctx->g_batch, s));
    ctx->last_launches = (ctx->kbb ? 1 : 0) +
                         (ctx->kgroup ? (ctx->g_batch_B + ctx->grid / ctx->lane_grid - 1) / (ctx->grid / ctx->lane_grid)
                                      : ctx->g_batch_B);
    return 0;
}

extern "C" int csvd_step_batch_host(csvd_ctx *ctx, int32_t B, const double *H, const csvd_config *cfg,
                                    csvd_result *res, int64_t *ids, double *logits, int64_t cap) {
    if (!ctx || !cfg || !H || !res) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc = batch_prepare(ctx, B, cfg, true, s);
    if (rc) return rc;
    static const bool prof = getenv("CSVD_PROFILE_HOST") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    memcpy(ctx->H_pin, H, sizeof(double) * B * ctx->D.d);
    for (int b = 0; b < B; ++b) ctx->res_map_b[b].kind = CSVD_KIND_NONE - 1;  // sentinels, overwritten by the lanes
    auto t1 = now();
    CK(cudaGraphLaunch(ctx->g_batch, s));
    ctx->last_launches = (ctx->kbb ? 1 : 0) +
                         (ctx->kgroup ? (ctx->g_batch_B + ctx->grid / ctx->lane_grid - 1) / (ctx->grid / ctx->lane_grid)
                                      : ctx->g_batch_B);
    auto t2 = now();
    // every lane publishes its result into mapped memory; busy-poll the stream
    cudaError_t q;
    while ((q = cudaStreamQuery(s)) == cudaErrorNotReady) {
    }
    if (q != cudaSuccess) return fail(ctx, CSVD_ECUDA, std::string("batch: ") + cudaGetErrorString(q));
    int ready = 0;
    for (int b = 0; b < B; ++b) ready += ctx->res_map_b[b].kind != CSVD_KIND_NONE - 1;
    if (ready < B) {  // a lane ended without publishing: device error
        CK(cudaStreamSynchronize(s));
        std::vector<csvd_result> rr(B);
        CK(cudaMemcpy(rr.data(), ctx->d_res_all, sizeof(csvd_result) * B, cudaMemcpyDeviceToHost));
        bool value_err = false;
        for (auto &r : rr) value_err = value_err || r.error == CSVD_EVALUE;

        CK(cudaMemset(ctx->d_res_all, 0, sizeof(csvd_result) * B));
        for (Lane &l : ctx->lanes) {
            CK(cudaMemset(l.D.bar, 0, 16));
        }
        if (value_err) return fail(ctx, CSVD_EVALUE, "bounds must be finite");
        return fail(ctx, CSVD_ESTATE, "device state error in a batch lane (grid barrier timeout)");
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (prof) {
        auto t3 = now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        fprintf(stderr, "batch host: stage %.1f us, graph launch %.1f us, wait %.1f us\n", us(t0, t1), us(t1, t2),
                us(t2, t3));
    }
    const int64_t V = ctx->D.V;
    for (int b = 0; b < B; ++b) {
        memcpy(&res[b], (const void *)(ctx->res_map_b + b), sizeof(csvd_result));
        if (res[b].error) {
            const int e = res[b].error;
            return fail(ctx, e, e == CSVD_EVALUE ? "bounds must be finite" : "device state error");
        }
        const int64_t n = res[b].sub_size;
        if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
        if (ids) memcpy(ids + (size_t)b * cap, ctx->ids_map_b + (size_t)b * V, sizeof(int64_t) * n);
        if (logits) memcpy(logits + (size_t)b * cap, ctx->logits_map_b + (size_t)b * V, sizeof(double) * n);
    }
    return 0;
}

extern "C" int csvd_batch_lanes(csvd_ctx *ctx, int32_t *lanes, int32_t *grid_per_lane) {
    if (!ctx) return CSVD_ESTATE;
    if (lanes) *lanes = (int32_t)ctx->lanes.size();
    if (grid_per_lane) *grid_per_lane = ctx->lane_grid;
    return 0;
}

extern "C" int csvd_reserve_k(csvd_ctx *ctx, int32_t k) {
    if (!ctx) return CSVD_ESTATE;
    if (k <= ctx->D.K) return 0;
    if (k < 1 || (long long)k > (long long)ctx->D.V) return fail(ctx, CSVD_ECONFIG, "need 1 <= k <= V");
    int K = 32;
    while (K < k) K <<= 1;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));  // queued graphs still reference the old buffers
    int rc;
    free_lanes(ctx);  // lanes are rebuilt for the new K on the next batch
    if ((rc = alloc_k(ctx, K))) return rc;  // all-or-nothing: the old K stays valid on failure
    if ((rc = configure(ctx)) || (rc = build_graphs(ctx))) {
        // no graph may keep pointing at buffers of a half-applied K
        for (cudaGraphExec_t *g : {&ctx->g_step, &ctx->g_host, &ctx->g_bounds, &ctx->g_dense, &ctx->g_step_head,
                                   &ctx->g_host_head}) {
            if (*g) cudaGraphExecDestroy(*g);
            *g = nullptr;
        }
        drop_head_src(ctx);
        return rc;
    }
    return 0;
}

static int create_impl(csvd_ctx **out, int device, const csvd_table_desc *t, const csvd_index_desc *ix,
                       const uint8_t *owned) {
    if (!out || !t || !ix) return CSVD_ECONFIG;
    csvd_ctx *ctx = new csvd_ctx();
    *out = ctx;
    ctx->device = device;
    CK(cudaSetDevice(device));
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) return fail(ctx, CSVD_ECUDA, "device does not support cooperative launch");
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    Dev &D = ctx->D;
    if (t->vocab_size < 1 || t->hidden_dim < 1 || t->vocab_size >= (1ll << 31))
        return fail(ctx, CSVD_EDIM, "bad table dims");
    if (ix->n_clusters < 1 || ix->n_clusters > 4096)
        return fail(ctx, CSVD_ECONFIG, "n_clusters must be in [1, 4096]");
    D.V = (int)t->vocab_size;
    D.d = (int)t->hidden_dim;
    D.C = ix->n_clusters;
    D.Cp = 1;
    while (D.Cp < D.C) D.Cp <<= 1;
    if (D.Cp < 2) D.Cp = 2;
    D.mode = ix->mode;
    D.bd = D.d + (ix->mode == CSVD_MODE_BIAS_AUGMENTED ? 1 : 0);
    D.wdtype = t->w_dtype;
    if (D.d > 16384) return fail(ctx, CSVD_EDIM, "hidden_dim > 16384 unsupported");
    // pairwise plans (+ interleaved source tables for CPL < 8 regular plans)
    make_plan(D.d, D.wplan, ctx->wleaves, ctx->wprog);
    make_plan(D.bd, D.bplan, ctx->bleaves, ctx->bprog);
    if (D.wplan.nleaf > CSVD_MAX_LEAVES / 4 || D.bplan.nleaf > CSVD_MAX_LEAVES / 4)
        return fail(ctx, CSVD_EDIM, "too many pairwise leaves");
    int rc;
    int2 *dl;
    short *dp;
    int *di;
    if ((rc = dupload(ctx, &dl, ctx->wleaves.data(), ctx->wleaves.size()))) return rc;
    if ((rc = dupload(ctx, &dp, ctx->wprog.data(), ctx->wprog.size()))) return rc;
    D.wplan.leaves = dl;
    D.wplan.prog = dp;
    if ((rc = dupload(ctx, &dl, ctx->bleaves.data(), ctx->bleaves.size()))) return rc;
    if ((rc = dupload(ctx, &dp, ctx->bprog.data(), ctx->bprog.size()))) return rc;
    D.bplan.leaves = dl;
    D.bplan.prog = dp;
    for (int which = 0; which < 2; ++which) {
        const PwPlan &pl = which ? D.bplan : D.wplan;
        const int *src_dev = nullptr;
        if (pl.regular && pl.cpl < 8) {
            std::vector<int> src(pl.n);
            for (int idx = 0; idx < pl.n; ++idx) src[idx] = pw_hs_source(pl, idx);
            if ((rc = dupload(ctx, &di, src.data(), src.size()))) return rc;
            src_dev = di;
        }
        if (which) D.bsrc = src_dev; else D.wsrc = src_dev;
    }
    // --- table: upload in original order, permute on device (weights == NULL:
    //     bounds-only context for cluster_bounds(index, h), which has no table)
    const long long V = D.V;
    const size_t esz = (D.wdtype == CSVD_W_BF16) ? 2 : 4;
    const size_t row_bytes = esz * (size_t)D.d;
    // local rows: every row (unsharded) or the owned clusters' rows, cluster by
    // cluster in id order (each cluster stays one contiguous row range)
    const int Cn = ix->n_clusters;
    ctx->shard = owned != nullptr;
    ctx->owned.assign(Cn, 1);
    if (owned)
        for (int c = 0; c < Cn; ++c) ctx->owned[c] = owned[c] ? 1 : 0;
    std::vector<int> wrow0(Cn, -1), lpos;
    std::vector<long long> lperm;  // local row -> original token id
    {
        int lr = 0;
        for (int c = 0; c < Cn; ++c) {
            if (!ctx->owned[c]) continue;
            wrow0[c] = lr;
            for (long long i = 0; i < ix->sizes[c]; ++i) {
                const long long pos = ix->starts[c] + i;
                if (pos < 0 || pos >= V) return fail(ctx, CSVD_ECONFIG, "cluster ranges out of range");
                lpos.push_back((int)pos);
                lperm.push_back(ix->perm[pos]);
                ++lr;
            }
        }
        D.Vl = lr;
    }
    ctx->local_tokens.assign(lperm.begin(), lperm.end());
    std::sort(ctx->local_tokens.begin(), ctx->local_tokens.end());
    if (t->weights) {
        void *Wtmp = nullptr, *W = nullptr;
        CK(cudaMalloc(&Wtmp, row_bytes * V));
        CK(cudaMemcpy(Wtmp, t->weights, row_bytes * V, cudaMemcpyHostToDevice));
        long long *dperm64;
        if ((rc = dupload(ctx, &dperm64, lperm.data(), lperm.size()))) return rc;
        CK(cudaMalloc(&W, row_bytes * (size_t)(D.Vl > 0 ? D.Vl : 1) + 64));
        ctx->dev_allocs.push_back(W);
        if (D.Vl > 0)
            k_permute_rows<<<4096, 256>>>((const char *)Wtmp, (char *)W, dperm64, D.Vl, (long long)row_bytes);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaFree(Wtmp));
        D.W = W;
    } else {
        D.W = nullptr;
    }
    {
        int *dw;
        if ((rc = dupload(ctx, &dw, wrow0.data(), wrow0.size()))) return rc;
        D.wrow0 = dw;
        D.lpos = nullptr;
        if (owned) {
            if ((rc = dupload(ctx, &dw, lpos.data(), lpos.size() ? lpos.size() : 1))) return rc;
            D.lpos = dw;
        }
    }
    std::vector<double> biasp(V);
    std::vector<int> perm32(V);
    for (long long p = 0; p < V; ++p) {
        long long tok = ix->perm[p];
        if (tok < 0 || tok >= V) return fail(ctx, CSVD_ECONFIG, "perm out of range");
        perm32[p] = (int)tok;
        biasp[p] = t->bias ? t->bias[tok] : 0.0;
    }
    double *dbias;
    int *dperm;
    if ((rc = dupload(ctx, &dbias, biasp.data(), (size_t)V))) return rc;
    if ((rc = dupload(ctx, &dperm, perm32.data(), (size_t)V))) return rc;
    D.bias = dbias;
    D.perm = dperm;
    // --- index arrays
    const int C = D.C;
    std::vector<int> st32(C), sz32(C);
    std::vector<double> meanb(C);
    long long pos = 0;
    for (int c = 0; c < C; ++c) {
        st32[c] = (int)ix->starts[c];
        sz32[c] = (int)ix->sizes[c];
        if (ix->starts[c] != pos || ix->sizes[c] < 1)
            return fail(ctx, CSVD_ECONFIG, "cluster ranges must partition [0,V)");
        pos += ix->sizes[c];
        double s = 0;
        for (long long p = ix->starts[c]; p < ix->starts[c] + ix->sizes[c]; ++p) s += biasp[p];
        meanb[c] = s / (double)ix->sizes[c];
    }
    if (pos != V) return fail(ctx, CSVD_ECONFIG, "cluster ranges must cover [0,V)");
    double *dd;
    if ((rc = dupload(ctx, &dd, ix->centroids, (size_t)C * D.bd))) return rc;
    D.cent = dd;
    if ((rc = dupload(ctx, &dd, ix->radii, (size_t)C))) return rc;
    D.radii = dd;
    if ((rc = dupload(ctx, &dd, ix->max_biases, (size_t)C))) return rc;
    D.maxb = dd;
    if ((rc = dupload(ctx, &dd, ix->log_sizes, (size_t)C))) return rc;
    D.logsz = dd;
    if ((rc = dupload(ctx, &dd, meanb.data(), (size_t)C))) return rc;
    D.meanb = dd;
    if (D.mode == CSVD_MODE_SPHERICAL) {
        if (!ix->centroid_norms || !ix->angulars || !ix->max_norms || !ix->min_norms)
            return fail(ctx, CSVD_ECONFIG, "spherical index needs norms/angulars");
        if ((rc = dupload(ctx, &dd, ix->centroid_norms, (size_t)C))) return rc;
        D.cnorm = dd;
        if ((rc = dupload(ctx, &dd, ix->angulars, (size_t)C))) return rc;
        D.ang = dd;
        if ((rc = dupload(ctx, &dd, ix->max_norms, (size_t)C))) return rc;
        D.maxn = dd;
        if ((rc = dupload(ctx, &dd, ix->min_norms, (size_t)C))) return rc;
        D.minn = dd;
    }
    if ((rc = dupload(ctx, &di, st32.data(), (size_t)C))) return rc;
    D.starts = di;
    if ((rc = dupload(ctx, &di, sz32.data(), (size_t)C))) return rc;
    D.sizes = di;
    // --- per-step workspace
    if ((rc = dalloc(ctx, &ctx->d_h, (size_t)D.d))) return rc;
    D.h = ctx->d_h;
    if ((rc = dalloc(ctx, &ctx->d_cfg, 1))) return rc;
    D.cfg = ctx->d_cfg;
    if ((rc = dalloc(ctx, &D.U, C))) return rc;
    if ((rc = dalloc(ctx, &D.dots, C))) return rc;
    if ((rc = dalloc(ctx, &D.Uraw, C))) return rc;
    if ((rc = dalloc(ctx, &D.order_g, C))) return rc;
    if ((rc = dalloc(ctx, &D.cum_g, C + 1))) return rc;
    if ((rc = dalloc(ctx, &D.S_logits, (size_t)V))) return rc;
    if ((rc = dalloc(ctx, &D.S_ids, (size_t)V))) return rc;
    if ((rc = dalloc(ctx, &D.st, 1))) return rc;
    if ((rc = dalloc(ctx, &D.res, 1))) return rc;
    if ((rc = dalloc(ctx, &D.bar, 4))) return rc;
    CK(cudaMemset(D.bar, 0, 16));
    if ((rc = dalloc(ctx, &D.gsum, (size_t)D.C * (3 + 32)))) return rc;
    if ((rc = dalloc(ctx, &D.hcnt, (size_t)HW_TOTAL_INTS))) return rc;
    CK(cudaMemset(D.hcnt, 0, sizeof(int) * HW_TOTAL_INTS));
    if ((rc = dalloc(ctx, &D.bar64, 2))) return rc;
    CK(cudaMemset(D.bar64, 0, 16));
    CK(cudaMemset(D.st, 0, sizeof(ScanState)));
    CK(cudaMemset(D.res, 0, sizeof(csvd_result)));
    D.dbg = nullptr;
    D.pre_bounds = 0;
    D.lanes = nullptr;
    if (getenv("CSVD_DEBUG_TS") && atoi(getenv("CSVD_DEBUG_TS")) > 0) {
        if ((rc = dalloc(ctx, &D.dbg, 128 + 512))) return rc;  // + per-CTA start / end times
        CK(cudaMemset(D.dbg, 0, (128 + 512) * 8));
    }
    CK(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device));
    // --- pinned staging
    ctx->first_chunk = D.V < 4096 ? D.V : 4096;
    CK(cudaHostAlloc(&ctx->h_pin, sizeof(double) * (D.d + 1), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->h_map, sizeof(double) * (D.d + 1), cudaHostAllocMapped));
    ctx->h_zero_copy = getenv("CSVD_H_ZERO_COPY") != nullptr;  // measured: TMA from mapped host memory is slower than the copy node
    CK(cudaHostAlloc(&ctx->cfg_pin, sizeof(csvd_config), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->cfg_pin_b, sizeof(csvd_config), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->cfg_pin_fixed, sizeof(csvd_config), cudaHostAllocDefault));
    memset(ctx->cfg_pin_b, 0, sizeof(csvd_config));
    fixed_cfg(ctx->cfg_pin_fixed, D.V, 0);
    CK(cudaHostAlloc(&ctx->res_pin, sizeof(csvd_result), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->ids_pin, sizeof(long long) * V, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->logits_pin, sizeof(double) * V, cudaHostAllocDefault));
    memset(ctx->cfg_pin, 0, sizeof(csvd_config));
    CK(cudaHostAlloc(&ctx->res_map, sizeof(csvd_result), cudaHostAllocMapped));
    CK(cudaHostAlloc(&ctx->ids_map, sizeof(long long) * V, cudaHostAllocMapped));
    CK(cudaHostAlloc(&ctx->logits_map, sizeof(double) * V, cudaHostAllocMapped));
    D.res_host = nullptr;
    D.ids_host = nullptr;
    D.logits_host = nullptr;
    D.K = 32;
    if ((rc = configure(ctx))) return rc;  // grid size first (K buffers are per CTA / warp)
    if ((rc = alloc_k(ctx, 32))) return rc;
    if ((rc = configure(ctx))) return rc;
    return build_graphs(ctx);
}

extern "C" int csvd_create(csvd_ctx **out, int device, const csvd_table_desc *t, const csvd_index_desc *ix) {
    return create_impl(out, device, t, ix, nullptr);
}

extern "C" int csvd_create_shard(csvd_ctx **out, int device, const csvd_table_desc *t, const csvd_index_desc *ix,
                                 const uint8_t *owned) {
    if (!owned) return CSVD_ECONFIG;
    return create_impl(out, device, t, ix, owned);
}

extern "C" int csvd_destroy(csvd_ctx *ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (cudaGraphExec_t g : {ctx->g_step, ctx->g_host, ctx->g_bounds, ctx->g_dense, ctx->g_step_head, ctx->g_host_head})
        if (g) cudaGraphExecDestroy(g);
    drop_head_src(ctx);
    free_lanes(ctx);
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    for (void *p : ctx->dev_allocs) cudaFree(p);
    for (int i = 0; i < 4; ++i)
        if (ctx->k_buffers[i]) cudaFree(ctx->k_buffers[i]);
    if (ctx->flush_buf) cudaFree(ctx->flush_buf);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    if (ctx->h_map) cudaFreeHost(ctx->h_map);
    for (csvd_config *p : {ctx->cfg_pin, ctx->cfg_pin_b, ctx->cfg_pin_fixed})
        if (p) cudaFreeHost(p);
    if (ctx->res_pin) cudaFreeHost(ctx->res_pin);
    if (ctx->ids_pin) cudaFreeHost(ctx->ids_pin);
    if (ctx->logits_pin) cudaFreeHost(ctx->logits_pin);
    for (void *p : {(void *)ctx->res_map, (void *)ctx->ids_map, (void *)ctx->logits_map})
        if (p) cudaFreeHost(p);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return 0;
}

extern "C" const char *csvd_strerror(csvd_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

static int check_cfg(csvd_ctx *ctx, const csvd_config *cfg) {
    const Dev &D = ctx->D;
    if (!D.W) return fail(ctx, CSVD_ECONFIG, "bounds-only context (no table)");
    if (cfg->k < 1 || cfg->k > D.V) return fail(ctx, CSVD_ECONFIG, "need 1 <= k <= V");
    if (cfg->n_targets < 1 || cfg->n_targets > 3) return fail(ctx, CSVD_ECONFIG, "bad targets");
    if (!(cfg->epsilon > 0 && cfg->epsilon < 1)) return fail(ctx, CSVD_ECONFIG, "epsilon must lie in (0, 1)");
    if (cfg->n_levels < 1 || cfg->n_levels > CSVD_MAX_LEVELS) return fail(ctx, CSVD_ECONFIG, "bad fallback levels");
    if (cfg->k_max < 0) return fail(ctx, CSVD_ECONFIG, "K_max must be >= 0");
    int rc = 0;
    if (cfg->k > ctx->D.K) rc = csvd_reserve_k(ctx, cfg->k);
    return rc;
}

// device-side result error -> error code
static int result_error(csvd_ctx *ctx, const csvd_result &r) {
    if (!r.error) return 0;
    cudaMemset(&ctx->D.res->error, 0, sizeof(int32_t));
    if (r.error == CSVD_EVALUE) return fail(ctx, CSVD_EVALUE, "bounds must be finite");
    cudaMemset(ctx->D.bar, 0, 16);  // a timed-out barrier leaves stale counts
    cudaMemset(ctx->D.bar64, 0, 16);
    cudaMemset(ctx->D.hcnt, 0, sizeof(int) * HW_INTS);
    return fail(ctx, r.error, "device state error (grid barrier timeout)");
}

// make d_cfg hold *cfg (stream-ordered, synchronous on change: configs rarely
// change between steps, and a pinned staging buffer must not be rewritten
// while an earlier upload is still queued)
static int sync_cfg(csvd_ctx *ctx, const csvd_config *cfg, cudaStream_t s) {
    if (ctx->cfg_valid && memcmp(&ctx->cfg_dev, cfg, sizeof(csvd_config)) == 0) return 0;
    CK(cudaStreamSynchronize(s));
    *ctx->cfg_pin = *cfg;
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    ctx->cfg_dev = *cfg;
    ctx->cfg_valid = true;
    return 0;
}

extern "C" int csvd_step_device(csvd_ctx *ctx, const double *h_dev, const csvd_config *cfg, void *stream) {
    if (!ctx || !cfg) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    const bool head = !ctx->direct && ctx->g_step_head && head_config(cfg);
    const double *hsrc = h_dev ? h_dev : ctx->d_h;
    const bool in_place = head && ((uintptr_t)hsrc % 16 == 0) && head_graph_set_h(ctx, hsrc);
    if (!in_place) {
        if (head && !head_graph_set_h(ctx, ctx->d_h)) return fail(ctx, CSVD_ECUDA, "head graph: cannot reset h");
        if (h_dev && h_dev != ctx->d_h)
            CK(cudaMemcpyAsync(ctx->d_h, h_dev, sizeof(double) * ctx->D.d, cudaMemcpyDeviceToDevice, s));
    }
    if ((rc = sync_cfg(ctx, cfg, s))) return rc;
    if (ctx->direct) return launch(ctx, LAUNCH_STEP, s);
    cudaGraphExec_t g = head ? ctx->g_step_head : ctx->g_step;
    if (!g) return fail(ctx, CSVD_ESTATE, "no step graph (an earlier workspace change failed)");
    CK(cudaGraphLaunch(g, s));
    ctx->last_launches = 1;  // one step kernel (it runs the fallback chain itself)
    return 0;
}

extern "C" int csvd_outputs(csvd_ctx *ctx, int64_t **ids_dev, double **logits_dev, csvd_result **res_dev) {
    if (!ctx) return CSVD_ESTATE;
    if (ids_dev) *ids_dev = (int64_t *)ctx->D.S_ids;
    if (logits_dev) *logits_dev = ctx->D.S_logits;
    if (res_dev) *res_dev = ctx->D.res;
    return 0;
}

extern "C" int csvd_step_host(csvd_ctx *ctx, const double *h, const csvd_config *cfg, csvd_result *res, int64_t *ids,
                              double *logits, int64_t cap) {
    if (!ctx || !h || !cfg || !res) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    const int d = ctx->D.d;
    const int64_t first = ctx->first_chunk;
    if ((rc = sync_cfg(ctx, cfg, s))) return rc;
    const bool zc = !ctx->direct && ctx->g_host_head && head_config(cfg) && ctx->h_zero_copy;
    memcpy(zc ? ctx->h_map : ctx->h_pin, h, sizeof(double) * d);
    if (ctx->direct) {
        CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * d, cudaMemcpyHostToDevice, s));
        if ((rc = launch(ctx, LAUNCH_STEP, s))) return rc;
        CK(cudaMemcpyAsync(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->ids_pin, ctx->D.S_ids, sizeof(long long) * first, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->logits_pin, ctx->D.S_logits, sizeof(double) * first, cudaMemcpyDeviceToHost, s));
    } else {
        // zero-copy: the kernel writes ids / logits / result into mapped host
        // memory; busy-poll the stream (no blocking-sync wake-up) and read them
        // once the kernel has completed
        static const bool prof = getenv("CSVD_PROFILE_HOST") != nullptr;
        auto t1 = std::chrono::steady_clock::now();
        ctx->res_map->kind = CSVD_KIND_NONE - 1;  // sentinel: overwritten by the kernel
        cudaGraphExec_t g = (ctx->g_host_head && head_config(cfg)) ? ctx->g_host_head : ctx->g_host;
        if (!g) return fail(ctx, CSVD_ESTATE, "no step graph (an earlier workspace change failed)");
        CK(cudaGraphLaunch(g, s));
        ctx->last_launches = 1;  // one step kernel (it runs the fallback chain itself)
        auto t2 = std::chrono::steady_clock::now();
        cudaError_t q;
        while ((q = cudaStreamQuery(s)) == cudaErrorNotReady) {
        }
        if (q != cudaSuccess) return fail(ctx, CSVD_ECUDA, std::string("step: ") + cudaGetErrorString(q));
        const bool got = ctx->res_map->kind != CSVD_KIND_NONE - 1;
        if (got) {
            if (prof) {
                auto t3 = std::chrono::steady_clock::now();
                auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
                fprintf(stderr, "step host: graph launch %.1f us, wait %.1f us\n", us(t1, t2), us(t2, t3));
            }
            memcpy(res, (const void *)ctx->res_map, sizeof(csvd_result));
            if ((rc = result_error(ctx, *res))) return rc;
            const int64_t n = res->sub_size;
            if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
            if (ids) memcpy(ids, ctx->ids_map, sizeof(int64_t) * n);
            if (logits) memcpy(logits, ctx->logits_map, sizeof(double) * n);
            return 0;
        }
        // the step ended without publishing (device error): read its state
        CK(cudaMemcpy(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost));
        *res = *ctx->res_pin;
        if ((rc = result_error(ctx, *res))) return rc;
        return fail(ctx, CSVD_ESTATE, "step finished without publishing its result");
    }
    CK(cudaStreamSynchronize(s));
    *res = *ctx->res_pin;
    if ((rc = result_error(ctx, *res))) return rc;
    const int64_t n = res->sub_size;
    if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
    if (n > first) {
        CK(cudaMemcpyAsync(ctx->ids_pin + first, ctx->D.S_ids + first, sizeof(long long) * (n - first),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->logits_pin + first, ctx->D.S_logits + first, sizeof(double) * (n - first),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (ids) memcpy(ids, ctx->ids_pin, sizeof(int64_t) * n);
    if (logits) memcpy(logits, ctx->logits_pin, sizeof(double) * n);
    return 0;
}

static void fixed_cfg(csvd_config *cfg, long long V, int slack_f32) {
    memset(cfg, 0, sizeof(*cfg));
    cfg->k = 1;
    cfg->n_targets = 1;
    cfg->epsilon = 0.5;
    cfg->n_levels = 1;
    cfg->level_kind[0] = CSVD_FB_FULL_VOCAB;
    cfg->k_max = V;
    cfg->slack_f32 = slack_f32;
}

extern "C" int csvd_bounds_host(csvd_ctx *ctx, const double *h, int32_t slack_f32, double *values, double *qn,
                                double *slack) {
    if (!ctx || !h) return CSVD_ESTATE;
    if (ctx) ctx->cfg_valid = false;  // this path writes its own config into d_cfg
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    csvd_config fc;
    fixed_cfg(&fc, ctx->D.V, slack_f32);
    int rc;
    if ((rc = stage_pinned_cfg(ctx, ctx->cfg_pin_fixed, fc, s))) return rc;
    memcpy(ctx->h_pin, h, sizeof(double) * ctx->D.d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    if (ctx->direct) {
        CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin_fixed, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
        if ((rc = launch(ctx, LAUNCH_BOUNDS, s))) return rc;
    } else {
        CK(cudaGraphLaunch(ctx->g_bounds, s));
        ctx->last_launches = 1;
    }
    CK(cudaMemcpyAsync(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    if (values) CK(cudaMemcpyAsync(values, ctx->D.U, sizeof(double) * ctx->D.C, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (qn) *qn = ctx->res_pin->query_norm;
    if (slack) *slack = ctx->res_pin->slack;
    return result_error(ctx, *ctx->res_pin);
}

static int dense_async(csvd_ctx *ctx, cudaStream_t s) {
    if (ctx) ctx->cfg_valid = false;  // this path writes its own config into d_cfg
    if (!ctx->D.W) return fail(ctx, CSVD_ECONFIG, "bounds-only context (no table)");
    csvd_config fc;
    fixed_cfg(&fc, ctx->D.V, 0);
    int rc;
    if ((rc = stage_pinned_cfg(ctx, ctx->cfg_pin_fixed, fc, s))) return rc;
    if (ctx->direct) {
        CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin_fixed, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
        return launch(ctx, LAUNCH_DENSE, s);
    }
    CK(cudaGraphLaunch(ctx->g_dense, s));
    ctx->last_launches = 1;
    return 0;
}

extern "C" int csvd_dense_host(csvd_ctx *ctx, const double *h, double *logits) {
    if (!ctx || !h) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    memcpy(ctx->h_pin, h, sizeof(double) * ctx->D.d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    int rc = dense_async(ctx, s);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ctx->logits_pin, ctx->D.S_logits, sizeof(double) * ctx->D.V, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if ((rc = result_error(ctx, *ctx->res_pin))) return rc;
    memcpy(logits, ctx->logits_pin, sizeof(double) * ctx->D.V);
    return 0;
}

extern "C" int csvd_dense_device(csvd_ctx *ctx, const double *h_dev, void *stream) {
    if (!ctx) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    if (h_dev && h_dev != ctx->d_h)
        CK(cudaMemcpyAsync(ctx->d_h, h_dev, sizeof(double) * ctx->D.d, cudaMemcpyDeviceToDevice, s));
    return dense_async(ctx, s);
}

// ---------------------------------------------------------------------------
// shard entry points (sharded_decode_step, shard_sim.py:134-208)
// ---------------------------------------------------------------------------
extern "C" int csvd_shard_open(csvd_ctx *ctx, const double *h, const csvd_config *cfg, double *summary,
                               int64_t *positions, int64_t *ids, double *logits, int64_t cap, int64_t *n_out) {
    if (ctx) ctx->cfg_valid = false;  // this path writes its own config into d_cfg
    if (!ctx || !h || !cfg || !summary || !n_out) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    if (cfg->variant != CSVD_VARIANT_BATCHSELECT) return fail(ctx, CSVD_ECONFIG, "shard opens use batch-select order");
    const Dev &D = ctx->D;
    memcpy(ctx->h_pin, h, sizeof(double) * D.d);
    if ((rc = stage_pinned_cfg(ctx, ctx->cfg_pin, *cfg, s))) return rc;
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * D.d, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    if ((rc = launch(ctx, LAUNCH_SHARD, s))) return rc;
    const int K = D.K;
    ctx->sum_h.resize(CSVD_SH_TOPK + K);
    ctx->order_h.resize(D.C);
    ctx->cum_h.resize(D.C + 1);
    CK(cudaMemcpyAsync(ctx->res_pin, D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->sum_h.data(), D.shard_out, sizeof(double) * (CSVD_SH_TOPK + K), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->order_h.data(), D.order_g, sizeof(int) * D.C, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->cum_h.data(), D.cum_g, sizeof(int) * (D.C + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if ((rc = result_error(ctx, *ctx->res_pin))) return rc;
    const double *sm = ctx->sum_h.data();
    const int p_lo = (int)sm[CSVD_SH_P_LO], p_hi = (int)sm[CSVD_SH_P_HI];
    const long long c_lo = ctx->cum_h[p_lo], c_hi = ctx->cum_h[p_hi];
    const long long nrange = c_hi - c_lo;
    // this shard's tokens of the range, in opening order
    long long n = 0;
    for (int q = p_lo; q < p_hi; ++q)
        if (ctx->owned[ctx->order_h[q]]) n += ctx->cum_h[q + 1] - ctx->cum_h[q];
    *n_out = n;
    memcpy(summary, sm, sizeof(double) * (CSVD_SH_TOPK + cfg->k));
    if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
    if (n == 0 || (!positions && !ids && !logits)) return 0;
    ctx->sids_h.resize(nrange);
    ctx->slog_h.resize(nrange);
    CK(cudaMemcpyAsync(ctx->sids_h.data(), D.S_ids + c_lo, sizeof(long long) * nrange, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->slog_h.data(), D.S_logits + c_lo, sizeof(double) * nrange, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    long long j = 0;
    for (int q = p_lo; q < p_hi; ++q) {
        if (!ctx->owned[ctx->order_h[q]]) continue;
        for (long long r = ctx->cum_h[q]; r < ctx->cum_h[q + 1]; ++r, ++j) {
            if (positions) positions[j] = r;
            if (ids) ids[j] = ctx->sids_h[r - c_lo];
            if (logits) logits[j] = ctx->slog_h[r - c_lo];
        }
    }
    return 0;
}

extern "C" int csvd_shard_dense(csvd_ctx *ctx, const double *h, int32_t k, double *summary, int64_t *ids,
                                double *logits, int64_t cap, int64_t *n_out) {
    if (ctx) ctx->cfg_valid = false;  // this path writes its own config into d_cfg
    if (!ctx || !h || !summary || !n_out) return CSVD_ESTATE;
    if (!ctx->shard) return fail(ctx, CSVD_ECONFIG, "not a shard context");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const Dev &D0 = ctx->D;
    if (k < 1 || k > D0.V) return fail(ctx, CSVD_ECONFIG, "need 1 <= k <= V");
    int rc;
    if (k > D0.K && (rc = csvd_reserve_k(ctx, k))) return rc;
    const Dev &D = ctx->D;
    {
        csvd_config fc;
        fixed_cfg(&fc, D.V, 0);
        fc.k = k;
        if ((rc = stage_pinned_cfg(ctx, ctx->cfg_pin, fc, s))) return rc;
    }
    memcpy(ctx->h_pin, h, sizeof(double) * D.d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * D.d, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    if ((rc = launch(ctx, LAUNCH_DENSE, s))) return rc;
    ctx->sum_h.resize(CSVD_SH_TOPK + D.K);
    CK(cudaMemcpyAsync(ctx->res_pin, D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->sum_h.data(), D.shard_out, sizeof(double) * (CSVD_SH_TOPK + D.K), cudaMemcpyDeviceToHost, s));
    const long long V = D.V;
    CK(cudaMemcpyAsync(ctx->logits_pin, D.S_logits, sizeof(double) * V, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if ((rc = result_error(ctx, *ctx->res_pin))) return rc;
    const long long n = (long long)ctx->local_tokens.size();
    *n_out = n;
    memcpy(summary, ctx->sum_h.data(), sizeof(double) * (CSVD_SH_TOPK + k));
    if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
    for (long long j = 0; j < n; ++j) {
        const long long tok = ctx->local_tokens[j];
        if (ids) ids[j] = tok;
        if (logits) logits[j] = ctx->logits_pin[tok];
    }
    return 0;
}

extern "C" int csvd_info(csvd_ctx *ctx, int64_t *V, int64_t *d, int32_t *C, int32_t *bd, int32_t *wreg, int32_t *breg,
                         int32_t *grid) {
    if (!ctx) return CSVD_ESTATE;
    if (V) *V = ctx->D.V;
    if (d) *d = ctx->D.d;
    if (C) *C = ctx->D.C;
    if (bd) *bd = ctx->D.bd;
    if (wreg) *wreg = ctx->D.wplan.regular;
    if (breg) *breg = ctx->D.bplan.regular;
    if (grid) *grid = ctx->grid;
    return 0;
}

extern "C" int csvd_set_direct(csvd_ctx *ctx, int32_t direct) {
    if (!ctx) return CSVD_ESTATE;
    ctx->direct = direct ? 1 : 0;
    return 0;
}

extern "C" int csvd_l2_flush(csvd_ctx *ctx, void *stream) {
    if (!ctx) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    const size_t bytes = 384ull << 20;
    if (!ctx->flush_buf) {
        CK(cudaMalloc(&ctx->flush_buf, bytes + 64));
        CK(cudaMemset(ctx->flush_buf, 1, bytes));
    }
    k_l2_flush<<<ctx->nsm * 4, 512, 0, s>>>((const uint4 *)ctx->flush_buf, bytes / 16,
                                            (unsigned *)((char *)ctx->flush_buf + bytes));
    CK(cudaGetLastError());
    return 0;
}

extern "C" int csvd_debug_timestamps(csvd_ctx *ctx, unsigned long long *out64) {
    if (!ctx || !ctx->D.dbg) return CSVD_ESTATE;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out64, ctx->D.dbg, (128 + 512) * 8, cudaMemcpyDeviceToHost));
    return 0;
}

extern "C" int csvd_stream(csvd_ctx *ctx, void **stream) {
    if (!ctx || !stream) return CSVD_ESTATE;
    *stream = (void *)ctx->stream;
    return 0;
}

extern "C" int csvd_last_launches(csvd_ctx *ctx, int32_t *n) {
    if (!ctx || !n) return CSVD_ESTATE;
    *n = ctx->last_launches;  // kernels the last entry point launched (graph kernel nodes)
    return 0;
}

// ABI self-check for the ctypes mirrors (tests/test_abi.py)
extern "C" int csvd_test_sizes(int32_t *cfg_size, int32_t *res_size, int32_t *table_size, int32_t *index_size) {
    *cfg_size = (int32_t)sizeof(csvd_config);
    *res_size = (int32_t)sizeof(csvd_result);
    *table_size = (int32_t)sizeof(csvd_table_desc);
    *index_size = (int32_t)sizeof(csvd_index_desc);
    return 0;
}

// ---------------------------------------------------------------------------
// host-only test hook (no GPU needed): the scan state machine with the
// reference's sequential per-prefix arithmetic (tests/test_scan_host.py)
// ---------------------------------------------------------------------------
extern "C" int csvd_test_scan_host(const csvd_config *cfg, int C, long long V, int d, const int *cum, const double *Uo,
                                   const double *lrh, const double *sum_lse, const double *sum_min,
                                   const double *sum_max, const double *sum_topk, int K, const double *S_logits,
                                   int p_sel, csvd_result *res, int *p_final, int *phase_final) {
    ScanState st;
    memset(&st, 0, sizeof(st));
    st.phase = PH_MAIN;
    st.log_z = -INFINITY;
    ScanIn in{cfg, C, V, d, cum, Uo, lrh};
    ScalarSearch search;
    if (cfg->variant == CSVD_VARIANT_BATCHSELECT) st.p_sel = csvd_select_prefix(in, cfg->k_max, search);
    if (p_sel > 0 && p_sel != st.p_sel) return -100;  // selection restatement mismatch
    // per-prefix values, sequential (CertState.merge_cluster, certify.py:73-83)
    std::vector<double> lz(C), kth(C), mn(C), mx(C), rho(C), dl(C);
    std::vector<double> list, merged;
    double log_z = -INFINITY, smin = INFINITY, smax = -INFINITY;
    const int k = cfg->k;
    for (int q = 0; q < C; ++q) {
        const int size = cum[q + 1] - cum[q];
        const int kn = size < k ? size : k;
        merged.clear();
        size_t i = 0, j = 0;
        const double *B = sum_topk + (size_t)q * K;
        while ((int)merged.size() < k && (i < list.size() || (int)j < kn)) {
            if ((int)j >= kn || (i < list.size() && list[i] >= B[j])) merged.push_back(list[i++]);
            else merged.push_back(B[j++]);
        }
        list.swap(merged);
        smin = q == 0 ? sum_min[q] : (sum_min[q] < smin ? sum_min[q] : smin);
        smax = q == 0 ? sum_max[q] : (sum_max[q] > smax ? sum_max[q] : smax);
        const int p = q + 1;
        if (p % 64 == 0) {
            double s = 0.0;
            for (int e = 0; e < cum[p]; ++e) s += exp(S_logits[e] - smax);
            log_z = smax + log(s);
        } else {
            log_z = csvd_logaddexp(log_z, sum_lse[q]);
        }
        lz[q] = log_z;
        kth[q] = ((int)list.size() >= k && cum[p] >= k) ? list[k - 1] : -INFINITY;
        mn[q] = smin;
        mx[q] = smax;
        rho[q] = csvd_rho(log_z, lrh[p]);
        dl[q] = csvd_delta(log_z, lrh[p]);
    }
    csvd_result r;
    memset(&r, 0, sizeof(r));
    Chunk ch{0, C, lz.data(), kth.data(), mn.data(), mx.data(), rho.data(), dl.data()};
    Scan sc{in, st, r};
    sc.run(ch);
    *res = r;
    *p_final = st.p;
    *phase_final = st.phase;
    return 0;
}
