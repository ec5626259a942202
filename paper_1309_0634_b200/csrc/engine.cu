// engine.cu -- the C ABI of include/ss_b200.h and the per-batch pipeline.
//
// Build (see paper_1309_0634_b200/_build.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
//        -Xcompiler -fPIC -cudart static engine.cu -o libss_b200.so
//
// Pipeline of one batch (the loop body of harness.run, harness.py:99-117),
// every kernel a programmatic dependent launch (ss_launch), the whole step
// replayed as a CUDA graph:
//   K2  k_count_rows / k_count / k_key_count   per-chunk group histograms
//                                              (count_batch; int64 keys probed)
//       k_batch_stats*   gcount, gkept (never-stored runs dropped), tpt
//   K7  k_balance        policy on a side stream, overlapped with the rest;
//       k_split_*        hot-key split plan from the batch's own counts
//       k_scan_*         run starts (+ digit bases / live-chunk list)
//       k_reserve        grow occupancy-proportional rings (sparse store)
//   K3  k_rank_place     single-pass stable placement (G <= 2^14; few live
//                        chunks: sub-chunks via k_sub_hist / k_sub_scan), or
//       k_sort_pass      radix passes over the live chunks (G <= 2^17), or
//       k_os_*           look-back-free LSD passes (G >= 2^18)
//   K4  k_ingest         partition-parallel window exchange (+ split shares)
//   K5  k_finalize       fold deltas into the state, result rows;
//       k_mm_* / k_minmax_rescan   MIN/MAX of partially evicted windows
//       k_emit_host      rows into pinned host memory (streaming use)
//       k_apply_*        apply the policy's moves (in force from batch t+1)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ss_b200.h"
#include "common.cuh"
#include "partition.cuh"
#include "window.cuh"
#include "balance.cuh"
#include "split.cuh"
#include "keys.cuh"
#include "bucket.cuh"
#include "radix.cuh"
#include "trace.cuh"
#include "streamwin.cuh"

using namespace ss;

// every kernel launch of the library goes through `ss_note_launch(), k<<<...>>>`
// so the benchmark can report how many of our kernels ran (ss_launch_count)
static std::atomic<long long> g_launches{0};
static inline void ss_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// every launch: programmatic stream serialisation (SS_PDL_ENTRY in each
// kernel), so a kernel's launch and CTA rasterisation overlap the tail of
// its predecessor; SS_B200_NO_PDL=1 launches plainly (A/B)
static const bool g_pdl = !(getenv("SS_B200_NO_PDL") && getenv("SS_B200_NO_PDL")[0] == '1');
template <typename... KArgs, typename... Args>
static inline void ss_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    static_assert(sizeof...(KArgs) == sizeof...(Args), "every kernel argument is passed explicitly");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

namespace {

constexpr int64_t kCountChunk = 16384;
constexpr int64_t kDenseLimitBytes = int64_t(24) << 30;

struct DevReport {            // written by report_body (window.cuh) as 64-bit words, copied to the host
    unsigned long long bad;
    long long tuples;
    long long imbalance;
    long long moves;
    long long moves_before;
    long long scanned;
    long long max_load;
    long long touched;
    long long split_groups;
    long long n_res;
    long long load_sum;      // sum of the per-block loads max_load is taken over
    int oom;
    int pad;
};

// one emission buffer: columns are null when the aggregate is not configured
struct HostRows {
    int32_t* g;
    int32_t* cnt;
    long long* sum;
    double* avg;
    int32_t* mn;
    int32_t* mx;
    unsigned long long* hdr;    // [0] rows, [1] first bad tuple (kNoBad if none), [2] its group
};

}  // namespace

struct ss_engine {
    ss_config cfg{};
    int64_t G = 0, W = 0;
    int P = 0;
    bool dense = true;
    bool minmax = false;
    cudaStream_t st = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_stats = nullptr, ev_bal = nullptr;
    std::string err;

    // window store
    int32_t *fill = nullptr, *next_pos = nullptr, *mn = nullptr, *mx = nullptr, *cap = nullptr;
    long long* wsum = nullptr;
    int64_t* off = nullptr;
    int32_t* ring = nullptr;
    unsigned long long pool_cap = 0;
    unsigned long long* pool_top = nullptr;
    int* oom = nullptr;

    // assignment
    int32_t *pmap = nullptr, *order = nullptr, *offsets = nullptr, *new_order = nullptr, *new_off = nullptr;
    uint8_t* moved = nullptr;

    // batch scratch
    int64_t S = 0, max_batch = 0;
    int n_sub_max = 0;
    uint32_t* stage_keys = nullptr;
    int32_t* stage_vals = nullptr;
    int32_t *gcnt = nullptr, *gstart = nullptr, *gcount = nullptr, *bsum = nullptr;
    int32_t* gkept = nullptr;              // kept (possibly stored) tuples of each group in the batch
    int32_t* gpre = nullptr;               // [chunk][g] kept-count prefix over chunks (single-pass placement)
    int32_t* gsub = nullptr;               // [unit][g] sub-chunk prefixes (few live chunks)
    int32_t* subh = nullptr;               // [unit][g] sub-chunk counts
    int* sub_shift = nullptr;              // device: sub-chunks per live chunk = 2^sub_shift
    uint32_t* pwork = nullptr;             // per-partition window-update work of the batch (k_batch_stats)
    int* any_dead = nullptr;               // some tuple of the batch is never stored (set by k_batch_stats)
    int4* cta_map = nullptr;               // work-proportional K4 grid: slot of every CTA
    int* cta_used = nullptr;
    bool rank_place = false;               // G <= kRankMaxG: k_rank_place instead of the radix passes
    bool bucket = false;                   // G > kRankMaxG: bucketed two-pass placement (bucket.cuh)
    BucketArgs bk{};
    // G > kRankMaxG: look-back-free 7-bit LSD passes (radix.cuh)
    bool os = false;
    int os_digit = kOsBitsWide;            // digit width: kOsBitsWide (measured best: C4 0.42 ms vs 0.49 with 7 bits)
    int os_match = 1;                      // ranking: ballot matches (0), alternating with MATCH (1), MATCH (2)
    bool os2 = true;                       // 10-bit passes: 512-thread, 2-CTA-per-SM variant (measured +2.6 % at C4,
                                           // +3 % at C5 over the 1024-thread double-buffered kernel; SS_B200_OS2=0: A/B)
    int os_npass = 0, os_shift[kOsMaxPass] = {0, 0, 0, 0}, os_bits[kOsMaxPass] = {0, 0, 0, 0};
    uint32_t* os_hist = nullptr;
    uint32_t* os_bsum = nullptr;
    uint32_t* os_dtot = nullptr;
    // where the placement left the kept values (and, in trace mode, keys)
    int32_t* vals_final = nullptr;
    uint32_t* keys_final = nullptr;
    int32_t* n_live = nullptr;             // kept tuples of the batch (device)
    uint32_t* chunk_live = nullptr;        // live-chunk bitmap
    int32_t *lc = nullptr, *n_lc = nullptr;   // ordered live-chunk list
    uint32_t *chunk_h = nullptr, *chunk_base = nullptr;   // first-pass digit histograms / bases per live chunk
    int32_t* btile = nullptr;              // second-pass tile prefix over first-pass buckets
    long long* bdelta = nullptr;           // per-group batch delta
    int32_t *bmin = nullptr, *bmax = nullptr;
    unsigned long long* part_work = nullptr;
    RingCopy* copies = nullptr;            // ring growth copies (sparse store)
    unsigned* n_copies = nullptr;
    int32_t *hot_of = nullptr, *hot_g = nullptr;   // count-kernel hot cache (large G)
    int* n_hot_dev = nullptr;
    bool side_pending = false;             // policy/apply of the last batch still on the side stream
    cudaEvent_t ev_k4 = nullptr, ev_apply = nullptr;
    uint32_t* dhist = nullptr;
    unsigned long long *tpt = nullptr, *touched = nullptr, *bad = nullptr;
    uint32_t* kbuf = nullptr;
    int32_t* vbuf[2] = {nullptr, nullptr};
    int64_t sort_cap = 0;
    unsigned long long* status = nullptr;
    int64_t status_tiles = 0;
    uint32_t* tickets = nullptr;
    uint32_t* ep_dev = nullptr;            // look-back epoch (device; bumped per placement)
    DigitPlan plan{};
    int rb[2] = {0, 0};
    int nblk = 0;

    // balancer
    int cap_moves = 0;
    int4* moves = nullptr;
    int *front_top = nullptr, *back_first = nullptr, *mv_next = nullptr, *n_moves = nullptr;
    int32_t *keep_at = nullptr, *mv_pos = nullptr;   // list layout of the fused step's apply
    long long *scanned = nullptr, *final_tpt = nullptr;
    int* prev_moves = nullptr;

    uint32_t* kbuf2 = nullptr;             // sorted keys (reorder only)

    // int64 keys (key_bits == 64): key -> dense slot table
    bool keys64 = false;
    bool pre_counted = false;     // this batch was counted by the int64 key probe
    int key_agg = 0;              // warp-aggregated cold-key atomics in the probe + count (A/B: SS_B200_KEY_AGG; one atomic per cold tuple measured 3% faster at C4, 15.24 -> 15.76 G tuples/s: cold keys rarely repeat inside a warp)
    KeyTable kt{};
    long long* stage_keys64 = nullptr;

    // streaming input (ss_step / ss_step_keys64 with host buffers): the next
    // batch's H2D runs on a copy stream into the other staging buffer while
    // the current batch computes; a buffer is reused once the batch that
    // read it has finished its first placement pass
    cudaStream_t cp = nullptr;
    cudaEvent_t ev_staged[2] = {nullptr, nullptr}, ev_freed[2] = {nullptr, nullptr};
    bool freed_rec[2] = {false, false};
    int stg_next = 0, cur_stage = -1;
    uint32_t* skeys[2] = {nullptr, nullptr};
    int32_t* svals[2] = {nullptr, nullptr};
    long long* sk64[2] = {nullptr, nullptr};
    uint2* srec[2] = {nullptr, nullptr};      // replay records (ss_step_records)

    // host emission: each batch's rows (group + the configured aggregates)
    // written by a kernel straight into mapped pinned host memory
    // (double-buffered); h_emit[b] are the host views, d_emit[b] the
    // device aliases of the same pages
    bool host_emit = false;
    HostRows h_emit[2]{}, d_emit[2]{};
    cudaEvent_t ev_emit[2] = {nullptr, nullptr};
    long long emit_seq = 0, pull_seq = 0;

    // CUDA graphs of the fused step: one per (inputs, n, balancer, plan /
    // emission / staging parity); replays skip the per-launch host and GPU
    // front-end cost of ~15 kernels and memsets per batch
    const uint32_t* last_keys = nullptr;   // the last step's keys (names the bad tuple of a DataError)
    // stream-scope window (scope = 1): ring of the stream's
    // last W tuples; fill / wsum / mn / mx hold per-group COUNT / SUM / MIN / MAX
    bool stream_scope = false;
    uint32_t* sw_k = nullptr;
    int32_t* sw_v = nullptr;
    uint8_t* sw_touched = nullptr;
    long long* sw_cur = nullptr;           // device ring cursors (head, fill), see streamwin.cuh
    // per-tuple trace mode: no dead-tuple dropping, placed
    // groups kept, trace sums per placed tuple
    bool trace_on = false;
    long long* trace_s = nullptr;
    SegVal* trace_tile = nullptr;
    bool capturing = false;
    bool graphs_on = true;
    long long graph_hits = 0, graph_captures = 0;
    struct GraphEntry {
        const void* dk;
        const void* dv;
        int64_t n;
        ss_balancer bal;
        int plan_cur, plan_valid, emit_b, host_emit, stage, pre_counted;
        const void* gcnt;          // count rows the graph reads (alternating when the count is pipelined)
        cudaGraphExec_t exec;
        long long launches;
    };
    std::vector<GraphEntry> graphs;
    int32_t* kbsum = nullptr;

    // multi-GPU routing: group -> owning GPU
    int32_t* owner = nullptr;
    int n_dest = 0;
    unsigned long long* route_cnt = nullptr;   // [16]
    uint32_t* route_base = nullptr;            // [16]
    unsigned* fin_ticket = nullptr;            // k_finalize CTAs done (report fold)
    // int64 keys: the probe + count of batch t+1 on its own stream (kst)
    cudaStream_t kst = nullptr;
    cudaEvent_t ev_keys[2] = {nullptr, nullptr}, ev_fin[2] = {nullptr, nullptr}, ev_hot = nullptr;
    bool fin_rec[2] = {false, false}, hot_rec = false;
    bool key_pipe_dev = false;                 // device key inputs are ready when passed (ss_set_key_pipeline)
    bool inputs_on_stream = false;             // this step's device inputs are engine-stream work (records)
    // "ahead" mode (u32, G <= 2^14, single-pass placement, no policy or
    // split): count + statistics + scans + sub-chunk prefixes of batch t+1
    // run on the count stream while batch t places and updates windows;
    // the per-batch arrays they write alternate
    bool ahead_ok = false, ahead = false;
    struct AheadSet {
        int32_t *gcount, *gkept, *gpre, *gstart, *n_live, *lc, *n_lc, *gsub;
        int* sub_shift;
        unsigned long long *tpt, *touched;
    } aset[2] = {};
    cudaEvent_t ev_in = nullptr;
    int32_t* gcnt_buf[2] = {nullptr, nullptr};
    uint32_t* skeys_buf[2] = {nullptr, nullptr};
    unsigned long long* key_bad = nullptr;
    int kpar = 0;
    int32_t* bowner = nullptr;                 // int64 keys across GPUs: bucket -> GPU [kKeyBuckets]
    int32_t* bdst = nullptr;                   // moved bucket -> destination (export), -1 else
    int2* mig64 = nullptr;                     // exported (slot, destination) [kMig64Max]
    longlong4* mig64_copies = nullptr;         // their ring images (ring offset, blob word, span) [kMig64Max]
    int* n_mig64 = nullptr;
    int32_t* rec_vals = nullptr;               // attrs of a received int64-key record batch
    longlong4* mig_list = nullptr;             // [kMigMax] (ring offset, blob word, span, -) of exported groups
    int* mig_n = nullptr;

    // hot-key split plans (split.cuh), double-buffered: plan[cur] executes
    // batch t while the planner writes plan[cur ^ 1] for batch t+1
    SplitPlan plan_buf[2]{};
    SplitScratch spx{};
    int plan_cur = 0;
    bool plan_valid = false;
    int last_plan = -1;        // plan buffer the last batch executed with
    int maxS = 0, maxSh = 0;

    // emission / misc
    unsigned* n_res = nullptr;
    int32_t *r_g = nullptr, *r_cnt = nullptr, *r_mn = nullptr, *r_mx = nullptr;
    long long* r_sum = nullptr;
    double* r_avg = nullptr;
    int32_t* bal_ecnt = nullptr;           // k_bal_prep output (large G)
    uint8_t* bal_eflag = nullptr;
    int4* rescan = nullptr;
    unsigned* n_rescan = nullptr;
    // MIN/MAX chunk summaries of full windows (W > kMMSumMinW)
    int32_t* sum_idx = nullptr;
    uint8_t* sum_valid = nullptr;
    int* n_sum = nullptr;
    int2* sums = nullptr;
    unsigned long long* part_ns = nullptr;
    unsigned long long* loads = nullptr;   // per-partition load incl. split shares
    long long* fill_loads = nullptr;       // split planner: cold loads of the batch
    DevReport* d_rep = nullptr;
    DevReport* h_rep = nullptr;            // pinned
    unsigned long long* alg_bytes = nullptr;
    long long alg_input = 0;
    std::vector<void*> allocs;

    // kernel-class timing (bench.py)
    struct ProfPair { int cls; cudaEvent_t a, b; };
    bool prof = false;
    std::vector<ProfPair> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[SS_K_NCLASS] = {0};
    int64_t prof_n[SS_K_NCLASS] = {0};
};

namespace {
// NVTX ranges on the host timeline of a profiler (nsys / ncu --nvtx): the
// public entry points and every kernel class of a step, named as in
// DESIGN.md.  Enabled by SS_B200_NVTX=1 (header-only NVTX3: without a tool
// attached a push is one branch).
static const bool g_nvtx = getenv("SS_B200_NVTX") && getenv("SS_B200_NVTX")[0] == '1';
struct NvtxRange {
    bool on;
    explicit NvtxRange(const char* name) : on(g_nvtx) { if (on) nvtxRangePushA(name); }
    ~NvtxRange() { if (on) nvtxRangePop(); }
};
static const char* const kClassName[SS_K_NCLASS] = {"ss count", "ss stats+scan", "ss placement", "ss window update",
                                                     "ss finalize+emit", "ss apply moves", "ss policy / split plan"};

struct ProfScope {
    ss_engine* e;
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    NvtxRange nv;
    ProfScope(ss_engine* e_, int c, cudaStream_t st) : e(e_), cls(c), s(st), nv(kClassName[c]) {
        if (!e->prof) return;
        a = take();
        cudaEventRecord(a, s);
    }
    cudaEvent_t take() {
        if (e->ev_pool.empty()) {
            cudaEvent_t x;
            cudaEventCreate(&x);
            return x;
        }
        cudaEvent_t x = e->ev_pool.back();
        e->ev_pool.pop_back();
        return x;
    }
    ~ProfScope() {
        if (!e->prof) return;
        cudaEvent_t b = take();
        cudaEventRecord(b, s);
        e->prof_pending.push_back({cls, a, b});
    }
};
}  // namespace

// --------------------------------------------------------------------------
// helpers
// --------------------------------------------------------------------------
namespace {

int fail(ss_engine* e, int code, const std::string& msg) {
    if (e) e->err = msg;
    return code;
}

#define SS_CUDA(e, call)                                                              \
    do {                                                                              \
        cudaError_t _st = (call);                                                     \
        if (_st != cudaSuccess)                                                       \
            return fail((e), SS_E_EXEC, std::string(#call ": ") + cudaGetErrorString(_st)); \
    } while (0)

template <typename T>
int dalloc(ss_engine* e, T** p, size_t n) {
    void* q = nullptr;
    cudaError_t st = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
    if (st != cudaSuccess)
        return fail(e, SS_E_EXEC, std::string("cudaMalloc(") + std::to_string(n * sizeof(T)) + "): " +
                                      cudaGetErrorString(st));
    e->allocs.push_back(q);
    *p = (T*)q;
    return SS_OK;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// the device policy loop: one CTA; G <= kBalStageG stages the entry lists
// and counts in shared memory when they fit next to the per-partition state
constexpr size_t kBalSmemMax = 200 * 1024;   // dynamic shared memory opted in for k_balance
static void launch_balance(ss_engine* e, BalanceArgs& a, cudaStream_t st) {
    a.G = (int)e->G;
    const bool staged = e->G <= kBalStageG && bal_smem_bytes(e->P, (int)e->G, true) <= kBalSmemMax;
    if (staged) {
        ss_launch(k_balance<true>, 1, kBalThreads, bal_smem_bytes(e->P, (int)e->G, true), st, a);
    } else if (a.policy == SS_POLICY_ALL || a.policy == SS_POLICY_PROB || a.policy == SS_POLICY_BEST) {
        // donor scans over the whole CTA, from position-ordered counts / flags
        a.ecnt = e->bal_ecnt;
        a.eflag = e->bal_eflag;
        ss_note_launch(), ss_launch(k_bal_prep, 2 * kNumSM, 256, 0, st, a);
        ss_launch(k_balance<false, true>, 1, kBalThreads, bal_smem_bytes(e->P, (int)e->G, false), st, a);
    } else {
        ss_launch(k_balance<false>, 1, kBalThreads, bal_smem_bytes(e->P, (int)e->G, false), st, a);
    }
}

// single-pass placement kernel for keys < 2^bits (ballot matching)
using RankKernel = void (*)(const uint32_t*, const int32_t*, uint32_t*, int32_t*, int64_t, int, const int32_t*,
                            const int32_t*, const int32_t*, const int32_t*, uint32_t, const int32_t*,
                            const unsigned long long*, const int*, const int32_t*);
// grid of a per-group kernel (a thread per group and round): one group per
// thread up to 16 CTAs per SM -- G = 1M groups on 2 x 148 CTAs left each
// thread a chain of ~13 dependent load rounds (k_finalize 47 us at C4)
static unsigned group_grid(int64_t G) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((G + 255) / 256, 16 * kNumSM));
}
static RankKernel rank_kernel(int bits) {
    switch (bits) {
        case 0: case 1: case 2: case 3: case 4: case 5: case 6: case 7: case 8: return k_rank_place<8>;
        case 9: return k_rank_place<9>;
        case 10: return k_rank_place<10>;
        case 11: return k_rank_place<11>;
        case 12: return k_rank_place<12>;
        case 13: return k_rank_place<13>;
        default: return k_rank_place<14>;
    }
}

int bits_for(int64_t G) {
    int b = 1;
    while ((int64_t(1) << b) < G) ++b;
    return b;
}

int rb_for(int bits) { return bits < 4 ? 4 : (bits > 11 ? 11 : bits); }

template <int RB>
void launch_sort(cudaStream_t st, const uint32_t* kin, const int32_t* vin, uint32_t* kout, int32_t* vout,
                 int n, int shift, uint32_t mask, const uint32_t* base, unsigned long long* status,
                 const uint32_t* ep_dev, uint32_t ep_off, uint32_t* ticket, const unsigned long long* bad, int stream_in,
                 const int32_t* n_dev, const SortSeg* sg) {
    // mode 2 adds up to one partial tile per bucket
    const int tiles = (n + kSortTile - 1) / kSortTile + (sg && sg->mode == 2 ? sg->nb : 0);
    if (tiles == 0) return;
    // persistent: at most the co-resident CTAs (2 per SM), each looping over tickets
    ss_note_launch(), ss_launch(k_sort_pass<RB>, std::min(tiles, 2 * kNumSM), kSortThreads, SortSmem<RB>::bytes, st, kin, vin, kout, vout, n, shift, mask, base, status, ep_dev, ep_off, ticket, bad, stream_in, nullptr, n_dev,
        sg ? *sg : SortSeg{});
}

void sort_dispatch(int rb, cudaStream_t st, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                   int32_t* vout, int n, int shift, uint32_t mask, const uint32_t* base,
                   unsigned long long* status, const uint32_t* ep_dev, uint32_t ep_off, uint32_t* ticket,
                   const unsigned long long* bad, int stream_in, const int32_t* n_dev = nullptr,
                   const SortSeg* sg = nullptr) {
#define SS_SORT_CASE(R) launch_sort<R>(st, kin, vin, kout, vout, n, shift, mask, base, status, ep_dev, ep_off, ticket, bad, \
                                       stream_in, n_dev, sg)
    switch (rb) {
        case 4: SS_SORT_CASE(4); break;
        case 5: SS_SORT_CASE(5); break;
        case 6: SS_SORT_CASE(6); break;
        case 7: SS_SORT_CASE(7); break;
        case 8: SS_SORT_CASE(8); break;
        case 9: SS_SORT_CASE(9); break;
        case 10: SS_SORT_CASE(10); break;
        default: SS_SORT_CASE(11); break;
    }
#undef SS_SORT_CASE
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_dense_off(int64_t* off, int32_t* cap, int64_t G, int64_t W) { SS_PDL_ENTRY();
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
        off[g] = g * W;
        cap[g] = (int32_t)W;
    }
}
__global__ void k_set_bad(unsigned long long* bad) { SS_PDL_ENTRY(); *bad = (unsigned long long)kNoBad; }
__global__ void k_epoch_bump(uint32_t* ep) { SS_PDL_ENTRY(); *ep = epoch_next(*ep); }
// replay records (u32 group, i32 attr; datagen.py REPLAY_DTYPE) -> SoA keys / values
__global__ void k_deinterleave(const uint4* __restrict__ rec, int64_t n, uint32_t* __restrict__ keys,
                               int32_t* __restrict__ vals) { SS_PDL_ENTRY();
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = ld_stream_v4(rec + i);
        reinterpret_cast<uint2*>(keys)[i] = make_uint2(r.x, r.z);
        reinterpret_cast<int2*>(vals)[i] = make_int2((int)r.y, (int)r.w);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint2 last = reinterpret_cast<const uint2*>(rec)[n - 1];
        keys[n - 1] = last.x;
        vals[n - 1] = (int32_t)last.y;
    }
}
// the batch's rows (group + configured aggregate columns) into mapped
// pinned host memory (PCIe writes).  The header carries the row count and,
// for a rejected batch, the first bad tuple and its group, so the host
// raises DataError when it pulls that batch.
__global__ void k_emit_host(const unsigned* __restrict__ n_res, const unsigned long long* __restrict__ bad,
                            const uint32_t* __restrict__ keys, long long n_keys, const int32_t* __restrict__ g,
                            const int32_t* __restrict__ cnt, const long long* __restrict__ sum,
                            const double* __restrict__ avg, const int32_t* __restrict__ mn,
                            const int32_t* __restrict__ mx, HostRows h) { SS_PDL_ENTRY();
    const unsigned long long b = *bad;
    const unsigned n = (b == (unsigned long long)kNoBad) ? *n_res : 0u;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        h.g[i] = g[i];
        if (h.cnt) h.cnt[i] = cnt[i];
        if (h.sum) h.sum[i] = sum[i];
        if (h.avg) h.avg[i] = avg[i];
        if (h.mn) h.mn[i] = mn[i];
        if (h.mx) h.mx[i] = mx[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        h.hdr[0] = n;
        h.hdr[1] = b;
        h.hdr[2] = (b < (unsigned long long)n_keys) ? (unsigned long long)keys[b] : 0ull;
    }
}
__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_u64_to_i64(const unsigned long long* a, long long* b, int n) { SS_PDL_ENTRY();
    for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = (long long)a[i];
}

// map group ids to placement ranks (reorder_batch sorts by rank)
__global__ void k_to_rank(const uint32_t* __restrict__ g, int64_t n, const int32_t* __restrict__ rank,
                          uint32_t G, uint32_t* __restrict__ out, unsigned long long* bad) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = g[i];
        if (v >= G) {
            atomicMin(bad, (unsigned long long)i);
            out[i] = 0;
        } else {
            out[i] = (uint32_t)rank[v];
        }
    }
}
__global__ void k_rank_of(const int32_t* __restrict__ order, int64_t G, int32_t* __restrict__ rank) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x)
        rank[order[i]] = (int32_t)i;
}
__global__ void k_from_rank(uint32_t* __restrict__ k, int64_t n, const int32_t* __restrict__ order) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        k[i] = (uint32_t)order[k[i]];
}
__global__ void k_clear_moved(const int4* __restrict__ moves, const int* __restrict__ n_moves, uint8_t* moved) { SS_PDL_ENTRY();
    const int n = *n_moves;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) moved[moves[i].x] = 0;
}

// load monitor (K6): imbalance of the entry loads, max per-block load
// including split shares, and the report the host reads back.
__global__ void __launch_bounds__(1024)
k_report(ReportArgs a) { SS_PDL_ENTRY();
    report_body(a);
}

}  // namespace

static int join_side(ss_engine* e);
static int create_count_pipe(ss_engine* e);

// --------------------------------------------------------------------------
// lifecycle
// --------------------------------------------------------------------------
extern "C" const char* ss_version(void) { return "ss_b200 1.0 (sm_100a)"; }

#ifdef SS_K4_PROF
extern "C" int ss_debug_k4_prof(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_k4_prof, 8 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_k4_prof, z, sizeof(z));
    }
    return 0;
}
#endif
#ifdef SS_SORT_PROF
// experiment builds only: clock64 cycles per placement-tile phase, summed over CTAs
extern "C" int ss_debug_sort_prof(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_sort_prof, 8 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_sort_prof, z, sizeof(z));
    }
    return 0;
}
#endif

extern "C" int ss_set_graphs(ss_engine* e, int enable) {
    if (!e) return SS_E_CONFIG;
    e->graphs_on = enable != 0;
    return SS_OK;
}

extern "C" long long ss_sub_batch(ss_engine* e) { return e ? (long long)e->S : 0; }

extern "C" long long ss_launch_count(int reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}

extern "C" const char* ss_last_error(ss_engine* e) { return e ? e->err.c_str() : "null engine"; }

extern "C" void ss_destroy(ss_engine* e) {
    if (!e) return;
    cudaSetDevice(e->cfg.device);
    cudaStreamSynchronize(e->st);
    if (e->cp) cudaStreamSynchronize(e->cp);
    if (e->kst) cudaStreamSynchronize(e->kst);
    for (auto& g : e->graphs) cudaGraphExecDestroy(g.exec);
    for (void* p : e->allocs) cudaFree(p);
    if (e->h_rep) cudaFreeHost(e->h_rep);
    for (int b = 0; b < 2; ++b) {
        for (void* q : {(void*)e->h_emit[b].g, (void*)e->h_emit[b].cnt, (void*)e->h_emit[b].sum,
                        (void*)e->h_emit[b].avg, (void*)e->h_emit[b].mn, (void*)e->h_emit[b].mx,
                        (void*)e->h_emit[b].hdr})
            if (q) cudaFreeHost(q);
        if (e->ev_staged[b]) cudaEventDestroy(e->ev_staged[b]);
        if (e->ev_freed[b]) cudaEventDestroy(e->ev_freed[b]);
        if (e->ev_emit[b]) cudaEventDestroy(e->ev_emit[b]);
    }
    for (int b = 0; b < 2; ++b) {
        if (e->ev_keys[b]) cudaEventDestroy(e->ev_keys[b]);
        if (e->ev_fin[b]) cudaEventDestroy(e->ev_fin[b]);
    }
    if (e->ev_hot) cudaEventDestroy(e->ev_hot);
    if (e->ev_in) cudaEventDestroy(e->ev_in);
    if (e->kst) cudaStreamDestroy(e->kst);
    if (e->cp) cudaStreamDestroy(e->cp);
    if (e->side) cudaStreamDestroy(e->side);
    if (e->ev_stats) cudaEventDestroy(e->ev_stats);
    if (e->ev_bal) cudaEventDestroy(e->ev_bal);
    if (e->st && e->cfg.reserved == 0) cudaStreamDestroy(e->st);
    delete e;
}

static int engine_alloc_sort(ss_engine* e, int64_t n) {
    if (n <= e->sort_cap) return SS_OK;
    const int64_t cap = ((n + kSortTile - 1) / kSortTile) * kSortTile;
    int rc;
    if ((rc = dalloc(e, &e->kbuf, cap))) return rc;
    if ((rc = dalloc(e, &e->kbuf2, cap))) return rc;
    if ((rc = dalloc(e, &e->vbuf[0], cap))) return rc;
    if ((rc = dalloc(e, &e->vbuf[1], cap))) return rc;
    e->status_tiles = cap / kSortTile + kMaxBins;   // + one partial tile per bucket (SortSeg mode 2)
    if ((rc = dalloc(e, &e->status, (size_t)e->status_tiles * kMaxBins))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->status, 0, sizeof(unsigned long long) * e->status_tiles * kMaxBins, e->st));
    e->sort_cap = cap;
    return SS_OK;
}

extern "C" int ss_create(const ss_config* cfg, ss_engine** out) {
    if (!cfg || !out) return SS_E_CONFIG;
    *out = nullptr;
    ss_engine* e = new ss_engine();
    e->cfg = *cfg;
    e->cfg.reserved = 0;
    if (cfg->n_groups < 1 || cfg->n_groups > (int64_t(1) << 22)) {
        int rc = fail(e, SS_E_CONFIG, "n_groups must be in [1, 2^22]");
        *out = e;
        return rc;
    }
    if (cfg->window < 1 || cfg->window > (int64_t(1) << 30)) {
        int rc = fail(e, SS_E_CONFIG, "window must be in [1, 2^30]");
        *out = e;
        return rc;
    }
    if (cfg->max_batch > (int64_t(1) << 30)) {
        // batch ranks, ring positions and window fills are summed in 32 bits
        int rc = fail(e, SS_E_CONFIG, "max_batch must be <= 2^30");
        *out = e;
        return rc;
    }
    if (cfg->n_partitions < 1 || cfg->n_partitions > 4096) {
        int rc = fail(e, SS_E_CONFIG, "n_partitions must be in [1, 4096]");
        *out = e;
        return rc;
    }
    *out = e;
    e->G = cfg->n_groups;
    e->W = cfg->window;
    e->P = cfg->n_partitions;
    e->minmax = (cfg->agg_mask & (SS_AGG_MIN | SS_AGG_MAX)) != 0;
    SS_CUDA(e, cudaSetDevice(cfg->device));
    SS_CUDA(e, cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking));
    SS_CUDA(e, cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_stats, cudaEventDisableTiming));
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_bal, cudaEventDisableTiming));
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_k4, cudaEventDisableTiming));
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_apply, cudaEventDisableTiming));
    SS_CUDA(e, cudaStreamCreateWithFlags(&e->cp, cudaStreamNonBlocking));
    if (const char* ng = getenv("SS_B200_NO_GRAPHS")) e->graphs_on = !(ng[0] && ng[0] != '0');
    for (int b = 0; b < 2; ++b) {
        SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_staged[b], cudaEventDisableTiming));
        SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_freed[b], cudaEventDisableTiming));
        SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_emit[b], cudaEventDisableTiming));
    }

    const int64_t G = e->G, W = e->W;
    int rc;
    // -- window store
    if ((rc = dalloc(e, &e->fill, G)) || (rc = dalloc(e, &e->next_pos, G)) || (rc = dalloc(e, &e->wsum, G)) ||
        (rc = dalloc(e, &e->mn, G)) || (rc = dalloc(e, &e->mx, G)) || (rc = dalloc(e, &e->cap, G)) ||
        (rc = dalloc(e, &e->off, G)) || (rc = dalloc(e, &e->pool_top, 1)) || (rc = dalloc(e, &e->oom, 1)) ||
        (rc = dalloc(e, &e->n_copies, 1)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->fill, 0, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->next_pos, 0, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->wsum, 0, G * 8, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->mn, 0, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->mx, 0, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->oom, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->pool_top, 0, 8, e->st));
    e->stream_scope = cfg->scope == 1;
    if (cfg->scope != 0 && cfg->scope != 1) {
        *out = e;
        return fail(e, SS_E_CONFIG, "scope must be 0 (per-group window) or 1 (stream window)");
    }
    if (e->stream_scope) {
        if ((rc = dalloc(e, &e->sw_k, W)) || (rc = dalloc(e, &e->sw_v, W)) || (rc = dalloc(e, &e->sw_touched, G)) ||
            (rc = dalloc(e, &e->sw_cur, 2)))
            return rc;
        SS_CUDA(e, cudaMemsetAsync(e->sw_touched, 0, G, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->sw_k, 0, W * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->sw_v, 0, W * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->sw_cur, 0, 2 * 8, e->st));
    }
    // a stream-scope engine keeps no per-group rings (a token pool)
    const int64_t dense_vals = e->stream_scope ? 16 : G * W;
    e->dense = cfg->pool_values == 0 && dense_vals * 4 <= kDenseLimitBytes && !e->stream_scope;
    if (e->dense) {
        e->pool_cap = (unsigned long long)dense_vals;
        if ((rc = dalloc(e, &e->ring, dense_vals))) return rc;
        ss_note_launch(), ss_launch(k_dense_off, 296, 256, 0, e->st, e->off, e->cap, G, W);
    } else {
        int64_t pool = e->stream_scope ? 16 : cfg->pool_values;
        if (pool <= 0) {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            pool = std::min<int64_t>((int64_t)(fr / 4 / 2), int64_t(16) << 30);   // <= 64 GB of 180
            pool = std::min<int64_t>(pool, dense_vals);
        }
        e->pool_cap = (unsigned long long)pool;
        if ((rc = dalloc(e, &e->ring, pool))) return rc;
        SS_CUDA(e, cudaMemsetAsync(e->off, 0, G * 8, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->cap, 0, G * 4, e->st));
        // growth copies are listed in kCopyChunk pieces: at most one partial
        // piece per group plus the pool's worth of full pieces
        if ((rc = dalloc(e, &e->copies, G + pool / kCopyChunk + 1))) return rc;
    }
    // -- assignment: contiguous ranges (partition.py:97-114) until set
    if ((rc = dalloc(e, &e->pmap, G)) || (rc = dalloc(e, &e->order, G)) || (rc = dalloc(e, &e->new_order, G)) ||
        (rc = dalloc(e, &e->offsets, e->P + 1)) || (rc = dalloc(e, &e->new_off, e->P + 1)) ||
        (rc = dalloc(e, &e->moved, G)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->moved, 0, G, e->st));
    {
        std::vector<int32_t> order(G), pmap(G);
        std::vector<int32_t> offs(e->P + 1);
        const int64_t q = G / e->P, r = G % e->P;
        int64_t lo = 0;
        for (int t = 0; t < e->P; ++t) {
            offs[t] = (int32_t)lo;
            const int64_t sz = q + (t < r ? 1 : 0);
            for (int64_t g = lo; g < lo + sz; ++g) { order[g] = (int32_t)g; pmap[g] = t; }
            lo += sz;
        }
        offs[e->P] = (int32_t)G;
        SS_CUDA(e, cudaMemcpy(e->order, order.data(), G * 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->pmap, pmap.data(), G * 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->offsets, offs.data(), (e->P + 1) * 4, cudaMemcpyHostToDevice));
    }
    // -- batch scratch
    e->max_batch = cfg->max_batch > 0 ? cfg->max_batch : (int64_t(1) << 24);
    // count chunks: the granularity at which never-stored tuples are dropped
    // (a chunk with no kept tuple is never read again).  Power of two >=
    // 2^16, grown until the per-chunk histograms (n_chunk x G) stay <= 2^22
    // entries and n_chunk <= 4096.
    // (2^12..2^14-tuple chunks for few groups measured slower at C1: the
    // stats cost grows faster than the placement gains)
    const int s_min_log = 16;
    int64_t S = cfg->sub_batch;
    if (S <= 0) S = int64_t(1) << s_min_log;
    {
        int64_t p2 = int64_t(1) << s_min_log;
        while (p2 < S) p2 <<= 1;
        S = p2;
        auto nch = [&](int64_t c) { return (e->max_batch + c - 1) / c; };
        while ((cfg->sub_batch <= 0 && nch(S) * G > (int64_t(1) << 22) && S < e->max_batch) || nch(S) > 4096) S <<= 1;
    }
    e->S = S;
    e->n_sub_max = (int)((e->max_batch + S - 1) / S);
    const int nsub = e->n_sub_max;
    e->nblk = (int)((G + kScanBlk - 1) / kScanBlk);
    {
        const int bits = bits_for(G);
        if (bits <= 11) {
            e->plan.npass = 1;
            e->plan.shift[0] = 0; e->plan.bits[0] = bits;
            e->plan.shift[1] = 0; e->plan.bits[1] = 0;
        } else {
            e->plan.npass = 2;
            e->plan.bits[0] = bits / 2;
            e->plan.bits[1] = bits - bits / 2;
            e->plan.shift[0] = 0;
            e->plan.shift[1] = bits / 2;
        }
        e->rb[0] = rb_for(e->plan.bits[0]);
        e->rb[1] = rb_for(e->plan.bits[1]);
    }
    if ((rc = dalloc(e, &e->stage_keys, e->max_batch)) || (rc = dalloc(e, &e->stage_vals, e->max_batch)) ||
        (rc = dalloc(e, &e->gcnt, (size_t)nsub * G)) || (rc = dalloc(e, &e->gstart, (size_t)nsub * G)) ||
        (rc = dalloc(e, &e->gcount, G)) || (rc = dalloc(e, &e->bsum, (size_t)nsub * e->nblk)) ||
        (rc = dalloc(e, &e->dhist, (size_t)nsub * 2 * kMaxBins)) || (rc = dalloc(e, &e->tpt, e->P)) ||
        (rc = dalloc(e, &e->touched, 1)) || (rc = dalloc(e, &e->bad, 1)) ||
        (rc = dalloc(e, &e->tickets, (size_t)nsub * 2 + 2)) || (rc = dalloc(e, &e->gkept, G)) || (rc = dalloc(e, &e->n_live, nsub + 1)) ||
        (rc = dalloc(e, &e->chunk_live, nsub)) || (rc = dalloc(e, &e->lc, nsub)) || (rc = dalloc(e, &e->n_lc, 1)) ||
        (rc = dalloc(e, &e->chunk_h, (size_t)nsub * kMaxBins)) || (rc = dalloc(e, &e->chunk_base, (size_t)nsub * kMaxBins)) ||
        (rc = dalloc(e, &e->btile, kMaxBins + 1)) || (rc = dalloc(e, &e->ep_dev, 1)) ||
        (rc = dalloc(e, &e->bdelta, G)) || (rc = dalloc(e, &e->bmin, G)) || (rc = dalloc(e, &e->bmax, G)) ||
        (rc = dalloc(e, &e->hot_of, G)) || (rc = dalloc(e, &e->hot_g, kHotCache)) || (rc = dalloc(e, &e->n_hot_dev, 1)) ||
        (rc = dalloc(e, &e->fin_ticket, 1)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->fin_ticket, 0, 4, e->st));
    // single-pass placement whenever the cursors fit in shared memory; with
    // a small kept set (few live chunks, e.g. C1) every live chunk is cut
    // into sub-chunks so the placement still fills the GPU (one CTA per
    // live chunk left it idle, and the radix passes over the live chunks
    // were used instead: C1 placement 33 us)
    e->rank_place = G <= kRankMaxG;
    if (const char* rp = getenv("SS_B200_RANK_PLACE")) e->rank_place = G <= kRankMaxG && rp[0] != '0';
    if (e->rank_place &&
        ((rc = dalloc(e, &e->gpre, (size_t)nsub * G)) || (rc = dalloc(e, &e->gsub, (size_t)kSubUnitsMax * G)) ||
         (rc = dalloc(e, &e->subh, (size_t)kSubUnitsMax * G)) || (rc = dalloc(e, &e->sub_shift, 1))))
        return rc;
    if (e->rank_place) SS_CUDA(e, cudaMemsetAsync(e->sub_shift, 0, 4, e->st));
    // bucketed placement: every cold group (batch count < kBkTau) must keep
    // all its tuples, i.e. W >= kBkTau
    e->bucket = !e->rank_place && G > kRankMaxG && W >= kBkTau && e->max_batch <= kBkMaxBatch;
    {
        // A/B switch while the bucketed passes are tuned: off unless SS_B200_BUCKET=1
        const char* bp = getenv("SS_B200_BUCKET");
        e->bucket = e->bucket && bp && bp[0] == '1';
    }
    // look-back-free passes from 2^17 groups on (C4/C5: 0.63 -> 0.42 ms;
    // C3, 2^17: with the two-CTA pass and the parallel column scan 37.7 vs
    // 37.1 G tuples/s for the segmented radix passes over live chunks,
    // which stay in use for 2^14 < G <= 2^16)
    e->os = !e->rank_place && bits_for(G) >= 17;
    if (const char* op = getenv("SS_B200_ONESWEEP")) e->os = !e->rank_place && G > kRankMaxG && op[0] != '0';
    if (e->os) {
        const int bits = bits_for(G);
        if (const char* ob = getenv("SS_B200_OS_BITS")) e->os_digit = atoi(ob) == kOsBitsWide ? kOsBitsWide : kOsBits;
        if (const char* om = getenv("SS_B200_OS_MATCH")) e->os_match = atoi(om);
        if (const char* o2 = getenv("SS_B200_OS2")) e->os2 = o2[0] == '1';
        e->os_npass = (bits + e->os_digit - 1) / e->os_digit;
        if (e->os_npass > kOsMaxPass) e->os = false;
        int sh = 0;
        for (int p = 0; p < e->os_npass; ++p) {
            const int w = (bits - sh + (e->os_npass - p) - 1) / (e->os_npass - p);
            e->os_shift[p] = sh;
            e->os_bits[p] = w;
            sh += w;
        }
        const int64_t tiles = (e->max_batch + kOsTile - 1) / kOsTile;
        const int bins = 1 << e->os_digit;
        if (e->os && ((rc = dalloc(e, &e->os_hist, (size_t)tiles * bins)) ||
                      (rc = dalloc(e, &e->os_bsum, (size_t)((tiles + kOsBlkTiles - 1) / kOsBlkTiles) * bins)) ||
                      (rc = dalloc(e, &e->os_dtot, (size_t)bins))))
            return rc;
    }
    if (e->bucket) {
        BucketArgs& b = e->bk;
        if ((rc = dalloc(e, &b.bin_of, G)) || (rc = dalloc(e, &b.bin_first, kBkNBMax + 1)) ||
            (rc = dalloc(e, &b.bin_hot, kBkNBMax)) || (rc = dalloc(e, &b.n_bins, 1)) ||
            (rc = dalloc(e, &b.fsum, G / kBkBlk + 2)) || (rc = dalloc(e, &b.tbin, e->max_batch + 8)) ||
            (rc = dalloc(e, &b.hist, (size_t)kBkSupers * kBkNBMax)) || (rc = dalloc(e, &b.btot, kBkNBMax)) ||
            (rc = dalloc(e, &b.sbase, kBkNBMax)))
            return rc;
    }
    if ((rc = dalloc(e, &e->pwork, e->P)) || (rc = dalloc(e, &e->cta_map, 4 * kNumSM + e->P)) ||
        (rc = dalloc(e, &e->cta_used, 1)) || (rc = dalloc(e, &e->any_dead, 1)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->pwork, 0, (size_t)e->P * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->hot_of, 0xff, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->n_hot_dev, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->bdelta, 0, G * 8, e->st));
    ss_note_launch(), ss_launch(k_fill_i32, 296, 256, 0, e->st, e->bmin, G, 0x7fffffff);
    ss_note_launch(), ss_launch(k_fill_i32, 296, 256, 0, e->st, e->bmax, G, (int32_t)0x80000000);
    SS_CUDA(e, cudaMemsetAsync(e->gcnt, 0, (size_t)nsub * G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->gcount, 0, G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->chunk_live, 0, (size_t)nsub * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->ep_dev, 0, 4, e->st));
    ss_note_launch(), ss_launch(k_set_bad, 1, 1, 0, e->st, e->bad);
    if ((rc = engine_alloc_sort(e, e->max_batch))) return rc;
    e->vals_final = e->vbuf[0];
    e->keys_final = e->kbuf2;
    // -- int64 key table
    e->keys64 = cfg->key_bits == 64;
    if (const char* ka = getenv("SS_B200_KEY_AGG")) e->key_agg = atoi(ka);
    if (e->keys64) {
        uint64_t cap = 1;
        while (cap < 2 * (uint64_t)G) cap <<= 1;
        KeyTable& t = e->kt;
        if ((rc = dalloc(e, &t.ent, cap + 1)) || (rc = dalloc(e, &t.first, cap + 1)) ||
            (rc = dalloc(e, &t.pend, e->max_batch)) || (rc = dalloc(e, &t.pend_ent, e->max_batch)) ||
            (rc = dalloc(e, &t.n_pend, 1)) || (rc = dalloc(e, &t.slot_ent, G)) ||
            (rc = dalloc(e, &t.new_ent, G)) || (rc = dalloc(e, &t.n_new, 1)) || (rc = dalloc(e, &t.n_slots, 1)) ||
            (rc = dalloc(e, &t.mark, e->max_batch)) || (rc = dalloc(e, &t.slot_keys, G)) ||
            (rc = dalloc(e, &t.min_key_entry, 1)) || (rc = dalloc(e, &t.overflow, 1)) ||
            (rc = dalloc(e, &t.prev_slots, 1)) ||
            (rc = dalloc(e, &e->stage_keys64, e->max_batch)) ||
            (rc = dalloc(e, &e->kbsum, e->max_batch / kMarkBlk + 2)))
            return rc;
        t.cap_mask = cap - 1;
        t.G = (int)G;
        // pipelined key probe (large G: the probe also counts the batch)
        if (G > 16384 && !e->stream_scope && !getenv("SS_B200_NO_KEY_PIPE") && (rc = create_count_pipe(e)))
            return rc;
        ss_note_launch(), ss_launch(k_key_init, 296, 256, 0, e->st, t.ent, (int64_t)cap + 1);
        SS_CUDA(e, cudaMemsetAsync(t.first, 0xff, (cap + 1) * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(t.mark, 0xff, e->max_batch * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(t.n_new, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(t.n_slots, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(t.min_key_entry, 0xff, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(t.overflow, 0, 4, e->st));
    }
    // u32 groups: the count of batch t+1 likewise runs ahead
    if (!e->keys64 && !e->stream_scope && !getenv("SS_B200_NO_KEY_PIPE") && (rc = create_count_pipe(e)))
        return rc;
    // small G without a policy: statistics, scans and sub-chunk prefixes too
    if (e->kst && !e->keys64 && e->rank_place && !getenv("SS_B200_NO_AHEAD")) {
        const int nsub = e->n_sub_max;
        ss_engine::AheadSet& a0 = e->aset[0];
        a0 = {e->gcount, e->gkept, e->gpre, e->gstart, e->n_live, e->lc, e->n_lc, e->gsub, e->sub_shift,
              e->tpt, e->touched};
        ss_engine::AheadSet& a1 = e->aset[1];
        if ((rc = dalloc(e, &a1.gcount, G)) || (rc = dalloc(e, &a1.gkept, G)) ||
            (rc = dalloc(e, &a1.gpre, (size_t)nsub * G)) || (rc = dalloc(e, &a1.gstart, (size_t)nsub * G)) ||
            (rc = dalloc(e, &a1.n_live, nsub + 1)) || (rc = dalloc(e, &a1.lc, nsub)) || (rc = dalloc(e, &a1.n_lc, 1)) ||
            (rc = dalloc(e, &a1.gsub, (size_t)kSubUnitsMax * G)) || (rc = dalloc(e, &a1.sub_shift, 1)) ||
            (rc = dalloc(e, &a1.tpt, e->P)) || (rc = dalloc(e, &a1.touched, 1)))
            return rc;
        SS_CUDA(e, cudaMemsetAsync(a1.sub_shift, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(a1.gcount, 0, G * 4, e->st));
        e->ahead_ok = true;
    }
    // -- balancer
    // (used whenever the lists are not staged: large G, or large P)
    if ((rc = dalloc(e, &e->bal_ecnt, G)) || (rc = dalloc(e, &e->bal_eflag, G))) return rc;
    e->cap_moves = 4 * e->P;
    if ((rc = dalloc(e, &e->keep_at, e->P)) || (rc = dalloc(e, &e->mv_pos, e->cap_moves))) return rc;
    if ((rc = dalloc(e, &e->moves, e->cap_moves)) || (rc = dalloc(e, &e->front_top, e->P)) ||
        (rc = dalloc(e, &e->back_first, e->P)) || (rc = dalloc(e, &e->mv_next, e->cap_moves)) ||
        (rc = dalloc(e, &e->n_moves, 1)) || (rc = dalloc(e, &e->scanned, 1)) ||
        (rc = dalloc(e, &e->final_tpt, e->P)) || (rc = dalloc(e, &e->prev_moves, 1)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->n_moves, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->prev_moves, 0, 4, e->st));
    // -- hot-key split plans
    e->maxS = 2 * e->P + 2;
    e->maxSh = e->P + e->maxS + 1;
    for (int b = 0; b < 2; ++b) {
        SplitPlan& sp = e->plan_buf[b];
        if ((rc = dalloc(e, &sp.n_split, 1)) || (rc = dalloc(e, &sp.n_share, 1)) || (rc = dalloc(e, &sp.split_of, G)) ||
            (rc = dalloc(e, &sp.split_g, e->maxS)) || (rc = dalloc(e, &sp.split_den, e->maxS)) ||
            (rc = dalloc(e, &sp.part_soff, e->P + 1)) || (rc = dalloc(e, &sp.share_grp, e->maxSh)) ||
            (rc = dalloc(e, &sp.share_lo, e->maxSh)) || (rc = dalloc(e, &sp.share_hi, e->maxSh)))
            return rc;
        SS_CUDA(e, cudaMemsetAsync(sp.n_split, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(sp.n_share, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(sp.split_of, 0xff, G * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(sp.part_soff, 0, (e->P + 1) * 4, e->st));
    }
    if ((rc = dalloc(e, &e->spx.hot_g, e->maxS)) || (rc = dalloc(e, &e->spx.n_hot, 1)) ||
        (rc = dalloc(e, &e->spx.base, e->P)) || (rc = dalloc(e, &e->spx.hot_flag, G)) ||
        (rc = dalloc(e, &e->spx.n_stored, 1)))
        return rc;
    // -- emission
    if ((rc = dalloc(e, &e->n_res, 1)) || (rc = dalloc(e, &e->r_g, G)) || (rc = dalloc(e, &e->r_cnt, G)) ||
        (rc = dalloc(e, &e->r_sum, G)) || (rc = dalloc(e, &e->r_avg, G)) || (rc = dalloc(e, &e->r_mn, G)) ||
        (rc = dalloc(e, &e->r_mx, G)) || (rc = dalloc(e, &e->rescan, G)) || (rc = dalloc(e, &e->n_rescan, 1)) ||
        (rc = dalloc(e, &e->part_ns, e->P)) || (rc = dalloc(e, &e->loads, e->P)) || (rc = dalloc(e, &e->fill_loads, e->P)) || (rc = dalloc(e, &e->d_rep, 1)) ||
        (rc = dalloc(e, &e->part_work, e->P)) ||
        (rc = dalloc(e, &e->alg_bytes, 1)))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->alg_bytes, 0, 8, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->n_res, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->n_rescan, 0, 4, e->st));
    if (e->minmax && W > kMMSumMinW) {
        // every group whose window is full holds W ring values, so at most
        // (ring pool / W) of them -- the summaries cost pool / kMMChunk x 8 B
        const int64_t max_full = std::min<int64_t>(G, (int64_t)(e->pool_cap / (uint64_t)W) + 1);
        const int64_t nch = (W + kMMChunk - 1) / kMMChunk;
        if ((rc = dalloc(e, &e->sum_idx, G)) || (rc = dalloc(e, &e->sum_valid, G)) || (rc = dalloc(e, &e->n_sum, 1)) ||
            (rc = dalloc(e, &e->sums, (size_t)max_full * nch)))
            return rc;
        SS_CUDA(e, cudaMemsetAsync(e->sum_idx, 0xff, G * 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->sum_valid, 0, G, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->n_sum, 0, 4, e->st));
    }
    SS_CUDA(e, cudaMallocHost(&e->h_rep, sizeof(DevReport)));
    memset(e->h_rep, 0, sizeof(DevReport));
    e->h_rep->bad = (unsigned long long)kNoBad;
    SS_CUDA(e, cudaFuncSetAttribute(k_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    SS_CUDA(e, cudaFuncSetAttribute(k_count_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    SS_CUDA(e, cudaFuncSetAttribute(k_sub_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankMaxG * 4));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<4>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<5>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<6>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<7>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<8>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<9>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<10>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SortSmem<11>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_sort_pass<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SortSmem<4>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kIngestSmem));
    SS_CUDA(e, cudaFuncSetAttribute(k_bk_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kBkNBMax * 4));
    SS_CUDA(e, cudaFuncSetAttribute(k_os_pass<kOsBits>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)OsSmem<kOsBits>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_os_pass<kOsBitsWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)OsSmem<kOsBitsWide>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_os_pass2<kOsBitsWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)Os2Smem<kOsBitsWide>::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_bk_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BkSmem::bytes));
    SS_CUDA(e, cudaFuncSetAttribute(k_bk_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BkLocSmem::bytes));
    for (int b = 0; b <= 14; ++b) {
        const RankKernel rk = b ? rank_kernel(b) : k_rank_place<0>;
        SS_CUDA(e, cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rank_smem_bytes(kRankMaxG)));
    }
    SS_CUDA(e, cudaFuncSetAttribute(k_balance<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBalSmemMax));
    SS_CUDA(e, cudaFuncSetAttribute(k_balance<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBalSmemMax));
    SS_CUDA(e, cudaFuncSetAttribute(k_balance<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBalSmemMax));
    SS_CUDA(e, cudaFuncSetAttribute(k_split_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

extern "C" int ss_set_stream(ss_engine* e, void* stream) {
    if (!e) return SS_E_CONFIG;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (e->cfg.reserved == 0 && e->st) cudaStreamDestroy(e->st);
    e->st = (cudaStream_t)stream;
    e->cfg.reserved = 1;   // not owned
    return SS_OK;
}

// int64 keys: device key inputs are complete when ss_step_keys64 is called
// (not produced by pending engine-stream work), so the next batch's probe
// may run ahead on the key stream (host inputs always may)
extern "C" int ss_set_key_pipeline(ss_engine* e, int ready_inputs) {
    if (!e) return SS_E_CONFIG;
    e->key_pipe_dev = ready_inputs != 0;
    return SS_OK;
}

extern "C" int ss_sync(ss_engine* e) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    if (e->kst) SS_CUDA(e, cudaStreamSynchronize(e->kst));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// --------------------------------------------------------------------------
// input staging
// --------------------------------------------------------------------------
// make the engine stream wait for the last batch's side work (policy,
// apply, report) before anything that reads or writes the assignment
static int join_side(ss_engine* e) {
    if (e->side_pending) {
        SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_apply, 0));
        e->side_pending = false;
    }
    return SS_OK;
}

// streaming input: pick the batch's staging buffer; the copy stream waits
// until the batch that last read it has finished its first placement pass
static int begin_stage(ss_engine* e, bool keys64) {
    const int b = e->stg_next;
    e->stg_next ^= 1;
    int rc;
    if (!e->skeys[1]) {
        e->skeys[0] = e->stage_keys;
        e->svals[0] = e->stage_vals;
        if ((rc = dalloc(e, &e->skeys[1], e->max_batch)) || (rc = dalloc(e, &e->svals[1], e->max_batch))) return rc;
    }
    if (keys64 && !e->sk64[1]) {
        e->sk64[0] = e->stage_keys64;
        if ((rc = dalloc(e, &e->sk64[1], e->max_batch))) return rc;
    }
    if (e->freed_rec[b]) SS_CUDA(e, cudaStreamWaitEvent(e->cp, e->ev_freed[b], 0));
    e->cur_stage = b;
    return SS_OK;
}

// host -> staging buffer on the copy stream (device pointers pass through)
template <typename T>
static int stage_h2d(ss_engine* e, T* dst, const T* src, int64_t n, const T** out) {
    if (!src || is_device_ptr(src)) {
        *out = src;
        return SS_OK;
    }
    if (n) SS_CUDA(e, cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, e->cp));
    *out = dst;
    return SS_OK;
}

// the engine stream waits for the batch's copies
static int end_stage(ss_engine* e) {
    const int b = e->cur_stage;
    SS_CUDA(e, cudaEventRecord(e->ev_staged[b], e->cp));
    SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_staged[b], 0));
    return SS_OK;
}

static int stage_input(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                       const uint32_t** dk, const int32_t** dv) {
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    if (is_device_ptr(groups)) *dk = groups;
    else {
        if (n) SS_CUDA(e, cudaMemcpyAsync(e->stage_keys, groups, n * 4, cudaMemcpyHostToDevice, e->st));
        *dk = e->stage_keys;
    }
    if (dv) {
        if (!attrs) *dv = nullptr;
        else if (is_device_ptr(attrs)) *dv = attrs;
        else {
            if (n) SS_CUDA(e, cudaMemcpyAsync(e->stage_vals, attrs, n * 4, cudaMemcpyHostToDevice, e->st));
            *dv = e->stage_vals;
        }
    }
    return SS_OK;
}

// After a DataError the partially filled histograms are cleared so the
// engine state is exactly as before the failed call.
static int recover_bad(ss_engine* e) {
    cudaStreamSynchronize(e->side);
    e->side_pending = false;
    SS_CUDA(e, cudaMemsetAsync(e->gcnt, 0, (size_t)e->n_sub_max * e->G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->gcount, 0, e->G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->chunk_live, 0, (size_t)e->n_sub_max * 4, e->st));
    ss_note_launch(), ss_launch(k_set_bad, 1, 1, 0, e->st, e->bad);
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

static int data_error(ss_engine* e, unsigned long long idx, const uint32_t* dkeys) {
    uint32_t g = 0;
    cudaMemcpy(&g, dkeys + idx, 4, cudaMemcpyDeviceToHost);
    recover_bad(e);
    return fail(e, SS_E_DATA, "tuple " + std::to_string(idx) + " has group " + std::to_string(g) +
                                  ", outside [0, " + std::to_string(e->G) + ")");
}

// K2 over n tuples with sub-batch size S (n_sub = ceil(n / S))
static int launch_count(ss_engine* e, const uint32_t* dk, int64_t n, int64_t S, bool use_hot = false) {
    if (n == 0) return SS_OK;
    const int vec_ok = ((uintptr_t)dk % 16) == 0;
    if (e->G <= 16384) {
        // larger chunks amortise the per-CTA flush of the G-bin histogram
        const int64_t chunk = (e->G > 2048 && S % 65536 == 0) ? 65536 : kCountChunk;
        const int64_t grid = (n + chunk - 1) / chunk;
        ss_note_launch(), ss_launch(k_count<true>, (unsigned)grid, 512, e->G * 4, e->st, dk, n, (uint32_t)e->G, S, chunk, e->gcnt, e->bad,
                                                               vec_ok, nullptr, nullptr, 0);
    } else {
        // the hot cache holds the previous batch's hot groups; its size is
        // fixed at kHotCache slots (unused slots count nothing)
        const int64_t grid = (n + kCountChunk - 1) / kCountChunk;
        const int nh = use_hot ? kHotCache : 0;
        ss_note_launch(), ss_launch(k_count<false>, (unsigned)grid, 512, (size_t)nh * 4, e->st, dk, n, (uint32_t)e->G, S, kCountChunk, e->gcnt,
                                                                      e->bad, vec_ok, e->hot_of, e->hot_g, nh);
    }
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// batch statistics over n_chunk count rows; `step` also derives the kept
// counts and live chunks of the fused step
static int launch_stats(ss_engine* e, int n_chunk, bool step = false, bool want_work = false) {
    SS_CUDA(e, cudaMemsetAsync(e->tpt, 0, e->P * 8, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->touched, 0, 8, e->st));
    if (step) SS_CUDA(e, cudaMemsetAsync(e->any_dead, 0, 4, e->st));
    // many chunks (> 32): a CTA per 32 groups, warps over chunk ranges;
    // otherwise a thread per group, coalesced over consecutive groups
    if (n_chunk > 32) {
        const unsigned grid = (unsigned)std::min<int64_t>((e->G + 31) / 32, 8 * kNumSM);
        const bool small = e->G <= 4096;
        auto kern = small ? k_batch_stats_cols<32> : k_batch_stats_cols<16>;
        ss_note_launch(), ss_launch(kern, grid, small ? 1024 : 512, e->P * 8, e->st, e->gcnt, n_chunk, (uint32_t)e->G, e->pmap, e->P, e->gcount, step ? e->gkept : nullptr,
            step ? e->chunk_live : nullptr, e->tpt, e->touched, e->bad, e->fill, e->W, e->alg_bytes, e->trace_on ? 1 : 0,
            step && e->rank_place ? e->gpre : nullptr, want_work ? e->pwork : nullptr, step ? e->any_dead : nullptr);
    } else {
        const unsigned grid = (unsigned)std::min<int64_t>((e->G + 255) / 256, 16 * kNumSM);
        ss_note_launch(), ss_launch(k_batch_stats, grid, 256, e->P * 8, e->st, e->gcnt, n_chunk, (uint32_t)e->G, e->pmap, e->P, e->gcount, step ? e->gkept : nullptr,
            step ? e->chunk_live : nullptr, e->tpt, e->touched, e->bad, e->fill, e->W, e->alg_bytes, e->trace_on ? 1 : 0,
            step && e->rank_place ? e->gpre : nullptr, want_work ? e->pwork : nullptr, step ? e->any_dead : nullptr);
    }
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// G-sized scan of one count row -> run starts gstart[g] and the digit bases
// of every placement pass; with n_chunk > 0 also the live-chunk list
static int launch_scans(ss_engine* e, const int32_t* row, int n_chunk = 0) {
    if (e->G <= kScanSmallG) {
        // the single-pass placement needs no digit bases or bucket tiles
        DigitPlan plan = e->plan;
        const bool rank = n_chunk && e->rank_place;
        if (rank) plan.npass = 0;
        ss_note_launch(), ss_launch(k_scan_small, 1, 1024, 0, e->st, row, (uint32_t)e->G, plan, e->dhist, e->gstart, e->bad,
                                                              e->n_live, n_chunk ? e->chunk_live : nullptr, n_chunk,
                                                              e->lc, e->n_lc, n_chunk && !rank ? e->btile : nullptr,
                                                              e->ep_dev, rank ? e->sub_shift : nullptr);
        SS_CUDA(e, cudaGetLastError());
        return SS_OK;
    }
    SS_CUDA(e, cudaMemsetAsync(e->dhist, 0, (size_t)2 * kMaxBins * 4, e->st));
    dim3 g2(e->nblk, 1);
    ss_note_launch(), ss_launch(k_scan_reduce, g2, 1024, 0, e->st, row, (uint32_t)e->G, e->bsum, e->nblk, e->plan, e->dhist, e->bad);
    ss_note_launch(), ss_launch(k_scan_top, 1, 1024, 0, e->st, e->bsum, e->nblk, e->plan, e->dhist, e->bad, e->n_live,
                                                        n_chunk ? e->chunk_live : nullptr, n_chunk, e->lc, e->n_lc,
                                                        n_chunk ? e->btile : nullptr, e->ep_dev);
    ss_note_launch(), ss_launch(k_scan_down, g2, 1024, 0, e->st, row, (uint32_t)e->G, e->bsum, e->nblk, e->gstart, e->bad);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}


// reorder API: stable placement of all n tuples (keys -> kbuf2, values ->
// vbuf[0]); no tuple is dropped
static int launch_place_all(ss_engine* e, const uint32_t* dk, const int32_t* dv, int64_t n) {
    const uint32_t* base0 = e->dhist;
    const uint32_t* base1 = e->dhist + kMaxBins;
    const uint32_t m0 = (1u << e->plan.bits[0]) - 1u;
    if (e->plan.npass == 1) {
        sort_dispatch(e->rb[0], e->st, dk, dv, e->kbuf2, e->vbuf[0], (int)n, 0, m0, base0, e->status,
                      e->ep_dev, 0, e->tickets, e->bad, 0);
    } else {
        const uint32_t m1 = (1u << e->plan.bits[1]) - 1u;
        sort_dispatch(e->rb[0], e->st, dk, dv, e->kbuf, e->vbuf[1], (int)n, e->plan.shift[0], m0, base0, e->status,
                      e->ep_dev, 0, e->tickets, e->bad, 0);
        sort_dispatch(e->rb[1], e->st, e->kbuf, e->vbuf[1], e->kbuf2, e->vbuf[0], (int)n, e->plan.shift[1], m1, base1,
                      e->status, e->ep_dev, 1, e->tickets + 1, e->bad, 0);
    }
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

template <int BITS>
static void launch_os_pass_t(ss_engine* e, const OsArgs& a, unsigned tiles, unsigned blks) {
    ss_note_launch(), ss_launch(k_os_up<BITS>, (tiles + kOsUpTiles - 1) / kOsUpTiles, kOsThreads, 0, e->st, a);
    ss_note_launch(), ss_launch(k_os_red<BITS>, blks, 1024, 0, e->st, a);
    ss_note_launch(), ss_launch(k_os_top<BITS>, (1 << BITS) / 32, 1024, 0, e->st, a);
    ss_note_launch(), ss_launch(k_os_down<BITS>, blks, 1024, 0, e->st, a);
    if constexpr (BITS == kOsBitsWide) {
        if (e->os2) {
            ss_note_launch(), ss_launch(k_os_pass2<BITS>, std::min<unsigned>(tiles, 2 * kNumSM), kOs2Threads,
                                        Os2Smem<BITS>::bytes, e->st, a);
            return;
        }
    }
    ss_note_launch(), ss_launch(k_os_pass<BITS>, std::min<unsigned>(tiles, kNumSM), kOsThreads, OsSmem<BITS>::bytes, e->st, a);
}
static void launch_os_pass(ss_engine* e, const OsArgs& a, unsigned tiles, unsigned blks) {
    if (e->os_digit == kOsBitsWide) launch_os_pass_t<kOsBitsWide>(e, a, tiles, blks);
    else launch_os_pass_t<kOsBits>(e, a, tiles, blks);
}

// fused step: stable placement of the batch's kept tuples (values only) into
// vbuf[0].  The first pass walks the live chunks and drops never-stored
// tuples; a second pass (G > 2^11) consumes the compacted kept set.
static void use_ahead_set(ss_engine* e, int b) {
    const ss_engine::AheadSet& a = e->aset[b];
    e->gcount = a.gcount; e->gkept = a.gkept; e->gpre = a.gpre; e->gstart = a.gstart; e->n_live = a.n_live;
    e->lc = a.lc; e->n_lc = a.n_lc; e->gsub = a.gsub; e->sub_shift = a.sub_shift; e->tpt = a.tpt;
    e->touched = a.touched;
    e->gcnt = e->gcnt_buf[b];
}

// sub-chunk counts and prefixes of the single-pass placement (no-ops
// unless k_scan_small chose sub-chunks)
static void launch_sub_prefix(ss_engine* e, const uint32_t* dk, int64_t n, int cs) {
    ss_note_launch(), ss_launch(k_sub_hist, kSubUnitsMax, 512, e->G * 4, e->st, dk, n, cs, e->lc, e->n_lc, e->sub_shift,
                                (uint32_t)e->G, e->subh, e->bad);
    ss_note_launch(), ss_launch(k_sub_scan, 2 * kNumSM, 256, 0, e->st, e->gpre, e->lc, e->n_lc, e->sub_shift,
                                (uint32_t)e->G, e->subh, e->gsub, e->bad);
}

static int launch_place_step(ss_engine* e, const uint32_t* dk, const int32_t* dv, int64_t n) {
    const uint32_t* base0 = e->dhist;
    const uint32_t* base1 = e->dhist + kMaxBins;
    const uint32_t m0 = (1u << e->plan.bits[0]) - 1u;
    const int nb0 = 1 << e->plan.bits[0];
    const int n_chunk = (int)std::max<int64_t>(1, (n + e->S - 1) / e->S);
    int cs = 0;
    while ((int64_t(1) << cs) < e->S) ++cs;
    e->vals_final = e->vbuf[0];
    e->keys_final = e->kbuf2;
    if (e->os && !e->bucket) {
        // LSD passes: (dk, dv) -> (kbuf, vbuf1) -> (kbuf2, vbuf0) -> ...
        uint32_t* kb[2] = {e->kbuf, e->kbuf2};
        int32_t* vb[2] = {e->vbuf[1], e->vbuf[0]};
        const uint32_t* kin = dk;
        const int32_t* vin = dv;
        const unsigned tiles = (unsigned)((n + kOsTile - 1) / kOsTile);
        const unsigned blks = (tiles + kOsBlkTiles - 1) / kOsBlkTiles;
        for (int p = 0; p < e->os_npass; ++p) {
            const bool last = p == e->os_npass - 1;
            OsArgs a{};
            a.kin = kin;
            a.vin = vin;
            a.kout = (last && !e->trace_on) ? nullptr : kb[p & 1];
            a.vout = vb[p & 1];
            a.n = n;
            a.n_dev = p ? e->n_live : nullptr;
            a.shift = e->os_shift[p];
            a.mask = (1u << e->os_bits[p]) - 1u;
            a.hist = e->os_hist;
            a.bsum = e->os_bsum;
            a.dtot = e->os_dtot;
            a.live = p == 0 ? e->gcnt : nullptr;
            a.chunk_shift = cs;
            a.G = (uint32_t)e->G;
            a.any_dead = e->any_dead;
            a.match = e->os_match;
            a.bad = e->bad;
            launch_os_pass(e, a, tiles, blks);
            kin = a.kout;
            vin = a.vout;
            if (last) {
                e->vals_final = a.vout;
                e->keys_final = a.kout;
            }
        }
        SS_CUDA(e, cudaGetLastError());
        return SS_OK;
    }
    if (e->bucket && !e->trace_on) {
        BucketArgs a = e->bk;
        a.keys = dk;
        a.vals = dv;
        a.n = n;
        a.G = (uint32_t)e->G;
        a.gcount = e->gcount;
        a.gkept = e->gkept;
        a.gstart = e->gstart;
        a.skey = e->kbuf;
        a.sval = e->vbuf[1];
        a.vout = e->vbuf[0];
        a.bad = e->bad;
        const int nblk = (int)((e->G + kBkBlk - 1) / kBkBlk);
        ss_note_launch(), ss_launch(k_bk_flags_reduce, nblk, 1024, 0, e->st, a);
        ss_note_launch(), ss_launch(k_bk_flags_top, 1, 1024, 0, e->st, a, nblk);
        ss_note_launch(), ss_launch(k_bk_flags_down, nblk, 1024, 0, e->st, a);
        ss_note_launch(), ss_launch(k_bk_hist, kBkSupers, 1024, kBkNBMax * 4, e->st, a);
        ss_note_launch(), ss_launch(k_bk_colscan, kBkNBMax / 32, 1024, 0, e->st, a);
        ss_note_launch(), ss_launch(k_bk_binscan, 1, 1024, 0, e->st, a);
        ss_note_launch(), ss_launch(k_bk_scatter, kBkSupers, kBkThreads, BkSmem::bytes, e->st, a);
        ss_note_launch(), ss_launch(k_bk_local, 2 * kNumSM, kBkLocThreads, BkLocSmem::bytes, e->st, a);
        SS_CUDA(e, cudaGetLastError());
        return SS_OK;
    }
    if (e->rank_place) {
        // one CTA per live chunk, cursors from the chunk prefix (k_batch_stats)
        static const int use_match = getenv("SS_B200_RANK_MATCH") ? atoi(getenv("SS_B200_RANK_MATCH")) : 0;
        // (a chain-free variant with per-warp histograms of all G groups
        // per 4096-tuple piece, for G <= 2048, measured slower at C1: 21.4
        // against 16.7 us, and was dropped)
        auto kern = use_match ? k_rank_place<0> : rank_kernel(bits_for(e->G));
        const size_t rsm = rank_smem_bytes((uint32_t)e->G);
        // sub-chunk prefixes (no-ops unless k_scan_small chose sub-chunks)
        if (!e->ahead) launch_sub_prefix(e, dk, n, cs);
        ss_note_launch(), ss_launch(kern, std::max(n_chunk, kSubUnitsMax), kRankWarps * 32, rsm, e->st, dk, dv, e->trace_on ? e->kbuf2 : nullptr, e->vbuf[0], n, cs, e->lc, e->n_lc, e->gpre, e->gstart,
            (uint32_t)e->G, e->n_live, e->bad, e->sub_shift, e->gsub);
        SS_CUDA(e, cudaGetLastError());
        return SS_OK;
    }
    // per-live-chunk bin bases of the first pass
    // enough CTAs per chunk that every SM has a slice of ~4K groups or more
    const int slices = (int)std::max<int64_t>(1, std::min<int64_t>((e->G + 4095) / 4096, (2 * kNumSM + n_chunk - 1) / n_chunk));
    SS_CUDA(e, cudaMemsetAsync(e->chunk_h, 0, (size_t)n_chunk * nb0 * 4, e->st));
    ss_note_launch(), ss_launch(k_chunk_hist, dim3(n_chunk, slices), 1024, nb0 * 4, e->st, e->gcnt, (uint32_t)e->G, e->lc, e->n_lc,
                                                                                   m0, nb0, e->chunk_h, e->bad);
    ss_note_launch(), ss_launch(k_chunk_scan, (nb0 + 31) / 32, 1024, 0, e->st, e->chunk_h, e->n_lc, nb0, base0,
                                                                        e->chunk_base, e->bad);
    SortSeg s1{};
    s1.mode = 1;
    s1.live = e->gcnt;
    s1.lc = e->lc;
    s1.n_lc = e->n_lc;
    s1.chunk_shift = cs;
    s1.G = (uint32_t)e->G;
    s1.cbase = e->chunk_base;
    s1.any_dead = e->any_dead;
    if (e->plan.npass == 1) {
        sort_dispatch(e->rb[0], e->st, dk, dv, e->trace_on ? e->kbuf2 : nullptr, e->vbuf[0], (int)n, 0, m0, base0,
                      e->status, e->ep_dev, 0,
                      e->tickets, e->bad, 1, e->n_live, &s1);
    } else {
        const uint32_t m1 = (1u << e->plan.bits[1]) - 1u;
        sort_dispatch(e->rb[0], e->st, dk, dv, e->kbuf, e->vbuf[1], (int)n, e->plan.shift[0], m0, base0, e->status,
                      e->ep_dev, 0, e->tickets, e->bad, 1, e->n_live, &s1);
        SortSeg s2{};
        s2.mode = 2;
        s2.G = (uint32_t)e->G;
        s2.btile = e->btile;
        s2.bpos = base0;
        s2.nb = nb0;
        s2.b0 = e->plan.bits[0];
        s2.gstart = e->gstart;
        sort_dispatch(e->rb[1], e->st, e->kbuf, e->vbuf[1], e->trace_on ? e->kbuf2 : nullptr, e->vbuf[0], (int)n,
                      e->plan.shift[1], m1, base1,
                      e->status, e->ep_dev, 1, e->tickets + 1, e->bad, 0, e->n_live, &s2);
    }
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

static IngestArgs ingest_args(ss_engine* e, int plan) {
    IngestArgs a{};
    a.order = e->order;
    a.offsets = e->offsets;
    a.gcnt = e->gkept;          // each group's kept run ...
    a.gcount = e->gcount;       // ... is the suffix of its K batch tuples
    a.gstart = e->gstart;
    a.vals = e->vals_final;
    a.fill = e->fill;
    a.next_pos = e->next_pos;
    a.off = e->off;
    a.ring = e->ring;
    a.bdelta = e->bdelta;
    a.bmin = e->bmin;
    a.bmax = e->bmax;
    a.W = e->W;
    a.minmax = e->minmax;
    if (plan >= 0) {
        const SplitPlan& sp = e->plan_buf[plan];
        a.split_of = sp.split_of;
        a.share_off = sp.part_soff;
        a.share_grp = sp.share_grp;
        a.share_lo = sp.share_lo;
        a.share_hi = sp.share_hi;
        a.split_g = sp.split_g;
        a.split_den = sp.split_den;
    }
    a.part_ns = e->part_ns;
    a.part_work = e->part_work;
    a.n_live = e->n_live;
    a.bad = e->bad;
    return a;
}

static int move_cap(ss_engine* e, const ss_balancer* b);
static int enqueue_report(ss_engine* e, int64_t n, bool has_policy, cudaStream_t st);
static ReportArgs report_args(ss_engine* e, int64_t n, bool has_policy);
static int copy_report(ss_engine* e, cudaStream_t st);

// an event other streams (or the host) wait on: inside a stream capture it
// must be an external event-record node
static cudaError_t record_ext(ss_engine* e, cudaEvent_t ev, cudaStream_t st) {
    return e->capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal) : cudaEventRecord(ev, st);
}

// One batch (the loop body of harness.run, harness.py:99-117).
//   main stream: count -> [join last batch's side work] -> stats -> scans
//                -> reserve -> per sub-batch (place, window exchange)
//                -> finalize + emit (+ MIN/MAX rescans)
//   side stream: policy / split planner (from the stats) -> [wait for the
//                last window exchange] -> apply moves -> report
// The side work of batch t overlaps the rest of batch t and the count of
// batch t+1; batch t+1's stats wait for it (they read the new map).
static int run_batch(ss_engine* e, const uint32_t* dk, const int32_t* dv, int64_t n, const ss_balancer* bal,
                     bool emit) {
    const int n_chunk = (int)std::max<int64_t>(1, (n + e->S - 1) / e->S);
    int rc;
    const bool split = bal && bal->split;
    // split mode: hot groups are water-filled over the partitions, cold
    // groups move by the configured policy (any of the seven; the hot ones
    // are excluded from its picks); without split, the reference policy
    // runs unchanged
    const int pol = bal ? bal->policy : SS_POLICY_NO;
    const bool has_policy = pol != SS_POLICY_NO;
    const bool run_side = has_policy || split;
    // the reassignment policy alone leaves partitions hosting a top group
    // with several times the mean work: K4 CTAs in proportion to the work
    // (measured at C2: 4 x 148 CTAs in total beat 2, 8 and 16 x 148; with
    // static partitions, C1, the uniform grid is faster)
    constexpr int k4_waves = 4;
    const bool work_grid = has_policy && !split && e->P <= 1024;
    SS_CUDA(e, cudaMemsetAsync(e->tickets, 0, 2 * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->part_ns, 0, e->P * 8, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->part_work, 0, e->P * 8, e->st));
    if (emit) SS_CUDA(e, cudaMemsetAsync(e->n_res, 0, 4, e->st));
    if (e->minmax) SS_CUDA(e, cudaMemsetAsync(e->n_rescan, 0, 4, e->st));
    {
        ProfScope ps(e, SS_K_COUNT, e->st);
        if (e->G <= 16384) {
            // one CTA per count chunk, rows written whole (no zeroing needed)
            if (n && !e->pre_counted) {
                ss_note_launch(), ss_launch(k_count_rows, n_chunk, 512, e->G * 4, e->st, dk, n, (uint32_t)e->G, e->S, e->gcnt,
                                                                                 e->bad, ((uintptr_t)dk % 16) == 0);
                SS_CUDA(e, cudaGetLastError());
            }
        } else if (!e->pre_counted && (rc = launch_count(e, dk, n, e->S, true))) return rc;
    }
    if (e->side_pending) {
        SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_apply, 0));
        e->side_pending = false;
    }
    // hot-key split: this batch's plan, computed on the side stream from this
    // batch's counts while the placement runs; the window update waits for it
    const int plan = split ? (e->plan_cur ^ 1) : -1;
    e->last_plan = plan;
    {
        ProfScope ps(e, SS_K_STATS, e->st);
        if (!e->ahead && (rc = launch_stats(e, n_chunk, true, work_grid))) return rc;
        if (e->G > 16384) {
            // hot cache for the next batch's count: > 1/(4 kHotCache) of the batch
            SS_CUDA(e, cudaMemsetAsync(e->n_hot_dev, 0, 4, e->st));
            ss_note_launch(), ss_launch(k_hot_select, group_grid(e->G), 256, 0, e->st, e->gcount, (uint32_t)e->G,
                                                        std::max<long long>(32, n / (4 * kHotCache)), e->hot_of,
                                                        e->hot_g, e->n_hot_dev, e->bad,
                                                        e->keys64 ? (int32_t*)e->kt.ent : nullptr, e->kt.slot_ent);
            // the next batch's key probe (key stream) may start: it reads the hot cache
            if (e->kst) {
                SS_CUDA(e, record_ext(e, e->ev_hot, e->st));
                e->hot_rec = true;
            }
        }
    }
    e->alg_input += (e->keys64 ? 12 : 8) * n;   // the batch is read once: key + attr bytes
    if (run_side) {
        SS_CUDA(e, cudaEventRecord(e->ev_stats, e->st));
        SS_CUDA(e, cudaStreamWaitEvent(e->side, e->ev_stats, 0));
        ProfScope ps(e, SS_K_BALANCE, e->side);
        if (split) {
            SS_CUDA(e, cudaMemsetAsync(e->spx.base, 0, e->P * 8, e->side));
            SS_CUDA(e, cudaMemsetAsync(e->spx.n_hot, 0, 4, e->side));
            SS_CUDA(e, cudaMemsetAsync(e->spx.n_stored, 0, 8, e->side));
            ss_note_launch(), ss_launch(k_split_sum, group_grid(e->G), 256, 0, e->side, e->gcount, (uint32_t)e->G, e->W,
                                        e->spx.n_stored, e->bad);
            ss_note_launch(), ss_launch(k_split_hot, 2 * kNumSM, 256, e->P * 4, e->side, e->gcount, (uint32_t)e->G, e->pmap,
                                        (const unsigned long long*)e->spx.n_stored, e->maxS, e->spx, e->P, e->bad, e->W);
            // water-fill the hot groups over this batch's cold loads (the
            // policy's moves apply from the next batch on)
            const SplitPlan& nx = e->plan_buf[plan];
            ss_note_launch(), ss_launch(k_u64_to_i64, 1, 1024, 0, e->side, e->spx.base, e->fill_loads, e->P);
            const size_t smem = (size_t)e->maxS * 20 + 16 + (size_t)(e->P + 1) * 4;
            ss_note_launch(), ss_launch(k_split_fill, 1, 1024, smem, e->side, e->gcount, e->fill_loads, e->P, e->maxS, e->spx, nx, nx,
                                                                       e->bad, e->W);
            SS_CUDA(e, cudaMemsetAsync(e->loads, 0, e->P * 8, e->side));
            ss_note_launch(), ss_launch(k_split_loads, 2 * kNumSM, 256, e->P * 4, e->side, e->gcount, (uint32_t)e->G, e->pmap, e->P,
                                                                                    nx, e->loads, e->bad, e->W);
            SS_CUDA(e, cudaEventRecord(e->ev_bal, e->side));
        }
        if (has_policy) {
            BalanceArgs a{};
            a.policy = pol;
            a.threshold = bal->thread_threshold;
            a.pot = bal->pot;
            a.cap = move_cap(e, bal);
            a.P = e->P;
            a.order = e->order;
            a.offsets = e->offsets;
            a.gcount = e->gcount;
            a.tpt = e->tpt;
            a.moved = e->moved;
            a.moves = e->moves;
            a.front_top = e->front_top;
            a.back_first = e->back_first;
            a.mv_next = e->mv_next;
            a.new_off = e->new_off;
            a.keep_at = e->keep_at;
            a.mv_pos = e->mv_pos;
            a.n_moves = e->n_moves;
            a.scanned = e->scanned;
            a.final_tpt = e->final_tpt;
            a.bad = e->bad;
            if (split) {
                // cold groups only need to move off partitions above the mean:
                // the water level of the hot shares is >= the mean
                a.init_loads = e->spx.base;
                a.exclude = e->spx.hot_flag;
                a.stop_sum = e->spx.n_stored;      // the mean block load in values to store
            }
            ss_note_launch(), launch_balance(e, a, e->side);
        }
        SS_CUDA(e, cudaGetLastError());
    }
    if (!e->ahead) {
        ProfScope ps(e, SS_K_STATS, e->st);
        if ((rc = launch_scans(e, e->gkept, n_chunk))) return rc;
    }
    if (!e->dense) {
        ProfScope ps(e, SS_K_INGEST, e->st);
        SS_CUDA(e, cudaMemsetAsync(e->n_copies, 0, 4, e->st));
        ss_note_launch(), ss_launch(k_reserve, group_grid(e->G), 256, 0, e->st, e->gcount, (uint32_t)e->G, e->W, e->fill, e->off, e->cap,
                                                 e->pool_top, e->pool_cap, e->oom, e->copies, e->n_copies, e->bad);
        ss_note_launch(), ss_launch(k_ring_copy, 8 * kNumSM, 256, 0, e->st, e->copies, e->n_copies, e->ring);
    }
    {
        ProfScope ps(e, SS_K_PLACE, e->st);
        if ((rc = launch_place_step(e, dk, dv, n))) return rc;
    }
    if (e->trace_on) {
        // per-tuple trace sums, from the batch-start ring (before the window update)
        TraceArgs ta{};
        ta.keys = e->keys_final;
        ta.vals = e->vals_final;
        ta.n_dev = e->n_live;
        ta.gstart = e->gstart;
        ta.fill = e->fill;
        ta.next_pos = e->next_pos;
        ta.wsum = e->wsum;
        ta.off = e->off;
        ta.ring = e->ring;
        ta.W = e->W;
        ta.out = e->trace_s;
        ta.tile = e->trace_tile;
        ta.bad = e->bad;
        const unsigned tiles = (unsigned)((n + kTraceTile - 1) / kTraceTile);
        ss_note_launch(), ss_launch(k_trace_local, tiles, kTraceTile, 0, e->st, ta);
        ss_note_launch(), ss_launch(k_trace_tiles, 1, 1024, 0, e->st, ta);
        ss_note_launch(), ss_launch(k_trace_apply, tiles, kTraceTile, 0, e->st, ta);
        SS_CUDA(e, cudaGetLastError());
    }
    if (e->cur_stage >= 0) {
        // the staged input is not read again: the next-but-one batch may reuse it
        SS_CUDA(e, record_ext(e, e->ev_freed[e->cur_stage], e->st));
        e->freed_rec[e->cur_stage] = true;
        e->cur_stage = -1;
    }
    {
        // (the wait for the split plan is outside the timed scope: the
        // class time is the window update's own device time)
        if (split) SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_bal, 0));
        ProfScope ps(e, SS_K_INGEST, e->st);
        IngestArgs a = ingest_args(e, plan);
        // CTAs per partition: with hot-key splitting (or no balancer, static
        // partitions) one resident wave (2 per SM) is best; when the
        // group-reassignment policy runs alone a few partitions carry several
        // times the mean, and 4x the CTAs per partition (later waves,
        // partition-minor order) shortens their tail (measured: 8 CTAs per
        // partition at P = 148 saturates)
        a.cpp = std::max(1, ((split || !has_policy) ? 2 : 8) * kNumSM / e->P);
        unsigned grid = (unsigned)(e->P * a.cpp);
        if (work_grid) {
            ss_note_launch(), ss_launch(k_cta_map, 1, 1024, 0, e->st, e->pwork, e->P, k4_waves * kNumSM, e->cta_map,
                                                               e->cta_used);
            a.cta_map = e->cta_map;
            a.n_used = e->cta_used;
            grid = (unsigned)(k4_waves * kNumSM + e->P);
        }
        ss_note_launch(), ss_launch(k_ingest, grid, kIngestThreads, kIngestSmem, e->st, a);
        SS_CUDA(e, cudaGetLastError());
    }
    if (run_side) SS_CUDA(e, cudaEventRecord(e->ev_k4, e->st));
    {
        ProfScope ps(e, SS_K_EMIT, e->st);
        FinalizeArgs f{};
        f.gcount = e->gcount;
        f.gcnt = e->gcnt;
        f.n_sub = n_chunk;
        f.lc = e->lc;
        f.n_lc = e->n_lc;
        f.G = (uint32_t)e->G;
        f.W = e->W;
        f.fill = e->fill;
        f.next_pos = e->next_pos;
        f.wsum = e->wsum;
        f.mn = e->mn;
        f.mx = e->mx;
        f.bdelta = e->bdelta;
        f.bmin = e->bmin;
        f.bmax = e->bmax;
        f.minmax = e->minmax;
        f.emit = emit;
        f.n_res = e->n_res;
        f.r_g = e->r_g;
        f.r_cnt = e->r_cnt;
        f.r_sum = e->r_sum;
        f.r_avg = e->r_avg;
        f.r_mn = e->r_mn;
        f.r_mx = e->r_mx;
        f.rescan = e->rescan;
        f.n_rescan = e->n_rescan;
        f.sum_idx = e->sum_idx;
        f.sum_valid = e->sum_valid;
        f.n_sum = e->n_sum;
        f.bad = e->bad;
        if (!run_side) {
            // no side-stream work: the last finalize CTA writes the report
            f.report = report_args(e, n, false);
            f.ticket = e->fin_ticket;
        }
        // (at least two CTAs per SM: finalize also clears the live chunks' count rows,
        // 10 MB at C2)
        ss_note_launch(), ss_launch(k_finalize, std::max<unsigned>(group_grid(e->G), 2 * kNumSM), 256, 0, e->st, f);
        if (e->minmax) {
            if (e->sums) {
                ss_note_launch(), ss_launch(k_mm_refresh, 8 * kNumSM, 256, 0, e->st, e->rescan, e->n_rescan, e->ring, e->off, e->W,
                                                                               e->sum_idx, e->sum_valid, e->sums);
                ss_note_launch(), ss_launch(k_mm_fold, 2 * kNumSM, 256, 0, e->st, e->rescan, e->n_rescan, e->W, e->sum_idx,
                                                                            e->sum_valid, e->sums, e->mn, e->mx, e->r_mn,
                                                                            e->r_mx);
            } else {
                ss_note_launch(), ss_launch(k_rescan_reset, 4, 256, 0, e->st, e->rescan, e->n_rescan, e->mn, e->mx);
                ss_note_launch(), ss_launch(k_minmax_rescan, 8 * kNumSM, 256, 0, e->st, e->rescan, e->n_rescan, e->ring, e->off,
                                                                                 e->W, e->mn, e->mx);
                ss_note_launch(), ss_launch(k_rescan_rows, 4, 256, 0, e->st, e->rescan, e->n_rescan, e->mn, e->mx, e->r_mn, e->r_mx);
            }
        }
        if (emit && e->host_emit) {
            const int b = (int)(e->emit_seq & 1);
            ss_note_launch(), ss_launch(k_emit_host, kNumSM, 256, 0, e->st, e->n_res, e->bad, dk, (long long)n, e->r_g, e->r_cnt, e->r_sum,
                                                                     e->r_avg, e->r_mn, e->r_mx, e->d_emit[b]);
            SS_CUDA(e, record_ext(e, e->ev_emit[b], e->st));
            ++e->emit_seq;
        }
        SS_CUDA(e, cudaGetLastError());
    }
    if (run_side) {
        SS_CUDA(e, cudaStreamWaitEvent(e->side, e->ev_k4, 0));
        if (has_policy) {
            ProfScope ps(e, SS_K_APPLY, e->side);
            // (the new offsets and move positions come from k_balance)
            ss_note_launch(), ss_launch(k_apply_place, e->P, 256, 0, e->side, e->order, e->offsets, e->keep_at, e->moves,
                                                                       e->n_moves, e->mv_pos, e->moved, e->new_order);
            ss_note_launch(), ss_launch(k_apply_commit, 2 * kNumSM, 256, 0, e->side, e->order, e->offsets, e->new_order, e->new_off, (int)e->G,
                                                            e->P, e->moves, e->n_moves, e->pmap, e->moved);
            SS_CUDA(e, cudaGetLastError());
        }
        if ((rc = enqueue_report(e, n, has_policy, e->side))) return rc;
        SS_CUDA(e, cudaEventRecord(e->ev_apply, e->side));
        e->side_pending = true;
        if (e->capturing) {
            // a captured step joins its side branch before it ends
            SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_apply, 0));
            e->side_pending = false;
        }
    } else {
        if ((rc = copy_report(e, e->st))) return rc;
    }
    if (split) e->plan_cur ^= 1;
    e->plan_valid = split;
    return SS_OK;
}

// --------------------------------------------------------------------------
// report
// --------------------------------------------------------------------------
static ReportArgs report_args(ss_engine* e, int64_t n, bool has_policy) {
    const bool used_plan = e->last_plan >= 0;
    ReportArgs r{};
    r.tpt = e->tpt;
    r.loads = used_plan ? e->loads : nullptr;
    r.P = e->P;
    r.bad = e->bad;
    r.touched = e->touched;
    r.n_moves = e->n_moves;
    r.prev_moves = e->prev_moves;
    r.scanned = e->scanned;
    r.n_split = used_plan ? e->plan_buf[e->last_plan].n_split : nullptr;
    // (the result-row count is read from n_res by the result calls; the
    // side-stream report may run before finalize, so it is not copied here)
    r.n_res = nullptr;
    r.oom = e->oom;
    r.tuples = (long long)n;
    r.has_policy = has_policy ? 1 : 0;
    r.rep = (long long*)e->d_rep;
    return r;
}

// copy of the device report to the host (after k_report, or after the
// k_finalize that wrote it when no side-stream work ran)
static int copy_report(ss_engine* e, cudaStream_t st) {
    SS_CUDA(e, cudaMemcpyAsync(e->h_rep, e->d_rep, sizeof(DevReport), cudaMemcpyDeviceToHost, st));
    return SS_OK;
}

static int enqueue_report(ss_engine* e, int64_t n, bool has_policy, cudaStream_t st) {
    ss_note_launch(), ss_launch(k_report, 1, 1024, 0, st, report_args(e, n, has_policy));
    SS_CUDA(e, cudaGetLastError());
    return copy_report(e, st);
}


// the key stream's bad-tuple flag into the batch's (engine stream)
__global__ void k_merge_bad(unsigned long long* __restrict__ bad, unsigned long long* __restrict__ key_bad) { SS_PDL_ENTRY();
    if (threadIdx.x != 0) return;
    const unsigned long long k = *key_bad;
    if (k != (unsigned long long)kNoBad) {
        if (k < *bad) *bad = k;
        *key_bad = (unsigned long long)kNoBad;
    }
}

// free the key-table entries a rejected int64-key batch claimed
static void key_rollback(ss_engine* e) {
    const int64_t n_ent = (int64_t)e->kt.cap_mask + 2;
    ss_note_launch(), ss_launch(k_key_rollback, (unsigned)std::min<int64_t>((n_ent + 255) / 256, 16 * kNumSM), 256, 0,
                                e->st, e->kt, n_ent);
    cudaStreamSynchronize(e->st);
}

static int check_report(ss_engine* e, const uint32_t* dk) {
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->side));
    if (e->kst) SS_CUDA(e, cudaStreamSynchronize(e->kst));
    SS_CUDA(e, cudaGetLastError());
    if (e->h_rep->bad != (unsigned long long)kNoBad) {
        if (e->keys64) key_rollback(e);
        return data_error(e, e->h_rep->bad, dk);
    }
    if (e->h_rep->oom) return fail(e, SS_E_EXEC, "window ring pool exhausted (raise pool_values)");
    if (e->keys64) {
        int ov = 0;
        SS_CUDA(e, cudaMemcpy(&ov, e->kt.overflow, 4, cudaMemcpyDeviceToHost));
        if (ov) {
            key_rollback(e);
            recover_bad(e);
            return fail(e, SS_E_DATA, "more than n_groups distinct keys");
        }
    }
    return SS_OK;
}

static void fill_report(const ss_engine* e, ss_step_report* r) {
    const DevReport& d = *e->h_rep;
    r->tuples = d.tuples;
    r->imbalance = d.imbalance;
    r->moves = d.moves;
    r->moves_applied_before = d.moves_before;
    r->scanned = d.scanned;
    r->max_load = d.max_load;
    r->touched = d.touched;
    r->split_groups = d.split_groups;
    // max / mean over one unit: tuples without a split plan, values to
    // store (min(count, W) per group) with one (split.cuh)
    r->mean_load = e->P ? (double)d.load_sum / (double)e->P : 0.0;
    r->load_ratio = (d.load_sum > 0) ? (double)d.max_load / r->mean_load : 0.0;
}

// the count (or int64 probe + count) of batch t+1 on its own stream while
// batch t finishes: alternating count rows (and slot buffers for int64
// keys), the events ordering it, a separate bad-tuple flag
static int create_count_pipe(ss_engine* e) {
    int rc;
    SS_CUDA(e, cudaStreamCreateWithFlags(&e->kst, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_keys[b], cudaEventDisableTiming));
        SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_fin[b], cudaEventDisableTiming));
    }
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_hot, cudaEventDisableTiming));
    SS_CUDA(e, cudaEventCreateWithFlags(&e->ev_in, cudaEventDisableTiming));
    e->gcnt_buf[0] = e->gcnt;
    e->skeys_buf[0] = e->stage_keys;
    if ((rc = dalloc(e, &e->gcnt_buf[1], (size_t)e->n_sub_max * e->G)) || (rc = dalloc(e, &e->key_bad, 1)) ||
        (e->keys64 && (rc = dalloc(e, &e->skeys_buf[1], e->max_batch))))
        return rc;
    SS_CUDA(e, cudaMemsetAsync(e->gcnt_buf[1], 0, (size_t)e->n_sub_max * e->G * 4, e->st));
    ss_note_launch(), ss_launch(k_set_bad, 1, 1, 0, e->st, e->key_bad);
    return SS_OK;
}

static int ensure_moves(ss_engine* e, int64_t want) {
    want = std::min<int64_t>(want, e->G);
    if (want <= e->cap_moves) return SS_OK;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->side));
    int rc;
    if ((rc = dalloc(e, &e->moves, want)) || (rc = dalloc(e, &e->mv_next, want)) || (rc = dalloc(e, &e->mv_pos, want)))
        return rc;
    e->cap_moves = (int)want;
    // captured step graphs hold the old move buffers
    for (auto& g : e->graphs) cudaGraphExecDestroy(g.exec);
    e->graphs.clear();
    return SS_OK;
}

static int move_cap(ss_engine* e, const ss_balancer* b) {
    const int64_t want = b->max_moves > 0 ? b->max_moves : 4LL * e->P;
    return (int)std::min<int64_t>(want, e->cap_moves);
}

static int check_balancer(ss_engine* e, const ss_balancer* b) {
    if (!b) return SS_OK;
    if (b->policy < SS_POLICY_NO || b->policy > SS_POLICY_SHIFTLOCAL)
        return fail(e, SS_E_CONFIG, "unknown policy " + std::to_string(b->policy));
    if (b->thread_threshold < 1) return fail(e, SS_E_CONFIG, "thread_threshold must be >= 1");
    if (!(b->pot > 0.0 && b->pot <= 1.0)) return fail(e, SS_E_CONFIG, "pot must be in (0, 1]");
    if (b->max_moves < 0) return fail(e, SS_E_CONFIG, "max_moves must be >= 1 (0 = default)");
    return ensure_moves(e, b->max_moves > 0 ? b->max_moves : 4LL * e->P);
}

// --------------------------------------------------------------------------
// assignment
// --------------------------------------------------------------------------
extern "C" int ss_set_assignment(ss_engine* e, const int32_t* order, const int64_t* offsets) {
    if (!e || !order || !offsets) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    const int64_t G = e->G;
    const int P = e->P;
    if (offsets[0] != 0 || offsets[P] != G) return fail(e, SS_E_CONSISTENCY, "offsets must span [0, G]");
    std::vector<int32_t> pmap(G, -1), offs(P + 1);
    for (int p = 0; p < P; ++p) {
        if (offsets[p + 1] < offsets[p]) return fail(e, SS_E_CONSISTENCY, "offsets must be non-decreasing");
        offs[p] = (int32_t)offsets[p];
        for (int64_t i = offsets[p]; i < offsets[p + 1]; ++i) {
            const int32_t g = order[i];
            if (g < 0 || g >= G) return fail(e, SS_E_CONSISTENCY, "group " + std::to_string(g) + " out of range");
            if (pmap[g] >= 0) return fail(e, SS_E_CONSISTENCY, "group " + std::to_string(g) + " listed twice");
            pmap[g] = p;
        }
    }
    offs[P] = (int32_t)G;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaMemcpy(e->order, order, G * 4, cudaMemcpyHostToDevice));
    SS_CUDA(e, cudaMemcpy(e->pmap, pmap.data(), G * 4, cudaMemcpyHostToDevice));
    SS_CUDA(e, cudaMemcpy(e->offsets, offs.data(), (P + 1) * 4, cudaMemcpyHostToDevice));
    return SS_OK;
}

extern "C" int ss_get_assignment(ss_engine* e, int32_t* g2t, int32_t* order, int64_t* offsets) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (g2t) SS_CUDA(e, cudaMemcpy(g2t, e->pmap, e->G * 4, cudaMemcpyDeviceToHost));
    if (order) SS_CUDA(e, cudaMemcpy(order, e->order, e->G * 4, cudaMemcpyDeviceToHost));
    if (offsets) {
        std::vector<int32_t> o(e->P + 1);
        SS_CUDA(e, cudaMemcpy(o.data(), e->offsets, (e->P + 1) * 4, cudaMemcpyDeviceToHost));
        for (int p = 0; p <= e->P; ++p) offsets[p] = o[p];
    }
    return SS_OK;
}

// Sequential application with the reference's validation order
// (partition.py:181-203); the engine is untouched when a move fails.
extern "C" int ss_apply_moves(ss_engine* e, const ss_move* moves, int64_t n) {
    if (!e) return SS_E_CONFIG;
    const int64_t G = e->G;
    const int P = e->P;
    std::vector<int32_t> g2t(G), order(G);
    std::vector<int64_t> offs(P + 1);
    int rc = ss_get_assignment(e, g2t.data(), order.data(), offs.data());
    if (rc) return rc;
    std::vector<std::vector<int32_t>> lists(P);
    for (int p = 0; p < P; ++p) lists[p].assign(order.begin() + offs[p], order.begin() + offs[p + 1]);
    for (int64_t i = 0; i < n; ++i) {
        const ss_move& m = moves[i];
        if (m.placement != SS_FRONT && m.placement != SS_BACK)
            return fail(e, SS_E_CONFIG, "unknown placement " + std::to_string(m.placement));
        if (m.src < 0 || m.src >= P || m.dst < 0 || m.dst >= P)
            return fail(e, SS_E_CONFIG, "move " + std::to_string(i) + " names a thread out of range");
        if (m.group < 0 || m.group >= G)
            return fail(e, SS_E_CONFIG, "move " + std::to_string(i) + " names a group out of range");
        if (g2t[m.group] != m.src)
            return fail(e, SS_E_STALE_MOVE, "group " + std::to_string(m.group) + " is on thread " +
                                                std::to_string(g2t[m.group]) + ", not " + std::to_string(m.src));
        auto& src = lists[m.src];
        src.erase(std::find(src.begin(), src.end(), m.group));
        auto& dst = lists[m.dst];
        if (m.placement == SS_BACK) dst.push_back(m.group);
        else dst.insert(dst.begin(), m.group);
        g2t[m.group] = m.dst;
    }
    int64_t pos = 0;
    for (int p = 0; p < P; ++p) {
        offs[p] = pos;
        for (int32_t g : lists[p]) order[pos++] = g;
    }
    offs[P] = pos;
    return ss_set_assignment(e, order.data(), offs.data());
}

// --------------------------------------------------------------------------
// partition step
// --------------------------------------------------------------------------
static int64_t round_chunk(int64_t n) {
    return std::max<int64_t>(kCountChunk, ((n + kCountChunk - 1) / kCountChunk) * kCountChunk);
}

static int clear_counts_row0(ss_engine* e) {
    SS_CUDA(e, cudaMemsetAsync(e->gcnt, 0, e->G * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->gcount, 0, e->G * 4, e->st));
    return SS_OK;
}

extern "C" int ss_count(ss_engine* e, const uint32_t* groups, int64_t n, int64_t* group_counts, int64_t* tpt) {
    if (!e || n < 0) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    const uint32_t* dk;
    int rc;
    if ((rc = stage_input(e, groups, nullptr, n, &dk, nullptr))) return rc;
    if ((rc = launch_count(e, dk, n, round_chunk(n)))) return rc;
    if ((rc = launch_stats(e, 1))) return rc;
    unsigned long long bad;
    SS_CUDA(e, cudaMemcpyAsync(&bad, e->bad, 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (bad != (unsigned long long)kNoBad) return data_error(e, bad, dk);
    std::vector<int32_t> gc(e->G);
    std::vector<unsigned long long> tp(e->P);
    SS_CUDA(e, cudaMemcpy(gc.data(), e->gcount, e->G * 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(tp.data(), e->tpt, e->P * 8, cudaMemcpyDeviceToHost));
    if ((rc = clear_counts_row0(e))) return rc;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (group_counts)
        for (int64_t g = 0; g < e->G; ++g) group_counts[g] = gc[g];
    if (tpt)
        for (int p = 0; p < e->P; ++p) tpt[p] = (int64_t)tp[p];
    return SS_OK;
}

extern "C" int ss_reorder(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                          uint32_t* out_groups, int32_t* out_attrs, int64_t* indicator) {
    if (!e || n < 0) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    const uint32_t* dk;
    const int32_t* dv;
    int rc;
    if ((rc = stage_input(e, groups, attrs, n, &dk, &dv))) return rc;
    if ((rc = engine_alloc_sort(e, n))) return rc;
    int32_t* rank = e->new_order;   // scratch: only the apply kernels use it, inside a step
    ss_note_launch(), ss_launch(k_rank_of, 2 * kNumSM, 256, 0, e->st, e->order, e->G, rank);
    if (n) ss_note_launch(), ss_launch(k_to_rank, 2 * kNumSM, 256, 0, e->st, dk, n, rank, (uint32_t)e->G, e->stage_keys, e->bad);
    const uint32_t* rk = e->stage_keys;
    if ((rc = launch_count(e, rk, n, round_chunk(n)))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->tickets, 0, 8, e->st));
    if ((rc = launch_scans(e, e->gcnt))) return rc;
    if (n && (rc = launch_place_all(e, rk, dv, n))) return rc;
    if (n) ss_note_launch(), ss_launch(k_from_rank, 2 * kNumSM, 256, 0, e->st, e->kbuf2, n, e->order);
    unsigned long long bad;
    SS_CUDA(e, cudaMemcpyAsync(&bad, e->bad, 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (bad != (unsigned long long)kNoBad) {
        // report the original group of the offending tuple
        uint32_t g = 0;
        if (is_device_ptr(groups)) cudaMemcpy(&g, groups + bad, 4, cudaMemcpyDeviceToHost);
        else g = groups[bad];
        recover_bad(e);
        return fail(e, SS_E_DATA, "tuple " + std::to_string(bad) + " has group " + std::to_string(g) +
                                      ", outside [0, " + std::to_string(e->G) + ")");
    }
    if (n) {
        SS_CUDA(e, cudaMemcpy(out_groups, e->kbuf2, n * 4, is_device_ptr(out_groups) ? cudaMemcpyDeviceToDevice
                                                                                       : cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(out_attrs, e->vbuf[0], n * 4, is_device_ptr(out_attrs) ? cudaMemcpyDeviceToDevice
                                                                                      : cudaMemcpyDeviceToHost));
    }
    if (indicator) {
        std::vector<int32_t> offs(e->P + 1), gst(e->G);
        SS_CUDA(e, cudaMemcpy(offs.data(), e->offsets, (e->P + 1) * 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(gst.data(), e->gstart, e->G * 4, cudaMemcpyDeviceToHost));
        for (int p = 0; p <= e->P; ++p) indicator[p] = (offs[p] < e->G) ? gst[offs[p]] : n;
        if (n == 0)
            for (int p = 0; p <= e->P; ++p) indicator[p] = 0;
    }
    if ((rc = clear_counts_row0(e))) return rc;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// --------------------------------------------------------------------------
// aggregate update / balancer / fused step
// --------------------------------------------------------------------------
extern "C" int ss_ingest(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n) {
    if (!e || n < 0) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    if (n == 0) return SS_OK;
    const uint32_t* dk;
    const int32_t* dv;
    int rc;
    if ((rc = stage_input(e, groups, attrs, n, &dk, &dv))) return rc;
    e->last_plan = -1;
    if ((rc = run_batch(e, dk, dv, n, nullptr, false))) return rc;
    return check_report(e, dk);
}

extern "C" int ss_balance(ss_engine* e, const uint32_t* groups, int64_t n, const ss_balancer* cfg,
                          ss_move* moves, int64_t* n_moves, int64_t* scanned, int64_t* final_tpt) {
    if (!e || !cfg || n < 0) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    const uint32_t* dk;
    if ((rc = stage_input(e, groups, nullptr, n, &dk, nullptr))) return rc;
    if ((rc = launch_count(e, dk, n, round_chunk(n)))) return rc;
    if ((rc = launch_stats(e, 1))) return rc;
    int nm = 0;
    long long sc = 0;
    std::vector<long long> ft(e->P);
    if (cfg->policy == SS_POLICY_NO) {
        std::vector<unsigned long long> tp(e->P);
        SS_CUDA(e, cudaMemcpyAsync(tp.data(), e->tpt, e->P * 8, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaStreamSynchronize(e->st));
        for (int p = 0; p < e->P; ++p) ft[p] = (long long)tp[p];
    } else {
        BalanceArgs a{};
        a.policy = cfg->policy;
        a.threshold = cfg->thread_threshold;
        a.pot = cfg->pot;
        a.cap = move_cap(e, cfg);
        a.P = e->P;
        a.order = e->order;
        a.offsets = e->offsets;
        a.gcount = e->gcount;
        a.tpt = e->tpt;
        a.moved = e->moved;
        a.moves = e->moves;
        a.front_top = e->front_top;
        a.back_first = e->back_first;
        a.mv_next = e->mv_next;
        a.n_moves = e->n_moves;
        a.scanned = e->scanned;
        a.final_tpt = e->final_tpt;
        a.bad = e->bad;
        ss_note_launch(), launch_balance(e, a, e->st);
        SS_CUDA(e, cudaGetLastError());
        ss_note_launch(), ss_launch(k_clear_moved, 4, 256, 0, e->st, e->moves, e->n_moves, e->moved);
        SS_CUDA(e, cudaMemcpyAsync(&nm, e->n_moves, 4, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaMemcpyAsync(&sc, e->scanned, 8, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaMemcpyAsync(ft.data(), e->final_tpt, e->P * 8, cudaMemcpyDeviceToHost, e->st));
    }
    unsigned long long bad;
    SS_CUDA(e, cudaMemcpyAsync(&bad, e->bad, 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (bad != (unsigned long long)kNoBad) return data_error(e, bad, dk);
    if (nm > 0 && moves) {
        std::vector<int4> mv(nm);
        SS_CUDA(e, cudaMemcpy(mv.data(), e->moves, nm * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nm; ++i) moves[i] = ss_move{mv[i].x, mv[i].y, mv[i].z, mv[i].w};
    }
    if (n_moves) *n_moves = nm;
    if (scanned) *scanned = sc;
    if (final_tpt)
        for (int p = 0; p < e->P; ++p) final_tpt[p] = ft[p];
    // the MoveList is emitted but not applied (policies are pure)
    SS_CUDA(e, cudaMemsetAsync(e->n_moves, 0, 4, e->st));
    if ((rc = clear_counts_row0(e))) return rc;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// --------------------------------------------------------------------------
// the fused step as a replayed CUDA graph
// --------------------------------------------------------------------------
struct HostState {
    int plan_cur, last_plan;
    bool plan_valid, side_pending;
    long long emit_seq, alg_input;
    int cur_stage;
    bool freed0, freed1;
    bool operator==(const HostState& o) const {
        return plan_cur == o.plan_cur && last_plan == o.last_plan && plan_valid == o.plan_valid &&
               side_pending == o.side_pending && emit_seq == o.emit_seq && alg_input == o.alg_input &&
               cur_stage == o.cur_stage && freed0 == o.freed0 && freed1 == o.freed1;
    }
};
static HostState get_state(const ss_engine* e) {
    return {e->plan_cur, e->last_plan, e->plan_valid, e->side_pending, e->emit_seq, e->alg_input,
            e->cur_stage, e->freed_rec[0], e->freed_rec[1]};
}
static void set_state(ss_engine* e, const HostState& h) {
    e->plan_cur = h.plan_cur; e->last_plan = h.last_plan; e->plan_valid = h.plan_valid;
    e->side_pending = h.side_pending; e->emit_seq = h.emit_seq; e->alg_input = h.alg_input;
    e->cur_stage = h.cur_stage; e->freed_rec[0] = h.freed0; e->freed_rec[1] = h.freed1;
}
// the host bookkeeping run_batch(emit = true) performs, for a replayed graph
// (which joins its side branch before it ends)
static HostState step_transition(const ss_engine* e, int64_t n, const ss_balancer* bal) {
    HostState h = get_state(e);
    const bool split = bal && bal->split;
    h.last_plan = split ? (e->plan_cur ^ 1) : -1;
    h.alg_input += (e->keys64 ? 12 : 8) * n;
    if (split) h.plan_cur ^= 1;
    h.plan_valid = split;
    if (h.cur_stage == 0) h.freed0 = true;
    if (h.cur_stage == 1) h.freed1 = true;
    h.cur_stage = -1;
    if (e->host_emit) ++h.emit_seq;
    h.side_pending = false;
    return h;
}

static bool same_bal(const ss_balancer* a, const ss_balancer& b) {
    ss_balancer z{};
    const ss_balancer& x = a ? *a : z;
    return memcmp(&x, &b, sizeof(ss_balancer)) == 0;
}

static int run_step(ss_engine* e, const uint32_t* dk, const int32_t* dv, int64_t n, const ss_balancer* bal) {
    if (!e->graphs_on || e->prof || e->trace_on) return run_batch(e, dk, dv, n, bal, true);
    int rc;
    if (e->side_pending) {                       // graphs are self-contained: join the last side work
        SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_apply, 0));
        e->side_pending = false;
    }
    const int emit_b = (int)(e->emit_seq & 1);
    ss_engine::GraphEntry* hit = nullptr;
    for (auto& g : e->graphs)
        if (g.dk == dk && g.dv == dv && g.n == n && same_bal(bal, g.bal) && g.plan_cur == e->plan_cur &&
            g.plan_valid == (int)e->plan_valid && g.emit_b == emit_b && g.host_emit == (int)e->host_emit &&
            g.stage == e->cur_stage && g.pre_counted == (int)e->pre_counted && g.gcnt == (const void*)e->gcnt) {
            hit = &g;
            break;
        }
    if (hit) ++e->graph_hits;
    if (!hit && e->graph_captures >= 8 && e->graph_hits < 2 * e->graph_captures) {
        // inputs that change every batch (e.g. freshly exchanged buffers):
        // capturing would cost more than it saves
        e->graphs_on = false;
        return run_batch(e, dk, dv, n, bal, true);
    }
    if (!hit) {
        ++e->graph_captures;
        const HostState s0 = get_state(e);
        const HostState expect = step_transition(e, n, bal);
        const long long l0 = g_launches.load();
        cudaGraph_t graph = nullptr;
        e->capturing = true;
        cudaError_t err = cudaStreamBeginCapture(e->st, cudaStreamCaptureModeRelaxed);
        rc = (err == cudaSuccess) ? run_batch(e, dk, dv, n, bal, true) : SS_E_EXEC;
        const cudaError_t err2 = cudaStreamEndCapture(e->st, &graph);
        e->capturing = false;
        const HostState s1 = get_state(e);
        cudaGraphExec_t exec = nullptr;
        if (err == cudaSuccess && rc == SS_OK && err2 == cudaSuccess && graph)
            err = cudaGraphInstantiate(&exec, graph, 0);
        else
            err = cudaErrorStreamCaptureInvalidated;
        if (graph) cudaGraphDestroy(graph);
        const long long per_replay = g_launches.load() - l0;   // kernels recorded by the capture
        g_launches.store(l0);
        set_state(e, s0);
        if (err != cudaSuccess || !(s1 == expect)) {
            // capture not possible here (or the bookkeeping model disagrees):
            // run this and every later batch without graphs
            if (exec) cudaGraphExecDestroy(exec);
            cudaGetLastError();
            e->graphs_on = false;
            return run_batch(e, dk, dv, n, bal, true);
        }
        if (e->graphs.size() >= 16) {
            cudaGraphExecDestroy(e->graphs.front().exec);
            e->graphs.erase(e->graphs.begin());
        }
        ss_engine::GraphEntry ge{};
        ge.dk = dk;
        ge.dv = dv;
        ge.n = n;
        if (bal) ge.bal = *bal;
        ge.plan_cur = e->plan_cur;
        ge.plan_valid = (int)e->plan_valid;
        ge.emit_b = emit_b;
        ge.host_emit = (int)e->host_emit;
        ge.stage = e->cur_stage;
        ge.pre_counted = (int)e->pre_counted;
        ge.gcnt = e->gcnt;
        ge.exec = exec;
        ge.launches = per_replay;
        e->graphs.push_back(ge);
        hit = &e->graphs.back();
    }
    SS_CUDA(e, cudaGraphLaunch(hit->exec, e->st));
    g_launches.fetch_add(hit->launches);
    set_state(e, step_transition(e, n, bal));
    return SS_OK;
}

// stream-scope window: one batch (see streamwin.cuh)
__global__ void k_sw_report(const unsigned long long* bad, long long n, const unsigned long long* touched,
                            const unsigned* n_res, DevReport* rep) { SS_PDL_ENTRY();
    DevReport r{};
    r.bad = *bad;
    r.tuples = n;
    r.touched = (long long)*touched;
    r.n_res = *n_res;
    *rep = r;
}

static int run_stream(ss_engine* e, const uint32_t* dk, const int32_t* dv, int64_t n) {
    const int64_t W = e->W;
    const int64_t m = std::min<int64_t>(n, W);
    StreamWinArgs a{};
    a.keys = dk;
    a.vals = dv;
    a.n = n;
    a.m = m;
    a.ring_k = e->sw_k;
    a.ring_v = e->sw_v;
    a.W = W;
    a.cur = e->sw_cur;
    a.G = (uint32_t)e->G;
    a.count = e->fill;
    a.sum = e->wsum;
    a.mn = e->mn;
    a.mx = e->mx;
    a.touched = e->sw_touched;
    a.bad = e->bad;
    SS_CUDA(e, cudaMemsetAsync(e->n_res, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->touched, 0, 8, e->st));
    ss_note_launch(), ss_launch(k_sw_check, 4 * kNumSM, 256, 0, e->st, a);
    ss_note_launch(), ss_launch(k_sw_evict, 4 * kNumSM, 256, 0, e->st, a);
    ss_note_launch(), ss_launch(k_sw_add, 4 * kNumSM, 256, 0, e->st, a);
    if (e->minmax) {
        ss_note_launch(), ss_launch(k_sw_mm_reset, 2 * kNumSM, 256, 0, e->st, a);
        ss_note_launch(), ss_launch(k_sw_mm_scan, 4 * kNumSM, 256, 0, e->st, a);
    }
    StreamEmitArgs f{};
    f.G = (uint32_t)e->G;
    f.count = e->fill;
    f.sum = e->wsum;
    f.mn = e->mn;
    f.mx = e->mx;
    f.minmax = e->minmax;
    f.touched = e->sw_touched;
    f.n_res = e->n_res;
    f.r_g = e->r_g;
    f.r_cnt = e->r_cnt;
    f.r_sum = e->r_sum;
    f.r_avg = e->r_avg;
    f.r_mn = e->r_mn;
    f.r_mx = e->r_mx;
    f.touched_total = e->touched;
    f.bad = e->bad;
    ss_note_launch(), ss_launch(k_sw_emit, 2 * kNumSM, 256, 0, e->st, f);
    ss_note_launch(), ss_launch(k_sw_advance, 1, 1, 0, e->st, a);
    ss_note_launch(), ss_launch(k_sw_report, 1, 1, 0, e->st, e->bad, (long long)n, e->touched, e->n_res, e->d_rep);
    SS_CUDA(e, cudaMemcpyAsync(e->h_rep, e->d_rep, sizeof(DevReport), cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaGetLastError());
    if (e->cur_stage >= 0) {
        SS_CUDA(e, cudaEventRecord(e->ev_freed[e->cur_stage], e->st));
        e->freed_rec[e->cur_stage] = true;
        e->cur_stage = -1;
    }
    return SS_OK;
}

extern "C" int ss_step(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                       const ss_balancer* cfg, ss_step_report* rep) {
    NvtxRange nv_("ss_step");
    if (!e || n < 0) return SS_E_CONFIG;
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    const uint32_t* dk = groups;
    const int32_t* dv = attrs;
    bool staged_here = false;
    if (!is_device_ptr(groups) || (attrs && !is_device_ptr(attrs))) {
        // host buffers: H2D on the copy stream into this batch's staging
        // buffer, overlapped with the previous batch's compute
        staged_here = true;
        if ((rc = begin_stage(e, false))) return rc;
        const int b = e->cur_stage;
        if ((rc = stage_h2d(e, e->skeys[b], groups, n, &dk)) || (rc = stage_h2d(e, e->svals[b], attrs, n, &dv)) ||
            (rc = end_stage(e)))
            return rc;
    }
    e->last_keys = dk;
    const bool has_policy = cfg && cfg->policy != SS_POLICY_NO;
    e->last_plan = -1;
    if (e->stream_scope) {
        if (cfg && (cfg->policy != SS_POLICY_NO || cfg->split))
            return fail(e, SS_E_CONFIG, "the balancer works on per-group windows: use policy 'no' with scope 'stream'");
        if ((rc = run_stream(e, dk, dv, n))) return rc;
        if (rep) {
            if ((rc = check_report(e, dk))) {
                // a bad batch changes nothing: validation runs before any update
                return rc;
            }
            fill_report(e, rep);
        }
        return SS_OK;
    }
    const bool ahead = n > 0 && e->ahead_ok && !has_policy && !(cfg && cfg->split) && !e->trace_on && !e->prof &&
                       !e->pre_counted;
    if (ahead) {
        // count + statistics + scans + sub-chunk prefixes of this batch on
        // the count stream into the alternate per-batch arrays, while the
        // previous batch places and updates windows on the engine stream
        const int b = e->kpar;
        e->kpar ^= 1;
        if (staged_here) {
            SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_staged[e->cur_stage], 0));
        } else if (!e->key_pipe_dev || e->inputs_on_stream) {
            SS_CUDA(e, cudaEventRecord(e->ev_in, e->st));
            SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_in, 0));
        }
        if (e->fin_rec[b]) SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_fin[b], 0));
        use_ahead_set(e, b);
        const int n_chunk = (int)std::max<int64_t>(1, (n + e->S - 1) / e->S);
        int cs = 0;
        while ((int64_t(1) << cs) < e->S) ++cs;
        cudaStream_t const st0 = e->st;
        e->st = e->kst;                      // the launch helpers enqueue on e->st
        {
            NvtxRange nv2("ss count + stats + scans (ahead)");
            ss_note_launch(), ss_launch(k_count_rows, n_chunk, 512, e->G * 4, e->kst, dk, n, (uint32_t)e->G, e->S,
                                        e->gcnt, e->key_bad, ((uintptr_t)dk % 16) == 0);
            rc = launch_stats(e, n_chunk, true, false);
            if (!rc) rc = launch_scans(e, e->gkept, n_chunk);
            if (!rc) launch_sub_prefix(e, dk, n, cs);
        }
        e->st = st0;
        if (rc) {
            use_ahead_set(e, 0);
            return rc;
        }
        SS_CUDA(e, cudaGetLastError());
        SS_CUDA(e, cudaEventRecord(e->ev_keys[b], e->kst));
        SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_keys[b], 0));
        ss_note_launch(), ss_launch(k_merge_bad, 1, 32, 0, e->st, e->bad, e->key_bad);
        e->ahead = true;
        e->pre_counted = true;
        rc = run_step(e, dk, dv, n, cfg);
        e->pre_counted = false;
        e->ahead = false;
        use_ahead_set(e, 0);
        if (rc) return rc;
        SS_CUDA(e, cudaEventRecord(e->ev_fin[b], e->st));
        e->fin_rec[b] = true;
    } else if (n > 0 && e->kst && !e->keys64 && !e->pre_counted) {
        // the count rows of this batch on the count stream (overlapping the
        // previous batch's tail), into the alternate rows (see ss_step_keys64)
        const int b = e->kpar;
        e->kpar ^= 1;
        if (staged_here) {
            SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_staged[e->cur_stage], 0));
        } else if (!e->key_pipe_dev || e->inputs_on_stream) {
            // device keys may be produced by work already on the engine
            // stream (replay records split there): wait for it -- no overlap
            SS_CUDA(e, cudaEventRecord(e->ev_in, e->st));
            SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_in, 0));
        }
        if (e->fin_rec[b]) SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_fin[b], 0));
        const int n_chunk = (int)std::max<int64_t>(1, (n + e->S - 1) / e->S);
        {
            NvtxRange nv2("ss count (ahead)");
            if (e->G <= 16384) {
                ss_note_launch(), ss_launch(k_count_rows, n_chunk, 512, e->G * 4, e->kst, dk, n, (uint32_t)e->G, e->S,
                                            e->gcnt_buf[b], e->key_bad, ((uintptr_t)dk % 16) == 0);
            } else {
                // large G: the previous batch's hot-group cache (k_hot_select)
                // must be complete; the rows are zero (finalize / stats keep them so)
                if (e->hot_rec) SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_hot, 0));
                const int64_t grid = (n + kCountChunk - 1) / kCountChunk;
                ss_note_launch(), ss_launch(k_count<false>, (unsigned)grid, 512, (size_t)kHotCache * 4, e->kst, dk, n,
                                            (uint32_t)e->G, e->S, kCountChunk, e->gcnt_buf[b], e->key_bad,
                                            (int)(((uintptr_t)dk % 16) == 0), (const int32_t*)e->hot_of,
                                            (const int32_t*)e->hot_g, kHotCache);
            }
        }
        SS_CUDA(e, cudaGetLastError());
        SS_CUDA(e, cudaEventRecord(e->ev_keys[b], e->kst));
        SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_keys[b], 0));
        ss_note_launch(), ss_launch(k_merge_bad, 1, 32, 0, e->st, e->bad, e->key_bad);
        int32_t* const gcnt0 = e->gcnt;
        e->gcnt = e->gcnt_buf[b];
        e->pre_counted = true;
        rc = run_step(e, dk, dv, n, cfg);
        e->pre_counted = false;
        e->gcnt = gcnt0;
        if (rc) return rc;
        SS_CUDA(e, cudaEventRecord(e->ev_fin[b], e->st));
        e->fin_rec[b] = true;
    } else if (n > 0 && (rc = run_step(e, dk, dv, n, cfg))) {
        return rc;
    }
    if (n == 0) {
        if (e->side_pending) {
            SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_apply, 0));
            e->side_pending = false;
        }
        SS_CUDA(e, cudaMemsetAsync(e->tpt, 0, e->P * 8, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->touched, 0, 8, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->n_res, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->n_moves, 0, 4, e->st));
        SS_CUDA(e, cudaMemsetAsync(e->scanned, 0, 8, e->st));
        if ((rc = enqueue_report(e, 0, has_policy, e->st))) return rc;
    }
    if (rep) {
        if ((rc = check_report(e, dk))) return rc;
        fill_report(e, rep);
    }
    return SS_OK;
}

// replay ingest: a batch of 8-byte (u32 group, i32 attr)
// records -- the reference's replay-file format, datagen.py:29,250-296 --
// host (pinned: H2D on the copy stream, overlapped) or device; split into
// the engine's SoA staging buffers on the device, then the fused step
extern "C" int ss_step_records(ss_engine* e, const void* records, int64_t n, const ss_balancer* cfg,
                               ss_step_report* rep) {
    if (!e || n < 0 || (n && !records)) return SS_E_CONFIG;
    if (e->keys64) return fail(e, SS_E_CONFIG, "replay records carry 32-bit group ids (engine has key_bits = 64)");
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    if ((rc = begin_stage(e, false))) return rc;
    const int b = e->cur_stage;
    const uint2* rec = (const uint2*)records;
    if (n && !is_device_ptr(records)) {
        if (!e->srec[b] && (rc = dalloc(e, &e->srec[b], e->max_batch + 2))) return rc;
        SS_CUDA(e, cudaMemcpyAsync(e->srec[b], records, n * 8, cudaMemcpyHostToDevice, e->cp));
        rec = e->srec[b];
    }
    if ((rc = end_stage(e))) return rc;
    if (n) {
        if (((uintptr_t)rec & 15) != 0) return fail(e, SS_E_CONFIG, "device records must be 16-byte aligned");
        ss_note_launch(), ss_launch(k_deinterleave, 4 * kNumSM, 256, 0, e->st, (const uint4*)rec, n, e->skeys[b], e->svals[b]);
        SS_CUDA(e, cudaGetLastError());
    }
    e->inputs_on_stream = true;           // the split keys are engine-stream work
    rc = ss_step(e, e->skeys[b], e->svals[b], n, cfg, rep);
    e->inputs_on_stream = false;
    return rc;
}

extern "C" int ss_set_trace(ss_engine* e, int enable) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int rc;
    if (enable && !e->trace_s) {
        if ((rc = dalloc(e, &e->trace_s, e->max_batch)) ||
            (rc = dalloc(e, &e->trace_tile, e->max_batch / kTraceTile + 2)))
            return rc;
    }
    e->trace_on = enable != 0;
    return SS_OK;
}

extern "C" int ss_trace(ss_engine* e, int64_t cap, int32_t* groups, int64_t* sums, int64_t* n) {
    if (!e) return SS_E_CONFIG;
    if (!e->trace_on) return fail(e, SS_E_CONFIG, "trace mode is off (ss_set_trace)");
    { int jr = join_side(e); if (jr) return jr; }
    int32_t nl = 0;
    SS_CUDA(e, cudaMemcpyAsync(&nl, e->n_live, 4, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (n) *n = nl;
    const int64_t m = std::min<int64_t>(cap, nl);
    if (m > 0 && groups) SS_CUDA(e, cudaMemcpy(groups, e->kbuf2, m * 4, cudaMemcpyDeviceToHost));
    if (m > 0 && sums) SS_CUDA(e, cudaMemcpy(sums, e->trace_s, m * 8, cudaMemcpyDeviceToHost));
    return SS_OK;
}

extern "C" int ss_last_report(ss_engine* e, ss_step_report* rep) {
    if (!e) return SS_E_CONFIG;
    int rc = check_report(e, e->last_keys);
    if (rc) return rc;
    if (rep) fill_report(e, rep);
    return SS_OK;
}

extern "C" int ss_last_loads(ss_engine* e, int64_t* loads) {
    if (!e || !loads) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    std::vector<unsigned long long> t(e->P);
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaMemcpy(t.data(), e->last_plan >= 0 ? e->loads : e->tpt, e->P * 8, cudaMemcpyDeviceToHost));
    for (int p = 0; p < e->P; ++p) loads[p] = (int64_t)t[p];
    return SS_OK;
}

extern "C" int ss_last_part_ns(ss_engine* e, int64_t* ns) {
    if (!e || !ns) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    std::vector<unsigned long long> t(e->P);
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaMemcpy(t.data(), e->part_ns, e->P * 8, cudaMemcpyDeviceToHost));
    for (int p = 0; p < e->P; ++p) ns[p] = (int64_t)t[p];
    return SS_OK;
}

extern "C" int ss_last_part_work(ss_engine* e, int64_t* work) {
    if (!e || !work) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    std::vector<unsigned long long> t(e->P);
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaMemcpy(t.data(), e->part_work, e->P * 8, cudaMemcpyDeviceToHost));
    for (int p = 0; p < e->P; ++p) work[p] = (int64_t)t[p];
    return SS_OK;
}

extern "C" int ss_last_moves(ss_engine* e, ss_move* moves, int64_t cap, int64_t* n) {
    if (!e) return SS_E_CONFIG;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int nm = (int)e->h_rep->moves;
    if (n) *n = nm;
    if (moves && nm > 0) {
        nm = (int)std::min<int64_t>(nm, cap);
        std::vector<int4> mv(nm);
        SS_CUDA(e, cudaMemcpy(mv.data(), e->moves, nm * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nm; ++i) moves[i] = ss_move{mv[i].x, mv[i].y, mv[i].z, mv[i].w};
    }
    return SS_OK;
}

// --------------------------------------------------------------------------
// state export
// --------------------------------------------------------------------------
extern "C" int ss_snapshot(ss_engine* e, int64_t* fill, int64_t* next_pos, int64_t* window_sum, int32_t* mn,
                           int32_t* mx, double* avg) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    const int64_t G = e->G;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    std::vector<int32_t> f(G), np(G);
    std::vector<long long> s(G);
    SS_CUDA(e, cudaMemcpy(f.data(), e->fill, G * 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(np.data(), e->next_pos, G * 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(s.data(), e->wsum, G * 8, cudaMemcpyDeviceToHost));
    if (mn) SS_CUDA(e, cudaMemcpy(mn, e->mn, G * 4, cudaMemcpyDeviceToHost));
    if (mx) SS_CUDA(e, cudaMemcpy(mx, e->mx, G * 4, cudaMemcpyDeviceToHost));
    for (int64_t g = 0; g < G; ++g) {
        if (fill) fill[g] = f[g];
        if (next_pos) next_pos[g] = np[g];
        if (window_sum) window_sum[g] = s[g];
        if (avg) avg[g] = f[g] ? (double)s[g] / (double)f[g] : 0.0;
    }
    return SS_OK;
}

extern "C" int ss_export_values(ss_engine* e, int64_t group, int64_t* out, int64_t cap, int64_t* n) {
    if (!e || group < 0 || group >= e->G) return fail(e, SS_E_CONFIG, "group out of range");
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int32_t f, p;
    int64_t o;
    SS_CUDA(e, cudaMemcpy(&f, e->fill + group, 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(&p, e->next_pos + group, 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(&o, e->off + group, 8, cudaMemcpyDeviceToHost));
    if (n) *n = f;
    if (!out || f == 0) return SS_OK;
    const int64_t span = (f < e->W) ? f : e->W;     // filling windows are linear
    std::vector<int32_t> v(span);
    SS_CUDA(e, cudaMemcpy(v.data(), e->ring + o, span * 4, cudaMemcpyDeviceToHost));
    const int64_t m = std::min<int64_t>(cap, f);
    for (int64_t i = 0; i < m; ++i) out[i] = v[(p + i) % e->W];
    return SS_OK;
}

extern "C" int ss_results(ss_engine* e, int64_t cap, int32_t* groups, int64_t* count, int64_t* sum, double* avg,
                          int32_t* mn, int32_t* mx, int64_t* n) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    unsigned nr = 0;
    SS_CUDA(e, cudaMemcpy(&nr, e->n_res, 4, cudaMemcpyDeviceToHost));
    if (n) *n = nr;
    const int64_t m = std::min<int64_t>(cap, nr);
    if (m <= 0) return SS_OK;
    std::vector<int32_t> rg(nr), rc(nr), rmn(nr), rmx(nr);
    std::vector<long long> rs(nr);
    std::vector<double> ra(nr);
    SS_CUDA(e, cudaMemcpy(rg.data(), e->r_g, nr * 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(rc.data(), e->r_cnt, nr * 4, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(rs.data(), e->r_sum, nr * 8, cudaMemcpyDeviceToHost));
    SS_CUDA(e, cudaMemcpy(ra.data(), e->r_avg, nr * 8, cudaMemcpyDeviceToHost));
    if (e->minmax) {
        SS_CUDA(e, cudaMemcpy(rmn.data(), e->r_mn, nr * 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(rmx.data(), e->r_mx, nr * 4, cudaMemcpyDeviceToHost));
    }
    // emission order is by group id (rows are produced concurrently)
    std::vector<int> idx(nr);
    for (unsigned i = 0; i < nr; ++i) idx[i] = (int)i;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return rg[a] < rg[b]; });
    for (int64_t i = 0; i < m; ++i) {
        const int k = idx[i];
        if (groups) groups[i] = rg[k];
        if (count) count[i] = rc[k];
        if (sum) sum[i] = rs[k];
        if (avg) avg[i] = ra[k];
        if (mn) mn[i] = e->minmax ? rmn[k] : 0;
        if (mx) mx[i] = e->minmax ? rmx[k] : 0;
    }
    return SS_OK;
}

// --------------------------------------------------------------------------
// measurement
// --------------------------------------------------------------------------
extern "C" int ss_profile(ss_engine* e, int enable) {
    if (!e) return SS_E_CONFIG;
    e->prof = enable != 0;
    return SS_OK;
}

extern "C" int ss_profile_read(ss_engine* e, double* ms, int64_t* launches, int reset) {
    if (!e) return SS_E_CONFIG;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->side));
    for (auto& p : e->prof_pending) {
        float t = 0.f;
        SS_CUDA(e, cudaEventElapsedTime(&t, p.a, p.b));
        e->prof_ms[p.cls] += t;
        e->prof_n[p.cls] += 1;
        e->ev_pool.push_back(p.a);
        e->ev_pool.push_back(p.b);
    }
    e->prof_pending.clear();
    for (int c = 0; c < SS_K_NCLASS; ++c) {
        if (ms) ms[c] = e->prof_ms[c];
        if (launches) launches[c] = e->prof_n[c];
        if (reset) { e->prof_ms[c] = 0; e->prof_n[c] = 0; }
    }
    return SS_OK;
}

extern "C" int ss_alg_bytes(ss_engine* e, int64_t* bytes, int reset) {
    if (!e) return SS_E_CONFIG;
    unsigned long long b = 0;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaMemcpy(&b, e->alg_bytes, 8, cudaMemcpyDeviceToHost));
    if (bytes) *bytes = (int64_t)b + e->alg_input;
    if (reset) {
        SS_CUDA(e, cudaMemset(e->alg_bytes, 0, 8));
        e->alg_input = 0;
    }
    return SS_OK;
}

extern "C" int ss_results_raw(ss_engine* e, int64_t cap, int32_t* groups, double* avg, int64_t* n) {
    if (!e) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    unsigned nr = 0;
    SS_CUDA(e, cudaMemcpyAsync(&nr, e->n_res, 4, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (n) *n = nr;
    const int64_t m = std::min<int64_t>(cap, nr);
    if (m > 0 && groups) SS_CUDA(e, cudaMemcpyAsync(groups, e->r_g, m * 4, cudaMemcpyDeviceToHost, e->st));
    if (m > 0 && avg) SS_CUDA(e, cudaMemcpyAsync(avg, e->r_avg, m * 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// --------------------------------------------------------------------------
// multi-GPU: owner map, stable route by owner, direct-count policies,
// window-state migration
// --------------------------------------------------------------------------
extern "C" int ss_set_owner(ss_engine* e, const int32_t* owner_of, int n_dest) {
    if (!e || !owner_of || n_dest < 1 || n_dest > 16) return fail(e, SS_E_CONFIG, "n_dest must be in [1, 16]");
    { int jr = join_side(e); if (jr) return jr; }
    for (int64_t g = 0; g < e->G; ++g)
        if (owner_of[g] < 0 || owner_of[g] >= n_dest) return fail(e, SS_E_CONFIG, "owner out of range");
    int rc;
    if (!e->owner) {
        if ((rc = dalloc(e, &e->owner, e->G)) || (rc = dalloc(e, &e->route_cnt, 16)) ||
            (rc = dalloc(e, &e->route_base, 16)))
            return rc;
    }
    SS_CUDA(e, cudaMemcpyAsync(e->owner, owner_of, e->G * 4, cudaMemcpyHostToDevice, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    e->n_dest = n_dest;
    return SS_OK;
}

// Stable split of a batch by owning GPU: out = [tuples of GPU 0 in arrival
// order] ++ [GPU 1] ++ ...; counts[d] = tuples for GPU d.  One mapped
// multisplit pass (k_sort_pass<4, true>).
extern "C" int ss_route(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n, uint32_t* out_groups,
                        int32_t* out_attrs, int64_t* counts) {
    if (!e || n < 0) return SS_E_CONFIG;
    if (!e->owner) return fail(e, SS_E_CONFIG, "ss_set_owner first");
    { int jr = join_side(e); if (jr) return jr; }
    const uint32_t* dk;
    const int32_t* dv;
    int rc;
    if ((rc = stage_input(e, groups, attrs, n, &dk, &dv))) return rc;
    if ((rc = engine_alloc_sort(e, n))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->route_cnt, 0, 16 * 8, e->st));
    if (n) ss_note_launch(), ss_launch(k_owner_hist, 2 * kNumSM, 256, 0, e->st, dk, n, (uint32_t)e->G, e->owner, e->route_cnt, e->bad);
    unsigned long long hc[16];
    unsigned long long bad;
    SS_CUDA(e, cudaMemcpyAsync(hc, e->route_cnt, 16 * 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaMemcpyAsync(&bad, e->bad, 8, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (bad != (unsigned long long)kNoBad) return data_error(e, bad, dk);
    uint32_t base[16];
    uint64_t run = 0;
    for (int d = 0; d < 16; ++d) {
        base[d] = (uint32_t)run;
        run += hc[d];
        if (counts && d < e->n_dest) counts[d] = (int64_t)hc[d];
    }
    if (n == 0) return SS_OK;
    SS_CUDA(e, cudaMemcpyAsync(e->route_base, base, sizeof(base), cudaMemcpyHostToDevice, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->tickets, 0, 8, e->st));
    const bool dev_out = is_device_ptr(out_groups) && is_device_ptr(out_attrs);
    uint32_t* ko = dev_out ? out_groups : e->kbuf2;
    int32_t* vo = dev_out ? out_attrs : e->vbuf[0];
    ss_note_launch(), ss_launch(k_epoch_bump, 1, 1, 0, e->st, e->ep_dev);
    const int tiles = (int)((n + kSortTile - 1) / kSortTile);
    ss_note_launch(), ss_launch(k_sort_pass<4, true>, std::min(tiles, 2 * kNumSM), kSortThreads, SortSmem<4>::bytes, e->st, dk, dv, ko, vo, (int)n, 0, 15u, e->route_base, e->status, e->ep_dev, 0, e->tickets, e->bad, 0, e->owner, nullptr, SortSeg{});
    SS_CUDA(e, cudaGetLastError());
    if (!dev_out) {
        SS_CUDA(e, cudaMemcpyAsync(out_groups, ko, n * 4, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaMemcpyAsync(out_attrs, vo, n * 4, cudaMemcpyDeviceToHost, e->st));
    }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// batch group counts of the last step (valid until the next step).  A
// device destination is filled stream-ordered (no host synchronisation).
extern "C" int ss_group_counts(ss_engine* e, int32_t* counts) {
    if (!e || !counts) return SS_E_CONFIG;
    if (is_device_ptr(counts)) {
        SS_CUDA(e, cudaMemcpyAsync(counts, e->gcount, e->G * 4, cudaMemcpyDeviceToDevice, e->st));
        return SS_OK;
    }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->side));
    SS_CUDA(e, cudaMemcpy(counts, e->gcount, e->G * 4, cudaMemcpyDeviceToHost));
    return SS_OK;
}

__global__ void k_tpt_from_counts(const int32_t* __restrict__ counts, int64_t G, const int32_t* __restrict__ pmap,
                                  unsigned long long* __restrict__ tpt) { SS_PDL_ENTRY();
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x)
        if (counts[g]) atomicAdd(&tpt[pmap[g]], (unsigned long long)counts[g]);
}

// ---- device-resident multi-GPU data plane ---------------------------------
// Everything below is stream-ordered on the engine's stream and reads
// nothing back to the host: the caller (sharded.py) does one small control
// read per batch (route counts, the bad-tuple status and migration sizes),
// which NCCL's host API needs for the all-to-all split sizes.

// route bases from the owner histogram; counts_dev[d] for d < n_dest
__global__ void k_route_base(const unsigned long long* __restrict__ cnt, int n_dest, uint32_t* __restrict__ base,
                             int64_t* __restrict__ counts_dev) { SS_PDL_ENTRY();
    if (threadIdx.x != 0) return;
    uint32_t run = 0;
    for (int d = 0; d < 16; ++d) {
        base[d] = run;
        run += (uint32_t)cnt[d];
        if (d < n_dest) counts_dev[d] = (int64_t)cnt[d];
    }
}
// counts_dev[n_dest] = first bad tuple index (or -1); the route mutates no
// engine state, so the flag is cleared for the batch that follows
__global__ void k_route_done(unsigned long long* __restrict__ bad, int n_dest, int64_t* __restrict__ counts_dev) { SS_PDL_ENTRY();
    if (threadIdx.x != 0) return;
    const unsigned long long b = *bad;
    counts_dev[n_dest] = b == (unsigned long long)kNoBad ? -1 : (int64_t)b;
    *bad = (unsigned long long)kNoBad;
}

// Stable split by owning GPU into 8-byte (group, attr) records -- the one
// message the tuple all-to-all ships; counts_dev[n_dest + 1] on the device.
extern "C" int ss_route_records(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                                void* out_records, int64_t* counts_dev) {
    NvtxRange nv_("ss_route_records");
    if (!e || n < 0 || !counts_dev || (n && !out_records)) return SS_E_CONFIG;
    if (!e->owner) return fail(e, SS_E_CONFIG, "ss_set_owner first");
    if (!is_device_ptr(counts_dev) || (n && !is_device_ptr(out_records)))
        return fail(e, SS_E_CONFIG, "ss_route_records: device outputs required");
    { int jr = join_side(e); if (jr) return jr; }
    const uint32_t* dk;
    const int32_t* dv;
    int rc;
    if ((rc = stage_input(e, groups, attrs, n, &dk, &dv))) return rc;
    if ((rc = engine_alloc_sort(e, n))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->route_cnt, 0, 16 * 8, e->st));
    if (n) ss_note_launch(), ss_launch(k_owner_hist, 2 * kNumSM, 256, 0, e->st, dk, n, (uint32_t)e->G, e->owner, e->route_cnt, e->bad);
    ss_note_launch(), ss_launch(k_route_base, 1, 32, 0, e->st, e->route_cnt, e->n_dest, e->route_base, counts_dev);
    if (n) {
        SS_CUDA(e, cudaMemsetAsync(e->tickets, 0, 8, e->st));
        ss_note_launch(), ss_launch(k_epoch_bump, 1, 1, 0, e->st, e->ep_dev);
        const int tiles = (int)((n + kSortTile - 1) / kSortTile);
        ss_note_launch(), ss_launch(k_sort_pass<4, true>, std::min(tiles, 2 * kNumSM), kSortThreads, SortSmem<4>::bytes, e->st, dk, dv, (uint32_t*)out_records, nullptr, (int)n, 0, 15u, e->route_base, e->status, e->ep_dev, 0,
            e->tickets, e->bad, 0, e->owner, nullptr, SortSeg{});
    }
    ss_note_launch(), ss_launch(k_route_done, 1, 32, 0, e->st, e->bad, e->n_dest, counts_dev);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// The owner map from a device array (the GPU-level engine's own pmap)
extern "C" int ss_set_owner_dev(ss_engine* e, const int32_t* owner_dev, int n_dest) {
    if (!e || !owner_dev || n_dest < 1 || n_dest > 16) return fail(e, SS_E_CONFIG, "n_dest must be in [1, 16]");
    if (!is_device_ptr(owner_dev)) return fail(e, SS_E_CONFIG, "ss_set_owner_dev: device map required");
    int rc;
    if (!e->owner) {
        if ((rc = dalloc(e, &e->owner, e->G)) || (rc = dalloc(e, &e->route_cnt, 16)) ||
            (rc = dalloc(e, &e->route_base, 16)))
            return rc;
    }
    SS_CUDA(e, cudaMemcpyAsync(e->owner, owner_dev, e->G * 4, cudaMemcpyDeviceToDevice, e->st));
    e->n_dest = n_dest;
    return SS_OK;
}

// The policy on device per-group counts, its moves applied to this
// engine's assignment on the device (the GPU-level balancer: partitions =
// GPUs).  Copies the moves (int4 group, src, dst, placement), their count
// and the new group -> partition map into caller device buffers.
extern "C" int ss_balance_apply_dev(ss_engine* e, const int32_t* counts_dev, const ss_balancer* cfg, void* moves_dev,
                                    int32_t* n_moves_dev, int32_t* pmap_dev) {
    if (!e || !cfg || !counts_dev || !moves_dev || !n_moves_dev || !pmap_dev) return SS_E_CONFIG;
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    if (!is_device_ptr(counts_dev) || !is_device_ptr(moves_dev) || !is_device_ptr(n_moves_dev) ||
        !is_device_ptr(pmap_dev))
        return fail(e, SS_E_CONFIG, "ss_balance_apply_dev: device buffers required");
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaMemcpyAsync(e->gcount, counts_dev, e->G * 4, cudaMemcpyDeviceToDevice, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->tpt, 0, e->P * 8, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->n_moves, 0, 4, e->st));
    ss_note_launch(), ss_launch(k_tpt_from_counts, 2 * kNumSM, 256, 0, e->st, e->gcount, e->G, e->pmap, e->tpt);
    const int cap = move_cap(e, cfg);
    if (cfg->policy != SS_POLICY_NO) {
        BalanceArgs a{};
        a.policy = cfg->policy;
        a.threshold = cfg->thread_threshold;
        a.pot = cfg->pot;
        a.cap = cap;
        a.P = e->P;
        a.order = e->order;
        a.offsets = e->offsets;
        a.gcount = e->gcount;
        a.tpt = e->tpt;
        a.moved = e->moved;
        a.moves = e->moves;
        a.front_top = e->front_top;
        a.back_first = e->back_first;
        a.mv_next = e->mv_next;
        a.new_off = e->new_off;
        a.keep_at = e->keep_at;
        a.mv_pos = e->mv_pos;
        a.n_moves = e->n_moves;
        a.scanned = e->scanned;
        a.final_tpt = e->final_tpt;
        a.bad = e->bad;
        ss_note_launch(), launch_balance(e, a, e->st);
        ss_note_launch(), ss_launch(k_apply_place, e->P, 256, 0, e->st, e->order, e->offsets, e->keep_at, e->moves,
                                                                  e->n_moves, e->mv_pos, e->moved, e->new_order);
        ss_note_launch(), ss_launch(k_apply_commit, 2 * kNumSM, 256, 0, e->st, e->order, e->offsets, e->new_order, e->new_off,
                                                                        (int)e->G, e->P, e->moves, e->n_moves, e->pmap,
                                                                        e->moved);
    }
    SS_CUDA(e, cudaMemcpyAsync(moves_dev, e->moves, (size_t)cap * sizeof(int4), cudaMemcpyDeviceToDevice, e->st));
    SS_CUDA(e, cudaMemcpyAsync(n_moves_dev, e->n_moves, 4, cudaMemcpyDeviceToDevice, e->st));
    SS_CUDA(e, cudaMemcpyAsync(pmap_dev, e->pmap, e->G * 4, cudaMemcpyDeviceToDevice, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->gcount, 0, e->G * 4, e->st));
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// Window-state migration blobs (int32 words).  Per destination d, a segment
//   [n] ++ n records (g, fill, next_pos, sum_lo, sum_hi, min, max, span) ++ values
// (span = the ring image: fill values while filling, else all W slots, so
// next_pos carries over and the migrated group is bit-identical).
constexpr int kMigMax = 256;          // exported groups per batch (>= 4 x GPUs)
constexpr int kMigRec = 8;

__global__ void k_export_plan(const int4* __restrict__ moves, const int32_t* __restrict__ n_moves, int rank, int n_dest,
                              int64_t W, const int32_t* __restrict__ fill, const int32_t* __restrict__ next_pos,
                              const long long* __restrict__ wsum, const int32_t* __restrict__ mn,
                              const int32_t* __restrict__ mx, const int64_t* __restrict__ off, int32_t* __restrict__ blob,
                              int64_t blob_cap, int64_t* __restrict__ sizes, longlong4* __restrict__ list,
                              int* __restrict__ n_list) { SS_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int nm = min(*n_moves, kMigMax);
    int64_t ng[16] = {0}, nv[16] = {0};
    for (int i = 0; i < nm; ++i) {
        const int4 m = moves[i];
        if (m.y != rank || m.z == rank || m.z < 0 || m.z >= n_dest) continue;
        const int f = fill[m.x];
        ng[m.z] += 1;
        nv[m.z] += (int64_t)f < W ? f : W;
    }
    int64_t seg[16], base = 0;
    for (int d = 0; d < n_dest; ++d) {
        seg[d] = base;
        const int64_t words = ng[d] ? 1 + kMigRec * ng[d] + nv[d] : 0;
        sizes[d] = words;
        base += words;
    }
    if (base > blob_cap) {                          // caller raises: blob too small
        for (int d = 0; d < n_dest; ++d) sizes[d] = -1;
        *n_list = 0;
        return;
    }
    int64_t rec[16], val[16];
    for (int d = 0; d < n_dest; ++d) {
        if (ng[d]) blob[seg[d]] = (int32_t)ng[d];
        rec[d] = seg[d] + 1;
        val[d] = seg[d] + 1 + kMigRec * ng[d];
    }
    int nl = 0;
    for (int i = 0; i < nm; ++i) {
        const int4 m = moves[i];
        if (m.y != rank || m.z == rank || m.z < 0 || m.z >= n_dest) continue;
        const int g = m.x, d = m.z;
        const int f = fill[g];
        const int64_t span = (int64_t)f < W ? f : W;
        const unsigned long long s = (unsigned long long)wsum[g];
        int32_t* r = blob + rec[d];
        r[0] = g; r[1] = f; r[2] = next_pos[g];
        r[3] = (int32_t)(uint32_t)s; r[4] = (int32_t)(uint32_t)(s >> 32);
        r[5] = mn[g]; r[6] = mx[g]; r[7] = (int32_t)span;
        rec[d] += kMigRec;
        if (span) list[nl++] = make_longlong4(off[g], val[d], span, 0);
        val[d] += span;
    }
    *n_list = nl;
}

__global__ void __launch_bounds__(256)
k_export_vals(const longlong4* __restrict__ list, const int* __restrict__ n_list, const int32_t* __restrict__ ring,
              int32_t* __restrict__ blob) { SS_PDL_ENTRY();
    if ((int)blockIdx.x >= *n_list) return;
    const longlong4 c = list[blockIdx.x];
    for (int64_t j = threadIdx.x; j < c.z; j += blockDim.x) blob[c.y + j] = ring[c.x + j];
}

extern "C" int ss_export_moves_dev(ss_engine* e, const void* moves_dev, const int32_t* n_moves_dev, int rank,
                                   int32_t* blob_dev, int64_t blob_cap_words, int64_t* sizes_dev) {
    if (!e || !moves_dev || !n_moves_dev || !blob_dev || !sizes_dev) return SS_E_CONFIG;
    if (e->n_dest < 1) return fail(e, SS_E_CONFIG, "ss_set_owner first");
    int rc;
    if (!e->mig_list && ((rc = dalloc(e, &e->mig_list, kMigMax)) || (rc = dalloc(e, &e->mig_n, 1)))) return rc;
    ss_note_launch(), ss_launch(k_export_plan, 1, 32, 0, e->st, (const int4*)moves_dev, n_moves_dev, rank, e->n_dest, e->W,
                                                         e->fill, e->next_pos, e->wsum, e->mn, e->mx, e->off, blob_dev,
                                                         blob_cap_words, sizes_dev, e->mig_list, e->mig_n);
    ss_note_launch(), ss_launch(k_export_vals, kMigMax, 256, 0, e->st, e->mig_list, e->mig_n, e->ring, blob_dev);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

struct MigSegs {
    int64_t off[17];
    int n;
};

// CTA (j, s): record j of the segment from source s -- ring space (a bump
// reservation when the region is too small), values, state
__global__ void __launch_bounds__(256)
k_import(const int32_t* __restrict__ blob, MigSegs segs, int64_t W, int dense, int32_t* __restrict__ fill,
         int32_t* __restrict__ next_pos, long long* __restrict__ wsum, int32_t* __restrict__ mn,
         int32_t* __restrict__ mx, int64_t* __restrict__ off, int32_t* __restrict__ cap,
         unsigned long long* __restrict__ pool_top, unsigned long long pool_cap, int* __restrict__ oom,
         uint8_t* __restrict__ sum_valid, int32_t* __restrict__ ring, int64_t G) { SS_PDL_ENTRY();
    __shared__ int64_t sh_dst;
    const int s = blockIdx.y, j = blockIdx.x;
    if (segs.off[s + 1] == segs.off[s]) return;
    const int32_t* seg = blob + segs.off[s];
    const int ng = seg[0];
    if (j >= ng) return;
    const int32_t* r = seg + 1 + kMigRec * j;
    int64_t vpos = 1 + (int64_t)kMigRec * ng;
    for (int i = 0; i < j; ++i) vpos += seg[1 + kMigRec * i + 7];
    const int g = r[0];
    const int64_t span = r[7];
    if (g < 0 || g >= G) return;
    if (threadIdx.x == 0) {
        int64_t o = off[g];
        if (!dense && cap[g] < span) {
            const int64_t ncap = min64(W, max64(span, 16));
            const unsigned long long top = atomicAdd(pool_top, (unsigned long long)ncap);
            if (top + (unsigned long long)ncap > pool_cap) {
                *oom = 1;
                o = -1;
            } else {
                o = (int64_t)top;
                off[g] = o;
                cap[g] = (int32_t)ncap;
            }
        }
        sh_dst = o;
        if (o >= 0) {
            fill[g] = r[1];
            next_pos[g] = r[2];
            wsum[g] = (long long)(((unsigned long long)(uint32_t)r[4] << 32) | (uint32_t)r[3]);
            mn[g] = r[5];
            mx[g] = r[6];
            if (sum_valid) sum_valid[g] = 0;        // ring rewritten: chunk summaries stale
        }
    }
    __syncthreads();
    const int64_t o = sh_dst;
    if (o < 0) return;
    for (int64_t i = threadIdx.x; i < span; i += blockDim.x) ring[o + i] = seg[vpos + i];
}

extern "C" int ss_import_blob_dev(ss_engine* e, const int32_t* blob_dev, const int64_t* seg_off, int n_seg,
                                  int max_groups) {
    if (!e || n_seg < 0 || n_seg > 16 || (n_seg && !seg_off)) return SS_E_CONFIG;
    if (n_seg == 0 || max_groups <= 0 || seg_off[n_seg] == 0) return SS_OK;     // nothing received
    if (!blob_dev) return fail(e, SS_E_CONFIG, "ss_import_blob_dev: null blob");
    MigSegs s{};
    for (int i = 0; i <= n_seg; ++i) s.off[i] = seg_off[i];
    s.n = n_seg;
    if (s.off[n_seg] == 0) return SS_OK;
    ss_note_launch(), ss_launch(k_import, dim3((unsigned)std::min(max_groups, kMigMax), (unsigned)n_seg), 256, 0, e->st, blob_dev, s, e->W, e->dense ? 1 : 0, e->fill, e->next_pos, e->wsum, e->mn, e->mx, e->off, e->cap,
        e->pool_top, e->pool_cap, e->oom, e->sum_valid, e->ring, e->G);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}


// The policy on given per-group counts (BatchStats.group_counts) against
// the current assignment; nothing is applied.  Used by the GPU-level
// balancer (partitions = GPUs) and by the reference-signature policies.
extern "C" int ss_balance_counts(ss_engine* e, const int32_t* counts, const ss_balancer* cfg, ss_move* moves,
                                 int64_t* n_moves, int64_t* scanned, int64_t* final_tpt) {
    if (!e || !cfg || !counts) return SS_E_CONFIG;
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaMemcpyAsync(e->gcount, counts, e->G * 4,
                               is_device_ptr(counts) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->tpt, 0, e->P * 8, e->st));
    ss_note_launch(), ss_launch(k_tpt_from_counts, 2 * kNumSM, 256, 0, e->st, e->gcount, e->G, e->pmap, e->tpt);
    int nm = 0;
    long long sc = 0;
    std::vector<long long> ft(e->P);
    if (cfg->policy == SS_POLICY_NO) {
        std::vector<unsigned long long> tp(e->P);
        SS_CUDA(e, cudaMemcpyAsync(tp.data(), e->tpt, e->P * 8, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaStreamSynchronize(e->st));
        for (int p = 0; p < e->P; ++p) ft[p] = (long long)tp[p];
    } else {
        BalanceArgs a{};
        a.policy = cfg->policy;
        a.threshold = cfg->thread_threshold;
        a.pot = cfg->pot;
        a.cap = move_cap(e, cfg);
        a.P = e->P;
        a.order = e->order;
        a.offsets = e->offsets;
        a.gcount = e->gcount;
        a.tpt = e->tpt;
        a.moved = e->moved;
        a.moves = e->moves;
        a.front_top = e->front_top;
        a.back_first = e->back_first;
        a.mv_next = e->mv_next;
        a.n_moves = e->n_moves;
        a.scanned = e->scanned;
        a.final_tpt = e->final_tpt;
        a.bad = e->bad;
        ss_note_launch(), launch_balance(e, a, e->st);
        SS_CUDA(e, cudaGetLastError());
        ss_note_launch(), ss_launch(k_clear_moved, 4, 256, 0, e->st, e->moves, e->n_moves, e->moved);
        SS_CUDA(e, cudaMemcpyAsync(&nm, e->n_moves, 4, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaMemcpyAsync(&sc, e->scanned, 8, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaMemcpyAsync(ft.data(), e->final_tpt, e->P * 8, cudaMemcpyDeviceToHost, e->st));
        SS_CUDA(e, cudaStreamSynchronize(e->st));
    }
    if (nm > 0 && moves) {
        std::vector<int4> mv(nm);
        SS_CUDA(e, cudaMemcpy(mv.data(), e->moves, nm * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nm; ++i) moves[i] = ss_move{mv[i].x, mv[i].y, mv[i].z, mv[i].w};
    }
    if (n_moves) *n_moves = nm;
    if (scanned) *scanned = sc;
    if (final_tpt)
        for (int p = 0; p < e->P; ++p) final_tpt[p] = ft[p];
    SS_CUDA(e, cudaMemsetAsync(e->n_moves, 0, 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->gcount, 0, e->G * 4, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// Window state of `groups` in ring-slot layout: meta[5*i..] = (fill,
// next_pos, window_sum, min, max); values = concatenated ring images of
// span = fill (< W, linear) or W slots.  Import writes the same layout, so
// a migrated group is bit-identical (next_pos included).
static int64_t state_span(int32_t fill, int64_t W) { return fill < W ? fill : W; }

extern "C" int ss_export_state(ss_engine* e, const int32_t* groups, int64_t n, int64_t* meta, int32_t* values,
                               int64_t cap, int64_t* n_values) {
    if (!e || n < 0) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t g = groups[i];
        if (g < 0 || g >= e->G) return fail(e, SS_E_CONFIG, "group out of range");
        int32_t f, np, lo, hi;
        long long s;
        int64_t o;
        SS_CUDA(e, cudaMemcpy(&f, e->fill + g, 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(&np, e->next_pos + g, 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(&s, e->wsum + g, 8, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(&lo, e->mn + g, 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(&hi, e->mx + g, 4, cudaMemcpyDeviceToHost));
        SS_CUDA(e, cudaMemcpy(&o, e->off + g, 8, cudaMemcpyDeviceToHost));
        if (meta) {
            meta[5 * i + 0] = f; meta[5 * i + 1] = np; meta[5 * i + 2] = s;
            meta[5 * i + 3] = lo; meta[5 * i + 4] = hi;
        }
        const int64_t span = state_span(f, e->W);
        if (values && pos + span <= cap && span)
            SS_CUDA(e, cudaMemcpy(values + pos, e->ring + o, span * 4, cudaMemcpyDeviceToHost));
        pos += span;
    }
    if (n_values) *n_values = pos;
    return SS_OK;
}

extern "C" int ss_import_state(ss_engine* e, const int32_t* groups, int64_t n, const int64_t* meta,
                               const int32_t* values) {
    if (!e || n < 0 || (n && (!meta || !groups))) return SS_E_CONFIG;
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t g = groups[i];
        if (g < 0 || g >= e->G) return fail(e, SS_E_CONFIG, "group out of range");
        const int32_t f = (int32_t)meta[5 * i + 0], np = (int32_t)meta[5 * i + 1];
        const long long s = meta[5 * i + 2];
        const int32_t lo = (int32_t)meta[5 * i + 3], hi = (int32_t)meta[5 * i + 4];
        const int64_t span = state_span(f, e->W);
        int64_t o;
        SS_CUDA(e, cudaMemcpy(&o, e->off + g, 8, cudaMemcpyDeviceToHost));
        if (!e->dense) {
            int32_t c;
            SS_CUDA(e, cudaMemcpy(&c, e->cap + g, 4, cudaMemcpyDeviceToHost));
            if (c < span) {
                unsigned long long top;
                SS_CUDA(e, cudaMemcpy(&top, e->pool_top, 8, cudaMemcpyDeviceToHost));
                const int64_t ncap = std::min<int64_t>(e->W, std::max<int64_t>(span, 16));
                if (top + ncap > e->pool_cap) return fail(e, SS_E_EXEC, "window ring pool exhausted");
                o = (int64_t)top;
                top += ncap;
                const int32_t c32 = (int32_t)ncap;
                SS_CUDA(e, cudaMemcpy(e->pool_top, &top, 8, cudaMemcpyHostToDevice));
                SS_CUDA(e, cudaMemcpy(e->off + g, &o, 8, cudaMemcpyHostToDevice));
                SS_CUDA(e, cudaMemcpy(e->cap + g, &c32, 4, cudaMemcpyHostToDevice));
            }
        }
        if (span) SS_CUDA(e, cudaMemcpy(e->ring + o, values + pos, span * 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->fill + g, &f, 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->next_pos + g, &np, 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->wsum + g, &s, 8, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->mn + g, &lo, 4, cudaMemcpyHostToDevice));
        SS_CUDA(e, cudaMemcpy(e->mx + g, &hi, 4, cudaMemcpyHostToDevice));
        if (e->sum_valid) SS_CUDA(e, cudaMemset(e->sum_valid + g, 0, 1));   // ring rewritten
        pos += span;
    }
    return SS_OK;
}

// ---- int64 keys across GPUs (keys.cuh: buckets) ------------------------------
constexpr int kMig64Max = 8192;          // keys migrated per batch and GPU (4 x GPUs buckets of ~G/2^16 keys)

static int ensure_bucket_owner(ss_engine* e) {
    if (!e->keys64) return fail(e, SS_E_CONFIG, "engine was created with key_bits = 32");
    int rc;
    if (!e->bowner) {
        if ((rc = dalloc(e, &e->bowner, kKeyBuckets)) || (rc = dalloc(e, &e->bdst, kKeyBuckets)) ||
            (rc = dalloc(e, &e->mig64, kMig64Max)) || (rc = dalloc(e, &e->mig64_copies, kMig64Max)) ||
            (rc = dalloc(e, &e->n_mig64, 1)) ||
            (rc = dalloc(e, &e->rec_vals, e->max_batch)))
            return rc;
        if (!e->route_cnt && ((rc = dalloc(e, &e->route_cnt, 16)) || (rc = dalloc(e, &e->route_base, 16)))) return rc;
        if (!e->mig_list && ((rc = dalloc(e, &e->mig_list, kMigMax)) || (rc = dalloc(e, &e->mig_n, 1)))) return rc;
    }
    return SS_OK;
}

// bucket -> GPU map (kKeyBuckets entries in [0, n_dest)), host or device
extern "C" int ss_set_bucket_owner(ss_engine* e, const int32_t* owner, int n_dest) {
    if (!e || !owner || n_dest < 1 || n_dest > 16) return fail(e, SS_E_CONFIG, "n_dest must be in [1, 16]");
    int rc;
    if ((rc = ensure_bucket_owner(e))) return rc;
    if (!is_device_ptr(owner))
        for (int b = 0; b < kKeyBuckets; ++b)
            if (owner[b] < 0 || owner[b] >= n_dest) return fail(e, SS_E_CONFIG, "owner out of range");
    SS_CUDA(e, cudaMemcpyAsync(e->bowner, owner, kKeyBuckets * 4, cudaMemcpyDefault, e->st));
    e->n_dest = n_dest;
    return SS_OK;
}

// stable split of an int64-key batch (device keys / attrs) by the owner of
// each key's bucket into 12-byte (key lo, key hi, attr) records (device);
// counts_dev[n_dest] per destination, counts_dev[n_dest] = -1 (no bad keys)
extern "C" int ss_route_records64(ss_engine* e, const int64_t* keys, const int32_t* attrs, int64_t n, void* out_records,
                                  int64_t* counts_dev) {
    NvtxRange nv_("ss_route_records64");
    if (!e || n < 0 || !counts_dev || (n && (!out_records || !keys || !attrs))) return SS_E_CONFIG;
    if (!e->bowner) return fail(e, SS_E_CONFIG, "ss_set_bucket_owner first");
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    if (n && (!is_device_ptr(keys) || !is_device_ptr(attrs) || !is_device_ptr(out_records)) || !is_device_ptr(counts_dev))
        return fail(e, SS_E_CONFIG, "ss_route_records64: device buffers required");
    { int jr = join_side(e); if (jr) return jr; }
    int rc;
    if ((rc = engine_alloc_sort(e, n))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->route_cnt, 0, 16 * 8, e->st));
    if (n) {
        ss_note_launch(), ss_launch(k_key_route_prep, 4 * kNumSM, 256, 0, e->st, (const long long*)keys, n, e->kbuf,
                                    e->vbuf[1]);
        ss_note_launch(), ss_launch(k_owner_hist, 2 * kNumSM, 256, 0, e->st, (const uint32_t*)e->kbuf, n,
                                    (uint32_t)kKeyBuckets, (const int32_t*)e->bowner, e->route_cnt, e->bad);
    }
    ss_note_launch(), ss_launch(k_route_base, 1, 32, 0, e->st, (const unsigned long long*)e->route_cnt, e->n_dest,
                                e->route_base, counts_dev);
    if (n) {
        SS_CUDA(e, cudaMemsetAsync(e->tickets, 0, 8, e->st));
        ss_note_launch(), ss_launch(k_epoch_bump, 1, 1, 0, e->st, e->ep_dev);
        const int tiles = (int)((n + kSortTile - 1) / kSortTile);
        ss_note_launch(), ss_launch(k_sort_pass<4, true>, std::min(tiles, 2 * kNumSM), kSortThreads, SortSmem<4>::bytes,
                                    e->st, (const uint32_t*)e->kbuf, (const int32_t*)e->vbuf[1], e->kbuf2, e->vbuf[0],
                                    (int)n, 0, 15u, (const uint32_t*)e->route_base, e->status,
                                    (const uint32_t*)e->ep_dev, 0u, e->tickets, (const unsigned long long*)e->bad, 0,
                                    (const int32_t*)e->bowner, (const int32_t*)nullptr, SortSeg{});
        ss_note_launch(), ss_launch(k_key_route_gather, 4 * kNumSM, 256, 0, e->st, (const long long*)keys, attrs,
                                    (const int32_t*)e->vbuf[0], n, (int32_t*)out_records);
    }
    ss_note_launch(), ss_launch(k_route_done, 1, 32, 0, e->st, e->bad, e->n_dest, counts_dev);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

extern "C" int ss_step_keys64(ss_engine* e, const int64_t* keys, const int32_t* attrs, int64_t n,
                              const ss_balancer* cfg, ss_step_report* rep);

// one batch of received 12-byte records (device) through the int64-key step
extern "C" int ss_step_records64(ss_engine* e, const void* records, int64_t n, const ss_balancer* cfg,
                                 ss_step_report* rep) {
    if (!e || n < 0 || (n && !records)) return SS_E_CONFIG;
    int rc;
    if ((rc = ensure_bucket_owner(e))) return rc;
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    if (n && !is_device_ptr(records)) return fail(e, SS_E_CONFIG, "ss_step_records64: device records required");
    if (n) ss_note_launch(), ss_launch(k_key_rec_split, 4 * kNumSM, 256, 0, e->st, (const int32_t*)records, n,
                                       e->stage_keys64, e->rec_vals);
    e->inputs_on_stream = true;           // the split keys are engine-stream work
    rc = ss_step_keys64(e, (const int64_t*)e->stage_keys64, e->rec_vals, n, cfg, rep);
    e->inputs_on_stream = false;
    return rc;
}

// per-bucket counts of the last batch (device, kKeyBuckets entries)
extern "C" int ss_bucket_counts_dev(ss_engine* e, int32_t* out) {
    if (!e || !out) return SS_E_CONFIG;
    int rc;
    if ((rc = ensure_bucket_owner(e))) return rc;
    SS_CUDA(e, cudaMemsetAsync(out, 0, kKeyBuckets * 4, e->st));
    ss_note_launch(), ss_launch(k_key_bucket_counts, group_grid(e->G), 256, 0, e->st, e->kt,
                                (const int32_t*)e->gcount, out);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// segments per destination: [n] ++ n x (key lo, key hi, fill, next_pos,
// sum lo, sum hi, min, max, span) ++ ring images
constexpr int kMigRec64 = 9;

__global__ void k_export_plan64(const int2* __restrict__ list, const int* __restrict__ n_list, int cap, int n_dest,
                                int64_t W, const unsigned long long* __restrict__ slot_keys,
                                const int32_t* __restrict__ fill, const int32_t* __restrict__ next_pos,
                                const long long* __restrict__ wsum, const int32_t* __restrict__ mn,
                                const int32_t* __restrict__ mx, const int64_t* __restrict__ off,
                                int32_t* __restrict__ blob, int64_t blob_cap, int64_t* __restrict__ sizes,
                                longlong4* __restrict__ copies, int* __restrict__ n_copies) { SS_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int nl = min(*n_list, cap);
    int64_t ng[16] = {0}, nv[16] = {0};
    for (int i = 0; i < nl; ++i) {
        const int2 m = list[i];
        const int f = fill[m.x];
        ng[m.y] += 1;
        nv[m.y] += (int64_t)f < W ? f : W;
    }
    int64_t seg[16], base = 0;
    for (int d = 0; d < n_dest; ++d) {
        seg[d] = base;
        const int64_t words = ng[d] ? 1 + kMigRec64 * ng[d] + nv[d] : 0;
        sizes[d] = words;
        base += words;
    }
    if (base > blob_cap || *n_list > cap) {
        for (int d = 0; d < n_dest; ++d) sizes[d] = -1;
        *n_copies = 0;
        return;
    }
    int64_t rec[16], val[16];
    for (int d = 0; d < n_dest; ++d) {
        if (ng[d]) blob[seg[d]] = (int32_t)ng[d];
        rec[d] = seg[d] + 1;
        val[d] = seg[d] + 1 + kMigRec64 * ng[d];
    }
    int nc = 0;
    for (int i = 0; i < nl; ++i) {
        const int g = list[i].x, d = list[i].y;
        const int f = fill[g];
        const int64_t span = (int64_t)f < W ? f : W;
        const unsigned long long k = slot_keys[g];
        const unsigned long long sm = (unsigned long long)wsum[g];
        int32_t* r = blob + rec[d];
        r[0] = (int32_t)(uint32_t)k; r[1] = (int32_t)(uint32_t)(k >> 32);
        r[2] = f; r[3] = next_pos[g];
        r[4] = (int32_t)(uint32_t)sm; r[5] = (int32_t)(uint32_t)(sm >> 32);
        r[6] = mn[g]; r[7] = mx[g]; r[8] = (int32_t)span;
        rec[d] += kMigRec64;
        if (span) copies[nc++] = make_longlong4(off[g], val[d], span, 0);
        val[d] += span;
    }
    *n_copies = nc;
}

// window state of the keys in the buckets this GPU gives away
extern "C" int ss_export_moves64_dev(ss_engine* e, const void* moves_dev, const int32_t* n_moves_dev, int rank,
                                     int32_t* blob_dev, int64_t blob_cap_words, int64_t* sizes_dev) {
    if (!e || !moves_dev || !n_moves_dev || !blob_dev || !sizes_dev) return SS_E_CONFIG;
    int rc;
    if ((rc = ensure_bucket_owner(e))) return rc;
    SS_CUDA(e, cudaMemsetAsync(e->bdst, 0xff, kKeyBuckets * 4, e->st));
    SS_CUDA(e, cudaMemsetAsync(e->n_mig64, 0, 4, e->st));
    ss_note_launch(), ss_launch(k_key_mig_mark, 4, 256, 0, e->st, (const int4*)moves_dev, n_moves_dev, rank, e->n_dest,
                                e->bdst);
    ss_note_launch(), ss_launch(k_key_mig_collect, group_grid(e->G), 256, 0, e->st, e->kt, (const int32_t*)e->bdst,
                                e->mig64, e->n_mig64, kMig64Max);
    ss_note_launch(), ss_launch(k_export_plan64, 1, 32, 0, e->st, (const int2*)e->mig64, (const int*)e->n_mig64, kMig64Max,
                                e->n_dest, e->W, (const unsigned long long*)e->kt.slot_keys, (const int32_t*)e->fill,
                                (const int32_t*)e->next_pos, (const long long*)e->wsum, (const int32_t*)e->mn,
                                (const int32_t*)e->mx, (const int64_t*)e->off, blob_dev, blob_cap_words, sizes_dev,
                                e->mig64_copies, e->n_mig64);
    ss_note_launch(), ss_launch(k_export_vals, kMig64Max, 256, 0, e->st, (const longlong4*)e->mig64_copies,
                                (const int*)e->n_mig64, (const int32_t*)e->ring, blob_dev);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// CTA s: the records of segment s, one warp per record (value offsets from
// a serial prefix over the segment's spans by the warp itself)
__global__ void __launch_bounds__(256)
k_import64(const int32_t* __restrict__ blob, MigSegs segs, int64_t W, int dense, KeyTable t,
           int32_t* __restrict__ fill, int32_t* __restrict__ next_pos, long long* __restrict__ wsum,
           int32_t* __restrict__ mn, int32_t* __restrict__ mx, int64_t* __restrict__ off, int32_t* __restrict__ cap,
           unsigned long long* __restrict__ pool_top, unsigned long long pool_cap, int* __restrict__ oom,
           uint8_t* __restrict__ sum_valid, int32_t* __restrict__ ring) { SS_PDL_ENTRY();
    const int s = blockIdx.x;
    if (segs.off[s + 1] == segs.off[s]) return;
    const int32_t* seg = blob + segs.off[s];
    const int ng = seg[0];
    const unsigned lane = lane_id();
    const int nw = blockDim.x >> 5;
    for (int j = (int)warp_id(); j < ng; j += nw) {
        const int32_t* r = seg + 1 + kMigRec64 * j;
        int64_t part = 0;                       // spans of the records before j
        for (int i = (int)lane; i < j; i += 32) part += seg[1 + kMigRec64 * i + 8];
        const int64_t vpos = 1 + (int64_t)kMigRec64 * ng + warp_sum(part);
        const unsigned long long k = ((unsigned long long)(uint32_t)r[1] << 32) | (uint32_t)r[0];
        const int64_t span = r[8];
        int64_t o = -1;
        if (lane == 0) {
            const int g = key_claim_slot(t, k);
            if (g >= 0) {
                o = off[g];
                if (!dense && cap[g] < span) {
                    const int64_t ncap = min64(W, max64(span, 16));
                    const unsigned long long top = atomicAdd(pool_top, (unsigned long long)ncap);
                    if (top + (unsigned long long)ncap > pool_cap) {
                        *oom = 1;
                        o = -1;
                    } else {
                        o = (int64_t)top;
                        off[g] = o;
                        cap[g] = (int32_t)ncap;
                    }
                }
                if (o >= 0) {
                    fill[g] = r[2];
                    next_pos[g] = r[3];
                    wsum[g] = (long long)(((unsigned long long)(uint32_t)r[5] << 32) | (uint32_t)r[4]);
                    mn[g] = r[6];
                    mx[g] = r[7];
                    if (sum_valid) sum_valid[g] = 0;
                }
            }
        }
        o = __shfl_sync(SS_FULL, o, 0);
        if (o < 0) continue;
        for (int64_t i = lane; i < span; i += 32) ring[o + i] = seg[vpos + i];
    }
}

extern "C" int ss_import_blob64_dev(ss_engine* e, const int32_t* blob_dev, const int64_t* seg_off, int n_seg) {
    if (!e || n_seg < 0 || n_seg > 16 || (n_seg && !seg_off)) return SS_E_CONFIG;
    int rc;
    if ((rc = ensure_bucket_owner(e))) return rc;
    if (n_seg == 0 || seg_off[n_seg] == 0) return SS_OK;
    if (!blob_dev) return fail(e, SS_E_CONFIG, "ss_import_blob64_dev: null blob");
    MigSegs sg{};
    for (int i = 0; i <= n_seg; ++i) sg.off[i] = seg_off[i];
    sg.n = n_seg;
    ss_note_launch(), ss_launch(k_import64, (unsigned)n_seg, 256, 0, e->st, blob_dev, sg, e->W, e->dense ? 1 : 0, e->kt,
                                e->fill, e->next_pos, e->wsum, e->mn, e->mx, e->off, e->cap, e->pool_top, e->pool_cap,
                                e->oom, e->sum_valid, e->ring);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// --------------------------------------------------------------------------
// int64 keys
// --------------------------------------------------------------------------
// keys -> slots (and, with `count`, the batch's group histogram: the
// fused step then skips its count kernel)
static int map_keys(ss_engine* e, const int64_t* keys, int64_t n, uint32_t* dout, bool count, cudaStream_t st,
                    int32_t* gcnt, unsigned long long* bad) {
    const long long* dk;
    if (is_device_ptr(keys)) dk = (const long long*)keys;
    else {
        if (n) SS_CUDA(e, cudaMemcpyAsync(e->stage_keys64, keys, n * 8, cudaMemcpyHostToDevice, st));
        dk = e->stage_keys64;
    }
    if (n == 0) return SS_OK;
    KeyTable& t = e->kt;
    NvtxRange nv_("ss key probe + count");
    SS_CUDA(e, cudaMemcpyAsync(t.prev_slots, t.n_slots, 4, cudaMemcpyDeviceToDevice, st));
    const int nblk = (int)((n + kMarkBlk - 1) / kMarkBlk);
    const int64_t range = kCountChunk;                   // divides the count chunk S
    const unsigned grid = (unsigned)((n + range - 1) / range);
    SS_CUDA(e, cudaMemsetAsync(t.n_pend, 0, 4, st));
    if (count)
        ss_note_launch(), ss_launch(k_key_count<true>, grid, 512, kHotCache * 4, st, dk, n, t, dout, e->S, range, gcnt,
                                                                              e->hot_g, kHotCache, e->key_agg);
    else
        ss_note_launch(), ss_launch(k_key_count<false>, grid, 512, 0, st, dk, n, t, dout, e->S, range, nullptr, nullptr, 0, 0);
    ss_note_launch(), ss_launch(k_key_rank_small, 1, 1024, 0, st, t);
    ss_note_launch(), ss_launch(k_key_mark, 2 * kNumSM, 256, 0, st, t);
    ss_note_launch(), ss_launch(k_key_mark_count, std::min(nblk, 2 * kNumSM), 1024, 0, st, t, n, e->kbsum);
    ss_note_launch(), ss_launch(k_key_mark_scan, 1, 1024, 0, st, t, e->kbsum, nblk);
    ss_note_launch(), ss_launch(k_key_mark_assign, std::min(nblk, 2 * kNumSM), 1024, 0, st, t, n, e->kbsum);
    ss_note_launch(), ss_launch(k_key_mark_done, 1, 1, 0, st, t);
    ss_note_launch(), ss_launch(k_key_map, 4 * kNumSM, 256, 0, st, dk, t, dout, e->S, count ? gcnt : nullptr, bad);
    SS_CUDA(e, cudaGetLastError());
    return SS_OK;
}

// key -> dense slot of a batch (slots assigned in first-appearance order)
extern "C" int ss_map_keys(ss_engine* e, const int64_t* keys, int64_t n, uint32_t* out_slots) {
    if (!e || n < 0) return SS_E_CONFIG;
    if (!e->keys64) return fail(e, SS_E_CONFIG, "engine was created with key_bits = 32");
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    { int jr = join_side(e); if (jr) return jr; }
    const bool dev = is_device_ptr(out_slots);
    int rc;
    if ((rc = map_keys(e, keys, n, dev ? out_slots : e->stage_keys, false, e->st, e->gcnt, e->bad))) return rc;
    if (!dev && n) SS_CUDA(e, cudaMemcpyAsync(out_slots, e->stage_keys, n * 4, cudaMemcpyDeviceToHost, e->st));
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    return SS_OK;
}

// the fused step on int64 keys: map to slots, then ss_step on the slots
extern "C" int ss_step_keys64(ss_engine* e, const int64_t* keys, const int32_t* attrs, int64_t n,
                              const ss_balancer* cfg, ss_step_report* rep) {
    NvtxRange nv_("ss_step_keys64");
    if (!e || n < 0) return SS_E_CONFIG;
    if (!e->keys64) return fail(e, SS_E_CONFIG, "engine was created with key_bits = 32");
    if (n > e->max_batch) return fail(e, SS_E_CONFIG, "batch larger than max_batch");
    int rc;
    if ((rc = check_balancer(e, cfg))) return rc;
    const int64_t* dk = keys;
    const int32_t* dv = attrs;
    if (!is_device_ptr(keys) || (attrs && !is_device_ptr(attrs))) {
        if ((rc = begin_stage(e, true))) return rc;
        const int b = e->cur_stage;
        const long long* k64 = nullptr;
        if ((rc = stage_h2d(e, e->sk64[b], (const long long*)keys, n, &k64)) ||
            (rc = stage_h2d(e, e->svals[b], attrs, n, &dv)) || (rc = end_stage(e)))
            return rc;
        dk = (const int64_t*)k64;
    }
    // large G: the key probe also counts the batch (one pass over the keys)
    const bool count = e->G > 16384 && !e->stream_scope;
    if (!e->kst) {
        if ((rc = map_keys(e, dk, n, e->stage_keys, count, e->st, e->gcnt, e->bad))) return rc;
        e->pre_counted = count;
        rc = ss_step(e, e->stage_keys, dv, n, cfg, rep);
        e->pre_counted = false;
        return rc;
    }
    // Pipelined: the probe + count of this batch runs on the key stream,
    // overlapping the previous batch's placement and window update, into
    // its own slot buffer and count rows (alternating).  It waits for the
    // previous batch's hot-group cache (k_hot_select) and for the batch
    // that last used these count rows (finalize clears them); the engine
    // stream waits for it.  A bad tuple is flagged on the key stream's own
    // flag and merged into the batch's flag on the engine stream.
    const int b = e->kpar;
    e->kpar ^= 1;
    if (e->cur_stage >= 0) {
        SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_staged[e->cur_stage], 0));
    } else if (!e->key_pipe_dev || e->inputs_on_stream) {
        // device keys may be produced by work already on the engine stream
        // (e.g. the multi-GPU record split): wait for it -- no overlap
        SS_CUDA(e, cudaEventRecord(e->ev_in, e->st));
        SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_in, 0));
    }
    if (e->hot_rec) SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_hot, 0));
    if (e->fin_rec[b]) SS_CUDA(e, cudaStreamWaitEvent(e->kst, e->ev_fin[b], 0));
    if ((rc = map_keys(e, dk, n, e->skeys_buf[b], count, e->kst, e->gcnt_buf[b], e->key_bad))) return rc;
    SS_CUDA(e, cudaEventRecord(e->ev_keys[b], e->kst));
    SS_CUDA(e, cudaStreamWaitEvent(e->st, e->ev_keys[b], 0));
    ss_note_launch(), ss_launch(k_merge_bad, 1, 32, 0, e->st, e->bad, e->key_bad);
    int32_t* const gcnt0 = e->gcnt;
    e->gcnt = e->gcnt_buf[b];
    e->pre_counted = count;
    rc = ss_step(e, e->skeys_buf[b], dv, n, cfg, rep);
    e->pre_counted = false;
    e->gcnt = gcnt0;
    if (rc == SS_OK) {
        SS_CUDA(e, cudaEventRecord(e->ev_fin[b], e->st));
        e->fin_rec[b] = true;
    }
    return rc;
}

extern "C" int ss_set_host_emit(ss_engine* e, int enable) {
    if (!e) return SS_E_CONFIG;
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    if (enable && !e->h_emit[0].g) {
        const uint32_t m = e->cfg.agg_mask;
        for (int b = 0; b < 2; ++b) {
            HostRows& h = e->h_emit[b];
            HostRows& d = e->d_emit[b];
            auto mapped = [&](auto** hp, auto** dp, size_t bytes) -> cudaError_t {
                cudaError_t st = cudaHostAlloc((void**)hp, bytes, cudaHostAllocMapped);
                if (st == cudaSuccess) st = cudaHostGetDevicePointer((void**)dp, (void*)*hp, 0);
                return st;
            };
            SS_CUDA(e, mapped(&h.g, &d.g, e->G * 4));
            SS_CUDA(e, mapped(&h.hdr, &d.hdr, 64));
            if (m & SS_AGG_COUNT) SS_CUDA(e, mapped(&h.cnt, &d.cnt, e->G * 4));
            if (m & SS_AGG_SUM) SS_CUDA(e, mapped(&h.sum, &d.sum, e->G * 8));
            if (m & SS_AGG_AVG) SS_CUDA(e, mapped(&h.avg, &d.avg, e->G * 8));
            if (e->minmax && (m & SS_AGG_MIN)) SS_CUDA(e, mapped(&h.mn, &d.mn, e->G * 4));
            if (e->minmax && (m & SS_AGG_MAX)) SS_CUDA(e, mapped(&h.mx, &d.mx, e->G * 4));
        }
    }
    e->host_emit = enable != 0;
    e->emit_seq = e->pull_seq = 0;
    return SS_OK;
}

extern "C" int ss_results_pull(ss_engine* e, int64_t cap, int32_t* groups, int64_t* count, int64_t* sum,
                               double* avg, int32_t* mn, int32_t* mx, int64_t* n) {
    if (!e) return SS_E_CONFIG;
    if (!e->host_emit) return fail(e, SS_E_CONFIG, "host emission is off (ss_set_host_emit)");
    if (e->pull_seq >= e->emit_seq) return fail(e, SS_E_CONFIG, "no emitted batch left to pull");
    if (e->emit_seq - e->pull_seq > 2)
        return fail(e, SS_E_EXEC, "emitted rows overwritten: pull at least every other batch");
    const int b = (int)(e->pull_seq & 1);
    SS_CUDA(e, cudaEventSynchronize(e->ev_emit[b]));
    const HostRows& h = e->h_emit[b];
    const volatile unsigned long long* hdr = h.hdr;
    if (hdr[1] != (unsigned long long)kNoBad) {
        // a rejected batch (engine.py:281-282: nothing of it was applied);
        // the batches issued after it were no-ops as well and are dropped
        const unsigned long long idx = hdr[1], g = hdr[2];
        e->pull_seq = e->emit_seq;
        int rc = recover_bad(e);
        if (rc) return rc;
        return fail(e, SS_E_DATA, "tuple " + std::to_string(idx) + " has group " + std::to_string(g) +
                                      ", outside [0, " + std::to_string(e->G) + ")");
    }
    const unsigned nr = (unsigned)hdr[0];
    if (n) *n = nr;
    const int64_t m = std::min<int64_t>(cap, nr);
    // rows [i0, i1) out of the kernel-written pinned buffers; large pulls
    // (C4: ~1M rows per batch) are split over host threads, so the copy out
    // of the pinned buffers does not serialise the next batch's issue
    auto rows = [&](int64_t i0, int64_t i1) {
        const int64_t k = i1 - i0;
        if (groups) memcpy(groups + i0, h.g + i0, k * 4);
        if (count) {
            if (h.cnt) for (int64_t i = i0; i < i1; ++i) count[i] = h.cnt[i];
            else memset(count + i0, 0, k * 8);
        }
        if (sum) {
            if (h.sum) memcpy(sum + i0, h.sum + i0, k * 8);
            else memset(sum + i0, 0, k * 8);
        }
        if (avg) {
            if (h.avg) memcpy(avg + i0, h.avg + i0, k * 8);
            else for (int64_t i = i0; i < i1; ++i) avg[i] = 0.0;
        }
        if (mn) {
            if (h.mn) memcpy(mn + i0, h.mn + i0, k * 4);
            else memset(mn + i0, 0, k * 4);
        }
        if (mx) {
            if (h.mx) memcpy(mx + i0, h.mx + i0, k * 4);
            else memset(mx + i0, 0, k * 4);
        }
    };
    if (m >= (1 << 16)) {
        const int nt = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        const int64_t per = (m + nt - 1) / nt;
        for (int t = 1; t < nt; ++t) {
            const int64_t i0 = std::min<int64_t>(m, t * per), i1 = std::min<int64_t>(m, i0 + per);
            if (i0 < i1) th.emplace_back(rows, i0, i1);
        }
        rows(0, std::min<int64_t>(m, per));
        for (auto& x : th) x.join();
    } else if (m > 0) {
        rows(0, m);
    }
    ++e->pull_seq;
    return SS_OK;
}

extern "C" int ss_slot_keys(ss_engine* e, int64_t* keys, int64_t* n_slots) {
    if (!e) return SS_E_CONFIG;
    if (!e->keys64) return fail(e, SS_E_CONFIG, "engine was created with key_bits = 32");
    { int jr = join_side(e); if (jr) return jr; }
    SS_CUDA(e, cudaStreamSynchronize(e->st));
    int ns = 0;
    SS_CUDA(e, cudaMemcpy(&ns, e->kt.n_slots, 4, cudaMemcpyDeviceToHost));
    if (n_slots) *n_slots = ns;
    if (keys && ns) SS_CUDA(e, cudaMemcpy(keys, e->kt.slot_keys, (size_t)ns * 8, cudaMemcpyDeviceToHost));
    return SS_OK;
}
