// streamwin.cuh -- stream-scope window (the D1 alternative
// of SURVEY 7.3): GROUP BY over the last W tuples of the whole stream
// (`[ROWS W]`), instead of each group's last W values (the reference,
// engine.py:51-70).  State: a ring of the last W (group, value) tuples of the
// stream plus per-group COUNT / SUM (and MIN / MAX recomputed over the window
// for the groups a batch touched).  Per batch of n tuples, the last
// m = min(n, W) enter the window and the e = max(0, fill + m - W) oldest ring
// tuples leave it -- exactly the ring slots the new tuples overwrite.
#pragma once

#include "common.cuh"

namespace ss {

struct StreamWinArgs {
    const uint32_t* keys;      // the batch
    const int32_t* vals;
    int64_t n;                 // batch size
    int64_t m;                 // tuples entering the window (the batch's last m)
    uint32_t* ring_k;          // [W] window ring
    int32_t* ring_v;
    int64_t W;
    long long* cur;            // device ring cursors: [0] next slot to write (the
                               // oldest slot when full), [1] window tuples.  Only
                               // k_sw_advance moves them, after a valid batch, so
                               // a rejected batch leaves the window untouched
    uint32_t G;
    int32_t* count;            // per-group COUNT (the engine's fill array)
    long long* sum;            // per-group SUM (the engine's window_sum array)
    int32_t* mn;
    int32_t* mx;
    uint8_t* touched;
    unsigned long long* bad;
};

// the batch's view of the ring, from the device cursors
struct SwView {
    int64_t head, evict_from, n_evict, fill_after;
};
__device__ __forceinline__ SwView sw_view(const StreamWinArgs& a) {
    const int64_t head = a.cur[0], fill = a.cur[1];
    SwView v;
    v.head = head;
    v.n_evict = max64(0, fill + a.m - a.W);
    v.evict_from = (head - fill + a.W) % a.W;      // the oldest tuple
    v.fill_after = min64(a.W, fill + a.m);
    return v;
}

// tuples leaving the window: before the new tuples overwrite their slots
__global__ void __launch_bounds__(256)
k_sw_evict(StreamWinArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const SwView w = sw_view(a);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < w.n_evict; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = (w.evict_from + j) % a.W;
        const uint32_t g = a.ring_k[slot];
        atomicSub(&a.count[g], 1);
        atomicAdd((unsigned long long*)&a.sum[g], (unsigned long long)(-(long long)a.ring_v[slot]));
        a.touched[g] = 1;
    }
}

// validation of the whole batch (first bad tuple wins) -- before any state change
__global__ void __launch_bounds__(256)
k_sw_check(StreamWinArgs a) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
        if (a.keys[i] >= a.G) atomicMin(a.bad, (unsigned long long)i);
}

// tuples entering the window
__global__ void __launch_bounds__(256)
k_sw_add(StreamWinArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const SwView w = sw_view(a);
    const int64_t lo = a.n - a.m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.m; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = a.keys[lo + k];
        const int32_t v = a.vals[lo + k];
        atomicAdd(&a.count[g], 1);
        atomicAdd((unsigned long long*)&a.sum[g], (unsigned long long)(long long)v);
        a.touched[g] = 1;
        const int64_t slot = (w.head + k) % a.W;
        a.ring_k[slot] = g;
        a.ring_v[slot] = v;
    }
}

// MIN / MAX of touched groups: reset, then one pass over the window
__global__ void __launch_bounds__(256)
k_sw_mm_reset(StreamWinArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < a.G; g += gridDim.x * blockDim.x)
        if (a.touched[g]) {
            a.mn[g] = 0x7fffffff;
            a.mx[g] = (int32_t)0x80000000;
        }
}

__global__ void __launch_bounds__(256)
k_sw_mm_scan(StreamWinArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const SwView w = sw_view(a);
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < w.fill_after; s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = a.ring_k[s];
        if (a.touched[g]) {
            atomicMin(&a.mn[g], a.ring_v[s]);
            atomicMax(&a.mx[g], a.ring_v[s]);
        }
    }
}

// the batch is in: move the ring cursors (a rejected batch changes nothing)
__global__ void k_sw_advance(StreamWinArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const SwView w = sw_view(a);
    a.cur[0] = (w.head + a.m) % a.W;
    a.cur[1] = w.fill_after;
}

// one result row per touched group; clears the touched flags
struct StreamEmitArgs {
    uint32_t G;
    int32_t* count;
    long long* sum;
    int32_t* mn;
    int32_t* mx;
    int minmax;
    uint8_t* touched;
    unsigned* n_res;
    int32_t* r_g;
    int32_t* r_cnt;
    long long* r_sum;
    double* r_avg;
    int32_t* r_mn;
    int32_t* r_mx;
    unsigned long long* touched_total;
    const unsigned long long* bad;
};

__global__ void __launch_bounds__(256)
k_sw_emit(StreamEmitArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const unsigned lane = lane_id();
    for (uint32_t g0 = blockIdx.x * blockDim.x; g0 < a.G; g0 += gridDim.x * blockDim.x) {
        const uint32_t g = g0 + threadIdx.x;
        const bool t = g < a.G && a.touched[g];
        const unsigned bal = __ballot_sync(SS_FULL, t);
        unsigned base = 0;
        if (lane == 0 && bal) {
            base = atomicAdd(a.n_res, (unsigned)__popc(bal));
            atomicAdd(a.touched_total, (unsigned long long)__popc(bal));
        }
        base = __shfl_sync(SS_FULL, base, 0);
        if (!t) continue;
        const unsigned slot = base + __popc(bal & lanemask_lt());
        const int c = a.count[g];
        const long long s = a.sum[g];
        a.r_g[slot] = (int32_t)g;
        a.r_cnt[slot] = c;
        a.r_sum[slot] = s;
        a.r_avg[slot] = c ? __ll2double_rn(s) / (double)c : 0.0;
        if (a.minmax) {
            if (c == 0) {
                a.mn[g] = 0;
                a.mx[g] = 0;
            }
            a.r_mn[slot] = a.mn[g];
            a.r_mx[slot] = a.mx[g];
        }
        a.touched[g] = 0;
    }
}

}  // namespace ss
