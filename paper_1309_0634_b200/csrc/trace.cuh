// trace.cuh -- per-tuple trace emission on the device.
//
// Reference: AggregateTrace / TraceBuffer (engine.py:125-164): one
// (group, window sum after the tuple) record per ingested tuple; traces are
// compared through grouped_projection (engine.py:138-145), i.e. per group in
// arrival order.  serial_reference (engine.py:432-445) is the oracle.
//
// In trace mode the step keeps every tuple (no dead-tuple dropping) and the
// last placement pass also writes the group of every placed tuple, so the
// placed batch is the batch's grouped projection.  For the tuple at run
// index j of group g (prior fill f0, next_pos p0, sum S0) the timeline is
// old window ++ run; the tuple adds a_j and evicts T[f0 + j - W] when that
// index is >= 0 (an old ring value if < f0, else run value a_{j-W}).  The
// trace sum is S0 + the inclusive segmented prefix of (a - evicted) over
// the run -- computed before the window update rewrites the ring.
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kTraceTile = 1024;    // one element per thread

struct SegVal {
    long long v;
    int head;                        // a segment starts at or before this element
};

__device__ __forceinline__ SegVal seg_op(SegVal a, SegVal b) {
    return SegVal{b.head ? b.v : a.v + b.v, a.head | b.head};
}

// inclusive block segmented scan (blockDim.x == kTraceTile); `sh` >= 33 entries
__device__ __forceinline__ SegVal block_seg_scan(SegVal x, SegVal* sh, SegVal* total) {
    const unsigned lane = lane_id(), w = warp_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegVal y;
        y.v = __shfl_up_sync(SS_FULL, x.v, o);
        y.head = __shfl_up_sync(SS_FULL, x.head, o);
        if ((int)lane >= o) x = seg_op(y, x);
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        SegVal s = (lane < (blockDim.x >> 5)) ? sh[lane] : SegVal{0, 0};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegVal y;
            y.v = __shfl_up_sync(SS_FULL, s.v, o);
            y.head = __shfl_up_sync(SS_FULL, s.head, o);
            if ((int)lane >= o) s = seg_op(y, s);
        }
        sh[lane] = s;                     // inclusive over warps
    }
    __syncthreads();
    if (w > 0) x = seg_op(sh[w - 1], x);
    *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return x;
}

struct TraceArgs {
    const uint32_t* keys;      // group of every placed tuple (grouped, arrival-stable)
    const int32_t* vals;       // placed values
    const int32_t* n_dev;      // placed tuples
    const int32_t* gstart;     // run start of every group
    const int32_t* fill;       // batch-start window state
    const int32_t* next_pos;
    const long long* wsum;
    const int64_t* off;
    const int32_t* ring;
    int64_t W;
    long long* out;            // trace sums (in), per placed tuple
    SegVal* tile;              // per-tile (aggregate, has head), then carry-in
    const unsigned long long* bad;
};

// phase 1: per tuple delta (heads carry the group's prior sum), tile-local
// segmented scan, tile aggregate
__global__ void __launch_bounds__(kTraceTile)
k_trace_local(TraceArgs a) { SS_PDL_ENTRY();
    __shared__ SegVal sh[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int n = *a.n_dev;
    const int64_t i = (int64_t)blockIdx.x * kTraceTile + threadIdx.x;
    if ((int64_t)blockIdx.x * kTraceTile >= n) return;
    SegVal x{0, 0};
    if (i < n) {
        const uint32_t g = a.keys[i];
        const int s = a.gstart[g];
        const int64_t j = i - s;
        const int64_t f0 = a.fill[g];
        const int64_t t = f0 + j - a.W;        // timeline index evicted by this tuple
        long long ev = 0;
        if (t >= 0) ev = (t < f0) ? a.ring[a.off[g] + (a.next_pos[g] + t) % a.W] : a.vals[s + (t - f0)];
        x.v = (long long)a.vals[i] - ev;
        x.head = (j == 0);
        if (x.head) x.v += a.wsum[g];
    }
    SegVal tot;
    x = block_seg_scan(x, sh, &tot);
    if (i < n) a.out[i] = x.v;
    if (threadIdx.x == 0) a.tile[blockIdx.x] = tot;
}

// phase 2: exclusive segmented scan over the tile aggregates (one CTA,
// rounds of 1024 tiles): tile[t] becomes the carry-in of tile t
__global__ void __launch_bounds__(1024)
k_trace_tiles(TraceArgs a) { SS_PDL_ENTRY();
    __shared__ SegVal sh[33];
    __shared__ SegVal sinc[1024];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int n = *a.n_dev;
    const int nt = (n + kTraceTile - 1) / kTraceTile;
    SegVal carry{0, 0};                          // inclusive over earlier rounds (all threads)
    for (int t0 = 0; t0 < nt; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const SegVal x = (t < nt) ? a.tile[t] : SegVal{0, 0};
        SegVal tot;
        const SegVal inc = block_seg_scan(x, sh, &tot);
        sinc[threadIdx.x] = inc;
        __syncthreads();
        const SegVal before = threadIdx.x ? sinc[threadIdx.x - 1] : SegVal{0, 0};
        if (t < nt) a.tile[t] = seg_op(carry, before);
        carry = seg_op(carry, tot);
        __syncthreads();
    }
}

// phase 3: add each tile's carry-in to its elements before the tile's first head
__global__ void __launch_bounds__(kTraceTile)
k_trace_apply(TraceArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int n = *a.n_dev;
    const int64_t i = (int64_t)blockIdx.x * kTraceTile + threadIdx.x;
    if (i >= n || blockIdx.x == 0) return;
    const SegVal c = a.tile[blockIdx.x];
    // an element is before the tile's first head iff no head in [tile start, i]
    const uint32_t g = a.keys[i];
    const int64_t s = a.gstart[g];
    if (s < (int64_t)blockIdx.x * kTraceTile) a.out[i] += c.v;
}

}  // namespace ss
