// keys.cuh -- int64 group keys (C4/C5) -> dense group slots.
//
// The reference's groups are dense ids (datagen.py:81-103); the C4 shape
// uses arbitrary int64 keys.  An open-addressing table (linear probing,
// capacity 2^k >= 2G) maps each key to a dense slot in [0, G), and slots
// are assigned in order of FIRST APPEARANCE in the stream, so the slot
// numbering -- which the balancer's lowest-id tie rules see -- is a pure
// function of the stream (equivalent to the reference run on the stream
// relabelled by first appearance, relabel_groups datagen.py:181-192).
//
// Per batch: k_key_probe claims entries for unseen keys (CAS on the key
// word; INT64_MIN is the empty marker and is handled by a dedicated
// entry) and records each new entry's first stream position with
// atomicMin; k_key_mark + k_key_compact order the batch's new entries by
// first position and hand out slots; k_key_map writes the slot of every
// tuple.  Batches without new keys skip the ordering work.
#pragma once

#include "common.cuh"

namespace ss {

constexpr unsigned long long kEmptyKey = 0x8000000000000000ull;   // INT64_MIN

__device__ __forceinline__ unsigned long long key_hash(unsigned long long x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27; x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

struct KeyTable {
    unsigned long long* keys;   // [cap] kEmptyKey = free
    int32_t* slot;              // [cap] dense slot (-1 until assigned)
    unsigned int* first;        // [cap] first position in the current batch (new entries)
    int32_t* ent;               // [n] entry index of each tuple of the batch
    int32_t* new_ent;           // [G] entries claimed in this batch
    int* n_new;
    int* n_slots;               // slots handed out so far
    int32_t* mark;              // [max_batch] entry whose first position is i, or -1
    unsigned long long* slot_keys;   // [G] key of each slot
    int* min_key_entry;         // entry index used for INT64_MIN (-1)
    int* overflow;              // more distinct keys than G
    int* pending;               // some tuple of the batch has a key without a slot yet
    unsigned long long cap_mask;
    int G;
};

// probe / claim.  The table has >= 2G entries, so probing terminates.
// A tuple whose key already has a slot gets it written straight away (the
// steady state: no second pass); a tuple of a key without a slot yet is
// marked pending (out = ~0) with its entry remembered for k_key_map.
constexpr int kProbeILP = 4;

__device__ __forceinline__ int key_entry(KeyTable& t, unsigned long long k, unsigned long long h) {
    while (true) {
        const unsigned long long cur = t.keys[h];
        if (cur == k) return (int)h;
        if (cur == kEmptyKey) {
            const unsigned long long prev = atomicCAS(&t.keys[h], kEmptyKey, k);
            if (prev == kEmptyKey) {
                const int k2 = atomicAdd(t.n_new, 1);
                if (k2 < t.G) t.new_ent[k2] = (int)h; else *t.overflow = 1;
                return (int)h;
            }
            if (prev == k) return (int)h;
        }
        h = (h + 1) & t.cap_mask;
    }
}

__global__ void __launch_bounds__(256)
k_key_probe(const long long* __restrict__ keys, int64_t n, KeyTable t, uint32_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kProbeILP;
    bool any_pending = false;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < n; i0 += stride) {
        unsigned long long k[kProbeILP], cur[kProbeILP], h[kProbeILP];
        // all first probes in flight together
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) {
            const int64_t i = i0 + (int64_t)u * gridDim.x * blockDim.x;
            k[u] = (i < n) ? (unsigned long long)keys[i] : kEmptyKey;
            h[u] = key_hash(k[u]) & t.cap_mask;
        }
        // first probes through the read-only path: the hottest keys' entries
        // are then L1 hits instead of a stream of requests to one L2 slice.
        // A stale read is harmless -- an entry claimed meanwhile is found
        // again by key_entry's CAS (prev == k) or probed past
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) cur[u] = __ldg(t.keys + h[u]);
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) {
            const int64_t i = i0 + (int64_t)u * gridDim.x * blockDim.x;
            if (i >= n) continue;
            int e;
            if (k[u] == kEmptyKey) {
                // the reserved marker value gets a dedicated entry: cap_mask + 1
                e = (int)(t.cap_mask + 1);
                if (atomicCAS(t.min_key_entry, -1, e) == -1) {
                    const int k2 = atomicAdd(t.n_new, 1);
                    if (k2 < t.G) t.new_ent[k2] = e; else *t.overflow = 1;
                }
            } else {
                e = (cur[u] == k[u]) ? (int)h[u] : key_entry(t, k[u], h[u]);
            }
            const int sl = __ldg(t.slot + e);      // slots are assigned by later kernels only
            if (sl >= 0) {
                out[i] = (uint32_t)sl;
            } else {
                out[i] = 0xffffffffu;
                t.ent[i] = e;
                atomicMin(&t.first[e], (unsigned int)i);
                any_pending = true;
            }
        }
    }
    // one flag write per warp (a store per pending tuple would serialise
    // on the flag's L2 slice)
    if (__any_sync(SS_FULL, any_pending) && lane_id() == 0) *t.pending = 1;
}

constexpr int kKeySmall = 2048;     // new keys ranked inside one CTA up to this many

// few new keys: rank them by first position inside one CTA
__global__ void __launch_bounds__(1024)
k_key_rank_small(KeyTable t) {
    __shared__ unsigned int f[kKeySmall];
    __shared__ int32_t en[kKeySmall];
    const int nn = min(*t.n_new, t.G);       // entries past G were never listed (overflow)
    if (nn == 0 || nn > kKeySmall) return;
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
        en[i] = t.new_ent[i];
        f[i] = t.first[en[i]];
    }
    __syncthreads();
    const int base = *t.n_slots;
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
        int r = 0;
        for (int j = 0; j < nn; ++j) r += f[j] < f[i];
        if (base + r < t.G) t.slot[en[i]] = base + r;
        else *t.overflow = 1;
        t.first[en[i]] = 0xffffffffu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *t.n_slots = min(base + nn, t.G);
        *t.n_new = 0;
    }
}
// n_new past kKeySmall is reset by k_key_mark_done

// many new keys: mark[first position] = entry, then an ordered
// compaction over the batch positions (count / scan / assign)
__global__ void __launch_bounds__(256)
k_key_mark(KeyTable t) {
    const int nn = min(*t.n_new, t.G);
    if (nn <= kKeySmall) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
        const int e = t.new_ent[i];
        t.mark[t.first[e]] = e;
    }
}

constexpr int kMarkBlk = 4096;

__global__ void __launch_bounds__(1024)
k_key_mark_count(KeyTable t, int64_t n, int32_t* __restrict__ bsum) {
    __shared__ int32_t red[33];
    if (min(*t.n_new, t.G) <= kKeySmall) return;
    int c = 0;
    for (int q = 0; q < 4; ++q) {
        const int64_t i = (int64_t)blockIdx.x * kMarkBlk + q * 1024 + threadIdx.x;
        c += (i < n && t.mark[i] >= 0);
    }
    int32_t tot;
    block_excl_scan(c, red, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024)
k_key_mark_scan(KeyTable t, int32_t* __restrict__ bsum, int nblk) {
    __shared__ int32_t red[33];
    if (min(*t.n_new, t.G) <= kKeySmall) return;
    int32_t carry = *t.n_slots;
    for (int b0 = 0; b0 < nblk; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const int32_t v = b < nblk ? bsum[b] : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan(v, red, &tot);
        if (b < nblk) bsum[b] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(1024)
k_key_mark_assign(KeyTable t, int64_t n, const int32_t* __restrict__ bsum) {
    __shared__ int32_t red[33];
    if (min(*t.n_new, t.G) <= kKeySmall) return;
    int32_t base = bsum[blockIdx.x];
    for (int q = 0; q < 4; ++q) {
        const int64_t i = (int64_t)blockIdx.x * kMarkBlk + q * 1024 + threadIdx.x;
        int e = -1;
        if (i < n) e = t.mark[i];
        int32_t tot;
        const int32_t ex = block_excl_scan(e >= 0 ? 1 : 0, red, &tot);
        if (e >= 0) {
            if (base + ex < t.G) t.slot[e] = base + ex;
            else *t.overflow = 1;
            t.first[e] = 0xffffffffu;
            t.mark[i] = -1;
        }
        base += tot;
    }
}

__global__ void k_key_mark_done(KeyTable t) {
    const int nn = min(*t.n_new, t.G);
    if (nn <= kKeySmall) return;
    *t.n_slots = min(*t.n_slots + nn, t.G);
    *t.n_new = 0;
}

// pending tuples -> slot; the first tuple of each freshly assigned key
// also records the slot's key
__global__ void __launch_bounds__(256)
k_key_map(const long long* __restrict__ keys, int64_t n, KeyTable t, uint32_t* __restrict__ out) {
    if (*t.pending == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (out[i] != 0xffffffffu) continue;
        const int e = t.ent[i];
        const int s = t.slot[e];
        out[i] = (uint32_t)s;
        if (t.first[e] == 0xffffffffu) {      // first tuple of a freshly assigned key writes it
            if (atomicExch(&t.first[e], 0xfffffffeu) == 0xffffffffu) t.slot_keys[s] = (unsigned long long)keys[i];
        }
    }
}

}  // namespace ss
