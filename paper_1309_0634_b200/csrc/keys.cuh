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
// Table entries are 16 bytes -- key, slot and the slot's hot-cache index
// -- so a probe that hits costs ONE sector read, and the table (32 MB at
// G = 1M) is read with an L2 evict_last policy while the streamed keys use
// evict_first, so it stays resident in the 126 MB L2.
//
// Per batch: k_key_count probes every tuple, writes its slot and counts it
// into the batch's group histogram (count_batch, partition.py:117-130):
// groups hot in the previous batch in shared memory, the rest with
// warp-aggregated global atomics -- the key lookup and the count are one
// pass over the keys.  Tuples of keys without a slot yet (new keys) are
// appended to a pending list and their entries' first stream positions
// recorded with atomicMin; k_key_mark + k_key_compact order the batch's new
// entries by first position and hand out slots; k_key_map writes and
// counts the pending tuples.  Batches without new keys skip that work.
#pragma once

#include "common.cuh"

namespace ss {

constexpr unsigned long long kEmptyKey = 0x8000000000000000ull;   // INT64_MIN

#ifdef SS_KEY_HASH32
// (A/B variant) one 32-bit multiply: fold, Fibonacci-scramble, spread
__device__ __forceinline__ unsigned long long key_hash(unsigned long long x) {
    const uint32_t f = ((uint32_t)x ^ (uint32_t)(x >> 32)) * 0x9E3779B1u;
    return (unsigned long long)(f ^ (f >> 15)) * 0x85EBCA6Bu;
}
#else
__device__ __forceinline__ unsigned long long key_hash(unsigned long long x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27; x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
#endif

struct __align__(16) KEntry {
    unsigned long long key;     // kEmptyKey = free
    int32_t slot;               // dense slot (-1 until assigned)
    int32_t hot;                // index in the count kernel's hot cache, -1 if none
};

struct KeyTable {
    KEntry* ent;                // [cap + 1]; entry cap is INT64_MIN's
    unsigned int* first;        // [cap + 1] first position in the current batch (new entries)
    int32_t* pend;              // [n] tuples whose key had no slot at probe time
    int32_t* pend_ent;          // [n] their entries
    int* n_pend;
    int32_t* new_ent;           // [G] entries claimed in this batch
    int* n_new;
    int* n_slots;               // slots handed out so far
    int32_t* mark;              // [max_batch] entry whose first position is i, or -1
    unsigned long long* slot_keys;   // [G] key of each slot
    int32_t* slot_ent;          // [G] entry of each slot
    int* min_key_entry;         // entry index used for INT64_MIN (-1)
    int* overflow;              // more distinct keys than G
    int* prev_slots;            // n_slots when the batch began (rollback of a rejected batch)
    unsigned long long cap_mask;
    int G;
};

// L2 cache policies: the streamed batch leaves first, the table stays
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ ulonglong2 ld_stream_u64x2(const void* p, unsigned long long pol) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(pol));
    return r;
}
// a table entry through the read-only path: the hottest keys' entries are
// L1 hits.  A stale read is harmless -- an entry claimed meanwhile is found
// again by key_entry's CAS (prev == k) or probed past; slots and hot
// indices are only written by later kernels
__device__ __forceinline__ KEntry ld_entry(const KEntry* p, unsigned long long pol) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;" : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(pol));
    KEntry e;
    e.key = r.x;
    e.slot = (int32_t)(r.y & 0xffffffffull);
    e.hot = (int32_t)(r.y >> 32);
    return e;
}

// probe / claim.  The table has >= 2G entries, so probing terminates.
__device__ __forceinline__ int key_entry(KeyTable& t, unsigned long long k, unsigned long long h) {
    while (true) {
        const unsigned long long cur = t.ent[h].key;
        if (cur == k) return (int)h;
        if (cur == kEmptyKey) {
            const unsigned long long prev = atomicCAS(&t.ent[h].key, kEmptyKey, k);
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

// K2 for int64 keys: probe + slot + count in one pass.  CTA b covers the
// contiguous tuple range [b*range, (b+1)*range) inside one count chunk of S
// tuples (range divides S), counted into row (b*range)/S of gcnt.
constexpr int kKeyItems = 4;
#ifndef SS_KEY_MINB
#define SS_KEY_MINB 2                   // CTAs per SM the register budget allows (A/B build switch)
#endif            // consecutive tuples per thread and round (2 x 16-byte loads)

template <bool COUNT>
__global__ void __launch_bounds__(512, SS_KEY_MINB)
k_key_count(const long long* __restrict__ keys, int64_t n, KeyTable t, uint32_t* __restrict__ out, int64_t S,
            int64_t range, int32_t* __restrict__ gcnt, const int32_t* __restrict__ hot_g, int n_hot, int agg) { SS_PDL_ENTRY();
    extern __shared__ int32_t sh_hist[];                  // [n_hot]
    const int64_t c0 = (int64_t)blockIdx.x * range;
    if (c0 >= n) return;
    const int64_t c1 = min64(n, c0 + range);
    int32_t* dst = COUNT ? gcnt + (c0 / S) * (int64_t)t.G : nullptr;
    if (COUNT) {
        for (int i = threadIdx.x; i < n_hot; i += blockDim.x) sh_hist[i] = 0;
        __syncthreads();
    }
    const unsigned long long pol_s = policy_evict_first(), pol_t = policy_evict_last();
    const unsigned lane = lane_id();
    const bool vec = ((uintptr_t)keys % 16) == 0 && ((uintptr_t)out % 16) == 0;
    for (int64_t base = c0; base < c1; base += (int64_t)kKeyItems * blockDim.x) {
        const int64_t i0 = base + (int64_t)kKeyItems * threadIdx.x;
        unsigned long long k[kKeyItems];
        const bool full = vec && i0 + kKeyItems <= c1;
        if (full) {
            const ulonglong2 a = ld_stream_u64x2(keys + i0, pol_s);
            const ulonglong2 b = ld_stream_u64x2(keys + i0 + 2, pol_s);
            k[0] = a.x; k[1] = a.y; k[2] = b.x; k[3] = b.y;
        } else {
#pragma unroll
            for (int u = 0; u < kKeyItems; ++u) k[u] = (i0 + u < c1) ? (unsigned long long)keys[i0 + u] : kEmptyKey;
        }
        KEntry en[kKeyItems];
        unsigned long long h[kKeyItems];
#pragma unroll
        for (int u = 0; u < kKeyItems; ++u) {
            h[u] = key_hash(k[u]) & t.cap_mask;
            en[u] = ld_entry(t.ent + h[u], pol_t);        // all first probes in flight together
        }
        uint32_t sl[kKeyItems];
        int hot[kKeyItems];
        // fast path: every key of the round at its home entry with a slot
        // (all but a batch's first appearances and probe collisions) --
        // branch-free; anything else goes through one warp-uniform slow path
        bool slow = false;
#pragma unroll
        for (int u = 0; u < kKeyItems; ++u) {
            const bool valid = i0 + u < c1;
            const bool ok = !valid || (en[u].key == k[u] && k[u] != kEmptyKey && en[u].slot >= 0);
            slow |= !ok;
            sl[u] = valid ? (uint32_t)en[u].slot : 0xffffffffu;
            hot[u] = valid ? en[u].hot : -1;
        }
        if (__any_sync(SS_FULL, slow)) {
#pragma unroll
            for (int u = 0; u < kKeyItems; ++u) {
                const int64_t i = i0 + u;
                bool pending = false;
                int e = -1;
                if (i < c1 && !(en[u].key == k[u] && k[u] != kEmptyKey && en[u].slot >= 0)) {
                    if (k[u] == kEmptyKey) {
                        // the reserved marker value gets a dedicated entry: cap_mask + 1
                        e = (int)(t.cap_mask + 1);
                        if (atomicCAS(t.min_key_entry, -1, e) == -1) {
                            const int k2 = atomicAdd(t.n_new, 1);
                            if (k2 < t.G) t.new_ent[k2] = e; else *t.overflow = 1;
                        }
                    } else {
                        e = key_entry(t, k[u], h[u]);
                    }
                    en[u] = ld_entry(t.ent + e, pol_t);
                    if (en[u].slot >= 0) {
                        sl[u] = (uint32_t)en[u].slot;
                        hot[u] = en[u].hot;
                    } else {
                        sl[u] = 0xffffffffu;
                        hot[u] = -1;
                        pending = true;
                        atomicMin(&t.first[e], (unsigned int)i);
                    }
                }
                // pending tuples: one warp-aggregated append to the pending list
                const unsigned pm = __ballot_sync(SS_FULL, pending);
                if (pm) {
                    int pb = 0;
                    if (lane == (unsigned)(__ffs(pm) - 1)) pb = atomicAdd(t.n_pend, __popc(pm));
                    pb = __shfl_sync(SS_FULL, pb, __ffs(pm) - 1);
                    if (pending) {
                        const int r = pb + __popc(pm & lanemask_lt());
                        t.pend[r] = (int32_t)i;
                        t.pend_ent[r] = e;
                    }
                }
            }
        }
        if (COUNT) {
            // count: hot groups in shared memory, the rest one global atomic
            // each (or warp-aggregated, agg: a key hot in this batch but
            // missing from the cache -- drifting skew -- costs one per warp)
#pragma unroll
            for (int u = 0; u < kKeyItems; ++u) {
                uint32_t g = sl[u];
                if (hot[u] >= 0 && hot[u] < n_hot) {
                    atomicAdd(&sh_hist[hot[u]], 1);
                    g = 0xffffffffu;
                }
                if (agg) {
                    const unsigned peers = __match_any_sync(SS_FULL, g);
                    if (g != 0xffffffffu && lane == 31u - __clz(peers)) atomicAdd(&dst[g], __popc(peers));
                } else if (g != 0xffffffffu) {
                    atomicAdd(&dst[g], 1);
                }
            }
        }
        if (full) {
            *(uint4*)(out + i0) = make_uint4(sl[0], sl[1], sl[2], sl[3]);
        } else {
#pragma unroll
            for (int u = 0; u < kKeyItems; ++u)
                if (i0 + u < c1) out[i0 + u] = sl[u];
        }
    }
    if (!COUNT) return;
    __syncthreads();
    for (int i = threadIdx.x; i < n_hot; i += blockDim.x) {
        const int32_t c = sh_hist[i];
        if (c) atomicAdd(&dst[hot_g[i]], c);
    }
}

__global__ void k_key_init(KEntry* ent, int64_t n) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        KEntry e;
        e.key = kEmptyKey;
        e.slot = -1;
        e.hot = -1;
        ent[i] = e;
    }
}

constexpr int kKeySmall = 2048;     // new keys ranked inside one CTA up to this many

__device__ __forceinline__ void assign_slot(KeyTable& t, int e, int s) {
    if (s < t.G) {
        t.ent[e].slot = s;
        t.slot_ent[s] = e;
    } else {
        *t.overflow = 1;
    }
    t.first[e] = 0xffffffffu;
}

// few new keys: rank them by first position inside one CTA
__global__ void __launch_bounds__(1024)
k_key_rank_small(KeyTable t) { SS_PDL_ENTRY();
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
        assign_slot(t, en[i], base + r);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *t.n_slots = min(base + nn, t.G);
        *t.n_new = 0;
    }
}
// n_new past kKeySmall is reset by k_key_mark_done

// A rejected batch (a bad tuple, or more distinct keys than G) must leave
// the engine as it was (validate before mutate, engine.py:281-282): the
// entries its new keys claimed are freed.  They were all claimed after
// every older key, so no older key's probe sequence passes through them
// (linear probing only ever inserts at free entries).
__global__ void __launch_bounds__(256)
k_key_rollback(KeyTable t, int64_t n_ent) { SS_PDL_ENTRY();
    const int keep = *t.prev_slots;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_ent; e += (int64_t)gridDim.x * blockDim.x) {
        const KEntry en = t.ent[e];
        if (en.key == kEmptyKey && e != (int64_t)t.cap_mask + 1) continue;
        if (en.slot >= 0 && en.slot < keep) continue;
        if (e == (int64_t)t.cap_mask + 1 && en.slot < 0 && *t.min_key_entry < 0) continue;
        KEntry z;
        z.key = kEmptyKey;
        z.slot = -1;
        z.hot = -1;
        t.ent[e] = z;
        t.first[e] = 0xffffffffu;
        if (e == (int64_t)t.cap_mask + 1) *t.min_key_entry = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *t.n_slots = keep;
        *t.n_new = 0;
        *t.n_pend = 0;
        *t.overflow = 0;
    }
}

// many new keys: mark[first position] = entry, then an ordered
// compaction over the batch positions (count / scan / assign)
__global__ void __launch_bounds__(256)
k_key_mark(KeyTable t) { SS_PDL_ENTRY();
    const int nn = min(*t.n_new, t.G);
    if (nn <= kKeySmall) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
        const int e = t.new_ent[i];
        t.mark[t.first[e]] = e;
    }
}

constexpr int kMarkBlk = 4096;

__global__ void __launch_bounds__(1024)
k_key_mark_count(KeyTable t, int64_t n, int32_t* __restrict__ bsum) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    if (min(*t.n_new, t.G) <= kKeySmall) return;
    // grid-stride over the 4096-position blocks (a grid of one CTA per
    // block cost ~7 us of launches per batch even when nothing is new)
    const int64_t nblk = (n + kMarkBlk - 1) / kMarkBlk;
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        int c = 0;
        for (int q = 0; q < 4; ++q) {
            const int64_t i = b * kMarkBlk + q * 1024 + threadIdx.x;
            c += (i < n && t.mark[i] >= 0);
        }
        int32_t tot;
        block_excl_scan(c, red, &tot);
        if (threadIdx.x == 0) bsum[b] = tot;
    }
}

__global__ void __launch_bounds__(1024)
k_key_mark_scan(KeyTable t, int32_t* __restrict__ bsum, int nblk) { SS_PDL_ENTRY();
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
k_key_mark_assign(KeyTable t, int64_t n, const int32_t* __restrict__ bsum) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    if (min(*t.n_new, t.G) <= kKeySmall) return;
    const int64_t nblk = (n + kMarkBlk - 1) / kMarkBlk;
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        int32_t base = bsum[b];
        for (int q = 0; q < 4; ++q) {
            const int64_t i = b * kMarkBlk + q * 1024 + threadIdx.x;
            int e = -1;
            if (i < n) e = t.mark[i];
            int32_t tot;
            const int32_t ex = block_excl_scan(e >= 0 ? 1 : 0, red, &tot);
            if (e >= 0) {
                assign_slot(t, e, base + ex);
                t.mark[i] = -1;
            }
            base += tot;
        }
    }
}

__global__ void k_key_mark_done(KeyTable t) { SS_PDL_ENTRY();
    const int nn = min(*t.n_new, t.G);
    if (nn <= kKeySmall) return;
    *t.n_slots = min(*t.n_slots + nn, t.G);
    *t.n_new = 0;
}

// pending tuples -> slot, counted into their chunk's row (a key without a
// slot after assignment -- more distinct keys than G -- is a bad tuple);
// the first tuple of each freshly assigned key records the slot's key
__global__ void __launch_bounds__(256)
k_key_map(const long long* __restrict__ keys, KeyTable t, uint32_t* __restrict__ out, int64_t S,
          int32_t* __restrict__ gcnt, unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    const int np = *t.n_pend;
    const int stride = gridDim.x * blockDim.x;
    // a warp's iterations stay converged (the bound is rounded up to warps)
    const int np_w = (np + 31) & ~31;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < np_w; r += stride) {
        uint32_t g = 0xffffffffu;
        int64_t row = -1;
        if (r < np) {
            const int64_t i = t.pend[r];
            const int e = t.pend_ent[r];
            const int s = t.ent[e].slot;
            out[i] = (uint32_t)s;
            if (s < 0) {
                atomicMin(bad, (unsigned long long)i);
            } else {
                g = (uint32_t)s;
                row = i / S;
                if (t.first[e] == 0xffffffffu) {     // first tuple of a freshly assigned key writes it
                    if (atomicExch(&t.first[e], 0xfffffffeu) == 0xffffffffu) t.slot_keys[s] = (unsigned long long)keys[i];
                }
            }
        }
        // pending tuples of one chunk row and group: one atomic per warp
        const unsigned peers = __match_any_sync(SS_FULL, (unsigned long long)row << 32 | g);
        if (gcnt && g != 0xffffffffu && lane_id() == 31u - __clz(peers))
            atomicAdd(&gcnt[row * t.G + g], __popc(peers));
    }
}

// ---- int64 keys across GPUs -------------------------------------------------
// Keys shard by a hash bucket: bucket(k) = top 16 bits of key_hash(k), and
// the GPU-level engine assigns BUCKETS to GPUs (its "groups" are the 2^16
// buckets), so routing needs no global key -> group dictionary and moving a
// bucket migrates every key of it.  Each GPU keeps its own key table.
constexpr int kKeyBuckets = 1 << 16;
__device__ __forceinline__ uint32_t key_bucket(unsigned long long k) { return (uint32_t)(key_hash(k) >> 48); }

__global__ void __launch_bounds__(256)
k_key_route_prep(const long long* __restrict__ keys, int64_t n, uint32_t* __restrict__ bkt,
                 int32_t* __restrict__ idx) { SS_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        bkt[i] = key_bucket((unsigned long long)keys[i]);
        idx[i] = (int32_t)i;
    }
}

// 12-byte records (key lo, key hi, attr) in the routed order
__global__ void __launch_bounds__(256)
k_key_route_gather(const long long* __restrict__ keys, const int32_t* __restrict__ attrs,
                   const int32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ rec) { SS_PDL_ENTRY();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = idx[j];
        const unsigned long long k = (unsigned long long)keys[i];
        rec[3 * j] = (int32_t)(uint32_t)k;
        rec[3 * j + 1] = (int32_t)(uint32_t)(k >> 32);
        rec[3 * j + 2] = attrs[i];
    }
}

__global__ void __launch_bounds__(256)
k_key_rec_split(const int32_t* __restrict__ rec, int64_t n, long long* __restrict__ keys,
                int32_t* __restrict__ attrs) { SS_PDL_ENTRY();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        keys[j] = (long long)(((unsigned long long)(uint32_t)rec[3 * j + 1] << 32) | (uint32_t)rec[3 * j]);
        attrs[j] = rec[3 * j + 2];
    }
}

// per-bucket counts of the last batch (the GPU-level policy's group counts)
__global__ void __launch_bounds__(256)
k_key_bucket_counts(KeyTable t, const int32_t* __restrict__ gcount, int32_t* __restrict__ out) { SS_PDL_ENTRY();
    const int ns = min(*t.n_slots, t.G);
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ns; g += gridDim.x * blockDim.x) {
        const int32_t c = gcount[g];
        if (c) atomicAdd(&out[key_bucket(t.slot_keys[g])], c);
    }
}

// migration of moved buckets: mark them with their destination, list this
// GPU's slots whose key falls in one
__global__ void __launch_bounds__(256)
k_key_mig_mark(const int4* __restrict__ moves, const int32_t* __restrict__ n_moves, int rank, int n_dest,
               int32_t* __restrict__ bdst) { SS_PDL_ENTRY();
    const int nm = *n_moves;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += gridDim.x * blockDim.x) {
        const int4 m = moves[i];
        if (m.y == rank && m.z != rank && m.z >= 0 && m.z < n_dest && m.x >= 0 && m.x < kKeyBuckets) bdst[m.x] = m.z;
    }
}
__global__ void __launch_bounds__(256)
k_key_mig_collect(KeyTable t, const int32_t* __restrict__ bdst, int2* __restrict__ list, int* __restrict__ n_list,
                  int cap) { SS_PDL_ENTRY();
    const int ns = min(*t.n_slots, t.G);
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ns; g += gridDim.x * blockDim.x) {
        const int d = bdst[key_bucket(t.slot_keys[g])];
        if (d >= 0) {
            const int i = atomicAdd(n_list, 1);
            if (i < cap) list[i] = make_int2(g, d);
        }
    }
}

// claim (or find) the entry of a migrated key and give it a slot at once
// (not through the batch's first-appearance ranking); -1: table full
__device__ __forceinline__ int key_claim_slot(KeyTable& t, unsigned long long k) {
    int e;
    if (k == kEmptyKey) {
        e = (int)(t.cap_mask + 1);
        atomicCAS(t.min_key_entry, -1, e);
    } else {
        unsigned long long h = key_hash(k) & t.cap_mask;
        while (true) {
            const unsigned long long prev = atomicCAS(&t.ent[h].key, kEmptyKey, k);
            if (prev == kEmptyKey || prev == k) break;
            h = (h + 1) & t.cap_mask;
        }
        e = (int)h;
    }
    int s = t.ent[e].slot;
    if (s < 0) {
        s = atomicAdd(t.n_slots, 1);
        if (s >= t.G) {
            *t.overflow = 1;
            return -1;
        }
        t.ent[e].slot = s;
        t.slot_ent[s] = e;
        t.slot_keys[s] = k;
    }
    return s;
}

}  // namespace ss
