// balance.cuh -- K6 (load monitor) + K7 (device rebalancer) + device
// apply_moves for the skewstream B200 pipeline.
//
// Reference (balance.py, partition.py):
//   _rebalance_extremes  balance.py:141-172  hottest->coolest greedy loop,
//                        cap = max_moves or 4P, lowest-id ties, a group
//                        moves at most once, receiver gets it at the BACK
//   get_first 181-200, check_all 203-227, prob_check 230-264,
//   best_balance 267-293, shift 296-342, shift_local 345-385,
//   apply_moves partition.py:181-203
//
// One CTA runs the policy's sequential loop for the whole GPU while the
// rest of the chip executes the batch (the moves only take effect at the
// next batch, harness.py:115-116).  The per-partition loads (and, for
// G <= kBalStageG, the entry lists and counts) live in shared memory; the
// extreme-pair policies run in one warp: donor picks that scan a
// partition's groups (check_all, prob_check, best_balance) are warp
// reductions over the partition's ENTRY list (the list at batch start).
// Working lists never need to be
// materialised: a group moves at most once per invocation, so a working
// list is  [fronts pushed into it, newest first] ++ [entry members not yet
// moved] ++ [backs pushed into it, in order].
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kBalThreads = 512;        // co-resides with a K4 CTA on its SM

struct BalanceArgs {
    int policy;
    long long threshold;
    double pot;
    int cap;
    int P;
    int G;
    const int32_t* order;       // entry lists (CSR)
    const int32_t* offsets;     // [P+1]
    const int32_t* gcount;      // batch group counts
    const unsigned long long* tpt;   // entry loads
    uint8_t* moved;             // [G] scratch, all zero on entry, cleared by apply
    int4* moves;                // (group, src, dst, placement)
    int* front_top;             // [P] newest FRONT-push move index (-1)
    int* back_first;            // [P] first BACK-push move index (-1)
    int* mv_next;               // [cap] next older front / next newer back
    int* n_moves;
    long long* scanned;
    long long* final_tpt;       // [P]
    const unsigned long long* bad;
    const unsigned long long* init_loads;   // split mode: cold-only loads (else tpt)
    const uint8_t* exclude;                 // split mode: hot groups never move
    long long stop_load;                    // split mode: done once max load <= this (0: off)
    const unsigned long long* stop_sum;     // or: ceil(*stop_sum / P), the mean block load (device)
    // large G (entry lists not staged): entry counts and moved/excluded flags
    // by entry POSITION, so a donor scan reads three coalesced arrays
    int32_t* ecnt;              // [G] gcount[order[i]]
    uint8_t* eflag;             // [G] excluded or moved in this invocation
    // fused step: the new list layout for k_apply_place (nullptr: not wanted)
    int32_t* new_off;           // [P+1] offsets of the rebuilt lists
    int32_t* keep_at;           // [P] where the unmoved entry members start
    int32_t* mv_pos;            // [cap] position of every move's group
};

struct BalSmem {
    long long* loads;
    int* ftop;      // newest front push
    int* fbot;      // oldest front push
    int* bfirst;
    int* blast;
    int* elo;       // entry cursor [elo, ehi)
    int* ehi;
    int* esize;     // live entry members
    int* nin;       // pushed-in members
    // staged (G <= kBalStageG): entry order, its batch counts by position and
    // the moved / excluded flag by group, all in shared memory, so a donor
    // scan is no chain of dependent global loads (nullptr otherwise)
    int* sorder;
    int* scnt;
    uint8_t* smv;
};
constexpr int kBalStageG = 16384;

__host__ __device__ inline size_t bal_smem_bytes(int P, int G, bool staged) {
    return (size_t)P * (8 + 8 * 4) + (staged ? (size_t)G * 9 : 0);
}

__device__ __forceinline__ int bal_size(const BalSmem& s, int p) { return s.esize[p] + s.nin[p]; }

// head / tail of a working list (single thread)
__device__ int bal_head(const BalanceArgs& a, const BalSmem& s, int p) {
    if (s.ftop[p] >= 0) return a.moves[s.ftop[p]].x;
    int c = s.elo[p];
    if (s.sorder) while (c < s.ehi[p] && s.smv[s.sorder[c]]) ++c;
    else while (c < s.ehi[p] && a.moved[a.order[c]]) ++c;
    s.elo[p] = c;
    if (c < s.ehi[p]) return s.sorder ? s.sorder[c] : a.order[c];
    if (s.bfirst[p] >= 0) return a.moves[s.bfirst[p]].x;
    return -1;
}
__device__ int bal_tail(const BalanceArgs& a, const BalSmem& s, int p) {
    if (s.blast[p] >= 0) return a.moves[s.blast[p]].x;
    int c = s.ehi[p];
    if (s.sorder) while (c > s.elo[p] && s.smv[s.sorder[c - 1]]) --c;
    else while (c > s.elo[p] && a.moved[a.order[c - 1]]) --c;
    s.ehi[p] = c;
    if (c > s.elo[p]) return s.sorder ? s.sorder[c - 1] : a.order[c - 1];
    if (s.fbot[p] >= 0) return a.moves[s.fbot[p]].x;
    return -1;
}

// record a move of g (an un-moved entry member of src) into dst; c = its
// batch count when the caller has it (< 0: read it)
__device__ void bal_move(const BalanceArgs& a, const BalSmem& s, int* nm, int g, int src, int dst,
                         int placement, long long c = -1) {
    const int mi = *nm;
    a.moves[mi] = make_int4(g, src, dst, placement);
    a.moved[g] = 1;
    if (s.smv) s.smv[g] = 1;
    s.esize[src] -= 1;
    s.nin[dst] += 1;
    a.mv_next[mi] = -1;
    if (placement == 1) {   // BACK
        if (s.blast[dst] >= 0) a.mv_next[s.blast[dst]] = mi;
        else s.bfirst[dst] = mi;
        s.blast[dst] = mi;
    } else {                // FRONT
        a.mv_next[mi] = s.ftop[dst];
        if (s.ftop[dst] < 0) s.fbot[dst] = mi;
        s.ftop[dst] = mi;
    }
    if (c < 0) c = a.gcount[g];
    s.loads[src] -= c;
    s.loads[dst] += c;
    *nm = mi + 1;
}

// entry counts and flags by position for the CTA-wide donor scans
__global__ void __launch_bounds__(256)
k_bal_prep(BalanceArgs a) { SS_PDL_ENTRY();
    if (*a.bad != (unsigned long long)kNoBad) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.G; i += gridDim.x * blockDim.x) {
        const int g = a.order[i];
        a.ecnt[i] = a.gcount[g];
        a.eflag[i] = a.exclude ? a.exclude[g] : 0;
    }
}

// CTA-wide lexicographic (key, id) minimum with a payload; result in every
// thread (uses sh_k / sh_i / sh_x of kBalThreads / 32 entries)
__device__ __forceinline__ void cta_argmin(long long& key, int& id, int& x, long long* sh_k, int* sh_i, int* sh_x) {
    const unsigned lane = lane_id(), w = warp_id();
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const long long ok = __shfl_xor_sync(SS_FULL, key, o);
        const int oi = __shfl_xor_sync(SS_FULL, id, o);
        const int ox = __shfl_xor_sync(SS_FULL, x, o);
        if (ok < key || (ok == key && oi < id)) { key = ok; id = oi; x = ox; }
    }
    if (lane == 0) { sh_k[w] = key; sh_i[w] = id; sh_x[w] = x; }
    __syncthreads();
    key = LLONG_MAX; id = 0x7fffffff; x = -1;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
        if (sh_k[q] < key || (sh_k[q] == key && sh_i[q] < id)) { key = sh_k[q]; id = sh_i[q]; x = sh_x[q]; }
    __syncthreads();
}

template <bool STAGED, bool WIDE = false>
__global__ void __launch_bounds__(kBalThreads)
k_balance(BalanceArgs a) { SS_PDL_ENTRY();
    extern __shared__ long long bal_sm[];
    __shared__ int red_i[72];
    const int P = a.P;
    BalSmem s;
    s.loads = bal_sm;
    int* ib = (int*)(bal_sm + P);
    s.ftop = ib; s.fbot = ib + P; s.bfirst = ib + 2 * P; s.blast = ib + 3 * P;
    s.elo = ib + 4 * P; s.ehi = ib + 5 * P; s.esize = ib + 6 * P; s.nin = ib + 7 * P;
    s.sorder = s.scnt = nullptr;
    s.smv = nullptr;
    if (STAGED) {
        s.sorder = ib + 8 * P;
        s.scnt = s.sorder + a.G;
        s.smv = (uint8_t*)(s.scnt + a.G);
    }
    if (*a.bad != (unsigned long long)kNoBad) {
        if (threadIdx.x == 0) *a.n_moves = 0;
        return;
    }
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        s.loads[p] = (long long)(a.init_loads ? a.init_loads[p] : a.tpt[p]);
        s.ftop[p] = s.fbot[p] = s.bfirst[p] = s.blast[p] = -1;
        s.elo[p] = a.offsets[p];
        s.ehi[p] = a.offsets[p + 1];
        s.esize[p] = a.offsets[p + 1] - a.offsets[p];
        s.nin[p] = 0;
    }
    if (STAGED) {
        for (int i = threadIdx.x; i < a.G; i += blockDim.x) {
            const int g = a.order[i];
            s.sorder[i] = g;
            s.scnt[i] = a.gcount[g];
            s.smv[i] = a.exclude ? a.exclude[i] : 0;
        }
    }
    __syncthreads();
    auto ORD = [&](int i) { return STAGED ? s.sorder[i] : a.order[i]; };
    auto CNT = [&](int i, int g) -> long long { return STAGED ? (long long)s.scnt[i] : (long long)a.gcount[g]; };
    auto MV = [&](int g) -> bool { return STAGED ? s.smv[g] != 0 : (a.moved[g] || (a.exclude && a.exclude[g])); };
    int nm = 0;                // valid in thread 0
    long long scanned = 0;
    const int pol = a.policy;
    const long long stop_load = a.stop_sum ? (long long)((*a.stop_sum + P - 1) / P) : a.stop_load;

    if (WIDE && (pol == 2 || pol == 3 || pol == 4)) {
        // large G: the donor's entry list is scanned by the whole CTA
        // (coalesced, by entry position), one move per round; the extreme
        // pair and the move itself are single-warp / single-thread as below
        __shared__ long long r_k[kBalThreads / 32];
        __shared__ int r_i[kBalThreads / 32], r_x[kBalThreads / 32];
        __shared__ int sh_hi, sh_lo, sh_stop, sh_pick;
        __shared__ long long sh_limit;
        const unsigned lane = lane_id();
        for (;;) {
            if (warp_id() == 0) {
                long long vmax = LLONG_MIN, vmin = LLONG_MAX;
                int imax = 0x7fffffff, imin = 0x7fffffff;
                for (int p = lane; p < P; p += 32) {
                    const long long v = s.loads[p];
                    if (v > vmax) { vmax = v; imax = p; }
                    if (v < vmin) { vmin = v; imin = p; }
                }
                long long nmax = imax == 0x7fffffff ? LLONG_MAX : -vmax;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    long long ok = __shfl_xor_sync(SS_FULL, nmax, o);
                    int oi = __shfl_xor_sync(SS_FULL, imax, o);
                    if (ok < nmax || (ok == nmax && oi < imax)) { nmax = ok; imax = oi; }
                    ok = __shfl_xor_sync(SS_FULL, vmin, o);
                    oi = __shfl_xor_sync(SS_FULL, imin, o);
                    if (ok < vmin || (ok == vmin && oi < imin)) { vmin = ok; imin = oi; }
                }
                if (lane == 0) {
                    const int hi = imax, lo = imin;
                    int stop = (nm >= a.cap) || (s.loads[hi] - s.loads[lo] <= a.threshold) ||
                               (stop_load > 0 && s.loads[hi] <= stop_load);
                    if (!stop && pol == 3) {
                        const int sz = bal_size(s, hi);
                        if (sz <= 0) stop = 1;
                        else sh_limit = (long long)ceil(a.pot * (double)s.loads[hi] / (double)sz);
                    }
                    sh_hi = hi;
                    sh_lo = lo;
                    sh_stop = stop;
                }
            }
            __syncthreads();
            if (sh_stop) break;
            const int hi = sh_hi, lo = sh_lo;
            const int e0 = a.offsets[hi], e1 = a.offsets[hi + 1];
            int pick = -1, pick_i = -1;
            long long pscan = 0, pick_c = -1;
            if (pol == 2 || pol == 4) {
                const long long dmax = s.loads[hi], dmin = s.loads[lo];
                long long bk = LLONG_MAX;
                int bg = 0x7fffffff, bi = -1;
                for (int i = e0 + (int)threadIdx.x; i < e1; i += blockDim.x) {
                    if (a.eflag[i]) continue;
                    const long long c = a.ecnt[i];
                    const int g = a.order[i];
                    long long key;
                    if (pol == 2) key = -c;
                    else {
                        const long long d = (dmax - c) - (dmin + c);
                        key = d < 0 ? -d : d;
                    }
                    if (key < bk || (key == bk && g < bg)) { bk = key; bg = g; bi = i; }
                }
                cta_argmin(bk, bg, bi, r_k, r_i, r_x);
                if (bg != 0x7fffffff) {
                    if (pol == 2) {
                        if (-bk > 0) { pick = bg; pick_i = bi; pscan = (long long)a.tpt[hi]; pick_c = -bk; }
                    } else if (bk < dmax - dmin) {
                        pick = bg;
                        pick_i = bi;
                    }
                }
            } else {
                // prob_check: the first un-moved entry (in list order) with
                // count >= limit; scanned = tuples of the entries before it
                // + limit.  Fallback: max count, lowest id.
                const long long limit = sh_limit;
                long long fk = LLONG_MAX, ck = LLONG_MAX;
                int fg = 0x7fffffff, fi = -1, cg = 0x7fffffff, ci = -1;
                for (int i = e0 + (int)threadIdx.x; i < e1; i += blockDim.x) {
                    if (a.eflag[i]) continue;
                    const long long c = a.ecnt[i];
                    if (c >= limit && ck == LLONG_MAX) { ck = i; cg = 0; ci = i; }   // first candidate of this thread
                    if (c > 0) {
                        const int g = a.order[i];
                        if (-c < fk || (-c == fk && g < fg)) { fk = -c; fg = g; fi = i; }
                    }
                }
                cta_argmin(ck, cg, ci, r_k, r_i, r_x);
                if (ci >= 0) {
                    long long pre = 0;
                    for (int i = e0 + (int)threadIdx.x; i < ci; i += blockDim.x) pre += a.ecnt[i];
                    pre = warp_sum(pre);
                    if (lane == 0) r_k[warp_id()] = pre;
                    __syncthreads();
                    pre = 0;
                    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) pre += r_k[q];
                    __syncthreads();
                    pick = a.order[ci];
                    pick_i = ci;
                    pscan = pre + limit;
                    pick_c = a.ecnt[ci];
                } else {
                    cta_argmin(fk, fg, fi, r_k, r_i, r_x);
                    if (fg != 0x7fffffff && -fk > 0) {
                        pick = fg;
                        pick_i = fi;
                        pscan = (long long)a.tpt[hi];
                        pick_c = -fk;
                    }
                }
            }
            if (threadIdx.x == 0) {
                sh_pick = pick;
                if (pick >= 0) {
                    bal_move(a, s, &nm, pick, hi, lo, 1, pick_c);
                    a.eflag[pick_i] = 1;
                    scanned += pscan;
                }
            }
            __syncthreads();
            if (sh_pick < 0) break;
        }
    } else if (pol == 1 || pol == 2 || pol == 3 || pol == 4) {
        // The extreme-pair loop is sequential: one warp runs it with warp
        // shuffles only (no CTA barriers); the shared-memory state is
        // updated by lane 0 and published to the warp by __syncwarp.
        if (warp_id() == 0) {
            const unsigned lane = lane_id();
            // lexicographic (key, id) minimum over the warp
            auto warp_argmin = [&](long long& key, int& id) {
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const long long ok = __shfl_xor_sync(SS_FULL, key, o);
                    const int oi = __shfl_xor_sync(SS_FULL, id, o);
                    if (ok < key || (ok == key && oi < id)) { key = ok; id = oi; }
                }
            };
            for (;;) {
                // hottest / coolest partition, lowest index on ties
                long long vmax = LLONG_MIN, vmin = LLONG_MAX;
                int imax = 0x7fffffff, imin = 0x7fffffff;
                for (int p = lane; p < P; p += 32) {
                    const long long v = s.loads[p];
                    if (v > vmax) { vmax = v; imax = p; }
                    if (v < vmin) { vmin = v; imin = p; }
                }
                long long nmax = imax == 0x7fffffff ? LLONG_MAX : -vmax;   // argmax as argmin of the negation
                warp_argmin(nmax, imax);
                warp_argmin(vmin, imin);
                const int hi = imax, lo = imin;
                const int nm_all = __shfl_sync(SS_FULL, nm, 0);
                if (nm_all >= a.cap) break;
                if (s.loads[hi] - s.loads[lo] <= a.threshold) break;
                if (stop_load > 0 && s.loads[hi] <= stop_load) break;
                const int e0 = a.offsets[hi], e1 = a.offsets[hi + 1];
                int pick = -1;
                long long pscan = 0, pick_c = -1;
                if (pol == 1) {                       // get_first
                    int r = -1;
                    if (lane == 0) {
                        const int g = bal_head(a, s, hi);
                        if (g >= 0 && !MV(g) && a.gcount[g] != 0) r = g;
                    }
                    pick = __shfl_sync(SS_FULL, r, 0);
                } else if (pol == 2 || pol == 4) {    // check_all / best_balance
                    long long bk = LLONG_MAX;
                    int bg = 0x7fffffff;
                    const long long dmax = s.loads[hi], dmin = s.loads[lo];
                    for (int i = e0 + (int)lane; i < e1; i += 32) {
                        const int g = ORD(i);
                        if (MV(g)) continue;
                        const long long c = CNT(i, g);
                        long long key;
                        if (pol == 2) key = -c;      // max count, lowest id
                        else {
                            const long long d = (dmax - c) - (dmin + c);
                            key = d < 0 ? -d : d;
                        }
                        if (key < bk || (key == bk && g < bg)) { bk = key; bg = g; }
                    }
                    warp_argmin(bk, bg);
                    if (bg != 0x7fffffff) {
                        if (pol == 2) {
                            if (-bk > 0) { pick = bg; pscan = (long long)a.tpt[hi]; pick_c = -bk; }
                        } else {
                            if (bk < dmax - dmin) pick = bg;
                        }
                    }
                } else {                               // prob_check
                    const int sz = bal_size(s, hi);
                    if (sz > 0) {
                        const long long limit = (long long)ceil(a.pot * (double)s.loads[hi] / (double)sz);
                        long long run = 0;             // tuples of the entries before this chunk
                        long long fb_key = LLONG_MAX;  // fallback: max count (as -c), lowest id
                        int fb_g = 0x7fffffff;
                        for (int c0 = e0; c0 < e1; c0 += 32) {
                            const int i = c0 + (int)lane;
                            int g = -1;
                            long long c = 0;
                            bool cand = false;
                            if (i < e1) {
                                g = ORD(i);
                                c = CNT(i, g);
                                const bool mv = MV(g);
                                cand = (c >= limit) && !mv;
                                if (!mv && c > 0) {
                                    const long long key = -c;
                                    if (key < fb_key || (key == fb_key && g < fb_g)) { fb_key = key; fb_g = g; }
                                }
                            }
                            const long long incl = warp_incl_scan(c);
                            const unsigned cb = __ballot_sync(SS_FULL, cand);
                            if (cb) {                  // first candidate in entry order
                                const int f = __ffs(cb) - 1;
                                pick = __shfl_sync(SS_FULL, g, f);
                                pscan = run + __shfl_sync(SS_FULL, incl - c, f) + limit;
                                pick_c = __shfl_sync(SS_FULL, c, f);
                                break;
                            }
                            run += __shfl_sync(SS_FULL, incl, 31);
                        }
                        if (pick < 0) {
                            warp_argmin(fb_key, fb_g);
                            if (fb_g != 0x7fffffff && -fb_key > 0) {
                                pick = fb_g;
                                pscan = (long long)a.tpt[hi];
                                pick_c = -fb_key;
                            }
                        }
                    }
                }
                if (pick < 0) break;
                __syncwarp();                          // every lane's reads of the moved flags precede the move
                if (lane == 0) {
                    bal_move(a, s, &nm, pick, hi, lo, 1, pick_c);
                    scanned += pscan;
                }
                __syncwarp();
            }
        }
    } else if (threadIdx.x == 0 && pol == 5) {     // shift
        while (nm < a.cap) {
            int hi = 0, lo = 0;
            for (int p = 1; p < P; ++p) {
                if (s.loads[p] > s.loads[hi]) hi = p;
                if (s.loads[p] < s.loads[lo]) lo = p;
            }
            if (s.loads[hi] - s.loads[lo] <= a.threshold) break;
            const bool down = hi > lo;
            const int b = down ? lo + 1 : hi, e = down ? hi + 1 : lo;
            int emitted = 0;
            for (int i = b; i < e; ++i) {
                if (nm >= a.cap) break;
                if (bal_size(s, i) == 0) continue;
                const int g = down ? bal_head(a, s, i) : bal_tail(a, s, i);
                if (g < 0 || MV(g)) continue;
                bal_move(a, s, &nm, g, i, down ? i - 1 : i + 1, down ? 1 : 0);
                ++emitted;
            }
            if (emitted == 0) break;
        }
    } else if (threadIdx.x == 0 && pol == 6) {     // shift_local
        for (int i = 0; i + 1 < P; ++i) {
            if (nm >= a.cap) break;
            int src, dst;
            bool last;
            if (s.loads[i] - s.loads[i + 1] > a.threshold) { src = i; dst = i + 1; last = true; }
            else if (s.loads[i + 1] - s.loads[i] > a.threshold) { src = i + 1; dst = i; last = false; }
            else continue;
            if (bal_size(s, src) == 0) continue;
            const int g = last ? bal_tail(a, s, src) : bal_head(a, s, src);
            if (g < 0 || MV(g)) continue;
            bal_move(a, s, &nm, g, src, dst, last ? 0 : 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *a.n_moves = nm;
        *a.scanned = scanned;
    }
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        a.final_tpt[p] = s.loads[p];
        a.front_top[p] = s.ftop[p];
        a.back_first[p] = s.bfirst[p];
    }
    if (a.new_off) {
        // new list of p = fronts pushed in (newest first) ++ entry members
        // not moved ++ backs pushed in (in order): offsets from the final
        // sizes, every move's position by walking p's push chains (thread p)
        __shared__ int32_t sh_carry;
        if (threadIdx.x == 0) sh_carry = 0;
        __syncthreads();
        for (int p0 = 0; p0 < P; p0 += blockDim.x) {
            const int p = p0 + threadIdx.x;
            const int32_t sz = p < P ? s.esize[p] + s.nin[p] : 0;
            int32_t tot;
            const int32_t ex = block_excl_scan(sz, red_i, &tot);
            if (p < P) {
                int pos = sh_carry + ex;
                a.new_off[p] = pos;
                for (int mi = s.ftop[p]; mi >= 0; mi = a.mv_next[mi]) a.mv_pos[mi] = pos++;
                a.keep_at[p] = pos;
                pos += s.esize[p];
                for (int mi = s.bfirst[p]; mi >= 0; mi = a.mv_next[mi]) a.mv_pos[mi] = pos++;
            }
            __syncthreads();
            if (threadIdx.x == 0) sh_carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) a.new_off[P] = sh_carry;
    }
}

// ---- device apply_moves (partition.py:181-203) ------------------------------
// new list(p) = fronts pushed into p (newest first) ++ entry members of p
// that did not move ++ backs pushed into p (in order); k_balance lays the
// new lists out (offsets, unmoved-member starts, move positions).
// fused step: the rebuilt lists from the layout k_balance computed (one
// CTA per partition places its unmoved entry members; the moved groups are
// scattered to their positions by all CTAs)
__global__ void __launch_bounds__(256)
k_apply_place(const int32_t* __restrict__ order, const int32_t* __restrict__ offsets,
              const int32_t* __restrict__ keep_at, const int4* __restrict__ moves, const int* __restrict__ n_moves,
              const int32_t* __restrict__ mv_pos, const uint8_t* __restrict__ moved, int32_t* __restrict__ new_order) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    const int nm = *n_moves;
    if (nm == 0) return;
    const int p = blockIdx.x;
    for (int mi = blockIdx.x * blockDim.x + threadIdx.x; mi < nm; mi += gridDim.x * blockDim.x)
        new_order[mv_pos[mi]] = moves[mi].x;
    int pos = keep_at[p];
    const int e0 = offsets[p], e1 = offsets[p + 1];
    for (int c0 = e0; c0 < e1; c0 += blockDim.x) {
        const int i = c0 + threadIdx.x;
        int g = -1;
        int keep = 0;
        if (i < e1) {
            g = order[i];
            keep = !moved[g];
        }
        int32_t tot;
        const int32_t ex = block_excl_scan(keep, red, &tot);
        if (keep) new_order[pos + ex] = g;
        pos += tot;
    }
}

// commit: copy the rebuilt lists, update the group->partition map, clear
// the moved flags
__global__ void __launch_bounds__(256)
k_apply_commit(int32_t* __restrict__ order, int32_t* __restrict__ offsets, const int32_t* __restrict__ new_order,
               const int32_t* __restrict__ new_off, int G, int P, const int4* __restrict__ moves,
               const int* __restrict__ n_moves, int32_t* __restrict__ pmap, uint8_t* __restrict__ moved) { SS_PDL_ENTRY();
    const int nm = *n_moves;
    if (nm == 0) return;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (int i = tid; i < G; i += nt) order[i] = new_order[i];
    for (int i = tid; i <= P; i += nt) offsets[i] = new_off[i];
    for (int i = tid; i < nm; i += nt) {
        const int4 m = moves[i];
        pmap[m.x] = m.z;
        moved[m.x] = 0;
    }
}

}  // namespace ss
