// hcb_solve.cu -- device-resident IPGC solve (hc_solve).
//
// Replaces the reference's whole `color_graph` round loop
// (pkg/src/hybridcolor/driver.py:122-176) together with the round functions
// (coloring.py:113-176), the kernels (_kernels.pyx:29-149) and the worklist
// swap (worklist.py:77-91) by ONE cooperatively launched persistent kernel
// (one 1024-thread CTA per SM): every round is
//     assign -> grid barrier -> resolve -> grid barrier
// with the hybrid mode decision, the worklist and the per-round records kept
// on the device, so there is no host round trip per round.
//
// State encoding (one 32-bit word per node, X[u]):
//   X[u] == 0                 never assigned
//   X[u] == T (bit31 clear)   uncolored; T = tentative color of the current /
//                             last round (a loser keeps its stale T)
//   X[u] == C | FBIT          permanently colored with C
// Equivalence with the reference's (colors_read, colors_write, stamp) triple
// (SURVEY.md Appendix A):
//   * assign reads only committed colors: it ignores words without FBIT, which
//     is exactly "active neighbours read 0" (colors_read of a loser is reset by
//     the commit at coloring.py:140/174).
//   * resolve counts v<u with color(X[v]) == T[u].  The reference's extra test
//     stamp[v]==round (_kernels.pyx:113) is implied: a neighbour committed in an
//     earlier round has a color T[u] avoided (T[u] is the mex over committed
//     neighbour colors), and every uncolored node is active in every round
//     (data: worklist == {C==0}; topo: activity C==0).  Winners of the current
//     round set FBIT during resolve without changing the color bits, so
//     concurrent readers see the same color either way; losers keep T so they
//     still count for higher neighbours (test_coloring.py:84-91).
//   * winners commit C[u]=T[u] in resolve itself; no separate commit pass.
//
// Work distribution (IrGL-style nested parallelism):
// nodes are binned once by degree -- small (thread per node), mid (warp per
// node), hub (CTA per node).  The always-maintained worklist is kept per bin
// and double buffered.  Each phase hands out units with ONE atomic per unit:
// hub nodes first (largest work first), then chunks of mid nodes, then chunks
// of small nodes.  Losers of chunk c are compacted (order-preserving for the
// small bin) into output segment c of the next worklist and the chunk writes
// its loser count; the next round rebuilds the segment prefix in shared
// memory.  So pushes need no global atomics, the worklist stays sorted by id
// (segments are in chunk order), and topology-driven rounds (static bin lists
// + activity test) and data-driven rounds (segmented dynamic lists) share the
// same code.
#include <algorithm>

#include "hcb_partition.cuh"

namespace hcb {
namespace solve {

constexpr int BLOCK = 1024;
constexpr int NW = BLOCK / 32;
constexpr int SMALL_MAX = 16;            // deg <= SMALL_MAX : thread per node (64-bit mask mex)
constexpr int MID_WORDS = 64;            // warp bitmap words -> mid nodes up to 2046 neighbours
constexpr int MID_MAX = MID_WORDS * 32 - 2;
constexpr int HUB_WORDS = 512;           // CTA bitmap window: 16384 colors per pass
constexpr int MAXSEG = 2048;             // output segments per bin per round
constexpr unsigned FBIT = 0x80000000u;
constexpr unsigned CMASK = 0x7fffffffu;

enum { BIN_SMALL = 0, BIN_MID = 1, BIN_HUB = 2, NBIN = 3 };

struct Ctrl {
    GridBarrier bar;
    int error;
    int pad0;
    unsigned long long nstat[NBIN];              // static bin sizes
    unsigned long long hub_cnt[2];               // hub worklist size per parity
    unsigned long long conflicts[2];
    unsigned int unit_ctr[2][2];                 // [phase][parity]
    long long rounds;
    long long rec_overflow;
    unsigned segcnt[2][2][MAXSEG];               // [parity][small|mid][segment] loser counts
};

struct Params {
    const long long *ro;
    const int *ci;
    long long n;
    unsigned *X;
    int *stat;                 // static lists, bins contiguous (small | mid | hub)
    int *dyn[2][NBIN];         // dynamic lists per parity and bin
    Ctrl *ctrl;
    hc_round_rec *rec;
    long long max_rec;
    long long *colors_out;
    int mode;
    long long thr;
    unsigned nblocks;
    long long *stats;          // optional int64[max_rec][2]: (assign edges, resolve lower edges)
};

struct Smem {
    unsigned prefix[2][MAXSEG + 1];   // segment prefix of the current small / mid lists
    unsigned mid_bm[NW][MID_WORDS];
    unsigned hub_bm[HUB_WORDS];
    unsigned warp_tmp[NW];
    unsigned long long red;
    int hub_first;
    unsigned unit;
    unsigned out_cnt;
};

// A bin's current list: dense (static list / round 1) or segmented (the
// previous round's output: nseg segments of capacity segcap).
struct List {
    const int *base;
    unsigned long long total;
    unsigned nseg, segcap;
    bool segmented;
};

__device__ __forceinline__ long long list_index(const List &L, const unsigned *prefix, unsigned long long v) {
    if (!L.segmented) return (long long)v;
    // last segment s with prefix[s] <= v (segments may be empty)
    unsigned lo = 0, hi = L.nseg;  // invariant prefix[lo] <= v < prefix[hi]
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (prefix[mid] <= v) lo = mid;
        else hi = mid;
    }
    return (long long)lo * L.segcap + (long long)(v - prefix[lo]);
}

// chunk size so a bin produces at most MAXSEG segments; multiple of `tile`
__device__ __forceinline__ unsigned chunk_size(unsigned long long total, unsigned tile) {
    unsigned long long c = (total + MAXSEG - 1) / MAXSEG;
    c = (c + tile - 1) / tile * tile;
    return (unsigned)max(c, (unsigned long long)tile);
}

// ------------------------------------------------------------------ small
__device__ __forceinline__ unsigned assign_small(const Params &P, int u) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned long long mask = 0;
    for (long long k = b; k < e; k += 4) {
        int v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (k + j < e) ? P.ci[k + j] : -1;
        unsigned x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = v[j] >= 0 ? P.X[v[j]] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned c = x[j] & CMASK;
            if ((x[j] & FBIT) && c <= 64u) mask |= 1ull << (c - 1u);
        }
    }
    return (unsigned)__ffsll((long long)~mask);  // deg <= SMALL_MAX < 64: a zero bit exists
}

__device__ __forceinline__ unsigned resolve_small(const Params &P, int u, unsigned T, unsigned &lower) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned cnt = 0, low = 0;
    for (long long k = b; k < e; k += 4) {
        int v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (k + j < e) ? P.ci[k + j] : 0x7fffffff;
        bool done = false;
        unsigned x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = v[j] < u ? P.X[v[j]] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (v[j] < u) { cnt += (x[j] & CMASK) == T; ++low; }
            else done = true;
        }
        if (done) break;  // adjacency is sorted ascending (graph.py:193-197)
    }
    lower = low;
    return cnt;
}

// ------------------------------------------------------------------ mid (warp)
__device__ __forceinline__ unsigned assign_mid(const Params &P, int u, unsigned *bm) {
    const unsigned lane = lane_id();
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;  // mex <= deg+1 (_kernels.pyx:49)
#pragma unroll
    for (int w = 0; w < MID_WORDS / 32; ++w) bm[lane + 32 * w] = 0u;
    __syncwarp();
    for (long long k = b + lane; k < e; k += 64) {
        const int v0 = P.ci[k];
        const int v1 = (k + 32 < e) ? P.ci[k + 32] : -1;
        const unsigned x0 = P.X[v0];
        const unsigned x1 = v1 >= 0 ? P.X[v1] : 0u;
        unsigned c = x0 & CMASK;
        if ((x0 & FBIT) && c <= lim) atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
        c = x1 & CMASK;
        if ((x1 & FBIT) && c <= lim) atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
    }
    __syncwarp();
    unsigned T = 0;
#pragma unroll
    for (int w = 0; w < MID_WORDS / 32; ++w) {
        const unsigned word = bm[lane + 32 * w];
        const unsigned bal = __ballot_sync(FULL, word != FULL);
        if (bal) {
            const int f = __ffs(bal) - 1;
            const unsigned fw = __shfl_sync(FULL, word, f);
            T = (unsigned)((w * 32 + f) * 32 + __ffs(~fw));
            break;
        }
    }
    __syncwarp();
    return T;
}

__device__ __forceinline__ unsigned resolve_mid(const Params &P, int u, unsigned T, unsigned &lower_out) {
    const unsigned lane = lane_id();
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned cnt = 0, low = 0;
    for (long long k0 = b; k0 < e; k0 += 32) {
        const long long k = k0 + lane;
        const int v = k < e ? P.ci[k] : 0x7fffffff;
        const bool lower = v < u;
        if (lower) { cnt += (P.X[v] & CMASK) == T; ++low; }
        if (__ballot_sync(FULL, !lower)) break;
    }
    lower_out = warp_sum(low);
    return warp_sum(cnt);
}

// ------------------------------------------------------------------ hub (CTA)
__device__ unsigned assign_hub(const Params &P, int u, Smem &sm) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;
    for (unsigned w0 = 0;; w0 += HUB_WORDS * 32) {
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK) sm.hub_bm[i] = 0u;
        if (threadIdx.x == 0) sm.hub_first = 0x7fffffff;
        __syncthreads();
        const unsigned hi = min(lim, w0 + HUB_WORDS * 32);
        for (long long k = b + threadIdx.x; k < e; k += 2 * BLOCK) {
            const int v0 = P.ci[k];
            const int v1 = (k + BLOCK < e) ? P.ci[k + BLOCK] : -1;
            const unsigned x0 = P.X[v0];
            const unsigned x1 = v1 >= 0 ? P.X[v1] : 0u;
            unsigned c = x0 & CMASK;
            if ((x0 & FBIT) && c > w0 && c <= hi)
                atomicOr(&sm.hub_bm[(c - w0 - 1u) >> 5], 1u << ((c - w0 - 1u) & 31u));
            c = x1 & CMASK;
            if ((x1 & FBIT) && c > w0 && c <= hi)
                atomicOr(&sm.hub_bm[(c - w0 - 1u) >> 5], 1u << ((c - w0 - 1u) & 31u));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK)
            if (sm.hub_bm[i] != FULL) { atomicMin(&sm.hub_first, i); break; }
        __syncthreads();
        const int f = sm.hub_first;
        if (f != 0x7fffffff) {
            const unsigned T = w0 + (unsigned)f * 32u + (unsigned)__ffs(~sm.hub_bm[f]);
            __syncthreads();
            return T;
        }
        __syncthreads();
    }
}

__device__ unsigned resolve_hub(const Params &P, int u, unsigned T, Smem &sm, unsigned &lower_out) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    if (threadIdx.x == 0) sm.red = 0;
    __syncthreads();
    unsigned cnt = 0, low = 0;
    for (long long k0 = b + (long long)warp * 32; k0 < e; k0 += (long long)BLOCK) {
        const long long k = k0 + lane;
        const int v = k < e ? P.ci[k] : 0x7fffffff;
        const bool lower = v < u;
        if (lower) { cnt += (P.X[v] & CMASK) == T; ++low; }
        if (__ballot_sync(FULL, !lower)) break;  // later chunks are all >= u
    }
    cnt = warp_sum(cnt);
    low = warp_sum(low);
    // counts packed: conflicts in the low 32 bits, lower-neighbour visits above
    if (lane == 0 && (cnt | low)) atomicAdd(&sm.red, (unsigned long long)cnt | ((unsigned long long)low << 32));
    __syncthreads();
    const unsigned long long r = sm.red;
    __syncthreads();
    lower_out = (unsigned)(r >> 32);
    return (unsigned)r;
}

// block-wide exclusive scan of one flag per thread; returns this thread's rank,
// *total = number of set flags.  All threads must call.
__device__ __forceinline__ unsigned block_rank(bool flag, unsigned *total, Smem &sm) {
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned bal = __ballot_sync(FULL, flag);
    if (lane == 0) sm.warp_tmp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
        const unsigned v = sm.warp_tmp[lane];
        const unsigned incl = warp_incl_scan(v);
        sm.warp_tmp[lane] = incl - v;
        if (lane == 31) sm.red = incl;  // reuse: total
    }
    __syncthreads();
    const unsigned r = sm.warp_tmp[warp] + __popc(bal & lanemask_lt());
    *total = (unsigned)sm.red;
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ kernel
template <bool STATS>
__global__ void __launch_bounds__(BLOCK, 1) solve_kernel(Params P) {
    __shared__ Smem sm;
    Ctrl *C = P.ctrl;
    const unsigned lane = lane_id();
    const unsigned warp = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long gthreads = (long long)P.nblocks * BLOCK;

    for (long long u = gtid; u < P.n; u += gthreads) P.X[u] = 0u;
    const unsigned long long nst[NBIN] = {C->nstat[0], C->nstat[1], C->nstat[2]};
    const int *stat_lists[NBIN] = {P.stat, P.stat + nst[0], P.stat + nst[0] + nst[1]};
    const bool ident_small = nst[0] == (unsigned long long)P.n;  // all nodes small: sweep ids
    grid_sync(&C->bar, P.nblocks);

    // previous round's output geometry (identical in every CTA)
    unsigned prev_nseg[2] = {0, 0}, prev_cap[2] = {0, 0};
    unsigned long long t_start = 0;
    long long wl_in_prev = 0;
    int topo_prev = 0;
    unsigned long long my_conf = 0;
    unsigned long long my_edges[2] = {0, 0};  // stats: assign edges, resolve lower edges
    constexpr bool stats = STATS;
    long long t = 1;
    for (;; ++t) {
        const int p = (int)(t & 1), np = p ^ 1;
        // ---- current worklist sizes: rebuild the segment prefix of the
        //      previous round's output (round 1: the full static lists)
        List L[NBIN];
        for (int b = 0; b < 2; ++b) {
            if (t == 1) {
                L[b] = List{stat_lists[b], nst[b], 0, 0, false};
            } else {
                const unsigned ns = prev_nseg[b];
                for (unsigned s = threadIdx.x; s < ns; s += BLOCK)
                    sm.prefix[b][s + 1] = __ldcg(&C->segcnt[p][b][s]);
                if (threadIdx.x == 0) sm.prefix[b][0] = 0;
                __syncthreads();
                // inclusive scan of prefix[1..ns] (ns <= MAXSEG = 2*BLOCK)
                {
                    const unsigned i0 = 1 + 2 * threadIdx.x, i1 = i0 + 1;
                    const unsigned a0 = i0 <= ns ? sm.prefix[b][i0] : 0u;
                    const unsigned a1 = i1 <= ns ? sm.prefix[b][i1] : 0u;
                    const unsigned pair = a0 + a1;
                    const unsigned incl = warp_incl_scan(pair);
                    if (lane == 31) sm.warp_tmp[warp] = incl;
                    __syncthreads();
                    if (warp == 0) {
                        const unsigned v = sm.warp_tmp[lane];
                        sm.warp_tmp[lane] = warp_incl_scan(v) - v;
                    }
                    __syncthreads();
                    const unsigned ex = sm.warp_tmp[warp] + incl - pair;
                    if (i0 <= ns) sm.prefix[b][i0] = ex + a0;
                    if (i1 <= ns) sm.prefix[b][i1] = ex + pair;
                    __syncthreads();
                }
                L[b] = List{P.dyn[p][b], sm.prefix[b][ns], ns, prev_cap[b], true};
            }
        }
        const unsigned long long hub_total = t == 1 ? nst[BIN_HUB] : ld_relaxed_u64(&C->hub_cnt[p]);
        L[BIN_HUB] = List{t == 1 ? stat_lists[BIN_HUB] : P.dyn[p][BIN_HUB], hub_total, 0, 0, false};
        const unsigned long long s = L[0].total + L[1].total + L[2].total;
        const bool topo = P.mode == HC_MODE_TOPO || (P.mode == HC_MODE_HYBRID && (long long)s > P.thr);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const unsigned long long now = globaltimer();
            if (t > 1) {  // finish the record of round t-1 (driver.py:159-168)
                const int q = np;
                if (t - 1 <= P.max_rec) {
                    hc_round_rec r;
                    r.round = t - 1;
                    r.topo = topo_prev;
                    r.wl_in = wl_in_prev;
                    r.wl_out = (long long)s;
                    r.conflicts = (long long)C->conflicts[q];
                    r.ns = (long long)(now - t_start);
                    P.rec[t - 2] = r;
                }
                C->conflicts[q] = 0;
                C->hub_cnt[q] = 0;
                C->unit_ctr[0][q] = C->unit_ctr[1][q] = 0;
            }
            t_start = now;
            wl_in_prev = (long long)s;
            topo_prev = topo;
        }
        if (s == 0) break;  // worklist drained (driver.py:145)

        if (topo) {  // topology-driven: sweep the static lists, activity test
            for (int b = 0; b < NBIN; ++b) L[b] = List{stat_lists[b], nst[b], 0, 0, false};
        }
        const bool ident = topo && ident_small;
        const unsigned csz[2] = {chunk_size(L[0].total, BLOCK), chunk_size(L[1].total, NW)};
        const unsigned nch[2] = {(unsigned)((L[0].total + csz[0] - 1) / csz[0]),
                                 (unsigned)((L[1].total + csz[1] - 1) / csz[1])};
        const unsigned n_hub = (unsigned)L[BIN_HUB].total;
        const unsigned units = n_hub + nch[1] + nch[0];

        for (int phase = 0; phase < 2; ++phase) {
            unsigned *ctr = &C->unit_ctr[phase][p];
            if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);
            __syncthreads();
            unsigned unit = sm.unit;
            __syncthreads();
            while (unit < units) {
                if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);  // prefetch the next unit
                if (unit < n_hub) {
                    // ---- hub: one CTA per node
                    const int u = L[BIN_HUB].base[unit];
                    const unsigned xu = P.X[u];
                    if (!(topo && (xu & FBIT))) {  // topology sweep: inactive (_kernels.pyx:76)
                        if (phase == 0) {
                            const unsigned T = assign_hub(P, u, sm);
                            if (threadIdx.x == 0) {
                                P.X[u] = T;
                                if (stats) my_edges[0] += P.ro[u + 1] - P.ro[u];
                            }
                        } else {
                            unsigned low;
                            const unsigned k = resolve_hub(P, u, xu, sm, low);
                            if (threadIdx.x == 0) {
                                my_conf += k;
                                if (stats) my_edges[1] += low;
                                if (k) P.dyn[np][BIN_HUB][atomicAdd(&C->hub_cnt[np], 1ull)] = u;
                                else P.X[u] = xu | FBIT;
                            }
                        }
                    }
                } else if (unit < n_hub + nch[1]) {
                    // ---- mid chunk: one warp per node
                    const unsigned c = unit - n_hub;
                    const unsigned long long lo = (unsigned long long)c * csz[1];
                    const unsigned long long hi = min(lo + csz[1], L[1].total);
                    int *out = P.dyn[np][BIN_MID] + (long long)c * csz[1];
                    if (threadIdx.x == 0) sm.out_cnt = 0;
                    __syncthreads();
                    for (unsigned long long v = lo + warp; v < hi; v += NW) {
                        const int u = L[1].base[list_index(L[1], sm.prefix[1], v)];
                        const unsigned xu = P.X[u];
                        if (topo && (xu & FBIT)) continue;
                        if (phase == 0) {
                            const unsigned T = assign_mid(P, u, sm.mid_bm[warp]);
                            if (lane == 0) {
                                P.X[u] = T;
                                if (stats) my_edges[0] += P.ro[u + 1] - P.ro[u];
                            }
                        } else {
                            unsigned low;
                            const unsigned k = resolve_mid(P, u, xu, low);
                            if (lane == 0) {
                                my_conf += k;
                                if (stats) my_edges[1] += low;
                                if (k) out[atomicAdd(&sm.out_cnt, 1u)] = u;
                                else P.X[u] = xu | FBIT;
                            }
                        }
                    }
                    __syncthreads();
                    if (phase == 1 && threadIdx.x == 0) C->segcnt[np][1][c] = sm.out_cnt;
                } else {
                    // ---- small chunk: one thread per node, ordered compaction
                    const unsigned c = unit - n_hub - nch[1];
                    const unsigned long long lo = (unsigned long long)c * csz[0];
                    const unsigned long long hi = min(lo + csz[0], L[0].total);
                    int *out = P.dyn[np][BIN_SMALL] + (long long)c * csz[0];
                    unsigned written = 0;
                    for (unsigned long long base = lo; base < hi; base += BLOCK) {
                        const unsigned long long v = base + threadIdx.x;
                        int u = -1;
                        unsigned xu = 0;
                        if (v < hi) {
                            u = ident ? (int)v : L[0].base[list_index(L[0], sm.prefix[0], v)];
                            xu = P.X[u];
                            if (topo && (xu & FBIT)) u = -1;
                        }
                        bool lost = false;
                        if (u >= 0) {
                            if (phase == 0) {
                                P.X[u] = assign_small(P, u);
                                if (stats) my_edges[0] += P.ro[u + 1] - P.ro[u];
                            } else {
                                unsigned low;
                                const unsigned k = resolve_small(P, u, xu, low);
                                my_conf += k;
                                if (stats) my_edges[1] += low;
                                lost = k != 0;
                                if (!lost) P.X[u] = xu | FBIT;
                            }
                        }
                        if (phase == 1) {
                            unsigned tot;
                            const unsigned r = block_rank(lost, &tot, sm);
                            if (lost) out[written + r] = u;
                            written += tot;
                        }
                    }
                    if (phase == 1 && threadIdx.x == 0) C->segcnt[np][0][c] = written;
                }
                __syncthreads();
                unit = sm.unit;
                __syncthreads();
            }
            if (phase == 0) grid_sync(&C->bar, P.nblocks);
        }
        // conflicts of this round: block reduce then one atomic per CTA
        {
            unsigned long long v = warp_sum(my_conf);
            my_conf = 0;
            if (threadIdx.x == 0) sm.red = 0;
            __syncthreads();
            if (lane == 0 && v) atomicAdd(&sm.red, v);
            __syncthreads();
            if (threadIdx.x == 0 && sm.red) atomicAdd(&C->conflicts[p], sm.red);
            if (stats) {
                __syncthreads();
                for (int q = 0; q < 2; ++q) {
                    const unsigned long long e = warp_sum(my_edges[q]);
                    my_edges[q] = 0;
                    if (lane == 0 && e && t <= P.max_rec)
                        atomicAdd((unsigned long long *)&P.stats[2 * (t - 1) + q], e);
                }
            }
        }
        prev_nseg[0] = nch[0]; prev_nseg[1] = nch[1];
        prev_cap[0] = csz[0]; prev_cap[1] = csz[1];
        grid_sync(&C->bar, P.nblocks);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->rounds = t - 1;
        if (t - 1 > P.max_rec) C->rec_overflow = 1;
    }
    for (long long u = gtid; u < P.n; u += gthreads) P.colors_out[u] = (long long)(P.X[u] & CMASK);
}

// degree classifier for the static bins
struct DegreeBin {
    const long long *ro;
    __device__ int operator()(long long i) const {
        const long long d = ro[i + 1] - ro[i];
        return d <= SMALL_MAX ? BIN_SMALL : (d <= MID_MAX ? BIN_MID : BIN_HUB);
    }
};
struct EmitI32 {
    __device__ int operator()(long long i) const { return (int)i; }
};

__global__ void copy_totals_kernel(const unsigned long long *totals, Ctrl *c) {
    if (threadIdx.x < NBIN) c->nstat[threadIdx.x] = totals[threadIdx.x];
}

// worst-case segmented capacity of a bin with `cnt` static nodes
inline size_t seg_capacity(long long cnt) {
    return (size_t)cnt + (size_t)cnt / MAXSEG + 2 * BLOCK;
}

struct Layout {
    size_t x, stat, dyn[2][NBIN], ctrl, part, total;
};

// The dynamic bin regions depend on the bin sizes, which are only known on
// the device; size each for the whole node count (upper bound of every bin).
static Layout layout(long long n) {
    Layout L;
    size_t o = 0;
    L.x = o; o = align_up(o + 4 * (size_t)n, 256);
    L.stat = o; o = align_up(o + 4 * (size_t)n, 256);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NBIN; ++b) {
            L.dyn[p][b] = o;
            o = align_up(o + 4 * (b == BIN_HUB ? (size_t)n : seg_capacity(n)), 256);
        }
    L.ctrl = o; o = align_up(o + sizeof(Ctrl), 256);
    L.part = o; o = align_up(o + part_scratch_bytes(NBIN, n), 256);
    L.total = o;
    return L;
}

static int occupancy() {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<false>, BLOCK, 0) != cudaSuccess)
        return 0;
    return per_sm;
}

}  // namespace solve
}  // namespace hcb

using namespace hcb;
using namespace hcb::solve;

extern "C" {

int hc_device_info(int *h_num_sms, int *h_ctas_per_sm) {
    if (h_num_sms) *h_num_sms = num_sms();
    if (h_ctas_per_sm) *h_ctas_per_sm = occupancy();
    return HC_OK;
}

size_t hc_solve_workspace_bytes(int64_t num_nodes, int64_t num_edges) {
    (void)num_edges;
    return layout(num_nodes < 0 ? 0 : num_nodes).total;
}

int hc_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
             int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
             int64_t max_rec, int64_t *h_rounds, void *d_ws, size_t ws_bytes, void *stream) {
    return hc_solve_stats(d_row_offsets, d_col_indices, num_nodes, num_edges, mode, thr_count,
                          d_colors, d_rec, max_rec, h_rounds, nullptr, d_ws, ws_bytes, stream);
}

int hc_solve_stats(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                   int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors,
                   hc_round_rec *d_rec, int64_t max_rec, int64_t *h_rounds, int64_t *d_stats,
                   void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(num_nodes >= 0 && num_nodes < 0x7fffffffLL, HC_ERR_INVALID,
               "hc_solve: num_nodes %lld out of range", (long long)num_nodes);
    HC_REQUIRE(mode >= HC_MODE_DATA && mode <= HC_MODE_HYBRID, HC_ERR_INVALID,
               "hc_solve: mode %d invalid", mode);
    HC_REQUIRE(max_rec >= 0, HC_ERR_INVALID, "hc_solve: max_rec < 0");
    cudaStream_t st = as_stream(stream);
    if (h_rounds) *h_rounds = 0;
    if (num_nodes == 0) return HC_OK;  // empty graph: 0 rounds (test_driver.py:88-93)
    HC_REQUIRE(d_row_offsets && d_colors && (num_edges == 0 || d_col_indices), HC_ERR_INVALID,
               "hc_solve: null pointer");
    const Layout L = layout(num_nodes);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_solve: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P;
    P.ro = reinterpret_cast<const long long *>(d_row_offsets);
    P.ci = d_col_indices;
    P.n = num_nodes;
    P.X = reinterpret_cast<unsigned *>(ws + L.x);
    P.stat = reinterpret_cast<int *>(ws + L.stat);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NBIN; ++b) P.dyn[p][b] = reinterpret_cast<int *>(ws + L.dyn[p][b]);
    P.ctrl = reinterpret_cast<Ctrl *>(ws + L.ctrl);
    P.rec = d_rec;
    P.max_rec = d_rec ? max_rec : 0;
    P.colors_out = reinterpret_cast<long long *>(d_colors);
    P.mode = mode;
    P.thr = thr_count;
    P.stats = reinterpret_cast<long long *>(d_stats);
    if (d_stats && P.max_rec)
        HC_CUDA_TRY(cudaMemsetAsync(d_stats, 0, sizeof(int64_t) * 2 * (size_t)P.max_rec, st));

    HC_CUDA_TRY(cudaMemsetAsync(P.ctrl, 0, offsetof(Ctrl, segcnt), st));
    unsigned long long *totals = nullptr;
    int rc = ordered_partition<NBIN>(num_nodes, DegreeBin{P.ro}, EmitI32{}, P.stat, ws + L.part,
                                     &totals, st);
    if (rc != HC_OK) return rc;
    copy_totals_kernel<<<1, 32, 0, st>>>(totals, P.ctrl);
    HC_CHECK_LAUNCH();

    const int per_sm = occupancy();
    const int sms = num_sms();
    HC_REQUIRE(per_sm > 0 && sms > 0, HC_ERR_CUDA, "hc_solve: occupancy query failed");
    P.nblocks = (unsigned)(per_sm * sms);
    void *args[] = {&P};
    const void *fn = d_stats ? (const void *)solve_kernel<true> : (const void *)solve_kernel<false>;
    HC_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(P.nblocks), dim3(BLOCK), args, 0, st));
    long long info[2];
    HC_CUDA_TRY(cudaMemcpyAsync(info, &P.ctrl->rounds, sizeof info, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    if (h_rounds) *h_rounds = info[0];
    HC_REQUIRE(!info[1], HC_ERR_RECORDS, "hc_solve: %lld rounds exceed the %lld-record buffer",
               info[0], (long long)max_rec);
    return HC_OK;
}

}  // extern "C"
