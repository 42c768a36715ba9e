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
// nodes are binned once by degree -- small (thread per node, NPT nodes per
// thread with all their loads batched for memory-level parallelism), mid
// (warp per node; CTA per node in rounds with few active mid nodes, where
// latency rather than throughput decides), hub (CTA per node).  The
// always-maintained worklist is kept per bin and double buffered.  Each phase
// hands out units with ONE atomic per unit: hub nodes first (largest work
// first), then chunks of mid nodes, then chunks of small nodes.  Losers of
// chunk c are compacted (order-preserving for the small bin) into output
// segment c of the next worklist and the chunk writes its loser count; the
// next round rebuilds the segment prefix in shared memory.  So pushes need no
// global atomics, the worklist stays sorted by id (segments are in chunk
// order), and topology-driven rounds (static bin lists + activity test) and
// data-driven rounds (segmented dynamic lists) share the same code.
//
// Row offsets are read as int32 when num_edges < 2^31 (a copy made in the
// preprocessing), halving the offset traffic; int64 otherwise.
#include <algorithm>

#include "hcb_partition.cuh"

namespace hcb {
namespace solve {

constexpr int BLOCK = 1024;
constexpr int NW = BLOCK / 32;
constexpr int NPT = 4;                   // small nodes per thread per tile
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
    const void *ro;            // int32 or int64 row offsets (template OffT)
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

// A bin's current list: dense (static list / round 1) or segmented (the
// previous round's output: nseg segments of capacity segcap).
struct List {
    const int *base;
    unsigned long long total;
    unsigned nseg, segcap;
    bool segmented;
};

// per-round, CTA-uniform configuration kept in shared memory (registers are
// the scarce resource at 1024 threads per SM)
struct RoundCfg {
    List L[NBIN];
    const int *stat_lists[NBIN];
    unsigned long long nst[NBIN];
    unsigned csz0, csz1, nch0, nch1, n_hub, units;
    unsigned prev_nseg[2], prev_cap[2];
    bool topo, ident, mid_by_cta, ident_small;
};

struct Smem {
    RoundCfg rc;
    unsigned prefix[2][MAXSEG + 1];   // segment prefix of the current small / mid lists
    unsigned mid_bm[NW][MID_WORDS];
    unsigned hub_bm[HUB_WORDS];
    unsigned warp_tmp[NPT * NW];
    unsigned long long red;
    int hub_first;
    unsigned unit;
    unsigned out_cnt;
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

__device__ __forceinline__ void mark(unsigned *bm, unsigned c) {
    atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
}

// ------------------------------------------------------------------ mid (warp)
template <typename OffT>
__device__ __forceinline__ unsigned assign_mid(const Params &P, const OffT *ro, int u, unsigned *bm,
                                               unsigned &deg_out) {
    const unsigned lane = lane_id();
    const long long b = ro[u], e = ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;  // mex <= deg+1 (_kernels.pyx:49)
    deg_out = lim - 1u;
#pragma unroll
    for (int w = 0; w < MID_WORDS / 32; ++w) bm[lane + 32 * w] = 0u;
    __syncwarp();
    for (long long k = b + lane; k < e; k += 128) {
        int v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (k + 32 * q < e) ? P.ci[k + 32 * q] : -1;
        unsigned x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = v[q] >= 0 ? P.X[v[q]] : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const unsigned c = x[q] & CMASK;
            if ((x[q] & FBIT) && c <= lim) mark(bm, c);
        }
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

template <typename OffT>
__device__ __forceinline__ unsigned resolve_mid(const Params &P, const OffT *ro, int u, unsigned T,
                                                unsigned &lower_out) {
    const unsigned lane = lane_id();
    const long long b = ro[u], e = ro[u + 1];
    unsigned cnt = 0, low = 0;
    for (long long k0 = b; k0 < e; k0 += 128) {
        int v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long k = k0 + 32 * q + lane;
            v[q] = k < e ? P.ci[k] : 0x7fffffff;
        }
        unsigned x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = v[q] < u ? P.X[v[q]] : 0u;
        bool stop = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (v[q] < u) { cnt += (x[q] & CMASK) == T; ++low; }
            else stop = true;
        }
        if (__any_sync(FULL, stop)) break;  // adjacency sorted: the rest is >= u
    }
    lower_out = warp_sum(low);
    return warp_sum(cnt);
}

// ------------------------------------------------------------------ hub (CTA)
template <typename OffT>
__device__ unsigned assign_hub(const Params &P, const OffT *ro, int u, Smem &sm) {
    const long long b = ro[u], e = ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;
    for (unsigned w0 = 0;; w0 += HUB_WORDS * 32) {
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK) sm.hub_bm[i] = 0u;
        if (threadIdx.x == 0) sm.hub_first = 0x7fffffff;
        __syncthreads();
        const unsigned hi = min(lim, w0 + HUB_WORDS * 32);
        for (long long k = b + threadIdx.x; k < e; k += 4 * BLOCK) {
            int v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = (k + q * BLOCK < e) ? P.ci[k + q * BLOCK] : -1;
            unsigned x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = v[q] >= 0 ? P.X[v[q]] : 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned c = x[q] & CMASK;
                if ((x[q] & FBIT) && c > w0 && c <= hi) mark(sm.hub_bm, c - w0);
            }
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

template <typename OffT>
__device__ unsigned resolve_hub(const Params &P, const OffT *ro, int u, unsigned T, Smem &sm,
                                unsigned &lower_out) {
    const long long b = ro[u], e = ro[u + 1];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    if (threadIdx.x == 0) sm.red = 0;
    __syncthreads();
    unsigned cnt = 0, low = 0;
    for (long long k0 = b + (long long)warp * 128; k0 < e; k0 += 128LL * NW) {
        int v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long k = k0 + 32 * q + lane;
            v[q] = k < e ? P.ci[k] : 0x7fffffff;
        }
        unsigned x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = v[q] < u ? P.X[v[q]] : 0u;
        bool stop = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (v[q] < u) { cnt += (x[q] & CMASK) == T; ++low; }
            else stop = true;
        }
        if (__any_sync(FULL, stop)) break;  // later chunks are all >= u
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

// ------------------------------------------------------------------ small
// Thread per node, NPT nodes per thread; all list / offset / first-four-
// neighbour loads of the NPT nodes are issued before any is consumed.
// Returns the loser flags (resolve) through `lost`.
template <typename OffT, bool STATS, int PHASE>
__device__ __forceinline__ void small_tile(const Params &P, const OffT *ro, const RoundCfg &rc,
                                           const unsigned *prefix, unsigned long long base,
                                           unsigned long long hi, int u[NPT], bool lost[NPT],
                                           unsigned long long &my_conf, unsigned long long *my_edges) {
    const List &L = rc.L[BIN_SMALL];
    const bool topo = rc.topo, ident = rc.ident;
    unsigned xu[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
        u[j] = v < hi ? (ident ? (int)v : L.base[list_index(L, prefix, v)]) : -1;
        lost[j] = false;
        xu[j] = 0u;
    }
    if (topo || PHASE == 1) {
#pragma unroll
        for (int j = 0; j < NPT; ++j) xu[j] = u[j] >= 0 ? P.X[u[j]] : 0u;
        if (topo) {
#pragma unroll
            for (int j = 0; j < NPT; ++j)
                if (xu[j] & FBIT) u[j] = -1;  // inactive (_kernels.pyx:76-77, 135-136)
        }
    }
    OffT rb[NPT], re[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        rb[j] = u[j] >= 0 ? ro[u[j]] : OffT(0);
        re[j] = u[j] >= 0 ? ro[u[j] + 1] : OffT(0);
    }
    int nb[NPT][4];
#pragma unroll
    for (int j = 0; j < NPT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) nb[j][q] = rb[j] + q < re[j] ? P.ci[rb[j] + q] : -1;
    if (PHASE == 0) {
        unsigned x[NPT][4];
#pragma unroll
        for (int j = 0; j < NPT; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) x[j][q] = nb[j][q] >= 0 ? P.X[nb[j][q]] : 0u;
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            if (u[j] < 0) continue;
            unsigned long long mask = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned cc = x[j][q] & CMASK;
                if ((x[j][q] & FBIT) && cc <= 64u) mask |= 1ull << (cc - 1u);
            }
            for (OffT k = rb[j] + 4; k < re[j]; k += 4) {  // deg 5..16
                int v2[4];
                unsigned x2[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? P.ci[k + q] : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) x2[q] = v2[q] >= 0 ? P.X[v2[q]] : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned cc = x2[q] & CMASK;
                    if ((x2[q] & FBIT) && cc <= 64u) mask |= 1ull << (cc - 1u);
                }
            }
            P.X[u[j]] = (unsigned)__ffsll((long long)~mask);  // deg <= 16: a zero bit exists
            if (STATS) my_edges[0] += re[j] - rb[j];
        }
    } else {
        unsigned x[NPT][4];
#pragma unroll
        for (int j = 0; j < NPT; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) x[j][q] = (nb[j][q] >= 0 && nb[j][q] < u[j]) ? P.X[nb[j][q]] : 0u;
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
            if (u[j] < 0) continue;
            const unsigned T = xu[j];
            unsigned cnt = 0, low = 0;
            bool stop = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (nb[j][q] >= 0 && nb[j][q] < u[j]) { cnt += (x[j][q] & CMASK) == T; ++low; }
                else stop = true;
            }
            for (OffT k = rb[j] + 4; !stop && k < re[j]; k += 4) {
                int v2[4];
                unsigned x2[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? P.ci[k + q] : 0x7fffffff;
#pragma unroll
                for (int q = 0; q < 4; ++q) x2[q] = v2[q] < u[j] ? P.X[v2[q]] : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (v2[q] < u[j]) { cnt += (x2[q] & CMASK) == T; ++low; }
                    else stop = true;  // adjacency sorted ascending (graph.py:193-197)
                }
            }
            my_conf += cnt;
            if (STATS) my_edges[1] += low;
            lost[j] = cnt != 0;
            if (!lost[j]) P.X[u[j]] = T | FBIT;
        }
    }
}

// Ordered compaction of a tile's losers (index order base + j*BLOCK + tid,
// i.e. j-major then thread) into out[written ...]; returns the tile's count.
__device__ __forceinline__ unsigned compact_tile(const int u[NPT], const bool lost[NPT], int *out,
                                                 unsigned written, Smem &sm) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned bal[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) bal[j] = __ballot_sync(FULL, lost[j]);
    if (lane < NPT) {
        unsigned mine = 0;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (lane == (unsigned)j) mine = __popc(bal[j]);
        sm.warp_tmp[lane * NW + warp] = mine;
    }
    __syncthreads();
    if (warp == 0) {  // scan NPT*NW = 128 counts, 4 per lane
        unsigned a[4], sum = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) { a[q] = sm.warp_tmp[4 * lane + q]; sum += a[q]; }
        const unsigned incl = warp_incl_scan(sum);
        unsigned run = incl - sum;
#pragma unroll
        for (int q = 0; q < 4; ++q) { sm.warp_tmp[4 * lane + q] = run; run += a[q]; }
        if (lane == 31) sm.out_cnt = incl;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NPT; ++j)
        if (lost[j]) out[written + sm.warp_tmp[j * NW + warp] + __popc(bal[j] & lanemask_lt())] = u[j];
    const unsigned tot = sm.out_cnt;
    __syncthreads();
    return tot;
}

// One unit of one phase.  All CTA-uniform inputs come from shared memory.
template <typename OffT, bool STATS, int PHASE>
__device__ __forceinline__ void run_unit(const Params &P, const OffT *ro, Smem &sm, unsigned unit,
                                         int p, unsigned long long &my_conf,
                                         unsigned long long *my_edges) {
    const RoundCfg &rc = sm.rc;
    const int np = p ^ 1;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned n_hub = rc.n_hub, nch1 = rc.nch1;
    const bool cta_unit = unit < n_hub || (rc.mid_by_cta && unit < n_hub + nch1);
    if (cta_unit) {
        // ---- hub (or mid node in the latency regime): one CTA per node
        const bool is_hub = unit < n_hub;
        const unsigned c = unit - n_hub;
        const int u = is_hub ? rc.L[BIN_HUB].base[unit] : rc.L[BIN_MID].base[list_index(rc.L[BIN_MID], sm.prefix[1], c)];
        const unsigned xu = P.X[u];
        unsigned pushed = 0;
        if (!(rc.topo && (xu & FBIT))) {  // topology sweep: inactive (_kernels.pyx:76)
            if (PHASE == 0) {
                const unsigned T = assign_hub(P, ro, u, sm);
                if (threadIdx.x == 0) {
                    P.X[u] = T;
                    if (STATS) my_edges[0] += ro[u + 1] - ro[u];
                }
            } else {
                unsigned low;
                const unsigned k = resolve_hub(P, ro, u, xu, sm, low);
                if (threadIdx.x == 0) {
                    my_conf += k;
                    if (STATS) my_edges[1] += low;
                    if (k) {
                        if (is_hub) P.dyn[np][BIN_HUB][atomicAdd(&P.ctrl->hub_cnt[np], 1ull)] = u;
                        else P.dyn[np][BIN_MID][c] = u;  // segment c, capacity 1
                        pushed = 1;
                    } else {
                        P.X[u] = xu | FBIT;
                    }
                }
            }
        }
        if (!is_hub && PHASE == 1 && threadIdx.x == 0) P.ctrl->segcnt[np][1][c] = pushed;
    } else if (unit < n_hub + nch1) {
        // ---- mid chunk: one warp per node
        const unsigned c = unit - n_hub;
        const unsigned csz1 = rc.csz1;
        const unsigned long long lo = (unsigned long long)c * csz1;
        const unsigned long long hi = min(lo + csz1, rc.L[BIN_MID].total);
        int *out = P.dyn[np][BIN_MID] + (long long)c * csz1;
        if (threadIdx.x == 0) sm.out_cnt = 0;
        __syncthreads();
        for (unsigned long long v = lo + warp; v < hi; v += NW) {
            const int u = rc.L[BIN_MID].base[list_index(rc.L[BIN_MID], sm.prefix[1], v)];
            const unsigned xu = P.X[u];
            if (rc.topo && (xu & FBIT)) continue;
            if (PHASE == 0) {
                unsigned deg;
                const unsigned T = assign_mid(P, ro, u, sm.mid_bm[warp], deg);
                if (lane == 0) {
                    P.X[u] = T;
                    if (STATS) my_edges[0] += deg;
                }
            } else {
                unsigned low;
                const unsigned k = resolve_mid(P, ro, u, xu, low);
                if (lane == 0) {
                    my_conf += k;
                    if (STATS) my_edges[1] += low;
                    if (k) out[atomicAdd(&sm.out_cnt, 1u)] = u;
                    else P.X[u] = xu | FBIT;
                }
            }
        }
        __syncthreads();
        if (PHASE == 1 && threadIdx.x == 0) P.ctrl->segcnt[np][1][c] = sm.out_cnt;
    } else {
        // ---- small chunk
        const unsigned c = unit - n_hub - nch1;
        const unsigned csz0 = rc.csz0;
        const unsigned long long lo = (unsigned long long)c * csz0;
        const unsigned long long hi = min(lo + csz0, rc.L[BIN_SMALL].total);
        int *out = P.dyn[np][BIN_SMALL] + (long long)c * csz0;
        unsigned written = 0;
        for (unsigned long long base = lo; base < hi; base += (unsigned long long)BLOCK * NPT) {
            int u[NPT];
            bool lost[NPT];
            small_tile<OffT, STATS, PHASE>(P, ro, rc, sm.prefix[0], base, hi, u, lost, my_conf, my_edges);
            if (PHASE == 1) written += compact_tile(u, lost, out, written, sm);
        }
        if (PHASE == 1 && threadIdx.x == 0) P.ctrl->segcnt[np][0][c] = written;
    }
}

template <typename OffT, bool STATS, int PHASE>
__device__ __forceinline__ void run_phase(const Params &P, const OffT *ro, Smem &sm, int p,
                                          unsigned long long &my_conf, unsigned long long *my_edges) {
    unsigned *ctr = &P.ctrl->unit_ctr[PHASE][p];
    if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);
    __syncthreads();
    unsigned unit = sm.unit;
    __syncthreads();
    while (unit < sm.rc.units) {
        if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);  // prefetch the next unit
        run_unit<OffT, STATS, PHASE>(P, ro, sm, unit, p, my_conf, my_edges);
        __syncthreads();
        unit = sm.unit;
        __syncthreads();
    }
}

// ------------------------------------------------------------------ kernel
template <typename OffT, bool STATS>
__global__ void __launch_bounds__(BLOCK, 1) solve_kernel(Params P) {
    __shared__ Smem sm;
    Ctrl *C = P.ctrl;
    const OffT *ro = reinterpret_cast<const OffT *>(P.ro);
    const unsigned lane = lane_id();
    const unsigned warp = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long gthreads = (long long)P.nblocks * BLOCK;
    RoundCfg &rc = sm.rc;

    for (long long u = gtid; u < P.n; u += gthreads) P.X[u] = 0u;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBIN; ++b) rc.nst[b] = C->nstat[b];
        rc.stat_lists[0] = P.stat;
        rc.stat_lists[1] = P.stat + rc.nst[0];
        rc.stat_lists[2] = P.stat + rc.nst[0] + rc.nst[1];
        rc.ident_small = rc.nst[0] == (unsigned long long)P.n;  // all nodes small: sweep ids
        rc.prev_nseg[0] = rc.prev_nseg[1] = rc.prev_cap[0] = rc.prev_cap[1] = 0;
    }
    grid_sync(&C->bar, P.nblocks);

    unsigned long long t_start = 0;  // block 0 / thread 0 record keeping
    long long wl_in_prev = 0;
    int topo_prev = 0;
    unsigned long long my_conf = 0;
    unsigned long long my_edges[2] = {0, 0};  // stats: assign edges, resolve lower edges
    long long t = 1;
    for (;; ++t) {
        const int p = (int)(t & 1), np = p ^ 1;
        // ---- current worklist sizes: rebuild the segment prefix of the
        //      previous round's output (round 1: the full static lists)
        if (t > 1) {
#pragma unroll 1
            for (int b = 0; b < 2; ++b) {
                const unsigned ns = rc.prev_nseg[b];
                for (unsigned s = threadIdx.x; s < ns; s += BLOCK)
                    sm.prefix[b][s + 1] = __ldcg(&C->segcnt[p][b][s]);
                if (threadIdx.x == 0) sm.prefix[b][0] = 0;
                __syncthreads();
                // inclusive scan of prefix[1..ns] (ns <= MAXSEG = 2*BLOCK)
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
        }
        if (threadIdx.x == 0) {
            for (int b = 0; b < 2; ++b)
                rc.L[b] = t == 1 ? List{rc.stat_lists[b], rc.nst[b], 0, 0, false}
                                 : List{P.dyn[p][b], sm.prefix[b][rc.prev_nseg[b]], rc.prev_nseg[b],
                                        rc.prev_cap[b], true};
            const unsigned long long hub_total = t == 1 ? rc.nst[BIN_HUB] : ld_relaxed_u64(&C->hub_cnt[p]);
            rc.L[BIN_HUB] = List{t == 1 ? rc.stat_lists[BIN_HUB] : P.dyn[p][BIN_HUB], hub_total, 0, 0, false};
            const unsigned long long s = rc.L[0].total + rc.L[1].total + rc.L[2].total;
            const bool topo = P.mode == HC_MODE_TOPO || (P.mode == HC_MODE_HYBRID && (long long)s > P.thr);
            // mid nodes at CTA granularity when few are active (latency regime)
            const bool mid_cta = rc.L[1].total <= 2ull * P.nblocks;
            if (topo)  // topology-driven: sweep the static lists, activity test
                for (int b = 0; b < NBIN; ++b) rc.L[b] = List{rc.stat_lists[b], rc.nst[b], 0, 0, false};
            rc.topo = topo;
            rc.ident = topo && rc.ident_small;
            rc.csz0 = chunk_size(rc.L[0].total, BLOCK * NPT);
            rc.csz1 = (mid_cta && rc.L[1].total <= MAXSEG) ? 1u : chunk_size(rc.L[1].total, NW);
            rc.nch0 = (unsigned)((rc.L[0].total + rc.csz0 - 1) / rc.csz0);
            rc.nch1 = (unsigned)((rc.L[1].total + rc.csz1 - 1) / rc.csz1);
            rc.mid_by_cta = rc.csz1 == 1u;
            rc.n_hub = (unsigned)rc.L[BIN_HUB].total;
            rc.units = s == 0 ? 0u : rc.n_hub + rc.nch1 + rc.nch0;
            sm.red = s;  // broadcast |W_t|
            if (blockIdx.x == 0) {
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
        }
        __syncthreads();
        const unsigned long long s = sm.red;
        __syncthreads();
        if (s == 0) break;  // worklist drained (driver.py:145)

        run_phase<OffT, STATS, 0>(P, ro, sm, p, my_conf, my_edges);
        grid_sync(&C->bar, P.nblocks);
        run_phase<OffT, STATS, 1>(P, ro, sm, p, my_conf, my_edges);

        // conflicts of this round: block reduce then one atomic per CTA
        {
            unsigned long long v = warp_sum(my_conf);
            my_conf = 0;
            if (threadIdx.x == 0) sm.red = 0;
            __syncthreads();
            if (lane == 0 && v) atomicAdd(&sm.red, v);
            __syncthreads();
            if (threadIdx.x == 0 && sm.red) atomicAdd(&C->conflicts[p], sm.red);
            if (STATS) {
                for (int q = 0; q < 2; ++q) {
                    const unsigned long long e = warp_sum(my_edges[q]);
                    my_edges[q] = 0;
                    if (lane == 0 && e && t <= P.max_rec)
                        atomicAdd((unsigned long long *)&P.stats[2 * (t - 1) + q], e);
                }
            }
        }
        if (threadIdx.x == 0) {
            rc.prev_nseg[0] = rc.nch0; rc.prev_nseg[1] = rc.nch1;
            rc.prev_cap[0] = rc.csz0; rc.prev_cap[1] = rc.csz1;
        }
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

__global__ void narrow_offsets_kernel(const long long *ro, int *ro32, long long count) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        ro32[i] = (int)ro[i];
}

// worst-case segmented capacity of a bin with `cnt` static nodes
inline size_t seg_capacity(long long cnt) {
    return (size_t)cnt + (size_t)cnt / MAXSEG + 2 * BLOCK * NPT;
}

struct Layout {
    size_t x, stat, dyn[2][NBIN], ro32, ctrl, part, total;
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
    L.ro32 = o; o = align_up(o + 4 * (size_t)(n + 1), 256);
    L.ctrl = o; o = align_up(o + sizeof(Ctrl), 256);
    L.part = o; o = align_up(o + part_scratch_bytes(NBIN, n), 256);
    L.total = o;
    return L;
}

template <typename OffT, bool STATS>
static const void *kernel_ptr() {
    return (const void *)solve_kernel<OffT, STATS>;
}

static int occupancy() {
    int per_sm = 0, per_sm64 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<int, false>, BLOCK, 0) != cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm64, solve_kernel<long long, false>, BLOCK, 0) !=
        cudaSuccess)
        return 0;
    return std::min(per_sm, per_sm64);
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
    HC_REQUIRE(num_edges >= 0, HC_ERR_INVALID, "hc_solve: num_edges < 0");
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
    const bool narrow = num_edges < 0x7fffffffLL;
    Params P;
    P.ro = narrow ? (const void *)(ws + L.ro32) : (const void *)d_row_offsets;
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
    const long long *ro64 = reinterpret_cast<const long long *>(d_row_offsets);
    int rc = ordered_partition<NBIN>(num_nodes, DegreeBin{ro64}, EmitI32{}, P.stat, ws + L.part,
                                     &totals, st);
    if (rc != HC_OK) return rc;
    copy_totals_kernel<<<1, 32, 0, st>>>(totals, P.ctrl);
    HC_CHECK_LAUNCH();
    if (narrow) {
        const int sms = std::max(1, num_sms());
        narrow_offsets_kernel<<<sms * 4, 256, 0, st>>>(ro64, reinterpret_cast<int *>(ws + L.ro32),
                                                       num_nodes + 1);
        HC_CHECK_LAUNCH();
    }

    const int per_sm = occupancy();
    const int sms = num_sms();
    HC_REQUIRE(per_sm > 0 && sms > 0, HC_ERR_CUDA, "hc_solve: occupancy query failed");
    P.nblocks = (unsigned)(per_sm * sms);
    void *args[] = {&P};
    const void *fn = narrow ? (d_stats ? kernel_ptr<int, true>() : kernel_ptr<int, false>())
                            : (d_stats ? kernel_ptr<long long, true>() : kernel_ptr<long long, false>());
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
